/*
 * silt_cuda.h — C ABI of the B200-native time-stepping path for the coupled
 * shallow-water + Exner (Grass or Shields-threshold bedload) relaxation solver
 * of arXiv 1307.0491.
 *
 * This is the drop-in boundary.  Every entry point takes plain pointers and
 * sizes; nothing here mentions torch, std::vector or CUDA types (streams are
 * passed as `void*` holding a cudaStream_t).  Each function returns a status
 * code (SILT_OK == 0); the message of the last failure on the calling thread
 * is available from silt_last_error().  The C++ shim
 * (paper_1307_0491_b200/csrc/silt_gpu.hpp) maps the codes back onto the
 * reference's exception types.
 *
 * Reference interfaces replaced (paths relative to the reference checkout
 * proj/core/):
 *   silt_problem / silt_bc ......... Grid, Physics, BedloadLaw, BoundarySpec,
 *                                    Scenario (include/silt/grid.hpp:12-27,
 *                                    physics.hpp:7-11, bedload.hpp:32-52,
 *                                    scenarios.hpp:24-49)
 *   silt_solver_create/upload ...... PaddedField::from_field, partition
 *                                    (src/stepper.cpp:13-18, src/parallel.cpp:150-177)
 *   silt_solver_begin .............. run_serial/run_parallel prologue + first
 *                                    cfl_dt (src/parallel.cpp:208-222, 261-316;
 *                                    src/stepper.cpp:38-58)
 *   silt_solver_step ............... one loop trip of run_serial/run_parallel:
 *                                    apply_bcs + cfl_dt + clip + step_2d/step_1d
 *                                    (src/parallel.cpp:221-250, 315-364;
 *                                    src/stepper.cpp:118-189; src/scenarios.cpp:78-144)
 *   silt_solver_reduce_slot /
 *   silt_solver_exchange_ptrs ...... global_dt + halo_exchange/pull_halo
 *                                    (src/parallel.cpp:43-99, 192-206)
 *   silt_solver_download ........... PaddedField::interior, gather
 *                                    (src/stepper.cpp:20-25, src/parallel.cpp:179-190)
 *   silt_solver_capture_resume ..... on_snapshot(t, gather(...)) at a landed
 *                                    snapshot time, asynchronously
 *                                    (src/parallel.cpp:333-342)
 *   silt_run ....................... run_serial (src/parallel.cpp:208-259)
 *   silt_cfl_dt .................... cfl_dt (include/silt/stepper.hpp:38-41)
 *   silt_step_padded ............... step_1d / step_2d on a halo-complete
 *                                    PaddedField (include/silt/stepper.hpp:47-54)
 *   silt_riemann_batch ............. equilibrate + celerity_bounds +
 *                                    interface_riemann (relax_state.hpp:27-51,
 *                                    riemann.hpp:33-35)
 *   silt_write_snapshot / _to_string write_snapshot / snapshot_to_string
 *                                    (src/snapshot.cpp:50-93), on the device
 *   silt_law_batch ................. normal_flux + normal_flux_derivative
 *                                    (include/silt/bedload.hpp:95-98)
 */
#ifndef SILT_CUDA_H
#define SILT_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SILT_ABI_VERSION 2

/* Status codes.  INVALID ~ std::invalid_argument, RUNTIME ~ std::runtime_error
 * in the reference (SURVEY §8b "Errors"). */
enum {
    SILT_OK = 0,
    SILT_ERR_INVALID = 1,
    SILT_ERR_RUNTIME = 2,
    SILT_ERR_CUDA = 3,
    SILT_ERR_UNSUPPORTED = 4
};

/* BcType, in the reference's enum order (include/silt/scenarios.hpp:17-22),
 * plus GIVEN: ghosts supplied by the caller (halo-complete PaddedField). */
enum {
    SILT_BC_INFLOW = 0,
    SILT_BC_OUTFLOW = 1,
    SILT_BC_WALL = 2,
    SILT_BC_PERIODIC = 3,
    SILT_BC_GIVEN = 4
};

/* BedloadLaw::Kind (include/silt/bedload.hpp:33). */
enum { SILT_LAW_GRASS = 0, SILT_LAW_SHIELDS = 1 };

/* ShieldsFormula, in the reference's enum order (include/silt/bedload.hpp:12-18). */
enum {
    SILT_SHIELDS_MPM = 0,       /* MeyerPeterMuller */
    SILT_SHIELDS_FLVB = 1,      /* FernandezLuqueVanBeek */
    SILT_SHIELDS_NIELSEN = 2,   /* Nielsen */
    SILT_SHIELDS_RIBBERINK = 3, /* Ribberink */
    SILT_SHIELDS_CAMENEN = 4    /* CamenenLarson */
};

/* FrictionModel (include/silt/bedload.hpp:20-23). */
enum { SILT_FRICTION_DARCY_WEISBACH = 0, SILT_FRICTION_MANNING = 1 };

/* Side order of Scenario::bc (include/silt/scenarios.hpp:15). */
enum { SILT_WEST = 0, SILT_EAST = 1, SILT_SOUTH = 2, SILT_NORTH = 3 };

/* Numerical variant of the kernels. FAST: contracted FMAs, reciprocals,
 * closed-form Grass terms; parity to 1e-9 normwise.  STRICT: the reference's
 * operation order, no FMA contraction, IEEE division and glibc's hypot
 * algorithm (bitwise-identical to the CPU reference for the Grass law and for
 * the Shields laws that need only sqrt: Darcy-Weisbach friction with MPM,
 * FLVB or Nielsen; Manning friction and the Ribberink / Camenen formulas call
 * pow/exp, where CUDA's libm may differ from glibc's by an ulp or two). */
enum { SILT_VARIANT_FAST = 0, SILT_VARIANT_STRICT = 1 };

/* Run state reported by silt_solver_status. */
enum {
    SILT_STATE_RUNNING = 0,  /* more steps would advance the run */
    SILT_STATE_DONE = 1,     /* t >= t_end or steps >= max_steps */
    SILT_STATE_PAUSED = 2,   /* landed on a snapshot time; call silt_solver_resume */
    SILT_STATE_FAILED = 3    /* a step raised an error (see error_code) */
};

typedef struct silt_bc {
    int32_t type;          /* SILT_BC_* */
    int32_t supercritical; /* Inflow: impose h0 as well */
    double q0;             /* Inflow: imposed normal discharge */
    double h0;             /* Inflow (supercritical): imposed depth */
} silt_bc;

/* One configured problem: grid + physics + bedload law + BCs + run knobs.
 * The law fields mirror BedloadLaw (include/silt/bedload.hpp:32-52) and are
 * validated like BedloadLaw::grass / BedloadLaw::shields (src/bedload.cpp:26-57). */
typedef struct silt_problem {
    int32_t dim;       /* 1 or 2 */
    int32_t nx, ny;    /* global cell counts (ny == 1 in 1D) */
    int32_t law_kind;  /* SILT_LAW_GRASS or SILT_LAW_SHIELDS */
    double dx, dy;     /* Grid::dx, Grid::dy (1D: dy = 1) */
    double gravity;    /* Physics::gravity */
    double h_dry;      /* Physics::h_dry */
    double a_g, m_g;   /* Grass: BedloadLaw::grass(a_g, m_g) */
    int32_t shields_formula; /* Shields: SILT_SHIELDS_* */
    int32_t friction_model;  /* Shields: SILT_FRICTION_* */
    double tau_cr;           /* Shields: critical Shields stress (>= 0) */
    double grain_diameter;   /* Shields: d_s (> 0) */
    double rel_density;      /* Shields: s (> 1) */
    double friction_coef;    /* Shields: Darcy f or Manning n (> 0) */
    double cfl;        /* Scenario::cfl, in (0, 1] */
    double safety;     /* Scenario::safety (>= 1) */
    silt_bc bc[4];     /* West, East, South, North */
} silt_problem;

/* Which rows of the global grid one solver owns (row strips, px = 1). */
typedef struct silt_strip {
    int32_t j0;              /* global index of local row 0 */
    int32_t ny_local;        /* rows owned */
    int32_t south_neighbor;  /* 1: ghost row -1 arrives from another strip */
    int32_t north_neighbor;  /* 1: ghost row ny_local arrives from another strip */
} silt_strip;

typedef struct silt_run_plan {
    double t_end;                 /* >= 0; +inf allowed */
    int64_t max_steps;            /* < 0: unlimited */
    const double* snapshot_times; /* host array, may be NULL */
    int32_t n_snapshots;
    int64_t dt_log_capacity;      /* device-side dt log length (0: none) */
} silt_run_plan;

typedef struct silt_status {
    double t;            /* simulated time reached */
    int64_t steps;       /* steps taken */
    int32_t state;       /* SILT_STATE_* */
    int32_t error_code;  /* SILT_OK or SILT_ERR_* when state == FAILED */
    double last_dt;      /* dt of the last step taken */
    int32_t snapshot_index; /* snapshots landed so far */
    int32_t pad_;
} silt_status;

/* Device pointers a multi-rank driver moves between strips after each step
 * (4 fields h,hu,hv,zb packed as [4][nx] doubles).  send_* are written by the
 * step kernel; recv_* are read by the next step.  NULL when the side has no
 * neighbour. */
typedef struct silt_exchange {
    double* send_south;
    double* send_north;
    double* recv_south;
    double* recv_north;
    int64_t row_doubles; /* 4 * nx */
} silt_exchange;

typedef struct silt_solver silt_solver;

int silt_abi_version(void);
/* sizeof of silt_bc, silt_problem, silt_strip, silt_run_plan, silt_status,
 * silt_exchange (in that order) into sizes[0..n); lets bindings verify their
 * mirrors without a GPU. */
int silt_abi_sizes(int64_t* sizes, int n);
const char* silt_last_error(void);
int silt_device_count(int* count);

/* ---- solver handle ------------------------------------------------------ */
int silt_solver_create(const silt_problem* problem, const silt_strip* strip,
                       int device, int variant, silt_solver** out);
int silt_solver_destroy(silt_solver* s);
int silt_solver_set_stream(silt_solver* s, void* cuda_stream);
/* AoS FlowState {h,hu,hv,zb} rows of this strip, ny_local * nx cells; host
 * pointer (pinned or pageable). */
int silt_solver_upload(silt_solver* s, const double* host_aos);
int silt_solver_download(silt_solver* s, double* host_aos);
/* Same with device pointers (AoS, nx*ny_local*4 doubles). */
int silt_solver_upload_device(silt_solver* s, const double* dev_aos);
int silt_solver_download_device(silt_solver* s, double* dev_aos);
/* Caller-supplied ghost cells (SILT_BC_GIVEN sides): AoS, west/east ny_local
 * cells, south/north nx cells; any pointer may be NULL. */
int silt_solver_set_ghosts(silt_solver* s, const double* west, const double* east,
                           const double* south, const double* north);
/* Reset the run clock to t = 0 and reduce state 0 (first cfl_dt). Async. */
int silt_solver_begin(silt_solver* s, const silt_run_plan* plan);
/* Enqueue n predicated steps (async; no host synchronisation). */
int silt_solver_step(silt_solver* s, int n);
/* One step with a caller-chosen dt (step_1d/step_2d semantics, no clipping). */
int silt_solver_step_fixed(silt_solver* s, double dt);
/* Synchronise and read the run state; returns the error of a failed step. */
int silt_solver_status(silt_solver* s, silt_status* st);
/* Continue after a snapshot pause. */
int silt_solver_resume(silt_solver* s);
/* Asynchronous snapshot gather: the on_snapshot + gather of a run
 * (src/parallel.cpp:333-342, 179-190) without holding the run.  For a PAUSED
 * solver: the state is copied on the device into a snapshot buffer, the
 * solver resumes, and the buffer streams to host_aos (nx * ny_local FlowState,
 * AoS) on a side stream while the following steps execute.  Use page-locked
 * host memory (silt_host_alloc) for the copy to overlap.  One capture is in
 * flight per solver; the next capture waits for it.  capture_wait blocks until
 * the last capture has landed; capture_query reports it without blocking. */
int silt_solver_capture_resume(silt_solver* s, double* host_aos);
int silt_solver_capture_wait(silt_solver* s);
int silt_solver_capture_query(silt_solver* s, int* landed);
/* write_snapshot of a paused solver without holding the run: the state is
 * copied on the device, the solver resumes, and a host thread formats the
 * copy on the device and writes `path` (header unless `append`) while the
 * next steps run.  silt_solver_capture_wait joins it and reports its error. */
int silt_solver_capture_write(silt_solver* s, double time, const char* path, int append);
/* Page-locked host memory (capture targets, fast uploads). */
int silt_host_alloc(int64_t bytes, void** out);
int silt_host_free(void* p);
/* dt of steps [0, n) from the device log (n <= capacity). */
int silt_solver_dt_log(silt_solver* s, double* host_out, int64_t n);
/* WorkerTiming.compute_seconds (include/silt/parallel.hpp:52-57; measured at
 * src/parallel.cpp:324-348): device seconds of this strip's step launches
 * since timing was last enabled (CUDA events around each launch, harvested
 * when the stream synchronises).  Synchronises; writes the current total to
 * *compute_seconds (may be NULL); enable = 1 / 0 switches timing on / off and
 * resets the total, enable < 0 only reads. */
int silt_solver_timing(silt_solver* s, int enable, double* compute_seconds);
/* Current cfl_dt of the uploaded state (synchronises). */
int silt_solver_cfl_dt(silt_solver* s, double* dt);
/* Multi-rank hooks. reduce_slot: device pointer to the {max_x, max_y} axis
 * speeds the NEXT step reads; a driver all-reduces it with MAX (per step, in
 * stream order) before enqueueing that step. */
int silt_solver_reduce_slot(silt_solver* s, double** dev_ptr);
int silt_solver_exchange_ptrs(silt_solver* s, silt_exchange* out);
/* Halo/compute overlap for multi-rank drivers: one step in two launches.
 * Part 1 runs the two boundary row blocks of the strip (they read the
 * received ghost rows and write the send rows), part 2 the interior blocks
 * and ends the step.  After part 1 (e.g. an event on the solver's stream) a
 * driver may move the edge rows to and from the neighbours while part 2
 * runs; the speed slot is complete after part 2.  *ok = 0 when the strip does
 * not split (1D, fewer than 3 row blocks, no neighbour, or a launch long
 * enough to use the dynamic row-block order): use silt_solver_step. */
int silt_solver_step_split_ok(silt_solver* s, int* ok);
int silt_solver_step_part(silt_solver* s, int part);
/* ---- multi-process strips over peer memory (CUDA IPC) ----------------------
 * The step exchange without a collective library: every rank exports its
 * exchange rows, Control block and step-flag array; after connect, the step
 * kernel stores the strip's edge rows straight into the neighbours' receive
 * rows (double-buffered by state parity), a one-warp kernel folds the strip's
 * axis-speed maxima into every rank's slot with remote atomics, and the
 * stream writes its step count into every rank's flag array; the next step
 * waits (a stream memory operation, no host synchronisation) until every
 * rank's count has arrived.  Replaces halo_exchange + global_dt
 * (src/parallel.cpp:43-99, 192-206) of run_parallel's loop.
 * Protocol: create the strip, export, all-gather the handles (any host
 * channel), connect; then per run: begin (its initial reduction already
 * stores the edge rows into the neighbours' memory), one MAX all-reduce of
 * the slot over the same channel (finishes global_dt and orders every rank's
 * initial kernels), and silt_solver_p2p_step on every rank with the same n. */
typedef struct silt_p2p_handle {
    char rows[64];   /* cudaIpcMemHandle_t of the exchange-row buffer */
    char ctl[64];    /* ... of the Control block */
    char flags[64];  /* ... of the step-flag array */
    int32_t nx;
    int32_t pad_;
} silt_p2p_handle;
int silt_solver_p2p_export(silt_solver* s, silt_p2p_handle* out);
int silt_solver_p2p_connect(silt_solver* s, int rank, int world, const silt_p2p_handle* all,
                            int south_rank, int north_rank);
int silt_solver_p2p_step(silt_solver* s, int n);
/* Number of kernel launches this handle has enqueued (for accounting). */
int silt_solver_launch_count(silt_solver* s, int64_t* count);

/* ---- in-process strip group: run_parallel(sc, 1, py) ---------------------
 * py row strips (block_range partition, src/parallel.cpp:25-30) in one
 * process, strip k on devices[k % n_devices].  Per step, with no host
 * synchronisation: the step kernels, ghost rows moved by device/peer copies
 * and the axis-speed maxima reduced on devices[0] (stream events order the
 * cross-device traffic).  Replaces run_parallel (src/parallel.cpp:261-386). */
typedef struct silt_group silt_group;
int silt_group_create(const silt_problem* problem, int py, const int* devices, int n_devices,
                      int variant, silt_group** out);
int silt_group_destroy(silt_group* g);
/* whole-grid AoS field (nx * ny cells) */
int silt_group_upload(silt_group* g, const double* host_aos);
int silt_group_download(silt_group* g, double* host_aos);
int silt_group_begin(silt_group* g, const silt_run_plan* plan);
int silt_group_step(silt_group* g, int n);
int silt_group_status(silt_group* g, silt_status* st);
int silt_group_resume(silt_group* g);
/* silt_solver_capture_resume / _wait over every strip (whole-grid host_aos) */
int silt_group_capture_resume(silt_group* g, double* host_aos);
int silt_group_capture_wait(silt_group* g);
int silt_group_dt_log(silt_group* g, double* host_out, int64_t n);
/* silt_solver_timing over the strips: per_strip[k] (py entries, may be NULL). */
int silt_group_timing(silt_group* g, int enable, double* per_strip);

/* ---- snapshot CSV, formatted on the device -------------------------------
 * write_snapshot / snapshot_to_string (src/snapshot.cpp:50-93; io.hpp:66-73):
 * header `x,h,u,zb,eta,time` (1D) or `x,y,h,u,v,zb,eta,time` (2D), one row
 * per cell, row-major, every number as snprintf("%.17g") prints it — the
 * bytes are identical to the reference's.  Rows are formatted by GPU kernels
 * (silt_csv.cu) in chunks and streamed through pinned memory to the sink.
 * `aos`: rows [j0, j0 + rows) of the problem's grid as FlowState AoS, in
 * host or device memory.  `append` != 0 appends without a header (strips
 * after the first). */
int silt_snapshot_to_string(const silt_problem* problem, const double* aos, int64_t j0,
                            int64_t rows, double time, int header, char* out, int64_t cap,
                            int64_t* len);
int silt_write_snapshot(const silt_problem* problem, const double* aos, int64_t j0,
                        int64_t rows, double time, const char* path, int append,
                        int64_t* bytes);
/* the solver's current state (its rows of the grid), straight from the device */
int silt_solver_write_snapshot(silt_solver* s, double time, const char* path, int append,
                               int64_t* bytes);
/* every strip in order: one file for the whole grid */
int silt_group_write_snapshot(silt_group* g, double time, const char* path, int64_t* bytes);

/* ---- one-shot conveniences (mirror the reference free functions) ---------- */
/* run_serial: whole run on one GPU; host AoS in/out; dt_log may be NULL. */
int silt_run(const silt_problem* problem, const double* init_aos,
             const silt_run_plan* plan, int variant, double* out_aos,
             double* dt_log, int64_t dt_log_capacity, silt_status* status);
/* cfl_dt over an interior field (AoS nx*ny). */
int silt_cfl_dt(const silt_problem* problem, const double* field_aos,
                int variant, double* dt);
/* step_1d/step_2d on a halo-complete padded field (AoS (nx+2)*(ny+2), ghost
 * frame included; 1D: 3 rows, the middle one used). In place. */
int silt_step_padded(const silt_problem* problem, double* padded_aos,
                     double dt, int variant);
/* Batch of interface solves: cells L[n][4], R[n][4] (FlowState h,hu,hv,zb),
 * axis 0 = X / 1 = Y.  out[n][5] = {F_h, F_hu_left, F_hu_right, F_hv, F_z}
 * (the reference FaceFlux, src/stepper.cpp:61-89). */
int silt_riemann_batch(const silt_problem* problem, const double* left,
                       const double* right, int64_t n, int axis, int variant,
                       double* out);

/* Batch of bedload-law evaluations as the step kernels make them: states[n][3]
 * = {h, u_n, u_t}; out[n][2] = {normal_flux(law, h, u_n, u_t, g),
 * normal_flux_derivative(law, h, u_n, u_t, g)} (src/bedload.cpp:207-223),
 * for either law kind.  Host arrays. */
int silt_law_batch(const silt_problem* problem, const double* states, int64_t n,
                   int variant, double* out);

/* Device math self-test (diagnostics): for k < n,
 *   out[4k+0] = FAST reciprocal of x[k]      out[4k+1] = IEEE 1/x[k]
 *   out[4k+2] = STRICT hypot(x[k], y[k])     out[4k+3] = FAST sqrt(x[k])
 * Host arrays. */
int silt_selftest_math(const double* x, const double* y, int64_t n, double* out);

#ifdef __cplusplus
}
#endif
#endif /* SILT_CUDA_H */
