// silt_kernels.cuh — the fused relaxation time step for sm_100a.
//
// Included by silt_fast.cu (S = false) and silt_strict.cu (S = true,
// compiled with -fmad=false).  See DESIGN.md §Kernels for the roofline.
//
// K1 step2d: one launch per time step.  Each warp owns a column strip of 30
// cells and marches up R rows.  Lane l holds column i0-1+l: lanes 1..30 own
// cells, lanes 0 and 31 are the x-halo.  Rows of state n arrive through a
// cp.async ring in shared memory (RING-1 rows in flight).  Per row:
//   per-cell relaxation terms for the x and y axes (computed once, shared by
//   both faces of the cell) -> y-face problem against the previous row (its
//   terms parked in shared memory) -> y update of the previous row ->
//   check_depth -> store state n+1 -> CFL/hmax candidates of state n+1 (the
//   NEXT step's cfl_dt) folded into registers -> x-face problem (right
//   neighbour's terms from shared memory) -> x update parked for the next row.
// Quiescent rows (FAST) are stored unchanged without any face solve, and a
// streak of them runs in a short inner loop (load, compare, vote, store).
// Every face is solved exactly once per launch: x faces by the lane left of
// them (the halo lanes 0 and 31 make each x face belong to exactly one warp),
// y faces by the owning column, so depth and bed updates telescope exactly.
//
// The run clock lives on the device (Control, triple-buffered per launch):
// every CTA derives dt_n from the previous launch's reduced axis speeds and
// the clipping rule of run_serial (src/parallel.cpp:221-237), so a batch of
// steps needs no host round trip.
#pragma once
#include <cooperative_groups.h>

#include "silt_layout.h"
#include "silt_physics.cuh"

namespace silt_dev {

__device__ __forceinline__ double shfl_down_d(double v, int d) {
    return __shfl_down_sync(0xffffffffu, v, d);
}
__device__ __forceinline__ double shfl_up_d(double v, int d) {
    return __shfl_up_sync(0xffffffffu, v, d);
}
__device__ __forceinline__ Side shfl_down_side(const Side& s) {
    Side o;
    o.h = shfl_down_d(s.h, 1);
    o.hun = shfl_down_d(s.hun, 1);
    o.pi = shfl_down_d(s.pi, 1);
    o.z = shfl_down_d(s.z, 1);
    o.omega = shfl_down_d(s.omega, 1);
    o.un = shfl_down_d(s.un, 1);
    o.ut = shfl_down_d(s.ut, 1);
    o.tau = shfl_down_d(s.tau, 1);
    o.a_side = shfl_down_d(s.a_side, 1);
    o.b2_side = shfl_down_d(s.b2_side, 1);
    const int packed = __shfl_down_sync(0xffffffffu, s.wet | (s.moving << 1), 1);
    o.wet = packed & 1;
    o.moving = (packed >> 1) & 1;
    return o;
}

// ---- control block --------------------------------------------------------
struct RunDecision {
    bool run;
    double dt, t_new;
    int next_state;
    int snap_idx;
    bool landed;
};

// Mirrors one trip of run_serial's loop head (src/parallel.cpp:221-237):
// loop condition, cfl_dt from the reduced speeds (src/stepper.cpp:38-58:
// min over cells of dx/s == dx / max s since RN division is monotone), clip
// to the next stop (next_stop, :129-132).
__device__ __forceinline__ RunDecision decide(const StepArgs& A, const Slot& cur) {
    const Control& C = *A.ctl;
    RunDecision d;
    d.run = false;
    d.dt = 0;
    d.t_new = cur.t;
    d.snap_idx = cur.snap_idx;
    d.landed = false;
    d.next_state = cur.state;
    if (cur.state != SILT_STATE_RUNNING) return d;
    if (cur.err) {
        d.next_state = SILT_STATE_FAILED;
        return d;
    }
    if (C.fixed_mode) {  // step_1d/step_2d(f, ..., dt): any dt, as given
        d.run = true;
        d.dt = C.fixed_dt;
        d.t_new = cur.t + d.dt;
        return d;
    }
    if (!(cur.t < C.t_end && (C.max_steps < 0 || cur.steps < C.max_steps))) {
        d.next_state = SILT_STATE_DONE;
        return d;
    }
    if (!cur.wet) {
        d.next_state = SILT_STATE_FAILED;
        return d;
    }
    const double sx = __longlong_as_double((long long)cur.max_sx);
    const double sy = __longlong_as_double((long long)cur.max_sy);
    double raw = A.dx / sx;
    if (A.dim == 2) raw = smin(raw, A.dy / sy);
    raw = A.cfl * raw;
    const double stop = (cur.snap_idx < C.n_snaps) ? smin(C.snaps[cur.snap_idx], C.t_end) : C.t_end;
    if (stop - cur.t <= raw) {
        d.dt = stop - cur.t;
        d.t_new = stop;
    } else {
        d.dt = raw;
        d.t_new = cur.t + d.dt;
    }
    d.run = true;
    if (cur.snap_idx < C.n_snaps && d.t_new == C.snaps[cur.snap_idx]) {
        d.landed = true;
        d.snap_idx = cur.snap_idx + 1;
        d.next_state = SILT_STATE_PAUSED;
    }
    return d;
}

// Block (0,0) thread 0: publish the next header, clear the slot after next.
__device__ __forceinline__ void control_epilogue(const StepArgs& A, int li, const Slot& cur,
                                                 const RunDecision& d) {
    Control& C = *A.ctl;
    Slot& nxt = C.slot[(li + 1) % 3];
    Slot& clr = C.slot[(li + 2) % 3];
    clr.max_sx = clr.max_sy = clr.hmax = 0ull;
    clr.wet = 0u;
    clr.err = 0u;
    C.item_ctr[(li + 2) % 3] = 0u;  // warp-item counter of launch li + 2
    if (d.run) {
        nxt.t = d.t_new;
        nxt.steps = cur.steps + 1;
        nxt.last_dt = d.dt;
        nxt.snap_idx = d.snap_idx;
        nxt.state = d.next_state;
        if (!C.fixed_mode && C.dt_log && cur.steps < C.dt_cap) C.dt_log[cur.steps] = d.dt;
    } else {
        nxt.t = cur.t;
        nxt.steps = cur.steps;
        nxt.last_dt = cur.last_dt;
        nxt.snap_idx = cur.snap_idx;
        nxt.state = d.next_state;
        nxt.max_sx = cur.max_sx;
        nxt.max_sy = cur.max_sy;
        nxt.hmax = cur.hmax;
        nxt.wet = cur.wet;
        nxt.err = cur.err | ((d.next_state == SILT_STATE_FAILED && !cur.err) ? kErrDry : 0u);
    }
}

__device__ __forceinline__ void record_error(const StepArgs& A, unsigned bit, int col, int row,
                                             const double* info6, Slot& nxt) {
    atomicOr(&nxt.err, bit);
    if (atomicCAS(&A.ctl->err_claim, 0u, 1u) == 0u) {
        A.ctl->err_bits = bit;
        A.ctl->err_col = col;
        A.ctl->err_row = row;
        for (int k = 0; k < 6; ++k) A.ctl->err_info[k] = info6 ? info6[k] : 0.0;
    }
}

// ---- cell access ----------------------------------------------------------
// Ghost value for a physical side (ghost_value, src/scenarios.cpp:43-74).
__device__ __forceinline__ void ghost_transform(const StepArgs& A, int side, double c[4]) {
    const int t = A.bc_type[side];
    const bool xside = side == SILT_WEST || side == SILT_EAST;
    if (t == SILT_BC_INFLOW) {
        if (A.bc_super[side]) c[0] = A.bc_h0[side];
        if (xside) {
            c[1] = A.bc_q0[side];
            c[2] = 0.0;
        } else {
            c[2] = A.bc_q0[side];
            c[1] = 0.0;
        }
    } else if (t == SILT_BC_WALL) {
        if (xside)
            c[1] = -c[1];
        else
            c[2] = -c[2];
    }
}

__device__ __forceinline__ void load_interior(const StepArgs& A, int p, int col, int row,
                                              double c[4]) {
    if (SILT_VIOLATED(row >= 0 && row < A.ny && col >= 0 && col < A.nx, 1, row, col)) return;
    const size_t off = (size_t)row * A.pitch + col;
#pragma unroll
    for (int f = 0; f < 4; ++f) c[f] = __ldg(A.state[p][f] + off);
}

// Cell (col, row) of state parity p, ghosts synthesised: rows -1 / ny come
// from the ghost-row buffers (BC rows written by the previous launch, or rows
// received from a neighbour strip); columns -1 / nx are built from the x-side
// boundary condition (apply_bc_side, src/scenarios.cpp:78-99) or wrap
// (periodic), or come from caller-supplied ghost columns (GIVEN).
__device__ __forceinline__ void load_cell(const StepArgs& A, int p, int col, int row, double c[4]) {
    const int nx = A.nx;
    if (row < 0 || row >= A.ny) {
        const double* g;
        if (row < 0)
            g = A.south_nbr ? A.recv_s[p] : A.ghost_s[p];
        else
            g = A.north_nbr ? A.recv_n[p] : A.ghost_n[p];
        const int cc = min(max(col, 0), nx - 1);
#pragma unroll
        for (int f = 0; f < 4; ++f) c[f] = g[(size_t)f * nx + cc];
        return;
    }
    if (col >= 0 && col < nx) {
        load_interior(A, p, col, row, c);
        return;
    }
    if (col < -1 || col > nx) {  // dead lane: any valid cell
        load_interior(A, p, col < 0 ? 0 : nx - 1, row, c);
        return;
    }
    const int side = col < 0 ? SILT_WEST : SILT_EAST;
    const int t = A.bc_type[side];
    if (t == SILT_BC_PERIODIC) {
        load_interior(A, p, col < 0 ? nx - 1 : 0, row, c);
        return;
    }
    if (t == SILT_BC_GIVEN) {
        const double* g = side == SILT_WEST ? A.ghost_w : A.ghost_e;
#pragma unroll
        for (int f = 0; f < 4; ++f) c[f] = g[(size_t)f * A.ny + row];
        return;
    }
    load_interior(A, p, col < 0 ? 0 : nx - 1, row, c);
    ghost_transform(A, side, c);
}

// Ghost rows of a freshly written edge row (row 0 or ny-1) for the next
// state parity q: physical BC ghost, periodic self-wrap, or the send buffer
// for a neighbour strip.
__device__ __forceinline__ void write_edges(const StepArgs& A, int q, int col, int row,
                                            const double c[4]) {
    if (SILT_VIOLATED(col >= 0 && col < A.nx, 2, row, col)) return;
    if (row == 0) {
        if (A.south_nbr) {
#pragma unroll
            for (int f = 0; f < 4; ++f) A.send_s[q][(size_t)f * A.nx + col] = c[f];
        } else if (A.per_y_self) {
#pragma unroll
            for (int f = 0; f < 4; ++f) A.ghost_n[q][(size_t)f * A.nx + col] = c[f];
        } else if (A.bc_type[SILT_SOUTH] != SILT_BC_GIVEN) {
            double g[4] = {c[0], c[1], c[2], c[3]};
            ghost_transform(A, SILT_SOUTH, g);
#pragma unroll
            for (int f = 0; f < 4; ++f) A.ghost_s[q][(size_t)f * A.nx + col] = g[f];
        }
    }
    if (row == A.ny - 1) {
        if (A.north_nbr) {
#pragma unroll
            for (int f = 0; f < 4; ++f) A.send_n[q][(size_t)f * A.nx + col] = c[f];
        } else if (A.per_y_self) {
#pragma unroll
            for (int f = 0; f < 4; ++f) A.ghost_s[q][(size_t)f * A.nx + col] = c[f];
        } else if (A.bc_type[SILT_NORTH] != SILT_BC_GIVEN) {
            double g[4] = {c[0], c[1], c[2], c[3]};
            ghost_transform(A, SILT_NORTH, g);
#pragma unroll
            for (int f = 0; f < 4; ++f) A.ghost_n[q][(size_t)f * A.nx + col] = g[f];
        }
    }
}

// Per-cell CFL candidates of a state (axis_speed, src/stepper.cpp:30-36, on
// primitives of a wet cell).
template <bool S, bool SH>
__device__ __forceinline__ void cell_speeds(const StepArgs& A, const double c[4], double& sx,
                                            double& sy) {
    const Params& P = A.P;
    const double h = c[0];
    if constexpr (S) {
        const double u = c[1] / h, v = c[2] / h;
        sx = axis_speed_ref<SH>(P, h, u, v);
        sy = (A.dim == 2) ? axis_speed_ref<SH>(P, h, v, u) : 0.0;
    } else {
        const double rh = rcp(h);
        const double u = c[1] * rh, v = c[2] * rh;
        const double gh = P.g * h;
        const double s2 = fma(u, u, v * v);
        double dqx = 0, dqy = 0, om;
        ShieldsRates LR;
        if constexpr (SH) {
            LR = shields_rates_fast(P, h, s2);
            shields_terms_fast(LR, u, s2, om, dqx);
        } else {
            grass_terms_fast(P, u, v, s2, om, dqx);
        }
        const double au = fabs(u), av = fabs(v);
        sx = au + fsqrt(smax(gh, fma(u, u, P.g * dqx)));
        if (A.dim == 2) {
            if constexpr (SH)
                shields_terms_fast(LR, v, s2, om, dqy);
            else
                grass_terms_fast(P, v, u, s2, om, dqy);
            sy = av + fsqrt(smax(gh, fma(v, v, P.g * dqy)));
        } else {
            sy = 0.0;
        }
    }
}

struct Reduce {
    double sx, sy, hmax;
    unsigned wet;
};

__device__ __forceinline__ void reduce_fold(const StepArgs& A, Reduce& R, const double c[4],
                                            double sx, double sy) {
    R.hmax = smax(R.hmax, c[0]);
    if (c[0] > A.P.h_dry) {
        R.wet = 1u;
        if (sx == sx) R.sx = smax(R.sx, sx);
        if (sy == sy) R.sy = smax(R.sy, sy);
    }
}

// CFL speeds of an updated row (the NEXT step's cfl_dt), folded into the
// lane's maxima.  (An fp32-screened fold — exact fp64 speeds only for cells
// whose fp32 estimate reaches the warp's running maximum — was bit-identical
// but measured 7 % slower on C5: DESIGN.md §7.)
template <bool S, bool SH>
__device__ __forceinline__ void fold_speeds(const StepArgs& A, Reduce& R, const double o[4],
                                            bool upd) {
    if (upd) {
        double sx, sy;
        cell_speeds<S, SH>(A, o, sx, sy);
        reduce_fold(A, R, o, sx, sy);
    }
}

// warp reduce + one conditional atomic per warp into the slot
__device__ __forceinline__ void reduce_flush(Reduce R, Slot& s) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        R.sx = smax(R.sx, __shfl_xor_sync(0xffffffffu, R.sx, o));
        R.sy = smax(R.sy, __shfl_xor_sync(0xffffffffu, R.sy, o));
        R.hmax = smax(R.hmax, __shfl_xor_sync(0xffffffffu, R.hmax, o));
        R.wet |= __shfl_xor_sync(0xffffffffu, R.wet, o);
    }
    if ((threadIdx.x & 31) == 0) {
        volatile Slot& vs = s;
        if (R.sx > 0 && R.sx > __longlong_as_double((long long)vs.max_sx))
            atomicMax(&s.max_sx, (unsigned long long)__double_as_longlong(R.sx));
        if (R.sy > 0 && R.sy > __longlong_as_double((long long)vs.max_sy))
            atomicMax(&s.max_sy, (unsigned long long)__double_as_longlong(R.sy));
        if (R.hmax > 0 && R.hmax > __longlong_as_double((long long)vs.hmax))
            atomicMax(&s.hmax, (unsigned long long)__double_as_longlong(R.hmax));
        if (R.wet && !vs.wet) atomicOr(&s.wet, 1u);
    }
}

template <bool S, bool SH>
__device__ __forceinline__ void make_sides(const StepArgs& A, const double c[4], Side& sx, Side& sy,
                                           bool need_x) {
    if constexpr (S) {
        if (need_x) sx = make_side_ref<SH>(A.P, c[0], c[1], c[2], c[3]);
        sy = make_side_ref<SH>(A.P, c[0], c[2], c[1], c[3]);
    } else {
        const CellPre pre = cell_pre_fast<SH>(A.P, c[0], c[1], c[2], c[3]);
        if (need_x) sx = make_side_fast<SH>(A.P, pre, true);
        sy = make_side_fast<SH>(A.P, pre, false);
    }
}

// ---- K1: fused 2D step ----------------------------------------------------
#ifndef SILT_STEP_MIN_BLOCKS
#define SILT_STEP_MIN_BLOCKS 3
#endif

// Per-lane source of the cp.async row prefetch.  The column mapping (interior
// column, periodic wrap, the interior cell a physical x-ghost is derived from,
// or a caller-given ghost column) is fixed per lane, so it is resolved once:
// interior rows then cost one multiply-add per field.  Rows -1 / ny come from
// the ghost-row buffers (physical BC rows, or rows received from a neighbour).
struct RowSrc {
    const double* base;  // field 0; field f at base + f * fstride
    size_t stride;       // row stride (pitch, or 1 for a given ghost column)
    size_t fstride;      // field stride (plane, or ny for a given ghost column)
    int col_clamped;
};

__device__ __forceinline__ RowSrc row_src(const StepArgs& A, int p, int col) {
    RowSrc s;
    const int nx = A.nx;
    int c;
    s.stride = A.pitch;
    if (col == -1 || col == nx) {
        const int side = col < 0 ? SILT_WEST : SILT_EAST;
        const int t = A.bc_type[side];
        if (t == SILT_BC_GIVEN) {
            const double* g = side == SILT_WEST ? A.ghost_w : A.ghost_e;
            s.base = g;
            s.fstride = A.ny;
            s.stride = 1;
            s.col_clamped = col < 0 ? 0 : nx - 1;
            return s;
        }
        c = (t == SILT_BC_PERIODIC) ? (col < 0 ? nx - 1 : 0) : (col < 0 ? 0 : nx - 1);
    } else {
        c = min(max(col, 0), nx - 1);  // dead lanes: any valid cell
    }
    s.base = A.state[p][0] + c;
    s.fstride = A.plane;
    s.col_clamped = min(max(col, 0), nx - 1);
    return s;
}

__device__ __forceinline__ const double* row_field(const StepArgs& A, const RowSrc& s, int p,
                                                   int row, int f) {
    if (row >= 0 && row < A.ny) return s.base + (size_t)f * s.fstride + (size_t)row * s.stride;
    const double* g = row < 0 ? (A.south_nbr ? A.recv_s[p] : A.ghost_s[p])
                              : (A.north_nbr ? A.recv_n[p] : A.ghost_n[p]);
    return g + (size_t)f * A.nx + s.col_clamped;
}

__device__ __forceinline__ void cp_async8_s(unsigned dst, const double* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(dst), "l"(src) : "memory");
}

// Prefetch the 4 fields of one row: a single range check and one 64-bit
// offset per row; dst = shared address of field 0's slot, fields kStepThreads
// doubles apart.
__device__ __forceinline__ void prefetch_row(const StepArgs& A, const RowSrc& s, int p, int row,
                                             unsigned dst) {
    constexpr unsigned kFieldBytes = kStepThreads * sizeof(double);
    if (SILT_VIOLATED(row >= -1 && row <= A.ny && s.col_clamped >= 0 && s.col_clamped < A.nx,
                      3, row, s.col_clamped))
        return;
    if (row >= 0 && row < A.ny) {
        const size_t off = (size_t)row * s.stride;
#pragma unroll
        for (int f = 0; f < 4; ++f)
            cp_async8_s(dst + f * kFieldBytes, s.base + (size_t)f * s.fstride + off);
    } else {
#pragma unroll
        for (int f = 0; f < 4; ++f) cp_async8_s(dst + f * kFieldBytes, row_field(A, s, p, row, f));
    }
}

// Physical x-boundary ghost (apply_bc_side, src/scenarios.cpp:78-99) applied
// to the interior cell the row prefetch copied (row_src).
__device__ __forceinline__ void fix_xghost(const StepArgs& A, int col, int row, double c[4]) {
    if (row < 0 || row >= A.ny || (col != -1 && col != A.nx)) return;
    const int side = col < 0 ? SILT_WEST : SILT_EAST;
    const int t = A.bc_type[side];
    if (t == SILT_BC_GIVEN || t == SILT_BC_PERIODIC) return;
    ghost_transform(A, side, c);
}

__device__ __forceinline__ void cp_async8(double* dst, const double* src) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(src) : "memory");
}
// "memory" clobbers: shared-memory reads of a slot must not move across the
// wait that makes it valid, nor across the copy that overwrites it.
__device__ __forceinline__ void cp_async_commit() {
    asm volatile("cp.async.commit_group;\n" ::: "memory");
}
__device__ __forceinline__ void cp_async_wait1() {
    asm volatile("cp.async.wait_group 1;\n" ::: "memory");
}
__device__ __forceinline__ void cp_async_wait2() {
    asm volatile("cp.async.wait_group 2;\n" ::: "memory");
}
#ifndef SILT_RING
#define SILT_RING 6
#endif
__device__ __forceinline__ void cp_async_wait_ring() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(SILT_RING - 2) : "memory");
}

template <int W>
__device__ __forceinline__ void side_to_ring(double (*ring)[W], int* flags, const Side& s, int lane) {
    ring[0][lane] = s.h;
    ring[1][lane] = s.hun;
    ring[2][lane] = s.pi;
    ring[3][lane] = s.z;
    ring[4][lane] = s.omega;
    ring[5][lane] = s.un;
    ring[6][lane] = s.ut;
    ring[7][lane] = s.tau;
    ring[8][lane] = s.a_side;
    ring[9][lane] = s.b2_side;
    flags[lane] = s.wet | (s.moving << 1);
}

template <int W>
__device__ __forceinline__ Side side_from_ring(const double (*ring)[W], const int* flags, int lane) {
    Side s;
    s.h = ring[0][lane];
    s.hun = ring[1][lane];
    s.pi = ring[2][lane];
    s.z = ring[3][lane];
    s.omega = ring[4][lane];
    s.un = ring[5][lane];
    s.ut = ring[6][lane];
    s.tau = ring[7][lane];
    s.a_side = ring[8][lane];
    s.b2_side = ring[9][lane];
    const int fl = flags[lane];
    s.wet = fl & 1;
    s.moving = (fl >> 1) & 1;
    return s;
}

template <bool S, bool SH>
__device__ __forceinline__ Side side_of(const StepArgs& A, const double c[4], bool xaxis) {
    if constexpr (S) {
        return xaxis ? make_side_ref<SH>(A.P, c[0], c[1], c[2], c[3])
                     : make_side_ref<SH>(A.P, c[0], c[2], c[1], c[3]);
    } else {
        const CellPre pre = cell_pre_fast<SH>(A.P, c[0], c[1], c[2], c[3]);
        return make_side_fast<SH>(A.P, pre, xaxis);
    }
}

template <bool S, bool SH>
__device__ __forceinline__ void sides_of(const StepArgs& A, const double c[4], Side& sx, Side& sy) {
#ifdef SILT_FAST_REF_SIDES  // diagnostics: FAST face solver on the reference's per-cell terms
    if constexpr (true) {
#else
    if constexpr (S) {
#endif
        sx = make_side_ref<SH>(A.P, c[0], c[1], c[2], c[3]);
        sy = make_side_ref<SH>(A.P, c[0], c[2], c[1], c[3]);
    } else {
        const CellPre pre = cell_pre_fast<SH>(A.P, c[0], c[1], c[2], c[3]);
        sx = make_side_fast<SH>(A.P, pre, true);
        sy = make_side_fast<SH>(A.P, pre, false);
    }
}

// SILT_PDL: 2D step launches with programmatic stream serialization (the next
// step's CTAs launch during this step's tail and wait in griddepcontrol.wait):
// C3 74.7 -> 73.1 us per step, bit-identical; long launches unchanged
#ifndef SILT_PDL
#define SILT_PDL 1
#endif
// SILT_RING: cp.async ring slots; rows are issued SILT_RING-1 ahead
// Per-CTA shared memory of the 2D step (dynamic: above the 48 KB static cap).
struct StepSmem {
    double row[SILT_RING][4][kStepThreads];  // cp.async ring
    double side[10][kStepThreads];        // y-side terms of row r-1
    double sx[10][kStepThreads + 1];      // x-side terms of row r (+1: lane 31 reads t+1)
    int side_fl[kStepThreads];            // their wet / moving flags
    int sx_fl[kStepThreads + 1];
    double xs[4][kStepThreads];           // x-updated row r-1
    double fy[4][kStepThreads];           // y face below row r-1: h, huR, hv, z
    int nfull[kStepThreads / 32];         // full-path rows of each warp (launch order)
};

// Rows of a warp's march on the full (non-quiescent) path above which its
// row block counts as hot for the next launch's order.
constexpr int kHotRows = 4;

template <bool S, bool SH, bool WI = false>
__global__ void __launch_bounds__(kStepThreads, SILT_STEP_MIN_BLOCKS) step2d_kernel(StepArgs A, int li) {
    // Per-thread march state in shared memory (SoA by thread: conflict-free),
    // so that registers at each face solve hold little beyond the solver.
    extern __shared__ __align__(16) unsigned char step_smem_raw[];
    StepSmem& sm = *reinterpret_cast<StepSmem*>(step_smem_raw);
#if SILT_PDL
    // Programmatic dependent launch: this grid may be launched while the
    // previous step's is still finishing; wait for it (and its memory) before
    // touching the control slot or the state, and let the next step's grid
    // launch as soon as every CTA of this one is running.
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;");
#endif
    auto& sh_side = sm.side;
    auto& sh_sx = sm.sx;
    auto& sh_xs = sm.xs;
    auto& sh_fy = sm.fy;
    auto& sh_row = sm.row;

    const Slot cur = A.ctl->slot[li % 3];
    const RunDecision d = decide(A, cur);
    if (A.epilogue && blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0)
        control_epilogue(A, li, cur, d);
    if (!d.run) return;
    Slot& nxt = A.ctl->slot[(li + 1) % 3];

    const int p = (int)(cur.steps & 1), q = p ^ 1;
    const int t = threadIdx.x;
    const int lane = t & 31;
    const double cx = d.dt / A.dx;
    const double cy = d.dt / A.dy;
    const double href = __longlong_as_double((long long)cur.hmax);
    Reduce R{0.0, 0.0, 0.0, 0u};
    // Work items.  Default: one (column band, row block) per warp, from the
    // launch grid.  Warp-item mode (WI: short launches, A.warp_items): the grid
    // is one wave of resident CTAs and every warp pulls (band, row block)
    // items from a per-launch counter until none are left — no partly empty
    // last wave and no CTA start-up per item; the maxima of all the warp's
    // items fold into one reduction.
    const int gwarp = (blockIdx.x + blockIdx.y * gridDim.x) * (kStepThreads / 32) + (t >> 5);
    int item = gwarp;
    do {
    {
    int strip, rbi;
    if constexpr (WI) {
        // items run row block by row block (bands fastest), in the launch's
        // row-block order when there is one (hot blocks spread, §3c)
        strip = item % A.bands;
        rbi = item / A.bands;
        if (A.rb_map) rbi = __ldg(A.rb_map + rbi);
    } else {
        strip = blockIdx.x * (kStepThreads / 32) + (t >> 5);
        rbi = A.rb_map ? __ldg(A.rb_map + blockIdx.y) : (int)blockIdx.y;
    }
    const int i0 = strip * kCellsPerWarp;
    if (i0 >= A.nx) goto item_done;  // warp-uniform
    const int col = i0 - 1 + lane;
    const bool owned = lane >= 1 && lane <= kCellsPerWarp && col < A.nx;
    const bool xface = lane <= kCellsPerWarp && col <= A.nx - 1;  // face at right of col
    const int jb = rbi * A.rows_per_block;
    const int je = min(jb + A.rows_per_block, A.ny);
    if (jb >= je) goto item_done;
    if (lane == 0) sm.nfull[t >> 5] = 0;
#ifdef SILT_TRACE
    unsigned long long tr_start = 0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tr_start));
#endif
    const RowSrc src = row_src(A, p, col);

    const unsigned row_sa0 = (unsigned)__cvta_generic_to_shared(&sh_row[0][0][t]);
    constexpr unsigned kSlotBytes = 4 * kStepThreads * sizeof(double);
    double* const out0 = A.state[q][0] + col;  // output cell (row 0) of field 0
    const size_t plane = A.plane;              // field f at out0 + f * plane
#pragma unroll
    for (int k = 0; k < SILT_RING - 1; ++k) {
        if (jb - 1 + k <= je) prefetch_row(A, src, p, jb - 1 + k, row_sa0 + k * kSlotBytes);
        cp_async_commit();
    }
    int buf = 0;  // ring slot of row r
    // Quiescent rows (FAST): when rows r-2, r-1 and r of this warp are bitwise
    // equal and uniform across the warp (and wet), every face touching row r-1
    // takes face_flux's exact uniform-state flux, so its update is exactly the
    // identity and the shared-memory march state is already correct; the row
    // is stored unchanged and its CFL speed comes from a one-entry cache.  The
    // result is bit-identical to the full path (tests: SILT_QUIET_SKIP=0).
    // Speeds of the current quiescent streak (the state is the same on every
    // skipped row of a streak), folded into the reduction once per streak.
    bool quiet_prev = false, qvalid = false;
    bool quiet_prev2 = false;  // STRICT: row r-2 equal to row r-3 on every lane
    double qsx = 0.0, qsy = 0.0;
    // streak loop (below): not in the warps holding an x-ghost column, whose
    // ghost cells are transformed after the load
    const bool xedge = i0 == 0 || i0 + kCellsPerWarp >= A.nx;
    bool have = false, eq_have = false;  // row r already loaded by the streak loop
#pragma unroll 1
    for (int r = jb - 1; r <= je; ++r) {
        // The slot of row r-1 is refilled (with row r+RING-1) only after row r
        // has been compared with it: RING-1 rows stay in flight while row r is
        // processed, and the quiescence test needs no copy of the previous row.
        const int prev = buf == 0 ? SILT_RING - 1 : buf - 1;  // slot of row r-1
        double c[4];
        unsigned long long dif = 0;  // row r vs row r-1, bitwise (as loaded)
        if (!have) {
            cp_async_wait_ring();  // row r landed; the later rows may be in flight
#pragma unroll
            for (int f = 0; f < 4; ++f) {
                c[f] = sh_row[buf][f][t];
                dif |= (unsigned long long)(__double_as_longlong(c[f]) ^
                                            __double_as_longlong(sh_row[prev][f][t]));
            }
            // every lane's reads of slot `prev` precede the refill (lanes of a
            // warp only ever touch their own column of a slot)
            if (r + SILT_RING - 1 <= je)
                prefetch_row(A, src, p, r + SILT_RING - 1, row_sa0 + prev * kSlotBytes);
            cp_async_commit();
        } else {  // waited for, compared and refilled by the streak loop
#pragma unroll
            for (int f = 0; f < 4; ++f) c[f] = sh_row[buf][f][t];
            dif = eq_have ? 0ull : 1ull;
            have = false;
        }
        buf = buf == SILT_RING - 1 ? 0 : buf + 1;
        if (SILT_VIOLATED(blockDim.x == kStepThreads && buf >= 0 && buf < SILT_RING, 4, buf,
                          blockDim.x))
            goto item_done;
        fix_xghost(A, col, r, c);
        const bool own_row = r >= jb && r < je;

        if constexpr (!S) {
            if (A.quiet_skip) {
                // vertical equality first (cheap); the horizontal test with
                // shuffles only when the whole warp passed it
                long long cb[4];
#pragma unroll
                for (int f = 0; f < 4; ++f) cb[f] = __double_as_longlong(c[f]);
                const bool eqy = r > jb - 1 && dif == 0ull;
                // Inside a streak one vote suffices: if every lane (halo and
                // dead lanes included) sees row r equal to row r-1, and row r-1
                // was verified uniform across the warp and wet, so is row r.
                bool quiet = quiet_prev && __all_sync(0xffffffffu, eqy);
                if (!quiet) {
                    const bool wet = c[0] > A.P.h_dry;
                    quiet = __all_sync(0xffffffffu, !owned || (eqy && wet));
                    if (quiet) {
                        unsigned long long difx = 0;
#pragma unroll
                        for (int f = 0; f < 4; ++f)  // every lane shuffles
                            difx |= (unsigned long long)(cb[f] ^
                                                         __shfl_down_sync(0xffffffffu, cb[f], 1));
                        quiet = __all_sync(0xffffffffu, !xface || (difx == 0ull && wet));
                    }
                }
                const bool skip = quiet && quiet_prev && r - 1 >= jb;
                quiet_prev = quiet;
                if (!skip) qvalid = false;
                if (skip) {
                    if (owned && !SILT_VIOLATED(r - 1 >= 0 && r - 1 < A.ny && col < A.nx, 6,
                                                r - 1, col)) {  // row r-1 is unchanged: o == c
                        const size_t off = (size_t)(r - 1) * A.pitch;
                        out0[off] = c[0];
                        out0[off + plane] = c[1];
                        out0[off + 2 * plane] = c[2];
                        out0[off + 3 * plane] = c[3];
                        if (r - 1 == 0 || r - 1 == A.ny - 1) write_edges(A, q, col, r - 1, c);
                        if (!qvalid) {  // first row of the streak: its speeds, folded once
                            cell_speeds<S, SH>(A, c, qsx, qsy);
                            reduce_fold(A, R, c, qsx, qsy);
                            qvalid = true;
                        }
                    }
                    // Streak loop: rows r-1 and r are quiet, so row r+1 is
                    // quiet iff every lane sees it equal to row r (the vote
                    // above), and then row r is stored unchanged.  A short
                    // dependency chain per row (no x-ghost fix, no second
                    // test, the previous row from registers); the first
                    // non-quiet row goes back to the loop above, already
                    // loaded.  Same decisions and stores as that loop.
                    if (!xedge) {
#pragma unroll 1
                        while (r < je) {
                            const int pv = buf == 0 ? SILT_RING - 1 : buf - 1;  // slot of row r
                            cp_async_wait_ring();  // row r+1 landed
                            unsigned long long dn = 0;
#pragma unroll
                            for (int f = 0; f < 4; ++f)
                                dn |= (unsigned long long)(__double_as_longlong(sh_row[buf][f][t]) ^
                                                           __double_as_longlong(c[f]));
                            if (r + SILT_RING <= je)
                                prefetch_row(A, src, p, r + SILT_RING, row_sa0 + pv * kSlotBytes);
                            cp_async_commit();
                            if (!__all_sync(0xffffffffu, dn == 0ull)) {
                                have = true;  // row r+1 is the next trip's row r
                                eq_have = dn == 0ull;
                                break;
                            }
                            buf = buf == SILT_RING - 1 ? 0 : buf + 1;
                            if (owned && !SILT_VIOLATED(r >= 0 && r < A.ny && col < A.nx, 7, r,
                                                        col)) {  // row r is unchanged: o == c
                                const size_t off = (size_t)r * A.pitch;
                                out0[off] = c[0];
                                out0[off + plane] = c[1];
                                out0[off + 2 * plane] = c[2];
                                out0[off + 3 * plane] = c[3];
                                if (r == 0 || r == A.ny - 1) write_edges(A, q, col, r, c);
                            }
                            ++r;
                        }
                    }
                    continue;  // warp-uniform
                }
            }
        } else {
            if (A.quiet_skip) {
                // Repeated rows (STRICT, the reference's arithmetic, which has
                // no exact uniform-state shortcut): when rows r-3 .. r of this
                // warp are equal column by column (every lane, halo and dead
                // lanes included), the faces of row r-1 see exactly the states
                // the faces of row r-2 saw, so row r-1's update is row r-2's,
                // bit for bit, whatever the flow: it is read back from the
                // output (this lane stored it one row ago, its CFL speeds are
                // already folded) and stored again.  The march state in shared
                // memory belongs to rows equal to row r-1, so it stays correct.
                const bool eqy = r > jb - 1 && dif == 0ull;
                const bool same = __all_sync(0xffffffffu, eqy);
                const bool skip = same && quiet_prev && quiet_prev2 && r - 2 >= jb;
                quiet_prev2 = quiet_prev;
                quiet_prev = same;
                if (skip) {
                    double qv[4] = {0.0, 0.0, 0.0, 0.0};
                    if (owned && !SILT_VIOLATED(r - 2 >= 0 && r - 1 < A.ny && col < A.nx, 6,
                                                r - 1, col)) {
                        const size_t off = (size_t)(r - 2) * A.pitch;
#pragma unroll
                        for (int f = 0; f < 4; ++f) qv[f] = out0[off + (size_t)f * plane];
                        const size_t off1 = off + A.pitch;
#pragma unroll
                        for (int f = 0; f < 4; ++f) out0[off1 + (size_t)f * plane] = qv[f];
                        if (r - 1 == 0 || r - 1 == A.ny - 1) write_edges(A, q, col, r - 1, qv);
                    }
                    // streak loop: row r+1 repeats iff every lane sees it equal
                    // to row r; then row r's update is the same again
                    if (!xedge) {
#pragma unroll 1
                        while (r < je) {
                            const int pv = buf == 0 ? SILT_RING - 1 : buf - 1;  // slot of row r
                            cp_async_wait_ring();  // row r+1 landed
                            unsigned long long dn = 0;
#pragma unroll
                            for (int f = 0; f < 4; ++f)
                                dn |= (unsigned long long)(__double_as_longlong(sh_row[buf][f][t]) ^
                                                           __double_as_longlong(c[f]));
                            if (r + SILT_RING <= je)
                                prefetch_row(A, src, p, r + SILT_RING, row_sa0 + pv * kSlotBytes);
                            cp_async_commit();
                            if (!__all_sync(0xffffffffu, dn == 0ull)) {
                                have = true;  // row r+1 is the next trip's row r
                                eq_have = dn == 0ull;
                                break;
                            }
                            buf = buf == SILT_RING - 1 ? 0 : buf + 1;
                            if (owned && !SILT_VIOLATED(r >= 0 && r < A.ny && col < A.nx, 7, r,
                                                        col)) {
                                const size_t off = (size_t)r * A.pitch;
                                out0[off] = qv[0];
                                out0[off + plane] = qv[1];
                                out0[off + 2 * plane] = qv[2];
                                out0[off + 3 * plane] = qv[3];
                                if (r == 0 || r == A.ny - 1) write_edges(A, q, col, r, qv);
                            }
                            ++r;
                        }
                    }
                    continue;  // warp-uniform
                }
            }
        }

        if (own_row && lane == 0) ++sm.nfull[t >> 5];
        // y face between rows r-1 and r (normal = v, transverse = u), solved
        // first; the x-side waits in shared memory for the x face
        Flux fy{0, 0, 0, 0, 0};
        {
            Side sx, sy;
            sides_of<S, SH>(A, c, sx, sy);
            if (own_row) side_to_ring(sh_sx, sm.sx_fl, sx, t);
            if (r > jb - 1 && owned) {
                const Side lo = side_from_ring(sh_side, sm.side_fl, t);
                if (!face_flux<S>(A.P, lo, sy, fy)) {
                    const double info[6] = {lo.h, lo.un, lo.z, sy.h, sy.un, sy.z};
                    record_error(A, kErrRiemann, col, r + A.j0, info, nxt);
                }
            }
            side_to_ring(sh_side, sm.side_fl, sy, t);
        }
        double o[4];
        bool upd = false;
        if (r - 1 >= jb && owned) {
            // y update of row r-1 (src/stepper.cpp:181-186) + check_depth
            o[0] = sh_xs[0][t] - cy * (fy.h - sh_fy[0][t]);
            o[2] = sh_xs[2][t] - cy * (fy.huL - sh_fy[1][t]);
            o[1] = sh_xs[1][t] - cy * (fy.hv - sh_fy[2][t]);
            o[3] = sh_xs[3][t] - cy * (fy.z - sh_fy[3][t]);
            if (!check_depth(o[0], href)) record_error(A, kErrNegDepth, col, r - 1 + A.j0, nullptr, nxt);
            if (!SILT_VIOLATED(r - 1 >= 0 && r - 1 < A.ny && col >= 0 && col < A.nx, 5, r - 1, col)) {
                const size_t off = (size_t)(r - 1) * A.pitch;
                out0[off] = o[0];
                out0[off + plane] = o[1];
                out0[off + 2 * plane] = o[2];
                out0[off + 3 * plane] = o[3];
                if (r - 1 == 0 || r - 1 == A.ny - 1) write_edges(A, q, col, r - 1, o);
                upd = true;
            }
        }
        fold_speeds<S, SH>(A, R, o, upd);
        if (!own_row) continue;  // warp-uniform
        sh_fy[0][t] = fy.h;
        sh_fy[1][t] = fy.huR;
        sh_fy[2][t] = fy.hv;
        sh_fy[3][t] = fy.z;
        __syncwarp();
        // x faces: this lane solves the face between col and col+1
        Flux fx{0, 0, 0, 0, 0};
        if (xface) {
            const Side sx = side_from_ring(sh_sx, sm.sx_fl, t);
            const Side right = side_from_ring(sh_sx, sm.sx_fl, t + 1);
            if (!face_flux<S>(A.P, sx, right, fx)) {
                const double info[6] = {sx.h, sx.un, sx.z, right.h, right.un, right.z};
                record_error(A, kErrRiemann, col, r + A.j0, info, nxt);
            }
        }
        const double lh = shfl_up_d(fx.h, 1), lhuR = shfl_up_d(fx.huR, 1);
        const double lhv = shfl_up_d(fx.hv, 1), lz = shfl_up_d(fx.z, 1);
        // x update (step_2d x sweep, src/stepper.cpp:165-170)
        sh_xs[0][t] = c[0] - cx * (fx.h - lh);
        sh_xs[1][t] = c[1] - cx * (fx.huL - lhuR);
        sh_xs[2][t] = c[2] - cx * (fx.hv - lhv);
        sh_xs[3][t] = c[3] - cx * (fx.z - lz);
        __syncwarp();
    }
    if (A.rb_order && lane == 0 && sm.nfull[t >> 5] > kHotRows) A.rb_hot[li][rbi] = 1;
#ifdef SILT_TRACE
    // (trace build only, launch-grid mode) per-warp fold into the CTA's
    // record; the buffer is initialised to {~0, 0, 0, 0} by the tool
    if (!S && !WI && g_trace && lane == 0) {
        unsigned long long tr_end;
        unsigned smid;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tr_end));
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        unsigned long long* rec = g_trace + 4 * ((size_t)blockIdx.y * gridDim.x + blockIdx.x);
        atomicMin(rec, tr_start);
        atomicMax(rec + 1, tr_end);
        rec[2] = smid | ((unsigned long long)blockIdx.x << 16);
        atomicAdd(rec + 3, (unsigned long long)(jb / A.rows_per_block) * (t == 0) +
                                ((unsigned long long)sm.nfull[t >> 5] << 32));
    }
#endif
    }
    item_done:
        if constexpr (!WI) break;
        {
            unsigned nxt_item = 0;
            if (lane == 0) nxt_item = atomicAdd(&A.ctl->item_ctr[li % 3], 1u);
            item = A.warps_total + (int)__shfl_sync(0xffffffffu, nxt_item, 0);
        }
    } while (item < A.n_items);
    reduce_flush(R, nxt);
}

// ---- K2: 1D step (step_1d, src/stepper.cpp:118-140) ----------------------
template <bool S, bool SH>
__device__ __forceinline__ void step1d_body(const StepArgs& A, int li) {
    const Slot cur = A.ctl->slot[li % 3];
    const RunDecision d = decide(A, cur);
    if (blockIdx.x == 0 && threadIdx.x == 0) control_epilogue(A, li, cur, d);
    if (!d.run) return;
    Slot& nxt = A.ctl->slot[(li + 1) % 3];
    const int p = (int)(cur.steps & 1), q = p ^ 1;
    const int lane = threadIdx.x & 31;
    const int strip = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
    const int i0 = strip * kCellsPerWarp;
    if (i0 >= A.nx) return;
    const int col = i0 - 1 + lane;
    const bool owned = lane >= 1 && lane <= kCellsPerWarp && col < A.nx;
    const bool xface = lane <= kCellsPerWarp && col <= A.nx - 1;
    const double c1 = d.dt / A.dx;
    const double href = __longlong_as_double((long long)cur.hmax);
    double c[4];
    load_cell(A, p, col, 0, c);
    Side sx;
    if constexpr (S) {
        sx = make_side_ref<SH>(A.P, c[0], c[1], c[2], c[3]);
    } else {
        const CellPre pre = cell_pre_fast<SH>(A.P, c[0], c[1], c[2], c[3]);
        sx = make_side_fast<SH>(A.P, pre, true);
    }
    const Side right = shfl_down_side(sx);
    Flux fx{0, 0, 0, 0, 0};
    if (xface && !face_flux<S>(A.P, sx, right, fx)) {
        const double info[6] = {sx.h, sx.un, sx.z, right.h, right.un, right.z};
        record_error(A, kErrRiemann, col, 0, info, nxt);
    }
    const double lh = shfl_up_d(fx.h, 1), lhuR = shfl_up_d(fx.huR, 1);
    const double lhv = shfl_up_d(fx.hv, 1), lz = shfl_up_d(fx.z, 1);
    Reduce R{0.0, 0.0, 0.0, 0u};
    if (owned) {
        double o[4];
        o[0] = c[0] - c1 * (fx.h - lh);
        o[1] = c[1] - c1 * (fx.huL - lhuR);
        o[2] = c[2] - c1 * (fx.hv - lhv);
        o[3] = c[3] - c1 * (fx.z - lz);
        if (!check_depth(o[0], href)) record_error(A, kErrNegDepth, col, 0, nullptr, nxt);
        if (!SILT_VIOLATED(col >= 0 && col < A.nx, 8, 0, col))
#pragma unroll
            for (int f = 0; f < 4; ++f) A.state[q][f][col] = o[f];
        double ssx, ssy;
        cell_speeds<S, SH>(A, o, ssx, ssy);
        reduce_fold(A, R, o, ssx, ssy);
    }
    reduce_flush(R, nxt);
}

template <bool S, bool SH>
__global__ void __launch_bounds__(kStepThreads) step1d_kernel(StepArgs A, int li) {
    step1d_body<S, SH>(A, li);
}

// ---- K2c: n 1D steps in one cooperative launch --------------------------------
// The 1D configurations are latency-bound (a few thousand cells: one face
// solve per lane, then the global reduction); a launch per step adds the
// launch and a cold start each time.  Here all CTAs stay resident and step n
// times, a grid-wide barrier between steps (it orders the state writes and
// the slot reductions of step k before step k+1 reads them).  Steps after the
// run stopped (done / paused / failed) only propagate the run clock, exactly
// as the per-step launches would, so launch index n keeps its meaning.
template <bool S, bool SH>
__global__ void __launch_bounds__(kStepThreads) step1d_coop_kernel(StepArgs A, int li0, int n) {
    cooperative_groups::grid_group g = cooperative_groups::this_grid();
    for (int k = 0; k < n; ++k) {
        step1d_body<S, SH>(A, (li0 + k) % 3);
        g.sync();
    }
}

// Grids that fit one thread-block cluster (up to 16 CTAs of 384 threads:
// 5760 cells, C1 and C2) keep the whole line on chip for the n steps: every
// CTA holds its 360 cells in shared memory (double-buffered by state parity),
// reads the two cells beyond its ends from the neighbouring CTAs' shared
// memory (DSMEM, map_shared_rank), and reduces the axis-speed maxima / hmax /
// wet / error bits through shared memory: a CTA partial, then one cluster
// barrier (release / acquire at cluster scope), then every warp folds the
// CTAs' partials.  Every thread runs the run clock itself (decide(), the same
// arithmetic on the same inputs in every CTA), so a step needs no global
// memory round trip; the state goes back to HBM at the end, the dt log as it
// is made, and the final run header lands in slot (li0 + n) % 3 exactly as n
// launches of step1d_kernel would leave it (after a stop, those launches only
// carry the header forward).  Per-face arithmetic is step1d_body's.
constexpr int kCluster1dThreads = 384;

// Global-memory variant (step1d_body per step, the cluster barrier between
// steps): measured faster than the resident one above 8 CTAs.
template <bool S, bool SH>
__global__ void __launch_bounds__(kCluster1dThreads, 1)
    step1d_cluster_kernel(StepArgs A, int li0, int n) {
    cooperative_groups::cluster_group cl = cooperative_groups::this_cluster();
    for (int k = 0; k < n; ++k) {
        step1d_body<S, SH>(A, (li0 + k) % 3);
        cl.sync();
    }
}

constexpr int kCluster1dWarps = kCluster1dThreads / 32;
#ifndef SILT_RESIDENT_MAX_CTAS
#define SILT_RESIDENT_MAX_CTAS 8
#endif
constexpr int kResidentMaxCtas = SILT_RESIDENT_MAX_CTAS;  // resident 1D kernel up to this many CTAs
constexpr int kCluster1dCells = kCluster1dWarps * kCellsPerWarp;  // 360 per CTA

template <bool S, bool SH>
__global__ void __launch_bounds__(kCluster1dThreads, 1)
    step1d_resident_kernel(StepArgs A, int li0, int n) {
    namespace cg = cooperative_groups;
    cg::cluster_group cl = cg::this_cluster();
    __shared__ double s_line[2][4][kCluster1dCells];  // this CTA's cells, by state parity
    __shared__ double s_wpart[kCluster1dWarps][4];    // warp partials: sx, sy, hmax, wet|err
    __shared__ double s_cta[2][4];                    // CTA partial, by parity of the new state
    const Control& C = *A.ctl;
    const int rank = (int)cl.block_rank();
    const int nctas = (int)cl.num_blocks();
    const int t = threadIdx.x, lane = t & 31, w = t >> 5;
    const int base = rank * kCluster1dCells;
    const int i0 = base + w * kCellsPerWarp;
    const int col = i0 - 1 + lane;
    const int nx = A.nx;
    const bool owned = lane >= 1 && lane <= kCellsPerWarp && col < nx;
    const bool xface = lane <= kCellsPerWarp && col <= nx - 1;
    Slot cur = C.slot[li0 % 3];
    // this lane's cell: interior owner CTA and index, or an x-ghost
    int src = col;
    if (col < -1 || col > nx) src = col < 0 ? 0 : nx - 1;  // dead lane: any valid cell
    const int side = col < 0 ? SILT_WEST : SILT_EAST;
    const bool ghost = col == -1 || col == nx;
    const int bct = ghost ? A.bc_type[side] : SILT_BC_OUTFLOW;
    if (ghost) src = (bct == SILT_BC_PERIODIC) ? (col < 0 ? nx - 1 : 0) : (col < 0 ? 0 : nx - 1);
    int owner = src / kCluster1dCells, idx = src - owner * kCluster1dCells;
    int oi = owned ? col - base : 0;  // this lane's slot in the CTA's line
    if (SILT_VIOLATED(oi >= 0 && oi < kCluster1dCells && idx >= 0 && idx < kCluster1dCells &&
                          owner >= 0 && owner < (int)cl.num_blocks(),
                      9, oi, owner))
        oi = idx = owner = 0;  // checked build: counted, clamped (no early exit: barriers)
    double* const own_cell[2] = {&s_line[0][0][oi], &s_line[1][0][oi]};
    double* const src_cell[2] = {cl.map_shared_rank(&s_line[0][0][idx], owner),
                                 cl.map_shared_rank(&s_line[1][0][idx], owner)};
    constexpr int kF = kCluster1dCells;  // field stride in s_line
    {
        const int p = (int)(cur.steps & 1);
        if (owned)
#pragma unroll
            for (int f = 0; f < 4; ++f) own_cell[p][f * kF] = A.state[p][f][col];
    }
    cl.sync();  // lines filled; every CTA has read the initial header
    unsigned errb = 0;
    // Software pipeline: the CTAs' partials of state n+1 are loaded (DSMEM)
    // right after the barrier but folded only after the next face solve,
    // which needs the cells and not dt; so is the run decision.
    bool pending = false;  // partials loaded, not folded into cur yet
    double pa = 0.0, pb = 0.0, ph = 0.0;
    long long pbits = 0;
    auto fold_partials = [&]() {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            pa = smax(pa, __shfl_xor_sync(0xffffffffu, pa, o));
            pb = smax(pb, __shfl_xor_sync(0xffffffffu, pb, o));
            ph = smax(ph, __shfl_xor_sync(0xffffffffu, ph, o));
            pbits |= __shfl_xor_sync(0xffffffffu, pbits, o);
        }
        cur.max_sx = pa > 0 ? (unsigned long long)__double_as_longlong(pa) : 0ull;
        cur.max_sy = pb > 0 ? (unsigned long long)__double_as_longlong(pb) : 0ull;
        cur.hmax = ph > 0 ? (unsigned long long)__double_as_longlong(ph) : 0ull;
        cur.wet = (unsigned)(pbits & 1);
        cur.err = (unsigned)(pbits >> 1);
        pending = false;
    };
    for (int k = 0; k < n; ++k) {
        const int p = (int)(cur.steps & 1), q = p ^ 1;
        double c[4];
        if (ghost && bct == SILT_BC_GIVEN) {
            const double* g = side == SILT_WEST ? A.ghost_w : A.ghost_e;
#pragma unroll
            for (int f = 0; f < 4; ++f) c[f] = g[(size_t)f * A.ny];
        } else {
#pragma unroll
            for (int f = 0; f < 4; ++f) c[f] = src_cell[p][f * kF];
            if (ghost && bct != SILT_BC_PERIODIC) ghost_transform(A, side, c);
        }
        Side sx;
        if constexpr (S) {
            sx = make_side_ref<SH>(A.P, c[0], c[1], c[2], c[3]);
        } else {
            const CellPre pre = cell_pre_fast<SH>(A.P, c[0], c[1], c[2], c[3]);
            sx = make_side_fast<SH>(A.P, pre, true);
        }
        const Side right = shfl_down_side(sx);
        Flux fx{0, 0, 0, 0, 0};
        const bool face_ok = !xface || face_flux<S>(A.P, sx, right, fx);
        const double lh = shfl_up_d(fx.h, 1), lhuR = shfl_up_d(fx.huR, 1);
        const double lhv = shfl_up_d(fx.hv, 1), lz = shfl_up_d(fx.z, 1);
        if (pending) fold_partials();
        const RunDecision d = decide(A, cur);
        if (!d.run) {  // what the remaining per-step launches would carry forward
            cur.err |= (d.next_state == SILT_STATE_FAILED && !cur.err) ? kErrDry : 0u;
            cur.state = d.next_state;
            break;
        }
        if (rank == 0 && t == 0 && !C.fixed_mode && C.dt_log && cur.steps < C.dt_cap)
            C.dt_log[cur.steps] = d.dt;
        if (!face_ok) {
            errb |= kErrRiemann;
            if (atomicCAS(&A.ctl->err_claim, 0u, 1u) == 0u) {
                A.ctl->err_bits = kErrRiemann;
                A.ctl->err_col = col;
                A.ctl->err_row = 0;
                const double info[6] = {sx.h, sx.un, sx.z, right.h, right.un, right.z};
                for (int m = 0; m < 6; ++m) A.ctl->err_info[m] = info[m];
            }
        }
        const double c1 = d.dt / A.dx;
        const double href = __longlong_as_double((long long)cur.hmax);
        Reduce R{0.0, 0.0, 0.0, 0u};
        if (owned) {
            double o[4];
            o[0] = c[0] - c1 * (fx.h - lh);
            o[1] = c[1] - c1 * (fx.huL - lhuR);
            o[2] = c[2] - c1 * (fx.hv - lhv);
            o[3] = c[3] - c1 * (fx.z - lz);
            if (!check_depth(o[0], href)) {
                errb |= kErrNegDepth;
                if (atomicCAS(&A.ctl->err_claim, 0u, 1u) == 0u) {
                    A.ctl->err_bits = kErrNegDepth;
                    A.ctl->err_col = col;
                    A.ctl->err_row = 0;
                    for (int m = 0; m < 6; ++m) A.ctl->err_info[m] = 0.0;
                }
            }
#pragma unroll
            for (int f = 0; f < 4; ++f) own_cell[q][f * kF] = o[f];
            double ssx, ssy;
            cell_speeds<S, SH>(A, o, ssx, ssy);
            reduce_fold(A, R, o, ssx, ssy);
        }
        // CTA partial (max of non-negative doubles; wet and error bits OR-ed)
        double fl = __longlong_as_double((long long)(R.wet | (errb << 1)));
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            R.sx = smax(R.sx, __shfl_xor_sync(0xffffffffu, R.sx, o));
            R.sy = smax(R.sy, __shfl_xor_sync(0xffffffffu, R.sy, o));
            R.hmax = smax(R.hmax, __shfl_xor_sync(0xffffffffu, R.hmax, o));
            fl = __longlong_as_double(__double_as_longlong(fl) |
                                      __double_as_longlong(__shfl_xor_sync(0xffffffffu, fl, o)));
        }
        if (lane == 0) {
            s_wpart[w][0] = R.sx;
            s_wpart[w][1] = R.sy;
            s_wpart[w][2] = R.hmax;
            s_wpart[w][3] = fl;
        }
        __syncthreads();
        if (w == 0) {
            double a = 0.0, b = 0.0, h = 0.0;
            long long bits = 0;
            if (lane < kCluster1dWarps) {
                a = s_wpart[lane][0];
                b = s_wpart[lane][1];
                h = s_wpart[lane][2];
                bits = __double_as_longlong(s_wpart[lane][3]);
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                a = smax(a, __shfl_xor_sync(0xffffffffu, a, o));
                b = smax(b, __shfl_xor_sync(0xffffffffu, b, o));
                h = smax(h, __shfl_xor_sync(0xffffffffu, h, o));
                bits |= __shfl_xor_sync(0xffffffffu, bits, o);
            }
            if (lane == 0) {
                s_cta[q][0] = a;
                s_cta[q][1] = b;
                s_cta[q][2] = h;
                s_cta[q][3] = __longlong_as_double(bits);
            }
        }
        cl.sync();  // the new line and the CTA partials are visible cluster-wide
        pa = pb = ph = 0.0;
        pbits = 0;
        if (lane < nctas) {
            const double* rp = cl.map_shared_rank(&s_cta[q][0], lane);
            pa = rp[0];
            pb = rp[1];
            ph = rp[2];
            pbits = __double_as_longlong(rp[3]);
        }
        pending = true;
        // the run clock of state n+1 (control_epilogue); its reductions follow
        cur.t = d.t_new;
        cur.steps = cur.steps + 1;
        cur.last_dt = d.dt;
        cur.snap_idx = d.snap_idx;
        cur.state = d.next_state;
    }
    if (pending) fold_partials();
    // state back to HBM (parity of its step count), header into the slot the
    // next launch reads, the one after it cleared for its reductions
    {
        const int p = (int)(cur.steps & 1);
        if (owned)
#pragma unroll
            for (int f = 0; f < 4; ++f) A.state[p][f][col] = own_cell[p][f * kF];
    }
    if (rank == 0 && t == 0) {
        Slot& fin = A.ctl->slot[(li0 + n) % 3];
        fin = cur;
        Slot& clr = A.ctl->slot[(li0 + n + 1) % 3];
        clr.max_sx = clr.max_sy = clr.hmax = 0ull;
        clr.wet = 0u;
        clr.err = 0u;
    }
    cl.sync();  // no CTA leaves while its shared memory may still be read
}

// ---- initial reduction of a state (first cfl_dt + hmax + ghost rows) --------
template <bool S, bool SH>
__global__ void __launch_bounds__(256) reduce_state_kernel(StepArgs A, int li) {
    Slot& s = A.ctl->slot[li % 3];
    const int p = (int)(s.steps & 1);
    Reduce R{0.0, 0.0, 0.0, 0u};
    const long long n = (long long)A.nx * A.ny;
    for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < n;
         k += (long long)gridDim.x * blockDim.x) {
        const int row = (int)(k / A.nx), col = (int)(k % A.nx);
        double c[4];
        load_interior(A, p, col, row, c);
        if (A.write_edges_in_reduce) write_edges(A, p, col, row, c);
        double sx = 0, sy = 0;
        if (c[0] > A.P.h_dry) cell_speeds<S, SH>(A, c, sx, sy);
        reduce_fold(A, R, c, sx, sy);
    }
    reduce_flush(R, s);
}

// ---- batch of interface problems (unit tests / ABI silt_riemann_batch) -------
template <bool S, bool SH>
__global__ void face_batch_kernel(Params P, const double* L, const double* Rr, long long n,
                                  int axis, double* out, unsigned* err) {
    const long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (k >= n) return;
    double l[4], r[4];
    for (int f = 0; f < 4; ++f) {
        l[f] = L[4 * k + f];
        r[f] = Rr[4 * k + f];
    }
    Side sl, sr;
    const int nn = axis == 0 ? 1 : 2, tt = axis == 0 ? 2 : 1;
    if constexpr (S) {
        sl = make_side_ref<SH>(P, l[0], l[nn], l[tt], l[3]);
        sr = make_side_ref<SH>(P, r[0], r[nn], r[tt], r[3]);
    } else {
        const CellPre pl = cell_pre_fast<SH>(P, l[0], l[1], l[2], l[3]);
        const CellPre pr = cell_pre_fast<SH>(P, r[0], r[1], r[2], r[3]);
        sl = make_side_fast<SH>(P, pl, axis == 0);
        sr = make_side_fast<SH>(P, pr, axis == 0);
    }
    Flux F;
    if (!face_flux<S>(P, sl, sr, F)) atomicOr(err, kErrRiemann);
    out[5 * k + 0] = F.h;
    out[5 * k + 1] = F.huL;
    out[5 * k + 2] = F.huR;
    out[5 * k + 3] = F.hv;
    out[5 * k + 4] = F.z;
}

// ---- batch of law evaluations (unit tests / ABI silt_law_batch) -------------
// Each variant evaluates the law the way its step kernels do: STRICT through
// normal_flux_ref / normal_flux_derivative_ref, FAST through the per-cell
// rates + planar terms of make_side_fast.
template <bool S, bool SH>
__global__ void law_batch_kernel(Params P, const double* X, long long n, double* out) {
    const long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (k >= n) return;
    const double h = X[3 * k], un = X[3 * k + 1], ut = X[3 * k + 2];
    double omega, dq;
    if constexpr (S) {
        omega = normal_flux_ref<SH>(P, h, un, ut);
        dq = normal_flux_derivative_ref<SH>(P, h, un, ut);
    } else {
        const double s2 = fma(un, un, ut * ut);
        if constexpr (SH)
            shields_terms_fast(shields_rates_fast(P, h, s2), un, s2, omega, dq);
        else
            grass_terms_fast(P, un, ut, s2, omega, dq);
    }
    out[2 * k] = omega;
    out[2 * k + 1] = dq;
}

}  // namespace silt_dev

#ifdef SILT_CHECKED
#define SILT_DEBUG_CHECKS_BODY                                                                 \
    cudaDeviceSynchronize();                                                                   \
    cudaMemcpyFromSymbol(out, silt_dev::g_check, sizeof(unsigned long long) * 4);              \
    const unsigned long long z[4] = {0, 0, 0, 0};                                              \
    cudaMemcpyToSymbol(silt_dev::g_check, z, sizeof z);                                        \
    return 1;
#else
#define SILT_DEBUG_CHECKS_BODY \
    (void)out;                 \
    return 0;
#endif

// Explicit instantiation hooks, defined by each TU with its own S; the law
// kind (A.P.shields) picks the kernel instantiation at launch.
#define SILT_DEFINE_LAUNCHERS(S, NAME)                                                          \
    template <bool SH>                                                                           \
    static void NAME##_step_t(const StepArgs& A, int li, dim3 grid, cudaStream_t st) {           \
        if (A.dim == 2) {                                                                        \
            /* the attribute is per device: one bit per device ordinal */                       \
            static unsigned long long attr_set = 0;                                              \
            int dev_ = 0;                                                                        \
            cudaGetDevice(&dev_);                                                                \
            if (!(attr_set >> (dev_ & 63) & 1ull)) {                                             \
                cudaFuncSetAttribute(silt_dev::step2d_kernel<S, SH, false>,                      \
                                     cudaFuncAttributeMaxDynamicSharedMemorySize,                \
                                     (int)sizeof(silt_dev::StepSmem));                           \
                cudaFuncSetAttribute(silt_dev::step2d_kernel<S, SH, true>,                       \
                                     cudaFuncAttributeMaxDynamicSharedMemorySize,                \
                                     (int)sizeof(silt_dev::StepSmem));                           \
                /* SILT_CARVEOUT=%: shared-memory carveout preference (A/B) */                  \
                if (const char* cv = std::getenv("SILT_CARVEOUT"))                               \
                    cudaFuncSetAttribute(silt_dev::step2d_kernel<S, SH, false>,                  \
                                         cudaFuncAttributePreferredSharedMemoryCarveout,         \
                                         std::atoi(cv));                                         \
                attr_set |= 1ull << (dev_ & 63);                                                 \
            }                                                                                    \
            if (SILT_PDL) {                                                                      \
                cudaLaunchConfig_t cfg{};                                                        \
                cfg.gridDim = grid;                                                              \
                cfg.blockDim = dim3(kStepThreads);                                               \
                cfg.dynamicSmemBytes = sizeof(silt_dev::StepSmem);                               \
                cfg.stream = st;                                                                 \
                cudaLaunchAttribute at[1];                                                       \
                at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;                   \
                at[0].val.programmaticStreamSerializationAllowed = 1;                            \
                cfg.attrs = at;                                                                  \
                cfg.numAttrs = 1;                                                                \
                StepArgs a_ = A;                                                                 \
                int li_ = li;                                                                    \
                if (A.warp_items)                                                                \
                    cudaLaunchKernelEx(&cfg, silt_dev::step2d_kernel<S, SH, true>, a_, li_);     \
                else                                                                             \
                    cudaLaunchKernelEx(&cfg, silt_dev::step2d_kernel<S, SH, false>, a_, li_);    \
            } else if (A.warp_items)                                                             \
                silt_dev::step2d_kernel<S, SH, true>                                             \
                    <<<grid, kStepThreads, sizeof(silt_dev::StepSmem), st>>>(A, li);             \
            else                                                                                 \
                silt_dev::step2d_kernel<S, SH, false>                                            \
                    <<<grid, kStepThreads, sizeof(silt_dev::StepSmem), st>>>(A, li);             \
        } else                                                                                   \
            silt_dev::step1d_kernel<S, SH><<<grid, kStepThreads, 0, st>>>(A, li);                \
    }                                                                                            \
    void NAME##_step(const StepArgs& A, int li, dim3 grid, cudaStream_t st) {                    \
        if (A.P.shields)                                                                         \
            NAME##_step_t<true>(A, li, grid, st);                                                \
        else                                                                                     \
            NAME##_step_t<false>(A, li, grid, st);                                               \
    }                                                                                            \
    int NAME##_step1d_coop(const StepArgs& A, int li0, int n, dim3 grid, cudaStream_t st) {      \
        StepArgs a = A;                                                                          \
        void* args[] = {&a, &li0, &n};                                                           \
        const void* f = A.P.shields ? (const void*)silt_dev::step1d_coop_kernel<S, true>         \
                                    : (const void*)silt_dev::step1d_coop_kernel<S, false>;       \
        return (int)cudaLaunchCooperativeKernel(f, grid, dim3(kStepThreads), args, 0, st);       \
    }                                                                                            \
    int NAME##_step1d_cluster(const StepArgs& A, int li0, int n, int ctas, cudaStream_t st) {    \
        StepArgs a = A;                                                                          \
        void* args[] = {&a, &li0, &n};                                                           \
        const char* renv = std::getenv("SILT_1D_RESIDENT"); /* per launch: tests switch it */   \
        const int resident_env = renv ? std::atoi(renv) : -1;                                    \
        const bool resident = resident_env >= 0 ? resident_env != 0 : ctas <= silt_dev::kResidentMaxCtas; \
        const void* f =                                                                          \
            resident ? (A.P.shields ? (const void*)silt_dev::step1d_resident_kernel<S, true>     \
                                    : (const void*)silt_dev::step1d_resident_kernel<S, false>)   \
                     : (A.P.shields ? (const void*)silt_dev::step1d_cluster_kernel<S, true>      \
                                    : (const void*)silt_dev::step1d_cluster_kernel<S, false>);   \
        cudaFuncSetAttribute(f, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);              \
        cudaLaunchConfig_t cfg{};                                                                \
        cfg.gridDim = dim3(ctas);                                                                \
        cfg.blockDim = dim3(silt_dev::kCluster1dThreads);                                        \
        cfg.stream = st;                                                                         \
        cudaLaunchAttribute at[1];                                                               \
        at[0].id = cudaLaunchAttributeClusterDimension;                                          \
        at[0].val.clusterDim.x = ctas;                                                           \
        at[0].val.clusterDim.y = 1;                                                              \
        at[0].val.clusterDim.z = 1;                                                              \
        cfg.attrs = at;                                                                          \
        cfg.numAttrs = 1;                                                                        \
        return (int)cudaLaunchKernelExC(&cfg, f, args);                                          \
    }                                                                                            \
    int NAME##_debug_checks(unsigned long long* out) {                                           \
        SILT_DEBUG_CHECKS_BODY                                                                   \
    }                                                                                            \
    int NAME##_step2d_ctas_per_sm(int shields) {                                                 \
        const void* f = shields ? (const void*)silt_dev::step2d_kernel<S, true>                  \
                                : (const void*)silt_dev::step2d_kernel<S, false>;                \
        cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize,                     \
                             (int)sizeof(silt_dev::StepSmem));                                   \
        int per_sm = 0;                                                                          \
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, f, kStepThreads,              \
                                                          sizeof(silt_dev::StepSmem)) != cudaSuccess) \
            per_sm = 0;                                                                          \
        return per_sm;                                                                           \
    }                                                                                            \
    int NAME##_step1d_coop_blocks(int shields) {                                                 \
        int per_sm = 0, sms = 0, dev = 0;                                                        \
        cudaGetDevice(&dev);                                                                     \
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);                       \
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(                                           \
            &per_sm,                                                                             \
            shields ? silt_dev::step1d_coop_kernel<S, true> : silt_dev::step1d_coop_kernel<S, false>, \
            kStepThreads, 0);                                                                    \
        return per_sm * sms;                                                                     \
    }                                                                                            \
    void NAME##_reduce(const StepArgs& A, int li, int blocks, cudaStream_t st) {                 \
        if (A.P.shields)                                                                         \
            silt_dev::reduce_state_kernel<S, true><<<blocks, 256, 0, st>>>(A, li);               \
        else                                                                                     \
            silt_dev::reduce_state_kernel<S, false><<<blocks, 256, 0, st>>>(A, li);              \
    }                                                                                            \
    void NAME##_faces(const silt_dev::Params& P, const double* L, const double* R, long long n,  \
                      int axis, double* out, unsigned* err, cudaStream_t st) {                   \
        const int b = 128;                                                                       \
        const unsigned g = (unsigned)((n + b - 1) / b);                                          \
        if (P.shields)                                                                           \
            silt_dev::face_batch_kernel<S, true><<<g, b, 0, st>>>(P, L, R, n, axis, out, err);   \
        else                                                                                     \
            silt_dev::face_batch_kernel<S, false><<<g, b, 0, st>>>(P, L, R, n, axis, out, err);  \
    }                                                                                            \
    void NAME##_law(const silt_dev::Params& P, const double* X, long long n, double* out,        \
                    cudaStream_t st) {                                                           \
        const unsigned g = (unsigned)((n + 127) / 128);                                          \
        if (P.shields)                                                                           \
            silt_dev::law_batch_kernel<S, true><<<g, 128, 0, st>>>(P, X, n, out);                \
        else                                                                                     \
            silt_dev::law_batch_kernel<S, false><<<g, 128, 0, st>>>(P, X, n, out);               \
    }
