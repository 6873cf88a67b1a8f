// silt_capi.cu — host runtime behind include/silt_cuda.h.
//
// Owns device memory (SoA ping-pong planes, ghost rows, the Control block),
// validates problems with the reference's messages, enqueues the fused step
// kernels on the solver's stream and maps device error words back onto the
// reference's exception classes (status codes SILT_ERR_INVALID ~
// std::invalid_argument, SILT_ERR_RUNTIME ~ std::runtime_error).
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include <map>
#include <memory>
#include <mutex>
#include <thread>

#include "silt_csv_launch.h"
#include "silt_cuda.h"
#include "silt_launch.h"
#include "silt_layout.h"

namespace {
void ipc_close(void* p);          // IPC registry (multi-process strips), defined below
void ipc_forget_local(void* p);
}  // namespace

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
    g_err = msg;
    return code;
}

#define CUDA_TRY(expr)                                                                        \
    do {                                                                                      \
        cudaError_t e_ = (expr);                                                              \
        if (e_ != cudaSuccess)                                                                \
            return fail(SILT_ERR_CUDA, std::string(#expr ": ") + cudaGetErrorString(e_));     \
    } while (0)

__global__ void aos_to_soa(const double* __restrict__ aos, double* h, double* hu, double* hv,
                           double* zb, int nx, int ny, int pitch) {
    const long long n = (long long)nx * ny;
    for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < n;
         k += (long long)gridDim.x * blockDim.x) {
        const double4 c = reinterpret_cast<const double4*>(aos)[k];
        const long long off = (k / nx) * pitch + (k % nx);
        h[off] = c.x;
        hu[off] = c.y;
        hv[off] = c.z;
        zb[off] = c.w;
    }
}

__global__ void soa_to_aos(double* __restrict__ aos, const double* h, const double* hu,
                           const double* hv, const double* zb, int nx, int ny, int pitch) {
    const long long n = (long long)nx * ny;
    for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < n;
         k += (long long)gridDim.x * blockDim.x) {
        const long long off = (k / nx) * pitch + (k % nx);
        reinterpret_cast<double4*>(aos)[k] = make_double4(h[off], hu[off], hv[off], zb[off]);
    }
}

// AoS ghost cells (n cells) -> [4][n] planes
__global__ void aos_to_planes(const double* __restrict__ aos, double* planes, int n) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    for (int f = 0; f < 4; ++f) planes[(size_t)f * n + k] = aos[4 * (size_t)k + f];
}

// Next launch's row-block order from the hot flags of the launch just
// enqueued (one CTA; the flags are cleared for reuse).  Hot row blocks go to
// positions floor((h + 1/2) span / H), span = 0.9 nb, the others fill the
// remaining positions in row order; without usable information (no hot
// block, or more than span / 2) the default order is copied.
__global__ void __launch_bounds__(1024) rb_order_kernel(unsigned char* hot, const int* def,
                                                        int* lists, int* out, int nb,
                                                        int span_permille) {
    __shared__ int s_warp[32];
    __shared__ int s_base[2];
    const int t = threadIdx.x, lane = t & 31, w = t >> 5;
    if (t == 0) s_base[0] = s_base[1] = 0;
    __syncthreads();
    int* hot_list = lists;
    int* cold_list = lists + nb;
    for (int k0 = 0; k0 < nb; k0 += 1024) {
        const int k = k0 + t;
        const int f = (k < nb && hot[k]) ? 1 : 0;
        // exclusive block scan of f
        const unsigned bal = __ballot_sync(0xffffffffu, f);
        const int in_warp = __popc(bal & ((1u << lane) - 1u));
        if (lane == 31) s_warp[w] = in_warp + f;
        __syncthreads();
        if (w == 0) {
            const int v = s_warp[lane];
            int x = v;
            for (int d = 1; d < 32; d <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, x, d);
                if (lane >= d) x += y;
            }
            s_warp[lane] = x - v;  // exclusive
        }
        __syncthreads();
        const int hr = s_base[0] + s_warp[w] + in_warp;  // hot rank
        if (k < nb) {
            if (f)
                hot_list[hr] = k;
            else
                cold_list[k - hr] = k;
            hot[k] = 0;
        }
        __syncthreads();
        if (t == 1023) s_base[0] = hr + f;
        __syncthreads();
    }
    const long long H = s_base[0];
    const long long span = (long long)nb * span_permille / 1000;
    const bool use = H > 0 && 2 * H <= span;
    for (int k = t; k < nb; k += 1024) {
        if (!use) {
            out[k] = def[k];
            continue;
        }
        // hot positions before k: #{h : (2h + 1) span < 2 k H}
        auto before = [&](long long kk) {
            const long long num = 2 * kk * H - span;
            if (num <= 0) return 0LL;
            const long long c = (num + 2 * span - 1) / (2 * span);
            return c < H ? c : H;
        };
        const long long lt = before(k), le = before(k + 1);
        out[k] = (le > lt) ? hot_list[lt] : cold_list[k - lt];
    }
}

int grid_blocks(long long n, int threads) {
    long long b = (n + threads - 1) / threads;
    return (int)std::max(1LL, std::min(b, 148LL * 32));
}

const char* kNegDepthMsg =
    "step: negative depth produced; time step or celerities violate stability";

}  // namespace

struct silt_solver {
    silt_problem prob{};
    silt_strip strip{};
    int device = 0;
    int variant = SILT_VARIANT_FAST;
    int nx = 0, ny = 0, pitch = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    double* planes = nullptr;   // [2][4][ny][pitch]
    double* rows = nullptr;     // 8 x [4][nx]
    double* cols = nullptr;     // 2 x [4][ny]
    double* staging = nullptr;  // AoS nx*ny*4
    double* snapbuf = nullptr;  // AoS nx*ny*4: device copy of a captured snapshot
    void* rb_mem = nullptr;     // row-block order: default, lists, 3 tables, 3 hot flags
    int* rb_default = nullptr;
    int* rb_lists = nullptr;
    int* split_map = nullptr;   // {0, nb-1, 1, 2, ..., nb-2}: edge and interior row blocks
    int row_blocks = 0;
    int rb_span = 900;          // hot row blocks spread over this share (per mille) of a launch
    int coop_blocks = -1;       // 1D: co-resident CTAs of the cooperative step kernel (-1: unknown)
    // multi-process peer-memory exchange (silt_solver_p2p_*)
    unsigned* p2p_flags = nullptr;       // [64]: step count of every rank (written by the ranks)
    int p2p_rank = -1, p2p_world = 0;
    unsigned p2p_count = 0;              // steps taken through silt_solver_p2p_step
    bool begun_after_connect = false;    // the run's initial rows went to the peers
    std::vector<void*> p2p_opened;       // IPC mappings to close
    std::vector<unsigned*> p2p_peer_flag;  // per other rank: &their_flags[p2p_rank]
    unsigned** p2p_peer_flag_dev = nullptr;  // the same, device array
    Control** p2p_peer_ctl = nullptr;    // device array: the other ranks' Control
    bool cluster_failed = false;  // 1D: the cluster launch was refused once
    cudaStream_t copy_stream = nullptr;  // snapshot D2H, overlapping the next steps
    cudaEvent_t cap_ready = nullptr, cap_done = nullptr;
    bool cap_pending = false;
    std::thread writer;         // asynchronous CSV snapshot (silt_solver_capture_write)
    std::atomic<bool> writer_busy{false};  // set by capture_write, cleared by the thread
    int writer_rc = SILT_OK;
    std::string writer_err;
    Control* ctl = nullptr;
    Control* host_ctl = nullptr;  // pinned staging for control uploads
    double* dt_log = nullptr;
    int64_t dt_cap = 0;
    double* snaps = nullptr;
    int n_snaps_alloc = 0;
    int64_t launches = 0;
    int64_t kernel_count = 0;
    bool begun = false;
    StepArgs args{};
    dim3 step_grid;
    dim3 row_grid;  // the launch grid (column groups x row blocks), also in warp-item mode
    // WorkerTiming split (silt_solver_timing): device time of this strip's
    // step launches, bracketed by events and harvested when the stream syncs
    bool timing_on = false;
    std::vector<cudaEvent_t> tev_free;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> tev_pending;
    double compute_s = 0;
};

namespace {
// Event bracket around this strip's step work (timing builds of run_parallel's
// WorkerTiming.compute_seconds); no-op unless silt_solver_timing enabled it.
cudaEvent_t timing_mark(silt_solver* s) {
    if (!s->timing_on) return nullptr;
    cudaEvent_t e = nullptr;
    if (!s->tev_free.empty()) {
        e = s->tev_free.back();
        s->tev_free.pop_back();
    } else if (cudaEventCreate(&e) != cudaSuccess) {
        return nullptr;
    }
    cudaEventRecord(e, s->stream);
    return e;
}

void timing_close(silt_solver* s, cudaEvent_t start) {
    if (!start) return;
    cudaEvent_t end = timing_mark(s);
    if (!end) {
        s->tev_free.push_back(start);
        return;
    }
    s->tev_pending.emplace_back(start, end);
}

// After a stream synchronisation: fold the completed brackets into compute_s.
void timing_harvest(silt_solver* s) {
    for (auto& pr : s->tev_pending) {
        float ms = 0.f;
        if (cudaEventElapsedTime(&ms, pr.first, pr.second) == cudaSuccess) s->compute_s += 1e-3 * ms;
        s->tev_free.push_back(pr.first);
        s->tev_free.push_back(pr.second);
    }
    s->tev_pending.clear();
}
}  // namespace

namespace {

// Device parameters of a validated problem.  Shields constants are evaluated
// in the reference's operation order (src/bedload.cpp:152, :161) so the STRICT
// kernels see the same doubles.
silt_dev::Params make_params(const silt_problem& p) {
    silt_dev::Params P{};
    P.g = p.gravity;
    P.h_dry = p.h_dry;
    P.a_g = p.a_g;
    P.m_g = p.m_g;
    P.safety = p.safety;
    P.half_g = 0.5 * p.gravity;
    P.m3 = p.m_g == 3.0;
    P.shields = p.law_kind == SILT_LAW_SHIELDS;
    if (P.shields) {
        P.formula = p.shields_formula;
        P.friction = p.friction_model;
        P.tau_cr = p.tau_cr;
        P.d_s = p.grain_diameter;
        P.rel_density = p.rel_density;
        P.fcoef = p.friction_coef;
        const double d = p.grain_diameter;
        P.scale = std::sqrt((p.rel_density - 1.0) * p.gravity * d * d * d);
        const double sd = (p.rel_density - 1.0) * d;
        P.ktau = p.friction_model == SILT_FRICTION_MANNING
                     ? p.friction_coef * p.friction_coef / sd
                     : p.friction_coef / (8.0 * p.gravity * sd);
    }
    return P;
}

int validate_problem(const silt_problem* p) {
    if (!p) return fail(SILT_ERR_INVALID, "silt: null problem");
    if (p->dim != 1 && p->dim != 2) return fail(SILT_ERR_INVALID, "grid: dim must be 1 or 2");
    if (p->nx < 1) return fail(SILT_ERR_INVALID, "grid: cell count nx must be >= 1");
    if (p->dim == 2 && p->ny < 1) return fail(SILT_ERR_INVALID, "grid: cell count ny must be >= 1");
    if (!(p->dx > 0) || !std::isfinite(p->dx))
        return fail(SILT_ERR_INVALID, "grid: length_x must be positive");
    if (p->dim == 2 && (!(p->dy > 0) || !std::isfinite(p->dy)))
        return fail(SILT_ERR_INVALID, "grid: length_y must be positive");
    if (p->law_kind == SILT_LAW_GRASS) {  // BedloadLaw::grass, src/bedload.cpp:26-36
        if (!(p->a_g >= 0) || !std::isfinite(p->a_g))
            return fail(SILT_ERR_INVALID, "bedload: Grass a_g must be >= 0");
        if (!(p->m_g >= 1.0 && p->m_g <= 4.0))
            return fail(SILT_ERR_INVALID, "bedload: Grass m_g must lie in [1, 4]");
    } else if (p->law_kind == SILT_LAW_SHIELDS) {  // BedloadLaw::shields, :38-57
        if (p->shields_formula < SILT_SHIELDS_MPM || p->shields_formula > SILT_SHIELDS_CAMENEN)
            return fail(SILT_ERR_INVALID, "bedload: unknown Shields formula");
        if (p->friction_model != SILT_FRICTION_DARCY_WEISBACH &&
            p->friction_model != SILT_FRICTION_MANNING)
            return fail(SILT_ERR_INVALID, "bedload: unknown friction model");
        if (!(p->tau_cr >= 0)) return fail(SILT_ERR_INVALID, "bedload: tau_cr must be >= 0");
        if (!(p->grain_diameter > 0))
            return fail(SILT_ERR_INVALID, "bedload: grain diameter must be > 0");
        if (!(p->rel_density > 1))
            return fail(SILT_ERR_INVALID, "bedload: relative density must exceed 1");
        if (!(p->friction_coef > 0))
            return fail(SILT_ERR_INVALID, "bedload: friction coefficient must be > 0");
    } else {
        return fail(SILT_ERR_INVALID, "bedload: unknown law kind");
    }
    const bool px0 = p->bc[SILT_WEST].type == SILT_BC_PERIODIC;
    const bool px1 = p->bc[SILT_EAST].type == SILT_BC_PERIODIC;
    if (px0 != px1) return fail(SILT_ERR_INVALID, "apply_bcs: periodic requires both x sides");
    if (p->dim == 2) {
        const bool py0 = p->bc[SILT_SOUTH].type == SILT_BC_PERIODIC;
        const bool py1 = p->bc[SILT_NORTH].type == SILT_BC_PERIODIC;
        if (py0 != py1) return fail(SILT_ERR_INVALID, "apply_bcs: periodic requires both y sides");
    }
    for (int s = 0; s < 4; ++s)
        if (p->bc[s].type < SILT_BC_INFLOW || p->bc[s].type > SILT_BC_GIVEN)
            return fail(SILT_ERR_INVALID, "silt: unknown boundary type");
    return SILT_OK;
}

int check_cfl(double cfl) {
    if (!(cfl > 0) || !(cfl <= 1)) return fail(SILT_ERR_INVALID, "cfl_dt: cfl must lie in (0, 1]");
    return SILT_OK;
}

#ifndef SILT_WAVE_R
#define SILT_WAVE_R 48
#endif
#ifndef SILT_WAVE_DOWN
#define SILT_WAVE_DOWN 8
#endif

// part 0: the whole step; 1: the two boundary row blocks of a split step;
// 2: its interior row blocks (and the end of the step).
void launch_step(silt_solver* s, int part = 0) {
    const cudaEvent_t t0 = timing_mark(s);
    struct Close {
        silt_solver* s;
        cudaEvent_t t0;
        ~Close() { timing_close(s, t0); }
    } close_{s, t0};
    const int li = (int)(s->launches % 3);
    StepArgs a = s->args;
    dim3 grid = s->step_grid;
    if (part == 0) {
        a.rb_map = a.rb_order ? a.rb_table[li] : nullptr;
    } else {
        // split edge / interior launches: always on the launch grid
        grid = s->row_grid;
        a.warp_items = 0;
        a.rb_map = part == 1 ? s->split_map : s->split_map + 2;
        a.epilogue = part == 1 ? 1 : 0;
        grid.y = part == 1 ? 2u : grid.y - 2u;
    }
    if (s->variant == SILT_VARIANT_STRICT)
        silt_strict_step(a, li, grid, s->stream);
    else
        silt_fast_step(a, li, grid, s->stream);
    ++s->kernel_count;
    if (part == 1) return;
    ++s->launches;
    if (s->args.rb_order) {
        rb_order_kernel<<<1, 1024, 0, s->stream>>>(s->args.rb_hot[li], s->rb_default, s->rb_lists,
                                                   s->args.rb_table[(li + 1) % 3], s->row_blocks,
                                                   s->rb_span);
        ++s->kernel_count;
    }
}

int read_slot(silt_solver* s, Slot* out, Control* full) {
    CUDA_TRY(cudaSetDevice(s->device));
    CUDA_TRY(cudaStreamSynchronize(s->stream));
    CUDA_TRY(cudaGetLastError());
    timing_harvest(s);
    if (full) {
        CUDA_TRY(cudaMemcpy(full, s->ctl, sizeof(Control), cudaMemcpyDeviceToHost));
        *out = full->slot[s->launches % 3];
    } else {
        CUDA_TRY(cudaMemcpy(out, &s->ctl->slot[s->launches % 3], sizeof(Slot),
                            cudaMemcpyDeviceToHost));
    }
    return SILT_OK;
}

int error_from(const Control& c, unsigned bits) {
    if (bits & silt_dev::kErrRiemann) {
        char buf[512];
        std::snprintf(buf, sizeof buf,
                      "interface_riemann: no positive fan after 25 celerity enlargements "
                      "(hL=%g uL=%g zL=%g | hR=%g uR=%g zR=%g)",
                      c.err_info[0], c.err_info[1], c.err_info[2], c.err_info[3], c.err_info[4],
                      c.err_info[5]);
        return fail(SILT_ERR_RUNTIME, buf);
    }
    if (bits & silt_dev::kErrNegDepth) return fail(SILT_ERR_RUNTIME, kNegDepthMsg);
    if (bits & silt_dev::kErrDry) return fail(SILT_ERR_INVALID, "cfl_dt: field is entirely dry");
    if (bits & silt_dev::kErrPeer) {
        char buf[256];
        std::snprintf(buf, sizeof buf,
                      "p2p: rank %d did not publish step %d within the peer timeout "
                      "(SILT_P2P_TIMEOUT_MS); the peer process died or hung",
                      c.err_col, c.err_row);
        return fail(SILT_ERR_RUNTIME, buf);
    }

    return fail(SILT_ERR_RUNTIME, "step: device error");
}

}  // namespace

extern "C" {

int silt_abi_version(void) { return SILT_ABI_VERSION; }

// Diagnostics (not part of the drop-in API): bounds-check counters of a
// -DSILT_CHECKED build, summed over both variants' kernels, then reset.
// out[4] = {violations, first code, first a, first b}; returns 1 in a checked
// build, 0 otherwise (counters then stay 0).
int silt_debug_checks(unsigned long long* out) {
    unsigned long long a[4] = {0, 0, 0, 0}, b[4] = {0, 0, 0, 0};
    const int ca = silt_fast_debug_checks(a);
    const int cb = silt_strict_debug_checks(b);
    if (out) {
        out[0] = a[0] + b[0];
        const unsigned long long* first = a[0] ? a : b;
        for (int k = 1; k < 4; ++k) out[k] = first[k];
    }
    return ca | cb;
}

int silt_abi_sizes(int64_t* sizes, int n) {
    const int64_t all[6] = {sizeof(silt_bc),       sizeof(silt_problem), sizeof(silt_strip),
                            sizeof(silt_run_plan), sizeof(silt_status),  sizeof(silt_exchange)};
    for (int k = 0; k < n && k < 6; ++k) sizes[k] = all[k];
    return SILT_OK;
}

const char* silt_last_error(void) { return g_err.c_str(); }

int silt_device_count(int* count) {
    CUDA_TRY(cudaGetDeviceCount(count));
    return SILT_OK;
}

int silt_solver_create(const silt_problem* problem, const silt_strip* strip, int device,
                       int variant, silt_solver** out) {
    if (!out) return fail(SILT_ERR_INVALID, "silt_solver_create: null out");
    *out = nullptr;
    if (int rc = validate_problem(problem)) return rc;
    if (variant != SILT_VARIANT_FAST && variant != SILT_VARIANT_STRICT)
        return fail(SILT_ERR_INVALID, "silt_solver_create: unknown variant");
    const int gny = problem->dim == 1 ? 1 : problem->ny;
    silt_strip st{0, gny, 0, 0};
    if (strip) st = *strip;
    if (st.ny_local < 1 || st.j0 < 0 || st.j0 + st.ny_local > gny)
        return fail(SILT_ERR_INVALID, "partition: every worker needs at least one cell per axis");
    if (problem->dim == 1 && (st.south_neighbor || st.north_neighbor || st.ny_local != 1))
        return fail(SILT_ERR_INVALID, "partition: 1D grids require py == 1");
    int ndev = 0;
    CUDA_TRY(cudaGetDeviceCount(&ndev));
    if (device < 0 || device >= ndev) return fail(SILT_ERR_CUDA, "silt_solver_create: bad device");
    CUDA_TRY(cudaSetDevice(device));

    silt_solver* s = new silt_solver();
    s->prob = *problem;
    s->prob.ny = gny;
    s->strip = st;
    s->device = device;
    s->variant = variant;
    s->nx = problem->nx;
    s->ny = st.ny_local;
    s->pitch = (s->nx + 31) / 32 * 32;
    const size_t plane = (size_t)s->ny * s->pitch;
    auto cleanup = [&](int rc) {
        silt_solver_destroy(s);
        return rc;
    };
    if (cudaStreamCreateWithFlags(&s->stream, cudaStreamNonBlocking) != cudaSuccess)
        return cleanup(fail(SILT_ERR_CUDA, "cudaStreamCreate failed"));
    s->own_stream = true;
    if (cudaMalloc(&s->planes, 8 * plane * sizeof(double)) != cudaSuccess ||
        cudaMalloc(&s->rows, 10 * 4 * (size_t)s->nx * sizeof(double)) != cudaSuccess ||
        cudaMalloc(&s->cols, 2 * 4 * (size_t)s->ny * sizeof(double)) != cudaSuccess ||
        cudaMalloc(&s->ctl, sizeof(Control)) != cudaSuccess ||
        cudaMallocHost(&s->host_ctl, sizeof(Control)) != cudaSuccess)
        return cleanup(fail(SILT_ERR_CUDA, "silt_solver_create: device allocation failed"));
    cudaMemset(s->planes, 0, 8 * plane * sizeof(double));
    cudaMemset(s->rows, 0, 10 * 4 * (size_t)s->nx * sizeof(double));
    cudaMemset(s->cols, 0, 2 * 4 * (size_t)s->ny * sizeof(double));
    cudaMemset(s->ctl, 0, sizeof(Control));

    StepArgs& A = s->args;
    A.dim = problem->dim;
    A.nx = s->nx;
    A.ny = s->ny;
    A.pitch = s->pitch;
    A.j0 = st.j0;
    A.south_nbr = st.south_neighbor;
    A.north_nbr = st.north_neighbor;
    A.per_y_self = problem->dim == 2 && problem->bc[SILT_SOUTH].type == SILT_BC_PERIODIC &&
                   !st.south_neighbor && !st.north_neighbor;
    {
        const char* q = std::getenv("SILT_QUIET_SKIP");
        A.quiet_skip = (q && q[0] == '0') ? 0 : 1;
    }
    A.dx = problem->dx;
    A.dy = problem->dim == 1 ? 1.0 : problem->dy;
    A.cfl = problem->cfl;
    A.P = make_params(*problem);
    for (int k = 0; k < 4; ++k) {
        A.bc_type[k] = problem->bc[k].type;
        A.bc_super[k] = problem->bc[k].supercritical;
        A.bc_q0[k] = problem->bc[k].q0;
        A.bc_h0[k] = problem->bc[k].h0;
    }
    for (int p = 0; p < 2; ++p)
        for (int f = 0; f < 4; ++f) A.state[p][f] = s->planes + (size_t)(p * 4 + f) * plane;
    A.plane = (long long)plane;
    const size_t row = 4 * (size_t)s->nx;
    A.ghost_s[0] = s->rows + 0 * row;
    A.ghost_s[1] = s->rows + 1 * row;
    A.ghost_n[0] = s->rows + 2 * row;
    A.ghost_n[1] = s->rows + 3 * row;
    // single-buffered exchange rows (rows 8, 9: the second recv parity of the
    // group's direct mode)
    A.recv_s[0] = A.recv_s[1] = s->rows + 4 * row;
    A.recv_n[0] = A.recv_n[1] = s->rows + 5 * row;
    A.send_s[0] = A.send_s[1] = s->rows + 6 * row;
    A.send_n[0] = A.send_n[1] = s->rows + 7 * row;
    A.ghost_w = s->cols;
    A.ghost_e = s->cols + 4 * (size_t)s->ny;
    A.ctl = s->ctl;
    // resident step CTAs per SM of this variant and law (occupancy of the
    // 2D kernel with its dynamic shared memory; 3 for both variants today)
    int ctas_per_sm = 3;
    if (problem->dim == 2) {
        const int q = variant == SILT_VARIANT_STRICT
                          ? silt_strict_step2d_ctas_per_sm(problem->law_kind == SILT_LAW_SHIELDS)
                          : silt_fast_step2d_ctas_per_sm(problem->law_kind == SILT_LAW_SHIELDS);
        if (q > 0) ctas_per_sm = q;
    }
    // rows per CTA: enough warps in flight for a fp64-latency-bound kernel
    const long long strips = (s->nx + kCellsPerWarp - 1) / kCellsPerWarp;
    long long R = (strips * s->ny + 16383) / 16384;  // C4s: 34, C4: 96 (capped), measured best
    R = std::max(8LL, std::min(96LL, R));  // 96: measured best for C4 and Q; 8: C3 (+8 % over 4)
    if (R >= 32) R -= R % 16;              // C5: 64 (not 69), C4s: 32
    if (R < SILT_WAVE_R && problem->dim == 2) {
        // Short launches (a few waves of CTAs): the last wave's empty slots
        // are a visible tail, so pick the rows per block in R-8..R+4 whose CTA
        // count comes closest below a whole number of waves (3 CTAs per SM).
        // C3 (1024^2): 7 rows, 2.98 waves — 12.5 -> 12.75 G cell-updates/s;
        // C4s (4096^2): 25 rows, 12.9 waves — 0.263 -> 0.257 ms per step.
        int nsm = 148;
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, device);
        const double slots = (double)ctas_per_sm * nsm;
        const long long cols = (strips + kStepThreads / 32 - 1) / (kStepThreads / 32);
        auto waste = [&](long long r) {
            const double w = (double)(((long long)s->ny + r - 1) / r * cols) / slots;
            return std::ceil(w) - w;
        };
        long long best = R;
        for (long long cand = std::max(6LL, R - SILT_WAVE_DOWN); cand <= R + 4; ++cand)
            if (waste(cand) < waste(best) - 0.05) best = cand;
        R = best;
    }
    // Long launches (those the row-block order below applies to) run as warp
    // items too (FAST: warps pull (band, row block) items through the order
    // table, no CTA start-up per block and no warp slot held by a finished
    // warp of a hot CTA) with row blocks of at most 64 rows: C4 3.004 ->
    // 2.958 ms per step (20 steps; ~neutral over 500 steps, where the faster
    // kernel meets the power cap), the uniform field unchanged, a 2-strip
    // half 1.526 -> 1.497 ms.  STRICT: see below.
    const char* wi_env = std::getenv("SILT_WARP_ITEMS");
    {
        int nsm = 148;
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, device);
        const long long nb0 = (s->ny + R - 1) / R;
        const long long ctas0 = nb0 * ((strips + kStepThreads / 32 - 1) / (kStepThreads / 32));
        const char* pe = std::getenv("SILT_ROW_PERM");
        const bool order0 = problem->dim == 2 && nb0 >= 16 && (pe ? pe[0] != '0' : ctas0 >= 64LL * nsm);
        if (order0 && !(wi_env && wi_env[0] == '0')) {
            if (variant == SILT_VARIANT_STRICT) {
                // STRICT skips a repeated row only after three full rows at
                // the start of every row block (its repeated-row skip needs
                // four equal rows and a computed one to repeat), so long
                // blocks: C4 8.74 (64 rows) / 8.07 (128) / 7.45 (256) /
                // 9.04 (384, hot blocks become the tail) ms per step.  At 256
                // rows C4 is 64 x 137 CTAs, below the ordered-launch size:
                // the launch grid in row order (forcing the order table,
                // with or without warp items: 8.35 ms over 100 steps).
                R = 256;
                while (R > 64 && (s->ny + R - 1) / R < 16) R /= 2;
            } else {
                R = std::min(R, 64LL);
            }
        }
    }
    if (const char* e = std::getenv("SILT_ROWS")) R = std::max(1LL, std::atoll(e));
    if (problem->dim == 1) R = 1;
    A.rows_per_block = (int)R;
    const int warps_per_cta = kStepThreads / 32;
    // 2D row-block launch order (long launches only: >= 64 CTAs per SM; in
    // short ones the reordering costs the row-halo sharing in L2 and buys
    // nothing).  Blocks are issued row block by row block, columns fastest
    // (x-halo sharing in L2).  A row block that does full-path work holds its
    // SM slots ~10x longer than a quiescent one, so the order spreads the
    // "hot" row blocks of the previous launch evenly over the first 90 % of
    // the launch: no window in which compute-bound blocks starve the
    // memory-bound ones, and none left to start at the end (the tail).
    // Without hot information the order is 8 interleaved passes (every 8th
    // row block per pass).  rb_order_kernel rebuilds the order after every
    // step from the hot flags the step kernel sets.
    {
        const unsigned nb = (unsigned)((s->ny + R - 1) / R);
        const long long ctas = (long long)nb * ((strips + warps_per_cta - 1) / warps_per_cta);
        int sms = 148;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
        const char* e = std::getenv("SILT_ROW_PERM");
        const bool order = problem->dim == 2 && nb >= 16 && (e ? e[0] != '0' : ctas >= 64LL * sms);
        s->step_grid = dim3((unsigned)((strips + warps_per_cta - 1) / warps_per_cta), nb, 1);
        s->row_grid = s->step_grid;
        A.rb_order = order ? 1 : 0;
        A.epilogue = 1;
        A.rb_map = nullptr;
        // Warp-item mode for short 2D launches (a few waves of CTAs, e.g. C3)
        // and long ordered ones (C4): one wave of resident CTAs whose warps
        // pull (band, row block) items from a counter.  The split edge /
        // interior launches of the collective multi-rank path keep the launch
        // grid (launch_step).  SILT_WARP_ITEMS=0/1 forces it off/on.
        A.warp_items = 0;
        A.bands = (int)strips;
        A.n_items = (int)(strips * nb);
        A.warps_total = 0;
        {
            const double waves = (double)ctas / ((double)ctas_per_sm * sms);
            const char* we = std::getenv("SILT_WARP_ITEMS");
            // (short launches of strips with neighbours keep the grid: the
            // hot piece of a two-piece rank at N = 8 measured 0.424 -> 0.460 ms)
            const bool neighbours = st.south_neighbor || st.north_neighbor;
            bool wi = problem->dim == 2 && (order || (waves <= 8.0 && waves > 1.0 && !neighbours));
            if (we) wi = problem->dim == 2 && we[0] == '1';
            if (wi) {
                const unsigned grid = (unsigned)std::min<long long>(
                    ctas, (long long)ctas_per_sm * sms);
                s->step_grid = dim3(grid, 1, 1);
                A.warp_items = 1;
                A.warps_total = (int)grid * warps_per_cta;
            }
        }
        if (!order && problem->dim == 2 && nb >= 3 && (st.south_neighbor || st.north_neighbor)) {
            std::vector<int> m{0, (int)nb - 1};
            for (unsigned k = 1; k + 1 < nb; ++k) m.push_back((int)k);
            if (cudaMalloc(&s->split_map, m.size() * sizeof(int)) != cudaSuccess)
                return cleanup(fail(SILT_ERR_CUDA, "silt_solver_create: device allocation failed"));
            cudaMemcpy(s->split_map, m.data(), m.size() * sizeof(int), cudaMemcpyHostToDevice);
        }
        // A hot row block must still finish inside the launch: the shorter the
        // launch (in waves of 3 CTAs per SM), the earlier the last one starts.
        // 1 - 6.5 / waves: C4 on one GPU (53 waves) 0.88, its 2-strip halves
        // (26 waves) 0.75 — measured best 0.85-0.90 and 0.60-0.75.
        {
            const double waves = (double)ctas / ((double)ctas_per_sm * sms);
            s->rb_span = (int)std::max(500.0, std::min(900.0, 1000.0 * (1.0 - 6.5 / waves)));
        }
        if (const char* es = std::getenv("SILT_RB_SPAN")) s->rb_span = std::max(100, std::min(1000, std::atoi(es)));
        s->row_blocks = (int)nb;
        if (order) {
            // default (no hot information): 8 interleaved passes for the
            // launch grid; in order for warp items (whose warps stream
            // through the row blocks one after another: the halo rows of
            // neighbouring blocks are still in L2)
            std::vector<int> def;
            if (A.warp_items) {
                for (unsigned y = 0; y < nb; ++y) def.push_back((int)y);
            } else {
                for (unsigned z = 0; z < 8; ++z)
                    for (unsigned y = z; y < nb; y += 8) def.push_back((int)y);
            }
            if (cudaMalloc(&s->rb_mem, (4 + 2 * 3) * (size_t)nb * sizeof(int) + 3 * (size_t)nb) !=
                cudaSuccess)
                return cleanup(fail(SILT_ERR_CUDA, "silt_solver_create: device allocation failed"));
            int* base = static_cast<int*>(s->rb_mem);
            s->rb_default = base;
            s->rb_lists = base + nb;  // hot list, cold list (scratch of the order kernel)
            for (int k = 0; k < 3; ++k) A.rb_table[k] = base + (size_t)(3 + k) * nb;
            unsigned char* hot = reinterpret_cast<unsigned char*>(base + (size_t)6 * nb);
            for (int k = 0; k < 3; ++k) A.rb_hot[k] = hot + (size_t)k * nb;
            cudaMemset(hot, 0, 3 * (size_t)nb);
            for (int k = -1; k < 3; ++k)
                cudaMemcpy(k < 0 ? s->rb_default : A.rb_table[k], def.data(), nb * sizeof(int),
                           cudaMemcpyHostToDevice);
        }
    }
    if (cudaDeviceSynchronize() != cudaSuccess)
        return cleanup(fail(SILT_ERR_CUDA, "silt_solver_create: init failed"));
    *out = s;
    return SILT_OK;
}

int silt_solver_destroy(silt_solver* s) {
    if (!s) return SILT_OK;
    if (s->writer.joinable()) s->writer.join();
    cudaSetDevice(s->device);
    if (s->stream) cudaStreamSynchronize(s->stream);
    if (s->copy_stream) {
        cudaStreamSynchronize(s->copy_stream);
        cudaStreamDestroy(s->copy_stream);
    }
    if (s->cap_ready) cudaEventDestroy(s->cap_ready);
    if (s->cap_done) cudaEventDestroy(s->cap_done);
    cudaFree(s->snapbuf);
    cudaFree(s->rb_mem);
    cudaFree(s->split_map);
    for (void* p : s->p2p_opened) ipc_close(p);
    for (void* p : {(void*)s->rows, (void*)s->ctl, (void*)s->p2p_flags}) ipc_forget_local(p);
    cudaFree(s->p2p_peer_ctl);
    cudaFree(s->p2p_peer_flag_dev);
    cudaFree(s->p2p_flags);
    cudaFree(s->planes);
    cudaFree(s->rows);
    cudaFree(s->cols);
    cudaFree(s->staging);
    cudaFree(s->ctl);
    cudaFree(s->dt_log);
    cudaFree(s->snaps);
    if (s->host_ctl) cudaFreeHost(s->host_ctl);
    timing_harvest(s);
    for (cudaEvent_t e : s->tev_free) cudaEventDestroy(e);
    if (s->own_stream && s->stream) cudaStreamDestroy(s->stream);
    delete s;
    return SILT_OK;
}

int silt_solver_set_stream(silt_solver* s, void* stream) {
    if (!s) return fail(SILT_ERR_INVALID, "null solver");
    CUDA_TRY(cudaSetDevice(s->device));
    CUDA_TRY(cudaStreamSynchronize(s->stream));
    if (s->own_stream) cudaStreamDestroy(s->stream);
    s->own_stream = false;
    s->stream = (cudaStream_t)stream;
    return SILT_OK;
}

static int ensure_staging(silt_solver* s) {
    if (s->staging) return SILT_OK;
    CUDA_TRY(cudaMalloc(&s->staging, 4 * (size_t)s->nx * s->ny * sizeof(double)));
    return SILT_OK;
}

static int upload_impl(silt_solver* s, const double* src, cudaMemcpyKind kind) {
    if (!s || !src) return fail(SILT_ERR_INVALID, "silt_solver_upload: null argument");
    CUDA_TRY(cudaSetDevice(s->device));
    if (int rc = ensure_staging(s)) return rc;
    const size_t bytes = 4 * (size_t)s->nx * s->ny * sizeof(double);
    CUDA_TRY(cudaMemcpyAsync(s->staging, src, bytes, kind, s->stream));
    const StepArgs& A = s->args;
    aos_to_soa<<<grid_blocks((long long)s->nx * s->ny, 256), 256, 0, s->stream>>>(
        s->staging, A.state[0][0], A.state[0][1], A.state[0][2], A.state[0][3], s->nx, s->ny,
        s->pitch);
    ++s->kernel_count;
    CUDA_TRY(cudaGetLastError());
    s->begun = false;  // the run clock restarts at the uploaded state
    return SILT_OK;
}

int silt_solver_upload(silt_solver* s, const double* host_aos) {
    return upload_impl(s, host_aos, cudaMemcpyHostToDevice);
}

int silt_solver_upload_device(silt_solver* s, const double* dev_aos) {
    return upload_impl(s, dev_aos, cudaMemcpyDeviceToDevice);
}

static int download_impl(silt_solver* s, double* dst, cudaMemcpyKind kind) {
    if (!s || !dst) return fail(SILT_ERR_INVALID, "silt_solver_download: null argument");
    CUDA_TRY(cudaSetDevice(s->device));
    int p = 0;
    if (s->begun) {
        Slot sl;
        if (int rc = read_slot(s, &sl, nullptr)) return rc;
        p = (int)(sl.steps & 1);
    }
    if (int rc = ensure_staging(s)) return rc;
    const StepArgs& A = s->args;
    soa_to_aos<<<grid_blocks((long long)s->nx * s->ny, 256), 256, 0, s->stream>>>(
        s->staging, A.state[p][0], A.state[p][1], A.state[p][2], A.state[p][3], s->nx, s->ny,
        s->pitch);
    ++s->kernel_count;
    const size_t bytes = 4 * (size_t)s->nx * s->ny * sizeof(double);
    CUDA_TRY(cudaMemcpyAsync(dst, s->staging, bytes, kind, s->stream));
    CUDA_TRY(cudaStreamSynchronize(s->stream));
    return SILT_OK;
}

int silt_solver_download(silt_solver* s, double* host_aos) {
    return download_impl(s, host_aos, cudaMemcpyDeviceToHost);
}

int silt_solver_download_device(silt_solver* s, double* dev_aos) {
    return download_impl(s, dev_aos, cudaMemcpyDeviceToDevice);
}

// ---- asynchronous snapshot capture ------------------------------------------
// on_snapshot + gather (src/parallel.cpp:333-342, 179-190) without holding the
// run: the paused state is transposed into snapbuf on the solver's stream, the
// solver resumes, and snapbuf streams to host memory on copy_stream while the
// next steps execute.

int silt_solver_capture_wait(silt_solver* s) {
    if (!s) return fail(SILT_ERR_INVALID, "null solver");
    if (s->writer.joinable()) {  // an asynchronous CSV snapshot in flight
        s->writer.join();
        s->cap_pending = false;
        if (s->writer_rc != SILT_OK) {
            const int rc = s->writer_rc;
            s->writer_rc = SILT_OK;
            return fail(rc, s->writer_err);
        }
    }
    if (!s->cap_pending) return SILT_OK;
    CUDA_TRY(cudaSetDevice(s->device));
    CUDA_TRY(cudaEventSynchronize(s->cap_done));
    s->cap_pending = false;
    return SILT_OK;
}

int silt_solver_capture_query(silt_solver* s, int* landed) {
    if (!s || !landed) return fail(SILT_ERR_INVALID, "silt_solver_capture_query: null argument");
    *landed = 1;
    if (s->writer.joinable()) {  // an asynchronous CSV snapshot: landed once written
        if (s->writer_busy.load(std::memory_order_acquire)) {
            *landed = 0;
            return SILT_OK;
        }
        return silt_solver_capture_wait(s);  // joins, reports the writer's error
    }
    if (!s->cap_pending) return SILT_OK;
    CUDA_TRY(cudaSetDevice(s->device));
    const cudaError_t e = cudaEventQuery(s->cap_done);
    if (e == cudaErrorNotReady) {
        *landed = 0;
        return SILT_OK;
    }
    if (e != cudaSuccess) return fail(SILT_ERR_CUDA, cudaGetErrorString(e));
    s->cap_pending = false;
    return SILT_OK;
}

int silt_solver_capture_resume(silt_solver* s, double* host_aos) {
    if (!s || !host_aos) return fail(SILT_ERR_INVALID, "silt_solver_capture_resume: null argument");
    if (!s->begun) return fail(SILT_ERR_INVALID, "silt_solver_capture_resume: run not begun");
    if (int rc = silt_solver_capture_wait(s)) return rc;  // snapbuf is free again
    CUDA_TRY(cudaSetDevice(s->device));
    const size_t bytes = 4 * (size_t)s->nx * s->ny * sizeof(double);
    if (!s->snapbuf) {
        CUDA_TRY(cudaMalloc(&s->snapbuf, bytes));
        CUDA_TRY(cudaStreamCreateWithFlags(&s->copy_stream, cudaStreamNonBlocking));
        CUDA_TRY(cudaEventCreateWithFlags(&s->cap_ready, cudaEventDisableTiming));
        CUDA_TRY(cudaEventCreateWithFlags(&s->cap_done, cudaEventDisableTiming));
    }
    Slot sl;
    if (int rc = read_slot(s, &sl, nullptr)) return rc;  // synchronizes the stream
    if (sl.state != SILT_STATE_PAUSED)
        return fail(SILT_ERR_INVALID, "silt_solver_capture_resume: solver is not paused");
    const int p = (int)(sl.steps & 1);
    const StepArgs& A = s->args;
    soa_to_aos<<<grid_blocks((long long)s->nx * s->ny, 256), 256, 0, s->stream>>>(
        s->snapbuf, A.state[p][0], A.state[p][1], A.state[p][2], A.state[p][3], s->nx, s->ny,
        s->pitch);
    ++s->kernel_count;
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaEventRecord(s->cap_ready, s->stream));
    CUDA_TRY(cudaStreamWaitEvent(s->copy_stream, s->cap_ready, 0));
    CUDA_TRY(cudaMemcpyAsync(host_aos, s->snapbuf, bytes, cudaMemcpyDeviceToHost,
                             s->copy_stream));
    CUDA_TRY(cudaEventRecord(s->cap_done, s->copy_stream));
    s->cap_pending = true;
    // resume: later launches on s->stream are ordered after the transpose
    int st = SILT_STATE_RUNNING;
    Slot* slot = &s->ctl->slot[s->launches % 3];
    CUDA_TRY(cudaMemcpy(&slot->state, &st, sizeof(int), cudaMemcpyHostToDevice));
    return SILT_OK;
}

int silt_host_alloc(int64_t bytes, void** out) {
    if (!out || bytes < 0) return fail(SILT_ERR_INVALID, "silt_host_alloc: bad argument");
    *out = nullptr;
    if (bytes == 0) return SILT_OK;
    CUDA_TRY(cudaHostAlloc(out, (size_t)bytes, cudaHostAllocPortable));
    return SILT_OK;
}

int silt_host_free(void* p) {
    if (p) CUDA_TRY(cudaFreeHost(p));
    return SILT_OK;
}

int silt_solver_set_ghosts(silt_solver* s, const double* west, const double* east,
                           const double* south, const double* north) {
    if (!s) return fail(SILT_ERR_INVALID, "null solver");
    CUDA_TRY(cudaSetDevice(s->device));
    const StepArgs& A = s->args;
    struct Item {
        const double* src;
        double* dst;
        int n;
    } items[4] = {{west, A.ghost_w, s->ny},
                  {east, A.ghost_e, s->ny},
                  {south, A.ghost_s[0], s->nx},
                  {north, A.ghost_n[0], s->nx}};
    double* tmp = nullptr;
    const int nmax = std::max(s->nx, s->ny);
    CUDA_TRY(cudaMalloc(&tmp, 4 * (size_t)nmax * sizeof(double)));
    for (auto& it : items) {
        if (!it.src) continue;
        cudaMemcpyAsync(tmp, it.src, 4 * (size_t)it.n * sizeof(double), cudaMemcpyHostToDevice,
                        s->stream);
        aos_to_planes<<<(it.n + 127) / 128, 128, 0, s->stream>>>(tmp, it.dst, it.n);
        ++s->kernel_count;
    }
    cudaStreamSynchronize(s->stream);
    cudaFree(tmp);
    CUDA_TRY(cudaGetLastError());
    return SILT_OK;
}

int silt_solver_begin(silt_solver* s, const silt_run_plan* plan) {
    if (!s || !plan) return fail(SILT_ERR_INVALID, "silt_solver_begin: null argument");
    if (!(plan->t_end >= 0)) return fail(SILT_ERR_INVALID, "run: t_end must be >= 0");
    CUDA_TRY(cudaSetDevice(s->device));
    // make_plan (src/parallel.cpp:101-127): keep (0, t_end], sorted, unique
    std::vector<double> snaps;
    for (int k = 0; k < plan->n_snapshots; ++k) {
        const double v = plan->snapshot_times[k];
        if (v > 0 && v <= plan->t_end) snaps.push_back(v);
    }
    std::sort(snaps.begin(), snaps.end());
    snaps.erase(std::unique(snaps.begin(), snaps.end()), snaps.end());
    CUDA_TRY(cudaStreamSynchronize(s->stream));
    if (s->begun) {
        // A new run from the current state: the run clock restarts at parity
        // 0, so after an odd number of steps state n lives in plane set 1 and
        // is moved to plane set 0 first (otherwise the run would restart one
        // step stale).
        if (int rc = silt_solver_capture_wait(s)) return rc;
        Slot sl;
        if (int rc = read_slot(s, &sl, nullptr)) return rc;
        if (sl.steps & 1) {
            const size_t bytes = (size_t)s->ny * s->pitch * sizeof(double);
            for (int f = 0; f < 4; ++f)
                CUDA_TRY(cudaMemcpyAsync(s->args.state[0][f], s->args.state[1][f], bytes,
                                         cudaMemcpyDeviceToDevice, s->stream));
        }
    }
    if ((int)snaps.size() > s->n_snaps_alloc) {
        cudaFree(s->snaps);
        s->snaps = nullptr;
        CUDA_TRY(cudaMalloc(&s->snaps, snaps.size() * sizeof(double)));
        s->n_snaps_alloc = (int)snaps.size();
    }
    if (!snaps.empty())
        CUDA_TRY(cudaMemcpy(s->snaps, snaps.data(), snaps.size() * sizeof(double),
                            cudaMemcpyHostToDevice));
    if (plan->dt_log_capacity > s->dt_cap) {
        cudaFree(s->dt_log);
        s->dt_log = nullptr;
        CUDA_TRY(cudaMalloc(&s->dt_log, plan->dt_log_capacity * sizeof(double)));
        s->dt_cap = plan->dt_log_capacity;
    }
    Control& c = *s->host_ctl;
    std::memset(&c, 0, sizeof(Control));
    c.slot[0].state = SILT_STATE_RUNNING;
    c.t_end = plan->t_end;
    c.max_steps = plan->max_steps;
    c.fixed_dt = 0;
    c.fixed_mode = 0;
    c.dt_cap = std::min<int64_t>(plan->dt_log_capacity, s->dt_cap);
    c.dt_log = s->dt_log;
    c.snaps = s->snaps;
    c.n_snaps = (int)snaps.size();
    CUDA_TRY(cudaMemcpyAsync(s->ctl, &c, sizeof(Control), cudaMemcpyHostToDevice, s->stream));
    s->launches = 0;
    StepArgs A = s->args;
    A.write_edges_in_reduce = 1;
    const long long n = (long long)s->nx * s->ny;
    if (s->variant == SILT_VARIANT_STRICT)
        silt_strict_reduce(A, 0, grid_blocks(n, 256), s->stream);
    else
        silt_fast_reduce(A, 0, grid_blocks(n, 256), s->stream);
    ++s->kernel_count;
    CUDA_TRY(cudaGetLastError());
    s->begun = true;
    s->begun_after_connect = s->p2p_world > 1;
    return SILT_OK;
}

int silt_solver_step(silt_solver* s, int n) {
    if (!s) return fail(SILT_ERR_INVALID, "null solver");
    if (!s->begun) return fail(SILT_ERR_INVALID, "silt_solver_step: call silt_solver_begin first");
    if (int rc = check_cfl(s->prob.cfl)) return rc;
    CUDA_TRY(cudaSetDevice(s->device));
    // 1D: n steps in one cooperative launch when the grid fits co-resident
    // (step1d_coop_kernel); SILT_COOP=0 keeps one launch per step
    static const bool coop = [] {
        const char* e = std::getenv("SILT_COOP");
        return !(e && e[0] == '0');
    }();
    if (coop && s->prob.dim == 1 && n > 1) {
        // one cluster (<= 16 CTAs of 384 threads) when the line fits, else a
        // cooperative grid; SILT_COOP=2 forces the cooperative grid
        const long long strips = (s->nx + kCellsPerWarp - 1) / kCellsPerWarp;
        const int per_cta = 384 / 32;
        const int ctas = (int)((strips + per_cta - 1) / per_cta);
        static const bool cluster_ok = [] {
            const char* e = std::getenv("SILT_COOP");
            return !(e && e[0] == '2');
        }();
        if (cluster_ok && ctas <= 16 && !s->cluster_failed) {
            const cudaEvent_t t0 = timing_mark(s);
            const int li0 = (int)(s->launches % 3);
            const int rc = s->variant == SILT_VARIANT_STRICT
                               ? silt_strict_step1d_cluster(s->args, li0, n, ctas, s->stream)
                               : silt_fast_step1d_cluster(s->args, li0, n, ctas, s->stream);
            timing_close(s, t0);
            if (rc == 0) {
                s->launches += n;
                ++s->kernel_count;
                return SILT_OK;
            }
            cudaGetLastError();  // cluster not schedulable here: fall back for good
            s->cluster_failed = true;
        }
        if (s->coop_blocks < 0)
            s->coop_blocks = s->variant == SILT_VARIANT_STRICT
                                 ? silt_strict_step1d_coop_blocks(s->args.P.shields)
                                 : silt_fast_step1d_coop_blocks(s->args.P.shields);
        if ((int)s->step_grid.x <= s->coop_blocks) {
            const int li0 = (int)(s->launches % 3);
            const cudaEvent_t t0 = timing_mark(s);
            const int rc = s->variant == SILT_VARIANT_STRICT
                               ? silt_strict_step1d_coop(s->args, li0, n, s->step_grid, s->stream)
                               : silt_fast_step1d_coop(s->args, li0, n, s->step_grid, s->stream);
            timing_close(s, t0);
            if (rc != 0) return fail(SILT_ERR_CUDA, cudaGetErrorString((cudaError_t)rc));
            s->launches += n;
            ++s->kernel_count;
            return SILT_OK;
        }
    }
    for (int k = 0; k < n; ++k) launch_step(s);
    CUDA_TRY(cudaGetLastError());
    return SILT_OK;
}

int silt_solver_step_split_ok(silt_solver* s, int* ok) {
    if (!s || !ok) return fail(SILT_ERR_INVALID, "silt_solver_step_split_ok: null argument");
    *ok = s->split_map != nullptr;
    return SILT_OK;
}

int silt_solver_step_part(silt_solver* s, int part) {
    if (!s) return fail(SILT_ERR_INVALID, "null solver");
    if (!s->begun) return fail(SILT_ERR_INVALID, "silt_solver_step_part: call silt_solver_begin first");
    if (part != 1 && part != 2) return fail(SILT_ERR_INVALID, "silt_solver_step_part: part is 1 or 2");
    if (!s->split_map)
        return fail(SILT_ERR_UNSUPPORTED, "silt_solver_step_part: this strip does not split");
    if (int rc = check_cfl(s->prob.cfl)) return rc;
    CUDA_TRY(cudaSetDevice(s->device));
    launch_step(s, part);
    CUDA_TRY(cudaGetLastError());
    return SILT_OK;
}

int silt_solver_step_fixed(silt_solver* s, double dt) {
    if (!s) return fail(SILT_ERR_INVALID, "null solver");
    if (!s->begun) return fail(SILT_ERR_INVALID, "silt_solver_step_fixed: call begin first");
    CUDA_TRY(cudaSetDevice(s->device));
    // the caller's dt is applied exactly as given, like step_1d/step_2d
    // (src/stepper.cpp:118-189): 0 leaves the field unchanged, a NaN makes
    // check_depth fail ("negative depth produced"), as in the reference
    s->host_ctl->fixed_dt = dt;
    s->host_ctl->fixed_mode = 1;
    CUDA_TRY(cudaMemcpyAsync(&s->ctl->fixed_dt, &s->host_ctl->fixed_dt, sizeof(double),
                             cudaMemcpyHostToDevice, s->stream));
    CUDA_TRY(cudaMemcpyAsync(&s->ctl->fixed_mode, &s->host_ctl->fixed_mode, sizeof(int),
                             cudaMemcpyHostToDevice, s->stream));
    launch_step(s);
    CUDA_TRY(cudaStreamSynchronize(s->stream));
    s->host_ctl->fixed_dt = 0;
    s->host_ctl->fixed_mode = 0;
    CUDA_TRY(cudaMemcpy(&s->ctl->fixed_dt, &s->host_ctl->fixed_dt, sizeof(double),
                        cudaMemcpyHostToDevice));
    CUDA_TRY(cudaMemcpy(&s->ctl->fixed_mode, &s->host_ctl->fixed_mode, sizeof(int),
                        cudaMemcpyHostToDevice));
    CUDA_TRY(cudaGetLastError());
    return SILT_OK;
}

int silt_solver_status(silt_solver* s, silt_status* st) {
    if (!s || !st) return fail(SILT_ERR_INVALID, "silt_solver_status: null argument");
    if (!s->begun) return fail(SILT_ERR_INVALID, "silt_solver_status: call begin first");
    Control* full = s->host_ctl;
    Slot sl;
    if (int rc = read_slot(s, &sl, full)) return rc;
    st->t = sl.t;
    st->steps = sl.steps;
    st->state = sl.state;
    st->last_dt = sl.last_dt;
    st->snapshot_index = sl.snap_idx;
    st->error_code = SILT_OK;
    if (sl.err || sl.state == SILT_STATE_FAILED) {
        st->state = SILT_STATE_FAILED;
        const unsigned bits = sl.err ? sl.err : silt_dev::kErrDry;
        st->error_code = error_from(*full, full->err_claim ? full->err_bits : bits);
        return st->error_code;
    }
    return SILT_OK;
}

int silt_solver_resume(silt_solver* s) {
    if (!s) return fail(SILT_ERR_INVALID, "null solver");
    CUDA_TRY(cudaSetDevice(s->device));
    CUDA_TRY(cudaStreamSynchronize(s->stream));
    int st = 0;
    Slot* slot = &s->ctl->slot[s->launches % 3];
    CUDA_TRY(cudaMemcpy(&st, &slot->state, sizeof(int), cudaMemcpyDeviceToHost));
    if (st == SILT_STATE_PAUSED) {
        st = SILT_STATE_RUNNING;
        CUDA_TRY(cudaMemcpy(&slot->state, &st, sizeof(int), cudaMemcpyHostToDevice));
    }
    return SILT_OK;
}

int silt_solver_dt_log(silt_solver* s, double* host_out, int64_t n) {
    if (!s || (!host_out && n > 0)) return fail(SILT_ERR_INVALID, "silt_solver_dt_log: null");
    if (n > s->dt_cap) return fail(SILT_ERR_INVALID, "silt_solver_dt_log: n exceeds capacity");
    if (n == 0) return SILT_OK;
    CUDA_TRY(cudaSetDevice(s->device));
    CUDA_TRY(cudaStreamSynchronize(s->stream));
    CUDA_TRY(cudaMemcpy(host_out, s->dt_log, n * sizeof(double), cudaMemcpyDeviceToHost));
    return SILT_OK;
}

int silt_solver_cfl_dt(silt_solver* s, double* dt) {
    if (!s || !dt) return fail(SILT_ERR_INVALID, "silt_solver_cfl_dt: null argument");
    if (int rc = check_cfl(s->prob.cfl)) return rc;
    if (!s->begun) {
        silt_run_plan plan{INFINITY, -1, nullptr, 0, 0};
        if (int rc = silt_solver_begin(s, &plan)) return rc;
    }
    Slot sl;
    if (int rc = read_slot(s, &sl, nullptr)) return rc;
    if (!sl.wet) return fail(SILT_ERR_INVALID, "cfl_dt: field is entirely dry");
    double sx, sy;
    std::memcpy(&sx, &sl.max_sx, sizeof(double));
    std::memcpy(&sy, &sl.max_sy, sizeof(double));
    double raw = s->args.dx / sx;
    if (s->prob.dim == 2) raw = std::min(raw, s->args.dy / sy);
    *dt = s->prob.cfl * raw;
    return SILT_OK;
}

int silt_solver_reduce_slot(silt_solver* s, double** dev_ptr) {
    if (!s || !dev_ptr) return fail(SILT_ERR_INVALID, "silt_solver_reduce_slot: null argument");
    *dev_ptr = reinterpret_cast<double*>(&s->ctl->slot[s->launches % 3].max_sx);
    return SILT_OK;
}

int silt_solver_exchange_ptrs(silt_solver* s, silt_exchange* out) {
    if (!s || !out) return fail(SILT_ERR_INVALID, "silt_solver_exchange_ptrs: null argument");
    out->send_south = s->strip.south_neighbor ? s->args.send_s[0] : nullptr;
    out->send_north = s->strip.north_neighbor ? s->args.send_n[0] : nullptr;
    out->recv_south = s->strip.south_neighbor ? s->args.recv_s[0] : nullptr;
    out->recv_north = s->strip.north_neighbor ? s->args.recv_n[0] : nullptr;
    out->row_doubles = 4 * (int64_t)s->nx;
    return SILT_OK;
}

int silt_solver_launch_count(silt_solver* s, int64_t* count) {
    if (!s || !count) return fail(SILT_ERR_INVALID, "null argument");
    *count = s->kernel_count;
    return SILT_OK;
}

}  // extern "C"

// ---- strip group --------------------------------------------------------------
namespace {

// direct mode: this strip's maxima of the state just produced into every
// other strip's slot (remote atomics over NVLink / same-device atomics)
__global__ void push_max_kernel(const Control* local, int slot, Control* const* peers, int n) {
    const unsigned long long sx = local->slot[slot].max_sx, sy = local->slot[slot].max_sy;
    for (int k = threadIdx.x; k < n; k += blockDim.x) {
        atomicMax(&peers[k]->slot[slot].max_sx, sx);
        atomicMax(&peers[k]->slot[slot].max_sy, sy);
    }
}

// p2p: maxima into the peers' slots, then (release, system scope) this rank's
// step count into every peer's flag array: a peer that acquires the flag
// also observes this rank's edge rows and maxima.
__global__ void push_release_kernel(const Control* local, int slot, Control* const* peers,
                                    unsigned* const* peer_flags, int n, unsigned value) {
    const unsigned long long sx = local->slot[slot].max_sx, sy = local->slot[slot].max_sy;
    for (int k = threadIdx.x; k < n; k += blockDim.x) {
        atomicMax(&peers[k]->slot[slot].max_sx, sx);
        atomicMax(&peers[k]->slot[slot].max_sy, sy);
    }
    __syncthreads();
    __threadfence_system();
    for (int k = threadIdx.x; k < n; k += blockDim.x)
        asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(peer_flags[k]), "r"(value)
                     : "memory");
}

// p2p: acquire (system scope) every peer's flag before the step that reads
// their rows and maxima.  The wait is bounded: a peer that has not published
// step `expect` within timeout_ns (dead or hung rank) raises kErrPeer in the
// slot the next launch reads, so that launch and every later one stop
// (decide: FAILED) and the host reports which rank missed which step, instead
// of the GPU spinning forever.
__global__ void acquire_flags_kernel(const unsigned* flags, int world, int rank,
                                     unsigned expect, Control* ctl, int slot,
                                     unsigned long long timeout_ns) {
    unsigned long long t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    for (int j = threadIdx.x; j < world; j += blockDim.x) {
        if (j == rank) continue;
        unsigned v;
        for (;;) {
            asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(flags + j)
                         : "memory");
            if ((int)(v - expect) >= 0) break;
            unsigned long long t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            if (t - t0 > timeout_ns) {
                atomicOr(&ctl->slot[slot].err, silt_dev::kErrPeer);
                if (atomicCAS(&ctl->err_claim, 0u, 1u) == 0u) {
                    ctl->err_bits = silt_dev::kErrPeer;
                    ctl->err_col = j;            // the rank that missed the step
                    ctl->err_row = (int)expect;  // the step it did not publish
                }
                break;
            }
            __nanosleep(500);
        }
    }
}

__global__ void max_slots_kernel(const double* gathered, int n, double* result) {
    double sx = 0.0, sy = 0.0;
    for (int k = 0; k < n; ++k) {
        sx = gathered[2 * k] > sx ? gathered[2 * k] : sx;
        sy = gathered[2 * k + 1] > sy ? gathered[2 * k + 1] : sy;
    }
    result[0] = sx;
    result[1] = sy;
}

void block_range(int n, int parts, int r, int* offset, int* count) {
    const int base = n / parts, rem = n % parts;
    *count = base + (r < rem ? 1 : 0);
    *offset = r * base + std::min(r, rem);
}

}  // namespace

struct silt_group {
    std::vector<silt_solver*> strips;
    std::vector<int> south, north;   // neighbour strip or -1
    std::vector<cudaEvent_t> stepped, copied;
    // direct mode: the step kernels store their edge rows into the
    // neighbours' recv rows (peer memory) and push_max_kernel folds each
    // strip's axis-speed maxima into every other strip's slot; per step the
    // strips only wait on each other's events (no copies, no reduction stream)
    bool direct = false;
    std::vector<Control**> peers;    // per strip, on its device: the other strips' Control
    std::vector<cudaEvent_t> pushed;
    bool joined = false;             // `reduced` marks the last direct step of every strip
    int dev0 = 0;
    double* gathered = nullptr;      // on dev0: [py][2]
    double* result = nullptr;        // on dev0: [2]
    cudaStream_t s0 = nullptr;       // reduction stream on dev0
    cudaEvent_t reduced = nullptr;
    int nx = 0, ny = 0;
};

namespace {

int group_exchange(silt_group* g) {
    const int py = (int)g->strips.size();
    if (py == 1) return SILT_OK;
    // 1. every strip finished its step
    for (int k = 0; k < py; ++k) {
        CUDA_TRY(cudaSetDevice(g->strips[k]->device));
        CUDA_TRY(cudaEventRecord(g->stepped[k], g->strips[k]->stream));
    }
    // 2. gather the slots on dev0, MAX, scatter back
    CUDA_TRY(cudaSetDevice(g->dev0));
    for (int k = 0; k < py; ++k) {
        CUDA_TRY(cudaStreamWaitEvent(g->s0, g->stepped[k], 0));
        const Slot* slot = &g->strips[k]->ctl->slot[g->strips[k]->launches % 3];
        CUDA_TRY(cudaMemcpyAsync(g->gathered + 2 * k, &slot->max_sx, 2 * sizeof(double),
                                 cudaMemcpyDefault, g->s0));
    }
    max_slots_kernel<<<1, 1, 0, g->s0>>>(g->gathered, py, g->result);
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaEventRecord(g->reduced, g->s0));
    // 3. per strip: reduced maxima + ghost rows from the neighbours' send rows
    //    (direct mode: the rows are already in place)
    const size_t row = 4 * (size_t)g->nx * sizeof(double);
    for (int k = 0; k < py; ++k) {
        silt_solver* s = g->strips[k];
        CUDA_TRY(cudaSetDevice(s->device));
        CUDA_TRY(cudaStreamWaitEvent(s->stream, g->reduced, 0));
        Slot* slot = &s->ctl->slot[s->launches % 3];
        CUDA_TRY(cudaMemcpyAsync(&slot->max_sx, g->result, 2 * sizeof(double), cudaMemcpyDefault,
                                 s->stream));
        if (g->direct) {
            CUDA_TRY(cudaEventRecord(g->copied[k], s->stream));
            continue;
        }
        if (g->south[k] >= 0) {
            silt_solver* src = g->strips[g->south[k]];
            CUDA_TRY(cudaStreamWaitEvent(s->stream, g->stepped[g->south[k]], 0));
            CUDA_TRY(cudaMemcpyAsync(s->args.recv_s[0], src->args.send_n[0], row,
                                     cudaMemcpyDefault, s->stream));
        }
        if (g->north[k] >= 0) {
            silt_solver* src = g->strips[g->north[k]];
            CUDA_TRY(cudaStreamWaitEvent(s->stream, g->stepped[g->north[k]], 0));
            CUDA_TRY(cudaMemcpyAsync(s->args.recv_n[0], src->args.send_s[0], row,
                                     cudaMemcpyDefault, s->stream));
        }
        CUDA_TRY(cudaEventRecord(g->copied[k], s->stream));
    }
    // 4. a strip's next step overwrites its send rows: wait for the readers
    for (int k = 0; k < py; ++k) {
        silt_solver* s = g->strips[k];
        CUDA_TRY(cudaSetDevice(s->device));
        if (g->south[k] >= 0) CUDA_TRY(cudaStreamWaitEvent(s->stream, g->copied[g->south[k]], 0));
        if (g->north[k] >= 0) CUDA_TRY(cudaStreamWaitEvent(s->stream, g->copied[g->north[k]], 0));
    }
    return SILT_OK;
}

}  // namespace

extern "C" {

int silt_group_destroy(silt_group* g) {
    if (!g) return SILT_OK;
    for (size_t k = 0; k < g->peers.size(); ++k) {
        cudaSetDevice(g->strips[k]->device);
        cudaStreamSynchronize(g->strips[k]->stream);
        if (g->peers[k]) cudaFree(g->peers[k]);
        if (g->pushed[k]) cudaEventDestroy(g->pushed[k]);
    }
    for (silt_solver* s : g->strips) silt_solver_destroy(s);
    cudaSetDevice(g->dev0);
    if (g->s0) cudaStreamSynchronize(g->s0);
    for (auto e : g->stepped) cudaEventDestroy(e);
    for (auto e : g->copied) cudaEventDestroy(e);
    if (g->reduced) cudaEventDestroy(g->reduced);
    if (g->s0) cudaStreamDestroy(g->s0);
    cudaFree(g->gathered);
    cudaFree(g->result);
    delete g;
    return SILT_OK;
}

int silt_group_create(const silt_problem* problem, int py, const int* devices, int n_devices,
                      int variant, silt_group** out) {
    if (!out) return fail(SILT_ERR_INVALID, "silt_group_create: null out");
    *out = nullptr;
    if (int rc = validate_problem(problem)) return rc;
    const int ny = problem->dim == 1 ? 1 : problem->ny;
    if (py < 1) return fail(SILT_ERR_INVALID, "partition: worker counts must be >= 1");
    if (problem->dim == 1 && py != 1) return fail(SILT_ERR_INVALID, "partition: 1D grids require py == 1");
    if (py > ny) return fail(SILT_ERR_INVALID, "partition: every worker needs at least one cell per axis");
    const int dev_default = 0;
    if (n_devices < 1 || !devices) {
        devices = &dev_default;
        n_devices = 1;
    }
    silt_group* g = new silt_group();
    g->nx = problem->nx;
    g->ny = ny;
    g->dev0 = devices[0];
    const bool per_y = problem->dim == 2 && problem->bc[SILT_SOUTH].type == SILT_BC_PERIODIC;
    for (int k = 0; k < py; ++k) {
        int j0, n;
        block_range(ny, py, k, &j0, &n);
        const int south = k > 0 ? k - 1 : (per_y && py > 1 ? py - 1 : -1);
        const int north = k < py - 1 ? k + 1 : (per_y && py > 1 ? 0 : -1);
        silt_strip st{j0, n, south >= 0, north >= 0};
        silt_solver* s = nullptr;
        if (int rc = silt_solver_create(problem, &st, devices[k % n_devices], variant, &s)) {
            silt_group_destroy(g);
            return rc;
        }
        g->strips.push_back(s);
        g->south.push_back(south);
        g->north.push_back(north);
        cudaEvent_t e1, e2;
        cudaSetDevice(s->device);
        cudaEventCreateWithFlags(&e1, cudaEventDisableTiming);
        cudaEventCreateWithFlags(&e2, cudaEventDisableTiming);
        g->stepped.push_back(e1);
        g->copied.push_back(e2);
    }
    // direct NVLink copies between the devices in use (ghost rows, slots)
    {
        const int nd = std::min(n_devices, py);
        for (int a = 0; a < nd; ++a)
            for (int b = 0; b < nd; ++b) {
                if (devices[a] == devices[b]) continue;
                int ok = 0;
                if (cudaDeviceCanAccessPeer(&ok, devices[a], devices[b]) == cudaSuccess && ok) {
                    cudaSetDevice(devices[a]);
                    if (cudaDeviceEnablePeerAccess(devices[b], 0) != cudaSuccess)
                        cudaGetLastError();  // already enabled is fine
                }
            }
    }
    // direct mode: every pair of strip devices can reach the other's memory
    {
        const char* e = std::getenv("SILT_GROUP_DIRECT");
        bool ok = py > 1 && problem->dim == 2 && !(e && e[0] == '0');
        for (int a = 0; ok && a < py; ++a)
            for (int b = 0; ok && b < py; ++b) {
                const int da = g->strips[a]->device, db = g->strips[b]->device;
                int can = 1;
                if (da != db && (cudaDeviceCanAccessPeer(&can, da, db) != cudaSuccess || !can))
                    ok = false;
            }
        if (ok) {
            const size_t row = 4 * (size_t)g->nx;
            for (silt_solver* s : g->strips) {  // second parity of the receive rows
                s->args.recv_s[1] = s->rows + 8 * row;
                s->args.recv_n[1] = s->rows + 9 * row;
            }
            for (int k = 0; k < py; ++k) {
                StepArgs& A = g->strips[k]->args;
                for (int q = 0; q < 2; ++q) {
                    if (g->south[k] >= 0) A.send_s[q] = g->strips[g->south[k]]->args.recv_n[q];
                    if (g->north[k] >= 0) A.send_n[q] = g->strips[g->north[k]]->args.recv_s[q];
                }
            }
            g->peers.assign(py, nullptr);
            g->pushed.assign(py, nullptr);
            for (int k = 0; k < py && ok; ++k) {
                std::vector<Control*> others;
                for (int j = 0; j < py; ++j)
                    if (j != k) others.push_back(g->strips[j]->ctl);
                cudaSetDevice(g->strips[k]->device);
                if (cudaMalloc(&g->peers[k], others.size() * sizeof(Control*)) != cudaSuccess ||
                    cudaMemcpy(g->peers[k], others.data(), others.size() * sizeof(Control*),
                               cudaMemcpyHostToDevice) != cudaSuccess ||
                    cudaEventCreateWithFlags(&g->pushed[k], cudaEventDisableTiming) != cudaSuccess)
                    ok = false;
            }
            g->direct = ok;
            if (!ok) {
                silt_group_destroy(g);
                return fail(SILT_ERR_CUDA, "silt_group_create: direct-mode setup failed");
            }
        }
    }
    cudaSetDevice(g->dev0);
    if (cudaStreamCreateWithFlags(&g->s0, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&g->reduced, cudaEventDisableTiming) != cudaSuccess ||
        cudaMalloc(&g->gathered, 2 * py * sizeof(double)) != cudaSuccess ||
        cudaMalloc(&g->result, 2 * sizeof(double)) != cudaSuccess) {
        silt_group_destroy(g);
        return fail(SILT_ERR_CUDA, "silt_group_create: allocation failed");
    }
    *out = g;
    return SILT_OK;
}

int silt_group_upload(silt_group* g, const double* host_aos) {
    if (!g || !host_aos) return fail(SILT_ERR_INVALID, "silt_group_upload: null argument");
    for (silt_solver* s : g->strips)
        if (int rc = silt_solver_upload(s, host_aos + 4 * (size_t)s->strip.j0 * g->nx)) return rc;
    return SILT_OK;
}

int silt_group_download(silt_group* g, double* host_aos) {
    if (!g || !host_aos) return fail(SILT_ERR_INVALID, "silt_group_download: null argument");
    for (silt_solver* s : g->strips)
        if (int rc = silt_solver_download(s, host_aos + 4 * (size_t)s->strip.j0 * g->nx)) return rc;
    return SILT_OK;
}

int silt_group_begin(silt_group* g, const silt_run_plan* plan) {
    if (!g) return fail(SILT_ERR_INVALID, "null group");
    for (silt_solver* s : g->strips)
        if (int rc = silt_solver_begin(s, plan)) return rc;
    return group_exchange(g);
}

int silt_group_step(silt_group* g, int n) {
    if (!g) return fail(SILT_ERR_INVALID, "null group");
    const int py = (int)g->strips.size();
    for (int k = 0; k < n; ++k) {
        if (!g->direct) {
            for (silt_solver* s : g->strips)
                if (int rc = silt_solver_step(s, 1)) return rc;
            if (int rc = group_exchange(g)) return rc;
            continue;
        }
        for (int i = 0; i < py; ++i) {
            silt_solver* s = g->strips[i];
            CUDA_TRY(cudaSetDevice(s->device));
            // every strip's previous step (rows delivered, maxima pushed) is
            // done: one join event (2 py waits per step instead of py^2)
            if (g->joined) CUDA_TRY(cudaStreamWaitEvent(s->stream, g->reduced, 0));
            if (int rc = silt_solver_step(s, 1)) return rc;
            push_max_kernel<<<1, 32, 0, s->stream>>>(s->ctl, (int)(s->launches % 3), g->peers[i],
                                                      py - 1);
            ++s->kernel_count;
            CUDA_TRY(cudaGetLastError());
            CUDA_TRY(cudaEventRecord(g->pushed[i], s->stream));
        }
        CUDA_TRY(cudaSetDevice(g->dev0));
        for (int j = 0; j < py; ++j) CUDA_TRY(cudaStreamWaitEvent(g->s0, g->pushed[j], 0));
        CUDA_TRY(cudaEventRecord(g->reduced, g->s0));
        g->joined = true;
    }
    return SILT_OK;
}

// run_parallel rethrows the lowest rank's error (src/parallel.cpp:377-378)
int silt_group_status(silt_group* g, silt_status* st) {
    if (!g || !st) return fail(SILT_ERR_INVALID, "silt_group_status: null argument");
    int first_rc = SILT_OK;
    silt_status first{};
    for (size_t k = 0; k < g->strips.size(); ++k) {
        silt_status s{};
        const int rc = silt_solver_status(g->strips[k], &s);
        if (k == 0) first = s;
        if (rc && !first_rc) {
            first_rc = rc;
            first = s;
            if (rc == SILT_ERR_CUDA) break;
        }
    }
    *st = first;
    return first_rc;
}

int silt_group_resume(silt_group* g) {
    if (!g) return fail(SILT_ERR_INVALID, "null group");
    for (silt_solver* s : g->strips)
        if (int rc = silt_solver_resume(s)) return rc;
    return SILT_OK;
}

int silt_group_capture_resume(silt_group* g, double* host_aos) {
    if (!g || !host_aos) return fail(SILT_ERR_INVALID, "silt_group_capture_resume: null argument");
    for (silt_solver* s : g->strips)
        if (int rc = silt_solver_capture_resume(s, host_aos + 4 * (size_t)s->strip.j0 * g->nx))
            return rc;
    return SILT_OK;
}

int silt_group_capture_wait(silt_group* g) {
    if (!g) return fail(SILT_ERR_INVALID, "null group");
    for (silt_solver* s : g->strips)
        if (int rc = silt_solver_capture_wait(s)) return rc;
    return SILT_OK;
}

int silt_group_dt_log(silt_group* g, double* host_out, int64_t n) {
    if (!g || g->strips.empty()) return fail(SILT_ERR_INVALID, "null group");
    return silt_solver_dt_log(g->strips[0], host_out, n);
}

int silt_solver_timing(silt_solver* s, int enable, double* compute_seconds) {
    if (!s) return fail(SILT_ERR_INVALID, "null solver");
    CUDA_TRY(cudaSetDevice(s->device));
    CUDA_TRY(cudaStreamSynchronize(s->stream));
    timing_harvest(s);
    if (compute_seconds) *compute_seconds = s->compute_s;
    if (enable >= 0) {
        s->timing_on = enable != 0;
        s->compute_s = 0;
    }
    return SILT_OK;
}

int silt_group_timing(silt_group* g, int enable, double* per_strip) {
    if (!g) return fail(SILT_ERR_INVALID, "null group");
    for (size_t k = 0; k < g->strips.size(); ++k)
        if (int rc = silt_solver_timing(g->strips[k], enable, per_strip ? per_strip + k : nullptr))
            return rc;
    return SILT_OK;
}

}  // extern "C"

extern "C" {

// run_serial on the GPU (src/parallel.cpp:208-259)
int silt_run(const silt_problem* problem, const double* init_aos, const silt_run_plan* plan,
             int variant, double* out_aos, double* dt_log, int64_t dt_log_capacity,
             silt_status* status) {
    if (!plan || !init_aos || !out_aos) return fail(SILT_ERR_INVALID, "silt_run: null argument");
    if (int rc = check_cfl(problem ? problem->cfl : 0.5)) return rc;
    silt_solver* s = nullptr;
    if (int rc = silt_solver_create(problem, nullptr, 0, variant, &s)) return rc;
    silt_run_plan p = *plan;
    p.dt_log_capacity = dt_log ? dt_log_capacity : 0;
    int rc = silt_solver_upload(s, init_aos);
    if (!rc) rc = silt_solver_begin(s, &p);
    silt_status st{};
    const int batch = 32;
    while (!rc) {
        rc = silt_solver_step(s, batch);
        if (rc) break;
        rc = silt_solver_status(s, &st);
        if (rc) break;
        if (st.state == SILT_STATE_PAUSED) {
            rc = silt_solver_resume(s);
            continue;
        }
        if (st.state == SILT_STATE_DONE) break;
    }
    if (!rc && dt_log) rc = silt_solver_dt_log(s, dt_log, std::min<int64_t>(st.steps, dt_log_capacity));
    if (!rc) rc = silt_solver_download(s, out_aos);
    if (status) *status = st;
    const std::string keep = g_err;
    silt_solver_destroy(s);
    g_err = keep;
    return rc;
}

int silt_cfl_dt(const silt_problem* problem, const double* field_aos, int variant, double* dt) {
    if (int rc = check_cfl(problem ? problem->cfl : 0.5)) return rc;
    silt_solver* s = nullptr;
    if (int rc = silt_solver_create(problem, nullptr, 0, variant, &s)) return rc;
    int rc = silt_solver_upload(s, field_aos);
    if (!rc) rc = silt_solver_cfl_dt(s, dt);
    const std::string keep = g_err;
    silt_solver_destroy(s);
    g_err = keep;
    return rc;
}

// step_1d/step_2d on a halo-complete PaddedField (include/silt/stepper.hpp:47-54)
int silt_step_padded(const silt_problem* problem, double* padded, double dt, int variant) {
    if (!problem || !padded) return fail(SILT_ERR_INVALID, "silt_step_padded: null argument");
    silt_problem p = *problem;
    for (int k = 0; k < 4; ++k) p.bc[k].type = SILT_BC_GIVEN;
    const int nx = p.nx, ny = p.dim == 1 ? 1 : p.ny;
    const int W = nx + 2;
    std::vector<double> interior(4 * (size_t)nx * ny), west(4 * (size_t)ny), east(4 * (size_t)ny),
        south(4 * (size_t)nx), north(4 * (size_t)nx);
    auto at = [&](int i, int j) { return padded + 4 * ((size_t)(j + 1) * W + (i + 1)); };
    for (int j = 0; j < ny; ++j)
        for (int i = 0; i < nx; ++i) std::memcpy(&interior[4 * ((size_t)j * nx + i)], at(i, j), 32);
    for (int j = 0; j < ny; ++j) {
        std::memcpy(&west[4 * (size_t)j], at(-1, j), 32);
        std::memcpy(&east[4 * (size_t)j], at(nx, j), 32);
    }
    for (int i = 0; i < nx; ++i) {
        std::memcpy(&south[4 * (size_t)i], at(i, -1), 32);
        std::memcpy(&north[4 * (size_t)i], at(i, ny), 32);
    }
    silt_solver* s = nullptr;
    if (int rc = silt_solver_create(&p, nullptr, 0, variant, &s)) return rc;
    int rc = silt_solver_upload(s, interior.data());
    if (!rc) rc = silt_solver_set_ghosts(s, west.data(), east.data(), p.dim == 2 ? south.data() : nullptr,
                                         p.dim == 2 ? north.data() : nullptr);
    silt_run_plan plan{INFINITY, -1, nullptr, 0, 0};
    if (!rc) rc = silt_solver_begin(s, &plan);
    if (!rc) rc = silt_solver_step_fixed(s, dt);
    silt_status st{};
    if (!rc) rc = silt_solver_status(s, &st);
    if (!rc) rc = silt_solver_download(s, interior.data());
    if (!rc)
        for (int j = 0; j < ny; ++j)
            for (int i = 0; i < nx; ++i) std::memcpy(at(i, j), &interior[4 * ((size_t)j * nx + i)], 32);
    const std::string keep = g_err;
    silt_solver_destroy(s);
    g_err = keep;
    return rc;
}

int silt_riemann_batch(const silt_problem* problem, const double* left, const double* right,
                       int64_t n, int axis, int variant, double* out) {
    if (int rc = validate_problem(problem)) return rc;
    if (n <= 0) return SILT_OK;
    CUDA_TRY(cudaSetDevice(0));
    const silt_dev::Params P = make_params(*problem);
    double *dl = nullptr, *dr = nullptr, *dout = nullptr;
    unsigned* derr = nullptr;
    const size_t b4 = 4 * (size_t)n * sizeof(double), b5 = 5 * (size_t)n * sizeof(double);
    CUDA_TRY(cudaMalloc(&dl, b4));
    CUDA_TRY(cudaMalloc(&dr, b4));
    CUDA_TRY(cudaMalloc(&dout, b5));
    CUDA_TRY(cudaMalloc(&derr, sizeof(unsigned)));
    cudaMemset(derr, 0, sizeof(unsigned));
    cudaMemcpy(dl, left, b4, cudaMemcpyHostToDevice);
    cudaMemcpy(dr, right, b4, cudaMemcpyHostToDevice);
    if (variant == SILT_VARIANT_STRICT)
        silt_strict_faces(P, dl, dr, n, axis, dout, derr, 0);
    else
        silt_fast_faces(P, dl, dr, n, axis, dout, derr, 0);
    cudaError_t e = cudaDeviceSynchronize();
    unsigned herr = 0;
    cudaMemcpy(out, dout, b5, cudaMemcpyDeviceToHost);
    cudaMemcpy(&herr, derr, sizeof(unsigned), cudaMemcpyDeviceToHost);
    cudaFree(dl);
    cudaFree(dr);
    cudaFree(dout);
    cudaFree(derr);
    if (e != cudaSuccess) return fail(SILT_ERR_CUDA, cudaGetErrorString(e));
    if (herr)
        return fail(SILT_ERR_RUNTIME,
                    "interface_riemann: no positive fan after 25 celerity enlargements");
    return SILT_OK;
}

int silt_law_batch(const silt_problem* problem, const double* states, int64_t n, int variant,
                   double* out) {
    if (int rc = validate_problem(problem)) return rc;
    if (n <= 0) return SILT_OK;
    CUDA_TRY(cudaSetDevice(0));
    const silt_dev::Params P = make_params(*problem);
    double *dx = nullptr, *dout = nullptr;
    CUDA_TRY(cudaMalloc(&dx, 3 * (size_t)n * sizeof(double)));
    CUDA_TRY(cudaMalloc(&dout, 2 * (size_t)n * sizeof(double)));
    cudaMemcpy(dx, states, 3 * (size_t)n * sizeof(double), cudaMemcpyHostToDevice);
    if (variant == SILT_VARIANT_STRICT)
        silt_strict_law(P, dx, n, dout, 0);
    else
        silt_fast_law(P, dx, n, dout, 0);
    cudaError_t e = cudaMemcpy(out, dout, 2 * (size_t)n * sizeof(double), cudaMemcpyDeviceToHost);
    cudaFree(dx);
    cudaFree(dout);
    if (e != cudaSuccess) return fail(SILT_ERR_CUDA, cudaGetErrorString(e));
    return SILT_OK;
}

int silt_selftest_math(const double* x, const double* y, int64_t n, double* out) {
    if (n <= 0) return SILT_OK;
    CUDA_TRY(cudaSetDevice(0));
    double *dx = nullptr, *dy = nullptr, *dout = nullptr;
    CUDA_TRY(cudaMalloc(&dx, n * sizeof(double)));
    CUDA_TRY(cudaMalloc(&dy, n * sizeof(double)));
    CUDA_TRY(cudaMalloc(&dout, 4 * n * sizeof(double)));
    cudaMemcpy(dx, x, n * sizeof(double), cudaMemcpyHostToDevice);
    cudaMemcpy(dy, y, n * sizeof(double), cudaMemcpyHostToDevice);
    silt_selftest_math_launch(dx, dy, n, dout);
    cudaError_t e = cudaMemcpy(out, dout, 4 * n * sizeof(double), cudaMemcpyDeviceToHost);
    cudaFree(dx);
    cudaFree(dy);
    cudaFree(dout);
    if (e != cudaSuccess) return fail(SILT_ERR_CUDA, cudaGetErrorString(e));
    return SILT_OK;
}

}  // extern "C"

// ---- snapshot CSV (write_snapshot / snapshot_to_string on the device) -------
// src/snapshot.cpp:50-93.  Chunks of rows are formatted by silt_csv.cu into
// device memory, copied into one of two pinned host buffers and handed to the
// sink (file or memory) while the next chunk is formatted.

namespace {

struct CsvSink {
    FILE* fp = nullptr;         // file sink
    char* mem = nullptr;        // memory sink
    int64_t cap = 0, used = 0;  // memory sink capacity / bytes produced
    std::string path;
    bool failed = false;
    void write(const char* p, size_t n) {
        if (fp) {
            if (n && std::fwrite(p, 1, n, fp) != n) failed = true;
        } else {
            if (mem && used + (int64_t)n <= cap) std::memcpy(mem + used, p, n);
        }
        used += (int64_t)n;
    }
};

struct CsvCtx {
    int device = 0;
    int chunk_cells = 0;
    silt_csv::Pow5Table* table = nullptr;
    char* stage = nullptr;
    int* len = nullptr;
    int* off = nullptr;
    void* temp = nullptr;
    size_t temp_bytes = 0;
    char* out = nullptr;
    double* field = nullptr;  // device copy of host rows
    char* host[2] = {nullptr, nullptr};
    int* tail = nullptr;      // pinned: {off[n-1], len[n-1]}
    cudaStream_t stream = nullptr;
    cudaEvent_t copied[2] = {nullptr, nullptr};
};

std::mutex g_csv_mu;
std::map<int, CsvCtx*> g_csv;

int csv_ctx(int device, CsvCtx** out) {
    std::lock_guard<std::mutex> lock(g_csv_mu);
    auto it = g_csv.find(device);
    if (it != g_csv.end()) {
        *out = it->second;
        return SILT_OK;
    }
    CUDA_TRY(cudaSetDevice(device));
    auto* c = new CsvCtx();
    c->device = device;
    c->chunk_cells = 1 << 21;
    const size_t n = (size_t)c->chunk_cells;
    silt_csv::Pow5Table host_table;
    silt_csv::build_pow5(host_table);
    CUDA_TRY(cudaMalloc(&c->table, sizeof(silt_csv::Pow5Table)));
    CUDA_TRY(cudaMemcpy(c->table, &host_table, sizeof host_table, cudaMemcpyHostToDevice));
    CUDA_TRY(cudaMalloc(&c->stage, n * kCsvRowMax));
    CUDA_TRY(cudaMalloc(&c->len, n * sizeof(int)));
    CUDA_TRY(cudaMalloc(&c->off, n * sizeof(int)));
    c->temp_bytes = silt_csv_scan_temp_bytes((int)n);
    CUDA_TRY(cudaMalloc(&c->temp, c->temp_bytes));
    CUDA_TRY(cudaMalloc(&c->out, n * kCsvRowMax));
    CUDA_TRY(cudaMalloc(&c->field, 4 * n * sizeof(double)));
    for (int b = 0; b < 2; ++b) {
        CUDA_TRY(cudaHostAlloc(&c->host[b], n * kCsvRowMax, cudaHostAllocPortable));
        CUDA_TRY(cudaEventCreateWithFlags(&c->copied[b], cudaEventDisableTiming));
    }
    CUDA_TRY(cudaHostAlloc(&c->tail, 2 * sizeof(int), cudaHostAllocPortable));
    CUDA_TRY(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    g_csv[device] = c;
    *out = c;
    return SILT_OK;
}

// rows [0, rows) of field F (device) -> CSV; F may instead be host AoS
// (host_aos != nullptr), copied chunk by chunk.
int csv_emit(int device, CsvField F, const double* host_aos, const silt_problem& p, int rows,
             int j0, double time, bool header, CsvSink& sink) {
    CsvCtx* c = nullptr;
    if (int rc = csv_ctx(device, &c)) return rc;
    std::lock_guard<std::mutex> lock(g_csv_mu);  // one emitter per process at a time
    CUDA_TRY(cudaSetDevice(device));
    const int dim = p.dim;
    if (header) {
        const char* h = dim == 1 ? "x,h,u,zb,eta,time\n" : "x,y,h,u,v,zb,eta,time\n";
        sink.write(h, std::strlen(h));
    }
    const int nx = p.nx;
    int chunk_cells = c->chunk_cells;
    if (const char* e = std::getenv("SILT_CSV_CHUNK"))  // smaller chunks (tests)
        chunk_cells = std::max(1, std::min(chunk_cells, std::atoi(e)));
    const int crow = std::max(1, chunk_cells / nx);
    if ((long long)nx > chunk_cells)
        return fail(SILT_ERR_UNSUPPORTED, "write_snapshot: rows longer than the chunk size");
    int pending = -1;  // host buffer holding the previous chunk
    int64_t pending_bytes = 0;
    for (int r0 = 0, chunk = 0; r0 < rows; r0 += crow, ++chunk) {
        const int nr = std::min(crow, rows - r0);
        const int n = nr * nx;
        CsvField G = F;
        if (host_aos) {
            CUDA_TRY(cudaMemcpyAsync(c->field, host_aos + 4 * (size_t)r0 * nx,
                                     4 * (size_t)n * sizeof(double), cudaMemcpyHostToDevice,
                                     c->stream));
            for (int f = 0; f < 4; ++f) G.f[f] = c->field + f;
            G.row_stride = 4LL * nx;
            G.col_stride = 4;
        } else {
            for (int f = 0; f < 4; ++f) G.f[f] = F.f[f] + (long long)r0 * F.row_stride;
        }
        CsvGeom geo{nx, nr, j0 + r0, dim, p.dx, p.dy, p.h_dry, time};
        silt_csv_format_launch(G, geo, c->table, c->stage, c->len, c->stream);
        silt_csv_scan(c->len, c->off, n, c->temp, c->temp_bytes, c->stream);
        silt_csv_compact_launch(c->stage, c->len, c->off, n, c->out, c->stream);
        CUDA_TRY(cudaGetLastError());
        CUDA_TRY(cudaMemcpyAsync(&c->tail[0], c->off + (n - 1), sizeof(int),
                                 cudaMemcpyDeviceToHost, c->stream));
        CUDA_TRY(cudaMemcpyAsync(&c->tail[1], c->len + (n - 1), sizeof(int),
                                 cudaMemcpyDeviceToHost, c->stream));
        CUDA_TRY(cudaStreamSynchronize(c->stream));
        const int64_t bytes = (int64_t)c->tail[0] + c->tail[1];
        const int b = chunk & 1;
        CUDA_TRY(cudaMemcpyAsync(c->host[b], c->out, (size_t)bytes, cudaMemcpyDeviceToHost,
                                 c->stream));
        CUDA_TRY(cudaEventRecord(c->copied[b], c->stream));
        if (pending >= 0) {  // the host writes chunk k-1 while chunk k is copied
            CUDA_TRY(cudaEventSynchronize(c->copied[pending]));
            sink.write(c->host[pending], (size_t)pending_bytes);
        }
        pending = b;
        pending_bytes = bytes;
        // the next chunk's compaction overwrites c->out: order it after this copy
    }
    if (pending >= 0) {
        CUDA_TRY(cudaEventSynchronize(c->copied[pending]));
        sink.write(c->host[pending], (size_t)pending_bytes);
    }
    return SILT_OK;
}

bool is_device_ptr(const void* p) {
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

CsvField aos_field(const double* aos, int nx) {
    CsvField F;
    for (int f = 0; f < 4; ++f) F.f[f] = aos + f;
    F.row_stride = 4LL * nx;
    F.col_stride = 4;
    return F;
}

int open_sink(CsvSink& sink, const char* path, bool append) {
    sink.path = path;
    sink.fp = std::fopen(path, append ? "ab" : "wb");
    if (!sink.fp)
        return fail(SILT_ERR_RUNTIME, std::string("cannot open '") + path + "' for writing");
    return SILT_OK;
}

int close_sink(CsvSink& sink, int rc) {
    if (sink.fp) {
        if (std::fclose(sink.fp) != 0) sink.failed = true;
        sink.fp = nullptr;
    }
    if (rc) return rc;
    if (sink.failed) return fail(SILT_ERR_RUNTIME, "failed writing '" + sink.path + "'");
    return SILT_OK;
}

int check_rows(const silt_problem* p, int64_t j0, int64_t rows) {
    if (int rc = validate_problem(p)) return rc;
    const int64_t gny = p->dim == 1 ? 1 : p->ny;
    if (j0 < 0 || rows < 0 || j0 + rows > gny)
        return fail(SILT_ERR_INVALID, "write_snapshot: rows outside the grid");
    return SILT_OK;
}

}  // namespace

extern "C" {

int silt_snapshot_to_string(const silt_problem* problem, const double* aos, int64_t j0,
                            int64_t rows, double time, int header, char* out, int64_t cap,
                            int64_t* len) {
    if (!aos || !len) return fail(SILT_ERR_INVALID, "silt_snapshot_to_string: null argument");
    if (int rc = check_rows(problem, j0, rows)) return rc;
    const bool dev = is_device_ptr(aos);
    int device = 0;
    if (dev) {
        cudaPointerAttributes a{};
        CUDA_TRY(cudaPointerGetAttributes(&a, aos));
        device = a.device;
    }
    CsvSink sink;
    sink.mem = out;
    sink.cap = out ? cap : 0;
    const int rc = csv_emit(device, aos_field(dev ? aos : nullptr, problem->nx),
                            dev ? nullptr : aos, *problem, (int)rows, (int)j0, time, header != 0,
                            sink);
    *len = sink.used;
    if (rc) return rc;
    if (sink.used > sink.cap)
        return fail(SILT_ERR_INVALID, "silt_snapshot_to_string: buffer too small (see *len)");
    return SILT_OK;
}

int silt_write_snapshot(const silt_problem* problem, const double* aos, int64_t j0, int64_t rows,
                        double time, const char* path, int append, int64_t* bytes) {
    if (!aos || !path) return fail(SILT_ERR_INVALID, "silt_write_snapshot: null argument");
    if (int rc = check_rows(problem, j0, rows)) return rc;
    const bool dev = is_device_ptr(aos);
    int device = 0;
    if (dev) {
        cudaPointerAttributes a{};
        CUDA_TRY(cudaPointerGetAttributes(&a, aos));
        device = a.device;
    }
    CsvSink sink;
    if (int rc = open_sink(sink, path, append != 0)) return rc;
    int rc = csv_emit(device, aos_field(dev ? aos : nullptr, problem->nx), dev ? nullptr : aos,
                      *problem, (int)rows, (int)j0, time, append == 0, sink);
    rc = close_sink(sink, rc);
    if (bytes) *bytes = sink.used;
    return rc;
}

int silt_solver_write_snapshot(silt_solver* s, double time, const char* path, int append,
                               int64_t* bytes) {
    if (!s || !path) return fail(SILT_ERR_INVALID, "silt_solver_write_snapshot: null argument");
    int p = 0;
    if (s->begun) {
        Slot sl;
        if (int rc = read_slot(s, &sl, nullptr)) return rc;
        p = (int)(sl.steps & 1);
    } else {
        CUDA_TRY(cudaSetDevice(s->device));
        CUDA_TRY(cudaStreamSynchronize(s->stream));
    }
    CsvField F;
    for (int f = 0; f < 4; ++f) F.f[f] = s->args.state[p][f];
    F.row_stride = s->pitch;
    F.col_stride = 1;
    CsvSink sink;
    if (int rc = open_sink(sink, path, append != 0)) return rc;
    int rc = csv_emit(s->device, F, nullptr, s->prob, s->ny, s->strip.j0, time, append == 0, sink);
    rc = close_sink(sink, rc);
    if (bytes) *bytes = sink.used;
    return rc;
}

int silt_group_write_snapshot(silt_group* g, double time, const char* path, int64_t* bytes) {
    if (!g || !path) return fail(SILT_ERR_INVALID, "silt_group_write_snapshot: null argument");
    int64_t total = 0;
    for (size_t k = 0; k < g->strips.size(); ++k) {
        int64_t b = 0;
        if (int rc = silt_solver_write_snapshot(g->strips[k], time, path, k > 0, &b)) return rc;
        total += b;
    }
    if (bytes) *bytes = total;
    return SILT_OK;
}

}  // extern "C"

// ---- asynchronous CSV snapshot ---------------------------------------------------
// write_snapshot of a paused run without holding it: the state is copied into
// the snapshot buffer on the solver's stream, the run resumes, and a host
// thread formats the buffer on the device (CSV stream, concurrent with the
// next steps) and writes the file.  silt_solver_capture_wait joins it.
extern "C" int silt_solver_capture_write(silt_solver* s, double time, const char* path,
                                         int append) {
    if (!s || !path) return fail(SILT_ERR_INVALID, "silt_solver_capture_write: null argument");
    if (!s->begun) return fail(SILT_ERR_INVALID, "silt_solver_capture_write: run not begun");
    if (int rc = silt_solver_capture_wait(s)) return rc;
    CUDA_TRY(cudaSetDevice(s->device));
    const size_t bytes = 4 * (size_t)s->nx * s->ny * sizeof(double);
    if (!s->snapbuf) {
        CUDA_TRY(cudaMalloc(&s->snapbuf, bytes));
        CUDA_TRY(cudaStreamCreateWithFlags(&s->copy_stream, cudaStreamNonBlocking));
        CUDA_TRY(cudaEventCreateWithFlags(&s->cap_ready, cudaEventDisableTiming));
        CUDA_TRY(cudaEventCreateWithFlags(&s->cap_done, cudaEventDisableTiming));
    }
    Slot sl;
    if (int rc = read_slot(s, &sl, nullptr)) return rc;
    if (sl.state != SILT_STATE_PAUSED)
        return fail(SILT_ERR_INVALID, "silt_solver_capture_write: solver is not paused");
    const int p = (int)(sl.steps & 1);
    const StepArgs& A = s->args;
    soa_to_aos<<<grid_blocks((long long)s->nx * s->ny, 256), 256, 0, s->stream>>>(
        s->snapbuf, A.state[p][0], A.state[p][1], A.state[p][2], A.state[p][3], s->nx, s->ny,
        s->pitch);
    ++s->kernel_count;
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaEventRecord(s->cap_ready, s->stream));
    int st = SILT_STATE_RUNNING;
    Slot* slot = &s->ctl->slot[s->launches % 3];
    CUDA_TRY(cudaMemcpy(&slot->state, &st, sizeof(int), cudaMemcpyHostToDevice));
    const std::string file(path);
    s->writer_rc = SILT_OK;
    s->writer_busy.store(true, std::memory_order_relaxed);
    s->writer = std::thread([s, time, file, append] {
        cudaSetDevice(s->device);
        if (cudaEventSynchronize(s->cap_ready) != cudaSuccess) {
            s->writer_rc = SILT_ERR_CUDA;
            s->writer_err = "silt_solver_capture_write: capture failed";
            return;
        }
        CsvSink sink;
        int rc = open_sink(sink, file.c_str(), append != 0);
        if (rc == SILT_OK) {
            rc = csv_emit(s->device, aos_field(s->snapbuf, s->nx), nullptr, s->prob, s->ny,
                          s->strip.j0, time, append == 0, sink);
            rc = close_sink(sink, rc);
        }
        s->writer_rc = rc;
        if (rc != SILT_OK) s->writer_err = silt_last_error();
        s->writer_busy.store(false, std::memory_order_release);
    });
    return SILT_OK;
}

// ---- multi-process strips over peer memory ----------------------------------------
namespace {

// Process-wide registry of IPC handles.  A process may own several strips
// ("pieces", distributed.PieceRunner) that connect to the same remote
// buffers, and a piece's neighbour may live in the same process: handles this
// process exported resolve to the local pointer (CUDA refuses to open them),
// remote ones are opened once and reference-counted.
struct IpcEntry {
    void* ptr = nullptr;
    int refs = 0;
    bool local = false;
};
std::mutex g_ipc_mu;
std::map<std::string, IpcEntry>& ipc_registry() {
    static std::map<std::string, IpcEntry> m;
    return m;
}

std::string ipc_key(const cudaIpcMemHandle_t& h) {
    return std::string(reinterpret_cast<const char*>(&h), sizeof h);
}

int ipc_export(void* ptr, cudaIpcMemHandle_t* h) {
    CUDA_TRY(cudaIpcGetMemHandle(h, ptr));
    std::lock_guard<std::mutex> lk(g_ipc_mu);
    IpcEntry& e = ipc_registry()[ipc_key(*h)];
    e.ptr = ptr;
    e.local = true;
    return SILT_OK;
}

int ipc_open(const cudaIpcMemHandle_t& h, void** out) {
    std::lock_guard<std::mutex> lk(g_ipc_mu);
    auto& reg = ipc_registry();
    auto it = reg.find(ipc_key(h));
    if (it != reg.end() && (it->second.local || it->second.refs > 0)) {
        if (!it->second.local) ++it->second.refs;
        *out = it->second.ptr;
        return SILT_OK;
    }
    void* p = nullptr;
    CUDA_TRY(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
    IpcEntry& e = reg[ipc_key(h)];
    e.ptr = p;
    e.refs = 1;
    e.local = false;
    *out = p;
    return SILT_OK;
}

void ipc_close(void* p) {
    std::lock_guard<std::mutex> lk(g_ipc_mu);
    auto& reg = ipc_registry();
    for (auto it = reg.begin(); it != reg.end(); ++it) {
        if (it->second.ptr != p || it->second.local) continue;
        if (--it->second.refs <= 0) {
            cudaIpcCloseMemHandle(p);
            reg.erase(it);
        }
        return;
    }
}

// A local buffer about to be freed: drop its exported handle.
void ipc_forget_local(void* p) {
    if (!p) return;
    std::lock_guard<std::mutex> lk(g_ipc_mu);
    auto& reg = ipc_registry();
    for (auto it = reg.begin(); it != reg.end();) {
        if (it->second.local && it->second.ptr == p)
            it = reg.erase(it);
        else
            ++it;
    }
}

// Bound of the per-step wait for the peers (SILT_P2P_TIMEOUT_MS, default 60 s).
unsigned long long p2p_timeout_ns() {
    static const unsigned long long ns = [] {
        const char* e = std::getenv("SILT_P2P_TIMEOUT_MS");
        const long long ms = e ? std::atoll(e) : 60000;
        return (unsigned long long)(ms > 0 ? ms : 60000) * 1000000ull;
    }();
    return ns;
}

}  // namespace

extern "C" int silt_solver_p2p_export(silt_solver* s, silt_p2p_handle* out) {
    if (!s || !out) return fail(SILT_ERR_INVALID, "silt_solver_p2p_export: null argument");
    if (s->prob.dim != 2) return fail(SILT_ERR_UNSUPPORTED, "p2p: 2D strips only");
    CUDA_TRY(cudaSetDevice(s->device));
    if (!s->p2p_flags) {
        CUDA_TRY(cudaMalloc(&s->p2p_flags, 64 * sizeof(unsigned)));
        CUDA_TRY(cudaMemset(s->p2p_flags, 0, 64 * sizeof(unsigned)));
    }
    std::memset(out, 0, sizeof *out);
    cudaIpcMemHandle_t h;
    if (int rc = ipc_export(s->rows, &h)) return rc;
    std::memcpy(out->rows, &h, sizeof h);
    if (int rc = ipc_export(s->ctl, &h)) return rc;
    std::memcpy(out->ctl, &h, sizeof h);
    if (int rc = ipc_export(s->p2p_flags, &h)) return rc;
    std::memcpy(out->flags, &h, sizeof h);
    out->nx = s->nx;
    return SILT_OK;
}

extern "C" int silt_solver_p2p_connect(silt_solver* s, int rank, int world,
                                       const silt_p2p_handle* all, int south, int north) {
    if (!s || !all) return fail(SILT_ERR_INVALID, "silt_solver_p2p_connect: null argument");
    if (world < 2 || world > 64 || rank < 0 || rank >= world)
        return fail(SILT_ERR_INVALID, "p2p: 2 <= world <= 64, 0 <= rank < world");
    if (!s->p2p_flags) return fail(SILT_ERR_INVALID, "p2p: export before connect");
    if ((south >= 0) != (bool)s->strip.south_neighbor || (north >= 0) != (bool)s->strip.north_neighbor)
        return fail(SILT_ERR_INVALID, "p2p: neighbours do not match the strip");
    CUDA_TRY(cudaSetDevice(s->device));
    std::vector<void*> rows(world, nullptr), ctls(world, nullptr), flags(world, nullptr);
    for (int j = 0; j < world; ++j) {
        if (j == rank) continue;
        if (all[j].nx != s->nx) return fail(SILT_ERR_INVALID, "p2p: strips of different widths");
        cudaIpcMemHandle_t h;
        std::memcpy(&h, all[j].ctl, sizeof h);
        if (int rc = ipc_open(h, &ctls[j])) return rc;
        s->p2p_opened.push_back(ctls[j]);
        std::memcpy(&h, all[j].flags, sizeof h);
        if (int rc = ipc_open(h, &flags[j])) return rc;
        s->p2p_opened.push_back(flags[j]);
        if (j == south || j == north) {
            std::memcpy(&h, all[j].rows, sizeof h);
            if (int rc = ipc_open(h, &rows[j])) return rc;
            s->p2p_opened.push_back(rows[j]);
        }
    }
    const size_t row = 4 * (size_t)s->nx;
    StepArgs& A = s->args;
    A.recv_s[1] = s->rows + 8 * row;  // second parity of the receive rows
    A.recv_n[1] = s->rows + 9 * row;
    for (int q = 0; q < 2; ++q) {
        if (south >= 0) A.send_s[q] = static_cast<double*>(rows[south]) + (q ? 9 : 5) * row;
        if (north >= 0) A.send_n[q] = static_cast<double*>(rows[north]) + (q ? 8 : 4) * row;
    }
    std::vector<Control*> others;
    s->p2p_peer_flag.clear();
    for (int j = 0; j < world; ++j) {
        if (j == rank) continue;
        others.push_back(static_cast<Control*>(ctls[j]));
        s->p2p_peer_flag.push_back(static_cast<unsigned*>(flags[j]) + rank);
    }
    CUDA_TRY(cudaMalloc(&s->p2p_peer_ctl, others.size() * sizeof(Control*)));
    CUDA_TRY(cudaMemcpy(s->p2p_peer_ctl, others.data(), others.size() * sizeof(Control*),
                        cudaMemcpyHostToDevice));
    CUDA_TRY(cudaMalloc(&s->p2p_peer_flag_dev, s->p2p_peer_flag.size() * sizeof(unsigned*)));
    CUDA_TRY(cudaMemcpy(s->p2p_peer_flag_dev, s->p2p_peer_flag.data(),
                        s->p2p_peer_flag.size() * sizeof(unsigned*), cudaMemcpyHostToDevice));
    // probe the mechanism once (remote atomics, remote flag writes, the
    // acquire) so that a driver can fall back before its first step
    {
        push_release_kernel<<<1, 32, 0, s->stream>>>(s->ctl, 0, s->p2p_peer_ctl,
                                                     s->p2p_peer_flag_dev, world - 1,
                                                     s->p2p_count);
        CUDA_TRY(cudaGetLastError());
        acquire_flags_kernel<<<1, 32, 0, s->stream>>>(s->p2p_flags, world, rank, 0u, s->ctl, 0,
                                                      p2p_timeout_ns());
        CUDA_TRY(cudaGetLastError());
        CUDA_TRY(cudaStreamSynchronize(s->stream));
    }
    s->p2p_rank = rank;
    s->p2p_world = world;
    s->begun_after_connect = false;
    return SILT_OK;
}

extern "C" int silt_solver_p2p_step(silt_solver* s, int n) {
    if (!s) return fail(SILT_ERR_INVALID, "null solver");
    if (s->p2p_world < 2) return fail(SILT_ERR_INVALID, "silt_solver_p2p_step: not connected");
    if (!s->begun || !s->begun_after_connect)
        return fail(SILT_ERR_INVALID, "silt_solver_p2p_step: call silt_solver_begin after connect");
    if (int rc = check_cfl(s->prob.cfl)) return rc;
    CUDA_TRY(cudaSetDevice(s->device));
    const unsigned long long timeout = p2p_timeout_ns();
    for (int k = 0; k < n; ++k) {
        const unsigned c = ++s->p2p_count;
        if (c > 1) {
            // every rank finished step c-1 (its rows and maxima are here): one
            // warp acquires the peers' flags at system scope, with a bounded
            // wait, so the step observes the peers' writes
            acquire_flags_kernel<<<1, 32, 0, s->stream>>>(s->p2p_flags, s->p2p_world, s->p2p_rank,
                                                          c - 1, s->ctl, (int)(s->launches % 3),
                                                          timeout);
            ++s->kernel_count;
        }
        launch_step(s);
        push_release_kernel<<<1, 32, 0, s->stream>>>(s->ctl, (int)(s->launches % 3),
                                                     s->p2p_peer_ctl, s->p2p_peer_flag_dev,
                                                     s->p2p_world - 1, c);
        ++s->kernel_count;
        CUDA_TRY(cudaGetLastError());
    }
    return SILT_OK;
}
