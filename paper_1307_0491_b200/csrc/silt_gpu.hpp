// silt_gpu.hpp — C++ drop-in for the reference's time-stepping API on B200.
//
// Header-only layer over the C ABI (include/silt_cuda.h, libsilt_b200.so).
// It takes the reference's OWN types from its public headers (silt::Field,
// PaddedField, BedloadLaw, Physics, Scenario, RunOptions, RunResult — the
// reference install's <silt/...> headers), so a caller switches the hot path by
// calling silt::gpu::X instead of silt::X:
//
//   silt::cfl_dt      (include/silt/stepper.hpp:38-41)   -> silt::gpu::cfl_dt
//   silt::step_1d/2d  (include/silt/stepper.hpp:47-54)   -> silt::gpu::step_1d/2d
//   silt::run_serial  (include/silt/parallel.hpp:80)     -> silt::gpu::run_serial
//   silt::run_parallel(include/silt/parallel.hpp:85-86)  -> silt::gpu::run_parallel
//   silt::write_snapshot / snapshot_to_string (io.hpp:69-73) -> silt::gpu::write_snapshot / ...
//
// Same argument meaning, same exception classes and messages:
// std::invalid_argument for preconditions, std::runtime_error for numerical
// failure (negative depth, no positive Riemann fan).  Differences, by design:
//   * both law kinds (Grass, Shields x 5 formulas x 2 friction models) run on
//     the GPU; there is no CPU fallback;
//   * run_parallel(sc, px, py) validates px/py like partition() and runs
//     px * py row strips (columns are never split: every layout is bitwise
//     identical, tests/test_parallel.cpp:215-238), strip k on CUDA device
//     k % devices; a 1D line is one strip;
//   * RunResult::timing holds one WorkerTiming per strip: compute_seconds is
//     the strip's step-kernel time on its device (CUDA events,
//     silt_group_timing), exchange_seconds the rest of the run loop's wall
//     time (halo/maxima delivery, waits on other strips, snapshot gathers).
#pragma once

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "silt/parallel.hpp"
#include "silt/scenarios.hpp"
#include "silt/stepper.hpp"
#include "silt_cuda.h"

namespace silt {
namespace gpu {

// SILT_VARIANT_FAST (default) or SILT_VARIANT_STRICT (bit-identical to the CPU
// reference, slower).
inline int& variant() {
    static thread_local int v = SILT_VARIANT_FAST;
    return v;
}

inline void check(int rc) {
    if (rc == SILT_OK) return;
    const std::string msg = silt_last_error();
    if (rc == SILT_ERR_INVALID || rc == SILT_ERR_UNSUPPORTED) throw std::invalid_argument(msg);
    throw std::runtime_error(msg);
}

namespace detail {

inline silt_problem problem(const Grid& g, const BedloadLaw& law, const Physics& phys, double cfl,
                            double safety) {
    silt_problem p{};
    p.dim = g.dim;
    p.nx = g.nx;
    p.ny = g.dim == 1 ? 1 : g.ny;
    p.law_kind = law.kind == BedloadLaw::Kind::Grass ? SILT_LAW_GRASS : SILT_LAW_SHIELDS;
    p.shields_formula = static_cast<int32_t>(law.formula);
    p.friction_model = law.friction.model == FrictionModel::Manning ? SILT_FRICTION_MANNING
                                                                    : SILT_FRICTION_DARCY_WEISBACH;
    p.tau_cr = law.tau_cr;
    p.grain_diameter = law.grain_diameter;
    p.rel_density = law.rel_density;
    p.friction_coef = law.friction.coefficient;
    p.dx = g.dx;
    p.dy = g.dim == 1 ? 1.0 : g.dy;
    p.gravity = phys.gravity;
    p.h_dry = phys.h_dry;
    p.a_g = law.a_g;
    p.m_g = law.m_g;
    p.cfl = cfl;
    p.safety = safety;
    for (int s = 0; s < 4; ++s) p.bc[s] = silt_bc{SILT_BC_GIVEN, 0, 0.0, 0.0};
    return p;
}

inline void set_bcs(silt_problem& p, const std::array<BoundarySpec, 4>& bc) {
    for (int s = 0; s < 4; ++s)
        p.bc[s] = silt_bc{static_cast<int32_t>(bc[s].type), bc[s].supercritical ? 1 : 0, bc[s].q0,
                          bc[s].h0};
}

inline const double* data(const std::vector<FlowState>& v) {
    static_assert(sizeof(FlowState) == 4 * sizeof(double), "FlowState must be 4 doubles");
    return reinterpret_cast<const double*>(v.data());
}
inline double* data(std::vector<FlowState>& v) { return reinterpret_cast<double*>(v.data()); }

}  // namespace detail

// cfl_dt (include/silt/stepper.hpp:38-41)
inline double cfl_dt(const Field& f, const BedloadLaw& law, const Physics& phys, double cfl) {
    silt_problem p = detail::problem(f.grid, law, phys, cfl, 1.0);
    for (int s = 0; s < 4; ++s) p.bc[s].type = SILT_BC_OUTFLOW;
    double dt = 0;
    check(silt_cfl_dt(&p, detail::data(f.cells), variant(), &dt));
    return dt;
}

inline double cfl_dt(const PaddedField& f, const BedloadLaw& law, const Physics& phys, double cfl) {
    return gpu::cfl_dt(f.interior(), law, phys, cfl);
}

// step_1d / step_2d on a halo-complete PaddedField (include/silt/stepper.hpp:47-54)
inline void step_1d(PaddedField& f, const BedloadLaw& law, const Physics& phys, double dt,
                    double safety) {
    if (f.grid.dim != 1) throw std::invalid_argument("step_1d: grid must be 1D");
    silt_problem p = detail::problem(f.grid, law, phys, 0.5, safety);
    check(silt_step_padded(&p, detail::data(f.cells), dt, variant()));
}

inline void step_2d(PaddedField& f, const BedloadLaw& law, const Physics& phys, double dt,
                    double safety) {
    if (f.grid.dim != 2) throw std::invalid_argument("step_2d: grid must be 2D");
    silt_problem p = detail::problem(f.grid, law, phys, 0.5, safety);
    check(silt_step_padded(&p, detail::data(f.cells), dt, variant()));
}

namespace detail {

class Group {
  public:
    Group(const silt_problem& p, int py) {
        int n = 0;
        check(silt_device_count(&n));
        if (n < 1) throw std::runtime_error("silt::gpu: no CUDA device");
        std::vector<int> devs(n);
        for (int k = 0; k < n; ++k) devs[k] = k;
        check(silt_group_create(&p, py, devs.data(), n, variant(), &g_));
    }
    ~Group() { silt_group_destroy(g_); }
    Group(const Group&) = delete;
    Group& operator=(const Group&) = delete;
    silt_group* get() const { return g_; }

  private:
    silt_group* g_ = nullptr;
};

// page-locked host memory for asynchronous snapshot captures
struct PinnedBuffer {
    double* ptr = nullptr;
    size_t bytes = 0;
    void alloc(size_t n) {
        void* p = nullptr;
        check(silt_host_alloc(static_cast<int64_t>(n), &p));
        ptr = static_cast<double*>(p);
        bytes = n;
    }
    ~PinnedBuffer() {
        if (ptr) silt_host_free(ptr);
    }
};

// make_plan + the run loop of run_serial / run_parallel
// (src/parallel.cpp:101-132, 208-259, 261-386)
inline RunResult run(const Scenario& sc, int py, const RunOptions& opt) {
    const auto wall0 = std::chrono::steady_clock::now();
    const double t_end = opt.t_end >= 0 ? opt.t_end : sc.t_end;
    const double cfl = opt.cfl > 0 ? opt.cfl : sc.cfl;
    const double safety = opt.safety > 0 ? opt.safety : sc.safety;
    if (!(t_end >= 0)) throw std::invalid_argument("run: t_end must be >= 0");
    silt_problem p = problem(sc.grid, sc.law, sc.phys, cfl, safety);
    set_bcs(p, sc.bc);
    bool snap_initial = false;
    for (double s : opt.snapshot_times)
        if (s == 0) snap_initial = true;
    PinnedBuffer pinned;  // declared before the group: outlives any in-flight copy
    Group g(p, py);
    check(silt_group_upload(g.get(), data(sc.initial.cells)));
    if (snap_initial && opt.on_snapshot) opt.on_snapshot(0.0, sc.initial);
    silt_run_plan plan{t_end, opt.max_steps, opt.snapshot_times.data(),
                       static_cast<int32_t>(opt.snapshot_times.size()), 0};
    check(silt_group_begin(g.get(), &plan));
    check(silt_group_timing(g.get(), 1, nullptr));  // WorkerTiming.compute_seconds from here
    const auto loop0 = std::chrono::steady_clock::now();
    silt_status st{};
    // Snapshots are gathered asynchronously: the paused state is captured on
    // the device, the run resumes, and the copy streams into page-locked host
    // memory while the next steps execute; on_snapshot runs once it landed.
    Field snap(sc.grid);
    double pending_t = -1;
    auto deliver = [&] {
        if (pending_t < 0) return;
        check(silt_group_capture_wait(g.get()));
        std::memcpy(data(snap.cells), pinned.ptr, pinned.bytes);
        opt.on_snapshot(pending_t, snap);
        pending_t = -1;
    };
    for (;;) {
        check(silt_group_step(g.get(), 16));
        check(silt_group_status(g.get(), &st));
        if (st.state == SILT_STATE_PAUSED) {
            if (opt.on_snapshot) {
                deliver();
                if (!pinned.ptr) pinned.alloc(snap.cells.size() * sizeof(FlowState));
                check(silt_group_capture_resume(g.get(), pinned.ptr));
                pending_t = st.t;
            } else {
                check(silt_group_resume(g.get()));
            }
            continue;
        }
        if (st.state == SILT_STATE_DONE) break;
    }
    deliver();
    std::vector<double> compute(py, 0.0);
    check(silt_group_timing(g.get(), 0, compute.data()));
    const double loop_s =
        std::chrono::duration<double>(std::chrono::steady_clock::now() - loop0).count();
    RunResult res;
    res.final_field = Field(sc.grid);
    check(silt_group_download(g.get(), data(res.final_field.cells)));
    res.time = st.t;
    res.steps = st.steps;
    // The reference's split (src/parallel.cpp:318-361): compute = local CFL +
    // stepping, exchange = ghost fill, gathers and synchronisation.  Here
    // compute is the strip's step-kernel time on its device (the fused step
    // includes the next CFL reduction); the rest of the run loop's wall time —
    // halo delivery, the maxima exchange, waits on the other strips, snapshot
    // gathers and host round trips — is exchange.
    for (int r = 0; r < py; ++r) {
        WorkerTiming w;
        w.rank = r;
        w.steps = st.steps;
        w.compute_seconds = compute[r];
        w.exchange_seconds = loop_s > compute[r] ? loop_s - compute[r] : 0.0;
        res.timing.push_back(w);
    }
    res.wall_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - wall0).count();
    return res;
}

}  // namespace detail

// snapshot_to_string / write_snapshot (include/silt/io.hpp:69-73), formatted
// on the GPU (silt_csv.cu): the same bytes as the reference's.
inline std::string snapshot_to_string(const Field& f, double time, const Physics& phys = {}) {
    silt_problem p = detail::problem(f.grid, BedloadLaw::grass(0.0), phys, 0.5, 1.0);
    const int64_t rows = f.grid.dim == 1 ? 1 : f.grid.ny;
    int64_t len = 0;
    const int rc = silt_snapshot_to_string(&p, detail::data(f.cells), 0, rows, time, 1, nullptr,
                                           0, &len);
    if (rc != SILT_OK && !(rc == SILT_ERR_INVALID && len > 0)) check(rc);
    std::string out(static_cast<size_t>(len), '\0');
    check(silt_snapshot_to_string(&p, detail::data(f.cells), 0, rows, time, 1, out.data(), len,
                                  &len));
    return out;
}

inline void write_snapshot(const Field& f, double time, const std::string& path,
                           const Physics& phys = {}) {
    silt_problem p = detail::problem(f.grid, BedloadLaw::grass(0.0), phys, 0.5, 1.0);
    const int64_t rows = f.grid.dim == 1 ? 1 : f.grid.ny;
    check(silt_write_snapshot(&p, detail::data(f.cells), 0, rows, time, path.c_str(), 0,
                              nullptr));
}

// run_serial (include/silt/parallel.hpp:80)
inline RunResult run_serial(const Scenario& sc, const RunOptions& opt = {}) {
    if ((sc.bc[0].type == BcType::Periodic) != (sc.bc[1].type == BcType::Periodic))
        throw std::invalid_argument("apply_bcs: periodic requires both x sides");
    if (sc.grid.dim == 2 &&
        (sc.bc[2].type == BcType::Periodic) != (sc.bc[3].type == BcType::Periodic))
        throw std::invalid_argument("apply_bcs: periodic requires both y sides");
    return detail::run(sc, 1, opt);
}

// run_parallel (include/silt/parallel.hpp:85-86)
inline RunResult run_parallel(const Scenario& sc, int px, int py, const RunOptions& opt = {}) {
    const double t_end = opt.t_end >= 0 ? opt.t_end : sc.t_end;
    if (!(t_end >= 0)) throw std::invalid_argument("run: t_end must be >= 0");
    if ((sc.bc[0].type == BcType::Periodic) != (sc.bc[1].type == BcType::Periodic))
        throw std::invalid_argument("run_parallel: periodic requires both x sides");
    if (sc.grid.dim == 2 &&
        (sc.bc[2].type == BcType::Periodic) != (sc.bc[3].type == BcType::Periodic))
        throw std::invalid_argument("run_parallel: periodic requires both y sides");
    if (px < 1 || py < 1) throw std::invalid_argument("partition: worker counts must be >= 1");
    if (sc.grid.dim == 1 && py != 1)
        throw std::invalid_argument("partition: 1D grids require py == 1");
    if (px > sc.grid.nx || py > sc.grid.ny)
        throw std::invalid_argument("partition: every worker needs at least one cell per axis");
    // The GPU decomposition is row strips: a px x py layout runs as px * py
    // strips (capped at one row each; a 1D line is one strip).  Every layout
    // gives the same fields bit for bit (tests/test_parallel.cpp:215-238), so
    // only the worker count carries over; res.timing has one entry per strip.
    const long long workers = (long long)px * py;
    const int strips = sc.grid.dim == 1 ? 1 : (int)std::min<long long>(workers, sc.grid.ny);
    return detail::run(sc, strips, opt);
}

}  // namespace gpu
}  // namespace silt
