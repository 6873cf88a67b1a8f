// oracle/ref_driver.cpp — TEST INFRASTRUCTURE ONLY.
//
// A thin extern "C" driver over the *unmodified* reference library (silt core,
// compiled from /root/reference/proj/core/src by oracle/Makefile into
// oracle/_ref/libsilt_ref.so).  It lets the Python tests, the golden-fixture
// generator and bench.py's CPU-baseline / --impl reference arm call the
// reference through its own public API.  Nothing in the product links this.
//
// All reference calls go through the public headers (proj/core/include/silt):
//   run loop ............ mirrors run_serial (src/parallel.cpp:208-259) step by
//                         step so the dt sequence can be logged
//   run_serial/parallel . silt::run_serial / silt::run_parallel (parallel.hpp:80-86)
//   cfl_dt .............. silt::cfl_dt (stepper.hpp:38-41)
//   step_1d/step_2d ..... stepper.hpp:47-54
//   face ................ equilibrate/primitives/celerity_bounds/interface_riemann,
//                         composed exactly like solve_face (src/stepper.cpp:69-89)
#include <algorithm>
#include <array>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <limits>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "silt/io.hpp"
#include "silt/parallel.hpp"
#include "silt/relax_state.hpp"
#include "silt/riemann.hpp"
#include "silt/scenarios.hpp"
#include "silt/stepper.hpp"
#include "silt_cuda.h"

using namespace silt;

namespace {

thread_local std::string g_err;

int fail(int code, const char* what) {
    g_err = what;
    return code;
}

template <class F>
int guarded(F&& fn) {
    try {
        fn();
        return SILT_OK;
    } catch (const std::invalid_argument& e) {
        return fail(SILT_ERR_INVALID, e.what());
    } catch (const std::runtime_error& e) {
        return fail(SILT_ERR_RUNTIME, e.what());
    } catch (const std::exception& e) {
        return fail(SILT_ERR_RUNTIME, e.what());
    }
}

Grid make_grid(const silt_problem& p) {
    Grid g;
    g.dim = p.dim;
    g.nx = p.nx;
    g.ny = p.dim == 1 ? 1 : p.ny;
    g.dx = p.dx;
    g.dy = p.dim == 1 ? 1.0 : p.dy;
    g.length_x = g.nx * g.dx;
    g.length_y = p.dim == 1 ? 0.0 : g.ny * g.dy;
    return g;
}

BoundarySpec make_bc(const silt_bc& b) {
    switch (b.type) {
        case SILT_BC_INFLOW:
            return b.supercritical ? BoundarySpec::inflow_supercritical(b.q0, b.h0)
                                   : BoundarySpec::inflow_subcritical(b.q0);
        case SILT_BC_WALL: return BoundarySpec::wall();
        case SILT_BC_PERIODIC: return BoundarySpec::periodic();
        default: return BoundarySpec::outflow();
    }
}

Physics make_phys(const silt_problem& p) {
    Physics ph;
    ph.gravity = p.gravity;
    ph.h_dry = p.h_dry;
    return ph;
}

Field make_field(const Grid& g, const double* aos) {
    Field f(g);
    for (std::size_t k = 0; k < f.cells.size(); ++k)
        f.cells[k] = {aos[4 * k], aos[4 * k + 1], aos[4 * k + 2], aos[4 * k + 3]};
    return f;
}

void store_field(const Field& f, double* aos) {
    for (std::size_t k = 0; k < f.cells.size(); ++k) {
        aos[4 * k] = f.cells[k].h;
        aos[4 * k + 1] = f.cells[k].hu;
        aos[4 * k + 2] = f.cells[k].hv;
        aos[4 * k + 3] = f.cells[k].zb;
    }
}

// BedloadLaw from the ABI problem, through the reference's own factories
// (src/bedload.cpp:26-57) so their validation applies.
BedloadLaw make_law(const silt_problem& p) {
    if (p.law_kind == SILT_LAW_GRASS) return BedloadLaw::grass(p.a_g, p.m_g);
    if (p.law_kind != SILT_LAW_SHIELDS) throw std::invalid_argument("bedload: unknown law kind");
    if (p.shields_formula < 0 || p.shields_formula > 4)
        throw std::invalid_argument("bedload: unknown Shields formula");
    FrictionLaw fric;
    fric.model = p.friction_model == SILT_FRICTION_MANNING ? FrictionModel::Manning
                                                           : FrictionModel::DarcyWeisbach;
    fric.coefficient = p.friction_coef;
    return BedloadLaw::shields(static_cast<ShieldsFormula>(p.shields_formula), fric, p.tau_cr,
                               p.grain_diameter, p.rel_density);
}

Scenario make_scenario(const silt_problem& p, const double* init, double t_end) {
    Scenario sc;
    sc.name = "oracle";
    sc.grid = make_grid(p);
    sc.initial = make_field(sc.grid, init);
    sc.law = make_law(p);
    sc.phys = make_phys(p);
    for (int s = 0; s < 4; ++s) sc.bc[s] = make_bc(p.bc[s]);
    sc.t_end = t_end;
    sc.cfl = p.cfl;
    sc.safety = p.safety;
    return sc;
}

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

// run_serial's loop (src/parallel.cpp:221-250) re-expressed through the public
// API so each dt can be logged: apply_bcs -> cfl_dt -> clip -> step_*.
int ref_run(const silt_problem* p, const double* init, double t_end,
            int64_t max_steps, const double* snaps, int n_snaps, double* out,
            double* dt_log, int64_t dt_cap, int64_t* steps_out, double* t_out) {
    return guarded([&] {
        const Scenario sc = make_scenario(*p, init, t_end);
        std::vector<double> plan;
        for (int k = 0; k < n_snaps; ++k)
            if (snaps[k] > 0 && snaps[k] <= t_end) plan.push_back(snaps[k]);
        std::sort(plan.begin(), plan.end());
        plan.erase(std::unique(plan.begin(), plan.end()), plan.end());
        PaddedField f = PaddedField::from_field(sc.initial);
        double t = 0;
        int64_t steps = 0;
        std::size_t snap = 0;
        while (t < t_end && (max_steps < 0 || steps < max_steps)) {
            apply_bcs(f, sc.bc);
            const double raw = cfl_dt(f, sc.law, sc.phys, sc.cfl);
            const double stop = snap < plan.size() ? std::min(plan[snap], t_end) : t_end;
            double dt, t_new;
            if (stop - t <= raw) {
                dt = stop - t;
                t_new = stop;
            } else {
                dt = raw;
                t_new = t + dt;
            }
            if (f.grid.dim == 1)
                step_1d(f, sc.law, sc.phys, dt, sc.safety);
            else
                step_2d(f, sc.law, sc.phys, dt, sc.safety);
            if (dt_log && steps < dt_cap) dt_log[steps] = dt;
            t = t_new;
            ++steps;
            if (snap < plan.size() && t == plan[snap]) ++snap;
        }
        store_field(f.interior(), out);
        *steps_out = steps;
        *t_out = t;
    });
}

// silt::run_serial / silt::run_parallel verbatim (parallel.hpp:80-86).
int ref_run_parallel(const silt_problem* p, const double* init, double t_end,
                     int64_t max_steps, int px, int py, double* out,
                     int64_t* steps_out, double* t_out, double* compute_seconds,
                     double* wall_seconds) {
    return guarded([&] {
        const Scenario sc = make_scenario(*p, init, t_end);
        RunOptions opt;
        opt.max_steps = max_steps;
        RunResult r = (px == 0 && py == 0) ? run_serial(sc, opt)
                                           : run_parallel(sc, px, py, opt);
        if (out) store_field(r.final_field, out);
        *steps_out = r.steps;
        *t_out = r.time;
        double cmax = 0;
        for (const WorkerTiming& w : r.timing) cmax = std::max(cmax, w.compute_seconds);
        if (compute_seconds) *compute_seconds = cmax;
        if (wall_seconds) *wall_seconds = r.wall_seconds;
    });
}

// run_parallel's step loop (src/parallel.cpp:315-364) for Topology{1, py},
// re-expressed through the public API so the dt sequence can be logged:
// halo_exchange + apply_bc_side on the physical sides, cfl_dt per block,
// global_dt, step_2d per block — the blocks' phases on `threads` host
// threads.  No snapshots, t_end = inf; every BC must be non-periodic.  Used
// to generate the large-grid fixtures (tests/golden/make_golden_big.py).
int ref_run_blocks(const silt_problem* p, const double* init, int64_t max_steps, int py,
                   int threads, double* out, double* dt_log, int64_t* steps_out,
                   double* t_out) {
    return guarded([&] {
        const Scenario sc = make_scenario(*p, init, std::numeric_limits<double>::infinity());
        for (int s = 0; s < 4; ++s)
            if (sc.bc[s].type == BcType::Periodic)
                throw std::invalid_argument("ref_run_blocks: periodic sides not supported");
        Topology topo;
        topo.px = 1;
        topo.py = py;
        std::vector<Subdomain> parts = partition(sc.initial, topo);
        std::vector<double> locals(parts.size());
        auto each = [&](auto&& fn) {
            std::vector<std::thread> pool;
            const int nt = std::max(1, std::min<int>(threads, (int)parts.size()));
            for (int w = 0; w < nt; ++w)
                pool.emplace_back([&, w] {
                    for (std::size_t k = w; k < parts.size(); k += nt) fn(k);
                });
            for (auto& th : pool) th.join();
        };
        double t = 0;
        int64_t steps = 0;
        while (max_steps < 0 || steps < max_steps) {
            halo_exchange(parts, topo, false);
            each([&](std::size_t k) {
                Subdomain& sd = parts[k];
                apply_bc_side(sd.field, Side::West, sc.bc[0]);
                apply_bc_side(sd.field, Side::East, sc.bc[1]);
                if (topo.neighbor(sd.rank, 0, -1) < 0)
                    apply_bc_side(sd.field, Side::South, sc.bc[2]);
                if (topo.neighbor(sd.rank, 0, +1) < 0)
                    apply_bc_side(sd.field, Side::North, sc.bc[3]);
                locals[k] = cfl_dt(sd.field, sc.law, sc.phys, sc.cfl);
            });
            const double dt = global_dt(locals);
            each([&](std::size_t k) {
                step_2d(parts[k].field, sc.law, sc.phys, dt, sc.safety);
            });
            if (dt_log) dt_log[steps] = dt;
            t = t + dt;
            ++steps;
        }
        store_field(gather(parts, topo, sc.grid), out);
        *steps_out = steps;
        *t_out = t;
    });
}

// The reference's bundled scenarios (build_scenario, src/scenarios.cpp:289-296
// with build_bump_2d's a_g / t_end arguments when name == "bump2d"): fills
// *p (grid, law, physics, cfl, safety, BCs), *t_end and, when init != NULL,
// the AoS initial field (query the cell count with init == NULL first).
int ref_build_scenario(const char* name, int cells_x, int cells_y, double a_g, silt_problem* p,
                       double* init, int64_t* cells, double* t_end) {
    return guarded([&] {
        const std::string n(name);
        const Scenario sc = n == "bump2d" ? build_bump_2d(cells_x, cells_y, a_g)
                                          : build_scenario(n, cells_x, cells_y);
        const Grid& g = sc.grid;
        std::memset(p, 0, sizeof *p);
        p->dim = g.dim;
        p->nx = g.nx;
        p->ny = g.dim == 1 ? 1 : g.ny;
        p->dx = g.dx;
        p->dy = g.dim == 1 ? 1.0 : g.dy;
        p->gravity = sc.phys.gravity;
        p->h_dry = sc.phys.h_dry;
        if (sc.law.kind != BedloadLaw::Kind::Grass)
            throw std::invalid_argument("ref_build_scenario: Grass scenarios only");
        p->law_kind = SILT_LAW_GRASS;
        p->a_g = sc.law.a_g;
        p->m_g = sc.law.m_g;
        p->cfl = sc.cfl;
        p->safety = sc.safety;
        for (int k = 0; k < 4; ++k) {
            const BoundarySpec& b = sc.bc[k];
            p->bc[k].type = b.type == BcType::Inflow     ? SILT_BC_INFLOW
                            : b.type == BcType::Wall     ? SILT_BC_WALL
                            : b.type == BcType::Periodic ? SILT_BC_PERIODIC
                                                         : SILT_BC_OUTFLOW;
            p->bc[k].supercritical = b.supercritical ? 1 : 0;
            p->bc[k].q0 = b.q0;
            p->bc[k].h0 = b.h0;
        }
        *cells = (int64_t)sc.initial.cells.size();
        *t_end = sc.t_end;
        if (init) store_field(sc.initial, init);
    });
}

// silt::run_serial with snapshot times (parallel.hpp:59-66, 80): the field
// at every landed snapshot, in order, into snaps_out[k] (AoS, cells * 4);
// *n_landed = how many landed.
int ref_run_snaps(const silt_problem* p, const double* init, double t_end, const double* times,
                  int n_times, double* snaps_out, int* n_landed, double* t_out,
                  int64_t* steps_out) {
    return guarded([&] {
        const Scenario sc = make_scenario(*p, init, t_end);
        RunOptions opt;
        opt.snapshot_times.assign(times, times + n_times);
        const std::size_t cells = sc.initial.cells.size();
        int k = 0;
        opt.on_snapshot = [&](double, const Field& f) {
            if (k < n_times) store_field(f, snaps_out + 4 * cells * (std::size_t)k);
            ++k;
        };
        const RunResult r = run_serial(sc, opt);
        *n_landed = k;
        *t_out = r.time;
        *steps_out = r.steps;
    });
}

int ref_cfl_dt(const silt_problem* p, const double* field, double* dt) {
    return guarded([&] {
        const Field f = make_field(make_grid(*p), field);
        *dt = cfl_dt(f, make_law(*p), make_phys(*p), p->cfl);
    });
}

// Halo-complete padded field (AoS, (nx+2)*(ny+2) cells; 1D: 3 rows).
int ref_step_padded(const silt_problem* p, double* padded, double dt) {
    return guarded([&] {
        PaddedField f(make_grid(*p));
        const std::size_t n = f.cells.size();
        for (std::size_t k = 0; k < n; ++k)
            f.cells[k] = {padded[4 * k], padded[4 * k + 1], padded[4 * k + 2],
                          padded[4 * k + 3]};
        const BedloadLaw law = make_law(*p);
        if (p->dim == 1)
            step_1d(f, law, make_phys(*p), dt, p->safety);
        else
            step_2d(f, law, make_phys(*p), dt, p->safety);
        for (std::size_t k = 0; k < n; ++k) {
            padded[4 * k] = f.cells[k].h;
            padded[4 * k + 1] = f.cells[k].hu;
            padded[4 * k + 2] = f.cells[k].hv;
            padded[4 * k + 3] = f.cells[k].zb;
        }
    });
}

int ref_apply_bcs(const silt_problem* p, double* padded) {
    return guarded([&] {
        PaddedField f(make_grid(*p));
        const std::size_t n = f.cells.size();
        for (std::size_t k = 0; k < n; ++k)
            f.cells[k] = {padded[4 * k], padded[4 * k + 1], padded[4 * k + 2],
                          padded[4 * k + 3]};
        std::array<BoundarySpec, 4> bc;
        for (int s = 0; s < 4; ++s) bc[s] = make_bc(p->bc[s]);
        apply_bcs(f, bc);
        for (std::size_t k = 0; k < n; ++k) {
            padded[4 * k] = f.cells[k].h;
            padded[4 * k + 1] = f.cells[k].hu;
            padded[4 * k + 2] = f.cells[k].hv;
            padded[4 * k + 3] = f.cells[k].zb;
        }
    });
}

// solve_face composed from the public API (src/stepper.cpp:69-89).
// out[k] = {F_h, F_hu_left, F_hu_right, F_hv, F_z}; info[k] = {a_eff, b_eff,
// enlargements, branch(0 inert,1 suppressed,2 solid-outer,3 fluid-outer)}.
int ref_face_batch(const silt_problem* p, const double* L, const double* R,
                   int64_t n, int axis, double* out, double* info) {
    return guarded([&] {
        const BedloadLaw law = make_law(*p);
        const Physics phys = make_phys(*p);
        const Axis ax = axis == 0 ? Axis::X : Axis::Y;
        for (int64_t k = 0; k < n; ++k) {
            const FlowState lc{L[4 * k], L[4 * k + 1], L[4 * k + 2], L[4 * k + 3]};
            const FlowState rc{R[4 * k], R[4 * k + 1], R[4 * k + 2], R[4 * k + 3]};
            const RelaxState l = equilibrate(lc, law, phys, ax);
            const RelaxState r = equilibrate(rc, law, phys, ax);
            const Primitives pl = primitives(lc, phys.h_dry);
            const Primitives pr = primitives(rc, phys.h_dry);
            const double vt_l = ax == Axis::X ? pl.v : pl.u;
            const double vt_r = ax == Axis::X ? pr.v : pr.u;
            const CelerityPair cel = celerity_bounds(l, r, vt_l, vt_r, law, phys, p->safety);
            const InterfaceSolution s = interface_riemann(l, r, cel, phys.gravity);
            out[5 * k + 0] = s.flux_h;
            out[5 * k + 1] = s.flux_hu_left;
            out[5 * k + 2] = s.flux_hu_right;
            out[5 * k + 3] = s.flux_h * (s.flux_h > 0 ? vt_l : s.flux_h < 0 ? vt_r : 0.0);
            out[5 * k + 4] = s.flux_z;
            if (info) {
                int branch = 0;
                if (cel.a > 0) {
                    if (s.celerity.b < 1e-12) branch = 1;
                    else if (s.celerity.b > s.celerity.a) branch = 2;
                    else branch = 3;
                }
                info[4 * k + 0] = s.celerity.a;
                info[4 * k + 1] = s.celerity.b;
                info[4 * k + 2] = s.enlargements;
                info[4 * k + 3] = branch;
            }
        }
    });
}

// interface_riemann on explicit relaxation states l/r = {h, hu, pi, z, omega}.
// out = {flux_h, flux_z, flux_hu_left, flux_hu_right, a_eff, b_eff,
//        enlargements, speed[5], region[6][5]} (42 doubles).
int ref_riemann(const double* l5, const double* r5, double a, double b, double g,
                double* out) {
    return guarded([&] {
        RelaxState l{l5[0], l5[1], l5[2], l5[3], l5[4]};
        RelaxState r{r5[0], r5[1], r5[2], r5[3], r5[4]};
        const InterfaceSolution s = interface_riemann(l, r, CelerityPair{a, b}, g);
        out[0] = s.flux_h;
        out[1] = s.flux_z;
        out[2] = s.flux_hu_left;
        out[3] = s.flux_hu_right;
        out[4] = s.celerity.a;
        out[5] = s.celerity.b;
        out[6] = s.enlargements;
        for (int w = 0; w < 5; ++w) out[7 + w] = s.speed[w];
        for (int k = 0; k < 6; ++k) {
            out[12 + 5 * k] = s.region[k].h;
            out[13 + 5 * k] = s.region[k].hu;
            out[14 + 5 * k] = s.region[k].pi;
            out[15 + 5 * k] = s.region[k].z;
            out[16 + 5 * k] = s.region[k].omega;
        }
    });
}

// equilibrate + celerity_bounds for a state pair (relax_state.hpp:27-51).
// out = {l(5), r(5), a, b}
int ref_relax(const silt_problem* p, const double* lc4, const double* rc4, int axis,
              double* out) {
    return guarded([&] {
        const BedloadLaw law = make_law(*p);
        const Physics phys = make_phys(*p);
        const Axis ax = axis == 0 ? Axis::X : Axis::Y;
        const FlowState lc{lc4[0], lc4[1], lc4[2], lc4[3]};
        const FlowState rc{rc4[0], rc4[1], rc4[2], rc4[3]};
        const RelaxState l = equilibrate(lc, law, phys, ax);
        const RelaxState r = equilibrate(rc, law, phys, ax);
        const Primitives pl = primitives(lc, phys.h_dry);
        const Primitives pr = primitives(rc, phys.h_dry);
        const CelerityPair c = celerity_bounds(l, r, ax == Axis::X ? pl.v : pl.u,
                                               ax == Axis::X ? pr.v : pr.u, law, phys,
                                               p->safety);
        const RelaxState* sides[2] = {&l, &r};
        for (int s = 0; s < 2; ++s) {
            out[5 * s + 0] = sides[s]->h;
            out[5 * s + 1] = sides[s]->hu;
            out[5 * s + 2] = sides[s]->pi;
            out[5 * s + 3] = sides[s]->z;
            out[5 * s + 4] = sides[s]->omega;
        }
        out[10] = c.a;
        out[11] = c.b;
    });
}

// Law probes (states[n][3] = h, u_n, u_t).  out[n][6] = {dimensional_flux(h,
// u_n), flux_derivatives(h, h u_n).dqs_du, normal_flux, normal_flux_derivative,
// shields_stress(h, u_n) (0 for Grass), friction_slope(u_n, h) (0 for Grass)}.
int ref_law_eval(const silt_problem* p, const double* X, int64_t n, double* out) {
    return guarded([&] {
        const BedloadLaw law = make_law(*p);
        const double g = p->gravity;
        const bool sh = law.kind == BedloadLaw::Kind::Shields;
        for (int64_t k = 0; k < n; ++k) {
            const double h = X[3 * k], un = X[3 * k + 1], ut = X[3 * k + 2];
            double* o = out + 6 * k;
            o[0] = dimensional_flux(law, h, un, g);
            o[1] = flux_derivatives(law, h, h * un, g).dqs_du;
            o[2] = normal_flux(law, h, un, ut, g);
            o[3] = normal_flux_derivative(law, h, un, ut, g);
            o[4] = sh ? shields_stress(law, h, un, g) : 0.0;
            o[5] = sh ? friction_slope(law.friction, un, h, g) : 0.0;
        }
    });
}

// out[n][2] = {shields_flux, shields_flux_derivative}(formula, tau[k], tau_cr[k])
int ref_shields_flux(int formula, const double* tau, const double* tau_cr, int64_t n,
                     double* out) {
    return guarded([&] {
        const ShieldsFormula f = static_cast<ShieldsFormula>(formula);
        for (int64_t k = 0; k < n; ++k) {
            out[2 * k] = shields_flux(f, tau[k], tau_cr[k]);
            out[2 * k + 1] = shields_flux_derivative(f, tau[k], tau_cr[k]);
        }
    });
}

// snapshot_to_string (src/snapshot.cpp:50-84) of an AoS field; *len = bytes
// needed; copies min(len, cap) bytes into out.
int ref_snapshot_to_string(const silt_problem* p, const double* aos, double time, char* out,
                           int64_t cap, int64_t* len) {
    return guarded([&] {
        const Grid g = make_grid(*p);
        const Field f = make_field(g, aos);
        const std::string s = snapshot_to_string(f, time, make_phys(*p));
        *len = static_cast<int64_t>(s.size());
        if (out) std::memcpy(out, s.data(), std::min<size_t>(s.size(), (size_t)cap));
    });
}

}  // extern "C"
