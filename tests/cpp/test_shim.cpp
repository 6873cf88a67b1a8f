// tests/cpp/test_shim.cpp — the C++ drop-in (silt::gpu, paper_1307_0491_b200/
// csrc/silt_gpu.hpp) against the reference itself, written like the
// reference's doctest suites (proj/tests/test_stepper.cpp, test_parallel.cpp).
// Linked with oracle/_ref/libsilt_ref.so (the unmodified reference core) for
// the scenario builders and the CPU run_serial it is compared with.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <functional>
#include <stdexcept>
#include <string>
#include <vector>

#include <fstream>
#include <sstream>
#include <stdlib.h>

#include "silt/io.hpp"
#include "silt/parallel.hpp"
#include "silt/scenarios.hpp"
#include "silt/stepper.hpp"
#include "silt_gpu.hpp"

using namespace silt;

static int g_fail = 0, g_pass = 0;
#define CHECK(c)                                                                      \
    do {                                                                              \
        if (c) {                                                                      \
            ++g_pass;                                                                 \
        } else {                                                                      \
            ++g_fail;                                                                 \
            std::fprintf(stderr, "%s:%d: CHECK(%s) failed\n", __FILE__, __LINE__, #c); \
        }                                                                             \
    } while (0)
template <class E, class F>
bool throws(F&& f) {
    try {
        f();
    } catch (const E&) {
        return true;
    } catch (...) {
        return false;
    }
    return false;
}

static bool same_bits(const Field& a, const Field& b) {
    if (a.cells.size() != b.cells.size()) return false;
    for (size_t k = 0; k < a.cells.size(); ++k)
        if (a.cells[k].h != b.cells[k].h || a.cells[k].hu != b.cells[k].hu ||
            a.cells[k].hv != b.cells[k].hv || a.cells[k].zb != b.cells[k].zb)
            return false;
    return true;
}

// per-field ||a-b||_inf / ||b||_inf
static double normwise(const Field& a, const Field& b) {
    double worst = 0;
    for (int f = 0; f < 4; ++f) {
        double num = 0, den = 0;
        for (size_t k = 0; k < a.cells.size(); ++k) {
            const double* x = &a.cells[k].h;
            const double* y = &b.cells[k].h;
            num = std::max(num, std::fabs(x[f] - y[f]));
            den = std::max(den, std::fabs(y[f]));
        }
        worst = std::max(worst, den > 0 ? num / den : num);
    }
    return worst;
}

static void test_cfl() {
    Field f(Grid::make_1d(10.0, 10));
    for (auto& c : f.cells) c = {1.0, 0.0, 0.0, 0.0};
    const BedloadLaw law = BedloadLaw::grass(1.0, 3.0);
    CHECK(std::fabs(gpu::cfl_dt(f, law, Physics{}, 0.5) - 0.15963771420352524) <= 1e-15);
    CHECK(gpu::cfl_dt(PaddedField::from_field(f), law, Physics{}, 0.5) ==
          gpu::cfl_dt(f, law, Physics{}, 0.5));
    CHECK(throws<std::invalid_argument>([&] { gpu::cfl_dt(f, law, Physics{}, 0.0); }));
    CHECK(throws<std::invalid_argument>([&] { gpu::cfl_dt(f, law, Physics{}, 1.5); }));
    Field dry(Grid::make_1d(1.0, 4));
    CHECK(throws<std::invalid_argument>([&] { gpu::cfl_dt(dry, law, Physics{}, 0.5); }));
}

static void test_steps_match_reference() {
    // a padded 2D field with reference BC ghosts: step_2d vs the CPU reference
    Scenario sc = build_bump_2d(40, 24, 1.0);
    PaddedField a = PaddedField::from_field(sc.initial);
    apply_bcs(a, sc.bc);
    PaddedField b = a;
    const double dt = cfl_dt(a, sc.law, sc.phys, 0.5);
    step_2d(a, sc.law, sc.phys, dt, 1.05);
    gpu::variant() = SILT_VARIANT_STRICT;
    gpu::step_2d(b, sc.law, sc.phys, dt, 1.05);
    CHECK(same_bits(a.interior(), b.interior()));
    // negative depth throws runtime_error (test_stepper.cpp:306-314)
    PaddedField n(Grid::make_1d(0.8, 8));
    for (int i = 0; i < 8; ++i) n.at(i) = {1.0, (i < 4) ? -10.0 : 10.0, 0.0, 0.0};
    n.at(-1) = n.at(0);
    n.at(8) = n.at(7);
    CHECK(throws<std::runtime_error>(
        [&] { gpu::step_1d(n, BedloadLaw::grass(0.0), Physics{}, 1.0, 1.05); }));
    // Shields laws run on the GPU path too.  Darcy-Weisbach + MPM needs only
    // IEEE arithmetic and sqrt, so STRICT reproduces the reference bit for bit.
    const BedloadLaw mpm = BedloadLaw::shields(ShieldsFormula::MeyerPeterMuller, FrictionLaw{});
    CHECK(cfl_dt(sc.initial, mpm, sc.phys, 0.5) == gpu::cfl_dt(sc.initial, mpm, sc.phys, 0.5));
    PaddedField c = PaddedField::from_field(sc.initial);
    apply_bcs(c, sc.bc);
    PaddedField d = c;
    const double dt2 = cfl_dt(c, mpm, sc.phys, 0.5);
    step_2d(c, mpm, sc.phys, dt2, 1.05);
    gpu::step_2d(d, mpm, sc.phys, dt2, 1.05);
    CHECK(same_bits(c.interior(), d.interior()));
}

static void test_runs(int variant) {
    gpu::variant() = variant;
    struct Case {
        Scenario sc;
        long steps;
    };
    std::vector<Case> cases = {{build_dune_1d(400), 300},
                               {build_antidune_1d(600), 400},
                               {build_bump_2d(48, 36, 1.0), 60},
                               {build_bump_2d(30, 30, 0.001), 40}};
    for (auto& c : cases) {
        RunOptions opt;
        opt.max_steps = c.steps;
        std::vector<double> seen_ref, seen_gpu;
        opt.snapshot_times = {0.0, 1.5, 3.0};
        opt.on_snapshot = [&](double t, const Field&) { seen_ref.push_back(t); };
        const RunResult ref = run_serial(c.sc, opt);
        opt.on_snapshot = [&](double t, const Field&) { seen_gpu.push_back(t); };
        const RunResult got = gpu::run_serial(c.sc, opt);
        CHECK(got.steps == ref.steps);
        CHECK(seen_gpu == seen_ref);
        if (variant == SILT_VARIANT_STRICT) {
            CHECK(got.time == ref.time);
            CHECK(same_bits(got.final_field, ref.final_field));
        } else {
            CHECK(std::fabs(got.time - ref.time) <= 1e-12 * ref.time);
            CHECK(normwise(got.final_field, ref.final_field) <= 1e-9);
        }
        if (c.sc.grid.dim == 2) {
            for (int py : {2, 3, 7}) {
                opt.on_snapshot = nullptr;
                const RunResult par = gpu::run_parallel(c.sc, 1, py, opt);
                CHECK(par.steps == ref.steps);
                if (variant == SILT_VARIANT_STRICT)
                    CHECK(same_bits(par.final_field, ref.final_field));
                else
                    CHECK(same_bits(par.final_field, got.final_field));
            }
        }
    }
    // partition / plan validation mirrors the reference
    const Scenario sc = build_bump_2d(8, 6, 1.0);
    CHECK(throws<std::invalid_argument>([&] { gpu::run_parallel(sc, 0, 1); }));
    CHECK(throws<std::invalid_argument>([&] { gpu::run_parallel(sc, 1, 7); }));
    RunOptions bad;
    bad.t_end = -1;
    Scenario neg = sc;
    neg.t_end = -5;
    CHECK(throws<std::invalid_argument>([&] { gpu::run_serial(neg, bad); }));
}

static std::string slurp(const std::string& path) {
    std::ifstream is(path, std::ios::binary);
    std::stringstream ss;
    ss << is.rdbuf();
    return ss.str();
}

// The CLI's simulate / bench-speedup flow (tools/src/main.cpp:100-203,
// 261-317) with silt::run_parallel swapped for silt::gpu::run_parallel and
// write_snapshot for silt::gpu::write_snapshot: snapshot files byte-identical
// to the CPU flow's (STRICT), timing.csv / speedup.csv from the reference's
// own report writers.
static void test_cli_flow() {
    char tmpl[] = "/tmp/silt_shim_XXXXXX";
    const std::string dir = mkdtemp(tmpl);
    const Scenario sc = build_bump_2d(64, 48, 1.0);
    RunOptions opt;
    opt.max_steps = 50;
    opt.snapshot_times = {0.0, 2.0, 4.0};
    int k_ref = 0, k_gpu = 0;
    opt.on_snapshot = [&](double t, const Field& f) {
        write_snapshot(f, t, dir + "/ref_" + std::to_string(k_ref++) + ".csv", sc.phys);
    };
    const RunResult ref = run_parallel(sc, 1, 2, opt);
    gpu::variant() = SILT_VARIANT_STRICT;
    opt.on_snapshot = [&](double t, const Field& f) {
        gpu::write_snapshot(f, t, dir + "/gpu_" + std::to_string(k_gpu++) + ".csv", sc.phys);
    };
    const RunResult got = gpu::run_parallel(sc, 1, 2, opt);
    CHECK(k_ref == 3 && k_gpu == 3);
    for (int k = 0; k < 3; ++k) {
        const std::string a = slurp(dir + "/ref_" + std::to_string(k) + ".csv");
        const std::string b = slurp(dir + "/gpu_" + std::to_string(k) + ".csv");
        CHECK(!a.empty() && a == b);
    }
    CHECK(snapshot_to_string(got.final_field, got.time, sc.phys) ==
          gpu::snapshot_to_string(got.final_field, got.time, sc.phys));
    gpu::write_snapshot(got.final_field, got.time, dir + "/final_gpu.csv", sc.phys);
    write_snapshot(ref.final_field, ref.time, dir + "/final_ref.csv", sc.phys);
    CHECK(slurp(dir + "/final_gpu.csv") == slurp(dir + "/final_ref.csv"));
    // timing.csv: one row per worker strip, the reference's writer
    const std::string timing = timing_to_csv(got.timing);
    CHECK(timing.rfind("rank,steps,compute_seconds,exchange_seconds\n", 0) == 0);
    CHECK(std::count(timing.begin(), timing.end(), '\n') == 3);
    CHECK(timing.find("\n1,50,") != std::string::npos);
    // bench-speedup: layouts 1x1 and 1x2 on the GPU runner
    gpu::variant() = SILT_VARIANT_FAST;
    RunOptions bo;
    bo.max_steps = 20;
    std::vector<std::pair<int, double>> timings;
    for (int py : {1, 2}) timings.emplace_back(py, gpu::run_parallel(sc, 1, py, bo).wall_seconds);
    const std::vector<SpeedupRow> rows = speedup_report(timings, 1);
    const std::string csv = speedup_to_csv(rows);
    CHECK(csv.rfind("workers,seconds,speedup,efficiency\n1,", 0) == 0);
    CHECK(rows.size() == 2 && rows[0].speedup == 1.0);
    std::remove((dir + "/final_gpu.csv").c_str());
    std::remove((dir + "/final_ref.csv").c_str());
    for (int k = 0; k < 3; ++k) {
        std::remove((dir + "/ref_" + std::to_string(k) + ".csv").c_str());
        std::remove((dir + "/gpu_" + std::to_string(k) + ".csv").c_str());
    }
    std::remove(dir.c_str());
}

int main() {
    test_cfl();
    test_cli_flow();
    test_steps_match_reference();
    test_runs(SILT_VARIANT_STRICT);
    test_runs(SILT_VARIANT_FAST);
    std::printf("test_shim: %d passed, %d failed\n", g_pass, g_fail);
    return g_fail ? 1 : 0;
}
