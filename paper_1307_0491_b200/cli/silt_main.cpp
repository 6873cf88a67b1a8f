// silt_main.cpp — the `silt` command line on the B200 time-stepping path.
//
//   silt-gpu simulate      --scenario bump2d --cells 400x400 --t-end 50 --workers 1x4 --out d ...
//   silt-gpu bench-speedup --scenario bump2d --cells 400x400 --layouts 1x1,1x2,1x4 --out s.csv
//   silt-gpu regime DEPTH VELOCITY [law flags]
//   silt-gpu flux-table [--tau-cr X] [--tau a,b,...] [--tau-max X] [--points N] [--out f]
//
// The reference's CLI (proj/tools/src/main.cpp: run_simulate :100-203,
// run_bench :261-317, run_regime :209-253, run_flux_table :321-367) with one
// change on the hot path: silt::run_parallel -> silt::gpu::run_parallel
// (paper_1307_0491_b200/csrc/silt_gpu.hpp, libsilt_b200.so) and snapshots
// formatted on the GPU (silt::gpu::write_snapshot, byte-identical CSV).  Config
// parsing/merging, scenario building, the timing / speedup / crest reports and
// the regime analysis are the reference's own library functions (silt::core),
// so the outputs keep their formats: snap_NNNN.csv, final.csv, timing.csv,
// config.txt, speedup CSV and the stdout lines.
//
// CLI11 (the reference's flag parser) is not available here; flags are parsed
// by the small parser below with the same names and value syntax.  Extra flag:
// --variant fast|strict (default fast; strict is bitwise the CPU reference).
//
// Compiled with -DSILT_CLI_REFERENCE the same source drives silt::run_parallel
// and silt::write_snapshot instead: the reference's CPU flow, used only by
// tests/test_cli.py as the expected output (tests/cpp/_build/silt-ref-cli).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <filesystem>
#include <fstream>
#include <iostream>
#include <map>
#include <optional>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "silt/io.hpp"
#include "silt/regime.hpp"
#ifndef SILT_CLI_REFERENCE
#include "silt_gpu.hpp"
#endif

namespace fs = std::filesystem;

namespace {

#ifdef SILT_CLI_REFERENCE
silt::RunResult run_strips(const silt::Scenario& sc, int px, int py, const silt::RunOptions& o) {
    return silt::run_parallel(sc, px, py, o);
}
void write_csv(const silt::Field& f, double t, const std::string& path,
                    const silt::Physics& phys) {
    silt::write_snapshot(f, t, path, phys);
}
#else
silt::RunResult run_strips(const silt::Scenario& sc, int px, int py, const silt::RunOptions& o) {
    return silt::gpu::run_parallel(sc, px, py, o);
}
void write_csv(const silt::Field& f, double t, const std::string& path,
                    const silt::Physics& phys) {
    silt::gpu::write_snapshot(f, t, path, phys);
}
#endif

std::string num(double v, const char* spec) {
    char buf[48];
    std::snprintf(buf, sizeof buf, spec, v);
    return buf;
}

// ---- flags -------------------------------------------------------------------
// argv after the subcommand: --name value pairs (or --name=value) and
// positionals.  `has` mirrors CLI11's count(): was the flag given at all.
struct Args {
    std::map<std::string, std::string> kv;
    std::vector<std::string> pos;

    Args(int argc, char** argv, int first, const std::vector<std::string>& known) {
        for (int i = first; i < argc; ++i) {
            std::string a = argv[i];
            if (a.rfind("--", 0) != 0) {
                pos.push_back(a);
                continue;
            }
            std::string name = a, value;
            const std::size_t eq = a.find('=');
            if (eq != std::string::npos) {
                name = a.substr(0, eq);
                value = a.substr(eq + 1);
            } else {
                if (i + 1 >= argc) throw std::invalid_argument(name + ": missing value");
                value = argv[++i];
            }
            if (std::find(known.begin(), known.end(), name) == known.end())
                throw std::invalid_argument("unknown option " + name);
            kv[name] = value;
        }
    }
    bool has(const std::string& k) const { return kv.count(k) != 0; }
    const std::string& str(const std::string& k) const { return kv.at(k); }
    double dbl(const std::string& k) const { return parse_double(kv.at(k), k); }
    long lng(const std::string& k) const {
        std::size_t used = 0;
        long v = 0;
        try {
            v = std::stol(kv.at(k), &used);
        } catch (const std::exception&) {
            used = 0;
        }
        if (used != kv.at(k).size()) throw std::invalid_argument(k + ": expected an integer");
        return v;
    }
    static double parse_double(const std::string& s, const std::string& what) {
        std::size_t used = 0;
        double v = 0;
        try {
            v = std::stod(s, &used);
        } catch (const std::exception&) {
            used = 0;
        }
        if (used != s.size() || s.empty()) throw std::invalid_argument(what + ": expected a number");
        return v;
    }
    std::vector<double> list(const std::string& k) const {
        std::vector<double> out;
        const std::string& s = kv.at(k);
        std::size_t p = 0;
        while (p <= s.size()) {
            std::size_t c = s.find(',', p);
            if (c == std::string::npos) c = s.size();
            out.push_back(parse_double(s.substr(p, c - p), k));
            p = c + 1;
        }
        return out;
    }
};

// "J" or "JxK" with positive integers (the reference's parse_dims, main.cpp:24-48)
std::pair<int, std::optional<int>> dims(const std::string& s, const std::string& flag) {
    auto one = [&](const std::string& tok) {
        std::size_t used = 0;
        int v = 0;
        try {
            v = std::stoi(tok, &used);
        } catch (const std::exception&) {
            used = 0;
        }
        if (used != tok.size() || v <= 0)
            throw std::invalid_argument(flag + ": expected positive integers like 200 or 200x100, got '" +
                                        s + "'");
        return v;
    };
    const std::size_t x = s.find('x');
    if (x == std::string::npos) return {one(s), std::nullopt};
    return {one(s.substr(0, x)), one(s.substr(x + 1))};
}

const std::vector<std::string> kLawFlags = {"--law", "--ag", "--mg", "--tau-cr", "--ds",
                                            "--rel-density", "--friction", "--friction-coef"};

void fill_law(const Args& a, silt::RunConfig& c) {
    if (a.has("--law")) c.law = a.str("--law");
    if (a.has("--ag")) c.a_g = a.dbl("--ag");
    if (a.has("--mg")) c.m_g = a.dbl("--mg");
    if (a.has("--tau-cr")) c.tau_cr = a.dbl("--tau-cr");
    if (a.has("--ds")) c.d_s = a.dbl("--ds");
    if (a.has("--rel-density")) c.rel_density = a.dbl("--rel-density");
    if (a.has("--friction")) c.friction = a.str("--friction");
    if (a.has("--friction-coef")) c.friction_coef = a.dbl("--friction-coef");
}

std::vector<std::string> with_law(std::vector<std::string> v) {
    v.insert(v.end(), kLawFlags.begin(), kLawFlags.end());
    v.push_back("--variant");
    return v;
}

void set_variant(const Args& a) {
    if (!a.has("--variant")) return;
    const std::string& v = a.str("--variant");
    if (v != "fast" && v != "strict") throw std::invalid_argument("--variant: fast or strict");
#ifndef SILT_CLI_REFERENCE
    silt::gpu::variant() = v == "strict" ? SILT_VARIANT_STRICT : SILT_VARIANT_FAST;
#endif
}

// ---- simulate (main.cpp:100-203) ----------------------------------------------
int simulate(int argc, char** argv) {
    const Args a(argc, argv, 2,
                 with_law({"--config", "--scenario", "--cells", "--t-end", "--cfl", "--safety",
                           "--gravity", "--workers", "--out", "--snap-every", "--snap-at",
                           "--max-steps", "--corner-exchange"}));
    set_variant(a);
    silt::RunConfig cfg;
    if (a.has("--config")) {
        if (!fs::exists(a.str("--config")))
            throw std::invalid_argument("--config: file does not exist: " + a.str("--config"));
        cfg = silt::parse_config_file(a.str("--config"));
    }
    silt::RunConfig over;
    if (a.has("--scenario")) over.scenario = a.str("--scenario");
    if (a.has("--cells")) {
        const auto d = dims(a.str("--cells"), "--cells");
        over.cells_x = d.first;
        over.cells_y = d.second;
    }
    if (a.has("--t-end")) over.t_end = a.dbl("--t-end");
    if (a.has("--cfl")) over.cfl = a.dbl("--cfl");
    if (a.has("--safety")) over.safety = a.dbl("--safety");
    if (a.has("--gravity")) over.gravity = a.dbl("--gravity");
    if (a.has("--workers")) {
        const auto d = dims(a.str("--workers"), "--workers");
        over.workers_x = d.first;
        over.workers_y = d.second.value_or(1);
    }
    if (a.has("--out")) over.out_dir = a.str("--out");
    if (a.has("--snap-every")) over.snap_every = a.dbl("--snap-every");
    if (a.has("--snap-at")) over.snap_at = a.list("--snap-at");
    if (a.has("--max-steps")) over.max_steps = a.lng("--max-steps");
    if (a.has("--corner-exchange")) {
        const std::string& v = a.str("--corner-exchange");
        if (v != "on" && v != "off") throw std::invalid_argument("--corner-exchange: on or off");
        over.corner_exchange = v == "on";
    }
    fill_law(a, over);

    cfg = silt::merge_config(cfg, over);
    const silt::Scenario sc = silt::scenario_from_config(cfg);
    const int px = cfg.workers_x.value_or(1);
    const int py = cfg.workers_y.value_or(1);
    silt::RunOptions opt;
    opt.max_steps = cfg.max_steps.value_or(-1);
    opt.exchange_corners = cfg.corner_exchange.value_or(true);

    std::vector<double> snaps = cfg.snap_at;
    if (cfg.snap_every) {
        if (!(*cfg.snap_every > 0)) throw std::invalid_argument("snap_every must be positive");
        for (long k = 0; k * *cfg.snap_every <= sc.t_end * (1.0 + 1e-12); ++k)
            snaps.push_back(k * *cfg.snap_every);
    }
    std::sort(snaps.begin(), snaps.end());
    snaps.erase(std::unique(snaps.begin(), snaps.end()), snaps.end());
    if (!snaps.empty() && !cfg.out_dir)
        throw std::invalid_argument("snapshots requested but no output directory given (--out)");
    fs::path dir;
    if (cfg.out_dir) {
        dir = *cfg.out_dir;
        fs::create_directories(dir);
    }
    int snap_idx = 0;
    opt.snapshot_times = snaps;
    if (!snaps.empty()) {
        opt.on_snapshot = [&](double t, const silt::Field& field) {
            char name[32];
            std::snprintf(name, sizeof name, "snap_%04d.csv", snap_idx++);
            write_csv(field, t, (dir / name).string(), sc.phys);
            std::cout << "snapshot t = " << num(t, "%g") << " s -> " << name << "\n";
        };
    }
    if (sc.choked_cells > 0)
        std::cout << "note: " << sc.choked_cells
                  << " cells start at critical depth (no steady supercritical profile there)\n";

    const silt::RunResult res = run_strips(sc, px, py, opt);

    if (cfg.out_dir) {
        write_csv(res.final_field, res.time, (dir / "final.csv").string(), sc.phys);
        std::ofstream(dir / "timing.csv") << silt::timing_to_csv(res.timing);
        std::ofstream(dir / "config.txt") << silt::emit_config(cfg);
    }
    const silt::CrestTrack track = silt::crest_track({{0.0, sc.initial}, {res.time, res.final_field}});
    const silt::Grid& g = sc.grid;
    std::cout << "scenario   " << sc.name << "  (";
    if (g.dim == 1)
        std::cout << g.nx << " cells, dx = " << num(g.dx, "%g") << " m";
    else
        std::cout << g.nx << "x" << g.ny << " cells, dx = " << num(g.dx, "%g")
                  << " m, dy = " << num(g.dy, "%g") << " m";
    std::cout << ")\n";
    std::cout << "law        " << sc.law.describe() << "\n";
    std::cout << "workers    " << px << "x" << py << "\n";
    std::cout << "steps      " << res.steps << "  (t = " << num(res.time, "%g") << " s)\n";
    std::cout << "wall time  " << num(res.wall_seconds, "%.3f") << " s\n";
    std::cout << "crest      x = " << num(track.x.front(), "%g") << " m -> "
              << num(track.x.back(), "%g") << " m (" << silt::to_string(track.verdict) << ")\n";
    if (cfg.out_dir) std::cout << "output     " << dir.string() << "\n";
    return 0;
}

// ---- bench-speedup (main.cpp:261-317) ------------------------------------------
int bench(int argc, char** argv) {
    const Args a(argc, argv, 2,
                 {"--scenario", "--cells", "--t-end", "--cfl", "--max-steps", "--layouts",
                  "--runs", "--ref", "--out", "--variant"});
    set_variant(a);
    const std::string layouts_s = a.has("--layouts") ? a.str("--layouts") : "1x1,2x1,2x2,4x2";
    std::vector<std::pair<int, int>> layouts;
    for (std::size_t p = 0; p <= layouts_s.size();) {
        std::size_t c = layouts_s.find(',', p);
        if (c == std::string::npos) c = layouts_s.size();
        const auto d = dims(layouts_s.substr(p, c - p), "--layouts");
        layouts.emplace_back(d.first, d.second.value_or(1));
        p = c + 1;
    }
    if (layouts.empty()) throw std::invalid_argument("--layouts: empty list");
    silt::RunConfig cfg;
    cfg.scenario = a.has("--scenario") ? a.str("--scenario") : std::string("bump2d");
    const auto cd = dims(a.has("--cells") ? a.str("--cells") : std::string("400x400"), "--cells");
    cfg.cells_x = cd.first;
    cfg.cells_y = cd.second;
    cfg.t_end = a.has("--t-end") ? a.dbl("--t-end") : 50.0;
    if (a.has("--cfl")) cfg.cfl = a.dbl("--cfl");
    const int runs = a.has("--runs") ? (int)a.lng("--runs") : 1;
    const int ref_w = a.has("--ref") ? (int)a.lng("--ref") : 0;

    std::cout << "host reports " << std::thread::hardware_concurrency() << " hardware threads\n";
    std::vector<std::pair<int, double>> timings;
    for (const auto& [px, py] : layouts) {
        const silt::Scenario sc = silt::scenario_from_config(cfg);
        silt::RunOptions opt;
        if (a.has("--max-steps")) opt.max_steps = a.lng("--max-steps");
        double best = 0;
        for (int r = 0; r < std::max(1, runs); ++r) {
            const silt::RunResult res = run_strips(sc, px, py, opt);
            if (r == 0 || res.wall_seconds < best) best = res.wall_seconds;
        }
        timings.emplace_back(px * py, best);
        std::cout << "layout " << px << "x" << py << ": " << num(best, "%.3f") << " s\n";
    }
    const int ref = ref_w > 0 ? ref_w : timings.front().first;
    const std::vector<silt::SpeedupRow> rows = silt::speedup_report(timings, ref);
    std::printf("\n%-9s %-11s %-9s %s\n", "workers", "seconds", "speedup", "efficiency");
    for (const silt::SpeedupRow& r : rows)
        std::printf("%-9d %-11.3f %-9.3f %.3f\n", r.workers, r.seconds, r.speedup, r.efficiency);
    std::fflush(stdout);
    if (a.has("--out")) {
        std::ofstream os(a.str("--out"));
        if (!os) throw std::runtime_error("cannot open '" + a.str("--out") + "' for writing");
        os << silt::speedup_to_csv(rows);
        std::cout << "\nwrote " << a.str("--out") << "\n";
    }
    return 0;
}

// ---- regime (main.cpp:209-253): diagnostics, the reference's own analysis ------
int regime(int argc, char** argv) {
    const Args a(argc, argv, 2, with_law({"--gravity"}));
    if (a.pos.size() != 2) throw std::invalid_argument("regime: expected DEPTH VELOCITY");
    const double h = Args::parse_double(a.pos[0], "depth");
    const double u = Args::parse_double(a.pos[1], "velocity");
    silt::RunConfig lc;
    fill_law(a, lc);
    const silt::BedloadLaw law =
        silt::law_from_config(lc, silt::BedloadLaw::grass(lc.a_g.value_or(1.0), lc.m_g.value_or(3.0)));
    silt::Physics phys;
    if (a.has("--gravity")) phys.gravity = a.dbl("--gravity");
    const silt::RegimeReport rep = silt::analyze_regime(h, u, law, phys);
    std::cout << "law        " << law.describe() << "\n";
    std::cout << "state      h = " << num(h, "%g") << " m, u = " << num(u, "%g") << " m/s\n";
    std::cout << "froude     " << num(rep.froude, "%.6g") << "\n";
    std::cout << "alpha      " << num(rep.derivs.alpha, "%.10g") << "\n";
    std::cout << "beta       " << num(rep.derivs.beta, "%.10g") << "\n";
    std::cout << "dqs_du     " << num(rep.derivs.dqs_du, "%.10g") << "\n";
    if (rep.cubic.real) {
        std::cout << "roots      " << num(rep.cubic.roots[0], "%.10g") << "  "
                  << num(rep.cubic.roots[1], "%.10g") << "  " << num(rep.cubic.roots[2], "%.10g")
                  << "\n";
        std::cout << "pattern    " << rep.sign_pattern << "\n";
        std::cout << "sediment   " << num(rep.sediment_root, "%.10g") << " m/s\n";
    } else {
        std::cout << "roots      " << num(rep.cubic.roots[0], "%.10g") << "  and  "
                  << num(rep.cubic.roots[1], "%.10g") << " +/- "
                  << num(std::abs(rep.cubic.roots[2]), "%.10g") << "i\n";
    }
    std::cout << "regime     " << silt::to_string(rep.regime) << "\n";
    if (rep.transcritical)
        std::cout << "note       near-critical flow (|Fr - 1| <= 0.05): classification is "
                     "unreliable here\n";
    return 0;
}

// ---- flux-table (main.cpp:321-367) -----------------------------------------------
int flux_table(int argc, char** argv) {
    const Args a(argc, argv, 2, {"--tau-cr", "--tau", "--tau-max", "--points", "--out"});
    const double tau_cr = a.has("--tau-cr") ? a.dbl("--tau-cr") : 0.047;
    std::vector<double> taus = a.has("--tau") ? a.list("--tau") : std::vector<double>{};
    if (taus.empty()) {
        const double tmax = a.has("--tau-max") ? a.dbl("--tau-max") : 0.5;
        const long pts = a.has("--points") ? a.lng("--points") : 101;
        if (pts < 2 || !(tmax > 0))
            throw std::invalid_argument("--points must be >= 2 and --tau-max positive");
        for (long k = 0; k < pts; ++k) taus.push_back(tmax * k / (pts - 1));
    }
    using silt::ShieldsFormula;
    const ShieldsFormula laws[] = {ShieldsFormula::MeyerPeterMuller,
                                   ShieldsFormula::FernandezLuqueVanBeek, ShieldsFormula::Nielsen,
                                   ShieldsFormula::Ribberink, ShieldsFormula::CamenenLarson};
    std::string out = "tau,mpm,flvb,nielsen,ribberink,camenen\n";
    for (double tau : taus) {
        out += num(tau, "%.17g");
        for (ShieldsFormula f : laws) out += "," + num(silt::shields_flux(f, tau, tau_cr), "%.17g");
        out += "\n";
    }
    if (a.has("--out")) {
        std::ofstream os(a.str("--out"));
        if (!os) throw std::runtime_error("cannot open '" + a.str("--out") + "' for writing");
        os << out;
        std::cout << "wrote " << a.str("--out") << "\n";
    } else {
        std::cout << out;
    }
    return 0;
}

}  // namespace

int main(int argc, char** argv) {
    const std::string usage =
        "usage: silt-gpu {simulate|bench-speedup|regime|flux-table} [options]\n"
        "  finite-volume shallow-water flow coupled to bedload transport, time\n"
        "  stepping on the GPU (libsilt_b200.so)\n";
    if (argc < 2 || std::string(argv[1]) == "--help" || std::string(argv[1]) == "-h") {
        std::cout << usage;
        return argc < 2 ? 2 : 0;
    }
    const std::string cmd = argv[1];
    try {
        if (cmd == "simulate") return simulate(argc, argv);
        if (cmd == "bench-speedup") return bench(argc, argv);
        if (cmd == "regime") return regime(argc, argv);
        if (cmd == "flux-table") return flux_table(argc, argv);
        std::cerr << usage;
        return 2;
    } catch (const std::exception& e) {
        std::cerr << "error: " << e.what() << "\n";
        return 1;
    }
}
