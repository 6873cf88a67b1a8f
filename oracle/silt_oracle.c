/*
 * oracle/silt_oracle.c — TEST INFRASTRUCTURE ONLY (the parity checker).
 *
 * A plain-C11 restatement of the reference's time-stepping path for the
 * coupled shallow-water + Exner relaxation scheme of arXiv 1307.0491 (Grass
 * and Shields-threshold bedload closures).
 * Every function follows the reference operation by operation (same operand
 * order, no FMA contraction: built with -ffp-contract=off) so that it agrees
 * bit for bit with the reference compiled with its Release flags; the tests
 * pin that against oracle/_ref (the reference itself) and tests/golden/.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg may
 * load this library.  The product (paper_1307_0491_b200) never does.
 *
 * Citations are paths under the reference checkout, proj/core/.
 */
#include <float.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "silt_cuda.h"

static char g_err[512];
const char* orc_last_error(void) { return g_err; }

static int set_err(int code, const char* msg) {
    snprintf(g_err, sizeof g_err, "%s", msg);
    return code;
}

static double dmax(double a, double b) { return (a < b) ? b : a; } /* std::max */
static double dmin(double a, double b) { return (b < a) ? b : a; } /* std::min */

/* ---- state layout (include/silt/grid.hpp:44-49) ------------------------- */
typedef struct { double h, hu, hv, zb; } cell_t;
typedef struct { double h, u, v, zb; } prim_t;
/* RelaxState (include/silt/relax_state.hpp:14-22) */
typedef struct { double h, hu, pi, z, omega; } relax_t;

/* primitives: src/grid.cpp:47-59 */
static prim_t primitives(cell_t s, double h_dry) {
    prim_t p;
    p.h = s.h;
    p.zb = s.zb;
    if (s.h > h_dry) {
        p.u = s.hu / s.h;
        p.v = s.hv / s.h;
    } else {
        p.u = 0;
        p.v = 0;
    }
    return p;
}

/* RelaxState::u (include/silt/relax_state.hpp:20) */
static double relax_u(const relax_t* s, double h_dry) { return s->h > h_dry ? s->hu / s->h : 0.0; }

/* ---- bedload closures: src/bedload.cpp ---------------------------------- */
#define K_UEPS 1e-10 /* src/bedload.cpp:11 */

/* BedloadLaw (include/silt/bedload.hpp:32-52) + Physics::gravity */
typedef struct {
    double gravity, h_dry;
    int kind;                  /* 0 Grass, 1 Shields */
    double a_g, m_g;           /* Grass */
    int formula, friction;     /* Shields: ShieldsFormula, FrictionModel (0 DW, 1 Manning) */
    double tau_cr, d_s, rel_density, fcoef;
} phys_t;

/* abs_pow: src/bedload.cpp:14-20 */
static double abs_pow(double au, double p) {
    if (p == 0.0) return 1.0;
    if (p == 1.0) return au;
    if (p == 2.0) return au * au;
    if (p == 3.0) return au * au * au;
    return pow(au, p);
}

/* positive_part: src/bedload.cpp:22 */
static double positive_part(double x) { return x > 0 ? x : 0.0; }

/* grass_flux: src/bedload.cpp:78-80 */
static double grass_flux(double u, double a_g, double m_g) {
    return a_g * u * abs_pow(fabs(u), m_g - 1.0);
}

/* friction_slope: src/bedload.cpp:82-92 */
static double friction_slope(const phys_t* P, double u, double h) {
    if (!(h > 0)) return 0.0;
    const double drag = u * fabs(u);
    if (P->friction == 0) return P->fcoef * drag / (8.0 * P->gravity * h);
    return P->fcoef * P->fcoef * drag / pow(h, 4.0 / 3.0);
}

/* shields_flux: src/bedload.cpp:94-116 */
static double shields_flux(int formula, double tau, double tau_cr) {
    double e;
    switch (formula) {
        case 0: e = positive_part(tau - tau_cr); return 8.0 * e * sqrt(e);
        case 1: e = positive_part(tau - tau_cr); return 5.7 * e * sqrt(e);
        case 2:
            if (tau <= 0) return 0.0;
            return 12.0 * sqrt(tau) * positive_part(tau - tau_cr);
        case 3: return 11.0 * pow(positive_part(tau - tau_cr), 1.65);
        case 4:
            if (tau <= 0) return 0.0;
            return 12.0 * tau * sqrt(tau) * exp(-4.5 * tau_cr / tau);
    }
    return 0.0;
}

/* shields_flux_derivative: src/bedload.cpp:118-147 */
static double shields_flux_derivative(int formula, double tau, double tau_cr) {
    double rt;
    switch (formula) {
        case 0:
            if (tau < tau_cr) return 0.0;
            return 12.0 * sqrt(tau - tau_cr);
        case 1:
            if (tau < tau_cr) return 0.0;
            return 8.55 * sqrt(tau - tau_cr);
        case 2:
            if (tau <= 0 || tau < tau_cr) return 0.0;
            rt = sqrt(tau);
            return 6.0 * (tau - tau_cr) / rt + 12.0 * rt;
        case 3:
            if (tau < tau_cr) return 0.0;
            return 11.0 * 1.65 * pow(positive_part(tau - tau_cr), 0.65);
        case 4:
            if (tau <= 0) return 0.0;
            rt = sqrt(tau);
            return 12.0 * exp(-4.5 * tau_cr / tau) * (1.5 * rt + 4.5 * tau_cr / rt);
    }
    return 0.0;
}

/* shields_stress: src/bedload.cpp:149-153 */
static double shields_stress(const phys_t* P, double h, double u) {
    if (!(h > 0)) return 0.0;
    const double sf = friction_slope(P, fabs(u), h);
    return h * sf / ((P->rel_density - 1.0) * P->d_s);
}

/* dimensional_flux: src/bedload.cpp:155-163 */
static double dimensional_flux(const phys_t* P, double h, double u) {
    if (P->kind == 0) return grass_flux(u, P->a_g, P->m_g);
    if (!(h > 0) || fabs(u) <= K_UEPS) return 0.0;
    const double tau = shields_stress(P, h, u);
    const double qstar = shields_flux(P->formula, tau, P->tau_cr);
    const double d = P->d_s;
    const double scale = sqrt((P->rel_density - 1.0) * P->gravity * d * d * d);
    return copysign(qstar * scale, u);
}

/* flux_derivatives(...).dqs_du: src/bedload.cpp:165-200 */
static double dqs_du(const phys_t* P, double h, double hu) {
    if (!(h > 0)) return 0.0;
    const double u = hu / h;
    if (P->kind == 0) return P->a_g * P->m_g * abs_pow(fabs(u), P->m_g - 1.0);
    if (fabs(u) <= K_UEPS) return 0.0;
    const double tau = shields_stress(P, h, u);
    const double dqstar = shields_flux_derivative(P->formula, tau, P->tau_cr);
    if (dqstar == 0.0) return 0.0;
    const double ds = P->d_s;
    const double scale = sqrt((P->rel_density - 1.0) * P->gravity * ds * ds * ds);
    const double dtau_du = 2.0 * tau / u;
    const double sgn = (u > 0) ? 1.0 : -1.0;
    return sgn * scale * dqstar * dtau_du;
}

/* normal_flux: src/bedload.cpp:207-213 */
static double normal_flux(const phys_t* P, double h, double un, double ut) {
    const double speed = hypot(un, ut);
    if (speed <= K_UEPS) return 0.0;
    return dimensional_flux(P, h, speed) * (un / speed);
}

/* normal_flux_derivative: src/bedload.cpp:215-223 */
static double normal_flux_derivative(const phys_t* P, double h, double un, double ut) {
    const double speed = hypot(un, ut);
    if (speed <= K_UEPS) return 0.0;
    const double rate = dimensional_flux(P, h, speed);
    const double drate = dqs_du(P, h, h * speed);
    const double ratio = un / speed;
    return rate / speed + ratio * ratio * (drate - rate / speed);
}

/* ---- relaxation state + celerities: src/relax_state.cpp ----------------- */
/* equilibrate: src/relax_state.cpp:8-21 */
static relax_t equilibrate(cell_t cell, const phys_t* P, int axis) {
    const prim_t p = primitives(cell, P->h_dry);
    const double un = axis == 0 ? p.u : p.v;
    const double ut = axis == 0 ? p.v : p.u;
    relax_t s;
    s.h = cell.h;
    s.hu = cell.h * un;
    s.pi = 0.5 * P->gravity * cell.h * cell.h;
    s.z = cell.zb;
    s.omega = normal_flux(P, cell.h, un, ut);
    return s;
}

/* bounds_impl: src/relax_state.cpp:25-53 */
static void celerity_bounds(const relax_t* l, const relax_t* r, double ut_l, double ut_r,
                            const phys_t* P, double safety, double* a_out, double* b_out) {
    const int wet_l = l->h > P->h_dry;
    const int wet_r = r->h > P->h_dry;
    *a_out = 0;
    *b_out = 0;
    if (!wet_l && !wet_r) return;
    const double g = P->gravity;
    double a = 0, b2 = 0;
    int still = 1;
    const relax_t* sides[2] = {l, r};
    for (int k = 0; k < 2; ++k) {
        const relax_t* s = sides[k];
        if (!(s->h > P->h_dry)) continue;
        const double un = relax_u(s, P->h_dry);
        const double ut = k == 0 ? ut_l : ut_r;
        a = dmax(a, s->h * sqrt(g * s->h));
        const double dq = normal_flux_derivative(P, s->h, un, ut);
        b2 = dmax(b2, s->hu * s->hu + g * s->h * s->h * dq);
        const double speed = hypot(un, ut);
        if (dimensional_flux(P, s->h, speed) != 0.0 || dq != 0.0 || s->omega != 0.0) still = 0;
    }
    *a_out = safety * a;
    *b_out = still ? 0.0 : safety * sqrt(b2);
}

/* ---- interface Riemann solver: src/riemann.cpp --------------------------- */
#define K_SUPPRESS_B 1e-12 /* src/riemann.cpp:42 */
#define K_GAP 1.1          /* :43 */
#define K_MAX_ENLARGE 25   /* :44 */
#define K_MAX_NEWTON 60    /* :45 */

typedef struct {
    relax_t region[6];
    double speed[5];
    double exchange[5];
} fan_t;

/* tau_of: src/riemann.cpp:50-52 */
static double tau_of(const relax_t* s) { return 1.0 / dmax(s->h, 1e-12); }

/* make_state: src/riemann.cpp:60-68 */
static relax_t make_state(double tau, double u, double pi, double z, double omega) {
    relax_t s;
    s.h = 1.0 / tau;
    s.hu = u / tau;
    s.pi = pi;
    s.z = z;
    s.omega = omega;
    return s;
}

/* solve_suppressed: src/riemann.cpp:72-94. Returns 0 when ill-posed. */
static int solve_suppressed(const relax_t* l, const relax_t* r, double a, double g, fan_t* f) {
    const double tl = tau_of(l), tr = tau_of(r);
    const double ul = relax_u(l, 0.0), ur = relax_u(r, 0.0);
    const double ustar = 0.5 * (ul + ur) + (l->pi - r->pi) / (2.0 * a);
    const double pstar = 0.5 * (l->pi + r->pi) + 0.5 * a * (ul - ur);
    const double tsl = tl + (ustar - ul) / a;
    const double tsr = tr + (ur - ustar) / a;
    if (!(tsl > 0) || !(tsr > 0)) return 0;
    memset(f, 0, sizeof *f);
    f->region[0] = *l;
    f->region[1] = make_state(tsl, ustar, pstar, l->z, l->omega);
    f->region[2] = f->region[1];
    f->region[3] = make_state(tsr, ustar, pstar, r->z, r->omega);
    f->region[4] = f->region[3];
    f->region[5] = *r;
    f->speed[0] = ul - a * tl;
    f->speed[1] = ustar;
    f->speed[2] = ustar;
    f->speed[3] = ustar;
    f->speed[4] = ur + a * tr;
    f->exchange[2] = g * 0.5 * (l->h + r->h) * (r->z - l->z);
    return 1;
}

/* solve_solid_outer: src/riemann.cpp:97-146 */
static int solve_solid_outer(const relax_t* l, const relax_t* r, double a, double b, double g,
                             fan_t* f) {
    const double tl = tau_of(l), tr = tau_of(r);
    const double ul = relax_u(l, 0.0), ur = relax_u(r, 0.0);
    const double k = g / (a * a - b * b);
    const double kl_side = l->pi + a * a * tl;
    const double kr_side = r->pi + a * a * tr;
    const double m2 = ul - b * tl;
    const double m4 = ur + b * tr;
    const double d = m4 - m2;
    if (!(d > 0)) return 0;
    const double jz = r->z - l->z;
    const double jw = r->omega - l->omega;
    const double dzl = (m4 * jz - jw) / d;
    const double dzr = (m2 * jz - jw) / d;
    const double zstar = l->z + dzl;
    const double wstar = l->omega + m2 * dzl;
    const double rad1 = tl * tl + 2.0 * k * dzl;
    const double rad4 = tr * tr + 2.0 * k * dzr;
    if (!(rad1 > 0) || !(rad4 > 0)) return 0;
    const double t1 = sqrt(rad1);
    const double t4 = sqrt(rad4);
    const double u1 = m2 + b * t1;
    const double u4 = m4 - b * t4;
    const double p1 = kl_side - a * a * t1;
    const double p4 = kr_side - a * a * t4;
    const double ustar = 0.5 * (u1 + u4) + (p1 - p4) / (2.0 * a);
    const double pstar = 0.5 * (p1 + p4) + 0.5 * a * (u1 - u4);
    const double t2 = t1 + (ustar - u1) / a;
    const double t3 = t4 + (u4 - ustar) / a;
    if (!(t2 > 0) || !(t3 > 0)) return 0;
    memset(f, 0, sizeof *f);
    f->region[0] = *l;
    f->region[1] = make_state(t1, u1, p1, zstar, wstar);
    f->region[2] = make_state(t2, ustar, pstar, zstar, wstar);
    f->region[3] = make_state(t3, ustar, pstar, zstar, wstar);
    f->region[4] = make_state(t4, u4, p4, zstar, wstar);
    f->region[5] = *r;
    f->speed[0] = m2;
    f->speed[1] = u1 - a * t1;
    f->speed[2] = ustar;
    f->speed[3] = u4 + a * t4;
    f->speed[4] = m4;
    f->exchange[0] = (a * a - b * b) * (t1 - tl);
    f->exchange[4] = (a * a - b * b) * (tr - t4);
    return 1;
}

/* Eval of solve_fluid_outer: src/riemann.cpp:166-185 */
typedef struct {
    double t1, t2, t3, t4, dzl, dzr, d, r1, r2;
    int valid;
} eval_t;

typedef struct {
    double lam, rho, amb, b, kappa, jz, jw, k;
} fo_ctx;

static eval_t fo_eval(const fo_ctx* c, double m2, double m4) {
    eval_t e;
    memset(&e, 0, sizeof e);
    e.t1 = (m2 - c->lam) / c->amb;
    e.t4 = (c->rho - m4) / c->amb;
    e.t2 = (m4 - m2 - c->b * c->kappa) / (2.0 * c->b);
    e.t3 = (m4 - m2 + c->b * c->kappa) / (2.0 * c->b);
    e.d = m4 - m2;
    e.valid = e.t1 > 0 && e.t2 > 0 && e.t3 > 0 && e.t4 > 0 && e.d > 0;
    if (!e.valid) return e;
    e.dzl = (m4 * c->jz - c->jw) / e.d;
    e.dzr = (m2 * c->jz - c->jw) / e.d;
    e.r1 = (e.t1 * e.t1 - e.t2 * e.t2) + (e.t3 * e.t3 - e.t4 * e.t4) + 2.0 * c->k * c->jz;
    e.r2 = (e.t1 * e.t1 - e.t2 * e.t2) + 2.0 * c->k * e.dzl;
    return e;
}

static double res_norm(const eval_t* v) { return dmax(fabs(v->r1), fabs(v->r2)); }

/* solve_fluid_outer: src/riemann.cpp:152-262 */
static int solve_fluid_outer(const relax_t* l, const relax_t* r, double a, double b, double g,
                             fan_t* f, int* newton_its) {
    const double tl = tau_of(l), tr = tau_of(r);
    const double ul = relax_u(l, 0.0), ur = relax_u(r, 0.0);
    fo_ctx c;
    c.k = g / (a * a - b * b);
    const double kl_side = l->pi + a * a * tl;
    const double kr_side = r->pi + a * a * tr;
    c.kappa = (kr_side - kl_side) / (a * a);
    c.lam = ul - a * tl;
    c.rho = ur + a * tr;
    c.jz = r->z - l->z;
    c.jw = r->omega - l->omega;
    c.amb = a - b;
    c.b = b;

    const double u0 = 0.5 * (ul + ur) + (l->pi - r->pi) / (2.0 * a);
    double tsl = tl + (u0 - ul) / a;
    double tsr = tr + (ur - u0) / a;
    const double tfloor = 1e-6 * dmin(tl, tr);
    tsl = dmax(tsl, tfloor);
    tsr = dmax(tsr, tfloor);
    double m2 = u0 - b * tsl;
    double m4 = u0 + b * tsr;

    eval_t e = fo_eval(&c, m2, m4);
    if (!e.valid) return 0;

    /* std::max({tl, tr, t1, t2, t3, t4}) keeps the first maximal element */
    double tmax = tl;
    const double cand[5] = {tr, e.t1, e.t2, e.t3, e.t4};
    for (int q = 0; q < 5; ++q)
        if (tmax < cand[q]) tmax = cand[q];
    const double res_scale = tmax * tmax + fabs(2.0 * c.k * c.jz) + fabs(2.0 * c.k * e.dzl) +
                             fabs(2.0 * c.k * e.dzr);
    const double tol = 1e-13 * res_scale + 1e-300;

    int it = 0;
    while (res_norm(&e) > tol) {
        if (++it > K_MAX_NEWTON) return 0;
        const double j11 = 2.0 * e.t1 / c.amb - c.kappa / b;
        const double j12 = 2.0 * e.t4 / c.amb + c.kappa / b;
        const double j21 = 2.0 * e.t1 / c.amb + e.t2 / b + 2.0 * c.k * e.dzl / e.d;
        const double j22 = -e.t2 / b + 2.0 * c.k * (c.jz - e.dzl) / e.d;
        const double det = j11 * j22 - j12 * j21;
        if (det == 0.0 || !isfinite(det)) return 0;
        const double step2 = (e.r1 * j22 - e.r2 * j12) / det;
        const double step4 = (e.r2 * j11 - e.r1 * j21) / det;
        double damp = 1.0;
        int accepted = 0;
        for (int bt = 0; bt < 40; ++bt) {
            const eval_t trial = fo_eval(&c, m2 - damp * step2, m4 - damp * step4);
            if (trial.valid && (res_norm(&trial) < res_norm(&e) || res_norm(&trial) <= tol)) {
                m2 -= damp * step2;
                m4 -= damp * step4;
                e = trial;
                accepted = 1;
                break;
            }
            damp *= 0.5;
        }
        if (!accepted) return 0;
    }
    if (newton_its) *newton_its = it;

    const double ustar = 0.5 * (m2 + m4 - b * c.kappa);
    const double zstar = l->z + e.dzl;
    const double wstar = l->omega + m2 * e.dzl;
    const double u1 = c.lam + a * e.t1;
    const double u4 = c.rho - a * e.t4;
    const double p1 = kl_side - a * a * e.t1;
    const double p2 = kl_side - a * a * e.t2;
    const double p3 = kr_side - a * a * e.t3;
    const double p4 = kr_side - a * a * e.t4;
    memset(f, 0, sizeof *f);
    f->region[0] = *l;
    f->region[1] = make_state(e.t1, u1, p1, l->z, l->omega);
    f->region[2] = make_state(e.t2, ustar, p2, zstar, wstar);
    f->region[3] = make_state(e.t3, ustar, p3, zstar, wstar);
    f->region[4] = make_state(e.t4, u4, p4, r->z, r->omega);
    f->region[5] = *r;
    f->speed[0] = c.lam;
    f->speed[1] = m2;
    f->speed[2] = ustar;
    f->speed[3] = m4;
    f->speed[4] = c.rho;
    f->exchange[1] = (a * a - b * b) * (e.t2 - e.t1);
    f->exchange[3] = (a * a - b * b) * (e.t4 - e.t3);
    return 1;
}

typedef struct {
    double flux_h, flux_z, flux_hu_left, flux_hu_right;
    double a_eff, b_eff;
    int enlargements;
    int branch; /* 0 inert, 1 suppressed, 2 solid-outer, 3 fluid-outer */
    fan_t fan;
} solution_t;

/* interface_riemann: src/riemann.cpp:266-338. Returns 0 on success, 1 when no
 * positive fan exists after kMaxEnlarge enlargements (runtime_error). */
static int interface_riemann(const relax_t* left, const relax_t* right, double a0, double b0,
                             double g, solution_t* out) {
    memset(out, 0, sizeof *out);
    out->fan.region[0] = *left;
    out->fan.region[5] = *right;
    out->a_eff = a0;
    out->b_eff = b0;
    if (a0 <= 0.0) return 0;
    double a = a0, b = b0;
    for (int attempt = 0; attempt <= K_MAX_ENLARGE; ++attempt) {
        double ae = a, be = b;
        if (be >= K_SUPPRESS_B) {
            if (ae >= be)
                ae = dmax(ae, K_GAP * be);
            else
                be = dmax(be, K_GAP * ae);
        }
        fan_t f;
        int ok, branch;
        if (be < K_SUPPRESS_B) {
            ok = solve_suppressed(left, right, ae, g, &f);
            branch = 1;
        } else if (be > ae) {
            ok = solve_solid_outer(left, right, ae, be, g, &f);
            branch = 2;
        } else {
            ok = solve_fluid_outer(left, right, ae, be, g, &f, NULL);
            branch = 3;
        }
        if (ok) {
            out->fan = f;
            out->a_eff = ae;
            out->b_eff = be;
            out->enlargements = attempt;
            out->branch = branch;
            int rg = 5;
            for (int w = 0; w < 5; ++w) {
                if (f.speed[w] >= 0.0) {
                    rg = w;
                    break;
                }
            }
            const relax_t* s0 = &f.region[rg];
            out->flux_h = s0->hu;
            out->flux_z = (be < K_SUPPRESS_B) ? 0.0 : s0->omega;
            const double base = s0->hu * relax_u(s0, 0.0) + s0->pi;
            double mneg = 0, mpos = 0;
            for (int w = 0; w < 5; ++w) {
                if (f.speed[w] < 0.0)
                    mneg += f.exchange[w];
                else
                    mpos += f.exchange[w];
            }
            out->flux_hu_left = base + mneg;
            out->flux_hu_right = base - mpos;
            return 0;
        }
        a *= 2.0;
        if (b > 0) b *= 2.0;
    }
    snprintf(g_err, sizeof g_err,
             "interface_riemann: no positive fan after %d celerity enlargements (hL=%g uL=%g "
             "zL=%g | hR=%g uR=%g zR=%g)",
             K_MAX_ENLARGE, left->h, relax_u(left, 0.0), left->z, right->h, relax_u(right, 0.0),
             right->z);
    return 1;
}

/* ---- stepper: src/stepper.cpp ------------------------------------------- */
typedef struct { double h, hu_left, hu_right, hv, z; } faceflux_t; /* :61-67 */

/* solve_face: src/stepper.cpp:69-89 */
static int solve_face(cell_t lc, cell_t rc, const phys_t* P, double safety, int axis,
                      faceflux_t* F, solution_t* sol_out) {
    const relax_t l = equilibrate(lc, P, axis);
    const relax_t r = equilibrate(rc, P, axis);
    const prim_t pl = primitives(lc, P->h_dry);
    const prim_t pr = primitives(rc, P->h_dry);
    const double vt_l = axis == 0 ? pl.v : pl.u;
    const double vt_r = axis == 0 ? pr.v : pr.u;
    double a, b;
    celerity_bounds(&l, &r, vt_l, vt_r, P, safety, &a, &b);
    solution_t sol;
    if (interface_riemann(&l, &r, a, b, P->gravity, &sol)) return 1;
    F->h = sol.flux_h;
    F->hu_left = sol.flux_hu_left;
    F->hu_right = sol.flux_hu_right;
    F->z = sol.flux_z;
    F->hv = sol.flux_h * (sol.flux_h > 0 ? vt_l : sol.flux_h < 0 ? vt_r : 0.0);
    if (sol_out) *sol_out = sol;
    return 0;
}

/* check_depth: src/stepper.cpp:91-100. Returns 1 on a real violation. */
static int check_depth(double* h, double href) {
    if (*h >= 0) return 0;
    if (*h > -1e-12 * dmax(href, 1.0)) {
        *h = 0;
        return 0;
    }
    return 1;
}

static const char* kNegDepth =
    "step: negative depth produced; time step or celerities violate stability";

/* axis_speed: src/stepper.cpp:30-36 */
static double axis_speed(const phys_t* P, double h, double un, double ut) {
    const double fluid = fabs(un) + sqrt(P->gravity * h);
    const double dq = normal_flux_derivative(P, h, un, ut);
    const double solid = fabs(un) + sqrt(un * un + P->gravity * dq);
    return dmax(fluid, solid);
}

typedef struct {
    int dim, nx, ny;
    double dx, dy;
    phys_t P;
    double cfl, safety;
    silt_bc bc[4];
} grid_t;

static grid_t make_grid(const silt_problem* p) {
    grid_t g;
    g.dim = p->dim;
    g.nx = p->nx;
    g.ny = p->dim == 1 ? 1 : p->ny;
    g.dx = p->dx;
    g.dy = p->dim == 1 ? 1.0 : p->dy;
    g.P.gravity = p->gravity;
    g.P.h_dry = p->h_dry;
    g.P.kind = p->law_kind;
    g.P.a_g = p->a_g;
    g.P.m_g = p->m_g;
    g.P.formula = p->shields_formula;
    g.P.friction = p->friction_model;
    g.P.tau_cr = p->tau_cr;
    g.P.d_s = p->grain_diameter;
    g.P.rel_density = p->rel_density;
    g.P.fcoef = p->friction_coef;
    g.cfl = p->cfl;
    g.safety = p->safety;
    memcpy(g.bc, p->bc, sizeof g.bc);
    return g;
}

/* PaddedField::at (include/silt/stepper.hpp:23-28): ghost frame of one cell */
#define PAT(f, g, i, j) ((f)[(size_t)((j) + 1) * (size_t)((g)->nx + 2) + (size_t)((i) + 1)])

/* cfl_dt_impl: src/stepper.cpp:38-58, over a padded field's interior */
static int cfl_dt_padded(const grid_t* g, const cell_t* f, double* dt_out) {
    if (!(g->cfl > 0) || !(g->cfl <= 1))
        return set_err(SILT_ERR_INVALID, "cfl_dt: cfl must lie in (0, 1]");
    double dt = INFINITY;
    int any_wet = 0;
    for (int j = 0; j < g->ny; ++j) {
        for (int i = 0; i < g->nx; ++i) {
            const cell_t s = PAT(f, g, i, j);
            if (!(s.h > g->P.h_dry)) continue;
            any_wet = 1;
            const prim_t p = primitives(s, g->P.h_dry);
            dt = dmin(dt, g->dx / axis_speed(&g->P, p.h, p.u, p.v));
            if (g->dim == 2) dt = dmin(dt, g->dy / axis_speed(&g->P, p.h, p.v, p.u));
        }
    }
    if (!any_wet) return set_err(SILT_ERR_INVALID, "cfl_dt: field is entirely dry");
    *dt_out = g->cfl * dt;
    return SILT_OK;
}

/* step_1d: src/stepper.cpp:118-140 */
static int step_1d(const grid_t* g, cell_t* f, double dt) {
    const int nx = g->nx;
    const double c = dt / g->dx;
    faceflux_t* flux = (faceflux_t*)malloc(sizeof(faceflux_t) * (size_t)(nx + 1));
    int rc = SILT_OK;
    for (int k = 0; k <= nx && rc == SILT_OK; ++k)
        if (solve_face(PAT(f, g, k - 1, 0), PAT(f, g, k, 0), &g->P, g->safety, 0, &flux[k], NULL))
            rc = SILT_ERR_RUNTIME;
    if (rc == SILT_OK) {
        double hmax = 0;
        for (int i = 0; i < nx; ++i) hmax = dmax(hmax, PAT(f, g, i, 0).h);
        for (int i = 0; i < nx; ++i) {
            cell_t* s = &PAT(f, g, i, 0);
            s->h -= c * (flux[i + 1].h - flux[i].h);
            s->hu -= c * (flux[i + 1].hu_left - flux[i].hu_right);
            s->hv -= c * (flux[i + 1].hv - flux[i].hv);
            s->zb -= c * (flux[i + 1].z - flux[i].z);
            if (check_depth(&s->h, hmax)) {
                rc = set_err(SILT_ERR_RUNTIME, kNegDepth);
                break;
            }
        }
    }
    free(flux);
    return rc;
}

/* step_2d: src/stepper.cpp:142-189 */
static int step_2d(const grid_t* g, cell_t* f, double dt) {
    const int nx = g->nx, ny = g->ny;
    const double cx = dt / g->dx;
    const double cy = dt / g->dy;
    const size_t ncell = (size_t)(nx + 2) * (size_t)(ny + 2);
    cell_t* old = (cell_t*)malloc(sizeof(cell_t) * ncell);
    memcpy(old, f, sizeof(cell_t) * ncell);
    double hmax = 0;
    for (int j = 0; j < ny; ++j)
        for (int i = 0; i < nx; ++i) hmax = dmax(hmax, PAT(old, g, i, j).h);

    int rc = SILT_OK;
    faceflux_t* fx = (faceflux_t*)malloc(sizeof(faceflux_t) * (size_t)(nx + 1));
    for (int j = 0; j < ny && rc == SILT_OK; ++j) {
        for (int k = 0; k <= nx; ++k)
            if (solve_face(PAT(old, g, k - 1, j), PAT(old, g, k, j), &g->P, g->safety, 0, &fx[k],
                           NULL)) {
                rc = SILT_ERR_RUNTIME;
                break;
            }
        if (rc != SILT_OK) break;
        for (int i = 0; i < nx; ++i) {
            cell_t* s = &PAT(f, g, i, j);
            s->h -= cx * (fx[i + 1].h - fx[i].h);
            s->hu -= cx * (fx[i + 1].hu_left - fx[i].hu_right);
            s->hv -= cx * (fx[i + 1].hv - fx[i].hv);
            s->zb -= cx * (fx[i + 1].z - fx[i].z);
        }
    }
    free(fx);
    faceflux_t* fy = (faceflux_t*)malloc(sizeof(faceflux_t) * (size_t)(ny + 1));
    for (int i = 0; i < nx && rc == SILT_OK; ++i) {
        for (int k = 0; k <= ny; ++k)
            if (solve_face(PAT(old, g, i, k - 1), PAT(old, g, i, k), &g->P, g->safety, 1, &fy[k],
                           NULL)) {
                rc = SILT_ERR_RUNTIME;
                break;
            }
        if (rc != SILT_OK) break;
        for (int j = 0; j < ny; ++j) {
            cell_t* s = &PAT(f, g, i, j);
            s->h -= cy * (fy[j + 1].h - fy[j].h);
            s->hv -= cy * (fy[j + 1].hu_left - fy[j].hu_right);
            s->hu -= cy * (fy[j + 1].hv - fy[j].hv);
            s->zb -= cy * (fy[j + 1].z - fy[j].z);
            if (check_depth(&s->h, hmax)) {
                rc = set_err(SILT_ERR_RUNTIME, kNegDepth);
                break;
            }
        }
    }
    free(fy);
    free(old);
    return rc;
}

/* ---- boundary conditions: src/scenarios.cpp:43-144 ----------------------- */
/* ghost_value: src/scenarios.cpp:43-74 */
static cell_t ghost_value(cell_t interior, int side, const silt_bc* spec) {
    cell_t gv = interior;
    const int xside = side == SILT_WEST || side == SILT_EAST;
    if (spec->type == SILT_BC_INFLOW) {
        if (spec->supercritical) gv.h = spec->h0;
        if (xside) {
            gv.hu = spec->q0;
            gv.hv = 0;
        } else {
            gv.hv = spec->q0;
            gv.hu = 0;
        }
    } else if (spec->type == SILT_BC_WALL) {
        if (xside)
            gv.hu = -gv.hu;
        else
            gv.hv = -gv.hv;
    }
    return gv;
}

/* apply_bc_side: src/scenarios.cpp:78-99 */
static void apply_bc_side(const grid_t* g, cell_t* f, int side, const silt_bc* spec) {
    const int nx = g->nx, ny = g->ny;
    if (side == SILT_WEST)
        for (int j = 0; j < ny; ++j) PAT(f, g, -1, j) = ghost_value(PAT(f, g, 0, j), side, spec);
    else if (side == SILT_EAST)
        for (int j = 0; j < ny; ++j) PAT(f, g, nx, j) = ghost_value(PAT(f, g, nx - 1, j), side, spec);
    else if (side == SILT_SOUTH)
        for (int i = 0; i < nx; ++i) PAT(f, g, i, -1) = ghost_value(PAT(f, g, i, 0), side, spec);
    else
        for (int i = 0; i < nx; ++i) PAT(f, g, i, ny) = ghost_value(PAT(f, g, i, ny - 1), side, spec);
}

/* apply_bcs: src/scenarios.cpp:101-144 */
static int apply_bcs(const grid_t* g, cell_t* f) {
    const int nx = g->nx, ny = g->ny;
    const int per_x = g->bc[0].type == SILT_BC_PERIODIC;
    const int per_y = g->bc[2].type == SILT_BC_PERIODIC;
    if (per_x != (g->bc[1].type == SILT_BC_PERIODIC))
        return set_err(SILT_ERR_INVALID, "apply_bcs: periodic requires both x sides");
    if (g->dim == 2 && per_y != (g->bc[3].type == SILT_BC_PERIODIC))
        return set_err(SILT_ERR_INVALID, "apply_bcs: periodic requires both y sides");
    if (per_x) {
        for (int j = 0; j < ny; ++j) {
            PAT(f, g, -1, j) = PAT(f, g, nx - 1, j);
            PAT(f, g, nx, j) = PAT(f, g, 0, j);
        }
    } else {
        apply_bc_side(g, f, SILT_WEST, &g->bc[0]);
        apply_bc_side(g, f, SILT_EAST, &g->bc[1]);
    }
    if (g->dim == 2) {
        if (per_y) {
            for (int i = 0; i < nx; ++i) {
                PAT(f, g, i, -1) = PAT(f, g, i, ny - 1);
                PAT(f, g, i, ny) = PAT(f, g, i, 0);
            }
        } else {
            apply_bc_side(g, f, SILT_SOUTH, &g->bc[2]);
            apply_bc_side(g, f, SILT_NORTH, &g->bc[3]);
        }
        const int both = per_x && per_y;
        PAT(f, g, -1, -1) = both ? PAT(f, g, nx - 1, ny - 1) : PAT(f, g, 0, 0);
        PAT(f, g, nx, -1) = both ? PAT(f, g, 0, ny - 1) : PAT(f, g, nx - 1, 0);
        PAT(f, g, -1, ny) = both ? PAT(f, g, nx - 1, 0) : PAT(f, g, 0, ny - 1);
        PAT(f, g, nx, ny) = both ? PAT(f, g, 0, 0) : PAT(f, g, nx - 1, ny - 1);
    }
    return SILT_OK;
}

/* ---- exported API (mirrors oracle/ref_driver.cpp) ------------------------ */
static cell_t* padded_from_aos(const grid_t* g, const double* aos) {
    const size_t n = (size_t)(g->nx + 2) * (size_t)(g->ny + 2);
    cell_t* f = (cell_t*)calloc(n, sizeof(cell_t));
    for (int j = 0; j < g->ny; ++j)
        for (int i = 0; i < g->nx; ++i) {
            const double* c = aos + 4 * ((size_t)j * (size_t)g->nx + (size_t)i);
            cell_t s = {c[0], c[1], c[2], c[3]};
            PAT(f, g, i, j) = s;
        }
    return f;
}

static int cmp_double(const void* a, const void* b) {
    const double x = *(const double*)a, y = *(const double*)b;
    return (x > y) - (x < y);
}

/* BedloadLaw::grass / BedloadLaw::shields validation: src/bedload.cpp:26-57 */
static int check_law(const silt_problem* p) {
    if (p->law_kind == 0) {
        if (!(p->a_g >= 0) || !isfinite(p->a_g))
            return set_err(SILT_ERR_INVALID, "bedload: Grass a_g must be >= 0");
        if (!(p->m_g >= 1.0 && p->m_g <= 4.0))
            return set_err(SILT_ERR_INVALID, "bedload: Grass m_g must lie in [1, 4]");
        return 0;
    }
    if (p->law_kind != 1 || p->shields_formula < 0 || p->shields_formula > 4 ||
        p->friction_model < 0 || p->friction_model > 1)
        return set_err(SILT_ERR_INVALID, "bedload: unknown law");
    if (!(p->tau_cr >= 0)) return set_err(SILT_ERR_INVALID, "bedload: tau_cr must be >= 0");
    if (!(p->grain_diameter > 0))
        return set_err(SILT_ERR_INVALID, "bedload: grain diameter must be > 0");
    if (!(p->rel_density > 1))
        return set_err(SILT_ERR_INVALID, "bedload: relative density must exceed 1");
    if (!(p->friction_coef > 0))
        return set_err(SILT_ERR_INVALID, "bedload: friction coefficient must be > 0");
    return 0;
}

/* run_serial loop: src/parallel.cpp:208-259 (make_plan :101-127, next_stop :129-132) */
int orc_run(const silt_problem* p, const double* init, double t_end, int64_t max_steps,
            const double* snaps, int n_snaps, double* out, double* dt_log, int64_t dt_cap,
            int64_t* steps_out, double* t_out) {
    if (check_law(p)) return SILT_ERR_INVALID;
    if (!(t_end >= 0)) return set_err(SILT_ERR_INVALID, "run: t_end must be >= 0");
    const grid_t g = make_grid(p);
    double* plan = (double*)malloc(sizeof(double) * (size_t)(n_snaps > 0 ? n_snaps : 1));
    int np = 0;
    for (int k = 0; k < n_snaps; ++k)
        if (snaps[k] > 0 && snaps[k] <= t_end) plan[np++] = snaps[k];
    qsort(plan, (size_t)np, sizeof(double), cmp_double);
    int nu = 0;
    for (int k = 0; k < np; ++k)
        if (nu == 0 || plan[nu - 1] != plan[k]) plan[nu++] = plan[k];
    np = nu;

    cell_t* f = padded_from_aos(&g, init);
    double t = 0;
    int64_t steps = 0;
    int snap = 0;
    int rc = SILT_OK;
    while (t < t_end && (max_steps < 0 || steps < max_steps)) {
        if ((rc = apply_bcs(&g, f)) != SILT_OK) break;
        double raw;
        if ((rc = cfl_dt_padded(&g, f, &raw)) != SILT_OK) break;
        const double stop = snap < np ? dmin(plan[snap], t_end) : t_end;
        double dt, t_new;
        if (stop - t <= raw) {
            dt = stop - t;
            t_new = stop;
        } else {
            dt = raw;
            t_new = t + dt;
        }
        rc = g.dim == 1 ? step_1d(&g, f, dt) : step_2d(&g, f, dt);
        if (rc != SILT_OK) break;
        if (dt_log && steps < dt_cap) dt_log[steps] = dt;
        t = t_new;
        ++steps;
        if (snap < np && t == plan[snap]) ++snap;
    }
    if (rc == SILT_OK) {
        for (int j = 0; j < g.ny; ++j)
            for (int i = 0; i < g.nx; ++i) {
                const cell_t s = PAT(f, &g, i, j);
                double* c = out + 4 * ((size_t)j * (size_t)g.nx + (size_t)i);
                c[0] = s.h;
                c[1] = s.hu;
                c[2] = s.hv;
                c[3] = s.zb;
            }
        *steps_out = steps;
        *t_out = t;
    }
    free(f);
    free(plan);
    return rc;
}

/* cfl_dt(const Field&): src/stepper.cpp:104-108 */
int orc_cfl_dt(const silt_problem* p, const double* field, double* dt) {
    const grid_t g = make_grid(p);
    cell_t* f = padded_from_aos(&g, field);
    const int rc = cfl_dt_padded(&g, f, dt);
    free(f);
    return rc;
}

int orc_step_padded(const silt_problem* p, double* padded, double dt) {
    const grid_t g = make_grid(p);
    const int rc = g.dim == 1 ? step_1d(&g, (cell_t*)padded, dt) : step_2d(&g, (cell_t*)padded, dt);
    return rc;
}

int orc_apply_bcs(const silt_problem* p, double* padded) {
    const grid_t g = make_grid(p);
    return apply_bcs(&g, (cell_t*)padded);
}

int orc_face_batch(const silt_problem* p, const double* L, const double* R, int64_t n, int axis,
                   double* out, double* info) {
    const grid_t g = make_grid(p);
    for (int64_t k = 0; k < n; ++k) {
        const cell_t lc = {L[4 * k], L[4 * k + 1], L[4 * k + 2], L[4 * k + 3]};
        const cell_t rc = {R[4 * k], R[4 * k + 1], R[4 * k + 2], R[4 * k + 3]};
        faceflux_t F;
        solution_t sol;
        if (solve_face(lc, rc, &g.P, g.safety, axis, &F, &sol)) return SILT_ERR_RUNTIME;
        out[5 * k + 0] = F.h;
        out[5 * k + 1] = F.hu_left;
        out[5 * k + 2] = F.hu_right;
        out[5 * k + 3] = F.hv;
        out[5 * k + 4] = F.z;
        if (info) {
            info[4 * k + 0] = sol.a_eff;
            info[4 * k + 1] = sol.b_eff;
            info[4 * k + 2] = sol.enlargements;
            info[4 * k + 3] = sol.branch;
        }
    }
    return SILT_OK;
}

int orc_riemann(const double* l5, const double* r5, double a, double b, double g, double* out) {
    const relax_t l = {l5[0], l5[1], l5[2], l5[3], l5[4]};
    const relax_t r = {r5[0], r5[1], r5[2], r5[3], r5[4]};
    solution_t s;
    if (interface_riemann(&l, &r, a, b, g, &s)) return SILT_ERR_RUNTIME;
    out[0] = s.flux_h;
    out[1] = s.flux_z;
    out[2] = s.flux_hu_left;
    out[3] = s.flux_hu_right;
    out[4] = s.a_eff;
    out[5] = s.b_eff;
    out[6] = s.enlargements;
    for (int w = 0; w < 5; ++w) out[7 + w] = s.fan.speed[w];
    for (int k = 0; k < 6; ++k) {
        out[12 + 5 * k] = s.fan.region[k].h;
        out[13 + 5 * k] = s.fan.region[k].hu;
        out[14 + 5 * k] = s.fan.region[k].pi;
        out[15 + 5 * k] = s.fan.region[k].z;
        out[16 + 5 * k] = s.fan.region[k].omega;
    }
    return SILT_OK;
}

/* equilibrate + celerity_bounds for a pair: out = {l(5), r(5), a, b} */
int orc_relax(const silt_problem* p, const double* lc4, const double* rc4, int axis, double* out) {
    const grid_t g = make_grid(p);
    const cell_t lc = {lc4[0], lc4[1], lc4[2], lc4[3]};
    const cell_t rc = {rc4[0], rc4[1], rc4[2], rc4[3]};
    const relax_t l = equilibrate(lc, &g.P, axis);
    const relax_t r = equilibrate(rc, &g.P, axis);
    const prim_t pl = primitives(lc, g.P.h_dry);
    const prim_t pr = primitives(rc, g.P.h_dry);
    double a, b;
    celerity_bounds(&l, &r, axis == 0 ? pl.v : pl.u, axis == 0 ? pr.v : pr.u, &g.P, g.safety, &a,
                    &b);
    const relax_t* sides[2] = {&l, &r};
    for (int s = 0; s < 2; ++s) {
        out[5 * s + 0] = sides[s]->h;
        out[5 * s + 1] = sides[s]->hu;
        out[5 * s + 2] = sides[s]->pi;
        out[5 * s + 3] = sides[s]->z;
        out[5 * s + 4] = sides[s]->omega;
    }
    out[10] = a;
    out[11] = b;
    return SILT_OK;
}

/* Law probes, same layout as ref_law_eval (oracle/ref_driver.cpp). */
int orc_law_eval(const silt_problem* p, const double* X, int64_t n, double* out) {
    if (check_law(p)) return SILT_ERR_INVALID;
    const grid_t g = make_grid(p);
    const phys_t* P = &g.P;
    for (int64_t k = 0; k < n; ++k) {
        const double h = X[3 * k], un = X[3 * k + 1], ut = X[3 * k + 2];
        double* o = out + 6 * k;
        o[0] = dimensional_flux(P, h, un);
        o[1] = dqs_du(P, h, h * un);
        o[2] = normal_flux(P, h, un, ut);
        o[3] = normal_flux_derivative(P, h, un, ut);
        o[4] = P->kind == 1 ? shields_stress(P, h, un) : 0.0;
        o[5] = P->kind == 1 ? friction_slope(P, un, h) : 0.0;
    }
    return 0;
}

int orc_shields_flux(int formula, const double* tau, const double* tau_cr, int64_t n,
                     double* out) {
    for (int64_t k = 0; k < n; ++k) {
        out[2 * k] = shields_flux(formula, tau[k], tau_cr[k]);
        out[2 * k + 1] = shields_flux_derivative(formula, tau[k], tau_cr[k]);
    }
    return 0;
}

/* snapshot_to_string: src/snapshot.cpp:14-18 (append_num), 50-84.  *len = bytes
 * needed; min(len, cap) bytes are copied into out. */
int orc_snapshot_to_string(const silt_problem* p, const double* aos, double time, char* out,
                           int64_t cap, int64_t* len) {
    const grid_t g = make_grid(p);
    int64_t used = 0;
    char buf[64];
#define ORC_PUT(str)                                                         \
    do {                                                                     \
        const char* s_ = (str);                                              \
        const size_t n_ = strlen(s_);                                        \
        if (out && used + (int64_t)n_ <= cap) memcpy(out + used, s_, n_);    \
        used += (int64_t)n_;                                                 \
    } while (0)
#define ORC_NUM(v)                                  \
    do {                                            \
        snprintf(buf, sizeof buf, "%.17g", (v));    \
        ORC_PUT(buf);                               \
    } while (0)
    ORC_PUT(g.dim == 1 ? "x,h,u,zb,eta,time\n" : "x,y,h,u,v,zb,eta,time\n");
    for (int j = 0; j < g.ny; ++j) {
        for (int i = 0; i < g.nx; ++i) {
            const double* c = aos + 4 * ((size_t)j * g.nx + i);
            cell_t s;
            s.h = c[0];
            s.hu = c[1];
            s.hv = c[2];
            s.zb = c[3];
            const prim_t pr = primitives(s, g.P.h_dry);
            ORC_NUM((i + 0.5) * g.dx);
            ORC_PUT(",");
            if (g.dim == 2) {
                ORC_NUM((j + 0.5) * g.dy);
                ORC_PUT(",");
            }
            ORC_NUM(s.h);
            ORC_PUT(",");
            ORC_NUM(pr.u);
            ORC_PUT(",");
            if (g.dim == 2) {
                ORC_NUM(pr.v);
                ORC_PUT(",");
            }
            ORC_NUM(s.zb);
            ORC_PUT(",");
            ORC_NUM(s.h + s.zb);
            ORC_PUT(",");
            ORC_NUM(time);
            ORC_PUT("\n");
        }
    }
#undef ORC_NUM
#undef ORC_PUT
    *len = used;
    return 0;
}
