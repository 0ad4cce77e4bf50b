/*
 * oracle/odp_oracle.c -- float64 CPU ORACLE of the time-dependent Hamilton-Jacobi level-set step
 * of OptimizedDP (Bui, Giovanis, Chen, Shriraman, arXiv 2204.05520): PAPER.md §3.2, Eq. 4
 * and Algorithm 2, with the grid/ghost rule of §3.4.1, the
 * RK/CFL rule of §3.4.3 and the derivative schemes of §3.4.4.
 *
 * THIS IS TEST INFRASTRUCTURE.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load it.  It shares no source, header, table or
 * constant with the CUDA path (paper_2204_05520_b200/) and never calls it.  The product path
 * never loads this library.
 *
 * Style: plain per-node loops in the order Algorithm 2 lists them, float64 everywhere, no
 * blocking or fusion.  Where the paper is silent/garbled the SURVEY.md §8(c) reading is taken;
 * each is named below as A<n> and listed in DESIGN.md §3:
 *   A1  tau = -s >= 0, V_tau = H(x, grad V), H = ext_u ext_d p.f (goal -1: min/reach, +1: max/avoid;
 *       the disturbance takes the opposite goal).
 *   A2  L = H + sum_d alpha_d (D+ - D-)/2   (the printed "-" of Alg. 2 l.163 is anti-diffusive).
 *   A3  costate p = (D- + D+)/2.
 *   A4  minD/maxD range over both D- and D+ of the current stage input.
 *   A5  alpha_{i,d} = max over p in [minD,maxD] of |dH/dp_d| = |f_d(x,u*(p),d*(p))| (exact).
 *   A6  per-node alpha in the dissipation, alpha^max only for dt.
 *   A7  CFL factor C (0.8 LOW, 0.5 MEDIUM by default); dt = C / sum_d alpha^max_d/dx_d.
 *   A8  RK2 stage 2 reuses dt of stage 1 and recomputes its own range and alpha.
 *   A9  dt clipped to the next save time; loop while tau_k - tau > 1e-12 max(1, tau_last).
 *   A10 TVD-RK2 = Heun: V1 = V + dt L(V); V2 = V1 + dt L(V1); V = (V + V2)/2.
 *   A11 BRT: V <- min(V, target) after every full step; BRS: nothing.
 *   A12 ghost(k) = v_e + k |v_e - v_in| sgn(v_e), sgn(0) = +1, periodic axes wrap.
 *   A13 ENO2 with second differences, tie |a| <= |b| picks the left candidate.
 *   A14 bang-bang sgn(0) = +1.    A15 periodic axes exclude the upper endpoint.
 *   A19 NaN or max|V| > 1e10 is a numerical failure.   A20 all alpha^max = 0 -> dt = tau_k - tau.
 *   A30 Eq. 7 (pairwise Dubins): evader control a (|a| <= abar, the goal's extremum),
 *       pursuer b (|b| <= bbar, the opposite); alpha over the sign set of q = p_x y - p_y x - p_th
 *       (its range over the costate box, linear in p) and, for the th axis, of p_th independently.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <float.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define OR_OK 0
#define OR_EINVAL 1
#define OR_ENUMERIC 2
#define OR_ENOMEM 5

/* oracle-local dynamics identifiers (mapped from names by oracle/__init__.py) */
enum { OR_HOLO_BALL = 0, OR_HOLO_BOX = 1, OR_DUBINS3D = 2, OR_CAR4D = 3, OR_CAR5D = 4, OR_DOUBLEINT6D = 5,
       OR_PAIR_DUBINS3D = 6 };
enum { OR_LOW = 1, OR_MEDIUM = 2 };
enum { OR_BRS = 0, OR_BRT = 1 };

static double sgn1(double v) { return v >= 0.0 ? 1.0 : -1.0; } /* A14: sgn(0) = +1 */

/* ------------------------------------------------------------------------------------------
 * Grid (§3.4.1): node counts, bounds, periodic dimensions.  Row-major, axis 0 outermost,
 * highest axis innermost (§4.1).
 * ---------------------------------------------------------------------------------------- */
typedef struct {
    int n;
    int64_t N[6], stride[6], P;
    double lo[6], hi[6], dx[6];
    int per[6];
    double *x[6];
} og;

static void og_free(og *g) { for (int d = 0; d < 6; ++d) { free(g->x[d]); g->x[d] = NULL; } }

static int og_init(og *g, int n, const int64_t *N, const double *lo, const double *hi, uint32_t pmask) {
    memset(g, 0, sizeof(*g));
    if (n < 1 || n > 6) return OR_EINVAL;
    g->n = n;
    for (int d = 0; d < n; ++d) {
        if (N[d] < 3 || !(lo[d] < hi[d])) return OR_EINVAL;
        g->N[d] = N[d]; g->lo[d] = lo[d]; g->hi[d] = hi[d];
        g->per[d] = (pmask >> d) & 1u;
        /* A15: periodic axes exclude the upper endpoint */
        g->dx[d] = g->per[d] ? (hi[d] - lo[d]) / (double)N[d] : (hi[d] - lo[d]) / (double)(N[d] - 1);
    }
    g->stride[n - 1] = 1;
    for (int d = n - 2; d >= 0; --d) g->stride[d] = g->stride[d + 1] * g->N[d + 1];
    g->P = g->stride[0] * g->N[0];
    for (int d = 0; d < n; ++d) {
        g->x[d] = (double *)malloc(sizeof(double) * (size_t)g->N[d]);
        if (!g->x[d]) { og_free(g); return OR_ENOMEM; }
        for (int64_t i = 0; i < g->N[d]; ++i) g->x[d][i] = g->lo[d] + (double)i * g->dx[d];
    }
    return OR_OK;
}

/* Value of W along axis d at index j (possibly outside [0,N)), through the node whose flat index
 * with idx[d] set to 0 is `base`.  Ghost rule A12 (addGhostExtrapolate). */
static double og_at(const og *g, const double *W, int64_t base, int d, int64_t j) {
    const int64_t N = g->N[d], s = g->stride[d];
    if (j >= 0 && j < N) return W[base + j * s];
    if (g->per[d]) {
        j %= N;
        if (j < 0) j += N;
        return W[base + j * s];
    }
    if (j < 0) {
        const double e = W[base], in = W[base + s];
        return e + (double)(-j) * fabs(e - in) * sgn1(e);
    } else {
        const double e = W[base + (N - 1) * s], in = W[base + (N - 2) * s];
        return e + (double)(j - (N - 1)) * fabs(e - in) * sgn1(e);
    }
}

/* A13: ENO2 selection -- the second difference with the smaller magnitude, left on ties. */
static double eno_pick(double a, double b) { return fabs(a) <= fabs(b) ? a : b; }

/* One-sided derivatives D-, D+ along axis d at node (idx, flat) -- §3.4.4.
 * LOW: first-order upwind differences.  MEDIUM: second-order ENO. */
/* ENO2 decision ambiguity (test support, reading A28): a pick whose two candidates are within
 * float32 evaluation noise of each other in magnitude (| |a| - |b| | <= 2e-5) while differing in
 * value (|a - b| > 2e-4, i.e. opposite signs) can legitimately go either way in a float32
 * evaluation; such nodes are reported so parity tests can exempt them. */
static int eno_ambiguous(double a, double b) { return fabs(fabs(a) - fabs(b)) <= 2e-5 && fabs(a - b) > 2e-4; }

static void og_deriv(const og *g, const double *W, const int64_t *idx, int64_t flat, int d, int acc,
                     double *dm, double *dp, unsigned char *amb) {
    const int64_t i = idx[d];
    const int64_t base = flat - i * g->stride[d];
    const double h = g->dx[d];
    if (acc == OR_LOW) {
        const double vm = og_at(g, W, base, d, i - 1), v0 = W[flat], vp = og_at(g, W, base, d, i + 1);
        *dm = (v0 - vm) / h;
        *dp = (vp - v0) / h;
    } else {
        const double vm2 = og_at(g, W, base, d, i - 2), vm1 = og_at(g, W, base, d, i - 1), v0 = W[flat];
        const double vp1 = og_at(g, W, base, d, i + 1), vp2 = og_at(g, W, base, d, i + 2);
        const double dd_m = vm2 - 2.0 * vm1 + v0;  /* delta^2 at i-1 */
        const double dd_0 = vm1 - 2.0 * v0 + vp1;  /* delta^2 at i   */
        const double dd_p = v0 - 2.0 * vp1 + vp2;  /* delta^2 at i+1 */
        *dm = (v0 - vm1) / h + eno_pick(dd_m, dd_0) / (2.0 * h);
        *dp = (vp1 - v0) / h - eno_pick(dd_0, dd_p) / (2.0 * h);
        if (amb && (eno_ambiguous(dd_m, dd_0) || eno_ambiguous(dd_0, dd_p))) *amb = 1;
    }
}

/* ------------------------------------------------------------------------------------------
 * Dynamics (reading A22).  Each functor gives the optimal control and
 * disturbance for a costate (Alg. 2 l.154, "u_opt <- argmax grad.f"), the state rate
 * (l.155, "zdot <- f(z, u_opt)") and the dissipation coefficient (l.162).
 * ---------------------------------------------------------------------------------------- */
typedef struct { int id, n; double prm[8]; } ofun;

static int of_init(ofun *f, int id, int n, const double *prm, int np) {
    static const int want_np[7] = {2, 3, 3, 5, 3, 3, 5};
    static const int want_n[7] = {0, 0, 3, 4, 5, 6, 3};
    if (id < 0 || id > 6) return OR_EINVAL;
    if (np != want_np[id]) return OR_EINVAL;
    if (want_n[id] != 0 && n != want_n[id]) return OR_EINVAL;
    if (n < 1 || n > 6) return OR_EINVAL;
    f->id = id; f->n = n;
    for (int k = 0; k < np; ++k) f->prm[k] = prm[k];
    const double goal = prm[np - 1];
    if (goal != 1.0 && goal != -1.0) return OR_EINVAL;
    return OR_OK;
}

/* optimal control u* and disturbance d* for costate p (bang-bang; ball control for HOLO_BALL) */
static void of_opt(const ofun *f, const double *x, const double *p, double *u, double *dd) {
    (void)x;
    const double *c = f->prm;
    switch (f->id) {
    case OR_HOLO_BALL: { /* xdot = u, |u|_2 <= ubar; u* = goal ubar p/|p| (0 if p = 0) */
        double nrm = 0.0;
        for (int d = 0; d < f->n; ++d) nrm += p[d] * p[d];
        nrm = sqrt(nrm);
        for (int d = 0; d < f->n; ++d) u[d] = nrm > 0.0 ? c[1] * c[0] * p[d] / nrm : 0.0;
        break; }
    case OR_HOLO_BOX: /* xdot_d = u_d + d_d */
        for (int d = 0; d < f->n; ++d) { u[d] = c[2] * c[0] * sgn1(p[d]); dd[d] = -c[2] * c[1] * sgn1(p[d]); }
        break;
    case OR_DUBINS3D: /* [v, wbar, goal]; u = w */
        u[0] = c[2] * c[1] * sgn1(p[2]);
        break;
    case OR_CAR4D: /* [abar, wbar, dxbar, dybar, goal]; u = (a, w), d = (dx, dy) */
        u[0] = c[4] * c[0] * sgn1(p[2]);
        u[1] = c[4] * c[1] * sgn1(p[3]);
        dd[0] = -c[4] * c[2] * sgn1(p[0]);
        dd[1] = -c[4] * c[3] * sgn1(p[1]);
        break;
    case OR_CAR5D: /* [abar, alphabar, goal]; u = (a, alpha) */
        u[0] = c[2] * c[0] * sgn1(p[3]);
        u[1] = c[2] * c[1] * sgn1(p[4]);
        break;
    case OR_DOUBLEINT6D: /* [ubar, dbar, goal]; u_i, d_i act on v_i (axes 1, 3, 5) */
        for (int i = 0; i < 3; ++i) {
            u[i] = c[2] * c[0] * sgn1(p[2 * i + 1]);
            dd[i] = -c[2] * c[1] * sgn1(p[2 * i + 1]);
        }
        break;
    case OR_PAIR_DUBINS3D: /* Eq. 7, [va, vb, abar, bbar, goal]; u = a (evader), d = b (pursuer)
                            * p.f = p_x(-va + vb cos th) + p_y va sin th + a (p_x y - p_y x - p_th) + b p_th */
        u[0] = c[4] * c[2] * sgn1(p[0] * x[1] - p[1] * x[0] - p[2]);
        dd[0] = -c[4] * c[3] * sgn1(p[2]);
        break;
    }
}

/* state rate f(x, u, d) */
static void of_rate(const ofun *f, const double *x, const double *u, const double *dd, double *fx) {
    const double *c = f->prm;
    switch (f->id) {
    case OR_HOLO_BALL:
        for (int d = 0; d < f->n; ++d) fx[d] = u[d];
        break;
    case OR_HOLO_BOX:
        for (int d = 0; d < f->n; ++d) fx[d] = u[d] + dd[d];
        break;
    case OR_DUBINS3D:
        fx[0] = c[0] * cos(x[2]);
        fx[1] = c[0] * sin(x[2]);
        fx[2] = u[0];
        break;
    case OR_CAR4D: /* (x, y, v, theta) */
        fx[0] = x[2] * cos(x[3]) + dd[0];
        fx[1] = x[2] * sin(x[3]) + dd[1];
        fx[2] = u[0];
        fx[3] = u[1];
        break;
    case OR_CAR5D: /* (x, y, theta, v, w) */
        fx[0] = x[3] * cos(x[2]);
        fx[1] = x[3] * sin(x[2]);
        fx[2] = x[4];
        fx[3] = u[0];
        fx[4] = u[1];
        break;
    case OR_DOUBLEINT6D: /* (px, vx, py, vy, pz, vz) */
        for (int i = 0; i < 3; ++i) {
            fx[2 * i] = x[2 * i + 1];
            fx[2 * i + 1] = u[i] + dd[i];
        }
        break;
    case OR_PAIR_DUBINS3D: /* Eq. 7: relative (x, y, th) of pursuer b w.r.t. evader a */
        fx[0] = -c[0] + c[1] * cos(x[2]) + u[0] * x[1];
        fx[1] = c[0] * sin(x[2]) - u[0] * x[0];
        fx[2] = dd[0] - u[0];
        break;
    }
}

/* number of distinct signs sgn(p) takes over p in [lo, hi] (A14), written into s[] */
static int sign_set(double lo, double hi, double *s) {
    int k = 0;
    if (hi >= 0.0) s[k++] = 1.0;
    if (lo < 0.0) s[k++] = -1.0;
    return k;
}

/* alpha_{i,d} = max_{p in [minD, maxD]} |dH/dp_d| (Alg. 2 l.162; A5).  For these control-affine
 * functors dH/dp_d = f_d(x, u*(p), d*(p)); u*, d* depend on p only through the sign of the one
 * costate component they multiply, so the maximum is over that component's sign set. */
static double of_alpha(const ofun *f, const double *x, int d, const double *minD, const double *maxD) {
    const double *c = f->prm;
    double s[2];
    double best = 0.0;
    int k;
    switch (f->id) {
    case OR_HOLO_BALL: { /* |dH/dp_d| = ubar |p_d| / |p|: maximal at |p_d| = M_d, |p_e| = m_e */
        double Md = fmax(fabs(minD[d]), fabs(maxD[d]));
        if (Md == 0.0) return 0.0;
        double den = Md * Md;
        for (int e = 0; e < f->n; ++e) {
            if (e == d) continue;
            double me = (minD[e] <= 0.0 && maxD[e] >= 0.0) ? 0.0 : fmin(fabs(minD[e]), fabs(maxD[e]));
            den += me * me;
        }
        return c[0] * Md / sqrt(den); }
    case OR_HOLO_BOX:
        k = sign_set(minD[d], maxD[d], s);
        for (int j = 0; j < k; ++j) best = fmax(best, fabs(c[2] * c[0] * s[j] - c[2] * c[1] * s[j]));
        return best;
    case OR_DUBINS3D:
        if (d == 0) return fabs(c[0] * cos(x[2]));
        if (d == 1) return fabs(c[0] * sin(x[2]));
        k = sign_set(minD[2], maxD[2], s);
        for (int j = 0; j < k; ++j) best = fmax(best, fabs(c[2] * c[1] * s[j]));
        return best;
    case OR_CAR4D:
        if (d == 0 || d == 1) {
            const double drift = d == 0 ? x[2] * cos(x[3]) : x[2] * sin(x[3]);
            const double dbar = d == 0 ? c[2] : c[3];
            k = sign_set(minD[d], maxD[d], s);
            for (int j = 0; j < k; ++j) best = fmax(best, fabs(drift - c[4] * dbar * s[j]));
            return best;
        }
        k = sign_set(minD[d], maxD[d], s);
        for (int j = 0; j < k; ++j) best = fmax(best, fabs(c[4] * (d == 2 ? c[0] : c[1]) * s[j]));
        return best;
    case OR_CAR5D:
        if (d == 0) return fabs(x[3] * cos(x[2]));
        if (d == 1) return fabs(x[3] * sin(x[2]));
        if (d == 2) return fabs(x[4]);
        k = sign_set(minD[d], maxD[d], s);
        for (int j = 0; j < k; ++j) best = fmax(best, fabs(c[2] * (d == 3 ? c[0] : c[1]) * s[j]));
        return best;
    case OR_DOUBLEINT6D:
        if ((d & 1) == 0) return fabs(x[d + 1]);
        k = sign_set(minD[d], maxD[d], s);
        for (int j = 0; j < k; ++j) best = fmax(best, fabs(c[2] * c[0] * s[j] - c[2] * c[1] * s[j]));
        return best;
    case OR_PAIR_DUBINS3D: {
        /* a* = goal abar sgn(q), q = p_x y - p_y x - p_th; b* = -goal bbar sgn(p_th) (A30).  The
         * range of q over the costate box is the sum of the ranges of its three terms (it is linear
         * in p); alpha takes the maximum over the sign set of q and, for d = th, the sign set of
         * p_th independently (an outer bound of the joint sign set, exact when both sets hold both
         * signs, reading A30). */
        double qlo = 0.0, qhi = 0.0;
        const double cx = x[1], cy = -x[0];               /* q = cx p_x + cy p_y - p_th */
        qlo += fmin(cx * minD[0], cx * maxD[0]); qhi += fmax(cx * minD[0], cx * maxD[0]);
        qlo += fmin(cy * minD[1], cy * maxD[1]); qhi += fmax(cy * minD[1], cy * maxD[1]);
        qlo += -maxD[2]; qhi += -minD[2];
        double sq[2], st[2];
        const int kq = sign_set(qlo, qhi, sq), kt = sign_set(minD[2], maxD[2], st);
        for (int j = 0; j < kq; ++j) {
            const double a = c[4] * c[2] * sq[j];
            if (d == 0) best = fmax(best, fabs(-c[0] + c[1] * cos(x[2]) + a * x[1]));
            else if (d == 1) best = fmax(best, fabs(c[0] * sin(x[2]) - a * x[0]));
            else
                for (int i = 0; i < kt; ++i) best = fmax(best, fabs(-c[4] * c[3] * st[i] - a));
        }
        return best; }
    }
    return 0.0;
}

/* H_i = grad(phi)^T zdot with zdot = f(z, u_opt, d_opt)   (Alg. 2 l.154-156) */
static double of_ham(const ofun *f, const double *x, const double *p) {
    double u[6] = {0}, dd[6] = {0}, fx[6] = {0};
    of_opt(f, x, p, u, dd);
    of_rate(f, x, u, dd, fx);
    double H = 0.0;
    for (int d = 0; d < f->n; ++d) H += p[d] * fx[d];
    return H;
}

/* ------------------------------------------------------------------------------------------
 * One evaluation of the semi-discrete right-hand side L(W) (step O3 of SURVEY.md §8(c)):
 *   pass A  -- Alg. 2 l.152-159: derivative range minD/maxD over every node and both sides (A4),
 *              plus the guard quantities max|W| and any NaN (A19);
 *   pass B  -- Alg. 2 l.152-156 and l.160-165: p, u*, d*, H, alpha_i, dissipation (A2), alpha^max.
 * ---------------------------------------------------------------------------------------- */
typedef struct { double minD[6], maxD[6], amax[6], maxabs; int nan; } ostage;

static void idx_of_row(const og *g, int64_t row, int64_t *idx) {
    /* row = flat index / N[n-1]; idx[n-1] set by the caller */
    for (int d = g->n - 2; d >= 0; --d) { idx[d] = row % g->N[d]; row /= g->N[d]; }
}

static void og_stage(const og *g, const ofun *f, const double *W, int acc, const double *amax_fixed,
                     double *L, ostage *st, unsigned char *amb) {
    const int n = g->n;
    const int64_t Nl = g->N[n - 1], rows = g->P / Nl;
    for (int d = 0; d < n; ++d) { st->minD[d] = INFINITY; st->maxD[d] = -INFINITY; st->amax[d] = 0.0; }
    st->maxabs = 0.0; st->nan = 0;

    /* pass A */
#pragma omp parallel
    {
        double mn[6], mx[6], mabs = 0.0; int nan = 0;
        int64_t idx[6];
        for (int d = 0; d < n; ++d) { mn[d] = INFINITY; mx[d] = -INFINITY; }
#pragma omp for schedule(static)
        for (int64_t row = 0; row < rows; ++row) {
            idx_of_row(g, row, idx);
            for (int64_t j = 0; j < Nl; ++j) {
                idx[n - 1] = j;
                const int64_t flat = row * Nl + j;
                const double w = W[flat];
                if (isnan(w)) nan = 1;
                if (fabs(w) > mabs) mabs = fabs(w);
                for (int d = 0; d < n; ++d) {
                    double dm, dp;
                    og_deriv(g, W, idx, flat, d, acc, &dm, &dp, NULL);
                    mn[d] = fmin(mn[d], fmin(dm, dp));   /* l.157 */
                    mx[d] = fmax(mx[d], fmax(dm, dp));   /* l.158 */
                }
            }
        }
#pragma omp critical
        {
            for (int d = 0; d < n; ++d) { st->minD[d] = fmin(st->minD[d], mn[d]); st->maxD[d] = fmax(st->maxD[d], mx[d]); }
            if (mabs > st->maxabs) st->maxabs = mabs;
            st->nan |= nan;
        }
    }

    /* pass B */
#pragma omp parallel
    {
        double am[6] = {0};
        int64_t idx[6];
        double x[6] = {0}, p[6], dm[6], dp[6];
#pragma omp for schedule(static)
        for (int64_t row = 0; row < rows; ++row) {
            idx_of_row(g, row, idx);
            for (int64_t j = 0; j < Nl; ++j) {
                idx[n - 1] = j;
                const int64_t flat = row * Nl + j;
                for (int d = 0; d < n; ++d) {
                    x[d] = g->x[d][idx[d]];
                    og_deriv(g, W, idx, flat, d, acc, &dm[d], &dp[d], amb ? amb + flat : NULL);  /* l.153 */
                    p[d] = 0.5 * (dm[d] + dp[d]);                       /* A3 */
                }
                double H = of_ham(f, x, p);                             /* l.154-156 */
                for (int d = 0; d < n; ++d) {
                    const double a = of_alpha(f, x, d, st->minD, st->maxD);     /* l.162 */
                    H += a * (dp[d] - dm[d]) / 2.0;                             /* l.163, A2 */
                    if (a > am[d]) am[d] = a;                                   /* l.164 */
                }
                L[flat] = H;
            }
        }
#pragma omp critical
        {
            for (int d = 0; d < n; ++d) if (am[d] > st->amax[d]) st->amax[d] = am[d];
        }
    }
    if (amax_fixed) for (int d = 0; d < n; ++d) st->amax[d] = amax_fixed[d];
}

static int guard_bad(const ostage *st) { return st->nan || !(st->maxabs <= 1e10); }   /* A19 */

static void scan_guard(const og *g, const double *W, ostage *st) {
    st->nan = 0; st->maxabs = 0.0;
    for (int64_t i = 0; i < g->P; ++i) {
        if (isnan(W[i])) st->nan = 1;
        if (fabs(W[i]) > st->maxabs) st->maxabs = fabs(W[i]);
    }
}

static double round_f32(double v) { return (double)(float)v; }

/* O4 / Alg. 2 l.167: dt = C (sum_d |alpha^max_d| / dx_d)^-1, clipped to the time left (A9, A20) */
static double og_dt(int n, const double *amax, const double *dx, double cfl, double remaining) {
    double sum = 0.0;
    for (int d = 0; d < n; ++d) sum += fabs(amax[d]) / dx[d];
    double dt = sum > 0.0 ? cfl / sum : remaining;
    return dt > remaining ? remaining : dt;
}

/* ------------------------------------------------------------------------------------------
 * Exported entry points
 * ---------------------------------------------------------------------------------------- */
int oracle_grid_axes(int n, const int64_t *N, const double *lo, const double *hi, uint32_t pmask,
                     double *dx_out, double *coords_out) {
    og g;
    int st = og_init(&g, n, N, lo, hi, pmask);
    if (st) { og_free(&g); return st; }
    int64_t off = 0;
    for (int d = 0; d < n; ++d) {
        dx_out[d] = g.dx[d];
        for (int64_t i = 0; i < g.N[d]; ++i) coords_out[off++] = g.x[d][i];
    }
    og_free(&g);
    return OR_OK;
}

/* 1-D ghost/neighbour value of a line W[0..N) at index j (unit pins of A12) */
double oracle_line_value(const double *W, int64_t N, int periodic, int64_t j) {
    og g;
    memset(&g, 0, sizeof(g));
    g.n = 1; g.N[0] = N; g.stride[0] = 1; g.per[0] = periodic; g.P = N;
    return og_at(&g, W, 0, 0, j);
}

/* D- and D+ of every node along every axis: Dm, Dp are n x P arrays (axis-major). */
int oracle_derivs(int n, const int64_t *N, const double *lo, const double *hi, uint32_t pmask,
                  const double *W, int acc, double *Dm, double *Dp) {
    og g;
    int st = og_init(&g, n, N, lo, hi, pmask);
    if (st) { og_free(&g); return st; }
    if (acc != OR_LOW && acc != OR_MEDIUM) { og_free(&g); return OR_EINVAL; }
    int64_t idx[6];
    for (int64_t flat = 0; flat < g.P; ++flat) {
        int64_t r = flat;
        for (int d = n - 1; d >= 0; --d) { idx[d] = r % g.N[d]; r /= g.N[d]; }
        for (int d = 0; d < n; ++d) og_deriv(&g, W, idx, flat, d, acc, &Dm[d * g.P + flat], &Dp[d * g.P + flat], NULL);
    }
    og_free(&g);
    return OR_OK;
}

/* H(x, p) with the optimal control/disturbance and the state rate it produces. */
int oracle_hamiltonian(int dyn, const double *prm, int np, int n, const double *x, const double *p,
                       double *H_out, double *u_out, double *d_out, double *f_out) {
    ofun f;
    int st = of_init(&f, dyn, n, prm, np);
    if (st) return st;
    double u[6] = {0}, dd[6] = {0}, fx[6] = {0};
    of_opt(&f, x, p, u, dd);
    of_rate(&f, x, u, dd, fx);
    double H = 0.0;
    for (int d = 0; d < n; ++d) H += p[d] * fx[d];
    *H_out = H;
    if (u_out) memcpy(u_out, u, sizeof(u));
    if (d_out) memcpy(d_out, dd, sizeof(dd));
    if (f_out) memcpy(f_out, fx, sizeof(fx));
    return OR_OK;
}

/* state rate for explicit (u, d) -- used by the brute-force optimality pins */
int oracle_rate(int dyn, const double *prm, int np, int n, const double *x, const double *u,
                const double *dd, double *f_out) {
    ofun f;
    int st = of_init(&f, dyn, n, prm, np);
    if (st) return st;
    of_rate(&f, x, u, dd, f_out);
    return OR_OK;
}

int oracle_alpha(int dyn, const double *prm, int np, int n, const double *x, const double *minD,
                 const double *maxD, double *alpha_out) {
    ofun f;
    int st = of_init(&f, dyn, n, prm, np);
    if (st) return st;
    for (int d = 0; d < n; ++d) alpha_out[d] = of_alpha(&f, x, d, minD, maxD);
    return OR_OK;
}

/* One L(W) evaluation (O3) on a whole grid. range_out = [minD(n), maxD(n), amax(n), maxabs, nan] */
int oracle_stage(int n, const int64_t *N, const double *lo, const double *hi, uint32_t pmask, int dyn,
                 const double *prm, int np, const double *W, int acc, double *L, double *range_out,
                 int nthreads) {
    og g;
    ofun f;
    int st = og_init(&g, n, N, lo, hi, pmask);
    if (st) { og_free(&g); return st; }
    if ((st = of_init(&f, dyn, n, prm, np))) { og_free(&g); return st; }
    if (acc != OR_LOW && acc != OR_MEDIUM) { og_free(&g); return OR_EINVAL; }
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#endif
    ostage s;
    og_stage(&g, &f, W, acc, NULL, L, &s, NULL);
    for (int d = 0; d < n; ++d) { range_out[d] = s.minD[d]; range_out[n + d] = s.maxD[d]; range_out[2 * n + d] = s.amax[d]; }
    range_out[3 * n] = s.maxabs;
    range_out[3 * n + 1] = s.nan;
    og_free(&g);
    return OR_OK;
}

/*
 * The full solve (steps O0-O9): V <- V0; for every save time tau_k, take CFL steps clipped to
 * tau_k (A9); LOW = upwind1 + forward Euler (Alg. 2 l.169 with the A2 sign), MEDIUM = ENO2 +
 * TVD-RK2 (A10); BRT min with the target after each full step (A11); guard (A19).
 *
 *   V0, target   float32 inputs promoted exactly (A18); target NULL -> V0
 *   out          (ntau-1) x P doubles (write_initial=0) or ntau x P (write_initial=1)
 *   store_f32    1 -> round V to float32 after every stage (precision-conditioning pin Z4)
 *   amax_fixed   non-NULL -> alpha^max used for dt (windowed oracle, pin Z12)
 *   amb_out      non-NULL -> P bytes, OR over all stages of the ENO2 decision ambiguity flag
 * Returns OR_OK, OR_EINVAL, OR_ENUMERIC (tau_reached/steps valid), OR_ENOMEM.
 */
int oracle_hj_solve(int n, const int64_t *N, const double *lo, const double *hi, uint32_t pmask,
                    int dyn, const double *prm, int np, const float *V0, const float *target,
                    const double *tau, int ntau, int acc, int mode, double cfl, int write_initial,
                    int store_f32, const double *amax_fixed, double *out, double *tau_reached,
                    int64_t *steps_taken, int64_t *stages_taken, int nthreads, unsigned char *amb_out) {
    og g;
    ofun f;
    int st = og_init(&g, n, N, lo, hi, pmask);
    if (st) { og_free(&g); return st; }
    if ((st = of_init(&f, dyn, n, prm, np))) { og_free(&g); return st; }
    if ((acc != OR_LOW && acc != OR_MEDIUM) || (mode != OR_BRS && mode != OR_BRT) || ntau < 2 || tau[0] != 0.0) {
        og_free(&g); return OR_EINVAL;
    }
    for (int k = 1; k < ntau; ++k) if (!(tau[k] > tau[k - 1])) { og_free(&g); return OR_EINVAL; }
    if (cfl <= 0.0) cfl = acc == OR_LOW ? 0.8 : 0.5;   /* A7 */
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#endif
    const int64_t P = g.P;
    double *V = (double *)malloc(sizeof(double) * (size_t)P);
    double *L = (double *)malloc(sizeof(double) * (size_t)P);
    double *V1 = acc == OR_MEDIUM ? (double *)malloc(sizeof(double) * (size_t)P) : NULL;
    if (!V || !L || (acc == OR_MEDIUM && !V1)) { free(V); free(L); free(V1); og_free(&g); return OR_ENOMEM; }
    const float *T = target ? target : V0;

    /* O1 */
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < P; ++i) V[i] = (double)V0[i];
    double t = 0.0;
    int64_t steps = 0, stages = 0;
    int k_out = 0;
    if (write_initial) { memcpy(out, V, sizeof(double) * (size_t)P); k_out = 1; }
    const double eps = 1e-12 * fmax(1.0, tau[ntau - 1]);
    int status = OR_OK;
    ostage s;

    for (int k = 1; k < ntau && status == OR_OK; ++k) {
        while (tau[k] - t > eps) {                                    /* O2 */
            og_stage(&g, &f, V, acc, amax_fixed, L, &s, amb_out);   /* O3 */
            ++stages;
            if (guard_bad(&s)) { status = OR_ENUMERIC; break; }
            const double dt = og_dt(n, s.amax, g.dx, cfl, tau[k] - t);   /* O4 */
            if (acc == OR_LOW) {                                      /* O5 */
#pragma omp parallel for schedule(static)
                for (int64_t i = 0; i < P; ++i) {
                    double v = V[i] + dt * L[i];
                    if (store_f32) v = round_f32(v);
                    if (mode == OR_BRT) v = fmin(v, (double)T[i]);   /* O7 */
                    V[i] = v;
                }
            } else {                                                  /* O6 */
#pragma omp parallel for schedule(static)
                for (int64_t i = 0; i < P; ++i) {
                    double v = V[i] + dt * L[i];
                    V1[i] = store_f32 ? round_f32(v) : v;
                }
                og_stage(&g, &f, V1, acc, amax_fixed, L, &s, amb_out);  /* A8: own range, dt kept */
                ++stages;
                if (guard_bad(&s)) { status = OR_ENUMERIC; break; }
#pragma omp parallel for schedule(static)
                for (int64_t i = 0; i < P; ++i) {
                    const double V2 = V1[i] + dt * L[i];
                    double v = 0.5 * (V[i] + V2);
                    if (store_f32) v = round_f32(v);
                    if (mode == OR_BRT) v = fmin(v, (double)T[i]);   /* O7 */
                    V[i] = v;
                }
            }
            t += dt;                                                  /* O8 */
            ++steps;
        }
        if (status != OR_OK) break;
        memcpy(out + (size_t)k_out * (size_t)P, V, sizeof(double) * (size_t)P);   /* O9 */
        ++k_out;
    }
    if (status == OR_OK) {
        scan_guard(&g, V, &s);
        if (guard_bad(&s)) status = OR_ENUMERIC;
    }
    if (tau_reached) *tau_reached = t;
    if (steps_taken) *steps_taken = steps;
    if (stages_taken) *stages_taken = stages;
    free(V); free(L); free(V1);
    og_free(&g);
    return status;
}

double oracle_cfl_dt(int n, const double *amax, const double *dx, double cfl, double remaining) {
    return og_dt(n, amax, dx, cfl, remaining);
}

/* ------------------------------------------------------------------------------------------
 * Time-to-reach by Lax-Friedrichs sweeping -- Algorithm 3 with Eq. 5-6
 * and the alternating sweep orderings of §4.3.  Readings:
 *   A31 the loop runs WHILE max |phi - phi_old| > eps (the printed "<" would never enter it);
 *       l.3 "phi <- phi_old" saves the previous iterate.
 *   A32 H_TTR(z, p) = max_u min_d (-p.f) - 1 (Eq. 6, min/max swapped by the Isaacs condition of
 *       these control-affine systems) = -H_reach(z, p) - 1, H_reach the Hamiltonian of the functor
 *       with goal -1 (the control minimises p.f); p by central differences (the LF form of l.11).
 *   A33 sigma_d(z) = max over all costates of |dH/dp_d| (the functor's alpha with every costate
 *       sign possible, i.e. on the box [-1, 1]^n); in n dimensions l.10-11 read
 *       phi_new = (-H + sum_d sigma_d (phi_{+d} + phi_{-d}) / (2 dz_d)) / (sum_d sigma_d / dz_d).
 *   A34 target nodes (V0 <= 0) keep phi = 0; "not in boundary" = index 1..N-2 on every
 *       non-periodic axis; after each sweep the boundary rule of l.14-15 is applied along each
 *       non-periodic axis in order 0..n-1 to that axis' face nodes.
 *   A35 (oracle side) sweep k visits axis d < 3 descending when bit d of (k mod 8) is set, axes >= 3
 *       ascending: the 8 alternating orderings of §4.3 ("a total of 8 different iterating
 *       directions"); Gauss-Seidel, in place, as Algorithm 3 prints.
 * ---------------------------------------------------------------------------------------- */
static double ttr_update(const og *g, const ofun *fr, const double *phi, const int64_t *idx, int64_t flat,
                         const double *x) {
    double p[6] = {0}, sig[6] = {0}, mn[6], mx[6];
    for (int d = 0; d < g->n; ++d) { mn[d] = -1.0; mx[d] = 1.0; }
    double num = 0.0, den = 0.0;
    for (int d = 0; d < g->n; ++d) {
        const int64_t base = flat - idx[d] * g->stride[d];
        const double vp = og_at(g, phi, base, d, idx[d] + 1), vm = og_at(g, phi, base, d, idx[d] - 1);
        p[d] = (vp - vm) / (2.0 * g->dx[d]);
        sig[d] = of_alpha(fr, x, d, mn, mx);
        num += sig[d] * (vp + vm) / (2.0 * g->dx[d]);
        den += sig[d] / g->dx[d];
    }
    const double H = -of_ham(fr, x, p) - 1.0;                       /* A32 */
    return den > 0.0 ? (num - H) / den : phi[flat];
}

int oracle_ttr_solve(int n, const int64_t *N, const double *lo, const double *hi, uint32_t pmask, int dyn,
                     const double *prm, int np, const float *V0, double big, double eps, int64_t max_sweeps,
                     double *out, int64_t *sweeps_out, double *last_change) {
    og g;
    ofun f;
    int st = og_init(&g, n, N, lo, hi, pmask);
    if (st) { og_free(&g); return st; }
    /* the control minimises p.f (goal -1) whatever the caller's goal says (A32) */
    double prm2[8];
    for (int k = 0; k < np && k < 8; ++k) prm2[k] = prm[k];
    if (np >= 1) prm2[np - 1] = -1.0;
    if ((st = of_init(&f, dyn, n, prm2, np))) { og_free(&g); return st; }
    if (!(eps > 0.0) || max_sweeps < 1) { og_free(&g); return OR_EINVAL; }
    const int64_t P = g.P;
    double *old = (double *)malloc(sizeof(double) * (size_t)P);
    if (!old) { og_free(&g); return OR_ENOMEM; }
    for (int64_t i = 0; i < P; ++i) out[i] = V0[i] <= 0.0f ? 0.0 : big;     /* l.1 */
    int64_t sweeps = 0;
    double change = INFINITY;
    while (change > eps && sweeps < max_sweeps) {                            /* l.2, A31 */
        memcpy(old, out, sizeof(double) * (size_t)P);                        /* l.3 */
        for (int64_t k = 0; k < P; ++k) {                                    /* l.4: one ordering */
            int64_t idx[6], r = k, flat = 0;
            int skip = 0;
            for (int d = n - 1; d >= 0; --d) {
                int64_t i = r % g.N[d];
                r /= g.N[d];
                if (d < 3 && (((sweeps & 7) >> d) & 1)) i = g.N[d] - 1 - i;       /* A35 */
                idx[d] = i;
                if (!g.per[d] && (i == 0 || i == g.N[d] - 1)) skip = 1;
            }
            if (skip) continue;
            for (int d = 0; d < n; ++d) flat += idx[d] * g.stride[d];
            if (V0[flat] <= 0.0f) continue;                                   /* A34 */
            double x[6];
            for (int d = 0; d < n; ++d) x[d] = g.x[d][idx[d]];
            const double nv = ttr_update(&g, &f, out, idx, flat, x);         /* l.5-11 */
            out[flat] = fmin(nv, out[flat]);                                  /* l.12 */
        }
        for (int d = 0; d < n; ++d) {                                         /* l.14-15 */
            if (g.per[d]) continue;
            const int64_t s = g.stride[d], Nd = g.N[d];
            for (int64_t k = 0; k < P; ++k) {
                const int64_t i = (k / s) % Nd;
                if (i != 0 && i != Nd - 1) continue;
                const int64_t a = i == 0 ? k + s : k - s, b = i == 0 ? k + 2 * s : k - 2 * s;
                out[k] = fmin(fmax(2.0 * out[a] - out[b], out[b]), out[k]);
            }
        }
        change = 0.0;
        for (int64_t i = 0; i < P; ++i) change = fmax(change, fabs(out[i] - old[i]));
        ++sweeps;
    }
    free(old);
    og_free(&g);
    if (sweeps_out) *sweeps_out = sweeps;
    if (last_change) *last_change = change;
    return OR_OK;
}

/* ------------------------------------------------------------------------------------------
 * Continuous-MDP value iteration -- Algorithm 1 with Eq. 1-3 and the
 * nearest-neighbour successor of the note under it.  Readings:
 *   A36 the MDP: S = the grid's nodes; a model gives a finite action set, K outcomes per action
 *       with probabilities p_k and displacements Delta(s, a, k); s' = the node nearest to
 *       s + Delta: per axis i' = i + round_half_up(Delta_d / dx_d) computed in FLOAT32 (the kernel's
 *       precision: an integer decided by floating point), wrapped on periodic axes, clamped to
 *       [0, N-1] on the others.  Models:
 *         MDP_HOLONOMIC [speed, dt, gamma]: actions {stay, +-e_d}, Delta = +-dt speed e_d, K = 1.
 *         MDP_DUBINS3D [vbar, wbar, dt, slip, pslip, gamma]: (x, y, th); actions v in {vbar/2, vbar}
 *         x w in {-wbar, 0, wbar}; outcomes sigma in {0, +slip, -slip} with p {1-2 pslip, pslip,
 *         pslip}; Delta = (dt v cos th - sigma sin th, dt v sin th + sigma cos th, dt w).
 *   A37 Q(s, a) = R(s) + gamma sum_k p_k V(s'_k): Eq. 3's discount (l.6 prints no gamma; without it
 *       the iteration diverges); the reward depends on the state only (R given per node).
 *   A38 V_0 = 0 (l.2); one iteration takes V_{t+1}(s) = max_a Q(s, a) from V_t (l.3-7; the
 *       max with V_{t+1}(s) initialised below every Q); stop after the first iteration with
 *       max_s |V_{t+1}(s) - V_t(s)| < threshold (l.8-10's break read as the global test).
 *       order 0: Jacobi (all of V_{t+1} from V_t); order 1: in place (Gauss-Seidel) with the 8
 *       alternating orderings of §4.3 (as for Algorithm 3).  gamma < 1 makes the
 *       Bellman operator a contraction, so both orders have the same fixed point.
 * ---------------------------------------------------------------------------------------- */
enum { OR_MDP_HOLONOMIC = 0, OR_MDP_DUBINS3D = 1 };

typedef struct {
    int model, n, na, K;
    float act[13][6];        /* per action (at most 2n + 1 = 13): float32 parameters of the model */
    float dt, slip;
    double p[3], gamma;
} omdp;

static int omdp_init(omdp *m, int model, int n, const double *prm, int np) {
    memset(m, 0, sizeof(*m));
    m->model = model; m->n = n;
    if (model == OR_MDP_HOLONOMIC) {
        if (np != 3 || n < 1 || n > 6) return OR_EINVAL;
        m->na = 2 * n + 1; m->K = 1; m->p[0] = 1.0;
        const float step = (float)prm[1] * (float)prm[0];            /* dt * speed */
        for (int a = 1; a < m->na; ++a) {                              /* a = 1 + 2d (+), 2 + 2d (-) */
            const int d = (a - 1) / 2;
            m->act[a][d] = (a - 1) % 2 == 0 ? step : -step;
        }
        m->gamma = prm[2];
    } else if (model == OR_MDP_DUBINS3D) {
        if (np != 6 || n != 3) return OR_EINVAL;
        m->na = 6; m->K = 3;
        const float vbar = (float)prm[0], wbar = (float)prm[1];
        for (int a = 0; a < 6; ++a) {
            m->act[a][0] = (a / 3) == 0 ? 0.5f * vbar : vbar;          /* v */
            m->act[a][1] = (float)(a % 3 - 1) * wbar;                   /* w in {-wbar, 0, wbar} */
        }
        m->dt = (float)prm[2];
        m->slip = (float)prm[3];
        m->p[1] = m->p[2] = prm[4];
        m->p[0] = 1.0 - 2.0 * prm[4];
        m->gamma = prm[5];
    } else {
        return OR_EINVAL;
    }
    if (!(m->gamma >= 0.0 && m->gamma < 1.0)) return OR_EINVAL;
    return OR_OK;
}

/* flat index of the successor of node idx under (a, k) -- A36 (float32 decision) */

/* nearest node along an axis for a displacement of q cells, in float32: round half up, i.e. ties
 * toward the larger index (SPEC nearest_index); q - floor(q) is exact in float32 */
static int64_t nearest_shift_f32(float q) {
    const float fl = floorf(q);
    const float fr = q - fl;
    return (int64_t)fl + (fr >= 0.5f ? 1 : 0);
}

static int64_t omdp_succ(const og *g, const omdp *m, const float *inv_dx, const int64_t *idx, int a, int k) {
    float delta[6] = {0};
    if (m->model == OR_MDP_HOLONOMIC) {
        for (int d = 0; d < g->n; ++d) delta[d] = m->act[a][d];
    } else {
        const double th = g->x[2][idx[2]];
        const float c = (float)cos(th), s = (float)sin(th);
        const float sig = k == 0 ? 0.0f : (k == 1 ? m->slip : -m->slip);
        const float dtv = m->dt * m->act[a][0];
        const float t0 = dtv * c, t1 = sig * s, t2 = dtv * s, t3 = sig * c;
        delta[0] = t0 - t1;
        delta[1] = t2 + t3;
        delta[2] = m->dt * m->act[a][1];
    }
    int64_t flat = 0;
    for (int d = 0; d < g->n; ++d) {
        const float q = delta[d] * inv_dx[d];
        int64_t j = idx[d] + nearest_shift_f32(q);
        if (g->per[d]) { j %= g->N[d]; if (j < 0) j += g->N[d]; }
        else j = j < 0 ? 0 : (j > g->N[d] - 1 ? g->N[d] - 1 : j);
        flat += j * g->stride[d];
    }
    return flat;
}

int oracle_vi_successor(int n, const int64_t *N, const double *lo, const double *hi, uint32_t pmask, int model,
                        const double *prm, int np, const int64_t *idx, int a, int k, int64_t *flat_out) {
    og g;
    omdp m;
    int st = og_init(&g, n, N, lo, hi, pmask);
    if (!st) st = omdp_init(&m, model, n, prm, np);
    if (!st && (a < 0 || a >= m.na || k < 0 || k >= m.K)) st = OR_EINVAL;
    if (!st) {
        float inv_dx[6];
        for (int d = 0; d < n; ++d) inv_dx[d] = (float)(1.0 / g.dx[d]);
        *flat_out = omdp_succ(&g, &m, inv_dx, idx, a, k);
    }
    og_free(&g);
    return st;
}

int oracle_vi_solve(int n, const int64_t *N, const double *lo, const double *hi, uint32_t pmask, int model,
                    const double *prm, int np, const float *R, double threshold, int64_t max_iters, int order,
                    double *out, int64_t *iters_out, double *last_change) {
    og g;
    omdp m;
    int st = og_init(&g, n, N, lo, hi, pmask);
    if (st) { og_free(&g); return st; }
    if ((st = omdp_init(&m, model, n, prm, np))) { og_free(&g); return st; }
    if (max_iters < 1 || (order != 0 && order != 1)) { og_free(&g); return OR_EINVAL; }
    const int64_t P = g.P;
    float inv_dx[6];
    for (int d = 0; d < n; ++d) inv_dx[d] = (float)(1.0 / g.dx[d]);
    double *old = (double *)malloc(sizeof(double) * (size_t)P);
    if (!old) { og_free(&g); return OR_ENOMEM; }
    for (int64_t i = 0; i < P; ++i) out[i] = 0.0;                              /* l.2 */
    int64_t it = 0;
    double change = INFINITY;
    while (it < max_iters) {                                                   /* l.3 */
        memcpy(old, out, sizeof(double) * (size_t)P);
        const double *src = order == 0 ? old : out;                           /* A38 */
        for (int64_t kk = 0; kk < P; ++kk) {                                   /* l.4 */
            int64_t idx[6], r = kk, flat = 0;
            for (int d = n - 1; d >= 0; --d) {
                int64_t i = r % g.N[d];
                r /= g.N[d];
                if (order == 1 && d < 3 && (((it & 7) >> d) & 1)) i = g.N[d] - 1 - i;   /* §4.3 */
                idx[d] = i;
            }
            for (int d = 0; d < n; ++d) flat += idx[d] * g.stride[d];
            double best = -INFINITY;
            for (int a = 0; a < m.na; ++a) {                                   /* l.5 */
                double ev = 0.0;
                for (int k = 0; k < m.K; ++k)
                    ev += m.p[k] * src[omdp_succ(&g, &m, inv_dx, idx, a, k)];
                const double Q = (double)R[flat] + m.gamma * ev;                /* l.6, A37 */
                best = fmax(best, Q);                                          /* l.7 */
            }
            out[flat] = best;
        }
        change = 0.0;
        for (int64_t i = 0; i < P; ++i) change = fmax(change, fabs(out[i] - old[i]));   /* l.8 */
        ++it;
        if (change < threshold) break;                                        /* l.9-10, A38 */
    }
    free(old);
    og_free(&g);
    if (iters_out) *iters_out = it;
    if (last_change) *last_change = change;
    return OR_OK;
}

int oracle_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
