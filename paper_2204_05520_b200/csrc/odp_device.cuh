// odp_device.cuh -- device-side data layout, stencil helpers and the compiled-in dynamics
// functors of the B200 HJ level-set step.  Independent of oracle/ (no shared code).
//
// Paper: Bui et al., OptimizedDP (arXiv 2204.05520), §3.2 Algorithm 2,
// §3.4.1 grid and ghost points, §3.4.4 derivatives.  Readings A1-A27: DESIGN.md §3.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace odp {

constexpr int MAXD = 6;

// ---------------------------------------------------------------------------------------------
// Layout of one (local) grid in HBM: a row-major float32 array, axis 0 outermost.  On a
// multi-GPU slab the local array is a contiguous range of axis-0 planes, preceded and followed by
// R halo planes in the same allocation (W points at local plane 0).
// ---------------------------------------------------------------------------------------------
struct GridDev {
    int n;
    int N[MAXD];             // local extents; N[0] = local axis-0 planes
    int Ng0;                 // global axis-0 extent
    int g0;                  // global index of local plane 0
    int per[MAXD];           // periodic flags
    long long stride[MAXD];  // element strides (stride[n-1] = 1)
    long long P;             // local points = N[0] * stride[0]
    float inv_dx[MAXD];      // float(1/dx_d)
    float hih[MAXD];         // 0.5f * inv_dx[d] = 1/(2 dx_d)
    float dx[MAXD];
    const float *tab;        // per axis: x[Ng_d], cos x[Ng_d], sin x[Ng_d] (float32 of float64 values)
    int tab_off[MAXD];       // offset of axis d's x-table in tab; cos at +Ng_d, sin at +2 Ng_d
    int Ng[MAXD];            // global extents
};

// Device-resident solver state: the time loop runs without host round trips (the host only
// polls `active`/`status` between launch chunks).
struct DevState {
    double tau;          // current time (float64, reading A9)
    double tau_target;   // next save time tau_k
    double eps;          // 1e-12 max(1, tau_last)
    double dt;           // step of the current time step (float64)
    double cfl;
    float dt_f;          // dt as used by the update kernels
    float minD[MAXD], maxD[MAXD];   // global derivative range of the current stage input (A4)
    float amax[MAXD];               // alpha^max of the current step (Alg. 2 l.164)
    float maxabs;
    int nan;
    int active;          // 1 while the current save interval still needs steps
    int status;          // 0 ok, 2 numeric failure (A19)
    int pending;         // single-pass: the last stage's OUTPUT failed the guard; fail at the next stage's start
    unsigned int work[3];  // dynamic work counters of the march launches: pass 1, pass 2, split pass 1 (boundary)
    long long steps, stages;
};

struct FParams { float c[8]; };

// Coordinates of one node that a functor may read.
struct Pt { float x[MAXD], c[MAXD], s[MAXD]; };

__device__ __forceinline__ float sgn1(float v) { return v >= 0.f ? 1.f : -1.f; }   // A14: sgn(0) = +1

// A12: sign-adjusted linear extrapolation, q >= 1 cells beyond the face with edge value e and the
// next inner value in: e + q |e - in| sgn(e)   (addGhostExtrapolate)
__device__ __forceinline__ float ghost(float e, float in, float q) {
    return fmaf(q, fabsf(e - in) * sgn1(e), e);
}

// A13: ENO2 selection -- the smaller second difference in magnitude, left on ties
__device__ __forceinline__ float eno_pick(float a, float b) { return fabsf(a) <= fabsf(b) ? a : b; }

// One-sided derivatives from the 2R+1 values v[0..2R] centred on the node (§3.4.4).
template <int R>
__device__ __forceinline__ void deriv(const float *v, float inv_h, float &dm, float &dp) {
    if constexpr (R == 1) {
        dm = (v[1] - v[0]) * inv_h;
        dp = (v[2] - v[1]) * inv_h;
    } else {
        const float d2m = fmaf(-2.f, v[1], v[0] + v[2]);   // delta^2 at i-1
        const float d20 = fmaf(-2.f, v[2], v[1] + v[3]);   // delta^2 at i
        const float d2p = fmaf(-2.f, v[3], v[2] + v[4]);   // delta^2 at i+1
        const float hh = 0.5f * inv_h;
        dm = fmaf(eno_pick(d2m, d20), hh, (v[2] - v[1]) * inv_h);
        dp = fmaf(-eno_pick(d20, d2p), hh, (v[3] - v[2]) * inv_h);
    }
}

// Replace the out-of-domain entries of a line window v[0..2R] (centre index i, extent N) by
// ghost values.  Non-periodic only; in-domain entries are untouched (periodic lines are loaded
// wrapped and never reach here).
template <int R>
__device__ __forceinline__ void fix_ghosts(float *v, int i, int N) {
    // (all window indices are compile-time constants so v stays in registers)
    if (i < R) {            // low face inside the window: face value at slot R - i, inner at R - i + 1
        float e = v[R], in = v[R + 1];
#pragma unroll
        for (int ii = 1; ii < R; ++ii)
            if (i == ii) { e = v[R - ii]; in = v[R - ii + 1]; }
#pragma unroll
        for (int k = 0; k < R; ++k)
            if (k < R - i) v[k] = ghost(e, in, float(R - i - k));
    }
    const int m = N - 1 - i;  // distance of the centre from the high face
    if (m < R) {              // high face at slot R + m, inner at R + m - 1
        float e = v[R], in = v[R - 1];
#pragma unroll
        for (int mm = 1; mm < R; ++mm)
            if (m == mm) { e = v[R + mm]; in = v[R + mm - 1]; }
#pragma unroll
        for (int k = R + 1; k <= 2 * R; ++k)
            if (k > R + m) v[k] = ghost(e, in, float(k - R - m));
    }
}

// ---------------------------------------------------------------------------------------------
// Dynamics functors (reading A22).  Each provides
//   NEED_X / NEED_TRIG  bitmasks of the axes whose coordinate / (cos, sin) the functor reads,
//   deps(d)             bitmask of the axes alpha_d depends on (<= 2 axes, or all 3 with DEPS3),
//   init(P, minD, maxD) per-stage constants from params and the global derivative range,
//   ham(pt, p)          H = p . f(x, u*, d*) with bang-bang u*, d* (Alg. 2 l.154-156, Eq. 4),
//   alpha(d, pt)        max over p in [minD, maxD] of |dH/dp_d| (Alg. 2 l.162, reading A5).
// goal = params[last]: -1 minimise (reach), +1 maximise (avoid); disturbance opposite (A1).
// ---------------------------------------------------------------------------------------------
struct SignSet {
    bool pos, neg;
    __device__ void set(float mn, float mx) { pos = mx >= 0.f; neg = mn < 0.f; }
    // max over s in the set of |a + b s|
    __device__ float maxabs(float a, float b) const {
        float r = 0.f;
        if (pos) r = fabsf(a + b);
        if (neg) r = fmaxf(r, fabsf(a - b));
        return r;
    }
};

template <int NDIM>
struct FHoloBall {   // [ubar, goal]: xdot = u, |u|_2 <= ubar
    // alpha_(i,d) does not depend on the stage's derivative range: false
    static constexpr bool RANGE_FREE = false;
    static constexpr bool SEPARABLE = true, DEPS3 = false;
    static constexpr int NEED_X = 0, NEED_TRIG = 0;
    static constexpr __host__ __device__ int deps(int) { return 0; }
    float kH, a[NDIM];
    __device__ void init(const FParams &P, const float *mn, const float *mx) {
        kH = P.c[1] * P.c[0];
#pragma unroll
        for (int d = 0; d < NDIM; ++d) {     // ubar M_d / sqrt(M_d^2 + sum_e m_e^2)
            const float Md = fmaxf(fabsf(mn[d]), fabsf(mx[d]));
            float den = Md * Md;
#pragma unroll
            for (int e = 0; e < NDIM; ++e) {
                if (e == d) continue;
                const float me = (mn[e] <= 0.f && mx[e] >= 0.f) ? 0.f : fminf(fabsf(mn[e]), fabsf(mx[e]));
                den = fmaf(me, me, den);
            }
            a[d] = Md == 0.f ? 0.f : P.c[0] * Md / sqrtf(den);
        }
    }
    __device__ float ham(const Pt &, const float *p) const {
        float s = 0.f;
#pragma unroll
        for (int d = 0; d < NDIM; ++d) s = fmaf(p[d], p[d], s);
        return kH * sqrtf(s);
    }
    __device__ float alpha(int d, const Pt &) const { return a[d]; }
};

template <int NDIM>
struct FHoloBox {    // [ubar, dbar, goal]: xdot_i = u_i + d_i
    // alpha_(i,d) does not depend on the stage's derivative range: true
    static constexpr bool RANGE_FREE = true;
    static constexpr bool SEPARABLE = true, DEPS3 = false;
    static constexpr int NEED_X = 0, NEED_TRIG = 0;
    static constexpr __host__ __device__ int deps(int) { return 0; }
    float kH, a[NDIM];
    __device__ void init(const FParams &P, const float *mn, const float *mx) {
        const float g = P.c[2];
        kH = g * P.c[0] - g * P.c[1];
#pragma unroll
        for (int d = 0; d < NDIM; ++d) {
            SignSet S; S.set(mn[d], mx[d]);
            a[d] = S.maxabs(0.f, kH);
        }
    }
    __device__ float ham(const Pt &, const float *p) const {
        float s = 0.f;
#pragma unroll
        for (int d = 0; d < NDIM; ++d) s += fabsf(p[d]);
        return kH * s;
    }
    __device__ float alpha(int d, const Pt &) const { return a[d]; }
};

struct FDubins3D {   // [v, wbar, goal]: (x, y, th) -> (v cos th, v sin th, w)
    // alpha_(i,d) does not depend on the stage's derivative range: true
    static constexpr bool RANGE_FREE = true;
    static constexpr bool SEPARABLE = true, DEPS3 = false;
    static constexpr int NDIM = 3;
    static constexpr int NEED_X = 0, NEED_TRIG = 1 << 2;
    static constexpr __host__ __device__ int deps(int d) { return d < 2 ? (1 << 2) : 0; }
    float v, kw, a2;
    __device__ void init(const FParams &P, const float *mn, const float *mx) {
        v = P.c[0];
        kw = P.c[2] * P.c[1];
        SignSet S; S.set(mn[2], mx[2]);
        a2 = S.maxabs(0.f, kw);
    }
    __device__ float ham(const Pt &q, const float *p) const {
        return fmaf(kw, fabsf(p[2]), fmaf(p[1], v * q.s[2], p[0] * (v * q.c[2])));
    }
    __device__ float alpha(int d, const Pt &q) const {
        return d == 0 ? fabsf(v * q.c[2]) : (d == 1 ? fabsf(v * q.s[2]) : a2);
    }
};

struct FCar4D {      // [abar, wbar, dxbar, dybar, goal]: (x, y, v, th)
    // alpha_(i,d) does not depend on the stage's derivative range: false
    static constexpr bool RANGE_FREE = false;
    static constexpr bool SEPARABLE = true, DEPS3 = false;
    static constexpr int NDIM = 4;
    static constexpr int NEED_X = 1 << 2, NEED_TRIG = 1 << 3;
    static constexpr __host__ __device__ int deps(int d) { return d < 2 ? ((1 << 2) | (1 << 3)) : 0; }
    float ka, kw, kdx, kdy, a2, a3;
    SignSet Sx, Sy;
    __device__ void init(const FParams &P, const float *mn, const float *mx) {
        const float g = P.c[4];
        ka = g * P.c[0]; kw = g * P.c[1];
        kdx = -g * P.c[2]; kdy = -g * P.c[3];     // disturbance takes the opposite goal
        Sx.set(mn[0], mx[0]); Sy.set(mn[1], mx[1]);
        SignSet Sv, St; Sv.set(mn[2], mx[2]); St.set(mn[3], mx[3]);
        a2 = Sv.maxabs(0.f, ka); a3 = St.maxabs(0.f, kw);
    }
    __device__ float ham(const Pt &q, const float *p) const {
        const float vx = q.x[2] * q.c[3], vy = q.x[2] * q.s[3];
        float H = p[0] * vx;
        H = fmaf(p[1], vy, H);
        H = fmaf(ka, fabsf(p[2]), H);
        H = fmaf(kw, fabsf(p[3]), H);
        H = fmaf(kdx, fabsf(p[0]), H);
        H = fmaf(kdy, fabsf(p[1]), H);
        return H;
    }
    __device__ float alpha(int d, const Pt &q) const {
        if (d == 0) return Sx.maxabs(q.x[2] * q.c[3], kdx);
        if (d == 1) return Sy.maxabs(q.x[2] * q.s[3], kdy);
        return d == 2 ? a2 : a3;
    }
};

struct FCar5D {      // [abar, alphabar, goal]: (x, y, th, v, w)
    // alpha_(i,d) does not depend on the stage's derivative range: true
    static constexpr bool RANGE_FREE = true;
    static constexpr bool SEPARABLE = true, DEPS3 = false;
    static constexpr int NDIM = 5;
    static constexpr int NEED_X = (1 << 3) | (1 << 4), NEED_TRIG = 1 << 2;
    static constexpr __host__ __device__ int deps(int d) {
        return d < 2 ? ((1 << 2) | (1 << 3)) : (d == 2 ? (1 << 4) : 0);
    }
    float ka, kal, a3, a4;
    __device__ void init(const FParams &P, const float *mn, const float *mx) {
        const float g = P.c[2];
        ka = g * P.c[0]; kal = g * P.c[1];
        SignSet Sv, Sw; Sv.set(mn[3], mx[3]); Sw.set(mn[4], mx[4]);
        a3 = Sv.maxabs(0.f, ka); a4 = Sw.maxabs(0.f, kal);
    }
    __device__ float ham(const Pt &q, const float *p) const {
        float H = p[0] * (q.x[3] * q.c[2]);
        H = fmaf(p[1], q.x[3] * q.s[2], H);
        H = fmaf(p[2], q.x[4], H);
        H = fmaf(ka, fabsf(p[3]), H);
        H = fmaf(kal, fabsf(p[4]), H);
        return H;
    }
    __device__ float alpha(int d, const Pt &q) const {
        if (d == 0) return fabsf(q.x[3] * q.c[2]);
        if (d == 1) return fabsf(q.x[3] * q.s[2]);
        if (d == 2) return fabsf(q.x[4]);
        return d == 3 ? a3 : a4;
    }
};

struct FDoubleInt6D {  // [ubar, dbar, goal]: (px, vx, py, vy, pz, vz) -> (v_i, u_i + d_i)
    // alpha_(i,d) does not depend on the stage's derivative range: true
    static constexpr bool RANGE_FREE = true;
    static constexpr bool SEPARABLE = true, DEPS3 = false;
    static constexpr int NDIM = 6;
    static constexpr int NEED_X = (1 << 1) | (1 << 3) | (1 << 5), NEED_TRIG = 0;
    static constexpr __host__ __device__ int deps(int d) { return (d & 1) == 0 ? (1 << (d + 1)) : 0; }
    float kv, av[3];
    __device__ void init(const FParams &P, const float *mn, const float *mx) {
        const float g = P.c[2];
        kv = g * P.c[0] - g * P.c[1];
#pragma unroll
        for (int i = 0; i < 3; ++i) { SignSet S; S.set(mn[2 * i + 1], mx[2 * i + 1]); av[i] = S.maxabs(0.f, kv); }
    }
    __device__ float ham(const Pt &q, const float *p) const {
        float H = 0.f;
#pragma unroll
        for (int i = 0; i < 3; ++i) {
            H = fmaf(p[2 * i], q.x[2 * i + 1], H);
            H = fmaf(kv, fabsf(p[2 * i + 1]), H);
        }
        return H;
    }
    __device__ float alpha(int d, const Pt &q) const {
        return (d & 1) == 0 ? fabsf(q.x[d + 1]) : av[d >> 1];
    }
};

struct FPairDubins3D {  // Eq. 7 [va, vb, abar, bbar, goal]: relative (x, y, th) of a pursuer b
                       // w.r.t. an evader a: xdot = -va + vb cos th + a y, ydot = va sin th - a x,
                       // thdot = b - a; a (control) takes the goal's extremum, b the opposite (A30)
    static constexpr int NDIM = 3;
    static constexpr int NEED_X = (1 << 0) | (1 << 1), NEED_TRIG = 1 << 2;
    // alpha_d depends on (x, y) through the switching function and on th through the drift
    static constexpr __host__ __device__ int deps(int) { return 0x7; }
    static constexpr bool RANGE_FREE = false;       // the sign set of q = p_x y - p_y x - p_th
    static constexpr bool SEPARABLE = false, DEPS3 = true;
    float va, vb, ka, kb;                            // ka = goal abar, kb = -goal bbar
    float mn[3], mx[3];                              // the stage's costate box (A4)
    __device__ void init(const FParams &P, const float *lo, const float *hi) {
        va = P.c[0]; vb = P.c[1];
        ka = P.c[4] * P.c[2];
        kb = -P.c[4] * P.c[3];
#pragma unroll
        for (int d = 0; d < 3; ++d) { mn[d] = lo[d]; mx[d] = hi[d]; }
    }
    __device__ float ham(const Pt &q, const float *p) const {
        const float x = q.x[0], y = q.x[1];
        const float sw = fmaf(p[0], y, -fmaf(p[1], x, p[2]));     // q = p_x y - p_y x - p_th
        const float a = ka * sgn1(sw), b = kb * sgn1(p[2]);
        float H = p[0] * fmaf(vb, q.c[2], fmaf(a, y, -va));
        H = fmaf(p[1], fmaf(va, q.s[2], -a * x), H);
        H = fmaf(p[2], b - a, H);
        return H;
    }
    // alpha_{i,d}: maximum of |f_d| over the sign set of q on the costate box (exact: q is linear
    // in p, its range is the sum of the ranges of its terms) and, for th, the sign set of p_th (A30)
    __device__ float alpha(int d, const Pt &q) const {
        const float x = q.x[0], y = q.x[1];
        const float qlo = fminf(y * mn[0], y * mx[0]) + fminf(-x * mn[1], -x * mx[1]) - mx[2];
        const float qhi = fmaxf(y * mn[0], y * mx[0]) + fmaxf(-x * mn[1], -x * mx[1]) - mn[2];
        float best = 0.f;
#pragma unroll
        for (int j = 0; j < 2; ++j) {
            const float sq = j == 0 ? 1.f : -1.f;
            if (j == 0 ? !(qhi >= 0.f) : !(qlo < 0.f)) continue;
            const float a = ka * sq;
            if (d == 0) best = fmaxf(best, fabsf(fmaf(vb, q.c[2], fmaf(a, y, -va))));
            else if (d == 1) best = fmaxf(best, fabsf(fmaf(va, q.s[2], -a * x)));
            else {
                if (mx[2] >= 0.f) best = fmaxf(best, fabsf(kb - a));
                if (mn[2] < 0.f) best = fmaxf(best, fabsf(-kb - a));
            }
        }
        return best;
    }
};

// Coordinates of axis a at global index i from the tables.
template <class F>
__device__ __forceinline__ void load_axis(const GridDev &g, Pt &q, int a, int i) {
    if ((F::NEED_X >> a) & 1) q.x[a] = __ldg(g.tab + g.tab_off[a] + i);
    if ((F::NEED_TRIG >> a) & 1) {
        q.c[a] = __ldg(g.tab + g.tab_off[a] + g.Ng[a] + i);
        q.s[a] = __ldg(g.tab + g.tab_off[a] + 2 * g.Ng[a] + i);
    }
}

enum StageKind { STAGE_EULER = 0, STAGE_RK1 = 1, STAGE_RK2 = 2 };

// The update of Alg. 2 l.169 (A2 sign in L) for one node, plus the BRT min (A11).
// Vn may alias the output (RK2 stage 2 updates Vn in place: each node reads its own Vn entry
// before writing it), so it is neither __restrict__ nor read through the non-coherent path.
__device__ __forceinline__ float stage_update(int kind, int brt, float w, float L, float dt,
                                              const float *Vn, const float *__restrict__ T,
                                              long long i) {
    float v;
    if (kind == STAGE_RK2) {
        const float v2 = fmaf(dt, L, w);            // V2 = V1 + dt L(V1)
        v = 0.5f * (Vn[i] + v2);                    // (Vn + V2) / 2   (A10)
    } else {
        v = fmaf(dt, L, w);                          // Euler / RK stage 1
    }
    if (brt && kind != STAGE_RK1) v = fminf(v, __ldg(T + i));
    return v;
}

}  // namespace odp
