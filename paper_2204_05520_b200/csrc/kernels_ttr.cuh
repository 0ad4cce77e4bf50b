// kernels_ttr.cuh -- time-to-reach by Lax-Friedrichs iteration (§3.3,
// Algorithm 3; readings A31-A35 in DESIGN.md §3).
//
// Algorithm 3 updates the grid in place in alternating orderings (Gauss-Seidel, §4.3).
// A sequential in-place sweep has no parallelism across the grid, so the GPU path iterates the
// same update as a Jacobi iteration (reading A35): every node of iteration k+1 is computed from
// iteration k, then the boundary rule of l.14-15 is applied along each non-periodic axis in order
// 0..n-1 (reading A34).  One iteration = one k_ttr_interior launch + one k_ttr_face launch per
// non-periodic axis + k_ttr_ctl; buffers alternate, the convergence test (A31) runs on the device.
//
//   k_ttr_init      l.1: phi = 0 on the target {V0 <= 0}, `big` elsewhere
//   k_ttr_interior  l.5-12 for every node not on a non-periodic face (A32, A33)
//   k_ttr_face<d>   l.14-15 along axis d on its two faces
//   k_ttr_ctl       l.2 (A31): stop once max |phi_new - phi_old| <= eps (or the iteration cap)
#pragma once

#include "odp_device.cuh"
#include "kernels_generic.cuh"

namespace odp {

struct TtrState {
    unsigned change[2];   // float bits of max |phi_new - phi_old| of the iteration writing parity p
    int done;             // 1 once the stop test passed
    int parity;           // buffer holding the result once done
    long long iters;      // iterations executed
    long long max_iters;
    float eps;
    int pad;
};

__device__ __forceinline__ void ttr_reduce_change(float c, TtrState *st, int par) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) c = fmaxf(c, __shfl_xor_sync(0xffffffffu, c, off));
    // |x| >= 0: IEEE order of non-negative floats is the order of their bit patterns
    if ((threadIdx.x & 31) == 0 && c > 0.f) atomicMax(&st->change[par], __float_as_uint(c));
}

__global__ void __launch_bounds__(256) k_ttr_init(long long P, const float *__restrict__ V0, float big,
                                                  float *__restrict__ phi) {
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < P; i += stride)
        phi[i] = __ldg(V0 + i) <= 0.f ? 0.f : big;                      // l.1
}

__global__ void k_ttr_reset(TtrState *st, long long max_iters, float eps) {
    st->change[0] = st->change[1] = 0u;
    st->done = 0; st->parity = 0; st->iters = 0;
    st->max_iters = max_iters; st->eps = eps;
}

// l.5-12 on every node; face nodes of non-periodic axes are copied (their value comes from
// k_ttr_face).  Reads src (iteration k), writes dst (iteration k+1).
template <class F, int NDIM>
__global__ void __launch_bounds__(256) k_ttr_interior(GridDev g, FParams fp, const float *__restrict__ V0,
                                                      const float *__restrict__ src, float *__restrict__ dst,
                                                      TtrState *st, int par) {
    if (st->done) return;
    F f;
    {
        float mn[MAXD], mx[MAXD];
#pragma unroll
        for (int d = 0; d < MAXD; ++d) { mn[d] = -1.f; mx[d] = 1.f; }        // A33: costate box [-1, 1]^n
        f.init(fp, mn, mx);
    }
    float cmax = 0.f;
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < g.P; i += stride) {
        int idx[NDIM];
        node_index<NDIM>(g, i, idx);
        const float old = src[i];
        bool face = false;
#pragma unroll
        for (int d = 0; d < NDIM; ++d) face |= !g.per[d] && (idx[d] == 0 || idx[d] == g.N[d] - 1);
        if (face || __ldg(V0 + i) <= 0.f) { dst[i] = old; continue; }     // A34: faces later, target fixed
        Pt q;
        float p[NDIM];
        float num = 0.f, den = 0.f;
#pragma unroll
        for (int d = 0; d < NDIM; ++d) load_axis<F>(g, q, d, idx[d]);   // alpha_d may read any axis
#pragma unroll
        for (int d = 0; d < NDIM; ++d) {
            const long long s = g.stride[d];
            long long op = s, om = -s;
            if (g.per[d]) {                              // periodic wrap (interior nodes never wrap otherwise)
                if (idx[d] == g.N[d] - 1) op = -(long long)(g.N[d] - 1) * s;
                if (idx[d] == 0) om = (long long)(g.N[d] - 1) * s;
            }
            const float vp = src[i + op], vm = src[i + om];
            p[d] = (vp - vm) * g.hih[d];                 // central difference (A32)
            num = fmaf(f.alpha(d, q) * g.hih[d], vp + vm, num);
            den = fmaf(f.alpha(d, q), g.inv_dx[d], den);
        }
        const float H = -f.ham(q, p) - 1.f;              // A32: H_TTR = -H_reach(goal -1) - 1
        const float nv = den > 0.f ? (num - H) / den : old;    // l.10-11 (A33)
        const float v = fminf(nv, old);                  // l.12
        dst[i] = v;
        cmax = fmaxf(cmax, fabsf(v - old));
    }
    ttr_reduce_change(cmax, st, par);
}

// l.14-15 along axis d: phi_face = min(max(2 phi_1 - phi_2, phi_2), phi_face) on both faces, from
// the values already in dst (after the interior update and the rules of axes < d).  Nodes whose
// highest non-periodic face axis is d are final here and enter the change.
template <int NDIM>
__global__ void __launch_bounds__(256) k_ttr_face(GridDev g, int d, const float *__restrict__ src, float *dst,
                                                  TtrState *st, int par) {
    if (st->done) return;
    const long long inner = g.stride[d];
    const long long outer = g.P / (inner * g.N[d]);
    const long long per_side = outer * inner;
    const int Nd = g.N[d];
    float cmax = 0.f;
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < 2 * per_side; t += stride) {
        const int side = t >= per_side;
        const long long r = side ? t - per_side : t;
        const long long o = r / inner, in = r - o * inner;
        const long long i = o * (inner * Nd) + (side ? (long long)(Nd - 1) * inner : 0) + in;
        const long long sa = side ? -inner : inner;
        const float a = dst[i + sa], b = dst[i + 2 * sa], cur = dst[i];
        const float v = fminf(fmaxf(2.f * a - b, b), cur);
        dst[i] = v;
        int idx[NDIM];
        node_index<NDIM>(g, i, idx);
        bool last = true;
#pragma unroll
        for (int e = 0; e < NDIM; ++e)
            if (e > d && !g.per[e] && (idx[e] == 0 || idx[e] == g.N[e] - 1)) last = false;
        if (last) cmax = fmaxf(cmax, fabsf(v - src[i]));
    }
    ttr_reduce_change(cmax, st, par);
}

// l.2 (A31): the iteration that wrote parity `par` is done; stop when its change <= eps.
__global__ void k_ttr_ctl(TtrState *st, int par) {
    if (st->done) return;
    st->iters += 1;
    const float c = __uint_as_float(st->change[par]);
    if (c <= st->eps || st->iters >= st->max_iters) { st->done = 1; st->parity = par; return; }
    st->change[par ^ 1] = 0u;
}

typedef void (*ttr_interior_fn)(GridDev, FParams, const float *, const float *, float *, TtrState *, int);
typedef void (*ttr_face_fn)(GridDev, int, const float *, float *, TtrState *, int);

struct TtrFns {
    ttr_interior_fn interior = nullptr;
    ttr_face_fn face = nullptr;
};

template <class F, int NDIM>
static TtrFns ttr_fns() {
    TtrFns t;
    t.interior = k_ttr_interior<F, NDIM>;
    t.face = k_ttr_face<NDIM>;
    return t;
}

}  // namespace odp
