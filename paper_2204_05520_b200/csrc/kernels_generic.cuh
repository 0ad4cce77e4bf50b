// kernels_generic.cuh -- the "generic" kernel family: one thread per node, every stencil
// neighbour read through L1/L2 (__ldg), any dims 1..6, any extents.  Correctness baseline and
// fallback for grids the tiled family does not cover (small or odd shapes).
//
//   k_pass1  Alg. 2 l.152-159: per-axis min/max of D-/D+ over all nodes (reading A4), max|W|, NaN
//   k_pass2  Alg. 2 l.152-156 + l.160-163 + l.169: D+-, p, H, alpha_i, L, stage update, BRT min
#pragma once

#include "odp_device.cuh"

namespace odp {

// Per-CTA partial of pass 1: [minD(n), maxD(n), maxabs, nan] floats at partials + blockIdx.x*(2n+2)
template <int NDIM>
__device__ __forceinline__ void block_reduce_range(float *mn, float *mx, float mabs, int nan, float *partials) {
    __shared__ float red[32][2 * MAXD + 2];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
#pragma unroll
        for (int d = 0; d < NDIM; ++d) {
            mn[d] = fminf(mn[d], __shfl_xor_sync(0xffffffffu, mn[d], off));
            mx[d] = fmaxf(mx[d], __shfl_xor_sync(0xffffffffu, mx[d], off));
        }
        mabs = fmaxf(mabs, __shfl_xor_sync(0xffffffffu, mabs, off));
        nan |= __shfl_xor_sync(0xffffffffu, nan, off);
    }
    if (lane == 0) {
#pragma unroll
        for (int d = 0; d < NDIM; ++d) { red[warp][d] = mn[d]; red[warp][NDIM + d] = mx[d]; }
        red[warp][2 * NDIM] = mabs;
        red[warp][2 * NDIM + 1] = (float)nan;
    }
    __syncthreads();
    const int nw = (blockDim.x + 31) >> 5;
    if (threadIdx.x < 2 * NDIM + 2) {
        const int q = threadIdx.x;
        float r = red[0][q];
        for (int w = 1; w < nw; ++w) {
            const float o = red[w][q];
            r = (q < NDIM) ? fminf(r, o) : fmaxf(r, o);
        }
        partials[(long long)blockIdx.x * (2 * NDIM + 2) + q] = r;
    }
}

// Load of a value array: through the non-coherent path for the launch-per-pass kernels (W is
// read-only for the launch), through L2 (ld.global.cg) inside k_resident, where the arrays are
// rewritten between the grid barriers of one launch.
template <bool CG>
__device__ __forceinline__ float ldw(const float *p) { return CG ? __ldcg(p) : __ldg(p); }

// Value of W at offset k (|k| <= R) from local node `i` (flat index) along axis d, whose index on
// that axis is `id` (local).  Periodic axes wrap; non-periodic out-of-domain slots are left for
// fix_ghosts.  Axis 0 consults the global index so halo planes of a slab are used.
template <int R, bool CG = false>
__device__ __forceinline__ void load_line(const GridDev &g, const float *__restrict__ W, long long i, int d,
                                          int id, float *v) {
    const long long s = g.stride[d];
    if (d == 0) {
        const int gid = g.g0 + id;
#pragma unroll
        for (int k = -R; k <= R; ++k) {
            const int gj = gid + k;
            if (gj >= 0 && gj < g.Ng0) v[k + R] = ldw<CG>(W + i + k * s);
            else if (g.per[0]) { int w = gj < 0 ? gj + g.Ng0 : gj - g.Ng0; v[k + R] = ldw<CG>(W + i + (long long)(w - gid) * s); }
            else v[k + R] = 0.f;
        }
        if (!g.per[0]) fix_ghosts<R>(v, gid, g.Ng0);
        return;
    }
    const int N = g.N[d];
#pragma unroll
    for (int k = -R; k <= R; ++k) {
        const int j = id + k;
        if (j >= 0 && j < N) v[k + R] = ldw<CG>(W + i + k * s);
        else if (g.per[d]) { int w = j < 0 ? j + N : j - N; v[k + R] = ldw<CG>(W + i + (long long)(w - id) * s); }
        else v[k + R] = 0.f;
    }
    if (!g.per[d]) fix_ghosts<R>(v, id, N);
}

template <int NDIM>
__device__ __forceinline__ void node_index(const GridDev &g, long long i, int *idx) {
    const long long r = (g.P <= 0x7fffffffLL) ? (long long)((unsigned)i / (unsigned)g.stride[0]) : i / g.stride[0];
    idx[0] = (int)r;
    int rem = (int)(i - r * g.stride[0]);
#pragma unroll
    for (int d = NDIM - 1; d >= 1; --d) {
        idx[d] = rem % g.N[d];
        rem /= g.N[d];
    }
}

// Pass 1 of one stage over all nodes, grid-stride; st may point to a CTA-local (shared) copy.
template <int NDIM, int R, bool CG>
__device__ __forceinline__ void pass1_generic_body(const GridDev &g, const float *__restrict__ W, float *partials,
                                                   const DevState *st) {
    if (!st->active) return;
    float mn[NDIM], mx[NDIM];
#pragma unroll
    for (int d = 0; d < NDIM; ++d) { mn[d] = __int_as_float(0x7f800000); mx[d] = -__int_as_float(0x7f800000); }
    float mabs = 0.f;
    int nan = 0;
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < g.P; i += stride) {
        int idx[NDIM];
        node_index<NDIM>(g, i, idx);
        const float w = ldw<CG>(W + i);
        nan |= (w != w);
        mabs = fmaxf(mabs, fabsf(w));
#pragma unroll
        for (int d = 0; d < NDIM; ++d) {
            float v[2 * R + 1], dm, dp;
            load_line<R, CG>(g, W, i, d, idx[d], v);
            deriv<R>(v, g.inv_dx[d], dm, dp);
            mn[d] = fminf(mn[d], fminf(dm, dp));
            mx[d] = fmaxf(mx[d], fmaxf(dm, dp));
        }
    }
    block_reduce_range<NDIM>(mn, mx, mabs, nan, partials);
}

template <int NDIM, int R>
__global__ void __launch_bounds__(256) k_pass1_generic(GridDev g, const float *__restrict__ W, float *partials,
                                                       const DevState *st) {
    pass1_generic_body<NDIM, R, false>(g, W, partials, st);
}

// Pass 2 of one stage over all nodes, grid-stride; st may point to a CTA-local (shared) copy.
template <class F, int NDIM, int R, bool CG>
__device__ __forceinline__ void pass2_generic_body(const GridDev &g, const float *__restrict__ W, const float *Vn,
                                                   const float *__restrict__ T, float *out, const DevState *st,
                                                   const FParams &fp, int kind, int brt) {
    if (!st->active) return;
    F f;
    f.init(fp, st->minD, st->maxD);
    const float dt = st->dt_f;
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < g.P; i += stride) {
        int idx[NDIM];
        node_index<NDIM>(g, i, idx);
        Pt q;
#pragma unroll
        for (int d = 0; d < NDIM; ++d) load_axis<F>(g, q, d, d == 0 ? g.g0 + idx[0] : idx[d]);
        float dm[NDIM], dp[NDIM], p[NDIM];
#pragma unroll
        for (int d = 0; d < NDIM; ++d) {
            float v[2 * R + 1];
            load_line<R, CG>(g, W, i, d, idx[d], v);
            deriv<R>(v, g.inv_dx[d], dm[d], dp[d]);
            p[d] = 0.5f * (dm[d] + dp[d]);                 // A3
        }
        float L = f.ham(q, p);                              // l.154-156
#pragma unroll
        for (int d = 0; d < NDIM; ++d) L = fmaf(f.alpha(d, q), 0.5f * (dp[d] - dm[d]), L);   // l.163 (A2)
        out[i] = stage_update(kind, brt, ldw<CG>(W + i), L, dt, Vn, T, i);
    }
}

template <class F, int NDIM, int R>
__global__ void __launch_bounds__(256) k_pass2_generic(GridDev g, const float *__restrict__ W,
                                                       const float *Vn, const float *__restrict__ T,
                                                       float *out, const DevState *st, FParams fp,
                                                       int kind, int brt) {
    pass2_generic_body<F, NDIM, R, false>(g, W, Vn, T, out, st, fp, kind, brt);
}

}  // namespace odp
