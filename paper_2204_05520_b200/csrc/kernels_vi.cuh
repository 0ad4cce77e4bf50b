// kernels_vi.cuh -- continuous-MDP value iteration (§3.1, Algorithm 1,
// P:117-133, Eq. 1-3; readings A36-A38 in DESIGN.md §3).
//
//   V_{t+1}(s) = max_a [ R(s) + gamma sum_k p_k V_t(s'_k) ],  s'_k = nearest node to s + Delta(s, a, k)
//
// One launch per iteration (Jacobi order, A38), the stop test in the last CTA (shared driver with
// the time-to-reach path).  Thread = one column (fixed indices of axes 1..n-1), marching axis 0.
// A model's displacement never depends on the axis-0 coordinate (both models here), so the
// successor of every (action, outcome) is, per column, a constant in-plane offset plus a constant
// axis-0 shift: the float32 snapping arithmetic of A36 runs once per column, and each node costs
// NA*K gathers (L1/L2 hits: successors are a few cells away), clamps and FMAs -- a gather-bound
// kernel.
#pragma once

#include "odp_device.cuh"
#include "kernels_ttr.cuh"

namespace odp {

struct MdpParams {
    float step;      // HOLONOMIC: dt * speed (float32 product, A36)
    float vbar, wbar, dt, slip;
    float p[3];      // outcome probabilities (float32)
    float gamma;
};

// Index shift of the nearest node for a displacement of q cells: ties toward the larger index
// (nearest_index, "round half up", S:65 / S:81).  q - floor(q) is exact in float32.
__device__ __forceinline__ int nearest_shift(float q) {
    const float fl = floorf(q);
    return (int)fl + (__fsub_rn(q, fl) >= 0.5f ? 1 : 0);
}

// Displacement Delta(s, a, k) in float32 with every product and sum rounded separately (no FMA
// contraction: the snapped node is an integer decided by float arithmetic, A36).
template <int NDIM>
struct MHolonomic {
    static constexpr int NA = 2 * NDIM + 1, K = 1;
    static constexpr int NEED_TRIG = 0;
    __device__ static void delta(const MdpParams &m, const Pt &, int a, int, float *dl) {
#pragma unroll
        for (int d = 0; d < NDIM; ++d) dl[d] = 0.f;
        if (a > 0) {
            const int d = (a - 1) >> 1;
#pragma unroll
            for (int e = 0; e < NDIM; ++e)
                if (e == d) dl[e] = ((a - 1) & 1) == 0 ? m.step : -m.step;
        }
    }
};

struct MDubins3D {
    static constexpr int NA = 6, K = 3;
    static constexpr int NEED_TRIG = 1 << 2;
    __device__ static void delta(const MdpParams &m, const Pt &q, int a, int k, float *dl) {
        const float v = a < 3 ? __fmul_rn(0.5f, m.vbar) : m.vbar;
        const float w = __fmul_rn((float)(a % 3 - 1), m.wbar);
        const float sig = k == 0 ? 0.f : (k == 1 ? m.slip : -m.slip);
        const float c = q.c[2], s = q.s[2];
        const float dtv = __fmul_rn(m.dt, v);
        dl[0] = __fsub_rn(__fmul_rn(dtv, c), __fmul_rn(sig, s));
        dl[1] = __fadd_rn(__fmul_rn(dtv, s), __fmul_rn(sig, c));
        dl[2] = __fmul_rn(m.dt, w);
    }
};

template <class M, int NDIM>
__global__ void __launch_bounds__(256) k_vi_march(GridDev g, MdpParams mp, const float *__restrict__ R,
                                                  const float *__restrict__ src, float *__restrict__ dst,
                                                  TtrState *st, int par, int seg_len) {
    if (st->done) return;
    constexpr int NS = M::NA * M::K;
    const int ncol = (int)g.stride[0];
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    const int N0 = g.N[0];
    const int a0 = blockIdx.y * seg_len, a1 = min(N0, a0 + seg_len);
    float cmax = 0.f;
    if (c < ncol) {
        int idx[NDIM];
        {
            int rem = c;
#pragma unroll
            for (int d = NDIM - 1; d >= 1; --d) {
                const int qd = rem / g.N[d];
                idx[d] = rem - qd * g.N[d];
                rem = qd;
            }
            idx[0] = 0;
        }
        Pt q;
#pragma unroll
        for (int d = 1; d < NDIM; ++d)
            if ((M::NEED_TRIG >> d) & 1) {
                q.c[d] = __ldg(g.tab + g.tab_off[d] + g.Ng[d] + idx[d]);
                q.s[d] = __ldg(g.tab + g.tab_off[d] + 2 * g.Ng[d] + idx[d]);
            }
        // per (action, outcome): in-plane offset and axis-0 shift of the nearest-node successor (A36)
        int off[NS], sh0[NS];
#pragma unroll
        for (int a = 0; a < M::NA; ++a)
#pragma unroll
            for (int k = 0; k < M::K; ++k) {
                float dl[NDIM];
                M::delta(mp, q, a, k, dl);
                int o = 0;
#pragma unroll
                for (int d = 1; d < NDIM; ++d) {
                    int j = idx[d] + nearest_shift(__fmul_rn(dl[d], g.inv_dx[d]));
                    if (g.per[d]) { j %= g.N[d]; if (j < 0) j += g.N[d]; }
                    else j = max(0, min(g.N[d] - 1, j));
                    o += (j - idx[d]) * (int)g.stride[d];
                }
                off[a * M::K + k] = o;
                sh0[a * M::K + k] = nearest_shift(__fmul_rn(dl[0], g.inv_dx[0]));
            }
        const bool per0 = g.per[0] != 0;
        const long long s0 = ncol;
        const float *col = src + c;
        for (int i0 = a0; i0 < a1; ++i0) {
            const long long i = i0 * s0 + c;
            const float r = __ldg(R + i);
            float best = -__int_as_float(0x7f800000);
#pragma unroll
            for (int a = 0; a < M::NA; ++a) {
                float ev = 0.f;
#pragma unroll
                for (int k = 0; k < M::K; ++k) {
                    int j0 = i0 + sh0[a * M::K + k];
                    if (per0) { j0 %= N0; if (j0 < 0) j0 += N0; }
                    else j0 = max(0, min(N0 - 1, j0));
                    const float v = col[j0 * s0 + off[a * M::K + k]];
                    ev = fmaf(mp.p[k], v, ev);
                }
                best = fmaxf(best, fmaf(mp.gamma, ev, r));   // l.6-7 (A37)
            }
            const float old = col[i0 * s0];
            dst[i] = best;
            cmax = fmaxf(cmax, fabsf(best - old));           // l.8
        }
    }
    ttr_reduce_change(cmax, st, par);
    ttr_last_cta_control(st, par);
}

typedef void (*vi_march_fn)(GridDev, MdpParams, const float *, const float *, float *, TtrState *, int, int);

static vi_march_fn vi_select(int model, int n) {
    if (model == 1) return k_vi_march<MDubins3D, 3>;
    switch (n) {
    case 1: return k_vi_march<MHolonomic<1>, 1>;
    case 2: return k_vi_march<MHolonomic<2>, 2>;
    case 3: return k_vi_march<MHolonomic<3>, 3>;
    case 4: return k_vi_march<MHolonomic<4>, 4>;
    case 5: return k_vi_march<MHolonomic<5>, 5>;
    default: return k_vi_march<MHolonomic<6>, 6>;
    }
}

}  // namespace odp
