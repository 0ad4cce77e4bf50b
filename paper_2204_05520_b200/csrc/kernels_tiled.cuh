// kernels_tiled.cuh -- the "tiled" kernel family of the B200 HJ level-set step.
//
// Unit of work: one inner TILE-PLANE = the M = N[n-2] * N[n-1] contiguous floats of the two
// innermost axes at a fixed outer index (i_0 .. i_{n-3}) -- the paper's "highest dimension as the
// most inner loop" memory order (§4.1) turned into a contiguous 2D tile.  Every stencil
// neighbour of a node along an OUTER axis d lies at the same in-plane offset of another
// tile-plane, so a CTA stages the centre tile-plane plus the 2R neighbour tile-planes of each outer
// axis in shared memory with 1-D TMA bulk copies (cp.async.bulk ... mbarrier::complete_tx), then
// every thread reads its 4 consecutive nodes with 128-bit LDS.  In-plane neighbours (axes n-2,
// n-1) come from the centre tile; ghost values (reading A12) and periodic wraps are formed in
// registers.  Persistent CTAs walk the tile-planes in memory order; several CTAs per SM overlap
// one CTA's TMA wait with another's arithmetic.
//
//   k_tiled<PASS2=false>  pass 1: per-axis min/max of D-/D+ (Alg. 2 l.157-158), max|W|, NaN
//   k_tiled<PASS2=true>   pass 2: D+-, p, H, alpha_i, L, Euler/RK stage, BRT min (l.153-169)
#pragma once

#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "kernels_generic.cuh"

namespace odp {

constexpr int TILED_VEC = 4;   // consecutive nodes per thread (one 128-bit shared load per slot)
#ifndef ODP_TILED_MINB
#define ODP_TILED_MINB 3           // CTAs per SM the register budget is sized for
#endif
#ifndef ODP_TILED_MAXSTAGES
#define ODP_TILED_MAXSTAGES 1      // TMA pipeline depth
#endif
#ifndef ODP_TILED_L2_BYTES
#define ODP_TILED_L2_BYTES 0       // L2 budget of the axis-0 reuse window (0 = plain memory order)
#endif

struct TiledArgs {
    int M;             // floats per tile-plane
    int NT;            // tile-planes in the local array
    int N2, N1;        // extents of axes n-2, n-1
    int per2, per1;    // periodic flags of axes n-2, n-1
    int stages;        // TMA pipeline depth (1 or 2)
    int stage_floats;  // floats per pipeline stage (nslots * M)
    // L2 blocking of the tile order: strips of B consecutive indices of outer axis 1, each swept
    // with axis 0 outermost, so axis-0 neighbours are re-read from L2 instead of HBM
    int S;             // tiles per (i0, i1) cell = prod_{2 <= o < n-2} N_o
    int B;             // strip width along axis 1 (B >= N_1 -> plain memory order)
    int blk_tiles;     // N_0 * B * S
};

// --- PTX helpers (mbarrier + 1-D TMA bulk copy) -------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n\t"
        "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity), "r"(0x989680u)   /* suspend-time hint: sleep (up to 10 ms) instead of spinning */
        : "memory");
}
__device__ __forceinline__ void tma_bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// Separable Hamiltonian accumulation: H = sum_d term(d, p_d) (all functors except the ball, whose
// H = ubar goal |p|_2 is accumulated as sum p_d^2 and finished with a square root).
template <class F> struct HamAcc;

template <class F>
__device__ __forceinline__ float ham_term(const F &f, int d, const Pt &q, float pd);

template <int NDIM>
__device__ __forceinline__ float ham_term(const FHoloBall<NDIM> &, int, const Pt &, float pd) { return pd * pd; }
template <int NDIM>
__device__ __forceinline__ float ham_term(const FHoloBox<NDIM> &f, int, const Pt &, float pd) { return f.kH * fabsf(pd); }
__device__ __forceinline__ float ham_term(const FDubins3D &f, int d, const Pt &q, float pd) {
    return d == 0 ? pd * (f.v * q.c[2]) : (d == 1 ? pd * (f.v * q.s[2]) : f.kw * fabsf(pd));
}
__device__ __forceinline__ float ham_term(const FCar4D &f, int d, const Pt &q, float pd) {
    if (d == 0) return fmaf(f.kdx, fabsf(pd), pd * (q.x[2] * q.c[3]));
    if (d == 1) return fmaf(f.kdy, fabsf(pd), pd * (q.x[2] * q.s[3]));
    return (d == 2 ? f.ka : f.kw) * fabsf(pd);
}
__device__ __forceinline__ float ham_term(const FCar5D &f, int d, const Pt &q, float pd) {
    if (d == 0) return pd * (q.x[3] * q.c[2]);
    if (d == 1) return pd * (q.x[3] * q.s[2]);
    if (d == 2) return pd * q.x[4];
    return (d == 3 ? f.ka : f.kal) * fabsf(pd);
}
__device__ __forceinline__ float ham_term(const FDoubleInt6D &f, int d, const Pt &q, float pd) {
    return (d & 1) == 0 ? pd * q.x[d + 1] : f.kv * fabsf(pd);
}
template <class F> __device__ __forceinline__ float ham_finish(const F &, float acc) { return acc; }
template <int NDIM> __device__ __forceinline__ float ham_finish(const FHoloBall<NDIM> &f, float acc) {
    return f.kH * sqrtf(acc);
}

// Unscaled one-sided differences u = h D-, w = h D+ from the 2R+1 window (§3.4.4): the 1/h scale
// is folded into the consumers (pass 1 scales its min/max once at the end -- 1/h > 0 is monotone --
// and pass 2 folds it into the costate and dissipation factors).
template <int R>
__device__ __forceinline__ void deriv_u(const float *v, float &u, float &w) {
    if constexpr (R == 1) {
        u = v[1] - v[0];
        w = v[2] - v[1];
    } else {
        const float d2m = fmaf(-2.f, v[1], v[0] + v[2]);   // delta^2 at i-1
        const float d20 = fmaf(-2.f, v[2], v[1] + v[3]);   // delta^2 at i
        const float d2p = fmaf(-2.f, v[3], v[2] + v[4]);   // delta^2 at i+1
        u = fmaf(0.5f, eno_pick(d2m, d20), v[2] - v[1]);   // A13
        w = fmaf(-0.5f, eno_pick(d20, d2p), v[3] - v[2]);
    }
}

// Per-axis contribution of one node: pass 1 folds h D-/h D+ into the running range, pass 2
// accumulates the Hamiltonian term at p = (D- + D+)/2 (A3) and the dissipation
// alpha (D+ - D-)/2 (A2); hih = 1/(2h).
template <class F, int R, bool PASS2>
__device__ __forceinline__ void axis_update(const F &f, int d, const Pt &q, const float *v, float hih, float &acc,
                                            float &dis, float &mn, float &mx) {
    float u, w;
    deriv_u<R>(v, u, w);
    if constexpr (PASS2) {
        acc += ham_term(f, d, q, (u + w) * hih);
        dis = fmaf(f.alpha(d, q) * hih, w - u, dis);
    } else {
        mn = fminf(mn, fminf(u, w));
        mx = fmaxf(mx, fmaxf(u, w));
    }
}

// work index u (the order CTAs sweep) -> tile-plane index t (memory order)
template <int NO>
__device__ __forceinline__ int tile_of(const TiledArgs &a, const GridDev &g, int u) {
    if constexpr (NO >= 2) {
        const int N1o = g.N[1];
        if (a.B < N1o) {
            int blk = u / a.blk_tiles;
            const int nblk = (N1o + a.B - 1) / a.B;
            if (blk > nblk - 1) blk = nblk - 1;
            const int w = min(a.B, N1o - blk * a.B);
            const int rem = u - blk * a.blk_tiles;
            const int ws = w * a.S;
            const int i0 = rem / ws;
            const int rem2 = rem - i0 * ws;
            const int i1 = blk * a.B + rem2 / a.S;
            const int r = rem2 - (rem2 / a.S) * a.S;
            return (i0 * N1o + i1) * a.S + r;
        }
    }
    return u;
}

template <int NO>
__device__ __forceinline__ void outer_index(const GridDev &g, int t, int *oid, int *oN) {
    int r = t;
#pragma unroll
    for (int o = NO - 1; o >= 1; --o) {
        const int q = r / g.N[o];
        oid[o] = r - q * g.N[o];
        oN[o] = g.N[o];
        r = q;
    }
    oid[0] = g.g0 + r;    // axis 0: global index (slabs)
    oN[0] = g.Ng0;
}

// Per-stage tile metadata, written by the issuing thread before its mbarrier arrive (release) and
// read by every thread after the wait (acquire): the outer multi-index is computed once per tile.
struct TileInfo {
    int t;
    int oid[MAXD];
    int ghost;   // any outer axis of this tile-plane within R of a non-periodic face
};

// Thread 0: stage tile-plane t (centre + the in-domain outer neighbours) into `dst` with 1-D TMA
// bulk copies that all complete on `bar`.
template <int NO, int R>
__device__ __forceinline__ void issue_tile(const GridDev &g, const float *W, int t, int M, float *dst, uint64_t *bar,
                                           TileInfo *info) {
    int oid[NO], oN[NO];
    outer_index<NO>(g, t, oid, oN);
    int gh = 0;
#pragma unroll
    for (int o = 0; o < NO; ++o) {
        info->oid[o] = oid[o];
        gh |= !g.per[o] && (oid[o] < R || oid[o] > oN[o] - 1 - R);
    }
    info->t = t;
    info->ghost = gh;
#ifdef ODP_TILED_DEBUG_NOLOAD
    mbar_expect_tx(bar, 0);
    return;
#endif
    const long long base = (long long)t * M;
    const uint32_t tb = (uint32_t)M * 4u;
    uint32_t bytes = tb;
    tma_bulk_g2s(dst, W + base, tb, bar);
#pragma unroll
    for (int o = 0; o < NO; ++o) {
#pragma unroll
        for (int k = -R; k <= R; ++k) {
            if (k == 0) continue;
            const int s = 1 + o * 2 * R + (k < 0 ? k + R : k + R - 1);
            int j = oid[o] + k;
            bool ok = true;
            if (j < 0 || j >= oN[o]) {
                if (g.per[o]) j = j < 0 ? j + oN[o] : j - oN[o];
                else ok = false;
            }
            if (ok) {
                tma_bulk_g2s(dst + (size_t)s * M, W + base + (long long)(j - oid[o]) * g.stride[o], tb, bar);
                bytes += tb;
            }
        }
    }
    mbar_expect_tx(bar, bytes);
}


// Shared-memory layout of one CTA (floats):
//   stage k (k < stages): [k*SF, (k+1)*SF), SF = nslots*M: TMA slots, slot 0 = centre tile-plane,
//       slot 1 + o*2R + j = outer axis o, offset -R..-1, 1..R (ghost slots materialised in place)
//   pad: the centre tile-plane padded by R ghost cells on each side of the two in-plane axes
//       (PW = N1 + 2R columns, N2 + 2R rows) -- every stencil read of the compute loop is branch-free
template <class F, int NDIM, int R, bool PASS2>
__global__ void __launch_bounds__(256, ODP_TILED_MINB) k_tiled(TiledArgs a, GridDev g, const float *__restrict__ W, const float *Vn,
                                                  const float *__restrict__ T, float *out, float *partials,
                                                  const DevState *st, FParams fp, int kind, int brt) {
    if (!st->active) return;
    constexpr int NO = NDIM - 2;                   // outer axes
    extern __shared__ __align__(128) float smem[];
    __shared__ uint64_t bar[2];
    __shared__ TileInfo tinfo[2];

    float mn[NDIM], mx[NDIM], mabs = 0.f;
    int nan = 0;
#pragma unroll
    for (int d = 0; d < NDIM; ++d) { mn[d] = __int_as_float(0x7f800000); mx[d] = -__int_as_float(0x7f800000); }

    F f;
    float dt = 0.f;
    if constexpr (PASS2) {
        f.init(fp, st->minD, st->maxD);
        dt = st->dt_f;
    }
    float hih[NDIM];
#pragma unroll
    for (int d = 0; d < NDIM; ++d) hih[d] = 0.5f * g.inv_dx[d];
    const int M = a.M, N1 = a.N1, N2 = a.N2;
    const int PW = N1 + 2 * R;
    float *pad = smem + (size_t)a.stages * a.stage_floats;
    const int G = gridDim.x;

    // ---- tile-invariant table of the in-plane ghost cells of the padded copy (A12; rows and
    //      columns, no corners): int4 {target, edge/source, inner, mode | q << 2}, mode 1 ghost, 2 copy
    int4 *gtab = reinterpret_cast<int4 *>(pad + (((size_t)(N2 + 2 * R) * PW + 3) & ~(size_t)3));   // 16-B aligned
    const int ncol = 2 * R * N2, nghost = 2 * R * (N1 + N2);
    for (int i = threadIdx.x; i < nghost; i += blockDim.x) {
        int T = 0, E = 0, I = 0, mode = 0, qd = 0;
        if (i < ncol) {                       // ghost columns of row r
            const int r = i / (2 * R), kk = i - r * 2 * R;
            const int prow = (r + R) * PW;
            if (kk < R) {
                qd = R - kk;
                T = prow + R - qd;
                if (a.per1) { mode = 2; E = prow + R + N1 - qd; }
                else { mode = 1; E = prow + R; I = prow + R + 1; }
            } else {
                qd = kk - R + 1;
                T = prow + R + N1 - 1 + qd;
                if (a.per1) { mode = 2; E = prow + R + qd - 1; }
                else { mode = 1; E = prow + R + N1 - 1; I = prow + R + N1 - 2; }
            }
        } else {                              // ghost rows of column c
            const int i2 = i - ncol;
            const int c = i2 / (2 * R), kk = i2 - c * 2 * R;
            const int pc = c + R;
            if (kk < R) {
                qd = R - kk;
                T = (R - qd) * PW + pc;
                if (a.per2) { mode = 2; E = (R + N2 - qd) * PW + pc; }
                else { mode = 1; E = R * PW + pc; I = (R + 1) * PW + pc; }
            } else {
                qd = kk - R + 1;
                T = (R + N2 - 1 + qd) * PW + pc;
                if (a.per2) { mode = 2; E = (R + qd - 1) * PW + pc; }
                else { mode = 1; E = (R + N2 - 1) * PW + pc; I = (R + N2 - 2) * PW + pc; }
            }
        }
        gtab[i] = make_int4(T, E, I, mode | (qd << 2));
    }

    // in-plane position of this thread's first quad (the same in every tile-plane)
    const int e0 = threadIdx.x * TILED_VEC;
    const int r0 = e0 / N1, c0 = e0 - r0 * N1;
    auto quad_rc = [&](int e, int &r, int &c) {
        if (e == e0) { r = r0; c = c0; }
        else { r = e / N1; c = e - r * N1; }
    };

    if (threadIdx.x == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        if ((int)blockIdx.x < a.NT) issue_tile<NO, R>(g, W, tile_of<NO>(a, g, blockIdx.x), M, smem, &bar[0], &tinfo[0]);
    }
    __syncthreads();

    uint32_t phase0 = 0, phase1 = 0;
    int it = 0;
    for (int u = blockIdx.x; u < a.NT; u += G, ++it) {
        const int sidx = a.stages == 2 ? (it & 1) : 0;
        float *stg = smem + (size_t)sidx * a.stage_floats;
        if (a.stages == 2 && threadIdx.x == 0 && u + G < a.NT)          // prefetch the next tile-plane
            issue_tile<NO, R>(g, W, tile_of<NO>(a, g, u + G), M, smem + (size_t)(sidx ^ 1) * a.stage_floats,
                              &bar[sidx ^ 1], &tinfo[sidx ^ 1]);
        if (sidx == 0) { mbar_wait(&bar[0], phase0); phase0 ^= 1u; }
        else { mbar_wait(&bar[1], phase1); phase1 ^= 1u; }
        const TileInfo &ti = tinfo[sidx];
        const long long base = (long long)ti.t * M;
        const bool any_ghost = ti.ghost;
        int oid[NO], oN[NO];
#pragma unroll
        for (int o = 0; o < NO; ++o) { oid[o] = ti.oid[o]; oN[o] = o == 0 ? g.Ng0 : g.N[o]; }
        Pt q;   // tile-uniform coordinates of the outer axes
        if constexpr (PASS2) {
#pragma unroll
            for (int o = 0; o < NO; ++o) load_axis<F>(g, q, o, oid[o]);
        }

        // ---- fill 1: padded in-plane copy of the centre; materialise outer ghost slots (A12) ----
        for (int e = e0; e < M; e += blockDim.x * TILED_VEC) {
            int r, c;
            quad_rc(e, r, c);
            const int P = e + 2 * R * r + R * PW + R;
            const float4 c4 = *reinterpret_cast<const float4 *>(stg + e);
            pad[P] = c4.x;
            pad[P + 1 + (c + 1 >= N1 ? 2 * R : 0)] = c4.y;
            pad[P + 2 + (c + 2 >= N1 ? 2 * R : 0)] = c4.z;
            pad[P + 3 + (c + 3 >= N1 ? 2 * R : 0)] = c4.w;
            if (any_ghost) {
#pragma unroll
                for (int o = 0; o < NO; ++o) {
                    if (g.per[o]) continue;
                    const int id = oid[o], Nd = oN[o];
                    if (id >= R && id <= Nd - 1 - R) continue;
                    auto slot = [&](int kk) -> float * {
                        return kk == 0 ? stg : stg + (size_t)(1 + o * 2 * R + (kk < 0 ? kk + R : kk + R - 1)) * M;
                    };
#pragma unroll
                    for (int kk = -R; kk <= R; ++kk) {
                        if (kk == 0) continue;
                        const int j = id + kk;
                        float qd;
                        const float *E, *I;
                        if (j < 0) { E = slot(-id); I = slot(1 - id); qd = (float)(-j); }
                        else if (j >= Nd) { E = slot(Nd - 1 - id); I = slot(Nd - 2 - id); qd = (float)(j - (Nd - 1)); }
                        else continue;
                        const float4 e4 = *reinterpret_cast<const float4 *>(E + e);
                        const float4 i4 = *reinterpret_cast<const float4 *>(I + e);
                        float4 gv;
                        gv.x = ghost(e4.x, i4.x, qd); gv.y = ghost(e4.y, i4.y, qd);
                        gv.z = ghost(e4.z, i4.z, qd); gv.w = ghost(e4.w, i4.w, qd);
                        *reinterpret_cast<float4 *>(slot(kk) + e) = gv;
                    }
                }
            }
        }
        __syncthreads();
        // ---- fill 2: in-plane ghost cells ----
        for (int i = threadIdx.x; i < nghost; i += blockDim.x) {
            const int4 d = gtab[i];
            const float e = pad[d.y];
            pad[d.x] = (d.w & 3) == 2 ? e : ghost(e, pad[d.z], (float)(d.w >> 2));
        }
        __syncthreads();

        // ---- compute: branch-free stencils for 4 consecutive nodes per thread ----
#ifdef ODP_TILED_DEBUG_NOCOMPUTE
        if (base < 0)
#endif
        for (int e = e0; e < M; e += blockDim.x * TILED_VEC) {
            const float4 c4 = *reinterpret_cast<const float4 *>(stg + e);
            const float cv[4] = {c4.x, c4.y, c4.z, c4.w};
            float acc[TILED_VEC], dis[TILED_VEC];
            int P0[TILED_VEC];
            Pt qv[TILED_VEC];
            int qr, qc;
            quad_rc(e, qr, qc);
            const int qP = e + 2 * R * qr + R * PW + R;
#pragma unroll
            for (int j = 0; j < TILED_VEC; ++j) {
                acc[j] = 0.f; dis[j] = 0.f;
                const bool wrap = qc + j >= N1;
                P0[j] = qP + j + (wrap ? 2 * R : 0);
                qv[j] = q;
                if constexpr (PASS2) {
                    load_axis<F>(g, qv[j], NDIM - 2, wrap ? qr + 1 : qr);
                    load_axis<F>(g, qv[j], NDIM - 1, wrap ? qc + j - N1 : qc + j);
                }
            }
            const float *sp = stg + e;
#pragma unroll
            for (int o = 0; o < NO; ++o) {
                float wv[2 * R + 1][TILED_VEC];
#pragma unroll
                for (int kk = -R; kk <= R; ++kk) {
                    if (kk == 0) {
#pragma unroll
                        for (int j = 0; j < TILED_VEC; ++j) wv[R][j] = cv[j];
                        continue;
                    }
                    const int s = 1 + o * 2 * R + (kk < 0 ? kk + R : kk + R - 1);
                    const float4 x = *reinterpret_cast<const float4 *>(sp + (size_t)s * M);
                    wv[kk + R][0] = x.x; wv[kk + R][1] = x.y; wv[kk + R][2] = x.z; wv[kk + R][3] = x.w;
                }
#pragma unroll
                for (int j = 0; j < TILED_VEC; ++j) {
                    float v[2 * R + 1];
#pragma unroll
                    for (int kk = 0; kk <= 2 * R; ++kk) v[kk] = wv[kk][j];
                    axis_update<F, R, PASS2>(f, o, qv[j], v, hih[o], acc[j], dis[j], mn[o], mx[o]);
                }
            }
#pragma unroll
            for (int j = 0; j < TILED_VEC; ++j) {
                float v[2 * R + 1];
#pragma unroll
                for (int kk = -R; kk <= R; ++kk) v[kk + R] = kk == 0 ? cv[j] : pad[P0[j] + kk * PW];
                axis_update<F, R, PASS2>(f, NDIM - 2, qv[j], v, hih[NDIM - 2], acc[j], dis[j], mn[NDIM - 2], mx[NDIM - 2]);
#pragma unroll
                for (int kk = -R; kk <= R; ++kk) v[kk + R] = kk == 0 ? cv[j] : pad[P0[j] + kk];
                axis_update<F, R, PASS2>(f, NDIM - 1, qv[j], v, hih[NDIM - 1], acc[j], dis[j], mn[NDIM - 1], mx[NDIM - 1]);
                if constexpr (PASS2) {
                    acc[j] = ham_finish(f, acc[j]) + dis[j];
                } else {
                    nan |= (cv[j] != cv[j]);
                    mabs = fmaxf(mabs, fabsf(cv[j]));
                }
            }
            if constexpr (PASS2) {
                const long long gi = base + e;
                float4 o4;
                o4.x = stage_update(kind, brt, cv[0], acc[0], dt, Vn, T, gi + 0);
                o4.y = stage_update(kind, brt, cv[1], acc[1], dt, Vn, T, gi + 1);
                o4.z = stage_update(kind, brt, cv[2], acc[2], dt, Vn, T, gi + 2);
                o4.w = stage_update(kind, brt, cv[3], acc[3], dt, Vn, T, gi + 3);
                *reinterpret_cast<float4 *>(out + gi) = o4;
            }
        }
        fence_proxy_async();   // order this tile's generic smem accesses before later TMA writes
        __syncthreads();       // the stage and pad are free again
        if (a.stages == 1 && threadIdx.x == 0 && u + G < a.NT)
            issue_tile<NO, R>(g, W, tile_of<NO>(a, g, u + G), M, smem, &bar[0], &tinfo[0]);
    }
    if constexpr (!PASS2) {
#pragma unroll
        for (int d = 0; d < NDIM; ++d) { mn[d] *= g.inv_dx[d]; mx[d] *= g.inv_dx[d]; }   // h D -> D
        block_reduce_range<NDIM>(mn, mx, mabs, nan, partials);
    }
}

// ------------------------------------------------------------------------------------------------
// host side
// ------------------------------------------------------------------------------------------------
typedef void (*tiled_fn)(TiledArgs, GridDev, const float *, const float *, const float *, float *, float *,
                         const DevState *, FParams, int, int);

struct TiledFns {
    tiled_fn pass1 = nullptr, pass2 = nullptr;
};

struct TiledPlan {
    TiledArgs a;
    int block = 0, grid = 0;
    size_t smem = 0;
};

template <class F, int NDIM, int R>
TiledFns tiled_fns() {
    TiledFns t;
    if constexpr (NDIM >= 3) {
        t.pass1 = k_tiled<F, NDIM, R, false>;
        t.pass2 = k_tiled<F, NDIM, R, true>;
    }
    return t;
}

// Decide whether the tiled family covers this grid and size its launch.  l2_bytes: the L2 budget
// for the axis-0 reuse window of the tile order.
inline bool tiled_plan(const GridDev &g, int R, int nsm, TiledPlan *p, double l2_bytes = ODP_TILED_L2_BYTES) {
    (void)nsm;
    if (g.n < 3) return false;
    const long long M = (long long)g.N[g.n - 2] * g.N[g.n - 1];
    if (M % TILED_VEC) return false;                       // 16-B aligned tile-planes and float4 lanes
    if (g.N[g.n - 2] < R + 1 || g.N[g.n - 1] < R + 1) return false;
    if (g.P / M > (1LL << 31) - 1) return false;
    const int nslots = 1 + 2 * R * (g.n - 2);
    const size_t stage = (size_t)nslots * M * sizeof(float);
    const size_t padb = (size_t)(g.N[g.n - 2] + 2 * R) * (g.N[g.n - 1] + 2 * R) * sizeof(float) +
                        (size_t)2 * R * (g.N[g.n - 2] + g.N[g.n - 1]) * 16 + 16;   // + ghost table (int4, 16-B aligned)
    const size_t cap = 220 * 1024;
    int stages = ODP_TILED_MAXSTAGES;
    if (2 * stage + padb > cap) stages = 1;
    if (stage + padb > cap) return false;
    TiledArgs &a = p->a;
    a.M = (int)M;
    a.NT = (int)(g.P / M);
    a.N2 = g.N[g.n - 2];
    a.N1 = g.N[g.n - 1];
    a.per2 = g.per[g.n - 2];
    a.per1 = g.per[g.n - 1];
    a.stages = stages;
    a.stage_floats = (int)(nslots * M);
    // tile order: strips along outer axis 1 sized so 2R strips of axis-0 planes stay in L2
    a.S = 1;
    for (int o = 2; o < g.n - 2; ++o) a.S *= g.N[o];
    a.B = g.n - 2 >= 2 ? g.N[1] : 1;
    if (const char *env = getenv("ODP_TILED_L2_BYTES")) l2_bytes = atof(env);   // tuning override
    if (g.n - 2 >= 2 && l2_bytes > 0) {
        const double per_b = 2.0 * R * a.S * (double)M * 4.0;     // bytes of the axis-0 window per unit B
        int B = (int)(l2_bytes / per_b);
        if (B < 1) B = 1;
        if (B < g.N[1]) a.B = B;
    }
    a.blk_tiles = g.N[0] * a.B * a.S;
    const int quads = (int)(M / TILED_VEC);
    p->block = quads >= 256 ? 256 : ((quads + 31) / 32) * 32;

    p->smem = (size_t)stages * stage + padb;
    p->grid = 0;
    return true;
}

inline int tiled_prepare(const TiledFns &t, TiledPlan &p, int nsm) {
    for (tiled_fn fn : {t.pass1, t.pass2}) {
        if (cudaFuncSetAttribute((const void *)fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p.smem) != cudaSuccess)
            return 1;
    }
    int occ1 = 0, occ2 = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ1, (const void *)t.pass1, p.block, p.smem) != cudaSuccess) return 1;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ2, (const void *)t.pass2, p.block, p.smem) != cudaSuccess) return 1;
    const int occ = std::max(1, std::min(occ1, occ2));
    p.grid = std::min(p.a.NT, nsm * occ);
    return 0;
}

inline void tiled_pass1(const TiledFns &t, const TiledPlan &p, const GridDev &g, const float *W, float *partials,
                        const DevState *st, cudaStream_t s) {
    FParams fp;
    memset(&fp, 0, sizeof fp);
    t.pass1<<<p.grid, p.block, p.smem, s>>>(p.a, g, W, nullptr, nullptr, nullptr, partials, st, fp, 0, 0);
}

inline void tiled_pass2(const TiledFns &t, const TiledPlan &p, const GridDev &g, const float *W, const float *Vn,
                        const float *T, float *out, const DevState *st, const FParams &fp, int kind, int brt,
                        cudaStream_t s) {
    t.pass2<<<p.grid, p.block, p.smem, s>>>(p.a, g, W, Vn, T, out, nullptr, st, fp, kind, brt);
}

}  // namespace odp
