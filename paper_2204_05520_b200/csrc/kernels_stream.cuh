// kernels_stream.cuh -- the "stream" kernel family (default) of the B200 HJ level-set step.
//
// Layout recap: row-major float32, axis 0 outermost.  The two innermost axes form an
// in-plane TILE of M = N[n-2] * N[n-1] contiguous floats; the remaining "outer" axes index tiles.
//
// Each CTA owns a COLUMN of tiles: a fixed index on every outer axis but the innermost one (the
// MARCHING axis, axis n-3, stride M), and walks a segment of the marching axis.  Per thread:
//   * VEC consecutive nodes of one in-plane row ("quad");
//   * the 2R+1 values of its quad along the marching axis live in a register shift window, so
//     each step loads ONE new tile quad for that axis (one step ahead, software prefetch);
//   * the 2R neighbour quads along every other outer axis are loaded straight from L2 with
//     vector loads (no reuse to exploit on chip: those tiles are 3.6 KB .. 100 MB apart);
//   * the in-plane neighbours come from a shared-memory copy of the centre tile, padded with the
//     in-plane ghost cells (A12) and laid out with 16-B aligned rows so every read is a
//     conflict-free 64/128-bit LDS; double-buffered so a step needs two barriers.
// Ghost values along outer axes are formed in registers (the face condition is CTA-uniform).
//
//   pass 1 (PASS2=false): min/max of D-/D+ per axis (Alg. 2 l.157-158), max|W|, NaN flag
//   pass 2 (PASS2=true):  p, H, alpha_i, dissipation, Euler/RK stage, BRT min (l.153-169)
#pragma once

#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "kernels_tiled.cuh"

namespace odp {

#ifndef ODP_STREAM_MINB2
#define ODP_STREAM_MINB2 2      // CTAs/SM the register budget of the VEC=2 kernels is sized for
#endif
#ifndef ODP_STREAM_MINB4
#define ODP_STREAM_MINB4 1      // ... and of the VEC=4 kernels (64 registers would spill)
#endif
constexpr int STREAM_MAXT = 512;   // threads per CTA (one quad per thread)

template <int V> struct VecT;
template <> struct VecT<2> { using type = float2; };
template <> struct VecT<4> { using type = float4; };

template <int V>
__device__ __forceinline__ void ld_vec(const float *p, float *v) {
    if constexpr (V == 4) {
        const float4 x = __ldg(reinterpret_cast<const float4 *>(p));
        v[0] = x.x; v[1] = x.y; v[2] = x.z; v[3] = x.w;
    } else {
        const float2 x = __ldg(reinterpret_cast<const float2 *>(p));
        v[0] = x.x; v[1] = x.y;
    }
}

// load VEC consecutive floats at p: one vector load when aligned and complete, else per element
template <int V>
__device__ __forceinline__ void load_quad(const float *__restrict__ p, bool vec_ok, int nvalid, float *v) {
    if (vec_ok) {
        ld_vec<V>(p, v);
    } else {
#pragma unroll
        for (int j = 0; j < V; ++j) v[j] = j < nvalid ? __ldg(p + j) : 0.f;
    }
}

template <int V>
__device__ __forceinline__ void lds_vec(const float *p, float *v) {
    if constexpr (V == 4) {
        const float4 x = *reinterpret_cast<const float4 *>(p);
        v[0] = x.x; v[1] = x.y; v[2] = x.z; v[3] = x.w;
    } else {
        const float2 x = *reinterpret_cast<const float2 *>(p);
        v[0] = x.x; v[1] = x.y;
    }
}

template <int V>
__device__ __forceinline__ void sts_vec(float *p, const float *v) {
    if constexpr (V == 4) *reinterpret_cast<float4 *>(p) = make_float4(v[0], v[1], v[2], v[3]);
    else *reinterpret_cast<float2 *>(p) = make_float2(v[0], v[1]);
}

struct StreamArgs {
    int M, N2, N1;      // tile size and in-plane extents
    int per2, per1;
    int QR;             // quads per row = ceil(N1 / VEC)
    int nquads;         // N2 * QR
    int PW;             // padded row width (floats, multiple of 4)
    int OFF;            // padded column of in-plane column 0 (multiple of 4, >= R)
    int pad_floats;     // floats per pad buffer (multiple of 4)
    int K;              // marching segment length
    int nseg;           // segments per column
    int ncols;          // columns = prod of the outer extents except the marching axis
    int units;          // ncols * nseg
};

template <class F, int NDIM, int R, int VEC, bool PASS2>
__global__ void __launch_bounds__(STREAM_MAXT, VEC == 2 ? ODP_STREAM_MINB2 : ODP_STREAM_MINB4) k_stream(StreamArgs a, GridDev g, const float *__restrict__ W,
                                                                  const float *Vn, const float *__restrict__ T, float *out,
                                                                  float *partials, const DevState *st, FParams fp,
                                                                  int kind, int brt) {
    if (!st->active) return;
    constexpr int NO = NDIM - 2;          // outer axes; the marching axis is NO-1
    constexpr int MA = NO - 1;
    constexpr int NW = 2 * R + 1;
    extern __shared__ __align__(128) float smem[];

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

    const int M = a.M, N1 = a.N1, N2 = a.N2, PW = a.PW;
    // ---- tile-invariant per-thread geometry ----
    const int qid = threadIdx.x;
    const bool active_q = qid < a.nquads;
    const int qrow = active_q ? qid / a.QR : 0;
    const int qc0 = active_q ? (qid - qrow * a.QR) * VEC : 0;
    const int lin = qrow * N1 + qc0;                           // linear in-plane offset of node 0
    // N1 % VEC == 0 (plan): quads never straddle rows and every quad load/store is a vector access
    const int padc = (qrow + R) * PW + a.OFF + qc0;            // padded index of node 0
    // in-plane ghost-cell table (rows and columns, no corners), int4 {target, edge, inner, mode|q<<2}
    float *pad0 = smem;
    float *pad1 = smem + a.pad_floats;
    int4 *gtab = reinterpret_cast<int4 *>(smem + 2 * a.pad_floats);
    const int ncolg = 2 * R * N2, nghost = 2 * R * (N1 + N2);
    for (int i = threadIdx.x; i < nghost; i += blockDim.x) {
        int Tg = 0, E = 0, I = 0, mode = 0, qd = 0;
        if (i < ncolg) {
            const int r = i / (2 * R), kk = i - r * 2 * R;
            const int prow = (r + R) * PW + a.OFF;
            if (kk < R) {
                qd = R - kk; Tg = prow - qd;
                if (a.per1) { mode = 2; E = prow + N1 - qd; } else { mode = 1; E = prow; I = prow + 1; }
            } else {
                qd = kk - R + 1; Tg = prow + N1 - 1 + qd;
                if (a.per1) { mode = 2; E = prow + qd - 1; } else { mode = 1; E = prow + N1 - 1; I = prow + N1 - 2; }
            }
        } else {
            const int i2 = i - ncolg;
            const int c = i2 / (2 * R), kk = i2 - c * 2 * R;
            const int pc = a.OFF + c;
            if (kk < R) {
                qd = R - kk; Tg = (R - qd) * PW + pc;
                if (a.per2) { mode = 2; E = (R + N2 - qd) * PW + pc; } else { mode = 1; E = R * PW + pc; I = (R + 1) * PW + pc; }
            } else {
                qd = kk - R + 1; Tg = (R + N2 - 1 + qd) * PW + pc;
                if (a.per2) { mode = 2; E = (R + qd - 1) * PW + pc; }
                else { mode = 1; E = (R + N2 - 1) * PW + pc; I = (R + N2 - 2) * PW + pc; }
            }
        }
        gtab[i] = make_int4(Tg, E, I, mode | (qd << 2));
    }
    // in-plane coordinates of the thread's nodes (pass 2)
    Pt qin[VEC];
    if constexpr (PASS2) {
#pragma unroll
        for (int j = 0; j < VEC; ++j) {
            load_axis<F>(g, qin[j], NDIM - 2, qrow);
            load_axis<F>(g, qin[j], NDIM - 1, qc0 + j);
        }
    }
    __syncthreads();

    const int Nm = MA == 0 ? g.Ng0 : g.N[MA];      // marching extent (global: face tests)
    const int mlo = MA == 0 ? g.g0 : 0;             // first marching index owned (slabs own part of axis 0)
    int step_parity = 0;
    for (int u = blockIdx.x; u < a.units; u += gridDim.x) {
        const int col = u / a.nseg, seg = u - col * a.nseg;
        // outer indices of the column (axes 0 .. MA-1) and the tile index of its marching start
        int oid[NO > 1 ? NO - 1 : 1], oN[NO > 1 ? NO - 1 : 1];
        {
            int r = col;
#pragma unroll
            for (int o = MA - 1; o >= 1; --o) { const int qv = r / g.N[o]; oid[o] = r - qv * g.N[o]; oN[o] = g.N[o]; r = qv; }
            if constexpr (MA >= 1) { oid[0] = g.g0 + r; oN[0] = g.Ng0; }
        }
        // element pointer of this thread's quad in the column's tile at local marching index 0
        const long long colbase = MA >= 1 ? (long long)col * g.N[MA] : 0;
        const float *cp = W + colbase * M + lin;
        const int m0 = mlo + seg * a.K, m1 = min(mlo + (MA == 0 ? g.N[0] : g.N[MA]), m0 + a.K);
        const bool mper = MA == 0 ? g.per[0] : g.per[MA];
        // local marching index of global index jg, clamped / wrapped into the domain (out-of-domain
        // window slots are overwritten by fix_ghosts)
        auto mloc = [&](int jg) -> int {
            int j = jg;
            if (j < 0 || j >= Nm) {
                if (mper) j = j < 0 ? j + Nm : j - Nm;
                else j = j < 0 ? 0 : Nm - 1;
            }
            return j - mlo;
        };
        // window of the marching axis: w[k] = values at marching index j + k - R
        float w[NW][VEC], pre[VEC];
#pragma unroll
        for (int k = 0; k < NW - 1; ++k) ld_vec<VEC>(cp + (long long)mloc(m0 + k - R) * M, w[k + 1]);
        ld_vec<VEC>(cp + (long long)mloc(m0 + R) * M, pre);
        // the other outer axes: face status and neighbour offsets (uniform over the CTA)
        bool oface[NO > 1 ? NO - 1 : 1];
        int noff[NO > 1 ? NO - 1 : 1][2 * R];
#pragma unroll
        for (int o = 0; o < MA; ++o) {
            oface[o] = !g.per[o] && (oid[o] < R || oid[o] > oN[o] - 1 - R);
#pragma unroll
            for (int k = -R; k <= R; ++k) {
                if (k == 0) continue;
                int j = oid[o] + k;
                if (j < 0 || j >= oN[o]) {
                    if (g.per[o]) j = j < 0 ? j + oN[o] : j - oN[o];
                    else j = oid[o];                        // placeholder; fixed by fix_ghosts
                }
                noff[o][k < 0 ? k + R : k + R - 1] = (int)((long long)(j - oid[o]) * g.stride[o]);
            }
        }
        Pt qcol;
        if constexpr (PASS2) {
#pragma unroll
            for (int o = 0; o < MA; ++o) load_axis<F>(g, qcol, o, oid[o]);
        }

        for (int jg = m0; jg < m1; ++jg) {
            // shift the window and take the prefetched quad; prefetch the next one
#pragma unroll
            for (int k = 0; k < NW - 1; ++k)
#pragma unroll
                for (int v = 0; v < VEC; ++v) w[k][v] = w[k + 1][v];
#pragma unroll
            for (int v = 0; v < VEC; ++v) w[NW - 1][v] = pre[v];
            if (jg + 1 < m1) ld_vec<VEC>(cp + (long long)mloc(jg + 1 + R) * M, pre);
            const float *cq = cp + (long long)(jg - mlo) * M;     // centre quad of this step
            const long long tb = colbase * M + (long long)(jg - mlo) * M;
            // neighbour quads along the other outer axes (issued before the barriers)
            float nb[NO > 1 ? NO - 1 : 1][2 * R][VEC];
#pragma unroll
            for (int o = 0; o < MA; ++o)
#pragma unroll
                for (int s2 = 0; s2 < 2 * R; ++s2) ld_vec<VEC>(cq + noff[o][s2], nb[o][s2]);
            // centre quad -> padded shared tile (double-buffered)
            float *pad = step_parity ? pad1 : pad0;
            step_parity ^= 1;
            if (active_q) sts_vec<VEC>(pad + padc, w[R]);
            __syncthreads();
            for (int i = threadIdx.x; i < nghost; i += blockDim.x) {
                const int4 d = gtab[i];
                const float e = pad[d.y];
                pad[d.x] = (d.w & 3) == 2 ? e : ghost(e, pad[d.z], (float)(d.w >> 2));
            }
            __syncthreads();
            if (!active_q) continue;

            Pt q = qcol;
            if constexpr (PASS2) load_axis<F>(g, q, MA, jg);
            float acc[VEC], dis[VEC];
#pragma unroll
            for (int v = 0; v < VEC; ++v) { acc[v] = 0.f; dis[v] = 0.f; }
            Pt qv[VEC];
#pragma unroll
            for (int v = 0; v < VEC; ++v) {
                qv[v] = q;
                if constexpr (PASS2) {
                    qv[v].x[NDIM - 2] = qin[v].x[NDIM - 2]; qv[v].c[NDIM - 2] = qin[v].c[NDIM - 2]; qv[v].s[NDIM - 2] = qin[v].s[NDIM - 2];
                    qv[v].x[NDIM - 1] = qin[v].x[NDIM - 1]; qv[v].c[NDIM - 1] = qin[v].c[NDIM - 1]; qv[v].s[NDIM - 1] = qin[v].s[NDIM - 1];
                }
            }
            // marching axis
            const bool mface = !mper && (jg < R || jg > Nm - 1 - R);
#pragma unroll
            for (int v = 0; v < VEC; ++v) {
                float x[NW];
#pragma unroll
                for (int k = 0; k < NW; ++k) x[k] = w[k][v];
                if (mface) fix_ghosts<R>(x, jg, Nm);
                axis_update<F, R, PASS2>(f, MA, qv[v], x, hih[MA], acc[v], dis[v], mn[MA], mx[MA]);
            }
            // other outer axes
#pragma unroll
            for (int o = 0; o < MA; ++o) {
#pragma unroll
                for (int v = 0; v < VEC; ++v) {
                    float x[NW];
#pragma unroll
                    for (int k = -R; k <= R; ++k) x[k + R] = k == 0 ? w[R][v] : nb[o][k < 0 ? k + R : k + R - 1][v];
                    if (oface[o]) fix_ghosts<R>(x, oid[o], oN[o]);
                    axis_update<F, R, PASS2>(f, o, qv[v], x, hih[o], acc[v], dis[v], mn[o], mx[o]);
                }
            }
            // in-plane: rows (axis n-2) and columns (axis n-1) from the padded tile
            {
                float rowv[2 * R][VEC];
#pragma unroll
                for (int k = -R; k <= R; ++k) {
                    if (k == 0) continue;
                    lds_vec<VEC>(pad + padc + k * PW, rowv[k < 0 ? k + R : k + R - 1]);
                }
                float lft[VEC], rgt[VEC];          // columns qc0-VEC .. qc0-1 and qc0+VEC .. qc0+2VEC-1
                lds_vec<VEC>(pad + padc - VEC, lft);
                lds_vec<VEC>(pad + padc + VEC, rgt);
#pragma unroll
                for (int v = 0; v < VEC; ++v) {
                    float x[NW];
#pragma unroll
                    for (int k = -R; k <= R; ++k) x[k + R] = k == 0 ? w[R][v] : rowv[k < 0 ? k + R : k + R - 1][v];
                    axis_update<F, R, PASS2>(f, NDIM - 2, qv[v], x, hih[NDIM - 2], acc[v], dis[v], mn[NDIM - 2], mx[NDIM - 2]);
                    // column window: element v + k of the concatenation lft | centre | rgt
#pragma unroll
                    for (int k = -R; k <= R; ++k) {
                        const int c = v + k;
                        x[k + R] = c < 0 ? lft[VEC + c] : (c < VEC ? w[R][c] : rgt[c - VEC]);
                    }
                    axis_update<F, R, PASS2>(f, NDIM - 1, qv[v], x, hih[NDIM - 1], acc[v], dis[v], mn[NDIM - 1], mx[NDIM - 1]);
                }
            }
            if constexpr (PASS2) {
                const long long gi = tb + lin;
                float o4[VEC];
#pragma unroll
                for (int v = 0; v < VEC; ++v) {
                    const float L = ham_finish(f, acc[v]) + dis[v];
                    o4[v] = stage_update(kind, brt, w[R][v], L, dt, Vn, T, gi + v);
                }
                sts_vec<VEC>(out + gi, o4);                 // vector store to global
            } else {
#pragma unroll
                for (int v = 0; v < VEC; ++v) {
                    nan |= (w[R][v] != w[R][v]);
                    mabs = fmaxf(mabs, fabsf(w[R][v]));
                }
            }
        }
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
typedef void (*stream_fn)(StreamArgs, GridDev, const float *, const float *, const float *, float *, float *,
                          const DevState *, FParams, int, int);

struct StreamFns {
    stream_fn pass1 = nullptr, pass2 = nullptr;
    int vec = 4;
};

struct StreamPlan {
    StreamArgs a;
    int block = 0, grid = 0;
    size_t smem = 0;
};

template <class F, int NDIM, int R, int VEC>
void stream_fns_v(stream_fn *p1, stream_fn *p2) {
    if constexpr (NDIM >= 3) {
        *p1 = k_stream<F, NDIM, R, VEC, false>;
        *p2 = k_stream<F, NDIM, R, VEC, true>;
    }
}

struct StreamFnsAll {
    stream_fn pass1[2] = {nullptr, nullptr}, pass2[2] = {nullptr, nullptr};   // [0]: VEC 2, [1]: VEC 4
};

template <class F, int NDIM, int R>
StreamFnsAll stream_fns() {
    StreamFnsAll t;
    stream_fns_v<F, NDIM, R, 2>(&t.pass1[0], &t.pass2[0]);
    stream_fns_v<F, NDIM, R, 4>(&t.pass1[1], &t.pass2[1]);
    return t;
}

// Decide whether the stream family covers this grid; picks the vector width from N1.
inline bool stream_plan(const GridDev &g, int R, const StreamFnsAll &all, StreamFns *fns, StreamPlan *p) {
    if (g.n < 3 || !all.pass1[0]) return false;
    const int N2 = g.N[g.n - 2], N1 = g.N[g.n - 1];
    const long long M = (long long)N2 * N1;
    if (M % 4) return false;                        // tile bases stay 16-B aligned
    if (N2 < R + 1 || N1 < R + 1) return false;
    int vec = N1 % 4 == 0 ? 4 : (N1 % 2 == 0 ? 2 : 0);
    if (const char *env = getenv("ODP_STREAM_VEC")) { const int v = atoi(env); if (N1 % v == 0) vec = v; }
    if (!vec || vec < R) return false;
    fns->pass1 = all.pass1[vec == 4];
    fns->pass2 = all.pass2[vec == 4];
    fns->vec = vec;
    StreamArgs &a = p->a;
    a.M = (int)M; a.N2 = N2; a.N1 = N1;
    a.per2 = g.per[g.n - 2]; a.per1 = g.per[g.n - 1];
    a.QR = N1 / vec;
    a.nquads = N2 * a.QR;
    if (a.nquads > STREAM_MAXT) return false;       // one quad per thread
    a.OFF = 4;
    a.PW = ((a.OFF + N1 + vec + 3) / 4) * 4;        // room for the last quad's right neighbours
    const int PH = N2 + 2 * R;
    a.pad_floats = ((PH * a.PW) + 3) / 4 * 4;
    const int MA = g.n - 3;
    const int Nm = g.N[MA];                         // locally owned marching extent
    a.ncols = 1;
    for (int o = 0; o < MA; ++o) a.ncols *= g.N[o];
    // segment length: whole columns when there are enough of them, else split for parallelism
    a.K = Nm;
    if ((long long)a.ncols < 148LL * 4) a.K = std::max(4, Nm / std::max(1, (148 * 8) / a.ncols));
    if (const char *env = getenv("ODP_STREAM_K")) a.K = std::max(1, atoi(env));
    a.K = std::min(a.K, Nm);
    a.nseg = (Nm + a.K - 1) / a.K;
    a.units = a.ncols * a.nseg;
    p->block = ((a.nquads + 31) / 32) * 32;
    p->smem = (size_t)2 * a.pad_floats * sizeof(float) + (size_t)2 * R * (N1 + N2) * 16 + 16;
    p->grid = 0;
    return true;
}

inline int stream_prepare(const StreamFns &t, StreamPlan &p, int nsm) {
    for (stream_fn fn : {t.pass1, t.pass2}) {
        if (cudaFuncSetAttribute((const void *)fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p.smem) != cudaSuccess)
            return 1;
    }
    int occ1 = 0, occ2 = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ1, (const void *)t.pass1, p.block, p.smem) != cudaSuccess) return 1;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ2, (const void *)t.pass2, p.block, p.smem) != cudaSuccess) return 1;
    const int occ = std::max(1, std::min(occ1, occ2));
    p.grid = std::min(p.a.units, nsm * occ);
    return 0;
}

inline void stream_pass1(const StreamFns &t, const StreamPlan &p, const GridDev &g, const float *W, float *partials,
                         const DevState *st, cudaStream_t s) {
    FParams fp;
    memset(&fp, 0, sizeof fp);
    t.pass1<<<p.grid, p.block, p.smem, s>>>(p.a, g, W, nullptr, nullptr, nullptr, partials, st, fp, 0, 0);
}

inline void stream_pass2(const StreamFns &t, const StreamPlan &p, const GridDev &g, const float *W, const float *Vn,
                         const float *T, float *out, const DevState *st, const FParams &fp, int kind, int brt,
                         cudaStream_t s) {
    t.pass2<<<p.grid, p.block, p.smem, s>>>(p.a, g, W, Vn, T, out, nullptr, st, fp, kind, brt);
}

}  // namespace odp
