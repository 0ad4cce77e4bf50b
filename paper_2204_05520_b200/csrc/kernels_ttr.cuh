// kernels_ttr.cuh -- time-to-reach by Lax-Friedrichs iteration (§3.3,
// Algorithm 3; readings A31-A35 in DESIGN.md §3).
//
// Algorithm 3 updates the grid in place in alternating orderings (Gauss-Seidel, §4.3).
// A sequential in-place sweep has no parallelism across the grid, so the GPU path iterates the
// same update as a Jacobi iteration (reading A35): every node of iteration k+1 is computed from
// iteration k, then the boundary rule of l.14-15 is applied along each non-periodic axis in order
// 0..n-1 (reading A34).  Buffers alternate and the convergence test
// (A31) runs on the device.  One iteration = 1 + (non-periodic axes) launches:
//
//   k_ttr_init      l.1: phi = 0 on the target {V0 <= 0}, `big` elsewhere
//   k_ttr_rows      l.5-12 on every node not on a non-periodic face (A32, A33); one CTA row group
//                   per iteration of its loop: the row's coordinates, face flags and index
//                   arithmetic are uniform, the innermost axis runs across the threads
//   k_ttr_face<d>   l.14-15 along non-periodic axis d on its two faces, in place, axes in order;
//                   the last CTA of the iteration's last launch runs l.2's stop test
//   k_ttr_finish    writes +0 over the target marker
//
// The target is carried in the value itself: a target node holds -0.0f (l.1, A34: never updated),
// every other node a value whose sign bit is clear (neighbour reads go through |x|, results are
// normalised with + 0.0f), so the iteration reads 8 bytes per node instead of 12 (no V0 stream).
#pragma once

#include "odp_device.cuh"

namespace odp {

struct TtrState {
    unsigned change[2];   // float bits of max |phi_new - phi_old| of the iteration writing parity p
    int done;             // 1 once the stop test passed
    int parity;           // buffer holding the result once done
    long long iters;      // iterations executed
    long long max_iters;
    float eps;
    unsigned blocks_done; // CTAs of the iteration's last launch that finished
    int strict;           // stop on change < eps (value iteration, A38) instead of <= eps (A31)
    int pad;
};

__device__ __forceinline__ bool is_target(float v) { return __float_as_uint(v) == 0x80000000u; }

__device__ __forceinline__ void ttr_reduce_change(float c, TtrState *st, int par) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) c = fmaxf(c, __shfl_xor_sync(0xffffffffu, c, off));
    // |x| >= 0: IEEE order of non-negative floats is the order of their bit patterns
    if ((threadIdx.x & 31) == 0 && c > 0.f) atomicMax(&st->change[par], __float_as_uint(c));
}

// Stop test of l.2 (A31) for the iteration that wrote `par`, run by the last CTA of the iteration's
// last launch: every CTA's atomicMax is visible after its fence + counter increment.
__device__ __forceinline__ void ttr_last_cta_control(TtrState *st, int par) {
    __shared__ bool last;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) last = atomicAdd(&st->blocks_done, 1u) == gridDim.x * gridDim.y * gridDim.z - 1;
    __syncthreads();
    if (last && threadIdx.x == 0) {
        __threadfence();
        st->blocks_done = 0u;
        st->iters += 1;
        const float c = __uint_as_float(atomicAdd(&st->change[par], 0u));
        const bool conv = st->strict ? c < st->eps : c <= st->eps;
        if (conv || st->iters >= st->max_iters) { st->done = 1; st->parity = par; }
        else st->change[par ^ 1] = 0u;
    }
}

__global__ void __launch_bounds__(256) k_ttr_init(long long P, const float *__restrict__ V0, float big,
                                                  float *__restrict__ phi) {
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < P; i += stride)
        phi[i] = __ldg(V0 + i) <= 0.f ? -0.f : big;                     // l.1 (target marker -0)
}

__global__ void __launch_bounds__(256) k_ttr_finish(long long P, const float *src, float *phi) {
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < P; i += stride)
        phi[i] = fabsf(src[i]);                                           // -0 target marker -> 0
}

__global__ void k_ttr_reset(TtrState *st, long long max_iters, float eps, int strict) {
    st->change[0] = st->change[1] = 0u;
    st->strict = strict;
    st->done = 0; st->parity = 0; st->iters = 0;
    st->max_iters = max_iters; st->eps = eps;
    st->blocks_done = 0u;
}

// l.5-12.  Rows = all axes but the innermost; RPB = rows per CTA step (blockDim / N_last, >= 1).
template <class F, int NDIM>
__global__ void __launch_bounds__(256) k_ttr_rows(GridDev g, FParams fp, const float *__restrict__ src,
                                                  float *__restrict__ dst, TtrState *st, int par, int last_launch) {
    if (st->done) return;
    constexpr int L = NDIM - 1;
    F f;
    {
        float mn[MAXD], mx[MAXD];
#pragma unroll
        for (int d = 0; d < MAXD; ++d) { mn[d] = -1.f; mx[d] = 1.f; }        // A33: costate box [-1, 1]^n
        f.init(fp, mn, mx);
    }
    const int NL = g.N[L];
    const int RPB = NL >= (int)blockDim.x ? 1 : (int)blockDim.x / NL;
    const int lr = NL >= (int)blockDim.x ? 0 : (int)threadIdx.x / NL;
    const int j0 = NL >= (int)blockDim.x ? (int)threadIdx.x : (int)threadIdx.x - lr * NL;
    const long long rows = g.P / NL;
    const bool perL = g.per[L] != 0;
    float cmax = 0.f;
    if (lr < RPB) {
        for (long long rg = blockIdx.x; rg * RPB < rows; rg += gridDim.x) {
            const long long r = rg * RPB + lr;
            if (r >= rows) break;
            int idx[NDIM];
            bool row_face = false;
            {
                long long rr = r;
#pragma unroll
                for (int d = L - 1; d >= 1; --d) {
                    const long long qd = rr / g.N[d];
                    idx[d] = (int)(rr - qd * g.N[d]);
                    rr = qd;
                }
                idx[0] = (int)rr;
#pragma unroll
                for (int d = 0; d < L; ++d) row_face |= !g.per[d] && (idx[d] == 0 || idx[d] == g.N[d] - 1);
            }
            const long long base = r * NL;
            if (row_face) {                              // A34: faces take l.14-15 in k_ttr_face
                for (int j = j0; j < NL; j += blockDim.x) dst[base + j] = src[base + j];
                continue;
            }
            Pt q;
#pragma unroll
            for (int d = 0; d < L; ++d) load_axis<F>(g, q, d, idx[d]);
            for (int j = j0; j < NL; j += blockDim.x) {
                const long long i = base + j;
                const float old = src[i];
                if (is_target(old) || (!perL && (j == 0 || j == NL - 1))) { dst[i] = old; continue; }   // A34
                idx[L] = j;
                load_axis<F>(g, q, L, j);
                float p[NDIM];
                float num = 0.f, den = 0.f;
#pragma unroll
                for (int d = 0; d < NDIM; ++d) {
                    const long long s = g.stride[d];
                    long long op = s, om = -s;
                    if (g.per[d]) {                      // periodic wrap (interior nodes never wrap otherwise)
                        if (idx[d] == g.N[d] - 1) op = -(long long)(g.N[d] - 1) * s;
                        if (idx[d] == 0) om = (long long)(g.N[d] - 1) * s;
                    }
                    const float vp = fabsf(src[i + op]), vm = fabsf(src[i + om]);
                    p[d] = (vp - vm) * g.hih[d];         // central difference (A32)
                    const float a = f.alpha(d, q);
                    num = fmaf(a * g.hih[d], vp + vm, num);
                    den = fmaf(a, g.inv_dx[d], den);
                }
                const float H = -f.ham(q, p) - 1.f;      // A32: H_TTR = -H_reach(goal -1) - 1
                const float nv = den > 0.f ? (num - H) / den : old;     // l.10-11 (A33)
                const float v = fminf(nv, old) + 0.f;    // l.12 (+0: never the target marker)
                dst[i] = v;
                cmax = fmaxf(cmax, fabsf(v - old));
            }
        }
    }
    ttr_reduce_change(cmax, st, par);
    if (last_launch) ttr_last_cta_control(st, par);
}

// l.5-12 for NDIM >= 2: thread = one column (fixed indices of axes 1..n-1, consecutive threads =
// consecutive addresses of an axis-0 plane), marching axis 0 over one segment of planes
// (blockIdx.y) with the axis-0 neighbours in a register window.  Per-column work (index
// decomposition, coordinates, wrapped neighbour offsets, face test) is done once per column.
template <class F, int NDIM>
__global__ void __launch_bounds__(256) k_ttr_march(GridDev g, FParams fp, const float *__restrict__ src,
                                                   float *__restrict__ dst, TtrState *st, int par, int last_launch,
                                                   int seg_len) {
    if (st->done) return;
    F f;
    {
        float mn[MAXD], mx[MAXD];
#pragma unroll
        for (int d = 0; d < MAXD; ++d) { mn[d] = -1.f; mx[d] = 1.f; }        // A33: costate box [-1, 1]^n
        f.init(fp, mn, mx);
    }
    const int ncol = (int)g.stride[0];
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    const int N0 = g.N[0];
    const int a0 = blockIdx.y * seg_len, a1 = min(N0, a0 + seg_len);
    float cmax = 0.f;
    if (c < ncol) {
        int idx[NDIM];
        bool col_face = false;
        int op[NDIM], om[NDIM];
        {
            int rem = c;
#pragma unroll
            for (int d = NDIM - 1; d >= 1; --d) {
                const int q = rem / g.N[d];
                idx[d] = rem - q * g.N[d];
                rem = q;
                const int sd = (int)g.stride[d];
                op[d] = sd; om[d] = -sd;
                if (g.per[d]) {
                    if (idx[d] == g.N[d] - 1) op[d] = -(g.N[d] - 1) * sd;
                    if (idx[d] == 0) om[d] = (g.N[d] - 1) * sd;
                } else if (idx[d] == 0 || idx[d] == g.N[d] - 1) {
                    col_face = true;
                }
            }
        }
        const long long s0 = (long long)ncol;
        if (col_face) {                                  // A34: faces take l.14-15 in k_ttr_face
            for (int i0 = a0; i0 < a1; ++i0) dst[i0 * s0 + c] = src[i0 * s0 + c];
        } else {
            Pt q;
#pragma unroll
            for (int d = 1; d < NDIM; ++d) load_axis<F>(g, q, d, idx[d]);
            const bool per0 = g.per[0] != 0;
            const float *col = src + c;
            auto at0 = [&](int i0) -> float {            // phi at plane i0 (wrapped if periodic)
                if (per0) i0 = i0 < 0 ? i0 + N0 : (i0 >= N0 ? i0 - N0 : i0);
                else i0 = max(0, min(N0 - 1, i0));
                return col[i0 * s0];
            };
            // U planes per batch: all loads of a batch are issued before its arithmetic (the
            // side-neighbour loads come from L2; the batch keeps U of them in flight per thread)
            constexpr int U = 4;
            float vm = fabsf(at0(a0 - 1)), vc = at0(a0);
            for (int ib = a0; ib < a1; ib += U) {
                float vn[U], sp[U][NDIM], sm[U][NDIM];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    if (ib + u < a1) {
                        vn[u] = at0(ib + u + 1);
                        const float *pc = col + (long long)(ib + u) * s0;
#pragma unroll
                        for (int d = 1; d < NDIM; ++d) { sp[u][d] = pc[op[d]]; sm[u][d] = pc[om[d]]; }
                    }
                }
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    if (ib + u >= a1) break;
                    const int i0 = ib + u;
                    const long long i = i0 * s0 + c;
                    const float old = vc;
                    if (is_target(old) || (!per0 && (i0 == 0 || i0 == N0 - 1))) {
                        dst[i] = old;                    // A34
                    } else {
                        load_axis<F>(g, q, 0, i0);
                        float p[NDIM];
                        const float vp0 = fabsf(vn[u]);
                        p[0] = (vp0 - vm) * g.hih[0];    // central difference (A32)
                        const float a0v = f.alpha(0, q);
                        float num = a0v * g.hih[0] * (vp0 + vm);
                        float den = a0v * g.inv_dx[0];
#pragma unroll
                        for (int d = 1; d < NDIM; ++d) {
                            const float vp = fabsf(sp[u][d]), vmd = fabsf(sm[u][d]);
                            p[d] = (vp - vmd) * g.hih[d];
                            const float a = f.alpha(d, q);
                            num = fmaf(a * g.hih[d], vp + vmd, num);
                            den = fmaf(a, g.inv_dx[d], den);
                        }
                        const float H = -f.ham(q, p) - 1.f;   // A32: H_TTR = -H_reach(goal -1) - 1
                        const float nv = den > 0.f ? (num - H) / den : old;   // l.10-11 (A33)
                        const float v = fminf(nv, old) + 0.f;               // l.12
                        dst[i] = v;
                        cmax = fmaxf(cmax, fabsf(v - old));
                    }
                    vm = fabsf(vc);
                    vc = vn[u];
                }
            }
        }
    }
    ttr_reduce_change(cmax, st, par);
    if (last_launch) ttr_last_cta_control(st, par);
}

// l.5-12 for NDIM >= 3 with an in-plane tile in shared memory: CTA = TY x TX nodes of the plane
// (axes n-2, n-1) for fixed middle-axis indices, marching axis 0 over a segment.  Each step stages
// the (TY+2) x (TX+2) tile of the next plane (halo wrapped on periodic axes), so the in-plane
// neighbours are LDS with constant offsets; axis-0 neighbours stay in registers (vm, vc) and the
// next plane's centre (vn) comes from the staged tile; middle axes (NDIM >= 4) through L1/L2.
constexpr int TTR_TX = 32, TTR_TY = 8;
constexpr int TTR_NPT = 4;                               // nodes per thread along the tile row
constexpr int TTR_TW = TTR_TX * TTR_NPT;                 // tile width (columns)

template <class F, int NDIM>
__global__ void __launch_bounds__(TTR_TX * TTR_TY) k_ttr_tile(GridDev g, FParams fp, const float *__restrict__ src,
                                                              float *__restrict__ dst, TtrState *st, int par,
                                                              int last_launch, int seg_len, int ntx, int nty) {
    if (st->done) return;
    constexpr int A = NDIM - 2, B = NDIM - 1;            // tile axes (rows, columns)
    constexpr int SW = TTR_TW + 2, SH = TTR_TY + 2, U = TTR_NPT;
    __shared__ float tile[3][SH * SW];
    F f;
    {
        float mn[MAXD], mx[MAXD];
#pragma unroll
        for (int d = 0; d < MAXD; ++d) { mn[d] = -1.f; mx[d] = 1.f; }        // A33: costate box [-1, 1]^n
        f.init(fp, mn, mx);
    }
    const int NA = g.N[A], NB = g.N[B];
    const int N0 = g.N[0];
    // block -> (tile column, tile row, middle-axis combination); blockIdx.y = axis-0 segment
    int bx = blockIdx.x;
    const int tcx = bx % ntx; bx /= ntx;
    const int tcy = bx % nty; bx /= nty;
    int idx[NDIM];
    long long mid = 0;                                   // offset of the middle-axis indices
#pragma unroll
    for (int d = A - 1; d >= 1; --d) {
        idx[d] = bx % g.N[d];
        bx /= g.N[d];
        mid += (long long)idx[d] * g.stride[d];
    }
    const int tx = threadIdx.x % TTR_TX, ty = threadIdx.x / TTR_TX;
    const int ja = tcy * TTR_TY + ty;
    idx[A] = ja;
    bool rowface = false;                                // on a non-periodic face of axes 1 .. n-2
#pragma unroll
    for (int d = 1; d < B; ++d) rowface |= !g.per[d] && (idx[d] == 0 || idx[d] == g.N[d] - 1);
    // this thread's U nodes: columns tcx TW + u TX + tx (lanes stay consecutive per node slot)
    bool inside[U], face[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
        const int jb = tcx * TTR_TW + u * TTR_TX + tx;
        inside[u] = ja < NA && jb < NB;
        face[u] = !inside[u] || rowface || (!g.per[B] && (jb == 0 || jb == NB - 1));
    }
    const long long s0 = g.stride[0];
    const int sA = (int)g.stride[A];
    const int a0 = blockIdx.y * seg_len, a1 = min(N0, a0 + seg_len);
    const bool per0 = g.per[0] != 0;
    // tile loader: this thread's tile elements, in-plane offsets fixed per CTA (halo wrapped on
    // periodic axes, clamped on the others: those values are only read by face nodes, which are not
    // updated here); cp.async into a 3-stage ring, one commit group per plane
    constexpr int NT = TTR_TX * TTR_TY, NE = (SH * SW + NT - 1) / NT;
    int eoff[NE];
    bool eok[NE];
#pragma unroll
    for (int k = 0; k < NE; ++k) {
        const int e = threadIdx.x + k * NT;
        eok[k] = e < SH * SW;
        const int r = e / SW, cc = e - r * SW;
        int ga = tcy * TTR_TY + r - 1, gb = tcx * TTR_TW + cc - 1;
        // full modulo on periodic axes: the tile (TW + 2 columns, TY + 2 rows) can reach more than
        // one period past the face when the extent is small (e.g. a 12-node theta axis)
        if (g.per[A]) ga = ((ga % NA) + NA) % NA; else ga = max(0, min(NA - 1, ga));
        if (g.per[B]) gb = ((gb % NB) + NB) % NB; else gb = max(0, min(NB - 1, gb));
        eoff[k] = ga * sA + gb;
    }
    auto at0 = [&](int i0) -> int {                      // wrapped / clamped plane index
        if (per0) return i0 < 0 ? i0 + N0 : (i0 >= N0 ? i0 - N0 : i0);
        return max(0, min(N0 - 1, i0));
    };
    const uint32_t tb0 = (uint32_t)__cvta_generic_to_shared(&tile[0][0]);
    constexpr uint32_t TB = 4u * SH * SW;                // bytes per stage
    auto issue = [&](uint32_t sb, const float *pl) {
#pragma unroll
        for (int k = 0; k < NE; ++k)
#ifdef ODP_CHECK
            if (eok[k] && !(pl + eoff[k] - src >= 0 && pl + eoff[k] - src < g.P)) {
                printf("odp check 60 failed: ttr tile source %lld of %lld (block %d)\n", (long long)(pl + eoff[k] - src),
                       (long long)g.P, blockIdx.x);
                __trap();
            } else
#endif
            if (eok[k])
                asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(sb + 4u * (uint32_t)(threadIdx.x + k * NT)),
                             "l"(pl + eoff[k]) : "memory");
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    auto plane = [&](int i0) -> const float * { return src + (long long)at0(i0) * s0 + mid; };
    Pt q[U];
#pragma unroll
    for (int u = 0; u < U; ++u)
        if (inside[u]) {
#pragma unroll
            for (int d = 1; d < B; ++d) load_axis<F>(g, q[u], d, idx[d]);
            load_axis<F>(g, q[u], B, tcx * TTR_TW + u * TTR_TX + tx);
        }
    const long long me = mid + (long long)ja * sA + tcx * TTR_TW + tx;   // element of node slot 0
    float cmax = 0.f;
    float vm[U], vc[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
        vm[u] = 0.f; vc[u] = 0.f;
        if (inside[u]) vm[u] = fabsf(src[(long long)at0(a0 - 1) * s0 + me + u * TTR_TX]);
    }
    uint32_t sc = tb0, sn = tb0 + TB, sf = tb0 + 2 * TB;   // stages: plane i0, i0 + 1, i0 + 2
    issue(sc, plane(a0));
    issue(sn, plane(a0 + 1));
    const float *pf = plane(a0 + 2);                     // next plane to fetch (interior: +s0 per step)
    float *dp = dst + (long long)a0 * s0 + me;
    auto ld = [](uint32_t addr) -> float {
        float v;
        asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(addr));
        return v;
    };
    const uint32_t ctr0 = 4u * (uint32_t)((ty + 1) * SW + tx + 1);
    for (int i0 = a0; i0 < a1; ++i0, dp += s0) {
        issue(sf, pf);                                   // (a group is committed even past the segment)
        pf = (i0 + 3 < N0) ? pf + s0 : plane(i0 + 3);
        asm volatile("cp.async.wait_group 1;" ::: "memory");   // planes i0 and i0 + 1 have landed
        __syncthreads();
        const bool face0 = !per0 && (i0 == 0 || i0 == N0 - 1);
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (!inside[u]) continue;
            const uint32_t c4 = ctr0 + 4u * (uint32_t)(u * TTR_TX);
            if (i0 == a0) vc[u] = ld(sc + c4);
            const float vn = ld(sn + c4);
            const float old = vc[u];
            float v = old;
            if (!face[u] && !face0 && !is_target(old)) {
                load_axis<F>(g, q[u], 0, i0);
                float p[NDIM];
                float num = 0.f, den = 0.f;
#pragma unroll
                for (int d = 0; d < NDIM; ++d) {
                    float vp, vmd;
                    if (d == 0) { vp = fabsf(vn); vmd = vm[u]; }
                    else if (d == A) { vp = fabsf(ld(sc + c4 + 4u * SW)); vmd = fabsf(ld(sc + c4 - 4u * SW)); }
                    else if (d == B) { vp = fabsf(ld(sc + c4 + 4u)); vmd = fabsf(ld(sc + c4 - 4u)); }
                    else {
                        const long long sd = g.stride[d];
                        long long op = sd, om = -sd;
                        if (g.per[d]) {
                            if (idx[d] == g.N[d] - 1) op = -(long long)(g.N[d] - 1) * sd;
                            if (idx[d] == 0) om = (long long)(g.N[d] - 1) * sd;
                        }
                        const float *pc = src + (dp - dst) + u * TTR_TX;
                        vp = fabsf(pc[op]); vmd = fabsf(pc[om]);
                    }
                    p[d] = (vp - vmd) * g.hih[d];        // central difference (A32)
                    const float a = f.alpha(d, q[u]);
                    num = fmaf(a * g.hih[d], vp + vmd, num);
                    den = fmaf(a, g.inv_dx[d], den);
                }
                const float H = -f.ham(q[u], p) - 1.f;   // A32: H_TTR = -H_reach(goal -1) - 1
                const float nv = den > 0.f ? (num - H) / den : old;   // l.10-11 (A33)
                v = fminf(nv, old) + 0.f;                // l.12
                cmax = fmaxf(cmax, fabsf(v - old));
            }
            dp[u * TTR_TX] = v;                          // (A34: target / faces keep their value)
            vm[u] = fabsf(vc[u]);
            vc[u] = vn;
        }
        __syncthreads();                                 // stage sc is refilled by the next issue
        const uint32_t t = sc; sc = sn; sn = sf; sf = t;
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    ttr_reduce_change(cmax, st, par);
    if (last_launch) ttr_last_cta_control(st, par);
}

// l.14-15 along axis d on its two faces, in place in dst (which holds the interior update and the
// rules of axes < d; face nodes were copied from src by k_ttr_rows).  The rule reads the nodes 1 and
// 2 cells inside, never on an axis-d face (N >= 4), so no value this launch writes is read.  Nodes
// whose highest non-periodic face axis is d are final and enter the change.
template <int NDIM>
__global__ void __launch_bounds__(256) k_ttr_face(GridDev g, int d, int last_launch, const float *__restrict__ src,
                                                  float *dst, TtrState *st, int par) {
    if (st->done) return;
    const long long inner = g.stride[d];
    const int Nd = g.N[d];
    const long long outer = g.P / (inner * Nd);
    const long long per_side = outer * inner;
    float cmax = 0.f;
    // index arithmetic in 32 bits when the face set and the element offsets fit (the usual case)
    auto body = [&](auto t, auto per_side_, auto inner_) {
        using I = decltype(t);
        const int side = t >= per_side_;
        const I r = side ? t - per_side_ : t;
        const I o = r / inner_, in = r - o * inner_;
        const long long i = (long long)o * ((long long)inner_ * Nd) + (side ? (long long)(Nd - 1) * inner_ : 0) + in;
        const float cur = dst[i];
        float v = cur;
        if (!is_target(cur)) {                           // A34: target nodes keep 0
            const long long sa = side ? -(long long)inner_ : (long long)inner_;
            const float a = fabsf(dst[i + sa]), b = fabsf(dst[i + 2 * sa]);
            v = fminf(fmaxf(2.f * a - b, b), cur) + 0.f;
            dst[i] = v;
        }
        // highest face axis of this node: the axes e > d are decoded from `in`
        bool last = true;
        I rem = in;
#pragma unroll
        for (int e = NDIM - 1; e > 0; --e) {
            if (e <= d) break;
            const I q = rem / (I)g.N[e];
            const int ie = (int)(rem - q * (I)g.N[e]);
            rem = q;
            if (!g.per[e] && (ie == 0 || ie == g.N[e] - 1)) last = false;
        }
        if (last) cmax = fmaxf(cmax, fabsf(v - src[i]));
    };
    if (2 * per_side < (1LL << 31)) {
        const unsigned ps = (unsigned)per_side, inn = (unsigned)inner, tot = 2u * ps;
        for (unsigned t = blockIdx.x * blockDim.x + threadIdx.x; t < tot; t += gridDim.x * blockDim.x) body(t, ps, inn);
    } else {
        const long long stride = (long long)gridDim.x * blockDim.x;
        for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < 2 * per_side; t += stride)
            body(t, per_side, inner);
    }
    ttr_reduce_change(cmax, st, par);
    if (last_launch) ttr_last_cta_control(st, par);
}

typedef void (*ttr_rows_fn)(GridDev, FParams, const float *, float *, TtrState *, int, int);
typedef void (*ttr_face_fn)(GridDev, int, int, const float *, float *, TtrState *, int);

typedef void (*ttr_march_fn)(GridDev, FParams, const float *, float *, TtrState *, int, int, int);
typedef void (*ttr_tile_fn)(GridDev, FParams, const float *, float *, TtrState *, int, int, int, int, int);

struct TtrFns {
    ttr_rows_fn rows = nullptr;       // NDIM == 1
    ttr_march_fn march = nullptr;     // NDIM >= 2
    ttr_tile_fn tile = nullptr;       // NDIM >= 3
    ttr_face_fn face = nullptr;
};

template <class F, int NDIM>
static TtrFns ttr_fns() {
    TtrFns t;
    if constexpr (NDIM == 1) t.rows = k_ttr_rows<F, NDIM>;
    else t.march = k_ttr_march<F, NDIM>;
    if constexpr (NDIM >= 3) t.tile = k_ttr_tile<F, NDIM>;
    t.face = k_ttr_face<NDIM>;
    return t;
}

}  // namespace odp
