// kernels_march.cuh -- the "march" kernel family (default) of the B200 HJ level-set step.
//
// Decomposition: a CTA owns a COLUMN of in-plane tiles (the two innermost, contiguous axes) at
// fixed indices of the "side" outer axes and marches the innermost outer axis (the MARCHING axis).
// Every tile a step reads -- the centre tile (row block + halo rows) and the 2R side-neighbour
// tiles per side axis -- is staged in shared memory by 1-D TMA bulk copies (cp.async.bulk, one
// lane of warp 0 per copy, completion on an mbarrier), issued one step ahead into double buffers,
// so threads read every stencil neighbour with a plain LDS at a fixed per-thread offset (the
// stream family spent ~45 % of its instructions on 64-bit global address arithmetic).  What the
// arithmetic does differently from the stream / generic families:
//
//  * EDGE SHARING.  The ENO2 selection of an edge i+1/2, m = pick(d2_i, d2_{i+1}), and its first
//    difference d1 = v_{i+1} - v_i give BOTH D+_i = d1 - m/2 and D-_{i+1} = d1 + m/2 (in units
//    of h; §3.4.4, reading A13).  Along the marching axis the edge of the previous step is
//    carried in registers (one second difference, one pick per node instead of three and two);
//    along the in-plane column axis the VEC nodes of a thread share their interior edges.
//  * EDGE-ASSIGNED PASS 1.  Pass 1 only needs the global range of {D-_i, D+_i} (Alg. 2
//    l.157-158, A4).  Every value is one side of an edge, so a node contributes its upper edge
//    (both sides) -- 3 loads, 2 second differences, 1 pick per side axis instead of 4, 3, 2 --
//    and min(D+, D-) = d1 - |m|/2, max = d1 + |m|/2 (exact: one of the two fma's).  Nodes on a
//    face add the one-sided values of the face edges (min/max are idempotent, so a value seen
//    twice is harmless; the only thing to avoid is a value that is not a node's D-/D+).
//  * PACKED FP32.  Two adjacent nodes of a row are one float2; every add/mul/fma on node pairs is
//    one FADD2/FMUL2/FFMA2 (sm_100a), the ENO picks are FSETP+FSEL per node, the range
//    accumulation is 3-input FMNMX3.
//  * NO CTA BARRIER IN THE LOOP.  One producer warp issues the copies and waits on "empty"
//    mbarriers (one arrive per compute warp and step); compute warps wait only on the "full"
//    mbarrier of their step, so warps drift freely within the two-stage pipeline.  In-plane ghost
//    cells (A12) are formed in registers by the threads on the tile faces (periodic halo rows are
//    copied by TMA, periodic columns read wrapped offsets).
//
// The arithmetic of every D-/D+ is the same sequence of IEEE float32 operations as in the stream
// and generic families (d2 = fma(-2, v_c, v_l + v_r); D = fma(+-0.5, m, d1)), so the derivative
// range of pass 1 is bit-identical across families.
//
//   pass 1 (PASS2=false): min/max of hD-/hD+ per axis, max|W| (NaN-propagating), per-CTA partials
//   pass 2 (PASS2=true):  p, H, alpha_i, dissipation, Euler/RK stage, BRT min (Alg. 2 l.153-169)
#pragma once

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <type_traits>

#include "kernels_stream.cuh"

namespace odp {

#ifndef ODP_MARCH_MINB1
#define ODP_MARCH_MINB1 2      // CTAs/SM the register budget of the NP=1 (VEC=2) kernels is sized for
#endif
#ifndef ODP_MARCH_MINB2
#define ODP_MARCH_MINB2 1      // ... and of the NP=2 (VEC=4) kernels
#endif
#ifndef ODP_MARCH_WAIT
#define ODP_MARCH_WAIT 1       // 1: mbarrier try_wait with a suspend hint; 0: try_wait + nanosleep back-off
#endif
#ifndef ODP_MARCH_LEANP
#define ODP_MARCH_LEANP 1      // producer: per-unit copy descriptors in registers (0: round-1 issue())
#endif
#ifndef ODP_MARCH_ECOUNT
#define ODP_MARCH_ECOUNT 0     // 1: stage release through a plain shared counter the producer polls
#endif
#ifndef ODP_MARCH_ECOUNT_NS
#define ODP_MARCH_ECOUNT_NS 32 // the producer's poll back-off (ODP_MARCH_ECOUNT = 1)
#endif
#ifndef ODP_MARCH_WAITP
#define ODP_MARCH_WAITP 1      // the producer's wait on a released stage (modes of mbar_wait_mode)
#endif
#ifndef ODP_MARCH_RELAY
#define ODP_MARCH_RELAY 0      // 1: one compute warp waits on the copies, named barrier for the rest
#endif
#ifndef ODP_MARCH_SLEEP_NS
#define ODP_MARCH_SLEEP_NS 64   // back-off of the ODP_MARCH_WAIT = 0 wait loop
#endif
#ifndef ODP_MARCH_KINDS
#define ODP_MARCH_KINDS 1      // MEDIUM shape-specialised pass 2 compiled per RK stage kind (0: runtime kind)
#endif
#ifndef ODP_MARCH_LDSTEP
#define ODP_MARCH_LDSTEP 1     // RK-stage-2 instances load Vn / T per step instead of one step ahead (0: off)
#endif
#ifndef ODP_MARCH_UNROLL
#define ODP_MARCH_UNROLL 1     // experiment: unroll the marching loop (window shifts become renames)
#endif
#ifndef ODP_MARCH_SELP
#define ODP_MARCH_SELP 0       // 1: ENO pick as FSET + 3 FMA-pipe ops instead of FSETP + FSEL
#endif
#ifdef ODP_MARCH_EXPERIMENTS
constexpr bool MARCH_EXP = true;   // timing experiments (ODP_MARCH_DBG): the kernels read MarchArgs::dbg
#else
constexpr bool MARCH_EXP = false;  // production: dbg is a compile-time 0
#endif
constexpr int MARCH_MAXT1 = 512;   // threads per CTA, NP = 1 (compute warps + the producer warp)
constexpr int MARCH_MAXT2 = 640;   // threads per CTA, NP = 2

// ---- packed fp32 helpers (FADD2 / FMUL2 / FFMA2 on sm_100a) -------------------------------------
__device__ __forceinline__ float2 f2(float a, float b) { return make_float2(a, b); }
__device__ __forceinline__ float2 f2s(float a) { return make_float2(a, a); }
__device__ __forceinline__ float2 add2(float2 a, float2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ float2 sub2(float2 a, float2 b) { return __fadd2_rn(a, make_float2(-b.x, -b.y)); }
__device__ __forceinline__ float2 mul2(float2 a, float2 b) { return __fmul2_rn(a, b); }
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }
// second difference d2 = fma(-2, c, l + r)  (bitwise the same as the scalar families)
__device__ __forceinline__ float2 d2p(float2 l, float2 c, float2 r) { return fma2(f2s(-2.f), c, add2(l, r)); }
__device__ __forceinline__ float d2s(float l, float c, float r) { return fmaf(-2.f, c, l + r); }

// A13: the smaller second difference in magnitude, the left one on ties
__device__ __forceinline__ float pick1(float a, float b) {
#if ODP_MARCH_SELP
    float p;   // p = 1 if |a| <= |b| else 0; a p + b (1 - p) is exact (one of the products is 0)
    asm("set.le.f32.f32 %0, %1, %2;" : "=f"(p) : "f"(fabsf(a)), "f"(fabsf(b)));
    return fmaf(b, 1.f - p, a * p);
#else
    return fabsf(a) <= fabsf(b) ? a : b;
#endif
}
__device__ __forceinline__ float2 pick2(float2 a, float2 b) { return f2(pick1(a.x, b.x), pick1(a.y, b.y)); }

// |x| on the FMA pipe (FADD RZ, |x|) rather than a LOP on the ALU pipe
__device__ __forceinline__ float absf(float x) { return fabsf(x) + 0.f; }
__device__ __forceinline__ float2 abs2(float2 a) { return f2(absf(a.x), absf(a.y)); }

__device__ __forceinline__ float min3f(float a, float b, float c) {
    float r;
    asm("min.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
    return r;
}
__device__ __forceinline__ float max3f(float a, float b, float c) {
    float r;
    asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
    return r;
}
__device__ __forceinline__ float max3nan(float a, float b, float c) {   // NaN-propagating (guard A19)
    float r;
    asm("max.NaN.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
    return r;
}

// |pick(a, b)| = min(|a|, |b|): the magnitude of the ENO2 selection without the selection itself
__device__ __forceinline__ float2 amin2(float2 a, float2 b) {
    return f2(fminf(fabsf(a.x), fabsf(b.x)), fminf(fabsf(a.y), fabsf(b.y)));
}
// range of the two sides of an edge {d1 - |m|/2, d1 + |m|/2} into [mn, mx] (both nodes of a pair);
// am = |m| (pass 1 never needs the sign of the selection)
__device__ __forceinline__ void inc_edge(float2 am, float2 d1, float &mn, float &mx) {
    const float2 lo = fma2(f2s(-0.5f), am, d1), hi = fma2(f2s(0.5f), am, d1);
    mn = min3f(mn, lo.x, lo.y);
    mx = max3f(mx, hi.x, hi.y);
}
__device__ __forceinline__ void inc_val(float2 v, float &mn, float &mx) {
    mn = min3f(mn, v.x, v.y);
    mx = max3f(mx, v.x, v.y);
}
__device__ __forceinline__ void inc_s(float v, float &mn, float &mx) {
    mn = fminf(mn, v);
    mx = fmaxf(mx, v);
}

// ---- ODP_CHECK builds (libodp_check.so, tests/test_gpu_checked.py): device-side bounds and
// alignment checks of every shared-memory read, TMA copy and global access of the march kernels,
// in place of compute-sanitizer (closed on this pool).  A failed check prints and traps. ----------
#ifdef ODP_CHECK
extern __shared__ __align__(128) float odp_dyn_smem[];
__device__ __noinline__ void odp_check_fail(int code, long long a, long long b) {
    printf("odp check %d failed: %lld %lld (block %d thread %d)\n", code, a, b, blockIdx.x, threadIdx.x);
    __trap();
}
#define ODP_CHK(cond, code, a, b) do { if (!(cond)) odp_check_fail((code), (long long)(a), (long long)(b)); } while (0)
__device__ __forceinline__ void odp_chk_smem(uint32_t addr, uint32_t bytes, int code) {
    uint32_t dsz;
    asm("mov.u32 %0, %%dynamic_smem_size;" : "=r"(dsz));
    const uint32_t base = smem_u32(odp_dyn_smem);
    ODP_CHK(addr >= base && addr + bytes <= base + dsz && (addr & (bytes >= 8 ? 7u : 3u)) == 0, code, addr - base, dsz);
}
#else
#define ODP_CHK(cond, code, a, b) ((void)0)
__device__ __forceinline__ void odp_chk_smem(uint32_t, uint32_t, int) {}
#endif

// 8-byte shared-memory load at a 32-bit shared address (one base register + immediate offsets)
__device__ __forceinline__ float2 lds2(uint32_t addr) {
    odp_chk_smem(addr, 8, 1);
    float2 v;
    asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"(addr));
    return v;
}

__device__ __forceinline__ bool mbar_test(uint64_t *bar, uint32_t parity) {   // non-blocking phase test
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n}"
        : "=r"(ok) : "r"(smem_u32(bar)), "r"(parity) : "memory");
    return ok != 0;
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// 1-D TMA bulk copy global -> shared (CTA-local destination address), completing on an mbarrier
__device__ __forceinline__ void tma_bulk_g2s_u32(uint32_t dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

// ghost value (A12) for a pair
__device__ __forceinline__ float2 ghost2(float2 e, float2 in, float q) { return f2(ghost(e.x, in.x, q), ghost(e.y, in.y, q)); }

// Fix the out-of-domain slots of a pair window x[0..2R] centred on index i of an axis of extent N
// (non-periodic): the pair version of fix_ghosts.
template <int R>
__device__ __forceinline__ void fix_ghosts2(float2 *x, int i, int N) {
    float xs[2 * R + 1], ys[2 * R + 1];
#pragma unroll
    for (int k = 0; k <= 2 * R; ++k) { xs[k] = x[k].x; ys[k] = x[k].y; }
    fix_ghosts<R>(xs, i, N);
    fix_ghosts<R>(ys, i, N);
#pragma unroll
    for (int k = 0; k <= 2 * R; ++k) x[k] = f2(xs[k], ys[k]);
}

// ---- vector memory helpers: NP float2 pairs = 2 NP consecutive floats ---------------------------
template <int NP>
__device__ __forceinline__ void ldg_p(const float *p, float2 *v) {
    if constexpr (NP == 2) {
        const float4 t = __ldg(reinterpret_cast<const float4 *>(p));
        v[0] = f2(t.x, t.y); v[1] = f2(t.z, t.w);
    } else {
        v[0] = __ldg(reinterpret_cast<const float2 *>(p));
    }
}
template <int NP>
__device__ __forceinline__ void ldg_plain(const float *p, float2 *v) {   // coherent load (may alias out)
    if constexpr (NP == 2) {
        const float4 t = *reinterpret_cast<const float4 *>(p);
        v[0] = f2(t.x, t.y); v[1] = f2(t.z, t.w);
    } else {
        v[0] = *reinterpret_cast<const float2 *>(p);
    }
}
template <int NP>
__device__ __forceinline__ void lds_p(const float *p, float2 *v) {
    if constexpr (NP == 2) {
        const float4 t = *reinterpret_cast<const float4 *>(p);
        v[0] = f2(t.x, t.y); v[1] = f2(t.z, t.w);
    } else {
        v[0] = *reinterpret_cast<const float2 *>(p);
    }
}
template <int NP>
__device__ __forceinline__ void st_p(float *p, const float2 *v) {
    if constexpr (NP == 2) *reinterpret_cast<float4 *>(p) = make_float4(v[0].x, v[0].y, v[1].x, v[1].y);
    else *reinterpret_cast<float2 *>(p) = v[0];
}

// ---- pass-2 per-axis terms ----------------------------------------------------------------------
// Every compiled-in functor except the ball has a separable Hamiltonian
//     H = sum_d [ c_d(x) p_d + k_d |p_d| ]     (table C-2; Eq. 4 with bang-bang u*, d*)
// with p_d = (D-_d + D+_d)/2 (A3); c_d, k_d below.  The ball accumulates sum p_d^2 (H = kH |p|_2).
// Inputs are s = h(D- + D+) and t = h(D+ - D-); hih = 1/(2h).
template <class F> struct Sep { static constexpr bool ball = false; };
template <int N> struct Sep<FHoloBall<N>> { static constexpr bool ball = true; };

template <int NDIM> __device__ __forceinline__ float lin_c(const FHoloBox<NDIM> &, int, const Pt &) { return 0.f; }
template <int NDIM> __device__ __forceinline__ float abs_k(const FHoloBox<NDIM> &f, int) { return f.kH; }
template <int NDIM> __device__ __forceinline__ float lin_c(const FHoloBall<NDIM> &, int, const Pt &) { return 0.f; }
template <int NDIM> __device__ __forceinline__ float abs_k(const FHoloBall<NDIM> &, int) { return 0.f; }
__device__ __forceinline__ float lin_c(const FDubins3D &f, int d, const Pt &q) {
    return d == 0 ? f.v * q.c[2] : (d == 1 ? f.v * q.s[2] : 0.f);
}
__device__ __forceinline__ float abs_k(const FDubins3D &f, int d) { return d == 2 ? f.kw : 0.f; }
__device__ __forceinline__ float lin_c(const FCar4D &, int d, const Pt &q) {
    return d == 0 ? q.x[2] * q.c[3] : (d == 1 ? q.x[2] * q.s[3] : 0.f);
}
__device__ __forceinline__ float abs_k(const FCar4D &f, int d) {
    return d == 0 ? f.kdx : (d == 1 ? f.kdy : (d == 2 ? f.ka : f.kw));
}
__device__ __forceinline__ float lin_c(const FCar5D &, int d, const Pt &q) {
    return d == 0 ? q.x[3] * q.c[2] : (d == 1 ? q.x[3] * q.s[2] : (d == 2 ? q.x[4] : 0.f));
}
__device__ __forceinline__ float abs_k(const FCar5D &f, int d) { return d == 3 ? f.ka : (d == 4 ? f.kal : 0.f); }
__device__ __forceinline__ float lin_c(const FDoubleInt6D &, int d, const Pt &q) { return (d & 1) == 0 ? q.x[d + 1] : 0.f; }
__device__ __forceinline__ float abs_k(const FDoubleInt6D &f, int d) { return (d & 1) ? f.kv : 0.f; }

// compile-time masks of the axes with a linear / an absolute-value term
template <class F> struct Terms { static constexpr unsigned LIN = 0, ABS = 0x3f; };   // holonomic box
template <int N> struct Terms<FHoloBall<N>> { static constexpr unsigned LIN = 0, ABS = 0; };
template <> struct Terms<FDubins3D> { static constexpr unsigned LIN = 0x3, ABS = 0x4; };
template <> struct Terms<FCar4D> { static constexpr unsigned LIN = 0x3, ABS = 0xf; };
template <> struct Terms<FCar5D> { static constexpr unsigned LIN = 0x7, ABS = 0x18; };
template <> struct Terms<FDoubleInt6D> { static constexpr unsigned LIN = 0x15, ABS = 0x2a; };

// Per axis, with u = hD-, w = hD+ (units of h) and hih = 1/(2h), H_d + dissipation_d is
//   c (u+w) hih + k |u+w| hih + alpha (w-u) hih          (A3, A2, A6)
// For an axis with a linear term only and alpha = |c| (PQ) this is 2 hih [min(c,0) u + max(c,0) w];
// for an |p| term only and alpha = |k| (AB) it is 2 |k| hih (k < 0 ? min(w, -u) : max(w, -u)) -- exact
// algebra, one accumulator, no separate dissipation sum.  alpha_d = |c| / |k| holds for every such
// axis of the compiled-in functors (table C-2; an AB axis's switching-costate sign set is never
// empty).  Axes with both terms (CAR4D x, y: alpha depends on the range) use the general form.
template <class F>
__device__ __forceinline__ void axis_terms(const F &f, int d, const Pt &q0, const Pt &q1, float hih, float2 u,
                                           float2 w, float2 &acc, float2 &dis, float2 *pv) {
    const bool lin = (Terms<F>::LIN >> d) & 1, ab = (Terms<F>::ABS >> d) & 1;
    if (F::SEPARABLE && !Sep<F>::ball && lin && !ab) {                      // PQ
        const float c0 = lin_c(f, d, q0), c1 = lin_c(f, d, q1), h2 = 2.f * hih;
        acc = fma2(f2(fminf(c0, 0.f) * h2, fminf(c1, 0.f) * h2), u, acc);
        acc = fma2(f2(fmaxf(c0, 0.f) * h2, fmaxf(c1, 0.f) * h2), w, acc);
        return;
    }
    if (F::SEPARABLE && !Sep<F>::ball && ab && !lin) {                      // AB
        const float k = abs_k(f, d);
        const float2 v = k < 0.f ? f2(fminf(w.x, -u.x), fminf(w.y, -u.y)) : f2(fmaxf(w.x, -u.x), fmaxf(w.y, -u.y));
        acc = fma2(f2s(2.f * fabsf(k) * hih), v, acc);
        return;
    }
    const float2 s = add2(u, w), t = sub2(w, u);
    if constexpr (!F::SEPARABLE) {
        pv[d] = mul2(s, f2s(hih));                   // p_d = (D- + D+)/2 (A3); H at the end of the node
    } else if constexpr (Sep<F>::ball) {
        const float2 sh = mul2(s, f2s(hih));
        acc = fma2(sh, sh, acc);
    } else {
        if (lin) acc = fma2(s, f2(lin_c(f, d, q0) * hih, lin_c(f, d, q1) * hih), acc);
        if (ab) {
            const float k = abs_k(f, d) * hih;
            acc = f2(fmaf(fabsf(s.x), k, acc.x), fmaf(fabsf(s.y), k, acc.y));
        }
    }
    dis = fma2(t, f2(f.alpha(d, q0) * hih, f.alpha(d, q1) * hih), dis);
}

template <class F>
__device__ __forceinline__ float2 ham_fin2(const F &f, float2 acc) {
    if constexpr (Sep<F>::ball) return f2(f.kH * sqrtf(acc.x), f.kH * sqrtf(acc.y));
    else return acc;
}
template <> struct Terms<FPairDubins3D> { static constexpr unsigned LIN = 0, ABS = 0; };
__device__ __forceinline__ float lin_c(const FPairDubins3D &, int, const Pt &) { return 0.f; }
__device__ __forceinline__ float abs_k(const FPairDubins3D &, int) { return 0.f; }

// ---- kernel -------------------------------------------------------------------------------------
//
// Unit of work: (column, marching segment, row block).  A COLUMN fixes the side-axis indices; the
// CTA marches the marching axis over the segment; a ROW BLOCK is B consecutive rows of the in-plane
// tile (B = N2 when the whole tile fits the CTA).  Shared memory per CTA:
//   ring  RS = R+2 slots, each the row block +-R halo rows of one centre tile (the tile of marching
//         index j is the centre of step j; slot = step counter mod RS);
//   side  2 buffers x NSS slots (NSS = 2R per side axis), each the row block of one side-neighbour
//         tile of the current step;
//   bars  two mbarriers (one per buffer parity).
// Warp 0 issues every copy as a 1-D TMA bulk copy (cp.async.bulk, one lane per copy) one step
// ahead: while step j computes, the tiles of step j+1 are in flight.  A thread's stencil
// neighbours are then plain LDS at fixed per-thread offsets -- no global address arithmetic in the
// loop (the stream family spent ~45 % of its instructions there).
struct MarchArgs {
    int M, N2, N1;        // tile size and in-plane extents
    int per2, per1;
    int xs;               // pass 2's streamed operands staged by TMA: bit 0 the target T, bit 1 Vn
    int B, nrb;           // rows per row block, row blocks per tile
    int nthr;             // B * QR
    int RSZ, SSZ;         // floats per ring / side slot
    int xoff;             // float offset of the T / Vn slots ([NST][xn] x SSZ)
    int xn;               // T / Vn slots per stage (0..2)
    int rmarg;            // leading margin of a ring slot (keeps TMA destinations 16-B aligned)
    int side_off;         // float offset of the side buffers
    int bar_off;          // float offset of the mbarriers
    int tab_off;          // float offset of the per-unit copy table
    int aux_off;          // float offset of the per-warp side geometry [16][2*3] and the marching coordinate table
    int mtab_n;           // entries of the marching coordinate table in shared memory (0: read the global table)
    int sn[3];            // local extents of the side axes (work order, march_col)
    int b1;               // axis-1 block of the work order (divides sn[1])
    int ncols;            // columns (product of the side extents)
    int dbg;              // 0 in the production build; ODP_MARCH_DBG under -DODP_MARCH_EXPERIMENTS only
    int K, nseg, units;   // marching segment length, segments per column, work units
    // axis-0 subset of the columns (multi-GPU overlap): 0 all, 1 interior planes
    // [i0r, N0 - i0r), 2 boundary planes [0, i0r) and [N0 - i0r, N0); s0n = planes in the subset
    int i0map, i0r, s0n;
    int wslot;            // dynamic work counter of this launch (st->work[wslot])
};
constexpr int MARCH_SMARG = 4;   // leading margin of a side slot (floats)

// Shared-memory geometry of a CTA (floats), a function of (R, N1, B, NSS) only; used by the host
// plan and -- for the shape-specialised instances -- as compile-time constants in the kernel, so
// every stencil read is an LDS at an immediate offset from one per-thread base register.
__host__ __device__ constexpr int geo_rmarg(int R, int N1) { return 4 + ((-R * N1) & 3); }
// ring slot: [rmarg][(B + 2R) rows x N1][slack][column-ghost table: (B + 2R) rows x 4 floats]
__host__ __device__ constexpr int geo_rgt(int R, int N1, int B) {
    return ((geo_rmarg(R, N1) + (B + 2 * R) * N1 + 4 + 3) / 4) * 4;
}
__host__ __device__ constexpr int geo_rsz(int R, int N1, int B) { return geo_rgt(R, N1, B) + 4 * (B + 2 * R); }
__host__ __device__ constexpr int geo_ssz(int N1, int B) { return ((MARCH_SMARG + B * N1 + 3) / 4) * 4; }
// NST pipeline stages: NST side buffers, R + NST ring slots
__host__ __device__ constexpr int geo_side_off(int R, int N1, int B, int NST) { return (R + NST) * geo_rsz(R, N1, B); }
__host__ __device__ constexpr int geo_bar_off(int R, int N1, int B, int NSS, int NST) {
    return ((geo_side_off(R, N1, B, NST) + NST * NSS * geo_ssz(N1, B)) + 3) / 4 * 4;
}
// 4 NST <= 16 mbarriers (128 B) + copy table: 32 x 8 B offsets + 32 x 4 B sizes + 8 x 4 B ring fields
// + unit queue (4 ints) + issued-step records (3 NST <= 12 ints)
__host__ __device__ constexpr int geo_smem_bytes(int R, int N1, int B, int NSS, int NST) {
    return geo_bar_off(R, N1, B, NSS, NST) * 4 + 144 + 32 * 8 + 32 * 4 + 8 * 4 + 16 + 52;
}

struct MarchUnit {
    int col, seg, rb, r0, nrow;   // column, segment, row block, first row, rows owned
    int m0, m1;                   // global marching range of the segment
    long long cbase;              // element offset of the column's tile at local marching index 0
};

// Work order of the columns (L2 reuse).  A column's side neighbours are the columns at +-1, +-2 on
// each side axis; CTAs run ~2 x 148 consecutive units at a time, so consecutive units should be
// side-axis neighbours: axis 0 (the largest stride) varies fastest, then -- for three side axes --
// axis 2 inside blocks of b1 consecutive axis-1 indices, so the +-2 neighbourhood of a wave stays
// resident in the 126 MB L2 instead of being re-read from HBM (ncu: 5.2x algorithmic DRAM bytes
// with the memory order).  Returns the memory-order column index.
__device__ __forceinline__ int march_i0(const MarchArgs &a, int i) {   // subset index -> axis-0 plane
    if (a.i0map == 1) return i + a.i0r;
    if (a.i0map == 2) return i < a.i0r ? i : a.sn[0] - 2 * a.i0r + i;
    return i;
}

template <int MA>
__device__ __forceinline__ int march_col(const MarchArgs &a, int c) {
    if constexpr (MA <= 1) {
        return march_i0(a, c);
    } else if constexpr (MA == 2) {
        const int i0 = march_i0(a, c % a.s0n), i1 = c / a.s0n;
        return i0 * a.sn[1] + i1;
    } else {
        const int i0 = march_i0(a, c % a.s0n);
        int r = c / a.s0n;
        const int i1l = r % a.b1;
        r /= a.b1;
        const int i2 = r % a.sn[2];
        const int i1 = (r / a.sn[2]) * a.b1 + i1l;
        return (i0 * a.sn[1] + i1) * a.sn[2] + i2;
    }
}

template <int MA>
__device__ __forceinline__ MarchUnit march_unit(const MarchArgs &a, int Nml, int mlo, int u) {
    MarchUnit U;
    const int rb = u % a.nrb;
    const int cs = u / a.nrb;
    U.seg = cs / a.ncols;                          // segments slowest: a wave spans many columns, few steps
    const int c = cs - U.seg * a.ncols;
    U.col = march_col<MA>(a, c);
    U.rb = rb;
    U.r0 = rb * a.B;
    U.nrow = min(a.B, a.N2 - U.r0);
    U.m0 = mlo + U.seg * a.K;
    U.m1 = min(mlo + Nml, U.m0 + a.K);
    U.cbase = (long long)U.col * Nml * a.M;
    return U;
}

// mbarrier wait with back-off: a warp that finds its data missing sleeps instead of spinning, so
// it does not take issue slots from the warps that are computing
// mode 2: non-blocking test_wait in a tight loop (fastest wake-up, spends issue slots);
// mode 3: try_wait without a suspend-time hint (the hardware's default time limit) in a loop
template <int MODE>
__device__ __forceinline__ void mbar_wait_mode(uint64_t *bar, uint32_t parity) {
    if constexpr (MODE == 2) {
        asm volatile(
            "{\n\t.reg .pred p;\n"
            "TW_%=:\n\t"
            "mbarrier.test_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
            "@!p bra TW_%=;\n}" ::"r"(smem_u32(bar)), "r"(parity) : "memory");
    } else if constexpr (MODE == 3) {
        asm volatile(
            "{\n\t.reg .pred p;\n"
            "TY_%=:\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
            "@!p bra TY_%=;\n}" ::"r"(smem_u32(bar)), "r"(parity) : "memory");
    } else {
        mbar_wait(bar, parity);
    }
}

__device__ __forceinline__ void mbar_wait_sleep(uint64_t *bar, uint32_t parity) {
#if ODP_MARCH_WAIT == 2 || ODP_MARCH_WAIT == 3
    mbar_wait_mode<ODP_MARCH_WAIT>(bar, parity);
    return;
#endif
#if ODP_MARCH_WAIT == 1
    mbar_wait(bar, parity);      // try_wait with a suspend-time hint: the hardware parks the warp
    return;
#endif
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n}"
        : "=r"(ok) : "r"(smem_u32(bar)), "r"(parity) : "memory");
    while (!ok) {
        __nanosleep(ODP_MARCH_SLEEP_NS);
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n}"
            : "=r"(ok) : "r"(smem_u32(bar)), "r"(parity) : "memory");
    }
}

// LBT / LBM: the launch bounds (threads per CTA, CTAs per SM) the register budget is sized for;
// shape-specialised instances with fewer rows per block may set them to their own block size
// KIND >= 0: pass 2 compiled for one stage kind (Euler / RK stage 1 / RK stage 2), -1: runtime `kind`
template <class F, int NDIM, int R, int NP, bool PASS2, int CN1 = 0, int CB = 0, int NST = 2,
          int LBT = MARCH_MAXT1, int LBM = ODP_MARCH_MINB1, int KIND = -1>
__global__ void __launch_bounds__(LBT, LBM)
k_march(MarchArgs a, GridDev g, const float *__restrict__ W, const float *Vn, const float *__restrict__ T,
        float *out, float *partials, const DevState *st, FParams fp, int kind, int brt) {
    static_assert(NP == 1, "the march family computes node pairs (VEC = 2)");
    static_assert(NST >= 2 && NST <= 4, "pipeline depth 2..4 (<= 18 mbarriers, unit queue of NST)");
    // dynamic work distribution: pass 1 takes units from work[0], pass 2 from work[1]; each pass
    // resets the other pass's counter (that launch has completed: same stream)
    unsigned int *wctr = const_cast<unsigned int *>(&st->work[a.wslot]);
    if (blockIdx.x == 0 && threadIdx.x == 0)          // the other launches' counters (stream order: not running)
        for (int k = 0; k < 3; ++k)
            if (k != a.wslot) const_cast<DevState *>(st)->work[k] = 0u;
    if (!st->active) return;
    constexpr int VEC = 2;
    constexpr int NO = NDIM - 2;     // outer axes
    constexpr int MA = NO - 1;       // marching axis; axes 0..MA-1 are the side axes
    constexpr int NSA = MA > 0 ? MA : 1;
    constexpr int RS = R + NST;      // ring slots
    constexpr bool CT = CN1 > 0;     // shape-specialised instance: geometry known at compile time
    constexpr int NSS = 2 * R * MA;  // side slots per stage
    // pass 2's T / Vn staged by TMA (a.xs): LOW instances only -- in the MEDIUM pass 2 the extra
    // live state costs spills and occupancy (c4 / c3 / c5-MEDIUM measured slower)
    constexpr bool XSC = PASS2 && R == 1;
    const int xs = XSC ? a.xs : 0;
    const int dbg = MARCH_EXP ? a.dbg : 0;
    // LOW (R = 1) is always forward Euler (odp.cu's step sequence); MEDIUM runs RK stages 1 and 2
    if constexpr (R == 1 && PASS2) kind = STAGE_EULER;
    if constexpr (KIND >= 0 && PASS2) kind = KIND;
    // RK stage 2 instances load Vn / T at the start of each step (no loop-carried registers); the
    // others keep the one-step-ahead load (DESIGN.md §7 third table)
    constexpr bool LDSTEP = ODP_MARCH_LDSTEP && KIND == STAGE_RK2;
    extern __shared__ __align__(128) float smem[];
    const int N1 = CT ? CN1 : a.N1;
    const int RSZ = CT ? geo_rsz(R, CN1, CB) : a.RSZ;
    const int SSZ = CT ? geo_ssz(CN1, CB) : a.SSZ;
    const int RMG = CT ? geo_rmarg(R, CN1) : a.rmarg;
    float *ring = smem;
    float *side = smem + (CT ? geo_side_off(R, CN1, CB, NST) : a.side_off);
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem + a.bar_off);
    // tma[b]:   the copies of a step with parity b landed (producer arrive.expect_tx + bytes)
    // empty[b]: every compute warp is done reading that step's buffers (one arrive per warp)
    // ubar[q]:  unit-queue entry q is written (producer arrive)
    uint64_t *tmab = bars, *empty = bars + NST, *ubar = bars + 2 * NST;

    float mn[NDIM], mx[NDIM], mabs = 0.f;
#pragma unroll
    for (int d = 0; d < NDIM; ++d) { mn[d] = __int_as_float(0x7f800000); mx[d] = -__int_as_float(0x7f800000); }
    F f;
    float dt = 0.f;
    const float *hih = g.hih;                 // 1/(2h) per axis (kernel-parameter space)
    if constexpr (PASS2) {
        f.init(fp, st->minD, st->maxD);
        dt = st->dt_f;
    }

    const int N2 = a.N2, M = a.M;
    const int QR = N1 / VEC;
    const int tid = threadIdx.x;
    const int nwc = (a.nthr + 31) >> 5;                // compute warps; warp nwc is the producer
    const int lrow = tid / QR;                         // row within the row block
    const int qc0 = (tid - lrow * QR) * VEC;           // first column of this thread's nodes
    const int toff = RMG + (lrow + R) * N1 + qc0;      // this thread's nodes in a ring slot
    const int sloc = MARCH_SMARG + lrow * N1 + qc0;    // ... in a side slot
    // left / right column pairs: the tile itself (wrapped within the row on a periodic column
    // axis); on a non-periodic column face the pair's ghost cells are formed in registers (A12)
    const bool cfirst = qc0 == 0, clast = qc0 + VEC == N1;
    const int loff = cfirst ? (a.per1 ? N1 - 2 : 0) : -2;
    const int roff = clast ? (a.per1 ? -(N1 - 2) : 0) : VEC;
    const bool gfirst = cfirst && !a.per1, glast = clast && !a.per1;
    Pt qcv[VEC];                                       // in-plane column coordinates (pass 2)
    if constexpr (PASS2) {
#pragma unroll
        for (int j = 0; j < VEC; ++j) load_axis<F>(g, qcv[j], NDIM - 1, qc0 + j);
    }

    const int Nm = MA == 0 ? g.Ng0 : g.N[MA];       // marching extent (global: face tests)
    const int mlo = MA == 0 ? g.g0 : 0;              // global index of local marching index 0
    const int Nml = MA == 0 ? g.N[0] : g.N[MA];      // locally owned marching extent
    const bool mper = g.per[MA] != 0;
    auto mloc = [&](int jg) -> int {                 // local marching index of global jg (clamped / wrapped)
        int j = jg;
        if (j < 0 || j >= Nm) {
            if (mper) j = j < 0 ? j + Nm : j - Nm;
            else j = j < 0 ? 0 : Nm - 1;
        }
        return j - mlo;
    };
    auto side_geom = [&](int col, int *oid, int *oN) {
        int r = col;
#pragma unroll
        for (int o = MA - 1; o >= 1; --o) { const int qv = r / g.N[o]; oid[o] = r - qv * g.N[o]; oN[o] = g.N[o]; r = qv; }
        if constexpr (MA >= 1) { oid[0] = g.g0 + r; oN[0] = g.Ng0; }
    };

    // ---- producer: copy table of a unit (lane l < NSS: side slot l; lane NSS: the ring tile) ----
    long long *t_soff = reinterpret_cast<long long *>(smem + a.tab_off);   // [32]
    uint32_t *t_snb = reinterpret_cast<uint32_t *>(t_soff + 32);           // [32] bytes (0 = skip)
    int *t_ring = reinterpret_cast<int *>(t_snb + 32);                      // [8]
    int *uq = t_ring + 8;                                                   // [NST] unit queue (producer -> compute warps)
    auto make_table = [&](const MarchUnit &U) {
        const int lane = tid & 31;
        int oid[NSA], oN[NSA];
        side_geom(U.col, oid, oN);
        if (lane < NSS) {
            const int o = lane / (2 * R), kk = lane - o * 2 * R;
            const int k = kk < R ? kk - R : kk - R + 1;
            int io = 0, no = 1, per = 0;
            long long so = 0;
#pragma unroll
            for (int q = 0; q < MA; ++q)
                if (q == o) { io = oid[q]; no = oN[q]; per = g.per[q]; so = g.stride[q]; }
            const bool face = !per && (io < R || io > no - 1 - R);
            int jo = io + k;
            bool ok = true;
            if (jo < 0 || jo >= no) {
                if (per) jo = jo < 0 ? jo + no : jo - no;
                else ok = false;
            }
            // pass 1 interior: edge i+1/2 only -- the -R tile (ENO2) / the -1 tile (upwind) is never read
            if (!PASS2 && !face && k == -R) ok = false;
            t_soff[lane] = (long long)(jo - io) * so + (long long)U.r0 * N1;
            t_snb[lane] = ok ? (uint32_t)U.nrow * N1 * 4 : 0u;
        }
        if (lane == 0) {
            const int va = U.r0 - R, vb = U.r0 + U.nrow + R;          // virtual rows [va, vb) of a ring slot
            const int ra = max(va, 0), rbb = min(vb, N2);
            int fa = ra * N1, fb = rbb * N1;
            fa &= ~3; fb = (fb + 3) & ~3;                              // 16-B granules inside the tile
            t_ring[0] = fa;
            t_ring[1] = (fb - fa) * 4;
            t_ring[2] = RMG + fa - va * N1;                            // destination float offset in the slot
            t_ring[3] = (a.per2 && va < 0) ? (-va) * N1 * 4 : 0;
            t_ring[4] = (a.per2 && vb > N2) ? (vb - N2) * N1 * 4 : 0;
            t_ring[5] = RMG + (N2 - va) * N1;
            t_ring[6] = (N2 + va) * N1;                                // wrap-lo source row offset
        }
        __syncwarp();
    };
    // copies of step `itx` = marching index j of unit U (ring tiles j+kb .. j+R), on tma[itx & 1]
    auto issue = [&](const MarchUnit &U, int j, int itx, int kb) {
        const int lane = tid & 31;
        const int stg = itx % NST;
        uint64_t *bar = &tmab[stg];
        const long long tj = U.cbase + (long long)(j - mlo) * M;
        uint32_t nb = 0, nbw0 = 0, nbw1 = 0;
        const float *src = nullptr;
        uint32_t dst = 0;
        long long tt = 0;
        float *slot = nullptr;
        if (lane < NSS) {
            nb = t_snb[lane];
            src = W + tj + t_soff[lane];
            dst = smem_u32(side + stg * NSS * SSZ + lane * SSZ + MARCH_SMARG);
        } else if (lane - NSS >= kb && lane - NSS <= R) {
            const int k = lane - NSS, mj = j + k;
            if (mj < U.m1) {
                tt = U.cbase + (long long)mloc(mj) * M;
                slot = ring + ((itx + k) % RS) * RSZ;
                nb = (uint32_t)t_ring[1];
                src = W + tt + t_ring[0];
                dst = smem_u32(slot + t_ring[2]);
                nbw0 = (uint32_t)t_ring[3];
                nbw1 = (uint32_t)t_ring[4];
            }
        }
        if (dbg & 4) nb = nbw0 = nbw1 = 0;          // experiment: no data movement (garbage tiles)
#ifdef ODP_CHECK
        {
            const long long wlo = -2LL * g.stride[0], whi = g.P + 2LL * g.stride[0];   // W: local planes + 2 halo planes
            auto chk_copy = [&](uint32_t d, const float *sp, uint32_t n, int code) {
                if (!n) return;
                const long long e = sp - W;
                ODP_CHK(e >= wlo && e + n / 4 <= whi, code, e, n);
                ODP_CHK(((uintptr_t)sp & 15) == 0 && (d & 15) == 0 && (n & 15) == 0, code + 1, (long long)(uintptr_t)sp, n);
                odp_chk_smem(d, n, code + 2);
            };
            chk_copy(dst, src, nb, 10);
            if (nbw0) chk_copy(smem_u32(slot + RMG), W + tt + t_ring[6], nbw0, 20);
            if (nbw1) chk_copy(smem_u32(slot + t_ring[5]), W + tt, nbw1, 30);
        }
#endif
        const uint32_t total = __reduce_add_sync(0xffffffffu, nb + nbw0 + nbw1);
        if (lane == 0) mbar_expect_tx(bar, total);
        __syncwarp();
        if (nb) tma_bulk_g2s_u32(dst, src, nb, bar);
        if (nbw0) tma_bulk_g2s_u32(smem_u32(slot + RMG), W + tt + t_ring[6], nbw0, bar);
        if (nbw1) tma_bulk_g2s_u32(smem_u32(slot + t_ring[5]), W + tt, nbw1, bar);
    };
    // per-warp side geometry (index and extent per side axis, read only on face columns) and the
    // marching axis' coordinate tables (x, cos, sin) staged once per launch
    int *wgeo = reinterpret_cast<int *>(smem + a.aux_off) + (tid >> 5) * 6;
    float *mtab = smem + a.aux_off + 96;
    if constexpr (PASS2) {
        if (((F::NEED_X | F::NEED_TRIG) >> MA) & 1)
            for (int jj = tid; jj < a.mtab_n; jj += blockDim.x) {
                if ((F::NEED_X >> MA) & 1) mtab[jj] = __ldg(g.tab + g.tab_off[MA] + jj);
                if ((F::NEED_TRIG >> MA) & 1) {
                    mtab[a.mtab_n + jj] = __ldg(g.tab + g.tab_off[MA] + g.Ng[MA] + jj);
                    mtab[2 * a.mtab_n + jj] = __ldg(g.tab + g.tab_off[MA] + 2 * g.Ng[MA] + jj);
                }
            }
    }
    auto load_march = [&](Pt &q, int jg) {            // coordinates of the marching axis at global index jg
        if (CT || a.mtab_n) {                        // (shape-specialised instances always stage it)
            if ((F::NEED_X >> MA) & 1) q.x[MA] = mtab[jg];
            if ((F::NEED_TRIG >> MA) & 1) { q.c[MA] = mtab[a.mtab_n + jg]; q.s[MA] = mtab[2 * a.mtab_n + jg]; }
        } else {
            load_axis<F>(g, q, MA, jg);
        }
    };

    if (tid == 0) {
        for (int b = 0; b < NST; ++b) {
            mbar_init(&tmab[b], 1);
#if ODP_MARCH_ECOUNT
            *reinterpret_cast<volatile unsigned int *>(&empty[b]) = 0u;   // plain release counter
#else
            mbar_init(&empty[b], nwc);
#endif
            mbar_init(&ubar[b], 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if ((tid >> 5) == nwc) {
        // ================= producer warp =================
        // Issues the copies of step sn as soon as step sn - NST released its buffers (every compute
        // warp arrived on empty), i.e. up to NST - 1 steps ahead of the slowest compute warp, and
        // nothing else: the ghost cells are formed by the compute warps in registers, so the only
        // serial work per step is the copy issue.  Units come from the launch's work counter in
        // order and are announced through a queue of NST entries (the units in flight on the whole
        // GPU stay a compact range of the L2-friendly work order).
        const int lane = tid & 31;
        int nu = 0;                                          // units announced to the compute warps
        auto grab = [&]() -> int {
            unsigned int v = 0;
            if (lane == 0) v = atomicAdd(wctr, 1u);
            v = __shfl_sync(0xffffffffu, v, 0);
            const int un = v < (unsigned)a.units ? (int)v : -1;
            if (lane == 0) {
                uq[nu % NST] = un;
                mbar_arrive(&ubar[nu % NST]);
            }
            ++nu;
            return un;
        };
        int ui = grab();
        int sn = 0;
        while (ui >= 0) {
            const MarchUnit U = march_unit<MA>(a, Nml, mlo, ui);
            make_table(U);
#if ODP_MARCH_LEANP
            // this lane's copy descriptor for the whole unit: only the marching offset, the stage and
            // the ring slot change from step to step (round 1's issue() re-derived everything from
            // the shared table every step, ~90 instructions + a REDUX on the producer's serial path)
            const long long colb = U.cbase - (long long)mlo * M;   // element offset of global marching index 0
            uint32_t d_nb = 0, d_w0 = 0, d_w1 = 0, d_dst = 0, d_d0 = 0, d_d1 = 0;
            long long d_src = 0, d_s0 = 0;
            const float *d_base = W;                        // source array of this lane's copy
            if (lane < NSS) {
                d_nb = t_snb[lane];
                d_src = colb + t_soff[lane];
                d_dst = smem_u32(side + lane * SSZ + MARCH_SMARG);
            } else if (lane - NSS <= R) {
                d_nb = (uint32_t)t_ring[1];
                d_src = colb + t_ring[0];
                d_dst = smem_u32(ring + t_ring[2]);
                d_w0 = (uint32_t)t_ring[3];
                d_w1 = (uint32_t)t_ring[4];
                d_s0 = colb + t_ring[6];
                d_d0 = smem_u32(ring + RMG);
                d_d1 = smem_u32(ring + t_ring[5]);
            } else if (XSC && lane - NSS - R - 1 < 2) {
                // pass 2's streamed operands: lane NSS+R+1 the target T, lane NSS+R+2 Vn (row block of
                // the step's tile, same element offsets as the centre tile)
                const int xl = lane - NSS - R - 1;
                if ((xs >> xl) & 1) {
                    d_nb = (uint32_t)U.nrow * N1 * 4;
                    d_src = colb + (long long)U.r0 * N1;
                    d_base = xl == 0 ? T : Vn;
                    d_dst = smem_u32(smem + a.xoff + (xl == 1 && (xs & 1) ? SSZ : 0) + MARCH_SMARG);
                }
            }
            if (dbg & 4) d_nb = d_w0 = d_w1 = 0;      // experiment: no data movement (garbage tiles)
            const uint32_t side_bytes = __reduce_add_sync(0xffffffffu, (lane < NSS || (XSC && lane > NSS + R)) ? d_nb : 0u);
            const uint32_t ring_bytes = (dbg & 4) ? 0u : (uint32_t)(t_ring[1] + t_ring[3] + t_ring[4]);
#endif
            for (int j = U.m0; j < U.m1; ++j, ++sn) {
                const int sr = sn - NST;                     // the step whose buffers step sn reuses
#if ODP_MARCH_ECOUNT
                if (sr >= 0) {       // the (sr / NST + 1)-th release of stage sr % NST: nwc arrivals each
                    const unsigned int want = (unsigned int)(sr / NST + 1) * (unsigned int)nwc;
                    const uint32_t ea = smem_u32(&empty[sr % NST]);
                    unsigned int have;
                    for (;;) {
                        asm volatile("ld.acquire.cta.shared::cta.u32 %0, [%1];" : "=r"(have) : "r"(ea) : "memory");
                        if ((int)(have - want) >= 0) break;
                        __nanosleep(ODP_MARCH_ECOUNT_NS);
                    }
                }
#else
                if (sr >= 0) mbar_wait_mode<ODP_MARCH_WAITP>(&empty[sr % NST], (uint32_t)((sr / NST) & 1));
#endif
#if ODP_MARCH_LEANP
                {
                    const int stg = sn % NST;
                    uint64_t *bar = &tmab[stg];
                    const int kb = j == U.m0 ? 0 : R;           // ring tiles j + kb .. j + klast
                    const int klast = min(R, U.m1 - 1 - j);
                    const uint32_t nring = klast >= kb ? (uint32_t)(klast - kb + 1) : 0u;
                    if (lane == 0) mbar_expect_tx(bar, side_bytes + nring * ring_bytes);
                    __syncwarp();
                    uint32_t n = 0, n0 = 0, n1 = 0, dd = 0, off = 0;
                    long long se = 0, mo = 0;
                    if (lane < NSS) {
                        n = d_nb;
                        dd = d_dst + (uint32_t)(stg * NSS * SSZ * 4);
                        se = d_src + (long long)j * M;
                    } else if (XSC && lane > NSS + R) {       // T / Vn (pass 2, LOW)
                        n = d_nb;
                        dd = d_dst + (uint32_t)(stg * a.xn * SSZ * 4);
                        se = d_src + (long long)j * M;
                    } else {
                        const int k = lane - NSS;
                        if (k >= kb && k <= klast) {
                            off = (uint32_t)(((sn + k) % RS) * RSZ * 4);
                            mo = (long long)(j + k) * M;
                            n = d_nb; n0 = d_w0; n1 = d_w1;
                            dd = d_dst + off;
                            se = d_src + mo;
                        }
                    }
#ifdef ODP_CHECK
                    {
                        const long long wlo = -2LL * g.stride[0], whi = g.P + 2LL * g.stride[0];
                        auto chk_copy = [&](uint32_t d, long long e, uint32_t nbytes, int code) {
                            if (!nbytes) return;
                            ODP_CHK(e >= wlo && e + nbytes / 4 <= whi, code, e, nbytes);
                            ODP_CHK(((uintptr_t)(W + e) & 15) == 0 && (d & 15) == 0 && (nbytes & 15) == 0, code + 1, e, nbytes);
                            odp_chk_smem(d, nbytes, code + 2);
                        };
                        if (XSC && lane > NSS + R) {          // T / Vn: the local slab [0, P)
                            if (n) {
                                ODP_CHK(se >= 0 && se + n / 4 <= g.P, 50, se, n);
                                ODP_CHK(((uintptr_t)(d_base + se) & 15) == 0 && (dd & 15) == 0 && (n & 15) == 0, 51, se, n);
                                odp_chk_smem(dd, n, 52);
                            }
                        } else {
                            chk_copy(dd, se, n, 10);
                        }
                        chk_copy(d_d0 + off, d_s0 + mo, n0, 20);
                        chk_copy(d_d1 + off, colb + mo, n1, 30);
                    }
#endif
                    if (n) tma_bulk_g2s_u32(dd, (XSC ? d_base : W) + se, n, bar);
                    if (n0) tma_bulk_g2s_u32(d_d0 + off, W + d_s0 + mo, n0, bar);
                    if (n1) tma_bulk_g2s_u32(d_d1 + off, W + colb + mo, n1, bar);
                }
#else
                issue(U, j, sn, j == U.m0 ? 0 : R);
#endif
#ifdef ODP_MARCH_PDELAY_NS             // experiment: a slower producer (is the copy issue on the critical path?)
                __nanosleep(ODP_MARCH_PDELAY_NS);
#endif
            }
            ui = grab();
        }
    } else {
        // ================= compute warps =================
        int it = 0;                                      // step counter of this CTA (buffer / phase)
        int rs0 = 0;                                     // it % RS (ring slot of the centre tile)
        int st0 = 0, sph = 0;                            // it % NST (stage), (it / NST) & 1
        const uint32_t rb_s = smem_u32(ring + toff);    // this thread's nodes in ring slot 0 (bytes)
        const uint32_t sb_s = smem_u32(side + sloc);    // ... in side slot 0 of stage 0
        const uint32_t xb_s = smem_u32(smem + a.xoff + sloc);   // ... in the T / Vn slots of stage 0 (pass 2)
        const uint32_t xvo = (xs & 1) ? (uint32_t)SSZ * 4u : 0u;  // Vn's slot after T's
        const uint32_t lof = 4u * (uint32_t)loff, rof = 4u * (uint32_t)roff;
        int rsw = R;                                     // (it + R) % RS: ring slot of the entering window tile
        for (int k = 0;; ++k) {
            mbar_wait_sleep(&ubar[k % NST], (uint32_t)((k / NST) & 1));
            const int u = uq[k % NST];
            if (u < 0) break;
            const MarchUnit U = march_unit<MA>(a, Nml, mlo, u);
            const int m0 = U.m0, m1 = U.m1;
            const bool act = lrow < U.nrow && tid < a.nthr;
            const int grow = U.r0 + lrow;                 // global row of this thread
            const bool rface = !a.per2 && (grow < R || grow > N2 - 1 - R);   // ghost rows in the row window
            int oid[NSA], oN[NSA];
            side_geom(U.col, oid, oN);
            uint32_t fmask = 0;                               // bit o: the column is within R of a face of side axis o
#pragma unroll
            for (int o = 0; o < MA; ++o)
                if (!g.per[o] && (oid[o] < R || oid[o] > oN[o] - 1 - R)) fmask |= 1u << o;
            __syncwarp();
            if ((tid & 31) == 0)
#pragma unroll
                for (int o = 0; o < MA; ++o) { wgeo[2 * o] = oid[o]; wgeo[2 * o + 1] = oN[o]; }
            __syncwarp();
            Pt qrow;
            if constexpr (PASS2) {
#pragma unroll
                for (int o = 0; o < MA; ++o) load_axis<F>(g, qrow, o, oid[o]);
                load_axis<F>(g, qrow, NDIM - 2, min(grow, N2 - 1));
            }
            const float *cb = W + U.cbase + grow * N1 + qc0;   // this thread's nodes at local marching index 0

            // ---- preamble: the window around m0 and the carried edge m0 - 1/2 (registers) ----
            float2 win[R + 1];
            float2 dd0, mL, dL;
            if (act) {
                float2 x[2 * R + 1];
#pragma unroll
                for (int k = -R; k <= R; ++k) {
                    ODP_CHK(cb + (long long)mloc(m0 + k) * M - W >= -2LL * g.stride[0] &&
                            cb + (long long)mloc(m0 + k) * M - W + 2 <= g.P + 2LL * g.stride[0], 40, m0 + k, 0);
                    x[k + R] = __ldg(reinterpret_cast<const float2 *>(cb + (long long)mloc(m0 + k) * M));
                }
                if (!mper && (m0 < R || m0 > Nm - 1 - R)) fix_ghosts2<R>(x, m0, Nm);
#pragma unroll
                for (int k = 0; k < R; ++k) win[k] = x[R + k];
                if constexpr (R == 2) {
                    dd0 = d2p(x[1], x[2], x[3]);
                    mL = pick2(d2p(x[0], x[1], x[2]), dd0);
                    dL = sub2(x[2], x[1]);
                    if constexpr (!PASS2) inc_val(fma2(f2s(0.5f), mL, dL), mn[MA], mx[MA]);   // D-_{m0}
                } else {
                    dL = sub2(x[1], x[0]);
                    if constexpr (!PASS2) inc_val(dL, mn[MA], mx[MA]);
                }
            }

            float2 vnv = f2s(0.f), ttv = f2s(0.f);         // Vn / target of the current step (pass 2), loaded a step ahead
            if constexpr (PASS2 && !LDSTEP) {              // (unless staged by TMA with the step's tiles: xs)
                if (act) {
                    const long long gi0 = U.cbase + (long long)(m0 - mlo) * M + grow * N1 + qc0;
                    ODP_CHK(gi0 >= 0 && gi0 + 2 <= g.P, 41, gi0, g.P);
                    if (kind == STAGE_RK2 && !(xs & 2)) vnv = *reinterpret_cast<const float2 *>(Vn + gi0);
                    if (brt && kind != STAGE_RK1 && !(xs & 1)) ttv = __ldg(reinterpret_cast<const float2 *>(T + gi0));
                }
            }

            long long gi = U.cbase + (long long)(m0 - mlo) * M + grow * N1 + qc0;   // element of node 0 (this step)
#if ODP_MARCH_UNROLL == 2
#pragma unroll 2
#elif ODP_MARCH_UNROLL == 3
#pragma unroll 3
#endif
            for (int jg = m0; jg < m1; ++jg, ++it, gi += M) {
                // window value entering at this step: v_{j+R} (ring inside the segment, else global / ghost)
                const int kin = jg + R;
                const bool in_ring = kin < m1;
                if constexpr (PASS2 && LDSTEP) {           // this step's Vn / target, before the copy wait
                    if (act) {
                        ODP_CHK(gi >= 0 && gi + 2 <= g.P, 41, gi, g.P);
                        if (kind == STAGE_RK2 && !(xs & 2)) vnv = *reinterpret_cast<const float2 *>(Vn + gi);
                        if (brt && kind != STAGE_RK1 && !(xs & 1)) ttv = __ldg(reinterpret_cast<const float2 *>(T + gi));
                    }
                }

                float2 vin = f2s(0.f);
                if (act && !in_ring) {
                    if (mper || kin < Nm) {
                        ODP_CHK(cb + (long long)mloc(kin) * M - W >= -2LL * g.stride[0] &&
                                cb + (long long)mloc(kin) * M - W + 2 <= g.P + 2LL * g.stride[0], 43, kin, 0);
                        vin = __ldg(reinterpret_cast<const float2 *>(cb + (long long)mloc(kin) * M));
                    } else {                                  // beyond the high face: ghost (A12)
                        const float2 e = __ldg(reinterpret_cast<const float2 *>(cb + (long long)(Nm - 1 - mlo) * M));
                        const float2 in = __ldg(reinterpret_cast<const float2 *>(cb + (long long)(Nm - 2 - mlo) * M));
                        vin = ghost2(e, in, (float)(kin - Nm + 1));
                    }
                }
#if ODP_MARCH_RELAY
                // the step's copies landed: compute warp 0 alone waits on the transaction barrier (its
                // waits wake on every copy's completion), then releases the other compute warps
                // through a hardware named barrier, where waiting warps take no issue slots
                if (tid < 32) mbar_wait_sleep(&tmab[st0], (uint32_t)sph);
                asm volatile("bar.sync 1, %0;" ::"r"(nwc * 32) : "memory");
#else
                mbar_wait_sleep(&tmab[st0], (uint32_t)sph);        // the step's copies landed
#endif
                const uint32_t rcs = rb_s + (uint32_t)(rs0 * RSZ * 4);      // this thread's nodes in the centre tile
                const uint32_t sbs = sb_s + (uint32_t)(st0 * NSS * SSZ * 4); // ... in side slot 0

                if (act && !(dbg & 2)) {
                    if (in_ring) vin = lds2(rb_s + (uint32_t)(rsw * RSZ * 4));
                    win[R] = vin;
                    const float2 v0 = win[0];
                    Pt q0;
                    if constexpr (PASS2) {
                        q0 = qrow;
                        load_march(q0, jg);
                    }
                    float2 acc = f2s(0.f), dis = f2s(0.f);
                    float2 pv[F::SEPARABLE ? 1 : NDIM];     // costate of the node pair (non-separable H)
                    auto node_pts = [&](Pt &a0, Pt &a1) {
                        a0 = q0; a1 = q0;
                        a0.x[NDIM - 1] = qcv[0].x[NDIM - 1]; a0.c[NDIM - 1] = qcv[0].c[NDIM - 1]; a0.s[NDIM - 1] = qcv[0].s[NDIM - 1];
                        a1.x[NDIM - 1] = qcv[1].x[NDIM - 1]; a1.c[NDIM - 1] = qcv[1].c[NDIM - 1]; a1.s[NDIM - 1] = qcv[1].s[NDIM - 1];
                    };
                    auto terms = [&](int d, float2 uu, float2 ww) {
                        Pt a0, a1;
                        node_pts(a0, a1);
                        axis_terms(f, d, a0, a1, hih[d], uu, ww, acc, dis, pv);
                    };
                    // one-sided derivatives of a full window x[0..2R] (classic): h D-, h D+
                    auto classic = [&](const float2 *x, float2 &uu, float2 &ww, float2 &mr, float2 &d1r) {
                        if constexpr (R == 2) {
                            const float2 dm = d2p(x[0], x[1], x[2]), dc = d2p(x[1], x[2], x[3]), dp = d2p(x[2], x[3], x[4]);
                            uu = fma2(f2s(0.5f), pick2(dm, dc), sub2(x[2], x[1]));
                            mr = pick2(dc, dp);
                            d1r = sub2(x[3], x[2]);
                            ww = fma2(f2s(-0.5f), mr, d1r);
                        } else {
                            uu = sub2(x[1], x[0]);
                            ww = sub2(x[2], x[1]);
                            mr = ww; d1r = ww;
                        }
                    };

                    // ---- marching axis: carried edge j-1/2, new edge j+1/2 ----
                    if constexpr (R == 2) {
                        const float2 dd1 = d2p(win[0], win[1], win[2]);      // d2_{j+1}
                        const float2 d1 = sub2(win[1], win[0]);
                        if constexpr (PASS2) {
                            const float2 m = pick2(dd0, dd1);
                            terms(MA, fma2(f2s(0.5f), mL, dL), fma2(f2s(-0.5f), m, d1));
                            mL = m;
                        } else {
                            if (!mper && jg == Nm - 1) inc_val(fma2(f2s(-0.5f), pick2(dd0, dd1), d1), mn[MA], mx[MA]);
                            else inc_edge(amin2(dd0, dd1), d1, mn[MA], mx[MA]);
                        }
                        dd0 = dd1; dL = d1;
                    } else {
                        const float2 d1 = sub2(win[1], win[0]);
                        if constexpr (PASS2) terms(MA, dL, d1);
                        else inc_val(d1, mn[MA], mx[MA]);
                        dL = d1;
                    }

                    // ---- side axes (CTA-uniform faces), neighbours from the side slots ----
#pragma unroll
                    for (int o = 0; o < MA; ++o) {
                        const uint32_t so = sbs + (uint32_t)(o * 2 * R * SSZ * 4);
                        const bool of = (fmask >> o) & 1u;
                        if (PASS2 || of) {
                            float2 x[2 * R + 1];
#pragma unroll
                            for (int k = -R; k <= R; ++k)
                                x[k + R] = k == 0 ? v0 : lds2(so + (uint32_t)((k < 0 ? k + R : k + R - 1) * SSZ * 4));
                            if (of) fix_ghosts2<R>(x, wgeo[2 * o], wgeo[2 * o + 1]);
                            float2 uu, ww, mr, d1r;
                            classic(x, uu, ww, mr, d1r);
                            if constexpr (PASS2) {
                                terms(o, uu, ww);
                            } else {
                                inc_val(uu, mn[o], mx[o]);
                                inc_val(ww, mn[o], mx[o]);
                                if (R == 2 && wgeo[2 * o] + 1 <= wgeo[2 * o + 1] - 1) inc_val(fma2(f2s(0.5f), mr, d1r), mn[o], mx[o]);   // D-_{i+1}
                            }
                        } else {
                            // pass 1, interior: the node's upper edge i+1/2 (both sides)
                            if constexpr (R == 2) {
                                const float2 s1 = lds2(so + (uint32_t)(1 * SSZ * 4));
                                const float2 s2 = lds2(so + (uint32_t)(2 * SSZ * 4));
                                const float2 s3 = lds2(so + (uint32_t)(3 * SSZ * 4));
                                inc_edge(amin2(d2p(s1, v0, s2), d2p(v0, s2, s3)), sub2(s2, v0), mn[o], mx[o]);
                            } else {
                                inc_val(sub2(lds2(so + (uint32_t)(1 * SSZ * 4)), v0), mn[o], mx[o]);
                            }
                        }
                    }

                    // ---- in-plane rows (axis n-2): rows beyond a non-periodic face are ghosts (A12) ----
                    {
                        float2 x[2 * R + 1];
                        if (!PASS2 && !rface) {
                            // pass 1, interior row: the node's upper edge r+1/2 (both sides)
                            const uint32_t rs = (uint32_t)(N1 * 4);
                            if constexpr (R == 2) {
                                const float2 s1 = lds2(rcs - rs), s2 = lds2(rcs + rs), s3 = lds2(rcs + 2 * rs);
                                inc_edge(amin2(d2p(s1, v0, s2), d2p(v0, s2, s3)), sub2(s2, v0), mn[NDIM - 2], mx[NDIM - 2]);
                            } else {
                                inc_val(sub2(lds2(rcs + rs), v0), mn[NDIM - 2], mx[NDIM - 2]);
                            }
                        } else if (!rface) {
#pragma unroll
                            for (int k = -R; k <= R; ++k) x[k + R] = k == 0 ? v0 : lds2(rcs + (uint32_t)(k * N1 * 4));
                        } else {
#pragma unroll
                            for (int k = -R; k <= R; ++k) {
                                const int rr = min(max(grow + k, 0), N2 - 1) - grow;
                                x[k + R] = k == 0 ? v0 : lds2(rcs + (uint32_t)(rr * N1 * 4));
                            }
                            // ghost rows (A12) from the face row e and the next inner row
                            if (grow == 0) {
                                x[R - 1] = ghost2(v0, x[R + 1], 1.f);
                                if (R == 2) x[0] = ghost2(v0, x[R + 1], 2.f);
                            } else if (R == 2 && grow == 1) {
                                x[0] = ghost2(x[1], v0, 1.f);
                            }
                            if (grow == N2 - 1) {
                                x[R + 1] = ghost2(v0, x[R - 1], 1.f);
                                if (R == 2) x[2 * R] = ghost2(v0, x[R - 1], 2.f);
                            } else if (R == 2 && grow == N2 - 2) {
                                x[2 * R] = ghost2(x[3], v0, 1.f);
                            }
                        }
                        if (PASS2 || rface) {
                            float2 uu, ww, mr, d1r;
                            classic(x, uu, ww, mr, d1r);
                            if constexpr (PASS2) {
                                terms(NDIM - 2, uu, ww);
                            } else {       // face row: D-, D+ and, below the last row, both sides of edge r+1/2
                                inc_val(uu, mn[NDIM - 2], mx[NDIM - 2]);
                                inc_val(ww, mn[NDIM - 2], mx[NDIM - 2]);
                                if (R == 2 && grow + 1 <= N2 - 1) inc_val(fma2(f2s(0.5f), mr, d1r), mn[NDIM - 2], mx[NDIM - 2]);
                            }
                        }
                    }

                    // ---- in-plane columns (axis n-1): left / right pairs (tile or ghost table) ----
                    {
                        float2 lp = lds2(rcs + lof);
                        float2 rp = lds2(rcs + rof);
                        if (gfirst) lp = f2(ghost(v0.x, v0.y, 2.f), ghost(v0.x, v0.y, 1.f));
                        if (glast) rp = f2(ghost(v0.y, v0.x, 1.f), ghost(v0.y, v0.x, 2.f));
                        float2 uu, ww;
                        if constexpr (!PASS2 && R == 2) {
                            // edges c+1/2 (both sides) and c+3/2 (both sides, or D+_{c+1} on the last pair
                            // of a non-periodic row); D-_c on the first pair (the face edge c-1/2)
                            const float d0 = d2s(lp.y, v0.x, v0.y), d1 = d2s(v0.x, v0.y, rp.x), d2 = d2s(v0.y, rp.x, rp.y);
                            const float fb = v0.y - v0.x, fc = rp.x - v0.y;
                            const float2 lo = fma2(f2s(-0.5f), f2(fminf(fabsf(d0), fabsf(d1)), fminf(fabsf(d1), fabsf(d2))), f2(fb, fc));
                            float2 hi = fma2(f2s(0.5f), f2(fminf(fabsf(d0), fabsf(d1)), fminf(fabsf(d1), fabsf(d2))), f2(fb, fc));
                            if (glast) hi.y = fmaf(-0.5f, pick1(d1, d2), fc);
                            float l2 = glast ? hi.y : lo.y;
                            mn[NDIM - 1] = min3f(mn[NDIM - 1], lo.x, l2);
                            mx[NDIM - 1] = max3f(mx[NDIM - 1], hi.x, hi.y);
                            if (gfirst) inc_s(fmaf(0.5f, pick1(d2s(lp.x, lp.y, v0.x), d0), v0.x - lp.y), mn[NDIM - 1], mx[NDIM - 1]);
                        } else if constexpr (R == 2) {
                            // columns -2 -1 | 0 1 | 2 3 ; second differences at -1 0 1 2 ; edges -1/2, 1/2, 3/2
                            const float dm1 = d2s(lp.x, lp.y, v0.x), d0 = d2s(lp.y, v0.x, v0.y);
                            const float d1 = d2s(v0.x, v0.y, rp.x), d2 = d2s(v0.y, rp.x, rp.y);
                            const float ea = pick1(dm1, d0), eb = pick1(d0, d1), ec = pick1(d1, d2);
                            const float fa = v0.x - lp.y, fb = v0.y - v0.x, fc = rp.x - v0.y;
                            uu = fma2(f2s(0.5f), f2(ea, eb), f2(fa, fb));
                            ww = fma2(f2s(-0.5f), f2(eb, ec), f2(fb, fc));
                        } else {
                            uu = f2(v0.x - lp.y, v0.y - v0.x);
                            ww = f2(v0.y - v0.x, rp.x - v0.y);
                        }
                        if constexpr (PASS2) terms(NDIM - 1, uu, ww);
                        else if constexpr (R == 1) {
                            inc_val(ww, mn[NDIM - 1], mx[NDIM - 1]);          // D+_c, D+_{c+1} (= D-_{c+1}, D-_{c+2})
                            if (gfirst) inc_s(uu.x, mn[NDIM - 1], mx[NDIM - 1]);   // D-_0
                        }
                    }

                    if constexpr (PASS2) {
                        if constexpr (!F::SEPARABLE) {             // H = p.f(x, u*, d*) per node (Alg. 2 l.154-156)
                            Pt a0, a1;
                            node_pts(a0, a1);
                            float p0[NDIM], p1[NDIM];
#pragma unroll
                            for (int d = 0; d < NDIM; ++d) { p0[d] = pv[d].x; p1[d] = pv[d].y; }
                            acc = f2(f.ham(a0, p0), f.ham(a1, p1));
                        }
                        if (xs) {                            // staged operands of this step
                            const uint32_t xs0 = xb_s + (uint32_t)(st0 * a.xn * SSZ * 4);
                            if (xs & 1) ttv = lds2(xs0);
                            if (xs & 2) vnv = lds2(xs0 + xvo);
                        }
                        const float2 L = add2(ham_fin2(f, acc), dis);
                        float2 v = fma2(f2s(dt), L, v0);                        // W + dt L
                        if (kind == STAGE_RK2) v = mul2(f2s(0.5f), add2(vnv, v));  // (Vn + V2)/2 (A10)
                        if (brt && kind != STAGE_RK1) v = f2(fminf(v.x, ttv.x), fminf(v.y, ttv.y));
                        ODP_CHK(gi >= 0 && gi + 2 <= g.P, 42, gi, g.P);
                        *reinterpret_cast<float2 *>(out + gi) = v;
                        mabs = max3nan(mabs, fabsf(v.x), fabsf(v.y));   // output guard (single-pass solves)
                        if (!LDSTEP && jg + 1 < m1) {         // the next step's Vn / target
                            if (kind == STAGE_RK2 && !(xs & 2)) vnv = *reinterpret_cast<const float2 *>(Vn + gi + M);
                            if (brt && kind != STAGE_RK1 && !(xs & 1)) ttv = __ldg(reinterpret_cast<const float2 *>(T + gi + M));
                        }
                    } else {
                        mabs = max3nan(mabs, fabsf(v0.x), fabsf(v0.y));
                    }
#pragma unroll
                    for (int k = 0; k < R; ++k) win[k] = win[k + 1];
                }
                __syncwarp();
#if ODP_MARCH_ECOUNT
                // this warp is done with the step's buffers: a plain shared-memory release counter (an
                // mbarrier arrive would wake every warp sleeping on the copy barriers, 15 times a step)
                if ((tid & 31) == 0)
                    asm volatile("red.release.cta.shared::cta.add.u32 [%0], 1;" ::"r"(smem_u32(&empty[st0])) : "memory");
#else
                if ((tid & 31) == 0) mbar_arrive(&empty[st0]);   // this warp is done with the step's buffers
#endif
                if (++rs0 == RS) rs0 = 0;
                if (++rsw == RS) rsw = 0;
                if (++st0 == NST) { st0 = 0; sph ^= 1; }
            }
        }
    }
    if constexpr (!PASS2) {
#pragma unroll
        for (int d = 0; d < NDIM; ++d) { mn[d] *= g.inv_dx[d]; mx[d] *= g.inv_dx[d]; }   // h D -> D
        const int nan = mabs != mabs;
        block_reduce_range<NDIM>(mn, mx, nan ? 0.f : mabs, nan, partials);
    } else if (partials) {
        // single-pass solves: the guard of A19 on this stage's OUTPUT -- the next
        // stage's input -- in place of pass 1 (the range entries stay neutral)
        const int nan = mabs != mabs;
        block_reduce_range<NDIM>(mn, mx, nan ? 0.f : mabs, nan, partials);
    }
}

// ------------------------------------------------------------------------------------------------
// host side
// ------------------------------------------------------------------------------------------------
typedef void (*march_fn)(MarchArgs, GridDev, const float *, const float *, const float *, float *, float *,
                         const DevState *, FParams, int, int);

// The generic (runtime-geometry) instance plus shape-specialised ones for the tile shapes of the
// BASELINE.json configs (c1 36x(21), c2 60x(15), c3 40x(20), c4 30x(30), c5 48x(16); the row
// block B in parentheses is what march_plan picks for those shapes).  Any other grid runs the
// generic instance -- same code, geometry from MarchArgs.
struct MarchInst {
    int n1 = 0, b = 0, nst = 2;
    march_fn pass1 = nullptr, pass2 = nullptr;
    march_fn pass2k[3] = {nullptr, nullptr, nullptr};   // per stage kind (null: pass2 with the runtime kind)
};
constexpr int MARCH_MAX_INST = 12;
struct MarchFnsAll {
    march_fn pass1 = nullptr, pass2 = nullptr;   // generic
    MarchInst inst[MARCH_MAX_INST];
    int ninst = 0;
};
struct MarchFns {
    march_fn pass1 = nullptr, pass2 = nullptr;
    march_fn pass2k[3] = {nullptr, nullptr, nullptr};
    int specialised = 0;
};
struct MarchPlan {
    MarchArgs a;
    int block = 0, grid = 0;
    size_t smem = 0;
    bool t_ok = false;    // the target is 16-B aligned (TMA source)
    size_t smem_noxs = 0; // dynamic shared memory without the T / Vn staging slots
};

template <class F, int NDIM, int R, int CN1, int CB, int NST = 2, int LBT = MARCH_MAXT1, int LBM = ODP_MARCH_MINB1>
void march_add(MarchFnsAll &t) {
    if constexpr (NDIM >= 3) {
        MarchInst &m = t.inst[t.ninst++];
        m.n1 = CN1; m.b = CB; m.nst = NST;
        m.pass1 = k_march<F, NDIM, R, 1, false, CN1, CB, NST, LBT, LBM>;
        m.pass2 = k_march<F, NDIM, R, 1, true, CN1, CB, NST, LBT, LBM>;
#if ODP_MARCH_KINDS
        if constexpr (R == 2) {      // MEDIUM: the RK stage 1 launch carries no Vn / target code at all
            m.pass2k[STAGE_RK1] = k_march<F, NDIM, R, 1, true, CN1, CB, NST, LBT, LBM, STAGE_RK1>;
            m.pass2k[STAGE_RK2] = k_march<F, NDIM, R, 1, true, CN1, CB, NST, LBT, LBM, STAGE_RK2>;
        }
#endif
    }
}

template <class F, int NDIM, int R>
MarchFnsAll march_fns() {
    MarchFnsAll t;
    if constexpr (NDIM >= 3) {
        t.pass1 = k_march<F, NDIM, R, 1, false>;
        t.pass2 = k_march<F, NDIM, R, 1, true>;
        if constexpr (std::is_same<F, FDoubleInt6D>::value) {     // c4 (30^6), c5 (64 x 48^5)
            march_add<F, NDIM, R, 30, 30, 2>(t);
#ifdef ODP_MARCH_EXPERIMENTS       // register budget vs warps per SM (tried and not kept)
            if constexpr (R == 2) {
                march_add<F, NDIM, R, 30, 30, 4, 512, 1>(t);     // 1 CTA/SM, no spills, deep pipeline
                march_add<F, NDIM, R, 30, 10, 3, 192, 4>(t);     // 4 CTAs/SM, 80 registers
                march_add<F, NDIM, R, 30, 10, 2, 192, 4>(t);
            }
#endif
            march_add<F, NDIM, R, 48, 16, 2>(t);
            if constexpr (R == 1) march_add<F, NDIM, R, 48, 16, 4>(t);   // c5 LOW
#ifdef ODP_MARCH_XINST             // smaller row blocks: 3 CTAs/SM for c5 LOW (ODP_MARCH_B=12 / 8)
            if constexpr (R == 1) { march_add<F, NDIM, R, 48, 12, 4>(t); march_add<F, NDIM, R, 48, 8, 4>(t); }
#endif
        } else if constexpr (std::is_same<F, FCar5D>::value && R == 2) {   // c3
            march_add<F, NDIM, R, 40, 20, 2>(t);
            march_add<F, NDIM, R, 40, 20, 3>(t);
        } else if constexpr (std::is_same<F, FCar4D>::value && R == 1) {   // c2
            march_add<F, NDIM, R, 60, 15, 2>(t);
            march_add<F, NDIM, R, 60, 15, 4>(t);
        } else if constexpr (std::is_same<F, FDubins3D>::value && R == 1) { // c1
            march_add<F, NDIM, R, 36, 21, 2>(t);
            march_add<F, NDIM, R, 36, 21, 3>(t);
        }
    }
    return t;
}

// Whether the march family covers this grid (and the alignment of the arrays it vector-loads).
inline bool march_plan(const GridDev &g, int R, const MarchFnsAll &all, const void *T, const void *W,
                       MarchFns *fns, MarchPlan *p) {
    if (g.n < 3 || !all.pass1) return false;
    const int N2 = g.N[g.n - 2], N1 = g.N[g.n - 1];
    const long long M = (long long)N2 * N1;
    if (N2 < 2 * R + 1 || N1 < 2 * R || N1 % 2) return false;
    if (M % 4) return false;                                     // tile bases 16-B aligned
    if (g.per[g.n - 2] && (R * N1) % 4) return false;             // periodic halo rows copied exactly
    if (T && ((uintptr_t)T % 8)) return false;
    if ((uintptr_t)W % 16) return false;
    const int MA = g.n - 3;
    const int NSS = 2 * R * MA;
    const int QR = N1 / 2;
    // rows per block: among the B (B N1 % 4 == 0 unless B = N2, <= 512 threads) whose shared
    // memory leaves room for 2 CTAs per SM (else 1), the one wasting the fewest rows in the last
    // (ragged) block, the larger on ties
    // rows per block B and pipeline depth NST: the deepest pipeline (NST = 4, 3, 2) of a compiled
    // instance whose shared memory still leaves room for 2 CTAs per SM; B among those that fit,
    // the one wasting the fewest rows in the last (ragged) block, the larger on ties.  NST > 2
    // exists only as shape-specialised instances; the generic instance runs NST = 2.
    const bool generic_only = getenv("ODP_MARCH_GENERIC") != nullptr;
    int nst_env = 0, b_env = 0;
    if (const char *env = getenv("ODP_MARCH_NST")) nst_env = std::min(4, std::max(2, atoi(env)));
    if (const char *env = getenv("ODP_MARCH_B")) b_env = atoi(env);
    const bool one_cta = getenv("ODP_MARCH_1CTA") != nullptr;
    auto pick_b = [&](int nst, int cap) {
        int bb = 0, best_waste = 1 << 30;
        for (int B = std::min(N2, (MARCH_MAXT1 - 32) / QR); B >= 1; --B) {
            if (B != N2 && (B * N1) % 4) continue;
            if (geo_smem_bytes(R, N1, B, NSS, nst) > cap) continue;
            const int waste = ((N2 + B - 1) / B) * B - N2;
            if (waste < best_waste) { best_waste = waste; bb = B; }
        }
        if (b_env >= 1 && b_env <= N2 && b_env * QR + 32 <= MARCH_MAXT1 && (b_env == N2 || (b_env * N1) % 4 == 0)) bb = b_env;
        return bb;
    };
    // shape-specialised instances read the marching coordinate table from shared memory only
    const bool mtab_ok = g.N[g.n - 3] <= 1024 && (g.n - 3 != 0 || g.Ng0 <= 1024);
    auto has_inst = [&](int B, int nst) {
        if (generic_only) return nst == 2;
        for (int i = 0; i < all.ninst; ++i)
            if (all.inst[i].n1 == N1 && all.inst[i].b == B && all.inst[i].nst == nst) return mtab_ok;
        return nst == 2;
    };
    int best = 0, nst = 2;
    for (int pass = one_cta ? 1 : 0; pass < 2 && !best; ++pass) {
        const int cap = pass == 0 ? 113 * 1024 : 226 * 1024;
        for (int cand = nst_env ? nst_env : 4; cand >= 2 && !best; --cand) {
            const int B = pick_b(cand, cap);
            if (B && has_inst(B, cand)) { best = B; nst = cand; }
            if (nst_env) break;
        }
    }
    if (!best) return false;
    fns->pass1 = all.pass1;
    fns->pass2 = all.pass2;
    fns->specialised = 0;
    for (int i = 0; i < all.ninst && !generic_only && mtab_ok; ++i)
        if (all.inst[i].n1 == N1 && all.inst[i].b == best && all.inst[i].nst == nst) {
            fns->pass1 = all.inst[i].pass1;
            fns->pass2 = all.inst[i].pass2;
            for (int k = 0; k < 3; ++k) fns->pass2k[k] = all.inst[i].pass2k[k];
            fns->specialised = 1;
        }
    MarchArgs &a = p->a;
    a.M = (int)M; a.N2 = N2; a.N1 = N1;
    a.per2 = g.per[g.n - 2]; a.per1 = g.per[g.n - 1];
    a.B = best;
    a.nrb = (N2 + best - 1) / best;
    a.nthr = best * QR;
    a.RSZ = geo_rsz(R, N1, best);
    a.SSZ = geo_ssz(N1, best);
    a.rmarg = geo_rmarg(R, N1);
    a.side_off = geo_side_off(R, N1, best, nst);
    a.bar_off = geo_bar_off(R, N1, best, NSS, nst);
    a.tab_off = a.bar_off + 36;                     // 2 NST + R + NST + NST <= 18 mbarriers (144 B)
    a.aux_off = a.tab_off + 112;                    // copy table (64 + 32 + 8 + 4 floats) rounded
    {
        const int NmG = MA == 0 ? g.Ng0 : g.N[MA];
        a.mtab_n = NmG <= 1024 ? NmG : 0;
    }
    for (int o = 0; o < 3; ++o) a.sn[o] = o < MA ? g.N[o] : 1;
    a.b1 = 1;
    if (MA == 3) {
        int want = 3;                               // c4 sweep (ODP_MARCH_B1 = 1..30): 3 best, +1.7 % over 6
        if (const char *env = getenv("ODP_MARCH_B1")) want = std::max(1, atoi(env));
        for (int b = std::min(want, g.N[1]); b >= 1; --b)
            if (g.N[1] % b == 0) { a.b1 = b; break; }
    }
    const int Nm = g.N[MA];
    long long ncols = 1;
    for (int o = 0; o < MA; ++o) ncols *= g.N[o];
    const long long cols_rb = ncols * a.nrb;
    a.ncols = (int)std::min<long long>(ncols, 1LL << 30);
    a.K = Nm;
    // few columns: split the marching axis into segments, ~6 units per SM (c2 sweep of ODP_MARCH_K:
    // 20 best, 1.43e11 vs 1.36e11 at the ~8 per SM segment length 15 and 1.20e11 unsegmented)
    if (cols_rb < 148LL * 4) a.K = std::max(4, Nm / (int)std::max<long long>(1, (148 * 6) / cols_rb));

    if (const char *env = getenv("ODP_MARCH_K")) a.K = std::max(1, atoi(env));
    a.K = std::min(a.K, Nm);
    a.nseg = (Nm + a.K - 1) / a.K;
    if (cols_rb * a.nseg > (1LL << 31) - 1) return false;
    a.units = (int)(cols_rb * a.nseg);
    a.dbg = 0;
#ifdef ODP_MARCH_EXPERIMENTS       // timing experiments only: never in the production build (wrong results)
    if (const char *env = getenv("ODP_MARCH_DBG")) a.dbg = atoi(env);
#endif
    a.i0map = 0; a.i0r = 0; a.s0n = a.sn[0];
    a.wslot = 0;                                    // pass 2 launches use slot 1 (march_pass2)
    p->block = ((a.nthr + 31) / 32) * 32 + 32;      // compute warps + the producer warp
    p->smem = (size_t)(a.aux_off + 96 + 3 * a.mtab_n) * 4;
    p->smem = std::max(p->smem, (size_t)geo_smem_bytes(R, N1, best, NSS, nst));
    // pass 2's streamed operands (target T, Vn of RK stage 2) staged by TMA with the step's tiles:
    // as many slots per stage (0..2) as the shared memory of the chosen occupancy leaves room for
    // (ODP_MARCH_XS = 0 keeps them as per-thread global loads one step ahead, the round-1 path)
    a.xs = 0;
    p->smem_noxs = p->smem;
    a.xoff = (int)((p->smem / 4 + 31) / 32 * 32);   // 128-B aligned
    a.xn = 0;
    {
        // (march_prepare drops the slots again if, with the static shared memory, they cost a CTA/SM)
        const size_t cap = (!one_cta && geo_smem_bytes(R, N1, best, NSS, nst) <= 113 * 1024) ? 113 * 1024 : 226 * 1024;
        int want = ODP_MARCH_LEANP ? 2 : 0;
        if (const char *env = getenv("ODP_MARCH_XS")) want = std::min(want, std::max(0, atoi(env)));
        if (R != 1) want = 0;
        for (int xn = want; xn >= 1; --xn)
            if ((size_t)(a.xoff + xn * nst * a.SSZ) * 4 <= cap) { a.xn = xn; break; }
        if (a.xn) p->smem = (size_t)(a.xoff + a.xn * nst * a.SSZ) * 4;
    }
    p->t_ok = T && ((uintptr_t)T % 16) == 0;
    p->grid = 0;
    return true;
}

inline int march_prepare(const MarchFns &t, MarchPlan &p, int nsm) {
    int occ1 = 0, occ2 = 0;
    for (int attempt = 0; attempt < 2; ++attempt) {
        for (march_fn fn : {t.pass1, t.pass2, t.pass2k[0], t.pass2k[1], t.pass2k[2]}) {
            if (fn && cudaFuncSetAttribute((const void *)fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p.smem) != cudaSuccess)
                return 1;
        }
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ1, (const void *)t.pass1, p.block, p.smem) != cudaSuccess) return 1;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ2, (const void *)t.pass2, p.block, p.smem) != cudaSuccess) return 1;
        // the T / Vn staging slots must not cost a CTA per SM (static shared memory counts too)
        if (p.a.xn == 0 || p.smem_noxs == p.smem) break;
        int occ0 = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ0, (const void *)t.pass2, p.block, p.smem_noxs) != cudaSuccess) return 1;
        if (occ0 <= std::min(occ1, occ2)) break;
        p.a.xn = 0;
        p.smem = p.smem_noxs;
    }
    const int occ = std::max(1, std::min(occ1, occ2));
    p.grid = std::min(p.a.units, nsm * occ);
    if (getenv("ODP_MARCH_VERBOSE"))
        fprintf(stderr, "march plan: B=%d threads=%d smem=%zu occupancy=%d/%d grid=%d units=%d K=%d specialised=%d\n",
                p.a.B, p.block, p.smem, occ1, occ2, p.grid, p.a.units, p.a.K, t.specialised);
    return 0;
}

inline void march_pass1(const MarchFns &t, const MarchPlan &p, const GridDev &g, const float *W, float *partials,
                        const DevState *st, cudaStream_t s) {
    FParams fp;
    memset(&fp, 0, sizeof fp);
    t.pass1<<<p.grid, p.block, p.smem, s>>>(p.a, g, W, nullptr, nullptr, nullptr, partials, st, fp, 0, 0);
}

inline void march_pass2(const MarchFns &t, const MarchPlan &p, const GridDev &g, const float *W, const float *Vn,
                        const float *T, float *out, const DevState *st, const FParams &fp, int kind, int brt,
                        cudaStream_t s, float *guard_partials = nullptr) {
    MarchArgs a = p.a;
    a.wslot = 1;
    // stage T (and Vn) by TMA where the plan left slots: T first (BRT), then Vn (RK stage 2)
    const int need = ((brt && kind != STAGE_RK1 && p.t_ok) ? 1 : 0) |
                     ((kind == STAGE_RK2 && ((uintptr_t)Vn % 16) == 0) ? 2 : 0);
    a.xs = 0;
    if (a.xn >= 2) a.xs = need;
    else if (a.xn == 1) a.xs = (need & 1) ? 1 : need;
    const march_fn fn = (kind >= 0 && kind < 3 && t.pass2k[kind]) ? t.pass2k[kind] : t.pass2;
    fn<<<p.grid, p.block, p.smem, s>>>(a, g, W, Vn, T, out, guard_partials, st, fp, kind, brt);
}

// Pass 1 split by axis-0 planes (multi-GPU overlap): the interior planes [R, N0 - R)
// need no halo, the boundary planes [0, R) and [N0 - R, N0) do.  Both launches use the full grid so
// the partials are 2 x grid records (interior first).  map: 1 interior, 2 boundary.
inline MarchArgs march_subset(const MarchArgs &a0, int map, int R) {
    MarchArgs a = a0;
    a.i0map = map;
    a.i0r = R;
    a.s0n = map == 1 ? a0.sn[0] - 2 * R : 2 * R;
    const long long per_plane = a0.ncols / a0.sn[0];
    a.ncols = (int)(per_plane * a.s0n);
    a.units = a.ncols * a.nrb * a.nseg;
    a.wslot = map == 1 ? 0 : 2;
    return a;
}

inline void march_pass1_split(const MarchFns &t, const MarchPlan &p, const MarchArgs &a, const GridDev &g,
                              const float *W, float *partials, const DevState *st, cudaStream_t s) {
    FParams fp;
    memset(&fp, 0, sizeof fp);
    t.pass1<<<p.grid, p.block, p.smem, s>>>(a, g, W, nullptr, nullptr, nullptr, partials, st, fp, 0, 0);
}

}  // namespace odp
