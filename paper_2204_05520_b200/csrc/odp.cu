// odp.cu -- C-ABI (include/odp.h), host orchestrator and kernel instantiation of the B200 HJ
// level-set step.  One translation unit: libodp.so.
//
// Host orchestration of Algorithm 2 per save interval (reading A9):
//   begin(tau_k) -> chunks of steps [pass1 -> finalize -> pass2 (-> pass1 -> finalize -> pass2)
//   -> advance] launched back to back; every kernel early-exits once the device state says the
//   interval is done, so the host polls the 80-byte state only between chunks.
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <algorithm>
#include <cstdarg>
#include <cstdint>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <chrono>
#include <condition_variable>
#include <functional>
#include <mutex>
#include <thread>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>   // header-only NVTX: ranges are free unless a profiler injects itself

#include "../../include/odp.h"
#include "kernels_march.cuh"
#include "kernels_ttr.cuh"
#include "kernels_vi.cuh"

// NVTX ranges around the host orchestration (SURVEY.md §5 tracing): solve, save interval, halo
// exchange, range allreduce, resident launch -- visible in Nsight Systems / ncu --nvtx filters
struct NvtxRange {
    explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange &) = delete;
    NvtxRange &operator=(const NvtxRange &) = delete;
};

using namespace odp;

// ------------------------------------------------------------------------------------------------
// errors
// ------------------------------------------------------------------------------------------------
static thread_local std::string g_err;

static odp_status fail(odp_status s, const char *fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return s;
}

#define CUDA_TRY(expr)                                                                            \
    do {                                                                                          \
        cudaError_t e_ = (expr);                                                                  \
        if (e_ != cudaSuccess)                                                                    \
            return fail(e_ == cudaErrorMemoryAllocation ? ODP_ENOMEM : ODP_ECUDA, "%s: %s (%s:%d)", \
                        #expr, cudaGetErrorString(e_), __FILE__, __LINE__);                       \
    } while (0)

// ------------------------------------------------------------------------------------------------
// NCCL, loaded on first use (dlopen of libnccl.so.2: the copy torch.distributed already mapped, else
// the system one), so single-GPU use of the library has no NCCL dependency
// ------------------------------------------------------------------------------------------------
namespace nccl {
typedef int result_t;
typedef void *comm_t;
struct UniqueId { char internal[128]; };
enum { Float32 = 7 };
enum { Max = 2 };
struct Api {
    bool ok = false;
    result_t (*GetUniqueId)(UniqueId *) = nullptr;
    result_t (*CommInitRank)(comm_t *, int, UniqueId, int) = nullptr;
    result_t (*CommDestroy)(comm_t) = nullptr;
    result_t (*Send)(const void *, size_t, int, int, comm_t, cudaStream_t) = nullptr;
    result_t (*Recv)(void *, size_t, int, int, comm_t, cudaStream_t) = nullptr;
    result_t (*AllReduce)(const void *, void *, size_t, int, int, comm_t, cudaStream_t) = nullptr;
    result_t (*GroupStart)() = nullptr;
    result_t (*GroupEnd)() = nullptr;
    const char *(*GetErrorString)(result_t) = nullptr;
    result_t (*CommGetAsyncError)(comm_t, result_t *) = nullptr;   // failure detection (optional)
    result_t (*CommAbort)(comm_t) = nullptr;
};
static Api &api() {
    static Api a;
    static bool tried = false;
    if (tried) return a;
    tried = true;
    void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return a;
    a.GetUniqueId = (result_t(*)(UniqueId *))dlsym(h, "ncclGetUniqueId");
    a.CommInitRank = (result_t(*)(comm_t *, int, UniqueId, int))dlsym(h, "ncclCommInitRank");
    a.CommDestroy = (result_t(*)(comm_t))dlsym(h, "ncclCommDestroy");
    a.Send = (result_t(*)(const void *, size_t, int, int, comm_t, cudaStream_t))dlsym(h, "ncclSend");
    a.Recv = (result_t(*)(void *, size_t, int, int, comm_t, cudaStream_t))dlsym(h, "ncclRecv");
    a.AllReduce = (result_t(*)(const void *, void *, size_t, int, int, comm_t, cudaStream_t))dlsym(h, "ncclAllReduce");
    a.GroupStart = (result_t(*)())dlsym(h, "ncclGroupStart");
    a.GroupEnd = (result_t(*)())dlsym(h, "ncclGroupEnd");
    a.GetErrorString = (const char *(*)(result_t))dlsym(h, "ncclGetErrorString");
    a.CommGetAsyncError = (result_t(*)(comm_t, result_t *))dlsym(h, "ncclCommGetAsyncError");
    a.CommAbort = (result_t(*)(comm_t))dlsym(h, "ncclCommAbort");
    a.ok = a.GetUniqueId && a.CommInitRank && a.CommDestroy && a.Send && a.Recv && a.AllReduce && a.GroupStart &&
           a.GroupEnd && a.GetErrorString;
    return a;
}
}  // namespace nccl

#define NCCL_TRY(expr)                                                                            \
    do {                                                                                          \
        nccl::result_t r_ = (expr);                                                               \
        if (r_ != 0)                                                                              \
            return fail(ODP_ENCCL, "%s: %s (%s:%d)", #expr, nccl::api().GetErrorString(r_), __FILE__, __LINE__); \
    } while (0)

// ------------------------------------------------------------------------------------------------
// finalize / time-loop control kernels (Alg. 2 l.164-167; readings A7, A9, A19, A20)
// ------------------------------------------------------------------------------------------------
// Per-CTA partials of pass 1 -> one range record [-minD(n), maxD(n), maxabs, nan] (every entry a
// max, so ranks combine records with a single allreduce(max); exact in any order).
template <int NDIM>
__global__ void __launch_bounds__(256) k_reduce_partials(const float *__restrict__ partials, int nparts,
                                                         const DevState *st, float *range) {
    if (!st->active) return;
    constexpr int Q = 2 * NDIM + 2;
    __shared__ float red[Q][8];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int q = 0; q < Q; ++q) {
        float r = q < NDIM ? __int_as_float(0x7f800000) : (q < 2 * NDIM ? -__int_as_float(0x7f800000) : 0.f);
        for (int p = threadIdx.x; p < nparts; p += blockDim.x) {
            const float o = partials[(long long)p * Q + q];
            r = q < NDIM ? fminf(r, o) : fmaxf(r, o);
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            const float o = __shfl_xor_sync(0xffffffffu, r, off);
            r = q < NDIM ? fminf(r, o) : fmaxf(r, o);
        }
        if (lane == 0) red[q][warp] = r;
    }
    __syncthreads();
    if (threadIdx.x < Q) {
        const int q = threadIdx.x;
        float r = red[q][0];
        for (int w = 1; w < (int)(blockDim.x >> 5); ++w) r = q < NDIM ? fminf(r, red[q][w]) : fmaxf(r, red[q][w]);
        range[q] = q < NDIM ? -r : r;
    }
}

// The body of k_finalize; k_resident runs it in every CTA on a CTA-local copy of the state (CG:
// partials read through L2, they are rewritten between the grid barriers of that launch).
template <class F, int NDIM, bool CG>
__device__ __forceinline__ void finalize_body(const float *partials, int nparts, DevState *st,
                                              const GridDev &g, const FParams &fp, const double *__restrict__ dxd,
                                              int stage_in_step, int final_check, const float *__restrict__ range,
                                              const float *__restrict__ amax_parts, int namax,
                                              bool reuse_amax = false) {
    if (!st->active) return;
    constexpr int Q = 2 * NDIM + 2;
    __shared__ float red[Q][8];
    __shared__ float rng[Q];
    __shared__ int bad;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (range) {            // multi-GPU: the range record was allreduced over the ranks
        if (threadIdx.x < Q) rng[threadIdx.x] = threadIdx.x < NDIM ? -range[threadIdx.x] : range[threadIdx.x];
    } else
    // reduce the per-CTA partials of pass 1 (min/max are exact: any order gives the same bits);
    // all Q entries of a record are loaded before any reduction so the loads overlap
    {
        float r[Q];
#pragma unroll
        for (int q = 0; q < Q; ++q) r[q] = q < NDIM ? __int_as_float(0x7f800000) : (q < 2 * NDIM ? -__int_as_float(0x7f800000) : 0.f);
        for (int p = threadIdx.x; p < nparts; p += blockDim.x) {
            float o[Q];
#pragma unroll
            for (int q = 0; q < Q; ++q) o[q] = ldw<CG>(partials + (long long)p * Q + q);
#pragma unroll
            for (int q = 0; q < Q; ++q) r[q] = q < NDIM ? fminf(r[q], o[q]) : fmaxf(r[q], o[q]);
        }
#pragma unroll
        for (int q = 0; q < Q; ++q) {
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) {
                const float o = __shfl_xor_sync(0xffffffffu, r[q], off);
                r[q] = q < NDIM ? fminf(r[q], o) : fmaxf(r[q], o);
            }
            if (lane == 0) red[q][warp] = r[q];
        }
    }
    __syncthreads();
    if (!range && threadIdx.x < Q) {
        const int q = threadIdx.x;
        float r = red[q][0];
        for (int w = 1; w < (int)(blockDim.x >> 5); ++w) r = q < NDIM ? fminf(r, red[q][w]) : fmaxf(r, red[q][w]);
        rng[q] = r;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int d = 0; d < NDIM; ++d) { st->minD[d] = rng[d]; st->maxD[d] = rng[NDIM + d]; }
        st->maxabs = rng[2 * NDIM];
        st->nan = rng[2 * NDIM + 1] != 0.f;
        bad = st->nan || !(rng[2 * NDIM] <= 1e10f);
        if (bad) { st->status = ODP_ENUMERIC; st->active = 0; }
        else if (final_check) st->active = 0;
        else st->stages += 1;
    }
    __syncthreads();
    if (bad || final_check || stage_in_step != 0) return;

    // alpha^max_d = max over the nodes of alpha_{i,d}: enumerate the (<= 2) coordinate axes that
    // alpha_d depends on (functor deps); any other coordinate is irrelevant to alpha_d.
    F f;
    f.init(fp, rng, rng + NDIM);
    __shared__ float am[NDIM];
    if (F::RANGE_FREE && reuse_amax) {   // k_resident: alpha^max of a RANGE_FREE functor is the
        if (threadIdx.x < NDIM) am[threadIdx.x] = st->amax[threadIdx.x];   // previous step's, bit for bit
        __syncthreads();
    } else if constexpr (F::DEPS3) {   // alpha_d depends on 3 coordinates: per-CTA maxima from k_amax3
        float a[NDIM];                  // block-wide max over the records (exact in any order)
#pragma unroll
        for (int d = 0; d < NDIM; ++d) a[d] = 0.f;
        for (int p = threadIdx.x; p < namax; p += blockDim.x)
#pragma unroll
            for (int d = 0; d < NDIM; ++d) a[d] = fmaxf(a[d], ldw<CG>(amax_parts + p * NDIM + d));
#pragma unroll
        for (int d = 0; d < NDIM; ++d) {
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) a[d] = fmaxf(a[d], __shfl_xor_sync(0xffffffffu, a[d], off));
            if (lane == 0) red[d][warp] = a[d];
        }
        __syncthreads();
        if (threadIdx.x < NDIM) {
            float r = red[threadIdx.x][0];
            for (int w = 1; w < (int)(blockDim.x >> 5); ++w) r = fmaxf(r, red[threadIdx.x][w]);
            am[threadIdx.x] = r;
        }
        __syncthreads();
    } else
    for (int d = 0; d < NDIM; ++d) {
        const int m = F::deps(d);
        int ax[2] = {-1, -1}, na = 0;
        for (int a = 0; a < NDIM; ++a) if ((m >> a) & 1) ax[na++] = a;
        const int n0 = na > 0 ? g.Ng[ax[0]] : 1, n1 = na > 1 ? g.Ng[ax[1]] : 1;
        float r = 0.f;
        for (int t = threadIdx.x; t < n0 * n1; t += blockDim.x) {
            Pt q;
            if (na > 0) load_axis<F>(g, q, ax[0], t % n0);
            if (na > 1) load_axis<F>(g, q, ax[1], t / n0);
            r = fmaxf(r, f.alpha(d, q));
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) r = fmaxf(r, __shfl_xor_sync(0xffffffffu, r, off));
        if (lane == 0) red[0][warp] = r;
        __syncthreads();
        if (threadIdx.x == 0) {
            float a = red[0][0];
            for (int w = 1; w < (int)(blockDim.x >> 5); ++w) a = fmaxf(a, red[0][w]);
            am[d] = a;
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        double sum = 0.0;                                             // Alg. 2 l.167
        for (int d = 0; d < NDIM; ++d) { st->amax[d] = am[d]; sum += fabs((double)am[d]) / dxd[d]; }
        const double rem = st->tau_target - st->tau;
        double dt = sum > 0.0 ? st->cfl / sum : rem;                 // A20
        if (dt > rem) dt = rem;                                       // A9
        st->dt = dt;
        st->dt_f = (float)dt;
    }
}

template <class F, int NDIM>
__global__ void __launch_bounds__(256) k_finalize(const float *__restrict__ partials, int nparts, DevState *st,
                                                  GridDev g, FParams fp, const double *__restrict__ dxd,
                                                  int stage_in_step, int final_check, const float *__restrict__ range,
                                                  const float *__restrict__ amax_parts, int namax) {
    finalize_body<F, NDIM, false>(partials, nparts, st, g, fp, dxd, stage_in_step, final_check, range, amax_parts,
                                  namax);
}

__global__ void k_init_state(DevState *st, double cfl, double eps) {
    st->tau = 0.0; st->tau_target = 0.0; st->eps = eps; st->dt = 0.0; st->cfl = cfl; st->dt_f = 0.f;
    st->maxabs = 0.f; st->nan = 0; st->active = 0; st->status = 0; st->steps = 0; st->stages = 0; st->pending = 0;
    st->work[0] = st->work[1] = st->work[2] = 0u;
    for (int d = 0; d < MAXD; ++d) { st->minD[d] = 0.f; st->maxD[d] = 0.f; st->amax[d] = 0.f; }
}

__device__ __forceinline__ void begin_body(DevState *st, double tau_k) {
    if (st->pending) { st->status = ODP_ENUMERIC; st->pending = 0; }
    st->tau_target = tau_k;
    st->active = (st->status == 0 && tau_k - st->tau > st->eps) ? 1 : 0;
}
__global__ void k_begin(DevState *st, double tau_k) { begin_body(st, tau_k); }

__device__ __forceinline__ void force_active_body(DevState *st) {
    if (st->pending) { st->status = ODP_ENUMERIC; st->pending = 0; }
    st->active = st->status == 0 ? 1 : 0;
}
__global__ void k_force_active(DevState *st) { force_active_body(st); }

// For functors whose alpha_d depends on three coordinates (DEPS3, e.g. Eq. 7): the stage's range is
// stored first (k_store_range: the same exact min/max reduction as k_finalize), then k_amax3 takes
// the maximum of alpha_{i,d} over the nodes of that coordinate grid with many CTAs (the
// one-CTA enumeration of k_finalize would cost N0 N1 N2 / 256 iterations per stage).
template <int NDIM, bool CG>
__device__ __forceinline__ void store_range_body(const float *partials, int nparts, DevState *st) {
    constexpr int Q = 2 * NDIM + 2;
    __shared__ float red[Q][8];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int q = 0; q < 2 * NDIM; ++q) {
        float r = q < NDIM ? __int_as_float(0x7f800000) : -__int_as_float(0x7f800000);
        for (int p = threadIdx.x; p < nparts; p += blockDim.x) {
            const float o = ldw<CG>(partials + (long long)p * Q + q);
            r = q < NDIM ? fminf(r, o) : fmaxf(r, o);
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            const float o = __shfl_xor_sync(0xffffffffu, r, off);
            r = q < NDIM ? fminf(r, o) : fmaxf(r, o);
        }
        if (lane == 0) red[q][warp] = r;
    }
    __syncthreads();
    if (threadIdx.x < 2 * NDIM) {
        const int q = threadIdx.x;
        float r = red[q][0];
        for (int w = 1; w < (int)(blockDim.x >> 5); ++w) r = q < NDIM ? fminf(r, red[q][w]) : fmaxf(r, red[q][w]);
        if (q < NDIM) st->minD[q] = r; else st->maxD[q - NDIM] = r;
    }
}

template <int NDIM>
__global__ void __launch_bounds__(256) k_store_range(const float *__restrict__ partials, int nparts, DevState *st,
                                                     const float *__restrict__ range) {
    if (!st->active) return;
    if (range) {
        if (threadIdx.x < NDIM) { st->minD[threadIdx.x] = -range[threadIdx.x]; st->maxD[threadIdx.x] = range[NDIM + threadIdx.x]; }
        return;
    }
    store_range_body<NDIM, false>(partials, nparts, st);
}

template <class F, int NDIM>
__device__ __forceinline__ void amax3_body(const GridDev &g, const FParams &fp, const DevState *st, float *parts) {
    F f;
    f.init(fp, st->minD, st->maxD);
    float a[NDIM];
#pragma unroll
    for (int d = 0; d < NDIM; ++d) a[d] = 0.f;
    const long long n = (long long)g.Ng[0] * g.Ng[1] * g.Ng[2];
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const int i2 = (int)(i % g.Ng[2]);
        const long long r = i / g.Ng[2];
        const int i1 = (int)(r % g.Ng[1]), i0 = (int)(r / g.Ng[1]);
        Pt q;
        load_axis<F>(g, q, 0, i0);
        load_axis<F>(g, q, 1, i1);
        load_axis<F>(g, q, 2, i2);
#pragma unroll
        for (int d = 0; d < NDIM; ++d) a[d] = fmaxf(a[d], f.alpha(d, q));
    }
    __shared__ float red[NDIM][8];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int d = 0; d < NDIM; ++d) {
        float r = a[d];
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) r = fmaxf(r, __shfl_xor_sync(0xffffffffu, r, off));
        if (lane == 0) red[d][warp] = r;
    }
    __syncthreads();
    if (threadIdx.x < NDIM) {
        float r = red[threadIdx.x][0];
        for (int w = 1; w < (int)(blockDim.x >> 5); ++w) r = fmaxf(r, red[threadIdx.x][w]);
        parts[blockIdx.x * NDIM + threadIdx.x] = r;
    }
}

template <class F, int NDIM>
__global__ void __launch_bounds__(256) k_amax3(GridDev g, FParams fp, const DevState *st, float *parts) {
    if (!st->active) return;
    amax3_body<F, NDIM>(g, fp, st, parts);
}

// One launch in place of k_store_range + k_amax3 + k_finalize (one rank, stage 0 of a step): every
// CTA reduces pass 1's partials into a CTA-local range (the same exact min/max), takes its share of
// the alpha^max enumeration, and the LAST CTA to finish (arrival counter, reset by that CTA) runs the
// finalize on the global state, reading the per-CTA maxima through L2.  Bitwise the three launches.
template <class F, int NDIM>
__global__ void __launch_bounds__(256) k_amax3_fin(const float *__restrict__ partials, int nparts, DevState *st,
                                                   GridDev g, FParams fp, const double *__restrict__ dxd,
                                                   float *parts, unsigned *ctr) {
    if (!st->active) return;
    __shared__ DevState loc;
    __shared__ bool last;
    store_range_body<NDIM, false>(partials, nparts, &loc);
    __syncthreads();
    amax3_body<F, NDIM>(g, fp, &loc, parts);
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        last = atomicAdd(ctr, 1u) == gridDim.x - 1;
        if (last) *ctr = 0u;
    }
    __syncthreads();
    if (!last) return;
    __threadfence();
    finalize_body<F, NDIM, true>(partials, nparts, st, g, fp, dxd, 0, 0, nullptr, parts, (int)gridDim.x);
}

// Single-pass solves: for a functor whose alpha_(i,d) does not depend on the
// derivative range (RANGE_FREE), alpha^max is the same at every step, so pass 1 is dead work apart
// from the guard of A19.  k_dt re-derives dt from the stored alpha^max exactly as k_finalize does
// (same float64 expression); k_guard checks the stage OUTPUT (= the next stage's input) from the
// max|V| / NaN partials pass 2 wrote, and counts the stage.
__global__ void k_dt(DevState *st, const double *__restrict__ dxd, int n) {
    st->work[1] = 0u;              // the previous launch may have been a pass 2 (k_march work counters)
    if (!st->active) return;
    if (st->pending) { st->status = ODP_ENUMERIC; st->active = 0; return; }   // detected at this stage's input
    double sum = 0.0;                                                 // Alg. 2 l.167
    for (int d = 0; d < n; ++d) sum += fabs((double)st->amax[d]) / dxd[d];
    const double rem = st->tau_target - st->tau;
    double dt = sum > 0.0 ? st->cfl / sum : rem;                      // A20
    if (dt > rem) dt = rem;                                           // A9
    st->dt = dt;
    st->dt_f = (float)dt;
}

template <int NDIM>
__global__ void __launch_bounds__(256) k_guard(const float *__restrict__ partials, int nparts, DevState *st,
                                               const float *__restrict__ range, int last_stage) {
    if (!st->active) return;
    constexpr int Q = 2 * NDIM + 2;
    __shared__ float red[2][8];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    float ma = 0.f, nn = 0.f;
    if (range) {
        ma = range[2 * NDIM]; nn = range[2 * NDIM + 1];
    } else {
        for (int p = threadIdx.x; p < nparts; p += blockDim.x) {
            ma = fmaxf(ma, partials[(long long)p * Q + 2 * NDIM]);
            nn = fmaxf(nn, partials[(long long)p * Q + 2 * NDIM + 1]);
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            ma = fmaxf(ma, __shfl_xor_sync(0xffffffffu, ma, off));
            nn = fmaxf(nn, __shfl_xor_sync(0xffffffffu, nn, off));
        }
        if (lane == 0) { red[0][warp] = ma; red[1][warp] = nn; }
        __syncthreads();
        if (threadIdx.x == 0)
            for (int w = 1; w < (int)(blockDim.x >> 5); ++w) { ma = fmaxf(ma, red[0][w]); nn = fmaxf(nn, red[1][w]); }
    }
    if (threadIdx.x == 0) {
        st->stages += 1;                                              // the stage ran on a checked input
        if (nn != 0.f || !(ma <= 1e10f)) {
            // the two-pass solve detects this at the next stage's input: within the step (RK stage 1)
            // that stops the step; after its last stage the step completes (tau advances) first
            st->nan = nn != 0.f;
            if (last_stage) st->pending = 1;
            else { st->status = ODP_ENUMERIC; st->active = 0; }
        }
        st->maxabs = ma;
        st->work[1] = 0u;          // single-pass: pass 2 follows pass 2 (see k_march's work counters)
    }
}

__device__ __forceinline__ void advance_body(DevState *st) {           // O8: tau += dt (float64)
    if (!st->active) return;
    st->tau += st->dt;
    st->steps += 1;
    if (st->tau_target - st->tau <= st->eps) st->active = 0;
}
__global__ void k_advance(DevState *st) { advance_body(st); }

// ------------------------------------------------------------------------------------------------
// k_resident: the whole solve of a small grid in ONE cooperative launch (ODP_KERNEL_RESIDENT).
// A grid that fits in L2 many times over (c1: 61k nodes, 242 KB per array) spends its time on
// launch gaps and host round trips, not on HBM: ~10 launches per step and a D2H + host sync per
// save interval, each a few us, against ~1 us of arithmetic per pass.  Here every save interval,
// time step, RK stage, finalize and snapshot runs inside one kernel: the passes are the generic
// family's per-node bodies (so the result is bitwise the generic family's: same arithmetic per
// node, min/max partials exact in any order), arrays read through L2 (ld.global.cg), and the
// control kernels (k_begin, k_finalize, k_advance, k_force_active) run redundantly in EVERY CTA
// on a CTA-local copy of DevState -- same inputs, same float64 operations, so every copy takes
// the same decisions and the only grid-wide synchronisation is one barrier after each pass.
// CTA 0 writes the state back at the end.  Launched with cudaLaunchCooperativeKernel (all CTAs
// co-resident, required by the spin barrier).
// ------------------------------------------------------------------------------------------------
constexpr int ODP_AMAX_PARTS = 4096;   // per-CTA alpha^max records (k_amax3: nsm CTAs; k_resident: its grid)
struct ResidentArgs {
    float *buf0, *buf1;          // V ping-pong (local slab layout, no halo use: one rank)
    const float *T;              // BRT target
    float *out;                  // snapshots, out + k * P
    const double *tau;           // device copy of the save times
    int ntau, k_out0;
    float *partials;             // gridDim.x * (2n + 2) floats
    const double *dxd;
    DevState *st;
    unsigned *bar;               // grid barrier counter, zeroed before the launch
    float *amax_parts;           // DEPS3 functors: per-CTA alpha^max, gridDim.x * n floats
    int low, brt;
};

// Grid-wide barrier: monotonic arrival counter, CTA b waits until gen * gridDim.x arrivals.  The
// __syncthreads + gpu-scope fence before the arrival release the CTA's writes; the acquire load
// orders the reads after it.
__device__ __forceinline__ void grid_barrier(unsigned *bar, unsigned &gen) {
    __syncthreads();
    gen += 1;
    if (threadIdx.x == 0) {
        __threadfence();
        atomicAdd(bar, 1u);
        const unsigned target = gen * gridDim.x;
        unsigned v;
        do {
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(bar) : "memory");
        } while ((int)(v - target) < 0);
    }
    __syncthreads();
}

template <class F, int NDIM, int R>
__global__ void __launch_bounds__(256) k_resident(GridDev g, FParams fp, ResidentArgs a) {
    __shared__ DevState sst;
    if (threadIdx.x == 0) sst = *a.st;
    __syncthreads();
    unsigned gen = 0;
    float *buf[2] = {a.buf0, a.buf1};
    const long long P = g.P;
    const int np = gridDim.x;
    int cur = 0, k_out = a.k_out0;
    auto ctl = [&](auto &&fn) {                 // one control step on the CTA-local state
        __syncthreads();
        if (threadIdx.x == 0) fn();
        __syncthreads();
    };
    bool have_amax = false;                     // RANGE_FREE: alpha^max computed once (bitwise the same)
    auto fin = [&](int stage, int final_check) {
        if constexpr (F::DEPS3) {
            // alpha_d depends on 3 coordinates (Eq. 7): k_store_range + k_amax3 of the multi-launch
            // path, here by every CTA over its share of the coordinate grid, one more grid barrier;
            // the branch is uniform over the grid (every CTA holds the same state)
            if (stage == 0 && !final_check && sst.active) {
                store_range_body<NDIM, true>(a.partials, np, &sst);
                __syncthreads();
                amax3_body<F, NDIM>(g, fp, &sst, a.amax_parts);
                grid_barrier(a.bar, gen);
            }
        }
        finalize_body<F, NDIM, true>(a.partials, np, &sst, g, fp, a.dxd, stage, final_check, nullptr, a.amax_parts,
                                     F::DEPS3 ? np : 0, have_amax);
        __syncthreads();
        if (stage == 0 && !final_check && sst.active) have_amax = true;
    };
    for (int k = 1; k < a.ntau; ++k) {
        ctl([&] { begin_body(&sst, a.tau[k]); });
        while (sst.active) {
            const long long s0 = sst.steps;
            if (a.low) {                          // Alg. 2, Euler (LOW): pass 1, finalize, pass 2
                pass1_generic_body<NDIM, R, true>(g, buf[cur], a.partials, &sst);
                grid_barrier(a.bar, gen);
                fin(0, 0);
                pass2_generic_body<F, NDIM, R, true>(g, buf[cur], nullptr, a.T, buf[cur ^ 1], &sst, fp, STAGE_EULER, a.brt);
                grid_barrier(a.bar, gen);
            } else {                              // TVD-RK2 (MEDIUM): two stages (A10)
                pass1_generic_body<NDIM, R, true>(g, buf[0], a.partials, &sst);
                grid_barrier(a.bar, gen);
                fin(0, 0);
                pass2_generic_body<F, NDIM, R, true>(g, buf[0], nullptr, a.T, buf[1], &sst, fp, STAGE_RK1, a.brt);
                grid_barrier(a.bar, gen);
                pass1_generic_body<NDIM, R, true>(g, buf[1], a.partials, &sst);
                grid_barrier(a.bar, gen);
                fin(1, 0);
                pass2_generic_body<F, NDIM, R, true>(g, buf[1], buf[0], a.T, buf[0], &sst, fp, STAGE_RK2, a.brt);
                grid_barrier(a.bar, gen);
            }
            ctl([&] { advance_body(&sst); });
            if (a.low && sst.steps != s0) cur ^= 1;
        }
        if (sst.status) break;                    // numeric failure: no snapshot, no final guard
        const float *src = buf[a.low ? cur : 0];
        float *dst = a.out + (long long)k_out * P;
        for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < P; i += (long long)gridDim.x * blockDim.x)
            dst[i] = __ldcg(src + i);
        ++k_out;
    }
    if (!sst.status) {                            // final guard on the last V (reading A19)
        ctl([&] { force_active_body(&sst); });
        pass1_generic_body<NDIM, R, true>(g, buf[a.low ? cur : 0], a.partials, &sst);
        grid_barrier(a.bar, gen);
        fin(0, 1);
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) *a.st = sst;
}

// ------------------------------------------------------------------------------------------------
// kernel tables
// ------------------------------------------------------------------------------------------------
typedef void (*pass1_fn)(GridDev, const float *, float *, const DevState *);
typedef void (*pass2_fn)(GridDev, const float *, const float *, const float *, float *, const DevState *, FParams,
                         int, int);
typedef void (*fin_fn)(const float *, int, DevState *, GridDev, FParams, const double *, int, int, const float *,
                       const float *, int);
typedef void (*srange_fn)(const float *, int, DevState *, const float *);
typedef void (*amax3_fn)(GridDev, FParams, const DevState *, float *);
typedef void (*amax3fin_fn)(const float *, int, DevState *, GridDev, FParams, const double *, float *, unsigned *);
typedef void (*red_fn)(const float *, int, const DevState *, float *);
typedef void (*guard_fn)(const float *, int, DevState *, const float *, int);
typedef void (*res_fn)(GridDev, FParams, ResidentArgs);

struct KernelSet {
    pass1_fn pass1 = nullptr;
    pass2_fn pass2 = nullptr;
    fin_fn fin = nullptr;
    red_fn red = nullptr;
    guard_fn guard = nullptr;
    srange_fn srange = nullptr;   // DEPS3 functors only
    amax3_fn amax3 = nullptr;
    amax3fin_fn amax3fin = nullptr;   // DEPS3, one rank: range + alpha^max + finalize in one launch
    res_fn res = nullptr;         // k_resident
    bool range_free = false;
    TiledFns tiled;      // tiled family (may be empty)
    StreamFnsAll stream; // stream family (may be empty)
    MarchFnsAll march;   // march family (may be empty)
};

template <class F, int NDIM, int R>
static KernelSet make_set() {
    KernelSet k;
    k.pass1 = k_pass1_generic<NDIM, R>;
    k.pass2 = k_pass2_generic<F, NDIM, R>;
    k.fin = k_finalize<F, NDIM>;
    k.red = k_reduce_partials<NDIM>;
    k.guard = k_guard<NDIM>;
    k.range_free = F::RANGE_FREE;
    if constexpr (F::DEPS3) {
        k.srange = k_store_range<NDIM>;
        k.amax3 = k_amax3<F, NDIM>;
        k.amax3fin = k_amax3_fin<F, NDIM>;
    }
    k.res = k_resident<F, NDIM, R>;
    if constexpr (F::SEPARABLE) {      // the tiled / stream families assemble separable Hamiltonians only
        k.tiled = tiled_fns<F, NDIM, R>();
        k.stream = stream_fns<F, NDIM, R>();
    }
    k.march = march_fns<F, NDIM, R>();
    return k;
}

template <template <int> class FH, int R>
static KernelSet holo_set(int n) {
    switch (n) {
    case 1: return make_set<FH<1>, 1, R>();
    case 2: return make_set<FH<2>, 2, R>();
    case 3: return make_set<FH<3>, 3, R>();
    case 4: return make_set<FH<4>, 4, R>();
    case 5: return make_set<FH<5>, 5, R>();
    default: return make_set<FH<6>, 6, R>();
    }
}

template <int R>
static KernelSet select_set_r(int dyn, int n) {
    switch (dyn) {
    case ODP_DYN_HOLONOMIC_BALL: return holo_set<FHoloBall, R>(n);
    case ODP_DYN_HOLONOMIC_BOX: return holo_set<FHoloBox, R>(n);
    case ODP_DYN_DUBINS3D: return make_set<FDubins3D, 3, R>();
    case ODP_DYN_CAR4D: return make_set<FCar4D, 4, R>();
    case ODP_DYN_CAR5D: return make_set<FCar5D, 5, R>();
    case ODP_DYN_PAIR_DUBINS3D: return make_set<FPairDubins3D, 3, R>();
    default: return make_set<FDoubleInt6D, 6, R>();
    }
}

static KernelSet select_set(int dyn, int n, int R) { return R == 1 ? select_set_r<1>(dyn, n) : select_set_r<2>(dyn, n); }

// ------------------------------------------------------------------------------------------------
// grid handle
// ------------------------------------------------------------------------------------------------
struct odp_loopback;
extern "C" void odp_loopback_destroy(odp_loopback *lb);
struct odp_grid {
    int n = 0;
    int64_t N[MAXD] = {0};
    double lo[MAXD] = {0}, hi[MAXD] = {0}, dx[MAXD] = {0};
    int per[MAXD] = {0};
    int64_t P = 0;                // points of the whole grid
    // axis-0 slab partition (odp_grid_partition); unpartitioned: rank 0 of 1 owning [0, N[0])
    int rank = 0, nranks = 1;
    int64_t i0b = 0, n0 = 0;      // first owned axis-0 plane, owned planes
    nccl::comm_t comm = nullptr;
    odp_loopback *lb = nullptr;   // test transport: slabs of one process on one GPU (odp_grid_partition_loopback)
    float *d_range = nullptr;     // [-minD, maxD, maxabs, nan] of the current stage (allreduced)
    float *d_amax = nullptr;      // per-CTA alpha^max of k_amax3 (DEPS3 functors)
    double *d_tau = nullptr;      // k_resident: device copy of the save times (capacity tau_cap)
    int tau_cap = 0;
    unsigned *d_bar = nullptr;    // k_resident: grid barrier counter
    unsigned *d_ctr = nullptr;    // k_amax3_fin: arrival counter (zero between launches)
    // device cache (allocated lazily on the device current at the first solve)
    int device = -1;
    float *d_tab = nullptr;
    int tab_off[MAXD] = {0};
    double *d_dx = nullptr;
    float *d_buf[2] = {nullptr, nullptr};
    size_t buf_elems = 0;
    int64_t halo_elems = 0;       // R_MAX planes before local plane 0
    float *d_partials = nullptr;
    int max_parts = 0;
    DevState *d_state = nullptr;
    DevState *h_state = nullptr;  // pinned
    cudaStream_t own_stream = nullptr;
    cudaStream_t side_stream = nullptr;     // NCCL halo exchange overlapped with interior pass 1
    cudaEvent_t ev_in = nullptr, ev_halo = nullptr;
    cudaEvent_t ev_join[2] = {nullptr, nullptr};   // NULL-stream callers: order own_stream after / before the legacy stream
    std::vector<cudaEvent_t> events;
    long long launches = 0;
    float *d_stage = nullptr;     // staging buffers of the *_host entry points (grown on demand)
    size_t stage_elems = 0;
    TtrState *d_ttr = nullptr;    // time-to-reach iteration state (odp_ttr_solve)
    TtrState *h_ttr = nullptr;    // pinned
};

static constexpr int R_MAX = 2;

static void free_device(odp_grid *g) {
    if (g->device < 0) return;
    int cur = -1;
    cudaGetDevice(&cur);
    cudaSetDevice(g->device);
    cudaFree(g->d_tab); cudaFree(g->d_dx);
    cudaFree(g->d_buf[0]); cudaFree(g->d_buf[1]);
    cudaFree(g->d_partials); cudaFree(g->d_state); cudaFree(g->d_range); cudaFree(g->d_amax);
    if (g->h_state) cudaFreeHost(g->h_state);
    cudaFree(g->d_ttr);
    if (g->h_ttr) cudaFreeHost(g->h_ttr);
    cudaFree(g->d_stage);
    g->d_stage = nullptr; g->stage_elems = 0;
    cudaFree(g->d_tau); cudaFree(g->d_bar); cudaFree(g->d_ctr);
    g->d_tau = nullptr; g->tau_cap = 0; g->d_bar = nullptr; g->d_ctr = nullptr;
    g->d_ttr = nullptr; g->h_ttr = nullptr;
    if (g->own_stream) cudaStreamDestroy(g->own_stream);
    if (g->side_stream) cudaStreamDestroy(g->side_stream);
    if (g->ev_in) cudaEventDestroy(g->ev_in);
    if (g->ev_halo) cudaEventDestroy(g->ev_halo);
    for (auto &e : g->ev_join) { if (e) cudaEventDestroy(e); e = nullptr; }
    g->side_stream = nullptr; g->ev_in = nullptr; g->ev_halo = nullptr;
    for (auto e : g->events) cudaEventDestroy(e);
    g->events.clear();
    g->d_tab = nullptr; g->d_dx = nullptr; g->d_buf[0] = g->d_buf[1] = nullptr; g->d_partials = nullptr;
    g->d_state = nullptr; g->h_state = nullptr; g->own_stream = nullptr; g->d_range = nullptr; g->d_amax = nullptr;
    g->max_parts = 0; g->buf_elems = 0;
    g->device = -1;
    if (cur >= 0) cudaSetDevice(cur);
}

extern "C" odp_status odp_grid_create(int dims, const double *lo, const double *hi, const int64_t *N,
                                      uint32_t periodic_mask, odp_grid **out) {
    g_err.clear();
    if (!out) return fail(ODP_EINVAL, "out is NULL");
    *out = nullptr;
    if (dims < 1 || dims > MAXD) return fail(ODP_EINVAL, "dims=%d not in 1..6", dims);
    if (!lo || !hi || !N) return fail(ODP_EINVAL, "NULL lo/hi/N");
    odp_grid *g = new (std::nothrow) odp_grid();
    if (!g) return fail(ODP_ENOMEM, "host allocation");
    g->n = dims;
    g->P = 1;
    for (int d = 0; d < dims; ++d) {
        if (N[d] < 3) { delete g; return fail(ODP_EINVAL, "N[%d]=%lld < 3", d, (long long)N[d]); }
        if (!(lo[d] < hi[d])) { delete g; return fail(ODP_EINVAL, "lo[%d] >= hi[%d]", d, d); }
        if (N[d] > (int64_t)1 << 30) { delete g; return fail(ODP_EINVAL, "N[%d] too large", d); }
        g->N[d] = N[d]; g->lo[d] = lo[d]; g->hi[d] = hi[d];
        g->per[d] = (periodic_mask >> d) & 1u;
        g->dx[d] = g->per[d] ? (hi[d] - lo[d]) / (double)N[d] : (hi[d] - lo[d]) / (double)(N[d] - 1);   // A15
        if (g->P > INT64_MAX / N[d]) { delete g; return fail(ODP_EINVAL, "point count overflows int64 at axis %d", d); }
        g->P *= N[d];
    }
    if (dims > 1 && g->P / g->N[0] > ((int64_t)1 << 31) - 1) { delete g; return fail(ODP_EINVAL, "axis-0 plane exceeds 2^31 points"); }
    g->i0b = 0;
    g->n0 = g->N[0];
    *out = g;
    return ODP_OK;
}

extern "C" void odp_grid_destroy(odp_grid *g) {
    if (!g) return;
    free_device(g);
    if (g->comm && nccl::api().ok) nccl::api().CommDestroy(g->comm);
    delete g;
}

static int64_t plane_of(const odp_grid *g) { return g->P / g->N[0]; }
static int64_t local_points(const odp_grid *g) { return g->n0 * plane_of(g); }

// Balanced contiguous axis-0 slabs: rank r owns [b, b + c) with c = floor(N0 / P) or + 1 (the first
// N0 mod P ranks take one more plane).
extern "C" odp_status odp_partition_extent(int64_t N0, int nranks, int rank, int64_t *i0_begin, int64_t *i0_count) {
    g_err.clear();
    if (nranks < 1 || rank < 0 || rank >= nranks || N0 < 1) return fail(ODP_EINVAL, "bad partition request");
    const int64_t q = N0 / nranks, r = N0 % nranks;
    const int64_t c = q + (rank < r ? 1 : 0);
    const int64_t b = rank * q + (rank < r ? rank : r);
    if (i0_begin) *i0_begin = b;
    if (i0_count) *i0_count = c;
    return ODP_OK;
}

extern "C" odp_status odp_comm_unique_id(void *id128) {
    g_err.clear();
    if (!id128) return fail(ODP_EINVAL, "NULL id");
    nccl::Api &a = nccl::api();
    if (!a.ok) return fail(ODP_ENCCL, "libnccl.so.2 not loadable: %s", dlerror());
    nccl::UniqueId id;
    NCCL_TRY(a.GetUniqueId(&id));
    memcpy(id128, &id, sizeof id);
    return ODP_OK;
}

// Axis-0 slab partition (north_star: slabs along axis 0, NCCL halo exchange + allreduce per stage).
extern "C" odp_status odp_grid_partition(odp_grid *g, int rank, int nranks, const void *id128, int device) {
    g_err.clear();
    if (!g) return fail(ODP_EINVAL, "NULL grid");
    if (nranks < 1 || rank < 0 || rank >= nranks) return fail(ODP_EINVAL, "rank %d of %d", rank, nranks);
    if (nranks > 1 && g->per[0]) return fail(ODP_EINVAL, "axis 0 is periodic: slab partition not supported");
    if (nranks > 1 && g->N[0] < (int64_t)R_MAX * nranks)
        return fail(ODP_EINVAL, "N[0]=%lld < %d planes per rank", (long long)g->N[0], R_MAX);
    if (nranks > 1 && !id128) return fail(ODP_EINVAL, "NULL NCCL id");
    int64_t b = 0, c = 0;
    odp_status st = odp_partition_extent(g->N[0], nranks, rank, &b, &c);
    if (st) return st;
    free_device(g);                       // working buffers are sized by the slab
    if (g->comm && nccl::api().ok) nccl::api().CommDestroy(g->comm);
    g->comm = nullptr;
    g->lb = nullptr;
    g->rank = rank; g->nranks = nranks; g->i0b = b; g->n0 = c;
    if (id128) {            // (nranks = 1 with an id: a 1-rank communicator -- the multi-GPU code path)
        nccl::Api &a = nccl::api();
        if (!a.ok) return fail(ODP_ENCCL, "libnccl.so.2 not loadable");
        CUDA_TRY(cudaSetDevice(device));
        nccl::UniqueId id;
        memcpy(&id, id128, sizeof id);
        NCCL_TRY(a.CommInitRank(&g->comm, nranks, id, rank));
    }
    return ODP_OK;
}

extern "C" odp_status odp_grid_local_extent(const odp_grid *g, int64_t *i0_begin, int64_t *i0_count) {
    g_err.clear();
    if (!g) return fail(ODP_EINVAL, "NULL grid");
    if (i0_begin) *i0_begin = g->i0b;
    if (i0_count) *i0_count = g->n0;
    return ODP_OK;
}

extern "C" odp_status odp_grid_info(const odp_grid *g, int *dims, int64_t *N, double *dx, int64_t *points) {
    g_err.clear();
    if (!g) return fail(ODP_EINVAL, "NULL grid");
    if (dims) *dims = g->n;
    for (int d = 0; d < g->n; ++d) {
        if (N) N[d] = g->N[d];
        if (dx) dx[d] = g->dx[d];
    }
    if (points) *points = local_points(g);
    return ODP_OK;
}

extern "C" long long odp_last_launch_count(const odp_grid *g) { return g ? g->launches : 0; }
extern "C" const char *odp_last_error(void) { return g_err.c_str(); }
extern "C" const char *odp_version(void) { return "odp-b200 0.1 sm_100a"; }

static odp_status ensure_device(odp_grid *g, int nparts_needed) {
    int dev = 0;
    CUDA_TRY(cudaGetDevice(&dev));
    if (g->device >= 0 && g->device != dev) free_device(g);
    const int64_t plane = plane_of(g);
    if (g->device < 0) {
        g->device = dev;
        // coordinate tables x, cos x, sin x per axis: float64 host values rounded to float32 (A26)
        std::vector<float> tab;
        for (int d = 0; d < g->n; ++d) {
            g->tab_off[d] = (int)tab.size();
            for (int k = 0; k < 3; ++k)
                for (int64_t i = 0; i < g->N[d]; ++i) {
                    const double x = g->lo[d] + (double)i * g->dx[d];
                    tab.push_back((float)(k == 0 ? x : (k == 1 ? std::cos(x) : std::sin(x))));
                }
        }
        CUDA_TRY(cudaMalloc(&g->d_tab, tab.size() * sizeof(float)));
        CUDA_TRY(cudaMemcpy(g->d_tab, tab.data(), tab.size() * sizeof(float), cudaMemcpyHostToDevice));
        CUDA_TRY(cudaMalloc(&g->d_dx, MAXD * sizeof(double)));
        CUDA_TRY(cudaMemcpy(g->d_dx, g->dx, MAXD * sizeof(double), cudaMemcpyHostToDevice));
        CUDA_TRY(cudaMalloc(&g->d_state, sizeof(DevState)));
        CUDA_TRY(cudaMallocHost(&g->h_state, sizeof(DevState)));
        CUDA_TRY(cudaStreamCreateWithFlags(&g->own_stream, cudaStreamNonBlocking));
        for (auto &e : g->ev_join) CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    if (!g->d_buf[0]) {
        g->halo_elems = R_MAX * plane;
        g->buf_elems = (size_t)(local_points(g) + 2 * g->halo_elems);
        for (int b = 0; b < 2; ++b) {
            CUDA_TRY(cudaMalloc(&g->d_buf[b], g->buf_elems * sizeof(float)));
            CUDA_TRY(cudaMemset(g->d_buf[b], 0, g->buf_elems * sizeof(float)));
        }
    }
    if (g->max_parts < nparts_needed) {
        cudaFree(g->d_partials);
        g->d_partials = nullptr;
        CUDA_TRY(cudaMalloc(&g->d_partials, (size_t)nparts_needed * (2 * MAXD + 2) * sizeof(float)));
        g->max_parts = nparts_needed;
    }
    if (!g->d_range) CUDA_TRY(cudaMalloc(&g->d_range, (2 * MAXD + 2) * sizeof(float)));
    if (!g->d_amax) CUDA_TRY(cudaMalloc(&g->d_amax, ODP_AMAX_PARTS * MAXD * sizeof(float)));
    return ODP_OK;
}

// Device staging area of the *_host entry points: kept in the handle so that repeated end-to-end
// calls do not pay a multi-GB allocation each time.
static odp_status stage_buffer(odp_grid *g, size_t elems, float **out) {
    if (g->stage_elems < elems) {
        cudaFree(g->d_stage);
        g->d_stage = nullptr;
        g->stage_elems = 0;
        CUDA_TRY(cudaMalloc(&g->d_stage, elems * sizeof(float)));
        g->stage_elems = elems;
    }
    *out = g->d_stage;
    return ODP_OK;
}

// The stream a call runs on.  A NULL opts->stream (torch's legacy default stream reports handle 0)
// means "the caller's default stream": the call then runs on the handle's own non-blocking stream,
// ordered AFTER everything already enqueued on the legacy default stream (the caller may have just
// produced V0 / target / R there) and, on exit, the legacy stream is ordered after the call (the
// caller may reuse the output memory at once).  An explicit stream is used as given.
struct StreamScope {
    cudaStream_t s = nullptr, legacy_join = nullptr;
    cudaEvent_t done = nullptr;
    StreamScope(odp_grid *g, void *user) {
        if (user) { s = (cudaStream_t)user; return; }
        s = g->own_stream;
        cudaEventRecord(g->ev_join[0], cudaStreamLegacy);
        cudaStreamWaitEvent(s, g->ev_join[0], 0);
        legacy_join = s;
        done = g->ev_join[1];
    }
    ~StreamScope() {
        if (!legacy_join) return;
        cudaEventRecord(done, legacy_join);
        cudaStreamWaitEvent(cudaStreamLegacy, done, 0);
    }
};

static GridDev make_griddev(const odp_grid *g) {
    GridDev d;
    memset(&d, 0, sizeof d);
    d.n = g->n;
    for (int k = 0; k < g->n; ++k) {
        d.N[k] = (int)g->N[k];
        d.Ng[k] = (int)g->N[k];
        d.per[k] = g->per[k];
        d.inv_dx[k] = (float)(1.0 / g->dx[k]);
        d.hih[k] = 0.5f * d.inv_dx[k];
        d.dx[k] = (float)g->dx[k];
        d.tab_off[k] = g->tab_off[k];
    }
    d.stride[g->n - 1] = 1;
    for (int k = g->n - 2; k >= 0; --k) d.stride[k] = d.stride[k + 1] * g->N[k + 1];
    d.N[0] = (int)g->n0;
    d.P = local_points(g);
    d.Ng0 = (int)g->N[0];
    d.g0 = (int)g->i0b;
    d.tab = g->d_tab;
    return d;
}

// ------------------------------------------------------------------------------------------------
// Loopback transport (tests: the multi-rank slab path on ONE GPU).  The P slab handles of one
// process, each driven by its own host thread, exchange halo planes by device-to-device copies and
// reduce their range records with a max kernel.  Ordering uses only stream events plus a host
// barrier per collective (every rank enqueues the same collectives in the same order, as with
// NCCL: same dt sequence, same launch chunks); nothing on the device waits on another rank's
// kernel, so ranks may run concurrently or one after the other.
// ------------------------------------------------------------------------------------------------
struct odp_loopback {
    int n = 0;
    std::mutex m;
    std::condition_variable cv;
    long long gen = 0;
    int count = 0;
    std::vector<odp_grid *> g;            // by rank
    std::vector<float *> w;               // each rank's stage input of the current exchange
    std::vector<cudaEvent_t> ready, done; // per rank: my data is final / I finished reading the others'
    float *rec = nullptr;                 // [n][2 MAXD + 2] range records (device, on the ranks' GPU)
    void barrier() {
        std::unique_lock<std::mutex> lk(m);
        const long long g0 = gen;
        if (++count == n) { count = 0; ++gen; cv.notify_all(); }
        else cv.wait(lk, [&] { return gen != g0; });
    }
};

__global__ void k_rec_max(const float *rec, int nr, int cnt, float *out) {
    const int q = threadIdx.x;
    if (q >= cnt) return;
    float r = rec[q];
    for (int k = 1; k < nr; ++k) r = fmaxf(r, rec[k * (2 * MAXD + 2) + q]);
    out[q] = r;
}

extern "C" odp_status odp_loopback_create(int nranks, odp_loopback **out) {
    g_err.clear();
    if (!out || nranks < 1 || nranks > 64) return fail(ODP_EINVAL, "loopback of %d ranks", nranks);
    odp_loopback *lb = new (std::nothrow) odp_loopback();
    if (!lb) return fail(ODP_ENOMEM, "host allocation");
    lb->n = nranks;
    lb->g.assign(nranks, nullptr);
    lb->w.assign(nranks, nullptr);
    lb->ready.assign(nranks, nullptr);
    lb->done.assign(nranks, nullptr);
    for (int r = 0; r < nranks; ++r) {
        if (cudaEventCreateWithFlags(&lb->ready[r], cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&lb->done[r], cudaEventDisableTiming) != cudaSuccess) {
            odp_loopback_destroy(lb);
            return fail(ODP_ECUDA, "loopback events");
        }
    }
    if (cudaMalloc(&lb->rec, (size_t)nranks * (2 * MAXD + 2) * sizeof(float)) != cudaSuccess) {
        odp_loopback_destroy(lb);
        return fail(ODP_ECUDA, "loopback records");
    }
    *out = lb;
    return ODP_OK;
}

extern "C" void odp_loopback_destroy(odp_loopback *lb) {
    if (!lb) return;
    for (auto e : lb->ready) if (e) cudaEventDestroy(e);
    for (auto e : lb->done) if (e) cudaEventDestroy(e);
    cudaFree(lb->rec);
    delete lb;
}

extern "C" odp_status odp_grid_partition_loopback(odp_grid *g, int rank, odp_loopback *lb) {
    g_err.clear();
    if (!g || !lb) return fail(ODP_EINVAL, "NULL grid / loopback");
    const int nranks = lb->n;
    if (rank < 0 || rank >= nranks) return fail(ODP_EINVAL, "rank %d of %d", rank, nranks);
    if (nranks > 1 && g->per[0]) return fail(ODP_EINVAL, "axis 0 is periodic: slab partition not supported");
    if (nranks > 1 && g->N[0] < (int64_t)R_MAX * nranks)
        return fail(ODP_EINVAL, "N[0]=%lld < %d planes per rank", (long long)g->N[0], R_MAX);
    int64_t b = 0, c = 0;
    odp_status st = odp_partition_extent(g->N[0], nranks, rank, &b, &c);
    if (st) return st;
    free_device(g);
    if (g->comm && nccl::api().ok) nccl::api().CommDestroy(g->comm);
    g->comm = nullptr;
    g->rank = rank; g->nranks = nranks; g->i0b = b; g->n0 = c;
    g->lb = lb;
    lb->g[rank] = g;
    return ODP_OK;
}

static odp_status lb_halo_exchange(odp_grid *g, float *W, int R, cudaStream_t s) {
    odp_loopback *lb = g->lb;
    const int me = g->rank;
    const size_t plane = (size_t)plane_of(g), cnt = (size_t)R * plane;
    lb->w[me] = W;
    CUDA_TRY(cudaEventRecord(lb->ready[me], s));
    lb->barrier();                                           // every rank's W recorded
    if (me > 0) {                                            // rank-1's last R planes -> my low halo
        const odp_grid *o = lb->g[me - 1];
        CUDA_TRY(cudaStreamWaitEvent(s, lb->ready[me - 1], 0));
        CUDA_TRY(cudaMemcpyAsync(W - cnt, lb->w[me - 1] + (size_t)(o->n0 - R) * plane, cnt * sizeof(float),
                                 cudaMemcpyDeviceToDevice, s));
    }
    if (me < lb->n - 1) {                                    // rank+1's first R planes -> my high halo
        CUDA_TRY(cudaStreamWaitEvent(s, lb->ready[me + 1], 0));
        CUDA_TRY(cudaMemcpyAsync(W + (size_t)g->n0 * plane, lb->w[me + 1], cnt * sizeof(float),
                                 cudaMemcpyDeviceToDevice, s));
    }
    CUDA_TRY(cudaEventRecord(lb->done[me], s));
    lb->barrier();                                           // every rank's reads enqueued
    if (me > 0) CUDA_TRY(cudaStreamWaitEvent(s, lb->done[me - 1], 0));   // my planes read before I overwrite them
    if (me < lb->n - 1) CUDA_TRY(cudaStreamWaitEvent(s, lb->done[me + 1], 0));
    return ODP_OK;
}

static odp_status lb_range_allreduce(odp_grid *g, int n, cudaStream_t s) {
    odp_loopback *lb = g->lb;
    const int me = g->rank, cnt = 2 * n + 2;
    CUDA_TRY(cudaMemcpyAsync(lb->rec + (size_t)me * (2 * MAXD + 2), g->d_range, cnt * sizeof(float),
                             cudaMemcpyDeviceToDevice, s));
    CUDA_TRY(cudaEventRecord(lb->ready[me], s));
    lb->barrier();
    for (int r = 0; r < lb->n; ++r)
        if (r != me) CUDA_TRY(cudaStreamWaitEvent(s, lb->ready[r], 0));
    k_rec_max<<<1, 32, 0, s>>>(lb->rec, lb->n, cnt, g->d_range);
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaEventRecord(lb->done[me], s));
    lb->barrier();
    for (int r = 0; r < lb->n; ++r)                          // every rank read my record before I rewrite it
        if (r != me) CUDA_TRY(cudaStreamWaitEvent(s, lb->done[r], 0));
    return ODP_OK;
}

// Halo planes of a stage input W (local plane 0) from the axis-0 neighbours (north_star: NCCL
// send/recv per RK stage): my first R planes go to rank-1's high halo, my last R planes to rank+1's
// low halo.  Slabs are contiguous row-major ranges, so every message is one contiguous range.
static odp_status halo_exchange(odp_grid *g, float *W, int R, cudaStream_t s) {
    if (g->nranks <= 1) return ODP_OK;
    NvtxRange nv("odp halo_exchange");
    if (g->lb) return lb_halo_exchange(g, W, R, s);
    nccl::Api &a = nccl::api();
    const size_t plane = (size_t)plane_of(g), cnt = (size_t)R * plane;
    NCCL_TRY(a.GroupStart());
    if (g->rank > 0) {
        NCCL_TRY(a.Send(W, cnt, nccl::Float32, g->rank - 1, g->comm, s));
        NCCL_TRY(a.Recv(W - cnt, cnt, nccl::Float32, g->rank - 1, g->comm, s));
    }
    if (g->rank < g->nranks - 1) {
        NCCL_TRY(a.Send(W + (size_t)(g->n0 - R) * plane, cnt, nccl::Float32, g->rank + 1, g->comm, s));
        NCCL_TRY(a.Recv(W + (size_t)g->n0 * plane, cnt, nccl::Float32, g->rank + 1, g->comm, s));
    }
    NCCL_TRY(a.GroupEnd());
    return ODP_OK;
}

// allreduce(max) of the stage's range record [-minD, maxD, maxabs, nan] over the ranks
static odp_status range_allreduce(odp_grid *g, int n, cudaStream_t s) {
    NvtxRange nv("odp range_allreduce");
    if (g->lb) return lb_range_allreduce(g, n, s);
    if (!g->comm) return ODP_OK;
    NCCL_TRY(nccl::api().AllReduce(g->d_range, g->d_range, (size_t)(2 * n + 2), nccl::Float32, nccl::Max, g->comm, s));
    return ODP_OK;
}

// Host wait for a stream of a partitioned solve.  With an NCCL communicator the wait polls (no
// blocking synchronize): a peer that failed or vanished leaves our NCCL kernels waiting forever, so
// ncclCommGetAsyncError is checked every millisecond and the communicator is aborted on an error or
// after ODP_NCCL_TIMEOUT_S seconds (default 600) without progress -- the solve then returns
// ODP_ENCCL instead of hanging.
static odp_status sync_stream(odp_grid *g, cudaStream_t s) {
    if (!g->comm) {
        CUDA_TRY(cudaStreamSynchronize(s));
        return ODP_OK;
    }
    nccl::Api &a = nccl::api();
    double limit = 600.0;
    if (const char *e = getenv("ODP_NCCL_TIMEOUT_S")) limit = atof(e);
    const auto t0 = std::chrono::steady_clock::now();
    for (;;) {
        const cudaError_t q = cudaStreamQuery(s);
        if (q == cudaSuccess) return ODP_OK;
        if (q != cudaErrorNotReady) return fail(ODP_ECUDA, "stream: %s", cudaGetErrorString(q));
        nccl::result_t ae = 0;
        if (a.CommGetAsyncError && a.CommGetAsyncError(g->comm, &ae) == 0 && ae != 0) {
            if (a.CommAbort) a.CommAbort(g->comm);
            g->comm = nullptr;
            return fail(ODP_ENCCL, "NCCL asynchronous error: %s (communicator aborted)", a.GetErrorString(ae));
        }
        const double el = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        if (el > limit) {
            if (a.CommAbort) a.CommAbort(g->comm);
            g->comm = nullptr;
            return fail(ODP_ENCCL, "no progress for %.0f s (peer failure?): communicator aborted", el);
        }
        std::this_thread::sleep_for(std::chrono::microseconds(200));
    }
}

static const int kWantParams[7] = {2, 3, 3, 5, 3, 3, 5};
static const int kWantDims[7] = {0, 0, 3, 4, 5, 6, 3};

static odp_status validate_dyn(const odp_grid *g, int dyn, const double *params, int nparams) {
    if (!g) return fail(ODP_EINVAL, "NULL grid");
    if (dyn < 0 || dyn > 6) return fail(ODP_EINVAL, "unknown dynamics id %d", dyn);
    if (!params || nparams != kWantParams[dyn]) return fail(ODP_EINVAL, "dynamics %d takes %d params (got %d)", dyn, kWantParams[dyn], nparams);
    if (kWantDims[dyn] && kWantDims[dyn] != g->n) return fail(ODP_EINVAL, "dynamics %d needs dims=%d (grid has %d)", dyn, kWantDims[dyn], g->n);
    const double goal = params[nparams - 1];
    if (goal != 1.0 && goal != -1.0) return fail(ODP_EINVAL, "goal must be -1 or +1");
    for (int k = 0; k < nparams; ++k) if (!std::isfinite(params[k])) return fail(ODP_EINVAL, "param %d not finite", k);
    return ODP_OK;
}

static odp_status validate(const odp_grid *g, int dyn, const double *params, int nparams, const double *tau,
                           int ntau, int accuracy, int mode) {
    odp_status st = validate_dyn(g, dyn, params, nparams);
    if (st) return st;
    if (accuracy != ODP_LOW && accuracy != ODP_MEDIUM) return fail(ODP_EINVAL, "accuracy %d", accuracy);
    if (mode != ODP_BRS && mode != ODP_BRT) return fail(ODP_EINVAL, "mode %d", mode);
    if (!tau || ntau < 2) return fail(ODP_EINVAL, "need ntau >= 2");
    if (tau[0] != 0.0) return fail(ODP_EINVAL, "tau[0] must be 0");
    for (int k = 1; k < ntau; ++k) if (!(tau[k] > tau[k - 1])) return fail(ODP_EINVAL, "tau not strictly increasing at %d", k);
    return ODP_OK;
}

namespace {
struct Launch {
    int kind;          // 0 pass1, 1 pass2, 2 finalize/control, 3 pass2 of RK stage 2
    int ev;            // index of the start event (stop = ev + 1), -1 if untimed
};
}

static odp_status solve_device(odp_grid *g, int dyn, const double *params, int nparams, const float *V0,
                               const double *tau, int ntau, int accuracy, int mode, float *out,
                               const odp_solve_opts *opts) {
    odp_status st = validate(g, dyn, params, nparams, tau, ntau, accuracy, mode);
    if (st) return st;
    if (!V0 || !out) return fail(ODP_EINVAL, "NULL V0/out");
    const int R = accuracy == ODP_LOW ? 1 : 2;
    const int n = g->n;
    KernelSet ks = select_set(dyn, n, R);

    const int want_kernel = opts ? opts->kernel : ODP_KERNEL_AUTO;
    GridDev gd_probe;
    memset(&gd_probe, 0, sizeof gd_probe);

    // launch geometry of the generic family
    const int block = 256;
    int nsm = 148;
    {
        int dev = 0;
        CUDA_TRY(cudaGetDevice(&dev));
        CUDA_TRY(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    }
    long long want_blocks = (local_points(g) + block - 1) / block;
    int grid_generic = (int)std::min<long long>(want_blocks, (long long)nsm * 8);

    if ((st = ensure_device(g, std::max(grid_generic, nsm * 8)))) return st;
    GridDev gd = make_griddev(g);

    const float *Tcheck = (opts && opts->target) ? opts->target : V0;
    bool use_march = false, use_stream = false, use_tiled = false;
    MarchPlan mp;
    MarchFns mfn;
    StreamPlan sp;
    StreamFns sfn;
    TiledPlan tp;
    if (want_kernel == ODP_KERNEL_AUTO || want_kernel == ODP_KERNEL_MARCH)
        use_march = march_plan(gd, R, ks.march, Tcheck, g->d_buf[0] + g->halo_elems, &mfn, &mp);
    if (want_kernel == ODP_KERNEL_MARCH && !use_march) return fail(ODP_EINVAL, "march kernels do not cover this grid");
    if (!use_march && (want_kernel == ODP_KERNEL_AUTO || want_kernel == ODP_KERNEL_STREAM))
        use_stream = stream_plan(gd, R, ks.stream, &sfn, &sp);
    if (want_kernel == ODP_KERNEL_STREAM && !use_stream) return fail(ODP_EINVAL, "stream kernels do not cover this grid");
    if (!use_march && !use_stream && (want_kernel == ODP_KERNEL_AUTO || want_kernel == ODP_KERNEL_TILED) && ks.tiled.pass1)
        use_tiled = tiled_plan(gd, R, nsm, &tp);
    if (want_kernel == ODP_KERNEL_TILED && !use_tiled) return fail(ODP_EINVAL, "tiled kernels do not cover this grid");
    // resident (one cooperative launch per solve): asked for, or AUTO on a small single-rank grid
    // without per-launch timing (ODP_RESIDENT_MAX_POINTS, default 2^18 nodes: ~1 MB per array)
    const long long res_max = getenv("ODP_RESIDENT_MAX_POINTS") ? atoll(getenv("ODP_RESIDENT_MAX_POINTS")) : (1LL << 18);
    const bool res_ok = ks.res && g->nranks == 1 && !g->comm && !g->lb && !(opts && opts->kernel_ms) &&
                        !(opts && opts->single_pass);
    if (want_kernel == ODP_KERNEL_RESIDENT && !res_ok)
        return fail(ODP_EINVAL, "resident kernel: one rank, no kernel_ms / single_pass");
    const bool use_resident = want_kernel == ODP_KERNEL_RESIDENT ||
                              (want_kernel == ODP_KERNEL_AUTO && res_ok && local_points(g) <= res_max);
    if (use_resident) use_march = use_stream = use_tiled = false;
    if (use_march) {
        if (march_prepare(mfn, mp, nsm)) return fail(ODP_ECUDA, "march kernel attribute setup failed");
        if ((st = ensure_device(g, mp.grid))) return st;
    }
    if (use_stream) {
        if (stream_prepare(sfn, sp, nsm)) return fail(ODP_ECUDA, "stream kernel attribute setup failed");
        if ((st = ensure_device(g, sp.grid))) return st;
    }
    if (use_tiled) {
        if (tiled_prepare(ks.tiled, tp, nsm)) return fail(ODP_ECUDA, "tiled kernel attribute setup failed");
        if ((st = ensure_device(g, tp.grid))) return st;
    }
    const int nparts = use_march ? mp.grid : use_stream ? sp.grid : (use_tiled ? tp.grid : grid_generic);
    // multi-GPU overlap: pass 1 on the interior axis-0 planes runs while the NCCL halo
    // exchange is in flight on a side stream, then pass 1 on the R boundary planes at each slab end.
    // Needs an axis-0 side axis (march family, dims >= 4) and interior planes; ODP_SPLIT_PASS1=1
    // forces the split on one rank (tests: bitwise equal to the unsplit solve)
    const bool force_split = getenv("ODP_SPLIT_PASS1") && atoi(getenv("ODP_SPLIT_PASS1")) == 1;
    const bool split = use_march && n >= 4 && g->n0 >= 2 * R + 1 && (g->nranks > 1 || force_split) &&
                       !(getenv("ODP_SPLIT_PASS1") && atoi(getenv("ODP_SPLIT_PASS1")) == 0);
    MarchArgs ma_int, ma_bnd;
    if (split) {
        ma_int = march_subset(mp.a, 1, R);
        ma_bnd = march_subset(mp.a, 2, R);
        if ((st = ensure_device(g, 2 * mp.grid))) return st;
        if (!g->side_stream) {
            CUDA_TRY(cudaStreamCreateWithFlags(&g->side_stream, cudaStreamNonBlocking));
            CUDA_TRY(cudaEventCreateWithFlags(&g->ev_in, cudaEventDisableTiming));
            CUDA_TRY(cudaEventCreateWithFlags(&g->ev_halo, cudaEventDisableTiming));
        }
    }
    const int nparts1 = split ? 2 * mp.grid : nparts;      // pass-1 partial records (launch_fin)

    StreamScope sscope(g, opts ? opts->stream : nullptr);
    cudaStream_t s = sscope.s;
    const double cfl = (opts && opts->cfl > 0.0) ? opts->cfl : (accuracy == ODP_LOW ? 0.8 : 0.5);   // A7
    const double eps = 1e-12 * std::max(1.0, tau[ntau - 1]);
    const int brt = mode == ODP_BRT;
    const float *T = (opts && opts->target) ? opts->target : V0;
    const int write_initial = opts ? opts->write_initial : 0;
    const bool timed = opts && opts->kernel_ms;
    double kms[4] = {0, 0, 0, 0};       // pass 1, pass 2, control, pass 2 of RK stage 2 (subset of pass 2)

    FParams fp;
    memset(&fp, 0, sizeof fp);
    for (int k = 0; k < nparams; ++k) fp.c[k] = (float)params[k];

    float *buf[2] = {g->d_buf[0] + g->halo_elems, g->d_buf[1] + g->halo_elems};
    const size_t bytes = (size_t)local_points(g) * sizeof(float);
    g->launches = 0;

    CUDA_TRY(cudaMemcpyAsync(buf[0], V0, bytes, cudaMemcpyDeviceToDevice, s));
    k_init_state<<<1, 1, 0, s>>>(g->d_state, cfl, eps);
    ++g->launches;
    CUDA_TRY(cudaGetLastError());
    int k_out = 0;
    if (write_initial) {
        CUDA_TRY(cudaMemcpyAsync(out, V0, bytes, cudaMemcpyDeviceToDevice, s));
        k_out = 1;
    }

    if (use_resident) {
        int occ = 0;
        CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, ks.res, block, 0));
        if (occ < 1) return fail(ODP_ECUDA, "k_resident does not fit on an SM");
        long long nb = std::min<long long>(std::min<long long>(want_blocks, (long long)occ * nsm), ODP_AMAX_PARTS);
        if (getenv("ODP_RESIDENT_CTAS")) nb = std::max(1LL, std::min<long long>(nb, atoll(getenv("ODP_RESIDENT_CTAS"))));
        if ((st = ensure_device(g, (int)nb))) return st;
        if (g->tau_cap < ntau) {
            cudaFree(g->d_tau);
            g->d_tau = nullptr;
            g->tau_cap = 0;
            CUDA_TRY(cudaMalloc(&g->d_tau, (size_t)ntau * sizeof(double)));
            g->tau_cap = ntau;
        }
        if (!g->d_bar) CUDA_TRY(cudaMalloc(&g->d_bar, sizeof(unsigned)));
        CUDA_TRY(cudaMemcpyAsync(g->d_tau, tau, (size_t)ntau * sizeof(double), cudaMemcpyHostToDevice, s));
        CUDA_TRY(cudaMemsetAsync(g->d_bar, 0, sizeof(unsigned), s));
        ResidentArgs ra;
        ra.buf0 = buf[0]; ra.buf1 = buf[1]; ra.T = T; ra.out = out; ra.tau = g->d_tau; ra.ntau = ntau;
        ra.k_out0 = k_out; ra.partials = g->d_partials; ra.dxd = g->d_dx; ra.st = g->d_state; ra.bar = g->d_bar;
        ra.amax_parts = g->d_amax;
        ra.low = accuracy == ODP_LOW; ra.brt = brt;
        void *kargs[] = {&gd, &fp, &ra};
        NvtxRange nv("odp k_resident (whole solve)");
        CUDA_TRY(cudaLaunchCooperativeKernel((const void *)ks.res, dim3((unsigned)nb), dim3(block), kargs, 0, s));
        ++g->launches;
        CUDA_TRY(cudaMemcpyAsync(g->h_state, g->d_state, sizeof(DevState), cudaMemcpyDeviceToHost, s));
        if (odp_status ss = sync_stream(g, s)) return ss;
        if (opts) {
            if (opts->tau_reached) *opts->tau_reached = g->h_state->tau;
            if (opts->steps_taken) *opts->steps_taken = g->h_state->steps;
            if (opts->stages_taken) *opts->stages_taken = g->h_state->stages;
            if (opts->single_pass_used) *opts->single_pass_used = 0;
        }
        if (g->h_state->status)
            return fail(ODP_ENUMERIC, "numerical failure (NaN or |V| > 1e10) at tau = %.9g", g->h_state->tau);
        return ODP_OK;
    }

    std::vector<Launch> launches;
    auto ensure_events = [&](size_t nev) -> odp_status {
        while (g->events.size() < nev) {
            cudaEvent_t e;
            CUDA_TRY(cudaEventCreate(&e));
            g->events.push_back(e);
        }
        return ODP_OK;
    };

    auto launch_pass1 = [&](const float *W) {
        if (use_march) march_pass1(mfn, mp, gd, W, g->d_partials, g->d_state, s);
        else if (use_stream) stream_pass1(sfn, sp, gd, W, g->d_partials, g->d_state, s);
        else if (use_tiled) tiled_pass1(ks.tiled, tp, gd, W, g->d_partials, g->d_state, s);
        else ks.pass1<<<grid_generic, block, 0, s>>>(gd, W, g->d_partials, g->d_state);
    };
    // single-pass: opted in, RANGE_FREE functor, march family
    const bool single = opts && opts->single_pass && ks.range_free && use_march;
    bool have_amax = false;              // alpha^max of this solve computed by a two-pass step
    auto launch_pass2 = [&](const float *W, const float *Vn, float *o, int kind, bool guard = false) {
        if (use_march) march_pass2(mfn, mp, gd, W, Vn, T, o, g->d_state, fp, kind, brt, s, guard ? g->d_partials : nullptr);
        else if (use_stream) stream_pass2(sfn, sp, gd, W, Vn, T, o, g->d_state, fp, kind, brt, s);
        else if (use_tiled) tiled_pass2(ks.tiled, tp, gd, W, Vn, T, o, g->d_state, fp, kind, brt, s);
        else ks.pass2<<<grid_generic, block, 0, s>>>(gd, W, Vn, T, o, g->d_state, fp, kind, brt);
    };
    odp_status cst = ODP_OK;     // first communication failure (NCCL calls are enqueued, not checked per launch)
    auto launch_guard = [&](int last_stage) {
        if (g->comm || g->lb) {
            ks.red<<<1, 256, 0, s>>>(g->d_partials, nparts, g->d_state, g->d_range);
            if (cst == ODP_OK) cst = range_allreduce(g, n, s);
            ks.guard<<<1, 256, 0, s>>>(g->d_partials, nparts, g->d_state, g->d_range, last_stage);
        } else {
            ks.guard<<<1, 256, 0, s>>>(g->d_partials, nparts, g->d_state, nullptr, last_stage);
        }
    };
    auto exch = [&](float *Wx) {
        if (g->nranks > 1 && cst == ODP_OK) cst = halo_exchange(g, Wx, R, s);
    };
    // k_amax3 CTAs (DEPS3 functors): 3 per SM -- the enumeration is a chain of dependent table loads
    // per node, latency-bound at one CTA per SM (f2 100^3: ~27 nodes per thread); f2 sweep of
    // ODP_AMAX3_CPS 1/2/3/4/6/8/16: 26.1/29.3/30.0/29.7/27.0/26.8/21.7 Gpt-st/s
    const int namax = ks.amax3 ? std::min(ODP_AMAX_PARTS, nsm * (getenv("ODP_AMAX3_CPS") ? std::max(1, atoi(getenv("ODP_AMAX3_CPS"))) : 3)) : 0;
    if (ks.amax3fin && !g->d_ctr) {
        CUDA_TRY(cudaMalloc(&g->d_ctr, sizeof(unsigned)));
        CUDA_TRY(cudaMemsetAsync(g->d_ctr, 0, sizeof(unsigned), s));
    }
    auto launch_fin = [&](int stage_in_step, int final_check) {
        const float *rng = nullptr;
        if (g->comm || g->lb) {
            ks.red<<<1, 256, 0, s>>>(g->d_partials, nparts1, g->d_state, g->d_range);
            if (cst == ODP_OK) cst = range_allreduce(g, n, s);
            rng = g->d_range;
        }
        if (ks.amax3fin && !rng && stage_in_step == 0 && !final_check && !getenv("ODP_AMAX3_SPLIT")) {
            ks.amax3fin<<<namax, 256, 0, s>>>(g->d_partials, nparts1, g->d_state, gd, fp, g->d_dx, g->d_amax, g->d_ctr);
            return;
        }
        if (ks.amax3 && stage_in_step == 0 && !final_check) {
            ks.srange<<<1, 256, 0, s>>>(g->d_partials, nparts1, g->d_state, rng);
            ks.amax3<<<namax, 256, 0, s>>>(gd, fp, g->d_state, g->d_amax);
        }
        ks.fin<<<1, 256, 0, s>>>(g->d_partials, nparts1, g->d_state, gd, fp, g->d_dx, stage_in_step, final_check,
                                 rng, g->d_amax, namax);
    };

    // one timed/untimed launch wrapper; events are recorded only when kernel times are requested
    int ev_next = 0;
    auto rec = [&](int kind, auto &&fn) -> odp_status {
        int ev = -1;
        if (timed) {
            odp_status e = ensure_events((size_t)ev_next + 2);
            if (e) return e;
            ev = ev_next;
            ev_next += 2;
            CUDA_TRY(cudaEventRecord(g->events[ev], s));
        }
        fn();
        ++g->launches;
        if (timed) CUDA_TRY(cudaEventRecord(g->events[ev + 1], s));
        launches.push_back({kind, ev});
        return ODP_OK;
    };

    // the stage's halo exchange + pass 1: overlapped (split) or in sequence
    auto split_pass1 = [&](float *Wx) {
        cudaEventRecord(g->ev_in, s);                    // W complete (previous pass 2)
        cudaStreamWaitEvent(g->side_stream, g->ev_in, 0);
        if (g->nranks > 1 && cst == ODP_OK) cst = halo_exchange(g, Wx, R, g->side_stream);
        cudaEventRecord(g->ev_halo, g->side_stream);
        march_pass1_split(mfn, mp, ma_int, gd, Wx, g->d_partials, g->d_state, s);
        cudaStreamWaitEvent(s, g->ev_halo, 0);
        march_pass1_split(mfn, mp, ma_bnd, gd, Wx, g->d_partials + (size_t)mp.grid * (2 * n + 2), g->d_state, s);
    };
    auto exch_pass1 = [&](float *Wx) -> odp_status {
        odp_status r = ODP_OK;
        if (split) {
            r = rec(0, [&] { split_pass1(Wx); });
            ++g->launches;                                // two pass-1 launches (rec counts one)
            return r;
        }
        if (g->nranks > 1 && (r = rec(2, [&] { exch(Wx); }))) return r;
        return rec(0, [&] { launch_pass1(Wx); });
    };

    int cur = 0;                       // index of the buffer holding the current V
    odp_status rs = ODP_OK;
    // one time step (Alg. 2 l.150-170) as a launch sequence; a = buffer of the current V (LOW)
    auto step = [&](int a, bool sp_mode) -> odp_status {
        const int b = a ^ 1;
        odp_status r = ODP_OK;
        if (sp_mode) {
            // pass 2 only: dt from the fixed alpha^max, the guard on each stage's output
            if ((r = rec(2, [&] { k_dt<<<1, 1, 0, s>>>(g->d_state, g->d_dx, n); }))) return r;
            if (accuracy == ODP_LOW) {
                if (g->nranks > 1 && (r = rec(2, [&] { exch(buf[a]); }))) return r;
                if ((r = rec(1, [&] { launch_pass2(buf[a], nullptr, buf[b], STAGE_EULER, true); }))) return r;
                if ((r = rec(2, [&] { launch_guard(1); }))) return r;
            } else {
                if (g->nranks > 1 && (r = rec(2, [&] { exch(buf[0]); }))) return r;
                if ((r = rec(1, [&] { launch_pass2(buf[0], nullptr, buf[1], STAGE_RK1, true); }))) return r;
                if ((r = rec(2, [&] { launch_guard(0); }))) return r;
                if (g->nranks > 1 && (r = rec(2, [&] { exch(buf[1]); }))) return r;
                if ((r = rec(3, [&] { launch_pass2(buf[1], buf[0], buf[0], STAGE_RK2, true); }))) return r;
                if ((r = rec(2, [&] { launch_guard(1); }))) return r;
            }
        } else if (accuracy == ODP_LOW) {
            if ((r = exch_pass1(buf[a]))) return r;
            if ((r = rec(2, [&] { launch_fin(0, 0); }))) return r;
            if ((r = rec(1, [&] { launch_pass2(buf[a], nullptr, buf[b], STAGE_EULER); }))) return r;
        } else {
            if ((r = exch_pass1(buf[0]))) return r;
            if ((r = rec(2, [&] { launch_fin(0, 0); }))) return r;
            if ((r = rec(1, [&] { launch_pass2(buf[0], nullptr, buf[1], STAGE_RK1); }))) return r;
            if ((r = exch_pass1(buf[1]))) return r;
            if ((r = rec(2, [&] { launch_fin(1, 0); }))) return r;
            if ((r = rec(3, [&] { launch_pass2(buf[1], buf[0], buf[0], STAGE_RK2); }))) return r;
        }
        return rec(2, [&] { k_advance<<<1, 1, 0, s>>>(g->d_state); });
    };
    // CUDA graphs (opts.use_graph: 0 auto = grids up to 2^25 local points, 1 on, -1 off): GS steps
    // captured once per (step kind, buffer parity) and replayed as one launch; every kernel
    // early-exits once the interval is done, exactly like the direct launches.  Not with kernel
    // timing (per-launch events) or an NCCL communicator.
    constexpr int GS = 8;
    const int ug = opts ? opts->use_graph : 0;
    const bool graphs = !timed && !g->comm && !g->lb && (ug == 1 || (ug == 0 && local_points(g) <= (1LL << 25)));
    cudaGraphExec_t gexec[2][2] = {{nullptr, nullptr}, {nullptr, nullptr}};
    long long glaunch[2] = {0, 0};          // kernel launches per replay, by step kind
    auto graph_of = [&](int kind_sp, int a0, cudaGraphExec_t *out_exec) -> odp_status {
        if (gexec[kind_sp][a0]) { *out_exec = gexec[kind_sp][a0]; return ODP_OK; }
        const long long l0 = g->launches;
        cudaGraph_t graph = nullptr;
        CUDA_TRY(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
        odp_status r = ODP_OK;
        for (int j = 0; j < GS && r == ODP_OK; ++j) r = step((a0 + j) & 1, kind_sp != 0);
        const cudaError_t ce = cudaStreamEndCapture(s, &graph);
        if (r) { if (graph) cudaGraphDestroy(graph); return r; }
        if (ce != cudaSuccess) return fail(ODP_ECUDA, "graph capture: %s", cudaGetErrorString(ce));
        const cudaError_t ie = cudaGraphInstantiate(&gexec[kind_sp][a0], graph, 0);
        cudaGraphDestroy(graph);
        if (ie != cudaSuccess) return fail(ODP_ECUDA, "graph instantiate: %s", cudaGetErrorString(ie));
        glaunch[kind_sp] = g->launches - l0;
        g->launches = l0;
        *out_exec = gexec[kind_sp][a0];
        return ODP_OK;
    };
    auto free_graphs = [&]() {
        for (auto &row : gexec)
            for (auto &e : row)
                if (e) { cudaGraphExecDestroy(e); e = nullptr; }
    };
    struct GraphGuard { std::function<void()> f; ~GraphGuard() { f(); } } graph_guard{free_graphs};
    for (int k = 1; k < ntau && rs == ODP_OK; ++k) {
        NvtxRange nv("odp save interval");
        k_begin<<<1, 1, 0, s>>>(g->d_state, tau[k]);
        ++g->launches;
        CUDA_TRY(cudaMemcpyAsync(g->h_state, g->d_state, sizeof(DevState), cudaMemcpyDeviceToHost, s));
        if (odp_status ss = sync_stream(g, s)) return ss;
        long long s0 = g->h_state->steps;
        int chunk = 2;
        std::vector<int> step_of_launch;
        while (g->h_state->active) {
            launches.clear();
            step_of_launch.clear();
            ev_next = 0;
            const bool sp_now = single && have_amax;
            if (graphs && chunk >= GS && (!single || have_amax)) {
                cudaGraphExec_t ex = nullptr;
                if ((rs = graph_of(sp_now ? 1 : 0, cur & 1, &ex))) return rs;
                for (int r = 0; r < (chunk + GS - 1) / GS; ++r) {
                    CUDA_TRY(cudaGraphLaunch(ex, s));
                    g->launches += glaunch[sp_now ? 1 : 0];
                }
            } else {
                for (int j = 0; j < chunk; ++j) {
                    if ((rs = step((cur + j) & 1, single && have_amax))) return rs;
                    have_amax = true;
                    while (step_of_launch.size() < launches.size()) step_of_launch.push_back(j);
                }
            }
            CUDA_TRY(cudaGetLastError());
            if (cst) return cst;
            CUDA_TRY(cudaMemcpyAsync(g->h_state, g->d_state, sizeof(DevState), cudaMemcpyDeviceToHost, s));
            if (odp_status ss = sync_stream(g, s)) return ss;
            const long long done = g->h_state->steps - s0;
            s0 = g->h_state->steps;
            if (accuracy == ODP_LOW && (done & 1)) cur ^= 1;
            if (timed) {
                for (size_t q = 0; q < launches.size(); ++q) {
                    if (step_of_launch[q] >= done) continue;      // launches that found the interval done
                    float ms = 0.f;
                    CUDA_TRY(cudaEventElapsedTime(&ms, g->events[launches[q].ev], g->events[launches[q].ev + 1]));
                    kms[launches[q].kind == 3 ? 1 : launches[q].kind] += ms;
                    if (launches[q].kind == 3) kms[3] += ms;
                }
            }
            if (g->h_state->status) { rs = ODP_ENUMERIC; break; }
            // size the next chunk from the remaining time and the current dt (+1 for the clipped step)
            const double rem = g->h_state->tau_target - g->h_state->tau;
            const long long est = g->h_state->dt > 0 ? (long long)std::ceil(rem / g->h_state->dt) + 1 : 2;
            chunk = (int)std::max<long long>(1, std::min<long long>(est, 256));
        }
        if (rs != ODP_OK) break;
        CUDA_TRY(cudaMemcpyAsync(out + (size_t)k_out * local_points(g), buf[accuracy == ODP_LOW ? cur : 0], bytes,
                                 cudaMemcpyDeviceToDevice, s));
        ++k_out;
    }
    if (rs == ODP_OK) {
        // final guard on the last V (reading A19)
        const float *Wf = buf[accuracy == ODP_LOW ? cur : 0];
        k_force_active<<<1, 1, 0, s>>>(g->d_state);
        if (split) {
            split_pass1(const_cast<float *>(Wf));
            ++g->launches;
        } else {
            exch(const_cast<float *>(Wf));
            launch_pass1(Wf);
        }
        launch_fin(0, 1);
        if (cst) return cst;
        g->launches += 3;
        CUDA_TRY(cudaGetLastError());
        CUDA_TRY(cudaMemcpyAsync(g->h_state, g->d_state, sizeof(DevState), cudaMemcpyDeviceToHost, s));
        if (odp_status ss = sync_stream(g, s)) return ss;
        if (g->h_state->status) rs = ODP_ENUMERIC;
    }
    if (opts) {
        if (opts->tau_reached) *opts->tau_reached = g->h_state->tau;
        if (opts->steps_taken) *opts->steps_taken = g->h_state->steps;
        if (opts->stages_taken) *opts->stages_taken = g->h_state->stages;
        if (opts->kernel_ms) for (int q = 0; q < 4; ++q) opts->kernel_ms[q] = kms[q];
        if (opts->single_pass_used) *opts->single_pass_used = single ? 1 : 0;
    }
    if (rs == ODP_ENUMERIC)
        return fail(ODP_ENUMERIC, "numerical failure (NaN or |V| > 1e10) at tau = %.9g", g->h_state->tau);
    return rs;
}

extern "C" odp_status odp_hj_solve(odp_grid *g, int dynamics_id, const double *params, int nparams, const float *V0,
                                   const double *tau, int ntau, int accuracy, int mode, float *out,
                                   const odp_solve_opts *opts) {
    g_err.clear();
    NvtxRange nv("odp_hj_solve");
    return solve_device(g, dynamics_id, params, nparams, V0, tau, ntau, accuracy, mode, out, opts);
}

extern "C" odp_status odp_hj_solve_host(odp_grid *g, int dynamics_id, const double *params, int nparams,
                                        const float *V0, const double *tau, int ntau, int accuracy, int mode,
                                        float *out, const odp_solve_opts *opts) {
    g_err.clear();
    NvtxRange nv("odp_hj_solve_host");
    odp_status st = validate(g, dynamics_id, params, nparams, tau, ntau, accuracy, mode);
    if (st) return st;
    if (!V0 || !out) return fail(ODP_EINVAL, "NULL V0/out");
    if ((st = ensure_device(g, 1))) return st;
    const int nout = (opts && opts->write_initial) ? ntau : ntau - 1;
    const size_t P = (size_t)local_points(g), bytes = P * sizeof(float);
    StreamScope sscope(g, opts ? opts->stream : nullptr);
    cudaStream_t s = sscope.s;
    const bool has_t = opts && opts->target;
    float *base = nullptr;
    if ((st = stage_buffer(g, P * (size_t)(1 + nout + (has_t ? 1 : 0)), &base))) return st;
    float *dV0 = base, *dout = base + P, *dT = has_t ? base + P * (size_t)(1 + nout) : nullptr;
    odp_solve_opts o;
    memset(&o, 0, sizeof o);
    if (opts) o = *opts;
    o.stream = s;
    if (has_t) {
        CUDA_TRY(cudaMemcpyAsync(dT, opts->target, bytes, cudaMemcpyHostToDevice, s));
        o.target = dT;
    }
    CUDA_TRY(cudaMemcpyAsync(dV0, V0, bytes, cudaMemcpyHostToDevice, s));
    st = solve_device(g, dynamics_id, params, nparams, dV0, tau, ntau, accuracy, mode, dout, &o);
    if (st == ODP_OK || st == ODP_ENUMERIC) {
        cudaError_t e = cudaMemcpyAsync(out, dout, bytes * nout, cudaMemcpyDeviceToHost, s);
        if (e == cudaSuccess) e = cudaStreamSynchronize(s);
        if (e != cudaSuccess && st == ODP_OK) st = fail(ODP_ECUDA, "copy out: %s", cudaGetErrorString(e));
    }
    cudaStreamSynchronize(s);
    return st;
}

// ------------------------------------------------------------------------------------------------
// time-to-reach (Algorithm 3; readings A31-A35)
// ------------------------------------------------------------------------------------------------
template <template <int> class FH>
static TtrFns ttr_holo(int n) {
    switch (n) {
    case 1: return ttr_fns<FH<1>, 1>();
    case 2: return ttr_fns<FH<2>, 2>();
    case 3: return ttr_fns<FH<3>, 3>();
    case 4: return ttr_fns<FH<4>, 4>();
    case 5: return ttr_fns<FH<5>, 5>();
    default: return ttr_fns<FH<6>, 6>();
    }
}

static TtrFns ttr_select(int dyn, int n) {
    switch (dyn) {
    case ODP_DYN_HOLONOMIC_BALL: return ttr_holo<FHoloBall>(n);
    case ODP_DYN_HOLONOMIC_BOX: return ttr_holo<FHoloBox>(n);
    case ODP_DYN_DUBINS3D: return ttr_fns<FDubins3D, 3>();
    case ODP_DYN_CAR4D: return ttr_fns<FCar4D, 4>();
    case ODP_DYN_CAR5D: return ttr_fns<FCar5D, 5>();
    case ODP_DYN_PAIR_DUBINS3D: return ttr_fns<FPairDubins3D, 3>();
    default: return ttr_fns<FDoubleInt6D, 6>();
    }
}

// ------------------------------------------------------------------------------------------------
// iterate-to-convergence driver shared by time-to-reach (Alg. 3) and value iteration (Alg. 1):
// chunks of G iterations (direct launches or one CUDA graph per chunk), each iteration's launches
// early-exit once the device state says done; the host reads the 40-byte TtrState per chunk.
// launch_iter(k, ev) launches iteration k of a chunk (k even: buffer 0 -> 1), recording ev[0..2]
// around its two launch groups when ev is non-null (per-launch timing, direct launches only).
// ------------------------------------------------------------------------------------------------
static odp_status iterate_to_convergence(odp_grid *g, cudaStream_t s, int per_iter, bool use_graph, bool per_launch,
                                         const std::function<void(int, const cudaEvent_t *)> &launch_iter,
                                         double *ms_total, double *ms_a, double *ms_b) {
    const int G = 16;                                           // iterations per chunk (even)
    std::vector<cudaEvent_t> pev;
    struct EvGuard { std::vector<cudaEvent_t> &v; ~EvGuard() { for (auto e : v) cudaEventDestroy(e); } } pev_guard{pev};
    if (per_launch) {
        pev.resize(3 * G);
        for (auto &e : pev) CUDA_TRY(cudaEventCreate(&e));
    }
    auto chunk = [&](void) -> cudaError_t {
        for (int k = 0; k < G; ++k) launch_iter(k, per_launch ? &pev[3 * k] : nullptr);
        return cudaGetLastError();
    };
    cudaGraphExec_t exec = nullptr;
    if (use_graph) {
        cudaGraph_t graph = nullptr;
        CUDA_TRY(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
        cudaError_t e = chunk();
        cudaError_t e2 = cudaStreamEndCapture(s, &graph);
        if (e != cudaSuccess || e2 != cudaSuccess) {
            if (graph) cudaGraphDestroy(graph);
            return fail(ODP_ECUDA, "graph capture: %s", cudaGetErrorString(e != cudaSuccess ? e : e2));
        }
        e = cudaGraphInstantiate(&exec, graph, 0);
        cudaGraphDestroy(graph);
        if (e != cudaSuccess) return fail(ODP_ECUDA, "graph instantiate: %s", cudaGetErrorString(e));
    }
    cudaEvent_t ev[2];
    CUDA_TRY(cudaEventCreate(&ev[0]));
    CUDA_TRY(cudaEventCreate(&ev[1]));
    *ms_total = 0.0; *ms_a = 0.0; *ms_b = 0.0;
    long long iters_before = 0;
    odp_status rs = ODP_OK;
    int reps = 1;                       // graph replays per host check: 1, 2, 4, 8 (long solves sync rarely)
    for (;;) {
        cudaError_t e = cudaEventRecord(ev[0], s);
        if (use_graph) {
            for (int r = 0; r < reps && e == cudaSuccess; ++r) e = cudaGraphLaunch(exec, s);
        } else if (e == cudaSuccess) {
            e = chunk();
        }
        if (e == cudaSuccess) e = cudaEventRecord(ev[1], s);
        if (e == cudaSuccess) e = cudaMemcpyAsync(g->h_ttr, g->d_ttr, sizeof(TtrState), cudaMemcpyDeviceToHost, s);
        if (e == cudaSuccess) e = cudaStreamSynchronize(s);
        if (e != cudaSuccess) { rs = fail(ODP_ECUDA, "iteration: %s", cudaGetErrorString(e)); break; }
        float ms = 0.f;
        cudaEventElapsedTime(&ms, ev[0], ev[1]);
        *ms_total += ms;
        g->launches += (long long)G * per_iter * (use_graph ? reps : 1);
        if (use_graph) reps = std::min(reps * 2, 8);
        if (per_launch) {                    // only the iterations that ran (the rest early-exit)
            const long long ran = g->h_ttr->iters - iters_before;
            for (int k = 0; k < G && k < ran; ++k) {
                float a = 0.f, b = 0.f;
                cudaEventElapsedTime(&a, pev[3 * k], pev[3 * k + 1]);
                cudaEventElapsedTime(&b, pev[3 * k + 1], pev[3 * k + 2]);
                *ms_a += a;
                *ms_b += b;
            }
        }
        iters_before = g->h_ttr->iters;
        if (g->h_ttr->done) break;
    }
    if (exec) cudaGraphExecDestroy(exec);
    cudaEventDestroy(ev[0]);
    cudaEventDestroy(ev[1]);
    return rs;
}

static odp_status ttr_device(odp_grid *g, int dyn, const double *params, int nparams, const float *V0, float *phi,
                             const odp_ttr_opts *opts) {
    odp_status st = validate_dyn(g, dyn, params, nparams);
    if (st) return st;
    if (!V0 || !phi) return fail(ODP_EINVAL, "NULL V0/phi");
    if (V0 == phi) return fail(ODP_EINVAL, "phi aliases V0");
    if (g->nranks > 1 || g->comm) return fail(ODP_EINVAL, "time-to-reach runs on an unpartitioned grid");
    for (int d = 0; d < g->n; ++d)
        if (!g->per[d] && g->N[d] < 4) return fail(ODP_EINVAL, "N[%d]=%lld < 4 on a non-periodic axis", d, (long long)g->N[d]);
    const double eps = (opts && opts->eps > 0.0) ? opts->eps : 1e-6;
    const long long max_iters = (opts && opts->max_iters > 0) ? opts->max_iters : 100000;
    const double big = (opts && opts->big > 0.0) ? opts->big : 100.0;
    const bool use_graph = opts ? opts->use_graph != 0 : true;
    if ((st = ensure_device(g, 1))) return st;
    if (!g->d_ttr) {
        CUDA_TRY(cudaMalloc(&g->d_ttr, sizeof(TtrState)));
        CUDA_TRY(cudaMallocHost(&g->h_ttr, sizeof(TtrState)));
    }
    StreamScope sscope(g, opts ? opts->stream : nullptr);
    cudaStream_t s = sscope.s;
    const int n = g->n;
    const TtrFns fn = ttr_select(dyn, n);
    GridDev gd = make_griddev(g);
    FParams fp;
    memset(&fp, 0, sizeof fp);
    for (int k = 0; k < nparams; ++k) fp.c[k] = (float)params[k];
    fp.c[nparams - 1] = -1.f;                                   // A32: the control minimises p.f
    int nsm = 148, dev = 0;
    CUDA_TRY(cudaGetDevice(&dev));
    CUDA_TRY(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    const int block = 256;
    const long long P = local_points(g);
    const int grid_all = (int)std::min<long long>((P + block - 1) / block, (long long)nsm * 8);
    const int NL = (int)g->N[n - 1];
    const long long rows = P / NL;
    const int RPB = NL >= block ? 1 : block / NL;
    const int grid_rows = (int)std::min<long long>((rows + RPB - 1) / RPB, (long long)nsm * 8);
    // march kernel: columns = one axis-0 plane; axis 0 split into segments so that ~8 CTAs per SM run
    const long long ncol = P / g->n0;
    const int col_blocks = (int)((ncol + block - 1) / block);
    int nseg = (int)std::max<long long>(1, std::min<long long>(g->n0, ((long long)nsm * 8 + col_blocks - 1) / col_blocks));
    const int seg_len = (int)((g->n0 + nseg - 1) / nseg);
    nseg = (int)((g->n0 + seg_len - 1) / seg_len);
    const dim3 grid_march(col_blocks, nseg);
    // tile kernel (NDIM >= 3): TY x TX in-plane tiles x middle-axis combinations x axis-0 segments
    const bool use_tile = fn.tile != nullptr && !(getenv("ODP_TTR_TILE") && atoi(getenv("ODP_TTR_TILE")) == 0);
    int ntx = 1, nty = 1, tile_seg = 1;
    dim3 grid_tile(1, 1);
    if (use_tile) {
        ntx = (int)((g->N[n - 1] + TTR_TW - 1) / TTR_TW);
        nty = (int)((g->N[n - 2] + TTR_TY - 1) / TTR_TY);
        long long nb = (long long)ntx * nty;
        for (int d = 1; d < n - 2; ++d) nb *= g->N[d];
        int ns = (int)std::max<long long>(1, std::min<long long>(g->n0, ((long long)nsm * 6 + nb - 1) / nb));
        tile_seg = (int)((g->n0 + ns - 1) / ns);
        ns = (int)((g->n0 + tile_seg - 1) / tile_seg);
        grid_tile = dim3((unsigned)nb, (unsigned)ns);
    }
    int grid_face[MAXD] = {0}, last_axis = -1;
    for (int d = 0; d < n; ++d) {
        grid_face[d] = (int)std::min<long long>((2 * (P / g->N[d]) + block - 1) / block, (long long)nsm * 8);
        if (!g->per[d]) last_axis = d;
    }
    float *buf[2] = {phi, g->d_buf[0] + g->halo_elems};
    g->launches = 0;

    k_ttr_reset<<<1, 1, 0, s>>>(g->d_ttr, max_iters, (float)eps, 0);
    k_ttr_init<<<grid_all, block, 0, s>>>(P, V0, (float)big, buf[0]);
    g->launches += 2;
    CUDA_TRY(cudaGetLastError());
    const int per_iter = 1 + [&] { int c = 0; for (int d = 0; d < n; ++d) c += g->per[d] ? 0 : 1; return c; }();
    const bool per_launch = opts && opts->kernel_ms && !use_graph;
    double ms_total = 0.0, ms_interior = 0.0, ms_faces = 0.0;
    st = iterate_to_convergence(g, s, per_iter, use_graph, per_launch, [&](int k, const cudaEvent_t *ev) {
        const int par = (k + 1) & 1;
        const float *src = buf[k & 1];
        float *dst = buf[par];
        if (ev) cudaEventRecord(ev[0], s);
        if (use_tile) fn.tile<<<grid_tile, TTR_TX * TTR_TY, 0, s>>>(gd, fp, src, dst, g->d_ttr, par, last_axis < 0 ? 1 : 0,
                                                                  tile_seg, ntx, nty);
        else if (fn.march) fn.march<<<grid_march, block, 0, s>>>(gd, fp, src, dst, g->d_ttr, par, last_axis < 0 ? 1 : 0, seg_len);
        else fn.rows<<<grid_rows, block, 0, s>>>(gd, fp, src, dst, g->d_ttr, par, last_axis < 0 ? 1 : 0);
        if (ev) cudaEventRecord(ev[1], s);
        for (int d = 0; d < n; ++d)
            if (!g->per[d]) fn.face<<<grid_face[d], block, 0, s>>>(gd, d, d == last_axis ? 1 : 0, src, dst, g->d_ttr, par);
        if (ev) cudaEventRecord(ev[2], s);
    }, &ms_total, &ms_interior, &ms_faces);
    if (st) return st;
    k_ttr_finish<<<grid_all, block, 0, s>>>(P, buf[g->h_ttr->parity], phi);
    g->launches += 1;
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaStreamSynchronize(s));
    if (opts) {
        if (opts->iters_taken) *opts->iters_taken = g->h_ttr->iters;
        if (opts->last_change) *opts->last_change = (double)__builtin_bit_cast(float, g->h_ttr->change[g->h_ttr->parity]);
        if (opts->kernel_ms) {
            opts->kernel_ms[0] = ms_total;
            opts->kernel_ms[1] = per_launch ? ms_interior : -1.0;
            opts->kernel_ms[2] = per_launch ? ms_faces : -1.0;
        }
    }
    return ODP_OK;
}

extern "C" odp_status odp_ttr_solve(odp_grid *g, int dynamics_id, const double *params, int nparams,
                                    const float *V0, float *phi, const odp_ttr_opts *opts) {
    g_err.clear();
    NvtxRange nv("odp_ttr_solve");
    return ttr_device(g, dynamics_id, params, nparams, V0, phi, opts);
}

extern "C" odp_status odp_ttr_solve_host(odp_grid *g, int dynamics_id, const double *params, int nparams,
                                         const float *V0, float *phi, const odp_ttr_opts *opts) {
    g_err.clear();
    odp_status st = validate_dyn(g, dynamics_id, params, nparams);
    if (st) return st;
    if (!V0 || !phi) return fail(ODP_EINVAL, "NULL V0/phi");
    if ((st = ensure_device(g, 1))) return st;
    const size_t bytes = (size_t)local_points(g) * sizeof(float);
    StreamScope sscope(g, opts ? opts->stream : nullptr);
    cudaStream_t s = sscope.s;
    float *dV0 = nullptr, *dphi = nullptr;
    if ((st = stage_buffer(g, 2 * (size_t)local_points(g), &dV0))) return st;
    dphi = dV0 + local_points(g);
    odp_ttr_opts o;
    memset(&o, 0, sizeof o);
    if (opts) o = *opts; else o.use_graph = 1;
    o.stream = s;
    CUDA_TRY(cudaMemcpyAsync(dV0, V0, bytes, cudaMemcpyHostToDevice, s));
    st = ttr_device(g, dynamics_id, params, nparams, dV0, dphi, &o);
    if (st == ODP_OK) {
        cudaError_t e = cudaMemcpyAsync(phi, dphi, bytes, cudaMemcpyDeviceToHost, s);
        if (e == cudaSuccess) e = cudaStreamSynchronize(s);
        if (e != cudaSuccess) st = fail(ODP_ECUDA, "copy out: %s", cudaGetErrorString(e));
    }
    cudaStreamSynchronize(s);
    return st;
}

// ------------------------------------------------------------------------------------------------
// value iteration (Algorithm 1; readings A36-A38)
// ------------------------------------------------------------------------------------------------
static odp_status vi_device(odp_grid *g, int model, const double *params, int nparams, const float *R, float *V,
                            const odp_vi_opts *opts) {
    if (!g) return fail(ODP_EINVAL, "NULL grid");
    if (model != ODP_MDP_HOLONOMIC && model != ODP_MDP_DUBINS3D) return fail(ODP_EINVAL, "unknown MDP model %d", model);
    const int want = model == ODP_MDP_HOLONOMIC ? 3 : 6;
    if (!params || nparams != want) return fail(ODP_EINVAL, "MDP model %d takes %d params (got %d)", model, want, nparams);
    for (int k = 0; k < nparams; ++k) if (!std::isfinite(params[k])) return fail(ODP_EINVAL, "param %d not finite", k);
    if (model == ODP_MDP_DUBINS3D && g->n != 3) return fail(ODP_EINVAL, "MDP model 1 needs dims=3 (grid has %d)", g->n);
    const double gamma = params[nparams - 1];
    if (!(gamma >= 0.0 && gamma < 1.0)) return fail(ODP_EINVAL, "gamma must be in [0, 1)");
    if (model == ODP_MDP_DUBINS3D && !(params[4] >= 0.0 && params[4] <= 0.5)) return fail(ODP_EINVAL, "pslip must be in [0, 0.5]");
    if (!R || !V) return fail(ODP_EINVAL, "NULL R/V");
    if (R == V) return fail(ODP_EINVAL, "V aliases R");
    if (g->nranks > 1 || g->comm) return fail(ODP_EINVAL, "value iteration runs on an unpartitioned grid");
    const double thr = (opts && opts->threshold > 0.0) ? opts->threshold : 1e-6;
    const long long max_iters = (opts && opts->max_iters > 0) ? opts->max_iters : 100000;
    const bool fixed = opts && opts->fixed_iters;
    const bool use_graph = opts ? opts->use_graph != 0 : true;
    odp_status st;
    if ((st = ensure_device(g, 1))) return st;
    if (!g->d_ttr) {
        CUDA_TRY(cudaMalloc(&g->d_ttr, sizeof(TtrState)));
        CUDA_TRY(cudaMallocHost(&g->h_ttr, sizeof(TtrState)));
    }
    StreamScope sscope(g, opts ? opts->stream : nullptr);
    cudaStream_t s = sscope.s;
    MdpParams mp;
    memset(&mp, 0, sizeof mp);
    if (model == ODP_MDP_HOLONOMIC) {
        mp.step = (float)params[1] * (float)params[0];
        mp.p[0] = 1.f;
    } else {
        mp.vbar = (float)params[0]; mp.wbar = (float)params[1]; mp.dt = (float)params[2]; mp.slip = (float)params[3];
        mp.p[0] = (float)(1.0 - 2.0 * params[4]); mp.p[1] = mp.p[2] = (float)params[4];
    }
    mp.gamma = (float)gamma;
    const vi_march_fn fn = vi_select(model, g->n);
    GridDev gd = make_griddev(g);
    int nsm = 148, dev = 0;
    CUDA_TRY(cudaGetDevice(&dev));
    CUDA_TRY(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    const int block = 256;
    const long long P = local_points(g);
    const long long ncol = P / g->n0;
    const int col_blocks = (int)((ncol + block - 1) / block);
    int nseg = (int)std::max<long long>(1, std::min<long long>(g->n0, ((long long)nsm * 8 + col_blocks - 1) / col_blocks));
    const int seg_len = (int)((g->n0 + nseg - 1) / nseg);
    nseg = (int)((g->n0 + seg_len - 1) / seg_len);
    const dim3 grid_march(col_blocks, nseg);
    float *buf[2] = {V, g->d_buf[0] + g->halo_elems};
    g->launches = 0;
    k_ttr_reset<<<1, 1, 0, s>>>(g->d_ttr, max_iters, fixed ? -1.f : (float)thr, 1);
    CUDA_TRY(cudaMemsetAsync(buf[0], 0, (size_t)P * sizeof(float), s));           // l.2: V_0 = 0
    g->launches += 1;
    CUDA_TRY(cudaGetLastError());
    const bool per_launch = opts && opts->kernel_ms && !use_graph;
    double ms_total = 0.0, ms_iter = 0.0, ms_unused = 0.0;
    st = iterate_to_convergence(g, s, 1, use_graph, per_launch, [&](int k, const cudaEvent_t *ev) {
        const int par = (k + 1) & 1;
        if (ev) cudaEventRecord(ev[0], s);
        fn<<<grid_march, block, 0, s>>>(gd, mp, R, buf[k & 1], buf[par], g->d_ttr, par, seg_len);
        if (ev) { cudaEventRecord(ev[1], s); cudaEventRecord(ev[2], s); }
    }, &ms_total, &ms_iter, &ms_unused);
    if (st) return st;
    if (g->h_ttr->parity == 1) {
        CUDA_TRY(cudaMemcpyAsync(V, buf[1], (size_t)P * sizeof(float), cudaMemcpyDeviceToDevice, s));
    }
    CUDA_TRY(cudaStreamSynchronize(s));
    if (opts) {
        if (opts->iters_taken) *opts->iters_taken = g->h_ttr->iters;
        if (opts->last_change) *opts->last_change = (double)__builtin_bit_cast(float, g->h_ttr->change[g->h_ttr->parity]);
        if (opts->kernel_ms) {
            opts->kernel_ms[0] = ms_total;
            opts->kernel_ms[1] = per_launch ? ms_iter : -1.0;
        }
    }
    return ODP_OK;
}

extern "C" odp_status odp_vi_solve(odp_grid *g, int model_id, const double *params, int nparams, const float *R,
                                   float *V, const odp_vi_opts *opts) {
    g_err.clear();
    NvtxRange nv("odp_vi_solve");
    return vi_device(g, model_id, params, nparams, R, V, opts);
}

extern "C" odp_status odp_vi_solve_host(odp_grid *g, int model_id, const double *params, int nparams,
                                        const float *R, float *V, const odp_vi_opts *opts) {
    g_err.clear();
    if (!g) return fail(ODP_EINVAL, "NULL grid");
    if (!R || !V) return fail(ODP_EINVAL, "NULL R/V");
    odp_status st;
    if ((st = ensure_device(g, 1))) return st;
    const size_t bytes = (size_t)local_points(g) * sizeof(float);
    StreamScope sscope(g, opts ? opts->stream : nullptr);
    cudaStream_t s = sscope.s;
    float *dR = nullptr, *dV = nullptr;
    if ((st = stage_buffer(g, 2 * (size_t)local_points(g), &dR))) return st;
    dV = dR + local_points(g);
    odp_vi_opts o;
    memset(&o, 0, sizeof o);
    if (opts) o = *opts; else o.use_graph = 1;
    o.stream = s;
    CUDA_TRY(cudaMemcpyAsync(dR, R, bytes, cudaMemcpyHostToDevice, s));
    st = vi_device(g, model_id, params, nparams, dR, dV, &o);
    if (st == ODP_OK) {
        cudaError_t e = cudaMemcpyAsync(V, dV, bytes, cudaMemcpyDeviceToHost, s);
        if (e == cudaSuccess) e = cudaStreamSynchronize(s);
        if (e != cudaSuccess) st = fail(ODP_ECUDA, "copy out: %s", cudaGetErrorString(e));
    }
    cudaStreamSynchronize(s);
    return st;
}
