// L2 -> SM bandwidth microbenchmark (design input for the stencil kernels, not product code).
// A buffer of S bytes is read over and over by every CTA:
//   mode 0: 1-D TMA bulk copies (cp.async.bulk) of CHUNK bytes into a ring of NBUF smem slots,
//           one elected thread issues, every warp waits on the slot's mbarrier (like k_march)
//   mode 1: LDG.128 by every thread (coalesced), summed so nothing is dead
// S = 48 MB stays L2-resident (126 MB L2); S = 4 GB measures DRAM.  Prints GB/s.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o l2bw tools/l2bw.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int NBUF>
__global__ void __launch_bounds__(256) k_tma(const float *src, size_t nchunks, int chunk, int iters, float *out) {
    extern __shared__ __align__(128) unsigned char sm[];
    __shared__ __align__(8) uint64_t bar[NBUF];
    if (threadIdx.x == 0) {
        for (int b = 0; b < NBUF; ++b) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[b])));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    float acc = 0.f;
    size_t c = (size_t)blockIdx.x * 7919u % nchunks;
    auto issue = [&](int b, size_t ch) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar[b])), "r"(chunk) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"(su32(sm + (size_t)b * chunk)), "l"((const char *)src + ch * chunk), "r"(chunk), "r"(su32(&bar[b])) : "memory");
    };
    const int total = iters;
    if (threadIdx.x == 0)
        for (int b = 0; b < NBUF && b < total; ++b) { issue(b, c); c = (c + gridDim.x) % nchunks; }
    for (int it = 0; it < total; ++it) {
        const int b = it % NBUF;
        const uint32_t ph = (it / NBUF) & 1;
        asm volatile("{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W;\n}" ::"r"(su32(&bar[b])), "r"(ph) : "memory");
        acc += reinterpret_cast<const float *>(sm + (size_t)b * chunk)[threadIdx.x];
        __syncthreads();
        if (threadIdx.x == 0 && it + NBUF < total) { issue(b, c); c = (c + gridDim.x) % nchunks; }
    }
    if (acc == 1234.5f) out[0] = acc;
}

__global__ void __launch_bounds__(256) k_ldg(const float4 *src, size_t n4, int iters, float *out) {
    float4 a = make_float4(0, 0, 0, 0);
    size_t i = ((size_t)blockIdx.x * 7919u * 256 + threadIdx.x) % n4;
    const size_t stride = (size_t)gridDim.x * 256;
    for (int it = 0; it < iters; ++it) {
        float4 v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) { v[u] = __ldcg(src + i); i += stride; if (i >= n4) i -= n4; }
#pragma unroll
        for (int u = 0; u < 4; ++u) { a.x += v[u].x; a.y += v[u].y; a.z += v[u].z; a.w += v[u].w; }
    }
    if (a.x + a.y + a.z + a.w == 1234.5f) out[0] = a.x;
}

int main() {
    int sm;
    cudaDeviceGetAttribute(&sm, cudaDevAttrMultiProcessorCount, 0);
    float *out;
    cudaMalloc(&out, 4);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (size_t S : {(size_t)48 << 20, (size_t)4 << 30}) {
        char *buf;
        cudaMalloc(&buf, S);
        cudaMemset(buf, 1, S);
        for (int chunk : {1024, 3600, 4096, 16384}) {
            for (int occ : {1, 2, 4}) {
                const int nbuf = 8;
                const size_t smem = (size_t)nbuf * chunk;
                if (smem > 200 * 1024 / occ) continue;
                cudaFuncSetAttribute(k_tma<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
                const size_t nch = S / chunk;
                const int iters = (int)((size_t)256 << 20) / chunk / (sm * occ) + 8;   // ~256 MB per launch... x16 below
                const int it2 = iters * 16;
                k_tma<8><<<sm * occ, 256, smem>>>((const float *)buf, nch, chunk, it2, out);
                cudaEventRecord(e0);
                k_tma<8><<<sm * occ, 256, smem>>>((const float *)buf, nch, chunk, it2, out);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                float ms;
                cudaEventElapsedTime(&ms, e0, e1);
                const double bytes = (double)sm * occ * it2 * chunk;
                printf("S=%5zu MB TMA chunk=%5d CTAs/SM=%d : %7.1f GB/s  (%s)\n", S >> 20, chunk, occ, bytes / ms / 1e6,
                       cudaGetErrorString(cudaGetLastError()));
            }
        }
        for (int occ : {2, 4, 8}) {
            const size_t n4 = S / 16;
            const int iters = 4096;
            k_ldg<<<sm * occ, 256>>>((const float4 *)buf, n4, iters, out);
            cudaEventRecord(e0);
            k_ldg<<<sm * occ, 256>>>((const float4 *)buf, n4, iters, out);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            const double bytes = (double)sm * occ * 256 * iters * 4 * 16;
            printf("S=%5zu MB LDG.128 CTAs/SM=%d : %7.1f GB/s  (%s)\n", S >> 20, occ, bytes / ms / 1e6,
                   cudaGetErrorString(cudaGetLastError()));
        }
        cudaFree(buf);
    }
    return 0;
}
