// Issue-rate microbenchmark for the instruction classes the HJ stencil kernels use (FFMA, FFMA2,
// FADD2, FMNMX, FMNMX3, FSETP+FSEL pick, mixes).  Prints warp-instructions / cycle / SM.
#include <cstdio>
#include <cuda_runtime.h>
#define NCH 8
#define ITERS 4096
__device__ __forceinline__ float min3f(float a, float b, float c) { float r; asm("min.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c)); return r; }

template <int K> __global__ void kb(float *o, float a, float b) {
  float x[NCH], y[NCH]; float2 z[NCH];
  for (int c = 0; c < NCH; ++c) { x[c] = threadIdx.x * 1e-3f + c; y[c] = x[c] * 0.5f; z[c] = make_float2(x[c], y[c]); }
  const float2 A = make_float2(a, a), B = make_float2(b, b);
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int c = 0; c < NCH; ++c) {
      if (K == 0) x[c] = fmaf(x[c], a, b);
      if (K == 1) z[c] = __ffma2_rn(z[c], A, B);
      if (K == 2) z[c] = __fadd2_rn(z[c], B);
      if (K == 3) x[c] = fminf(x[c], y[c] + 0.f), y[c] = fmaxf(y[c], x[c]);
      if (K == 4) x[c] = min3f(x[c], y[c], a), y[c] = min3f(y[c], x[c], b);
      if (K == 5) { x[c] = fabsf(x[c]) <= fabsf(y[c]) ? y[c] : x[c]; }
      if (K == 6) { z[c] = __ffma2_rn(z[c], A, B); x[c] = fminf(x[c], y[c]); }
      if (K == 7) { x[c] = fmaf(x[c], a, b); y[c] = fminf(y[c], b); }
      if (K == 8) { z[c] = __ffma2_rn(z[c], A, B); x[c] = fmaf(x[c], a, b); }
    }
  }
  float s = 0; for (int c = 0; c < NCH; ++c) s += x[c] + y[c] + z[c].x + z[c].y;
  if (s == 12345.f) o[0] = s;
}
int main() {
  float *o; cudaMalloc(&o, 4);
  int sm; cudaDeviceGetAttribute(&sm, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const char *names[] = {"FFMA", "FFMA2", "FADD2", "FMNMX x2", "FMNMX3 x2", "FSETP+FSEL", "FFMA2+FMNMX", "FFMA+FMNMX", "FFMA2+FFMA"};
  const double ipc_inst[] = {1, 1, 1, 2, 2, 2, 2, 2, 2};   // warp instructions per chain-iteration
  void (*ks[])(float *, float, float) = {kb<0>, kb<1>, kb<2>, kb<3>, kb<4>, kb<5>, kb<6>, kb<7>, kb<8>};
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int k = 0; k < 9; ++k) {
    for (int occ : {4, 8}) {
      const int blocks = sm * occ, thr = 256;
      ks[k]<<<blocks, thr>>>(o, 1.0001f, 1e-7f);
      cudaEventRecord(e0);
      ks[k]<<<blocks, thr>>>(o, 1.0001f, 1e-7f);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      const double winst = (double)blocks * thr / 32 * ITERS * NCH * ipc_inst[k];
      const double cyc = ms * 1e-3 * clk * 1e3;   // at the nominal max clock
      printf("%-14s warps/SMSP=%2d  %.3f ms  warp-inst/clk/SM = %.2f\n", names[k], occ * 8 / 4, ms, winst / cyc / sm);
    }
  }
  return 0;
}
