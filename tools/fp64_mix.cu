// Are DMMA and DFMA separate pipes on B200, and what saturates DMMA?  (diagnostics)
// mode 0: all warps DMMA; 1: all DFMA; 2: even warps DMMA + odd warps DFMA;
// 3: even warps DMMA, odd idle; 4: odd warps DFMA, even idle.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}
template <int NACC>
__global__ void mix(double* out, int iters, int mode) {
  const int warp = threadIdx.x >> 5;
  const int half = (warp >> 2) & 1;  // same SMSP mix: warps 0-3 vs 4-7, ...
  if ((mode == 3 && half) || (mode == 4 && half == 0)) return;
  const bool do_mma = mode == 0 || ((mode == 2 || mode == 3) && half == 0);
  double s = 0;
  if (do_mma) {
    double acc[NACC][2];
    double a = 1.0 + threadIdx.x * 1e-12, b = 1.0 - threadIdx.x * 1e-12;
    for (int i = 0; i < NACC; ++i) acc[i][0] = acc[i][1] = 0;
    for (int it = 0; it < iters; ++it)
#pragma unroll
      for (int i = 0; i < NACC; ++i) dmma884(acc[i][0], acc[i][1], a, b);
    for (int i = 0; i < NACC; ++i) s += acc[i][0] + acc[i][1];
  } else {
    double x[NACC];
    for (int i = 0; i < NACC; ++i) x[i] = threadIdx.x * 1e-9 + i;
    for (int it = 0; it < iters; ++it)
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int i = 0; i < NACC; ++i) x[i] = fma(x[i], 0.999999, 1e-7);
    for (int i = 0; i < NACC; ++i) s += x[i];
  }
  if (s == 12345.678) out[0] = s;
}
template <int NACC>
void run(int threads, double* out, int sms) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 4096, grid = sms;
  for (int mode = 0; mode < 5; ++mode) {
    mix<NACC><<<grid, threads>>>(out, 16, mode);
    cudaEventRecord(e0);
    mix<NACC><<<grid, threads>>>(out, iters, mode);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    const double warps = grid * threads / 32.0;
    const double mma_w = mode == 0 ? warps : (mode == 2 || mode == 3 ? warps / 2 : 0);
    const double fma_w = mode == 1 ? warps : (mode == 2 || mode == 4 ? warps / 2 : 0);
    const double fm = mma_w * iters * NACC * 512.0, ff = fma_w * 32 * iters * NACC * 4 * 2.0;
    printf("chains %2d threads %4d mode %d: %.3f ms  DMMA %.1f TF  DFMA %.1f TF  total %.1f TF\n", NACC, threads, mode,
           ms, fm / ms / 1e9, ff / ms / 1e9, (fm + ff) / ms / 1e9);
  }
}
int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  double* out; cudaMalloc(&out, 64);
  run<8>(512, out, p.multiProcessorCount);
  run<16>(512, out, p.multiProcessorCount);
  run<8>(1024, out, p.multiProcessorCount);
  return 0;
}
