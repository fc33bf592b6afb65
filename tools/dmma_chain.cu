// DMMA.8x8x4 issue rate vs warps per SMSP and independent accumulator chains per warp
// (one CTA per SM).  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/dmma_chain tools/dmma_chain.cu
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}
template <int NC>
__global__ void k(double* out, int iters) {
  double acc[NC][2];
  double a = 1.0 + threadIdx.x * 1e-12, b = 1.0 - threadIdx.x * 1e-12;
#pragma unroll
  for (int i = 0; i < NC; ++i) acc[i][0] = acc[i][1] = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NC; ++i) dmma(acc[i][0], acc[i][1], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NC; ++i) s += acc[i][0] + acc[i][1];
  if (s == 12345.0) out[0] = s;
}
template <int NC>
void run(int warps, int sms, double* out) {
  int iters = 4096 * 8 / NC;
  k<NC><<<sms, 32 * warps>>>(out, 16);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<NC><<<sms, 32 * warps>>>(out, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double dm = (double)iters * NC * warps * sms;
  printf("{\"test\": \"dmma_chain\", \"warps_per_sm\": %d, \"chains\": %d, \"tflops\": %.2f, \"clk_per_dmma_per_smsp\": %.2f}\n",
         warps, NC, dm * 512 / ms / 1e9, ms * 1e-3 * 1.965e9 / (dm / sms / 4));
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out; cudaMalloc(&out, 8);
  for (int w : {4, 8, 12, 16}) {
    run<1>(w, sms, out); run<2>(w, sms, out); run<4>(w, sms, out); run<6>(w, sms, out); run<8>(w, sms, out);
  }
  return 0;
}
