// FP64 roofline microbenchmarks for B200 (sm_100a): DFMA and DMMA (mma.sync f64)
// peaks, plus a single-warp check of the m8n8k4 f64 fragment layout that the
// tall-panel kernels rely on.  Build: see tools/run_peaks.sh.  Prints JSON lines.
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1);} } while (0)

__global__ void dfma_loop(double* out, int iters, double a, double b) {
  double x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-9 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 16; ++r)
#pragma unroll
      for (int i = 0; i < 8; ++i) x[i] = fma(x[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += x[i];
  if (s == 12345.678) out[0] = s;
}

__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

template <int NACC>
__global__ void dmma_loop(double* out, int iters) {
  double acc[NACC][2];
  double a = 1.0 + threadIdx.x * 1e-12, b = 1.0 - threadIdx.x * 1e-12;
#pragma unroll
  for (int i = 0; i < NACC; ++i) { acc[i][0] = 0; acc[i][1] = 0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) dmma884(acc[i][0], acc[i][1], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += acc[i][0] + acc[i][1];
  if (s == 12345.678) out[0] = s;
}

// one warp: D = A(8x4, row-major) * B(4x8) using the documented fragment map
__global__ void dmma_layout(const double* A, const double* B, double* D) {
  int lane = threadIdx.x;
  double a = A[(lane >> 2) * 4 + (lane & 3)];          // row=g, col=t
  double b = B[(lane & 3) * 8 + (lane >> 2)];          // row=t, col=g
  double d0 = 0, d1 = 0;
  dmma884(d0, d1, a, b);
  int r = lane >> 2, c = (lane & 3) * 2;
  D[r * 8 + c] = d0;
  D[r * 8 + c + 1] = d1;
}

int main() {
  int dev = 0; cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, dev));
  int sms = p.multiProcessorCount;
  double* out; CK(cudaMalloc(&out, 64));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  // layout check
  {
    double hA[32], hB[32], hD[64], ref[64];
    for (int i = 0; i < 32; ++i) { hA[i] = 1 + i; hB[i] = 0.5 * (i % 7) - 1; }
    for (int r = 0; r < 8; ++r) for (int c = 0; c < 8; ++c) {
      double s = 0; for (int k = 0; k < 4; ++k) s += hA[r * 4 + k] * hB[k * 8 + c]; ref[r * 8 + c] = s; }
    double *dA, *dB, *dD; CK(cudaMalloc(&dA, 256)); CK(cudaMalloc(&dB, 256)); CK(cudaMalloc(&dD, 512));
    CK(cudaMemcpy(dA, hA, 256, cudaMemcpyHostToDevice)); CK(cudaMemcpy(dB, hB, 256, cudaMemcpyHostToDevice));
    dmma_layout<<<1, 32>>>(dA, dB, dD); CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(hD, dD, 512, cudaMemcpyDeviceToHost));
    double err = 0; for (int i = 0; i < 64; ++i) err = fmax(err, fabs(hD[i] - ref[i]));
    printf("{\"test\": \"dmma_m8n8k4_layout\", \"max_abs_err\": %.3e}\n", err);
  }
  for (int blocksPerSm : {1, 2, 4}) {
    int iters = 4096, threads = 256, grid = sms * blocksPerSm;
    dfma_loop<<<grid, threads>>>(out, 16, 1.0000001, 1e-9); CK(cudaDeviceSynchronize());
    cudaEventRecord(e0); dfma_loop<<<grid, threads>>>(out, iters, 1.0000001, 1e-9); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1)); float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 8 * 16 * (double)iters * grid * threads;
    printf("{\"test\": \"dfma_peak\", \"blocks_per_sm\": %d, \"tflops\": %.3f, \"ms\": %.3f}\n", blocksPerSm, flops / ms / 1e9, ms);
  }
  for (int warps : {4, 8, 16}) {
    int iters = 8192, grid = sms * 2, threads = 32 * warps;
    dmma_loop<8><<<grid, threads>>>(out, 16); CK(cudaDeviceSynchronize());
    cudaEventRecord(e0); dmma_loop<8><<<grid, threads>>>(out, iters); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1)); float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 256 * 8 * (double)iters * grid * warps;
    printf("{\"test\": \"dmma_peak\", \"warps_per_block\": %d, \"blocks\": %d, \"tflops\": %.3f, \"ms\": %.3f}\n", warps, grid, flops / ms / 1e9, ms);
  }
  // HBM copy (read + write bytes)
  {
    size_t n = (size_t)1 << 30;  // 1 Gi doubles per buffer = 8 GiB
    double *a, *b; CK(cudaMalloc(&a, n * 8)); CK(cudaMalloc(&b, n * 8));
    CK(cudaMemset(a, 0, n * 8));
    CK(cudaMemcpy(b, a, n * 8, cudaMemcpyDeviceToDevice)); CK(cudaDeviceSynchronize());
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(e0); CK(cudaMemcpyAsync(b, a, n * 8, cudaMemcpyDeviceToDevice)); cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1)); float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
    }
    printf("{\"test\": \"hbm_copy\", \"gbs\": %.1f}\n", 2.0 * n * 8 / best / 1e6);
  }
  printf("{\"test\": \"device\", \"name\": \"%s\", \"sms\": %d, \"l2_bytes\": %d, \"smem_optin\": %zu}\n",
         p.name, sms, p.l2CacheSize, p.sharedMemPerBlockOptin);
  return 0;
}
