// Latency probe for the one-CTA eigensolver's dependent chains (diagnostics only).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void probe(double* out, long long* t, double a, double b, int n) {
  double x = a, y = b;
  long long c0 = clock64();
  for (int i = 0; i < n; ++i) x = fma(x, y, a);            // DFMA chain
  long long c1 = clock64();
  for (int i = 0; i < n; ++i) x = sqrt(x + 2.0);            // sqrt chain
  long long c2 = clock64();
  for (int i = 0; i < n; ++i) x = a / (x + 1.0);            // div chain
  long long c3 = clock64();
  for (int i = 0; i < n; ++i) x += __shfl_xor_sync(0xffffffffu, x, 1);  // shfl+add chain
  long long c4 = clock64();
  __shared__ double sm[64];
  sm[threadIdx.x] = x;
  __syncwarp();
  int idx = threadIdx.x;
  for (int i = 0; i < n; ++i) { x = sm[(idx + (int)x) & 31] + 1.0; }  // LDS chain
  long long c5 = clock64();
  for (int i = 0; i < n; ++i) { x = x * y + a; x = x - b; }            // DMUL+DADD chain pair
  long long c6 = clock64();
  for (int i = 0; i < n; ++i) x = 1.0 / x;                  // rcp chain
  long long c7 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) { t[0] = c1 - c0; t[1] = c2 - c1; t[2] = c3 - c2; t[3] = c4 - c3; t[4] = c5 - c4; t[5] = c6 - c5; t[6] = c7 - c6; }
}
__global__ void bar_probe(long long* t, int n) {
  long long c0 = clock64();
  for (int i = 0; i < n; ++i) __syncthreads();
  long long c1 = clock64();
  if (threadIdx.x == 0) t[7] = c1 - c0;
}
int main() {
  double* o; long long* t;
  cudaMalloc(&o, 64 * 8); cudaMallocManaged(&t, 16 * 8);
  const int n = 1000;
  for (int r = 0; r < 2; ++r) { probe<<<1, 32>>>(o, t, 0.5, 0.999, n); bar_probe<<<1, 512>>>(t, n); }
  cudaDeviceSynchronize();
  const char* nm[8] = {"dfma", "sqrt", "div", "shfl+add", "lds+add", "mul+add,sub", "rcp", "syncthreads(512)"};
  for (int i = 0; i < 8; ++i) printf("%-18s %.1f cycles\n", nm[i], (double)t[i] / n);
  return 0;
}
