// HBM read bandwidth of a column-major M x N fp64 panel streamed in row chunks of R rows
// (each column contributes R*8 contiguous bytes per chunk), as the tall passes stream it.
// One CTA per SM, each CTA walks its row range chunk by chunk, loads every column's R rows
// with 16-byte loads and sums them (so the loads are not dead).  Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/colmajor_bw tools/colmajor_bw.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int R>
__global__ void __launch_bounds__(512) stream_kernel(const double* __restrict__ A, long long ld, long long M, int N,
                                                     long long rows_per_cta, double* out) {
  const long long r0 = blockIdx.x * rows_per_cta, r1 = min(M, r0 + rows_per_cta);
  constexpr int V = R / 2;                 // double2 per column chunk
  const int tid = threadIdx.x;
  double acc = 0.0;
  for (long long r = r0; r < r1; r += R) {
    // (column, vector) pairs of this chunk spread over the CTA's threads
    for (int i = tid; i < N * V; i += blockDim.x) {
      const int c = i / V, v = i % V;
      const double2 x = __ldg(reinterpret_cast<const double2*>(A + (size_t)c * ld + r) + v);
      acc += x.x + x.y;
    }
  }
  if (acc == 1234.5) out[0] = acc;
}

template <int R>
void run(const double* A, long long ld, long long M, int N, double* out, int sms, int ctas_per_sm) {
  const int grid = sms * ctas_per_sm;
  const long long rows = ((M + grid - 1) / grid + R - 1) / R * R;
  stream_kernel<R><<<grid, 512>>>(A, ld, M, N, rows, out);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int i = 0; i < 5; ++i) stream_kernel<R><<<grid, 512>>>(A, ld, M, N, rows, out);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  printf("{\"test\": \"colmajor_bw\", \"rows_per_chunk\": %d, \"cols\": %d, \"ctas_per_sm\": %d, \"gbs\": %.1f}\n", R, N,
         ctas_per_sm, 5.0 * M * N * 8 / (ms * 1e-3) / 1e9);
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const long long M = 1 << 20;
  const int N = 200;
  double *A, *out;
  cudaMalloc(&A, (size_t)M * N * 8);
  cudaMalloc(&out, 8);
  cudaMemset(A, 0, (size_t)M * N * 8);
  for (int cps : {1, 2, 4}) {
    run<16>(A, M, M, N, out, sms, cps);
    run<32>(A, M, M, N, out, sms, cps);
    run<64>(A, M, M, N, out, sms, cps);
    run<128>(A, M, M, N, out, sms, cps);
  }
  return 0;
}
