// Streaming bandwidth of a column-major M x C fp64 panel in 16-row stages when the stage's box lines
// are split between the TMA engine (columns [0, C1): one 2-D box of 16 rows per <= 256 columns) and
// cp.async 16-byte copies by NCP producer warps (columns [C1, C): 8 lanes per 128-byte column piece).
// The 16-row TMA stream is capped by the engine's per-line rate (~4.6 TB/s, tools/tma_stream_bw.cu);
// the question is whether the LSU path adds to it.  No math: one consumer warp releases the slots.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/hybrid tools/hybrid_stream_bw.cu -lcuda
#include <cstdio>
#include <cuda.h>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned saddr(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* b, unsigned c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(saddr(b)), "r"(c));
}
__device__ __forceinline__ void mbar_wait(unsigned long long* b, unsigned ph) {
  asm volatile("{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W;\n}\n" ::"r"(saddr(b)),
               "r"(ph));
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(saddr(b)));
}
__device__ __forceinline__ void mbar_expect(unsigned long long* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(saddr(b)), "r"(bytes));
}

constexpr int R = 16;

// warp 0 lane 0: TMA; warp 1: consumer; warps 2 .. 2 + NCP - 1: cp.async producers
__global__ void __launch_bounds__(256) hybrid_stream(const __grid_constant__ CUtensorMap map,
                                                     const __grid_constant__ CUtensorMap map64, const double* A, long long M,
                                                     int C, int C1, int ncp, int ns, long long rows_per_cta) {
  extern __shared__ __align__(1024) unsigned char sm[];
  unsigned char* base = sm + ((1024 - (saddr(sm) & 1023)) & 1023);
  const unsigned stage = (unsigned)R * C * 8;
  unsigned long long* full = reinterpret_cast<unsigned long long*>(base + (size_t)ns * stage);
  unsigned long long* empty = full + ns;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < ns; ++i) {
      mbar_init(&full[i], 1 + 32 * ncp);
      mbar_init(&empty[i], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const long long r0 = blockIdx.x * rows_per_cta, r1 = min(M, r0 + rows_per_cta);
  const long long nst = (r1 - r0 + R - 1) / R;
  if (warp == 0) {
    if (lane == 0) {
      for (long long s = 0; s < nst; ++s) {
        const int b = (int)(s % ns);
        if (s >= ns) mbar_wait(&empty[b], (unsigned)(((s / ns) - 1) & 1));
        mbar_expect(&full[b], (unsigned)(R * C1 * 8));
        const int row = (int)(r0 + s * R);
        for (int c = 0; c < C1;) {  // 256-column boxes, then 64-column ones (C1 a multiple of 64)
          const bool big = c + 256 <= C1;
          asm volatile(
              "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::
                  "r"(saddr(base + (size_t)b * stage + (size_t)c * R * 8)),
              "l"(big ? &map : &map64), "r"(row), "r"(c), "r"(saddr(&full[b]))
              : "memory");
          c += big ? 256 : 64;
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0)
      for (long long s = 0; s < nst; ++s) {
        const int b = (int)(s % ns);
        mbar_wait(&full[b], (unsigned)((s / ns) & 1));
        mbar_arrive(&empty[b]);
      }
  } else if (warp < 2 + ncp) {
    const int t = threadIdx.x - 64, nt = 32 * ncp;
    const int nchunk = (C - C1) * 8;  // 16-byte chunks per stage
    for (long long s = 0; s < nst; ++s) {
      const int b = (int)(s % ns);
      if (s >= ns) mbar_wait(&empty[b], (unsigned)(((s / ns) - 1) & 1));
      const long long row = r0 + s * R;
      unsigned char* dst0 = base + (size_t)b * stage + (size_t)C1 * R * 8;
      for (int i = t; i < nchunk; i += nt) {
        const int c = i >> 3, part = i & 7;
        const double* src = A + (size_t)(C1 + c) * M + row + part * 2;
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(saddr(dst0 + (size_t)c * R * 8 + part * 16)),
                     "l"(src)
                     : "memory");
      }
      asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(saddr(&full[b])) : "memory");
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
  }
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const long long M = 1 << 20;
  const int C = 448;  // ~ the deterministic fused pass's panel ([U_{b-1} | A_b | A_{b+1}] at B = 200: 424)
  double* A;
  cudaMalloc(&A, (size_t)M * C * 8);
  cudaMemset(A, 0, (size_t)M * C * 8);
  CUtensorMap map, map64;
  cuuint64_t dims[2] = {(cuuint64_t)M, (cuuint64_t)C};
  cuuint64_t str[1] = {(cuuint64_t)M * 8};
  cuuint32_t box[2] = {16, 256};
  cuuint32_t es[2] = {1, 1};
  if (cuTensorMapEncodeTiled(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, A, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                             CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
    printf("encode failed\n");
    return 1;
  }
  box[1] = 64;
  if (cuTensorMapEncodeTiled(&map64, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, A, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                             CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
    printf("encode failed\n");
    return 1;
  }
  for (int C1 : {448, 320, 256, 192, 128, 0})
    for (int ncp : {1, 2, 4, 6}) {
      if (C1 == C && ncp > 1) continue;
      for (int ns : {3, 4}) {
        const int stage = R * C * 8;
        const size_t smem = (size_t)ns * stage + 1024 + 256;
        if (smem > 227 * 1024) continue;
        cudaFuncSetAttribute(hybrid_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        const long long rows = ((M + sms - 1) / sms + R - 1) / R * R;
        hybrid_stream<<<sms, 256, smem>>>(map, map64, A, M, C, C1, ncp, ns, rows);
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaEventRecord(e0);
        for (int i = 0; i < 5; ++i) hybrid_stream<<<sms, 256, smem>>>(map, map64, A, M, C, C1, ncp, ns, rows);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("{\"test\": \"hybrid_stream\", \"cols\": %d, \"tma_cols\": %d, \"cp_warps\": %d, \"stages\": %d, \"gbs\": %.1f, "
               "\"err\": \"%s\"}\n",
               C, C1, ncp, ns, 5.0 * M * C * 8 / (ms * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
      }
    }
  return 0;
}
