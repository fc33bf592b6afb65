// Pure TMA streaming bandwidth of a column-major M x C fp64 panel (no math): one CTA per SM,
// one producer lane, one consumer warp that releases ring slots as they land.
//   2d: a 16-row x C box per stage (128 contiguous bytes of every column per request)
//   3d: a (16 rows, R/16 row blocks, C) box per stage: R*8 contiguous bytes of every column
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tma_stream_bw tools/tma_stream_bw.cu -lcuda
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

template <int DIM>
__global__ void __launch_bounds__(64) tma_stream(const __grid_constant__ CUtensorMap map,
                                                 const __grid_constant__ CUtensorMap pmap, long long M, int C, int R,
                                                 int ns, long long rows_per_cta, int pf_rows) {
  extern __shared__ __align__(1024) unsigned char sm[];
  unsigned char* base = sm + ((1024 - (saddr(sm) & 1023)) & 1023);
  const unsigned stage = (unsigned)R * C * 8;
  unsigned long long* full = reinterpret_cast<unsigned long long*>(base + (size_t)ns * stage);
  unsigned long long* empty = full + ns;
  if (threadIdx.x == 0) {
    for (int i = 0; i < ns; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], 1); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const long long r0 = blockIdx.x * rows_per_cta, r1 = min(M, r0 + rows_per_cta);
  const long long nst = (r1 - r0 + R - 1) / R;
  if (threadIdx.x == 0) {
    for (long long s = 0; s < nst; ++s) {
      const int b = (int)(s % ns);
      if (s >= ns) mbar_wait(&empty[b], (unsigned)(((s / ns) - 1) & 1));
      mbar_expect(&full[b], stage);
      const int row = (int)(r0 + s * R);
      // optional L2 prefetch of pf_rows-row blocks (3-D box) one block ahead: longer contiguous DRAM runs per column
      if (pf_rows > 0 && ((s * R) % pf_rows) == 0) {
        const long long prow = row + pf_rows;
        if (prow < r1)
          asm volatile("cp.async.bulk.prefetch.tensor.3d.L2.global.tile [%0, {%1, %2, %3}];" ::"l"(&pmap), "r"(0),
                       "r"((int)(prow / 16)), "r"(0)
                       : "memory");
      }
      if (DIM == 2) {
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::
                "r"(saddr(base + (size_t)b * stage)), "l"(&map), "r"(row), "r"(0), "r"(saddr(&full[b]))
            : "memory");
      } else {
        asm volatile(
            "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::
                "r"(saddr(base + (size_t)b * stage)), "l"(&map), "r"(0), "r"(row / 16), "r"(0), "r"(saddr(&full[b]))
            : "memory");
      }
    }
  } else if (threadIdx.x == 32) {
    for (long long s = 0; s < nst; ++s) {
      const int b = (int)(s % ns);
      mbar_wait(&full[b], (unsigned)((s / ns) & 1));
      mbar_arrive(&empty[b]);
    }
  }
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const long long M = 1 << 20;
  const int C = 200;
  double* A; cudaMalloc(&A, (size_t)M * C * 8); cudaMemset(A, 0, (size_t)M * C * 8);
  CUtensorMap pmaps[3];
  const int pfs[3] = {0, 128, 256};
  for (int i = 1; i < 3; ++i) {
    cuuint64_t dims[3] = {16, (cuuint64_t)(M / 16), (cuuint64_t)C};
    cuuint64_t str[2] = {128, (cuuint64_t)M * 8};
    cuuint32_t box[3] = {16, (cuuint32_t)(pfs[i] / 16), (cuuint32_t)C};
    cuuint32_t es[3] = {1, 1, 1};
    CUresult e = cuTensorMapEncodeTiled(&pmaps[i], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, A, dims, str, box, es,
                                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (e != CUDA_SUCCESS) printf("pmap encode failed %d\n", (int)e);
  }
  pmaps[0] = pmaps[1];
  for (int pfi = 0; pfi < 3; ++pfi)
  for (int dim : {2, 3}) {
    for (int R : {16, 32, 64}) {
      if (pfi > 0 && !(dim == 2 || R == 32)) continue;
      if (dim == 2 && R != 16) continue;
      CUtensorMap map;
      CUresult e;
      if (dim == 2) {
        cuuint64_t dims[2] = {(cuuint64_t)M, (cuuint64_t)C};
        cuuint64_t str[1] = {(cuuint64_t)M * 8};
        cuuint32_t box[2] = {16, (cuuint32_t)C};
        cuuint32_t es[2] = {1, 1};
        e = cuTensorMapEncodeTiled(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, A, dims, str, box, es,
                                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      } else {
        cuuint64_t dims[3] = {16, (cuuint64_t)(M / 16), (cuuint64_t)C};
        cuuint64_t str[2] = {128, (cuuint64_t)M * 8};
        cuuint32_t box[3] = {16, (cuuint32_t)(R / 16), (cuuint32_t)C};
        cuuint32_t es[3] = {1, 1, 1};
        e = cuTensorMapEncodeTiled(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, A, dims, str, box, es,
                                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      }
      if (e != CUDA_SUCCESS) { printf("encode failed %d (dim %d R %d)\n", (int)e, dim, R); continue; }
      for (int budget_kb : {96, 160, 200}) {
        const int stage = R * C * 8;
        const int ns = budget_kb * 1024 / stage;
        if (ns < 2) continue;
        const size_t smem = (size_t)ns * stage + 1024 + 256;
        auto kern = dim == 2 ? tma_stream<2> : tma_stream<3>;
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        const long long rows = ((M + sms - 1) / sms + R - 1) / R * R;
        const int pf = pfs[pfi];
        kern<<<sms, 64, smem>>>(map, pmaps[pfi], M, C, R, ns, rows, pf);
        cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
        cudaEventRecord(e0);
        for (int i = 0; i < 5; ++i) kern<<<sms, 64, smem>>>(map, pmaps[pfi], M, C, R, ns, rows, pf);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        cudaError_t err = cudaGetLastError();
        printf("{\"test\": \"tma_stream\", \"dim\": %d, \"rows_per_stage\": %d, \"cols\": %d, \"stages\": %d, \"pf_rows\": %d, \"gbs\": %.1f, \"err\": \"%s\"}\n",
               dim, R, C, ns, pf, 5.0 * M * C * 8 / (ms * 1e-3) / 1e9, cudaGetErrorString(err));
      }
    }
  }
  return 0;
}
