// Tall-skinny FP64 GEMMs on DMMA for panels too wide for the fused passes
// (randomized update at configs 3/4: n = K + B up to ~1000, sketch width l up to 128).
//
//   tgemm_nn:  C (M x N) = [P_0 | P_1 | ...] (M x K) * W (K x N)        (sketch Y = C Omega,
//              Y <- Y T, U = Y W_f).  CTA = 128 rows x 64 output columns (N <= 64) or 64 rows x
//              128, K in 32-column chunks through a cp.async double buffer, 8 warps x (4 or 2 row
//              blocks x NB/16 column blocks) of 8x8 DMMA tiles.  Each output element is written once.
//              The sym case of tgemm_tn (P == Y) skips the tiles below the diagonal.
//   tgemm_tn:  X (K x N) = P^T Y with the M rows split over CTAs (split-K): CTA = (row chunk,
//              64 x 64 output tile), 32-row stages; per-chunk partial tiles are summed in a fixed
//              order by tgemm_tn_reduce (bitwise reproducible), optionally row-scaled by d.
//   colmax_rows: per-chunk (value at max |u|, global row) of each column, first occurrence.
#include <algorithm>
#include <cstdlib>

#include "psvd_gemm.cuh"

namespace psvd {

namespace {

constexpr int GT = 256;           // threads

// 8-byte global->shared async copy (W / T operands: any leading dimension)
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, int src_bytes) {
  uint32_t sa = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(sa), "l"(gmem), "r"(src_bytes));
}
constexpr int BM = 64, BK = 32;   // rows per CTA, K chunk

constexpr int WSTR = BK + 4;      // smem stride of a W column chunk

struct ColTable {
  const double* ptr[GEMM_MAX_SEG];
  int64_t ld[GEMM_MAX_SEG];
  int c0[GEMM_MAX_SEG + 1];  // prefix column offsets
  int nseg;
};

// per-column base pointers of the segmented panel, built once per CTA in shared memory
__device__ __forceinline__ void build_cols(const ColTable& t, int K, const double** cols) {
  for (int k = threadIdx.x; k < K; k += blockDim.x) {
    const double* p = t.ptr[0] + (int64_t)k * t.ld[0];
    if (t.nseg > 1 && k >= t.c0[1]) p = t.ptr[1] + (int64_t)(k - t.c0[1]) * t.ld[1];
    if (t.nseg > 2 && k >= t.c0[2]) p = t.ptr[2] + (int64_t)(k - t.c0[2]) * t.ld[2];
    if (t.nseg > 3 && k >= t.c0[3]) p = t.ptr[3] + (int64_t)(k - t.c0[3]) * t.ld[3];
    cols[k] = p;
  }
}

size_t nn_smem(int NB, int K, int BMT = BM) {
  return sizeof(double) * (2 * BK * (size_t)(BMT + 4) + 2 * (size_t)NB * WSTR) + 8 * (size_t)K + 16;
}

template <int NB, int BMT = BM>  // output columns per CTA (64 or 128); rows per CTA (64 or 128)
__global__ void __launch_bounds__(GT) tgemm_nn_kernel(int64_t M, ColTable P, int K, const double* __restrict__ W,
                                                      int64_t ldw, int N, double* __restrict__ C, int64_t ldc) {
  constexpr int CBW = NB / 8 / 2;  // column blocks per warp (warp pair shares the row blocks)
  constexpr int RBW = BMT / 32;    // row blocks per warp (4 warps over the rows)
  constexpr int PS = BMT + 4;      // smem stride of a P column chunk (= 4 mod 16)
  extern __shared__ __align__(16) double gsm[];
  double (*sP)[BK * PS] = reinterpret_cast<double (*)[BK * PS]>(gsm);
  double (*sW)[NB * WSTR] = reinterpret_cast<double (*)[NB * WSTR]>(gsm + 2 * BK * PS);
  const double** cols = reinterpret_cast<const double**>(gsm + 2 * BK * PS + 2 * NB * WSTR);
  build_cols(P, K, cols);
  __syncthreads();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, tq = lane & 3;
  const int64_t r0 = (int64_t)blockIdx.x * BMT;
  const int n0 = blockIdx.y * NB;
  const int rbase = (warp & 3) * RBW;         // row blocks rbase .. rbase + RBW - 1
  const int cbase = (warp >> 2) * CBW;        // column blocks cbase .. cbase + CBW - 1
  double acc[RBW][CBW][2];
#pragma unroll
  for (int a = 0; a < RBW; ++a)
#pragma unroll
    for (int b = 0; b < CBW; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;

  const int nchunk = (K + BK - 1) / BK;
  const bool w16 = (ldw & 1) == 0 && (reinterpret_cast<uintptr_t>(W) & 15) == 0;
  auto load = [&](int ch, int buf) {
    const int k0 = ch * BK;
    // P: BK columns x BMT rows in 16-byte pieces
    for (int q = tid; q < BK * (BMT / 2); q += GT) {
      const int kk = q / (BMT / 2), pc = q % (BMT / 2);
      const int k = k0 + kk;
      const int64_t r = r0 + 2 * pc;
      double* dst = &sP[buf][kk * PS + 2 * pc];
      const int64_t valid = M - r;
      const int bytes = (k < K) ? (valid >= 2 ? 16 : (valid == 1 ? 8 : 0)) : 0;
      const double* src = (bytes > 0) ? cols[k] + r : P.ptr[0];
      cp_async16(dst, src, bytes);
    }
    // W: NB columns x BK rows (k); W is small and L2-resident.  16-byte pieces when every column chunk is
    // 16-byte aligned (even ld, aligned base; k0 is a multiple of BK), else 8-byte ones (any ld)
    if (w16) {
      for (int q = tid; q < NB * (BK / 2); q += GT) {
        const int nn = q / (BK / 2), kk = 2 * (q % (BK / 2));
        const int n = n0 + nn, k = k0 + kk;
        const int bytes = (n < N && k < K) ? (k + 1 < K ? 16 : 8) : 0;
        cp_async16(&sW[buf][nn * WSTR + kk], (bytes > 0) ? W + (int64_t)n * ldw + k : W, bytes);
      }
    } else {
      for (int q = tid; q < NB * BK; q += GT) {
        const int nn = q / BK, kk = q % BK;
        const int n = n0 + nn, k = k0 + kk;
        const int bytes = (n < N && k < K) ? 8 : 0;
        cp_async8(&sW[buf][nn * WSTR + kk], (bytes > 0) ? W + (int64_t)n * ldw + k : W, bytes);
      }
    }
  };
  load(0, 0);
  cp_async_commit();
  for (int ch = 0; ch < nchunk; ++ch) {
    const int buf = ch & 1;
    if (ch + 1 < nchunk) load(ch + 1, buf ^ 1);
    cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();
    const double* p = sP[buf];
    const double* w = sW[buf];
#pragma unroll
    for (int ks = 0; ks < BK / 4; ++ks) {
      const int k = ks * 4 + tq;
      double fa[RBW], fb[CBW];
#pragma unroll
      for (int a = 0; a < RBW; ++a) fa[a] = p[k * PS + (rbase + a) * 8 + g];
#pragma unroll
      for (int b = 0; b < CBW; ++b) fb[b] = w[((cbase + b) * 8 + g) * WSTR + k];
#pragma unroll
      for (int a = 0; a < RBW; ++a)
#pragma unroll
        for (int b = 0; b < CBW; ++b) dmma884(acc[a][b][0], acc[a][b][1], fa[a], fb[b]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int a = 0; a < RBW; ++a) {
    const int64_t r = r0 + (rbase + a) * 8 + g;
    if (r >= M) continue;
#pragma unroll
    for (int b = 0; b < CBW; ++b) {
      const int n = n0 + (cbase + b) * 8 + 2 * tq;
      if (n < N) C[(int64_t)n * ldc + r] = acc[a][b][0];
      if (n + 1 < N) C[(int64_t)(n + 1) * ldc + r] = acc[a][b][1];
    }
  }
}

constexpr int TR = 32;          // rows per stage of tgemm_tn
constexpr int TSTR = TR + 4;    // = 4 mod 16
constexpr int TO = 64;          // output tile edge
#ifndef TN_CTAS_PER_SM
#define TN_CTAS_PER_SM 3        // split-K CTAs per SM (3 fit by shared memory)
#endif

// partial[(chunk * ntk + kt) * ntn + nt][64 x TON] (row-major, row = P column).  TON = 64, or 112 for
// 64 < N <= 112 (config 4's l = 110 sketch: one column tile, so P is read once per row chunk and the tile
// pads to 112 instead of 128)
template <int TON>
__global__ void __launch_bounds__(GT) tgemm_tn_kernel(int64_t M, int64_t rows_per_chunk, ColTable P, int K,
                                                      const double* __restrict__ Y, int64_t ldy, int N, int ntk,
                                                      int ntn, int sym, double* __restrict__ partial) {
  // sym: P == Y (a Gram): tiles below the diagonal are not computed (the reduce mirrors them)
  if (sym && (int)(blockIdx.x % (ntk * ntn)) / ntn > (int)(blockIdx.x % (ntk * ntn)) % ntn) return;
  constexpr int BW = TON / 16;  // 8-column blocks per warp (two warp groups over the TON columns)
  extern __shared__ __align__(16) double gsm[];
  double (*sA)[TO * TSTR] = reinterpret_cast<double (*)[TO * TSTR]>(gsm);
  double (*sB)[TON * TSTR] = reinterpret_cast<double (*)[TON * TSTR]>(gsm + 2 * TO * TSTR);
  const double** cols = reinterpret_cast<const double**>(gsm + 2 * TO * TSTR + 2 * TON * TSTR);
  build_cols(P, K, cols);
  __syncthreads();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, tq = lane & 3;
  const int tile = blockIdx.x % (ntk * ntn);
  const int64_t chunk = blockIdx.x / (ntk * ntn);
  const int kt = tile / ntn, nt = tile % ntn;
  const int64_t rb = chunk * rows_per_chunk, re = (M < rb + rows_per_chunk) ? M : rb + rows_per_chunk;
  const int m0 = kt * TO, n0 = nt * TON;
  const int abase = (warp & 3) * 2, bbase = (warp >> 2) * BW;
  double acc[2][BW][2];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < BW; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
  const int64_t nst = re > rb ? (re - rb + TR - 1) / TR : 0;
  auto load = [&](int64_t s, int buf) {
    const int64_t r0 = rb + s * TR;
    for (int q = tid; q < (TO + TON) * (TR / 2); q += GT) {
      const int which = q >= TO * (TR / 2);
      const int qq = which ? q - TO * (TR / 2) : q;
      const int cc = qq / (TR / 2), pc = qq % (TR / 2);
      const int64_t r = r0 + 2 * pc;
      const int64_t valid = re - r;
      int bytes = valid >= 2 ? 16 : (valid == 1 ? 8 : 0);
      const double* src;
      if (which == 0) {
        const int k = m0 + cc;
        if (k >= K) bytes = 0;
        src = bytes > 0 ? cols[k] + r : P.ptr[0];
        cp_async16(&sA[buf][cc * TSTR + 2 * pc], src, bytes);
      } else {
        const int n = n0 + cc;
        if (n >= N) bytes = 0;
        src = bytes > 0 ? Y + (int64_t)n * ldy + r : Y;
        cp_async16(&sB[buf][cc * TSTR + 2 * pc], src, bytes);
      }
    }
  };
  if (nst > 0) load(0, 0);
  cp_async_commit();
  for (int64_t s = 0; s < nst; ++s) {
    const int buf = (int)(s & 1);
    if (s + 1 < nst) load(s + 1, buf ^ 1);
    cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();
    const double* A = sA[buf];
    const double* B = sB[buf];
#pragma unroll
    for (int ks = 0; ks < TR / 4; ++ks) {
      const int k = ks * 4 + tq;
      double fa[2], fb[BW];
#pragma unroll
      for (int a = 0; a < 2; ++a) fa[a] = A[((abase + a) * 8 + g) * TSTR + k];
#pragma unroll
      for (int b = 0; b < BW; ++b) fb[b] = B[((bbase + b) * 8 + g) * TSTR + k];
#pragma unroll
      for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int b = 0; b < BW; ++b) dmma884(acc[a][b][0], acc[a][b][1], fa[a], fb[b]);
    }
    __syncthreads();
  }
  double* dst = partial + (size_t)blockIdx.x * TO * TON;
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < BW; ++b)
      *reinterpret_cast<double2*>(dst + ((abase + a) * 8 + g) * TON + (bbase + b) * 8 + 2 * tq) =
          make_double2(acc[a][b][0], acc[a][b][1]);
}

// X[m + n*ldx] = d[m] * sum_chunks partial(chunk, m, n), chunks in order
__global__ void tgemm_tn_reduce_kernel(const double* __restrict__ partial, int nchunks, int K, int N, int ntk,
                                       int ntn, int ton, int sym, const double* __restrict__ d, double* __restrict__ X,
                                       int ldx) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (int64_t)K * N) return;
  int m = (int)(idx % K), n = (int)(idx / K);
  const int mo = m;
  if (sym && m / TO > n / TO) {  // below-diagonal tile of a Gram: its mirror (same sums, same order)
    const int t = m;
    m = n;
    n = t;
  }
  const int kt = m / TO, nt = n / ton;  // sym tiles are square (ton == TO)
  const size_t off = (size_t)(m % TO) * ton + (n % ton);
  double s = 0.0;
  for (int c = 0; c < nchunks; ++c) s += partial[((size_t)c * ntk * ntn + kt * ntn + nt) * TO * ton + off];
  const int no = (int)(idx / K);
  X[(int64_t)no * ldx + mo] = d != nullptr ? d[mo] * s : s;
}

// per-chunk (value at max |u|, global row) of each column; ties -> first row
__global__ void colmax_rows_kernel(const double* __restrict__ U, int64_t ld, int64_t M, int K, int64_t rows_per_chunk,
                                   int64_t row_offset, double* __restrict__ out) {
  const int k = blockIdx.y;
  const int64_t chunk = blockIdx.x;
  const int64_t rb = chunk * rows_per_chunk, re = (M < rb + rows_per_chunk) ? M : rb + rows_per_chunk;
  double best = -1.0, val = 0.0;
  int64_t row = -1;
  for (int64_t r = rb + threadIdx.x; r < re; r += blockDim.x) {
    const double v = U[(int64_t)k * ld + r];
    if (fabs(v) > best) { best = fabs(v); val = v; row = r; }
  }
  __shared__ double sb[256], sv[256];
  __shared__ long long sr[256];
  sb[threadIdx.x] = best; sv[threadIdx.x] = val; sr[threadIdx.x] = row;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o) {
      const int j = threadIdx.x + o;
      const bool take = sb[j] > sb[threadIdx.x] ||
                        (sb[j] == sb[threadIdx.x] && sr[j] >= 0 && (sr[threadIdx.x] < 0 || sr[j] < sr[threadIdx.x]));
      if (take) { sb[threadIdx.x] = sb[j]; sv[threadIdx.x] = sv[j]; sr[threadIdx.x] = sr[j]; }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    double* dst = out + ((size_t)chunk * K + k) * 2;
    dst[0] = sv[0];
    dst[1] = (double)(sr[0] + row_offset);
  }
}

ColTable make_table(const GemmSeg* segs, int nseg) {
  ColTable t{};
  t.nseg = nseg;
  t.c0[0] = 0;
  for (int i = 0; i < nseg; ++i) {
    t.ptr[i] = segs[i].ptr;
    t.ld[i] = segs[i].ld;
    t.c0[i + 1] = t.c0[i] + segs[i].ncols;
  }
  for (int i = nseg; i < GEMM_MAX_SEG; ++i) {
    t.ptr[i] = segs[0].ptr;
    t.ld[i] = segs[0].ld;
    t.c0[i + 1] = 1 << 30;
  }
  return t;
}

}  // namespace

void launch_tgemm_nn(int64_t M, const GemmSeg* segs, int nseg, const double* W, int64_t ldw, int N, double* C,
                     int64_t ldc, cudaStream_t st) {
  const ColTable t = make_table(segs, nseg);
  const int K = t.c0[nseg];
  const unsigned gx = (unsigned)((M + BM - 1) / BM);
  static const int bm128 = getenv("PSVD_NN_BM64") ? 0 : 1;  // A/B switch: 64-row CTAs
  if (N <= 64 && bm128) {
    // 128-row CTAs: 4 row blocks x 4 column blocks per warp, 8 fragment loads per 16 DMMAs
    const size_t sm = nn_smem(64, K, 128);
    cudaFuncSetAttribute(tgemm_nn_kernel<64, 128>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    tgemm_nn_kernel<64, 128><<<dim3((unsigned)((M + 127) / 128), 1), GT, sm, st>>>(M, t, K, W, ldw, N, C, ldc);
  } else if (N <= 64) {
    const size_t sm = nn_smem(64, K);
    cudaFuncSetAttribute(tgemm_nn_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    tgemm_nn_kernel<64><<<dim3(gx, 1), GT, sm, st>>>(M, t, K, W, ldw, N, C, ldc);
  } else if (N <= 112) {
    // 14 column blocks (the l = K + p = 110 sketch of config 4 pads to 112 instead of 128)
    const size_t sm = nn_smem(112, K);
    cudaFuncSetAttribute(tgemm_nn_kernel<112>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    tgemm_nn_kernel<112><<<dim3(gx, 1), GT, sm, st>>>(M, t, K, W, ldw, N, C, ldc);
  } else {
    const size_t sm = nn_smem(128, K);
    cudaFuncSetAttribute(tgemm_nn_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    tgemm_nn_kernel<128><<<dim3(gx, (unsigned)((N + 127) / 128)), GT, sm, st>>>(M, t, K, W, ldw, N, C, ldc);
  }
}

static int tn_width(int N, bool sym) { return (!sym && N > 64 && N <= 112) ? 112 : TO; }

static size_t tn_partial(int64_t M, int K, int N, int ton, int num_sms) {
  const int ntk = (K + TO - 1) / TO, ntn = (N + ton - 1) / ton;
  const int64_t want = std::max<int64_t>(1, (int64_t)TN_CTAS_PER_SM * num_sms / (ntk * ntn));
  const int64_t nchunks = std::min<int64_t>(want, (M + TR - 1) / TR);
  return (size_t)std::max<int64_t>(nchunks, 1) * ntk * ntn * TO * ton;
}

size_t tgemm_tn_partial_doubles(int64_t M, int K, int N, int num_sms) {
  // sized for either tile width (the launch picks it from N and whether the product is a Gram)
  return std::max(tn_partial(M, K, N, TO, num_sms), tn_partial(M, K, N, tn_width(N, false), num_sms));
}

void launch_tgemm_tn(int64_t M, const GemmSeg* segs, int nseg, const double* Y, int64_t ldy, int N,
                     const double* d, double* X, int ldx, double* partial, int num_sms, cudaStream_t st) {
  const ColTable t = make_table(segs, nseg);
  const int K = t.c0[nseg];
  const int sym = (nseg == 1 && segs[0].ptr == Y && segs[0].ld == ldy && K == N) ? 1 : 0;
  const int ton = tn_width(N, sym);
  const int ntk = (K + TO - 1) / TO, ntn = (N + ton - 1) / ton;
  const int64_t want = std::max<int64_t>(1, (int64_t)TN_CTAS_PER_SM * num_sms / (ntk * ntn));
  int64_t nchunks = std::max<int64_t>(1, std::min<int64_t>(want, (M + TR - 1) / TR));
  const int64_t rows = ((M + nchunks - 1) / nchunks + TR - 1) / TR * TR;
  nchunks = (M + rows - 1) / rows;
  const size_t sm = sizeof(double) * 2 * (TO + ton) * TSTR + 8 * (size_t)K + 16;
  const unsigned grid = (unsigned)(nchunks * ntk * ntn);
  if (ton == 112) {
    cudaFuncSetAttribute(tgemm_tn_kernel<112>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    tgemm_tn_kernel<112><<<grid, GT, sm, st>>>(M, rows, t, K, Y, ldy, N, ntk, ntn, sym, partial);
  } else {
    cudaFuncSetAttribute(tgemm_tn_kernel<TO>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    tgemm_tn_kernel<TO><<<grid, GT, sm, st>>>(M, rows, t, K, Y, ldy, N, ntk, ntn, sym, partial);
  }
  const int64_t tot = (int64_t)K * N;
  tgemm_tn_reduce_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(partial, (int)nchunks, K, N, ntk, ntn, ton,
                                                                        sym, d, X, ldx);
}

int64_t colmax_rows_chunks(int64_t M) { return std::max<int64_t>(1, std::min<int64_t>(256, (M + 4095) / 4096)); }

void launch_colmax_rows(const double* U, int64_t ld, int64_t M, int K, int64_t row_offset, double* out,
                        cudaStream_t st) {
  const int64_t nchunks = colmax_rows_chunks(M);
  const int64_t rows = (M + nchunks - 1) / nchunks;
  colmax_rows_kernel<<<dim3((unsigned)nchunks, (unsigned)K), 256, 0, st>>>(U, ld, M, K, rows, row_offset, out);
}

}  // namespace psvd
