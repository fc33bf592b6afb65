// Tall-skinny DMMA GEMMs for wide panels (see psvd_gemm.cu).
#pragma once
#include "psvd_common.cuh"

namespace psvd {

constexpr int GEMM_MAX_SEG = 4;

struct GemmSeg {
  const double* ptr;  // column-major, 16-byte aligned, even ld
  int64_t ld;
  int ncols;
};

// C (M x N, ld ldc) = [segs] (M x K) * W (K x N, col-major, ld ldw even, 16-byte aligned).
// C must not alias any segment.
void launch_tgemm_nn(int64_t M, const GemmSeg* segs, int nseg, const double* W, int64_t ldw, int N, double* C,
                     int64_t ldc, cudaStream_t st);
// X (K x N, ld ldx) = diag(d) [segs]^T Y (d may be null); partial: tgemm_tn_partial_doubles(...) doubles.
size_t tgemm_tn_partial_doubles(int64_t M, int K, int N, int num_sms);
void launch_tgemm_tn(int64_t M, const GemmSeg* segs, int nseg, const double* Y, int64_t ldy, int N,
                     const double* d, double* X, int ldx, double* partial, int num_sms, cudaStream_t st);
// per-chunk (value at max |u|, row + row_offset) of each of the K columns: out[chunk][K][2]
int64_t colmax_rows_chunks(int64_t M);
void launch_colmax_rows(const double* U, int64_t ld, int64_t M, int K, int64_t row_offset, double* out,
                        cudaStream_t st);

}  // namespace psvd
