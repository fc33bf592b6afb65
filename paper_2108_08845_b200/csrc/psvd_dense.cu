// C ABI of the dense factorizations behind the reference's linalg boundary (qr_factor, svd_full,
// randomized_range's products, parallel_qr's Cholesky factors; include/psvd.h).
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>
#include <algorithm>
#include <cstdlib>

#include "psvd_ctx.cuh"

using namespace psvd;
using namespace psvd_internal;

namespace psvd_internal {

// Y (rows x cols, column-major, ld ldy) = the row-major X (rows x cols, row stride ldx): 32 x 32 tiles
// through shared memory (padded against bank conflicts), coalesced on both sides.
__global__ void __launch_bounds__(256) transpose_kernel(const double* __restrict__ X, int64_t ldx, int64_t rows,
                                                       int64_t cols, double* __restrict__ Y, int64_t ldy) {
  __shared__ double t[32][33];
  const int64_t r0 = (int64_t)blockIdx.x * 32, c0 = (int64_t)blockIdx.y * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
  for (int k = ty; k < 32; k += 8) {
    const int64_t r = r0 + k, c = c0 + tx;
    t[k][tx] = (r < rows && c < cols) ? X[r * ldx + c] : 0.0;
  }
  __syncthreads();
  for (int k = ty; k < 32; k += 8) {
    const int64_t c = c0 + k, r = r0 + tx;
    if (r < rows && c < cols) Y[c * ldy + r] = t[tx][k];
  }
}

__global__ void scale_cols_any_kernel(double* __restrict__ X, int64_t ld, int64_t rows, int cols,
                                      const double* __restrict__ s, int invert) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int j = blockIdx.y;
  if (i >= rows || j >= cols) return;
  const double f = s[j];
  double& x = X[(size_t)j * ld + i];
  x = invert ? (f != 0.0 ? x / f : 0.0) : x * f;
}

int chol_any(psvd_ctx* c, const double* G, int n, double* T, int* illcond, int* status, double* Rout,
             cudaStream_t st) {
  if (n <= CHOL_NMAX) {
    launch_chol_inv(G, n, T, st, illcond, status, Rout);
    c->launches++;
    return cuda_check(c, "chol");
  }
  int rc = ensure(c, c->bigws, sizeof(double) * chol_big_workspace_doubles(n));
  if (rc) return rc;
  launch_chol_big(G, n, T, illcond, status, Rout, (double*)c->bigws.ptr, st);
  c->launches += chol_big_launches(n);
  return cuda_check(c, "chol big");
}

int jacobi_any(psvd_ctx* c, const double* X, int64_t ldx, int64_t m, int n, int transpose, double* S, double* V,
               int64_t ldv, double* U, int64_t ldu, cudaStream_t st) {
  int rc = ensure(c, c->bigjac, sizeof(double) * jacobi_big_workspace_doubles(m, n));
  if (rc) return rc;
  const int e = launch_jacobi_big(X, ldx, m, n, transpose, S, V, ldv, U, ldu, (double*)c->bigjac.ptr, c->d_status,
                                  nullptr, c->num_sms, st);
  c->launches += 2;
  if (e != 0) return fail(c, PSVD_ECUDA, "jacobi launch: %s", cudaGetErrorString((cudaError_t)e));
  return cuda_check(c, "jacobi big");
}

}  // namespace psvd_internal

extern "C" {

// ---- dense factorizations behind the reference's linalg boundary (qr_factor / svd_full /
// randomized_range, linalg.py:94-147; parallel_qr, dsvd.py:176-202).  Library utilities, not
// the streaming update: psvd_qr reads one condition flag back (one host sync).

int psvd_chol(psvd_ctx* c, const double* G, int n, double* R, double* T, void* stream) {
  if (!c) return PSVD_EINVAL;
  if (n < 1 || !G || !T) return fail(c, PSVD_EINVAL, "bad Cholesky n=%d", n);
  return chol_any(c, G, n, T, c->d_status + 3, c->d_status, R, (cudaStream_t)stream);
}

int psvd_chol_shift(psvd_ctx* c, double* G, int n, int64_t M, void* stream) {
  if (!c) return PSVD_EINVAL;
  if (n < 1 || !G || M < 1) return fail(c, PSVD_EINVAL, "bad shift arguments");
  launch_chol_shift(G, n, M, (cudaStream_t)stream);
  c->launches++;
  return cuda_check(c, "chol shift");
}

int psvd_chol_illcond(psvd_ctx* c, int* flag, void* stream) {
  if (!c || !flag) return PSVD_EINVAL;
  cudaStream_t st = (cudaStream_t)stream;
  cudaMemcpyAsync(c->h_status, c->d_status + 3, sizeof(int), cudaMemcpyDeviceToHost, st);
  if (cudaStreamSynchronize(st) != cudaSuccess) return cuda_check(c, "chol flag");
  *flag = *c->h_status;
  return PSVD_OK;
}

int psvd_nn_product(psvd_ctx* c, int64_t M, const double* A, int64_t lda, int n, const double* W, int64_t ldw, int w,
                    double* Y, int64_t ldy, void* stream) {
  if (!c) return PSVD_EINVAL;
  int rc;
  if (M < 1 || n < 1 || w < 1 || !W || ldw < n) return fail(c, PSVD_EINVAL, "bad nn_product shape");
  if ((rc = check_mat(c, "A", A, lda, M, n)) || (rc = check_mat(c, "Y", Y, ldy, M, w))) return rc;
  const GemmSeg ga{A, lda, n};
  launch_tgemm_nn(M, &ga, 1, W, ldw, w, Y, ldy, (cudaStream_t)stream);
  c->launches++;
  return cuda_check(c, "nn product");
}

int psvd_small_matmul(psvd_ctx* c, const double* A, int lda, int transA, const double* B, int ldb, double* C, int ldc,
                      int m, int k, int n, void* stream) {
  if (!c) return PSVD_EINVAL;
  if (m < 1 || k < 1 || n < 1 || !A || !B || !C || ldc < m) return fail(c, PSVD_EINVAL, "bad small matmul");
  launch_small_gemm(A, lda, transA, B, ldb, C, ldc, m, k, n, nullptr, (cudaStream_t)stream);
  c->launches++;
  return cuda_check(c, "small matmul");
}

// Tall QR (M >= n, any n: one-CTA Cholesky up to CHOL_NMAX, the global-memory one beyond): CholeskyQR2
// (R = R2 R1 from two Gram passes), or psvd_qr_robust (psvd_accurate.cu: Gram deflation + Householder
// QR of the small factor) when the first Cholesky flags cond(A) beyond CholeskyQR2's range or a rank
// deficiency.  diag(R) >= 0 (qr_factor's sign convention, linalg.py:94-104).  R: n x n, ld n.
int psvd_qr(psvd_ctx* c, int64_t M, int n, const double* A, int64_t lda, double* Q, int64_t ldq, double* R,
            void* stream) {
  if (!c) return PSVD_EINVAL;
  cudaStream_t st = (cudaStream_t)stream;
  int rc;
  if (n < 1 || M < n) return fail(c, PSVD_EINVAL, "qr needs M >= n >= 1 (M=%lld n=%d)", (long long)M, n);
  if ((rc = check_mat(c, "A", A, lda, M, n)) || (rc = check_mat(c, "Q", Q, ldq, M, n))) return rc;
  if (!R) return fail(c, PSVD_EINVAL, "R is null");
  const size_t nn = (size_t)n * n;
  const int64_t ldt = M + (M & 1);
  if ((rc = ensure(c, c->dense, sizeof(double) * 5 * nn)) || (rc = ensure(c, c->dense2, sizeof(double) * ldt * n)))
    return rc;
  double* G = (double*)c->dense.ptr;
  double* R1 = G + nn;
  double* T1 = R1 + nn;
  double* R2 = T1 + nn;
  double* T2 = R2 + nn;
  double* tmp = (double*)c->dense2.ptr;
  auto gram = [&](const double* X, int64_t ldx) { return psvd_gram(c, M, nullptr, 0, nullptr, 1.0, 0, X, ldx, n, G, st); };
  auto mul = [&](const double* X, int64_t ldx, const double* T, double* Y, int64_t ldy) {
    const GemmSeg gx{X, ldx, n};
    launch_tgemm_nn(M, &gx, 1, T, n, n, Y, ldy, st);
    c->launches++;
  };
  auto refine = [&](double* Rk, double* Tk) -> int {  // Q <- Q chol(Q^T Q)^-1, returns the new factor in Rk
    int r;
    if ((r = gram(Q, ldq))) return r;
    if ((r = chol_any(c, G, n, Tk, nullptr, c->d_status, Rk, st))) return r;
    mul(Q, ldq, Tk, tmp, ldt);
    cudaMemcpy2DAsync(Q, ldq * sizeof(double), tmp, ldt * sizeof(double), M * sizeof(double), n,
                      cudaMemcpyDeviceToDevice, st);
    c->launches++;
    return cuda_check(c, "qr refine");
  };
  // CholeskyQR2
  if ((rc = gram(A, lda))) return rc;
  if ((rc = chol_any(c, G, n, T1, c->d_status + 3, c->d_status, R1, st))) return rc;
  int ill = 0;
  if ((rc = psvd_chol_illcond(c, &ill, stream))) return rc;
  if (ill) return psvd_qr_robust(c, M, n, A, lda, Q, ldq, R, stream);  // beyond CholeskyQR2's range / rank deficient
  mul(A, lda, T1, Q, ldq);
  if ((rc = refine(R2, T2))) return rc;
  launch_small_gemm(R2, n, 0, R1, n, R, n, n, n, n, nullptr, st);  // R2 R1
  c->launches++;
  return cuda_check(c, "qr");
}

// One-sided Jacobi SVD of X (m x n, m >= n, n <= JACOBI_NMAX): S (n, descending), V (n x n, ld ldv;
// X = U diag(S) V^T).  Relative accuracy (no squaring); X is packed first.
int psvd_jacobi(psvd_ctx* c, const double* X, int64_t ldx, int64_t m, int n, double* S, double* V, int64_t ldv,
                void* stream) {
  if (!c) return PSVD_EINVAL;
  cudaStream_t st = (cudaStream_t)stream;
  int rc;
  if (n < 1 || m < n || m > (int64_t)INT32_MAX)
    return fail(c, PSVD_EINVAL, "jacobi needs m >= n >= 1 (m=%lld n=%d)", (long long)m, n);
  if (!X || !S || !V || ldx < m || ldv < n) return fail(c, PSVD_EINVAL, "bad jacobi arguments");
  if (n > JACOBI_NMAX) return jacobi_any(c, X, ldx, m, n, 0, S, V, ldv, nullptr, 0, st);
  const size_t mn = (size_t)m * n;
  if ((rc = ensure(c, c->dense2, sizeof(double) * (mn + (size_t)n * n))) ||
      (rc = ensure(c, c->jacws, sizeof(double) * jacobi_workspace_doubles((int)m, n))))
    return rc;
  double* Xp = (double*)c->dense2.ptr;
  double* J = Xp + mn;
  cudaMemcpy2DAsync(Xp, m * sizeof(double), X, ldx * sizeof(double), m * sizeof(double), n, cudaMemcpyDeviceToDevice,
                    st);
  launch_jacobi_svd(Xp, (int)m, n, S, J, (double*)c->jacws.ptr, c->d_status, st);
  cudaMemcpy2DAsync(V, ldv * sizeof(double), J, n * sizeof(double), n * sizeof(double), n, cudaMemcpyDeviceToDevice, st);
  c->launches++;
  return cuda_check(c, "jacobi");
}

// One-sided Jacobi SVD of any width on the global-memory kernel: X (m x n, ld ldx) or, with
// transpose = 1, X^T of an n x m X.  S (n) descending, V (n x n, ld ldv), optional U = X V S^-1.
int psvd_jacobi_uv(psvd_ctx* c, const double* X, int64_t ldx, int64_t m, int n, int transpose, double* S, double* V,
                   int64_t ldv, double* U, int64_t ldu, void* stream) {
  if (!c) return PSVD_EINVAL;
  if (n < 1 || m < 1 || !X || !S || !V || ldv < n || (U && ldu < m) || ldx < (transpose ? n : m))
    return fail(c, PSVD_EINVAL, "bad jacobi_uv arguments (m=%lld n=%d)", (long long)m, n);
  return jacobi_any(c, X, ldx, m, n, transpose, S, V, ldv, U, ldu, (cudaStream_t)stream);
}

// The reference's sign rule (linalg.py:81-91): per column of U (rows x cols) the entry of largest
// magnitude (first occurrence) is made positive; the same flips go to the columns of V (vrows x
// cols, may be null: the rows of vt).
int psvd_sign_pair(psvd_ctx* c, double* U, int64_t ldu, int64_t rows, int cols, double* V, int64_t ldv, int64_t vrows,
                   void* stream) {
  if (!c) return PSVD_EINVAL;
  cudaStream_t st = (cudaStream_t)stream;
  int rc;
  if (rows < 1 || cols < 1 || !U || ldu < rows || (V && ldv < vrows)) return fail(c, PSVD_EINVAL, "bad sign arguments");
  const int64_t nch = colmax_rows_chunks(rows);
  if ((rc = ensure(c, c->colmax, sizeof(double) * (size_t)nch * cols * 2)) ||
      (rc = ensure(c, c->xpairs, sizeof(double) * (size_t)cols)))
    return rc;
  double* sgn = (double*)c->xpairs.ptr;
  launch_colmax_rows(U, ldu, rows, cols, 0, (double*)c->colmax.ptr, st);
  launch_colmax_sign((const double*)c->colmax.ptr, (int)nch, cols, sgn, st);
  launch_scale_cols(U, ldu, rows, cols, sgn, st);
  c->launches += 3;
  if (V) {
    launch_scale_cols(V, ldv, vrows, cols, sgn, st);
    c->launches++;
  }
  return cuda_check(c, "sign pair");
}

// Column-major copy of a row-major device matrix (C-ordered numpy / torch input, as the reference's
// burgers_matrix returns): X rows x cols with row stride ldx -> Y column-major, ld ldy (even).
int psvd_transpose(psvd_ctx* c, const double* X, int64_t ldx, int64_t rows, int64_t cols, double* Y, int64_t ldy,
                   void* stream) {
  if (!c) return PSVD_EINVAL;
  if (!X || !Y || rows < 1 || cols < 1 || ldx < cols || ldy < rows) return fail(c, PSVD_EINVAL, "bad transpose");
  dim3 g((unsigned)((rows + 31) / 32), (unsigned)((cols + 31) / 32));
  if (g.y > 65535u) return fail(c, PSVD_EINVAL, "transpose: too many columns for one launch");
  transpose_kernel<<<g, 256, 0, (cudaStream_t)stream>>>(X, ldx, rows, cols, Y, ldy);
  c->launches++;
  return cuda_check(c, "transpose");
}

// X[:, j] *= s_j (invert = 0) or /= s_j with 0 for s_j == 0 (invert = 1)
int psvd_scale_cols(psvd_ctx* c, double* X, int64_t ld, int64_t rows, int cols, const double* s, int invert,
                    void* stream) {
  if (!c) return PSVD_EINVAL;
  if (!X || !s || rows < 1 || cols < 1 || ld < rows) return fail(c, PSVD_EINVAL, "bad scale_cols arguments");
  dim3 g((unsigned)((rows + 255) / 256), (unsigned)cols);
  scale_cols_any_kernel<<<g, 256, 0, (cudaStream_t)stream>>>(X, ld, rows, cols, s, invert);
  c->launches++;
  return cuda_check(c, "scale cols");
}

}  // extern "C"
