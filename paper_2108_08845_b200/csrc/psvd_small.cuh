// Small-core kernels: one CTA, operate on n x n (n <= a few hundred) data that
// the tall passes reduced out of the M-row panel.  They run on the device
// stream between the tall passes, so an update never syncs with the host.
#pragma once
#include "psvd_common.cuh"

namespace psvd {

constexpr int SMALL_THREADS = 1024;
constexpr int EIG_NMAX_SMEM = 224;   // packed lower triangle kept in shared memory up to this n
constexpr int EIG_FAST_NMAX = 216;   // column-oriented lane-owned-rows path (7 rows per lane, 16 warps)
constexpr int EIG_FAST_THREADS = 512;

// Extract the n x n Gram block (rows/cols [c0, c0+n) of the combined column space)
// from reduced 32x32 tiles (tile id I*NB+J, I <= J computed), scaled symmetrically
// by d (length n, may be null): out[i][j] = d_i d_j T(c0+i, c0+j).  col-major, ld n.
void launch_extract_sym(const double* tiles, int NB, int c0, int n, const double* d, double* out,
                        cudaStream_t st);
// Assemble the streaming Gram from the narrow [U | A] pass tiles and the A^T A pass tiles.
void launch_assemble_gram(const double* tua, int nbua, const double* taa, int nbaa, int K, int B, const double* d,
                          double* G, cudaStream_t st);
void launch_assemble_gram_fused(const double* tf, int nbf, int a0, int yb, const double* UU, const double* scale,
                                const int* gate, const double* T, const double* taa, int nbaa, int K, int B,
                                const double* d, double* G, cudaStream_t st, double uu_w = 1.0);
// Extract the rectangular block rows [r0, r0+nr) x cols [c0, c0+nc) (r-block <= c-block),
// scaled by row factors d (length nr, may be null).  col-major, ld nr.
void launch_extract_rect(const double* tiles, int NB, int r0, int nr, int c0, int nc, const double* d,
                         double* out, cudaStream_t st);

// Top-K eigenpairs of the symmetric PSD n x n matrix G (col-major, ld n) and the
// recompose weights of the streaming update:
//   sigma_k = sqrt(lambda_k) (descending), V_k eigenvectors,
//   sign_k from the reference's rule applied to U_R = R V Sigma^-1 with
//   R = chol(G) (the R of qr(C), diag >= 0 — linalg.py:94-104, 81-91),
//   W[:, k] = dscale .* V[:, k] * sign_k / sigma_k   (dscale may be null).
// ws: global scratch of eig_workspace_doubles(n, K) doubles.
size_t eig_workspace_doubles(int n, int K);
// timers (optional, device): clock64() at the 9 phase boundaries (diagnostics).
void launch_eig_topk(const double* G, int n, int K, const double* dscale, double* W, double* sigma,
                     double* ws, int* status, long long* timers, cudaStream_t st, double rank_tol = 0.0,
                     int split = 0, const int* gate = nullptr);

// Subspace-iteration fast path (psvd_subspace.cu): Ritz pairs of G from span(G^2 Q0), block 32.
// Writes Z (n x K, ld n) and sigma = sqrt(theta) like the split-mode solver and sets *gate = 0
// when every residual ||G x_k - theta_k x_k|| <= SS_TOL * theta_0, else *gate = 1 (the gated
// full solver then runs).  ss_ws: subspace_workspace_doubles(n) doubles.
#ifndef PSVD_SS_P
#define PSVD_SS_P 32
#endif
constexpr int SS_P = PSVD_SS_P;
constexpr int SS_THREADS = 512;
constexpr int SS_KMAX = 12;
constexpr int SS_ITERS = 2;
constexpr double SS_TOL = 2e-14;
bool subspace_supported(int n, int K);
size_t subspace_workspace_doubles(int n);
void launch_subspace_eig(const double* G, int n, int K, double* ss_ws, double* Zout, double* sigma_out, int* gate,
                         cudaStream_t st);
// Split core (n <= EIG_FAST_NMAX): eig with split = 1 leaves Z in ws + n(n+1)/2 and sqrt(lambda)
// in sigma; ldlt_pack (concurrent, needs only G) writes chol(G + delta I) packed to Lout;
// sign_weights then applies the sign rule and writes W.
bool eig_split_supported(int n, int K);
void launch_ldlt_pack(const double* G, int n, double* Lout, cudaStream_t st);
void launch_sign_weights(const double* Lg, const double* Z, const double* sigma, int n, int K, const double* dscale,
                         double* W, double* sigma_out, int* status, double rank_tol, cudaStream_t st);
bool eig_supported(int n, int K);

// Rayleigh refinement of sigma from the recomposed columns' norms (see psvd_small.cu); sets
// PSVD_ST_ILLCOND in *status when sigma_1 / sigma_K > GRAM_KAPPA_MAX (the Gram route's accuracy gate).
constexpr double GRAM_KAPPA_MAX = 300.0;
void launch_normalize_gram(double* UtU, int K, double* sigma, double* scale, int* status, cudaStream_t st);

// Drift check of streaming.py:106-115 on the K x K Gram UtU = U_new^T U_new:
// if max|UtU - I| > tol: T = rr^{-1}[:, order] with rr = chol(UtU) (= qr(U).R),
// sigma <- (sigma * |diag rr|)[order] (stable descending), *gate = 1; else *gate = 0.
void launch_drift_check(const double* UtU, int K, double tol, double* sigma, double* T, int* gate,
                        int* status, cudaStream_t st);
// the check keeps (2 K^2 + K + 65 + (K + 1) / 2) doubles in shared memory: K <= 120 within 227 KB
constexpr int DRIFT_SMEM_KMAX = 120;

// ---- randomized-update helpers (psvd_rand.cu)
void launch_small_gemm(const double* A, int lda, int transA, const double* B, int ldb, double* C, int ldc, int m,
                       int k1, int k2, const double* rowscale, cudaStream_t st);
size_t jacobi_workspace_doubles(int n, int l);
constexpr int JACOBI_NMAX = 160;  // the rotation accumulator J (n x n) lives in shared memory
void launch_jacobi_svd(const double* Z, int n, int l, double* S, double* J, double* ws, int* status, cudaStream_t st,
                       const int* gate = nullptr);
void launch_chol_inv(const double* G, int l, double* T, cudaStream_t st, int* illcond = nullptr, int* status = nullptr,
                     double* Rout = nullptr);
constexpr int CHOL_NMAX = 112;  // chol_inv keeps R and R^-1 in shared memory
void launch_chol_shift(double* G, int n, int64_t M, cudaStream_t st);
void launch_colmax_sign(const double* colmax, int nchunks, int K, double* sign, cudaStream_t st);
void launch_colmax_reduce(const double* colmax, int nchunks, int K, double* out, cudaStream_t st);
void launch_svqb_scale(double* T, const double* S, int l, double tol, cudaStream_t st, const int* gate = nullptr,
                       int* status = nullptr);
void launch_scale_cols(double* U, int64_t ld, int64_t M, int K, const double* s, cudaStream_t st);
void launch_scale_rows(const double* X, int ldx, int m, int k, const double* d, double* Y, int ldy, cudaStream_t st);

// ---- any-width dense kernels, operands in global memory (psvd_big.cu)
// chol_big: same contract as launch_chol_inv (T = R^-1, optional Rout, zero rows for numerically null
// pivots, *illcond for cond > ~1e6) for any n; ws: chol_big_workspace_doubles(n).
size_t chol_big_workspace_doubles(int n);
void launch_chol_big(const double* G, int n, double* T, int* illcond, int* status, double* Rout, double* ws,
                     cudaStream_t st);
int chol_big_launches(int n);
// jacobi_big: one-sided Jacobi SVD of X (m x n, ld ldx; transpose = 1 takes X^T of an n x m X):
// S (n, descending), V (n x n, ld ldv) the accumulated rotations (right singular vectors), optional
// U (m x n, ld ldu) = X V S^-1.  ws: jacobi_big_workspace_doubles(m, n).  Returns a cudaError_t.
size_t jacobi_big_workspace_doubles(int64_t m, int n);
int launch_jacobi_big(const double* X, int64_t ldx, int64_t m, int n, int transpose, double* S, double* V,
                      int64_t ldv, double* U, int64_t ldu, double* ws, int* status, int* sweeps_out, int num_sms,
                      cudaStream_t st);

// ---- pipelined randomized stream glue (psvd_rand.cu; see psvd_rand_stream_run)
void launch_rs_prep(const double* sgn, const double* Wf, int lq, int K, const double* sigma, double ff,
                    const double* Om, int ldom, const double* QtQ, const double* tiles, int NB, int q_c0, int y_c0,
                    int l, int have_q, double* Etop, double* C, double* G1, cudaStream_t st);
void launch_rs_wb(const double* C, int lq, const double* T1, int l, int have_q, double* Wb, cudaStream_t st);
void launch_rs_post(const double* tiles, int NB, int q_c0, int a_c0, int y_c0, int lq, int B, int l,
                    const double* Etop, int K, int have_q, double* G2, double* X, cudaStream_t st);
void launch_rs_w0(const double* Etop, int lq, int K, const double* Qz, int n, int B, int l, int have_q, double* W0,
                  cudaStream_t st);
void launch_rs_ident(double* I, double* ones, int K, cudaStream_t st);
// U = Q W (optional write) with per-CTA column argmax pairs for the sign rule: qw_colmax_chunks
// CTAs over contiguous row ranges (chunk order = row order).
int64_t qw_colmax_rows(int64_t M, int num_sms);
int qw_colmax_chunks(int64_t M, int num_sms);
bool qw_colmax_supported(int l, int K);
void launch_qw_colmax(const double* Q, int64_t ldq, int64_t M, int l, const double* W, int K, double* U, int64_t ldu,
                      int64_t row_offset, double* colmax, int num_sms, cudaStream_t st);

}  // namespace psvd
