/* psvd.h — C ABI of the B200-native streaming-SVD library (libpsvd.so).
 *
 * Drop-in boundary for the hot path of the reference `parsvd` package
 * (arXiv 2108.08845 / PyParSVD, /root/reference/pkg/src/parsvd).  The
 * reference is pure Python + numpy; its "FFI" for this path is numpy's
 * LAPACK/BLAS calls inside the functions cited per entry point below.  The
 * Python package paper_2108_08845_b200 binds these symbols with ctypes and
 * mirrors the reference's public functions (StreamConfig/StreamState/
 * stream_initialize/stream_incorporate/stream_all, parallel_stream_*,
 * gather_modes, RandomSketchConfig/low_rank_svd).
 *
 * Conventions
 *   - All matrices are column-major fp64 device memory with an explicit
 *     leading dimension (snapshot-contiguous, as the reference's PARSVD01
 *     file and wire formats, io.py:1-13 / comm.py:9-13).  Leading
 *     dimensions must be even and base pointers 16-byte aligned (128-bit
 *     loads); the Python layer pads when needed.
 *   - The caller owns every buffer passed in; the library owns only its
 *     context workspace.
 *   - Every call is asynchronous on `stream` (a cudaStream_t; NULL = legacy
 *     default stream) and never synchronizes with the host, except
 *     psvd_read_status.
 *   - Return codes: PSVD_OK, PSVD_EINVAL (-> ValueError), PSVD_ENOCONV
 *     (-> ConvergenceError, linalg.py:117-121), PSVD_ECUDA (-> RuntimeError).
 *   - One context per device per host thread; a context is not thread-safe.
 */
#ifndef PSVD_H_
#define PSVD_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PSVD_OK 0
#define PSVD_EINVAL 1
#define PSVD_ENOCONV 2
#define PSVD_ECUDA 3

/* device status bits (psvd_read_status) */
#define PSVD_ST_NONFINITE 1  /* a non-finite entry reached the update (linalg.py:76-77 ValueError) */
#define PSVD_ST_NOCONVERGE 2 /* small factorization failed (linalg.py:117-121 ConvergenceError) */
#define PSVD_ST_RESCUE 4     /* orthogonality-drift rescue ran (streaming.py:106-115) */
#define PSVD_ST_RANKDEF 8    /* a kept singular value is exactly zero */
#define PSVD_ST_CHOLFAIL 16  /* sketch Cholesky needed the shifted retry */
#define PSVD_ST_ILLCOND 32   /* deterministic Gram route: kept spectrum sigma_1 / sigma_K > 300, so the
                                update must be redone on the accurate route (psvd_stream_update_accurate) */
#define PSVD_ST_SKETCHCOND 64 /* randomized update: a sketch (or power-iteration) block had a direction at or below
                                3e-7 of its largest one, where the Gram-based orthonormalization (SVQB) drops or
                                blurs it while the reference's Householder qr keeps it (linalg.py:94-104, 143-147):
                                the caller redoes the update on the accurate route (psvd_qr after every product) */

typedef struct psvd_ctx psvd_ctx;

int psvd_version(void);
int psvd_create(int device, psvd_ctx** out);
int psvd_destroy(psvd_ctx* ctx);
const char* psvd_last_error(psvd_ctx* ctx);

/* Orthogonality-drift threshold of the streaming updates (default 1e-8 =
 * streaming.py:25 ORTHO_DRIFT_TOL).  A negative value forces the rescue
 * branch (tests). */
int psvd_set_drift_tol(psvd_ctx* ctx, double tol);

/* Row-partitioned randomized update: collective hooks the
 * library calls, in stream order on `stream`, at the exchange points of
 * psvd_rand_update — allreduce (sum in rank order, in place) of Y^T Y (l x l),
 * (Y T)^T (Y T) (l x l) and D P^T Y (n x l), and an allgather of the per-rank
 * (value, global row) argmax pairs (K x 2) for the tall sign rule.  row_offset
 * is the global index of this rank's first row.  Pass NULL hooks to go back to
 * the single-GPU update.  The hooks return 0 on success. */
typedef int (*psvd_allreduce_fn)(void* user, double* buf, int64_t count, void* stream);
typedef int (*psvd_allgather_fn)(void* user, const double* send, int64_t count, double* recv, void* stream);
int psvd_set_exchange(psvd_ctx* ctx, psvd_allreduce_fn allreduce, psvd_allgather_fn allgather, void* user,
                      int nranks, int64_t row_offset);

/* NCCL data plane of the same exchange points (no Python in the loop): the caller creates one
 * communicator per context from a unique id it distributes (psvd_nccl_unique_id on one rank, then a
 * broadcast, then psvd_nccl_init on every rank; libnccl.so.2 is loaded at run time) and enables it
 * around row-partitioned calls.  Each exchange is then an in-stream ncclAllGather on the library's
 * stream plus a rank-ordered sum, bitwise identical on every rank (replaces the reference's
 * gather / send / broadcast, dsvd.py:176-202).  Mutually exclusive with psvd_set_exchange. */
int psvd_nccl_available(int* ok);
int psvd_nccl_unique_id(psvd_ctx* ctx, unsigned char* id128);
int psvd_nccl_init(psvd_ctx* ctx, int nranks, int rank, const unsigned char* id128);
int psvd_nccl_enable(psvd_ctx* ctx, int on, int64_t row_offset);
int psvd_nccl_destroy(psvd_ctx* ctx);
/* Exchange accounting since context creation (the reference's CommStats, comm.py:74-88):
 * out[0] collectives issued at the exchange points, out[1] bytes received from other ranks. */
int psvd_exchange_stats(psvd_ctx* ctx, long long* out2);

/* Which core solver produced the last split-mode core solve (diagnostics, syncs the
 * device): *full = 0 when the subspace-iteration fast path converged, 1 when the
 * gated full Householder solver ran. */
int psvd_last_core_path(psvd_ctx* ctx, int* full);

/* Pass-kernel counters since context creation (diagnostics): out[0] narrow TMA passes,
 * out[1] TMA-fed Gram passes, out[2] cp.async Gram passes, out[3] general cp.async passes,
 * out[4] wide-route tall-skinny GEMM updates. */
int psvd_path_counters(psvd_ctx* ctx, long long* out5);

/* Number of kernels this context has enqueued so far (launch accounting). */
long long psvd_launch_count(psvd_ctx* ctx);

/* Diagnostics (with PSVD_EIG_TIMERS set in the environment): SM clock64()
 * stamps of the 9 phase boundaries of the last core eigensolver launch and 5
 * tridiagonalization sub-phase sums (14 entries; synchronous copy). */
int psvd_eig_phase_cycles(psvd_ctx* ctx, long long* out14);

/* Copy the context's device status word to *status (synchronizes `stream`);
 * reset != 0 clears it afterwards (stream-ordered). */
int psvd_read_status(psvd_ctx* ctx, int* status, int reset, void* stream);

/* ---- deterministic streaming update (streaming.py:63-116, dsvd.py:205-242) ----
 *
 * Panel C = [ff * U * diag(sigma) | A] with U (M x Kc, ld ldu), A (M x B, ld lda),
 * Kc = 0 for stream_initialize (then U, sigma are ignored).
 */

/* Local Gram G = C^T C (n x n, n = Kc + B, col-major ld n) — replaces the
 * np.concatenate + np.linalg.qr R-factor of streaming.py:97-98 / dsvd.py:187
 * (G = R^T R).  Reduction order is fixed: bitwise reproducible. */
int psvd_gram(psvd_ctx* ctx, int64_t M, const double* U, int64_t ldu, const double* sigma, double ff,
              int Kc, const double* A, int64_t lda, int B, double* G, void* stream);

/* Core factorization of a (summed) Gram: top-K eigenpairs, sigma_k =
 * sqrt(lambda_k) descending (= svd_full(R).s, linalg.py:107-123), the
 * reference sign rule on U_R (linalg.py:81-91) and the recompose weights
 * W (n x K, col-major ld n) such that U_new = [U | A] * W
 * (= q @ u[:, order] of streaming.py:102-103).  sigma_out: device, K. */
int psvd_core_eig(psvd_ctx* ctx, const double* G, int n, const double* sigma_in, double ff, int Kc, int K,
                  double* W, double* sigma_out, void* stream);

/* U_out (M x K, ld ldo) = [U | A] * W; optionally UtU (K x K) = U_out^T U_out
 * for the drift check.  U_out must not alias U or A. */
int psvd_recompose(psvd_ctx* ctx, int64_t M, const double* U, int64_t ldu, int Kc, const double* A,
                   int64_t lda, int B, const double* W, int K, double* U_out, int64_t ldo, double* UtU,
                   void* stream);

/* The fused pass of the pipelined stream as a call of its own (streaming.py:97-103 composed with the next
 * update's projection): U_out = [U | A] * W, UtU = U_out^T U_out (K x K) and AtU = A_next^T U_out
 * (Bn x K, col-major ld Bn) from one read of [U | A | A_next].  mode 0: the narrow TMA pass (16-row
 * stages: the round-1 kernel, kept as the fallback and as the A/B reference); mode 1: the split-ring
 * kernel (32-row 3-D TMA boxes; PSVD_EINVAL when the shapes do not qualify: K <= 24, M a multiple of
 * 16, the rings within shared memory).  With mode 1 and noff > 0 the
 * pass also forms the 32 x 32 blocks (2t, 2t + 1), t < noff <= 3, of A_next^T A_next (work taken off
 * the look-ahead Gram) into off_tiles, a (ceil(Bn / 32))^2 array of row-major 32 x 32 tiles. */
int psvd_fused_pass(psvd_ctx* ctx, int64_t M, const double* U, int64_t ldu, int Kc, const double* A, int64_t lda,
                    int B, const double* A_next, int64_t ldan, int Bn, const double* W, int K, double* U_out,
                    int64_t ldo, double* UtU, double* AtU, int mode, int noff, double* off_tiles, void* stream);

/* Rayleigh refinement after a recompose: with UtU = U^T U (K x K, summed over
 * ranks in the row-parallel case), sigma_k <- sigma_k * sqrt(UtU_kk) (= ||C v_k||),
 * U[:, k] /= sqrt(UtU_kk), UtU normalized in place.  Second-order accurate in
 * the Gram eigenvector error (sqrt(lambda) alone is eps*kappa^2). */
int psvd_refine_normalize(psvd_ctx* ctx, int64_t M, double* U, int64_t ldu, int K, double* UtU, double* sigma,
                          void* stream);

/* Drift rescue of streaming.py:106-115 driven by UtU on the device: if
 * max|UtU - I| > tol, U <- qr(U).q reordered and sigma <- sigma*|diag r|
 * reordered (stable descending); otherwise a no-op.  In place. */
int psvd_drift_rescue(psvd_ctx* ctx, int64_t M, double* U, int64_t ldu, int K, const double* UtU,
                      double* sigma, double tol, void* stream);

/* One whole single-GPU update = gram + core_eig + recompose (+ drift rescue
 * when rescue != 0): stream_initialize (Kc = 0) / stream_incorporate.
 * Gram route: its kept singular values carry eps (sigma_1 / sigma_k)^2 error terms.  When the
 * kept spectrum is wider than sigma_1 / sigma_K = 300 it sets PSVD_ST_ILLCOND in the status
 * word; the caller then redoes the update with psvd_stream_update_accurate. */
int psvd_stream_update(psvd_ctx* ctx, int64_t M, const double* U, int64_t ldu, const double* sigma,
                       double ff, int Kc, const double* A, int64_t lda, int B, int K, int rescue,
                       double* U_out, int64_t ldo, double* sigma_out, void* stream);

/* Whole deterministic stream (stream_all, streaming.py:119-133, or its
 * continuation from a state when Kc == K) over nb batches A[b] (M x B[b],
 * device pointers in a host array).  Same per-batch arithmetic as
 * psvd_stream_update; the A^T A Gram of batch b+1 runs on a low-priority
 * internal stream while the core solve of batch b runs on a high-priority
 * one.  Updates alternate between U_a and U_b (M x K, ld ldo; U_in must not
 * alias U_a); *final_buf receives 0 or 1.  sigma_hist: device, nb x K (the
 * singular values after every step).  Ordered after prior work on `stream`
 * and joined back into it.  batch_ready (optional, nb cudaEvent_t or NULL
 * entries): batch j is read only after its event, so host->device copies of
 * later batches can overlap the updates of earlier ones. */
/* 1 in *ok when psvd_stream_run supports batches of up to Bmax columns with K modes on M rows
 * (its look-ahead Gram and fused pass plan within the kernels' limits), else 0: stream those
 * batches through psvd_stream_update. */
int psvd_stream_run_supported(psvd_ctx* ctx, int64_t M, int K, int Bmax, int* ok);
/* In-step timing of psvd_stream_run's dominant kernel (benchmark evidence): mode 1 starts recording
 * CUDA-event pairs on the library's low-priority stream around every look-ahead A^T A Gram; mode 0
 * stops, synchronizes and returns out3 = {summed ms, launches timed, summed flops M B (B + 1)}. */
int psvd_gram_timing(psvd_ctx* ctx, int mode, double* out3);
int psvd_stream_run(psvd_ctx* ctx, int64_t M, const double* U_in, int64_t ldu, const double* sigma_in, int Kc,
                    int nb, const double* const* A, const int64_t* lda, const int* B, int K, double ff, int rescue,
                    double* U_a, double* U_b, int64_t ldo, double* sigma_hist, int* final_buf,
                    void* const* batch_ready, void* stream);

/* The accurate route of one deterministic update (same arguments and result as
 * psvd_stream_update) at any conditioning and rank: an orthonormal basis Q of the explicit
 * panel C = [ff U S | A] by Gram deflation (levels of Gram -> Jacobi eig -> keep lambda >
 * 1e-10 lambda_max -> CholeskyQR2 -> project out, until the residual is at rounding level),
 * B = Q^T C, the multi-CTA one-sided Jacobi SVD of B^T (relative accuracy, no squaring), the
 * reference's sign rule on U_R = R V S^-1 with R the Householder R of B (= the R of
 * qr(C), diag >= 0; streaming.py:97-103, linalg.py:81-104), U_out = Q U_B[:, :K] (orthonormal
 * by construction), then the drift rescue when rescue != 0.  Synchronizes the host (the
 * deflation levels are sized from device values).  Uses the exchange hooks when set: every
 * Gram / projection is summed over the row-partitioned ranks. */
int psvd_stream_update_accurate(psvd_ctx* ctx, int64_t M, const double* U, int64_t ldu, const double* sigma,
                                double ff, int Kc, const double* A, int64_t lda, int B, int K, int rescue,
                                double* U_out, int64_t ldo, double* sigma_out, void* stream);

/* qr_factor at any conditioning and rank (linalg.py:94-104): the same Gram-deflation basis,
 * completed to n orthonormal columns (deterministic pseudo-random candidates, projected out),
 * B = Q^T A, Householder QR of B (one CTA), Q <- Q Q_B.  psvd_qr takes this route itself when
 * the first Cholesky flags cond(A) > ~1e6.  Synchronizes the host.  Q: M x n (ld ldq), R: n x n. */
int psvd_qr_robust(psvd_ctx* ctx, int64_t M, int n, const double* A, int64_t lda, double* Q, int64_t ldq, double* R,
                   void* stream);

/* ---- one-shot distributed SVD helpers (APMOS, dsvd.py:80-173) ----
 * Top-k eigenpairs of a symmetric PSD n x n matrix G (col-major, ld n): V (n x k,
 * ld ldv) the eigenvectors, s = sqrt(max(lambda, 0)) descending (the right singular
 * vectors / values of any C with C^T C = G; generate_right_vectors' "gram" route). */
int psvd_sym_topk(psvd_ctx* ctx, const double* G, int n, int k, double* V, int64_t ldv, double* s, void* stream);

/* X (n x m, ld ldx) = A^T Y for tall A (M x n) and Y (M x m), both column-major with even
 * leading dimensions: the rows are split over CTAs and summed in a fixed order. */
int psvd_tn_product(psvd_ctx* ctx, int64_t M, const double* A, int64_t lda, int n, const double* Y, int64_t ldy,
                    int m, double* X, int64_t ldx, void* stream);

/* Column sign rule of linalg.py:81-91 in place: the largest-|.| entry of each column of
 * X (rows x cols, ld even) becomes positive (first row wins ties). */
int psvd_sign_by_peak(psvd_ctx* ctx, double* X, int64_t ld, int64_t rows, int cols, void* stream);

/* ---- randomized streaming update (low_rank_svd of the panel,
 * linalg.py:126-162) ----
 * U_out, sigma_out = low_rank_svd([ff U diag(sigma) | A], target_rank = K,
 * sketch width l = K + oversampling, q power iterations) with the Gaussian
 * test matrix Omega (n x l, n = Kc + B, col-major ld n) supplied by the caller
 * (the reference's Philox(seed).standard_normal((n, l)), linalg.py:141-142).
 * Range basis by SVQB (eigen-orthonormalization of the sketch Gram,
 * numerically null directions dropped) + one CholeskyQR refinement pass, projection B = Q^T C, one-sided
 * Jacobi SVD of B, and the tall sign rule on U (global argmax per column,
 * lowest row on ties, linalg.py:81-91, 161).  Kc = 0 for the first batch. */
int psvd_rand_update(psvd_ctx* ctx, int64_t M, const double* U, int64_t ldu, const double* sigma, double ff,
                     int Kc, const double* A, int64_t lda, int B, int K, int l, int q, const double* Omega,
                     double* U_out, int64_t ldo, double* sigma_out, void* stream);

/* Randomized stream over nb device batches (reference: stream_all with the R9 composition,
 * i.e. low_rank_svd([ff U S | A_b]) per batch, linalg.py:126-162 + streaming.py:119-133),
 * pipelined: the state between updates stays a sketch basis (U is written once, to U_out), and
 * the state-independent sketch A_{b+1} Omega[K:] of the next batch runs on a low-priority stream
 * while the one-CTA small solves of batch b run.  Omega[b]: the (n_b x l) test matrix of batch b
 * (col-major, ld n_b; n_b = K + B[b] after the first update, B[0] when Kc = 0).  sigma_hist:
 * nb x K singular values per update.  Requires l <= 32 (returns PSVD_EINVAL otherwise: use
 * psvd_rand_update per batch).  Row-partitioned with the exchange set (hooks or NCCL): every
 * exchange is issued on the library's high-priority stream in the same order on every rank. */
/* 1 in *ok when psvd_rand_stream_run's passes plan for batches of up to Bmax columns (sketch
 * width l, K modes, q power iterations) on M rows, else 0: use psvd_rand_update per batch. */
int psvd_rand_stream_run_supported(psvd_ctx* ctx, int64_t M, int K, int l, int q, int Bmax, int* ok);
int psvd_rand_stream_run(psvd_ctx* ctx, int64_t M, const double* U_in, int64_t ldu, const double* sigma_in, int Kc,
                         int nb, const double* const* A, const int64_t* lda, const int* B, int K, int l, int q,
                         double ff, const double* const* Omega, double* U_out, int64_t ldo, double* sigma_hist,
                         void* const* batch_ready, void* stream);

/* ---- dense factorizations behind the reference's linalg boundary ----
 * qr_factor (linalg.py:94-104): psvd_qr, tall A (M >= n, any n): CholeskyQR2, or the shifted
 * CholeskyQR3 when the first Cholesky flags cond(A) beyond CholeskyQR2's range (one host sync to
 * read that flag).  Q: M x n (ld ldq), R: n x n (ld n) upper with diag(R) >= 0.
 * svd_full (linalg.py:107-123): psvd_jacobi, one-sided Jacobi SVD of X (m x n, m >= n, any n;
 * S descending, V n x n), composed with psvd_qr for tall inputs; psvd_sign_pair applies the
 * reference's sign rule (linalg.py:81-91) to U and the same flips to V.
 * randomized_range (linalg.py:126-147): psvd_nn_product (Y = A W, A tall) with psvd_tn_product
 * and psvd_qr.  parallel_qr (dsvd.py:176-202): psvd_gram + rank-ordered sum + psvd_chol
 * (R and R^-1 of a Gram, any n) + psvd_nn_product + psvd_small_matmul (C = op(A) B, small). */
int psvd_chol(psvd_ctx* ctx, const double* G, int n, double* R, double* T, void* stream);
int psvd_chol_shift(psvd_ctx* ctx, double* G, int n, int64_t M, void* stream);
int psvd_chol_illcond(psvd_ctx* ctx, int* flag, void* stream);
int psvd_nn_product(psvd_ctx* ctx, int64_t M, const double* A, int64_t lda, int n, const double* W, int64_t ldw, int w,
                    double* Y, int64_t ldy, void* stream);
int psvd_small_matmul(psvd_ctx* ctx, const double* A, int lda, int transA, const double* B, int ldb, double* C,
                      int ldc, int m, int k, int n, void* stream);
int psvd_qr(psvd_ctx* ctx, int64_t M, int n, const double* A, int64_t lda, double* Q, int64_t ldq, double* R,
            void* stream);
int psvd_jacobi(psvd_ctx* ctx, const double* X, int64_t ldx, int64_t m, int n, double* S, double* V, int64_t ldv,
                void* stream);
int psvd_sign_pair(psvd_ctx* ctx, double* U, int64_t ldu, int64_t rows, int cols, double* V, int64_t ldv,
                   int64_t vrows, void* stream);
/* svd_full's core for any width (linalg.py:107-123; the reference's dgesdd of the R factor):
 * multi-CTA one-sided Jacobi on X (m x n, ld ldx) or, with transpose = 1, on X^T of an n x m X.
 * S (n) descending, V (n x n, ld ldv) the right singular vectors, optional U (m x n, ld ldu) =
 * X V S^-1 (0 columns for zero singular values).  Bitwise reproducible.  psvd_qr and psvd_chol take
 * any n as well (one-CTA kernels up to 112 columns, blocked global-memory kernels beyond). */
int psvd_jacobi_uv(psvd_ctx* ctx, const double* X, int64_t ldx, int64_t m, int n, int transpose, double* S,
                   double* V, int64_t ldv, double* U, int64_t ldu, void* stream);

/* Y (rows x cols, column-major, ld ldy) from a row-major X (row stride ldx): C-ordered input
 * (the reference's burgers_matrix returns C order) enters the library's column-major layout. */
int psvd_transpose(psvd_ctx* ctx, const double* X, int64_t ldx, int64_t rows, int64_t cols, double* Y, int64_t ldy,
                   void* stream);

/* X[:, j] *= s_j, or /= s_j (0 where s_j == 0) with invert = 1. */
int psvd_scale_cols(psvd_ctx* ctx, double* X, int64_t ld, int64_t rows, int cols, const double* s, int invert,
                    void* stream);
/* low_rank_svd's right factor (linalg.py:157-162) from the last psvd_rand_update on this context
 * (same stream, right after it): vt (K x n, ld ldvt), rows signed like the returned U's columns. */
int psvd_rand_last_vt(psvd_ctx* ctx, int n, int l, int K, double* Vt, int64_t ldvt, void* stream);

/* ---- row-parallel helpers ---- */

/* out (n x n) = sum_r parts[r] in rank order (parts: P contiguous n x n blocks);
 * used after an allgather so every GPU holds bitwise-identical sums. */
int psvd_sum_ordered(psvd_ctx* ctx, const double* parts, int P, int64_t count, double* out, void* stream);

/* ---- input generation (datagen.py:49-90 formula, device side) ----
 * out(i, j) = burgers u(x[row0 + i], t[col0 + j]) with x = linspace(0, length, grid),
 * t = linspace(0, t_final, n_snap); i < rows, j < cols; col-major ld ldo. */
int psvd_burgers(psvd_ctx* ctx, double* out, int64_t ldo, int64_t row0, int64_t rows, int64_t grid,
                 int col0, int cols, int n_snap, double length, double t_final, double reynolds,
                 void* stream);

#ifdef __cplusplus
}
#endif
#endif /* PSVD_H_ */
