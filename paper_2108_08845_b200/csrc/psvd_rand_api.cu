// C ABI of the randomized update (include/psvd.h): per batch (psvd_rand_update) and the pipelined
// stream (psvd_rand_stream_run), low_rank_svd's right factor (reference linalg.py:126-162 composed
// per batch).
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

__global__ void rand_vt_kernel(const double* __restrict__ Bt, int n, int l, const double* __restrict__ J,
                               const double* __restrict__ S, const double* __restrict__ sgn, int K,
                               double* __restrict__ Vt, int64_t ldvt) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= n * K) return;
  const int k = idx % K, j = idx / K;
  double v = 0.0;
  for (int i = 0; i < l; ++i) v = fma(Bt[(size_t)i * n + j], J[(size_t)k * l + i], v);
  Vt[(size_t)j * ldvt + k] = S[k] != 0.0 ? sgn[k] * v / S[k] : 0.0;
}

// G (w x w, ld w) = Y^T Y of a tall M x w panel on the Gram pass (upper 32 x 32 tiles, fixed-order reduce);
// unlike psvd_gram it leaves the context's panel scaling (dvec) alone
int narrow_gram(psvd_ctx* c, int64_t M, const double* Y, int64_t ldy, int w, double* G, cudaStream_t st) {
  Pass ps;
  int rc = plan_pass(c, ps, M, {Seg{Y, ldy, w, 0}}, 0, 0, 0, nullptr, 0, true, false, false);
  if (rc) return rc;
  if ((rc = run_pass(c, ps, st))) return rc;
  launch_extract_sym((const double*)c->tiles.ptr, ps.NB, 0, w, nullptr, G, st);
  c->launches++;
  return cuda_check(c, "narrow gram");
}

// sign rule over ranks: local per-chunk pairs -> one pair per column -> allgather -> sign
int exchange_sign(psvd_ctx* c, const double* local_pairs, int nchunks, int K, double* sgn, cudaStream_t st) {
  if (!ex_active(c)) {
    launch_colmax_sign(local_pairs, nchunks, K, sgn, st);
    c->launches++;
    return PSVD_OK;
  }
  int rc;
  if ((rc = ensure(c, c->xpairs, sizeof(double) * (size_t)(c->ex_nranks + 1) * K * 2))) return rc;
  double* mine = (double*)c->xpairs.ptr;
  double* all = mine + (size_t)K * 2;
  launch_colmax_reduce(local_pairs, nchunks, K, mine, st);
  if (c->nccl_on) {
    if ((rc = nccl_allgather(c, mine, (int64_t)K * 2, all, st))) return rc;
  } else {
    c->ex_calls++;
    c->ex_bytes += 16 * (int64_t)K * (c->ex_nranks - 1);
    if (c->ex_allgather(c->ex_user, mine, (int64_t)K * 2, all, (void*)st) != 0)
      return fail(c, PSVD_ECUDA, "allgather hook failed");
  }
  launch_colmax_sign(all, c->ex_nranks, K, sgn, st);  // rank order = global row order: first rank wins ties
  c->launches += 2;
  return PSVD_OK;
}

// SVQB weights T = V diag(lambda^-1/2) of the l x l sketch Gram (numerically null directions
// dropped at 1e-7 relative), from a one-sided Jacobi eigen-decomposition of the Gram.
int svqb(psvd_ctx* c, const double* Gs, int l, double* T, double* sig_scratch, cudaStream_t st) {
  int rc = ensure(c, c->eigws, sizeof(double) * std::max(eig_workspace_doubles(l, l), jacobi_workspace_doubles(l, l)));
  if (rc) return rc;
  // CholeskyQR weights T = R^-1 first (one short kernel); when the sketch is ill conditioned
  // (max R_ii / min R_ii > 1e6 or a dropped pivot) the gated Jacobi SVQB overwrites them
  int* illcond = c->d_status + 3;
  launch_chol_inv(Gs, l, T, st, illcond, c->d_status);
  launch_jacobi_svd(Gs, l, l, sig_scratch, T, (double*)c->eigws.ptr, c->d_status, st, illcond);
  launch_svqb_scale(T, sig_scratch, l, 1e-7, st, illcond, c->d_status);
  c->launches += 3;
  return cuda_check(c, "svqb");
}

}  // namespace psvd_internal

extern "C" {

int psvd_rand_update(psvd_ctx* c, int64_t M, const double* U, int64_t ldu, const double* sigma, double ff, int Kc,
                     const double* A, int64_t lda, int B, int K, int l, int q, const double* Omega, double* U_out,
                     int64_t ldo, double* sigma_out, void* stream) {
  if (!c) return PSVD_EINVAL;
  cudaStream_t st = (cudaStream_t)stream;
  const int n = Kc + B;
  int rc;
  if (M < 1 || B < 1 || Kc < 0 || K < 1 || l < K || q < 0) return fail(c, PSVD_EINVAL, "bad randomized shape");
  // the sketch's Cholesky / SVQB / Jacobi solvers are the one-CTA kernels: wider sketches are the caller's
  // (linalg.randomized_update composes them from the any-width products, psvd_qr and the multi-CTA Jacobi)
  if (l > CHOL_NMAX)
    return fail(c, PSVD_EINVAL, "sketch width %d exceeds the %d columns of psvd_rand_update", l, CHOL_NMAX);
  // (row-partitioned: M is this rank's block, which may be shorter than the sketch; the caller checks the global rows)
  const int64_t rows_chk = ex_active(c) ? std::max<int64_t>(M, l) : M;
  if (l > std::min<int64_t>(rows_chk, n))
    return fail(c, PSVD_EINVAL, "sketch width %d exceeds min(a.shape) = %lld", l, (long long)std::min<int64_t>(rows_chk, n));
  if ((rc = check_mat(c, "U", U, ldu, M, Kc)) || (rc = check_mat(c, "A", A, lda, M, B)) ||
      (rc = check_mat(c, "U_out", U_out, ldo, M, K)))
    return rc;
  if (!Omega || !sigma_out || (Kc > 0 && !sigma)) return fail(c, PSVD_EINVAL, "null pointer");
  const int64_t ldy = M + (M & 1);
  if ((rc = ensure(c, c->ybuf, sizeof(double) * (size_t)ldy * l))) return rc;
  // small buffers: W0 (n x l), G1, T1, G2, T2 (l x l), X, Z, Z1, Qz, Bt (n x l), S (l), J (l x l), Wf (l x K), sign (K)
  const size_t nl = (size_t)n * l, ll = (size_t)l * l;
  if ((rc = ensure(c, c->rsmall, sizeof(double) * (6 * nl + 6 * ll + 2 * l + (size_t)l * K + K + 64)))) return rc;
  double* base = (double*)c->rsmall.ptr;
  double* W0 = base;
  double* X = W0 + nl;
  double* Z = X + nl;
  double* Z1 = Z + nl;
  double* Qz = Z1 + nl;
  double* Bt = Qz + nl;
  double* G1 = Bt + nl;
  double* T1 = G1 + ll;
  double* G2 = T1 + ll;
  double* T2 = G2 + ll;
  double* J = T2 + ll;
  double* Tz = J + ll;
  double* S = Tz + ll;
  double* sscr = S + l;
  double* Wf = sscr + l;
  double* sgn = Wf + (size_t)l * K;
  double* Y = (double*)c->ybuf.ptr;
  if ((rc = ensure(c, c->jacws, sizeof(double) * jacobi_workspace_doubles(n, l)))) return rc;
  if ((rc = make_dvec(c, sigma, ff, Kc, n, st))) return rc;
  const double* d = (const double*)c->dvec.ptr;
  launch_scale_rows(Omega, n, n, l, d, W0, n, st);  // Y = [ff U S | A] Omega = [U | A] (D Omega)
  c->launches++;
  // Panels too wide for the fused passes (sketch + Gram tiles in one read, W resident in smem)
  // take the tall-skinny GEMM route: same sequence of products, one product per launch.
  std::vector<Seg> pa = panel(U, ldu, Kc, A, lda, B);
  std::vector<Seg> pb = pa;
  pb.push_back(Seg{Y, ldy, l, 0});
  // the projection pass writes Y1 = Y T1 to a second buffer: with more than one slice CTA per row
  // chunk an in-place update would race (slice 0 writes rows the other slices still read)
  if ((rc = ensure(c, c->ybuf2, sizeof(double) * (size_t)ldy * l))) return rc;
  double* Y1b = (double*)c->ybuf2.ptr;
  bool wide = l > MAX_W || getenv("PSVD_FORCE_WIDE") != nullptr;
  if (!wide) {  // dry-run plans of the fused passes (no launches): wide when they do not fit
    Pass t1, t2;
    wide = plan_pass(c, t1, M, pa, 0, n, l, W0, n, false, true, false) != PSVD_OK ||
           plan_pass(c, t2, M, pb, n, l, l, T1, l, false, true, true, n) != PSVD_OK;
  }
  if (wide) {
    c->path_count[4]++;
    if ((rc = ensure(c, c->ybuf2, sizeof(double) * (size_t)ldy * l))) return rc;
    double* Y2 = (double*)c->ybuf2.ptr;
    const size_t part = std::max(tgemm_tn_partial_doubles(M, n, l, c->num_sms), tgemm_tn_partial_doubles(M, l, l, c->num_sms));
    if ((rc = ensure(c, c->partial, sizeof(double) * part))) return rc;
    double* pbuf = (double*)c->partial.ptr;
    std::vector<GemmSeg> gp;
    if (Kc > 0) gp.push_back(GemmSeg{U, ldu, Kc});
    gp.push_back(GemmSeg{A, lda, B});
    const GemmSeg gy{Y, ldy, l}, gy2{Y2, ldy, l};
    for (int it = 0; it <= q; ++it) {
      launch_tgemm_nn(M, gp.data(), (int)gp.size(), W0, n, l, Y, ldy, st);           // Y = P W0
      c->launches++;
      // G1 = Y^T Y on the Gram pass (upper 32 x 32 tiles, TMA-fed, unread sub-blocks trimmed): about half
      // the DMMA work of the 64 x 64 tiles of the general TN product
      if ((rc = narrow_gram(c, M, Y, ldy, l, G1, st))) return rc;
      if ((rc = ex_allreduce(c, G1, (int64_t)l * l, st))) return rc;
      if ((rc = svqb(c, G1, l, T1, sscr, st))) return rc;
      launch_tgemm_nn(M, &gy, 1, T1, l, l, Y2, ldy, st);                              // Y1 = Y T1
      c->launches++;
      if ((rc = narrow_gram(c, M, Y2, ldy, l, G2, st))) return rc;  // G2 = Y1^T Y1
      // (the Gram pass may have grown the shared partial-tile workspace: take its current address)
      if ((rc = ensure(c, c->partial, sizeof(double) * part))) return rc;
      pbuf = (double*)c->partial.ptr;
      launch_tgemm_tn(M, gp.data(), (int)gp.size(), Y2, ldy, l, d, X, n, pbuf, c->num_sms, st);  // X = D P^T Y1
      c->launches += 2;
      if ((rc = ex_allreduce(c, G2, (int64_t)l * l, st)) || (rc = ex_allreduce(c, X, (int64_t)n * l, st))) return rc;
      launch_chol_inv(G2, l, T2, st);
      launch_small_gemm(X, n, 0, T2, l, (it < q) ? Z : Bt, n, n, l, l, nullptr, st);
      c->launches += 2;
      if (it < q) {
        launch_small_gemm(Z, n, 1, Z, n, G1, l, l, n, l, nullptr, st);
        c->launches++;
        if ((rc = svqb(c, G1, l, Tz, sscr, st))) return rc;
        launch_small_gemm(Z, n, 0, Tz, l, Z1, n, n, l, l, nullptr, st);
        launch_small_gemm(Z1, n, 1, Z1, n, G1, l, l, n, l, nullptr, st);
        launch_chol_inv(G1, l, Tz, st);
        launch_small_gemm(Z1, n, 0, Tz, l, Qz, n, n, l, l, nullptr, st);
        launch_scale_rows(Qz, n, n, l, d, W0, n, st);
        c->launches += 5;
      }
    }
    if (n >= 2 * l && l <= CHOL_NMAX) {
      // small SVD of B through a QR of B^T (CholeskyQR2, n x l) and one-sided Jacobi on R (l x l):
      // B^T J = Q (R J) gives the same J and column norms, and rotating columns of length l
      // instead of n costs n / l times less; an ill-conditioned B^T (max R_ii / min R_ii > 1e6)
      // takes the gated Jacobi on B^T itself
      int* illcond = c->d_status + 3;
      double* R1 = Tz;
      double* R2 = Z;
      double* Rq = Qz;
      launch_small_gemm(Bt, n, 1, Bt, n, G1, l, l, n, l, nullptr, st);    // B B^T
      launch_chol_inv(G1, l, T1, st, illcond, c->d_status, R1);
      launch_small_gemm(Bt, n, 0, T1, l, Z1, n, n, l, l, nullptr, st);    // Q1 = B^T R1^-1
      launch_small_gemm(Z1, n, 1, Z1, n, G2, l, l, n, l, nullptr, st);
      launch_chol_inv(G2, l, X, st, nullptr, nullptr, R2);
      launch_small_gemm(R2, l, 0, R1, l, Rq, l, l, l, l, nullptr, st);    // R = R2 R1
      launch_jacobi_svd(Rq, l, l, S, J, (double*)c->jacws.ptr, c->d_status, st);
      launch_jacobi_svd(Bt, n, l, S, J, (double*)c->jacws.ptr, c->d_status, st, illcond);
      c->launches += 8;
    } else {
      launch_jacobi_svd(Bt, n, l, S, J, (double*)c->jacws.ptr, c->d_status, st);
    }
    launch_small_gemm(T2, l, 0, J, l, Wf, l, l, l, K, nullptr, st);
    launch_tgemm_nn(M, &gy2, 1, Wf, l, K, U_out, ldo, st);  // U = Y1 (T2 U_B[:, :K])
    const int64_t nch = colmax_rows_chunks(M);
    if ((rc = ensure(c, c->colmax, sizeof(double) * (size_t)nch * K * 2))) return rc;
    launch_colmax_rows(U_out, ldo, M, K, c->ex_row_offset, (double*)c->colmax.ptr, st);
    if ((rc = exchange_sign(c, (const double*)c->colmax.ptr, (int)nch, K, sgn, st))) return rc;
    launch_scale_cols(U_out, ldo, M, K, sgn, st);
    cudaMemcpyAsync(sigma_out, S, sizeof(double) * K, cudaMemcpyDeviceToDevice, st);
    c->launches += 5;
    return cuda_check(c, "randomized update (wide)");
  }
  for (int it = 0; it <= q; ++it) {
    // pass A: Y = P W0, Y^T Y
    Pass ps;
    if ((rc = plan_pass(c, ps, M, pa, 0, n, l, W0, n, false, true, false))) return rc;
    ps.p.Yout = Y;
    ps.p.ldy = ldy;
    if ((rc = run_pass(c, ps, st))) return rc;
    launch_extract_sym((const double*)c->tiles.ptr, ps.NB, ps.p.np_pad, l, nullptr, G1, st);
    c->launches++;
    if ((rc = ex_allreduce(c, G1, (int64_t)l * l, st))) return rc;
    if ((rc = svqb(c, G1, l, T1, sscr, st))) return rc;
    // pass B: Y1 = Y T1 (into the second buffer), (Y1^T Y1, D P^T Y1)
    Pass pb_;
    if ((rc = plan_pass(c, pb_, M, pb, n, l, l, T1, l, false, true, true, n))) return rc;
    pb_.p.Yout = Y1b;
    pb_.p.ldy = ldy;
    if ((rc = run_pass(c, pb_, st))) return rc;
    launch_extract_sym((const double*)c->tiles.ptr, pb_.NB, pb_.p.np_pad, l, nullptr, G2, st);
    launch_extract_rect((const double*)c->tiles.ptr, pb_.NB, 0, n, pb_.p.np_pad, l, d, X, st);
    c->launches += 2;
    if ((rc = ex_allreduce(c, G2, (int64_t)l * l, st)) || (rc = ex_allreduce(c, X, (int64_t)n * l, st))) return rc;
    launch_chol_inv(G2, l, T2, st);  // refinement pass: G2 ~ I, Cholesky is exact enough
    c->launches++;
    // Z = C^T Q = (D P^T Y1) T2 = X T2  (= B^T after the last iteration)
    launch_small_gemm(X, n, 0, T2, l, (it < q) ? Z : Bt, n, n, l, l, nullptr, st);
    c->launches++;
    if (it < q) {  // power iteration: Qz = orth(Z) by SVQB twice, next sketch W0 = D Qz
      launch_small_gemm(Z, n, 1, Z, n, G1, l, l, n, l, nullptr, st);
      c->launches++;
      if ((rc = svqb(c, G1, l, Tz, sscr, st))) return rc;
      launch_small_gemm(Z, n, 0, Tz, l, Z1, n, n, l, l, nullptr, st);
      launch_small_gemm(Z1, n, 1, Z1, n, G1, l, l, n, l, nullptr, st);
      launch_chol_inv(G1, l, Tz, st);
      c->launches += 3;
      launch_small_gemm(Z1, n, 0, Tz, l, Qz, n, n, l, l, nullptr, st);
      launch_scale_rows(Qz, n, n, l, d, W0, n, st);
      c->launches += 2;
    }
  }
  // small SVD of B = Q^T C (l x n) through B^T = Bt: U_B = J, S descending
  launch_jacobi_svd(Bt, n, l, S, J, (double*)c->jacws.ptr, c->d_status, st);
  // U = Q U_B[:, :K] = Y1 (T2 J[:, :K])
  launch_small_gemm(T2, l, 0, J, l, Wf, l, l, l, K, nullptr, st);
  c->launches += 2;
  int nchunks;
  if (qw_colmax_supported(l, K)) {
    nchunks = qw_colmax_chunks(M, c->num_sms);
    if ((rc = ensure(c, c->colmax, sizeof(double) * (size_t)nchunks * K * 2))) return rc;
    launch_qw_colmax(Y1b, ldy, M, l, Wf, K, U_out, ldo, c->ex_row_offset, (double*)c->colmax.ptr, c->num_sms, st);
    c->launches++;
  } else {
    Pass pc;
    if ((rc = plan_pass(c, pc, M, {Seg{Y1b, ldy, l, 0}}, 0, l, K, Wf, l, false, false, false))) return rc;
    nchunks = pc.map.nchunks;
    if ((rc = ensure(c, c->colmax, sizeof(double) * (size_t)nchunks * K * 2))) return rc;
    pc.p.Yout = U_out;
    pc.p.ldy = ldo;
    pc.p.colmax = (double*)c->colmax.ptr;
    pc.p.row_offset = c->ex_row_offset;
    if ((rc = run_pass(c, pc, st))) return rc;
  }
  if ((rc = exchange_sign(c, (const double*)c->colmax.ptr, nchunks, K, sgn, st))) return rc;
  launch_scale_cols(U_out, ldo, M, K, sgn, st);
  cudaMemcpyAsync(sigma_out, S, sizeof(double) * K, cudaMemcpyDeviceToDevice, st);
  c->launches += 1;
  return cuda_check(c, "randomized update");
}

// Pipelined randomized stream (SURVEY §8 R9 over a batch list; reference linalg.py:126-162 composed
// per batch).  The state between updates is the sketch basis Q_b = Y1_b (M x l) plus small weights
// (U_b = Q_b Wf_b diag(s_b)), so U is materialized once, at the end.  Per update b:
//   hi:  sign pass over Q_{b-1} (argmax of Q Wf)  ->  G1 = Y^T Y for Y = Q C + Z_b (small)  ->  SVQB
//        ->  projection pass over [Q_{b-1} | Z_b | A_b]: Y1 = (Q C + Z_b) T1, Y1^T Y1, [Q | A]^T Y1
//        ->  [power iterations: sketch pass over [Q | A], projection pass]  ->  Cholesky, Jacobi SVD
//   lo:  Z_{b+1} = A_{b+1} Omega[K:] with Q_b^T Z_{b+1} and Z^T Z (the state-independent half of the
//        next sketch), started as soon as Q_b is final so it overlaps the one-SM small solves.
// Same arithmetic as psvd_rand_update per batch up to rounding (U is replaced by Q Wf diag(s)).
int psvd_rand_stream_run(psvd_ctx* c, int64_t M, const double* U_in, int64_t ldu, const double* sigma_in, int Kc,
                         int nb, const double* const* A, const int64_t* lda, const int* B, int K, int l, int q,
                         double ff, const double* const* Omega, double* U_out, int64_t ldo, double* sigma_hist,
                         void* const* batch_ready, void* stream) {
  if (!c) return PSVD_EINVAL;
  if (nb < 1 || !A || !lda || !B || !Omega || !U_out || !sigma_hist)
    return fail(c, PSVD_EINVAL, "bad rand_stream_run arguments");
  if (K < 1 || l < K || q < 0) return fail(c, PSVD_EINVAL, "bad sketch K=%d l=%d q=%d", K, l, q);
  if (l > TMA_MAX_Y || !tma_available() || !qw_colmax_supported(l, K))
    return fail(c, PSVD_EINVAL, "sketch width %d not supported by the pipelined run (use psvd_rand_update)", l);
  if (Kc != 0 && Kc != K) return fail(c, PSVD_EINVAL, "initial state carries %d modes, K=%d", Kc, K);
  if (Kc > 0 && (!U_in || !sigma_in)) return fail(c, PSVD_EINVAL, "null initial state");
  int rc;
  int bmax = 0;
  for (int b = 0; b < nb; ++b) {
    if ((rc = check_mat(c, "A", A[b], lda[b], M, B[b]))) return rc;
    if (B[b] < 1) return fail(c, PSVD_EINVAL, "empty batch");
    if (!Omega[b]) return fail(c, PSVD_EINVAL, "null Omega");
    const int n = ((b > 0 || Kc > 0) ? K : 0) + B[b];
    const int64_t rows_chk = ex_active(c) ? std::max<int64_t>(M, l) : M;  // row-partitioned: the caller checks the global rows
    if (l > std::min<int64_t>(rows_chk, n))
      return fail(c, PSVD_EINVAL, "sketch width %d exceeds min(a.shape) = %lld", l, (long long)std::min<int64_t>(rows_chk, n));
    bmax = std::max(bmax, B[b]);
  }
  if (Kc == 0 && B[0] < K) return fail(c, PSVD_EINVAL, "initial batch has %d columns, need at least k_modes=%d", B[0], K);
  if ((rc = check_mat(c, "U_out", U_out, ldo, M, K))) return rc;
  if (Kc > 0 && (rc = check_mat(c, "U_in", U_in, ldu, M, K))) return rc;
  const int64_t ldq = M + (M & 1);
  if ((rc = ensure(c, c->ybuf, sizeof(double) * (size_t)ldq * l)) ||
      (rc = ensure(c, c->ybuf2, sizeof(double) * (size_t)ldq * l)) ||
      (rc = ensure(c, c->zbuf, sizeof(double) * (size_t)ldq * l)))
    return rc;
  double* Qb[2] = {(double*)c->ybuf.ptr, (double*)c->ybuf2.ptr};
  double* Zt = (double*)c->zbuf.ptr;
  const int nmax = K + bmax;
  const size_t ll = (size_t)l * l, nl = (size_t)nmax * l;
  const size_t need = (size_t)l * K + 4 * ll + 2 * ll + 2 * ll + ll + 5 * nl + ll + (size_t)(l + bmax) * l + 2 * l +
                      2 * (size_t)l * K + K + 2 * (size_t)K * K + K + 64;
  if ((rc = ensure(c, c->rs2, sizeof(double) * need))) return rc;
  double* p_ = (double*)c->rs2.ptr;
  auto take = [&](size_t n_) { double* r = p_; p_ += n_; return r; };
  double* Etop = take((size_t)l * K);
  double* Cm = take(ll);
  double* G1 = take(ll);
  double* T1 = take(ll);
  double* Wb = take(2 * ll);
  double* G2[2] = {take(ll), take(ll)};
  double* T2 = take(ll);
  double* X = take(nl);
  double* Zs = take(nl);
  double* Z1 = take(nl);
  double* Qz = take(nl);
  double* Bt = take(nl);
  double* Tz = take(ll);
  double* W0 = take((size_t)(l + bmax) * l);
  double* S = take(l);
  double* sscr = take(l);
  double* J = take(ll);
  double* Wf[2] = {take((size_t)l * K), take((size_t)l * K)};
  double* sgn = take(K);
  double* WfI = take((size_t)K * K);
  double* QtQ0 = take((size_t)K * K);
  double* ones = take(K);
  if ((rc = ensure(c, c->jacws, sizeof(double) * jacobi_workspace_doubles(nmax, l)))) return rc;
  cudaStream_t user = (cudaStream_t)stream, hi = c->s_hi, lo = c->s_lo;
  // PSVD_TRACE=1: timeline of the two streams on stderr (diagnostics; %globaltimer stamps)
  static const bool trace = getenv("PSVD_TRACE") != nullptr;
  std::vector<std::string> tl;
  unsigned long long* tbuf = nullptr;
  if (trace) cudaMallocManaged(&tbuf, 512 * sizeof(unsigned long long));
  auto mark = [&](const char* what, int b, cudaStream_t s_) {
    if (!trace || tl.size() >= 512) return;
    launch_stamp(tbuf + tl.size(), s_);
    tl.push_back(std::string(what) + "[" + std::to_string(b) + "]");
  };
  mark("start", 0, user);
  cudaEventRecord(c->ev_fork, user);
  cudaStreamWaitEvent(hi, c->ev_fork, 0);
  cudaStreamWaitEvent(lo, c->ev_fork, 0);
  if (Kc > 0) {  // user state: Q = U_in, Wf = I, signs +1, Q^T Q from one narrow pass
    launch_rs_ident(WfI, ones, K, hi);
    c->launches++;
    Pass pu;
    if ((rc = plan_pass(c, pu, M, {Seg{U_in, ldu, K, 0}}, 0, K, K, WfI, K, false, true, false))) return rc;
    if ((rc = run_pass(c, pu, hi))) return rc;
    launch_extract_sym((const double*)c->tiles.ptr, pu.NB, pu.p.np_pad, K, nullptr, QtQ0, hi);
    c->launches++;
    if ((rc = ex_allreduce(c, QtQ0, (int64_t)K * K, hi))) return rc;  // row-partitioned: global U^T U
    cudaEventRecord(c->ev_qready, hi);
  }
  int la_nb[2] = {0, 0}, la_y[2] = {0, 0};
  static const int nsub_env = getenv("PSVD_LA_NSUB") ? atoi(getenv("PSVD_LA_NSUB")) : 1;
  const int nsub = (int)std::max<int64_t>(1, std::min<int64_t>(nsub_env, M / 65536));
  // look-ahead sketch of batch j on the low-priority stream: Z = A_j Omega_j[K:], tiles Q^T Z, Z^T Z
  auto la = [&](int j) -> int {
    const bool hq = j > 0 || Kc > 0;
    const int lq = j > 0 ? l : Kc;
    const double* Qp = j > 0 ? Qb[(j - 1) & 1] : U_in;
    const int64_t ldqp = j > 0 ? ldq : ldu;
    const int nj = (hq ? K : 0) + B[j];
    if (hq) cudaStreamWaitEvent(lo, c->ev_qready, 0);
    if (j >= 2) cudaStreamWaitEvent(lo, c->ev_asm[j & 1], 0);  // tiles2[j&1] consumed by update j-2
    if (batch_ready && batch_ready[j]) cudaStreamWaitEvent(lo, (cudaEvent_t)batch_ready[j], 0);
    const int64_t rows_sub = (M + nsub - 1) / nsub / 32 * 32 + 32;
    Pass first;
    size_t part_off = 0;
    int nchunks_total = 0;
    mark("lo:la_begin", j, lo);
    for (int k = 0; k < nsub; ++k) {
      const int64_t r0 = (int64_t)k * rows_sub;
      if (r0 >= M) break;
      const int64_t mk = std::min(M, r0 + rows_sub) - r0;
      std::vector<Seg> segs;
      if (hq) segs.push_back(Seg{Qp + r0, ldqp, lq, 0});
      segs.push_back(Seg{A[j] + r0, lda[j], B[j], 0});
      Pass pa;
      int r = plan_pass(c, pa, mk, segs, hq ? lq : 0, B[j], l, Omega[j] + (hq ? K : 0), nj, false, true, hq,
                        hq ? lq : -1, -1, &c->partial2, &c->tiles2[j & 1], c->num_sms - 2, 0, true);
      if (r) return r;
      const size_t need_p = part_off + (size_t)pa.grid * SLOTS * 1024;
      if (k == 0) {
        if ((r = ensure(c, c->partial2, sizeof(double) * need_p * nsub))) return r;
        first = pa;
      }
      pa.p.partial = (double*)c->partial2.ptr + part_off;
      pa.p.Yout = Zt + r0;
      pa.p.ldy = ldq;
      c->path_count[pa.tma ? 0 : 3]++;
      // the split-ring kernel when the pass qualifies (group A = A_j under W, group B = Q for Q^T Z)
      if (pa.tma && nsub == 1 && try_fused_split(c, pa, {}, 1)) {
        launch_fused_split(pa.p, pa.maps3, pa.x, pa.fs, pa.grid, lo);
        first.map = pa.map;  // the split kernel's own slot map
      } else if (pa.tma)
        launch_pass_tma(pa.p, pa.maps, pa.x, pa.grid, lo);
      else
        launch_tall(pa.p, pa.grid, lo);
      c->launches++;
      if ((r = cuda_check(c, "look-ahead sketch"))) return r;
      part_off += (size_t)pa.grid * SLOTS * 1024;
      nchunks_total += pa.map.nchunks;
    }
    first.map.nchunks = nchunks_total;
    launch_tall_reduce((const double*)c->partial2.ptr, first.map, (double*)c->tiles2[j & 1].ptr, lo);
    c->launches++;
    la_nb[j & 1] = first.NB;
    la_y[j & 1] = first.p.np_pad;
    mark("lo:la_end", j, lo);
    cudaEventRecord(c->ev_aa[j & 1], lo);
    return cuda_check(c, "look-ahead reduce");
  };
  if ((rc = la(0))) return rc;
  for (int b = 0; b < nb; ++b) {
    const bool hq = b > 0 || Kc > 0;
    const int lq = b > 0 ? l : Kc, kq = hq ? K : 0, n = kq + B[b];
    const double* Qp = b > 0 ? Qb[(b - 1) & 1] : U_in;
    const int64_t ldqp = b > 0 ? ldq : ldu;
    const double* Wfp = b > 0 ? Wf[(b - 1) & 1] : WfI;
    const double* sgp = b > 0 ? sgn : ones;
    const double* sigp = b > 0 ? sigma_hist + (size_t)(b - 1) * K : sigma_in;
    const double* QtQ = b > 0 ? G2[(b - 1) & 1] : QtQ0;
    double* Qn = Qb[b & 1];
    double* G2c = G2[b & 1];
    mark("hi:update", b, hi);
    if (b > 0) {  // tall sign rule of U_{b-1} = Q Wf (linalg.py:161, 81-91): argmax pass, no write
      const int nch = qw_colmax_chunks(M, c->num_sms);
      if ((rc = ensure(c, c->colmax, sizeof(double) * (size_t)nch * K * 2))) return rc;
      launch_qw_colmax(Qp, ldqp, M, l, Wfp, K, nullptr, 0, c->ex_row_offset, (double*)c->colmax.ptr, c->num_sms, hi);
      c->launches++;
      if ((rc = exchange_sign(c, (const double*)c->colmax.ptr, nch, K, sgn, hi))) return rc;
    }
    mark("hi:sign_end", b, hi);
    cudaStreamWaitEvent(hi, c->ev_aa[b & 1], 0);
    // row-partitioned: the look-ahead tiles (Q^T Z, Z^T Z) summed over the ranks, on this stream (every
    // exchange of the run is issued on hi, in the same order on every rank)
    if ((rc = ex_allreduce(c, (double*)c->tiles2[b & 1].ptr, (int64_t)la_nb[b & 1] * la_nb[b & 1] * 1024, hi)))
      return rc;
    mark("hi:prep", b, hi);
    launch_rs_prep(sgp, Wfp, lq, K, sigp, ff, Omega[b], n, QtQ, (const double*)c->tiles2[b & 1].ptr, la_nb[b & 1], 0,
                   la_y[b & 1], l, hq, Etop, Cm, G1, hi);
    c->launches++;
    cudaEventRecord(c->ev_asm[b & 1], hi);
    if ((rc = svqb(c, G1, l, T1, sscr, hi))) return rc;
    mark("hi:svqb_end", b, hi);
    launch_rs_wb(Cm, lq, T1, l, hq, Wb, hi);
    c->launches++;
    if (batch_ready && batch_ready[b]) cudaStreamWaitEvent(hi, (cudaEvent_t)batch_ready[b], 0);
    // projection pass: Y1 = [Q | Z] Wb, Y1^T Y1, [Q | Z | A]^T Y1
    {
      std::vector<Seg> segs;
      if (hq) segs.push_back(Seg{Qp, ldqp, lq, 0});
      segs.push_back(Seg{Zt, ldq, l, 2});  // Z^T Y1 is not needed: no P^T Y rows for Z
      segs.push_back(Seg{A[b], lda[b], B[b], 0});
      const int wk = (hq ? lq : 0) + l;
      Pass pb;
      if ((rc = plan_pass(c, pb, M, segs, 0, wk, l, Wb, wk, false, true, true, -1, -1, nullptr, nullptr, 0, 0, true)))
        return rc;
      pb.p.Yout = Qn;
      pb.p.ldy = ldq;
      mark("hi:projB", b, hi);
      if ((rc = run_pass(c, pb, hi))) return rc;
      mark("hi:projB_end", b, hi);
      if (q == 0) {
        cudaEventRecord(c->ev_qready, hi);
        if (b + 1 < nb && (rc = la(b + 1))) return rc;
      }
      launch_rs_post((const double*)c->tiles.ptr, pb.NB, hq ? pb.p.seg[0].col0 : 0, pb.p.seg[hq ? 2 : 1].col0,
                     pb.p.np_pad, lq, B[b], l, Etop, K, hq, G2c, X, hi);
      c->launches++;
      if ((rc = ex_allreduce(c, G2c, (int64_t)l * l, hi)) || (rc = ex_allreduce(c, X, (int64_t)n * l, hi))) return rc;
    }
    launch_chol_inv(G2c, l, T2, hi);
    launch_small_gemm(X, n, 0, T2, l, q > 0 ? Zs : Bt, n, n, l, l, nullptr, hi);
    c->launches += 2;
    for (int it = 1; it <= q; ++it) {
      // power iteration (linalg.py:143-145): Qz = orth(C^T Q) by SVQB + CholeskyQR, next sketch P (D Qz)
      launch_small_gemm(Zs, n, 1, Zs, n, G1, l, l, n, l, nullptr, hi);
      c->launches++;
      if ((rc = svqb(c, G1, l, Tz, sscr, hi))) return rc;
      launch_small_gemm(Zs, n, 0, Tz, l, Z1, n, n, l, l, nullptr, hi);
      launch_small_gemm(Z1, n, 1, Z1, n, G1, l, l, n, l, nullptr, hi);
      launch_chol_inv(G1, l, Tz, hi);
      launch_small_gemm(Z1, n, 0, Tz, l, Qz, n, n, l, l, nullptr, hi);
      const int rows = (hq ? lq : 0) + B[b];
      launch_rs_w0(Etop, lq, K, Qz, n, B[b], l, hq, W0, hi);
      c->launches += 5;
      std::vector<Seg> segs;
      if (hq) segs.push_back(Seg{Qp, ldqp, lq, 0});
      segs.push_back(Seg{A[b], lda[b], B[b], 0});
      Pass pA;  // sketch pass: Y = [Q | A] (E Qz), Y^T Y (into Z's buffer: Z_b was consumed by the first projection)
      if ((rc = plan_pass(c, pA, M, segs, 0, rows, l, W0, rows, false, true, false))) return rc;
      pA.p.Yout = Zt;
      pA.p.ldy = ldq;
      if ((rc = run_pass(c, pA, hi))) return rc;
      launch_extract_sym((const double*)c->tiles.ptr, pA.NB, pA.p.np_pad, l, nullptr, G1, hi);
      c->launches++;
      if ((rc = ex_allreduce(c, G1, (int64_t)l * l, hi))) return rc;
      if ((rc = svqb(c, G1, l, T1, sscr, hi))) return rc;
      segs.push_back(Seg{Zt, ldq, l, 2});  // (no Z^T Y1 rows)
      Pass pB;  // projection pass: Y1 = Y T1 (not in place: slices), Y1^T Y1, [Q | A]^T Y1
      if ((rc = plan_pass(c, pB, M, segs, rows, l, l, T1, l, false, true, true, -1, -1, nullptr, nullptr, 0, 0, true)))
        return rc;
      pB.p.Yout = Qn;
      pB.p.ldy = ldq;
      if ((rc = run_pass(c, pB, hi))) return rc;
      if (it == q) {
        cudaEventRecord(c->ev_qready, hi);
        if (b + 1 < nb && (rc = la(b + 1))) return rc;
      }
      launch_rs_post((const double*)c->tiles.ptr, pB.NB, hq ? pB.p.seg[0].col0 : 0, pB.p.seg[hq ? 1 : 0].col0,
                     pB.p.np_pad, lq, B[b], l, Etop, K, hq, G2c, X, hi);
      if ((rc = ex_allreduce(c, G2c, (int64_t)l * l, hi)) || (rc = ex_allreduce(c, X, (int64_t)n * l, hi))) return rc;
      launch_chol_inv(G2c, l, T2, hi);
      launch_small_gemm(X, n, 0, T2, l, it < q ? Zs : Bt, n, n, l, l, nullptr, hi);
      c->launches += 3;
    }
    // small SVD of B = Q^T C through B^T = Bt (U_B = J); Wf = T2 J[:, :K]
    mark("hi:jacobi", b, hi);
    launch_jacobi_svd(Bt, n, l, S, J, (double*)c->jacws.ptr, c->d_status, hi);
    mark("hi:jacobi_end", b, hi);
    launch_small_gemm(T2, l, 0, J, l, Wf[b & 1], l, l, l, K, nullptr, hi);
    cudaMemcpyAsync(sigma_hist + (size_t)b * K, S, sizeof(double) * K, cudaMemcpyDeviceToDevice, hi);
    c->launches += 2;
    if ((rc = cuda_check(c, "randomized stream update"))) return rc;
  }
  {  // U = Q Wf with the sign rule, written once
    const double* Ql = Qb[(nb - 1) & 1];
    const int nch = qw_colmax_chunks(M, c->num_sms);
    if ((rc = ensure(c, c->colmax, sizeof(double) * (size_t)nch * K * 2))) return rc;
    launch_qw_colmax(Ql, ldq, M, l, Wf[(nb - 1) & 1], K, U_out, ldo, c->ex_row_offset, (double*)c->colmax.ptr,
                     c->num_sms, hi);
    if ((rc = exchange_sign(c, (const double*)c->colmax.ptr, nch, K, sgn, hi))) return rc;
    launch_scale_cols(U_out, ldo, M, K, sgn, hi);
    c->launches += 2;
  }
  cudaEventRecord(c->ev_join, lo);
  cudaStreamWaitEvent(user, c->ev_join, 0);
  cudaEventRecord(c->ev_join, hi);
  cudaStreamWaitEvent(user, c->ev_join, 0);
  if (trace) {
    mark("end", 0, user);
    cudaDeviceSynchronize();
    for (size_t i = 0; i < tl.size(); ++i)
      fprintf(stderr, "psvd_trace %-18s %9.3f ms\n", tl[i].c_str(), (double)(tbuf[i] - tbuf[0]) * 1e-6);
    cudaFree(tbuf);
  }
  return cuda_check(c, "rand_stream_run");
}

// 1 when psvd_rand_stream_run's passes plan for batches of up to Bmax columns (sketch width l,
// K modes, q power iterations) on M rows; 0: use psvd_rand_update per batch (its wide route).
int psvd_rand_stream_run_supported(psvd_ctx* c, int64_t M, int K, int l, int q, int Bmax, int* ok) {
  if (!c || !ok || M < 1 || K < 1 || l < K || Bmax < 1 || q < 0) return PSVD_EINVAL;
  *ok = 0;
  if (l > TMA_MAX_Y || !tma_available() || !qw_colmax_supported(l, K)) return PSVD_OK;
  const double* fake = reinterpret_cast<const double*>(uintptr_t(1) << 20);
  const int64_t ld = M + (M & 1);
  std::string saved = c->err;
  Pass p1, p2, p3, p4;
  bool fit = plan_pass(c, p1, M, {Seg{fake, ld, l, 0}, Seg{fake, ld, Bmax, 0}}, l, Bmax, l, fake, K + Bmax, false,
                       true, true, l, -1, &c->partial2, &c->tiles2[0], c->num_sms - 2, 0, true) == PSVD_OK &&
             p1.tma &&
             plan_pass(c, p2, M, {Seg{fake, ld, l, 0}, Seg{fake, ld, l, 0}, Seg{fake, ld, Bmax, 0}}, 0, 2 * l, l,
                       fake, 2 * l, false, true, true, -1, -1, nullptr, nullptr, 0, 0, true) == PSVD_OK;
  if (fit && q > 0)
    fit = plan_pass(c, p3, M, {Seg{fake, ld, l, 0}, Seg{fake, ld, Bmax, 0}}, 0, l + Bmax, l, fake, l + Bmax, false,
                    true, false) == PSVD_OK &&
          plan_pass(c, p4, M, {Seg{fake, ld, l, 0}, Seg{fake, ld, Bmax, 0}, Seg{fake, ld, l, 0}}, l + Bmax, l, l,
                    fake, l, false, true, true, -1, -1, nullptr, nullptr, 0, 0, true) == PSVD_OK;
  c->err = saved;
  *ok = fit ? 1 : 0;
  return PSVD_OK;
}

// vt (K x n, ld ldvt) of the last psvd_rand_update on this context (low_rank_svd's right factor,
// linalg.py:157-162): vt[k] = sign_k (B^T U_B[:, k])^T / S_k from the update's small matrices.
// Valid on the same stream right after that update.
int psvd_rand_last_vt(psvd_ctx* c, int n, int l, int K, double* Vt, int64_t ldvt, void* stream) {
  if (!c) return PSVD_EINVAL;
  if (!Vt || n < 1 || l < K || K < 1 || ldvt < K) return fail(c, PSVD_EINVAL, "bad rand_last_vt arguments");
  const size_t nl = (size_t)n * l, ll = (size_t)l * l;
  const size_t need = sizeof(double) * (6 * nl + 6 * ll + 2 * l + (size_t)l * K + K);
  if (c->rsmall.bytes < need) return fail(c, PSVD_EINVAL, "no randomized update of this shape to read");
  const double* base = (const double*)c->rsmall.ptr;
  const double* Bt = base + 5 * nl;
  const double* J = Bt + nl + 4 * ll;
  const double* S = J + 2 * ll;
  const double* sgn = S + 2 * l + (size_t)l * K;
  rand_vt_kernel<<<(unsigned)((n * K + 127) / 128), 128, 0, (cudaStream_t)stream>>>(Bt, n, l, J, S, sgn, K, Vt, ldvt);
  c->launches++;
  return cuda_check(c, "rand vt");
}

}  // extern "C"
