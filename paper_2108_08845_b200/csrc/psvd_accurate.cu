// Rank-robust factorizations of tall panels: the accurate route of the deterministic update and the
// any-rank qr_factor / svd_full (reference: np.linalg.qr / np.linalg.svd, Householder-based and
// backward stable at any conditioning, linalg.py:94-123; streaming.py:97-99).
//
// CholeskyQR (even shifted CholeskyQR3) assumes cond(A) < 1/eps; a numerically rank-deficient panel
// (a Burgers batch has ~30 significant directions out of 200) breaks it.  Instead:
//
//   range_basis:  an orthonormal basis Q of range(X) by Gram deflation.  Level l: G = X^T X
//                 (DMMA TN product, summed over ranks), eig(G) by the multi-CTA Jacobi, keep the
//                 directions with lambda > tau lambda_max (tau = 1e-10: their Gram eigenvectors give
//                 columns Y = X V Lambda^-1/2 with cond(Y) ~ 1 + eps / tau), orthogonalize Y against
//                 the basis so far (twice) and by CholeskyQR2, append, and project Y out of X (twice).
//                 Each level resolves another factor sqrt(tau) = 1e-5 of the spectrum; the residual
//                 ends at rounding level (||X_res||_F <= 4 eps sqrt(n) ||X||_F) after <= 4 levels.
//                 Every decision is taken from allreduced, bitwise-identical values: the ranks of a
//                 row-partitioned panel follow the same control flow.
//   hh_qr:        one-CTA Householder QR of a small m x n matrix (global-memory working copy),
//                 diag(R) >= 0 (qr_factor's convention), optional explicit Q (m x qcols).
//
// Then X = Q B with B = Q^T X (n x n), and:
//   qr_factor (psvd_qr_robust):  B = Q_B R (Householder), Q <- Q Q_B  (svd_full then runs its Jacobi
//               on this R);
//   the accurate update:  the one-sided Jacobi of B^T (relative accuracy): B^T J = U~ S, so
//               X = (Q J) S U~^T; the reference's sign rule is taken on U_R = R U~ S^-1 with R the
//               Householder R of B (= the R of qr(X), diag >= 0).
#include <algorithm>
#include <cfloat>
#include <cmath>
#include <cstring>
#include <vector>

#include "psvd_ctx.cuh"

using namespace psvd;
using namespace psvd_internal;

namespace {

constexpr int HH_THREADS = 1024;
constexpr double RB_TAU = 1e-10;   // kept eigenvalue ratio per deflation level
constexpr int RB_MAX_LEVELS = 6;

// One CTA: Householder QR of A (m x n; trans = 1 reads A^T of an n x m A, ld lda).  W: m x n
// workspace (ld m), tau: min(m, n).  R (min(m, n) x n, ld ldr) upper with diag >= 0; Q (m x qcols,
// ld ldq, qcols in [min(m, n), m]) explicit, or null.
__global__ void __launch_bounds__(HH_THREADS) hh_qr_kernel(const double* __restrict__ A, int64_t lda, int trans,
                                                           int m, int n, double* __restrict__ W,
                                                           double* __restrict__ tau, double* __restrict__ R, int ldr,
                                                           double* __restrict__ Q, int ldq, int qcols) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarp = blockDim.x >> 5;
  for (int64_t idx = tid; idx < (int64_t)m * n; idx += blockDim.x) {
    const int i = (int)(idx % m), j = (int)(idx / m);
    W[idx] = trans ? A[(int64_t)i * lda + j] : A[(int64_t)j * lda + i];
  }
  __syncthreads();
  const int p = min(m, n);
  __shared__ double s_tau;
  for (int k = 0; k < p; ++k) {
    double* wk = W + (size_t)k * m;
    if (warp == 0) {  // reflector of W[k:m, k] (dlarfg)
      double ss = 0.0;
      for (int i = k + 1 + lane; i < m; i += 32) ss = fma(wk[i], wk[i], ss);
      ss = warp_sum(ss);
      const double alpha = wk[k];
      double t = 0.0, beta = alpha, scal = 0.0;
      if (ss > 0.0) {
        beta = -copysign(sqrt(fma(alpha, alpha, ss)), alpha);
        t = (beta - alpha) / beta;
        scal = 1.0 / (alpha - beta);
      }
      __syncwarp();
      for (int i = k + 1 + lane; i < m; i += 32) wk[i] = ss > 0.0 ? wk[i] * scal : 0.0;
      if (lane == 0) {
        wk[k] = beta;
        tau[k] = t;
        s_tau = t;
      }
    }
    __syncthreads();
    const double t = s_tau;
    if (t != 0.0) {
      for (int j = k + 1 + warp; j < n; j += nwarp) {
        double* wj = W + (size_t)j * m;
        double w = 0.0;
        for (int i = k + 1 + lane; i < m; i += 32) w = fma(wk[i], wj[i], w);
        w = warp_sum(w) + wj[k];
        const double tw = t * w;
        if (lane == 0) wj[k] -= tw;
        for (int i = k + 1 + lane; i < m; i += 32) wj[i] = fma(-tw, wk[i], wj[i]);
      }
    }
    __syncthreads();
  }
  // R with diag >= 0: row k times sign(R_kk)
  for (int64_t idx = tid; idx < (int64_t)p * n; idx += blockDim.x) {
    const int i = (int)(idx % p), j = (int)(idx / p);
    const double s = W[(size_t)i * m + i] < 0.0 ? -1.0 : 1.0;
    R[(size_t)j * ldr + i] = i <= j ? s * W[(size_t)j * m + i] : 0.0;
  }
  if (Q == nullptr) return;
  // Q = H_0 ... H_{p-1} [I; 0] by backward accumulation (columns j >= k change at step k)
  for (int64_t idx = tid; idx < (int64_t)m * qcols; idx += blockDim.x) {
    const int i = (int)(idx % m), j = (int)(idx / m);
    Q[(size_t)j * ldq + i] = i == j ? 1.0 : 0.0;
  }
  __syncthreads();
  for (int k = p - 1; k >= 0; --k) {
    const double t = tau[k];
    const double* vk = W + (size_t)k * m;  // v = [1; W[k+1:m, k]]
    if (t != 0.0) {
      for (int j = k + warp; j < qcols; j += nwarp) {
        double* qj = Q + (size_t)j * ldq;
        double w = 0.0;
        for (int i = k + 1 + lane; i < m; i += 32) w = fma(vk[i], qj[i], w);
        w = warp_sum(w) + qj[k];
        const double tw = t * w;
        if (lane == 0) qj[k] -= tw;
        for (int i = k + 1 + lane; i < m; i += 32) qj[i] = fma(-tw, vk[i], qj[i]);
      }
    }
    __syncthreads();
  }
  for (int64_t idx = tid; idx < (int64_t)m * p; idx += blockDim.x) {
    const int i = (int)(idx % m), j = (int)(idx / m);
    if (W[(size_t)j * m + j] < 0.0) Q[(size_t)j * ldq + i] = -Q[(size_t)j * ldq + i];
  }
}

__global__ void trace_kernel(const double* __restrict__ G, int n, double* __restrict__ out) {
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int i = 0; i < n; ++i) t += G[(size_t)i * n + i];
    *out = t;
  }
}

// [I; -Z] (k + r) x k, column-major ld (k + r): the weights of Y - Q Z through one segmented NN product
__global__ void ident_negz_kernel(const double* __restrict__ Z, int r, int k, double* __restrict__ Wt) {
  const int ld = k + r;
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < ld * k; idx += gridDim.x * blockDim.x) {
    const int i = idx % ld, j = idx / ld;
    Wt[idx] = i < k ? (i == j ? 1.0 : 0.0) : -Z[(size_t)j * r + (i - k)];
  }
}

// deterministic pseudo-random candidates in [-1, 1) keyed by (global row, column): the orthonormal
// completion of a rank-deficient basis (same values on every rank for a given global row)
__global__ void candidates_kernel(double* __restrict__ Z, int64_t ldz, int64_t M, int k, int64_t row_offset,
                                  unsigned long long seed) {
  const int64_t total = M * (int64_t)k;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = idx % M, j = idx / M;
    unsigned long long x = seed ^ ((unsigned long long)(i + row_offset) * 0x9E3779B97F4A7C15ull) ^
                           ((unsigned long long)j * 0xC2B2AE3D27D4EB4Full);
    x ^= x >> 30; x *= 0xBF58476D1CE4E5B9ull;
    x ^= x >> 27; x *= 0x94D049BB133111EBull;
    x ^= x >> 31;
    Z[j * ldz + i] = (double)(x >> 11) * (2.0 / 9007199254740992.0) - 1.0;
  }
}

__global__ void scale_cols_small_kernel(double* __restrict__ X, int ld, int m, int n, const double* __restrict__ s,
                                        int invert) {
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < m * n; idx += gridDim.x * blockDim.x) {
    const int i = idx % m, j = idx / m;
    const double f = s[j];
    X[(size_t)j * ld + i] = invert ? (f > 0.0 ? X[(size_t)j * ld + i] / f : 0.0) : X[(size_t)j * ld + i] * f;
  }
}

// sign rule of linalg.py:81-91 on the columns of U_R (r x K): the first entry of largest magnitude
// made positive; sgn[k] = +-1.  Rows of R whose pivot is below SIGN_ROW_TOL max|R_ii| are skipped: their
// entries carry errors up to eps |C|^2 / |R_ii| >= their size in ANY backward-stable R (Householder's
// included), so they cannot decide the reference's sign; the reference's own choice is set by the
// determined rows whenever it is reproducible at all.
constexpr double SIGN_ROW_TOL = 1e-8;
__global__ void small_colsign_kernel(const double* __restrict__ UR, int ld, int r, int K, const double* __restrict__ Rb,
                                     int ldr, double* __restrict__ sgn) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= K) return;
  double dmax = 0.0;
  for (int i = 0; i < r; ++i) dmax = fmax(dmax, fabs(Rb[(size_t)i * ldr + i]));
  double best = -1.0, v = 0.0;
  for (int i = 0; i < r; ++i) {
    if (!(fabs(Rb[(size_t)i * ldr + i]) >= SIGN_ROW_TOL * dmax)) continue;
    const double x = UR[(size_t)k * ld + i];
    if (fabs(x) > best) { best = fabs(x); v = x; }
  }
  sgn[k] = v < 0.0 ? -1.0 : 1.0;
}

}  // namespace

namespace psvd_internal {

void launch_hh_qr(const double* A, int64_t lda, int trans, int m, int n, double* ws, double* R, int ldr, double* Q,
                  int ldq, int qcols, cudaStream_t st) {
  hh_qr_kernel<<<1, HH_THREADS, 0, st>>>(A, lda, trans, m, n, ws, ws + (size_t)m * n, R, ldr, Q, ldq, qcols);
}
size_t hh_qr_workspace_doubles(int m, int n) { return (size_t)m * n + std::min(m, n) + 8; }

// The accurate factorization workspace: small matrices in accws, four tall M x n buffers in accq.
struct AccWs {
  double *G, *lam, *V, *Z, *Wt, *T, *scal, *trace;
  double *X, *X2, *Q, *Y2;  // tall M x n buffers (ld): residual (ping-pong), basis, temporary
  int64_t ld;
};

static int acc_workspace(psvd_ctx* c, int64_t M, int n, AccWs& w) {
  const size_t nn = (size_t)n * n;
  int rc = ensure(c, c->accws, sizeof(double) * (6 * nn + 4 * (size_t)n + 64));
  if (rc) return rc;
  const int64_t ld = M + (M & 1);
  if ((rc = ensure(c, c->accq, sizeof(double) * 4 * (size_t)ld * n))) return rc;
  double* s = (double*)c->accws.ptr;
  w.G = s;
  w.V = w.G + nn;
  w.Z = w.V + nn;
  w.Wt = w.Z + nn;       // (2n) x n
  w.T = w.Wt + 2 * nn;
  w.lam = w.T + nn;
  w.scal = w.lam + n;
  w.trace = w.scal + n;
  double* t = (double*)c->accq.ptr;
  w.ld = ld;
  w.X = t;
  w.X2 = t + (size_t)ld * n;
  w.Q = t + 2 * (size_t)ld * n;
  w.Y2 = t + 3 * (size_t)ld * n;
  return PSVD_OK;
}

// X^T Y (k x m, ld ldx) summed over ranks
static int tn(psvd_ctx* c, int64_t M, const double* X, int64_t ldx, int k, const double* Y, int64_t ldy, int m,
              double* out, cudaStream_t st) {
  int rc = ensure(c, c->partial, sizeof(double) * tgemm_tn_partial_doubles(M, k, m, c->num_sms));
  if (rc) return rc;
  const GemmSeg g{X, ldx, k};
  launch_tgemm_tn(M, &g, 1, Y, ldy, m, nullptr, out, k, (double*)c->partial.ptr, c->num_sms, st);
  c->launches += 2;
  if ((rc = cuda_check(c, "tn"))) return rc;
  return ex_allreduce(c, out, (int64_t)k * m, st);
}

// Y <- Y - B (B^T Y) twice (B: M x r orthonormal), through [Y | B] [I; -Z] into tmp; Y, tmp swapped
static int project_out(psvd_ctx* c, int64_t M, const double* B, int64_t ldb, int r, double*& Y, double*& tmp,
                       int64_t ld, int k, AccWs& w, cudaStream_t st) {
  if (r == 0 || k == 0) return PSVD_OK;
  for (int pass = 0; pass < 2; ++pass) {
    int rc = tn(c, M, B, ldb, r, Y, ld, k, w.Z, st);
    if (rc) return rc;
    ident_negz_kernel<<<std::max(1, std::min(1024, ((k + r) * k + 255) / 256)), 256, 0, st>>>(w.Z, r, k, w.Wt);
    const GemmSeg segs[2] = {{Y, ld, k}, {B, ldb, r}};
    launch_tgemm_nn(M, segs, 2, w.Wt, k + r, k, tmp, ld, st);
    c->launches += 2;
    std::swap(Y, tmp);
  }
  return cuda_check(c, "project out");
}

// CholeskyQR2 of Y (M x k, well conditioned): Y <- Y R^-1 twice
static int cqr2(psvd_ctx* c, int64_t M, double*& Y, double*& tmp, int64_t ld, int k, AccWs& w, cudaStream_t st) {
  for (int pass = 0; pass < 2; ++pass) {
    int rc = tn(c, M, Y, ld, k, Y, ld, k, w.G, st);
    if (rc) return rc;
    if ((rc = chol_any(c, w.G, k, w.T, nullptr, c->d_status, nullptr, st))) return rc;
    const GemmSeg g{Y, ld, k};
    launch_tgemm_nn(M, &g, 1, w.T, k, k, tmp, ld, st);
    c->launches++;
    std::swap(Y, tmp);
  }
  return cuda_check(c, "cqr2");
}

static int read_doubles(psvd_ctx* c, const double* d, double* h, int n, cudaStream_t st) {
  if (cudaMemcpyAsync(h, d, sizeof(double) * n, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
      cudaStreamSynchronize(st) != cudaSuccess)
    return cuda_check(c, "read back");
  return PSVD_OK;
}

// Orthonormal basis of range(X) into w.Q (columns [0, r)); X = w.X (M x n) is overwritten by the
// residual (ping-pong with w.X2).
int range_basis(psvd_ctx* c, int64_t M, int n, AccWs& w, int* r_out, cudaStream_t st) {
  int r = 0;
  double fro0 = 0.0;
  std::vector<double> lam(n), scal(n);
  double* X = w.X;
  double* Xt = w.X2;
  for (int level = 0; level < RB_MAX_LEVELS && r < n; ++level) {
    int rc = tn(c, M, X, w.ld, n, X, w.ld, n, w.G, st);
    if (rc) return rc;
    trace_kernel<<<1, 32, 0, st>>>(w.G, n, w.trace);
    c->launches++;
    double tr = 0.0;
    if ((rc = read_doubles(c, w.trace, &tr, 1, st))) return rc;
    if (!std::isfinite(tr)) return fail(c, PSVD_EINVAL, "panel contains non-finite entries");
    if (level == 0) fro0 = tr;
    if (tr <= 0.0 || tr <= 16.0 * DBL_EPSILON * DBL_EPSILON * n * fro0) break;  // rounding level
    if ((rc = jacobi_any(c, w.G, n, n, n, 0, w.lam, w.V, n, nullptr, 0, st))) return rc;
    if ((rc = read_doubles(c, w.lam, lam.data(), n, st))) return rc;
    int k = 0;
    while (k < n - r && lam[k] > RB_TAU * lam[0] && lam[k] > 0.0) ++k;
    if (k == 0) break;
    for (int i = 0; i < k; ++i) scal[i] = 1.0 / std::sqrt(lam[i]);
    cudaMemcpyAsync(w.scal, scal.data(), sizeof(double) * k, cudaMemcpyHostToDevice, st);
    // the new block is built in place in the basis (columns r .. r + k); its two-pass projections and
    // CholeskyQR2 ping-pong with Y2 an even number of times, so it ends where it started
    double* Qk = w.Q + (size_t)r * w.ld;
    double* Y = Qk;
    double* Yt = w.Y2;
    const GemmSeg gx{X, w.ld, n};
    launch_tgemm_nn(M, &gx, 1, w.V, n, k, Y, w.ld, st);  // Y = X V_k Lambda_k^-1/2
    launch_scale_cols(Y, w.ld, M, k, w.scal, st);
    c->launches += 2;
    if ((rc = project_out(c, M, w.Q, w.ld, r, Y, Yt, w.ld, k, w, st))) return rc;
    if ((rc = cqr2(c, M, Y, Yt, w.ld, k, w, st))) return rc;
    if (Y != Qk) return fail(c, PSVD_ECUDA, "range basis: block not back in place");
    if ((rc = project_out(c, M, Qk, w.ld, k, X, Xt, w.ld, n, w, st))) return rc;  // X <- X - Qk (Qk^T X)
    r += k;
  }
  *r_out = r;
  return cuda_check(c, "range basis");
}

// Complete w.Q (M x r orthonormal) to M x ncols: pseudo-random candidates, projected out twice, CholeskyQR2.
int complete_basis(psvd_ctx* c, int64_t M, int r, int ncols, AccWs& w, cudaStream_t st) {
  const int k = ncols - r;
  if (k <= 0) return PSVD_OK;
  double* Qk = w.Q + (size_t)r * w.ld;  // built in place (an even number of ping-pongs with Y2)
  double* Y = Qk;
  double* tmp = w.Y2;
  candidates_kernel<<<(unsigned)std::min<int64_t>(4096, (M * k + 255) / 256), 256, 0, st>>>(
      Y, w.ld, M, k, c->ex_row_offset, 0x5eed5eedULL + (unsigned long long)r);
  c->launches++;
  int rc;
  if ((rc = project_out(c, M, w.Q, w.ld, r, Y, tmp, w.ld, k, w, st))) return rc;
  if ((rc = cqr2(c, M, Y, tmp, w.ld, k, w, st))) return rc;
  if ((rc = project_out(c, M, w.Q, w.ld, r, Y, tmp, w.ld, k, w, st))) return rc;
  if ((rc = cqr2(c, M, Y, tmp, w.ld, k, w, st))) return rc;
  if (Y != Qk) return fail(c, PSVD_ECUDA, "complete basis: block not back in place");
  return cuda_check(c, "complete basis");
}

}  // namespace psvd_internal

extern "C" {

// Any-rank tall QR (M >= n): Q (M x n, ld ldq) orthonormal, R (n x n, ld n) upper with diag >= 0,
// A = Q R to rounding (qr_factor, linalg.py:94-104; Householder semantics for rank-deficient input:
// numerically null directions get tiny rows of R and an orthonormal completion in Q).
int psvd_qr_robust(psvd_ctx* c, int64_t M, int n, const double* A, int64_t lda, double* Q, int64_t ldq, double* R,
                   void* stream) {
  if (!c) return PSVD_EINVAL;
  cudaStream_t st = (cudaStream_t)stream;
  int rc;
  // a row-partitioned rank (exchange hooks set) may hold fewer rows than columns
  if (n < 1 || M < 1 || (!ex_active(c) && M < n))
    return fail(c, PSVD_EINVAL, "qr needs M >= n >= 1 (M=%lld n=%d)", (long long)M, n);
  if ((rc = check_mat(c, "A", A, lda, M, n)) || (rc = check_mat(c, "Q", Q, ldq, M, n))) return rc;
  if (!R) return fail(c, PSVD_EINVAL, "R is null");
  AccWs w;
  if ((rc = acc_workspace(c, M, n, w))) return rc;
  if ((rc = ensure(c, c->dense, sizeof(double) * (hh_qr_workspace_doubles(n, n) + (size_t)n * n)))) return rc;
  cudaMemcpy2DAsync(w.X, w.ld * sizeof(double), A, lda * sizeof(double), M * sizeof(double), n,
                    cudaMemcpyDeviceToDevice, st);
  int r = 0;
  if ((rc = range_basis(c, M, n, w, &r, st))) return rc;
  if ((rc = complete_basis(c, M, r, n, w, st))) return rc;
  // B = Q^T A (n x n); B = Q_B R; Q <- Q Q_B
  if ((rc = tn(c, M, w.Q, w.ld, n, A, lda, n, w.G, st))) return rc;
  double* hw = (double*)c->dense.ptr;
  double* QB = hw + hh_qr_workspace_doubles(n, n);
  launch_hh_qr(w.G, n, 0, n, n, hw, R, n, QB, n, n, st);
  const GemmSeg gq{w.Q, w.ld, n};
  launch_tgemm_nn(M, &gq, 1, QB, n, n, Q, ldq, st);
  c->launches += 2;
  return cuda_check(c, "qr robust");
}

// The accurate route of one deterministic update (streaming.py:97-116 at any conditioning): the
// same result as psvd_stream_update, computed from an explicit panel C = [ff U S | A] through the
// rank-robust basis (range_basis), the Jacobi SVD of B = Q^T C and the sign rule on the Householder R
// of B.  U_out = Q J[:, :K] diag(sign) (orthonormal by construction).  Synchronizes the host (the
// deflation levels size their products from device values).  Runs the exchange hooks when set, so a
// row-partitioned panel gets the same factorization on every rank.
int psvd_stream_update_accurate(psvd_ctx* c, int64_t M, const double* U, int64_t ldu, const double* sigma, double ff,
                                int Kc, const double* A, int64_t lda, int B, int K, int rescue, double* U_out,
                                int64_t ldo, double* sigma_out, void* stream) {
  if (!c) return PSVD_EINVAL;
  cudaStream_t st = (cudaStream_t)stream;
  const int n = Kc + B;
  int rc;
  if (M < 1 || B < 1 || Kc < 0 || K < 1 || K > n) return fail(c, PSVD_EINVAL, "bad accurate update shape");
  if ((rc = check_mat(c, "U", U, ldu, M, Kc)) || (rc = check_mat(c, "A", A, lda, M, B)) ||
      (rc = check_mat(c, "U_out", U_out, ldo, M, K)))
    return rc;
  AccWs w;
  if ((rc = acc_workspace(c, M, n, w))) return rc;
  const size_t nn = (size_t)n * n;
  if ((rc = ensure(c, c->dense, sizeof(double) * (hh_qr_workspace_doubles(n, n) + 4 * nn + 4 * (size_t)n + 8))))
    return rc;
  double* hw = (double*)c->dense.ptr;
  double* Bt = hw + hh_qr_workspace_doubles(n, n);  // n x r
  double* J = Bt + nn;                               // r x r
  double* Ut = J + nn;                               // n x r
  double* UR = Ut + nn;                              // r x K
  double* S = UR + nn;                               // r
  double* sgn = S + n;                               // K
  if ((rc = make_dvec(c, sigma, ff, Kc, n, st))) return rc;
  const double* d = (const double*)c->dvec.ptr;
  // explicit panel [U diag(d) | A]
  if (Kc > 0) {
    cudaMemcpy2DAsync(w.X, w.ld * sizeof(double), U, ldu * sizeof(double), M * sizeof(double), Kc,
                      cudaMemcpyDeviceToDevice, st);
    launch_scale_cols(w.X, w.ld, M, Kc, d, st);
    c->launches++;
  }
  cudaMemcpy2DAsync(w.X + (size_t)Kc * w.ld, w.ld * sizeof(double), A, lda * sizeof(double), M * sizeof(double), B,
                    cudaMemcpyDeviceToDevice, st);
  int r = 0;
  if ((rc = range_basis(c, M, n, w, &r, st))) return rc;
  if (r < K) {  // fewer numerically independent directions than modes: complete with zero singular values
    if ((rc = complete_basis(c, M, r, K, w, st))) return rc;
  }
  const int rr = std::max(r, K);
  // B^T = C^T Q = diag(d) [U | A]^T Q  (n x rr)
  if ((rc = ensure(c, c->partial, sizeof(double) * tgemm_tn_partial_doubles(M, n, rr, c->num_sms)))) return rc;
  std::vector<GemmSeg> gp;
  if (Kc > 0) gp.push_back(GemmSeg{U, ldu, Kc});
  gp.push_back(GemmSeg{A, lda, B});
  launch_tgemm_tn(M, gp.data(), (int)gp.size(), w.Q, w.ld, rr, d, Bt, n, (double*)c->partial.ptr, c->num_sms, st);
  c->launches += 2;
  if ((rc = ex_allreduce(c, Bt, (int64_t)n * rr, st))) return rc;
  // Jacobi on B^T (n x rr): B^T J = Ut S  ->  C = (Q J) S Ut^T
  if ((rc = jacobi_any(c, Bt, n, n, rr, 0, S, J, rr, Ut, n, st))) return rc;
  // sign rule on U_R = R Ut[:, :K] S^-1, R = the Householder R of B (rr x n, diag >= 0)
  double* Rb = w.G;  // rr x n, ld rr
  launch_hh_qr(Bt, n, 1, rr, n, hw, Rb, rr, nullptr, 0, 0, st);
  launch_small_gemm(Rb, rr, 0, Ut, n, UR, rr, rr, n, K, nullptr, st);
  small_colsign_kernel<<<(K + 127) / 128, 128, 0, st>>>(UR, rr, std::min(rr, n), K, Rb, rr, sgn);
  // (the 1/S scaling does not change the argmax)
  scale_cols_small_kernel<<<std::max(1, std::min(1024, (rr * K + 255) / 256)), 256, 0, st>>>(J, rr, rr, K, sgn, 0);
  c->launches += 4;
  // U_out = Q J[:, :K] diag(sign); sigma_out = S[:K]
  const GemmSeg gq{w.Q, w.ld, rr};
  launch_tgemm_nn(M, &gq, 1, J, rr, K, U_out, ldo, st);
  c->launches++;
  cudaMemcpyAsync(sigma_out, S, sizeof(double) * K, cudaMemcpyDeviceToDevice, st);
  if (rescue) {
    if ((rc = ensure(c, c->utu, sizeof(double) * (size_t)K * K))) return rc;
    if ((rc = tn(c, M, U_out, ldo, K, U_out, ldo, K, (double*)c->utu.ptr, st))) return rc;
    if ((rc = psvd_drift_rescue(c, M, U_out, ldo, K, (const double*)c->utu.ptr, sigma_out, c->drift_tol, stream)))
      return rc;
  }
  return cuda_check(c, "accurate update");
}

}  // extern "C"
