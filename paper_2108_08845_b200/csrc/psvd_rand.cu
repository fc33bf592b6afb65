// Small kernels of the randomized update (reference linalg.py:126-162 composed
// per batch): one-sided Jacobi SVD of the projected core, tiny
// dense products, and the tall sign rule (linalg.py:161, 81-91).
#include <cfloat>
#include <cstdio>
#include <algorithm>
#include <cstdlib>

#include "psvd_small.cuh"

namespace psvd {

// ---------------------------------------------------------------- small dense GEMM
// C (m x k2) = op(A) (m x k1) * B (k1 x k2), col-major; op(A) = A (lda rows) or A^T.
// One thread per output entry, fixed summation order (deterministic).
__global__ void small_gemm_kernel(const double* __restrict__ A, int lda, int transA, const double* __restrict__ B,
                                  int ldb, double* __restrict__ C, int ldc, int m, int k1, int k2,
                                  const double* __restrict__ rowscale) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (int64_t)m * k2) return;
  const int i = (int)(idx % m), j = (int)(idx / m);
  double s = 0.0;
  if (transA) {
    for (int k = 0; k < k1; ++k) s = fma(A[(size_t)i * lda + k], B[(size_t)j * ldb + k], s);
  } else {
    for (int k = 0; k < k1; ++k) s = fma(A[(size_t)k * lda + i], B[(size_t)j * ldb + k], s);
  }
  if (rowscale) s *= rowscale[i];
  C[(size_t)j * ldc + i] = s;
}

void launch_small_gemm(const double* A, int lda, int transA, const double* B, int ldb, double* C, int ldc, int m,
                       int k1, int k2, const double* rowscale, cudaStream_t st) {
  const int64_t tot = (int64_t)m * k2;
  small_gemm_kernel<<<(unsigned)((tot + 127) / 128), 128, 0, st>>>(A, lda, transA, B, ldb, C, ldc, m, k1, k2,
                                                                    rowscale);
}

// ---------------------------------------------------------------- one-sided Jacobi SVD
// Z (n x l, col-major ld n) = V S J^T.  Outputs S (l, descending) and J (l x l,
// col-major, columns in the order of S): for Z = B^T (B = Q^T C) J is U_B of
// svd(B).  Parallel round-robin ordering, one warp per column pair.
template <bool SMEM>
__global__ void __launch_bounds__(1024, 1)
jacobi_svd_kernel(const double* __restrict__ Zin, int n, int l, double* __restrict__ S, double* __restrict__ Jout,
                  double* __restrict__ ws, int* __restrict__ status, const int* __restrict__ gate) {
  if (gate != nullptr && *gate == 0) return;  // the CholeskyQR route was well conditioned
  extern __shared__ double sm[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
  const int le = l + (l & 1);  // even number of columns (a zero column pads odd l)
  double* Z = SMEM ? sm : ws;
  double* J = SMEM ? sm + (size_t)n * le : sm;
  double* red = J + (size_t)le * le;  // 32 doubles of block_sum scratch
  double* nrm = red + 32;
  int* order = reinterpret_cast<int*>(nrm + le);
  int* flag = order + le + 1;
  for (int64_t i = tid; i < (int64_t)n * le; i += blockDim.x) {
    const int c = (int)(i / n);
    Z[i] = c < l ? Zin[i] : 0.0;
  }
  for (int i = tid; i < le * le; i += blockDim.x) J[i] = (i % le == i / le) ? 1.0 : 0.0;
  // ||Z||_F^2 is invariant under the rotations: pairs whose inner product is below
  // eps^2 ||Z||_F^2 are at fp64 noise level relative to the matrix (rank-deficient
  // sketches) and are left alone, so the sweep converges instead of churning noise.
  double fro = 0.0;
  for (int64_t i = tid; i < (int64_t)n * le; i += blockDim.x) fro = fma(Z[i], Z[i], fro);
  fro = block_sum(fro, red);
  const double cfloor = DBL_EPSILON * DBL_EPSILON * fro;
  const double ctol = (double)max(n, 2) * DBL_EPSILON;  // orthogonality target (LAPACK-style m*eps)
  const int npair = le / 2;
  for (int sweep = 0; sweep < 40; ++sweep) {
    if (tid == 0) *flag = 0;
    __syncthreads();
    for (int r = 0; r < le - 1; ++r) {
      for (int k = warp; k < npair; k += nwarps) {
        int p, q;
        if (k == 0) {
          p = le - 1;
          q = r;
        } else {
          p = (r + k) % (le - 1);
          q = (r - k + le - 1) % (le - 1);
        }
        if (p > q) { const int t = p; p = q; q = t; }
        double* zp = Z + (size_t)p * n;
        double* zq = Z + (size_t)q * n;
        double a = 0.0, b = 0.0, c = 0.0;
        for (int i = lane; i < n; i += 32) {
          const double x = zp[i], y = zq[i];
          a = fma(x, x, a);
          b = fma(y, y, b);
          c = fma(x, y, c);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {  // three interleaved butterflies
          a += __shfl_xor_sync(0xffffffffu, a, o);
          b += __shfl_xor_sync(0xffffffffu, b, o);
          c += __shfl_xor_sync(0xffffffffu, c, o);
        }
        if (c != 0.0 && c * c > ctol * ctol * (a * b) && fabs(c) > cfloor) {
          // t = tan(theta) of the Hestenes rotation, smaller root: t = 2c sgn(b - a) / (|b - a| + sqrt((b - a)^2 + 4c^2))
          // (one sqrt, one division, one rsqrt per pair: the FP64 div/sqrt chains set the round latency)
          const double d = b - a;
          const double t = (d >= 0.0 ? 2.0 * c : -2.0 * c) / (fabs(d) + sqrt(fma(d, d, 4.0 * c * c)));
          const double cs = rsqrt(fma(t, t, 1.0)), sn = cs * t;
          for (int i = lane; i < n; i += 32) {
            const double x = zp[i], y = zq[i];
            zp[i] = cs * x - sn * y;
            zq[i] = sn * x + cs * y;
          }
          double* jp = J + (size_t)p * le;
          double* jq = J + (size_t)q * le;
          for (int i = lane; i < le; i += 32) {
            const double x = jp[i], y = jq[i];
            jp[i] = cs * x - sn * y;
            jq[i] = sn * x + cs * y;
          }
          if (lane == 0) *flag = 1;
        }
      }
      __syncthreads();
    }
    const int f = *flag;
    __syncthreads();
#ifdef PSVD_JACOBI_DEBUG
    if (tid == 0) printf("sweep %d flag %d clock %lld\n", sweep, f, (long long)clock64());
#endif
    if (f == 0) break;
    if (sweep == 39 && tid == 0) atomicOr(status, PSVD_ST_NOCONVERGE);
  }
  for (int c = warp; c < le; c += nwarps) {
    double s = 0.0;
    for (int i = lane; i < n; i += 32) s = fma(Z[(size_t)c * n + i], Z[(size_t)c * n + i], s);
    s = warp_sum(s);
    if (lane == 0) nrm[c] = sqrt(s);
  }
  __syncthreads();
  if (tid == 0) {  // stable sort by descending singular value
    for (int c = 0; c < le; ++c) order[c] = c;
    for (int a = 1; a < le; ++a) {
      const int oa = order[a];
      int b = a - 1;
      while (b >= 0 && nrm[order[b]] < nrm[oa]) { order[b + 1] = order[b]; --b; }
      order[b + 1] = oa;
    }
  }
  __syncthreads();
  for (int i = tid; i < l; i += blockDim.x) S[i] = nrm[order[i]];
  for (int i = tid; i < l * l; i += blockDim.x) {
    const int r = i % l, c = i / l;
    Jout[(size_t)c * l + r] = J[(size_t)order[c] * le + r];
  }
}

size_t jacobi_workspace_doubles(int n, int l) { return (size_t)n * (l + 1); }

// SVQB weights from the Jacobi eigen-decomposition of an l x l SPD Gram (S = eigenvalues,
// descending; T = eigenvectors): T[:, k] *= 1 / sqrt(S_k), or 0 for directions with
// sqrt(S_k) <= tol * sqrt(S_0) (numerically null, dropped).
__global__ void svqb_scale_kernel(double* __restrict__ T, const double* __restrict__ S, int l, double tol,
                                  const int* __restrict__ gate, int* __restrict__ status) {
  if (gate != nullptr && *gate == 0) return;
  const int k = blockIdx.x;
  const double s0 = sqrt(fmax(S[0], 0.0)), sk = sqrt(fmax(S[k], 0.0));
  const double inv = (sk > 0.0 && sk > tol * s0) ? 1.0 / sk : 0.0;
  // a direction this small is dropped or only roughly resolved by the Gram's eigenpairs: the result is a
  // valid randomized SVD, but no longer the reference's to 1e-10 (its Householder qr keeps the direction)
  if (status != nullptr && threadIdx.x == 0 && !(sk > 3.0 * tol * s0)) atomicOr(status, PSVD_ST_SKETCHCOND);
  for (int i = threadIdx.x; i < l; i += blockDim.x) T[(size_t)k * l + i] *= inv;
}

void launch_svqb_scale(double* T, const double* S, int l, double tol, cudaStream_t st, const int* gate, int* status) {
  svqb_scale_kernel<<<l, 32, 0, st>>>(T, S, l, tol, gate, status);
}

void launch_jacobi_svd(const double* Z, int n, int l, double* S, double* J, double* ws, int* status, cudaStream_t st,
                       const int* gate) {
  const int le = l + (l & 1);
  const size_t small = (size_t)le * le + 32 + le + le + 8;
  const size_t limit = 227 * 1024 / sizeof(double);
  if ((size_t)n * le + small <= limit) {
    const size_t smem = ((size_t)n * le + small) * sizeof(double);
    cudaFuncSetAttribute(jacobi_svd_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    // one warp per column pair (fewer idle warps at the round barriers for small l)
    const int thr = std::min(1024, std::max(64, 32 * (le / 2)));
    jacobi_svd_kernel<true><<<1, thr, smem, st>>>(Z, n, l, S, J, ws, status, gate);
  } else {
    const size_t smem = small * sizeof(double);
    cudaFuncSetAttribute(jacobi_svd_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    jacobi_svd_kernel<false><<<1, 1024, smem, st>>>(Z, n, l, S, J, ws, status, gate);
  }
}

// ---------------------------------------------------------------- Cholesky refinement
// T = R^{-1} for R = chol(G) (upper, G = R^T R, l <= 128).  Used for the second
// orthonormalization pass of a sketch whose Gram is already ~I (CholeskyQR2's
// refinement step); columns of a numerically null direction (pivot <= tiny)
// are zeroed, matching the first (SVQB) pass which dropped them.
__global__ void __launch_bounds__(1024, 1) chol_inv_kernel(const double* __restrict__ G, int l, double* __restrict__ T,
                                                           int* __restrict__ illcond, int* __restrict__ status,
                                                           double* __restrict__ Rout) {
  extern __shared__ double sm[];
  double* R = sm;          // l x l col-major, upper used
  double* X = R + l * l;   // inverse
  const int tid = threadIdx.x, nthr = blockDim.x;
  for (int idx = tid; idx < l * l; idx += nthr) R[idx] = G[idx];
  __syncthreads();
  double dmax = 0.0;
  bool finite = true;
  for (int i = 0; i < l; ++i) {  // the diagonal from the shared copy (same scan order)
    const double g = R[(size_t)i * l + i];
    finite = finite && isfinite(g);
    dmax = fmax(dmax, g);
  }
  // a non-finite snapshot entry reaches every sketch column (Gaussian Omega): its Gram diagonal
  if (!finite && status != nullptr && threadIdx.x == 0) atomicOr(status, PSVD_ST_NONFINITE);
  const double tiny = 64.0 * DBL_EPSILON * dmax;
  const int lane = tid & 31, warp = tid >> 5, nwarp = nthr >> 5;
  // right-looking Cholesky on the upper triangle: R[k][j] for j >= k (column j of R at R + j l)
  for (int k = 0; k < l; ++k) {
    const double piv = R[(size_t)k * l + k];
    const bool ok = piv > tiny;
    const double rk = ok ? sqrt(piv) : 0.0;
    __syncthreads();
    for (int j = k + tid; j < l; j += nthr) R[(size_t)j * l + k] = ok ? (j == k ? rk : R[(size_t)j * l + k] / rk) : 0.0;
    __syncthreads();
    // trailing update: warp per column j, lanes over rows i in (k, j]
    for (int j = k + 1 + warp; j < l; j += nwarp) {
      const double rkj = R[(size_t)j * l + k];
      for (int i = k + 1 + lane; i <= j; i += 32) R[(size_t)j * l + i] -= R[(size_t)i * l + k] * rkj;
    }
    __syncthreads();
  }
  // X = R^{-1} (upper), warp per column j: column-oriented back substitution, the right-hand
  // side b (= e_j) held by the lanes (row i in lane i % 32, slot i / 32); zero rows for zero pivots
  constexpr int SLOTS_MAX = (CHOL_NMAX + 31) / 32;
  for (int j = warp; j < l; j += nwarp) {
    double b[SLOTS_MAX];
#pragma unroll
    for (int t = 0; t < SLOTS_MAX; ++t) b[t] = (t * 32 + lane == j) ? 1.0 : 0.0;
#pragma unroll
    for (int t = SLOTS_MAX - 1; t >= 0; --t) {
      if (t * 32 > j) continue;
      for (int r = 31; r >= 0; --r) {
        const int q = t * 32 + r;
        if (q > j) continue;
        const double d = R[(size_t)q * l + q];
        const double xq = d != 0.0 ? __shfl_sync(0xffffffffu, b[t], r) / d : 0.0;
        if (lane == r) b[t] = xq;
#pragma unroll
        for (int u = 0; u <= t; ++u) {
          const int i = u * 32 + lane;
          if (i < q) b[u] -= R[(size_t)q * l + i] * xq;
        }
      }
    }
#pragma unroll
    for (int t = 0; t < SLOTS_MAX; ++t) {
      const int i = t * 32 + lane;
      if (i < l) X[(size_t)j * l + i] = i <= j ? b[t] : 0.0;
    }
  }
  __syncthreads();
  for (int idx = tid; idx < l * l; idx += nthr) T[idx] = X[idx];
  if (Rout != nullptr)
    for (int idx = tid; idx < l * l; idx += nthr) Rout[idx] = (idx % l <= idx / l) ? R[idx] : 0.0;
  if (illcond != nullptr && tid == 0) {
    // CholeskyQR2 keeps O(eps) orthogonality for cond(Y) < ~1e7: flag anything beyond
    // cond(Y) ~ max R_ii / min R_ii > 1e6, or a dropped pivot, for the SVQB route
    double rmax = 0.0, rmin = DBL_MAX;
    for (int i = 0; i < l; ++i) {
      const double d = R[(size_t)i * l + i];
      rmax = fmax(rmax, d);
      rmin = fmin(rmin, d);
    }
    *illcond = !(rmin > 0.0 && rmax <= 1e6 * rmin);
  }
}

// The same factorization for l <= 32 on one warp (lane j owns column j of R and of R^-1; row-major
// shared copies with a 33-double stride): same operations in the same order as chol_inv_kernel,
// without its 3 CTA barriers per column and single-thread columns of the inverse.
__global__ void __launch_bounds__(32, 1) chol_inv_warp_kernel(const double* __restrict__ G, int l,
                                                               double* __restrict__ T, int* __restrict__ illcond,
                                                               int* __restrict__ status, double* __restrict__ Rout) {
  __shared__ double R[32 * 33];
  __shared__ double X[32 * 33];
  const int lane = threadIdx.x;
  const bool mine = lane < l;
  double dmax = 0.0;
  bool finite = true;
  for (int i = 0; i < l; ++i) {  // identical scan order to chol_inv_kernel's
    const double g = G[(size_t)i * l + i];
    finite = finite && isfinite(g);
    dmax = fmax(dmax, g);
  }
  if (!finite && status != nullptr && lane == 0) atomicOr(status, PSVD_ST_NONFINITE);
  const double tiny = 64.0 * DBL_EPSILON * dmax;
  if (mine)
    for (int i = 0; i < l; ++i) R[i * 33 + lane] = G[(size_t)lane * l + i];  // R[i][j] = G(i, j)
  __syncwarp();
  for (int k = 0; k < l; ++k) {
    const double piv = R[k * 33 + k];
    const bool ok = piv > tiny;
    const double rk = ok ? sqrt(piv) : 0.0;
    __syncwarp();
    if (mine && lane >= k) R[k * 33 + lane] = ok ? (lane == k ? rk : R[k * 33 + lane] / rk) : 0.0;
    __syncwarp();
    if (mine) {
      const double rkj = R[k * 33 + lane];
      for (int i = k + 1; i <= lane; ++i) R[i * 33 + lane] -= R[k * 33 + i] * rkj;
    }
    __syncwarp();
  }
  if (mine) {
    const int j = lane;
    for (int i = l - 1; i >= 0; --i) {
      double v = (i == j) ? 1.0 : 0.0;
      for (int q = i + 1; q <= j; ++q) v -= R[i * 33 + q] * X[q * 33 + j];
      const double d = R[i * 33 + i];
      X[i * 33 + j] = (i <= j && d != 0.0) ? v / d : 0.0;
    }
    for (int i = 0; i < l; ++i) T[(size_t)j * l + i] = X[i * 33 + j];
    if (Rout != nullptr)
      for (int i = 0; i < l; ++i) Rout[(size_t)j * l + i] = i <= j ? R[i * 33 + j] : 0.0;
  }
  if (illcond != nullptr && lane == 0) {
    double rmax = 0.0, rmin = DBL_MAX;
    for (int i = 0; i < l; ++i) {
      const double d = R[i * 33 + i];
      rmax = fmax(rmax, d);
      rmin = fmin(rmin, d);
    }
    *illcond = !(rmin > 0.0 && rmax <= 1e6 * rmin);
  }
}

void launch_chol_inv(const double* G, int l, double* T, cudaStream_t st, int* illcond, int* status, double* Rout) {
  static const bool no_warp = getenv("PSVD_NO_WARP_CHOL") != nullptr;
  if (l <= 32 && !no_warp) {
    chol_inv_warp_kernel<<<1, 32, 0, st>>>(G, l, T, illcond, status, Rout);
    return;
  }
  const size_t smem = 2 * (size_t)l * l * sizeof(double);
  cudaFuncSetAttribute(chol_inv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  chol_inv_kernel<<<1, 1024, smem, st>>>(G, l, T, illcond, status, Rout);
}

// G += shift I with shift = 11 (M n + n (n + 1)) u tr(G): the shifted CholeskyQR of Fukaya et al.
// (an R that exists for any cond(A) < 1/u; two unshifted CholeskyQR passes then restore orthogonality)
__global__ void chol_shift_kernel(double* __restrict__ G, int n, double mfac) {
  __shared__ double tr;
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int i = 0; i < n; ++i) t += G[(size_t)i * n + i];
    tr = t;
  }
  __syncthreads();
  const double sh = 11.0 * mfac * DBL_EPSILON * 0.5 * tr;
  for (int i = threadIdx.x; i < n; i += blockDim.x) G[(size_t)i * n + i] += sh;
}

void launch_chol_shift(double* G, int n, int64_t M, cudaStream_t st) {
  const double mfac = (double)M * n + (double)n * (n + 1);
  chol_shift_kernel<<<1, 128, 0, st>>>(G, n, mfac);
}

// ---------------------------------------------------------------- tall sign rule
// colmax: [nchunks][K][2] = (signed value at max |u|, global row) per chunk in row
// order; the first chunk wins ties (lowest row, numpy argmax).  One CTA per column: each
// thread scans a strided subset of the chunks in increasing order, then a tree reduction
// that prefers the larger |value| and, on ties, the lower chunk index.
constexpr int CM_THREADS = 256;

__device__ void colmax_best(const double* __restrict__ colmax, int nchunks, int K, int k, double& val, double& row) {
  __shared__ double sa[CM_THREADS], sv[CM_THREADS], sr[CM_THREADS];
  __shared__ int sc[CM_THREADS];
  double best = -1.0, v = 0.0, r = -1.0;
  int bc = 0x7fffffff;
  for (int c = threadIdx.x; c < nchunks; c += CM_THREADS) {
    const double x = colmax[((size_t)c * K + k) * 2];
    if (fabs(x) > best) {
      best = fabs(x);
      v = x;
      r = colmax[((size_t)c * K + k) * 2 + 1];
      bc = c;
    }
  }
  sa[threadIdx.x] = best; sv[threadIdx.x] = v; sr[threadIdx.x] = r; sc[threadIdx.x] = bc;
  __syncthreads();
  for (int o = CM_THREADS / 2; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o) {
      const int j = threadIdx.x + o;
      if (sa[j] > sa[threadIdx.x] || (sa[j] == sa[threadIdx.x] && sc[j] < sc[threadIdx.x])) {
        sa[threadIdx.x] = sa[j]; sv[threadIdx.x] = sv[j]; sr[threadIdx.x] = sr[j]; sc[threadIdx.x] = sc[j];
      }
    }
    __syncthreads();
  }
  val = sv[0];
  row = sr[0];
}

__global__ void colmax_sign_kernel(const double* __restrict__ colmax, int nchunks, int K, double* __restrict__ sign) {
  double v, r;
  colmax_best(colmax, nchunks, K, blockIdx.x, v, r);
  if (threadIdx.x == 0) sign[blockIdx.x] = v < 0.0 ? -1.0 : 1.0;  // applied with scale_cols (multiplies by +-1)
}

// one (value, row) pair per column from the per-chunk pairs (first chunk wins ties)
__global__ void colmax_reduce_kernel(const double* __restrict__ colmax, int nchunks, int K, double* __restrict__ out) {
  double v, r;
  colmax_best(colmax, nchunks, K, blockIdx.x, v, r);
  if (threadIdx.x == 0) {
    out[(size_t)blockIdx.x * 2] = v;
    out[(size_t)blockIdx.x * 2 + 1] = r;
  }
}

void launch_colmax_reduce(const double* colmax, int nchunks, int K, double* out, cudaStream_t st) {
  colmax_reduce_kernel<<<K, CM_THREADS, 0, st>>>(colmax, nchunks, K, out);
}

void launch_colmax_sign(const double* colmax, int nchunks, int K, double* sign, cudaStream_t st) {
  colmax_sign_kernel<<<K, CM_THREADS, 0, st>>>(colmax, nchunks, K, sign);
}

__global__ void scale_cols_kernel(double* __restrict__ U, int64_t ld, int64_t M, int K, const double* __restrict__ s) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int k = blockIdx.y;
  if (i >= M || k >= K) return;
  const double f = s[k];
  if (f != 1.0) U[(size_t)k * ld + i] *= f;
}

void launch_scale_cols(double* U, int64_t ld, int64_t M, int K, const double* s, cudaStream_t st) {
  dim3 g((unsigned)((M + 255) / 256), (unsigned)K);
  scale_cols_kernel<<<g, 256, 0, st>>>(U, ld, M, K, s);
}

__global__ void scale_rows_kernel(const double* __restrict__ X, int ldx, int m, int k, const double* __restrict__ d,
                                  double* __restrict__ Y, int ldy) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (int64_t)m * k) return;
  const int i = (int)(idx % m), j = (int)(idx / m);
  Y[(size_t)j * ldy + i] = d[i] * X[(size_t)j * ldx + i];
}

void launch_scale_rows(const double* X, int ldx, int m, int k, const double* d, double* Y, int ldy, cudaStream_t st) {
  const int64_t tot = (int64_t)m * k;
  scale_rows_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(X, ldx, m, k, d, Y, ldy);
}

// ================================================================ pipelined randomized stream glue
// The pipelined stream (psvd_rand_stream_run) keeps the state of update b-1 as a sketch basis
// Q = Y1_{b-1} (M x lq, the once-orthonormalized sketch), weights Wf (lq x K), sigma (K) and the
// column signs s of the sign rule, U_{b-1} = Q Wf diag(s).  The panel of update b,
// [ff U S | A] = [Q | A] E with E = blockdiag(Wf diag(s ff sigma), I) ((lq + B) x (K + B)),
// is never formed: every product with it goes through E (reference: linalg.py:126-162 composed
// per batch, streaming.py:97-98).
namespace {
__device__ __forceinline__ double tile_at(const double* __restrict__ tiles, int NB, int gi, int gj) {
  return tiles[((size_t)(gi >> 5) * NB + (gj >> 5)) * 1024 + (gi & 31) * 32 + (gj & 31)];
}
__device__ __forceinline__ double tile_sym(const double* __restrict__ tiles, int NB, int gi, int gj) {
  return gi <= gj ? tile_at(tiles, NB, gi, gj) : tile_at(tiles, NB, gj, gi);
}
}  // namespace

// Etop = Wf diag(s ff sigma) (lq x K); C = Etop Omega[0:K, :] (lq x l);
// G1 = Y^T Y for Y = Q C + Z:  C^T QtQ C + C^T QtZ + QtZ^T C + ZtZ, where QtZ / ZtZ come from the
// look-ahead pass tiles (Q at panel columns [q_c0, q_c0 + lq), Z = its Y block at y_c0).
// have_q == 0 (first batch, no state): G1 = ZtZ.  One CTA.
__global__ void rs_prep_kernel(const double* __restrict__ sgn, const double* __restrict__ Wf, int lq, int K,
                               const double* __restrict__ sigma, double ff, const double* __restrict__ Om, int ldom,
                               const double* __restrict__ QtQ, const double* __restrict__ tiles, int NB, int q_c0,
                               int y_c0, int l, int have_q, double* __restrict__ Etop, double* __restrict__ C,
                               double* __restrict__ G1) {
  extern __shared__ double sm[];
  const int tid = threadIdx.x, nt = blockDim.x;
  if (!have_q) {
    for (int i = tid; i < l * l; i += nt) {
      const int r = i % l, cc = i / l;
      G1[i] = tile_sym(tiles, NB, y_c0 + r, y_c0 + cc);
    }
    return;
  }
  double* E = sm;              // lq x K
  double* Cs = E + lq * K;     // lq x l
  double* QZ = Cs + lq * l;    // lq x l
  double* H = QZ + lq * l;     // lq x l: QtQ C + QtZ
  for (int i = tid; i < lq * K; i += nt) {
    const int k = i / lq;
    const double e = Wf[i] * (sgn[k] * (ff * sigma[k]));
    E[i] = e;
    Etop[i] = e;
  }
  for (int i = tid; i < lq * l; i += nt) {
    const int r = i % lq, cc = i / lq;
    QZ[i] = tile_at(tiles, NB, q_c0 + r, y_c0 + cc);
  }
  __syncthreads();
  for (int i = tid; i < lq * l; i += nt) {
    const int r = i % lq, cc = i / lq;
    double s = 0.0;
    for (int k = 0; k < K; ++k) s = fma(E[k * lq + r], Om[(size_t)cc * ldom + k], s);
    Cs[i] = s;
    C[i] = s;
  }
  __syncthreads();
  for (int i = tid; i < lq * l; i += nt) {
    const int r = i % lq, cc = i / lq;
    double s = QZ[i];
    for (int m = 0; m < lq; ++m) s = fma(QtQ[m * lq + r], Cs[cc * lq + m], s);
    H[i] = s;
  }
  __syncthreads();
  for (int i = tid; i < l * l; i += nt) {
    const int r = i % l, cc = i / l;
    if (r > cc) continue;
    double s = tile_sym(tiles, NB, y_c0 + r, y_c0 + cc);
    for (int m = 0; m < lq; ++m) s += Cs[r * lq + m] * H[cc * lq + m] + QZ[m + r * lq] * Cs[cc * lq + m];
    G1[cc * l + r] = s;
    G1[r * l + cc] = s;
  }
}

void launch_rs_prep(const double* sgn, const double* Wf, int lq, int K, const double* sigma, double ff,
                    const double* Om, int ldom, const double* QtQ, const double* tiles, int NB, int q_c0, int y_c0,
                    int l, int have_q, double* Etop, double* C, double* G1, cudaStream_t st) {
  const size_t smem = sizeof(double) * ((size_t)lq * K + 3 * (size_t)lq * l);
  rs_prep_kernel<<<1, 256, smem, st>>>(sgn, Wf, lq, K, sigma, ff, Om, ldom, QtQ, tiles, NB, q_c0, y_c0, l, have_q,
                                       Etop, C, G1);
}

// Wb ((lq + l) x l) = [C T1; T1] (the weights of Y1 = [Q | Z] Wb = (Q C + Z) T1); have_q == 0: Wb = T1.
__global__ void rs_wb_kernel(const double* __restrict__ C, int lq, const double* __restrict__ T1, int l, int have_q,
                             double* __restrict__ Wb) {
  const int rows = have_q ? lq + l : l;
  for (int i = threadIdx.x; i < rows * l; i += blockDim.x) {
    const int r = i % rows, cc = i / rows;
    double v;
    if (have_q && r < lq) {
      v = 0.0;
      for (int m = 0; m < l; ++m) v = fma(C[m * lq + r], T1[cc * l + m], v);
    } else {
      v = T1[cc * l + (have_q ? r - lq : r)];
    }
    Wb[i] = v;
  }
}

void launch_rs_wb(const double* C, int lq, const double* T1, int l, int have_q, double* Wb, cudaStream_t st) {
  rs_wb_kernel<<<1, 256, 0, st>>>(C, lq, T1, l, have_q, Wb);
}

// After a projection pass (Y1 at y_c0, Q at q_c0, A at a_c0):  G2 = Y1^T Y1 (l x l) and
// X = E^T [Q | A]^T Y1 (n x l, n = K + B with Q, else B): X[k] = sum_i Etop[i, k] (Q^T Y1)[i],
// X[K + r] = (A^T Y1)[r]  (= D P^T Y1 of the unpipelined update).
__global__ void rs_post_kernel(const double* __restrict__ tiles, int NB, int q_c0, int a_c0, int y_c0, int lq, int B,
                               int l, const double* __restrict__ Etop, int K, int have_q, double* __restrict__ G2,
                               double* __restrict__ X) {
  const int tid = blockIdx.x * blockDim.x + threadIdx.x, nt = gridDim.x * blockDim.x;
  for (int i = tid; i < l * l; i += nt) {
    const int r = i % l, cc = i / l;
    G2[i] = tile_sym(tiles, NB, y_c0 + r, y_c0 + cc);
  }
  const int kq = have_q ? K : 0, n = kq + B;
  for (int i = tid; i < n * l; i += nt) {
    const int r = i % n, cc = i / n;
    double v;
    if (r < kq) {
      v = 0.0;
      for (int m = 0; m < lq; ++m) v = fma(Etop[r * lq + m], tile_at(tiles, NB, q_c0 + m, y_c0 + cc), v);
    } else {
      v = tile_at(tiles, NB, a_c0 + (r - kq), y_c0 + cc);
    }
    X[i] = v;
  }
}

void launch_rs_post(const double* tiles, int NB, int q_c0, int a_c0, int y_c0, int lq, int B, int l,
                    const double* Etop, int K, int have_q, double* G2, double* X, cudaStream_t st) {
  const int n = (have_q ? K : 0) + B;
  const int tot = std::max(l * l, n * l);
  rs_post_kernel<<<(tot + 255) / 256, 256, 0, st>>>(tiles, NB, q_c0, a_c0, y_c0, lq, B, l, Etop, K, have_q, G2, X);
}

// Power-iteration sketch weights W0 = E Qz ((lq + B) x l): [Etop Qz[0:K]; Qz[K:]]; have_q == 0: W0 = Qz.
__global__ void rs_w0_kernel(const double* __restrict__ Etop, int lq, int K, const double* __restrict__ Qz, int n,
                             int B, int l, int have_q, double* __restrict__ W0) {
  const int rows = have_q ? lq + B : B, kq = have_q ? K : 0;
  const int tid = blockIdx.x * blockDim.x + threadIdx.x, nt = gridDim.x * blockDim.x;
  for (int i = tid; i < rows * l; i += nt) {
    const int r = i % rows, cc = i / rows;
    double v;
    if (have_q && r < lq) {
      v = 0.0;
      for (int k = 0; k < K; ++k) v = fma(Etop[k * lq + r], Qz[(size_t)cc * n + k], v);
    } else {
      v = Qz[(size_t)cc * n + kq + (r - (have_q ? lq : 0))];
    }
    W0[i] = v;
  }
}

void launch_rs_w0(const double* Etop, int lq, int K, const double* Qz, int n, int B, int l, int have_q, double* W0,
                  cudaStream_t st) {
  const int rows = have_q ? lq + B : B;
  rs_w0_kernel<<<(rows * l + 255) / 256, 256, 0, st>>>(Etop, lq, K, Qz, n, B, l, have_q, W0);
}

// identity (K x K) and ones (K): the weights / signs of a user-supplied initial state
__global__ void rs_ident_kernel(double* __restrict__ I, double* __restrict__ ones, int K) {
  for (int i = threadIdx.x; i < K * K; i += blockDim.x) I[i] = (i % K == i / K) ? 1.0 : 0.0;
  for (int i = threadIdx.x; i < K; i += blockDim.x) ones[i] = 1.0;
}

void launch_rs_ident(double* I, double* ones, int K, cudaStream_t st) { rs_ident_kernel<<<1, 256, 0, st>>>(I, ones, K); }


// ---------------------------------------------------------------- U = Q W with the column argmax
// Narrow recompose for the sign rule of the randomized path (linalg.py:161, 81-91): Q (M x l,
// l <= 32) times W (l x K, K <= 16), optionally written to U, and per CTA (a contiguous row
// range, so CTA order = row order) the (signed value at max |u|, global row) of every column,
// ties to the lowest row.  A plain bandwidth kernel: a handful of FMAs per loaded double, many
// CTAs per SM (the TMA pass's one-CTA-per-SM ring is latency-bound on panels this narrow).
constexpr int QW_THREADS = 256;
constexpr int QW_KMAX = 16;

template <int LM, int KM>
__global__ void __launch_bounds__(QW_THREADS, 2) qw_colmax_kernel(const double* __restrict__ Q, int64_t ldq, int64_t M,
                                                                  int l, const double* __restrict__ W, int K,
                                                                  double* __restrict__ U, int64_t ldu,
                                                                  int64_t rows_per_cta, int64_t row_offset,
                                                                  double* __restrict__ colmax) {
  __shared__ double sW[LM * KM];
  // per thread and column: |u| max in a register, (row << 1 | negative) of it in shared memory
  __shared__ long long srow[KM][QW_THREADS];
  __shared__ double rb[QW_THREADS / 32][KM];
  __shared__ long long rr[QW_THREADS / 32][KM];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int i = tid; i < LM * KM; i += QW_THREADS) {
    const int j = i / KM, k = i % KM;
    sW[i] = (j < l && k < K) ? W[(size_t)k * l + j] : 0.0;  // sW[j][k], zero padded
  }
#pragma unroll
  for (int k = 0; k < KM; ++k) srow[k][tid] = -1;
  __syncthreads();
  const int64_t r0 = (int64_t)blockIdx.x * rows_per_cta, r1 = min(M, r0 + rows_per_cta);
  double ba[KM];
#pragma unroll
  for (int k = 0; k < KM; ++k) ba[k] = -1.0;
  for (int64_t r = r0 + tid; r < r1; r += QW_THREADS) {
    double q[LM];
#pragma unroll
    for (int j = 0; j < LM; ++j) q[j] = j < l ? __ldg(Q + (size_t)j * ldq + r) : 0.0;  // l loads in flight
#pragma unroll
    for (int k = 0; k < KM; ++k) {
      double u = 0.0;
#pragma unroll
      for (int j = 0; j < LM; ++j) u = fma(q[j], sW[j * KM + k], u);
      if (k < K) {
        if (U != nullptr) U[(size_t)k * ldu + r] = u;
        if (fabs(u) > ba[k]) {
          ba[k] = fabs(u);
          srow[k][tid] = (r << 1) | (u < 0.0 ? 1 : 0);
        }
      }
    }
  }
  if (colmax == nullptr) return;
  // warp then block reduction, ties to the smaller row (numpy argmax: first occurrence)
#pragma unroll
  for (int k = 0; k < KM; ++k) {
    double a = ba[k];
    long long rw = srow[k][tid];
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      const double oa = __shfl_xor_sync(0xffffffffu, a, off);
      const long long orw = __shfl_xor_sync(0xffffffffu, rw, off);
      if (oa > a || (oa == a && orw >= 0 && (rw < 0 || (orw >> 1) < (rw >> 1)))) { a = oa; rw = orw; }
    }
    if (lane == 0) { rb[warp][k] = a; rr[warp][k] = rw; }
  }
  __syncthreads();
  if (tid < K) {
    double a = -1.0;
    long long rw = -1;
    for (int w = 0; w < QW_THREADS / 32; ++w) {
      const double oa = rb[w][tid];
      const long long orw = rr[w][tid];
      if (oa > a || (oa == a && orw >= 0 && (rw < 0 || (orw >> 1) < (rw >> 1)))) { a = oa; rw = orw; }
    }
    double* dst = colmax + ((size_t)blockIdx.x * K + tid) * 2;
    dst[0] = rw < 0 ? 0.0 : ((rw & 1) ? -a : a);
    dst[1] = rw < 0 ? -1.0 : (double)(rw >> 1) + (double)row_offset;
  }
}

// rows per CTA (multiple of 32) and the CTA count = number of argmax chunks
int64_t qw_colmax_rows(int64_t M, int num_sms) {
  const int64_t target = std::max<int64_t>(1, std::min<int64_t>((int64_t)num_sms * 4, (M + 255) / 256));
  return ((M + target - 1) / target + 31) / 32 * 32;
}
int qw_colmax_chunks(int64_t M, int num_sms) {
  const int64_t rows = qw_colmax_rows(M, num_sms);
  return (int)((M + rows - 1) / rows);
}

bool qw_colmax_supported(int l, int K) { return l >= 1 && l <= 32 && K >= 1 && K <= QW_KMAX; }

void launch_qw_colmax(const double* Q, int64_t ldq, int64_t M, int l, const double* W, int K, double* U, int64_t ldu,
                      int64_t row_offset, double* colmax, int num_sms, cudaStream_t st) {
  const int64_t rows = qw_colmax_rows(M, num_sms);
  const int grid = (int)((M + rows - 1) / rows);
#define QW_LAUNCH(LM_, KM_) \
  qw_colmax_kernel<LM_, KM_><<<grid, QW_THREADS, 0, st>>>(Q, ldq, M, l, W, K, U, ldu, rows, row_offset, colmax)
  if (l <= 16) {
    if (K <= 8) QW_LAUNCH(16, 8); else QW_LAUNCH(16, 16);
  } else if (l <= 24) {
    if (K <= 8) QW_LAUNCH(24, 8); else if (K <= 12) QW_LAUNCH(24, 12); else QW_LAUNCH(24, 16);
  } else {
    if (K <= 8) QW_LAUNCH(32, 8); else QW_LAUNCH(32, 16);
  }
#undef QW_LAUNCH
}

}  // namespace psvd
