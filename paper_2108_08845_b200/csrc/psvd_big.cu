// Dense factorizations of any width, with the matrix in global memory (L2 resident at these sizes).
// The one-CTA kernels of psvd_rand.cu / psvd_small.cu keep their operands in shared memory and stop at
// CHOL_NMAX = 112 / JACOBI_NMAX = 160 columns; these take the reference's shapes beyond that
// (qr_factor / svd_full of any width, linalg.py:94-123; parallel_qr of the K + B = 210-column streaming
// concatenation, dsvd.py:176-202, 238; the accurate R-factor route of the deterministic update,
// streaming.py:97-99).
//
//   chol_big:   G = R^T R, right-looking over 32-column panels: one CTA factors the 32 x 32 diagonal
//               block (lane-owned columns, as chol_inv_warp_kernel) and solves the block row; a grid
//               applies the rank-32 update to the trailing upper triangle.  Pivots below
//               64 eps max(diag G) give zero rows (numerically null directions, as chol_inv).  Then
//               T = R^-1 by column-oriented back substitution, one warp per column.
//   jacobi_big: one-sided (Hestenes) Jacobi SVD of X (m x n), cooperative kernel: the n columns are
//               paired by the round-robin (circle) schedule, one warp per pair per round, a grid
//               barrier between rounds; every pair recomputes its three inner products from the
//               current columns (relative accuracy, no squaring) and rotates X and the accumulated V.
//               A sweep with no rotation ends the iteration; the singular values are the column norms,
//               sorted descending (ties: lower column first).  Fixed pairing and fixed reduction
//               order: bitwise reproducible, so replicated factorizations agree across GPUs.
#include <cfloat>
#include <cooperative_groups.h>

#include "psvd_small.cuh"

namespace cg = cooperative_groups;

namespace psvd {

namespace {

constexpr int CB = 32;  // Cholesky panel width

// max diag(G) and finiteness of the diagonal (one CTA): stats[0] = dmax, stats[1] = 1 if finite
__global__ void chol_stats_kernel(const double* __restrict__ G, int n, double* __restrict__ A,
                                  double* __restrict__ stats, int* __restrict__ status) {
  __shared__ double red[32];
  double dmax = 0.0;
  int bad = 0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const double g = G[(size_t)i * n + i];
    bad |= !isfinite(g);
    dmax = fmax(dmax, g);
  }
  dmax = warp_max(dmax);
  bad = __any_sync(0xffffffffu, bad);
  __shared__ int sbad;
  if (threadIdx.x == 0) sbad = 0;
  __syncthreads();
  if ((threadIdx.x & 31) == 0) {
    red[threadIdx.x >> 5] = dmax;
    if (bad) atomicOr(&sbad, 1);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double m = 0.0;
    for (int w = 0; w < (int)(blockDim.x + 31) / 32; ++w) m = fmax(m, red[w]);
    stats[0] = m;
    stats[1] = sbad ? 0.0 : 1.0;
    if (sbad && status != nullptr) atomicOr(status, PSVD_ST_NONFINITE);
  }
  // working copy of the upper triangle (the lower one is never read)
  for (size_t idx = threadIdx.x; idx < (size_t)n * n; idx += blockDim.x) {
    const int i = (int)(idx % n), j = (int)(idx / n);
    A[idx] = i <= j ? G[idx] : 0.0;
  }
}

// Factor the diagonal block [k0, k0 + kb) and solve the block row R[k0:k1, k1:n] = R_kk^-T A[k0:k1, k1:n]
__global__ void __launch_bounds__(1024) chol_panel_kernel(double* __restrict__ A, int n, int k0,
                                                          const double* __restrict__ stats) {
  __shared__ double D[CB][CB + 1];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int kb = min(CB, n - k0);
  const double tiny = 64.0 * DBL_EPSILON * stats[0];
  for (int idx = threadIdx.x; idx < CB * CB; idx += blockDim.x) {
    const int i = idx % CB, j = idx / CB;
    D[i][j] = (i < kb && j < kb && i <= j) ? A[(size_t)(k0 + j) * n + k0 + i] : 0.0;
  }
  __syncthreads();
  if (warp == 0) {  // lane j owns column j (chol_inv_warp_kernel's order of operations)
    const bool mine = lane < kb;
    for (int k = 0; k < kb; ++k) {
      const double piv = D[k][k];
      const bool ok = piv > tiny;
      const double rk = ok ? sqrt(piv) : 0.0;
      __syncwarp();
      if (mine && lane >= k) D[k][lane] = ok ? (lane == k ? rk : D[k][lane] / rk) : 0.0;
      __syncwarp();
      if (mine) {
        const double rkj = D[k][lane];
        for (int i = k + 1; i <= lane; ++i) D[i][lane] -= D[k][i] * rkj;
      }
      __syncwarp();
    }
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < kb * kb; idx += blockDim.x) {
    const int i = idx % kb, j = idx / kb;
    if (i <= j) A[(size_t)(k0 + j) * n + k0 + i] = D[i][j];
  }
  // block row: warp per column j >= k1, lane i holds A[k0 + i, j]; forward substitution with D^T
  const int k1 = k0 + kb;
  for (int j = k1 + warp; j < n; j += 32) {
    double* col = A + (size_t)j * n + k0;
    double a = lane < kb ? col[lane] : 0.0;
    for (int p = 0; p < kb; ++p) {
      const double d = D[p][p];
      const double xp = d != 0.0 ? __shfl_sync(0xffffffffu, a, p) / d : 0.0;
      if (lane == p) a = xp;
      if (lane > p && lane < kb) a -= D[p][lane] * xp;
    }
    if (lane < kb) col[lane] = a;
  }
}

// Trailing update of the upper triangle: A[i][j] -= sum_p R[p][i] R[p][j], p in [k0, k1), k1 <= i <= j.
// One CTA per 32 x 32 output tile (ti <= tj), 256 threads x 4 outputs.
__global__ void __launch_bounds__(256) chol_update_kernel(double* __restrict__ A, int n, int k0, int kb, int nt) {
  __shared__ double Ri[CB][CB + 1], Rj[CB][CB + 1];
  // tile index -> (ti, tj), ti <= tj, over nt tiles per side
  int t = blockIdx.x, ti = 0;
  while (t >= nt - ti) { t -= nt - ti; ++ti; }
  const int tj = ti + t;
  const int k1 = k0 + kb;
  const int i0 = k1 + ti * CB, j0 = k1 + tj * CB;
  for (int idx = threadIdx.x; idx < CB * CB; idx += blockDim.x) {
    const int p = idx % CB, c = idx / CB;
    Ri[p][c] = (p < kb && i0 + c < n) ? A[(size_t)(i0 + c) * n + k0 + p] : 0.0;
    Rj[p][c] = (p < kb && j0 + c < n) ? A[(size_t)(j0 + c) * n + k0 + p] : 0.0;
  }
  __syncthreads();
  const int r = threadIdx.x % CB, c0 = threadIdx.x / CB;  // rows r, columns c0 + 8 q
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int c = c0 + 8 * q;
    const int i = i0 + r, j = j0 + c;
    if (i < n && j < n && i <= j) {
      double s = 0.0;
      for (int p = 0; p < kb; ++p) s = fma(Ri[p][r], Rj[p][c], s);
      A[(size_t)j * n + i] -= s;
    }
  }
}

// T = R^-1 (upper; zero rows for zero pivots), Rout = R with zeros below the diagonal.
// Warp per column j, the right-hand side in shared memory (8 warps x n doubles per CTA).
__global__ void __launch_bounds__(256) tri_inv_kernel(const double* __restrict__ A, int n, double* __restrict__ T,
                                                      double* __restrict__ Rout) {
  extern __shared__ double sb[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int j = blockIdx.x * 8 + warp;
  if (j >= n) return;
  double* b = sb + (size_t)warp * n;
  for (int i = lane; i <= j; i += 32) b[i] = i == j ? 1.0 : 0.0;
  double* out = T + (size_t)j * n;
  for (int q = j; q >= 0; --q) {
    __syncwarp();
    const double d = A[(size_t)q * n + q];
    const double xq = d != 0.0 ? b[q] / d : 0.0;
    if (lane == 0) out[q] = xq;
    const double* rq = A + (size_t)q * n;
    for (int i = lane; i < q; i += 32) b[i] -= rq[i] * xq;
  }
  for (int i = j + 1 + lane; i < n; i += 32) out[i] = 0.0;
  if (Rout != nullptr) {
    const double* aj = A + (size_t)j * n;
    for (int i = lane; i < n; i += 32) Rout[(size_t)j * n + i] = i <= j ? aj[i] : 0.0;
  }
}

__global__ void chol_flag_kernel(const double* __restrict__ A, int n, int* __restrict__ illcond) {
  if (threadIdx.x != 0) return;
  double rmax = 0.0, rmin = DBL_MAX;
  for (int i = 0; i < n; ++i) {
    const double d = A[(size_t)i * n + i];
    rmax = fmax(rmax, d);
    rmin = fmin(rmin, d);
  }
  *illcond = !(rmin > 0.0 && rmax <= 1e6 * rmin);  // chol_inv_kernel's CholeskyQR2 range check
}

// ------------------------------------------------------------------------------------------ Jacobi

constexpr int JB_WARPS = 8;
constexpr int JB_THREADS = JB_WARPS * 32;

// round-robin (circle method) pairing of np (even) players: round r, slot p -> (i, j), i < j
__device__ __forceinline__ void rr_pair(int r, int p, int np, int& i, int& j) {
  const int m = np - 1;
  int a, b;
  if (p == 0) {
    a = r;
    b = m;
  } else {
    a = (r + p) % m;
    b = (r - p + m) % m;
  }
  i = min(a, b);
  j = max(a, b);
}

struct JacobiArgs {
  double* X;   // m x n, ld m (working copy)
  double* V;   // n x n, ld n (accumulated rotations)
  int64_t m;
  int n;
  int max_sweeps;
  double tol;
  int* sweep_flags;  // max_sweeps ints, zeroed
  double* norms;     // n
  int* perm;         // n
  double* S;         // n, output (descending)
  double* Vout;      // n x n, ld ldv, output (columns permuted)
  int64_t ldv;
  double* Uout;      // optional m x n, ld ldu: X[:, perm] / S (0 for S == 0)
  int64_t ldu;
  int* status;
  int* sweeps_out;
  int presort;       // pair order by decreasing initial column norm
};

__global__ void __launch_bounds__(JB_THREADS) jacobi_big_kernel(JacobiArgs a) {
  cg::grid_group grid = cg::this_grid();
  const int lane = threadIdx.x & 31;
  const int gwarp = blockIdx.x * JB_WARPS + (threadIdx.x >> 5);
  const int nwarps = gridDim.x * JB_WARPS;
  const int n = a.n;
  const int64_t m = a.m;
  const int np = n + (n & 1);
  // V = I
  for (size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x; idx < (size_t)n * n;
       idx += (size_t)gridDim.x * blockDim.x)
    a.V[idx] = (idx % n == idx / n) ? 1.0 : 0.0;
  // pair order by decreasing initial column norm (de Rijk): on a matrix graded the other way (small columns
  // first, e.g. Burgers rows near x = 1, whose early snapshots are ~1e-80) the cyclic sweeps otherwise stall
  for (int j = gwarp; j < n; j += nwarps) {
    const double* xj = a.X + (size_t)j * m;
    double s = 0.0;
    for (int64_t k = lane; k < m; k += 32) s = fma(xj[k], xj[k], s);
    s = warp_sum(s);
    if (lane == 0) a.norms[j] = s;
  }
  grid.sync();
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
    const double sj = a.norms[j];
    int rank = 0;
    for (int i = 0; i < n; ++i) {
      const double si = a.norms[i];
      rank += (si > sj) || (si == sj && i < j);
    }
    a.perm[a.presort ? rank : j] = j;
  }
  grid.sync();
  __shared__ int rotated;
  int sweep = 0;
  bool converged = n < 2;
  for (; sweep < a.max_sweeps && !converged; ++sweep) {
    if (threadIdx.x == 0) rotated = 0;
    __syncthreads();
    for (int r = 0; r < np - 1; ++r) {
      for (int p = gwarp; p < np / 2; p += nwarps) {
        int i, j;
        rr_pair(r, p, np, i, j);
        if (j >= n) continue;
        i = a.perm[i];
        j = a.perm[j];
        double* xi = a.X + (size_t)i * m;
        double* xj = a.X + (size_t)j * m;
        double s_ii = 0.0, s_jj = 0.0, s_ij = 0.0;
        for (int64_t k = lane; k < m; k += 32) {
          const double u = xi[k], v = xj[k];
          s_ii = fma(u, u, s_ii);
          s_jj = fma(v, v, s_jj);
          s_ij = fma(u, v, s_ij);
        }
        s_ii = warp_sum(s_ii);
        s_jj = warp_sum(s_jj);
        s_ij = warp_sum(s_ij);
        if (s_ii == 0.0 || s_jj == 0.0) continue;
        if (!(fabs(s_ij) > a.tol * sqrt(s_ii) * sqrt(s_jj))) continue;
        // Rutishauser's rotation: zeta = (s_jj - s_ii) / (2 s_ij), t = sign(zeta) / (|zeta| + sqrt(1 + zeta^2))
        const double zeta = (s_jj - s_ii) / (2.0 * s_ij);
        const double t = copysign(1.0, zeta) / (fabs(zeta) + hypot(1.0, zeta));
        const double cs = 1.0 / hypot(1.0, t);
        const double sn = cs * t;
        for (int64_t k = lane; k < m; k += 32) {
          const double u = xi[k], v = xj[k];
          xi[k] = cs * u - sn * v;
          xj[k] = sn * u + cs * v;
        }
        double* vi = a.V + (size_t)i * n;
        double* vj = a.V + (size_t)j * n;
        for (int k = lane; k < n; k += 32) {
          const double u = vi[k], v = vj[k];
          vi[k] = cs * u - sn * v;
          vj[k] = sn * u + cs * v;
        }
        if (lane == 0) rotated = 1;
      }
      grid.sync();
    }
    __syncthreads();
    if (threadIdx.x == 0 && rotated) atomicOr(a.sweep_flags + sweep, 1);
    grid.sync();
    converged = *((volatile int*)(a.sweep_flags + sweep)) == 0;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    if (!converged && a.status != nullptr) atomicOr(a.status, PSVD_ST_NOCONVERGE);
    if (a.sweeps_out != nullptr) *a.sweeps_out = sweep;
  }
  // column norms (fixed order)
  for (int j = gwarp; j < n; j += nwarps) {
    const double* xj = a.X + (size_t)j * m;
    double s = 0.0;
    for (int64_t k = lane; k < m; k += 32) s = fma(xj[k], xj[k], s);
    s = warp_sum(s);
    if (lane == 0) a.norms[j] = sqrt(s);
  }
  grid.sync();
  // rank of every column: larger norm first, ties -> lower column first
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
    const double sj = a.norms[j];
    int rank = 0;
    for (int i = 0; i < n; ++i) {
      const double si = a.norms[i];
      rank += (si > sj) || (si == sj && i < j);
    }
    a.perm[rank] = j;
    a.S[rank] = sj;
  }
  grid.sync();
  for (size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x; idx < (size_t)n * n;
       idx += (size_t)gridDim.x * blockDim.x) {
    const int row = (int)(idx % n), c = (int)(idx / n);
    a.Vout[(size_t)c * a.ldv + row] = a.V[(size_t)a.perm[c] * n + row];
  }
  if (a.Uout != nullptr) {
    for (int c = gwarp; c < n; c += nwarps) {
      const double s = a.S[c];
      const double inv = s > 0.0 ? 1.0 / s : 0.0;
      const double* src = a.X + (size_t)a.perm[c] * m;
      double* dst = a.Uout + (size_t)c * a.ldu;
      for (int64_t k = lane; k < m; k += 32) dst[k] = src[k] * inv;
    }
  }
}

__global__ void pack_cols_kernel(const double* __restrict__ X, int64_t ldx, int64_t m, int n, double* __restrict__ Y,
                                 int transpose) {
  const size_t total = (size_t)m * n;
  for (size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total; idx += (size_t)gridDim.x * blockDim.x) {
    const int64_t i = (int64_t)(idx % m);
    const int64_t j = (int64_t)(idx / m);
    // transpose: Y (m x n) = X^T with X (n x m, ld ldx)
    Y[idx] = transpose ? X[i * ldx + j] : X[j * ldx + i];
  }
}

}  // namespace

size_t chol_big_workspace_doubles(int n) { return (size_t)n * n + 8; }

void launch_chol_big(const double* G, int n, double* T, int* illcond, int* status, double* Rout, double* ws,
                     cudaStream_t st) {
  double* A = ws;
  double* stats = ws + (size_t)n * n;
  chol_stats_kernel<<<1, 1024, 0, st>>>(G, n, A, stats, status);
  for (int k0 = 0; k0 < n; k0 += CB) {
    const int kb = n - k0 < CB ? n - k0 : CB;
    chol_panel_kernel<<<1, 1024, 0, st>>>(A, n, k0, stats);
    const int rest = n - k0 - kb;
    if (rest > 0) {
      const int nt = (rest + CB - 1) / CB;
      chol_update_kernel<<<nt * (nt + 1) / 2, 256, 0, st>>>(A, n, k0, kb, nt);
    }
  }
  const size_t smem = sizeof(double) * 8 * (size_t)n;
  cudaFuncSetAttribute(tri_inv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  tri_inv_kernel<<<(n + 7) / 8, 256, smem, st>>>(A, n, T, Rout);
  if (illcond != nullptr) chol_flag_kernel<<<1, 32, 0, st>>>(A, n, illcond);
}

int chol_big_launches(int n) { return 2 + ((n + CB - 1) / CB) * 2 + 1; }

size_t jacobi_big_workspace_doubles(int64_t m, int n) {
  return (size_t)m * n + (size_t)n * n + 2 * (size_t)n + 64 + 8;
}

int launch_jacobi_big(const double* X, int64_t ldx, int64_t m, int n, int transpose, double* S, double* V,
                      int64_t ldv, double* U, int64_t ldu, double* ws, int* status, int* sweeps_out, int num_sms,
                      cudaStream_t st) {
  // ws: Xw (m x n) | Vw (n x n) | norms (n) | perm (n ints, as doubles) | sweep flags (64 ints)
  double* Xw = ws;
  double* Vw = Xw + (size_t)m * n;
  double* norms = Vw + (size_t)n * n;
  int* perm = (int*)(norms + n);
  int* flags = (int*)(norms + 2 * (size_t)n);
  static const char* env_sweeps = getenv("PSVD_JACOBI_SWEEPS");  // diagnostics (at most 128: the flags' room)
  const int max_sweeps = env_sweeps ? std::max(1, std::min(128, atoi(env_sweeps))) : 100;
  const size_t total = (size_t)m * n;
  pack_cols_kernel<<<(unsigned)std::min<size_t>((total + 255) / 256, 4096), 256, 0, st>>>(X, ldx, m, n, Xw,
                                                                                          transpose);
  cudaMemsetAsync(flags, 0, sizeof(int) * max_sweeps, st);
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, jacobi_big_kernel, JB_THREADS, 0);
  const int want = std::max(1, ((n + 1) / 2 + JB_WARPS - 1) / JB_WARPS);
  const int grid = std::max(1, std::min(want, per_sm * num_sms));
  JacobiArgs a;
  a.X = Xw;
  a.V = Vw;
  a.m = m;
  a.n = n;
  a.max_sweeps = max_sweeps;
  a.tol = DBL_EPSILON * sqrt((double)m);
  a.sweep_flags = flags;
  a.norms = norms;
  a.perm = perm;
  a.S = S;
  a.Vout = V;
  a.ldv = ldv;
  a.Uout = U;
  a.ldu = ldu;
  a.status = status;
  a.sweeps_out = sweeps_out;
  static const char* env_presort = getenv("PSVD_JACOBI_PRESORT");  // diagnostics: 0 = the plain cyclic order
  a.presort = env_presort ? atoi(env_presort) != 0 : 1;
  void* args[] = {&a};
  return (int)cudaLaunchCooperativeKernel((const void*)jacobi_big_kernel, dim3(grid), dim3(JB_THREADS), args, 0, st);
}

}  // namespace psvd
