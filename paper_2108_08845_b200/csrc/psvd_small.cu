// Small-core kernels (one CTA each).  See psvd_small.cuh.
//
// The deterministic streaming update needs the top-K singular triplets of the
// (K+B) x (K+B) core.  We reach them through the Gram G = C^T C of the panel
// C = [ff U S | A] (G = R^T R for the reference's R, streaming.py:98-99):
//   1. Householder tridiagonalization of G (packed lower triangle in smem),
//   2. top-K eigenvalues by 33-point multisection of Sturm counts (one warp
//      per eigenvalue),
//   3. eigenvectors of T by the twisted (forward/backward LDL^T) factorization
//      at the index of minimal |gamma| (one thread per eigenvalue), re-
//      orthogonalized (MGS twice) inside clusters of close eigenvalues,
//   4. back-transformation through the Householder reflectors,
//   5. R = chol(G + delta I) and the reference's sign rule on U_R = R V S^-1
//      (linalg.py:81-91), giving W = V S^-1 diag(sign) for the recompose.
#include <cfloat>
#include "psvd_small.cuh"

namespace psvd {

__device__ __forceinline__ int pidx(int n, int r, int c) {  // r >= c, column-packed lower
  return c * n - (c * (c - 1)) / 2 + (r - c);
}

// ---------------------------------------------------------------- extraction

__global__ void extract_sym_kernel(const double* __restrict__ tiles, int NB, int c0, int n,
                                   const double* __restrict__ d, double* __restrict__ out) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (int64_t)n * n) return;
  const int i = (int)(idx % n), j = (int)(idx / n);
  int gi = c0 + i, gj = c0 + j;
  if (gi > gj) { const int t = gi; gi = gj; gj = t; }  // always read the upper element: exact symmetry
  const int I = gi >> 5, J = gj >> 5;
  double v = tiles[((size_t)I * NB + J) * 1024 + (gi & 31) * 32 + (gj & 31)];
  if (d != nullptr) v = d[i] * d[j] * v;
  out[idx] = v;
}

__global__ void extract_rect_kernel(const double* __restrict__ tiles, int NB, int r0, int nr, int c0, int nc,
                                    const double* __restrict__ d, double* __restrict__ out) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (int64_t)nr * nc) return;
  const int i = (int)(idx % nr), j = (int)(idx / nr);
  const int gi = r0 + i, gj = c0 + j;
  const int I = gi >> 5, J = gj >> 5;
  double v = tiles[((size_t)I * NB + J) * 1024 + (gi & 31) * 32 + (gj & 31)];
  if (d != nullptr) v = d[i] * v;
  out[idx] = v;
}

void launch_extract_sym(const double* tiles, int NB, int c0, int n, const double* d, double* out,
                        cudaStream_t st) {
  const int64_t tot = (int64_t)n * n;
  extract_sym_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(tiles, NB, c0, n, d, out);
}

// G (n x n, n = K + B) = [[d d^T .* (U^T U), d .* (U^T A)], [., A^T A]] from the tiles of the
// narrow [U | A] pass (first tile rows) and of the A^T A pass.
__global__ void assemble_gram_kernel(const double* __restrict__ tua, int nbua, const double* __restrict__ taa,
                                     int nbaa, int K, int B, const double* __restrict__ d, double* __restrict__ G) {
  const int n = K + B;
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (int64_t)n * n) return;
  int i = (int)(idx % n), j = (int)(idx / n);
  if (i > j) { const int t = i; i = j; j = t; }
  double v;
  if (i < K) {
    v = tua[((size_t)(i >> 5) * nbua + (j >> 5)) * 1024 + (i & 31) * 32 + (j & 31)] * d[i];
    if (j < K) v *= d[j];
  } else {
    const int a = i - K, b = j - K;
    v = taa[((size_t)(a >> 5) * nbaa + (b >> 5)) * 1024 + (a & 31) * 32 + (b & 31)];
  }
  G[idx] = v;
}

void launch_assemble_gram(const double* tua, int nbua, const double* taa, int nbaa, int K, int B, const double* d,
                          double* G, cudaStream_t st) {
  const int64_t tot = (int64_t)(K + B) * (K + B);
  assemble_gram_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(tua, nbua, taa, nbaa, K, B, d, G);
}

// Streaming Gram for batch b+1 from the fused recompose pass of batch b:
//   UU = Uhat^T Uhat (already normalized by the Rayleigh refinement, K x K),
//   UA(k, j) = scale_k * (A_{b+1}^T Y)(j, k) read from the tiles (block a0 + j/32, Y block yb),
//   and, when the drift rescue ran (*gate), U <- U T:  UU <- T^T UU T,  UA <- T^T UA.
//   G = [[d d^T .* UU, d .* UA], [., A^T A]].
__global__ void assemble_gram_fused_kernel(const double* __restrict__ tf, int nbf, int a0, int yb,
                                           const double* __restrict__ UU, const double* __restrict__ scale,
                                           const int* __restrict__ gate, const double* __restrict__ T,
                                           const double* __restrict__ taa, int nbaa, int K, int B,
                                           const double* __restrict__ d, double* __restrict__ G, double uu_w) {
  const int n = K + B;
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (int64_t)n * n) return;
  int i = (int)(idx % n), j = (int)(idx / n);
  if (i > j) { const int t = i; i = j; j = t; }
  const bool rot = gate != nullptr && *gate != 0;
  double v;
  if (j < K) {
    if (!rot) {
      v = UU[(size_t)j * K + i];
    } else {
      v = 0.0;
      for (int a = 0; a < K; ++a) {
        double s = 0.0;
        for (int b2 = 0; b2 < K; ++b2) s += UU[(size_t)b2 * K + a] * T[(size_t)j * K + b2];
        v += T[(size_t)i * K + a] * s;
      }
    }
    v *= d[i] * d[j] * uu_w;  // uu_w: 0 on all but the first rank when the local Grams are summed
  } else if (i < K) {
    const int col = j - K;
    auto ua = [&](int k) {
      return scale[k] * tf[((size_t)(a0 + (col >> 5)) * nbf + yb + (k >> 5)) * 1024 + (col & 31) * 32 + (k & 31)];
    };
    if (!rot) {
      v = ua(i);
    } else {
      v = 0.0;
      for (int k = 0; k < K; ++k) v += T[(size_t)i * K + k] * ua(k);
    }
    v *= d[i];
  } else {
    const int a = i - K, b = j - K;
    v = taa[((size_t)(a >> 5) * nbaa + (b >> 5)) * 1024 + (a & 31) * 32 + (b & 31)];
  }
  G[idx] = v;
}

void launch_assemble_gram_fused(const double* tf, int nbf, int a0, int yb, const double* UU, const double* scale,
                                const int* gate, const double* T, const double* taa, int nbaa, int K, int B,
                                const double* d, double* G, cudaStream_t st, double uu_w) {
  const int64_t tot = (int64_t)(K + B) * (K + B);
  assemble_gram_fused_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(tf, nbf, a0, yb, UU, scale, gate, T, taa,
                                                                             nbaa, K, B, d, G, uu_w);
}

void launch_extract_rect(const double* tiles, int NB, int r0, int nr, int c0, int nc, const double* d,
                         double* out, cudaStream_t st) {
  const int64_t tot = (int64_t)nr * nc;
  extract_rect_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(tiles, NB, r0, nr, c0, nc, d, out);
}

// ---------------------------------------------------------------- eigensolver

size_t eig_workspace_doubles(int n, int K) {
  return (size_t)n * (n + 1) / 2 + (size_t)n * K + 2 * (size_t)n * K + 64;
}

__device__ __forceinline__ double fix_pivot(double q, double pivmin) {
  return fabs(q) < pivmin ? (q < 0.0 ? -pivmin : pivmin) : q;
}

// deterministic pseudo-random start vector entry in (-1, 1)
__device__ __forceinline__ double prand(unsigned a, unsigned b) {
  unsigned h = a * 0x9E3779B1u ^ (b + 0x7F4A7C15u) * 0x85EBCA77u;
  h ^= h >> 15; h *= 0x2C1B3C6Du; h ^= h >> 12; h *= 0x297A2D39u; h ^= h >> 15;
  return ((double)h / 4294967296.0) * 2.0 - 1.0;
}

// FAST (n <= EIG_FAST_NMAX, 512 threads): phases B and G are column-oriented with
// lane-owned rows (row r lives in lane r % 32, slot r / 32, of every warp): the
// trailing update of column j-1 and the symmetric mat-vec of column j are one
// sweep where each element costs LDS + 2 FMA + STS + 2 FMA and the vectors
// v, w sit in registers; row sums are combined across warps in a fixed order.
template <bool SMEM, bool FAST>
__global__ void __launch_bounds__(FAST ? EIG_FAST_THREADS : SMALL_THREADS, 1)
eig_topk_kernel(const double* __restrict__ G, int n, int K, const double* __restrict__ dscale,
                double* __restrict__ W, double* __restrict__ sigma_out, double* __restrict__ ws,
                int* __restrict__ status, long long* __restrict__ timers, double rank_tol, int split,
                const int* __restrict__ gate) {
  if (gate != nullptr && *gate == 0) return;  // the subspace fast path already converged
  extern __shared__ double sm[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nthr = blockDim.x, nwarps = nthr >> 5;
  const unsigned full = 0xffffffffu;
  const size_t npk = (size_t)n * (n + 1) / 2;
  double* Lp = SMEM ? sm : ws;
  double* vec = SMEM ? sm + npk : sm;       // small vectors always in smem
  double* v = vec;
  double* p = v + n;
  double* dd = p + n;
  double* ee = dd + n;
  double* tau = ee + n;
  double* e2 = tau + n;
  double* lam = e2 + n;                     // K
  double* red = lam + K;                    // 64 scratch
  int* clus = reinterpret_cast<int*>(red + 64);  // K cluster leaders
  // FAST-only arrays (after clus): column starts, double-buffered v / w, row partials
  constexpr int NT = (EIG_FAST_NMAX + 31) / 32;
  const int npad = ((n + 31) / 32) * 32;
  double* fbase = red + 64 + K + 1;
  int* cs = reinterpret_cast<int*>(fbase);                 // n ints
  double* vsA = fbase + (n + 1) / 2 + 1;
  double* vsB = vsA + npad;
  double* wsv = vsB + npad;
  double* ydot = wsv + npad;
  double* psm = ydot + npad;
  double* ypart = psm + npad;                              // [nwarps][npad]
  double* Z = ws + npk;                     // n x K (col-major, ld n)
  double* Dp = Z + (size_t)n * K;           // K x n
  double* Dm = Dp + (size_t)n * K;          // K x n
  auto stamp = [&](int i) {
    if (timers != nullptr && tid == 0) timers[i] = clock64();
  };
  stamp(0);

  // ---- A: load the lower triangle
  for (int64_t idx = tid; idx < (int64_t)n * n; idx += nthr) {
    const int i = (int)(idx % n), j = (int)(idx / n);
    if (i >= j) Lp[pidx(n, i, j)] = G[idx];
  }
  __syncthreads();

  stamp(1);
  if constexpr (FAST) {
    // ---- B (fast): column-oriented Householder tridiagonalization, lane-owned rows
    for (int c = tid; c < n; c += nthr) cs[c] = pidx(n, c, c);
    for (int i = tid; i < npad; i += nthr) { vsA[i] = 0.0; vsB[i] = 0.0; wsv[i] = 0.0; ydot[i] = 0.0; psm[i] = 0.0; }
    __syncthreads();
    double vO[NT], wO[NT], vN[NT];
#pragma unroll
    for (int t = 0; t < NT; ++t) { vO[t] = 0.0; wO[t] = 0.0; vN[t] = 0.0; }
    double* vs_old = vsA;
    double* vs_new = vsB;
    long long sub[5] = {0, 0, 0, 0, 0}, tsub = 0;
    auto tick = [&](int i) {  // diagnostics only (timers != null): barrier-accurate sub-phase clocks
      if (timers == nullptr) return;
      __syncthreads();
      const long long now = clock64();
      if (i >= 0) sub[i] += now - tsub;
      tsub = now;
    };
    tick(-1);
    // Per column j, three barriers:
    //   (e+a) every thread: w_{j-1} = p + kc v_{j-1} (registers + smem);  the owner warp of
    //         column j applies step j-1's update to it and turns it into reflector v_j
    //   (c)   fused sweep over columns > j: update with (v_{j-1}, w_{j-1}), symv with v_j
    //   (d)   p = tau_j y, partials of p.v
    for (int j = 0; j + 2 < n; ++j) {
      double kc = 0.0;
      if (j > 0) {
        double ptv = lane < nwarps ? red[lane] : 0.0;
        ptv = warp_sum(ptv);
        kc = -0.5 * tau[j - 1] * ptv;
#pragma unroll
        for (int t = 0; t < NT; ++t) {
          const int r = lane + 32 * t;
          vO[t] = vN[t];
          wO[t] = (r < npad) ? fma(kc, vN[t], psm[r]) : 0.0;
        }
        for (int r = tid; r < npad; r += nthr) wsv[r] = fma(kc, vs_old[r], psm[r]);
      }
      if (warp == (j % nwarps)) {
        const double vj = vs_old[j];
        const double wj = fma(kc, vj, psm[j]);
        double part = 0.0, xa = 0.0;
        double xs[NT];
#pragma unroll
        for (int t = 0; t < NT; ++t) {
          const int r = lane + 32 * t;
          xs[t] = 0.0;
          if (32 * t + 31 < j) continue;
          if (r >= j && r < n) {
            const double x = Lp[cs[j] + (r - j)] - (vO[t] * wj + wO[t] * vj);
            xs[t] = x;
            if (r >= j + 2) part = fma(x, x, part);
            if (r == j + 1) xa = x;
            if (r == j) dd[j] = x;
          }
        }
        const double xn2 = warp_sum(part);
        const double alpha = __shfl_sync(full, xa, (j + 1) & 31);
        double tj = 0.0, beta = alpha, scl = 0.0;
        if (xn2 != 0.0) {
          beta = -copysign(sqrt(alpha * alpha + xn2), alpha);
          tj = (beta - alpha) / beta;
          scl = 1.0 / (alpha - beta);
        }
#pragma unroll
        for (int t = 0; t < NT; ++t) {
          const int r = lane + 32 * t;
          double vr = 0.0;
          if (tj != 0.0 && r >= j + 1 && r < n) vr = (r == j + 1) ? 1.0 : xs[t] * scl;
          if (r < npad) vs_new[r] = vr;
          if (r >= j && r < n) Lp[cs[j] + (r - j)] = (r >= j + 2 && tj != 0.0) ? vr : xs[t];
        }
        if (lane == 0) { ee[j] = beta; tau[j] = tj; }
      }
      __syncthreads();
      tick(0);
      const double tj = tau[j];
#pragma unroll
      for (int t = 0; t < NT; ++t) {
        const int r = lane + 32 * t;
        vN[t] = r < npad ? vs_new[r] : 0.0;
      }
      tick(1);
      // (c) fused sweep over columns c >= j+1: update with (v_old, w_old), symv with v_new
      double yp[NT];
#pragma unroll
      for (int t = 0; t < NT; ++t) yp[t] = 0.0;
      // two columns per iteration: independent dot chains / warp reductions overlap
      for (int c = j + 1 + ((warp - (j + 1)) % nwarps + nwarps) % nwarps; c < n; c += 2 * nwarps) {
        const int c1 = c + nwarps;
        const bool has1 = c1 < n;
        const int c1s = has1 ? c1 : c;
        const double wpc = wsv[c], vpc = vs_old[c], vnc = vs_new[c];
        const double wpc1 = wsv[c1s], vpc1 = vs_old[c1s], vnc1 = has1 ? vs_new[c1s] : 0.0;
        const int base = cs[c] - c, base1 = cs[c1s] - c1s;
        double dot = 0.0, dot1 = 0.0;
#pragma unroll
        for (int t = 0; t < NT; ++t) {
          if (32 * t + 31 < c) continue;  // warp-uniform: whole slot above the diagonal
          const int r = lane + 32 * t;
          // branch-free body: loads from a clamped address, predicated store, masked sums
          const bool in0 = r >= c && r < n;
          const int a0 = in0 ? base + r : base + c;
          const double x = Lp[a0] - (vO[t] * wpc + wO[t] * vpc);
          if (in0) Lp[a0] = x;
          yp[t] = fma(in0 ? x : 0.0, vnc, yp[t]);
          dot = fma(r > c && r < n ? x : 0.0, vN[t], dot);
          if (has1) {
            const bool in1 = r >= c1 && r < n;
            const int a1 = in1 ? base1 + r : base1 + c1s;
            const double x1 = Lp[a1] - (vO[t] * wpc1 + wO[t] * vpc1);
            if (in1) Lp[a1] = x1;
            yp[t] = fma(in1 ? x1 : 0.0, vnc1, yp[t]);
            dot1 = fma(r > c1 && r < n ? x1 : 0.0, vN[t], dot1);
          }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          dot += __shfl_xor_sync(full, dot, o);
          dot1 += __shfl_xor_sync(full, dot1, o);
        }
        if (lane == 0) {
          ydot[c] = dot;
          if (has1) ydot[c1] = dot1;
        }
      }
#pragma unroll
      for (int t = 0; t < NT; ++t) {
        const int r = lane + 32 * t;
        if (r < npad) ypart[(size_t)warp * npad + r] = yp[t];
      }
      __syncthreads();
      tick(2);
      // (d) p = tau * y (rows >= j+1), partials of p.v
      double pv = 0.0;
      for (int r = tid; r < npad; r += nthr) {
        double y = 0.0;
        if (r >= j + 1 && r < n) {
          for (int w = 0; w < nwarps; ++w) y += ypart[(size_t)w * npad + r];
          y += ydot[r];
        }
        const double pr = tj * y;
        psm[r] = pr;
        pv = fma(pr, vs_new[r], pv);
      }
      pv = warp_sum(pv);
      if (lane == 0) red[warp] = pv;
      double* tmp = vs_old;
      vs_old = vs_new;
      vs_new = tmp;
      __syncthreads();
      tick(3);
    }
    if (timers != nullptr && tid == 0)
      for (int i = 0; i < 5; ++i) timers[9 + i] = sub[i];
    // w of the last reflector, then the pending update of the trailing 2x2 block
    if (n >= 3) {
      double ptv = lane < nwarps ? red[lane] : 0.0;
      ptv = warp_sum(ptv);
      const double kc = -0.5 * tau[n - 3] * ptv;
      for (int r = tid; r < npad; r += nthr) wsv[r] = fma(kc, vs_old[r], psm[r]);
      __syncthreads();
      if (tid == 0) {
        for (int c = n - 2; c < n; ++c)
          for (int r = c; r < n; ++r) {
            const int a = cs[c] + (r - c);
            Lp[a] -= vs_old[r] * wsv[c] + wsv[r] * vs_old[c];
          }
      }
    }
    __syncthreads();
  } else {
  // ---- B: Householder tridiagonalization (lower, dsytd2-style)
  for (int j = 0; j + 2 < n; ++j) {
    const int m = n - j - 1;
    const int cj = pidx(n, j, j);
    double part = 0.0;
    for (int i = 1 + tid; i < m; i += nthr) {
      const double x = Lp[cj + 1 + i];
      part += x * x;
    }
    const double xn2 = block_sum(part, red);
    const double alpha = Lp[cj + 1];
    if (xn2 == 0.0) {
      if (tid == 0) { tau[j] = 0.0; ee[j] = alpha; dd[j] = Lp[cj]; }
      __syncthreads();
      continue;
    }
    const double beta = -copysign(sqrt(alpha * alpha + xn2), alpha);
    const double tj = (beta - alpha) / beta;
    const double scl = 1.0 / (alpha - beta);
    for (int i = tid; i < m; i += nthr) v[i] = (i == 0) ? 1.0 : Lp[cj + 1 + i] * scl;
    if (tid == 0) { tau[j] = tj; ee[j] = beta; dd[j] = Lp[cj]; }
    __syncthreads();
    for (int i = 1 + tid; i < m; i += nthr) Lp[cj + 1 + i] = v[i];
    // p = tau * A22 * v, four threads per row (fixed order -> deterministic)
    for (int base = 0; base < m; base += nthr / 4) {
      const int row = base + (tid >> 2), q4 = tid & 3;
      double s = 0.0;
      if (row < m) {
        const int gr = j + 1 + row;
        for (int k = q4; k < m; k += 4) {
          const int gk = j + 1 + k;
          const double a = (k <= row) ? Lp[pidx(n, gr, gk)] : Lp[pidx(n, gk, gr)];
          s = fma(a, v[k], s);
        }
      }
      s += __shfl_xor_sync(full, s, 1);
      s += __shfl_xor_sync(full, s, 2);
      if (row < m && q4 == 0) p[row] = tj * s;
    }
    __syncthreads();
    part = 0.0;
    for (int i = tid; i < m; i += nthr) part += p[i] * v[i];
    const double pv = block_sum(part, red);
    const double kc = -0.5 * tj * pv;
    for (int i = tid; i < m; i += nthr) p[i] = fma(kc, v[i], p[i]);  // w
    __syncthreads();
    for (int c = warp; c < m; c += nwarps) {
      const int b0 = pidx(n, j + 1 + c, j + 1 + c);
      const double vc = v[c], wc = p[c];
      for (int r = c + lane; r < m; r += 32) Lp[b0 + (r - c)] -= v[r] * wc + p[r] * vc;
    }
    __syncthreads();
  }
  }
  if (tid == 0) {
    if (n >= 2) {
      dd[n - 2] = Lp[pidx(n, n - 2, n - 2)];
      ee[n - 2] = Lp[pidx(n, n - 1, n - 2)];
      tau[n - 2] = 0.0;
    }
    dd[n - 1] = Lp[pidx(n, n - 1, n - 1)];
    ee[n - 1] = 0.0;
    tau[n - 1] = 0.0;
  }
  __syncthreads();
  for (int i = tid; i < n; i += nthr) e2[i] = (i + 1 < n) ? ee[i] * ee[i] : 0.0;
  __syncthreads();

  stamp(2);
  // ---- C: Gerschgorin bounds, multisection bisection (one warp per eigenvalue)
  double glo = DBL_MAX, ghi = -DBL_MAX, emax2 = 0.0;
  for (int i = lane; i < n; i += 32) {
    const double r = (i > 0 ? fabs(ee[i - 1]) : 0.0) + (i + 1 < n ? fabs(ee[i]) : 0.0);
    glo = fmin(glo, dd[i] - r);
    ghi = fmax(ghi, dd[i] + r);
    emax2 = fmax(emax2, e2[i]);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    glo = fmin(glo, __shfl_xor_sync(full, glo, o));
    ghi = fmax(ghi, __shfl_xor_sync(full, ghi, o));
    emax2 = fmax(emax2, __shfl_xor_sync(full, emax2, o));
  }
  const double tnorm = fmax(fabs(glo), fabs(ghi));
  const double pivmin = DBL_MIN * fmax(1.0, emax2);
  glo -= 2.0 * DBL_EPSILON * tnorm * n + 2.0 * pivmin;
  ghi += 2.0 * DBL_EPSILON * tnorm * n + 2.0 * pivmin;
  for (int k = warp; k < K; k += nwarps) {
    const int aidx = n - 1 - k;  // ascending index of the k-th largest
    double lo = glo, hi = ghi;
    for (int it = 0; it < 80; ++it) {
      const double x = lo + (hi - lo) * ((double)(lane + 1) / 33.0);
      double q = fix_pivot(dd[0] - x, pivmin);
      int cnt = q < 0.0;
      for (int i = 1; i < n; ++i) {
        q = fix_pivot((dd[i] - x) - e2[i - 1] / q, pivmin);
        cnt += q < 0.0;
      }
      const unsigned mask = __ballot_sync(full, cnt > aidx);
      const int f = mask ? __ffs(mask) - 1 : 32;
      const double xf = __shfl_sync(full, x, f & 31);
      const double xb = __shfl_sync(full, x, (f + 31) & 31);
      const double nhi = f < 32 ? xf : hi;
      const double nlo = f > 0 ? xb : lo;
      const bool stall = (nhi == hi && nlo == lo);
      lo = nlo;
      hi = nhi;
      if (stall || hi - lo <= 2.0 * DBL_EPSILON * fmax(fabs(lo), fabs(hi)) + pivmin) break;
    }
    if (lane == 0) lam[k] = 0.5 * (lo + hi);
  }
  __syncthreads();

  stamp(3);
  // ---- D: twisted-factorization eigenvectors of T: forward (dp) and backward (dm)
  // recurrences on two threads per eigenvalue, twist index = first argmin |gamma_r|
  // (warp per eigenvalue), then the two halves of z on two threads again.
  int* rsel = clus + K;  // K ints after the cluster leaders
  for (int u = tid; u < 2 * K; u += nthr) {
    const int k = u % K;
    const double lk = lam[k];
    if (u < K) {
      double* dp = Dp + (size_t)k * n;
      double q = fix_pivot(dd[0] - lk, pivmin);
      dp[0] = q;
      for (int i = 1; i < n; ++i) {
        q = fix_pivot((dd[i] - lk) - e2[i - 1] / q, pivmin);
        dp[i] = q;
      }
    } else {
      double* dm = Dm + (size_t)k * n;
      double q = fix_pivot(dd[n - 1] - lk, pivmin);
      dm[n - 1] = q;
      for (int i = n - 2; i >= 0; --i) {
        q = fix_pivot((dd[i] - lk) - e2[i] / q, pivmin);
        dm[i] = q;
      }
    }
  }
  __syncthreads();
  for (int k = warp; k < K; k += nwarps) {
    const double lk = lam[k];
    const double* dp = Dp + (size_t)k * n;
    const double* dm = Dm + (size_t)k * n;
    double gb = DBL_MAX;
    int rb = n;
    for (int i = lane; i < n; i += 32) {
      const double gm = fabs(dp[i] + dm[i] - (dd[i] - lk));
      if (gm < gb) { gb = gm; rb = i; }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double og = __shfl_xor_sync(full, gb, o);
      const int orr = __shfl_xor_sync(full, rb, o);
      if (og < gb || (og == gb && orr < rb)) { gb = og; rb = orr; }
    }
    if (lane == 0) rsel[k] = rb;
  }
  __syncthreads();
  for (int u = tid; u < 2 * K; u += nthr) {
    const int k = u % K;
    const int r = rsel[k];
    double* z = Z + (size_t)k * n;
    if (u < K) {
      const double* dp = Dp + (size_t)k * n;
      double zi = 1.0;
      z[r] = 1.0;
      for (int i = r - 1; i >= 0; --i) { zi = -ee[i] * zi / dp[i]; z[i] = zi; }
    } else {
      const double* dm = Dm + (size_t)k * n;
      double zi = 1.0;
      for (int i = r + 1; i < n; ++i) { zi = -ee[i - 1] * zi / dm[i]; z[i] = zi; }
    }
  }
  __syncthreads();
  // cluster leaders: consecutive eigenvalues closer than 1e-3 ||T|| (dstein's ORTOL)
  if (tid == 0) {
    int lead = 0;
    for (int k = 0; k < K; ++k) {
      if (k > 0 && lam[k - 1] - lam[k] > 1e-3 * tnorm) lead = k;
      clus[k] = lead;
    }
  }
  __syncthreads();

  stamp(4);
  // ---- E: normalize; MGS (twice) inside clusters; rescue collapsed vectors
  for (int k0 = warp; k0 < K; k0 += nwarps) {
    if (clus[k0] != k0) continue;  // this warp owns the cluster led by k0
    int kend = k0 + 1;
    while (kend < K && clus[kend] == k0) ++kend;
    for (int k = k0; k < kend; ++k) {
      double* z = Z + (size_t)k * n;
      for (int attempt = 0; attempt < 3; ++attempt) {
        double s = 0.0;
        for (int i = lane; i < n; i += 32) s += z[i] * z[i];
        double nrm = sqrt(warp_sum(s));
        for (int i = lane; i < n; i += 32) z[i] /= nrm;
        __syncwarp();
        for (int pass = 0; pass < 2; ++pass) {
          for (int q2 = k0; q2 < k; ++q2) {
            const double* zq = Z + (size_t)q2 * n;
            double c = 0.0;
            for (int i = lane; i < n; i += 32) c += zq[i] * z[i];
            c = warp_sum(c);
            for (int i = lane; i < n; i += 32) z[i] -= c * zq[i];
            __syncwarp();
          }
        }
        s = 0.0;
        for (int i = lane; i < n; i += 32) s += z[i] * z[i];
        nrm = sqrt(warp_sum(s));
        if (nrm > 0.5) {
          for (int i = lane; i < n; i += 32) z[i] /= nrm;
          __syncwarp();
          break;
        }
        // collapsed (degenerate cluster): two steps of LDL^T inverse iteration from a
        // pseudo-random start, re-orthogonalized on the next attempt
        const double* dp = Dp + (size_t)k * n;
        for (int i = lane; i < n; i += 32) z[i] = prand(k * 7919u + attempt, i);
        __syncwarp();
        for (int step = 0; step < 2; ++step) {
          if (lane == 0) {
            for (int i = 1; i < n; ++i) z[i] -= (ee[i - 1] / dp[i - 1]) * z[i - 1];
            for (int i = 0; i < n; ++i) z[i] /= dp[i];
            for (int i = n - 2; i >= 0; --i) z[i] -= (ee[i] / dp[i]) * z[i + 1];
            double mx = 0.0;
            for (int i = 0; i < n; ++i) mx = fmax(mx, fabs(z[i]));
            if (mx > 0.0) for (int i = 0; i < n; ++i) z[i] /= mx;
          }
          __syncwarp();
        }
      }
    }
  }
  __syncthreads();

  stamp(5);
  // ---- F: back-transform Z <- H_0 ... H_{n-3} Z  (warp per column, no block sync)
  if constexpr (FAST) {
    // z in registers (lane-owned rows), reflector j read from column j of the packed storage
    for (int k = warp; k < K; k += nwarps) {
      double* zg = Z + (size_t)k * n;
      double zr[NT];
#pragma unroll
      for (int t = 0; t < NT; ++t) {
        const int r = lane + 32 * t;
        zr[t] = r < n ? zg[r] : 0.0;
      }
      for (int j = n - 3; j >= 0; --j) {
        const double tj = tau[j];
        if (tj == 0.0) continue;
        const int base = cs[j] - j;
        double vr[NT];
        double s = 0.0;
#pragma unroll
        for (int t = 0; t < NT; ++t) {
          const int r = lane + 32 * t;
          if (32 * t + 31 < j + 1) { vr[t] = 0.0; continue; }  // warp-uniform
          const bool in = r >= j + 2 && r < n;
          const double lv = Lp[in ? base + r : base + j];     // clamped address, no branch
          vr[t] = in ? lv : (r == j + 1 ? 1.0 : 0.0);
          s = fma(vr[t], zr[t], s);
        }
        s = warp_sum(s) * tj;
#pragma unroll
        for (int t = 0; t < NT; ++t) zr[t] = fma(-s, vr[t], zr[t]);
      }
#pragma unroll
      for (int t = 0; t < NT; ++t) {
        const int r = lane + 32 * t;
        if (r < n) zg[r] = zr[t];
      }
    }
  } else {
    for (int k = warp; k < K; k += nwarps) {
      double* z = Z + (size_t)k * n;
      for (int j = n - 3; j >= 0; --j) {
        const double tj = tau[j];
        if (tj == 0.0) continue;
        const int cj = pidx(n, j, j);
        double s = 0.0;
        for (int i = j + 2 + lane; i < n; i += 32) s += Lp[cj + (i - j)] * z[i];
        s = warp_sum(s) + z[j + 1];
        s *= tj;
        if (lane == 0) z[j + 1] -= s;
        for (int i = j + 2 + lane; i < n; i += 32) z[i] -= s * Lp[cj + (i - j)];
        __syncwarp();
      }
    }
  }
  __syncthreads();

  stamp(6);
  if (split) {  // phases G/H run in ldlt_pack_kernel (concurrently) and sign_weights_kernel
    for (int k = tid; k < K; k += nthr) sigma_out[k] = sqrt(fmax(lam[k], 0.0));
    if (tid == 0) {
      for (int i = 0; i < n; ++i)
        if (!isfinite(dd[i]) || !isfinite(G[(size_t)i * n + i])) { atomicOr(status, PSVD_ST_NONFINITE); break; }
    }
    return;
  }
  // ---- G: R = chol(G + delta I), delta = 10 n eps max(diag G).
  // The reference's R is Householder's (well-determined only in the rows
  // where |R_ii| >> sqrt(eps)|C|); an unshifted Cholesky of the Gram turns the
  // remaining rows into O(1) garbage that can win the sign rule's argmax.
  // The shift bounds those rows by ~sqrt(delta) (their true U_R entries are
  // below ~1e-7 kappa_k anyway) and leaves the well-determined rows unchanged
  // to O(delta / R_ii^2).
  double dmax = 0.0;
  for (int i = tid; i < n; i += nthr) dmax = fmax(dmax, G[(size_t)i * n + i]);
  dmax = warp_max(dmax);
  if (lane == 0) red[warp] = dmax;
  __syncthreads();
  if (tid == 0) {
    double m = 0.0;
    for (int w = 0; w < nwarps; ++w) m = fmax(m, red[w]);
    red[40] = m;
  }
  __syncthreads();
  const double delta = 10.0 * (double)n * DBL_EPSILON * red[40];
  for (int64_t idx = tid; idx < (int64_t)n * n; idx += nthr) {
    const int i = (int)(idx % n), j = (int)(idx / n);
    if (i >= j) Lp[pidx(n, i, j)] = G[idx] + (i == j ? delta : 0.0);
  }
  __syncthreads();
  if constexpr (FAST) {
    // LDL^T, one barrier per column: column k is read-only in step k; rows lane-owned.
    // Stored: diagonal D_k and the unscaled column A'[r][k] = L[r][k] D_k; R = D^-1/2 A'^T.
    for (int k = 0; k + 1 < n; ++k) {
      const double piv = Lp[cs[k]];
      if (piv > 0.0) {
        const double ipiv = 1.0 / piv;
        double lr[NT];
#pragma unroll
        for (int t = 0; t < NT; ++t) {
          const int r = lane + 32 * t;
          lr[t] = (r > k && r < n) ? Lp[cs[k] + (r - k)] : 0.0;
        }
        for (int c = k + 1 + ((warp - (k + 1)) % nwarps + nwarps) % nwarps; c < n; c += nwarps) {
          const double lc = Lp[cs[k] + (c - k)] * ipiv;
          const int base = cs[c] - c;
#pragma unroll
          for (int t = 0; t < NT; ++t) {
            const int r = lane + 32 * t;
            if (r >= c && r < n) Lp[base + r] -= lr[t] * lc;
          }
        }
      }
      __syncthreads();
    }
    // convert to the Cholesky form used by phase H: column k -> A'[r][k] / sqrt(D_k)
    for (int k = warp; k < n; k += nwarps) {
      const double dk = Lp[cs[k]];
      const double inv = dk > 0.0 ? 1.0 / sqrt(dk) : 0.0;
      for (int r = k + lane; r < n; r += 32) Lp[cs[k] + (r - k)] *= inv;
    }
    __syncthreads();
  } else {
  for (int k = 0; k < n; ++k) {
    const int ck = pidx(n, k, k);
    const double piv = Lp[ck];
    __syncthreads();
    const bool ok = piv > 0.0;
    const double rk = ok ? sqrt(piv) : 0.0;
    for (int i = tid; i < n - k; i += nthr) Lp[ck + i] = ok ? (i == 0 ? rk : Lp[ck + i] / rk) : 0.0;
    __syncthreads();
    if (ok) {
      for (int c = k + 1 + warp; c < n; c += nwarps) {
        const int bc = pidx(n, c, c);
        const double lck = Lp[ck + (c - k)];
        for (int r = c + lane; r < n; r += 32) Lp[bc + (r - c)] -= Lp[ck + (r - k)] * lck;
      }
    }
    __syncthreads();
  }

  }
  stamp(7);
  // ---- H: sign rule on U_R = R V (R = L^T), weights, singular values
  for (int k = warp; k < K; k += nwarps) {
    const double* z = Z + (size_t)k * n;
    double best_abs = -1.0, best_val = 0.0;
    for (int i = 0; i < n; ++i) {
      const int ci = pidx(n, i, i);
      double s = 0.0;
      for (int jj = i + lane; jj < n; jj += 32) s += Lp[ci + (jj - i)] * z[jj];
      s = warp_sum(s);
      if (fabs(s) > best_abs) { best_abs = fabs(s); best_val = s; }
    }
    const double sg = best_val < 0.0 ? -1.0 : 1.0;
    const double sk = sqrt(fmax(lam[k], 0.0));
    const double s0 = sqrt(fmax(lam[0], 0.0));
    const bool keep = sk > 0.0 && sk > rank_tol * s0;  // rank_tol > 0: drop numerically null directions
    const double inv = keep ? sg / sk : 0.0;
    if (sk == 0.0 && rank_tol == 0.0 && lane == 0) atomicOr(status, PSVD_ST_RANKDEF);
    for (int i = lane; i < n; i += 32) W[(size_t)k * n + i] = (dscale ? dscale[i] : 1.0) * z[i] * inv;
    if (lane == 0) sigma_out[k] = sk;
  }
  if (tid == 0) {
    for (int i = 0; i < n; ++i)
      if (!isfinite(dd[i]) || !isfinite(G[(size_t)i * n + i])) { atomicOr(status, PSVD_ST_NONFINITE); break; }
  }
  __syncthreads();
  stamp(8);
}

bool eig_supported(int n, int K) { return n >= 1 && K >= 1 && K <= n && K <= 1024; }

void launch_eig_topk(const double* G, int n, int K, const double* dscale, double* W, double* sigma,
                     double* ws, int* status, long long* timers, cudaStream_t st, double rank_tol, int split,
                     const int* gate) {
  const int npad = (n + 31) / 32 * 32;
  const size_t vec = (size_t)6 * n + K + 64 + K + 2;  // ... + clus (K ints) + rsel (K ints)
  const size_t fast_extra = (size_t)(n + 1) / 2 + 1 + 5 * (size_t)npad + (size_t)(EIG_FAST_THREADS / 32) * npad + 8;
  const size_t npk = (size_t)n * (n + 1) / 2;
  const size_t limit = 227 * 1024;
  if (n <= EIG_FAST_NMAX && (npk + vec + fast_extra) * sizeof(double) <= limit) {
    const size_t smem = (npk + vec + fast_extra) * sizeof(double);
    cudaFuncSetAttribute(eig_topk_kernel<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    eig_topk_kernel<true, true><<<1, EIG_FAST_THREADS, smem, st>>>(G, n, K, dscale, W, sigma, ws, status, timers,
                                                                    rank_tol, split, gate);
  } else if (n <= EIG_NMAX_SMEM) {
    const size_t smem = (npk + vec) * sizeof(double);
    cudaFuncSetAttribute(eig_topk_kernel<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    eig_topk_kernel<true, false><<<1, SMALL_THREADS, smem, st>>>(G, n, K, dscale, W, sigma, ws, status, timers,
                                                                  rank_tol, split, gate);
  } else {
    const size_t smem = vec * sizeof(double);
    cudaFuncSetAttribute(eig_topk_kernel<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    eig_topk_kernel<false, false><<<1, SMALL_THREADS, smem, st>>>(G, n, K, dscale, W, sigma, ws, status, timers,
                                                                   rank_tol, split, gate);
  }
}

// ---------------------------------------------------------------- split core: LDL^T and sign/weights
// The sign rule's factor R = chol(G + delta I) depends only on G, so it runs as its
// own one-CTA kernel on an auxiliary stream, concurrently with the eigensolver.
bool eig_split_supported(int n, int K) {
  const size_t npk = (size_t)n * (n + 1) / 2;
  return n <= EIG_FAST_NMAX && (npk + n) * sizeof(double) <= 227 * 1024 && K <= 1024;
}

__global__ void __launch_bounds__(EIG_FAST_THREADS, 1)
ldlt_pack_kernel(const double* __restrict__ G, int n, double* __restrict__ Lout) {
  extern __shared__ double sm[];
  constexpr int NT = (EIG_FAST_NMAX + 31) / 32;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nthr = blockDim.x, nwarps = nthr >> 5;
  const size_t npk = (size_t)n * (n + 1) / 2;
  double* Lp = sm;
  int* cs = reinterpret_cast<int*>(sm + npk);
  double* red = sm + npk + (n + 1) / 2 + 1;
  for (int c = tid; c < n; c += nthr) cs[c] = pidx(n, c, c);
  double dmax = 0.0;
  for (int i = tid; i < n; i += nthr) dmax = fmax(dmax, G[(size_t)i * n + i]);
  dmax = warp_max(dmax);
  if (lane == 0) red[warp] = dmax;
  __syncthreads();
  double gmax = 0.0;
  for (int w = 0; w < nwarps; ++w) gmax = fmax(gmax, red[w]);
  const double delta = 10.0 * (double)n * DBL_EPSILON * gmax;  // see the eigensolver's phase G
  for (int64_t idx = tid; idx < (int64_t)n * n; idx += nthr) {
    const int i = (int)(idx % n), j = (int)(idx / n);
    if (i >= j) Lp[cs[j] + (i - j)] = G[idx] + (i == j ? delta : 0.0);
  }
  __syncthreads();
  for (int k = 0; k + 1 < n; ++k) {
    const double piv = Lp[cs[k]];
    if (piv > 0.0) {
      const double ipiv = 1.0 / piv;
      double lr[NT];
#pragma unroll
      for (int t = 0; t < NT; ++t) {
        const int r = lane + 32 * t;
        lr[t] = (r > k && r < n) ? Lp[cs[k] + (r - k)] : 0.0;
      }
      for (int c = k + 1 + ((warp - (k + 1)) % nwarps + nwarps) % nwarps; c < n; c += nwarps) {
        const double lc = Lp[cs[k] + (c - k)] * ipiv;
        const int base = cs[c] - c;
#pragma unroll
        for (int t = 0; t < NT; ++t) {
          const int r = lane + 32 * t;
          if (r >= c && r < n) Lp[base + r] -= lr[t] * lc;
        }
      }
    }
    __syncthreads();
  }
  for (int k = warp; k < n; k += nwarps) {  // Cholesky columns A'[r][k] / sqrt(D_k), packed to global
    const double dk = Lp[cs[k]];
    const double inv = dk > 0.0 ? 1.0 / sqrt(dk) : 0.0;
    for (int r = k + lane; r < n; r += 32) Lout[cs[k] + (r - k)] = Lp[cs[k] + (r - k)] * inv;
  }
}

__global__ void __launch_bounds__(EIG_FAST_THREADS, 1)
sign_weights_kernel(const double* __restrict__ Lg, const double* __restrict__ Z, const double* __restrict__ sigma_in,
                    int n, int K, const double* __restrict__ dscale, double* __restrict__ W,
                    double* __restrict__ sigma_out, int* __restrict__ status, double rank_tol) {
  extern __shared__ double sm[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nthr = blockDim.x, nwarps = nthr >> 5;
  const size_t npk = (size_t)n * (n + 1) / 2;
  double* Lp = sm;
  for (size_t i = tid; i < npk; i += nthr) Lp[i] = Lg[i];
  __syncthreads();
  // U_R[i][k] = (R v_k)_i = sum_{j >= i} L[j][i] z_k[j]: thread per (i, k), written to W as scratch
  for (int q = tid; q < n * K; q += nthr) {
    const int i = q % n, k = q / n;
    const int ci = pidx(n, i, i);
    const double* z = Z + (size_t)k * n;
    double s = 0.0;
    for (int jj = i; jj < n; ++jj) s = fma(Lp[ci + (jj - i)], z[jj], s);
    W[(size_t)k * n + i] = s;
  }
  __syncthreads();
  for (int k = warp; k < K; k += nwarps) {
    double ba = -1.0, bv = 0.0;
    int bi = n;
    for (int i = lane; i < n; i += 32) {
      const double u = W[(size_t)k * n + i];
      if (fabs(u) > ba) { ba = fabs(u); bv = u; bi = i; }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {  // max |u|, lowest row on ties (numpy argmax)
      const double oa = __shfl_xor_sync(0xffffffffu, ba, o);
      const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (oa > ba || (oa == ba && oi < bi)) { ba = oa; bv = ov; bi = oi; }
    }
    const double sg = bv < 0.0 ? -1.0 : 1.0;
    const double sk = sigma_in[k];
    const double s0 = sigma_in[0];
    const bool keep = sk > 0.0 && sk > rank_tol * s0;
    const double inv = keep ? sg / sk : 0.0;
    if (sk == 0.0 && rank_tol == 0.0 && lane == 0) atomicOr(status, PSVD_ST_RANKDEF);
    __syncwarp();
    const double* z = Z + (size_t)k * n;
    for (int i = lane; i < n; i += 32) W[(size_t)k * n + i] = (dscale ? dscale[i] : 1.0) * z[i] * inv;
    if (lane == 0 && sigma_out != sigma_in) sigma_out[k] = sk;
  }
}

// The same factor, blocked: chol(G + delta I) over 32-column panels held in shared memory as dense
// (n - 32p) x 32 column-major blocks (202 KB at n = 210).  Per panel: warp 0 factors the 32 x 32
// diagonal block (lane-owned rows, syncwarp only), every thread solves one row below it (forward
// substitution against the block), and the warps apply the rank-32 trailing update as 8 x 8 DMMA
// tiles of the lower triangle: 3 CTA barriers per panel instead of one per column (ldlt_pack_kernel:
// ~367 us at n = 210, one barrier per column and n^3 / 6 shared-memory FMAs).  Zero / negative pivots
// give zero columns, as ldlt_pack_kernel's.
constexpr int CP = 8;  // panel width (8: one DMMA k-step pair per trailing tile, a short pivot chain per panel)

__host__ __device__ inline int cp_panels(int n) { return (n + CP - 1) / CP; }
__host__ __device__ inline size_t cp_doubles(int n) {
  size_t t = 0;
  for (int p = 0; p < cp_panels(n); ++p) t += (size_t)(n - CP * p) * CP;
  return t;
}

__global__ void __launch_bounds__(EIG_FAST_THREADS, 1)
chol_panels_kernel(const double* __restrict__ G, int n, double* __restrict__ Lout) {
  extern __shared__ double sm[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nthr = blockDim.x, nwarps = nthr >> 5;
  const int P = cp_panels(n);
  __shared__ int pb[64];  // panel base offsets (n <= 512)
  __shared__ double red[32];
  if (tid == 0) {
    int off = 0;
    for (int p = 0; p < P; ++p) {
      pb[p] = off;
      off += (n - CP * p) * CP;
    }
  }
  double dmax = 0.0;
  for (int i = tid; i < n; i += nthr) dmax = fmax(dmax, G[(size_t)i * n + i]);
  dmax = warp_max(dmax);
  if (lane == 0) red[warp] = dmax;
  __syncthreads();
  double gmax = 0.0;
  for (int w = 0; w < nwarps; ++w) gmax = fmax(gmax, red[w]);
  const double delta = 10.0 * (double)n * DBL_EPSILON * gmax;  // ldlt_pack_kernel's shift
  // element (r, c), r >= c: panel p = c / 32, column j = c % 32, row r - 32 p of the (n - 32 p) rows
  auto at = [&](int r, int c) -> double& {
    const int p = c / CP;
    return sm[pb[p] + (c - CP * p) * (n - CP * p) + (r - CP * p)];
  };
  for (int j = warp; j < n; j += nwarps) {  // column j: coalesced reads, one panel lookup
    const int pj = j / CP;
    double* col = sm + pb[pj] + (j - CP * pj) * (n - CP * pj) - CP * pj;  // col[r] = element (r, j)
    for (int i = j + lane; i < n; i += 32) col[i] = G[(size_t)j * n + i] + (i == j ? delta : 0.0);
  }
  __syncthreads();
  for (int p = 0; p < P; ++p) {
    const int c0 = CP * p, w = min(CP, n - c0), nr = n - c0;
    double* Pp = sm + pb[p];  // nr x CP, column j at Pp + j nr, local row i
    if (warp == 0) {
      // the CP x CP diagonal block in registers, lane i = local row i (padded with the identity past w):
      // straight-line code, shuffles only
      double row[CP];
#pragma unroll
      for (int j = 0; j < CP; ++j)
        row[j] = (lane < w && j < w) ? (j <= lane ? Pp[j * nr + lane] : 0.0) : (j == lane ? 1.0 : 0.0);
#pragma unroll
      for (int k = 0; k < CP; ++k) {
        const double d = __shfl_sync(0xffffffffu, row[k], k);
        const bool ok = d > 0.0;
        const double lkk = ok ? sqrt(d) : 0.0;
        const double inv = ok ? 1.0 / lkk : 0.0;
        const double lik = lane == k ? lkk : (lane > k ? row[k] * inv : 0.0);
        row[k] = lik;
#pragma unroll
        for (int j = k + 1; j < CP; ++j) {
          const double ljk = __shfl_sync(0xffffffffu, lik, j);  // L(j, k), held by lane j
          row[j] = lane >= j ? fma(-lik, ljk, row[j]) : row[j];
        }
      }
#pragma unroll
      for (int j = 0; j < CP; ++j)
        if (lane < w && j <= lane && j < w) Pp[j * nr + lane] = row[j];
    }
    __syncthreads();
    // rows below the block: l_i = a_i L_d^-T, one thread per row, forward substitution in place
    for (int i = w + tid; i < nr; i += nthr) {
      for (int k = 0; k < w; ++k) {
        const double lkk = Pp[k * nr + k];
        double v = Pp[k * nr + i];
        for (int j = 0; j < k; ++j) v = fma(-Pp[j * nr + i], Pp[j * nr + k], v);
        Pp[k * nr + i] = lkk > 0.0 ? v / lkk : 0.0;
      }
    }
    __syncthreads();
    // trailing update on 8 x 8 DMMA tiles: A(r, c) -= sum_k L(r, k) L(c, k), r >= c >= c0 + w
    const int t0 = c0 + w;
    if (t0 < n) {
      const int nb = (n - t0 + 7) / 8;
      const int ntiles = nb * (nb + 1) / 2;
      const int g = lane >> 2, tq = lane & 3;
      for (int t = warp; t < ntiles; t += nwarps) {
        int bi = 0, rem = t;  // tile t -> (bi >= bj), row-major over the lower triangle
        while (rem > bi) { rem -= bi + 1; ++bi; }
        const int bj = rem;
        const int r0 = t0 + 8 * bi, cc0 = t0 + 8 * bj;
        double d0 = 0.0, d1 = 0.0;
        const int ra = r0 + g, cb = cc0 + g;
        for (int k0 = 0; k0 < w; k0 += 4) {
          const int k = k0 + tq;
          const double a = (ra < n && k < w) ? Pp[k * nr + (ra - c0)] : 0.0;
          const double b = (cb < n && k < w) ? Pp[k * nr + (cb - c0)] : 0.0;
          dmma884(d0, d1, a, b);
        }
        // d{0,1} = D[g][2 tq + {0,1}]: rows r0 + g, columns cc0 + 2 tq (+1)
        const int r = r0 + g;
        const int ca = cc0 + 2 * tq;
        if (r < n && ca < n && r >= ca) at(r, ca) -= d0;
        if (r < n && ca + 1 < n && r >= ca + 1) at(r, ca + 1) -= d1;
      }
    }
    __syncthreads();
  }
  // packed lower output (ldlt_pack's layout: column c at pidx(n, c, c))
  for (int j = warp; j < n; j += nwarps) {
    const int pj = j / CP;
    const double* col = sm + pb[pj] + (j - CP * pj) * (n - CP * pj) - CP * pj;
    double* out = Lout + pidx(n, j, j) - j;
    for (int i = j + lane; i < n; i += 32) out[i] = col[i];
  }
}

void launch_ldlt_pack(const double* G, int n, double* Lout, cudaStream_t st) {
  static const bool old = getenv("PSVD_OLD_LDLT") != nullptr;  // A/B: the unblocked kernel
  const size_t blocked = cp_doubles(n) * sizeof(double);
  if (!old && blocked <= 227 * 1024 && cp_panels(n) <= 64) {
    cudaFuncSetAttribute(chol_panels_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)blocked);
    chol_panels_kernel<<<1, EIG_FAST_THREADS, blocked, st>>>(G, n, Lout);
    return;
  }
  const size_t smem = ((size_t)n * (n + 1) / 2 + (n + 1) / 2 + 1 + 32) * sizeof(double);
  cudaFuncSetAttribute(ldlt_pack_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  ldlt_pack_kernel<<<1, EIG_FAST_THREADS, smem, st>>>(G, n, Lout);
}

void launch_sign_weights(const double* Lg, const double* Z, const double* sigma, int n, int K, const double* dscale,
                         double* W, double* sigma_out, int* status, double rank_tol, cudaStream_t st) {
  const size_t smem = ((size_t)n * (n + 1) / 2) * sizeof(double);
  cudaFuncSetAttribute(sign_weights_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  sign_weights_kernel<<<1, EIG_FAST_THREADS, smem, st>>>(Lg, Z, sigma, n, K, dscale, W, sigma_out, status, rank_tol);
}

// ---------------------------------------------------------------- Rayleigh refinement
// U = C V S^-1 from the Gram route has ||u_k|| = ||C v_k|| / s_k, and ||C v_k|| is
// the Rayleigh estimate of the singular value (second-order accurate in the
// eigenvector error, vs eps*kappa^2 for sqrt(lambda)).  sigma_k <- ||C v_k||,
// UtU <- D^-1 UtU D^-1 (D = diag ||u_k||) and scale_k = 1 / ||u_k|| for the columns.
__global__ void normalize_gram_kernel(double* __restrict__ UtU, int K, double* __restrict__ sigma,
                                      double* __restrict__ scale, int* __restrict__ status) {
  __shared__ double nk[1024];
  for (int k = threadIdx.x; k < K; k += blockDim.x) {
    const double d = UtU[(size_t)k * K + k];
    nk[k] = d > 0.0 ? sqrt(d) : 1.0;
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < K * K; idx += blockDim.x) {
    const int i = idx % K, j = idx / K;
    UtU[idx] = UtU[idx] / (nk[i] * nk[j]);
  }
  for (int k = threadIdx.x; k < K; k += blockDim.x) {
    sigma[k] *= nk[k];
    scale[k] = 1.0 / nk[k];
  }
  // conditioning gate of the Gram route: its kept values carry eps (s_1 / s_k)^2 error terms, so a
  // kept spectrum wider than GRAM_KAPPA_MAX flags the update for the accurate (R-factor) route
  __syncthreads();
  if (threadIdx.x == 0 && status != nullptr && K > 0 && !(sigma[K - 1] * GRAM_KAPPA_MAX >= sigma[0]))
    atomicOr(status, PSVD_ST_ILLCOND);
}

void launch_normalize_gram(double* UtU, int K, double* sigma, double* scale, int* status, cudaStream_t st) {
  normalize_gram_kernel<<<1, 1024, 0, st>>>(UtU, K, sigma, scale, status);
}

// ---------------------------------------------------------------- drift check / rescue

__global__ void __launch_bounds__(1024, 1)
drift_check_kernel(const double* __restrict__ UtU, int K, double tol, double* __restrict__ sigma,
                   double* __restrict__ T, int* __restrict__ gate, int* __restrict__ status) {
  extern __shared__ double sm[];
  double* A = sm;               // K x K
  double* X = A + K * K;        // K x K (inverse of rr)
  double* vals = X + K * K;     // K
  double* red = vals + K;       // 64
  int* order = reinterpret_cast<int*>(red + 64);
  const int tid = threadIdx.x, nthr = blockDim.x;
  double dev = 0.0;
  for (int idx = tid; idx < K * K; idx += nthr) {
    const double a = UtU[idx];
    A[idx] = a;
    const int i = idx % K, j = idx / K;
    dev = fmax(dev, fabs(a - (i == j ? 1.0 : 0.0)));
  }
  dev = warp_max(dev);
  if ((tid & 31) == 0) red[tid >> 5] = dev;
  __syncthreads();
  if (tid == 0) {
    double m = 0.0;
    for (int w = 0; w < (nthr + 31) / 32; ++w) m = fmax(m, red[w]);
    red[40] = m;
  }
  __syncthreads();
  if (!(red[40] > tol)) {
    if (tid == 0) *gate = 0;
    return;
  }
  // Cholesky A = L L^T (upper rr = L^T), column by column
  for (int k = 0; k < K; ++k) {
    if (tid == 0) A[k * K + k] = sqrt(fmax(A[k * K + k], 0.0));
    __syncthreads();
    const double rk = A[k * K + k];
    for (int i = k + 1 + tid; i < K; i += nthr) A[k * K + i] = rk > 0.0 ? A[k * K + i] / rk : 0.0;
    __syncthreads();
    for (int idx = tid; idx < K * K; idx += nthr) {
      const int i = idx % K, j = idx / K;
      if (j > k && i >= j) A[j * K + i] -= A[k * K + i] * A[k * K + j];
    }
    __syncthreads();
  }
  // X = rr^{-1}, rr upper with rr[i][j] = L[j][i] = A[i*K + j] (i <= j)
  for (int j = tid; j < K; j += nthr) {
    for (int i = K - 1; i >= 0; --i) {
      double s = (i == j) ? 1.0 : 0.0;
      for (int q = i + 1; q <= j; ++q) s -= A[i * K + q] * X[j * K + q];
      const double d = A[i * K + i];
      X[j * K + i] = (i <= j && d != 0.0) ? s / d : 0.0;
    }
  }
  for (int k = tid; k < K; k += nthr) vals[k] = sigma[k] * fabs(A[k * K + k]);
  __syncthreads();
  if (tid == 0) {
    for (int k = 0; k < K; ++k) order[k] = k;
    for (int a = 1; a < K; ++a) {  // stable insertion sort, descending
      const int oa = order[a];
      int b = a - 1;
      while (b >= 0 && vals[order[b]] < vals[oa]) { order[b + 1] = order[b]; --b; }
      order[b + 1] = oa;
    }
    *gate = 1;
    atomicOr(status, PSVD_ST_RESCUE);
  }
  __syncthreads();
  for (int idx = tid; idx < K * K; idx += nthr) {
    const int i = idx % K, c = idx / K;
    T[(size_t)c * K + i] = X[order[c] * K + i];
  }
  for (int c = tid; c < K; c += nthr) sigma[c] = vals[order[c]];
}

void launch_drift_check(const double* UtU, int K, double tol, double* sigma, double* T, int* gate,
                        int* status, cudaStream_t st) {
  const size_t smem = (2 * (size_t)K * K + K + 64 + (K + 1) / 2 + 1) * sizeof(double);
  cudaFuncSetAttribute(drift_check_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  drift_check_kernel<<<1, 1024, smem, st>>>(UtU, K, tol, sigma, T, gate, status);
}

}  // namespace psvd
