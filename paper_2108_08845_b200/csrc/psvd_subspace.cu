// Subspace-iteration fast path of the core solve (top-K eigenpairs of the n x n Gram).
//
// The streaming Gram of a numerically low-rank snapshot stream (Burgers: lambda_33 /
// lambda_10 < 1e-7) has its top K eigenvectors inside the span of G^m Q0 after m = 2
// applications.  So before the one-CTA Householder eigensolver (O(n^3) latency-bound
// steps) we try:
//   ss_iterate:  X0 = [e_0..e_{K-1} | pseudo-random] (n x 32), Q <- orth(G Q) twice from Q = X0,
//                W = G Q, H = Q^T W (32 x 32).  G Q on DMMA with G streamed from L2,
//                orth = Householder QR in shared memory (one CTA).
//   eig_topk(H): Ritz values / vectors (the existing solver at n = 32).
//   ss_finish:   X = Q Z_H, GX = W Z_H, residuals ||GX_k - theta_k X_k||; if all are below
//                tol * theta_0 the Ritz pairs are the result (same buffers as the full
//                solver's split mode) and the gate skips the full solver; otherwise the
//                full solver runs unchanged.  Either way the result is exact to the
//                working precision: a Ritz pair with residual r has eigenvalue error
//                <= r^2 / gap and angle <= r / gap (Davis-Kahan), the bounds of the full
//                solver at r ~ eps ||G||.
#include <algorithm>
#include <cfloat>
#include <cstdlib>

#include "psvd_small.cuh"

namespace psvd {

namespace {

constexpr int SP = SS_P;  // block width (4 DMMA column blocks)

__device__ __forceinline__ double prand_ss(unsigned a, unsigned b) {
  unsigned h = a * 0x9E3779B1u ^ (b + 0x7F4A7C15u) * 0x85EBCA77u;
  h ^= h >> 15; h *= 0x2C1B3C6Du; h ^= h >> 12; h *= 0x297A2D39u; h ^= h >> 15;
  return ((double)h / 4294967296.0) * 2.0 - 1.0;
}

// Ws (n x SP, ld ldq, rows >= n zero) = G (n x n, col-major, global) * Qs (smem, rows >= n zero)
__device__ void gq_product(const double* __restrict__ G, int n, const double* Qs, int ldq, double* Ws) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  const int g = lane >> 2, tq = lane & 3;
  const int nrb = (n + 7) / 8;
  const int kend = (n + 7) / 8 * 8;
  for (int rb = warp; rb < nrb; rb += nwarps) {
    const int row = rb * 8 + g;
    const bool rv = row < n;
    constexpr int CB = SP / 8;  // 8-column DMMA blocks of Q
    double acc[CB][2][2];
#pragma unroll
    for (int c = 0; c < CB; ++c) acc[c][0][0] = acc[c][0][1] = acc[c][1][0] = acc[c][1][1] = 0.0;
#pragma unroll 4
    for (int k0 = 0; k0 < kend; k0 += 8) {  // unrolled: several k steps' loads of G (L2) in flight
      const int ka = k0 + tq, kb = k0 + 4 + tq;
      const double a0 = (rv && ka < n) ? __ldg(G + (size_t)ka * n + row) : 0.0;
      const double a1 = (rv && kb < n) ? __ldg(G + (size_t)kb * n + row) : 0.0;
#pragma unroll
      for (int c = 0; c < CB; ++c) {
        dmma884(acc[c][0][0], acc[c][0][1], a0, Qs[(size_t)(c * 8 + g) * ldq + ka]);
        dmma884(acc[c][1][0], acc[c][1][1], a1, Qs[(size_t)(c * 8 + g) * ldq + kb]);
      }
    }
#pragma unroll
    for (int c = 0; c < CB; ++c) {
      Ws[(size_t)(c * 8 + 2 * tq) * ldq + row] = rv ? acc[c][0][0] + acc[c][1][0] : 0.0;
      Ws[(size_t)(c * 8 + 2 * tq + 1) * ldq + row] = rv ? acc[c][0][1] + acc[c][1][1] : 0.0;
    }
  }
}

// Rows per lane of the fixed-trip loops below (n <= EIG_FAST_NMAX): every load of a column segment
// is issued before the first use, instead of one shared-memory round trip per loop iteration
constexpr int HR = (EIG_FAST_NMAX + 31) / 32;

// Householder reflector of column j of Y (rows j .. n-1), by one warp: v = Y[j+1:, j] scaled in
// place (v_j = 1 implied), tau into *tau_out; Y[j, j] keeps alpha (R is not needed).
__device__ __forceinline__ void house_reflector(double* v, int j, int n, double* tau_out) {
  const int lane = threadIdx.x & 31;
  double x[HR];
#pragma unroll
  for (int t = 0; t < HR; ++t) {
    const int i = j + 1 + lane + 32 * t;
    x[t] = i < n ? v[i] : 0.0;
  }
  double part = 0.0;
#pragma unroll
  for (int t = 0; t < HR; ++t) part = fma(x[t], x[t], part);
  const double xn2 = warp_sum(part);
  const double alpha = v[j];
  double tau = 0.0, scl = 0.0;
  if (xn2 != 0.0) {
    const double beta = -copysign(sqrt(alpha * alpha + xn2), alpha);
    tau = (beta - alpha) / beta;
    scl = 1.0 / (alpha - beta);
  }
#pragma unroll
  for (int t = 0; t < HR; ++t) {
    const int i = j + 1 + lane + 32 * t;
    if (i < n) v[i] = x[t] * scl;
  }
  if (lane == 0) *tau_out = tau;
}

// y <- H_j y = y - tau v (v^T y) on rows j .. n-1, by one warp (v_j = 1 implied)
__device__ __forceinline__ void house_apply(const double* v, double tau, int j, int n, double* y) {
  const int lane = threadIdx.x & 31;
  double vv[HR], yy[HR];
#pragma unroll
  for (int t = 0; t < HR; ++t) {
    const int i = j + 1 + lane + 32 * t;
    vv[t] = i < n ? v[i] : 0.0;
    yy[t] = i < n ? y[i] : 0.0;
  }
  double s = 0.0;
#pragma unroll
  for (int t = 0; t < HR; ++t) s = fma(vv[t], yy[t], s);
  s = (warp_sum(s) + y[j]) * tau;
  __syncwarp();
  if (lane == 0) y[j] -= s;
#pragma unroll
  for (int t = 0; t < HR; ++t) {
    const int i = j + 1 + lane + 32 * t;
    if (i < n) y[i] = fma(-s, vv[t], yy[t]);
  }
  __syncwarp();
}

// Householder QR of Y (n x SP in smem, ld ldq); Q (explicit, n x SP) into Qs.  Y is destroyed.
// One CTA barrier per column: the warp that updates column j + 1 (warp 0) forms its reflector
// right away while the other warps update theirs.  Q column c = H_0 ... H_c e_c (the reflectors
// after c leave e_c alone), one warp per column, no barriers.
__device__ void house_qr(double* Ys, int n, int ldq, double* Qs, double* stau) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  if (warp == 0) house_reflector(Ys, 0, n, &stau[0]);
  __syncthreads();
  for (int j = 0; j < SP - 1; ++j) {
    const double* v = Ys + (size_t)j * ldq;
    const double tau = stau[j];
    for (int c = j + 1 + warp; c < SP; c += nwarps) {
      double* y = Ys + (size_t)c * ldq;
      house_apply(v, tau, j, n, y);
      if (c == j + 1) house_reflector(y, j + 1, n, &stau[j + 1]);  // warp 0: the next reflector
    }
    __syncthreads();
  }
  // columns c and SP - 1 - c on one warp (equal work: c + 1 + SP - c reflector applications)
  for (int w = warp; w < SP / 2; w += nwarps)
    for (int h = 0; h < 2; ++h) {
      const int c = h ? SP - 1 - w : w;
      double* q = Qs + (size_t)c * ldq;
      for (int i = lane; i < ldq; i += 32) q[i] = (i == c) ? 1.0 : 0.0;
      __syncwarp();
      for (int j = c; j >= 0; --j) house_apply(Ys + (size_t)j * ldq, stau[j], j, n, q);
    }
  __syncthreads();
}

__global__ void __launch_bounds__(SS_THREADS, 1)
    ss_iterate_kernel(const double* __restrict__ G, int n, int K, int iters, double* __restrict__ Qg,
                      double* __restrict__ Wg, double* __restrict__ Hg) {
  extern __shared__ double ssm[];
  const int ldq = (n + 15) / 16 * 16 + 4;  // = 4 (mod 16): conflict-free B fragments
  double* Qs = ssm;
  double* Ys = Qs + (size_t)SP * ldq;
  double* stau = Ys + (size_t)SP * ldq;
  // X0 = [e_0 .. e_{K-1} | pseudo-random], rows >= n zero.  No QR of X0: span(G^m X0) does not
  // depend on the basis of span(X0), and X0 is well conditioned (unit vectors next to random
  // columns), so the first product takes X0 as it is
  for (int i = threadIdx.x; i < SP * ldq; i += blockDim.x) {
    const int c = i / ldq, r = i % ldq;
    double v = 0.0;
    if (r < n) v = (c < K) ? (r == c ? 1.0 : 0.0) : prand_ss(7919u * c + 17u, r);
    Qs[i] = v;
  }
  __syncthreads();
  for (int it = 0; it < iters; ++it) {
    gq_product(G, n, Qs, ldq, Ys);
    __syncthreads();
    house_qr(Ys, n, ldq, Qs, stau);
  }
  gq_product(G, n, Qs, ldq, Ys);  // W = G Q
  __syncthreads();
  for (int i = threadIdx.x; i < SP * n; i += blockDim.x) {
    const int c = i / n, r = i % n;
    Qg[i] = Qs[(size_t)c * ldq + r];
    Wg[i] = Ys[(size_t)c * ldq + r];
  }
  // H = sym(Q^T W)
  for (int e = threadIdx.x; e < SP * SP; e += blockDim.x) {
    const int a = e % SP, b = e / SP;
    if (a > b) continue;
    const double* qa = Qs + (size_t)a * ldq;
    const double* wb = Ys + (size_t)b * ldq;
    const double* qb = Qs + (size_t)b * ldq;
    const double* wa = Ys + (size_t)a * ldq;
    double s1 = 0.0, s2 = 0.0;
    for (int i = 0; i < n; ++i) {
      s1 = fma(qa[i], wb[i], s1);
      s2 = fma(qb[i], wa[i], s2);
    }
    const double h = 0.5 * (s1 + s2);
    Hg[(size_t)b * SP + a] = h;
    Hg[(size_t)a * SP + b] = h;
  }
}

// Ritz pairs from eig(H): X = Q Z_H, residual check, outputs in the full solver's split-mode slots.
__global__ void __launch_bounds__(SS_THREADS, 1)
    ss_finish_kernel(int n, int K, const double* __restrict__ Qg, const double* __restrict__ Wg,
                     const double* __restrict__ ZH, const double* __restrict__ sigH, double tol,
                     double* __restrict__ Zout, double* __restrict__ sigma_out, int* __restrict__ gate) {
  __shared__ double zh[SP * 16];
  __shared__ double res[16];
  __shared__ int bad;
  if (threadIdx.x == 0) bad = 0;
  for (int i = threadIdx.x; i < SP * K; i += blockDim.x) zh[i] = ZH[i];
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  const double th0 = sigH[0] * sigH[0];
  for (int k = warp; k < K; k += nwarps) {
    const double th = sigH[k] * sigH[k];
    double r2 = 0.0;
    for (int i = lane; i < n; i += 32) {
      double x = 0.0, gx = 0.0;
#pragma unroll 8
      for (int c = 0; c < SP; ++c) {
        x = fma(Qg[(size_t)c * n + i], zh[k * SP + c], x);
        gx = fma(Wg[(size_t)c * n + i], zh[k * SP + c], gx);
      }
      Zout[(size_t)k * n + i] = x;
      const double d = gx - th * x;
      r2 = fma(d, d, r2);
    }
    r2 = warp_sum(r2);
    if (lane == 0) res[k] = sqrt(r2);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int ok = isfinite(th0) && th0 > 0.0;
    for (int k = 0; k < K; ++k) ok = ok && isfinite(res[k]) && res[k] <= tol * th0;
    bad = !ok;
    *gate = bad;  // 1: run the full solver
  }
  __syncthreads();
  if (!bad)
    for (int k = threadIdx.x; k < K; k += blockDim.x) sigma_out[k] = sigH[k];
}

}  // namespace

bool subspace_supported(int n, int K) { return K <= SS_KMAX && n >= 2 * SP && n <= EIG_FAST_NMAX; }

size_t subspace_workspace_doubles(int n) {
  // Q, W (n x SP), H (SP x SP), eig(H) workspace, sigma(H), status
  return 2 * (size_t)n * SP + SP * SP + eig_workspace_doubles(SP, SS_KMAX) + SP + 8;
}

void launch_subspace_eig(const double* G, int n, int K, double* ss_ws, double* Zout, double* sigma_out, int* gate,
                         cudaStream_t st) {
  double* Qg = ss_ws;
  double* Wg = Qg + (size_t)n * SP;
  double* Hg = Wg + (size_t)n * SP;
  double* hws = Hg + SP * SP;
  double* sigH = hws + eig_workspace_doubles(SP, SS_KMAX);
  int* hstat = reinterpret_cast<int*>(sigH + SP);
  const int ldq = (n + 15) / 16 * 16 + 4;
  const size_t smem = sizeof(double) * (2 * (size_t)SP * ldq + SP);
  cudaFuncSetAttribute(ss_iterate_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  ss_iterate_kernel<<<1, SS_THREADS, smem, st>>>(G, n, K, SS_ITERS, Qg, Wg, Hg);
  cudaMemsetAsync(hstat, 0, sizeof(int), st);
  // (measured alternatives for this 32 x 32 Rayleigh-Ritz solve, both slower than the general solver's
  // 0.18 ms: the one-CTA one-sided Jacobi 0.26 ms, a one-warp cyclic two-sided Jacobi 1.2 ms)
  launch_eig_topk(Hg, SP, K, nullptr, hws /* W unused in split mode */, sigH, hws, hstat, nullptr, st, 0.0, 1);
  const double* ZH = hws + (size_t)SP * (SP + 1) / 2;
  ss_finish_kernel<<<1, SS_THREADS, 0, st>>>(n, K, Qg, Wg, ZH, sigH, SS_TOL, Zout, sigma_out, gate);
}

}  // namespace psvd
