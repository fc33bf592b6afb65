// Timing / convergence probe of the one-CTA Jacobi SVD (diagnostics).
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include "../paper_2108_08845_b200/csrc/psvd_small.cuh"
using namespace psvd;
int main() {
  for (int n : {20, 210}) {
    const int l = 20;
    for (int cond : {0, 8, 16}) {
      std::vector<double> h((size_t)n * l);
      srand(1);
      // columns with geometric scales 10^(-cond * k / l)
      for (int c = 0; c < l; ++c)
        for (int r = 0; r < n; ++r) h[(size_t)c * n + r] = (rand() / (double)RAND_MAX - 0.5) * pow(10.0, -cond * (double)c / l);
      if (n == l) {  // symmetric PSD: G = X^T X
        std::vector<double> g((size_t)l * l, 0.0);
        for (int i = 0; i < l; ++i) for (int j = 0; j < l; ++j) { double s = 0; for (int r = 0; r < l; ++r) s += h[(size_t)i * l + r] * h[(size_t)j * l + r]; g[(size_t)j * l + i] = s; }
        h = g;
      }
      double *dZ, *dS, *dJ, *dws; int* dst;
      cudaMalloc(&dZ, h.size() * 8); cudaMalloc(&dS, l * 8); cudaMalloc(&dJ, l * l * 8); cudaMalloc(&dws, (size_t)n * (l + 2) * 8); cudaMalloc(&dst, 4);
      cudaMemcpy(dZ, h.data(), h.size() * 8, cudaMemcpyHostToDevice); cudaMemset(dst, 0, 4);
      cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
      launch_jacobi_svd(dZ, n, l, dS, dJ, dws, dst, 0);
      cudaEventRecord(e0);
      launch_jacobi_svd(dZ, n, l, dS, dJ, dws, dst, 0);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      int st; cudaMemcpy(&st, dst, 4, cudaMemcpyDeviceToHost);
      double s[64]; cudaMemcpy(s, dS, l * 8, cudaMemcpyDeviceToHost);
      printf("n=%d l=%d cond=1e%d: %.1f us status=%d s0=%.3e s_last=%.3e err=%s\n", n, l, cond, ms * 1e3, st, s[0], s[l - 1], cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
