// Internal to libpsvd.so: the context behind the opaque psvd_ctx handle of include/psvd.h, a planned
// tall pass, and the host helpers the C-ABI translation units share (psvd_api.cu, psvd_stream.cu,
// psvd_rand_api.cu, psvd_dense.cu).  Not part of the boundary.
#pragma once
#include <cstdint>
#include <string>
#include <utility>
#include <vector>

#include "../../include/psvd.h"
#include "psvd_small.cuh"
#include "psvd_gemm.cuh"
#include "psvd_tall.cuh"

using namespace psvd;

struct Buf {
  void* ptr = nullptr;
  size_t bytes = 0;
};

constexpr int SMEM_LIMIT = 227 * 1024;

struct psvd_ctx {
  int device = 0;
  int num_sms = 148;
  std::string err;
  int* d_status = nullptr;  // device status word
  int* d_gate = nullptr;
  long long* d_timers = nullptr;  // eig phase clocks (diagnostics)
  int* h_status = nullptr;  // pinned
  long long launches = 0;   // kernels enqueued by this context (bench evidence)
  long long path_count[5] = {0, 0, 0, 0, 0};  // narrow TMA, TMA Gram, cp.async Gram, general, wide route
  double drift_tol = 1e-8;  // streaming.py:25 ORTHO_DRIFT_TOL (psvd_set_drift_tol overrides, e.g. to force the rescue)
  Buf partial, tiles, gram, eigws, wbuf, utu, tbuf, dvec, colmax;
  Buf ybuf, rsmall, jacws;  // randomized path: sketch Y (M x l), small matrices, Jacobi scratch
  Buf ybuf2;                // wide randomized path: second sketch buffer (Y T1 out of place)
  Buf xpairs;               // row-partitioned sign rule: local and gathered argmax pairs
  Buf ssws;                 // subspace-iteration core solve: Q, W, H, eig(H) scratch
  int* d_ssgate = nullptr;  // 1: the subspace path did not converge, run the full solver
  psvd_allreduce_fn ex_allreduce = nullptr;  // row-partitioned randomized update (psvd_set_exchange)
  psvd_allgather_fn ex_allgather = nullptr;
  void* ex_user = nullptr;
  int ex_nranks = 1;
  int64_t ex_row_offset = 0;
  Buf partial2, tiles2[2];  // A^T A passes on the low-priority stream (double-buffered tiles)
  Buf zbuf, rs2;            // pipelined randomized stream: look-ahead sketch Z = A Omega_A, small matrices
  Buf dense, dense2;        // dense utilities (psvd_qr / psvd_jacobi): small factors, a tall temporary
  Buf bigws, bigjac;        // any-width Cholesky / Jacobi workspaces (psvd_big.cu)
  Buf accws, accq;          // accurate R-factor route of the deterministic update: small factors, tall Q
  void* nccl_comm = nullptr;  // NCCL data plane of the exchange points (psvd_nccl.cu)
  bool nccl_on = false;
  int nccl_nranks = 1, nccl_rank = 0;
  Buf nccl_parts;             // allgather landing buffer of the rank-ordered sums
  long long ex_calls = 0, ex_bytes = 0;  // collectives issued / bytes received at the exchange points
  // in-step timing of the look-ahead A^T A Gram launches of psvd_stream_run (psvd_gram_timing):
  // event pairs on the low-priority stream around each batch's Gram sub-launches
  bool timing_on = false;
  std::vector<cudaEvent_t> tev;
  int tev_used = 0;
  double timed_flops = 0.0;
  cudaEvent_t ev_qready = nullptr;  // pipelined randomized stream: the sketch basis of the last update is final
  cudaStream_t s_hi = nullptr, s_lo = nullptr;  // pipelined stream_run: critical chain / look-ahead Grams
  cudaStream_t s_aux = nullptr;                  // concurrent LDL^T of the split core solve
  cudaEvent_t ev_ldlt_fork = nullptr, ev_ldlt_join = nullptr, ev_eig_start = nullptr;
  cudaEvent_t ev_fdone = nullptr;  // psvd_stream_run: the fused pass kernel of an update has left the SMs
  cudaEvent_t ev_aa[2] = {nullptr, nullptr}, ev_asm[2] = {nullptr, nullptr}, ev_fork = nullptr, ev_join = nullptr;
};

// A planned tall pass: params + reduce map + grid.
struct Pass {
  TallParams p;
  ReduceMap map;
  int grid = 0;
  int NB = 0;
  bool ws = false;      // warp-specialized Gram kernel
  bool tma = false;     // warp-specialized TMA pass (narrow panels)
  bool gtma = false;    // TMA-fed Gram-only pass
  TmaMaps maps;
  TmaExtra x;
  Buf* part = nullptr;  // partial-tile workspace of the stream this pass runs on
  Buf* tl = nullptr;    // reduced tiles
  bool fsplit = false;  // split-ring fused pass (fused_split_kernel) instead of the narrow TMA pass
  FusedSplit fs;
  TmaMaps maps3;        // its 3-D tensor maps
  ReduceMap offmap;     // its offloaded Gram tiles (reduced into the look-ahead Gram's tile array)
};

namespace psvd_internal {

int fail(psvd_ctx* c, int code, const char* fmt, ...);
int cuda_check(psvd_ctx* c, const char* what);
int ensure(psvd_ctx* c, Buf& b, size_t bytes);  // grow-only workspace (growth synchronizes)
inline int rup(int x, int m) { return (x + m - 1) / m * m; }
bool aligned16(const void* p);
int check_mat(psvd_ctx* c, const char* name, const double* p, int64_t ld, int64_t M, int cols);
// Common pass setup.  segs: panel segments; w/W: optional Y = P[:, wlo:wlo+wk] * W.
int plan_pass(psvd_ctx* c, Pass& ps, int64_t M, const std::vector<Seg>& segs, int wlo, int wk, int w,
              const double* W, int64_t ldw, bool gram_pp, bool gram_yy, bool gram_py, int py_cols = -1,
              int pp_rows = -1, Buf* part = nullptr, Buf* tl = nullptr, int max_ctas = 0, int py_lo = 0,
              bool gaps_ok = false, const std::vector<std::pair<int, int>>* skip_pp = nullptr);
int run_pass(psvd_ctx* c, Pass& ps, cudaStream_t st);
// Split-ring variant of a planned fused pass [U | A_b | A_next] (psvd_tall.cuh: FusedSplit): sets ps.fsplit
// when it qualifies; off = 32-column block pairs of A_next^T A_next to compute in the pass (off_nb tile
// columns in the look-ahead Gram's tile array).  run_fused_split launches it and both reductions.
bool try_fused_split(psvd_ctx* c, Pass& ps, const std::vector<std::pair<int, int>>& off, int off_nb);
int run_fused_split(psvd_ctx* c, Pass& ps, cudaStream_t st, double* off_tiles);
int make_dvec(psvd_ctx* c, const double* sigma, double ff, int Kc, int n, cudaStream_t st);
std::vector<Seg> panel(const double* U, int64_t ldu, int Kc, const double* A, int64_t lda, int B);
void launch_stamp(unsigned long long* out, cudaStream_t st);  // device clock into *out (trace marks)
// Core solve of a Gram: eig (+ concurrent LDL^T on the aux stream when the split path applies)
int core_solve(psvd_ctx* c, const double* G, int n, int K, const double* dscale, double* W, double* sigma,
               cudaStream_t st, long long* timers);
// sigma_k <- ||C v_k|| and unit columns (Rayleigh refinement), UtU normalized in place
int refine_normalize(psvd_ctx* c, int64_t M, double* U, int64_t ld, int K, double* UtU, double* sigma,
                     cudaStream_t st);
// drift rescue beyond the one-CTA check (K > DRIFT_SMEM_KMAX): host-checked, psvd_qr based
int drift_rescue_wide(psvd_ctx* c, int64_t M, double* U, int64_t ldu, int K, const double* UtU, double* sigma,
                      double tol, cudaStream_t st);
// exchange points of the row-partitioned updates (no-ops on one GPU): NCCL in-stream when a
// communicator is enabled, else the caller's hooks
int ex_allreduce(psvd_ctx* c, double* buf, int64_t count, cudaStream_t st);
bool ex_active(const psvd_ctx* c);  // a row-partitioned exchange is set (NCCL or hooks)
int nccl_allgather(psvd_ctx* c, const double* send, int64_t count, double* recv, cudaStream_t st);
int nccl_allreduce_ordered(psvd_ctx* c, double* buf, int64_t count, cudaStream_t st);
// Cholesky R and R^-1 of an n x n Gram for any n (the one-CTA kernel up to CHOL_NMAX, psvd_big.cu beyond)
int chol_any(psvd_ctx* c, const double* G, int n, double* T, int* illcond, int* status, double* Rout,
             cudaStream_t st);
// one-sided Jacobi SVD for any n (psvd_big.cu): S, V (ld ldv), optional U = X V S^-1 (ld ldu)
int jacobi_any(psvd_ctx* c, const double* X, int64_t ldx, int64_t m, int n, int transpose, double* S, double* V,
               int64_t ldv, double* U, int64_t ldu, cudaStream_t st);

}  // namespace psvd_internal
