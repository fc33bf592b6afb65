// C ABI of the pipelined deterministic stream (include/psvd.h: psvd_stream_run, the reference's
// stream_all, streaming.py:119-133, and the row-partitioned stream of dsvd.py:205-242).
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

namespace {

// Deferred normalization (psvd_stream_run): the previous update's U is left as the fused pass wrote
// it, U_raw, and U = U_raw diag(scale) T (T the drift rescue's transform when its gate fired, else
// I).  The panel product [U | A] W then equals [U_raw | A] W' with the top K rows of W replaced by
// diag(scale) T W_top: one CTA, fixed summation order.
__global__ void fold_w_kernel(double* W, int64_t ldw, int K, const double* scale, const double* T, const int* gate) {
  extern __shared__ double wt[];  // K x K, col-major
  const bool rot = gate != nullptr && *gate != 0;
  for (int i = threadIdx.x; i < K * K; i += blockDim.x) wt[i] = W[(int64_t)(i / K) * ldw + i % K];
  __syncthreads();
  for (int i = threadIdx.x; i < K * K; i += blockDim.x) {
    const int r = i % K, col = i / K;
    double v = wt[i];
    if (rot) {
      v = 0.0;
      for (int l = 0; l < K; ++l) v += T[(int64_t)l * K + r] * wt[col * K + l];
    }
    W[(int64_t)col * ldw + r] = scale[r] * v;
  }
}

}  // namespace

extern "C" {

// Whole stream with look-ahead: the A^T A Gram of batch b+1 runs on a
// low-priority stream (one SM left free) while the one-CTA core solve of batch
// b runs on the high-priority stream; U^T [U | A_{b+1}] is a narrow pass after
// the recompose.  Same arithmetic as psvd_stream_update per batch.
int psvd_stream_run(psvd_ctx* c, int64_t M, const double* U_in, int64_t ldu, const double* sigma_in, int Kc,
                    int nb, const double* const* A, const int64_t* lda, const int* B, int K, double ff, int rescue,
                    double* U_a, double* U_b, int64_t ldo, double* sigma_hist, int* final_buf, void* const* batch_ready, void* stream) {
  if (!c || nb < 1 || !A || !lda || !B || !U_a || !U_b || !sigma_hist || !final_buf)
    return fail(c, PSVD_EINVAL, "bad stream_run arguments");
  if (Kc != 0 && Kc != K) return fail(c, PSVD_EINVAL, "initial state carries %d modes, K=%d", Kc, K);
  if (Kc > 0 && (!U_in || !sigma_in)) return fail(c, PSVD_EINVAL, "null initial state");
  if (U_in == U_a) return fail(c, PSVD_EINVAL, "U_in must not alias U_a");
  int rc;
  for (int b = 0; b < nb; ++b) {
    if ((rc = check_mat(c, "A", A[b], lda[b], M, B[b]))) return rc;
    if (B[b] < 1) return fail(c, PSVD_EINVAL, "empty batch");
  }
  if ((rc = check_mat(c, "U_a", U_a, ldo, M, K)) || (rc = check_mat(c, "U_b", U_b, ldo, M, K))) return rc;
  if (Kc == 0 && B[0] < K) return fail(c, PSVD_EINVAL, "initial batch has %d columns, need at least k_modes=%d", B[0], K);
  int nmax = 0;
  for (int b = 0; b < nb; ++b) nmax = std::max(nmax, K + B[b]);
  if ((rc = ensure(c, c->gram, sizeof(double) * (size_t)nmax * nmax))) return rc;
  if ((rc = ensure(c, c->wbuf, sizeof(double) * (size_t)nmax * K))) return rc;
  if ((rc = ensure(c, c->utu, sizeof(double) * (size_t)K * K))) return rc;
  if ((rc = ensure(c, c->dvec, sizeof(double) * (size_t)nmax))) return rc;
  if ((rc = ensure(c, c->eigws, sizeof(double) * eig_workspace_doubles(nmax, K)))) return rc;
  if ((rc = ensure(c, c->tbuf, sizeof(double) * ((size_t)K * K + K)))) return rc;
  cudaStream_t user = (cudaStream_t)stream, hi = c->s_hi, lo = c->s_lo;
  // PSVD_TRACE=1: timeline of the two streams on stderr (diagnostics; %globaltimer stamps)
  static const bool trace = getenv("PSVD_TRACE") != nullptr;
  std::vector<std::string> tl;
  unsigned long long* tbuf = nullptr;
  if (trace) cudaMallocManaged(&tbuf, 256 * sizeof(unsigned long long));
  auto mark = [&](const char* what, int b, cudaStream_t s_) {
    if (!trace || tl.size() >= 256) return;
    launch_stamp(tbuf + tl.size(), s_);
    tl.push_back(std::string(what) + "[" + std::to_string(b) + "]");
  };
  mark("start", 0, user);
  cudaEventRecord(c->ev_fork, user);
  cudaStreamWaitEvent(hi, c->ev_fork, 0);
  cudaStreamWaitEvent(lo, c->ev_fork, 0);
  double* G = (double*)c->gram.ptr;
  double* W = (double*)c->wbuf.ptr;
  double* UtU = (double*)c->utu.ptr;
  double* bufs[2] = {U_a, U_b};
  int nbaa[2] = {0, 0};
  int nbua = 0, fused_a0 = 0, fused_y = 0;
  bool prev_resc = false;
  // A^T A of batch j on the low-priority stream into tiles2[j & 1]
  // The look-ahead Gram is cut into row sub-ranges launched back to back: CTAs of a
  // low-priority kernel cannot be preempted, so short launches let the high-priority
  // recompose / U^T A passes take the SMs between them.  All sub-ranges write disjoint
  // partial sets and one fixed-order reduction sums them (bitwise reproducible).
  // The fused pass of batch b waits for the look-ahead Gram of b+1 rather than time-sharing SMs with it
  // (both kernels hold whole SMs, so sharing bought nothing: 9.04 vs 9.10 ms per config-2 step, and it
  // cut the Gram's in-step rate from 29.9 to 21 TF/s); the Gram runs as one launch on all SMs but the one
  // the core solve of batch b occupies.  PSVD_LA_SHARED=1 restores the time-shared schedule (4 row
  // sub-launches on num_sms - 2 CTAs).
  static const bool la_serial = getenv("PSVD_LA_SHARED") == nullptr;
  // Between an update's fused pass and the next look-ahead Gram only one-CTA kernels remain when the
  // column normalization (and a fired drift rescue) of U is folded into the next update's W instead of
  // rewriting U (fold_w_kernel): the Gram then starts as soon as the fused pass leaves the SMs and the
  // one-CTA tail runs on the SM it leaves free.  PSVD_NO_DEFER_NORM=1: normalize U in place.
  static const bool defer_env = getenv("PSVD_NO_DEFER_NORM") == nullptr;
  const bool defer = defer_env && la_serial && K <= DRIFT_SMEM_KMAX;
  const int nsub = la_serial ? 1 : (int)std::max<int64_t>(1, std::min<int64_t>(4, M / 65536));
  const int la_ctas = la_serial ? c->num_sms - 1 : c->num_sms - 2;
  // Fused passes planned up front: the ones that qualify run on the split-ring kernel (32-row 3-D boxes,
  // psvd_tall.cuh: FusedSplit), which also computes a few 32 x 32 tiles of the next batch's A^T A; the
  // look-ahead Gram of that batch then skips them (skip_pp[j]).  PSVD_NO_FSPLIT=1: the narrow TMA pass for
  // all of them; PSVD_FS_NOFF=n: tiles taken off the Gram (default 3).
  static const int fs_noff = getenv("PSVD_FS_NOFF") ? std::max(0, std::min(FS_MAX_OFF, atoi(getenv("PSVD_FS_NOFF")))) : 3;
  std::vector<Pass> fpass(nb > 1 ? nb - 1 : 0);
  std::vector<std::vector<std::pair<int, int>>> skip_pp(nb);
  for (int b = 0; b + 1 < nb; ++b) {
    const int kc = (b == 0) ? Kc : K;
    const double* up = b == 0 ? (Kc > 0 ? U_in : nullptr) : bufs[(b - 1) & 1];
    const int64_t ldp = b == 0 ? (Kc > 0 ? ldu : 0) : ldo;
    std::vector<Seg> segs = panel(up, ldp, kc, A[b], lda[b], B[b]);
    segs.push_back(Seg{A[b + 1], lda[b + 1], B[b + 1], 1});
    const int wk = kc + B[b];
    static const int fused_ctas = getenv("PSVD_FUSED_CTAS") ? atoi(getenv("PSVD_FUSED_CTAS")) : 0;
    if ((rc = plan_pass(c, fpass[b], M, segs, 0, wk, K, W, wk, false, true, true, -1, -1, nullptr, nullptr, fused_ctas, -1)))
      return rc;
    // full off-diagonal blocks (0,1), (2,3), ... of A_{b+1}^T A_{b+1}
    std::vector<std::pair<int, int>> off;
    const int nfull = B[b + 1] / 32;
    for (int t = 0; 2 * t + 1 < nfull && (int)off.size() < fs_noff; ++t) off.push_back({2 * t, 2 * t + 1});
    if (la_serial && try_fused_split(c, fpass[b], off, (B[b + 1] + 31) / 32))
      for (int o = 0; o < fpass[b].offmap.nout; ++o)
        skip_pp[b + 1].push_back({fpass[b].offmap.out_id[o] / ((B[b + 1] + 31) / 32), fpass[b].offmap.out_id[o] % ((B[b + 1] + 31) / 32)});
  }
  auto aa_pass = [&](int j) -> int {
    if (j >= 2) cudaStreamWaitEvent(lo, c->ev_asm[j & 1], 0);  // tiles2[j&1] consumed by batch j-2's assembly
    // start A^T A of batch j with the core solve of batch j-1: it then overlaps that one-SM
    // solve (the longer of the two) instead of competing with the recompose pass for SMs.  With the
    // deferred normalization it only waits for the fused pass of batch j-2 to leave the SMs: the
    // one-CTA tail of that update (extract, Rayleigh refinement, drift check) and the assembly of
    // batch j-1 then run on the SM the Gram leaves free
    if (j >= 2 && defer)
      cudaStreamWaitEvent(lo, c->ev_fdone, 0);
    else if (j >= 1)
      cudaStreamWaitEvent(lo, c->ev_eig_start, 0);
    if (batch_ready && batch_ready[j]) cudaStreamWaitEvent(lo, (cudaEvent_t)batch_ready[j], 0);
    const int64_t rows_sub = (M + nsub - 1) / nsub / 32 * 32 + 32;
    Pass first;
    size_t part_off = 0;
    int nchunks_total = 0;
    mark("lo:aa_begin", j, lo);
    cudaEvent_t te1 = nullptr;
    if (c->timing_on && c->tev_used + 2 <= (int)c->tev.size()) {
      cudaEventRecord(c->tev[c->tev_used], lo);
      te1 = c->tev[c->tev_used + 1];
      c->tev_used += 2;
      // upper triangle of A^T A (DMMA tiles), less the 32 x 32 tiles the split-ring fused pass computes
      c->timed_flops += (double)M * B[j] * (B[j] + 1) - 2048.0 * M * skip_pp[j].size();
    }
    for (int k = 0; k < nsub; ++k) {
      const int64_t r0 = (int64_t)k * rows_sub;
      if (r0 >= M) break;
      const int64_t mk = std::min(M, r0 + rows_sub) - r0;
      Pass pa;
      int r = plan_pass(c, pa, mk, {Seg{A[j] + r0, lda[j], B[j], 0}}, 0, 0, 0, nullptr, 0, true, false, false, -1,
                        -1, &c->partial2, &c->tiles2[j & 1], la_ctas, 0, false, skip_pp[j].empty() ? nullptr : &skip_pp[j]);
      if (r) return r;
      const size_t need = part_off + (size_t)pa.grid * SLOTS * 1024;
      if (k == 0) {  // size the partial buffer for all sub-ranges once
        if ((r = ensure(c, c->partial2, sizeof(double) * need * nsub))) return r;
        first = pa;
      }
      pa.p.partial = (double*)c->partial2.ptr + part_off;
      c->path_count[pa.gtma ? 1 : pa.ws ? 2 : 3]++;
      if (pa.gtma)
        launch_gram_tma(pa.p, pa.maps, pa.x, pa.grid, lo);
      else if (pa.ws)
        launch_gram_ws(pa.p, pa.grid, lo);
      else
        launch_tall(pa.p, pa.grid, lo);
      c->launches++;
      if ((r = cuda_check(c, "look-ahead gram"))) return r;
      part_off += (size_t)pa.grid * SLOTS * 1024;
      nchunks_total += pa.map.nchunks;
    }
    if (te1) cudaEventRecord(te1, lo);
    first.map.nchunks = nchunks_total;
    launch_tall_reduce((const double*)c->partial2.ptr, first.map, (double*)c->tiles2[j & 1].ptr, lo);
    c->launches++;
    nbaa[j & 1] = first.NB;
    mark("lo:aa_end", j, lo);
    cudaEventRecord(c->ev_aa[j & 1], lo);
    return cuda_check(c, "look-ahead reduce");
  };
  if ((rc = aa_pass(0))) return rc;
  const double* Uprev = Kc > 0 ? U_in : nullptr;
  int64_t ldprev = Kc > 0 ? ldu : 0;
  const double* sprev = Kc > 0 ? sigma_in : nullptr;
  int cur = 0;
  bool prev_raw = false;  // Uprev = U_raw of the previous update (scale and T in c->tbuf)
  double* const tb_T = (double*)c->tbuf.ptr;
  double* const tb_scale = tb_T + (size_t)K * K;
  if (Kc > 0) {  // U^T [U | A_0] for the initial state
    if (batch_ready && batch_ready[0]) cudaStreamWaitEvent(hi, (cudaEvent_t)batch_ready[0], 0);
    Pass pu;
    if ((rc = plan_pass(c, pu, M, {Seg{U_in, ldu, K, 0}, Seg{A[0], lda[0], B[0], 0}}, 0, 0, 0, nullptr, 0, true,
                        false, false, -1, K)))
      return rc;
    nbua = pu.NB;
    if ((rc = run_pass(c, pu, hi))) return rc;
  }
  for (int b = 0; b < nb; ++b) {
    const int kc = (b == 0) ? Kc : K;
    const int n = kc + B[b];
    cudaStreamWaitEvent(hi, c->ev_aa[b & 1], 0);
    cudaEventRecord(c->ev_eig_start, hi);
    if (b + 1 < nb && (rc = aa_pass(b + 1))) return rc;
    mark("hi:eig_begin", b, hi);
    if ((rc = make_dvec(c, sprev, ff, kc, n, hi))) return rc;
    if (b == 0) {
      launch_assemble_gram((const double*)c->tiles.ptr, nbua, (const double*)c->tiles2[b & 1].ptr, nbaa[b & 1], kc,
                           B[b], (const double*)c->dvec.ptr, G, hi);
    } else {
      // row-partitioned (exchange hooks): U^T U is already the global, normalized Gram; the other
      // blocks are local.  Only the first rank keeps the U^T U block, so the rank-ordered sum
      // below reproduces it exactly
      const double uu_w = (ex_active(c) && c->ex_row_offset != 0) ? 0.0 : 1.0;
      const double* tb = (const double*)c->tbuf.ptr;
      launch_assemble_gram_fused((const double*)c->tiles.ptr, nbua, fused_a0, fused_y, UtU, tb + (size_t)K * K,
                                 prev_resc ? c->d_gate : nullptr, tb, (const double*)c->tiles2[b & 1].ptr,
                                 nbaa[b & 1], K, B[b], (const double*)c->dvec.ptr, G, hi, uu_w);
    }
    c->launches++;
    // row-partitioned: the streaming Gram is the rank-ordered sum of the local ones
    if ((rc = ex_allreduce(c, G, (int64_t)n * n, hi))) return rc;
    cudaEventRecord(c->ev_asm[b & 1], hi);
    double* sig_b = sigma_hist + (size_t)b * K;
    if ((rc = core_solve(c, G, n, K, (const double*)c->dvec.ptr, W, sig_b, hi, nullptr))) return rc;
    mark("hi:eig_end", b, hi);
    double* Uout = bufs[cur];
    const bool resc = rescue && kc > 0;
    if (prev_raw) {
      fold_w_kernel<<<1, 256, sizeof(double) * K * K, hi>>>(W, kc + B[b], K, tb_scale, tb_T,
                                                            prev_resc ? c->d_gate : nullptr);
      c->launches++;
    }
    if (b + 1 < nb) {
      // fused: U_b = [U_{b-1} | A_b] W, with U_b^T U_b and U_b^T A_{b+1} from the same pass
      if (batch_ready && batch_ready[b + 1]) cudaStreamWaitEvent(hi, (cudaEvent_t)batch_ready[b + 1], 0);
      if (la_serial) cudaStreamWaitEvent(hi, c->ev_aa[(b + 1) & 1], 0);
      Pass& pf = fpass[b];
      const int wk = kc + B[b];
      pf.p.partial = (double*)pf.part->ptr;  // the workspace may have grown since the plan
      const int a0 = pf.p.seg[pf.p.nseg - 1].col0 / 32;
      pf.p.Yout = Uout;
      pf.p.ldy = ldo;
      if (pf.fsplit) {
        if ((rc = run_fused_split(c, pf, hi, (double*)c->tiles2[(b + 1) & 1].ptr))) return rc;
      } else if ((rc = run_pass(c, pf, hi))) {
        return rc;
      }
      cudaEventRecord(c->ev_fdone, hi);
      if (getenv("PSVD_DUMP_FUSED")) {  // diagnostics: tiles + Y of the fused pass
        cudaStreamSynchronize(hi);
        std::vector<double> h((size_t)pf.NB * pf.NB * 1024), y((size_t)M * K);
        cudaMemcpy(h.data(), c->tiles.ptr, h.size() * 8, cudaMemcpyDeviceToHost);
        cudaMemcpy2D(y.data(), M * 8, Uout, ldo * 8, M * 8, K, cudaMemcpyDeviceToHost);
        char fn[256];
        snprintf(fn, sizeof(fn), "%s_%d.bin", getenv("PSVD_DUMP_FUSED"), b);
        FILE* f = fopen(fn, "wb");
        int hdr[4] = {pf.NB, a0, pf.p.np_pad / 32, (int)M};
        fwrite(hdr, 4, 4, f);
        fwrite(h.data(), 8, h.size(), f);
        fwrite(y.data(), 8, y.size(), f);
        std::vector<double> u((size_t)M * K, 0.0), wv((size_t)wk * K);
        if (kc > 0) cudaMemcpy2D(u.data(), M * 8, Uprev, ldprev * 8, M * 8, K, cudaMemcpyDeviceToHost);
        cudaMemcpy(wv.data(), W, wv.size() * 8, cudaMemcpyDeviceToHost);
        fwrite(u.data(), 8, u.size(), f);
        fwrite(wv.data(), 8, wv.size(), f);
        fclose(f);
      }
      launch_extract_sym((const double*)c->tiles.ptr, pf.NB, pf.p.np_pad, K, nullptr, UtU, hi);
      c->launches++;
      if ((rc = ex_allreduce(c, UtU, (int64_t)K * K, hi))) return rc;  // global U^T U
      nbua = pf.NB;
      fused_a0 = a0;
      fused_y = pf.p.np_pad / 32;
    } else {
      if ((rc = psvd_recompose(c, M, Uprev, ldprev, kc, A[b], lda[b], B[b], W, K, Uout, ldo, UtU, hi))) return rc;
      if ((rc = ex_allreduce(c, UtU, (int64_t)K * K, hi))) return rc;
    }
    if (defer && b + 1 < nb) {
      // Rayleigh refinement and the drift check without touching U: both fold into the next W
      launch_normalize_gram(UtU, K, sig_b, tb_scale, c->d_status, hi);
      c->launches++;
      if (resc) {
        launch_drift_check(UtU, K, c->drift_tol, sig_b, tb_T, c->d_gate, c->d_status, hi);
        c->launches++;
      }
      if ((rc = cuda_check(c, "deferred refine"))) return rc;
      prev_raw = true;
    } else {
      if ((rc = refine_normalize(c, M, Uout, ldo, K, UtU, sig_b, hi))) return rc;
      if (resc && (rc = psvd_drift_rescue(c, M, Uout, ldo, K, UtU, sig_b, c->drift_tol, hi))) return rc;
      prev_raw = false;
    }
    prev_resc = resc;
    mark("hi:recompose_end", b, hi);
    Uprev = Uout;
    ldprev = ldo;
    sprev = sig_b;
    *final_buf = cur;
    cur ^= 1;
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
  return cuda_check(c, "stream_run");
}

// In-step timing of the dominant kernel (bench roofline): mode 1 starts recording event pairs around
// every look-ahead A^T A Gram of psvd_stream_run; mode 0 stops, synchronizes and returns
// out3 = {summed milliseconds, launches timed, summed flops M B (B + 1)}.
int psvd_gram_timing(psvd_ctx* c, int mode, double* out3) {
  if (!c) return PSVD_EINVAL;
  if (mode == 1) {
    if (c->tev.empty()) {
      c->tev.resize(1024);
      for (auto& e : c->tev) cudaEventCreate(&e);
    }
    c->tev_used = 0;
    c->timed_flops = 0.0;
    c->timing_on = true;
    return cuda_check(c, "timing start");
  }
  c->timing_on = false;
  double ms = 0.0;
  for (int i = 0; i + 1 < c->tev_used; i += 2) {
    cudaEventSynchronize(c->tev[i + 1]);
    float t = 0.f;
    cudaEventElapsedTime(&t, c->tev[i], c->tev[i + 1]);
    ms += t;
  }
  if (out3) {
    out3[0] = ms;
    out3[1] = c->tev_used / 2;
    out3[2] = c->timed_flops;
  }
  return cuda_check(c, "timing read");
}

// 1 when psvd_stream_run can take batches of up to Bmax columns with K modes on M rows: its
// look-ahead Gram (one pass of 32x32 tiles) and its fused pass [U | A_b | A_{b+1}] plan within
// the kernels' limits; 0 otherwise (stream batch by batch through psvd_stream_update instead).
int psvd_stream_run_supported(psvd_ctx* c, int64_t M, int K, int Bmax, int* ok) {
  if (!c || !ok || M < 1 || K < 1 || Bmax < 1) return PSVD_EINVAL;
  *ok = 0;
  const int nb32 = (Bmax + 31) / 32;
  if (nb32 * (nb32 + 1) / 2 > MAX_OUT_TILES) return PSVD_OK;
  // dry-run plans on placeholder 16-byte aligned pointers (plans launch nothing)
  const double* fake = reinterpret_cast<const double*>(uintptr_t(1) << 20);
  const int64_t ld = M + (M & 1);
  Pass pa, pf;
  std::string saved = c->err;
  bool fit = plan_pass(c, pa, M, {Seg{fake, ld, Bmax, 0}}, 0, 0, 0, nullptr, 0, true, false, false) == PSVD_OK &&
             plan_pass(c, pf, M, {Seg{fake, ld, K, 0}, Seg{fake, ld, Bmax, 0}, Seg{fake, ld, Bmax, 1}}, 0, K + Bmax,
                       K, fake, K + Bmax, false, true, true, -1, -1, nullptr, nullptr, 0, -1) == PSVD_OK;
  c->err = saved;
  *ok = fit ? 1 : 0;
  return PSVD_OK;
}

}  // extern "C"
