// C ABI (include/psvd.h): context, workspace, pass planning and the update
// orchestration.  Everything is enqueued on the caller's stream; nothing here
// synchronizes with the host except psvd_read_status.
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>
#include <algorithm>
#include <cstdlib>

#include "../../include/psvd.h"
#include "psvd_small.cuh"
#include "psvd_gemm.cuh"
#include "psvd_tall.cuh"

using namespace psvd;

namespace {

struct Buf {
  void* ptr = nullptr;
  size_t bytes = 0;
};

constexpr int SMEM_LIMIT = 227 * 1024;

}  // namespace

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
  cudaEvent_t ev_qready = nullptr;  // pipelined randomized stream: the sketch basis of the last update is final
  cudaStream_t s_hi = nullptr, s_lo = nullptr;  // pipelined stream_run: critical chain / look-ahead Grams
  cudaStream_t s_aux = nullptr;                  // concurrent LDL^T of the split core solve
  cudaEvent_t ev_ldlt_fork = nullptr, ev_ldlt_join = nullptr, ev_eig_start = nullptr;
  cudaEvent_t ev_aa[2] = {nullptr, nullptr}, ev_asm[2] = {nullptr, nullptr}, ev_fork = nullptr, ev_join = nullptr;
};

namespace {

int fail(psvd_ctx* c, int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  if (c) c->err = buf;
  return code;
}

int cuda_check(psvd_ctx* c, const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(c, PSVD_ECUDA, "%s: %s", what, cudaGetErrorString(e));
  return PSVD_OK;
}

// Grow-only workspace.  Growth synchronizes the device (rare; warm-up sizes it).
int ensure(psvd_ctx* c, Buf& b, size_t bytes) {
  if (b.bytes >= bytes) return PSVD_OK;
  if (b.ptr) {
    cudaDeviceSynchronize();
    cudaFree(b.ptr);
    b.ptr = nullptr;
    b.bytes = 0;
  }
  size_t want = std::max<size_t>(bytes, 4096);
  if (cudaMalloc(&b.ptr, want) != cudaSuccess) {
    cudaGetLastError();
    return fail(c, PSVD_ECUDA, "workspace allocation of %zu bytes failed", want);
  }
  b.bytes = want;
  return PSVD_OK;
}

inline int rup(int x, int m) { return (x + m - 1) / m * m; }

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

int check_mat(psvd_ctx* c, const char* name, const double* p, int64_t ld, int64_t M, int cols) {
  if (cols == 0) return PSVD_OK;
  if (p == nullptr) return fail(c, PSVD_EINVAL, "%s is null", name);
  if (ld < M) return fail(c, PSVD_EINVAL, "%s: leading dimension %lld < rows %lld", name, (long long)ld, (long long)M);
  if (ld % 2 != 0) return fail(c, PSVD_EINVAL, "%s: leading dimension %lld must be even", name, (long long)ld);
  if (!aligned16(p)) return fail(c, PSVD_EINVAL, "%s: base pointer must be 16-byte aligned", name);
  return PSVD_OK;
}

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
};

// Fill the warp plans / reduce map for a tile list (I <= J, 32-col blocks of [P | Y]).
int plan_tiles(psvd_ctx* c, Pass& ps, const std::vector<std::pair<int, int>>& tiles, bool allow_ksplit,
               int warps_avail = NWARP) {
  const int nt = (int)tiles.size();
  memset(ps.p.plan, 0, sizeof(ps.p.plan));
  memset(&ps.map, 0, sizeof(ps.map));
  if (nt == 0) {
    ps.p.nslices = 1;
    return PSVD_OK;
  }
  if (nt > MAX_OUT_TILES) return fail(c, PSVD_EINVAL, "too many Gram tiles (%d)", nt);
  const int nwarp_needed = (nt + TPW - 1) / TPW;
  const int nslices = (nwarp_needed + warps_avail - 1) / warps_avail;
  if (nslices > MAX_SLICES) return fail(c, PSVD_EINVAL, "panel too wide (%d tiles)", nt);
  ps.p.nslices = nslices;
  const int per = (nt + nslices - 1) / nslices;
  ps.map.nout = nt;
  for (int s = 0; s < nslices; ++s) {
    const int t0 = s * per, t1 = std::min(nt, t0 + per);
    const int ns = t1 - t0;
    if (ns <= 0) continue;
    if (ns >= warps_avail) {
      for (int w = 0; w < warps_avail; ++w) {
        WarpPlan& wp = ps.p.plan[s][w];
        wp.ksplit = 1;
        wp.kpart = 0;
        for (int t = 0; t < TPW; ++t) {
          const int li = w + t * warps_avail;
          if (li < ns) {
            wp.ti[wp.ntile] = (signed char)tiles[t0 + li].first;
            wp.tj[wp.ntile] = (signed char)tiles[t0 + li].second;
            const int o = t0 + li;
            ps.map.src[o][ps.map.nsrc[o]++] = (unsigned char)(s * SLOTS + w * TPW + wp.ntile);
            wp.ntile++;
          }
        }
      }
    } else {
      int ksplit = 1;
      while (allow_ksplit && ksplit * 2 * ns <= warps_avail) ksplit *= 2;
      for (int w = 0; w < ns * ksplit; ++w) {
        WarpPlan& wp = ps.p.plan[s][w];
        const int li = w % ns;
        wp.ksplit = (unsigned char)ksplit;
        wp.kpart = (unsigned char)(w / ns);
        wp.ti[0] = (signed char)tiles[t0 + li].first;
        wp.tj[0] = (signed char)tiles[t0 + li].second;
        wp.ntile = 1;
        const int o = t0 + li;
        ps.map.src[o][ps.map.nsrc[o]++] = (unsigned char)(s * SLOTS + w * TPW);
      }
    }
  }
  for (int o = 0; o < nt; ++o) ps.map.out_id[o] = (short)(tiles[o].first * ps.NB + tiles[o].second);
  return PSVD_OK;
}

// Warp-specialized Gram: spread the tiles over (slice, SMSP) bins so that every SMSP's DMMA
// pipe gets the same number of 8x8 blocks per k-step (warp w issues on SMSP w % 4; a diagonal
// tile needs 10 of 16 blocks, a tile on the panel's last partial block fewer).  Longest-
// processing-time greedy; the kernel's pace is the busiest SMSP of the busiest slice.
static int plan_tiles_balanced(psvd_ctx* c, Pass& ps, const std::vector<std::pair<int, int>>& tiles, int np,
                                int ncons = NWARP - WS_PRODUCERS) {  // the last warps load
  const int nt = (int)tiles.size();
  const int nslices = (nt + ncons - 1) / ncons;
  if (nt > MAX_OUT_TILES || nslices > MAX_SLICES) return fail(c, PSVD_EINVAL, "panel too wide (%d tiles)", nt);
  memset(ps.p.plan, 0, sizeof(ps.p.plan));
  memset(&ps.map, 0, sizeof(ps.map));
  ps.p.nslices = nslices;
  ps.map.nout = nt;
  auto cost = [&](int I, int J) {
    const int na = std::min(4, (np - I * 32 + 7) / 8), nb = std::min(4, (np - J * 32 + 7) / 8);
    if (I != J) return na * nb;
    int k = 0;
    for (int a = 0; a < na; ++a) k += std::max(0, nb - a);
    return k;
  };
  std::vector<int> order(nt);
  for (int i = 0; i < nt; ++i) order[i] = i;
  std::stable_sort(order.begin(), order.end(), [&](int x, int y) {
    return cost(tiles[x].first, tiles[x].second) > cost(tiles[y].first, tiles[y].second);
  });
  // bins: (slice, smsp); slots of smsp q in a slice: warps q, q+4, q+8, q+12 below ncons
  std::vector<int> load(nslices * 4, 0), used(nslices * 4, 0), slice_load(nslices, 0);
  auto slots_of = [&](int q) { int k = 0; for (int w = q; w < ncons; w += 4) ++k; return k; };
  for (int o : order) {
    const int cst = cost(tiles[o].first, tiles[o].second);
    int best = -1;
    for (int b = 0; b < nslices * 4; ++b) {
      if (used[b] >= slots_of(b % 4)) continue;
      if (best < 0 || load[b] < load[best] || (load[b] == load[best] && slice_load[b / 4] < slice_load[best / 4]))
        best = b;
    }
    if (best < 0) return fail(c, PSVD_EINVAL, "tile balancing failed");
    const int sl = best / 4, q = best % 4;
    const int w = q + 4 * used[best];
    used[best]++;
    load[best] += cst;
    slice_load[sl] += cst;
    WarpPlan& wp = ps.p.plan[sl][w];
    wp.ksplit = 1;
    wp.kpart = 0;
    wp.ti[0] = (signed char)tiles[o].first;
    wp.tj[0] = (signed char)tiles[o].second;
    wp.ntile = 1;
    ps.map.src[o][ps.map.nsrc[o]++] = (unsigned char)(sl * SLOTS + w * TPW);
  }
  for (int o = 0; o < nt; ++o) ps.map.out_id[o] = (short)(tiles[o].first * ps.NB + tiles[o].second);
  return PSVD_OK;
}

// TMA pass: tiles on the Gram warps (after the 2*ncb Y warps), one tile each, no k-split.
static int plan_tiles_tma(psvd_ctx* c, Pass& ps, const std::vector<std::pair<int, int>>& tiles) {
  const int nt = (int)tiles.size();
  memset(ps.p.plan, 0, sizeof(ps.p.plan));
  memset(&ps.map, 0, sizeof(ps.map));
  // Y warps: 2 row blocks x ncb column blocks; with 32-row stages (M a multiple of 16) a second
  // set of warps takes the second 16-row half when the Gram tiles still fit one slice (3 Y warps
  // per SMSP instead of 1.5: the Y product is bound by each warp's load -> DMMA chains)
  const int nyo = 2 * (ps.p.w_pad / 8);
  static const bool no_yh = getenv("PSVD_NO_YH") != nullptr;
  const int yh = (!no_yh && ps.p.M % 16 == 0 && 2 * nyo + nt <= NWARP - 1) ? 2 : 1;
  ps.p.yh = yh;
  // register-resident W (32-row stages): column block x k part warps, most parts that fit
  const int ncb = ps.p.w_pad / 8;
  static const int kp_max = getenv("PSVD_YKP") ? atoi(getenv("PSVD_YKP")) : 4;
  const int kspan_est = rup(ps.p.wk, 8) + 8 * ps.p.nseg;  // physical k span, gaps included
  int ykp = 1;
  if (ps.p.M % 16 == 0)
    for (int kp = std::min(kp_max, 4); kp >= 2; --kp)
      if (ncb * kp + nt <= NWARP - 1 && ncb * kp >= nyo && (kspan_est / 4 + kp - 1) / kp <= 16) {
        ykp = kp;
        break;
      }
  ps.p.ykp = ykp;
  static const int cap = getenv("PSVD_TMA_SLICE_WARPS") ? atoi(getenv("PSVD_TMA_SLICE_WARPS")) : 0;  // diagnostics
  const int warp0 = ykp > 1 ? ncb * ykp : nyo * yh, nwarps = cap > 0 ? std::min(cap, NWARP - 1 - warp0) : NWARP - 1 - warp0;
  const int nslices = std::max(1, (nt + nwarps - 1) / nwarps);
  if (nt > MAX_OUT_TILES || nslices > MAX_SLICES) return fail(c, PSVD_EINVAL, "panel too wide (%d tiles)", nt);
  ps.p.nslices = nslices;
  ps.map.nout = nt;
  const int per = (nt + nslices - 1) / nslices;
  for (int o = 0; o < nt; ++o) {
    const int sl = o / per, w = warp0 + o % per;
    WarpPlan& wp = ps.p.plan[sl][w];
    wp.ksplit = 1;
    wp.kpart = 0;
    wp.ti[0] = (signed char)tiles[o].first;
    wp.tj[0] = (signed char)tiles[o].second;
    wp.ntile = 1;
    ps.map.src[o][ps.map.nsrc[o]++] = (unsigned char)(sl * SLOTS + w * TPW);
    ps.map.out_id[o] = (short)(tiles[o].first * ps.NB + tiles[o].second);
  }
  return PSVD_OK;
}

// Common pass setup.  segs: panel segments; w/W: optional Y = P[:, wlo:wlo+wk] * W.
int plan_pass(psvd_ctx* c, Pass& ps, int64_t M, const std::vector<Seg>& segs, int wlo, int wk, int w,
              const double* W, int64_t ldw, bool gram_pp, bool gram_yy, bool gram_py, int py_cols = -1,
              int pp_rows = -1, Buf* part = nullptr, Buf* tl = nullptr, int max_ctas = 0, int py_lo = 0,
              bool gaps_ok = false) {
  memset(&ps.p, 0, sizeof(ps.p));
  ps.part = part ? part : &c->partial;
  ps.tl = tl ? tl : &c->tiles;
  TallParams& p = ps.p;
  p.M = M;
  p.nseg = (int)segs.size();
  // Narrow passes (Y of <= 16 columns, Gram tiles only against Y) run on the TMA kernel,
  // whose segments start on 8-column boundaries; P-tiles at explicit blocks (py_lo >= 0)
  // need that layout to coincide with the contiguous one.
  static const bool no_tma = getenv("PSVD_NO_TMA") != nullptr;
  bool tma = !no_tma && w > 0 && w <= TMA_MAX_Y && !gram_pp && tma_available();
  auto layout = [&](int align) {
    int n_ = 0;
    for (size_t i = 0; i < segs.size(); ++i) {
      p.seg[i] = segs[i];
      n_ = (segs[i].col0 == 1) ? rup(n_, 32) : rup(n_, align);  // col0 == 1: start on a 32-column block
      p.seg[i].col0 = n_;
      n_ += segs[i].ncols;
    }
    return n_;
  };
  int np = layout(1);
  int pshift = 0;
  if (tma) {
    std::vector<int> c1(segs.size());
    for (size_t i = 0; i < segs.size(); ++i) c1[i] = p.seg[i].col0;
    const int np8 = layout(8);
    bool same = true;
    for (size_t i = 0; i < segs.size(); ++i) same = same && c1[i] == p.seg[i].col0;
    for (size_t i = 0; i < segs.size(); ++i)
      tma = tma && aligned16(segs[i].ptr) && segs[i].ld % 2 == 0 && segs[i].ncols > 0;
    bool use_gaps = true;
    // gaps_ok: the caller extracts by segment (p.seg[i].col0), so the gapped layout is fine
    if (gram_py && py_lo >= 0 && !same && !gaps_ok) {
      // P-tiles at fixed logical blocks: keep the contiguous layout, shifted right by pshift so
      // that every segment after the first starts on an 8-column boundary (the first one's box
      // starts out of bounds, zero filled)
      pshift = c1.size() > 1 ? (8 - c1[1] % 8) % 8 : 0;
      bool ok = c1.size() > 1;
      for (size_t i = 1; i < c1.size(); ++i) ok = ok && (c1[i] + pshift) % 8 == 0;
      if (!ok) tma = false;
      use_gaps = false;
    }
    // + 8 per 256-column box boundary: equal boxes may end up to 8 columns past the panel
    int nbig = 0;
    for (size_t i = 0; i < segs.size(); ++i) nbig += (segs[i].ncols + 7) / 256;
    const int pw = (use_gaps ? rup(np8, 32) : rup(np, 32) + 8) + 8 * nbig;
    if (tma && tma_pass_smem_bytes(pw, rup(wk, 8) + 8 * (int)segs.size(), rup(w, 8)) > (size_t)SMEM_LIMIT) {
      tma = false;
      pshift = 0;
    }
    if (tma && use_gaps) {
      np = np8;
    } else {
      np = layout(1);
    }
  }
  if (py_lo < 0) {  // P-tiles over the last segment (its own 32-column block)
    const Seg& l = p.seg[segs.size() - 1];
    py_lo = l.col0 / 32;
    py_cols = l.col0 + l.ncols;
  }
  p.np = np;
  int np_pad = rup(std::max(np, 1), 32);
  if (w > 0) np_pad = std::max(np_pad, rup(wlo + rup(wk, 4), 32));
  p.np_pad = np_pad;
  p.W = W;
  p.ldw = ldw;
  p.wlo = wlo;
  p.wk = wk;
  p.w = w;
  p.w_pad = w > 0 ? rup(w, 8) : 0;
  if (w > MAX_W) return fail(c, PSVD_EINVAL, "Y width %d exceeds %d", w, MAX_W);
  // stage height: 32 rows unless the smem budget forces 16 (the TMA pass has its own 16-row ring)
  p.ks = 32;
  p.nstage = 3;
  if (!tma) {
    if (tall_smem_bytes(32, np_pad, wk, w, 3) > (size_t)SMEM_LIMIT) p.nstage = 2;
    if (tall_smem_bytes(32, np_pad, wk, w, 2) > (size_t)SMEM_LIMIT) p.ks = 16;
    if (tall_smem_bytes(p.ks, np_pad, wk, w, p.nstage) > (size_t)SMEM_LIMIT)
      return fail(c, PSVD_EINVAL, "panel of %d columns (+%d) does not fit shared memory", np, w);
  }
  const int NBp = np_pad / 32, NBy = w > 0 ? rup(w, 32) / 32 : 0;
  ps.NB = NBp + NBy;
  std::vector<std::pair<int, int>> tiles;
  if (gram_pp)
    for (int I = 0; I < (pp_rows < 0 ? NBp : std::min(NBp, (pp_rows + 31) / 32)); ++I)
      for (int J = I; J < NBp; ++J) tiles.push_back({I, J});
  if (gram_py)
    for (int I = py_lo; I < (py_cols < 0 ? NBp : (py_cols + 31) / 32); ++I)
      for (int J = 0; J < NBy; ++J) tiles.push_back({I, NBp + J});
  if (gram_yy)
    for (int I = 0; I < NBy; ++I)
      for (int J = I; J < NBy; ++J) tiles.push_back({NBp + I, NBp + J});
  // narrow tiles: all Gram tiles end in the Y block and Y has <= 16 columns
  p.narrow = (w > 0 && w <= 16 && !gram_pp && !tiles.empty()) ? 1 : 0;
  // Gram-only passes with enough tiles run warp-specialized (one producer warp, no k-split)
  ps.ws = (w == 0 && (int)tiles.size() >= 8 &&
           gram_ws_smem_bytes(np_pad, 3) <= (size_t)SMEM_LIMIT);
  if (ps.ws && !no_tma && tma_available() && gram_tma_smem_bytes(np_pad) <= (size_t)SMEM_LIMIT) {
    // TMA-fed Gram when every segment already starts on an 8-column boundary
    bool ok = true;
    for (int i = 0; i < p.nseg; ++i)
      ok = ok && (p.seg[i].col0 & 7) == 0 && aligned16(p.seg[i].ptr) && p.seg[i].ld % 2 == 0 && p.seg[i].ncols > 0;
    ps.gtma = ok;
  }
  ps.tma = tma;
  if (tma) p.narrow = 1;
  int rc = tma ? plan_tiles_tma(c, ps, tiles)
               : ps.gtma ? plan_tiles_balanced(c, ps, tiles, np, TMA_GRAM_CONS)
               : ps.ws ? plan_tiles_balanced(c, ps, tiles, np) : plan_tiles(c, ps, tiles, w == 0);
  {
    static const char* dbg = getenv("PSVD_GRAM_DBG");
    p.dbg = dbg ? atoi(dbg) : 0;
  }
  if (rc) return rc;
  // grid: one CTA per SM (1 CTA/SM by smem), chunks of 32-row multiples
  const int64_t stages32 = (M + 31) / 32;
  const int ctas = max_ctas > 0 ? std::min(max_ctas, c->num_sms) : c->num_sms;
  int64_t nchunks = std::max<int64_t>(1, std::min<int64_t>(stages32, std::max(1, ctas / p.nslices)));
  int64_t rows = (stages32 + nchunks - 1) / nchunks * 32;
  nchunks = (M + rows - 1) / rows;
  p.rows_per_cta = rows;
  ps.grid = (int)(nchunks * p.nslices);
  ps.map.nchunks = (int)nchunks;
  ps.map.nslices = p.nslices;
  if (!tiles.empty()) {
    int rc2 = ensure(c, *ps.part, sizeof(double) * (size_t)ps.grid * SLOTS * 1024);
    if (rc2) return rc2;
    rc2 = ensure(c, *ps.tl, sizeof(double) * (size_t)ps.NB * ps.NB * 1024);
    if (rc2) return rc2;
    p.partial = (double*)ps.part->ptr;
  }
  if ((tma || ps.gtma) && tma_pass_prepare(p, ps.maps, ps.x, tma ? pshift : 0, tma) != 0)
    return fail(c, PSVD_ECUDA, "TMA descriptor setup failed");
  if (tma && tma_pass_smem_bytes(ps.x.pwidth, ps.x.kp_hi - ps.x.kp_lo, p.w_pad, ps.x.ns, ps.x.rb) > (size_t)SMEM_LIMIT)
    return fail(c, PSVD_EINVAL, "narrow pass ring of %d columns exceeds shared memory", ps.x.pwidth);
  return PSVD_OK;
}

int run_pass(psvd_ctx* c, Pass& ps, cudaStream_t st) {
  if (ps.p.Yout != nullptr && ps.p.nslices > 1)
    for (int i = 0; i < ps.p.nseg; ++i)
      if (ps.p.seg[i].ptr == ps.p.Yout)
        return fail(c, PSVD_EINVAL, "in-place pass with %d slices would race", ps.p.nslices);
  c->path_count[ps.tma ? 0 : ps.gtma ? 1 : ps.ws ? 2 : 3]++;
  if (ps.tma)
    launch_pass_tma(ps.p, ps.maps, ps.x, ps.grid, st);
  else if (ps.gtma)
    launch_gram_tma(ps.p, ps.maps, ps.x, ps.grid, st);
  else if (ps.ws)
    launch_gram_ws(ps.p, ps.grid, st);
  else
    launch_tall(ps.p, ps.grid, st);
  c->launches += 1 + (ps.map.nout > 0);
  int rc = cuda_check(c, "tall pass");
  if (rc) {
    char buf[400];
    snprintf(buf, sizeof(buf), " [%s pass: np=%d np_pad=%d w=%d wk=%d nseg=%d grid=%d pwidth=%d kspan=%d ns=%d smem=%zu]",
             ps.tma ? "narrow TMA" : ps.gtma ? "TMA Gram" : ps.ws ? "ws Gram" : "general", ps.p.np, ps.p.np_pad, ps.p.w,
             ps.p.wk, ps.p.nseg, ps.grid, ps.x.pwidth, ps.x.kp_hi - ps.x.kp_lo, ps.x.ns,
             ps.tma ? tma_pass_smem_bytes(ps.x.pwidth, ps.x.kp_hi - ps.x.kp_lo, ps.p.w_pad, ps.x.ns, ps.x.rb)
                    : tall_smem_bytes(ps.p.ks, ps.p.np_pad, ps.p.wk, ps.p.w, ps.p.nstage));
    c->err += buf;
    return rc;
  }
  if (ps.map.nout > 0) {
    launch_tall_reduce((const double*)ps.part->ptr, ps.map, (double*)ps.tl->ptr, st);
    rc = cuda_check(c, "tall reduce");
  }
  return rc;
}

__global__ void make_dvec_kernel(const double* __restrict__ sigma, double ff, int Kc, int n, double* d) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) d[i] = i < Kc ? ff * sigma[i] : 1.0;
}

int make_dvec(psvd_ctx* c, const double* sigma, double ff, int Kc, int n, cudaStream_t st) {
  int rc = ensure(c, c->dvec, sizeof(double) * (size_t)std::max(n, 1));
  if (rc) return rc;
  make_dvec_kernel<<<(n + 255) / 256, 256, 0, st>>>(sigma, ff, Kc, n, (double*)c->dvec.ptr);
  c->launches++;
  return cuda_check(c, "dvec");
}

std::vector<Seg> panel(const double* U, int64_t ldu, int Kc, const double* A, int64_t lda, int B) {
  std::vector<Seg> s;
  if (Kc > 0) s.push_back(Seg{U, ldu, Kc, 0});
  if (B > 0) s.push_back(Seg{A, lda, B, 0});
  return s;
}

__global__ void stamp_kernel(unsigned long long* out) {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  *out = t;
}

__global__ void scale_cols_any_kernel(double* __restrict__ X, int64_t ld, int64_t rows, int cols,
                                      const double* __restrict__ s, int invert) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int j = blockIdx.y;
  if (i >= rows || j >= cols) return;
  const double f = s[j];
  double& x = X[(size_t)j * ld + i];
  x = invert ? (f != 0.0 ? x / f : 0.0) : x * f;
}

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

__global__ void sum_ordered_kernel(const double* __restrict__ parts, int P, int64_t count, double* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= count) return;
  double s = 0.0;
  for (int r = 0; r < P; ++r) s += parts[(int64_t)r * count + i];
  out[i] = s;
}

// log(1 + exp(v)) exactly as numpy's logaddexp(0, v) branches (npy_logaddexp)
__device__ double logaddexp0(double v) {
  if (v == 0.0) return 0.6931471805599453;  // LOGE2
  return v > 0.0 ? v + log1p(exp(-v)) : log1p(exp(v));
}

__global__ void burgers_kernel(double* __restrict__ out, int64_t ldo, int64_t row0, int64_t rows, int64_t grid,
                               int col0, int cols, int n_snap, double length, double t_final, double re) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int j = blockIdx.y;
  if (i >= rows || j >= cols) return;
  const int64_t gi = row0 + i;
  const int gj = col0 + j;
  // numpy.linspace: fl(k * step) + start, last sample pinned to stop
  const double dx = length / (double)(grid - 1);
  const double x = (gi == grid - 1) ? length : (double)gi * dx;
  const double dt = n_snap > 1 ? t_final / (double)(n_snap - 1) : 0.0;
  const double t = (n_snap > 1 && gj == n_snap - 1) ? t_final : (double)gj * dt;
  const double expo = 0.5 * (log1p(t) - re / 8.0) + re * x * x / (4.0 * (t + 1.0));
  out[(int64_t)j * ldo + i] = (x / (t + 1.0)) * exp(-logaddexp0(expo));
}

}  // namespace

static int core_solve(psvd_ctx* c, const double* G, int n, int K, const double* dscale, double* W, double* sigma,
                      cudaStream_t st, long long* timers);
static int refine_normalize(psvd_ctx* c, int64_t M, double* U, int64_t ld, int K, double* UtU, double* sigma,
                            cudaStream_t st);

// ============================================================================ C ABI

extern "C" {

int psvd_version(void) { return 1; }

int psvd_create(int device, psvd_ctx** out) {
  if (!out) return PSVD_EINVAL;
  *out = nullptr;
  if (cudaSetDevice(device) != cudaSuccess) {
    cudaGetLastError();
    return PSVD_ECUDA;
  }
  psvd_ctx* c = new psvd_ctx();
  c->device = device;
  cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device);
  if (cudaMalloc(&c->d_status, 4 * sizeof(int)) != cudaSuccess || cudaMallocHost(&c->h_status, sizeof(int)) != cudaSuccess) {
    cudaGetLastError();
    delete c;
    return PSVD_ECUDA;
  }
  c->d_gate = c->d_status + 1;
  c->d_ssgate = c->d_status + 2;
  if (cudaMalloc(&c->d_timers, 16 * sizeof(long long)) != cudaSuccess) {
    cudaGetLastError();
    return PSVD_ECUDA;
  }
  cudaMemset(c->d_status, 0, 4 * sizeof(int));
  {
    int lo = 0, hi = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);  // numerically: hi <= lo (smaller = higher priority)
    cudaStreamCreateWithPriority(&c->s_hi, cudaStreamNonBlocking, hi);
    cudaStreamCreateWithPriority(&c->s_lo, cudaStreamNonBlocking, lo);
    cudaStreamCreateWithPriority(&c->s_aux, cudaStreamNonBlocking, hi);
    cudaEventCreateWithFlags(&c->ev_ldlt_fork, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&c->ev_ldlt_join, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&c->ev_eig_start, cudaEventDisableTiming);
    for (int i = 0; i < 2; ++i) {
      cudaEventCreateWithFlags(&c->ev_aa[i], cudaEventDisableTiming);
      cudaEventCreateWithFlags(&c->ev_asm[i], cudaEventDisableTiming);
    }
    cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&c->ev_qready, cudaEventDisableTiming);
  }
  cudaDeviceSynchronize();
  *out = c;
  return PSVD_OK;
}

int psvd_destroy(psvd_ctx* c) {
  if (!c) return PSVD_OK;
  cudaSetDevice(c->device);
  cudaDeviceSynchronize();
  Buf* bufs[] = {&c->partial, &c->tiles, &c->gram, &c->eigws, &c->wbuf, &c->utu, &c->tbuf, &c->dvec, &c->colmax,
                 &c->ybuf, &c->ybuf2, &c->xpairs, &c->ssws, &c->rsmall, &c->jacws, &c->partial2, &c->tiles2[0], &c->tiles2[1],
                 &c->zbuf, &c->rs2, &c->dense, &c->dense2};
  for (Buf* b : bufs)
    if (b->ptr) cudaFree(b->ptr);
  if (c->s_hi) cudaStreamDestroy(c->s_hi);
  if (c->s_lo) cudaStreamDestroy(c->s_lo);
  if (c->s_aux) cudaStreamDestroy(c->s_aux);
  if (c->ev_ldlt_fork) cudaEventDestroy(c->ev_ldlt_fork);
  if (c->ev_ldlt_join) cudaEventDestroy(c->ev_ldlt_join);
  if (c->ev_eig_start) cudaEventDestroy(c->ev_eig_start);
  for (int i = 0; i < 2; ++i) {
    if (c->ev_aa[i]) cudaEventDestroy(c->ev_aa[i]);
    if (c->ev_asm[i]) cudaEventDestroy(c->ev_asm[i]);
  }
  if (c->ev_fork) cudaEventDestroy(c->ev_fork);
  if (c->ev_join) cudaEventDestroy(c->ev_join);
  if (c->ev_qready) cudaEventDestroy(c->ev_qready);
  cudaFree(c->d_status);
  cudaFree(c->d_timers);
  cudaFreeHost(c->h_status);
  delete c;
  return PSVD_OK;
}

const char* psvd_last_error(psvd_ctx* c) { return c ? c->err.c_str() : "null context"; }

long long psvd_launch_count(psvd_ctx* c) { return c ? c->launches : -1; }

int psvd_set_exchange(psvd_ctx* c, psvd_allreduce_fn allreduce, psvd_allgather_fn allgather, void* user, int nranks,
                      int64_t row_offset) {
  if (!c) return PSVD_EINVAL;
  if ((allreduce == nullptr) != (allgather == nullptr) || nranks < 1 || row_offset < 0)
    return fail(c, PSVD_EINVAL, "bad exchange hooks");
  c->ex_allreduce = allreduce;
  c->ex_allgather = allgather;
  c->ex_user = user;
  c->ex_nranks = allreduce ? nranks : 1;
  c->ex_row_offset = allreduce ? row_offset : 0;
  return PSVD_OK;
}

int psvd_path_counters(psvd_ctx* c, long long* out5) {
  if (!c || !out5) return PSVD_EINVAL;
  for (int i = 0; i < 5; ++i) out5[i] = c->path_count[i];
  return PSVD_OK;
}

int psvd_last_core_path(psvd_ctx* c, int* full) {
  if (!c || !full) return PSVD_EINVAL;
  if (cudaMemcpy(full, c->d_ssgate, sizeof(int), cudaMemcpyDeviceToHost) != cudaSuccess)
    return cuda_check(c, "core path");
  return PSVD_OK;
}

int psvd_set_drift_tol(psvd_ctx* c, double tol) {
  if (!c) return PSVD_EINVAL;
  c->drift_tol = tol;
  return PSVD_OK;
}

int psvd_eig_phase_cycles(psvd_ctx* c, long long* out9) {
  if (!c || !out9) return PSVD_EINVAL;
  if (cudaMemcpy(out9, c->d_timers, 14 * sizeof(long long), cudaMemcpyDeviceToHost) != cudaSuccess)
    return cuda_check(c, "eig timers");
  return PSVD_OK;
}

int psvd_read_status(psvd_ctx* c, int* status, int reset, void* stream) {
  if (!c || !status) return PSVD_EINVAL;
  cudaStream_t st = (cudaStream_t)stream;
  cudaMemcpyAsync(c->h_status, c->d_status, sizeof(int), cudaMemcpyDeviceToHost, st);
  if (reset) cudaMemsetAsync(c->d_status, 0, sizeof(int), st);
  if (cudaStreamSynchronize(st) != cudaSuccess) return cuda_check(c, "read status");
  *status = *c->h_status;
  return cuda_check(c, "read status");
}

int psvd_gram(psvd_ctx* c, int64_t M, const double* U, int64_t ldu, const double* sigma, double ff, int Kc,
              const double* A, int64_t lda, int B, double* G, void* stream) {
  if (!c) return PSVD_EINVAL;
  cudaStream_t st = (cudaStream_t)stream;
  if (M < 1 || B < 0 || Kc < 0 || Kc + B < 1) return fail(c, PSVD_EINVAL, "bad shape M=%lld Kc=%d B=%d", (long long)M, Kc, B);
  int rc;
  if ((rc = check_mat(c, "U", U, ldu, M, Kc)) || (rc = check_mat(c, "A", A, lda, M, B))) return rc;
  if (Kc > 0 && sigma == nullptr) return fail(c, PSVD_EINVAL, "sigma is null");
  if (G == nullptr) return fail(c, PSVD_EINVAL, "G is null");
  const int n = Kc + B;
  const int nb32 = (n + 31) / 32;
  if (nb32 * (nb32 + 1) / 2 > MAX_OUT_TILES) {
    // too many 32x32 tiles for one pass: the tall-skinny TN GEMM (full n x n, split over rows),
    // [U | A]^T U and [U | A]^T A, then the d_i d_j scaling of the panel [ff U S | A]
    c->path_count[4]++;
    if ((rc = ensure(c, c->partial, sizeof(double) * tgemm_tn_partial_doubles(M, n, std::max(B, std::max(Kc, 1)),
                                                                              c->num_sms))))
      return rc;
    std::vector<GemmSeg> gp;
    if (Kc > 0) gp.push_back(GemmSeg{U, ldu, Kc});
    if (B > 0) gp.push_back(GemmSeg{A, lda, B});
    if ((rc = make_dvec(c, sigma, ff, Kc, n, st))) return rc;
    const double* d = Kc > 0 ? (const double*)c->dvec.ptr : nullptr;
    if (Kc > 0) {
      launch_tgemm_tn(M, gp.data(), (int)gp.size(), U, ldu, Kc, d, G, n, (double*)c->partial.ptr, c->num_sms, st);
      c->launches += 2;
    }
    if (B > 0) {
      launch_tgemm_tn(M, gp.data(), (int)gp.size(), A, lda, B, d, G + (size_t)Kc * n, n, (double*)c->partial.ptr,
                      c->num_sms, st);
      c->launches += 2;
    }
    if (Kc > 0) {
      launch_scale_cols(G, n, n, Kc, d, st);  // columns of the U block: d_j = ff sigma_j
      c->launches++;
    }
    return cuda_check(c, "wide gram");
  }
  Pass ps;
  if ((rc = plan_pass(c, ps, M, panel(U, ldu, Kc, A, lda, B), 0, 0, 0, nullptr, 0, true, false, false))) return rc;
  if ((rc = run_pass(c, ps, st))) return rc;
  if ((rc = make_dvec(c, sigma, ff, Kc, n, st))) return rc;
  launch_extract_sym((const double*)c->tiles.ptr, ps.NB, 0, n, (const double*)c->dvec.ptr, G, st);
  c->launches++;
  return cuda_check(c, "extract gram");
}

int psvd_sym_topk(psvd_ctx* c, const double* G, int n, int k, double* V, int64_t ldv, double* s, void* stream) {
  if (!c) return PSVD_EINVAL;
  cudaStream_t st = (cudaStream_t)stream;
  if (n < 1 || k < 1 || k > n) return fail(c, PSVD_EINVAL, "bad eig shape n=%d k=%d", n, k);
  if (!G || !V || !s || ldv < n) return fail(c, PSVD_EINVAL, "bad eig arguments");
  int rc;
  if ((rc = ensure(c, c->eigws, sizeof(double) * eig_workspace_doubles(n, k)))) return rc;
  double* ws = (double*)c->eigws.ptr;
  launch_eig_topk(G, n, k, nullptr, ws /* W unused */, s, ws, c->d_status, nullptr, st, 0.0, 1);
  cudaMemcpy2DAsync(V, ldv * sizeof(double), ws + (size_t)n * (n + 1) / 2, n * sizeof(double), n * sizeof(double), k,
                    cudaMemcpyDeviceToDevice, st);
  c->launches++;
  return cuda_check(c, "sym topk");
}

int psvd_tn_product(psvd_ctx* c, int64_t M, const double* A, int64_t lda, int n, const double* Y, int64_t ldy, int m,
                    double* X, int64_t ldx, void* stream) {
  if (!c) return PSVD_EINVAL;
  int rc;
  if (M < 1 || n < 1 || m < 1 || ldx < n || !X) return fail(c, PSVD_EINVAL, "bad tn_product shape");
  if ((rc = check_mat(c, "A", A, lda, M, n)) || (rc = check_mat(c, "Y", Y, ldy, M, m))) return rc;
  if ((rc = ensure(c, c->partial, sizeof(double) * tgemm_tn_partial_doubles(M, n, m, c->num_sms)))) return rc;
  const GemmSeg ga{A, lda, n};
  launch_tgemm_tn(M, &ga, 1, Y, ldy, m, nullptr, X, (int)ldx, (double*)c->partial.ptr, c->num_sms,
                  (cudaStream_t)stream);
  c->launches += 2;
  return cuda_check(c, "tn product");
}

int psvd_sign_by_peak(psvd_ctx* c, double* X, int64_t ld, int64_t rows, int cols, void* stream) {
  if (!c) return PSVD_EINVAL;
  cudaStream_t st = (cudaStream_t)stream;
  int rc;
  if ((rc = check_mat(c, "X", X, ld, rows, cols))) return rc;
  if (cols == 0) return PSVD_OK;
  const int64_t nch = colmax_rows_chunks(rows);
  if ((rc = ensure(c, c->colmax, sizeof(double) * (size_t)nch * cols * 2)) ||
      (rc = ensure(c, c->xpairs, sizeof(double) * (size_t)cols))) return rc;
  launch_colmax_rows(X, ld, rows, cols, 0, (double*)c->colmax.ptr, st);
  launch_colmax_sign((const double*)c->colmax.ptr, (int)nch, cols, (double*)c->xpairs.ptr, st);
  launch_scale_cols(X, ld, rows, cols, (const double*)c->xpairs.ptr, st);
  c->launches += 3;
  return cuda_check(c, "sign by peak");
}

int psvd_core_eig(psvd_ctx* c, const double* G, int n, const double* sigma_in, double ff, int Kc, int K, double* W,
                  double* sigma_out, void* stream) {
  if (!c) return PSVD_EINVAL;
  cudaStream_t st = (cudaStream_t)stream;
  if (n < 1 || K < 1 || K > n || Kc < 0 || Kc > n) return fail(c, PSVD_EINVAL, "bad core shape n=%d K=%d Kc=%d", n, K, Kc);
  if (!G || !W || !sigma_out || (Kc > 0 && !sigma_in)) return fail(c, PSVD_EINVAL, "null pointer");
  if (!eig_supported(n, K)) return fail(c, PSVD_EINVAL, "core of size %d with K=%d is not supported", n, K);
  int rc;
  if ((rc = make_dvec(c, sigma_in, ff, Kc, n, st))) return rc;
  if ((rc = ensure(c, c->eigws, sizeof(double) * eig_workspace_doubles(n, K)))) return rc;
  static const bool eig_timers = getenv("PSVD_EIG_TIMERS") != nullptr;  // diagnostics: phase clocks
  return core_solve(c, G, n, K, (const double*)c->dvec.ptr, W, sigma_out, st, eig_timers ? c->d_timers : nullptr);
}

int psvd_recompose(psvd_ctx* c, int64_t M, const double* U, int64_t ldu, int Kc, const double* A, int64_t lda, int B,
                   const double* W, int K, double* U_out, int64_t ldo, double* UtU, void* stream) {
  if (!c) return PSVD_EINVAL;
  cudaStream_t st = (cudaStream_t)stream;
  int rc;
  if (M < 1 || K < 1 || Kc + B < 1) return fail(c, PSVD_EINVAL, "bad shape");
  if ((rc = check_mat(c, "U", U, ldu, M, Kc)) || (rc = check_mat(c, "A", A, lda, M, B)) ||
      (rc = check_mat(c, "U_out", U_out, ldo, M, K)))
    return rc;
  const int n = Kc + B;
  Pass ps;
  if (plan_pass(c, ps, M, panel(U, ldu, Kc, A, lda, B), 0, n, K, W, n, false, UtU != nullptr, false) != PSVD_OK) {
    // panel + W beyond one pass's shared memory: U_out = [U | A] W and U_out^T U_out on the
    // tall-skinny GEMMs (the panel is read once per product)
    c->path_count[4]++;
    std::vector<GemmSeg> gp;
    if (Kc > 0) gp.push_back(GemmSeg{U, ldu, Kc});
    gp.push_back(GemmSeg{A, lda, B});
    launch_tgemm_nn(M, gp.data(), (int)gp.size(), W, n, K, U_out, ldo, st);
    c->launches++;
    if (UtU) {
      if ((rc = ensure(c, c->partial, sizeof(double) * tgemm_tn_partial_doubles(M, K, K, c->num_sms)))) return rc;
      const GemmSeg gu{U_out, ldo, K};
      launch_tgemm_tn(M, &gu, 1, U_out, ldo, K, nullptr, UtU, K, (double*)c->partial.ptr, c->num_sms, st);
      c->launches += 2;
    }
    return cuda_check(c, "wide recompose");
  }
  ps.p.Yout = U_out;
  ps.p.ldy = ldo;
  if ((rc = run_pass(c, ps, st))) return rc;
  if (UtU) {
    launch_extract_sym((const double*)c->tiles.ptr, ps.NB, ps.p.np_pad, K, nullptr, UtU, st);
    c->launches++;
    rc = cuda_check(c, "extract UtU");
  }
  return rc;
}

int psvd_drift_rescue(psvd_ctx* c, int64_t M, double* U, int64_t ldu, int K, const double* UtU, double* sigma,
                      double tol, void* stream) {
  if (!c) return PSVD_EINVAL;
  cudaStream_t st = (cudaStream_t)stream;
  int rc;
  if ((rc = check_mat(c, "U", U, ldu, M, K))) return rc;
  if (K > MAX_W) return fail(c, PSVD_EINVAL, "K=%d too large for the rescue pass", K);
  if ((rc = ensure(c, c->tbuf, sizeof(double) * ((size_t)K * K + K)))) return rc;
  launch_drift_check(UtU, K, tol, sigma, (double*)c->tbuf.ptr, c->d_gate, c->d_status, st);
  c->launches++;
  if ((rc = cuda_check(c, "drift check"))) return rc;
  Pass ps;
  if ((rc = plan_pass(c, ps, M, {Seg{U, ldu, K, 0}}, 0, K, K, (const double*)c->tbuf.ptr, K, false, false, false)))
    return rc;
  ps.p.Yout = U;  // in place: every stage is fully staged in smem before its rows are rewritten
  ps.p.ldy = ldu;
  ps.p.gate = c->d_gate;
  return run_pass(c, ps, st);
}

}  // extern "C"

// Core solve of a Gram: eig (+ concurrent LDL^T on the aux stream when the split path applies)
static int core_solve(psvd_ctx* c, const double* G, int n, int K, const double* dscale, double* W, double* sigma,
                      cudaStream_t st, long long* timers) {
  int rc = ensure(c, c->eigws, sizeof(double) * eig_workspace_doubles(n, K));
  if (rc) return rc;
  double* ws = (double*)c->eigws.ptr;
  if (eig_split_supported(n, K) && timers == nullptr) {
    cudaEventRecord(c->ev_ldlt_fork, st);
    cudaStreamWaitEvent(c->s_aux, c->ev_ldlt_fork, 0);
    launch_ldlt_pack(G, n, ws, c->s_aux);  // packed L in the (unused in smem mode) first n(n+1)/2 doubles
    cudaEventRecord(c->ev_ldlt_join, c->s_aux);
    static const bool no_ss = getenv("PSVD_NO_SUBSPACE") != nullptr;
    if (!no_ss && subspace_supported(n, K)) {
      // subspace-iteration fast path; the full solver below is gated off when it converged
      if ((rc = ensure(c, c->ssws, sizeof(double) * subspace_workspace_doubles(n)))) return rc;
      launch_subspace_eig(G, n, K, (double*)c->ssws.ptr, ws + (size_t)n * (n + 1) / 2, sigma, c->d_ssgate, st);
      launch_eig_topk(G, n, K, dscale, W, sigma, ws, c->d_status, nullptr, st, 0.0, 1, c->d_ssgate);
      c->launches += 4;
    } else {
      cudaMemsetAsync(c->d_ssgate, 0xff, sizeof(int), st);  // reads as "full solver"
      launch_eig_topk(G, n, K, dscale, W, sigma, ws, c->d_status, nullptr, st, 0.0, 1);
    }
    cudaStreamWaitEvent(st, c->ev_ldlt_join, 0);
    launch_sign_weights(ws, ws + (size_t)n * (n + 1) / 2, sigma, n, K, dscale, W, sigma, c->d_status, 0.0, st);
    c->launches += 3;
  } else {
    launch_eig_topk(G, n, K, dscale, W, sigma, ws, c->d_status, timers, st);
    c->launches++;
  }
  return cuda_check(c, "core solve");
}

// sigma_k <- ||C v_k|| and unit columns (Rayleigh refinement), UtU normalized in place
static int refine_normalize(psvd_ctx* c, int64_t M, double* U, int64_t ld, int K, double* UtU, double* sigma,
                            cudaStream_t st) {
  int rc = ensure(c, c->tbuf, sizeof(double) * ((size_t)K * K + K));
  if (rc) return rc;
  double* scale = (double*)c->tbuf.ptr + (size_t)K * K;
  launch_normalize_gram(UtU, K, sigma, scale, st);
  launch_scale_cols(U, ld, M, K, scale, st);
  c->launches += 2;
  return cuda_check(c, "refine");
}

extern "C" {

int psvd_stream_update(psvd_ctx* c, int64_t M, const double* U, int64_t ldu, const double* sigma, double ff, int Kc,
                       const double* A, int64_t lda, int B, int K, int rescue, double* U_out, int64_t ldo,
                       double* sigma_out, void* stream) {
  if (!c) return PSVD_EINVAL;
  const int n = Kc + B;
  if (K < 1 || K > n) return fail(c, PSVD_EINVAL, "K=%d must be in [1, %d]", K, n);
  int rc;
  if ((rc = ensure(c, c->gram, sizeof(double) * (size_t)n * n))) return rc;
  if ((rc = ensure(c, c->wbuf, sizeof(double) * (size_t)n * K))) return rc;
  if ((rc = ensure(c, c->utu, sizeof(double) * (size_t)K * K))) return rc;
  double* G = (double*)c->gram.ptr;
  double* W = (double*)c->wbuf.ptr;
  double* UtU = (double*)c->utu.ptr;
  if ((rc = psvd_gram(c, M, U, ldu, sigma, ff, Kc, A, lda, B, G, stream))) return rc;
  if ((rc = psvd_core_eig(c, G, n, sigma, ff, Kc, K, W, sigma_out, stream))) return rc;
  if ((rc = psvd_recompose(c, M, U, ldu, Kc, A, lda, B, W, K, U_out, ldo, UtU, stream))) return rc;
  if ((rc = refine_normalize(c, M, U_out, ldo, K, UtU, sigma_out, (cudaStream_t)stream))) return rc;
  if (rescue) rc = psvd_drift_rescue(c, M, U_out, ldo, K, UtU, sigma_out, c->drift_tol, stream);
  return rc;
}

// SVQB orthonormalizer of a sketch Gram: T = V diag(1/sqrt(lambda)) with numerically
// null directions (sigma below rank_tol * sigma_max) dropped (zero columns).
// exchange points of the row-partitioned randomized update (no-ops on one GPU)
static int ex_allreduce(psvd_ctx* c, double* buf, int64_t count, cudaStream_t st) {
  if (!c->ex_allreduce) return PSVD_OK;
  if (c->ex_allreduce(c->ex_user, buf, count, (void*)st) != 0) return fail(c, PSVD_ECUDA, "allreduce hook failed");
  return PSVD_OK;
}

// sign rule over ranks: local per-chunk pairs -> one pair per column -> allgather -> sign
static int exchange_sign(psvd_ctx* c, const double* local_pairs, int nchunks, int K, double* sgn, cudaStream_t st) {
  if (!c->ex_allgather) {
    launch_colmax_sign(local_pairs, nchunks, K, sgn, st);
    c->launches++;
    return PSVD_OK;
  }
  int rc;
  if ((rc = ensure(c, c->xpairs, sizeof(double) * (size_t)(c->ex_nranks + 1) * K * 2))) return rc;
  double* mine = (double*)c->xpairs.ptr;
  double* all = mine + (size_t)K * 2;
  launch_colmax_reduce(local_pairs, nchunks, K, mine, st);
  if (c->ex_allgather(c->ex_user, mine, (int64_t)K * 2, all, (void*)st) != 0)
    return fail(c, PSVD_ECUDA, "allgather hook failed");
  launch_colmax_sign(all, c->ex_nranks, K, sgn, st);  // rank order = global row order: first rank wins ties
  c->launches += 2;
  return PSVD_OK;
}

// SVQB weights T = V diag(lambda^-1/2) of the l x l sketch Gram (numerically null directions
// dropped at 1e-7 relative), from a one-sided Jacobi eigen-decomposition of the Gram.
static int svqb(psvd_ctx* c, const double* Gs, int l, double* T, double* sig_scratch, cudaStream_t st) {
  int rc = ensure(c, c->eigws, sizeof(double) * std::max(eig_workspace_doubles(l, l), jacobi_workspace_doubles(l, l)));
  if (rc) return rc;
  // CholeskyQR weights T = R^-1 first (one short kernel); when the sketch is ill conditioned
  // (max R_ii / min R_ii > 1e6 or a dropped pivot) the gated Jacobi SVQB overwrites them
  int* illcond = c->d_status + 3;
  launch_chol_inv(Gs, l, T, st, illcond, c->d_status);
  launch_jacobi_svd(Gs, l, l, sig_scratch, T, (double*)c->eigws.ptr, c->d_status, st, illcond);
  launch_svqb_scale(T, sig_scratch, l, 1e-7, st, illcond);
  c->launches += 3;
  return cuda_check(c, "svqb");
}

int psvd_rand_update(psvd_ctx* c, int64_t M, const double* U, int64_t ldu, const double* sigma, double ff, int Kc,
                     const double* A, int64_t lda, int B, int K, int l, int q, const double* Omega, double* U_out,
                     int64_t ldo, double* sigma_out, void* stream) {
  if (!c) return PSVD_EINVAL;
  cudaStream_t st = (cudaStream_t)stream;
  const int n = Kc + B;
  int rc;
  if (M < 1 || B < 1 || Kc < 0 || K < 1 || l < K || q < 0) return fail(c, PSVD_EINVAL, "bad randomized shape");
  if (l > std::min<int64_t>(M, n))
    return fail(c, PSVD_EINVAL, "sketch width %d exceeds min(a.shape) = %lld", l, (long long)std::min<int64_t>(M, n));
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
      launch_tgemm_tn(M, &gy, 1, Y, ldy, l, nullptr, G1, l, pbuf, c->num_sms, st);    // G1 = Y^T Y
      c->launches += 3;
      if ((rc = ex_allreduce(c, G1, (int64_t)l * l, st))) return rc;
      if ((rc = svqb(c, G1, l, T1, sscr, st))) return rc;
      launch_tgemm_nn(M, &gy, 1, T1, l, l, Y2, ldy, st);                              // Y1 = Y T1
      launch_tgemm_tn(M, &gy2, 1, Y2, ldy, l, nullptr, G2, l, pbuf, c->num_sms, st);  // G2 = Y1^T Y1
      launch_tgemm_tn(M, gp.data(), (int)gp.size(), Y2, ldy, l, d, X, n, pbuf, c->num_sms, st);  // X = D P^T Y1
      c->launches += 5;
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
    launch_jacobi_svd(Bt, n, l, S, J, (double*)c->jacws.ptr, c->d_status, st);
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
    stamp_kernel<<<1, 1, 0, s_>>>(tbuf + tl.size());
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
  const int nsub = (int)std::max<int64_t>(1, std::min<int64_t>(4, M / 65536));
  auto aa_pass = [&](int j) -> int {
    if (j >= 2) cudaStreamWaitEvent(lo, c->ev_asm[j & 1], 0);  // tiles2[j&1] consumed by batch j-2's assembly
    // start A^T A of batch j with the core solve of batch j-1: it then overlaps that one-SM
    // solve (the longer of the two) instead of competing with the recompose pass for SMs
    if (j >= 1) cudaStreamWaitEvent(lo, c->ev_eig_start, 0);
    if (batch_ready && batch_ready[j]) cudaStreamWaitEvent(lo, (cudaEvent_t)batch_ready[j], 0);
    const int64_t rows_sub = (M + nsub - 1) / nsub / 32 * 32 + 32;
    Pass first;
    size_t part_off = 0;
    int nchunks_total = 0;
    mark("lo:aa_begin", j, lo);
    for (int k = 0; k < nsub; ++k) {
      const int64_t r0 = (int64_t)k * rows_sub;
      if (r0 >= M) break;
      const int64_t mk = std::min(M, r0 + rows_sub) - r0;
      Pass pa;
      int r = plan_pass(c, pa, mk, {Seg{A[j] + r0, lda[j], B[j], 0}}, 0, 0, 0, nullptr, 0, true, false, false, -1,
                        -1, &c->partial2, &c->tiles2[j & 1], c->num_sms - 2);
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
      const double uu_w = (c->ex_allreduce && c->ex_row_offset != 0) ? 0.0 : 1.0;
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
    if (b + 1 < nb) {
      // fused: U_b = [U_{b-1} | A_b] W, with U_b^T U_b and U_b^T A_{b+1} from the same pass
      std::vector<Seg> segs = panel(Uprev, ldprev, kc, A[b], lda[b], B[b]);
      segs.push_back(Seg{A[b + 1], lda[b + 1], B[b + 1], 1});
      if (batch_ready && batch_ready[b + 1]) cudaStreamWaitEvent(hi, (cudaEvent_t)batch_ready[b + 1], 0);
      Pass pf;
      const int wk = kc + B[b];
      if ((rc = plan_pass(c, pf, M, segs, 0, wk, K, W, wk, false, true, true, -1, -1, nullptr, nullptr, 0, -1)))
        return rc;
      const int a0 = pf.p.seg[pf.p.nseg - 1].col0 / 32;
      pf.p.Yout = Uout;
      pf.p.ldy = ldo;
      if ((rc = run_pass(c, pf, hi))) return rc;
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
    if ((rc = refine_normalize(c, M, Uout, ldo, K, UtU, sig_b, hi))) return rc;
    if (resc && (rc = psvd_drift_rescue(c, M, Uout, ldo, K, UtU, sig_b, c->drift_tol, hi))) return rc;
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
  if (c->ex_allreduce) return fail(c, PSVD_EINVAL, "the pipelined randomized run is single-GPU");
  if (Kc != 0 && Kc != K) return fail(c, PSVD_EINVAL, "initial state carries %d modes, K=%d", Kc, K);
  if (Kc > 0 && (!U_in || !sigma_in)) return fail(c, PSVD_EINVAL, "null initial state");
  int rc;
  int bmax = 0;
  for (int b = 0; b < nb; ++b) {
    if ((rc = check_mat(c, "A", A[b], lda[b], M, B[b]))) return rc;
    if (B[b] < 1) return fail(c, PSVD_EINVAL, "empty batch");
    if (!Omega[b]) return fail(c, PSVD_EINVAL, "null Omega");
    const int n = ((b > 0 || Kc > 0) ? K : 0) + B[b];
    if (l > std::min<int64_t>(M, n))
      return fail(c, PSVD_EINVAL, "sketch width %d exceeds min(a.shape) = %lld", l, (long long)std::min<int64_t>(M, n));
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
    stamp_kernel<<<1, 1, 0, s_>>>(tbuf + tl.size());
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
      if (pa.tma)
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
      segs.push_back(Seg{Zt, ldq, l, 0});
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
      if ((rc = svqb(c, G1, l, T1, sscr, hi))) return rc;
      segs.push_back(Seg{Zt, ldq, l, 0});
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

// ---- dense factorizations behind the reference's linalg boundary (qr_factor / svd_full /
// randomized_range, linalg.py:94-147; parallel_qr, dsvd.py:176-202).  Library utilities, not
// the streaming update: psvd_qr reads one condition flag back (one host sync).

int psvd_chol(psvd_ctx* c, const double* G, int n, double* R, double* T, void* stream) {
  if (!c) return PSVD_EINVAL;
  if (n < 1 || n > CHOL_NMAX || !G || !T) return fail(c, PSVD_EINVAL, "bad Cholesky n=%d (1..%d)", n, CHOL_NMAX);
  launch_chol_inv(G, n, T, (cudaStream_t)stream, c->d_status + 3, c->d_status, R);
  c->launches++;
  return cuda_check(c, "chol");
}

int psvd_chol_shift(psvd_ctx* c, double* G, int n, int64_t M, void* stream) {
  if (!c) return PSVD_EINVAL;
  if (n < 1 || !G || M < 1) return fail(c, PSVD_EINVAL, "bad shift arguments");
  launch_chol_shift(G, n, M, (cudaStream_t)stream);
  c->launches++;
  return cuda_check(c, "chol shift");
}

int psvd_chol_illcond(psvd_ctx* c, int* flag, void* stream) {
  if (!c || !flag) return PSVD_EINVAL;
  cudaStream_t st = (cudaStream_t)stream;
  cudaMemcpyAsync(c->h_status, c->d_status + 3, sizeof(int), cudaMemcpyDeviceToHost, st);
  if (cudaStreamSynchronize(st) != cudaSuccess) return cuda_check(c, "chol flag");
  *flag = *c->h_status;
  return PSVD_OK;
}

int psvd_nn_product(psvd_ctx* c, int64_t M, const double* A, int64_t lda, int n, const double* W, int64_t ldw, int w,
                    double* Y, int64_t ldy, void* stream) {
  if (!c) return PSVD_EINVAL;
  int rc;
  if (M < 1 || n < 1 || w < 1 || !W || ldw < n) return fail(c, PSVD_EINVAL, "bad nn_product shape");
  if ((rc = check_mat(c, "A", A, lda, M, n)) || (rc = check_mat(c, "Y", Y, ldy, M, w))) return rc;
  const GemmSeg ga{A, lda, n};
  launch_tgemm_nn(M, &ga, 1, W, ldw, w, Y, ldy, (cudaStream_t)stream);
  c->launches++;
  return cuda_check(c, "nn product");
}

int psvd_small_matmul(psvd_ctx* c, const double* A, int lda, int transA, const double* B, int ldb, double* C, int ldc,
                      int m, int k, int n, void* stream) {
  if (!c) return PSVD_EINVAL;
  if (m < 1 || k < 1 || n < 1 || !A || !B || !C || ldc < m) return fail(c, PSVD_EINVAL, "bad small matmul");
  launch_small_gemm(A, lda, transA, B, ldb, C, ldc, m, k, n, nullptr, (cudaStream_t)stream);
  c->launches++;
  return cuda_check(c, "small matmul");
}

// Tall QR (M >= n, n <= CHOL_NMAX): CholeskyQR2 (R = R2 R1 from two Gram passes), or the shifted
// CholeskyQR3 when the first Cholesky flags cond(A) beyond CholeskyQR2's range.  diag(R) >= 0 by
// construction (qr_factor's sign convention, linalg.py:94-104); numerically null directions give zero
// rows of R and zero columns of Q.  R: n x n, ld n.
int psvd_qr(psvd_ctx* c, int64_t M, int n, const double* A, int64_t lda, double* Q, int64_t ldq, double* R,
            void* stream) {
  if (!c) return PSVD_EINVAL;
  cudaStream_t st = (cudaStream_t)stream;
  int rc;
  if (n < 1 || n > CHOL_NMAX || M < n) return fail(c, PSVD_EINVAL, "qr needs M >= n and n <= %d (M=%lld n=%d)",
                                                  CHOL_NMAX, (long long)M, n);
  if ((rc = check_mat(c, "A", A, lda, M, n)) || (rc = check_mat(c, "Q", Q, ldq, M, n))) return rc;
  if (!R) return fail(c, PSVD_EINVAL, "R is null");
  const size_t nn = (size_t)n * n;
  const int64_t ldt = M + (M & 1);
  if ((rc = ensure(c, c->dense, sizeof(double) * 8 * nn)) || (rc = ensure(c, c->dense2, sizeof(double) * ldt * n)))
    return rc;
  double* G = (double*)c->dense.ptr;
  double* R1 = G + nn;
  double* T1 = R1 + nn;
  double* R2 = T1 + nn;
  double* T2 = R2 + nn;
  double* R3 = T2 + nn;
  double* T3 = R3 + nn;
  double* Rt = T3 + nn;
  double* tmp = (double*)c->dense2.ptr;
  auto gram = [&](const double* X, int64_t ldx) { return psvd_gram(c, M, nullptr, 0, nullptr, 1.0, 0, X, ldx, n, G, st); };
  auto mul = [&](const double* X, int64_t ldx, const double* T, double* Y, int64_t ldy) {
    const GemmSeg gx{X, ldx, n};
    launch_tgemm_nn(M, &gx, 1, T, n, n, Y, ldy, st);
    c->launches++;
  };
  auto refine = [&](double* Rk, double* Tk) -> int {  // Q <- Q chol(Q^T Q)^-1, returns the new factor in Rk
    int r;
    if ((r = gram(Q, ldq))) return r;
    launch_chol_inv(G, n, Tk, st, nullptr, c->d_status, Rk);
    mul(Q, ldq, Tk, tmp, ldt);
    cudaMemcpy2DAsync(Q, ldq * sizeof(double), tmp, ldt * sizeof(double), M * sizeof(double), n,
                      cudaMemcpyDeviceToDevice, st);
    c->launches++;
    return cuda_check(c, "qr refine");
  };
  // CholeskyQR2
  if ((rc = gram(A, lda))) return rc;
  launch_chol_inv(G, n, T1, st, c->d_status + 3, c->d_status, R1);
  c->launches++;
  int ill = 0;
  if ((rc = psvd_chol_illcond(c, &ill, stream))) return rc;
  if (ill) {  // shifted CholeskyQR3
    if ((rc = gram(A, lda))) return rc;
    launch_chol_shift(G, n, M, st);
    launch_chol_inv(G, n, T1, st, nullptr, c->d_status, R1);
    c->launches += 2;
  }
  mul(A, lda, T1, Q, ldq);
  if ((rc = refine(R2, T2))) return rc;
  launch_small_gemm(R2, n, 0, R1, n, ill ? Rt : R, n, n, n, n, nullptr, st);  // R2 R1
  c->launches++;
  if (ill) {
    if ((rc = refine(R3, T3))) return rc;
    launch_small_gemm(R3, n, 0, Rt, n, R, n, n, n, n, nullptr, st);  // R3 R2 R1
    c->launches++;
  }
  return cuda_check(c, "qr");
}

// One-sided Jacobi SVD of X (m x n, m >= n, n <= JACOBI_NMAX): S (n, descending), V (n x n, ld ldv;
// X = U diag(S) V^T).  Relative accuracy (no squaring); X is packed first.
int psvd_jacobi(psvd_ctx* c, const double* X, int64_t ldx, int64_t m, int n, double* S, double* V, int64_t ldv,
                void* stream) {
  if (!c) return PSVD_EINVAL;
  cudaStream_t st = (cudaStream_t)stream;
  int rc;
  if (n < 1 || n > JACOBI_NMAX || m < n || m > (int64_t)INT32_MAX)
    return fail(c, PSVD_EINVAL, "jacobi needs m >= n and n <= %d (m=%lld n=%d)", JACOBI_NMAX, (long long)m, n);
  if (!X || !S || !V || ldx < m || ldv < n) return fail(c, PSVD_EINVAL, "bad jacobi arguments");
  const size_t mn = (size_t)m * n;
  if ((rc = ensure(c, c->dense2, sizeof(double) * (mn + (size_t)n * n))) ||
      (rc = ensure(c, c->jacws, sizeof(double) * jacobi_workspace_doubles((int)m, n))))
    return rc;
  double* Xp = (double*)c->dense2.ptr;
  double* J = Xp + mn;
  cudaMemcpy2DAsync(Xp, m * sizeof(double), X, ldx * sizeof(double), m * sizeof(double), n, cudaMemcpyDeviceToDevice,
                    st);
  launch_jacobi_svd(Xp, (int)m, n, S, J, (double*)c->jacws.ptr, c->d_status, st);
  cudaMemcpy2DAsync(V, ldv * sizeof(double), J, n * sizeof(double), n * sizeof(double), n, cudaMemcpyDeviceToDevice, st);
  c->launches++;
  return cuda_check(c, "jacobi");
}

// The reference's sign rule (linalg.py:81-91): per column of U (rows x cols) the entry of largest
// magnitude (first occurrence) is made positive; the same flips go to the columns of V (vrows x
// cols, may be null: the rows of vt).
int psvd_sign_pair(psvd_ctx* c, double* U, int64_t ldu, int64_t rows, int cols, double* V, int64_t ldv, int64_t vrows,
                   void* stream) {
  if (!c) return PSVD_EINVAL;
  cudaStream_t st = (cudaStream_t)stream;
  int rc;
  if (rows < 1 || cols < 1 || !U || ldu < rows || (V && ldv < vrows)) return fail(c, PSVD_EINVAL, "bad sign arguments");
  const int64_t nch = colmax_rows_chunks(rows);
  if ((rc = ensure(c, c->colmax, sizeof(double) * (size_t)nch * cols * 2)) ||
      (rc = ensure(c, c->xpairs, sizeof(double) * (size_t)cols)))
    return rc;
  double* sgn = (double*)c->xpairs.ptr;
  launch_colmax_rows(U, ldu, rows, cols, 0, (double*)c->colmax.ptr, st);
  launch_colmax_sign((const double*)c->colmax.ptr, (int)nch, cols, sgn, st);
  launch_scale_cols(U, ldu, rows, cols, sgn, st);
  c->launches += 3;
  if (V) {
    launch_scale_cols(V, ldv, vrows, cols, sgn, st);
    c->launches++;
  }
  return cuda_check(c, "sign pair");
}

// X[:, j] *= s_j (invert = 0) or /= s_j with 0 for s_j == 0 (invert = 1)
int psvd_scale_cols(psvd_ctx* c, double* X, int64_t ld, int64_t rows, int cols, const double* s, int invert,
                    void* stream) {
  if (!c) return PSVD_EINVAL;
  if (!X || !s || rows < 1 || cols < 1 || ld < rows) return fail(c, PSVD_EINVAL, "bad scale_cols arguments");
  dim3 g((unsigned)((rows + 255) / 256), (unsigned)cols);
  scale_cols_any_kernel<<<g, 256, 0, (cudaStream_t)stream>>>(X, ld, rows, cols, s, invert);
  c->launches++;
  return cuda_check(c, "scale cols");
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

int psvd_refine_normalize(psvd_ctx* c, int64_t M, double* U, int64_t ldu, int K, double* UtU, double* sigma,
                          void* stream) {
  if (!c) return PSVD_EINVAL;
  int rc;
  if ((rc = check_mat(c, "U", U, ldu, M, K))) return rc;
  if (!UtU || !sigma || K > 1024) return fail(c, PSVD_EINVAL, "bad refine arguments");
  return refine_normalize(c, M, U, ldu, K, UtU, sigma, (cudaStream_t)stream);
}

int psvd_sum_ordered(psvd_ctx* c, const double* parts, int P, int64_t count, double* out, void* stream) {
  if (!c || !parts || !out || P < 1 || count < 0) return fail(c, PSVD_EINVAL, "bad sum_ordered args");
  if (count == 0) return PSVD_OK;
  sum_ordered_kernel<<<(unsigned)((count + 255) / 256), 256, 0, (cudaStream_t)stream>>>(parts, P, count, out);
  c->launches++;
  return cuda_check(c, "sum ordered");
}

int psvd_burgers(psvd_ctx* c, double* out, int64_t ldo, int64_t row0, int64_t rows, int64_t grid, int col0, int cols,
                 int n_snap, double length, double t_final, double reynolds, void* stream) {
  if (!c || !out || rows < 0 || cols < 0 || grid < 2 || n_snap < 1 || ldo < rows || row0 < 0 || row0 + rows > grid ||
      col0 < 0 || col0 + cols > n_snap)
    return fail(c, PSVD_EINVAL, "bad burgers args");
  if (rows == 0 || cols == 0) return PSVD_OK;
  dim3 g((unsigned)((rows + 255) / 256), (unsigned)cols);
  burgers_kernel<<<g, 256, 0, (cudaStream_t)stream>>>(out, ldo, row0, rows, grid, col0, cols, n_snap, length, t_final,
                                                       reynolds);
  return cuda_check(c, "burgers");
}

}  // extern "C"
