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

#include "psvd_ctx.cuh"

namespace psvd_internal {

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

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

int check_mat(psvd_ctx* c, const char* name, const double* p, int64_t ld, int64_t M, int cols) {
  if (cols == 0) return PSVD_OK;
  if (p == nullptr) return fail(c, PSVD_EINVAL, "%s is null", name);
  if (ld < M) return fail(c, PSVD_EINVAL, "%s: leading dimension %lld < rows %lld", name, (long long)ld, (long long)M);
  if (ld % 2 != 0) return fail(c, PSVD_EINVAL, "%s: leading dimension %lld must be even", name, (long long)ld);
  if (!aligned16(p)) return fail(c, PSVD_EINVAL, "%s: base pointer must be 16-byte aligned", name);
  return PSVD_OK;
}


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
int plan_tiles_balanced(psvd_ctx* c, Pass& ps, const std::vector<std::pair<int, int>>& tiles, int np,
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
int plan_tiles_tma(psvd_ctx* c, Pass& ps, const std::vector<std::pair<int, int>>& tiles,
                   const std::vector<unsigned char>& sub) {
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
  // warp of each tile: in order, or (one slice, register-W Y warps) longest-first onto the SMSP
  // (warp % 4) with the least Gram work so far -- the Y parts' k split then evens the SMSPs out
  std::vector<int> warp_of(nt);
  for (int o = 0; o < nt; ++o) warp_of[o] = warp0 + o % per;
  static const bool no_lpt = getenv("PSVD_TMA_NO_LPT") != nullptr;  // diagnostics: tiles in order
  if (nslices == 1 && ykp > 1 && !no_lpt) {
    const int NBp = ps.p.np_pad / 32;
    std::vector<int> cost(nt), order(nt);
    for (int o = 0; o < nt; ++o) {
      const int I = tiles[o].first;
      const int na = I >= NBp ? ncb : sub[o] ? (sub[o] >> 4) : std::min(4, (ps.p.np - I * 32 + 7) / 8);
      cost[o] = na * ncb;
      order[o] = o;
    }
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return cost[a] > cost[b]; });
    int load[4] = {0, 0, 0, 0};
    std::vector<char> used(NWARP, 0);
    for (int o : order) {
      int best = -1;
      for (int w = warp0; w < warp0 + nwarps; ++w)
        if (!used[w] && (best < 0 || load[w % 4] < load[best % 4])) best = w;
      used[best] = 1;
      load[best % 4] += cost[o];
      warp_of[o] = best;
    }
    // pairwise swaps across SMSPs while they lower the busiest SMSP (then the spread)
    auto score = [&](const int* L) {
      int mx = 0, sq = 0;
      for (int q = 0; q < 4; ++q) mx = std::max(mx, L[q]), sq += L[q] * L[q];
      return std::make_pair(mx, sq);
    };
    for (bool improved = true; improved;) {
      improved = false;
      for (int a = 0; a < nt && !improved; ++a)
        for (int b = a + 1; b < nt && !improved; ++b) {
          const int qa = warp_of[a] % 4, qb = warp_of[b] % 4;
          if (qa == qb || cost[a] == cost[b]) continue;
          int L[4] = {load[0], load[1], load[2], load[3]};
          L[qa] += cost[b] - cost[a];
          L[qb] += cost[a] - cost[b];
          if (score(L) < score(load)) {
            std::swap(warp_of[a], warp_of[b]);
            for (int q = 0; q < 4; ++q) load[q] = L[q];
            improved = true;
          }
        }
    }
  }
  for (int o = 0; o < nt; ++o) {
    const int sl = o / per, w = warp_of[o];
    WarpPlan& wp = ps.p.plan[sl][w];
    wp.ksplit = 1;
    wp.kpart = 0;
    wp.ti[0] = (signed char)tiles[o].first;
    wp.tj[0] = (signed char)tiles[o].second;
    wp.ntile = 1;
    wp.sub = sub[o];
    ps.map.src[o][ps.map.nsrc[o]++] = (unsigned char)(sl * SLOTS + w * TPW);
    ps.map.out_id[o] = (short)(tiles[o].first * ps.NB + tiles[o].second);
  }
  return PSVD_OK;
}

// Common pass setup.  segs: panel segments; w/W: optional Y = P[:, wlo:wlo+wk] * W.
int plan_pass(psvd_ctx* c, Pass& ps, int64_t M, const std::vector<Seg>& segs, int wlo, int wk, int w,
              const double* W, int64_t ldw, bool gram_pp, bool gram_yy, bool gram_py, int py_cols,
              int pp_rows, Buf* part, Buf* tl, int max_ctas, int py_lo, bool gaps_ok,
              const std::vector<std::pair<int, int>>* skip_pp) {
  memset(&ps.p, 0, sizeof(ps.p));
  ps.fsplit = false;
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
      for (int J = I; J < NBp; ++J) {
        // tiles another pass computes (the split-ring fused pass takes some off the look-ahead Gram)
        if (skip_pp && std::find(skip_pp->begin(), skip_pp->end(), std::make_pair(I, J)) != skip_pp->end()) continue;
        tiles.push_back({I, J});
      }
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
  // narrow TMA pass: P-tiles compute only the 8-column sub-blocks that hold wanted rows, the
  // columns of segments not flagged "no P^T Y" (col0 == 2 on input) inside [py_lo block, py_cols)
  std::vector<unsigned char> sub(tiles.size(), 0);
  if (tma && gram_py) {
    std::vector<char> want((size_t)np_pad / 8, 0);
    const int lo = py_lo * 32, hi = py_cols < 0 ? np_pad : std::min(np_pad, py_cols);
    for (size_t i = 0; i < segs.size(); ++i) {
      if (segs[i].col0 == 2) continue;
      const int c0 = std::max(lo, p.seg[i].col0), c1 = std::min(hi, p.seg[i].col0 + p.seg[i].ncols);
      for (int sb = c0 / 8; sb * 8 < c1; ++sb) want[sb] = 1;
    }
    for (size_t o = 0; o < tiles.size(); ++o) {
      if (tiles[o].first >= NBp) continue;
      int a0 = -1, a1 = -1;
      for (int a = 0; a < 4; ++a)
        if (want[(size_t)tiles[o].first * 4 + a]) {
          if (a0 < 0) a0 = a;
          a1 = a;
        }
      if (a0 >= 0) sub[o] = (unsigned char)(a0 | ((a1 - a0 + 1) << 4));
    }
  }
  int rc = tma ? plan_tiles_tma(c, ps, tiles, sub)
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
  // narrow TMA passes go to the split-ring kernel when they qualify (32-row 3-D boxes, W in registers;
  // psvd_tall.cuh: FusedSplit); passes planned with offloaded tiles are launched by their owners
  if (ps.tma && !ps.fsplit) try_fused_split(c, ps, {}, 1);
  if (ps.fsplit && ps.offmap.nout == 0) return run_fused_split(c, ps, st, nullptr);
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

bool try_fused_split(psvd_ctx* c, Pass& ps, const std::vector<std::pair<int, int>>& off, int off_nb) {
  ps.fsplit = false;
  static const bool disabled = getenv("PSVD_NO_FSPLIT") != nullptr;  // A/B switch: narrow TMA pass everywhere
  if (disabled || !ps.tma || c->num_sms < 1) return false;
  static const int fs_dbg = getenv("PSVD_FS_DBG") ? atoi(getenv("PSVD_FS_DBG")) : 0;  // timing diagnostics (wrong results)
  if (fs_dbg) ps.p.dbg = fs_dbg;
  int offs[FS_MAX_OFF][2];
  int noff = 0;
  for (const auto& t : off)
    if (noff < FS_MAX_OFF) offs[noff][0] = t.first, offs[noff][1] = t.second, ++noff;
  if (fused_split_prepare(ps.p, ps.x, ps.map, ps.NB, offs, noff, ps.fs, ps.maps3, ps.offmap, off_nb) != 0) return false;
  ps.fsplit = true;
  return true;
}

int run_fused_split(psvd_ctx* c, Pass& ps, cudaStream_t st, double* off_tiles) {
  c->path_count[0]++;
  launch_fused_split(ps.p, ps.maps3, ps.x, ps.fs, ps.grid, st);
  c->launches += 1 + (ps.map.nout > 0) + (ps.offmap.nout > 0);
  int rc = cuda_check(c, "split-ring fused pass");
  if (rc) return rc;
  launch_tall_reduce((const double*)ps.part->ptr, ps.map, (double*)ps.tl->ptr, st);
  if (ps.offmap.nout > 0) launch_tall_reduce((const double*)ps.part->ptr, ps.offmap, off_tiles, st);
  return cuda_check(c, "split-ring reduce");
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

void launch_stamp(unsigned long long* out, cudaStream_t st) { stamp_kernel<<<1, 1, 0, st>>>(out); }

}  // namespace psvd_internal

using namespace psvd_internal;

// ============================================================================ C ABI

extern "C" {

int psvd_version(void) { return 1; }

// The caller's current device is restored on return (the context's kernels run on `device`; the
// Python layer enters that device around every call).
struct DeviceGuard {
  int prev = -1;
  DeviceGuard() { cudaGetDevice(&prev); }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

int psvd_create(int device, psvd_ctx** out) {
  if (!out) return PSVD_EINVAL;
  *out = nullptr;
  DeviceGuard guard;
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
    cudaFree(c->d_status);
    cudaFreeHost(c->h_status);
    delete c;
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
    cudaEventCreateWithFlags(&c->ev_fdone, cudaEventDisableTiming);
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
  DeviceGuard guard;
  cudaSetDevice(c->device);
  cudaDeviceSynchronize();
  Buf* bufs[] = {&c->partial, &c->tiles, &c->gram, &c->eigws, &c->wbuf, &c->utu, &c->tbuf, &c->dvec, &c->colmax,
                 &c->ybuf, &c->ybuf2, &c->xpairs, &c->ssws, &c->rsmall, &c->jacws, &c->partial2, &c->tiles2[0], &c->tiles2[1],
                 &c->zbuf, &c->rs2, &c->dense, &c->dense2, &c->bigws, &c->bigjac, &c->accws, &c->accq,
                 &c->nccl_parts};
  psvd_nccl_destroy(c);
  for (auto& e : c->tev) cudaEventDestroy(e);
  for (Buf* b : bufs)
    if (b->ptr) cudaFree(b->ptr);
  if (c->s_hi) cudaStreamDestroy(c->s_hi);
  if (c->s_lo) cudaStreamDestroy(c->s_lo);
  if (c->s_aux) cudaStreamDestroy(c->s_aux);
  if (c->ev_ldlt_fork) cudaEventDestroy(c->ev_ldlt_fork);
  if (c->ev_ldlt_join) cudaEventDestroy(c->ev_ldlt_join);
  if (c->ev_eig_start) cudaEventDestroy(c->ev_eig_start);
  if (c->ev_fdone) cudaEventDestroy(c->ev_fdone);
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
  if (allreduce && c->nccl_on) return fail(c, PSVD_EINVAL, "the NCCL exchange is enabled (psvd_nccl_enable)");
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
    // (one workspace for both products, each sized on its own: a narrower Y splits the rows into more chunks
    // and can need more partial tiles than the wider one)
    if ((rc = ensure(c, c->partial,
                     sizeof(double) * std::max(tgemm_tn_partial_doubles(M, n, std::max(Kc, 1), c->num_sms),
                                               tgemm_tn_partial_doubles(M, n, std::max(B, 1), c->num_sms)))))
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
  if ((rc = run_pass(c, ps, st))) return rc;  // the split-ring kernel with group A alone when the pass qualifies
  if (UtU) {
    launch_extract_sym((const double*)c->tiles.ptr, ps.NB, ps.p.np_pad, K, nullptr, UtU, st);
    c->launches++;
    rc = cuda_check(c, "extract UtU");
  }
  return rc;
}

int psvd_fused_pass(psvd_ctx* c, int64_t M, const double* U, int64_t ldu, int Kc, const double* A, int64_t lda, int B,
                    const double* A_next, int64_t ldan, int Bn, const double* W, int K, double* U_out, int64_t ldo,
                    double* UtU, double* AtU, int mode, int noff, double* off_tiles, void* stream) {
  if (!c) return PSVD_EINVAL;
  cudaStream_t st = (cudaStream_t)stream;
  int rc;
  if (M < 1 || K < 1 || B < 1 || Bn < 1 || Kc < 0 || !W || !UtU || !AtU) return fail(c, PSVD_EINVAL, "bad fused_pass arguments");
  if ((rc = check_mat(c, "U", U, ldu, M, Kc)) || (rc = check_mat(c, "A", A, lda, M, B)) ||
      (rc = check_mat(c, "A_next", A_next, ldan, M, Bn)) || (rc = check_mat(c, "U_out", U_out, ldo, M, K)))
    return rc;
  std::vector<Seg> segs = panel(U, ldu, Kc, A, lda, B);
  segs.push_back(Seg{A_next, ldan, Bn, 1});
  const int wk = Kc + B;
  Pass pf;
  if ((rc = plan_pass(c, pf, M, segs, 0, wk, K, W, wk, false, true, true, -1, -1, nullptr, nullptr, 0, -1))) return rc;
  pf.p.Yout = U_out;
  pf.p.ldy = ldo;
  const int off_nb = (Bn + 31) / 32;
  if (mode == 1) {
    std::vector<std::pair<int, int>> off;
    for (int t = 0; 2 * t + 1 < Bn / 32 && t < noff && off_tiles; ++t) off.push_back({2 * t, 2 * t + 1});
    if (!try_fused_split(c, pf, off, off_nb)) return fail(c, PSVD_EINVAL, "the pass does not qualify for the split-ring kernel");
    if ((rc = run_fused_split(c, pf, st, off_tiles))) return rc;
  } else if (!pf.tma) {  // no narrow TMA plan (e.g. an odd leading dimension): the general tall pass
    if ((rc = run_pass(c, pf, st))) return rc;
  } else {  // mode 0: the narrow TMA pass itself (run_pass would pick the split-ring kernel)
    c->path_count[0]++;
    launch_pass_tma(pf.p, pf.maps, pf.x, pf.grid, st);
    c->launches += 2;
    if ((rc = cuda_check(c, "narrow fused pass"))) return rc;
    launch_tall_reduce((const double*)pf.part->ptr, pf.map, (double*)pf.tl->ptr, st);
  }
  const int a0 = pf.p.seg[pf.p.nseg - 1].col0 / 32;
  launch_extract_sym((const double*)c->tiles.ptr, pf.NB, pf.p.np_pad, K, nullptr, UtU, st);
  launch_extract_rect((const double*)c->tiles.ptr, pf.NB, a0 * 32, Bn, pf.p.np_pad, K, nullptr, AtU, st);
  c->launches += 2;
  return cuda_check(c, "fused pass extract");
}

int psvd_drift_rescue(psvd_ctx* c, int64_t M, double* U, int64_t ldu, int K, const double* UtU, double* sigma,
                      double tol, void* stream) {
  if (!c) return PSVD_EINVAL;
  cudaStream_t st = (cudaStream_t)stream;
  int rc;
  if ((rc = check_mat(c, "U", U, ldu, M, K))) return rc;
  if (K > DRIFT_SMEM_KMAX) return drift_rescue_wide(c, M, U, ldu, K, UtU, sigma, tol, st);
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

__global__ void or_status_kernel(int* status, int bits) { atomicOr(status, bits); }

// Drift rescue for K beyond the one-CTA check's shared memory (K > DRIFT_SMEM_KMAX): the deviation
// max|UtU - I| is read back (one host sync), and when it exceeds tol U <- qr(U).q, sigma <- sigma |diag r|,
// both reordered stable-descending (streaming.py:106-115) through psvd_qr (any K, rank robust).
int psvd_internal::drift_rescue_wide(psvd_ctx* c, int64_t M, double* U, int64_t ldu, int K, const double* UtU,
                                     double* sigma, double tol, cudaStream_t st) {
  std::vector<double> h((size_t)K * K), sg(K), dg(K);
  if (cudaMemcpyAsync(h.data(), UtU, sizeof(double) * h.size(), cudaMemcpyDeviceToHost, st) != cudaSuccess ||
      cudaStreamSynchronize(st) != cudaSuccess)
    return cuda_check(c, "drift read");
  double dev = 0.0;
  for (int j = 0; j < K; ++j)
    for (int i = 0; i < K; ++i) dev = std::max(dev, std::fabs(h[(size_t)j * K + i] - (i == j ? 1.0 : 0.0)));
  if (!(dev > tol)) return PSVD_OK;
  const int64_t ldq = M + (M & 1);
  Buf q, r;
  int rc = PSVD_OK;
  if (cudaMalloc(&q.ptr, sizeof(double) * ldq * K) != cudaSuccess ||
      cudaMalloc(&r.ptr, sizeof(double) * (size_t)K * K) != cudaSuccess) {
    cudaFree(q.ptr);
    return fail(c, PSVD_ECUDA, "drift rescue allocation");
  }
  double* Q = (double*)q.ptr;
  double* R = (double*)r.ptr;
  if ((rc = psvd_qr(c, M, K, U, ldu, Q, ldq, R, st)) == PSVD_OK) {
    cudaMemcpyAsync(sg.data(), sigma, sizeof(double) * K, cudaMemcpyDeviceToHost, st);
    cudaMemcpy2DAsync(dg.data(), sizeof(double), R, sizeof(double) * (K + 1), sizeof(double), K,
                      cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    std::vector<int> order(K);
    for (int k = 0; k < K; ++k) {
      sg[k] *= std::fabs(dg[k]);
      order[k] = k;
    }
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return sg[a] > sg[b]; });
    std::vector<double> so(K);
    for (int k = 0; k < K; ++k) {
      so[k] = sg[order[k]];
      cudaMemcpyAsync(U + (size_t)k * ldu, Q + (size_t)order[k] * ldq, sizeof(double) * M, cudaMemcpyDeviceToDevice,
                      st);
    }
    cudaMemcpyAsync(sigma, so.data(), sizeof(double) * K, cudaMemcpyHostToDevice, st);
    or_status_kernel<<<1, 1, 0, st>>>(c->d_status, PSVD_ST_RESCUE);
    c->launches++;
    cudaStreamSynchronize(st);  // so's host buffer
  }
  cudaFree(q.ptr);
  cudaFree(r.ptr);
  return rc ? rc : cuda_check(c, "drift rescue wide");
}

// Core solve of a Gram: eig (+ concurrent LDL^T on the aux stream when the split path applies)
int psvd_internal::core_solve(psvd_ctx* c, const double* G, int n, int K, const double* dscale, double* W, double* sigma,
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
int psvd_internal::refine_normalize(psvd_ctx* c, int64_t M, double* U, int64_t ld, int K, double* UtU,
                                    double* sigma, cudaStream_t st) {
  int rc = ensure(c, c->tbuf, sizeof(double) * ((size_t)K * K + K));
  if (rc) return rc;
  double* scale = (double*)c->tbuf.ptr + (size_t)K * K;
  launch_normalize_gram(UtU, K, sigma, scale, c->d_status, st);
  launch_scale_cols(U, ld, M, K, scale, st);
  c->launches += 2;
  return cuda_check(c, "refine");
}

// exchange points of the row-partitioned randomized update (no-ops on one GPU)
int psvd_internal::ex_allreduce(psvd_ctx* c, double* buf, int64_t count, cudaStream_t st) {
  if (c->nccl_on) return nccl_allreduce_ordered(c, buf, count, st);
  if (!c->ex_allreduce) return PSVD_OK;
  c->ex_calls++;
  c->ex_bytes += 8 * count * (c->ex_nranks - 1);
  if (c->ex_allreduce(c->ex_user, buf, count, (void*)st) != 0) return fail(c, PSVD_ECUDA, "allreduce hook failed");
  return PSVD_OK;
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
