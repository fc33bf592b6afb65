// Warp-specialized TMA pass for narrow panels (see psvd_tall.cuh, "narrow"): Y = P W for a Y of
// <= 32 columns and the Gram tiles P^T Y, Y^T Y in one read of the panel P = [seg_0 | seg_1 | ...].
//
// One CTA per SM streams its row chunk in stages landing in an NS-deep ring signalled by mbarriers
// (complete_tx).  With M a multiple of 16 and two stages fitting, a stage is 32 rows brought by 3-D
// TMA boxes {16 rows, 2, <= 256 columns} (256 contiguous bytes of every column per request); else 16
// rows from 2-D boxes.  128-byte swizzle: the 16-byte chunks of a column are XOR-ed with its unit
// index (swzr).  Warp roles:
//
//   last warp    producer: one lane issues the stage's TMA boxes once the ring slot is released;
//   Y warps      32-row stages: W held in registers, each (8-column block, k part) warp forms all 32
//                rows of its block over its k part, the parts' partial sums meet in the Y tile in
//                part order through an mbarrier chain; the k split is weighted per SMSP by the Gram
//                work placed there.  16-row stages: fragment-reloading Y warps (one 8x8 output block
//                each).  The last part writes Y to global (slice 0) and folds the per-column argmax
//                of |y|;
//   Gram warps   one tile (I, Y) of [P | Y] each, compile-time sub-block shape, sub-blocks nobody
//                reads trimmed at plan time, tiles placed longest-first onto the least-loaded SMSP.
//
// No CTA-wide barrier inside the stage loop: full / empty (panel ring), ydone / yfree (Y double
// buffer) and chain mbarriers only.  Results are bitwise identical run to run (fixed per-warp
// accumulation order, fixed-order tall_reduce afterwards).
#include <cuda.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <type_traits>
#include <vector>

#include "psvd_tall.cuh"

namespace psvd {

namespace {

constexpr int TKS = 16;       // rows per 128-byte swizzled column piece (a stage is TKS or 2 TKS rows)
constexpr int TNS_MAX = 8;    // ring depth: x.ns stages, as many as fit (3 .. 8 of 16 rows, 2 .. 8 of 32)
constexpr int YMAXC = 32;     // widest Y of the narrow pass (4 column blocks)
constexpr int YKP_WR = 16;    // W fragments held in registers per Y warp (k steps of 4 columns)
constexpr int YB = 2;         // Y ring depth (Y warps run up to YB stages ahead of the Gram warps; 4 measured no faster)
constexpr int PROD_WARP = NWARP - 1;
// sW row stride (doubles, = 4 mod 16: 2 wavefronts per B-fragment load), sized by the Y width
// W row stride in doubles: the four W rows of a fragment load must tile the 16 double-banks
// exactly twice (stride = 8 mod 16: w_pad 8 or 24 itself; 4 or 12 mod 16: 20 and 36 for 16 and 32)
__host__ __device__ inline int w_stride(int w_pad) {
  return (w_pad & 15) == 8 ? w_pad : (w_pad <= 16 ? 20 : 36);
}

PSVD_DEV uint32_t saddr(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

PSVD_DEV void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(saddr(bar)), "r"(bytes) : "memory");
}

PSVD_DEV void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::
          "r"(saddr(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(saddr(bar))
      : "memory");
}

// multicast variant: the box lands at the same smem offset in every CTA of ctaMask and
// signals the mbarrier at the same offset in each of them
PSVD_DEV void tma_load_2d_mc(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar, uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.multicast::cluster "
      "[%0], [%1, {%2, %3}], [%4], %5;\n" ::"r"(saddr(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(saddr(bar)), "h"(mask)
      : "memory");
}

// element (column c, stage row k) of a 128B-swizzled 16-row stage, in doubles
PSVD_DEV int swz(int c, int k) { return c * 16 + ((((k >> 1) ^ (c & 7)) << 1) | (k & 1)); }

// RB row blocks of 16 per stage: column c's rows are RB consecutive 128-byte units (the layout a
// 3-D TMA box {16 rows, RB row blocks, columns} lands in), unit u = c RB + (k >> 4) swizzled by u & 7
template <int RB>
PSVD_DEV int swzr(int c, int k) {
  const int u = c * RB + (k >> 4);
  return u * 16 + (((((k & 15) >> 1) ^ (u & 7)) << 1) | (k & 1));
}

PSVD_DEV void tma_load_3d(void* dst, const CUtensorMap* map, int c0, int c1, int c2, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];\n" ::
          "r"(saddr(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(saddr(bar))
      : "memory");
}

}  // namespace

size_t tma_pass_smem_bytes(int pwidth, int kp_span, int w_pad, int ns, int rb) {
  size_t b = 1024;  // alignment slack for the 1024-byte swizzle atoms
  const int sr = TKS * std::max(1, rb);
  b += sizeof(double) * (size_t)ns * pwidth * sr;    // panel ring
  b += sizeof(double) * YB * std::max(w_pad, 8) * sr;  // Y ring (w_pad <= 32 columns)
  b += sizeof(double) * (size_t)kp_span * w_stride(w_pad);  // W
  b += 64 * sizeof(uint64_t);                        // barriers
  b += sizeof(double) * 4 * YMAXC * 3;               // argmax scratch
  return b;
}

template <int RB, bool AOFF = false>
__global__ void __launch_bounds__(NTHR, 1)
    pass_tma_kernel(const __grid_constant__ TallParams p, const __grid_constant__ TmaMaps maps, const TmaExtra x) {
  if (p.gate != nullptr && *p.gate == 0) return;  // gated pass (drift rescue) not needed
  constexpr int SR = TKS * RB;  // rows per stage
  extern __shared__ unsigned char smem_raw[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, tq = lane & 3;
  const int slice = blockIdx.x % p.nslices;
  const int64_t chunk = blockIdx.x / p.nslices;
  const int64_t row_begin = chunk * p.rows_per_cta;
  const int64_t row_end = min(p.M, row_begin + p.rows_per_cta);
  const int np_pad = p.np_pad;  // logical panel width (Y block index boundary)
  const int pw = x.pwidth;       // physical ring width (>= np_pad + pshift)
  const int kspan = x.kp_hi - x.kp_lo;
  const int WSP = w_stride(p.w_pad);
  const int ncb = p.w_pad >> 3;  // Y column blocks (1..4)
  const int nyo = 2 * ncb;       // Y output blocks (2 row blocks of 8 x ncb) per 16-row block
  // 32-row stages: the two 16-row halves of a block go to one warp (yh = 1) or to two (yh = 2)
  const int yh = (RB == 2 && p.yh == 2) ? 2 : 1;
  // 32-row stages, register-resident W: Y warp (cb, kp) holds the W fragments of its k part and
  // forms all 32 rows of column block cb over that part; the ykp partials meet in the Y tile in
  // part order through a chain of mbarriers
  const int ykp = (RB == 2 && p.ykp > 1) ? p.ykp : 1;

  unsigned char* base = smem_raw + ((1024 - (saddr(smem_raw) & 1023)) & 1023);
  double* sP = reinterpret_cast<double*>(base);
  const int TNS = x.ns;
  double* sY = sP + (size_t)TNS * pw * SR;
  const int YC = max(p.w_pad, 8);  // Y ring columns
  double* sW = sY + YB * YC * SR;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sW + (size_t)kspan * WSP);
  uint64_t* full = bars;
  uint64_t* empty = bars + TNS;
  uint64_t* ydone = bars + 2 * TNS;
  uint64_t* yfree = ydone + YB;
  double* cmx = reinterpret_cast<double*>(bars + 64);  // [2 rb][32 cols][val, abs, row]

  uint64_t* chain = bars + 24;  // [YB][4 cb][3 links] (ykp > 1)
  int ngram = 0;
  const int ny = ykp > 1 ? ncb * ykp : nyo * yh;  // Y warps 0 .. ny-1
  for (int w = ny; w < PROD_WARP; ++w) ngram += p.plan[slice][w].ntile > 0;

  // one-time setup: zero the panel columns no TMA box writes (alignment gaps), the Y
  // buffers (columns >= w stay zero), stage W with zero rows for gap columns
  for (int i = tid; i < TNS * pw; i += NTHR) {
    const int c = i % pw;
    if (!x.written[c >> 3]) {
      double* col = sP + (size_t)i * SR;
#pragma unroll
      for (int k = 0; k < SR; ++k) col[k] = 0.0;
    }
  }
  for (int i = tid; i < YB * YC * SR; i += NTHR) sY[i] = 0.0;
  for (int i = tid; i < kspan * WSP; i += NTHR) {
    const int kk = i / WSP, o = i % WSP;
    // rows of each full 8-column step are stored in the Y warps' k order: step half h reads
    // columns 2h + {0, 1, 4, 5} (see the Y warps); the 4-column tail keeps the natural order
    int kperm = kk;
    if (RB == 1 && kk < ((kspan >> 3) << 3)) {
      const int r = kk & 7, h = r >> 2, t = r & 3;
      kperm = (kk & ~7) + 2 * h + (t & 1) + 4 * (t >> 1);
    }
    const int pc = x.kp_lo + kperm;  // physical panel column
    double v = 0.0;
    if (o < p.w) {
      for (int s = 0; s < p.nseg; ++s) {
        const int c0 = p.seg[s].col0 + x.pshift;  // physical start
        if (x.wrow0[s] != TMA_NOT_IN_W && pc >= c0 && pc < c0 + p.seg[s].ncols) {
          const int wr = x.wrow0[s] + (pc - c0);
          if (wr >= 0 && wr < p.wk) v = p.W[(int64_t)o * p.ldw + wr];
        }
      }
    }
    sW[i] = v;
  }
  if (tid == 0) {
    for (int b = 0; b < TNS; ++b) {
      mbar_init(&full[b], 1);
      mbar_init(&empty[b], (unsigned)(ny + ngram));
    }
    for (int b = 0; b < YB; ++b) {
      mbar_init(&ydone[b], 32u * (ykp > 1 ? ncb : ny));
      mbar_init(&yfree[b], (unsigned)max(32 * ngram, 1));
    }
    if (ykp > 1)
      for (int i = 0; i < YB * 4 * 3; ++i) mbar_init(&chain[i], 32u);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");  // zero fills before the first TMA writes
  __syncthreads();
  const int64_t nstage = row_end > row_begin ? (row_end - row_begin + SR - 1) / SR : 0;

  if (warp == PROD_WARP) {
    if (lane == 0) {
      // stages are issued in groups of x.grp consecutive ones, box by box, so each column's
      // grp x 128 contiguous bytes reach DRAM back to back (a lone 128-byte piece per column
      // and stage is a poor DRAM access: tools/colmajor_bw.cu measured 16-row chunks at ~60%
      // of the 64-row rate)
      const int G = x.grp;
      for (int64_t s0 = 0; s0 < nstage; s0 += G) {
        const int64_t s1 = min(nstage, s0 + G);
        for (int64_t s = s0; s < s1; ++s) {
          const int si = (int)s, b = si % TNS;
          if (si >= TNS) mbar_wait(&empty[b], (unsigned)(((si / TNS) - 1) & 1));
          mbar_expect_tx(&full[b], p.dbg == 2 ? 0u : x.stage_bytes);  // dbg 2: no loads (compute-only timing)
        }
        if (p.dbg == 2) continue;
        for (int o = 0; o < x.nops; ++o)
          for (int64_t s = s0; s < s1; ++s) {
            const int b = (int)s % TNS;
            double* dst = sP + (size_t)b * pw * SR + (size_t)x.op_pcol[o] * SR;
            const int r0 = (int)(row_begin + s * SR);
            if (RB == 1)
              tma_load_2d(dst, &maps.m[x.op_seg[o]], r0, x.op_col[o], &full[b]);
            else  // rows r0 .. r0 + SR - 1 of every column: SR * 8 contiguous bytes per column
              tma_load_3d(dst, &maps.m[x.op_seg[o]], 0, r0 / TKS, x.op_col[o], &full[b]);
          }
      }
    }
    return;
  }

  if (RB == 2 && ykp > 1 && warp < ny) {
    // ---------------------------------------------------------------- Y warps, W in registers
    const int cb = warp % ncb, kp = warp / ncb;
    // k steps of 4 columns of this part: sized on the host so that every SMSP carries the same
    // DMMA count per stage, its Gram tiles included (nj <= YKP_WR)
    const int j0 = p.ykj0[warp], nj = p.yknj[warp];
    double wr[YKP_WR];
#pragma unroll
    for (int j = 0; j < YKP_WR; ++j)
      wr[j] = j < nj ? sW[(size_t)(4 * (j0 + j) + tq) * WSP + cb * 8 + g] : 0.0;
    const bool last = kp == ykp - 1;
    const bool do_y = slice == 0 && last;
    // element (column kp_lo + 4 (j0 + j) + tq, row 16 h + rr) of a stage is unit u = 2 kp_lo + 8 (j0 + j)
    // + 2 tq + h with u & 7 = 2 tq + h whatever j (kp_lo is a multiple of 8): swzr<2> = a per-lane offset
    // + 128 j, no address arithmetic per load
    int aoff[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int h = q >> 1, rr = (q & 1) * 8 + g;
      aoff[q] = (2 * (x.kp_lo + 4 * j0 + tq) + h) * 16 + ((((rr >> 1) ^ (2 * tq + h)) << 1) | (rr & 1));
    }
    double cm_val[2] = {0.0, 0.0}, cm_abs[2] = {-1.0, -1.0};
    int64_t cm_row[2] = {-1, -1};
    int b = 0;
    unsigned ph = 0;
    for (int64_t s = 0; s < nstage; ++s, (++b == TNS ? (b = 0, ph ^= 1u) : 0u)) {
      const int yb = (int)(s & (YB - 1));
      const unsigned yph = (unsigned)(((int)s / YB) & 1);
      mbar_wait(&full[b], ph);
      const double* P = sP + (size_t)b * pw * SR;
      // 4 row blocks of 8 (q = 2 h + rb), 4 independent accumulator chains; column c of step j is
      // unit 2c + h, phase (2 (k0 + tq) + h) & 7: conflict-free across tq
      double acc[4][2];
#pragma unroll
      for (int q = 0; q < 4; ++q) acc[q][0] = acc[q][1] = 0.0;
      const int cbase = x.kp_lo + 4 * j0 + tq;
      // AOFF: precomputed per-lane offsets, no address arithmetic per load.  Measured faster for one or
      // two Y column blocks (the recompose: 0.43 -> 0.38 ms) and slower for three (the randomized passes'
      // 12 Y warps: 0.53 -> 0.63 ms), so the launch picks the instantiation by Y width
#pragma unroll
      for (int j = 0; j < YKP_WR; ++j) {
        if (j < nj && p.dbg != 1) {
          const int c = cbase + 4 * j;
          double a[4];
#pragma unroll
          for (int q = 0; q < 4; ++q)
            a[q] = AOFF ? P[aoff[q] + 128 * j] : P[swzr<2>(c, (q >> 1) * 16 + (q & 1) * 8 + g)];
#pragma unroll
          for (int q = 0; q < 4; ++q) dmma884(acc[q][0], acc[q][1], a[q], wr[j]);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[b]);  // panel slot no longer read by this warp
      double* Ys = sY + (size_t)yb * YC * SR;
      const int o0 = cb * 8 + 2 * tq;
      if (kp == 0 || p.dbg == 3) {  // dbg 3 (timing only, wrong Y): parts do not wait for each other
        if ((kp == 0 || last) && s >= YB && ngram > 0) mbar_wait(&yfree[yb], yph ^ 1u);
      } else {
        mbar_wait(&chain[(yb * 4 + cb) * 3 + kp - 1], yph);  // the partial sum of parts 0 .. kp-1
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int r = (q >> 1) * 16 + (q & 1) * 8 + g;
          acc[q][0] = Ys[swzr<2>(o0, r)] + acc[q][0];
          acc[q][1] = Ys[swzr<2>(o0 + 1, r)] + acc[q][1];
        }
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int r = (q >> 1) * 16 + (q & 1) * 8 + g;
        Ys[swzr<2>(o0, r)] = acc[q][0];
        Ys[swzr<2>(o0 + 1, r)] = acc[q][1];
      }
      if (!last) {
        mbar_arrive(&chain[(yb * 4 + cb) * 3 + kp]);
        continue;
      }
      mbar_arrive(&ydone[yb]);
      if (do_y) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {  // q = 2 h + rb: rows 8 q + g, increasing (first occurrence kept)
          const int64_t row = row_begin + s * SR + 8 * q + g;
          const double y0 = acc[q][0], y1 = acc[q][1];
          if (row >= row_end) continue;
          if (p.Yout != nullptr) {
            if (o0 < p.w) p.Yout[(int64_t)o0 * p.ldy + row] = y0;
            if (o0 + 1 < p.w) p.Yout[(int64_t)(o0 + 1) * p.ldy + row] = y1;
          }
          if (p.colmax != nullptr) {
            if (fabs(y0) > cm_abs[0]) { cm_abs[0] = fabs(y0); cm_val[0] = y0; cm_row[0] = row; }
            if (fabs(y1) > cm_abs[1]) { cm_abs[1] = fabs(y1); cm_val[1] = y1; cm_row[1] = row; }
          }
        }
      }
    }
    if (do_y && p.colmax != nullptr) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
#pragma unroll
        for (int off = 4; off < 32; off <<= 1) {
          const double oa = __shfl_xor_sync(0xffffffffu, cm_abs[e], off);
          const double ov = __shfl_xor_sync(0xffffffffu, cm_val[e], off);
          const long long orow = __shfl_xor_sync(0xffffffffu, (long long)cm_row[e], off);
          if (oa > cm_abs[e] || (oa == cm_abs[e] && orow >= 0 && (cm_row[e] < 0 || orow < cm_row[e]))) {
            cm_abs[e] = oa; cm_val[e] = ov; cm_row[e] = orow;
          }
        }
        const int o = cb * 8 + 2 * tq + e;
        if (g == 0 && o < p.w) {
          double* dst = p.colmax + ((size_t)chunk * p.w + o) * 2;
          dst[0] = cm_val[e];
          dst[1] = (double)cm_row[e] + (double)p.row_offset;
        }
      }
    }
    return;
  }

  if (warp < ny) {
    // ---------------------------------------------------------------- Y warps
    // warp -> output block blk = (rb, cb) of every 16-row block h it owns (all of a stage's
    // halves when yh == 1, half hp when yh == 2), over the whole k range
    const int blk = warp % nyo, hp = warp / nyo;
    const int rb = blk & 1, cb = blk >> 1;
    const int h_lo = yh == 2 ? hp : 0, h_hi = yh == 2 ? hp + 1 : RB;
    const int k_lo = x.kp_lo, k_hi = x.kp_hi;
    double cm_val[2] = {0.0, 0.0}, cm_abs[2] = {-1.0, -1.0};
    int64_t cm_row[2] = {-1, -1};
    const bool do_y = slice == 0;
    // ring position (b, phase) advanced per stage: no 64-bit divisions in the stage loop
    int b = 0;
    unsigned ph = 0;
    for (int64_t s = 0; s < nstage; ++s, (++b == TNS ? (b = 0, ph ^= 1u) : 0u)) {
      const int yb = (int)(s & (YB - 1));
      mbar_wait(&full[b], ph);
      const double* P = sP + (size_t)b * pw * SR;
      const int kr = rb * 8 + g;
      double y0h[RB], y1h[RB];
#pragma unroll
      for (int h = 0; h < RB; ++h) {
        y0h[h] = y1h[h] = 0.0;
        if (h < h_lo || h >= h_hi) continue;
        // RB == 1: kp_lo is a multiple of 8, so the swizzle phase of a column is fixed per lane and
        // the fragment addresses advance by 8 columns per step.  Step half h of an 8-column step
        // reads columns k0 + 2h + {0, 1, 4, 5}[tq] (the four columns of a fragment then fall in
        // both 64-byte halves of the swizzled rows: 2 wavefronts per LDS); W's rows follow.
        // RB == 2: the unit phase is (2 c + h) & 7, already spread by the natural order k0 + tq.
        // Groups of 4 steps: 16 independent loads, then 8 DMMAs on 4 chains (the per-warp
        // load -> DMMA latency chain bounded the one-step loop).
        int colA, colB, phA, phB;
        if (RB == 1) {
          colA = (tq & 1) + 4 * (tq >> 1);
          colB = colA + 2;
          phA = colA;
          phB = colB;
        } else {
          colA = tq;
          colB = tq + 4;
          phA = (RB * tq + h) & 7;
          phB = phA;
        }
        const double* pa = P + (size_t)(RB * (k_lo + colA) + h) * 16 + ((((kr >> 1) ^ phA) << 1) | (kr & 1));
        const double* pb = P + (size_t)(RB * (k_lo + colB) + h) * 16 + ((((kr >> 1) ^ phB) << 1) | (kr & 1));
        constexpr int STEP = 128 * RB;  // doubles per 8 columns
        const double* wa = sW + (size_t)(k_lo - x.kp_lo + tq) * WSP + cb * 8 + g;
        const double* wbp = wa + (size_t)4 * WSP;
        double c0 = 0.0, c1 = 0.0, c2 = 0.0, c3 = 0.0, c4 = 0.0, c5 = 0.0, c6 = 0.0, c7 = 0.0;
        const int n8 = p.dbg == 1 ? 0 : (k_hi - k_lo) >> 3;
        int i = 0;
#pragma unroll 1
        for (; i + 4 <= n8; i += 4) {
          double fa[8], fw[8];
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            fa[2 * j] = pa[(size_t)(i + j) * STEP];
            fa[2 * j + 1] = pb[(size_t)(i + j) * STEP];
            fw[2 * j] = wa[(size_t)(8 * (i + j)) * WSP];
            fw[2 * j + 1] = wbp[(size_t)(8 * (i + j)) * WSP];
          }
          dmma884(c0, c1, fa[0], fw[0]);
          dmma884(c2, c3, fa[1], fw[1]);
          dmma884(c4, c5, fa[2], fw[2]);
          dmma884(c6, c7, fa[3], fw[3]);
          dmma884(c0, c1, fa[4], fw[4]);
          dmma884(c2, c3, fa[5], fw[5]);
          dmma884(c4, c5, fa[6], fw[6]);
          dmma884(c6, c7, fa[7], fw[7]);
        }
        for (; i < n8; ++i) {
          dmma884(c0, c1, pa[(size_t)i * STEP], wa[(size_t)(8 * i) * WSP]);
          dmma884(c2, c3, pb[(size_t)i * STEP], wbp[(size_t)(8 * i) * WSP]);
        }
        if (p.dbg != 1 && k_lo + 8 * n8 < k_hi)  // kp span is a multiple of 4; natural order
          dmma884(c4, c5, P[swzr<RB>(k_lo + 8 * n8 + tq, kr + 16 * h)], wa[(size_t)(8 * n8) * WSP]);
        y0h[h] = (c0 + c4) + (c2 + c6);
        y1h[h] = (c1 + c5) + (c3 + c7);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[b]);  // panel slot no longer read by this warp
      if (s >= YB && ngram > 0) mbar_wait(&yfree[yb], (unsigned)((((int)s / YB) - 1) & 1));
      double* Ys = sY + (size_t)yb * YC * SR;
      const int o0 = cb * 8 + 2 * tq;
#pragma unroll
      for (int h = 0; h < RB; ++h) {
        if (h < h_lo || h >= h_hi) continue;
        Ys[swzr<RB>(o0, kr + 16 * h)] = y0h[h];
        Ys[swzr<RB>(o0 + 1, kr + 16 * h)] = y1h[h];
      }
      mbar_arrive(&ydone[yb]);
#pragma unroll
      for (int h = 0; h < RB; ++h) {
        if (h < h_lo || h >= h_hi) continue;
        const int64_t r = row_begin + s * SR + 16 * h + kr;
        const double y0 = y0h[h], y1 = y1h[h];
        if (do_y && r < row_end) {
          if (p.Yout != nullptr) {
            if (o0 < p.w) p.Yout[(int64_t)o0 * p.ldy + r] = y0;
            if (o0 + 1 < p.w) p.Yout[(int64_t)(o0 + 1) * p.ldy + r] = y1;
          }
          if (p.colmax != nullptr) {
            if (fabs(y0) > cm_abs[0]) { cm_abs[0] = fabs(y0); cm_val[0] = y0; cm_row[0] = r; }
            if (fabs(y1) > cm_abs[1]) { cm_abs[1] = fabs(y1); cm_val[1] = y1; cm_row[1] = r; }
          }
        }
      }
    }
    if (do_y && p.colmax != nullptr) {
      // combine over g (lanes 4 apart), ties to the smaller row (first occurrence)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
#pragma unroll
        for (int off = 4; off < 32; off <<= 1) {
          const double oa = __shfl_xor_sync(0xffffffffu, cm_abs[e], off);
          const double ov = __shfl_xor_sync(0xffffffffu, cm_val[e], off);
          const long long orow = __shfl_xor_sync(0xffffffffu, (long long)cm_row[e], off);
          if (oa > cm_abs[e] || (oa == cm_abs[e] && orow >= 0 && (cm_row[e] < 0 || orow < cm_row[e]))) {
            cm_abs[e] = oa; cm_val[e] = ov; cm_row[e] = orow;
          }
        }
      }
      if (g == 0) {
        for (int e = 0; e < 2; ++e) {
          double* d = cmx + ((size_t)(rb + 2 * hp) * YMAXC + cb * 8 + 2 * tq + e) * 3;
          d[0] = cm_val[e]; d[1] = cm_abs[e]; d[2] = (double)cm_row[e];
        }
      }
      asm volatile("bar.sync 1, %0;\n" ::"r"(32 * ny) : "memory");
      if (rb == 0 && hp == 0 && g == 0) {
        for (int e = 0; e < 2; ++e) {
          const int o = cb * 8 + 2 * tq + e;
          if (o >= p.w) continue;
          const double* d = cmx + (size_t)o * 3;
          for (int q = 1; q < 2 * yh; ++q) {  // ties: the smaller row (first occurrence)
            const double* d1 = cmx + ((size_t)q * YMAXC + o) * 3;
            if (d1[1] > d[1] || (d1[1] == d[1] && d1[2] >= 0 && (d[2] < 0 || d1[2] < d[2]))) d = d1;
          }
          double* dst = p.colmax + ((size_t)chunk * p.w + o) * 2;
          dst[0] = d[0];
          dst[1] = d[2] + (double)p.row_offset;
        }
      }
    }
    return;
  }

  // ---------------------------------------------------------------- Gram warps
  const WarpPlan wp = p.plan[slice][warp];
  if (wp.ntile == 0) return;
  const int I = wp.ti[0];
  const bool i_is_y = I * 32 >= np_pad;
  // P-tile: the wanted 8-column sub-blocks a0 .. a0 + na - 1 (plan_pass trims unwanted rows)
  const int a0 = (!i_is_y && wp.sub != 0) ? (wp.sub & 15) : 0;
  const int na = i_is_y ? ncb : wp.sub != 0 ? (wp.sub >> 4) : min(4, (p.np - I * 32 + 7) / 8);
  const int acol = I * 32 + x.pshift + a0 * 8;  // physical first column of a panel tile
  double acc[4][4][2];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int c = 0; c < 4; ++c) acc[a][c][0] = acc[a][c][1] = 0.0;
  auto stage_loop = [&](auto na_t, auto nb_t) {
    constexpr int NA = decltype(na_t)::value, NB = decltype(nb_t)::value;
    int b = 0;
    unsigned ph = 0;
    for (int64_t s = 0; s < nstage; ++s, (++b == TNS ? (b = 0, ph ^= 1u) : 0u)) {
      const int yb = (int)(s & (YB - 1));
      mbar_wait(&full[b], ph);
      mbar_wait(&ydone[yb], (unsigned)(((int)s / YB) & 1));
      const double* Ys = sY + (size_t)yb * YC * SR;
      const double* Abase = sP + (size_t)b * pw * SR;
#pragma unroll
      for (int kk = 0; kk < SR / 4; ++kk) {
        const int k = kk * 4 + tq;
        double fa[NA], fb[NB];
#pragma unroll
        for (int q = 0; q < NA; ++q)
          fa[q] = i_is_y ? Ys[swzr<RB>(q * 8 + g, k)] : Abase[swzr<RB>(acol + q * 8 + g, k)];
#pragma unroll
        for (int q = 0; q < NB; ++q) fb[q] = Ys[swzr<RB>(q * 8 + g, k)];
        if (p.dbg != 1)
#pragma unroll
          for (int a = 0; a < NA; ++a)
#pragma unroll
            for (int c = 0; c < NB; ++c) dmma884(acc[a][c][0], acc[a][c][1], fa[a], fb[c]);
      }
      mbar_arrive(&yfree[yb]);
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[b]);
    }
  };
  using I1 = std::integral_constant<int, 1>;
  using I2 = std::integral_constant<int, 2>;
  using I3 = std::integral_constant<int, 3>;
  using I4 = std::integral_constant<int, 4>;
  auto with_na = [&](auto nb_t) {
    if (na == 4) stage_loop(I4{}, nb_t);
    else if (na == 3) stage_loop(I3{}, nb_t);
    else if (na == 2) stage_loop(I2{}, nb_t);
    else stage_loop(I1{}, nb_t);
  };
  if (ncb == 4) with_na(I4{});
  else if (ncb == 3) with_na(I3{});
  else if (ncb == 2) with_na(I2{});
  else with_na(I1{});
  double* dst = p.partial + ((size_t)blockIdx.x * SLOTS + warp * TPW) * 1024;
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      // accumulator a holds sub-block a0 + a: rows outside the computed range are zero
      double v0 = 0.0, v1 = 0.0;
#pragma unroll
      for (int s = 0; s < 4; ++s)
        if (s + a0 == a) v0 = acc[s][c][0], v1 = acc[s][c][1];
      *reinterpret_cast<double2*>(dst + (a * 8 + g) * 32 + c * 8 + 2 * tq) = make_double2(v0, v1);
    }
}

// ---------------------------------------------------------------- TMA Gram (w == 0)
// Gram-only pass fed by TMA: 32-row stages (two 16-row 128B-swizzled boxes per segment)
// in a GNS-deep ring; warp 15 lane 0 issues the boxes, warps 0..14 each own one 32x32
// tile (compile-time block shape, as gram_ws_kernel) and never meet at a CTA barrier.
constexpr int GNS = 3;

size_t gram_tma_smem_bytes(int np_pad) {
  return 1024 + sizeof(double) * (size_t)GNS * 2 * np_pad * TKS + 2 * GNS * sizeof(uint64_t) + 64;
}

// MC: the two slice CTAs of a row chunk form a cluster and share every stage through
// TMA multicast (each producer loads one 16-row half into both CTAs), so the panel is
// read from HBM/L2 once instead of once per slice.  Consumers release a ring slot on
// both CTAs' empty barriers (the producer overwrites it in both).
template <bool MC>
__global__ void __launch_bounds__(NTHR, 1)
    gram_tma_kernel(const __grid_constant__ TallParams p, const __grid_constant__ TmaMaps maps, const TmaExtra x) {
  if (p.gate != nullptr && *p.gate == 0) return;  // uniform over the grid (and a cluster)
  extern __shared__ unsigned char smem_raw[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, tq = lane & 3;
  const int slice = blockIdx.x % p.nslices;
  const int64_t chunk = blockIdx.x / p.nslices;
  const int64_t row_begin = chunk * p.rows_per_cta;
  const int64_t row_end = min(p.M, row_begin + p.rows_per_cta);
  const int np_pad = p.np_pad;
  unsigned char* base = smem_raw + ((1024 - (saddr(smem_raw) & 1023)) & 1023);
  double* sP = reinterpret_cast<double*>(base);  // [stage][half][np_pad][16]
  uint64_t* full = reinterpret_cast<uint64_t*>(sP + (size_t)GNS * 2 * np_pad * TKS);
  uint64_t* empty = full + GNS;
  unsigned crank = 0;
  if (MC) asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(crank));
  int ncons = 0;
  for (int w = 0; w < PROD_WARP; ++w) ncons += p.plan[slice][w].ntile > 0;
  int nrel = ncons;  // arrivals that release a ring slot
  if (MC) {
    nrel = 0;
    for (int s2 = 0; s2 < 2; ++s2)
      for (int w = 0; w < PROD_WARP; ++w) nrel += p.plan[s2][w].ntile > 0;
  }
  for (int i = tid; i < GNS * 2 * np_pad; i += NTHR) {
    const int c = i % np_pad;
    if (!x.written[c >> 3]) {
      double* col = sP + (size_t)i * TKS;
#pragma unroll
      for (int k = 0; k < TKS; ++k) col[k] = 0.0;
    }
  }
  if (tid == 0) {
    for (int b = 0; b < GNS; ++b) {
      mbar_init(&full[b], 1);
      mbar_init(&empty[b], (unsigned)max(nrel, 1));
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  __syncthreads();
  if (MC) asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
  const int64_t nstage = row_end > row_begin ? (row_end - row_begin + 2 * TKS - 1) / (2 * TKS) : 0;

  if (warp == PROD_WARP) {
    if (lane == 0) {
      for (int64_t s = 0; s < nstage; ++s) {
        const int b = (int)(s % GNS);
        if (s >= GNS) mbar_wait(&empty[b], (unsigned)(((s / GNS) - 1) & 1));
        mbar_expect_tx(&full[b], 2 * x.stage_bytes);  // both halves land here (one per producer when MC)
        for (int h = MC ? (int)crank : 0; h < (MC ? (int)crank + 1 : 2); ++h) {
          double* dst = sP + ((size_t)b * 2 + h) * np_pad * TKS;
          const int r0 = (int)(row_begin + s * 2 * TKS + h * TKS);
          for (int o = 0; o < x.nops; ++o) {
            if (MC)
              tma_load_2d_mc(dst + (size_t)x.op_pcol[o] * TKS, &maps.m[x.op_seg[o]], r0, x.op_col[o], &full[b], 0x3);
            else
              tma_load_2d(dst + (size_t)x.op_pcol[o] * TKS, &maps.m[x.op_seg[o]], r0, x.op_col[o], &full[b]);
          }
        }
      }
    }
  } else if (p.plan[slice][warp].ntile > 0) {
    const WarpPlan wp = p.plan[slice][warp];
    double acc[4][4][2];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int c = 0; c < 4; ++c) acc[a][c][0] = acc[a][c][1] = 0.0;
    const int I = wp.ti[0], J = wp.tj[0];
    const int nva = min(4, (p.np - I * 32 + 7) / 8), nvb = min(4, (p.np - J * 32 + 7) / 8);
    // element (column 8 q + g, row 4 kk + tq) of a 16-row half is swz = 128 q + goff[kk] (the swizzle phase
    // of a column is g whatever q): per-lane offsets, no address arithmetic per load
    int goff[TKS / 4];
#pragma unroll
    for (int kk = 0; kk < TKS / 4; ++kk) goff[kk] = swz(g, kk * 4 + tq);
    uint32_t peer_empty = 0;
    if (MC) {
      const uint32_t loc = saddr(&empty[0]);
      asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(peer_empty) : "r"(loc), "r"(crank ^ 1u));
    }
    auto stage_loop = [&](auto na_t, auto nb_t, auto diag_t) {
      constexpr int NA = decltype(na_t)::value, NB = decltype(nb_t)::value;
      constexpr bool DIAG = decltype(diag_t)::value;
      for (int64_t s = 0; s < nstage; ++s) {
        const int b = (int)(s % GNS);
        mbar_wait(&full[b], (unsigned)((s / GNS) & 1));
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const double* H = sP + ((size_t)b * 2 + h) * np_pad * TKS;
          const double* bI = H + (size_t)I * 32 * TKS;
          const double* bJ = H + (size_t)J * 32 * TKS;
#pragma unroll
          for (int kk = 0; kk < TKS / 4; ++kk) {
            double fa[NA], fb[NB];
#pragma unroll
            for (int q = 0; q < NA; ++q) fa[q] = bI[goff[kk] + 128 * q];
#pragma unroll
            for (int q = 0; q < NB; ++q) fb[q] = bJ[goff[kk] + 128 * q];
#pragma unroll
            for (int a = 0; a < NA; ++a)
#pragma unroll
              for (int c = 0; c < NB; ++c)
                if (!DIAG || c >= a) dmma884(acc[a][c][0], acc[a][c][1], fa[a], fb[c]);
          }
        }
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(&empty[b]);
          if (MC) {
            const uint32_t remote = peer_empty + (uint32_t)(b * sizeof(uint64_t));
            asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];\n" ::"r"(remote) : "memory");
          }
        }
      }
    };
    using F = std::false_type;
    using T = std::true_type;
    using I1 = std::integral_constant<int, 1>;
    using I2 = std::integral_constant<int, 2>;
    using I3 = std::integral_constant<int, 3>;
    using I4 = std::integral_constant<int, 4>;
    if (I != J) {
      if (nvb == 4) stage_loop(I4{}, I4{}, F{});
      else if (nvb == 3) stage_loop(I4{}, I3{}, F{});
      else if (nvb == 2) stage_loop(I4{}, I2{}, F{});
      else stage_loop(I4{}, I1{}, F{});
    } else {
      if (nva == 4) stage_loop(I4{}, I4{}, T{});
      else if (nva == 3) stage_loop(I3{}, I3{}, T{});
      else if (nva == 2) stage_loop(I2{}, I2{}, T{});
      else stage_loop(I1{}, I1{}, T{});
    }
    double* dst = p.partial + ((size_t)blockIdx.x * SLOTS + warp * TPW) * 1024;
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int c = 0; c < 4; ++c)
        *reinterpret_cast<double2*>(dst + (a * 8 + g) * 32 + c * 8 + 2 * tq) =
            make_double2(acc[a][c][0], acc[a][c][1]);
  }
  // neither CTA may exit while its peer can still multicast into it or arrive on its barriers
  if (MC) {
    __syncwarp();
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
  }
}

void launch_gram_tma(const TallParams& p, const TmaMaps& maps, const TmaExtra& x, int grid, cudaStream_t st) {
  const size_t smem = gram_tma_smem_bytes(p.np_pad);
  // Multicast halves the panel traffic of a two-slice Gram but couples the two CTAs' pace
  // (measured slower at B = 200: 25.8 vs 29.7 TF/s), so it is opt-in (PSVD_GRAM_MULTICAST=1).
  static const bool mc = getenv("PSVD_GRAM_MULTICAST") != nullptr;
  if (p.nslices == 2 && grid % 2 == 0 && mc) {
    cudaFuncSetAttribute(gram_tma_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3(NTHR);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, gram_tma_kernel<true>, p, maps, x);
    return;
  }
  cudaFuncSetAttribute(gram_tma_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  gram_tma_kernel<false><<<grid, NTHR, smem, st>>>(p, maps, x);
}

// ---------------------------------------------------------------- split-ring pass
// First built for the deterministic stream's fused pass over [U | A_b | A_next] (psvd_tall.cuh:
// FusedSplit): a 32-row stage of that whole panel does not fit shared memory twice, which had left the
// pass on 16-row stages (128 contiguous bytes per column and request, ~4.5 TB/s).  Here a stage is split
// by column group: group A = the segments under W (read by the Y warps) and group B = the others (read
// by the tile warps), each group in its own ring of 3-D boxes {16 rows, 2, columns} (256 contiguous bytes
// per column); a slot is released by its own readers.  W lives in the Y warps' registers (nkp k parts per
// column block, partial sums met in the Y tile in part order, as in pass_tma_kernel), staged once through
// ring memory.  Tile warps: P^T Y over runs of 8-column sub-blocks of either group, Y^T Y, and offloaded
// 32 x 32 tiles of group B's Gram that the look-ahead Gram then skips.  Every load address is a per-lane
// offset plus a compile-time constant (the swizzle phase of a column repeats every 8 columns).
namespace {

PSVD_DEV bool mbar_test(uint64_t* bar, unsigned parity) {
  uint32_t ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok)
      : "r"(saddr(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}

}  // namespace

constexpr int FS_YB = 2;  // Y ring depth: the Y warps run up to FS_YB stages ahead of the tile warps

size_t fused_split_smem_bytes(const FusedSplit& fs) {
  return 1024 + sizeof(double) * (size_t)fs.ns * (fs.pwA + fs.pwB) * 32 + sizeof(double) * FS_YB * 8 * (size_t)fs.ncb * 32 +
         64 * sizeof(uint64_t);
}

template <int NCB>
__global__ void __launch_bounds__(NTHR, 1)
    fused_split_kernel(const __grid_constant__ TallParams p, const __grid_constant__ TmaMaps maps,
                       const __grid_constant__ TmaExtra x, const __grid_constant__ FusedSplit fs) {
  constexpr int SR = 32, YC = 8 * NCB;
  extern __shared__ unsigned char smem_raw[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, tq = lane & 3;
  const int64_t row_begin = (int64_t)blockIdx.x * p.rows_per_cta;
  const int64_t row_end = min(p.M, row_begin + p.rows_per_cta);
  unsigned char* base = smem_raw + ((1024 - (saddr(smem_raw) & 1023)) & 1023);
  const size_t szA = (size_t)fs.pwA * SR, szB = (size_t)fs.pwB * SR;  // doubles per slot
  const int NS = fs.ns;                                               // slots per ring (2 .. FS_NS_MAX)
  double* ring = reinterpret_cast<double*>(base);                     // [A0 | B0 | A1 | B1 | ...]
  double* sY = ring + (size_t)NS * (szA + szB);                       // [FS_YB][YC columns][32 rows], swzr<2>
  uint64_t* bars = reinterpret_cast<uint64_t*>(sY + FS_YB * YC * SR);
  uint64_t *fullA = bars, *emptyA = bars + FS_NS_MAX, *fullB = bars + 2 * FS_NS_MAX, *emptyB = bars + 3 * FS_NS_MAX,
           *ydone = bars + 4 * FS_NS_MAX, *yfree = ydone + FS_YB, *chain = yfree + FS_YB;  // chain[(yb * NCB + cb) * 3 + link]
  const int WSP = w_stride(YC);
  double* sW = ring;  // W staged through slot A0 before the first box lands there

  for (int i = tid; i < fs.n4 * 4 * WSP; i += NTHR) {
    const int pc = fs.colA0 + i / WSP, o = i % WSP;  // physical panel column, Y column
    double v = 0.0;
    if (o < p.w) {
      for (int s = 0; s < p.nseg; ++s) {
        const int c0 = p.seg[s].col0;
        if (x.wrow0[s] != TMA_NOT_IN_W && pc >= c0 && pc < c0 + p.seg[s].ncols) {
          const int wr = x.wrow0[s] + (pc - c0);
          if (wr >= 0 && wr < p.wk) v = p.W[(int64_t)o * p.ldw + wr];
        }
      }
    }
    sW[i] = v;
  }
  for (int i = tid; i < FS_YB * YC * SR; i += NTHR) sY[i] = 0.0;
  if (tid == 0) {
    for (int b = 0; b < NS; ++b) {
      mbar_init(&fullA[b], 1);
      mbar_init(&fullB[b], 1);
      mbar_init(&emptyA[b], (unsigned)max(fs.nA, 1));
      mbar_init(&emptyB[b], (unsigned)max(fs.nB, 1));
    }
    for (int b = 0; b < FS_YB; ++b) {
      mbar_init(&ydone[b], 32u * NCB);
      mbar_init(&yfree[b], (unsigned)max(32 * fs.npy, 1));
    }
    for (int i = 0; i < FS_YB * NCB * 3; ++i) mbar_init(&chain[i], 32u);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  const int role = fs.role[warp];
  double wr[FS_WR];
  if (role == FS_Y) {
    const int cb = fs.ycb[warp], j0 = fs.yj0[warp], nj = fs.ynj[warp];
#pragma unroll
    for (int j = 0; j < FS_WR; ++j) wr[j] = j < nj ? sW[(size_t)(4 * (j0 + j) + tq) * WSP + cb * 8 + g] : 0.0;
  }
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");  // generic accesses of the ring before the boxes
  __syncthreads();
  const int64_t nstage = row_end > row_begin ? (row_end - row_begin + SR - 1) / SR : 0;
  // tile warps: element (column 8 b + g, row 4 kk + tq) of a 32-row stage is swzr<2> = 256 b + eoff[kk]:
  // unit 16 b + 2 g + (kk >> 2), phase (2 g + (kk >> 2)) & 7 -- per-lane offsets, no arithmetic per load
  int eoff[SR / 4];
#pragma unroll
  for (int kk = 0; kk < SR / 4; ++kk) eoff[kk] = swzr<2>(g, kk * 4 + tq);

  if (role == FS_PROD) {
    if (lane == 0) {
      // one lane feeds both rings: whichever group's slot is free gets its next stage
      int64_t a = 0, b = 0;
      int pia = 0, pib = 0;       // ring positions of stages a and b
      unsigned pha = 1, phb = 1;  // parity of the release that frees them: ((stage / NS) - 1) & 1
      while (a < nstage || b < nstage) {
        if (a < nstage) {
          const int pi = pia;
          if (a < NS || mbar_test(&emptyA[pi], pha)) {
            mbar_expect_tx(&fullA[pi], p.dbg == 2 ? 0u : fs.bytesA);  // dbg 2: no loads (compute-only timing)
            double* dst = ring + (size_t)pi * (szA + szB);
            const int r16 = (int)((row_begin + a * SR) / TKS);
            for (int o = 0; o < (p.dbg == 2 ? 0 : fs.nopsA); ++o)
              tma_load_3d(dst + (size_t)fs.opd[o] * SR, &maps.m[fs.opm[o]], 0, r16, fs.opc[o], &fullA[pi]);
            ++a;
            if (++pia == NS) pia = 0, pha ^= 1u;
          }
        }
        if (fs.nopsB == 0) b = nstage;  // no group B (a recompose)
        if (b < nstage) {
          const int pi = pib;
          if (b < NS || mbar_test(&emptyB[pi], phb)) {
            mbar_expect_tx(&fullB[pi], p.dbg == 2 ? 0u : fs.bytesB);
            double* dst = ring + (size_t)pi * (szA + szB) + szA;
            const int r16 = (int)((row_begin + b * SR) / TKS);
            for (int o = fs.nopsA; o < (p.dbg == 2 ? 0 : fs.nopsA + fs.nopsB); ++o)
              tma_load_3d(dst + (size_t)fs.opd[o] * SR, &maps.m[fs.opm[o]], 0, r16, fs.opc[o], &fullB[pi]);
            ++b;
            if (++pib == NS) pib = 0, phb ^= 1u;
          }
        }
      }
    }
    return;
  }

  if (role == FS_Y) {
    const int cb = fs.ycb[warp], kp = fs.ykp[warp], j0 = fs.yj0[warp], nj = fs.ynj[warp];
    const bool last = kp == fs.nkp - 1;
    const int o0 = cb * 8 + 2 * tq;
    // element (column 4 (j0 + j) + tq, row 16 h + rr) of a stage is unit u = 8 (j0 + j) + 2 tq + h with
    // u & 7 = 2 tq + h whatever j: swzr<2> = a per-lane offset + 128 j, no address arithmetic per load
    int aoff[4], yoff[4][2];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int h = q >> 1, rr = (q & 1) * 8 + g;
      aoff[q] = (8 * j0 + 2 * tq + h) * 16 + ((((rr >> 1) ^ (2 * tq + h)) << 1) | (rr & 1));
      yoff[q][0] = swzr<2>(o0, 16 * h + rr);
      yoff[q][1] = swzr<2>(o0 + 1, 16 * h + rr);
    }
    // the step count of a part is a compile-time constant of its stage loop: no branch per step and the
    // fragment loads of later steps issue under the DMMAs of earlier ones
    const bool y0_ok = p.Yout != nullptr && o0 < p.w, y1_ok = p.Yout != nullptr && o0 + 1 < p.w;
    double* const yo0 = p.Yout + (int64_t)o0 * p.ldy + row_begin + g;
    double* const yo1 = yo0 + p.ldy;
    auto yrun = [&](auto nj_t) {
      constexpr int NJ = decltype(nj_t)::value;
      int pi = 0;
      unsigned ph = 0;
      for (int64_t s = 0; s < nstage; ++s, (++pi == NS ? (pi = 0, ph ^= 1u) : 0u)) {
        mbar_wait(&fullA[pi], ph);
        const double* P = ring + (size_t)pi * (szA + szB);
        const double* pq[4] = {P + aoff[0], P + aoff[1], P + aoff[2], P + aoff[3]};
        double acc[4][2];
#pragma unroll
        for (int q = 0; q < 4; ++q) acc[q][0] = acc[q][1] = 0.0;
#pragma unroll
        for (int j = 0; j < NJ; ++j) {
          double a[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) a[q] = pq[q][128 * j];
#pragma unroll
          for (int q = 0; q < 4; ++q) dmma884(acc[q][0], acc[q][1], a[q], wr[j]);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&emptyA[pi]);
        const int yb = (int)(s % FS_YB);
        const unsigned yph = (unsigned)((s / FS_YB) & 1);
        double* Ys = sY + (size_t)yb * YC * SR;
        if (kp == 0) {
          if (s >= FS_YB && fs.npy > 0) mbar_wait(&yfree[yb], yph ^ 1u);  // the tile warps are done with Y of stage s - FS_YB
        } else {
          mbar_wait(&chain[(yb * NCB + cb) * 3 + kp - 1], yph);  // the partial sum of parts 0 .. kp - 1
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            acc[q][0] = Ys[yoff[q][0]] + acc[q][0];
            acc[q][1] = Ys[yoff[q][1]] + acc[q][1];
          }
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          Ys[yoff[q][0]] = acc[q][0];
          Ys[yoff[q][1]] = acc[q][1];
        }
        if (!last) {
          mbar_arrive(&chain[(yb * NCB + cb) * 3 + kp]);
          continue;
        }
        mbar_arrive(&ydone[yb]);
        const int64_t r0 = s * SR;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          if (row_begin + r0 + 8 * q + g >= row_end) continue;
          if (y0_ok) yo0[r0 + 8 * q] = acc[q][0];
          if (y1_ok) yo1[r0 + 8 * q] = acc[q][1];
        }
      }
    };
    switch (nj) {
#define PSVD_FS_NJ(N) case N: yrun(std::integral_constant<int, N>{}); break;
      PSVD_FS_NJ(1) PSVD_FS_NJ(2) PSVD_FS_NJ(3) PSVD_FS_NJ(4) PSVD_FS_NJ(5) PSVD_FS_NJ(6) PSVD_FS_NJ(7)
      PSVD_FS_NJ(8) PSVD_FS_NJ(9) PSVD_FS_NJ(10) PSVD_FS_NJ(11) PSVD_FS_NJ(12) PSVD_FS_NJ(13) PSVD_FS_NJ(14)
      PSVD_FS_NJ(15) PSVD_FS_NJ(16) PSVD_FS_NJ(17) PSVD_FS_NJ(18) PSVD_FS_NJ(19)
#undef PSVD_FS_NJ
      default: yrun(std::integral_constant<int, FS_WR>{}); break;
    }
    return;
  }

  if (role == FS_PY) {
    const int sb0 = fs.py_sb0[warp];
    // the group whose slots this warp's sub-blocks live in (A: e.g. Q^T Y of a projection pass)
    const bool onA = fs.py_onA[warp] != 0;
    uint64_t* const fullX = onA ? fullA : fullB;
    uint64_t* const emptyX = onA ? emptyA : emptyB;
    const size_t xoff = (onA ? 0 : szA) + 256 * (size_t)sb0;
    auto run = [&](auto na_t, auto yy_t) {
      constexpr int NA = decltype(na_t)::value;
      constexpr bool YY = decltype(yy_t)::value;
      constexpr int NAX = NA > 0 ? NA : 1;
      double acc[NAX][NCB][2], accy[NCB][NCB][2];
#pragma unroll
      for (int a = 0; a < NAX; ++a)
#pragma unroll
        for (int c = 0; c < NCB; ++c) acc[a][c][0] = acc[a][c][1] = 0.0;
#pragma unroll
      for (int a = 0; a < NCB; ++a)
#pragma unroll
        for (int c = 0; c < NCB; ++c) accy[a][c][0] = accy[a][c][1] = 0.0;
      int pi = 0;
      unsigned ph = 0;
      for (int64_t s = 0; s < nstage; ++s, (++pi == NS ? (pi = 0, ph ^= 1u) : 0u)) {
        const int yb = (int)(s % FS_YB);
        if (NA > 0) mbar_wait(&fullX[pi], ph);
        mbar_wait(&ydone[yb], (unsigned)((s / FS_YB) & 1));
        const double* Bp = ring + (size_t)pi * (szA + szB) + xoff;
        const double* Ys = sY + (size_t)yb * YC * SR;
#pragma unroll
        for (int kk = 0; kk < SR / 4; ++kk) {
          double fa[NAX], fb[NCB];
#pragma unroll
          for (int c = 0; c < NCB; ++c) fb[c] = Ys[eoff[kk] + 256 * c];
          if (NA > 0) {
#pragma unroll
            for (int a = 0; a < NAX; ++a) fa[a] = Bp[eoff[kk] + 256 * a];
#pragma unroll
            for (int a = 0; a < NAX; ++a)
#pragma unroll
              for (int c = 0; c < NCB; ++c) dmma884(acc[a][c][0], acc[a][c][1], fa[a], fb[c]);
          }
          if (YY) {
#pragma unroll
            for (int a = 0; a < NCB; ++a)
#pragma unroll
              for (int c = 0; c < NCB; ++c) dmma884(accy[a][c][0], accy[a][c][1], fb[a], fb[c]);
          }
        }
        mbar_arrive(&yfree[yb]);
        __syncwarp();
        if (NA > 0 && lane == 0) mbar_arrive(&emptyX[pi]);
      }
      // full 32 x 32 slots (the fixed-order reduce sums every element): sub-block a lands in row block
      // (rb0 + a) & 3 of the warp's tile (rb0 + a) >> 2, zeros everywhere else
      const int rb0 = fs.py_rb0[warp], nt = fs.py_nt[warp];
      for (int t = 0; t < nt; ++t) {
        double* dst = p.partial + ((size_t)blockIdx.x * SLOTS + fs.py_slot[warp][t]) * 1024;
        for (int rb = 0; rb < 4; ++rb) {
          const int a = 4 * t + rb - rb0;
          if (a >= 0 && a < NA) continue;  // written below
#pragma unroll
          for (int c = 0; c < 4; ++c)
            *reinterpret_cast<double2*>(dst + (rb * 8 + g) * 32 + c * 8 + 2 * tq) = make_double2(0.0, 0.0);
        }
      }
#pragma unroll
      for (int a = 0; a < NA; ++a) {
        double* dst = p.partial + ((size_t)blockIdx.x * SLOTS + fs.py_slot[warp][(rb0 + a) >> 2]) * 1024;
        const int rb = (rb0 + a) & 3;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          double v0 = 0.0, v1 = 0.0;
          if (c < NCB) v0 = acc[a % NAX][c % NCB][0], v1 = acc[a % NAX][c % NCB][1];
          *reinterpret_cast<double2*>(dst + (rb * 8 + g) * 32 + c * 8 + 2 * tq) = make_double2(v0, v1);
        }
      }
      if (YY) {
        double* dst = p.partial + ((size_t)blockIdx.x * SLOTS + fs.yy_slot) * 1024;
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            double v0 = 0.0, v1 = 0.0;
            if (a < NCB && c < NCB) v0 = accy[a % NCB][c % NCB][0], v1 = accy[a % NCB][c % NCB][1];
            *reinterpret_cast<double2*>(dst + (a * 8 + g) * 32 + c * 8 + 2 * tq) = make_double2(v0, v1);
          }
      }
    };
    using F = std::false_type;
    using T = std::true_type;
    const int na = fs.py_na[warp];
    if (fs.py_yy[warp]) {
      switch (na) {
        case 0: run(std::integral_constant<int, 0>{}, T{}); break;
        case 1: run(std::integral_constant<int, 1>{}, T{}); break;
        case 2: run(std::integral_constant<int, 2>{}, T{}); break;
        case 3: run(std::integral_constant<int, 3>{}, T{}); break;
        default: run(std::integral_constant<int, 4>{}, T{}); break;
      }
    } else {
      switch (na) {
        case 1: run(std::integral_constant<int, 1>{}, F{}); break;
        case 2: run(std::integral_constant<int, 2>{}, F{}); break;
        case 3: run(std::integral_constant<int, 3>{}, F{}); break;
        case 4: run(std::integral_constant<int, 4>{}, F{}); break;
        case 5: run(std::integral_constant<int, 5>{}, F{}); break;
        default:  // 6 .. 8 sub-blocks: one or two Y column blocks only (the accumulators of three would not fit)
          if constexpr (NCB <= 2) {
            if (na == 6) run(std::integral_constant<int, 6>{}, F{});
            else if (na == 7) run(std::integral_constant<int, 7>{}, F{});
            else run(std::integral_constant<int, 8>{}, F{});
          }
          break;
      }
    }
    return;
  }

  if (role == FS_OFF) {
    const int I = fs.off_i[warp], J = fs.off_j[warp];
    double acc[4][4][2];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int c = 0; c < 4; ++c) acc[a][c][0] = acc[a][c][1] = 0.0;
    auto run = [&](auto diag_t) {
      constexpr bool DIAG = decltype(diag_t)::value;
      int pi = 0;
      unsigned ph = 0;
      for (int64_t s = 0; s < nstage; ++s, (++pi == NS ? (pi = 0, ph ^= 1u) : 0u)) {
        mbar_wait(&fullB[pi], ph);
        const double* Bp = ring + (size_t)pi * (szA + szB) + szA;
        const double* bI = Bp + 1024 * I;
        const double* bJ = Bp + 1024 * J;
#pragma unroll
        for (int kk = 0; kk < SR / 4; ++kk) {
          double fa[4], fb[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) fa[q] = bI[eoff[kk] + 256 * q];
#pragma unroll
          for (int q = 0; q < 4; ++q) fb[q] = DIAG ? fa[q] : bJ[eoff[kk] + 256 * q];
#pragma unroll
          for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int c = 0; c < 4; ++c)
              if (!DIAG || c >= a) dmma884(acc[a][c][0], acc[a][c][1], fa[a], fb[c]);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&emptyB[pi]);
      }
    };
    if (I == J) run(std::true_type{});
    else run(std::false_type{});
    double* dst = p.partial + ((size_t)blockIdx.x * SLOTS + fs.off_slot[warp]) * 1024;
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int c = 0; c < 4; ++c)
        *reinterpret_cast<double2*>(dst + (a * 8 + g) * 32 + c * 8 + 2 * tq) = make_double2(acc[a][c][0], acc[a][c][1]);
  }
}

void launch_fused_split(const TallParams& p, const TmaMaps& maps3, const TmaExtra& x, const FusedSplit& fs, int grid,
                        cudaStream_t st) {
  const size_t smem = fused_split_smem_bytes(fs);
  if (fs.ncb == 3) {
    cudaFuncSetAttribute(fused_split_kernel<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    fused_split_kernel<3><<<grid, NTHR, smem, st>>>(p, maps3, x, fs);
  } else if (fs.ncb == 2) {
    cudaFuncSetAttribute(fused_split_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    fused_split_kernel<2><<<grid, NTHR, smem, st>>>(p, maps3, x, fs);
  } else {
    cudaFuncSetAttribute(fused_split_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    fused_split_kernel<1><<<grid, NTHR, smem, st>>>(p, maps3, x, fs);
  }
}

// ---------------------------------------------------------------- host side

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(f);
    cudaGetLastError();
  }
  return fn;
}

bool tma_available() { return encode_fn() != nullptr; }

int tma_pass_prepare(TallParams& p, TmaMaps& maps, TmaExtra& x, int pshift, bool narrow) {
  EncodeTiledFn enc = encode_fn();
  if (!enc) return -1;
  memset(&x, 0, sizeof(x));
  x.pshift = pshift;
  int nops = 0;
  uint32_t bytes = 0;
  int logical = 0;
  int kp_lo = 1 << 30, kp_hi = 0, pend = 0;
  for (int s = 0; s < p.nseg; ++s) {
    const Seg& sg = p.seg[s];
    const int P = sg.col0 + pshift;         // physical first column
    const int lead = P & 7;                 // only the first segment may start off an 8-column boundary
    if ((lead != 0 && (s != 0 || P != pshift)) || (reinterpret_cast<uintptr_t>(sg.ptr) & 15) != 0 ||
        (sg.ld & 1) != 0)
      return -1;
    // boxes of 256 columns, then one tail box of the remaining columns rounded up to 8 (its own
    // tensor map): a box may overhang the segment by < 8 columns only, so it never lands on the
    // next segment's columns (which start on the next 8-column boundary)
    const int span = sg.ncols + lead;
    const int nfull = span > 256 ? span / 256 : 0;
    const int tail = span - 256 * nfull;
    cuuint64_t dims[2] = {(cuuint64_t)p.M, (cuuint64_t)sg.ncols};
    cuuint64_t strides[1] = {(cuuint64_t)sg.ld * sizeof(double)};
    cuuint32_t es[2] = {1, 1};
    auto encode = [&](int map, int bw) {
      cuuint32_t box[2] = {(cuuint32_t)TKS, (cuuint32_t)bw};
      return enc(&maps.m[map], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(sg.ptr), dims, strides, box, es,
                 CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                 CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
    };
    if (nfull > 0 && !encode(s, 256)) return -1;
    const int tw = (tail + 7) / 8 * 8;
    if (tail > 0 && !encode(nfull > 0 ? MAX_SEG + s : s, tw)) return -1;
    // boxes start at tensor column -lead (out of bounds -> zero filled) so they land 1024-byte aligned
    for (int k = 0; k < nfull + (tail > 0); ++k) {
      if (nops >= TMA_MAX_OPS) return -1;
      const int c = -lead + 256 * k;
      const int bw = k < nfull ? 256 : tw;
      const int dst = P + c;
      x.op_seg[nops] = (short)(k < nfull ? s : (nfull > 0 ? MAX_SEG + s : s));
      x.op_col[nops] = (short)c;
      x.op_pcol[nops] = (short)dst;
      x.op_bw[nops] = (short)bw;
      for (int q = dst >> 3; q < (dst + bw) >> 3 && q < TMA_MAX_BLK; ++q) x.written[q] = 1;
      bytes += (uint32_t)(TKS * bw * sizeof(double));
      pend = std::max(pend, dst + bw);
      ++nops;
    }
    x.wrow0[s] = TMA_NOT_IN_W;
    const int lo = std::max(logical, p.wlo), hi = std::min(logical + sg.ncols, p.wlo + p.wk);
    if (p.w > 0 && lo < hi) {
      x.wrow0[s] = logical - p.wlo;
      kp_lo = std::min(kp_lo, P + (lo - logical));
      kp_hi = std::max(kp_hi, P + (hi - logical));
    }
    logical += sg.ncols;
  }
  if (p.w > 0) {
    x.kp_lo = kp_lo / 8 * 8;
    x.kp_hi = (kp_hi + 3) / 4 * 4;
  }
  x.nops = nops;
  x.stage_bytes = bytes;
  x.pwidth = std::max((p.np_pad + pshift + 7) / 8 * 8, (pend + 7) / 8 * 8);
  // 32-row stages (narrow passes, M a multiple of 16, a 2-deep ring fits): one 3-D box per
  // column block brings 256 contiguous bytes of every column per request -- 16-row boxes (128
  // bytes per column) cap TMA streaming at ~4.6 TB/s, 32-row ones reach ~6.9
  // (tools/tma_stream_bw.cu)
  static const bool no_rb2 = getenv("PSVD_TMA_RB1") != nullptr;
  x.rb = 1;
  if (narrow && !no_rb2 && p.M % TKS == 0 &&
      tma_pass_smem_bytes(x.pwidth, x.kp_hi - x.kp_lo, p.w_pad, 2, 2) <= (size_t)(227 * 1024)) {
    x.rb = 2;
    for (int o = 0; o < nops; ++o) {
      const int m = x.op_seg[o], sidx = m % MAX_SEG;
      const Seg& sg = p.seg[sidx];
      cuuint64_t dims[3] = {(cuuint64_t)TKS, (cuuint64_t)(p.M / TKS), (cuuint64_t)sg.ncols};
      cuuint64_t strides[2] = {(cuuint64_t)TKS * sizeof(double), (cuuint64_t)sg.ld * sizeof(double)};
      cuuint32_t box[3] = {(cuuint32_t)TKS, 2, (cuuint32_t)x.op_bw[o]};
      cuuint32_t es[3] = {1, 1, 1};
      if (enc(&maps.m[m], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(sg.ptr), dims, strides, box, es,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return -1;
    }
    x.stage_bytes = 2 * bytes;
  }
  if (x.rb != 2) p.yh = 1;  // 16-row stages: the second half-warps of the plan stay idle
  if (p.ykp > 1 && (x.rb != 2 || ((x.kp_hi - x.kp_lo) / 4 + p.ykp - 1) / p.ykp > YKP_WR)) {
    p.ykp = 1;  // the plan's Y warps 0 .. 2 ncb - 1 then run the fragment-reloading path
    p.yh = 1;
  }
  if (p.ykp > 1) {
    // split each column block's k steps over its ykp parts in proportion to what the parts'
    // SMSPs (warp w issues on SMSP w % 4) have left after their Gram tiles: a Y step is 4
    // DMMAs per stage (4 row blocks), a Gram tile na x nb DMMAs per 4 rows
    const int n4 = (x.kp_hi - x.kp_lo) / 4, ncb = p.w_pad / 8, ny = ncb * p.ykp;
    double gload[4] = {0.0, 0.0, 0.0, 0.0};  // Gram DMMAs per 32-row stage per SMSP (slice 0 stands for all)
    for (int w = ny; w < NWARP - 1; ++w) {
      const WarpPlan& wp = p.plan[0][w];
      if (wp.ntile == 0) continue;
      const int I = wp.ti[0];
      const int na = I * 32 >= p.np_pad ? ncb : wp.sub != 0 ? (wp.sub >> 4) : std::min(4, (p.np - I * 32 + 7) / 8);
      gload[w % 4] += (double)na * ncb * (2 * TKS / 4);
    }
    int ywarps[4] = {0, 0, 0, 0};
    for (int v = 0; v < ny; ++v) ywarps[v % 4]++;
    const double share = (gload[0] + gload[1] + gload[2] + gload[3] + 4.0 * n4 * ncb) / 4.0;
    for (int cb = 0; cb < ncb; ++cb) {
      // part kp's weight: what its SMSP has left of the even share after the Gram tiles, split
      // over the Y warps issuing there (a Y step is 4 DMMAs per stage)
      double wgt[4], sum = 0.0;
      for (int kp = 0; kp < p.ykp; ++kp) {
        const int q = (cb + ncb * kp) % 4;
        wgt[kp] = std::max(1.0, (share - gload[q]) / std::max(1, ywarps[q]));
        sum += wgt[kp];
      }
      int j = 0;
      for (int kp = 0; kp < p.ykp; ++kp) {
        const int w = cb + ncb * kp;
        int nj = kp == p.ykp - 1 ? n4 - j : (int)(n4 * wgt[kp] / sum + 0.5);
        nj = std::max(0, std::min(nj, std::min(YKP_WR, n4 - j)));
        p.ykj0[w] = (unsigned char)j;
        p.yknj[w] = (unsigned char)nj;
        j += nj;
      }
      if (j != n4 || p.yknj[cb + ncb * (p.ykp - 1)] > YKP_WR) {  // fall back to the even split
        for (int kp = 0; kp < p.ykp; ++kp) {
          const int w = cb + ncb * kp;
          p.ykj0[w] = (unsigned char)(n4 * kp / p.ykp);
          p.yknj[w] = (unsigned char)(n4 * (kp + 1) / p.ykp - n4 * kp / p.ykp);
        }
      }
    }
  }
  // ring depth: as many stages as shared memory holds (3 .. TNS_MAX; 2 .. for 32-row stages)
  x.ns = x.rb == 2 ? 2 : 3;
  while (x.ns < TNS_MAX &&
         tma_pass_smem_bytes(x.pwidth, x.kp_hi - x.kp_lo, p.w_pad, x.ns + 1, x.rb) <= (size_t)(227 * 1024))
    ++x.ns;
  if (const char* e = getenv("PSVD_TMA_NS")) x.ns = std::max(2, std::min(x.ns, atoi(e)));
  // issue groups: half the ring (two groups in flight), at most 4 stages = 64 rows
  x.grp = 1;  // grouped issue (consecutive stages box by box) measured no faster: off by default
  if (const char* e = getenv("PSVD_TMA_GROUP")) x.grp = std::max(1, std::min(x.ns, atoi(e)));
  return 0;
}

// Split-ring pass: qualifies a planned narrow TMA pass (p, x: tma_pass_prepare's box list; map: its reduce
// map with NB tile columns, replaced by the split kernel's own on success) and builds the warp roles, the k
// split and the 3-D tensor maps.  Group A = the segments W covers (contiguous), group B = the others (all
// before or all after group A; none for a recompose).  The wanted tiles come from the plan: (I, Y) for the
// 8-column sub-blocks the plan kept, (Y, Y).  off[i] = {I, J}: 32-column block pairs of group B's (single)
// segment whose Gram tile is computed here (full blocks only, I <= J), reduced by offmap into a tile array
// with off_nb tile columns.  Returns 0 when the pass runs on fused_split_kernel, -1 when it stays on
// pass_tma_kernel.
int fused_split_prepare(const TallParams& p, const TmaExtra& x, ReduceMap& map, int NB, const int (*off)[2],
                        int noff, FusedSplit& fs, TmaMaps& maps3, ReduceMap& offmap, int off_nb) {
  EncodeTiledFn enc = encode_fn();
  memset(&fs, 0, sizeof(fs));
  memset(&offmap, 0, sizeof(offmap));
  if (!enc || p.nseg < 1 || p.nslices != 1 || x.pshift != 0 || p.w < 1 || p.M % TKS != 0 ||
      (p.w_pad != 8 && p.w_pad != 16 && p.w_pad != 24) || p.colmax != nullptr || p.gate != nullptr ||
      (p.dbg != 0 && p.dbg != 2))
    return -1;
  // groups
  int a0s = -1, a1s = -1, b0s = -1, b1s = -1;
  for (int s = 0; s < p.nseg; ++s) {
    if ((p.seg[s].col0 & 7) != 0) return -1;
    if (x.wrow0[s] != TMA_NOT_IN_W) {
      if (a0s < 0) a0s = s;
      else if (a1s != s - 1) return -1;  // W's segments are contiguous
      a1s = s;
    } else {
      if (b0s < 0) b0s = s;
      else if (b1s != s - 1) return -1;  // and so are the others: all before or all after group A
      b1s = s;
    }
  }
  if (a0s < 0) return -1;
  const bool hasB = b0s >= 0;
  const int colA0 = p.seg[a0s].col0, endA = p.seg[a1s].col0 + p.seg[a1s].ncols;
  const int colB0 = hasB ? p.seg[b0s].col0 : 0, endB = hasB ? p.seg[b1s].col0 + p.seg[b1s].ncols : 0;
  fs.colA0 = colA0;
  fs.pwA = (endA - colA0 + 7) / 8 * 8;
  fs.pwB = hasB ? (endB - colB0 + 7) / 8 * 8 : 0;
  fs.ncb = p.w_pad / 8;
  if (hasB && !(colB0 >= colA0 + fs.pwA || colA0 >= colB0 + fs.pwB)) return -1;
  if (x.kp_lo != colA0 || x.kp_hi > colA0 + fs.pwA || fs.pwA > 256 + 8 || fs.pwB > 256 + 8) return -1;
  fs.n4 = (x.kp_hi - x.kp_lo) / 4;
  fs.nkp = fs.n4 > 24 ? 4 : fs.n4 > 12 ? 2 : 1;
  if (fs.n4 < 1 || fs.n4 > fs.nkp * FS_WR) return -1;
  fs.ns = 2;
  if (fused_split_smem_bytes(fs) > (size_t)(227 * 1024)) return -1;
  static const int ns_cap = getenv("PSVD_FS_NS") ? std::max(2, std::min(FS_NS_MAX, atoi(getenv("PSVD_FS_NS")))) : FS_NS_MAX;
  while (fs.ns < ns_cap) {  // as many slots per ring as shared memory holds
    fs.ns++;
    if (fused_split_smem_bytes(fs) > (size_t)(227 * 1024)) {
      fs.ns--;
      break;
    }
  }
  if ((size_t)fs.n4 * 4 * w_stride(p.w_pad) > (size_t)fs.pwA * 32) return -1;  // W is staged through slot A0
  // boxes: group A first, then group B; every 8-column block of both slots must be covered
  std::vector<char> covA(fs.pwA / 8, 0), covB(fs.pwB / 8, 0);
  int n = 0;
  for (int pass = 0; pass < 2; ++pass)
    for (int o = 0; o < x.nops; ++o) {
      const int m = x.op_seg[o], sidx = m % MAX_SEG;
      const bool inB = x.wrow0[sidx] == TMA_NOT_IN_W;
      if (inB != (pass == 1)) continue;
      const int dst = x.op_pcol[o] - (inB ? colB0 : colA0), bw = x.op_bw[o];
      if (dst < 0 || (dst & 7) != 0 || x.op_col[o] < 0 || dst + bw > (inB ? fs.pwB : fs.pwA)) return -1;
      fs.opm[n] = (short)m;
      fs.opc[n] = x.op_col[o];
      fs.opd[n] = (short)dst;
      for (int q = dst / 8; q < (dst + bw) / 8; ++q) (inB ? covB : covA)[q] = 1;
      (inB ? fs.bytesB : fs.bytesA) += (unsigned)(2 * TKS * bw * sizeof(double));
      (inB ? fs.nopsB : fs.nopsA)++;
      const Seg& sg = p.seg[sidx];
      cuuint64_t dims[3] = {(cuuint64_t)TKS, (cuuint64_t)(p.M / TKS), (cuuint64_t)sg.ncols};
      cuuint64_t strides[2] = {(cuuint64_t)TKS * sizeof(double), (cuuint64_t)sg.ld * sizeof(double)};
      cuuint32_t box[3] = {(cuuint32_t)TKS, 2, (cuuint32_t)bw};
      cuuint32_t es[3] = {1, 1, 1};
      if (enc(&maps3.m[m], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(sg.ptr), dims, strides, box, es,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return -1;
      ++n;
    }
  for (char c : covA) if (!c) return -1;
  for (char c : covB) if (!c) return -1;
  // the planned tiles: (I, Y block) with the plan's wanted 8-column sub-blocks, and (Y block, Y block)
  const int yblk = p.np_pad / 32;
  if (NB != yblk + 1) return -1;
  std::vector<int> wantA, wantB;  // slot-relative sub-blocks
  bool has_yy = false;
  for (int w = 0; w < NWARP; ++w) {
    const WarpPlan& wp = p.plan[0][w];
    if (wp.ntile == 0) continue;
    const int I = wp.ti[0], J = wp.tj[0];
    if (wp.ntile != 1 || J != yblk) return -1;
    if (I == yblk) { has_yy = true; continue; }
    if (I > yblk) return -1;
    const int s0 = wp.sub != 0 ? (wp.sub & 15) : 0;
    const int na = wp.sub != 0 ? (wp.sub >> 4) : std::min(4, (p.np - I * 32 + 7) / 8);
    for (int a = 0; a < na; ++a) {
      const int col = (4 * I + s0 + a) * 8;
      if (col >= colA0 && col < colA0 + fs.pwA) wantA.push_back((col - colA0) / 8);
      else if (hasB && col >= colB0 && col < colB0 + fs.pwB) wantB.push_back((col - colB0) / 8);
      else return -1;
    }
  }
  if (!has_yy) return -1;
  std::sort(wantA.begin(), wantA.end());
  std::sort(wantB.begin(), wantB.end());
  // Roles are built for every chunk size of the tile warps (namax sub-blocks per warp, up to what the
  // accumulators allow) and the one with the lightest busiest SMSP is kept
  const FusedSplit fs0 = fs;
  ReduceMap nm;
  auto build = [&](int namax, bool yy_own, FusedSplit& fs, ReduceMap& nm, ReduceMap& offmap) -> double {
    memset(&nm, 0, sizeof(nm));
    memset(&offmap, 0, sizeof(offmap));
    // fixed items: tile warps over runs of wanted sub-blocks, Y^T Y on the lightest of them when its
    // accumulators fit (else a warp of its own), offloaded tiles, the producer
    struct Item { int kind, cost, sb0, na, onA, I, J; };
    std::vector<Item> items;
    auto add_runs = [&](const std::vector<int>& want, int onA) {
      size_t i = 0;
      while (i < want.size()) {
        size_t j = i + 1;
        while (j < want.size() && want[j] == want[j - 1] + 1) ++j;
        // a run of wanted sub-blocks, cut into chunks of namax (the remainder last: it can carry Y^T Y)
        const int len = (int)(j - i);
        for (int lo = 0; lo < len; lo += namax) {
          const int hi = std::min(len, lo + namax);
          items.push_back({FS_PY, (hi - lo) * fs.ncb * 8, want[i] + lo, hi - lo, onA, 0, 0});
        }
        i = j;
      }
    };
    add_runs(wantB, 0);
    add_runs(wantA, 1);
    int yy_item = -1;
    for (size_t i = 0; i < items.size() && !yy_own; ++i)
      if (items[i].na <= 4 && items[i].na * fs.ncb + fs.ncb * fs.ncb <= 18 &&
          (yy_item < 0 || items[i].na < items[yy_item].na))
        yy_item = (int)i;
    if (yy_item < 0) {
      items.push_back({FS_PY, 0, 0, 0, 1, 0, 0});
      yy_item = (int)items.size() - 1;
    }
    items[yy_item].cost += fs.ncb * fs.ncb * 8;
    const int nfullB = (hasB && b0s == b1s) ? p.seg[b0s].ncols / 32 : 0;
    for (int i = 0; i < noff && fs.noff < FS_MAX_OFF; ++i) {
      const int I = off[i][0], J = off[i][1];
      if (I < 0 || I > J || J >= nfullB) continue;
      items.push_back({FS_OFF, (I == J ? 10 : 16) * 8, 0, 0, 0, I, J});
      fs.noff++;
    }
    items.push_back({FS_PROD, 0, 0, 0, 0, 0, 0});
    const int nyw = fs.ncb * fs.nkp;
    if ((int)items.size() + nyw > NWARP) return -1.0;
    // longest first onto the least-loaded SMSP (warp w issues on SMSP w % 4) with a free slot
    std::vector<int> order(items.size());
    for (size_t i = 0; i < order.size(); ++i) order[i] = (int)i;
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return items[a].cost > items[b].cost; });
    int load[4] = {0, 0, 0, 0}, cnt[4] = {0, 0, 0, 0};
    int next_slot = 0;
    auto add_src = [&](int out_id, int slot) {
      int o = 0;
      while (o < nm.nout && nm.out_id[o] != out_id) ++o;
      if (o == nm.nout) {
        if (nm.nout >= MAX_OUT_TILES) return false;
        nm.out_id[nm.nout++] = (short)out_id;
      }
      if (nm.nsrc[o] >= NWARP) return false;
      nm.src[o][nm.nsrc[o]++] = (unsigned char)slot;
      return true;
    };
    for (int it : order) {
      int q = -1;
      for (int c = 0; c < 4; ++c)
        if (cnt[c] < 4 && (q < 0 || load[c] < load[q] || (load[c] == load[q] && cnt[c] < cnt[q]))) q = c;
      if (q < 0) return -1.0;
      const int w = q + 4 * cnt[q];
      cnt[q]++;
      load[q] += items[it].cost;
      const Item& im = items[it];
      fs.role[w] = (unsigned char)im.kind;
      if (im.kind == FS_PY) {
        const int g0 = ((im.onA ? colA0 : colB0) / 8) + im.sb0;  // global sub-block of the first one
        fs.py_sb0[w] = (unsigned char)im.sb0;
        fs.py_na[w] = (unsigned char)im.na;
        fs.py_onA[w] = (unsigned char)im.onA;
        fs.py_rb0[w] = (unsigned char)(g0 & 3);
        fs.py_yy[w] = (unsigned char)(it == yy_item);
        const int nt = im.na > 0 ? (g0 + im.na - 1) / 4 - g0 / 4 + 1 : 0;
        if (nt > 3) return -1.0;
        fs.py_nt[w] = (unsigned char)nt;
        for (int t = 0; t < nt; ++t) {
          if (next_slot >= SLOTS || !add_src((g0 / 4 + t) * NB + yblk, next_slot)) return -1.0;
          fs.py_slot[w][t] = (unsigned char)next_slot++;
        }
        if (it == yy_item) {
          if (next_slot >= SLOTS || !add_src(yblk * NB + yblk, next_slot)) return -1.0;
          fs.yy_slot = (unsigned char)next_slot++;
        }
        fs.npy++;
        if (im.na > 0) (im.onA ? fs.nA : fs.nB)++;
      } else if (im.kind == FS_OFF) {
        if (next_slot >= SLOTS) return -1.0;
        fs.off_i[w] = (unsigned char)im.I;
        fs.off_j[w] = (unsigned char)im.J;
        fs.off_slot[w] = (unsigned char)next_slot;
        const int o = offmap.nout++;
        offmap.out_id[o] = (short)(im.I * off_nb + im.J);
        offmap.nsrc[o] = 1;
        offmap.src[o][0] = (unsigned char)next_slot++;
        fs.nB++;
      }
    }
    fs.nA += nyw;
    // Y warps take the remaining slots; column blocks alternate so that each gets nkp parts
    std::vector<int> yw;
    for (int i = 0; i < 4; ++i)
      for (int q = 0; q < 4; ++q)
        if (i >= cnt[q] && (int)yw.size() < nyw) yw.push_back(q + 4 * i);
    if ((int)yw.size() != nyw) return -1.0;
    std::sort(yw.begin(), yw.end(), [](int a, int b) { return a % 4 != b % 4 ? a % 4 < b % 4 : a < b; });
    int ywarps[4] = {0, 0, 0, 0};
    for (int w : yw) ywarps[w % 4]++;
    const double target = (load[0] + load[1] + load[2] + load[3] + 4.0 * fs.n4 * fs.ncb) / 4.0;
    std::vector<std::vector<int>> wcb(fs.ncb);
    for (size_t i = 0; i < yw.size(); ++i) wcb[i % fs.ncb].push_back(yw[i]);
    for (int cb = 0; cb < fs.ncb; ++cb) {
      // a part's weight: what its SMSP has left of the even share, split over the Y warps issuing there
      std::vector<double> wgt(fs.nkp);
      double sum = 0.0;
      for (int kp = 0; kp < fs.nkp; ++kp) {
        const int q = wcb[cb][kp] % 4;
        wgt[kp] = std::max(4.0, (target - load[q]) / std::max(1, ywarps[q]));
        sum += wgt[kp];
      }
      std::vector<int> nj(fs.nkp);
      int tot = 0;
      for (int kp = 0; kp < fs.nkp; ++kp) {
        nj[kp] = std::max(1, std::min(FS_WR, (int)(fs.n4 * wgt[kp] / sum + 0.5)));
        tot += nj[kp];
      }
      for (int guard = 0; tot != fs.n4 && guard < 1000; ++guard) {  // fix the rounding, heaviest weights first
        int best = -1;
        for (int kp = 0; kp < fs.nkp; ++kp) {
          if (tot < fs.n4 && nj[kp] >= FS_WR) continue;
          if (tot > fs.n4 && nj[kp] <= 1) continue;
          if (best < 0 || (tot < fs.n4 ? wgt[kp] / nj[kp] > wgt[best] / nj[best] : wgt[kp] / nj[kp] < wgt[best] / nj[best]))
            best = kp;
        }
        if (best < 0) return -1.0;
        nj[best] += tot < fs.n4 ? 1 : -1;
        tot += tot < fs.n4 ? 1 : -1;
      }
      if (tot != fs.n4) return -1.0;
      int j = 0;
      for (int kp = 0; kp < fs.nkp; ++kp) {
        const int w = wcb[cb][kp];
        fs.role[w] = FS_Y;
        fs.ycb[w] = (unsigned char)cb;
        fs.ykp[w] = (unsigned char)kp;
        fs.yj0[w] = (unsigned char)j;
        fs.ynj[w] = (unsigned char)nj[kp];
        j += nj[kp];
      }
    }

    // DMMAs per stage of the busiest SMSP; a single warp is a serial chain, so the heaviest tile warp
    // counts half as much again
    double mx = 0.0;
    int yl[4] = {0, 0, 0, 0};
    for (int w = 0; w < NWARP; ++w)
      if (fs.role[w] == FS_Y) yl[w % 4] += 4 * fs.ynj[w];
    for (int q = 0; q < 4; ++q) mx = std::max(mx, (double)load[q] + yl[q]);
    for (const Item& im : items) mx = std::max(mx, 1.5 * im.cost);
    return mx;
  };
  int best_na = -1;
  bool best_own = false;
  double best_load = 0.0;
  for (int own = 0; own < 2; ++own)
    for (int namax = fs0.ncb <= 2 ? 8 : 5; namax >= 2; --namax) {
      FusedSplit t = fs0;
      ReduceMap m1, m2;
      const double ld = build(namax, own != 0, t, m1, m2);
      if (ld >= 0.0 && (best_na < 0 || ld < best_load - 0.5)) best_na = namax, best_own = own != 0, best_load = ld;
    }
  if (best_na < 0) return -1;
  fs = fs0;
  if (build(best_na, best_own, fs, nm, offmap) < 0.0) return -1;
  nm.nchunks = map.nchunks;
  nm.nslices = 1;
  map = nm;
  offmap.nchunks = map.nchunks;
  offmap.nslices = 1;
  static const bool verbose = getenv("PSVD_PASS_VERBOSE") != nullptr;
  if (verbose) {
    fprintf(stderr, "fused_split: ns=%d colA0=%d pwA=%d pwB=%d n4=%d ncb=%d nkp=%d npy=%d noff=%d nA=%d nB=%d smem=%zu roles:",
            fs.ns, fs.colA0, fs.pwA, fs.pwB, fs.n4, fs.ncb, fs.nkp, fs.npy, fs.noff, fs.nA, fs.nB, fused_split_smem_bytes(fs));
    for (int w = 0; w < NWARP; ++w) {
      if (fs.role[w] == FS_Y) fprintf(stderr, " w%d:Y(cb%d,kp%d,%d+%d)", w, fs.ycb[w], fs.ykp[w], fs.yj0[w], fs.ynj[w]);
      else if (fs.role[w] == FS_PY)
        fprintf(stderr, " w%d:PY%s(sb%d+%d%s)", w, fs.py_onA[w] ? "a" : "", fs.py_sb0[w], fs.py_na[w], fs.py_yy[w] ? ",yy" : "");
      else if (fs.role[w] == FS_OFF) fprintf(stderr, " w%d:OFF(%d,%d)", w, fs.off_i[w], fs.off_j[w]);
      else if (fs.role[w] == FS_PROD) fprintf(stderr, " w%d:PROD", w);
    }
    fprintf(stderr, "\n");
  }
  return 0;
}

void launch_pass_tma(const TallParams& p, const TmaMaps& maps, const TmaExtra& x, int grid, cudaStream_t st) {
  const size_t smem = tma_pass_smem_bytes(x.pwidth, x.kp_hi - x.kp_lo, p.w_pad, x.ns, x.rb);
  static int verbose = getenv("PSVD_PASS_VERBOSE") ? atoi(getenv("PSVD_PASS_VERBOSE")) : 0;
  if (verbose > 0) {  // diagnostics: the geometry of the first launches
    --verbose;
    fprintf(stderr, "pass_tma: grid=%d M=%lld np=%d np_pad=%d w=%d wk=%d pwidth=%d kspan=%d ns=%d rb=%d ykp=%d yh=%d "
            "nslices=%d smem=%zu tiles:", grid, (long long)p.M, p.np, p.np_pad, p.w, p.wk, x.pwidth, x.kp_hi - x.kp_lo,
            x.ns, x.rb, p.ykp, p.yh, p.nslices, smem);
    for (int w = 0; w < NWARP; ++w)
      if (p.plan[0][w].ntile) fprintf(stderr, " w%d(%d,%d,sub%02x)", w, p.plan[0][w].ti[0], p.plan[0][w].tj[0], p.plan[0][w].sub);
    if (p.ykp > 1)
      for (int w = 0; w < (p.w_pad / 8) * p.ykp; ++w) fprintf(stderr, " y%d[%d+%d]", w, p.ykj0[w], p.yknj[w]);
    fprintf(stderr, "\n");
  }
  static const bool drop_gram = getenv("PSVD_DBG_DROP_GRAM") != nullptr;  // timing diagnostics only: wrong tiles
  if (drop_gram && x.rb == 2) {
    TallParams q = p;
    const int ny = p.ykp > 1 ? (p.w_pad / 8) * p.ykp : 0;
    for (int sl = 0; sl < MAX_SLICES; ++sl)
      for (int w = ny; w < NWARP; ++w) q.plan[sl][w].ntile = 0;
    cudaFuncSetAttribute(pass_tma_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    pass_tma_kernel<2><<<grid, NTHR, smem, st>>>(q, maps, x);
    return;
  }
  if (x.rb == 2 && p.w_pad <= 16) {
    cudaFuncSetAttribute(pass_tma_kernel<2, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    pass_tma_kernel<2, true><<<grid, NTHR, smem, st>>>(p, maps, x);
  } else if (x.rb == 2) {
    cudaFuncSetAttribute(pass_tma_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    pass_tma_kernel<2><<<grid, NTHR, smem, st>>>(p, maps, x);
  } else {
    cudaFuncSetAttribute(pass_tma_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    pass_tma_kernel<1><<<grid, NTHR, smem, st>>>(p, maps, x);
  }
}

}  // namespace psvd
