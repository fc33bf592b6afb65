// Tall-panel pass: the one kernel family that touches the M-row data.
//
// A "panel" P is the virtual column concatenation of up to 4 column-major
// device matrices (segments), e.g. [U | A_batch] = the reference's
// np.concatenate([ff*U*S, A]) (streaming.py:97-98) without materializing it,
// or [U | A | Y] for the randomized passes.  One pass streams P in 32-row
// stages through shared memory (cp.async, double buffered) and, per stage:
//
//   1. optionally forms Y = P[:, wlo:wlo+wk] * W on FP64 tensor cores (DMMA),
//      W small (wk x w) and resident in smem; Y goes to smem, optionally to
//      global (coalesced) and into a running per-column (max|y|, row) argmax;
//   2. accumulates a selected set of 32x32 tiles of the Gram matrix of the
//      combined column space [P | Y] in registers (DMMA), e.g. the upper
//      triangle of P^T P (deterministic update), Y^T Y and P^T Y (sketch).
//
// Per-CTA partial tiles are summed across CTAs in a fixed order by
// tall_reduce (bitwise reproducible; no atomics), so replicated small
// factorizations on every GPU see identical input.
#pragma once
#include <cuda.h>

#include "psvd_common.cuh"

namespace psvd {

// rows per stage KS is a template parameter (32, or 16 when the panel + W do not
// fit 227 KB); the smem column stride KS + 4 is 4 (mod 16) -> conflict-free fragments.
constexpr int NWARP = 16;  // 4 warps per SMSP keep the DMMA pipe fed through LDS/barrier latency
constexpr int NTHR = NWARP * 32;
constexpr int TPW = 1;     // Gram tiles per warp (64 accumulator doubles -> <= 128 registers)
constexpr int WS_PRODUCERS = 2;  // cp.async producer warps of the warp-specialized Gram
constexpr int MAX_SEG = 4;
constexpr int SLOTS = NWARP * TPW;  // partial tile slots per CTA
constexpr int MAX_SLICES = 4;
constexpr int MAX_OUT_TILES = 64;
constexpr int MAX_W = 128;   // widest Y

struct Seg {
  const double* ptr;
  int64_t ld;
  int ncols;
  int col0;  // first column in the panel space (plan_pass fills it). On input: 1 = start on a
             // 32-column block, 2 = no P^T Y rows wanted for this segment (narrow TMA pass)
};

struct WarpPlan {
  signed char ti[2], tj[2];  // 32-column block indices into [P | Y]
  unsigned char ntile, kpart, ksplit;
  unsigned char sub;  // narrow TMA pass, P-tile: first wanted 8-column sub-block | count << 4 (0: all)
};

struct TallParams {
  int64_t M;
  int64_t rows_per_cta;  // multiple of 32
  int ks;                // rows per stage (32 or 16)
  int nstage;            // cp.async pipeline depth (2 or 3)
  int narrow;            // every Gram tile ends in the Y block (Y <= 16 columns; <= 32 on the TMA pass)
  int dbg;               // diagnostics (PSVD_GRAM_DBG): 1 = skip DMMA, 2 = skip global loads
  int nseg;
  Seg seg[MAX_SEG];
  int np, np_pad;        // panel columns; padded to a multiple of 32 (start of the Y block)
  const double* W;       // Y = P[:, wlo:wlo+wk] * W; W col-major (wk x w), ld ldw; w == 0 -> no Y
  int64_t ldw;
  int wlo, wk, w, w_pad;  // w_pad = round8(w) columns computed; S_Y holds round32(w) columns
  double* Yout;          // optional global copy of Y (col-major, ld ldy)
  int64_t ldy;
  int nslices;
  int yh;                // narrow TMA pass with 32-row stages: 2 = one Y warp per 16-row half of a block
  int ykp;               // narrow TMA pass with 32-row stages: > 1 = W in registers, k split into ykp parts
  unsigned char ykj0[NWARP], yknj[NWARP];  // per Y warp: first k step and step count of its part
  WarpPlan plan[MAX_SLICES][NWARP];
  double* partial;       // [grid][SLOTS][1024]
  double* colmax;        // optional [grid][w][2] = (signed value at max |y|, global row)
  int64_t row_offset;    // global row index of local row 0 (multi-GPU argmax)
  const int* gate;       // optional: skip the pass unless *gate != 0
};

struct ReduceMap {
  int nout;
  int nchunks, nslices;
  short out_id[MAX_OUT_TILES];                    // destination tile id (I * NB + J)
  unsigned char nsrc[MAX_OUT_TILES];
  unsigned char src[MAX_OUT_TILES][NWARP];        // slice * SLOTS + slot
};

size_t tall_smem_bytes(int ks, int np_pad, int wk, int w, int nstage);

void launch_tall(const TallParams& p, int grid, cudaStream_t st);
// Warp-specialized Gram-only pass (w == 0, KS = 32, <= NWARP-1 tiles per slice, ksplit == 1).
size_t gram_ws_smem_bytes(int np_pad, int ns);
void launch_gram_ws(const TallParams& p, int grid, cudaStream_t st);
void launch_tall_reduce(const double* partial, const ReduceMap& map, double* tiles, cudaStream_t st);

// Warp-specialized TMA pass for narrow panels (w <= 32, Gram tiles only against Y):
// every segment starts on an 8-column boundary of the panel (1024-byte swizzle atoms).
constexpr int TMA_MAX_OPS = 16;
constexpr int TMA_NOT_IN_W = -(1 << 30);
constexpr int TMA_MAX_BLK = 192;  // 8-column blocks of the panel
// narrow TMA pass: warps 0 .. 2*ncb-1 form Y (ncb = Y column blocks, w <= 32), the following
// ones own one Gram tile each, the last warp is the TMA producer
constexpr int TMA_MAX_Y = 32;
struct TmaMaps {
  CUtensorMap m[2 * MAX_SEG];  // per segment: 256-column boxes, and the narrower tail box [MAX_SEG + s]
};
struct TmaExtra {
  int nops;
  short op_seg[TMA_MAX_OPS], op_col[TMA_MAX_OPS], op_pcol[TMA_MAX_OPS];  // op_seg: tensor map index
  short op_bw[TMA_MAX_OPS];  // box width (columns)
  int wrow0[MAX_SEG];        // W row of the segment's first column (TMA_NOT_IN_W: outside Y's range)
  int kp_lo, kp_hi;          // Y's k range in physical panel columns
  int pshift;                // physical column = logical column + pshift (narrow pass)
  int pwidth;                // physical ring width (columns)
  unsigned stage_bytes;
  int ns;                    // ring depth (stages)
  int grp;                   // stages issued together (consecutive rows of every column back to back)
  int rb;                    // 16-row blocks per stage of the narrow pass (1: 2-D boxes; 2: 3-D boxes)
  unsigned char written[TMA_MAX_BLK];  // 8-column panel blocks covered by a TMA box
};
bool tma_available();
size_t tma_pass_smem_bytes(int pwidth, int kp_span, int w_pad, int ns = 3, int ny = 1);
int tma_pass_prepare(TallParams& p, TmaMaps& maps, TmaExtra& x, int pshift = 0, bool narrow = false);
void launch_pass_tma(const TallParams& p, const TmaMaps& maps, const TmaExtra& x, int grid, cudaStream_t st);
// Split-ring pass (fused_split_kernel): a narrow pass Y = P_A W with Gram tiles against Y, streamed as
// 32-row stages of two column groups -- group A = the segments W covers (read by the Y warps), group B =
// the others (read by the tile warps) -- each in its own ring of 2 .. FS_NS_MAX slots of 3-D TMA boxes
// (256 contiguous bytes per column and request).  W lives in the Y warps' registers; tile warps own the
// P^T Y sub-blocks of either group and Y^T Y; up to FS_MAX_OFF warps compute 32 x 32 tiles of the Gram of
// group B's segment (the deterministic stream's fused pass over [U | A_b | A_next]: work taken off the
// look-ahead Gram of A_next, whose pass is DMMA-bound while this one is HBM-bound).  run_pass sends every
// narrow TMA pass that qualifies here (fused_split_prepare); the others stay on pass_tma_kernel.
constexpr int FS_WR = 20;      // W fragments (k steps of 4 columns) a Y warp holds in registers
constexpr int FS_NKP = 4;      // k parts per Y column block
constexpr int FS_MAX_OFF = 3;  // offloaded Gram tiles
constexpr int FS_NS_MAX = 4;   // slots per ring
enum { FS_IDLE = 0, FS_Y = 1, FS_PY = 2, FS_OFF = 3, FS_PROD = 4 };
struct FusedSplit {
  int colA0;                     // first panel column of group A (= the first k column of W)
  int pwA, pwB;                  // slot widths in columns (multiples of 8)
  int nopsA, nopsB;              // TMA boxes per stage of each group (group A's come first)
  short opm[TMA_MAX_OPS], opc[TMA_MAX_OPS], opd[TMA_MAX_OPS];  // tensor map, tensor column, slot column
  unsigned bytesA, bytesB;       // bytes per stage of each group
  int ncb;                       // Y column blocks (1 .. 3)
  int n4;                        // k steps of 4 physical panel columns
  int nkp;                       // k parts per Y column block (1, 2 or FS_NKP)
  int ns;                        // slots per ring (2 .. FS_NS_MAX, as shared memory allows)
  int npy, noff;                 // warps with P^T Y (or Y^T Y) tiles / offloaded Gram tiles
  int nA, nB;                    // warps that read group A / group B (they release its ring slots)
  unsigned char role[NWARP];
  unsigned char ycb[NWARP], ykp[NWARP], yj0[NWARP], ynj[NWARP];     // Y warps: column block, part, k steps
  // tile warps: na sub-blocks of 8 columns from sub-block sb0 of their group's slot; rb0 = position of the
  // first one inside its 32-column tile, nt tiles touched, one partial-tile slot each
  unsigned char py_sb0[NWARP], py_na[NWARP], py_yy[NWARP], py_onA[NWARP], py_rb0[NWARP], py_nt[NWARP];
  unsigned char py_slot[NWARP][3], yy_slot;
  unsigned char off_i[NWARP], off_j[NWARP], off_slot[NWARP];       // offloaded tile (I, J) of the B segment's Gram
};
size_t fused_split_smem_bytes(const FusedSplit& fs);
void launch_fused_split(const TallParams& p, const TmaMaps& maps3, const TmaExtra& x, const FusedSplit& fs, int grid,
                        cudaStream_t st);
// builds fs and the 3-D tensor maps from a planned narrow TMA pass (p, x, its reduce map); off: wanted
// offloaded tiles (block pairs of the last segment); returns 0 when the pass qualifies
int fused_split_prepare(const TallParams& p, const TmaExtra& x, ReduceMap& map, int NB, const int (*off)[2],
                        int noff, FusedSplit& fs, TmaMaps& maps3, ReduceMap& offmap, int off_nb);

// TMA-fed Gram-only pass (w == 0, segments on 8-column boundaries, <= NWARP - 1 tiles per slice)
constexpr int TMA_GRAM_CONS = NWARP - 1;
size_t gram_tma_smem_bytes(int np_pad);
void launch_gram_tma(const TallParams& p, const TmaMaps& maps, const TmaExtra& x, int grid, cudaStream_t st);

}  // namespace psvd
