// Tall-panel pass kernels (see psvd_tall.cuh for the contract).
#include <type_traits>

#include "psvd_tall.cuh"

namespace psvd {

__host__ __device__ static inline int round_up(int x, int m) { return (x + m - 1) / m * m; }

size_t tall_smem_bytes(int ks, int np_pad, int wk, int w, int nstage) {
  const int ksp = ks + 4;
  size_t b = 0;
  b += sizeof(const double*) * (size_t)np_pad;  // column base pointers
  b = (b + 15) / 16 * 16;
  b += sizeof(double) * nstage * (size_t)np_pad * ksp;  // multi-buffered panel stages
  if (w > 0) {
    b += sizeof(double) * (size_t)round_up(w, 32) * ksp;                    // Y stage
    b += sizeof(double) * (size_t)round_up(wk, 4) * (round_up(w, 8) + 4);   // W
  }
  return b;
}

// NJB: 8-column blocks computed per Gram tile column (4 = full 32x32 tile; 2 when
// every tile's column block is a Y block of <= 16 columns, e.g. U^T U and A^T U
// for K <= 16 — halves the DMMA work of the fused recompose pass).
template <int KS, int MAXCB, int NS, int NJB>
__global__ void __launch_bounds__(NTHR, 1) tall_pass_kernel(const TallParams p) {
  constexpr int KSP = KS + 4;   // = 4 (mod 16)
  constexpr int RB = KS / 8;    // 8-row blocks per stage
  constexpr int CG = NWARP / RB;  // warp groups over Y column blocks
  if (p.gate != nullptr && *p.gate == 0) return;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, tq = lane & 3;
  const int slice = blockIdx.x % p.nslices;
  const int64_t chunk = blockIdx.x / p.nslices;
  const int64_t row_begin = chunk * p.rows_per_cta;
  const int64_t row_end = min(p.M, row_begin + p.rows_per_cta);
  const int np_pad = p.np_pad, w_pad = p.w_pad;
  const bool has_y = p.w > 0;
  const int wk_pad = (p.wk + 3) & ~3;
  const int wsp = w_pad + 4;
  const int ycols = has_y ? round_up(p.w, 32) : 0;

  const double** colptr = reinterpret_cast<const double**>(smem_raw);
  size_t off = ((sizeof(const double*) * (size_t)np_pad) + 15) / 16 * 16;
  double* sP = reinterpret_cast<double*>(smem_raw + off);
  off += sizeof(double) * NS * (size_t)np_pad * KSP;
  double* sY = reinterpret_cast<double*>(smem_raw + off);
  double* sW = sY + (size_t)ycols * KSP;

  for (int c = tid; c < np_pad; c += NTHR) {
    const double* ptr = nullptr;
    for (int s = 0; s < p.nseg; ++s) {
      const int c0 = p.seg[s].col0;
      if (c >= c0 && c < c0 + p.seg[s].ncols) ptr = p.seg[s].ptr + (int64_t)(c - c0) * p.seg[s].ld;
    }
    colptr[c] = ptr;
  }
  __syncthreads();
  // zero the padding columns (no source) of every stage buffer; cp.async never writes them
  for (int i = tid; i < NS * np_pad * KSP; i += NTHR) {
    const int c = (i / KSP) % np_pad;
    if (colptr[c] == nullptr) sP[i] = 0.0;
  }
  if (has_y) {
    for (int i = tid; i < ycols * KSP; i += NTHR) sY[i] = 0.0;
    for (int i = tid; i < wk_pad * wsp; i += NTHR) {
      const int k = i / wsp, o = i % wsp;
      sW[i] = (k < p.wk && o < p.w) ? p.W[(int64_t)o * p.ldw + k] : 0.0;
    }
  }
  __syncthreads();

  const int64_t nstage = row_end > row_begin ? (row_end - row_begin + KS - 1) / KS : 0;
  const int nchunk16 = p.np * (KS / 2);

  auto prefetch = [&](int64_t s, int buf) {
    const int64_t r0 = row_begin + s * KS;
    double* dst_base = sP + (size_t)buf * np_pad * KSP;
    for (int q = tid; q < nchunk16; q += NTHR) {
      const int c = q / (KS / 2), pc = q % (KS / 2);
      const int64_t r = r0 + 2 * pc;
      const int64_t valid = row_end - r;
      const int bytes = valid >= 2 ? 16 : (valid == 1 ? 8 : 0);
      const double* cp = colptr[c];
      if (cp == nullptr) continue;  // padding column: stays zero
      cp_async16(dst_base + (size_t)c * KSP + 2 * pc, cp + (bytes > 0 ? r : row_begin), bytes);
    }
  };

  const WarpPlan wp = p.plan[slice][warp];
  double acc[TPW][4][4][2];
#pragma unroll
  for (int t = 0; t < TPW; ++t)
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) acc[t][a][b][0] = acc[t][a][b][1] = 0.0;

  double cm_val = 0.0, cm_abs = -1.0;
  int64_t cm_row = -1;
  const bool do_cm = has_y && p.colmax != nullptr && slice == 0 && tid < p.w;

  // NS-stage cp.async pipeline: stage s lives in buffer s % NS; the barrier at the top of
  // iteration s also retires iteration s-1, whose buffer the new prefetch reuses
#pragma unroll
  for (int s0 = 0; s0 < NS - 1; ++s0) {
    if (s0 < nstage) prefetch(s0, s0);
    cp_async_commit();
  }

  for (int64_t s = 0; s < nstage; ++s) {
    const int buf = (int)(s % NS);
    cp_async_wait<NS - 2>();
    __syncthreads();
    if (s + NS - 1 < nstage) prefetch(s + NS - 1, (int)((s + NS - 1) % NS));
    cp_async_commit();
    const double* P = sP + (size_t)buf * np_pad * KSP;
    const int64_t r0 = row_begin + s * KS;

    if (has_y) {
      // Y(KS x w_pad) = P[:, wlo:wlo+wk] * W on DMMA; warp -> row block rb, column blocks cb0 + CG*j
      const int rb = warp % RB, cb0 = warp / RB, ncb = w_pad >> 3;
      double ya[MAXCB][2], yb[MAXCB][2];  // two accumulator chains (even / odd k-steps)
#pragma unroll
      for (int j = 0; j < MAXCB; ++j) ya[j][0] = ya[j][1] = yb[j][0] = yb[j][1] = 0.0;
      const double* pa = P + (size_t)(p.wlo + tq) * KSP + rb * 8 + g;
      const double* pb = sW + (size_t)tq * wsp + g;
      int k0 = 0;
      for (; k0 + 8 <= wk_pad; k0 += 8) {
        const double a0 = pa[(size_t)k0 * KSP], a1 = pa[(size_t)(k0 + 4) * KSP];
#pragma unroll
        for (int j = 0; j < MAXCB; ++j) {
          const int cb = cb0 + CG * j;
          if (cb < ncb) {
            dmma884(ya[j][0], ya[j][1], a0, pb[(size_t)k0 * wsp + cb * 8]);
            dmma884(yb[j][0], yb[j][1], a1, pb[(size_t)(k0 + 4) * wsp + cb * 8]);
          }
        }
      }
      if (k0 < wk_pad) {
        const double a0 = pa[(size_t)k0 * KSP];
#pragma unroll
        for (int j = 0; j < MAXCB; ++j) {
          const int cb = cb0 + CG * j;
          if (cb < ncb) dmma884(ya[j][0], ya[j][1], a0, pb[(size_t)k0 * wsp + cb * 8]);
        }
      }
#pragma unroll
      for (int j = 0; j < MAXCB; ++j) {
        ya[j][0] += yb[j][0];
        ya[j][1] += yb[j][1];
      }
#pragma unroll
      for (int j = 0; j < MAXCB; ++j) {
        const int cb = cb0 + CG * j;
        if (cb < ncb) {
          sY[(size_t)(cb * 8 + 2 * tq) * KSP + rb * 8 + g] = ya[j][0];
          sY[(size_t)(cb * 8 + 2 * tq + 1) * KSP + rb * 8 + g] = ya[j][1];
        }
      }
      __syncthreads();
      if (slice == 0) {
        if (p.Yout != nullptr) {
          for (int q = tid; q < p.w * (KS / 2); q += NTHR) {
            const int o = q / (KS / 2), pc = q % (KS / 2);
            const int64_t r = r0 + 2 * pc;
            double* dst = p.Yout + (int64_t)o * p.ldy + r;
            const double v0 = sY[(size_t)o * KSP + 2 * pc], v1 = sY[(size_t)o * KSP + 2 * pc + 1];
            if (r + 1 < row_end) {
              *reinterpret_cast<double2*>(dst) = make_double2(v0, v1);
            } else if (r < row_end) {
              dst[0] = v0;
            }
          }
        }
        if (do_cm) {
          const int nr = (int)((row_end - r0) < KS ? (row_end - r0) : KS);
          for (int r = 0; r < nr; ++r) {
            const double v = sY[(size_t)tid * KSP + r];
            if (fabs(v) > cm_abs) {
              cm_abs = fabs(v);
              cm_val = v;
              cm_row = r0 + r;
            }
          }
        }
      }
    }

    // Gram tiles over the combined [P | Y] column space
    if (wp.ntile > 0 && wp.ksplit == 1) {
#pragma unroll
      for (int kk = 0; kk < KS / 4; ++kk) {
        const int k0 = kk * 4;
#pragma unroll
        for (int t = 0; t < TPW; ++t) {
          if (t < wp.ntile) {
            const int I = wp.ti[t], J = wp.tj[t];
            const double* bI = (I * 32 < np_pad) ? P + (size_t)I * 32 * KSP : sY + (size_t)(I * 32 - np_pad) * KSP;
            const double* bJ = (J * 32 < np_pad) ? P + (size_t)J * 32 * KSP : sY + (size_t)(J * 32 - np_pad) * KSP;
            double fa[4], fb[NJB];
#pragma unroll
            for (int q = 0; q < 4; ++q) fa[q] = bI[(size_t)(q * 8 + g) * KSP + k0 + tq];
#pragma unroll
            for (int q = 0; q < NJB; ++q) fb[q] = bJ[(size_t)(q * 8 + g) * KSP + k0 + tq];
#pragma unroll
            for (int a = 0; a < 4; ++a)
#pragma unroll
              for (int b = 0; b < NJB; ++b) dmma884(acc[t][a][b][0], acc[t][a][b][1], fa[a], fb[b]);
          }
        }
      }
    } else if (wp.ntile > 0) {
      for (int kk = wp.kpart; kk < KS / 4; kk += wp.ksplit) {
        const int k0 = kk * 4;
#pragma unroll
        for (int t = 0; t < TPW; ++t) {
          if (t < wp.ntile) {
            const int I = wp.ti[t], J = wp.tj[t];
            const double* bI = (I * 32 < np_pad) ? P + (size_t)I * 32 * KSP : sY + (size_t)(I * 32 - np_pad) * KSP;
            const double* bJ = (J * 32 < np_pad) ? P + (size_t)J * 32 * KSP : sY + (size_t)(J * 32 - np_pad) * KSP;
            double fa[4], fb[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              fa[q] = bI[(size_t)(q * 8 + g) * KSP + k0 + tq];
              fb[q] = bJ[(size_t)(q * 8 + g) * KSP + k0 + tq];
            }
#pragma unroll
            for (int a = 0; a < 4; ++a)
#pragma unroll
              for (int b = 0; b < 4; ++b) dmma884(acc[t][a][b][0], acc[t][a][b][1], fa[a], fb[b]);
          }
        }
      }
    }
  }
  cp_async_wait<0>();

  if (wp.ntile > 0) {
#pragma unroll
    for (int t = 0; t < TPW; ++t) {
      if (t < wp.ntile) {
        double* dst = p.partial + ((size_t)blockIdx.x * SLOTS + warp * TPW + t) * 1024;
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int b = 0; b < 4; ++b)
            *reinterpret_cast<double2*>(dst + (a * 8 + g) * 32 + b * 8 + 2 * tq) =
                make_double2(acc[t][a][b][0], acc[t][a][b][1]);
      }
    }
  }
  if (do_cm) {
    double* dst = p.colmax + ((size_t)chunk * p.w + tid) * 2;
    dst[0] = cm_val;
    dst[1] = (double)(cm_row + p.row_offset);
  }
}

// Fixed-order reduction of the per-CTA partial tiles: block (32 elements of one
// output tile) x 8 warps; warp w sums sources w, w+8, ... (chunk-major order),
// then the 8 warp sums are added in warp order.  Bitwise reproducible.
// ---------------------------------------------------------------- warp-specialized Gram
// Gram-only passes (no Y): warp NWARP-1 streams 32-row stages into an NS-deep
// ring with cp.async + mbarrier (full[b]: 32 producer lanes, empty[b]: the
// consumer warps); warps 0..NWARP-2 each own one 32x32 tile and never wait on
// a CTA barrier, so the DMMA pipe is not drained at stage boundaries.
size_t gram_ws_smem_bytes(int np_pad, int ns) {
  size_t b = sizeof(const double*) * (size_t)np_pad;
  b = (b + 15) / 16 * 16;
  b += 2 * ns * sizeof(uint64_t);
  b = (b + 15) / 16 * 16;
  return b + sizeof(double) * ns * (size_t)np_pad * 36;
}

template <int NS>
__global__ void __launch_bounds__(NTHR, 1) gram_ws_kernel(const TallParams p) {
  constexpr int KS = 32, KSP = 36;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, tq = lane & 3;
  const int slice = blockIdx.x % p.nslices;
  const int64_t chunk = blockIdx.x / p.nslices;
  const int64_t row_begin = chunk * p.rows_per_cta;
  const int64_t row_end = min(p.M, row_begin + p.rows_per_cta);
  const int np_pad = p.np_pad;
  const double** colptr = reinterpret_cast<const double**>(smem_raw);
  size_t off = ((sizeof(const double*) * (size_t)np_pad) + 15) / 16 * 16;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw + off);
  uint64_t* empty = full + NS;
  off += (2 * NS * sizeof(uint64_t) + 15) / 16 * 16;
  double* sP = reinterpret_cast<double*>(smem_raw + off);
  constexpr int PROD = NWARP - WS_PRODUCERS;  // first producer warp
  int ncons = 0;  // consumer warps of this slice (all arrive on `empty`)
  for (int w = 0; w < PROD; ++w) ncons += p.plan[slice][w].ntile > 0;
  for (int c = tid; c < np_pad; c += NTHR) {
    const double* ptr = nullptr;
    for (int s = 0; s < p.nseg; ++s) {
      const int c0 = p.seg[s].col0;
      if (c >= c0 && c < c0 + p.seg[s].ncols) ptr = p.seg[s].ptr + (int64_t)(c - c0) * p.seg[s].ld;
    }
    colptr[c] = ptr;
  }
  __syncthreads();
  // zero the padding columns (no source) of every stage buffer; cp.async never writes them
  for (int i = tid; i < NS * np_pad * KSP; i += NTHR) {
    const int c = (i / KSP) % np_pad;
    if (colptr[c] == nullptr) sP[i] = 0.0;
  }
  if (tid == 0) {
    for (int b = 0; b < NS; ++b) {
      mbar_init(&full[b], 32 * WS_PRODUCERS);
      mbar_init(&empty[b], (unsigned)max(ncons, 1));
    }
  }
  __syncthreads();
  const int64_t nstage = row_end > row_begin ? (row_end - row_begin + KS - 1) / KS : 0;

  if (warp >= PROD) {
    // producer lanes: fixed 16-byte row piece pc, columns c = cstream + k * cstride
    const int pl = (warp - PROD) * 32 + lane;
    const int pc = pl & 15, cstream = pl >> 4, cstride = (32 * WS_PRODUCERS) >> 4;
    for (int64_t s = 0; s < nstage; ++s) {
      const int b = (int)(s % NS);
      if (s >= NS) mbar_wait(&empty[b], (unsigned)(((s / NS) - 1) & 1));
      const int64_t r = row_begin + s * KS + 2 * pc;
      const int64_t valid = row_end - r;
      const int bytes = valid >= 2 ? 16 : (valid == 1 ? 8 : 0);
      const int64_t roff = bytes > 0 ? r : row_begin;
      double* dst = sP + (size_t)b * np_pad * KSP + 2 * pc;
      if (!(p.dbg & 2)) {
        for (int c = cstream; c < p.np; c += cstride) {
          const double* cp = colptr[c];
          if (cp != nullptr) cp_async16(dst + (size_t)c * KSP, cp + roff, bytes);
        }
      }
      cp_async_mbar_arrive(&full[b]);
    }
    cp_async_wait<0>();
    return;
  }

  const WarpPlan wp = p.plan[slice][warp];
  if (wp.ntile == 0) return;
  double acc[4][4][2];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
  const int I = wp.ti[0], J = wp.tj[0];
  // Which 8x8 blocks this warp's tile needs: diagonal tiles only b >= a (extraction reads
  // row <= col), blocks past the last panel column are skipped.  The shape is fixed for
  // the whole kernel, so each warp runs one specialized stage loop (no per-step branches).
  const int nva = min(4, (p.np - I * 32 + 7) / 8), nvb = min(4, (p.np - J * 32 + 7) / 8);
  // Tile shape, compile-time in the stage loop (a DMMA under a runtime predicate costs a
  // warp reconvergence each; such warps would pace the whole CTA through the ring):
  //   DIAG: block (a, c) needed iff c >= a (extraction reads row <= col);
  //   NA x NB: valid 8-row / 8-column blocks (last panel block partially filled).
  auto stage_loop = [&](auto na_t, auto nb_t, auto diag_t) {
    constexpr int NA = decltype(na_t)::value, NB = decltype(nb_t)::value;
    constexpr bool DIAG = decltype(diag_t)::value;
    for (int64_t s = 0; s < nstage; ++s) {
      const int b = (int)(s % NS);
      mbar_wait(&full[b], (unsigned)((s / NS) & 1));
      const double* P = sP + (size_t)b * np_pad * KSP;
      const double* bI = P + (size_t)I * 32 * KSP + g * KSP + tq;
      const double* bJ = P + (size_t)J * 32 * KSP + g * KSP + tq;
#pragma unroll
      for (int kk = 0; kk < KS / 4; ++kk) {
        double fa[NA], fb[NB];
#pragma unroll
        for (int q = 0; q < NA; ++q) fa[q] = bI[(size_t)q * 8 * KSP + kk * 4];
#pragma unroll
        for (int q = 0; q < NB; ++q) fb[q] = bJ[(size_t)q * 8 * KSP + kk * 4];
#pragma unroll
        for (int a = 0; a < NA; ++a)
#pragma unroll
          for (int c = 0; c < NB; ++c)
            if (!DIAG || c >= a) {
              if (!(p.dbg & 1)) dmma884(acc[a][c][0], acc[a][c][1], fa[a], fb[c]);
            }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[b]);
    }
  };
  using F = std::false_type;
  using T = std::true_type;
  auto C = [](auto v) { return std::integral_constant<int, decltype(v)::value>{}; };
  (void)C;
  if (I != J) {
    if (nva == 4 && nvb == 4) stage_loop(std::integral_constant<int, 4>{}, std::integral_constant<int, 4>{}, F{});
    else if (nvb == 3) stage_loop(std::integral_constant<int, 4>{}, std::integral_constant<int, 3>{}, F{});
    else if (nvb == 2) stage_loop(std::integral_constant<int, 4>{}, std::integral_constant<int, 2>{}, F{});
    else stage_loop(std::integral_constant<int, 4>{}, std::integral_constant<int, 1>{}, F{});
  } else {
    if (nva == 4) stage_loop(std::integral_constant<int, 4>{}, std::integral_constant<int, 4>{}, T{});
    else if (nva == 3) stage_loop(std::integral_constant<int, 3>{}, std::integral_constant<int, 3>{}, T{});
    else if (nva == 2) stage_loop(std::integral_constant<int, 2>{}, std::integral_constant<int, 2>{}, T{});
    else stage_loop(std::integral_constant<int, 1>{}, std::integral_constant<int, 1>{}, T{});
  }
  double* dst = p.partial + ((size_t)blockIdx.x * SLOTS + warp * TPW) * 1024;
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int c = 0; c < 4; ++c)
      *reinterpret_cast<double2*>(dst + (a * 8 + g) * 32 + c * 8 + 2 * tq) = make_double2(acc[a][c][0], acc[a][c][1]);
}

void launch_gram_ws(const TallParams& p, int grid, cudaStream_t st) {
  const size_t smem = gram_ws_smem_bytes(p.np_pad, 3);
  cudaFuncSetAttribute(gram_ws_kernel<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  gram_ws_kernel<3><<<grid, NTHR, smem, st>>>(p);
}

__global__ void __launch_bounds__(256) tall_reduce_kernel(const double* __restrict__ partial, const ReduceMap map,
                                                          double* __restrict__ tiles) {
  __shared__ double red[8][33];
  const int o = blockIdx.y;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int e = blockIdx.x * 32 + lane;
  const int ns = map.nsrc[o];
  const int total = map.nchunks * ns;
  double s = 0.0;
  for (int q = warp; q < total; q += 8) {
    const int c = q / ns, i = q % ns;
    const int sl = map.src[o][i] / SLOTS, slot = map.src[o][i] % SLOTS;
    s += partial[((size_t)(c * map.nslices + sl) * SLOTS + slot) * 1024 + e];
  }
  red[warp][lane] = s;
  __syncthreads();
  if (warp == 0) {
    double t = 0.0;
#pragma unroll
    for (int w = 0; w < 8; ++w) t += red[w][lane];
    tiles[(size_t)map.out_id[o] * 1024 + e] = t;
  }
}

template <int KS, int NS, int NJB>
static void launch_ks(const TallParams& p, int grid, size_t smem, cudaStream_t st) {
  const int ncb = p.w_pad / 8;
  constexpr int CG = NWARP / (KS / 8);
  const int per = (ncb + CG - 1) / CG;
#define PSVD_LAUNCH(MCB)                                                                                   \
  do {                                                                                                     \
    cudaFuncSetAttribute(tall_pass_kernel<KS, MCB, NS, NJB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
    tall_pass_kernel<KS, MCB, NS, NJB><<<grid, NTHR, smem, st>>>(p);                                       \
  } while (0)
  if (per <= 1)
    PSVD_LAUNCH(1);
  else if (per <= 2)
    PSVD_LAUNCH(2);
  else
    PSVD_LAUNCH(4);  // w <= MAX_W = 128 -> at most 16 column blocks over CG = 4 warp groups
#undef PSVD_LAUNCH
}

void launch_tall(const TallParams& p, int grid, cudaStream_t st) {
  const size_t smem = tall_smem_bytes(p.ks, p.np_pad, p.wk, p.w, p.nstage);
  if (p.narrow) {
    if (p.ks == 32 && p.nstage == 3)
      launch_ks<32, 3, 2>(p, grid, smem, st);
    else if (p.ks == 32)
      launch_ks<32, 2, 2>(p, grid, smem, st);
    else
      launch_ks<16, 2, 2>(p, grid, smem, st);
  } else if (p.ks == 32 && p.nstage == 3) {
    launch_ks<32, 3, 4>(p, grid, smem, st);
  } else if (p.ks == 32) {
    launch_ks<32, 2, 4>(p, grid, smem, st);
  } else {
    launch_ks<16, 2, 4>(p, grid, smem, st);
  }
}

void launch_tall_reduce(const double* partial, const ReduceMap& map, double* tiles, cudaStream_t st) {
  if (map.nout == 0) return;
  dim3 grid(1024 / 32, map.nout);
  tall_reduce_kernel<<<grid, 256, 0, st>>>(partial, map, tiles);
}

}  // namespace psvd
