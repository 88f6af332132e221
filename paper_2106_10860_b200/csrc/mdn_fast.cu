// Fast sm_100a kernels for the MADDNESS hot path.
//
// k_amm_ws: the fused g + f + dequant (mdn_amm) and the encode-only variant
// (mdn_encode). One persistent CTA per SM, warp-specialised:
//
//   warp 0          TMA producer: 2-D tensor copies of A row tiles into a ring
//                   of NS shared-memory stages (mbarrier complete_tx)
//   warps 1..E      encoders: Algorithm 1 on every
//                   (row, codebook) of a stage, fp32 compares against thresholds
//                   resident in shared memory; packed 4-bit codes go to a ring
//                   of NB code tiles in shared memory (never to HBM)
//   warps E+1..E+S  scanners: one row per thread; the C x 16 x M uint8 tables
//                   stay resident in shared memory as 32-bit words holding 4
//                   output columns ("f"; the paper's column-pair
//                   fusion, App. D, generalised to 4 columns per lookup);
//                   exact sums in 2 x 16-bit SWAR lanes, or the App. D
//                   averaging tree (4-lane byte average, L335, L697-706); then
//                   out = alpha * S + beta (Eq. 1) and coalescing-friendly
//                   128-bit stores.
//
// Stage layout: A rows [y, y + R) are fetched as nslab boxes of
// (SW + 4) x R floats (slab k covers columns [k SW, k SW + SW + 4)); the 4
// extra columns pad each row to a pitch of SW + 4 words (== 4 mod 32 for
// SW = 128 or 32), which spreads the encoders' per-row reads over banks; the
// tail beyond column D and rows beyond N are zero-filled by the TMA unit.
//
// k_scan_fast: mdn_scan from packed codes in HBM, thread per row, tables in
// shared memory.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdlib>
#include <map>
#include <mutex>

#include "mdn_internal.h"
#include "mdn_tma.cuh"
#include "mdn_scan.cuh"

namespace mdn {
namespace fast {

constexpr int BR = 256;                  // rows per tile
constexpr int NB = 3;                    // code ring depth (tiles)
constexpr int NS_MAX = 16;               // A stage ring depth cap
constexpr int BAR_BYTES = 384;           // full/empty[NS_MAX] + cfull/cempty[NB] mbarriers
static_assert((2 * NS_MAX + 2 * NB) * 8 <= BAR_BYTES, "mbarriers must fit below the tables");
constexpr int CM = -1;                   // SUBF value of the column-major-A variant

// Shared-memory word offsets of codebook c's 16 thresholds / 4 split offsets.
// The encoder lanes of a warp cover up to NG = C / 8 codebook groups (one
// codebook 8g + i each at step i); padding by 8 (4) words per group puts the
// groups' threshold (offset) blocks in different banks: conflict-free gathers
// for NG <= 4, 2-way for NG = 8.
__host__ __device__ constexpr int thr_base(int c) { return 16 * c + 8 * (c >> 3); }
__host__ __device__ constexpr int off_base(int c) { return 4 * c + 4 * (c >> 3); }

// Warp roles. Per row an encoder spends ~25 instructions per codebook
// (4 split-dim loads, 4 threshold gathers, compares), a scanner ~4W per
// codebook (W table words of 4 columns), so the encoder:scanner split follows
// 25 : 4W -- 2:8 for the 100-column tables, 6:4 for 10-16 columns, 8:2 for
// <= 8 columns (ncu on the image config: scanners idle 63% at 2:8).
// Exact-mode pipe mix of the scanner warps (mdn_scan.cuh) in the column-major
// kernel, whose scanners bound cls100 (ALU pipe 75%): on for the wide tables
// only (same box, mix vs ALU-only: cls100 (W = 25) 4.14 -> 4.20e9 rows/s;
// scale (W = 4) 1.04 -> 1.02e10, cls10_c16 -5%). The row-major kernel keeps
// ALU-only adds (the mix cost cls100 5% there).
#ifndef MDN_CM_MIX
#define MDN_CM_MIX 3
#endif

#ifndef MDN_E_WIDE
#define MDN_E_WIDE 2         // encoder warps of the row-major kernel for W >= 8 (cls100)
#endif
#ifndef MDN_CM_E
#define MDN_CM_E 6           // encoder warps of the column-major kernel for W >= 8 (cls100)
#endif
#ifndef MDN_E_MID
#define MDN_E_MID 6          // encoder warps for 3 <= W < 8 (tuning experiments: -DMDN_E_MID=...)
#endif
#ifndef MDN_S_MID
#define MDN_S_MID 4          // scanner warps for 3 <= W < 8 (tuning experiments: -DMDN_S_MID=...)
#endif

template <int W, bool ENC_ONLY, bool CMV = false>
struct Roles {
  // Column-major A with wide tables runs ~35% more rows/s than row-major
  // (fewer bytes per row), so it gets 6 encoder warps instead of 2 (cls100:
  // 3.65 -> 4.11e9 rows/s; 2 encoder warps could not keep up).
  static constexpr int E = ENC_ONLY ? 8 : (W >= 8 ? (CMV ? MDN_CM_E : MDN_E_WIDE) : (W >= 3 ? MDN_E_MID : 8));
  static constexpr int S = ENC_ONLY ? 0 : (W >= 8 ? 8 : (W >= 3 ? MDN_S_MID : 2));
  static constexpr int THREADS = 32 * (1 + E + S);
  static constexpr int ROWS_PER_SCANNER = ENC_ONLY ? 0 : BR / (32 * S);
};

struct Params {
  int64_t N;
  int64_t n_tiles;
  int64_t ldo;
  int D, SW, nslab, R, NS;
  int slab_e;                     // shared-memory elements (of the input type) per slab, 128-B aligned
  int pad_e;                      // row pitch = SW + pad_e elements (16 bytes of padding)
  int M;
  int ntile;                      // TILED: column tiles of W words (ceil(Wfull / W))
  int Wfull;                      // TILED: the tables' full width in words (ceil(M / 4))
  bool pair;                      // M even, ldo even, out 8-B aligned: 8-byte stores
  int l2_hint;                    // 0 none (default), 1 evict_first, 2 evict_last, 3 evict_normal
  float alpha_eff, beta32;
  const uint32_t* lut;            // global [C][W][16]
  const uint16_t* dims;           // global [C][4]
  const uint16_t* sub;            // global [C] subspace begin
  const float* thr;               // global [C][16]
  const uint16_t* q;              // global [C][16] 8-bit split values ceil(v) (uint8 input)
  const uint16_t* slot;           // column-major A: global [D] stage slot of each split column
  const uint16_t* cols;           // column-major A: global [n_cols] split column of each slot
  int n_cols;                     // column-major A: distinct split columns (nslab = n_cols rounded up to 4)
  float* out;
  uint8_t* codes;                 // encode-only output
};

// ------------------------------------------------------------ fused kernel --

__device__ __forceinline__ float pick4(const float4& v, int s) {
  const float a = (s & 1) ? v.y : v.x;
  const float b = (s & 1) ? v.w : v.z;
  return (s & 2) ? b : a;
}

// fp32 input (TIn = float):
//   SUBF = 0: the 4 split-dim values are read one by one (s_off: offsets).
//   SUBF = 1 / 2: the codebook's whole subspace (<= 4 / <= 8 columns, 16-B
//   aligned) is read with 1 / 2 conflict-free LDS.128 (row pitch == 4 mod 32
//   words) and the split dims picked with warp-uniform selects (s_off: column
//   within the subspace, s_base: subspace offset) -- 4x / 2x fewer shared
//   wavefronts than four 4-way-conflicted LDS.32.
// 8-bit input (TIn = uint8_t): thresholds are the
// integer split values q = ceil(v) (App. B, reading R11) and x >= q is an
//   integer compare. SUBF = 1 / 2: every subspace is exactly 4 / 8 bytes, so
//   the unit's G codebooks occupy 4G / 8G contiguous bytes, fetched with
//   LDS.128 and split into bytes with PRMT.
__device__ __forceinline__ uint32_t byte_of(uint32_t lo, uint32_t hi, int sel) {
  return __byte_perm(lo, hi, (uint32_t)sel) & 0xFFu;     // byte sel (0..7) of {hi:lo}
}

template <class TIn, int C, int SUBF>
__device__ __forceinline__ uint32_t encode_group(const TIn* __restrict__ rowp,
                                                 const int* __restrict__ s_off,
                                                 const int* __restrict__ s_base,
                                                 const float* __restrict__ s_thr, int c0) {
  constexpr int G = C >= 8 ? 8 : C;
  uint32_t word = 0;
  if constexpr (sizeof(TIn) == 1) {
    const int* s_q = reinterpret_cast<const int*>(s_thr);
    uint32_t wv[SUBF <= 0 ? 1 : G * SUBF];
    if constexpr (SUBF > 0) {
      const uint4* src = reinterpret_cast<const uint4*>(rowp + s_base[c0]);
#pragma unroll
      for (int k = 0; k < G * SUBF / 4; ++k) {
        const uint4 v = src[k];
        wv[4 * k] = v.x, wv[4 * k + 1] = v.y, wv[4 * k + 2] = v.z, wv[4 * k + 3] = v.w;
      }
    }
#pragma unroll
    for (int i = 0; i < G; ++i) {
      const int c = c0 + i;
      const int4 o = *reinterpret_cast<const int4*>(s_off + off_base(c));
      int x0, x1, x2, x3;
      if constexpr (SUBF <= 0) {
        x0 = rowp[o.x], x1 = rowp[o.y], x2 = rowp[o.z], x3 = rowp[o.w];
      } else if constexpr (SUBF == 1) {
        x0 = byte_of(wv[i], 0u, o.x), x1 = byte_of(wv[i], 0u, o.y);
        x2 = byte_of(wv[i], 0u, o.z), x3 = byte_of(wv[i], 0u, o.w);
      } else {
        x0 = byte_of(wv[2 * i], wv[2 * i + 1], o.x), x1 = byte_of(wv[2 * i], wv[2 * i + 1], o.y);
        x2 = byte_of(wv[2 * i], wv[2 * i + 1], o.z), x3 = byte_of(wv[2 * i], wv[2 * i + 1], o.w);
      }
      const int* th = s_q + thr_base(c);
      uint32_t p = x0 >= th[0] ? 1u : 0u;
      p = 2u * p + (x1 >= th[1 + p] ? 1u : 0u);
      p = 2u * p + (x2 >= th[3 + p] ? 1u : 0u);
      p = 2u * p + (x3 >= th[7 + p] ? 1u : 0u);
      word |= p << (4 * i);
    }
    return word;
  } else {
#pragma unroll
  for (int i = 0; i < G; ++i) {
    const int c = c0 + i;
    const int4 o = *reinterpret_cast<const int4*>(s_off + off_base(c));
    float x0, x1, x2, x3;
    if constexpr (SUBF <= 0) {
      x0 = rowp[o.x], x1 = rowp[o.y], x2 = rowp[o.z], x3 = rowp[o.w];
    } else {
      const float4* vb = reinterpret_cast<const float4*>(rowp + s_base[c]);
      const float4 v0 = vb[0];
      if constexpr (SUBF == 1) {
        x0 = pick4(v0, o.x), x1 = pick4(v0, o.y), x2 = pick4(v0, o.z), x3 = pick4(v0, o.w);
      } else {
        const float4 v1 = vb[1];
        x0 = (o.x & 4) ? pick4(v1, o.x) : pick4(v0, o.x);
        x1 = (o.y & 4) ? pick4(v1, o.y) : pick4(v0, o.y);
        x2 = (o.z & 4) ? pick4(v1, o.z) : pick4(v0, o.z);
        x3 = (o.w & 4) ? pick4(v1, o.w) : pick4(v0, o.w);
      }
    }
    const float* th = s_thr + thr_base(c);
    // Algorithm 1: i <- 2i - 1 + [x_{j^t} >= v^t_i]  (0-based: p <- 2p + b)
    uint32_t p = x0 >= th[0] ? 1u : 0u;
    p = 2u * p + (x1 >= th[1 + p] ? 1u : 0u);
    p = 2u * p + (x2 >= th[3 + p] ? 1u : 0u);
    p = 2u * p + (x3 >= th[7 + p] ? 1u : 0u);
    word |= p << (4 * i);
  }
  return word;
  }
}

// PROBE (mdn_amm_probe): the same kernel -- producer, TMA boxes, stage and code
// rings, barriers, grid, warp roles, output stores -- with Algorithm 1 and the
// table scan removed (encoders only hand the stages back, scanners store
// beta32 for every output): the data-movement ceiling of this pipeline.
// TILED: table widths without a compiled kernel. The tables are cut into
// p.ntile column tiles of W words (16 output columns for W = 4), laid out
// [tile][c][W][16] after the stage ring, and every scanner row walks the
// tiles: scan_core of tile t, then the row's columns [16 t, 16 t + 16). The
// encoders and the code hand-off are unchanged; warp roles are the wide-table
// ones (E2:S8 from W = 8), since a row then costs ntile times a W-word scan.
// Wide-table output rows staged through shared memory (MDN_SCAN_STAGE): with
// lane = row every float4 store of a warp hit 32 different rows (32 partial
// sectors per instruction), and those stores share the L1 / shared-memory
// data path with the table lookups -- the scan's own arithmetic alone reaches
// 0.94 of the 128 B/clk crossbar, with the per-row stores 0.41
// (scripts/micro/lds_rate.cu). Staged, each half row set (32 rows x <= 52
// columns) leaves in coalesced runs of whole rows.
#ifndef MDN_SCAN_STAGE
#define MDN_SCAN_STAGE 1
#endif
template <int W, bool VEC>
constexpr bool scan_stage() {
  return MDN_SCAN_STAGE != 0 && VEC && W >= 8;
}
// staging float4 per row: ceil(W / 2) (the larger half) rounded up to odd, so
// the lanes' row pitches land on distinct 4-bank groups per quarter warp
template <int W>
constexpr int scan_stage_pitch() {
  return ((W + 1) / 2) | 1;
}
template <int W>
constexpr int scan_stage_floats() {
  return 32 * 4 * scan_stage_pitch<W>();
}
// Column-major fused kernel (k_amm_ws<..., CM>), wide tables: its 8 scanner
// warps stage their rows in 4 parts of CM_PART words (odd), which keeps two
// R = 128 gather4 stages in shared memory (MDN_CM_STAGE=0 at build: off).
#ifndef MDN_CM_STAGE
#define MDN_CM_STAGE 1
#endif
template <int W>
constexpr int CM_PART() {
  return ((W + 3) / 4) | 1;
}
// Their parts leave by TMA tensor stores (MDN_CM_TSTORE, as k_scan_ts; one
// buffer per warp, each part waits for the previous part's read). Same box,
// cls100 column-major rows/s (exact / avg): LDS + STG readback 5.01 / 3.88e9
// (0.698 of HBM), TMA stores 5.60 / 4.22e9 (0.779); MDN_CM_TSTORE=0 restores
// the readback.
#ifndef MDN_CM_TSTORE
#define MDN_CM_TSTORE 1
#endif
template <int W, bool ENC_ONLY, bool CMV>
constexpr int cm_ostg_bytes() {
  return MDN_CM_STAGE != 0 && CMV && !ENC_ONLY && W >= 8 && W - 3 * CM_PART<W>() > 0 ? 8 * 32 * 16 * CM_PART<W>() : 0;
}

// One part of a warp's 32 output rows (words [H0, H0 + NH)) through the
// warp's staging buffer (pitch P float4 per row, P odd).
template <int W, int H0, int NH, int P>
__device__ __forceinline__ void stage_part(float* __restrict__ stg, float* __restrict__ out, int64_t r0,
                                           int64_t N, int64_t ldo, const uint32_t (&ae)[W],
                                           const uint32_t (&ao)[W], float a, float b, int lane) {
  static_assert(NH <= P && (P & 1), "part must fit the odd row pitch");
#pragma unroll
  for (int j = 0; j < NH; ++j) {
    const int w = H0 + j;
    float4 f;
    f.x = __fmaf_rn(a, (float)(ae[w] & 0xFFFFu), b);
    f.y = __fmaf_rn(a, (float)(ao[w] & 0xFFFFu), b);
    f.z = __fmaf_rn(a, (float)(ae[w] >> 16), b);
    f.w = __fmaf_rn(a, (float)(ao[w] >> 16), b);
    reinterpret_cast<float4*>(stg)[lane * P + j] = f;
  }
  __syncwarp();
  // 32 x NH float4: item i = row i / NH, word i % NH; consecutive lanes write
  // consecutive 16-B pieces of a row
#pragma unroll
  for (int it = 0; it < NH; ++it) {
    const int i = it * 32 + lane;
    const int r = i / NH, j = i - r * NH;
    if (r0 + r < N)
      *reinterpret_cast<float4*>(out + (r0 + r) * ldo + 4 * (H0 + j)) = reinterpret_cast<const float4*>(stg)[r * P + j];
  }
  __syncwarp();
}

template <class TIn, int C, int W, int U, bool VEC, bool ENC_ONLY, int SUBF, bool PROBE = false,
          bool TILED = false>
__global__ void __launch_bounds__(Roles<(TILED ? 8 : W), ENC_ONLY, SUBF == CM>::THREADS, 1)
    k_amm_ws(const __grid_constant__ CUtensorMap tmap, const Params p,
             const __grid_constant__ CUtensorMap omap) {
  constexpr int G = C >= 8 ? 8 : C;      // codebooks per encoder unit (one code word)
  constexpr int NG = C / G;
  constexpr int CBW = NG;                // code words per row
  constexpr int WR = TILED ? 8 : W;       // table width the warp roles are sized for
  constexpr int EW = Roles<WR, ENC_ONLY, SUBF == CM>::E;
  constexpr int SWN = Roles<WR, ENC_ONLY, SUBF == CM>::S;
  constexpr int KR = Roles<WR, ENC_ONLY, SUBF == CM>::ROWS_PER_SCANNER;
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);
  uint64_t* empty = full + NS_MAX;
  uint64_t* cfull = empty + NS_MAX;
  uint64_t* cempty = cfull + NB;
  // Carve with integer offsets from `smem` so every pointer stays provably in
  // the shared window (plain LDS/STS, no generic loads).
  constexpr int OFF_THR = BAR_BYTES;
  constexpr int OFF_OFF = OFF_THR + thr_base(C) * 4;
  constexpr int OFF_BASE = OFF_OFF + off_base(C) * 4;
  constexpr int OFF_COLS = OFF_BASE + C * 4;
  constexpr int OFF_LUT = (OFF_COLS + (SUBF == CM ? 4 * C * 4 : 0) + 15) & ~15;
  constexpr int OFF_CODES = OFF_LUT + (ENC_ONLY || TILED ? 0 : C * W * 16 * 4);
  // column-major wide tables: the scanner warps' output staging (cm_ostg_bytes)
  // (128-B aligned for the TMA stores of MDN_CM_TSTORE; plan_cm budgets the slack)
  constexpr int OFF_OSTG = (OFF_CODES + (ENC_ONLY ? 0 : NB * BR * CBW * 4) + 127) & ~127;
  constexpr int OFF_STAGE = (OFF_OSTG + cm_ostg_bytes<W, ENC_ONLY, SUBF == CM>() + 127) & ~127;
  float* s_thr = reinterpret_cast<float*>(smem + OFF_THR);
  int* s_off = reinterpret_cast<int*>(smem + OFF_OFF);
  int* s_base = reinterpret_cast<int*>(smem + OFF_BASE);
  int* s_cols = reinterpret_cast<int*>(smem + OFF_COLS);
  uint32_t* s_codes = reinterpret_cast<uint32_t*>(smem + OFF_CODES);
  TIn* s_stage = reinterpret_cast<TIn*>(smem + OFF_STAGE);
  const int tid = threadIdx.x;
  const int pitch = p.SW + p.pad_e;                 // elements of TIn per shared row
  const int stage_e = p.nslab * p.slab_e;
  // tiled tables live after the stage ring (their size is a runtime value)
  uint32_t* s_lut = reinterpret_cast<uint32_t*>(
      smem + (TILED ? OFF_STAGE + (size_t)p.NS * stage_e * sizeof(TIn) : (size_t)OFF_LUT));

  // ---- setup: trees, split-dim offsets, tables, barriers ----
  for (int i = tid; i < 16 * C; i += blockDim.x) {
    const int si = thr_base(i / 16) + i % 16;
    if constexpr (sizeof(TIn) == 1)
      reinterpret_cast<int*>(s_thr)[si] = p.q[i];  // integer split values (App. B, R11)
    else
      s_thr[si] = p.thr[i];
  }
  for (int i = tid; i < 4 * C; i += blockDim.x) {
    const int d = p.dims[i];
    const int si = off_base(i / 4) + i % 4;
    if constexpr (SUBF == CM)
      s_off[si] = p.slot[d] * p.slab_e;              // slot-major stage: [slot][row]
    else
      s_off[si] = SUBF ? d - p.sub[i / 4] : (d / p.SW) * p.slab_e + (d % p.SW);
  }
  if constexpr (SUBF == CM)
    for (int k = tid; k < p.nslab; k += blockDim.x) s_cols[k] = p.cols[k < p.n_cols ? k : p.n_cols - 1];
  for (int c = tid; c < C; c += blockDim.x) {
    const int b = p.sub[c];
    s_base[c] = (b / p.SW) * p.slab_e + (b % p.SW);
  }
  if constexpr (TILED) {
    // [c][Wfull][16] -> [tile][c][W][16], words past the table width zero
    const int n = p.ntile * C * W * 16;
    for (int i = tid; i < n; i += blockDim.x) {
      const int k = i & 15, w = (i >> 4) % W, c = (i / (16 * W)) % C, t = i / (16 * W * C);
      const int gw = t * W + w;
      s_lut[i] = gw < p.Wfull ? p.lut[((size_t)c * p.Wfull + gw) * 16 + k] : 0u;
    }
  } else if constexpr (!ENC_ONLY) {
    const uint4* src = reinterpret_cast<const uint4*>(p.lut);
    uint4* dst = reinterpret_cast<uint4*>(s_lut);
    for (int i = tid; i < C * W * 4; i += blockDim.x) dst[i] = src[i];
  }
  if (tid == 0) {
    for (int s = 0; s < p.NS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], EW * 32);
    }
    for (int b = 0; b < NB; ++b) {
      mbar_init(&cfull[b], EW * 32);
      mbar_init(&cempty[b], SWN > 0 ? SWN * 32 : 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap)) : "memory");
  }
  __syncthreads();

  const int warp = tid >> 5, lane = tid & 31;
  const int stages_per_tile = BR / p.R;
  if (warp == 0) {
    // ---------------- TMA producer ----------------
    // Row-major A: lane 0 issues the nslab slab boxes of a stage. Column-major
    // A: |S| single-column boxes per stage, issued by all 32 lanes (one lane
    // issuing them serially caps the stage rate at ~140 cycles per box).
    constexpr bool ALL_LANES = SUBF == CM;
    if (ALL_LANES || lane == 0) {
      const uint32_t bytes = (uint32_t)(p.nslab * p.R * pitch * sizeof(TIn));
      const uint64_t pol = l2_policy(p.l2_hint);
      uint32_t q = 0;
      for (int64_t tile = blockIdx.x; tile < p.n_tiles; tile += gridDim.x) {
        for (int st = 0; st < stages_per_tile; ++st, ++q) {
          const int s = q % p.NS;
          mbar_wait(&empty[s], ((q / p.NS) & 1u) ^ 1u);
          const int64_t y = tile * BR + (int64_t)st * p.R;
          if (y >= p.N) {            // stage entirely past the last row: nothing to fetch
            if (lane == 0) mbar_arrive(&full[s]);
            continue;
          }
          if (lane == 0) mbar_arrive_tx(&full[s], bytes);
          TIn* dst = s_stage + (size_t)s * stage_e;
          if constexpr (SUBF == CM) {
            // column-major A: TMA gather4 -- one instruction fetches R rows of
            // 4 split columns (4 rows of At) into 4 consecutive slots; the
            // slot count is padded to a multiple of 4 with the last column.
            __syncwarp();            // expect_tx before any complete_tx of this phase
            for (int k = 4 * lane; k < p.nslab; k += 128)
              tma_gather4(dst + k * p.slab_e, &tmap, (int)y, s_cols[k], s_cols[k + 1], s_cols[k + 2],
                          s_cols[k + 3], &full[s]);
          } else {
            for (int k = 0; k < p.nslab; ++k)
              tma_load_2d(dst + k * p.slab_e, &tmap, k * p.SW, (int)y, &full[s], p.l2_hint, pol);
          }
        }
      }
    }
  } else if (warp <= EW) {
    // ---------------- encoders ----------------
    const int etid = tid - 32;
    uint32_t q = 0, z = 0;
    for (int64_t tile = blockIdx.x; tile < p.n_tiles; tile += gridDim.x, ++z) {
      const int b = z % NB;
      if constexpr (!ENC_ONLY) mbar_wait(&cempty[b], ((z / NB) & 1u) ^ 1u);
      for (int st = 0; st < stages_per_tile; ++st, ++q) {
        const int s = q % p.NS;
        mbar_wait(&full[s], (q / p.NS) & 1u);
        const TIn* stg = s_stage + (size_t)s * stage_e;
        for (int u = etid; u < (PROBE ? 0 : p.R * NG); u += EW * 32) {
          // Group-fastest units: the lanes of a warp cover NG codebook groups of
          // 32 / NG rows, so their split columns differ and the per-row reads
          // (pitch == 4 mod 32 words) spread over more banks than 32 rows of
          // one column would (4-way conflicts: +47% shared wavefronts on scale).
          // (Column-major stages are [slot][row]: there rows-fastest lanes read
          // 32 consecutive words of one slot, conflict-free, while groups-fastest
          // lanes would put 4 slots' rows on the same banks.)
          constexpr bool ROWS_FAST = SUBF == CM || NG == 1;
          const int g = ROWS_FAST ? u / p.R : u % NG, r = ROWS_FAST ? u % p.R : u / NG;
          const uint32_t word = encode_group<TIn, C, SUBF>(stg + r * pitch, s_off, s_base, s_thr, g * G);
          const int row_local = st * p.R + r;
          if constexpr (ENC_ONLY) {
            const int64_t row = tile * BR + row_local;
            if (row < p.N) {
              if constexpr (C >= 8)
                reinterpret_cast<uint32_t*>(p.codes + row * (C / 2))[g] = word;
              else if constexpr (C == 4)
                reinterpret_cast<uint16_t*>(p.codes + row * 2)[0] = (uint16_t)word;
              else
                p.codes[row] = (uint8_t)word;
            }
          } else {
            s_codes[(b * BR + row_local) * CBW + g] = word;
          }
        }
        mbar_arrive(&empty[s]);
      }
      if constexpr (!ENC_ONLY) mbar_arrive(&cfull[b]);
    }
  } else if constexpr (!ENC_ONLY) {
    // ---------------- scanners ----------------
    const int stid = tid - 32 * (1 + EW);
    uint32_t z = 0;
    for (int64_t tile = blockIdx.x; tile < p.n_tiles; tile += gridDim.x, ++z) {
      const int b = z % NB;
      mbar_wait(&cfull[b], (z / NB) & 1u);
#pragma unroll 1
      for (int k = 0; k < KR; ++k) {
        const int rl = stid + k * SWN * 32;
        const int64_t row = tile * BR + rl;
        const uint32_t* myc = s_codes + (b * BR + rl) * CBW;
        uint32_t ae[W], ao[W];
        if constexpr (TILED) {
#pragma unroll 1
          for (int t = 0; t < p.ntile; ++t) {
            scan_core<C, W, U, false, 0>(s_lut + (size_t)t * C * W * 16, [&](int g) { return myc[g]; }, ae, ao);
            if (row < p.N)
              store_row<W, false>(p.out + row * p.ldo + 4 * W * t, p.M - 4 * W * t, ae, ao, p.alpha_eff,
                                  p.beta32, p.pair);
          }
          if (k == KR - 1) mbar_arrive(&cempty[b]);
          continue;
        }
        if constexpr (PROBE) {
#pragma unroll
          for (int w = 0; w < W; ++w) ae[w] = 0u, ao[w] = 0u;
        } else {
          scan_core<C, W, U, false, (SUBF == CM && W >= 8) ? MDN_CM_MIX : 0>(s_lut, [&](int g) { return myc[g]; }, ae, ao);
        }
        if (k == KR - 1) mbar_arrive(&cempty[b]);
        if constexpr (VEC && cm_ostg_bytes<W, ENC_ONLY, SUBF == CM>() > 0) {
          // coalesced row stores in 4 parts of <= CM_PART words (see scan_stage)
          constexpr int Q = CM_PART<W>();
          float* stg = reinterpret_cast<float*>(smem + OFF_OSTG) + (size_t)(stid >> 5) * 32 * 4 * Q;
          const int64_t r0 = row - (stid & 31);
          const int lane = stid & 31;
          if constexpr (MDN_CM_TSTORE != 0) {
            // TMA tensor stores of the 4 parts (last part starts at W - Q)
            auto tpart = [&](int h0) {
              if (lane == 0) bulk_wait_read<0>();
              __syncwarp();
#pragma unroll
              for (int j = 0; j < Q; ++j) {
                const int w = h0 + j;
                float4 f;
                f.x = __fmaf_rn(p.alpha_eff, (float)(ae[w] & 0xFFFFu), p.beta32);
                f.y = __fmaf_rn(p.alpha_eff, (float)(ao[w] & 0xFFFFu), p.beta32);
                f.z = __fmaf_rn(p.alpha_eff, (float)(ae[w] >> 16), p.beta32);
                f.w = __fmaf_rn(p.alpha_eff, (float)(ao[w] >> 16), p.beta32);
                reinterpret_cast<float4*>(stg)[lane * Q + j] = f;
              }
              fence_proxy_async_smem();
              __syncwarp();
              if (lane == 0) {
                tma_store_2d(&omap, stg, 4 * h0, (int)r0);
                bulk_commit();
              }
            };
            tpart(0);
            tpart(Q);
            tpart(2 * Q);
            tpart(W - Q);
            continue;
          }
          stage_part<W, 0, Q, Q>(stg, p.out, r0, p.N, p.ldo, ae, ao, p.alpha_eff, p.beta32, lane);
          stage_part<W, Q, Q, Q>(stg, p.out, r0, p.N, p.ldo, ae, ao, p.alpha_eff, p.beta32, lane);
          stage_part<W, 2 * Q, Q, Q>(stg, p.out, r0, p.N, p.ldo, ae, ao, p.alpha_eff, p.beta32, lane);
          stage_part<W, 3 * Q, W - 3 * Q, Q>(stg, p.out, r0, p.N, p.ldo, ae, ao, p.alpha_eff, p.beta32, lane);
        } else if (row < p.N) {
          store_row<W, VEC>(p.out + row * p.ldo, p.M, ae, ao, p.alpha_eff, p.beta32, p.pair);
        }
      }
    }
    if constexpr (MDN_CM_TSTORE != 0 && VEC && cm_ostg_bytes<W, ENC_ONLY, SUBF == CM>() > 0)
      if ((stid & 31) == 0) bulk_wait_all();
  }
}

// ------------------------------------------------------------ scan kernel --

// Code-word software pipelining of mdn_scan (the next row's code words are
// loaded before this row is scanned): 0 = off, 1 = on with the codebook-group
// loop rolled (words picked by selects), 2 = on with it unrolled. Measured
// (same box, rows/s, mode 2 / 1 / 0): scale (C 32, W 4) 3.56 / 3.17 / 3.27e10,
// cls10_c32 3.75 / 3.28 / 3.49e10, cls10_c64 2.12 / 1.83 / 1.80e10; cls100
// (W 25) 1: 4.78 vs 0: 5.06e9 (unrolled: 3.95e9, register pressure); C = 16
// within 2%. MDN_SCAN_PF (build flag) forces one mode for A/B.
template <int C, int W>
constexpr int scan_pf_mode() {
#ifdef MDN_SCAN_PF
  return MDN_SCAN_PF;
#else
  return C >= 32 && W <= 4 ? 2 : 0;
#endif
}

// The row's packed code words (8 codes each); `vec`: rows 16-B (C = 32) or
// 8-B (C = 16) aligned, one vector load.
template <int C>
__device__ __forceinline__ void load_code_words(const uint8_t* __restrict__ codes, int64_t row,
                                                uint32_t (&cw)[C >= 8 ? C / 8 : 1], bool vec) {
  const uint8_t* cr = codes + row * ((C + 1) / 2);
  if constexpr (C == 32) {
    if (vec) {
      const uint4 v = __ldg(reinterpret_cast<const uint4*>(cr));
      cw[0] = v.x, cw[1] = v.y, cw[2] = v.z, cw[3] = v.w;
      return;
    }
  } else if constexpr (C == 16) {
    if (vec) {
      const uint2 v = __ldg(reinterpret_cast<const uint2*>(cr));
      cw[0] = v.x, cw[1] = v.y;
      return;
    }
  }
  if constexpr (C >= 8) {
#pragma unroll
    for (int g = 0; g < C / 8; ++g) cw[g] = __ldg(reinterpret_cast<const uint32_t*>(cr) + g);
  } else if constexpr (C == 4) {
    cw[0] = __ldg(reinterpret_cast<const uint16_t*>(cr));
  } else {
    cw[0] = __ldg(cr);
  }
}

// k_scan_fast's body; two entry points that differ only in their launch
// bounds. __launch_bounds__(256, 1) lets ptxas keep the wide tables' row in
// registers (cls100: 99 -> 127 registers, 2 blocks/SM) and schedule more
// lookups ahead; it pays for the wide tables and costs the narrow ones
// (same box, rows/s: cls100 5.05 -> 5.51e9, cls10_c64 2.15 -> 2.23e10, but
// scale 3.57 -> 3.24e10, image 2.46 -> 2.39e11, cls10_c16 and tiny flat).
template <int C, int W>
constexpr bool scan_lb1() {
  return W >= 8 || C >= 64;
}
template <int C, int W, int U, bool VEC, int MIX>
__device__ __forceinline__ void scan_fast_body(const uint32_t* __restrict__ lut_g,
                                               const uint8_t* __restrict__ codes, int64_t N, int M,
                                               int32_t* __restrict__ sums, float* __restrict__ out,
                                               int64_t ldo, float a, float b, int scale, bool pair,
                                               bool vec_codes) {
  extern __shared__ __align__(128) unsigned char smem[];
  uint32_t* s_lut = reinterpret_cast<uint32_t*>(smem);
  for (int i = threadIdx.x; i < C * W * 4; i += blockDim.x)
    reinterpret_cast<uint4*>(s_lut)[i] = reinterpret_cast<const uint4*>(lut_g)[i];
  __syncthreads();
  constexpr int NW = C >= 8 ? C / 8 : 1;
  constexpr int PF = scan_pf_mode<C, W>();
  if constexpr (scan_stage<W, VEC>()) {
    if (out) {
      // warp-uniform row loop: lanes past N scan code 0 and store nothing
      constexpr int H = (W + 1) / 2;
      const int lane = threadIdx.x & 31;
      float* stg = reinterpret_cast<float*>(smem + (size_t)C * W * 16 * 4) +
                   (size_t)(threadIdx.x >> 5) * scan_stage_floats<W>();
      const int64_t stride = (int64_t)gridDim.x * blockDim.x;
      for (int64_t r0 = (int64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31); r0 < N; r0 += stride) {
        const int64_t row = r0 + lane;
        uint32_t cw[NW];
        if (row < N) {
          load_code_words<C>(codes, row, cw, vec_codes);
        } else {
#pragma unroll
          for (int g = 0; g < NW; ++g) cw[g] = 0u;
        }
        uint32_t ae[W], ao[W];
        auto words = [&](int g) {
          uint32_t r = cw[0];
#pragma unroll
          for (int k = 1; k < NW; ++k) r = g == k ? cw[k] : r;
          return r;
        };
        scan_core<C, W, U, PF == 2, MIX>(s_lut, words, ae, ao);
        if (sums && row < N) store_sums<W>(sums + row * M, M, scale, ae, ao);
        stage_part<W, 0, H, scan_stage_pitch<W>()>(stg, out, r0, N, ldo, ae, ao, a, b, lane);
        stage_part<W, H, W - H, scan_stage_pitch<W>()>(stg, out, r0, N, ldo, ae, ao, a, b, lane);
      }
      return;
    }
  }
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t row = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  uint32_t cw[NW];
  if (PF && row < N) load_code_words<C>(codes, row, cw, vec_codes);
  for (; row < N; row += stride) {
    uint32_t nx[NW];
    if constexpr (PF != 0) {
      if (row + stride < N) load_code_words<C>(codes, row + stride, nx, vec_codes);
    } else {
      load_code_words<C>(codes, row, cw, vec_codes);
    }
    uint32_t ae[W], ao[W];
    auto words = [&](int g) {
      uint32_t r = cw[0];
#pragma unroll
      for (int k = 1; k < NW; ++k) r = g == k ? cw[k] : r;   // register select, no local memory
      return r;
    };
    scan_core<C, W, U, PF == 2, MIX>(s_lut, words, ae, ao);
    if (sums) store_sums<W>(sums + row * M, M, scale, ae, ao);
    if (out) store_row<W, VEC>(out + row * ldo, M, ae, ao, a, b, pair);
    if constexpr (PF != 0) {
#pragma unroll
      for (int g = 0; g < NW; ++g) cw[g] = nx[g];
    }
  }
}

#define MDN_SCAN_ARGS                                                                         \
  const uint32_t *__restrict__ lut_g, const uint8_t *__restrict__ codes, int64_t N, int M,     \
      int32_t *__restrict__ sums, float *__restrict__ out, int64_t ldo, float a, float b,       \
      int scale, bool pair, bool vec_codes
template <int C, int W, int U, bool VEC, int MIX>
__global__ void __launch_bounds__(256) k_scan_fast(MDN_SCAN_ARGS) {
  scan_fast_body<C, W, U, VEC, MIX>(lut_g, codes, N, M, sums, out, ldo, a, b, scale, pair, vec_codes);
}
#ifndef MDN_SCAN_LB1_TPB
#define MDN_SCAN_LB1_TPB 512   // threads per block of the wide-table scan (one block per SM)
#endif
template <int C, int W, int U, bool VEC, int MIX>
__global__ void __launch_bounds__(MDN_SCAN_LB1_TPB, 1) k_scan_fast_lb1(MDN_SCAN_ARGS) {
  scan_fast_body<C, W, U, VEC, MIX>(lut_g, codes, N, M, sums, out, ldo, a, b, scale, pair, vec_codes);
}
#undef MDN_SCAN_ARGS

// Wide-table mdn_scan with TMA tensor stores of the staged rows
// (MDN_SCAN_TSTORE). The staging buffer of a warp is already a dense box
// (32 rows x P float4, P odd), so instead of reading it back (LDS) and
// storing it from the registers (STG through the L1 path the lookups use),
// one lane hands the box to the TMA unit: per 32 rows and part, one
// instruction instead of P LDS.128 + P STG.128 per lane, and the rows past N
// are clipped by the tensor map. Part 1 starts at word W - P (it overlaps
// part 0 by 2P - W words, written twice with the same values). NBUF buffers
// per warp: with 2 the second part never waits for the first part's read.
// Same box, cls100 rows/s (exact / avg): LDS + STG readback 6.89 / 4.87e9,
// TMA stores with 1 buffer (512 threads) 8.10 / 5.66e9, with 2 buffers (384
// threads) 8.09 / 5.63e9; kept: 1 buffer. MDN_SCAN_TSTORE=0 (build flag)
// restores the readback.
#ifndef MDN_SCAN_TSTORE
#define MDN_SCAN_TSTORE 1
#endif
#ifndef MDN_SCAN_TS_NBUF
#define MDN_SCAN_TS_NBUF 1
#endif
#ifndef MDN_SCAN_TS_TPB
#define MDN_SCAN_TS_TPB (MDN_SCAN_TS_NBUF == 1 ? 512 : 384)
#endif
template <int C, int W, int U, int MIX>
__global__ void __launch_bounds__(MDN_SCAN_TS_TPB, 1)
    k_scan_ts(const __grid_constant__ CUtensorMap om, const uint32_t* __restrict__ lut_g,
              const uint8_t* __restrict__ codes, int64_t N, int M, int32_t* __restrict__ sums,
              float a, float b, int scale, bool vec_codes) {
  extern __shared__ __align__(128) unsigned char smem[];
  uint32_t* s_lut = reinterpret_cast<uint32_t*>(smem);
  for (int i = threadIdx.x; i < C * W * 4; i += blockDim.x)
    reinterpret_cast<uint4*>(s_lut)[i] = reinterpret_cast<const uint4*>(lut_g)[i];
  __syncthreads();
  constexpr int NW = C >= 8 ? C / 8 : 1;
  constexpr int PF = scan_pf_mode<C, W>();
  constexpr int P = scan_stage_pitch<W>();
  constexpr int H1 = W - P;
  static_assert(H1 > 0 && H1 <= P, "two parts of P words cover the row");
  constexpr int NBUF = MDN_SCAN_TS_NBUF;
  const int lane = threadIdx.x & 31;
  float* stg0 = reinterpret_cast<float*>(smem + (size_t)C * W * 16 * 4) +
                (size_t)(threadIdx.x >> 5) * NBUF * scan_stage_floats<W>();
  float* stg1 = stg0 + (NBUF - 1) * scan_stage_floats<W>();
  auto part = [&](float* stg, int h0, const uint32_t(&ae)[W], const uint32_t(&ao)[W]) {
#pragma unroll
    for (int j = 0; j < P; ++j) {
      const int w = h0 + j;
      float4 f;
      f.x = __fmaf_rn(a, (float)(ae[w] & 0xFFFFu), b);
      f.y = __fmaf_rn(a, (float)(ao[w] & 0xFFFFu), b);
      f.z = __fmaf_rn(a, (float)(ae[w] >> 16), b);
      f.w = __fmaf_rn(a, (float)(ao[w] >> 16), b);
      reinterpret_cast<float4*>(stg)[lane * P + j] = f;
    }
  };
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t r0 = (int64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31); r0 < N; r0 += stride) {
    const int64_t row = r0 + lane;
    uint32_t cw[NW];
    if (row < N) {
      load_code_words<C>(codes, row, cw, vec_codes);
    } else {
#pragma unroll
      for (int g = 0; g < NW; ++g) cw[g] = 0u;
    }
    uint32_t ae[W], ao[W];
    auto words = [&](int g) {
      uint32_t r = cw[0];
#pragma unroll
      for (int k = 1; k < NW; ++k) r = g == k ? cw[k] : r;
      return r;
    };
    scan_core<C, W, U, PF == 2, MIX>(s_lut, words, ae, ao);
    if (sums && row < N) store_sums<W>(sums + row * M, M, scale, ae, ao);
    // part 0: its buffer's previous store must have been read (NBUF = 2: the
    // one group allowed to be pending is the other buffer's)
    if (lane == 0) bulk_wait_read<NBUF - 1>();
    __syncwarp();
    part(stg0, 0, ae, ao);
    fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0) {
      tma_store_2d(&om, stg0, 0, (int)r0);
      bulk_commit();
      bulk_wait_read<NBUF - 1>();
    }
    __syncwarp();
    part(stg1, H1, ae, ao);
    fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0) {
      tma_store_2d(&om, stg1, 4 * H1, (int)r0);
      bulk_commit();
    }
  }
  if (lane == 0) bulk_wait_all();
}

// mdn_scan for table widths without a compiled kernel: the tables cut into
// ntile column tiles of WT words ([tile][c][WT][16] in shared memory, words
// past the width zero); a thread's row walks the tiles with its code words
// in registers.
template <int C, int WT, int U>
__global__ void __launch_bounds__(256) k_scan_tiled(const uint32_t* __restrict__ lut_g, int Wfull,
                                                    int ntile, const uint8_t* __restrict__ codes,
                                                    int64_t N, int M, int32_t* __restrict__ sums,
                                                    float* __restrict__ out, int64_t ldo, float a,
                                                    float b, int scale, bool pair, bool vec_codes) {
  extern __shared__ __align__(128) unsigned char smem[];
  uint32_t* s_lut = reinterpret_cast<uint32_t*>(smem);
  const int n = ntile * C * WT * 16;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const int k = i & 15, w = (i >> 4) % WT, c = (i / (16 * WT)) % C, t = i / (16 * WT * C);
    const int gw = t * WT + w;
    s_lut[i] = gw < Wfull ? lut_g[((size_t)c * Wfull + gw) * 16 + k] : 0u;
  }
  __syncthreads();
  constexpr int NW = C >= 8 ? C / 8 : 1;
  for (int64_t row = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; row < N;
       row += (int64_t)gridDim.x * blockDim.x) {
    uint32_t cw[NW];
    load_code_words<C>(codes, row, cw, vec_codes);
#pragma unroll 1
    for (int t = 0; t < ntile; ++t) {
      uint32_t ae[WT], ao[WT];
      scan_core<C, WT, U, false, 0>(
          s_lut + (size_t)t * C * WT * 16,
          [&](int g) {
            uint32_t r = cw[0];
#pragma unroll
            for (int q = 1; q < NW; ++q) r = g == q ? cw[q] : r;
            return r;
          },
          ae, ao);
      const int m0 = 4 * WT * t;
      if (sums) store_sums<WT>(sums + row * M + m0, M - m0, scale, ae, ao);
      if (out) store_row<WT, false>(out + row * ldo + m0, M - m0, ae, ao, a, b, pair);
    }
  }
}

// ------------------------------------------------------------ host side --

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(ptr);
  });
  return fn;
}

cudaError_t ensure_smem(const void* kernel, size_t smem) {
  int dev = 0;
  cudaGetDevice(&dev);
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, size_t> done;
  {
    std::lock_guard<std::mutex> g(mu);
    auto it = done.find({kernel, dev});
    if (it != done.end() && it->second >= smem) return cudaSuccess;
  }
  cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e == cudaSuccess) {
    std::lock_guard<std::mutex> g(mu);
    size_t& v = done[{kernel, dev}];
    if (smem > v) v = smem;
  }
  return e;
}

DevInfo dev_info() {
  static DevInfo cache[16];
  static bool have[16] = {};
  static std::mutex mu;
  int d = 0;
  cudaGetDevice(&d);
  std::lock_guard<std::mutex> g(mu);
  if (d < 16 && have[d]) return cache[d];
  DevInfo di;
  cudaDeviceGetAttribute(&di.sms, cudaDevAttrMultiProcessorCount, d);
  cudaDeviceGetAttribute(&di.smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, d);
  if (d < 16) {
    cache[d] = di;
    have[d] = true;
  }
  return di;
}

int env_int(const char* name, int dflt);

struct Geometry {
  bool ok = false;
  int SW, nslab, R, NS, slab_e, pad_e;
  size_t smem;
};

// Slab width SW dividing D such that a box of SW + pad_e elements (pad_e =
// 16 bytes of padding) fits the 256-element TMA box limit and is a multiple of
// 16 bytes; then the largest rows-per-stage R (dividing the 256-row tile) that
// leaves room for >= 4 stages (>= 2 at worst). es = input element size.
Geometry plan(int C, int W, int D, bool enc_only, int es, int ntile) {
  Geometry g;
  const int pad_e = 16 / es;
  if (D % pad_e != 0) return g;
  int nslab = 0;
  for (int n = 1; n <= 64; ++n)
    if (D % n == 0 && (D / n) % pad_e == 0 && D / n + pad_e <= 256) {
      nslab = n;
      break;
    }
  if (!nslab) return g;
  g.nslab = nslab;
  g.SW = D / nslab;
  g.pad_e = pad_e;
  const int CBW = C >= 8 ? C / 8 : 1;
  size_t fixed = BAR_BYTES + thr_base(C) * 4 + off_base(C) * 4 + C * 4 + 16;
  if (!enc_only) fixed += (size_t)C * W * 16 * 4 * ntile + (size_t)NB * BR * CBW * 4;
  fixed = (fixed + 127) & ~size_t(127);
  const size_t budget = (size_t)dev_info().smem_optin;
  const int align_e = 128 / es;
  static const int rmax = env_int("MDN_WS_RMAX", 256);   // A/B knob: cap on rows per stage
  static const int mns = env_int("MDN_WS_MINNS", 3);     // fewest stages for the largest R (A/B knob)
  for (int min_ns : {mns, 2}) {
    for (int R : {256, 128, 64, 32, 16, 8}) {
      if (R > rmax) continue;
      int slab_e = ((R * (g.SW + pad_e)) + align_e - 1) / align_e * align_e;
      size_t stage = (size_t)nslab * slab_e * es;
      if (fixed + stage * min_ns > budget) continue;
      int NS = (int)((budget - fixed) / stage);
      if (NS > NS_MAX) NS = NS_MAX;
      g.R = R;
      g.NS = NS;
      g.slab_e = slab_e;
      g.smem = fixed + stage * NS;
      g.ok = true;
      return g;
    }
  }
  return g;
}

// Tuning knobs for experiments (read once): MDN_TMA_L2PROMO in {0,64,128,256}
// (default 256) and MDN_TMA_HINT in {0..3} (default 0). Not part of the ABI.
int env_int(const char* name, int dflt) {
  const char* v = getenv(name);
  return v ? atoi(v) : dflt;
}
int knob_promo() {
  static int v = env_int("MDN_TMA_L2PROMO", 256);
  return v;
}
// MDN_NO_RT=1 disables the register-tree kernel (A/B comparisons only).
bool rt_enabled() {
  static int v = env_int("MDN_NO_RT", 0);
  return v == 0;
}
// MDN_NO_BQ=1 disables the byte-threshold encoder of the 8-bit path (A/B only).
bool knob_bq() {
  static int v = env_int("MDN_NO_BQ", 0);
  return v == 0;
}
int knob_hint() {
  static int v = env_int("MDN_TMA_HINT", 0);
  return v;
}

bool make_tmap(CUtensorMap* m, const void* A, int64_t N, int64_t lda, int D, int SW, int R,
               int es) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return false;
  const int pr = knob_promo();
  const CUtensorMapL2promotion promo =
      pr == 0 ? CU_TENSOR_MAP_L2_PROMOTION_NONE
              : pr == 64 ? CU_TENSOR_MAP_L2_PROMOTION_L2_64B
                         : pr == 128 ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B
                                     : CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
  cuuint64_t dims[2] = {(cuuint64_t)D, (cuuint64_t)N};
  cuuint64_t strides[1] = {(cuuint64_t)lda * es};
  cuuint32_t box[2] = {(cuuint32_t)(SW + 16 / es), (cuuint32_t)R};
  cuuint32_t estr[2] = {1, 1};
  return fn(m, es == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_UINT8, 2,
            const_cast<void*>(A), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, promo,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

bool make_tmap_out(CUtensorMap* m, float* out, int64_t N, int M, int64_t ldo, int bw, int bh) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {(cuuint64_t)M, (cuuint64_t)N};
  cuuint64_t strides[1] = {(cuuint64_t)ldo * 4};
  cuuint32_t box[2] = {(cuuint32_t)bw, (cuuint32_t)bh};
  cuuint32_t estr[2] = {1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, out, dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
            CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <class TIn, int C, int W, int U, bool VEC, bool ENC, int SUBF, bool PROBE = false,
          bool TILED = false>
cudaError_t launch_ws_sf(const CUtensorMap& tm, const Params& p, size_t smem, cudaStream_t s,
                         const CUtensorMap* om = nullptr) {
  auto k = k_amm_ws<TIn, C, W, U, VEC, ENC, SUBF, PROBE, TILED>;
  cudaError_t attr_err = ensure_smem(reinterpret_cast<const void*>(k), smem);
  if (attr_err != cudaSuccess) return attr_err;
  int64_t grid = p.n_tiles < dev_info().sms ? p.n_tiles : dev_info().sms;
  k<<<(unsigned)grid, Roles<(TILED ? 8 : W), ENC, SUBF == CM>::THREADS, smem, s>>>(tm, p, om ? *om : tm);
  return cudaGetLastError();
}

// Subspace-vector encoders are compiled for the small-D tables (C <= 8).
template <class TIn, int C, int W, int U, bool VEC, bool ENC>
cudaError_t launch_ws_t(const CUtensorMap& tm, const Params& p, int subf, size_t smem,
                        cudaStream_t s) {
  if constexpr (C <= 8) {
    if (subf == 1) return launch_ws_sf<TIn, C, W, U, VEC, ENC, 1>(tm, p, smem, s);
    if (subf == 2) return launch_ws_sf<TIn, C, W, U, VEC, ENC, 2>(tm, p, smem, s);
  }
  return launch_ws_sf<TIn, C, W, U, VEC, ENC, 0>(tm, p, smem, s);
}

// Exact-mode pipe mix of the standalone scan (mdn_scan.cuh). With the mask
// form the mix paid (cls100 +7%, scale +8%, cls10_c64 +8%); with the raw-word
// form (one PRMT per word) ALU-only is as fast or faster (same box, rows/s,
// ALU-only vs mix: cls100 5.96 vs 5.91e9, scale 3.89 vs 3.89e10, cls10_c64
// 2.61 vs 2.43e10, cls10_c16 6.02 vs 5.96e10), so the default is ALU-only.
// MDN_SCAN_MIX=3 forces the mix (every MDN_SCAN_MIXK-th word on the ALU).
#ifndef MDN_SCAN_MIXK
#define MDN_SCAN_MIXK 3   // the mixed form: every MIXK-th word's adds on the ALU pipe
#endif
static int scan_mix(int C) {
  static const int v = env_int("MDN_SCAN_MIX", -1);
  return v < 0 ? 0 : v;
}

template <int C, int W, int U, bool VEC>
cudaError_t launch_scan_t(const LutsDev& l, const uint8_t* codes, int64_t N, int32_t* sums,
                          float* out, int64_t ldo, cudaStream_t s) {
  using KFn = void (*)(const uint32_t*, const uint8_t*, int64_t, int, int32_t*, float*, int64_t, float,
                      float, int, bool, bool);
  if constexpr (MDN_SCAN_TSTORE != 0 && scan_stage<W, VEC>()) {
    constexpr int P = scan_stage_pitch<W>();
    CUtensorMap om;
    if (out && N > 0 && scan_mix(C) == 0 && make_tmap_out(&om, out, N, l.M, ldo, 4 * P, 32)) {
      auto kt = k_scan_ts<C, W, U, 0>;
      constexpr int tpb = MDN_SCAN_TS_TPB;
      const size_t smem =
          (size_t)C * W * 16 * 4 + (size_t)(tpb / 32) * MDN_SCAN_TS_NBUF * scan_stage_floats<W>() * 4;
      cudaError_t e = ensure_smem(reinterpret_cast<const void*>(kt), smem);
      if (e != cudaSuccess) return e;
      int per_sm = 0;
      e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kt, tpb, smem);
      if (e != cudaSuccess) return e;
      if (per_sm < 1) per_sm = 1;
      int64_t blocks = (N + tpb - 1) / tpb;
      const int64_t cap = (int64_t)dev_info().sms * per_sm;
      if (blocks > cap) blocks = cap;
      const bool vec_codes = (reinterpret_cast<uintptr_t>(codes) & (C == 32 ? 15u : 7u)) == 0;
      kt<<<(unsigned)blocks, tpb, smem, s>>>(om, l.words, codes, N, l.M, sums, l.alpha_eff, l.beta32,
                                             l.U == 0 ? 1 : l.U, vec_codes);
      return cudaGetLastError();
    }
  }
  KFn k;
  if constexpr (scan_lb1<C, W>()) {
    k = k_scan_fast_lb1<C, W, U, VEC, 0>;
    if constexpr (U == 0)
      if (scan_mix(C) == 3) k = k_scan_fast_lb1<C, W, U, VEC, MDN_SCAN_MIXK>;
  } else {
    k = k_scan_fast<C, W, U, VEC, 0>;
    if constexpr (U == 0)
      if (scan_mix(C) == 3) k = k_scan_fast<C, W, U, VEC, MDN_SCAN_MIXK>;
  }
  const int tpb = scan_lb1<C, W>() ? MDN_SCAN_LB1_TPB : 256;
  size_t smem = (size_t)C * W * 16 * 4;
  if constexpr (scan_stage<W, VEC>()) smem += (size_t)(tpb / 32) * scan_stage_floats<W>() * 4;
  cudaError_t attr_err = ensure_smem(reinterpret_cast<const void*>(k), smem);
  if (attr_err != cudaSuccess) return attr_err;
  // One wave of resident blocks (grid-stride): a grid above the occupancy
  // limit leaves a tail wave running at a fraction of the SM (cls100: 80
  // registers -> 3 blocks/SM, so the old 4/SM grid ran its last quarter alone).
  int per_sm = 0;
  cudaError_t oe = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, tpb, smem);
  if (oe != cudaSuccess) return oe;
  static const int bps = env_int("MDN_SCAN_BPS", 0);   // tuning knob: cap blocks/SM
  if (bps > 0 && per_sm > bps) per_sm = bps;
  if (per_sm < 1) per_sm = 1;
  int64_t blocks = (N + tpb - 1) / tpb;
  const int64_t cap = (int64_t)dev_info().sms * per_sm;
  if (blocks > cap) blocks = cap;
  const bool pair = l.M % 2 == 0 && ldo % 2 == 0 && (reinterpret_cast<uintptr_t>(out) & 7u) == 0;
  const bool vec_codes = (reinterpret_cast<uintptr_t>(codes) & (C == 32 ? 15u : 7u)) == 0;
  k<<<(unsigned)blocks, tpb, smem, s>>>(l.words, codes, N, l.M, sums, out, ldo, l.alpha_eff,
                                        l.beta32, l.U == 0 ? 1 : l.U, pair, vec_codes);
  return cudaGetLastError();
}

// (C, W, U) combinations with compiled fast kernels: every BASELINE config in
// both modes (U = C for C < 16, else 16), plus common neighbours.
#define MDN_FAST_COMBOS(X) \
  X(4, 1, 0) X(4, 1, 4) X(8, 1, 0) X(8, 1, 8) X(8, 2, 0) X(8, 2, 8)                    \
  X(16, 1, 0) X(16, 1, 16) X(16, 3, 0) X(16, 3, 16) X(16, 4, 0) X(16, 4, 16)            \
  X(32, 1, 0) X(32, 1, 16) X(32, 3, 0) X(32, 3, 16) X(32, 4, 0) X(32, 4, 16)            \
  X(32, 25, 0) X(32, 25, 16) X(64, 3, 0) X(64, 3, 16) X(64, 4, 0) X(64, 4, 16)

bool has_combo(int C, int W, int U) {
#define X(c, w, u) \
  if (C == c && W == w && U == u) return true;
  MDN_FAST_COMBOS(X)
#undef X
  return false;
}

bool has_encoder(int C) { return C == 4 || C == 8 || C == 16 || C == 32 || C == 64; }

}  // namespace fast

using namespace fast;

static bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

// es = input element size (4: fp32 A, 1: uint8 A).
static int subf_for(const TreesDev& t, const Geometry& g, int es) {
  // Subspace loads stay inside one slab. (Allowing them across the two
  // 128-column slabs of the scale config -- 32 uniform 8-column subspaces --
  // cost 21%: 4.62 vs 5.86e9 rows/s, same box; the groups' 16-B loads land
  // on the same banks.)
  if (g.nslab != 1) return 0;
  return es == 4 ? t.subf : t.subf_u8;
}

static bool amm_fast_ok(const TreesDev& t, const LutsDev& l, const void* A, int64_t lda, int es,
                        Geometry* geo) {
  if (!has_combo(t.C, l.W, l.U)) return false;
  if (!aligned16(A) || (lda * es) % 16 != 0) return false;
  if (!encode_fn()) return false;
  *geo = plan(t.C, l.W, t.D, false, es, 1);
  return geo->ok;
}

// Table widths without a compiled kernel: the tile width with a compiled
// (C, WT, U) kernel (4 words = 16 columns for C >= 16) and the tile count;
// false if no tiled kernel serves these shapes (the generic kernel then runs).
static bool tiled_plan(const TreesDev& t, const LutsDev& l, const void* A, int64_t lda, int es,
                       int* WT, int* ntile, Geometry* geo) {
  if (has_combo(t.C, l.W, l.U) || es != 4) return false;
  const int wt = t.C >= 16 ? 4 : (t.C == 8 ? 2 : (t.C == 4 ? 1 : 0));
  if (!wt || !has_combo(t.C, wt, l.U) || l.W <= wt) return false;
  if (!aligned16(A) || (lda * es) % 16 != 0 || !encode_fn()) return false;
  *WT = wt;
  *ntile = (l.W + wt - 1) / wt;
  *geo = plan(t.C, wt, t.D, false, es, *ntile);
  return geo->ok;
}

const char* amm_variant_name(const TreesDev& t, const LutsDev& l, const float* A, int64_t lda,
                             const float* out, int64_t ldo) {
  Geometry g;
  if (rt_enabled() && amm_rt_applies(t, l, 4))
    return (l.M == 2 || l.M == 4) && ldo % l.M == 0 ? "rt_vec" : "rt";
  if (!amm_fast_ok(t, l, A, lda, 4, &g)) {
    int wt, nt;
    return tiled_plan(t, l, A, lda, 4, &wt, &nt, &g) ? "ws_tma_tiled" : "generic";
  }
  const bool vec = l.M % 4 == 0 && ldo % 4 == 0 && aligned16(out);
  static const char* names[2][3] = {{"ws_tma", "ws_tma_sub4", "ws_tma_sub8"},
                                    {"ws_tma_vec", "ws_tma_vec_sub4", "ws_tma_vec_sub8"}};
  return names[vec][subf_for(t, g, 4)];
}

cudaError_t launch_encode_generic(const TreesDev&, const void*, int, int64_t, int64_t, uint8_t*,
                                  cudaStream_t);
cudaError_t launch_scan_generic(const LutsDev&, const uint8_t*, int64_t, int32_t*, float*, int64_t,
                                cudaStream_t);
cudaError_t launch_amm_generic(const TreesDev&, const LutsDev&, const void*, int, int64_t, int64_t,
                               float*, int64_t, cudaStream_t);

static Params base_params(const TreesDev& t, const Geometry& g, int64_t N) {
  Params p{};
  p.N = N;
  p.n_tiles = (N + BR - 1) / BR;
  p.D = t.D;
  p.SW = g.SW;
  p.nslab = g.nslab;
  p.R = g.R;
  p.NS = g.NS;
  p.slab_e = g.slab_e;
  p.pad_e = g.pad_e;
  p.dims = t.dims;
  p.sub = t.sub;
  p.l2_hint = knob_hint();
  p.thr = t.thr;
  p.q = t.q;
  return p;
}

// Tiled fused kernel for table widths without a compiled kernel (fp32 rows).
static cudaError_t amm_tiled(const TreesDev& t, const LutsDev& l, const float* A, int64_t N,
                             int64_t lda, float* out, int64_t ldo, cudaStream_t s, bool* done) {
  *done = false;
  Geometry g;
  int wt = 0, nt = 0;
  if (!tiled_plan(t, l, A, lda, 4, &wt, &nt, &g)) return cudaSuccess;
  CUtensorMap tm;
  if (!make_tmap(&tm, A, N, lda, t.D, g.SW, g.R, 4)) return cudaSuccess;
  Params p = base_params(t, g, N);
  const int sf = subf_for(t, g, 4);
  p.ldo = ldo;
  p.M = l.M;
  p.pair = l.M % 2 == 0 && ldo % 2 == 0 && (reinterpret_cast<uintptr_t>(out) & 7u) == 0;
  p.alpha_eff = l.alpha_eff;
  p.beta32 = l.beta32;
  p.lut = l.words;
  p.out = out;
  p.ntile = nt;
  p.Wfull = l.W;
  *done = true;
#define TL(c, w, u, sfv)                                                                  \
  if (t.C == c && wt == w && l.U == u && sf == sfv)                                       \
    return launch_ws_sf<float, c, w, u, false, false, sfv, false, true>(tm, p, g.smem, s);
  TL(4, 1, 0, 0) TL(4, 1, 4, 0) TL(4, 1, 0, 1) TL(4, 1, 4, 1) TL(4, 1, 0, 2) TL(4, 1, 4, 2)
  TL(8, 2, 0, 0) TL(8, 2, 8, 0) TL(8, 2, 0, 1) TL(8, 2, 8, 1) TL(8, 2, 0, 2) TL(8, 2, 8, 2)
#undef TL
  // C >= 16: the per-split-dim encoder (SUBF 0) serves every subspace layout
#define TL(c, w, u)                                                                      \
  if (t.C == c && wt == w && l.U == u)                                                   \
    return launch_ws_sf<float, c, w, u, false, false, 0, false, true>(tm, p, g.smem, s);
  TL(16, 4, 0) TL(16, 4, 16) TL(32, 4, 0) TL(32, 4, 16) TL(64, 4, 0) TL(64, 4, 16)
#undef TL
  *done = false;
  return cudaSuccess;
}

template <class TIn>
static cudaError_t amm_fast(const TreesDev& t, const LutsDev& l, const TIn* A, int64_t N,
                            int64_t lda, float* out, int64_t ldo, cudaStream_t s, bool* done) {
  constexpr int es = sizeof(TIn);
  *done = false;
  Geometry g;
  if (N > (int64_t)0x7FFFFF00) return cudaSuccess;
  if (!amm_fast_ok(t, l, A, lda, es, &g)) {
    if constexpr (es == 4) return amm_tiled(t, l, A, N, lda, out, ldo, s, done);
    return cudaSuccess;
  }
  CUtensorMap tm;
  if (!make_tmap(&tm, A, N, lda, t.D, g.SW, g.R, es)) return cudaSuccess;
  Params p = base_params(t, g, N);
  const int sf = subf_for(t, g, es);
  p.ldo = ldo;
  p.M = l.M;
  p.pair = l.M % 2 == 0 && ldo % 2 == 0 && (reinterpret_cast<uintptr_t>(out) & 7u) == 0;
  p.alpha_eff = l.alpha_eff;
  p.beta32 = l.beta32;
  p.lut = l.words;
  p.out = out;
  const bool vec = l.M % 4 == 0 && ldo % 4 == 0 && aligned16(out);
  *done = true;
#define X(c, w, u)                                                                  \
  if (t.C == c && l.W == w && l.U == u)                                             \
    return vec ? launch_ws_t<TIn, c, w, u, true, false>(tm, p, sf, g.smem, s)       \
               : launch_ws_t<TIn, c, w, u, false, false>(tm, p, sf, g.smem, s);
  MDN_FAST_COMBOS(X)
#undef X
  *done = false;
  return cudaSuccess;
}

// mdn_amm_probe: amm_fast's geometry and launch with PROBE (row-major fp32 A).
static cudaError_t amm_probe_fast(const TreesDev& t, const LutsDev& l, const float* A, int64_t N,
                                  int64_t lda, float* out, int64_t ldo, cudaStream_t s, bool* done) {
  *done = false;
  Geometry g;
  if (N > (int64_t)0x7FFFFF00 || !amm_fast_ok(t, l, A, lda, 4, &g)) return cudaSuccess;
  CUtensorMap tm;
  if (!make_tmap(&tm, A, N, lda, t.D, g.SW, g.R, 4)) return cudaSuccess;
  Params p = base_params(t, g, N);
  p.ldo = ldo;
  p.M = l.M;
  p.pair = l.M % 2 == 0 && ldo % 2 == 0 && (reinterpret_cast<uintptr_t>(out) & 7u) == 0;
  p.alpha_eff = l.alpha_eff;
  p.beta32 = l.beta32;
  p.lut = l.words;
  p.out = out;
  const bool vec = l.M % 4 == 0 && ldo % 4 == 0 && aligned16(out);
  *done = true;
#define X(c, w, u)                                                                             \
  if (u == 0 && t.C == c && l.W == w)                                                          \
    return vec ? launch_ws_sf<float, c, w, 0, true, false, 0, true>(tm, p, g.smem, s)          \
               : launch_ws_sf<float, c, w, 0, false, false, 0, true>(tm, p, g.smem, s);
  MDN_FAST_COMBOS(X)
#undef X
  *done = false;
  return cudaSuccess;
}

cudaError_t launch_amm_probe(const TreesDev& t, const LutsDev& l, const float* A, int64_t N,
                             int64_t lda, float* out, int64_t ldo, cudaStream_t s, bool* done) {
  *done = false;
  if (rt_enabled() && amm_rt_applies(t, l, 4)) return cudaSuccess;   // mdn_amm runs k_amm_rt here
  return amm_probe_fast(t, l, A, N, lda, out, ldo, s, done);
}

template <class TIn>
static cudaError_t encode_fast(const TreesDev& t, const TIn* A, int64_t N, int64_t lda,
                               uint8_t* codes, cudaStream_t s, bool* done) {
  constexpr int es = sizeof(TIn);
  *done = false;
  if (N > (int64_t)0x7FFFFF00 || !has_encoder(t.C) || !aligned16(A) || (lda * es) % 16 != 0 ||
      !encode_fn())
    return cudaSuccess;
  if (t.C >= 8 && (reinterpret_cast<uintptr_t>(codes) & 3u)) return cudaSuccess;
  if (t.C == 4 && (reinterpret_cast<uintptr_t>(codes) & 1u)) return cudaSuccess;
  Geometry g = plan(t.C, 1, t.D, true, es, 1);
  if (!g.ok) return cudaSuccess;
  CUtensorMap tm;
  if (!make_tmap(&tm, A, N, lda, t.D, g.SW, g.R, es)) return cudaSuccess;
  Params p = base_params(t, g, N);
  const int sf = subf_for(t, g, es);
  p.codes = codes;
  *done = true;
  switch (t.C) {
    case 4: return launch_ws_t<TIn, 4, 1, 0, false, true>(tm, p, sf, g.smem, s);
    case 8: return launch_ws_t<TIn, 8, 1, 0, false, true>(tm, p, sf, g.smem, s);
    case 16: return launch_ws_t<TIn, 16, 1, 0, false, true>(tm, p, sf, g.smem, s);
    case 32: return launch_ws_t<TIn, 32, 1, 0, false, true>(tm, p, sf, g.smem, s);
    case 64: return launch_ws_t<TIn, 64, 1, 0, false, true>(tm, p, sf, g.smem, s);
  }
  *done = false;
  return cudaSuccess;
}

// ------------------------------------------------ column-major A --
// Stage layout [slot][R rows]: one TMA box of {R rows x 1 column} per distinct
// split column, so only 4 |S| bytes per row leave HBM; an encoder's "row" is
// stg + r with element offset slot(j) * R for split column j (pitch 1).
static Geometry plan_cm(int C, int W, int n_cols, bool enc_only) {
  Geometry g;
  if (n_cols < 1 || n_cols > 4 * C) return g;
  g.nslab = (n_cols + 3) & ~3;                     // gather4 fills slots in fours
  g.SW = 1;
  g.pad_e = 0;
  const int CBW = C >= 8 ? C / 8 : 1;
  size_t fixed = BAR_BYTES + thr_base(C) * 4 + off_base(C) * 4 + C * 4 + 4 * C * 4 + 16;
  if (!enc_only) fixed += (size_t)C * W * 16 * 4 + (size_t)NB * BR * CBW * 4 + 16;
  if (!enc_only && MDN_CM_STAGE != 0 && W >= 8 && W - 3 * (((W + 3) / 4) | 1) > 0)
    fixed += (size_t)8 * 32 * 16 * (((W + 3) / 4) | 1) + 128;   // cm_ostg_bytes (scanner output staging) + alignment
  fixed = (fixed + 127) & ~size_t(127);
  const size_t budget = (size_t)dev_info().smem_optin;
  // Largest R with >= 2 stages: the column boxes are R * 4 bytes and the TMA
  // rate per box, not the bytes, bounds small boxes (cls100, measured: R = 32 /
  // 64 / 128 -> 1.2 / 2.2 / 3.5e9 rows/s).
  const int force_r = env_int("MDN_CM_R", 0);       // experiment knob: fixed rows per stage
  for (int min_ns : {2}) {
    for (int R : {256, 128, 64, 32}) {
      if (force_r && R != force_r) continue;
      const size_t stage = (size_t)g.nslab * R * 4;
      if (fixed + stage * min_ns > budget) continue;
      int NS = (int)((budget - fixed) / stage);
      if (NS > NS_MAX) NS = NS_MAX;
      g.R = R;
      g.NS = NS;
      g.slab_e = R;
      g.smem = fixed + stage * NS;
      g.ok = true;
      return g;
    }
  }
  return g;
}

static bool make_tmap_cm(CUtensorMap* m, const float* At, int64_t N, int64_t ldt, int D, int R) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {(cuuint64_t)N, (cuuint64_t)D};
  cuuint64_t strides[1] = {(cuuint64_t)ldt * 4};
  cuuint32_t box[2] = {(cuuint32_t)R, 1};
  cuuint32_t estr[2] = {1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(At), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

static bool cm_ok(const TreesDev& t, const float* At, int64_t N, int64_t ldt) {
  return N <= (int64_t)0x7FFFFF00 && aligned16(At) && ldt % 4 == 0 && encode_fn() != nullptr &&
         t.n_cols >= 1;
}

cudaError_t launch_amm_ws_cm(const TreesDev& t, const LutsDev& l, const float* At, int64_t N,
                             int64_t ldt, float* out, int64_t ldo, cudaStream_t s, bool* done) {
  *done = false;
  // With TMA gather4 (4 split columns per box) this beats the thread-per-row
  // kernel of mdn_colmajor.cu from 16 codebooks up (scale 8.5 vs 5.5e9,
  // cls10_c16 1.97e10 vs 1.17e10, cls100 3.57 vs 2.56e9 rows/s); with 4-8
  // codebooks of 32-value rows the thread-per-row kernel is faster (tiny 7.2
  // vs 6.6e10, image 4.6 vs 4.2e10).
  if (t.C < 16 || !cm_ok(t, At, N, ldt) || !has_combo(t.C, l.W, l.U)) return cudaSuccess;
  Geometry g = plan_cm(t.C, l.W, t.n_cols, false);
  if (!g.ok) return cudaSuccess;
  CUtensorMap tm;
  if (!make_tmap_cm(&tm, At, N, ldt, t.D, g.R)) return cudaSuccess;
  Params p = base_params(t, g, N);
  p.slot = t.slot;
  p.cols = t.cols;
  p.n_cols = t.n_cols;
  p.ldo = ldo;
  p.M = l.M;
  p.pair = l.M % 2 == 0 && ldo % 2 == 0 && (reinterpret_cast<uintptr_t>(out) & 7u) == 0;
  p.alpha_eff = l.alpha_eff;
  p.beta32 = l.beta32;
  p.lut = l.words;
  p.out = out;
  const bool vec = l.M % 4 == 0 && ldo % 4 == 0 && aligned16(out);
  // wide tables, VEC: the scanners' staged parts leave by TMA (MDN_CM_TSTORE)
  CUtensorMap om;
  const bool ts = MDN_CM_TSTORE != 0 && vec && MDN_CM_STAGE != 0 && l.W >= 8 &&
                  l.W - 3 * (((l.W + 3) / 4) | 1) > 0;
  if (ts && !make_tmap_out(&om, out, N, l.M, ldo, 4 * (((l.W + 3) / 4) | 1), 32)) return cudaSuccess;
  *done = true;
#define X(c, w, u)                                                                   \
  if constexpr (c >= 16)                                                             \
    if (t.C == c && l.W == w && l.U == u)                                            \
      return vec ? launch_ws_sf<float, c, w, u, true, false, CM>(tm, p, g.smem, s, ts ? &om : nullptr) \
                 : launch_ws_sf<float, c, w, u, false, false, CM>(tm, p, g.smem, s);
  MDN_FAST_COMBOS(X)
#undef X
  *done = false;
  return cudaSuccess;
}

cudaError_t launch_encode_ws_cm(const TreesDev& t, const float* At, int64_t N, int64_t ldt,
                                uint8_t* codes, cudaStream_t s, bool* done) {
  *done = false;
  if (t.C < 16 || !cm_ok(t, At, N, ldt) || !has_encoder(t.C)) return cudaSuccess;
  if (reinterpret_cast<uintptr_t>(codes) & 3u) return cudaSuccess;
  Geometry g = plan_cm(t.C, 1, t.n_cols, true);
  if (!g.ok) return cudaSuccess;
  CUtensorMap tm;
  if (!make_tmap_cm(&tm, At, N, ldt, t.D, g.R)) return cudaSuccess;
  Params p = base_params(t, g, N);
  p.slot = t.slot;
  p.cols = t.cols;
  p.n_cols = t.n_cols;
  p.codes = codes;
  *done = true;
  switch (t.C) {
    case 16: return launch_ws_sf<float, 16, 1, 0, false, true, CM>(tm, p, g.smem, s);
    case 32: return launch_ws_sf<float, 32, 1, 0, false, true, CM>(tm, p, g.smem, s);
    case 64: return launch_ws_sf<float, 64, 1, 0, false, true, CM>(tm, p, g.smem, s);
  }
  *done = false;
  return cudaSuccess;
}

cudaError_t launch_amm(const TreesDev& t, const LutsDev& l, const float* A, int64_t N, int64_t lda,
                       float* out, int64_t ldo, cudaStream_t s) {
  bool done = false;
  cudaError_t e;
  if (rt_enabled()) {
    e = launch_amm_rt(t, l, A, N, lda, out, ldo, s, &done);
    if (done) return e;
  }
  e = amm_fast<float>(t, l, A, N, lda, out, ldo, s, &done);
  return done ? e : launch_amm_generic(t, l, A, 4, N, lda, out, ldo, s);
}

cudaError_t launch_amm_u8(const TreesDev& t, const LutsDev& l, const uint8_t* A, int64_t N,
                          int64_t lda, float* out, int64_t ldo, cudaStream_t s) {
  bool done = false;
  cudaError_t e;
  if (rt_enabled()) {
    e = launch_amm_rt_u8(t, l, A, N, lda, out, ldo, s, &done);
    if (done) return e;
  }
  e = amm_fast<uint8_t>(t, l, A, N, lda, out, ldo, s, &done);
  return done ? e : launch_amm_generic(t, l, A, 1, N, lda, out, ldo, s);
}

cudaError_t launch_encode(const TreesDev& t, const float* A, int64_t N, int64_t lda, uint8_t* codes,
                          cudaStream_t s) {
  bool done = false;
  cudaError_t e;
  if (rt_enabled()) {
    e = launch_encode_rt(t, A, N, lda, codes, s, &done);
    if (done) return e;
  }
  e = encode_fast<float>(t, A, N, lda, codes, s, &done);
  return done ? e : launch_encode_generic(t, A, 4, N, lda, codes, s);
}

cudaError_t launch_encode_u8(const TreesDev& t, const uint8_t* A, int64_t N, int64_t lda,
                             uint8_t* codes, cudaStream_t s) {
  bool done = false;
  cudaError_t e;
  if (rt_enabled()) {
    e = launch_encode_rt_u8(t, A, N, lda, codes, s, &done);
    if (done) return e;
  }
  e = encode_fast<uint8_t>(t, A, N, lda, codes, s, &done);
  return done ? e : launch_encode_generic(t, A, 1, N, lda, codes, s);
}

cudaError_t launch_scan(const LutsDev& l, const uint8_t* codes, int64_t N, int32_t* sums,
                        float* out, int64_t ldo, cudaStream_t s) {
  const bool codes_ok = l.C >= 8 ? (reinterpret_cast<uintptr_t>(codes) & 3u) == 0
                                 : (reinterpret_cast<uintptr_t>(codes) & 1u) == 0;
  if (!codes_ok) return launch_scan_generic(l, codes, N, sums, out, ldo, s);
  if (!has_combo(l.C, l.W, l.U)) {
    const int wt = l.C >= 16 ? 4 : (l.C == 8 ? 2 : (l.C == 4 ? 1 : 0));
    if (wt && has_combo(l.C, wt, l.U) && l.W > wt) {
      const int nt = (l.W + wt - 1) / wt;
      const size_t smem = (size_t)nt * l.C * wt * 16 * 4;
      if (smem <= (size_t)dev_info().smem_optin) {
        auto launch_tiled = [&](auto kern) -> cudaError_t {
          cudaError_t e = ensure_smem(reinterpret_cast<const void*>(kern), smem);
          if (e != cudaSuccess) return e;
          int per_sm = 0;
          e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 256, smem);
          if (e != cudaSuccess) return e;
          if (per_sm < 1) per_sm = 1;
          int64_t blocks = (N + 255) / 256;
          const int64_t cap = (int64_t)dev_info().sms * per_sm;
          if (blocks > cap) blocks = cap;
          const bool pair = l.M % 2 == 0 && ldo % 2 == 0 && (reinterpret_cast<uintptr_t>(out) & 7u) == 0;
          const bool vec_codes = (reinterpret_cast<uintptr_t>(codes) & (l.C == 32 ? 15u : 7u)) == 0;
          kern<<<(unsigned)blocks, 256, smem, s>>>(l.words, l.W, nt, codes, N, l.M, sums, out, ldo,
                                                   l.alpha_eff, l.beta32, l.U == 0 ? 1 : l.U, pair,
                                                   vec_codes);
          return cudaGetLastError();
        };
#define TS(c, w, u) \
        if (l.C == c && wt == w && l.U == u) return launch_tiled(k_scan_tiled<c, w, u>);
        TS(4, 1, 0) TS(4, 1, 4) TS(8, 2, 0) TS(8, 2, 8) TS(16, 4, 0) TS(16, 4, 16)
        TS(32, 4, 0) TS(32, 4, 16) TS(64, 4, 0) TS(64, 4, 16)
#undef TS
      }
    }
    return launch_scan_generic(l, codes, N, sums, out, ldo, s);
  }
  const bool vec = out && l.M % 4 == 0 && ldo % 4 == 0 && aligned16(out);
#define X(c, w, u)                                                                  \
  if (l.C == c && l.W == w && l.U == u)                                             \
    return vec ? launch_scan_t<c, w, u, true>(l, codes, N, sums, out, ldo, s)       \
               : launch_scan_t<c, w, u, false>(l, codes, N, sums, out, ldo, s);
  MDN_FAST_COMBOS(X)
#undef X
  return launch_scan_generic(l, codes, N, sums, out, ldo, s);
}

}  // namespace mdn
