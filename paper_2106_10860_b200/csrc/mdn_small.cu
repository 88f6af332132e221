// Register-tree kernel for the small-row MADDNESS configurations (C <= 8
// codebooks, M <= 4 output columns: the Tiny and image-filter workloads, and
// the 8-bit image path of SURVEY N1).
//
// With rows of 32 values the fused path must sustain 4-16e10 rows/s, i.e. a
// budget of roughly 200 thread-instructions per row at full issue, and the
// general kernel (mdn_fast.cu: thread per row, thresholds gathered from shared
// memory at every level, 4 output columns per table word) spends ~480 on the
// 8-bit image rows. This kernel is organised so that nothing per-codebook is
// looked up at run time:
//
//   warp 0        TMA producer: one 2-D box of R = 256 rows per stage into an
//                 NS-deep shared-memory ring (mbarrier complete_tx).
//   warps 1..NWK  workers, in NG groups of 8; group g takes every NG-th stage
//                 and warp k of the group its rows [32k, 32k + 32):
//     encode      lane -> (row lane / C, codebook lane % C), C iterations per
//                 32 rows. Each lane owns ONE codebook for the whole kernel,
//                 so its tree -- 15 thresholds and 4 split
//                 dims -- lives in registers. Algorithm 1 (L228-248) becomes
//                 4 compares and 11 selects (the threshold of level t is picked
//                 by the bits already decided, L239), no shared gathers.
//                 8-bit rows: the codebook's 4-byte subspace is one 32-bit
//                 shared load and each split value one PRMT (App. B split
//                 values q = ceil(v), reading R11).
//     hand-off    the code (pre-scaled to a table byte offset) goes to a
//                 warp-private shared buffer; __syncwarp.
//     scan        lane -> row. Tables are the 16-bit-lane layout
//                 words16[c][k][w] = T[c][k][2w] | T[c][k][2w+1] << 16, so an
//                 exact sum is ONE add per (row, codebook, 2 columns), and an
//                 App. D average mu(a,b) = (a+b+1) >> 1 is 3 ops per 2 columns
//                 (vs 5 for __vavgu4 on 4 byte lanes).
//     dequant     out = fl32(alpha_eff * S + beta32) (Eq. 1), S -> fp32
//                 by the 2^23 magic-number trick (exact for S < 2^23), one
//                 FFMA rounding; 8- or 16-byte stores.
//
// ENC (mdn_encode / mdn_encode_u8 for C in {4, 8}): the same producer and
// encode, no tables and no scan; the C lanes of a row group hold a C x C
// nibble matrix (rows x codebooks) which log2(C) rotate / shuffle / merge
// stages transpose, so each lane ends with one row's packed codes and the
// warp's 32 rows leave in one coalesced store.
#include <cuda.h>
#include <cuda_runtime.h>

#include <type_traits>

#include "mdn_internal.h"
#include "mdn_tma.cuh"

namespace mdn {
namespace fast {
namespace small {

constexpr int R = 256;                   // rows per stage (= TMA box rows)
#ifndef MDN_RT_LANE_LUT
#define MDN_RT_LANE_LUT 1
#endif
// Scan tables replicated per scanner lane: word (c, k, w) of lane l at
// ((c 16 + k) W2 + w) 32 + l, so lane l's lookups always hit bank l -- any
// code mix is conflict-free (one shared copy of 16 words per codebook put the
// 32 rows' random codes on 16 banks: ~38% of the kernel's shared-load
// wavefronts were conflicts). 16 KB for W2 = 1. On for 8-bit rows (image_u8
// 1.341 -> 1.366e11 rows/s, same box); fp32 rows are HBM-bound and their
// W2 = 2 tables (32 KB) cost the tiny config a stage (-0.8%), so not there.
template <class TIn> constexpr int lanes_lut() { return sizeof(TIn) == 1 && MDN_RT_LANE_LUT ? 32 : 1; }
constexpr int NWK = 16;                  // worker warps
constexpr int THREADS = 32 * (1 + NWK);
#ifndef MDN_RT_SUBS_U8_ENC
#define MDN_RT_SUBS_U8_ENC 2 // 32-row chunks an 8-bit encode-only worker takes per stage
#endif
// A worker takes SUBS consecutive 32-row chunks of a stage (one barrier wait
// and release per SUBS chunks); CPS workers share a stage, NG groups rotate.
// Two chunks per wait pay only where the per-stage overhead is a visible share
// of the work: the 8-bit encode-only kernel (same box: 1.285 -> 1.389e11
// rows/s); the fused 8-bit kernel lost 2.4% with it, fp32 rows are HBM-bound.
template <class TIn, bool ENC> constexpr int subs_of() {
  return sizeof(TIn) == 1 && ENC ? MDN_RT_SUBS_U8_ENC : 1;
}
template <class TIn, bool ENC> constexpr int cps_of() { return R / (32 * subs_of<TIn, ENC>()); }
template <class TIn, bool ENC> constexpr int ng_of() { return NWK / cps_of<TIn, ENC>(); }
#ifndef MDN_RT_NS_MAX
#define MDN_RT_NS_MAX 16
#endif
// Stage ring depth cap. 8-bit stages are 8 KB (256 rows x 32 B): 8 stages keep
// only 64 KB per SM in flight, under the bytes HBM latency needs at 35 GB/s
// per SM; 16 (the barrier block's 256 bytes hold 2 x 16) lift that to 128 KB.
constexpr int NS_MAX = MDN_RT_NS_MAX;
static_assert(2 * NS_MAX * 8 <= 256, "full/empty barriers must fit below OFF_LUT");
#ifndef MDN_RT_CTAS_U8
#define MDN_RT_CTAS_U8 1     // resident CTAs per SM of the 8-bit variants (tuning: -DMDN_RT_CTAS_U8=2)
#endif

struct SParams {
  int64_t N, n_tiles, ldo;
  int pitch_e;                   // elements per shared row (fp32: D + 4; 8-bit: D)
  int stage_b;                   // bytes per stage, 128-aligned
  int NS;
  int M;
  float alpha_eff, beta32;
  const uint32_t* lut16;         // global [C][16][W2]
  const uint16_t* dims;          // global [C][4]
  const uint16_t* sub;           // global [C]
  const float* thr;              // global [C][16]
  const uint16_t* q;             // global [C][16]
  float* out;
  uint8_t* codes;                // encode-only: packed 4-bit codes, N x C/2
};

// Code rows are C words (one table address per codebook). C = 8: rows whose
// index has bit 2 set store their two 16-B halves swapped (word c ^ 4), and
// the scanner's lane-per-row LDS.128 reads apply the same swizzle, so the
// encoder's stores (4 rows x 8 codebooks) and the reads (a quarter-warp =
// rows 8k..8k+7) both cover all 32 banks once, and every lane sees its
// codebooks in order.
template <int C>
struct CodeStride {
  static constexpr int value = C;
};

// Algorithm 1 with the tree in registers: p <- 2p + [x_t >= v^t_p] where the
// level-t threshold v^t_p is selected by the bits b_0..b_{t-1} already taken.
template <class V>
__device__ __forceinline__ uint32_t tree_code(V x0, V x1, V x2, V x3, const V (&t)[15]) {
  const bool b0 = x0 >= t[0];
  const bool b1 = x1 >= (b0 ? t[2] : t[1]);
  const V u2 = b0 ? (b1 ? t[6] : t[5]) : (b1 ? t[4] : t[3]);
  const bool b2 = x2 >= u2;
  const V e0 = b2 ? t[8] : t[7], e1 = b2 ? t[10] : t[9];
  const V e2 = b2 ? t[12] : t[11], e3 = b2 ? t[14] : t[13];
  const V u3 = b0 ? (b1 ? e3 : e2) : (b1 ? e1 : e0);
  const bool b3 = x3 >= u3;
  return (b0 ? 8u : 0u) + (b1 ? 4u : 0u) + (b2 ? 2u : 0u) + (b3 ? 1u : 0u);
}

// 8-bit rows whose split values all fit a byte (q <= 255; always true for a
// model trained on 8-bit data, App. B): Algorithm 1 with one byte-shuffle per
// level instead of a select tree, and the rest as adds / multiplies so that
// ptxas can spread the work over the FMA pipe as well as the ALU pipe (the
// select-tree version saturates the ALU pipe at 85% on the image_u8 config).
//   lt_t = [x_t < v_t] = 1 - b_t is the sign bit of x_t - v_t;
//   n_{t+1} = 2 n_t + lt_t is the complemented node index (n_4 = 15 - code).
//   Levels 2 and 3 pick their threshold with PRMT from the byte-packed level
//   table (complemented node order) with selector n: byte 0 holds the
//   threshold, bytes 1-3 byte 0 of the table (g); the split value is packed
//   the same way (x, g, g, g), so the word difference is x - v and its sign
//   is the compare.
struct ByteTree {
  int q0, q2, d12;                 // level 0 threshold; level 1: v = q2 + lt0 * (q1 - q2)
  uint32_t s01;                    // PRMT selector: x1 in bits 0-7, x0 in bits 16-23
  uint32_t q0s, nq2s, nd12s;       // q0 << 16, -(q2 << 16), -((q1 - q2) << 16)
  uint32_t Q2, Q3lo, Q3hi;         // level tables, byte n = threshold of complemented node n
  uint32_t s0, s1, s2, s3;         // PRMT selectors of the split values in the subspace word
  uint32_t g2, g3;                 // byte 0 of Q2 / Q3lo (pad bytes of the packed compares)
  uint32_t base;                   // table address of code 15 (n_4 = 0)
  uint32_t oh[4];                  // dp4a forms: one-hot byte of split dim t in the subspace word
  uint32_t nq0, nd12, nq2;         // -q0, -(q1 - q2), -q2
};

// Raw PRMT / shift: __byte_perm masks its selector (LOP3 & 0x7777) to hide
// PRMT's sign-replicate bit, and a plain (x - v) >> 31 is pattern-matched back
// into ISETP + SEL (ALU pipe); our selectors never set bit 3 of a nibble.
__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t s) {
  uint32_t d;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(s));
  return d;
}
__device__ __forceinline__ uint32_t sign_bit(uint32_t x) {
  uint32_t d;
  asm("shr.u32 %0, %1, 31;" : "=r"(d) : "r"(x));
  return d;
}

// n' = 2n + [d < 0] in one funnel shift: the upper word of {n, d} << 1.
__device__ __forceinline__ uint32_t push_sign(uint32_t n, uint32_t d) {
  uint32_t r;
  asm("shf.l.wrap.b32 %0, %1, %2, 1;" : "=r"(r) : "r"(d), "r"(n));
  return r;
}

#ifndef MDN_BQ01
#define MDN_BQ01 1   // levels 0 and 1 from one PRMT (x1 + (x0 << 16)); 0: one PRMT each
#endif
// Byte-tree levels in the dp4a form (template DP, a bitmask; bit 0: levels 0+1,
// bit 1: level 2, bit 2: level 3): x_j - v as dp4a(w, onehot_j, -v) or
// dp4a(V, -1 @ byte 0, x_j) on the FMA pipe instead of PRMT + subtract on the
// ALU pipe, which the byte trees saturate. Same-box A/B (rows/s, image_u8):
// fused 0: 1.364e11, 6: 1.375e11, 7: 1.255e11 (the FMA pipe then carries the
// scan's adds as well); encode-only 0: 1.414e11, 4: 1.483e11, 6: 1.475e11,
// 7: 1.495e11. MDN_BQ_DP (build flag) forces one form for A/B.
template <bool ENC>
constexpr int bq_dp() {
#ifdef MDN_BQ_DP
  return MDN_BQ_DP;
#else
  return ENC ? 7 : 6;
#endif
}

// x_j - v on the FMA pipe: dp4a(w, onehot_j, c) = x_j + c, and
// dp4a(V, 0x000000FF, x) = x - byte0(V) (signed b: -1 at byte 0, 0 elsewhere).
__device__ __forceinline__ uint32_t dp4a_uu(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d;
  asm("dp4a.u32.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}
__device__ __forceinline__ uint32_t dp4a_us(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d;
  asm("dp4a.u32.s32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}
static __constant__ uint32_t k_shift16 = 65536u;   // opaque to ptxas: the multiply stays an IMAD

__device__ __forceinline__ uint32_t mad_lo(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d;
  asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}

// 15 - code (the complemented leaf index n_4) for 8-bit rows; see byte_tree_addr.
// Levels 0 and 1 (MDN_BQ01): r = x1 + (x0 << 16) from one PRMT; r - (q0 << 16)
// is negative iff x0 < q0 (x1 < 2^16 cannot carry into the sign), and
// r * 2^16 - (v1 << 16) = (x1 - v1) << 16 has the sign of x1 - v1 (|x1 - v1|
// < 2^8), both products on the FMA pipe.
template <int DP>
__device__ __forceinline__ uint32_t byte_tree_n4(uint32_t w, const ByteTree& b) {
  uint32_t n2;
  if constexpr ((DP & 1) != 0) {
    // dp4a form: x0 - q0 and x1 - v1 (v1 = q2 + lt0 (q1 - q2)) as dp4a(w, onehot, -v)
    const uint32_t lt0 = sign_bit(dp4a_uu(w, b.oh[0], b.nq0));
    n2 = push_sign(lt0, dp4a_uu(w, b.oh[1], mad_lo(lt0, b.nd12, b.nq2)));
  } else {
#if MDN_BQ01
    const uint32_t r = prmt(w, 0u, b.s01);
    const uint32_t lt0 = sign_bit(r - b.q0s);
    n2 = push_sign(lt0, mad_lo(r, k_shift16, mad_lo(lt0, b.nd12s, b.nq2s)));
#else
    const uint32_t lt0 = sign_bit(prmt(w, 0u, b.s0) - (uint32_t)b.q0);
    const uint32_t v1 = (uint32_t)b.q2 + lt0 * (uint32_t)b.d12;
    n2 = push_sign(lt0, prmt(w, 0u, b.s1) - v1);
#endif
  }
  uint32_t n3;
  if constexpr ((DP & 2) != 0)
    n3 = push_sign(n2, dp4a_us(prmt(b.Q2, b.Q2, n2), 0x000000FFu, dp4a_uu(w, b.oh[2], 0u)));
  else
    n3 = push_sign(n2, prmt(w, b.g2, b.s2) - prmt(b.Q2, b.Q2, n2));
  if constexpr ((DP & 4) != 0)
    return push_sign(n3, dp4a_us(prmt(b.Q3lo, b.Q3hi, n3), 0x000000FFu, dp4a_uu(w, b.oh[3], 0u)));
  else
    return push_sign(n3, prmt(w, b.g3, b.s3) - prmt(b.Q3lo, b.Q3hi, n3));
}

template <int W2>
__device__ __forceinline__ uint32_t byte_tree_addr(uint32_t w, const ByteTree& b) {
  return b.base - byte_tree_n4<bq_dp<false>()>(w, b) * (4u * W2 * lanes_lut<uint8_t>());   // 15 - n4 = code
}

// mu(a, b) = floor((a + b + 1) / 2) on two 16-bit lanes holding values < 256
// (App. D): the sum is < 512, so no carry crosses lanes; the shift moves
// the high lane's bit 0 into bit 15, which the mask clears.
__device__ __forceinline__ uint32_t avg16(uint32_t a, uint32_t b) {
  return ((a + b + 0x00010001u) >> 1) & 0x7FFF7FFFu;
}

__device__ __forceinline__ uint32_t lds_u32(uint32_t addr) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr));
  return v;
}

__device__ __forceinline__ float u16_to_f(uint32_t s) {
  return __uint_as_float(0x4B000000u | s) - 8388608.0f;   // exact for s < 2^23
}

// TIn = float: fp32 rows. TIn = uint8_t: 8-bit rows whose codebooks are
// 4-byte subspaces [4c, 4c + 4) (the image config; other byte layouts use the
// general kernel). VEC: 0 = guarded scalar stores, 1 = M == 2 W2 with 8-byte
// (W2 odd) or 16-byte (W2 even) aligned rows.
// ENC: encode only (mdn_encode / mdn_encode_u8): the C lanes of a row OR
// their nibbles together with shuffles and one lane stores the row's packed
// codes; no tables, no scan.
template <class TIn, int D, int C, int W2, int U, int VEC, bool BQ, bool ENC = false>
__global__ void __launch_bounds__(THREADS, sizeof(TIn) == 1 ? MDN_RT_CTAS_U8 : 1)
    k_amm_rt(const __grid_constant__ CUtensorMap tmap, const SParams p) {
  // Shared row pitch (elements): fp32 rows D + 4 (pitch == 4 mod 32 words);
  // 8-bit rows D bytes unpadded, so the encoder's 4-row x 8-codebook word
  // loads hit 32 distinct banks (a 48-byte pitch made them 2-way conflicted)
  // and the stage holds a third fewer bytes.
  constexpr int PITCH = sizeof(TIn) == 1 ? D : D + 16 / (int)sizeof(TIn);
  constexpr int RPW = 32 / C;                       // rows per encode iteration
  constexpr int SUBS = subs_of<TIn, ENC>(), CPS = cps_of<TIn, ENC>(), NG = ng_of<TIn, ENC>();
  constexpr int CS = CodeStride<C>::value;
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);
  uint64_t* empty = full + NS_MAX;
  constexpr int OFF_LUT = 256;
  constexpr int LANES_LUT = lanes_lut<TIn>();
  constexpr bool LANE_LUT = LANES_LUT > 1;
  constexpr int OFF_CODE = OFF_LUT + C * 16 * W2 * 4 * LANES_LUT;
  constexpr int OFF_STAGE = ENC ? 256 : (OFF_CODE + NWK * 32 * CS * 4 + 127) & ~127;
  uint32_t* s_lut = reinterpret_cast<uint32_t*>(smem + OFF_LUT);
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;

  if constexpr (!ENC)
    for (int i = tid; i < C * 16 * W2 * LANES_LUT; i += blockDim.x) s_lut[i] = p.lut16[i / LANES_LUT];
  if (tid == 0) {
    for (int s = 0; s < p.NS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], CPS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap)) : "memory");
  }
  __syncthreads();

  // Local stage sequence of this CTA: tiles blockIdx.x, blockIdx.x + grid, ...
  // stages of this CTA (< 2^31: N < 2^31 rows are checked on the host)
  const int n_local = (int)((p.n_tiles - blockIdx.x + gridDim.x - 1) / gridDim.x);

  if (warp == 0) {
    // ---------------- TMA producer ----------------
    if (lane == 0) {
      const uint32_t bytes = (uint32_t)(R * p.pitch_e * sizeof(TIn));
      int s = 0;
      uint32_t ph = 0;
      for (int q = 0; q < n_local; ++q) {
        mbar_wait_sleep(&empty[s], ph ^ 1u);
        mbar_arrive_tx(&full[s], bytes);
        const int64_t y = (blockIdx.x + q * gridDim.x) * (int64_t)R;
        tma_load_2d(smem + OFF_STAGE + (size_t)s * p.stage_b, &tmap, 0, (int)y, &full[s], 0, 0);
        if (++s == p.NS) s = 0, ph ^= 1u;
      }
    }
    return;
  }

  // ---------------- workers ----------------
  const int wk = warp - 1;
  const int grp = wk / CPS, chunk = wk % CPS;
  const int c = lane % C;                            // this lane's codebook (fixed)
  const int rs = lane / C;
  uint32_t* s_code = reinterpret_cast<uint32_t*>(smem + OFF_CODE) + wk * 32 * CS;

  // The lane's tree in registers.
  using V = typename std::conditional<sizeof(TIn) == 1, int, float>::type;
  V th[15];
#pragma unroll
  for (int i = 0; i < 15; ++i) {
    if constexpr (sizeof(TIn) == 1) th[i] = (int)p.q[c * 16 + i];
    else th[i] = p.thr[c * 16 + i];
  }
  int o[4];                                          // split-dim element offsets
  uint32_t sel[4];                                   // 8-bit rows: PRMT selectors
  const int sub = p.sub[c];
#pragma unroll
  for (int t = 0; t < 4; ++t) {
    o[t] = p.dims[c * 4 + t];
    sel[t] = (uint32_t)(o[t] - sub) | 0x4440u;       // zero-extend the selected byte
  }

  // Per-lane addressing, fixed for the kernel: the lane reads row rs of each
  // RPW-row group; the codebook's table base (absolute shared address) is
  // folded into the stored code so the scanner's lookups need no adds.
  // (with per-lane tables: + 4 rs, the scanner lane of this lane's row in each
  // RPW-row group; the group's 4 RPW it is added per iteration)
  const uint32_t lut_c = su32(s_lut) + (uint32_t)(c * 16 * W2 * 4 * LANES_LUT) +
                         (LANE_LUT ? 4u * (uint32_t)rs : 0u);
  ByteTree bt{};
  if constexpr (BQ) {
    const uint16_t* qc = p.q + c * 16;             // heap order; complemented node n at level t
    bt.q0 = qc[0];                                 //   is heap index 2^(t+1) - 2 - n
    bt.q2 = qc[2];
    bt.d12 = (int)qc[1] - (int)qc[2];
    bt.Q2 = 0u, bt.Q3lo = 0u, bt.Q3hi = 0u;
#pragma unroll
    for (int n = 0; n < 4; ++n) bt.Q2 |= (uint32_t)qc[6 - n] << (8 * n);
#pragma unroll
    for (int n = 0; n < 4; ++n) bt.Q3lo |= (uint32_t)qc[14 - n] << (8 * n);
#pragma unroll
    for (int n = 0; n < 4; ++n) bt.Q3hi |= (uint32_t)qc[10 - n] << (8 * n);
    bt.g2 = bt.Q2 & 0xFFu;
    bt.g3 = bt.Q3lo & 0xFFu;
    const uint32_t j0 = o[0] - sub, j1 = o[1] - sub, j2 = o[2] - sub, j3 = o[3] - sub;
    bt.s0 = j0 | 0x4440u;
    bt.s1 = j1 | 0x4440u;
    bt.s01 = j1 | 0x40u | (j0 << 8) | 0x4000u;    // (x1, 0, x0, 0)
    bt.q0s = (uint32_t)bt.q0 << 16;
    bt.nq2s = 0u - ((uint32_t)bt.q2 << 16);
    bt.nd12s = 0u - ((uint32_t)bt.d12 << 16);
    bt.s2 = j2 | 0x4440u;                          // (x, g, g, g)
    bt.s3 = j3 | 0x4440u;
    bt.base = lut_c + 15u * 4u * W2 * LANES_LUT;
    bt.oh[0] = 1u << (8 * j0), bt.oh[1] = 1u << (8 * j1), bt.oh[2] = 1u << (8 * j2), bt.oh[3] = 1u << (8 * j3);
    bt.nq0 = 0u - (uint32_t)bt.q0;
    bt.nd12 = 0u - (uint32_t)bt.d12;
    bt.nq2 = 0u - (uint32_t)bt.q2;
  }
  // ENC transpose constants: stage k exchanges with lane c ^ 2^k; a lane whose
  // bit k is b keeps the nibbles whose index has bit k == b and receives the
  // partner's rotated by 4 * 2^k the other way.
  constexpr int LOGC = C == 8 ? 3 : 2;
  uint32_t t_rot[LOGC], t_sel[LOGC];
#pragma unroll
  for (int k = 0; k < LOGC; ++k) {
    const uint32_t lo = k == 0 ? 0x0F0F0F0Fu : (k == 1 ? 0x00FF00FFu : 0x0000FFFFu);
    const bool b = (c >> k) & 1;
    t_rot[k] = b ? 32u - (4u << k) : (4u << k);
    t_sel[k] = (b ? ~lo : lo) | (C == 4 ? 0xFFFF0000u : 0u);
  }
  int s = grp, ph = 0;
  while (s >= p.NS) s -= p.NS, ph ^= 1;
  // This lane's output row and pointer, advanced by a constant stride per stage.
  // 32-bit row counter: N <= 0x7FFFFF00 (host check), unsigned wrap past the
  // last stage is never compared
  uint32_t row = ((uint32_t)blockIdx.x + (uint32_t)grp * gridDim.x) * R + chunk * 32 * SUBS + lane;
  const uint32_t row_step = (uint32_t)NG * gridDim.x * R;
  const uint32_t n_rows = (uint32_t)p.N;
  float* o_row = p.out + (int64_t)row * p.ldo;
  const int64_t o_step = (int64_t)row_step * p.ldo;
  const float alpha = p.alpha_eff, beta = p.beta32;
  for (int q = grp; q < n_local; q += NG, row += row_step, o_row += o_step) {
    mbar_wait_sleep(&full[s], (uint32_t)ph);
#pragma unroll 1
    for (int hs = 0; hs < SUBS; ++hs) {
    const TIn* stg = reinterpret_cast<const TIn*>(smem + OFF_STAGE + (size_t)s * p.stage_b) +
                     (size_t)(chunk * 32 * SUBS + hs * 32 + rs) * PITCH;
    // ---- encode 32 rows: C iterations of RPW rows x C codebooks ----
    // All loads first, then the (independent) trees, then the stores, so the
    // compiler may interleave the C dependency chains.
    uint32_t code[C];                                // table entry addresses
    if constexpr (sizeof(TIn) == 1) {
      uint32_t w[C];
#pragma unroll
      for (int it = 0; it < C; ++it)
        w[it] = *reinterpret_cast<const uint32_t*>(stg + it * RPW * PITCH + sub);
#pragma unroll
      for (int it = 0; it < C; ++it) {
        if constexpr (BQ && ENC)
          code[it] = 15u - byte_tree_n4<bq_dp<true>()>(w[it], bt);
        else if constexpr (BQ)
          code[it] = byte_tree_addr<W2>(w[it], bt) + (LANE_LUT ? 4u * RPW * it : 0u);
        else
          code[it] = (ENC ? 0u : lut_c + (LANE_LUT ? 4u * RPW * it : 0u)) + (ENC ? 1u : 4u * W2 * LANES_LUT) *
                     tree_code<int>((int)__byte_perm(w[it], 0u, sel[0]), (int)__byte_perm(w[it], 0u, sel[1]),
                                    (int)__byte_perm(w[it], 0u, sel[2]), (int)__byte_perm(w[it], 0u, sel[3]), th);
      }
    } else {
      float x[C][4];
#pragma unroll
      for (int it = 0; it < C; ++it)
#pragma unroll
        for (int t = 0; t < 4; ++t) x[it][t] = stg[it * RPW * PITCH + o[t]];
#pragma unroll
      for (int it = 0; it < C; ++it)
        code[it] = (ENC ? 0u : lut_c + (LANE_LUT ? 4u * RPW * it : 0u)) + (ENC ? 1u : 4u * W2 * LANES_LUT) *
                   tree_code<float>(x[it][0], x[it][1], x[it][2], x[it][3], th);
    }
    if constexpr (ENC) {
      // Lane (rs, c) holds codebook c of rows it * RPW + rs: a C x C nibble
      // matrix over the group's lanes. Pack it (nibble it), then transpose it
      // with log2(C) butterfly stages (rotate, shuffle, merge) so that lane
      // (rs, c) holds row c * RPW + rs, and the warp's 32 rows leave in one
      // coalesced store (low nibble = even codebook, L147 / L608).
      uint32_t keep = code[C - 1];
#pragma unroll
      for (int it = C - 2; it >= 0; --it) keep = keep * 16u + code[it];
#pragma unroll
      for (int k = 0; k < LOGC; ++k) {
        const uint32_t t = __funnelshift_r(keep, keep, t_rot[k]);
        const uint32_t r = __shfl_xor_sync(0xffffffffu, t, 1 << k);
        keep = (keep & t_sel[k]) | (r & ~t_sel[k]);
      }
      const int64_t r = ((int64_t)blockIdx.x + (int64_t)q * gridDim.x) * R + chunk * 32 * SUBS + hs * 32 +
                        c * RPW + rs;
      if (r < p.N) {
        if constexpr (C == 8)
          reinterpret_cast<uint32_t*>(p.codes)[r] = keep;
        else
          reinterpret_cast<uint16_t*>(p.codes)[r] = (uint16_t)keep;
      }
      __syncwarp();
      if (hs == SUBS - 1 && lane == 0) mbar_arrive(&empty[s]);
      continue;                                      // next chunk of this stage
    }
#pragma unroll
    for (int it = 0; it < C; ++it) {
      const int rr = it * RPW + rs;
      s_code[rr * CS + (C == 8 ? (c ^ (rr & 4)) : c)] = code[it];
    }
    __syncwarp();
    if (hs == SUBS - 1 && lane == 0) mbar_arrive(&empty[s]);   // the stage's rows are consumed
    // ---- scan row `lane` ----
    uint32_t off[C];
#pragma unroll
    for (int k = 0; k < C; k += 4) {
      // read with the store's swizzle: a quarter-warp's 8 rows then cover the 32
      // banks once (unswizzled reads of rows r and r + 4 hit the same 4 banks:
      // ncu, image_u8: 8 wavefronts per LDS.128 for an ideal 4)
      const uint4 v = *reinterpret_cast<const uint4*>(s_code + lane * CS + (C == 8 ? (k ^ (lane & 4)) : k));
      off[k] = v.x, off[k + 1] = v.y, off[k + 2] = v.z, off[k + 3] = v.w;
    }
    __syncwarp();                                    // s_code may be rewritten next stage
    uint32_t acc[W2];
#pragma unroll
    for (int w = 0; w < W2; ++w) acc[w] = 0u;
    if constexpr (U == 0) {
#pragma unroll
      for (int cc = 0; cc < C; ++cc)
#pragma unroll
        for (int w = 0; w < W2; ++w)
          acc[w] += lds_u32(off[cc] + 4 * LANES_LUT * w);
    } else {
      static_assert((U & (U - 1)) == 0 && C % U == 0, "U must be a power of two dividing C");
#pragma unroll
      for (int blk = 0; blk < C / U; ++blk)
#pragma unroll
        for (int w = 0; w < W2; ++w) {
          uint32_t v[U];
#pragma unroll
          for (int i = 0; i < U; ++i) {
            const int cc = blk * U + i;
            v[i] = lds_u32(off[cc] + 4 * LANES_LUT * w);
          }
#pragma unroll
          for (int st = 1; st < U; st *= 2)          // halves recursion = adjacent pairs (R17)
#pragma unroll
            for (int i = 0; i < U; i += 2 * st) v[i] = avg16(v[i], v[i + st]);
          acc[w] += v[0];
        }
    }
    if (row + hs * 32 < n_rows) {
      float* o_h = o_row + (int64_t)hs * 32 * p.ldo;
      float f[2 * W2];
#pragma unroll
      for (int w = 0; w < W2; ++w) {
        f[2 * w] = __fmaf_rn(alpha, u16_to_f(acc[w] & 0xFFFFu), beta);
        f[2 * w + 1] = __fmaf_rn(alpha, u16_to_f(acc[w] >> 16), beta);
      }
      if constexpr (VEC) {
        if constexpr (W2 % 2 == 0) {
#pragma unroll
          for (int w = 0; w < W2; w += 2)
            *reinterpret_cast<float4*>(o_h + 2 * w) = make_float4(f[2 * w], f[2 * w + 1], f[2 * w + 2], f[2 * w + 3]);
        } else {
#pragma unroll
          for (int w = 0; w < W2; ++w)
            *reinterpret_cast<float2*>(o_h + 2 * w) = make_float2(f[2 * w], f[2 * w + 1]);
        }
      } else {
#pragma unroll
        for (int m = 0; m < 2 * W2; ++m)
          if (m < p.M) o_h[m] = f[m];
      }
    }
    }  // chunks of the stage
    // next ring slot of this group: NS % NG == 0 and NG <= NS, so one wrap at most
    s += NG;
    if (s >= p.NS) s -= p.NS, ph ^= 1;
  }
}

// ---------------------------------------------------------------------------
// k_u8_rows: the 8-bit byte-tree path with lane = row for BOTH halves.
//
// k_amm_rt maps lane -> (row, codebook) for the encode so that each lane keeps
// one codebook's tree in registers, and then hands the codes to lane -> row
// for the scan through a shared buffer (per 32 rows and C = 8: 8 word loads,
// 8 code stores, 2 x LDS.128 back, two __syncwarp; encode-only: a 3-stage
// nibble transpose). For 8-bit rows whose codebooks are the 4-byte words of
// the row (App. B; image_u8) all of that can go: the lane loads its own
// 32-byte row (2 x LDS.128) and walks all C trees itself. The trees' byte
// tables and selectors are the same for every lane, so they are kernel
// parameters (constant bank operands of PRMT / IMAD / IDP4A) rather than
// per-lane registers; only the PRMT sources Q2, Q3lo, Q3hi need registers.
// Per (row, codebook) the encode is the same byte tree as k_amm_rt (one PRMT
// per level picks the node's split value; sign-bit
// compares, Alg. 1), the table address one IMAD, the lookup one LDS.
// Encode-only: the row's codes pack into one register (no transpose) and leave
// in one coalesced 4-byte store per lane.
// Stage ring cap (8 KB stages). Same-box A/B (exact / avg / encode rows/s):
// 16 stages 1.400 / 1.273 / 1.552e11, 24: 1.377 / 1.271 / 1.521e11, 32:
// 1.377 / 1.273 / 1.501e11 -- not bound by bytes in flight.
#ifndef MDN_U8ROWS_NS_MAX
#define MDN_U8ROWS_NS_MAX 16
#endif
constexpr int U8_NS_MAX = MDN_U8ROWS_NS_MAX;
#ifndef MDN_U8ROWS_NWK
#define MDN_U8ROWS_NWK 16      // worker warps of k_u8_rows
#endif
constexpr int U8_NWK = MDN_U8ROWS_NWK;
constexpr int U8_THREADS = 32 * (1 + U8_NWK);
struct RParams {
  SParams p;
  ByteTree cb[8];   // per codebook; ByteTree::base unused (lane-independent)
};

template <int C, int W2, int U, int VEC, bool ENC, int DP, int SUBS>
__global__ void __launch_bounds__(U8_THREADS, 1)
    k_u8_rows(const __grid_constant__ CUtensorMap tmap, const __grid_constant__ RParams rp) {
  static_assert(C == 8, "codebooks are the 4-byte words of a 32-byte row");
  constexpr int D = 32;
  constexpr int CPS = R / (32 * SUBS), NG = U8_NWK / CPS;
  constexpr int LROW = 128;                        // bytes per (c, k, w) table row: 32 lanes
  constexpr int OFF_LUT = 16 * U8_NS_MAX;          // full / empty barriers below
  constexpr int OFF_STAGE = (OFF_LUT + (ENC ? 0 : C * 16 * W2 * LROW) + 127) & ~127;
  const SParams& p = rp.p;
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);
  uint64_t* empty = full + U8_NS_MAX;
  uint32_t* s_lut = reinterpret_cast<uint32_t*>(smem + OFF_LUT);
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;

  // per-lane replicated tables: word (c, k, w) of lane l at ((c 16 + k) W2 + w) 32 + l
  if constexpr (!ENC)
    for (int i = tid; i < C * 16 * W2 * 32; i += blockDim.x) s_lut[i] = p.lut16[i >> 5];
  if (tid == 0) {
    for (int s = 0; s < p.NS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], CPS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap)) : "memory");
  }
  __syncthreads();
  const int n_local = (int)((p.n_tiles - blockIdx.x + gridDim.x - 1) / gridDim.x);

  if (warp == 0) {
    if (lane == 0) {
      const uint32_t bytes = (uint32_t)(R * D);
      int s = 0;
      uint32_t ph = 0;
      for (int q = 0; q < n_local; ++q) {
        mbar_wait_sleep(&empty[s], ph ^ 1u);
        mbar_arrive_tx(&full[s], bytes);
        const int64_t y = (blockIdx.x + q * gridDim.x) * (int64_t)R;
        tma_load_2d(smem + OFF_STAGE + (size_t)s * p.stage_b, &tmap, 0, (int)y, &full[s], 0, 0);
        if (++s == p.NS) s = 0, ph ^= 1u;
      }
    }
    return;
  }

  const int wk = warp - 1;
  const int grp = wk / CPS, chunk = wk % CPS;
  // table address of (c, k = 15, w = 0) for this lane; code k = 15 - n4
  const uint32_t lbase = su32(s_lut) + 4u * (uint32_t)lane + 15u * W2 * LROW;
  int s = grp, ph = 0;
  while (s >= p.NS) s -= p.NS, ph ^= 1;
  uint32_t row = ((uint32_t)blockIdx.x + (uint32_t)grp * gridDim.x) * R + chunk * 32 * SUBS + lane;
  const uint32_t row_step = (uint32_t)NG * gridDim.x * R;
  const uint32_t n_rows = (uint32_t)p.N;
  float* o_row = p.out + (int64_t)row * p.ldo;
  const int64_t o_step = (int64_t)row_step * p.ldo;
  const float alpha = p.alpha_eff, beta = p.beta32;

  for (int q = grp; q < n_local; q += NG, row += row_step, o_row += o_step) {
    mbar_wait_sleep(&full[s], (uint32_t)ph);
#pragma unroll 1
    for (int hs = 0; hs < SUBS; ++hs) {
      const unsigned char* rp_row =
          smem + OFF_STAGE + (size_t)s * p.stage_b + (size_t)(chunk * 32 * SUBS + hs * 32 + lane) * D;
      const uint4 lo = *reinterpret_cast<const uint4*>(rp_row);
      const uint4 hi = *reinterpret_cast<const uint4*>(rp_row + 16);
      const uint32_t xw[8] = {lo.x, lo.y, lo.z, lo.w, hi.x, hi.y, hi.z, hi.w};
      // The rows now live in registers: release the slot before the compute
      // (the arrive's release semantics order the warp's loads before it).
      __syncwarp();
      if (hs == SUBS - 1 && lane == 0) mbar_arrive(&empty[s]);
      uint32_t n4[C];
#pragma unroll
      for (int c = 0; c < C; ++c) n4[c] = byte_tree_n4<DP>(xw[c], rp.cb[c]);
      const uint32_t r = row + hs * 32;
      if constexpr (ENC) {
        // packed codes, low nibble = codebook 0 (L147 / L608): sum_c (15 - n4_c) 16^c
        uint32_t acc = n4[0];
#pragma unroll
        for (int c = 1; c < C; ++c) acc = mad_lo(n4[c], 1u << (4 * c), acc);
        if (r < n_rows) reinterpret_cast<uint32_t*>(p.codes)[r] = ~acc;
        continue;
      }
      uint32_t addr[C];
#pragma unroll
      for (int c = 0; c < C; ++c) addr[c] = mad_lo(n4[c], 0u - (uint32_t)(W2 * LROW), lbase);
      uint32_t acc[W2];
#pragma unroll
      for (int w = 0; w < W2; ++w) acc[w] = 0u;
      if constexpr (U == 0) {
#pragma unroll
        for (int c = 0; c < C; ++c)
#pragma unroll
          for (int w = 0; w < W2; ++w) acc[w] += lds_u32(addr[c] + (uint32_t)((c * 16 * W2 + w) * LROW));
      } else {
        static_assert((U & (U - 1)) == 0 && C % U == 0, "U must be a power of two dividing C");
#pragma unroll
        for (int blk = 0; blk < C / U; ++blk)
#pragma unroll
          for (int w = 0; w < W2; ++w) {
            uint32_t v[U];
#pragma unroll
            for (int i = 0; i < U; ++i) {
              const int c = blk * U + i;
              v[i] = lds_u32(addr[c] + (uint32_t)((c * 16 * W2 + w) * LROW));
            }
#pragma unroll
            for (int st = 1; st < U; st *= 2)          // halves recursion = adjacent pairs (R17)
#pragma unroll
              for (int i = 0; i < U; i += 2 * st) v[i] = avg16(v[i], v[i + st]);
            acc[w] += v[0];
          }
      }
      if (r < n_rows) {
        float* o_h = o_row + (int64_t)hs * 32 * p.ldo;
        float f[2 * W2];
#pragma unroll
        for (int w = 0; w < W2; ++w) {
          f[2 * w] = __fmaf_rn(alpha, u16_to_f(acc[w] & 0xFFFFu), beta);
          f[2 * w + 1] = __fmaf_rn(alpha, u16_to_f(acc[w] >> 16), beta);
        }
        if constexpr (VEC) {
          if constexpr (W2 % 2 == 0) {
#pragma unroll
            for (int w = 0; w < W2; w += 2)
              *reinterpret_cast<float4*>(o_h + 2 * w) = make_float4(f[2 * w], f[2 * w + 1], f[2 * w + 2], f[2 * w + 3]);
          } else {
#pragma unroll
            for (int w = 0; w < W2; ++w)
              *reinterpret_cast<float2*>(o_h + 2 * w) = make_float2(f[2 * w], f[2 * w + 1]);
          }
        } else {
#pragma unroll
          for (int m = 0; m < 2 * W2; ++m)
            if (m < p.M) o_h[m] = f[m];
        }
      }
    }
    s += NG;
    if (s >= p.NS) s -= p.NS, ph ^= 1;
  }
}

// The per-codebook byte-tree constants (as k_amm_rt's lanes build them, from
// the model's host copies of the split dims, subspace starts and 8-bit split
// values q, heap order).
static void host_byte_tree(const TreesDev& t, int c, ByteTree* b) {
  const uint16_t* qc = t.h_q + c * 16;
  *b = ByteTree{};
  b->q0 = qc[0];
  b->q2 = qc[2];
  b->d12 = (int)qc[1] - (int)qc[2];
  for (int n = 0; n < 4; ++n) b->Q2 |= (uint32_t)qc[6 - n] << (8 * n);
  for (int n = 0; n < 4; ++n) b->Q3lo |= (uint32_t)qc[14 - n] << (8 * n);
  for (int n = 0; n < 4; ++n) b->Q3hi |= (uint32_t)qc[10 - n] << (8 * n);
  b->g2 = b->Q2 & 0xFFu;
  b->g3 = b->Q3lo & 0xFFu;
  uint32_t j[4];
  for (int l = 0; l < 4; ++l) j[l] = (uint32_t)(t.h_dims[c * 4 + l] - t.h_sub[c]);
  b->s0 = j[0] | 0x4440u;
  b->s1 = j[1] | 0x4440u;
  b->s01 = j[1] | 0x40u | (j[0] << 8) | 0x4000u;
  b->q0s = (uint32_t)b->q0 << 16;
  b->nq2s = 0u - ((uint32_t)b->q2 << 16);
  b->nd12s = 0u - ((uint32_t)b->d12 << 16);
  b->s2 = j[2] | 0x4440u;
  b->s3 = j[3] | 0x4440u;
  b->base = 0u;
  for (int l = 0; l < 4; ++l) b->oh[l] = 1u << (8 * j[l]);
  b->nq0 = 0u - (uint32_t)b->q0;
  b->nd12 = 0u - (uint32_t)b->d12;
  b->nq2 = 0u - (uint32_t)b->q2;
}

// Per mode: 32-row chunks per stage wait (SUBS) and the byte-tree level forms
// (DP, as bq_dp). Same-box A/B, image_u8 rows/s: exact SUBS 1 -> 2 1.24 ->
// 1.40e11 (DP 7: 1.21 / 1.20e11); encode-only SUBS 2, DP 6 1.55e11 (SUBS 1
// 1.36e11; DP 7 1.25e11); averaging SUBS 1, DP 7 1.39e11 (SUBS 2: DP 6
// 1.27e11, DP 7 1.19e11). Build flags override (A/B only).
#ifndef MDN_U8ROWS_SUBS
#define MDN_U8ROWS_SUBS 2
#endif
#ifndef MDN_U8ROWS_SUBS_AVG
#define MDN_U8ROWS_SUBS_AVG 1
#endif
#ifndef MDN_U8ROWS_SUBS_ENC
#define MDN_U8ROWS_SUBS_ENC 2
#endif
#ifndef MDN_U8ROWS_DP
#define MDN_U8ROWS_DP 6
#endif
#ifndef MDN_U8ROWS_DP_AVG
#define MDN_U8ROWS_DP_AVG 7
#endif
#ifndef MDN_U8ROWS_DP_ENC
#define MDN_U8ROWS_DP_ENC 6
#endif
template <bool ENC, int U>
struct U8Cfg {
  static constexpr int SUBS = ENC ? MDN_U8ROWS_SUBS_ENC : (U ? MDN_U8ROWS_SUBS_AVG : MDN_U8ROWS_SUBS);
  static constexpr int DP = ENC ? MDN_U8ROWS_DP_ENC : (U ? MDN_U8ROWS_DP_AVG : MDN_U8ROWS_DP);
  static constexpr int NG = U8_NWK / (R / (32 * SUBS));   // worker groups rotating over stages
};

// Is k_u8_rows applicable? 8-bit rows of 32 bytes, 8 codebooks on the row's
// 4-byte words, every split value a byte, host copies of the trees.
static bool u8_rows_ok(const TreesDev& t) {
  static const int on = env_int("MDN_U8_ROWS", 1);   // 0: k_amm_rt (A/B only)
  return on != 0 && t.C == 8 && t.D == 32 && t.subf_u8 == 1 && t.q_byte && t.h_q && t.h_dims &&
         t.h_sub;
}

template <int W2, int U, int VEC, bool ENC>
static cudaError_t launch_u8_rows(const CUtensorMap& tm, const RParams& rp, size_t smem,
                                  cudaStream_t st) {
  using Cfg = U8Cfg<ENC, U>;
  auto k = k_u8_rows<8, W2, U, VEC, ENC, Cfg::DP, Cfg::SUBS>;
  cudaError_t e = ensure_smem(reinterpret_cast<const void*>(k), smem);
  if (e != cudaSuccess) return e;
  const int64_t cap = (int64_t)dev_info().sms;
  const int64_t grid = rp.p.n_tiles < cap ? rp.p.n_tiles : cap;
  k<<<(unsigned)grid, U8_THREADS, smem, st>>>(tm, rp);
  return cudaGetLastError();
}

// Fused (codes == nullptr) or encode-only (out == nullptr) 8-bit rows.
static cudaError_t u8_rows(const TreesDev& t, const LutsDev* l, const uint8_t* A, int64_t N,
                           int64_t lda, float* out, int64_t ldo, uint8_t* codes, cudaStream_t st,
                           bool* done) {
  *done = false;
  const bool enc = codes != nullptr;
  if (N > (int64_t)0x7FFFFF00 || !u8_rows_ok(t)) return cudaSuccess;
  if ((reinterpret_cast<uintptr_t>(A) & 15u) || lda % 16) return cudaSuccess;
  if (enc && (reinterpret_cast<uintptr_t>(codes) & 3u)) return cudaSuccess;
  int W2 = 1;
  if (!enc) {
    if (l->M > 4 || !l->words16 || !(l->U == 0 || l->U == 8)) return cudaSuccess;
    W2 = (l->M + 1) / 2;
  }
  const int stage_b = R * 32;
  const size_t fixed = ((16 * U8_NS_MAX + (enc ? 0 : (size_t)8 * 16 * W2 * 128)) + 127) & ~size_t(127);
  const size_t budget = (size_t)dev_info().smem_optin;
  const bool avg = !enc && l->U != 0;
  const int NG = enc ? U8Cfg<true, 0>::NG : (avg ? U8Cfg<false, 8>::NG : U8Cfg<false, 0>::NG);
  if (fixed + (size_t)2 * NG * stage_b > budget) return cudaSuccess;
  int NS = (int)((budget - fixed) / stage_b);
  static const int ns_cap = env_int("MDN_U8ROWS_NS", U8_NS_MAX);   // ring-depth A/B knob
  if (NS > U8_NS_MAX) NS = U8_NS_MAX;
  if (NS > ns_cap) NS = ns_cap;
  NS -= NS % NG;                                    // each group owns its ring slots
  if (NS < NG) NS = NG;                             // (2 NG stages fit: checked above)
  CUtensorMap tm;
  if (!make_tmap(&tm, A, N, lda, 32, 16, R, 1)) return cudaSuccess;
  RParams rp{};
  SParams& p = rp.p;
  p.N = N;
  p.n_tiles = (N + R - 1) / R;
  p.ldo = ldo;
  p.pitch_e = 32;
  p.stage_b = stage_b;
  p.NS = NS;
  if (!enc) {
    p.M = l->M;
    p.alpha_eff = l->alpha_eff;
    p.beta32 = l->beta32;
    p.lut16 = l->words16;
  }
  p.out = out;
  p.codes = codes;
  for (int c = 0; c < 8; ++c) host_byte_tree(t, c, &rp.cb[c]);
  const size_t smem = fixed + (size_t)NS * stage_b;
  *done = true;
  if (enc) return launch_u8_rows<1, 0, 0, true>(tm, rp, smem, st);
  const uintptr_t oa = reinterpret_cast<uintptr_t>(out);
  const bool vec = l->M == 2 * W2 &&
                   (W2 % 2 == 0 ? (ldo % 4 == 0 && (oa & 15u) == 0) : (ldo % 2 == 0 && (oa & 7u) == 0));
  if (W2 == 1)
    return avg ? (vec ? launch_u8_rows<1, 8, 1, false>(tm, rp, smem, st) : launch_u8_rows<1, 8, 0, false>(tm, rp, smem, st))
               : (vec ? launch_u8_rows<1, 0, 1, false>(tm, rp, smem, st) : launch_u8_rows<1, 0, 0, false>(tm, rp, smem, st));
  return avg ? (vec ? launch_u8_rows<2, 8, 1, false>(tm, rp, smem, st) : launch_u8_rows<2, 8, 0, false>(tm, rp, smem, st))
             : (vec ? launch_u8_rows<2, 0, 1, false>(tm, rp, smem, st) : launch_u8_rows<2, 0, 0, false>(tm, rp, smem, st));
}

template <class TIn, int C, int W2, int U, int VEC, bool BQ>
cudaError_t launch(const CUtensorMap& tm, const SParams& p, size_t smem, cudaStream_t st) {
  auto k = k_amm_rt<TIn, 32, C, W2, U, VEC, BQ>;
  cudaError_t e = ensure_smem(reinterpret_cast<const void*>(k), smem);
  if (e != cudaSuccess) return e;
  const int64_t cap = (int64_t)dev_info().sms * (sizeof(TIn) == 1 ? MDN_RT_CTAS_U8 : 1);
  const int64_t grid = p.n_tiles < cap ? p.n_tiles : cap;
  k<<<(unsigned)grid, THREADS, smem, st>>>(tm, p);
  return cudaGetLastError();
}

template <class TIn, int C, bool BQ>
cudaError_t launch_enc(const CUtensorMap& tm, const SParams& p, size_t smem, cudaStream_t st) {
  auto k = k_amm_rt<TIn, 32, C, 1, 0, 0, BQ, true>;
  cudaError_t e = ensure_smem(reinterpret_cast<const void*>(k), smem);
  if (e != cudaSuccess) return e;
  const int64_t cap = (int64_t)dev_info().sms * (sizeof(TIn) == 1 ? MDN_RT_CTAS_U8 : 1);
  const int64_t grid = p.n_tiles < cap ? p.n_tiles : cap;
  k<<<(unsigned)grid, THREADS, smem, st>>>(tm, p);
  return cudaGetLastError();
}

template <class TIn, int C, int W2, int U>
cudaError_t launch_v(const CUtensorMap& tm, const SParams& p, size_t smem, bool vec, bool bq,
                     cudaStream_t st) {
  if constexpr (sizeof(TIn) == 1) {
    if (bq)
      return vec ? launch<TIn, C, W2, U, 1, true>(tm, p, smem, st)
                 : launch<TIn, C, W2, U, 0, true>(tm, p, smem, st);
  }
  return vec ? launch<TIn, C, W2, U, 1, false>(tm, p, smem, st)
             : launch<TIn, C, W2, U, 0, false>(tm, p, smem, st);
}

}  // namespace small
}  // namespace fast

using namespace fast;
using namespace fast::small;

// Is the register-tree kernel applicable? C in {4, 8}, M <= 4, U in {0, C},
// the padded row fits one TMA box, 16-B aligned A; 8-bit rows additionally need
// 4-byte subspaces [4c, 4c + 4) (t.subf_u8 == 1).
static bool rt_ok(const TreesDev& t, const LutsDev& l, const void* A, int64_t lda, int es) {
  if (!(t.C == 4 || t.C == 8) || l.M > 4 || !l.words16) return false;
  if (!(l.U == 0 || l.U == t.C)) return false;
  if ((reinterpret_cast<uintptr_t>(A) & 15u) || (lda * es) % 16) return false;
  if (t.D != 32) return false;                     // compiled row width (Tiny / image configs)
  if (es == 1 && t.subf_u8 != 1) return false;
  return true;
}

template <class TIn>
static cudaError_t amm_rt(const TreesDev& t, const LutsDev& l, const TIn* A, int64_t N,
                          int64_t lda, float* out, int64_t ldo, cudaStream_t st, bool* done) {
  constexpr int es = sizeof(TIn);
  *done = false;
  if (N > (int64_t)0x7FFFFF00 || !rt_ok(t, l, A, lda, es)) return cudaSuccess;
  if constexpr (es == 1) {
    if (knob_bq()) {
      cudaError_t e = u8_rows(t, &l, A, N, lda, out, ldo, nullptr, st, done);
      if (*done || e != cudaSuccess) return e;
    }
  }
  const int pitch_e = es == 1 ? t.D : t.D + 16 / es;     // must match the kernel's PITCH
  const int stage_b = ((R * pitch_e * es) + 127) & ~127;
  const int W2 = (l.M + 1) / 2;
  const size_t fixed = ((256 + (size_t)t.C * 16 * W2 * 4 * lanes_lut<TIn>() + (size_t)NWK * 32 * (t.C == 8 ? 12 : 4) * 4) + 127) & ~size_t(127);
  size_t budget = (size_t)dev_info().smem_optin;
  if (es == 1 && MDN_RT_CTAS_U8 > 1) budget = std::min(budget, (size_t)(233472 / MDN_RT_CTAS_U8 - 1024));
  constexpr int NG = ng_of<TIn, false>();
  if (fixed + (size_t)2 * NG * stage_b > budget) return cudaSuccess;
  int NS = (int)((budget - fixed) / stage_b);
  if (NS > NS_MAX) NS = NS_MAX;
  // Each worker group must own its ring slots (NS % NG == 0): a slot shared by
  // two groups could be waited on for phase k+1 by one group while phase k is
  // still incomplete, which the parity wait cannot tell apart.
  NS -= NS % NG;
  CUtensorMap tm;
  // box inner = SW + 16/es elements (make_tmap's padded box); SW = D - 16 for
  // 8-bit rows gives the unpadded D-byte box
  if (!make_tmap(&tm, A, N, lda, t.D, es == 1 ? t.D - 16 : t.D, R, es)) return cudaSuccess;
  SParams p{};
  p.N = N;
  p.n_tiles = (N + R - 1) / R;
  p.ldo = ldo;
  p.pitch_e = pitch_e;
  p.stage_b = stage_b;
  p.NS = NS;
  p.M = l.M;
  p.alpha_eff = l.alpha_eff;
  p.beta32 = l.beta32;
  p.lut16 = l.words16;
  p.dims = t.dims;
  p.sub = t.sub;
  p.thr = t.thr;
  p.q = t.q;
  p.out = out;
  const size_t smem = fixed + (size_t)NS * stage_b;
  const uintptr_t oa = reinterpret_cast<uintptr_t>(out);
  const bool vec = l.M == 2 * W2 &&
                   (W2 % 2 == 0 ? (ldo % 4 == 0 && (oa & 15u) == 0) : (ldo % 2 == 0 && (oa & 7u) == 0));
  *done = true;
  const bool avg = l.U != 0;
  const bool bq = t.q_byte && knob_bq();
  if (t.C == 4 && W2 == 1) return avg ? launch_v<TIn, 4, 1, 4>(tm, p, smem, vec, bq, st) : launch_v<TIn, 4, 1, 0>(tm, p, smem, vec, bq, st);
  if (t.C == 4 && W2 == 2) return avg ? launch_v<TIn, 4, 2, 4>(tm, p, smem, vec, bq, st) : launch_v<TIn, 4, 2, 0>(tm, p, smem, vec, bq, st);
  if (t.C == 8 && W2 == 1) return avg ? launch_v<TIn, 8, 1, 8>(tm, p, smem, vec, bq, st) : launch_v<TIn, 8, 1, 0>(tm, p, smem, vec, bq, st);
  if (t.C == 8 && W2 == 2) return avg ? launch_v<TIn, 8, 2, 8>(tm, p, smem, vec, bq, st) : launch_v<TIn, 8, 2, 0>(tm, p, smem, vec, bq, st);
  *done = false;
  return cudaSuccess;
}

// Encode-only variant: same pipeline, same trees, packed codes out.
template <class TIn>
static cudaError_t encode_rt(const TreesDev& t, const TIn* A, int64_t N, int64_t lda,
                             uint8_t* codes, cudaStream_t st, bool* done) {
  constexpr int es = sizeof(TIn);
  *done = false;
  if (N > (int64_t)0x7FFFFF00 || !(t.C == 4 || t.C == 8) || t.D != 32) return cudaSuccess;
  if ((reinterpret_cast<uintptr_t>(A) & 15u) || (lda * es) % 16) return cudaSuccess;
  if (es == 1 && t.subf_u8 != 1) return cudaSuccess;
  if (reinterpret_cast<uintptr_t>(codes) & (uintptr_t)(t.C / 2 - 1)) return cudaSuccess;
  if constexpr (es == 1) {
    if (knob_bq()) {
      cudaError_t e = u8_rows(t, nullptr, A, N, lda, nullptr, 0, codes, st, done);
      if (*done || e != cudaSuccess) return e;
    }
  }
  const int pitch_e = es == 1 ? t.D : t.D + 16 / es;
  const int stage_b = ((R * pitch_e * es) + 127) & ~127;
  const size_t fixed = 256;                          // barriers only (kernel's OFF_STAGE)
  size_t budget = (size_t)dev_info().smem_optin;
  if (es == 1 && MDN_RT_CTAS_U8 > 1) budget = std::min(budget, (size_t)(233472 / MDN_RT_CTAS_U8 - 1024));
  constexpr int NG = ng_of<TIn, true>();
  int NS = (int)((budget - fixed) / stage_b);
  if (NS > NS_MAX) NS = NS_MAX;
  NS -= NS % NG;
  if (NS < NG) return cudaSuccess;
  CUtensorMap tm;
  if (!make_tmap(&tm, A, N, lda, t.D, es == 1 ? t.D - 16 : t.D, R, es)) return cudaSuccess;
  SParams p{};
  p.N = N;
  p.n_tiles = (N + R - 1) / R;
  p.pitch_e = pitch_e;
  p.stage_b = stage_b;
  p.NS = NS;
  p.dims = t.dims;
  p.sub = t.sub;
  p.thr = t.thr;
  p.q = t.q;
  p.codes = codes;
  const size_t smem = fixed + (size_t)NS * stage_b;
  const bool bq = es == 1 && t.q_byte && knob_bq();
  *done = true;
  if constexpr (es == 1) {
    if (bq) return t.C == 4 ? launch_enc<TIn, 4, true>(tm, p, smem, st) : launch_enc<TIn, 8, true>(tm, p, smem, st);
  }
  return t.C == 4 ? launch_enc<TIn, 4, false>(tm, p, smem, st) : launch_enc<TIn, 8, false>(tm, p, smem, st);
}

cudaError_t launch_encode_rt(const TreesDev& t, const float* A, int64_t N, int64_t lda,
                             uint8_t* codes, cudaStream_t st, bool* done) {
  return encode_rt<float>(t, A, N, lda, codes, st, done);
}

cudaError_t launch_encode_rt_u8(const TreesDev& t, const uint8_t* A, int64_t N, int64_t lda,
                                uint8_t* codes, cudaStream_t st, bool* done) {
  return encode_rt<uint8_t>(t, A, N, lda, codes, st, done);
}

cudaError_t launch_amm_rt(const TreesDev& t, const LutsDev& l, const float* A, int64_t N,
                          int64_t lda, float* out, int64_t ldo, cudaStream_t st, bool* done) {
  return amm_rt<float>(t, l, A, N, lda, out, ldo, st, done);
}

cudaError_t launch_amm_rt_u8(const TreesDev& t, const LutsDev& l, const uint8_t* A, int64_t N,
                             int64_t lda, float* out, int64_t ldo, cudaStream_t st, bool* done) {
  return amm_rt<uint8_t>(t, l, A, N, lda, out, ldo, st, done);
}

bool amm_rt_applies(const TreesDev& t, const LutsDev& l, int es) {
  return rt_ok(t, l, reinterpret_cast<const void*>(256), t.D, es);
}

}  // namespace mdn
