// Scan core shared by the TMA-fed fused kernel (mdn_fast.cu) and the
// column-major kernel (mdn_colmajor.cu): table lookups of 32-bit words holding
// 4 output columns, exact 16-bit SWAR sums or the App. D averaging tree, and
// the dequantising row store.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace mdn {
namespace fast {

// ------------------------------------------------------------ scan core --

// Accumulate the W table words of every codebook for one row.
//   words(g): the g-th 32-bit word of the row's packed codes (8 codes, low
//   nibble first; for C < 8 only the low 4C bits are used).
// Exact mode (U == 0): ae[w] / ao[w] hold the even / odd output columns of
// word w in two 16-bit lanes (S <= 255 C < 2^16 for C <= 256).
// Averaging mode: per block of U consecutive codebooks the halves-recursion
// tree of rounded averages (mu(a,b) = (a+b+1)>>1 per byte, avg8), and the
// block results are summed exactly (App. D, reading R16/R17).
// mu(a, b) = floor((a + b + 1) / 2) on 4 byte lanes (App. D) as
// (a | b) - (((a ^ b) & 0xFE..) >> 1): per byte a | b = (a & b) + (a ^ b) can
// never borrow, and the mask keeps each byte's low bit from shifting into its
// neighbour. 4 ALU ops (LOP3, LOP3, SHF, IADD) against 5 for __vavgu4.
__device__ __forceinline__ uint32_t avg8(uint32_t a, uint32_t b) {
  uint32_t x;   // (a ^ b) & 0xFEFEFEFE in one LOP3 (inline: LLVM would re-canonicalise it)
  asm("lop3.b32 %0, %1, %2, %3, 0x28;" : "=r"(x) : "r"(a), "r"(b), "r"(0xFEFEFEFEu));
  return (a | b) - (x >> 1);
}

// Three-instruction form (MDN_AVG_LEA, default). On complemented bytes the
// rounded-up average is the rounded-down one: 255 - mu(a, b) = floor(((255 -
// a) + (255 - b)) / 2) = (a' & b') + (((a' ^ b') & 0xFE..) >> 1), and ptxas
// fuses the shift and the add into one LEA.HI (the subtraction of avg8 does
// not fuse): LOP3, LOP3, LEA.HI. avg8_c1 takes raw a, b (a' & b' = ~(a | b),
// a' ^ b' = a ^ b) and returns the complemented average; avg8_c takes and
// returns complemented values. The tree's root stays complemented and is
// SUBTRACTED from lane sums pre-loaded with 255 per block (scan_core), so no
// instruction is spent on complementing. Bit-identical to avg8 (R16/R17).
#ifndef MDN_AVG_LEA
#define MDN_AVG_LEA 1
#endif
__device__ __forceinline__ uint32_t avg8_c1(uint32_t a, uint32_t b) {
  uint32_t x, n;
  asm("lop3.b32 %0, %1, %2, %3, 0x28;" : "=r"(x) : "r"(a), "r"(b), "r"(0xFEFEFEFEu));
  asm("lop3.b32 %0, %1, %2, %3, 0x03;" : "=r"(n) : "r"(a), "r"(b), "r"(0u));
  return n + (x >> 1);
}
__device__ __forceinline__ uint32_t avg8_c(uint32_t a, uint32_t b) {
  uint32_t x;
  asm("lop3.b32 %0, %1, %2, %3, 0x28;" : "=r"(x) : "r"(a), "r"(b), "r"(0xFEFEFEFEu));
  return (a & b) + (x >> 1);
}

// Pipe balancing. The exact accumulate is LOP/PRMT (split a word into its
// even and odd byte lanes) + adds, all on the ALU pipe by default, which then
// saturates (ncu: ALU 73%, issue 51% on cls100 mdn_scan) while the FMA pipe
// idles. An add written as mad.lo with a multiplier ptxas cannot see (k_one,
// a __constant__ 1 it cannot fold) stays an IMAD on the FMA pipe. Per pair of
// words: ALU-only = 2 LDS + 6 ALU; IMAD form = 2 LDS + 4 ALU + 4 FMA. Mixing
// one ALU-form word in three balances the two pipes against issue.
static __constant__ uint32_t k_one = 1u;

__device__ __forceinline__ uint32_t mad_add(uint32_t acc, uint32_t x, uint32_t one) {
  uint32_t r;
  asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(r) : "r"(x), "r"(one), "r"(acc));
  return r;
}

// Raw-word exact sums (MDN_SCAN_RAW, default). A table word holds 4 columns
// w = x0 + 2^8 x1 + 2^16 x2 + 2^24 x3; the odd bytes need their own 16-bit
// lanes, o = prmt(w, 0x4341) = x1 + 2^16 x3, but the even ones need not be
// split out at all: accumulating the RAW words, sum w = E + 2^8 O (mod 2^32)
// with E = E0 + 2^16 E2 and O = O1 + 2^16 O3 the even / odd lane sums, so
// E = sum w - 2^8 O (mod 2^32) is exact once per row and word (every lane
// sum <= 255 C < 2^16 for C <= 256, so E < 2^32). Per word one PRMT and two
// accumulations instead of a LOP3 mask, a PRMT and two accumulations.
#ifndef MDN_SCAN_RAW
#define MDN_SCAN_RAW 1
#endif

// MIX (exact mode): 0 = ALU only; k > 0 = every k-th word on the ALU, the rest
// IMAD adds (raw form: the odd-lane sums of those words as IMAD adds).
template <int C, int W, int U, bool UNROLL_G = false, int MIX = 0, class Words>
__device__ __forceinline__ void scan_core(const uint32_t* __restrict__ lut, Words words,
                                          uint32_t (&ae)[W], uint32_t (&ao)[W]) {
#pragma unroll
  for (int w = 0; w < W; ++w) ae[w] = ao[w] = 0u;
  const uint32_t one = k_one;
  if constexpr (U == 0) {
    constexpr int G = C >= 8 ? 8 : C;
    constexpr int NGU = UNROLL_G ? C / G : 1;
#pragma unroll NGU
    for (int g = 0; g < C / G; ++g) {
      const uint32_t cw = words(g);
      const uint32_t* lg = lut + g * G * W * 16;
#pragma unroll
      for (int i = 0; i < G; i += 2) {
        const uint32_t* p0 = lg + (i * W) * 16 + ((cw >> (4 * i)) & 15u);
        const uint32_t* p1 = lg + ((i + 1) * W) * 16 + ((cw >> (4 * i + 4)) & 15u);
#pragma unroll
        for (int w = 0; w < W; ++w) {
          const uint32_t a = p0[w * 16], b = p1[w * 16];
          if constexpr (MDN_SCAN_RAW != 0) {
            ae[w] += a + b;                            // raw words (ae = sum w until the fix-up)
            if (MIX == 0 || w % (MIX > 0 ? MIX : 1) == 0)
              ao[w] += __byte_perm(a, 0u, 0x4341) + __byte_perm(b, 0u, 0x4341);
            else
              ao[w] = mad_add(mad_add(ao[w], __byte_perm(a, 0u, 0x4341), one), __byte_perm(b, 0u, 0x4341), one);
          } else if (MIX == 0 || w % (MIX > 0 ? MIX : 1) == 0) {
            ae[w] += (a & 0x00FF00FFu) + (b & 0x00FF00FFu);
            ao[w] += __byte_perm(a, 0u, 0x4341) + __byte_perm(b, 0u, 0x4341);
          } else {
            ae[w] = mad_add(mad_add(ae[w], a & 0x00FF00FFu, one), b & 0x00FF00FFu, one);
            ao[w] = mad_add(mad_add(ao[w], __byte_perm(a, 0u, 0x4341), one), __byte_perm(b, 0u, 0x4341), one);
          }
        }
      }
    }
    if constexpr (MDN_SCAN_RAW != 0) {
#pragma unroll
      for (int w = 0; w < W; ++w) ae[w] -= ao[w] << 8;   // E = sum w - 2^8 O (mod 2^32)
    }
  } else {
    static_assert((U & (U - 1)) == 0 && C % U == 0, "U must be a power of two dividing C");
    constexpr int NBU = UNROLL_G ? C / U : 1;
    constexpr bool CPL = MDN_AVG_LEA != 0 && U >= 2;   // complemented tree roots
    if constexpr (CPL) {
      // every 16-bit lane starts 255 per block ahead and loses 255 - mu per
      // block: it never goes negative, so no lane borrows from its neighbour
#pragma unroll
      for (int w = 0; w < W; ++w) {
        ae[w] += (uint32_t)(255 * (C / U)) * 0x00010001u;
        ao[w] += (uint32_t)(255 * (C / U)) * 0x00010001u;
      }
    }
#pragma unroll NBU
    for (int blk = 0; blk < C / U; ++blk) {
      const uint32_t* p[U];
#pragma unroll
      for (int i = 0; i < U; ++i) {
        const int c = blk * U + i;  // runtime blk, static i
        uint32_t cw;
        if constexpr (U >= 8) {
          cw = words(blk * (U / 8) + i / 8);
          p[i] = lut + (c * W) * 16 + ((cw >> (4 * (i % 8))) & 15u);
        } else {
          const int cc = blk * U + i;
          cw = words(cc >> 3);
          p[i] = lut + (c * W) * 16 + ((cw >> (4 * (cc & 7))) & 15u);
        }
      }
#pragma unroll
      for (int w = 0; w < W; ++w) {
        uint32_t v[U];
#pragma unroll
        for (int i = 0; i < U; ++i) v[i] = p[i][w * 16];
#pragma unroll
        for (int s = 1; s < U; s *= 2)
#pragma unroll
          for (int i = 0; i < U; i += 2 * s) {
            if constexpr (!CPL) v[i] = avg8(v[i], v[i + s]);
            else v[i] = s == 1 ? avg8_c1(v[i], v[i + s]) : avg8_c(v[i], v[i + s]);
          }
        if constexpr (CPL) {
          ae[w] -= v[0] & 0x00FF00FFu;
          ao[w] -= __byte_perm(v[0], 0u, 0x4341);
        } else {
          ae[w] += v[0] & 0x00FF00FFu;
          ao[w] += __byte_perm(v[0], 0u, 0x4341);
        }
      }
    }
  }
}

// out[m] = fl32(alpha_eff * S'[m] + beta32): S' < 2^16 is exact in fp32 and
// alpha_eff a power of two, so the FMA's single rounding equals the oracle's.
// pair: (non-VEC) M even and the row 8-byte aligned -> 8-byte stores.
template <int W, bool VEC>
__device__ __forceinline__ void store_row(float* __restrict__ o, int M, const uint32_t (&ae)[W],
                                          const uint32_t (&ao)[W], float a, float b,
                                          bool pair = false) {
#pragma unroll
  for (int w = 0; w < W; ++w) {
    float4 f;
    f.x = __fmaf_rn(a, (float)(ae[w] & 0xFFFFu), b);
    f.y = __fmaf_rn(a, (float)(ao[w] & 0xFFFFu), b);
    f.z = __fmaf_rn(a, (float)(ae[w] >> 16), b);
    f.w = __fmaf_rn(a, (float)(ao[w] >> 16), b);
    if constexpr (VEC) {
      *reinterpret_cast<float4*>(o + 4 * w) = f;
    } else if (pair) {
      const int m = 4 * w;
      if (m + 1 < M) *reinterpret_cast<float2*>(o + m) = make_float2(f.x, f.y);
      if (m + 3 < M) *reinterpret_cast<float2*>(o + m + 2) = make_float2(f.z, f.w);
    } else {
      const int m = 4 * w;
      if (m + 0 < M) o[m + 0] = f.x;
      if (m + 1 < M) o[m + 1] = f.y;
      if (m + 2 < M) o[m + 2] = f.z;
      if (m + 3 < M) o[m + 3] = f.w;
    }
  }
}

template <int W>
__device__ __forceinline__ void store_sums(int32_t* __restrict__ o, int M, int scale,
                                           const uint32_t (&ae)[W], const uint32_t (&ao)[W]) {
#pragma unroll
  for (int w = 0; w < W; ++w) {
    const int m = 4 * w;
    const int v[4] = {(int)(ae[w] & 0xFFFFu), (int)(ao[w] & 0xFFFFu), (int)(ae[w] >> 16),
                      (int)(ao[w] >> 16)};
#pragma unroll
    for (int i = 0; i < 4; ++i)
      if (m + i < M) o[m + i] = v[i] * scale;
  }
}

}  // namespace fast
}  // namespace mdn
