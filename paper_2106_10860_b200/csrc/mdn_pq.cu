// Product Quantization encoder: the comparator MADDNESS replaces.
//
// g^(c)(a) = argmin_k sum_{j in J^(c)} (a_j - P^(c)_{k,j})^2  (PAPER.md Eq.
// pqLoss, L182-184), K = 16 prototypes per subspace learned offline by
// K-means (L155-163; oracle/pq.py). The codes use the same 4-bit packing as
// mdn_encode and feed the same mdn_scan / tables (h(B) from the dense P).
//
// Floating point decides the integer code. The oracle takes the first argmin
// of the fp64 definition; this kernel evaluates the argmin-invariant expanded
// form e_k = ||p_k||^2 - 2 <a, p_k> (||a||^2 is common to every k) in fp32
// with fused multiply-adds, and DESIGN.md reading P1 accepts its code iff the
// code's fp64 distance is within the fp32 rounding bound of the minimum
// (oracle.check_pq_codes); ties go to the lowest k.
//
// k_encode_pq<DS, R>: a thread owns one codebook c (lane % C) and R rows; the
// 16 x DS scaled prototypes q = -2 p of c are read from shared memory (layout
// [k][j/4][c][4]: one conflict-free LDS.128 per 4 dims, reused for the R
// rows) next to ||p_k||^2 ([k][c]); one FFMA per (row, prototype, dim), two
// accumulator chains per row: 16 D FMAs per row (cls100: 8,192), so the
// kernel is bound by HBM (4 D bytes per row) or by the fp32 pipe, whichever
// is nearer (Sec. 5.1).
#include <cuda_runtime.h>

#include "mdn_internal.h"
#include "mdn_tma.cuh"

namespace mdn {
namespace fast {
namespace pq {

constexpr int THREADS = 256;
#ifndef MDN_PQ_PF
// prefetch the next row group's x while this one is encoded: cost 25-30%
// (more registers, fewer resident warps) on every config; off
#define MDN_PQ_PF 0
#endif
// Also measured and rejected: packed fp32x2 FMAs (FFMA2, row pairs, the
// prototype value as the broadcast scalar operand -- half the FMA
// instructions) ran at 0.75 of the scalar-FFMA kernel (cls100 1.32 vs 1.76e9,
// scale 2.36 vs 3.11e9, tiny 1.87 vs 2.50e10 rows/s): FFMA2 does not double
// the fp32 rate and halves the independent accumulator chains.
#ifndef MDN_PQ_R4
#define MDN_PQ_R4 8     // rows per thread for 4-column subspaces
#endif
#ifndef MDN_PQ_R8
#define MDN_PQ_R8 8
#endif
#ifndef MDN_PQ_R16
#define MDN_PQ_R16 4    // (2 rows: cls100 1.37 vs 1.76e9 rows/s)
#endif
#ifndef MDN_PQ_R32
#define MDN_PQ_R32 2
#endif

template <int DS, int R>
__device__ __forceinline__ void load_x(const float* __restrict__ A, int64_t N, int64_t lda, int c,
                                       int64_t row0, float (&x)[R][DS]) {
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int64_t row = row0 + r < N ? row0 + r : N - 1;       // clamp the tail (not stored)
    const float4* src = reinterpret_cast<const float4*>(A + row * lda + (int64_t)c * DS);
#pragma unroll
    for (int j4 = 0; j4 < DS / 4; ++j4) {
      const float4 v = __ldg(src + j4);
      x[r][4 * j4] = v.x, x[r][4 * j4 + 1] = v.y, x[r][4 * j4 + 2] = v.z, x[r][4 * j4 + 3] = v.w;
    }
  }
}

template <int DS, int R>
__global__ void __launch_bounds__(THREADS) k_encode_pq(const float* __restrict__ A, int64_t N,
                                                       int64_t lda, int C,
                                                       const float4* __restrict__ cent_g,
                                                       uint8_t* __restrict__ codes) {
  extern __shared__ __align__(16) unsigned char smem[];
  float4* s_cent = reinterpret_cast<float4*>(smem);             // [16][DS/4][C] of -2 p
  const int n4 = 16 * (DS / 4) * C + 4 * C;                     // + ||p||^2 [16][C]
  for (int i = threadIdx.x; i < n4; i += blockDim.x) s_cent[i] = cent_g[i];
  __syncthreads();
  const float* s_pn = reinterpret_cast<const float*>(s_cent + 16 * (DS / 4) * C);
  const int c = threadIdx.x % C;
  const int rg = threadIdx.x / C;
  const int groups_per_block = THREADS / C;
  const int64_t rows_per_block = (int64_t)groups_per_block * R;
  // Block-uniform trip count (the code packing shuffles need every lane).
  const int64_t step = (int64_t)gridDim.x * rows_per_block;
  float x[R][DS];
  if (MDN_PQ_PF) load_x<DS, R>(A, N, lda, c, (int64_t)blockIdx.x * rows_per_block + (int64_t)rg * R, x);
  for (int64_t base = (int64_t)blockIdx.x * rows_per_block; base < N; base += step) {
    const int64_t row0 = base + (int64_t)rg * R;
    float xn[MDN_PQ_PF ? R : 1][MDN_PQ_PF ? DS : 1];
    if constexpr (MDN_PQ_PF) {
      if (base + step < N) load_x<DS, R>(A, N, lda, c, row0 + step, xn);
    } else {
      load_x<DS, R>(A, N, lda, c, row0, x);
    }
    float best[R];
    uint32_t bk[R];
#pragma unroll
    for (int r = 0; r < R; ++r) best[r] = __int_as_float(0x7f800000), bk[r] = 0u;   // +inf
#pragma unroll 1
    for (int k = 0; k < 16; ++k) {
      float d0[R], d1[R];
      const float pn = s_pn[k * C + c];
#pragma unroll
      for (int r = 0; r < R; ++r) d0[r] = pn, d1[r] = 0.f;
#pragma unroll
      for (int j4 = 0; j4 < DS / 4; ++j4) {
        const float4 q = s_cent[(k * (DS / 4) + j4) * C + c];
#pragma unroll
        for (int r = 0; r < R; ++r) {
          d0[r] = __fmaf_rn(x[r][4 * j4], q.x, d0[r]);
          d1[r] = __fmaf_rn(x[r][4 * j4 + 1], q.y, d1[r]);
          d0[r] = __fmaf_rn(x[r][4 * j4 + 2], q.z, d0[r]);
          d1[r] = __fmaf_rn(x[r][4 * j4 + 3], q.w, d1[r]);
        }
      }
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const float d = __fadd_rn(d0[r], d1[r]);
        if (d < best[r]) best[r] = d, bk[r] = (uint32_t)k;     // strict: ties keep the lowest k
      }
    }
    // pack two codes per byte: low nibble = even codebook (L147, L608)
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const uint32_t hi = __shfl_down_sync(0xffffffffu, bk[r], 1);
      if ((c & 1) == 0 && row0 + r < N)
        codes[(row0 + r) * (C / 2) + c / 2] = (uint8_t)(bk[r] | (hi << 4));
    }
    if constexpr (MDN_PQ_PF) {
#pragma unroll
      for (int r = 0; r < R; ++r)
#pragma unroll
        for (int j = 0; j < DS; ++j) x[r][j] = xn[r % (MDN_PQ_PF ? R : 1)][j % (MDN_PQ_PF ? DS : 1)];
    }
  }
}

// Which kernel per subspace width (same box, rows/s, lane-per-row R = 4 vs
// lane-per-codebook): DS = 32 (cls10_c16) 1.63 vs 1.10e9; DS = 16 (cls100)
// 1.65 vs 1.76e9; DS = 8 (scale) 2.98 vs 3.16e9; DS = 4 (tiny) 2.45 vs
// 2.50e10 (lane-per-row R = 1 / 2 slower still). MDN_PQ_ROWS (build flag)
// forces one kernel for A/B.
template <int DS>
constexpr bool pq_rows_kernel() {
#ifdef MDN_PQ_ROWS
  return MDN_PQ_ROWS != 0;
#else
  return DS == 32;
#endif
}
#ifndef MDN_PQ_RR
#define MDN_PQ_RR 4     // rows per lane of the lane-per-row kernel
#endif

// k_encode_pq_rows<DS, R>: a warp takes one codebook pair (2p, 2p + 1) of 32 R
// consecutive rows, lane l rows l, l + 32, ...: every prototype read is a
// warp-uniform shared-memory broadcast (one wavefront per LDS.128, 4 R FFMAs
// each), so the fp32 pipe, not shared-memory bandwidth, bounds the inner loop;
// the row's subspace comes straight from global memory (each row's DS floats
// are one or two 32-B sectors, reused across the float4 loads through L1).
template <int DS, int R>
__global__ void __launch_bounds__(THREADS) k_encode_pq_rows(const float* __restrict__ A, int64_t N,
                                                            int64_t lda, int C,
                                                            const float4* __restrict__ cent_g,
                                                            uint8_t* __restrict__ codes) {
  extern __shared__ __align__(16) unsigned char smem[];
  float4* s_cent = reinterpret_cast<float4*>(smem);             // [16][DS/4][C] of -2 p
  const int n4 = 16 * (DS / 4) * C + 4 * C;                     // + ||p||^2 [16][C]
  for (int i = threadIdx.x; i < n4; i += blockDim.x) s_cent[i] = cent_g[i];
  __syncthreads();
  const float* s_pn = reinterpret_cast<const float*>(s_cent + 16 * (DS / 4) * C);
  const int lane = threadIdx.x & 31;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t n_warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int n_pairs = C / 2;
  const int64_t n_tiles = (N + 32 * R - 1) / (32 * R);
  for (int64_t item = gw; item < n_tiles * n_pairs; item += n_warps) {
    const int64_t tile = item / n_pairs;
    const int pair = (int)(item % n_pairs);
    uint32_t code[R];
#pragma unroll
    for (int r = 0; r < R; ++r) code[r] = 0u;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int c = 2 * pair + h;
      float x[R][DS];
#pragma unroll
      for (int r = 0; r < R; ++r) {
        int64_t row = tile * 32 * R + r * 32 + lane;
        row = row < N ? row : N - 1;                          // clamp the tail (not stored)
        const float4* src = reinterpret_cast<const float4*>(A + row * lda + (int64_t)c * DS);
#pragma unroll
        for (int j4 = 0; j4 < DS / 4; ++j4) {
          const float4 v = __ldg(src + j4);
          x[r][4 * j4] = v.x, x[r][4 * j4 + 1] = v.y, x[r][4 * j4 + 2] = v.z, x[r][4 * j4 + 3] = v.w;
        }
      }
      float best[R];
      uint32_t bk[R];
#pragma unroll
      for (int r = 0; r < R; ++r) best[r] = __int_as_float(0x7f800000), bk[r] = 0u;   // +inf
#pragma unroll 2
      for (int k = 0; k < 16; ++k) {
        float d0[R], d1[R];
        const float pn = s_pn[k * C + c];
#pragma unroll
        for (int r = 0; r < R; ++r) d0[r] = pn, d1[r] = 0.f;
#pragma unroll
        for (int j4 = 0; j4 < DS / 4; ++j4) {
          const float4 q = s_cent[(k * (DS / 4) + j4) * C + c];    // warp-uniform: broadcast
#pragma unroll
          for (int r = 0; r < R; ++r) {
            d0[r] = __fmaf_rn(x[r][4 * j4], q.x, d0[r]);
            d1[r] = __fmaf_rn(x[r][4 * j4 + 1], q.y, d1[r]);
            d0[r] = __fmaf_rn(x[r][4 * j4 + 2], q.z, d0[r]);
            d1[r] = __fmaf_rn(x[r][4 * j4 + 3], q.w, d1[r]);
          }
        }
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const float d = __fadd_rn(d0[r], d1[r]);
          if (d < best[r]) best[r] = d, bk[r] = (uint32_t)k;   // strict: ties keep the lowest k
        }
      }
#pragma unroll
      for (int r = 0; r < R; ++r) code[r] |= bk[r] << (4 * h);   // low nibble = even codebook
    }
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int64_t row = tile * 32 * R + r * 32 + lane;
      if (row < N) codes[row * n_pairs + pair] = (uint8_t)code[r];
    }
  }
}

// Any subspace layout / C: thread per (row, codebook), prototypes from the
// dense P in global memory.
__global__ void k_encode_pq_generic(const float* __restrict__ A, int64_t N, int64_t lda, int C,
                                    int D, const uint16_t* __restrict__ sub_b,
                                    const uint16_t* __restrict__ sub_e,
                                    const float* __restrict__ P, uint8_t* __restrict__ codes) {
  const int nb = (C + 1) / 2;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < N * nb;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = i / nb;
    const int pair = (int)(i % nb);
    uint32_t out = 0;
    for (int h = 0; h < 2; ++h) {
      const int c = 2 * pair + h;
      if (c >= C) break;
      float best = __int_as_float(0x7f800000);
      uint32_t bk = 0;
      for (int k = 0; k < 16; ++k) {
        float d = 0.f;
        for (int j = sub_b[c]; j < sub_e[c]; ++j) {
          const float t = __fsub_rn(A[row * lda + j], P[(int64_t)(16 * c + k) * D + j]);
          d = __fadd_rn(d, __fmul_rn(t, t));
        }
        if (d < best) best = d, bk = (uint32_t)k;
      }
      out |= bk << (4 * h);
    }
    codes[row * nb + pair] = (uint8_t)out;
  }
}

template <int DS, int R>
cudaError_t launch(const float* A, int64_t N, int64_t lda, int C, const float* cent,
                   uint8_t* codes, cudaStream_t s) {
  if constexpr (pq_rows_kernel<DS>()) {
    auto k = k_encode_pq_rows<DS, MDN_PQ_RR>;
    const size_t smem = ((size_t)16 * DS * C + 16 * C) * 4;
    cudaError_t e = ensure_smem(reinterpret_cast<const void*>(k), smem);
    if (e != cudaSuccess) return e;
    int per_sm = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, THREADS, smem);
    if (e != cudaSuccess) return e;
    if (per_sm < 1) per_sm = 1;
    const int64_t items = (N + 32 * MDN_PQ_RR - 1) / (32 * MDN_PQ_RR) * (C / 2);
    int64_t blocks = (items + THREADS / 32 - 1) / (THREADS / 32);
    const int64_t cap = (int64_t)dev_info().sms * per_sm;
    if (blocks > cap) blocks = cap;
    k<<<(unsigned)blocks, THREADS, smem, s>>>(A, N, lda, C, reinterpret_cast<const float4*>(cent),
                                              codes);
    return cudaGetLastError();
  }
  auto k = k_encode_pq<DS, R>;
  const size_t smem = ((size_t)16 * DS * C + 16 * C) * 4;
  cudaError_t e = ensure_smem(reinterpret_cast<const void*>(k), smem);
  if (e != cudaSuccess) return e;
  int per_sm = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, THREADS, smem);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) per_sm = 1;
  const int64_t rows_per_block = (int64_t)(THREADS / C) * R;
  int64_t blocks = (N + rows_per_block - 1) / rows_per_block;
  const int64_t cap = (int64_t)dev_info().sms * per_sm;
  if (blocks > cap) blocks = cap;
  k<<<(unsigned)blocks, THREADS, smem, s>>>(A, N, lda, C, reinterpret_cast<const float4*>(cent),
                                            codes);
  return cudaGetLastError();
}

}  // namespace pq
}  // namespace fast

using namespace fast::pq;

// t.pq_cent: [16][DS/4][C][4] scaled prototypes -2 p, then ||p||^2 [16][C], when every subspace is [c DS, (c+1) DS)
// with DS in {4, 8, 16, 32} and THREADS % C == 0 (else null: generic kernel).
cudaError_t launch_encode_pq(const TreesDev& t, const float* P_dense, const uint16_t* sub_b,
                             const uint16_t* sub_e, const float* A, int64_t N, int64_t lda,
                             uint8_t* codes, cudaStream_t s) {
  const bool fast_ok = t.pq_cent && t.pq_ds > 0 && (reinterpret_cast<uintptr_t>(A) & 15u) == 0 &&
                       lda % 4 == 0 && t.C % 2 == 0 &&
                       ((size_t)16 * t.pq_ds * t.C + 16 * t.C) * 4 <= (size_t)fast::dev_info().smem_optin;
  if (fast_ok) {
    switch (t.pq_ds) {
      case 4: return launch<4, MDN_PQ_R4>(A, N, lda, t.C, t.pq_cent, codes, s);
      case 8: return launch<8, MDN_PQ_R8>(A, N, lda, t.C, t.pq_cent, codes, s);
      case 16: return launch<16, MDN_PQ_R16>(A, N, lda, t.C, t.pq_cent, codes, s);
      case 32: return launch<32, MDN_PQ_R32>(A, N, lda, t.C, t.pq_cent, codes, s);
    }
  }
  const int64_t work = N * ((t.C + 1) / 2);
  int64_t blocks = (work + 255) / 256;
  const int64_t cap = (int64_t)fast::dev_info().sms * 8;
  if (blocks > cap) blocks = cap;
  k_encode_pq_generic<<<(unsigned)blocks, 256, 0, s>>>(A, N, lda, t.C, t.D, sub_b, sub_e, P_dense,
                                                      codes);
  return cudaGetLastError();
}

}  // namespace mdn
