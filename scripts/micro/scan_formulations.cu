// Microbenchmark: exact-mode cls100 scan (C=32, W=25, M=100) formulations.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -o scanbench scanbench.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <vector>
#include <algorithm>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)

constexpr int C = 32, W = 25, M = 100, W2 = (W + 1) / 2;
static __constant__ uint32_t k_one = 1u;

__device__ __forceinline__ uint32_t mad_add(uint32_t acc, uint32_t x, uint32_t one) {
  uint32_t r;
  asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(r) : "r"(x), "r"(one), "r"(acc));
  return r;
}
__device__ __forceinline__ uint64_t mad_wide_add(uint64_t acc, uint32_t x, uint32_t one) {
  uint64_t r;
  asm("mad.wide.u32 %0, %1, %2, %3;" : "=l"(r) : "r"(x), "r"(one), "l"(acc));
  return r;
}

__device__ __forceinline__ uint32_t dp4a(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t r;
  asm("dp4a.u32.u32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(c));
  return r;
}
static __constant__ uint32_t k_one24 = 1u << 24;
__device__ __forceinline__ uint32_t mad_hi_add(uint32_t acc, uint32_t x, uint32_t m) {
  uint32_t r;
  asm("mad.hi.u32 %0, %1, %2, %3;" : "=r"(r) : "r"(x), "r"(m), "r"(acc));
  return r;
}

__device__ __forceinline__ void store_row(float* o, const uint32_t (&ae)[W], const uint32_t (&ao)[W], float a, float b) {
#pragma unroll
  for (int w = 0; w < W; ++w) {
    float4 f;
    f.x = __fmaf_rn(a, (float)(ae[w] & 0xFFFFu), b);
    f.y = __fmaf_rn(a, (float)(ao[w] & 0xFFFFu), b);
    f.z = __fmaf_rn(a, (float)(ae[w] >> 16), b);
    f.w = __fmaf_rn(a, (float)(ao[w] >> 16), b);
    *reinterpret_cast<float4*>(o + 4 * w) = f;
  }
}

// V: 0 baseline (MIX 3); 1 rolled e IADD raw WIDE; 2 rolled e IMAD raw WIDE;
// 3 rolled alternating; 4 = 3 with LDS.64; 5 = 1 with LDS.64; 6 unrolled pairs raw (ptxas IADD3.X)
// 7 = rolled pairs of codebooks, e IADD3, raw WIDE on two accumulator sets? (no) -> rolled 2 cb, raw WIDE per cb with separate asm volatile
template <int V, int MB>
__global__ void __launch_bounds__(256, MB) k_scan(const uint32_t* __restrict__ lut_g, const uint4* __restrict__ codes,
                                              int64_t N, float* __restrict__ out, float a, float b) {
  extern __shared__ __align__(16) uint32_t s_lut[];
  constexpr int NWORDS = (V == 5) ? C * W2 * 32 : C * W * 16;
  for (int i = threadIdx.x; i < NWORDS; i += blockDim.x) s_lut[i] = lut_g[i];
  __syncthreads();
  const uint32_t one = k_one, one24 = k_one24;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t row = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; row < N; row += stride) {
    const uint4 cv = __ldg(codes + row);
    const uint32_t cw[4] = {cv.x, cv.y, cv.z, cv.w};
    uint32_t ae[W], ao[W];
#pragma unroll
    for (int w = 0; w < W; ++w) ae[w] = ao[w] = 0u;
    if constexpr (V == 0) {
#pragma unroll 1
      for (int g = 0; g < 4; ++g) {
        uint32_t c0 = cw[0];
        c0 = g == 1 ? cw[1] : c0; c0 = g == 2 ? cw[2] : c0; c0 = g == 3 ? cw[3] : c0;
        const uint32_t* lg = s_lut + g * 8 * W * 16;
#pragma unroll
        for (int i = 0; i < 8; i += 2) {
          const uint32_t* p0 = lg + (i * W) * 16 + ((c0 >> (4 * i)) & 15u);
          const uint32_t* p1 = lg + ((i + 1) * W) * 16 + ((c0 >> (4 * i + 4)) & 15u);
#pragma unroll
          for (int w = 0; w < W; ++w) {
            const uint32_t x = p0[w * 16], y = p1[w * 16];
            if (w % 3 == 0) {
              ae[w] += (x & 0x00FF00FFu) + (y & 0x00FF00FFu);
              ao[w] += __byte_perm(x, 0u, 0x4341) + __byte_perm(y, 0u, 0x4341);
            } else {
              ae[w] = mad_add(mad_add(ae[w], x & 0x00FF00FFu, one), y & 0x00FF00FFu, one);
              ao[w] = mad_add(mad_add(ao[w], __byte_perm(x, 0u, 0x4341), one), __byte_perm(y, 0u, 0x4341), one);
            }
          }
        }
      }
    } else {
      // E = sum (w & 0x00FF00FF) = S0 + 2^16 S2; B = sum (w >> 8) = S1 + 2^8 S2 + 2^16 S3
      uint32_t r3[W];
#pragma unroll
      for (int w = 0; w < W; ++w) r3[w] = 0u;
#pragma unroll 1
      for (int g = 0; g < 4; ++g) {
        uint32_t c0 = cw[0];
        c0 = g == 1 ? cw[1] : c0; c0 = g == 2 ? cw[2] : c0; c0 = g == 3 ? cw[3] : c0;
        if constexpr (V == 5) {
          const uint2* lg = reinterpret_cast<const uint2*>(s_lut) + g * 8 * W2 * 16;
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const uint2* p = lg + (i * W2) * 16 + ((c0 >> (4 * i)) & 15u);
#pragma unroll
            for (int w2 = 0; w2 < W2; ++w2) {
              const uint2 v = p[w2 * 16];
#pragma unroll
              for (int h = 0; h < 2; ++h) {
                const int w = 2 * w2 + h;
                if (w < W) {
                  const uint32_t x = h ? v.y : v.x;
                  ae[w] = mad_add(ae[w], x & 0x00FF00FFu, one);
                  ao[w] += x >> 8;
                }
              }
            }
          }
        } else {
        const uint32_t* lg = s_lut + g * 8 * W * 16;
#pragma unroll
        for (int i = 0; i < 8; i += 2) {
          const uint32_t* p0 = lg + (i * W) * 16 + ((c0 >> (4 * i)) & 15u);
          const uint32_t* p1 = lg + ((i + 1) * W) * 16 + ((c0 >> (4 * i + 4)) & 15u);
#pragma unroll
          for (int w = 0; w < W; ++w) {
            const uint32_t x = p0[w * 16], y = p1[w * 16];
            if constexpr (V == 1) {
              ae[w] = mad_add(mad_add(ae[w], x & 0x00FF00FFu, one), y & 0x00FF00FFu, one);
              ao[w] += x >> 8;
              ao[w] += y >> 8;
            } else if constexpr (V == 2) {
              ae[w] += (x & 0x00FF00FFu) + (y & 0x00FF00FFu);
              ao[w] += x >> 8;
              ao[w] += y >> 8;
            } else if constexpr (V == 3) {
              if (w & 1) ae[w] += (x & 0x00FF00FFu) + (y & 0x00FF00FFu);
              else ae[w] = mad_add(mad_add(ae[w], x & 0x00FF00FFu, one), y & 0x00FF00FFu, one);
              ao[w] += x >> 8;
              ao[w] += y >> 8;
            } else if constexpr (V == 4) {
              ae[w] += (x & 0x00FF00FFu) + (y & 0x00FF00FFu);
              ao[w] = mad_hi_add(mad_hi_add(ao[w], x, one24), y, one24);
            } else if constexpr (V == 7) {   // D1: raw r0 (in ao), S3 via dp4a (in r3)
              ae[w] += (x & 0x00FF00FFu) + (y & 0x00FF00FFu);
              ao[w] += x + y;
              r3[w] = dp4a(y, 0x01000000u, dp4a(x, 0x01000000u, r3[w]));
            } else if constexpr (V == 8) {   // D3: S1 via dp4a (ao), S3 via dp4a (r3)
              ae[w] += (x & 0x00FF00FFu) + (y & 0x00FF00FFu);
              ao[w] = dp4a(y, 0x00000100u, dp4a(x, 0x00000100u, ao[w]));
              r3[w] = dp4a(y, 0x01000000u, dp4a(x, 0x01000000u, r3[w]));
            } else if constexpr (V == 9) {   // D1 with IMAD e-adds
              ae[w] = mad_add(mad_add(ae[w], x & 0x00FF00FFu, one), y & 0x00FF00FFu, one);
              ao[w] += x + y;
              r3[w] = dp4a(y, 0x01000000u, dp4a(x, 0x01000000u, r3[w]));
            } else {  // V6: e IADD3 pairs, o alternate LEA / IMAD.HI
              ae[w] += (x & 0x00FF00FFu) + (y & 0x00FF00FFu);
              if (w % 3 == 0) ao[w] = mad_hi_add(mad_hi_add(ao[w], x, one24), y, one24);
              else { ao[w] += x >> 8; ao[w] += y >> 8; }
            }
          }
        }
        }
      }
      if constexpr (V == 7 || V == 9) {
#pragma unroll
        for (int w = 0; w < W; ++w) ao[w] = (((ao[w] - ae[w]) >> 8) & 0xFFFFu) | (r3[w] << 16);
      } else if constexpr (V == 8) {
#pragma unroll
        for (int w = 0; w < W; ++w) ao[w] |= r3[w] << 16;
      } else {
#pragma unroll
        for (int w = 0; w < W; ++w) ao[w] -= (ae[w] & 0xFFFF0000u) >> 8;
      }
    }
    store_row(out + row * M, ae, ao, a, b);
  }
}

template <int V, int MB = 1>
float run(const uint32_t* lut, const uint32_t* lut64, const uint4* codes, int64_t N, float* out, int sms, int reps) {
  auto k = k_scan<V, MB>;
  const size_t smem = (V == 5) ? (size_t)C * W2 * 32 * 4 : (size_t)C * W * 16 * 4;
  CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int per_sm = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, 256, smem));
  int64_t blocks = std::min<int64_t>((N + 255) / 256, (int64_t)sms * per_sm);
  const uint32_t* l = (V == 5) ? lut64 : lut;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  std::vector<float> ts;
  for (int r = 0; r < reps + 2; ++r) {
    cudaEventRecord(e0);
    k<<<(unsigned)blocks, 256, smem>>>(l, codes, N, out, 0.5f, -3.0f);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    if (r >= 2) ts.push_back(ms);
  }
  CK(cudaGetLastError());
  std::sort(ts.begin(), ts.end());
  cudaFuncAttributes fa; cudaFuncGetAttributes(&fa, k);
  printf("V%d/MB%d regs=%d blocks/SM=%d  best %.3f ms  median %.3f ms  -> %.3e rows/s (median)\n", V, MB, fa.numRegs, per_sm,
         ts[0], ts[ts.size() / 2], N / (ts[ts.size() / 2] * 1e-3));
  return ts[ts.size() / 2];
}

int main() {
  const int64_t N = 1 << 21;
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  std::vector<uint8_t> tq((size_t)C * 16 * M);
  srand(1);
  for (auto& v : tq) v = (uint8_t)(rand() & 255);
  // words: [c][w][k] word = bytes m = 4w..4w+3 of code k
  std::vector<uint32_t> lw((size_t)C * W * 16, 0), l64((size_t)C * W2 * 32, 0);
  for (int c = 0; c < C; ++c)
    for (int k = 0; k < 16; ++k)
      for (int w = 0; w < W; ++w) {
        uint32_t x = 0;
        for (int j = 0; j < 4; ++j) {
          int m = 4 * w + j;
          if (m < M) x |= (uint32_t)tq[((size_t)c * 16 + k) * M + m] << (8 * j);
        }
        lw[((size_t)c * W + w) * 16 + k] = x;
        l64[(((size_t)c * W2 + w / 2) * 16 + k) * 2 + (w & 1)] = x;
      }
  std::vector<uint8_t> codes((size_t)N * 16);
  for (auto& v : codes) v = (uint8_t)(rand() & 255);
  uint32_t *d_l, *d_l64; uint4* d_c; float *d_o, *d_ref;
  CK(cudaMalloc(&d_l, lw.size() * 4)); CK(cudaMalloc(&d_l64, l64.size() * 4));
  CK(cudaMalloc(&d_c, codes.size())); CK(cudaMalloc(&d_o, (size_t)N * M * 4)); CK(cudaMalloc(&d_ref, (size_t)N * M * 4));
  CK(cudaMemcpy(d_l, lw.data(), lw.size() * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(d_l64, l64.data(), l64.size() * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(d_c, codes.data(), codes.size(), cudaMemcpyHostToDevice));
  const int reps = 20;
  run<0>(d_l, d_l64, d_c, N, d_ref, sms, reps);
  // host check of a few rows of the baseline
  {
    std::vector<float> o(64 * M);
    CK(cudaMemcpy(o.data(), d_ref, o.size() * 4, cudaMemcpyDeviceToHost));
    int bad = 0;
    for (int r = 0; r < 64; ++r)
      for (int m = 0; m < M; ++m) {
        int s = 0;
        for (int c = 0; c < C; ++c) {
          int k = (codes[(size_t)r * 16 + c / 2] >> (4 * (c & 1))) & 15;
          s += tq[((size_t)c * 16 + k) * M + m];
        }
        if (o[r * M + m] != 0.5f * s - 3.0f) ++bad;
      }
    printf("baseline host check: %d bad\n", bad);
  }
  auto cmp = [&](const char* name) {
    std::vector<uint32_t> x((size_t)N * M), y((size_t)N * M);
    CK(cudaMemcpy(x.data(), d_o, x.size() * 4, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(y.data(), d_ref, y.size() * 4, cudaMemcpyDeviceToHost));
    size_t bad = 0;
    for (size_t i = 0; i < x.size(); ++i) bad += x[i] != y[i];
    printf("  %s mismatches: %zu\n", name, bad);
  };
  run<7>(d_l, d_l64, d_c, N, d_o, sms, reps); cmp("V7");
  run<8>(d_l, d_l64, d_c, N, d_o, sms, reps); cmp("V8");
  run<9>(d_l, d_l64, d_c, N, d_o, sms, reps); cmp("V9");
  run<1>(d_l, d_l64, d_c, N, d_o, sms, reps); cmp("V1");
  run<0>(d_l, d_l64, d_c, N, d_o, sms, reps); cmp("V0");
  return 0;
}
