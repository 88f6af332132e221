// Microbenchmark: the shared-memory load rate the table scan can reach on
// this GPU, with the scan's own access pattern (random 4-bit codes into
// 16-entry table rows laid out so that the 16 codes hit 16 distinct banks,
// one table row per (codebook, word)), and nothing else in the loop but the
// load and one XOR per loaded word (ALU: 1 LOP3 per LDS; the LDS is the
// bound if the crossbar is). Variants: 4-, 8- and 16-byte loads (the wider
// ones with the row layout [c][w/V][k][V] so a phase still covers 16
// distinct codes -> for 16-byte loads two codes per 4-bank group: conflicts
// by design, reported). Prints loaded bytes per clock per SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o lds_rate lds_rate.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)

constexpr int C = 32, W = 24;   // 24 words so every width divides it

template <int V>
__global__ void __launch_bounds__(512, 1) k_lds(const uint32_t* __restrict__ codes_g, uint32_t* out, int reps) {
  extern __shared__ __align__(16) uint32_t s[];
  for (int i = threadIdx.x; i < C * W * 16; i += blockDim.x) s[i] = i * 2654435761u;
  __syncthreads();
  uint32_t cw[4];
  for (int g = 0; g < 4; ++g) cw[g] = codes_g[(blockIdx.x * blockDim.x + threadIdx.x) * 4 + g];
  uint32_t acc0 = 0, acc1 = 0, acc2 = 0, acc3 = 0;
  for (int r = 0; r < reps; ++r) {
#pragma unroll 1
    for (int g = 0; g < 4; ++g) {
      const uint32_t c = cw[g] ^ (uint32_t)r;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int cb = g * 8 + i;
        const uint32_t k = (c >> (4 * i)) & 15u;
        if constexpr (V == 1) {
          const uint32_t* p = s + cb * W * 16 + k;
#pragma unroll
          for (int w = 0; w < W; ++w) acc0 ^= p[w * 16];
        } else if constexpr (V == 2) {
          const uint2* p = reinterpret_cast<const uint2*>(s) + cb * (W / 2) * 16 + k;
#pragma unroll
          for (int w = 0; w < W / 2; ++w) { const uint2 v = p[w * 16]; acc0 ^= v.x; acc1 ^= v.y; }
        } else {
          const uint4* p = reinterpret_cast<const uint4*>(s) + cb * (W / 4) * 16 + k;
#pragma unroll
          for (int w = 0; w < W / 4; ++w) {
            const uint4 v = p[w * 16];
            acc0 ^= v.x; acc1 ^= v.y; acc2 ^= v.z; acc3 ^= v.w;
          }
        }
      }
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc0 ^ acc1 ^ acc2 ^ acc3;
}

// The scan's arithmetic on top of the same loads (raw-word form): per word
// acc_w += w and acc_o += prmt(w, 0x4341), W accumulator pairs per thread.
// V = 5: adds as IADD3 (ALU); V = 6: odd-lane adds as IMAD (FMA pipe);
// V = 7: as 5 with 8-byte loads ([c][w/2][k][2] rows); V = 8: as 6 plus the
// real kernel's per-row float4 output stores (8 distinct row sets, > L2).
static __constant__ uint32_t k_one = 1u;
__device__ __forceinline__ uint32_t mad_add(uint32_t acc, uint32_t x, uint32_t one) {
  uint32_t r;
  asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(r) : "r"(x), "r"(one), "r"(acc));
  return r;
}
template <int V>
__global__ void __launch_bounds__(512, 1) k_scan(const uint32_t* __restrict__ codes_g, uint32_t* out, int reps) {
  extern __shared__ __align__(16) uint32_t s[];
  for (int i = threadIdx.x; i < C * W * 16; i += blockDim.x) s[i] = i * 2654435761u;
  __syncthreads();
  uint32_t cw[4];
  for (int g = 0; g < 4; ++g) cw[g] = codes_g[(blockIdx.x * blockDim.x + threadIdx.x) * 4 + g];
  const uint32_t one = k_one;
  uint32_t res = 0;
  for (int r = 0; r < reps; ++r) {
    uint32_t ae[W], ao[W];
#pragma unroll
    for (int w = 0; w < W; ++w) ae[w] = ao[w] = 0u;
#pragma unroll 1
    for (int g = 0; g < 4; ++g) {
      const uint32_t c = cw[g] ^ (uint32_t)r;
#pragma unroll
      for (int i = 0; i < 8; i += 2) {
        const int cb = g * 8 + i;
        const uint32_t k0 = (c >> (4 * i)) & 15u, k1 = (c >> (4 * i + 4)) & 15u;
        if constexpr (V == 7) {
          const uint2* p0 = reinterpret_cast<const uint2*>(s) + cb * (W / 2) * 16 + k0;
          const uint2* p1 = reinterpret_cast<const uint2*>(s) + (cb + 1) * (W / 2) * 16 + k1;
#pragma unroll
          for (int w = 0; w < W / 2; ++w) {
            const uint2 a = p0[w * 16], b = p1[w * 16];
            ae[2 * w] += a.x + b.x;
            ao[2 * w] += __byte_perm(a.x, 0u, 0x4341) + __byte_perm(b.x, 0u, 0x4341);
            ae[2 * w + 1] += a.y + b.y;
            ao[2 * w + 1] += __byte_perm(a.y, 0u, 0x4341) + __byte_perm(b.y, 0u, 0x4341);
          }
        } else {
          const uint32_t* p0 = s + cb * W * 16 + k0;
          const uint32_t* p1 = s + (cb + 1) * W * 16 + k1;
#pragma unroll
          for (int w = 0; w < W; ++w) {
            const uint32_t a = p0[w * 16], b = p1[w * 16];
            ae[w] += a + b;
            if constexpr (V == 6 || V == 8)
              ao[w] = mad_add(mad_add(ao[w], __byte_perm(a, 0u, 0x4341), one), __byte_perm(b, 0u, 0x4341), one);
            else
              ao[w] += __byte_perm(a, 0u, 0x4341) + __byte_perm(b, 0u, 0x4341);
          }
        }
      }
    }
    if constexpr (V == 8) {
      // the real scan's epilogue: each lane stores its row's W float4 (16-B
      // pieces of 32 different rows per warp store instruction)
      float* o = reinterpret_cast<float*>(out) + 1024 +
                 ((size_t)(blockIdx.x * blockDim.x + threadIdx.x) + (size_t)(r & 7) * gridDim.x * blockDim.x) * (4 * W);
#pragma unroll
      for (int w = 0; w < W; ++w) {
        const uint32_t e = ae[w] - (ao[w] << 8);
        *reinterpret_cast<float4*>(o + 4 * w) =
            make_float4((float)(e & 0xFFFFu), (float)(ao[w] & 0xFFFFu), (float)(e >> 16), (float)(ao[w] >> 16));
      }
    } else {
#pragma unroll
      for (int w = 0; w < W; ++w) res ^= (ae[w] - (ao[w] << 8)) ^ ao[w];
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = res;
}

template <int V>
void run(const uint32_t* dcodes, uint32_t* dout, int sms, int clk_khz) {
  auto k = V <= 4 ? k_lds<V <= 4 ? V : 1> : k_scan<V>;
  const size_t smem = (size_t)C * W * 16 * 4;
  CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int reps = 200;
  k<<<sms, 512, smem>>>(dcodes, dout, 2);
  CK(cudaDeviceSynchronize());
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b));
  float best = 1e30f;
  for (int t = 0; t < 5; ++t) {
    CK(cudaEventRecord(a));
    k<<<sms, 512, smem>>>(dcodes, dout, reps);
    CK(cudaEventRecord(b));
    CK(cudaEventSynchronize(b));
    float ms; CK(cudaEventElapsedTime(&ms, a, b));
    if (ms < best) best = ms;
  }
  const double bytes = (double)sms * 512 * reps * C * W * 4;   // loaded bytes (all lanes)
  const double clocks = best * 1e-3 * clk_khz * 1e3;
  printf("V=%d (%2d-byte loads%s): %.3f ms, %.1f B/clk/SM loaded (%.3f of 128), %.3e lookups(words)/s\n", V,
         V == 7 ? 8 : (V > 4 ? 4 : 4 * V), V == 5 ? ", raw-word scan, ALU adds" : V == 6 ? ", raw-word scan, IMAD odd adds"
         : V == 7 ? ", raw-word scan" : V == 8 ? ", raw-word scan + row stores" : "",
         best, bytes / clocks / sms, bytes / clocks / sms / 128.0, bytes / 4 / (best * 1e-3));
}

int main() {
  int sms = 0, clk = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0));
  const int n = sms * 512 * 4;
  uint32_t* h = (uint32_t*)malloc(n * 4);
  uint64_t x = 88172645463325252ull;
  for (int i = 0; i < n; ++i) { x ^= x << 13; x ^= x >> 7; x ^= x << 17; h[i] = (uint32_t)x; }
  uint32_t *dcodes, *dout;
  CK(cudaMalloc(&dcodes, n * 4));
  CK(cudaMalloc(&dout, 4096 + (size_t)8 * sms * 512 * 4 * W * 4));   // V = 8 row outputs
  CK(cudaMemcpy(dcodes, h, n * 4, cudaMemcpyHostToDevice));
  printf("SMs %d, clock %d MHz (max; the timed kernels run at the clock the driver allows)\n", sms, clk / 1000);
  run<1>(dcodes, dout, sms, clk);
  run<2>(dcodes, dout, sms, clk);
  run<4>(dcodes, dout, sms, clk);
  run<5>(dcodes, dout, sms, clk);
  run<6>(dcodes, dout, sms, clk);
  run<7>(dcodes, dout, sms, clk);
  run<8>(dcodes, dout, sms, clk);
  return 0;
}
