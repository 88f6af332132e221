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

template <int V>
void run(const uint32_t* dcodes, uint32_t* dout, int sms, int clk_khz) {
  auto k = k_lds<V>;
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
  printf("V=%d (%2d-byte loads): %.3f ms, %.1f B/clk/SM loaded (%.3f of 128), %.3e lookups(words)/s\n", V, 4 * V,
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
  CK(cudaMalloc(&dcodes, n * 4)); CK(cudaMalloc(&dout, sms * 512 * 4));
  CK(cudaMemcpy(dcodes, h, n * 4, cudaMemcpyHostToDevice));
  printf("SMs %d, clock %d MHz (max; the timed kernels run at the clock the driver allows)\n", sms, clk / 1000);
  run<1>(dcodes, dout, sms, clk);
  run<2>(dcodes, dout, sms, clk);
  run<4>(dcodes, dout, sms, clk);
  return 0;
}
