// Generic (any shape / alignment) kernels for g, f and the fused path.
// Thread per row, no shape templates: the correctness baseline that every
// specialised kernel is tested against, and the fallback for shapes / strides
// the fast kernels do not cover.
#include <cuda_runtime.h>

#include "mdn_internal.h"

namespace mdn {
namespace {

constexpr int GEN_THREADS = 256;

// Algorithm 1 for one codebook of one row:
// p <- 2p + [x_{j^t} >= v^t_p], t = 1..4 (0-based heap node 2^t - 1 + p).
__device__ __forceinline__ int hash_row(const float* __restrict__ a, const int* s_dims,
                                        const float* s_thr, int c) {
  int p = 0;
#pragma unroll
  for (int t = 0; t < 4; ++t) {
    float x = __ldg(a + s_dims[c * 4 + t]);
    float v = s_thr[c * THR_STRIDE + (1 << t) - 1 + p];
    p = 2 * p + (x >= v ? 1 : 0);
  }
  return p;
}

__device__ __forceinline__ void load_trees(const TreesDev& t, int* s_dims, float* s_thr) {
  for (int i = threadIdx.x; i < t.C * 4; i += blockDim.x) s_dims[i] = t.dims[i];
  for (int i = threadIdx.x; i < t.C * THR_STRIDE; i += blockDim.x) s_thr[i] = t.thr[i];
}

__global__ void k_encode_generic(TreesDev t, const float* __restrict__ A, int64_t N, int64_t lda,
                                 uint8_t* __restrict__ codes) {
  extern __shared__ __align__(16) unsigned char smem[];
  float* s_thr = reinterpret_cast<float*>(smem);
  int* s_dims = reinterpret_cast<int*>(s_thr + t.C * THR_STRIDE);
  load_trees(t, s_dims, s_thr);
  __syncthreads();
  const int nb = (t.C + 1) / 2;
  for (int64_t row = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; row < N;
       row += (int64_t)gridDim.x * blockDim.x) {
    const float* a = A + row * lda;
    uint8_t* out = codes + row * nb;
    for (int c = 0; c < t.C; c += 2) {
      int lo = hash_row(a, s_dims, s_thr, c);
      int hi = c + 1 < t.C ? hash_row(a, s_dims, s_thr, c + 1) : 0;
      out[c / 2] = (uint8_t)(lo | (hi << 4));
    }
  }
}

// S for one (row, column m): exact sum, or the App. D estimator with a
// binary-counter evaluation of the halves recursion (identical to
// s^_U(x) = mu(s^_U(x_left), s^_U(x_right)) with mu(a,b) = (a+b+1)>>1).
__device__ __forceinline__ int sum_entry(const uint8_t* __restrict__ tq, const uint8_t* code_row,
                                         int C, int M, int U, int m) {
  if (U == 0) {
    int s = 0;
    for (int c = 0; c < C; ++c) {
      int k = (code_row[c >> 1] >> (4 * (c & 1))) & 15;
      s += tq[((int64_t)c * K + k) * M + m];
    }
    return s;
  }
  int total = 0;
  for (int b = 0; b < C / U; ++b) {
    int stack[8];
    int top = 0;
    for (int i = 0; i < U; ++i) {
      int c = b * U + i;
      int k = (code_row[c >> 1] >> (4 * (c & 1))) & 15;
      int v = tq[((int64_t)c * K + k) * M + m];
      int lvl = 0;
      for (int ii = i; ii & 1; ii >>= 1) v = (stack[lvl++] + v + 1) >> 1;
      stack[lvl] = v;
      top = lvl;
    }
    total += stack[top];
  }
  return total;  // the block-sum; S = U * total
}

__global__ void k_scan_generic(LutsDev l, const uint8_t* __restrict__ codes, int64_t N,
                               int32_t* __restrict__ sums, float* __restrict__ out, int64_t ldo) {
  const int nb = (l.C + 1) / 2;
  const int scale = l.U == 0 ? 1 : l.U;
  for (int64_t row = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; row < N;
       row += (int64_t)gridDim.x * blockDim.x) {
    const uint8_t* cr = codes + row * nb;
    for (int m = 0; m < l.M; ++m) {
      int s = sum_entry(l.tq, cr, l.C, l.M, l.U, m);
      if (sums) sums[row * l.M + m] = s * scale;
      if (out) out[row * ldo + m] = __fmaf_rn(l.alpha_eff, (float)s, l.beta32);
    }
  }
}

__global__ void k_amm_generic(TreesDev t, LutsDev l, const float* __restrict__ A, int64_t N,
                              int64_t lda, float* __restrict__ out, int64_t ldo) {
  extern __shared__ __align__(16) unsigned char smem[];
  float* s_thr = reinterpret_cast<float*>(smem);
  int* s_dims = reinterpret_cast<int*>(s_thr + t.C * THR_STRIDE);
  load_trees(t, s_dims, s_thr);
  __syncthreads();
  uint8_t code_row[MAX_C / 2];
  for (int64_t row = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; row < N;
       row += (int64_t)gridDim.x * blockDim.x) {
    const float* a = A + row * lda;
    for (int c = 0; c < t.C; c += 2) {
      int lo = hash_row(a, s_dims, s_thr, c);
      int hi = c + 1 < t.C ? hash_row(a, s_dims, s_thr, c + 1) : 0;
      code_row[c / 2] = (uint8_t)(lo | (hi << 4));
    }
    for (int m = 0; m < l.M; ++m) {
      int s = sum_entry(l.tq, code_row, l.C, l.M, l.U, m);
      out[row * ldo + m] = __fmaf_rn(l.alpha_eff, (float)s, l.beta32);
    }
  }
}

unsigned grid_for(int64_t N) {
  int64_t blocks = (N + GEN_THREADS - 1) / GEN_THREADS;
  int64_t cap = 148 * 16;
  return (unsigned)(blocks < cap ? blocks : cap);
}

}  // namespace

cudaError_t launch_encode_generic(const TreesDev& t, const float* A, int64_t N, int64_t lda,
                                  uint8_t* codes, cudaStream_t s) {
  size_t sm = (size_t)t.C * (THR_STRIDE * 4 + 16);
  k_encode_generic<<<grid_for(N), GEN_THREADS, sm, s>>>(t, A, N, lda, codes);
  return cudaGetLastError();
}

cudaError_t launch_scan_generic(const LutsDev& l, const uint8_t* codes, int64_t N, int32_t* sums,
                                float* out, int64_t ldo, cudaStream_t s) {
  k_scan_generic<<<grid_for(N), GEN_THREADS, 0, s>>>(l, codes, N, sums, out, ldo);
  return cudaGetLastError();
}

cudaError_t launch_amm_generic(const TreesDev& t, const LutsDev& l, const float* A, int64_t N,
                               int64_t lda, float* out, int64_t ldo, cudaStream_t s) {
  size_t sm = (size_t)t.C * (THR_STRIDE * 4 + 16);
  k_amm_generic<<<grid_for(N), GEN_THREADS, sm, s>>>(t, l, A, N, lda, out, ldo);
  return cudaGetLastError();
}

}  // namespace mdn

// ---------------------------------------------------------------------------
// Diagnostics: a plain streaming kernel with the fused path's byte mix (read
// every element of A, write M floats per row), no table work. Its bandwidth is
// the achievable ceiling the fused kernel is compared against.
namespace mdn {
namespace {
constexpr int PROBE_ROWS = 4;   // rows per warp iteration (loads in flight)

__global__ void __launch_bounds__(256) k_stream_probe(const float* __restrict__ A, int64_t N,
                                                      int64_t lda, int D, float* __restrict__ out,
                                                      int64_t ldo, int M) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int D4 = D / 4;
  for (int64_t r0 = warp * PROBE_ROWS; r0 < N; r0 += nwarps * PROBE_ROWS) {
    float acc[PROBE_ROWS];
#pragma unroll
    for (int k = 0; k < PROBE_ROWS; ++k) {
      acc[k] = 0.f;
      const int64_t r = r0 + k;
      if (r < N) {
        const float4* a = reinterpret_cast<const float4*>(A + r * lda);
        for (int i = lane; i < D4; i += 32) {
          const float4 v = __ldcs(a + i);
          acc[k] += (v.x + v.y) + (v.z + v.w);
        }
      }
    }
#pragma unroll
    for (int k = 0; k < PROBE_ROWS; ++k) {
      float v = acc[k];
      for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      const int64_t r = r0 + k;
      if (r < N)
        for (int m = lane; m < M; m += 32) out[r * ldo + m] = v;
    }
  }
}
}  // namespace

cudaError_t launch_stream_probe(const float* A, int64_t N, int64_t lda, int D, float* out,
                                int64_t ldo, int M, cudaStream_t s) {
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  k_stream_probe<<<sms * 8, 256, 0, s>>>(A, N, lda, D, out, ldo, M);
  return cudaGetLastError();
}
}  // namespace mdn
