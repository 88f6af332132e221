// Generic (any shape / alignment) kernels for g, f and the fused path.
// Thread per row, no shape templates: the correctness baseline that every
// specialised kernel is tested against, and the fallback for shapes / strides
// the fast kernels do not cover.
#include <cuda_runtime.h>

#include "mdn_internal.h"
#include "mdn_tma.cuh"

namespace mdn {
namespace {

constexpr int GEN_THREADS = 256;

// Algorithm 1 for one codebook of one row:
// p <- 2p + [x_{j^t} >= v^t_p], t = 1..4 (0-based heap node 2^t - 1 + p).
// fp32 A: x >= v in fp32. uint8 A: x >= q with the integer split
// values q = ceil(v) (App. B, reading R11), stored in s_thr as ints.
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

__device__ __forceinline__ int hash_row(const uint8_t* __restrict__ a, const int* s_dims,
                                        const float* s_thr, int c) {
  const int* s_q = reinterpret_cast<const int*>(s_thr);
  int p = 0;
#pragma unroll
  for (int t = 0; t < 4; ++t) {
    int x = __ldg(a + s_dims[c * 4 + t]);
    int q = s_q[c * THR_STRIDE + (1 << t) - 1 + p];
    p = 2 * p + (x >= q ? 1 : 0);
  }
  return p;
}

template <class TIn>
__device__ __forceinline__ void load_trees(const TreesDev& t, int* s_dims, float* s_thr) {
  for (int i = threadIdx.x; i < t.C * 4; i += blockDim.x) s_dims[i] = t.dims[i];
  for (int i = threadIdx.x; i < t.C * THR_STRIDE; i += blockDim.x) {
    if constexpr (sizeof(TIn) == 1)
      reinterpret_cast<int*>(s_thr)[i] = t.q[i];
    else
      s_thr[i] = t.thr[i];
  }
}

template <class TIn>
__global__ void k_encode_generic(TreesDev t, const TIn* __restrict__ A, int64_t N, int64_t lda,
                                 uint8_t* __restrict__ codes) {
  extern __shared__ __align__(16) unsigned char smem[];
  float* s_thr = reinterpret_cast<float*>(smem);
  int* s_dims = reinterpret_cast<int*>(s_thr + t.C * THR_STRIDE);
  load_trees<TIn>(t, s_dims, s_thr);
  __syncthreads();
  const int nb = (t.C + 1) / 2;
  for (int64_t row = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; row < N;
       row += (int64_t)gridDim.x * blockDim.x) {
    const TIn* a = A + row * lda;
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
    int stack[AVG_STACK];
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

template <class TIn>
__global__ void k_amm_generic(TreesDev t, LutsDev l, const TIn* __restrict__ A, int64_t N,
                              int64_t lda, float* __restrict__ out, int64_t ldo) {
  extern __shared__ __align__(16) unsigned char smem[];
  float* s_thr = reinterpret_cast<float*>(smem);
  int* s_dims = reinterpret_cast<int*>(s_thr + t.C * THR_STRIDE);
  load_trees<TIn>(t, s_dims, s_thr);
  __syncthreads();
  uint8_t code_row[MAX_C / 2];
  for (int64_t row = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; row < N;
       row += (int64_t)gridDim.x * blockDim.x) {
    const TIn* a = A + row * lda;
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
  const int64_t cap = (int64_t)fast::dev_info().sms * 16;   // grid-stride fallback kernels
  return (unsigned)(blocks < cap ? blocks : cap);
}

}  // namespace

cudaError_t launch_encode_generic(const TreesDev& t, const void* A, int es, int64_t N, int64_t lda,
                                  uint8_t* codes, cudaStream_t s) {
  size_t sm = (size_t)t.C * (THR_STRIDE * 4 + 16);
  if (es == 1)
    k_encode_generic<uint8_t><<<grid_for(N), GEN_THREADS, sm, s>>>(
        t, static_cast<const uint8_t*>(A), N, lda, codes);
  else
    k_encode_generic<float><<<grid_for(N), GEN_THREADS, sm, s>>>(
        t, static_cast<const float*>(A), N, lda, codes);
  return cudaGetLastError();
}

cudaError_t launch_scan_generic(const LutsDev& l, const uint8_t* codes, int64_t N, int32_t* sums,
                                float* out, int64_t ldo, cudaStream_t s) {
  k_scan_generic<<<grid_for(N), GEN_THREADS, 0, s>>>(l, codes, N, sums, out, ldo);
  return cudaGetLastError();
}

cudaError_t launch_amm_generic(const TreesDev& t, const LutsDev& l, const void* A, int es,
                               int64_t N, int64_t lda, float* out, int64_t ldo, cudaStream_t s) {
  size_t sm = (size_t)t.C * (THR_STRIDE * 4 + 16);
  if (es == 1)
    k_amm_generic<uint8_t><<<grid_for(N), GEN_THREADS, sm, s>>>(
        t, l, static_cast<const uint8_t*>(A), N, lda, out, ldo);
  else
    k_amm_generic<float><<<grid_for(N), GEN_THREADS, sm, s>>>(
        t, l, static_cast<const float*>(A), N, lda, out, ldo);
  return cudaGetLastError();
}

}  // namespace mdn

// ---------------------------------------------------------------------------
// Diagnostics: a plain streaming kernel with the fused path's byte mix: every
// float of A read once (flat, fully coalesced float4 grid-stride when lda == D)
// and N x M floats of out written once, interleaved, no table work. Its
// bandwidth is the achievable ceiling for this read:write mix.
namespace mdn {
namespace {
__global__ void __launch_bounds__(256) k_stream_probe(const float4* __restrict__ A4, int64_t n4,
                                                      float4* __restrict__ out4, int64_t w4) {
  // Reads every float4 of A (8 independent 16-byte loads in flight per
  // thread), then writes the M columns of every row: the fused path's byte
  // mix with no other work (the earlier version spread the writes with a
  // 64-bit modulo per element and was instruction-bound at 5.3 TB/s).
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  float acc = 0.f;
  int64_t j = tid;
  for (; j + 7 * stride < n4; j += 8 * stride) {
    float4 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = __ldg(A4 + j + u * stride);
#pragma unroll
    for (int u = 0; u < 8; ++u) acc += (v[u].x + v[u].y) + (v[u].z + v[u].w);
  }
  for (; j < n4; j += stride) {
    const float4 v = __ldg(A4 + j);
    acc += (v.x + v.y) + (v.z + v.w);
  }
  for (int64_t k = tid; k < w4; k += stride) out4[k] = make_float4(acc, acc, acc, acc);
}
}  // namespace

cudaError_t launch_stream_probe(const float* A, int64_t N, int64_t lda, int D, float* out,
                                int64_t ldo, int M, cudaStream_t s) {
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int64_t n4 = N * lda / 4;            // lda == D for the bench inputs
  const int64_t w4 = N * ldo / 4;
  k_stream_probe<<<sms * 8, 256, 0, s>>>(reinterpret_cast<const float4*>(A), n4,
                                          reinterpret_cast<float4*>(out), w4);
  return cudaGetLastError();
}
}  // namespace mdn
