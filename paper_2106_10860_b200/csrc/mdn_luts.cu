// h(B) on the device: table construction (Sec. 3; dense
// prototypes per L896, Theta(MKCD)) and the 8-bit quantisation of App. A
// (L593-604). Off the timed path; run once per B ("set_operator").
//
// Exactness contract: every product P*B of two fp32
// values is exact in fp64, so the only rounding is the fp64 addition, done in
// ascending j by one thread per table entry; min / max reductions are exact
// in any order. Hence Tq bytes, l, alpha and beta32 are bit-identical to any
// other implementation of the same definition.
#include <cuda_runtime.h>

#include "mdn_internal.h"

namespace mdn {
namespace {

// T[(c*16+k)*M + m] = sum_{j=0}^{D-1} P[c*16+k][j] * B[j][m]   (fp64, ascending j)
__global__ void k_tables(const float* __restrict__ P, const float* __restrict__ B, int KC, int D,
                         int M, double* __restrict__ T) {
  int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (int64_t)KC * M) return;
  int row = (int)(idx / M), m = (int)(idx % M);
  const float* p = P + (int64_t)row * D;
  double acc = 0.0;
  for (int j = 0; j < D; ++j)
    acc = __dadd_rn(acc, __dmul_rn((double)p[j], (double)B[(int64_t)j * M + m]));
  T[idx] = acc;
}

// One block per codebook: delta_c = min T[c], range_c = max (T[c] - delta_c).
__global__ void k_minmax(const double* __restrict__ T, int M, double* delta, double* range) {
  const int c = blockIdx.x, n = K * M;
  const double* t = T + (int64_t)c * n;
  __shared__ double red[256];
  double mn = INFINITY;
  for (int i = threadIdx.x; i < n; i += blockDim.x) mn = fmin(mn, t[i]);
  red[threadIdx.x] = mn;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) red[threadIdx.x] = fmin(red[threadIdx.x], red[threadIdx.x + s]);
    __syncthreads();
  }
  const double d = red[0];
  __syncthreads();
  double mx = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) mx = fmax(mx, __dsub_rn(t[i], d));
  red[threadIdx.x] = mx;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) red[threadIdx.x] = fmax(red[threadIdx.x], red[threadIdx.x + s]);
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    delta[c] = d;
    range[c] = red[0];
  }
}

// l = max{ l : 2^l R <= 255 } with R = max_c range_c (reading R14); alpha = 2^-l;
// beta32 = fl32(sum_c delta_c + alpha * debias) (reading R18), ascending c.
__global__ void k_scalars(const double* delta, const double* range, int C, int U_or_0,
                          LutScalars* out) {
  double R = 0.0;
  for (int c = 0; c < C; ++c) R = fmax(R, range[c]);
  int l = 0;
  if (R > 0.0) {
    l = (int)floor(log2(255.0 / R));
    while (ldexp(R, l + 1) <= 255.0) ++l;
    while (ldexp(R, l) > 255.0) --l;
  }
  LutScalars s;
  s.err = (l > 100 || l < -100) ? 1 : 0;
  s.l = l;
  s.alpha = (float)ldexp(1.0, -l);
  double debias = 0.0;
  if (U_or_0 > 1) {
    int lg = 0;
    while ((1 << lg) < U_or_0) ++lg;
    debias = -(double)C * (double)lg / 4.0;  // App. D Theorem (L766-771), sign per R16
  }
  double sum = 0.0;
  for (int c = 0; c < C; ++c) sum = __dadd_rn(sum, delta[c]);
  s.beta32 = __double2float_rn(__dadd_rn(sum, __dmul_rn((double)s.alpha, debias)));
  *out = s;
}

// Tq = rint(2^l (T - delta_c)), ties to even (reading R15).
__global__ void k_quant(const double* __restrict__ T, const double* __restrict__ delta, int M,
                        int64_t n, const LutScalars* sc, uint8_t* __restrict__ tq) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n || sc->err) return;
  int c = (int)(i / (K * M));
  double q = rint(ldexp(__dsub_rn(T[i], delta[c]), sc->l));
  q = fmin(fmax(q, 0.0), 255.0);  // no-op by construction of l
  tq[i] = (uint8_t)q;
}

// Scan layout: words[(c*W + w)*16 + k] = Tq[c][k][4w .. 4w+3] (little-endian bytes,
// zero beyond M). For fixed (c, w) the 16 code entries are 16 consecutive words,
// i.e. 16 distinct shared-memory banks, so threads with arbitrary codes never
// conflict.
__global__ void k_pack_words(const uint8_t* __restrict__ tq, int C, int M,
                             uint32_t* __restrict__ words) {
  const int W = (M + 3) / 4;
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (int64_t)C * W * K) return;
  int k = (int)(i % K), w = (int)((i / K) % W), c = (int)(i / ((int64_t)K * W));
  uint32_t v = 0;
  for (int b = 0; b < 4; ++b) {
    int m = 4 * w + b;
    uint32_t byte = m < M ? tq[((int64_t)c * K + k) * M + m] : 0u;
    v |= byte << (8 * b);
  }
  words[i] = v;
}

// Small-M scan layout (mdn_small.cu): words16[(c*16 + k)*W2 + w] =
// Tq[c][k][2w] | Tq[c][k][2w+1] << 16 (zero beyond M). Exact sums of up to
// 257 such words cannot carry across the 16-bit lanes (255 C < 2^16).
__global__ void k_pack_words16(const uint8_t* __restrict__ tq, int C, int M,
                               uint32_t* __restrict__ words16) {
  const int W2 = (M + 1) / 2;
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (int64_t)C * K * W2) return;
  const int w = (int)(i % W2);
  const int64_t ck = i / W2;                       // c * 16 + k
  uint32_t v = 0;
  for (int b = 0; b < 2; ++b) {
    int m = 2 * w + b;
    uint32_t byte = m < M ? tq[ck * M + m] : 0u;
    v |= byte << (16 * b);
  }
  words16[i] = v;
}

}  // namespace

cudaError_t pack_words_dev(const uint8_t* dTq, int C, int M, uint32_t* dWords,
                           uint32_t* dWords16, cudaStream_t s) {
  int64_t n = (int64_t)C * ((M + 3) / 4) * K;
  k_pack_words<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(dTq, C, M, dWords);
  if (dWords16) {
    int64_t n16 = (int64_t)C * K * ((M + 1) / 2);
    k_pack_words16<<<(unsigned)((n16 + 255) / 256), 256, 0, s>>>(dTq, C, M, dWords16);
  }
  return cudaGetLastError();
}

cudaError_t build_tables_dev(const float* dP, const float* dB, int C, int D, int M, int U_or_0,
                             double* dT, double* dDelta, double* dRange, LutScalars* dScal,
                             uint8_t* dTq, uint32_t* dWords, uint32_t* dWords16, cudaStream_t s) {
  const int KC = K * C;
  int64_t n = (int64_t)KC * M;
  k_tables<<<(unsigned)((n + 127) / 128), 128, 0, s>>>(dP, dB, KC, D, M, dT);
  k_minmax<<<C, 256, 0, s>>>(dT, M, dDelta, dRange);
  k_scalars<<<1, 1, 0, s>>>(dDelta, dRange, C, U_or_0, dScal);
  k_quant<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(dT, dDelta, M, n, dScal, dTq);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  e = pack_words_dev(dTq, C, M, dWords, dWords16, s);
  if (e != cudaSuccess) return e;
  return cudaStreamSynchronize(s);
}

}  // namespace mdn
