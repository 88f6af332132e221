// Column-major A: the split-column gather encoder.
//
// Algorithm 1 "only depends on a constant number of indices in the input
// vector, and can easily be vectorized provided that the matrix whose rows are
// being encoded is stored in column-major order", and its cost
// per row is O(C) rather than O(D) (L431). With A stored column-major (At =
// A^T, D x N, row stride ldt >= N) the kernel reads ONLY the <= 4C split
// columns, each as fully coalesced 128-byte warp loads (lane = row), so the
// HBM bytes per row are 4 |S| + 4M (|S| = distinct split dims) instead of
// 4D + 4M: 912 vs 2448 for the CIFAR-100-shaped config.
//
// For C >= 16 the fused path and the encoder run the warp-specialised TMA
// kernel of mdn_fast.cu with a [slot][row] stage layout filled by TMA gather4
// (launch_amm_ws_cm / launch_encode_ws_cm) whenever its shapes are
// supported; the kernel here serves C <= 8 (tiny, image) and is the fallback.
//
// k_amm_cm: a thread owns RPT consecutive rows (4 for C = 4, 2 for C = 8 when
// the columns are aligned for vector loads, else 1). For each group of 8
// codebooks the split values are loaded (streaming, evict-first: each is used
// once; one vector load per column covers the thread's rows), Algorithm 1
// runs on thresholds resident in shared memory, and the packed codes feed the
// same shared-memory table scan as the row-major fused kernel (mdn_scan.cuh);
// the codes never leave registers. ENC_ONLY writes the packed codes instead
// (one 8-byte store per thread when RPT rows of codes make 8 bytes).
#include <cuda_runtime.h>

#include <cstdlib>

#include "mdn_internal.h"
#include "mdn_scan.cuh"
#include "mdn_tma.cuh"

namespace mdn {
namespace fast {
namespace colmajor {

constexpr int THREADS = 256;

// Streaming (evict-first) loads.
__device__ __forceinline__ float ld_stream(const float* p) { return __ldcs(p); }

// RPT consecutive rows of one split column (At[col][row .. row + RPT)): one
// vector load (RPT = 2: 8 B, 4: 16 B aligned), so a warp reads RPT x 128
// contiguous bytes per column instead of 128.
template <int RPT>
__device__ __forceinline__ void ld_stream_v(const float* p, float (&v)[RPT]) {
  if constexpr (RPT == 4) {
    const float4 t = __ldcs(reinterpret_cast<const float4*>(p));
    v[0] = t.x, v[1] = t.y, v[2] = t.z, v[3] = t.w;
  } else if constexpr (RPT == 2) {
    const float2 t = __ldcs(reinterpret_cast<const float2*>(p));
    v[0] = t.x, v[1] = t.y;
  } else {
    v[0] = ld_stream(p);
  }
}

// Algorithm 1 (L228-248) for G codebooks of one row; x[i][t] = the row's value
// in split column dims[c0 + i][t]. 0-based: p <- 2p + [x_t >= v^t_p].
template <int G>
__device__ __forceinline__ uint32_t encode_group(const float (&x)[G][4], const float* __restrict__ s_thr,
                                                 int c0) {
  uint32_t word = 0;
#pragma unroll
  for (int i = 0; i < G; ++i) {
    const float* th = s_thr + 16 * (c0 + i);
    uint32_t p = x[i][0] >= th[0] ? 1u : 0u;
    p = 2u * p + (x[i][1] >= th[1 + p] ? 1u : 0u);
    p = 2u * p + (x[i][2] >= th[3 + p] ? 1u : 0u);
    p = 2u * p + (x[i][3] >= th[7 + p] ? 1u : 0u);
    word |= p << (4 * i);
  }
  return word;
}

struct CmParams {
  const float* At;
  int64_t N, ldt, ldo;
  const uint16_t* dims;   // [C][4]
  const float* thr;       // [C][16]
  const uint32_t* lut;    // [C][W][16]
  float* out;
  uint8_t* codes;
  int M;
  bool pair;
  bool pack2;             // M == 2, ldo == 2, out 16-B aligned: 2 rows per float4 store
  float alpha_eff, beta32;
};

// Per-row code stores (encode) or scan + dequantised stores (fused).
template <int C, int W, int U, bool VEC, bool ENC_ONLY, int RPT>
__device__ __forceinline__ void cm_store(const CmParams& p, int64_t row0,
                                         const uint32_t (&cw)[RPT][C >= 8 ? C / 8 : 1],
                                         const uint32_t* s_lut) {
  constexpr int NG = C >= 8 ? C / 8 : 1;
  if constexpr (!ENC_ONLY && RPT == 2 && W == 1) {
    if (p.pack2) {
      // M = 2, ldo = 2: the two rows' outputs are 16 contiguous bytes
      float4 o;
      uint32_t ae[W], ao[W];
      scan_core<C, W, U, true>(s_lut, [&](int g) { return cw[0][g]; }, ae, ao);
      o.x = __fmaf_rn(p.alpha_eff, (float)(ae[0] & 0xFFFFu), p.beta32);
      o.y = __fmaf_rn(p.alpha_eff, (float)(ao[0] & 0xFFFFu), p.beta32);
      scan_core<C, W, U, true>(s_lut, [&](int g) { return cw[1][g]; }, ae, ao);
      o.z = __fmaf_rn(p.alpha_eff, (float)(ae[0] & 0xFFFFu), p.beta32);
      o.w = __fmaf_rn(p.alpha_eff, (float)(ao[0] & 0xFFFFu), p.beta32);
      *reinterpret_cast<float4*>(p.out + row0 * 2) = o;
      return;
    }
  }
#pragma unroll
  for (int r = 0; r < RPT; ++r) {
    const int64_t row = row0 + r;
    if constexpr (ENC_ONLY) {
      if constexpr (C >= 8) {
#pragma unroll
        for (int g = 0; g < NG; ++g) reinterpret_cast<uint32_t*>(p.codes + row * (C / 2))[g] = cw[r][g];
      } else if constexpr (C == 4) {
        reinterpret_cast<uint16_t*>(p.codes + row * 2)[0] = (uint16_t)cw[r][0];
      } else {
        p.codes[row] = (uint8_t)cw[r][0];
      }
    } else {
      uint32_t ae[W], ao[W];
      scan_core<C, W, U, true>(s_lut, [&](int g) { return cw[r][g]; }, ae, ao);
      store_row<W, VEC>(p.out + row * p.ldo, p.M, ae, ao, p.alpha_eff, p.beta32, p.pair);
    }
  }
}

// RPT consecutive rows row0 .. row0 + RPT - 1 (all < N) of one thread: each
// split column is one vector load of the RPT values (RPT = 1: scalar).
template <int C, int W, int U, bool VEC, bool ENC_ONLY, int RPT>
__device__ __forceinline__ void cm_rows(const CmParams& p, int64_t row0, const float* s_thr,
                                        const int64_t* s_col, const uint32_t* s_lut) {
  constexpr int G = C >= 8 ? 8 : C;
  constexpr int NG = C / G;
  const float* a = p.At + row0;
  uint32_t cw[RPT][NG];
#pragma unroll
  for (int g = 0; g < NG; ++g) {
    float x[RPT][G][4];
#pragma unroll
    for (int i = 0; i < G; ++i)
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        float v[RPT];
        ld_stream_v<RPT>(a + s_col[(g * G + i) * 4 + t], v);
#pragma unroll
        for (int r = 0; r < RPT; ++r) x[r][i][t] = v[r];
      }
    // every split-column load of the group is issued before the first tree
    // consumes one (left alone, the compiler interleaved them at 38 registers
    // in the fused variant: long-scoreboard stalls 18 per issue)
    asm volatile("" ::: "memory");
#pragma unroll
    for (int r = 0; r < RPT; ++r) cw[r][g] = encode_group<G>(x[r], s_thr, g * G);
  }
  if constexpr (ENC_ONLY && RPT > 1 && C * RPT == 16) {
    // the rows' codes are 8 contiguous bytes (C = 4: 4 rows x 2 B; C = 8:
    // 2 rows x 4 B): one 8-byte store (the launcher checked the alignment)
    uint64_t v = 0;
#pragma unroll
    for (int r = 0; r < RPT; ++r) v |= (uint64_t)cw[r][0] << (r * 4 * C);
    *reinterpret_cast<uint64_t*>(p.codes + row0 * (C / 2)) = v;
  } else {
    cm_store<C, W, U, VEC, ENC_ONLY, RPT>(p, row0, cw, s_lut);
  }
}

// Thread per RPT consecutive rows (RPT > 1 for C <= 8 with 16-B / 8-B aligned
// columns; the N % RPT tail rows then run one per thread).
template <int C, int W, int U, bool VEC, bool ENC_ONLY, int RPT = 1>
__global__ void __launch_bounds__(THREADS, 1) k_amm_cm(const CmParams p) {
  extern __shared__ __align__(16) unsigned char smem[];
  float* s_thr = reinterpret_cast<float*>(smem);                       // [C][16]
  int64_t* s_col = reinterpret_cast<int64_t*>(s_thr + 16 * C);         // [C][4] element offsets
  uint32_t* s_lut = reinterpret_cast<uint32_t*>(s_col + 4 * C);        // [C][W][16]
  for (int i = threadIdx.x; i < 16 * C; i += blockDim.x) s_thr[i] = p.thr[i];
  for (int i = threadIdx.x; i < 4 * C; i += blockDim.x) s_col[i] = (int64_t)p.dims[i] * p.ldt;
  if constexpr (!ENC_ONLY) {
    const uint4* src = reinterpret_cast<const uint4*>(p.lut);
    uint4* dst = reinterpret_cast<uint4*>(s_lut);
    for (int i = threadIdx.x; i < C * W * 4; i += blockDim.x) dst[i] = src[i];
  }
  __syncthreads();
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t n_full = p.N / RPT;
  for (int64_t gi = tid; gi < n_full; gi += stride)
    cm_rows<C, W, U, VEC, ENC_ONLY, RPT>(p, gi * RPT, s_thr, s_col, s_lut);
  if constexpr (RPT > 1)
    for (int64_t row = n_full * RPT + tid; row < p.N; row += stride)
      cm_rows<C, W, U, VEC, ENC_ONLY, 1>(p, row, s_thr, s_col, s_lut);
}

// Generic fallback: any C (<= MAX_C), any M / U, any alignment.
__global__ void k_amm_cm_generic(TreesDev t, LutsDev l, const float* __restrict__ At, int64_t N,
                                 int64_t ldt, float* __restrict__ out, int64_t ldo,
                                 uint8_t* __restrict__ codes) {
  extern __shared__ __align__(16) unsigned char smem[];
  float* s_thr = reinterpret_cast<float*>(smem);
  int* s_dims = reinterpret_cast<int*>(s_thr + t.C * THR_STRIDE);
  for (int i = threadIdx.x; i < t.C * THR_STRIDE; i += blockDim.x) s_thr[i] = t.thr[i];
  for (int i = threadIdx.x; i < t.C * 4; i += blockDim.x) s_dims[i] = t.dims[i];
  __syncthreads();
  uint8_t code_row[MAX_C / 2];
  const int nb = (t.C + 1) / 2;
  for (int64_t row = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; row < N;
       row += (int64_t)gridDim.x * blockDim.x) {
    for (int i = 0; i < nb; ++i) code_row[i] = 0;
    for (int c = 0; c < t.C; ++c) {
      int q = 0;
      for (int lv = 0; lv < 4; ++lv) {
        const float x = At[(int64_t)s_dims[c * 4 + lv] * ldt + row];
        q = 2 * q + (x >= s_thr[c * THR_STRIDE + (1 << lv) - 1 + q] ? 1 : 0);
      }
      code_row[c >> 1] |= (uint8_t)(q << (4 * (c & 1)));
    }
    if (codes) {
      for (int i = 0; i < nb; ++i) codes[row * nb + i] = code_row[i];
      continue;
    }
    for (int m = 0; m < l.M; ++m) {
      int s = 0;
      if (l.U == 0) {
        for (int c = 0; c < l.C; ++c)
          s += l.tq[((int64_t)c * K + ((code_row[c >> 1] >> (4 * (c & 1))) & 15)) * l.M + m];
      } else {
        // App. D halves recursion, evaluated as a binary counter (as mdn_generic.cu)
        for (int b = 0; b < l.C / l.U; ++b) {
          int stack[AVG_STACK], top = 0;
          for (int i = 0; i < l.U; ++i) {
            const int c = b * l.U + i;
            int v = l.tq[((int64_t)c * K + ((code_row[c >> 1] >> (4 * (c & 1))) & 15)) * l.M + m];
            int lvl = 0;
            for (int ii = i; ii & 1; ii >>= 1) v = (stack[lvl++] + v + 1) >> 1;
            stack[lvl] = v;
            top = lvl;
          }
          s += stack[top];
        }
      }
      out[row * ldo + m] = __fmaf_rn(l.alpha_eff, (float)s, l.beta32);
    }
  }
}

template <int C, int W, int U, bool VEC, bool ENC, int RPT = 1>
cudaError_t launch(const CmParams& p, cudaStream_t s) {
  auto k = k_amm_cm<C, W, U, VEC, ENC, RPT>;
  const size_t smem = 16 * C * 4 + 4 * C * 8 + (ENC ? 0 : (size_t)C * W * 16 * 4);
  cudaError_t e = ensure_smem(reinterpret_cast<const void*>(k), smem);
  if (e != cudaSuccess) return e;
  int per_sm = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, THREADS, smem);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) per_sm = 1;
  int64_t blocks = ((p.N + RPT - 1) / RPT + THREADS - 1) / THREADS;
  const int64_t cap = (int64_t)dev_info().sms * per_sm;
  if (blocks > cap) blocks = cap;
  k<<<(unsigned)blocks, THREADS, smem, s>>>(p);
  return cudaGetLastError();
}

#define MDN_CM_COMBOS(X) \
  X(4, 1, 0) X(4, 1, 4) X(8, 1, 0) X(8, 1, 8) X(8, 2, 0) X(8, 2, 8)                    \
  X(16, 1, 0) X(16, 1, 16) X(16, 3, 0) X(16, 3, 16) X(16, 4, 0) X(16, 4, 16)            \
  X(32, 1, 0) X(32, 1, 16) X(32, 3, 0) X(32, 3, 16) X(32, 4, 0) X(32, 4, 16)            \
  X(32, 25, 0) X(32, 25, 16) X(64, 3, 0) X(64, 3, 16) X(64, 4, 0) X(64, 4, 16)

}  // namespace colmajor
}  // namespace fast

using namespace fast::colmajor;

static cudaError_t cm_generic(const TreesDev& t, const LutsDev* l, const float* At, int64_t N,
                              int64_t ldt, float* out, int64_t ldo, uint8_t* codes, cudaStream_t s) {
  const size_t smem = (size_t)t.C * THR_STRIDE * 4 + (size_t)t.C * 4 * 4;
  int64_t blocks = (N + 255) / 256;
  const int64_t cap = (int64_t)fast::dev_info().sms * 8;
  if (blocks > cap) blocks = cap;
  LutsDev ld{};
  if (l) ld = *l;
  k_amm_cm_generic<<<(unsigned)blocks, 256, smem, s>>>(t, ld, At, N, ldt, out, ldo, codes);
  return cudaGetLastError();
}

// MDN_CM_SIMPLE=1 forces the thread-per-row kernel below (A/B comparisons only).
static bool cm_simple() {
  static int v = [] { const char* e = getenv("MDN_CM_SIMPLE"); return e ? atoi(e) : 0; }();
  return v != 0;
}
// MDN_CM_WS_ENCODE=0 keeps mdn_encode_cm on the thread-per-row kernel (A/B).
static bool cm_ws_encode() {
  static int v = [] { const char* e = getenv("MDN_CM_WS_ENCODE"); return e ? atoi(e) : 1; }();
  return v != 0;
}

// Rows per thread of k_amm_cm for C <= 8: 4 (C = 4) or 2 (C = 8) when the
// columns allow the vector loads, else 1. MDN_CM_RPT=1 forces 1 (A/B only).
static int cm_rpt(int C, const float* At, int64_t ldt) {
  static int knob = [] { const char* e = getenv("MDN_CM_RPT"); return e ? atoi(e) : 0; }();
  if (knob == 1 || C > 8) return 1;
  const uintptr_t a = reinterpret_cast<uintptr_t>(At);
  if (C <= 4 && (a & 15u) == 0 && ldt % 4 == 0) return 4;
  if ((a & 7u) == 0 && ldt % 2 == 0) return 2;
  return 1;
}

template <int C, int W, int U, bool VEC, bool ENC>
static cudaError_t launch_r(const CmParams& p, int rpt, cudaStream_t s) {
  if constexpr (C <= 4)
    if (rpt == 4) return launch<C, W, U, VEC, ENC, 4>(p, s);
  if constexpr (C <= 8)
    if (rpt >= 2) return launch<C, W, U, VEC, ENC, 2>(p, s);
  return launch<C, W, U, VEC, ENC, 1>(p, s);
}

cudaError_t launch_amm_cm(const TreesDev& t, const LutsDev& l, const float* At, int64_t N,
                          int64_t ldt, float* out, int64_t ldo, cudaStream_t s) {
  if (!cm_simple()) {
    bool done = false;
    cudaError_t e = launch_amm_ws_cm(t, l, At, N, ldt, out, ldo, s, &done);
    if (done) return e;
  }
  CmParams p{};
  p.At = At;
  p.N = N;
  p.ldt = ldt;
  p.ldo = ldo;
  p.dims = t.dims;
  p.thr = t.thr;
  p.lut = l.words;
  p.out = out;
  p.M = l.M;
  p.pair = l.M % 2 == 0 && ldo % 2 == 0 && (reinterpret_cast<uintptr_t>(out) & 7u) == 0;
  p.alpha_eff = l.alpha_eff;
  p.beta32 = l.beta32;
  const bool vec = l.M % 4 == 0 && ldo % 4 == 0 && (reinterpret_cast<uintptr_t>(out) & 15u) == 0;
  p.pack2 = l.M == 2 && ldo == 2 && (reinterpret_cast<uintptr_t>(out) & 15u) == 0;
  const int rpt = cm_rpt(t.C, At, ldt);
#define X(c, w, u)                                                                   \
  if (t.C == c && l.W == w && l.U == u)                                              \
    return vec ? launch_r<c, w, u, true, false>(p, rpt, s) : launch_r<c, w, u, false, false>(p, rpt, s);
  MDN_CM_COMBOS(X)
#undef X
  return cm_generic(t, &l, At, N, ldt, out, ldo, nullptr, s);
}

cudaError_t launch_encode_cm(const TreesDev& t, const float* At, int64_t N, int64_t ldt,
                             uint8_t* codes, cudaStream_t s) {
  if (!cm_simple() && cm_ws_encode()) {
    bool done = false;
    cudaError_t e = launch_encode_ws_cm(t, At, N, ldt, codes, s, &done);
    if (done) return e;
  }
  CmParams p{};
  p.At = At;
  p.N = N;
  p.ldt = ldt;
  p.dims = t.dims;
  p.thr = t.thr;
  p.codes = codes;
  const uintptr_t ca = reinterpret_cast<uintptr_t>(codes);
  const bool aligned = t.C >= 8 ? (ca & 3u) == 0 : (t.C == 4 ? (ca & 1u) == 0 : true);
  if (aligned) {
    switch (t.C) {
      // several rows per thread only with 8-byte aligned codes (one store per group)
      case 4: return launch_r<4, 1, 0, false, true>(p, (ca & 7u) ? 1 : cm_rpt(4, At, ldt), s);
      case 8: return launch_r<8, 1, 0, false, true>(p, (ca & 7u) ? 1 : cm_rpt(8, At, ldt), s);
      case 16: return launch<16, 1, 0, false, true>(p, s);
      case 32: return launch<32, 1, 0, false, true>(p, s);
      case 64: return launch<64, 1, 0, false, true>(p, s);
    }
  }
  return cm_generic(t, nullptr, At, N, ldt, nullptr, 0, codes, s);
}

}  // namespace mdn
