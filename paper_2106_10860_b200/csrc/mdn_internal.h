// Internal declarations shared by the host side and the kernels of libmaddness.
// (Product code only; nothing here is shared with the oracle.)
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "../../include/maddness.h"

namespace mdn {

constexpr int K = MDN_K;           // leaves per tree
constexpr int THR_STRIDE = 16;     // 15 heap-ordered thresholds + 1 pad per codebook
constexpr int MAX_C = 256;         // S <= 255 * C must fit the 16-bit SWAR lanes
// Training rows are int32 indices; the block-stride loops (i += blockDim <= 1024)
// need headroom below INT32_MAX so that i + stride never overflows.
constexpr int64_t MDN_TRAIN_MAX_N = 0x7FFFFFFF - (1 << 20);
constexpr int MAX_U = 64;          // largest averaging block (App. D; U = 16 default)
constexpr int AVG_STACK = 7;       // log2(MAX_U) + 1 levels of the halves-recursion stack
static_assert((1 << (AVG_STACK - 1)) == MAX_U, "averaging stack depth must match MAX_U");
constexpr int MAX_W2 = 4;          // words16 tables are kept for M <= 8

// Tree parameters as the kernels consume them (device).
struct TreesDev {
  const uint16_t* dims;  // [C][4] global column of each level's split
  const float* thr;      // [C][16] heap order, pad slot 15 unused
  const uint16_t* sub;   // [C] first column of each codebook's subspace J^(c)
  const uint16_t* q;     // [C][16] 8-bit split values ceil(v) in [0, 256] (uint8 input)
  int C;
  int D;
  int subf;              // fp32: 1 / 2 = every subspace 16-B aligned and <= 4 / 8 wide
  int subf_u8;           // uint8: 1 / 2 = every subspace exactly 4 / 8 bytes, contiguous
  int q_byte;            // every 8-bit split value q <= 255 (fits a byte)
  const uint16_t* cols;  // distinct split columns, ascending [n_cols] (column-major A)
  const uint16_t* slot;  // [D] index of each split column in `cols` (0xFFFF otherwise)
  int n_cols;
  const float* pq_cent;  // PQ model: prototypes [16][DS/4][C][4] (equal subspaces), or null
  int pq_ds;             // PQ subspace width DS of pq_cent (0 if null)
  // Host copies (the model's): launchers that pass per-codebook constants as
  // kernel parameters read them here.
  const uint16_t* h_dims = nullptr;
  const uint16_t* h_sub = nullptr;
  const uint16_t* h_q = nullptr;
};

// Quantised tables as the kernels consume them (device).
struct LutsDev {
  const uint8_t* tq;     // canonical [C][16][M]
  const uint32_t* words; // scan layout [C][W][16]: word (c,w,k) = Tq[c][k][4w..4w+3]
  const uint32_t* words16; // small-M scan layout [C][16][W2]: 2 columns per word in 16-bit
                           // lanes (T[c][k][2w] | T[c][k][2w+1] << 16); null if M > 2*MAX_W2
  int C, M, W;
  int U;                 // 0 = exact sum; else averaging block size (power of two)
  float alpha_eff;       // alpha (exact) or alpha * U (avg): out = alpha_eff * S' + beta
  float beta32;
};

// Kernel entry points (mdn_kernels.cu / mdn_luts.cu / mdn_amm_tma.cu).
cudaError_t launch_encode(const TreesDev& t, const float* A, int64_t N, int64_t lda,
                          uint8_t* codes, cudaStream_t s);
cudaError_t launch_scan(const LutsDev& l, const uint8_t* codes, int64_t N, int32_t* sums,
                        float* out, int64_t ldo, cudaStream_t s);
cudaError_t launch_amm(const TreesDev& t, const LutsDev& l, const float* A, int64_t N,
                       int64_t lda, float* out, int64_t ldo, cudaStream_t s);
cudaError_t launch_encode_u8(const TreesDev& t, const uint8_t* A, int64_t N, int64_t lda,
                             uint8_t* codes, cudaStream_t s);
cudaError_t launch_amm_u8(const TreesDev& t, const LutsDev& l, const uint8_t* A, int64_t N,
                          int64_t lda, float* out, int64_t ldo, cudaStream_t s);
// Register-tree kernel for C <= 8, M <= 4 (mdn_small.cu); *done = false when
// the shapes are not covered (the caller then uses the general kernels).
cudaError_t launch_amm_rt(const TreesDev& t, const LutsDev& l, const float* A, int64_t N,
                          int64_t lda, float* out, int64_t ldo, cudaStream_t s, bool* done);
cudaError_t launch_amm_rt_u8(const TreesDev& t, const LutsDev& l, const uint8_t* A, int64_t N,
                             int64_t lda, float* out, int64_t ldo, cudaStream_t s, bool* done);
bool amm_rt_applies(const TreesDev& t, const LutsDev& l, int es);
cudaError_t launch_encode_rt(const TreesDev& t, const float* A, int64_t N, int64_t lda,
                             uint8_t* codes, cudaStream_t s, bool* done);
cudaError_t launch_encode_rt_u8(const TreesDev& t, const uint8_t* A, int64_t N, int64_t lda,
                                uint8_t* codes, cudaStream_t s, bool* done);
// PQ encoder (mdn_pq.cu).
cudaError_t launch_encode_pq(const TreesDev& t, const float* P_dense, const uint16_t* sub_b,
                             const uint16_t* sub_e, const float* A, int64_t N, int64_t lda,
                             uint8_t* codes, cudaStream_t s);
// Column-major A (mdn_colmajor.cu).
cudaError_t launch_amm_cm(const TreesDev& t, const LutsDev& l, const float* At, int64_t N,
                          int64_t ldt, float* out, int64_t ldo, cudaStream_t s);
cudaError_t launch_encode_cm(const TreesDev& t, const float* At, int64_t N, int64_t ldt,
                             uint8_t* codes, cudaStream_t s);
// Warp-specialised TMA-gather4 variant of the fused path for column-major A
// (mdn_fast.cu); *done = false when not applicable (the caller then uses
// mdn_colmajor.cu's thread-per-row kernel).
cudaError_t launch_amm_ws_cm(const TreesDev& t, const LutsDev& l, const float* At, int64_t N,
                             int64_t ldt, float* out, int64_t ldo, cudaStream_t s, bool* done);
cudaError_t launch_encode_ws_cm(const TreesDev& t, const float* At, int64_t N, int64_t ldt,
                                uint8_t* codes, cudaStream_t s, bool* done);
const char* amm_variant_name(const TreesDev& t, const LutsDev& l, const float* A, int64_t lda,
                             const float* out, int64_t ldo);

// LUT build (device fp64), writes tq/words and the scalars.
struct LutScalars {
  int l;
  int err;        // 1 = |l| > 100
  float alpha;
  float beta32;
};
cudaError_t build_tables_dev(const float* dP, const float* dB, int C, int D, int M,
                             int U_or_0, double* dT, double* dDelta, double* dRange,
                             LutScalars* dScal, uint8_t* dTq, uint32_t* dWords,
                             uint32_t* dWords16, cudaStream_t s);
cudaError_t pack_words_dev(const uint8_t* dTq, int C, int M, uint32_t* dWords,
                           uint32_t* dWords16, cudaStream_t s);

uint64_t fnv1a64(const uint8_t* p, size_t n);

// GPU training (mdn_train.cu): trees + prototypes -> model.mdnm v1.
size_t train_blob_size(int C, int D);
cudaError_t train_model(const float* A, int64_t N, int64_t lda, int D, int C, double lam,
                        std::vector<uint8_t>& blob, int* err);

}  // namespace mdn

struct mdn_model {
  int device;
  int C, D;
  uint32_t flags;
  double lambda;
  uint64_t n_train, seed, fingerprint;
  std::vector<uint16_t> h_dims;   // [C][4]
  std::vector<float> h_thr;       // [C][16]
  std::vector<uint16_t> h_sub;    // [C] subspace begin
  std::vector<uint16_t> h_q;      // [C][16] 8-bit split values
  int subf = 0, subf_u8 = 0, q_byte = 0;
  std::vector<uint16_t> h_cols, h_slot;
  uint16_t* d_cols = nullptr;
  uint16_t* d_slot = nullptr;
  bool pq = false;                // flags bit1: PQ comparator model, no trees
  int pq_ds = 0;
  std::vector<uint16_t> h_sub_e;  // [C] subspace end
  uint16_t* d_sub_e = nullptr;
  float* d_pqcent = nullptr;      // [16][DS/4][C][4]
  uint16_t* d_dims = nullptr;
  float* d_thr = nullptr;
  uint16_t* d_sub = nullptr;
  uint16_t* d_q = nullptr;
  float* d_P = nullptr;           // [16C][D]
  mdn::TreesDev trees() const {
    return {d_dims, d_thr, d_sub, d_q, C, D, subf, subf_u8, q_byte, d_cols, d_slot,
            (int)h_cols.size(), d_pqcent, d_pqcent ? pq_ds : 0,
            h_dims.data(), h_sub.data(), h_q.data()};
  }
};

struct mdn_luts {
  int device;
  int C, M, W, mode, U, l;
  float alpha, beta32;
  uint64_t model_fp;
  std::vector<double> delta;
  uint8_t* d_tq = nullptr;       // [C][16][M]
  uint32_t* d_words = nullptr;   // [C][W][16]
  uint32_t* d_words16 = nullptr; // [C][16][W2], M <= 2 * MAX_W2 only
  mdn::LutsDev dev() const {
    float ae = mode == MDN_SUM_AVG ? alpha * (float)U : alpha;   // exact: power of two
    return {d_tq, d_words, d_words16, C, M, W, mode == MDN_SUM_AVG ? U : 0, ae, beta32};
  }
};
