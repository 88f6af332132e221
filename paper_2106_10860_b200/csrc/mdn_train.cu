// GPU training of the MADDNESS hash trees and prototypes.
//
// The offline step before the hot path (untimed in the paper),
// restated from Sec. 4.2-4.3 and App. C in the paper's order, with the same
// readings as the oracle (R1-R12):
//
//   per codebook c (subspace J^(c), R1/R2), 4 times Algorithm 2 (L272-305):
//     candidates  top-4 dims by L(j) = sum over buckets of the per-dim SSE
//                 (L265; ties -> lower index, R3), evaluated ascending
//     score       for each candidate j and bucket B: Algorithm 3 (L626-644)
//                 on B sorted by x_j -- prefix / suffix SSE over all subspace
//                 dims (Alg. 4, R4-R6), positions with x[n] < x[n+1] only
//                 (R7, R9), first minimum (R8); keep j if the bucket-summed
//                 loss is strictly smaller (L289)
//     split       children {x_j < v}, {x_j >= v} (L296-302, L240), order kept
//   prototypes    ridge P = (G^T G + lambda I)^-1 G^T A~ (L318-321) with G
//                 from the leaves (R12), or bucket means for lambda = 0 (L218)
//
// Device layout: the rows of each bucket are a contiguous range of `perm`
// (ascending row id inside a bucket, as the oracle's index arrays). Sorting a
// bucket by x_j is a CUB segmented stable sort (a library primitive); the
// prefix sums, losses, argmins and partitions are the kernels below; the SPD
// solve is cuSOLVER's Cholesky (potrf / potrs).
//
// Precision: fp64 statistics as the oracle; the loss of a position sums the
// subspace dims in ascending order. Block-parallel prefix sums add in a
// different order than the oracle's sequential cumsum, so on fp32 data a split
// whose loss ties another within rounding may differ (both are optimal to
// rounding); on integer-valued data (8-bit pixels) every sum is exact and the
// trees are bit-identical (tests/test_gpu_train.py).
#include <cuda_runtime.h>
#include <cusolverDn.h>

#include <cub/block/block_reduce.cuh>
#include <cub/block/block_scan.cuh>
#include <cub/device/device_segmented_sort.cuh>

#include <algorithm>
#include <array>
#include <cmath>
#include <cstring>
#include <vector>

#include "mdn_internal.h"

namespace mdn {
namespace train {

constexpr int TB = 256;   // threads per block of the per-bucket kernels
constexpr int BS = 17;    // bucket-offset stride per codebook (<= 16 buckets + 1)

// All codebooks are trained together: blockIdx.{y,z} selects the codebook c,
// whose rows sit in perm[c N ..), buckets at bstart[c BS ..), subspace at
// col0[c] with d[c] dims.

// L(j, B) for every subspace dim of every bucket (two-pass: mean, then squared
// deviations; L259). grid (nb, dmax, C); out[(c 16 + b) 64 + jj].
__global__ void k_dim_sse(const float* __restrict__ A, int64_t lda, const int* __restrict__ perm,
                          const int* __restrict__ bstart, const int* __restrict__ col0,
                          const int* __restrict__ dims_n, int N, double* __restrict__ out) {
  using BR = cub::BlockReduce<double, TB>;
  __shared__ typename BR::TempStorage tmp;
  __shared__ double s_mean;
  const int b = blockIdx.x, jj = blockIdx.y, c = blockIdx.z;
  if (jj >= dims_n[c]) return;
  const int* pc = perm + (size_t)c * N;
  const int s = bstart[c * BS + b], e = bstart[c * BS + b + 1], n = e - s;
  const int col = col0[c] + jj;
  double* o = out + ((size_t)c * 16 + b) * 64 + jj;
  if (n == 0) {
    if (threadIdx.x == 0) *o = 0.0;
    return;
  }
  double acc = 0.0;
  for (int i = s + threadIdx.x; i < e; i += TB) acc += (double)A[(int64_t)pc[i] * lda + col];
  double tot = BR(tmp).Sum(acc);
  if (threadIdx.x == 0) s_mean = tot / n;
  __syncthreads();
  const double mean = s_mean;
  acc = 0.0;
  for (int i = s + threadIdx.x; i < e; i += TB) {
    const double t = (double)A[(int64_t)pc[i] * lda + col] - mean;
    acc += t * t;
  }
  tot = BR(tmp).Sum(acc);
  if (threadIdx.x == 0) *o = tot;
}

// Sort keys for each codebook's candidate column: x_j of the rows in perm
// order (-0 -> +0). grid (x, C).
__global__ void k_gather_keys(const float* __restrict__ A, int64_t lda, const int* __restrict__ perm,
                              int N, const int* __restrict__ cols, float* __restrict__ keys,
                              int* __restrict__ vals) {
  const int c = blockIdx.y;
  const int col = cols[c];
  const size_t off = (size_t)c * N;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int r = perm[off + i];
    keys[off + i] = A[(int64_t)r * lda + col] + 0.0f;
    vals[off + i] = r;
  }
}

__device__ __forceinline__ float midpoint_threshold(float a, float b) {
  // Alg. 3 line 9 (L639) with reading R9: a < v <= b in fp32.
  float v = __double2float_rn(__dadd_rn((double)a, __ddiv_rn(__dsub_rn((double)b, (double)a), 2.0)));
  if (v <= a) v = nextafterf(a, INFINITY);
  return v;
}

// Algorithm 3 on every bucket of every codebook for one candidate column each,
// split over row tiles of TR rows so large buckets use many CTAs. Rows of
// bucket b of codebook c are keys/vals[c N + bstart[c BS + b] ..) sorted by x_j.
//   k_tile_sums      per (codebook, bucket, tile, dim): sum x, sum x^2
//   k_split_tiles    per tile: prefix sums = earlier tiles' sums (ascending) +
//                    in-tile block scans; the loss of every realisable
//                    position (Alg. 3 L634-635 with Alg. 4, dims
//                    ascending); the tile's first minimum
//   k_split_reduce   per bucket: first minimum over the tiles (R8), the
//                    threshold (R9) or the constant-column / empty cases
constexpr int TR = 4096;   // rows per tile
constexpr int DS = 64;     // per-dim stride of the tile sums (max subspace width)

__device__ __forceinline__ void bucket_range(const int* bstart, int c, int b, int tile, int& s,
                                             int& e, int& start, int& end) {
  s = bstart[c * BS + b], e = bstart[c * BS + b + 1];
  start = s + tile * TR;
  end = min(start + TR, e);
}

__global__ void __launch_bounds__(TB) k_tile_sums(const float* __restrict__ A, int64_t lda,
                                                  const int* __restrict__ vals_all,
                                                  const int* __restrict__ bstart,
                                                  const int* __restrict__ col0_a,
                                                  const int* __restrict__ dims_n, int Nrows, int Tmax,
                                                  double* __restrict__ tsum) {
  using BR = cub::BlockReduce<double, TB>;
  __shared__ typename BR::TempStorage tmp;
  const int tile = blockIdx.x, b = blockIdx.y, c = blockIdx.z;
  int s, e, start, end;
  bucket_range(bstart, c, b, tile, s, e, start, end);
  if (start >= e) return;
  const int* vals = vals_all + (size_t)c * Nrows;
  const int col0 = col0_a[c], d = dims_n[c];
  double* out = tsum + (((size_t)c * 16 + b) * Tmax + tile) * DS * 2;
  for (int jj = 0; jj < d; ++jj) {
    double a1 = 0.0, a2 = 0.0;
    for (int i = start + threadIdx.x; i < end; i += TB) {
      const double x = (double)A[(int64_t)vals[i] * lda + col0 + jj];
      a1 += x, a2 += x * x;
    }
    const double t1 = BR(tmp).Sum(a1);
    __syncthreads();
    const double t2 = BR(tmp).Sum(a2);
    if (threadIdx.x == 0) out[2 * jj] = t1, out[2 * jj + 1] = t2;
    __syncthreads();
  }
}

template <int DMAX>
__global__ void __launch_bounds__(TB) k_split_tiles(const float* __restrict__ A, int64_t lda,
                                                    const float* __restrict__ keys_all,
                                                    const int* __restrict__ vals_all,
                                                    const int* __restrict__ bstart,
                                                    const int* __restrict__ col0_a,
                                                    const int* __restrict__ dims_n, int Nrows,
                                                    int Tmax, const double* __restrict__ tsum,
                                                    double* __restrict__ tbest_l,
                                                    int* __restrict__ tbest_n) {
  using BSc = cub::BlockScan<double, TB>;
  __shared__ typename BSc::TempStorage scan_tmp;
  __shared__ double s_T1[DMAX], s_T2[DMAX], s_c1[DMAX], s_c2[DMAX];
  __shared__ double s_bl[TB];
  __shared__ int s_bn[TB];
  const int tile = blockIdx.x, b = blockIdx.y, c = blockIdx.z;
  int s, e, start, end;
  bucket_range(bstart, c, b, tile, s, e, start, end);
  if (start >= e) return;
  const float* keys = keys_all + (size_t)c * Nrows;
  const int* vals = vals_all + (size_t)c * Nrows;
  const int col0 = col0_a[c], d = dims_n[c];
  const int N = e - s;
  const int ntiles = (N + TR - 1) / TR;
  const double* ts = tsum + ((size_t)c * 16 + b) * Tmax * DS * 2;
  for (int jj = threadIdx.x; jj < d; jj += TB) {          // carry-in and totals, tiles ascending
    double c1 = 0.0, c2 = 0.0, t1 = 0.0, t2 = 0.0;
    for (int t = 0; t < ntiles; ++t) {
      const double v1 = ts[(size_t)t * DS * 2 + 2 * jj], v2 = ts[(size_t)t * DS * 2 + 2 * jj + 1];
      if (t < tile) c1 += v1, c2 += v2;
      t1 += v1, t2 += v2;
    }
    s_c1[jj] = c1, s_c2[jj] = c2, s_T1[jj] = t1, s_T2[jj] = t2;
  }
  __syncthreads();
  double best = INFINITY;
  int best_n = -1;
  for (int base = start; base < end; base += TB) {
    const int i = base + threadIdx.x;                      // absolute index in keys / vals
    const int n = i - s;                                   // position in the bucket (0-based)
    const bool in = i < end;
    const bool valid = in && n + 1 < N && keys[i] < keys[i + 1];     // R7 + R9
    const int row = in ? vals[i] : 0;
    double head = 0.0, tail = 0.0;
    for (int jj = 0; jj < d; ++jj) {
      const double x = in ? (double)A[(int64_t)row * lda + col0 + jj] : 0.0;
      double p1, p2, agg1, agg2;
      BSc(scan_tmp).InclusiveSum(x, p1, agg1);
      __syncthreads();
      BSc(scan_tmp).InclusiveSum(x * x, p2, agg2);
      __syncthreads();
      p1 += s_c1[jj], p2 += s_c2[jj];
      const double cnt = (double)(n + 1), rest = (double)(N - n - 1);
      head += p2 - p1 * p1 / cnt;                          // Alg. 4, dims ascending
      if (rest > 1) {                                      // rest == 1: L662's out[0] = 0
        const double r1 = s_T1[jj] - p1, r2 = s_T2[jj] - p2;
        tail += r2 - r1 * r1 / rest;
      }
      __syncthreads();
      if (threadIdx.x == TB - 1) s_c1[jj] += agg1, s_c2[jj] += agg2;
      __syncthreads();
    }
    if (n == 0) head = 0.0;                                // L662: out[0] = 0
    if (valid) {
      const double l = head + tail;                        // L634-635
      if (l < best) best = l, best_n = n;
    }
  }
  s_bl[threadIdx.x] = best;
  s_bn[threadIdx.x] = best_n;
  __syncthreads();
  if (threadIdx.x == 0) {
    double bl = INFINITY;
    int bn = -1;
    for (int t = 0; t < TB; ++t)                           // lowest position on ties (R8)
      if (s_bn[t] >= 0 && (s_bl[t] < bl || (s_bl[t] == bl && s_bn[t] < bn))) bl = s_bl[t], bn = s_bn[t];
    const size_t o = ((size_t)c * 16 + b) * Tmax + tile;
    tbest_l[o] = bl;
    tbest_n[o] = bn;
  }
}

__global__ void k_split_reduce(const float* __restrict__ keys_all, const int* __restrict__ bstart,
                               const int* __restrict__ dims_n, int Nrows, int Tmax,
                               const double* __restrict__ tsum, const double* __restrict__ tbest_l,
                               const int* __restrict__ tbest_n, double* __restrict__ loss_out,
                               float* __restrict__ thr_out) {
  const int b = blockIdx.x, c = blockIdx.y;
  if (threadIdx.x != 0) return;
  const int s = bstart[c * BS + b], e = bstart[c * BS + b + 1], N = e - s;
  const int ob = c * 16 + b;
  if (N == 0) {                                            // R10
    loss_out[ob] = 0.0, thr_out[ob] = 0.f;
    return;
  }
  const float* keys = keys_all + (size_t)c * Nrows;
  const int ntiles = (N + TR - 1) / TR;
  double bl = INFINITY;
  int bn = -1;
  for (int t = 0; t < ntiles; ++t) {                       // tiles ascending: strict < keeps the first
    const size_t o = (size_t)ob * Tmax + t;
    if (tbest_n[o] >= 0 && tbest_l[o] < bl) bl = tbest_l[o], bn = tbest_n[o];
  }
  if (bn < 0) {
    // constant column: (the value, SSE of the bucket), every row goes right
    const double* ts = tsum + (size_t)ob * Tmax * DS * 2;
    double sse = 0.0;
    for (int jj = 0; jj < dims_n[c]; ++jj) {
      double t1 = 0.0, t2 = 0.0;
      for (int t = 0; t < ntiles; ++t) t1 += ts[(size_t)t * DS * 2 + 2 * jj], t2 += ts[(size_t)t * DS * 2 + 2 * jj + 1];
      sse += t2 - t1 * t1 / (double)N;
    }
    loss_out[ob] = sse;
    thr_out[ob] = keys[s];
  } else {
    loss_out[ob] = bl;
    thr_out[ob] = midpoint_threshold(keys[s + bn], keys[s + bn + 1]);
  }
}

// Stable partition of each bucket by x_j >= v (L296-302): left child 2b,
// right child 2b+1, ascending row id kept inside each. grid (nb, C).
__global__ void k_partition(const float* __restrict__ A, int64_t lda, const int* __restrict__ perm_all,
                            const int* __restrict__ bstart, int Nrows, const int* __restrict__ cols,
                            const float* __restrict__ thr, int* __restrict__ perm_out_all,
                            int* __restrict__ nleft_out) {
  using BSi = cub::BlockScan<int, TB>;
  using BR = cub::BlockReduce<int, TB>;
  __shared__ typename BSi::TempStorage scan_tmp;
  __shared__ typename BR::TempStorage red_tmp;
  __shared__ int s_left, s_carry_l, s_carry_r;
  const int b = blockIdx.x, c = blockIdx.y;
  const int* perm = perm_all + (size_t)c * Nrows;
  int* perm_out = perm_out_all + (size_t)c * Nrows;
  const int col = cols[c];
  const int s = bstart[c * BS + b], e = bstart[c * BS + b + 1];
  const float v = thr[c * 16 + b];
  int cl = 0;
  for (int i = s + threadIdx.x; i < e; i += TB) cl += (A[(int64_t)perm[i] * lda + col] < v) ? 1 : 0;
  const int nl = BR(red_tmp).Sum(cl);
  if (threadIdx.x == 0) s_left = nl, s_carry_l = 0, s_carry_r = 0, nleft_out[c * 16 + b] = nl;
  __syncthreads();
  const int left_total = s_left;
  for (int base = s; base < e; base += TB) {
    const int i = base + threadIdx.x;
    const bool in = i < e;
    const int r = in ? perm[i] : 0;
    const int isl = in && A[(int64_t)r * lda + col] < v ? 1 : 0;
    const int isr = in && !isl ? 1 : 0;
    int pl, pr, al, ar;
    BSi(scan_tmp).ExclusiveSum(isl, pl, al);
    __syncthreads();
    BSi(scan_tmp).ExclusiveSum(isr, pr, ar);
    if (isl) perm_out[s + s_carry_l + pl] = r;
    if (isr) perm_out[s + left_total + s_carry_r + pr] = r;
    __syncthreads();
    if (threadIdx.x == 0) s_carry_l += al, s_carry_r += ar;
    __syncthreads();
  }
}

// codes[row * C + c] = leaf of row for codebook c. grid (16, C).
__global__ void k_leaf_codes(const int* __restrict__ perm, const int* __restrict__ bstart, int N,
                             int C, uint8_t* __restrict__ codes) {
  const int b = blockIdx.x, c = blockIdx.y;
  const int* pc = perm + (size_t)c * N;
  for (int i = bstart[c * BS + b] + threadIdx.x; i < bstart[c * BS + b + 1]; i += blockDim.x)
    codes[(int64_t)pc[i] * C + c] = (uint8_t)b;
}

// G^T G co-occurrence counts (L318): M[(c,k),(c',k')] += 1 per row.
__global__ void k_gtg(const uint8_t* __restrict__ codes, int N, int C, unsigned* __restrict__ M) {
  const int KC = 16 * C;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < (int64_t)N * C * C;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int row = (int)(i / ((int64_t)C * C));
    const int cc = (int)(i % ((int64_t)C * C));
    const int c1 = cc / C, c2 = cc % C;
    const int a = 16 * c1 + codes[(int64_t)row * C + c1], bb = 16 * c2 + codes[(int64_t)row * C + c2];
    atomicAdd(&M[(int64_t)a * KC + bb], 1u);
  }
}

// G^T A~ for one leaf (c, k): sum of its rows over every column j (leaf rows
// are the contiguous perm range of the final level). Column-major for potrs:
// out[j * KC + 16c + k]. With bucket means (lambda = 0) the mean is taken
// over the subspace only and written row-major into P directly.
__global__ void k_gta(const float* __restrict__ A, int64_t lda, int D, const int* __restrict__ perm_all,
                      const int* __restrict__ bstart, int N, int KC, double* __restrict__ GtA) {
  using BR = cub::BlockReduce<double, TB>;
  __shared__ typename BR::TempStorage tmp;
  const int k = blockIdx.x % 16, c = blockIdx.x / 16;      // grid (16 C, column blocks)
  const int* perm = perm_all + (size_t)c * N;
  const int s = bstart[c * BS + k], e = bstart[c * BS + k + 1];
  for (int j = blockIdx.y; j < D; j += gridDim.y) {
    double acc = 0.0;
    for (int i = s + threadIdx.x; i < e; i += TB) acc += (double)A[(int64_t)perm[i] * lda + j];
    const double tot = BR(tmp).Sum(acc);
    if (threadIdx.x == 0) GtA[(int64_t)j * KC + 16 * c + k] = tot;
    __syncthreads();
  }
}

__global__ void k_add_ridge(const unsigned* __restrict__ cnt, double* __restrict__ M, int KC,
                            double lam) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < (int64_t)KC * KC;
       i += (int64_t)gridDim.x * blockDim.x)
    M[i] = (double)cnt[i] + ((i / KC) == (i % KC) ? lam : 0.0);
}

}  // namespace train

using namespace train;

namespace {

struct DevBuf {
  std::vector<void*> ptrs;
  template <class T>
  T* get(size_t n) {
    void* p = nullptr;
    if (cudaMalloc(&p, (n ? n : 1) * sizeof(T)) != cudaSuccess) return nullptr;
    ptrs.push_back(p);
    return static_cast<T*>(p);
  }
  ~DevBuf() {
    for (void* p : ptrs) cudaFree(p);
  }
};

template <class T>
void put(std::vector<uint8_t>& o, T v) {
  const uint8_t* b = reinterpret_cast<const uint8_t*>(&v);
  o.insert(o.end(), b, b + sizeof(T));
}

}  // namespace

size_t train_blob_size(int C, int D) { return 48 + (size_t)76 * C + (size_t)64 * C * D + 8; }

// Trains on device rows A (N x D, lda) and serialises "model.mdnm v1" into
// `blob`. Returns a cudaError_t; *err = MDN_* for non-CUDA failures.
cudaError_t train_model(const float* A, int64_t N64, int64_t lda, int D, int C, double lam,
                        std::vector<uint8_t>& blob, int* err) {
  *err = MDN_OK;
  const int N = (int)N64;
  const int KC = 16 * C;
  // R1: contiguous subspaces, the first D mod C one column wider.
  std::vector<int> sb(C), se(C);
  {
    const int base = D / C, extra = D % C;
    int b = 0;
    for (int c = 0; c < C; ++c) {
      sb[c] = b;
      b += base + (c < extra ? 1 : 0);
      se[c] = b;
    }
  }
  int dmax = 0;
  for (int c = 0; c < C; ++c) dmax = std::max(dmax, se[c] - sb[c]);
  if (dmax > 64) {
    *err = MDN_EINVAL;     // the split-loss kernel keeps <= 64 per-dim totals in shared memory
    return cudaSuccess;
  }
  DevBuf buf;
  const size_t CN = (size_t)C * N;
  int* perm = buf.get<int>(CN);
  int* perm2 = buf.get<int>(CN);
  int* vals = buf.get<int>(CN);
  int* vals_s = buf.get<int>(CN);
  float* keys = buf.get<float>(CN);
  float* keys_s = buf.get<float>(CN);
  int* d_bstart = buf.get<int>((size_t)C * BS);
  int* d_nleft = buf.get<int>((size_t)C * 16);
  int* d_col0 = buf.get<int>(C);
  int* d_dn = buf.get<int>(C);
  int* d_cols = buf.get<int>(C);
  int* d_segb = buf.get<int>((size_t)C * 8);
  int* d_sege = buf.get<int>((size_t)C * 8);
  double* d_L = buf.get<double>((size_t)C * 16 * 64);
  double* d_loss = buf.get<double>((size_t)C * 16);
  const int Tmax = (N + TR - 1) / TR;
  double* d_tsum = buf.get<double>((size_t)C * 16 * Tmax * DS * 2);
  double* d_tbl = buf.get<double>((size_t)C * 16 * Tmax);
  int* d_tbn = buf.get<int>((size_t)C * 16 * Tmax);
  float* d_thr = buf.get<float>((size_t)C * 16);
  uint8_t* d_codes = buf.get<uint8_t>((size_t)N * C);
  unsigned* d_cnt = buf.get<unsigned>((size_t)KC * KC);
  double* d_M = buf.get<double>((size_t)KC * KC);
  double* d_GtA = buf.get<double>((size_t)KC * D);
  if (!perm || !perm2 || !vals || !vals_s || !keys || !keys_s || !d_bstart || !d_nleft || !d_col0 ||
      !d_dn || !d_cols || !d_segb || !d_sege || !d_L || !d_loss || !d_thr || !d_codes || !d_cnt ||
      !d_M || !d_GtA || !d_tsum || !d_tbl || !d_tbn) {
    *err = MDN_ENOMEM;
    return cudaSuccess;
  }
  cudaError_t e = cudaMemset(d_GtA, 0, (size_t)KC * D * sizeof(double));
  if (e != cudaSuccess) return e;
  auto h2d = [&](void* dst, const void* src, size_t bytes) {
    return cudaMemcpy(dst, src, bytes, cudaMemcpyHostToDevice);
  };
  auto d2h = [&](void* dst, const void* src, size_t bytes) {
    return cudaMemcpy(dst, src, bytes, cudaMemcpyDeviceToHost);
  };
  {
    std::vector<int> h_perm(CN), dn(C);
    for (int c = 0; c < C; ++c) {
      dn[c] = se[c] - sb[c];
      for (int i = 0; i < N; ++i) h_perm[(size_t)c * N + i] = i;
    }
    if ((e = h2d(perm, h_perm.data(), CN * 4)) != cudaSuccess) return e;
    if ((e = h2d(d_col0, sb.data(), C * 4)) != cudaSuccess) return e;
    if ((e = h2d(d_dn, dn.data(), C * 4)) != cudaSuccess) return e;
  }
  // CUB temp storage (sized for the largest call: C N items, 8 C segments)
  size_t cub_bytes = 0;
  for (int nseg : {1, 2, 4, 8}) {
    size_t bb = 0;
    cub::DeviceSegmentedSort::StableSortPairs(nullptr, bb, keys, keys_s, vals, vals_s, (int)CN,
                                              nseg * C, d_segb, d_sege);
    cub_bytes = std::max(cub_bytes, bb);
  }
  void* cub_tmp = buf.get<uint8_t>(cub_bytes);
  if (!cub_tmp) {
    *err = MDN_ENOMEM;
    return cudaSuccess;
  }
  std::vector<uint16_t> dims((size_t)C * 4);
  std::vector<float> thr((size_t)C * 15, 0.f);
  const int gk_blocks = std::min(1024, (N + 255) / 256);
  // bucket offsets per codebook, host side: bst[c * BS + b]
  std::vector<int> bst((size_t)C * BS, 0);
  for (int c = 0; c < C; ++c) bst[(size_t)c * BS + 1] = N;
  for (int t = 0; t < 4; ++t) {
    const int nb = 1 << t;
    if ((e = h2d(d_bstart, bst.data(), bst.size() * 4)) != cudaSuccess) return e;
    // candidates (L265): top-4 of L(j) summed over buckets in bucket order
    k_dim_sse<<<dim3(nb, dmax, C), TB>>>(A, lda, perm, d_bstart, d_col0, d_dn, N, d_L);
    std::vector<double> hL((size_t)C * 16 * 64);
    if ((e = d2h(hL.data(), d_L, hL.size() * 8)) != cudaSuccess) return e;
    std::vector<std::array<int, 4>> cand(C);
    for (int c = 0; c < C; ++c) {
      const int d = se[c] - sb[c];
      std::vector<double> L(d, 0.0);
      for (int b = 0; b < nb; ++b)
        for (int jj = 0; jj < d; ++jj) L[jj] += hL[((size_t)c * 16 + b) * 64 + jj];
      std::vector<int> order(d);
      for (int jj = 0; jj < d; ++jj) order[jj] = jj;
      std::stable_sort(order.begin(), order.end(), [&](int x, int y) { return L[x] > L[y]; });
      std::vector<int> cs(order.begin(), order.begin() + std::min(4, d));
      std::sort(cs.begin(), cs.end());
      for (int q = 0; q < 4; ++q) cand[c][q] = cs[std::min(q, (int)cs.size() - 1)];   // pad: re-evaluation ties, kept out by L289's strict <
    }
    // segments of the sort: bucket b of codebook c
    {
      std::vector<int> sbg((size_t)C * nb), seg((size_t)C * nb);
      for (int c = 0; c < C; ++c)
        for (int b = 0; b < nb; ++b) {
          sbg[(size_t)c * nb + b] = (int)((size_t)c * N + bst[(size_t)c * BS + b]);
          seg[(size_t)c * nb + b] = (int)((size_t)c * N + bst[(size_t)c * BS + b + 1]);
        }
      if ((e = h2d(d_segb, sbg.data(), sbg.size() * 4)) != cudaSuccess) return e;
      if ((e = h2d(d_sege, seg.data(), seg.size() * 4)) != cudaSuccess) return e;
    }
    int tiles_lv = 1;                                  // tiles of the largest bucket
    for (int c = 0; c < C; ++c)
      for (int b = 0; b < nb; ++b)
        tiles_lv = std::max(tiles_lv, (bst[(size_t)c * BS + b + 1] - bst[(size_t)c * BS + b] + TR - 1) / TR);
    // score each candidate (Alg. 2 l.4-15), all codebooks at once
    std::vector<double> l_min(C, INFINITY);
    std::vector<int> j_min(C, -1);
    std::vector<float> v_min((size_t)C * 16, 0.f);
    for (int q = 0; q < 4; ++q) {
      std::vector<int> cols(C);
      for (int c = 0; c < C; ++c) cols[c] = sb[c] + cand[c][q];
      if ((e = h2d(d_cols, cols.data(), C * 4)) != cudaSuccess) return e;
      k_gather_keys<<<dim3(gk_blocks, C), 256>>>(A, lda, perm, N, d_cols, keys, vals);
      size_t bytes = cub_bytes;
      e = cub::DeviceSegmentedSort::StableSortPairs(cub_tmp, bytes, keys, keys_s, vals, vals_s, (int)CN,
                                                    nb * C, d_segb, d_sege);
      if (e != cudaSuccess) return e;
      const dim3 tg(tiles_lv, nb, C);
      k_tile_sums<<<tg, TB>>>(A, lda, vals_s, d_bstart, d_col0, d_dn, N, Tmax, d_tsum);
      if (dmax <= 16)
        k_split_tiles<16><<<tg, TB>>>(A, lda, keys_s, vals_s, d_bstart, d_col0, d_dn, N, Tmax, d_tsum,
                                      d_tbl, d_tbn);
      else
        k_split_tiles<64><<<tg, TB>>>(A, lda, keys_s, vals_s, d_bstart, d_col0, d_dn, N, Tmax, d_tsum,
                                      d_tbl, d_tbn);
      k_split_reduce<<<dim3(nb, C), 32>>>(keys_s, d_bstart, d_dn, N, Tmax, d_tsum, d_tbl, d_tbn, d_loss,
                                          d_thr);
      std::vector<double> hl((size_t)C * 16);
      std::vector<float> hv((size_t)C * 16);
      if ((e = d2h(hl.data(), d_loss, hl.size() * 8)) != cudaSuccess) return e;
      if ((e = d2h(hv.data(), d_thr, hv.size() * 4)) != cudaSuccess) return e;
      for (int c = 0; c < C; ++c) {
        double l = 0.0;
        for (int b = 0; b < nb; ++b) l += hl[(size_t)c * 16 + b];          // L287, bucket order
        if (l < l_min[c]) {                                                  // L289 (strict)
          l_min[c] = l, j_min[c] = cand[c][q];
          for (int b = 0; b < nb; ++b) v_min[(size_t)c * 16 + b] = hv[(size_t)c * 16 + b];
        }
      }
    }
    std::vector<int> cols(C);
    for (int c = 0; c < C; ++c) {
      cols[c] = sb[c] + j_min[c];
      dims[(size_t)c * 4 + t] = (uint16_t)cols[c];
      for (int b = 0; b < nb; ++b) thr[(size_t)c * 15 + (1 << t) - 1 + b] = v_min[(size_t)c * 16 + b];
    }
    // split (L296-302)
    if ((e = h2d(d_cols, cols.data(), C * 4)) != cudaSuccess) return e;
    if ((e = h2d(d_thr, v_min.data(), v_min.size() * 4)) != cudaSuccess) return e;
    k_partition<<<dim3(nb, C), TB>>>(A, lda, perm, d_bstart, N, d_cols, d_thr, perm2, d_nleft);
    std::vector<int> nl((size_t)C * 16);
    if ((e = d2h(nl.data(), d_nleft, nl.size() * 4)) != cudaSuccess) return e;
    std::vector<int> nbst((size_t)C * BS, 0);
    for (int c = 0; c < C; ++c) {
      for (int b = 0; b < nb; ++b) {
        nbst[(size_t)c * BS + 2 * b] = bst[(size_t)c * BS + b];
        nbst[(size_t)c * BS + 2 * b + 1] = bst[(size_t)c * BS + b] + nl[(size_t)c * 16 + b];
      }
      nbst[(size_t)c * BS + 2 * nb] = N;
    }
    bst.swap(nbst);
    std::swap(perm, perm2);
  }
  // leaves -> codes (R12: membership == re-encoding under R9) and G^T A~
  if ((e = h2d(d_bstart, bst.data(), bst.size() * 4)) != cudaSuccess) return e;
  k_leaf_codes<<<dim3(16, C), 256>>>(perm, d_bstart, N, C, d_codes);
  k_gta<<<dim3(16 * C, std::min(D, 256)), TB>>>(A, lda, D, perm, d_bstart, N, KC, d_GtA);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  // prototypes
  std::vector<float> P((size_t)KC * D, 0.f);
  std::vector<double> X((size_t)KC * D);
  if (lam > 0) {
    if ((e = cudaMemset(d_cnt, 0, (size_t)KC * KC * 4)) != cudaSuccess) return e;
    k_gtg<<<4096, 256>>>(d_codes, N, C, d_cnt);
    k_add_ridge<<<1024, 256>>>(d_cnt, d_M, KC, lam);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    cusolverDnHandle_t h = nullptr;
    if (cusolverDnCreate(&h) != CUSOLVER_STATUS_SUCCESS) {
      *err = MDN_ECUDA;
      return cudaSuccess;
    }
    int lwork = 0;
    int* d_info = buf.get<int>(1);
    cusolverStatus_t cs = cusolverDnDpotrf_bufferSize(h, CUBLAS_FILL_MODE_LOWER, KC, d_M, KC, &lwork);
    double* work = buf.get<double>((size_t)std::max(lwork, 1));
    if (cs == CUSOLVER_STATUS_SUCCESS)
      cs = cusolverDnDpotrf(h, CUBLAS_FILL_MODE_LOWER, KC, d_M, KC, work, lwork, d_info);
    if (cs == CUSOLVER_STATUS_SUCCESS)
      cs = cusolverDnDpotrs(h, CUBLAS_FILL_MODE_LOWER, KC, D, d_M, KC, d_GtA, KC, d_info);
    cusolverDnDestroy(h);
    int info = 0;
    if ((e = cudaMemcpy(&info, d_info, 4, cudaMemcpyDeviceToHost)) != cudaSuccess) return e;
    if (cs != CUSOLVER_STATUS_SUCCESS || info != 0) {
      *err = MDN_ECUDA;
      return cudaSuccess;
    }
    if ((e = cudaMemcpy(X.data(), d_GtA, X.size() * 8, cudaMemcpyDeviceToHost)) != cudaSuccess) return e;
    for (int ck = 0; ck < KC; ++ck)
      for (int j = 0; j < D; ++j) P[(size_t)ck * D + j] = (float)X[(size_t)j * KC + ck];
  } else {
    // bucket means over the subspace (L218, MADDNESS-PQ), zero for empty leaves (R10)
    std::vector<uint8_t> hc((size_t)N * C);
    if ((e = cudaMemcpy(X.data(), d_GtA, X.size() * 8, cudaMemcpyDeviceToHost)) != cudaSuccess) return e;
    if ((e = cudaMemcpy(hc.data(), d_codes, hc.size(), cudaMemcpyDeviceToHost)) != cudaSuccess) return e;
    std::vector<int64_t> cnt((size_t)KC, 0);
    for (int n = 0; n < N; ++n)
      for (int c = 0; c < C; ++c) cnt[16 * c + hc[(size_t)n * C + c]]++;
    for (int c = 0; c < C; ++c)
      for (int k = 0; k < 16; ++k) {
        const int ck = 16 * c + k;
        if (!cnt[ck]) continue;
        for (int j = sb[c]; j < se[c]; ++j) P[(size_t)ck * D + j] = (float)(X[(size_t)j * KC + ck] / cnt[ck]);
      }
  }
  // serialise model.mdnm v1 (include/maddness.h)
  blob.clear();
  blob.insert(blob.end(), {'M', 'D', 'N', 'M'});
  put<uint32_t>(blob, 1);
  put<uint32_t>(blob, (uint32_t)C);
  put<uint32_t>(blob, (uint32_t)D);
  put<uint32_t>(blob, 16);
  put<uint32_t>(blob, lam > 0 ? 1u : 0u);
  put<double>(blob, lam);
  put<uint64_t>(blob, (uint64_t)N);
  put<uint64_t>(blob, 0);
  for (int c = 0; c < C; ++c) {
    put<uint32_t>(blob, (uint32_t)sb[c]);
    put<uint32_t>(blob, (uint32_t)se[c]);
    for (int t = 0; t < 4; ++t) put<uint16_t>(blob, dims[(size_t)c * 4 + t]);
    for (int i = 0; i < 15; ++i) put<float>(blob, thr[(size_t)c * 15 + i]);
  }
  const uint8_t* pb = reinterpret_cast<const uint8_t*>(P.data());
  blob.insert(blob.end(), pb, pb + P.size() * 4);
  put<uint64_t>(blob, fnv1a64(blob.data(), blob.size()));
  return cudaSuccess;
}

}  // namespace mdn
