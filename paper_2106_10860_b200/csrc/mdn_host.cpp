// libmaddness host side: file parsing, handle lifetime, validation, dispatch,
// and the pipelined host-buffer executor. See include/maddness.h for the
// contract of every entry point.
#include <cuda_runtime.h>
#include <string.h>

#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <memory>
#include <mutex>
#include <new>
#include <vector>

#include <nvtx3/nvToolsExt.h>   // header-only NVTX3: no-ops unless a profiler attaches

#include "mdn_internal.h"

namespace mdn {

cudaError_t launch_amm_probe(const TreesDev& t, const LutsDev& l, const float* A, int64_t N,
                             int64_t lda, float* out, int64_t ldo, cudaStream_t s, bool* done);
cudaError_t launch_stream_probe(const float* A, int64_t N, int64_t lda, int D, float* out,
                                int64_t ldo, int M, cudaStream_t s);

uint64_t fnv1a64(const uint8_t* p, size_t n) {
  uint64_t h = 0xCBF29CE484222325ull;
  for (size_t i = 0; i < n; ++i) {
    h ^= p[i];
    h *= 0x100000001B3ull;
  }
  return h;
}

namespace {

// Makes `dev` current for the scope of an entry point, restoring the caller's.
struct DeviceGuard {
  int prev = -1;
  bool ok = true;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    if (prev != dev) ok = cudaSetDevice(dev) == cudaSuccess;
  }
  ~DeviceGuard() {
    int cur = -1;
    if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
  }
};

struct Reader {
  const uint8_t* p;
  size_t len, off = 0;
  bool fail = false;
  size_t fail_off = 0;
  template <class T>
  T get() {
    T v{};
    if (off + sizeof(T) > len) {
      if (!fail) fail_off = off;
      fail = true;
      return v;
    }
    memcpy(&v, p + off, sizeof(T));
    off += sizeof(T);
    return v;
  }
  bool need(size_t n) {
    if (off + n > len) {
      if (!fail) fail_off = off;
      fail = true;
    }
    return !fail;
  }
};

template <class T>
void put(std::vector<uint8_t>& o, T v) {
  const uint8_t* b = reinterpret_cast<const uint8_t*>(&v);
  o.insert(o.end(), b, b + sizeof(T));
}

int cuda_status(cudaError_t e) {
  if (e == cudaSuccess) return MDN_OK;
  static const bool debug = getenv("MDN_DEBUG") != nullptr;
  if (debug) fprintf(stderr, "libmaddness: CUDA error %d: %s\n", (int)e, cudaGetErrorString(e));
  if (e == cudaErrorMemoryAllocation) return MDN_ENOMEM;
  return MDN_ECUDA;
}

template <class T>
int dalloc(T** p, size_t count) {
  *p = nullptr;
  if (count == 0) count = 1;
  cudaError_t e = cudaMalloc(reinterpret_cast<void**>(p), count * sizeof(T));
  return cuda_status(e);
}

bool is_pow2(int u) { return u >= 1 && (u & (u - 1)) == 0; }

// The fast kernels address rows with 32-bit TMA coordinates; larger calls
// run as consecutive 2^30-row launches on the same stream (an 8-bit A of
// 2^31 rows x 32 bytes fits a 180 GB B200).
// MDN_ROW_CHUNK (a multiple of 256) overrides the chunk for tests.
int64_t row_chunk() {
  static const int64_t v = [] {
    const char* e = getenv("MDN_ROW_CHUNK");
    const int64_t c = e ? atoll(e) : 0;
    return c >= 256 && c % 256 == 0 && c <= (int64_t(1) << 30) ? c : int64_t(1) << 30;
  }();
  return v;
}

template <class F>
cudaError_t for_row_chunks(int64_t N, F&& launch) {
  const int64_t ch = row_chunk();
  cudaError_t e = cudaSuccess;
  for (int64_t r0 = 0; r0 < N && e == cudaSuccess; r0 += ch) e = launch(r0, N - r0 < ch ? N - r0 : ch);
  return e;
}

int set_err(size_t* err_off, size_t off, int st) {
  if (err_off) *err_off = off;
  return st;
}

}  // namespace
}  // namespace mdn

using namespace mdn;

extern "C" {

const char* mdn_status_str(int s) {
  switch (s) {
    case MDN_OK: return "ok";
    case MDN_EINVAL: return "invalid argument";
    case MDN_ESHAPE: return "shape mismatch";
    case MDN_EFORMAT: return "bad or truncated stream";
    case MDN_EVERSION: return "unsupported format version";
    case MDN_ESTATE: return "luts were not built from this model";
    case MDN_ECUDA: return "CUDA error";
    case MDN_ENOMEM: return "out of memory";
    case MDN_ERANGE: return "table scale exponent out of range";
    default: return "unknown status";
  }
}

int mdn_abi_version(void) { return MDN_ABI_VERSION; }

// ----------------------------------------------------------------- model --

void mdn_model_free(mdn_model* m) {
  if (!m) return;
  {
    DeviceGuard g(m->device);
    cudaFree(m->d_dims);
    cudaFree(m->d_thr);
    cudaFree(m->d_P);
    cudaFree(m->d_sub);
    cudaFree(m->d_q);
    cudaFree(m->d_cols);
    cudaFree(m->d_slot);
    cudaFree(m->d_sub_e);
    cudaFree(m->d_pqcent);
  }
  delete m;
}

int mdn_model_load(const void* buf, size_t len, int device, mdn_model** out, size_t* err_off) {
  if (!buf || !out) return MDN_EINVAL;
  *out = nullptr;
  Reader r{static_cast<const uint8_t*>(buf), len};
  if (!r.need(48) || memcmp(r.p, "MDNM", 4) != 0) return set_err(err_off, 0, MDN_EFORMAT);
  r.off = 4;
  uint32_t ver = r.get<uint32_t>(), C = r.get<uint32_t>(), D = r.get<uint32_t>();
  uint32_t k = r.get<uint32_t>(), flags = r.get<uint32_t>();
  if (ver != 1) return set_err(err_off, 4, MDN_EVERSION);
  if (k != (uint32_t)K) return set_err(err_off, 16, MDN_EINVAL);
  if (C < 1 || C > (uint32_t)MAX_C || D < 1 || D > 65535 || C > D)
    return set_err(err_off, 8, MDN_EINVAL);
  std::unique_ptr<mdn_model> m(new (std::nothrow) mdn_model());
  if (!m) return MDN_ENOMEM;
  m->device = device;
  m->C = (int)C;
  m->D = (int)D;
  m->flags = flags;
  m->lambda = r.get<double>();
  m->n_train = r.get<uint64_t>();
  m->seed = r.get<uint64_t>();
  m->h_dims.assign((size_t)C * 4, 0);
  m->h_thr.assign((size_t)C * THR_STRIDE, 0.f);
  m->h_sub.assign(C, 0);
  m->h_sub_e.assign(C, 0);
  m->pq = (flags & 2u) != 0;
  int max_w = 0;
  bool aligned = true;
  for (uint32_t c = 0; c < C; ++c) {
    size_t rec = r.off;
    uint32_t b = r.get<uint32_t>(), e = r.get<uint32_t>();
    m->h_sub[c] = (uint16_t)b;
    m->h_sub_e[c] = (uint16_t)e;
    if ((int)(e - b) > max_w) max_w = (int)(e - b);
    if (b % 4) aligned = false;
    for (int t = 0; t < 4; ++t) m->h_dims[c * 4 + t] = r.get<uint16_t>();
    for (int i = 0; i < 15; ++i) m->h_thr[c * THR_STRIDE + i] = r.get<float>();
    if (r.fail) return set_err(err_off, r.fail_off, MDN_EFORMAT);
    if (b > e || e > D) return set_err(err_off, rec, MDN_EFORMAT);
    // a NaN threshold has no 8-bit split value and no meaning in Alg. 1
    for (int i = 0; i < 15; ++i)
      if (std::isnan(m->h_thr[c * THR_STRIDE + i])) return set_err(err_off, rec + 16 + 4 * i, MDN_EINVAL);
    for (int t = 0; t < 4; ++t) {
      if (m->h_dims[c * 4 + t] >= D) return set_err(err_off, rec + 8 + 2 * t, MDN_EINVAL);
      // split dims must lie in the codebook's subspace (reading R2)
      if (m->h_dims[c * 4 + t] < b || m->h_dims[c * 4 + t] >= e)
        return set_err(err_off, rec + 8 + 2 * t, MDN_EFORMAT);
    }
  }
  m->subf = aligned && max_w <= 4 ? 1 : (aligned && max_w <= 8 ? 2 : 0);
  // uint8 input: every subspace exactly 4 (or 8) bytes, back to back
  m->subf_u8 = 0;
  for (int w : {4, 8}) {
    bool ok = (int)D == w * (int)C;
    for (uint32_t c = 0; c < C && ok; ++c) ok = m->h_sub[c] == w * c;
    if (ok) m->subf_u8 = w / 4;
  }
  // App. B 8-bit split values for natively 8-bit x (reading R11): q = ceil(v),
  // clamped to [0, 256] so that x >= q <=> x >= v for every byte x.
  m->h_q.assign((size_t)C * THR_STRIDE, 0);
  for (size_t i = 0; i < m->h_q.size(); ++i) {
    double q = std::ceil((double)m->h_thr[i]);
    m->h_q[i] = (uint16_t)(q < 0 ? 0 : (q > 256 ? 256 : q));
  }
  // Distinct split columns (column-major A reads only these).
  m->h_slot.assign(D, 0xFFFF);
  for (size_t i = 0; i < m->h_dims.size(); ++i) m->h_slot[m->h_dims[i]] = 0;
  for (uint32_t d = 0; d < D; ++d)
    if (m->h_slot[d] == 0) {
      m->h_slot[d] = (uint16_t)m->h_cols.size();
      m->h_cols.push_back((uint16_t)d);
    }
  m->q_byte = 1;
  for (uint32_t cc = 0; cc < C; ++cc)
    for (int i = 0; i < 15; ++i) m->q_byte &= m->h_q[cc * THR_STRIDE + i] <= 255 ? 1 : 0;
  size_t p_bytes = (size_t)K * C * D * sizeof(float);
  if (!r.need(p_bytes + 8)) return set_err(err_off, r.fail_off, MDN_EFORMAT);
  const uint8_t* P = r.p + r.off;
  r.off += p_bytes;
  uint64_t fp_stored = r.get<uint64_t>();
  uint64_t fp = fnv1a64(r.p, r.off - 8);
  if (fp != fp_stored) return set_err(err_off, r.off - 8, MDN_EFORMAT);
  m->fingerprint = fp;
  // PQ model (flags bit1): prototypes re-laid out [16][DS/4][C][4]
  // for the fast encoder when every subspace is [c DS, (c+1) DS), DS in
  // {4, 8, 16, 32} and C divides 256 (else the generic PQ kernel reads P).
  std::vector<float> h_pqcent;
  if (m->pq) {
    const int DS = (int)(D / C);
    bool eq = (int)D == DS * (int)C && (DS == 4 || DS == 8 || DS == 16 || DS == 32) &&
              256 % C == 0 && C % 2 == 0;
    for (uint32_t cc = 0; cc < C && eq; ++cc) eq = m->h_sub[cc] == DS * cc && m->h_sub_e[cc] == DS * (cc + 1);
    if (eq) {
      // fast encoder operands of the expanded form ||p||^2 - 2 <a, p> (reading
      // P1): q = -2 p (exact in fp32) in [k][j/4][c][4], then ||p_k||^2 of
      // every (k, c) summed in fp64 and rounded once, [k][c]
      m->pq_ds = DS;
      h_pqcent.assign((size_t)16 * D + 16 * C, 0.f);
      for (int k = 0; k < 16; ++k)
        for (uint32_t cc = 0; cc < C; ++cc) {
          double pn = 0.0;
          for (int j = 0; j < DS; ++j) {
            float v;
            memcpy(&v, P + (((size_t)(16 * cc + k) * D + cc * DS + j) * 4), 4);
            h_pqcent[(((size_t)k * (DS / 4) + j / 4) * C + cc) * 4 + (j % 4)] = -2.0f * v;
            pn += (double)v * (double)v;
          }
          h_pqcent[(size_t)16 * D + (size_t)k * C + cc] = (float)pn;
        }
    }
  }

  DeviceGuard g(device);
  if (!g.ok) return MDN_ECUDA;
  int st;
  if ((st = dalloc(&m->d_dims, m->h_dims.size())) != MDN_OK) return st;
  if ((st = dalloc(&m->d_thr, m->h_thr.size())) != MDN_OK) {
    mdn_model_free(m.release());
    return st;
  }
  if ((st = dalloc(&m->d_P, (size_t)K * C * D)) != MDN_OK ||
      (st = dalloc(&m->d_sub, (size_t)C)) != MDN_OK ||
      (st = dalloc(&m->d_q, m->h_q.size())) != MDN_OK ||
      (st = dalloc(&m->d_cols, m->h_cols.size())) != MDN_OK ||
      (st = dalloc(&m->d_slot, m->h_slot.size())) != MDN_OK ||
      (st = dalloc(&m->d_sub_e, (size_t)C)) != MDN_OK ||
      (!h_pqcent.empty() && (st = dalloc(&m->d_pqcent, h_pqcent.size())) != MDN_OK)) {
    mdn_model_free(m.release());
    return st;
  }
  cudaError_t e1 = cudaMemcpy(m->d_dims, m->h_dims.data(), m->h_dims.size() * 2, cudaMemcpyHostToDevice);
  cudaError_t e2 = cudaMemcpy(m->d_thr, m->h_thr.data(), m->h_thr.size() * 4, cudaMemcpyHostToDevice);
  cudaError_t e3 = cudaMemcpy(m->d_P, P, p_bytes, cudaMemcpyHostToDevice);
  cudaError_t e4 = cudaMemcpy(m->d_sub, m->h_sub.data(), C * 2, cudaMemcpyHostToDevice);
  cudaError_t e5 = cudaMemcpy(m->d_q, m->h_q.data(), m->h_q.size() * 2, cudaMemcpyHostToDevice);
  cudaError_t e6 = cudaMemcpy(m->d_cols, m->h_cols.data(), m->h_cols.size() * 2, cudaMemcpyHostToDevice);
  cudaError_t e7 = cudaMemcpy(m->d_slot, m->h_slot.data(), m->h_slot.size() * 2, cudaMemcpyHostToDevice);
  cudaError_t e8 = cudaMemcpy(m->d_sub_e, m->h_sub_e.data(), C * 2, cudaMemcpyHostToDevice);
  cudaError_t e9 = h_pqcent.empty() ? cudaSuccess
                                    : cudaMemcpy(m->d_pqcent, h_pqcent.data(), h_pqcent.size() * 4,
                                                 cudaMemcpyHostToDevice);
  if (e1 != cudaSuccess || e2 != cudaSuccess || e3 != cudaSuccess || e4 != cudaSuccess ||
      e5 != cudaSuccess || e6 != cudaSuccess || e7 != cudaSuccess || e8 != cudaSuccess ||
      e9 != cudaSuccess) {
    mdn_model_free(m.release());
    return MDN_ECUDA;
  }
  *out = m.release();
  return MDN_OK;
}

int mdn_train(const float* A, int64_t N, int64_t lda, int D, int C, double lambda, int device,
              void* buf, size_t* len) {
  if (!len || C < 1 || D < 1 || C > D || C > MAX_C || D > 65535 || !(lambda >= 0)) return MDN_EINVAL;
  const size_t need = train_blob_size(C, D);
  if (!buf) {
    *len = need;
    return MDN_OK;
  }
  if (*len < need || !A || N < 1 || N > MDN_TRAIN_MAX_N || lda < D) return MDN_EINVAL;
  DeviceGuard g(device);
  if (!g.ok) return MDN_ECUDA;
  std::vector<uint8_t> blob;
  int err = MDN_OK;
  cudaError_t e = train_model(A, N, lda, D, C, lambda, blob, &err);
  if (e != cudaSuccess) return cuda_status(e);
  if (err != MDN_OK) return err;
  if (blob.size() != need) return MDN_ECUDA;
  memcpy(buf, blob.data(), need);
  *len = need;
  return MDN_OK;
}

int mdn_model_info(const mdn_model* m, int* C, int* D, uint64_t* fp) {
  if (!m) return MDN_EINVAL;
  if (C) *C = m->C;
  if (D) *D = m->D;
  if (fp) *fp = m->fingerprint;
  return MDN_OK;
}

// ------------------------------------------------------------------ luts --

void mdn_luts_free(mdn_luts* l) {
  if (!l) return;
  {
    DeviceGuard g(l->device);
    cudaFree(l->d_tq);
    cudaFree(l->d_words);
    cudaFree(l->d_words16);
  }
  delete l;
}

static int alloc_luts(int device, int C, int M, mdn_luts** out) {
  std::unique_ptr<mdn_luts> l(new (std::nothrow) mdn_luts());
  if (!l) return MDN_ENOMEM;
  l->device = device;
  l->C = C;
  l->M = M;
  l->W = (M + 3) / 4;
  int st;
  if ((st = dalloc(&l->d_tq, (size_t)C * K * M)) != MDN_OK) return st;
  if ((st = dalloc(&l->d_words, (size_t)C * l->W * K)) != MDN_OK) {
    cudaFree(l->d_tq);
    return st;
  }
  if (M <= 2 * MAX_W2 && (st = dalloc(&l->d_words16, (size_t)C * K * ((M + 1) / 2))) != MDN_OK) {
    cudaFree(l->d_tq);
    cudaFree(l->d_words);
    return st;
  }
  *out = l.release();
  return MDN_OK;
}

int mdn_build_luts(const mdn_model* m, const float* B, int64_t M, int64_t ldb, int mode, int U,
                   mdn_luts** out) {
  if (!m || !B || !out || M < 1 || M > 4096 || ldb < M) return MDN_EINVAL;
  if (mode != MDN_SUM_EXACT && mode != MDN_SUM_AVG) return MDN_EINVAL;
  if (mode == MDN_SUM_AVG && (!is_pow2(U) || m->C % U != 0 || U > MAX_U)) return MDN_EINVAL;
  if (mode == MDN_SUM_EXACT) U = 1;
  *out = nullptr;
  DeviceGuard g(m->device);
  if (!g.ok) return MDN_ECUDA;
  const int C = m->C, D = m->D;
  mdn_luts* l = nullptr;
  int st = alloc_luts(m->device, C, (int)M, &l);
  if (st != MDN_OK) return st;
  l->mode = mode;
  l->U = U;
  l->model_fp = m->fingerprint;
  // Host B (D x M, ldb) -> dense device copy.
  std::vector<float> hb((size_t)D * M);
  for (int64_t j = 0; j < D; ++j) memcpy(&hb[j * M], B + j * ldb, M * sizeof(float));
  float* dB = nullptr;
  double *dT = nullptr, *dDelta = nullptr, *dRange = nullptr;
  LutScalars* dScal = nullptr;
  LutScalars hs{};
  cudaError_t e = cudaSuccess;
  if ((st = dalloc(&dB, hb.size())) || (st = dalloc(&dT, (size_t)K * C * M)) ||
      (st = dalloc(&dDelta, C)) || (st = dalloc(&dRange, C)) || (st = dalloc(&dScal, 1))) {
    goto fail;
  }
  e = cudaMemcpy(dB, hb.data(), hb.size() * 4, cudaMemcpyHostToDevice);
  if (e == cudaSuccess)
    e = build_tables_dev(m->d_P, dB, C, D, (int)M, mode == MDN_SUM_AVG ? U : 0, dT, dDelta, dRange,
                         dScal, l->d_tq, l->d_words, l->d_words16, 0);
  if (e == cudaSuccess) e = cudaMemcpy(&hs, dScal, sizeof(hs), cudaMemcpyDeviceToHost);
  if (e == cudaSuccess) {
    l->delta.resize(C);
    e = cudaMemcpy(l->delta.data(), dDelta, C * sizeof(double), cudaMemcpyDeviceToHost);
  }
  if (e != cudaSuccess) {
    st = cuda_status(e);
    goto fail;
  }
  if (hs.err) {
    st = MDN_ERANGE;
    goto fail;
  }
  l->l = hs.l;
  l->alpha = hs.alpha;
  l->beta32 = hs.beta32;
  cudaFree(dB);
  cudaFree(dT);
  cudaFree(dDelta);
  cudaFree(dRange);
  cudaFree(dScal);
  *out = l;
  return MDN_OK;
fail:
  cudaFree(dB);
  cudaFree(dT);
  cudaFree(dDelta);
  cudaFree(dRange);
  cudaFree(dScal);
  mdn_luts_free(l);
  return st;
}

int mdn_luts_serialize(const mdn_luts* l, void* buf, size_t* len) {
  if (!l || !len) return MDN_EINVAL;
  size_t tq = (size_t)l->C * K * l->M;
  size_t need = 4 + 6 * 4 + 4 + 4 + 4 + 8 + 8 * (size_t)l->C + tq + 8;
  if (!buf) {
    *len = need;
    return MDN_OK;
  }
  if (*len < need) return MDN_EINVAL;
  std::vector<uint8_t> o;
  o.reserve(need);
  o.insert(o.end(), {'M', 'D', 'N', 'L'});
  put<uint32_t>(o, 1);
  put<uint32_t>(o, l->C);
  put<uint32_t>(o, l->M);
  put<uint32_t>(o, K);
  put<uint32_t>(o, l->mode);
  put<uint32_t>(o, l->U);
  put<int32_t>(o, l->l);
  put<float>(o, l->alpha);
  put<float>(o, l->beta32);
  put<uint64_t>(o, l->model_fp);
  for (double d : l->delta) put<double>(o, d);
  size_t at = o.size();
  o.resize(at + tq);
  {
    DeviceGuard g(l->device);
    if (cudaMemcpy(o.data() + at, l->d_tq, tq, cudaMemcpyDeviceToHost) != cudaSuccess) return MDN_ECUDA;
  }
  put<uint64_t>(o, fnv1a64(o.data(), o.size()));
  memcpy(buf, o.data(), o.size());
  *len = o.size();
  return MDN_OK;
}

int mdn_luts_load(const void* buf, size_t len, int device, mdn_luts** out, size_t* err_off) {
  if (!buf || !out) return MDN_EINVAL;
  *out = nullptr;
  Reader r{static_cast<const uint8_t*>(buf), len};
  if (!r.need(52) || memcmp(r.p, "MDNL", 4) != 0) return set_err(err_off, 0, MDN_EFORMAT);
  r.off = 4;
  uint32_t ver = r.get<uint32_t>(), C = r.get<uint32_t>(), M = r.get<uint32_t>();
  uint32_t k = r.get<uint32_t>(), mode = r.get<uint32_t>(), U = r.get<uint32_t>();
  if (ver != 1) return set_err(err_off, 4, MDN_EVERSION);
  if (k != (uint32_t)K || C < 1 || C > (uint32_t)MAX_C || M < 1 || M > 4096 || mode > 1 ||
      !is_pow2((int)U) || C % U != 0 || U > (uint32_t)MAX_U ||
      (mode == MDN_SUM_EXACT && U != 1))
    return set_err(err_off, 8, MDN_EINVAL);   // same U rule as mdn_build_luts
  int32_t lexp = r.get<int32_t>();
  float alpha = r.get<float>(), beta = r.get<float>();
  uint64_t mfp = r.get<uint64_t>();
  std::vector<double> delta(C);
  for (uint32_t c = 0; c < C; ++c) delta[c] = r.get<double>();
  size_t tq = (size_t)C * K * M;
  if (r.fail || !r.need(tq + 8)) return set_err(err_off, r.fail_off, MDN_EFORMAT);
  const uint8_t* tqp = r.p + r.off;
  r.off += tq;
  uint64_t fp_stored = r.get<uint64_t>();
  if (fnv1a64(r.p, r.off - 8) != fp_stored) return set_err(err_off, r.off - 8, MDN_EFORMAT);
  DeviceGuard g(device);
  if (!g.ok) return MDN_ECUDA;
  mdn_luts* l = nullptr;
  int st = alloc_luts(device, (int)C, (int)M, &l);
  if (st != MDN_OK) return st;
  l->mode = (int)mode;
  l->U = (int)U;
  l->l = lexp;
  l->alpha = alpha;
  l->beta32 = beta;
  l->model_fp = mfp;
  l->delta = delta;
  cudaError_t e = cudaMemcpy(l->d_tq, tqp, tq, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = pack_words_dev(l->d_tq, l->C, l->M, l->d_words, l->d_words16, 0);
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    mdn_luts_free(l);
    return cuda_status(e);
  }
  *out = l;
  return MDN_OK;
}

int mdn_luts_info(const mdn_luts* l, int* C, int* M, int* mode, int* U, int* lexp, float* alpha,
                  float* beta32, uint64_t* mfp) {
  if (!l) return MDN_EINVAL;
  if (C) *C = l->C;
  if (M) *M = l->M;
  if (mode) *mode = l->mode;
  if (U) *U = l->U;
  if (lexp) *lexp = l->l;
  if (alpha) *alpha = l->alpha;
  if (beta32) *beta32 = l->beta32;
  if (mfp) *mfp = l->model_fp;
  return MDN_OK;
}

// -------------------------------------------------------------- hot path --

int mdn_encode(const mdn_model* m, const float* A, int64_t N, int64_t lda, uint8_t* codes,
               void* stream) {
  if (!m || N < 0) return MDN_EINVAL;
  if (m->pq) return MDN_ESTATE;              // PQ model: no hash trees (mdn_encode_pq)
  if (N == 0) return MDN_OK;
  if (!A || !codes || lda < m->D) return MDN_EINVAL;
  DeviceGuard g(m->device);
  if (!g.ok) return MDN_ECUDA;
  const int64_t nb = (m->C + 1) / 2;
  return cuda_status(for_row_chunks(N, [&](int64_t r0, int64_t n) {
    return launch_encode(m->trees(), A + r0 * lda, n, lda, codes + r0 * nb, (cudaStream_t)stream);
  }));
}

int mdn_scan(const mdn_luts* l, const uint8_t* codes, int64_t N, int32_t* sums, float* out,
             int64_t ldo, void* stream) {
  if (!l || N < 0) return MDN_EINVAL;
  if (N == 0) return MDN_OK;
  if (!codes || (!sums && !out) || (out && ldo < l->M)) return MDN_EINVAL;
  DeviceGuard g(l->device);
  if (!g.ok) return MDN_ECUDA;
  const int64_t nb = (l->C + 1) / 2;
  return cuda_status(for_row_chunks(N, [&](int64_t r0, int64_t n) {
    return launch_scan(l->dev(), codes + r0 * nb, n, sums ? sums + r0 * l->M : nullptr,
                       out ? out + r0 * ldo : nullptr, ldo, (cudaStream_t)stream);
  }));
}

int mdn_amm(const mdn_model* m, const mdn_luts* l, const float* A, int64_t N, int64_t lda,
            float* out, int64_t ldo, void* stream) {
  if (!m || !l || N < 0) return MDN_EINVAL;
  if (l->C != m->C) return MDN_ESHAPE;
  if (l->model_fp != m->fingerprint || m->pq) return MDN_ESTATE;
  if (l->device != m->device) return MDN_EINVAL;
  if (N == 0) return MDN_OK;
  if (!A || !out || lda < m->D || ldo < l->M) return MDN_EINVAL;
  DeviceGuard g(m->device);
  if (!g.ok) return MDN_ECUDA;
  return cuda_status(for_row_chunks(N, [&](int64_t r0, int64_t n) {
    return launch_amm(m->trees(), l->dev(), A + r0 * lda, n, lda, out + r0 * ldo, ldo,
                      (cudaStream_t)stream);
  }));
}

int mdn_amm_probe(const mdn_model* m, const mdn_luts* l, const float* A, int64_t N, int64_t lda,
                  float* out, int64_t ldo, void* stream) {
  if (!m || !l || N < 0) return MDN_EINVAL;
  if (l->C != m->C) return MDN_ESHAPE;
  if (l->model_fp != m->fingerprint || m->pq) return MDN_ESTATE;
  if (l->device != m->device) return MDN_EINVAL;
  if (N == 0) return MDN_OK;
  if (!A || !out || lda < m->D || ldo < l->M) return MDN_EINVAL;
  DeviceGuard g(m->device);
  if (!g.ok) return MDN_ECUDA;
  bool all_done = true;
  int st = cuda_status(for_row_chunks(N, [&](int64_t r0, int64_t n) {
    bool done = false;
    cudaError_t e = launch_amm_probe(m->trees(), l->dev(), A + r0 * lda, n, lda, out + r0 * ldo,
                                     ldo, (cudaStream_t)stream, &done);
    all_done = all_done && done;
    return e;
  }));
  if (st != MDN_OK) return st;
  return all_done ? MDN_OK : MDN_EINVAL;   // no general (k_amm_ws) pipeline for this shape
}

int mdn_encode_u8(const mdn_model* m, const uint8_t* A, int64_t N, int64_t lda, uint8_t* codes,
                  void* stream) {
  if (!m || N < 0) return MDN_EINVAL;
  if (m->pq) return MDN_ESTATE;              // PQ model: no hash trees (mdn_encode_pq)
  if (N == 0) return MDN_OK;
  if (!A || !codes || lda < m->D) return MDN_EINVAL;
  DeviceGuard g(m->device);
  if (!g.ok) return MDN_ECUDA;
  const int64_t nb = (m->C + 1) / 2;
  return cuda_status(for_row_chunks(N, [&](int64_t r0, int64_t n) {
    return launch_encode_u8(m->trees(), A + r0 * lda, n, lda, codes + r0 * nb, (cudaStream_t)stream);
  }));
}

int mdn_amm_u8(const mdn_model* m, const mdn_luts* l, const uint8_t* A, int64_t N, int64_t lda,
               float* out, int64_t ldo, void* stream) {
  if (!m || !l || N < 0) return MDN_EINVAL;
  if (l->C != m->C) return MDN_ESHAPE;
  if (l->model_fp != m->fingerprint || m->pq) return MDN_ESTATE;
  if (l->device != m->device) return MDN_EINVAL;
  if (N == 0) return MDN_OK;
  if (!A || !out || lda < m->D || ldo < l->M) return MDN_EINVAL;
  DeviceGuard g(m->device);
  if (!g.ok) return MDN_ECUDA;
  return cuda_status(for_row_chunks(N, [&](int64_t r0, int64_t n) {
    return launch_amm_u8(m->trees(), l->dev(), A + r0 * lda, n, lda, out + r0 * ldo, ldo,
                         (cudaStream_t)stream);
  }));
}

int mdn_encode_pq(const mdn_model* m, const float* A, int64_t N, int64_t lda, uint8_t* codes,
                  void* stream) {
  if (!m || N < 0) return MDN_EINVAL;
  if (!m->pq) return MDN_ESTATE;              // not a PQ model (flags bit1)
  if (N == 0) return MDN_OK;
  if (!A || !codes || lda < m->D) return MDN_EINVAL;
  DeviceGuard g(m->device);
  if (!g.ok) return MDN_ECUDA;
  const int64_t nb = (m->C + 1) / 2;
  return cuda_status(for_row_chunks(N, [&](int64_t r0, int64_t n) {
    return launch_encode_pq(m->trees(), m->d_P, m->d_sub, m->d_sub_e, A + r0 * lda, n, lda,
                            codes + r0 * nb, (cudaStream_t)stream);
  }));
}

int mdn_encode_cm(const mdn_model* m, const float* At, int64_t N, int64_t ldt, uint8_t* codes,
                  void* stream) {
  if (!m || N < 0) return MDN_EINVAL;
  if (m->pq) return MDN_ESTATE;              // PQ model: no hash trees (mdn_encode_pq)
  if (N == 0) return MDN_OK;
  if (!At || !codes || ldt < N) return MDN_EINVAL;
  DeviceGuard g(m->device);
  if (!g.ok) return MDN_ECUDA;
  const int64_t nb = (m->C + 1) / 2;
  return cuda_status(for_row_chunks(N, [&](int64_t r0, int64_t n) {
    return launch_encode_cm(m->trees(), At + r0, n, ldt, codes + r0 * nb, (cudaStream_t)stream);
  }));
}

int mdn_amm_cm(const mdn_model* m, const mdn_luts* l, const float* At, int64_t N, int64_t ldt,
               float* out, int64_t ldo, void* stream) {
  if (!m || !l || N < 0) return MDN_EINVAL;
  if (l->C != m->C) return MDN_ESHAPE;
  if (l->model_fp != m->fingerprint || m->pq) return MDN_ESTATE;
  if (l->device != m->device) return MDN_EINVAL;
  if (N == 0) return MDN_OK;
  if (!At || !out || ldt < N || ldo < l->M) return MDN_EINVAL;
  DeviceGuard g(m->device);
  if (!g.ok) return MDN_ECUDA;
  return cuda_status(for_row_chunks(N, [&](int64_t r0, int64_t n) {
    return launch_amm_cm(m->trees(), l->dev(), At + r0, n, ldt, out + r0 * ldo, ldo,
                         (cudaStream_t)stream);
  }));
}

int mdn_amm_variant(const mdn_model* m, const mdn_luts* l, int64_t lda, char* buf, size_t len) {
  if (!m || !l || !buf || len == 0) return MDN_EINVAL;
  // Report for a 16-B aligned A / out with ldo == M.
  const char* name = amm_variant_name(m->trees(), l->dev(), reinterpret_cast<const float*>(256),
                                      lda, reinterpret_cast<const float*>(256), l->M);
  snprintf(buf, len, "%s", name);
  return MDN_OK;
}

int mdn_stream_probe(const float* A, int64_t N, int64_t lda, int64_t D, float* out, int64_t ldo,
                     int64_t M, void* stream) {
  if (N < 0 || D < 4 || D % 4 || M < 1 || lda < D || ldo < M || lda % 4 || (N * ldo) % 4) return MDN_EINVAL;
  if (N == 0) return MDN_OK;
  if (!A || !out || (reinterpret_cast<uintptr_t>(A) & 15u) || (reinterpret_cast<uintptr_t>(out) & 15u))
    return MDN_EINVAL;
  return cuda_status(mdn::launch_stream_probe(A, N, lda, (int)D, out, ldo, (int)M,
                                              (cudaStream_t)stream));
}

// ------------------------------------------------------ host executor (e2e) --

struct mdn_exec {
  const mdn_model* model;
  const mdn_luts* luts;
  int device;
  int64_t chunk;
  int n_slots;
  std::vector<cudaStream_t> streams;
  std::vector<float*> dA, dOut;
  std::vector<uint8_t*> dC;       // packed codes of a chunk (mdn_encode_host / mdn_scan_host)
  std::mutex mu;                  // held for a whole host call: the slots are per handle
};

void mdn_exec_free(mdn_exec* x) {
  if (!x) return;
  {
    DeviceGuard g(x->device);
    for (auto s : x->streams) cudaStreamDestroy(s);
    for (auto p : x->dA) cudaFree(p);
    for (auto p : x->dOut) cudaFree(p);
    for (auto p : x->dC) cudaFree(p);
  }
  delete x;
}

int mdn_exec_create(const mdn_model* m, const mdn_luts* l, int64_t chunk_rows, int n_slots,
                    mdn_exec** out) {
  if (!m || !l || !out || chunk_rows < 1 || n_slots < 1 || n_slots > 8) return MDN_EINVAL;
  if (l->C != m->C) return MDN_ESHAPE;
  if (l->model_fp != m->fingerprint) return MDN_ESTATE;
  if (l->device != m->device) return MDN_EINVAL;   // as mdn_amm: tables on the model's device
  *out = nullptr;
  DeviceGuard g(m->device);
  if (!g.ok) return MDN_ECUDA;
  std::unique_ptr<mdn_exec> x(new (std::nothrow) mdn_exec());
  if (!x) return MDN_ENOMEM;
  x->model = m;
  x->luts = l;
  x->device = m->device;
  x->chunk = chunk_rows;
  x->n_slots = n_slots;
  for (int i = 0; i < n_slots; ++i) {
    cudaStream_t s;
    float *a = nullptr, *o = nullptr;
    if (cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking) != cudaSuccess) {
      mdn_exec_free(x.release());
      return MDN_ECUDA;
    }
    x->streams.push_back(s);
    uint8_t* c = nullptr;
    int st = dalloc(&a, (size_t)chunk_rows * m->D);
    if (st == MDN_OK) st = dalloc(&o, (size_t)chunk_rows * l->M);
    if (st == MDN_OK) st = dalloc(&c, (size_t)chunk_rows * ((m->C + 1) / 2));
    x->dA.push_back(a);
    x->dOut.push_back(o);
    x->dC.push_back(c);
    if (st != MDN_OK) {
      mdn_exec_free(x.release());
      return st;
    }
  }
  *out = x.release();
  return MDN_OK;
}

}  // extern "C"

// ------------------------------------------------ host-buffer pipelines --
//
// Every host call runs the same driver: chunk q of the rows goes through slot
// q % n_slots on the slot's stream -- host->device copy, the device op, the
// device->host copy -- so the copies of one chunk overlap the kernels of the
// others; stream order serialises the reuse of a slot (chunk q's upload waits
// for chunk q - n_slots' download). The per-op part is a chunk function.
namespace {

template <class ChunkFn>
int run_pipeline(mdn_exec* x, int64_t N, ChunkFn&& chunk) {
  // The staging slots are mutable state of the handle: one call at a time
  // (maddness.h: concurrent calls on one executor serialise here).
  std::lock_guard<std::mutex> lock(x->mu);
  nvtxRangePushA("mdn_host_pipeline");          // timeline: one range per host call
  struct PopRange {
    ~PopRange() { nvtxRangePop(); }
  } pop_range;
  DeviceGuard g(x->device);
  if (!g.ok) return MDN_ECUDA;
  cudaError_t e = cudaSuccess;
  const int64_t nchunks = (N + x->chunk - 1) / x->chunk;
  for (int64_t q = 0; q < nchunks && e == cudaSuccess; ++q) {
    const int s = (int)(q % x->n_slots);
    const int64_t r0 = q * x->chunk, n = N - r0 < x->chunk ? N - r0 : x->chunk;
    e = chunk(s, x->streams[s], r0, n);
  }
  for (auto st : x->streams) {
    cudaError_t e2 = cudaStreamSynchronize(st);
    if (e == cudaSuccess) e = e2;
  }
  return cuda_status(e);
}

// n rows of w elements (host row stride ld) into a packed device tile. A
// contiguous block goes as one linear copy: a 2-D copy of narrow rows (8-bit
// A, small M) runs row by row far below the PCIe rate.
template <class T>
cudaError_t upload_rows(T* dst, const T* src, int64_t ld, int64_t w, int64_t n, cudaStream_t st) {
  return ld == w ? cudaMemcpyAsync(dst, src, (size_t)n * w * sizeof(T), cudaMemcpyHostToDevice, st)
                 : cudaMemcpy2DAsync(dst, w * sizeof(T), src, ld * sizeof(T), w * sizeof(T), n,
                                     cudaMemcpyHostToDevice, st);
}

template <class T>
cudaError_t download_rows(T* dst, int64_t ld, const T* src, int64_t w, int64_t n, cudaStream_t st) {
  return ld == w ? cudaMemcpyAsync(dst, src, (size_t)n * w * sizeof(T), cudaMemcpyDeviceToHost, st)
                 : cudaMemcpy2DAsync(dst, ld * sizeof(T), src, w * sizeof(T), w * sizeof(T), n,
                                     cudaMemcpyDeviceToHost, st);
}

// Chunk [r0, r0 + n) of the split columns of host At (D x N, ldt) into the
// slot's D x chunk column-major tile (ldt = chunk); rows of At that are not
// split columns are never copied and never read. Adjacent columns as one 2-D
// copy of n-float rows.
cudaError_t upload_split_columns(const mdn_exec* x, float* dAt, const float* At, int64_t ldt,
                                 int64_t r0, int64_t n, cudaStream_t st) {
  const std::vector<uint16_t>& cols = x->model->h_cols;
  cudaError_t e = cudaSuccess;
  for (size_t i = 0; i < cols.size() && e == cudaSuccess;) {
    size_t j = i + 1;
    while (j < cols.size() && cols[j] == cols[j - 1] + 1) ++j;
    const int64_t c0 = cols[i];
    e = cudaMemcpy2DAsync(dAt + c0 * x->chunk, (size_t)x->chunk * sizeof(float),
                          At + c0 * ldt + r0, (size_t)ldt * sizeof(float),
                          (size_t)n * sizeof(float), j - i, cudaMemcpyHostToDevice, st);
    i = j;
  }
  return e;
}

// Fused g + f on host rows (fp32 or natively 8-bit).
template <class TIn>
int amm_host(mdn_exec* x, const TIn* A, int64_t N, int64_t lda, float* out, int64_t ldo) {
  if (!x || N < 0) return MDN_EINVAL;
  if (x->model->pq) return MDN_ESTATE;                 // PQ model: mdn_amm_pq_host
  if (N == 0) return MDN_OK;
  const int D = x->model->D, M = x->luts->M;
  if (!A || !out || lda < D || ldo < M) return MDN_EINVAL;
  return run_pipeline(x, N, [&](int s, cudaStream_t st, int64_t r0, int64_t n) {
    TIn* dA = reinterpret_cast<TIn*>(x->dA[s]);        // sized for fp32 rows: 8-bit rows fit
    cudaError_t e = upload_rows(dA, A + r0 * lda, lda, D, n, st);
    if (e != cudaSuccess) return e;
    if constexpr (sizeof(TIn) == 1)
      e = launch_amm_u8(x->model->trees(), x->luts->dev(), dA, n, D, x->dOut[s], M, st);
    else
      e = launch_amm(x->model->trees(), x->luts->dev(), dA, n, D, x->dOut[s], M, st);
    if (e != cudaSuccess) return e;
    return download_rows(out + r0 * ldo, ldo, x->dOut[s], M, n, st);
  });
}

// g alone on host rows (fp32 or 8-bit): packed codes back.
template <class TIn>
int encode_host(mdn_exec* x, const TIn* A, int64_t N, int64_t lda, uint8_t* codes) {
  if (!x || N < 0) return MDN_EINVAL;
  if (x->model->pq) return MDN_ESTATE;                 // PQ model: mdn_encode_pq_host
  if (N == 0) return MDN_OK;
  const int D = x->model->D;
  const int64_t nb = (x->model->C + 1) / 2;
  if (!A || !codes || lda < D) return MDN_EINVAL;
  return run_pipeline(x, N, [&](int s, cudaStream_t st, int64_t r0, int64_t n) {
    TIn* dA = reinterpret_cast<TIn*>(x->dA[s]);
    cudaError_t e = upload_rows(dA, A + r0 * lda, lda, D, n, st);
    if (e != cudaSuccess) return e;
    if constexpr (sizeof(TIn) == 1)
      e = launch_encode_u8(x->model->trees(), dA, n, D, x->dC[s], st);
    else
      e = launch_encode(x->model->trees(), dA, n, D, x->dC[s], st);
    if (e != cudaSuccess) return e;
    return download_rows(codes + r0 * nb, nb, x->dC[s], nb, n, st);
  });
}

// The PQ comparator: codes only (out == null) or codes + scan +
// dequant per chunk on the device (the two-launch PQ amm).
int pq_host(mdn_exec* x, const float* A, int64_t N, int64_t lda, uint8_t* codes, float* out,
            int64_t ldo) {
  if (!x || N < 0) return MDN_EINVAL;
  const mdn_model* m = x->model;
  if (!m->pq) return MDN_ESTATE;
  if (N == 0) return MDN_OK;
  const int D = m->D, M = x->luts->M;
  const int64_t nb = (m->C + 1) / 2;
  if (!A || lda < D || (!codes && !out) || (out && ldo < M)) return MDN_EINVAL;
  return run_pipeline(x, N, [&](int s, cudaStream_t st, int64_t r0, int64_t n) {
    cudaError_t e = upload_rows(x->dA[s], A + r0 * lda, lda, D, n, st);
    if (e != cudaSuccess) return e;
    e = launch_encode_pq(m->trees(), m->d_P, m->d_sub, m->d_sub_e, x->dA[s], n, D, x->dC[s], st);
    if (e != cudaSuccess) return e;
    if (!out) return download_rows(codes + r0 * nb, nb, x->dC[s], nb, n, st);
    e = launch_scan(x->luts->dev(), x->dC[s], n, nullptr, x->dOut[s], M, st);
    if (e != cudaSuccess) return e;
    return download_rows(out + r0 * ldo, ldo, x->dOut[s], M, n, st);
  });
}

}  // namespace

extern "C" {

int mdn_amm_host(mdn_exec* x, const float* A, int64_t N, int64_t lda, float* out, int64_t ldo) {
  return amm_host<float>(x, A, N, lda, out, ldo);
}

int mdn_amm_host_u8(mdn_exec* x, const uint8_t* A, int64_t N, int64_t lda, float* out,
                    int64_t ldo) {
  return amm_host<uint8_t>(x, A, N, lda, out, ldo);
}

int mdn_encode_host(mdn_exec* x, const float* A, int64_t N, int64_t lda, uint8_t* codes) {
  return encode_host<float>(x, A, N, lda, codes);
}

int mdn_encode_host_u8(mdn_exec* x, const uint8_t* A, int64_t N, int64_t lda, uint8_t* codes) {
  return encode_host<uint8_t>(x, A, N, lda, codes);
}

// f alone: host codes in, dequantised host rows out, with the executor's tables.
int mdn_scan_host(mdn_exec* x, const uint8_t* codes, int64_t N, float* out, int64_t ldo) {
  if (!x || N < 0) return MDN_EINVAL;
  if (N == 0) return MDN_OK;
  const int M = x->luts->M;
  const int64_t nb = (x->model->C + 1) / 2;
  if (!codes || !out || ldo < M) return MDN_EINVAL;
  return run_pipeline(x, N, [&](int s, cudaStream_t st, int64_t r0, int64_t n) {
    cudaError_t e = upload_rows(x->dC[s], codes + r0 * nb, nb, nb, n, st);
    if (e != cudaSuccess) return e;
    e = launch_scan(x->luts->dev(), x->dC[s], n, nullptr, x->dOut[s], M, st);
    if (e != cudaSuccess) return e;
    return download_rows(out + r0 * ldo, ldo, x->dOut[s], M, n, st);
  });
}

int mdn_encode_pq_host(mdn_exec* x, const float* A, int64_t N, int64_t lda, uint8_t* codes) {
  if (!codes) return MDN_EINVAL;
  return pq_host(x, A, N, lda, codes, nullptr, 0);
}

int mdn_amm_pq_host(mdn_exec* x, const float* A, int64_t N, int64_t lda, float* out, int64_t ldo) {
  if (!out) return MDN_EINVAL;
  return pq_host(x, A, N, lda, nullptr, out, ldo);
}

// Column-major host A: only the split columns cross PCIe
// (4 |S| instead of 4 D bytes per row).
int mdn_amm_cm_host(mdn_exec* x, const float* At, int64_t N, int64_t ldt, float* out,
                    int64_t ldo) {
  if (!x || N < 0) return MDN_EINVAL;
  if (x->model->pq) return MDN_ESTATE;
  if (N == 0) return MDN_OK;
  const int M = x->luts->M;
  if (!At || !out || ldt < N || ldo < M) return MDN_EINVAL;
  return run_pipeline(x, N, [&](int s, cudaStream_t st, int64_t r0, int64_t n) {
    cudaError_t e = upload_split_columns(x, x->dA[s], At, ldt, r0, n, st);
    if (e != cudaSuccess) return e;
    e = launch_amm_cm(x->model->trees(), x->luts->dev(), x->dA[s], n, x->chunk, x->dOut[s], M, st);
    if (e != cudaSuccess) return e;
    return download_rows(out + r0 * ldo, ldo, x->dOut[s], M, n, st);
  });
}

int mdn_encode_cm_host(mdn_exec* x, const float* At, int64_t N, int64_t ldt, uint8_t* codes) {
  if (!x || N < 0) return MDN_EINVAL;
  if (x->model->pq) return MDN_ESTATE;
  if (N == 0) return MDN_OK;
  if (!At || !codes || ldt < N) return MDN_EINVAL;
  const int64_t nb = (x->model->C + 1) / 2;
  return run_pipeline(x, N, [&](int s, cudaStream_t st, int64_t r0, int64_t n) {
    cudaError_t e = upload_split_columns(x, x->dA[s], At, ldt, r0, n, st);
    if (e != cudaSuccess) return e;
    e = launch_encode_cm(x->model->trees(), x->dA[s], n, x->chunk, x->dC[s], st);
    if (e != cudaSuccess) return e;
    return download_rows(codes + r0 * nb, nb, x->dC[s], nb, n, st);
  });
}

}  // extern "C"
