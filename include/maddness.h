/*
 * libmaddness -- B200 (sm_100a) hot path of MADDNESS (Blalock & Guttag,
 * "Multiplying Matrices Without Multiplying", ICML 2021, arXiv 2106.10860).
 *
 * The paper's problem statement (Sec. 1.1, Eq. 1): construct
 * g(.) (encoding of A), h(.) (tables from B), f(.,.) (aggregation) and
 * constants alpha, beta with  alpha f(g(A), h(B)) + beta  ~  A B.
 * This library implements the inference side on the GPU:
 *
 *   mdn_encode      g(A)          Algorithm 1 (L228-248): 4-level hash trees,
 *                                 4-bit code per codebook
 *   mdn_build_luts  h(B)          T = P B (L190-192, dense P per L896) and the
 *                                 8-bit quantisation of App. A (L593-604)
 *   mdn_scan        f + dequant   out[n,m] = alpha * sum_c Tq[c][code][m] + beta
 *                                 (L331), exact or averaging (App. D)
 *   mdn_amm         all three fused; codes never touch HBM
 *
 * Training (Alg. 2-4, ridge prototypes, L252-323) is offline and lives in the
 * oracle; the library consumes the serialized model ("model.mdnm v1" below).
 *
 * Conventions for every entry point
 *  - Return value: MDN_OK (0) or a negative mdn_status. Argument and shape
 *    validation is synchronous; kernel launch errors return MDN_ECUDA;
 *    asynchronous device faults surface at the caller's next stream sync.
 *  - Ownership: the caller allocates and owns every data buffer (A, B, codes,
 *    sums, out); the library owns only its opaque handles, created by
 *    *_load / *_build / *_create and released by the matching *_free.
 *    No allocation happens on the hot path (encode / scan / amm).
 *  - Device pointers ("device" below) must be on the handle's device; the
 *    library makes that device current for the call and restores the caller's
 *    current device before returning. `stream` is a cudaStream_t (NULL = the
 *    legacy default stream); all work of a call is enqueued on it.
 *  - Layouts are row-major with explicit leading dimensions in elements.
 *  - Model and LUT handles are immutable after creation and may be used
 *    concurrently from several host threads / streams. An executor
 *    (mdn_exec) owns mutable staging slots: concurrent host calls on ONE
 *    executor are serialised by its internal lock (safe, not parallel); use
 *    one executor per thread for parallel host pipelines.
 *  - N = 0 is a no-op returning MDN_OK.
 */
#ifndef MADDNESS_H_
#define MADDNESS_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MDN_ABI_VERSION 1
#define MDN_K 16 /* prototypes per codebook: 16 leaves of a 4-level tree (L224, L608) */

typedef enum {
  MDN_OK = 0,
  MDN_EINVAL = -1,   /* null pointer, bad enum, U not a power of two dividing C,
                        lda < D, ldo < M, N < 0 */
  MDN_ESHAPE = -2,   /* luts.C != model.C, D mismatch */
  MDN_EFORMAT = -3,  /* bad magic / truncated / corrupt stream; *err_off = byte offset */
  MDN_EVERSION = -4, /* unsupported format version */
  MDN_ESTATE = -5,   /* luts were built from a different model (fingerprint) --
                        "apply before set_operator" */
  MDN_ECUDA = -6,    /* CUDA runtime / launch error */
  MDN_ENOMEM = -7,   /* device or host allocation failed */
  MDN_ERANGE = -8    /* table scale exponent |l| > 100 (tables not representable) */
} mdn_status;

typedef enum {
  MDN_SUM_EXACT = 0, /* exact integer sum of the C looked-up bytes (L331-333) */
  MDN_SUM_AVG = 1    /* averaging integer sum estimator, blocks of U (App. D) */
} mdn_sum_mode;

typedef struct mdn_model mdn_model; /* trees + prototypes, resident on one device */
typedef struct mdn_luts mdn_luts;   /* quantised tables + alpha, beta, on one device */
typedef struct mdn_exec mdn_exec;   /* host-buffer pipelined executor (e2e path) */

/* ---------------------------------------------------------------- model -- */

/* Parse a "model.mdnm v1" byte stream (host memory, `len` bytes) and upload
 * the split dims, thresholds and prototypes to `device`.
 * Errors: MDN_EFORMAT (with *err_off = offending byte offset; err_off may be
 * NULL), MDN_EVERSION, MDN_EINVAL (split dim >= D, C < 1, K != 16, a NaN threshold),
 * MDN_ENOMEM, MDN_ECUDA. */
int mdn_model_load(const void* buf, size_t len, int device, mdn_model** out,
                   size_t* err_off);
void mdn_model_free(mdn_model* model);
/* C, D and the file's FNV-1a fingerprint; any output pointer may be NULL. */
int mdn_model_info(const mdn_model* model, int* C, int* D, uint64_t* fingerprint);

/* GPU training: the offline step before the hot path (PAPER.md
 * L379), Sec. 4.2-4.3 and App. C -- per codebook 4 x Algorithm 2 with
 * Algorithms 3/4 (L252-305, L621-682), then ridge prototypes
 * P = (G^T G + lambda I)^-1 G^T A~ (L318-321), or bucket means for lambda = 0
 * (L218) -- with the readings R1-R12 of DESIGN.md.
 *   A       device fp32 training rows A~, N x D, row stride lda >= D;
 *           1 <= N <= 2^31 - 2^20 - 1 (int32 row indices with loop headroom).
 *   buf     host buffer receiving a "model.mdnm v1" stream (load it with
 *           mdn_model_load); buf == NULL: *len receives the size needed,
 *           48 + 76 C + 64 C D + 8 bytes. Otherwise *len is the capacity in,
 *           bytes written out.
 * Synchronous. Errors: MDN_EINVAL (bad sizes, a subspace wider than 64
 * columns, lambda < 0), MDN_ENOMEM, MDN_ECUDA (incl. a failed Cholesky). */
int mdn_train(const float* A, int64_t N, int64_t lda, int D, int C, double lambda, int device,
              void* buf, size_t* len);

/* ------------------------------------------------------------------ luts -- */

/* h(B) + App. A quantisation (the "set_operator" step), computed on the device.
 *   B     HOST fp32, D x M row-major, row stride ldb >= M (elements).
 *   mode  MDN_SUM_EXACT or MDN_SUM_AVG.
 *   U     averaging block (power of two dividing C, U <= 64); ignored in
 *         exact mode (stored as 1).
 * Arithmetic (reading R13-R15, R18 of DESIGN.md):
 *   T[c][k][m] = sum_{j ascending} (double)P[16c+k][j] * (double)B[j][m]
 *   delta_c = min_{k,m} T[c];  R = max_c max_{k,m}(T[c] - delta_c)
 *   l = max{ l : 2^l R <= 255 } (0 if R == 0);  alpha = 2^-l
 *   Tq = rint(2^l (T - delta_c))  (ties to even)
 *   beta32 = (float)(sum_{c ascending} delta_c + alpha * debias),
 *   debias = 0 (exact) or -C log2(U) / 4 (avg, App. D Theorem, L766-771)
 * Synchronous: returns when the tables are resident. MDN_ERANGE if |l| > 100. */
int mdn_build_luts(const mdn_model* model, const float* B, int64_t M, int64_t ldb,
                   int mode, int U, mdn_luts** out);
/* Serialize to "luts.mdnl v1". buf == NULL: *len receives the size needed.
 * Otherwise *len is the capacity in, bytes written out (MDN_EINVAL if small). */
int mdn_luts_serialize(const mdn_luts* luts, void* buf, size_t* len);
/* Load a "luts.mdnl v1" stream (e.g. after an NCCL broadcast) onto `device`.
 * Validates what mdn_build_luts enforces: bad magic / truncation / checksum
 * -> MDN_EFORMAT (*err_off = offending byte), version != 1 -> MDN_EVERSION,
 * C outside [1, 256], M outside [1, 4096], unknown mode, U not a power of
 * two dividing C, U > 64, or U != 1 in exact mode -> MDN_EINVAL. */
int mdn_luts_load(const void* buf, size_t len, int device, mdn_luts** out,
                  size_t* err_off);
void mdn_luts_free(mdn_luts* luts);
/* Any output pointer may be NULL. */
int mdn_luts_info(const mdn_luts* luts, int* C, int* M, int* mode, int* U, int* l,
                  float* alpha, float* beta32, uint64_t* model_fingerprint);

/* ------------------------------------------------------------- hot path -- */

/* g(A): Algorithm 1 on every row (fp32 compares, x >= v goes right, L240).
 *   A      device fp32, N x D, row stride lda >= D (elements).
 *   codes  device u8, N x ceil(C/2), row stride ceil(C/2): two 4-bit codes per
 *          byte, low nibble = codebook 2i, high nibble = codebook 2i+1 (L147,
 *          L608); an odd last codebook leaves the high nibble 0. */
int mdn_encode(const mdn_model* model, const float* A, int64_t N, int64_t lda,
               uint8_t* codes, void* stream);

/* f and dequantisation from packed codes.
 *   codes  device u8, N x ceil(C/2) as produced by mdn_encode.
 *   sums   device int32 N x M (row stride M), or NULL: the integer estimate
 *          S (exact: sum_c Tq; avg: U * sum_blocks s^_U, App. D L697 + L687).
 *   out    device fp32 N x M (row stride ldo >= M), or NULL:
 *          out = fl32(alpha * S + beta32)  (Eq. 1; one rounding).
 * At least one of sums / out must be non-NULL. */
int mdn_scan(const mdn_luts* luts, const uint8_t* codes, int64_t N, int32_t* sums,
             float* out, int64_t ldo, void* stream);

/* Fused g + f + dequant: out = alpha f(g(A), h(B)) + beta.
 *   A device fp32 N x D (lda), out device fp32 N x M (ldo). The luts must have
 *   been built from `model` (else MDN_ESTATE). */
int mdn_amm(const mdn_model* model, const mdn_luts* luts, const float* A, int64_t N,
            int64_t lda, float* out, int64_t ldo, void* stream);

/* ------------------------------------------------ 8-bit input -- */

/* g and the fused path for natively 8-bit A ("MADDNESS can operate on 8-bit
 * data directly"), with App. B's 8-bit split values (L606-616):
 * for byte inputs the x-quantiser is the identity and each threshold v becomes
 * q = ceil(v) clamped to [0, 256], so x >= q <=> x >= v and the codes equal
 * mdn_encode's on the same values as fp32 (reading R11).
 *   A  device u8, N x D, row stride lda >= D (bytes). Other arguments, layouts
 *   and errors as mdn_encode / mdn_amm. A quarter of the fp32 path's A bytes. */
int mdn_encode_u8(const mdn_model* model, const uint8_t* A, int64_t N, int64_t lda,
                  uint8_t* codes, void* stream);
int mdn_amm_u8(const mdn_model* model, const mdn_luts* luts, const uint8_t* A, int64_t N,
               int64_t lda, float* out, int64_t ldo, void* stream);

/* ------------------------------------------- column-major A -- */

/* g and the fused path for COLUMN-MAJOR A: "[Algorithm 1] only depends on a
 * constant number of indices in the input vector, and can easily be
 * vectorized provided that the matrix whose rows are being encoded is stored
 * in column-major order"; its cost per row is O(C), not O(D)
 * (L431). Only the <= 4C split columns of A are read.
 *   At     device fp32, D x N row-major (= A column-major): element (n, j) of
 *          A is At[j * ldt + n]; ldt >= N (elements).
 *   codes  as mdn_encode (row-major N x ceil(C/2)); out as mdn_amm (row-major
 *          N x M, ldo >= M). Results are bit-identical to mdn_encode /
 *          mdn_amm on the same A stored row-major.
 * Errors as mdn_encode / mdn_amm (ldt < N: MDN_EINVAL). */
int mdn_encode_cm(const mdn_model* model, const float* At, int64_t N, int64_t ldt,
                  uint8_t* codes, void* stream);
int mdn_amm_cm(const mdn_model* model, const mdn_luts* luts, const float* At, int64_t N,
               int64_t ldt, float* out, int64_t ldo, void* stream);

/* --------------------------------------------- PQ comparator -- */

/* g(A) of Product Quantization, the encoder MADDNESS replaces (PAPER.md Sec.
 * 3, Eq. pqLoss): per codebook the index of the nearest of the 16
 * K-means prototypes (L155-163) in squared Euclidean distance over the
 * codebook's subspace, evaluated in fp32 with every subtract / multiply / add
 * rounded separately, dims ascending; ties go to the lowest index.
 *   model  a PQ model: "model.mdnm" with flags bit1 set; its P holds the
 *          prototypes (row 16c + k, zero outside subspace c). MDN_ESTATE for
 *          a MADDNESS model (and the tree-based calls refuse PQ models).
 *   A, codes as mdn_encode. The codes feed mdn_scan with tables from
 *   mdn_build_luts(model, B, ...) exactly like MADDNESS codes. */
int mdn_encode_pq(const mdn_model* model, const float* A, int64_t N, int64_t lda,
                  uint8_t* codes, void* stream);

/* ----------------------------------------------------- end-to-end (host) -- */

/* A pipelined executor for HOST buffers: row chunks are copied host->device,
 * run through the device op and copied back, with the copies of one chunk
 * overlapping the kernel of another (`n_slots` device staging slots of
 * `chunk_rows` rows, one stream each; chunk q uses slot q % n_slots and stream
 * order serialises a slot's reuse). Owns its device staging buffers and
 * streams; `model` and `luts` are borrowed and must outlive the executor.
 * For overlap the host buffers should be page-locked. Every host call below
 * is synchronous (returns when the host outputs hold every row); N = 0 is a
 * no-op; null buffers or short strides -> MDN_EINVAL; a call for the other
 * model kind (tree calls on a PQ executor, PQ calls on a MADDNESS one) ->
 * MDN_ESTATE; CUDA failures -> MDN_ECUDA.
 * Errors: luts from another model -> MDN_ESTATE, C mismatch -> MDN_ESHAPE,
 * chunk_rows < 1 or n_slots outside [1, 8], or luts on another device than
 * the model -> MDN_EINVAL, allocation -> MDN_ENOMEM. Host calls on one
 * executor from several threads run one after another (internal lock). */
int mdn_exec_create(const mdn_model* model, const mdn_luts* luts, int64_t chunk_rows,
                    int n_slots, mdn_exec** out);
void mdn_exec_free(mdn_exec* exec);
/* A_host fp32 N x D (lda), out_host fp32 N x M (ldo). Synchronous: returns
 * when out_host holds every row. */
int mdn_amm_host(mdn_exec* exec, const float* A_host, int64_t N, int64_t lda,
                 float* out_host, int64_t ldo);
/* The same pipeline for natively 8-bit rows (mdn_amm_u8): A_host
 * u8 N x D (lda bytes) -- a quarter of the host->device bytes per row. */
int mdn_amm_host_u8(mdn_exec* exec, const uint8_t* A_host, int64_t N, int64_t lda,
                    float* out_host, int64_t ldo);
/* The unfused halves through the same executor (slots, streams): g on host
 * rows -> host codes (codes_host u8 N x ceil(C/2), contiguous), and f on host
 * codes -> host out (fp32 N x M, ldo >= M) with the executor's tables. Same
 * errors as mdn_amm_host. */
int mdn_encode_host(mdn_exec* exec, const float* A_host, int64_t N, int64_t lda,
                    uint8_t* codes_host);
int mdn_scan_host(mdn_exec* exec, const uint8_t* codes_host, int64_t N, float* out_host,
                  int64_t ldo);
/* g on natively 8-bit host rows (mdn_encode_u8), lda in bytes. */
int mdn_encode_host_u8(mdn_exec* exec, const uint8_t* A_host, int64_t N, int64_t lda,
                       uint8_t* codes_host);
/* The same pipeline for column-major host A (mdn_amm_cm; SURVEY N2, P:L246,
 * P:L431): At_host fp32 D x N, row stride ldt >= N (column n of A = row n of
 * the result). Per chunk only the model's distinct split columns of At are
 * copied host->device (4 |S| bytes per row instead of 4 D), into the slot
 * buffer used as a D x chunk_rows column-major tile. Same errors as
 * mdn_amm_host; ldt < N -> MDN_EINVAL. */
int mdn_amm_cm_host(mdn_exec* exec, const float* At_host, int64_t N, int64_t ldt,
                    float* out_host, int64_t ldo);
/* The PQ comparator through the same executor, which must have
 * been created with a PQ model: host rows -> host codes (mdn_encode_pq), or
 * host rows -> host out (mdn_encode_pq + mdn_scan per chunk on the device).
 * The tree-based host calls return MDN_ESTATE for a PQ executor and these
 * two for a MADDNESS one. */
int mdn_encode_pq_host(mdn_exec* exec, const float* A_host, int64_t N, int64_t lda,
                       uint8_t* codes_host);
int mdn_amm_pq_host(mdn_exec* exec, const float* A_host, int64_t N, int64_t lda,
                    float* out_host, int64_t ldo);
/* g on column-major host A: split columns in, packed codes (N x ceil(C/2),
 * contiguous host u8) out. */
int mdn_encode_cm_host(mdn_exec* exec, const float* At_host, int64_t N, int64_t ldt,
                       uint8_t* codes_host);

/* --------------------------------------------------------- diagnostics -- */

/* Roofline probe (not part of the method): a plain streaming kernel with the
 * fused path's byte mix -- reads every element of A (device fp32 N x D, lda,
 * D % 4 == 0, 16-B aligned) and writes M floats per row of out (device,
 * ldo) -- so bench.py can report the achievable bandwidth for this mix next
 * to the fused kernel's. */
int mdn_stream_probe(const float* A, int64_t N, int64_t lda, int64_t D, float* out,
                     int64_t ldo, int64_t M, void* stream);
/* Pipeline ceiling probe (not part of the method): the fused kernel that
 * mdn_amm would launch for these arguments (the general warp-specialised
 * k_amm_ws: same TMA boxes, stage ring, code ring, grid, warp roles and
 * output stores) with Algorithm 1 and the table scan removed -- every output
 * element is beta32. Its time is the achievable ceiling of mdn_amm's own data
 * movement. Arguments, layouts and errors as mdn_amm; MDN_EINVAL also when
 * mdn_amm would not use the general pipeline for these shapes (register-tree
 * or generic kernels). */
int mdn_amm_probe(const mdn_model* model, const mdn_luts* luts, const float* A, int64_t N,
                  int64_t lda, float* out, int64_t ldo, void* stream);

/* --------------------------------------------------------------- misc -- */

const char* mdn_status_str(int status);
int mdn_abi_version(void);
/* Kernel variant the last-chosen dispatch would use for these shapes
 * (for tests/bench reporting): writes a NUL-terminated name into buf. */
int mdn_amm_variant(const mdn_model* model, const mdn_luts* luts, int64_t lda,
                    char* buf, size_t len);

/*
 * File formats (little-endian). They are the only thing the oracle and this
 * library share; each side has its own reader/writer.
 *
 * model.mdnm v1
 *   char[4] "MDNM" | u32 ver = 1 | u32 C | u32 D | u32 K = 16 | u32 flags (bit0 ridge,
 *   bit1 PQ model: P = K-means prototypes, tree fields unused)
 *   f64 lambda | u64 n_train | u64 seed
 *   C records: u32 sub_begin | u32 sub_end | u16 dim[4] | f32 thr[15]
 *              (thr in heap order: level t node p at 2^t - 1 + p)
 *   f32 P[16C][D]
 *   u64 fingerprint = FNV-1a 64 of all preceding bytes
 *
 * luts.mdnl v1
 *   char[4] "MDNL" | u32 ver = 1 | u32 C | u32 M | u32 K = 16 | u32 mode | u32 U
 *   i32 l | f32 alpha | f32 beta32 | u64 model_fingerprint | f64 delta[C]
 *   u8 Tq[C][16][M]
 *   u64 fingerprint = FNV-1a 64 of all preceding bytes
 */

#ifdef __cplusplus
}
#endif
#endif /* MADDNESS_H_ */
