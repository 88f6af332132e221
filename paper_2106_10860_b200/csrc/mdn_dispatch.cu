// Kernel selection for the hot-path entry points.
#include <cuda_runtime.h>

#include "mdn_internal.h"

namespace mdn {

cudaError_t launch_encode_generic(const TreesDev&, const float*, int64_t, int64_t, uint8_t*,
                                  cudaStream_t);
cudaError_t launch_scan_generic(const LutsDev&, const uint8_t*, int64_t, int32_t*, float*, int64_t,
                                cudaStream_t);
cudaError_t launch_amm_generic(const TreesDev&, const LutsDev&, const float*, int64_t, int64_t,
                               float*, int64_t, cudaStream_t);

cudaError_t launch_encode(const TreesDev& t, const float* A, int64_t N, int64_t lda, uint8_t* codes,
                          cudaStream_t s) {
  return launch_encode_generic(t, A, N, lda, codes, s);
}

cudaError_t launch_scan(const LutsDev& l, const uint8_t* codes, int64_t N, int32_t* sums,
                        float* out, int64_t ldo, cudaStream_t s) {
  return launch_scan_generic(l, codes, N, sums, out, ldo, s);
}

const char* amm_variant_name(const TreesDev&, const LutsDev&, const float*, int64_t, const float*,
                             int64_t) {
  return "generic";
}

cudaError_t launch_amm(const TreesDev& t, const LutsDev& l, const float* A, int64_t N, int64_t lda,
                       float* out, int64_t ldo, cudaStream_t s) {
  return launch_amm_generic(t, l, A, N, lda, out, ldo, s);
}

}  // namespace mdn
