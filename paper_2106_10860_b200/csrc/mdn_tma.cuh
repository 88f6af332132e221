// sm_100a PTX helpers shared by the TMA-fed kernels (mdn_fast.cu, mdn_small.cu):
// mbarrier init / arrive / wait, 2-D TMA tensor loads, L2 cache policies, and
// the host-side tensor-map / device-attribute helpers defined in mdn_fast.cu.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace mdn {
namespace fast {

__device__ __forceinline__ uint32_t su32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  uint32_t ok = 0;
  const uint32_t a = su32(b);
  do {
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(ok)
        : "r"(a), "r"(parity)
        : "memory");
  } while (!ok);
}
// As mbar_wait, but the waiting thread is suspended (up to the hint, in ns)
// until the phase completes instead of spinning: the spin loop's
// YIELD / TRYWAIT / BRA otherwise takes issue slots from the compute warps.
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* b, uint32_t parity) {
  uint32_t ok = 0;
  const uint32_t a = su32(b);
  do {
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3; selp.u32 %0, 1, 0, p; }"
        : "=r"(ok)
        : "r"(a), "r"(parity), "r"(1000000u)
        : "memory");
  } while (!ok);
}
// Optional L2 cache policy for the A tiles (Params::l2_hint; 0 = none, the
// default: measured on cls100, evict_first costs 9% -- 2.45e9 vs 2.70e9 rows/s).
__device__ __forceinline__ uint64_t l2_policy(int hint) {
  uint64_t pol = 0;
  if (hint == 1) asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  if (hint == 2) asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  if (hint == 3) asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int x, int y,
                                            uint64_t* bar, int hint, uint64_t policy) {
  if (hint == 0) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3}], [%4];" ::"r"(su32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(su32(bar))
        : "memory");
  } else {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(su32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(su32(bar)), "l"(policy)
        : "memory");
  }
}

// TMA gather4 (sm_100a): rows r0..r3 of a 2-D tensor, `box inner` elements
// each from column x, land back to back at dst (box height 1 in the map).
__device__ __forceinline__ void tma_gather4(void* dst, const CUtensorMap* map, int x, int r0, int r1,
                                            int r2, int r3, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(su32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(su32(bar))
      : "memory");
}

// 2-D TMA tensor store (shared -> global, bulk-group completion): the box at
// (x, y) of the map's tensor is written from dense shared memory at src;
// elements outside the tensor (rows >= N, columns >= M) are not written.
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, const void* src, int x, int y) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(x), "r"(y), "r"(su32(src))
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
// at most N of this thread's committed bulk groups still READING shared memory
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
// all of this thread's bulk groups complete (writes performed)
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
// this thread's generic-proxy shared-memory writes visible to the async proxy (TMA)
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// Host helpers (mdn_fast.cu).
struct DevInfo {
  int sms = 148;
  int smem_optin = 232448;
};
DevInfo dev_info();
// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (kernel, device,
// size): the attribute costs ~1 us per call, more than a small launch.
cudaError_t ensure_smem(const void* kernel, size_t smem);
bool make_tmap(CUtensorMap* m, const void* A, int64_t N, int64_t lda, int D, int SW, int R, int es);
// fp32 output [N][M] at row pitch ldo (floats), stored in boxes of bw columns x bh rows
bool make_tmap_out(CUtensorMap* m, float* out, int64_t N, int M, int64_t ldo, int bw, int bh);
int knob_hint();
bool knob_bq();
int env_int(const char* name, int dflt);   // tuning knobs (mdn_fast.cu)

}  // namespace fast
}  // namespace mdn
