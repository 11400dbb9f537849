// dev_util.cuh -- small sm_100a device helpers: mbarrier + bulk-copy (TMA
// engine, cp.async.bulk) PTX wrappers and warp reductions.
#pragma once

#include <cstdint>
#include <cstdio>

// Device-side invariant checks (bounds of every queue / run / list index the
// kernels compute).  Compiled in only for the checked build
// (-DFIZI_DEVICE_CHECKS, libfizi_checked.so): a violated check traps, which
// surfaces as a sticky CUDA error in the calling test.
#ifdef FIZI_DEVICE_CHECKS
#define FIZI_DCHECK(cond)                                                              \
  do {                                                                                 \
    if (!(cond)) {                                                                     \
      printf("FIZI_DCHECK failed: %s at %s:%d (block %d thread %d)\n", #cond, __FILE__, \
             __LINE__, (int)blockIdx.x, (int)threadIdx.x);                             \
      __trap();                                                                        \
    }                                                                                  \
  } while (0)
#else
#define FIZI_DCHECK(cond) \
  do {                    \
  } while (0)
#endif

namespace fizi {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}

__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

// One bulk global->shared copy completing on `bar` (bytes % 16 == 0, both
// addresses 16-byte aligned).  Streams through L2 with evict-first priority:
// every frame byte is read exactly once.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}

// One bulk shared->global copy (TMA engine), tracked by the issuing thread's
// bulk async-group; call bulk_s2g_wait before the shared buffer is reused.
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, uint32_t bytes) {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // generic smem writes -> async proxy
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst),
               "r"(smem_u32(src)), "r"(bytes)
               : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}

__device__ __forceinline__ void bulk_s2g_wait() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}

__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      " .reg .pred p;\n"
      "WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// 4 bits -> 4 bytes {0,1} (bit i -> byte i)
__device__ __forceinline__ uint32_t expand4(uint32_t v) { return (v * 0x00204081u) & 0x01010101u; }

__device__ __forceinline__ uint32_t warp_sum_u32(uint32_t v) {
  return __reduce_add_sync(0xFFFFFFFFu, v);
}

}  // namespace fizi
