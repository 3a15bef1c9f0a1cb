// TMA-engine bulk copies (cp.async.bulk, non-tensor) completing on shared
// memory mbarriers: the producer side of the warp-specialised row rings used by
// the Gower stream (contiguous tiles) and the piece kernels (gathered rows).
#pragma once
#include <cstdint>

namespace bulk {
__device__ __forceinline__ unsigned saddr(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void bar_init(uint64_t* b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(saddr(b)), "r"(count));
}
__device__ __forceinline__ void bar_fence() {
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
__device__ __forceinline__ void arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(saddr(b)) : "memory");
}
// one arrival that also announces `bytes` of bulk-copy completions for the phase
__device__ __forceinline__ void arrive_expect(uint64_t* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(saddr(b)),
               "r"(bytes) : "memory");
}
// a bulk copy global -> shared (16-byte aligned, size a multiple of 16)
__device__ __forceinline__ void copy(void* dst, const void* src, unsigned bytes, uint64_t* b) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
      ::"r"(saddr(dst)), "l"(src), "r"(bytes), "r"(saddr(b)) : "memory");
}
__device__ __forceinline__ void load(void* dst, const void* src, unsigned bytes, uint64_t* b) {
  arrive_expect(b, bytes);
  copy(dst, src, bytes, b);
}
__device__ __forceinline__ void wait(uint64_t* b, unsigned phase) {
  asm volatile(
      "{\n.reg .pred P;\nWAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n"
      "@!P bra WAIT_%=;\n}\n" ::"r"(saddr(b)), "r"(phase) : "memory");
}
}  // namespace bulk
