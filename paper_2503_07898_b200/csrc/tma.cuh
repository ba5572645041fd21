// tma.cuh -- the Blackwell bulk-copy (TMA) path for whole-block staging:
// one elected thread moves a contiguous global span into shared memory with
// cp.async.bulk (SASS UBLKCP), completion tracked by an mbarrier's
// transaction count; the CTA's threads sleep on the barrier (try_wait) while
// their own metadata loads overlap the copy. Used by the block-sparse step
// kernels, whose 8^3 blocks keep each block's Q population planes in one
// contiguous span (BlockField layout ((b*Q)+c)*E^3 + local, sparse.hpp:62-86).
#pragma once

#include <cstdint>

namespace voxl_b200 {

__device__ __forceinline__ unsigned smem_addr(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}

/// mbarrier with `count` expected arrivals (one thread).
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
    // make the initialised barrier visible to the async (TMA) proxy
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

/// Arrive (one of the expected arrivals) and add `bytes` to the phase's
/// expected transaction count.
__device__ __forceinline__ void mbar_arrive_expect_tx(unsigned long long* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
                 : "memory");
}

/// Bulk copy of `bytes` (multiple of 16; both addresses 16-byte aligned)
/// global -> shared, completing `bytes` transactions on `bar`.
__device__ __forceinline__ void tma_bulk_g2s(void* smem, const void* gmem, unsigned bytes, unsigned long long* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_addr(smem)),
                 "l"(gmem), "r"(bytes), "r"(smem_addr(bar))
                 : "memory");
}

/// Sleep until the barrier's phase `parity` has completed.
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
    asm volatile(
        "{\n"
        "  .reg .pred done;\n"
        "WAIT_%=:\n"
        "  mbarrier.try_wait.parity.shared::cta.b64 done, [%0], %1;\n"
        "  @!done bra WAIT_%=;\n"
        "}\n" ::"r"(smem_addr(bar)),
        "r"(parity)
        : "memory");
}

} // namespace voxl_b200
