// PTX helpers used only by the microbenchmarks in tools/ (not by the library):
// TMA tensor gather4 (measured slower than the cp.async gather, membench11/13/14).
#pragma once

#include <cuda.h>
#include "tw_ptx.cuh"

namespace tw {
namespace ptx {

__device__ __forceinline__ void prefetch_tmap(const CUtensorMap *m) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(m)) : "memory");
}
// 4 arbitrary rows (r0..r3) x box-width columns starting at column c0 of a
// 2-D tensor -> 4 consecutive box rows in shared memory (swizzled per the
// tensor map).  Out-of-bounds rows/columns are zero-filled.
__device__ __forceinline__ void tma_gather4(void *smem_dst, const CUtensorMap *m, uint64_t *bar, int32_t c0,
                                            int4 rows, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3, %4, %5, %6}], [%7], %8;" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(c0), "r"(rows.x), "r"(rows.y), "r"(rows.z), "r"(rows.w),
      "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}

}  // namespace ptx
}  // namespace tw
