// Tensor-map (TMA descriptor) cache for the paged KV pool.
#pragma once
#include <cuda.h>
#include <stdint.h>

namespace ds {
// 2D bf16 map over a head-major pool layer viewed as [rows][128] (row = kv_head *
// head_stride + cell, 256-byte rows), box = 64 columns (128 B, SWIZZLE_128B) x
// box_rows rows.  Cached by (base, rows, box_rows); returns nullptr on failure.
const CUtensorMap* kv_tensor_map(const void* base, int64_t rows, int box_rows);
// 3D bf16 map over a row-major matrix [rows][cols] viewed as (64, rows, cols/64)
// - 128-byte column slabs - with box (64, box_rows, box_slabs), SWIZZLE_128B:
// one TMA op moves box_rows x (64*box_slabs) elements, landing as
// [box_slabs][box_rows][128 B] with 16-byte chunk c of smem row R at c ^ (R & 7).
// Rows >= `rows` are zero-filled.  Cached; nullptr on failure.
const CUtensorMap* slab_tensor_map(const void* base, int64_t rows, int64_t cols, int box_rows,
                                   int box_slabs);
}  // namespace ds

#ifdef __CUDACC__
namespace ds {
// 2D TMA tile load, completion counted on an mbarrier (tx bytes)
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes "
      "[%0], [%1, {%2, %3}], [%4];\n" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(dst))),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1),
      "r"(static_cast<uint32_t>(__cvta_generic_to_shared(bar)))
      : "memory");
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int c0, int c1,
                                            int c2, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes "
      "[%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(dst))),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2),
      "r"(static_cast<uint32_t>(__cvta_generic_to_shared(bar)))
      : "memory");
}
__device__ __forceinline__ void tma_prefetch_desc(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}
}  // namespace ds
#endif
