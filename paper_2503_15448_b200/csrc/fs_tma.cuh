// TMA tensor loads and 128-byte-swizzled tcgen05 operand descriptors
// (sm_100a, inline PTX), for kernels whose operands are staged by
// cp.async.bulk.tensor from row-major global matrices.
//
// A tensor map describes a 3-D bf16 array [slot][row][col] whose innermost
// dimension (col) is contiguous; boxes are 64 columns (128 B, one swizzle
// row) by `box_rows` rows, landing in shared memory as box_rows rows of
// 128 B, 16-byte chunks XOR-swizzled within 1024-byte (8-row) atoms.
// Out-of-range rows/columns of a box are zero-filled by the TMA unit.
//
// The same smem image serves both operand majors of tcgen05.mma:
//   K-major  (K along the 64 columns, M/N along rows): SBO = 1024 B between
//            8-row groups; a K step of 16 elements advances the start by 32 B.
//   MN-major (M/N along the 64 columns, K along rows): SBO = 1024 B between
//            8-row (8-k) groups, LBO = byte distance between consecutive
//            64-column boxes along M/N; a K step of 16 advances by 2048 B.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "fs_tc.cuh"

namespace fs {
namespace tma {

// ------------------------------------------------------------------ host
// cuTensorMapEncodeTiled through the runtime's driver entry point (no libcuda link)
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

inline EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}

// bf16 [slots][rows][cols], row stride `ld` elements (ld*2 % 16 == 0), slot
// stride `slot_bytes` (% 16 == 0); box = 64 cols x box_rows rows x 1 slot.
inline bool make_map(CUtensorMap* m, const void* base, int64_t cols, int64_t rows, int64_t slots, int64_t ld,
                     int64_t slot_bytes, int box_rows) {
  EncodeTiledFn fn = encode_fn();
  if (!fn || cols < 1 || rows < 1 || slots < 1 || (ld * 2) % 16 || slot_bytes % 16 || box_rows < 1 ||
      box_rows > 256 || (reinterpret_cast<uintptr_t>(base) & 15))
    return false;
  cuuint64_t dim[3] = {(cuuint64_t)cols, (cuuint64_t)rows, (cuuint64_t)slots};
  cuuint64_t stride[2] = {(cuuint64_t)(ld * 2), (cuuint64_t)(slots > 1 ? slot_bytes : ld * 2 * rows)};
  cuuint32_t box[3] = {64u, (cuuint32_t)box_rows, 1u};
  cuuint32_t estr[3] = {1u, 1u, 1u};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dim, stride, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// ------------------------------------------------------------------ device
__device__ __forceinline__ void prefetch_map(const CUtensorMap* m) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(m)) : "memory");
}
__device__ __forceinline__ void expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(tc::smem_u32(bar)), "r"(bytes)
               : "memory");
}
// one box at (col, row, slot) into 1024-byte-aligned shared memory; completes on `bar`
__device__ __forceinline__ void load_3d(void* dst, const CUtensorMap* m, int col, int row, int slot, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::
          "r"(tc::smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(col), "r"(row), "r"(slot), "r"(tc::smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(tc::smem_u32(bar)) : "memory");
}

// tcgen05 shared-memory descriptor, SWIZZLE_128B (layout code 2), sm100 version 1
__device__ __forceinline__ uint64_t desc_sw128(uint32_t saddr, uint32_t lbo_bytes, uint32_t sbo_bytes) {
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)((lbo_bytes >> 4) & 0x3FFFu) << 16) |
         ((uint64_t)((sbo_bytes >> 4) & 0x3FFFu) << 32) | (1ull << 46) | (2ull << 61);
}
// K-major operand: rows = M/N, 64 K columns per box; K slice kk (16 elements)
__device__ __forceinline__ uint64_t kmajor(uint32_t saddr, int kk) {
  return desc_sw128(saddr + 32u * (uint32_t)kk, 16u, 1024u);
}
// MN-major operand: boxes of 64 M/N columns x K rows, `box_bytes` apart along M/N; K slice kk (16 rows)
__device__ __forceinline__ uint64_t mnmajor(uint32_t saddr, int kk, uint32_t box_bytes) {
  return desc_sw128(saddr + 2048u * (uint32_t)kk, box_bytes, 1024u);
}

}  // namespace tma
}  // namespace fs
