// k_tile_tma.cu -- the TMA-loaded tile sort (bitonic_tma.cuh) and its tensor map.
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include "bitonic_tma.cuh"
#include "kernel_tables.hpp"

namespace b200 {

TmaTileFn find_tile_tma_kernel(int C) {
  switch (C) {
    case 10: return &tile_sort_tma_kernel<10>;
    case 11: return &tile_sort_tma_kernel<11>;
    case 12: return &tile_sort_tma_kernel<12>;
    case 13: return &tile_sort_tma_kernel<13>;
    default: return nullptr;
  }
}

// keys[0..total) viewed as rows of 32 uint32 (128 bytes), boxes of 2^(C-5)
// rows, 128-byte swizzle.
bool make_tile_tensor_map(CUtensorMap* map, const uint32_t* keys, uint64_t total, int C) {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      fn = nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }();
  if (encode == nullptr || total % 32 != 0 || C < 8 || C > 13) return false;
  cuuint64_t dims[2] = {32, total / 32};
  cuuint64_t strides[1] = {128};
  cuuint32_t box[2] = {32, 1u << (C - 5)};
  cuuint32_t estr[2] = {1, 1};
  return encode(map, CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, const_cast<uint32_t*>(keys), dims,
                strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace b200
