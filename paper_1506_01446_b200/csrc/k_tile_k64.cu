// k_tile_k64.cu -- tile-sort kernels for 64-bit keys (hi/lo word arrays,
// 16 keys per thread), in their own translation unit to keep builds parallel.
#include "bitonic_static.cuh"
#include "kernel_tables.hpp"

namespace b200 {

PassFn find_tile_kernel_k64(int C, int R) {
  constexpr int MODE = 2;
  if (R != (C < 4 ? C : 4)) return nullptr;
  switch (C) {
    case 1: return &tile_sort_kernel<1, 1, MODE>;
    case 2: return &tile_sort_kernel<2, 2, MODE>;
    case 3: return &tile_sort_kernel<3, 3, MODE>;
    case 4: return &tile_sort_kernel<4, 4, MODE>;
    case 5: return &tile_sort_kernel<5, 4, MODE>;
    case 6: return &tile_sort_kernel<6, 4, MODE>;
    case 7: return &tile_sort_kernel<7, 4, MODE>;
    case 8: return &tile_sort_kernel<8, 4, MODE>;
    case 9: return &tile_sort_kernel<9, 4, MODE>;
    case 10: return &tile_sort_kernel<10, 4, MODE>;
    case 11: return &tile_sort_kernel<11, 4, MODE>;
    case 12: return &tile_sort_kernel<12, 4, MODE>;
    case 13: return &tile_sort_kernel<13, 4, MODE>;
    default: return nullptr;
  }
}

}  // namespace b200
