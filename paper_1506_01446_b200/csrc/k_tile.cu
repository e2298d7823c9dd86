// k_tile.cu -- tile-sort kernels (all tile sizes) and the table lookups.
#include "bitonic_static.cuh"
#include "kernel_tables.hpp"

namespace b200 {

// key + payload tiles: 16 pairs per thread (keys + payloads = 32 registers)
static PassFn kv_tile(int C) {
  constexpr int MODE = 1;
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

PassFn find_tile_kernel(int C, int R, int mode) {
  if (mode == 1) return R == (C < 4 ? C : 4) ? kv_tile(C) : nullptr;
  if (mode == 2) return find_tile_kernel_k64(C, R);
  if (R == 6) {  // 64 keys per thread: fewer shared-memory rounds
    switch (C) {
      case 12: return &tile_sort_kernel<12, 6>;
      case 13: return &tile_sort_kernel<13, 6>;
      case 14: return &tile_sort_kernel<14, 6>;
      default: return nullptr;
    }
  }
  if (R == 4) {
    switch (C) {
      case 10: return &tile_sort_kernel<10, 4>;
      case 11: return &tile_sort_kernel<11, 4>;
      case 12: return &tile_sort_kernel<12, 4>;
      case 13: return &tile_sort_kernel<13, 4>;
      case 14: return &tile_sort_kernel<14, 4>;
      default: return nullptr;
    }
  }
  if (R != 5 && C >= 5) return nullptr;
  switch (C) {
    case 1: return &tile_sort_kernel<1>;
    case 2: return &tile_sort_kernel<2>;
    case 3: return &tile_sort_kernel<3>;
    case 4: return &tile_sort_kernel<4>;
    case 5: return &tile_sort_kernel<5>;
    case 6: return &tile_sort_kernel<6>;
    case 7: return &tile_sort_kernel<7>;
    case 8: return &tile_sort_kernel<8>;
    case 9: return &tile_sort_kernel<9>;
    case 10: return &tile_sort_kernel<10>;
    case 11: return &tile_sort_kernel<11>;
    case 12: return &tile_sort_kernel<12>;
    case 13: return &tile_sort_kernel<13>;
    case 14: return &tile_sort_kernel<14>;
    case 15: return &tile_sort_kernel<15>;
    default: return nullptr;
  }
}

namespace {
struct Tables {
  MergeTable t[kMergeCMax + 1];
  MergeTable t4[kMergeCMax + 1];
  MergeTable tkv[kMergeCMax + 1];
  MergeTable tk64[kMergeCMax + 1];
  Tables() {
    for (auto& x : t) x = MergeTable{};
    for (auto& x : t4) x = MergeTable{};
    for (auto& x : tkv) x = MergeTable{};
    fill_merge_table_12_kv(tkv[12]);
    fill_merge_table_13_kv(tkv[13]);
    for (auto& x : tk64) x = MergeTable{};
    fill_merge_table_12_k64(tk64[12]);
    fill_merge_table_13_k64(tk64[13]);
    fill_merge_table_12_r4(t4[12]);
    fill_merge_table_13_r4(t4[13]);
    fill_merge_table_14_r4(t4[14]);
    fill_merge_table_11(t[11]);
    fill_merge_table_12(t[12]);
    fill_merge_table_13(t[13]);
    fill_merge_table_14(t[14]);
    fill_merge_table_15(t[15]);
  }
};
const Tables& tables() {
  static Tables tb;
  return tb;
}
}  // namespace

PassFn find_merge_kernel(int C, int SA, int SB, int R, int mode) {
  if (C < kMergeCMin || C > kMergeCMax) return nullptr;
  if (R != 5 && R != 4) return nullptr;
  if (mode != 0 && R != 4) return nullptr;
  const MergeTable& t = mode == 1   ? tables().tkv[C]
                        : mode == 2 ? tables().tk64[C]
                                    : (R == 5 ? tables().t[C] : tables().t4[C]);
  if (SB >= 0 && SA == SB - 1 && SB < 16) return t.th[SB];
  if (SA < 0 && SB >= 0 && SB < 16) return t.ho[SB];
  if (SB < 0 && SA >= 0 && SA < 16) return t.to[SA];
  return nullptr;
}

}  // namespace b200
