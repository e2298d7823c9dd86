// merge_table.cuh -- instantiates every merge shape of one tile size C.
#pragma once

#include <utility>

#include "bitonic_static.cuh"
#include "kernel_tables.hpp"

namespace b200 {

template <int C, int A, int R, int MODE, bool VIRT = false>
PassFn th_entry() {
  if constexpr (A >= 2 && A <= C - 1) return &merge_kernel<C, A - 1, A, R, MODE, VIRT>;
  else return nullptr;
}
template <int C, int A, int R, int MODE, bool VIRT = false>
PassFn ho_entry() {
  if constexpr (A >= 2 && A <= C - 1) return &merge_kernel<C, -1, A, R, MODE, VIRT>;
  else return nullptr;
}
template <int C, int SA, int R, int MODE, bool VIRT = false>
PassFn to_entry() {
  if constexpr (SA >= 0 && SA <= C - 1) return &merge_kernel<C, SA, -1, R, MODE, VIRT>;
  else return nullptr;
}
template <int C, int R, int MODE, bool VIRT = false, int... I>
void fill_merge_table(MergeTable& t, std::integer_sequence<int, I...>) {
  ((t.th[I] = th_entry<C, I, R, MODE, VIRT>()), ...);
  ((t.ho[I] = ho_entry<C, I, R, MODE, VIRT>()), ...);
  ((t.to[I] = to_entry<C, I, R, MODE, VIRT>()), ...);
}

}  // namespace b200

#define B200_DEFINE_MERGE_TABLE(CC)                                      \
  namespace b200 {                                                       \
  void fill_merge_table_##CC(MergeTable& t) {                            \
    fill_merge_table<CC, 5, 0>(t, std::make_integer_sequence<int, 16>{}); \
  }                                                                      \
  }

#define B200_DEFINE_MERGE_TABLE_R4(CC)                                   \
  namespace b200 {                                                       \
  void fill_merge_table_##CC##_r4(MergeTable& t) {                       \
    fill_merge_table<CC, 4, 0>(t, std::make_integer_sequence<int, 16>{}); \
  }                                                                      \
  }

#define B200_DEFINE_MERGE_TABLE_KV(CC)                                   \
  namespace b200 {                                                       \
  void fill_merge_table_##CC##_kv(MergeTable& t) {                       \
    fill_merge_table<CC, 4, 1>(t, std::make_integer_sequence<int, 16>{}); \
  }                                                                      \
  }

#define B200_DEFINE_MERGE_TABLE_K64(CC)                                  \
  namespace b200 {                                                       \
  void fill_merge_table_##CC##_k64(MergeTable& t) {                      \
    fill_merge_table<CC, 4, 2>(t, std::make_integer_sequence<int, 16>{}); \
  }                                                                      \
  }
