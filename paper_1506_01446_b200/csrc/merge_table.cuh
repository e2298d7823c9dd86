// merge_table.cuh -- instantiates every merge shape of one tile size C.
#pragma once

#include <utility>

#include "bitonic_static.cuh"
#include "kernel_tables.hpp"

namespace b200 {

template <int C, int A>
PassFn th_entry() {
  if constexpr (A >= 2 && A <= C - 1) return &merge_kernel<C, A - 1, A>;
  else return nullptr;
}
template <int C, int A>
PassFn ho_entry() {
  if constexpr (A >= 2 && A <= C - 1) return &merge_kernel<C, -1, A>;
  else return nullptr;
}
template <int C, int SA>
PassFn to_entry() {
  if constexpr (SA >= 0 && SA <= C - 1) return &merge_kernel<C, SA, -1>;
  else return nullptr;
}
template <int C, int... I>
void fill_merge_table(MergeTable& t, std::integer_sequence<int, I...>) {
  ((t.th[I] = th_entry<C, I>()), ...);
  ((t.ho[I] = ho_entry<C, I>()), ...);
  ((t.to[I] = to_entry<C, I>()), ...);
}

}  // namespace b200

#define B200_DEFINE_MERGE_TABLE(CC)                                      \
  namespace b200 {                                                       \
  void fill_merge_table_##CC(MergeTable& t) {                            \
    fill_merge_table<CC>(t, std::make_integer_sequence<int, 16>{});      \
  }                                                                      \
  }
