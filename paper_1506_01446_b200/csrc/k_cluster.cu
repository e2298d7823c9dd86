// k_cluster.cu -- the 2-CTA cluster merge passes (bitonic_cluster.cuh).
#include "bitonic_cluster.cuh"
#include "kernel_tables.hpp"

namespace b200 {

namespace {
template <int B, int R>
PassFn cl_entry() {
  if constexpr (B >= 4 && B <= 13) return &cluster_merge_kernel<B, R>;
  else return nullptr;
}
template <int R, int... I>
void fill(PassFn* t, std::integer_sequence<int, I...>) {
  ((t[I] = cl_entry<I, R>()), ...);
}
struct ClusterTable {
  PassFn r5[16] = {};
  ClusterTable() { fill<5>(r5, std::make_integer_sequence<int, 16>{}); }
};
}  // namespace

PassFn find_cluster_kernel(int B, int R) {
  static const ClusterTable t;
  if (B < 0 || B > 15 || R != 5) return nullptr;
  return t.r5[B];
}

}  // namespace b200
