// k_virt.cu -- the virtual-padding kernels (non-power-of-two single arrays,
// bitonic_static.cuh VIRT): 2^13-key tile sort and merge passes on 2^13-key
// cosets, 32 keys per thread; the planner restricts virtual plans to these.
#include "merge_table.cuh"

namespace b200 {

namespace {
struct VirtTable {
  MergeTable t13;
  VirtTable() {
    t13 = MergeTable{};
    fill_merge_table<13, 5, 0, true>(t13, std::make_integer_sequence<int, 16>{});
  }
};
}  // namespace

PassFn find_virtual_kernel(bool tile, int C, int SA, int SB, int R) {
  static const VirtTable vt;
  if (C != 13 || R != 5) return nullptr;
  if (tile) return &tile_sort_kernel<13, 5, 0, true>;
  const MergeTable& t = vt.t13;
  if (SB >= 0 && SA == SB - 1 && SB < 16) return t.th[SB];
  if (SA < 0 && SB >= 0 && SB < 16) return t.ho[SB];
  if (SB < 0 && SA >= 0 && SA < 16) return t.to[SA];
  return nullptr;
}

}  // namespace b200
