// merge_consts.hpp -- tile geometry of the merge-path kernels (merge_split.cuh),
// shared with the host code that sizes their scratch.
#pragma once

#include <cstdint>

namespace b200 {

// merge_bitonic_kernel: one 2^kMergeC-key bitonic tile per CTA
constexpr int kMergeC = 13;
constexpr uint64_t kMergeTile = uint64_t{1} << kMergeC;

}  // namespace b200
