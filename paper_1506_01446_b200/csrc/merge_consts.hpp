// merge_consts.hpp -- tile geometry of the merge-path kernels (merge_split.cuh),
// shared with the host code that sizes their scratch.
#pragma once

#include <cstdint>

namespace b200 {

constexpr int kMergeThreads = 256;
constexpr int kMergeItems = 8;
constexpr uint64_t kMergeTile = (uint64_t)kMergeThreads * kMergeItems;

}  // namespace b200
