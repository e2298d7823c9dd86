// kernel_tables.hpp -- lookup of the compile-time specialised pass kernels.
#pragma once

#include "bitonic_engine.cuh"

struct CUtensorMap_st;

namespace b200 {

using PassFn = void (*)(PassParams);

// Tile-sort kernel for a 2^C tile (C in [1, 15]) with 2^R keys per thread
// (R = 5, or R = 4 for the instantiated latency-bound sizes).
// mode: 0 keys only, 1 key + payload, 2 64-bit keys (hi/lo word arrays)
PassFn find_tile_kernel(int C, int R = 5, int mode = 0);
// Specialised merge kernel for local bits SA..0 then C-1..SB, or nullptr when
// that shape was not instantiated (the caller then uses the runtime-dispatched
// bitonic_pass_kernel<C>).
PassFn find_merge_kernel(int C, int SA, int SB, int R = 5, int mode = 0);
PassFn find_tile_kernel_k64(int C, int R);  // k_tile_k64.cu
// 2-CTA cluster pass (bitonic_cluster.cuh): tail bits B..0 fused with the
// head of the next phase on a 2^15-key coset (B in [4, 13]); nullptr otherwise.
PassFn find_cluster_kernel(int B, int R = 5);
// Virtual-padding kernels (k_virt.cu): 2^13-key tile / merge shapes, R = 5.
PassFn find_virtual_kernel(bool tile, int C, int SA, int SB, int R);
// TMA-loaded tile sort (bitonic_tma.cuh), C in [10, 13], 32 keys per thread
using TmaTileFn = void (*)(PassParams, const CUtensorMap_st);
TmaTileFn find_tile_tma_kernel(int C);
bool make_tile_tensor_map(CUtensorMap_st* map, const uint32_t* keys, uint64_t total, int C);

// Instantiated merge tile sizes.
constexpr int kMergeCMin = 11;
constexpr int kMergeCMax = 15;

struct MergeTable {
  PassFn th[16];  // SA = A-1, SB = A   (tail + head),  A in [2, C-1]
  PassFn ho[16];  // SA = -1,  SB = A   (head only),    A in [2, C-1]
  PassFn to[16];  // SA,       SB = -1  (tail only),    SA in [0, C-1]
};

void fill_merge_table_11(MergeTable& t);
void fill_merge_table_12(MergeTable& t);
void fill_merge_table_13(MergeTable& t);
void fill_merge_table_14(MergeTable& t);
void fill_merge_table_15(MergeTable& t);
void fill_merge_table_12_r4(MergeTable& t);
void fill_merge_table_13_r4(MergeTable& t);
void fill_merge_table_14_r4(MergeTable& t);
void fill_merge_table_12_kv(MergeTable& t);
void fill_merge_table_13_kv(MergeTable& t);
void fill_merge_table_12_k64(MergeTable& t);
void fill_merge_table_13_k64(MergeTable& t);

}  // namespace b200
