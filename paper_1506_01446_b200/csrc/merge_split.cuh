// merge_split.cuh -- merge-split of two sorted shards (the compare-exchange
// of the rank-level bitonic network in the partitioned sort).
//
// The reference has no multi-device path; north_star adds one:
// each rank sorts its contiguous shard (work_slice rule, worker_pool.hpp:
// 22-25), then every CE of a bitonic network over the G shards is replaced by
// a merge-split: the lower rank of an ascending pair keeps the m smallest
// keys of the 2m union, the upper rank the m largest (block 0-1 principle).
//
// Implementation: merge path.  merge_partition_kernel finds, for every
// 2048-key output tile, how many keys come from the local shard (a binary
// search on the diagonal of the virtual merge).  merge_tile_kernel then
// stages the two input windows in shared memory, each thread finds its own
// 8-key sub-diagonal, merges serially and the CTA writes the tile back
// coalesced.  `partner` may be a peer-device pointer: the reads then travel
// over NVLink inside this kernel (no separate copy), which is the fused
// exchange + merge.
#pragma once

#include <cstdint>

namespace b200 {

constexpr int kMergeThreads = 256;
constexpr int kMergeItems = 8;
constexpr uint64_t kMergeTile = (uint64_t)kMergeThreads * kMergeItems;

// Number of keys of A among the first d keys of merge(A, B) (A first on ties).
__device__ __forceinline__ uint64_t corank_global(uint64_t d, uint64_t m,
                                                  const uint32_t* A,
                                                  const uint32_t* B,
                                                  uint32_t kx) {
  uint64_t lo = d > m ? d - m : 0;
  uint64_t hi = d < m ? d : m;
  while (lo < hi) {
    const uint64_t mid = (lo + hi) >> 1;
    if ((A[mid] ^ kx) <= (B[d - mid - 1] ^ kx)) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

__global__ void merge_partition_kernel(const uint32_t* __restrict__ A,
                                       const uint32_t* __restrict__ B,
                                       uint64_t m, int keep_high, uint32_t kx,
                                       uint64_t* __restrict__ coranks,
                                       uint64_t nb) {
  const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nb) return;
  const uint64_t off = keep_high ? m : 0;
  uint64_t d = t * kMergeTile;
  if (d > m) d = m;
  coranks[t] = corank_global(off + d, m, A, B, kx);
}

__global__ void __launch_bounds__(kMergeThreads)
merge_tile_kernel(const uint32_t* __restrict__ A, const uint32_t* __restrict__ B,
                  uint64_t m, int keep_high, uint32_t kx,
                  const uint64_t* __restrict__ coranks,
                  uint32_t* __restrict__ out) {
  __shared__ uint32_t s_in[kMergeTile];
  __shared__ uint32_t s_out[kMergeTile];
  const uint64_t off = keep_high ? m : 0;
  const uint64_t c = blockIdx.x;
  const uint64_t o0 = c * kMergeTile;
  const uint64_t o1 = (o0 + kMergeTile < m) ? o0 + kMergeTile : m;
  const uint64_t d0 = off + o0, d1 = off + o1;
  const uint64_t i0 = coranks[c], i1 = coranks[c + 1];
  const uint64_t j0 = d0 - i0, j1 = d1 - i1;
  const int la = (int)(i1 - i0), lb = (int)(j1 - j0), L = la + lb;

  for (int x = threadIdx.x; x < la; x += kMergeThreads) s_in[x] = A[i0 + x] ^ kx;
  for (int x = threadIdx.x; x < lb; x += kMergeThreads) s_in[la + x] = B[j0 + x] ^ kx;
  __syncthreads();

  const uint32_t* sA = s_in;
  const uint32_t* sB = s_in + la;
  int dt = threadIdx.x * kMergeItems;
  if (dt > L) dt = L;
  // corank of dt inside the tile
  int lo = dt > lb ? dt - lb : 0;
  int hi = dt < la ? dt : la;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (sA[mid] <= sB[dt - mid - 1]) lo = mid + 1;
    else hi = mid;
  }
  int i = lo, j = dt - lo;
#pragma unroll
  for (int q = 0; q < kMergeItems; ++q) {
    const int o = dt + q;
    if (o < L) {
      const bool takeA = (j >= lb) || (i < la && sA[i] <= sB[j]);
      s_out[o] = takeA ? sA[i] : sB[j];
      i += takeA ? 1 : 0;
      j += takeA ? 0 : 1;
    }
  }
  __syncthreads();
  for (int x = threadIdx.x; x < L; x += kMergeThreads) out[o0 + x] = s_out[x] ^ kx;
}

}  // namespace b200
