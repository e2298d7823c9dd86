// merge_split.cuh -- merge path kernels: merge-split of two sorted shards (the
// compare-exchange of the rank-level bitonic network in the partitioned
// sort) and a general two-way merge.
//
// The reference has no multi-device path; north_star adds one:
// each rank sorts its contiguous shard (work_slice rule, worker_pool.hpp:
// 22-25), then every CE of a bitonic network over the G shards is replaced by
// a merge-split: the lower rank of an ascending pair keeps the m smallest
// keys of the 2m union, the upper rank the m largest (block 0-1 principle).
//
// Both operations are "output window [o_begin, o_begin + o_len) of
// merge(A[0..la), B[0..lb))".  merge_partition_kernel finds, for every
// 2048-key output tile, how many keys come from A (binary search on the
// diagonal of the virtual merge, A first on ties); merge_tile_kernel stages
// the two input windows in shared memory, each thread finds its own 8-key
// sub-diagonal, merges serially and the CTA writes the tile back coalesced.
// A or B may be a peer-device pointer: each CTA then reads only the part of
// the partner shard that lands in its output tile, over NVLink, inside the
// kernel (the exchange is fused into the merge and moves ~m/2 keys).
#pragma once

#include <cstdint>

#include "merge_consts.hpp"

namespace b200 {


// Number of keys of A among the first d keys of merge(A, B) (A first on ties).
__device__ __forceinline__ uint64_t corank_global(uint64_t d, const uint32_t* A,
                                                  uint64_t la, const uint32_t* B,
                                                  uint64_t lb, uint32_t kx) {
  uint64_t lo = d > lb ? d - lb : 0;
  uint64_t hi = d < la ? d : la;
  while (lo < hi) {
    const uint64_t mid = (lo + hi) >> 1;
    if ((A[mid] ^ kx) <= (B[d - mid - 1] ^ kx)) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

__global__ void merge_partition_kernel(const uint32_t* __restrict__ A, uint64_t la,
                                       const uint32_t* __restrict__ B, uint64_t lb,
                                       uint64_t o_begin, uint64_t o_len, uint32_t kx,
                                       uint64_t* __restrict__ coranks, uint64_t nb) {
  const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nb) return;
  uint64_t d = t * kMergeTile;
  if (d > o_len) d = o_len;
  coranks[t] = corank_global(o_begin + d, A, la, B, lb, kx);
}

__global__ void __launch_bounds__(kMergeThreads)
merge_tile_kernel(const uint32_t* __restrict__ A, uint64_t la,
                  const uint32_t* __restrict__ B, uint64_t lb, uint64_t o_begin,
                  uint64_t o_len, uint32_t kx, const uint64_t* __restrict__ coranks,
                  uint32_t* __restrict__ out) {
  __shared__ uint32_t s_in[kMergeTile];
  __shared__ uint32_t s_out[kMergeTile];
  const uint64_t c = blockIdx.x;
  const uint64_t o0 = c * kMergeTile;
  const uint64_t o1 = (o0 + kMergeTile < o_len) ? o0 + kMergeTile : o_len;
  const uint64_t d0 = o_begin + o0, d1 = o_begin + o1;
  const uint64_t i0 = coranks[c], i1 = coranks[c + 1];
  const uint64_t j0 = d0 - i0, j1 = d1 - i1;
  const int na = (int)(i1 - i0), nbk = (int)(j1 - j0), L = na + nbk;

  for (int x = threadIdx.x; x < na; x += kMergeThreads) s_in[x] = A[i0 + x] ^ kx;
  for (int x = threadIdx.x; x < nbk; x += kMergeThreads) s_in[na + x] = B[j0 + x] ^ kx;
  __syncthreads();

  const uint32_t* sA = s_in;
  const uint32_t* sB = s_in + na;
  int dt = threadIdx.x * kMergeItems;
  if (dt > L) dt = L;
  int lo = dt > nbk ? dt - nbk : 0;
  int hi = dt < na ? dt : na;
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
      const bool takeA = (j >= nbk) || (i < na && sA[i] <= sB[j]);
      s_out[o] = takeA ? sA[i] : sB[j];
      i += takeA ? 1 : 0;
      j += takeA ? 0 : 1;
    }
  }
  __syncthreads();
  for (int x = threadIdx.x; x < L; x += kMergeThreads) out[o0 + x] = s_out[x] ^ kx;
}

}  // namespace b200
