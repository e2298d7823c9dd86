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
// 8192-key output tile, how many keys come from A (binary search on the
// diagonal of the virtual merge, A first on ties); merge_bitonic_kernel
// stages the tile's two input windows (B reversed) in shared memory and
// sorts the resulting bitonic sequence with the last phase of the network.
// A or B may be a peer-device pointer: each CTA then reads only the part of
// the partner shard that lands in its output tile, over NVLink, inside the
// kernel (the exchange is fused into the merge and moves ~m/2 keys).
#pragma once

#include <cstdint>

#include "bitonic_static.cuh"
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

// One thread per output-tile boundary: binary search on the diagonal.  (A
// 33-ary warp search -- 32 lanes probing at once -- cut the dependent loads
// from 29 to 6 at 2^29 keys but read ~8x more DRAM sectors; measured
// slower on B200 at every size from 2^24 up.)
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

// One output tile per CTA, merged as a bitonic sequence: the tile's A window
// (ascending) followed by its B window reversed is a bitonic sequence of
// kMergeTile = 2^kMergeC keys for ANY split na + nb, so the last phase of
// the network -- steps on local bits kMergeC-1..0, all ascending -- sorts
// it.  That phase runs on the round engine of the sort passes
// (bitonic_static.cuh: registers + conflict-free padded shared memory), so
// the merge has no data-dependent shared-memory traffic (the serial
// per-thread merge it replaced was bank-conflict bound: 2.3-2.6 TB/s on a
// 2^29-key merge-split).  A partial last tile is padded with the order's
// maximum between the two runs (keeping it bitonic); the padding sorts to
// the end and is not stored.
//
// (.nc measured faster than .lu here: 2^28 merge-path sort 7.8 vs 8.5 ms)
#ifndef B200_MP_LD
#define B200_MP_LD ".nc"
#endif
// Register e of round 0 (slot offset D = dep_reg(e) from the thread's slot):
// A[tj + D] when D < room, else B[-(tj + D)] -- D is a compile-time immediate.
template <int D>
__device__ __forceinline__ uint32_t ld_split(const uint32_t* ta, const uint32_t* tb, int room) {
  uint32_t x;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.gt.s32 p, %1, %4;\n\t"
      "@p ld.global" B200_MP_LD ".u32 %0, [%2+%5];\n\t"
      "@!p ld.global" B200_MP_LD ".u32 %0, [%3+%6];\n\t}"
      : "=r"(x)
      : "r"(room), "l"(ta), "l"(tb), "n"(D), "n"(4 * D), "n"(-4 * D));
  return x;
}

//
// merge_tile: the body, for one output tile o[0..L) = keys i0..i1 of A and
// keys j1-(L-(i1-i0)) .. j1 of B (both in the order kx selects).
template <class L0, int NR, int E = 0>
__device__ __forceinline__ void load_full_regs(const uint32_t* ta, const uint32_t* tb, int room,
                                               uint32_t kx, uint32_t (&v)[NR]) {
  if constexpr (E < NR) {
    v[E] = ld_split<(int)L0::dep_reg(E)>(ta, tb, room) ^ kx;
    load_full_regs<L0, NR, E + 1>(ta, tb, room, kx, v);
  }
}

template <int C, int R>
__device__ __forceinline__ void merge_tile(const uint32_t* __restrict__ A,
                                           const uint32_t* __restrict__ B, uint64_t i0,
                                           uint64_t i1, uint64_t j1, int L, uint32_t kx,
                                           uint32_t* __restrict__ o, uint32_t one,
                                           uint32_t mone, uint32_t* smem) {
  using Body = PassBody<C, 1, C - 1, -1, R, 0>;
  constexpr int T = threads_for<C, R>();
  constexpr int N = 1 << C;
  const uint64_t o0 = 0;
  uint32_t* const out = o;
  const int na = (int)(i1 - i0);
  // Slot j of the tile: A[i0 + j] for j < na (ascending), the maximum for
  // the padding, B backwards in the last nb slots (descending): ascending,
  // flat, descending is bitonic.
  typename Body::Ctx cx;
  cx.keys = out;
  cx.vals = nullptr;
  cx.gbase = o0;
  cx.y = C;
  cx.uA = cx.uB = cx.uC = 0u;  // one ascending phase, no direction bit
  cx.gin = cx.gout = cx.gin_lo = cx.gout_lo = 0u;
  cx.fs = FmaSplit{one, mone};
  using L0 = typename Body::template L<0>;
  uint32_t v[1 << R];
  uint32_t w[1 << R];
  if constexpr (Body::template direct_ok<L0>()) {
    // Round 0's lanes own 32 consecutive slots: each register is one
    // coalesced (possibly misaligned) warp load straight from A or B into
    // the first round's layout -- no staging copy, no barrier.
    const int nbk = L - na;
    const uint32_t* pa = A + i0;                    // slot j < na        -> pa[j]
    const uint32_t* pb = B + (j1 - 1) + (N - nbk);  // slot j >= N - nbk -> pb[-j]
    const uint32_t tj = L0::thread_j();
    static_assert(L0::tpos(0) == 0 && L0::tpos(4) == 4, "round 0: lanes on local bits 0..4");
    if (L == N) {
      // Full tile (every merge-path phase tile): no padding, slot j is A[i0+j]
      // below na, else B backwards.  Per register one compare against an
      // immediate and two predicated loads with immediate offsets from two
      // per-thread bases (3 instructions; no per-register address math).
      const uint32_t* ta = pa + tj;
      const uint32_t* tb = pb - tj;
      const int room = na - (int)tj;  // slot tj + d is in A iff d < room
      load_full_regs<L0, (1 << R)>(ta, tb, room, kx, v);
    } else {
    const int lane = (int)(tj & 31u);
    const uint32_t wbase = tj & ~31u;  // the warp's part of the slot index
#pragma unroll
    for (int e = 0; e < (1 << R); ++e) {
      // a register's 32 slots are consecutive: classify the chunk once per
      // warp (uniform branches); only the <= 2 chunks that straddle a window
      // edge select per lane
      const int J = (int)(wbase | L0::dep_reg(e));
      const int j = J + lane;
      uint32_t x;
      if (J + 32 <= na) {
        x = __ldg(pa + j);
      } else if (J >= N - nbk) {
        x = __ldg(pb - j);
      } else {
        x = j < na ? __ldg(pa + j) : (j >= N - nbk ? __ldg(pb - j) : ~kx);
      }
      v[e] = x ^ kx;
    }
    }
  } else {
  {
      // 16-byte loads on the aligned interior of both windows (the edges, at
      // most 3 + 3 keys per window, and the padding are stored separately).
      // Chunk u of the concatenated chunk list is A chunk u or B chunk u-nA4;
      // each thread issues all its chunk loads before any store.
      const int nbk = L - na;
      const uint64_t j0 = j1 - (uint64_t)nbk;
      const uint64_t a0 = (i0 + 3) & ~uint64_t{3}, a1e = i1 & ~uint64_t{3};
      const uint64_t b0 = (j0 + 3) & ~uint64_t{3}, b1e = j1 & ~uint64_t{3};
      const bool va = ((reinterpret_cast<uintptr_t>(A) & 15u) == 0) && a1e > a0 && a0 <= i1;
      const bool vb = ((reinterpret_cast<uintptr_t>(B) & 15u) == 0) && b1e > b0 && b0 <= j1;
      const int nA4 = va ? (int)((a1e - a0) >> 2) : 0;
      const int nB4 = vb ? (int)((b1e - b0) >> 2) : 0;
      constexpr int Q = N / 4 / T;  // chunk slots per thread
      uint4 x[Q];
  #pragma unroll
      for (int q = 0; q < Q; ++q) {
        const int u = threadIdx.x + q * T;
        const uint4* src = u < nA4 ? reinterpret_cast<const uint4*>(A + a0) + u
                                   : reinterpret_cast<const uint4*>(B + b0) + (u - nA4);
        if (u < nA4 + nB4) x[q] = __ldg(src);
      }
  #pragma unroll
      for (int q = 0; q < Q; ++q) {
        const int u = threadIdx.x + q * T;
        if (u < nA4) {
          const uint32_t j = (uint32_t)(a0 - i0) + 4u * (uint32_t)u;  // A slot
          smem[smem_pad(j)] = x[q].x ^ kx;
          smem[smem_pad(j + 1)] = x[q].y ^ kx;
          smem[smem_pad(j + 2)] = x[q].z ^ kx;
          smem[smem_pad(j + 3)] = x[q].w ^ kx;
        } else if (u < nA4 + nB4) {
          // B[g] -> slot N - 1 - (g - j0)
          const uint32_t j = (uint32_t)(N - 1) - (uint32_t)(b0 - j0) - 4u * (uint32_t)(u - nA4);
          smem[smem_pad(j)] = x[q].x ^ kx;
          smem[smem_pad(j - 1)] = x[q].y ^ kx;
          smem[smem_pad(j - 2)] = x[q].z ^ kx;
          smem[smem_pad(j - 3)] = x[q].w ^ kx;
        }
      }
      // edges (keys outside the 16-byte interiors) and padding
      const uint64_t ea0 = va ? a0 : i1, ea1 = va ? a1e : i1;  // A interior [ea0, ea1)
      const uint64_t eb0 = vb ? b0 : j1, eb1 = vb ? b1e : j1;
      for (uint64_t g = i0 + threadIdx.x; g < ea0; g += T) smem[smem_pad((uint32_t)(g - i0))] = A[g] ^ kx;
      for (uint64_t g = ea1 + threadIdx.x; g < i1; g += T) smem[smem_pad((uint32_t)(g - i0))] = A[g] ^ kx;
      for (uint64_t g = j0 + threadIdx.x; g < eb0; g += T)
        smem[smem_pad((uint32_t)(N - 1) - (uint32_t)(g - j0))] = B[g] ^ kx;
      for (uint64_t g = eb1 + threadIdx.x; g < j1; g += T)
        smem[smem_pad((uint32_t)(N - 1) - (uint32_t)(g - j0))] = B[g] ^ kx;
      for (int j = na + threadIdx.x; j < N - nbk; j += T) smem[smem_pad((uint32_t)j)] = 0xFFFFFFFFu;
    }
    __syncthreads();
    L0::lds(smem, v);
  }
  Body::template rounds<0>(cx, smem, v, w);
  Body::tail(cx, v, w);
  using LL = typename Body::template L<Body::NRE - 1>;
  if constexpr (Body::template direct_ok<LL>()) {
    // The last round's lanes own consecutive vectors (64 keys per thread:
    // rounds {12..7}, {6..1}, {0}+fillers): coalesced stores straight from
    // registers, one shared-memory round trip fewer than the transpose below.
    if (L == N && (reinterpret_cast<uintptr_t>(o) & 15u) == 0) {
      cx.gout = kx;
      Body::store(cx, smem, v, w);
      return;
    }
  }
  // (A direct 16-byte store from a layout whose lanes sit 32 bytes apart --
  // half a sector per instruction -- measured 518 vs 394 us per 2^28-key
  // phase: L1/LSU-bound.  The shared-memory transpose keeps every store a
  // full 512-byte warp line.)
  LL::sts(smem, v);
  __syncthreads();
  if (L == N && (reinterpret_cast<uintptr_t>(o) & 15u) == 0) {
#pragma unroll 4
    for (int q = threadIdx.x; q < N / 4; q += T) {
      const uint32_t p = smem_pad(4u * q);
      reinterpret_cast<uint4*>(o)[q] =
          make_uint4(smem[p] ^ kx, smem[p + 1] ^ kx, smem[p + 2] ^ kx, smem[p + 3] ^ kx);
    }
  } else {
    for (int j = threadIdx.x; j < L; j += T) o[j] = smem[smem_pad((uint32_t)j)] ^ kx;
  }
}

template <int C = kMergeC, int R = 5>
__global__ void __launch_bounds__(threads_for<C, R>(), min_blocks_for<C, R>())
merge_bitonic_kernel(const uint32_t* __restrict__ A, const uint32_t* __restrict__ B,
                     uint64_t o_begin, uint64_t o_len, uint32_t kx,
                     const uint64_t* __restrict__ coranks, uint32_t* __restrict__ out,
                     uint32_t one, uint32_t mone) {
  constexpr int N = 1 << C;
  extern __shared__ uint32_t smem[];
  const uint64_t c = blockIdx.x;
  const uint64_t o0 = c * (uint64_t)N;
  const uint64_t o1 = (o0 + N < o_len) ? o0 + N : o_len;
  const uint64_t i0 = coranks[c], i1 = coranks[c + 1];
  merge_tile<C, R>(A, B, i0, i1, o_begin + o1 - i1, (int)(o1 - o0), kx, out + o0, one, mone,
                   smem);
}

// ---- merge-path phases (the "mergepath" sort variant) --------------------------
// Phase p of a sort whose 2^(p-1)-key runs are all ascending (in the order kx
// selects): the bitonic merger of each run pair, with its p-C large-stride
// half-cleaner steps replaced by a co-rank partition -- every 2^C-key output
// tile holds exactly the keys of ranks [t 2^C, (t+1) 2^C) of the pair's merge,
// which is what the half-cleaners route to it -- and its last C steps run by
// merge_tile.  One HBM round trip per phase; src -> dst (out of place).
// Tiles never straddle a pair (2^p >= 2^(C+1)).
template <int WB = kMergeC>
__global__ void mergepath_partition_kernel(const uint32_t* __restrict__ src, int p, uint32_t kx,
                                           uint64_t* __restrict__ coranks, uint64_t ntiles) {
  const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  pdl_wait();  // the previous phase's output (PDL launch; no-op otherwise)
  pdl_trigger();
  if (t >= ntiles) return;
  const uint64_t half = uint64_t{1} << (p - 1);
  const uint64_t o = t << WB;
  const uint64_t base = o & ~((half << 1) - 1);
  const uint64_t d = o - base;
  if (d == 0) {
    coranks[t] = 0;
    return;
  }
  // (a 4-ary search -- three independent probes per level, 14 instead of 27
  // dependent levels at 2^28 -- measured slower: 19-40 vs 13-33 us per
  // phase; the extra probe sectors cost more than the saved round trips)
  coranks[t] = corank_global(d, src + base, half, src + base + half, half, kx);
}

// (capping the 64-key variant at 80 registers for six CTAs per SM measured
// slower than 86 registers and five: 2^28 8.00 vs 7.39 ms)
#ifndef B200_MP_MINB6
#define B200_MP_MINB6 4
#endif
template <int C = kMergeC, int R = 5>
__global__ void __launch_bounds__(threads_for<C, R>(), (R == 6 && C == 13) ? B200_MP_MINB6 : min_blocks_for<C, R>())
mergepath_merge_kernel(const uint32_t* __restrict__ src, uint32_t* __restrict__ dst, int p,
                       uint32_t kx, const uint64_t* __restrict__ coranks, uint32_t one,
                       uint32_t mone) {
  constexpr int N = 1 << C;
  extern __shared__ uint32_t smem[];
  const uint64_t t = blockIdx.x;
  const uint64_t half = uint64_t{1} << (p - 1);
  const uint64_t o = t * (uint64_t)N;
  const uint64_t base = o & ~((half << 1) - 1);
  const uint64_t d = o - base;  // the tile's first rank in its pair's merge
  pdl_wait();  // the partition's coranks (PDL launch; no-op otherwise)
  const uint64_t i0 = coranks[t];
  const uint64_t i1 = (d + N == (half << 1)) ? half : coranks[t + 1];
  merge_tile<C, R>(src + base, src + base + half, i0, i1, d + N - i1, N, kx, dst + o, one, mone,
                   smem);
  pdl_trigger();
}

}  // namespace b200
