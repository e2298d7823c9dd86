// bitonic_tma.cuh -- tile sort whose load is one TMA tensor copy.
//
// The tile sort's first round holds local bits 0..4 in registers with thread
// t owning row t of the tile (keys 32t .. 32t+31, bitonic_rounds.cuh
// Layout<C, 0x1F>).  Instead of the staged load (LDG.128 -> STS into padded
// shared memory -> barrier -> LDS), one elected thread issues a single
// cp.async.bulk.tensor copy of the whole 2^C-key tile (2^(C-5) rows of 128
// bytes) into shared memory with the 128-byte swizzle (16-byte chunk c of
// row r lands at chunk c ^ (r & 7)), the CTA waits on an mbarrier, and every
// thread reads its row with eight conflict-free LDS.128 (a quarter warp's
// eight rows hit eight different chunk positions).  The rest of the pass is
// the ordinary round engine; the swizzled buffer is then reused as the
// padded round buffer.  Reference: run_shared_block's block load,
// engine.cpp:56-70.
#pragma once

#include <cuda.h>

#include "bitonic_static.cuh"

namespace b200 {

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  const uint32_t a = (uint32_t)__cvta_generic_to_shared(bar);
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  const uint32_t a = (uint32_t)__cvta_generic_to_shared(bar);
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(a), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t a = (uint32_t)__cvta_generic_to_shared(bar);
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(a),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d(uint32_t* dst, const CUtensorMap* map, int c0, int c1,
                                            uint64_t* bar) {
  const uint32_t d = (uint32_t)__cvta_generic_to_shared(dst);
  const uint32_t b = (uint32_t)__cvta_generic_to_shared(bar);
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(d),
      "l"(map), "r"(c0), "r"(c1), "r"(b)
      : "memory");
}
__device__ __forceinline__ uint4 lds128(const uint32_t* p) {
  uint4 v;
  const uint32_t a = (uint32_t)__cvta_generic_to_shared(p);
  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "r"(a));
  return v;
}

// Layout whose thread bits are local bits 5, 6, ... in order: thread t owns
// the 32 keys of row t.
template <class L>
constexpr bool row_layout() {
  for (int i = 0; i < L::NT; ++i)
    if (L::tpos(i) != 5 + i) return false;
  return true;
}

// 2^C-key tiles, C in [8, 13] (one box of 2^(C-5) <= 256 rows).
template <int C, int R = reg_bits(C)>
__global__ void __launch_bounds__(threads_for<C, R>(), min_blocks_for<C, R>())
tile_sort_tma_kernel(PassParams P, const __grid_constant__ CUtensorMap map) {
  static_assert(C >= 8 && C <= 13 && R == 5, "TMA tile sort: 2^8..2^13 keys, 32 per thread");
  extern __shared__ __align__(16) uint8_t smem_raw[];
  __shared__ uint64_t bar;
  // the 128-byte swizzle pattern repeats every 1024 bytes of the SHARED
  // address: align the box to that in the shared window
  const uint32_t s0 = (uint32_t)__cvta_generic_to_shared(smem_raw);
  uint32_t* sm = reinterpret_cast<uint32_t*>(smem_raw + (((s0 + 1023u) & ~1023u) - s0));
  using B = PassBody<C, 0, -1, -1, R, 0>;
  static_assert(B::RD::mask(0) == 0x1Fu && row_layout<typename B::template L<0>>(),
                "TMA tile sort: round 0 must hold local bits 0..4, thread t = row t");
  typename B::Ctx c;
  c.keys = P.keys;
  c.vals = P.vals;
  const uint64_t blk = pass_block(P);
  c.gbase = blk << C;
  c.y = C;
  c.uA = c.uB = 0u;
  c.uC = 0u - dir_bit_global(c.gbase, C, P.kd);
  c.gin = P.gmask_in;
  c.gout = P.gmask_out;
  c.gin_lo = c.gout_lo = 0u;
  c.fs = FmaSplit{P.one, P.mone};
  constexpr int ROWS = 1 << (C - 5);
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  pdl_wait();
  if (threadIdx.x == 0) {
    mbar_expect_tx(&bar, (uint32_t)(ROWS * 128));
    tma_load_2d(sm, &map, 0, (int)(blk * ROWS), &bar);
  }
  mbar_wait(&bar, 0);
  uint32_t v[32];
  uint32_t w[32];
  {
    // round-0 layout: registers = local bits 0..4, thread t = row t
    const uint32_t t = threadIdx.x;
    const uint32_t* row = sm + t * 32;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const uint4 x = lds128(row + ((q ^ (t & 7)) << 2));
      v[4 * q + 0] = x.x ^ c.gin;
      v[4 * q + 1] = x.y ^ c.gin;
      v[4 * q + 2] = x.z ^ c.gin;
      v[4 * q + 3] = x.w ^ c.gin;
    }
  }
  __syncthreads();  // the swizzled tile becomes the padded round buffer
  B::template rounds<0>(c, sm, v, w);
  B::tail(c, v, w);
  B::store(c, sm, v, w);
  pdl_trigger();
}

}  // namespace b200
