// bitonic_cluster.cuh -- merge passes on 2^15-key cosets held by a CTA pair.
//
// One SM holds at most a 2^14-key coset at the occupancy the HBM-bound merge
// passes need, and a pass covers at most as many network steps as its coset
// has bits.  A thread-block cluster of two CTAs (on two SMs) jointly owns a
// 2^15-key coset S = [0, b+1) U [y, y+h), h = 14 - b, and runs the tail of
// phase p (bits b..0) fused with the head of phase p+1 (bits p..p-h+1): 15
// steps per HBM round trip instead of 14, which removes ~4 of the 29 passes
// of a 2^28-key sort (planner.hpp).
//
// At any moment each CTA holds the half of S with one coset bit fixed to its
// cluster rank c (the "cluster bit"):
//   part 1 (tail, bits b..0)  -- cluster bit = the coset's top bit (global bit
//           y+h-1 = p, which is also phase p's direction bit, so the tail's
//           direction is CTA-uniform);
//   exchange -- keys move through distributed shared memory so that the
//           cluster bit becomes b (a tail bit, done);
//   part 2 (head, bits 14..b+1 of S) -- on the sub-coset [0,b) U [y,y+h).
// Each part is an ordinary 2^14-key pass body (bitonic_static.cuh); the
// exchange replaces the HBM store + load between the two equivalent 14-bit
// passes: every key is written once to its own CTA's padded shared memory,
// and the first round of part 2 reads half of its registers from the peer
// CTA (ld.shared::cluster), the other half locally.
//
// Reference: the pass fuses steps of the network like the reference's
// register-paired / shared launches (engine.cpp:40-70, :229-246); its
// build_plan (engine.cpp:86-145) never crosses a phase boundary.
#pragma once

#include "bitonic_static.cuh"

namespace b200 {

__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t cluster_id_x() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(r));
  return r;
}
// shared::cluster address of `p` (a shared-memory pointer) in CTA `rank`
__device__ __forceinline__ uint32_t cluster_map(const void* p, uint32_t rank) {
  uint32_t a = (uint32_t)__cvta_generic_to_shared(p), r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
  return r;
}
__device__ __forceinline__ uint32_t ld_cluster(uint32_t addr) {
  uint32_t v;
  asm volatile("ld.shared::cluster.u32 %0, [%1];" : "=r"(v) : "r"(addr) : "memory");
  return v;
}
__device__ __forceinline__ void cluster_arrive() {
  asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_wait() {
  asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// 14-bit part-2 index j' -> part-1 index j of the same key (drops coset bit
// 14, the old cluster bit, and re-inserts coset bit b = 0): j' bits [0,b)
// stay, j' bits [b,13) move up by one.  Additive over disjoint bit fields.
template <int B>
__host__ __device__ constexpr uint32_t xmap(uint32_t jp) {
  return (jp & ((1u << B) - 1u)) | (((jp >> B) & ((1u << (13 - B)) - 1u)) << (B + 1));
}

template <int B, int R>
struct ClusterPass {
  static constexpr int C = 14;  // keys per CTA = 2^14
  // part 1: tail bits B..0 on [0, B+1) U [y, y+13-B)   (cluster bit y+13-B)
  using B1 = PassBody<C, 1, B, -1, R, 0, B + 1>;
  // part 2: head bits 13..B on [0, B) U [y, y+14-B)     (cluster bit B)
  using B2 = PassBody<C, 1, -1, B, R, 0, B>;
  static constexpr int NR = 1 << R;
  static_assert(B >= 2 && B <= 13, "cluster pass: tail top bit out of range");

  // Part 2's first layout, filled from both CTAs' shared memory.
  __device__ __forceinline__ static void exchange_load(const uint32_t* sm, uint32_t c,
                                                       uint32_t (&v)[NR]) {
    using L = typename B2::template L<0>;
    const uint32_t tj = L::thread_j();
    const uint32_t own = (tj >> 13) & 1u;  // owner CTA when bit 13 is a thread bit
    const uint32_t base_self = cluster_map(sm, c);
    const uint32_t base_peer = cluster_map(sm, c ^ 1u);
    const uint32_t toff = 4u * (smem_pad(xmap<B>(tj & 0x1FFFu)) + smem_pad(c << B));
#pragma unroll
    for (int e = 0; e < NR; ++e) {
      const uint32_t d = L::dep_reg(e);
      const uint32_t owner = own ^ ((d >> 13) & 1u);
      const uint32_t base = (owner == c) ? base_self : base_peer;
      v[e] = ld_cluster(base + toff + 4u * smem_pad(xmap<B>(d & 0x1FFFu)));
    }
  }

  __device__ __forceinline__ static void run(const PassParams& P, uint32_t* sm) {
    const uint32_t c = cluster_ctarank();
    const uint64_t cid = cluster_id_x();
    const int y = P.y;
    constexpr int A15 = B + 1;
    // base of the cluster's 15-bit coset [0, B+1) U [y, y+14-B)
    const uint64_t base15 = Coset<15, A15>::base(cid, y);
    typename B1::Ctx c1;
    c1.keys = P.keys;
    c1.vals = nullptr;
    c1.y = y;
    c1.gbase = base15 + ((uint64_t)c << (y + 13 - B));
    // phase pA's direction bit is global bit pA = y+13-B = the cluster bit
    c1.uA = P.pA >= P.kd ? 0u : 0u - c;
    c1.uB = 0u;
    c1.uC = 0u;
    c1.gin = 0u;
    c1.gout = 0u;
    c1.gin_lo = c1.gout_lo = 0u;
    c1.fs = FmaSplit{P.one, P.mone};
    typename B2::Ctx c2;
    c2.keys = P.keys;
    c2.vals = nullptr;
    c2.y = y;
    c2.gbase = base15 + ((uint64_t)c << B);
    c2.uA = 0u;
    c2.uC = 0u;
    c2.gin = 0u;
    c2.gin_lo = 0u;
    c2.fs = c1.fs;
    c2.uB = 0u - dir_bit_global(base15, P.pB, P.kd);
    c2.gout = P.gmask_out;
    c2.gout_lo = P.gmask_out_lo;

    uint32_t v[NR];
    uint32_t w[NR];
    pdl_wait();
    B1::load(c1, sm, v, w);
    B1::template rounds<0>(c1, sm, v, w);
    B1::tail(c1, v, w);
    // leave phase A's domain, enter phase B's (both CTA-uniform; phase B's is
    // the same in both CTAs, so the peer's keys arrive in the right domain)
    using LL = typename B1::template L<B1::NRE - 1>;
    const uint32_t m = c1.uA ^ c2.uB;
#pragma unroll
    for (int e = 0; e < NR; ++e) v[e] ^= m;
    jitter(5);
    LL::sts(sm, v);
    cluster_arrive();  // this CTA's keys are in its shared memory ...
    cluster_wait();    // ... and so are the peer's
    jitter(6);
    exchange_load(sm, c, v);
    cluster_arrive();  // done reading both CTAs' shared memory
    B2::template steps<0, B2::RD::begin(0)>(c2, v, w);
    cluster_wait();    // the peer has read ours: shared memory may be reused
    jitter(7);
    B2::template rounds<1>(c2, sm, v, w);
    B2::tail(c2, v, w);
    B2::store(c2, sm, v, w);
    pdl_trigger();
  }
};

template <int B, int R = 5>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(threads_for<14, R>(), min_blocks_for<14, R>())
cluster_merge_kernel(PassParams P) {
  extern __shared__ uint32_t smem[];
  ClusterPass<B, R>::run(P, smem);
}

}  // namespace b200
