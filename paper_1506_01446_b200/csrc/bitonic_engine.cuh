// bitonic_engine.cuh -- the sm_100a bitonic-network engine.
//
// One CTA owns a "coset" of 2^C keys of the global array: the keys whose
// global index varies only in a set S of C bit positions.  S is always
//   S = [0, a)  U  [y, y + C - a)
// i.e. a run of 2^a contiguous keys (coalesced HBM access, a >= 2) repeated
// 2^(C-a) times at global stride 2^y.  Inside the CTA the coset is addressed
// by a C-bit LOCAL index j; every compare-exchange (CE) of the network that
// falls inside the pass is a CE on one local bit.  The reference runs the same
// network one step (run_global_step, engine.cpp:31-38), two steps
// (register_paired_kernel, engine.cpp:229-246) or one block-local phase tail
// (run_shared_block, engine.cpp:56-70) per launch; here one launch runs every
// step whose bit lies in S -- the whole first C phases (tile sort), or the
// tail of phase p plus the head of phase p+1 (fused merge pass).
//
// Data path inside the CTA (keys never leave the SM between steps):
//   * registers: each thread holds NR = 2^R (R = 5) keys.  In layout L_z the
//     thread's keys are the 32 local indices with local bits [z, z+5) = the
//     register index e, so a CE on a local bit in [z, z+5) is a pure
//     register min/max (VIMNMX) with no data movement.
//   * shared memory: a layout change is one STS of the 32 registers, one
//     __syncthreads and one LDS in the new layout.  Addresses are padded by one
//     word per 32 (pad(j) = j + j/32), which makes every layout used here
//     bank-conflict free AND keeps every register's address an immediate
//     offset from a per-thread base (the padding map is additive over the
//     disjoint thread/register bit fields).
//
// Direction handling (no per-CE select).  The reference decides each CE's
// direction from bit p (the phase) of the lower index: ascending iff
// (i & 2^p) == 0 (engine.cpp:36, schedule.cpp:333).  Here keys are held in
// the "phase domain" v = u ^ D_p(i) with D_p(i) = -(bit p of i) (all ones for
// descending blocks).  In that domain every CE of phase p is ascending: for
// a descending pair both keys are complemented and min on complements is
// max on the keys.  Moving from phase p to p+1 XORs each key with
// D_p ^ D_{p+1} -- at most one XOR per key per phase, done in layout L_0
// where both bits are per-thread uniform.  The overall key order is folded in
// the same way: u = x ^ gmask with gmask = 0x80000000 for signed int32 keys
// (u32 order of x^0x80000000 == i32 order of x) and ~0 for descending output.
#pragma once

#include <cstdint>

namespace b200 {

constexpr int kRegBits = 5;
constexpr int kMaxTileBits = 15;

__host__ __device__ constexpr int reg_bits(int C) {
  return C < kRegBits ? C : kRegBits;
}
// Shared-memory padding: pad(j) = j + j/32 + j/1024.  Additive over
// disjoint bit fields (so register addresses are immediates), and for any 5
// lane bits with distinct residues mod 5 the 32 lanes hit 32 distinct banks.
__host__ __device__ constexpr uint32_t smem_pad(uint32_t j) {
  return j + (j >> 5) + (j >> 10);
}
// Padded shared-memory words for a 2^C tile.
__host__ __device__ constexpr int tile_smem_words(int C) {
  return (int)smem_pad((1u << C) - 1u) + 1;
}
__host__ __device__ constexpr int tile_threads(int C) {
  return 1 << (C - reg_bits(C));
}

// Runtime description of one pass (one kernel launch).  Built on the host by
// the planner (planner.cpp) and passed by value.
struct PassParams {
  uint32_t* keys;     // whole array (all batches), in place
  uint32_t* vals;     // payloads moved with the keys (key-value kernels only)
  uint32_t gmask_in;  // XOR applied at load  (key order transform, first pass)
  uint32_t gmask_out; // XOR applied at store (inverse transform, last pass)
  uint32_t gmask_in_lo;   // low-word transforms of 64-bit keys
  uint32_t gmask_out_lo;
  int a;              // local bits [0,a) -> global bits [0,a)
  int y;              // local bits [a,C) -> global bits [y, y+C-a)
  int kd;             // log2 of one sorted array: phase kd has no direction bit
  int tile_sort;      // 1: run phases 1..p_end (first pass); 0: merge pass
  int p_end;          // last phase of a tile-sort pass (min(C, kd))
  // Segment A (tail of a phase): CEs on local bits segA_hi..0, phase pA.
  int segA_hi;        // -1 when absent
  int pA;             // global phase (its direction bit is global bit pA)
  // Segment B (head / middle of a phase): CEs on local bits C-1..segB_lo.
  int segB_lo;        // -1 when absent
  int pB;
  // 1 and 0xFFFFFFFF, opaque to the compiler: operands of the IMAD form of
  // max() that moves part of the compare-exchange work to the FMA pipe
  uint32_t one, mone;
  // Virtual padding (non-power-of-two lengths, *_VIRT kernels): keys at
  // indices >= nreal are virtual; phase p's direction bit is bit p of
  // (index ^ dxor), dxor = nreal - 1.  Ignored by the other kernels.
  uint64_t nreal;
  uint64_t dxor;
  // 1: CTAs take their cosets in reverse order.  Consecutive passes run in
  // opposite directions, so a pass starts on the cosets the previous pass
  // wrote last -- still in L2 when the array is larger than L2.
  int reverse;
  // Tile-sort passes only: store the sorted tiles here instead of in place
  // (nullptr: in place).  The merge-path variant's first pass.
  uint32_t* keys_out;
};

// Coset index of this CTA (see PassParams::reverse).
__device__ __forceinline__ uint64_t pass_block(const PassParams& P) {
  return P.reverse ? (uint64_t)(gridDim.x - 1u - blockIdx.x) : (uint64_t)blockIdx.x;
}

// Operands of the FMA-pipe max (see Layout::mm).
struct FmaSplit {
  uint32_t one, mone;
};

template <int C>
struct Tile {
  static constexpr int R = reg_bits(C);
  static constexpr int NR = 1 << R;       // keys per thread
  static constexpr int T = 1 << (C - R);  // threads per CTA
  static constexpr int N = 1 << C;        // keys per CTA
  // Register-chunk layouts: L_Z0 (local bits 0..4 in registers), L_Z1, L_Z2.
  static constexpr int Z0 = 0;
  static constexpr int Z1 = (C >= 10) ? 5 : ((C > 5) ? C - 5 : 0);
  static constexpr int Z2 = (C > 10) ? C - 5 : Z1;

  // Which layout holds local bit b in registers.
  __device__ __forceinline__ static int chunk_of(int b) {
    if (b < R) return 0;
    if (C <= 10 || b < 10) return 1;
    return 2;
  }

  __device__ __forceinline__ static uint32_t pad(uint32_t j) {
    return smem_pad(j);
  }
  template <int Z>
  __device__ __forceinline__ static uint32_t spread(uint32_t t) {
    return (t & ((1u << Z) - 1u)) | ((t >> Z) << (Z + R));
  }
  template <int Z>
  __device__ __forceinline__ static uint32_t base_addr() {
    return pad(spread<Z>(threadIdx.x));
  }
  template <int Z, int E>
  __device__ __forceinline__ static constexpr uint32_t reg_off() {
    return ((uint32_t)E << Z) + (((uint32_t)E << Z) >> 5);
  }

  // ---- register <-> shared memory in layout L_Z ---------------------------
  template <int Z>
  __device__ __forceinline__ static void sts(uint32_t* sm, const uint32_t (&v)[NR]) {
    const uint32_t b = base_addr<Z>();
#pragma unroll
    for (int e = 0; e < NR; ++e) sm[b + smem_pad((uint32_t)e << Z)] = v[e];
  }
  template <int Z>
  __device__ __forceinline__ static void lds(const uint32_t* sm, uint32_t (&v)[NR]) {
    const uint32_t b = base_addr<Z>();
#pragma unroll
    for (int e = 0; e < NR; ++e) v[e] = sm[b + smem_pad((uint32_t)e << Z)];
  }
  __device__ __forceinline__ static void sts_layout(int L, uint32_t* sm, const uint32_t (&v)[NR]) {
    if (L == 0) sts<Z0>(sm, v);
    else if (L == 1) sts<Z1>(sm, v);
    else sts<Z2>(sm, v);
  }
  __device__ __forceinline__ static void lds_layout(int L, const uint32_t* sm, uint32_t (&v)[NR]) {
    if (L == 0) lds<Z0>(sm, v);
    else if (L == 1) lds<Z1>(sm, v);
    else lds<Z2>(sm, v);
  }

  // ---- compare-exchange on register bit Q (ascending in the phase domain) -
  template <int Q>
  __device__ __forceinline__ static void ce(uint32_t (&v)[NR]) {
#pragma unroll
    for (int e = 0; e < NR; ++e) {
      if (!(e & (1 << Q))) {
        const uint32_t x = v[e], y = v[e | (1 << Q)];
        v[e] = min(x, y);
        v[e | (1 << Q)] = max(x, y);
      }
    }
  }
  // Same, with the direction taken from register bit D (phases p < R of the
  // tile sort, where bit p of the local index is a register bit of L_0).
  template <int Q, int D>
  __device__ __forceinline__ static void ce_dir(uint32_t (&v)[NR]) {
#pragma unroll
    for (int e = 0; e < NR; ++e) {
      if (!(e & (1 << Q))) {
        const uint32_t x = v[e], y = v[e | (1 << Q)];
        const bool desc = (D < R) && ((e >> D) & 1);
        v[e] = desc ? max(x, y) : min(x, y);
        v[e | (1 << Q)] = desc ? min(x, y) : max(x, y);
      }
    }
  }
  __device__ __forceinline__ static void ce_q(int q, uint32_t (&v)[NR]) {
    switch (q) {
      case 0: ce<0>(v); break;
      case 1: if constexpr (R > 1) ce<1>(v); break;
      case 2: if constexpr (R > 2) ce<2>(v); break;
      case 3: if constexpr (R > 3) ce<3>(v); break;
      default: if constexpr (R > 4) ce<4>(v); break;
    }
  }
  __device__ __forceinline__ static int z_of(int L) {
    return L == 0 ? Z0 : (L == 1 ? Z1 : Z2);
  }

  // Phases 1..R-1 of the tile sort: every CE and its direction bit are
  // register bits of L_0, so these phases are straight-line min/max code.
  template <int P, int S, bool DIR>
  __device__ __forceinline__ static void reg_phase_steps(uint32_t (&v)[NR]) {
    if constexpr (S >= 0) {
      if constexpr (DIR) ce_dir<S, P>(v);
      else ce<S>(v);
      reg_phase_steps<P, S - 1, DIR>(v);
    }
  }
  // Runs phases P..min(R-1, p_end); phase kd (the array length) has no
  // direction bit (ascending), exactly like merge_span = n in the reference.
  template <int P>
  __device__ __forceinline__ static void reg_phases(uint32_t (&v)[NR], int p_end, int kd) {
    if constexpr (P < R) {
      if (P > p_end) return;
      if (P < kd) reg_phase_steps<P, P - 1, true>(v);
      else reg_phase_steps<P, P - 1, false>(v);
      reg_phases<P + 1>(v, p_end, kd);
    }
  }

  __device__ __forceinline__ static void xor_all(uint32_t (&v)[NR], uint32_t m) {
#pragma unroll
    for (int e = 0; e < NR; ++e) v[e] ^= m;
  }
};

// Programmatic dependent launch: a pass may be launched before the previous
// pass finished (its launch latency overlaps the previous pass's tail); it
// waits here until the previous grid's memory is visible.  No-ops when the
// kernel was launched without the PDL attribute.
__device__ __forceinline__ void pdl_wait() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
}
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// Direction bit (0/1) of global phase p for the key at global index gi.
__device__ __forceinline__ uint32_t dir_bit_global(uint64_t gi, int p, int kd) {
  return p >= kd ? 0u : (uint32_t)((gi >> p) & 1u);
}

template <int C>
__global__ void __launch_bounds__(Tile<C>::T, (Tile<C>::T >= 1024 ? 1 : (1024 / Tile<C>::T > 16 ? 16 : 1024 / Tile<C>::T)))
bitonic_pass_kernel(PassParams P) {
  using TL = Tile<C>;
  constexpr int NR = TL::NR;
  constexpr int T = TL::T;
  constexpr int N = TL::N;
  extern __shared__ uint32_t smem[];
  pdl_wait();

  // ---- global base of this CTA's coset ----------------------------------
  const int a = P.a, y = P.y, h = C - a;
  const uint64_t b = pass_block(P);
  uint64_t gbase;
  if (h == 0 || y == a) {
    gbase = b << C;  // contiguous tile
  } else {
    const int gap = y - a;  // fixed bits between the low run and the high range
    const uint64_t blo = b & ((1ull << gap) - 1ull);
    const uint64_t bhi = b >> gap;
    gbase = (blo << a) | (bhi << (y + h));
  }
  const uint32_t amask = (1u << a) - 1u;
  auto gidx = [&](uint32_t j) -> uint64_t {
    return gbase + (j & amask) + ((uint64_t)(j >> a) << y);
  };

  // Phase-domain entry mask for the first CE segment and exit mask for the
  // last one, as functions of the local index (only used at staging).
  // Merge pass:  entry phase = pA if segment A exists else pB.
  //              its direction bit is local C-1 when it lies in the high
  //              range (tail+head pass), else CTA-uniform.
  int p_first, p_last;
  if (P.tile_sort) {
    p_first = -1;  // tile sort enters the phase domain later (phase R)
    p_last = P.p_end;
  } else {
    p_first = P.segA_hi >= 0 ? P.pA : P.pB;
    p_last = P.segB_lo >= 0 ? P.pB : P.pA;
  }
  // local bit holding global bit p (or -1)
  auto local_of = [&](int p) -> int {
    if (p < a) return p;
    if (p >= y && p < y + h) return a + (p - y);
    return -1;
  };
  auto dmask_at = [&](int p, uint32_t j) -> uint32_t {
    if (p < 0) return 0u;
    const int l = local_of(p);
    uint32_t bit;
    if (l >= 0) bit = (j >> l) & 1u;
    else bit = dir_bit_global(gbase, p, P.kd);
    if (p >= P.kd) bit = 0u;
    return 0u - bit;
  };

  // ---- staging load: coalesced global -> padded shared -----------------
  if constexpr (N / T >= 4) {
    constexpr int IT = N / 4 / T;
    uint4 buf[IT];
#pragma unroll
    for (int it = 0; it < IT; ++it) {
      const uint32_t j = 4u * (uint32_t)(it * T + threadIdx.x);
      buf[it] = *reinterpret_cast<const uint4*>(P.keys + gidx(j));
    }
#pragma unroll
    for (int it = 0; it < IT; ++it) {
      const uint32_t j = 4u * (uint32_t)(it * T + threadIdx.x);
      const uint32_t m = P.gmask_in ^ dmask_at(p_first, j);
      const uint32_t pj = TL::pad(j);
      smem[pj + 0] = buf[it].x ^ m;
      smem[pj + 1] = buf[it].y ^ m;
      smem[pj + 2] = buf[it].z ^ m;
      smem[pj + 3] = buf[it].w ^ m;
    }
  } else {
    for (uint32_t j = threadIdx.x; j < (uint32_t)N; j += T) {
      smem[TL::pad(j)] = P.keys[gidx(j)] ^ P.gmask_in ^ dmask_at(p_first, j);
    }
  }
  __syncthreads();

  uint32_t v[NR];
  int cur = -1;  // current register layout (-1: keys are in shared memory)
  auto go = [&](int L) {
    if (cur == L) return;
    if (cur >= 0) {
      TL::sts_layout(cur, smem, v);
      __syncthreads();
    }
    TL::lds_layout(L, smem, v);
    cur = L;
  };
  auto step = [&](int lb) {
    const int L = TL::chunk_of(lb);
    go(L);
    TL::ce_q(lb - TL::z_of(L), v);
  };
  // In L_0 the thread's local index is (threadIdx.x << R) | e: local bits
  // >= R are per-thread uniform.
  auto l0_bit = [&](int p) -> uint32_t {
    // direction bit of phase p for this thread in layout L_0 (p's local bit
    // must be >= R or p must be outside S)
    if (p >= P.kd) return 0u;
    const int l = local_of(p);
    if (l >= 0) return (threadIdx.x >> (l - TL::R)) & 1u;
    return dir_bit_global(gbase, p, P.kd);
  };

  if (P.tile_sort) {
    // Phases 1..R-1: straight-line register code in L_0.
    go(0);
    TL::template reg_phases<1>(v, P.p_end, P.kd);
    if (P.p_end >= TL::R) {
      // Enter the phase domain at phase R.
      TL::xor_all(v, 0u - l0_bit(TL::R));
      for (int p = TL::R; p <= P.p_end; ++p) {
        for (int lb = p - 1; lb >= 0; --lb) step(lb);
        // now in L_0; move to phase p+1's domain (or leave it after p_end)
        const uint32_t nxt = (p < P.p_end) ? l0_bit(p + 1) : 0u;
        TL::xor_all(v, 0u - (l0_bit(p) ^ nxt));
      }
    }
    TL::xor_all(v, P.gmask_out);
  } else {
    if (P.segA_hi >= 0) {
      for (int lb = P.segA_hi; lb >= 0; --lb) step(lb);
      // in L_0: switch from phase pA's domain to pB's (or to plain keys)
      uint32_t m = 0u - l0_bit(P.pA);
      if (P.segB_lo >= 0) m ^= 0u - l0_bit(P.pB);
      TL::xor_all(v, m);
    }
    if (P.segB_lo >= 0) {
      for (int lb = C - 1; lb >= P.segB_lo; --lb) step(lb);
      // leave phase pB's domain at the staging store (dmask_at(p_last, j))
    }
  }

  // ---- staging store: registers -> shared -> coalesced global ------------
  if (cur >= 0) {
    TL::sts_layout(cur, smem, v);
  }
  __syncthreads();
  const bool exit_at_store = !P.tile_sort && P.segB_lo >= 0;
  if constexpr (N / T >= 4) {
    constexpr int IT = N / 4 / T;
#pragma unroll
    for (int it = 0; it < IT; ++it) {
      const uint32_t j = 4u * (uint32_t)(it * T + threadIdx.x);
      const uint32_t m = exit_at_store ? (dmask_at(p_last, j) ^ P.gmask_out)
                                       : (P.tile_sort ? 0u : P.gmask_out);
      const uint32_t pj = TL::pad(j);
      uint4 q;
      q.x = smem[pj + 0] ^ m;
      q.y = smem[pj + 1] ^ m;
      q.z = smem[pj + 2] ^ m;
      q.w = smem[pj + 3] ^ m;
      *reinterpret_cast<uint4*>(P.keys + gidx(j)) = q;
    }
  } else {
    for (uint32_t j = threadIdx.x; j < (uint32_t)N; j += T) {
      const uint32_t m = exit_at_store ? (dmask_at(p_last, j) ^ P.gmask_out)
                                       : (P.tile_sort ? 0u : P.gmask_out);
      P.keys[gidx(j)] = smem[TL::pad(j)] ^ m;
    }
  }
  pdl_trigger();
}

}  // namespace b200
