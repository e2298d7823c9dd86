// bitonic_static.cuh -- compile-time specialised passes.
//
// Same engine as bitonic_engine.cuh (coset tile in registers + padded shared
// memory, phase-domain direction trick), but every pass shape is a template:
// the sequence of CE bits, the register layout before every step and each
// layout change are fixed at compile time.  The steps then compile to
// straight-line VIMNMX blocks with no dispatch, no loop-carried register
// moves and no per-key index arithmetic (the runtime-dispatched
// bitonic_pass_kernel spent ~70% of its issue slots on that overhead).
//
// Pass shapes (local bit space of a C-bit tile, see planner.hpp):
//   tile_sort_kernel<C>        phases 1..p_end of every 2^C tile
//   merge_kernel<C, SA, SB>    CEs on local bits SA..0 (tail of phase pA),
//                              then C-1..SB (head of phase pB); SA or SB may
//                              be -1 (absent).  The coset's low run is
//                              a = SB (or C when SB < 0) keys long.
#pragma once

#include "bitonic_engine.cuh"

namespace b200 {

template <int C>
struct Static {
  using TL = Tile<C>;
  static constexpr int R = TL::R;
  static constexpr int NR = TL::NR;
  static constexpr int T = TL::T;
  static constexpr int N = TL::N;

  __host__ __device__ static constexpr int chunk_of(int b) {
    return b < R ? 0 : ((C <= 10 || b < 10) ? 1 : 2);
  }
  __host__ __device__ static constexpr int z_of(int L) {
    return L == 0 ? TL::Z0 : (L == 1 ? TL::Z1 : TL::Z2);
  }
  __host__ __device__ static constexpr int chunk_lo(int L) { return L == 0 ? 0 : (L == 1 ? R : 10); }
  // layout after running the descending bit run [HI..LO] from layout PREV
  __host__ __device__ static constexpr int after_run(int HI, int LO, int PREV) {
    return HI >= LO ? chunk_of(LO) : PREV;
  }

  template <int L>
  __device__ __forceinline__ static void sts_L(uint32_t* sm, const uint32_t (&v)[NR]) {
    TL::template sts<z_of(L)>(sm, v);
  }
  template <int L>
  __device__ __forceinline__ static void lds_L(const uint32_t* sm, uint32_t (&v)[NR]) {
    TL::template lds<z_of(L)>(sm, v);
  }
  template <int FROM, int TO>
  __device__ __forceinline__ static void switch_to(uint32_t* sm, uint32_t (&v)[NR]) {
    if constexpr (FROM != TO) {
      if constexpr (FROM >= 0) {
        sts_L<FROM>(sm, v);
        __syncthreads();
      }
      lds_L<TO>(sm, v);
    }
  }
  template <int QH, int QL>
  __device__ __forceinline__ static void steps_q(uint32_t (&v)[NR]) {
    if constexpr (QH >= QL) {
      TL::template ce<QH>(v);
      steps_q<QH - 1, QL>(v);
    }
  }
  // CEs on local bits HI, HI-1, ..., LO (all ascending in the phase domain),
  // entering in layout PREV (-1: keys are in shared memory).
  template <int HI, int LO, int PREV>
  __device__ __forceinline__ static void run(uint32_t* sm, uint32_t (&v)[NR]) {
    if constexpr (HI >= LO) {
      constexpr int L = chunk_of(HI);
      switch_to<PREV, L>(sm, v);
      constexpr int LOW = chunk_lo(L) > LO ? chunk_lo(L) : LO;
      constexpr int Z = z_of(L);
      steps_q<HI - Z, LOW - Z>(v);
      run<LOW - 1, LO, L>(sm, v);
    }
  }
};

// ---- staging (coalesced HBM <-> padded shared memory) ----------------------
template <int C, int A>
struct Coset {
  // Global index of local index j for CTA base gbase: the low A local bits
  // are contiguous, the rest sit at global stride 2^y.
  __device__ __forceinline__ static uint64_t gidx(uint64_t gbase, uint32_t j, int y) {
    if constexpr (A >= C) {
      return gbase + j;
    } else {
      return gbase + (j & ((1u << A) - 1u)) + ((uint64_t)(j >> A) << y);
    }
  }
  __device__ __forceinline__ static uint64_t base(uint64_t b, int y) {
    if constexpr (A >= C) {
      return b << C;
    } else {
      const int gap = y - A;
      const uint64_t blo = b & ((1ull << gap) - 1ull);
      const uint64_t bhi = b >> gap;
      return (blo << A) | (bhi << (y + (C - A)));
    }
  }
};

// Load the CTA's coset into padded shared memory, XOR-ing each key with
// m_uniform ^ (bit DBIT of its local index ? ~0 : 0) (DBIT < 0: none).
template <int C, int A, int DBIT>
__device__ __forceinline__ void stage_in(uint32_t* sm, const uint32_t* keys,
                                         uint64_t gbase, int y, uint32_t m_uniform) {
  using TL = Tile<C>;
  constexpr int T = TL::T, N = TL::N;
  if constexpr (N / T >= 4) {
    constexpr int IT = N / 4 / T;
    uint4 buf[IT];
#pragma unroll
    for (int it = 0; it < IT; ++it) {
      const uint32_t j = 4u * (uint32_t)(it * T + threadIdx.x);
      buf[it] = *reinterpret_cast<const uint4*>(keys + Coset<C, A>::gidx(gbase, j, y));
    }
#pragma unroll
    for (int it = 0; it < IT; ++it) {
      const uint32_t j = 4u * (uint32_t)(it * T + threadIdx.x);
      uint32_t m = m_uniform;
      if constexpr (DBIT >= 0) m ^= 0u - ((j >> DBIT) & 1u);
      const uint32_t pj = TL::pad(j);
      sm[pj + 0] = buf[it].x ^ m;
      sm[pj + 1] = buf[it].y ^ m;
      sm[pj + 2] = buf[it].z ^ m;
      sm[pj + 3] = buf[it].w ^ m;
    }
  } else {
    for (uint32_t j = threadIdx.x; j < (uint32_t)N; j += T) {
      uint32_t m = m_uniform;
      if constexpr (DBIT >= 0) m ^= 0u - ((j >> DBIT) & 1u);
      sm[TL::pad(j)] = keys[Coset<C, A>::gidx(gbase, j, y)] ^ m;
    }
  }
  __syncthreads();
}

template <int C, int A>
__device__ __forceinline__ void stage_out(const uint32_t* sm, uint32_t* keys,
                                          uint64_t gbase, int y, uint32_t m) {
  using TL = Tile<C>;
  constexpr int T = TL::T, N = TL::N;
  __syncthreads();
  if constexpr (N / T >= 4) {
    constexpr int IT = N / 4 / T;
#pragma unroll
    for (int it = 0; it < IT; ++it) {
      const uint32_t j = 4u * (uint32_t)(it * T + threadIdx.x);
      const uint32_t pj = TL::pad(j);
      uint4 q;
      q.x = sm[pj + 0] ^ m;
      q.y = sm[pj + 1] ^ m;
      q.z = sm[pj + 2] ^ m;
      q.w = sm[pj + 3] ^ m;
      *reinterpret_cast<uint4*>(keys + Coset<C, A>::gidx(gbase, j, y)) = q;
    }
  } else {
    for (uint32_t j = threadIdx.x; j < (uint32_t)N; j += T) {
      keys[Coset<C, A>::gidx(gbase, j, y)] = sm[TL::pad(j)] ^ m;
    }
  }
}

template <int C>
constexpr int min_blocks_for() {
  return Tile<C>::T >= 1024 ? 1 : (1024 / Tile<C>::T > 32 ? 32 : 1024 / Tile<C>::T);
}

// ---- tile sort: phases 1..p_end of every 2^C tile ----------------------------
template <int C>
struct TileSortBody {
  using S = Static<C>;
  using TL = Tile<C>;
  static constexpr int R = TL::R;
  static constexpr int NR = TL::NR;

  // Direction bit of phase P for this thread in layout L_0.
  template <int P>
  __device__ __forceinline__ static uint32_t dbit(int kd) {
    if (P >= kd) return 0u;
    if constexpr (P < C) {
      return (threadIdx.x >> (P - R)) & 1u;  // local bit P >= R: a thread bit
    } else {
      return (uint32_t)(blockIdx.x & 1u);    // global bit C of a contiguous tile
    }
  }
  template <int P>
  __device__ __forceinline__ static void phases(uint32_t* sm, uint32_t (&v)[NR],
                                                int p_end, int kd) {
    if constexpr (P <= C) {
      if (P > p_end) return;
      S::template run<P - 1, 0, 0>(sm, v);
      uint32_t m = dbit<P>(kd);
      if (P < p_end) m ^= dbit<P + 1>(kd);
      TL::xor_all(v, 0u - m);
      phases<P + 1>(sm, v, p_end, kd);
    }
  }
};

template <int C>
__global__ void __launch_bounds__(Tile<C>::T, min_blocks_for<C>())
tile_sort_kernel(PassParams P) {
  using TL = Tile<C>;
  using S = Static<C>;
  constexpr int NR = TL::NR;
  extern __shared__ uint32_t smem[];
  const uint64_t gbase = (uint64_t)blockIdx.x << C;
  stage_in<C, C, -1>(smem, P.keys, gbase, C, P.gmask_in);
  uint32_t v[NR];
  S::template lds_L<0>(smem, v);
  TL::template reg_phases<1>(v, P.p_end, P.kd);
  if (P.p_end >= TL::R) {
    TL::xor_all(v, 0u - TileSortBody<C>::template dbit<TL::R>(P.kd));
    TileSortBody<C>::template phases<TL::R>(smem, v, P.p_end, P.kd);
  }
  TL::xor_all(v, P.gmask_out);
  S::template sts_L<0>(smem, v);
  stage_out<C, C>(smem, P.keys, gbase, C, 0u);
}

// ---- merge pass: tail of phase pA (local bits SA..0), head of phase pB -------
template <int C, int SA, int SB>
__global__ void __launch_bounds__(Tile<C>::T, min_blocks_for<C>())
merge_kernel(PassParams P) {
  using TL = Tile<C>;
  using S = Static<C>;
  constexpr int NR = TL::NR;
  constexpr int R = TL::R;
  constexpr int A = SB >= 0 ? SB : C;  // low contiguous run (local bits [0, A))
  static_assert(SA >= 0 || SB >= 0, "empty pass");
  static_assert(SA < A, "tail bits must lie in the low run");
  extern __shared__ uint32_t smem[];

  const int y = P.y;
  const uint64_t gbase = Coset<C, A>::base(blockIdx.x, y);
  // Uniform direction bits (phase outside the coset, or p >= kd).
  const uint32_t dB = SB >= 0 ? dir_bit_global(gbase, P.pB, P.kd) : 0u;
  uint32_t v[NR];

  if constexpr (SA >= 0) {
    // Phase pA's direction bit: local C-1 when the head of pB follows (the
    // coset's high range then ends at bit pA), else a CTA-uniform bit.
    if constexpr (SB >= 0) {
      stage_in<C, A, C - 1>(smem, P.keys, gbase, y, P.gmask_in);
    } else {
      stage_in<C, A, -1>(smem, P.keys, gbase, y,
                         P.gmask_in ^ (0u - dir_bit_global(gbase, P.pA, P.kd)));
    }
    S::template run<SA, 0, -1>(smem, v);
    // now in L_0: leave phase pA's domain, enter pB's
    uint32_t m;
    if constexpr (SB >= 0) {
      m = ((threadIdx.x >> (C - 1 - R)) & 1u) ^ dB;
    } else {
      m = dir_bit_global(gbase, P.pA, P.kd);
    }
    TL::xor_all(v, 0u - m);
    if constexpr (SB >= 0) {
      S::template run<C - 1, SB, 0>(smem, v);
    }
  } else {
    stage_in<C, A, -1>(smem, P.keys, gbase, y, P.gmask_in ^ (0u - dB));
    S::template run<C - 1, SB, -1>(smem, v);
  }
  constexpr int FL = SB >= 0 ? S::chunk_of(SB) : 0;
  S::template sts_L<FL>(smem, v);
  stage_out<C, A>(smem, P.keys, gbase, y, P.gmask_out ^ (0u - dB));
}

}  // namespace b200
