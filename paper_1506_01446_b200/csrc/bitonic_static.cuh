// bitonic_static.cuh -- compile-time specialised passes built from rounds.
//
// Every pass shape is a template, so the CE sequence, the register set of
// every round (bitonic_rounds.cuh), each layout change, each phase-direction
// change and the choice between direct and staged HBM access are fixed at
// compile time.  The steps compile to straight-line VIMNMX blocks with no
// dispatch, no loop-carried register moves and no per-key index arithmetic.
//
//   tile_sort_kernel<C>        phases 1..C of every contiguous 2^C tile
//   merge_kernel<C, SA, SB>    CEs on local bits SA..0 (tail of phase pA),
//                              then C-1..SB (head of phase pB); SA or SB may
//                              be -1 (absent).  The coset's low run is
//                              A = SB (or C when SB < 0) keys long.
#pragma once

#include "bitonic_engine.cuh"
#include "bitonic_rounds.cuh"

namespace b200 {

// ---- coset geometry ----------------------------------------------------------
template <int C, int A>
struct Coset {
  // global offset of local index j (additive over disjoint bit fields)
  __device__ __forceinline__ static uint64_t goff(uint32_t j, int y) {
    if constexpr (A >= C) {
      return j;
    } else {
      return (uint64_t)(j & ((1u << A) - 1u)) + ((uint64_t)(j >> A) << y);
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

// ---- staging (coalesced HBM <-> padded shared memory) ------------------------
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
      buf[it] = *reinterpret_cast<const uint4*>(keys + gbase + Coset<C, A>::goff(j, y));
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
      sm[TL::pad(j)] = keys[gbase + Coset<C, A>::goff(j, y)] ^ m;
    }
  }
  __syncthreads();
}

template <int C, int A>
__device__ __forceinline__ void stage_out(const uint32_t* sm, uint32_t* keys,
                                          uint64_t gbase, int y) {
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
      q.x = sm[pj + 0];
      q.y = sm[pj + 1];
      q.z = sm[pj + 2];
      q.w = sm[pj + 3];
      *reinterpret_cast<uint4*>(keys + gbase + Coset<C, A>::goff(j, y)) = q;
    }
  } else {
    for (uint32_t j = threadIdx.x; j < (uint32_t)N; j += T) {
      keys[gbase + Coset<C, A>::goff(j, y)] = sm[TL::pad(j)];
    }
  }
}

template <int C>
constexpr int min_blocks_for() {
  return Tile<C>::T >= 1024 ? 1 : (1024 / Tile<C>::T > 32 ? 32 : 1024 / Tile<C>::T);
}

// ---- the pass body -------------------------------------------------------------
// Direction sources (phase-domain XOR, see bitonic_engine.cuh):
//   tile sort, phase p < R : natural domain, CEs use ce_dir (bit p is a
//                            register bit of round 0)
//   tile sort, phase p <  C: local bit p          (DL = p)
//   tile sort, phase C     : CTA-uniform          (DL = -1, value u[C])
//   merge, phase A         : local bit C-1 when segment B follows, else uniform
//   merge, phase B         : uniform
template <int C, int KIND, int SA, int SB>
struct PassBody {
  using S = Seq<C, KIND, SA, SB>;
  static constexpr int R = reg_bits(C);
  static constexpr int NR = 1 << R;
  using RD = Rounds<S, C, R>;
  static constexpr int NRND = RD::count();
  static constexpr int A = KIND == 0 ? C : (SB >= 0 ? SB : C);
  template <int r>
  using L = Layout<C, RD::mask(r)>;

  // local direction bit of phase id ph (-1: uniform / none)
  static constexpr int dloc(int ph) {
    if (KIND == 0) return ph < C ? ph : -1;
    if (ph == 0) return SB >= 0 ? C - 1 : -1;
    return -1;
  }
  // is phase id ph in the natural domain (tile sort phases < R)
  static constexpr bool natural(int ph) { return KIND == 0 && ph < R; }

  struct Ctx {
    uint32_t* keys;
    uint64_t gbase;
    int y;
    uint32_t uA, uB;      // uniform direction masks (merge)
    uint32_t uC;          // uniform direction mask of phase C (tile sort)
    uint32_t gin, gout;   // key-order transforms
  };

  // uniform mask for phase id ph when its direction bit is not local
  __device__ __forceinline__ static uint32_t uni(const Ctx& c, int ph) {
    if constexpr (KIND == 0) return c.uC;
    return ph == 0 ? c.uA : c.uB;
  }

  // Mask of register e, layout LR, phase id ph (0 / ~0).
  template <class LR, int PH>
  __device__ __forceinline__ static uint32_t dmask(const Ctx& c, int e, uint32_t tj) {
    if constexpr (natural(PH)) {
      return 0u;
    } else {
      constexpr int lb = dloc(PH);
      if constexpr (lb >= 0) {
        if constexpr (LR::qof(lb) >= 0) {
          return ((e >> LR::qof(lb)) & 1) ? 0xFFFFFFFFu : 0u;
        } else {
          return 0u - ((tj >> lb) & 1u);
        }
      } else {
        return uni(c, PH);
      }
    }
  }

  template <class LR, int PH0, int PH1>
  __device__ __forceinline__ static void transition(const Ctx& c, uint32_t (&v)[NR],
                                                    uint32_t extra) {
    const uint32_t tj = LR::thread_j();
#pragma unroll
    for (int e = 0; e < NR; ++e) {
      const uint32_t m = dmask<LR, PH0>(c, e, tj) ^ dmask<LR, PH1>(c, e, tj) ^ extra;
      v[e] ^= m;
    }
  }

  template <class LR, int I>
  __device__ __forceinline__ static void one_step(uint32_t (&v)[NR]) {
    constexpr int ph = S::phase(I);
    constexpr int b = S::bit(I);
    if constexpr (natural(ph)) {
      if constexpr (ph == 0) {
        LR::template ce<b>(v);
      } else {
        LR::template ce_dir<b, ph>(v);
      }
    } else {
      LR::template ce<b>(v);
    }
  }

  template <int r, int I>
  __device__ __forceinline__ static void steps(const Ctx& c, uint32_t (&v)[NR]) {
    if constexpr (I < RD::begin(r + 1)) {
      if constexpr (I > 0 && S::phase(I) != S::phase(I - 1)) {
        transition<L<r>, S::phase(I - 1), S::phase(I)>(c, v, 0u);
      }
      one_step<L<r>, I>(v);
      steps<r, I + 1>(c, v);
    }
  }

  // Keys -> registers in round 0's layout (phase domain of the first step).
  __device__ __forceinline__ static void load(const Ctx& c, uint32_t* sm, uint32_t (&v)[NR]) {
    using L0 = L<0>;
    constexpr int PH = S::phase(0);
    if constexpr (KIND == 1 && L0::lanes_low() && A >= 5) {
      const uint32_t tj = L0::thread_j();
      const uint32_t* base = c.keys + c.gbase + Coset<C, A>::goff(tj, c.y);
#pragma unroll
      for (int e = 0; e < NR; ++e) {
        v[e] = base[Coset<C, A>::goff(L0::dep_reg(e), c.y)];
      }
#pragma unroll
      for (int e = 0; e < NR; ++e) v[e] ^= dmask<L0, PH>(c, e, tj) ^ c.gin;
    } else {
      constexpr int db = natural(PH) ? -1 : dloc(PH);
      const uint32_t u = (natural(PH) || db >= 0) ? 0u : uni(c, PH);
      stage_in<C, A, db>(sm, c.keys, c.gbase, c.y, c.gin ^ u);
      L0::lds(sm, v);
    }
  }

  // Registers (last round's layout, last phase's domain) -> keys.
  __device__ __forceinline__ static void store(const Ctx& c, uint32_t* sm, uint32_t (&v)[NR]) {
    using LL = L<NRND - 1>;
    constexpr int PH = S::phase(S::len() - 1);
    const uint32_t tj = LL::thread_j();
#pragma unroll
    for (int e = 0; e < NR; ++e) v[e] ^= dmask<LL, PH>(c, e, tj) ^ c.gout;
    if constexpr (KIND == 1 && LL::lanes_low() && A >= 5) {
      uint32_t* base = c.keys + c.gbase + Coset<C, A>::goff(tj, c.y);
#pragma unroll
      for (int e = 0; e < NR; ++e) {
        base[Coset<C, A>::goff(LL::dep_reg(e), c.y)] = v[e];
      }
    } else {
      LL::sts(sm, v);
      stage_out<C, A>(sm, c.keys, c.gbase, c.y);
    }
  }

  template <int r>
  __device__ __forceinline__ static void rounds(const Ctx& c, uint32_t* sm, uint32_t (&v)[NR]) {
    if constexpr (r < NRND) {
      if constexpr (r > 0) {
        L<r - 1>::sts(sm, v);
        __syncthreads();
        L<r>::lds(sm, v);
      }
      steps<r, RD::begin(r)>(c, v);
      rounds<r + 1>(c, sm, v);
    }
  }

  __device__ __forceinline__ static void run(const Ctx& c, uint32_t* sm) {
    uint32_t v[NR];
    pdl_wait();
    load(c, sm, v);
    rounds<0>(c, sm, v);
    store(c, sm, v);
    pdl_trigger();
  }
};

template <int C>
__global__ void __launch_bounds__(Tile<C>::T, min_blocks_for<C>())
tile_sort_kernel(PassParams P) {
  extern __shared__ uint32_t smem[];
  using B = PassBody<C, 0, -1, -1>;
  typename B::Ctx c;
  c.keys = P.keys;
  c.gbase = (uint64_t)blockIdx.x << C;
  c.y = C;
  c.uA = c.uB = 0u;
  c.uC = 0u - dir_bit_global(c.gbase, C, P.kd);
  c.gin = P.gmask_in;
  c.gout = P.gmask_out;
  B::run(c, smem);
}

template <int C, int SA, int SB>
__global__ void __launch_bounds__(Tile<C>::T, min_blocks_for<C>())
merge_kernel(PassParams P) {
  static_assert(SA >= 0 || SB >= 0, "empty pass");
  extern __shared__ uint32_t smem[];
  using B = PassBody<C, 1, SA, SB>;
  constexpr int A = B::A;
  typename B::Ctx c;
  c.keys = P.keys;
  c.y = P.y;
  c.gbase = Coset<C, A>::base(blockIdx.x, P.y);
  c.uA = 0u - dir_bit_global(c.gbase, P.pA, P.kd);
  c.uB = 0u - dir_bit_global(c.gbase, P.pB, P.kd);
  c.uC = 0u;
  c.gin = P.gmask_in;
  c.gout = P.gmask_out;
  B::run(c, smem);
}

}  // namespace b200
