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

#include <type_traits>

#include "bitonic_engine.cuh"
#include "bitonic_rounds.cuh"

namespace b200 {

// ---- global access primitives ---------------------------------------------------
// Inline PTX keeps the 32 per-register accesses in register order (volatile
// asm is not reordered), which keeps the DRAM access order of all CTAs alike;
// B200_LDG_OP / B200_STG_OP select the cache operator (experiments).
#ifndef B200_LDG_OP
#define B200_LDG_OP ".lu"  // last use: measured best for the streaming passes
#endif
#ifndef B200_STG_OP
#define B200_STG_OP ""
#endif
__device__ __forceinline__ uint32_t ldg32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.global" B200_LDG_OP ".u32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ uint2 ldg64(const uint32_t* p) {
  uint2 v;
  asm volatile("ld.global" B200_LDG_OP ".v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "l"(p));
  return v;
}
__device__ __forceinline__ uint4 ldg128(const uint32_t* p) {
  uint4 v;
  asm volatile("ld.global" B200_LDG_OP ".v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  return v;
}
__device__ __forceinline__ void stg32(uint32_t* p, uint32_t v) {
  asm volatile("st.global" B200_STG_OP ".u32 [%0], %1;" :: "l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void stg64(uint32_t* p, uint32_t a, uint32_t b) {
  asm volatile("st.global" B200_STG_OP ".v2.u32 [%0], {%1, %2};" :: "l"(p), "r"(a), "r"(b) : "memory");
}
__device__ __forceinline__ void stg128(uint32_t* p, uint4 v) {
  asm volatile("st.global" B200_STG_OP ".v4.u32 [%0], {%1, %2, %3, %4};"
               :: "l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}

// ---- race stress (test builds only) ------------------------------------------
// With -DB200_JITTER every shared-memory hand-off point first sleeps a
// pseudo-random 0..1023 ns (per lane, per call site, per CTA, per clock), so
// the relative timing of threads, warps and CTAs differs from any production
// run; a missing barrier would surface as wrong output in the tests run
// against this build (tests/test_gpu_jitter.py).  No-op otherwise.
__device__ __forceinline__ void jitter(uint32_t site) {
#ifdef B200_JITTER
  uint32_t h = (blockIdx.x * 0x9E3779B9u) ^ (threadIdx.x * 0x85EBCA6Bu) ^ (site * 0xC2B2AE35u) ^
               (uint32_t)clock();
  h ^= h >> 15;
  h *= 0x2C1B3C6Du;
  h ^= h >> 12;
  if ((h & 3u) == 0u) __nanosleep((h >> 20) & 1023u);
#else
  (void)site;
#endif
}

// ---- coset geometry ----------------------------------------------------------
template <int C, int A>
struct Coset {
  // global offset of local index j (additive over disjoint bit fields)
  __host__ __device__ __forceinline__ static uint64_t goff(uint32_t j, int y) {
    if constexpr (A >= C) {
      return j;
    } else {
      return (uint64_t)(j & ((1u << A) - 1u)) + ((uint64_t)(j >> A) << y);
    }
  }
  __host__ __device__ __forceinline__ static uint64_t base(uint64_t b, int y) {
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
// Thread t moves the uint4 at local index j = 4t + it*4T for it = 0..IT-1.
// The two terms occupy disjoint local bits, so the global offset is
// goff(4t) + goff(it*4T): one per-thread base plus a uniform per-iteration
// offset (no per-key index arithmetic).
// The staging copies' shared-memory side: lane l of warp w writes / reads
// word q of the uint4 at local index 4(32w + l) + it*4T, padded.  Every such
// access of a warp must hit 32 distinct banks (the round layouts are checked
// by Layout::conflict_free; this covers the staging path).
template <int C, int R>
constexpr bool staging_conflict_free() {
  constexpr int T = 1 << (C - R), N = 1 << C;
  if (N / T < 4 || T < 32) return true;
  for (int w = 0; w < T / 32; ++w)
    for (int it = 0; it < N / 4 / T; ++it)
      for (int q = 0; q < 4; ++q) {
        uint32_t seen = 0;
        for (int l = 0; l < 32; ++l) {
          const uint32_t j = 4u * (uint32_t)(32 * w + l) + (uint32_t)(it * 4 * T) + (uint32_t)q;
          const uint32_t bank = smem_pad(j) & 31u;
          if (seen & (1u << bank)) return false;
          seen |= 1u << bank;
        }
      }
  return true;
}

template <int C, int A, int DBIT, int R>
__device__ __forceinline__ void stage_in(uint32_t* sm, const uint32_t* keys,
                                         uint64_t gbase, int y, uint32_t m_uniform) {
  using TL = Tile<C>;
  constexpr int T = 1 << (C - R), N = TL::N;
  static_assert(staging_conflict_free<C, R>(), "staging copy has bank conflicts");
  if constexpr (N / T >= 4) {
    constexpr int IT = N / 4 / T;
    const uint32_t j0 = 4u * threadIdx.x;
    const uint32_t* base = keys + gbase + Coset<C, A>::goff(j0, y);
    uint4 buf[IT];
#pragma unroll
    for (int it = 0; it < IT; ++it) {
      buf[it] = ldg128(base + Coset<C, A>::goff((uint32_t)(it * 4 * T), y));
    }
    jitter(1);
#pragma unroll
    for (int it = 0; it < IT; ++it) {
      const uint32_t j = j0 + (uint32_t)(it * 4 * T);
      const uint32_t pj = TL::pad(j);
      if constexpr (DBIT >= 0 && DBIT < 2) {
        // the direction bit varies inside the 4-key vector (the virtual
        // tile sort's phase-1 domain): one mask per key
        sm[pj + 0] = buf[it].x ^ m_uniform ^ (0u - (((j + 0u) >> DBIT) & 1u));
        sm[pj + 1] = buf[it].y ^ m_uniform ^ (0u - (((j + 1u) >> DBIT) & 1u));
        sm[pj + 2] = buf[it].z ^ m_uniform ^ (0u - (((j + 2u) >> DBIT) & 1u));
        sm[pj + 3] = buf[it].w ^ m_uniform ^ (0u - (((j + 3u) >> DBIT) & 1u));
      } else {
        uint32_t m = m_uniform;
        if constexpr (DBIT >= 0) m ^= 0u - ((j >> DBIT) & 1u);
        sm[pj + 0] = buf[it].x ^ m;
        sm[pj + 1] = buf[it].y ^ m;
        sm[pj + 2] = buf[it].z ^ m;
        sm[pj + 3] = buf[it].w ^ m;
      }
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

template <int C, int A, int R>
__device__ __forceinline__ void stage_out(const uint32_t* sm, uint32_t* keys,
                                          uint64_t gbase, int y) {
  using TL = Tile<C>;
  constexpr int T = 1 << (C - R), N = TL::N;
  jitter(2);
  __syncthreads();
  jitter(3);
  if constexpr (N / T >= 4) {
    constexpr int IT = N / 4 / T;
    const uint32_t j0 = 4u * threadIdx.x;
    uint32_t* base = keys + gbase + Coset<C, A>::goff(j0, y);
#pragma unroll
    for (int it = 0; it < IT; ++it) {
      const uint32_t pj = TL::pad(j0 + (uint32_t)(it * 4 * T));
      uint4 q;
      q.x = sm[pj + 0];
      q.y = sm[pj + 1];
      q.z = sm[pj + 2];
      q.w = sm[pj + 3];
      stg128(base + Coset<C, A>::goff((uint32_t)(it * 4 * T), y), q);
    }
  } else {
    for (uint32_t j = threadIdx.x; j < (uint32_t)N; j += T) {
      keys[gbase + Coset<C, A>::goff(j, y)] = sm[TL::pad(j)];
    }
  }
}

// ---- virtual padding (non-power-of-two lengths, no copy) -----------------------
// The array holds nreal keys; indices nreal .. 2^k - 1 are virtual.  A
// virtual key never reaches memory: loads give the phase domain's maximum
// (0xFFFFFFFF), stores skip it.  With the direction rule of the virtual plans
// (phase p's block is descending iff bit p of (index ^ (nreal - 1)) is set)
// the block holding index nreal - 1 is ascending at every level, so in the
// phase domain every compare-exchange that pairs a real key with a virtual
// one keeps the real key in place (the virtual index is the higher one) --
// the reference's pad_to_pow2 + sort + truncate (bench.cpp:366-377) without
// the padded copy.  Only CTAs whose coset straddles nreal take these paths.
template <int C, int A, int DBIT, int R>
__device__ __forceinline__ void stage_in_virtual(uint32_t* sm, const uint32_t* keys,
                                                 uint64_t gbase, int y, uint32_t m_uniform,
                                                 uint64_t nreal) {
  using TL = Tile<C>;
  constexpr int T = 1 << (C - R), N = TL::N;
  for (uint32_t j = threadIdx.x; j < (uint32_t)N; j += T) {
    uint32_t m = m_uniform;
    if constexpr (DBIT >= 0) m ^= 0u - ((j >> DBIT) & 1u);
    const uint64_t g = gbase + Coset<C, A>::goff(j, y);
    sm[TL::pad(j)] = g < nreal ? (keys[g] ^ m) : 0xFFFFFFFFu;
  }
  __syncthreads();
}

template <int C, int A, int R>
__device__ __forceinline__ void stage_out_virtual(const uint32_t* sm, uint32_t* keys,
                                                  uint64_t gbase, int y, uint64_t nreal) {
  using TL = Tile<C>;
  constexpr int T = 1 << (C - R), N = TL::N;
  __syncthreads();
  for (uint32_t j = threadIdx.x; j < (uint32_t)N; j += T) {
    const uint64_t g = gbase + Coset<C, A>::goff(j, y);
    if (g < nreal) keys[g] = sm[TL::pad(j)];
  }
}

template <int C, int R>
constexpr int threads_for() {
  return 1 << (C - R);
}
template <int C, int R, int MODE = 0>
constexpr int min_blocks_for() {
  // a 64-register budget per thread (1024 threads per SM at full use); two
  // register arrays of 32 keys get 128 registers (512 threads per SM)
  constexpr int slots = R >= 6 ? (MODE != 0 ? 256 : 512) : ((MODE != 0 && R >= 5) ? 512 : 1024);
  return threads_for<C, R>() >= slots ? 1
         : (slots / threads_for<C, R>() > 32 ? 32 : slots / threads_for<C, R>());
}

// ---- the pass body -------------------------------------------------------------
// Direction sources (phase-domain XOR, see bitonic_engine.cuh):
//   tile sort, phase p < R : natural domain, CEs use ce_dir (bit p is a
//                            register bit of round 0)
//   tile sort, phase p <  C: local bit p          (DL = p)
//   tile sort, phase C     : CTA-uniform          (DL = -1, value u[C])
//   merge, phase A         : local bit C-1 when segment B follows, else uniform
//   merge, phase B         : uniform
// MODE 0: keys only.  MODE 1: key + 32-bit payload (the payload array
// follows its key).  MODE 2: 64-bit keys split into a hi-word array (v) and
// a lo-word array (w), compared lexicographically.
// ---- shuffle tail ---------------------------------------------------------------
// When the steps of a pass's LAST round all touch lane bits of the round
// before it, those steps run as warp shuffles (SHFL.BFLY + one min/max per
// key) in that layout and the final shared-memory round trip (STS + barrier
// + LDS of every key) disappears.  B200_SHFL_TAIL = the most steps done this
// way (0 = off).  E.g. the 2^13-key tile sort's 17th round is the single
// step on bit 0 -- a lane bit of round 16's layout.
// Measured on B200 (tools/perf_probe.py, tools/pass_times.py, A/B against
// -DB200_SHFL_TAIL=0): no gain at any size -- 2^16 22.3/22.5 us, 2^20 49.1
// both, 2^24 479/475 us, 2^28 11.06/10.99 ms, batched 102-105 us both --
// and the 2^28 sort's last pass lost its direct store (366 vs 315 us); the
// tile sort saves one of 18 round trips but is ALU-bound.  Off by default.
#ifndef B200_SHFL_TAIL
#define B200_SHFL_TAIL 0
#endif

template <class LP>
constexpr int lane_of(int b) {
  const int lanes = LP::NT < 5 ? LP::NT : 5;
  for (int i = 0; i < lanes; ++i)
    if (LP::tpos(i) == b) return i;
  return -1;
}

template <class S, class RD, class LP, int NRND, int KIND, int R>
constexpr bool shfl_tail_ok() {
  if (B200_SHFL_TAIL <= 0 || NRND < 2 || LP::NT < 5) return false;
  const int b0 = RD::begin(NRND - 1), e = S::len();
  if (e - b0 > B200_SHFL_TAIL) return false;
  for (int i = b0; i < e; ++i) {
    if (lane_of<LP>(S::bit(i)) < 0) return false;
    if (KIND == 0 && S::phase(i) < R) return false;  // natural-domain phases
    if (S::phase(i) != S::phase(b0)) return false;
  }
  return true;
}

// AO >= 0 overrides the coset's low-run length A (the cluster passes run a
// tail on a 2^C sub-coset whose low run is shorter than C).
// VIRT: the virtual-padding variant (non-power-of-two single arrays).
template <int C, int KIND, int SA, int SB, int RR = reg_bits(C), int MODE = 0, int AO = -1,
          bool VIRT = false>
struct PassBody {
  static constexpr bool KV = MODE != 0;   // two register arrays
  // FMA-pipe share of the compare-exchange max (Layout::mm)
  static constexpr int FN = KIND == 0 ? B200_FMA_TILE_NUM : B200_FMA_NUM;
  static constexpr int FD = KIND == 0 ? B200_FMA_TILE_DEN : B200_FMA_DEN;
  static constexpr bool K64 = MODE == 2;
  using S = Seq<C, KIND, SA, SB>;
  static constexpr int R = RR;
  static constexpr int NR = 1 << R;
  static constexpr int A = AO >= 0 ? AO : (KIND == 0 ? C : (SB >= 0 ? SB : C));
  // Shared-memory round trips of a round cut: one per layout change, plus
  // one for a staged load / store when the first / last layout cannot talk
  // to HBM directly.
  template <class RX>
  static constexpr int smem_trips() {
    using F = Layout<C, RX::mask(0)>;
    using La = Layout<C, RX::mask(RX::count() - 1)>;
    const bool dl = KIND == 1 && F::lanes_low() && A >= F::vec_bits() + 5;
    const bool ds = KIND == 1 && La::lanes_low() && A >= La::vec_bits() + 5;
    return (RX::count() - 1) + (dl ? 0 : 1) + (ds ? 0 : 1);
  }
  using RD_GREEDY = Rounds<S, C, R, A, false>;
  using RD_DF = Rounds<S, C, R, A, true>;
  using RD = typename std::conditional<(KIND == 1 && smem_trips<RD_DF>() < smem_trips<RD_GREEDY>()),
                                       RD_DF, RD_GREEDY>::type;
  static constexpr int NRND = RD::count();
  template <int r>
  using L = Layout<C, RD::mask(r)>;
  // keys only: the last round may run as shuffles in the previous layout
  static constexpr bool SHT =
      MODE == 0 && !VIRT && shfl_tail_ok<S, RD, Layout<C, RD::mask(NRND >= 2 ? NRND - 2 : 0)>, NRND, KIND, R>();
  static constexpr int NRE = SHT ? NRND - 1 : NRND;  // rounds through shared memory

  // local direction bit of phase id ph (-1: uniform / none)
  static constexpr int dloc(int ph) {
    if (KIND == 0) return ph < C ? ph : -1;
    if (ph == 0) return SB >= 0 ? C - 1 : -1;
    return -1;
  }
  // is phase id ph in the natural domain (tile sort phases < R)
  // (the virtual variant runs every phase in the phase domain: its
  // directions carry a runtime flip, see flip())
  static constexpr bool natural(int ph) { return !VIRT && KIND == 0 && ph < R; }

  struct Ctx {
    uint32_t* keys;
    uint32_t* vals;       // payloads (KV)
    uint64_t gbase;
    int y;
    uint32_t uA, uB;      // uniform direction masks (merge)
    uint32_t uC;          // uniform direction mask of phase C (tile sort)
    uint32_t gin, gout;   // key-order transforms
    uint32_t gin_lo, gout_lo;  // low-word transforms (MODE 2)
    FmaSplit fs;               // opaque 1 / -1 (FMA-pipe max)
    // virtual padding (VIRT): real key count, direction flips of the local-
    // bit phases (bit p of nreal-1), and whether this coset straddles nreal
    uint64_t nreal;
    uint32_t xloc, xA;
    int partial;
  };

  // Runtime direction flip of phase PH when its direction bit is local.
  template <int PH>
  __device__ __forceinline__ static uint32_t flip(const Ctx& c) {
    if constexpr (!VIRT) {
      return 0u;
    } else if constexpr (KIND == 0) {
      if constexpr (PH < C) return 0u - ((c.xloc >> PH) & 1u);
      else return 0u;
    } else {
      if constexpr (PH == 0 && SB >= 0) return c.xA;
      else return 0u;
    }
  }

  // uniform mask for phase id ph when its direction bit is not local
  __device__ __forceinline__ static uint32_t uni(const Ctx& c, int ph) {
    if constexpr (KIND == 0) return c.uC;
    return ph == 0 ? c.uA : c.uB;
  }

  // Direction source of phase id PH in layout LR:
  //   register bit (compile-time per register), thread bit (runtime, maybe
  //   warp-uniform), CTA-uniform value, or none (natural domain).
  template <class LR, int PH>
  static constexpr int reg_q() {
    if (natural(PH)) return -1;
    constexpr int lb = dloc(PH);
    if (lb < 0) return -1;
    return LR::qof(lb);
  }
  template <class LR, int PH>
  static constexpr bool warp_uniform() {
    if (natural(PH)) return true;
    constexpr int lb = dloc(PH);
    if (lb < 0) return true;            // CTA-uniform
    if (LR::qof(lb) >= 0) return true;  // register part: no runtime value
    return LR::is_warp_bit(lb);
  }
  // runtime (non-register) part of phase PH's mask for this thread: 0 / ~0
  template <class LR, int PH>
  __device__ __forceinline__ static uint32_t uni_part(const Ctx& c, uint32_t tj) {
    if constexpr (natural(PH)) {
      return 0u;
    } else {
      constexpr int lb = dloc(PH);
      if constexpr (lb < 0) {
        return uni(c, PH);
      } else if constexpr (LR::qof(lb) >= 0) {
        return flip<PH>(c);
      } else {
        return (0u - ((tj >> lb) & 1u)) ^ flip<PH>(c);
      }
    }
  }

  // XOR register e with D_PH0(e) ^ D_PH1(e) ^ extra (PH < 0: no phase).
  // When the runtime part is warp-uniform the branch is divergence-free and
  // only the registers that actually flip are complemented.
  template <class LR, int PH0, int PH1, bool EXTRA_WARP_UNIFORM>
  __device__ __forceinline__ static void apply_mask1(const Ctx& c, uint32_t (&v)[NR],
                                                     uint32_t extra) {
    constexpr int q0 = PH0 >= 0 ? reg_q<LR, PH0>() : -1;
    constexpr int q1 = PH1 >= 0 ? reg_q<LR, PH1>() : -1;
    // (measured: helps the ALU-bound tile sort, hurts the latency-bound
    // merge passes at 2^20 -- so merges keep the straight XOR)
    constexpr bool wu = KIND == 0 && EXTRA_WARP_UNIFORM && (PH0 < 0 || warp_uniform<LR, PH0>()) &&
                        (PH1 < 0 || warp_uniform<LR, PH1>());
    const uint32_t tj = LR::thread_j();
    uint32_t u = 0u;  // runtime direction part: 0 or ~0
    if constexpr (PH0 >= 0) u ^= uni_part<LR, PH0>(c, tj);
    if constexpr (PH1 >= 0) u ^= uni_part<LR, PH1>(c, tj);
    auto rbit = [](int e) -> bool {
      bool r = false;
      if (q0 >= 0) r ^= ((e >> (q0 < 0 ? 0 : q0)) & 1) != 0;
      if (q1 >= 0) r ^= ((e >> (q1 < 0 ? 0 : q1)) & 1) != 0;
      return r;
    };
    if constexpr (wu) {
      if (u) {
#pragma unroll
        for (int e = 0; e < NR; ++e)
          if (!rbit(e)) v[e] = ~v[e];
      } else {
#pragma unroll
        for (int e = 0; e < NR; ++e)
          if (rbit(e)) v[e] = ~v[e];
      }
      // key-order transform (arbitrary CTA-uniform constant, usually 0)
      if (extra) {
#pragma unroll
        for (int e = 0; e < NR; ++e) v[e] ^= extra;
      }
    } else {
#pragma unroll
      for (int e = 0; e < NR; ++e) v[e] ^= (rbit(e) ? ~u : u) ^ extra;
    }
  }

  // Keys (both words of a 64-bit key in MODE 2; payloads never change).
  template <class LR, int PH0, int PH1, bool EXTRA_WARP_UNIFORM>
  __device__ __forceinline__ static void apply_mask(const Ctx& c, uint32_t (&v)[NR],
                                                    uint32_t (&w)[NR], uint32_t extra,
                                                    uint32_t extra_lo) {
    apply_mask1<LR, PH0, PH1, EXTRA_WARP_UNIFORM>(c, v, extra);
    if constexpr (K64) apply_mask1<LR, PH0, PH1, EXTRA_WARP_UNIFORM>(c, w, extra_lo);
  }

  template <class LR, int PH0, int PH1>
  __device__ __forceinline__ static void transition(const Ctx& c, uint32_t (&v)[NR],
                                                    uint32_t (&w)[NR]) {
    apply_mask<LR, PH0, PH1, true>(c, v, w, 0u, 0u);
  }

  template <class LR, int I>
  __device__ __forceinline__ static void one_step(const Ctx& c, uint32_t (&v)[NR],
                                                  uint32_t (&w)[NR]) {
    constexpr int ph = S::phase(I);
    constexpr int b = S::bit(I);
    if constexpr (natural(ph) && ph != 0) {
      if constexpr (K64) LR::template ce_dir_k64<b, ph>(v, w, c.fs);
      else if constexpr (KV) LR::template ce_dir_kv<b, ph>(v, w, c.fs);
      else LR::template ce_dir<b, ph, FN, FD>(v, c.fs);
    } else {
      if constexpr (K64) LR::template ce_k64<b>(v, w, c.fs);
      else if constexpr (KV) LR::template ce_kv<b>(v, w, c.fs);
      else LR::template ce<b, FN, FD>(v, c.fs);
    }
  }

  template <int r, int I>
  __device__ __forceinline__ static void steps(const Ctx& c, uint32_t (&v)[NR],
                                               uint32_t (&w)[NR]) {
    if constexpr (I < RD::begin(r + 1)) {
      if constexpr (I > 0 && S::phase(I) != S::phase(I - 1)) {
        transition<L<r>, S::phase(I - 1), S::phase(I)>(c, v, w);
        if constexpr (VIRT) {
          if (c.partial) reset_virtual<L<r>>(c, v);
        }
      }
      one_step<L<r>, I>(c, v, w);
      steps<r, I + 1>(c, v, w);
    }
  }

  // Direct (coalesced) HBM access is possible for a round's layout when its
  // lanes sit on 5 contiguous bits v..v+4 above a low register run of v <= 2
  // bits, all inside the contiguous low run of the coset (A >= v + 5).
  template <class LR>
  static constexpr bool direct_ok() {
    return KIND == 1 && LR::lanes_low() && A >= LR::vec_bits() + 5;
  }
  // Virtual keys back to the phase domain's maximum (after a transition XOR).
  template <class LR>
  __device__ __forceinline__ static void reset_virtual(const Ctx& c, uint32_t (&v)[NR]) {
    const uint64_t base = c.gbase + Coset<C, A>::goff(LR::thread_j(), c.y);
    const uint64_t lim = c.nreal > base ? c.nreal - base : 0;  // offsets >= lim are virtual
#pragma unroll
    for (int e = 0; e < NR; ++e)
      if (Coset<C, A>::goff(LR::dep_reg(e), c.y) >= lim) v[e] = 0xFFFFFFFFu;
  }
  template <class LR>
  __device__ __forceinline__ static void gload(const Ctx& c, uint32_t tj, uint32_t (&v)[NR]) {
    constexpr int V = LR::vec_bits();
    const uint32_t* base = c.keys + c.gbase + Coset<C, A>::goff(tj, c.y);
    if constexpr (V == 0) {
#pragma unroll
      for (int e = 0; e < NR; ++e) v[e] = ldg32(base + Coset<C, A>::goff(LR::dep_reg(e), c.y));
    } else if constexpr (V == 1) {
#pragma unroll
      for (int e = 0; e < NR; e += 2) {
        const uint2 q = ldg64(base + Coset<C, A>::goff(LR::dep_reg(e), c.y));
        v[e] = q.x;
        v[e + 1] = q.y;
      }
    } else {
#pragma unroll
      for (int e = 0; e < NR; e += 4) {
        const uint4 q = ldg128(base + Coset<C, A>::goff(LR::dep_reg(e), c.y));
        v[e] = q.x;
        v[e + 1] = q.y;
        v[e + 2] = q.z;
        v[e + 3] = q.w;
      }
    }
  }
  template <class LR>
  __device__ __forceinline__ static void gstore(const Ctx& c, uint32_t tj, const uint32_t (&v)[NR]) {
    constexpr int V = LR::vec_bits();
    // Re-derive the addresses instead of keeping the load's 32 pointers
    // live across the rounds (ptxas would spill them: merge_kernel<13,-1,9>
    // had 40 bytes of stack before this): an opaque copy of y
    // defeat the common-subexpression elimination (y * 1 with the 1 read
    // from a kernel parameter, like the FMA-split operands).
    const int y = c.y * (int)c.fs.one;
    uint32_t* base = c.keys + c.gbase + Coset<C, A>::goff(tj, y);
    if constexpr (V == 0) {
#pragma unroll
      for (int e = 0; e < NR; ++e) stg32(base + Coset<C, A>::goff(LR::dep_reg(e), y), v[e]);
    } else if constexpr (V == 1) {
#pragma unroll
      for (int e = 0; e < NR; e += 2) {
        stg64(base + Coset<C, A>::goff(LR::dep_reg(e), y), v[e], v[e + 1]);
      }
    } else {
#pragma unroll
      for (int e = 0; e < NR; e += 4) {
        stg128(base + Coset<C, A>::goff(LR::dep_reg(e), y),
               make_uint4(v[e], v[e + 1], v[e + 2], v[e + 3]));
      }
    }
  }

  // shared-memory words of one tile array (keys; payloads follow when KV)
  static constexpr uint32_t TW = (uint32_t)tile_smem_words(C);

  // Keys (and payloads) -> registers in round 0's layout (phase domain of
  // the first step).
  __device__ __forceinline__ static void load(const Ctx& c, uint32_t* sm, uint32_t (&v)[NR],
                                              uint32_t (&w)[NR]) {
    using L0 = L<0>;
    constexpr int PH = S::phase(0);
    if constexpr (VIRT) {
      if (c.partial) {  // keys only (the virtual plans are u32 / i32)
        // a straddling coset always goes through shared memory (scalar,
        // bounds-checked loads; few registers)
        constexpr int db = natural(PH) ? -1 : dloc(PH);
        const uint32_t u = natural(PH) ? 0u : (db >= 0 ? flip<PH>(c) : uni(c, PH));
        stage_in_virtual<C, A, db, R>(sm, c.keys, c.gbase, c.y, c.gin ^ u, c.nreal);
        L0::lds(sm, v);
        return;
      }
    }
    if constexpr (direct_ok<L0>()) {
      const uint32_t tj = L0::thread_j();
      gload<L0>(c, tj, v);
      if constexpr (KV) {
        Ctx cv = c;
        cv.keys = c.vals;
        gload<L0>(cv, tj, w);
      }
      apply_mask<L0, PH, -1, true>(c, v, w, c.gin, c.gin_lo);
    } else {
      constexpr int db = natural(PH) ? -1 : dloc(PH);
      const uint32_t u = natural(PH) ? 0u : (db >= 0 ? flip<PH>(c) : uni(c, PH));
      stage_in<C, A, db, R>(sm, c.keys, c.gbase, c.y, c.gin ^ u);
      if constexpr (K64) stage_in<C, A, db, R>(sm + TW, c.vals, c.gbase, c.y, c.gin_lo ^ u);
      else if constexpr (KV) stage_in<C, A, -1, R>(sm + TW, c.vals, c.gbase, c.y, 0u);
      L0::lds(sm, v);
      if constexpr (KV) L0::lds(sm + TW, w);
    }
  }

  // The shuffle tail (SHT): steps I.. on lane bits of layout L<NRE-1>.
  template <int I>
  __device__ __forceinline__ static void shfl_steps(const Ctx& c, uint32_t (&v)[NR],
                                                    uint32_t (&w)[NR]) {
    if constexpr (I < S::len()) {
      using LP = L<NRE - 1>;
      if constexpr (I > 0 && S::phase(I) != S::phase(I - 1)) {
        transition<LP, S::phase(I - 1), S::phase(I)>(c, v, w);
      }
      constexpr int li = lane_of<LP>(S::bit(I));
      static_assert(li >= 0, "shuffle step on a non-lane bit");
      const bool upper = (threadIdx.x >> li) & 1u;  // keeps the max (ascending domain)
#pragma unroll
      for (int e = 0; e < NR; ++e) {
        const uint32_t p = __shfl_xor_sync(0xFFFFFFFFu, v[e], 1u << li);
        v[e] = upper ? max(v[e], p) : min(v[e], p);
      }
      shfl_steps<I + 1>(c, v, w);
    }
  }

  // After the shared-memory rounds: the shuffle tail, if any.  The keys are
  // then in layout L<NRE - 1>.
  __device__ __forceinline__ static void tail(const Ctx& c, uint32_t (&v)[NR], uint32_t (&w)[NR]) {
    if constexpr (SHT) shfl_steps<RD::begin(NRND - 1)>(c, v, w);
  }

  // Registers (last round's layout, last phase's domain) -> keys (+ payloads).
  __device__ __forceinline__ static void store(const Ctx& c, uint32_t* sm, uint32_t (&v)[NR],
                                               uint32_t (&w)[NR]) {
    using LL = L<NRE - 1>;
    constexpr int PH = S::phase(S::len() - 1);
    const uint32_t tj = LL::thread_j();
    apply_mask<LL, PH, -1, true>(c, v, w, c.gout, c.gout_lo);
    if constexpr (VIRT) {
      if (c.partial) {
        LL::sts(sm, v);
        stage_out_virtual<C, A, R>(sm, c.keys, c.gbase, c.y, c.nreal);
        return;
      }
    }
    if constexpr (direct_ok<LL>()) {
      gstore<LL>(c, tj, v);
      if constexpr (KV) {
        Ctx cv = c;
        cv.keys = c.vals;
        gstore<LL>(cv, tj, w);
      }
    } else {
      jitter(4);
      LL::sts(sm, v);
      if constexpr (KV) LL::sts(sm + TW, w);
      stage_out<C, A, R>(sm, c.keys, c.gbase, c.y);
      if constexpr (KV) stage_out<C, A, R>(sm + TW, c.vals, c.gbase, c.y);
    }
  }

  template <int r>
  __device__ __forceinline__ static void rounds(const Ctx& c, uint32_t* sm, uint32_t (&v)[NR],
                                                uint32_t (&w)[NR]) {
    if constexpr (r < NRE) {
      if constexpr (r > 0) {
        jitter(10 + 2 * r);
        L<r - 1>::sts(sm, v);
        if constexpr (KV) L<r - 1>::sts(sm + TW, w);
        if constexpr (same_warp_bits<L<r - 1>, L<r>>()) {
          __syncwarp();
        } else {
          __syncthreads();
        }
        jitter(11 + 2 * r);
        L<r>::lds(sm, v);
        if constexpr (KV) L<r>::lds(sm + TW, w);
      }
      steps<r, RD::begin(r)>(c, v, w);
      rounds<r + 1>(c, sm, v, w);
    }
  }

  __device__ __forceinline__ static void run(const Ctx& c, uint32_t* sm) {
    uint32_t v[NR];
    uint32_t w[NR];  // payload registers (dead code unless KV)
    pdl_wait();
    load(c, sm, v, w);
    rounds<0>(c, sm, v, w);
    tail(c, v, w);
    store(c, sm, v, w);
    pdl_trigger();
  }
};

template <int C, int R = reg_bits(C), int MODE = 0, bool VIRT = false>
__global__ void __launch_bounds__(threads_for<C, R>(), min_blocks_for<C, R, MODE>())
tile_sort_kernel(PassParams P) {
  extern __shared__ uint32_t smem[];
  using B = PassBody<C, 0, -1, -1, R, MODE, -1, VIRT>;
  typename B::Ctx c;
  c.keys = P.keys;
  c.vals = P.vals;
  c.gbase = pass_block(P) << C;
  c.y = C;
  c.uA = c.uB = 0u;
  c.gin = P.gmask_in;
  c.gout = P.gmask_out;
  c.gin_lo = P.gmask_in_lo;
  c.gout_lo = P.gmask_out_lo;
  c.fs = FmaSplit{P.one, P.mone};
  if constexpr (VIRT) {
    if (c.gbase >= P.nreal) return;  // every key of this tile is virtual
    c.nreal = P.nreal;
    c.partial = c.gbase + ((1u << C) - 1u) >= P.nreal;
    c.xloc = (uint32_t)(P.dxor & ((1ull << C) - 1ull));
    c.xA = 0u;
    c.uC = 0u - dir_bit_global(c.gbase ^ P.dxor, C, P.kd);
  } else {
    c.uC = 0u - dir_bit_global(c.gbase, C, P.kd);
  }
  uint32_t v[B::NR];
  uint32_t w[B::NR];
  pdl_wait();
  B::load(c, smem, v, w);
  B::template rounds<0>(c, smem, v, w);
  B::tail(c, v, w);
  if (P.keys_out != nullptr) c.keys = P.keys_out;  // out of place (merge-path variant)
  B::store(c, smem, v, w);
  pdl_trigger();
}

template <int C, int SA, int SB, int R = reg_bits(C), int MODE = 0, bool VIRT = false>
__global__ void __launch_bounds__(threads_for<C, R>(), min_blocks_for<C, R, MODE>())
merge_kernel(PassParams P) {
  static_assert(SA >= 0 || SB >= 0, "empty pass");
  extern __shared__ uint32_t smem[];
  using B = PassBody<C, 1, SA, SB, R, MODE, -1, VIRT>;
  constexpr int A = B::A;
  typename B::Ctx c;
  c.keys = P.keys;
  c.vals = P.vals;
  c.y = P.y;
  c.gbase = Coset<C, A>::base(pass_block(P), P.y);
  c.uC = 0u;
  c.gin = 0u;  // a merge pass never runs first: keys are already transformed
  c.gout = P.gmask_out;
  c.gin_lo = 0u;
  c.gout_lo = P.gmask_out_lo;
  c.fs = FmaSplit{P.one, P.mone};
  if constexpr (VIRT) {
    if (c.gbase >= P.nreal) return;  // every key of this coset is virtual
    c.nreal = P.nreal;
    c.partial = c.gbase + Coset<C, A>::goff((1u << C) - 1u, P.y) >= P.nreal;
    c.xloc = 0u;
    c.xA = 0u - (uint32_t)((P.dxor >> P.pA) & 1u);
    c.uA = 0u - dir_bit_global(c.gbase ^ P.dxor, P.pA, P.kd);
    c.uB = 0u - dir_bit_global(c.gbase ^ P.dxor, P.pB, P.kd);
  } else {
    c.uA = 0u - dir_bit_global(c.gbase, P.pA, P.kd);
    c.uB = 0u - dir_bit_global(c.gbase, P.pB, P.kd);
  }
  B::run(c, smem);
}

}  // namespace b200
