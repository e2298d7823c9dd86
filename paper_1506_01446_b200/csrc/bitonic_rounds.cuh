// bitonic_rounds.cuh -- compile-time "round" engine for the specialised passes.
//
// A pass applies a fixed sequence of compare-exchange (CE) steps to the
// CTA's 2^C-key coset (see bitonic_engine.cuh for the coset / phase-domain
// conventions).  Here the sequence is cut, at compile time, into ROUNDS: a
// round is a maximal run of consecutive steps touching at most R = 5
// distinct local bits.  For a round, the thread's 32 registers hold the 32
// keys whose local index varies exactly in those 5 bits (register set RM),
// so every CE of the round is a register min/max.  Between rounds the tile
// is re-partitioned through padded shared memory (one STS + one LDS per
// key).  Compared with fixed 5-bit chunks this packs steps from different
// phases / bit ranges into one round (fewer shared-memory round trips, the
// dominant cost measured by ncu), and it lets the first and last round of a
// merge pass talk to HBM directly: when a round's registers avoid local bits
// 0..4, the 32 lanes of a warp own 32 consecutive keys, so each register is
// one coalesced 128-byte LDG/STG and the shared-memory staging copy
// disappears.
//
// Thread layout of a round with register set RM: thread index bits are
// deposited, in order, into the non-register local bits (so the lane = the
// 5 lowest non-register bits).  Shared address pad(j) = j + j/32 is additive
// over the disjoint thread / register fields, so register e always sits at a
// compile-time immediate offset from a per-thread base, and every layout
// whose lanes lie below bit 10 is bank-conflict free (checked by
// static_assert below).
#pragma once

#include <cstdint>

#include "bitonic_engine.cuh"

// CEs whose max runs on the FMA pipe: NUM of every DEN (measured on B200:
// 2/3 for the merge passes, 1/3 for the tile sort, whose issue slots and
// shared-memory pipe are as busy as its ALU pipe).
#ifndef B200_FMA_NUM
#define B200_FMA_NUM 2
#endif
#ifndef B200_FMA_DEN
#define B200_FMA_DEN 3
#endif
#ifndef B200_FMA_TILE_NUM
#define B200_FMA_TILE_NUM 1
#endif
#ifndef B200_FMA_TILE_DEN
#define B200_FMA_TILE_DEN 3
#endif

namespace b200 {

// ---- compile-time step sequences -----------------------------------------
// KIND 0: tile sort, phases 1..C (step s of phase p touches bit p-1-s).
// KIND 1: merge, bits SA..0 (phase "A"), then C-1..SB (phase "B").
template <int C, int KIND, int SA, int SB>
struct Seq {
  static constexpr int len() {
    return KIND == 0 ? C * (C + 1) / 2 : (SA + 1) + (SB >= 0 ? C - SB : 0);
  }
  // phase id of step i: tile sort -> p (1..C); merge -> 0 (A) or 1 (B)
  static constexpr int phase(int i) {
    if (KIND == 0) {
      int p = 1;
      while (i >= p) {
        i -= p;
        ++p;
      }
      return p;
    }
    return i < SA + 1 ? 0 : 1;
  }
  static constexpr int bit(int i) {
    if (KIND == 0) {
      int p = 1;
      while (i >= p) {
        i -= p;
        ++p;
      }
      return p - 1 - i;
    }
    return i < SA + 1 ? SA - i : C - 1 - (i - (SA + 1));
  }
};

constexpr int popc(uint32_t x) {
  int c = 0;
  while (x) {
    c += x & 1u;
    x >>= 1;
  }
  return c;
}

// A register set leaves, for every residue r mod 5, a free (thread) bit
// position p = r (mod 5) below C: then 5 lanes with distinct residues exist
// and the layout is bank-conflict free under smem_pad.
template <int C>
constexpr bool lanes_feasible(uint32_t m) {
  for (int r = 0; r < 5; ++r) {
    bool ok = false;
    for (int p = r; p < C; p += 5)
      if (!(m & (1u << p))) ok = true;
    if (!ok) return false;
  }
  return true;
}

// Greedy rounds: round r covers steps [begin(r), begin(r+1)).  A round also
// ends early when its register set would make a conflict-free lane choice
// impossible (only enforced for C >= 10, where every residue has two
// positions).
// DF ("direct first"): round 0 stops before the first step on a bit < 5, so
// its lanes can sit on bits 0..4 and the pass loads straight from HBM
// instead of staging through shared memory (PassBody picks whichever cut
// needs fewer shared-memory round trips).
template <class S, int C, int R, int A = C, bool DF = false>
struct Rounds {
  static constexpr bool enforce = C >= 10 && C - R >= 5;
  static constexpr int next_begin(int b) {
    uint32_t m = 0;
    int i = b;
    while (i < S::len()) {
      const uint32_t nm = m | (1u << S::bit(i));
      if (popc(nm) > R) break;
      if (enforce && !lanes_feasible<C>(nm)) break;
      if (DF && b == 0 && i > 0 && S::bit(i) < 5) break;
      m = nm;
      ++i;
    }
    return i;
  }
  static constexpr int begin(int r) {
    int b = 0;
    for (int k = 0; k < r; ++k) b = next_begin(b);
    return b;
  }
  static constexpr int count() {
    int r = 0, b = 0;
    while (b < S::len()) {
      b = next_begin(b);
      ++r;
    }
    return r;
  }
  // Register set of round r: its step bits, padded to R bits.  Fillers come
  // first from [5, A) -- above the lanes but inside the coset's contiguous
  // run, so direct HBM access needs fewer per-register pointers -- then from
  // the top (keeps the lanes on the low bits).
  static constexpr uint32_t mask(int r) {
    uint32_t m = 0;
    const int e = begin(r + 1);
    for (int i = begin(r); i < e; ++i) m |= 1u << S::bit(i);
    for (int b = A - 1; b >= 5 && popc(m) < R; --b) {
      if (m & (1u << b)) continue;
      if (enforce && !lanes_feasible<C>(m | (1u << b))) continue;
      m |= 1u << b;
    }
    for (int b = C - 1; b >= 0 && popc(m) < R; --b) {
      if (m & (1u << b)) continue;
      if (enforce && !lanes_feasible<C>(m | (1u << b))) continue;
      m |= 1u << b;
    }
    return m;
  }
};

// Two layouts of the same tile whose warp bits (thread bits 5 and up) sit on
// the same local bits give every warp the same set of keys: a re-partition
// between them only moves keys inside each warp's own shared-memory
// addresses, so a warp barrier suffices (no CTA barrier).
template <class LA, class LB>
constexpr bool same_warp_bits() {
  static_assert(LA::NT == LB::NT, "layouts of different thread counts");
  for (int i = 5; i < LA::NT; ++i)
    if (LA::tpos(i) != LB::tpos(i)) return false;
  return true;
}

// ---- layouts ---------------------------------------------------------------
template <int C, uint32_t RM>
struct Layout {
  static constexpr int R = popc(RM);
  static constexpr int NR = 1 << R;
  static constexpr int NT = C - R;  // thread bits
  // position of the i-th register bit / i-th thread bit
  static constexpr int rpos(int i) {
    int k = -1;
    for (int b = 0; b < C; ++b)
      if (RM & (1u << b)) {
        if (++k == i) return b;
      }
    return -1;
  }
  // i-th free (non-register) position, ascending
  static constexpr int free_pos(int i) {
    int k = -1;
    for (int b = 0; b < C; ++b)
      if (!(RM & (1u << b))) {
        if (++k == i) return b;
      }
    return -1;
  }
  // lane bit r -> the lowest free position with residue r (mod 5)
  static constexpr int lane_pos(int r) {
    for (int p = r; p < C; p += 5)
      if (!(RM & (1u << p))) return p;
    return -1;
  }
  static constexpr bool residue_lanes() {
    if (C - R < 5) return false;
    for (int r = 0; r < 5; ++r)
      if (lane_pos(r) < 0) return false;
    return true;
  }
  static constexpr bool is_lane_pos(int p) {
    for (int r = 0; r < 5; ++r)
      if (lane_pos(r) == p) return true;
    return false;
  }
  // number of consecutive register bits starting at bit 0
  static constexpr int vec_bits() {
    int v = 0;
    while (v < C && (RM & (1u << v))) ++v;
    return v;
  }
  // lanes on the 5 bits just above the low register run: a warp then owns
  // 32 x 2^v consecutive keys (coalesced vector access, v <= 2)
  static constexpr bool contiguous_lanes() {
    const int v = vec_bits();
    if (C - R < 5 || v > 2 || v + 5 > C) return false;
    for (int b = v; b < v + 5; ++b)
      if (RM & (1u << b)) return false;
    return true;
  }
  // position of thread bit i: lanes first (5 contiguous bits when possible,
  // else one per residue), then the remaining free positions ascending
  static constexpr int tpos(int i) {
    if (contiguous_lanes()) {
      const int v = vec_bits();
      if (i < 5) return v + i;
      int k = 4;
      for (int b = 0; b < C; ++b)
        if (!(RM & (1u << b)) && !(b >= v && b < v + 5)) {
          if (++k == i) return b;
        }
      return -1;
    }
    if (!residue_lanes()) return free_pos(i);
    if (i < 5) return lane_pos(i);
    int k = 4;
    for (int b = 0; b < C; ++b)
      if (!(RM & (1u << b)) && !is_lane_pos(b)) {
        if (++k == i) return b;
      }
    return -1;
  }
  // index of local bit b among the register bits (-1: thread bit)
  static constexpr int qof(int b) {
    if (!(RM & (1u << b))) return -1;
    int k = 0;
    for (int x = 0; x < b; ++x)
      if (RM & (1u << x)) ++k;
    return k;
  }
  static constexpr uint32_t dep_reg(int e) {
    uint32_t j = 0;
    for (int i = 0; i < R; ++i)
      if (e & (1 << i)) j |= 1u << rpos(i);
    return j;
  }
  static constexpr uint32_t pad(uint32_t j) { return smem_pad(j); }
  static constexpr uint32_t reg_off(int e) { return pad(dep_reg(e)); }
  static constexpr uint32_t dep_thr(uint32_t t) {
    uint32_t j = 0;
    for (int i = 0; i < C - R; ++i)
      if (t & (1u << i)) j |= 1u << tpos(i);
    return j;
  }
  static constexpr bool conflict_free() {
    const int lanes = (C - R) < 5 ? (1 << (C - R)) : 32;
    for (int a = 0; a < lanes; ++a)
      for (int b = a + 1; b < lanes; ++b)
        if ((pad(dep_thr(a)) & 31u) == (pad(dep_thr(b)) & 31u)) return false;
    return true;
  }
  static_assert(C < 10 || conflict_free(), "shared-memory layout has bank conflicts");
  // local bit b is a warp bit (a thread bit that is not one of the 5 lanes)
  static constexpr bool is_warp_bit(int b) {
    if (RM & (1u << b)) return false;
    const int lanes = (C - R) < 5 ? (C - R) : 5;
    for (int i = 0; i < lanes; ++i)
      if (tpos(i) == b) return false;
    return true;
  }
  // lanes own consecutive 2^v-key vectors (direct coalesced global access)
  static constexpr bool lanes_low() { return contiguous_lanes(); }

  // length of the run of consecutive thread bits starting at thread bit i
  // that land on consecutive local bits
  static constexpr int run_len(int i) {
    int n = 1;
    while (i + n < C - R && tpos(i + n) == tpos(i) + n) ++n;
    return n;
  }
  template <int I>
  __device__ __forceinline__ static uint32_t tj_rec(uint32_t t) {
    if constexpr (I >= C - R) {
      return 0u;
    } else {
      constexpr int len = run_len(I);
      constexpr uint32_t lm = (len >= 32) ? 0xFFFFFFFFu : ((1u << len) - 1u);
      return (((t >> I) & lm) << tpos(I)) | tj_rec<I + len>(t);
    }
  }
  // Runtime deposit of this thread's index into the thread bits.
  __device__ __forceinline__ static uint32_t thread_j() { return tj_rec<0>(threadIdx.x); }
  __device__ __forceinline__ static void sts(uint32_t* sm, const uint32_t (&v)[NR]) {
    const uint32_t b = pad(thread_j());
#pragma unroll
    for (int e = 0; e < NR; ++e) sm[b + reg_off(e)] = v[e];
  }
  __device__ __forceinline__ static void lds(const uint32_t* sm, uint32_t (&v)[NR]) {
    const uint32_t b = pad(thread_j());
#pragma unroll
    for (int e = 0; e < NR; ++e) v[e] = sm[b + reg_off(e)];
  }
  // min and max of one compare-exchange.  VIMNMX issues at 64/clk/SM on the
  // ALU pipe, so a CE costs two ALU slots; for two CEs in three, max is
  // computed as x + y - min by two IMADs on the otherwise idle FMA pipe
  // (exact in mod-2^32 arithmetic).  tools/mb_minmax.cu: 45 CE/clk/SM with
  // this 2:1 split vs 32 with VIMNMX pairs.  `one`/`mone` come from the
  // kernel parameters so ptxas cannot turn the IMADs back into IADD3s.
  template <int NUM, int DEN>
  __device__ __forceinline__ static void mm(int idx, uint32_t x, uint32_t y, uint32_t& lo,
                                            uint32_t& hi, FmaSplit f) {
    lo = min(x, y);
    if (idx % DEN < NUM) {
      uint32_t s;
      asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(s) : "r"(x), "r"(f.one), "r"(y));
      asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(hi) : "r"(lo), "r"(f.mone), "r"(s));
    } else {
      hi = max(x, y);
    }
  }
  // CE on local bit B (ascending in the phase domain)
  template <int B, int NUM, int DEN>
  __device__ __forceinline__ static void ce(uint32_t (&v)[NR], FmaSplit f) {
    constexpr int q = qof(B);
    static_assert(q >= 0, "CE bit must be a register bit");
#pragma unroll
    for (int e = 0; e < NR; ++e) {
      if (!(e & (1 << q))) {
        const int idx = (e & ((1 << q) - 1)) | ((e >> (q + 1)) << q);
        mm<NUM, DEN>(idx, v[e], v[e | (1 << q)], v[e], v[e | (1 << q)], f);
      }
    }
  }
  // CE on local bit B, direction from local bit D (a register bit)
  template <int B, int D, int NUM, int DEN>
  __device__ __forceinline__ static void ce_dir(uint32_t (&v)[NR], FmaSplit f) {
    constexpr int q = qof(B);
    constexpr int qd = qof(D);
    static_assert(q >= 0 && qd >= 0, "CE and direction bits must be register bits");
#pragma unroll
    for (int e = 0; e < NR; ++e) {
      if (!(e & (1 << q))) {
        const int idx = (e & ((1 << q) - 1)) | ((e >> (q + 1)) << q);
        uint32_t lo, hi;
        mm<NUM, DEN>(idx, v[e], v[e | (1 << q)], lo, hi, f);
        const bool desc = (e >> qd) & 1;
        v[e] = desc ? hi : lo;
        v[e | (1 << q)] = desc ? lo : hi;
      }
    }
  }
  // Key-value CE: keys as ce<B>; the payload follows its key.  The swap
  // happens only when strictly out of order (compare_exchange,
  // engine.cpp:16-22), so equal keys keep their payloads in place -- the
  // reference network's own payload order.
  template <int B>
  __device__ __forceinline__ static void ce_kv(uint32_t (&v)[NR], uint32_t (&w)[NR],
                                               FmaSplit fs) {
    constexpr int q = qof(B);
    static_assert(q >= 0, "CE bit must be a register bit");
#pragma unroll
    for (int e = 0; e < NR; ++e) {
      if (!(e & (1 << q))) {
        const int f = e | (1 << q);
        const int idx = (e & ((1 << q) - 1)) | ((e >> (q + 1)) << q);
        const uint32_t x = v[e], y = v[f];
        const bool sw = x > y;
        mm<B200_FMA_NUM, B200_FMA_DEN>(idx, x, y, v[e], v[f], fs);
        const uint32_t a = w[e], b = w[f];
        w[e] = sw ? b : a;
        w[f] = sw ? a : b;
      }
    }
  }
  template <int B, int D>
  __device__ __forceinline__ static void ce_dir_kv(uint32_t (&v)[NR], uint32_t (&w)[NR],
                                                   FmaSplit fs) {
    constexpr int q = qof(B);
    constexpr int qd = qof(D);
    static_assert(q >= 0 && qd >= 0, "CE and direction bits must be register bits");
#pragma unroll
    for (int e = 0; e < NR; ++e) {
      if (!(e & (1 << q))) {
        const int f = e | (1 << q);
        const int idx = (e & ((1 << q) - 1)) | ((e >> (q + 1)) << q);
        const uint32_t x = v[e], y = v[f];
        const bool desc = (e >> qd) & 1;
        const bool sw = desc ? (x < y) : (x > y);
        uint32_t lo, hi;
        mm<B200_FMA_NUM, B200_FMA_DEN>(idx, x, y, lo, hi, fs);
        v[e] = desc ? hi : lo;
        v[f] = desc ? lo : hi;
        const uint32_t a = w[e], b = w[f];
        w[e] = sw ? b : a;
        w[f] = sw ? a : b;
      }
    }
  }
  // 64-bit keys held as (hi word in v, lo word in w): lexicographic CE,
  // swap only when strictly out of order.
  template <int B>
  __device__ __forceinline__ static void ce_k64(uint32_t (&v)[NR], uint32_t (&w)[NR],
                                                FmaSplit fs) {
    constexpr int q = qof(B);
    static_assert(q >= 0, "CE bit must be a register bit");
#pragma unroll
    for (int e = 0; e < NR; ++e) {
      if (!(e & (1 << q))) {
        const int f = e | (1 << q);
        const int idx = (e & ((1 << q) - 1)) | ((e >> (q + 1)) << q);
        // x > y implies hi(x) >= hi(y): the high words are a plain min/max,
        // only the low words follow the 64-bit predicate.
        const uint64_t x = ((uint64_t)v[e] << 32) | w[e];
        const uint64_t y = ((uint64_t)v[f] << 32) | w[f];
        const bool sw = x > y;
        const uint32_t a = w[e], b = w[f];
        uint32_t h0, h1;
        mm<B200_FMA_NUM, B200_FMA_DEN>(idx, v[e], v[f], h0, h1, fs);
        v[e] = h0;
        v[f] = h1;
        w[e] = sw ? b : a;
        w[f] = sw ? a : b;
      }
    }
  }
  template <int B, int D>
  __device__ __forceinline__ static void ce_dir_k64(uint32_t (&v)[NR], uint32_t (&w)[NR],
                                                    FmaSplit fs) {
    constexpr int q = qof(B);
    constexpr int qd = qof(D);
    static_assert(q >= 0 && qd >= 0, "CE and direction bits must be register bits");
#pragma unroll
    for (int e = 0; e < NR; ++e) {
      if (!(e & (1 << q))) {
        const int f = e | (1 << q);
        const int idx = (e & ((1 << q) - 1)) | ((e >> (q + 1)) << q);
        const uint64_t x = ((uint64_t)v[e] << 32) | w[e];
        const uint64_t y = ((uint64_t)v[f] << 32) | w[f];
        const bool desc = (e >> qd) & 1;
        const bool sw = desc ? (x < y) : (x > y);
        const uint32_t a = w[e], b = w[f];
        uint32_t h0, h1;
        mm<B200_FMA_NUM, B200_FMA_DEN>(idx, v[e], v[f], h0, h1, fs);
        v[e] = desc ? h1 : h0;
        v[f] = desc ? h0 : h1;
        w[e] = sw ? b : a;
        w[f] = sw ? a : b;
      }
    }
  }
  // XOR register e with all-ones when bit LB of its local index is set
  // (LB a register bit) -- or with the per-thread uniform u when LB is a
  // thread bit -- or with u when LB < 0 (uniform source).
  template <int LB>
  __device__ __forceinline__ static uint32_t dmask_e(int e, uint32_t u) {
    if constexpr (LB >= 0 && qof(LB) >= 0) {
      return ((e >> qof(LB)) & 1) ? 0xFFFFFFFFu : 0u;
    } else {
      return u;
    }
  }
};

}  // namespace b200
