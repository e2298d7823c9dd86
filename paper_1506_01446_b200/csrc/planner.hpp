// planner.hpp -- host-side pass planner for the bitonic network.
//
// Generalises the reference's build_plan (proj/src/engine.cpp:86-145).  The
// reference packs the schedule (generate_schedule, schedule.cpp:20-36: phase
// p = 1..k, steps on bits p-1..0) into launches of three fixed kinds: one
// step, two paired steps, or the block-local tail of one phase.  Here a
// launch ("pass") may cover ANY run of consecutive steps whose bits fit in a
// C-bit coset S = [0,a) U [y, y+C-a) of the index space, so one HBM round
// trip covers up to C steps:
//   * pass 0 (tile sort): phases 1..C of every 2^C tile;
//   * merge passes, greedily: the tail of phase p (bits b..0, all < C) fused
//     with the head of phase p+1 (bits p..p-h+1), or, when a phase has too
//     many bits, a middle run of h = C - lrun high bits.
// Every pass keeps at least 2^lrun contiguous keys per run (lrun >= 2 so the
// kernels use 128-bit accesses; 5 = one 128 B line).  Concatenating the
// passes' steps reproduces the schedule's step order exactly -- the same
// invariant the reference tests for its plans (test_engine.cpp:99-118) -- and
// the CE total equals predicted_counts (schedule.cpp:71-78).
#pragma once

#include <algorithm>
#include <cstdint>
#include <functional>
#include <stdexcept>
#include <string>
#include <vector>

namespace b200 {

struct PlanPass {
  int C = 0;          // tile bits
  int a = 0, y = 0;   // coset shape
  int tile_sort = 0;  // phases 1..p_end in one tile
  int p_end = 0;      // last phase of a tile-sort pass
  int segA_hi = -1, pA = 0;
  int segB_lo = -1, pB = 0;
  uint64_t ctas = 0;
  uint64_t ces = 0;
  int R = 5;          // log2 keys per thread (5 = 32; 4 = 16 for latency-bound sizes)
  int cluster = 0;    // 1: 2-CTA cluster pass on a 2^15-key coset (bitonic_cluster.cuh)
};

// ---- cost model: shared-memory round trips of one merge pass ---------------
// Mirrors the kernels' compile-time round cutting (bitonic_rounds.cuh:
// Rounds, Layout::lanes_low; bitonic_static.cuh: PassBody::smem_trips) so
// the planner can prefer pass shapes that load/store HBM directly.
namespace detail {

inline int popcount32(uint32_t x) {
  int c = 0;
  while (x) {
    c += x & 1u;
    x >>= 1;
  }
  return c;
}

inline bool lanes_feasible(int C, uint32_t m) {
  for (int r = 0; r < 5; ++r) {
    bool ok = false;
    for (int p = r; p < C; p += 5)
      if (!(m & (1u << p))) ok = true;
    if (!ok) return false;
  }
  return true;
}

inline std::vector<uint32_t> cut_rounds(const std::vector<int>& bits, int C, int R, int A,
                                        bool DF) {
  const bool enforce = C >= 10 && C - R >= 5;
  std::vector<uint32_t> masks;
  size_t i = 0;
  while (i < bits.size()) {
    uint32_t m = 0;
    const size_t b = i;
    while (i < bits.size()) {
      const uint32_t nm = m | (1u << bits[i]);
      if (popcount32(nm) > R) break;
      if (enforce && !lanes_feasible(C, nm)) break;
      if (DF && b == 0 && i > 0 && bits[i] < 5) break;
      m = nm;
      ++i;
    }
    for (int x = A - 1; x >= 5 && popcount32(m) < R; --x) {
      if (m & (1u << x)) continue;
      if (enforce && !lanes_feasible(C, m | (1u << x))) continue;
      m |= 1u << x;
    }
    for (int x = C - 1; x >= 0 && popcount32(m) < R; --x) {
      if (m & (1u << x)) continue;
      if (enforce && !lanes_feasible(C, m | (1u << x))) continue;
      m |= 1u << x;
    }
    masks.push_back(m);
  }
  return masks;
}

inline bool direct(int C, int R, int A, uint32_t m) {
  int v = 0;
  while (v < C && (m & (1u << v))) ++v;
  if (C - R < 5 || v > 2 || v + 5 > C) return false;
  for (int b = v; b < v + 5; ++b)
    if (m & (1u << b)) return false;
  return A >= v + 5;
}

// Shared-memory round trips of merge pass (SA, SB) on a 2^C tile (low run
// of A keys: SB when a head follows, else C, unless given).
inline int merge_trips(int C, int R, int SA, int SB, int A_override = -1) {
  const int A = A_override >= 0 ? A_override : (SB >= 0 ? SB : C);
  std::vector<int> bits;
  for (int b = SA; b >= 0; --b) bits.push_back(b);
  if (SB >= 0)
    for (int b = C - 1; b >= SB; --b) bits.push_back(b);
  int best = 1 << 20;
  for (bool df : {false, true}) {
    const auto m = cut_rounds(bits, C, R, A, df);
    const int t = (int)m.size() - 1 + (direct(C, R, A, m.front()) ? 0 : 1) +
                  (direct(C, R, A, m.back()) ? 0 : 1);
    if (t < best) best = t;
  }
  return best;
}

}  // namespace detail

struct PlanOptions {
  int cmax = 15;   // largest tile (2^cmax keys per CTA)
  int lrun = 5;    // min contiguous run per merge pass (2^lrun keys)
  int min_ctas = 128;  // shrink the tile until the grid has this many CTAs
  int cmin = 6;    // ... but not below this tile size
  int regbits = 0; // keys per thread = 2^regbits (0 = automatic)
  int tile_regbits = 0;  // override for the tile-sort pass only (0 = same)
  bool dp = true;  // cost-model planner (false: greedy packing)
  bool kv = false; // key-value plan: 16 pairs per thread, 2^12 / 2^13 tiles
  int cmerge = 0;  // merge-pass coset size when it differs from the tile (0 = auto)
  bool mixed_c = true;         // choose the coset size per merge pass (tile's or cmerge)
  double wide_tail_cost = -1;  // extra cost of a tail pass on the larger cosets (<0: auto)
  double trip_cost = 0.10;  // extra cost of a shared-memory round trip, in passes
  // 2-CTA cluster passes (tail of phase p + head of p+1 on a 2^15-key coset,
  // bitonic_cluster.cuh) for single-array key-only sorts of >= 2^cluster_min_k.
  // Off by default: measured on B200 (tools/pass_times.py, 2^28) a cluster
  // pass takes 530-600 us against 325-415 us for the 14-bit passes it
  // replaces -- the DSMEM exchange (~17 B/clk/SM) and the two cluster
  // barriers cost more than the HBM round trip they save (12.7 vs 11.1 ms).
  bool cluster = false;
  int cluster_min_k = 24;
  double cluster_cost = 0.05;  // the DSMEM exchange, in passes
  int mid_lrun = 5;            // shortest run of a middle pass (k >= 24 plans)
  int regbits14 = 0;           // keys per thread of the 14-bit merge passes (0 = as R)
  int tile_c = 0;              // tile-sort size for single arrays (0 = per-size default)
  bool virt = false;           // virtual-padding plan: 2^13-key cosets only, 32 keys/thread
};

inline int ctz64(uint64_t x) {
  int r = 0;
  while (!(x & 1ull)) {
    x >>= 1;
    ++r;
  }
  return r;
}

// One entry per steps-run, in execution order.  k = log2(keys per array),
// batch = number of contiguous arrays (each sorted independently).
inline std::vector<PlanPass> make_plan(int k, uint64_t batch,
                                       const PlanOptions& opt) {
  if (k < 1 || k > 40) throw std::invalid_argument("k out of range");
  if (batch < 1) throw std::invalid_argument("batch must be >= 1");
  const uint64_t total = batch << k;
  const int kt = k + ctz64(batch);  // tiles must divide the whole buffer
  std::vector<PlanPass> plan;

  // Tile size.  With an explicit tuning (cmin == cmax) use it; otherwise the
  // per-size choice measured best on B200 (PDL between passes):
  //   k <= 12  one CTA sorts the whole array (single launch)
  //   13..22   2^12-key tiles: the passes are latency-bound (L2-resident
  //            data), so more, smaller CTAs per SM win over fewer passes
  //   >= 23    2^13-key tiles: four CTAs per SM keep the HBM-bound merge
  //            passes streaming (2^14-key tiles need fewer passes but fit
  //            only two CTAs per SM and measured slower: 12.3 vs 12.0 ms at
  //            2^28)
  int C;
  if (opt.cmin == opt.cmax) {
    C = opt.cmax;
  } else if (k <= 12) {
    C = k;
  } else if (k <= 22) {
    C = 12;
  } else {
    C = 13;
  }
  if (opt.tile_c > 0 && opt.cmin != opt.cmax && batch == 1 && k > opt.tile_c) C = opt.tile_c;
  if (opt.virt) {
    // the virtual-padding kernels exist for 2^13-key tiles and cosets only
    if (k < 14 || batch != 1 || opt.kv) throw std::invalid_argument("virtual plan needs k >= 14");
    C = 13;
  }
  if (C > opt.cmax) C = opt.cmax > k ? k : opt.cmax;
  if (batch > 1) {
    // Batched arrays of >= 2^8 keys: one array per CTA (the specialised
    // tile sort runs exactly phases 1..C); smaller arrays share a tile.
    if (k >= 8 && k <= 15) C = k;
    else if (k < 8) C = opt.cmax;
    while (C > k && C > opt.cmin && (total >> C) < (uint64_t)opt.min_ctas) --C;
  }
  if (C > kt) C = kt;
  if (opt.kv) {
    // key-value kernels exist for tiles up to 2^13 and merges on 2^12 / 2^13
    if (C > 13) C = 13;
    if (k > C && C < 12) C = 12;
    if (C > kt) C = kt;
  }
  // Merge passes need a coalescing run below the high range and a phase
  // direction bit that is per-thread uniform in layout L_0 (C - 1 >= 5).
  if (k > C && C < opt.lrun + 1) C = opt.lrun + 1;
  if (k > C && C < 6) C = 6;
  if (C > kt) C = kt;

  PlanPass t;
  t.C = C;
  t.a = C;
  t.y = C;
  t.tile_sort = 1;
  t.p_end = k < C ? k : C;
  t.ctas = total >> C;
  t.ces = (total / 2) * (uint64_t)(t.p_end * (t.p_end + 1) / 2);
  plan.push_back(t);
  // 16 keys per thread (twice the warps per SM) up to 2^21 keys, where the
  // passes are latency-bound, and for batched tiles (ALU-bound: more warps
  // overlap the shared-memory rounds); 32 keys per thread elsewhere
  // (measured on B200).
  int R = opt.regbits > 0 ? opt.regbits
                          : ((k <= 21 && batch == 1) || (batch > 1 && C >= 10 && C <= 14) ? 4 : 5);
  if (opt.virt) R = 5;
  if (opt.kv) R = C < 4 ? C : 4;
  for (auto& q : plan) q.R = R;
  if (opt.tile_regbits > 0 && !opt.kv) plan.front().R = opt.tile_regbits;
  if (k <= C) return plan;

  // Merge passes may use larger cosets than the tile sort: the tile sort is
  // ALU-bound (smaller tiles do fewer steps per key), the merge passes are
  // HBM-bound (larger cosets need fewer passes).
  // Measured on B200 (13-bit tile + 14-bit merges vs 13/13): 2^26 2.50 vs
  // 2.57 ms, 2^28 equal, 2^30 54.4 vs 56.6 ms; 2^24 prefers 13/13.  With the
  // coset size chosen per pass (mixed_c: 14-bit middle passes, 13-bit tail
  // passes where the wide ones are register-limited): 2^24 0.471 (vs 0.481),
  // 2^25 1.157, 2^26 2.405, 2^28 10.97, 2^30 52.9 ms.
  const int CT = C;
  int cm = opt.cmerge;
  if (cm == 0 && opt.cmin != opt.cmax && k >= 24) cm = 14;
  if (opt.virt) cm = 13;
  // (cm <= C + 2: the first merge state, phase C+1 from bit C, must have its
  // direction bit at or above local bit cm-1 -- see the tail-only / tail+head
  // rules in the DP below.)
  if (cm > C && cm <= C + 2 && cm <= 15 && cm <= kt && !opt.kv && batch == 1) {
    C = cm;
    // 16 keys per thread stays for the latency-bound sizes (16-key merge
    // kernels exist for 2^12- and 2^13-key cosets); 32 elsewhere
    R = opt.regbits > 0 ? opt.regbits : (R == 4 && C <= 13 ? 4 : 5);
  }
  const int lrun = opt.lrun;
  auto push_tail_head = [&](int p, int b, int h) {
    PlanPass m;
    m.C = C;
    m.R = (C == 14 && opt.regbits14 > 0) ? opt.regbits14 : R;
    m.ctas = total >> C;
    m.segA_hi = b;
    m.pA = p;
    if (h > 0) {
      m.a = C - h;
      m.y = p - h + 1;
      m.segB_lo = m.a;
      m.pB = p + 1;
      m.ces = (total / 2) * (uint64_t)((b + 1) + h);
    } else {
      m.a = C;
      m.y = C;
      m.ces = (total / 2) * (uint64_t)(b + 1);
    }
    plan.push_back(m);
  };
  auto push_middle = [&](int p, int b, int h) {
    PlanPass m;
    m.C = C;
    m.R = (C == 14 && opt.regbits14 > 0) ? opt.regbits14 : R;
    m.ctas = total >> C;
    m.a = C - h;
    m.y = b - h + 1;
    m.segB_lo = m.a;
    m.pB = p;
    m.ces = (total / 2) * (uint64_t)h;
    plan.push_back(m);
  };

  if (opt.dp || opt.kv) {
    // Dynamic program over (phase p, next step bit b): each pass costs 1 plus
    // trip_cost per extra shared-memory round trip; shapes are restricted to
    // the instantiated kernel families (tail-only, tail+head with a = b+1,
    // middle runs of h high bits).  With opt.mixed_c every pass may instead
    // use the tile's coset size (CT) or the merge coset size (C); the larger
    // cosets' tail passes are charged opt.wide_tail_cost more (they run at 2
    // CTAs per SM, measured on B200).
    const int K = k + 2;
    std::vector<double> best((size_t)K * K, -1.0);
    std::vector<int> choice((size_t)K * K, 0);  // 0 tail-only, >0 tail+head h, <0 middle -h
    std::vector<int> choice_c((size_t)K * K, C);
    std::vector<char> choice_cl((size_t)K * K, 0);
    const bool use_cluster = opt.cluster && !opt.virt && !opt.kv && batch == 1 && k >= opt.cluster_min_k &&
                             C >= 14 && !(opt.cmin == opt.cmax);
    const int mid_lrun = (!opt.kv && !opt.virt && batch == 1 && k >= opt.cluster_min_k &&
                          !(opt.cmin == opt.cmax)) ? std::min(opt.mid_lrun, lrun) : lrun;
    std::vector<int> cands = {C};
    if (opt.mixed_c && CT < C && CT >= 12)
      for (int c = C - 1; c >= CT; --c) cands.push_back(c);
    if (opt.mixed_c && CT == C && C == 14 && opt.tile_c == 14) cands.push_back(13);
    // measured best on B200: 0.3 up to 2^26 keys, 0.2 for 2^27..2^28, 0.1 above
    const double wide_tail = opt.wide_tail_cost >= 0 ? opt.wide_tail_cost
                             : (k <= 26 ? 0.3 : (k <= 28 ? 0.2 : 0.1));
    auto cost_of = [&](int Cc, int SA, int SB) {
      double c = 1.0 + opt.trip_cost * (detail::merge_trips(Cc, R, SA, SB) - 1);
      // (wide tail passes run fewer CTAs per SM: charged against the tile's
      // coset size; with a 14-bit tile, against the 13-bit alternative)
      if (SA >= 0) {
        if (Cc > CT) c += wide_tail * (Cc - CT);
        else if (opt.tile_c == 14 && Cc == 14) c += wide_tail;
      }
      return c;
    };
    std::function<double(int, int)> solve = [&](int p, int b) -> double {
      if (p > k) return 0.0;
      double& memo = best[(size_t)p * K + b];
      if (memo >= 0) return memo;
      double bc = 1e30;
      int bch = 0, bcc = C;
      bool bcl = false;
      if (use_cluster && b >= 4 && b <= 13 && b + 1 >= lrun && p >= 14 && p < k) {
        // cluster pass: tail bits b..0 on [0,b+1) U (13-b high bits), DSMEM
        // exchange, head bits 13..b on [0,b) U (14-b high bits)
        const int h = 14 - b;
        const int trips = detail::merge_trips(14, R, b, -1, b + 1) +
                          detail::merge_trips(14, R, -1, b) + 1;
        const double t = 1.0 + opt.cluster_cost + opt.trip_cost * (trips - 1) +
                         solve(p + 1, p - h);
        if (t < bc - 1e-9) {
          bc = t;
          bch = h;
          bcc = 15;
          bcl = true;
        }
      }
      for (int Cc : cands) {
        if (b < Cc) {
          // A tail-only pass takes phase p's direction as CTA-uniform: valid
          // only when bit p lies above the coset (p >= Cc; after a smaller
          // tile sort, p < Cc happens and the tail must be fused with a head).
          if (p >= Cc) {
            const double t0 = cost_of(Cc, b, -1) + solve(p + 1, p);
            if (t0 < bc - 1e-9) {
              bc = t0;
              bch = 0;
              bcc = Cc;
              bcl = false;
            }
          }
          const int h = Cc - (b + 1);
          // tail+head: phase p's direction bit must be the coset's top local
          // bit Cc-1 (p >= Cc-1), which also keeps the head above the tail
          if (p < k && p >= Cc - 1 && b + 1 >= lrun && h >= 1) {
            const double t1 = cost_of(Cc, b, b + 1) + solve(p + 1, p - h);
            if (t1 < bc - 1e-9) {
              bc = t1;
              bch = h;
              bcc = Cc;
              bcl = false;
            }
          }
        } else {
          for (int h = 1; h <= Cc - mid_lrun && h <= b; ++h) {
            const double t = cost_of(Cc, -1, Cc - h) + solve(p, b - h);
            if (t < bc - 1e-9) {
              bc = t;
              bch = -h;
              bcc = Cc;
              bcl = false;
            }
          }
        }
      }
      choice[(size_t)p * K + b] = bch;
      choice_c[(size_t)p * K + b] = bcc;
      choice_cl[(size_t)p * K + b] = bcl ? 1 : 0;
      memo = bc;
      return bc;
    };
    solve(CT + 1, CT);
    int p = CT + 1, b = CT;
    const int Cmax = C;
    while (p <= k) {
      const int ch = choice[(size_t)p * K + b];
      C = choice_c[(size_t)p * K + b];  // the push helpers read C
      if (choice_cl[(size_t)p * K + b]) {
        push_tail_head(p, b, ch);  // C = 15: a = b+1, y = p-h+1
        plan.back().cluster = 1;
        plan.back().ctas = total >> 14;
        plan.back().R = 5;
        b = p - ch;
        p = p + 1;
      } else if (b < C) {
        push_tail_head(p, b, ch);
        if (ch > 0) {
          b = p - ch;
          p = p + 1;
        } else {
          p = p + 1;
          b = p - 1;
        }
      } else {
        push_middle(p, b, -ch);
        b -= -ch;
      }
    }
    C = Cmax;
    return plan;
  }

  int p = CT + 1;  // current phase
  int b = CT;      // next step bit of phase p (steps run b, b-1, ..., 0)
  while (p <= k) {
    if (b < C) {
      // Tail of phase p fits in the low bits: fuse the head of phase p+1.
      const int low = (b + 1 > lrun) ? b + 1 : lrun;
      int h = C - low;
      if (p == k && p >= C) h = 0;
      push_tail_head(p, b, h > 0 ? h : 0);
      if (h > 0) {
        b = p - h;  // next step bit of phase p+1
        p = p + 1;
      } else {
        p = p + 1;
        b = p - 1;
      }
    } else {
      // Middle of phase p: h high bits b..b-h+1 plus a coalescing run.
      int h = C - lrun;
      if (h > b) h = b;
      push_middle(p, b, h);
      b -= h;
    }
  }
  return plan;
}

}  // namespace b200
