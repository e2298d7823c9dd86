// check_sync.cu -- host-side proof obligations for the kernels' shared-memory
// synchronisation and coset partitioning (compiled by nvcc, runs on the CPU;
// the analogue of the reference's static disjointness check,
// proj/tests/test_engine.cpp:395-437, for the B200 pass structure).
//
// For every instantiated pass shape (tile sorts, merge tables of 11..15-bit
// cosets with 16 and 32 keys per thread, the 2-CTA cluster passes):
//   1. every round layout maps (thread, register) -> local index bijectively,
//      and distinct indices get distinct padded shared-memory words: a
//      thread's STS in layout L writes exactly the words it read with LDS in
//      L, so no other thread touches them within a round (no barrier needed
//      between a round's LDS and its STS);
//   2. every layout transition the engine orders with __syncwarp only
//      (same_warp_bits) keeps each warp's word set: warp w reads in L<r>
//      exactly the words warp w wrote in L<r-1>, so no cross-warp data flow
//      is left unsynchronised;
//   3. every layout and the staging copies are bank-conflict free;
//   4. the cluster pass's DSMEM exchange reads every key written by the two
//      CTAs exactly once;
// and for every plan of k = 1..21 keys (batches of 3 and 8 up to k = 15,
// four tunings):
//   5. each pass's CTA cosets partition the index space (every key belongs
//      to exactly one CTA), and the passes' steps concatenate to the schedule.
// Exit code 0 and "OK" when every check holds.
#include <algorithm>
#include <cstdio>
#include <utility>
#include <vector>

#include "../../paper_1506_01446_b200/csrc/bitonic_cluster.cuh"
#include "../../paper_1506_01446_b200/csrc/planner.hpp"

using namespace b200;

static int failures = 0;
static long checks = 0;
#define EXPECT(cond, ...)                    \
  do {                                       \
    ++checks;                                \
    if (!(cond)) {                           \
      if (++failures < 20) {                 \
        std::printf("FAIL %s:%d ", __FILE__, __LINE__); \
        std::printf(__VA_ARGS__);            \
        std::printf("\n");                   \
      }                                      \
    }                                        \
  } while (0)

template <class L, int C>
void check_layout(const char* what) {
  constexpr int NT = 1 << L::NT;
  constexpr int NR = L::NR;
  std::vector<unsigned char> seen(1u << C, 0), word(smem_pad((1u << C) - 1u) + 1u, 0);
  for (uint32_t t = 0; t < (uint32_t)NT; ++t)
    for (int e = 0; e < NR; ++e) {
      const uint32_t j = L::dep_thr(t) | L::dep_reg(e);
      EXPECT(j < (1u << C) && (L::dep_thr(t) & L::dep_reg(e)) == 0, "%s: index out of range", what);
      if (j >= (1u << C)) continue;
      EXPECT(seen[j] == 0, "%s: index %u held twice", what, j);
      seen[j] = 1;
      const uint32_t wd = smem_pad(L::dep_thr(t)) + smem_pad(L::dep_reg(e));
      EXPECT(wd == smem_pad(j), "%s: padding not additive at %u", what, j);
      EXPECT(word[wd] == 0, "%s: word %u shared", what, wd);
      word[wd] = 1;
    }
  if (C >= 10) {
    EXPECT(L::conflict_free(), "%s: bank conflicts", what);
  }
}

template <class LA, class LB, int C>
void check_warp_transition(const char* what) {
  if (!same_warp_bits<LA, LB>()) return;
  constexpr int NT = 1 << LA::NT;
  const int warps = NT >= 32 ? NT / 32 : 1;
  const int lanes = NT >= 32 ? 32 : NT;
  for (int w = 0; w < warps; ++w) {
    std::vector<uint32_t> a, b;
    for (int l = 0; l < lanes; ++l) {
      const uint32_t t = (uint32_t)(w * 32 + l);
      for (int e = 0; e < LA::NR; ++e) a.push_back(LA::dep_thr(t) | LA::dep_reg(e));
      for (int e = 0; e < LB::NR; ++e) b.push_back(LB::dep_thr(t) | LB::dep_reg(e));
    }
    std::sort(a.begin(), a.end());
    std::sort(b.begin(), b.end());
    EXPECT(a == b, "%s: __syncwarp transition moves keys between warps (warp %d)", what, w);
  }
}

template <class B, int C, int r>
void check_rounds(const char* what) {
  if constexpr (r < B::NRND) {
    check_layout<typename B::template L<r>, C>(what);
    if constexpr (r > 0)
      check_warp_transition<typename B::template L<r - 1>, typename B::template L<r>, C>(what);
    check_rounds<B, C, r + 1>(what);
  }
}

template <int C, int KIND, int SA, int SB, int R, int AO = -1>
void check_body() {
  using B = PassBody<C, KIND, SA, SB, R, 0, AO>;
  char what[96];
  std::snprintf(what, sizeof what, "PassBody<C=%d,%s,SA=%d,SB=%d,R=%d>", C,
                KIND == 0 ? "tile" : "merge", SA, SB, R);
  check_rounds<B, C, 0>(what);
  EXPECT((staging_conflict_free<C, R>()), "%s: staging bank conflicts", what);
}

template <int C, int R, int I>
void check_shape() {
  // th: SA = A-1, SB = A; ho: SB = A; to: SA (the three tables of merge_table.cuh)
  if constexpr (I >= 2 && I <= C - 1) {
    check_body<C, 1, I - 1, I, R>();
    check_body<C, 1, -1, I, R>();
  }
  if constexpr (I <= C - 1) check_body<C, 1, I, -1, R>();
}

template <int C, int R, int... I>
void check_merge_family(std::integer_sequence<int, I...>) {
  (check_shape<C, R, I>(), ...);
}

template <int B>
void check_cluster() {
  using P = ClusterPass<B, 5>;
  check_body<14, 1, B, -1, 5, B + 1>();
  check_body<14, 1, -1, B, 5, B>();
  // every key written by CTA c in part 1 (index j, coset bit 14 = c) is read
  // exactly once in part 2 by the CTA owning its coset bit B
  using L = typename P::B2::template L<0>;
  std::vector<unsigned char> got(2u << 14, 0);
  for (uint32_t c = 0; c < 2; ++c)
    for (uint32_t t = 0; t < (1u << L::NT); ++t)
      for (int e = 0; e < L::NR; ++e) {
        const uint32_t jp = L::dep_thr(t) | L::dep_reg(e);
        const uint32_t owner = (jp >> 13) & 1u;
        const uint32_t j = xmap<B>(jp & 0x1FFFu) | (c << B);
        const uint32_t slot = (owner << 14) | j;
        EXPECT(got[slot] == 0, "cluster<%d>: key read twice", B);
        got[slot] = 1;
      }
  for (uint32_t s = 0; s < (2u << 14); ++s) EXPECT(got[s] == 1, "cluster<%d>: key %u lost", B, s);
}

template <int I>
void check_cluster_if() {
  if constexpr (I >= 4) check_cluster<I>();
}
template <int... I>
void check_clusters(std::integer_sequence<int, I...>) {
  (check_cluster_if<I>(), ...);
}

// ---- coset partitions of real plans -------------------------------------------
template <int C, int A>
uint64_t gidx(uint64_t b, uint32_t j, int y) {
  return Coset<C, A>::base(b, y) + Coset<C, A>::goff(j, y);
}

template <int C>
uint64_t gidx_rt(int a, uint64_t b, uint32_t j, int y) {
  switch (a) {
#define CASE(AA) \
  case AA: return gidx<C, (AA <= C ? AA : C)>(b, j, y);
    CASE(1) CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7) CASE(8) CASE(9) CASE(10)
    CASE(11) CASE(12) CASE(13) CASE(14) CASE(15)
#undef CASE
    default: return ~0ull;
  }
}

uint64_t gidx_any(int C, int a, uint64_t b, uint32_t j, int y) {
  switch (C) {
#define CC(X) \
  case X: return gidx_rt<X>(a, b, j, y);
    CC(1) CC(2) CC(3) CC(4) CC(5) CC(6) CC(7) CC(8) CC(9) CC(10) CC(11) CC(12) CC(13) CC(14) CC(15)
#undef CC
    default: return ~0ull;
  }
}

void check_plans() {
  for (int k = 1; k <= 21; ++k)
    for (uint64_t batch : {1ull, 3ull, 8ull}) {
      if (batch > 1 && k > 15) continue;
      for (int tile : {0, 7, 10, 13}) {
        PlanOptions o;
        if (tile) o.cmin = o.cmax = tile;
        const auto plan = make_plan(k, batch, o);
        const uint64_t total = batch << k;
        std::vector<std::pair<int, int>> steps;
        for (const auto& q : plan) {
          const int C = q.C, a = q.tile_sort ? q.C : q.a;
          std::vector<unsigned char> seen(total, 0);
          const uint64_t cosets = total >> C;
          for (uint64_t b = 0; b < cosets; ++b)
            for (uint32_t j = 0; j < (1u << C); ++j) {
              const uint64_t g = q.tile_sort ? ((b << C) + j) : gidx_any(C, a, b, j, q.y);
              EXPECT(g < total, "k=%d pass C=%d a=%d y=%d: index outside the array", k, C, a, q.y);
              if (g >= total) continue;
              EXPECT(seen[g] == 0, "k=%d pass C=%d a=%d y=%d: key in two cosets", k, C, a, q.y);
              seen[g] = 1;
            }
          if (q.tile_sort) {
            for (int p = 1; p <= q.p_end; ++p)
              for (int bb = p - 1; bb >= 0; --bb) steps.push_back({p, bb});
          } else {
            auto glob = [&](int l) { return l < q.a ? l : q.y + (l - q.a); };
            for (int l = q.segA_hi; l >= 0; --l) steps.push_back({q.pA, glob(l)});
            if (q.segB_lo >= 0)
              for (int l = C - 1; l >= q.segB_lo; --l) steps.push_back({q.pB, glob(l)});
          }
        }
        std::vector<std::pair<int, int>> want;
        for (int p = 1; p <= k; ++p)
          for (int bb = p - 1; bb >= 0; --bb) want.push_back({p, bb});
        EXPECT(steps == want, "k=%d batch=%llu tile=%d: steps differ from the schedule", k,
               (unsigned long long)batch, tile);
      }
    }
}

int main() {
  // tile sorts
  check_body<8, 0, -1, -1, 5>();
  check_body<10, 0, -1, -1, 4>();
  check_body<10, 0, -1, -1, 5>();
  check_body<11, 0, -1, -1, 4>();
  check_body<11, 0, -1, -1, 5>();
  check_body<12, 0, -1, -1, 4>();
  check_body<12, 0, -1, -1, 5>();
  check_body<13, 0, -1, -1, 4>();
  check_body<13, 0, -1, -1, 5>();
  check_body<14, 0, -1, -1, 5>();
  check_body<15, 0, -1, -1, 5>();
  // merge tables (merge_table.cuh), 32 and 16 keys per thread
  check_merge_family<11, 5>(std::make_integer_sequence<int, 16>{});
  check_merge_family<12, 5>(std::make_integer_sequence<int, 16>{});
  check_merge_family<13, 5>(std::make_integer_sequence<int, 16>{});
  check_merge_family<14, 5>(std::make_integer_sequence<int, 16>{});
  check_merge_family<15, 5>(std::make_integer_sequence<int, 16>{});
  check_merge_family<12, 4>(std::make_integer_sequence<int, 16>{});
  check_merge_family<13, 4>(std::make_integer_sequence<int, 16>{});
  check_merge_family<14, 4>(std::make_integer_sequence<int, 16>{});
  check_clusters(std::make_integer_sequence<int, 14>{});
  check_plans();
  std::printf("%s: %ld checks, %d failures\n", failures ? "FAILED" : "OK", checks, failures);
  return failures ? 1 : 0;
}
