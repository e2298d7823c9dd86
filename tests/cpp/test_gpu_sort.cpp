// C++ shim test (run by tests/test_cpp_shim.py on a GPU box).  Mirrors the
// reference's own test shapes for the sort entry point:
//   test_engine.cpp:217-227  canonical bitonic sequence
//   test_engine.cpp:229-235  sorted input (with negatives) is a fixed point
//   test_engine.cpp:237-253  random arrays vs the reference quicksort
//   test_engine.cpp:439-449  sequential sort agrees; odd length throws
#include <algorithm>
#include <cstdio>
#include <cstdint>
#include <functional>
#include <numeric>
#include <random>
#include <vector>

#include "bitonic/gpu_sort.hpp"

static int failures = 0;
#define CHECK(c)                                                   \
  do {                                                             \
    if (!(c)) {                                                    \
      std::printf("FAIL %s:%d %s\n", __FILE__, __LINE__, #c);      \
      ++failures;                                                  \
    }                                                              \
  } while (0)
#define CHECK_THROWS_AS(expr, T)                                   \
  do {                                                             \
    bool thrown = false;                                           \
    try {                                                          \
      expr;                                                        \
    } catch (const T&) {                                           \
      thrown = true;                                               \
    } catch (...) {                                                \
    }                                                              \
    CHECK(thrown);                                                 \
  } while (0)

int main() {
  using bitonic::gpu::sequential_bitonic_sort;
  using bitonic::gpu::sort;
  {
    std::vector<std::int32_t> keys = {1, 5, 9, 10, 12, 8, 7, 2};
    sequential_bitonic_sort(keys);
    CHECK((keys == std::vector<std::int32_t>{1, 2, 5, 7, 8, 9, 10, 12}));
  }
  {
    std::vector<std::int32_t> keys(64);
    std::iota(keys.begin(), keys.end(), -12);
    const auto copy = keys;
    sequential_bitonic_sort(keys);
    CHECK(keys == copy);
  }
  std::mt19937_64 rng(1000);
  for (unsigned k = 1; k <= 22; ++k) {
    std::vector<std::int32_t> keys(std::size_t{1} << k);
    for (auto& v : keys) v = static_cast<std::int32_t>(static_cast<std::uint32_t>(rng()));
    auto expected = keys;
    std::sort(expected.begin(), expected.end());
    auto desc = keys;
    sort(keys);
    CHECK(keys == expected);
    sort(std::span<std::int32_t>(desc), /*ascending=*/false);
    std::reverse(expected.begin(), expected.end());
    CHECK(desc == expected);
    std::vector<std::uint32_t> u(keys.size());
    for (auto& v : u) v = static_cast<std::uint32_t>(rng());
    auto ue = u;
    std::sort(ue.begin(), ue.end());
    sort(std::span<std::uint32_t>(u));
    CHECK(u == ue);
  }
  {
    // execute(plan, keys, workers) shape (engine.hpp:86-92, test_engine.cpp:255-269)
    struct PlanLike {
      unsigned k;
    };
    std::vector<std::int32_t> keys(1u << 12);
    for (auto& v : keys) v = static_cast<std::int32_t>(static_cast<std::uint32_t>(rng()));
    auto expected = keys;
    std::sort(expected.begin(), expected.end());
    const auto r = bitonic::gpu::execute(PlanLike{12}, keys, 4);
    CHECK(r.keys == expected);
    CHECK(r.counters.compare_exchanges == (std::uint64_t{1} << 11) * 78);
    CHECK(r.counters.global_reads == r.counters.kernel_launches << 12);
    CHECK_THROWS_AS(bitonic::gpu::execute(PlanLike{13}, keys, 4), bitonic::invalid_size_error);
    CHECK_THROWS_AS(bitonic::gpu::execute(PlanLike{12}, keys, 0), bitonic::config_error);
    // both arguments bad: workers is checked first (engine.cpp:177-185)
    CHECK_THROWS_AS(bitonic::gpu::execute(PlanLike{13}, keys, 0), bitonic::config_error);
    // a plan with the reference's launches list: counters are account() of
    // that plan (test_engine.cpp:354-370 compares them with plan totals)
    struct StepLike {};
    struct LaunchLike {
      std::vector<StepLike> steps;
    };
    struct PlanWithLaunches {
      unsigned k;
      std::vector<LaunchLike> launches;
    };
    PlanWithLaunches pl{12, {LaunchLike{std::vector<StepLike>(1)},
                             LaunchLike{std::vector<StepLike>(2)},
                             LaunchLike{std::vector<StepLike>(9)}}};
    const auto r2 = bitonic::gpu::execute(pl, keys, 2);
    CHECK(r2.keys == expected);
    CHECK(r2.counters.kernel_launches == 3);
    CHECK(r2.counters.global_reads == 3u << 12);
    CHECK(r2.counters.global_writes == 3u << 12);
    CHECK(r2.counters.compare_exchanges == (std::uint64_t{1} << 11) * 12);
  }
  {
    std::vector<std::int32_t> odd(6);
    CHECK_THROWS_AS(sequential_bitonic_sort(odd), bitonic::invalid_size_error);
    std::vector<std::int32_t> one(1);
    CHECK_THROWS_AS(sequential_bitonic_sort(one), bitonic::invalid_size_error);
    CHECK_THROWS_AS(bitonic::gpu::sort_device(static_cast<std::uint32_t*>(nullptr), 16),
                    bitonic::config_error);
  }
  std::printf("%s (%d failures)\n", failures ? "FAILED" : "OK", failures);
  return failures ? 1 : 0;
}
