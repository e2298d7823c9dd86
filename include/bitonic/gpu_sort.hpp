// bitonic/gpu_sort.hpp -- C++ drop-in for the reference's sort entry points,
// running the B200 (sm_100a) bitonic network through the C ABI in
// b200_bitonic.h.
//
// Reference interface replaced (/root/reference/proj/include/bitonic):
//   void sequential_bitonic_sort(std::span<std::int32_t>)   engine.hpp:102-104
//   ExecutionResult execute(const LaunchPlan&, KeyArray, unsigned)
//                                                            engine.hpp:86-92
// Same call shapes, same exception types: a non-power-of-two length throws
// bitonic::invalid_size_error (engine.cpp:250-253), bad arguments throw
// bitonic::config_error (error.hpp:19-23).  When the reference's
// bitonic/error.hpp is on the include path its types are used, so existing
// CHECK_THROWS_AS(..., invalid_size_error) tests keep working unchanged.
#ifndef BITONIC_GPU_SORT_HPP
#define BITONIC_GPU_SORT_HPP

#include <cstdint>
#include <span>
#include <utility>
#include <vector>
#include <stdexcept>
#include <string>

#include "../b200_bitonic.h"

#if __has_include("bitonic/error.hpp")
#include "bitonic/error.hpp"
#else
namespace bitonic {
// Same names and bases as the reference's error.hpp:11-23.
class invalid_size_error : public std::invalid_argument {
 public:
  explicit invalid_size_error(const std::string& what) : std::invalid_argument(what) {}
};
class config_error : public std::invalid_argument {
 public:
  explicit config_error(const std::string& what) : std::invalid_argument(what) {}
};
}  // namespace bitonic
#endif

namespace bitonic::gpu {

// A CUDA runtime failure (no reference counterpart: the reference has no GPU).
class cuda_error : public std::runtime_error {
 public:
  explicit cuda_error(const std::string& what) : std::runtime_error(what) {}
};

inline void check(int status) {
  switch (status) {
    case B200_OK:
      return;
    case B200_INVALID_SIZE:
      throw invalid_size_error(b200_bitonic_last_error());
    case B200_CONFIG:
      throw config_error(b200_bitonic_last_error());
    default:
      throw cuda_error(b200_bitonic_last_error());
  }
}

// Host-memory entries (H2D, sort on the GPU, D2H; synchronous).
inline void sort(std::span<std::int32_t> keys, bool ascending = true) {
  check(b200_bitonic_sort_host_i32(keys.data(), keys.size(), ascending ? 0 : 1));
}
inline void sort(std::span<std::uint32_t> keys, bool ascending = true) {
  check(b200_bitonic_sort_host_u32(keys.data(), keys.size(), ascending ? 0 : 1));
}

// Name-for-name replacement of bitonic::sequential_bitonic_sort.
inline void sequential_bitonic_sort(std::span<std::int32_t> keys) { sort(keys, true); }

// Device-pointer entries (in place, stream-ordered, no allocation).
inline void sort_device(std::int32_t* d_keys, std::uint64_t n, bool ascending = true,
                        b200_stream_t stream = nullptr) {
  check(b200_bitonic_sort_i32(d_keys, n, ascending ? 0 : 1, stream));
}
inline void sort_device(std::uint32_t* d_keys, std::uint64_t n, bool ascending = true,
                        b200_stream_t stream = nullptr) {
  check(b200_bitonic_sort_u32(d_keys, n, ascending ? 0 : 1, stream));
}
// The merge-path variant: same output, one HBM pass per global phase
// (allocates an n-key scratch buffer from the library's pool).
inline void sort_device_mergepath(std::int32_t* d_keys, std::uint64_t n, bool ascending = true,
                                  b200_stream_t stream = nullptr) {
  check(b200_bitonic_sort_mergepath_i32(d_keys, n, ascending ? 0 : 1, stream));
}
inline void sort_device_mergepath(std::uint32_t* d_keys, std::uint64_t n, bool ascending = true,
                                  b200_stream_t stream = nullptr) {
  check(b200_bitonic_sort_mergepath_u32(d_keys, n, ascending ? 0 : 1, stream));
}
inline void sort_device_batched(std::uint32_t* d_keys, std::uint64_t n_per_array,
                                std::uint64_t batch, bool ascending = true,
                                b200_stream_t stream = nullptr) {
  check(b200_bitonic_sort_u32_batched(d_keys, n_per_array, batch, ascending ? 0 : 1,
                                      stream));
}

// Counterparts of bitonic::Counters / ExecutionResult (engine.hpp:55-75),
// same field names, so call sites reading r.keys and r.counters compile
// unchanged.  The counters are the GPU plan's, in the reference's cost model
// (account(), engine.cpp:147-173): one launch = n reads + n writes; CEs =
// predicted_counts (schedule.cpp:71-78).
struct Counters {
  std::uint64_t kernel_launches = 0;
  std::uint64_t global_reads = 0;
  std::uint64_t global_writes = 0;
  std::uint64_t compare_exchanges = 0;
  friend bool operator==(const Counters&, const Counters&) = default;
};

struct ExecutionResult {
  std::vector<std::int32_t> keys;
  Counters counters;
};

inline Counters counters(std::uint64_t n, std::uint64_t batch = 1) {
  std::uint64_t c[4] = {0, 0, 0, 0};
  check(b200_bitonic_counters(n, batch, c));
  return Counters{c[0], c[1], c[2], c[3]};
}

// Drop-in for bitonic::execute(const LaunchPlan&, KeyArray, unsigned)
// (engine.hpp:86-92, engine.cpp:175-227): takes the keys by value, returns
// them sorted with counters.  Any plan type with the reference's `k` member
// is accepted; the GPU runs its own plan (the caller's strategy and block
// capacity describe CPU launches).  Same failures in the same order as
// engine.cpp:177-185: workers < 1 throws config_error first, then
// keys.size() != 2^k throws invalid_size_error.
//
// Counters: when the plan carries the reference's `launches` list, r.counters
// are that plan's, charged exactly as account() (engine.cpp:147-173) does --
// one launch = n reads + n writes, (n/2) x steps compare-exchanges -- so
// `r.counters == plan_totals(plan)` style assertions keep holding after the
// swap.  For a plan type without `launches` they are the GPU plan's
// (bitonic::gpu::counters(n)), in the same cost model.
template <class Plan>
inline Counters plan_counters(const Plan& plan, std::uint64_t n) {
  if constexpr (requires { plan.launches.begin(); }) {
    Counters c;
    for (const auto& launch : plan.launches) {
      c.kernel_launches += 1;
      c.global_reads += n;
      c.global_writes += n;
      c.compare_exchanges += (n / 2) * static_cast<std::uint64_t>(launch.steps.size());
    }
    return c;
  } else {
    return counters(n);
  }
}

template <class Plan>
inline ExecutionResult execute(const Plan& plan, std::vector<std::int32_t> keys,
                               unsigned workers) {
  if (workers < 1) throw config_error("execute: workers must be >= 1");
  if (plan.k >= 64 || keys.size() != (std::uint64_t{1} << plan.k)) {
    throw invalid_size_error("execute: key count does not match the plan's 2^k");
  }
  sort(std::span<std::int32_t>(keys), true);
  const std::uint64_t n = keys.size();
  Counters c = plan_counters(plan, n);
  return ExecutionResult{std::move(keys), c};
}

}  // namespace bitonic::gpu

#endif  // BITONIC_GPU_SORT_HPP
