// oracle/ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// A thin extern "C" wrapper around the UNMODIFIED reference implementation,
// compiled directly from its sources under /root/reference/proj/src by
// oracle/Makefile into oracle/_ref/libbitonic_ref.so.  It lets the Python
// tests, the golden-fixture generator and bench.py's reference arm call the
// reference's own functions:
//
//   ref_sequential_bitonic_sort_i32  -> bitonic::sequential_bitonic_sort
//                                       (proj/include/bitonic/engine.hpp:102-104)
//   ref_quicksort_i32                -> bitonic::reference_quicksort
//                                       (proj/include/bitonic/verify.hpp:18-22)
//   ref_execute_i32                  -> bitonic::execute(build_plan(...))
//                                       (engine.hpp:77-92)
//   ref_generate_input               -> bitonic::generate_input (bench.hpp:86-89)
//   ref_pad_to_pow2                  -> bitonic::pad_to_pow2 (bench.hpp:91-94)
//   ref_predicted_counts             -> bitonic::predicted_counts (schedule.hpp:59-61)
//   ref_plan_counters                -> sum of bitonic::account over a plan
//   ref_check_zero_one               -> bitonic::check_zero_one (verify.hpp:24-29)
//
// Status codes follow the product's C ABI: 0 ok, 1 invalid_size_error,
// 2 config_error, 5 other exception.  Nothing here is on the product path.
#include <cstdint>
#include <chrono>
#include <cstring>
#include <exception>
#include <span>
#include <vector>

#include "bitonic/engine.hpp"
#include "bitonic/error.hpp"
#include "bitonic/schedule.hpp"
#include "bitonic/verify.hpp"
#ifndef REF_NO_BENCH
#include "bitonic/bench.hpp"
#endif

namespace {

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const bitonic::invalid_size_error&) {
    return 1;
  } catch (const bitonic::config_error&) {
    return 2;
  } catch (...) {
    return 5;
  }
}

}  // namespace

extern "C" {

int ref_sequential_bitonic_sort_i32(int32_t* keys, uint64_t n) {
  return guarded([&] {
    bitonic::sequential_bitonic_sort(std::span<int32_t>(keys, n));
  });
}

int ref_quicksort_i32(int32_t* keys, uint64_t n) {
  return guarded(
      [&] { bitonic::reference_quicksort(std::span<int32_t>(keys, n)); });
}

// strategy: 0 baseline, 1 shared, 2 fused.  counters (optional) receives
// {kernel_launches, global_reads, global_writes, compare_exchanges}.
int ref_execute_i32(int32_t* keys, uint64_t n, int strategy, uint64_t cap,
                    unsigned workers, uint64_t* counters) {
  return guarded([&] {
    if (n < 2 || (n & (n - 1)) != 0) {
      throw bitonic::invalid_size_error("length must be a power of two");
    }
    unsigned k = 0;
    while ((uint64_t{1} << k) < n) ++k;
    const auto plan = bitonic::build_plan(
        bitonic::generate_schedule(k), static_cast<bitonic::Strategy>(strategy),
        cap);
    bitonic::KeyArray v(keys, keys + n);
    auto result = bitonic::execute(plan, std::move(v), workers);
    std::memcpy(keys, result.keys.data(), n * sizeof(int32_t));
    if (counters) {
      counters[0] = result.counters.kernel_launches;
      counters[1] = result.counters.global_reads;
      counters[2] = result.counters.global_writes;
      counters[3] = result.counters.compare_exchanges;
    }
  });
}

// run_cell's timing discipline (bench.cpp:92-107): the keys are copied into
// the vector outside the timed region; generate_schedule + build_plan +
// execute are timed with steady_clock; *ms receives the elapsed time.
int ref_execute_timed_i32(int32_t* keys, uint64_t n, int strategy, uint64_t cap,
                          unsigned workers, double* ms) {
  return guarded([&] {
    if (n < 2 || (n & (n - 1)) != 0) {
      throw bitonic::invalid_size_error("length must be a power of two");
    }
    unsigned k = 0;
    while ((uint64_t{1} << k) < n) ++k;
    bitonic::KeyArray v(keys, keys + n);
    const auto t0 = std::chrono::steady_clock::now();
    const auto plan = bitonic::build_plan(
        bitonic::generate_schedule(k), static_cast<bitonic::Strategy>(strategy),
        cap);
    auto result = bitonic::execute(plan, std::move(v), workers);
    const auto t1 = std::chrono::steady_clock::now();
    *ms = std::chrono::duration<double, std::milli>(t1 - t0).count();
    std::memcpy(keys, result.keys.data(), n * sizeof(int32_t));
  });
}

int ref_plan_counters(unsigned k, int strategy, uint64_t cap,
                      uint64_t* counters) {
  return guarded([&] {
    const auto plan = bitonic::build_plan(
        bitonic::generate_schedule(k), static_cast<bitonic::Strategy>(strategy),
        cap);
    bitonic::Counters total;
    for (const auto& launch : plan.launches) {
      total += bitonic::account(launch, std::size_t{1} << k);
    }
    counters[0] = total.kernel_launches;
    counters[1] = total.global_reads;
    counters[2] = total.global_writes;
    counters[3] = total.compare_exchanges;
  });
}

int ref_predicted_counts(unsigned k, uint64_t* rounds, uint64_t* ces) {
  return guarded([&] {
    const auto c = bitonic::predicted_counts(k);
    *rounds = c.rounds;
    *ces = c.compare_exchanges;
  });
}

int ref_check_zero_one(unsigned k, int* ok) {
  return guarded([&] { *ok = bitonic::check_zero_one(k) ? 1 : 0; });
}

int ref_has_bench(void) {
#ifdef REF_NO_BENCH
  return 0;
#else
  return 1;
#endif
}

#ifndef REF_NO_BENCH
int ref_generate_input(int32_t* out, uint64_t n, uint64_t seed) {
  return guarded([&] {
    const auto v = bitonic::generate_input(n, seed);
    std::memcpy(out, v.data(), n * sizeof(int32_t));
  });
}

// out must hold max(2, bit_ceil(n)) keys; *padded_len receives that length.
int ref_pad_to_pow2(const int32_t* in, uint64_t n, int32_t* out,
                    uint64_t* padded_len) {
  return guarded([&] {
    const auto p = bitonic::pad_to_pow2(std::span<const int32_t>(in, n));
    std::memcpy(out, p.keys.data(), p.keys.size() * sizeof(int32_t));
    *padded_len = p.keys.size();
  });
}
#endif

}  // extern "C"
