// bitonic_sort.cu -- launcher, plans, graphs, merge path and the device entries.
//
// Host side of the B200-native bitonic sort.  Replaces, behind the C ABI in
// include/b200_bitonic.h, the reference's execute() (engine.cpp:175-227):
// where the reference runs each launch of a LaunchPlan on a fork-join worker
// pool with a full barrier in between (worker_pool.cpp:28-44), this enqueues
// one sm_100a kernel per planned pass on a CUDA stream; stream order is the
// barrier.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/b200_bitonic.h"
#include "bitonic_engine.cuh"
#include "kernel_tables.hpp"
#include "merge_split.cuh"
#include "planner.hpp"
#include "runtime.hpp"

namespace b200::rt {

thread_local std::string g_last_error;

std::atomic<int> g_tile_bits{0};  // 0 = automatic
std::atomic<int> g_min_run_bits{5};

int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

int cuda_fail(cudaError_t e, const char* what) {
  return fail(B200_CUDA_ERROR,
              std::string(what) + ": " + cudaGetErrorString(e));
}

b200::PlanOptions plan_options() {
  b200::PlanOptions o;
  const int tb = g_tile_bits.load();
  if (tb > 0) {
    o.cmax = tb;
    o.cmin = tb;  // explicit tile size: no automatic shrinking
  }
  o.lrun = g_min_run_bits.load();
  if (const char* e = std::getenv("B200_BITONIC_REGBITS")) o.regbits = std::atoi(e);
  if (const char* e = std::getenv("B200_BITONIC_PLANNER")) o.dp = std::strcmp(e, "greedy") != 0;
  if (const char* e = std::getenv("B200_BITONIC_TILE_REGBITS")) o.tile_regbits = std::atoi(e);
  if (const char* e = std::getenv("B200_BITONIC_CMERGE")) o.cmerge = std::atoi(e);
  if (const char* e = std::getenv("B200_BITONIC_TRIP_COST")) o.trip_cost = std::atof(e);
  if (const char* e = std::getenv("B200_BITONIC_MIXED_C")) o.mixed_c = std::atoi(e) != 0;
  if (const char* e = std::getenv("B200_BITONIC_WIDE_TAIL_COST")) o.wide_tail_cost = std::atof(e);
  if (const char* e = std::getenv("B200_BITONIC_CLUSTER")) o.cluster = std::atoi(e) != 0;
  if (const char* e = std::getenv("B200_BITONIC_CLUSTER_COST")) o.cluster_cost = std::atof(e);
  if (const char* e = std::getenv("B200_BITONIC_MID_LRUN")) o.mid_lrun = std::atoi(e);
  if (const char* e = std::getenv("B200_BITONIC_R14")) o.regbits14 = std::atoi(e);
  if (const char* e = std::getenv("B200_BITONIC_TILE_C")) o.tile_c = std::atoi(e);
  return o;
}

int log2_exact(uint64_t n) {
  int k = 0;
  while ((uint64_t{1} << k) < n) ++k;
  return k;
}

bool is_pow2(uint64_t n) { return n >= 1 && (n & (n - 1)) == 0; }

// ---- kernel selection and launch --------------------------------------------
// Specialised (compile-time step sequence) kernels are used for every pass
// shape that was instantiated; anything else runs on the runtime-dispatched
// bitonic_pass_kernel<C>.  Both are sm_100a code; there is no host fallback.
template <int C>
b200::PassFn generic_kernel_c() {
  return &b200::bitonic_pass_kernel<C>;
}

b200::PassFn generic_kernel(int C) {
  switch (C) {
    case 1: return generic_kernel_c<1>();
    case 2: return generic_kernel_c<2>();
    case 3: return generic_kernel_c<3>();
    case 4: return generic_kernel_c<4>();
    case 5: return generic_kernel_c<5>();
    case 6: return generic_kernel_c<6>();
    case 7: return generic_kernel_c<7>();
    case 8: return generic_kernel_c<8>();
    case 9: return generic_kernel_c<9>();
    case 10: return generic_kernel_c<10>();
    case 11: return generic_kernel_c<11>();
    case 12: return generic_kernel_c<12>();
    case 13: return generic_kernel_c<13>();
    case 14: return generic_kernel_c<14>();
    default: return generic_kernel_c<15>();
  }
}

// Scratch memory (padded copies, 64-bit word planes, merge coranks, host
// staging) comes from one library-owned stream-ordered pool per device that
// keeps freed memory (release threshold = max): after the first call of a
// given size, allocation is a pool lookup instead of a fresh mapping.
std::mutex g_pool_mu;
std::vector<cudaMemPool_t> g_pools;

cudaError_t scratch_alloc(void** p, size_t bytes, cudaStream_t s) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  cudaMemPool_t pool = nullptr;
  {
    std::lock_guard<std::mutex> lk(g_pool_mu);
    if ((int)g_pools.size() <= dev) g_pools.resize(dev + 1, nullptr);
    if (g_pools[dev] == nullptr) {
      cudaMemPoolProps props{};
      props.allocType = cudaMemAllocationTypePinned;
      props.location.type = cudaMemLocationTypeDevice;
      props.location.id = dev;
      e = cudaMemPoolCreate(&g_pools[dev], &props);
      if (e != cudaSuccess) return e;
      uint64_t keep = ~uint64_t{0};
      cudaMemPoolSetAttribute(g_pools[dev], cudaMemPoolAttrReleaseThreshold, &keep);
    }
    pool = g_pools[dev];
  }
  return cudaMallocFromPoolAsync(p, bytes, pool, s);
}


cudaError_t trim_scratch_pools() {
  std::lock_guard<std::mutex> lk(g_pool_mu);
  for (cudaMemPool_t p : g_pools) {
    if (p == nullptr) continue;
    cudaError_t e = cudaMemPoolTrimTo(p, 0);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

std::atomic<int> g_force_generic{0};
// alternate the coset order of consecutive passes (PassParams::reverse)
bool reverse_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("B200_BITONIC_REVERSE");
    return !(e && std::strcmp(e, "0") == 0);
  }();
  return on;
}
std::atomic<int> g_pdl{1};  // programmatic dependent launch between passes

// Returns the kernel and its keys-per-thread exponent (the block size is
// 2^(C - R)).  Shapes without a 16-keys-per-thread instantiation fall back to
// 32 keys per thread.
// mode: 0 keys, 1 key + payload, 2 64-bit keys (two word arrays).
b200::PassFn select_kernel(const b200::PlanPass& q, int* R_out, int mode) {
  if (mode == 3) {  // virtual padding (keys only)
    *R_out = 5;
    return b200::find_virtual_kernel(q.tile_sort != 0, q.C, q.segA_hi, q.segB_lo, q.R);
  }
  if (q.cluster) {
    *R_out = 5;
    return mode == 0 ? b200::find_cluster_kernel(q.segA_hi, 5) : nullptr;
  }
  if (mode != 0) {
    *R_out = q.R;
    return q.tile_sort ? (q.p_end == q.C ? b200::find_tile_kernel(q.C, q.R, mode) : nullptr)
                       : b200::find_merge_kernel(q.C, q.segA_hi, q.segB_lo, q.R, mode);
  }
  if (!g_force_generic.load()) {
    for (int R : {q.R, 5}) {
      b200::PassFn f = q.tile_sort
                           ? (q.p_end == q.C ? b200::find_tile_kernel(q.C, R) : nullptr)
                           : b200::find_merge_kernel(q.C, q.segA_hi, q.segB_lo, R);
      if (f) {
        *R_out = R == 5 ? b200::reg_bits(q.C) : R;
        return f;
      }
    }
  }
  *R_out = b200::reg_bits(q.C);
  return generic_kernel(q.C);
}

// Max-dynamic-shared-memory attribute, set once per (device, kernel).
std::mutex g_attr_mu;
std::vector<std::vector<const void*>> g_attr_done;

cudaError_t ensure_attr(const void* fn, int C, int arrays) {
  const int bytes = b200::tile_smem_words(C) * 4 * arrays;
  if (bytes <= 48 * 1024) return cudaSuccess;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lk(g_attr_mu);
  if ((int)g_attr_done.size() <= dev) g_attr_done.resize(dev + 1);
  auto& done = g_attr_done[dev];
  if (std::find(done.begin(), done.end(), fn) != done.end()) return cudaSuccess;
  e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) done.push_back(fn);
  return e;
}

// The tile sort's load as one TMA tensor copy (bitonic_tma.cuh).
bool tma_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("B200_BITONIC_TMA");
    return e && std::strcmp(e, "1") == 0;
  }();
  return on;
}

cudaError_t launch_tile_tma(const b200::PlanPass& q, b200::PassParams p, uint64_t total,
                            cudaStream_t s, bool* done) {
  *done = false;
  b200::TmaTileFn f = b200::find_tile_tma_kernel(q.C);
  CUtensorMap map;
  if (f == nullptr || !b200::make_tile_tensor_map(&map, p.keys, total, q.C)) return cudaSuccess;
  const void* fn = reinterpret_cast<const void*>(f);
  const size_t smem = (size_t)b200::tile_smem_words(q.C) * 4 + 1024;  // + swizzle alignment
  cudaError_t e = cudaSuccess;
  {
    std::lock_guard<std::mutex> lk(g_attr_mu);
    int dev = 0;
    cudaGetDevice(&dev);
    if ((int)g_attr_done.size() <= dev) g_attr_done.resize(dev + 1);
    auto& d = g_attr_done[dev];
    if (std::find(d.begin(), d.end(), fn) == d.end()) {
      e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e == cudaSuccess) d.push_back(fn);
    }
  }
  if (e != cudaSuccess) return e;
  void* args[] = {&p, &map};
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)q.ctas);
  cfg.blockDim = dim3(1u << (q.C - 5));
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = g_pdl.load() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  *done = true;
  return cudaLaunchKernelExC(&cfg, fn, args);
}

// mode: 0 keys, 1 key + payload, 2 64-bit keys, 3 keys with virtual padding
cudaError_t launch_pass(const b200::PlanPass& q, b200::PassParams p, cudaStream_t s,
                        int mode) {
  if (q.tile_sort && mode == 0 && q.R == 5 && q.p_end == q.C && tma_enabled() &&
      !g_force_generic.load() && p.keys_out == nullptr) {
    bool done = false;
    cudaError_t e = launch_tile_tma(q, p, q.ctas << q.C, s, &done);
    if (done || e != cudaSuccess) return e;
  }
  int R = 5;
  const bool kv = mode == 1 || mode == 2;
  b200::PassFn f = select_kernel(q, &R, mode);
  if (f == nullptr) return cudaErrorNotSupported;  // no such key-value shape
  const void* fn = reinterpret_cast<const void*>(f);
  const int Cb = q.cluster ? 14 : q.C;  // keys per CTA = 2^Cb (a cluster pass: 2 CTAs)
  cudaError_t e = ensure_attr(fn, Cb, kv ? 2 : 1);
  if (e != cudaSuccess) return e;
  const size_t smem = (size_t)b200::tile_smem_words(Cb) * 4 * (kv ? 2 : 1);
  void* args[] = {&p};
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)q.ctas);
  cfg.blockDim = dim3(1u << (Cb - R));
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = g_pdl.load() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelExC(&cfg, fn, args);
}

// Plans are pure functions of (k, batch, options): cache the last few so a
// repeated sort costs only its kernel launches on the host.
std::mutex g_plan_mu;
struct PlanKey {
  int k;
  uint64_t batch;
  int cmax, cmin, lrun, min_ctas, regbits, tile_regbits, cmerge;
  bool dp, kv;
  double trip_cost;
  bool mixed_c;
  double wide_tail_cost;
  bool virt;
  bool cluster;
  double cluster_cost;
  int mid_lrun, regbits14, tile_c;
  bool operator==(const PlanKey& o) const {
    return k == o.k && batch == o.batch && cmax == o.cmax && cmin == o.cmin &&
           lrun == o.lrun && min_ctas == o.min_ctas && regbits == o.regbits && dp == o.dp &&
           kv == o.kv && tile_regbits == o.tile_regbits && cmerge == o.cmerge &&
           trip_cost == o.trip_cost && mixed_c == o.mixed_c &&
           wide_tail_cost == o.wide_tail_cost && virt == o.virt && cluster == o.cluster &&
           cluster_cost == o.cluster_cost && mid_lrun == o.mid_lrun &&
           regbits14 == o.regbits14 && tile_c == o.tile_c;
  }
};
std::vector<std::pair<PlanKey, std::vector<b200::PlanPass>>> g_plans;

std::vector<b200::PlanPass> cached_plan(int k, uint64_t batch, const b200::PlanOptions& o) {
  const PlanKey key{k, batch, o.cmax, o.cmin, o.lrun, o.min_ctas, o.regbits, o.tile_regbits,
                    o.cmerge, o.dp, o.kv, o.trip_cost, o.mixed_c, o.wide_tail_cost,
                    o.virt, o.cluster, o.cluster_cost, o.mid_lrun, o.regbits14, o.tile_c};
  std::lock_guard<std::mutex> lk(g_plan_mu);
  for (auto& e : g_plans)
    if (e.first == key) return e.second;
  auto plan = b200::make_plan(k, batch, o);
  if (g_plans.size() >= 16) g_plans.erase(g_plans.begin());
  g_plans.emplace_back(key, plan);
  return plan;
}

// ---- CUDA graphs for repeated launches -------------------------------------
// A sort is 1..31 dependent launches; enqueueing them costs ~3.5 us each on
// the host, which at 2^20 keys is as long as the sort itself.  The second
// time the same (device, buffers, shape, direction, tuning) is seen, the
// launch sequence is captured once (on a private capture stream, so the
// caller's stream may be the legacy default stream) and every later call
// is a single cudaGraphLaunch on the caller's stream.  Calls made while the
// caller's stream is itself being captured launch directly (they become
// part of the caller's graph).  B200_BITONIC_GRAPHS=0 disables this.
std::mutex g_graph_mu;
std::vector<GraphEntry> g_graphs;
thread_local cudaStream_t t_capture_stream[64] = {};

bool graphs_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("B200_BITONIC_GRAPHS");
    return !(e && std::strcmp(e, "0") == 0);
  }();
  return on;
}

GraphKey make_key(int kind, const void* p0, const void* p1, uint64_t n, uint64_t batch,
                  int desc, uint32_t kx, int mode, int G, const b200::PlanOptions& o) {
  GraphKey key;
  std::memset(&key, 0, sizeof(key));  // padding bytes take part in the compare
  cudaGetDevice(&key.dev);
  key.kind = kind;
  key.p0 = p0;
  key.p1 = p1;
  key.n = n;
  key.batch = batch;
  key.desc = desc;
  key.kx = kx;
  key.mode = mode;
  key.G = G;
  key.cmax = o.cmax;
  key.cmin = o.cmin;
  key.lrun = o.lrun;
  key.regbits = o.regbits;
  key.tile_regbits = o.tile_regbits;
  key.cmerge = o.cmerge;
  key.trip_cost = o.trip_cost;
  key.wide_tail_cost = o.wide_tail_cost;
  key.mixed_c = o.mixed_c;
  key.cluster = o.cluster;
  key.mid_lrun = o.mid_lrun;
  key.regbits14 = o.regbits14;
  key.tile_c = o.tile_c;
  key.cluster_cost = o.cluster_cost;
  key.dp = o.dp;
  key.generic = g_force_generic.load();
  key.pdl = g_pdl.load();
  return key;
}

GraphExecPtr own_exec(cudaGraphExec_t e) {
  return GraphExecPtr(e, [](cudaGraphExec_t x) {
    if (x) cudaGraphExecDestroy(x);
  });
}

void drop_graphs() {
  std::vector<GraphEntry> old;
  {
    std::lock_guard<std::mutex> lk(g_graph_mu);
    old.swap(g_graphs);
  }
  // execs still held by a launcher are destroyed when it lets go
}

// Validates and runs the whole plan (or only pass `only`, when >= 0).
// key_xor: 0x80000000 for int32 keys (for 64-bit keys: applied to the hi
// word).  d_vals: payloads (mode 1) or the lo words of 64-bit keys whose hi
// words are d_keys (mode 2).
int sort_impl(uint32_t* d_keys, uint64_t n_per, uint64_t batch, int descending,
              uint32_t key_xor, cudaStream_t stream, int only, uint32_t* d_vals, int mode,
              uint64_t nreal) {
  if (mode < 0) mode = d_vals != nullptr ? 1 : 0;
  bool virt = nreal != 0 && nreal < n_per;
  // testing aid: B200_BITONIC_VIRT_DEBUG=<dxor> runs a power-of-two sort
  // through the virtual-padding kernels (nreal = n, the given direction xor)
  uint64_t dbg_dxor = ~uint64_t{0};
  if (const char* e = std::getenv("B200_BITONIC_VIRT_DEBUG")) {
    if (!virt && batch == 1 && d_vals == nullptr && mode == 0) {
      virt = true;
      nreal = n_per;
      dbg_dxor = std::strtoull(e, nullptr, 0);
    }
  }
  if (virt && (batch != 1 || d_vals != nullptr || mode != 0)) {
    return fail(B200_CONFIG, "virtual padding: single key-only arrays");
  }
  if (mode != 0 && d_vals == nullptr) return fail(B200_CONFIG, "null second array");
  if (n_per < 2 || !is_pow2(n_per)) {
    return fail(B200_INVALID_SIZE,
                "length must be a power of two >= 2, got " +
                    std::to_string(n_per));
  }
  if (batch < 1) return fail(B200_CONFIG, "batch must be >= 1");
  const int k = log2_exact(n_per);
  if (k > 34 || (batch << k) >> k != batch || (batch << k) > (uint64_t{1} << 35)) {
    return fail(B200_INVALID_SIZE, "array too large for one device");
  }
  if (descending != 0 && descending != 1) {
    return fail(B200_CONFIG, "descending must be 0 or 1");
  }
  if (d_keys == nullptr) return fail(B200_CONFIG, "null key pointer");
  std::vector<b200::PlanPass> plan;
  b200::PlanOptions popt = plan_options();
  popt.kv = d_vals != nullptr;
  if (virt) {
    popt = b200::PlanOptions{};  // the virtual kernels' fixed shapes (no tuning knobs)
    popt.virt = true;
  }
  try {
    plan = cached_plan(k, batch, popt);
  } catch (const std::exception& e) {
    return fail(B200_CONFIG, e.what());
  }
  if (plan.front().C >= 2 && ((reinterpret_cast<uintptr_t>(d_keys) & 15u) != 0 ||
                                (reinterpret_cast<uintptr_t>(d_vals) & 15u) != 0)) {
    return fail(B200_CONFIG, "device pointers must be 16-byte aligned");
  }
  const uint32_t gmask = key_xor ^ (descending ? 0xFFFFFFFFu : 0u);
  const uint32_t gmask_lo = (mode == 2 && descending) ? 0xFFFFFFFFu : 0u;
  if (only >= (int)plan.size()) return fail(B200_CONFIG, "pass index outside the plan");
  auto launch_all = [&](cudaStream_t st) -> int {
    for (size_t i = 0; i < plan.size(); ++i) {
      if (only >= 0 && (int)i != only) continue;
      const b200::PlanPass& q = plan[i];
      b200::PassParams p{};
      p.keys = d_keys;
      p.vals = d_vals;
      p.gmask_in = (i == 0) ? gmask : 0u;
      p.gmask_out = (i + 1 == plan.size()) ? gmask : 0u;
      p.gmask_in_lo = (i == 0) ? gmask_lo : 0u;
      p.gmask_out_lo = (i + 1 == plan.size()) ? gmask_lo : 0u;
      p.a = q.a;
      p.y = q.y;
      p.kd = k;
      p.tile_sort = q.tile_sort;
      p.p_end = q.p_end;
      p.segA_hi = q.segA_hi;
      p.pA = q.pA;
      p.segB_lo = q.segB_lo;
      p.pB = q.pB;
      p.one = 1u;
      p.mone = 0xFFFFFFFFu;
      p.reverse = (reverse_enabled() && (i & 1) && !q.cluster) ? 1 : 0;
      p.nreal = virt ? nreal : ~uint64_t{0};
      p.dxor = virt ? (dbg_dxor != ~uint64_t{0} ? dbg_dxor : nreal - 1) : 0;
      cudaError_t e = launch_pass(q, p, st, virt ? 3 : mode);
      if (e == cudaErrorNotSupported) {
        return fail(B200_CONFIG,
                    "no key-value kernel for this tile size (use tile_bits 0, 12 or 13)");
      }
      if (e != cudaSuccess) return cuda_fail(e, "bitonic pass launch");
    }
    return B200_OK;
  };
  if (only >= 0 || plan.size() < 2) return launch_all(stream);
  GraphKey gk = make_key(0, d_keys, d_vals, n_per, batch, descending, key_xor, mode, 0, popt);
  gk.nreal = virt ? nreal : 0;
  return run_graphed(gk, stream, launch_all);
}

// ---- merge path ----------------------------------------------------------------
// Output window [o_begin, o_begin + o_len) of merge(A[0..la), B[0..lb)).
int merge_window_impl(const uint32_t* A, uint64_t la, const uint32_t* B, uint64_t lb,
                      uint64_t o_begin, uint64_t o_len, uint32_t key_xor, uint32_t* out,
                      uint64_t* scratch_coranks, cudaStream_t s) {
  if (o_len == 0) return B200_OK;
  const uint64_t tiles = (o_len + b200::kMergeTile - 1) / b200::kMergeTile;
  const uint64_t nb = tiles + 1;
  b200::merge_partition_kernel<<<(unsigned)((nb + 255) / 256), 256, 0, s>>>(
      A, la, B, lb, o_begin, o_len, key_xor, scratch_coranks, nb);
  constexpr int C = b200::kMergeC;
  // keys per thread of the merge tiles: 2^6 by default (two shared-memory
  // trips and coalesced direct stores for full tiles, as the merge-path
  // phases); B200_BITONIC_MERGE_R=4|5 (experiment knob)
  static const int mr = [] {
    const char* e = std::getenv("B200_BITONIC_MERGE_R");
    return e ? std::atoi(e) : 6;
  }();
  cudaError_t e;
  auto launch = [&](auto kern, int threads) -> cudaError_t {
    cudaError_t x = ensure_attr(reinterpret_cast<const void*>(kern), C, 1);
    if (x != cudaSuccess) return x;
    kern<<<(unsigned)tiles, threads, b200::tile_smem_words(C) * 4, s>>>(
        A, B, o_begin, o_len, key_xor, scratch_coranks, out, 1u, 0xFFFFFFFFu);
    return cudaSuccess;
  };
  if (mr == 4) e = launch(&b200::merge_bitonic_kernel<C, 4>, b200::threads_for<C, 4>());
  else if (mr == 5) e = launch(&b200::merge_bitonic_kernel<C, 5>, b200::threads_for<C, 5>());
  else e = launch(&b200::merge_bitonic_kernel<C, 6>, b200::threads_for<C, 6>());
  if (e != cudaSuccess) return cuda_fail(e, "merge kernel attribute");
  e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "merge launch");
  return B200_OK;
}

// ---- merge-path variant ---------------------------------------------------------
// The same result as the network sort (keys only), with each global phase in
// ONE HBM round trip: the tile sort leaves every 2^13-key tile ascending,
// then phase p (p = 14..k) merges run pairs by co-rank partition + bitonic
// tile merge (merge_split.cuh), ping-ponging between the array and one
// n-key scratch buffer so the last phase lands in the array.  k - 12 passes
// instead of the network's P(k) (2^28: 16 vs 29), at the price of an n-key
// scratch buffer and of the network's intermediate states (payload order of
// ties would differ, so key-value sorts stay on the network).
int mergepath_impl(uint32_t* d_keys, uint64_t n, int descending, uint32_t key_xor,
                   cudaStream_t s) {
  if (n < 2 || !is_pow2(n)) {
    return fail(B200_INVALID_SIZE,
                "length must be a power of two >= 2, got " + std::to_string(n));
  }
  if (descending != 0 && descending != 1) return fail(B200_CONFIG, "descending must be 0 or 1");
  if (d_keys == nullptr) return fail(B200_CONFIG, "null key pointer");
  constexpr int C = b200::kMergeC;  // merge window: 2^13 keys
  // tile-sort size: 2^14-key tiles (one phase fewer) measured 0.5-3% faster
  // than 2^13 from 2^24 keys (2^28: 7.72 vs 7.78 ms); experiment knob
  static const int tc_env = [] {
    const char* x = std::getenv("B200_BITONIC_MERGEPATH_TILE");
    return x ? std::atoi(x) : 14;
  }();
  const int TC = (tc_env >= C && tc_env <= 15) ? tc_env : C;
  const int k = log2_exact(n);
  if (k <= TC || k > 34) return sort_impl(d_keys, n, 1, descending, key_xor, s);
  if ((reinterpret_cast<uintptr_t>(d_keys) & 15u) != 0) {
    return fail(B200_CONFIG, "device pointers must be 16-byte aligned");
  }
  const uint32_t kx = key_xor ^ (descending ? 0xFFFFFFFFu : 0u);
  uint32_t kx_arg = kx;
  const int phases = k - TC;
  const uint64_t wins = n >> C;
  uint32_t* tmp = nullptr;
  uint64_t* cor = nullptr;
  B200_CUDA_TRY(scratch_alloc(reinterpret_cast<void**>(&tmp), n * 4, s));
  cudaError_t e = scratch_alloc(reinterpret_cast<void**>(&cor), (wins + 1) * sizeof(uint64_t), s);
  if (e != cudaSuccess) {
    cudaFreeAsync(tmp, s);
    return cuda_fail(e, "scratch");
  }
  int rc = B200_OK;
  // phase i (1-based) writes buf[i & 1]; the tile sort writes buf[0]
  uint32_t* buf[2] = {(phases & 1) ? tmp : d_keys, (phases & 1) ? d_keys : tmp};
  static const int tile_r = [] {  // keys per thread of the tile sort (experiment knob)
    const char* x = std::getenv("B200_BITONIC_MERGEPATH_TILE_R");
    return x ? std::atoi(x) : 5;
  }();
  {
    b200::PlanPass q;
    q.C = TC;
    q.R = tile_r;
    q.a = q.y = TC;
    q.tile_sort = 1;
    q.p_end = TC;
    q.ctas = n >> TC;
    b200::PassParams p{};
    p.keys = d_keys;
    p.keys_out = buf[0] == d_keys ? nullptr : buf[0];
    p.gmask_in = p.gmask_out = kx;  // every tile ascending in the order kx selects
    p.a = p.y = TC;
    p.kd = TC;
    p.tile_sort = 1;
    p.p_end = TC;
    p.segA_hi = p.segB_lo = -1;
    p.one = 1u;
    p.mone = 0xFFFFFFFFu;
    p.nreal = ~uint64_t{0};
    e = launch_pass(q, p, s, 0);
    if (e != cudaSuccess) rc = cuda_fail(e, "merge-path tile sort");
  }
  // keys per thread of the merge windows: 2^6 (rounds {12..7}, {6..1},
  // {0}: coalesced stores straight from registers, two shared-memory trips)
  // measured 7.39 vs 7.72 ms at 2^28 against 2^5 (three trips); knob kept
  static const int mr = [] {
    const char* x = std::getenv("B200_BITONIC_MERGEPATH_R");
    return x ? std::atoi(x) : 6;
  }();
  if (rc == B200_OK) {
    e = ensure_attr(mr == 6 ? reinterpret_cast<const void*>(&b200::mergepath_merge_kernel<C, 6>)
                            : reinterpret_cast<const void*>(&b200::mergepath_merge_kernel<C>),
                    C, 1);
    if (e != cudaSuccess) rc = cuda_fail(e, "merge kernel attribute");
  }
  // every phase kernel is launched with programmatic dependent launch: its
  // CTAs become resident while the previous kernel drains and wait in
  // griddepcontrol.wait for its memory (the kernels call pdl_wait first)
  auto pdl_launch = [&](const void* fn, unsigned grid, unsigned block, size_t smem,
                        void** args) -> cudaError_t {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(block);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = g_pdl.load() ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelExC(&cfg, fn, args);
  };
  // merge-window size: 2^13 keys (experiment knob B200_BITONIC_MERGEPATH_WIN=14)
  static const int wb_env = [] {
    const char* x = std::getenv("B200_BITONIC_MERGEPATH_WIN");
    return x ? std::atoi(x) : 13;
  }();
  const int WB = (wb_env == 14 && TC >= 14) ? 14 : 13;
  const uint64_t nwin = n >> WB;
  const void* merge_fn =
      WB == 14 ? reinterpret_cast<const void*>(&b200::mergepath_merge_kernel<14, 6>)
      : mr == 6 ? reinterpret_cast<const void*>(&b200::mergepath_merge_kernel<C, 6>)
                : reinterpret_cast<const void*>(&b200::mergepath_merge_kernel<C>);
  const void* part_fn = WB == 14
                            ? reinterpret_cast<const void*>(&b200::mergepath_partition_kernel<14>)
                            : reinterpret_cast<const void*>(&b200::mergepath_partition_kernel<C>);
  const unsigned merge_threads = WB == 14   ? b200::threads_for<14, 6>()
                                 : mr == 6 ? b200::threads_for<C, 6>()
                                           : b200::threads_for<C, 5>();
  if (WB == 14 && rc == B200_OK) {
    e = ensure_attr(merge_fn, 14, 1);
    if (e != cudaSuccess) rc = cuda_fail(e, "merge kernel attribute");
  }
  for (int i = 1; i <= phases && rc == B200_OK; ++i) {
    const uint32_t* src = buf[(i - 1) & 1];
    uint32_t* dst = buf[i & 1];
    int p = TC + i;
    uint32_t one = 1u, mone = 0xFFFFFFFFu;
    uint64_t nw = nwin;
    void* pargs[] = {&src, &p, &kx_arg, &cor, &nw};
    e = pdl_launch(part_fn, (unsigned)((nwin + 255) / 256), 256, 0, pargs);
    if (e == cudaSuccess) {
      void* margs[] = {&src, &dst, &p, &kx_arg, &cor, &one, &mone};
      e = pdl_launch(merge_fn, (unsigned)nwin, merge_threads,
                     (size_t)b200::tile_smem_words(WB) * 4, margs);
    }
    if (e != cudaSuccess) rc = cuda_fail(e, "merge-path phase");
  }
  cudaFreeAsync(cor, s);
  cudaFreeAsync(tmp, s);
  return rc;
}

int merge_split_impl(const uint32_t* local, const uint32_t* partner, uint64_t m,
                     int keep_high, uint32_t key_xor, uint32_t* out,
                     uint64_t* scratch_coranks, cudaStream_t s) {
  return merge_window_impl(local, m, partner, m, keep_high ? m : 0, m, key_xor, out,
                           scratch_coranks, s);
}

// float32 <-> order-preserving uint32 (IEEE totalOrder)
__global__ void f32_to_key_kernel(uint32_t* d, uint64_t n, int inverse) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const uint32_t x = d[i];
    if (!inverse) {
      d[i] = x ^ ((uint32_t)((int32_t)x >> 31) | 0x80000000u);
    } else {
      d[i] = x ^ ((uint32_t)((int32_t)~x >> 31) | 0x80000000u);
    }
  }
}

// 64-bit keys <-> (hi, lo) word planes.  kind 2 (float64) applies the
// totalOrder bit map x ^ (sign ? ~0 : 1 << 63) on the way in, undoes it on
// the way out.
__global__ void split64_kernel(const uint64_t* __restrict__ src, uint32_t* __restrict__ hi,
                               uint32_t* __restrict__ lo, uint64_t n, int kind) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    uint64_t x = src[i];
    if (kind == 2) x ^= (uint64_t)((int64_t)x >> 63) | 0x8000000000000000ull;
    hi[i] = (uint32_t)(x >> 32);
    lo[i] = (uint32_t)x;
  }
}

__global__ void join64_kernel(uint64_t* __restrict__ dst, const uint32_t* __restrict__ hi,
                              const uint32_t* __restrict__ lo, uint64_t n, int kind) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    uint64_t x = ((uint64_t)hi[i] << 32) | lo[i];
    if (kind == 2) x ^= (uint64_t)((int64_t)~x >> 63) | 0x8000000000000000ull;
    dst[i] = x;
  }
}

// kind: 0 uint64, 1 int64, 2 float64
int sort64_impl(uint64_t* d_keys, uint64_t n, int descending, int kind, cudaStream_t s) {
  if (n < 2 || !is_pow2(n)) {
    return fail(B200_INVALID_SIZE,
                "length must be a power of two >= 2, got " + std::to_string(n));
  }
  if (d_keys == nullptr) return fail(B200_CONFIG, "null key pointer");
  if (descending != 0 && descending != 1) {
    return fail(B200_CONFIG, "descending must be 0 or 1");
  }
  uint32_t* planes = nullptr;
  B200_CUDA_TRY(scratch_alloc(&planes, n * 8, s));
  uint32_t* hi = planes;
  uint32_t* lo = planes + n;
  const unsigned grid = (unsigned)std::min<uint64_t>((n + 255) / 256, 148 * 16);
  split64_kernel<<<grid, 256, 0, s>>>(d_keys, hi, lo, n, kind);
  int rc = sort_impl(hi, n, 1, descending, kind == 1 ? 0x80000000u : 0u, s, -1, lo, 2);
  if (rc == B200_OK) join64_kernel<<<grid, 256, 0, s>>>(d_keys, hi, lo, n, kind);
  cudaFreeAsync(planes, s);
  cudaError_t e = cudaGetLastError();
  if (rc == B200_OK && e != cudaSuccess) rc = cuda_fail(e, "64-bit key transform");
  return rc;
}

__global__ void pad_fill_kernel(uint32_t* dst, const uint32_t* src, uint64_t n,
                                uint64_t m, uint32_t pad) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += stride) {
    dst[i] = i < n ? src[i] : pad;
  }
}

// Virtual padding from 2^26 padded keys (B200: 2^28 - 1 keys 11.98 vs
// 11.97 ms with the copy, 0.81 x 2^28 keys 10.73 vs 11.86 ms, and no 1 GiB
// scratch; below that the copy path's size-tuned plans win, e.g. 2^20 - 1
// keys 0.075 vs 0.141 ms).  B200_BITONIC_VIRTUAL=1 forces it from 2^15
// (tests), =0 disables it.
bool use_virtual_padding(uint64_t m) {
  const char* e = std::getenv("B200_BITONIC_VIRTUAL");
  if (e && std::strcmp(e, "0") == 0) return false;
  if (e && std::strcmp(e, "1") == 0) return m >= (uint64_t{1} << 15);
  return m >= (uint64_t{1} << 26);
}

int padded_impl(uint32_t* d_keys, uint64_t n, int descending, uint32_t key_xor,
                cudaStream_t s) {
  if (n < 1) return fail(B200_INVALID_SIZE, "length must be >= 1");
  if (d_keys == nullptr) return fail(B200_CONFIG, "null key pointer");
  if (descending != 0 && descending != 1) {
    return fail(B200_CONFIG, "descending must be 0 or 1");
  }
  if (n == 1) return B200_OK;
  const bool aligned = (reinterpret_cast<uintptr_t>(d_keys) & 15u) == 0;
  if (is_pow2(n) && aligned) {
    return sort_impl(d_keys, n, 1, descending, key_xor, s);
  }
  uint64_t m = 2;
  while (m < n) m <<= 1;
  if (aligned && n >= (uint64_t{1} << 20) && n - m / 2 <= m / 4) {
    // Just above a power of two, padding would double the work: sort the
    // 2^j-key prefix in place, the r-key rest recursively (padded), and merge
    // the two runs (merge path) through one scratch buffer.  Same result as
    // pad + sort + truncate, ~1.5 instead of ~2.2 sorts of 2^j keys.
    const uint64_t h = m / 2, r = n - h;
    int rc = sort_impl(d_keys, h, 1, descending, key_xor, s);
    if (rc == B200_OK) rc = padded_impl(d_keys + h, r, descending, key_xor, s);
    if (rc != B200_OK) return rc;
    const uint32_t kx = key_xor ^ (descending ? 0xFFFFFFFFu : 0u);
    const uint64_t tiles = (n + b200::kMergeTile - 1) / b200::kMergeTile;
    uint32_t* out = nullptr;
    uint64_t* cor = nullptr;
    B200_CUDA_TRY(scratch_alloc(&out, n * 4, s));
    B200_CUDA_TRY(scratch_alloc(&cor, (tiles + 1) * sizeof(uint64_t), s));
    rc = merge_window_impl(d_keys, h, d_keys + h, r, 0, n, kx, out, cor, s);
    if (rc == B200_OK) {
      cudaError_t e = cudaMemcpyAsync(d_keys, out, n * 4, cudaMemcpyDeviceToDevice, s);
      if (e != cudaSuccess) rc = cuda_fail(e, "copy back");
    }
    cudaFreeAsync(cor, s);
    cudaFreeAsync(out, s);
    return rc;
  }
  if (aligned && use_virtual_padding(m)) {
    // Virtual padding: the 2^j-key network runs in place on the n real keys;
    // the m - n virtual keys are never loaded or stored (bitonic_static.cuh,
    // VIRT kernels) -- no scratch copy, no copy back.
    return sort_impl(d_keys, m, 1, descending, key_xor, s, -1, nullptr, 0, n);
  }
  // padding = the largest key in the sort's order (sorts last, discarded)
  const uint32_t gmask = key_xor ^ (descending ? 0xFFFFFFFFu : 0u);
  const uint32_t pad = ~gmask;
  uint32_t* tmp = nullptr;
  B200_CUDA_TRY(scratch_alloc(&tmp, m * 4, s));
  const unsigned grid = (unsigned)std::min<uint64_t>((m + 255) / 256, 148 * 8);
  pad_fill_kernel<<<grid, 256, 0, s>>>(tmp, d_keys, n, m, pad);
  int rc = sort_impl(tmp, m, 1, descending, key_xor, s);
  if (rc == B200_OK) {
    cudaError_t e = cudaMemcpyAsync(d_keys, tmp, n * 4, cudaMemcpyDeviceToDevice, s);
    if (e != cudaSuccess) rc = cuda_fail(e, "copy back");
  }
  cudaFreeAsync(tmp, s);
  if (rc == B200_OK) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) rc = cuda_fail(e, "padded sort");
  }
  return rc;
}


}  // namespace b200::rt

using namespace b200::rt;

extern "C" {



int b200_bitonic_sort_pairs_u32(uint32_t* d_keys, uint32_t* d_vals, uint64_t n,
                                int descending, b200_stream_t stream) {
  if (d_vals == nullptr) return fail(B200_CONFIG, "null value pointer");
  return sort_impl(d_keys, n, 1, descending, 0u, reinterpret_cast<cudaStream_t>(stream), -1,
                   d_vals);
}

int b200_bitonic_sort_pairs_i32(int32_t* d_keys, uint32_t* d_vals, uint64_t n,
                                int descending, b200_stream_t stream) {
  if (d_vals == nullptr) return fail(B200_CONFIG, "null value pointer");
  return sort_impl(reinterpret_cast<uint32_t*>(d_keys), n, 1, descending, 0x80000000u,
                   reinterpret_cast<cudaStream_t>(stream), -1, d_vals);
}

int b200_bitonic_sort_pairs_u32_batched(uint32_t* d_keys, uint32_t* d_vals,
                                        uint64_t n_per_array, uint64_t batch,
                                        int descending, b200_stream_t stream) {
  if (d_vals == nullptr) return fail(B200_CONFIG, "null value pointer");
  return sort_impl(d_keys, n_per_array, batch, descending, 0u,
                   reinterpret_cast<cudaStream_t>(stream), -1, d_vals);
}

int b200_bitonic_sort_f32(float* d_keys, uint64_t n, int descending,
                          b200_stream_t stream) {
  if (n < 2 || !is_pow2(n)) {
    return fail(B200_INVALID_SIZE,
                "length must be a power of two >= 2, got " + std::to_string(n));
  }
  if (d_keys == nullptr) return fail(B200_CONFIG, "null key pointer");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  uint32_t* d = reinterpret_cast<uint32_t*>(d_keys);
  const unsigned grid = (unsigned)std::min<uint64_t>((n + 255) / 256, 148 * 16);
  f32_to_key_kernel<<<grid, 256, 0, s>>>(d, n, 0);
  int rc = sort_impl(d, n, 1, descending, 0u, s);
  f32_to_key_kernel<<<grid, 256, 0, s>>>(d, n, 1);
  cudaError_t e = cudaGetLastError();
  if (rc == B200_OK && e != cudaSuccess) rc = cuda_fail(e, "f32 key transform");
  return rc;
}

int b200_bitonic_sort_u64(uint64_t* d_keys, uint64_t n, int descending,
                          b200_stream_t stream) {
  return sort64_impl(d_keys, n, descending, 0, reinterpret_cast<cudaStream_t>(stream));
}

int b200_bitonic_sort_i64(int64_t* d_keys, uint64_t n, int descending,
                          b200_stream_t stream) {
  return sort64_impl(reinterpret_cast<uint64_t*>(d_keys), n, descending, 1,
                     reinterpret_cast<cudaStream_t>(stream));
}

int b200_bitonic_sort_f64(double* d_keys, uint64_t n, int descending,
                          b200_stream_t stream) {
  return sort64_impl(reinterpret_cast<uint64_t*>(d_keys), n, descending, 2,
                     reinterpret_cast<cudaStream_t>(stream));
}

int b200_bitonic_sort_u64_planes(uint32_t* d_hi, uint32_t* d_lo, uint64_t n,
                                 int descending, b200_stream_t stream) {
  if (d_lo == nullptr) return fail(B200_CONFIG, "null low-word pointer");
  return sort_impl(d_hi, n, 1, descending, 0u, reinterpret_cast<cudaStream_t>(stream), -1,
                   d_lo, 2);
}

int b200_bitonic_sort_mergepath_u32(uint32_t* d_keys, uint64_t n, int descending,
                                    b200_stream_t stream) {
  return mergepath_impl(d_keys, n, descending, 0u, reinterpret_cast<cudaStream_t>(stream));
}

int b200_bitonic_sort_mergepath_i32(int32_t* d_keys, uint64_t n, int descending,
                                    b200_stream_t stream) {
  return mergepath_impl(reinterpret_cast<uint32_t*>(d_keys), n, descending, 0x80000000u,
                        reinterpret_cast<cudaStream_t>(stream));
}

int b200_bitonic_sort_padded_u32(uint32_t* d_keys, uint64_t n, int descending,
                                 b200_stream_t stream) {
  return padded_impl(d_keys, n, descending, 0u, reinterpret_cast<cudaStream_t>(stream));
}

int b200_bitonic_sort_padded_i32(int32_t* d_keys, uint64_t n, int descending,
                                 b200_stream_t stream) {
  return padded_impl(reinterpret_cast<uint32_t*>(d_keys), n, descending, 0x80000000u,
                     reinterpret_cast<cudaStream_t>(stream));
}

int b200_bitonic_sort_u32(uint32_t* d_keys, uint64_t n, int descending,
                          b200_stream_t stream) {
  return sort_impl(d_keys, n, 1, descending, 0u,
                   reinterpret_cast<cudaStream_t>(stream));
}

int b200_bitonic_sort_i32(int32_t* d_keys, uint64_t n, int descending,
                          b200_stream_t stream) {
  return sort_impl(reinterpret_cast<uint32_t*>(d_keys), n, 1, descending,
                   0x80000000u, reinterpret_cast<cudaStream_t>(stream));
}

int b200_bitonic_sort_u32_batched(uint32_t* d_keys, uint64_t n_per_array,
                                  uint64_t batch, int descending,
                                  b200_stream_t stream) {
  return sort_impl(d_keys, n_per_array, batch, descending, 0u,
                   reinterpret_cast<cudaStream_t>(stream));
}

int b200_bitonic_sort_i32_batched(int32_t* d_keys, uint64_t n_per_array,
                                  uint64_t batch, int descending,
                                  b200_stream_t stream) {
  return sort_impl(reinterpret_cast<uint32_t*>(d_keys), n_per_array, batch,
                   descending, 0x80000000u,
                   reinterpret_cast<cudaStream_t>(stream));
}

int b200_bitonic_plan(uint64_t n, uint64_t batch, b200_pass_info* out,
                      int max_passes, int* n_passes) {
  if (n < 2 || !is_pow2(n)) {
    return fail(B200_INVALID_SIZE,
                "length must be a power of two >= 2, got " + std::to_string(n));
  }
  if (batch < 1) return fail(B200_CONFIG, "batch must be >= 1");
  std::vector<b200::PlanPass> plan;
  try {
    plan = b200::make_plan(log2_exact(n), batch, plan_options());
  } catch (const std::exception& e) {
    return fail(B200_CONFIG, e.what());
  }
  if (n_passes) *n_passes = (int)plan.size();
  for (int i = 0; i < (int)plan.size() && i < max_passes && out; ++i) {
    const auto& q = plan[i];
    out[i].tile_bits = q.C;
    out[i].a = q.a;
    out[i].y = q.y;
    out[i].tile_sort = q.tile_sort;
    out[i].segA_hi = q.segA_hi;
    out[i].pA = q.tile_sort ? q.p_end : q.pA;
    out[i].segB_lo = q.segB_lo;
    out[i].pB = q.pB;
    out[i].ctas = q.ctas;
    out[i].compare_exchanges = q.ces;
    out[i].cluster = q.cluster ? 2 : 1;
  }
  return B200_OK;
}

int b200_bitonic_run_pass_u32(uint32_t* d_keys, uint64_t n_per_array,
                              uint64_t batch, int descending, int pass_index,
                              b200_stream_t stream) {
  if (pass_index < 0) return fail(B200_CONFIG, "pass index must be >= 0");
  return sort_impl(d_keys, n_per_array, batch, descending, 0u,
                   reinterpret_cast<cudaStream_t>(stream), pass_index);
}

int b200_bitonic_counters(uint64_t n, uint64_t batch, uint64_t out[4]) {
  int np = 0;
  int rc = b200_bitonic_plan(n, batch, nullptr, 0, &np);
  if (rc) return rc;
  std::vector<b200_pass_info> v(np);
  b200_bitonic_plan(n, batch, v.data(), np, &np);
  uint64_t ces = 0;
  for (auto& p : v) ces += p.compare_exchanges;
  out[0] = (uint64_t)np;
  out[1] = (uint64_t)np * n * batch;
  out[2] = (uint64_t)np * n * batch;
  out[3] = ces;
  return B200_OK;
}

int b200_bitonic_set_tuning(int tile_bits, int min_run_bits) {
  // min_run_bits >= 100 selects the runtime-dispatched kernels (testing aid):
  // b200_bitonic_set_tuning(t, 100 + r) == (t, r) with generic kernels.
  // min_run_bits >= 1000 disables programmatic dependent launch (testing aid)
  g_pdl.store(min_run_bits >= 1000 ? 0 : 1);
  if (min_run_bits >= 1000) min_run_bits -= 1000;
  g_force_generic.store(min_run_bits >= 100 ? 1 : 0);
  if (min_run_bits >= 100) min_run_bits -= 100;
  if (tile_bits != 0 && (tile_bits < 6 || tile_bits > b200::kMaxTileBits)) {
    return fail(B200_CONFIG, "tile_bits must be 0 (auto) or in [6, 15]");
  }
  if (min_run_bits < 2 || min_run_bits > 10) {
    return fail(B200_CONFIG, "min_run_bits must be in [2, 10]");
  }
  g_tile_bits.store(tile_bits);
  g_min_run_bits.store(min_run_bits);
  return B200_OK;
}

const char* b200_bitonic_last_error(void) { return g_last_error.c_str(); }

const char* b200_bitonic_version(void) { return "b200-bitonic 0.1 (sm_100a)"; }

}  // extern "C"
