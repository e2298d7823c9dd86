// runtime.hpp -- internal interface between the host translation units of
// the library (bitonic_sort.cu: launcher, plans, graphs, merge path and the
// device entries; host_entry.cu: the pipelined host-span entry; multi.cu: the
// multi-GPU, merge and peer-memory entries).  Not installed, not part of the
// C ABI.
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/b200_bitonic.h"
#include "merge_consts.hpp"
#include "planner.hpp"

namespace b200::rt {

// ---- errors: status code + thread-local message (b200_bitonic_last_error)
extern thread_local std::string g_last_error;
int fail(int code, const std::string& msg);
int cuda_fail(cudaError_t e, const char* what);

#define B200_CUDA_TRY(expr)                        \
  do {                                             \
    cudaError_t _e = (expr);                       \
    if (_e != cudaSuccess) return cuda_fail(_e, #expr); \
  } while (0)

// ---- process-wide tuning (b200_bitonic_set_tuning) and the plan options
extern std::atomic<int> g_tile_bits;
extern std::atomic<int> g_min_run_bits;
extern std::atomic<int> g_force_generic;
extern std::atomic<int> g_pdl;
b200::PlanOptions plan_options();

int log2_exact(uint64_t n);
bool is_pow2(uint64_t n);

// ---- retained stream-ordered scratch pool, one per device
cudaError_t scratch_alloc(void** p, size_t bytes, cudaStream_t s);
template <class T>
cudaError_t scratch_alloc(T** p, size_t bytes, cudaStream_t s) {
  return scratch_alloc(reinterpret_cast<void**>(p), bytes, s);
}
cudaError_t trim_scratch_pools();

// ---- CUDA graphs for repeated launch sequences (bitonic_sort.cu)
struct GraphKey {
  int dev, kind, mode, desc, k, G;
  const void* p0;
  const void* p1;
  uint64_t n, batch;
  uint32_t kx;
  int cmax, cmin, lrun, regbits, tile_regbits, cmerge, dp, generic, pdl;
  double trip_cost, wide_tail_cost, cluster_cost;
  int mixed_c, cluster, mid_lrun, regbits14, tile_c;
  uint64_t nreal;  // virtual padding: real keys (0 = none)
  bool operator==(const GraphKey& o) const { return std::memcmp(this, &o, sizeof(*this)) == 0; }
};
// An instantiated graph is shared between the cache and every caller that is
// about to launch it: the exec is destroyed only when the last owner lets go
// (cache eviction / drop_graphs and an in-flight launcher can race).
using GraphExecPtr = std::shared_ptr<CUgraphExec_st>;
GraphExecPtr own_exec(cudaGraphExec_t e);
struct GraphEntry {
  GraphKey key;
  int hits = 0;
  GraphExecPtr exec;
};
extern std::mutex g_graph_mu;
extern std::vector<GraphEntry> g_graphs;
extern thread_local cudaStream_t t_capture_stream[64];
bool graphs_enabled();
GraphKey make_key(int kind, const void* p0, const void* p1, uint64_t n, uint64_t batch,
                  int desc, uint32_t kx, int mode, int G, const b200::PlanOptions& o);
void drop_graphs();

// Runs fn(stream) directly, or through a cached graph once `key` repeats.
template <class Fn>
int run_graphed(const GraphKey& key, cudaStream_t s, Fn&& fn) {
  cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
  if (!graphs_enabled() || cudaStreamIsCapturing(s, &st) != cudaSuccess ||
      st != cudaStreamCaptureStatusNone) {
    cudaGetLastError();
    return fn(s);
  }
  GraphExecPtr exec;
  bool capture = false;
  {
    std::lock_guard<std::mutex> lk(g_graph_mu);
    auto it = std::find_if(g_graphs.begin(), g_graphs.end(),
                           [&](const GraphEntry& e) { return e.key == key; });
    if (it == g_graphs.end()) {
      if (g_graphs.size() >= 64) g_graphs.erase(g_graphs.begin());  // FIFO eviction
      GraphEntry e;
      e.key = key;
      e.hits = 1;
      g_graphs.push_back(e);
    } else {
      exec = it->exec;  // shared ownership: eviction cannot free it under us
      capture = !exec;
      ++it->hits;
    }
  }
  if (!exec && !capture) return fn(s);  // first sighting: launch directly
  if (!exec) {
    cudaStream_t& cs = t_capture_stream[key.dev & 63];
    if (cs == nullptr) B200_CUDA_TRY(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
    B200_CUDA_TRY(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
    int rc = fn(cs);
    cudaGraph_t g = nullptr;
    cudaError_t e = cudaStreamEndCapture(cs, &g);
    if (rc != B200_OK) {
      if (g) cudaGraphDestroy(g);
      return rc;
    }
    if (e != cudaSuccess) return cuda_fail(e, "graph capture");
    cudaGraphExec_t raw = nullptr;
    e = cudaGraphInstantiateWithFlags(&raw, g, 0);
    cudaGraphDestroy(g);
    if (e != cudaSuccess) return cuda_fail(e, "graph instantiate");
    exec = own_exec(raw);
    std::lock_guard<std::mutex> lk(g_graph_mu);
    auto it = std::find_if(g_graphs.begin(), g_graphs.end(),
                           [&](const GraphEntry& x) { return x.key == key; });
    if (it != g_graphs.end() && !it->exec) it->exec = exec;
    // else: another thread won the race (or the entry was evicted); ours is
    // launched once below and freed with its last owner
  }
  B200_CUDA_TRY(cudaGraphLaunch(exec.get(), s));
  return B200_OK;
}

// ---- multi-GPU context (multi.cu): cached streams / scratch of sort_u32_multi
void release_multi_ctx();

// ---- the sort and the merge path
// Validates and runs the whole plan (or only pass `only`, when >= 0).
// key_xor: 0x80000000 for int32 keys (for 64-bit keys: applied to the hi
// word).  d_vals: payloads (mode 1) or the lo words of 64-bit keys whose hi
// words are d_keys (mode 2).
int sort_impl(uint32_t* d_keys, uint64_t n_per, uint64_t batch, int descending,
              uint32_t key_xor, cudaStream_t stream, int only = -1,
              uint32_t* d_vals = nullptr, int mode = -1, uint64_t nreal = 0);
// Output window [o_begin, o_begin + o_len) of merge(A[0..la), B[0..lb)).
int merge_window_impl(const uint32_t* A, uint64_t la, const uint32_t* B, uint64_t lb,
                      uint64_t o_begin, uint64_t o_len, uint32_t key_xor, uint32_t* out,
                      uint64_t* scratch_coranks, cudaStream_t s);
int merge_split_impl(const uint32_t* local, const uint32_t* partner, uint64_t m,
                     int keep_high, uint32_t key_xor, uint32_t* out,
                     uint64_t* scratch_coranks, cudaStream_t s);

}  // namespace b200::rt
