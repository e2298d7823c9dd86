// host_entry.cu -- the host-span entries (b200_bitonic_sort_host_*), the
// drop-ins for the reference's sequential_bitonic_sort(span)
// (engine.hpp:102-104), and b200_bitonic_release_scratch.
#include <cuda_runtime.h>

#include <chrono>
#include <cstdio>
#include <random>

#include "runtime.hpp"

namespace b200::rt {

// ---- host-span entry: pipelined H2D / sort / D2H ----------------------------
// The reference's entry points sort host spans (sequential_bitonic_sort,
// engine.hpp:102-104).  Here the span is cut into G chunks: chunk j's H2D
// copy overlaps the bitonic sort of the chunks already on the device (one
// stream per chunk); the sorted chunks are combined by a merge-path tree
// (the merge kernels of the multi-GPU path), and the last merge is cut into
// output windows so each window's D2H copy overlaps the merge of the next.
// Device buffers and streams are cached per device (retained pool memory).
struct HostPipe {
  static constexpr int kMaxChunks = 8;
  bool init = false;
  cudaStream_t h2d = nullptr, d2h = nullptr, comp[kMaxChunks] = {};
  std::vector<cudaEvent_t> ev;
  std::mutex mu;
  void* block = nullptr;  // device buffers, see pipe_buffers
  size_t cap = 0;
};
std::mutex g_pipe_mu;
std::vector<std::vector<HostPipe*>> g_pipes;  // per device; live for the process
constexpr int kMaxPipesPerDevice = 4;

// A free pipeline context of device `dev`, returned locked: concurrent host
// sorts on one device each get their own buffers and streams (up to
// kMaxPipesPerDevice, then they queue on the first).
HostPipe* host_pipe(int dev, std::unique_lock<std::mutex>& held) {
  HostPipe* wait_on = nullptr;
  {
    std::lock_guard<std::mutex> lk(g_pipe_mu);
    if ((int)g_pipes.size() <= dev) g_pipes.resize(dev + 1);
    auto& v = g_pipes[dev];
    for (HostPipe* hp : v) {
      std::unique_lock<std::mutex> t(hp->mu, std::try_to_lock);
      if (t.owns_lock()) {
        held = std::move(t);
        return hp;
      }
    }
    if ((int)v.size() < kMaxPipesPerDevice) {
      v.push_back(new HostPipe());
      held = std::unique_lock<std::mutex>(v.back()->mu);
      return v.back();
    }
    wait_on = v.front();
  }
  held = std::unique_lock<std::mutex>(wait_on->mu);
  return wait_on;
}

cudaError_t pipe_init(HostPipe& P) {
  if (P.init) return cudaSuccess;
  cudaError_t e = cudaStreamCreateWithFlags(&P.h2d, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&P.d2h, cudaStreamNonBlocking);
  for (int j = 0; j < HostPipe::kMaxChunks && e == cudaSuccess; ++j)
    e = cudaStreamCreateWithFlags(&P.comp[j], cudaStreamNonBlocking);
  while (e == cudaSuccess && P.ev.size() < 64) {
    cudaEvent_t x;
    e = cudaEventCreateWithFlags(&x, cudaEventDisableTiming);
    if (e == cudaSuccess) P.ev.push_back(x);
  }
  if (e == cudaSuccess) P.init = true;
  return e;
}

// Chunk count: chunks of >= 2^22 keys (16 MiB), at most 8 (measured on B200
// + PCIe 5: up to 2^22 keys one chunk wins; at 2^24, 4 chunks save ~10%).
int pipe_chunks(uint64_t n) {
  if (const char* e = std::getenv("B200_BITONIC_HOST_CHUNKS")) {
    int g = std::atoi(e);
    if (g >= 1 && g <= HostPipe::kMaxChunks && (g & (g - 1)) == 0 && n / g >= 2) return g;
  }
  int g = 1;
  while (g < HostPipe::kMaxChunks && n / (uint64_t)(2 * g) >= (uint64_t{1} << 22)) g *= 2;
  return g;
}

// Device buffers for the host entry: [A: n keys | B: n keys | coranks],
// one allocation per device, grown on demand and kept (graphs refer to it).
cudaError_t pipe_buffers(HostPipe& P, uint64_t n, uint64_t cor_words) {
  const size_t need = n * 8 + cor_words * 8;
  if (P.cap >= need) return cudaSuccess;
  if (P.block) {
    // every earlier call on this pipe joined into comp[0] and was waited for
    // (the caller holds P.mu); sync it anyway instead of the whole device
    cudaError_t e = cudaStreamSynchronize(P.comp[0]);
    if (e != cudaSuccess) return e;
    drop_graphs();  // captured pipelines refer to the old block
    cudaFree(P.block);
    P.block = nullptr;
    P.cap = 0;
  }
  cudaError_t e = cudaMalloc(&P.block, need);
  if (e == cudaSuccess) P.cap = need;
  return e;
}

int host_sort(uint32_t* h, uint64_t n, int descending, uint32_t key_xor) {
  if (n < 2 || !is_pow2(n)) {
    return fail(B200_INVALID_SIZE,
                "length must be a power of two >= 2, got " + std::to_string(n));
  }
  if (h == nullptr) return fail(B200_CONFIG, "null key pointer");
  if (descending != 0 && descending != 1) {
    return fail(B200_CONFIG, "descending must be 0 or 1");
  }
  int dev = 0;
  B200_CUDA_TRY(cudaGetDevice(&dev));
  std::unique_lock<std::mutex> lk;
  HostPipe& P = *host_pipe(dev, lk);
  B200_CUDA_TRY(pipe_init(P));
  const int G = pipe_chunks(n);
  const uint64_t c = n / G;
  const uint32_t kx = key_xor ^ (descending ? 0xFFFFFFFFu : 0u);
  const uint64_t cor_per_round = n / b200::kMergeTile + 2 * HostPipe::kMaxChunks + 2;
  int rounds = 0;
  while ((1 << rounds) < G) ++rounds;
  B200_CUDA_TRY(pipe_buffers(P, n, cor_per_round * (rounds + 1)));
  uint32_t* A = reinterpret_cast<uint32_t*>(P.block);
  uint32_t* B = A + n;
  uint64_t* cor = reinterpret_cast<uint64_t*>(B + n);

  // The whole pipeline, forked from and joined back into `origin`.
  auto pipeline = [&](cudaStream_t origin) -> int {
    int rc = B200_OK;
    size_t evi = 0;
    auto dep = [&](cudaStream_t from, cudaStream_t to) {
      if (from == to) return;
      cudaEvent_t x = P.ev[evi++ % P.ev.size()];
      cudaEventRecord(x, from);
      cudaStreamWaitEvent(to, x, 0);
    };
    if (G == 1) {
      cudaError_t e = cudaMemcpyAsync(A, h, n * 4, cudaMemcpyHostToDevice, origin);
      if (e != cudaSuccess) return cuda_fail(e, "H2D copy");
      rc = sort_impl(A, n, 1, descending, key_xor, origin);
      if (rc != B200_OK) return rc;
      e = cudaMemcpyAsync(h, A, n * 4, cudaMemcpyDeviceToHost, origin);
      return e == cudaSuccess ? B200_OK : cuda_fail(e, "D2H copy");
    }
    dep(origin, P.h2d);
    for (int j = 0; j < G; ++j) dep(origin, P.comp[j]);
    // 1. chunk j: H2D on the copy stream, then its sort on stream j
    for (int j = 0; j < G && rc == B200_OK; ++j) {
      cudaError_t e = cudaMemcpyAsync(A + j * c, h + j * c, c * 4, cudaMemcpyHostToDevice,
                                      P.h2d);
      if (e != cudaSuccess) {
        rc = cuda_fail(e, "H2D copy");
        break;
      }
      dep(P.h2d, P.comp[j]);
      rc = sort_impl(A + j * c, c, 1, descending, key_xor, P.comp[j]);
    }
    // 2. merge tree: run r lives on stream comp[owner[r]]
    std::vector<int> owner(G);
    for (int j = 0; j < G; ++j) owner[j] = j;
    uint32_t* src = A;
    uint32_t* dst = B;
    uint64_t len = c;
    int runs = G, round = 0;
    while (runs > 2 && rc == B200_OK) {
      std::vector<int> nowner(runs / 2);
      for (int q = 0; q < runs / 2 && rc == B200_OK; ++q) {
        cudaStream_t sq = P.comp[owner[2 * q]];
        dep(P.comp[owner[2 * q + 1]], sq);
        uint64_t* cq = cor + round * cor_per_round + q * (2 * len / b200::kMergeTile + 2);
        rc = merge_window_impl(src + 2 * q * len, len, src + (2 * q + 1) * len, len, 0,
                               2 * len, kx, dst + 2 * q * len, cq, sq);
        nowner[q] = owner[2 * q];
      }
      owner = nowner;
      std::swap(src, dst);
      len *= 2;
      runs /= 2;
      ++round;
    }
    // 3. last merge in output windows, each copied back as soon as it is done
    if (rc == B200_OK) {
      cudaStream_t sm = P.comp[owner[0]];
      dep(P.comp[owner[1]], sm);
      const int W = G;
      const uint64_t ow = n / W;
      uint64_t* cw = cor + round * cor_per_round;
      for (int w = 0; w < W && rc == B200_OK; ++w) {
        rc = merge_window_impl(src, len, src + len, len, w * ow, ow, kx, dst + w * ow, cw, sm);
        if (rc != B200_OK) break;
        dep(sm, P.d2h);
        cudaError_t e = cudaMemcpyAsync(h + w * ow, dst + w * ow, ow * 4,
                                        cudaMemcpyDeviceToHost, P.d2h);
        if (e != cudaSuccess) rc = cuda_fail(e, "D2H copy");
      }
    }
    // join every stream back into the origin
    dep(P.d2h, origin);
    dep(P.h2d, origin);
    for (int j = 0; j < G; ++j) dep(P.comp[j], origin);
    return rc;
  };

  // Graph only page-locked spans (a pageable copy cannot be captured).
  cudaPointerAttributes attr{};
  const bool pinned = cudaPointerGetAttributes(&attr, h) == cudaSuccess &&
                      attr.type == cudaMemoryTypeHost;
  cudaGetLastError();
  cudaStream_t s0 = P.comp[0];
  int rc;
  if (pinned) {
    rc = run_graphed(make_key(1, h, P.block, n, 1, descending, key_xor, 0, G, plan_options()),
                     s0, pipeline);
  } else {
    rc = pipeline(s0);
  }
  cudaError_t e = cudaStreamSynchronize(s0);
  if (rc == B200_OK && e != cudaSuccess) rc = cuda_fail(e, "host sort");
  return rc;
}

}  // namespace b200::rt

using namespace b200::rt;

extern "C" {

int b200_bitonic_release_scratch(void) {
  drop_graphs();
  release_multi_ctx();
  {
    std::lock_guard<std::mutex> lk(g_pipe_mu);
    for (auto& dv : g_pipes) {
      for (HostPipe* hp : dv) {
        if (hp == nullptr || hp->block == nullptr) continue;
        std::lock_guard<std::mutex> lk2(hp->mu);
        if (hp->init) cudaStreamSynchronize(hp->comp[0]);
        cudaFree(hp->block);
        hp->block = nullptr;
        hp->cap = 0;
      }
    }
  }
  const cudaError_t e = trim_scratch_pools();
  return e == cudaSuccess ? B200_OK : cuda_fail(e, "trim scratch pool");
}

int b200_bitonic_sort_host_i32(int32_t* h_keys, uint64_t n, int descending) {
  return host_sort(reinterpret_cast<uint32_t*>(h_keys), n, descending,
                   0x80000000u);
}

int b200_bitonic_sort_host_u32(uint32_t* h_keys, uint64_t n, int descending) {
  return host_sort(h_keys, n, descending, 0u);
}

// The reference's bench input (generate_input, bench.cpp:354-364): the low
// 32 bits of successive std::mt19937_64(seed) outputs.  Host-side input
// generation for benchmarks and callers that want the reference's workload;
// not part of the sort.
int b200_bitonic_generate_input(uint32_t* h_out, uint64_t n, uint64_t seed) {
  if (n < 1) return fail(B200_INVALID_SIZE, "input size must be >= 1");
  if (h_out == nullptr) return fail(B200_CONFIG, "null output pointer");
  std::mt19937_64 rng(seed);
  for (uint64_t i = 0; i < n; ++i) h_out[i] = static_cast<uint32_t>(rng());
  return B200_OK;
}

}  // extern "C"
