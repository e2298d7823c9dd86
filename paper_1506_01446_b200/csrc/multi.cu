// multi.cu -- merge-path entries and the partitioned (multi-GPU) sort: the
// merge-split compare-exchange of the rank-level bitonic network, the
// one-process multi-device driver (peer reads inside the merge kernel) and
// the CUDA IPC helpers of the one-process-per-GPU driver (dist.py).
#include <cuda_runtime.h>

#include <algorithm>
#include <mutex>
#include <utility>
#include <vector>

#include "runtime.hpp"

using namespace b200::rt;

namespace {
// *count += keys of the output window [o_begin, o_begin + o_len) that came
// from B (the partner): o_len - (keys from A) = o_len - (cor[last] - cor[0]).
__global__ void count_partner_keys(const uint64_t* cor, uint64_t tiles, uint64_t o_len,
                                   unsigned long long* count) {
  atomicAdd(count, (unsigned long long)(o_len - (cor[tiles] - cor[0])));
}
}  // namespace

namespace b200::rt {
struct MultiCtx {
  std::vector<int> devs;
  uint64_t m = 0;
  std::vector<cudaStream_t> st;
  std::vector<cudaEvent_t> ev;
  std::vector<uint32_t*> scratch;
  std::vector<uint64_t*> cor;
  void release() {
    for (size_t r = 0; r < devs.size(); ++r) {
      cudaSetDevice(devs[r]);
      if (r < st.size() && st[r]) cudaStreamSynchronize(st[r]);
      if (r < scratch.size() && scratch[r]) cudaFree(scratch[r]);
      if (r < cor.size() && cor[r]) cudaFree(cor[r]);
      if (r < ev.size() && ev[r]) cudaEventDestroy(ev[r]);
      if (r < st.size() && st[r]) cudaStreamDestroy(st[r]);
    }
    devs.clear();
    st.clear();
    ev.clear();
    scratch.clear();
    cor.clear();
    m = 0;
  }
};
std::mutex g_multi_mu;
MultiCtx g_multi;
std::vector<std::pair<int, int>> g_peer_enabled;

void release_multi_ctx() {
  std::lock_guard<std::mutex> lk(g_multi_mu);
  int prev = 0;
  cudaGetDevice(&prev);
  g_multi.release();
  cudaSetDevice(prev);
}

}  // namespace b200::rt

extern "C" {

int b200_bitonic_merge_u32(const uint32_t* a, uint64_t la, const uint32_t* b,
                           uint64_t lb, uint32_t key_xor, uint32_t* out,
                           b200_stream_t stream) {
  if (la + lb == 0) return B200_OK;
  if ((la && !a) || (lb && !b) || !out) return fail(B200_CONFIG, "null pointer");
  if ((la && out == a) || (lb && out == b)) {
    return fail(B200_CONFIG, "out must not alias the inputs");
  }
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const uint64_t tiles = (la + lb + b200::kMergeTile - 1) / b200::kMergeTile;
  uint64_t* cor = nullptr;
  B200_CUDA_TRY(scratch_alloc(&cor, (tiles + 1) * sizeof(uint64_t), s));
  int rc = merge_window_impl(a, la, b, lb, 0, la + lb, key_xor, out, cor, s);
  cudaFreeAsync(cor, s);
  return rc;
}

int b200_bitonic_merge_split_u32(const uint32_t* local, const uint32_t* partner,
                                 uint64_t m, int keep_high, uint32_t key_xor,
                                 uint32_t* out, b200_stream_t stream) {
  if (m < 1) return fail(B200_INVALID_SIZE, "shard must hold >= 1 key");
  if (!local || !partner || !out) return fail(B200_CONFIG, "null pointer");
  if (out == local || out == partner) {
    return fail(B200_CONFIG, "out must not alias the inputs");
  }
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const uint64_t tiles = (m + b200::kMergeTile - 1) / b200::kMergeTile;
  uint64_t* cor = nullptr;
  B200_CUDA_TRY(scratch_alloc(&cor, (tiles + 1) * sizeof(uint64_t), s));
  int rc = merge_split_impl(local, partner, m, keep_high, key_xor, out, cor, s);
  cudaFreeAsync(cor, s);
  return rc;
}

int b200_bitonic_merge_split_u32_count(const uint32_t* local, const uint32_t* partner,
                                       uint64_t m, int keep_high, uint32_t key_xor,
                                       uint32_t* out, b200_stream_t stream,
                                       uint64_t* d_partner_keys) {
  if (m < 1) return fail(B200_INVALID_SIZE, "shard must hold >= 1 key");
  if (!local || !partner || !out) return fail(B200_CONFIG, "null pointer");
  if (out == local || out == partner) {
    return fail(B200_CONFIG, "out must not alias the inputs");
  }
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const uint64_t tiles = (m + b200::kMergeTile - 1) / b200::kMergeTile;
  uint64_t* cor = nullptr;
  B200_CUDA_TRY(scratch_alloc(&cor, (tiles + 1) * sizeof(uint64_t), s));
  int rc = merge_split_impl(local, partner, m, keep_high, key_xor, out, cor, s);
  if (rc == B200_OK && d_partner_keys) {
    count_partner_keys<<<1, 1, 0, s>>>(cor, tiles, m,
                                       reinterpret_cast<unsigned long long*>(d_partner_keys));
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) rc = cuda_fail(e, "partner key count");
  }
  cudaFreeAsync(cor, s);
  return rc;
}

// ---- cross-process stream ordering (interprocess events) -------------------
int b200_bitonic_ipc_event_create(void** event, b200_ipc_handle* handle) {
  if (!event || !handle) return fail(B200_CONFIG, "bad ipc_event_create arguments");
  static_assert(sizeof(cudaIpcEventHandle_t) <= sizeof(b200_ipc_handle), "handle size");
  cudaEvent_t e = nullptr;
  B200_CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming | cudaEventInterprocess));
  cudaIpcEventHandle_t h;
  cudaError_t err = cudaIpcGetEventHandle(&h, e);
  if (err != cudaSuccess) {
    cudaEventDestroy(e);
    return cuda_fail(err, "cudaIpcGetEventHandle");
  }
  std::memset(handle, 0, sizeof(*handle));
  std::memcpy(handle->bytes, &h, sizeof(h));
  *event = e;
  return B200_OK;
}

int b200_bitonic_ipc_event_open(const b200_ipc_handle* handle, void** event) {
  if (!event || !handle) return fail(B200_CONFIG, "bad ipc_event_open arguments");
  cudaIpcEventHandle_t h;
  std::memcpy(&h, handle->bytes, sizeof(h));
  cudaEvent_t e = nullptr;
  B200_CUDA_TRY(cudaIpcOpenEventHandle(&e, h));
  *event = e;
  return B200_OK;
}

int b200_bitonic_event_destroy(void* event) {
  if (event) B200_CUDA_TRY(cudaEventDestroy(reinterpret_cast<cudaEvent_t>(event)));
  return B200_OK;
}

int b200_bitonic_event_record(void* event, b200_stream_t stream) {
  if (!event) return fail(B200_CONFIG, "null event");
  B200_CUDA_TRY(cudaEventRecord(reinterpret_cast<cudaEvent_t>(event),
                                reinterpret_cast<cudaStream_t>(stream)));
  return B200_OK;
}

int b200_bitonic_stream_wait_event(b200_stream_t stream, void* event) {
  if (!event) return fail(B200_CONFIG, "null event");
  B200_CUDA_TRY(cudaStreamWaitEvent(reinterpret_cast<cudaStream_t>(stream),
                                    reinterpret_cast<cudaEvent_t>(event), 0));
  return B200_OK;
}

int b200_bitonic_ipc_alloc(uint64_t bytes, void** d_ptr, b200_ipc_handle* handle) {
  if (!d_ptr || !handle || bytes == 0) return fail(B200_CONFIG, "bad ipc_alloc arguments");
  static_assert(sizeof(cudaIpcMemHandle_t) <= sizeof(b200_ipc_handle), "handle size");
  B200_CUDA_TRY(cudaMalloc(d_ptr, bytes));
  cudaIpcMemHandle_t h;
  cudaError_t e = cudaIpcGetMemHandle(&h, *d_ptr);
  if (e != cudaSuccess) {
    cudaFree(*d_ptr);
    *d_ptr = nullptr;
    return cuda_fail(e, "cudaIpcGetMemHandle");
  }
  std::memset(handle, 0, sizeof(*handle));
  std::memcpy(handle->bytes, &h, sizeof(h));
  return B200_OK;
}

int b200_bitonic_ipc_free(void* d_ptr) {
  if (d_ptr) B200_CUDA_TRY(cudaFree(d_ptr));
  return B200_OK;
}

int b200_bitonic_ipc_open(const b200_ipc_handle* handle, void** d_ptr) {
  if (!d_ptr || !handle) return fail(B200_CONFIG, "bad ipc_open arguments");
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle->bytes, sizeof(h));
  B200_CUDA_TRY(cudaIpcOpenMemHandle(d_ptr, h, cudaIpcMemLazyEnablePeerAccess));
  return B200_OK;
}

int b200_bitonic_ipc_close(void* d_ptr) {
  if (d_ptr) B200_CUDA_TRY(cudaIpcCloseMemHandle(d_ptr));
  return B200_OK;
}

int b200_bitonic_copy(void* dst, const void* src, uint64_t bytes, b200_stream_t stream) {
  if (bytes == 0) return B200_OK;
  if (!dst || !src) return fail(B200_CONFIG, "null pointer");
  B200_CUDA_TRY(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice,
                                reinterpret_cast<cudaStream_t>(stream)));
  return B200_OK;
}

// Rank-level bitonic network over G sorted shards (block bitonic sort with
// merge-split compare-exchanges).  Same direction rule as the reference's
// network (schedule.cpp:58-67) applied to shard indices.  The streams,
// events, scratch shards and corank buffers of the last (devices, m) are
// kept for the next call (released by b200_bitonic_release_scratch), and
// peer access is enabled once per device pair.
int b200_bitonic_sort_u32_multi(uint32_t* const* d_shards, const int* devices,
                                int ngpu, uint64_t n_total, int descending) {
  if (ngpu != 1 && ngpu != 2 && ngpu != 4 && ngpu != 8) {
    return fail(B200_CONFIG, "ngpu must be 1, 2, 4 or 8");
  }
  if (!d_shards || !devices) return fail(B200_CONFIG, "null pointer");
  if (n_total < 2 || !is_pow2(n_total) || n_total < (uint64_t)ngpu * 2) {
    return fail(B200_INVALID_SIZE,
                "n_total must be a power of two >= 2*ngpu");
  }
  if (descending != 0 && descending != 1) {
    return fail(B200_CONFIG, "descending must be 0 or 1");
  }
  const uint64_t m = n_total / ngpu;
  const uint32_t gmask = descending ? 0xFFFFFFFFu : 0u;
  std::lock_guard<std::mutex> lk(g_multi_mu);
  int prev_dev = 0;
  B200_CUDA_TRY(cudaGetDevice(&prev_dev));
  struct Restore {
    int d;
    ~Restore() { cudaSetDevice(d); }
  } restore{prev_dev};

  // Enable peer access between distinct devices (once per ordered pair).
  for (int r = 0; r < ngpu; ++r) {
    for (int q = 0; q < ngpu; ++q) {
      if (devices[r] == devices[q]) continue;
      const std::pair<int, int> pr{devices[r], devices[q]};
      if (std::find(g_peer_enabled.begin(), g_peer_enabled.end(), pr) != g_peer_enabled.end())
        continue;
      int can = 0;
      B200_CUDA_TRY(cudaDeviceCanAccessPeer(&can, devices[r], devices[q]));
      if (!can) return fail(B200_CONFIG, "no peer access between devices");
      B200_CUDA_TRY(cudaSetDevice(devices[r]));
      cudaError_t e = cudaDeviceEnablePeerAccess(devices[q], 0);
      if (e == cudaErrorPeerAccessAlreadyEnabled) {
        cudaGetLastError();
      } else if (e != cudaSuccess) {
        return cuda_fail(e, "cudaDeviceEnablePeerAccess");
      }
      g_peer_enabled.push_back(pr);
    }
  }

  // Reuse the cached streams / events / scratch when (devices, m) repeats.
  MultiCtx& X = g_multi;
  const std::vector<int> devs(devices, devices + ngpu);
  const uint64_t tiles = (m + b200::kMergeTile - 1) / b200::kMergeTile;
  if (X.devs != devs || X.m != m) {
    X.release();
    X.devs = devs;
    X.m = m;
    X.st.assign(ngpu, nullptr);
    X.ev.assign(ngpu, nullptr);
    X.scratch.assign(ngpu, nullptr);
    X.cor.assign(ngpu, nullptr);
    for (int r = 0; r < ngpu; ++r) {
      cudaError_t e = cudaSetDevice(devices[r]);
      if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&X.st[r], cudaStreamNonBlocking);
      if (e == cudaSuccess) e = cudaEventCreateWithFlags(&X.ev[r], cudaEventDisableTiming);
      if (e == cudaSuccess && ngpu > 1) e = cudaMalloc(&X.scratch[r], m * 4);
      if (e == cudaSuccess && ngpu > 1) e = cudaMalloc(&X.cor[r], (tiles + 1) * sizeof(uint64_t));
      if (e != cudaSuccess) {
        X.release();
        return cuda_fail(e, "multi-GPU context");
      }
    }
  }
  std::vector<uint32_t*> cur(d_shards, d_shards + ngpu), tmp(X.scratch);
  int rc = B200_OK;
#define MTRY(expr)                                   \
  do {                                               \
    cudaError_t _e = (expr);                         \
    if (_e != cudaSuccess) return cuda_fail(_e, #expr); \
  } while (0)

  // the caller's writes to the shards (other streams) come first
  for (int r = 0; r < ngpu; ++r) {
    MTRY(cudaSetDevice(devices[r]));
    MTRY(cudaDeviceSynchronize());
  }
  // 1. local sorts (each shard ascending in the requested order)
  for (int r = 0; r < ngpu; ++r) {
    MTRY(cudaSetDevice(devices[r]));
    rc = sort_impl(cur[r], m, 1, descending, 0u, X.st[r]);
    if (rc != B200_OK) return rc;
  }
  // 2. rank-level network: phases q = 1..g, steps s = q..1
  int g = 0;
  while ((1 << g) < ngpu) ++g;
  for (int q = 1; q <= g; ++q) {
    for (int s = q; s >= 1; --s) {
      for (int r = 0; r < ngpu; ++r) {
        MTRY(cudaSetDevice(devices[r]));
        MTRY(cudaEventRecord(X.ev[r], X.st[r]));
      }
      for (int r = 0; r < ngpu; ++r) {
        const int partner = r ^ (1 << (s - 1));
        MTRY(cudaSetDevice(devices[r]));
        MTRY(cudaStreamWaitEvent(X.st[r], X.ev[partner], 0));
        const bool ascending = ((r >> q) & 1) == 0;
        const bool lower = r < partner;
        const int keep_high = (lower == ascending) ? 0 : 1;
        rc = merge_split_impl(cur[r], cur[partner], m, keep_high, gmask, tmp[r], X.cor[r],
                              X.st[r]);
        if (rc != B200_OK) return rc;
      }
      // both halves of every pair must finish reading before buffers swap
      for (int r = 0; r < ngpu; ++r) {
        MTRY(cudaSetDevice(devices[r]));
        MTRY(cudaEventRecord(X.ev[r], X.st[r]));
      }
      for (int r = 0; r < ngpu; ++r) {
        const int partner = r ^ (1 << (s - 1));
        MTRY(cudaSetDevice(devices[r]));
        MTRY(cudaStreamWaitEvent(X.st[r], X.ev[partner], 0));
      }
      std::swap(cur, tmp);
    }
  }
  // 3. results must end in the caller's buffers
  for (int r = 0; r < ngpu; ++r) {
    if (cur[r] != d_shards[r]) {
      MTRY(cudaSetDevice(devices[r]));
      MTRY(cudaMemcpyAsync(d_shards[r], cur[r], m * 4, cudaMemcpyDeviceToDevice, X.st[r]));
    }
  }
  for (int r = 0; r < ngpu; ++r) {
    MTRY(cudaSetDevice(devices[r]));
    MTRY(cudaStreamSynchronize(X.st[r]));
  }
#undef MTRY
  return B200_OK;
}

}  // extern "C"
