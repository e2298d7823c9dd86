// multi.cu -- merge-path entries and the partitioned (multi-GPU) sort: the
// merge-split compare-exchange of the rank-level bitonic network, the
// one-process multi-device driver (peer reads inside the merge kernel) and
// the CUDA IPC helpers of the one-process-per-GPU driver (dist.py).
#include <cuda_runtime.h>

#include "runtime.hpp"

using namespace b200::rt;

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
// network (schedule.cpp:58-67) applied to shard indices.
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
  int prev_dev = 0;
  B200_CUDA_TRY(cudaGetDevice(&prev_dev));

  // Enable peer access between distinct devices.
  for (int r = 0; r < ngpu; ++r) {
    for (int q = 0; q < ngpu; ++q) {
      if (devices[r] == devices[q]) continue;
      int can = 0;
      B200_CUDA_TRY(cudaDeviceCanAccessPeer(&can, devices[r], devices[q]));
      if (!can) {
        cudaSetDevice(prev_dev);
        return fail(B200_CONFIG, "no peer access between devices");
      }
      B200_CUDA_TRY(cudaSetDevice(devices[r]));
      cudaError_t e = cudaDeviceEnablePeerAccess(devices[q], 0);
      if (e == cudaErrorPeerAccessAlreadyEnabled) {
        cudaGetLastError();
      } else if (e != cudaSuccess) {
        cudaSetDevice(prev_dev);
        return cuda_fail(e, "cudaDeviceEnablePeerAccess");
      }
    }
  }

  std::vector<cudaStream_t> st(ngpu, nullptr);
  std::vector<cudaEvent_t> ev(ngpu, nullptr);
  std::vector<uint32_t*> cur(d_shards, d_shards + ngpu), tmp(ngpu, nullptr);
  std::vector<uint32_t*> scratch(ngpu, nullptr);
  std::vector<uint64_t*> cor(ngpu, nullptr);
  const uint64_t tiles = (m + b200::kMergeTile - 1) / b200::kMergeTile;
  int rc = B200_OK;
  auto cleanup = [&]() {
    for (int r = 0; r < ngpu; ++r) {
      cudaSetDevice(devices[r]);
      if (st[r]) cudaStreamSynchronize(st[r]);
      if (scratch[r]) cudaFree(scratch[r]);
      if (cor[r]) cudaFree(cor[r]);
      if (ev[r]) cudaEventDestroy(ev[r]);
      if (st[r]) cudaStreamDestroy(st[r]);
    }
    cudaSetDevice(prev_dev);
  };
#define MTRY(expr)                                   \
  do {                                               \
    cudaError_t _e = (expr);                         \
    if (_e != cudaSuccess) {                         \
      rc = cuda_fail(_e, #expr);                     \
      cleanup();                                     \
      return rc;                                     \
    }                                                \
  } while (0)

  for (int r = 0; r < ngpu; ++r) {
    MTRY(cudaSetDevice(devices[r]));
    MTRY(cudaStreamCreateWithFlags(&st[r], cudaStreamNonBlocking));
    MTRY(cudaEventCreateWithFlags(&ev[r], cudaEventDisableTiming));
    if (ngpu > 1) {
      MTRY(cudaMalloc(&scratch[r], m * 4));
      tmp[r] = scratch[r];
      MTRY(cudaMalloc(&cor[r], (tiles + 1) * sizeof(uint64_t)));
    }
  }
  // 1. local sorts (each shard ascending in the requested order)
  for (int r = 0; r < ngpu; ++r) {
    MTRY(cudaSetDevice(devices[r]));
    rc = sort_impl(cur[r], m, 1, descending, 0u, st[r]);
    if (rc != B200_OK) {
      std::string msg = g_last_error;
      cleanup();
      g_last_error = msg;
      return rc;
    }
  }
  // 2. rank-level network: phases q = 1..g, steps s = q..1
  int g = 0;
  while ((1 << g) < ngpu) ++g;
  for (int q = 1; q <= g; ++q) {
    for (int s = q; s >= 1; --s) {
      for (int r = 0; r < ngpu; ++r) {
        MTRY(cudaSetDevice(devices[r]));
        MTRY(cudaEventRecord(ev[r], st[r]));
      }
      for (int r = 0; r < ngpu; ++r) {
        const int partner = r ^ (1 << (s - 1));
        MTRY(cudaSetDevice(devices[r]));
        MTRY(cudaStreamWaitEvent(st[r], ev[partner], 0));
        const bool ascending = ((r >> q) & 1) == 0;
        const bool lower = r < partner;
        const int keep_high = (lower == ascending) ? 0 : 1;
        rc = merge_split_impl(cur[r], cur[partner], m, keep_high, gmask,
                              tmp[r], cor[r], st[r]);
        if (rc != B200_OK) {
          std::string msg = g_last_error;
          cleanup();
          g_last_error = msg;
          return rc;
        }
      }
      // both halves of every pair must finish reading before buffers swap
      for (int r = 0; r < ngpu; ++r) {
        MTRY(cudaSetDevice(devices[r]));
        MTRY(cudaEventRecord(ev[r], st[r]));
      }
      for (int r = 0; r < ngpu; ++r) {
        const int partner = r ^ (1 << (s - 1));
        MTRY(cudaSetDevice(devices[r]));
        MTRY(cudaStreamWaitEvent(st[r], ev[partner], 0));
      }
      std::swap(cur, tmp);
    }
  }
  // 3. results must end in the caller's buffers
  for (int r = 0; r < ngpu; ++r) {
    if (cur[r] != d_shards[r]) {
      MTRY(cudaSetDevice(devices[r]));
      MTRY(cudaMemcpyAsync(d_shards[r], cur[r], m * 4, cudaMemcpyDeviceToDevice,
                           st[r]));
    }
  }
  for (int r = 0; r < ngpu; ++r) {
    MTRY(cudaSetDevice(devices[r]));
    MTRY(cudaStreamSynchronize(st[r]));
  }
  cleanup();
#undef MTRY
  return B200_OK;
}

}  // extern "C"
