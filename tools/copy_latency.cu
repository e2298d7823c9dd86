// Host wall time vs device time of H2D + D2H of 4 MiB pinned (dev probe).
#include <cuda_runtime.h>
#include <chrono>
#include <cstdio>
#include <vector>
#include <algorithm>
int main() {
  const size_t bytes = 4 << 20;
  void *h, *d;
  cudaHostAlloc(&h, bytes, 0);
  cudaMalloc(&d, bytes);
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int chunks : {1, 2, 4, 8}) {
    std::vector<double> wall, dev;
    for (int r = 0; r < 30; ++r) {
      auto t0 = std::chrono::steady_clock::now();
      cudaEventRecord(a, s);
      for (int c = 0; c < chunks; ++c)
        cudaMemcpyAsync((char*)d + c * bytes / chunks, (char*)h + c * bytes / chunks,
                        bytes / chunks, cudaMemcpyHostToDevice, s);
      for (int c = 0; c < chunks; ++c)
        cudaMemcpyAsync((char*)h + c * bytes / chunks, (char*)d + c * bytes / chunks,
                        bytes / chunks, cudaMemcpyDeviceToHost, s);
      cudaEventRecord(b, s);
      cudaStreamSynchronize(s);
      auto t1 = std::chrono::steady_clock::now();
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (r >= 5) {
        wall.push_back(std::chrono::duration<double, std::micro>(t1 - t0).count());
        dev.push_back(ms * 1e3);
      }
    }
    std::sort(wall.begin(), wall.end());
    std::sort(dev.begin(), dev.end());
    printf("chunks %d: host wall %.1f us, device %.1f us\n", chunks, wall[wall.size() / 2],
           dev[dev.size() / 2]);
  }
  // spin vs blocking sync flags make no difference to DMA latency; also try a
  // device-side dummy kernel-free path: H2D only
  return 0;
}
