// Host wall time of b200_bitonic_sort_host_u32 on a pinned 2^20 span, called
// from C++ (no Python in the loop).  Development probe.
#include <cuda_runtime.h>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <random>
#include <vector>
#include <algorithm>
#include "../include/b200_bitonic.h"
int main(int argc, char** argv) {
  const int k = argc > 1 ? atoi(argv[1]) : 20;
  const uint64_t n = 1ull << k;
  uint32_t *h, *src;
  cudaHostAlloc((void**)&h, n * 4, 0);
  src = (uint32_t*)malloc(n * 4);
  std::mt19937 g(1);
  for (uint64_t i = 0; i < n; ++i) src[i] = g();
  std::vector<double> t;
  for (int r = 0; r < 40; ++r) {
    memcpy(h, src, n * 4);
    auto t0 = std::chrono::steady_clock::now();
    int rc = b200_bitonic_sort_host_u32(h, n, 0);
    auto t1 = std::chrono::steady_clock::now();
    if (rc) { printf("rc %d %s\n", rc, b200_bitonic_last_error()); return 1; }
    if (r >= 5) t.push_back(std::chrono::duration<double, std::micro>(t1 - t0).count());
  }
  for (uint64_t i = 1; i < n; ++i) if (h[i - 1] > h[i]) { printf("unsorted\n"); return 1; }
  std::sort(t.begin(), t.end());
  printf("k=%d host entry from C++: median %.1f us min %.1f us (%.2f Gkeys/s)\n", k,
         t[t.size() / 2], t[0], n / t[t.size() / 2] / 1e3);
  return 0;
}
