// H2D / D2H bandwidth for different host-buffer kinds (development probe).
#include <cuda_runtime.h>
#include <sys/mman.h>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <algorithm>
#include <vector>

static float timed(cudaStream_t s, void* dst, const void* src, size_t bytes, cudaMemcpyKind kind) {
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  std::vector<float> t;
  for (int r = 0; r < 15; ++r) {
    cudaEventRecord(a, s);
    cudaMemcpyAsync(dst, src, bytes, kind, s);
    cudaEventRecord(b, s);
    cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    if (r >= 3) t.push_back(ms);
  }
  std::sort(t.begin(), t.end());
  return t[t.size() / 2] * 1e3f;
}

int main() {
  cudaStream_t s; cudaStreamCreate(&s);
  for (size_t bytes : {size_t(4) << 20, size_t(64) << 20}) {
    void* d; cudaMalloc(&d, bytes);
    struct K { const char* name; void* p; } kinds[4];
    void* p0; cudaHostAlloc(&p0, bytes, cudaHostAllocDefault); kinds[0] = {"hostalloc", p0};
    void* p1; cudaHostAlloc(&p1, bytes, cudaHostAllocWriteCombined); kinds[1] = {"writecombined", p1};
    void* p2 = aligned_alloc(4096, bytes); memset(p2, 1, bytes);
    cudaHostRegister(p2, bytes, cudaHostRegisterDefault); kinds[2] = {"register4k", p2};
    void* p3 = mmap(nullptr, bytes, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
    madvise(p3, bytes, MADV_HUGEPAGE); memset(p3, 1, bytes);
    cudaHostRegister(p3, bytes, cudaHostRegisterDefault); kinds[3] = {"register_thp", p3};
    for (auto& k : kinds) {
      memset(k.p, 2, bytes);
      float h2d = timed(s, d, k.p, bytes, cudaMemcpyHostToDevice);
      float d2h = timed(s, k.p, d, bytes, cudaMemcpyDeviceToHost);
      printf("%3zu MB %-14s H2D %8.1f us (%5.1f GB/s)  D2H %8.1f us (%5.1f GB/s)\n", bytes >> 20,
             k.name, h2d, bytes / h2d / 1e3, d2h, bytes / d2h / 1e3);
    }
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
