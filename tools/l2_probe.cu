// l2_probe.cu -- how fast is a read+write pass over an L2-resident block?
//
// An in-place streaming pass (every 16-byte vector read and written back,
// coalesced, grid = 148 x 8 CTAs x 256 threads, grid-stride) over a buffer
// of S bytes, repeated back to back; reports read+write bytes / time for S
// from 4 MB to 256 MB and three load cache policies: default (.ca), .lu
// (last use, the sort's streaming loads) and L2::evict_last.  If the 126 MB
// L2 keeps a block resident across passes, passes on it run at L2 rather
// than HBM bandwidth.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o l2_probe l2_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int MODE>
__global__ void pass(uint4* __restrict__ p, size_t nvec) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (; i < nvec; i += stride) {
    uint4 v;
    if (MODE == 0) {
      asm volatile("ld.global.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p + i));
    } else if (MODE == 1) {
      asm volatile("ld.global.lu.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p + i));
    } else {
      uint64_t pol;
      asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
      asm volatile("ld.global.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p + i), "l"(pol));
    }
    v.x ^= 1u;
    if (MODE == 2) {
      uint64_t pol;
      asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
      asm volatile("st.global.L2::cache_hint.v4.u32 [%0], {%1,%2,%3,%4}, %5;" :: "l"(p + i), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w), "l"(pol) : "memory");
    } else {
      asm volatile("st.global.v4.u32 [%0], {%1,%2,%3,%4};" :: "l"(p + i), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
    }
  }
}

int main() {
  const size_t maxb = 256ull << 20;
  uint4* d;
  cudaMalloc(&d, maxb);
  cudaMemset(d, 1, maxb);
  uint4* flush;
  cudaMalloc(&flush, 512ull << 20);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const size_t sizes_mb[] = {4, 8, 16, 24, 32, 48, 64, 80, 96, 128, 256};
  const char* names[] = {"default", "lu", "evict_last"};
  for (int mode = 0; mode < 3; ++mode) {
    for (size_t mb : sizes_mb) {
      const size_t bytes = mb << 20, nvec = bytes / 16;
      const int reps = 50;
      cudaMemset(flush, 0, 512ull << 20);
      auto launch = [&]() {
        if (mode == 0) pass<0><<<148 * 8, 256>>>(d, nvec);
        else if (mode == 1) pass<1><<<148 * 8, 256>>>(d, nvec);
        else pass<2><<<148 * 8, 256>>>(d, nvec);
      };
      launch();  // warm: bring the block in
      cudaEventRecord(e0);
      for (int r = 0; r < reps; ++r) launch();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      const double gbs = 2.0 * bytes * reps / (ms * 1e-3) / 1e9;
      printf("%-10s %4zu MB  %8.2f us/pass  %8.0f GB/s (read+write)\n", names[mode], mb,
             1e3 * ms / reps, gbs);
    }
  }
  cudaError_t err = cudaGetLastError();
  printf("status: %s\n", cudaGetErrorString(err));
  return 0;
}
