// Persistent alternative to 15 dependent launches: one cooperative kernel that
// runs 15 in-place 4 MiB passes separated by a grid-wide barrier (a
// hand-rolled sense-reversing barrier on a global counter, and
// cooperative_groups::this_grid().sync()).  Development probe.
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <vector>
#include <algorithm>
namespace cg = cooperative_groups;

__device__ __forceinline__ void pass_body(uint4* d, int blk, int nblk) {
  for (int b = blk; b < 256; b += nblk) {
    const int i = b * 256 * 4 + threadIdx.x;
    uint4 v[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) v[j] = d[i + j * 256];
#pragma unroll
    for (int j = 0; j < 4; ++j) v[j].x ^= 1;
#pragma unroll
    for (int j = 0; j < 4; ++j) d[i + j * 256] = v[j];
  }
}

__global__ void __launch_bounds__(256) persistent_cg(uint4* d, int passes) {
  cg::grid_group g = cg::this_grid();
  for (int p = 0; p < passes; ++p) {
    pass_body(d, blockIdx.x, gridDim.x);
    g.sync();
  }
}

__device__ unsigned int g_bar_count = 0;
__device__ volatile unsigned int g_bar_gen = 0;

__device__ __forceinline__ void grid_barrier(unsigned int nblk) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned int gen = g_bar_gen;
    __threadfence();
    if (atomicAdd(&g_bar_count, 1) == nblk - 1) {
      g_bar_count = 0;
      __threadfence();
      g_bar_gen = gen + 1;
    } else {
      while (g_bar_gen == gen) { }
    }
    __threadfence();
  }
  __syncthreads();
}

__global__ void __launch_bounds__(256) persistent_atomic(uint4* d, int passes) {
  for (int p = 0; p < passes; ++p) {
    pass_body(d, blockIdx.x, gridDim.x);
    grid_barrier(gridDim.x);
  }
}

int main() {
  uint4* d;
  cudaMalloc(&d, (1 << 20) * 4);
  cudaStream_t s;
  cudaStreamCreate(&s);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int grid : {148, 256}) {
    for (int kind = 0; kind < 2; ++kind) {
      std::vector<float> t;
      for (int r = 0; r < 30; ++r) {
        int passes = 15;
        void* args[] = {&d, &passes};
        cudaEventRecord(a, s);
        if (kind == 0)
          cudaLaunchCooperativeKernel((void*)persistent_cg, grid, 256, args, 0, s);
        else
          cudaLaunchCooperativeKernel((void*)persistent_atomic, grid, 256, args, 0, s);
        cudaEventRecord(b, s);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (r >= 5) t.push_back(ms * 1e3f);
      }
      std::sort(t.begin(), t.end());
      printf("grid %d %s: 15 passes %.1f us (%.2f us/pass)  %s\n", grid,
             kind == 0 ? "cg::grid.sync" : "atomic barrier", t[t.size() / 2],
             t[t.size() / 2] / 15, cudaGetErrorString(cudaGetLastError()));
    }
  }
}
