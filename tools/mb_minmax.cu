// microbenchmark: VIMNMX throughput, and CE via min+IMAD trick
#include <cstdio>
#include <cstdint>
__global__ void k_minmax(uint32_t* out, int iters) {
  uint32_t v[32];
  for (int i = 0; i < 32; ++i) v[i] = threadIdx.x * 2654435761u + i * 40503u;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int q = 0; q < 5; ++q)
#pragma unroll
      for (int e = 0; e < 32; ++e) if (!(e & (1 << q))) { uint32_t a = v[e], b = v[e | (1<<q)]; v[e] = min(a,b); v[e|(1<<q)] = max(a,b); }
  }
  uint32_t s = 0; for (int i = 0; i < 32; ++i) s ^= v[i] * (i+1);
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_trick(uint32_t* out, int iters, uint32_t one, uint32_t mone) {
  uint32_t v[32];
  for (int i = 0; i < 32; ++i) v[i] = threadIdx.x * 2654435761u + i * 40503u;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int q = 0; q < 5; ++q)
#pragma unroll
      for (int e = 0; e < 32; ++e) if (!(e & (1 << q))) { uint32_t a = v[e], b = v[e | (1<<q)]; uint32_t mn = min(a,b);
         uint32_t s; asm("mad.lo.u32 %0, %1, %3, %2;" : "=r"(s) : "r"(a), "r"(b), "r"(one));
         uint32_t mx; asm("mad.lo.u32 %0, %1, %3, %2;" : "=r"(mx) : "r"(mn), "r"(s), "r"(mone));
         v[e] = mn; v[e|(1<<q)] = mx; }
  }
  uint32_t s = 0; for (int i = 0; i < 32; ++i) s ^= v[i] * (i+1);
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
// mixed: CE number c uses the IMAD form when (c % D) < NUM (fraction NUM/D),
// the VIMNMX pair otherwise: min/max work split over the ALU and FMA pipes
template <int NUM, int D>
__global__ void k_mixed(uint32_t* out, int iters, uint32_t one, uint32_t mone) {
  uint32_t v[32];
  for (int i = 0; i < 32; ++i) v[i] = threadIdx.x * 2654435761u + i * 40503u;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int q = 0; q < 5; ++q) {
      int c = 0;
#pragma unroll
      for (int e = 0; e < 32; ++e) if (!(e & (1 << q))) {
        uint32_t a = v[e], b = v[e | (1<<q)]; uint32_t mn = min(a,b), mx;
        if ((c % D) < NUM) {
          uint32_t s; asm("mad.lo.u32 %0, %1, %3, %2;" : "=r"(s) : "r"(a), "r"(b), "r"(one));
          asm("mad.lo.u32 %0, %1, %3, %2;" : "=r"(mx) : "r"(mn), "r"(s), "r"(mone));
        } else {
          mx = max(a, b);
        }
        v[e] = mn; v[e|(1<<q)] = mx; ++c;
      }
    }
  }
  uint32_t s = 0; for (int i = 0; i < 32; ++i) s ^= v[i] * (i+1);
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int NUM, int D>
void run_mixed(uint32_t* d, int blocks, int threads, int iters, cudaEvent_t a, cudaEvent_t b) {
  k_mixed<NUM, D><<<blocks, threads>>>(d, 10, 1u, 0xFFFFFFFFu);
  cudaEventRecord(a); k_mixed<NUM, D><<<blocks, threads>>>(d, iters, 1u, 0xFFFFFFFFu); cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  double ces = (double)blocks * threads * iters * 5 * 16;
  printf("mixed %d/%d threads=%d: %.3f ms, %.2f CE/clk/SM\n", NUM, D, threads, ms, ces/(ms*1e-3)/148/1.965e9);
}

int main() {
  uint32_t* d; cudaMalloc(&d, 148*8*1024*4);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  int iters = 2000;
  for (int rep = 0; rep < 2; ++rep) {
  for (int threads : {256, 512, 1024}) {
    int blocks = 148 * (2048 / threads) / 2;
    k_minmax<<<blocks, threads>>>(d, 10);
    cudaEventRecord(a); k_minmax<<<blocks, threads>>>(d, iters); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    double ces = (double)blocks * threads * iters * 5 * 16;
    printf("minmax threads=%d blocks=%d: %.3f ms, %.1f G CE/s, %.2f minmax ops/clk/SM @1.965GHz\n", threads, blocks, ms, ces/ms/1e6, ces*2/(ms*1e-3)/148/1.965e9);
    k_trick<<<blocks, threads>>>(d, 10, 1u, 0xFFFFFFFFu);
    cudaEventRecord(a); k_trick<<<blocks, threads>>>(d, iters, 1u, 0xFFFFFFFFu); cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    printf("trick  threads=%d blocks=%d: %.3f ms, %.1f G CE/s, %.2f CE/clk/SM\n", threads, blocks, ms, ces/ms/1e6, ces/(ms*1e-3)/148/1.965e9);
    run_mixed<1, 2>(d, blocks, threads, iters, a, b);
    run_mixed<2, 3>(d, blocks, threads, iters, a, b);
    run_mixed<3, 5>(d, blocks, threads, iters, a, b);
  }}
  return 0;
}
