// Floor of a chain of dependent 4 MiB in-place passes (L2-resident), with and
// without programmatic dependent launch: what a 15-pass 2^20 sort could reach
// if each pass were a pure copy.  Development probe.
#include <cuda_runtime.h>
#include <cstdio>
#include <vector>
#include <algorithm>

__global__ void __launch_bounds__(256) pass_kernel(uint4* d, int pdl) {
  if (pdl) asm volatile("griddepcontrol.wait;" ::: "memory");
  const int i = blockIdx.x * 256 * 4 + threadIdx.x;
  uint4 v[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) v[j] = d[i + j * 256];
#pragma unroll
  for (int j = 0; j < 4; ++j) { v[j].x ^= 1; }
  if (pdl) asm volatile("griddepcontrol.launch_dependents;");
#pragma unroll
  for (int j = 0; j < 4; ++j) d[i + j * 256] = v[j];
}

int main() {
  const int n = 1 << 20;  // keys
  uint4* d;
  cudaMalloc(&d, n * 4);
  cudaStream_t s;
  cudaStreamCreate(&s);
  for (int ctas : {256, 148 * 2}) {
    for (int pdl = 0; pdl < 2; ++pdl) {
      for (int graph = 0; graph < 2; ++graph) {
        auto chain = [&](cudaStream_t st) {
          for (int p = 0; p < 15; ++p) {
            cudaLaunchConfig_t cfg{};
            cfg.gridDim = dim3(256);  // 256 CTAs x 256 threads x 16 keys = 2^20
            cfg.blockDim = dim3(256);
            cfg.stream = st;
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
            at[0].val.programmaticStreamSerializationAllowed = pdl;
            cfg.attrs = at;
            cfg.numAttrs = 1;
            cudaLaunchKernelEx(&cfg, pass_kernel, d, pdl);
          }
        };
        cudaGraphExec_t ex = nullptr;
        if (graph) {
          cudaStream_t cs;
          cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking);
          cudaGraph_t g;
          cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal);
          chain(cs);
          cudaStreamEndCapture(cs, &g);
          cudaGraphInstantiate(&ex, g, 0);
        }
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        std::vector<float> t;
        for (int r = 0; r < 30; ++r) {
          cudaEventRecord(a, s);
          if (graph) cudaGraphLaunch(ex, s); else chain(s);
          cudaEventRecord(b, s);
          cudaEventSynchronize(b);
          float ms;
          cudaEventElapsedTime(&ms, a, b);
          if (r >= 5) t.push_back(ms * 1e3f);
        }
        std::sort(t.begin(), t.end());
        printf("ctas %d pdl %d graph %d: 15 passes %.1f us (%.2f us/pass)\n", ctas, pdl, graph,
               t[t.size() / 2], t[t.size() / 2] / 15);
      }
    }
    break;
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
