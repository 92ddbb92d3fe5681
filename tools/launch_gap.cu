// Kernel-to-kernel cost inside one CUDA graph on this GPU: a graph of K
// dependent launches of an (almost) empty kernel with the fast path's grid
// shapes, replayed; CUDA-event time / K.  Also one-CTA kernels, and kernels
// whose CTAs spin for a fixed time (so launch/drain overheads show against a
// known body).  Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/launch_gap.cu -o /tmp/launch_gap
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_empty(int* p) {
  if (p && threadIdx.x == 0 && blockIdx.x == 0) p[0] = 1;
}
__global__ void k_spin(int* p, long long ns) {
  long long t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  long long t = t0;
  while (t - t0 < ns) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  if (p && threadIdx.x == 0 && blockIdx.x == 0) p[0] = 1;
}

static float run(int K, int grid, int block, size_t smem, long long spin_ns) {
  cudaStream_t st;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  int* p;
  cudaMalloc(&p, 4);
  if (smem > 48 * 1024) {
    cudaFuncSetAttribute(k_empty, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(k_spin, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  }
  cudaGraph_t g;
  cudaGraphExec_t ge;
  cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal);
  for (int i = 0; i < K; ++i) {
    if (spin_ns)
      k_spin<<<grid, block, smem, st>>>(p, spin_ns);
    else
      k_empty<<<grid, block, smem, st>>>(p);
  }
  cudaStreamEndCapture(st, &g);
  cudaGraphInstantiate(&ge, g, 0);
  for (int w = 0; w < 3; ++w) cudaGraphLaunch(ge, st);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int R = 20;
  cudaEventRecord(a, st);
  for (int r = 0; r < R; ++r) cudaGraphLaunch(ge, st);
  cudaEventRecord(b, st);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  cudaGraphExecDestroy(ge);
  cudaGraphDestroy(g);
  cudaFree(p);
  cudaStreamDestroy(st);
  return ms * 1e3f / (R * K);  // us per kernel
}

int main() {
  const int K = 50;
  struct C { const char* name; int grid, block; size_t smem; long long spin; } cs[] = {
      {"1 CTA x 32, empty", 1, 32, 0, 0},
      {"592 x 256, empty", 592, 256, 0, 0},
      {"592 x 256, 52 KB smem, empty", 592, 256, 52 * 1024, 0},
      {"1160 x 128, empty", 1160, 128, 0, 0},
      {"444 x 256, 60 KB smem, empty", 444, 256, 60 * 1024, 0},
      {"896 x 256, empty", 896, 256, 0, 0},
      {"592 x 256, spin 10 us", 592, 256, 0, 10000},
      {"444 x 256, 60 KB, spin 10 us", 444, 256, 60 * 1024, 10000},
  };
  for (auto& c : cs)
    std::printf("%-34s %7.2f us per kernel%s\n", c.name, run(K, c.grid, c.block, c.smem, c.spin),
                c.spin ? " (10 us body)" : "");
  return 0;
}
