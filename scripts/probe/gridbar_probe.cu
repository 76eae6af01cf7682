// Probe: cost of a software grid barrier (atomic arrival counter + generation
// flag) among all co-resident blocks of a cooperative launch, vs. a kernel
// boundary inside a CUDA graph.  Decides whether a persistent PCG kernel pays.
#include <cuda_runtime.h>
#include <cstdio>

__device__ __forceinline__ unsigned ld_acq(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ void grid_barrier(unsigned* count, unsigned* gen, unsigned nblocks) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned g = ld_acq(gen);
    __threadfence();
    if (atomicAdd(count, 1u) == nblocks - 1) {
      *count = 0;
      __threadfence();
      atomicAdd(gen, 1u);
    } else {
      while (ld_acq(gen) == g) {
      }
    }
  }
  __syncthreads();
}
__global__ void k_bar(unsigned* count, unsigned* gen, int iters, float* sink) {
  float acc = threadIdx.x;
  for (int i = 0; i < iters; ++i) {
    acc = acc * 1.0001f + 1.f;
    grid_barrier(count, gen, gridDim.x);
  }
  if (acc == 12345.f) *sink = acc;
}
__global__ void k_empty(float* sink, int v) {
  if (v == 12345 && threadIdx.x == 0) *sink = 1.f;
}
int main() {
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  unsigned *c, *g;
  float* sink;
  cudaMalloc(&c, 8);
  cudaMalloc(&g, 8);
  cudaMalloc(&sink, 4);
  cudaMemset(c, 0, 8);
  cudaMemset(g, 0, 8);
  cudaStream_t st;
  cudaStreamCreate(&st);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int bps : {1, 2, 4}) {
    const int grid = nsm * bps, iters = 1000;
    void* args[] = {&c, &g, (void*)&iters, &sink};
    cudaLaunchCooperativeKernel((void*)k_bar, grid, 256, args, 0, st);
    cudaEventRecord(a, st);
    cudaLaunchCooperativeKernel((void*)k_bar, grid, 256, args, 0, st);
    cudaEventRecord(b, st);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("grid barrier, %d blocks: %.3f us per barrier (%s)\n", grid, ms * 1000 / iters,
           cudaGetErrorString(cudaGetLastError()));
  }
  // kernel boundaries in a graph: 1000 dependent launches of 592 blocks
  cudaGraph_t gr;
  cudaGraphExec_t ge;
  cudaStreamBeginCapture(st, cudaStreamCaptureModeRelaxed);
  for (int i = 0; i < 1000; ++i) k_empty<<<nsm * 4, 256, 0, st>>>(sink, i);
  cudaStreamEndCapture(st, &gr);
  cudaGraphInstantiate(&ge, gr, 0);
  cudaGraphLaunch(ge, st);
  cudaEventRecord(a, st);
  cudaGraphLaunch(ge, st);
  cudaEventRecord(b, st);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  printf("graph kernel boundary (%d blocks): %.3f us per kernel\n", nsm * 4, ms * 1000 / 1000);
  return 0;
}
