// Standalone probe: 2-D TMA load of a float field box into smem via a
// __grid_constant__ tensor-map parameter (same helpers as mo_device.cuh).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <vector>
#include "../../paper_1604_06525_b200/csrc/mo_device.cuh"

extern __shared__ __align__(128) unsigned char dsm[];
__global__ void k(const __grid_constant__ mo_tmaps T, float* out, int c0, int r0, int boxw) {
  unsigned long long* mb = reinterpret_cast<unsigned long long*>(dsm + 8192);
  if (threadIdx.x == 0) { mo_mbar_init(mb, 1); mo_mbar_fence_init(); }
  __syncthreads();
  if (threadIdx.x == 0) {
    mo_mbar_expect_tx(mb, boxw * 8 * 4);
    mo_tma_load_2d(dsm, &T.m[0], c0, r0, mb);
  }
  mo_mbar_wait(mb, 0);
  for (int i = threadIdx.x; i < boxw * 8; i += blockDim.x) out[i] = reinterpret_cast<float*>(dsm)[i];
}
using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
int main() {
  const int W = 64, Hh = 32, boxw = 36;
  std::vector<float> h(W * Hh);
  for (int i = 0; i < W * Hh; ++i) h[i] = float(i);
  float *d, *o;
  cudaMalloc(&d, h.size() * 4);
  cudaMalloc(&o, boxw * 8 * 4);
  cudaMemcpy(d, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
  void* f = nullptr;
  cudaDriverEntryPointQueryResult q;
  printf("entry %d\n", (int)cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q));
  mo_tmaps T;
  memset(&T, 0, sizeof T);
  cuuint64_t dims[2] = {W, Hh}, str[1] = {W * 4};
  cuuint32_t box[2] = {boxw, 8}, es[2] = {1, 1};
  CUresult r = ((EncodeFn)f)((CUtensorMap*)&T.m[0], CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, d, dims, str, box, es,
                             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode %d sizeof %zu\n", (int)r, sizeof(mo_tmaps));
  for (int c0 : {0, 4, -4, 40, 60}) {
    k<<<1, 128, 8192 + 64>>>(T, o, c0, -1, boxw);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<float> ho(boxw * 8);
    cudaMemcpy(ho.data(), o, ho.size() * 4, cudaMemcpyDeviceToHost);
    printf("c0=%d err=%s row0: %g %g %g row1: %g %g %g\n", c0, cudaGetErrorString(e), ho[0], ho[1], ho[2], ho[boxw],
           ho[boxw + 1], ho[boxw + 2]);
    if (e) return 1;
  }
  return 0;
}
