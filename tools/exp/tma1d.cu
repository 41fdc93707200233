// standalone check: 1-D TMA tensor store constraints (global start alignment, smem source alignment, box 188)
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdint.h>
#include "../../paper_2603_15603_b200/csrc/tc_sm100.cuh"

__global__ void k_test(const __grid_constant__ CUtensorMap tm, int off, int box, int soff) {
  extern __shared__ __align__(1024) uint8_t sm[];
  float* s = reinterpret_cast<float*>(sm + soff);
  for (int i = threadIdx.x; i < box; i += blockDim.x) s[i] = 1000.0f + i;
  tc::fence_async_smem();
  __syncthreads();
  if (threadIdx.x == 0) {
    tc::tma_store_1d(&tm, off, s);
    tc::bulk_commit();
    tc::bulk_wait0();
  }
}

int main() {
  const int n = 4096;
  float* d;
  cudaMalloc(&d, n * 4);
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  const int cases[4][3] = {{8, 188, 128}, {12, 192, 256}, {4, 188, 384}, {0, 192, 128}};  // off, box, smem offset
  for (int v = 0; v < 4; ++v) {
    cudaMemset(d, 0, n * 4);
    CUtensorMap tm;
    cuuint64_t dims[1] = {(cuuint64_t)n};
    cuuint64_t strides[1] = {(cuuint64_t)n * 4};
    cuuint32_t bx[1] = {(cuuint32_t)cases[v][1]};
    cuuint32_t es[1] = {1};
    CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 1, d, dims, strides, bx, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    k_test<<<1, 128, 4096>>>(tm, cases[v][0], cases[v][1], cases[v][2]);
    cudaError_t e = cudaDeviceSynchronize();
    float h[4];
    cudaMemcpy(h, d + cases[v][0] + cases[v][1] - 2, 4 * 4, cudaMemcpyDeviceToHost);
    printf("case %d enc %d err %s last two %.0f %.0f after %.0f\n", v, (int)r, cudaGetErrorString(e), h[0], h[1], h[2]);
    if (e != cudaSuccess) return 1;
  }
  return 0;
}
