// Hardware self-test of the tcgen05 building blocks (tc_sm100.cuh):
// C (128 x N, f32) = A (128 x K) * B (N x K)^T with A packed by threads into
// the K-major canonical layout, B copied pre-packed with one bulk (TMA) copy,
// the MMAs issued by one thread into TMEM and drained with tcgen05.ld.
// Exercised by tests/test_gpu_tcgen05.py before the fused kernels rely on it.
#include "fsb_common.cuh"
#include "tc_sm100.cuh"

__global__ void __launch_bounds__(128) k_tc_selftest(const __nv_bfloat16* __restrict__ A,
                                                     const uint8_t* __restrict__ Bpacked, int N, int K,
                                                     float* __restrict__ C) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar_load, bar_mma;
  __shared__ uint32_t tmem_base;
  uint8_t* sA = sm;
  uint8_t* sB = sm + 128 * K * 2;
  const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
  if (tid == 0) {
    tc::mbar_init(&bar_load, 1);
    tc::mbar_init(&bar_mma, 1);
    tc::mbar_fence_init();
  }
  if (warp == 0) {
    uint32_t cols = 32;
    while (cols < (uint32_t)N) cols <<= 1;
    tc::tmem_alloc(&tmem_base, cols);
  }
  // each thread packs one row of A
  for (int k = 0; k < K; k += 8) {
    uint4 v;
    const __nv_bfloat16* src = A + (size_t)tid * K + k;
    v = *reinterpret_cast<const uint4*>(src);
    *reinterpret_cast<uint4*>(sA + tc::kmajor_off(tid, k, K)) = v;
  }
  tc::fence_async_smem();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tbase = tmem_base;
  if (tid == 0) {
    const uint32_t bytes = (uint32_t)N * K * 2;
    tc::mbar_expect_tx(&bar_load, bytes);
    tc::bulk_g2s(sB, Bpacked, bytes, &bar_load);
    tc::mbar_wait(&bar_load, 0);
    const uint32_t idesc = tc::idesc_bf16(128, N);
    const uint32_t a0 = tc::smem_u32(sA), b0 = tc::smem_u32(sB);
    for (int k = 0; k < K; k += 16)
      tc::mma_bf16(tbase, tc::kmajor_desc(a0, K, k), tc::kmajor_desc(b0, K, k), idesc, k > 0);
    tc::mma_commit(&bar_mma);
  }
  __syncwarp();
  tc::mbar_wait(&bar_mma, 0);
  tc::fence_after();
  const uint32_t lane_base = tbase + ((uint32_t)(warp * 32) << 16);
  for (int c = 0; c < N; c += 16) {
    float v[16];
    tc::tmem_ld16(lane_base + c, v);
    for (int i = 0; i < 16; ++i) C[(size_t)(warp * 32 + lane) * N + c + i] = v[i];
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 0) {
    uint32_t cols = 32;
    while (cols < (uint32_t)N) cols <<= 1;
    tc::tmem_dealloc(tbase, cols);
  }
}

cudaError_t launch_tc_selftest(const void* A, const void* Bpacked, int N, int K, float* C, cudaStream_t st) {
  if (N < 16 || N > 256 || N % 16 || K < 16 || K % 16 || K > 512) return cudaErrorInvalidValue;
  const size_t smem = (size_t)(128 + N) * K * 2;
  cudaError_t e = cudaFuncSetAttribute(k_tc_selftest, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  k_tc_selftest<<<1, 128, smem, st>>>(static_cast<const __nv_bfloat16*>(A), static_cast<const uint8_t*>(Bpacked),
                                      N, K, C);
  return cudaGetLastError();
}
