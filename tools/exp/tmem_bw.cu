// standalone microbenchmark: tcgen05.ld (32x32b.x32) throughput per SM for
// 4 / 8 / 16 warps, and the cost of one ld + wait round (latency).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/tmem_bw tools/exp/tmem_bw.cu && /tmp/tmem_bw
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdint.h>
#include "../../paper_2603_15603_b200/csrc/tc_sm100.cuh"

__global__ void k_tmem_bw(int iters, int batch, float* out, unsigned long long* cyc) {
  __shared__ uint32_t taddr;
  if (threadIdx.x < 32) tc::tmem_alloc(&taddr, 512);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t base = taddr + ((uint32_t)(((threadIdx.x >> 5) & 3) * 32) << 16) + 32 * ((threadIdx.x >> 7) & 15);
  float acc = 0.0f;
  __syncthreads();
  const long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    if (batch == 1) {
      float v[32];
      tc::tmem_ld32(base, v);
#pragma unroll
      for (int k = 0; k < 32; ++k) acc += v[k];
    } else {  // four loads in flight before one wait
      uint32_t r[4][32];
#pragma unroll
      for (int b = 0; b < 4; ++b)
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
            "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
            "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
            : "=r"(r[b][0]), "=r"(r[b][1]), "=r"(r[b][2]), "=r"(r[b][3]), "=r"(r[b][4]), "=r"(r[b][5]),
              "=r"(r[b][6]), "=r"(r[b][7]), "=r"(r[b][8]), "=r"(r[b][9]), "=r"(r[b][10]), "=r"(r[b][11]),
              "=r"(r[b][12]), "=r"(r[b][13]), "=r"(r[b][14]), "=r"(r[b][15]), "=r"(r[b][16]), "=r"(r[b][17]),
              "=r"(r[b][18]), "=r"(r[b][19]), "=r"(r[b][20]), "=r"(r[b][21]), "=r"(r[b][22]), "=r"(r[b][23]),
              "=r"(r[b][24]), "=r"(r[b][25]), "=r"(r[b][26]), "=r"(r[b][27]), "=r"(r[b][28]), "=r"(r[b][29]),
              "=r"(r[b][30]), "=r"(r[b][31])
            : "r"(base + 128 * b));
      asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
      for (int b = 0; b < 4; ++b)
#pragma unroll
        for (int k = 0; k < 32; ++k) acc += __uint_as_float(r[b][k]);
    }
  }
  const long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = (unsigned long long)(t1 - t0);
  tc::fence_before();
  __syncthreads();
  if (threadIdx.x < 32) tc::tmem_dealloc(taddr, 512);
}

int main() {
  float* out;
  unsigned long long* cyc;
  cudaMalloc(&out, 148 * 1024 * 4);
  cudaMalloc(&cyc, 148 * 8);
  for (int batch = 1; batch <= 4; batch += 3)
    for (int warps = 4; warps <= 16; warps *= 2) {
      const int iters = 2000;
      k_tmem_bw<<<1, 32 * warps>>>(iters, batch, out, cyc);
      k_tmem_bw<<<1, 32 * warps>>>(iters, batch, out, cyc);
      cudaError_t e = cudaDeviceSynchronize();
      unsigned long long c = 0;
      cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
      const double bytes = (double)warps * 32 * 32 * 4 * iters * batch;
      printf("batch %d warps %2d: %llu cycles, %.1f B/cyc/SM, %.1f cyc per ld round (err %s)\n", batch, warps, c,
             bytes / c, (double)c / iters, cudaGetErrorString(e));
    }
  return 0;
}
