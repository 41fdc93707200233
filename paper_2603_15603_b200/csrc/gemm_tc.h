// Generic TMA + tcgen05 GEMM (k_gemm_tc.cu): C[M, N] = A[M, K] . W[N, K]^T
// with the fused epilogues of the large-config encoder.
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

enum { EPI_BIAS_BF16 = 0, EPI_RELU_BF16 = 1, EPI_RESID_F32 = 2, EPI_EMBED_F32 = 3 };

struct GemmEpi {
  const float* bias;        // (N)
  __nv_bfloat16* out_bf16;  // (M, ldo)
  float* x_f32;             // (M, ldo) residual stream
  const float* pos;         // (T, N) for EPI_EMBED_F32
  int ldo;
  int T;
  int kind;
};

cudaError_t launch_gemm_tc(const __nv_bfloat16* A, int lda, const __nv_bfloat16* W, int ldw, int M, int N, int K,
                           const GemmEpi& epi, cudaStream_t st);
// row-major bf16 (rows x cols, leading dimension ld) as a 2-D tensor map of
// (box_rows x 64) boxes with 128-byte swizzle
bool make_tmap_bf16(CUtensorMap* map, const void* base, uint64_t rows, uint64_t cols, uint64_t ld, uint32_t box_rows);
