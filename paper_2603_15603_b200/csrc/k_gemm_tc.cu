// Generic bf16 GEMM on tcgen05 for the large-config encoder (C4, ViT-L size):
//   C[M, N] = A[M, K] . W[N, K]^T  (+ fused epilogue)
// A and W are row-major bf16 (K contiguous, i.e. both operands K-major).
//
// One CTA computes a 128 x BN tile.  Warp 0 is the TMA producer (128-byte
// swizzled boxes of 64 K-elements), warp 1 issues tcgen05.mma from one lane
// into a TMEM accumulator, warps 2-5 drain TMEM through the epilogue; a
// STAGES-deep ring of full/empty mbarriers keeps TMA, MMA and the previous
// tile's epilogue overlapped.  Epilogues (decoder.py:247-257 semantics):
//   EPI_BIAS_BF16   out_bf16 = acc + bias                       (Q|K|V)
//   EPI_RELU_BF16   out_bf16 = relu(acc + bias)                 (MLP W1)
//   EPI_RESID_F32   x_f32   += acc + bias                       (Wo, W2)
//   EPI_EMBED_F32   x_f32    = (acc + bias) + pos[row % T]      (patch embed)
#include <cuda.h>
#include <cudaTypedefs.h>
#include <stdio.h>

#include "fsb_common.cuh"
#include "tc_sm100.cuh"

#include "gemm_tc.h"

namespace {
constexpr int BM = 128, BK = 64, STAGES = 4;
constexpr int GEMM_THREADS = 192;
}

template <int BN>
__global__ void __launch_bounds__(GEMM_THREADS, 1)
    k_gemm_tc(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, int M, int N, int K,
              GemmEpi epi) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 1024-byte alignment for the 128B swizzle atoms
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  constexpr uint32_t A_BYTES = BM * BK * 2, B_BYTES = BN * BK * 2, STAGE_BYTES = A_BYTES + B_BYTES;
  __shared__ uint64_t full[STAGES], empty[STAGES], done;
  __shared__ uint32_t tmem_base;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  const int nk = (K + BK - 1) / BK;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      tc::mbar_init(&full[s], 1);
      tc::mbar_init(&empty[s], 1);
    }
    tc::mbar_init(&done, 1);
    tc::mbar_fence_init();
    tc::prefetch_tmap(&tmA);
    tc::prefetch_tmap(&tmB);
  }
  if (warp == 1) tc::tmem_alloc(&tmem_base, BN < 32 ? 32 : BN);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = tmem_base;

  if (warp == 0 && lane == 0) {
    // TMA producer
    for (int kb = 0; kb < nk; ++kb) {
      const int s = kb % STAGES;
      if (kb >= STAGES) tc::mbar_wait(&empty[s], (uint32_t)(((kb / STAGES) - 1) & 1));
      uint8_t* sa = smem + s * STAGE_BYTES;
      tc::mbar_expect_tx(&full[s], STAGE_BYTES);
      tc::tma_load_2d(sa, &tmA, kb * BK, m0, &full[s]);
      tc::tma_load_2d(sa + A_BYTES, &tmB, kb * BK, n0, &full[s]);
    }
  } else if (warp == 1 && lane == 0) {
    // MMA issuer
    const uint32_t idesc = tc::idesc_bf16(BM, BN);
    const uint32_t sbase = tc::smem_u32(smem);
    for (int kb = 0; kb < nk; ++kb) {
      const int s = kb % STAGES;
      tc::mbar_wait(&full[s], (uint32_t)((kb / STAGES) & 1));
      tc::fence_after();
      const uint32_t a = sbase + s * STAGE_BYTES, b = a + A_BYTES;
#pragma unroll
      for (int k = 0; k < BK / 16; ++k)
        tc::mma_bf16(tmem, tc::sw128_kmajor_desc(a + 32 * k), tc::sw128_kmajor_desc(b + 32 * k), idesc,
                     (kb | k) != 0);
      tc::mma_commit(&empty[s]);  // frees the stage once these MMAs have read it
    }
    tc::mma_commit(&done);
  } else if (warp >= 2) {
    // epilogue: warp w reads TMEM lanes 32 * (w % 4) .. +31 (rows of the tile)
    tc::mbar_wait(&done, 0);
    tc::fence_after();
    const int quad = warp % 4;
    const int row = m0 + quad * 32 + lane;
    const uint32_t taddr = tmem + ((uint32_t)(quad * 32) << 16);
#pragma unroll 1
    for (int c = 0; c < BN; c += 16) {
      float v[16];
      tc::tmem_ld16(taddr + c, v);
      const int col = n0 + c;
      if (row >= M || col >= N) continue;
#pragma unroll
      for (int i = 0; i < 16; ++i) v[i] += __ldg(epi.bias + col + i);
      if (epi.kind == EPI_BIAS_BF16 || epi.kind == EPI_RELU_BF16) {
        if (epi.kind == EPI_RELU_BF16)
#pragma unroll
          for (int i = 0; i < 16; ++i) v[i] = fmaxf(v[i], 0.0f);
        uint4 u0, u1;
        u0.x = tc::pack_bf16(v[0], v[1]); u0.y = tc::pack_bf16(v[2], v[3]);
        u0.z = tc::pack_bf16(v[4], v[5]); u0.w = tc::pack_bf16(v[6], v[7]);
        u1.x = tc::pack_bf16(v[8], v[9]); u1.y = tc::pack_bf16(v[10], v[11]);
        u1.z = tc::pack_bf16(v[12], v[13]); u1.w = tc::pack_bf16(v[14], v[15]);
        uint4* dst = reinterpret_cast<uint4*>(epi.out_bf16 + (size_t)row * epi.ldo + col);
        dst[0] = u0;
        dst[1] = u1;
      } else {
        float* x = epi.x_f32 + (size_t)row * epi.ldo + col;
        if (epi.kind == EPI_EMBED_F32) {
          const float* p = epi.pos + (size_t)(row % epi.T) * N + col;
#pragma unroll
          for (int i = 0; i < 16; i += 4) {
            const float4 q = __ldg(reinterpret_cast<const float4*>(p + i));
            *reinterpret_cast<float4*>(x + i) = make_float4(v[i] + q.x, v[i + 1] + q.y, v[i + 2] + q.z, v[i + 3] + q.w);
          }
        } else {
#pragma unroll
          for (int i = 0; i < 16; i += 4) {
            float4 r = *reinterpret_cast<float4*>(x + i);
            r.x += v[i]; r.y += v[i + 1]; r.z += v[i + 2]; r.w += v[i + 3];
            *reinterpret_cast<float4*>(x + i) = r;
          }
        }
      }
    }
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 1) tc::tmem_dealloc(tmem, BN < 32 ? 32 : BN);
}

// ---------------------------------------------------------------------------
// host side: tensor maps (driver entry point through the runtime) and launch

static PFN_cuTensorMapEncodeTiled_v12000 tmap_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// row-major bf16 matrix (rows x cols, leading dimension ld elements) as a
// 2-D tensor map with (box_rows x 64)-element boxes, 128-byte swizzle
bool make_tmap_bf16(CUtensorMap* map, const void* base, uint64_t rows, uint64_t cols, uint64_t ld, uint32_t box_rows) {
  auto enc = tmap_encoder();
  if (!enc) return false;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {ld * 2};
  cuuint32_t box[2] = {64, box_rows};
  cuuint32_t es[2] = {1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int BN>
static constexpr size_t gemm_smem() {
  return (size_t)STAGES * (BM * BK * 2 + BN * BK * 2) + 1024;
}

cudaError_t init_attrs_gemm_tc() {
  cudaError_t e = cudaFuncSetAttribute(k_gemm_tc<256>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)gemm_smem<256>());
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(k_gemm_tc<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)gemm_smem<128>());
  return e;
}

// A (M x K, lda), W (N x K, ldw): bf16 row-major.  N must be a multiple of 16,
// K a multiple of 8 (16-byte TMA strides).
cudaError_t launch_gemm_tc(const __nv_bfloat16* A, int lda, const __nv_bfloat16* W, int ldw, int M, int N, int K,
                           const GemmEpi& epi, cudaStream_t st) {
  if (M == 0 || N == 0) return cudaSuccess;
  if (N % 16 || K % 8 || lda % 8 || ldw % 8) return cudaErrorInvalidValue;
  static bool attrs = false;
  if (!attrs) {
    cudaError_t e = init_attrs_gemm_tc();
    if (e != cudaSuccess) return e;
    attrs = true;
  }
  CUtensorMap ta, tb;
  const int BN = (N % 256 == 0) ? 256 : 128;
  if (!make_tmap_bf16(&ta, A, M, K, lda, BM) || !make_tmap_bf16(&tb, W, N, K, ldw, BN))
    return cudaErrorInvalidValue;
  dim3 grid((N + BN - 1) / BN, (M + BM - 1) / BM);
  if (BN == 256)
    k_gemm_tc<256><<<grid, GEMM_THREADS, gemm_smem<256>(), st>>>(ta, tb, M, N, K, epi);
  else
    k_gemm_tc<128><<<grid, GEMM_THREADS, gemm_smem<128>(), st>>>(ta, tb, M, N, K, epi);
  return cudaGetLastError();
}

// debug / test entry (tests/test_gpu_tcgen05.py): plain C = A W^T + bias
extern "C" int fsb_debug_gemm(const void* A, const void* W, const float* bias, int M, int N, int K, int kind,
                              void* out_bf16, float* x_f32, const float* pos, int T, void* stream) {
  GemmEpi e{bias, static_cast<__nv_bfloat16*>(out_bf16), x_f32, pos, N, T, kind};
  cudaError_t r = launch_gemm_tc(static_cast<const __nv_bfloat16*>(A), K, static_cast<const __nv_bfloat16*>(W), K, M,
                                 N, K, e, (cudaStream_t)stream);
  if (r != cudaSuccess) fprintf(stderr, "fsb_debug_gemm: %s\n", cudaGetErrorString(r));
  return r == cudaSuccess ? 0 : 4;
}
