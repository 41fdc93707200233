// Projector MLP on tcgen05 (bf16 mode): projection._projector_mlp
// (projection.py:468-472), relu(x W1 + b1) -> relu(. W2 + b2) -> (. W3 + b3) * mask.
//
// Every operand lives in HBM as a "tile image": 128 x 128 bf16 tiles in the
// UMMA K-major canonical layout, tile (row_tile, k_tile) at
// (row_tile * KT + k_tile) * 32 KB.  The projector-input kernel writes x
// straight into this layout, the weights are packed once on upload, and each
// reduce epilogue writes the next layer's A image, so a CTA stages every
// operand tile with one cp.async.bulk (TMA) copy and the tensor core reads it
// in place.
//
// One CTA computes a 128 x 128 output tile over a fixed group of G k-tiles
// (two-stage bulk-copy ring, MMAs accumulate in TMEM) and writes an fp32
// partial; k_tile_reduce adds the partials of all groups in order and applies
// bias / ReLU / mask.  The K partition depends on K only, so a mesh gives the
// same bits in a batch of 4096 as alone.
#include "fsb_common.cuh"
#include "tc_sm100.cuh"

namespace {
constexpr uint32_t kTileBytes = 128 * 128 * 2;
}

// grid: (n_tiles, splits, m_tiles); block 128
__global__ void __launch_bounds__(128, 1) k_tile_gemm(const uint8_t* __restrict__ Aimg, int KT,
                                                      const uint8_t* __restrict__ Bimg, int G, int M, int N,
                                                      float* __restrict__ partial) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar_load[2], bar_mma[2], bar_done;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid / 32;
  const int nt = blockIdx.x, split = blockIdx.y, mt = blockIdx.z;
  const int kt0 = split * G, nk = min(G, KT - kt0);
  pdl_wait();  // the A image comes from the previous kernel
  if (tid == 0) {
    for (int i = 0; i < 2; ++i) {
      tc::mbar_init(&bar_load[i], 1);
      tc::mbar_init(&bar_mma[i], 1);
    }
    tc::mbar_init(&bar_done, 1);
    tc::mbar_fence_init();
  }
  if (warp == 0) tc::tmem_alloc(&tmem_base, 128);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = tmem_base;
  const uint32_t sbase = tc::smem_u32(smem);
  if (tid == 0) {
    const uint32_t idesc = tc::idesc_bf16(128, 128);
    auto load = [&](int i) {
      const int s = i & 1;
      tc::mbar_expect_tx(&bar_load[s], 2 * kTileBytes);
      tc::bulk_g2s(smem + s * 2 * kTileBytes, Aimg + ((size_t)mt * KT + kt0 + i) * kTileBytes, kTileBytes,
                   &bar_load[s]);
      tc::bulk_g2s(smem + s * 2 * kTileBytes + kTileBytes, Bimg + ((size_t)nt * KT + kt0 + i) * kTileBytes,
                   kTileBytes, &bar_load[s]);
    };
    load(0);
    if (nk > 1) load(1);
    for (int i = 0; i < nk; ++i) {
      const int s = i & 1;
      tc::mbar_wait(&bar_load[s], (uint32_t)((i >> 1) & 1));
      tc::fence_after();
      const uint32_t a = sbase + s * 2 * kTileBytes, b = a + kTileBytes;
      for (int k = 0; k < 128; k += 16)
        tc::mma_bf16(tmem, tc::kmajor_desc(a, 128, k), tc::kmajor_desc(b, 128, k), idesc, (i | k) != 0);
      tc::mma_commit(&bar_mma[s]);
      if (i + 2 < nk) {
        tc::mbar_wait(&bar_mma[s], (uint32_t)((i >> 1) & 1));  // slot free again
        load(i + 2);
      }
    }
    tc::mma_commit(&bar_done);  // tracks every MMA issued above
  }
  __syncwarp();
  tc::mbar_wait(&bar_done, 0);
  tc::fence_after();
  const int row = mt * 128 + tid;
  const uint32_t taddr = tmem + ((uint32_t)(warp * 32) << 16);
  float* dst = partial + ((size_t)split * M + row) * N + nt * 128;
#pragma unroll 1
  for (int c = 0; c < 128; c += 64) {
    float v[64];
    tc::tmem_ld64(taddr + c, v);
    if (row < M)
#pragma unroll
      for (int i = 0; i < 64; i += 4) {
        if (nt * 128 + c + i < N)
          *reinterpret_cast<float4*>(dst + c + i) = make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
      }
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc(tmem, 128);
}

// out = act(sum_s P[s] + b) (* mask); written as fp32 (ldo) and/or as the
// bf16 A-tile image of the next layer (KT_out k-tiles per row tile)
__global__ void k_tile_reduce(const float* __restrict__ P, int S, int M, int N, const float* __restrict__ bias,
                              const float* __restrict__ mask, int relu, float* __restrict__ out, int ldo,
                              uint8_t* __restrict__ out_img, int KT_out, int* nonfinite) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  pdl_wait();
  if (idx >= (int64_t)M * N) return;
  const int m = (int)(idx / N), n = (int)(idx % N);
  float v = P[idx];
  for (int s = 1; s < S; ++s) v += P[(int64_t)s * M * N + idx];
  v += bias[n];
  if (relu) v = fmaxf(v, 0.0f);
  if (mask != nullptr) v *= mask[n];
  flag_nonfinite(nonfinite, v);
  if (out != nullptr) out[(int64_t)m * ldo + n] = v;
  if (out_img != nullptr) {
    const size_t tile = (size_t)(m >> 7) * KT_out + (n >> 7);
    *reinterpret_cast<__nv_bfloat16*>(out_img + tile * kTileBytes + tc::kmajor_off(m & 127, n & 127, 128)) =
        __float2bfloat16_rn(v);
  }
}

cudaError_t init_attrs_mlp_tc() {
  return cudaFuncSetAttribute(k_tile_gemm, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(4 * kTileBytes));
}

// one layer: C (M x N) = A_img (M x 128*KT) * B_img^T, K grouped in G k-tiles
cudaError_t launch_tile_layer(const uint8_t* Aimg, const uint8_t* Bimg, int KT, int G, int M, int N,
                              float* partial, const float* bias, const float* mask, int relu, float* out, int ldo,
                              uint8_t* out_img, int KT_out, int* nonfinite, cudaStream_t st) {
  if (M == 0) return cudaSuccess;
  const int S = (KT + G - 1) / G;
  dim3 grid((N + 127) / 128, S, (M + 127) / 128);
  cudaError_t e = launch_pdl(k_tile_gemm, grid, dim3(128), 4 * kTileBytes, st, Aimg, KT, Bimg, G, M, N, partial);
  if (e != cudaSuccess) return e;
  const int64_t tot = (int64_t)M * N;
  return launch_pdl(k_tile_reduce, dim3((unsigned)((tot + 255) / 256)), dim3(256), 0, st, partial, S, M, N, bias, mask,
                    relu, out, ldo, out_img, KT_out, nonfinite);
}
