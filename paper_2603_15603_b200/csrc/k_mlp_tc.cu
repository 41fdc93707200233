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
#include <cstdlib>
#include <utility>

#include "fsb_common.cuh"
#include "fsb_weights.h"
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

// ---------------------------------------------------------------------------
// Large batches (C3: 4096 meshes, 1152 output-tile x K-group items for W1):
// the same items and the same MMA sequence per item as k_tile_gemm (so the
// partials, and every mesh's bits, do not depend on the batch), computed by
// a persistent warp-specialised CTA per SM: warp 4 streams the A / B tiles
// of consecutive items through a 3-deep bulk-copy ring, warp 5 issues the
// MMAs into one of two TMEM accumulators, warps 0-3 drain the other one --
// loads, MMAs and the partial-sum stores of neighbouring items overlap
// instead of running back to back in one-item CTAs.
// ---------------------------------------------------------------------------
constexpr int kPStages = 3;

__global__ void __launch_bounds__(192, 1) k_tile_gemm_p(const uint8_t* __restrict__ Aimg, int KT,
                                                        const uint8_t* __restrict__ Bimg, int G, int M, int N,
                                                        int S, int NT, int MT, float* __restrict__ partial) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar_load[kPStages], bar_free[kPStages], bar_full[2], bar_tfree[2];
  __shared__ uint32_t tmem_base;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int items = MT * S * NT;
  if (threadIdx.x == 0) {
    for (int i = 0; i < kPStages; ++i) {
      tc::mbar_init(&bar_load[i], 1);
      tc::mbar_init(&bar_free[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      tc::mbar_init(&bar_full[i], 1);
      tc::mbar_init(&bar_tfree[i], 4);
    }
    tc::mbar_fence_init();
  }
  if (warp == 0) tc::tmem_alloc(&tmem_base, 256);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = tmem_base;
  const uint32_t sbase = tc::smem_u32(smem);
  pdl_wait();  // the A image comes from the previous kernel
  // item i: n-tile fastest, then K group, then m-tile
  auto decode = [&](int i, int& mt, int& split, int& nt) {
    nt = i % NT;
    split = (i / NT) % S;
    mt = i / (NT * S);
  };
  if (warp == 4) {
    if (lane == 0) {  // producer
      int q = 0;
      for (int i = blockIdx.x; i < items; i += gridDim.x) {
        int mt, split, nt;
        decode(i, mt, split, nt);
        const int kt0 = split * G, nk = min(G, KT - kt0);
        for (int k = 0; k < nk; ++k, ++q) {
          const int s = q % kPStages, u = q / kPStages;
          if (u > 0) tc::mbar_wait(&bar_free[s], (uint32_t)((u - 1) & 1));
          tc::mbar_expect_tx(&bar_load[s], 2 * kTileBytes);
          tc::bulk_g2s(smem + s * 2 * kTileBytes, Aimg + ((size_t)mt * KT + kt0 + k) * kTileBytes, kTileBytes,
                       &bar_load[s]);
          tc::bulk_g2s(smem + s * 2 * kTileBytes + kTileBytes, Bimg + ((size_t)nt * KT + kt0 + k) * kTileBytes,
                       kTileBytes, &bar_load[s]);
        }
      }
    }
  } else if (warp == 5) {
    if (lane == 0) {  // MMA issue
      const uint32_t idesc = tc::idesc_bf16(128, 128);
      int q = 0, t = 0;
      for (int i = blockIdx.x; i < items; i += gridDim.x, ++t) {
        int mt, split, nt;
        decode(i, mt, split, nt);
        const int kt0 = split * G, nk = min(G, KT - kt0);
        const int b = t & 1, ut = t >> 1;
        if (ut > 0) tc::mbar_wait(&bar_tfree[b], (uint32_t)((ut - 1) & 1));
        tc::fence_after();
        const uint32_t d = tmem + b * 128;
        for (int k = 0; k < nk; ++k, ++q) {
          const int s = q % kPStages, u = q / kPStages;
          tc::mbar_wait(&bar_load[s], (uint32_t)(u & 1));
          tc::fence_after();
          const uint32_t a = sbase + s * 2 * kTileBytes, bb = a + kTileBytes;
          for (int kk = 0; kk < 128; kk += 16)
            tc::mma_bf16(d, tc::kmajor_desc(a, 128, kk), tc::kmajor_desc(bb, 128, kk), idesc, (k | kk) != 0);
          tc::mma_commit(&bar_free[s]);  // slot s free once these MMAs have read it
        }
        tc::mma_commit(&bar_full[b]);
      }
    }
  } else {  // warps 0-3: epilogue, TMEM lane quadrant = warp
    int t = 0;
    for (int i = blockIdx.x; i < items; i += gridDim.x, ++t) {
      int mt, split, nt;
      decode(i, mt, split, nt);
      const int b = t & 1, ut = t >> 1;
      tc::mbar_wait(&bar_full[b], (uint32_t)(ut & 1));
      tc::fence_after();
      const int row = mt * 128 + warp * 32 + lane;
      const uint32_t taddr = tmem + b * 128 + ((uint32_t)(warp * 32) << 16);
      float* dst = partial + ((size_t)split * M + row) * N + nt * 128;
#pragma unroll 1
      for (int c = 0; c < 128; c += 64) {
        float v[64];
        tc::tmem_ld64(taddr + c, v);
        if (row < M)
#pragma unroll
          for (int j = 0; j < 64; j += 4) {
            if (nt * 128 + c + j < N)
              *reinterpret_cast<float4*>(dst + c + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
          }
      }
      tc::fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&bar_tfree[b]);
    }
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc(tmem, 256);
}

// ---------------------------------------------------------------------------
// Large batches, split-K reduced on chip: one persistent CTA per output tile
// item (m-tile, n-tile) walks the layer's K groups (and, in split-bf16 mode,
// the three passes) in the order k_tile_reduce8 adds the partial slices;
// each group's 128 x 128 product lands in one of two TMEM accumulators and
// the eight epilogue warps (lane quadrant w & 3, column half w >> 2) add it
// into a running sum in registers, then apply bias / ReLU / mask and write
// the outputs exactly as k_tile_reduce8 would.  Same bits as the partial-
// buffer path (the same fp32 adds in the same order); the S x M x N fp32
// partials (75 MB for layer 1 at 4096 meshes) never touch HBM.
// Warps 0-7 epilogue, warp 8 producer (bulk copies into a 3-deep ring),
// warp 9 MMA issue.
// ---------------------------------------------------------------------------
struct TileOperands {
  const uint8_t* a[3];
  const uint8_t* b[3];
};

// RELU / MASK / LO: the layer's epilogue variant (one instantiation each keeps
// the kernel small: the generic form measured i-cache bound on short layers)
template <bool RELU, bool MASK, bool LO>
__global__ void __launch_bounds__(320, 1) k_tile_gemm_f(TileOperands ops, int passes, int KT, int G, int M, int N,
                                                        int NT, int MT, const float* __restrict__ bias,
                                                        const float* __restrict__ mask, float* __restrict__ out,
                                                        int ldo, uint8_t* __restrict__ out_img, int KT_out,
                                                        int* nonfinite, uint8_t* __restrict__ out_img_lo) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar_load[kPStages], bar_free[kPStages], bar_full[2], bar_tfree[2];
  __shared__ uint32_t tmem_base;
  __shared__ float s_bias[128], s_mask[128];
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int items = MT * NT;
  const int S = (KT + G - 1) / G;
  const int units = passes * S;  // (pass, group) products per item, in the reduce's slice order
  if (threadIdx.x == 0) {
    for (int i = 0; i < kPStages; ++i) {
      tc::mbar_init(&bar_load[i], 1);
      tc::mbar_init(&bar_free[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      tc::mbar_init(&bar_full[i], 1);
      tc::mbar_init(&bar_tfree[i], 8);
    }
    tc::mbar_fence_init();
  }
  if (warp == 0) tc::tmem_alloc(&tmem_base, 256);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = tmem_base;
  const uint32_t sbase = tc::smem_u32(smem);
  pdl_wait();  // the A image comes from the previous kernel
  if (warp == 8) {
    if (lane == 0) {  // producer
      int q = 0;
      for (int i = blockIdx.x; i < items; i += gridDim.x) {
        const int nt = i % NT, mt = i / NT;
        for (int u = 0; u < units; ++u) {
          const int ps = u / S, kt0 = (u % S) * G, nk = min(G, KT - kt0);
          for (int k = 0; k < nk; ++k, ++q) {
            const int s = q % kPStages, r = q / kPStages;
            if (r > 0) tc::mbar_wait(&bar_free[s], (uint32_t)((r - 1) & 1));
            tc::mbar_expect_tx(&bar_load[s], 2 * kTileBytes);
            tc::bulk_g2s(smem + s * 2 * kTileBytes, ops.a[ps] + ((size_t)mt * KT + kt0 + k) * kTileBytes, kTileBytes,
                         &bar_load[s]);
            tc::bulk_g2s(smem + s * 2 * kTileBytes + kTileBytes, ops.b[ps] + ((size_t)nt * KT + kt0 + k) * kTileBytes,
                         kTileBytes, &bar_load[s]);
          }
        }
      }
    }
  } else if (warp == 9) {
    if (lane == 0) {  // MMA issue
      const uint32_t idesc = tc::idesc_bf16(128, 128);
      int q = 0, t = 0;
      for (int i = blockIdx.x; i < items; i += gridDim.x) {
        for (int u = 0; u < units; ++u, ++t) {
          const int kt0 = (u % S) * G, nk = min(G, KT - kt0);
          const int b = t & 1, ut = t >> 1;
          if (ut > 0) tc::mbar_wait(&bar_tfree[b], (uint32_t)((ut - 1) & 1));
          tc::fence_after();
          const uint32_t d = tmem + b * 128;
          for (int k = 0; k < nk; ++k, ++q) {
            const int s = q % kPStages, r = q / kPStages;
            tc::mbar_wait(&bar_load[s], (uint32_t)(r & 1));
            tc::fence_after();
            const uint32_t a = sbase + s * 2 * kTileBytes, bb = a + kTileBytes;
            for (int kk = 0; kk < 128; kk += 16)
              tc::mma_bf16(d, tc::kmajor_desc(a, 128, kk), tc::kmajor_desc(bb, 128, kk), idesc, (k | kk) != 0);
            tc::mma_commit(&bar_free[s]);
          }
          tc::mma_commit(&bar_full[b]);
        }
      }
    }
  } else {  // warps 0-7: running sums of one row x 64 columns
    const int quad = warp & 3, half = warp >> 2;
    int t = 0;
    for (int i = blockIdx.x; i < items; i += gridDim.x) {
      const int nt = i % NT, mt = i / NT;
      const int m = mt * 128 + quad * 32 + lane;
      // the item's 128 bias / mask columns into shared memory while its
      // first products are computed (per-element global loads in the
      // epilogue serialised into L2 round trips)
      asm volatile("bar.sync 1, 256;" ::: "memory");  // the previous item's epilogue is done with them
      if (threadIdx.x < 128) {
        const int n = nt * 128 + threadIdx.x;
        s_bias[threadIdx.x] = n < N ? bias[n] : 0.0f;
        s_mask[threadIdx.x] = n < N && mask != nullptr ? mask[n] : 1.0f;
      }
      asm volatile("bar.sync 1, 256;" ::: "memory");
      float v[64];
      for (int u = 0; u < units; ++u, ++t) {
        const int b = t & 1, ut = t >> 1;
        tc::mbar_wait(&bar_full[b], (uint32_t)(ut & 1));
        tc::fence_after();
#pragma unroll
        for (int hq = 0; hq < 2; ++hq) {  // two 32-column loads: fewer live registers
          float p[32];
          tc::tmem_ld32(tmem + b * 128 + ((uint32_t)(quad * 32) << 16) + 64 * half + 32 * hq, p);
          if (u == 0) {
#pragma unroll
            for (int j = 0; j < 32; ++j) v[32 * hq + j] = p[j];
          } else {
#pragma unroll
            for (int j = 0; j < 32; ++j) v[32 * hq + j] += p[j];
          }
        }
        tc::fence_before();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(&bar_tfree[b]);
      }
      if (m >= M) continue;
      // the k_tile_reduce8 epilogue, eight columns at a time
      bool bad = false;
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const int n0 = nt * 128 + 64 * half + 8 * c;
        if (n0 >= N) break;
        const bool hi = n0 + 4 < N;  // (N % 4 == 0: a chunk holds 4 or 8 columns)
        float w[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int cl = 64 * half + 8 * c + j;
          float x = v[8 * c + j] + s_bias[cl];
          if (RELU) x = fmaxf(x, 0.0f);
          if (MASK) x *= s_mask[cl];
          w[j] = (j < 4 || hi) ? x : 0.0f;
          bad = bad || !isfinite(w[j]);
        }
        if (out != nullptr) {
          *reinterpret_cast<float4*>(out + (int64_t)m * ldo + n0) = make_float4(w[0], w[1], w[2], w[3]);
          if (hi) *reinterpret_cast<float4*>(out + (int64_t)m * ldo + n0 + 4) = make_float4(w[4], w[5], w[6], w[7]);
        }
        if (out_img != nullptr) {
          const size_t tile = (size_t)(m >> 7) * KT_out + (n0 >> 7);
          const size_t off = tile * kTileBytes + tc::kmajor_off(m & 127, n0 & 127, 128);
          uint32_t h[4];
#pragma unroll
          for (int j = 0; j < 4; ++j) h[j] = tc::pack_bf16(w[2 * j], w[2 * j + 1]);
          *reinterpret_cast<uint4*>(out_img + off) = make_uint4(h[0], h[1], h[2], h[3]);
          if (LO) {
            uint32_t lo[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const float2 hf = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&h[j]));
              lo[j] = tc::pack_bf16(w[2 * j] - hf.x, w[2 * j + 1] - hf.y);
            }
            *reinterpret_cast<uint4*>(out_img_lo + off) = make_uint4(lo[0], lo[1], lo[2], lo[3]);
          }
        }
      }
      if (bad && nonfinite != nullptr) atomicOr(nonfinite, 1);
    }
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc(tmem, 256);
}

// ---------------------------------------------------------------------------
// Small batches (M = meshes <= 64: the frame path's 32): the same K groups,
// transposed -- D^T (128 outputs x Np meshes) = W^T tile (the A operand, M =
// 128) . X^T, the meshes as the N = Np operand (Np = M rounded up to 16).
// Only the first Np rows of each x k-tile are copied (the K-major row groups
// are contiguous: Np x 256 bytes instead of 32 KB) and each MMA is 128 x Np
// instead of 128 x 128 on a mostly-padding A tile.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(128, 1) k_tile_gemm_t(const uint8_t* __restrict__ Aimg, int KT,
                                                        const uint8_t* __restrict__ Bimg, int G, int M, int N, int Np,
                                                        float* __restrict__ partial) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar_load[2], bar_mma[2], bar_done;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid / 32;
  const int nt = blockIdx.x, split = blockIdx.y;
  const int kt0 = split * G, nk = min(G, KT - kt0);
  const uint32_t xbytes = (uint32_t)Np * 256u;  // Np rows of a K-major 128 x 128 tile
  pdl_wait();  // the A image comes from the previous kernel
  if (tid == 0) {
    for (int i = 0; i < 2; ++i) {
      tc::mbar_init(&bar_load[i], 1);
      tc::mbar_init(&bar_mma[i], 1);
    }
    tc::mbar_init(&bar_done, 1);
    tc::mbar_fence_init();
  }
  if (warp == 0) tc::tmem_alloc(&tmem_base, 64);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = tmem_base;
  const uint32_t sbase = tc::smem_u32(smem);
  constexpr uint32_t kStage = kTileBytes + 64 * 256;  // W^T tile + up to 64 x rows
  if (tid == 0) {
    const uint32_t idesc = tc::idesc_bf16(128, Np);
    auto load = [&](int i) {
      const int s = i & 1;
      tc::mbar_expect_tx(&bar_load[s], kTileBytes + xbytes);
      tc::bulk_g2s(smem + s * kStage, Bimg + ((size_t)nt * KT + kt0 + i) * kTileBytes, kTileBytes, &bar_load[s]);
      tc::bulk_g2s(smem + s * kStage + kTileBytes, Aimg + ((size_t)kt0 + i) * kTileBytes, xbytes, &bar_load[s]);
    };
    load(0);
    if (nk > 1) load(1);
    for (int i = 0; i < nk; ++i) {
      const int s = i & 1;
      tc::mbar_wait(&bar_load[s], (uint32_t)((i >> 1) & 1));
      tc::fence_after();
      const uint32_t w = sbase + s * kStage, x = w + kTileBytes;
      for (int k = 0; k < 128; k += 16)
        tc::mma_bf16(tmem, tc::kmajor_desc(w, 128, k), tc::kmajor_desc(x, 128, k), idesc, (i | k) != 0);
      tc::mma_commit(&bar_mma[s]);
      if (i + 2 < nk) {
        tc::mbar_wait(&bar_mma[s], (uint32_t)((i >> 1) & 1));
        load(i + 2);
      }
    }
    tc::mma_commit(&bar_done);
  }
  __syncwarp();
  tc::mbar_wait(&bar_done, 0);
  tc::fence_after();
  // lane = output unit n of this tile, columns = meshes
  const int n = nt * 128 + tid;
  const uint32_t taddr = tmem + ((uint32_t)(warp * 32) << 16);
  for (int c = 0; c < Np; c += 16) {
    float v[16];
    tc::tmem_ld16(taddr + c, v);
    if (n < N)
#pragma unroll
      for (int j = 0; j < 16; ++j)
        if (c + j < M) partial[((size_t)split * M + c + j) * N + n] = v[j];
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc(tmem, 64);
}

// k_tile_reduce with one 16-byte K-major chunk (8 consecutive n of a row)
// per thread: the same partial-sum order, bias / ReLU / mask, fp32 and bf16
// image stores as whole vectors (N % 4 == 0)
__global__ void k_tile_reduce8(const float* __restrict__ P, int S, int M, int N, const float* __restrict__ bias,
                               const float* __restrict__ mask, int relu, float* __restrict__ out, int ldo,
                               uint8_t* __restrict__ out_img, int KT_out, int* nonfinite,
                               uint8_t* __restrict__ out_img_lo) {
  const int N8 = (N + 7) / 8;
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  pdl_wait();
  if (idx >= (int64_t)M * N8) return;
  const int m = (int)(idx / N8), n0 = (int)(idx % N8) * 8;
  const bool hi = n0 + 4 < N;
  float v[8];
  auto ld = [&](int s) {
    const float* p = P + ((int64_t)s * M + m) * N + n0;
    const float4 a = *reinterpret_cast<const float4*>(p);
    const float4 b = hi ? *reinterpret_cast<const float4*>(p + 4) : make_float4(0.f, 0.f, 0.f, 0.f);
    return std::make_pair(a, b);
  };
  {
    const auto ab = ld(0);
    v[0] = ab.first.x; v[1] = ab.first.y; v[2] = ab.first.z; v[3] = ab.first.w;
    v[4] = ab.second.x; v[5] = ab.second.y; v[6] = ab.second.z; v[7] = ab.second.w;
  }
  for (int s = 1; s < S; ++s) {
    const auto ab = ld(s);
    v[0] += ab.first.x; v[1] += ab.first.y; v[2] += ab.first.z; v[3] += ab.first.w;
    v[4] += ab.second.x; v[5] += ab.second.y; v[6] += ab.second.z; v[7] += ab.second.w;
  }
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const int n = n0 + j;
    if (n < N) {
      v[j] += bias[n];
      if (relu) v[j] = fmaxf(v[j], 0.0f);
      if (mask != nullptr) v[j] *= mask[n];
      flag_nonfinite(nonfinite, v[j]);
    } else {
      v[j] = 0.0f;
    }
  }
  if (out != nullptr) {
    *reinterpret_cast<float4*>(out + (int64_t)m * ldo + n0) = make_float4(v[0], v[1], v[2], v[3]);
    if (hi) *reinterpret_cast<float4*>(out + (int64_t)m * ldo + n0 + 4) = make_float4(v[4], v[5], v[6], v[7]);
  }
  if (out_img != nullptr) {
    const size_t tile = (size_t)(m >> 7) * KT_out + (n0 >> 7);
    const size_t off = tile * kTileBytes + tc::kmajor_off(m & 127, n0 & 127, 128);
    uint32_t h[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) h[j] = tc::pack_bf16(v[2 * j], v[2 * j + 1]);
    *reinterpret_cast<uint4*>(out_img + off) = make_uint4(h[0], h[1], h[2], h[3]);
    if (out_img_lo != nullptr) {  // split-bf16: the remainders v - bf16(v)
      uint32_t l[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float2 hf = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&h[j]));
        l[j] = tc::pack_bf16(v[2 * j] - hf.x, v[2 * j + 1] - hf.y);
      }
      *reinterpret_cast<uint4*>(out_img_lo + off) = make_uint4(l[0], l[1], l[2], l[3]);
    }
  }
}

cudaError_t init_attrs_mlp_tc() {
  cudaError_t e = cudaFuncSetAttribute(k_tile_gemm, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(4 * kTileBytes));
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(k_tile_gemm_t, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)(2 * (kTileBytes + 64 * 256)));
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(k_tile_gemm_p, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)(2 * kPStages * kTileBytes));
  if (e != cudaSuccess) return e;
  for (auto f : {k_tile_gemm_f<true, false, false>, k_tile_gemm_f<false, true, false>, k_tile_gemm_f<true, false, true>,
                 k_tile_gemm_f<false, true, true>}) {
    e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(2 * kPStages * kTileBytes));
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

#ifndef FSB_TILE_PERSIST_M
#define FSB_TILE_PERSIST_M 1024  // batches from this size on: the persistent kernel
#endif

// one GEMM pass of a layer into `partial` (S split-K slices)
static cudaError_t tile_gemm_pass(const uint8_t* Aimg, const uint8_t* Bimg, int KT, int G, int M, int N, int S,
                                  float* partial, cudaStream_t st) {
  const int NT = (N + 127) / 128, MT = (M + 127) / 128;
  static const bool no_t = getenv("FSB_TILE_NO_T") != nullptr;  // A/B: the 128-row tiles at small M too
  if (M <= 64 && !no_t) {
    const int Np = (M + 15) / 16 * 16;
    return launch_pdl(k_tile_gemm_t, dim3(NT, S), dim3(128), 2 * (kTileBytes + 64 * 256), st, Aimg, KT, Bimg, G, M,
                      N, Np, partial);
  }
  if (M >= FSB_TILE_PERSIST_M) {
    const int items = MT * S * NT;
    return launch_pdl(k_tile_gemm_p, dim3(items < 148 ? items : 148), dim3(192), 2 * kPStages * kTileBytes, st, Aimg,
                      KT, Bimg, G, M, N, S, NT, MT, partial);
  }
  return launch_pdl(k_tile_gemm, dim3(NT, S, MT), dim3(128), 4 * kTileBytes, st, Aimg, KT, Bimg, G, M, N, partial);
}

// one layer: C (M x N) = A_img (M x 128*KT) * B_img^T, K grouped in G k-tiles.
// Split-bf16 (fp32 mode, Aimg_lo / Bimg_lo given): three passes hi.hi,
// hi.lo, lo.hi fill three slices of the partials (3 S in all), which the
// reduce adds in that order; it then writes the next layer's hi AND lo images.
cudaError_t launch_tile_layer(const uint8_t* Aimg, const uint8_t* Bimg, int KT, int G, int M, int N,
                              float* partial, const float* bias, const float* mask, int relu, float* out, int ldo,
                              uint8_t* out_img, int KT_out, int* nonfinite, cudaStream_t st, const uint8_t* Aimg_lo,
                              const uint8_t* Bimg_lo, uint8_t* out_img_lo) {
  if (M == 0) return cudaSuccess;
  const int S = (KT + G - 1) / G;
  const bool split = Aimg_lo != nullptr && Bimg_lo != nullptr;
  // large batches: the K groups reduced on chip (same bits as the partials +
  // k_tile_reduce8 below); FSB_TILE_PARTIALS=1 keeps the partial buffers
  static const bool partials = getenv("FSB_TILE_PARTIALS") != nullptr && atoi(getenv("FSB_TILE_PARTIALS")) != 0;
  if (M >= FSB_TILE_PERSIST_M && N % 4 == 0 && (out == nullptr || ldo % 4 == 0) && !partials &&
      ((relu != 0) != (mask != nullptr))) {
    TileOperands ops{{Aimg, Aimg, Aimg_lo}, {Bimg, Bimg_lo, Bimg}};
    const int NT = (N + 127) / 128, MT = (M + 127) / 128, items = NT * MT;
    const dim3 grid(items < 148 ? items : 148);
    const size_t smem = 2 * kPStages * kTileBytes;
    const int passes = split ? 3 : 1;
    uint8_t* lo = split ? out_img_lo : nullptr;
    if (relu)
      return split ? launch_pdl(k_tile_gemm_f<true, false, true>, grid, dim3(320), smem, st, ops, passes, KT, G, M, N,
                                NT, MT, bias, mask, out, ldo, out_img, KT_out, nonfinite, lo)
                   : launch_pdl(k_tile_gemm_f<true, false, false>, grid, dim3(320), smem, st, ops, passes, KT, G, M, N,
                                NT, MT, bias, mask, out, ldo, out_img, KT_out, nonfinite, lo);
    return split ? launch_pdl(k_tile_gemm_f<false, true, true>, grid, dim3(320), smem, st, ops, passes, KT, G, M, N, NT,
                              MT, bias, mask, out, ldo, out_img, KT_out, nonfinite, lo)
                 : launch_pdl(k_tile_gemm_f<false, true, false>, grid, dim3(320), smem, st, ops, passes, KT, G, M, N, NT,
                              MT, bias, mask, out, ldo, out_img, KT_out, nonfinite, lo);
  }
  cudaError_t e = tile_gemm_pass(Aimg, Bimg, KT, G, M, N, S, partial, st);
  if (e == cudaSuccess && split) e = tile_gemm_pass(Aimg, Bimg_lo, KT, G, M, N, S, partial + (size_t)S * M * N, st);
  if (e == cudaSuccess && split)
    e = tile_gemm_pass(Aimg_lo, Bimg, KT, G, M, N, S, partial + (size_t)2 * S * M * N, st);
  if (e != cudaSuccess) return e;
  const int St = split ? 3 * S : S;
  if (N % 4 == 0 && (out == nullptr || ldo % 4 == 0)) {
    const int64_t tot = (int64_t)M * ((N + 7) / 8);
    return launch_pdl(k_tile_reduce8, dim3((unsigned)((tot + 255) / 256)), dim3(256), 0, st, partial, St, M, N, bias,
                      mask, relu, out, ldo, out_img, KT_out, nonfinite, split ? out_img_lo : nullptr);
  }
  if (split) return cudaErrorInvalidValue;  // (the projector widths are multiples of 4)
  const int64_t tot = (int64_t)M * N;
  return launch_pdl(k_tile_reduce, dim3((unsigned)((tot + 255) / 256)), dim3(256), 0, st, partial, S, M, N, bias, mask,
                    relu, out, ldo, out_img, KT_out, nonfinite);
}

// ===========================================================================
// Fused projector (bf16 mode): the three MLP layers of
// projection._projector_mlp (projection.py:468-472), the output mask, the
// optional denoiser on theta[3:66] (projection.py:684-697) and the SMPL FK
// (bodymodel.py:266) for NM meshes in ONE launch: a cluster of CS CTAs,
// partial sums reduced through distributed shared memory instead of global
// partial buffers and separate reduce launches.
//
// Transposed formulation: D^T (outputs x meshes) = W^T (outputs x K, the
// uploaded K-major tile images, M = 128) . X^T, the meshes as the N = NM
// operand -- a 32-mesh batch costs a 32-wide MMA instead of a 128-row tile.
//   layer 1: CTA (mt = rank % 4, kq = rank / 4): h1 rows [128 mt, +128) over
//            k-tiles [kq KTq, (kq + 1) KTq) of x (the projector-input image:
//            rows = meshes); ranks 0..3 sum the four K quarters in order,
//            + b1, ReLU -> h1 k-tile mt as the next layer's bf16 operand
//   layer 2: rank u < 8: h2 rows [128 (u % 2), +128) x h1 k-tile u / 2
//            (pulled from rank u / 2); ranks 0, 1 sum + b2, ReLU
//   layer 3: ranks 0, 1: theta rows x h2 k-tile (own); rank 0 sums, + b3,
//            * mask -> theta
//   FK:      warp w of rank r takes mesh r + CS w (theta read from rank 0)
// Every reduction adds the partials in a fixed order, so a mesh gives the
// same bits at any batch position.
// ===========================================================================
namespace {
template <int NM>
constexpr int pf_stages() { return NM == 32 ? 3 : 2; }  // ring depth within the shared-memory budget

__device__ __forceinline__ float4 ld_dsmem_f4(uint32_t addr) {
  float4 v;
  asm volatile("ld.shared::cluster.v4.f32 {%0, %1, %2, %3}, [%4];\n"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "r"(addr));
  return v;
}
__device__ __forceinline__ uint4 ld_dsmem_u4(uint32_t addr) {
  uint4 v;
  asm volatile("ld.shared::cluster.v4.u32 {%0, %1, %2, %3}, [%4];\n"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "r"(addr));
  return v;
}
__device__ __forceinline__ float ld_dsmem_f(uint32_t addr) {
  float v;
  asm volatile("ld.shared::cluster.f32 %0, [%1];\n" : "=f"(v) : "r"(addr));
  return v;
}
}  // namespace

template <int NM, int CS>
__global__ void __launch_bounds__(128, 1)
    k_proj_fused(const uint8_t* __restrict__ ximg, ProjectorDev p, int B, float* __restrict__ theta,
                 const float* __restrict__ grest, float* __restrict__ joints, DenoiseW dn, int* nonfinite) {
  static_assert(NM == 32 || NM == 64, "meshes per cluster");
  static_assert(CS == 8 || CS == 16, "cluster size");
  constexpr int kPfStages = pf_stages<NM>();
  constexpr uint32_t kX = NM * 256;                    // x / h slice: NM rows x K = 128 bf16
  constexpr uint32_t kStage = kTileBytes + kX;
  constexpr uint32_t oRing = 0;
  constexpr uint32_t oPart = oRing + kPfStages * kStage;  // fp32 [128][NM]
  constexpr uint32_t oHt = oPart + 128 * NM * 4;         // this CTA's produced operand slice
  constexpr uint32_t oHb = oHt + kX;                     // the consumed (pulled) operand slice
  constexpr uint32_t oTh = oHb + kX;                     // theta [NM][80] (rank 0)
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ __align__(8) uint64_t bar_full[3], bar_free[3], bar_mma, bar_w;
  __shared__ uint32_t tmem_base;
  __shared__ FKOut fk[4];
  __shared__ float pose_s[4][66];
  __shared__ float dn_h[4][FSB_DN_MAX_HIDDEN];
  __shared__ float dn_o[4][64];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t rank = tc::cluster_rank();
  const int m0 = (int)(blockIdx.x / CS) * NM;            // first mesh of this cluster
  float* part = reinterpret_cast<float*>(smem + oPart);
  uint8_t* ht = smem + oHt;
  uint8_t* hb = smem + oHb;
  float* th = reinterpret_cast<float*>(smem + oTh);
  const uint32_t sbase = tc::smem_u32(smem);
  const uint32_t idesc = tc::idesc_bf16(128, NM);
  if (tid == 0) {
    for (int i = 0; i < kPfStages; ++i) {
      tc::mbar_init(&bar_full[i], 1);
      tc::mbar_init(&bar_free[i], 1);
    }
    tc::mbar_init(&bar_mma, 1);
    tc::mbar_init(&bar_w, 1);
    tc::mbar_fence_init();
  }
  if (warp == 0) tc::tmem_alloc(&tmem_base, NM < 32 ? 32 : NM);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = tmem_base;
  const uint32_t tl = tmem + ((uint32_t)(32 * warp) << 16);
  uint32_t mma_phase = 0;
  pdl_wait();  // x comes from the projector-input kernel

  // D (TMEM, lanes = output rows of this tile, columns = meshes) -> part
  auto drain = [&]() {
    tc::mbar_wait(&bar_mma, mma_phase);
    mma_phase ^= 1u;
    tc::fence_after();
#pragma unroll
    for (int c = 0; c < NM; c += 32) {
      float v[32];
      tc::tmem_ld32(tl + c, v);
#pragma unroll
      for (int i = 0; i < 32; i += 4)
        *reinterpret_cast<float4*>(part + tid * NM + c + i) = make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
    }
    tc::fence_before();
  };
  // sum of the partials of `nsrc` ranks (rank0 + step k), row tid, fixed order
  auto gather_sum = [&](int rank0, int step, int nsrc, float* acc) {
#pragma unroll
    for (int n = 0; n < NM; ++n) acc[n] = 0.0f;
    for (int k = 0; k < nsrc; ++k) {
      const uint32_t src = tc::mapa_shared(part + tid * NM, (uint32_t)(rank0 + step * k));
#pragma unroll
      for (int n = 0; n < NM; n += 4) {
        const float4 v = ld_dsmem_f4(src + 4 * n);
        acc[n] += v.x; acc[n + 1] += v.y; acc[n + 2] += v.z; acc[n + 3] += v.w;
      }
    }
  };
  // activations of rows [128 t0, +128) as the next layer's operand: mesh n,
  // K index tid (bf16, K-major over 128)
  auto store_operand = [&](const float* acc) {
#pragma unroll
    for (int n = 0; n < NM; ++n)
      *reinterpret_cast<__nv_bfloat16*>(ht + tc::kmajor_off(n, tid, 128)) =
          __float2bfloat16_rn(m0 + n < B ? acc[n] : 0.0f);
    tc::fence_async_smem();
  };

  // ---- layer 1 ------------------------------------------------------------
  constexpr int kNkq = CS / 4;  // K splits of layer 1
  const int KT1 = p.KT1, KTq = (KT1 + kNkq - 1) / kNkq;  // (>= 1 k-tile each for the projector's K)
  {
    const int mt = (int)rank & 3, kq = (int)rank >> 2;
    const int kt0 = kq * KTq, nk = max(0, min(KTq, KT1 - kt0));
    if (tid == 0) {
      const uint8_t* xsrc = ximg + ((size_t)(m0 / 128) * KT1) * kTileBytes + (size_t)((m0 % 128) / 8) * 2048;
      auto load = [&](int i) {
        const int s = i % kPfStages;
        tc::mbar_expect_tx(&bar_full[s], kStage);
        tc::bulk_g2s(smem + oRing + s * kStage, p.img_w1 + ((size_t)mt * KT1 + kt0 + i) * kTileBytes, kTileBytes,
                     &bar_full[s]);
        tc::bulk_g2s(smem + oRing + s * kStage + kTileBytes, xsrc + (size_t)(kt0 + i) * kTileBytes, kX,
                     &bar_full[s]);
      };
      for (int i = 0; i < min(nk, kPfStages); ++i) load(i);
      for (int i = 0; i < nk; ++i) {
        const int s = i % kPfStages;
        tc::mbar_wait(&bar_full[s], (uint32_t)((i / kPfStages) & 1));
        tc::fence_after();
        const uint32_t a = sbase + oRing + s * kStage, b = a + kTileBytes;
        for (int k = 0; k < 128; k += 16)
          tc::mma_bf16(tmem, tc::kmajor_desc(a, 128, k), tc::kmajor_desc(b, 128, k), idesc, (i | k) != 0);
        tc::mma_commit(&bar_free[s]);
        if (i + kPfStages < nk) {
          tc::mbar_wait(&bar_free[s], (uint32_t)((i / kPfStages) & 1));
          load(i + kPfStages);
        }
      }
      tc::mma_commit(&bar_mma);
    }
    __syncwarp();
    drain();
  }
  tc::cluster_sync_all();
  if (rank < 4) {  // h1 k-tile `rank`
    float acc[NM];
    gather_sum((int)rank, 4, kNkq, acc);
    const float b = __ldg(p.b1 + 128 * rank + tid);
#pragma unroll
    for (int n = 0; n < NM; ++n) acc[n] = fmaxf(acc[n] + b, 0.0f);
    store_operand(acc);
  }
  tc::cluster_sync_all();

  // ---- layer 2 ------------------------------------------------------------
  const int KT2 = p.KT2;  // 4 (h1 = 512)
  if ((int)rank < 2 * KT2) {
    const int mt2 = (int)rank & 1, kt2 = (int)rank >> 1;
    if (tid == 0) {
      tc::mbar_expect_tx(&bar_w, kTileBytes);
      tc::bulk_g2s(smem + oRing, p.img_w2 + ((size_t)mt2 * KT2 + kt2) * kTileBytes, kTileBytes, &bar_w);
    }
    const uint32_t src = tc::mapa_shared(ht, (uint32_t)kt2);
    for (uint32_t o = 16 * tid; o < kX; o += 16 * 128)
      *reinterpret_cast<uint4*>(hb + o) = ld_dsmem_u4(src + o);
    tc::fence_async_smem();
    __syncthreads();
    if (tid == 0) {
      tc::mbar_wait(&bar_w, 0);
      tc::fence_after();
      const uint32_t a = sbase + oRing, b = sbase + oHb;
      for (int k = 0; k < 128; k += 16)
        tc::mma_bf16(tmem, tc::kmajor_desc(a, 128, k), tc::kmajor_desc(b, 128, k), idesc, k != 0);
      tc::mma_commit(&bar_mma);
    }
    __syncwarp();
    drain();
  }
  tc::cluster_sync_all();
  if (rank < 2) {  // h2 k-tile `rank`
    float acc[NM];
    gather_sum((int)rank, 2, KT2, acc);
    const float b = __ldg(p.b2 + 128 * rank + tid);
#pragma unroll
    for (int n = 0; n < NM; ++n) acc[n] = fmaxf(acc[n] + b, 0.0f);
    store_operand(acc);
  }
  tc::cluster_sync_all();

  // ---- layer 3 ------------------------------------------------------------
  const int KT3 = p.KT3;  // 2 (h2 = 256)
  if ((int)rank < KT3) {
    if (tid == 0) {
      tc::mbar_expect_tx(&bar_w, kTileBytes);
      tc::bulk_g2s(smem + oRing, p.img_w3 + (size_t)rank * kTileBytes, kTileBytes, &bar_w);
      tc::mbar_wait(&bar_w, 1);
      tc::fence_after();
      const uint32_t a = sbase + oRing, b = sbase + oHt;  // h2 k-tile `rank` is this CTA's own
      for (int k = 0; k < 128; k += 16)
        tc::mma_bf16(tmem, tc::kmajor_desc(a, 128, k), tc::kmajor_desc(b, 128, k), idesc, k != 0);
      tc::mma_commit(&bar_mma);
    }
    __syncwarp();
    drain();
  }
  tc::cluster_sync_all();
  if (rank == 0 && tid < FSB_PARAM_DIM) {  // theta = (sum + b3) * mask
    float acc[NM];
    gather_sum(0, 1, KT3, acc);
    const float b = __ldg(p.b3 + tid), mk = __ldg(p.mask + tid);
#pragma unroll
    for (int n = 0; n < NM; ++n) {
      const float v = (acc[n] + b) * mk;
      th[n * 80 + tid] = v;
      if (m0 + n < B) {
        flag_nonfinite(nonfinite, v);
        theta[(int64_t)(m0 + n) * FSB_PARAM_DIM + tid] = v;
      }
    }
  }
  tc::cluster_sync_all();

  // ---- SMPL FK (+ denoiser) -------------------------------------------------
  for (int w = warp; joints != nullptr && w * CS < NM; w += 4) {  // (joints == nullptr: projector only)
    const int n = (int)rank + CS * w, b = m0 + n;
    if (b >= B) continue;  // warp-uniform
    const uint32_t src = tc::mapa_shared(th + n * 80, 0u);
    for (int i = lane; i < 66; i += 32) pose_s[warp][i] = ld_dsmem_f(src + 4 * i);
    __syncwarp();
    if (dn.H > 0) {
      denoise_warp(pose_s[warp] + 3, dn_h[warp], dn, lane, dn_o[warp], nonfinite);
      for (int i = lane; i < FSB_DN_IN; i += 32) {
        pose_s[warp][3 + i] = dn_o[warp][i];
        theta[(int64_t)b * FSB_PARAM_DIM + 3 + i] = dn_o[warp][i];
      }
      __syncwarp();
    }
    fk_warp(pose_s[warp], grest, fk[warp], lane);
    if (lane < FSB_NJ)
      for (int a = 0; a < 3; ++a) joints[((int64_t)b * FSB_NJ + lane) * 3 + a] = fk[warp].tw[lane][a];
    __syncwarp();
  }
  tc::cluster_sync_all();  // rank 0's theta and the operand slices stay alive until every CTA is done
  tc::fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc(tmem, NM < 32 ? 32 : NM);
}

namespace {
template <int NM, int CS>
constexpr uint32_t proj_fused_smem() {
  return pf_stages<NM>() * (kTileBytes + NM * 256) + 128 * NM * 4 + 2 * NM * 256 + NM * 80 * 4;
}
template <int NM, int CS>
cudaError_t launch_pf(const uint8_t* ximg, const ProjectorDev& p, int B, float* theta, const float* grest,
                      float* joints, const DenoiseW& dn, int* nonfinite, cudaStream_t st) {
  auto k = k_proj_fused<NM, CS>;
  static bool init = false;
  if (!init) {
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)proj_fused_smem<NM, CS>());
    if (e != cudaSuccess) return e;
    if (CS > 8) {
      e = cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      if (e != cudaSuccess) return e;
    }
    init = true;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)(((B + NM - 1) / NM) * CS));
  cfg.blockDim = dim3(128);
  cfg.dynamicSmemBytes = proj_fused_smem<NM, CS>();
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CS;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 2;
  return cudaLaunchKernelEx(&cfg, k, ximg, p, B, theta, grest, joints, dn, nonfinite);
}
}  // namespace

#ifndef FSB_PF_CS
#define FSB_PF_CS 8  // 16 measured slower under concurrent streams (cluster placement)
#endif
// true when the fused projector serves this projector's shape (h1 = 512,
// h2 = 256, theta = 76 outputs: the default (512, 256) widths)
bool proj_fused_ok(const ProjectorDev& p) { return p.h1 == 512 && p.h2 == 256 && p.KT2 == 4 && p.KT3 == 2; }

cudaError_t launch_proj_fused(const uint8_t* ximg, const ProjectorDev& p, int B, float* theta, const float* grest,
                              float* joints, const DenoiseW* dn, int* nonfinite, cudaStream_t st) {
  if (B == 0) return cudaSuccess;
  const DenoiseW d = dn ? *dn : DenoiseW{nullptr, nullptr, nullptr, nullptr, 0};
  if (B <= 32) return launch_pf<32, FSB_PF_CS>(ximg, p, B, theta, grest, joints, d, nonfinite, st);
  return launch_pf<64, FSB_PF_CS>(ximg, p, B, theta, grest, joints, d, nonfinite, st);
}
