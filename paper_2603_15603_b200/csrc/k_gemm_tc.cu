// Generic bf16 GEMM on tcgen05 for the large-config encoder (C4, ViT-L size):
//   C[M, N] = A[M, K] . W[N, K]^T  (+ fused epilogue)
// A and W are row-major bf16 (K contiguous, i.e. both operands K-major).
//
// Persistent kernel: one CTA per SM walks the 128 x BN output tiles
// (N-tile fastest, so CTAs running at the same time share A tiles in L2).
// Warp 0 is the TMA producer (128-byte swizzled boxes of 64 K-elements),
// warp 1 issues tcgen05.mma from one lane, warps 2-9 drain TMEM through the
// epilogue (two warps per TMEM lane quadrant, each on half the columns;
// 32-row blocks staged in swizzled shared memory and moved by TMA).  A STAGES-deep ring of full/empty mbarriers feeds the tensor
// core, and the accumulator is double-buffered in TMEM (2 x BN columns):
// the epilogue of tile i runs while the MMAs of tile i+1 accumulate into the
// other buffer.  Epilogues (decoder.py:247-257 semantics):
//   EPI_BIAS_BF16   out_bf16 = acc + bias                       (Q|K|V)
//   EPI_RELU_BF16   out_bf16 = relu(acc + bias)                 (MLP W1)
//   EPI_RESID_F32   x_f32   += acc + bias                       (Wo, W2)
//   EPI_EMBED_F32   x_f32    = (acc + bias) + pos[row % T]      (patch embed)
#include <cuda.h>
#include <cudaTypedefs.h>
#include <stdio.h>
#include <stdlib.h>

#include "fsb_common.cuh"
#include "tc_sm100.cuh"

#include "gemm_tc.h"

namespace {
#ifndef GEMM_STAGES
#define GEMM_STAGES 4
#endif
#ifndef GEMM_EPI_WARPS
#define GEMM_EPI_WARPS 4
#endif
constexpr int BM = 128, BK = 64, STAGES = GEMM_STAGES;
constexpr uint32_t EPI_BUF = 4096;  // per-warp staging buffer: 32 rows x 128 B, 128-byte swizzle
constexpr int EPI_WARPS = GEMM_EPI_WARPS;  // 4: one per TMEM lane quadrant; 8: two, each on half the columns
constexpr int GEMM_THREADS = 64 + 32 * EPI_WARPS;
}

// 128-byte-swizzled staging row: 16-byte chunk q of row r
__device__ __forceinline__ uint32_t sw128_off(int r, int q) { return (uint32_t)(r * 128 + ((q ^ (r & 7)) << 4)); }

template <int BN>
__global__ void __launch_bounds__(GEMM_THREADS, 1)
    k_gemm_tc(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
              const __grid_constant__ CUtensorMap tmC, int M, int N, int K, GemmEpi epi) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 1024-byte alignment for the 128B swizzle atoms
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  constexpr uint32_t A_BYTES = BM * BK * 2, B_BYTES = BN * BK * 2, STAGE_BYTES = A_BYTES + B_BYTES;
  constexpr uint32_t TMEM_COLS = 2 * BN;  // two accumulator buffers
  __shared__ uint64_t full[STAGES], empty[STAGES], acc_full[2], acc_empty[2], xbar[2 * EPI_WARPS];
  __shared__ uint32_t tmem_base;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int nk = (K + BK - 1) / BK;
  const int ntn = (N + BN - 1) / BN, ntm = (M + BM - 1) / BM;
  const int ntiles = ntm * ntn;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      tc::mbar_init(&full[s], 1);
      tc::mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      tc::mbar_init(&acc_full[b], 1);
      tc::mbar_init(&acc_empty[b], EPI_WARPS);
    }
    for (int i = 0; i < 2 * EPI_WARPS; ++i) tc::mbar_init(&xbar[i], 1);
    tc::mbar_fence_init();
    tc::prefetch_tmap(&tmA);
    tc::prefetch_tmap(&tmB);
    tc::prefetch_tmap(&tmC);
  }
  if (warp == 1) tc::tmem_alloc(&tmem_base, TMEM_COLS);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = tmem_base;

  if (warp == 0) {
    // TMA producer: the whole warp walks the schedule, lane 0 issues
    int it = 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
      const int m0 = (t / ntn) * BM, n0 = (t % ntn) * BN;
      for (int kb = 0; kb < nk; ++kb, ++it) {
        const int s = it % STAGES;
        if (it >= STAGES) tc::mbar_wait(&empty[s], (uint32_t)(((it / STAGES) - 1) & 1));
        if (lane == 0) {
          uint8_t* sa = smem + s * STAGE_BYTES;
          tc::mbar_expect_tx(&full[s], STAGE_BYTES);
          tc::tma_load_2d(sa, &tmA, kb * BK, m0, &full[s]);
          tc::tma_load_2d(sa + A_BYTES, &tmB, kb * BK, n0, &full[s]);
        }
        __syncwarp();
      }
    }
  } else if (warp == 1) {
    // MMA issuer: the whole warp walks the schedule, lane 0 issues
    const uint32_t idesc = tc::idesc_bf16(BM, BN);
    const uint32_t sbase = tc::smem_u32(smem);
    int it = 0, tc_count = 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++tc_count) {
      const int buf = tc_count & 1;
      if (tc_count >= 2) tc::mbar_wait(&acc_empty[buf], (uint32_t)(((tc_count >> 1) - 1) & 1));
      tc::fence_after();
      const uint32_t acc = tmem + (uint32_t)(buf * BN);
      for (int kb = 0; kb < nk; ++kb, ++it) {
        const int s = it % STAGES;
        tc::mbar_wait(&full[s], (uint32_t)((it / STAGES) & 1));
        tc::fence_after();
        if (lane == 0) {
          const uint32_t a = sbase + s * STAGE_BYTES, b = a + A_BYTES;
#pragma unroll
          for (int k = 0; k < BK / 16; ++k)
            tc::mma_bf16(acc, tc::sw128_kmajor_desc(a + 32 * k), tc::sw128_kmajor_desc(b + 32 * k), idesc,
                         (kb | k) != 0);
          tc::mma_commit(&empty[s]);  // frees the stage once these MMAs have read it
        }
        __syncwarp();
      }
      if (lane == 0) tc::mma_commit(&acc_full[buf]);  // accumulator of this tile complete
      __syncwarp();
    }
  } else if (warp >= 2) {
    // epilogue: warp w reads TMEM lanes 32 * (w % 4) .. +31 (rows of the
    // tile); warps w and w + 4 split the columns.  Each warp stages 32-row
    // blocks (128-byte rows: 32 fp32 or 64 bf16 columns) in two swizzled
    // shared-memory buffers and moves them with TMA: fp32 residual blocks
    // are TMA-loaded, updated in shared memory and TMA-stored; bf16 blocks
    // are written to shared memory and TMA-stored.  Global traffic is thus
    // whole 128-byte rows, issued by the TMA engine.
    const int ew = warp - 2, quad = warp % 4, half = ew / 4;
    constexpr int HALF = BN / (EPI_WARPS / 4);
    uint8_t* stg = smem + STAGES * STAGE_BYTES + ew * 2 * EPI_BUF;
    const bool f32 = epi.kind == EPI_RESID_F32 || epi.kind == EPI_EMBED_F32;
    const bool resid = epi.kind == EPI_RESID_F32;
    const int CB = f32 ? 32 : 64;  // columns per staged block
    int tc_count = 0, nblk = 0;    // nblk: blocks staged by this warp so far
    uint32_t xph[2] = {0u, 0u};
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++tc_count) {
      const int buf = tc_count & 1;
      const int m0 = (t / ntn) * BM, n0 = (t % ntn) * BN;
      const int r0 = m0 + quad * 32, row = r0 + lane;
      const int cbase = n0 + half * HALF;
      const uint32_t taddr = tmem + ((uint32_t)(quad * 32) << 16) + (uint32_t)(buf * BN + half * HALF);
      const int nb = HALF / CB;
      // residual blocks of this tile: the first two are fetched before the
      // MMAs finish (their staging buffers are free once earlier stores
      // have read them)
      auto fetch = [&](int k) {
        const int sb = (nblk + k) & 1;
        if (lane == 0) {
          tc::bulk_wait_read0();
          tc::mbar_expect_tx(&xbar[2 * ew + sb], EPI_BUF);
          tc::tma_load_2d(stg + sb * EPI_BUF, &tmC, cbase + k * CB, r0, &xbar[2 * ew + sb]);
        }
      };
      if (resid && r0 < M) {
        fetch(0);
        if (nb > 1) fetch(1);
      }
      tc::mbar_wait(&acc_full[buf], (uint32_t)((tc_count >> 1) & 1));
      tc::fence_after();
      for (int k = 0; k < nb; ++k) {
        const int sb = (nblk + k) & 1;
        uint8_t* sbuf = stg + sb * EPI_BUF;
        const int col = cbase + k * CB;
        float v[64];
        tc::tmem_ld32(taddr + k * CB, v);
        if (!f32) tc::tmem_ld32(taddr + k * CB + 32, v + 32);
        if (k + 1 == nb) {
          // last TMEM read of this tile by this warp: release the buffer
          tc::fence_before();
          __syncwarp();
          if (lane == 0) tc::mbar_arrive(&acc_empty[buf]);
        }
        if (r0 >= M || col >= N) continue;  // warp-uniform
#pragma unroll
        for (int i = 0; i < 32; i += 4) {  // + bias (same columns for every lane)
          const float4 q = __ldg(reinterpret_cast<const float4*>(epi.bias + col + i));
          v[i] += q.x; v[i + 1] += q.y; v[i + 2] += q.z; v[i + 3] += q.w;
        }
        if (!f32) {
          if (col + 32 < N)  // N is a multiple of 32; the TMA store clips columns >= N
#pragma unroll
            for (int i = 32; i < 64; i += 4) {
              const float4 q = __ldg(reinterpret_cast<const float4*>(epi.bias + col + i));
              v[i] += q.x; v[i + 1] += q.y; v[i + 2] += q.z; v[i + 3] += q.w;
            }
          if (epi.kind == EPI_RELU_BF16)
#pragma unroll
            for (int i = 0; i < 64; ++i) v[i] = fmaxf(v[i], 0.0f);
          if (lane == 0) tc::bulk_wait_read0();  // the store that last used this buffer has read it
          __syncwarp();
#pragma unroll
          for (int q = 0; q < 8; ++q)
            *reinterpret_cast<uint4*>(sbuf + sw128_off(lane, q)) =
                make_uint4(tc::pack_bf16(v[8 * q], v[8 * q + 1]), tc::pack_bf16(v[8 * q + 2], v[8 * q + 3]),
                           tc::pack_bf16(v[8 * q + 4], v[8 * q + 5]), tc::pack_bf16(v[8 * q + 6], v[8 * q + 7]));
        } else if (resid) {
          tc::mbar_wait(&xbar[2 * ew + sb], xph[sb]);
          xph[sb] ^= 1u;
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            float4* p = reinterpret_cast<float4*>(sbuf + sw128_off(lane, q));
            float4 x = *p;
            x.x += v[4 * q]; x.y += v[4 * q + 1]; x.z += v[4 * q + 2]; x.w += v[4 * q + 3];
            *p = x;
          }
        } else {  // EPI_EMBED_F32: x = (acc + bias) + pos[row % T]
          if (lane == 0) tc::bulk_wait_read0();
          __syncwarp();
          const float4* pr = reinterpret_cast<const float4*>(epi.pos + (size_t)(row % epi.T) * epi.ldo + col);
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const float4 pp = __ldg(pr + q);
            *reinterpret_cast<float4*>(sbuf + sw128_off(lane, q)) =
                make_float4(v[4 * q] + pp.x, v[4 * q + 1] + pp.y, v[4 * q + 2] + pp.z, v[4 * q + 3] + pp.w);
          }
        }
        tc::fence_async_smem();
        __syncwarp();
        if (lane == 0) {
          tc::tma_store_2d(&tmC, col, r0, sbuf);
          tc::bulk_commit();
        }
        if (resid && k + 2 < nb) fetch(k + 2);
      }
      nblk += nb;
    }
    if (lane == 0) tc::bulk_wait0();  // stores complete before the CTA exits
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 1) tc::tmem_dealloc(tmem, TMEM_COLS);
}

// ---------------------------------------------------------------------------
// CTA-pair variant (cta_group::2): a cluster of two CTAs on one TPC computes a
// 256 x 256 tile.  CTA r holds A rows [128 r, +128) and B rows (output
// columns) [128 r, +128) of every stage; the leader's single MMA lane issues
// M = 256 tcgen05.mma that read both CTAs' shared memory and accumulate into
// both CTAs' TMEM (rows [128 r, +128) in CTA r).  Per SM and k-block this
// moves 32 KB through shared memory instead of 48 KB (TMA writes + MMA reads
// of a 128 x 256 single-CTA tile exceed the 128 B/clk the SM provides).
//   full[s]     leader only: expect_tx by the leader's producer for both
//               CTAs' bytes; both CTAs' TMA loads complete on it
//   empty[s]    each CTA: the leader's commit multicasts to both
//   acc_full[b] each CTA: the leader's commit multicasts to both
//   acc_empty[b] leader only: 2 x EPI_WARPS arrivals, the peer's remote
// The epilogue is the single-CTA one on this CTA's 128 rows.
// ---------------------------------------------------------------------------
#ifndef GEMM2_STAGES
#define GEMM2_STAGES 5
#endif
#ifndef GEMM2_EPI_BUFS
#define GEMM2_EPI_BUFS 4
#endif
#ifndef GEMM2_EPI_WARPS
#define GEMM2_EPI_WARPS 4
#endif
namespace {
constexpr int STAGES2 = GEMM2_STAGES, BN2 = 256, NBUF2 = GEMM2_EPI_BUFS;  // NBUF2: staging buffers per epilogue warp
constexpr int EPI_WARPS2 = GEMM2_EPI_WARPS, GEMM_THREADS2 = 64 + 32 * EPI_WARPS2;
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(GEMM_THREADS2, 1)
    k_gemm_tc2(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
               const __grid_constant__ CUtensorMap tmC, int M, int N, int K, GemmEpi epi) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  constexpr uint32_t A_BYTES = BM * BK * 2, B_BYTES = (BN2 / 2) * BK * 2, STAGE_BYTES = A_BYTES + B_BYTES;
  constexpr uint32_t TMEM_COLS = 2 * BN2;
  __shared__ uint64_t full[STAGES2], empty[STAGES2], acc_full[2], acc_empty[2], xbar[NBUF2 * EPI_WARPS2];
  __shared__ uint32_t tmem_base;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const uint32_t rank = tc::cluster_rank();
  const bool leader = rank == 0;
  const int nk = (K + BK - 1) / BK;
  const int ntn = N / BN2, ntm = (M + 2 * BM - 1) / (2 * BM);
  const int ntiles = ntm * ntn;
  const int cid = blockIdx.x / 2, ncl = gridDim.x / 2;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES2; ++s) {
      tc::mbar_init(&full[s], 1);
      tc::mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      tc::mbar_init(&acc_full[b], 1);
      tc::mbar_init(&acc_empty[b], 2 * EPI_WARPS2);
    }
    for (int i = 0; i < NBUF2 * EPI_WARPS2; ++i) tc::mbar_init(&xbar[i], 1);
    tc::mbar_fence_init();
    tc::prefetch_tmap(&tmA);
    tc::prefetch_tmap(&tmB);
    tc::prefetch_tmap(&tmC);
  }
  if (warp == 1) tc::tmem_alloc_pair(&tmem_base, TMEM_COLS);
  tc::fence_before();
  __syncthreads();
  tc::cluster_sync_all();  // both CTAs' barriers initialised before any remote use
  tc::fence_after();
  const uint32_t tmem = tmem_base;

  if (warp == 0) {
    // TMA producer (both CTAs): this CTA's A and B halves of each stage
    int it = 0;
    for (int t = cid; t < ntiles; t += ncl) {
      const int m0 = (t / ntn) * 2 * BM + (int)rank * BM, n0 = (t % ntn) * BN2 + (int)rank * (BN2 / 2);
      for (int kb = 0; kb < nk; ++kb, ++it) {
        const int s = it % STAGES2;
        if (it >= STAGES2) tc::mbar_wait(&empty[s], (uint32_t)(((it / STAGES2) - 1) & 1));
        if (lane == 0) {
          uint8_t* sa = smem + s * STAGE_BYTES;
          if (leader) tc::mbar_expect_tx(&full[s], 2 * STAGE_BYTES);
          tc::tma_load_2d_pair(sa, &tmA, kb * BK, m0, &full[s]);
          tc::tma_load_2d_pair(sa + A_BYTES, &tmB, kb * BK, n0, &full[s]);
        }
        __syncwarp();
      }
    }
  } else if (warp == 1) {
    if (leader) {
      // MMA issuer (leader CTA only)
      const uint32_t idesc = tc::idesc_bf16(2 * BM, BN2);
      const uint32_t sbase = tc::smem_u32(smem);
      int it = 0, tc_count = 0;
      for (int t = cid; t < ntiles; t += ncl, ++tc_count) {
        const int buf = tc_count & 1;
        if (tc_count >= 2) tc::mbar_wait(&acc_empty[buf], (uint32_t)(((tc_count >> 1) - 1) & 1));
        tc::fence_after();
        const uint32_t acc = tmem + (uint32_t)(buf * BN2);
        for (int kb = 0; kb < nk; ++kb, ++it) {
          const int s = it % STAGES2;
          tc::mbar_wait(&full[s], (uint32_t)((it / STAGES2) & 1));
          tc::fence_after();
          if (lane == 0) {
            const uint32_t a = sbase + s * STAGE_BYTES, b = a + A_BYTES;
#pragma unroll
            for (int k = 0; k < BK / 16; ++k)
              tc::mma_bf16_pair(acc, tc::sw128_kmajor_desc(a + 32 * k), tc::sw128_kmajor_desc(b + 32 * k), idesc,
                                (kb | k) != 0);
            tc::mma_commit_pair(&empty[s], 0x3);  // frees the stage in both CTAs
          }
          __syncwarp();
        }
        if (lane == 0) tc::mma_commit_pair(&acc_full[buf], 0x3);  // both CTAs' accumulators complete
        __syncwarp();
      }
    }
  } else if (warp >= 2) {
    // epilogue on this CTA's 128 rows (as in k_gemm_tc)
    const int ew = warp - 2, quad = warp % 4, half = ew / 4;
    constexpr int HALF = BN2 / (EPI_WARPS2 / 4);
    uint8_t* stg = smem + STAGES2 * STAGE_BYTES + ew * NBUF2 * EPI_BUF;
    const bool f32 = epi.kind == EPI_RESID_F32 || epi.kind == EPI_EMBED_F32;
    const bool resid = epi.kind == EPI_RESID_F32;
    const int CB = f32 ? 32 : 64;
    const uint32_t acc_empty_leader0 = tc::mapa_shared(&acc_empty[0], 0);
    const uint32_t acc_empty_leader1 = tc::mapa_shared(&acc_empty[1], 0);
    int tc_count = 0, nblk = 0;
    uint32_t xph[NBUF2];
#pragma unroll
    for (int i = 0; i < NBUF2; ++i) xph[i] = 0u;
    for (int t = cid; t < ntiles; t += ncl, ++tc_count) {
      const int buf = tc_count & 1;
      const int m0 = (t / ntn) * 2 * BM + (int)rank * BM, n0 = (t % ntn) * BN2;
      const int r0 = m0 + quad * 32, row = r0 + lane;
      const int cbase = n0 + half * HALF;
      const uint32_t taddr = tmem + ((uint32_t)(quad * 32) << 16) + (uint32_t)(buf * BN2 + half * HALF);
      const int nb = HALF / CB;
      // residual blocks run NBUF2 ahead of their use (the epilogue of the
      // memory-bound Wo / W2 GEMMs is bound by these loads)
      auto fetch = [&](int k) {
        const int sb = (nblk + k) % NBUF2;
        if (lane == 0) {
          tc::bulk_wait_read0();
          tc::mbar_expect_tx(&xbar[NBUF2 * ew + sb], EPI_BUF);
          tc::tma_load_2d(stg + sb * EPI_BUF, &tmC, cbase + k * CB, r0, &xbar[NBUF2 * ew + sb]);
        }
      };
      if (resid && r0 < M)
        for (int k = 0; k < NBUF2 && k < nb; ++k) fetch(k);
      tc::mbar_wait(&acc_full[buf], (uint32_t)((tc_count >> 1) & 1));
      tc::fence_after();
      for (int k = 0; k < nb; ++k) {
        const int sb = (nblk + k) % NBUF2;
        uint8_t* sbuf = stg + sb * EPI_BUF;
        const int col = cbase + k * CB;
        float v[64];
        tc::tmem_ld32(taddr + k * CB, v);
        if (!f32) tc::tmem_ld32(taddr + k * CB + 32, v + 32);
        if (k + 1 == nb) {
          tc::fence_before();
          __syncwarp();
          if (lane == 0) tc::mbar_arrive_cluster(buf ? acc_empty_leader1 : acc_empty_leader0);
        }
        if (r0 >= M || col >= N) continue;  // warp-uniform
#pragma unroll
        for (int i = 0; i < 32; i += 4) {
          const float4 q = __ldg(reinterpret_cast<const float4*>(epi.bias + col + i));
          v[i] += q.x; v[i + 1] += q.y; v[i + 2] += q.z; v[i + 3] += q.w;
        }
        if (!f32) {
          if (col + 32 < N)
#pragma unroll
            for (int i = 32; i < 64; i += 4) {
              const float4 q = __ldg(reinterpret_cast<const float4*>(epi.bias + col + i));
              v[i] += q.x; v[i + 1] += q.y; v[i + 2] += q.z; v[i + 3] += q.w;
            }
          if (epi.kind == EPI_RELU_BF16)
#pragma unroll
            for (int i = 0; i < 64; ++i) v[i] = fmaxf(v[i], 0.0f);
          if (lane == 0) tc::bulk_wait_read0();
          __syncwarp();
#pragma unroll
          for (int q = 0; q < 8; ++q)
            *reinterpret_cast<uint4*>(sbuf + sw128_off(lane, q)) =
                make_uint4(tc::pack_bf16(v[8 * q], v[8 * q + 1]), tc::pack_bf16(v[8 * q + 2], v[8 * q + 3]),
                           tc::pack_bf16(v[8 * q + 4], v[8 * q + 5]), tc::pack_bf16(v[8 * q + 6], v[8 * q + 7]));
        } else if (resid) {
          tc::mbar_wait(&xbar[NBUF2 * ew + sb], xph[sb]);
          xph[sb] ^= 1u;
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            float4* p = reinterpret_cast<float4*>(sbuf + sw128_off(lane, q));
            float4 x = *p;
            x.x += v[4 * q]; x.y += v[4 * q + 1]; x.z += v[4 * q + 2]; x.w += v[4 * q + 3];
            *p = x;
          }
        } else {  // EPI_EMBED_F32
          if (lane == 0) tc::bulk_wait_read0();
          __syncwarp();
          const float4* pr = reinterpret_cast<const float4*>(epi.pos + (size_t)(row % epi.T) * epi.ldo + col);
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const float4 pp = __ldg(pr + q);
            *reinterpret_cast<float4*>(sbuf + sw128_off(lane, q)) =
                make_float4(v[4 * q] + pp.x, v[4 * q + 1] + pp.y, v[4 * q + 2] + pp.z, v[4 * q + 3] + pp.w);
          }
        }
        tc::fence_async_smem();
        __syncwarp();
        if (lane == 0) {
          tc::tma_store_2d(&tmC, col, r0, sbuf);
          tc::bulk_commit();
        }
        if (resid && k + NBUF2 < nb) fetch(k + NBUF2);
      }
      nblk += nb;
    }
    if (lane == 0) tc::bulk_wait0();
  }
  tc::fence_before();
  __syncthreads();
  tc::cluster_sync_all();  // the leader's MMAs into this CTA's TMEM / from its smem are done
  if (warp == 1) tc::tmem_dealloc_pair(tmem, TMEM_COLS);
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

// row-major fp32 matrix as a 2-D tensor map with (box_rows x 32)-element
// boxes (128-byte rows), 128-byte swizzle
static bool make_tmap_f32(CUtensorMap* map, const void* base, uint64_t rows, uint64_t cols, uint64_t ld,
                          uint32_t box_rows) {
  auto enc = tmap_encoder();
  if (!enc) return false;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {ld * 4};
  cuuint32_t box[2] = {32, box_rows};
  cuuint32_t es[2] = {1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(base), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int BN>
static constexpr size_t gemm_smem() {
  return (size_t)STAGES * (BM * BK * 2 + BN * BK * 2) + (size_t)EPI_WARPS * 2 * EPI_BUF + 1024;
}

static constexpr size_t gemm2_smem() {
  return (size_t)STAGES2 * (BM * BK * 2 + (BN2 / 2) * BK * 2) + (size_t)EPI_WARPS2 * NBUF2 * EPI_BUF + 1024;
}

cudaError_t init_attrs_gemm_tc() {
  cudaError_t e = cudaFuncSetAttribute(k_gemm_tc<256>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)gemm_smem<256>());
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(k_gemm_tc<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)gemm_smem<128>());
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(k_gemm_tc2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)gemm2_smem());
  return e;
}

// FSB_GEMM_PAIR=0 selects the single-CTA kernel for every shape (A/B runs)
static bool use_pair() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("FSB_GEMM_PAIR");
    v = (e != nullptr && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}

// A (M x K, lda), W (N x K, ldw): bf16 row-major.  N must be a multiple of 32,
// K a multiple of 8 (16-byte TMA strides).
cudaError_t launch_gemm_tc(const __nv_bfloat16* A, int lda, const __nv_bfloat16* W, int ldw, int M, int N, int K,
                           const GemmEpi& epi, cudaStream_t st) {
  if (M == 0 || N == 0) return cudaSuccess;
  if (N % 32 || K % 8 || lda % 8 || ldw % 8) return cudaErrorInvalidValue;
  static bool attrs = false;
  if (!attrs) {
    cudaError_t e = init_attrs_gemm_tc();
    if (e != cudaSuccess) return e;
    attrs = true;
  }
  CUtensorMap ta, tb, tc_;
  const int BN = (N % 256 == 0) ? 256 : 128;
  const bool pair = BN == 256 && M > BM && use_pair();
  if (!make_tmap_bf16(&ta, A, M, K, lda, BM) || !make_tmap_bf16(&tb, W, N, K, ldw, pair ? BN / 2 : BN))
    return cudaErrorInvalidValue;
  // epilogue blocks: 32 rows x 128 bytes (fp32: 32 columns, bf16: 64)
  const bool f32 = epi.kind == EPI_RESID_F32 || epi.kind == EPI_EMBED_F32;
  if (f32 ? !make_tmap_f32(&tc_, epi.x_f32, M, N, epi.ldo, 32) : !make_tmap_bf16(&tc_, epi.out_bf16, M, N, epi.ldo, 32))
    return cudaErrorInvalidValue;
  static int sms = 0;
  if (sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || sms <= 0) sms = 148;
  }
  if (pair) {  // persistent clusters of two CTAs, one 256 x 256 tile at a time
    const int64_t tiles = (int64_t)(N / BN2) * ((M + 2 * BM - 1) / (2 * BM));
    const int64_t ncl = tiles < sms / 2 ? tiles : sms / 2;
    k_gemm_tc2<<<dim3((unsigned)(2 * ncl)), GEMM_THREADS2, gemm2_smem(), st>>>(ta, tb, tc_, M, N, K, epi);
    return cudaGetLastError();
  }
  const int64_t tiles = (int64_t)((N + BN - 1) / BN) * ((M + BM - 1) / BM);
  const dim3 grid((unsigned)(tiles < sms ? tiles : sms));  // persistent: one CTA per SM
  if (BN == 256)
    k_gemm_tc<256><<<grid, GEMM_THREADS, gemm_smem<256>(), st>>>(ta, tb, tc_, M, N, K, epi);
  else
    k_gemm_tc<128><<<grid, GEMM_THREADS, gemm_smem<128>(), st>>>(ta, tb, tc_, M, N, K, epi);
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
