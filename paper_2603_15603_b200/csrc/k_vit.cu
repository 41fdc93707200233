// Large-config encoder (C4): Decoder.encode (decoder.py:231-260) at ViT-L
// size -- S=384 crops, p=16 patches (T=576 tokens), D=1024, 16 heads of 64.
//
// Per layer (pre-LN, decoder.py:214-218 / 205-212):
//   h   = LN1(x)                          k_layernorm  (fp32 -> bf16)
//   qkv = h Wqkv^T + bqkv                 k_gemm_tc    EPI_BIAS_BF16
//   ctx = softmax(q k^T / 8) v            k_attn_tc    (flash attention)
//   x  += ctx Wo^T + bo                   k_gemm_tc    EPI_RESID_F32
//   h   = LN2(x)                          k_layernorm
//   hid = relu(h W1^T + b1)               k_gemm_tc    EPI_RELU_BF16
//   x  += hid W2^T + b2                   k_gemm_tc    EPI_RESID_F32
// preceded by the patch embedding (k_patchify + EPI_EMBED_F32 GEMM) and
// followed by the final LayerNorm into the fp32 feature tensor.
#include <cuda.h>
#include <stdio.h>

#include "fsb_common.cuh"
#include "fsb_vit.h"
#include "gemm_tc.h"
#include "tc_sm100.cuh"

namespace {

// ---------------------------------------------------------------------------
// patchify: (n, S, S, 3) fp32 -> (n*T, p*p*3) bf16 rows in (py, px, c) order
// (the reshape/transpose of decoder.py:237-241).  Each patch row py is a
// contiguous run of p*3 floats in the crop, so 8 consecutive outputs are 8
// consecutive inputs whenever p*3 % 8 == 0 (p = 16: runs of 48).
__global__ void k_patchify(const float* __restrict__ crops, int n, int S, int p, __nv_bfloat16* __restrict__ out) {
  const int np = S / p, T = np * np, K = p * p * 3, run = p * 3;
  const int64_t total8 = (int64_t)n * T * K / 8;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total8; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = i * 8;
    const int64_t row = e / K;
    const int col = (int)(e - row * K);
    const int b = (int)(row / T), t = (int)(row - (int64_t)b * T);
    const int iy = t / np, ix = t - iy * np;
    const int py = col / run, rem = col - py * run;
    const float* src = crops + (((int64_t)b * S + iy * p + py) * S + (int64_t)ix * p) * 3 + rem;
    const float4 a = *reinterpret_cast<const float4*>(src);
    const float4 c = *reinterpret_cast<const float4*>(src + 4);
    uint4 u;
    u.x = tc::pack_bf16(a.x, a.y);
    u.y = tc::pack_bf16(a.z, a.w);
    u.z = tc::pack_bf16(c.x, c.y);
    u.w = tc::pack_bf16(c.z, c.w);
    *reinterpret_cast<uint4*>(out + e) = u;
  }
}

// ---------------------------------------------------------------------------
// LayerNorm (numkit.py:198-202, eps 1e-5): one warp per row, the row held in
// registers (D <= 2048, D % 128 == 0), two-pass mean / variance.
template <bool OUT_BF16, int MAXV>  // MAXV: float4 per lane (D / 128 when it is a power of two)
__global__ void k_layernorm(const float* __restrict__ x, int rows, int D, const float* __restrict__ g,
                            const float* __restrict__ b, void* __restrict__ out, int* nonfinite) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) / 32, lane = threadIdx.x % 32;
  if (warp >= rows) return;
  const int nv = D / 128;
  const float4* xr = reinterpret_cast<const float4*>(x + (size_t)warp * D);
  float4 v[MAXV];
  float s = 0.0f;
#pragma unroll
  for (int i = 0; i < MAXV; ++i)
    if (i < nv) {
      v[i] = __ldg(xr + i * 32 + lane);
      s += (v[i].x + v[i].y) + (v[i].z + v[i].w);
    }
  const float mean = warp_sum(s) / (float)D;
  float q = 0.0f;
#pragma unroll
  for (int i = 0; i < MAXV; ++i)
    if (i < nv) {
      v[i].x -= mean; v[i].y -= mean; v[i].z -= mean; v[i].w -= mean;
      q += (v[i].x * v[i].x + v[i].y * v[i].y) + (v[i].z * v[i].z + v[i].w * v[i].w);
    }
  const float rstd = 1.0f / sqrtf(warp_sum(q) / (float)D + 1e-5f);
  const float4* g4 = reinterpret_cast<const float4*>(g);
  const float4* b4 = reinterpret_cast<const float4*>(b);
#pragma unroll
  for (int i = 0; i < MAXV; ++i)
    if (i < nv) {
      const float4 gg = __ldg(g4 + i * 32 + lane), bb = __ldg(b4 + i * 32 + lane);
      float4 y;
      y.x = v[i].x * rstd * gg.x + bb.x;
      y.y = v[i].y * rstd * gg.y + bb.y;
      y.z = v[i].z * rstd * gg.z + bb.z;
      y.w = v[i].w * rstd * gg.w + bb.w;
      if (OUT_BF16) {
        uint2 u;
        u.x = tc::pack_bf16(y.x, y.y);
        u.y = tc::pack_bf16(y.z, y.w);
        reinterpret_cast<uint2*>(static_cast<__nv_bfloat16*>(out) + (size_t)warp * D)[i * 32 + lane] = u;
      } else {
        flag_nonfinite(nonfinite, y.x + y.y + y.z + y.w);
        reinterpret_cast<float4*>(static_cast<float*>(out) + (size_t)warp * D)[i * 32 + lane] = y;
      }
    }
}

// ---------------------------------------------------------------------------
// Flash attention on tcgen05 for head dim 64 (Decoder._attention,
// decoder.py:172-203: one crop's tokens attend to each other).
//
// CTA = one 128-query tile of one (crop, head); three CTAs share an SM
// (TMEM 128 columns and 72 KB of shared memory each).  5 warps:
//   warps 0-3  softmax, one query row per thread
//   warp 4     TMA (Q once; K chunks of 64 keys through a 2-deep ring, V
//              chunks through a 3-deep ring) and the tcgen05 issue, one
//              elected lane
// TMEM: S (128 x 64 fp32 scores) and O (128 x 64 fp32).
// The issue warp starts S(j+1) = Q K_{j+1}^T as soon as the softmax warps
// have copied S(j) into registers, so the tensor core works under the
// softmax of chunk j; P(j) = exp2(S c - m) is written as a bf16 tile to
// shared memory and O += P(j) V_j is issued when all four softmax warps
// have arrived.  The softmax warps only synchronise through mbarriers (no
// CTA-wide barrier per chunk).  The running max is rescaled lazily: O and l
// are corrected in TMEM only when the max grows by more than 2^8 (P stays
// <= 256; O / l is exact).  Keys past T are masked to -inf; query rows
// past T compute on the next crop's rows and are not stored.
#ifndef FSB_FA_PB
#define FSB_FA_PB 1  // P tiles in shared memory: 2 lets softmax(j) run under P(j-1).V (2 CTAs per SM)
#endif
constexpr int FA_THREADS = 160, FA_KC = 64, FA_KR = 2, FA_VR = 3, FA_PB = FSB_FA_PB;
constexpr uint32_t FA_Q = 0;                      // 16 KB
constexpr uint32_t FA_K = 16384;                  // FA_KR x 8 KB
constexpr uint32_t FA_V = FA_K + FA_KR * 8192;    // FA_VR x 8 KB
constexpr uint32_t FA_P = FA_V + FA_VR * 8192;    // FA_PB x 16 KB
constexpr uint32_t FA_SMEM = FA_P + FA_PB * 16384;
constexpr float FA_RESCALE = 8.0f;  // log2 units
static_assert(FA_PB == 1 || FA_PB == 2, "P buffers");

__global__ void __launch_bounds__(FA_THREADS, FA_PB == 1 ? 3 : 2)
    k_attn_tc(const __grid_constant__ CUtensorMap tmq, const __grid_constant__ CUtensorMap tmkv, int T, int D,
              float scale, __nv_bfloat16* __restrict__ ctx) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t q_full, k_full[FA_KR], v_full[FA_VR], s_full, s_free, p_full[FA_PB], o_full[2];
  __shared__ uint32_t tbase;
  const int qt = blockIdx.x, h = blockIdx.y, crop = blockIdx.z;
  const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
  const int row0 = crop * T;
  const int nch = (T + FA_KC - 1) / FA_KC;
  if (tid == 0) {
    tc::mbar_init(&q_full, 1);
    for (int i = 0; i < FA_KR; ++i) tc::mbar_init(&k_full[i], 1);
    for (int i = 0; i < FA_VR; ++i) tc::mbar_init(&v_full[i], 1);
    tc::mbar_init(&s_full, 1);
    tc::mbar_init(&s_free, 4);  // the four softmax warps copied S(j)
    for (int i = 0; i < FA_PB; ++i) tc::mbar_init(&p_full[i], 4);  // the four softmax warps wrote P(j)
    tc::mbar_init(&o_full[0], 1);  // P(j).V(j) done, j & 1 == b
    tc::mbar_init(&o_full[1], 1);
    tc::mbar_fence_init();
    tc::prefetch_tmap(&tmq);
    tc::prefetch_tmap(&tmkv);
  }
  if (warp == 0) tc::tmem_alloc(&tbase, 128);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  // TMEM columns: S at 0; O at 64
  const uint32_t sbase = tc::smem_u32(sm);
  const uint32_t tO = tbase + 64;

  if (warp == 4) {
    // TMA + MMA issue: the whole warp walks the schedule, lane 0 issues
    const bool leader = lane == 0;
    const uint32_t id_s = tc::idesc_bf16(128, FA_KC), id_o = tc::idesc_bf16_bmn(128, 64);
    auto load_k = [&](int j) {
      const int b = j % FA_KR;
      if (leader) {
        tc::mbar_expect_tx(&k_full[b], 8192u);
        tc::tma_load_2d(sm + FA_K + b * 8192, &tmkv, D + h * 64, row0 + j * FA_KC, &k_full[b]);
      }
      __syncwarp();
    };
    auto load_v = [&](int j) {
      const int b = j % FA_VR;
      if (leader) {
        tc::mbar_expect_tx(&v_full[b], 8192u);
        tc::tma_load_2d(sm + FA_V + b * 8192, &tmkv, 2 * D + h * 64, row0 + j * FA_KC, &v_full[b]);
      }
      __syncwarp();
    };
    auto issue_s = [&](int j) {
      tc::mbar_wait(&k_full[j % FA_KR], (uint32_t)((j / FA_KR) & 1));
      tc::fence_after();
      if (leader) {
        const uint32_t k = sbase + FA_K + (j % FA_KR) * 8192;
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          tc::mma_bf16(tbase, tc::sw128_kmajor_desc(sbase + FA_Q + 32 * kk), tc::sw128_kmajor_desc(k + 32 * kk), id_s,
                       kk > 0);
        tc::mma_commit(&s_full);
      }
      __syncwarp();
    };
    if (leader) {
      tc::mbar_expect_tx(&q_full, 16384u);
      tc::tma_load_2d(sm + FA_Q, &tmq, h * 64, row0 + qt * 128, &q_full);
    }
    __syncwarp();
    for (int j = 0; j < FA_KR && j < nch; ++j) load_k(j);
    for (int j = 0; j < FA_VR && j < nch; ++j) load_v(j);
    tc::mbar_wait(&q_full, 0);
    issue_s(0);
    for (int j = 0; j < nch; ++j) {
      if (j + 1 < nch) {
        // S(j+1) once the softmax warps hold S(j) in registers; S(j) has
        // completed, so its K slot takes chunk j+2
        tc::mbar_wait(&s_free, (uint32_t)(j & 1));
        tc::fence_after();
        issue_s(j + 1);
        if (j + 2 < nch) load_k(j + 2);
      }
      // O += P(j) V_j once the four softmax warps have written P(j)
      tc::mbar_wait(&p_full[j % FA_PB], (uint32_t)((j / FA_PB) & 1));
      tc::mbar_wait(&v_full[j % FA_VR], (uint32_t)((j / FA_VR) & 1));
      tc::fence_after();
      if (leader) {
        const uint32_t v = sbase + FA_V + (j % FA_VR) * 8192;
        const uint32_t pt = sbase + FA_P + (j % FA_PB) * 16384;
#pragma unroll
        for (int kk = 0; kk < FA_KC / 16; ++kk)
          tc::mma_bf16(tO, tc::kmajor_desc(pt, FA_KC, kk * 16), tc::sw128_mnmajor_desc(v + kk * 2048, 8192),
                       id_o, (j | kk) != 0);
        tc::mma_commit(&o_full[j & 1]);
      }
      __syncwarp();
      // V slot of chunk j-1 takes chunk j-1+VR once P(j-1).V(j-1) is done
      // (o_full phases are waited in order)
      if (j >= 1 && j - 1 + FA_VR < nch) {
        tc::mbar_wait(&o_full[(j - 1) & 1], (uint32_t)(((j - 1) >> 1) & 1));
        load_v(j - 1 + FA_VR);
      }
    }
  } else {
    // softmax: query row r = tid of the tile
    const uint32_t lane_off = (uint32_t)(warp * 32) << 16;
    uint8_t* prow0 = sm + FA_P + (tid >> 3) * (FA_KC * 16) + (tid & 7) * 16;
    const float c2 = scale * 1.4426950408889634f;
    float m = -INFINITY, l = 0.0f;
    for (int j = 0; j < nch; ++j) {
      tc::mbar_wait(&s_full, (uint32_t)(j & 1));
      tc::fence_after();
      float s[FA_KC];
      tc::tmem_ld64(tbase + lane_off, s);
      tc::fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&s_free);  // S may be overwritten by S(j+1)
      const int kvalid = T - j * FA_KC;
      if (kvalid < FA_KC) {
#pragma unroll
        for (int i = 0; i < FA_KC; ++i)
          if (i >= kvalid) s[i] = -INFINITY;
      }
      float m4[4] = {s[0], s[1], s[2], s[3]};
#pragma unroll
      for (int i = 4; i < FA_KC; ++i) m4[i & 3] = fmaxf(m4[i & 3], s[i]);
      const float mx = fmaxf(fmaxf(m4[0], m4[1]), fmaxf(m4[2], m4[3])) * c2;
      if (j >= FA_PB) {
        // P(j-PB).V(j-PB) done: P tile j % PB is free (PB = 1: O is stable too)
        tc::mbar_wait(&o_full[(j - FA_PB) & 1], (uint32_t)(((j - FA_PB) >> 1) & 1));
        tc::fence_after();
      }
      if (j == 0) {
        m = mx;
      } else {
        // lazy rescale: rows whose max grew by > 2^8 move to the new max.
        // TMEM accesses are warp-collective: the whole warp takes the branch
        // if any of its rows needs it (alpha = 1 elsewhere).
        const bool need = mx > m + FA_RESCALE;
        if (__any_sync(0xffffffffu, need)) {
          if (FA_PB == 2) {  // O must be stable: P(j-1).V(j-1) done
            tc::mbar_wait(&o_full[(j - 1) & 1], (uint32_t)(((j - 1) >> 1) & 1));
            tc::fence_after();
          }
          const float alpha = need ? ex2_approx(m - mx) : 1.0f;
#pragma unroll 1
          for (int c = 0; c < 64; c += 8) {
            float o[8];
            tc::tmem_ld8(tO + lane_off + c, o);
#pragma unroll
            for (int d = 0; d < 8; ++d) o[d] *= alpha;
            tc::tmem_st8(tO + lane_off + c, o);
          }
          l *= alpha;
          if (need) m = mx;
        }
      }
      const float nm = -m;
      uint8_t* prow = prow0 + (j % FA_PB) * 16384;
      float sum4[4] = {0.0f, 0.0f, 0.0f, 0.0f};
#pragma unroll
      for (int q = 0; q < FA_KC / 8; ++q) {
        uint32_t w[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const float p0 = ex2_approx(fmaf(s[8 * q + 2 * i], c2, nm));
          const float p1 = ex2_approx(fmaf(s[8 * q + 2 * i + 1], c2, nm));
          sum4[i] += p0 + p1;
          w[i] = tc::pack_bf16(p0, p1);
        }
        *reinterpret_cast<uint4*>(prow + q * 128) = make_uint4(w[0], w[1], w[2], w[3]);
      }
      l += (sum4[0] + sum4[1]) + (sum4[2] + sum4[3]);
      tc::fence_async_smem();  // P visible to the tensor core
      tc::fence_before();      // S(j) reads and the O rescale ordered before the arrive
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&p_full[j % FA_PB]);
    }
    tc::mbar_wait(&o_full[(nch - 1) & 1], (uint32_t)(((nch - 1) >> 1) & 1));
    tc::fence_after();
    const int qrow = qt * 128 + tid;
    const float inv = 1.0f / l;
#pragma unroll
    for (int half = 0; half < 2; ++half) {
      float o[32];
      tc::tmem_ld32(tO + lane_off + 32 * half, o);
      if (qrow < T) {
        uint4* dst = reinterpret_cast<uint4*>(ctx + (size_t)(row0 + qrow) * D + h * 64 + 32 * half);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const float* e = o + 8 * q;
          dst[q] = make_uint4(tc::pack_bf16(e[0] * inv, e[1] * inv), tc::pack_bf16(e[2] * inv, e[3] * inv),
                              tc::pack_bf16(e[4] * inv, e[5] * inv), tc::pack_bf16(e[6] * inv, e[7] * inv));
        }
      }
    }
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc(tbase, 128);
}

inline int ceil_div(int64_t a, int64_t b) { return (int)((a + b - 1) / b); }

template <bool OUT_BF16>
static void layernorm_launch(const float* x, int rows, int D, const float* g, const float* b, void* out,
                             int* nonfinite, cudaStream_t st) {
  const int blocks = ceil_div(rows, 8);
  switch (D / 128) {
    case 8: k_layernorm<OUT_BF16, 8><<<blocks, 256, 0, st>>>(x, rows, D, g, b, out, nonfinite); break;
    case 4: k_layernorm<OUT_BF16, 4><<<blocks, 256, 0, st>>>(x, rows, D, g, b, out, nonfinite); break;
    case 2: k_layernorm<OUT_BF16, 2><<<blocks, 256, 0, st>>>(x, rows, D, g, b, out, nonfinite); break;
    case 1: k_layernorm<OUT_BF16, 1><<<blocks, 256, 0, st>>>(x, rows, D, g, b, out, nonfinite); break;
    default: k_layernorm<OUT_BF16, 16><<<blocks, 256, 0, st>>>(x, rows, D, g, b, out, nonfinite); break;
  }
}

cudaError_t layernorm(const float* x, int rows, int D, const float* g, const float* b, void* out, bool bf16,
                      int* nonfinite, cudaStream_t st) {
  if (bf16)
    layernorm_launch<true>(x, rows, D, g, b, out, nonfinite, st);
  else
    layernorm_launch<false>(x, rows, D, g, b, out, nonfinite, st);
  return cudaGetLastError();
}

cudaError_t attention(const __nv_bfloat16* qkv, int crops, int T, int D, int H, __nv_bfloat16* ctx, cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(k_attn_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)FA_SMEM + 1024);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  CUtensorMap tmq, tmkv;
  if (!make_tmap_bf16(&tmq, qkv, (uint64_t)crops * T, 3 * (uint64_t)D, 3 * (uint64_t)D, 128) ||
      !make_tmap_bf16(&tmkv, qkv, (uint64_t)crops * T, 3 * (uint64_t)D, 3 * (uint64_t)D, FA_KC))
    return cudaErrorInvalidValue;
  dim3 grid(ceil_div(T, 128), H, crops);
  k_attn_tc<<<grid, FA_THREADS, FA_SMEM + 1024, st>>>(tmq, tmkv, T, D, 1.0f / sqrtf((float)(D / H)), ctx);
  return cudaGetLastError();
}

}  // namespace

size_t vit_ws_bytes(const VitW& w, int crops) {
  const size_t rows = (size_t)crops * w.T;
  const int K0 = w.p * w.p * 3;
  const size_t hcols = (size_t)(w.D > K0 ? w.D : K0);
  auto al = [](size_t b) { return (b + 1023) & ~size_t(1023); };
  return al(rows * w.D * 4) + al(rows * hcols * 2) + al(rows * 3 * w.D * 2) + al(rows * 4 * w.D * 2);
}

void vit_ws_carve(const VitW& w, int crops, void* base, VitWs* ws) {
  const size_t rows = (size_t)crops * w.T;
  const int K0 = w.p * w.p * 3;
  const size_t hcols = (size_t)(w.D > K0 ? w.D : K0);
  auto al = [](size_t b) { return (b + 1023) & ~size_t(1023); };
  uint8_t* p = static_cast<uint8_t*>(base);
  ws->max_crops = crops;
  ws->x = reinterpret_cast<float*>(p);
  p += al(rows * w.D * 4);
  ws->h = reinterpret_cast<__nv_bfloat16*>(p);
  p += al(rows * hcols * 2);
  ws->qkv = reinterpret_cast<__nv_bfloat16*>(p);
  p += al(rows * 3 * w.D * 2);
  ws->hid = reinterpret_cast<__nv_bfloat16*>(p);
}

cudaError_t launch_vit_encoder(const VitW& w, const VitWs& ws, const float* crops, int n, float* feats, int* nonfinite,
                               cudaStream_t st, int* launches) {
  const int D = w.D, T = w.T, K0 = w.p * w.p * 3;
  if (D % 128 || D > 2048 || D / w.H != 64 || K0 % 64) return cudaErrorInvalidValue;
  int nl = 0;
#define VIT_CHECK(expr)                  \
  do {                                   \
    cudaError_t e_ = (expr);             \
    if (e_ != cudaSuccess) return e_;    \
    ++nl;                                \
  } while (0)
  for (int c0 = 0; c0 < n; c0 += ws.max_crops) {
    const int nc = (n - c0 < ws.max_crops) ? n - c0 : ws.max_crops;
    const int M = nc * T;
    const float* cr = crops + (size_t)c0 * w.S * w.S * 3;
    float* out = feats + (size_t)c0 * T * D;
    const int64_t tot8 = (int64_t)M * K0 / 8;
    k_patchify<<<ceil_div(tot8, 256) < 148 * 16 ? ceil_div(tot8, 256) : 148 * 16, 256, 0, st>>>(cr, nc, w.S, w.p,
                                                                                                 ws.h);
    VIT_CHECK(cudaGetLastError());
    VIT_CHECK(launch_gemm_tc(ws.h, K0, w.wpatch, K0, M, D, K0,
                             GemmEpi{w.patch_b, nullptr, ws.x, w.pos, D, T, EPI_EMBED_F32}, st));
    for (const VitLayer& L : w.layers) {
      VIT_CHECK(layernorm(ws.x, M, D, L.ln1_g, L.ln1_b, ws.h, true, nullptr, st));
      VIT_CHECK(launch_gemm_tc(ws.h, D, L.wqkv, D, M, 3 * D, D,
                               GemmEpi{L.bqkv, ws.qkv, nullptr, nullptr, 3 * D, T, EPI_BIAS_BF16}, st));
      VIT_CHECK(attention(ws.qkv, nc, T, D, w.H, ws.h, st));
      VIT_CHECK(launch_gemm_tc(ws.h, D, L.wo, D, M, D, D, GemmEpi{L.bo, nullptr, ws.x, nullptr, D, T, EPI_RESID_F32},
                               st));
      VIT_CHECK(layernorm(ws.x, M, D, L.ln2_g, L.ln2_b, ws.h, true, nullptr, st));
      VIT_CHECK(launch_gemm_tc(ws.h, D, L.w1, D, M, 4 * D, D,
                               GemmEpi{L.b1, ws.hid, nullptr, nullptr, 4 * D, T, EPI_RELU_BF16}, st));
      VIT_CHECK(launch_gemm_tc(ws.hid, 4 * D, L.w2, 4 * D, M, D, 4 * D,
                               GemmEpi{L.b2, nullptr, ws.x, nullptr, D, T, EPI_RESID_F32}, st));
    }
    VIT_CHECK(layernorm(ws.x, M, D, w.norm_g, w.norm_b, out, false, nonfinite, st));
  }
#undef VIT_CHECK
  if (launches) *launches += nl;
  return cudaSuccess;
}

// debug / test entry (tests/test_gpu_vit.py): attention alone on a packed
// (crops*T, 3D) bf16 q|k|v matrix -> (crops*T, D) bf16 context
extern "C" int fsb_debug_attention(const void* qkv, int crops, int T, int D, int H, void* ctx, void* stream) {
  cudaError_t r = attention(static_cast<const __nv_bfloat16*>(qkv), crops, T, D, H, static_cast<__nv_bfloat16*>(ctx),
                            (cudaStream_t)stream);
  if (r != cudaSuccess) fprintf(stderr, "fsb_debug_attention: %s\n", cudaGetErrorString(r));
  return r == cudaSuccess ? 0 : 4;
}
