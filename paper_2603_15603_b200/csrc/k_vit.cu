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
template <bool OUT_BF16>
__global__ void k_layernorm(const float* __restrict__ x, int rows, int D, const float* __restrict__ g,
                            const float* __restrict__ b, void* __restrict__ out, int* nonfinite) {
  constexpr int MAXV = 16;  // float4 per lane
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
// decoder.py:172-203, one crop's tokens attend to each other).
//
// CTA = (128-query tile, head, crop), 128 threads, one query row per thread.
// Thread 0 drives TMA and the tensor core; everyone does the softmax.
//   S  = Q K^T      Q, K: TMA SW128 K-major boxes of the qkv matrix   TMEM [0,128)
//   P  = exp2(S*c - m) -> bf16, written to smem (no-swizzle K-major)
//   O' = P V        V: the same TMA box read MN-major                  TMEM [128,192)
//   O  = O * alpha + O'  in registers (online softmax), / l at the end.
// K chunks of 128 keys are double-buffered (the TMA of chunk j+1 runs under
// the MMAs and softmax of chunk j); V is single-buffered and refilled as soon
// as the P.V MMA of chunk j has consumed it (96 KB smem: two CTAs per SM).
// Keys past T are masked to -inf; query rows past T compute on the next
// crop's rows and are not stored.
constexpr int AT_THREADS = 128;
constexpr uint32_t AT_Q = 0, AT_K = 16384, AT_V = 49152, AT_P = 65536, AT_SMEM = 65536 + 32768;

__global__ void __launch_bounds__(AT_THREADS, 2)
    k_attn_tc(const __grid_constant__ CUtensorMap tm, int T, int D, float scale, __nv_bfloat16* __restrict__ ctx) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar_ld[2], bar_v, bar_s, bar_o;
  __shared__ uint32_t tbase;
  const int qt = blockIdx.x, h = blockIdx.y, crop = blockIdx.z;
  const int tid = threadIdx.x, warp = tid / 32;
  const int row0 = crop * T;
  const int nch = (T + 127) / 128;
  if (tid == 0) {
    tc::mbar_init(&bar_ld[0], 1);
    tc::mbar_init(&bar_ld[1], 1);
    tc::mbar_init(&bar_v, 1);
    tc::mbar_init(&bar_s, 1);
    tc::mbar_init(&bar_o, 1);
    tc::mbar_fence_init();
    tc::prefetch_tmap(&tm);
  }
  if (warp == 0) tc::tmem_alloc(&tbase, 256);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tS = tbase, tO = tbase + 128;
  const uint32_t lane_off = (uint32_t)(warp * 32) << 16;
  const uint32_t sbase = tc::smem_u32(sm);
  if (tid == 0) {
    tc::mbar_expect_tx(&bar_ld[0], 2 * 16384);
    tc::tma_load_2d(sm + AT_Q, &tm, h * 64, row0 + qt * 128, &bar_ld[0]);
    tc::tma_load_2d(sm + AT_K, &tm, D + h * 64, row0, &bar_ld[0]);
    tc::mbar_expect_tx(&bar_v, 16384);
    tc::tma_load_2d(sm + AT_V, &tm, 2 * D + h * 64, row0, &bar_v);
  }
  float o[64];
#pragma unroll
  for (int d = 0; d < 64; ++d) o[d] = 0.0f;
  float m = -1e30f, l = 0.0f;
  const float c2 = scale * 1.4426950408889634f;
  uint8_t* prow = sm + AT_P + (tid >> 3) * 2048 + (tid & 7) * 16;

  for (int j = 0; j < nch; ++j) {
    const int b = j & 1;
    if (tid == 0) {
      if (j + 1 < nch) {
        tc::mbar_expect_tx(&bar_ld[b ^ 1], 16384);
        tc::tma_load_2d(sm + AT_K + (b ^ 1) * 16384, &tm, D + h * 64, row0 + (j + 1) * 128, &bar_ld[b ^ 1]);
      }
      tc::mbar_wait(&bar_ld[b], (uint32_t)((j >> 1) & 1));
      tc::fence_after();
      const uint32_t q = sbase + AT_Q, k = sbase + AT_K + b * 16384;
      const uint32_t id = tc::idesc_bf16(128, 128);
#pragma unroll
      for (int kk = 0; kk < 4; ++kk)
        tc::mma_bf16(tS, tc::sw128_kmajor_desc(q + 32 * kk), tc::sw128_kmajor_desc(k + 32 * kk), id, kk > 0);
      tc::mma_commit(&bar_s);
    }
    tc::mbar_wait(&bar_s, (uint32_t)(j & 1));
    tc::fence_after();
    float s[128];
    tc::tmem_ld64(tS + lane_off, s);
    tc::tmem_ld64(tS + lane_off + 64, s + 64);
    const int kvalid = T - j * 128;
    float mx = m;
#pragma unroll
    for (int i = 0; i < 128; ++i) {
      s[i] = (i < kvalid) ? s[i] * c2 : -INFINITY;
      mx = fmaxf(mx, s[i]);
    }
    const float alpha = ex2_approx(m - mx);
    m = mx;
    float sum = 0.0f;
#pragma unroll
    for (int g = 0; g < 16; ++g) {
      uint32_t w[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        __nv_bfloat162 pb = __floats2bfloat162_rn(ex2_approx(s[8 * g + 2 * i] - mx), ex2_approx(s[8 * g + 2 * i + 1] - mx));
        const float2 pf = __bfloat1622float2(pb);
        sum += pf.x + pf.y;
        w[i] = *reinterpret_cast<uint32_t*>(&pb);
      }
      *reinterpret_cast<uint4*>(prow + g * 128) = make_uint4(w[0], w[1], w[2], w[3]);
    }
    l = l * alpha + sum;
    tc::fence_async_smem();
    tc::fence_before();
    __syncthreads();
    if (tid == 0) {
      tc::mbar_wait(&bar_v, (uint32_t)(j & 1));
      tc::fence_after();
      const uint32_t p = sbase + AT_P, v = sbase + AT_V;
      const uint32_t id = tc::idesc_bf16_bmn(128, 64);
#pragma unroll
      for (int kk = 0; kk < 8; ++kk)
        tc::mma_bf16(tO, tc::kmajor_desc(p, 128, kk * 16), tc::sw128_mnmajor_desc(v + kk * 2048, 8192), id, kk > 0);
      tc::mma_commit(&bar_o);
    }
    tc::mbar_wait(&bar_o, (uint32_t)(j & 1));
    tc::fence_after();
    if (tid == 0 && j + 1 < nch) {  // V of chunk j has been consumed
      tc::mbar_expect_tx(&bar_v, 16384);
      tc::tma_load_2d(sm + AT_V, &tm, 2 * D + h * 64, row0 + (j + 1) * 128, &bar_v);
    }
    float pv[64];
    tc::tmem_ld64(tO + lane_off, pv);
#pragma unroll
    for (int d = 0; d < 64; ++d) o[d] = fmaf(o[d], alpha, pv[d]);
  }
  const int qrow = qt * 128 + tid;
  if (qrow < T) {
    const float inv = 1.0f / l;
    uint4* dst = reinterpret_cast<uint4*>(ctx + (size_t)(row0 + qrow) * D + h * 64);
#pragma unroll
    for (int g = 0; g < 8; ++g) {
      const float* e = o + 8 * g;
      dst[g] = make_uint4(tc::pack_bf16(e[0] * inv, e[1] * inv), tc::pack_bf16(e[2] * inv, e[3] * inv),
                          tc::pack_bf16(e[4] * inv, e[5] * inv), tc::pack_bf16(e[6] * inv, e[7] * inv));
    }
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc(tbase, 256);
}

inline int ceil_div(int64_t a, int64_t b) { return (int)((a + b - 1) / b); }

cudaError_t layernorm(const float* x, int rows, int D, const float* g, const float* b, void* out, bool bf16,
                      int* nonfinite, cudaStream_t st) {
  const int blocks = ceil_div(rows, 8);
  if (bf16)
    k_layernorm<true><<<blocks, 256, 0, st>>>(x, rows, D, g, b, out, nonfinite);
  else
    k_layernorm<false><<<blocks, 256, 0, st>>>(x, rows, D, g, b, out, nonfinite);
  return cudaGetLastError();
}

cudaError_t attention(const __nv_bfloat16* qkv, int crops, int T, int D, int H, __nv_bfloat16* ctx, cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(k_attn_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)AT_SMEM + 1024);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  CUtensorMap tm;
  if (!make_tmap_bf16(&tm, qkv, (uint64_t)crops * T, 3 * (uint64_t)D, 3 * (uint64_t)D, 128))
    return cudaErrorInvalidValue;
  dim3 grid(ceil_div(T, 128), H, crops);
  k_attn_tc<<<grid, AT_THREADS, AT_SMEM + 1024, st>>>(tm, T, D, 1.0f / sqrtf((float)(D / H)), ctx);
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
