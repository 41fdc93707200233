// Reference-precision (fp32) encoder for ANY DecoderConfig (decoder.py:
// encode :231-260, _attention :172-203, _mlp :205-212, numkit.layer_norm
// :198-202) as a layer-by-layer pipeline of CUDA-core kernels: patchify ->
// patch GEMM (+ bias, + position) -> per layer [LayerNorm -> QKV GEMM ->
// attention -> Wo GEMM (+ residual) -> LayerNorm -> W1 GEMM (ReLU) -> W2 GEMM
// (+ residual)] -> final LayerNorm.
//
// This is the parity mode of the large configurations (the ViT-L-sized C4
// encoder at fp32, SURVEY §8(d) "run fp32 as well for parity"): every
// multiply-add is an fp32 FMA with fp32 accumulation, the reference's own
// arithmetic type, so it tracks the reference to ~1e-6 relative per layer.
// The tensor-core path (k_vit.cu, bf16 operands) is the throughput mode.
// The default config's fp32 encoder is the fused k_encoder_f32.
#include "fsb_common.cuh"
#include "fsb_enc_f32.h"

namespace {

inline int cdiv(int64_t a, int64_t b) { return (int)((a + b - 1) / b); }

// (n, S, S, 3) crops -> (n * np * np, p * p * 3) patch rows, in-patch order
// (py, px, c) and row-major patch order (decoder.py:247-248)
__global__ void k_patchify_f32(const float* __restrict__ crops, int n, int S, int p, float* __restrict__ P) {
  const int np = S / p, K0 = p * p * 3;
  const int64_t tot = (int64_t)n * np * np * K0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < tot; i += (int64_t)gridDim.x * blockDim.x) {
    const int k = (int)(i % K0);
    const int64_t row = i / K0;
    const int b = (int)(row / (np * np)), pi = (int)(row % (np * np));
    const int py = pi / np, px = pi % np;
    const int iy = k / (p * 3), ix = (k / 3) % p, c = k % 3;
    P[i] = crops[(((int64_t)b * S + py * p + iy) * S + px * p + ix) * 3 + c];
  }
}

// x[row, :] += pos[row % T, :]
__global__ void k_add_pos(float* __restrict__ x, const float* __restrict__ pos, int64_t rows, int T, int D) {
  const int64_t tot = rows * D;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < tot; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / D;
    x[i] += pos[(r % T) * D + i % D];
  }
}

// LayerNorm of any width, one warp per row: mean, then the mean of squared
// deviations (two passes, as numkit.layer_norm), eps 1e-5, affine
__global__ void k_layernorm_f32(const float* __restrict__ x, int64_t rows, int D, const float* __restrict__ g,
                                const float* __restrict__ b, float* __restrict__ out, int* nonfinite) {
  const int64_t row = (int64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  if (row >= rows) return;
  const float* xr = x + row * D;
  float s = 0.0f;
  for (int c = lane; c < D; c += 32) s += xr[c];
#pragma unroll
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  const float mu = s / (float)D;
  float q = 0.0f;
  for (int c = lane; c < D; c += 32) {
    const float d = xr[c] - mu;
    q = fmaf(d, d, q);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) q += __shfl_xor_sync(0xffffffffu, q, o);
  const float rs = 1.0f / sqrtf(q / (float)D + 1e-5f);
  float* orow = out + row * D;
  for (int c = lane; c < D; c += 32) {
    const float v = (xr[c] - mu) * rs * g[c] + b[c];
    flag_nonfinite(nonfinite, v);
    orow[c] = v;
  }
}

// Attention of one (crop, head) per blockIdx.(y, z), one query row per
// thread (blockIdx.x tiles the queries).  Keys / values are staged 32 at a
// time in shared memory; scores of a key block first, then one rescale of
// the running output (online softmax).  logits = (q . k) * f32(1/sqrt(dh))
// (decoder.py:190-196).  qkv rows: [q | k | v] (3D), ctx rows: D.
constexpr int kAtQ = 64;   // queries per CTA
constexpr int kAtKB = 32;  // keys per shared-memory block
template <int DH>
__global__ void __launch_bounds__(kAtQ) k_attn_f32(const float* __restrict__ qkv, int T, int D, float scale,
                                                   float* __restrict__ ctx) {
  __shared__ float Ks[kAtKB][DH + 1], Vs[kAtKB][DH];
  const int crop = blockIdx.z, h = blockIdx.y;
  const int qi = blockIdx.x * kAtQ + threadIdx.x;
  const int64_t base = (int64_t)crop * T;
  float q[DH], o[DH];
  const bool live = qi < T;
#pragma unroll
  for (int d = 0; d < DH; ++d) {
    q[d] = live ? qkv[(base + qi) * 3 * D + h * DH + d] : 0.0f;
    o[d] = 0.0f;
  }
  float m = -INFINITY, l = 0.0f;
  for (int k0 = 0; k0 < T; k0 += kAtKB) {
    const int nk = min(kAtKB, T - k0);
    __syncthreads();
    for (int i = threadIdx.x; i < kAtKB * DH; i += kAtQ) {
      const int r = i / DH, d = i % DH;
      const bool ok = r < nk;
      Ks[r][d] = ok ? qkv[(base + k0 + r) * 3 * D + D + h * DH + d] : 0.0f;
      Vs[r][d] = ok ? qkv[(base + k0 + r) * 3 * D + 2 * D + h * DH + d] : 0.0f;
    }
    __syncthreads();
    float s[kAtKB];
    float mb = -INFINITY;
#pragma unroll
    for (int r = 0; r < kAtKB; ++r) {
      float acc = 0.0f;
#pragma unroll
      for (int d = 0; d < DH; ++d) acc = fmaf(q[d], Ks[r][d], acc);
      s[r] = r < nk ? acc * scale : -INFINITY;
      mb = fmaxf(mb, s[r]);
    }
    const float mn = fmaxf(m, mb);
    const float corr = expf(m - mn);  // 0 on the first block (m = -inf)
    l *= corr;
#pragma unroll
    for (int d = 0; d < DH; ++d) o[d] *= corr;
#pragma unroll
    for (int r = 0; r < kAtKB; ++r) {
      const float pr = r < nk ? expf(s[r] - mn) : 0.0f;
      l += pr;
#pragma unroll
      for (int d = 0; d < DH; ++d) o[d] = fmaf(pr, Vs[r][d], o[d]);
    }
    m = mn;
  }
  if (!live) return;
  const float inv = 1.0f / l;
  float* out = ctx + (base + qi) * D + h * DH;
#pragma unroll
  for (int d = 0; d < DH; ++d) out[d] = o[d] * inv;
}

template <int DH>
cudaError_t attn_launch(const float* qkv, int crops, int T, int D, int H, float* ctx, cudaStream_t st) {
  dim3 grid(cdiv(T, kAtQ), H, crops);
  k_attn_f32<DH><<<grid, kAtQ, 0, st>>>(qkv, T, D, 1.0f / sqrtf((float)DH), ctx);
  return cudaGetLastError();
}

cudaError_t attention_f32(const float* qkv, int crops, int T, int D, int H, float* ctx, cudaStream_t st) {
  switch (D / H) {
    case 16: return attn_launch<16>(qkv, crops, T, D, H, ctx, st);
    case 32: return attn_launch<32>(qkv, crops, T, D, H, ctx, st);
    case 64: return attn_launch<64>(qkv, crops, T, D, H, ctx, st);
    case 128: return attn_launch<128>(qkv, crops, T, D, H, ctx, st);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t layernorm_f32(const float* x, int64_t rows, int D, const float* g, const float* b, float* out,
                          int* nonfinite, cudaStream_t st) {
  k_layernorm_f32<<<cdiv(rows, 8), 256, 0, st>>>(x, rows, D, g, b, out, nonfinite);
  return cudaGetLastError();
}

}  // namespace

bool enc_f32_supported(int D, int H) {
  const int dh = H > 0 && D % H == 0 ? D / H : 0;
  return dh == 16 || dh == 32 || dh == 64 || dh == 128;
}

size_t enc_f32_ws_bytes(const EncF32W& w, int crops) {
  const size_t rows = (size_t)crops * w.T;
  const int K0 = w.p * w.p * 3;
  auto al = [](size_t b) { return (b + 1023) & ~size_t(1023); };
  return al(rows * w.D * 4) + al(rows * (size_t)(w.D > K0 ? w.D : K0) * 4) + al(rows * 3 * w.D * 4) +
         al(rows * 4 * w.D * 4);
}

void enc_f32_ws_carve(const EncF32W& w, int crops, void* base, EncF32Ws* ws) {
  const size_t rows = (size_t)crops * w.T;
  const int K0 = w.p * w.p * 3;
  auto al = [](size_t b) { return (b + 1023) & ~size_t(1023); };
  uint8_t* p = static_cast<uint8_t*>(base);
  ws->max_crops = crops;
  ws->x = reinterpret_cast<float*>(p);
  p += al(rows * w.D * 4);
  ws->h = reinterpret_cast<float*>(p);
  p += al(rows * (size_t)(w.D > K0 ? w.D : K0) * 4);
  ws->qkv = reinterpret_cast<float*>(p);
  p += al(rows * 3 * w.D * 4);
  ws->hid = reinterpret_cast<float*>(p);
}

cudaError_t launch_enc_f32(const EncF32W& w, const EncF32Ws& ws, const float* crops, int n, float* feats,
                           int* nonfinite, cudaStream_t st, int* launches) {
  const int D = w.D, T = w.T, K0 = w.p * w.p * 3;
  if (!enc_f32_supported(D, w.H)) return cudaErrorInvalidValue;
  int nl = 0;
#define ENC_CHECK(expr)               \
  do {                                \
    cudaError_t e_ = (expr);          \
    if (e_ != cudaSuccess) return e_; \
    ++nl;                             \
  } while (0)
  for (int c0 = 0; c0 < n; c0 += ws.max_crops) {
    const int nc = (n - c0 < ws.max_crops) ? n - c0 : ws.max_crops;
    const int M = nc * T;
    const float* cr = crops + (size_t)c0 * w.S * w.S * 3;
    float* out = feats + (size_t)c0 * T * D;
    const int64_t tot = (int64_t)M * K0;
    k_patchify_f32<<<cdiv(tot, 256) < 148 * 32 ? cdiv(tot, 256) : 148 * 32, 256, 0, st>>>(cr, nc, w.S, w.p, ws.h);
    ENC_CHECK(cudaGetLastError());
    ENC_CHECK(launch_gemm_f32_acc(ws.h, K0, w.wpatch, w.patch_b, ws.x, D, M, D, K0, 0, 0, st));
    k_add_pos<<<cdiv((int64_t)M * D, 256) < 148 * 32 ? cdiv((int64_t)M * D, 256) : 148 * 32, 256, 0, st>>>(
        ws.x, w.pos, M, T, D);
    ENC_CHECK(cudaGetLastError());
    for (const EncF32Layer& L : w.layers) {
      ENC_CHECK(layernorm_f32(ws.x, M, D, L.ln1_g, L.ln1_b, ws.h, nullptr, st));
      ENC_CHECK(launch_gemm_f32_acc(ws.h, D, L.wqkv, L.bqkv, ws.qkv, 3 * D, M, 3 * D, D, 0, 0, st));
      ENC_CHECK(attention_f32(ws.qkv, nc, T, D, w.H, ws.h, st));
      ENC_CHECK(launch_gemm_f32_acc(ws.h, D, L.wo, L.bo, ws.x, D, M, D, D, 0, 1, st));  // x += ctx Wo + bo
      ENC_CHECK(layernorm_f32(ws.x, M, D, L.ln2_g, L.ln2_b, ws.h, nullptr, st));
      ENC_CHECK(launch_gemm_f32_acc(ws.h, D, L.w1, L.b1, ws.hid, 4 * D, M, 4 * D, D, 1, 0, st));
      ENC_CHECK(launch_gemm_f32_acc(ws.hid, 4 * D, L.w2, L.b2, ws.x, D, M, D, 4 * D, 0, 1, st));  // x += mlp
    }
    ENC_CHECK(layernorm_f32(ws.x, M, D, w.norm_g, w.norm_b, out, nonfinite, st));
  }
#undef ENC_CHECK
  if (launches) *launches += nl;
  return cudaSuccess;
}
