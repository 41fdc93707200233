// K2 (encoder) and K3 (body + hand decoders), fp32 mode, default model size
// (D = 64, 4 heads of 16, MLP 4D, 8x8 patches of a 64x64 crop).
//
// Reference: Decoder.encode (decoder.py:231-260), _attention (:172-203),
// _mlp (:205-212), _self_block/_cross_block (:214-227), _heads (:264-272),
// predict_kp2d (:274-282), _body_pass/decode_body (:284-356), decode_hand
// (:360-410), merge (:414-422).
//
// Design: one CTA owns one crop (encoder), one frame's body decode, or one
// hand decode, and keeps the whole residual stream, every intermediate and
// the current layer's weights in shared memory for the full depth of the
// network: HBM is touched once for the inputs, once for the outputs, and the
// ~0.8 M parameters stream from L2.  Inside a CTA every GEMM is a 4x4
// register-blocked FFMA tile over a transposed activation panel; LayerNorm
// and softmax are warp-shuffle row reductions; the body decoder's
// intermediate prediction (heads -> forward kinematics -> keypoint
// re-embedding) runs in-kernel on one warp, so the serial FK feedback of
// layers 0-2 costs no launches.  Rows of a batch never interact, so a frame
// decoded in a batch of 32 is bit-identical to the same frame decoded alone.
#include "fsb_common.cuh"
#include "fsb_weights.h"

namespace {

constexpr int D = 64;
constexpr int DH = 16;
constexpr int NT = 256;  // threads per CTA
constexpr int LDQKV = 3 * D + 4;   // row stride of the fused q|k|v panel
constexpr int LDKV = 2 * D + 4;    // row stride of the cross k|v panel
constexpr int WSTAGE = 256 * 64;   // floats of the weight staging buffer

// ---------------------------------------------------------------------------
// building blocks

// copy n floats (multiple of 4, 16-byte aligned) global -> shared
__device__ __forceinline__ void stage(float* __restrict__ dst, const float* __restrict__ src, int n) {
  const float4* s4 = reinterpret_cast<const float4*>(src);
  float4* d4 = reinterpret_cast<float4*>(dst);
  for (int i = threadIdx.x; i < n / 4; i += NT) d4[i] = __ldg(s4 + i);
}

// C(R x N) = A(R x K) @ W(K x N) with A given transposed (At[k * LDA + r])
// and W staged in shared memory (row-major, stride N).  Every output is one
// thread's sequential sum over k, so results do not depend on R or on which
// rows share the CTA.  epi(r, c, v) consumes each output.
template <int R, int K, int N, int LDA, class Epi>
__device__ __forceinline__ void gemm_tile(const float* __restrict__ At, const float* __restrict__ W, Epi epi) {
  constexpr int RG = R / 4, CG = N / 4, MT = RG * CG, PT = (MT + NT - 1) / NT;
  float acc[PT][4][4];
#pragma unroll
  for (int p = 0; p < PT; ++p)
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[p][i][j] = 0.0f;
  const int tid = threadIdx.x;
#pragma unroll 4
  for (int k = 0; k < K; ++k) {
#pragma unroll
    for (int p = 0; p < PT; ++p) {
      const int m = tid + p * NT;
      if (MT % NT == 0 || m < MT) {
        const int mr = m % RG, mc = m / RG;
        const float4 a = *reinterpret_cast<const float4*>(At + k * LDA + mr * 4);
        const float4 w = *reinterpret_cast<const float4*>(W + k * N + mc * 4);
        const float av[4] = {a.x, a.y, a.z, a.w};
        const float wv[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[p][i][j] = fmaf(av[i], wv[j], acc[p][i][j]);
      }
    }
  }
#pragma unroll
  for (int p = 0; p < PT; ++p) {
    const int m = tid + p * NT;
    if (MT % NT == 0 || m < MT) {
      const int mr = m % RG, mc = m / RG;
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) epi(mr * 4 + i, mc * 4 + j, acc[p][i][j]);
    }
  }
}

// epilogues --------------------------------------------------------------
struct EpiRow {  // dst[r * ld + c] = v + b[c]
  float* dst; int ld; const float* b;
  __device__ void operator()(int r, int c, float v) const { dst[r * ld + c] = v + __ldg(b + c); }
};
struct EpiT {  // dst[c * ld + r] = act(v + b[c])  (transposed panel for the next GEMM)
  float* dst; int ld; const float* b; bool relu;
  __device__ void operator()(int r, int c, float v) const {
    float y = v + __ldg(b + c);
    if (relu) y = fmaxf(y, 0.0f);
    dst[c * ld + r] = y;
  }
};
struct EpiAdd {  // x[r * ld + c] += v + b[c] for valid rows (residual update)
  float* x; int ld; const float* b; int nvalid;
  __device__ void operator()(int r, int c, float v) const {
    if (r < nvalid) x[r * ld + c] += v + __ldg(b + c);
  }
};

// LayerNorm (numkit.py:198-202) of rows [0, R) of a row-major panel, with an
// optional additive row term, written transposed into At (stride LDA).
// Rows >= nvalid are written as zeros.  TPR threads cooperate on a row.
struct NoPos {
  __device__ float operator()(int, int) const { return 0.0f; }
};
struct BodyPos {  // decoder.py:301-303: p2d on rows 5..26, p3d on rows 27..48
  const float* p2d; const float* p3d;
  __device__ float operator()(int r, int c) const {
    if (r >= 5 && r < 27) return p2d[(r - 5) * D + c];
    if (r >= 27 && r < 49) return p3d[(r - 27) * D + c];
    return 0.0f;
  }
};
struct HandPos {  // decoder.py:398: p_pts on rows 1..3
  const float* pts;
  __device__ float operator()(int r, int c) const { return (r >= 1 && r < 4) ? pts[(r - 1) * D + c] : 0.0f; }
};

template <int R, class Pos>
__device__ __forceinline__ void layer_norm_T(const float* __restrict__ X, int ldx, int nvalid, const float* g,
                                             const float* b, float* __restrict__ At, int LDA, Pos pos) {
  constexpr int TPR = NT / R;       // threads per row (4 for R = 64, 16 for R = 16)
  constexpr int CPT = D / TPR;      // columns per thread
  const int r = threadIdx.x / TPR, part = threadIdx.x % TPR;
  float v[CPT];
  float s = 0.0f;
#pragma unroll
  for (int i = 0; i < CPT; ++i) {
    const int c = part + i * TPR;
    v[i] = (r < nvalid) ? X[r * ldx + c] + pos(r, c) : 0.0f;
    s += v[i];
  }
#pragma unroll
  for (int o = TPR / 2; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  const float mu = s * (1.0f / D);
  float q = 0.0f;
#pragma unroll
  for (int i = 0; i < CPT; ++i) {
    v[i] -= mu;
    q += v[i] * v[i];
  }
#pragma unroll
  for (int o = TPR / 2; o > 0; o >>= 1) q += __shfl_xor_sync(0xffffffffu, q, o);
  const float sd = sqrtf(q * (1.0f / D) + 1e-5f);
#pragma unroll
  for (int i = 0; i < CPT; ++i) {
    const int c = part + i * TPR;
    At[c * LDA + r] = (r < nvalid) ? v[i] / sd * __ldg(g + c) + __ldg(b + c) : 0.0f;
  }
}

// LayerNorm of one row held in shared memory, by one warp (heads input)
__device__ __forceinline__ void layer_norm_row_warp(const float* x, const float* g, const float* b, float* out,
                                                    int lane) {
  float v0 = x[lane], v1 = x[lane + 32];
  const float mu = warp_sum(v0 + v1) * (1.0f / D);
  v0 -= mu;
  v1 -= mu;
  const float sd = sqrtf(warp_sum(v0 * v0 + v1 * v1) * (1.0f / D) + 1e-5f);
  out[lane] = v0 / sd * __ldg(g + lane) + __ldg(b + lane);
  out[lane + 32] = v1 / sd * __ldg(g + lane + 32) + __ldg(b + lane + 32);
}

// per-(head, query row) attention core (decoder.py:189-200): thread t serves
// head t / 64, query row t % 64.  Q, K, V row-major with the given strides;
// context written transposed into ctxT (stride LDA) for the output GEMM.
// Query q_base / key k_base offsets select a per-hand sub-panel.
__device__ __forceinline__ void attention_core(const float* __restrict__ Q, int ldq, const float* __restrict__ Kp,
                                               const float* __restrict__ Vp, int ldk, int nq, int nk,
                                               float* __restrict__ ctxT, int LDA) {
  const int h = threadIdx.x / 64, r = threadIdx.x % 64;
  if (r >= nq) return;
  float q[DH];
#pragma unroll
  for (int d = 0; d < DH; ++d) q[d] = Q[r * ldq + h * DH + d];
  float s[64];
  float mx = -INFINITY;
#pragma unroll
  for (int j = 0; j < 64; ++j) {
    if (j < nk) {
      const float* kr = Kp + j * ldk + h * DH;
      float acc = 0.0f;
#pragma unroll
      for (int d = 0; d < DH; ++d) acc = fmaf(q[d], kr[d], acc);
      s[j] = acc * 0.25f;  // f32(1/sqrt(16))
      mx = fmaxf(mx, s[j]);
    }
  }
  float sum = 0.0f;
#pragma unroll
  for (int j = 0; j < 64; ++j) {
    if (j < nk) {
      s[j] = expf(s[j] - mx);
      sum += s[j];
    }
  }
  float ctx[DH];
#pragma unroll
  for (int d = 0; d < DH; ++d) ctx[d] = 0.0f;
#pragma unroll
  for (int j = 0; j < 64; ++j) {
    if (j < nk) {
      const float pj = s[j] / sum;
      const float* vr = Vp + j * ldk + h * DH;
#pragma unroll
      for (int d = 0; d < DH; ++d) ctx[d] = fmaf(pj, vr[d], ctx[d]);
    }
  }
#pragma unroll
  for (int d = 0; d < DH; ++d) ctxT[(h * DH + d) * LDA + r] = ctx[d];
}

// y[j] = x . W[:, j] + b[j] for j < n (one thread per output; sequential k)
__device__ __forceinline__ void gemv_rows(const float* x, const float* W, const float* b, int k, int n, float* y) {
  for (int j = threadIdx.x; j < n; j += NT) {
    float acc = 0.0f;
    for (int i = 0; i < k; ++i) acc = fmaf(x[i], __ldg(W + i * n + j), acc);
    y[j] = acc + __ldg(b + j);
  }
}

// ---------------------------------------------------------------------------
// one pre-LN transformer sub-layer set on an R-row token panel

// self attention: X += Wo . attn(LN(X + pos)) + bo   (decoder.py:214-218)
template <int R, int LDA, class Pos>
__device__ void self_attention(float* X, int nvalid, const AttnW& w, Pos pos, float* A, float* QKV, float* Ws) {
  layer_norm_T<R>(X, D, nvalid, w.ln_g, w.ln_b, A, LDA, pos);
  stage(Ws, w.wqkv, D * 3 * D);
  __syncthreads();
  gemm_tile<R, D, 3 * D, LDA>(A, Ws, EpiRow{QKV, LDQKV, w.bqkv});
  __syncthreads();
  stage(Ws, w.wo, D * D);
  attention_core(QKV, LDQKV, QKV + D, QKV + 2 * D, LDQKV, nvalid, nvalid, A, LDA);
  __syncthreads();
  gemm_tile<R, D, D, LDA>(A, Ws, EpiAdd{X, D, w.bo, nvalid});
  __syncthreads();
}

// feature-side half of cross attention: K|V = LN_kv(F) @ [Wk|Wv] + b (64 rows)
__device__ void cross_kv(const float* F, const AttnW& w, float* Bt, float* KV, float* Ws) {
  layer_norm_T<64>(F, D, 64, w.ln2_g, w.ln2_b, Bt, 68, NoPos{});
  stage(Ws, w.wqkv, D * 3 * D);  // stage all of q|k|v; k|v are columns D..3D
  __syncthreads();
  // columns [D, 3D) of wqkv: shift the weight pointer and bias by D
  struct EpiKV {
    float* kv; const float* b;
    __device__ void operator()(int r, int c, float v) const { kv[r * LDKV + c] = v + __ldg(b + D + c); }
  };
  // W panel with row stride 3D: gemm_tile assumes stride N, so repack k|v
  // columns contiguously in place is not possible; use a strided view.
  {
    constexpr int R = 64, K = D, N = 2 * D;
    constexpr int RG = R / 4, CG = N / 4, MT = RG * CG, PT = MT / NT;
    float acc[PT][4][4];
#pragma unroll
    for (int p = 0; p < PT; ++p)
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[p][i][j] = 0.0f;
#pragma unroll 4
    for (int k = 0; k < K; ++k) {
#pragma unroll
      for (int p = 0; p < PT; ++p) {
        const int m = threadIdx.x + p * NT, mr = m % RG, mc = m / RG;
        const float4 a = *reinterpret_cast<const float4*>(Bt + k * 68 + mr * 4);
        const float4 wv4 = *reinterpret_cast<const float4*>(Ws + k * 3 * D + D + mc * 4);
        const float av[4] = {a.x, a.y, a.z, a.w};
        const float wv[4] = {wv4.x, wv4.y, wv4.z, wv4.w};
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[p][i][j] = fmaf(av[i], wv[j], acc[p][i][j]);
      }
    }
    EpiKV epi{KV, w.bqkv};
#pragma unroll
    for (int p = 0; p < PT; ++p) {
      const int m = threadIdx.x + p * NT, mr = m % RG, mc = m / RG;
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) epi(mr * 4 + i, mc * 4 + j, acc[p][i][j]);
    }
  }
}

// query-side half + attention + output: X += Wo . attn(LN_q(X), KV) + bo
template <int R, int LDA>
__device__ void cross_attention_q(float* X, int nvalid, const AttnW& w, const float* KV, int nk, float* A,
                                  float* Qb, float* Ws) {
  // Ws still holds q|k|v from cross_kv: q = columns [0, D)
  layer_norm_T<R>(X, D, nvalid, w.ln_g, w.ln_b, A, LDA, NoPos{});
  __syncthreads();
  {
    constexpr int RG = R / 4, CG = D / 4, MT = RG * CG, PT = (MT + NT - 1) / NT;
    float acc[PT][4][4];
#pragma unroll
    for (int p = 0; p < PT; ++p)
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[p][i][j] = 0.0f;
#pragma unroll 4
    for (int k = 0; k < D; ++k) {
#pragma unroll
      for (int p = 0; p < PT; ++p) {
        const int m = threadIdx.x + p * NT;
        if (MT % NT == 0 || m < MT) {
          const int mr = m % RG, mc = m / RG;
          const float4 a = *reinterpret_cast<const float4*>(A + k * LDA + mr * 4);
          const float4 wv4 = *reinterpret_cast<const float4*>(Ws + k * 3 * D + mc * 4);
          const float av[4] = {a.x, a.y, a.z, a.w};
          const float wv[4] = {wv4.x, wv4.y, wv4.z, wv4.w};
#pragma unroll
          for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) acc[p][i][j] = fmaf(av[i], wv[j], acc[p][i][j]);
        }
      }
    }
#pragma unroll
    for (int p = 0; p < PT; ++p) {
      const int m = threadIdx.x + p * NT;
      if (MT % NT == 0 || m < MT) {
        const int mr = m % RG, mc = m / RG;
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) Qb[(mr * 4 + i) * LDQKV + mc * 4 + j] = acc[p][i][j] + __ldg(w.bqkv + mc * 4 + j);
      }
    }
  }
  __syncthreads();
  stage(Ws, w.wo, D * D);
  attention_core(Qb, LDQKV, KV, KV + D, LDKV, nvalid, nk, A, LDA);
  __syncthreads();
  gemm_tile<R, D, D, LDA>(A, Ws, EpiAdd{X, D, w.bo, nvalid});
  __syncthreads();
}

// X += W2 . relu(W1 . LN(X) + b1) + b2   (decoder.py:205-212)
template <int R, int LDA>
__device__ void mlp_block(float* X, int nvalid, const MlpW& w, float* A, float* Ht, float* Ws) {
  layer_norm_T<R>(X, D, nvalid, w.ln_g, w.ln_b, A, LDA, NoPos{});
  stage(Ws, w.w1, D * 4 * D);
  __syncthreads();
  gemm_tile<R, D, 4 * D, LDA>(A, Ws, EpiT{Ht, LDA, w.b1, true});
  __syncthreads();
  stage(Ws, w.w2, 4 * D * D);
  __syncthreads();
  gemm_tile<R, 4 * D, D, LDA>(Ht, Ws, EpiAdd{X, D, w.b2, nvalid});
  __syncthreads();
}

}  // namespace

// ===========================================================================
// K2: encoder.  grid = ncrops, one crop per CTA.
// smem: X[64][64] | A[64][68] | H (qkv [64][196] / patches^T [192][68] /
// hidden^T [256][68]) | W stage [16384]
// ===========================================================================
constexpr int kEncSmemFloats = 64 * 64 + 64 * 68 + 256 * 68 + WSTAGE;

__global__ void __launch_bounds__(NT, 1) k_encoder_f32(const float* __restrict__ crops, int ncrops, EncW w,
                                                        float* __restrict__ feats, int* nonfinite) {
  extern __shared__ __align__(16) float sm[];
  float* X = sm;
  float* A = X + 64 * 64;
  float* H = A + 64 * 68;
  float* Ws = H + 256 * 68;
  const int cidx = blockIdx.x;
  const float* crop = crops + (int64_t)cidx * 64 * 64 * 3;
  const int tid = threadIdx.x;

  // patchify (decoder.py:247-248): row r = py*8+px, col k = (iy*8+ix)*3+c
  for (int idx = tid; idx < 64 * 192; idx += NT) {
    const int k = idx / 64, r = idx % 64;
    const int py = r / 8, px = r % 8, pix = k / 3, c = k % 3, iy = pix / 8, ix = pix % 8;
    H[k * 68 + r] = __ldg(crop + ((py * 8 + iy) * 64 + px * 8 + ix) * 3 + c);
  }
  stage(Ws, w.patch_w, 192 * D);
  __syncthreads();
  {
    struct EpiEmbed {
      float* X; const float* b; const float* pos;
      __device__ void operator()(int r, int c, float v) const {
        X[r * D + c] = (v + __ldg(b + c)) + __ldg(pos + r * D + c);
      }
    };
    gemm_tile<64, 192, D, 68>(H, Ws, EpiEmbed{X, w.patch_b, w.pos});
  }
  __syncthreads();
  for (int l = 0; l < w.layers; ++l) {
    self_attention<64, 68>(X, 64, w.self[l], NoPos{}, A, H, Ws);
    mlp_block<64, 68>(X, 64, w.mlp[l], A, H, Ws);
  }
  // final LN straight to HBM, row-major (B, 64, 64)
  {
    const int r = tid / 4, part = tid % 4;
    float v[16];
    float s = 0.0f;
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      v[i] = X[r * D + part + 4 * i];
      s += v[i];
    }
    s += __shfl_xor_sync(0xffffffffu, s, 1);
    s += __shfl_xor_sync(0xffffffffu, s, 2);
    const float mu = s * (1.0f / D);
    float q = 0.0f;
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      v[i] -= mu;
      q += v[i] * v[i];
    }
    q += __shfl_xor_sync(0xffffffffu, q, 1);
    q += __shfl_xor_sync(0xffffffffu, q, 2);
    const float sd = sqrtf(q * (1.0f / D) + 1e-5f);
    float* out = feats + ((int64_t)cidx * 64 + r) * D;
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const int c = part + 4 * i;
      const float y = v[i] / sd * __ldg(w.norm_g + c) + __ldg(w.norm_b + c);
      flag_nonfinite(nonfinite, y);
      out[c] = y;
    }
  }
}

// ===========================================================================
// K3: decoders.  grid = nbody + nhand CTAs: blocks [0, nbody) decode one
// frame's body crop, blocks [nbody, nbody + nhand) decode one hand crop.
// feats: (n, 64, 64); the body feature of frame f is feats[body_idx(f)], the
// hands' are given by hand_feat_idx.
// ===========================================================================

// layout of the body CTA's shared memory (floats)
constexpr int kBodyX = 0;                       // tokens [64][64]
constexpr int kBodyP2 = kBodyX + 64 * 64;       // p2d [22][64]
constexpr int kBodyP3 = kBodyP2 + 22 * 64;      // p3d [22][64]
constexpr int kBodyA = kBodyP3 + 22 * 64;       // A [64][68]
constexpr int kBodyB = kBodyA + 64 * 68;        // Bt [64][68] (LN_kv(feat)^T)
constexpr int kBodyH = kBodyB + 64 * 68;        // qkv [64][196] + kv [64][132]; hidden^T [256][68]
constexpr int kBodyHSize = 64 * LDQKV + 64 * LDKV;
constexpr int kBodyW = kBodyH + kBodyHSize;     // W stage
constexpr int kBodyS = kBodyW + WSTAGE;         // scratch (heads, FK)
constexpr int kDecSmemFloats = kBodyS + 1024 + (int)(sizeof(FKOut) / 4) + 16;

static_assert(kBodyHSize >= 256 * 68, "hidden panel must fit in the qkv/kv region");

__device__ void body_heads(const float* X, const BodyW& w, float* t0, float* params, float* cam, int warp,
                           int lane) {
  if (warp == 0) layer_norm_row_warp(X, w.norm_g, w.norm_b, t0, lane);
  __syncthreads();
  for (int j = threadIdx.x; j < FSB_PARAM_DIM + 3; j += NT) {
    const float* W = j < FSB_PARAM_DIM ? w.head_params_w : w.head_cam_w;
    const int n = j < FSB_PARAM_DIM ? FSB_PARAM_DIM : 3;
    const int jj = j < FSB_PARAM_DIM ? j : j - FSB_PARAM_DIM;
    float acc = 0.0f;
    for (int k = 0; k < D; ++k) acc = fmaf(t0[k], __ldg(W + k * n + jj), acc);
    if (j < FSB_PARAM_DIM)
      params[jj] = acc + __ldg(w.head_params_b + jj);
    else
      cam[jj] = acc + __ldg(w.head_cam_b + jj);
  }
  __syncthreads();
}

__device__ void decode_body_cta(const DecodeArgs& a, const BodyW& w, float* sm, int f) {
  float* X = sm + kBodyX;
  float* P2 = sm + kBodyP2;
  float* P3 = sm + kBodyP3;
  float* A = sm + kBodyA;
  float* Bt = sm + kBodyB;
  float* QKV = sm + kBodyH;
  float* KV = QKV + 64 * LDQKV;
  float* Ht = sm + kBodyH;
  float* Ws = sm + kBodyW;
  float* S = sm + kBodyS;
  float* t0 = S;              // 64
  float* params = S + 64;     // 76 (+pad)
  float* cam = S + 144;       // 3
  float* kp2d = S + 160;      // 44
  float* jc = S + 208;        // 66 centred joints
  float* boxtok = S + 288;    // 256
  FKOut& fk = *reinterpret_cast<FKOut*>(S + 1024);
  const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
  const float* feat = a.feats + (int64_t)f * a.body_feat_stride * 64 * D;

  // tokens = token_init (+ box prompt on rows 1..4); padded rows are zero
  for (int i = tid; i < 64 * D; i += NT) X[i] = (i < 51 * D) ? __ldg(w.token_init + i) : 0.0f;
  for (int i = tid; i < 22 * D; i += NT) {
    P2[i] = __ldg(w.p2d_init + i);
    P3[i] = __ldg(w.p3d_init + i);
  }
  if (tid < 8) S[1000 + tid] = a.prompts[(int64_t)f * 8 + tid];
  __syncthreads();
  gemv_rows(S + 1000, w.prompt_box_w, w.prompt_box_b, 8, 4 * D, boxtok);
  __syncthreads();
  X[D + tid] += boxtok[tid];  // rows 1..4 (tid < 256 == 4 * D)
  __syncthreads();

  for (int l = 0; l < w.layers; ++l) {
    self_attention<64, 68>(X, 51, w.self[l], BodyPos{P2, P3}, A, QKV, Ws);
    cross_kv(feat, w.cross[l], Bt, KV, Ws);
    cross_attention_q<64, 68>(X, 51, w.cross[l], KV, 64, A, QKV, Ws);
    mlp_block<64, 68>(X, 51, w.mlp[l], A, Ht, Ws);
    if ((a.body_sel >> l) & 1u) {
      // intermediate prediction (decoder.py:310-320)
      body_heads(X, w, t0, params, cam, warp, lane);
      if (warp == 0) fk_warp(params, w.joints_rest, fk, lane);
      __syncthreads();
      if (tid < FSB_NJ) {
        kp2d[2 * tid] = cam[0] * fk.tw[tid][0] + cam[1];
        kp2d[2 * tid + 1] = cam[0] * fk.tw[tid][1] + cam[2];
        for (int c = 0; c < 3; ++c) jc[3 * tid + c] = fk.tw[tid][c] - fk.tw[0][c];
      }
      __syncthreads();
      if (a.inter != nullptr) {
        float* dst = a.inter + ((int64_t)f * w.layers + l) * (FSB_PARAM_DIM + 3 + 44);
        for (int i = tid; i < FSB_PARAM_DIM + 3 + 44; i += NT)
          dst[i] = i < FSB_PARAM_DIM ? params[i] : (i < FSB_PARAM_DIM + 3 ? cam[i - FSB_PARAM_DIM] : kp2d[i - FSB_PARAM_DIM - 3]);
      }
      for (int i = tid; i < 22 * D; i += NT) {
        const int r = i / D, c = i % D;
        P2[i] = fmaf(kp2d[2 * r + 1], __ldg(w.phi2d_w + D + c), kp2d[2 * r] * __ldg(w.phi2d_w + c)) +
                __ldg(w.phi2d_b + c);
        P3[i] = fmaf(jc[3 * r + 2], __ldg(w.phi3d_w + 2 * D + c),
                     fmaf(jc[3 * r + 1], __ldg(w.phi3d_w + D + c), jc[3 * r] * __ldg(w.phi3d_w + c))) +
                __ldg(w.phi3d_b + c);
      }
      __syncthreads();
    }
  }
  body_heads(X, w, t0, params, cam, warp, lane);
  if (tid < FSB_PARAM_DIM) {
    const float v = params[tid];
    flag_nonfinite(a.nonfinite, v);
    a.body_params[(int64_t)f * FSB_PARAM_DIM + tid] = v;
    const bool hand_slot = (tid >= 51 && tid < 54) || (tid >= 63 && tid < 66);
    if (a.merged != nullptr && !hand_slot) a.merged[(int64_t)f * FSB_PARAM_DIM + tid] = v;
  }
  if (tid < 3) a.body_cam[(int64_t)f * 3 + tid] = cam[tid];
}

// hand CTA layout (floats)
constexpr int kHandX = 0;                   // tokens [16][64]
constexpr int kHandP = kHandX + 16 * 64;    // p_pts [3][64]
constexpr int kHandA = kHandP + 3 * 64 + 64;  // A [64][20]
constexpr int kHandB = kHandA + 64 * 20;    // Bt [64][68]
constexpr int kHandH = kHandB + 64 * 68;    // qkv [16][196] + kv [64][132]; hidden^T [256][20]
constexpr int kHandW = kHandH + 16 * LDQKV + 64 * LDKV;
constexpr int kHandS = kHandW + WSTAGE;
static_assert(kHandS + 256 <= kDecSmemFloats, "hand layout exceeds the decoder smem");

__device__ void decode_hand_cta(const DecodeArgs& a, const HandW& w, float* sm, int hnd) {
  float* X = sm + kHandX;
  float* P = sm + kHandP;
  float* A = sm + kHandA;
  float* Bt = sm + kHandB;
  float* QKV = sm + kHandH;
  float* KV = QKV + 16 * LDQKV;
  float* Ht = sm + kHandH;
  float* Ws = sm + kHandW;
  float* S = sm + kHandS;
  float* t0 = S;          // 64
  float* rc = S + 64;     // rots[3], cams[3]
  float* p2 = S + 80;     // 3 x 2
  const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
  const int frame = hnd / 2, side = hnd % 2;
  const int crop = a.hand_feat_first + frame * a.body_feat_stride + side;
  const float* feat = a.feats + (int64_t)crop * 64 * D;

  for (int i = tid; i < 16 * D; i += NT) X[i] = (i < 4 * D) ? __ldg(w.token_init + i) : 0.0f;
  for (int i = tid; i < 3 * D; i += NT) P[i] = __ldg(w.p_init + i);
  __syncthreads();

  auto heads = [&]() {
    if (warp == 0) layer_norm_row_warp(X, w.norm_g, w.norm_b, t0, lane);
    __syncthreads();
    if (tid < 6) {
      const float* W = tid < 3 ? w.head_rot_w : w.head_cam_w;
      const float* b = tid < 3 ? w.head_rot_b : w.head_cam_b;
      const int j = tid % 3;
      float acc = 0.0f;
      for (int k = 0; k < D; ++k) acc = fmaf(t0[k], __ldg(W + k * 3 + j), acc);
      rc[tid] = acc + __ldg(b + j);
    }
    __syncthreads();
  };

  for (int l = 0; l < w.layers; ++l) {
    self_attention<16, 20>(X, 4, w.self[l], HandPos{P}, A, QKV, Ws);
    cross_kv(feat, w.cross[l], Bt, KV, Ws);
    cross_attention_q<16, 20>(X, 4, w.cross[l], KV, 64, A, QKV, Ws);
    mlp_block<16, 20>(X, 4, w.mlp[l], A, Ht, Ws);
    if ((a.hand_sel >> l) & 1u) {
      // decoder.py:399-409: canonical points through the predicted rotation
      heads();
      if (tid == 0) {
        float R[9];
        rodrigues3(rc[0], rc[1], rc[2], R);
        for (int i = 0; i < 3; ++i) {
          float q[2];
          for (int ax = 0; ax < 2; ++ax)
            q[ax] = R[3 * ax] * __ldg(w.canon_pts + 3 * i) + R[3 * ax + 1] * __ldg(w.canon_pts + 3 * i + 1) +
                    R[3 * ax + 2] * __ldg(w.canon_pts + 3 * i + 2);
          p2[2 * i] = rc[3] * q[0] + rc[4];
          p2[2 * i + 1] = rc[3] * q[1] + rc[5];
        }
      }
      __syncthreads();
      for (int i = tid; i < 3 * D; i += NT) {
        const int r = i / D, c = i % D;
        P[i] = fmaf(p2[2 * r + 1], __ldg(w.phi2d_w + D + c), p2[2 * r] * __ldg(w.phi2d_w + c)) + __ldg(w.phi2d_b + c);
      }
      __syncthreads();
    }
  }
  heads();
  if (tid < 3) {
    const float v = rc[tid];
    flag_nonfinite(a.nonfinite, v);
    a.hand_rots[(int64_t)hnd * 3 + tid] = v;
    if (a.merged != nullptr) a.merged[(int64_t)frame * FSB_PARAM_DIM + (side == 0 ? 51 : 63) + tid] = v;
  }
}

__global__ void __launch_bounds__(NT, 1) k_decoders_f32(DecodeArgs a, BodyW bw, HandW hw) {
  extern __shared__ __align__(16) float sm[];
  if ((int)blockIdx.x < a.nbody)
    decode_body_cta(a, bw, sm, blockIdx.x);
  else
    decode_hand_cta(a, hw, sm, blockIdx.x - a.nbody);
}

cudaError_t init_attrs_transformer() {
  cudaError_t e = cudaFuncSetAttribute(k_encoder_f32, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)(kEncSmemFloats * sizeof(float)));
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(k_decoders_f32, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)(kDecSmemFloats * sizeof(float)));
}

cudaError_t launch_encoder_f32(const float* crops, int ncrops, const EncW& w, float* feats, int* nonfinite,
                               cudaStream_t st) {
  if (ncrops == 0) return cudaSuccess;
  const size_t smem = kEncSmemFloats * sizeof(float);
  k_encoder_f32<<<ncrops, NT, smem, st>>>(crops, ncrops, w, feats, nonfinite);
  return cudaGetLastError();
}

cudaError_t launch_decoders_f32(const DecodeArgs& a, const BodyW& bw, const HandW& hw, cudaStream_t st) {
  const int n = a.nbody + a.nhand;
  if (n == 0) return cudaSuccess;
  const size_t smem = kDecSmemFloats * sizeof(float);
  k_decoders_f32<<<n, NT, smem, st>>>(a, bw, hw);
  return cudaGetLastError();
}
