// K2 / K3 on the 5th-generation tensor cores (bf16 mode).
//
// Same math as the fp32 kernels in k_transformer.cu (reference decoder.py:
// encode :231-260, _attention :172-203, _mlp :205-212, decode_body
// :284-356, decode_hand :360-410) with every GEMM on tcgen05: operands are
// bf16 in shared memory (K-major UMMA layout, tc_sm100.cuh), accumulators
// are fp32 in TMEM, and the LayerNorm / softmax / residual / ReLU
// epilogues run in fp32 registers.
//
// One CTA = 4 warps = 128 TMEM lanes = 128 token rows, organised as two
// 64-row blocks: two crops (encoder), two frames' body tokens (51 valid
// rows each) or two hands (4 valid rows each).  Thread t owns row t for the
// whole network: its residual-stream row lives in 64 registers, LayerNorm
// and softmax are per-thread row reductions with no shuffles, and it writes
// its own row of every bf16 operand.  Attention of the two blocks is done
// as one 128 x 128 score tile whose off-diagonal block is masked to zero, so
// P.V stays a single MMA chain.  Weights (pre-packed bf16 W^T images) stream
// through two 32 KB slots with cp.async.bulk, one GEMM ahead of use.
#include "fsb_common.cuh"
#include "fsb_weights.h"
#include "tc_sm100.cuh"

namespace {

constexpr int D = 64, DH = 16, NTH = 128, BLK = 64;

// shared memory map (bytes)
constexpr uint32_t S_A = 0;         // 128 x 64 bf16 GEMM A operand           16 KB
constexpr uint32_t S_Q = 16384;     // 4 heads x (128 x 16) queries           16 KB
constexpr uint32_t S_K = 32768;     // 4 heads x (128 x 16) keys              16 KB
constexpr uint32_t S_VT = 49152;    // 4 heads x (16 x 128) values^T          16 KB
constexpr uint32_t S_HP = 65536;    // MLP hidden 128x256 | P 2x(128x128) | patches 128x192   64 KB
constexpr uint32_t S_W = 131072;    // 2 weight slots x 32 KB
constexpr uint32_t S_AUX = 196608;  // fp32 role scratch                      16 KB
constexpr uint32_t SMEM_TC = S_AUX + 16384;

// TMEM columns
constexpr uint32_t T_GEN = 0;   // GEMM accumulators / attention score pair
constexpr uint32_t T_O = 256;   // attention context (4 heads x 16)
constexpr uint32_t T_KV = 384;  // cross-attention K | V of the feature rows

constexpr int kMaxW = 64;

struct Shared {
  uint64_t wbar[2];
  uint64_t mbar;
  uint32_t tmem;
  int nw;
  const uint8_t* wptr[kMaxW];
  uint32_t wbytes[kMaxW];
};

// per-thread pipeline state (every thread tracks the same phases)
struct Pipe {
  Shared* sh;
  uint8_t* smem;
  uint32_t sbase;   // shared-space address of smem
  uint32_t tmem;
  uint32_t mphase;
  int wload, wuse;
  int tid;

  __device__ void prefetch() {  // next weight image into its ring slot
    if (wload < sh->nw) {
      if (tid == 0) {
        const int slot = wload & 1;
        tc::mbar_expect_tx(&sh->wbar[slot], sh->wbytes[wload]);
        tc::bulk_g2s(smem + S_W + slot * 32768u, sh->wptr[wload], sh->wbytes[wload], &sh->wbar[slot]);
      }
      ++wload;
    }
  }
  __device__ uint32_t acquire() {  // wait for the next weight image; returns its address
    const int slot = wuse & 1;
    tc::mbar_wait(&sh->wbar[slot], (uint32_t)((wuse >> 1) & 1));
    ++wuse;
    return sbase + S_W + slot * 32768u;
  }
  // operands written by threads -> visible to the tensor core; TMEM reads done
  __device__ void before_issue() {
    tc::fence_async_smem();
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
  }
  __device__ void commit_wait() {
    if (tid == 0) tc::mma_commit(&sh->mbar);
    tc::mbar_wait(&sh->mbar, mphase);
    mphase ^= 1u;
    tc::fence_after();
  }
  __device__ uint32_t lane_addr(uint32_t col) const {
    return tmem + ((uint32_t)((tid >> 5) * 32) << 16) + col;
  }
};

__device__ __forceinline__ void gemm(uint32_t a, int K, uint32_t b, int N, uint32_t dcol, uint32_t tmem) {
  const uint32_t id = tc::idesc_bf16(128, N);
  for (int k = 0; k < K; k += 16) tc::mma_bf16(tmem + dcol, tc::kmajor_desc(a, K, k), tc::kmajor_desc(b, K, k), id, k > 0);
}

// store 8 consecutive bf16 values of row r at column k0 of a K-major tile
__device__ __forceinline__ void st_row8(uint8_t* tile, int r, int k0, int K, const float* v) {
  uint4 u;
  u.x = tc::pack_bf16(v[0], v[1]);
  u.y = tc::pack_bf16(v[2], v[3]);
  u.z = tc::pack_bf16(v[4], v[5]);
  u.w = tc::pack_bf16(v[6], v[7]);
  *reinterpret_cast<uint4*>(tile + tc::kmajor_off(r, k0, K)) = u;
}

__device__ __forceinline__ void st_row_zero8(uint8_t* tile, int r, int k0, int K) {
  *reinterpret_cast<uint4*>(tile + tc::kmajor_off(r, k0, K)) = make_uint4(0u, 0u, 0u, 0u);
}

// 64-element row reductions with 8 independent partial chains
__device__ __forceinline__ float sum64(const float* v) {
  float p[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) p[i] = v[i];
#pragma unroll
  for (int c = 8; c < 64; ++c) p[c & 7] += v[c];
  return ((p[0] + p[1]) + (p[2] + p[3])) + ((p[4] + p[5]) + (p[6] + p[7]));
}

// mean and 1/sqrt(var + eps) of a 64-float row (numkit.py:198-202)
__device__ __forceinline__ void row_stats(const float* x, float& mu, float& rstd) {
  mu = sum64(x) * (1.0f / D);
  float p[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) p[i] = 0.0f;
#pragma unroll
  for (int c = 0; c < D; ++c) {
    const float d = x[c] - mu;
    p[c & 7] = fmaf(d, d, p[c & 7]);
  }
  const float q = ((p[0] + p[1]) + (p[2] + p[3])) + ((p[4] + p[5]) + (p[6] + p[7]));
  rstd = 1.0f / sqrtf(q * (1.0f / D) + 1e-5f);
}

// LayerNorm of the thread's row, bf16 into the A tile
__device__ __forceinline__ void ln_to_tile(const float* x, const float* g, const float* b, uint8_t* tile, int r) {
  float mu, rstd;
  row_stats(x, mu, rstd);
#pragma unroll
  for (int c0 = 0; c0 < D; c0 += 8) {
    float v[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = fmaf((x[c0 + i] - mu) * rstd, __ldg(g + c0 + i), __ldg(b + c0 + i));
    st_row8(tile, r, c0, D, v);
  }
}

__device__ __forceinline__ void ln_row(const float* x, const float* g, const float* b, float* y) {
  float mu, rstd;
  row_stats(x, mu, rstd);
#pragma unroll
  for (int c = 0; c < D; ++c) y[c] = fmaf((x[c] - mu) * rstd, __ldg(g + c), __ldg(b + c));
}

// q (cols qcol..+64 of TMEM) + bias -> per-head query tiles
__device__ void drain_q(Pipe& P, uint32_t qcol, const float* bq) {
  const int t = P.tid;
  float v[64];
  tc::tmem_ld64(P.lane_addr(qcol), v);
#pragma unroll
  for (int h = 0; h < 4; ++h) {
#pragma unroll
    for (int i = 0; i < 16; ++i) v[16 * h + i] += __ldg(bq + 16 * h + i);
    uint8_t* tq = P.smem + S_Q + h * 4096;
    st_row8(tq, t, 0, DH, v + 16 * h);
    st_row8(tq, t, 8, DH, v + 16 * h + 8);
  }
}

// k | v (cols kcol..+128) + bias -> per-head key tiles and transposed values
__device__ void drain_kv(Pipe& P, uint32_t kcol, const float* bk, const float* bv) {
  const int t = P.tid;
  float v[64];
  tc::tmem_ld64(P.lane_addr(kcol), v);
#pragma unroll
  for (int h = 0; h < 4; ++h) {
#pragma unroll
    for (int i = 0; i < 16; ++i) v[16 * h + i] += __ldg(bk + 16 * h + i);
    uint8_t* tk = P.smem + S_K + h * 4096;
    st_row8(tk, t, 0, DH, v + 16 * h);
    st_row8(tk, t, 8, DH, v + 16 * h + 8);
  }
  tc::tmem_ld64(P.lane_addr(kcol + 64), v);
  // V^T tile (16 x 128 per head): row d, column = this thread's key index
  const uint32_t col_off = (uint32_t)(t >> 3) * 128u + (uint32_t)(t & 7) * 2u;
#pragma unroll
  for (int h = 0; h < 4; ++h) {
    uint8_t* tv = P.smem + S_VT + h * 4096 + col_off;
#pragma unroll
    for (int d = 0; d < DH; ++d) {
      const __nv_bfloat16 hv = __float2bfloat16_rn(v[16 * h + d] + __ldg(bv + 16 * h + d));
      *reinterpret_cast<__nv_bfloat16*>(tv + (d >> 3) * 2048 + (d & 7) * 16) = hv;
    }
  }
}

// softmax of heads (2p, 2p+1) over the thread's own key block
__device__ void softmax_pair(Pipe& P, int nk) {
  const int t = P.tid, blk = t / BLK;
#pragma unroll 1
  for (int j = 0; j < 2; ++j) {
    float s[64];
    tc::tmem_ld64(P.lane_addr(T_GEN + 128 * j + 64 * blk), s);
    float m8[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) m8[i] = -INFINITY;
    // logits scaled by f32(1/sqrt(16)) and by log2(e) for the exp2 below
    constexpr float kScale = 0.25f * 1.4426950408889634f;
#pragma unroll
    for (int k = 0; k < 64; ++k) {
      s[k] = (k < nk) ? s[k] * kScale : -INFINITY;
      m8[k & 7] = fmaxf(m8[k & 7], s[k]);
    }
    const float mx = fmaxf(fmaxf(fmaxf(m8[0], m8[1]), fmaxf(m8[2], m8[3])),
                           fmaxf(fmaxf(m8[4], m8[5]), fmaxf(m8[6], m8[7])));
#pragma unroll
    for (int k = 0; k < 64; ++k) s[k] = (k < nk) ? exp2f(s[k] - mx) : 0.0f;
    const float inv = 1.0f / sum64(s);
    uint8_t* tp = P.smem + S_HP + j * 32768;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      float v[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) v[i] = s[8 * q + i] * inv;
      st_row8(tp, t, 64 * blk + 8 * q, 128, v);
      st_row_zero8(tp, t, 64 * (1 - blk) + 8 * q, 128);
    }
  }
}

// the four heads of one attention given sQ / sK / sVt; context -> ctx[64]
__device__ void attn_core(Pipe& P, int nk, float* ctx) {
  const uint32_t sq = P.sbase + S_Q, sk = P.sbase + S_K, sv = P.sbase + S_VT, sp = P.sbase + S_HP;
  const uint32_t id_s = tc::idesc_bf16(128, 128), id_o = tc::idesc_bf16(128, 16);
  P.before_issue();
  if (P.tid == 0)
    for (int j = 0; j < 2; ++j)
      tc::mma_bf16(P.tmem + T_GEN + 128 * j, tc::kmajor_desc(sq + j * 4096, DH, 0),
                   tc::kmajor_desc(sk + j * 4096, DH, 0), id_s, false);
  P.commit_wait();
#pragma unroll 1
  for (int pair = 0; pair < 2; ++pair) {
    softmax_pair(P, nk);
    P.before_issue();
    if (P.tid == 0) {
      for (int j = 0; j < 2; ++j) {
        const int h = 2 * pair + j;
        for (int k = 0; k < 128; k += 16)
          tc::mma_bf16(P.tmem + T_O + 16 * h, tc::kmajor_desc(sp + j * 32768, 128, k),
                       tc::kmajor_desc(sv + h * 4096, 128, k), id_o, k > 0);
      }
      if (pair == 0)
        for (int j = 0; j < 2; ++j)
          tc::mma_bf16(P.tmem + T_GEN + 128 * j, tc::kmajor_desc(sq + (2 + j) * 4096, DH, 0),
                       tc::kmajor_desc(sk + (2 + j) * 4096, DH, 0), id_s, false);
    }
    P.commit_wait();
  }
  tc::tmem_ld64(P.lane_addr(T_O), ctx);
}

// x += Wo . ctx + bo for valid rows
__device__ void out_proj(Pipe& P, const float* ctx, const float* bo, float* x, bool valid) {
  uint8_t* ta = P.smem + S_A;
#pragma unroll
  for (int c0 = 0; c0 < D; c0 += 8) st_row8(ta, P.tid, c0, D, ctx + c0);
  const uint32_t w = P.acquire();
  P.before_issue();
  if (P.tid == 0) gemm(P.sbase + S_A, D, w, D, T_GEN, P.tmem);
  P.prefetch();
  P.commit_wait();
  float v[64];
  tc::tmem_ld64(P.lane_addr(T_GEN), v);
  if (valid)
#pragma unroll
    for (int c = 0; c < D; ++c) x[c] += v[c] + __ldg(bo + c);
}

// self attention sub-layer: x += MHA(LN(x + pos))  (decoder.py:214-218)
__device__ void self_attn(Pipe& P, const AttnW& w, float* x, const float* pos, int nk, bool valid) {
  float a[D];
#pragma unroll
  for (int c = 0; c < D; ++c) a[c] = x[c] + pos[c];
  ln_to_tile(a, w.ln_g, w.ln_b, P.smem + S_A, P.tid);
  const uint32_t wq = P.acquire();
  P.before_issue();
  if (P.tid == 0) gemm(P.sbase + S_A, D, wq, 3 * D, T_GEN, P.tmem);
  P.prefetch();
  P.commit_wait();
  drain_q(P, T_GEN, w.bqkv);
  drain_kv(P, T_GEN + 64, w.bqkv + 64, w.bqkv + 128);
  float ctx[D];
  attn_core(P, nk, ctx);
  out_proj(P, ctx, w.bo, x, valid);
}

// cross attention sub-layer: x += MHA(LN_q(x), LN_kv(f))  (decoder.py:220-227)
__device__ void cross_attn(Pipe& P, const AttnW& w, float* x, const float* frow, bool valid) {
  float f[D];
#pragma unroll
  for (int c = 0; c < D; c += 4) {
    const float4 v = __ldg(reinterpret_cast<const float4*>(frow + c));
    f[c] = v.x; f[c + 1] = v.y; f[c + 2] = v.z; f[c + 3] = v.w;
  }
  ln_to_tile(f, w.ln2_g, w.ln2_b, P.smem + S_A, P.tid);
  const uint32_t wkv = P.acquire();
  P.before_issue();
  if (P.tid == 0) gemm(P.sbase + S_A, D, wkv, 2 * D, T_KV, P.tmem);
  P.prefetch();
  P.commit_wait();
  drain_kv(P, T_KV, w.bqkv + 64, w.bqkv + 128);
  ln_to_tile(x, w.ln_g, w.ln_b, P.smem + S_A, P.tid);
  const uint32_t wq = P.acquire();
  P.before_issue();
  if (P.tid == 0) gemm(P.sbase + S_A, D, wq, D, T_GEN, P.tmem);
  P.prefetch();
  P.commit_wait();
  drain_q(P, T_GEN, w.bqkv);
  float ctx[D];
  attn_core(P, BLK, ctx);
  out_proj(P, ctx, w.bo, x, valid);
}

// MLP sub-layer: x += W2 relu(W1 LN(x) + b1) + b2  (decoder.py:205-212)
__device__ void mlp(Pipe& P, const MlpW& w, float* x, bool valid) {
  ln_to_tile(x, w.ln_g, w.ln_b, P.smem + S_A, P.tid);
  const uint32_t w1 = P.acquire();
  P.before_issue();
  if (P.tid == 0) gemm(P.sbase + S_A, D, w1, 4 * D, T_GEN, P.tmem);
  P.prefetch();
  P.commit_wait();
  uint8_t* th = P.smem + S_HP;
#pragma unroll 1
  for (int q = 0; q < 4; ++q) {
    float v[64];
    tc::tmem_ld64(P.lane_addr(T_GEN + 64 * q), v);
#pragma unroll
    for (int i = 0; i < 64; ++i) v[i] = fmaxf(v[i] + __ldg(w.b1 + 64 * q + i), 0.0f);
#pragma unroll
    for (int i = 0; i < 64; i += 8) st_row8(th, P.tid, 64 * q + i, 4 * D, v + i);
  }
  const uint32_t w2 = P.acquire();
  P.before_issue();
  if (P.tid == 0) gemm(P.sbase + S_HP, 4 * D, w2, D, T_GEN, P.tmem);
  P.prefetch();
  P.commit_wait();
  float v[64];
  tc::tmem_ld64(P.lane_addr(T_GEN), v);
  if (valid)
#pragma unroll
    for (int c = 0; c < D; ++c) x[c] += v[c] + __ldg(w.b2 + c);
}

__device__ void setup(Pipe& P, Shared& sh, uint8_t* smem) {
  P.sh = &sh;
  P.smem = smem;
  P.sbase = tc::smem_u32(smem);
  P.tid = threadIdx.x;
  P.mphase = 0;
  P.wload = 0;
  P.wuse = 0;
  if (P.tid == 0) {
    tc::mbar_init(&sh.wbar[0], 1);
    tc::mbar_init(&sh.wbar[1], 1);
    tc::mbar_init(&sh.mbar, 1);
    tc::mbar_fence_init();
  }
  if (P.tid < 32) tc::tmem_alloc(&sh.tmem, 512);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  P.tmem = sh.tmem;
  P.prefetch();
}

__device__ void teardown(Pipe& P) {
  tc::fence_before();
  __syncthreads();
  if (P.tid < 32) tc::tmem_dealloc(P.tmem, 512);
}

}  // namespace

// ===========================================================================
// encoder: grid = ceil(ncrops / 2); block f of CTA b encodes crop 2b + f
// ===========================================================================
__global__ void __launch_bounds__(NTH, 1) k_encoder_tc(const float* __restrict__ crops, int ncrops, EncW w,
                                                       float* __restrict__ feats, int* nonfinite) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ Shared sh;
  const int t = threadIdx.x, blk = t / BLK, p = t % BLK;
  const int crop = 2 * blockIdx.x + blk;
  const bool valid = crop < ncrops;
  if (t == 0) {
    int n = 0;
    sh.wptr[n] = w.t_patch;
    sh.wbytes[n++] = 192 * D * 2;
    for (int l = 0; l < w.layers; ++l) {
      sh.wptr[n] = w.self[l].t_qkv; sh.wbytes[n++] = 3 * D * D * 2;
      sh.wptr[n] = w.self[l].t_o;   sh.wbytes[n++] = D * D * 2;
      sh.wptr[n] = w.mlp[l].t_w1;   sh.wbytes[n++] = 4 * D * D * 2;
      sh.wptr[n] = w.mlp[l].t_w2;   sh.wbytes[n++] = 4 * D * D * 2;
    }
    sh.nw = n;
  }
  __syncthreads();
  Pipe P;
  setup(P, sh, smem);

  // patchify row p of this crop (decoder.py:247-248) into the K = 192 tile
  {
    uint8_t* tile = smem + S_HP;
    const int py = p / 8, px = p % 8;
    const float* src = crops + (int64_t)(valid ? crop : 0) * 64 * 64 * 3;
#pragma unroll 1
    for (int iy = 0; iy < 8; ++iy) {
      const float* row = src + ((py * 8 + iy) * 64 + px * 8) * 3;
#pragma unroll
      for (int q = 0; q < 3; ++q) {
        float v[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) v[i] = valid ? __ldg(row + 8 * q + i) : 0.0f;
        st_row8(tile, t, iy * 24 + 8 * q, 192, v);
      }
    }
  }
  float x[D];
  {
    const uint32_t wp = P.acquire();
    P.before_issue();
    if (t == 0) gemm(P.sbase + S_HP, 192, wp, D, T_GEN, P.tmem);
    P.prefetch();
    P.commit_wait();
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      float v[16];
      tc::tmem_ld16(P.lane_addr(T_GEN + 16 * q), v);
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const int c = 16 * q + i;
        x[c] = valid ? (v[i] + __ldg(w.patch_b + c)) + __ldg(w.pos + p * D + c) : 0.0f;
      }
    }
  }
  float zero[D];
#pragma unroll
  for (int c = 0; c < D; ++c) zero[c] = 0.0f;
  for (int l = 0; l < w.layers; ++l) {
    self_attn(P, w.self[l], x, zero, BLK, valid);
    mlp(P, w.mlp[l], x, valid);
  }
  float y[D];
  ln_row(x, w.norm_g, w.norm_b, y);
  if (valid) {
    float* out = feats + ((int64_t)crop * 64 + p) * D;
#pragma unroll
    for (int c = 0; c < D; c += 4) {
      flag_nonfinite(nonfinite, y[c] + y[c + 1] + y[c + 2] + y[c + 3]);
      *reinterpret_cast<float4*>(out + c) = make_float4(y[c], y[c + 1], y[c + 2], y[c + 3]);
    }
  }
  teardown(P);
}

// ===========================================================================
// decoders: CTAs [0, nb) decode two frames' bodies, CTAs [nb, nb + nh) two
// hands each.
// ===========================================================================
struct BodyAux {  // fp32 scratch per block
  float t0[2][D];
  float params[2][80];
  float cam[2][4];
  float kp2d[2][44];
  float jc[2][66];
  int pred[2];
  FKOut fk[2];
  float boxtok[2][4 * D];
};
struct HandAux {
  float t0[2][D];
  float rc[2][8];   // rots[3], cams[3]
  float pts[2][6];  // 3 x (x, y) projected canonical points
  int pred[2];
};
static_assert(sizeof(BodyAux) <= 16384 && sizeof(HandAux) <= 16384, "aux scratch");

__device__ void body_heads(Pipe& P, BodyAux& ax, const BodyW& w, const float* x) {
  const int t = P.tid, blk = t / BLK, r = t % BLK;
  if (r == 0) {
    float y[D];
    ln_row(x, w.norm_g, w.norm_b, y);
#pragma unroll
    for (int c = 0; c < D; ++c) ax.t0[blk][c] = y[c];
  }
  __syncthreads();
  // thread (blk, r) evaluates outputs r and r + 64 of its block's 79 head
  // outputs (76 params + 3 camera); 64 independent loads per output
  for (int o = r; o < 79; o += 64) {
    const bool is_p = o < FSB_PARAM_DIM;
    const float* W = is_p ? w.head_params_w : w.head_cam_w;
    const int n = is_p ? FSB_PARAM_DIM : 3, oo = is_p ? o : o - FSB_PARAM_DIM;
    float acc[4] = {0.0f, 0.0f, 0.0f, 0.0f};
#pragma unroll
    for (int k = 0; k < D; ++k) acc[k & 3] = fmaf(ax.t0[blk][k], __ldg(W + k * n + oo), acc[k & 3]);
    const float v = (acc[0] + acc[1]) + (acc[2] + acc[3]);
    if (is_p)
      ax.params[blk][oo] = v + __ldg(w.head_params_b + oo);
    else
      ax.cam[blk][oo] = v + __ldg(w.head_cam_b + oo);
  }
  __syncthreads();
}

__global__ void __launch_bounds__(NTH, 1) k_decoders_tc(DecodeArgs a, BodyW bw, HandW hw) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ Shared sh;
  const int t = threadIdx.x, blk = t / BLK, r = t % BLK;
  const int nbc = (a.nbody + 1) / 2;
  const bool body = (int)blockIdx.x < nbc;
  const int unit = body ? 2 * blockIdx.x + blk : 2 * (blockIdx.x - nbc) + blk;  // frame or hand index
  const int nunit = body ? a.nbody : a.nhand;
  const bool uvalid = unit < nunit;
  const int nrows = body ? 51 : 4;
  const bool valid = uvalid && r < nrows;
  const int layers = body ? bw.layers : hw.layers;
  if (t == 0) {
    int n = 0;
    for (int l = 0; l < layers; ++l) {
      const AttnW& s = body ? bw.self[l] : hw.self[l];
      const AttnW& c = body ? bw.cross[l] : hw.cross[l];
      const MlpW& m = body ? bw.mlp[l] : hw.mlp[l];
      sh.wptr[n] = s.t_qkv; sh.wbytes[n++] = 3 * D * D * 2;
      sh.wptr[n] = s.t_o;   sh.wbytes[n++] = D * D * 2;
      sh.wptr[n] = c.t_kv;  sh.wbytes[n++] = 2 * D * D * 2;
      sh.wptr[n] = c.t_q;   sh.wbytes[n++] = D * D * 2;
      sh.wptr[n] = c.t_o;   sh.wbytes[n++] = D * D * 2;
      sh.wptr[n] = m.t_w1;  sh.wbytes[n++] = 4 * D * D * 2;
      sh.wptr[n] = m.t_w2;  sh.wbytes[n++] = 4 * D * D * 2;
    }
    sh.nw = n;
  }
  __syncthreads();
  Pipe P;
  setup(P, sh, smem);

  // feature row of this thread for cross attention
  int crop;
  if (body) {
    crop = (uvalid ? unit : 0) * a.body_feat_stride;
  } else {
    const int hnd = uvalid ? unit : 0;
    crop = a.hand_feat_first + (hnd / 2) * a.body_feat_stride + (hnd % 2);
  }
  const float* frow = a.feats + ((int64_t)crop * 64 + r) * D;

  float x[D], pos[D];
  BodyAux& bx = *reinterpret_cast<BodyAux*>(smem + S_AUX);
  HandAux& hx = *reinterpret_cast<HandAux*>(smem + S_AUX);
  if (body) {
    // tokens = token_init, rows 1..4 += prompt_box(prompt)  (decoder.py:287-293);
    // the 2 x 256 box-token outputs are spread over the CTA, 4 per thread
    for (int i = 0; i < 4; ++i) {
      const int idx = 4 * t + i, b = idx / (4 * D), o = idx % (4 * D);
      const int u = 2 * blockIdx.x + b;
      float acc = 0.0f;
      if (u < a.nbody) {
#pragma unroll
        for (int k = 0; k < 8; ++k) acc = fmaf(a.prompts[(int64_t)u * 8 + k], __ldg(bw.prompt_box_w + k * 4 * D + o), acc);
      }
      bx.boxtok[b][o] = acc + __ldg(bw.prompt_box_b + o);
    }
    if (t < 2) bx.pred[t] = 0;
    __syncthreads();
#pragma unroll
    for (int c = 0; c < D; ++c) {
      float v = valid ? __ldg(bw.token_init + r * D + c) : 0.0f;
      if (valid && r >= 1 && r < 5) v += bx.boxtok[blk][(r - 1) * D + c];
      x[c] = v;
    }
  } else {
#pragma unroll
    for (int c = 0; c < D; ++c) x[c] = valid ? __ldg(hw.token_init + r * D + c) : 0.0f;
    if (t < 2) hx.pred[t] = 0;
  }
  __syncthreads();

  for (int l = 0; l < layers; ++l) {
    // positional terms of the self-attention input
    if (body) {
      const bool pr2 = r >= 5 && r < 27, pr3 = r >= 27 && r < 49;
#pragma unroll
      for (int c = 0; c < D; ++c) {
        float v = 0.0f;
        if (valid && pr2) {
          const int j = r - 5;
          v = bx.pred[blk] ? fmaf(bx.kp2d[blk][2 * j + 1], __ldg(bw.phi2d_w + D + c),
                                  bx.kp2d[blk][2 * j] * __ldg(bw.phi2d_w + c)) + __ldg(bw.phi2d_b + c)
                           : __ldg(bw.p2d_init + j * D + c);
        } else if (valid && pr3) {
          const int j = r - 27;
          v = bx.pred[blk] ? fmaf(bx.jc[blk][3 * j + 2], __ldg(bw.phi3d_w + 2 * D + c),
                                  fmaf(bx.jc[blk][3 * j + 1], __ldg(bw.phi3d_w + D + c),
                                       bx.jc[blk][3 * j] * __ldg(bw.phi3d_w + c))) + __ldg(bw.phi3d_b + c)
                           : __ldg(bw.p3d_init + j * D + c);
        }
        pos[c] = v;
      }
    } else {
#pragma unroll
      for (int c = 0; c < D; ++c) {
        float v = 0.0f;
        if (valid && r >= 1) {
          const int j = r - 1;
          v = hx.pred[blk] ? fmaf(hx.pts[blk][2 * j + 1], __ldg(hw.phi2d_w + D + c),
                                  hx.pts[blk][2 * j] * __ldg(hw.phi2d_w + c)) + __ldg(hw.phi2d_b + c)
                           : __ldg(hw.p_init + j * D + c);
        }
        pos[c] = v;
      }
    }
    self_attn(P, body ? bw.self[l] : hw.self[l], x, pos, nrows, valid);
    cross_attn(P, body ? bw.cross[l] : hw.cross[l], x, frow, valid);
    mlp(P, body ? bw.mlp[l] : hw.mlp[l], x, valid);
    const unsigned sel = body ? a.body_sel : a.hand_sel;
    if ((sel >> l) & 1u) {
      if (body) {
        body_heads(P, bx, bw, x);
        if (t < 64) {  // warp 0 -> block 0, warp 1 -> block 1
          const int b = t / 32;
          fk_warp(bx.params[b], bw.joints_rest, bx.fk[b], t % 32);
        }
        __syncthreads();
        if (t < 2 * FSB_NJ) {
          const int b = t / FSB_NJ, j = t % FSB_NJ;
          bx.kp2d[b][2 * j] = bx.cam[b][0] * bx.fk[b].tw[j][0] + bx.cam[b][1];
          bx.kp2d[b][2 * j + 1] = bx.cam[b][0] * bx.fk[b].tw[j][1] + bx.cam[b][2];
          for (int c = 0; c < 3; ++c) bx.jc[b][3 * j + c] = bx.fk[b].tw[j][c] - bx.fk[b].tw[0][c];
        }
        if (t < 2) bx.pred[t] = 1;
        __syncthreads();
        if (a.inter != nullptr && r == 0 && uvalid) {
          float* dst = a.inter + ((int64_t)unit * layers + l) * (FSB_PARAM_DIM + 3 + 44);
          for (int i = 0; i < FSB_PARAM_DIM; ++i) dst[i] = bx.params[blk][i];
          for (int i = 0; i < 3; ++i) dst[FSB_PARAM_DIM + i] = bx.cam[blk][i];
          for (int i = 0; i < 44; ++i) dst[FSB_PARAM_DIM + 3 + i] = bx.kp2d[blk][i];
        }
      } else {
        if (r == 0) {
          float y[D];
          ln_row(x, hw.norm_g, hw.norm_b, y);
          float rc[6];
          for (int o = 0; o < 6; ++o) {
            const float* W = o < 3 ? hw.head_rot_w : hw.head_cam_w;
            float acc = 0.0f;
            for (int k = 0; k < D; ++k) acc = fmaf(y[k], __ldg(W + k * 3 + o % 3), acc);
            rc[o] = acc + __ldg((o < 3 ? hw.head_rot_b : hw.head_cam_b) + o % 3);
          }
          float R[9];
          rodrigues3(rc[0], rc[1], rc[2], R);
          for (int i = 0; i < 3; ++i) {
            float q[2];
            for (int ax = 0; ax < 2; ++ax)
              q[ax] = R[3 * ax] * __ldg(hw.canon_pts + 3 * i) + R[3 * ax + 1] * __ldg(hw.canon_pts + 3 * i + 1) +
                      R[3 * ax + 2] * __ldg(hw.canon_pts + 3 * i + 2);
            hx.pts[blk][2 * i] = rc[3] * q[0] + rc[4];
            hx.pts[blk][2 * i + 1] = rc[3] * q[1] + rc[5];
          }
          hx.pred[blk] = 1;
        }
        __syncthreads();
      }
    }
  }
  // final heads and outputs
  if (body) {
    body_heads(P, bx, bw, x);
    if (uvalid && r < FSB_PARAM_DIM) {
      const float v = bx.params[blk][r];
      flag_nonfinite(a.nonfinite, v);
      a.body_params[(int64_t)unit * FSB_PARAM_DIM + r] = v;
      const bool hand_slot = (r >= 51 && r < 54) || (r >= 63 && r < 66);
      if (a.merged != nullptr && !hand_slot) a.merged[(int64_t)unit * FSB_PARAM_DIM + r] = v;
      if (r < 3) a.body_cam[(int64_t)unit * 3 + r] = bx.cam[blk][r];
    }
    // params 64..75 (rows only go to 63)
    if (uvalid && r < FSB_PARAM_DIM - 64) {
      const int o = 64 + r;
      const float v = bx.params[blk][o];
      a.body_params[(int64_t)unit * FSB_PARAM_DIM + o] = v;
      const bool hand_slot = (o >= 51 && o < 54) || (o >= 63 && o < 66);
      if (a.merged != nullptr && !hand_slot) a.merged[(int64_t)unit * FSB_PARAM_DIM + o] = v;
    }
  } else {
    if (r == 0 && uvalid) {
      float y[D];
      ln_row(x, hw.norm_g, hw.norm_b, y);
      for (int o = 0; o < 3; ++o) {
        float acc = 0.0f;
        for (int k = 0; k < D; ++k) acc = fmaf(y[k], __ldg(hw.head_rot_w + k * 3 + o), acc);
        const float v = acc + __ldg(hw.head_rot_b + o);
        flag_nonfinite(a.nonfinite, v);
        a.hand_rots[(int64_t)unit * 3 + o] = v;
        if (a.merged != nullptr)
          a.merged[(int64_t)(unit / 2) * FSB_PARAM_DIM + ((unit % 2) == 0 ? 51 : 63) + o] = v;
      }
    }
  }
  teardown(P);
}

cudaError_t init_attrs_transformer_tc() {
  cudaError_t e = cudaFuncSetAttribute(k_encoder_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM_TC);
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(k_decoders_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM_TC);
}

cudaError_t launch_encoder_tc(const float* crops, int ncrops, const EncW& w, float* feats, int* nonfinite,
                              cudaStream_t st) {
  if (ncrops == 0) return cudaSuccess;
  k_encoder_tc<<<(ncrops + 1) / 2, NTH, SMEM_TC, st>>>(crops, ncrops, w, feats, nonfinite);
  return cudaGetLastError();
}

cudaError_t launch_decoders_tc(const DecodeArgs& a, const BodyW& bw, const HandW& hw, cudaStream_t st) {
  const int n = (a.nbody + 1) / 2 + (a.nhand + 1) / 2;
  if (n == 0) return cudaSuccess;
  k_decoders_tc<<<n, NTH, SMEM_TC, st>>>(a, bw, hw);
  return cudaGetLastError();
}
