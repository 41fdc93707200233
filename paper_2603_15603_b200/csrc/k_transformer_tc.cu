// K2 / K3 on the 5th-generation tensor cores (bf16 mode).
//
// Same math as the fp32 kernels in k_transformer.cu (reference decoder.py:
// encode :231-260, _attention :172-203, _mlp :205-212, decode_body
// :284-356, decode_hand :360-410) with every GEMM on tcgen05: operands are
// bf16 in shared memory (K-major UMMA layout, tc_sm100.cuh), accumulators
// are fp32 in TMEM, and the LayerNorm / softmax / residual / ReLU
// epilogues run in fp32 registers.
//
// One CTA = 8 warps = 256 threads over 128 TMEM lanes = 128 token rows,
// organised as two 64-row blocks: two crops (encoder), two frames' body
// tokens (51 valid rows each) or two hands (4 valid rows each).  Row r is
// owned by threads r and r + 128 (warps w and w + 4 read the same TMEM lane
// quadrant): each holds 32 of the row's 64 residual-stream values in
// registers, LayerNorm sums are combined through a double-buffered shared
// exchange (one barrier per reduction), and in attention each of the two
// threads runs the softmax of a different head.  Attention of the two
// blocks is one 128 x 128 score tile whose off-diagonal block is masked to
// zero, so P.V stays a single MMA chain.  Weights (pre-packed bf16 W^T
// images) stream through two 32 KB slots with cp.async.bulk, one GEMM ahead.
#include "fsb_common.cuh"
#include "fsb_weights.h"
#include "tc_sm100.cuh"

namespace {

constexpr int D = 64, DH = 16, NTH = 256, ROWS = 128, BLK = 64, HC = 32;  // HC: columns per thread

// shared memory map (bytes)
constexpr uint32_t S_A = 0;         // 128 x 64 bf16 GEMM A operand           16 KB
constexpr uint32_t S_Q = 16384;     // 4 heads x (128 x 16) queries           16 KB
constexpr uint32_t S_K = 32768;     // 4 heads x (128 x 16) keys              16 KB
constexpr uint32_t S_VT = 49152;    // 4 heads x (16 x 128) values^T          16 KB
constexpr uint32_t S_HP = 65536;    // MLP hidden 128x256 | P 2x(128x128) | patches 128x192   64 KB
constexpr uint32_t S_W = 131072;    // 2 weight slots x 32 KB
constexpr uint32_t S_AUX = 196608;  // fp32 role scratch                      16 KB
constexpr uint32_t S_PRM = S_AUX + 16384;  // 2 slots of the per-layer TCP_* parameter block
constexpr uint32_t PRM_BYTES = TCP_FLOATS * 4;
constexpr uint32_t SMEM_TC = S_PRM + 2 * PRM_BYTES;
static_assert(SMEM_TC <= 227 * 1024, "shared memory budget");

// TMEM columns
constexpr uint32_t T_GEN = 0;   // GEMM accumulators / attention score pair
constexpr uint32_t T_O = 256;   // attention context (4 heads x 16)
constexpr uint32_t T_KV = 384;  // cross-attention K | V of the feature rows

constexpr int kMaxW = 64;

struct Shared {
  uint64_t wbar[2];
  uint64_t pbar[2];
  uint64_t mbar;
  uint32_t tmem;
  int nw;
  const uint8_t* wptr[kMaxW];
  uint32_t wbytes[kMaxW];
  float xch[2][2 * ROWS];  // row-reduction exchange, double buffered
};

#ifdef FSB_PROFILE
// cycle attribution of CTA 0 / thread 0 (build with FSB_PROFILE=1):
// [0] total, [1] MMA waits, [2] weight waits, [3] issue barriers,
// [4] row-exchange barriers
__device__ unsigned long long g_tc_prof[2][2][16];  // [role][thread 0 | thread 255][counter]
#define PROF_T0() const long long prof_t0_ = clock64()
#define PROF_ADD(i) (prof[i] += clock64() - prof_t0_)
#else
#define PROF_T0()
#define PROF_ADD(i)
#endif

// per-thread pipeline state (every thread tracks the same phases)
struct Pipe {
  Shared* sh;
  uint8_t* smem;
  uint32_t sbase;  // shared-space address of smem
  uint32_t tmem;
  uint32_t mphase;
  int wload, wuse, xc, pload, puse;
  int tid, r, h;
#ifdef FSB_PROFILE
  long long prof[16];
#endif

  // per-layer parameter block ring (TCP_* layout): thread 0 issues, every
  // thread waits on the slot it reads
  __device__ void pprefetch(const float* src) {
    if (tid == 0 && src != nullptr) {
      const int slot = pload & 1;
      tc::mbar_expect_tx(&sh->pbar[slot], PRM_BYTES);
      tc::bulk_g2s(smem + S_PRM + slot * PRM_BYTES, src, PRM_BYTES, &sh->pbar[slot]);
    }
    ++pload;
  }
  __device__ const float* pacquire() {
    const int slot = puse & 1;
    tc::mbar_wait(&sh->pbar[slot], (uint32_t)((puse >> 1) & 1));
    ++puse;
    return reinterpret_cast<const float*>(smem + S_PRM + slot * PRM_BYTES);
  }

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
    PROF_T0();
    const int slot = wuse & 1;
    tc::mbar_wait(&sh->wbar[slot], (uint32_t)((wuse >> 1) & 1));
    ++wuse;
    PROF_ADD(2);
    return sbase + S_W + slot * 32768u;
  }
  // operands written by threads -> visible to the tensor core; TMEM reads done
  __device__ void before_issue() {
    PROF_T0();
    tc::fence_async_smem();
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    PROF_ADD(3);
  }
  __device__ void commit_wait() {
    PROF_T0();
    if (tid == 0) tc::mma_commit(&sh->mbar);
    tc::mbar_wait(&sh->mbar, mphase);
    mphase ^= 1u;
    tc::fence_after();
    PROF_ADD(1);
  }
  __device__ uint32_t lane_addr(uint32_t col) const {
    return tmem + ((uint32_t)(((tid >> 5) & 3) * 32) << 16) + col;
  }
  // sum of the two threads' partials of row r (one barrier)
  __device__ float row_total(float part) {
    float* b = sh->xch[xc & 1];
    ++xc;
    b[h * ROWS + r] = part;
    PROF_T0();
    __syncthreads();
    PROF_ADD(4);
    return b[r] + b[ROWS + r];
  }
};

__device__ __forceinline__ void gemm(uint32_t a, int K, uint32_t b, int N, uint32_t dcol, uint32_t tmem) {
  const uint32_t id = tc::idesc_bf16(128, N);
  for (int k = 0; k < K; k += 16) tc::mma_bf16(tmem + dcol, tc::kmajor_desc(a, K, k), tc::kmajor_desc(b, K, k), id, k > 0);
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float* v) {
  tc::tmem_ld16(taddr, v);
  tc::tmem_ld16(taddr + 16, v + 16);
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

// 32-element sum with 8 independent partial chains
__device__ __forceinline__ float sum32(const float* v) {
  float p[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) p[i] = v[i];
#pragma unroll
  for (int c = 8; c < 32; ++c) p[c & 7] += v[c];
  return ((p[0] + p[1]) + (p[2] + p[3])) + ((p[4] + p[5]) + (p[6] + p[7]));
}

// LayerNorm (numkit.py:198-202) of row r split over the thread pair: this
// thread's 32 columns [32h, 32h + 32) normalised into y
__device__ __forceinline__ void ln_half(Pipe& P, const float* x, const float* g, const float* b, float* y) {
  const float mu = P.row_total(sum32(x)) * (1.0f / D);
  float d[HC];
#pragma unroll
  for (int c = 0; c < HC; ++c) {
    const float e = x[c] - mu;
    d[c] = e * e;
  }
  const float rstd = 1.0f / sqrtf(P.row_total(sum32(d)) * (1.0f / D) + 1e-5f);
  const int c0 = HC * P.h;
#pragma unroll
  for (int c = 0; c < HC; ++c) y[c] = fmaf((x[c] - mu) * rstd, g[c0 + c], b[c0 + c]);  // g, b: shared or global
}

__device__ __forceinline__ void ln_half_to_tile(Pipe& P, const float* x, const float* g, const float* b) {
  float y[HC];
  ln_half(P, x, g, b, y);
#pragma unroll
  for (int q = 0; q < HC; q += 8) st_row8(P.smem + S_A, P.r, HC * P.h + q, D, y + q);
}

// query columns [qcol, +64) + bias -> heads 2h, 2h+1 of the query tiles
__device__ void drain_q(Pipe& P, uint32_t qcol, const float* bq) {
  float v[HC];
  tmem_ld32(P.lane_addr(qcol + HC * P.h), v);
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    const int hd = 2 * P.h + j;
#pragma unroll
    for (int i = 0; i < 16; ++i) v[16 * j + i] += bq[16 * hd + i];
    uint8_t* tq = P.smem + S_Q + hd * 4096;
    st_row8(tq, P.r, 0, DH, v + 16 * j);
    st_row8(tq, P.r, 8, DH, v + 16 * j + 8);
  }
}

// key | value columns [kcol, +128) + bias -> key tiles and transposed values
__device__ void drain_kv(Pipe& P, uint32_t kcol, const float* bk, const float* bv) {
  float v[HC];
  tmem_ld32(P.lane_addr(kcol + HC * P.h), v);
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    const int hd = 2 * P.h + j;
#pragma unroll
    for (int i = 0; i < 16; ++i) v[16 * j + i] += bk[16 * hd + i];
    uint8_t* tk = P.smem + S_K + hd * 4096;
    st_row8(tk, P.r, 0, DH, v + 16 * j);
    st_row8(tk, P.r, 8, DH, v + 16 * j + 8);
  }
  tmem_ld32(P.lane_addr(kcol + 64 + HC * P.h), v);
  // V^T tile per head (16 x 128): row d, column = this row's key index
  const uint32_t col_off = (uint32_t)(P.r >> 3) * 128u + (uint32_t)(P.r & 7) * 2u;
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    const int hd = 2 * P.h + j;
    uint8_t* tv = P.smem + S_VT + hd * 4096 + col_off;
#pragma unroll
    for (int d = 0; d < DH; ++d) {
      const __nv_bfloat16 hv = __float2bfloat16_rn(v[16 * j + d] + bv[16 * hd + d]);
      *reinterpret_cast<__nv_bfloat16*>(tv + (d >> 3) * 2048 + (d & 7) * 16) = hv;
    }
  }
}

// softmax of head (pair + 2 h) over the first NK keys of the row's own key
// block -> P tile h, unnormalised (the context is scaled by the returned
// 1 / sum after P.V: 16 multiplies instead of 64).  NK is the number of
// valid keys (64 for encoder self-attention and cross-attention, 51 body
// tokens, 4 hand tokens), so masking is resolved at compile time.
template <int NK>
__device__ float softmax_head(Pipe& P, bool active = true) {
  static_assert(NK >= 1 && NK <= 64, "keys per block");
  constexpr int NL = NK <= 16 ? 16 : (NK <= 32 ? 32 : 64);  // TMEM columns loaded
  const int blk = P.r / BLK;
  float s[64];
  const uint32_t ta = P.lane_addr(T_GEN + 128 * P.h + 64 * blk);
  if (NL == 64) tc::tmem_ld64(ta, s);
  else if (NL == 32) tmem_ld32(ta, s);
  else tc::tmem_ld16(ta, s);
  if (!active) {  // a row outside this round: P row of zeros
#pragma unroll
    for (int q = 0; q < 16; ++q) st_row_zero8(P.smem + S_HP + P.h * 32768, P.r, 8 * q, 128);
    return 0.0f;
  }
  float m4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
  for (int k = 0; k < NK; ++k) m4[k & 3] = fmaxf(m4[k & 3], s[k]);
  constexpr float kScale = 0.25f * 1.4426950408889634f;  // f32(1/sqrt(16)) * log2(e)
  const float nms = -fmaxf(fmaxf(m4[0], m4[1]), fmaxf(m4[2], m4[3])) * kScale;
  float p4[4] = {0.0f, 0.0f, 0.0f, 0.0f};
#pragma unroll
  for (int k = 0; k < NK; ++k) {
    s[k] = ex2_approx(fmaf(s[k], kScale, nms));
    p4[k & 3] += s[k];
  }
  uint8_t* tp = P.smem + S_HP + P.h * 32768;
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    if (8 * q < NK) {
      float v[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) v[i] = (8 * q + i < NK) ? s[8 * q + i] : 0.0f;
      st_row8(tp, P.r, 64 * blk + 8 * q, 128, v);
    } else {
      st_row_zero8(tp, P.r, 64 * blk + 8 * q, 128);
    }
    st_row_zero8(tp, P.r, 64 * (1 - blk) + 8 * q, 128);
  }
  return 1.0f / ((p4[0] + p4[1]) + (p4[2] + p4[3]));
}

// softmax of head (pair + 2 h) for hand tiles: every hand's four token rows
// [4 g, 4 g + 4) attend to the same four keys (decoder.py:393-398), so a
// warp's 32 rows need the 32 key columns of its own lane quadrant; the
// row's four are picked out of them.  Same arithmetic as softmax_head<4>.
__device__ float softmax_group4(Pipe& P) {
  float s[32];
  tmem_ld32(P.lane_addr(T_GEN + 128 * P.h + 32 * (P.r >> 5)), s);
  const int g = (P.r & 31) >> 2;
  float a[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    a[k] = s[k];
#pragma unroll
    for (int gg = 1; gg < 8; ++gg) a[k] = g == gg ? s[4 * gg + k] : a[k];
  }
  constexpr float kScale = 0.25f * 1.4426950408889634f;
  const float nms = -fmaxf(fmaxf(a[0], a[1]), fmaxf(a[2], a[3])) * kScale;
  float e[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) e[k] = ex2_approx(fmaf(a[k], kScale, nms));
  uint8_t* tp = P.smem + S_HP + P.h * 32768;
  const int qk = P.r >> 3;               // 8-column chunk holding the group's keys
  const bool hi = ((P.r >> 2) & 1) != 0;  // keys in its upper half
#pragma unroll
  for (int q = 0; q < 16; ++q) {
    if (q == qk) {
      float v[8];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        v[k] = hi ? 0.0f : e[k];
        v[4 + k] = hi ? e[k] : 0.0f;
      }
      st_row8(tp, P.r, 8 * q, 128, v);
    } else {
      st_row_zero8(tp, P.r, 8 * q, 128);
    }
  }
  return 1.0f / ((e[0] + e[1]) + (e[2] + e[3]));
}

// the four heads of one attention given sQ / sK / sVt; the context is
// written as bf16 straight into the A tile of the output projection.
// Pair p of the two passes runs heads p (threads h = 0) and p + 2
// (threads h = 1), so each thread ends up owning the softmax sums of the
// two heads whose context columns [32 h, 32 h + 32) it holds.
// One round: S = Q K^T, softmax, O (+)= P V.  Rows with active == false
// contribute a zero P row, so several rounds over different key sets (the
// hand tiles' cross attention) accumulate into one context; inv keeps the
// 1 / sum of the round in which the row was active.  G4: grouped hand
// self-attention (softmax_group4).
template <int NK, bool G4 = false>
__device__ void attn_round(Pipe& P, bool active, bool accumulate, float* inv) {
  const uint32_t sq = P.sbase + S_Q, sk = P.sbase + S_K, sv = P.sbase + S_VT, sp = P.sbase + S_HP;
  const uint32_t id_s = tc::idesc_bf16(128, 128), id_o = tc::idesc_bf16(128, 16);
  P.before_issue();
  if (P.tid == 0)
    for (int j = 0; j < 2; ++j)
      tc::mma_bf16(P.tmem + T_GEN + 128 * j, tc::kmajor_desc(sq + (2 * j) * 4096, DH, 0),
                   tc::kmajor_desc(sk + (2 * j) * 4096, DH, 0), id_s, false);
  P.commit_wait();
#pragma unroll 1
  for (int pair = 0; pair < 2; ++pair) {
    const float iv = G4 ? softmax_group4(P) : softmax_head<NK>(P, active);
    if (active) inv[pair] = iv;
    P.before_issue();
    if (P.tid == 0) {
      for (int j = 0; j < 2; ++j) {
        const int hd = pair + 2 * j;
        for (int k = 0; k < 128; k += 16)
          tc::mma_bf16(P.tmem + T_O + 16 * hd, tc::kmajor_desc(sp + j * 32768, 128, k),
                       tc::kmajor_desc(sv + hd * 4096, 128, k), id_o, accumulate || k > 0);
      }
      if (pair == 0)
        for (int j = 0; j < 2; ++j)
          tc::mma_bf16(P.tmem + T_GEN + 128 * j, tc::kmajor_desc(sq + (1 + 2 * j) * 4096, DH, 0),
                       tc::kmajor_desc(sk + (1 + 2 * j) * 4096, DH, 0), id_s, false);
    }
    P.commit_wait();
  }
}

// context (scaled by the deferred 1 / sum) as bf16 into the A tile
__device__ void attn_ctx(Pipe& P, const float* inv) {
  float ctx[HC];
  tmem_ld32(P.lane_addr(T_O + HC * P.h), ctx);
#pragma unroll
  for (int c = 0; c < HC; ++c) ctx[c] *= inv[c / 16];
#pragma unroll
  for (int q = 0; q < HC; q += 8) st_row8(P.smem + S_A, P.r, HC * P.h + q, D, ctx + q);
}

template <int NK, bool G4 = false>
__device__ void attn_core(Pipe& P) {
  float inv[2];
  attn_round<NK, G4>(P, true, false, inv);
  attn_ctx(P, inv);
}

// x += Wo . ctx + bo for valid rows (ctx already in the A tile)
__device__ void out_proj(Pipe& P, const float* bo, float* x, bool valid) {
  const uint32_t w = P.acquire();
  P.before_issue();
  if (P.tid == 0) gemm(P.sbase + S_A, D, w, D, T_GEN, P.tmem);
  P.prefetch();
  P.commit_wait();
  float v[HC];
  tmem_ld32(P.lane_addr(T_GEN + HC * P.h), v);
  if (valid)
#pragma unroll
    for (int c = 0; c < HC; ++c) x[c] += v[c] + bo[HC * P.h + c];
}

// Sub-layers.  `prm` is the layer's TCP_* parameter block staged in shared
// memory (LayerNorm affine and biases); the weight images come from the ring.

// self attention: x += MHA(LN(x + pos))  (decoder.py:214-218)
template <int NK, bool G4 = false>
__device__ void self_attn(Pipe& P, const float* prm, float* x, const float* pos, bool valid) {
  float a[HC];
#pragma unroll
  for (int c = 0; c < HC; ++c) a[c] = x[c] + pos[c];
#ifdef FSB_PROFILE
  long long q0 = clock64();
#endif
  ln_half_to_tile(P, a, prm + TCP_S_LN_G, prm + TCP_S_LN_B);
#ifdef FSB_PROFILE
  long long q1 = clock64();
  P.prof[12] += q1 - q0;
#endif
  const uint32_t wq = P.acquire();
  P.before_issue();
  if (P.tid == 0) gemm(P.sbase + S_A, D, wq, 3 * D, T_GEN, P.tmem);
  P.prefetch();
  P.commit_wait();
#ifdef FSB_PROFILE
  long long q2 = clock64();
  P.prof[13] += q2 - q1;
#endif
  drain_q(P, T_GEN, prm + TCP_S_BQKV);
  drain_kv(P, T_GEN + 64, prm + TCP_S_BQKV + 64, prm + TCP_S_BQKV + 128);
#ifdef FSB_PROFILE
  long long q3 = clock64();
  P.prof[14] += q3 - q2;
#endif
  attn_core<NK, G4>(P);
#ifdef FSB_PROFILE
  P.prof[15] += clock64() - q3;
#endif
  out_proj(P, prm + TCP_S_BO, x, valid);
}

// cross attention: x += MHA(LN_q(x), LN_kv(f))  (decoder.py:220-227)
__device__ void cross_attn(Pipe& P, const float* prm, float* x, const float* frow, bool valid) {
  float f[HC];
#pragma unroll
  for (int c = 0; c < HC; c += 4) {
    const float4 v = __ldg(reinterpret_cast<const float4*>(frow + HC * P.h + c));
    f[c] = v.x; f[c + 1] = v.y; f[c + 2] = v.z; f[c + 3] = v.w;
  }
  ln_half_to_tile(P, f, prm + TCP_C_LNKV_G, prm + TCP_C_LNKV_B);
  const uint32_t wkv = P.acquire();
  P.before_issue();
  if (P.tid == 0) gemm(P.sbase + S_A, D, wkv, 2 * D, T_KV, P.tmem);
  P.prefetch();
  P.commit_wait();
  drain_kv(P, T_KV, prm + TCP_C_BQKV + 64, prm + TCP_C_BQKV + 128);
  ln_half_to_tile(P, x, prm + TCP_C_LNQ_G, prm + TCP_C_LNQ_B);
  const uint32_t wq = P.acquire();
  P.before_issue();
  if (P.tid == 0) gemm(P.sbase + S_A, D, wq, D, T_GEN, P.tmem);
  P.prefetch();
  P.commit_wait();
  drain_q(P, T_GEN, prm + TCP_C_BQKV);
  attn_core<BLK>(P);
  out_proj(P, prm + TCP_C_BO, x, valid);
}

// cross attention of a hand tile (decoder.py:220-227 per hand): the queries
// once, then one round per pair of hand slots (2c, 2c + 1): LN_kv of their
// two crops' feature rows (block b of the 128 rows = slot 2c + b), K | V,
// and an attention round in which only the slots' token rows are active.
// Weight images in order t_q, t_kv (kept in its ring slot for all rounds),
// t_o.
__device__ void cross_attn_hands(Pipe& P, const float* prm, float* x, const DecodeArgs& a, int hand0, int nslots,
                                 bool valid) {
  ln_half_to_tile(P, x, prm + TCP_C_LNQ_G, prm + TCP_C_LNQ_B);
  const uint32_t wq = P.acquire();
  P.before_issue();
  if (P.tid == 0) gemm(P.sbase + S_A, D, wq, D, T_GEN, P.tmem);
  P.prefetch();
  P.commit_wait();
  drain_q(P, T_GEN, prm + TCP_C_BQKV);
  const uint32_t wkv = P.acquire();
  const int blk = P.r / BLK, rb = P.r % BLK;
  const int nr = (nslots + 1) / 2;
  float inv[2] = {0.0f, 0.0f};
#pragma unroll 1
  for (int c = 0; c < nr; ++c) {
    const int slot = 2 * c + blk;
    float f[HC];
    if (slot < nslots) {
      const int u = hand0 + slot;
      const int crop = a.hand_feat_first + (u / 2) * a.body_feat_stride + (u % 2);
      const float* frow = a.feats + ((int64_t)crop * 64 + rb) * D + HC * P.h;
#pragma unroll
      for (int q = 0; q < HC; q += 4) {
        const float4 v = __ldg(reinterpret_cast<const float4*>(frow + q));
        f[q] = v.x; f[q + 1] = v.y; f[q + 2] = v.z; f[q + 3] = v.w;
      }
    } else {
#pragma unroll
      for (int q = 0; q < HC; ++q) f[q] = 0.0f;
    }
    ln_half_to_tile(P, f, prm + TCP_C_LNKV_G, prm + TCP_C_LNKV_B);
    P.before_issue();
    if (P.tid == 0) gemm(P.sbase + S_A, D, wkv, 2 * D, T_KV, P.tmem);
    if (c == 0) P.prefetch();  // t_o into the slot t_q has left
    P.commit_wait();
    drain_kv(P, T_KV, prm + TCP_C_BQKV + 64, prm + TCP_C_BQKV + 128);
    attn_round<BLK>(P, (rb >> 2) == c, c > 0, inv);
  }
  attn_ctx(P, inv);
  out_proj(P, prm + TCP_C_BO, x, valid);
}

// MLP: x += W2 relu(W1 LN(x) + b1) + b2  (decoder.py:205-212)
__device__ void mlp(Pipe& P, const float* prm, float* x, bool valid) {
  ln_half_to_tile(P, x, prm + TCP_M_LN_G, prm + TCP_M_LN_B);
  const uint32_t w1 = P.acquire();
  P.before_issue();
  if (P.tid == 0) gemm(P.sbase + S_A, D, w1, 4 * D, T_GEN, P.tmem);
  P.prefetch();
  P.commit_wait();
  uint8_t* th = P.smem + S_HP;
#pragma unroll 1
  for (int q = 0; q < 2; ++q) {
    const int c0 = 128 * P.h + 64 * q;
    float v[64];
    tc::tmem_ld64(P.lane_addr(T_GEN + c0), v);
#pragma unroll
    for (int i = 0; i < 64; ++i) v[i] = fmaxf(v[i] + prm[TCP_M_B1 + c0 + i], 0.0f);
#pragma unroll
    for (int i = 0; i < 64; i += 8) st_row8(th, P.r, c0 + i, 4 * D, v + i);
  }
  const uint32_t w2 = P.acquire();
  P.before_issue();
  if (P.tid == 0) gemm(P.sbase + S_HP, 4 * D, w2, D, T_GEN, P.tmem);
  P.prefetch();
  P.commit_wait();
  float v[HC];
  tmem_ld32(P.lane_addr(T_GEN + HC * P.h), v);
  if (valid)
#pragma unroll
    for (int c = 0; c < HC; ++c) x[c] += v[c] + prm[TCP_M_B2 + HC * P.h + c];
}

__device__ void setup(Pipe& P, Shared& sh, uint8_t* smem) {
  P.sh = &sh;
  P.smem = smem;
  P.sbase = tc::smem_u32(smem);
  P.tid = threadIdx.x;
  P.r = threadIdx.x & (ROWS - 1);
  P.h = threadIdx.x / ROWS;
  P.mphase = 0;
  P.wload = 0;
  P.wuse = 0;
  P.xc = 0;
  P.pload = 0;
  P.puse = 0;
#ifdef FSB_PROFILE
  for (int i = 0; i < 16; ++i) P.prof[i] = 0;
  P.prof[0] = -clock64();
#endif
  if (P.tid == 0) {
    tc::mbar_init(&sh.wbar[0], 1);
    tc::mbar_init(&sh.wbar[1], 1);
    tc::mbar_init(&sh.pbar[0], 1);
    tc::mbar_init(&sh.pbar[1], 1);
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

__device__ void teardown(Pipe& P, int role) {
  tc::fence_before();
  __syncthreads();
  if (P.tid < 32) tc::tmem_dealloc(P.tmem, 512);
#ifdef FSB_PROFILE
  P.prof[0] += clock64();
  if ((P.tid == 0 || P.tid == NTH - 1) && blockIdx.x == 0)
    for (int i = 0; i < 16; ++i) g_tc_prof[role][P.tid ? 1 : 0][i] = (unsigned long long)P.prof[i];
#else
  (void)role;
#endif
}

}  // namespace

// ===========================================================================
// encoder: grid = ceil(ncrops / 2); block f of CTA b encodes crop 2b + f
// ===========================================================================
__global__ void __launch_bounds__(NTH, 1) k_encoder_tc(const float* __restrict__ crops, int ncrops, EncW w,
                                                       float* __restrict__ feats, int* nonfinite) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ Shared sh;
  const int t = threadIdx.x;
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
  if (w.layers > 0) P.pprefetch(w.tc_params[0]);
  const int blk = P.r / BLK, p = P.r % BLK;
  const int crop = 2 * blockIdx.x + blk;
  const bool valid = crop < ncrops;

  // patchify (decoder.py:247-248): this thread packs image rows iy in
  // [4h, 4h + 4) of patch p into the K = 192 tile (k = iy*24 + ix*3 + c)
  {
    uint8_t* tile = smem + S_HP;
    const int py = p / 8, px = p % 8;
    const float* src = crops + (int64_t)(valid ? crop : 0) * 64 * 64 * 3;
#pragma unroll 1
    for (int iy = 4 * P.h; iy < 4 * P.h + 4; ++iy) {
      const float* row = src + ((py * 8 + iy) * 64 + px * 8) * 3;
#pragma unroll
      for (int q = 0; q < 3; ++q) {
        float v[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) v[i] = valid ? __ldg(row + 8 * q + i) : 0.0f;
        st_row8(tile, P.r, iy * 24 + 8 * q, 192, v);
      }
    }
  }
  float x[HC];
  {
    const uint32_t wp = P.acquire();
    P.before_issue();
    if (t == 0) gemm(P.sbase + S_HP, 192, wp, D, T_GEN, P.tmem);
    P.prefetch();
    P.commit_wait();
    float v[HC];
    tmem_ld32(P.lane_addr(T_GEN + HC * P.h), v);
#pragma unroll
    for (int i = 0; i < HC; ++i) {
      const int c = HC * P.h + i;
      x[i] = valid ? (v[i] + __ldg(w.patch_b + c)) + __ldg(w.pos + p * D + c) : 0.0f;
    }
  }
  float zero[HC];
#pragma unroll
  for (int c = 0; c < HC; ++c) zero[c] = 0.0f;
  for (int l = 0; l < w.layers; ++l) {
    const float* prm = P.pacquire();
    __syncthreads();  // every thread is past layer l - 1: its slot may be refilled
    if (l + 1 < w.layers) P.pprefetch(w.tc_params[l + 1]);
    self_attn<BLK>(P, prm, x, zero, valid);
    mlp(P, prm, x, valid);
  }
  float y[HC];
  ln_half(P, x, w.norm_g, w.norm_b, y);
  if (valid) {
    float* out = feats + ((int64_t)crop * 64 + p) * D + HC * P.h;
    float bad = 0.0f;
#pragma unroll
    for (int c = 0; c < HC; c += 4) {
      bad += y[c] + y[c + 1] + y[c + 2] + y[c + 3];
      *reinterpret_cast<float4*>(out + c) = make_float4(y[c], y[c + 1], y[c + 2], y[c + 3]);
    }
    flag_nonfinite(nonfinite, bad);
  }
  teardown(P, 0);
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
// Hand tiles hold kHandsPerCta hands: slot i sits in row block i % 2, rows
// 64 (i % 2) + 4 (i / 2) + token, so the two slots of a cross-attention
// round (2c, 2c + 1) use key blocks 0 and 1 and every warp sees one.
#ifndef FSB_HANDS_PER_CTA
#define FSB_HANDS_PER_CTA 8
#endif
constexpr int kHandsPerCta = FSB_HANDS_PER_CTA;
static_assert(kHandsPerCta >= 2 && kHandsPerCta <= 32 && kHandsPerCta % 2 == 0, "hand slots per tile");
struct HandAux {
  float t0[kHandsPerCta][D];
  float rc[kHandsPerCta][8];   // rots[3], cams[3]
  float pts[kHandsPerCta][6];  // 3 x (x, y) projected canonical points
  int pred;
};
static_assert(sizeof(BodyAux) <= 16384 && sizeof(HandAux) <= 16384, "aux scratch");

// LN(token 0) -> head params / camera of both blocks (decoder.py:264-272)
__device__ void body_heads(Pipe& P, BodyAux& ax, const BodyW& w, const float* x) {
  float y[HC];
  ln_half(P, x, w.norm_g, w.norm_b, y);
  const int blk = P.r / BLK;
  if (P.r % BLK == 0)
#pragma unroll
    for (int c = 0; c < HC; ++c) ax.t0[blk][HC * P.h + c] = y[c];
  __syncthreads();
  {
    const int b = P.tid / 128, o = P.tid % 128;  // one head output per thread
    if (o < 79) {
      const bool is_p = o < FSB_PARAM_DIM;
      const float* W = is_p ? w.head_params_w : w.head_cam_w;
      const int n = is_p ? FSB_PARAM_DIM : 3, oo = is_p ? o : o - FSB_PARAM_DIM;
      float acc[4] = {0.0f, 0.0f, 0.0f, 0.0f};
#pragma unroll
      for (int k = 0; k < D; ++k) acc[k & 3] = fmaf(ax.t0[b][k], __ldg(W + k * n + oo), acc[k & 3]);
      const float v = (acc[0] + acc[1]) + (acc[2] + acc[3]);
      if (is_p)
        ax.params[b][oo] = v + __ldg(w.head_params_b + oo);
      else
        ax.cam[b][oo] = v + __ldg(w.head_cam_b + oo);
    }
  }
  __syncthreads();
}

// LN(token 0) -> hand rotation / camera of every slot (decoder.py:384-391)
__device__ void hand_heads(Pipe& P, HandAux& ax, const HandW& w, const float* x) {
  float y[HC];
  ln_half(P, x, w.norm_g, w.norm_b, y);
  const int slot = 2 * ((P.r % BLK) >> 2) + P.r / BLK;
  if ((P.r & 3) == 0 && slot < kHandsPerCta)
#pragma unroll
    for (int c = 0; c < HC; ++c) ax.t0[slot][HC * P.h + c] = y[c];
  __syncthreads();
  if (P.tid < 6 * kHandsPerCta) {
    const int b = P.tid / 6, o = P.tid % 6;
    const float* W = o < 3 ? w.head_rot_w : w.head_cam_w;
    float acc[4] = {0.0f, 0.0f, 0.0f, 0.0f};
#pragma unroll
    for (int k = 0; k < D; ++k) acc[k & 3] = fmaf(ax.t0[b][k], __ldg(W + k * 3 + o % 3), acc[k & 3]);
    ax.rc[b][o] = (acc[0] + acc[1]) + (acc[2] + acc[3]) + __ldg((o < 3 ? w.head_rot_b : w.head_cam_b) + o % 3);
  }
  __syncthreads();
}

__global__ void __launch_bounds__(NTH, 1) k_decoders_tc(DecodeArgs a, BodyW bw, HandW hw) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ Shared sh;
  const int t = threadIdx.x;
  const int nbc = (a.nbody + 1) / 2;
  const bool body = (int)blockIdx.x < nbc;
  const int layers = body ? bw.layers : hw.layers;
  if (t == 0) {
    int n = 0;
    for (int l = 0; l < layers; ++l) {
      const AttnW& s = body ? bw.self[l] : hw.self[l];
      const AttnW& c = body ? bw.cross[l] : hw.cross[l];
      const MlpW& m = body ? bw.mlp[l] : hw.mlp[l];
      sh.wptr[n] = s.t_qkv; sh.wbytes[n++] = 3 * D * D * 2;
      sh.wptr[n] = s.t_o;   sh.wbytes[n++] = D * D * 2;
      if (body) {
        sh.wptr[n] = c.t_kv;  sh.wbytes[n++] = 2 * D * D * 2;
        sh.wptr[n] = c.t_q;   sh.wbytes[n++] = D * D * 2;
      } else {  // cross_attn_hands: queries first
        sh.wptr[n] = c.t_q;   sh.wbytes[n++] = D * D * 2;
        sh.wptr[n] = c.t_kv;  sh.wbytes[n++] = 2 * D * D * 2;
      }
      sh.wptr[n] = c.t_o;   sh.wbytes[n++] = D * D * 2;
      sh.wptr[n] = m.t_w1;  sh.wbytes[n++] = 4 * D * D * 2;
      sh.wptr[n] = m.t_w2;  sh.wbytes[n++] = 4 * D * D * 2;
    }
    sh.nw = n;
  }
  __syncthreads();
  Pipe P;
  setup(P, sh, smem);
  if (layers > 0) P.pprefetch(body ? bw.tc_params[0] : hw.tc_params[0]);
  const int r = P.r, blk = r / BLK, c0 = HC * P.h;
  // body: frame 2 x + blk, token rb; hand: slot hs = 2 (r % 64 / 4) + blk, token rb
  const int hand0 = kHandsPerCta * ((int)blockIdx.x - nbc);
  const int nslots = body ? 0 : min(kHandsPerCta, a.nhand - hand0);
  const int hs = 2 * ((r % BLK) >> 2) + blk;
  const int rb = body ? r % BLK : (r & 3);
  const bool valid = body ? (2 * (int)blockIdx.x + blk < a.nbody && rb < 51) : hs < nslots;
  const int unit = body ? 2 * blockIdx.x + blk : 0;  // frame index (body tiles)

  // feature row of this thread for the body's cross attention
  const int crop = (body && unit < a.nbody ? unit : 0) * a.body_feat_stride;
  const float* frow = a.feats + ((int64_t)crop * 64 + (r % BLK)) * D;

  float x[HC], pos[HC];
  BodyAux& bx = *reinterpret_cast<BodyAux*>(smem + S_AUX);
  HandAux& hx = *reinterpret_cast<HandAux*>(smem + S_AUX);
  if (body) {
    // tokens = token_init, rows 1..4 += prompt_box(prompt)  (decoder.py:287-293)
    for (int i = 0; i < 2; ++i) {
      const int idx = 2 * t + i, b = idx / (4 * D), o = idx % (4 * D);
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
    for (int c = 0; c < HC; ++c) {
      float v = valid ? __ldg(bw.token_init + rb * D + c0 + c) : 0.0f;
      if (valid && rb >= 1 && rb < 5) v += bx.boxtok[blk][(rb - 1) * D + c0 + c];
      x[c] = v;
    }
  } else {
#pragma unroll
    for (int c = 0; c < HC; ++c) x[c] = valid ? __ldg(hw.token_init + rb * D + c0 + c) : 0.0f;
    if (t == 0) hx.pred = 0;
  }
  __syncthreads();

#ifdef FSB_PROFILE
  P.prof[8] += clock64() + P.prof[0];  // setup: kernel start (prof[0] = -start) -> layer loop
  long long tpos;
#endif
  for (int l = 0; l < layers; ++l) {
#ifdef FSB_PROFILE
    tpos = clock64();
#endif
    // positional terms of the self-attention input (decoder.py:300-303,
    // :397-398).  They change only when a prediction has been made, so they
    // are kept in registers and recomputed at layer 0 and after each
    // selected layer, with 16-byte loads of this thread's 32 columns.
    const unsigned psel = body ? a.body_sel : a.hand_sel;
    if (l == 0 || ((psel >> (l - 1)) & 1u)) {
#pragma unroll
      for (int i = 0; i < HC; ++i) pos[i] = 0.0f;
      int j = -1, kind = 0;  // kind 1: 2-D keypoint row, 2: 3-D joint row
      if (valid) {
        if (body) {
          if (rb >= 5 && rb < 27) j = rb - 5, kind = 1;
          else if (rb >= 27 && rb < 49) j = rb - 27, kind = 2;
        } else if (rb >= 1) {
          j = rb - 1, kind = 1;
        }
      }
      const int pred = body ? bx.pred[blk] : hx.pred;
      if (kind != 0 && !pred) {
        const float* init = body ? (kind == 1 ? bw.p2d_init : bw.p3d_init) : hw.p_init;
        const float4* src = reinterpret_cast<const float4*>(init + j * D + c0);
#pragma unroll
        for (int q = 0; q < HC / 4; ++q) {
          const float4 v = __ldg(src + q);
          pos[4 * q] = v.x; pos[4 * q + 1] = v.y; pos[4 * q + 2] = v.z; pos[4 * q + 3] = v.w;
        }
      } else if (kind == 1) {
        const float* w = body ? bw.phi2d_w : hw.phi2d_w;
        const float* bb = body ? bw.phi2d_b : hw.phi2d_b;
        const float k0 = body ? bx.kp2d[blk][2 * j] : hx.pts[hs][2 * j];
        const float k1 = body ? bx.kp2d[blk][2 * j + 1] : hx.pts[hs][2 * j + 1];
#pragma unroll
        for (int q = 0; q < HC / 4; ++q) {
          const float4 w0 = __ldg(reinterpret_cast<const float4*>(w + c0) + q);
          const float4 w1 = __ldg(reinterpret_cast<const float4*>(w + D + c0) + q);
          const float4 b4 = __ldg(reinterpret_cast<const float4*>(bb + c0) + q);
          pos[4 * q] = fmaf(k1, w1.x, k0 * w0.x) + b4.x;
          pos[4 * q + 1] = fmaf(k1, w1.y, k0 * w0.y) + b4.y;
          pos[4 * q + 2] = fmaf(k1, w1.z, k0 * w0.z) + b4.z;
          pos[4 * q + 3] = fmaf(k1, w1.w, k0 * w0.w) + b4.w;
        }
      } else if (kind == 2) {
        const float g0 = bx.jc[blk][3 * j], g1 = bx.jc[blk][3 * j + 1], g2 = bx.jc[blk][3 * j + 2];
#pragma unroll
        for (int q = 0; q < HC / 4; ++q) {
          const float4 w0 = __ldg(reinterpret_cast<const float4*>(bw.phi3d_w + c0) + q);
          const float4 w1 = __ldg(reinterpret_cast<const float4*>(bw.phi3d_w + D + c0) + q);
          const float4 w2 = __ldg(reinterpret_cast<const float4*>(bw.phi3d_w + 2 * D + c0) + q);
          const float4 b4 = __ldg(reinterpret_cast<const float4*>(bw.phi3d_b + c0) + q);
          pos[4 * q] = fmaf(g2, w2.x, fmaf(g1, w1.x, g0 * w0.x)) + b4.x;
          pos[4 * q + 1] = fmaf(g2, w2.y, fmaf(g1, w1.y, g0 * w0.y)) + b4.y;
          pos[4 * q + 2] = fmaf(g2, w2.z, fmaf(g1, w1.z, g0 * w0.z)) + b4.z;
          pos[4 * q + 3] = fmaf(g2, w2.w, fmaf(g1, w1.w, g0 * w0.w)) + b4.w;
        }
      }
    }
    const float* prm = P.pacquire();
    __syncthreads();  // every thread is past layer l - 1: its slot may be refilled
    if (l + 1 < layers) P.pprefetch(body ? bw.tc_params[l + 1] : hw.tc_params[l + 1]);
#ifdef FSB_PROFILE
    long long ts0 = clock64();
    P.prof[9] += ts0 - tpos;
#endif
    if (body)
      self_attn<51>(P, prm, x, pos, valid);
    else
      self_attn<4, true>(P, prm, x, pos, valid);
#ifdef FSB_PROFILE
    long long ts1 = clock64();
    P.prof[5] += ts1 - ts0;
#endif
    if (body)
      cross_attn(P, prm, x, frow, valid);
    else
      cross_attn_hands(P, prm, x, a, hand0, nslots, valid);
#ifdef FSB_PROFILE
    long long ts2 = clock64();
    P.prof[6] += ts2 - ts1;
#endif
    mlp(P, prm, x, valid);
#ifdef FSB_PROFILE
    long long ts3 = clock64();
    P.prof[7] += ts3 - ts2;
#endif
    const unsigned sel = body ? a.body_sel : a.hand_sel;
    if ((sel >> l) & 1u) {
      if (body) {
        // intermediate prediction: heads -> FK -> kp2d / centred joints
        body_heads(P, bx, bw, x);
#ifdef FSB_PROFILE
        long long th = clock64();
        P.prof[10] += th - ts3;
#endif
        if (t < 64) fk_warp<true>(bx.params[t / 32], bw.joints_rest, bx.fk[t / 32], t % 32);
        __syncthreads();
#ifdef FSB_PROFILE
        P.prof[11] += clock64() - th;
#endif
        if (t < 2 * FSB_NJ) {
          const int b = t / FSB_NJ, j = t % FSB_NJ;
          bx.kp2d[b][2 * j] = bx.cam[b][0] * bx.fk[b].tw[j][0] + bx.cam[b][1];
          bx.kp2d[b][2 * j + 1] = bx.cam[b][0] * bx.fk[b].tw[j][1] + bx.cam[b][2];
          for (int c = 0; c < 3; ++c) bx.jc[b][3 * j + c] = bx.fk[b].tw[j][c] - bx.fk[b].tw[0][c];
        }
        if (t < 2) bx.pred[t] = 1;
        __syncthreads();
        if (a.inter != nullptr && t < 2 * 123) {
          const int b = t / 123, i = t % 123, u = 2 * blockIdx.x + b;
          if (u < a.nbody) {
            float* dst = a.inter + ((int64_t)u * layers + l) * (FSB_PARAM_DIM + 3 + 44);
            dst[i] = i < FSB_PARAM_DIM ? bx.params[b][i]
                                       : (i < FSB_PARAM_DIM + 3 ? bx.cam[b][i - FSB_PARAM_DIM]
                                                                : bx.kp2d[b][i - FSB_PARAM_DIM - 3]);
          }
        }
      } else {
        // canonical points through the predicted rotation (decoder.py:399-409)
        hand_heads(P, hx, hw, x);
        if (t < kHandsPerCta) {
          const float* rc = hx.rc[t];
          float R[9];
          rodrigues3<true>(rc[0], rc[1], rc[2], R);
          for (int i = 0; i < 3; ++i) {
            float q[2];
            for (int ax = 0; ax < 2; ++ax)
              q[ax] = R[3 * ax] * __ldg(hw.canon_pts + 3 * i) + R[3 * ax + 1] * __ldg(hw.canon_pts + 3 * i + 1) +
                      R[3 * ax + 2] * __ldg(hw.canon_pts + 3 * i + 2);
            hx.pts[t][2 * i] = rc[3] * q[0] + rc[4];
            hx.pts[t][2 * i + 1] = rc[3] * q[1] + rc[5];
          }
        }
        if (t == 0) hx.pred = 1;
        __syncthreads();
      }
    }
  }
#ifdef FSB_PROFILE
  long long tfin = clock64();
#endif
  // final heads and outputs
  if (body) {
    body_heads(P, bx, bw, x);
    if (t < 2 * FSB_PARAM_DIM) {
      const int b = t / FSB_PARAM_DIM, o = t % FSB_PARAM_DIM, u = 2 * blockIdx.x + b;
      if (u < a.nbody) {
        const float v = bx.params[b][o];
        flag_nonfinite(a.nonfinite, v);
        a.body_params[(int64_t)u * FSB_PARAM_DIM + o] = v;
        const bool hand_slot = (o >= 51 && o < 54) || (o >= 63 && o < 66);
        if (a.merged != nullptr && !hand_slot) a.merged[(int64_t)u * FSB_PARAM_DIM + o] = v;
        if (o < 3) a.body_cam[(int64_t)u * 3 + o] = bx.cam[b][o];
      }
    }
  } else {
    hand_heads(P, hx, hw, x);
    if (t < 3 * kHandsPerCta) {
      const int b = t / 3, o = t % 3, u = hand0 + b;
      if (b < nslots) {
        const float v = hx.rc[b][o];
        flag_nonfinite(a.nonfinite, v);
        a.hand_rots[(int64_t)u * 3 + o] = v;
        if (a.merged != nullptr) a.merged[(int64_t)(u / 2) * FSB_PARAM_DIM + ((u % 2) == 0 ? 51 : 63) + o] = v;
      }
    }
  }
#ifdef FSB_PROFILE
  P.prof[8] += clock64() - tfin;
#endif
  teardown(P, 1);
}

// debug export of the FSB_PROFILE cycle counters (not part of the public ABI)
extern "C" int fsb_debug_tc_profile(unsigned long long* out32) {
#ifdef FSB_PROFILE
  return cudaMemcpyFromSymbol(out32, g_tc_prof, sizeof(unsigned long long) * 64) == cudaSuccess ? 0 : 4;
#else
  for (int i = 0; i < 64; ++i) out32[i] = 0;
  return 3;
#endif
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
  const int n = (a.nbody + 1) / 2 + (a.nhand + kHandsPerCta - 1) / kHandsPerCta;
  if (n == 0) return cudaSuccess;
  k_decoders_tc<<<n, NTH, SMEM_TC, st>>>(a, bw, hw);
  return cudaGetLastError();
}
