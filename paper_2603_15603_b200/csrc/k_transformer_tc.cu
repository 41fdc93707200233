// K2 / K3 on the 5th-generation tensor cores (bf16 mode).
//
// Same math as the fp32 kernels in k_transformer.cu (reference decoder.py:
// encode :231-260, _attention :172-203, _mlp :205-212, decode_body
// :284-356, decode_hand :360-410) with every GEMM on tcgen05: operands are
// bf16 in shared memory (K-major UMMA layout, tc_sm100.cuh) or in TMEM,
// accumulators are fp32 in TMEM, and the LayerNorm / softmax / residual /
// ReLU epilogues run in fp32 registers.
//
// A tile = 128 token rows = 128 TMEM lanes, organised as two 64-row blocks:
// two crops (encoder), two frames' body tokens (51 valid rows each) or
// kHandsPerCta hands (4 rows each).  One CTA runs TWO independent tiles
// ("groups" of 8 warps, 256 threads, 256 TMEM columns each) so that one
// group's element-wise phases overlap the other's tensor-core, TMEM and
// barrier latencies: the decoder is a long serial chain of small GEMMs and
// one tile alone leaves the SM mostly idle.  The groups share the weight
// stream: pre-packed bf16 W^T images flow through a two-slot ring filled by
// cp.async.bulk, and a slot is refilled by whichever group releases it last.
//
// Within a group, row r is owned by threads r and r + 128 (warps w and w + 4
// read the same TMEM lane quadrant): each holds 32 of the row's 64
// residual-stream values in registers; LayerNorm sums are combined through a
// double-buffered shared exchange (one group barrier per reduction).
// Attention runs two heads at a time: S = Q K^T for both (2 x 128 TMEM
// columns), the softmax writes P as packed bf16 back over S, and P.V reads P
// straight from TMEM (tcgen05.mma with A in TMEM).  The MLP hidden layer is
// likewise packed in place and read by the second GEMM from TMEM, so no
// 128 x 256 operand ever goes through shared memory.
#include <cstdlib>

#include "fsb_common.cuh"
#include "fsb_weights.h"
#include "tc_sm100.cuh"

namespace {

constexpr int D = 64, DH = 16, GT = 256, NG = 2, NTH = NG * GT, ROWS = 128, BLK = 64, HC = 32;

// shared memory map (bytes).  Per group g at g * S_GROUP:
constexpr uint32_t S_A = 0;       // 128 x 64 bf16 GEMM A operand / attention context    16 KB
constexpr uint32_t S_Q = 16384;   // 4 heads x (128 x 16) queries                        16 KB
constexpr uint32_t S_K = 32768;   // 4 heads x (128 x 16) keys                           16 KB
constexpr uint32_t S_VT = 49152;  // 4 heads x (16 x 128) values^T                       16 KB
constexpr uint32_t S_GROUP = 65536;
// (encoder: the patch operand, 128 x 192 bf16 = 48 KB, spans S_A..S_K)
// shared by both groups:
constexpr uint32_t S_W = NG * S_GROUP;             // 2 weight slots x 32 KB
constexpr uint32_t W_SLOT = 32768;
constexpr uint32_t S_PRM = S_W + 2 * W_SLOT;        // 2 slots of the per-layer TCP_* parameter block
constexpr uint32_t PRM_BYTES = TCP_FLOATS * 4;
constexpr uint32_t S_AUX = S_PRM + 2 * PRM_BYTES;   // per group role scratch
constexpr uint32_t AUX_BYTES = 7168;
constexpr uint32_t SMEM_TC = S_AUX + NG * AUX_BYTES;
static_assert(SMEM_TC + 6 * 1024 <= 227 * 1024, "shared memory budget");

// TMEM: 512 columns, group g at 256 g.  Within a group:
//   [0, 256)  GEMM accumulators (QKV 192, KV 128, W1 256, out 64) and the
//             attention score pair (head j of the pair at 128 j; P packed
//             over its first 64 columns)
//   [64, 96)  P.V output of the pair (outside both P regions)
constexpr uint32_t T_GEN = 0;
constexpr uint32_t T_PV = 64;

struct alignas(16) Shared {
  TcStream tab;         // this role's weight stream (copied from global by setup)
  uint64_t wbar[2];     // weight slot full
  uint64_t pbar[2];     // parameter slot full
  uint64_t mbar[NG];    // per-group MMA completion
  uint64_t kvb[NG][3];  // per-group cross-attention K / V stages (body: [0] one 32 KB image per layer)
  uint32_t tmem;
  unsigned wrel[2];     // releases of each weight slot (monotonic)
  unsigned prel[2];     // releases of each parameter slot
  unsigned nact;        // groups of this CTA with work (1 or 2): releases per slot reuse
  float xch[NG][2][2 * ROWS];  // row-reduction exchange, per group, double buffered
};
static_assert(sizeof(TcStream) % 16 == 0, "vector copy of the weight stream table");

#ifdef FSB_PROFILE
// cycle attribution of CTA 0 / group 0 (build with FSB_PROFILE=1):
// [0] total, [1] MMA waits, [2] weight waits, [3] issue barriers,
// [4] row-exchange barriers, [5..] per-phase (see the kernels)
__device__ unsigned long long g_tc_prof[3][2][16];  // [encoder | body | hand][thread 0 | thread 255][counter]
#define PROF_T0() const long long prof_t0_ = clock64()
#define PROF_ADD(i) (prof[i] += clock64() - prof_t0_)
#else
#define PROF_T0()
#define PROF_ADD(i)
#endif

// per-thread pipeline state (every thread of a group tracks the same phases)
struct Pipe {
  Shared* sh;
  uint8_t* smem;   // this group's region
  uint8_t* sall;   // CTA shared base
  uint32_t sbase;  // shared-space address of this group's region
  uint32_t wbase;  // shared-space address of the weight ring
  uint32_t tmem;   // this group's TMEM base
  uint32_t mphase;
  int wuse, xc, puse;
  int kvuse;  // cross-attention K / V stages consumed (kvb parity)
  int g, tid, r, h;
#ifdef FSB_PROFILE
  long long prof[16];
#endif

  __device__ void sync() const { asm volatile("bar.sync %0, %1;\n" ::"r"(1 + g), "r"(GT) : "memory"); }

  // weight ring: image i lives in slot i & 1.  The last of the two groups to
  // release image i - 1 loads image i + 1 into its slot.
  __device__ void load_image(int i) {
    if (i < sh->tab.nw) {
      const int slot = i & 1;
      tc::mbar_expect_tx(&sh->wbar[slot], sh->tab.wbytes[i]);
      tc::bulk_g2s(sall + S_W + slot * W_SLOT, sh->tab.wptr[i], sh->tab.wbytes[i], &sh->wbar[slot]);
    }
  }
  __device__ uint32_t acquire() {  // wait for the next weight image; returns its address
    PROF_T0();
    const int slot = wuse & 1;
    tc::mbar_wait(&sh->wbar[slot], (uint32_t)((wuse >> 1) & 1));
    ++wuse;
    PROF_ADD(2);
    return wbase + slot * W_SLOT;
  }
  // called once per acquired image, after the GEMM that reads it has been
  // issued: image wuse - 2's GEMM has completed by then
  __device__ void prefetch() {
    const int done = wuse - 2;
    if (done >= 0 && tid == 0) {
      const unsigned prior = atomicAdd(&sh->wrel[done & 1], 1u);
      if ((prior % sh->nact) == sh->nact - 1) load_image(done + 2);
    }
  }

  // per-layer parameter blocks: same protocol, one block per layer
  __device__ void load_prm(int l) {
    if (l < sh->tab.nprm) {
      const int slot = l & 1;
      tc::mbar_expect_tx(&sh->pbar[slot], PRM_BYTES);
      tc::bulk_g2s(sall + S_PRM + slot * PRM_BYTES, sh->tab.pptr[l], PRM_BYTES, &sh->pbar[slot]);
    }
  }
  __device__ const float* pacquire() {
    const int slot = puse & 1;
    tc::mbar_wait(&sh->pbar[slot], (uint32_t)((puse >> 1) & 1));
    ++puse;
    return reinterpret_cast<const float*>(sall + S_PRM + slot * PRM_BYTES);
  }
  // every thread of the group is past layer puse - 2 (call after a group
  // barrier at the start of layer puse - 1)
  __device__ void prelease() {
    const int done = puse - 2;
    if (done >= 0 && tid == 0) {
      const unsigned prior = atomicAdd(&sh->prel[done & 1], 1u);
      if ((prior % sh->nact) == sh->nact - 1) load_prm(done + 2);
    }
  }

  // operands written by threads -> visible to the tensor core; TMEM reads done
  __device__ void before_issue() {
    PROF_T0();
    tc::fence_async_smem();
    tc::fence_before();
    sync();
    tc::fence_after();
    PROF_ADD(3);
  }
  __device__ void commit_wait() {
    PROF_T0();
    if (tid == 0) tc::mma_commit(&sh->mbar[g]);
    tc::mbar_wait(&sh->mbar[g], mphase);
    mphase ^= 1u;
    tc::fence_after();
    PROF_ADD(1);
  }
  __device__ uint32_t lane_addr(uint32_t col) const {
    return tmem + ((uint32_t)(((tid >> 5) & 3) * 32) << 16) + col;
  }
  // sum of the two threads' partials of row r (one group barrier)
  __device__ float row_total(float part) {
    float* b = sh->xch[g][xc & 1];
    ++xc;
    b[h * ROWS + r] = part;
    PROF_T0();
    sync();
    PROF_ADD(4);
    return b[r] + b[ROWS + r];
  }
};

__device__ __forceinline__ void gemm(uint32_t a, int K, uint32_t b, int N, uint32_t dcol, uint32_t tmem) {
  const uint32_t id = tc::idesc_bf16(128, N);
  for (int k = 0; k < K; k += 16) tc::mma_bf16(tmem + dcol, tc::kmajor_desc(a, K, k), tc::kmajor_desc(b, K, k), id, k > 0);
}

// 32 lanes x 32 columns: one tcgen05.ld, one wait
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float* v) { tc::tmem_ld32(taddr, v); }

// store 8 consecutive bf16 values of row r at column k0 of a K-major tile
__device__ __forceinline__ void st_row8(uint8_t* tile, int r, int k0, int K, const float* v) {
  uint4 u;
  u.x = tc::pack_bf16(v[0], v[1]);
  u.y = tc::pack_bf16(v[2], v[3]);
  u.z = tc::pack_bf16(v[4], v[5]);
  u.w = tc::pack_bf16(v[6], v[7]);
  *reinterpret_cast<uint4*>(tile + tc::kmajor_off(r, k0, K)) = u;
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

// sum of squared deviations, same partial-chain order as sum32 over d[c]
__device__ __forceinline__ float sumsq32(const float* x, float mu) {
  float p[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const float e = x[i] - mu;
    p[i] = e * e;
  }
#pragma unroll
  for (int c = 8; c < 32; ++c) {
    const float e = x[c] - mu;
    p[c & 7] += e * e;
  }
  return ((p[0] + p[1]) + (p[2] + p[3])) + ((p[4] + p[5]) + (p[6] + p[7]));
}

// LayerNorm (numkit.py:198-202) of row r split over the thread pair: mean
// and 1 / std of the row (this thread holds columns [32h, 32h + 32))
__device__ __forceinline__ void ln_stats(Pipe& P, const float* x, float& mu, float& rstd) {
  mu = P.row_total(sum32(x)) * (1.0f / D);
  rstd = 1.0f / sqrtf(P.row_total(sumsq32(x, mu)) * (1.0f / D) + 1e-5f);
}

__device__ __forceinline__ void ln_half(Pipe& P, const float* x, const float* g, const float* b, float* y) {
  float mu, rstd;
  ln_stats(P, x, mu, rstd);
  const int c0 = HC * P.h;
#pragma unroll
  for (int c = 0; c < HC; ++c) y[c] = fmaf((x[c] - mu) * rstd, g[c0 + c], b[c0 + c]);  // g, b: shared or global
}

// LN straight into a bf16 K-major tile, 8 columns at a time
__device__ __forceinline__ void ln_half_to_tile(Pipe& P, const float* x, const float* g, const float* b,
                                                uint32_t tile = S_A) {
  float mu, rstd;
  ln_stats(P, x, mu, rstd);
  const int c0 = HC * P.h;
#pragma unroll
  for (int q = 0; q < HC; q += 8) {
    float y[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) y[c] = fmaf((x[q + c] - mu) * rstd, g[c0 + q + c], b[c0 + q + c]);
    st_row8(P.smem + tile, P.r, c0 + q, D, y);
  }
}

// fp32 row tile over [S_Q, S_Q + 32 KB) (free between layers and before
// the QKV GEMM): row r, 16-byte chunk q at r * 256 + 16 (q ^ (r & 7)), so a
// warp's rows hit distinct banks.  Holds the self-attention input x + pos
// and the residual stream across the heads / FK block, keeping both out of
// registers (a thread has 128 of them with two groups per SM).
__device__ __forceinline__ float4* xrow(Pipe& P, int q) {
  return reinterpret_cast<float4*>(P.smem + S_Q + P.r * 256 + ((q ^ (P.r & 7)) << 4));
}
__device__ __forceinline__ void save_row(Pipe& P, const float* x) {
#pragma unroll
  for (int k = 0; k < 8; ++k) *xrow(P, 8 * P.h + k) = make_float4(x[4 * k], x[4 * k + 1], x[4 * k + 2], x[4 * k + 3]);
}
__device__ __forceinline__ void load_row(Pipe& P, float* x) {
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const float4 v = *xrow(P, 8 * P.h + k);
    x[4 * k] = v.x; x[4 * k + 1] = v.y; x[4 * k + 2] = v.z; x[4 * k + 3] = v.w;
  }
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

// key columns [kcol, +64) + bias -> key tiles (heads 2h, 2h+1) at dst
// (default: this group's S_K; the encoder's K / V epilogue: global memory)
__device__ void drain_k(Pipe& P, uint32_t kcol, const float* bk, uint8_t* dst = nullptr) {
  float v[HC];
  tmem_ld32(P.lane_addr(kcol + HC * P.h), v);
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    const int hd = 2 * P.h + j;
#pragma unroll
    for (int i = 0; i < 16; ++i) v[16 * j + i] += bk[16 * hd + i];
    uint8_t* tk = (dst ? dst : P.smem + S_K) + hd * 4096;
    st_row8(tk, P.r, 0, DH, v + 16 * j);
    st_row8(tk, P.r, 8, DH, v + 16 * j + 8);
  }
}

// Values arrive transposed: the K | V GEMM is also issued with the weight
// image as the A operand and the token tile as B, so TMEM lanes 64..127 hold
// V^T (lane 64 + d = value dim d, columns = keys).  The threads of lane
// quadrants 2 and 3 write the per-head V^T tiles (16 x 128, K-major along
// keys) with 16-byte stores; thread h takes keys [64 h, 64 h + 64).
__device__ void drain_vt(Pipe& P, uint32_t vtcol, const float* bv, uint8_t* dst = nullptr) {
  if (P.r < 64) return;  // warp-uniform: lane quadrants 0, 1 hold K^T
  const int d = P.r - 64, hd = d >> 4;
  const float b = bv[d];
  uint8_t* tv = (dst ? dst : P.smem + S_VT) + hd * 4096;
#pragma unroll 1
  for (int c = 0; c < 2; ++c) {
    const int k0 = 64 * P.h + 32 * c;
    float v[32];
    tmem_ld32(P.lane_addr(vtcol + k0), v);
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] += b;
#pragma unroll
    for (int q = 0; q < 32; q += 8) st_row8(tv, d & 15, k0 + q, 128, v + q);
  }
}

// V^T[m][key] = sum_k W[row0 + m][k] tok[key][k] for m < 128: the weight
// image rows [row0, row0 + 128) as A, the 128 x 64 token tile as B
__device__ __forceinline__ void gemm_t(uint32_t w, int row0, uint32_t tok, uint32_t dcol, uint32_t tmem) {
  const uint32_t id = tc::idesc_bf16(128, 128);
  const uint32_t a = w + (uint32_t)(row0 / 8) * (D * 16);
  for (int k = 0; k < D; k += 16) tc::mma_bf16(tmem + dcol, tc::kmajor_desc(a, D, k), tc::kmajor_desc(tok, D, k), id, k > 0);
}

constexpr float kScale = 0.25f * 1.4426950408889634f;  // f32(1/sqrt(16)) * log2(e)

// softmax of head (pair + 2 h) over the first NK keys of the row's own key
// block; P (unnormalised, bf16) is packed over the head's S columns
// [128 h, 128 h + 64): the own block's 64 keys in 32 columns, zeros for the
// other block.  Returns 1 / sum (the context is scaled after P.V: 16
// multiplies instead of 64).  NK: 64 (encoder self-attention, cross
// attention), 51 (body tokens).  inactive rows write a zero P row.
// ONE_PASS (the encoder, whose register budget allows 64 live scores): one
// 64-column TMEM read instead of two passes of two 32-column reads.
template <int NK, bool ONE_PASS = false>
__device__ float softmax_head(Pipe& P, bool active = true) {
  static_assert(NK > 32 && NK <= 64, "keys per block");
  const int blk = P.r / BLK;
  const uint32_t tcol = T_GEN + 128 * P.h;
  const uint32_t sa = P.lane_addr(tcol + 64 * blk);
  if constexpr (ONE_PASS) {
    float s[64];
    tc::tmem_ld64(sa, s);
    float m4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
    for (int i = 0; i < NK; ++i) m4[i & 3] = fmaxf(m4[i & 3], s[i]);
    const float nms = -fmaxf(fmaxf(m4[0], m4[1]), fmaxf(m4[2], m4[3])) * kScale;
    float p4[4] = {0.0f, 0.0f, 0.0f, 0.0f};
#pragma unroll
    for (int half = 0; half < 2; ++half) {
      uint32_t u[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const int k = 32 * half + 2 * i;
        float e0 = 0.0f, e1 = 0.0f;
        if (k < NK) {
          e0 = ex2_approx(fmaf(s[k], kScale, nms));
          p4[k & 3] += e0;
        }
        if (k + 1 < NK) {
          e1 = ex2_approx(fmaf(s[k + 1], kScale, nms));
          p4[(k + 1) & 3] += e1;
        }
        u[i] = active ? tc::pack_bf16(e0, e1) : 0u;
      }
      tc::tmem_st16u_nowait(P.lane_addr(tcol + 32 * blk + 16 * half), u);
    }
    const uint32_t z[16] = {0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u};
    tc::tmem_st16u_nowait(P.lane_addr(tcol + 32 * (1 - blk)), z);
    tc::tmem_st16u_nowait(P.lane_addr(tcol + 32 * (1 - blk) + 16), z);
    return active ? 1.0f / ((p4[0] + p4[1]) + (p4[2] + p4[3])) : 0.0f;
  }
  // two passes over 32-column halves (32 live registers instead of 64):
  // the maximum, then exponentials packed as bf16 over the half just read
  float s[32];
  float m4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
  for (int half = 0; half < 2; ++half) {
    tmem_ld32(sa + 32 * half, s);
#pragma unroll
    for (int i = 0; i < 32; ++i)
      if (32 * half + i < NK) m4[i & 3] = fmaxf(m4[i & 3], s[i]);
  }
  const float nms = -fmaxf(fmaxf(m4[0], m4[1]), fmaxf(m4[2], m4[3])) * kScale;
  float p4[4] = {0.0f, 0.0f, 0.0f, 0.0f};
#pragma unroll
  for (int half = 0; half < 2; ++half) {
    tmem_ld32(sa + 32 * half, s);
    uint32_t u[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const int k = 32 * half + 2 * i;
      float e0 = 0.0f, e1 = 0.0f;
      if (k < NK) {
        e0 = ex2_approx(fmaf(s[2 * i], kScale, nms));
        p4[(2 * i) & 3] += e0;
      }
      if (k + 1 < NK) {
        e1 = ex2_approx(fmaf(s[2 * i + 1], kScale, nms));
        p4[(2 * i + 1) & 3] += e1;
      }
      u[i] = active ? tc::pack_bf16(e0, e1) : 0u;
    }
    tc::tmem_st16u_nowait(P.lane_addr(tcol + 32 * blk + 16 * half), u);
  }
  const uint32_t z[16] = {0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u};
  tc::tmem_st16u_nowait(P.lane_addr(tcol + 32 * (1 - blk)), z);
  tc::tmem_st16u_nowait(P.lane_addr(tcol + 32 * (1 - blk) + 16), z);
  return active ? 1.0f / ((p4[0] + p4[1]) + (p4[2] + p4[3])) : 0.0f;
}

// softmax of head (pair + 2 h) for hand tiles: every hand's four token rows
// [4 g, 4 g + 4) attend to the same four keys (decoder.py:393-398).  A warp's
// 32 rows need the 32 key columns of its own lane quadrant; the row's four
// are picked out of them.  Same arithmetic as the NK = 4 softmax.  P: the
// quadrant's 32 keys packed in 16 columns, zeros elsewhere.
__device__ float softmax_group4(Pipe& P) {
  const uint32_t tcol = T_GEN + 128 * P.h;
  const int q = P.r >> 5;
  float s[32];
  tmem_ld32(P.lane_addr(tcol + 32 * q), s);
  const int g = (P.r & 31) >> 2;
  float a[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    a[k] = s[k];
#pragma unroll
    for (int gg = 1; gg < 8; ++gg) a[k] = g == gg ? s[4 * gg + k] : a[k];
  }
  const float nms = -fmaxf(fmaxf(a[0], a[1]), fmaxf(a[2], a[3])) * kScale;
  float e[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) e[k] = ex2_approx(fmaf(a[k], kScale, nms));
  const uint32_t lo = tc::pack_bf16(e[0], e[1]), hi = tc::pack_bf16(e[2], e[3]);
  uint32_t u[32];
#pragma unroll
  for (int i = 0; i < 16; ++i) u[i] = i == 2 * g ? lo : (i == 2 * g + 1 ? hi : 0u);
  tc::tmem_st16u_nowait(P.lane_addr(tcol + 16 * q), u);
#pragma unroll
  for (int i = 0; i < 32; ++i) u[i] = 0u;
  // the other 48 packed columns of [tcol, tcol + 64)
  if (q == 0) {
    tc::tmem_st16u_nowait(P.lane_addr(tcol + 16), u);
    tc::tmem_st32u_nowait(P.lane_addr(tcol + 32), u);
  } else if (q == 1) {
    tc::tmem_st16u_nowait(P.lane_addr(tcol), u);
    tc::tmem_st32u_nowait(P.lane_addr(tcol + 32), u);
  } else if (q == 2) {
    tc::tmem_st32u_nowait(P.lane_addr(tcol), u);
    tc::tmem_st16u_nowait(P.lane_addr(tcol + 48), u);
  } else {
    tc::tmem_st32u_nowait(P.lane_addr(tcol), u);
    tc::tmem_st16u_nowait(P.lane_addr(tcol + 32), u);
  }
  return 1.0f / ((e[0] + e[1]) + (e[2] + e[3]));
}

// Attention of the four heads given sQ / sK / sVt, two heads at a time:
// S pair -> softmax (P packed over S) -> P.V from TMEM -> the pair's
// context columns, scaled by 1 / sum, as bf16 into `ctx_tile` for rows with
// active == true.  Thread h handles head (pair + 2 h) of each pair, so it
// ends up writing context columns [32 h, 32 h + 32) (heads 2h, 2h+1).
// Several calls with disjoint active rows and different K / V (the hand
// tiles' cross-attention rounds) assemble one context tile.
template <int NK, bool G4 = false, bool ONE_PASS = false>
__device__ void attention(Pipe& P, bool active, uint32_t ctx_tile = S_A) {
  const uint32_t sq = P.sbase + S_Q, sk = P.sbase + S_K, sv = P.sbase + S_VT;
  const uint32_t id_s = tc::idesc_bf16(128, 128), id_o = tc::idesc_bf16(128, 16);
#pragma unroll 1
  for (int pair = 0; pair < 2; ++pair) {
    P.before_issue();
    if (P.tid == 0)
      for (int j = 0; j < 2; ++j)
        tc::mma_bf16(P.tmem + T_GEN + 128 * j, tc::kmajor_desc(sq + (pair + 2 * j) * 4096, DH, 0),
                     tc::kmajor_desc(sk + (pair + 2 * j) * 4096, DH, 0), id_s, false);
    P.commit_wait();
    float inv;
    if constexpr (G4)
      inv = softmax_group4(P);
    else
      inv = softmax_head<NK, ONE_PASS>(P, active);
    tc::tmem_wait_st();
    P.before_issue();
    if (P.tid == 0)
      for (int j = 0; j < 2; ++j) {
        const int hd = pair + 2 * j;
        for (int k = 0; k < 8; ++k)
          tc::mma_bf16_ts(P.tmem + T_PV + 16 * j, P.tmem + T_GEN + 128 * j + 8 * k,
                          tc::kmajor_desc(sv + hd * 4096, 128, 16 * k), id_o, k > 0);
      }
    P.commit_wait();
    float o[16];
    tc::tmem_ld16(P.lane_addr(T_PV + 16 * P.h), o);
    if (active) {
#pragma unroll
      for (int i = 0; i < 16; ++i) o[i] *= inv;
      const int hd = pair + 2 * P.h;
      st_row8(P.smem + ctx_tile, P.r, 16 * hd, D, o);
      st_row8(P.smem + ctx_tile, P.r, 16 * hd + 8, D, o + 8);
    }
  }
}

// x += Wo . ctx + bo for valid rows (ctx in the A tile)
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

// self attention: x += MHA(LN(a)), a = x + pos  (decoder.py:214-218)
// (a == nullptr: a is in the fp32 row tile, written by the caller)
template <int NK, bool G4 = false, bool ONE_PASS = false>
__device__ void self_attn(Pipe& P, const float* prm, float* x, const float* a, bool valid) {
#ifdef FSB_PROFILE
  long long q0 = clock64();
#endif
  if (a != nullptr) {
    ln_half_to_tile(P, a, prm + TCP_S_LN_G, prm + TCP_S_LN_B);
  } else {
    float av[HC];
    load_row(P, av);
    ln_half_to_tile(P, av, prm + TCP_S_LN_G, prm + TCP_S_LN_B);
  }
#ifdef FSB_PROFILE
  long long q1 = clock64();
  P.prof[12] += q1 - q0;
#endif
  const uint32_t wq = P.acquire();
  P.before_issue();
  if (P.tid == 0) {
    gemm(P.sbase + S_A, D, wq, 2 * D, T_GEN, P.tmem);  // Q | K
    gemm_t(wq, D, P.sbase + S_A, T_GEN + 128, P.tmem);  // (K | V)^T: V^T in lanes 64..127
  }
  P.prefetch();
  P.commit_wait();
#ifdef FSB_PROFILE
  long long q2 = clock64();
  P.prof[13] += q2 - q1;
#endif
  drain_q(P, T_GEN, prm + TCP_S_BQKV);
  drain_k(P, T_GEN + 64, prm + TCP_S_BQKV + 64);
  drain_vt(P, T_GEN + 128, prm + TCP_S_BQKV + 128);
#ifdef FSB_PROFILE
  long long q3 = clock64();
  P.prof[14] += q3 - q2;
#endif
  attention<NK, G4, ONE_PASS>(P, true);
#ifdef FSB_PROFILE
  P.prof[15] += clock64() - q3;
#endif
  out_proj(P, prm + TCP_S_BO, x, valid);
}

// cross attention: x += MHA(LN_q(x), LN_kv(f))  (decoder.py:220-227).  The
// tile's keys and values were projected ahead of the decoder (kv_project);
// one bulk copy brings this layer's 32 KB image into S_K | S_VT while the
// queries are formed.
__device__ void cross_attn(Pipe& P, const float* prm, float* x, const uint8_t* kvimg, bool valid) {
  uint64_t* bar = &P.sh->kvb[P.g][0];
  if (P.tid == 0) {  // S_K / S_VT are free: the self-attention's MMAs have completed
    tc::mbar_expect_tx(bar, FSB_KV_BODY_TILE);
    tc::bulk_g2s(P.smem + S_K, kvimg, FSB_KV_BODY_TILE, bar);
  }
  ln_half_to_tile(P, x, prm + TCP_C_LNQ_G, prm + TCP_C_LNQ_B);
  const uint32_t wq = P.acquire();
  P.before_issue();
  if (P.tid == 0) gemm(P.sbase + S_A, D, wq, D, T_GEN, P.tmem);
  P.prefetch();
  P.commit_wait();
  drain_q(P, T_GEN, prm + TCP_C_BQKV);
  tc::mbar_wait(bar, (uint32_t)(P.kvuse & 1));
  ++P.kvuse;
  attention<BLK>(P, true);
  out_proj(P, prm + TCP_C_BO, x, valid);
}

// bf16 pair (low half = even element) -> fp32 pair
__device__ __forceinline__ float2 bf2(uint32_t u) {
  return make_float2(__uint_as_float(u << 16), __uint_as_float(u & 0xffff0000u));
}
// packed FP32x2 FMA (sm_100 FFMA2): a * b + c on both lanes
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
  float2 d;
  asm("{\n\t.reg .b64 ra, rb, rc, rd;\n\t"
      "mov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\tmov.b64 rc, {%6, %7};\n\t"
      "fma.rn.f32x2 rd, ra, rb, rc;\n\tmov.b64 {%0, %1}, rd;\n\t}"
      : "=f"(d.x), "=f"(d.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
  return d;
}

// cross attention of a hand tile (decoder.py:220-227 per hand): each hand's
// four query rows attend to its own crop's 64 keys, so the tile's 32 hands
// need 32 different key / value sets -- a batched GEMM with M = 4 per batch
// entry, which the 128-row tensor-core tiles cannot serve without running
// one round per crop pair.  The queries come from one tcgen05 GEMM; the
// scores, softmax and P.V run on the CUDA cores (FFMA2) over the
// precomputed bf16 K / V, streamed two keys (16 KB, all 32 hands) at a time
// through a three-slot shared-memory ring filled by cp.async.bulk (one
// 16 KB copy per key pair, issued by the group's first thread).  The 64 keys
// run as two halves merged at the end (hand_merge below), on both thread
// groups of a one-tile CTA or in sequence on one group.
// The four threads of a hand (tokens t = 0..3, column half h) split each
// key by 16-byte chunks: thread t reads chunk t (dims 32 h + 8 t .. + 8, of
// head 2 h + t / 2) once and forms the partial scores of all four query rows
// on it; a lane-pair shuffle completes each head's 16-dim score, so both
// threads of a pair hold the head's four rows' scores, run the online softmax
// for them and accumulate P.V on their chunk of the values.  A warp's 32
// lanes read 32 distinct chunks (eight hands x four): no broadcast waste.
constexpr int KV_STAGES = 3;
constexpr uint32_t KV_STAGE_BYTES = 32 * 512;  // two keys of 32 hands
constexpr int KV_STAGES_PER_LAYER = 64 / 2;
static_assert(KV_STAGES * KV_STAGE_BYTES <= 3 * 16384, "the ring spans S_Q, S_K, S_VT");

#ifndef FSB_HKV_EXP
#define FSB_HKV_EXP 0  // experiments: 1 = no copies / waits (compute only), 2 = no compute (copies only)
#endif
// online-softmax state of one thread's four query rows over a run of keys
struct HandState {
  float2 o[4][4];
  float m[4], l[4];
};
constexpr int KV_HALF = KV_STAGES_PER_LAYER / 2;  // key pairs per half

// qc[tp][k]: query row 4 i + tp (+ bias, pre-scaled by 1/sqrt(16) log2(e)),
// on this thread's chunk (column 32 h + 8 t + 2k, + 1), from the query
// accumulator at TMEM lane address `qaddr`
__device__ __forceinline__ void hand_queries(const Pipe& P, uint32_t qaddr, const float* prm, float2 (&qc)[4][4]) {
  const int t = P.r & 3, lane = P.r & 31;
  float q[HC];
  tmem_ld32(qaddr, q);
#pragma unroll
  for (int i = 0; i < HC; ++i) q[i] = (q[i] + prm[TCP_C_BQKV + HC * P.h + i]) * kScale;
#pragma unroll
  for (int sc = 0; sc < 4; ++sc)
#pragma unroll
    for (int k = 0; k < 8; k += 2)
#pragma unroll
      for (int tp = 0; tp < 4; ++tp) {
        const float a0 = __shfl_sync(0xffffffffu, q[8 * sc + k], (lane & ~3) | tp);
        const float a1 = __shfl_sync(0xffffffffu, q[8 * sc + k + 1], (lane & ~3) | tp);
        if (t == sc) qc[tp][k / 2] = make_float2(a0, a1);
      }
}

// 40 state floats of a thread <-> 40 TMEM columns of its lane
__device__ __forceinline__ void hand_state_st(uint32_t addr, const HandState& S) {
  float v[40];
#pragma unroll
  for (int tp = 0; tp < 4; ++tp) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      v[8 * tp + 2 * k] = S.o[tp][k].x;
      v[8 * tp + 2 * k + 1] = S.o[tp][k].y;
    }
    v[32 + tp] = S.m[tp];
    v[36 + tp] = S.l[tp];
  }
  tc::tmem_st32(addr, v);
  tc::tmem_st8(addr + 32, v + 32);
}
__device__ __forceinline__ void hand_state_ld(uint32_t addr, HandState& S) {
  float v[40];
  tmem_ld32(addr, v);
  tc::tmem_ld8(addr + 32, v + 32);
#pragma unroll
  for (int tp = 0; tp < 4; ++tp) {
#pragma unroll
    for (int k = 0; k < 4; ++k) S.o[tp][k] = make_float2(v[8 * tp + 2 * k], v[8 * tp + 2 * k + 1]);
    S.m[tp] = v[32 + tp];
    S.l[tp] = v[36 + tp];
  }
}

// The two halves of the keys (pairs [0, 16) and [16, 32)) always run as two
// separate online-softmax passes merged by hand_merge: by one group in
// sequence, or -- in a hand CTA holding one tile, whose second thread group
// would idle -- by the two groups side by side.  Same arithmetic either way,
// so a hand's bits do not depend on the launch shape.
__device__ __forceinline__ void hand_merge(HandState& A, const HandState& B) {
#pragma unroll
  for (int tp = 0; tp < 4; ++tp) {
    const float mm = fmaxf(A.m[tp], B.m[tp]);
    const float ca = ex2_approx(A.m[tp] - mm), cb = ex2_approx(B.m[tp] - mm);
    A.l[tp] = fmaf(A.l[tp], ca, B.l[tp] * cb);
    A.m[tp] = mm;
    const float2 ca2 = make_float2(ca, ca), cb2 = make_float2(cb, cb);
#pragma unroll
    for (int k = 0; k < 4; ++k) A.o[tp][k] = ffma2(A.o[tp][k], ca2, __fmul2_rn(B.o[tp][k], cb2));
  }
}

__device__ __forceinline__ void hand_state_reset(HandState& S) {
#pragma unroll
  for (int tp = 0; tp < 4; ++tp) {
    S.m[tp] = -INFINITY;
    S.l[tp] = 0.0f;
#pragma unroll
    for (int k = 0; k < 4; ++k) S.o[tp][k] = make_float2(0.0f, 0.0f);
  }
}

// `count` key pairs through this group's ring: pair j is layer pair
// first + j in slot (u0 + j) % 3; the caller issued pairs 0..2.  With
// `save_at` in range, the state of pairs [0, save_at) is parked in TMEM at
// `save_addr` and the pass restarts (the sequential two-half schedule).
__device__ void hand_keys(Pipe& P, const uint8_t* src, int first, int count, int u0, const float2 (&qc)[4][4],
                          HandState& S, int save_at, uint32_t save_addr) {
  const int t = P.r & 3;
  auto issue = [&](int j) {
    const int slot = (u0 + j) % KV_STAGES;
    uint64_t* bar = &P.sh->kvb[P.g][slot];
    tc::mbar_expect_tx(bar, KV_STAGE_BYTES);
    tc::bulk_g2s(P.smem + S_Q + slot * KV_STAGE_BYTES, src + (size_t)(first + j) * KV_STAGE_BYTES, KV_STAGE_BYTES,
                 bar);
  };
  hand_state_reset(S);
  // this thread's chunks: hand i's 512 bytes, chunk q = kk 16 + kv 8 + 4 h + t
  // at position q ^ (i & 7)
  const int hi = P.r >> 2;
  const uint32_t off = (uint32_t)hi * 512u;
  const uint32_t pk = (uint32_t)(((4 * P.h + t) ^ (hi & 7)) * 16);  // K chunk of key 0 (V: + 128, key 1: + 256)
#pragma unroll 1
  for (int j = 0; j < count; ++j) {
    if (j == save_at) {  // warp-uniform: park the first half, restart
      hand_state_st(save_addr, S);
      hand_state_reset(S);
    }
    const int n = u0 + j, slot = n % KV_STAGES;
    if (FSB_HKV_EXP != 1) tc::mbar_wait(&P.sh->kvb[P.g][slot], (uint32_t)((n / KV_STAGES) & 1));
    const uint8_t* st = P.smem + S_Q + slot * KV_STAGE_BYTES + off;
    if (FSB_HKV_EXP != 2) {
    float sc[2][4];
#pragma unroll
    for (int kk = 0; kk < 2; ++kk) {
      const uint4 u = *reinterpret_cast<const uint4*>(st + kk * 256 + pk);
      const float2 kx = bf2(u.x), ky = bf2(u.y), kz = bf2(u.z), kw = bf2(u.w);
#pragma unroll
      for (int tp = 0; tp < 4; ++tp) {
        float2 acc = __fmul2_rn(qc[tp][0], kx);
        acc = ffma2(qc[tp][1], ky, acc);
        acc = ffma2(qc[tp][2], kz, acc);
        acc = ffma2(qc[tp][3], kw, acc);
        sc[kk][tp] = acc.x + acc.y;
      }
    }
#pragma unroll
    for (int kk = 0; kk < 2; ++kk)
#pragma unroll
      for (int tp = 0; tp < 4; ++tp) sc[kk][tp] += __shfl_xor_sync(0xffffffffu, sc[kk][tp], 1);
    // online softmax (scores in log2 units): sc becomes the probabilities;
    // the accumulators are rescaled only when a row of the warp raised its
    // maximum (one warp-uniform test for the four rows; rows whose maximum
    // held are multiplied by exactly 1, so the bits are those of a per-row
    // test; rare after the first keys)
    float corr[4];
    bool grew = false;
#pragma unroll
    for (int tp = 0; tp < 4; ++tp) {
      const float mn = fmaxf(S.m[tp], fmaxf(sc[0][tp], sc[1][tp]));
      corr[tp] = ex2_approx(S.m[tp] - mn);
      S.m[tp] = mn;
      sc[0][tp] = ex2_approx(sc[0][tp] - mn);
      sc[1][tp] = ex2_approx(sc[1][tp] - mn);
      S.l[tp] = fmaf(S.l[tp], corr[tp], sc[0][tp] + sc[1][tp]);
      grew = grew || corr[tp] != 1.0f;
    }
    if (__any_sync(0xffffffffu, grew)) {
#pragma unroll
      for (int tp = 0; tp < 4; ++tp) {
        const float2 c2 = make_float2(corr[tp], corr[tp]);
#pragma unroll
        for (int k = 0; k < 4; ++k) S.o[tp][k] = __fmul2_rn(S.o[tp][k], c2);
      }
    }
#pragma unroll
    for (int kk = 0; kk < 2; ++kk) {
      const uint4 u = *reinterpret_cast<const uint4*>(st + kk * 256 + 128 + pk);
      const float2 vv[4] = {bf2(u.x), bf2(u.y), bf2(u.z), bf2(u.w)};
#pragma unroll
      for (int tp = 0; tp < 4; ++tp) {
        const float2 pp = make_float2(sc[kk][tp], sc[kk][tp]);
#pragma unroll
        for (int k = 0; k < 4; ++k) S.o[tp][k] = ffma2(pp, vv[k], S.o[tp][k]);
      }
    }
    }
    // (a group barrier per key pair; per-slot release barriers that let a
    // warp run ahead measured slower: hand CTA 173 -> 182 us)
    P.sync();  // every thread is done with the slot
    if (FSB_HKV_EXP != 1 && P.tid == 0 && j + KV_STAGES < count) issue(j + KV_STAGES);
  }
}

// the CTA-wide barrier between a hand tile's group and its helper group
// (the two groups reach it from different code sites: the non-.aligned
// form; after a spin on an mbarrier the warp's threads may leave the loop
// apart: reconverge for the tcgen05 loads that follow)
__device__ __forceinline__ void cta_pair_sync() {
  __syncwarp();
  asm volatile("barrier.sync 3, %0;\n" ::"r"(NTH) : "memory");
  __syncwarp();
}

// first three key pairs [first, first + 3) of a layer into this group's ring
__device__ __forceinline__ void hand_ring_start(Pipe& P, const uint8_t* src, int first, int u0) {
  if (FSB_HKV_EXP != 1 && P.tid == 0)
    for (int j = 0; j < KV_STAGES; ++j) {
      const int slot = (u0 + j) % KV_STAGES;
      uint64_t* bar = &P.sh->kvb[P.g][slot];
      tc::mbar_expect_tx(bar, KV_STAGE_BYTES);
      tc::bulk_g2s(P.smem + S_Q + slot * KV_STAGE_BYTES, src + (size_t)(first + j) * KV_STAGE_BYTES, KV_STAGE_BYTES,
                   bar);
    }
}

// TMEM columns where a half's state waits: the tile group's own free
// columns [64 + 128 h, +40) (sequential schedule), or the helper group's
__device__ __forceinline__ uint32_t hand_park(const Pipe& P, uint32_t group_off) {
  return P.lane_addr(64u + 128u * (uint32_t)P.h) + group_off;
}

__device__ void cross_attn_hands(Pipe& P, const float* prm, float* x, const uint8_t* hkv, int hand0, int nslots,
                                 int l, int L, bool valid, bool helped) {
  const int u0 = P.kvuse;
  // key pair s of this layer (16 KB: the tile's 32 hands x 512 bytes)
  const uint8_t* src = hkv + ((size_t)(hand0 / FSB_HANDS_PER_TILE) * L + l) * (32 * KV_STAGE_BYTES);
  hand_ring_start(P, src, 0, u0);  // S_Q..S_VT are free: the self-attention's MMAs have completed
  ln_half_to_tile(P, x, prm + TCP_C_LNQ_G, prm + TCP_C_LNQ_B);
  const uint32_t wq = P.acquire();
  P.before_issue();
  if (P.tid == 0) gemm(P.sbase + S_A, D, wq, D, T_GEN, P.tmem);
  P.prefetch();
  P.commit_wait();
  // the residual stream waits in TMEM columns [128 + 32 h, +32) (the query
  // accumulator uses [0, 64))
  {
    uint32_t xu[HC];
#pragma unroll
    for (int c = 0; c < HC; ++c) xu[c] = __float_as_uint(x[c]);
    tc::tmem_st32u_nowait(P.lane_addr(T_GEN + 128 + HC * P.h), xu);
  }
  if (helped) {  // the queries are in TMEM: the helper group may read them
    tc::fence_before();
    cta_pair_sync();
    tc::fence_after();
  }
  const int t = P.r & 3;
  float2 qc[4][4];
  hand_queries(P, P.lane_addr(T_GEN + HC * P.h), prm, qc);
  HandState A, B;
  if (helped) {
    hand_keys(P, src, 0, KV_HALF, u0, qc, A, -1, 0);
    P.kvuse = u0 + KV_HALF;
    cta_pair_sync();  // the helper's half is parked in its TMEM columns
    tc::fence_after();
    hand_state_ld(hand_park(P, 256u), B);
  } else {
    hand_keys(P, src, 0, KV_STAGES_PER_LAYER, u0, qc, B, KV_HALF, hand_park(P, 0u));
    P.kvuse = u0 + KV_STAGES_PER_LAYER;
    hand_state_ld(hand_park(P, 0u), A);
  }
  hand_merge(A, B);
  // context: rows 4 i + tp, columns 32 h + 8 t (head 2 h + t / 2) -> the A
  // tile of the output projection
  if (valid) {
#pragma unroll
    for (int tp = 0; tp < 4; ++tp) {
      const float inv = 1.0f / A.l[tp];
      float v[8];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        v[2 * k] = A.o[tp][k].x * inv;
        v[2 * k + 1] = A.o[tp][k].y * inv;
      }
      st_row8(P.smem + S_A, (P.r & ~3) | tp, HC * P.h + 8 * t, D, v);
    }
  }
  tc::tmem_wait_st();
  tmem_ld32(P.lane_addr(T_GEN + 128 + HC * P.h), x);
  out_proj(P, prm + TCP_C_BO, x, valid);
}

// The idle second group of a one-tile hand CTA runs the second half of every
// layer's keys (pairs [16, 32)) through its own ring and parks its state in
// its TMEM columns for the tile group (cross_attn_hands, helped = true).
__device__ void hand_helper(Pipe& P, const uint8_t* hkv, int hand0, int L) {
  for (int l = 0; l < L; ++l) {
    const uint8_t* src = hkv + ((size_t)(hand0 / FSB_HANDS_PER_TILE) * L + l) * (32 * KV_STAGE_BYTES);
    const int u0 = P.kvuse;
    hand_ring_start(P, src, KV_HALF, u0);  // this group's ring is free: its previous pass has ended
    const int slot = l & 1;                // the layer's parameter block (one pacquire per layer)
    tc::mbar_wait(&P.sh->pbar[slot], (uint32_t)((l >> 1) & 1));
    const float* prm = reinterpret_cast<const float*>(P.sall + S_PRM + slot * PRM_BYTES);
    cta_pair_sync();  // the tile group's queries are in its TMEM columns
    tc::fence_after();
    float2 qc[4][4];
    hand_queries(P, P.lane_addr(T_GEN + HC * P.h) - 256u, prm, qc);
    HandState B;
    hand_keys(P, src, KV_HALF, KV_HALF, u0, qc, B, -1, 0);
    P.kvuse = u0 + KV_HALF;
    hand_state_st(hand_park(P, 0u), B);
    tc::fence_before();
    cta_pair_sync();
  }
}

// MLP: x += W2 relu(W1 LN(x) + b1) + b2  (decoder.py:205-212).  The hidden
// layer is packed as bf16 over the first half of each 64-column chunk of the
// W1 accumulator (this thread's own chunks: no cross-thread hazard) and the
// second GEMM reads it from TMEM in two N = 32 halves whose outputs land in
// the chunks' free second halves: [32, 64) and [96, 128).
__device__ void mlp(Pipe& P, const float* prm, float* x, bool valid) {
  ln_half_to_tile(P, x, prm + TCP_M_LN_G, prm + TCP_M_LN_B);
  const uint32_t w1 = P.acquire();
  P.before_issue();
  if (P.tid == 0) gemm(P.sbase + S_A, D, w1, 4 * D, T_GEN, P.tmem);
  P.prefetch();
  P.commit_wait();
  // 32 fp32 columns at a time: piece p of a chunk packs into [c0 + 16 p, +16),
  // columns this thread has already read
#pragma unroll 1
  for (int q = 0; q < 4; ++q) {
    const int c0 = 128 * P.h + 64 * (q >> 1), p = q & 1;
    float v[32];
    tmem_ld32(P.lane_addr(T_GEN + c0 + 32 * p), v);
    uint32_t u[16];
#pragma unroll
    for (int i = 0; i < 16; ++i)
      u[i] = tc::pack_bf16(fmaxf(v[2 * i] + prm[TCP_M_B1 + c0 + 32 * p + 2 * i], 0.0f),
                           fmaxf(v[2 * i + 1] + prm[TCP_M_B1 + c0 + 32 * p + 2 * i + 1], 0.0f));
    tc::tmem_st16u_nowait(P.lane_addr(T_GEN + c0 + 16 * p), u);
  }
  tc::tmem_wait_st();
  const uint32_t w2 = P.acquire();
  P.before_issue();
  if (P.tid == 0) {
    const uint32_t id = tc::idesc_bf16(128, 32);
    for (int nh = 0; nh < 2; ++nh)
      for (int s = 0; s < 16; ++s)
        tc::mma_bf16_ts(P.tmem + T_GEN + 32 + 64 * nh, P.tmem + T_GEN + 64 * (s >> 2) + 8 * (s & 3),
                        tc::kmajor_desc(w2 + 16384u * nh, 4 * D, 16 * s), id, s > 0);
  }
  P.prefetch();
  P.commit_wait();
  float v[HC];
  tmem_ld32(P.lane_addr(T_GEN + 32 + 64 * P.h), v);
  if (valid)
#pragma unroll
    for (int c = 0; c < HC; ++c) x[c] += v[c] + prm[TCP_M_B2 + HC * P.h + c];
}

// CTA setup: copy the role's weight stream table (16-byte loads), barriers,
// TMEM, then the first two weight images and parameter blocks in flight
// nact: groups of the CTA that have work; a group without work (the second
// tile of a CTA at the end of the batch) leaves right after setup, so the
// other runs alone on the SM and is the only one releasing weight slots.
__device__ void setup(Pipe& P, Shared& sh, uint8_t* smem, const TcStream* tab, unsigned nact) {
  {
    const uint4* src = reinterpret_cast<const uint4*>(tab);
    uint4* dst = reinterpret_cast<uint4*>(&sh.tab);
    for (int i = threadIdx.x; i < (int)(sizeof(TcStream) / 16); i += NTH) dst[i] = __ldg(src + i);
  }
  P.sh = &sh;
  P.sall = smem;
  P.g = threadIdx.x / GT;
  P.smem = smem + P.g * S_GROUP;
  P.sbase = tc::smem_u32(P.smem);
  P.wbase = tc::smem_u32(smem + S_W);
  P.tid = threadIdx.x % GT;
  P.r = P.tid & (ROWS - 1);
  P.h = P.tid / ROWS;
  P.mphase = 0;
  P.kvuse = 0;
  P.wuse = 0;
  P.xc = 0;
  P.puse = 0;
#ifdef FSB_PROFILE
  for (int i = 0; i < 16; ++i) P.prof[i] = 0;
  P.prof[0] = -clock64();
#endif
  if (threadIdx.x == 0) {
    sh.nact = nact;
    for (int i = 0; i < 2; ++i) {
      tc::mbar_init(&sh.wbar[i], 1);
      tc::mbar_init(&sh.pbar[i], 1);
      sh.wrel[i] = 0;
      sh.prel[i] = 0;
    }
    for (int i = 0; i < NG; ++i) {
      tc::mbar_init(&sh.mbar[i], 1);
      for (int k = 0; k < 3; ++k) tc::mbar_init(&sh.kvb[i][k], 1);
    }
    tc::mbar_fence_init();
  }
  if (threadIdx.x < 32) tc::tmem_alloc(&sh.tmem, 512);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  P.tmem = sh.tmem + 256u * (uint32_t)P.g;
  if (threadIdx.x == 0) {
    P.load_image(0);
    P.load_image(1);
    P.load_prm(0);
    P.load_prm(1);
  }
}

__device__ void teardown(Pipe& P, int role) {
  pdl_trigger();  // the next kernel's prologue may start (it waits for this grid's completion)
  tc::fence_before();
  __syncthreads();
  if (threadIdx.x < 32) tc::tmem_dealloc(P.sh->tmem, 512);
#ifdef FSB_PROFILE
  P.prof[0] += clock64();
  // CTA 0 (encoder / body decoder) and the last CTA (hand decoder), group 0
  const bool rec = role == 0 ? blockIdx.x == 0 : (role == 1 ? blockIdx.x == 0 : blockIdx.x == gridDim.x - 1);
  if (P.g == 0 && (P.tid == 0 || P.tid == GT - 1) && rec)
    for (int i = 0; i < 16; ++i) g_tc_prof[role][P.tid ? 1 : 0][i] = (unsigned long long)P.prof[i];
#else
  (void)role;
#endif
}

}  // namespace

// ===========================================================================
// K / V of every decoder layer (kv_project) from this tile's final features
// y (decoder.py:220-227, each layer's LN_kv(f) Wk + bk, LN_kv(f) Wv + bv).
// The features are normalised once (n(f), bf16 A tile); each layer's LN_kv
// affine is folded into its weights and biases at upload (fsb_capi.cu), so
// two layers' K | V come out of ONE N = 256 GEMM.  The bias-added bf16
// results go straight to global memory in the decoders' layout (FSB_KV_* in
// fsb_weights.h): hands row-major chunks; body tiles the decoder's shared-
// memory image, V^T produced by staging V rows in shared memory and
// transposing 8 x 8 blocks with ldmatrix.trans (one coalesced 128-byte
// store per block).  Images / parameter blocks continue the CTA's stream.
// ===========================================================================
__device__ __forceinline__ void ldsm_x4_trans(uint32_t addr, uint32_t* d) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0, %1, %2, %3}, [%4];\n"
               : "=r"(d[0]), "=r"(d[1]), "=r"(d[2]), "=r"(d[3])
               : "r"(addr));
}

__device__ void kv_project(Pipe& P, const float* y, bool body, int tile, const KvArgs& kv) {
  const int L = kv.layers[body ? 0 : 1];
  const int c0 = HC * P.h;
  {
    float mu, rstd;
    ln_stats(P, y, mu, rstd);
#pragma unroll
    for (int q = 0; q < HC; q += 8) {
      float v[8];
#pragma unroll
      for (int c = 0; c < 8; ++c) v[c] = (y[q + c] - mu) * rstd;
      st_row8(P.smem + S_A, P.r, c0 + q, D, v);
    }
  }
  const int u = 2 * tile + P.r / BLK, j = P.r % BLK;  // hands: hand and key of this row
  const int warp = (P.tid >> 5) & 7, lane = P.tid & 31;
#pragma unroll 1
  for (int l0 = 0; l0 < L; l0 += 2) {
    const int nl = min(2, L - l0);
    const float* prm = P.pacquire();
    P.sync();  // every thread of the group is past the previous pair (TMEM drained, staging read)
    P.prelease();
    const uint32_t w = P.acquire();
    P.before_issue();
    if (P.tid == 0) gemm(P.sbase + S_A, D, w, 128 * nl, T_GEN, P.tmem);  // layers l0, l0 + 1: K | V each
    P.prefetch();
    P.commit_wait();
#pragma unroll 1
    for (int jl = 0; jl < nl; ++jl) {
      const int l = l0 + jl, cb = 128 * jl;
      float kk[HC], vv[HC];
      tmem_ld32(P.lane_addr(T_GEN + cb + c0), kk);
      tmem_ld32(P.lane_addr(T_GEN + cb + 64 + c0), vv);
#pragma unroll
      for (int i = 0; i < HC; ++i) {
        kk[i] += prm[cb + c0 + i];
        vv[i] += prm[cb + 64 + c0 + i];
      }
#ifndef FSB_KVP_EXP
#define FSB_KVP_EXP 0  // experiments: 1 = no hand stores, 2 = no body stores / transposes
#endif
      if (body) {
        if (FSB_KVP_EXP == 2) continue;
        uint8_t* dst = kv.body_kv + ((size_t)tile * L + l) * FSB_KV_BODY_TILE;
#pragma unroll
        for (int e = 0; e < 2; ++e) {  // K rows of heads 2h, 2h + 1
          st_row8(dst + (2 * P.h + e) * 4096, P.r, 0, DH, kk + 16 * e);
          st_row8(dst + (2 * P.h + e) * 4096, P.r, 8, DH, kk + 16 * e + 8);
        }
        // V rows -> staging (S_Q / S_K by layer parity), 16-byte chunk q of
        // row r at r * 128 + 16 (q ^ (r & 7))
        uint8_t* stg = P.smem + (jl ? S_K : S_Q);
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          uint4 w4;
          w4.x = tc::pack_bf16(vv[8 * c], vv[8 * c + 1]);
          w4.y = tc::pack_bf16(vv[8 * c + 2], vv[8 * c + 3]);
          w4.z = tc::pack_bf16(vv[8 * c + 4], vv[8 * c + 5]);
          w4.w = tc::pack_bf16(vv[8 * c + 6], vv[8 * c + 7]);
          *reinterpret_cast<uint4*>(stg + P.r * 128 + (((4 * P.h + c) ^ (P.r & 7)) << 4)) = w4;
        }
        P.sync();
        // warp w: token blocks 2w, 2w + 1 x the 8 dim blocks, four 8 x 8
        // blocks per ldmatrix.x4; lane i then holds (dim 8 db + i / 4,
        // keys 8 tb + 2 (i % 4), + 1) -> V^T image (head db / 2)
        const uint32_t sstg = tc::smem_u32(stg);
        uint8_t* vt = dst + 16384;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int tb = 2 * warp + (q >> 1);
          const int tok = 8 * tb + (lane & 7), db_l = 4 * (q & 1) + (lane >> 3);
          uint32_t d4[4];
          ldsm_x4_trans(sstg + tok * 128 + ((db_l ^ (tok & 7)) << 4), d4);
#pragma unroll
          for (int m = 0; m < 4; ++m) {
            const int db = 4 * (q & 1) + m;
            *reinterpret_cast<uint32_t*>(vt + (db >> 1) * 4096 + (db & 1) * 2048 + tb * 128 + (lane >> 2) * 16 +
                                         (lane & 3) * 4) = d4[m];
          }
        }
      } else if (FSB_KVP_EXP != 1) {
        // hand rows -> staging (S_Q: per hand 32 key pairs x 512 bytes in
        // the global chunk order, additionally XOR-ed with the key pair so
        // the stores spread over the banks) -> global: the tile's two hands
        // are adjacent, 1 KB contiguous per key pair
        const int sp = j >> 1;
        uint8_t* stg = P.smem + S_Q + (P.r / BLK) * FSB_KV_HAND + sp * 512;
#pragma unroll
        for (int kvi = 0; kvi < 2; ++kvi) {
          const float* v = kvi ? vv : kk;
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            uint4 w4;
            w4.x = tc::pack_bf16(v[8 * c], v[8 * c + 1]);
            w4.y = tc::pack_bf16(v[8 * c + 2], v[8 * c + 3]);
            w4.z = tc::pack_bf16(v[8 * c + 4], v[8 * c + 5]);
            w4.w = tc::pack_bf16(v[8 * c + 6], v[8 * c + 7]);
            const int q = (j & 1) * 16 + kvi * 8 + 4 * P.h + c;
            *reinterpret_cast<uint4*>(stg + ((q ^ (u & 7) ^ (sp & 7)) << 4)) = w4;
          }
        }
        P.sync();
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const int n = P.tid + GT * k, hb = n >> 10, o = n & 1023, osp = o >> 5;
          const int uu = 2 * tile + hb;
          const uint4 w4 = *reinterpret_cast<const uint4*>(P.smem + S_Q + hb * FSB_KV_HAND + o * 16);
          if (uu < kv.nhand)
            *reinterpret_cast<uint4*>(kv.hand_kv +
                                      ((((size_t)(uu / FSB_HANDS_PER_TILE) * L + l) * 32 + osp) * 32 +
                                       uu % FSB_HANDS_PER_TILE) * 512 + (((o & 31) ^ (osp & 7)) << 4)) = w4;
        }
        if (jl + 1 < nl) P.sync();  // staging reused by the pair's second layer
      }
    }
  }
}

// ===========================================================================
// encoder.  kv.mode 0: grid = ceil(ncrops / 4); group g, block f of CTA b
// encodes crop 4b + 2g + f.  kv.mode 1 (frames) / 2 (given features): body
// CTAs first, then hand CTAs; group g of a CTA takes tile 2 c + g of its
// role, whose blocks are frames (hands) 2 tile, 2 tile + 1 -- the decoders'
// body tiles pair the same frames -- and after the encoder (mode 1) or the
// feature load (mode 2) projects the role's K / V for every decoder layer.
// ===========================================================================
__global__ void __launch_bounds__(NTH, 1) k_encoder_tc(const float* __restrict__ crops, int ncrops, EncW w,
                                                       float* __restrict__ feats, int* nonfinite, KvArgs kv) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ Shared sh;
  Pipe P;
  const int nbc = ((kv.nbody + 1) / 2 + 1) / 2;  // body CTAs (modes 1, 2)
  const bool body = kv.mode != 0 && (int)blockIdx.x < nbc;
  const int nunits = body ? kv.nbody : kv.nhand;
  const int cta = body ? (int)blockIdx.x : (int)blockIdx.x - nbc;
  bool has0, has1;
  if (kv.mode == 0) {
    has0 = true;
    has1 = 4 * (int)blockIdx.x + 2 < ncrops;
  } else {
    has0 = 2 * (2 * cta) < nunits;
    has1 = 2 * (2 * cta + 1) < nunits;
  }
  setup(P, sh, smem, kv.mode == 0 ? w.tcs : kv.tcs[body ? 0 : 1], has1 ? 2u : 1u);
  pdl_wait();  // the weight stream is constant; crops / features come from the previous kernel
  const int blk = P.r / BLK, p = P.r % BLK;
  const int tile = 2 * cta + P.g;
  int crop;
  bool valid;
  if (kv.mode == 0) {
    crop = 4 * blockIdx.x + 2 * P.g + blk;
    valid = crop < ncrops;
  } else {
    const int unit = 2 * tile + blk;
    valid = unit < nunits;
    crop = body ? unit * kv.body_feat_stride : kv.hand_feat_first + (unit / 2) * kv.body_feat_stride + unit % 2;
  }
  // a group without a crop skips to the common teardown (one barrier site)
  if (kv.mode == 0 ? 4 * (int)blockIdx.x + 2 * P.g < ncrops : (P.g == 0 ? has0 : has1)) {

  float y[HC];
#ifdef FSB_PROFILE
  long long efin = 0;
#endif
  if (kv.mode != 2) {
  // patchify (decoder.py:247-248): this thread packs image rows iy in
  // [4h, 4h + 4) of patch p into the K = 192 tile (k = iy*24 + ix*3 + c),
  // which spans this group's A, Q and K tiles
  {
    uint8_t* tile_a = P.smem + S_A;
    const int py = p / 8, px = p % 8;
    const float* src = crops + (int64_t)(valid ? crop : 0) * 64 * 64 * 3;
#pragma unroll 1
    for (int iy = 4 * P.h; iy < 4 * P.h + 4; ++iy) {
      const float* row = src + ((py * 8 + iy) * 64 + px * 8) * 3;
      float4 f4[6];
#pragma unroll
      for (int q = 0; q < 6; ++q)
        f4[q] = valid ? __ldg(reinterpret_cast<const float4*>(row) + q) : make_float4(0.0f, 0.0f, 0.0f, 0.0f);
#pragma unroll
      for (int q = 0; q < 3; ++q) {
        const float v[8] = {f4[2 * q].x, f4[2 * q].y, f4[2 * q].z, f4[2 * q].w,
                            f4[2 * q + 1].x, f4[2 * q + 1].y, f4[2 * q + 1].z, f4[2 * q + 1].w};
        st_row8(tile_a, P.r, iy * 24 + 8 * q, 192, v);
      }
    }
  }
  float x[HC];
  {
#ifdef FSB_PROFILE
    const long long ep0 = clock64();
    P.prof[10] += ep0 + P.prof[0];  // kernel start -> patchify done
#endif
    const uint32_t wp = P.acquire();
#ifdef FSB_PROFILE
    const long long ep1 = clock64();
#endif
    P.before_issue();
    if (P.tid == 0) gemm(P.sbase + S_A, 192, wp, D, T_GEN, P.tmem);
    P.prefetch();
    P.commit_wait();
#ifdef FSB_PROFILE
    P.prof[11] += clock64() - ep0;  // embedding weights wait + GEMM
#endif
    // patch bias and position rows as 16-byte loads, all in flight at once
    // (32 + 32 scalar loads serialised into ~20 L2 round trips: ~17K cycles)
    float4 b4[HC / 4], p4[HC / 4];
    const float4* pb = reinterpret_cast<const float4*>(w.patch_b + HC * P.h);
    const float4* pp = reinterpret_cast<const float4*>(w.pos + p * D + HC * P.h);
#pragma unroll
    for (int q = 0; q < HC / 4; ++q) {
      b4[q] = __ldg(pb + q);
      p4[q] = __ldg(pp + q);
    }
    float v[HC];
    tmem_ld32(P.lane_addr(T_GEN + HC * P.h), v);
#pragma unroll
    for (int q = 0; q < HC / 4; ++q) {
      const float bq[4] = {b4[q].x, b4[q].y, b4[q].z, b4[q].w}, pq[4] = {p4[q].x, p4[q].y, p4[q].z, p4[q].w};
#pragma unroll
      for (int j = 0; j < 4; ++j) x[4 * q + j] = valid ? (v[4 * q + j] + bq[j]) + pq[j] : 0.0f;
    }
  }
#ifdef FSB_PROFILE
  P.prof[8] += clock64() + P.prof[0];  // kernel start -> layer loop (setup, patchify, embedding)
#endif
  for (int l = 0; l < w.layers; ++l) {
#ifdef FSB_PROFILE
    const long long e0 = clock64();
#endif
    const float* prm = P.pacquire();
    P.sync();  // every thread of the group is past layer l - 1
    P.prelease();
    self_attn<BLK, false, true>(P, prm, x, x, valid);
#ifdef FSB_PROFILE
    const long long e1 = clock64();
    P.prof[5] += e1 - e0;
#endif
    mlp(P, prm, x, valid);
#ifdef FSB_PROFILE
    P.prof[7] += clock64() - e1;
#endif
  }
#ifdef FSB_PROFILE
  efin = clock64();
#endif
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
  } else {  // mode 2: the features are given
    const float* in = kv.feats_in + ((int64_t)(valid ? crop : 0) * 64 + p) * D + HC * P.h;
#pragma unroll
    for (int c = 0; c < HC; c += 4) {
      const float4 v = valid ? __ldg(reinterpret_cast<const float4*>(in + c)) : make_float4(0.0f, 0.0f, 0.0f, 0.0f);
      y[c] = v.x; y[c + 1] = v.y; y[c + 2] = v.z; y[c + 3] = v.w;
    }
  }
#ifdef FSB_PROFILE
  if (kv.mode != 2) P.prof[9] += clock64() - efin;  // final LN + feature stores
  const long long ekv = clock64();
#endif
  if (kv.mode != 0) kv_project(P, y, body, tile, kv);
#ifdef FSB_PROFILE
  P.prof[6] += clock64() - ekv;
#endif
  }  // group has crops
  teardown(P, 0);
}

// ===========================================================================
// decoders: CTAs [0, nbc) hold two body tiles (four frames), CTAs
// [nbc, nbc + nhc) two hand tiles (2 kHandsPerCta hands).
// ===========================================================================
struct BodyAux {  // fp32 scratch per body tile
  float t0[2][D];
  float params[2][80];
  float cam[2][4];
  float kp2d[2][44];
  float jc[2][66];
  int pred[2];
  FKOut fk[2];
  float boxtok[2][4 * D];
};
// Hand tiles hold FSB_HANDS_PER_TILE = 32 hands: slot i in rows [4 i, 4 i + 4)
// (token t at row 4 i + t), so every warp holds eight whole hands.
constexpr int kHandsPerCta = FSB_HANDS_PER_TILE;  // per tile
#ifndef FSB_HAND_LATENCY_TILES
#define FSB_HAND_LATENCY_TILES 2
#endif
constexpr int kHandLatencyTiles = FSB_HAND_LATENCY_TILES;
struct HandAux {
  float part[2][kHandsPerCta][6];  // head partial sums of the two column halves
  float rc[kHandsPerCta][8];       // rots[3], cams[3]
  float pts[kHandsPerCta][6];      // 3 x (x, y) projected canonical points
  int pred;
};
static_assert(sizeof(BodyAux) <= AUX_BYTES && sizeof(HandAux) <= AUX_BYTES, "aux scratch");

// LN(token 0) -> head params / camera of both blocks (decoder.py:264-272)
// (x == nullptr: the residual stream is in the fp32 row tile)
__device__ void body_heads(Pipe& P, BodyAux& ax, const BodyW& w, const float* x) {
  float y[HC];
  if (x != nullptr) {
    ln_half(P, x, w.norm_g, w.norm_b, y);
  } else {
    load_row(P, y);
    ln_half(P, y, w.norm_g, w.norm_b, y);
  }
  const int blk = P.r / BLK;
  if (P.r % BLK == 0)
#pragma unroll
    for (int c = 0; c < HC; ++c) ax.t0[blk][HC * P.h + c] = y[c];
  P.sync();
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
  P.sync();
}

// LN(token 0) -> hand rotation / camera of every slot (decoder.py:384-391):
// each token-0 thread dots its 32 normalised columns with the six head
// columns; the two halves meet in shared memory
__device__ void hand_heads(Pipe& P, HandAux& ax, const HandW& w, const float* x) {
  float y[HC];
  if (x != nullptr) {
    ln_half(P, x, w.norm_g, w.norm_b, y);
  } else {
    load_row(P, y);
    ln_half(P, y, w.norm_g, w.norm_b, y);
  }
  if ((P.r & 3) == 0) {
    const int slot = P.r >> 2, c0 = HC * P.h;
#pragma unroll 1
    for (int o = 0; o < 6; ++o) {
      const float* W = (o < 3 ? w.head_rot_w : w.head_cam_w) + o % 3;
      float acc[4] = {0.0f, 0.0f, 0.0f, 0.0f};
#pragma unroll
      for (int k = 0; k < HC; ++k) acc[k & 3] = fmaf(y[k], __ldg(W + (c0 + k) * 3), acc[k & 3]);
      ax.part[P.h][slot][o] = (acc[0] + acc[1]) + (acc[2] + acc[3]);
    }
  }
  P.sync();
  if (P.tid < 6 * kHandsPerCta) {
    const int b = P.tid / 6, o = P.tid % 6;
    ax.rc[b][o] = (ax.part[0][b][o] + ax.part[1][b][o]) + __ldg((o < 3 ? w.head_rot_b : w.head_cam_b) + o % 3);
  }
  P.sync();
}

__global__ void __launch_bounds__(NTH, 1) k_decoders_tc(DecodeArgs a, BodyW bw, HandW hw) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ Shared sh;
  const int nbt = (a.nbody + 1) / 2;                          // body tiles
  const int nbc = (nbt + NG - 1) / NG;                        // body CTAs
  const bool body = (int)blockIdx.x < nbc;
  const int layers = body ? bw.layers : hw.layers;
  Pipe P;
  // tiles per CTA: body NG; hands a.hand_tiles_per_cta (1: latency, 2: SM-time)
  const int tpc = body ? NG : a.hand_tiles_per_cta;
  // groups with work in this CTA: tile 2 x + 1 exists?
  const int tile1 = tpc * (body ? (int)blockIdx.x : (int)blockIdx.x - nbc) + 1;
  const bool has1 = tpc == 2 && (body ? 2 * tile1 < a.nbody : kHandsPerCta * tile1 < a.nhand);
  setup(P, sh, smem, body ? bw.tcs : hw.tcs, has1 ? 2u : 1u);
  pdl_wait();
  const int t = P.tid;
  const int r = P.r, blk = r / BLK, c0 = HC * P.h;
  const int tile = tpc * (body ? (int)blockIdx.x : (int)blockIdx.x - nbc) + P.g;
  // body: frame 2 tile + blk, token rb; hand: slot hs = r / 4, token rb
  const int hand0 = kHandsPerCta * tile;
  const int nslots = body ? 0 : max(0, min(kHandsPerCta, a.nhand - hand0));
  const int hs = r >> 2;
  const int rb = body ? r % BLK : (r & 3);
  const int unit = body ? 2 * tile + blk : 0;  // frame index (body tiles)
  const bool valid = body ? (unit < a.nbody && rb < 51) : hs < nslots;
  const int fb0 = 2 * tile;                    // first frame of a body tile
  // a one-tile hand CTA: its second group runs half of every layer's cross-
  // attention keys (hand_helper); FSB_HAND_SPLIT=0 in the launcher turns
  // this off (same bits: the halves are merged the same way in sequence)
  const bool helped = !body && tpc == 1 && a.hand_split;
  if (helped && P.g == 1) hand_helper(P, a.hand_kv, kHandsPerCta * ((int)blockIdx.x - nbc), hw.layers);
  // a group without a tile skips to the common teardown (one barrier site)
  if (P.g == 0 || has1) {

  // this tile's projected cross-attention keys / values, one block per layer
  const uint8_t* kvt = body ? a.body_kv + (size_t)tile * layers * FSB_KV_BODY_TILE
                            : a.hand_kv;

  float x[HC];
  BodyAux& bx = *reinterpret_cast<BodyAux*>(smem + S_AUX + P.g * AUX_BYTES);
  HandAux& hx = *reinterpret_cast<HandAux*>(smem + S_AUX + P.g * AUX_BYTES);
  if (body) {
    // tokens = token_init, rows 1..4 += prompt_box(prompt)  (decoder.py:287-293)
    for (int i = 0; i < 2; ++i) {
      const int idx = 2 * t + i, b = idx / (4 * D), o = idx % (4 * D);
      const int u = fb0 + b;
      float acc = 0.0f;
      if (u < a.nbody) {
#pragma unroll
        for (int k = 0; k < 8; ++k) acc = fmaf(a.prompts[(int64_t)u * 8 + k], __ldg(bw.prompt_box_w + k * 4 * D + o), acc);
      }
      bx.boxtok[b][o] = acc + __ldg(bw.prompt_box_b + o);
    }
    // the token row as 16-byte loads, all in flight before the barrier
    // (scalar loads serialised into L2 round trips, as in the encoder)
    float4 ti[HC / 4];
    const float4* tsrc = reinterpret_cast<const float4*>(bw.token_init + (valid ? rb : 0) * D + c0);
#pragma unroll
    for (int q = 0; q < HC / 4; ++q) ti[q] = __ldg(tsrc + q);
    if (t < 2) bx.pred[t] = 0;
    P.sync();
#pragma unroll
    for (int q = 0; q < HC / 4; ++q) {
      const float tv[4] = {ti[q].x, ti[q].y, ti[q].z, ti[q].w};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int c = 4 * q + j;
        float v = valid ? tv[j] : 0.0f;
        if (valid && rb >= 1 && rb < 5) v += bx.boxtok[blk][(rb - 1) * D + c0 + c];
        x[c] = v;
      }
    }
  } else {
    const float4* tsrc = reinterpret_cast<const float4*>(hw.token_init + (valid ? rb : 0) * D + c0);
#pragma unroll
    for (int q = 0; q < HC / 4; ++q) {
      const float4 tv = __ldg(tsrc + q);
      x[4 * q] = valid ? tv.x : 0.0f;
      x[4 * q + 1] = valid ? tv.y : 0.0f;
      x[4 * q + 2] = valid ? tv.z : 0.0f;
      x[4 * q + 3] = valid ? tv.w : 0.0f;
    }
    if (t == 0) hx.pred = 0;
  }
  P.sync();

#ifdef FSB_PROFILE
  P.prof[8] += clock64() + P.prof[0];  // setup: kernel start (prof[0] = -start) -> layer loop
  long long tpos;
#endif
  for (int l = 0; l < layers; ++l) {
#ifdef FSB_PROFILE
    tpos = clock64();
#endif
    // a = x + positional term of the self-attention input (decoder.py:
    // 300-303, :397-398), recomputed every layer from the small tables
    // (16-byte loads of this thread's 32 columns)
    {
      float av[HC];
#pragma unroll
      for (int i = 0; i < HC; ++i) av[i] = x[i];
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
          av[4 * q] += v.x; av[4 * q + 1] += v.y; av[4 * q + 2] += v.z; av[4 * q + 3] += v.w;
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
          av[4 * q] += fmaf(k1, w1.x, k0 * w0.x) + b4.x;
          av[4 * q + 1] += fmaf(k1, w1.y, k0 * w0.y) + b4.y;
          av[4 * q + 2] += fmaf(k1, w1.z, k0 * w0.z) + b4.z;
          av[4 * q + 3] += fmaf(k1, w1.w, k0 * w0.w) + b4.w;
        }
      } else if (kind == 2) {
        const float g0 = bx.jc[blk][3 * j], g1 = bx.jc[blk][3 * j + 1], g2 = bx.jc[blk][3 * j + 2];
#pragma unroll
        for (int q = 0; q < HC / 4; ++q) {
          const float4 w0 = __ldg(reinterpret_cast<const float4*>(bw.phi3d_w + c0) + q);
          const float4 w1 = __ldg(reinterpret_cast<const float4*>(bw.phi3d_w + D + c0) + q);
          const float4 w2 = __ldg(reinterpret_cast<const float4*>(bw.phi3d_w + 2 * D + c0) + q);
          const float4 b4 = __ldg(reinterpret_cast<const float4*>(bw.phi3d_b + c0) + q);
          av[4 * q] += fmaf(g2, w2.x, fmaf(g1, w1.x, g0 * w0.x)) + b4.x;
          av[4 * q + 1] += fmaf(g2, w2.y, fmaf(g1, w1.y, g0 * w0.y)) + b4.y;
          av[4 * q + 2] += fmaf(g2, w2.z, fmaf(g1, w1.z, g0 * w0.z)) + b4.z;
          av[4 * q + 3] += fmaf(g2, w2.w, fmaf(g1, w1.w, g0 * w0.w)) + b4.w;
        }
      }
      save_row(P, av);  // S_Q is free: the previous layer's attention is done
    }
    const float* prm = P.pacquire();
    P.sync();  // every thread of the group is past layer l - 1
    P.prelease();
#ifdef FSB_PROFILE
    long long ts0 = clock64();
    P.prof[9] += ts0 - tpos;
#endif
    if (body)
      self_attn<51>(P, prm, x, nullptr, valid);
    else
      self_attn<4, true>(P, prm, x, nullptr, valid);
#ifdef FSB_PROFILE
    long long ts1 = clock64();
    P.prof[5] += ts1 - ts0;
#endif
    if (body)
      cross_attn(P, prm, x, kvt + (size_t)l * FSB_KV_BODY_TILE, valid);
    else
      cross_attn_hands(P, prm, x, kvt, hand0, nslots, l, layers, valid, helped);
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
      save_row(P, x);  // the residual stream waits in shared memory across heads / FK
      if (body) {
        // intermediate prediction: heads -> FK -> kp2d / centred joints
        body_heads(P, bx, bw, nullptr);
#ifdef FSB_PROFILE
        long long th = clock64();
        P.prof[10] += th - ts3;
#endif
        if (t < 64) fk_warp<true>(bx.params[t / 32], bw.joints_rest, bx.fk[t / 32], t % 32);
        P.sync();
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
        P.sync();
        if (a.inter != nullptr && t < 2 * 123) {
          const int b = t / 123, i = t % 123, u = fb0 + b;
          if (u < a.nbody) {
            float* dst = a.inter + ((int64_t)u * layers + l) * (FSB_PARAM_DIM + 3 + 44);
            dst[i] = i < FSB_PARAM_DIM ? bx.params[b][i]
                                       : (i < FSB_PARAM_DIM + 3 ? bx.cam[b][i - FSB_PARAM_DIM]
                                                                : bx.kp2d[b][i - FSB_PARAM_DIM - 3]);
          }
        }
      } else {
        // canonical points through the predicted rotation (decoder.py:399-409)
        hand_heads(P, hx, hw, nullptr);
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
        P.sync();
      }
      load_row(P, x);
    }
  }
#ifdef FSB_PROFILE
  long long tfin = clock64();
#endif
  // final heads and outputs
  if (body) {
    body_heads(P, bx, bw, x);
    if (t < 2 * FSB_PARAM_DIM) {
      const int b = t / FSB_PARAM_DIM, o = t % FSB_PARAM_DIM, u = fb0 + b;
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
  }  // group has a tile
  teardown(P, body ? 1 : 2);
}

// debug export of the FSB_PROFILE cycle counters (not part of the public ABI)
extern "C" int fsb_debug_tc_profile(unsigned long long* out32) {
#ifdef FSB_PROFILE
  return cudaMemcpyFromSymbol(out32, g_tc_prof, sizeof(unsigned long long) * 96) == cudaSuccess ? 0 : 4;
#else
  for (int i = 0; i < 96; ++i) out32[i] = 0;
  return 3;
#endif
}

cudaError_t init_attrs_transformer_tc() {
  cudaError_t e = cudaFuncSetAttribute(k_encoder_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM_TC);
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(k_decoders_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM_TC);
}

cudaError_t launch_encoder_tc(const float* crops, int ncrops, const EncW& w, float* feats, int* nonfinite,
                              const KvArgs& kv, cudaStream_t st) {
  int grid;
  if (kv.mode == 0) {
    grid = (ncrops + 2 * NG - 1) / (2 * NG);
  } else {
    const int bt = (kv.nbody + 1) / 2, ht = (kv.nhand + 1) / 2;
    grid = (bt + NG - 1) / NG + (ht + NG - 1) / NG;
  }
  if (grid == 0) return cudaSuccess;
  return launch_pdl(k_encoder_tc, dim3(grid), dim3(NTH), SMEM_TC, st, crops, ncrops, w, feats, nonfinite, kv);
}

cudaError_t launch_decoders_tc(const DecodeArgs& a_in, const BodyW& bw, const HandW& hw, cudaStream_t st) {
  DecodeArgs a = a_in;
  const int nbt = (a.nbody + 1) / 2, nht = (a.nhand + kHandsPerCta - 1) / kHandsPerCta;
  // hand tiles per CTA: one each while the hands fit a few CTAs (the hand
  // tiles' CUDA-core cross attention then has the SM to itself: latency),
  // two per CTA for large batches (SM-time).  FSB_HAND_TPC overrides.
  static const int forced = [] {
    const char* e = getenv("FSB_HAND_TPC");
    return e ? atoi(e) : 0;
  }();
  a.hand_tiles_per_cta = forced == 1 || forced == 2 ? forced : (nht <= kHandLatencyTiles ? 1 : 2);
  static const bool split = [] {
    const char* e = getenv("FSB_HAND_SPLIT");
    return e == nullptr || atoi(e) != 0;
  }();
  a.hand_split = split ? 1 : 0;
  const int n = (nbt + NG - 1) / NG + (nht + a.hand_tiles_per_cta - 1) / a.hand_tiles_per_cta;
  if (n == 0) return cudaSuccess;
  return launch_pdl(k_decoders_tc, dim3(n), dim3(NTH), SMEM_TC, st, a, bw, hw);
}
