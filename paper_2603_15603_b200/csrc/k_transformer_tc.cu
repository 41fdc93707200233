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

// key columns [kcol, +64) + bias -> key tiles (heads 2h, 2h+1)
__device__ void drain_k(Pipe& P, uint32_t kcol, const float* bk) {
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
}

// Values arrive transposed: the K | V GEMM is also issued with the weight
// image as the A operand and the token tile as B, so TMEM lanes 64..127 hold
// V^T (lane 64 + d = value dim d, columns = keys).  The threads of lane
// quadrants 2 and 3 write the per-head V^T tiles (16 x 128, K-major along
// keys) with 16-byte stores; thread h takes keys [64 h, 64 h + 64).
__device__ void drain_vt(Pipe& P, uint32_t vtcol, const float* bv) {
  if (P.r < 64) return;  // warp-uniform: lane quadrants 0, 1 hold K^T
  const int d = P.r - 64, hd = d >> 4;
  const float b = bv[d];
  uint8_t* tv = P.smem + S_VT + hd * 4096;
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

// cross attention: x += MHA(LN_q(x), LN_kv(f))  (decoder.py:220-227).
// LN_kv(f) is staged in the V^T tile (free until drain_kv refills it after
// the K | V GEMM has read it).
__device__ void cross_attn(Pipe& P, const float* prm, float* x, const float* frow, bool valid) {
  float f[HC];
#pragma unroll
  for (int c = 0; c < HC; c += 4) {
    const float4 v = __ldg(reinterpret_cast<const float4*>(frow + HC * P.h + c));
    f[c] = v.x; f[c + 1] = v.y; f[c + 2] = v.z; f[c + 3] = v.w;
  }
  ln_half_to_tile(P, f, prm + TCP_C_LNKV_G, prm + TCP_C_LNKV_B, S_VT);
  const uint32_t wkv = P.acquire();
  P.before_issue();
  if (P.tid == 0) {
    gemm(P.sbase + S_VT, D, wkv, D, T_GEN, P.tmem);        // K
    gemm_t(wkv, 0, P.sbase + S_VT, T_GEN + 128, P.tmem);  // (K | V)^T
  }
  P.prefetch();
  P.commit_wait();
  drain_k(P, T_GEN, prm + TCP_C_BQKV + 64);
  drain_vt(P, T_GEN + 128, prm + TCP_C_BQKV + 128);
  ln_half_to_tile(P, x, prm + TCP_C_LNQ_G, prm + TCP_C_LNQ_B);
  const uint32_t wq = P.acquire();
  P.before_issue();
  if (P.tid == 0) gemm(P.sbase + S_A, D, wq, D, T_GEN, P.tmem);
  P.prefetch();
  P.commit_wait();
  drain_q(P, T_GEN, prm + TCP_C_BQKV);
  attention<BLK>(P, true);
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
  if (nr == 0) P.prefetch();  // an empty tile still releases t_q (the other group waits for t_o)
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
    ln_half_to_tile(P, f, prm + TCP_C_LNKV_G, prm + TCP_C_LNKV_B, S_VT);
    P.before_issue();
    if (P.tid == 0) {
      gemm(P.sbase + S_VT, D, wkv, D, T_GEN, P.tmem);
      gemm_t(wkv, 0, P.sbase + S_VT, T_GEN + 128, P.tmem);
    }
    if (c == 0) P.prefetch();  // t_q's slot may be refilled
    P.commit_wait();
    drain_k(P, T_GEN, prm + TCP_C_BQKV + 64);
    drain_vt(P, T_GEN + 128, prm + TCP_C_BQKV + 128);
    attention<BLK>(P, (rb >> 2) == c);
  }
  out_proj(P, prm + TCP_C_BO, x, valid);
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
    for (int i = 0; i < NG; ++i) tc::mbar_init(&sh.mbar[i], 1);
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
// encoder: grid = ceil(ncrops / 4); group g, block f of CTA b encodes crop
// 4b + 2g + f
// ===========================================================================
__global__ void __launch_bounds__(NTH, 1) k_encoder_tc(const float* __restrict__ crops, int ncrops, EncW w,
                                                       float* __restrict__ feats, int* nonfinite) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ Shared sh;
  Pipe P;
  setup(P, sh, smem, w.tcs, 4 * (int)blockIdx.x + 2 < ncrops ? 2u : 1u);
  const int blk = P.r / BLK, p = P.r % BLK;
  const int crop = 4 * blockIdx.x + 2 * P.g + blk;
  const bool valid = crop < ncrops;
  // a group without a crop skips to the common teardown (one barrier site)
  if (4 * (int)blockIdx.x + 2 * P.g < ncrops) {

  // patchify (decoder.py:247-248): this thread packs image rows iy in
  // [4h, 4h + 4) of patch p into the K = 192 tile (k = iy*24 + ix*3 + c),
  // which spans this group's A, Q and K tiles
  {
    uint8_t* tile = P.smem + S_A;
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
        st_row8(tile, P.r, iy * 24 + 8 * q, 192, v);
      }
    }
  }
  float x[HC];
  {
    const uint32_t wp = P.acquire();
    P.before_issue();
    if (P.tid == 0) gemm(P.sbase + S_A, 192, wp, D, T_GEN, P.tmem);
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
  for (int l = 0; l < w.layers; ++l) {
    const float* prm = P.pacquire();
    P.sync();  // every thread of the group is past layer l - 1
    P.prelease();
    self_attn<BLK, false, true>(P, prm, x, x, valid);
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
// Hand tiles hold kHandsPerCta hands: slot i sits in row block i % 2, rows
// 64 (i % 2) + 4 (i / 2) + token, so the two slots of a cross-attention
// round (2c, 2c + 1) use key blocks 0 and 1 and every warp sees one.
#ifndef FSB_HANDS_PER_CTA
#define FSB_HANDS_PER_CTA 8  // 2 / 4 / 8 / 16 measured: DESIGN.md §4
#endif
constexpr int kHandsPerCta = FSB_HANDS_PER_CTA;  // per tile
static_assert(kHandsPerCta >= 2 && kHandsPerCta <= 16 && kHandsPerCta % 2 == 0, "hand slots per tile");
struct HandAux {
  float t0[kHandsPerCta][D];
  float rc[kHandsPerCta][8];   // rots[3], cams[3]
  float pts[kHandsPerCta][6];  // 3 x (x, y) projected canonical points
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

// LN(token 0) -> hand rotation / camera of every slot (decoder.py:384-391)
__device__ void hand_heads(Pipe& P, HandAux& ax, const HandW& w, const float* x) {
  float y[HC];
  if (x != nullptr) {
    ln_half(P, x, w.norm_g, w.norm_b, y);
  } else {
    load_row(P, y);
    ln_half(P, y, w.norm_g, w.norm_b, y);
  }
  const int slot = 2 * ((P.r % BLK) >> 2) + P.r / BLK;
  if ((P.r & 3) == 0 && slot < kHandsPerCta)
#pragma unroll
    for (int c = 0; c < HC; ++c) ax.t0[slot][HC * P.h + c] = y[c];
  P.sync();
  if (P.tid < 6 * kHandsPerCta) {
    const int b = P.tid / 6, o = P.tid % 6;
    const float* W = o < 3 ? w.head_rot_w : w.head_cam_w;
    float acc[4] = {0.0f, 0.0f, 0.0f, 0.0f};
#pragma unroll
    for (int k = 0; k < D; ++k) acc[k & 3] = fmaf(ax.t0[b][k], __ldg(W + k * 3 + o % 3), acc[k & 3]);
    ax.rc[b][o] = (acc[0] + acc[1]) + (acc[2] + acc[3]) + __ldg((o < 3 ? w.head_rot_b : w.head_cam_b) + o % 3);
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
  // groups with work in this CTA: tile 2 x + 1 exists?
  const int tile1 = NG * (body ? (int)blockIdx.x : (int)blockIdx.x - nbc) + 1;
  const bool has1 = body ? 2 * tile1 < a.nbody : kHandsPerCta * tile1 < a.nhand;
  setup(P, sh, smem, body ? bw.tcs : hw.tcs, has1 ? 2u : 1u);
  const int t = P.tid;
  const int r = P.r, blk = r / BLK, c0 = HC * P.h;
  const int tile = NG * (body ? (int)blockIdx.x : (int)blockIdx.x - nbc) + P.g;
  // body: frame 2 tile + blk, token rb; hand: slot hs = 2 (r % 64 / 4) + blk, token rb
  const int hand0 = kHandsPerCta * tile;
  const int nslots = body ? 0 : max(0, min(kHandsPerCta, a.nhand - hand0));
  const int hs = 2 * ((r % BLK) >> 2) + blk;
  const int rb = body ? r % BLK : (r & 3);
  const int unit = body ? 2 * tile + blk : 0;  // frame index (body tiles)
  const bool valid = body ? (unit < a.nbody && rb < 51) : hs < nslots;
  const int fb0 = 2 * tile;                    // first frame of a body tile
  // a group without a tile skips to the common teardown (one barrier site)
  if (P.g == 0 || has1) {

  // feature row of this thread for the body's cross attention
  const int crop = (body && unit < a.nbody ? unit : 0) * a.body_feat_stride;
  const float* frow = a.feats + ((int64_t)crop * 64 + (r % BLK)) * D;

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
    if (t < 2) bx.pred[t] = 0;
    P.sync();
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
                              cudaStream_t st) {
  if (ncrops == 0) return cudaSuccess;
  k_encoder_tc<<<(ncrops + 2 * NG - 1) / (2 * NG), NTH, SMEM_TC, st>>>(crops, ncrops, w, feats, nonfinite);
  return cudaGetLastError();
}

cudaError_t launch_decoders_tc(const DecodeArgs& a, const BodyW& bw, const HandW& hw, cudaStream_t st) {
  const int nbt = (a.nbody + 1) / 2, nht = (a.nhand + kHandsPerCta - 1) / kHandsPerCta;
  const int n = (nbt + NG - 1) / NG + (nht + NG - 1) / NG;
  if (n == 0) return cudaSuccess;
  k_decoders_tc<<<n, NTH, SMEM_TC, st>>>(a, bw, hw);
  return cudaGetLastError();
}
