// K4: forward kinematics, MHR linear-blend skinning, the barycentric bridge
// into the projector input, the projector MLP (fp32 path) and SMPL FK.
//
// Reference: bodymodel.fk_batch (bodymodel.py:266-297), skin_batch (:334-368,
// correctives off), projection.bridge (projection.py:187-203),
// _projector_inputs (:447-465), _projector_mlp (:468-472).
//
// LBS is the bandwidth-bound kernel of the path: per mesh it writes
// Nv x 12 B of vertices and reads ~1 KB of per-pose transforms.  The
// template (rest vertices, 1-2 nonzero skin weights per vertex, shape basis;
// ~4 MB at 18,439 vertices) is read once per CTA into registers and reused
// across a group of meshes, so HBM traffic is the vertex stream itself.
#include <cstdlib>

#include "fsb_common.cuh"
#include "fsb_weights.h"
#include "tc_sm100.cuh"

// ---------------------------------------------------------------------------
// FK: one warp per pose.  rel (B, 22, 3, 4) = [R_world | t_world - R_world g]
// ---------------------------------------------------------------------------
// lbs_in (nullable): the k_lbs_tc chunk records (fsb_weights.h
// FSB_LBS_REC_*): transforms interleaved by mesh pairs and the shape
// coefficients split into bf16 hi + lo (hi = bf16(s), lo = bf16(s - hi)).
// dn.H > 0 (the SMPL FK of the frame path with a denoiser loaded): the body
// pose theta[3:66] is first replaced by denoise(theta[3:66]) (projection.py:
// 684-697), in `poses` too, so FK, skinning and the returned theta see it
// (SURVEY §8(f) row 1 as a K4 epilogue).
__global__ void __launch_bounds__(128) k_fk(float* __restrict__ poses, int ld_pose, int B,
                                            const float* __restrict__ grest, float* __restrict__ joints,
                                            float* __restrict__ rel, uint8_t* __restrict__ lbs_in, DenoiseW dn,
                                            int* nonfinite) {
  __shared__ FKOut fk[4];
  __shared__ float pose_s[4][66];
  __shared__ float dn_h[4][FSB_DN_MAX_HIDDEN];
  __shared__ float dn_o[4][64];
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int b = blockIdx.x * 4 + warp;
  pdl_wait();
  if (b >= B) return;  // warp-uniform
  for (int i = lane; i < 66; i += 32) pose_s[warp][i] = poses[(int64_t)b * ld_pose + i];
  __syncwarp();
  if (dn.H > 0) {
    denoise_warp(pose_s[warp] + 3, dn_h[warp], dn, lane, dn_o[warp], nonfinite);
    for (int i = lane; i < FSB_DN_IN; i += 32) {
      pose_s[warp][3 + i] = dn_o[warp][i];
      poses[(int64_t)b * ld_pose + 3 + i] = dn_o[warp][i];
    }
    __syncwarp();
  }
  fk_warp(pose_s[warp], grest, fk[warp], lane);
  if (lane < FSB_NJ) {
    const int j = lane;
    if (joints != nullptr)
      for (int a = 0; a < 3; ++a) joints[((int64_t)b * FSB_NJ + j) * 3 + a] = fk[warp].tw[j][a];
    if (rel != nullptr) {
      float* r = rel + ((int64_t)b * FSB_NJ + j) * 12;
      for (int a = 0; a < 3; ++a) {
        r[4 * a + 0] = fk[warp].rw[j][3 * a + 0];
        r[4 * a + 1] = fk[warp].rw[j][3 * a + 1];
        r[4 * a + 2] = fk[warp].rw[j][3 * a + 2];
        r[4 * a + 3] = fk[warp].at[j][a];
      }
    }
    if (lbs_in != nullptr) {
      uint8_t* rec = lbs_in + (int64_t)(b / FSB_LBS_N) * FSB_LBS_REC_BYTES;
      const int m = b % FSB_LBS_N;
      float* a2 = reinterpret_cast<float*>(rec) + ((m >> 1) * FSB_NJ * FSB_LBS_JS + j * FSB_LBS_JS) * 2 + (m & 1);
      for (int a = 0; a < 3; ++a) {
        a2[2 * (4 * a + 0)] = fk[warp].rw[j][3 * a + 0];
        a2[2 * (4 * a + 1)] = fk[warp].rw[j][3 * a + 1];
        a2[2 * (4 * a + 2)] = fk[warp].rw[j][3 * a + 2];
        a2[2 * (4 * a + 3)] = fk[warp].at[j][a];
      }
    }
  }
  if (lbs_in != nullptr && lane < 16) {  // shape coefficient k = lane (zero padding k >= 10)
    uint8_t* rec = lbs_in + (int64_t)(b / FSB_LBS_N) * FSB_LBS_REC_BYTES;
    const int m = b % FSB_LBS_N, k = lane;
    const float sv = k < 10 ? poses[(int64_t)b * ld_pose + 66 + k] : 0.0f;
    const __nv_bfloat16 hi = __float2bfloat16_rn(sv);
    const __nv_bfloat16 lo = __float2bfloat16_rn(sv - __bfloat162float(hi));
    const uint32_t off = tc::kmajor_off(m, k, 16);
    *reinterpret_cast<__nv_bfloat16*>(rec + FSB_LBS_REC_A2 + off) = hi;
    *reinterpret_cast<__nv_bfloat16*>(rec + FSB_LBS_REC_A2 + FSB_LBS_REC_B + off) = lo;
  }
}

// ---------------------------------------------------------------------------
// one vertex of LBS given the mesh's joint transforms A (22 x 12) and shape
// coefficients (10): blend the nonzero joints, add shape offsets, apply.
// ---------------------------------------------------------------------------
template <int NZ>
struct VertexTmpl {
  int j[NZ];
  float w[NZ];
  float vr[3];
  float sb[30];
  // one vectorised read of the vertex record (fsb_weights.h: TemplateDev::rec)
  __device__ void load(const TemplateDev& t, int v) {
    constexpr int RS = vertex_record_floats(NZ);
    float f[RS];
    const float4* src = reinterpret_cast<const float4*>(t.rec) + (int64_t)v * (RS / 4);
#pragma unroll
    for (int q = 0; q < RS / 4; ++q) {
      const float4 x = __ldg(src + q);
      f[4 * q] = x.x; f[4 * q + 1] = x.y; f[4 * q + 2] = x.z; f[4 * q + 3] = x.w;
    }
    unpack(f);
  }
  // from a record already in registers / shared memory
  __device__ void unpack(const float* f) {
#pragma unroll
    for (int c = 0; c < 3; ++c) vr[c] = f[c];
#pragma unroll
    for (int k = 0; k < 30; ++k) sb[k] = f[4 + k];
#pragma unroll
    for (int z = 0; z < NZ; ++z) {
      w[z] = f[34 + z];
      j[z] = __float_as_int(f[34 + NZ + z]);
    }
  }
  __device__ void apply(const float* A, const float* shp, float out[3]) const {
    float T[12];
#pragma unroll
    for (int e = 0; e < 12; ++e) T[e] = 0.0f;
#pragma unroll
    for (int z = 0; z < NZ; ++z) {
      const float4* a4 = reinterpret_cast<const float4*>(A + 12 * j[z]);
#pragma unroll
      for (int q = 0; q < 3; ++q) {
        const float4 r = a4[q];
        T[4 * q + 0] = fmaf(w[z], r.x, T[4 * q + 0]);
        T[4 * q + 1] = fmaf(w[z], r.y, T[4 * q + 1]);
        T[4 * q + 2] = fmaf(w[z], r.z, T[4 * q + 2]);
        T[4 * q + 3] = fmaf(w[z], r.w, T[4 * q + 3]);
      }
    }
    float vs[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      float o = 0.0f;
#pragma unroll
      for (int k = 0; k < 10; ++k) o = fmaf(shp[k], sb[10 * c + k], o);
      vs[c] = o + vr[c];
    }
#pragma unroll
    for (int a = 0; a < 3; ++a) out[a] = fmaf(T[4 * a + 2], vs[2], fmaf(T[4 * a + 1], vs[1], T[4 * a] * vs[0])) + T[4 * a + 3];
  }
};

// packed FP32x2 FMA (sm_100 FFMA2): d = a * b + c on both lanes
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
  float2 d;
  asm("{\n\t.reg .b64 ra, rb, rc, rd;\n\t"
      "mov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\tmov.b64 rc, {%6, %7};\n\t"
      "fma.rn.f32x2 rd, ra, rb, rc;\n\tmov.b64 {%0, %1}, rd;\n\t}"
      : "=f"(d.x), "=f"(d.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
  return d;
}

#ifndef FSB_LBS_VPT
#define FSB_LBS_VPT 2
#endif
#ifndef FSB_LBS_MESHES
#define FSB_LBS_MESHES 32
#endif
#ifndef FSB_LBS_GROUP_CTAS
#define FSB_LBS_GROUP_CTAS 8
#endif
#ifndef FSB_LBS_MIN_BLOCKS
#define FSB_LBS_MIN_BLOCKS 2
#endif
constexpr int kLbsThreads = 256;
constexpr int kLbsVPT = FSB_LBS_VPT;            // consecutive vertices per thread
constexpr int kLbsMeshes = FSB_LBS_MESHES;      // meshes per group, as pairs
constexpr int kLbsGroupCTAs = FSB_LBS_GROUP_CTAS;  // CTAs along the mesh axis (each walks groups y, y + G, ...)
constexpr int kLbsWarpFloats = 32 * kLbsVPT * 3;   // V floats of one warp's vertices of one mesh

// LBS of a vertex tile for a run of 32-mesh groups.  Each thread keeps its
// two vertices' template records in registers for the whole run and walks
// the meshes two at a time: the per-mesh transforms and shape coefficients
// of a mesh pair are interleaved in shared memory as float2, so every
// multiply-add of the blend, shape offset and apply is one FFMA2 serving
// both meshes.  The next group's transforms are copied in with cp.async
// (4-byte scatter into the interleaved layout) while the current group is
// computed: two shared-memory buffers.
// grid: (ceil(nv / 512), min(groups, kLbsGroupCTAs)); group g of CTA y is
// y, y + gridDim.y, ...
struct LbsStage {
  float2 A2[kLbsMeshes / 2][FSB_NJ * 12];
  float2 S2[kLbsMeshes / 2][10];
};

__device__ __forceinline__ void cp_async4(void* dst, const void* src, bool valid) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(tc::smem_u32(dst)), "l"(src),
               "r"(valid ? 4 : 0)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait1() { asm volatile("cp.async.wait_group 1;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait0() { asm volatile("cp.async.wait_group 0;\n" ::: "memory"); }

// copy group g's transforms and shape coefficients into `st` (zero beyond B)
__device__ __forceinline__ void lbs_stage(LbsStage& st, const float* __restrict__ rel, const float* __restrict__ poses,
                                          int ld_pose, int B, int g) {
  const int m0 = g * kLbsMeshes;
  constexpr int PAIR = 2 * FSB_NJ * 12;  // floats per interleaved pair
  for (int pr = 0; pr < kLbsMeshes / 2; ++pr) {
    float* dst = reinterpret_cast<float*>(st.A2[pr]);
    for (int j = threadIdx.x; j < PAIR; j += kLbsThreads) {
      const int e = j >> 1, m = m0 + 2 * pr + (j & 1);
      const bool ok = m < B;
      cp_async4(dst + j, rel + (int64_t)(ok ? m : 0) * FSB_NJ * 12 + e, ok);
    }
  }
  for (int j = threadIdx.x; j < kLbsMeshes * 10; j += kLbsThreads) {
    const int pr = j / 20, half = (j / 10) & 1, k = j % 10, m = m0 + 2 * pr + half;
    const bool ok = m < B;
    cp_async4(reinterpret_cast<float*>(&st.S2[pr][k]) + half, poses + (int64_t)(ok ? m : 0) * ld_pose + 66 + k, ok);
  }
}

template <int NZ>
__global__ void __launch_bounds__(kLbsThreads, FSB_LBS_MIN_BLOCKS) k_lbs(TemplateDev t, const float* __restrict__ rel,
                                                        const float* __restrict__ poses, int ld_pose, int B,
                                                        float* __restrict__ verts, int* nonfinite) {
  extern __shared__ __align__(16) uint8_t lbs_smem[];
  LbsStage* stage = reinterpret_cast<LbsStage*>(lbs_smem);
  const int ngroups = (B + kLbsMeshes - 1) / kLbsMeshes;
  int g = blockIdx.y;
  if (g >= ngroups) return;  // CTA-uniform
  lbs_stage(stage[0], rel, poses, ld_pose, B, g);
  cp_async_commit();
  VertexTmpl<NZ> vt[kLbsVPT];
  const int v0 = (blockIdx.x * kLbsThreads + threadIdx.x) * kLbsVPT;
#pragma unroll
  for (int q = 0; q < kLbsVPT; ++q) {
    if (v0 + q < t.nv) {
      vt[q].load(t, v0 + q);
    } else {  // past the last vertex: harmless zeros (never stored)
#pragma unroll
      for (int z = 0; z < NZ; ++z) vt[q].j[z] = 0, vt[q].w[z] = 0.0f;
#pragma unroll
      for (int c = 0; c < 3; ++c) vt[q].vr[c] = 0.0f;
#pragma unroll
      for (int k = 0; k < 30; ++k) vt[q].sb[k] = 0.0f;
    }
  }
  const bool live = v0 < t.nv;
  // adjacent vertices of a thread mostly share their joints: where every
  // thread of the warp does, each transform row read from shared memory
  // serves all kLbsVPT vertices (shared-memory wavefronts bound this kernel)
  bool same = true;
#pragma unroll
  for (int q = 1; q < kLbsVPT; ++q)
#pragma unroll
    for (int z = 0; z < NZ; ++z) same = same && vt[q].j[z] == vt[0].j[z];
  const bool reuse = __all_sync(0xffffffffu, same);
  // per-warp output staging: the warp's 64 vertices of a mesh are 192
  // consecutive floats in V; they leave as fully coalesced 128-byte rows
  // (a lane's own 6 floats at a 24-byte stride would touch 3x the L2 sectors)
  float* wout = reinterpret_cast<float*>(lbs_smem + 2 * sizeof(LbsStage)) + (threadIdx.x >> 5) * 2 * kLbsWarpFloats;
  const int lane = threadIdx.x & 31;
  const int vw = (blockIdx.x * kLbsThreads + (threadIdx.x & ~31)) * kLbsVPT;  // the warp's first vertex
  const int nfw = max(0, min(32 * kLbsVPT, t.nv - vw)) * 3;                   // floats of its block
  float2 chk = make_float2(0.0f, 0.0f);
  const float2 one2 = make_float2(1.0f, 1.0f);
  for (int it = 0; g < ngroups; g += gridDim.y, ++it) {
    const int gn = g + gridDim.y;
    if (gn < ngroups) lbs_stage(stage[(it + 1) & 1], rel, poses, ld_pose, B, gn);
    cp_async_commit();
    cp_async_wait1();  // this group's copies have landed
    __syncthreads();
    const LbsStage& st = stage[it & 1];
    const int m0 = g * kLbsMeshes;
    const int nm = min(kLbsMeshes, B - m0);
    const int npair = (nm + 1) / 2;
    {
      for (int pr = 0; pr < npair; ++pr) {
        float2 sh[10];
#pragma unroll
        for (int k = 0; k < 10; ++k) sh[k] = st.S2[pr][k];
        float2 o[kLbsVPT][3];
        // shaped rest positions: v_rest + basis . shape (accumulated onto v_rest)
        float2 vs[kLbsVPT][3];
#pragma unroll
        for (int q = 0; q < kLbsVPT; ++q)
#pragma unroll
          for (int c = 0; c < 3; ++c) {
            float2 acc = make_float2(vt[q].vr[c], vt[q].vr[c]);
#pragma unroll
            for (int k = 0; k < 10; ++k)
              acc = ffma2(make_float2(vt[q].sb[10 * c + k], vt[q].sb[10 * c + k]), sh[k], acc);
            vs[q][c] = acc;
          }
        // sum_z w_z (R_z vs + t_z): each joint's transform applied, then
        // weighted (24 FFMA2 for two joints instead of blending the 3 x 4
        // transforms first, 33)
        if (reuse) {
#pragma unroll
          for (int z = 0; z < NZ; ++z) {
            const float4* row = reinterpret_cast<const float4*>(&st.A2[pr][12 * vt[0].j[z]]);
#pragma unroll
            for (int a = 0; a < 3; ++a) {
              const float4 r01 = row[2 * a], r23 = row[2 * a + 1];  // (R_a0, R_a1 | R_a2, t_a) x 2 meshes
#pragma unroll
              for (int q = 0; q < kLbsVPT; ++q) {
                float2 pa = ffma2(make_float2(r01.x, r01.y), vs[q][0], make_float2(r23.z, r23.w));
                pa = ffma2(make_float2(r01.z, r01.w), vs[q][1], pa);
                pa = ffma2(make_float2(r23.x, r23.y), vs[q][2], pa);
                o[q][a] = ffma2(make_float2(vt[q].w[z], vt[q].w[z]), pa, z == 0 ? make_float2(0.0f, 0.0f) : o[q][a]);
              }
            }
          }
        } else {
#pragma unroll
          for (int q = 0; q < kLbsVPT; ++q)
#pragma unroll
            for (int z = 0; z < NZ; ++z) {
              const float2 wz = make_float2(vt[q].w[z], vt[q].w[z]);
              const float4* row = reinterpret_cast<const float4*>(&st.A2[pr][12 * vt[q].j[z]]);
#pragma unroll
              for (int a = 0; a < 3; ++a) {
                const float4 r01 = row[2 * a], r23 = row[2 * a + 1];
                float2 pa = ffma2(make_float2(r01.x, r01.y), vs[q][0], make_float2(r23.z, r23.w));
                pa = ffma2(make_float2(r01.z, r01.w), vs[q][1], pa);
                pa = ffma2(make_float2(r23.x, r23.y), vs[q][2], pa);
                o[q][a] = ffma2(wz, pa, z == 0 ? make_float2(0.0f, 0.0f) : o[q][a]);
              }
            }
        }
#pragma unroll
        for (int q = 0; q < kLbsVPT; ++q)
#pragma unroll
          for (int a = 0; a < 3; ++a)
            if (v0 + q < t.nv) chk = ffma2(o[q][a], one2, chk);
        // mesh 2 pr (.x lanes) and 2 pr + 1 (.y lanes) through the warp's
        // staging rows
#pragma unroll
        for (int q = 0; q < kLbsVPT; ++q)
#pragma unroll
          for (int a = 0; a < 3; ++a) {
            wout[(lane * kLbsVPT + q) * 3 + a] = o[q][a].x;
            wout[kLbsWarpFloats + (lane * kLbsVPT + q) * 3 + a] = o[q][a].y;
          }
        __syncwarp();
        const int m = m0 + 2 * pr;
#pragma unroll
        for (int half = 0; half < 2; ++half) {
          if (2 * pr + half >= nm) break;
          float* d = verts + ((int64_t)(m + half) * t.nv + vw) * 3;
#pragma unroll
          for (int i = 0; i < 3 * kLbsVPT; ++i) {
            const int idx = 32 * i + lane;
            if (idx < nfw) __stcs(d + idx, wout[kLbsWarpFloats * half + idx]);
          }
        }
        __syncwarp();  // the staging rows are rewritten by the next pair
      }
    }
    __syncthreads();  // buffer it & 1 is refilled two groups later
  }
  cp_async_wait0();
  if (live && nonfinite != nullptr && !(isfinite(chk.x) && isfinite(chk.y))) atomicOr(nonfinite, 1);
}

// ---------------------------------------------------------------------------
// k_lbs_tc: LBS with the shape blend on the tensor cores.
//
// The shape offsets  off[b, v, c] = sum_k basis[v, c, k] * shape[b, k]
// (bodymodel.py:350-356; 30 of the 57 FMA pairs per vertex pair of meshes in
// the all-CUDA-core k_lbs) form a GEMM with K = 10: per 256-vertex tile and
// chunk of FSB_LBS_N meshes, tcgen05.mma (M = 128 rows = the tile's even or
// odd vertices, N = meshes, K = 16 padded) computes them into TMEM with a
// bf16 hi / lo split of both operands (hi.hi + hi.lo + lo.hi; ~2^-16
// relative per product) and fp32 accumulation.  The CUDA cores apply the 1-2
// weighted joint transforms (FFMA2 over mesh pairs).
//
// Shared-memory wavefronts, not FLOPs, bound this kernel (ncu: L1 ~80 %): a
// thread owns two ADJACENT vertices (TMEM lane i = vertices 2i, 2i + 1), so
// where a warp's vertex pairs share their joints (warp-uniform test, decided
// once from the template) each transform row read from shared memory serves
// both; the vertex rows leave through per-warp staging as coalesced stores.
//
// grid (vertex tiles, chunk CTAs); 256 threads: warps w and w + 4 own TMEM
// lane quadrant w % 4 (64 vertices) and take meshes [0, N/2) and [N/2, N) of
// each chunk.
// Per chunk: the k_fk record (transforms + shape images, one bulk copy) lands
// in one of two stage buffers; thread 0 issues the next chunk's MMAs into the
// other TMEM buffer while every thread applies the current one.
// ---------------------------------------------------------------------------
#ifndef FSB_LBS_WARPS
#define FSB_LBS_WARPS 8
#endif
constexpr int kLtWarps = FSB_LBS_WARPS;   // 8: 2 CTAs per SM; 16: 1 CTA per SM, half the chunk barriers
constexpr int kLtThreads = 32 * kLtWarps;
constexpr int kLtN = FSB_LBS_N;
constexpr int kLtCols = 2 * 3 * kLtN;     // TMEM columns per chunk buffer: [even x,y,z | odd x,y,z]
constexpr int kLtTmem = 2 * kLtCols <= 256 ? 256 : 512;  // two chunk buffers, power of two
constexpr int kLtHalf = kLtN / (kLtWarps / 4);  // meshes per warp and chunk
constexpr int kLtRow = 2 * 32 * 3;        // staging floats per (warp, mesh): 64 vertices
constexpr uint32_t kLtBasis = 0;
constexpr uint32_t kLtStage = FSB_LBS_BASIS_BYTES;
constexpr uint32_t kLtOut = kLtStage + 2 * FSB_LBS_REC_BYTES;  // per warp: 2 meshes x kLtRow
constexpr uint32_t kLtSmem = kLtOut + kLtWarps * 2 * kLtRow * 4;
static_assert(2 * kLtCols <= kLtTmem, "two chunk buffers in TMEM");
static_assert(kLtHalf % 2 == 0, "mesh pairs per warp");

template <int NZ>
__device__ __forceinline__ void lbs_apply(const float2* pairA, const int* jj, const float* w, const float2* vs,
                                          float2* o, int nzw) {
#pragma unroll
  for (int z = 0; z < NZ; ++z) {
    if (z >= nzw) break;  // warp-uniform: no vertex of the warp uses slot z
    const float2 wz = make_float2(w[z], w[z]);
    const float4* row = reinterpret_cast<const float4*>(pairA + FSB_LBS_JS * jj[z]);
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const float4 r01 = row[2 * a], r23 = row[2 * a + 1];  // (R_a0, R_a1 | R_a2, t_a) x 2 meshes
      float2 pa = ffma2(make_float2(r01.x, r01.y), vs[0], make_float2(r23.z, r23.w));
      pa = ffma2(make_float2(r01.z, r01.w), vs[1], pa);
      pa = ffma2(make_float2(r23.x, r23.y), vs[2], pa);
      o[a] = ffma2(wz, pa, z == 0 ? make_float2(0.0f, 0.0f) : o[a]);
    }
  }
}

template <int NZ>
__global__ void __launch_bounds__(kLtThreads, 512 / kLtTmem)
    k_lbs_tc(TemplateDev t, const uint8_t* __restrict__ lbs_in, int B, float* __restrict__ verts, int* nonfinite,
             CornerOut cu) {
  extern __shared__ __align__(1024) uint8_t lsm[];
  __shared__ __align__(8) uint64_t bar_basis, bar_stage[2], bar_mma[2];
  __shared__ uint32_t tmem_base;
  const int nchunks = (B + kLtN - 1) / kLtN;
  const int c0 = blockIdx.y;
  if (c0 >= nchunks) return;  // CTA-uniform
  const int G = gridDim.y;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int quad = warp & 3, mh = warp >> 2;  // TMEM lane quadrant, mesh slice of the chunk
  const int vw = blockIdx.x * FSB_LBS_TILE + 64 * quad;  // the warp's first vertex
  const int va = vw + 2 * lane;                           // this thread's vertices va, va + 1
  if (threadIdx.x == 0) {
    tc::mbar_init(&bar_basis, 1);
    for (int i = 0; i < 2; ++i) {
      tc::mbar_init(&bar_stage[i], 1);
      tc::mbar_init(&bar_mma[i], 1);
    }
    tc::mbar_fence_init();
  }
  if (warp == 0) tc::tmem_alloc(&tmem_base, kLtTmem);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = tmem_base;
  auto stage_in = [&](int chunk, int buf) {
    tc::mbar_expect_tx(&bar_stage[buf], FSB_LBS_REC_BYTES);
    tc::bulk_g2s(lsm + kLtStage + buf * FSB_LBS_REC_BYTES, lbs_in + (int64_t)chunk * FSB_LBS_REC_BYTES,
                 FSB_LBS_REC_BYTES, &bar_stage[buf]);
  };
  if (threadIdx.x == 0) {
    tc::mbar_expect_tx(&bar_basis, FSB_LBS_BASIS_BYTES);
    tc::bulk_g2s(lsm + kLtBasis, t.basis_img + (int64_t)blockIdx.x * FSB_LBS_BASIS_BYTES, FSB_LBS_BASIS_BYTES,
                 &bar_basis);
    pdl_wait();  // the chunk records come from k_fk
    stage_in(c0, 0);
    if (c0 + G < nchunks) stage_in(c0 + G, 1);
  }
  // the two vertices' rest positions and skin weights stay in registers
  float vr[2][3], w[2][NZ];
  int jj[2][NZ];
#pragma unroll
  for (int e = 0; e < 2; ++e) {
    const int v = va + e;
    const bool live = v < t.nv;
#pragma unroll
    for (int z = 0; z < NZ; ++z) {
      w[e][z] = live ? __ldg(t.skin_w + (int64_t)v * NZ + z) : 0.0f;
      jj[e][z] = live ? (int)t.skin_j[(int64_t)v * NZ + z] : 0;
    }
#pragma unroll
    for (int c = 0; c < 3; ++c) vr[e][c] = live ? __ldg(t.v_rest + (int64_t)v * 3 + c) : 0.0f;
  }
  // this thread's vertices' slots in the compacted corner buffer (-1: not
  // a projector corner)
  int slot[2];
#pragma unroll
  for (int e = 0; e < 2; ++e) slot[e] = cu.vu != nullptr && va + e < cu.nvslot ? __ldg(cu.vslot + va + e) : -1;
  pdl_wait();  // (the template reads above are constant data)
  // every vertex pair of the warp has one joint set: one row read serves both
  bool same = true;
#pragma unroll
  for (int z = 0; z < NZ; ++z) same = same && jj[0][z] == jj[1][z];
  const bool reuse = __all_sync(0xffffffffu, same);
  // joint slots any vertex of the warp uses (the rest carry weight 0: a
  // fused multiply-add of 0 leaves the sum unchanged, so skipping them is
  // exact).  ~40 % of MHR's 64-vertex blocks ride one bone only: 24 % fewer
  // shared-memory wavefronts at C3 (the kernel time is set by the CTA's
  // slowest warp, so the gain shows in SM issue slots, not in C3's time)
  int zmax = 1;
#pragma unroll
  for (int e = 0; e < 2; ++e)
#pragma unroll
    for (int z = 1; z < NZ; ++z)
      if (w[e][z] != 0.0f) zmax = max(zmax, z + 1);
  const int nzw = __reduce_max_sync(0xffffffffu, zmax);
  // NZ == 2 (MHR): the union of the two vertices' joints (<= 4), each joint's
  // rows read ONCE for both vertices, each vertex with its own weight (0 for
  // a joint it does not use -- exact).  A vertex's joints keep their order
  // within the union (vertex 0's first), so its sum is formed as before.
  // Pairs straddling two bones (7 % of the blocks) read 3 joints' rows
  // instead of 2 x 2.
  int ju[4] = {0, 0, 0, 0};
  float wu[2][4] = {{0.0f, 0.0f, 0.0f, 0.0f}, {0.0f, 0.0f, 0.0f, 0.0f}};
  int nuw = 1;
  if constexpr (NZ == 2) {
    int nu = 0;
#pragma unroll
    for (int e = 0; e < 2; ++e)
#pragma unroll
      for (int z = 0; z < 2; ++z) {
        if (w[e][z] == 0.0f) continue;
        int k = nu;
#pragma unroll
        for (int q = 0; q < 4; ++q)
          if (q < nu && ju[q] == jj[e][z]) k = q;
#pragma unroll
        for (int q = 0; q < 4; ++q)
          if (q == k) {
            ju[q] = jj[e][z];
            wu[e][q] = w[e][z];
          }
        nu += k == nu;
      }
    nuw = max(1, __reduce_max_sync(0xffffffffu, nu));
  }
  const uint32_t sbase = tc::smem_u32(lsm);
  auto issue = [&](int buf) {  // D[e][c] = basis(e, c) . shape^T: hi.hi + hi.lo + lo.hi
    const uint32_t bimg = sbase + kLtStage + buf * FSB_LBS_REC_BYTES + FSB_LBS_REC_A2;
    const uint32_t id = tc::idesc_bf16(128, kLtN);
#pragma unroll
    for (int e = 0; e < 2; ++e)
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const uint32_t d = tmem + buf * kLtCols + (3 * e + c) * kLtN;
        const uint32_t ahi = sbase + kLtBasis + (e * 6 + c) * 4096, alo = ahi + 3 * 4096;
        tc::mma_bf16(d, tc::kmajor_desc(ahi, 16, 0), tc::kmajor_desc(bimg, 16, 0), id, false);
        tc::mma_bf16(d, tc::kmajor_desc(ahi, 16, 0), tc::kmajor_desc(bimg + FSB_LBS_REC_B, 16, 0), id, true);
        tc::mma_bf16(d, tc::kmajor_desc(alo, 16, 0), tc::kmajor_desc(bimg, 16, 0), id, true);
      }
    tc::mma_commit(&bar_mma[buf]);
  };
  if (threadIdx.x == 0) {
    tc::mbar_wait(&bar_basis, 0);
    tc::mbar_wait(&bar_stage[0], 0);
    tc::fence_after();
    issue(0);
  }
  float* stg = reinterpret_cast<float*>(lsm + kLtOut) + warp * 2 * kLtRow;
  const int nfw = max(0, min(64, t.nv - vw)) * 3;  // floats of the warp's vertex block
  const uint32_t tl = tmem + ((uint32_t)(32 * quad) << 16);
  float2 chk = make_float2(0.0f, 0.0f);
  for (int it = 0, ch = c0; ch < nchunks; ++it, ch += G) {
    const int buf = it & 1;
    if (threadIdx.x == 0 && ch + G < nchunks) {  // next chunk's MMAs into the other buffer
      tc::mbar_wait(&bar_stage[buf ^ 1], (uint32_t)(((it + 1) >> 1) & 1));
      tc::fence_after();
      issue(buf ^ 1);
    }
    tc::mbar_wait(&bar_mma[buf], (uint32_t)((it >> 1) & 1));
    tc::fence_after();
    float off[2][3][kLtHalf];
#pragma unroll
    for (int e = 0; e < 2; ++e)
#pragma unroll
      for (int c = 0; c < 3; ++c) tc::tmem_ld8(tl + buf * kLtCols + (3 * e + c) * kLtN + kLtHalf * mh, off[e][c]);
    const float2* A2 = reinterpret_cast<const float2*>(lsm + kLtStage + buf * FSB_LBS_REC_BYTES);
    const int m0 = ch * kLtN + kLtHalf * mh;  // first mesh of this warp's half
    const int nm = min(kLtHalf, B - m0);
#pragma unroll
    for (int p = 0; p < kLtHalf / 2; ++p) {
      if (2 * p >= nm) continue;  // warp-uniform (the last chunk of a batch)
      const float2* pairA = A2 + (kLtHalf / 2 * mh + p) * (FSB_NJ * FSB_LBS_JS);
      float2 vs[2][3], o[2][3];
#pragma unroll
      for (int e = 0; e < 2; ++e)
#pragma unroll
        for (int c = 0; c < 3; ++c) vs[e][c] = make_float2(vr[e][c] + off[e][c][2 * p], vr[e][c] + off[e][c][2 * p + 1]);
      if constexpr (NZ == 2) {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          if (k >= nuw) break;  // warp-uniform
          const float4* row = reinterpret_cast<const float4*>(pairA + FSB_LBS_JS * ju[k]);
#pragma unroll
          for (int a = 0; a < 3; ++a) {
            const float4 r01 = row[2 * a], r23 = row[2 * a + 1];
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              float2 pa = ffma2(make_float2(r01.x, r01.y), vs[e][0], make_float2(r23.z, r23.w));
              pa = ffma2(make_float2(r01.z, r01.w), vs[e][1], pa);
              pa = ffma2(make_float2(r23.x, r23.y), vs[e][2], pa);
              o[e][a] = ffma2(make_float2(wu[e][k], wu[e][k]), pa, k == 0 ? make_float2(0.0f, 0.0f) : o[e][a]);
            }
          }
        }
      } else if (reuse) {  // one read of each transform row for both vertices
#pragma unroll
        for (int z = 0; z < NZ; ++z) {
          if (z >= nzw) break;  // warp-uniform
          const float4* row = reinterpret_cast<const float4*>(pairA + FSB_LBS_JS * jj[0][z]);
#pragma unroll
          for (int a = 0; a < 3; ++a) {
            const float4 r01 = row[2 * a], r23 = row[2 * a + 1];
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              float2 pa = ffma2(make_float2(r01.x, r01.y), vs[e][0], make_float2(r23.z, r23.w));
              pa = ffma2(make_float2(r01.z, r01.w), vs[e][1], pa);
              pa = ffma2(make_float2(r23.x, r23.y), vs[e][2], pa);
              const float2 wz = make_float2(w[e][z], w[e][z]);
              o[e][a] = ffma2(wz, pa, z == 0 ? make_float2(0.0f, 0.0f) : o[e][a]);
            }
          }
        }
      } else {
        lbs_apply<NZ>(pairA, jj[0], w[0], vs[0], o[0], nzw);
        lbs_apply<NZ>(pairA, jj[1], w[1], vs[1], o[1], nzw);
      }
#pragma unroll
      for (int e = 0; e < 2; ++e)
        if (va + e < t.nv)
#pragma unroll
          for (int a = 0; a < 3; ++a) chk = ffma2(o[e][a], make_float2(1.0f, 1.0f), chk);
      // projector corners into the compacted (B, nu, 3) buffer (a warp-contiguous
      // run gathered from the staging rows measured slower)
#pragma unroll
      for (int e = 0; e < 2; ++e)
        if (slot[e] >= 0) {
          float* u = cu.vu + ((int64_t)(m0 + 2 * p) * cu.nu + slot[e]) * 3;
#pragma unroll
          for (int a = 0; a < 3; ++a) u[a] = o[e][a].x;
          if (2 * p + 1 < nm)
#pragma unroll
            for (int a = 0; a < 3; ++a) u[(int64_t)cu.nu * 3 + a] = o[e][a].y;
        }
      // the warp's 64 vertices of meshes m, m + 1 leave as coalesced rows
      // through its staging buffer (2 x 192 floats).  Measured alternatives
      // (DESIGN.md §4): cp.async.bulk of the 16-byte-aligned interior and
      // 1-D TMA tensor stores of 188 / 192-float boxes (a mesh row of 18,439
      // x 12 B is 16-byte aligned only for every fourth mesh) were slower
      // (391 / 356 us vs 271 us at C3): ~750-byte bulk stores do not keep up.
#pragma unroll
      for (int half = 0; half < 2; ++half) {
        float* row = stg + half * kLtRow + 6 * lane;  // this lane's 6 floats (2 vertices x 3)
#pragma unroll
        for (int q = 0; q < 3; ++q) {
          const int e = (2 * q) / 3, a = (2 * q) % 3, e1 = (2 * q + 1) / 3, a1 = (2 * q + 1) % 3;
          *reinterpret_cast<float2*>(row + 2 * q) =
              half ? make_float2(o[e][a].y, o[e1][a1].y) : make_float2(o[e][a].x, o[e1][a1].x);
        }
      }
      __syncwarp();
      const int m = m0 + 2 * p;
#pragma unroll
      for (int half = 0; half < 2; ++half) {
        if (2 * p + half >= nm) break;
        float* dst = verts + ((int64_t)(m + half) * t.nv + vw) * 3;
#pragma unroll
        for (int i = 0; i < 6; ++i) {
          const int idx = 32 * i + lane;
          if (idx < nfw) __stcs(dst + idx, stg[half * kLtRow + idx]);
        }
      }
      __syncwarp();  // the staging rows are rewritten by the next pair
    }
    tc::fence_before();
    __syncthreads();  // TMEM buffer `buf` and stage buffer `buf` are free
    if (threadIdx.x == 0 && ch + 2 * G < nchunks) stage_in(ch + 2 * G, buf);
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc(tmem, kLtTmem);
  if (va < t.nv && nonfinite != nullptr && !(isfinite(chk.x) && isfinite(chk.y))) atomicOr(nonfinite, 1);
}

// ---------------------------------------------------------------------------
// projector input (projection.py:447-465): centre the source mesh on vertex
// 0, bridge the subsampled targets through their three corners, remove the
// subsample centroid.  From given vertices (V_mhr just written, or
// project_batch's input): k_proj_inputs_vc, one CTA per mesh.  Without V_mhr
// the needed MHR vertices are re-skinned from the L2-resident template:
// k_proj_inputs + k_proj_center.
// ---------------------------------------------------------------------------

// Re-skinned path: the targets of one mesh are spread over kProjChunks CTAs
// (one target per thread); each CTA writes its bridged, vertex-0-centred
// targets and its partial sum, and k_proj_center removes the centroid
// (partials added in chunk order, so the result does not depend on the batch).
constexpr int kProjChunks = 8;

// x = sub - centroid (projection.py:464), as fp32 (in place) and/or as the
// bf16 A-tile image of the tensor-core MLP (k_mlp_tc.cu)
__global__ void k_proj_center(float* __restrict__ sub, const float* __restrict__ psum, int B, int n_sub,
                              int write_f32, __nv_bfloat16* __restrict__ xb) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int K = 3 * n_sub;
  if (idx >= (int64_t)B * K) return;
  const int b = (int)(idx / K), i = (int)(idx % K), a = i % 3;
  float s = 0.0f;
#pragma unroll
  for (int q = 0; q < kProjChunks; ++q) s += psum[((int64_t)b * kProjChunks + q) * 3 + a];
  const float v = sub[idx] - s / (float)n_sub;
  if (write_f32) sub[idx] = v;
  if (xb != nullptr) {
    const int KT = (K + 127) / 128;
    const size_t tile = (size_t)(b >> 7) * KT + (i >> 7);
    xb[tile * 16384 + tc::kmajor_off(b & 127, i & 127, 128) / 2] = __float2bfloat16_rn(v);
  }
}

// Re-skinned projector inputs for a group of kProjMeshes meshes: the three
// corner records of this thread's target are read from the template once
// and applied to every mesh of the group (the transforms and shape
// coefficients of the group are staged in shared memory), so a batch of 32
// meshes is 32 CTAs instead of 256.  Same per-target arithmetic and the same
// per-chunk partial-sum order as k_proj_center expects.
constexpr int kProjMeshes = 8;

template <int NZ>
__global__ void __launch_bounds__(256) k_proj_inputs(TemplateDev t, ProjectorDev p, const float* __restrict__ rel,
                                                     const float* __restrict__ poses, int ld_pose, int B, int gpc,
                                                     float* __restrict__ sub, float* __restrict__ psum) {
  // gpc groups of kProjMeshes meshes per CTA (large batches): the corner
  // records stay in registers across the groups
  constexpr int RS = vertex_record_floats(NZ);
  __shared__ __align__(16) float A[kProjMeshes][FSB_NJ * 12];
  __shared__ float shp[kProjMeshes][10];
  __shared__ float v0[kProjMeshes][3];
  __shared__ float rec0[RS];  // template record of vertex 0
  __shared__ float red[kProjMeshes][32][3];
  const int chunk = blockIdx.x, tid = threadIdx.x;
  for (int i = tid; i < RS; i += blockDim.x) rec0[i] = __ldg(t.rec + i);
  const int per = (p.n_sub + kProjChunks - 1) / kProjChunks;
  const int i = chunk * per + tid;
  const bool act = tid < per && i < p.n_sub;
  VertexTmpl<NZ> vt[3];
  float wc[3];
  if (act)
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      vt[c].load(t, p.corners[3 * i + c]);
      wc[c] = p.bw[3 * i + c];
    }
  const int warp = tid / 32, lane = tid % 32;
#pragma unroll 1
  for (int gi = 0; gi < gpc; ++gi) {
    const int m0 = ((int)blockIdx.y * gpc + gi) * kProjMeshes;
    if (m0 >= B) break;  // CTA-uniform
    const int nm = min(kProjMeshes, B - m0);
    if (gi > 0) __syncthreads();  // the previous group's A / shp / red reads are done
    for (int k = tid; k < nm * FSB_NJ * 12; k += blockDim.x) (&A[0][0])[k] = rel[(int64_t)m0 * FSB_NJ * 12 + k];
    for (int k = tid; k < nm * 10; k += blockDim.x)
      shp[k / 10][k % 10] = poses[(int64_t)(m0 + k / 10) * ld_pose + 66 + k % 10];
    __syncthreads();
    if (tid < nm) {
      VertexTmpl<NZ> r0;
      r0.unpack(rec0);
      r0.apply(A[tid], shp[tid], v0[tid]);
    }
    __syncthreads();
    // per-mesh sums are reduced after the loop (independent shuffle chains)
    float acc[kProjMeshes][3];
#pragma unroll
    for (int m = 0; m < kProjMeshes; ++m) {
      acc[m][0] = acc[m][1] = acc[m][2] = 0.0f;
      if (act && m < nm) {
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          float o[3];
          vt[c].apply(A[m], shp[m], o);
#pragma unroll
          for (int a = 0; a < 3; ++a) acc[m][a] = fmaf(wc[c], o[a] - v0[m][a], acc[m][a]);
        }
#pragma unroll
        for (int a = 0; a < 3; ++a) sub[((int64_t)(m0 + m) * p.n_sub + i) * 3 + a] = acc[m][a];
      }
    }
#pragma unroll
    for (int m = 0; m < kProjMeshes; ++m)
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        const float r = warp_sum(acc[m][a]);
        if (lane == 0) red[m][warp][a] = r;
      }
    __syncthreads();
    if (tid < 3 * nm) {
      const int m = tid / 3, a = tid % 3;
      float tot = 0.0f;
      for (int w = 0; w < (int)blockDim.x / 32; ++w) tot += red[m][w][a];
      psum[((int64_t)(m0 + m) * kProjChunks + chunk) * 3 + a] = tot;
    }
  }
}

// Projector input of one mesh per CTA from its skinned vertices
// (projection.py:447-465): centre on vertex 0, bridge each target through
// its three corners, remove the subsample centroid, and write x as fp32
// and/or straight into the bf16 A-tile image of the tensor-core MLP -- the
// centroid is a CTA reduction (fixed order, so a mesh gives the same bits
// in any batch), no partial-sum buffer and no second kernel.
// STAGED: V is the LBS kernel's compacted (B, nu, 3) corner buffer; a CTA
// walks `mpc` consecutive meshes, each mesh's nu x 12 bytes bulk-copied
// into one of two shared-memory buffers (the next mesh lands while this one
// is bridged), and keeps its targets' corners and weights in registers
// across them.  The bridged targets are collected in shared memory (xs) and
// leave after the centroid removal as whole rows: fp32 with coalesced
// stores, the bf16 A-tile image as one 16-byte K-major chunk (8 consecutive
// k of the mesh's row) per store.
constexpr int kProjVcThreads = 512, kProjVcPer = 4;  // targets per thread (n_sub <= 2048)

template <bool STAGED>
__global__ void __launch_bounds__(kProjVcThreads) k_proj_inputs_vc(const float* __restrict__ V, int nv,
                                                                   ProjectorDev p, const int32_t* __restrict__ corners,
                                                                   float* __restrict__ x32,
                                                                   __nv_bfloat16* __restrict__ xb, int B, int mpc,
                                                                   __nv_bfloat16* __restrict__ xb_lo) {
  __shared__ float red[kProjVcThreads / 32][3];
  __shared__ float cen[3];
  __shared__ __align__(8) uint64_t bar[2];
  extern __shared__ __align__(16) float vsm[];
  const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
  const int K = 3 * p.n_sub, KT = (K + 127) / 128;
  float* xs = vsm + (STAGED ? 2 * nv * 3 : 0);  // (K) bridged targets, vertex-0 centred
  const int b0 = blockIdx.x * mpc, nb = min(mpc, B - b0);
  int cr[kProjVcPer][3];
  float wc[kProjVcPer][3];
#pragma unroll
  for (int q = 0; q < kProjVcPer; ++q) {
    const int t = tid + q * kProjVcThreads;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      cr[q][c] = t < p.n_sub ? __ldg(corners + 3 * t + c) : 0;
      wc[q][c] = t < p.n_sub ? __ldg(p.bw + 3 * t + c) : 0.0f;
    }
  }
  const uint32_t vbytes = (uint32_t)nv * 12;
  if (STAGED && tid == 0) {
    tc::mbar_init(&bar[0], 1);
    tc::mbar_init(&bar[1], 1);
    tc::mbar_fence_init();
  }
  if (STAGED) __syncthreads();
  pdl_wait();
  auto fetch = [&](int i) {  // mesh b0 + i into buffer i & 1 (thread 0)
    tc::mbar_expect_tx(&bar[i & 1], vbytes);
    tc::bulk_g2s(vsm + (i & 1) * nv * 3, V + (int64_t)(b0 + i) * nv * 3, vbytes, &bar[i & 1]);
  };
  if (STAGED && tid == 0) {
    fetch(0);
    if (nb > 1) fetch(1);
  }
  for (int i = 0; i < nb; ++i) {
    const int b = b0 + i;
    const float* Vb;
    if (STAGED) {
      tc::mbar_wait(&bar[i & 1], (uint32_t)((i >> 1) & 1));
      Vb = vsm + (i & 1) * nv * 3;
    } else {
      Vb = V + (int64_t)b * nv * 3;
    }
    const float o0 = Vb[0], o1 = Vb[1], o2 = Vb[2];
    float part[3] = {0.0f, 0.0f, 0.0f};
#pragma unroll
    for (int q = 0; q < kProjVcPer; ++q) {
      const int t = tid + q * kProjVcThreads;
      if (t < p.n_sub) {
        float acc[3] = {0.0f, 0.0f, 0.0f};
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          const float* vc = Vb + 3 * cr[q][c];
          acc[0] = fmaf(wc[q][c], vc[0] - o0, acc[0]);
          acc[1] = fmaf(wc[q][c], vc[1] - o1, acc[1]);
          acc[2] = fmaf(wc[q][c], vc[2] - o2, acc[2]);
        }
#pragma unroll
        for (int a = 0; a < 3; ++a) {
          part[a] += acc[a];
          xs[3 * t + a] = acc[a];
        }
      }
    }
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const float r = warp_sum(part[a]);
      if (lane == 0) red[warp][a] = r;
    }
    __syncthreads();  // xs, red complete; buffer i & 1 no longer read
    if (STAGED && tid == 0 && i + 2 < nb) {
      tc::fence_async_smem();
      fetch(i + 2);
    }
    if (tid < 3) {
      float sum = 0.0f;
      for (int w = 0; w < kProjVcThreads / 32; ++w) sum += red[w][tid];
      cen[tid] = sum / (float)p.n_sub;
    }
    __syncthreads();
    const float c0 = cen[0], c1 = cen[1], c2 = cen[2];
    auto val = [&](int k) { return k < K ? xs[k] - (k % 3 == 0 ? c0 : (k % 3 == 1 ? c1 : c2)) : 0.0f; };
    if (x32 != nullptr)
      for (int k = tid; k < K; k += kProjVcThreads) x32[(int64_t)b * K + k] = val(k);
    if (xb != nullptr) {
      uint8_t* img = reinterpret_cast<uint8_t*>(xb) + (size_t)(b >> 7) * KT * 32768;
      for (int ch = tid; ch < (K + 7) / 8; ch += kProjVcThreads) {
        const int k0 = 8 * ch;
        float v8[8];
        *reinterpret_cast<float4*>(v8) = *reinterpret_cast<const float4*>(xs + k0);  // (xs: K + 8 floats)
        *reinterpret_cast<float4*>(v8 + 4) = *reinterpret_cast<const float4*>(xs + k0 + 4);
        uint32_t w[4];
        int r = k0 % 3;  // coordinate of k0
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          v8[j] = k0 + j < K ? v8[j] - (r == 0 ? c0 : (r == 1 ? c1 : c2)) : 0.0f;
          r = r == 2 ? 0 : r + 1;
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const __nv_bfloat162 h = __floats2bfloat162_rn(v8[2 * j], v8[2 * j + 1]);
          w[j] = *reinterpret_cast<const uint32_t*>(&h);
        }
        const size_t off = (size_t)(k0 >> 7) * 32768 + tc::kmajor_off(b & 127, k0 & 127, 128);
        *reinterpret_cast<uint4*>(img + off) = make_uint4(w[0], w[1], w[2], w[3]);
        if (xb_lo != nullptr) {  // fp32 mode: the remainders v - bf16(v)
          uint32_t wl[4];
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const __nv_bfloat162 h = *reinterpret_cast<const __nv_bfloat162*>(&w[j]);
            const float2 hf = __bfloat1622float2(h);
            const __nv_bfloat162 l = __floats2bfloat162_rn(v8[2 * j] - hf.x, v8[2 * j + 1] - hf.y);
            wl[j] = *reinterpret_cast<const uint32_t*>(&l);
          }
          *reinterpret_cast<uint4*>(reinterpret_cast<uint8_t*>(xb_lo) + (size_t)(b >> 7) * KT * 32768 + off) =
              make_uint4(wl[0], wl[1], wl[2], wl[3]);
        }
      }
    }
    __syncthreads();  // xs, red and cen are rewritten by the next mesh
  }
}

// ---------------------------------------------------------------------------
// fp32 GEMM for the projector MLP: C = act(A @ W + b) * mask, A (M, K) with
// leading dim lda, W (K, N) row-major.  64x64 tiles, 4x4 per thread.  The
// K axis is cut into a fixed number of chunks per layer (blockIdx.z), chosen
// from K alone: each chunk's partial sum lands in P[split][M][N] and a
// second kernel adds the partials in split order.  The partition never
// depends on M, so a mesh projected in a batch of 4096 is bit-identical to
// the same mesh projected alone, while a batch of 32 still fills the GPU
// (W1 is 4500 x 512: 8 column tiles alone would occupy 8 SMs).
// ---------------------------------------------------------------------------
constexpr int kGT = 64, kGK = 16;

__global__ void __launch_bounds__(256) k_gemm_f32(const float* __restrict__ A, int lda,
                                                   const float* __restrict__ W, const float* __restrict__ bias,
                                                   const float* __restrict__ mask, float* __restrict__ C, int ldc,
                                                   int M, int N, int K, int relu, int* nonfinite, int kchunk,
                                                   float* __restrict__ P, int accumulate = 0) {
  __shared__ __align__(16) float As[kGK][kGT + 4];
  __shared__ __align__(16) float Bs[kGK][kGT + 4];
  const int tid = threadIdx.x, tx = tid % 16, ty = tid / 16;
  const int m0 = blockIdx.y * kGT, n0 = blockIdx.x * kGT;
  const int kb0 = blockIdx.z * kchunk, kb1 = min(K, kb0 + kchunk);
  float acc[4][4] = {};
  for (int k0 = kb0; k0 < kb1; k0 += kGK) {
    for (int i = tid; i < kGT * kGK; i += 256) {
      const int r = i / kGK, kk = i % kGK;  // A tile: coalesced along k
      const int gm = m0 + r, gk = k0 + kk;
      As[kk][r] = (gm < M && gk < kb1) ? A[(int64_t)gm * lda + gk] : 0.0f;
      const int kb = i / kGT, c = i % kGT;  // W tile: coalesced along n
      const int wk = k0 + kb, wn = n0 + c;
      Bs[kb][c] = (wk < kb1 && wn < N) ? __ldg(W + (int64_t)wk * N + wn) : 0.0f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < kGK; ++kk) {
      const float4 a = *reinterpret_cast<const float4*>(&As[kk][ty * 4]);
      const float4 w = *reinterpret_cast<const float4*>(&Bs[kk][tx * 4]);
      const float av[4] = {a.x, a.y, a.z, a.w}, wv[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(av[i], wv[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int gm = m0 + ty * 4 + i;
    if (gm >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int gn = n0 + tx * 4 + j;
      if (gn >= N) continue;
      if (P != nullptr) {
        P[((int64_t)blockIdx.z * M + gm) * N + gn] = acc[i][j];
        continue;
      }
      float v = acc[i][j] + bias[gn];
      if (relu) v = fmaxf(v, 0.0f);
      if (mask != nullptr) v *= mask[gn];
      if (accumulate) v += C[(int64_t)gm * ldc + gn];  // residual stream (k_enc_f32.cu)
      flag_nonfinite(nonfinite, v);
      C[(int64_t)gm * ldc + gn] = v;
    }
  }
}

// C = act(A W + bias) (+ C): the fp32 encoder's GEMMs (large M, no split)
cudaError_t launch_gemm_f32_acc(const float* A, int lda, const float* W, const float* bias, float* C, int ldc, int M,
                                int N, int K, int relu, int accumulate, cudaStream_t st) {
  if (M == 0 || N == 0) return cudaSuccess;
  dim3 grid((N + kGT - 1) / kGT, (M + kGT - 1) / kGT, 1);
  if (grid.y > 65535) return cudaErrorInvalidValue;
  k_gemm_f32<<<grid, 256, 0, st>>>(A, lda, W, bias, nullptr, C, ldc, M, N, K, relu, nullptr, K, nullptr, accumulate);
  return cudaGetLastError();
}

// C = act(sum_s P[s] + b) * mask, partials added in split order
__global__ void k_splitk_reduce(const float* __restrict__ P, int S, int M, int N, const float* __restrict__ bias,
                                const float* __restrict__ mask, float* __restrict__ C, int ldc, int relu,
                                int* nonfinite) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (int64_t)M * N) return;
  const int m = (int)(idx / N), n = (int)(idx % N);
  float v = P[idx];
  for (int s = 1; s < S; ++s) v += P[(int64_t)s * M * N + idx];
  v += bias[n];
  if (relu) v = fmaxf(v, 0.0f);
  if (mask != nullptr) v *= mask[n];
  flag_nonfinite(nonfinite, v);
  C[(int64_t)m * ldc + n] = v;
}

// ---------------------------------------------------------------------------
// launchers
// ---------------------------------------------------------------------------
cudaError_t launch_fk(const float* poses, int ld_pose, int B, const float* grest, float* joints, float* rel,
                      cudaStream_t st, uint8_t* lbs_in, const DenoiseW* dn, int* nonfinite) {
  if (B == 0) return cudaSuccess;
  const DenoiseW d = dn ? *dn : DenoiseW{nullptr, nullptr, nullptr, nullptr, 0};
  // (poses is written only with a denoiser: the caller passes a writable theta then)
  return launch_pdl(k_fk, dim3((B + 3) / 4), dim3(128), 0, st, const_cast<float*>(poses), ld_pose, B, grest, joints,
                    rel, lbs_in, d, nonfinite);
}

// grid: (vertex tiles, chunk CTAs); each chunk CTA walks chunks y, y + G, ...
// with G chosen so the grid fills ~2 CTAs per SM
cudaError_t launch_lbs_tc(const TemplateDev& t, const uint8_t* lbs_in, int B, float* verts, int* nonfinite,
                          cudaStream_t st, CornerOut cu) {
  if (B == 0) return cudaSuccess;
  if (t.basis_img == nullptr) return cudaErrorInvalidValue;
  const int tiles = (t.nv + FSB_LBS_TILE - 1) / FSB_LBS_TILE;
  const int nchunks = (B + kLtN - 1) / kLtN;
  int G = (512 / kLtTmem) * 148 / tiles;  // whole waves
  // at least two chunks per CTA: a small batch (the frame path's 32 meshes =
  // 2 chunks) then runs one CTA per vertex tile, whose setup (48 KB basis
  // image, template registers, TMEM) serves both chunks -- LBS saturated cost
  // 3.08 -> 2.68 us per batch, C2 +0.8 % (FSB_LBS_MINCH overrides)
  static const int min_chunks = [] {
    const char* e = getenv("FSB_LBS_MINCH");
    return e ? atoi(e) : 2;
  }();
  if (min_chunks > 1 && G > (nchunks + min_chunks - 1) / min_chunks) G = (nchunks + min_chunks - 1) / min_chunks;
  G = G < 1 ? 1 : (G > nchunks ? nchunks : G);
  dim3 grid(tiles, G);
  switch (t.nnz) {
    case 2: return launch_pdl(k_lbs_tc<2>, grid, dim3(kLtThreads), kLtSmem, st, t, lbs_in, B, verts, nonfinite, cu);
    case 4: return launch_pdl(k_lbs_tc<4>, grid, dim3(kLtThreads), kLtSmem, st, t, lbs_in, B, verts, nonfinite, cu);
    case 8: return launch_pdl(k_lbs_tc<8>, grid, dim3(kLtThreads), kLtSmem, st, t, lbs_in, B, verts, nonfinite, cu);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_lbs(const TemplateDev& t, const float* rel, const float* poses, int ld_pose, int B, float* verts,
                       int* nonfinite, cudaStream_t st) {
  if (B == 0) return cudaSuccess;
  const int ngroups = (B + kLbsMeshes - 1) / kLbsMeshes;
  dim3 grid((t.nv + kLbsThreads * kLbsVPT - 1) / (kLbsThreads * kLbsVPT),
            ngroups < kLbsGroupCTAs ? ngroups : kLbsGroupCTAs);
  const size_t smem = 2 * sizeof(LbsStage) + kLbsThreads / 32 * 2 * kLbsWarpFloats * sizeof(float);
  switch (t.nnz) {
    case 2: k_lbs<2><<<grid, kLbsThreads, smem, st>>>(t, rel, poses, ld_pose, B, verts, nonfinite); break;
    case 4: k_lbs<4><<<grid, kLbsThreads, smem, st>>>(t, rel, poses, ld_pose, B, verts, nonfinite); break;
    case 8: k_lbs<8><<<grid, kLbsThreads, smem, st>>>(t, rel, poses, ld_pose, B, verts, nonfinite); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

cudaError_t init_attrs_body() {
  const int smem = (int)(2 * sizeof(LbsStage) + kLbsThreads / 32 * 2 * kLbsWarpFloats * sizeof(float));
  cudaError_t e = cudaFuncSetAttribute(k_lbs<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(k_lbs<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(k_lbs<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(k_lbs_tc<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kLtSmem);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(k_lbs_tc<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kLtSmem);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(k_lbs_tc<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kLtSmem);
  return e;
}

static inline int proj_threads(const ProjectorDev& p) {
  const int per = (p.n_sub + kProjChunks - 1) / kProjChunks;
  return (per + 31) / 32 * 32;
}

static cudaError_t launch_proj_center(const ProjectorDev& p, int B, float* sub, const float* psum, bool f32,
                                      __nv_bfloat16* xb, cudaStream_t st) {
  const int64_t tot = (int64_t)B * 3 * p.n_sub;
  k_proj_center<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(sub, psum, B, p.n_sub, f32 ? 1 : 0, xb);
  return cudaGetLastError();
}

// sub: (B, n_sub, 3) fp32 scratch that receives x when f32 is set;
// xb: the bf16 A-tile image (or null)
cudaError_t launch_proj_inputs(const TemplateDev& t, const ProjectorDev& p, const float* rel, const float* poses,
                               int ld_pose, int B, float* sub, bool f32, __nv_bfloat16* xb, float* psum,
                               cudaStream_t st) {
  if (B == 0) return cudaSuccess;
  const int nt = proj_threads(p);
  if (nt > 256) return cudaErrorInvalidValue;  // n_sub <= 2048 (launch bounds)
  // small batches: one group of kProjMeshes per CTA (latency); large ones
  // (C3): 8 groups per CTA so each target's corner records are read once per
  // 64 meshes
  const int groups = (B + kProjMeshes - 1) / kProjMeshes;
  const int gpc = B >= 1024 ? 8 : 1;
  const dim3 grid(kProjChunks, (groups + gpc - 1) / gpc);
  switch (t.nnz) {
    case 2: k_proj_inputs<2><<<grid, nt, 0, st>>>(t, p, rel, poses, ld_pose, B, gpc, sub, psum); break;
    case 4: k_proj_inputs<4><<<grid, nt, 0, st>>>(t, p, rel, poses, ld_pose, B, gpc, sub, psum); break;
    case 8: k_proj_inputs<8><<<grid, nt, 0, st>>>(t, p, rel, poses, ld_pose, B, gpc, sub, psum); break;
    default: return cudaErrorInvalidValue;
  }
  cudaError_t e = cudaGetLastError();
  return e != cudaSuccess ? e : launch_proj_center(p, B, sub, psum, f32, xb, st);
}

cudaError_t launch_proj_inputs_v(const float* V, int nv, const ProjectorDev& p, int B, float* sub, bool f32,
                                 __nv_bfloat16* xb, float* psum, cudaStream_t st, bool compacted,
                                 __nv_bfloat16* xb_lo) {
  if (B == 0) return cudaSuccess;
  if (p.n_sub > kProjVcThreads * kProjVcPer) return cudaErrorInvalidValue;
  (void)psum;
  // compacted: V is the LBS kernel's (B, nu, 3) corner buffer, indexed by slot
  static bool attr = false;
  if (!attr) {
    for (auto* k : {k_proj_inputs_vc<false>, k_proj_inputs_vc<true>}) {
      cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      if (e != cudaSuccess) return e;
    }
    attr = true;
  }
  const size_t xs_bytes = (size_t)p.n_sub * 12 + 32;
  if (!compacted)
    return launch_pdl(k_proj_inputs_vc<false>, dim3(B), dim3(kProjVcThreads), xs_bytes, st, V, nv, p, p.corners,
                      f32 ? sub : nullptr, xb, B, 1, xb_lo);
  // meshes per CTA: 1 while that leaves SMs idle (latency of small batches),
  // up to 4 for large batches (register-held corners reused, loads overlapped)
  const int mpc = B >= 4 * 148 * 2 ? 4 : (B >= 2 * 148 * 2 ? 2 : 1);
  return launch_pdl(k_proj_inputs_vc<true>, dim3((B + mpc - 1) / mpc), dim3(kProjVcThreads),
                    (size_t)nv * 24 + xs_bytes, st, V, nv, p, p.ucorners, f32 ? sub : nullptr, xb, B, mpc, xb_lo);
}

// number of K chunks of a layer: a function of K only (batch independence);
// ~288-wide chunks, at most 16
int gemm_f32_splits(int K) {
  const int s = (K + 287) / 288;
  return s < 1 ? 1 : (s > 16 ? 16 : s);
}

cudaError_t launch_gemm_f32(const float* A, int lda, const float* W, const float* bias, const float* mask, float* C,
                            int ldc, int M, int N, int K, int relu, int* nonfinite, float* partial,
                            cudaStream_t st) {
  if (M == 0) return cudaSuccess;
  const int S = partial ? gemm_f32_splits(K) : 1;
  int kchunk = (K + S - 1) / S;
  kchunk = (kchunk + kGK - 1) / kGK * kGK;
  const int Seff = (K + kchunk - 1) / kchunk;
  dim3 grid((N + kGT - 1) / kGT, (M + kGT - 1) / kGT, Seff);
  k_gemm_f32<<<grid, 256, 0, st>>>(A, lda, W, bias, mask, C, ldc, M, N, K, relu, nonfinite, kchunk,
                                   Seff > 1 ? partial : nullptr);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess || Seff == 1) return e;
  const int64_t tot = (int64_t)M * N;
  k_splitk_reduce<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(partial, Seff, M, N, bias, mask, C, ldc, relu,
                                                                 nonfinite);
  return cudaGetLastError();
}

// projection.bridge (projection.py:187-203): out[b, t] = sum_c w[t, c] V[b, corner[t, c]]
__global__ void k_bridge(const float* __restrict__ V, int B, int nv, const int32_t* __restrict__ corners,
                         const float* __restrict__ w, int nt, float* __restrict__ out) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (int64_t)B * nt) return;
  const int b = (int)(idx / nt), t = (int)(idx % nt);
  const float* Vb = V + (int64_t)b * nv * 3;
  float acc[3] = {0.0f, 0.0f, 0.0f};
  for (int c = 0; c < 3; ++c) {
    const int v = corners[3 * t + c];
    const float wc = w[3 * t + c];
    for (int a = 0; a < 3; ++a) acc[a] = fmaf(wc, Vb[3 * v + a], acc[a]);
  }
  for (int a = 0; a < 3; ++a) out[idx * 3 + a] = acc[a];
}

cudaError_t launch_bridge(const float* V, int B, int nv, const int32_t* corners, const float* w, int nt, float* out,
                          cudaStream_t st) {
  const int64_t tot = (int64_t)B * nt;
  if (tot == 0) return cudaSuccess;
  k_bridge<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(V, B, nv, corners, w, nt, out);
  return cudaGetLastError();
}
