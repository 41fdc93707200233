// Shared definitions for the sm_100a kernels of the frame -> SMPL path.
#pragma once
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>

#define FSB_NJ 22
#define FSB_PARAM_DIM 76
#define FSB_PROMPT_DIM 8


// kinematic tree (reference bodymodel.py:29-32); identical for mhr and smpl
__constant__ __device__ static const int8_t kParents[FSB_NJ] = {
    -1, 0, 1, 2, 3, 4, 0, 6, 7, 8, 0, 10, 11, 12, 3, 14, 15, 16, 3, 18, 19, 20};

// Programmatic dependent launch (frame-path kernels are launched with
// launch_pdl): the next kernel of the stream may be scheduled while this one
// finishes; every such kernel calls pdl_wait() before it touches data a
// predecessor wrote (and before writing anything a predecessor reads), and
// pdl_trigger() once its own prologue-hiding point is reached.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory"); }

#ifndef FSB_NO_PDL
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}
#else
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args&&... args) {
  kernel<<<grid, block, smem, st>>>(static_cast<KArgs>(args)...);
  return cudaGetLastError();
}
#endif

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// sets the context's device-side non-finite flag (mapped to NumericError)
// 2^x on the SFU (MUFU.EX2, ~2 ulp); arguments are <= 0 where it is used
__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ void flag_nonfinite(int* flag, float v) {
  if (flag != nullptr && !isfinite(v)) atomicOr(flag, 1);
}

// ---------------------------------------------------------------------------
// forward kinematics (reference bodymodel.py:172-240).  One warp per pose:
// lanes 0..21 evaluate Rodrigues for their joint, then lane 0 walks the
// chain in joint order (parents[j] < j).  Output per joint: world rotation
// rw[9], world translation tw[3], rest-relative translation at[3].
// ---------------------------------------------------------------------------
struct FKOut {
  float rw[FSB_NJ][9];
  float tw[FSB_NJ][3];
  float at[FSB_NJ][3];
};

// FAST: MUFU sine/cosine and approximate division (bf16-mode kernels, where
// the bar is MPJPE <= 0.5 mm; abs error of __sinf/__cosf ~1e-6 for |x| < pi).
template <bool FAST = false>
__device__ __forceinline__ void rodrigues3(float wx, float wy, float wz, float* r) {
  const float t2 = __fadd_rn(__fadd_rn(__fmul_rn(wx, wx), __fmul_rn(wy, wy)), __fmul_rn(wz, wz));
  const bool small = t2 < 1e-12f;
  float s, c;
  if (small) {
    s = 1.0f - t2 * (1.0f / 6.0f);
    c = 0.5f - t2 * (1.0f / 24.0f);
  } else {
    const float th = sqrtf(t2);
    float sn, cs;
    if (FAST) {
      __sincosf(th, &sn, &cs);
      s = __fdividef(sn, th);
      c = __fdividef(1.0f - cs, t2);
    } else {
      sincosf(th, &sn, &cs);
      s = sn / th;
      c = (1.0f - cs) / t2;
    }
  }
  r[0] = 1.0f - (wy * wy + wz * wz) * c;
  r[1] = wx * wy * c - wz * s;
  r[2] = wx * wz * c + wy * s;
  r[3] = wx * wy * c + wz * s;
  r[4] = 1.0f - (wx * wx + wz * wz) * c;
  r[5] = wy * wz * c - wx * s;
  r[6] = wx * wz * c - wy * s;
  r[7] = wy * wz * c + wx * s;
  r[8] = 1.0f - (wx * wx + wy * wy) * c;
}

// depth of each joint in the kinematic tree (depth[j] = depth[parent] + 1)
__constant__ __device__ static const int8_t kDepth[FSB_NJ] = {0, 1, 2, 3, 4, 5, 1, 2, 3, 4, 1,
                                                            2, 3, 4, 4, 5, 6, 7, 4, 5, 6, 7};

// warp-cooperative FK; `pose` points at the 66 rotation params (shared or
// global), `grest` at the 22x3 rest joints.  All lanes of the warp must call.
// Lane j owns joint j: Rodrigues in parallel, then the chain is composed one
// tree level at a time (8 levels instead of 22 serial joints), each joint
// with the reference's fixed three-term accumulation order.
template <bool FAST = false>
__device__ __forceinline__ void fk_warp(const float* pose, const float* grest, FKOut& o, int lane) {
  const int j = lane;
  // (parent and depth read once: the lanes' distinct constant-bank addresses
  // serialise, and a per-level reload of kDepth[j] was the kernel's hottest
  // stall)
  const int p = j < FSB_NJ ? kParents[j] : -1;
  const int dj = j < FSB_NJ ? (int)kDepth[j] : -1;
  float loc[9], tl[3], g[3];
  if (j < FSB_NJ) {
    rodrigues3<FAST>(pose[3 * j], pose[3 * j + 1], pose[3 * j + 2], loc);
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      g[a] = grest[3 * j + a];
      tl[a] = (p < 0) ? g[a] : g[a] - grest[3 * p + a];
    }
    if (p < 0) {
#pragma unroll
      for (int e = 0; e < 9; ++e) o.rw[0][e] = loc[e];
#pragma unroll
      for (int a = 0; a < 3; ++a) o.tw[0][a] = tl[a];
    }
  }
  __syncwarp();
#pragma unroll 1
  for (int lvl = 1; lvl < 8; ++lvl) {
    if (dj == lvl) {
      float rp[9], tp[3];
#pragma unroll
      for (int e = 0; e < 9; ++e) rp[e] = o.rw[p][e];
#pragma unroll
      for (int a = 0; a < 3; ++a) tp[a] = o.tw[p][a];
#pragma unroll
      for (int a = 0; a < 3; ++a) {
#pragma unroll
        for (int b = 0; b < 3; ++b)
          o.rw[j][3 * a + b] = rp[3 * a] * loc[b] + rp[3 * a + 1] * loc[3 + b] + rp[3 * a + 2] * loc[6 + b];
        o.tw[j][a] = (rp[3 * a] * tl[0] + rp[3 * a + 1] * tl[1] + rp[3 * a + 2] * tl[2]) + tp[a];
      }
    }
    __syncwarp();
  }
  if (j < FSB_NJ) {
    const float* rj = o.rw[j];
#pragma unroll
    for (int a = 0; a < 3; ++a)
      o.at[j][a] = o.tw[j][a] - (rj[3 * a] * g[0] + rj[3 * a + 1] * g[1] + rj[3 * a + 2] * g[2]);
  }
  __syncwarp();
}

// ---------------------------------------------------------------------------
// kinematic-prior denoiser (reference projection.py:684-697,
// _denoise_forward :684-686): out = x + (relu(x W1 + b1) W2 + b2) on a
// (63,) body pose, one warp.  Both products follow numkit.matmul
// (numkit.py:78-90): every dot product is a left-to-right sum from +0 with a
// separately rounded product and add, so the result is bit-identical to the
// reference.  Lane j owns hidden units j, j + 32, ...; outputs m = lane,
// lane + 32.  Used by k_denoise and as the optional epilogue of the SMPL FK
// (k_fk) on the frame path.
// ---------------------------------------------------------------------------
struct DenoiseW {
  const float* w1;  // (63, H)
  const float* b1;
  const float* w2;  // (H, 63)
  const float* b2;
  int H;            // 0: no denoiser
};
#define FSB_DN_IN 63
#define FSB_DN_MAX_HIDDEN 128

// xs: the pose (shared, 63); hs: hidden scratch (shared, H); out: 63 values
// (may alias nothing the warp still reads)
__device__ __forceinline__ void denoise_warp(const float* xs, float* hs, const DenoiseW& d, int lane, float* out,
                                             int* nonfinite) {
  for (int j = lane; j < d.H; j += 32) {
    float acc = 0.0f;
    for (int k = 0; k < FSB_DN_IN; ++k) acc = __fadd_rn(acc, __fmul_rn(xs[k], __ldg(d.w1 + (int64_t)k * d.H + j)));
    hs[j] = fmaxf(__fadd_rn(acc, __ldg(d.b1 + j)), 0.0f);
  }
  __syncwarp();
  for (int m = lane; m < FSB_DN_IN; m += 32) {
    float acc = 0.0f;
    for (int j = 0; j < d.H; ++j) acc = __fadd_rn(acc, __fmul_rn(hs[j], __ldg(d.w2 + (int64_t)j * FSB_DN_IN + m)));
    const float v = __fadd_rn(xs[m], __fadd_rn(acc, __ldg(d.b2 + m)));
    flag_nonfinite(nonfinite, v);
    out[m] = v;
  }
  __syncwarp();
}

