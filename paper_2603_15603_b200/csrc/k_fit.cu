// projection.fit_batch on the GPU (reference projection.py:211-370; SURVEY
// §8(f) row 2): the iterative MHR -> SMPL conversion the feed-forward
// projector replaces.  Per mesh, `steps` Adam iterations (_Adam
// :237-263, cosine-decayed step size :361-363) on
//     L(theta) = sum_v |skin(theta)_v - target_v|^2
//              + lambda_pose |theta[3:66]|^2 + lambda_shape |theta[66:76]|^2
// (_fit_terms :266-287) with the gradient computed analytically -- through
// the LBS, the kinematic chain (bodymodel.py:208-240) and Rodrigues
// (bodymodel.py:172-205) -- instead of the reference's reverse-mode tape.
// The best iterate per mesh (mean Euclidean vertex gap, float64,
// _vertex_gap :290-293) is tracked as in _track_best (:311-318).
//
// One CTA (256 threads) per mesh runs every step:
//   warp 0     Rodrigues per joint, the chain composed one tree level at a
//              time, A_j = [R_w | t_w - R_w g]
//   all        per-vertex pass: skinned vertex, gap, dL/dp = 2 (p - t), the
//              shape gradient, (dL/dp, s_v) to a per-mesh scratch
//   warp/joint dL/dA_j = sum_v w_vj dL/dp_v [s_v; 1]^T over the joint's
//              vertex list (CSR by joint, built at template upload)
//   warp 0     chain backward one level at a time (children gathered by
//              their parent), Rodrigues backward (s, c and their
//              derivatives in float64)
//   76 thr.    Adam update with the reference's float32 operation order
#include "fsb_common.cuh"
#include "fsb_weights.h"

namespace {
constexpr int kFitThreads = 256;
constexpr int kFitWarps = kFitThreads / 32;
constexpr int kMaxLevel = 8;

struct FitShared {
  float theta[FSB_PARAM_DIM], m[FSB_PARAM_DIM], v[FSB_PARAM_DIM], best[FSB_PARAM_DIM], grad[FSB_PARAM_DIM];
  float rl[FSB_NJ][9], rw[FSB_NJ][9], tw[FSB_NJ][3], A[FSB_NJ][12];
  float dA[FSB_NJ][12], drw[FSB_NJ][9], dtw[FSB_NJ][3];
  float dbeta[kFitWarps][10];
  double err[kFitWarps];
  double best_err;
};

// d(s)/dt, d(c)/dt at t = theta^2 for s = sin(th)/th, c = (1 - cos th)/th^2
// (the reference's Taylor branch below 1e-12)
__device__ __forceinline__ void sc_derivs(float t2, double& ds, double& dc) {
  if (t2 < 1e-12f) {
    ds = -1.0 / 6.0;
    dc = -1.0 / 24.0;
    return;
  }
  const double t = t2, th = sqrt(t);
  double sn, cs;
  sincos(th, &sn, &cs);
  ds = (th * cs - sn) / (2.0 * th * t);
  dc = (th * sn - 2.0 * (1.0 - cs)) / (2.0 * t * t);
}

// dL/domega of R = rodrigues(omega) given G = dL/dR (row-major 3x3), with
// the reference's entry formulas r_ab(wx, wy, wz, s, c)
__device__ __forceinline__ void rodrigues_backward(const float* w, const float* G, float* out) {
  const float wx = w[0], wy = w[1], wz = w[2];
  const float t2 = wx * wx + wy * wy + wz * wz;
  float s, c;
  if (t2 < 1e-12f) {
    s = 1.0f - t2 * (1.0f / 6.0f);
    c = 0.5f - t2 * (1.0f / 24.0f);
  } else {
    const float th = sqrtf(t2);
    s = sinf(th) / th;
    c = (1.0f - cosf(th)) / t2;
  }
  double ds, dc;
  sc_derivs(t2, ds, dc);
  const float G00 = G[0], G01 = G[1], G02 = G[2], G10 = G[3], G11 = G[4], G12 = G[5], G20 = G[6], G21 = G[7],
              G22 = G[8];
  const float Gs = -wz * G01 + wy * G02 + wz * G10 - wx * G12 - wy * G20 + wx * G21;
  const float Gc = -(wy * wy + wz * wz) * G00 - (wx * wx + wz * wz) * G11 - (wx * wx + wy * wy) * G22 +
                   wx * wy * (G01 + G10) + wx * wz * (G02 + G20) + wy * wz * (G12 + G21);
  const float k = (float)(2.0 * (Gs * ds + Gc * dc));
  out[0] = c * (-2.0f * wx * G11 - 2.0f * wx * G22 + wy * (G01 + G10) + wz * (G02 + G20)) + s * (G21 - G12) + wx * k;
  out[1] = c * (-2.0f * wy * G00 - 2.0f * wy * G22 + wx * (G01 + G10) + wz * (G12 + G21)) + s * (G02 - G20) + wy * k;
  out[2] = c * (-2.0f * wz * G00 - 2.0f * wz * G11 + wx * (G02 + G20) + wy * (G12 + G21)) + s * (G10 - G01) + wz * k;
}

__constant__ int8_t kFitDepth[FSB_NJ] = {0, 1, 2, 3, 4, 5, 1, 2, 3, 4, 1, 2, 3, 4, 4, 5, 6, 7, 4, 5, 6, 7};
}  // namespace

__global__ void __launch_bounds__(kFitThreads) k_fit(TemplateDev t, const float* __restrict__ target, int B,
                                                     const float* __restrict__ init, int steps, double lr,
                                                     float lambda_pose, float lambda_shape, float* __restrict__ scratch,
                                                     float* __restrict__ best_out, double* __restrict__ err_out,
                                                     double* __restrict__ curve_out, float* __restrict__ grad0,
                                                     int* nonfinite) {
  __shared__ FitShared sh;
  const int b = blockIdx.x;
  const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
  // this lane's joint: parent, tree depth and children (bit c set when
  // parents[c] == joint), read from the constant bank once -- per-level
  // reloads with the lanes' distinct addresses serialise (as in fk_warp)
  const int jl = lane < FSB_NJ ? lane : 0;
  const int par_l = lane < FSB_NJ ? (int)kParents[jl] : -1;
  const int dep_l = lane < FSB_NJ ? (int)kFitDepth[jl] : -1;
  uint32_t kids_l = 0;
  for (int c = 0; c < FSB_NJ; ++c)  // (c is warp-uniform: broadcast reads)
    if (lane < FSB_NJ && kParents[c] == lane) kids_l |= 1u << c;
  const int nv = t.nv;
  const float* tgt = target + (int64_t)b * nv * 3;
  float* gs = scratch + (int64_t)b * nv * 6;  // (dL/dp, s) per vertex
  if (tid < FSB_PARAM_DIM) {
    sh.theta[tid] = init ? init[(int64_t)b * FSB_PARAM_DIM + tid] : 0.0f;
    sh.m[tid] = 0.0f;
    sh.v[tid] = 0.0f;
  }
  __syncthreads();
  const float b1 = 0.9f, b2 = 0.999f, eps = 1e-8f;
  for (int step = 0; step <= steps; ++step) {
    // ---- FK forward (warp 0): local rotations, world transforms, A -------
    if (warp == 0) {
      const int j = lane;
      float g[3], tl[3];
      if (j < FSB_NJ) {
        rodrigues3<false>(sh.theta[3 * j], sh.theta[3 * j + 1], sh.theta[3 * j + 2], sh.rl[j]);
        const int p = par_l;
        for (int a = 0; a < 3; ++a) {
          g[a] = t.joints_rest[3 * j + a];
          tl[a] = p < 0 ? g[a] : g[a] - t.joints_rest[3 * p + a];
        }
        if (p < 0) {
          for (int e = 0; e < 9; ++e) sh.rw[0][e] = sh.rl[0][e];
          for (int a = 0; a < 3; ++a) sh.tw[0][a] = tl[a];
        }
      }
      __syncwarp();
      for (int lvl = 1; lvl < kMaxLevel; ++lvl) {
        if (dep_l == lvl) {
          const int p = par_l;
          float rp[9], tp[3];
          for (int e = 0; e < 9; ++e) rp[e] = sh.rw[p][e];
          for (int a = 0; a < 3; ++a) tp[a] = sh.tw[p][a];
          for (int a = 0; a < 3; ++a) {
            for (int q = 0; q < 3; ++q)
              sh.rw[j][3 * a + q] = rp[3 * a] * sh.rl[j][q] + rp[3 * a + 1] * sh.rl[j][3 + q] + rp[3 * a + 2] * sh.rl[j][6 + q];
            sh.tw[j][a] = (rp[3 * a] * tl[0] + rp[3 * a + 1] * tl[1] + rp[3 * a + 2] * tl[2]) + tp[a];
          }
        }
        __syncwarp();
      }
      if (j < FSB_NJ) {
        for (int a = 0; a < 3; ++a) {
          for (int q = 0; q < 3; ++q) sh.A[j][4 * a + q] = sh.rw[j][3 * a + q];
          sh.A[j][4 * a + 3] = sh.tw[j][a] - (sh.rw[j][3 * a] * g[0] + sh.rw[j][3 * a + 1] * g[1] + sh.rw[j][3 * a + 2] * g[2]);
        }
      }
    }
    __syncthreads();
    // ---- per-vertex pass -------------------------------------------------
    float dbeta[10];
    for (int k = 0; k < 10; ++k) dbeta[k] = 0.0f;
    double err = 0.0;
    for (int v = tid; v < nv; v += kFitThreads) {
      float T[12];
      for (int e = 0; e < 12; ++e) T[e] = 0.0f;
      for (int z = 0; z < t.nnz; ++z) {
        const float w = t.skin_w[(int64_t)v * t.nnz + z];
        if (w == 0.0f) continue;
        const float* Aj = sh.A[t.skin_j[(int64_t)v * t.nnz + z]];
        for (int e = 0; e < 12; ++e) T[e] = fmaf(w, Aj[e], T[e]);
      }
      const float* bs = t.shape_basis + (int64_t)v * 30;
      float s[3];
      for (int a = 0; a < 3; ++a) {
        float o = 0.0f;
        for (int k = 0; k < 10; ++k) o = fmaf(bs[10 * a + k], sh.theta[66 + k], o);
        s[a] = o + t.v_rest[(int64_t)v * 3 + a];
      }
      float d[3];
      double e2 = 0.0;
      for (int a = 0; a < 3; ++a) {
        const float p = fmaf(T[4 * a + 2], s[2], fmaf(T[4 * a + 1], s[1], T[4 * a] * s[0])) + T[4 * a + 3];
        const float tv = tgt[(int64_t)v * 3 + a];
        d[a] = p - tv;
        const double dd = (double)p - (double)tv;
        e2 += dd * dd;
      }
      err += sqrt(e2);
      float* o = gs + (int64_t)v * 6;
      for (int a = 0; a < 3; ++a) {
        o[a] = 2.0f * d[a];
        o[3 + a] = s[a];
      }
      // shape gradient: B_v^T (T[:, :3]^T dL/dp)
      float u[3];
      for (int q = 0; q < 3; ++q) u[q] = 2.0f * (T[q] * d[0] + T[4 + q] * d[1] + T[8 + q] * d[2]);
      for (int k = 0; k < 10; ++k) dbeta[k] += u[0] * bs[k] + u[1] * bs[10 + k] + u[2] * bs[20 + k];
    }
    for (int k = 0; k < 10; ++k) dbeta[k] = warp_sum(dbeta[k]);
    for (int off = 16; off > 0; off >>= 1) err += __shfl_xor_sync(0xffffffffu, err, off);
    if (lane == 0) {
      for (int k = 0; k < 10; ++k) sh.dbeta[warp][k] = dbeta[k];
      sh.err[warp] = err;
    }
    __syncthreads();
    // ---- best iterate (before the update, as in the reference loop) -----
    if (tid == 0) {
      double e = 0.0;
      for (int w = 0; w < kFitWarps; ++w) e += sh.err[w];
      e /= (double)nv;
      if (!isfinite(e) && nonfinite) atomicOr(nonfinite, 1);
      if (step == 0 || e < sh.best_err) {
        sh.best_err = e;
        for (int i = 0; i < FSB_PARAM_DIM; ++i) sh.best[i] = sh.theta[i];
      }
      curve_out[(int64_t)b * (steps + 1) + step] = sh.best_err;
    }
    if (step == steps) break;
    // ---- dL/dA_j over each joint's vertex list ---------------------------
    for (int j = warp; j < FSB_NJ; j += kFitWarps) {
      float acc[12];
      for (int e = 0; e < 12; ++e) acc[e] = 0.0f;
      for (int i = t.joint_off[j] + lane; i < t.joint_off[j + 1]; i += 32) {
        const int v = t.joint_v[i];
        const float w = t.joint_w[i];
        const float* o = gs + (int64_t)v * 6;
        const float g0 = w * o[0], g1 = w * o[1], g2 = w * o[2];
        const float s0 = o[3], s1 = o[4], s2 = o[5];
        acc[0] += g0 * s0; acc[1] += g0 * s1; acc[2] += g0 * s2; acc[3] += g0;
        acc[4] += g1 * s0; acc[5] += g1 * s1; acc[6] += g1 * s2; acc[7] += g1;
        acc[8] += g2 * s0; acc[9] += g2 * s1; acc[10] += g2 * s2; acc[11] += g2;
      }
      for (int e = 0; e < 12; ++e) {
        const float r = warp_sum(acc[e]);
        if (lane == 0) sh.dA[j][e] = r;
      }
    }
    __syncthreads();
    // ---- chain backward + Rodrigues backward (warp 0) --------------------
    if (warp == 0) {
      const int j = lane;
      float g[3];
      if (j < FSB_NJ) {
        for (int a = 0; a < 3; ++a) g[a] = t.joints_rest[3 * j + a];
        // A_j = [R_w | t_w - R_w g]: own contributions
        for (int a = 0; a < 3; ++a) {
          const float dat = sh.dA[j][4 * a + 3];
          sh.dtw[j][a] = dat;
          for (int q = 0; q < 3; ++q) sh.drw[j][3 * a + q] = sh.dA[j][4 * a + q] - dat * g[q];
        }
      }
      __syncwarp();
      // children into parents, deepest level first
      for (int lvl = kMaxLevel - 2; lvl >= 0; --lvl) {
        if (dep_l == lvl) {
          for (int c = j + 1; c < FSB_NJ; ++c) {
            if (!((kids_l >> c) & 1u)) continue;
            float tl[3];
            for (int a = 0; a < 3; ++a) tl[a] = t.joints_rest[3 * c + a] - g[a];
            for (int a = 0; a < 3; ++a) {
              for (int q = 0; q < 3; ++q)  // dR_w[j] += dR_w[c] R_l[c]^T + dt_w[c] tl^T
                sh.drw[j][3 * a + q] += sh.drw[c][3 * a] * sh.rl[c][3 * q] + sh.drw[c][3 * a + 1] * sh.rl[c][3 * q + 1] +
                                        sh.drw[c][3 * a + 2] * sh.rl[c][3 * q + 2] + sh.dtw[c][a] * tl[q];
              sh.dtw[j][a] += sh.dtw[c][a];
            }
          }
        }
        __syncwarp();
      }
      if (j < FSB_NJ) {
        // dR_l[j] = R_w[p]^T dR_w[j] (root: dR_w[0])
        const int p = par_l;
        float G[9];
        for (int a = 0; a < 3; ++a)
          for (int q = 0; q < 3; ++q)
            G[3 * a + q] = p < 0 ? sh.drw[j][3 * a + q]
                                 : sh.rw[p][a] * sh.drw[j][q] + sh.rw[p][3 + a] * sh.drw[j][3 + q] +
                                       sh.rw[p][6 + a] * sh.drw[j][6 + q];
        float go[3];
        rodrigues_backward(&sh.theta[3 * j], G, go);
        for (int a = 0; a < 3; ++a) {
          const int i = 3 * j + a;
          sh.grad[i] = go[a] + (i >= 3 ? 2.0f * lambda_pose * sh.theta[i] : 0.0f);
        }
      }
      if (lane < 10) {
        float s = 0.0f;
        for (int w = 0; w < kFitWarps; ++w) s += sh.dbeta[w][lane];
        sh.grad[66 + lane] = s + 2.0f * lambda_shape * sh.theta[66 + lane];
      }
    }
    __syncthreads();
    if (grad0 != nullptr && step == 0 && tid < FSB_PARAM_DIM) grad0[(int64_t)b * FSB_PARAM_DIM + tid] = sh.grad[tid];
    // ---- Adam (projection.py:249-263), float32 in the reference's order ---
    if (tid < FSB_PARAM_DIM) {
      const double tt = (double)(step + 1);
      // the reference's betas are float32 values widened to Python floats
      const float c1 = (float)(1.0 - pow((double)0.9f, tt)), c2 = (float)(1.0 - pow((double)0.999f, tt));
      const float step_lr = (float)(lr * 0.5 * (1.0 + cos(3.141592653589793 * (double)step / (double)steps)));
      const float gg = sh.grad[tid];
      float m = __fmul_rn(sh.m[tid], b1);
      m = __fadd_rn(m, __fmul_rn(__fsub_rn(1.0f, b1), gg));
      float v = __fmul_rn(sh.v[tid], b2);
      v = __fadd_rn(v, __fmul_rn(__fsub_rn(1.0f, b2), __fmul_rn(gg, gg)));
      sh.m[tid] = m;
      sh.v[tid] = v;
      const float upd = __fdiv_rn(__fmul_rn(step_lr, __fdiv_rn(m, c1)), __fadd_rn(__fsqrt_rn(__fdiv_rn(v, c2)), eps));
      sh.theta[tid] = __fsub_rn(sh.theta[tid], upd);
    }
    __syncthreads();
  }
  if (tid < FSB_PARAM_DIM) best_out[(int64_t)b * FSB_PARAM_DIM + tid] = sh.best[tid];
  if (tid == 0) err_out[b] = sh.best_err;
}

cudaError_t launch_fit(const TemplateDev& t, const float* target, int B, const float* init, int steps, double lr,
                       float lambda_pose, float lambda_shape, float* scratch, float* best, double* err, double* curve,
                       float* grad0, int* nonfinite, cudaStream_t st) {
  if (B == 0) return cudaSuccess;
  k_fit<<<B, kFitThreads, 0, st>>>(t, target, B, init, steps, lr, lambda_pose, lambda_shape, scratch, best, err, curve,
                                   grad0, nonfinite);
  return cudaGetLastError();
}
