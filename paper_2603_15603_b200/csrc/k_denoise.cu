// projection.denoise (reference projection.py:684-697, _denoise_forward
// :684-686): out = x + (relu(x W1 + b1) W2 + b2) on (B, 63) body poses, the
// kinematic-prior residual MLP.
//
// One warp per pose.  Both matrix products follow numkit.matmul
// (numkit.py:78-90): every dot product is a left-to-right sum from +0 with a
// separately rounded product and add, so the result is bit-identical to the
// reference; lane j owns hidden units j, j + 32, ..., lanes own outputs
// m = lane and m = lane + 32.  Weights are read from global memory (L2
// resident, 16 KB at the default width).
#include "fsb_common.cuh"

namespace {
constexpr int kDnWarps = 4;
}  // namespace

// one warp per pose (denoise_warp, fsb_common.cuh)
__global__ void __launch_bounds__(32 * kDnWarps) k_denoise(const float* __restrict__ x, int B, DenoiseW d,
                                                          float* __restrict__ out, int* nonfinite) {
  __shared__ float xs[kDnWarps][64];
  __shared__ float hs[kDnWarps][FSB_DN_MAX_HIDDEN];
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int b = blockIdx.x * kDnWarps + warp;
  if (b >= B) return;  // warp-uniform
  const float* xb = x + (int64_t)b * FSB_DN_IN;
  for (int k = lane; k < FSB_DN_IN; k += 32) xs[warp][k] = xb[k];
  __syncwarp();
  denoise_warp(xs[warp], hs[warp], d, lane, out + (int64_t)b * FSB_DN_IN, nonfinite);
}

cudaError_t launch_denoise(const float* x, int B, const float* w1, const float* b1, const float* w2, const float* b2,
                           int H, float* out, int* nonfinite, cudaStream_t st) {
  if (B == 0) return cudaSuccess;
  if (H <= 0 || H > FSB_DN_MAX_HIDDEN) return cudaErrorInvalidValue;
  const DenoiseW d{w1, b1, w2, b2, H};
  k_denoise<<<(B + kDnWarps - 1) / kDnWarps, 32 * kDnWarps, 0, st>>>(x, B, d, out, nonfinite);
  return cudaGetLastError();
}
