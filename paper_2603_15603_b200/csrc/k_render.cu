// Synthetic-frame renderer (priors.render_scene, priors.py:237-252) on the
// GPU: gradient background plus one Gaussian blob per keypoint, float32 in
// [0, 1], (B, H, W, 3).  It is the input generator of the benchmark stream
// (94 ms/frame on the CPU).  Every op is rounded as in
// the numpy original (explicit _rn intrinsics, no FMA contraction); only the
// float32 exp may differ from numpy's by an ulp.
#include "fsb_common.cuh"

struct SceneRender {
  float kp[2 * FSB_NJ];
  float half_color[FSB_NJ * 3];  // 0.5 * colors, float32
  float inv;                     // float32(-0.5 / sigma^2)
  float pad;
  double gdir[2];
};

__global__ void __launch_bounds__(256) k_render(const SceneRender* __restrict__ scenes, int H, int W,
                                                float* __restrict__ out) {
  __shared__ SceneRender s;
  const int f = blockIdx.y;
  if (threadIdx.x < sizeof(SceneRender) / 4)
    reinterpret_cast<float*>(&s)[threadIdx.x] = reinterpret_cast<const float*>(scenes + f)[threadIdx.x];
  __syncthreads();
  const int64_t npx = (int64_t)H * W;
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < npx; p += (int64_t)gridDim.x * blockDim.x) {
    const int y = (int)(p / W), x = (int)(p % W);
    const float xf = (float)x, yf = (float)y;
    const double ramp_d = __dadd_rn(__ddiv_rn(__dmul_rn(s.gdir[0], (double)xf), (double)W),
                                    __ddiv_rn(__dmul_rn(s.gdir[1], (double)yf), (double)H));
    const float ramp = __double2float_rn(ramp_d);
    const float base = __fadd_rn(0.10f, __fmul_rn(0.05f, ramp));
    float acc[3] = {base, base, base};
    for (int j = 0; j < FSB_NJ; ++j) {
      const float dx = __fsub_rn(xf, s.kp[2 * j]), dy = __fsub_rn(yf, s.kp[2 * j + 1]);
      const float d2 = __fadd_rn(__fmul_rn(dx, dx), __fmul_rn(dy, dy));
      const float e = expf(__fmul_rn(d2, s.inv));
#pragma unroll
      for (int c = 0; c < 3; ++c) acc[c] = __fadd_rn(acc[c], __fmul_rn(e, s.half_color[3 * j + c]));
    }
    float* o = out + ((int64_t)f * npx + p) * 3;
#pragma unroll
    for (int c = 0; c < 3; ++c) o[c] = fminf(fmaxf(acc[c], 0.0f), 1.0f);
  }
}

cudaError_t launch_render(const void* scenes, int B, int H, int W, float* out, cudaStream_t st) {
  if (B == 0) return cudaSuccess;
  static_assert(sizeof(SceneRender) % 8 == 0 && sizeof(SceneRender) / 4 <= 256, "scene record layout");
  dim3 grid((unsigned)(((int64_t)H * W + 255) / 256 < 1024 ? ((int64_t)H * W + 255) / 256 : 1024), B);
  k_render<<<grid, 256, 0, st>>>(static_cast<const SceneRender*>(scenes), H, W, out);
  return cudaGetLastError();
}
