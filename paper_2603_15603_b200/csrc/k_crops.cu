// K1: extremity boxes from 2D keypoints + the batched 3-crop bilinear gather.
//
// Reference: priors._body_box_from_keypoints (priors.py:166-176),
// priors.hand_box (priors.py:198-217), pipeline._box_prompt (pipeline.py:318-329),
// priors.crop_grid (priors.py:220-230), numkit.bilinear_sample
// (numkit.py:123-154), pipeline.prepare_crops / batch assembly
// (pipeline.py:295-315, :415-425).
//
// Boxes, prompt, grid coordinates and tap indices are bit-exact with the
// reference; every float op below is an explicit round-to-nearest intrinsic
// so ptxas cannot contract it into an FMA (the numpy originals round each
// multiply and add separately).  See SURVEY Appendix B for the numpy-2
// promotion rules each line follows.
//
// Layout: images (B, H, W, 3) f32 NHWC in HBM; keypoints (B, 22, 2) f32;
// crops out (B, 3, S, S, 3) f32 (crop 0 = body, 1 = left hand, 2 = right).
// Grid: one CTA per (frame, crop, row band); each recomputes its frame's
// box (22 keypoints, a few hundred flops) instead of a separate launch.
#include "fsb_common.cuh"

namespace {

struct FrameBoxes {
  double box[3][4];   // body, left hand, right hand (x0, y0, x1, y1)
  float prompt[8];
};

// body box: float32 sequential sums, float64 divide by the count, then
// weak-scalar float32 corner arithmetic (Appendix B items 2-5).
__device__ void body_box(const float* kp, int W, int H, double out[4]) {
  float c[2], half_f[2];
  for (int ax = 0; ax < 2; ++ax) {
    float s = 0.0f;
    for (int i = 0; i < FSB_NJ; ++i) s = __fadd_rn(s, kp[2 * i + ax]);
    const float cen = __double2float_rn(__ddiv_rn((double)s, (double)FSB_NJ));
    float q = 0.0f;
    for (int i = 0; i < FSB_NJ; ++i) {
      const float d = __fsub_rn(kp[2 * i + ax], cen);
      q = __fadd_rn(q, __fmul_rn(d, d));
    }
    const float var = __double2float_rn(__ddiv_rn((double)q, (double)FSB_NJ));
    const float sd = __fsqrt_rn(var);
    const double half = __dadd_rn(__dmul_rn(2.6, (double)sd), 8.0);
    c[ax] = cen;
    half_f[ax] = __double2float_rn(half);
  }
  const int lim[2] = {W, H};
  float lo[2];
  for (int ax = 0; ax < 2; ++ax) {
    float v = __fsub_rn(c[ax], half_f[ax]);
    v = fminf(fmaxf(v, 0.0f), __double2float_rn((double)lim[ax] - 2.0));
    lo[ax] = v;
  }
  for (int ax = 0; ax < 2; ++ax) {
    float v = __fadd_rn(c[ax], half_f[ax]);
    const float vlo = __double2float_rn(__dadd_rn((double)lo[ax], 1.0));
    v = fminf(fmaxf(v, vlo), __double2float_rn((double)lim[ax] - 1.0));
    out[2 + ax] = (double)v;
  }
  out[0] = (double)lo[0];
  out[1] = (double)lo[1];
}

// wrist-centred square (float64 throughout, Appendix B item 6)
__device__ void hand_box(double wx_f, double wy_f, const double body[4], double alpha, int W, int H,
                         double out[4]) {
  const double bw = __dsub_rn(body[2], body[0]);
  const double bh = __dsub_rn(body[3], body[1]);
  const double s = __ddiv_rn(fmin(bw, bh), alpha);
  const double wm = (double)W - 1.0, hm = (double)H - 1.0;
  const double wx = fmin(fmax(wx_f, 0.0), wm);
  const double wy = fmin(fmax(wy_f, 0.0), hm);
  const double sx = fmin(s, wm), sy = fmin(s, hm);
  const double halfs = __ddiv_rn(s, 2.0);
  const double x0 = fmin(fmax(__dsub_rn(wx, halfs), 0.0), __dsub_rn(wm, sx));
  const double y0 = fmin(fmax(__dsub_rn(wy, halfs), 0.0), __dsub_rn(hm, sy));
  out[0] = x0;
  out[1] = y0;
  out[2] = __dadd_rn(x0, sx);
  out[3] = __dadd_rn(y0, sy);
}

__device__ void frame_boxes(const float* kp, int W, int H, double alpha, FrameBoxes& fb) {
  body_box(kp, W, H, fb.box[0]);
  hand_box(kp[2 * 16], kp[2 * 16 + 1], fb.box[0], alpha, W, H, fb.box[1]);
  hand_box(kp[2 * 20], kp[2 * 20 + 1], fb.box[0], alpha, W, H, fb.box[2]);
  const double w = W, h = H;
  const double* b = fb.box[0];
  fb.prompt[0] = __double2float_rn(__ddiv_rn(b[0], w));
  fb.prompt[1] = __double2float_rn(__ddiv_rn(b[1], h));
  fb.prompt[2] = __double2float_rn(__ddiv_rn(b[2], w));
  fb.prompt[3] = __double2float_rn(__ddiv_rn(b[3], h));
  fb.prompt[4] = __double2float_rn(__ddiv_rn(__dsub_rn(b[2], b[0]), w));
  fb.prompt[5] = __double2float_rn(__ddiv_rn(__dsub_rn(b[3], b[1]), h));
  fb.prompt[6] = __double2float_rn(__ddiv_rn(__dadd_rn(b[0], b[2]), __dmul_rn(2.0, w)));
  fb.prompt[7] = __double2float_rn(__ddiv_rn(__dadd_rn(b[1], b[3]), __dmul_rn(2.0, h)));
}

// np.linspace(a, b, S, dtype=float32)[i]
__device__ __forceinline__ float lin_f32(double a, double b, int S, int i) {
  if (i == S - 1) return __double2float_rn(b);
  const double step = __ddiv_rn(__dsub_rn(b, a), (double)(S - 1));
  return __double2float_rn(__dadd_rn(__dmul_rn((double)i, step), a));
}

constexpr int kRowsPerCTA = 16;

}  // namespace

// grid: (S / kRowsPerCTA, 3, B); block: 256 threads
__global__ void __launch_bounds__(256) k_boxes_crops(
    const float* __restrict__ images, const float* __restrict__ kps, int B, int H, int W, int S,
    double alpha, int64_t img_stride, double* __restrict__ boxes_out, float* __restrict__ prompt_out,
    float* __restrict__ crops_out, int32_t* __restrict__ taps_out, int* nonfinite) {
  __shared__ FrameBoxes fb;
  __shared__ float kp_s[2 * FSB_NJ];
  __shared__ float gx[512], gy[512];  // S <= 512 (checked by the launcher)
  const int f = blockIdx.z, crop = blockIdx.y, band = blockIdx.x;
  const int tid = threadIdx.x;
  if (tid < 2 * FSB_NJ) kp_s[tid] = kps[(int64_t)f * 2 * FSB_NJ + tid];
  __syncthreads();
  if (tid == 0) {
    frame_boxes(kp_s, W, H, alpha, fb);
    if (band == 0 && crop == 0) {
      for (int c = 0; c < 3; ++c)
        for (int e = 0; e < 4; ++e) boxes_out[((int64_t)f * 3 + c) * 4 + e] = fb.box[c][e];
      for (int e = 0; e < 8; ++e) prompt_out[(int64_t)f * 8 + e] = fb.prompt[e];
    }
  }
  __syncthreads();
  const double* bx = fb.box[crop];
  for (int i = tid; i < S; i += blockDim.x) {
    gx[i] = lin_f32(bx[0], bx[2], S, i);
    gy[i] = lin_f32(bx[1], bx[3], S, i);
  }
  __syncthreads();
  if (crops_out == nullptr && taps_out == nullptr) return;
  const float* img = images + (int64_t)f * img_stride;
  const float wmax = (float)(W - 1), hmax = (float)(H - 1);
  const int r0 = band * kRowsPerCTA;
  const int npx = kRowsPerCTA * S;
  for (int p = tid; p < npx; p += blockDim.x) {
    const int r = r0 + p / S, c = p % S;
    if (r >= S) break;
    const float x = fminf(fmaxf(gx[c], 0.0f), wmax);
    const float y = fminf(fmaxf(gy[r], 0.0f), hmax);
    const int x0 = (int)floorf(x), y0 = (int)floorf(y);
    const int x1 = min(x0 + 1, W - 1), y1 = min(y0 + 1, H - 1);
    const float fx = __fsub_rn(x, (float)x0), fy = __fsub_rn(y, (float)y0);
    const float ofx = __fsub_rn(1.0f, fx), ofy = __fsub_rn(1.0f, fy);
    const float* p00 = img + ((int64_t)y0 * W + x0) * 3;
    const float* p01 = img + ((int64_t)y0 * W + x1) * 3;
    const float* p10 = img + ((int64_t)y1 * W + x0) * 3;
    const float* p11 = img + ((int64_t)y1 * W + x1) * 3;
    const int64_t o = ((((int64_t)f * 3 + crop) * S + r) * S + c);
    if (taps_out != nullptr) {
      int32_t* t = taps_out + o * 4;
      t[0] = x0; t[1] = y0; t[2] = x1; t[3] = y1;
    }
    if (crops_out != nullptr) {
#pragma unroll
      for (int ch = 0; ch < 3; ++ch) {
        const float a = __ldg(p00 + ch), b = __ldg(p01 + ch), cc = __ldg(p10 + ch), d = __ldg(p11 + ch);
        const float top = __fadd_rn(__fmul_rn(a, ofx), __fmul_rn(b, fx));
        const float bot = __fadd_rn(__fmul_rn(cc, ofx), __fmul_rn(d, fx));
        const float v = __fadd_rn(__fmul_rn(top, ofy), __fmul_rn(bot, fy));
        flag_nonfinite(nonfinite, v);
        crops_out[o * 3 + ch] = v;
      }
    }
  }
}

// Stand-alone numkit.bilinear_sample (numkit.py:136-154): image (H, W, C),
// grid (n, 2) of (x, y) -> out (n, C).  One thread per sample point.
__global__ void k_bilinear(const float* __restrict__ img, int H, int W, int C, const float* __restrict__ grid,
                           int64_t n, float* __restrict__ out, int* nonfinite) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const float x = fminf(fmaxf(grid[2 * i], 0.0f), (float)(W - 1));
  const float y = fminf(fmaxf(grid[2 * i + 1], 0.0f), (float)(H - 1));
  const int x0 = (int)floorf(x), y0 = (int)floorf(y);
  const int x1 = min(x0 + 1, W - 1), y1 = min(y0 + 1, H - 1);
  const float fx = __fsub_rn(x, (float)x0), fy = __fsub_rn(y, (float)y0);
  const float ofx = __fsub_rn(1.0f, fx), ofy = __fsub_rn(1.0f, fy);
  for (int ch = 0; ch < C; ++ch) {
    const float a = img[((int64_t)y0 * W + x0) * C + ch], b = img[((int64_t)y0 * W + x1) * C + ch];
    const float c = img[((int64_t)y1 * W + x0) * C + ch], d = img[((int64_t)y1 * W + x1) * C + ch];
    const float top = __fadd_rn(__fmul_rn(a, ofx), __fmul_rn(b, fx));
    const float bot = __fadd_rn(__fmul_rn(c, ofx), __fmul_rn(d, fx));
    const float v = __fadd_rn(__fmul_rn(top, ofy), __fmul_rn(bot, fy));
    flag_nonfinite(nonfinite, v);
    out[i * C + ch] = v;
  }
}

cudaError_t launch_boxes_crops(const float* images, const float* kps, int B, int H, int W, int S, double alpha,
                               double* boxes, float* prompt, float* crops, int32_t* taps, int* nonfinite,
                               cudaStream_t st) {
  if (B == 0) return cudaSuccess;
  if (S < 2 || S > 512) return cudaErrorInvalidValue;
  dim3 grid((S + kRowsPerCTA - 1) / kRowsPerCTA, 3, B);
  k_boxes_crops<<<grid, 256, 0, st>>>(images, kps, B, H, W, S, alpha, (int64_t)H * W * 3, boxes, prompt, crops,
                                      taps, nonfinite);
  return cudaGetLastError();
}

cudaError_t launch_bilinear(const float* img, int H, int W, int C, const float* grid, int64_t n, float* out,
                            int* nonfinite, cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  k_bilinear<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(img, H, W, C, grid, n, out, nonfinite);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// stand-alone box / grid entry points (same arithmetic as k_boxes_crops)
// ---------------------------------------------------------------------------
__global__ void k_body_boxes(const float* __restrict__ kps, int n, int W, int H, double* __restrict__ out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  float kp[2 * FSB_NJ];
  for (int e = 0; e < 2 * FSB_NJ; ++e) kp[e] = kps[(int64_t)i * 2 * FSB_NJ + e];
  double b[4];
  body_box(kp, W, H, b);
  for (int e = 0; e < 4; ++e) out[4 * (int64_t)i + e] = b[e];
}

// priors.hand_box; W <= 0 means image_size=None (no clamping, priors.py:207-208)
__global__ void k_hand_boxes(const double* __restrict__ wrists, const double* __restrict__ body, int n, double alpha,
                             int W, int H, double* __restrict__ out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double b[4] = {body[4 * i], body[4 * i + 1], body[4 * i + 2], body[4 * i + 3]};
  double o[4];
  if (W > 0) {
    hand_box(wrists[2 * i], wrists[2 * i + 1], b, alpha, W, H, o);
  } else {
    const double s = __ddiv_rn(fmin(__dsub_rn(b[2], b[0]), __dsub_rn(b[3], b[1])), alpha);
    const double hs = __ddiv_rn(s, 2.0);
    const double wx = wrists[2 * i], wy = wrists[2 * i + 1];
    o[0] = __dsub_rn(wx, hs);
    o[1] = __dsub_rn(wy, hs);
    o[2] = __dadd_rn(wx, hs);
    o[3] = __dadd_rn(wy, hs);
  }
  for (int e = 0; e < 4; ++e) out[4 * (int64_t)i + e] = o[e];
}

// priors.crop_grid: boxes (n, 4) f64 -> (n, S, S, 2) f32
__global__ void k_crop_grid(const double* __restrict__ boxes, int n, int S, float* __restrict__ out) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (int64_t)n * S * S) return;
  const int i = (int)(idx / ((int64_t)S * S)), r = (int)((idx / S) % S), c = (int)(idx % S);
  const double* b = boxes + 4 * (int64_t)i;
  out[2 * idx] = lin_f32(b[0], b[2], S, c);
  out[2 * idx + 1] = lin_f32(b[1], b[3], S, r);
}

cudaError_t launch_body_boxes(const float* kps, int n, int W, int H, double* out, cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  k_body_boxes<<<(n + 127) / 128, 128, 0, st>>>(kps, n, W, H, out);
  return cudaGetLastError();
}

cudaError_t launch_hand_boxes(const double* wrists, const double* body, int n, double alpha, int W, int H, double* out,
                              cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  k_hand_boxes<<<(n + 127) / 128, 128, 0, st>>>(wrists, body, n, alpha, W, H, out);
  return cudaGetLastError();
}

cudaError_t launch_crop_grid(const double* boxes, int n, int S, float* out, cudaStream_t st) {
  const int64_t tot = (int64_t)n * S * S;
  if (tot == 0) return cudaSuccess;
  k_crop_grid<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(boxes, n, S, out);
  return cudaGetLastError();
}
