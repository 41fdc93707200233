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

// detect_stub (priors.py:188-190) clips the keypoints into the frame before
// the body box: np.clip of float32 values against the integral bounds
// [0, W-1] x [0, H-1] is exact in float32.  e = flat index into (22, 2).
__device__ __forceinline__ float clip_kp(float v, int e, int W, int H) {
  return fminf(fmaxf(v, 0.0f), (float)((e & 1) ? H - 1 : W - 1));
}

// kp: the frame's keypoints already clipped by clip_kp
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
// Boxes and prompt of every frame, one thread per frame (the serial float
// sums of the reference), ahead of the gather CTAs that read them.
__global__ void k_frame_boxes(const float* __restrict__ kps, int B, int W, int H, double alpha,
                              double* __restrict__ boxes_out, float* __restrict__ prompt_out) {
  pdl_wait();
  pdl_trigger();  // the gather CTAs may be scheduled right away (they wait for these boxes)
  const int f = blockIdx.x * blockDim.x + threadIdx.x;
  if (f >= B) return;
  float kp[2 * FSB_NJ];
#pragma unroll
  for (int i = 0; i < 2 * FSB_NJ; ++i) kp[i] = clip_kp(kps[(int64_t)f * 2 * FSB_NJ + i], i, W, H);
  FrameBoxes fb;
  frame_boxes(kp, W, H, alpha, fb);
  for (int c = 0; c < 3; ++c)
    for (int e = 0; e < 4; ++e) boxes_out[((int64_t)f * 3 + c) * 4 + e] = fb.box[c][e];
  for (int e = 0; e < 8; ++e) prompt_out[(int64_t)f * 8 + e] = fb.prompt[e];
}

// SELF (a batch of one or two frames, the latency case): thread 0 derives
// the frame's boxes itself (the same frame_boxes as k_frame_boxes; CTA
// (0, 0) of each frame writes them out) instead of waiting for a separate
// k_frame_boxes launch.
template <bool SELF>
__global__ void __launch_bounds__(256) k_boxes_crops(
    const float* __restrict__ images, const float* __restrict__ kps, int B, int H, int W, int S,
    double alpha, int64_t img_stride, double* __restrict__ boxes_out, float* __restrict__ prompt_out,
    float* __restrict__ crops_out, int32_t* __restrict__ taps_out, int* nonfinite) {
  __shared__ double bx[4];
  __shared__ float gx[512], gy[512];  // S <= 512 (checked by the launcher)
  const int f = blockIdx.z, crop = blockIdx.y, band = blockIdx.x;
  const int tid = threadIdx.x;
  pdl_wait();
  if (SELF) {
    if (tid == 0) {
      float kp[2 * FSB_NJ];
      for (int i = 0; i < 2 * FSB_NJ; ++i) kp[i] = clip_kp(kps[(int64_t)f * 2 * FSB_NJ + i], i, W, H);
      FrameBoxes fb;
      frame_boxes(kp, W, H, alpha, fb);
      for (int e = 0; e < 4; ++e) bx[e] = fb.box[crop][e];
      if (band == 0 && crop == 0) {
        for (int c = 0; c < 3; ++c)
          for (int e = 0; e < 4; ++e) boxes_out[((int64_t)f * 3 + c) * 4 + e] = fb.box[c][e];
        for (int e = 0; e < 8; ++e) prompt_out[(int64_t)f * 8 + e] = fb.prompt[e];
      }
    }
  } else {
    // the frame's boxes come from k_frame_boxes (same stream, launched first)
    if (tid < 4) bx[tid] = boxes_out[((int64_t)f * 3 + crop) * 4 + tid];
  }
  __syncthreads();
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

// ---------------------------------------------------------------------------
// Row-span streaming variant (the production K1).  A CTA owns `rows_per_cta`
// consecutive output rows of one crop and walks them in sub-bands of RB = 4
// rows.  For each sub-band the image rows it taps (y0 / y1 of each sample
// row, each image row once when the band's rows are contiguous) are staged
// in shared memory over the crop's x-span only: thread 0 plans the rows and
// issues one cp.async.bulk (TMA 1-D) copy per row into one of two buffers,
// so sub-band k+1 is in flight while sub-band k is blended from shared
// memory.  It serves frames in pinned host memory, read in place over PCIe
// so only the crop footprints cross the bus (measured 49 GB/s, PCIe-bound;
// per-tap reads of host frames reach 45 GB/s).  Frames resident in HBM use
// the per-tap kernel above, which is faster there (10.7 us vs 25 us for 32
// frames: L1 absorbs the tap overlap and the grid is wider).  Arithmetic is
// identical to k_boxes_crops (bit-exact).
// ---------------------------------------------------------------------------
#include "tc_sm100.cuh"

namespace {
constexpr int kStreamThreads = 256;
constexpr int kRB = 4;        // sample rows per sub-band
constexpr int kSlots = 2 * kRB;  // image rows per sub-band buffer

struct BandPlan {
  int nrows;
  int slot0[kRB], slot1[kRB];
  int rowoff[kSlots];  // floats between the staged row's first vector and pixel xa
};
}  // namespace

__global__ void __launch_bounds__(kStreamThreads) k_crops_stream(
    const float* __restrict__ images, const float* __restrict__ kps, int B, int H, int W, int S, double alpha,
    int64_t img_stride, int rowcap4, int rows_per_cta, double* __restrict__ boxes_out,
    float* __restrict__ prompt_out, float* __restrict__ crops_out, int32_t* __restrict__ taps_out, int* nonfinite,
    unsigned long long* bytes_in) {
  extern __shared__ __align__(128) float4 bufs4[];  // 2 buffers x kSlots rows x rowcap4
  __shared__ FrameBoxes fb;
  __shared__ float kp_s[2 * FSB_NJ];
  __shared__ float gx[512], gy[512];
  __shared__ BandPlan plan[2];
  __shared__ __align__(8) uint64_t bar[2];
  const int f = blockIdx.z, crop = blockIdx.y;
  const int tid = threadIdx.x;
  const int r_begin = blockIdx.x * rows_per_cta;
  const int r_end = min(S, r_begin + rows_per_cta);
  pdl_wait();
  if (r_begin >= S) return;
  if (tid < 2 * FSB_NJ) kp_s[tid] = clip_kp(kps[(int64_t)f * 2 * FSB_NJ + tid], tid, W, H);
  if (tid == 0) {
    tc::mbar_init(&bar[0], 1);
    tc::mbar_init(&bar[1], 1);
    tc::mbar_fence_init();
  }
  __syncthreads();
  if (tid == 0) {
    frame_boxes(kp_s, W, H, alpha, fb);
    if (blockIdx.x == 0 && crop == 0) {
      for (int c = 0; c < 3; ++c)
        for (int e = 0; e < 4; ++e) boxes_out[((int64_t)f * 3 + c) * 4 + e] = fb.box[c][e];
      for (int e = 0; e < 8; ++e) prompt_out[(int64_t)f * 8 + e] = fb.prompt[e];
    }
  }
  __syncthreads();
  const double* bx = fb.box[crop];
  for (int i = tid; i < S; i += kStreamThreads) gx[i] = lin_f32(bx[0], bx[2], S, i);
  for (int i = r_begin + tid; i < r_end; i += kStreamThreads) gy[i] = lin_f32(bx[1], bx[3], S, i);
  __syncthreads();
  if (crops_out == nullptr && taps_out == nullptr) return;
  const float wmax = (float)(W - 1), hmax = (float)(H - 1);
  const int nsub = (r_end - r_begin + kRB - 1) / kRB;
  const int rowcap = rowcap4 * 4;
  // x-span of the crop: taps of column 0 to column S-1 (the grid is monotone)
  const int xlo = (int)floorf(fminf(fmaxf(gx[0], 0.0f), wmax));
  const int xhi = min((int)floorf(fminf(fmaxf(gx[S - 1], 0.0f), wmax)) + 1, W - 1);
  const int span = (xhi - xlo + 1) * 3;
  const int64_t img0 = (int64_t)f * img_stride;
  unsigned long long bytes = 0;  // thread 0 only

  // thread 0: choose the image rows of sub-band k and start staging them
  auto plan_band = [&](int k) {
    const int b = k & 1;
    BandPlan& pl = plan[b];
    const int r0 = r_begin + k * kRB, nr = min(kRB, r_end - r0);
    int y0s[kRB], y1s[kRB];
    for (int i = 0; i < nr; ++i) {
      const int y0 = (int)floorf(fminf(fmaxf(gy[r0 + i], 0.0f), hmax));
      y0s[i] = y0;
      y1s[i] = min(y0 + 1, H - 1);
    }
    const int ymin = y0s[0], ymax = y1s[nr - 1];
    bool contiguous = ymax >= ymin && ymax - ymin + 1 <= kSlots;
    for (int i = 0; i < nr; ++i) contiguous = contiguous && y0s[i] >= ymin && y1s[i] <= ymax;
    int ys[kSlots];
    int n = 0;
    if (contiguous) {  // each image row of the band once
      for (int y = ymin; y <= ymax; ++y) ys[n++] = y;
      for (int i = 0; i < nr; ++i) {
        pl.slot0[i] = y0s[i] - ymin;
        pl.slot1[i] = y1s[i] - ymin;
      }
    } else {
      for (int i = 0; i < nr; ++i) {
        ys[n] = y0s[i];
        pl.slot0[i] = n++;
        ys[n] = y1s[i];
        pl.slot1[i] = n++;
      }
    }
    pl.nrows = n;
    uint32_t tx = 0;
    int64_t v0s[kSlots];
    int nvs[kSlots];
    for (int sl = 0; sl < n; ++sl) {
      const int64_t e0 = img0 + ((int64_t)ys[sl] * W + xlo) * 3;  // first float of the span
      const int64_t v0 = e0 >> 2, v1 = (e0 + span + 3) >> 2;
      pl.rowoff[sl] = (int)(e0 - 4 * v0);
      v0s[sl] = v0;
      nvs[sl] = (int)(v1 - v0);
      tx += (uint32_t)(v1 - v0) * 16u;
    }
    bytes += tx;
    tc::mbar_expect_tx(&bar[b], tx);
    for (int sl = 0; sl < n; ++sl)
      tc::bulk_g2s(bufs4 + (b * kSlots + sl) * rowcap4, reinterpret_cast<const float4*>(images) + v0s[sl],
                   (uint32_t)nvs[sl] * 16u, &bar[b]);
  };

  if (tid == 0) {
    plan_band(0);
    if (nsub > 1) plan_band(1);
  }
  __syncthreads();
  for (int k = 0; k < nsub; ++k) {
    const int b = k & 1;
    tc::mbar_wait(&bar[b], (uint32_t)((k >> 1) & 1));
    const BandPlan& pl = plan[b];
    const float* rows = reinterpret_cast<const float*>(bufs4) + (size_t)b * kSlots * rowcap;
    const int r0 = r_begin + k * kRB, nr = min(kRB, r_end - r0);
    for (int p = tid; p < nr * S; p += kStreamThreads) {
      const int i = p / S, c = p - i * S, r = r0 + i;
      const float x = fminf(fmaxf(gx[c], 0.0f), wmax);
      const float y = fminf(fmaxf(gy[r], 0.0f), hmax);
      const int x0 = (int)floorf(x), y0 = (int)floorf(y);
      const int x1 = min(x0 + 1, W - 1), y1 = min(y0 + 1, H - 1);
      const float fx = __fsub_rn(x, (float)x0), fy = __fsub_rn(y, (float)y0);
      const float ofx = __fsub_rn(1.0f, fx), ofy = __fsub_rn(1.0f, fy);
      const int s0 = pl.slot0[i], s1 = pl.slot1[i];
      const float* ra = rows + s0 * rowcap + pl.rowoff[s0] - xlo * 3;
      const float* rb = rows + s1 * rowcap + pl.rowoff[s1] - xlo * 3;
      const int64_t o = ((((int64_t)f * 3 + crop) * S + r) * S + c);
      if (taps_out != nullptr) {
        int32_t* t = taps_out + o * 4;
        t[0] = x0; t[1] = y0; t[2] = x1; t[3] = y1;
      }
      if (crops_out != nullptr) {
#pragma unroll
        for (int ch = 0; ch < 3; ++ch) {
          const float a = ra[x0 * 3 + ch], bb = ra[x1 * 3 + ch], cc = rb[x0 * 3 + ch], d = rb[x1 * 3 + ch];
          const float top = __fadd_rn(__fmul_rn(a, ofx), __fmul_rn(bb, fx));
          const float bot = __fadd_rn(__fmul_rn(cc, ofx), __fmul_rn(d, fx));
          const float v = __fadd_rn(__fmul_rn(top, ofy), __fmul_rn(bot, fy));
          flag_nonfinite(nonfinite, v);
          crops_out[o * 3 + ch] = v;
        }
      }
    }
    __syncthreads();  // buffer b and its plan are free again
    if (tid == 0 && k + 2 < nsub) plan_band(k + 2);
  }
  if (tid == 0 && bytes_in != nullptr) atomicAdd(bytes_in, bytes);
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

static size_t stream_smem(int rowcap4) { return (size_t)2 * kSlots * rowcap4 * sizeof(float4); }
constexpr size_t kStreamSmemCap = 120 * 1024;

cudaError_t init_attrs_crops() {
  return cudaFuncSetAttribute(k_crops_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kStreamSmemCap);
}

// host_frames: `images` is pinned (mapped) host memory; bytes_in (nullable)
// then accumulates the bytes K1 read over PCIe
cudaError_t launch_boxes_crops(const float* images, const float* kps, int B, int H, int W, int S, double alpha,
                               bool host_frames, double* boxes, float* prompt, float* crops, int32_t* taps,
                               int* nonfinite, unsigned long long* bytes_in, cudaStream_t st) {
  if (B == 0) return cudaSuccess;
  if (S < 2 || S > 512) return cudaErrorInvalidValue;
  const int64_t stride = (int64_t)H * W * 3;
  const int rowcap4 = (W * 3 + 7) / 4 + 1;
  const bool aligned = (reinterpret_cast<uintptr_t>(images) & 15u) == 0;
  if (host_frames && aligned && stream_smem(rowcap4) <= kStreamSmemCap) {
    // enough CTAs for ~2 per SM: bands of rows_per_cta (a multiple of kRB)
    const int nsub_total = (S + kRB - 1) / kRB;
    int bands = (296 + 3 * B - 1) / (3 * B);
    bands = max(1, min(bands, nsub_total));
    const int rows_per_cta = ((nsub_total + bands - 1) / bands) * kRB;
    bands = (S + rows_per_cta - 1) / rows_per_cta;
    dim3 grid(bands, 3, B);
    return launch_pdl(k_crops_stream, grid, dim3(kStreamThreads), stream_smem(rowcap4), st, images, kps, B, H, W, S,
                      alpha, stride, rowcap4, rows_per_cta, boxes, prompt, crops, taps, nonfinite, bytes_in);
  } else {  // HBM-resident (or very wide / unaligned host) frames: per-tap reads
    dim3 grid((S + kRowsPerCTA - 1) / kRowsPerCTA, 3, B);
    if (B <= 2)  // latency: one launch, each CTA derives its frame's boxes
      return launch_pdl(k_boxes_crops<true>, grid, dim3(256), 0, st, images, kps, B, H, W, S, alpha, stride, boxes,
                        prompt, crops, taps, nonfinite);
    cudaError_t e = launch_pdl(k_frame_boxes, dim3((B + 63) / 64), dim3(64), 0, st, kps, B, W, H, alpha, boxes, prompt);
    if (e != cudaSuccess) return e;
    return launch_pdl(k_boxes_crops<false>, grid, dim3(256), 0, st, images, kps, B, H, W, S, alpha, stride, boxes,
                      prompt, crops, taps, nonfinite);
  }
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

// ---------------------------------------------------------------------------
// Host-read peak (bench.py's e2e roofline denominator): stream `bytes` from
// pinned, mapped host memory to HBM the way K1 reads host frames -- each CTA
// pulls 16 KB chunks with cp.async.bulk into a two-slot shared-memory ring
// and writes them out with 16-byte stores.  Test hook, not in the header.
// ---------------------------------------------------------------------------
constexpr uint32_t kHrChunk = 16384;

__global__ void __launch_bounds__(256) k_host_read(const uint8_t* __restrict__ src, size_t nchunks,
                                                   uint8_t* __restrict__ dst) {
  extern __shared__ __align__(128) uint8_t hr_smem[];
  __shared__ __align__(8) uint64_t bar[2];
  if (threadIdx.x == 0) {
    tc::mbar_init(&bar[0], 1);
    tc::mbar_init(&bar[1], 1);
    tc::mbar_fence_init();
  }
  __syncthreads();
  auto fetch = [&](size_t c, int s) {
    tc::mbar_expect_tx(&bar[s], kHrChunk);
    tc::bulk_g2s(hr_smem + s * kHrChunk, src + c * kHrChunk, kHrChunk, &bar[s]);
  };
  size_t c = blockIdx.x;
  if (threadIdx.x == 0) {
    if (c < nchunks) fetch(c, 0);
    if (c + gridDim.x < nchunks) fetch(c + gridDim.x, 1);
  }
  for (int it = 0; c < nchunks; c += gridDim.x, ++it) {
    const int s = it & 1;
    tc::mbar_wait(&bar[s], (uint32_t)((it >> 1) & 1));
    const uint4* in = reinterpret_cast<const uint4*>(hr_smem + s * kHrChunk);
    uint4* out = reinterpret_cast<uint4*>(dst + c * kHrChunk);
    for (int i = threadIdx.x; i < (int)(kHrChunk / 16); i += blockDim.x) out[i] = in[i];
    __syncthreads();
    if (threadIdx.x == 0 && c + 2 * gridDim.x < nchunks) {
      tc::fence_async_smem();
      fetch(c + 2 * gridDim.x, s);
    }
  }
}

extern "C" int fsb_debug_host_read(const void* host_src, size_t bytes, void* dst, int ctas, void* stream) {
  if (bytes % kHrChunk) return 1;
  static bool attr = false;
  if (!attr && cudaFuncSetAttribute(k_host_read, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * kHrChunk) !=
                   cudaSuccess)
    return 2;
  attr = true;
  k_host_read<<<ctas, 256, 2 * kHrChunk, (cudaStream_t)stream>>>(static_cast<const uint8_t*>(host_src),
                                                                  bytes / kHrChunk, static_cast<uint8_t*>(dst));
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) fprintf(stderr, "fsb_debug_host_read: %s\n", cudaGetErrorString(e));
  return e == cudaSuccess ? 0 : 3;
}
