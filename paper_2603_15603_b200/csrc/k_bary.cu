// projection.bary_map_from_arrays / precompute_bary (reference
// projection.py:38-184): attach every target point to
// the closest point of the source surface, float64 over every (target,
// face) pair, ties to the lowest face index, zero-area faces projected onto
// their longest edge.
//
// One CTA per target point; its threads stride over the faces keeping the
// (distance, face) minimum, then a block argmin.  Every float64 operation
// is the reference's numpy operation in the same order with explicit
// round-to-nearest intrinsics (no FMA contraction), so the winning face and
// the weights are bit-identical: 3-term sums are ((x0 + x1) + x2),
// np.select takes the first true region, argmin keeps the first minimum.
#include "fsb_common.cuh"

namespace {
constexpr int kBaryThreads = 256;

struct V3 {
  double x, y, z;
};
__device__ __forceinline__ V3 ld3(const double* p) { return {p[0], p[1], p[2]}; }
__device__ __forceinline__ V3 sub(V3 a, V3 b) { return {__dsub_rn(a.x, b.x), __dsub_rn(a.y, b.y), __dsub_rn(a.z, b.z)}; }
__device__ __forceinline__ double dot(V3 a, V3 b) {
  return __dadd_rn(__dadd_rn(__dmul_rn(a.x, b.x), __dmul_rn(a.y, b.y)), __dmul_rn(a.z, b.z));
}

// _tri_regions (projection.py:38-83) for one (triangle, point)
__device__ void tri_regions(V3 a, V3 b, V3 c, V3 p, double w[3]) {
  const V3 ab = sub(b, a), ac = sub(c, a), ap = sub(p, a);
  const double d1 = dot(ab, ap), d2 = dot(ac, ap);
  const V3 bp = sub(p, b);
  const double d3 = dot(ab, bp), d4 = dot(ac, bp);
  const V3 cp = sub(p, c);
  const double d5 = dot(ab, cp), d6 = dot(ac, cp);
  const double vc = __dsub_rn(__dmul_rn(d1, d4), __dmul_rn(d3, d2));
  const double vb = __dsub_rn(__dmul_rn(d5, d2), __dmul_rn(d1, d6));
  const double va = __dsub_rn(__dmul_rn(d3, d6), __dmul_rn(d4, d5));
  if (d1 <= 0.0 && d2 <= 0.0) {  // vertex A
    w[0] = 1.0; w[1] = 0.0; w[2] = 0.0;
  } else if (d3 >= 0.0 && d4 <= d3) {  // vertex B
    w[0] = 0.0; w[1] = 1.0; w[2] = 0.0;
  } else if (vc <= 0.0 && d1 >= 0.0 && d3 <= 0.0) {  // edge AB
    const double t = __ddiv_rn(d1, __dsub_rn(d1, d3));
    w[0] = __dsub_rn(1.0, t); w[1] = t; w[2] = 0.0;
  } else if (d6 >= 0.0 && d5 <= d6) {  // vertex C
    w[0] = 0.0; w[1] = 0.0; w[2] = 1.0;
  } else if (vb <= 0.0 && d2 >= 0.0 && d6 <= 0.0) {  // edge AC
    const double t = __ddiv_rn(d2, __dsub_rn(d2, d6));
    w[0] = __dsub_rn(1.0, t); w[1] = 0.0; w[2] = t;
  } else if (va <= 0.0 && d4 >= d3 && d5 >= d6) {  // edge BC
    const double t = __ddiv_rn(__dsub_rn(d4, d3), __dadd_rn(__dsub_rn(d4, d3), __dsub_rn(d5, d6)));
    w[0] = 0.0; w[1] = __dsub_rn(1.0, t); w[2] = t;
  } else {  // interior
    const double denom = __dadd_rn(__dadd_rn(va, vb), vc);
    const double v = __ddiv_rn(vb, denom), ww = __ddiv_rn(vc, denom);
    w[0] = __dsub_rn(__dsub_rn(1.0, v), ww); w[1] = v; w[2] = ww;
  }
}

// bary weights and squared distance of point p to face f (degenerate faces:
// _segment_bary on the longest edge, projection.py:86-93, :128-141)
__device__ double face_bary(const double* verts, const int64_t* faces, const uint8_t* degen, int f, V3 p, double w[3]) {
  const int64_t ia = faces[3 * f], ib = faces[3 * f + 1], ic = faces[3 * f + 2];
  const V3 a = ld3(verts + 3 * ia), b = ld3(verts + 3 * ib), c = ld3(verts + 3 * ic);
  if (degen[f]) {
    const double e0 = dot(sub(b, a), sub(b, a)), e1 = dot(sub(c, b), sub(c, b)), e2 = dot(sub(a, c), sub(a, c));
    int longest = 0;  // np.argmax: first maximum
    double best = e0;
    if (e1 > best) { best = e1; longest = 1; }
    if (e2 > best) { longest = 2; }
    const int su = longest, sv = (longest + 1) % 3;
    const V3 cor[3] = {a, b, c};
    const V3 u = cor[su], d = sub(cor[sv], u);
    const double den = dot(d, d);
    double t = den > 0.0 ? __ddiv_rn(dot(sub(p, u), d), den) : 0.0;
    t = fmin(fmax(t, 0.0), 1.0);
    w[0] = w[1] = w[2] = 0.0;
    w[su] = __dsub_rn(1.0, t);
    w[sv] = t;
  } else {
    tri_regions(a, b, c, p, w);
  }
  // pos = sum_c w_c corner_c (summed over the corner axis in order)
  const V3 pos = {__dadd_rn(__dadd_rn(__dmul_rn(w[0], a.x), __dmul_rn(w[1], b.x)), __dmul_rn(w[2], c.x)),
                  __dadd_rn(__dadd_rn(__dmul_rn(w[0], a.y), __dmul_rn(w[1], b.y)), __dmul_rn(w[2], c.y)),
                  __dadd_rn(__dadd_rn(__dmul_rn(w[0], a.z), __dmul_rn(w[1], b.z)), __dmul_rn(w[2], c.z))};
  const V3 dd = sub(p, pos);
  return dot(dd, dd);
}
}  // namespace

// degenerate-face flags (projection.py:121-125)
__global__ void k_bary_degenerate(const double* __restrict__ verts, const int64_t* __restrict__ faces, int F,
                                  uint8_t* __restrict__ degen) {
  const int f = blockIdx.x * blockDim.x + threadIdx.x;
  if (f >= F) return;
  const V3 a = ld3(verts + 3 * faces[3 * f]), b = ld3(verts + 3 * faces[3 * f + 1]), c = ld3(verts + 3 * faces[3 * f + 2]);
  const V3 ab = sub(b, a), ac = sub(c, a);
  // np.cross: (ab_y ac_z - ab_z ac_y, ab_z ac_x - ab_x ac_z, ab_x ac_y - ab_y ac_x)
  const V3 n = {__dsub_rn(__dmul_rn(ab.y, ac.z), __dmul_rn(ab.z, ac.y)),
                __dsub_rn(__dmul_rn(ab.z, ac.x), __dmul_rn(ab.x, ac.z)),
                __dsub_rn(__dmul_rn(ab.x, ac.y), __dmul_rn(ab.y, ac.x))};
  const double area2 = dot(n, n);
  const double scale2 = __dmul_rn(dot(ab, ab), dot(ac, ac));
  degen[f] = area2 <= __dmul_rn(1e-12, fmax(scale2, 1e-300)) ? 1 : 0;
}

__global__ void __launch_bounds__(kBaryThreads) k_bary(const double* __restrict__ verts, const int64_t* __restrict__ faces,
                                                       int F, const uint8_t* __restrict__ degen,
                                                       const double* __restrict__ tgts, int64_t* __restrict__ face_out,
                                                       float* __restrict__ w_out) {
  __shared__ double sd[kBaryThreads];
  __shared__ int sf[kBaryThreads];
  const int t = blockIdx.x, tid = threadIdx.x;
  const V3 p = ld3(tgts + 3 * (int64_t)t);
  double best = INFINITY;
  int bf = 0x7fffffff;
  for (int f = tid; f < F; f += kBaryThreads) {
    double w[3];
    const double d2 = face_bary(verts, faces, degen, f, p, w);
    if (d2 < best) {  // f increases per thread: the first minimum is kept
      best = d2;
      bf = f;
    }
  }
  sd[tid] = best;
  sf[tid] = bf;
  __syncthreads();
  for (int s = kBaryThreads / 2; s > 0; s >>= 1) {
    if (tid < s) {
      const double o = sd[tid + s];
      const int of = sf[tid + s];
      if (o < sd[tid] || (o == sd[tid] && of < sf[tid])) {
        sd[tid] = o;
        sf[tid] = of;
      }
    }
    __syncthreads();
  }
  if (tid == 0) {
    const int f = sf[0];
    double w[3];
    face_bary(verts, faces, degen, f, p, w);
    // w = clip(w, 0); w /= w.sum(); float32 (projection.py:170-171, :175)
    for (int k = 0; k < 3; ++k) w[k] = fmax(w[k], 0.0);
    const double s = __dadd_rn(__dadd_rn(w[0], w[1]), w[2]);
    face_out[t] = f;
    for (int k = 0; k < 3; ++k) w_out[3 * (int64_t)t + k] = __double2float_rn(__ddiv_rn(w[k], s));
  }
}

cudaError_t launch_bary(const double* verts, const int64_t* faces, int F, const double* tgts, int nt, uint8_t* degen,
                        int64_t* face_out, float* w_out, cudaStream_t st) {
  if (F <= 0 || nt <= 0) return cudaSuccess;
  k_bary_degenerate<<<(F + 255) / 256, 256, 0, st>>>(verts, faces, F, degen);
  k_bary<<<nt, kBaryThreads, 0, st>>>(verts, faces, F, degen, tgts, face_out, w_out);
  return cudaGetLastError();
}
