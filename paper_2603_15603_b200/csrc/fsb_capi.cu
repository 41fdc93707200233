#include <stdlib.h>
// C ABI (include/fsb_b200.h): context, model upload/repacking, workspace,
// stage entry points and the CUDA-graph replay of the whole frame batch.
#include <cuda_runtime.h>
#include <stdarg.h>
#include <stdio.h>
#include <string.h>

#include <map>
#include <memory>
#include <string>
#include <vector>

#include "../../include/fsb_b200.h"
#include "fsb_common.cuh"
#include "fsb_enc_f32.h"
#include "fsb_vit.h"
#include "fsb_weights.h"

// ---- kernels (other translation units) ------------------------------------
cudaError_t launch_boxes_crops(const float* images, const float* kps, int B, int H, int W, int S, double alpha,
                               bool host_frames, double* boxes, float* prompt, float* crops, int32_t* taps,
                               int* nonfinite, unsigned long long* bytes_in, cudaStream_t st);
cudaError_t init_attrs_crops();
cudaError_t launch_bilinear(const float* img, int H, int W, int C, const float* grid, int64_t n, float* out,
                            int* nonfinite, cudaStream_t st);
cudaError_t launch_encoder_f32(const float* crops, int ncrops, const EncW& w, float* feats, int* nonfinite,
                               cudaStream_t st);
cudaError_t launch_decoders_f32(const DecodeArgs& a, const BodyW& bw, const HandW& hw, cudaStream_t st);
bool proj_fused_ok(const ProjectorDev& p);
// The one-launch cluster projector (k_proj_fused) is opt-in (FSB_PROJ_FUSED=1):
// measured against the split-K tile GEMMs it lowers the saturated per-batch
// cost (3.59 vs 4.46 us at cluster size 8) but raises the batch latency
// (33 vs 23 us) and the C3 time (0.66 vs 0.54 ms) -- DESIGN.md §4.
static bool proj_fused_on() {
  static const bool on = getenv("FSB_PROJ_FUSED") != nullptr;
  return on;
}
cudaError_t launch_proj_fused(const uint8_t* ximg, const ProjectorDev& p, int B, float* theta, const float* grest,
                              float* joints, const DenoiseW* dn, int* nonfinite, cudaStream_t st);
cudaError_t launch_fk(const float* poses, int ld_pose, int B, const float* grest, float* joints, float* rel,
                      cudaStream_t st, uint8_t* lbs_in = nullptr, const DenoiseW* dn = nullptr,
                      int* nonfinite = nullptr);
cudaError_t launch_lbs_tc(const TemplateDev& t, const uint8_t* lbs_in, int B, float* verts, int* nonfinite,
                          cudaStream_t st, CornerOut cu = CornerOut());
cudaError_t launch_lbs(const TemplateDev& t, const float* rel, const float* poses, int ld_pose, int B, float* verts,
                       int* nonfinite, cudaStream_t st);
cudaError_t launch_proj_inputs(const TemplateDev& t, const ProjectorDev& p, const float* rel, const float* poses,
                               int ld_pose, int B, float* sub, bool f32, __nv_bfloat16* xb, float* psum,
                               cudaStream_t st);
cudaError_t launch_proj_inputs_v(const float* V, int nv, const ProjectorDev& p, int B, float* sub, bool f32,
                                 __nv_bfloat16* xb, float* psum, cudaStream_t st, bool compacted = false,
                                 __nv_bfloat16* xb_lo = nullptr);
cudaError_t launch_gemm_f32(const float* A, int lda, const float* W, const float* bias, const float* mask, float* C,
                            int ldc, int M, int N, int K, int relu, int* nonfinite, float* partial,
                            cudaStream_t st);
int gemm_f32_splits(int K);

cudaError_t launch_body_boxes(const float* kps, int n, int W, int H, double* out, cudaStream_t st);
cudaError_t launch_hand_boxes(const double* wrists, const double* body, int n, double alpha, int W, int H, double* out,
                              cudaStream_t st);
cudaError_t launch_crop_grid(const double* boxes, int n, int S, float* out, cudaStream_t st);
cudaError_t launch_bridge(const float* V, int B, int nv, const int32_t* corners, const float* w, int nt, float* out,
                          cudaStream_t st);
cudaError_t launch_render(const void* scenes, int B, int H, int W, float* out, cudaStream_t st);
cudaError_t launch_fit(const TemplateDev& t, const float* target, int B, const float* init, int steps, double lr,
                       float lambda_pose, float lambda_shape, float* scratch, float* best, double* err, double* curve,
                       float* grad0, int* nonfinite, cudaStream_t st);
cudaError_t launch_bary(const double* verts, const int64_t* faces, int F, const double* tgts, int nt, uint8_t* degen,
                        int64_t* face_out, float* w_out, cudaStream_t st);
cudaError_t launch_denoise(const float* x, int B, const float* w1, const float* b1, const float* w2, const float* b2,
                           int H, float* out, int* nonfinite, cudaStream_t st);
cudaError_t init_attrs_transformer();
cudaError_t init_attrs_transformer_tc();
cudaError_t init_attrs_mlp_tc();
cudaError_t init_attrs_gemm_tc();
cudaError_t launch_tile_layer(const uint8_t* Aimg, const uint8_t* Bimg, int KT, int G, int M, int N, float* partial,
                              const float* bias, const float* mask, int relu, float* out, int ldo, uint8_t* out_img,
                              int KT_out, int* nonfinite, cudaStream_t st, const uint8_t* Aimg_lo = nullptr,
                              const uint8_t* Bimg_lo = nullptr, uint8_t* out_img_lo = nullptr);
cudaError_t launch_encoder_tc(const float* crops, int ncrops, const EncW& w, float* feats, int* nonfinite,
                              const KvArgs& kv, cudaStream_t st);
cudaError_t launch_decoders_tc(const DecodeArgs& a, const BodyW& bw, const HandW& hw, cudaStream_t st);
cudaError_t init_attrs_body();

namespace {

// byte offset of element (r, k) in a K-major no-swizzle UMMA tile (see tc_sm100.cuh)
inline size_t tc_kmajor_off(int r, int k, int K) {
  return (size_t)(r >> 3) * (K * 16) + (k >> 3) * 128 + (r & 7) * 16 + (k & 7) * 2;
}

struct DevMem {
  void* p = nullptr;
  size_t n = 0;
  ~DevMem() { release(); }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
  cudaError_t alloc(size_t bytes) {
    release();
    n = bytes;
    return bytes ? cudaMalloc(&p, bytes) : cudaSuccess;
  }
};

// host-side packer: append arrays at 256-byte aligned offsets, then one H2D
struct Packer {
  std::vector<unsigned char> host;
  size_t add(const void* src, size_t bytes) {
    const size_t off = (host.size() + 255) & ~size_t(255);
    host.resize(off + bytes);
    if (src) memcpy(host.data() + off, src, bytes);
    return off;
  }
};

struct GraphKey {
  int B, H, W, precision;
  uint32_t bsel, hsel;
  double alpha;
  const void* ptrs[16];
  cudaStream_t stream;
  bool operator==(const GraphKey& o) const { return memcmp(this, &o, sizeof(GraphKey)) == 0; }
};

}  // namespace

// The uploaded model (decoder weights and their tcgen05 images, templates,
// projector): read-only on the device once uploaded, so contexts created
// with fsb_ctx_create_shared point at one copy (one per GPU) instead of one
// per in-flight stream.  `version` counts uploads; a context whose graphs
// and workspace were built against another version rebuilds them.
struct fsb_model {
  uint64_t version = 1;
  // decoder
  bool has_decoder = false;
  fsb_decoder_config cfg{};
  DevMem dec_mem;
  DevMem tcs_mem;  // TcStream tables of the encoder, body and hand decoders, K / V projection
  const TcStream* kv_tcs[2][2] = {{nullptr, nullptr}, {nullptr, nullptr}};  // [encoder + K/V | K/V only][body | hand]
  EncW enc{};
  BodyW body{};
  HandW hand{};
  // non-default DecoderConfig: the encoder as a layer pipeline, bf16 on the
  // tensor cores (k_vit.cu, when the shape fits it) and fp32 on the CUDA
  // cores (k_enc_f32.cu, any shape)
  bool vit = false;
  bool vit_tc = false;
  VitW vitw;
  DevMem encf32_mem;
  EncF32W encw;
  // templates / projector
  bool has_tmpl[2] = {false, false};
  DevMem tmpl_mem[2];
  TemplateDev tmpl[2]{};
  bool has_proj = false;
  DevMem proj_mem;
  ProjectorDev proj{};
  // optional kinematic-prior denoiser, applied to theta[3:66] by the frame
  // path's SMPL FK (fsb_load_denoiser)
  DevMem dn_mem;
  DenoiseW dn{nullptr, nullptr, nullptr, nullptr, 0};
};

struct fsb_ctx {
  int device = 0;
  std::string err;
  int* d_flag = nullptr;
  unsigned long long* d_bytes_in = nullptr;  // frame bytes K1 read (HBM or, for host frames, PCIe)
  fsb_counters_t counters{};
  int64_t launches = 0;
  std::shared_ptr<fsb_model> mp;
  fsb_model* m = nullptr;
  uint64_t seen_version = 0;  // model version the workspace / graphs were built for
  // streams this context enqueued work on (top-level calls), with an event
  // recorded after the call: fsb_nonfinite / fsb_input_bytes wait on these
  // instead of synchronising the whole device
  std::vector<std::pair<cudaStream_t, cudaEvent_t>> done;
  cudaStream_t aux = nullptr;  // private non-blocking stream for flag reads
  int* h_flag = nullptr;                  // pinned read-back slots (a pageable target turns the
  unsigned long long* h_bytes = nullptr;  // 4-byte copy into a staged, synchronous transfer)
  // large-config encoder workspaces
  DevMem vit_ws_mem;
  VitWs vit_ws{};
  DevMem encf32_ws_mem;
  EncF32Ws encf32_ws{};
  // workspace
  int ws_frames = 0;
  DevMem ws;
  double* w_boxes = nullptr;
  float *w_prompt = nullptr, *w_crops = nullptr, *w_feats = nullptr, *w_params = nullptr, *w_cam = nullptr,
        *w_rots = nullptr, *w_rel = nullptr, *w_rel2 = nullptr, *w_x = nullptr, *w_h1 = nullptr, *w_h2 = nullptr,
        *w_theta = nullptr, *w_part = nullptr, *w_psum = nullptr, *w_vu = nullptr;
  __nv_bfloat16* w_xb = nullptr;  // projector input as a bf16 A-tile image
  uint8_t *w_lbsin = nullptr, *w_lbsin2 = nullptr;  // k_lbs_tc chunk records (MHR, SMPL)
  uint8_t *w_bkv = nullptr, *w_hkv = nullptr;  // projected cross-attention K / V (bf16 decoders)
  // fsb_encode_frames projected K / V for (kv_feats, kv_frames):
  // fsb_decode_frames on those features reads them instead of re-projecting
  // until the next encode / projection on this context
  const float* kv_feats = nullptr;
  int kv_frames = 0;
  unsigned char *w_h1img = nullptr, *w_h2img = nullptr;
  unsigned char *w_xbl = nullptr, *w_h1l = nullptr, *w_h2l = nullptr;  // fp32 mode: remainder images
  // graphs
  bool graphs = true;
  struct GraphEntry {
    GraphKey key;
    cudaGraphExec_t exec;
    int nodes;
    uint64_t used;
  };
  std::vector<GraphEntry> gcache;  // LRU of captured frame-batch graphs
  uint64_t gclock = 0;
  void drop_graphs() {
    for (auto& e : gcache) cudaGraphExecDestroy(e.exec);
    gcache.clear();
  }
};

namespace {

int fail(fsb_ctx* c, int code, const char* fmt, ...) __attribute__((format(printf, 3, 4)));
int fail(fsb_ctx* c, int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  if (c) c->err = buf;
  return code;
}

#define FSB_CUDA(c, expr)                                                                          \
  do {                                                                                             \
    cudaError_t e_ = (expr);                                                                       \
    if (e_ != cudaSuccess) return fail((c), FSB_ERR_CUDA, "%s: %s", #expr, cudaGetErrorString(e_)); \
  } while (0)

bool default_model(const fsb_decoder_config& c) {
  return c.crop_size == 64 && c.patch == 8 && c.dim == 64 && c.heads == 4 && c.enc_layers <= FSB_MAX_LAYERS &&
         c.body_layers <= 8 && c.hand_layers <= 8;
}

#ifndef FSB_VIT_CHUNK
#define FSB_VIT_CHUNK 256  // 128 / 256 / 384 / 768 measured equal within 2 %; 256 uses the least memory
#endif
constexpr int kVitChunk = FSB_VIT_CHUNK;  // crops per large-config encoder pass

int layer_count(uint32_t sel) { return __builtin_popcount(sel); }

bool capturing(cudaStream_t st) {
  cudaStreamCaptureStatus s = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(st, &s) != cudaSuccess) return false;
  return s != cudaStreamCaptureStatusNone;
}

// The (possibly shared) model was re-uploaded since this context built its
// graphs and workspace: both are stale.
void model_sync(fsb_ctx* c) {
  if (c->seen_version == c->m->version) return;
  c->kv_feats = nullptr;
  c->drop_graphs();
  c->ws_frames = 0;
  c->vit_ws_mem.release();
  c->vit_ws = VitWs{};
  c->encf32_ws_mem.release();
  c->encf32_ws = EncF32Ws{};
  c->seen_version = c->m->version;
}

void model_changed(fsb_ctx* c) {
  ++c->m->version;
  model_sync(c);
}

// record "this context's work on `st` is enqueued up to here" (top-level,
// non-capturing calls only; a captured graph records on its launch)
void note_stream(fsb_ctx* c, cudaStream_t st) {
  if (capturing(st)) return;
  for (auto& d : c->done)
    if (d.first == st) {
      cudaEventRecord(d.second, st);
      return;
    }
  cudaEvent_t ev = nullptr;
  if (cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) != cudaSuccess) return;
  cudaEventRecord(ev, st);
  c->done.push_back({st, ev});
}

// wait for this context's enqueued work only (not the whole device)
cudaError_t wait_own_work(fsb_ctx* c) {
  for (auto& d : c->done) {
    cudaError_t e = cudaEventSynchronize(d.second);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

int ensure_ws(fsb_ctx* c, int frames, cudaStream_t st) {
  model_sync(c);
  if (frames <= c->ws_frames) return FSB_OK;
  if (capturing(st))
    return fail(c, FSB_ERR_USAGE, "workspace for %d frames not reserved before graph capture", frames);
  return fsb_reserve(c, frames);
}

// Large-config encoder upload: bf16 W^T (N x K row-major) per linear layer,
// q|k|v stacked to (3D x D); fp32 biases, LayerNorm affine and positions.
// Only the encoder is device-resident for such configs;
// the decoders stay on the default configuration.
int load_enc_f32(fsb_ctx* c, const fsb_decoder_config& cfg,
                 const std::map<std::string, std::pair<const float*, int64_t>>& tab);

int load_vit(fsb_ctx* c, const fsb_decoder_config& cfg, const std::map<std::string, std::pair<const float*, int64_t>>& tab) {
  const int D = cfg.dim, p = cfg.patch, K0 = p * p * 3;
  // fp32 (reference precision) tables first: any shape with a supported head dim
  int rc = load_enc_f32(c, cfg, tab);
  if (rc) return rc;
  c->m->vit_tc = !(D % 128 || D > 2048 || D / cfg.heads != 64 || D % cfg.heads || K0 % 64);
  if (!c->m->vit_tc) {  // bf16 encode will raise; fp32 runs
    c->m->vit = true;
    c->m->cfg = cfg;
    c->m->has_decoder = true;
    model_changed(c);
    return FSB_OK;
  }
  const int np = cfg.crop_size / p, T = np * np;
  Packer pk;
  std::map<std::string, size_t> off;
  std::string missing;
  auto find = [&](const std::string& name, int64_t n) -> const float* {
    auto it = tab.find(name);
    if (it == tab.end() || it->second.second != n) {
      if (missing.empty()) missing = name;
      return nullptr;
    }
    return it->second.first;
  };
  auto put = [&](const std::string& name, int64_t n) {
    const float* a = find(name, n);
    if (a) off[name] = pk.add(a, (size_t)n * 4);
  };
  // (K x N_i) matrices -> one (sum N_i x K) bf16 W^T, 32x32 blocked transpose
  auto put_t = [&](const std::string& key, std::vector<std::string> mats, int K, int N) {
    std::vector<const float*> src;
    for (auto& m : mats) src.push_back(find(m, (int64_t)K * N));
    for (auto* a : src)
      if (!a) return;
    const int R = N * (int)mats.size();
    const size_t o = pk.add(nullptr, (size_t)R * K * 2);
    __nv_bfloat16* dst = reinterpret_cast<__nv_bfloat16*>(pk.host.data() + o);
    for (size_t t = 0; t < src.size(); ++t)
      for (int k0 = 0; k0 < K; k0 += 32)
        for (int n0 = 0; n0 < N; n0 += 32)
          for (int k = k0; k < k0 + 32 && k < K; ++k)
            for (int n = n0; n < n0 + 32 && n < N; ++n)
              dst[(size_t)(t * N + n) * K + k] = __float2bfloat16_rn(src[t][(size_t)k * N + n]);
    off[key] = o;
  };
  put_t("enc.wpatch", {"enc.patch_w"}, K0, D);
  put("enc.patch_b", D);
  put("enc.pos", (int64_t)T * D);
  put("enc.norm_g", D);
  put("enc.norm_b", D);
  for (int l = 0; l < cfg.enc_layers; ++l) {
    const std::string a = "enc.l" + std::to_string(l) + ".self", m = "enc.l" + std::to_string(l) + ".mlp";
    put_t(a + ".wqkv_t", {a + ".wq", a + ".wk", a + ".wv"}, D, D);
    put_t(a + ".wo_t", {a + ".wo"}, D, D);
    put_t(m + ".w1_t", {m + ".w1"}, D, 4 * D);
    put_t(m + ".w2_t", {m + ".w2"}, 4 * D, D);
    put(a + ".ln_g", D);
    put(a + ".ln_b", D);
    put(a + ".bo", D);
    put(m + ".ln_g", D);
    put(m + ".ln_b", D);
    put(m + ".b1", 4 * D);
    put(m + ".b2", D);
    // q|k|v biases stacked
    const float *bq = find(a + ".bq", D), *bk = find(a + ".bk", D), *bv = find(a + ".bv", D);
    if (bq && bk && bv) {
      std::vector<float> b(3 * (size_t)D);
      memcpy(b.data(), bq, D * 4);
      memcpy(b.data() + D, bk, D * 4);
      memcpy(b.data() + 2 * D, bv, D * 4);
      off[a + ".bqkv"] = pk.add(b.data(), b.size() * 4);
    }
  }
  if (!missing.empty()) return fail(c, FSB_ERR_SHAPE, "encoder weight table: missing or mis-sized '%s'", missing.c_str());
  c->vit_ws_mem.release();
  c->vit_ws = VitWs{};
  FSB_CUDA(c, c->m->dec_mem.alloc(pk.host.size()));
  FSB_CUDA(c, cudaMemcpy(c->m->dec_mem.p, pk.host.data(), pk.host.size(), cudaMemcpyHostToDevice));
  const uint8_t* base = static_cast<const uint8_t*>(c->m->dec_mem.p);
  auto F = [&](const std::string& n) { return reinterpret_cast<const float*>(base + off.at(n)); };
  auto B = [&](const std::string& n) { return reinterpret_cast<const __nv_bfloat16*>(base + off.at(n)); };
  VitW& w = c->m->vitw;
  w.S = cfg.crop_size;
  w.p = p;
  w.D = D;
  w.H = cfg.heads;
  w.T = T;
  w.wpatch = B("enc.wpatch");
  w.patch_b = F("enc.patch_b");
  w.pos = F("enc.pos");
  w.norm_g = F("enc.norm_g");
  w.norm_b = F("enc.norm_b");
  w.layers.clear();
  for (int l = 0; l < cfg.enc_layers; ++l) {
    const std::string a = "enc.l" + std::to_string(l) + ".self", m = "enc.l" + std::to_string(l) + ".mlp";
    w.layers.push_back(VitLayer{B(a + ".wqkv_t"), B(a + ".wo_t"), B(m + ".w1_t"), B(m + ".w2_t"), F(a + ".ln_g"),
                                F(a + ".ln_b"), F(a + ".bqkv"), F(a + ".bo"), F(m + ".ln_g"), F(m + ".ln_b"),
                                F(m + ".b1"), F(m + ".b2")});
  }
  c->m->cfg = cfg;
  c->m->has_decoder = true;
  c->m->vit = true;
  model_changed(c);
  return FSB_OK;
}

// fp32 tables of a non-default encoder (k_enc_f32.cu): the reference's
// (in, out) matrices as they are, q|k|v concatenated to (D, 3D)
int load_enc_f32(fsb_ctx* c, const fsb_decoder_config& cfg,
                 const std::map<std::string, std::pair<const float*, int64_t>>& tab) {
  const int D = cfg.dim, p = cfg.patch, K0 = p * p * 3;
  if (!enc_f32_supported(D, cfg.heads))
    return fail(c, FSB_ERR_USAGE, "encoder head dim %d not supported (16, 32, 64 or 128)",
                cfg.heads ? D / cfg.heads : 0);
  const int np = cfg.crop_size / p, T = np * np;
  Packer pk;
  std::map<std::string, size_t> off;
  std::string missing;
  auto find = [&](const std::string& name, int64_t n) -> const float* {
    auto it = tab.find(name);
    if (it == tab.end() || it->second.second != n) {
      if (missing.empty()) missing = name;
      return nullptr;
    }
    return it->second.first;
  };
  auto put = [&](const std::string& name, int64_t n) {
    const float* a = find(name, n);
    if (a) off[name] = pk.add(a, (size_t)n * 4);
  };
  put("enc.patch_w", (int64_t)K0 * D);
  put("enc.patch_b", D);
  put("enc.pos", (int64_t)T * D);
  put("enc.norm_g", D);
  put("enc.norm_b", D);
  for (int l = 0; l < cfg.enc_layers; ++l) {
    const std::string a = "enc.l" + std::to_string(l) + ".self", m = "enc.l" + std::to_string(l) + ".mlp";
    const float *wq = find(a + ".wq", (int64_t)D * D), *wk = find(a + ".wk", (int64_t)D * D),
                *wv = find(a + ".wv", (int64_t)D * D);
    const float *bq = find(a + ".bq", D), *bk = find(a + ".bk", D), *bv = find(a + ".bv", D);
    if (wq && wk && wv && bq && bk && bv) {
      const size_t o = pk.add(nullptr, (size_t)D * 3 * D * 4);
      float* w = reinterpret_cast<float*>(pk.host.data() + o);
      for (int r = 0; r < D; ++r) {
        memcpy(w + (size_t)r * 3 * D, wq + (size_t)r * D, D * 4);
        memcpy(w + (size_t)r * 3 * D + D, wk + (size_t)r * D, D * 4);
        memcpy(w + (size_t)r * 3 * D + 2 * D, wv + (size_t)r * D, D * 4);
      }
      off[a + ".wqkv32"] = o;
      std::vector<float> b(3 * (size_t)D);
      memcpy(b.data(), bq, D * 4);
      memcpy(b.data() + D, bk, D * 4);
      memcpy(b.data() + 2 * D, bv, D * 4);
      off[a + ".bqkv32"] = pk.add(b.data(), b.size() * 4);
    }
    put(a + ".wo", (int64_t)D * D);
    put(a + ".bo", D);
    put(a + ".ln_g", D);
    put(a + ".ln_b", D);
    put(m + ".ln_g", D);
    put(m + ".ln_b", D);
    put(m + ".w1", (int64_t)D * 4 * D);
    put(m + ".b1", 4 * D);
    put(m + ".w2", (int64_t)4 * D * D);
    put(m + ".b2", D);
  }
  if (!missing.empty()) return fail(c, FSB_ERR_SHAPE, "encoder weight table: missing or mis-sized '%s'", missing.c_str());
  FSB_CUDA(c, c->m->encf32_mem.alloc(pk.host.size()));
  FSB_CUDA(c, cudaMemcpy(c->m->encf32_mem.p, pk.host.data(), pk.host.size(), cudaMemcpyHostToDevice));
  const uint8_t* base = static_cast<const uint8_t*>(c->m->encf32_mem.p);
  auto F = [&](const std::string& n) { return reinterpret_cast<const float*>(base + off.at(n)); };
  EncF32W& w = c->m->encw;
  w.S = cfg.crop_size;
  w.p = p;
  w.D = D;
  w.H = cfg.heads;
  w.T = T;
  w.wpatch = F("enc.patch_w");
  w.patch_b = F("enc.patch_b");
  w.pos = F("enc.pos");
  w.norm_g = F("enc.norm_g");
  w.norm_b = F("enc.norm_b");
  w.layers.clear();
  for (int l = 0; l < cfg.enc_layers; ++l) {
    const std::string a = "enc.l" + std::to_string(l) + ".self", m = "enc.l" + std::to_string(l) + ".mlp";
    w.layers.push_back(EncF32Layer{F(a + ".wqkv32"), F(a + ".bqkv32"), F(a + ".wo"), F(a + ".bo"), F(a + ".ln_g"),
                                   F(a + ".ln_b"), F(m + ".ln_g"), F(m + ".ln_b"), F(m + ".w1"), F(m + ".b1"),
                                   F(m + ".w2"), F(m + ".b2")});
  }
  return FSB_OK;
}

}  // namespace

extern "C" {

const char* fsb_build_info(void) { return "fsb_b200 sm_100a (" __DATE__ ")"; }

static int ctx_new(int device, std::shared_ptr<fsb_model> model, fsb_ctx** out) {
  if (!out) return FSB_ERR_USAGE;
  *out = nullptr;
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) return FSB_ERR_CUDA;
  fsb_ctx* c = new fsb_ctx();
  c->device = device;
  c->mp = model ? model : std::make_shared<fsb_model>();
  c->m = c->mp.get();
  c->seen_version = c->m->version;
  if (init_attrs_transformer() != cudaSuccess || init_attrs_transformer_tc() != cudaSuccess ||
      init_attrs_mlp_tc() != cudaSuccess || init_attrs_gemm_tc() != cudaSuccess ||
      init_attrs_body() != cudaSuccess || init_attrs_crops() != cudaSuccess) {
    delete c;
    return FSB_ERR_CUDA;
  }
  if (cudaMalloc(&c->d_flag, sizeof(int)) != cudaSuccess || cudaMemset(c->d_flag, 0, sizeof(int)) != cudaSuccess ||
      cudaMalloc(&c->d_bytes_in, sizeof(unsigned long long)) != cudaSuccess ||
      cudaMemset(c->d_bytes_in, 0, sizeof(unsigned long long)) != cudaSuccess ||
      cudaStreamCreateWithFlags(&c->aux, cudaStreamNonBlocking) != cudaSuccess ||
      cudaMallocHost(&c->h_flag, sizeof(int)) != cudaSuccess ||
      cudaMallocHost(&c->h_bytes, sizeof(unsigned long long)) != cudaSuccess) {
    fsb_ctx_destroy(c);
    return FSB_ERR_CUDA;
  }
  *out = c;
  return FSB_OK;
}

int fsb_ctx_create(int device, fsb_ctx** out) { return ctx_new(device, nullptr, out); }

int fsb_ctx_create_shared(fsb_ctx* model_owner, fsb_ctx** out) {
  if (!model_owner) return FSB_ERR_USAGE;
  return ctx_new(model_owner->device, model_owner->mp, out);
}

void fsb_ctx_destroy(fsb_ctx* c) {
  if (!c) return;
  c->drop_graphs();
  for (auto& d : c->done) cudaEventDestroy(d.second);
  if (c->aux) cudaStreamDestroy(c->aux);
  if (c->d_flag) cudaFree(c->d_flag);
  if (c->d_bytes_in) cudaFree(c->d_bytes_in);
  if (c->h_flag) cudaFreeHost(c->h_flag);
  if (c->h_bytes) cudaFreeHost(c->h_bytes);
  delete c;  // the model is freed with its last context
}

const char* fsb_last_error(const fsb_ctx* c) { return c ? c->err.c_str() : "null context"; }

int fsb_set_graphs(fsb_ctx* c, int enabled) {
  c->graphs = enabled != 0;
  return FSB_OK;
}

int fsb_reserve(fsb_ctx* c, int max_frames) {
  model_sync(c);
  if (max_frames <= c->ws_frames) return FSB_OK;
  const int S = c->m->has_decoder ? c->m->cfg.crop_size : 0;
  const int T = c->m->has_decoder ? (S / c->m->cfg.patch) * (S / c->m->cfg.patch) : 0;
  const int Dm = c->m->has_decoder ? c->m->cfg.dim : 0;
  const int nsub = c->m->has_proj ? c->m->proj.n_sub : 1500;
  const int h1 = c->m->has_proj ? c->m->proj.h1 : 512, h2 = c->m->has_proj ? c->m->proj.h2 : 256;
  const size_t F = (size_t)max_frames;
  size_t off = 0;
  auto take = [&](size_t bytes) {
    const size_t o = off;
    off += (bytes + 255) & ~size_t(255);
    return o;
  };
  const size_t o_boxes = take(F * 12 * sizeof(double));
  const size_t o_prompt = take(F * 8 * 4);
  const size_t o_crops = take(F * 3 * S * S * 3 * 4);
  const size_t o_feats = take(F * 3 * T * Dm * 4);
  const size_t o_params = take(F * 76 * 4);
  const size_t o_cam = take(F * 3 * 4);
  const size_t o_rots = take(F * 6 * 4);
  const size_t o_rel = take(F * FSB_NJ * 12 * 4);
  const size_t o_rel2 = take(F * FSB_NJ * 12 * 4);
  const size_t o_x = take(F * 3 * nsub * 4);
  // bf16 A-tile images of the tensor-core projector (k_mlp_tc.cu)
  const size_t mtiles = (F + 127) / 128;
  const size_t ximg_bytes = mtiles * ((3 * (size_t)nsub + 127) / 128) * 32768;
  const size_t h1img_bytes = mtiles * ((h1 + 127) / 128) * 32768;
  const size_t h2img_bytes = mtiles * ((h2 + 127) / 128) * 32768;
  const size_t o_xb = take(ximg_bytes);
  const size_t o_h1i = take(h1img_bytes);
  const size_t o_h2i = take(h2img_bytes);
  // fp32 mode's remainder images (split-bf16), right behind (one memset)
  const size_t o_xbl = take(ximg_bytes);
  const size_t o_h1l = take(h1img_bytes);
  const size_t o_h2l = take(h2img_bytes);
  const size_t o_h1 = take(F * h1 * 4);
  const size_t o_h2 = take(F * h2 * 4);
  const size_t o_theta = take(F * 76 * 4);
  const int hmax = h1 > h2 ? (h1 > 76 ? h1 : 76) : (h2 > 76 ? h2 : 76);
  const size_t o_part = take(F * 48 * (size_t)hmax * 4);  // split-K partials (<= 16 chunks; x 3 split-bf16)
  const size_t o_psum = take(F * 8 * 3 * 4);               // projector-input centroid partials
  const size_t o_vu = take(F * (size_t)(c->m->has_proj ? c->m->proj.nu : 1) * 3 * 4);  // compacted corners
  const size_t lbsin_bytes = (F + FSB_LBS_N - 1) / FSB_LBS_N * (size_t)FSB_LBS_REC_BYTES;
  const size_t o_lbsin = take(lbsin_bytes);
  const size_t o_lbsin2 = take(lbsin_bytes);
  const int Lb = c->m->has_decoder ? c->m->cfg.body_layers : 0, Lh = c->m->has_decoder ? c->m->cfg.hand_layers : 0;
  const size_t o_bkv = take((F + 1) / 2 * (size_t)Lb * FSB_KV_BODY_TILE);
  const size_t o_hkv = take((2 * F + FSB_HANDS_PER_TILE - 1) / FSB_HANDS_PER_TILE * FSB_HANDS_PER_TILE * (size_t)Lh *
                            FSB_KV_HAND);
  c->drop_graphs();
  c->kv_feats = nullptr;
  FSB_CUDA(c, c->ws.alloc(off));
  unsigned char* b = static_cast<unsigned char*>(c->ws.p);
  // zero padding of the tile images (k columns past K, rows past B) must stay
  // finite: clear once, kernels only ever write the live region
  FSB_CUDA(c, cudaMemset(b + o_xb, 0, o_h2l + h2img_bytes - o_xb));
  c->w_h1img = b + o_h1i;
  c->w_h2img = b + o_h2i;
  c->w_xbl = b + o_xbl;
  c->w_h1l = b + o_h1l;
  c->w_h2l = b + o_h2l;
  c->w_boxes = reinterpret_cast<double*>(b + o_boxes);
  c->w_prompt = reinterpret_cast<float*>(b + o_prompt);
  c->w_crops = reinterpret_cast<float*>(b + o_crops);
  c->w_feats = reinterpret_cast<float*>(b + o_feats);
  c->w_params = reinterpret_cast<float*>(b + o_params);
  c->w_cam = reinterpret_cast<float*>(b + o_cam);
  c->w_rots = reinterpret_cast<float*>(b + o_rots);
  c->w_rel = reinterpret_cast<float*>(b + o_rel);
  c->w_rel2 = reinterpret_cast<float*>(b + o_rel2);
  c->w_x = reinterpret_cast<float*>(b + o_x);
  c->w_xb = reinterpret_cast<__nv_bfloat16*>(b + o_xb);
  c->w_h1 = reinterpret_cast<float*>(b + o_h1);
  c->w_h2 = reinterpret_cast<float*>(b + o_h2);
  c->w_theta = reinterpret_cast<float*>(b + o_theta);
  c->w_part = reinterpret_cast<float*>(b + o_part);
  c->w_psum = reinterpret_cast<float*>(b + o_psum);
  c->w_vu = reinterpret_cast<float*>(b + o_vu);
  // the shape images' K padding (k >= 10) and meshes past B stay zero
  FSB_CUDA(c, cudaMemset(b + o_lbsin, 0, o_lbsin2 - o_lbsin + lbsin_bytes));
  c->w_lbsin = b + o_lbsin;
  c->w_lbsin2 = b + o_lbsin2;
  c->w_bkv = b + o_bkv;
  c->w_hkv = b + o_hkv;
  c->ws_frames = max_frames;
  return FSB_OK;
}

// ---------------------------------------------------------------------------
// model upload

int fsb_load_decoder(fsb_ctx* c, const fsb_decoder_config* cfg, int n, const char* const* names,
                     const float* const* arrays, const int64_t* numel) {
  if (!cfg || n <= 0) return fail(c, FSB_ERR_USAGE, "fsb_load_decoder: empty weight table");
  std::map<std::string, std::pair<const float*, int64_t>> tab;
  for (int i = 0; i < n; ++i) tab[names[i]] = {arrays[i], numel[i]};
  const int Dm = cfg->dim;
  if (Dm <= 0 || cfg->heads <= 0 || Dm % cfg->heads || cfg->patch <= 0 || cfg->crop_size % cfg->patch)
    return fail(c, FSB_ERR_SHAPE, "inconsistent decoder config");
  if (cfg->enc_layers > FSB_MAX_LAYERS || cfg->body_layers > 8 || cfg->hand_layers > 8)
    return fail(c, FSB_ERR_USAGE, "too many layers for the device tables");
  if (!default_model(*cfg)) return load_vit(c, *cfg, tab);
  Packer pk;
  std::map<std::string, size_t> off;
  std::string missing;
  auto put = [&](const std::string& name, int64_t expect) -> bool {
    auto it = tab.find(name);
    if (it == tab.end()) {
      missing = name;
      return false;
    }
    if (expect >= 0 && it->second.second != expect) {
      missing = name + " (size)";
      return false;
    }
    off[name] = pk.add(it->second.first, (size_t)it->second.second * 4);
    return true;
  };
  // q|k|v concatenated to (D, 3D) and the biases to (3D)
  auto put_qkv = [&](const std::string& p) -> bool {
    const char* ws[3] = {".wq", ".wk", ".wv"};
    const char* bs[3] = {".bq", ".bk", ".bv"};
    std::vector<float> w((size_t)Dm * 3 * Dm), b((size_t)3 * Dm);
    for (int t = 0; t < 3; ++t) {
      auto iw = tab.find(p + ws[t]);
      auto ib = tab.find(p + bs[t]);
      if (iw == tab.end() || ib == tab.end() || iw->second.second != (int64_t)Dm * Dm || ib->second.second != Dm) {
        missing = p + ws[t];
        return false;
      }
      for (int r = 0; r < Dm; ++r)
        for (int q = 0; q < Dm; ++q) w[(size_t)r * 3 * Dm + t * Dm + q] = iw->second.first[(size_t)r * Dm + q];
      for (int q = 0; q < Dm; ++q) b[t * Dm + q] = ib->second.first[q];
    }
    off[p + ".wqkv"] = pk.add(w.data(), w.size() * 4);
    off[p + ".bqkv"] = pk.add(b.data(), b.size() * 4);
    return true;
  };
  // bf16 image of W^T for the tensor-core kernels: the column concatenation
  // of (K x N_i) matrices, packed in the K-major UMMA layout (tc_sm100.cuh)
  auto put_img = [&](const std::string& key, std::vector<std::string> mats, int K) -> bool {
    std::vector<std::pair<const float*, int>> src;
    int Ntot = 0;
    for (auto& m : mats) {
      auto it = tab.find(m);
      if (it == tab.end() || it->second.second % K) {
        missing = m + " (image)";
        return false;
      }
      src.push_back({it->second.first, (int)(it->second.second / K)});
      Ntot += src.back().second;
    }
    if (Ntot % 8 || K % 8) {
      missing = key + " (image shape)";
      return false;
    }
    std::vector<__nv_bfloat16> img((size_t)Ntot * K);
    int n0 = 0;
    for (auto& s : src) {
      for (int nn = 0; nn < s.second; ++nn)
        for (int k = 0; k < K; ++k)
          img[tc_kmajor_off(n0 + nn, k, K) / 2] = __float2bfloat16_rn(s.first[(size_t)k * s.second + nn]);
      n0 += s.second;
    }
    off[key] = pk.add(img.data(), img.size() * 2);
    return true;
  };
  auto attn = [&](const std::string& p, bool cross) -> bool {
    bool ok = cross ? (put(p + ".lnq_g", Dm) && put(p + ".lnq_b", Dm) && put(p + ".lnkv_g", Dm) &&
                       put(p + ".lnkv_b", Dm))
                    : (put(p + ".ln_g", Dm) && put(p + ".ln_b", Dm));
    ok = ok && (cross ? (put_img(p + ".t_q", {p + ".wq"}, Dm) && put_img(p + ".t_kv", {p + ".wk", p + ".wv"}, Dm))
                      : put_img(p + ".t_qkv", {p + ".wq", p + ".wk", p + ".wv"}, Dm));
    return ok && put_qkv(p) && put(p + ".wo", (int64_t)Dm * Dm) && put(p + ".bo", Dm) &&
           put_img(p + ".t_o", {p + ".wo"}, Dm);
  };
  auto mlp = [&](const std::string& p) -> bool {
    return put(p + ".ln_g", Dm) && put(p + ".ln_b", Dm) && put(p + ".w1", (int64_t)Dm * 4 * Dm) &&
           put(p + ".b1", 4 * Dm) && put(p + ".w2", (int64_t)4 * Dm * Dm) && put(p + ".b2", Dm) &&
           put_img(p + ".t_w1", {p + ".w1"}, Dm) && put_img(p + ".t_w2", {p + ".w2"}, 4 * Dm);
  };
  const int np = (cfg->crop_size / cfg->patch) * (cfg->crop_size / cfg->patch);
  bool ok = put("enc.patch_w", (int64_t)cfg->patch * cfg->patch * 3 * Dm) && put("enc.patch_b", Dm) &&
            put("enc.pos", (int64_t)np * Dm) && put("enc.norm_g", Dm) && put("enc.norm_b", Dm) &&
            put_img("enc.t_patch", {"enc.patch_w"}, cfg->patch * cfg->patch * 3);
  for (int l = 0; ok && l < cfg->enc_layers; ++l)
    ok = attn("enc.l" + std::to_string(l) + ".self", false) && mlp("enc.l" + std::to_string(l) + ".mlp");
  ok = ok && put("body.token_init", 51 * Dm) && put("body.p2d_init", 22 * Dm) && put("body.p3d_init", 22 * Dm) &&
       put("body.norm_g", Dm) && put("body.norm_b", Dm);
  for (int l = 0; ok && l < cfg->body_layers; ++l) {
    const std::string p = "body.l" + std::to_string(l);
    ok = attn(p + ".self", false) && attn(p + ".cross", true) && mlp(p + ".mlp");
  }
  ok = ok && put("body.head_params.w", (int64_t)Dm * 76) && put("body.head_params.b", 76) &&
       put("body.head_cam.w", (int64_t)Dm * 3) && put("body.head_cam.b", 3) && put("body.phi2d.w", 2 * Dm) &&
       put("body.phi2d.b", Dm) && put("body.phi3d.w", 3 * Dm) && put("body.phi3d.b", Dm) &&
       put("body.prompt_box.w", 8 * 4 * Dm) && put("body.prompt_box.b", 4 * Dm);
  ok = ok && put("hand.token_init", 4 * Dm) && put("hand.p_init", 3 * Dm) && put("hand.norm_g", Dm) &&
       put("hand.norm_b", Dm);
  for (int l = 0; ok && l < cfg->hand_layers; ++l) {
    const std::string p = "hand.l" + std::to_string(l);
    ok = attn(p + ".self", false) && attn(p + ".cross", true) && mlp(p + ".mlp");
  }
  ok = ok && put("hand.head_rot.w", (int64_t)Dm * 3) && put("hand.head_rot.b", 3) &&
       put("hand.head_cam.w", (int64_t)Dm * 3) && put("hand.head_cam.b", 3) && put("hand.phi2d.w", 2 * Dm) &&
       put("hand.phi2d.b", Dm) && put("hand.canon_pts", 9);
  // per-layer TCP_* parameter blocks of the tensor-core kernels (fsb_weights.h)
  auto put_params = [&](const std::string& key, const std::string& ps, const std::string& pc,
                        const std::string& pm) -> bool {
    std::vector<float> blk(TCP_FLOATS, 0.0f);
    auto cp = [&](const std::string& name, int at, int n) -> bool {
      auto it = tab.find(name);
      if (it == tab.end() || it->second.second != n) {
        missing = name + " (param block)";
        return false;
      }
      memcpy(blk.data() + at, it->second.first, (size_t)n * 4);
      return true;
    };
    bool good = cp(ps + ".ln_g", TCP_S_LN_G, Dm) && cp(ps + ".ln_b", TCP_S_LN_B, Dm) &&
                cp(ps + ".bq", TCP_S_BQKV, Dm) && cp(ps + ".bk", TCP_S_BQKV + Dm, Dm) &&
                cp(ps + ".bv", TCP_S_BQKV + 2 * Dm, Dm) && cp(ps + ".bo", TCP_S_BO, Dm) &&
                cp(pm + ".ln_g", TCP_M_LN_G, Dm) && cp(pm + ".ln_b", TCP_M_LN_B, Dm) &&
                cp(pm + ".b1", TCP_M_B1, 4 * Dm) && cp(pm + ".b2", TCP_M_B2, Dm);
    if (good && !pc.empty())
      good = cp(pc + ".lnq_g", TCP_C_LNQ_G, Dm) && cp(pc + ".lnq_b", TCP_C_LNQ_B, Dm) &&
             cp(pc + ".lnkv_g", TCP_C_LNKV_G, Dm) && cp(pc + ".lnkv_b", TCP_C_LNKV_B, Dm) &&
             cp(pc + ".bq", TCP_C_BQKV, Dm) && cp(pc + ".bk", TCP_C_BQKV + Dm, Dm) &&
             cp(pc + ".bv", TCP_C_BQKV + 2 * Dm, Dm) && cp(pc + ".bo", TCP_C_BO, Dm);
    if (good) off[key] = pk.add(blk.data(), blk.size() * 4);
    return good;
  };
  if (ok && Dm == 64) {
    for (int l = 0; ok && l < cfg->enc_layers; ++l) {
      const std::string p = "enc.l" + std::to_string(l);
      ok = put_params(p + ".tcp", p + ".self", "", p + ".mlp");
    }
    for (int l = 0; ok && l < cfg->body_layers; ++l) {
      const std::string p = "body.l" + std::to_string(l);
      ok = put_params(p + ".tcp", p + ".self", p + ".cross", p + ".mlp");
    }
    for (int l = 0; ok && l < cfg->hand_layers; ++l) {
      const std::string p = "hand.l" + std::to_string(l);
      ok = put_params(p + ".tcp", p + ".self", p + ".cross", p + ".mlp");
    }
    // The K / V projection ahead of the decoders (kv_project, k_transformer_tc.cu)
    // normalises the features once and folds each layer's LN_kv affine into
    // its weights: LN_l(f) [Wk | Wv] + [bk | bv] = n(f) (diag(g_l) [Wk | Wv])
    // + (b_l [Wk | Wv] + [bk | bv]).  Layers are packed in pairs: a bf16
    // image of 256 rows (layer 2p's 128 K | V columns, then 2p + 1's) and a
    // parameter block holding the folded biases at [0, 256).
    for (int role = 0; ok && role < 2; ++role) {
      const std::string rn = role == 0 ? "body" : "hand";
      const int L = role == 0 ? cfg->body_layers : cfg->hand_layers;
      for (int l0 = 0; ok && l0 < L; l0 += 2) {
        const int nl = L - l0 < 2 ? L - l0 : 2;
        std::vector<__nv_bfloat16> img((size_t)nl * 128 * Dm);
        std::vector<float> blk(TCP_FLOATS, 0.0f);
        for (int j = 0; ok && j < nl; ++j) {
          const std::string p = rn + ".l" + std::to_string(l0 + j) + ".cross";
          auto g = tab.find(p + ".lnkv_g"), be = tab.find(p + ".lnkv_b");
          auto wk = tab.find(p + ".wk"), wv = tab.find(p + ".wv"), bk = tab.find(p + ".bk"), bv = tab.find(p + ".bv");
          if (g == tab.end() || be == tab.end() || wk == tab.end() || wv == tab.end() || bk == tab.end() ||
              bv == tab.end()) {
            missing = p + " (K / V projection)";
            ok = false;
            break;
          }
          for (int n = 0; n < 2 * Dm; ++n) {
            const float* W = n < Dm ? wk->second.first : wv->second.first;
            const int nn = n % Dm;
            double acc = (n < Dm ? bk->second.first : bv->second.first)[nn];
            for (int k = 0; k < Dm; ++k) {
              const float w = W[(size_t)k * Dm + nn];
              img[tc_kmajor_off(128 * j + n, k, Dm) / 2] = __float2bfloat16_rn(g->second.first[k] * w);
              acc += (double)be->second.first[k] * w;
            }
            blk[128 * j + n] = (float)acc;
          }
        }
        if (!ok) break;
        off[rn + ".kvimg" + std::to_string(l0 / 2)] = pk.add(img.data(), img.size() * 2);
        off[rn + ".kvprm" + std::to_string(l0 / 2)] = pk.add(blk.data(), blk.size() * 4);
      }
    }
  }
  if (!ok) return fail(c, FSB_ERR_SHAPE, "decoder weight table: missing or mis-sized '%s'", missing.c_str());
  FSB_CUDA(c, c->m->dec_mem.alloc(pk.host.size()));
  FSB_CUDA(c, cudaMemcpy(c->m->dec_mem.p, pk.host.data(), pk.host.size(), cudaMemcpyHostToDevice));
  const unsigned char* base = static_cast<const unsigned char*>(c->m->dec_mem.p);
  auto P = [&](const std::string& name) { return reinterpret_cast<const float*>(base + off.at(name)); };
  auto I = [&](const std::string& name) { return reinterpret_cast<const uint8_t*>(base + off.at(name)); };
  auto fill_attn = [&](AttnW& a, const std::string& p, bool cross) {
    a.ln_g = P(p + (cross ? ".lnq_g" : ".ln_g"));
    a.ln_b = P(p + (cross ? ".lnq_b" : ".ln_b"));
    a.ln2_g = cross ? P(p + ".lnkv_g") : nullptr;
    a.ln2_b = cross ? P(p + ".lnkv_b") : nullptr;
    a.wqkv = P(p + ".wqkv");
    a.bqkv = P(p + ".bqkv");
    a.wo = P(p + ".wo");
    a.bo = P(p + ".bo");
    a.t_qkv = cross ? nullptr : I(p + ".t_qkv");
    a.t_q = cross ? I(p + ".t_q") : nullptr;
    a.t_kv = cross ? I(p + ".t_kv") : nullptr;
    a.t_o = I(p + ".t_o");
  };
  auto fill_mlp = [&](MlpW& m, const std::string& p) {
    m.ln_g = P(p + ".ln_g");
    m.ln_b = P(p + ".ln_b");
    m.w1 = P(p + ".w1");
    m.b1 = P(p + ".b1");
    m.w2 = P(p + ".w2");
    m.b2 = P(p + ".b2");
    m.t_w1 = I(p + ".t_w1");
    m.t_w2 = I(p + ".t_w2");
  };
  EncW& e = c->m->enc;
  e.t_patch = I("enc.t_patch");
  e.patch_w = P("enc.patch_w");
  e.patch_b = P("enc.patch_b");
  e.pos = P("enc.pos");
  e.norm_g = P("enc.norm_g");
  e.norm_b = P("enc.norm_b");
  e.layers = cfg->enc_layers;
  auto PT = [&](const std::string& name) { return off.count(name) ? P(name) : nullptr; };
  for (int l = 0; l < cfg->enc_layers; ++l) {
    fill_attn(e.self[l], "enc.l" + std::to_string(l) + ".self", false);
    fill_mlp(e.mlp[l], "enc.l" + std::to_string(l) + ".mlp");
    e.tc_params[l] = PT("enc.l" + std::to_string(l) + ".tcp");
  }
  BodyW& b = c->m->body;
  b.token_init = P("body.token_init");
  b.p2d_init = P("body.p2d_init");
  b.p3d_init = P("body.p3d_init");
  b.norm_g = P("body.norm_g");
  b.norm_b = P("body.norm_b");
  b.head_params_w = P("body.head_params.w");
  b.head_params_b = P("body.head_params.b");
  b.head_cam_w = P("body.head_cam.w");
  b.head_cam_b = P("body.head_cam.b");
  b.phi2d_w = P("body.phi2d.w");
  b.phi2d_b = P("body.phi2d.b");
  b.phi3d_w = P("body.phi3d.w");
  b.phi3d_b = P("body.phi3d.b");
  b.prompt_box_w = P("body.prompt_box.w");
  b.prompt_box_b = P("body.prompt_box.b");
  b.layers = cfg->body_layers;
  for (int l = 0; l < cfg->body_layers; ++l) {
    const std::string p = "body.l" + std::to_string(l);
    fill_attn(b.self[l], p + ".self", false);
    fill_attn(b.cross[l], p + ".cross", true);
    fill_mlp(b.mlp[l], p + ".mlp");
    b.tc_params[l] = PT(p + ".tcp");
  }
  HandW& h = c->m->hand;
  h.token_init = P("hand.token_init");
  h.p_init = P("hand.p_init");
  h.norm_g = P("hand.norm_g");
  h.norm_b = P("hand.norm_b");
  h.head_rot_w = P("hand.head_rot.w");
  h.head_rot_b = P("hand.head_rot.b");
  h.head_cam_w = P("hand.head_cam.w");
  h.head_cam_b = P("hand.head_cam.b");
  h.phi2d_w = P("hand.phi2d.w");
  h.phi2d_b = P("hand.phi2d.b");
  h.canon_pts = P("hand.canon_pts");
  h.layers = cfg->hand_layers;
  for (int l = 0; l < cfg->hand_layers; ++l) {
    const std::string p = "hand.l" + std::to_string(l);
    fill_attn(h.self[l], p + ".self", false);
    fill_attn(h.cross[l], p + ".cross", true);
    fill_mlp(h.mlp[l], p + ".mlp");
    h.tc_params[l] = PT(p + ".tcp");
  }
  // tcgen05 weight streams in consumption order (k_transformer_tc.cu)
  if (Dm == 64) {
    TcStream ts[7]{};
    auto img = [&](TcStream& t, const uint8_t* ptr, uint32_t bytes) {
      if (t.nw < FSB_TC_MAX_IMAGES) {
        t.wptr[t.nw] = ptr;
        t.wbytes[t.nw] = bytes;
      }
      ++t.nw;
    };
    const uint32_t DD = 64 * 64 * 2;
    img(ts[0], e.t_patch, 192 * 64 * 2);
    for (int l = 0; l < e.layers; ++l) {
      img(ts[0], e.self[l].t_qkv, 3 * DD);
      img(ts[0], e.self[l].t_o, DD);
      img(ts[0], e.mlp[l].t_w1, 4 * DD);
      img(ts[0], e.mlp[l].t_w2, 4 * DD);
      ts[0].pptr[l] = e.tc_params[l];
    }
    ts[0].nprm = e.layers;
    for (int role = 0; role < 2; ++role) {
      TcStream& t = ts[1 + role];
      const int L = role == 0 ? b.layers : h.layers;
      for (int l = 0; l < L; ++l) {
        const AttnW& sa = role == 0 ? b.self[l] : h.self[l];
        const AttnW& ca = role == 0 ? b.cross[l] : h.cross[l];
        const MlpW& m = role == 0 ? b.mlp[l] : h.mlp[l];
        img(t, sa.t_qkv, 3 * DD);
        img(t, sa.t_o, DD);
        img(t, ca.t_q, DD);  // K | V were projected ahead (kv_project)
        img(t, ca.t_o, DD);
        img(t, m.t_w1, 4 * DD);
        img(t, m.t_w2, 4 * DD);
        t.pptr[l] = role == 0 ? b.tc_params[l] : h.tc_params[l];
      }
      t.nprm = L;
      // K / V projection streams: after the encoder's (frame encode) or
      // alone (given features); one folded image + bias block per layer pair
      for (int mode = 0; mode < 2; ++mode) {
        TcStream& k = ts[3 + 2 * mode + role];
        if (mode == 0) k = ts[0];
        const std::string rn = role == 0 ? "body" : "hand";
        for (int l0 = 0; l0 < L; l0 += 2) {
          const int nl = L - l0 < 2 ? L - l0 : 2;
          img(k, I(rn + ".kvimg" + std::to_string(l0 / 2)), (uint32_t)nl * 2 * DD);
          k.pptr[k.nprm++] = PT(rn + ".kvprm" + std::to_string(l0 / 2));
        }
      }
    }
    for (int i = 0; i < 7; ++i)
      if (ts[i].nw > FSB_TC_MAX_IMAGES)
        return fail(c, FSB_ERR_USAGE, "decoder too deep for the tcgen05 weight stream (%d images > %d)", ts[i].nw,
                    FSB_TC_MAX_IMAGES);
    FSB_CUDA(c, c->m->tcs_mem.alloc(sizeof ts));
    FSB_CUDA(c, cudaMemcpy(c->m->tcs_mem.p, ts, sizeof ts, cudaMemcpyHostToDevice));
    const TcStream* dts = static_cast<const TcStream*>(c->m->tcs_mem.p);
    e.tcs = dts;
    b.tcs = dts + 1;
    h.tcs = dts + 2;
    for (int mode = 0; mode < 2; ++mode)
      for (int role = 0; role < 2; ++role) c->m->kv_tcs[mode][role] = dts + 3 + 2 * mode + role;
  }
  // the body decoder's FK uses the decoder template's rest joints; the
  // body template upload patches it in (fsb_load_template)
  c->m->body.joints_rest = c->m->has_tmpl[FSB_SMPL] ? c->m->tmpl[FSB_SMPL].joints_rest : nullptr;
  c->m->cfg = *cfg;
  c->m->has_decoder = true;
  c->m->vit = false;
  model_changed(c);
  return FSB_OK;
}

int fsb_load_template(fsb_ctx* c, int which, int nv, const float* v_rest, const float* joints_rest,
                      const int64_t* parents, const float* skin_weights, const float* shape_basis) {
  if (which != FSB_MHR && which != FSB_SMPL) return fail(c, FSB_ERR_USAGE, "template id must be 0 (mhr) or 1 (smpl)");
  if (nv <= 0) return fail(c, FSB_ERR_SHAPE, "template needs vertices");
  static const int64_t kPar[FSB_NJ] = {-1, 0, 1, 2, 3, 4, 0, 6, 7, 8, 0, 10, 11, 12, 3, 14, 15, 16, 3, 18, 19, 20};
  for (int j = 0; j < FSB_NJ; ++j)
    if (parents[j] != kPar[j]) return fail(c, FSB_ERR_USAGE, "only the 22-joint toy kinematic tree is supported");
  int maxnz = 0;
  for (int v = 0; v < nv; ++v) {
    int nz = 0;
    for (int j = 0; j < FSB_NJ; ++j) nz += skin_weights[(size_t)v * FSB_NJ + j] != 0.0f;
    maxnz = nz > maxnz ? nz : maxnz;
  }
  const int NZ = maxnz <= 2 ? 2 : (maxnz <= 4 ? 4 : (maxnz <= 8 ? 8 : -1));
  if (NZ < 0) return fail(c, FSB_ERR_USAGE, "skin weights with %d nonzeros per vertex (max 8)", maxnz);
  std::vector<int16_t> sj((size_t)nv * NZ, 0);
  std::vector<float> sw((size_t)nv * NZ, 0.0f);
  for (int v = 0; v < nv; ++v) {
    int z = 0;
    for (int j = 0; j < FSB_NJ; ++j) {
      const float w = skin_weights[(size_t)v * FSB_NJ + j];
      if (w != 0.0f) {
        sj[(size_t)v * NZ + z] = (int16_t)j;
        sw[(size_t)v * NZ + z] = w;
        ++z;
      }
    }
  }
  // vertex records for vectorised loads (fsb_weights.h)
  const int RS = vertex_record_floats(NZ);
  std::vector<float> rec((size_t)nv * RS, 0.0f);
  for (int v = 0; v < nv; ++v) {
    float* r = rec.data() + (size_t)v * RS;
    for (int a = 0; a < 3; ++a) r[a] = v_rest[(size_t)v * 3 + a];
    for (int k = 0; k < 30; ++k) r[4 + k] = shape_basis[(size_t)v * 30 + k];
    for (int z = 0; z < NZ; ++z) {
      r[34 + z] = sw[(size_t)v * NZ + z];
      const int jid = sj[(size_t)v * NZ + z];
      memcpy(&r[34 + NZ + z], &jid, 4);
    }
  }
  // skin weights by joint (CSR) for the iterative fit
  std::vector<int> joff(FSB_NJ + 1, 0), jv;
  std::vector<float> jw;
  for (int j = 0; j < FSB_NJ; ++j) {
    joff[j] = (int)jv.size();
    for (int v = 0; v < nv; ++v) {
      const float w = skin_weights[(size_t)v * FSB_NJ + j];
      if (w != 0.0f) {
        jv.push_back(v);
        jw.push_back(w);
      }
    }
  }
  joff[FSB_NJ] = (int)jv.size();
  // bf16 hi / lo images of the shape basis per 256-vertex tile (k_lbs_tc):
  // row i of parity e is vertex 2 i + e
  const int ntiles = (nv + FSB_LBS_TILE - 1) / FSB_LBS_TILE;
  std::vector<uint8_t> bimg((size_t)ntiles * FSB_LBS_BASIS_BYTES, 0);
  for (int tile = 0; tile < ntiles; ++tile)
    for (int i = 0; i < 128; ++i)
      for (int e = 0; e < 2; ++e) {
        const int v = tile * FSB_LBS_TILE + 2 * i + e;
        if (v >= nv) continue;
        for (int cc = 0; cc < 3; ++cc)
          for (int k = 0; k < 10; ++k) {
            const float x = shape_basis[(size_t)v * 30 + cc * 10 + k];
            const __nv_bfloat16 hi = __float2bfloat16_rn(x);
            const __nv_bfloat16 lo = __float2bfloat16_rn(x - __bfloat162float(hi));
            uint8_t* base = bimg.data() + (size_t)tile * FSB_LBS_BASIS_BYTES + tc_kmajor_off(i, k, 16);
            memcpy(base + (e * 6 + cc) * 4096, &hi, 2);
            memcpy(base + (e * 6 + 3 + cc) * 4096, &lo, 2);
          }
      }
  Packer pk;
  const size_t o_v = pk.add(v_rest, (size_t)nv * 12);
  const size_t o_s = pk.add(shape_basis, (size_t)nv * 30 * 4);
  const size_t o_j = pk.add(sj.data(), sj.size() * 2);
  const size_t o_w = pk.add(sw.data(), sw.size() * 4);
  const size_t o_g = pk.add(joints_rest, FSB_NJ * 12);
  const size_t o_r = pk.add(rec.data(), rec.size() * 4);
  const size_t o_jo = pk.add(joff.data(), joff.size() * 4);
  const size_t o_jv = pk.add(jv.data(), jv.size() * 4 + 4);
  const size_t o_jw = pk.add(jw.data(), jw.size() * 4 + 4);
  const size_t o_bi = pk.add(bimg.data(), bimg.size());
  DevMem& m = c->m->tmpl_mem[which];
  FSB_CUDA(c, m.alloc(pk.host.size()));
  FSB_CUDA(c, cudaMemcpy(m.p, pk.host.data(), pk.host.size(), cudaMemcpyHostToDevice));
  const unsigned char* base = static_cast<const unsigned char*>(m.p);
  TemplateDev& t = c->m->tmpl[which];
  t.nv = nv;
  t.nnz = NZ;
  t.v_rest = reinterpret_cast<const float*>(base + o_v);
  t.shape_basis = reinterpret_cast<const float*>(base + o_s);
  t.skin_j = reinterpret_cast<const int16_t*>(base + o_j);
  t.skin_w = reinterpret_cast<const float*>(base + o_w);
  t.joints_rest = reinterpret_cast<const float*>(base + o_g);
  t.rec = reinterpret_cast<const float*>(base + o_r);
  t.joint_off = reinterpret_cast<const int*>(base + o_jo);
  t.joint_v = reinterpret_cast<const int*>(base + o_jv);
  t.joint_w = reinterpret_cast<const float*>(base + o_jw);
  t.basis_img = base + o_bi;
  c->m->has_tmpl[which] = true;
  if (which == FSB_SMPL) c->m->body.joints_rest = t.joints_rest;
  model_changed(c);
  return FSB_OK;
}

int fsb_load_projector(fsb_ctx* c, int n_sub, int h1, int h2, const int64_t* corners, const float* bary,
                       const float* w1, const float* b1, const float* w2, const float* b2, const float* w3,
                       const float* b3, const float* mask) {
  if (n_sub <= 0 || h1 <= 0 || h2 <= 0) return fail(c, FSB_ERR_SHAPE, "projector sizes must be positive");
  const int K = 3 * n_sub;
  std::vector<int32_t> cr((size_t)n_sub * 3);
  int32_t cmax = 0;
  for (size_t i = 0; i < cr.size(); ++i) {
    cr[i] = (int32_t)corners[i];
    if (cr[i] < 0) return fail(c, FSB_ERR_SHAPE, "projector corner %d is negative", cr[i]);
    cmax = cr[i] > cmax ? cr[i] : cmax;
  }
  // compacted corner slots (ProjectorDev::nu): vertex 0 first, then the
  // distinct corners in vertex order
  std::vector<int32_t> vslot((size_t)cmax + 1, -1), ucr(cr.size());
  std::vector<char> used(vslot.size(), 0);
  for (int32_t v : cr) used[v] = 1;
  int32_t nu = 0;
  vslot[0] = nu++;
  for (size_t v = 1; v < vslot.size(); ++v)
    if (used[v]) vslot[v] = nu++;
  for (size_t i = 0; i < cr.size(); ++i) ucr[i] = vslot[cr[i]];
  // bf16 tile images of W^T (k_mlp_tc.cu): [n_tile][k_tile] 128 x 128
  // K-major tiles, zero padded in both n and k
  // lo = true: the remainder image bf16(W - bf16(W)) (fp32 mode's split-bf16)
  auto tile_image = [](const float* W, int Kin, int Nout, bool lo) {
    const int KT = (Kin + 127) / 128, NT = (Nout + 127) / 128;
    std::vector<__nv_bfloat16> img((size_t)NT * KT * 128 * 128, __float2bfloat16_rn(0.0f));
    for (int k = 0; k < Kin; ++k)
      for (int n = 0; n < Nout; ++n) {
        const size_t tile = (size_t)(n / 128) * KT + (k / 128);
        const float w = W[(size_t)k * Nout + n];
        const __nv_bfloat16 hi = __float2bfloat16_rn(w);
        img[tile * 16384 + tc_kmajor_off(n % 128, k % 128, 128) / 2] =
            lo ? __float2bfloat16_rn(w - __bfloat162float(hi)) : hi;
      }
    return img;
  };
  const bool tc_ok = h1 % 128 == 0 && h2 % 128 == 0;
  std::vector<__nv_bfloat16> i1, i2, i3, l1, l2, l3;
  if (tc_ok) {
    i1 = tile_image(w1, K, h1, false);
    i2 = tile_image(w2, h1, h2, false);
    i3 = tile_image(w3, h2, 76, false);
    l1 = tile_image(w1, K, h1, true);
    l2 = tile_image(w2, h1, h2, true);
    l3 = tile_image(w3, h2, 76, true);
  }
  Packer pk;
  const size_t o_c = pk.add(cr.data(), cr.size() * 4);
  const size_t o_bw = pk.add(bary, (size_t)n_sub * 12);
  const size_t o_vs = pk.add(vslot.data(), vslot.size() * 4);
  const size_t o_uc = pk.add(ucr.data(), ucr.size() * 4);
  const size_t o_w1 = pk.add(w1, (size_t)K * h1 * 4);
  const size_t o_b1 = pk.add(b1, (size_t)h1 * 4);
  const size_t o_w2 = pk.add(w2, (size_t)h1 * h2 * 4);
  const size_t o_b2 = pk.add(b2, (size_t)h2 * 4);
  const size_t o_w3 = pk.add(w3, (size_t)h2 * 76 * 4);
  const size_t o_b3 = pk.add(b3, 76 * 4);
  const size_t o_m = pk.add(mask, 76 * 4);
  const size_t o_i1 = pk.add(i1.data(), i1.size() * 2);
  const size_t o_i2 = pk.add(i2.data(), i2.size() * 2);
  const size_t o_i3 = pk.add(i3.data(), i3.size() * 2);
  const size_t o_l1 = pk.add(l1.data(), l1.size() * 2);
  const size_t o_l2 = pk.add(l2.data(), l2.size() * 2);
  const size_t o_l3 = pk.add(l3.data(), l3.size() * 2);
  FSB_CUDA(c, c->m->proj_mem.alloc(pk.host.size()));
  FSB_CUDA(c, cudaMemcpy(c->m->proj_mem.p, pk.host.data(), pk.host.size(), cudaMemcpyHostToDevice));
  const unsigned char* base = static_cast<const unsigned char*>(c->m->proj_mem.p);
  ProjectorDev& p = c->m->proj;
  p.n_sub = n_sub;
  p.h1 = h1;
  p.h2 = h2;
  p.corners = reinterpret_cast<const int32_t*>(base + o_c);
  p.bw = reinterpret_cast<const float*>(base + o_bw);
  p.nu = (nu + 3) & ~3;  // mesh stride of the buffer a multiple of 16 bytes (staged with 16-byte loads)
  p.nvslot = (int)vslot.size();
  p.vslot = reinterpret_cast<const int32_t*>(base + o_vs);
  p.ucorners = reinterpret_cast<const int32_t*>(base + o_uc);
  p.w1 = reinterpret_cast<const float*>(base + o_w1);
  p.b1 = reinterpret_cast<const float*>(base + o_b1);
  p.w2 = reinterpret_cast<const float*>(base + o_w2);
  p.b2 = reinterpret_cast<const float*>(base + o_b2);
  p.w3 = reinterpret_cast<const float*>(base + o_w3);
  p.b3 = reinterpret_cast<const float*>(base + o_b3);
  p.mask = reinterpret_cast<const float*>(base + o_m);
  p.img_w1 = tc_ok ? base + o_i1 : nullptr;
  p.img_w2 = tc_ok ? base + o_i2 : nullptr;
  p.img_w3 = tc_ok ? base + o_i3 : nullptr;
  p.img_w1_lo = tc_ok ? base + o_l1 : nullptr;
  p.img_w2_lo = tc_ok ? base + o_l2 : nullptr;
  p.img_w3_lo = tc_ok ? base + o_l3 : nullptr;
  p.KT1 = (K + 127) / 128;
  p.KT2 = (h1 + 127) / 128;
  p.KT3 = (h2 + 127) / 128;
  c->m->has_proj = true;
  model_changed(c);
  return FSB_OK;
}

// ---------------------------------------------------------------------------
// stages

int fsb_boxes_crops(fsb_ctx* c, const float* images, int B, int H, int W, const float* kp, double alpha, int S,
                    double* boxes, float* prompt, float* crops, int32_t* taps, void* stream) {
  if (B < 0 || H < 2 || W < 2) return fail(c, FSB_ERR_SHAPE, "boxes_crops: bad image shape %dx%d", H, W);
  if (S < 2 || S > 512) return fail(c, FSB_ERR_USAGE, "out_size must be in [2, 512]");
  if (!(alpha > 0)) return fail(c, FSB_ERR_USAGE, "alpha must be positive");
  if (!boxes || !prompt) return fail(c, FSB_ERR_USAGE, "boxes and prompt outputs are required");
  bool host_frames = false;
  if (B > 0) {
    // frames and keypoints may live in HBM or in pinned (mapped) host memory;
    // pageable host memory is not reachable from the device
    for (int i = 0; i < 2; ++i) {
      cudaPointerAttributes at{};
      if (cudaPointerGetAttributes(&at, i ? (const void*)kp : (const void*)images) != cudaSuccess ||
          at.type == cudaMemoryTypeUnregistered) {
        cudaGetLastError();
        return fail(c, FSB_ERR_USAGE, "boxes_crops: frames/keypoints must be device or pinned host memory");
      }
      if (i == 0) host_frames = at.type == cudaMemoryTypeHost;
    }
  }
  FSB_CUDA(c, launch_boxes_crops(images, kp, B, H, W, S, alpha, host_frames, boxes, prompt, crops, taps, c->d_flag,
                                 c->d_bytes_in, (cudaStream_t)stream));
  c->launches += B > 0 ? (host_frames || B <= 2 ? 1 : 2) : 0;  // HBM frames from 3 on: k_frame_boxes + k_boxes_crops
  note_stream(c, (cudaStream_t)stream);
  return FSB_OK;
}

int fsb_bilinear(fsb_ctx* c, const float* image, int H, int W, int C, const float* grid, int64_t n, float* out,
                 void* stream) {
  if (H < 1 || W < 1 || C < 1 || n < 0) return fail(c, FSB_ERR_SHAPE, "bilinear: bad shapes");
  FSB_CUDA(c, launch_bilinear(image, H, W, C, grid, n, out, c->d_flag, (cudaStream_t)stream));
  c->launches += n > 0;
  note_stream(c, (cudaStream_t)stream);
  return FSB_OK;
}

int fsb_body_boxes(fsb_ctx* c, const float* kp, int n, int W, int H, double* out, void* stream) {
  if (n < 0 || W < 2 || H < 2) return fail(c, FSB_ERR_SHAPE, "body_boxes: bad shapes");
  FSB_CUDA(c, launch_body_boxes(kp, n, W, H, out, (cudaStream_t)stream));
  c->launches += n > 0;
  note_stream(c, (cudaStream_t)stream);
  return FSB_OK;
}

int fsb_hand_boxes(fsb_ctx* c, const double* wrists, const double* body, int n, double alpha, int W, int H,
                   double* out, void* stream) {
  if (!(alpha > 0)) return fail(c, FSB_ERR_USAGE, "alpha must be positive");
  FSB_CUDA(c, launch_hand_boxes(wrists, body, n, alpha, W, H, out, (cudaStream_t)stream));
  c->launches += n > 0;
  note_stream(c, (cudaStream_t)stream);
  return FSB_OK;
}

int fsb_crop_grid(fsb_ctx* c, const double* boxes, int n, int S, float* out, void* stream) {
  if (S < 2) return fail(c, FSB_ERR_USAGE, "out_size must be >= 2");
  FSB_CUDA(c, launch_crop_grid(boxes, n, S, out, (cudaStream_t)stream));
  c->launches += n > 0;
  note_stream(c, (cudaStream_t)stream);
  return FSB_OK;
}

int fsb_bridge(fsb_ctx* c, const float* v, int B, int nv, const int32_t* corners, const float* w, int nt, float* out,
               void* stream) {
  if (B < 0 || nv <= 0 || nt < 0) return fail(c, FSB_ERR_SHAPE, "bridge: bad shapes");
  FSB_CUDA(c, launch_bridge(v, B, nv, corners, w, nt, out, (cudaStream_t)stream));
  c->launches += (int64_t)B * nt > 0;
  note_stream(c, (cudaStream_t)stream);
  return FSB_OK;
}

int fsb_encode(fsb_ctx* c, const float* crops, int n, float* feats, int precision, void* stream) {
  if (!c->m->has_decoder) return fail(c, FSB_ERR_USAGE, "encode: no decoder loaded");
  c->kv_feats = nullptr;
  if (precision != FSB_FP32 && precision != FSB_BF16) return fail(c, FSB_ERR_USAGE, "encode: bad precision %d", precision);
  model_sync(c);
  if (c->m->vit && precision == FSB_FP32) {  // reference precision, any config (k_enc_f32.cu)
    if (n <= 0) return FSB_OK;
    constexpr int kF32Chunk = 64;
    const int want = n < kF32Chunk ? n : kF32Chunk;
    if (c->encf32_ws.max_crops < want) {
      if (capturing((cudaStream_t)stream))
        return fail(c, FSB_ERR_USAGE, "encode: encoder workspace for %d crops not allocated before graph capture", want);
      FSB_CUDA(c, cudaStreamSynchronize((cudaStream_t)stream));
      FSB_CUDA(c, c->encf32_ws_mem.alloc(enc_f32_ws_bytes(c->m->encw, want)));
      enc_f32_ws_carve(c->m->encw, want, c->encf32_ws_mem.p, &c->encf32_ws);
    }
    int nl = 0;
    FSB_CUDA(c, launch_enc_f32(c->m->encw, c->encf32_ws, crops, n, feats, c->d_flag, (cudaStream_t)stream, &nl));
    c->counters.encode += 1;
    c->counters.encoded_crops += n;
    c->launches += nl;
    note_stream(c, (cudaStream_t)stream);
    return FSB_OK;
  }
  if (c->m->vit) {
    if (!c->m->vit_tc)
      return fail(c, FSB_ERR_USAGE,
                  "encode: the bf16 tensor-core encoder needs dim %% 128 == 0 (<= 2048), head dim 64 and "
                  "patch*patch*3 %% 64 == 0; precision='fp32' runs any config");
    if (n <= 0) return FSB_OK;
    const int want = n < kVitChunk ? n : kVitChunk;
    if (c->vit_ws.max_crops < want) {
      if (capturing((cudaStream_t)stream))
        return fail(c, FSB_ERR_USAGE, "encode: encoder workspace for %d crops not allocated before graph capture", want);
      FSB_CUDA(c, cudaStreamSynchronize((cudaStream_t)stream));
      FSB_CUDA(c, c->vit_ws_mem.alloc(vit_ws_bytes(c->m->vitw, want)));
      vit_ws_carve(c->m->vitw, want, c->vit_ws_mem.p, &c->vit_ws);
    }
    int nl = 0;
    FSB_CUDA(c, launch_vit_encoder(c->m->vitw, c->vit_ws, crops, n, feats, c->d_flag, (cudaStream_t)stream, &nl));
    c->counters.encode += 1;
    c->counters.encoded_crops += n;
    c->launches += nl;
    note_stream(c, (cudaStream_t)stream);
    return FSB_OK;
  }
  if (!default_model(c->m->cfg))
    return fail(c, FSB_ERR_USAGE, "encode: the fused fp32 encoder supports the default DecoderConfig only");
  if (precision == FSB_BF16)
    FSB_CUDA(c, launch_encoder_tc(crops, n, c->m->enc, feats, c->d_flag, KvArgs{}, (cudaStream_t)stream));
  else
    FSB_CUDA(c, launch_encoder_f32(crops, n, c->m->enc, feats, c->d_flag, (cudaStream_t)stream));
  c->counters.encode += 1;
  c->counters.encoded_crops += n;
  c->launches += n > 0;
  note_stream(c, (cudaStream_t)stream);
  return FSB_OK;
}

// K / V projection arguments for a decode of `a` (crop mapping as DecodeArgs)
static KvArgs kv_args(fsb_ctx* c, const DecodeArgs& a, int mode) {
  KvArgs kv{};
  kv.mode = mode;
  kv.nbody = a.nbody;
  kv.nhand = a.nhand;
  kv.body_feat_stride = a.body_feat_stride;
  kv.hand_feat_first = a.hand_feat_first;
  kv.feats_in = a.feats;
  kv.body_kv = c->w_bkv;
  kv.hand_kv = c->w_hkv;
  kv.tcs[0] = c->m->kv_tcs[mode - 1][0];
  kv.tcs[1] = c->m->kv_tcs[mode - 1][1];
  kv.layers[0] = c->m->cfg.body_layers;
  kv.layers[1] = c->m->cfg.hand_layers;
  return kv;
}

static int decode_common(fsb_ctx* c, DecodeArgs& a, int precision, cudaStream_t st) {
  if (!c->m->has_decoder) return fail(c, FSB_ERR_USAGE, "decode: no decoder loaded");
  if (a.nbody > 0 && !c->m->has_tmpl[FSB_SMPL])
    return fail(c, FSB_ERR_USAGE, "decode: the body decoder needs its template (fsb_load_template SMPL)");
  if (precision != FSB_FP32 && precision != FSB_BF16) return fail(c, FSB_ERR_USAGE, "decode: bad precision %d", precision);
  if (!default_model(c->m->cfg))
    return fail(c, FSB_ERR_USAGE, "decode: the fused fp32 decoders support the default DecoderConfig only");
  if ((a.body_sel >> c->m->cfg.body_layers) != 0u || (a.hand_sel >> c->m->cfg.hand_layers) != 0u)
    return fail(c, FSB_ERR_USAGE, "selection out of range");
  a.nonfinite = c->d_flag;
  if (precision == FSB_BF16 && a.body_kv == nullptr) {
    // the bf16 decoders read the cross-attention K / V projected ahead:
    // project them from the given features (k_encoder_tc mode 2)
    const int frames = a.nbody > (a.nhand + 1) / 2 ? a.nbody : (a.nhand + 1) / 2;
    int rc = ensure_ws(c, frames, st);
    if (rc) return rc;
    FSB_CUDA(c, launch_encoder_tc(nullptr, 0, c->m->enc, nullptr, c->d_flag, kv_args(c, a, 2), st));
    c->launches += (a.nbody + a.nhand) > 0;
    a.body_kv = c->w_bkv;
    a.hand_kv = c->w_hkv;
    c->kv_feats = nullptr;
  }
  if (precision == FSB_BF16)
    FSB_CUDA(c, launch_decoders_tc(a, c->m->body, c->m->hand, st));
  else
    FSB_CUDA(c, launch_decoders_f32(a, c->m->body, c->m->hand, st));
  c->launches += (a.nbody + a.nhand) > 0;
  const int nb = layer_count(a.body_sel);
  c->counters.fk += (int64_t)a.nbody * nb + (int64_t)a.nhand * layer_count(a.hand_sel);
  c->counters.project += (int64_t)a.nbody * nb + (int64_t)a.nhand * layer_count(a.hand_sel);
  c->counters.intermediate += (int64_t)a.nbody * nb;
  note_stream(c, st);
  return FSB_OK;
}

int fsb_decode_body(fsb_ctx* c, const float* feats, int B, int feat_stride, const float* prompts, uint32_t sel,
                    float* params, float* cam, float* inter, int precision, void* stream) {
  DecodeArgs a{};
  a.feats = feats;
  a.prompts = prompts;
  a.nbody = B;
  a.nhand = 0;
  a.body_feat_stride = feat_stride;
  a.body_sel = sel;
  a.body_params = params;
  a.body_cam = cam;
  a.inter = inter;
  return decode_common(c, a, precision, (cudaStream_t)stream);
}

int fsb_decode_hands(fsb_ctx* c, const float* feats, int n, uint32_t sel, float* rots, int precision, void* stream) {
  DecodeArgs a{};
  a.feats = feats;
  a.nbody = 0;
  a.nhand = n;
  a.body_feat_stride = 2;
  a.hand_feat_first = 0;
  a.hand_sel = sel;
  a.hand_rots = rots;
  return decode_common(c, a, precision, (cudaStream_t)stream);
}

int fsb_encode_frames(fsb_ctx* c, const float* crops, int B, float* feats, int precision, void* stream) {
  if (precision != FSB_BF16 || c->m->vit || !c->m->has_decoder || !default_model(c->m->cfg))
    return fsb_encode(c, crops, 3 * B, feats, precision, stream);
  cudaStream_t st = (cudaStream_t)stream;
  int rc = ensure_ws(c, B, st);
  if (rc) return rc;
  // encoder + every decoder layer's cross-attention K / V in one launch
  // (k_encoder_tc mode 1)
  DecodeArgs a{};
  a.feats = feats;
  a.nbody = B;
  a.nhand = 2 * B;
  a.body_feat_stride = 3;
  a.hand_feat_first = 1;
  FSB_CUDA(c, launch_encoder_tc(crops, 3 * B, c->m->enc, feats, c->d_flag, kv_args(c, a, 1), st));
  c->counters.encode += 1;
  c->counters.encoded_crops += 3 * B;
  c->launches += B > 0;
  c->kv_feats = feats;
  c->kv_frames = B;
  note_stream(c, st);
  return FSB_OK;
}

int fsb_decode_frames(fsb_ctx* c, const float* feats, int B, const float* prompts, uint32_t body_sel,
                      uint32_t hand_sel, float* params, float* cam, float* rots, float* merged, int precision,
                      void* stream) {
  DecodeArgs a{};
  if (precision == FSB_BF16 && c->kv_feats == feats && c->kv_frames == B && feats != nullptr) {
    a.body_kv = c->w_bkv;  // projected by fsb_encode_frames
    a.hand_kv = c->w_hkv;
  }
  a.feats = feats;
  a.prompts = prompts;
  a.nbody = B;
  a.nhand = 2 * B;
  a.body_feat_stride = 3;
  a.hand_feat_first = 1;
  a.body_sel = body_sel;
  a.hand_sel = hand_sel;
  a.body_params = params;
  a.body_cam = cam;
  a.hand_rots = rots;
  a.merged = merged;
  return decode_common(c, a, precision, (cudaStream_t)stream);
}

int fsb_fk(fsb_ctx* c, int which, const float* poses, int B, float* joints, float* rel, void* stream) {
  if (which != FSB_MHR && which != FSB_SMPL) return fail(c, FSB_ERR_USAGE, "bad template id");
  if (!c->m->has_tmpl[which]) return fail(c, FSB_ERR_USAGE, "fk: template %d not loaded", which);
  FSB_CUDA(c, launch_fk(poses, FSB_PARAM_DIM, B, c->m->tmpl[which].joints_rest, joints, rel, (cudaStream_t)stream));
  c->launches += B > 0;
  note_stream(c, (cudaStream_t)stream);
  return FSB_OK;
}

// FK (rel transforms + the k_lbs_tc chunk records) then LBS.  FSB_LBS_SIMT=1
// selects the all-CUDA-core k_lbs (measured alternative).
static bool lbs_simt() {
  static const bool v = getenv("FSB_LBS_SIMT") != nullptr;
  return v;
}

static int fk_lbs(fsb_ctx* c, int which, const float* poses, int B, float* rel, uint8_t* lbsin, float* joints,
                  float* verts, cudaStream_t st, const DenoiseW* dn = nullptr, CornerOut cu = CornerOut()) {
  const TemplateDev& t = c->m->tmpl[which];
  const bool tc = verts != nullptr && !lbs_simt();
  FSB_CUDA(c, launch_fk(poses, FSB_PARAM_DIM, B, t.joints_rest, joints, rel, st, tc ? lbsin : nullptr, dn, c->d_flag));
  c->launches += B > 0;
  if (verts == nullptr) return FSB_OK;
  if (tc)
    FSB_CUDA(c, launch_lbs_tc(t, lbsin, B, verts, c->d_flag, st, cu));
  else
    FSB_CUDA(c, launch_lbs(t, rel, poses, FSB_PARAM_DIM, B, verts, c->d_flag, st));
  c->launches += B > 0;
  return FSB_OK;
}

int fsb_skin(fsb_ctx* c, int which, const float* poses, int B, float* verts, void* stream) {
  if (which != FSB_MHR && which != FSB_SMPL) return fail(c, FSB_ERR_USAGE, "bad template id");
  if (!c->m->has_tmpl[which]) return fail(c, FSB_ERR_USAGE, "skin: template %d not loaded", which);
  cudaStream_t st = (cudaStream_t)stream;
  int rc = ensure_ws(c, B, st);
  if (rc) return rc;
  rc = fk_lbs(c, which, poses, B, c->w_rel, c->w_lbsin, nullptr, verts, st);
  if (rc) return rc;
  note_stream(c, (cudaStream_t)stream);
  return FSB_OK;
}

// K tiles per reduction group of the tensor-core projector layers; fixed, so
// the K partition (and the bits of a mesh's output) never depend on B
constexpr int kMlpGroup = 4;

static bool mlp_tc(const fsb_ctx* c, int precision) { return precision == FSB_BF16 && c->m->proj.img_w1 != nullptr; }
// fp32 mode on the tensor cores: every product as hi.hi + hi.lo + lo.hi of
// bf16 halves (x = hi + lo, hi = bf16(x), lo = bf16(x - hi)), fp32
// accumulation; FSB_MLP_SIMT=1 keeps the CUDA-core fp32 GEMM
static bool mlp_split(const fsb_ctx* c, int precision) {
  static const bool simt = getenv("FSB_MLP_SIMT") != nullptr;
  return precision == FSB_FP32 && c->m->proj.img_w1_lo != nullptr && !simt;
}

static int run_mlp(fsb_ctx* c, int B, float* theta, int precision, cudaStream_t st, bool split) {
  const ProjectorDev& p = c->m->proj;
  if (split) {
    // the three split-bf16 GEMMs of a layer fill three slices of the split-K
    // partials; the reduce adds all of them in a fixed order and writes the
    // next layer's hi and lo images
    const uint8_t* ximg = reinterpret_cast<const uint8_t*>(c->w_xb);
    FSB_CUDA(c, launch_tile_layer(ximg, p.img_w1, p.KT1, kMlpGroup, B, p.h1, c->w_part, p.b1, nullptr, 1, nullptr, 0,
                                  c->w_h1img, p.KT2, nullptr, st, c->w_xbl, p.img_w1_lo, c->w_h1l));
    FSB_CUDA(c, launch_tile_layer(c->w_h1img, p.img_w2, p.KT2, kMlpGroup, B, p.h2, c->w_part, p.b2, nullptr, 1,
                                  nullptr, 0, c->w_h2img, p.KT3, nullptr, st, c->w_h1l, p.img_w2_lo, c->w_h2l));
    FSB_CUDA(c, launch_tile_layer(c->w_h2img, p.img_w3, p.KT3, kMlpGroup, B, FSB_PARAM_DIM, c->w_part, p.b3, p.mask,
                                  0, theta, FSB_PARAM_DIM, nullptr, 0, c->d_flag, st, c->w_h2l, p.img_w3_lo,
                                  nullptr));
    c->launches += 12;
    return FSB_OK;
  }
  if (mlp_tc(c, precision)) {
    // relu(x W1 + b1) -> relu(h1 W2 + b2) -> (h2 W3 + b3) * mask on tcgen05;
    // each reduce writes the next layer's bf16 A-tile image
    const uint8_t* ximg = reinterpret_cast<const uint8_t*>(c->w_xb);
    FSB_CUDA(c, launch_tile_layer(ximg, p.img_w1, p.KT1, kMlpGroup, B, p.h1, c->w_part, p.b1, nullptr, 1, nullptr, 0,
                                  c->w_h1img, p.KT2, nullptr, st));
    FSB_CUDA(c, launch_tile_layer(c->w_h1img, p.img_w2, p.KT2, kMlpGroup, B, p.h2, c->w_part, p.b2, nullptr, 1,
                                  nullptr, 0, c->w_h2img, p.KT3, nullptr, st));
    FSB_CUDA(c, launch_tile_layer(c->w_h2img, p.img_w3, p.KT3, kMlpGroup, B, FSB_PARAM_DIM, c->w_part, p.b3, p.mask,
                                  0, theta, FSB_PARAM_DIM, nullptr, 0, c->d_flag, st));
    c->launches += 6;
    return FSB_OK;
  }
  FSB_CUDA(c, launch_gemm_f32(c->w_x, 3 * p.n_sub, p.w1, p.b1, nullptr, c->w_h1, p.h1, B, p.h1, 3 * p.n_sub, 1,
                              nullptr, c->w_part, st));
  FSB_CUDA(c, launch_gemm_f32(c->w_h1, p.h1, p.w2, p.b2, nullptr, c->w_h2, p.h2, B, p.h2, p.h1, 1, nullptr,
                              c->w_part, st));
  FSB_CUDA(c, launch_gemm_f32(c->w_h2, p.h2, p.w3, p.b3, p.mask, theta, FSB_PARAM_DIM, B, FSB_PARAM_DIM, p.h2, 0,
                              c->d_flag, c->w_part, st));
  c->launches += 3 + (gemm_f32_splits(3 * p.n_sub) > 1) + (gemm_f32_splits(p.h1) > 1) + (gemm_f32_splits(p.h2) > 1);
  return FSB_OK;
}

int fsb_project_vertices(fsb_ctx* c, const float* v_mhr, int B, int nv, float* theta, int precision,
                         void* stream) {
  if (!c->m->has_proj) return fail(c, FSB_ERR_USAGE, "project: no projector loaded");
  if (nv <= 0) return fail(c, FSB_ERR_SHAPE, "project: bad vertex count");
  cudaStream_t st = (cudaStream_t)stream;
  int rc = ensure_ws(c, B, st);
  if (rc) return rc;
  const bool tc = mlp_tc(c, precision), split = mlp_split(c, precision), img = tc || split;
  FSB_CUDA(c, launch_proj_inputs_v(v_mhr, nv, c->m->proj, B, c->w_x, !img, img ? c->w_xb : nullptr, c->w_psum, st,
                                   false, split ? reinterpret_cast<__nv_bfloat16*>(c->w_xbl) : nullptr));
  c->launches += B > 0;  // bridge + centre in one kernel
  if (tc && proj_fused_ok(c->m->proj) && proj_fused_on()) {  // the MLP in one launch
    FSB_CUDA(c, launch_proj_fused(reinterpret_cast<const uint8_t*>(c->w_xb), c->m->proj, B, theta, nullptr, nullptr,
                                  nullptr, c->d_flag, st));
    c->launches += B > 0;
    note_stream(c, st);
    return FSB_OK;
  }
  rc = run_mlp(c, B, theta, precision, st, split);
  if (rc == FSB_OK) note_stream(c, st);
  return rc;
}

static int skin_project_impl(fsb_ctx* c, const float* params, int B, float* v_mhr, float* theta, float* j_smpl,
                             float* v_smpl, int precision, cudaStream_t st) {
  if (!c->m->has_proj || !c->m->has_tmpl[FSB_MHR] || !c->m->has_tmpl[FSB_SMPL])
    return fail(c, FSB_ERR_USAGE, "skin_project: projector or templates missing");
  const TemplateDev& mhr = c->m->tmpl[FSB_MHR];
  const ProjectorDev& pj = c->m->proj;
  const bool bridge = v_mhr && getenv("FSB_PROJ_RESKIN") == nullptr;
  // the LBS kernel also writes the projector's corner vertices compacted
  // (tensor-core LBS only; FSB_PROJ_SCATTER=1 bridges from V_mhr's rows)
  CornerOut cu;
  if (bridge && !lbs_simt() && pj.nvslot <= mhr.nv && getenv("FSB_PROJ_SCATTER") == nullptr) {
    cu.vu = c->w_vu;
    cu.vslot = pj.vslot;
    cu.nvslot = pj.nvslot;
    cu.nu = pj.nu;
  }
  int rc = fk_lbs(c, FSB_MHR, params, B, c->w_rel, c->w_lbsin, nullptr, v_mhr, st, nullptr, cu);
  if (rc) return rc;
  const bool tc = mlp_tc(c, precision);
  // fp32 mode's split-bf16 MLP takes its inputs from the bridge kernel (the
  // re-skin path without V_mhr keeps the CUDA-core fp32 GEMMs)
  const bool split = bridge && mlp_split(c, precision), img = tc || split;
  __nv_bfloat16* xbl = split ? reinterpret_cast<__nv_bfloat16*>(c->w_xbl) : nullptr;
  if (bridge) {
    // V_mhr was just written: bridge its corner vertices (what the reference
    // projects, projection.py:447-465) instead of re-skinning them -- from
    // the compacted corner buffer when the LBS kernel filled it
    if (cu.vu)
      FSB_CUDA(c, launch_proj_inputs_v(cu.vu, pj.nu, pj, B, c->w_x, !img, img ? c->w_xb : nullptr, c->w_psum, st,
                                       true, xbl));
    else
      FSB_CUDA(c, launch_proj_inputs_v(v_mhr, mhr.nv, pj, B, c->w_x, !img, img ? c->w_xb : nullptr, c->w_psum, st,
                                       false, xbl));
    c->launches += 1;  // bridge + centre
  } else {
    FSB_CUDA(c, launch_proj_inputs(mhr, c->m->proj, c->w_rel, params, FSB_PARAM_DIM, B, c->w_x, !tc,
                                   tc ? c->w_xb : nullptr, c->w_psum, st));
    c->launches += 2;  // re-skinned inputs, centre
  }
  const DenoiseW* dn = c->m->dn.H > 0 ? &c->m->dn : nullptr;
  if (tc && v_smpl == nullptr && proj_fused_ok(c->m->proj) && proj_fused_on()) {
    // MLP (3 layers, mask), denoiser and SMPL FK in one cluster launch (k_mlp_tc.cu)
    FSB_CUDA(c, launch_proj_fused(reinterpret_cast<const uint8_t*>(c->w_xb), c->m->proj, B, theta,
                                  c->m->tmpl[FSB_SMPL].joints_rest, j_smpl, dn, c->d_flag, st));
    c->launches += B > 0;
    return FSB_OK;
  }
  rc = run_mlp(c, B, theta, precision, st, split);
  if (rc) return rc;
  // SMPL FK (+ the denoiser epilogue on theta[3:66] when one is loaded)
  return fk_lbs(c, FSB_SMPL, theta, B, v_smpl ? c->w_rel2 : nullptr, c->w_lbsin2, j_smpl, v_smpl, st, dn);
}

int fsb_skin_project(fsb_ctx* c, const float* params, int B, float* v_mhr, float* theta, float* j_smpl,
                     float* v_smpl, int precision, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  int rc = ensure_ws(c, B, st);
  if (rc) return rc;
  rc = skin_project_impl(c, params, B, v_mhr, theta, j_smpl, v_smpl, precision, st);
  if (rc == FSB_OK) note_stream(c, st);
  return rc;
}

static int frame_batch_launches(fsb_ctx* c, const float* images, int B, int H, int W, const float* kp, double alpha,
                                uint32_t bsel, uint32_t hsel, int precision, const fsb_frame_outputs& o,
                                cudaStream_t st) {
  const int S = c->m->cfg.crop_size;
  double* boxes = o.boxes ? o.boxes : c->w_boxes;
  float* prompt = o.prompt ? o.prompt : c->w_prompt;
  float* crops = o.crops ? o.crops : c->w_crops;
  float* feats = o.feats ? o.feats : c->w_feats;
  float* params = o.body_params ? o.body_params : c->w_params;
  float* cam = o.body_cam ? o.body_cam : c->w_cam;
  float* rots = o.hand_rots ? o.hand_rots : c->w_rots;
  int rc = fsb_boxes_crops(c, images, B, H, W, kp, alpha, S, boxes, prompt, crops, nullptr, st);
  if (rc) return rc;
  rc = fsb_encode_frames(c, crops, B, feats, precision, st);
  if (rc) return rc;
  rc = fsb_decode_frames(c, feats, B, prompt, bsel, hsel, params, cam, rots, o.merged, precision, st);
  if (rc || !o.theta) return rc;  // front half only (Pipeline.run without the SMPL tail)
  return skin_project_impl(c, o.merged, B, o.v_mhr, o.theta, o.j_smpl, o.v_smpl, precision, st);
}

int fsb_frame_batch(fsb_ctx* c, const float* images, int B, int H, int W, const float* kp, double alpha,
                    uint32_t body_sel, uint32_t hand_sel, int precision, const fsb_frame_outputs* out,
                    void* stream) {
  if (!out || !out->merged || (!out->theta) != (!out->j_smpl))
    return fail(c, FSB_ERR_USAGE, "frame_batch: merged is required, theta and j_smpl together or neither");
  const bool tail = out->theta != nullptr;
  if (!c->m->has_decoder || !c->m->has_tmpl[FSB_SMPL] || (tail && (!c->m->has_proj || !c->m->has_tmpl[FSB_MHR])))
    return fail(c, FSB_ERR_USAGE, "frame_batch: decoder and SMPL template (and for the tail: MHR template and "
                                  "projector) must be loaded");
  if (!tail && (out->v_mhr || out->v_smpl))
    return fail(c, FSB_ERR_USAGE, "frame_batch: v_mhr / v_smpl need the SMPL tail outputs");
  if (B <= 0) return FSB_OK;
  cudaStream_t st = (cudaStream_t)stream;
  int rc = ensure_ws(c, B, st);
  if (rc) return rc;
  const bool use_graph = c->graphs && st != nullptr && !capturing(st);
  if (!use_graph) return frame_batch_launches(c, images, B, H, W, kp, alpha, body_sel, hand_sel, precision, *out, st);
  GraphKey k{};
  k.B = B;
  k.H = H;
  k.W = W;
  k.precision = precision;
  k.bsel = body_sel;
  k.hsel = hand_sel;
  k.alpha = alpha;
  const void* ptrs[16] = {images, kp, out->boxes, out->prompt, out->crops, out->feats, out->body_params,
                          out->body_cam, out->hand_rots, out->merged, out->v_mhr, out->theta, out->j_smpl,
                          out->v_smpl, nullptr, nullptr};
  memcpy(k.ptrs, ptrs, sizeof ptrs);
  k.stream = st;
  fsb_ctx::GraphEntry* hit = nullptr;
  for (auto& e : c->gcache)
    if (e.key == k) hit = &e;
  if (!hit) {
    constexpr size_t kMaxGraphs = 32;
    if (c->gcache.size() >= kMaxGraphs) {
      size_t lru = 0;
      for (size_t i = 1; i < c->gcache.size(); ++i)
        if (c->gcache[i].used < c->gcache[lru].used) lru = i;
      cudaGraphExecDestroy(c->gcache[lru].exec);
      c->gcache.erase(c->gcache.begin() + lru);
    }
    const fsb_counters_t saved = c->counters;
    const int64_t saved_l = c->launches;
    FSB_CUDA(c, cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
    rc = frame_batch_launches(c, images, B, H, W, kp, alpha, body_sel, hand_sel, precision, *out, st);
    cudaGraph_t g = nullptr;
    cudaError_t ce = cudaStreamEndCapture(st, &g);
    c->counters = saved;
    c->launches = saved_l;
    if (rc) {
      if (g) cudaGraphDestroy(g);
      return rc;
    }
    if (ce != cudaSuccess) return fail(c, FSB_ERR_CUDA, "graph capture: %s", cudaGetErrorString(ce));
    size_t nn = 0;
    cudaGraphGetNodes(g, nullptr, &nn);
    cudaGraphExec_t ex = nullptr;
    ce = cudaGraphInstantiate(&ex, g, 0);
    cudaGraphDestroy(g);
    if (ce != cudaSuccess) return fail(c, FSB_ERR_CUDA, "graph instantiate: %s", cudaGetErrorString(ce));
    c->gcache.push_back({k, ex, (int)nn, 0});
    hit = &c->gcache.back();
  }
  hit->used = ++c->gclock;
  FSB_CUDA(c, cudaGraphLaunch(hit->exec, st));
  c->launches += hit->nodes;
  c->counters.encode += 1;
  c->counters.encoded_crops += 3 * B;
  const int nb = layer_count(body_sel), nh = layer_count(hand_sel);
  c->counters.fk += (int64_t)B * (nb + 2 * nh);
  c->counters.project += (int64_t)B * (nb + 2 * nh);
  c->counters.intermediate += (int64_t)B * nb;
  note_stream(c, (cudaStream_t)stream);
  return FSB_OK;
}

int fsb_fit_batch(fsb_ctx* c, const float* target, int B, int nv, const float* init, int steps, double lr,
                  float lambda_pose, float lambda_shape, float* scratch, float* best_params, double* vertex_error,
                  double* err_curve, float* grad0, void* stream) {
  if (!c->m->has_tmpl[FSB_SMPL]) return fail(c, FSB_ERR_USAGE, "fit_batch: no target template loaded (FSB_SMPL slot)");
  const TemplateDev& t = c->m->tmpl[FSB_SMPL];
  if (B < 0 || nv != t.nv) return fail(c, FSB_ERR_SHAPE, "fit_batch: targets have %d vertices, template %d", nv, t.nv);
  if (steps < 1) return fail(c, FSB_ERR_USAGE, "FitConfig.steps must be at least 1");
  if (!scratch || !best_params || !vertex_error || !err_curve)
    return fail(c, FSB_ERR_USAGE, "fit_batch: scratch and outputs are required");
  FSB_CUDA(c, launch_fit(t, target, B, init, steps, lr, lambda_pose, lambda_shape, scratch, best_params, vertex_error,
                         err_curve, grad0, c->d_flag, (cudaStream_t)stream));
  c->launches += B > 0;
  note_stream(c, (cudaStream_t)stream);
  return FSB_OK;
}

int fsb_bary_map(fsb_ctx* c, const double* src_verts, int nv, const int64_t* src_faces, int F, const double* tgt_verts,
                 int nt, uint8_t* degenerate, int64_t* face_index, float* weights, void* stream) {
  if (nv <= 0 || F <= 0 || nt < 0) return fail(c, FSB_ERR_SHAPE, "bary_map: bad shapes");
  if (!degenerate || !face_index || !weights) return fail(c, FSB_ERR_USAGE, "bary_map: outputs are required");
  FSB_CUDA(c, launch_bary(src_verts, src_faces, F, tgt_verts, nt, degenerate, face_index, weights,
                          (cudaStream_t)stream));
  c->launches += 2 * (nt > 0);
  note_stream(c, (cudaStream_t)stream);
  return FSB_OK;
}

int fsb_load_denoiser(fsb_ctx* c, const float* w1, const float* b1, const float* w2, const float* b2, int hidden) {
  if (hidden == 0 || w1 == nullptr) {  // remove
    c->m->dn = DenoiseW{nullptr, nullptr, nullptr, nullptr, 0};
    c->m->dn_mem.release();
    model_changed(c);
    return FSB_OK;
  }
  if (hidden < 0 || hidden > FSB_DN_MAX_HIDDEN)
    return fail(c, FSB_ERR_USAGE, "denoiser: hidden width %d not in [1, %d]", hidden, FSB_DN_MAX_HIDDEN);
  if (!b1 || !w2 || !b2) return fail(c, FSB_ERR_USAGE, "denoiser: null weight");
  const size_t n1 = (size_t)FSB_DN_IN * hidden, n2 = (size_t)hidden * FSB_DN_IN;
  const size_t tot = n1 + hidden + n2 + FSB_DN_IN;
  std::vector<float> h(tot);
  memcpy(h.data(), w1, n1 * 4);
  memcpy(h.data() + n1, b1, (size_t)hidden * 4);
  memcpy(h.data() + n1 + hidden, w2, n2 * 4);
  memcpy(h.data() + n1 + hidden + n2, b2, FSB_DN_IN * 4);
  FSB_CUDA(c, c->m->dn_mem.alloc(tot * 4));
  FSB_CUDA(c, cudaMemcpy(c->m->dn_mem.p, h.data(), tot * 4, cudaMemcpyHostToDevice));
  const float* d = static_cast<const float*>(c->m->dn_mem.p);
  c->m->dn = DenoiseW{d, d + n1, d + n1 + hidden, d + n1 + hidden + n2, hidden};
  model_changed(c);
  return FSB_OK;
}

int fsb_denoise(fsb_ctx* c, const float* poses, int B, const float* w1, const float* b1, const float* w2,
                const float* b2, int hidden, float* out, void* stream) {
  if (B < 0) return fail(c, FSB_ERR_SHAPE, "denoise: negative batch");
  if (hidden <= 0 || hidden > 128) return fail(c, FSB_ERR_USAGE, "denoise: hidden width %d not in [1, 128]", hidden);
  FSB_CUDA(c, launch_denoise(poses, B, w1, b1, w2, b2, hidden, out, c->d_flag, (cudaStream_t)stream));
  c->launches += B > 0;
  note_stream(c, (cudaStream_t)stream);
  return FSB_OK;
}

int fsb_render(fsb_ctx* c, const void* scenes, int B, int H, int W, float* out, void* stream) {
  if (B < 0 || H < 1 || W < 1) return fail(c, FSB_ERR_SHAPE, "render: bad shapes");
  FSB_CUDA(c, launch_render(scenes, B, H, W, out, (cudaStream_t)stream));
  c->launches += B > 0;
  note_stream(c, (cudaStream_t)stream);
  return FSB_OK;
}

int fsb_nonfinite(fsb_ctx* c, int* flag, int reset) {
  FSB_CUDA(c, wait_own_work(c));
  FSB_CUDA(c, cudaMemcpyAsync(c->h_flag, c->d_flag, sizeof(int), cudaMemcpyDeviceToHost, c->aux));
  if (reset) FSB_CUDA(c, cudaMemsetAsync(c->d_flag, 0, sizeof(int), c->aux));
  FSB_CUDA(c, cudaStreamSynchronize(c->aux));
  if (flag) *flag = *c->h_flag;
  return FSB_OK;
}

int fsb_nonfinite_enqueue(fsb_ctx* c, int* host_dst, int reset, void* stream) {
  if (!c || !host_dst) return FSB_ERR_USAGE;
  cudaStream_t st = (cudaStream_t)stream;
  FSB_CUDA(c, cudaMemcpyAsync(host_dst, c->d_flag, sizeof(int), cudaMemcpyDeviceToHost, st));
  if (reset) FSB_CUDA(c, cudaMemsetAsync(c->d_flag, 0, sizeof(int), st));
  return FSB_OK;
}

int fsb_input_bytes(fsb_ctx* c, int64_t* total, int reset) {
  if (!c || !total) return FSB_ERR_USAGE;
  FSB_CUDA(c, wait_own_work(c));
  FSB_CUDA(c, cudaMemcpyAsync(c->h_bytes, c->d_bytes_in, sizeof *c->h_bytes, cudaMemcpyDeviceToHost, c->aux));
  if (reset) FSB_CUDA(c, cudaMemsetAsync(c->d_bytes_in, 0, sizeof *c->h_bytes, c->aux));
  FSB_CUDA(c, cudaStreamSynchronize(c->aux));
  *total = (int64_t)*c->h_bytes;
  return FSB_OK;
}

int fsb_counters(const fsb_ctx* c, fsb_counters_t* out) {
  if (!c || !out) return FSB_ERR_USAGE;
  *out = c->counters;
  return FSB_OK;
}

int64_t fsb_kernel_launches(const fsb_ctx* c) { return c ? c->launches : 0; }

}  // extern "C"

cudaError_t launch_tc_selftest(const void* A, const void* Bpacked, int N, int K, float* C, cudaStream_t st);

extern "C" int fsb_selftest_umma(fsb_ctx* c, const void* A, const void* Bpacked, int N, int K, float* C,
                                 void* stream) {
  FSB_CUDA(c, launch_tc_selftest(A, Bpacked, N, K, C, (cudaStream_t)stream));
  c->launches += 1;
  return FSB_OK;
}
