/*
 * fsb_b200.h — C ABI of the B200 (sm_100a) implementation of the Fast SAM
 * 3D Body accelerated inference path (crop -> encode -> pruned decode ->
 * MHR LBS -> MHR->SMPL projector -> SMPL FK).
 *
 * The reference (arxiv/paper_2603_15603, package `fsb`) has no FFI layer: its
 * boundary is the Python API.  Each entry point below replaces the reference
 * function named in its comment (paths relative to pkg/src/fsb/); the Python
 * package paper_2603_15603_b200 binds them with ctypes and keeps the
 * reference signatures on top.
 *
 * Conventions
 *   - All tensor arguments are DEVICE pointers (float32 C-contiguous unless
 *     stated), `stream` is a cudaStream_t passed as void*.  Calls are
 *     asynchronous on that stream.  Nothing is freed across the boundary.
 *   - One fsb_ctx per (GPU, host thread).  A context is not thread-safe
 *     (one pipeline instance per thread).
 *   - Return codes mirror the reference exception classes
 *     (numkit.py:33-42): FSB_ERR_SHAPE -> ShapeError, FSB_ERR_NUMERIC ->
 *     NumericError (device non-finite flag), FSB_ERR_USAGE -> UsageError,
 *     FSB_ERR_CUDA -> CUDA runtime failure.  fsb_last_error() gives text.
 *   - precision: FSB_FP32 (parity mode, <= 1e-4 relative vs the CPU
 *     oracle) or FSB_BF16 (tensor-core mode, bf16 operands / fp32
 *     accumulate; LN, softmax, residuals, heads and FK stay fp32).
 */
#ifndef FSB_B200_H
#define FSB_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FSB_OK 0
#define FSB_ERR_SHAPE 1
#define FSB_ERR_NUMERIC 2
#define FSB_ERR_USAGE 3
#define FSB_ERR_CUDA 4

#define FSB_FP32 0
#define FSB_BF16 1

#define FSB_MHR 0
#define FSB_SMPL 1

typedef struct fsb_ctx fsb_ctx;

/* decoder.DecoderConfig (decoder.py:42-50) */
typedef struct {
  int crop_size, patch, dim, heads, enc_layers, body_layers, hand_layers;
} fsb_decoder_config;

/* cumulative stage counters, the reference's counters dict (decoder.py:69-71) */
typedef struct {
  int64_t encode, encoded_crops, fk, project, intermediate;
} fsb_counters_t;

/* per-frame outputs of fsb_frame_batch; nullable fields use ctx workspace */
typedef struct {
  double* boxes;       /* (B, 3, 4) f64: body, left hand, right hand */
  float* prompt;       /* (B, 8) */
  float* crops;        /* (B, 3, S, S, 3) */
  float* feats;        /* (B, 3, T, D) */
  float* body_params;  /* (B, 76) */
  float* body_cam;     /* (B, 3) */
  float* hand_rots;    /* (B, 2, 3) */
  float* merged;       /* (B, 76)  required */
  float* v_mhr;        /* (B, Nv_mhr, 3) */
  float* theta;        /* (B, 76)  required */
  float* j_smpl;       /* (B, 22, 3) required */
  float* v_smpl;       /* (B, Nv_smpl, 3) */
} fsb_frame_outputs;

/* ---- lifetime ---------------------------------------------------------- */
int fsb_ctx_create(int device, fsb_ctx** out);
/* a second context on model_owner's GPU that shares its uploaded model
 * (decoder weights, templates, projector: one device copy) but owns its
 * workspace, graphs, flags and counters -- one per in-flight stream
 * (pipelines are per thread, the frozen model is not mutated).
 * An upload through any sharing context is seen by all of them. */
int fsb_ctx_create_shared(fsb_ctx* model_owner, fsb_ctx** out);
void fsb_ctx_destroy(fsb_ctx* ctx);
const char* fsb_last_error(const fsb_ctx* ctx);
const char* fsb_build_info(void);
/* preallocate workspace for up to max_frames frames per call (call before
 * graph capture); 0 on success */
int fsb_reserve(fsb_ctx* ctx, int max_frames);
/* enable/disable CUDA-graph replay inside fsb_frame_batch (default on) */
int fsb_set_graphs(fsb_ctx* ctx, int enabled);

/* ---- model upload (host pointers; copied and repacked) ----------------- */
/* decoder.Decoder weight table (decoder.py:74-154, 160-164): n named
 * float32 arrays, names exactly as the reference dict keys */
int fsb_load_decoder(fsb_ctx* ctx, const fsb_decoder_config* cfg, int n, const char* const* names,
                     const float* const* arrays, const int64_t* numel);
/* bodymodel.BodyTemplate (bodymodel.py:90-104); which = FSB_MHR | FSB_SMPL */
int fsb_load_template(fsb_ctx* ctx, int which, int nv, const float* vertices_rest, const float* joints_rest,
                      const int64_t* parents, const float* skin_weights, const float* shape_basis);
/* projection.ProjectorWeights (projection.py:395-444) with the BaryMap rows
 * of the subsampled targets: corners (n_sub, 3) int64, bary (n_sub, 3) */
int fsb_load_projector(fsb_ctx* ctx, int n_sub, int h1, int h2, const int64_t* corners, const float* bary,
                       const float* w1, const float* b1, const float* w2, const float* b2, const float* w3,
                       const float* b3, const float* mask);

/* ---- stage entry points (device pointers) ------------------------------ */
/* priors.detect_stub(sigma=0) + _body_box_from_keypoints + hand_box x2 +
 * pipeline._box_prompt + prepare_crops (priors.py:166-230,
 * pipeline.py:295-329): images (B, H, W, 3), kp (B, 22, 2) -> boxes
 * (B, 3, 4) f64, prompt (B, 8), crops (B, 3, S, S, 3) and optional int32
 * taps (B, 3, S, S, 4) = (x0, y0, x1, y1).  Bit-exact with the reference.
 * `images` and `kp` may also be pinned host memory (cudaHostAlloc /
 * torch pin_memory): K1 then reads only the crop footprints over PCIe. */
int fsb_boxes_crops(fsb_ctx* ctx, const float* images, int B, int H, int W, const float* kp, double alpha, int S,
                    double* boxes, float* prompt, float* crops, int32_t* taps, void* stream);
/* priors._body_box_from_keypoints (priors.py:166-176): kp (n, 22, 2) ->
 * (n, 4) f64 boxes, bit-exact */
int fsb_body_boxes(fsb_ctx* ctx, const float* kp, int n, int W, int H, double* out, void* stream);
/* priors.hand_box (priors.py:198-217): wrists (n, 2) f32, body (n, 4) f64
 * -> (n, 4) f64; W <= 0 means image_size=None */
int fsb_hand_boxes(fsb_ctx* ctx, const double* wrists, const double* body, int n, double alpha, int W, int H,
                   double* out, void* stream);
/* priors.crop_grid (priors.py:220-230): boxes (n, 4) f64 -> (n, S, S, 2) */
int fsb_crop_grid(fsb_ctx* ctx, const double* boxes, int n, int S, float* out, void* stream);
/* projection.bridge (projection.py:187-203): v (B, nv, 3), corners (nt, 3)
 * int32 and weights (nt, 3) device arrays -> (B, nt, 3) */
int fsb_bridge(fsb_ctx* ctx, const float* v, int B, int nv, const int32_t* corners, const float* w, int nt,
               float* out, void* stream);
/* numkit.bilinear_sample (numkit.py:136-154): image (H, W, C), grid (n, 2) */
int fsb_bilinear(fsb_ctx* ctx, const float* image, int H, int W, int C, const float* grid, int64_t n, float* out,
                 void* stream);
/* Decoder.encode (decoder.py:231-260): crops (n, S, S, 3) -> feats (n, T, D) */
int fsb_encode(fsb_ctx* ctx, const float* crops, int n, float* feats, int precision, void* stream);
/* Decoder.decode_body (decoder.py:324-356, refine=False) for B frames:
 * feature of frame f at feats + f * feat_stride crops; selection bitmask;
 * inter (B, body_layers, 76 + 3 + 44) receives the intermediate prediction
 * (params, camera, kp2d) of every selected layer (nullable) */
int fsb_decode_body(fsb_ctx* ctx, const float* feats, int B, int feat_stride, const float* prompts, uint32_t sel,
                    float* params, float* cam, float* inter, int precision, void* stream);
/* Decoder.decode_hand (decoder.py:360-410): feats (n, T, D) -> rots (n, 3) */
int fsb_decode_hands(fsb_ctx* ctx, const float* feats, int n, uint32_t sel, float* rots, int precision,
                     void* stream);
/* Decoder.encode (decoder.py:231-260) of B frames' body + hand crops
 * (B, 3, S, S, 3) -> feats (B, 3, T, D); in bf16 mode the same launch also
 * projects every decoder layer's cross-attention keys / values
 * (decoder.py:220-227) into the context: fsb_decode_frames on this context
 * with the same feats and B reads them instead of projecting them again,
 * until the next encode on this context (fsb_frame_batch runs the pair;
 * the feats must not be modified in between) */
int fsb_encode_frames(fsb_ctx* ctx, const float* crops, int B, float* feats, int precision, void* stream);
/* body + both hands of B frames in one launch, merged (decoder.py:414-422) */
int fsb_decode_frames(fsb_ctx* ctx, const float* feats, int B, const float* prompts, uint32_t body_sel,
                      uint32_t hand_sel, float* params, float* cam, float* rots, float* merged, int precision,
                      void* stream);
/* bodymodel.fk_batch (bodymodel.py:266-323): poses (B, 76) -> joints
 * (B, 22, 3), rel (B, 22, 3, 4) (either nullable) */
int fsb_fk(fsb_ctx* ctx, int which, const float* poses, int B, float* joints, float* rel, void* stream);
/* bodymodel.skin_batch (bodymodel.py:334-368, correctives=False) */
int fsb_skin(fsb_ctx* ctx, int which, const float* poses, int B, float* verts, void* stream);
/* projection.project_batch (projection.py:475-483) on given MHR vertices */
int fsb_project_vertices(fsb_ctx* ctx, const float* v_mhr, int B, int nv, float* theta, int precision,
                         void* stream);
/* fused MHR skin -> bridge -> projector -> SMPL FK from MHR parameters */
int fsb_skin_project(fsb_ctx* ctx, const float* params, int B, float* v_mhr, float* theta, float* j_smpl,
                     float* v_smpl, int precision, void* stream);
/* the whole frame -> SMPL path for B frames (SURVEY §3.2 composition),
 * replayed from a CUDA graph; with out->theta == out->j_smpl == NULL only the
 * front half (boxes, crops, encode, decoders, merge: pipeline.Pipeline.run,
 * pipeline.py:377-506) runs */
int fsb_frame_batch(fsb_ctx* ctx, const float* images, int B, int H, int W, const float* kp, double alpha,
                    uint32_t body_sel, uint32_t hand_sel, int precision, const fsb_frame_outputs* out,
                    void* stream);

/* projection.fit_batch (projection.py:321-370): `steps` Adam iterations of
 * the fit objective (_fit_terms :266-287) per mesh against the bridged
 * targets (B, nv, 3) on the template loaded in the FSB_SMPL slot, from init
 * (B, 76) or the rest pose (NULL); analytic gradient.  scratch: B*nv*6
 * floats.  Outputs: best_params (B, 76), vertex_error (B,) f64 mean vertex
 * gap of the best iterate, err_curve (B, steps + 1) f64 best-so-far gap per
 * evaluated iterate (the reference's curve is its mean over the batch);
 * grad0 (B, 76), nullable: the objective's gradient at init
 * (projection.fit_objective_grad, :303-309). */
int fsb_fit_batch(fsb_ctx* ctx, const float* target, int B, int nv, const float* init, int steps, double lr,
                  float lambda_pose, float lambda_shape, float* scratch, float* best_params, double* vertex_error,
                  double* err_curve, float* grad0, void* stream);

/* projection.bary_map_from_arrays (projection.py:96-177): device float64
 * source vertices (nv, 3), int64 faces (F, 3) and float64 targets (nt, 3) ->
 * degenerate (F) u8 face flags, face_index (nt) int64, weights (nt, 3) f32;
 * bit-identical to the reference (same float64 operation order, first
 * minimum on ties) */
int fsb_bary_map(fsb_ctx* ctx, const double* src_verts, int nv, const int64_t* src_faces, int F,
                 const double* tgt_verts, int nt, uint8_t* degenerate, int64_t* face_index, float* weights,
                 void* stream);

/* Load (hidden > 0, host arrays w1 (63, hidden), b1 (hidden), w2 (hidden, 63),
 * b2 (63)) or remove (hidden == 0) the kinematic-prior denoiser of
 * projection.denoise (projection.py:684-697) as an epilogue of the SMPL tail:
 * fsb_skin_project / fsb_frame_batch then return theta with theta[3:66]
 * denoised and the SMPL joints of the denoised pose.  Part of the (shared)
 * model. */
int fsb_load_denoiser(fsb_ctx* ctx, const float* w1, const float* b1, const float* w2, const float* b2, int hidden);
/* projection.denoise (projection.py:684-697): poses (B, 63) body-pose
 * parameters -> out (B, 63) = x + relu(x W1 + b1) W2 + b2, W1 (63, hidden),
 * W2 (hidden, 63), hidden <= 128; bit-identical to the reference's
 * numkit.matmul order */
int fsb_denoise(fsb_ctx* ctx, const float* poses, int B, const float* w1, const float* b1, const float* w2,
                const float* b2, int hidden, float* out, void* stream);

/* priors.render_scene (priors.py:237-252) for B scenes: `scenes` is a
 * device array of 464-byte records {float kp[44]; float half_color[66];
 * float inv_two_sigma2; float pad; double gdir[2]} -> (B, H, W, 3) f32 */
int fsb_render(fsb_ctx* ctx, const void* scenes, int B, int H, int W, float* out, void* stream);

/* ---- host staging ------------------------------------------------------- */
/* The single-frame path's input check and staging (numkit.bilinear_sample's
 * check_finite, numkit.py:136-140, + the copy of the caller's host image
 * into the pinned frame K1 reads over PCIe) in one pass on a small
 * persistent pool of host threads: dst[i] = src[i] for i < n (HOST
 * pointers), *nonfinite = 1 if any value is NaN / inf (else 0).  Returns
 * FSB_OK; no context, no device work. */
int fsb_stage_frame(const float* src, float* dst, int64_t n, int* nonfinite);

/* ---- diagnostics -------------------------------------------------------- */
/* reads (and optionally clears) this context's non-finite flag; waits only
 * for the work this context enqueued (an event per stream it used), never
 * for the whole device */
int fsb_nonfinite(fsb_ctx* ctx, int* flag, int reset);
/* the same read enqueued on `stream` (ordered after the work enqueued there
 * before it; no host wait): the flag lands in `host_dst` (pinned host
 * memory) when the stream reaches it, then is cleared if `reset`.  The
 * single-frame path reads it together with its results (one sync). */
int fsb_nonfinite_enqueue(fsb_ctx* ctx, int* host_dst, int reset, void* stream);
int fsb_counters(const fsb_ctx* ctx, fsb_counters_t* out);
/* bytes of frame data the crop gather (K1) has read from pinned host frames
 * since the last reset, i.e. the bytes that crossed PCIe (only the crop
 * footprints are read; HBM-resident frames are not counted); waits for this
 * context's work like fsb_nonfinite */
int fsb_input_bytes(fsb_ctx* ctx, int64_t* total, int reset);
/* number of kernels this context launched (graph replays count their nodes) */
int64_t fsb_kernel_launches(const fsb_ctx* ctx);
/* tcgen05 self-test: C (128 x N) f32 = A (128 x K, bf16 row-major) * B^T,
 * B (N x K) given pre-packed in the K-major canonical UMMA layout */
int fsb_selftest_umma(fsb_ctx* ctx, const void* A, const void* Bpacked, int N, int K, float* C, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* FSB_B200_H */
