// Device-side weight tables of the frozen encoder/decoders and body models.
// All pointers are device addresses into one arena owned by the fsb_ctx.
// Linear weights are stored (in, out) row-major like the reference
// (decoder.py:74-154: y = x @ W + b); Q|K|V are concatenated to one (D, 3D)
// matrix so a block issues one projection GEMM.
#pragma once
#include <stdint.h>
#include <cuda_bf16.h>

#define FSB_MAX_LAYERS 32

// Per-layer block of the small fp32 parameters (LayerNorm affine, biases)
// that the tensor-core kernels stage into shared memory with one bulk copy
// per layer (offsets in floats, D = 64):
//   self attention : ln_g, ln_b, bq|bk|bv, bo
//   cross attention: lnq_g, lnq_b, lnkv_g, lnkv_b, bq|bk|bv, bo
//   MLP            : ln_g, ln_b, b1 (4D), b2
#define TCP_S_LN_G 0
#define TCP_S_LN_B 64
#define TCP_S_BQKV 128
#define TCP_S_BO 320
#define TCP_C_LNQ_G 384
#define TCP_C_LNQ_B 448
#define TCP_C_LNKV_G 512
#define TCP_C_LNKV_B 576
#define TCP_C_BQKV 640
#define TCP_C_BO 832
#define TCP_M_LN_G 896
#define TCP_M_LN_B 960
#define TCP_M_B1 1024
#define TCP_M_B2 1280
#define TCP_FLOATS 1344

struct AttnW {
  const float* ln_g;   // self: ln; cross: lnq
  const float* ln_b;
  const float* ln2_g;  // cross only: lnkv
  const float* ln2_b;
  const float* wqkv;   // (D, 3D)
  const float* bqkv;   // (3D)
  const float* wo;     // (D, D)
  const float* bo;
  // bf16 images in the K-major UMMA layout (tc_sm100.cuh), W^T: (N, K)
  const uint8_t* t_qkv;  // self: (3D, D)
  const uint8_t* t_q;    // cross: (D, D)
  const uint8_t* t_kv;   // cross: (2D, D)
  const uint8_t* t_o;    // (D, D)
};

struct MlpW {
  const float* ln_g;
  const float* ln_b;
  const float* w1;  // (D, 4D)
  const float* b1;
  const float* w2;  // (4D, D)
  const float* b2;
  const uint8_t* t_w1;  // bf16 image (4D, D)
  const uint8_t* t_w2;  // bf16 image (D, 4D)
};

// The weight-image / parameter-block sequence one tensor-core role
// (encoder, body decoder, hand decoder) consumes, in consumption order.
// Built on the host at upload and copied into shared memory by each CTA with
// a few vector loads (k_transformer_tc.cu).
#define FSB_TC_MAX_IMAGES 64
struct TcStream {
  const uint8_t* wptr[FSB_TC_MAX_IMAGES];
  uint32_t wbytes[FSB_TC_MAX_IMAGES];
  const float* pptr[FSB_MAX_LAYERS + 8];
  int nw, nprm;
  int pad[2];
};

struct EncW {
  const uint8_t* t_patch;  // bf16 image (D, p*p*3)
  const float* patch_w;  // (p*p*3, D)
  const float* patch_b;
  const float* pos;      // (n_patch, D)
  const float* norm_g;
  const float* norm_b;
  int layers;
  AttnW self[FSB_MAX_LAYERS];
  MlpW mlp[FSB_MAX_LAYERS];
  const float* tc_params[FSB_MAX_LAYERS];  // TCP_* blocks (cross part unused)
  const TcStream* tcs;                     // device copy of the tcgen05 weight stream
};

struct BodyW {
  const float* token_init;  // (51, D)
  const float* p2d_init;    // (22, D)
  const float* p3d_init;    // (22, D)
  const float* norm_g;
  const float* norm_b;
  const float* head_params_w;  // (D, 76)
  const float* head_params_b;
  const float* head_cam_w;     // (D, 3)
  const float* head_cam_b;
  const float* phi2d_w;        // (2, D)
  const float* phi2d_b;
  const float* phi3d_w;        // (3, D)
  const float* phi3d_b;
  const float* prompt_box_w;   // (8, 4D)
  const float* prompt_box_b;
  const float* joints_rest;    // (22, 3) of the decoder's template
  int layers;
  AttnW self[8];
  AttnW cross[8];
  MlpW mlp[8];
  const float* tc_params[8];  // TCP_* blocks
  const TcStream* tcs;        // device copy of the tcgen05 weight stream
};

struct HandW {
  const float* token_init;  // (4, D)
  const float* p_init;      // (3, D)
  const float* norm_g;
  const float* norm_b;
  const float* head_rot_w;  // (D, 3)
  const float* head_rot_b;
  const float* head_cam_w;
  const float* head_cam_b;
  const float* phi2d_w;     // (2, D)
  const float* phi2d_b;
  const float* canon_pts;   // (3, 3)
  int layers;
  AttnW self[8];
  AttnW cross[8];
  MlpW mlp[8];
  const float* tc_params[8];  // TCP_* blocks
  const TcStream* tcs;        // device copy of the tcgen05 weight stream
};

// floats per vertex record: rest xyz + pad, shape basis (3 x 10), nnz skin
// weights, nnz joint ids (int bits), padded to a multiple of 4 (float4 loads)
__host__ __device__ constexpr int vertex_record_floats(int nnz) { return (34 + 2 * nnz + 3) / 4 * 4; }

// body template on device (LBS / FK)
struct TemplateDev {
  int nv;
  int nnz;                   // padded skin nonzeros per vertex (2, 4 or 8)
  const float* rec;          // (nv, vertex_record_floats(nnz)) packed vertex records
  const float* v_rest;       // (nv, 3)
  const float* shape_basis;  // (nv, 3, 10)
  const int16_t* skin_j;     // (nv, nnz) joint ids, ascending, padded with 0
  const float* skin_w;       // (nv, nnz) weights, padded with 0
  const float* joints_rest;  // (22, 3)
  // skin weights by joint (CSR) for the fit's dL/dA reduction (k_fit.cu)
  const int* joint_off;      // (23)
  const int* joint_v;        // vertex ids
  const float* joint_w;      // weights
  // shape basis of each 256-vertex tile as bf16 hi / lo UMMA images for the
  // tensor-core shape blend of k_lbs_tc (k_body.cu): per tile 12 x 4 KB =
  // [even | odd vertices][hi | lo][x, y, z], each 128 rows x K = 16 K-major
  // (row i = vertex 2 i + parity of the tile)
  const uint8_t* basis_img;
};

// k_lbs_tc: vertices per tile (two per TMEM lane) and meshes per chunk
#define FSB_LBS_TILE 256
#ifndef FSB_LBS_N
#define FSB_LBS_N 16
#endif
#define FSB_LBS_BASIS_BYTES (12 * 128 * 16 * 2)
// per-chunk record written by k_fk (lbs_in): the chunk's joint transforms
// interleaved by mesh pairs (float2 [N/2][22 * 12]) and its shape
// coefficients as bf16 hi / lo images (N meshes x K = 16, K-major)
// float2 slots per joint in the interleaved transforms (12 used; padding to
// 14 or 16 to spread the joints over the banks measured no faster at C3)
#ifndef FSB_LBS_JS
#define FSB_LBS_JS 12
#endif
#define FSB_LBS_REC_A2 (FSB_LBS_N / 2 * 22 * FSB_LBS_JS * 8)
#define FSB_LBS_REC_B (FSB_LBS_N * 16 * 2)
#define FSB_LBS_REC_BYTES (FSB_LBS_REC_A2 + 2 * FSB_LBS_REC_B)

// barycentric map + projector
struct ProjectorDev {
  int n_sub;              // V_sub
  int h1, h2;             // hidden widths
  const int32_t* corners; // (n_sub, 3) source vertex ids of the subsampled targets
  const float* bw;        // (n_sub, 3) barycentric weights
  const float* w1;        // (3*n_sub, h1) f32
  const float* b1;
  const float* w2;        // (h1, h2)
  const float* b2;
  const float* w3;        // (h2, 76)
  const float* b3;
  const float* mask;      // (76)
  // bf16 tile images of W^T for the tensor-core MLP (k_mlp_tc.cu):
  // [n_tile][k_tile] 128 x 128 K-major tiles, zero padded
  const uint8_t* img_w1;  // (h1 / 128) x KT1, KT1 = ceil(3 * n_sub / 128)
  const uint8_t* img_w2;  // (h2 / 128) x KT2, KT2 = h1 / 128
  const uint8_t* img_w3;  // 1 x KT3 (76 rows used), KT3 = h2 / 128
  // fp32 (reference-precision) mode on the same tensor-core kernels: the
  // remainders W - bf16(W) as bf16 images (split-bf16: hi.hi + hi.lo + lo.hi)
  const uint8_t* img_w1_lo;
  const uint8_t* img_w2_lo;
  const uint8_t* img_w3_lo;
  int KT1, KT2, KT3;
  // compacted corner vertices: the LBS kernel writes the nu distinct corner
  // vertices of every mesh (vertex 0, the bridge origin, is slot 0) to a
  // (B, nu, 3) buffer as it skins them, and the bridge gathers from that
  // instead of from scattered rows of V_mhr
  int nu;                 // distinct corner vertices (+ vertex 0)
  int nvslot;             // length of vslot (max corner id + 1)
  const int32_t* vslot;   // (nvslot) slot of a source vertex in the compacted buffer, -1 if unused
  const int32_t* ucorners;  // (n_sub, 3) corners as slots
};

// optional compacted corner output of the LBS kernel (ProjectorDev::nu)
struct CornerOut {
  float* vu = nullptr;             // (B, nu, 3) or null
  const int32_t* vslot = nullptr;  // ProjectorDev::vslot
  int nvslot = 0, nu = 0;
};

// arguments of the fused decoder launch (k_transformer.cu)
struct DecodeArgs {
  const float* feats;       // (ncrops, T, D)
  const float* prompts;     // (nbody, 8)
  int nbody, nhand;
  int body_feat_stride;     // crop index of frame f's body feature = f * stride
  int hand_feat_first;      // crop of hand h = first + (h / 2) * stride + (h % 2)
  unsigned body_sel, hand_sel;
  float* body_params;       // (nbody, 76)
  float* body_cam;          // (nbody, 3)
  float* hand_rots;         // (nhand, 3)
  float* merged;            // (nbody, 76) or null: body params with hand rotations overwritten
  float* inter;             // (nbody, body_layers, 76 + 3 + 44) or null: intermediate predictions
  int* nonfinite;
  // bf16 mode: the cross-attention keys / values of every layer, projected
  // ahead of the decoders from the features (KvArgs below)
  const uint8_t* body_kv;   // FSB_KV_BODY_TILE bytes per (body tile, layer)
  const uint8_t* hand_kv;   // FSB_KV_HAND bytes per (hand, layer), 32 hands per tile
  int hand_tiles_per_cta;   // set by the launcher
  int hand_split;           // set by the launcher: one-tile hand CTAs split the cross-attention keys over both groups
};

// Cross-attention K / V of the decoders depend only on the features
// (decoder.py:220-227: LN_kv(f) Wk + bk, LN_kv(f) Wv + bv), so the bf16 path
// projects them for every layer right after the encoder (k_encoder_tc, or
// the same kernel on given features) instead of inside the decoders' serial
// layer chain.
//  * body tile T (frames 2T, 2T + 1), layer l: the decoder's shared-memory
//    image of the tile's keys and values, [K: 4 heads x (128 x 16, K-major)]
//    [V^T: 4 heads x (16 x 128 keys, K-major)], 32 KB, loaded with one bulk
//    copy per layer;
//  * hand tile T (hands 32 T + i), layer l: 32 key pairs s of 16 KB
//    ([hand i][512 bytes]); in hand i's 512 bytes the 16-byte chunk
//    q = kk 16 + kv 8 + h 4 + c (key 2 s + kk, K | V, column half h, chunk c
//    of the half) sits at position q ^ (i & 7), so a key pair lands in shared
//    memory with one 16 KB bulk copy and a warp's eight hands x four chunks
//    read distinct banks.
#define FSB_KV_BODY_TILE 32768
#define FSB_HANDS_PER_TILE 32
#define FSB_KV_HAND 16384
struct KvArgs {
  int mode;                 // 0: encode only; 1: encode frames + K / V; 2: K / V of the given features
  int nbody, nhand;         // modes 1, 2: crops as DecodeArgs (body of frame f = f * stride, hand u =
  int body_feat_stride;     //   first + (u / 2) * stride + u % 2)
  int hand_feat_first;
  const float* feats_in;    // mode 2
  uint8_t* body_kv;
  uint8_t* hand_kv;
  const TcStream* tcs[2];   // body / hand: (mode 1) encoder images + the role's K | V images, (mode 2) K | V only
  int layers[2];            // body / hand decoder layers
};
