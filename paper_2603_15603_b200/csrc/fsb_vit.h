// Large-config encoder (the ViT-L-sized Decoder.encode,
// decoder.py:231-260) as a layer-by-layer pipeline of tcgen05 kernels:
// LayerNorm -> TMA/tcgen05 GEMM with fused epilogue -> flash attention.
// Weights live as bf16 W^T (N x K, row-major) so both GEMM operands are
// K-major TMA boxes; biases, LayerNorm affine and the position table stay fp32.
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <vector>

struct VitLayer {
  const __nv_bfloat16 *wqkv, *wo, *w1, *w2;  // (3D x D), (D x D), (4D x D), (D x 4D)
  const float *ln1_g, *ln1_b, *bqkv, *bo;    // self block
  const float *ln2_g, *ln2_b, *b1, *b2;      // mlp block
};

struct VitW {
  int S = 0, p = 0, D = 0, H = 0, T = 0;
  const __nv_bfloat16* wpatch = nullptr;  // (D x p*p*3)
  const float *patch_b = nullptr, *pos = nullptr, *norm_g = nullptr, *norm_b = nullptr;
  std::vector<VitLayer> layers;
};

// activations for `rows` = crops * T token rows
struct VitWs {
  int max_crops = 0;
  float* x = nullptr;                // (rows, D) fp32 residual stream
  __nv_bfloat16* h = nullptr;        // (rows, max(D, p*p*3)) LN output / attention context / patches
  __nv_bfloat16* qkv = nullptr;      // (rows, 3D)
  __nv_bfloat16* hid = nullptr;      // (rows, 4D)
};

size_t vit_ws_bytes(const VitW& w, int crops);
void vit_ws_carve(const VitW& w, int crops, void* base, VitWs* ws);
// feats (n, T, D) fp32; crops (n, S, S, 3) fp32.  Runs in chunks of ws.max_crops.
cudaError_t launch_vit_encoder(const VitW& w, const VitWs& ws, const float* crops, int n, float* feats, int* nonfinite,
                               cudaStream_t st, int* launches);
