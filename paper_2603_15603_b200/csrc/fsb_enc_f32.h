// Reference-precision (fp32) encoder for any DecoderConfig (k_enc_f32.cu).
// Linear weights fp32 (in, out) row-major as the reference stores them
// (decoder.py:74-154), q|k|v concatenated to (D, 3D).
#pragma once
#include <cuda_runtime.h>

#include <vector>

struct EncF32Layer {
  const float *wqkv, *bqkv, *wo, *bo;  // (D, 3D), (3D), (D, D), (D)
  const float *ln1_g, *ln1_b, *ln2_g, *ln2_b;
  const float *w1, *b1, *w2, *b2;      // (D, 4D), (4D), (4D, D), (D)
};

struct EncF32W {
  int S = 0, p = 0, D = 0, H = 0, T = 0;
  const float *wpatch = nullptr, *patch_b = nullptr, *pos = nullptr, *norm_g = nullptr, *norm_b = nullptr;
  std::vector<EncF32Layer> layers;
};

struct EncF32Ws {
  int max_crops = 0;
  float *x = nullptr, *h = nullptr, *qkv = nullptr, *hid = nullptr;
};

bool enc_f32_supported(int D, int H);
size_t enc_f32_ws_bytes(const EncF32W& w, int crops);
void enc_f32_ws_carve(const EncF32W& w, int crops, void* base, EncF32Ws* ws);
cudaError_t launch_enc_f32(const EncF32W& w, const EncF32Ws& ws, const float* crops, int n, float* feats,
                           int* nonfinite, cudaStream_t st, int* launches);

// C = act(A W + bias) (+ C when accumulate): CUDA-core fp32 GEMM (k_body.cu)
cudaError_t launch_gemm_f32_acc(const float* A, int lda, const float* W, const float* bias, float* C, int ldc, int M,
                                int N, int K, int relu, int accumulate, cudaStream_t st);
