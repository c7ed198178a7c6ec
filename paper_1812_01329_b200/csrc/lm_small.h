// lm_small.h — single-launch fp32 LSTM-LM step (lm_small.cu).
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>

#include "step_kernels.h"

namespace jk {

constexpr int SMALL_MAX_L = 4;

struct SmallLmArgs {
  int V = 0, E = 0, H = 0, L = 0, B = 0, W = 0, T = 0;  // W = token-matrix width
  const int *tok = nullptr, *tgt = nullptr;
  const int *lens = nullptr;  // While mode (masked rows, device trip count); nullptr = unrolled T
  float *Emb = nullptr;
  float *Wih[SMALL_MAX_L] = {}, *Whh[SMALL_MAX_L] = {}, *bias[SMALL_MAX_L] = {};
  float *Wdec = nullptr, *bdec = nullptr;
  float *h[SMALL_MAX_L] = {}, *c[SMALL_MAX_L] = {};
  int *tag = nullptr;
  int tag_specialised = 1;  // TYPE_TAG assumed: read the state; else Switch on the device tag
  int upd_E = 1, upd_Wih[SMALL_MAX_L] = {1, 1, 1, 1}, upd_Whh[SMALL_MAX_L] = {1, 1, 1, 1},
      upd_b[SMALL_MAX_L] = {1, 1, 1, 1}, upd_Wdec = 1, upd_bdec = 1;
  float lr = 0.f;
  GuardList gl{};
  float *ws = nullptr;
  DevStatus *st = nullptr;
};

size_t small_lm_ws_floats(int V, int E, int H, int L, int B, int W);
cudaError_t launch_small_lm(const SmallLmArgs &a, cudaStream_t s);

}  // namespace jk
