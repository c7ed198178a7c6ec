// lm_rec.h — persistent recurrent LSTM kernels (lm_rec.cu).
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>

namespace jk {

struct RecFwdArgs {
  int B = 0, H = 0, T = 0;       // T = steps (unrolled) or the max width (While mode)
  const int *T_dev = nullptr;    // While mode: device-resident trip count (nullptr: use T)
  const int *lens = nullptr;     // While mode: per-row lengths (rows t >= len carry h, c)
  float *G = nullptr;            // [T*B][4H] input projection + bias (interleaved); overwritten
                                 // with the gate activations (i, f, g, o) for backward
  __nv_bfloat16 *Hs = nullptr;   // [(T+1)*B][ldh] h (bf16); row block 0 = h0
  float *Cs = nullptr;           // [(T+1)*B][ldh] c (fp32); row block 0 = c0
  int ldh = 0;
  const float *h0 = nullptr, *c0 = nullptr;  // [B][H] initial state (fp32)
  float *hT = nullptr, *cT = nullptr;        // [B][H] final state (fp32)
  unsigned int *barrier = nullptr;           // zeroed before the launch: rec_flag_words(grid) u32
  const int *fail = nullptr;                 // nonzero: skip (cooperative cancellation)
  const int *tag = nullptr;                  // state type tag; != 1 -> h0 = c0 = 0 (device Switch)
  unsigned long long *dbg = nullptr;         // optional %globaltimer probe of CTA 0 (8 per step)
  // exchange copy of h in the consumers' shared-memory layout: [T+1][nk chunks][Bp rows][128 B],
  // 128-B swizzled, so a step's operand is fetched with a few large bulk copies
  __nv_bfloat16 *Hsw = nullptr;
};

struct RecBwdArgs {
  int B = 0, H = 0, T = 0;
  const int *T_dev = nullptr;
  const int *lens = nullptr;
  const float *G = nullptr;       // gate activations from the forward kernel
  const float *Cs = nullptr;      // c history
  int ldh = 0;
  const float *dHin = nullptr;    // [T*B][ldd] gradient into h_t from above (decoder / next layer)
  int ldd = 0;
  __nv_bfloat16 *DZ = nullptr;    // [T*B][ldz] out: rb(dz), interleaved columns
  int ldz = 0;                    // >= 64 * ceil(4H / 64), zero padding beyond 4H
  unsigned int *barrier = nullptr;
  const int *fail = nullptr;
  unsigned long long *dbg = nullptr;
  __nv_bfloat16 *DZsw = nullptr;  // exchange copy of dz: [T][nk chunks][Bp rows][128 B] swizzled
};

// step-flag words a launch of `ctas` CTAs needs (one 128-B line per CTA)
constexpr int rec_flag_words(int ctas) { return ctas * 32; }

// bytes of the swizzled exchange buffers
size_t rec_hsw_bytes(int H, int B, int T);
size_t rec_dzsw_bytes(int H, int B, int T);

int rec_grid(int H);
cudaError_t lstm_rec_fwd(const RecFwdArgs &a, const __nv_bfloat16 *Whh, int ldw, bool masked,
                         cudaStream_t st);
// Both layers of a 2-layer stack in one launch (wavefront: layer 1's step t runs with layer 0's
// step t+1). Layer 1's input projection is computed in-kernel (its G buffer receives the gate
// activations only); Wih1 / Whh1 interleaved [4H x ldw] bf16, bias1_il interleaved fp32 [4H].
int rec_fwd_wf_grid(int H);
cudaError_t lstm_rec_fwd_wavefront(const RecFwdArgs &a0, const RecFwdArgs &a1, const __nv_bfloat16 *Whh0,
                                   const __nv_bfloat16 *Wih1, const __nv_bfloat16 *Whh1, int ldw,
                                   const float *bias1_il, bool masked, cudaStream_t st);
// Backward of a 2-layer stack in one launch (wavefront: layer 0's step t runs with layer 1's step
// t-1; W_ih1^T dz1_t, the dgrad of layer 1's input, is folded into layer 0's recurrent MMA, so
// a0.dHin must be null). B <= 64. WihT1: W_ih1 transposed, gate-interleaved [H x ldwt] bf16.
int rec_bwd_wf_grid(int H);
cudaError_t lstm_rec_bwd_wavefront(const RecBwdArgs &a1, const RecBwdArgs &a0, const __nv_bfloat16 *WhhT1,
                                   const __nv_bfloat16 *WihT1, const __nv_bfloat16 *WhhT0, int ldwt,
                                   bool masked, cudaStream_t st);
cudaError_t lstm_rec_bwd(const RecBwdArgs &a, const __nv_bfloat16 *WhhT, int ldwt, bool masked,
                         cudaStream_t st);

}  // namespace jk
