// lm_small.cu — the whole speculative training step of a small fp32 LSTM language model (C1:
// B4 T8 H16, fp32) as ONE launch of one CTA: AssertOps -> state snapshot ->
// unrolled or device-While loop -> softmax xent -> backward -> commit
// predicated on every assumption holding. All reductions run in a fixed order in one
// thread per output element, so results are bit-reproducible.
#include "common.cuh"
#include "lm_small.h"

namespace jk {

__device__ __forceinline__ void sync() { __syncthreads(); }

__global__ void __launch_bounds__(1024, 1) lm_small_f32_kernel(SmallLmArgs a) {
  const int tid = threadIdx.x, nt = blockDim.x;
  const int V = a.V, E = a.E, H = a.H, L = a.L, B = a.B, W = a.W, G4 = 4 * a.H;
  DevStatus *st = a.st;
  __shared__ unsigned long long s_key;
  __shared__ int s_err, s_T;
  // ---------------------------------------------------------------- phase 0: guards
  if (tid == 0) {
    s_key = KEY_PASS;
    s_err = 0;
    int T = a.T;
    if (a.lens) {
      T = 0;
      for (int b = 0; b < B; ++b) T = max(T, a.lens[b]);
      T = min(max(T, 0), W);
    }
    s_T = T;
  }
  sync();
  const unsigned long long imask = (1ull << IDX_BITS) - 1;
  for (int k = 0; k < a.gl.n; ++k) {
    const GuardDesc g = a.gl.g[k];
    if (g.kind == G_FORCED) {
      if (tid == 0) atomicMin(&s_key, ((unsigned long long)g.id << IDX_BITS) | imask);
      continue;
    }
    const long long n = g.kind == G_FIRST_EQ ? 1 : g.n;
    for (long long i = tid; i < n; i += nt) {
      const long long v = g.data[i];
      const bool bad = g.kind == G_RANGE ? (v < g.lo || v > g.hi) : v != g.value;
      if (bad) atomicMin(&s_key, ((unsigned long long)g.id << IDX_BITS) | (unsigned long long)i);
    }
  }
  const int T = s_T;
  const bool masked = a.lens != nullptr;
  // runtime errors: token ids of the executed steps, targets of the valid rows
  for (int i = tid; i < T * B; i += nt) {
    const int t = i / B, b = i % B;
    const int id = a.tok[b * W + t];
    if (id < 0 || id >= V) atomicOr(&s_err, 1);
    const bool valid = !masked || t < a.lens[b];
    const int tg = a.tgt[b * W + t];
    if (valid && (tg < 0 || tg >= V)) atomicOr(&s_err, 2);
  }
  sync();
  if (s_key != KEY_PASS || s_err) {
    if (tid == 0) {
      st->key = s_key;
      st->runtime_err = s_err;
      st->trip = T;
      if (s_key != KEY_PASS) {
        st->status = 1;
        const unsigned id = (unsigned)(s_key >> IDX_BITS);
        const unsigned long long idx = s_key & imask;
        long long obs = -1;
        if (idx != imask)
          for (int k = 0; k < a.gl.n; ++k)
            if (a.gl.g[k].id == id && a.gl.g[k].kind != G_FORCED) obs = a.gl.g[k].data[idx];
        st->observed = obs;
      } else {
        st->status = 4;
      }
    }
    return;  // nothing mutated: all-or-nothing
  }
  float *ws = a.ws;
  // workspace carve-up (floats)
  auto take = [&](size_t n) { float *p = ws; ws += (n + 3) & ~size_t(3); return p; };
  float *Hh[SMALL_MAX_L], *Cc[SMALL_MAX_L], *Gt[SMALL_MAX_L];
  for (int l = 0; l < L; ++l) {
    Hh[l] = take((size_t)(W + 1) * B * H);
    Cc[l] = take((size_t)(W + 1) * B * H);
    Gt[l] = take((size_t)W * B * G4);
  }
  float *Xe = take((size_t)W * B * E);        // gathered embeddings
  float *dy = take((size_t)W * B * V);        // logits, then dy
  float *rowloss = take((size_t)W * B);
  float *dHa = take((size_t)W * B * H), *dHb = take((size_t)W * B * H);
  float *dz = take((size_t)B * G4), *dhrec = take((size_t)B * H), *dc = take((size_t)B * H);
  float *carry = take((size_t)B * H), *dxt = take((size_t)B * (E > H ? E : H));
  float *gE = take((size_t)V * E);
  float *gWih[SMALL_MAX_L], *gWhh[SMALL_MAX_L], *gb[SMALL_MAX_L];
  for (int l = 0; l < L; ++l) {
    gWih[l] = take((size_t)G4 * (l ? H : E));
    gWhh[l] = take((size_t)G4 * H);
    gb[l] = take(G4);
  }
  float *gWd = take((size_t)V * H), *gbd = take(V);
  for (int i = tid; i < V * E; i += nt) gE[i] = 0.f;
  // ---------------------------------------------------------------- state snapshot (local copies)
  // self.state may be None (tag 0): the Switch/Merge of the generic graph picks zeros.
  const bool is_tensor = a.tag_specialised || a.tag[0] == 1;
  for (int l = 0; l < L; ++l)
    for (int i = tid; i < B * H; i += nt) {
      Hh[l][i] = is_tensor ? a.h[l][i] : 0.f;
      Cc[l][i] = is_tensor ? a.c[l][i] : 0.f;
    }
  for (int i = tid; i < T * B * E; i += nt) {
    const int r = i / E, k = i % E, t = r / B, b = r % B;
    Xe[i] = a.Emb[(size_t)a.tok[b * W + t] * E + k];
  }
  sync();
  // ---------------------------------------------------------------- forward loop frame
  for (int l = 0; l < L; ++l) {
    const int In = l ? H : E;
    for (int t = 0; t < T; ++t) {
      const float *x = l ? Hh[l - 1] + (size_t)(t + 1) * B * H : Xe + (size_t)t * B * E;
      const float *hp = Hh[l] + (size_t)t * B * H;
      float *g = Gt[l] + (size_t)t * B * G4;
      for (int i = tid; i < B * G4; i += nt) {
        const int b = i / G4, r = i % G4;
        float z = a.bias[l][r];
        for (int k = 0; k < In; ++k) z += x[b * In + k] * a.Wih[l][(size_t)r * In + k];
        for (int k = 0; k < H; ++k) z += hp[b * H + k] * a.Whh[l][(size_t)r * H + k];
        g[i] = z;
      }
      sync();
      for (int i = tid; i < B * H; i += nt) {
        const int b = i / H, u = i % H;
        float *gr = g + (size_t)b * G4;
        const float ig = sigmoidf_(gr[u]), fg = sigmoidf_(gr[H + u]);
        const float gg = tanhf(gr[2 * H + u]), og = sigmoidf_(gr[3 * H + u]);
        const float cp = Cc[l][(size_t)t * B * H + i];
        float c2 = fg * cp + ig * gg, h2 = og * tanhf(c2);
        if (masked && t >= a.lens[b]) { c2 = cp; h2 = hp[i]; }
        gr[u] = ig; gr[H + u] = fg; gr[2 * H + u] = gg; gr[3 * H + u] = og;
        Cc[l][(size_t)(t + 1) * B * H + i] = c2;
        Hh[l][(size_t)(t + 1) * B * H + i] = h2;
      }
      sync();
    }
  }
  // ---------------------------------------------------------------- decoder + softmax xent
  const float *htop = Hh[L - 1] + (size_t)B * H;
  const int R = T * B;
  for (int i = tid; i < R * V; i += nt) {
    const int r = i / V, v = i % V;
    float z = a.bdec[v];
    for (int k = 0; k < H; ++k) z += htop[(size_t)r * H + k] * a.Wdec[(size_t)v * H + k];
    dy[i] = z;
  }
  sync();
  __shared__ float s_nv;
  if (tid == 0) {
    int nvalid = 0;
    for (int b = 0; b < B; ++b) nvalid += masked ? min(a.lens[b], T) : T;
    s_nv = (float)max(nvalid, 1);
  }
  sync();
  for (int r = tid; r < R; r += nt) {
    const int t = r / B, b = r % B;
    float *y = dy + (size_t)r * V;
    const bool valid = !masked || t < a.lens[b];
    float m = -INFINITY;
    for (int v = 0; v < V; ++v) m = fmaxf(m, y[v]);
    float s = 0.f;
    for (int v = 0; v < V; ++v) s += expf(y[v] - m);
    const float lse = m + logf(s);
    const int tg = a.tgt[b * W + t];
    rowloss[r] = valid ? (lse - y[tg]) / s_nv : 0.f;
    for (int v = 0; v < V; ++v)
      y[v] = valid ? (expf(y[v] - lse) - (v == tg ? 1.f : 0.f)) / s_nv : 0.f;
  }
  sync();
  // decoder backward: dW_dec, db_dec, dh_top
  for (int i = tid; i < V * H; i += nt) {
    const int v = i / H, k = i % H;
    float acc = 0.f;
    for (int r = 0; r < R; ++r) acc += dy[(size_t)r * V + v] * htop[(size_t)r * H + k];
    gWd[i] = acc;
  }
  for (int v = tid; v < V; v += nt) {
    float acc = 0.f;
    for (int r = 0; r < R; ++r) acc += dy[(size_t)r * V + v];
    gbd[v] = acc;
  }
  for (int i = tid; i < R * H; i += nt) {
    const int r = i / H, k = i % H;
    float acc = 0.f;
    for (int v = 0; v < V; ++v) acc += dy[(size_t)r * V + v] * a.Wdec[(size_t)v * H + k];
    dHa[i] = acc;
  }
  sync();
  // ---------------------------------------------------------------- backward loop (reverse frame)
  float *dHin = dHa, *dHout = dHb;
  for (int l = L - 1; l >= 0; --l) {
    const int In = l ? H : E;
    for (int i = tid; i < G4 * In; i += nt) gWih[l][i] = 0.f;
    for (int i = tid; i < G4 * H; i += nt) gWhh[l][i] = 0.f;
    for (int i = tid; i < G4; i += nt) gb[l][i] = 0.f;
    for (int i = tid; i < B * H; i += nt) { dhrec[i] = 0.f; dc[i] = 0.f; carry[i] = 0.f; }
    sync();
    for (int t = T - 1; t >= 0; --t) {
      const float *g = Gt[l] + (size_t)t * B * G4;
      const float *x = l ? Hh[l - 1] + (size_t)(t + 1) * B * H : Xe + (size_t)t * B * E;
      const float *hp = Hh[l] + (size_t)t * B * H;
      for (int i = tid; i < B * H; i += nt) {
        const int b = i / H, u = i % H;
        const float dh = dHin[(size_t)t * B * H + i] + dhrec[i] + carry[i];
        const float *gr = g + (size_t)b * G4;
        float *dzr = dz + (size_t)b * G4;
        if (masked && t >= a.lens[b]) {
          carry[i] = dh;
          dzr[u] = dzr[H + u] = dzr[2 * H + u] = dzr[3 * H + u] = 0.f;
        } else {
          carry[i] = 0.f;
          const float ig = gr[u], fg = gr[H + u], gg = gr[2 * H + u], og = gr[3 * H + u];
          const float ct = Cc[l][(size_t)(t + 1) * B * H + i], cp = Cc[l][(size_t)t * B * H + i];
          const float tc = tanhf(ct);
          const float dout = dh * tc;
          const float dcc = dc[i] + dh * og * (1.f - tc * tc);
          dzr[u] = dcc * gg * ig * (1.f - ig);
          dzr[H + u] = dcc * cp * fg * (1.f - fg);
          dzr[2 * H + u] = dcc * ig * (1.f - gg * gg);
          dzr[3 * H + u] = dout * og * (1.f - og);
          dc[i] = dcc * fg;
        }
      }
      sync();
      for (int i = tid; i < B * H; i += nt) {
        const int b = i / H, u = i % H;
        float acc = 0.f;
        for (int r = 0; r < G4; ++r) acc += dz[(size_t)b * G4 + r] * a.Whh[l][(size_t)r * H + u];
        dhrec[i] = acc;
      }
      for (int i = tid; i < B * In; i += nt) {
        const int b = i / In, k = i % In;
        float acc = 0.f;
        for (int r = 0; r < G4; ++r) acc += dz[(size_t)b * G4 + r] * a.Wih[l][(size_t)r * In + k];
        dxt[i] = acc;
      }
      for (int i = tid; i < G4 * In; i += nt) {
        const int r = i / In, k = i % In;
        float acc = 0.f;
        for (int b = 0; b < B; ++b) acc += dz[(size_t)b * G4 + r] * x[(size_t)b * In + k];
        gWih[l][i] += acc;
      }
      for (int i = tid; i < G4 * H; i += nt) {
        const int r = i / H, k = i % H;
        float acc = 0.f;
        for (int b = 0; b < B; ++b) acc += dz[(size_t)b * G4 + r] * hp[(size_t)b * H + k];
        gWhh[l][i] += acc;
      }
      for (int r = tid; r < G4; r += nt) {
        float acc = 0.f;
        for (int b = 0; b < B; ++b) acc += dz[(size_t)b * G4 + r];
        gb[l][r] += acc;
      }
      sync();
      if (l > 0) {
        for (int i = tid; i < B * H; i += nt) dHout[(size_t)t * B * H + i] = dxt[i];
      } else {
        // embedding gradient: rows of this step in ascending b (segmented sum order per word)
        for (int k = tid; k < E; k += nt)
          for (int b = 0; b < B; ++b) gE[(size_t)a.tok[b * W + t] * E + k] += dxt[(size_t)b * E + k];
      }
      sync();
    }
    float *tmp = dHin; dHin = dHout; dHout = tmp;
  }
  // ---------------------------------------------------------------- finalize + commit
  __shared__ float s_loss;
  if (tid == 0) {
    float acc = 0.f;
    for (int r = 0; r < R; ++r) acc += rowloss[r];
    s_loss = acc;
    st->loss = acc;
    st->key = KEY_PASS;
    st->status = 0;
    st->runtime_err = 0;
    st->observed = 0;
    st->trip = T;
  }
  sync();
  const float lr = a.lr;
  if (a.upd_E) for (int i = tid; i < V * E; i += nt) a.Emb[i] -= lr * gE[i];
  for (int l = 0; l < L; ++l) {
    const int In = l ? H : E;
    if (a.upd_Wih[l]) for (int i = tid; i < G4 * In; i += nt) a.Wih[l][i] -= lr * gWih[l][i];
    if (a.upd_Whh[l]) for (int i = tid; i < G4 * H; i += nt) a.Whh[l][i] -= lr * gWhh[l][i];
    if (a.upd_b[l]) for (int i = tid; i < G4; i += nt) a.bias[l][i] -= lr * gb[l][i];
    for (int i = tid; i < B * H; i += nt) {
      a.h[l][i] = Hh[l][(size_t)T * B * H + i];
      a.c[l][i] = Cc[l][(size_t)T * B * H + i];
    }
  }
  if (a.upd_Wdec) for (int i = tid; i < V * H; i += nt) a.Wdec[i] -= lr * gWd[i];
  if (a.upd_bdec) for (int i = tid; i < V; i += nt) a.bdec[i] -= lr * gbd[i];
  if (tid == 0 && a.tag) a.tag[0] = 1;
}

size_t small_lm_ws_floats(int V, int E, int H, int L, int B, int W) {
  const size_t G4 = 4 * (size_t)H;
  auto r4 = [](size_t n) { return (n + 3) & ~size_t(3); };
  size_t n = 0;
  for (int l = 0; l < L; ++l) n += 2 * r4((size_t)(W + 1) * B * H) + r4((size_t)W * B * G4);
  n += r4((size_t)W * B * E) + r4((size_t)W * B * V) + r4((size_t)W * B) + 2 * r4((size_t)W * B * H);
  n += r4((size_t)B * G4) + 3 * r4((size_t)B * H) + r4((size_t)B * (E > H ? E : H));
  n += r4((size_t)V * E);
  for (int l = 0; l < L; ++l) n += r4(G4 * (l ? H : E)) + r4(G4 * H) + r4(G4);
  n += r4((size_t)V * H) + r4(V);
  return n + 64;
}

cudaError_t launch_small_lm(const SmallLmArgs &a, cudaStream_t s) {
  if (a.L > SMALL_MAX_L) return cudaErrorInvalidValue;
  lm_small_f32_kernel<<<1, 1024, 0, s>>>(a);
  return cudaGetLastError();
}

}  // namespace jk
