// lm_rec.cu — the loop of the Figure 1 program (`for item in sequence: state =
// rnn_cell(state, item)`) executed as ONE persistent launch per layer and direction: the loop
// frame lives on the device — unrolled to the asserted trip count or, in While
// mode, bounded by a trip count computed on the device — with no host round trip.
//
// Weight-stationary tcgen05 design. CTA j owns hidden units [16j, 16j+16) (all 4 gates):
//   forward : its 64 gate-interleaved rows of W_hh stay in shared memory for all T steps; per step
//             h_{t-1} (bf16, [B x H]) streams in by TMA, D[b, 4u+g] = h_{t-1} . W_slice^T lands in
//             TMEM (M = 128 batch rows, N = 64, K = 16 per MMA), and the cell update runs in the
//             epilogue thread that owns batch row b — c and the fp32 h stay in registers.
//   backward: its 16 columns of W_hh (stored transposed, [units x 4H]) stay in shared memory;
//             per step dz_{t+1} (bf16 [B x 4H]) streams in, D[b, u] = dz_{t+1} . W_hh[:, u] gives the
//             recurrent dh, and the cell backward runs in registers (dc carried in registers).
// Warp roles (192 threads): warps 0-3 epilogue (thread = batch row = TMEM lane), warp 4 producer
// (polls the producers' step flags, then fetches many 64-column chunks per TMA op through a 3-D
// tensor map), warp 5 MMA issuer. Each step is latency-bound, so every chunk of a step is in
// flight at once when shared memory allows, and the step's other operands are loaded before the
// MMA wait. Synchronisation is dataflow (per-CTA release flags), not a grid barrier.
// Gate-interleaved order: row 4u+g of the working copies = canonical row g*H+u (g = i,f,g,o).
#include <algorithm>

#include "common.cuh"
#include "gemm_tc.h"
#include "lm_rec.h"

namespace jk {

// MMA-issuing warps (one tcgen05.mma stream each, own accumulator): with the elect.sync issue one
// warp keeps the M = 64 MMAs pipe-bound (round 1 used four to hide a slow per-MMA issue)
constexpr int REC_NMW = 1;
constexpr int REC_THREADS = 160 + 32 * REC_NMW;
constexpr int REC_UPC = 16;      // hidden units per CTA
constexpr int REC_MAX_SLOTS = 48;
constexpr int SMEM_BUDGET = 232448 - 1024;

// fp32-accurate activations on the fast exp path (|error| ~1e-7)
JN_DEV float sig_f(float x) { return __fdividef(1.f, 1.f + __expf(-x)); }
JN_DEV float tanh_f(float x) {
  const float e = __expf(-2.f * fabsf(x));
  const float t = __fdividef(1.f - e, 1.f + e);
  return copysignf(t, x);
}

// Step flags are REC_FS words apart (one 128-B line each): a CTA's release store then shares its
// line with no other producer while ~100 consumers poll.
constexpr int REC_FS = 32;

// Dataflow synchronisation between the CTAs of a recurrent launch. Every step writes a fresh row
// block (h_t / dz_t), so there are no write-after-read hazards — only read-after-write: a CTA
// publishes "my slice of step t is written" with a release store of its per-CTA flag, and the
// consumer's producer warp waits for the flags of all producers, then fences once.
JN_DEV void publish_flag(unsigned int *flag, unsigned int v) {
  __syncthreads();  // all of this CTA's stores of the step precede the release (bar.sync cumulativity)
  if (threadIdx.x == 0) asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(flag), "r"(v) : "memory");
}
// Executed by a whole warp: lanes poll the n producer flags in parallel, two per 8-B relaxed load
// (flags must be 8-B aligned), then one acquire fence and one generic->async proxy fence for the
// bulk copies lane 0 issues next.
JN_DEV void wait_flags_warp(const unsigned int *flags, int n, unsigned int v) {
  const int lane = threadIdx.x & 31;
  for (int c = lane; c < n; c += 32) {
    unsigned x;
    do {
      asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(x) : "l"(flags + c * REC_FS) : "memory");
    } while (x < v);
  }
  __syncwarp();
  asm volatile("fence.acq_rel.gpu;" ::: "memory");
  fence_proxy_async_global();  // the bulk copies (async proxy) read what the generic proxy wrote
}

// Producer side of an exchange step: its generic-proxy stores of the exchange block, before the
// release (the consumer fences generic -> async proxy itself after its acquire, before the copy)
JN_DEV void prod_proxy_fence() { fence_proxy_async_global(); }
// Named barrier of the four epilogue warps (threads 0-127) — the other warps run ahead.
JN_DEV void epi_bar() { asm volatile("bar.sync 1, 128;" ::: "memory"); }
// Epilogue: this step's exchange-block writes are done (fenced for the async proxy by the caller);
// thread 0 releases the CTA's step flag once all four epilogue warps got here. (Measured slower:
// each epilogue warp releasing its own rows with a red.release.gpu.add.)
JN_DEV void epi_publish(unsigned int *flag, unsigned int v) {
  epi_bar();
  if (threadIdx.x == 0) asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(flag), "r"(v) : "memory");
}
// Epilogue warp: its TMEM reads of this step completed -> the MMA warps may overwrite the tiles.
JN_DEV void epi_tmem_release(uint64_t *tempty) {
  tc_fence_before();
  __syncwarp();
  if ((threadIdx.x & 31) == 0) mbar_arrive(tempty);
}

struct RecLayout {
  int nk;       // 64-column chunks of the streamed operand per step (run A, then run B)
  int nka;      // chunks of run A (the wavefront kernel's layer-1 CTAs stream two exchange blocks)
  int wbytes;   // resident weight slice bytes (1 KB aligned)
  int cb;       // bytes per chunk in smem = Bp * 128 (Bp = B rounded up to 8)
  int bp;       // rows per chunk fetched
  int ch;       // chunks per TMA op
  int nops;     // TMA ops per step
  int nslots;   // ring slots (one op each)
  int pad;      // bytes after the ring: an M=128 MMA reads 128 rows from a chunk base
};

// optional timeline probe (every CTA): dbg[(cta * T + t) * 16 + k] = %globaltimer (ns)
#define PROBE(t_, k_)                                                            \
  do {                                                                           \
    if (a.dbg) {                                                                 \
      unsigned long long ts_;                                                    \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ts_));                    \
      a.dbg[((size_t)blockIdx.x * a.T + (t_)) * 16 + (k_)] = ts_;                \
    }                                                                            \
  } while (0)

// Epilogue: this CTA's 16 units of batch row b (bf16) into exchange block `blk` — chunk u0/64,
// two 16-B granules at their swizzled positions (the layout the consumer's MMA descriptors read).
JN_DEV void write_xchg(uint8_t *xbuf, int blk, int nk, int cb, int u0, int b,
                       const __nv_bfloat16 (&hb)[16]) {
  uint8_t *chunk = xbuf + ((size_t)blk * nk + (u0 >> 6)) * cb;
  const uint32_t g0 = (uint32_t)(u0 & 63) >> 3;
  *reinterpret_cast<uint4 *>(chunk + sw128_off(b, g0)) = reinterpret_cast<const uint4 *>(hb)[0];
  *reinterpret_cast<uint4 *>(chunk + sw128_off(b, g0 + 1)) = reinterpret_cast<const uint4 *>(hb)[1];
}

// Ops of a step: run A's chunks [0, nka) in ops of up to ch chunks, then run B's [nka, nk).
JN_DEV int ops_a(const RecLayout &ly) { return (ly.nka + ly.ch - 1) / ly.ch; }
JN_DEV void op_range(const RecLayout &ly, int k, int &first, int &n) {
  const int oa = ops_a(ly);
  if (k < oa) {
    first = k * ly.ch;
    n = min(ly.ch, ly.nka - first);
  } else {
    first = ly.nka + (k - oa) * ly.ch;
    n = min(ly.ch, ly.nk - first);
  }
}

// Producer (warp 4, lane 0): op k of step `st` copies its chunks of the step's exchange block(s)
// (already in the swizzled shared-memory layout, contiguous) into ring slot (st*nops + k) %
// nslots with one bulk copy. srcA holds chunks [0, nka), srcB chunks [nka, nk).
// q0 >= 0: ring position of the step's first op (steps with varying op counts); else st * nops.
JN_DEV void issue_step(const uint8_t *srcA, const uint8_t *srcB, const RecLayout &ly, uint8_t *sA,
                       uint64_t *full, uint64_t *empty, int st, int k_begin = 0, int k_end = 1 << 30,
                       int q0 = -1) {
  for (int k = k_begin; k < min(ly.nops, k_end); ++k) {
    const int q = (q0 >= 0 ? q0 : st * ly.nops) + k, s = q % ly.nslots, r = q / ly.nslots;
    if (r > 0) mbar_wait(&empty[s], (r - 1) & 1);
    int first, nch;
    op_range(ly, k, first, nch);
    const uint8_t *src = first < ly.nka ? srcA + (size_t)first * ly.cb : srcB + (size_t)(first - ly.nka) * ly.cb;
    mbar_expect_tx(&full[s], nch * ly.cb);
    bulk_load(sA + (size_t)s * ly.ch * ly.cb, src, nch * ly.cb, &full[s]);
  }
}

// MMA issuers (warps 5 .. 5+REC_NMW-1, one elected lane each, four MMAs per asm statement: a
// single thread then issues back to back at ~35 cycles per M = 64 MMA, scripts/bench_mma_issue.cu;
// under `lane == 0` with per-MMA descriptors it was ~130-150 cycles, scripts/bench_mma.cu), and the
// recurrent MMAs are small (N = 64 / 32 / 16), so the step's K chunks are dealt round-robin to
// REC_NMW warps, each accumulating into its own TMEM tile (columns w * NCOL); the epilogue sums
// the tiles. Warp w: D_w = sum over chunks j = w (mod REC_NMW) of A_j . W_j^T (W chunk j at
// sW + j * wchunk bytes).
template <int NCOL>
JN_DEV void mma_step(const RecLayout &ly, uint8_t *sA, uint8_t *sW, int wchunk, uint64_t *full,
                     uint64_t *empty, uint64_t *tfull, uint64_t *tempty, uint32_t tmem, uint32_t idesc,
                     int st, int w, unsigned long long *pr, int q0 = -1) {
  const uint32_t acc = tmem + (uint32_t)(w * NCOL);
  for (int k = 0; k < ly.nops; ++k) {
    const int q = (q0 >= 0 ? q0 : st * ly.nops) + k, s = q % ly.nslots, r = q / ly.nslots;
    if (k == 0 && st > 0) mbar_wait(tempty, (st - 1) & 1);  // the epilogue drained step st-1's tiles
    mbar_wait(&full[s], r & 1);
    if (pr && k < 4) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(pr[8 + 2 * k]));
    tc_fence_after();
    int first, nch;
    op_range(ly, k, first, nch);
    const uint32_t sa = smem_u32(sA + (size_t)s * ly.ch * ly.cb);
    for (int c = 0; c < nch; ++c) {
      const int j = first + c;
      if (j % REC_NMW != w) continue;
      const uint32_t ca = sa + c * ly.cb, cw = smem_u32(sW + (size_t)j * wchunk);
      umma_bf16_k64(acc, umma_desc_sw128(ca, 16, 1024), umma_desc_sw128(cw, 16, 1024), idesc, j != w ? 1u : 0u,
                    2, 2);
    }
    umma_commit(&empty[s]);  // the slot is free once every issuing warp's MMAs on it completed
    if (pr && k < 4) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(pr[9 + 2 * k]));
  }
  umma_commit(tfull);
}

// ---------------------------------------------------------------------------------- forward
// One forward recurrence role: a CTA owning UPC units (4 UPC gate-interleaved rows) of one layer.
// Single-layer launch: every CTA streams its own layer's h_{t-1} (run A). Wavefront launch (two
// layers in one kernel): layer-1 CTAs compute W_ih1 h0_t + W_hh1 h1_{t-1} in one accumulation —
// run A = layer 0's exchange block t+1 (h0_t), run B = their own block t (h1_{t-1}) — so layer 1's
// step t runs concurrently with layer 0's step t+1 and no input-projection GEMM is needed.
struct FwdCtx {
  RecFwdArgs a;                  // this layer's buffers; a.barrier = this layer's step flags
  const __nv_bfloat16 *hswA;     // run-A exchange buffer (own Hsw, or the layer below's)
  int blkA_off;                  // run-A block = t + blkA_off
  const unsigned int *flagsA;    // producers of run A: wait flagsA[i] >= t + 1 + blkA_off
  int nflagsA;
  const unsigned int *flagsB;    // producers of run B (own layer): wait flagsB[i] >= t + 1
  int nflagsB;
  const float *bias;             // gate-interleaved bias (z init) when G is not pre-filled
  int cta;                       // CTA index within the layer
  int upcA, upcB;                // units per producer CTA of run A / run B (chunk -> flags)
};

JN_DEV void wait_flag_set(const unsigned int *flags, int n, unsigned int v) {
  const int lane = threadIdx.x & 31;
  for (int c = lane; c < n; c += 32) {
    unsigned x;
    do {
      asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(x) : "l"(flags + c * REC_FS) : "memory");
    } while (x < v);
  }
}

// tcgen05.ld .16x32bx2: lanes 0-15 of the warp's TMEM quadrant; threads 0-15 read N columns from
// taddr, threads 16-31 the N columns from taddr + N (both halves of an M = 64 accumulator row).
template <int N>
JN_DEV void tmem_ld_16x2(uint32_t taddr, uint32_t (&r)[N]) {
  static_assert(N == 16 || N == 32, "tmem_ld_16x2");
  if constexpr (N == 32) {
    asm volatile(
        "tcgen05.ld.sync.aligned.16x32bx2.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
        "%11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, "
        "%29, %30, %31}, [%32], 32;"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
          "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
          "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
          "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
  } else {
    asm volatile(
        "tcgen05.ld.sync.aligned.16x32bx2.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
        "%11, %12, %13, %14, %15}, [%16], 16;"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
          "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
  }
}

// Producer warp: wait (every lane polls a share, acquire loads) until flags[p0, p1) >= v.
JN_DEV void wait_flags_acq(const unsigned int *flags, int p0, int p1, unsigned int v) {
  for (int c = p0 + (int)(threadIdx.x & 31); c < p1; c += 32) {
    unsigned x;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(x) : "l"(flags + c * REC_FS) : "memory");
    } while (x < v);
  }
  __syncwarp();  // bar.warp.sync orders every lane's acquire before lane 0's copy issue
}

// M64 (B <= 64): M = 64 MMAs — half the A-operand shared-memory reads of M = 128, whose upper 64
// rows would be padding. The accumulator row i then sits in TMEM lane (i % 16) + 32 (i / 16);
// .16x32bx2 loads give epilogue warp w's lanes 0-15 AND 16-31 batch rows 16 w .. 16 w + 15, the
// low and high half of the CTA's units respectively (all 128 epilogue threads busy).
template <int UPC, bool MASKED, bool M64>
JN_DEV void fwd_body(const FwdCtx &cx, const CUtensorMap *tmWa, const CUtensorMap *tmWb,
                     const RecLayout &ly) {
  constexpr int NG = 4 * UPC;           // gate rows / MMA N / TMEM columns per accumulator
  constexpr int WCH = NG * 128;         // bytes per weight chunk
  constexpr int UH = M64 ? UPC / 2 : UPC;  // units per epilogue thread
  constexpr int GH = 4 * UH;               // gate columns per epilogue thread
  const RecFwdArgs &a = cx.a;
  extern __shared__ uint8_t smem_raw[];
  uint8_t *base = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                              ~uintptr_t(1023));
  const int nk = ly.nk, S = ly.nslots;
  uint8_t *sW = base;
  uint8_t *sA = sW + ly.wbytes;
  uint64_t *full = reinterpret_cast<uint64_t *>(sA + (size_t)S * ly.ch * ly.cb + ly.pad);
  uint64_t *empty = full + S;
  uint64_t *tfull = empty + S;
  uint64_t *wfull = tfull + 1;
  uint64_t *tempty = wfull + 1;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(tempty + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // batch row owned in the epilogue (warps 0-3) and the first of its UH units within the CTA
  const int b = M64 ? 16 * warp + (lane & 15) : (int)threadIdx.x;
  const int uoff = M64 ? (lane >> 4) * UH : 0;
  const int u0 = cx.cta * UPC;
  const int B = a.B, H = a.H;
  const int nkh = (H + 63) / 64;             // chunks of one h block
  const int ldg = 64 * ((4 * H + 63) / 64);  // G pitch (whole 64-column groups)
  const int nu = max(0, min(UPC, H - u0));
  if (a.fail && *a.fail) return;

  if (threadIdx.x == 128) {
    tma_prefetch_desc(tmWa);
    if (tmWb != tmWa) tma_prefetch_desc(tmWb);
    for (int s = 0; s < S; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], REC_NMW); }
    mbar_init(tfull, REC_NMW);
    mbar_init(wfull, 1);
    mbar_init(tempty, 4);
    fence_barrier_init();
  }
  if (warp == 5) tmem_alloc(tmem_slot, 64 * REC_NMW);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  if (threadIdx.x == 128) {
    mbar_expect_tx(wfull, nk * WCH);
    for (int j = 0; j < nk; ++j) {
      if (j < ly.nka) tma_load_2d(sW + j * WCH, tmWa, wfull, j * 64, NG * cx.cta);
      else tma_load_2d(sW + j * WCH, tmWb, wfull, (j - ly.nka) * 64, NG * cx.cta);
    }
  }
  // initial state -> registers, row block 0 of Hs / Cs and exchange block 0
  float hreg[UH], creg[UH];
  const bool row = warp < 4 && b < B;
  // `state = self.state` or zeros when it is still None: Switch/Merge on the device
  const bool is_tensor = a.tag == nullptr || *a.tag == 1;
#pragma unroll
  for (int u = 0; u < UH; ++u) {
    const int gu = u0 + uoff + u;
    hreg[u] = (row && gu < H && is_tensor) ? a.h0[(size_t)b * H + gu] : 0.f;
    creg[u] = (row && gu < H && is_tensor) ? a.c0[(size_t)b * H + gu] : 0.f;
    if (row && gu < H) {
      a.Hs[(size_t)b * a.ldh + gu] = __float2bfloat16_rn(hreg[u]);
      a.Cs[(size_t)b * a.ldh + gu] = creg[u];
    }
  }
  uint8_t *hsw = reinterpret_cast<uint8_t *>(a.Hsw);
  const uint8_t *hswA = reinterpret_cast<const uint8_t *>(cx.hswA);
  // exchange copy: this thread's UH units of row b (UH * 2 bytes, 16-B granule aligned for UH = 8,
  // half a granule for UH = 4) at its swizzled position in chunk (u0 + uoff) / 64
  auto write_x = [&](int blk, const __nv_bfloat16 *hb) {
    const int uc = u0 + uoff;
    uint8_t *chunk = hsw + ((size_t)blk * nkh + (uc >> 6)) * ly.cb;
    const uint32_t g0 = (uint32_t)(uc & 63) >> 3;
    if constexpr (UH % 8 == 0) {
#pragma unroll
      for (int q = 0; q < UH / 8; ++q)
        *reinterpret_cast<uint4 *>(chunk + sw128_off(b, g0 + q)) = reinterpret_cast<const uint4 *>(hb)[q];
    } else {
      static_assert(UH == 4, "write_x");
      *reinterpret_cast<uint2 *>(chunk + sw128_off(b, g0) + (uc & 7) * 2) = *reinterpret_cast<const uint2 *>(hb);
    }
  };
  if (row) {
    __align__(16) __nv_bfloat16 h0b[UH];
#pragma unroll
    for (int u = 0; u < UH; ++u) h0b[u] = __float2bfloat16_rn(uoff + u < nu ? hreg[u] : 0.f);
    write_x(0, h0b);
  }
  const int len_b = (MASKED && row) ? a.lens[b] : 0;
  unsigned int *flags = a.barrier;  // flags[c] = 1 + last step whose h block CTA c has written
  fence_proxy_async_global();
  publish_flag(&flags[cx.cta * REC_FS], (1));
  const int T = a.T_dev ? *a.T_dev : a.T;
  constexpr uint32_t idesc = umma_idesc_bf16(M64 ? 64 : 128, NG, 0, 0);
  const int nacc = min(REC_NMW, nk);  // accumulator tiles in use
  if (warp >= 5) mbar_wait(wfull, 0);

  for (int t = 0; t < T; ++t) {
    if (warp == 4) {
      if (threadIdx.x == 128) PROBE(t, 0);
      // op by op: wait only for the producers of the op's chunks, then issue its copy, so the
      // early chunks' copies and MMAs overlap the arrival of the later producers. Run A = h_{t-1}
      // of this layer (or h_t of the layer below, which runs ahead), run B = this layer's h_{t-1}.
      const uint8_t *srcA = hswA + (size_t)(t + cx.blkA_off) * nkh * ly.cb;
      const uint8_t *srcB = hsw + (size_t)t * nkh * ly.cb;
      // the producers' step flags of an op, its flag target
      auto op_flags = [&](int k, int &p0, int &p1, const unsigned int *&fl, unsigned &tgt) {
        int first, nch;
        op_range(ly, k, first, nch);
        const bool run_a = first < ly.nka;
        const int upc = run_a ? cx.upcA : cx.upcB;
        const int c0 = (run_a ? first : first - ly.nka) * 64;  // first unit of the op
        p0 = c0 / upc;
        p1 = min(run_a ? cx.nflagsA : cx.nflagsB, (c0 + 64 * nch + upc - 1) / upc);
        fl = run_a ? cx.flagsA : cx.flagsB;
        tgt = (run_a ? (unsigned)(t + 1 + cx.blkA_off) : (unsigned)t + 1);
      };
      for (int k = 0; k < ly.nops; ++k) {
        int p0, p1;
        const unsigned int *fl;
        unsigned tgt;
        op_flags(k, p0, p1, fl, tgt);
        wait_flags_acq(fl, p0, p1, tgt);
        if (threadIdx.x == 128) {
          if (k == 0) PROBE(t, 1);
          fence_proxy_async_global();  // generic-proxy writes of the producers -> async-proxy reads
          issue_step(srcA, srcB, ly, sA, full, empty, t, k, k + 1);
        }
        __syncwarp();
      }
      if (threadIdx.x == 128) PROBE(t, 2);
    } else if (warp >= 5) {
      if (elect_one_sync()) {
        mma_step<NG>(ly, sA, sW, WCH, full, empty, tfull, tempty, tmem, idesc, t, warp - 5,
                     (a.dbg && warp == 5) ? a.dbg + ((size_t)blockIdx.x * a.T + t) * 16 : nullptr);
        if (warp == 5) PROBE(t, 4);
      }
      __syncwarp();
    } else {
      // input projection of this step (independent of h_{t-1}): load while the MMA runs. G rows
      // are padded to whole 64-column groups, so every CTA moves whole rows; padding units
      // compute junk that is never published (hb = 0 there)
      float z[GH];
      float *g = a.G + (size_t)(t * B + (row ? b : 0)) * ldg + (size_t)NG * cx.cta + 4 * uoff;
      if (cx.bias) {
#pragma unroll
        for (int q = 0; q < GH; ++q) z[q] = cx.bias[min(NG * cx.cta + 4 * uoff + q, 4 * H - 1)];
      } else {
#pragma unroll
        for (int q = 0; q < GH / 4; ++q) {
          const float4 x = row ? reinterpret_cast<const float4 *>(g)[q] : make_float4(0.f, 0.f, 0.f, 0.f);
          z[4 * q] = x.x; z[4 * q + 1] = x.y; z[4 * q + 2] = x.z; z[4 * q + 3] = x.w;
        }
      }
      mbar_wait(tfull, t & 1);
      if (threadIdx.x == 0) PROBE(t, 5);
      __syncwarp();
      tc_fence_after();
      {
        const uint32_t ta = tmem + ((uint32_t)(warp * 32) << 16);
        for (int w = 0; w < nacc; ++w) {  // an accumulator's loads in flight together, one wait
          if constexpr (M64) {
            uint32_t v[GH];
            tmem_ld_16x2<GH>(ta + w * NG, v);
            tmem_ld_wait();
            tmem_pin(v);
#pragma unroll
            for (int i = 0; i < GH; ++i) z[i] += __uint_as_float(v[i]);
          } else {
            uint32_t v[NG / 32][32];
#pragma unroll
            for (int h = 0; h < NG / 32; ++h) tmem_ld32_nw(ta + w * NG + 32 * h, v[h]);
            tmem_ld_wait();
#pragma unroll
            for (int h = 0; h < NG / 32; ++h)
#pragma unroll
              for (int i = 0; i < 32; ++i) z[32 * h + i] += __uint_as_float(v[h][i]);
          }
        }
      }
      epi_tmem_release(tempty);
      const bool valid = !MASKED || t < len_b;
      __align__(16) __nv_bfloat16 hb[UH];
#pragma unroll
      for (int u = 0; u < UH; ++u) {
        const float ig = sig_f(z[4 * u]), fg = sig_f(z[4 * u + 1]);
        const float gg = tanh_f(z[4 * u + 2]), og = sig_f(z[4 * u + 3]);
        const float c2 = fg * creg[u] + ig * gg;
        const float h2 = og * tanh_f(c2);
        z[4 * u] = ig; z[4 * u + 1] = fg; z[4 * u + 2] = gg; z[4 * u + 3] = og;
        if (valid) { creg[u] = c2; hreg[u] = h2; }
        hb[u] = __float2bfloat16_rn(uoff + u < nu ? hreg[u] : 0.f);
      }
      // critical path first: the exchange copy of h_t, then the step flag; the rest after
      if (row) write_x(t + 1, hb);
      prod_proxy_fence();
      if (threadIdx.x == 0) PROBE(t, 6);
      epi_publish(&flags[cx.cta * REC_FS], (unsigned)t + 2);
      if (threadIdx.x == 0) PROBE(t, 7);
      if (row) {
        const size_t ro = (size_t)((t + 1) * B + b) * a.ldh + u0 + uoff;
#pragma unroll
        for (int q = 0; q < GH / 4; ++q)
          reinterpret_cast<float4 *>(g)[q] = make_float4(z[4 * q], z[4 * q + 1], z[4 * q + 2], z[4 * q + 3]);
        float4 *cd = reinterpret_cast<float4 *>(a.Cs + ro);  // ldh >= 64 * ceil(H / 64)
#pragma unroll
        for (int q = 0; q < UH / 4; ++q) cd[q] = make_float4(creg[4 * q], creg[4 * q + 1], creg[4 * q + 2], creg[4 * q + 3]);
#pragma unroll
        for (int u = 0; u < UH; ++u)  // column H of Hs is the GEMMs' ones column
          if (uoff + u == nu) hb[u] = __float2bfloat16_rn(1.f);
        if constexpr (UH % 8 == 0) {
          uint4 *hd = reinterpret_cast<uint4 *>(a.Hs + ro);
#pragma unroll
          for (int q = 0; q < UH / 8; ++q) hd[q] = reinterpret_cast<const uint4 *>(hb)[q];
        } else {
          *reinterpret_cast<uint2 *>(a.Hs + ro) = *reinterpret_cast<const uint2 *>(hb);
        }
      }
    }
  }
  // final state (committed by the commit phase only if every assumption held)
  if (row) {
#pragma unroll
    for (int u = 0; u < UH; ++u)
      if (uoff + u < nu) {
        a.hT[(size_t)b * H + u0 + uoff + u] = hreg[u];
        a.cT[(size_t)b * H + u0 + uoff + u] = creg[u];
      }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 5) tmem_dealloc(tmem, 64 * REC_NMW);
}

template <bool MASKED, bool M64>
__global__ void __launch_bounds__(REC_THREADS, 1)
    lstm_rec_fwd_kernel(const __grid_constant__ CUtensorMap tmW,  // W_hh interleaved [4H x H], box {64,64}
                        FwdCtx cx, RecLayout ly) {
  cx.cta = blockIdx.x;
  fwd_body<REC_UPC, MASKED, M64>(cx, &tmW, &tmW, ly);
}

// Wavefront: CTAs [0, g0) run layer 0 (16 units each), CTAs [g0, g0 + g1) run layer 1 (8 units).
template <bool MASKED, bool M64>
__global__ void __launch_bounds__(REC_THREADS, 1)
    lstm_rec_fwd_wf_kernel(const __grid_constant__ CUtensorMap tmW0,    // W_hh0, box {64,64}
                           const __grid_constant__ CUtensorMap tmWih1,  // W_ih1, box {64,32}
                           const __grid_constant__ CUtensorMap tmWhh1,  // W_hh1, box {64,32}
                           FwdCtx c0, FwdCtx c1, RecLayout ly0, RecLayout ly1, int g0) {
  if ((int)blockIdx.x < g0) {
    c0.cta = blockIdx.x;
    fwd_body<REC_UPC, MASKED, M64>(c0, &tmW0, &tmW0, ly0);
  } else {
    c1.cta = blockIdx.x - g0;
    fwd_body<REC_UPC / 2, MASKED, M64>(c1, &tmWih1, &tmWhh1, ly1);
  }
}

// ---------------------------------------------------------------------------------- backward
template <bool MASKED>
__global__ void __launch_bounds__(REC_THREADS, 1)
    lstm_rec_bwd_kernel(const __grid_constant__ CUtensorMap tmWT,  // W_hh^T [H x 4H], box {64,16}
                        RecBwdArgs a, RecLayout ly) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t *base = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                              ~uintptr_t(1023));
  const int ldg = 64 * gridDim.x;  // G pitch
  const int nk = ly.nk, S = ly.nslots;
  uint8_t *sW = base;
  uint8_t *sA = sW + ly.wbytes;
  uint64_t *full = reinterpret_cast<uint64_t *>(sA + (size_t)S * ly.ch * ly.cb + ly.pad);
  uint64_t *empty = full + S;
  uint64_t *tfull = empty + S;
  uint64_t *wfull = tfull + 1;
  uint64_t *tempty = wfull + 1;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(tempty + 1);

  const int warp = threadIdx.x >> 5;
  const int b = threadIdx.x;
  const int u0 = blockIdx.x * REC_UPC;
  const int B = a.B, H = a.H;
  if (a.fail && *a.fail) return;

  if (threadIdx.x == 128) {
    tma_prefetch_desc(&tmWT);
    for (int s = 0; s < S; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], REC_NMW); }
    mbar_init(tfull, REC_NMW);
    mbar_init(wfull, 1);
    mbar_init(tempty, 4);
    fence_barrier_init();
  }
  if (warp == 5) tmem_alloc(tmem_slot, 16 * REC_NMW < 32 ? 32 : 16 * REC_NMW);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  if (threadIdx.x == 128) {
    mbar_expect_tx(wfull, nk * 2048);
    for (int j = 0; j < nk; ++j) tma_load_2d(sW + j * 2048, &tmWT, wfull, j * 64, u0);
  }
  const int T = a.T_dev ? *a.T_dev : a.T;
  const bool row = warp < 4 && b < B;
  const int nu = min(REC_UPC, H - u0);
  // While mode: dz rows of the steps beyond the device trip count must not contribute to wgrads
  if (MASKED && row) {
    for (int t = T; t < a.T; ++t)
      for (int q = 0; q < 4 * nu; ++q)
        a.DZ[(size_t)(t * B + b) * a.ldz + (size_t)blockIdx.x * 64 + q] = __float2bfloat16_rn(0.f);
  }
  const int len_b = (MASKED && row) ? a.lens[b] : 0;
  float dcreg[REC_UPC], carry[REC_UPC];
#pragma unroll
  for (int u = 0; u < REC_UPC; ++u) { dcreg[u] = 0.f; carry[u] = 0.f; }
  constexpr uint32_t idesc = umma_idesc_bf16(128, 16, 0, 0);
  const int nacc = min(REC_NMW, nk);
  if (warp >= 5) mbar_wait(wfull, 0);
  unsigned int *flags = a.barrier;  // flags[c] = number of steps CTA c has completed
  uint8_t *dzsw = reinterpret_cast<uint8_t *>(a.DZsw);
  int nmma = 0;                     // steps that issued MMAs (tfull phase)

  for (int t = T - 1; t >= 0; --t) {
    const bool has_next = t + 1 < T;  // dz_{t+1} exists
    const int ti = T - 1 - t;          // probe / ring index
    if (warp == 4) {
      if (has_next) {
        if (threadIdx.x == 128) PROBE(ti, 0);
        wait_flags_warp(flags, gridDim.x, ((unsigned)(T - 1 - t)));  // dz_{t+1} fully written
        if (threadIdx.x == 128) {
          PROBE(ti, 1);
          issue_step(dzsw + (size_t)(t + 1) * nk * ly.cb, nullptr, ly, sA, full, empty, nmma);
          PROBE(ti, 2);
        }
      }
      __syncwarp();
    } else if (warp >= 5) {
      if (has_next && elect_one_sync()) {
        mma_step<16>(ly, sA, sW, 2048, full, empty, tfull, tempty, tmem, idesc, nmma, warp - 5,
                           (a.dbg && warp == 5) ? a.dbg + ((size_t)blockIdx.x * a.T + ti) * 16 : nullptr);
        if (warp == 5) PROBE(ti, 4);
      }
      __syncwarp();
    } else {
      // per-step operands independent of dz_{t+1}: load while the MMA runs
      const size_t r = (size_t)(t * B + (row ? b : 0));
      float gt[64], ct[REC_UPC], cp[REC_UPC], din[REC_UPC];
      {
        // padded pitches (G: 64 per CTA, Cs / dHin: >= 64 * ceil(H / 64)): whole-row vector loads
        const float *g = a.G + r * ldg + (size_t)blockIdx.x * 64;
        const float *pc = a.Cs + (r + B) * a.ldh + u0;
        const float *pp = a.Cs + r * a.ldh + u0;
        const float *pd = a.dHin + r * a.ldd + u0;
        const float4 zero4 = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int k = 0; k < 16; ++k) {
          const float4 x = row ? reinterpret_cast<const float4 *>(g)[k] : zero4;
          gt[4 * k] = x.x; gt[4 * k + 1] = x.y; gt[4 * k + 2] = x.z; gt[4 * k + 3] = x.w;
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const float4 x = row ? reinterpret_cast<const float4 *>(pc)[k] : zero4;
          const float4 y = row ? reinterpret_cast<const float4 *>(pp)[k] : zero4;
          const float4 w = row ? reinterpret_cast<const float4 *>(pd)[k] : zero4;
          ct[4 * k] = x.x; ct[4 * k + 1] = x.y; ct[4 * k + 2] = x.z; ct[4 * k + 3] = x.w;
          cp[4 * k] = y.x; cp[4 * k + 1] = y.y; cp[4 * k + 2] = y.z; cp[4 * k + 3] = y.w;
          din[4 * k] = w.x; din[4 * k + 1] = w.y; din[4 * k + 2] = w.z; din[4 * k + 3] = w.w;
        }
      }
      float dh[REC_UPC];
      if (has_next) {
        mbar_wait(tfull, nmma & 1);
        if (threadIdx.x == 0) PROBE(ti, 5);
        __syncwarp();
        tc_fence_after();
        tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16), dh);
        for (int w = 1; w < nacc; ++w) {
          float d2[REC_UPC];
          tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16) + w * 16, d2);
#pragma unroll
          for (int u = 0; u < REC_UPC; ++u) dh[u] += d2[u];
        }
        epi_tmem_release(tempty);
      } else {
#pragma unroll
        for (int u = 0; u < REC_UPC; ++u) dh[u] = 0.f;
      }
      const bool valid = !MASKED || t < len_b;
      __align__(16) __nv_bfloat16 dzb[64];
#pragma unroll
      for (int u = 0; u < REC_UPC; ++u) {
        const float dhu = dh[u] + din[u] + carry[u];
        const float ig = gt[4 * u], fg = gt[4 * u + 1], gg = gt[4 * u + 2], og = gt[4 * u + 3];
        if (valid) {
          const float tc = tanh_f(ct[u]);
          const float dout = dhu * tc;
          const float dc = dcreg[u] + dhu * og * (1.f - tc * tc);
          const float di = dc * gg, dg = dc * ig, df = dc * cp[u];
          dcreg[u] = dc * fg;
          carry[u] = 0.f;
          dzb[4 * u] = __float2bfloat16_rn(di * ig * (1.f - ig));
          dzb[4 * u + 1] = __float2bfloat16_rn(df * fg * (1.f - fg));
          dzb[4 * u + 2] = __float2bfloat16_rn(dg * (1.f - gg * gg));
          dzb[4 * u + 3] = __float2bfloat16_rn(dout * og * (1.f - og));
        } else {
          carry[u] = dhu;  // masked step: (h, c) passed through unchanged
        }
        if (!valid || u >= nu)
          dzb[4 * u] = dzb[4 * u + 1] = dzb[4 * u + 2] = dzb[4 * u + 3] = __float2bfloat16_rn(0.f);
      }
      if (row) {  // critical path first: the exchange copy of dz_t, then the step flag
        uint8_t *chunk = dzsw + ((size_t)t * nk + blockIdx.x) * ly.cb;
#pragma unroll
        for (int k = 0; k < 8; ++k)
          *reinterpret_cast<uint4 *>(chunk + sw128_off(b, k)) = reinterpret_cast<const uint4 *>(dzb)[k];
      }
      prod_proxy_fence();
      if (threadIdx.x == 0) PROBE(ti, 6);
      epi_publish(&flags[blockIdx.x * REC_FS], (unsigned)(T - t));
      if (threadIdx.x == 0) PROBE(ti, 7);
      if (row) {  // ldz >= 64 * grid: padding columns get the zeros computed for the padding units
        uint4 *d4 = reinterpret_cast<uint4 *>(a.DZ + r * a.ldz + (size_t)blockIdx.x * 64);
#pragma unroll
        for (int k = 0; k < 8; ++k) d4[k] = reinterpret_cast<const uint4 *>(dzb)[k];
      }
    }
    if (has_next) ++nmma;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 5) tmem_dealloc(tmem, 16 * REC_NMW < 32 ? 32 : 16 * REC_NMW);
}

// ------------------------------------------------------------------ backward, K-split clusters
// dh_t = W_hh^T dz_{t+1} has K = 4H: every CTA of the plain backward kernel streams the WHOLE of
// dz_{t+1} (B x 4H bf16, 328 KB at C2) through shared memory each step and issues 4H/16 MMAs —
// the step is bound by that stream and by the MMA issue rate. Here a cluster of KS_CL CTAs owns
// KS_UPC = 64 units; CTA r of the cluster holds W_hh^T[units x K-slice r] and streams only dz
// columns of K-slice r (1/KS_CL of the data, 1/KS_CL of the MMAs, N = 64). The KS_CL partial dh
// tiles are exchanged through distributed shared memory: CTA r keeps the 16 units it owns
// (u0 = 16 * blockIdx.x, the same ownership, dz exchange layout and flags as the plain kernel)
// and receives their partials from its KS_CL-1 peers, summed in a fixed order (deterministic).
constexpr int KS_CL = 4;
template <int UPC>
struct KsCfg {
  static constexpr int CUNITS = KS_CL * UPC;              // units per cluster = MMA N
  static constexpr int WCH = CUNITS * 128;                 // bytes per resident weight chunk
  static constexpr int TILE = 64 * UPC * 4;                // one peer's partial tile [row < 64][UPC] fp32
  static constexpr int RED = (2 * (KS_CL - 1) + KS_CL) * TILE;  // red[parity][sender] + stage[group]
  static constexpr int HU = UPC / 2;                       // units per epilogue thread
};

// One backward-recurrence role (a layer). K space of a step: run A = the layer above's dz_t
// (wavefront layer 0 only: dX_t = W_ih^T dz_t of the layer above, folded into this layer's dh
// instead of a separate dgrad GEMM), then run B = this layer's dz_{t+1}.
struct KsCtx {
  RecBwdArgs a;                  // this layer; a.barrier = its step flags, a.DZsw its exchange buffer
  int base;                      // first CTA of this layer in the launch (multiple of KS_CL)
  int nk_all;                    // chunks of one dz block = ceil(4H / 64)
  const __nv_bfloat16 *dzswA;    // run A: the layer above's exchange buffer (block t)
  const unsigned int *flagsA;    // its step flags (16 units = one chunk per producer CTA)
  int nkA;                       // chunks of run A (0: none)
};

template <int UPC, bool MASKED>
JN_DEV void ks_body(const KsCtx &cx, const CUtensorMap *tmWa, const CUtensorMap *tmWb, const RecLayout &ly) {
  using C = KsCfg<UPC>;
  constexpr int HU = C::HU;
  const RecBwdArgs &a = cx.a;
  extern __shared__ uint8_t smem_raw[];
  uint8_t *base = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                              ~uintptr_t(1023));
  const int nkr = ly.nk, S = ly.nslots;
  uint8_t *sW = base;
  uint8_t *sA = sW + ly.wbytes;
  float *red = reinterpret_cast<float *>(sA + (size_t)S * ly.ch * ly.cb + ly.pad);  // [2][CL-1][64][UPC]
  float *stage = red + 2 * (KS_CL - 1) * 64 * UPC;                                // [CL][64][UPC]
  uint64_t *full = reinterpret_cast<uint64_t *>(reinterpret_cast<uint8_t *>(red) + C::RED);
  uint64_t *empty = full + S;
  uint64_t *tfull = empty + S;
  uint64_t *wfull = tfull + 1;
  uint64_t *tempty = wfull + 1;
  uint64_t *redfull = tempty + 1;  // [2], one per parity
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(redfull + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int lcta = blockIdx.x - cx.base;  // CTA index within the layer
  const int rank = (int)cluster_ctarank(), cl = lcta / KS_CL;
  const int nkA = cx.nkA, nk_all = cx.nk_all, nkt = nkA + nk_all;
  const int s0 = rank * nkr, nks = max(0, min(nkr, nkt - s0));  // my K-slice
  const int na = max(0, min(s0 + nks, nkA) - s0);               // ... of which run A
  const int nb = nks - na, b0 = max(0, s0 - nkA);               // ... and run B (from chunk b0)
  const int B = a.B, H = a.H;
  const int u0 = UPC * lcta;
  // a CTA whose gate columns lie inside the dz chunk grid publishes its slice every step (zeros
  // for units >= H): consumers wait on every producer of a chunk
  const bool active = 4 * u0 < 64 * nk_all;
  const int ldg = 64 * nk_all;  // G pitch
  // epilogue mapping: thread q owns batch row q % 64 and units HU (q / 64) .. + HU - 1
  const int eb = threadIdx.x & 63, eh = (threadIdx.x >> 6) & 1;
  const int ue = u0 + HU * eh;                    // first unit of my epilogue share
  const int nuh = max(0, min(HU, H - ue));        // real units of my share
  if (a.fail && *a.fail) return;  // uniform: every CTA reads the same flag

  if (threadIdx.x == 128) {
    if (nkA) tma_prefetch_desc(tmWa);
    tma_prefetch_desc(tmWb);
    for (int s = 0; s < S; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], REC_NMW); }
    mbar_init(tfull, REC_NMW);
    mbar_init(wfull, 1);
    mbar_init(tempty, 4);
    mbar_init(&redfull[0], 1);  // the owner's arrive.expect_tx; the peers' bulk copies complete_tx
    mbar_init(&redfull[1], 1);
    fence_barrier_init();
  }
  if (warp == 5) tmem_alloc(tmem_slot, 64 * REC_NMW);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  cluster_sync_all();  // peers' barriers are initialised before any bulk copy targets them
  const uint32_t tmem = *tmem_slot;
  if (threadIdx.x == 128 && nks > 0) {
    mbar_expect_tx(wfull, nks * C::WCH);
    for (int j = 0; j < nks; ++j) {
      const int g = s0 + j;
      if (g < nkA) tma_load_2d(sW + j * C::WCH, tmWa, wfull, g * 64, C::CUNITS * cl);
      else tma_load_2d(sW + j * C::WCH, tmWb, wfull, (g - nkA) * 64, C::CUNITS * cl);
    }
  }
  const int T = a.T_dev ? *a.T_dev : a.T;
  const bool row = warp < 4 && eb < B && active;
  if (MASKED && row) {  // While mode: dz rows beyond the device trip count stay out of the wgrads
    for (int t = T; t < a.T; ++t)
      for (int q = 0; q < 4 * nuh; ++q)
        a.DZ[(size_t)(t * B + eb) * a.ldz + 4 * (size_t)ue + q] = __float2bfloat16_rn(0.f);
  }
  const int len_b = (MASKED && row) ? a.lens[eb] : 0;
  float dcreg[HU], carry[HU];
#pragma unroll
  for (int u = 0; u < HU; ++u) { dcreg[u] = 0.f; carry[u] = 0.f; }
  constexpr uint32_t idesc = umma_idesc_bf16(64, C::CUNITS, 0, 0);  // B <= 64: M = 64
  if (warp >= 5 && nks > 0) mbar_wait(wfull, 0);
  unsigned int *flags = a.barrier;  // flags[c] = number of steps CTA c of this layer has completed
  uint8_t *dzsw = reinterpret_cast<uint8_t *>(a.DZsw);
  const uint8_t *dzswA = reinterpret_cast<const uint8_t *>(cx.dzswA);
  int q_ring = 0;  // ring position (ops), producer and MMA warps advance it identically
  int nm = 0;      // steps in which this CTA issued MMAs (tfull / tempty phase)
  int nx = 0;      // exchange steps (redfull phase; uniform across the cluster)

  for (int t = T - 1; t >= 0; --t) {
    const int ti = T - 1 - t;
    const bool has_b = t + 1 < T;                 // dz_{t+1} of this layer exists
    const int nbs = has_b ? nb : 0;               // run-B chunks of my slice this step
    const int nstep = na + nbs;                   // chunks I multiply this step
    const bool has_x = nkA > 0 || has_b;          // the cluster exchanges partials this step
    RecLayout lys = ly;
    lys.nk = nstep;
    lys.nka = na;
    lys.nops = (na + ly.ch - 1) / ly.ch + (nbs + ly.ch - 1) / ly.ch;
    if (warp == 4) {
      if (nstep > 0) {
        if (threadIdx.x == 128) PROBE(ti, 0);
        const uint8_t *srcA = dzswA ? dzswA + ((size_t)t * nk_all + s0) * ly.cb : nullptr;
        const uint8_t *srcB = dzsw + ((size_t)(t + 1) * nk_all + b0) * ly.cb;
        const int opsA = (na + ly.ch - 1) / ly.ch;
        if (na > 0) {  // the layer above's dz_t: producer CTA g of that layer per chunk g
          for (int c = s0 + lane; c < s0 + na; c += 32) {
            unsigned x;
            do {
              asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(x) : "l"(cx.flagsA + c * REC_FS) : "memory");
            } while (x < ((unsigned)(T - t)));
          }
          __syncwarp();
          asm volatile("fence.acq_rel.gpu;" ::: "memory");
          fence_proxy_async_global();
          if (threadIdx.x == 128) issue_step(srcA, srcB, lys, sA, full, empty, 0, 0, opsA, q_ring);
        }
        if (nbs > 0) {  // this layer's dz_{t+1}: chunk j is produced by CTAs [16 j / UPC, 16 (j + 1) / UPC)
          const int p0 = b0 * 16 / UPC, p1 = (b0 + nbs) * 16 / UPC;
          for (int c = p0 + lane; c < p1; c += 32) {
            unsigned x;
            do {
              asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(x) : "l"(flags + c * REC_FS) : "memory");
            } while (x < ((unsigned)(T - 1 - t)));
          }
          __syncwarp();
          asm volatile("fence.acq_rel.gpu;" ::: "memory");
          fence_proxy_async_global();
          if (threadIdx.x == 128) issue_step(srcA, srcB, lys, sA, full, empty, 0, opsA, 1 << 30, q_ring);
        }
        if (threadIdx.x == 128) PROBE(ti, 2);
      }
      __syncwarp();
    } else if (warp >= 5) {
      if (nstep > 0 && elect_one_sync()) {
        mma_step<C::CUNITS>(lys, sA, sW, C::WCH, full, empty, tfull, tempty, tmem, idesc, nm, warp - 5,
                            (a.dbg && warp == 5) ? a.dbg + ((size_t)blockIdx.x * a.T + ti) * 16 : nullptr,
                            q_ring);
        if (warp == 5) PROBE(ti, 4);
      }
      __syncwarp();
    } else {
      // per-step operands of my (row, HU units), independent of the dz's: load while the MMA runs
      const size_t r = (size_t)(t * B + (row ? eb : 0));
      float gt[4 * HU], ct[HU], cp[HU], din[HU];
      {
        const float *g = a.G + r * ldg + 4 * (size_t)ue;
        const float *pc = a.Cs + (r + B) * a.ldh + ue;
        const float *pp = a.Cs + r * a.ldh + ue;
        const float *pd = a.dHin ? a.dHin + r * a.ldd + ue : nullptr;
        const float4 zero4 = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int k = 0; k < HU; ++k) {
          const float4 x = row ? reinterpret_cast<const float4 *>(g)[k] : zero4;
          gt[4 * k] = x.x; gt[4 * k + 1] = x.y; gt[4 * k + 2] = x.z; gt[4 * k + 3] = x.w;
        }
#pragma unroll
        for (int k = 0; k < HU / 4; ++k) {
          const float4 x = row ? reinterpret_cast<const float4 *>(pc)[k] : zero4;
          const float4 y = row ? reinterpret_cast<const float4 *>(pp)[k] : zero4;
          const float4 w = (row && pd) ? reinterpret_cast<const float4 *>(pd)[k] : zero4;
          ct[4 * k] = x.x; ct[4 * k + 1] = x.y; ct[4 * k + 2] = x.z; ct[4 * k + 3] = x.w;
          cp[4 * k] = y.x; cp[4 * k + 1] = y.y; cp[4 * k + 2] = y.z; cp[4 * k + 3] = y.w;
          din[4 * k] = w.x; din[4 * k + 1] = w.y; din[4 * k + 2] = w.z; din[4 * k + 3] = w.w;
        }
      }
      float dh[HU];
#pragma unroll
      for (int u = 0; u < HU; ++u) dh[u] = 0.f;
      if (has_x) {
        const int par = nx & 1;
        // partial dh tiles leave straight from registers: st.async of each 16-B piece into the
        // peer's red[par] slot, completing on the peer's redfull[par] (no staging, proxy fence or
        // single-thread bulk issue); only this CTA's own partial goes through `stage`
        static_assert(REC_NMW == 1, "one accumulator");
        if (threadIdx.x == 0) mbar_expect_tx(&redfull[par], (KS_CL - 1) * C::TILE);
        if (nstep > 0) {
          mbar_wait(tfull, nm & 1);
          if (threadIdx.x == 0) PROBE(ti, 5);
          __syncwarp();
          tc_fence_after();
        }
        epi_bar();  // every thread summed the previous step's stage
        {  // M = 64: accumulator row i in TMEM lane (i % 16) + 32 (i / 16); lanes 16-31 idle
          const int srow = 16 * warp + lane;
          const uint32_t ta = tmem + ((uint32_t)(warp * 32) << 16);
          uint32_t r[KS_CL][UPC];
          if (nstep > 0) {
#pragma unroll
            for (int p = 0; p < KS_CL; ++p) {
              if constexpr (UPC == 16) tmem_ld16_nw(ta + UPC * p, r[p]);
              else tmem_ld8_nw(ta + UPC * p, r[p]);
            }
            tmem_ld_wait();
#pragma unroll
            for (int p = 0; p < KS_CL; ++p) tmem_pin(r[p]);
          } else {
#pragma unroll
            for (int p = 0; p < KS_CL; ++p)
#pragma unroll
              for (int i = 0; i < UPC; ++i) r[p][i] = 0u;
          }
          if (nstep > 0) epi_tmem_release(tempty);
          if (lane < 16) {
#pragma unroll
            for (int p = 0; p < KS_CL; ++p) {
              const float *v = reinterpret_cast<const float *>(r[p]);
              if (p == rank) {
                float4 *dst = reinterpret_cast<float4 *>(stage + ((size_t)p * 64 + srow) * UPC);
#pragma unroll
                for (int q = 0; q < UPC / 4; ++q) dst[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
              } else {
                const int slot = rank < p ? rank : rank - 1;  // my sender slot inside peer p
                const uint32_t dst =
                    mapa_shared(smem_u32(red + ((size_t)(par * (KS_CL - 1) + slot) * 64 + srow) * UPC), p);
                const uint32_t pbar = mapa_shared(smem_u32(&redfull[par]), p);
#pragma unroll
                for (int q = 0; q < UPC / 4; ++q)
                  st_async_v4(dst + 16 * q, v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3], pbar);
              }
            }
          }
        }
        if (threadIdx.x == 0) PROBE(ti, 3);
        epi_bar();  // own partial rows visible to every summing thread
        if (threadIdx.x == 0) PROBE(ti, 14);
        mbar_wait_cluster(&redfull[par], (nx >> 1) & 1);
        if (threadIdx.x == 0) PROBE(ti, 15);
#pragma unroll
        for (int p = 0; p < KS_CL; ++p) {  // fixed order over the K-slices: deterministic
          const float *src = p == rank ? stage + (size_t)rank * 64 * UPC
                                       : red + (size_t)(par * (KS_CL - 1) + (p < rank ? p : p - 1)) * 64 * UPC;
          const float4 *s4 = reinterpret_cast<const float4 *>(src + (size_t)eb * UPC + HU * eh);
#pragma unroll
          for (int q = 0; q < HU / 4; ++q) {
            const float4 v = s4[q];
            dh[4 * q] += v.x; dh[4 * q + 1] += v.y; dh[4 * q + 2] += v.z; dh[4 * q + 3] += v.w;
          }
        }
      }
      const bool valid = !MASKED || t < len_b;
      __align__(16) __nv_bfloat16 dzb[4 * HU];
#pragma unroll
      for (int u = 0; u < HU; ++u) {
        const float dhu = dh[u] + din[u] + carry[u];
        const float ig = gt[4 * u], fg = gt[4 * u + 1], gg = gt[4 * u + 2], og = gt[4 * u + 3];
        if (valid) {
          const float tc = tanh_f(ct[u]);
          const float dout = dhu * tc;
          const float dc = dcreg[u] + dhu * og * (1.f - tc * tc);
          const float di = dc * gg, dg = dc * ig, df = dc * cp[u];
          dcreg[u] = dc * fg;
          carry[u] = 0.f;
          dzb[4 * u] = __float2bfloat16_rn(di * ig * (1.f - ig));
          dzb[4 * u + 1] = __float2bfloat16_rn(df * fg * (1.f - fg));
          dzb[4 * u + 2] = __float2bfloat16_rn(dg * (1.f - gg * gg));
          dzb[4 * u + 3] = __float2bfloat16_rn(dout * og * (1.f - og));
        } else {
          carry[u] = dhu;
        }
        if (!valid || u >= nuh)
          dzb[4 * u] = dzb[4 * u + 1] = dzb[4 * u + 2] = dzb[4 * u + 3] = __float2bfloat16_rn(0.f);
      }
      if (row) {  // exchange copy: gate columns 4 ue .. 4 ue + 4 HU of row eb
        const int col = 4 * ue;
        uint8_t *chunk = dzsw + ((size_t)t * nk_all + (col >> 6)) * ly.cb;
        const int g0 = (col & 63) >> 3;
#pragma unroll
        for (int k = 0; k < HU / 2; ++k)
          *reinterpret_cast<uint4 *>(chunk + sw128_off(eb, g0 + k)) = reinterpret_cast<const uint4 *>(dzb)[k];
      }
      prod_proxy_fence();
      if (threadIdx.x == 0) PROBE(ti, 6);
      if (active) epi_publish(&flags[lcta * REC_FS], (unsigned)(T - t));
      if (threadIdx.x == 0) PROBE(ti, 7);
      if (row) {
        uint4 *d4 = reinterpret_cast<uint4 *>(a.DZ + r * a.ldz + 4 * (size_t)ue);
#pragma unroll
        for (int k = 0; k < HU / 2; ++k) d4[k] = reinterpret_cast<const uint4 *>(dzb)[k];
      }
    }
    if (nstep > 0) ++nm;
    if (has_x) ++nx;
    q_ring += lys.nops;
  }
  if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();  // no CTA leaves while a peer may still address its shared memory
  if (warp == 5) tmem_dealloc(tmem, 64 * REC_NMW);
}

template <bool MASKED>
__global__ void __launch_bounds__(REC_THREADS, 1)
    lstm_rec_bwd_ks_kernel(const __grid_constant__ CUtensorMap tmWT,  // W_hh^T [H x 4H], box {64,64}
                           KsCtx cx, RecLayout ly) {
  ks_body<REC_UPC, MASKED>(cx, &tmWT, &tmWT, ly);
}

// Backward wavefront of a 2-layer stack: CTAs [0, g1) run layer 1 (16 units), CTAs [g1, g1 + g0)
// layer 0 (8 units), whose K space starts with layer 1's dz_t (W_ih1^T fused, no dgrad GEMM).
template <bool MASKED>
__global__ void __launch_bounds__(REC_THREADS, 1)
    lstm_rec_bwd_wf_kernel(const __grid_constant__ CUtensorMap tmWT1,   // W_hh1^T, box {64,64}
                           const __grid_constant__ CUtensorMap tmWihT1, // W_ih1^T, box {64,32}
                           const __grid_constant__ CUtensorMap tmWT0,   // W_hh0^T, box {64,32}
                           KsCtx c1, KsCtx c0, RecLayout ly1, RecLayout ly0) {
  if ((int)blockIdx.x < c0.base) ks_body<REC_UPC, MASKED>(c1, &tmWT1, &tmWT1, ly1);
  else ks_body<REC_UPC / 2, MASKED>(c0, &tmWihT1, &tmWT0, ly0);
}

// ---------------------------------------------------------------------------------- host
static RecLayout layout(int wbytes, int nk, int B, int extra = 0, bool m64 = false) {
  RecLayout l;
  l.nk = nk;
  l.wbytes = (wbytes + 1023) & ~1023;
  l.bp = (B + 7) & ~7;
  l.cb = l.bp * 128;
  l.pad = std::max(0, (m64 ? 64 : 128) - l.bp) * 128;  // rows an MMA reads past the last chunk
  const int avail = SMEM_BUDGET - l.wbytes - l.pad - extra - 1024 /*barriers*/;
  const int max_chunks = avail / l.cb;  // chunks that fit in flight
  // two ring slots (TMA of op k+1 overlaps the MMAs of op k); a whole step in flight if it fits
  l.nslots = 2;
  l.ch = std::min((nk + 1) / 2, max_chunks / 2);
  l.ch = std::max(1, std::min(l.ch, 256));
  if (const char *e = getenv("JANUS_REC_CH")) {  // experiment knob: chunks per TMA op
    const int ch = atoi(e);
    if (ch >= 1) {
      l.ch = std::min(ch, nk);
      l.nslots = std::max(2, std::min(REC_MAX_SLOTS, max_chunks / l.ch));
    }
  }
  l.nka = nk;
  l.nops = (nk + l.ch - 1) / l.ch;
  return l;
}
static int smem_of(const RecLayout &l, int extra = 0) {
  return 1024 + l.wbytes + l.nslots * l.ch * l.cb + l.pad + extra + 1024;
}

static size_t xchg_block(int cols, int B) { return (size_t)((cols + 63) / 64) * ((B + 7) & ~7) * 128; }
size_t rec_hsw_bytes(int H, int B, int T) { return (size_t)(T + 1) * xchg_block(H, B); }
size_t rec_dzsw_bytes(int H, int B, int T) { return (size_t)T * xchg_block(4 * H, B); }

int rec_grid(int H) { return (H + REC_UPC - 1) / REC_UPC; }

static cudaError_t coop_launch(const void *fn, int grid, int smem, void **args, cudaStream_t st) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(REC_THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;
  at[0].val.cooperative = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelExC(&cfg, fn, args);
}

cudaError_t lstm_rec_fwd(const RecFwdArgs &a, const __nv_bfloat16 *Whh, int ldw, bool masked,
                         cudaStream_t st) {
  if (a.B > 128 || a.B < 1) return cudaErrorInvalidValue;
  const int nk = (a.H + 63) / 64;
  RecLayout ly = layout(nk * 8192, nk, a.B, 0, a.B <= 64);
  if (ly.ch < 1 || smem_of(ly) > 232448) return cudaErrorInvalidValue;
  if (!a.Hsw) return cudaErrorInvalidValue;
  CUtensorMap tmW;
  if (!make_tmap_bf16(&tmW, Whh, a.H, 4ull * a.H, ldw, 64)) return cudaErrorInvalidValue;
  const int smem = smem_of(ly);
  const bool m64 = a.B <= 64;
  const void *fn = masked ? (m64 ? (const void *)lstm_rec_fwd_kernel<true, true> : (const void *)lstm_rec_fwd_kernel<true, false>)
                          : (m64 ? (const void *)lstm_rec_fwd_kernel<false, true> : (const void *)lstm_rec_fwd_kernel<false, false>);
  cudaError_t e = set_smem_once((const void *)fn, smem);
  if (e != cudaSuccess) return e;
  FwdCtx cx = {};
  cx.a = a;
  cx.hswA = a.Hsw;
  cx.blkA_off = 0;
  cx.flagsA = a.barrier;
  cx.nflagsA = rec_grid(a.H);
  cx.upcA = cx.upcB = REC_UPC;
  void *args[] = {&tmW, &cx, &ly};
  return coop_launch(fn, rec_grid(a.H), smem, args, st);
}

int rec_fwd_wf_grid(int H) { return rec_grid(H) + (H + REC_UPC / 2 - 1) / (REC_UPC / 2); }

cudaError_t lstm_rec_fwd_wavefront(const RecFwdArgs &a0, const RecFwdArgs &a1, const __nv_bfloat16 *Whh0,
                                   const __nv_bfloat16 *Wih1, const __nv_bfloat16 *Whh1, int ldw,
                                   const float *bias1_il, bool masked, cudaStream_t st) {
  if (a0.B > 128 || a0.B < 1 || a0.H != a1.H || !a0.Hsw || !a1.Hsw) return cudaErrorInvalidValue;
  const int H = a0.H, nkh = (H + 63) / 64;
  RecLayout ly0 = layout(nkh * 8192, nkh, a0.B, 0, a0.B <= 64);
  RecLayout ly1 = layout(2 * nkh * 4096, 2 * nkh, a0.B, 0, a0.B <= 64);
  ly1.nka = nkh;
  ly1.nops = (nkh + ly1.ch - 1) / ly1.ch * 2;
  const int smem = std::max(smem_of(ly0), smem_of(ly1));
  if (ly0.ch < 1 || ly1.ch < 1 || smem > 232448) return cudaErrorInvalidValue;
  CUtensorMap tm0, tmi, tmh;
  if (!make_tmap_bf16(&tm0, Whh0, H, 4ull * H, ldw, 64) || !make_tmap_bf16(&tmi, Wih1, H, 4ull * H, ldw, 32) ||
      !make_tmap_bf16(&tmh, Whh1, H, 4ull * H, ldw, 32))
    return cudaErrorInvalidValue;
  const bool m64 = a0.B <= 64;
  const void *fn = masked ? (m64 ? (const void *)lstm_rec_fwd_wf_kernel<true, true> : (const void *)lstm_rec_fwd_wf_kernel<true, false>)
                          : (m64 ? (const void *)lstm_rec_fwd_wf_kernel<false, true> : (const void *)lstm_rec_fwd_wf_kernel<false, false>);
  cudaError_t e = set_smem_once((const void *)fn, smem);
  if (e != cudaSuccess) return e;
  const int g0 = rec_grid(H), g1 = rec_fwd_wf_grid(H) - g0;
  FwdCtx c0 = {}, c1 = {};
  c0.a = a0;
  c0.hswA = a0.Hsw;
  c0.flagsA = a0.barrier;
  c0.nflagsA = g0;
  c1.a = a1;
  c1.hswA = a0.Hsw;  // h0_t = layer 0's exchange block t + 1
  c1.blkA_off = 1;
  c1.flagsA = a0.barrier;
  c1.nflagsA = g0;
  c1.flagsB = a1.barrier;
  c1.nflagsB = g1;
  c1.bias = bias1_il;
  c0.upcA = c0.upcB = REC_UPC;
  c1.upcA = REC_UPC;       // run A: layer 0's CTAs
  c1.upcB = REC_UPC / 2;   // run B: layer 1's CTAs
  int g0_ = g0;
  void *args[] = {&tm0, &tmi, &tmh, &c0, &c1, &ly0, &ly1, &g0_};
  return coop_launch(fn, g0 + g1, smem, args, st);
}

static cudaError_t lstm_rec_bwd_plain(const RecBwdArgs &a, const __nv_bfloat16 *WhhT, int ldwt,
                                      bool masked, cudaStream_t st) {
  const int nk = (4 * a.H + 63) / 64;
  RecLayout ly = layout(nk * 2048, nk, a.B);
  if (ly.ch < 1 || smem_of(ly) > 232448) return cudaErrorInvalidValue;
  CUtensorMap tmWT;
  if (!make_tmap_bf16(&tmWT, WhhT, 4ull * a.H, a.H, ldwt, 16)) return cudaErrorInvalidValue;
  const int smem = smem_of(ly);
  const void *fn = masked ? (const void *)lstm_rec_bwd_kernel<true> : (const void *)lstm_rec_bwd_kernel<false>;
  cudaError_t e = set_smem_once((const void *)fn, smem);
  if (e != cudaSuccess) return e;
  RecBwdArgs aa = a;
  void *args[] = {&tmWT, &aa, &ly};
  return coop_launch(fn, rec_grid(a.H), smem, args, st);
}

static cudaError_t cluster_launch(const void *fn, int grid, int smem, void **args, cudaStream_t st) {
  cudaError_t e = set_smem_once((const void *)fn, smem);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(REC_THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = KS_CL;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  // The CTAs wait on each other's step flags, so all clusters must be resident at once. A
  // cooperative launch would guarantee it but cannot be combined with clusters under the
  // profiler's replay; check instead that the device can hold every cluster simultaneously
  // (one CTA per SM; the launch runs alone on the stream).
  static const void *c_fn[8];
  static int c_smem[8], c_max[8], c_n = 0;
  int max_clusters = -1;
  for (int i = 0; i < c_n; ++i)
    if (c_fn[i] == fn && c_smem[i] == smem) max_clusters = c_max[i];
  if (max_clusters < 0) {  // occupancy query once per kernel and size (host cost)
    if (cudaOccupancyMaxActiveClusters(&max_clusters, fn, &cfg) != cudaSuccess) max_clusters = 0;
    if (c_n < 8) { c_fn[c_n] = fn; c_smem[c_n] = smem; c_max[c_n] = max_clusters; ++c_n; }
  }
  if (grid / KS_CL > max_clusters) return cudaErrorCooperativeLaunchTooLarge;
  return cudaLaunchKernelExC(&cfg, fn, args);
}

template <int UPC>
static RecLayout ks_layout(int nkt, int B) {
  const int nkr = (nkt + KS_CL - 1) / KS_CL;
  return layout(nkr * KsCfg<UPC>::WCH, nkr, B, KsCfg<UPC>::RED, true);  // B <= 64: M = 64 MMAs
}

static int ks_grid(int H, int upc) { return KS_CL * ((H + KS_CL * upc - 1) / (KS_CL * upc)); }

static cudaError_t lstm_rec_bwd_ks(const RecBwdArgs &a, const __nv_bfloat16 *WhhT, int ldwt, bool masked,
                                   cudaStream_t st) {
  const int nk_all = (4 * a.H + 63) / 64;
  RecLayout ly = ks_layout<REC_UPC>(nk_all, a.B);
  const int smem = smem_of(ly, KsCfg<REC_UPC>::RED);
  if (ly.ch < 1 || smem > 232448) return cudaErrorInvalidValue;
  CUtensorMap tmWT;
  if (!make_tmap_bf16(&tmWT, WhhT, 4ull * a.H, a.H, ldwt, 64)) return cudaErrorInvalidValue;
  const void *fn = masked ? (const void *)lstm_rec_bwd_ks_kernel<true> : (const void *)lstm_rec_bwd_ks_kernel<false>;
  KsCtx cx = {};
  cx.a = a;
  cx.base = 0;
  cx.nk_all = nk_all;
  void *args[] = {&tmWT, &cx, &ly};
  return cluster_launch(fn, ks_grid(a.H, REC_UPC), smem, args, st);
}

int rec_bwd_wf_grid(int H) { return ks_grid(H, REC_UPC) + ks_grid(H, REC_UPC / 2); }

cudaError_t lstm_rec_bwd_wavefront(const RecBwdArgs &a1, const RecBwdArgs &a0, const __nv_bfloat16 *WhhT1,
                                   const __nv_bfloat16 *WihT1, const __nv_bfloat16 *WhhT0, int ldwt,
                                   bool masked, cudaStream_t st) {
  if (a1.B > 64 || a1.B < 1 || a1.H != a0.H || !a1.DZsw || !a0.DZsw) return cudaErrorInvalidValue;
  const int H = a1.H, nk_all = (4 * H + 63) / 64;
  RecLayout ly1 = ks_layout<REC_UPC>(nk_all, a1.B);
  RecLayout ly0 = ks_layout<REC_UPC / 2>(2 * nk_all, a1.B);
  const int smem = std::max(smem_of(ly1, KsCfg<REC_UPC>::RED), smem_of(ly0, KsCfg<REC_UPC / 2>::RED));
  if (ly1.ch < 1 || ly0.ch < 1 || smem > 232448) return cudaErrorInvalidValue;
  CUtensorMap t1, ti, t0;
  if (!make_tmap_bf16(&t1, WhhT1, 4ull * H, H, ldwt, 64) || !make_tmap_bf16(&ti, WihT1, 4ull * H, H, ldwt, 32) ||
      !make_tmap_bf16(&t0, WhhT0, 4ull * H, H, ldwt, 32))
    return cudaErrorInvalidValue;
  const void *fn = masked ? (const void *)lstm_rec_bwd_wf_kernel<true> : (const void *)lstm_rec_bwd_wf_kernel<false>;
  KsCtx c1 = {}, c0 = {};
  c1.a = a1;
  c1.base = 0;
  c1.nk_all = nk_all;
  c0.a = a0;
  c0.base = ks_grid(H, REC_UPC);
  c0.nk_all = nk_all;
  c0.dzswA = a1.DZsw;
  c0.flagsA = a1.barrier;
  c0.nkA = nk_all;
  void *args[] = {&t1, &ti, &t0, &c1, &c0, &ly1, &ly0};
  return cluster_launch(fn, rec_bwd_wf_grid(H), smem, args, st);
}

cudaError_t lstm_rec_bwd(const RecBwdArgs &a, const __nv_bfloat16 *WhhT, int ldwt, bool masked,
                         cudaStream_t st) {
  if (a.B > 128 || a.B < 1) return cudaErrorInvalidValue;
  if (!a.DZsw) return cudaErrorInvalidValue;
  const char *e = getenv("JANUS_REC_BWD");
  // the K-split kernel exchanges partial tiles of at most 64 batch rows
  if ((e && e[0] == 'p') || a.B > 64) return lstm_rec_bwd_plain(a, WhhT, ldwt, masked, st);
  const cudaError_t r = lstm_rec_bwd_ks(a, WhhT, ldwt, masked, st);
  if (r == cudaErrorCooperativeLaunchTooLarge) {
    (void)cudaGetLastError();
    return lstm_rec_bwd_plain(a, WhhT, ldwt, masked, st);
  }
  return r;
}

}  // namespace jk
