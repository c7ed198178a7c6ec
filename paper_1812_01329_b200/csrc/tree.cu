// tree.cu — level-batched TreeLSTM training step (config C3).
//
// The TreeNN program recurses through InvokeOp (P:316 fn6: "recursion-based
// implementation"). Under the TREE_BINARY assumption (every node a leaf or a binary node whose
// children precede it in the same tree) the recursion is flattened into levels (reading Q8:
// level = height, stable by node id) — exactly the parallelism +PARL exploits "in multiple
// independent tree nodes" — and runs on the device:
//   guard (AssertOp over the forest) -> schedule (stable counting sort by height) ->
//   forward: one cooperative launch walks leaf level + internal levels with grid barriers; each
//            level is a tcgen05 GEMM (rows = the level's nodes, gate-interleaved weight tiles) with
//            the cell update fused in the TMEM epilogue, scattering h / c into the parent's
//            staging row (each child has exactly one parent: no atomics) ->
//   root classifier + xent -> backward: one cooperative launch walks the levels top-down.
// Gate-interleaved rows: U_il row 5u+g = U row g*H+u (g = i, f_l, f_r, o, u); W_leaf_il row 3u+g
// = W_leaf row g*H+u (g = i, o, u). Bias b has blocks (i, f, o, u) (reading Q5).
#include <string.h>

#include "common.cuh"
#include "gemm_tc.h"
#include "tree.h"

namespace jk {

// MMA-issuing warps (one accumulator each); measured with the elect.sync issue: 2 -> C3 B=25
// 0.271 -> 0.264 ms against 4 (B=256 0.562 -> 0.570), 1 -> 0.264 / 0.577
constexpr int T_NMW = 2;
constexpr int TT = 160 + 32 * T_NMW;
  // threads: warps 0-3 epilogue, warp 4 TMA, warps 5.. MMA
// ring stages: a multiple of T_NMW, so a stage is always consumed by the same MMA warp (it owns
// chunks q = w mod T_NMW) and that warp can never wait on a stage two phases ahead of its loads
constexpr int T_STAGES = 8;  // backward ring; the forward uses 6 (or 4) to fit its staging buffers
constexpr int T_ASTAGE = 128 * 128;  // A chunk: 128 rows x 64 bf16
constexpr int T_BSTAGE = 80 * 128;   // B chunk: up to 80 rows x 64 bf16

JN_DEV float sig_t(float x) { return __fdividef(1.f, 1.f + __expf(-x)); }
JN_DEV float tanh_t(float x) {
  const float e = __expf(-2.f * fabsf(x));
  return copysignf(__fdividef(1.f - e, 1.f + e), x);
}

JN_DEV unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Epilogue row helpers: a thread owns one node row and up to 16 consecutive units of it. Every
// global load of the row is issued before the TMEM accumulator is ready (tile_loop's `pre`), so the
// epilogue proper has no load behind a store to a possibly aliasing pointer; runs of 4 values move
// as 16-byte vectors (vec: H % 4 == 0 keeps every row and unit group 16-B aligned), the tail of a
// run that ends inside a group moves element by element.
JN_DEV void ld_run(const float *p, bool vec, int n, float *o) {  // 16 values
#pragma unroll
  for (int g = 0; g < 4; ++g) {
    if (vec && n >= 4 * g + 4) {
      const float4 v = *reinterpret_cast<const float4 *>(p + 4 * g);
      o[4 * g] = v.x; o[4 * g + 1] = v.y; o[4 * g + 2] = v.z; o[4 * g + 3] = v.w;
    } else {
#pragma unroll
      for (int i = 0; i < 4; ++i) o[4 * g + i] = 4 * g + i < n ? p[4 * g + i] : 0.f;
    }
  }
}
JN_DEV void ld4_s(const float *p, bool vec, int n, float *o) {  // shared memory, 4 values
  if (vec && n >= 4) {
    const float4 v = *reinterpret_cast<const float4 *>(p);
    o[0] = v.x; o[1] = v.y; o[2] = v.z; o[3] = v.w;
  } else {
#pragma unroll
    for (int i = 0; i < 4; ++i) o[i] = i < n ? p[i] : 0.f;
  }
}
JN_DEV void ld4_nc(const float *p, bool vec, int n, float *o) {  // read-only data, 4 values
  if (vec && n >= 4) {
    const float4 v = __ldg(reinterpret_cast<const float4 *>(p));
    o[0] = v.x; o[1] = v.y; o[2] = v.z; o[3] = v.w;
  } else {
#pragma unroll
    for (int i = 0; i < 4; ++i) o[i] = i < n ? __ldg(p + i) : 0.f;
  }
}
template <int NV>  // NV floats, a multiple of 4
JN_DEV void st_run(float *p, bool vec, int n, const float *v) {
#pragma unroll
  for (int g = 0; g < NV / 4; ++g) {
    if (vec && n >= 4 * g + 4) {
      *reinterpret_cast<float4 *>(p + 4 * g) = make_float4(v[4 * g], v[4 * g + 1], v[4 * g + 2], v[4 * g + 3]);
    } else {
#pragma unroll
      for (int i = 0; i < 4; ++i)
        if (4 * g + i < n) p[4 * g + i] = v[4 * g + i];
    }
  }
}
JN_DEV void st4_bf16(__nv_bfloat16 *p, bool vec, int n, const float *v) {  // 4 values, one 8-B store
  if (vec && n >= 4) {
    __nv_bfloat162 a = __floats2bfloat162_rn(v[0], v[1]);
    __nv_bfloat162 b = __floats2bfloat162_rn(v[2], v[3]);
    uint2 w;
    w.x = *reinterpret_cast<uint32_t *>(&a);
    w.y = *reinterpret_cast<uint32_t *>(&b);
    *reinterpret_cast<uint2 *>(p) = w;
  } else {
#pragma unroll
    for (int i = 0; i < 4; ++i)
      if (i < n) p[i] = __float2bfloat16_rn(v[i]);
  }
}

JN_DEV void grid_sync(unsigned int *ctr, unsigned int target, unsigned long long *dbg = nullptr) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned int k = target / gridDim.x;
    if (dbg && k < 256) dbg[((size_t)k * 256 + blockIdx.x) * 2] = gtimer();
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(ctr) : "memory");
    unsigned int v;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
    } while (v < target);
    if (dbg && k < 256) dbg[((size_t)k * 256 + blockIdx.x) * 2 + 1] = gtimer();
  }
  __syncthreads();
  fence_proxy_async_global();
}

// =============================================================================== guard
// TREE_BINARY (janus.h): elements 0..N-1 are nodes, N..N+B the tree_off entries; the minimum
// failing element is reported (observed = off[t] for offsets, kind[n] for nodes).
constexpr int TREE_GUARD_SMEM_INTS = 48 * 1024;  // offsets + parent counts in shared memory up to 192 KB

JN_DEV void tree_guard_body(const TreeBufs &t, const TreeDims &d, const TreeSched &s, unsigned id,
                            long long V, long long maxn, DevStatus *st) {
  __shared__ int s_badoff;
  __shared__ int s_badnode;
  const int N = d.N, B = d.B;
  if (threadIdx.x == 0) { s_badoff = 0x7fffffff; s_badnode = 0x7fffffff; }
  __syncthreads();
  for (int i = threadIdx.x; i <= B; i += blockDim.x) {
    bool ok;
    if (i == 0) ok = t.off[0] == 0;
    else {
      const int sz = t.off[i] - t.off[i - 1];
      ok = sz >= 1 && sz <= maxn && (i < B || t.off[B] == N);
    }
    if (!ok) atomicMin(&s_badoff, i);
  }
  __syncthreads();
  const unsigned long long mask = (1ull << IDX_BITS) - 1;
  if (s_badoff != 0x7fffffff) {
    if (threadIdx.x == 0)
      atomicMin(&st->key, ((unsigned long long)id << IDX_BITS) | (unsigned long long)(N + s_badoff));
    return;
  }
  // tree offsets and parent counts in shared memory when they fit (binary searches and atomics
  // on chip); otherwise in global memory
  extern __shared__ int s_off[];
  const bool sm = B + 1 + N <= TREE_GUARD_SMEM_INTS;
  const int *offp = sm ? s_off : t.off;
  int *pc = sm ? s_off + B + 1 : s.pcount;
  for (int n = threadIdx.x; n < N; n += blockDim.x) pc[n] = 0;
  if (sm)
    for (int i = threadIdx.x; i <= B; i += blockDim.x) s_off[i] = t.off[i];
  __syncthreads();
  for (int n = threadIdx.x; n < N; n += blockDim.x) {
    int lo_t = 0, hi_t = B - 1;  // tree containing n: largest t with off[t] <= n
    while (lo_t < hi_t) {
      const int mid = (lo_t + hi_t + 1) >> 1;
      if (offp[mid] <= n) lo_t = mid; else hi_t = mid - 1;
    }
    s.tree_of[n] = lo_t;
    const int lo = offp[lo_t];
    // the forest arrays are read-only here: non-coherent loads may run ahead of the stores
    const int k = __ldg(t.kind + n);
    const int wd = __ldg(t.word + n), l = __ldg(t.left + n), r = __ldg(t.right + n);
    bool bad = false;
    if (k == 0) bad = !(wd >= 0 && wd < V);
    else if (k == 1) {
      if (l >= lo && l < n && r >= lo && r < n && l != r) {
        atomicAdd(&pc[l], 1);
        atomicAdd(&pc[r], 1);
      } else bad = true;
    } else bad = true;
    if (bad) atomicMin(&s_badnode, n);
  }
  __syncthreads();
  for (int n = threadIdx.x; n < N; n += blockDim.x) {
    const bool root = n == offp[s.tree_of[n] + 1] - 1;
    if (root ? pc[n] != 0 : pc[n] != 1) atomicMin(&s_badnode, n);
  }
  __syncthreads();
  if (threadIdx.x == 0 && s_badnode != 0x7fffffff)
    atomicMin(&st->key, ((unsigned long long)id << IDX_BITS) | (unsigned long long)s_badnode);
  (void)mask;
}
__global__ void __launch_bounds__(1024) tree_guard_kernel(TreeBufs t, TreeDims d, TreeSched s,
                                                          unsigned id, long long V, long long maxn,
                                                          DevStatus *st) {
  pdl_enter();
  tree_guard_body(t, d, s, id, V, maxn, st);
}

cudaError_t launch_tree_guard(const TreeBufs &t, const TreeDims &d, const TreeSched &s, unsigned id,
                              long long V, long long max_nodes, DevStatus *st, cudaStream_t str) {
  const int smem = d.B + 1 + d.N <= TREE_GUARD_SMEM_INTS ? (d.B + 1 + d.N) * 4 : 0;
  cudaError_t e = set_smem_once((const void *)tree_guard_kernel, TREE_GUARD_SMEM_INTS * 4);
  if (e != cudaSuccess) return e;
  {
    const cudaError_t pe_ = launch_pdl(tree_guard_kernel, dim3(1), dim3(1024), smem, str, t, d, s, id, V, max_nodes, st);
    if (pe_ != cudaSuccess) return pe_;
  }
  return cudaGetLastError();
}

// =============================================================================== schedule
// Single block. Heights by a per-tree scan in post-order (children precede parents); then a
// stable counting sort by height in node-id order (warp match + per-level prefix over warps).
constexpr int TREE_SCHED_SMEM_NODES = 13 * 1024;  // heights + children in shared memory up to 156 KB
constexpr int TREE_SCHED_SMEM_OFF = 4096;         // + the tree offsets (16 KB)

JN_DEV void tree_schedule_body(const TreeBufs &t, const TreeDims &d, const TreeSched &s, const DevStatus *st) {
  __shared__ int hist[TREE_MAX_LEVELS + 1];
  __shared__ int running[TREE_MAX_LEVELS + 1];
  __shared__ unsigned short wcnt[32][TREE_MAX_LEVELS];
  __shared__ int s_L;
  const int N = d.N, B = d.B;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (*reinterpret_cast<const volatile unsigned long long *>(&st->key) != KEY_PASS) {
    // the forest failed its AssertOp: nothing downstream may run
    if (tid == 0) { s.meta[0] = 0; s.meta[1] = 0; s.meta[2] = 0; s.meta[3] = 0; }
    return;
  }
  unsigned long long *pb = t.dbg ? t.dbg + 4 * 256 * 256 * 2 : nullptr;  // dev probe: phase times
  if (pb && tid == 0) pb[0] = gtimer();
  for (int i = tid; i <= TREE_MAX_LEVELS; i += blockDim.x) { hist[i] = 0; running[i] = 0; }
  if (tid == 0) s_L = 1;
  __syncthreads();
  // heights (robust to malformed input: the guard has already decided the commit). One thread
  // walks each tree in node order (children precede parents); the heights live in shared memory
  // when the forest fits, so the walk is not a chain of global-memory round trips.
  extern __shared__ int sh_height[];
  const bool in_smem = N <= TREE_SCHED_SMEM_NODES;
  int *hh = in_smem ? sh_height : s.height;
  // children of internal nodes (kl = INT_MIN marks a leaf) staged in shared memory first
  int *kl = sh_height + N, *kr = sh_height + 2 * N;
  constexpr int LEAF = -2147483647 - 1;
  if (in_smem) {
    for (int n = tid; n < N; n += blockDim.x) {
      const bool in = t.kind[n] == 1;
      kl[n] = in ? t.left[n] : LEAF;
      kr[n] = in ? t.right[n] : LEAF;
    }
    __syncthreads();
  }
  if (pb && tid == 0) pb[1] = gtimer();
  // small forests (<= 2 nodes per thread): parallel relaxation; large ones: the per-tree walk (a
  // sweep over 10 nodes per thread costs more than walking the largest tree)
  const bool relax = in_smem && N <= 2 * (int)blockDim.x;
  if (relax) {
    // heights by parallel relaxation over all nodes: h = 1 + max(h_l, h_r) from h = 0 rises
    // monotonically to the longest leaf path, one level per sweep, so max height + 1 sweeps,
    // each one node per thread, instead of one thread walking each whole tree. Children with
    // ids >= the node are ignored (the guard reports them), so no cycle can keep it rising.
    // Jacobi sweeps (read one buffer, write the other): no thread reads a height another thread
    // writes in the same sweep (race-free under compute-sanitizer racecheck).
    int *h2 = sh_height + 3 * N + TREE_SCHED_SMEM_OFF;  // second buffer (relax: N <= 2048)
    for (int n = tid; n < N; n += blockDim.x) { hh[n] = 0; h2[n] = 0; }
    __syncthreads();
    int *cur = hh, *nxt = h2;
    bool more = true;
    while (more) {
      bool changed = false;
      for (int n = tid; n < N; n += blockDim.x) {
        const int l = kl[n];
        int h = 0;
        if (l != LEAF) {
          const int r = kr[n];
          const int hl = (l >= 0 && l < n) ? cur[l] : 0;
          const int hr = (r >= 0 && r < n) ? cur[r] : 0;
          h = min(1 + max(hl, hr), TREE_MAX_LEVELS - 1);
        }
        nxt[n] = h;
        changed |= h != cur[n];
      }
      more = __syncthreads_or(changed);
      int *tmp = cur; cur = nxt; nxt = tmp;
    }
    if (cur != hh)  // the fixpoint is in h2: copy it back
      for (int n = tid; n < N; n += blockDim.x) hh[n] = cur[n];
  }
  for (int tr = relax ? B : tid; tr < B; tr += blockDim.x) {  // one thread walks each tree
    const int lo = max(0, t.off[tr]), hi = min(N, t.off[tr + 1]);
    for (int n = lo; n < hi; ++n) {
      int h = 0;
      const bool internal = in_smem ? kl[n] != LEAF : t.kind[n] == 1;
      if (internal) {
        const int l = in_smem ? kl[n] : t.left[n], r = in_smem ? kr[n] : t.right[n];
        const int hl = (l >= lo && l < n) ? hh[l] : 0;
        const int hr = (r >= lo && r < n) ? hh[r] : 0;
        h = min(1 + max(hl, hr), TREE_MAX_LEVELS - 1);
      }
      hh[n] = h;
      if (!in_smem) s.tree_of[n] = tr;  // (in shared memory: the parallel pass below)
    }
  }
  __syncthreads();
  // tree_of, pslot, heights to global in parallel over nodes (the walk above is one thread per
  // tree: it carries only the on-chip height chain); tree of a node by binary search in the
  // offsets (shared memory)
  if (in_smem) {
    int *soff = sh_height + 3 * N;
    const bool off_sm = B + 1 <= TREE_SCHED_SMEM_OFF;
    if (off_sm)
      for (int i = tid; i <= B; i += blockDim.x) soff[i] = t.off[i];
    __syncthreads();
    const int *offp = off_sm ? soff : t.off;
    for (int n = tid; n < N; n += blockDim.x) {
      int lo_t = 0, hi_t = B - 1;
      while (lo_t < hi_t) {
        const int mid = (lo_t + hi_t + 1) >> 1;
        if (offp[mid] <= n) lo_t = mid; else hi_t = mid - 1;
      }
      s.tree_of[n] = lo_t;
      s.height[n] = hh[n];
    }
  }
  for (int n = tid; n < N; n += blockDim.x) s.pslot[n] = -1;
  __syncthreads();
  if (pb && tid == 0) pb[2] = gtimer();
  for (int n = tid; n < N; n += blockDim.x) {
    atomicAdd(&hist[hh[n]], 1);
    atomicMax(&s_L, hh[n] + 1);
  }
  __syncthreads();
  const int L = s_L;
  if (tid == 0) {
    int acc = 0;
    for (int l = 0; l <= L; ++l) {
      s.lvl_off[l] = acc;
      if (l < L) acc += hist[l];
    }
    s.meta[0] = L;
    s.meta[1] = N;
    s.meta[2] = hist[0];
    s.meta[3] = N - hist[0];
  }
  __syncthreads();
  if (pb && tid == 0) pb[3] = gtimer();
  // stable placement, chunk by chunk of 1024 ids
  for (int c0 = 0; c0 < N; c0 += blockDim.x) {
    for (int i = tid; i < 32 * TREE_MAX_LEVELS; i += blockDim.x) (&wcnt[0][0])[i] = 0;
    __syncthreads();
    const int n = c0 + tid;
    const bool live = n < N;
    const int h = live ? hh[n] : TREE_MAX_LEVELS - 1;
    const unsigned same = __match_any_sync(0xffffffff, live ? h : -1 - lane);
    const int rank_w = __popc(same & ((1u << lane) - 1));
    if (live && rank_w == 0) wcnt[warp][h] = (unsigned short)__popc(same);
    __syncthreads();
    // per level: exclusive prefix over warps (in place), then advance the running count
    for (int l = tid; l < L; l += blockDim.x) {
      int acc = running[l];
      for (int w = 0; w < 32; ++w) {
        const int c = wcnt[w][l];
        wcnt[w][l] = (unsigned short)(acc - running[l]);
        acc += c;
      }
      hist[l] = running[l];  // base of this chunk for level l
      running[l] = acc;
    }
    __syncthreads();
    if (live) {
      const int pos = s.lvl_off[h] + hist[h] + wcnt[warp][h] + rank_w;
      s.order[pos] = n;
      s.irank[n] = h > 0 ? pos - s.lvl_off[1] : -1 - pos;  // leaves: -1 - (level-0 position)
    }
    __syncthreads();
  }
  if (pb && tid == 0) pb[4] = gtimer();
  // parent slots
  for (int n = tid; n < N; n += blockDim.x) {
    if (t.kind[n] == 1 && hh[n] > 0) {
      const int l = t.left[n], r = t.right[n];
      if (l >= 0 && l < N) s.pslot[l] = (s.irank[n] << 1) | 0;
      if (r >= 0 && r < N) s.pslot[r] = (s.irank[n] << 1) | 1;
    }
  }
  __syncthreads();
  if (pb && tid == 0) pb[5] = gtimer();
  (void)st;
}
__global__ void __launch_bounds__(1024) tree_schedule_kernel(TreeBufs t, TreeDims d, TreeSched s,
                                                             const DevStatus *st) {
  pdl_enter();
  tree_schedule_body(t, d, s, st);
}
// TREE_BINARY guard and level schedule in one single-block launch (both are one block of 1024
// threads; bar.sync orders the guard's key proposals before the schedule reads the key)
__global__ void __launch_bounds__(1024) tree_guard_schedule_kernel(TreeBufs t, TreeDims d, TreeSched s,
                                                                   unsigned id, long long V, long long maxn,
                                                                   DevStatus *st) {
  pdl_enter();
  tree_guard_body(t, d, s, id, V, maxn, st);
  __syncthreads();
  tree_schedule_body(t, d, s, st);
}

cudaError_t launch_tree_schedule(const TreeBufs &t, const TreeDims &d, const TreeSched &s,
                                 const DevStatus *st, cudaStream_t str) {
  const int smem = d.N <= TREE_SCHED_SMEM_NODES
                       ? (3 * d.N + TREE_SCHED_SMEM_OFF + (d.N <= 2048 ? d.N : 0)) * 4 : 0;
  cudaError_t e = set_smem_once((const void *)tree_schedule_kernel, (3 * TREE_SCHED_SMEM_NODES + TREE_SCHED_SMEM_OFF) * 4);
  if (e != cudaSuccess) return e;
  {
    const cudaError_t pe_ = launch_pdl(tree_schedule_kernel, dim3(1), dim3(1024), smem, str, t, d, s, st);
    if (pe_ != cudaSuccess) return pe_;
  }
  return cudaGetLastError();
}

cudaError_t launch_tree_guard_schedule(const TreeBufs &t, const TreeDims &d, const TreeSched &s, unsigned id,
                                       long long V, long long max_nodes, DevStatus *st, cudaStream_t str) {
  const int gsmem = d.B + 1 + d.N <= TREE_GUARD_SMEM_INTS ? (d.B + 1 + d.N) * 4 : 0;
  const int ssmem = d.N <= TREE_SCHED_SMEM_NODES
                        ? (3 * d.N + TREE_SCHED_SMEM_OFF + (d.N <= 2048 ? d.N : 0)) * 4 : 0;
  cudaError_t e = set_smem_once((const void *)tree_guard_schedule_kernel,
                                std::max(TREE_GUARD_SMEM_INTS, 3 * TREE_SCHED_SMEM_NODES + TREE_SCHED_SMEM_OFF) * 4);
  if (e != cudaSuccess) return e;
  {
    const cudaError_t pe_ = launch_pdl(tree_guard_schedule_kernel, dim3(1), dim3(1024), std::max(gsmem, ssmem), str, t, d,
                                       s, id, V, max_nodes, st);
    if (pe_ != cudaSuccess) return pe_;
  }
  return cudaGetLastError();
}

// =============================================================================== GEMM tiles
// Persistent tile loop shared by the forward and backward kernels: rows [row0, row0 + M) of the
// A map times B rows [0, NTOT) in tiles of 128 x NT; the epilogue functor receives (row index,
// tile column base, z[NT]) for rows < M.
struct Ring {
  uint64_t *full, *empty, *tfull;
  uint8_t *sA, *sB;
  uint32_t tmem;
  int q;      // chunk counter (both producer and MMA advance it identically)
  int tiles;  // tiles processed by this CTA (tfull phase)
  float *zst; // STAGED tile loops: the accumulator tile [128][NT + 1] in shared memory
  // resident B (optional): this CTA's NT-row slice of the B operand, all K chunks, loaded once
  // per launch; the CTA then always takes tiles of column block bres_nn and only streams A
  const uint8_t *sBres = nullptr;
  uint64_t *bres_bar = nullptr;
  int bres_nn = -1, bres_groups = 0;
  bool bres_ready = false;  // (MMA thread) the resident slice has landed
};

// STAGED: the epilogue threads park the accumulator tile in shared memory and the epilogue
// functor receives (first row of the tile, valid rows, tile column base) on all 128 threads, so
// a level with few nodes spreads its (row, unit) work over the whole epilogue instead of one
// thread per row; otherwise it receives (row, tile column base, z[NT], pre's context) per row.
// tmA32 (optional): the A map with a 32-row box, used for tiles with <= 32 valid rows (the
// upper levels of a forest): the MMA still reads 128 smem rows, but rows past the box only feed
// accumulator rows the epilogue discards, and the level's A traffic drops 4x.
template <int NT, int STAGED = 0, int NS = T_STAGES, typename Pre, typename Epi>
JN_DEV void tile_loop(Ring &rg, const CUtensorMap *tmA, const CUtensorMap *tmB, int row0, int M,
                      int NTOT, int K, Pre pre, Epi epi, int nmw, unsigned long long *pr = nullptr,
                      const CUtensorMap *tmA32 = nullptr) {
  nmw = min(nmw, T_NMW);        // the launch has T_NMW MMA warps
  while (NS % nmw) nmw >>= 1;  // a fixed MMA warp per ring stage
  // nmw in {1, 2, 4} MMA warps take part (T_STAGES % nmw == 0 keeps a fixed owner per stage):
  // more warps for long reductions, fewer TMEM tiles for the epilogue to sum on short ones
  const int warp = threadIdx.x >> 5;
  const int ntile_n = (NTOT + NT - 1) / NT;
  const int mtiles = (M + 127) / 128;
  const int tiles = mtiles * ntile_n;
  const int nk = (K + 63) / 64;
  const bool res = rg.sBres != nullptr;
  constexpr uint32_t idesc = umma_idesc_bf16(128, NT, 0, 0);
  // tile sequence of this CTA: all tiles round robin, or (resident B) the M blocks of its column
  const int t0 = res ? (rg.bres_nn < 0 ? tiles : blockIdx.x / ntile_n) : blockIdx.x;
  const int tstep = res ? rg.bres_groups : gridDim.x;
  const int tend = res ? mtiles : tiles;
  for (int it = t0; it < tend; it += tstep) {
    const int m = res ? it : it / ntile_n, nn = res ? rg.bres_nn : it % ntile_n;
    if (warp == 4) {
      const bool small = tmA32 && M - m * 128 <= 32;
      const CUtensorMap *ta = small ? tmA32 : tmA;
      if ((threadIdx.x & 31) == 0)
        for (int kc = 0; kc < nk; ++kc) {
          const int q = rg.q + kc, s = q % NS, r = q / NS;
          if (r > 0) mbar_wait(&rg.empty[s], (r - 1) & 1);
          mbar_expect_tx(&rg.full[s], (small ? 32 * 128 : T_ASTAGE) + (res ? 0 : NT * 128));
          tma_load_2d(rg.sA + s * T_ASTAGE, ta, &rg.full[s], kc * 64, row0 + m * 128);
          if (!res) tma_load_2d(rg.sB + s * T_BSTAGE, tmB, &rg.full[s], kc * 64, nn * NT);
        }
      __syncwarp();
    } else if (warp >= 5) {
      // ring chunk q goes to MMA warp q % T_NMW (a fixed owner per stage), accumulating into
      // its own TMEM tile
      const int w = warp - 5;
      if (elect_one_sync()) {
        if (res && !rg.bres_ready) {
          mbar_wait(rg.bres_bar, 0);
          rg.bres_ready = true;
        }
        const uint32_t acc = rg.tmem + (uint32_t)(w * NT);
        const int kc0 = w < nmw ? ((w - rg.q) % nmw + nmw) % nmw : nk;  // my first chunk of this tile
        for (int kc = kc0; kc < nk; kc += nmw) {
          const int q = rg.q + kc, s = q % NS, r = q / NS;
          mbar_wait(&rg.full[s], r & 1);
          tc_fence_after();
          const uint32_t a = smem_u32(rg.sA + s * T_ASTAGE);
          const uint32_t b = res ? smem_u32(rg.sBres + kc * NT * 128) : smem_u32(rg.sB + s * T_BSTAGE);
          umma_bf16_k64(acc, umma_desc_sw128(a, 16, 1024), umma_desc_sw128(b, 16, 1024), idesc,
                        kc != kc0 ? 1u : 0u, 2, 2);
          umma_commit(&rg.empty[s]);
        }
        umma_commit(rg.tfull);  // arrives even with no chunk (nk < T_NMW)
      }
      __syncwarp();
    } else {
      const int row = m * 128 + threadIdx.x;
      const auto ctx = pre(row < M ? row : -1, nn * NT);  // row metadata while the MMAs run
      mbar_wait(rg.tfull, rg.tiles & 1);
      __syncwarp();
      tc_fence_after();
      if (pr && threadIdx.x == 0) pr[0] = gtimer();
      float z[NT];
#pragma unroll
      for (int i = 0; i < NT; ++i) z[i] = 0.f;
      const uint32_t ta = rg.tmem + ((uint32_t)(warp * 32) << 16);
      const int nacc = min(nmw, nk);  // the owners of chunks 0 .. nacc-1 of this tile
      for (int i = 0; i < nacc; ++i) {
        const int w = (rg.q + i) % nmw;
#pragma unroll
        for (int c = 0; c + 32 <= NT; c += 32) {
          float v[32];
          tmem_ld32(ta + w * NT + c, v);
#pragma unroll
          for (int i = 0; i < 32; ++i) z[c + i] += v[i];
        }
        if (NT % 32) {
          float v[16];
          tmem_ld16(ta + w * NT + (NT / 32) * 32, v);
#pragma unroll
          for (int i = 0; i < 16; ++i) z[(NT / 32) * 32 + i] += v[i];
        }
      }
      if (pr) {
        asm volatile("bar.sync 1, 128;" ::: "memory");
        if (threadIdx.x == 0) pr[2] = gtimer();
      }
      if constexpr (STAGED == 2) {  // staged for every warp of the CTA (below)
        float *zr = rg.zst + threadIdx.x * (NT + 1);
#pragma unroll
        for (int i = 0; i < NT; ++i) zr[i] = z[i];
        (void)ctx;
      } else if constexpr (STAGED) {
        float *zr = rg.zst + threadIdx.x * (NT + 1);
#pragma unroll
        for (int i = 0; i < NT; ++i) zr[i] = z[i];
        asm volatile("bar.sync 1, 128;" ::: "memory");
        epi(m * 128, min(128, M - m * 128), nn * NT);
        (void)ctx;
      } else {
        if (row < M) epi(row, nn * NT, z, ctx);
      }
      if (pr) {
        asm volatile("bar.sync 1, 128;" ::: "memory");
        if (threadIdx.x == 0) pr[1] = gtimer();
        if (threadIdx.x == 0) pr[3] = pr[1];
      }
    }
    if constexpr (STAGED == 2) {  // the producer and MMA warps are idle now: all warps share the epilogue
      __syncthreads();
      epi(m * 128, min(128, M - m * 128), nn * NT);
    }
    rg.q += nk;
    rg.tiles += 1;
    tc_fence_before();
    __syncthreads();  // TMEM accumulator free for the next tile
    tc_fence_after();
    if (STAGED == 2 && pr && threadIdx.x == 0) { pr[1] = gtimer(); pr[3] = pr[1]; }
  }
}

// =============================================================================== forward
struct TreeFwdMaps {
  CUtensorMap x_leaf, w_leaf, stage_h, u, stage_h32;
};

template <int NS, bool RNN>
__global__ void __launch_bounds__(TT, 1) tree_fwd_kernel(const __grid_constant__ TreeFwdMaps mp,
                                                         TreeBufs t, TreeDims d, TreeSched s,
                                                         const DevStatus *st) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t *base = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                              ~uintptr_t(1023));
  Ring rg;
  rg.sA = base;
  rg.sB = base + NS * T_ASTAGE;
  rg.full = reinterpret_cast<uint64_t *>(rg.sB + NS * T_BSTAGE);
  rg.empty = rg.full + NS;
  rg.tfull = rg.empty + NS;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(rg.tfull + 1);
  float *sbias = reinterpret_cast<float *>(base + NS * (T_ASTAGE + T_BSTAGE) + 256);
  const int H = d.H, E = d.E;
  rg.zst = sbias + ((4 * H + 3) & ~3);            // [128][NT + 1] accumulator tile
  int *s_ps = reinterpret_cast<int *>(rg.zst + 128 * 81);  // per tile row: parent slot
  int *s_tr = s_ps + 128;                          //               tree (roots)
  float *s_cc = reinterpret_cast<float *>(s_tr + 128);  // [128][32] children c (c_l | c_r)
  const int warp = threadIdx.x >> 5;
  if (st->key != KEY_PASS) return;  // assumption failed: skip (uniform across CTAs)
  if (threadIdx.x == 128) {
    for (int i = 0; i < NS; ++i) { mbar_init(&rg.full[i], 1); mbar_init(&rg.empty[i], 1); }
    mbar_init(rg.tfull, T_NMW);
    fence_barrier_init();
  }
  if (warp == 5) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  rg.tmem = *tmem_slot;
  rg.q = 0;
  rg.tiles = 0;
  const int L = s.meta[0], n0 = s.meta[2], nint = s.meta[3];
  unsigned int ep = 0;
  // ---- phase 0: leaf inputs in level-0 order (R1: rb(E[word])), ones columns for bias grads
  {
    const int gt = blockIdx.x * blockDim.x + threadIdx.x, gs = gridDim.x * blockDim.x;
    if constexpr (RNN) {
      // TreeRNN: a leaf IS its word vector (E = H, R2: rounded where it feeds a GEMM), written
      // straight into its parent's staging row (or the root features of a one-leaf tree)
      for (long long e = gt; e < (long long)n0 * H; e += gs) {
        const int pos = (int)(e / H), k = (int)(e % H);
        const int n = s.order[pos], ps = s.pslot[n];
        int w = t.word[n];
        w = (w >= 0 && w < d.V) ? w : 0;
        const __nv_bfloat16 hb = __float2bfloat16_rn(t.E[(size_t)w * E + k]);
        if (ps >= 0) t.stage_h[(size_t)(ps >> 1) * d.P2 + (ps & 1) * H + k] = hb;
        else t.root_h[(size_t)s.tree_of[n] * H + k] = __bfloat162float(hb);
      }
    } else {
      for (long long e = gt; e < (long long)n0 * d.Ep; e += gs) {
        const int pos = (int)(e / d.Ep), k = (int)(e % d.Ep);
        int w = t.word[s.order[pos]];
        w = (w >= 0 && w < d.V) ? w : 0;
        const float v = k < E ? t.E[(size_t)w * E + k] : (k == E ? 1.f : 0.f);
        t.x_leaf[(size_t)pos * d.Ep + k] = __float2bfloat16_rn(v);
      }
    }
    for (int i = gt; i < nint; i += gs) t.stage_h[(size_t)i * d.P2 + 2 * H] = __float2bfloat16_rn(1.f);
    // the bias (4H floats; TreeRNN: H) lives in shared memory for every epilogue of the launch
    for (int i = threadIdx.x; i < (RNN ? H : 4 * H); i += blockDim.x) sbias[i] = t.b[i];
    // the per-level arrival counters (first used after the leaf level's grid barrier)
    if (blockIdx.x == 0)
      for (int l = threadIdx.x; l < TREE_MAX_LEVELS; l += blockDim.x) {
        t.barrier[64 + l * 32] = 0;
        t.bwd_lvl[l * 32] = 0;  // the backward launch's counters (it runs after this kernel)
      }
  }
  fence_proxy_async_global();
  grid_sync(t.barrier, ++ep * gridDim.x, t.dbg);
  const float *b = sbias;
  // ---- level 0: leaves. z = x W_leaf^T; i, o = sigmoid, u = tanh; c = i u; h = o tanh(c)
  const bool vec = (H % 4) == 0;
  if constexpr (!RNN) {
  const int leaf_workers = min((int)gridDim.x, ((n0 + 127) / 128) * ((3 * H + 47) / 48));  // tiles of the leaf GEMM
  tile_loop<48, true, NS>(rg, &mp.x_leaf, &mp.w_leaf, 0, n0, 3 * H, E, [&](int pos, int) {
    if (pos >= 0) {  // row metadata into shared memory while the MMAs run
      const int n = s.order[pos], ps = s.pslot[n];
      s_ps[threadIdx.x] = ps;
      s_tr[threadIdx.x] = ps < 0 ? s.tree_of[n] : 0;
    }
    return 0;
  }, [&](int pbase, int nrows, int col0) {
    const int u0 = col0 / 3, nu = min(16, H - u0);
    for (int i0 = threadIdx.x; i0 < nrows * 16; i0 += 512) {  // item = (row, unit), 4 in flight
      float zv[4][3], bv[4][3];
      bool ok[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int i = i0 + 128 * j;
        ok[j] = i < nrows * 16 && (i & 15) < nu;
        if (ok[j]) {
          const float *zz = rg.zst + (i >> 4) * 49 + 3 * (i & 15);
          const int u = u0 + (i & 15);
#pragma unroll
          for (int g = 0; g < 3; ++g) { zv[j][g] = zz[g]; bv[j][g] = b[(g == 0 ? 0 : g + 1) * H + u]; }
        }
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) {
      if (!ok[j]) continue;
      const int i = i0 + 128 * j, r = i >> 4, uu = i & 15;
      const int u = u0 + uu, pos = pbase + r, ps = s_ps[r];
      const float ig = sig_t(zv[j][0] + bv[j][0]);
      const float og = sig_t(zv[j][1] + bv[j][1]);
      const float ug = tanh_t(zv[j][2] + bv[j][2]);
      const float c = ig * ug, h = og * tanh_t(c);
      float *gl = t.gates_leaf + (size_t)pos * 3 * H + 3 * u;
      gl[0] = ig; gl[1] = og; gl[2] = ug;
      t.c_leaf[(size_t)pos * H + u] = c;
      if (ps >= 0) {
        const int pi = ps >> 1, side = ps & 1;
        t.stage_h[(size_t)pi * d.P2 + side * H + u] = __float2bfloat16_rn(h);
        t.stage_c[(size_t)pi * 2 * H + side * H + u] = c;
      } else {
        t.root_h[(size_t)s_tr[r] * H + u] = h;
      }
      }
    }
  }, (E + 63) / 64 >= 8 ? 2 : 1);
  fence_proxy_async_global();
  // the leaf level's workers arrive on level 0's counter (the first internal level waits for it,
  // as every internal level waits for the one below) instead of a grid barrier
  if ((int)blockIdx.x < leaf_workers) {
    __syncthreads();
    if (threadIdx.x == 0) asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(t.barrier + 64) : "memory");
  }
  }  // !RNN (TreeRNN leaves were placed in phase 0)
  // ---- internal levels: z = [h_l; h_r] U^T; c = i u + f_l c_l + f_r c_r; h = o tanh(c)
  // Internal levels: only the CTAs with tiles at a level take part in it. A CTA waits for the
  // previous level's workers (its arrival counter, one 128-B line per level) before its own tiles
  // and then arrives on this level's counter — the chain of release/acquire pairs orders every
  // earlier level too — instead of all CTAs meeting at a grid barrier per level.
  unsigned int *lvl_ctr = t.barrier + 64;
  const int NGH = RNN ? H : 5 * H;  // gate rows of the cell weight (U: 5H interleaved; W: H)
  const int ntn = (NGH + 79) / 80;
  auto workers = [&](int l) {
    const int c = s.lvl_off[l + 1] - s.lvl_off[l];
    return min((int)gridDim.x, ((c + 127) / 128) * ntn);
  };
  for (int l = 1; l < L; ++l) {
    const int p0 = s.lvl_off[l], cnt = s.lvl_off[l + 1] - p0, r0 = p0 - s.lvl_off[1];
    if ((int)blockIdx.x >= workers(l)) continue;
    if (l > 1 || !RNN) {  // level 1 waits for the leaf level's workers (TreeRNN: placed in phase 0)
      if (threadIdx.x == 0) {
        const unsigned int target =
            (unsigned)(l > 1 ? workers(l - 1) : min((int)gridDim.x, ((n0 + 127) / 128) * ((3 * H + 47) / 48)));
        unsigned int v;
        do {
          asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(lvl_ctr + (l - 1) * 32) : "memory");
        } while (v < target);
      }
      __syncthreads();
      fence_proxy_async_global();
    }
    if constexpr (RNN) {
    // TreeRNN: z = [h_l; h_r] W^T + b, h = tanh(z); a tile = 80 units of 128 nodes
    tile_loop<80, true, NS>(rg, &mp.stage_h, &mp.u, r0, cnt, H, 2 * H, [&](int row, int) {
      if (row >= 0) {
        const int n = s.order[p0 + row], ps = s.pslot[n];
        s_ps[threadIdx.x] = ps;
        s_tr[threadIdx.x] = ps < 0 ? s.tree_of[n] : 0;
      }
      return 0;
    }, [&](int rbase, int nrows, int col0) {
      const int nu = min(80, H - col0);
      for (int i0 = threadIdx.x; i0 < nrows * 80; i0 += 512) {  // item = (row, unit), 4 in flight
        float zv[4];
        bool ok[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int i = i0 + 128 * j, r = i / 80, uu = i - 80 * r;
          ok[j] = i < nrows * 80 && uu < nu;
          zv[j] = ok[j] ? rg.zst[r * 81 + uu] + b[col0 + uu] : 0.f;
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          if (!ok[j]) continue;
          const int i = i0 + 128 * j, r = i / 80, u = col0 + i - 80 * r;
          const int ir = r0 + rbase + r, ps = s_ps[r];
          const float h = tanh_t(zv[j]);
          t.c_int[(size_t)ir * H + u] = h;
          if (ps >= 0) t.stage_h[(size_t)(ps >> 1) * d.P2 + (ps & 1) * H + u] = __float2bfloat16_rn(h);
          else t.root_h[(size_t)s_tr[r] * H + u] = h;
        }
      }
    }, (2 * H + 63) / 64 >= 16 ? 4 : ((2 * H + 63) / 64 >= 8 ? 2 : 1),
       t.dbg ? t.dbg + 2 * 256 * 256 * 2 + ((size_t)l * 256 + blockIdx.x) * 4 : nullptr, &mp.stage_h32);
    } else {
    tile_loop<80, true, NS>(rg, &mp.stage_h, &mp.u, r0, cnt, 5 * H, 2 * H, [&](int row, int col0) {
      const int u0 = col0 / 5, nu = min(16, H - u0);
      if (row >= 0 && nu > 0) {  // row metadata + children c into shared memory during the MMAs
        const int n = s.order[p0 + row], ps = s.pslot[n];
        s_ps[threadIdx.x] = ps;
        s_tr[threadIdx.x] = ps < 0 ? s.tree_of[n] : 0;
        const float *sc = t.stage_c + (size_t)(r0 + row) * 2 * H;
        float cl[16], cr[16];
        ld_run(sc + u0, vec, nu, cl);
        ld_run(sc + H + u0, vec, nu, cr);
        float *dst = s_cc + threadIdx.x * 32;
#pragma unroll
        for (int k = 0; k < 16; ++k) { dst[k] = cl[k]; dst[16 + k] = cr[k]; }
      }
      return 0;
    }, [&](int rbase, int nrows, int col0) {
      const int u0 = col0 / 5, nu = min(16, H - u0);
      // item = (row, unit), 16 per row; four items per thread in flight (all shared-memory reads
      // first, then the math and the stores): one warp per SM sub-partition has no other latency
      // hiding
      for (int i0 = threadIdx.x; i0 < nrows * 16; i0 += 512) {
        float zv[4][5], bv[4][4], cl[4], cr[4];
        int rr[4], uu[4];
        bool ok[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int i = i0 + 128 * j;
          rr[j] = i >> 4; uu[j] = i & 15;
          ok[j] = i < nrows * 16 && uu[j] < nu;
          if (ok[j]) {
            const float *zz = rg.zst + rr[j] * 81 + 5 * uu[j];
            const int u = u0 + uu[j];
#pragma unroll
            for (int g = 0; g < 5; ++g) zv[j][g] = zz[g];
#pragma unroll
            for (int g = 0; g < 4; ++g) bv[j][g] = b[g * H + u];
            cl[j] = s_cc[rr[j] * 32 + uu[j]];
            cr[j] = s_cc[rr[j] * 32 + 16 + uu[j]];
          }
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          if (!ok[j]) continue;
          const int r = rr[j], u = u0 + uu[j], ir = r0 + rbase + r, ps = s_ps[r];
          const float ig = sig_t(zv[j][0] + bv[j][0]);
          const float fl = sig_t(zv[j][1] + bv[j][1]);
          const float fr = sig_t(zv[j][2] + bv[j][1]);
          const float og = sig_t(zv[j][3] + bv[j][2]);
          const float ug = tanh_t(zv[j][4] + bv[j][3]);
          const float c = ig * ug + fl * cl[j] + fr * cr[j];
          const float h = og * tanh_t(c);
          float *gi = t.gates_int + (size_t)ir * 5 * H + 5 * u;
          gi[0] = ig; gi[1] = fl; gi[2] = fr; gi[3] = og; gi[4] = ug;
          t.c_int[(size_t)ir * H + u] = c;
          if (ps >= 0) {
            const int pi = ps >> 1, side = ps & 1;
            t.stage_h[(size_t)pi * d.P2 + side * H + u] = __float2bfloat16_rn(h);
            t.stage_c[(size_t)pi * 2 * H + side * H + u] = c;
          } else {
            t.root_h[(size_t)s_tr[r] * H + u] = h;
          }
        }
      }
    }, (2 * H + 63) / 64 >= 16 ? 4 : ((2 * H + 63) / 64 >= 8 ? 2 : 1),
       t.dbg ? t.dbg + 2 * 256 * 256 * 2 + ((size_t)l * 256 + blockIdx.x) * 4 : nullptr, &mp.stage_h32);
    }  // RNN / LSTM cell
    fence_proxy_async_global();
    __syncthreads();
    if (threadIdx.x == 0) asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(lvl_ctr + l * 32) : "memory");
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 5) tmem_dealloc(rg.tmem, 512);
  (void)st;
}

static int tree_smem(int ns = T_STAGES) { return 1024 + ns * (T_ASTAGE + T_BSTAGE) + 256; }
// forward: + bias [4H] + accumulator tile [128][81] + row metadata [2][128] + children c [128][32]
static int tree_smem_fwd(int ns, int H) {
  return tree_smem(ns) + 4 * ((4 * H + 3) & ~3) + 4 * 128 * 81 + 8 * 128 + 4 * 128 * 32;
}

static cudaError_t coop(const void *fn, int grid, int smem, void **args, cudaStream_t st) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(TT);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;
  at[0].val.cooperative = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelExC(&cfg, fn, args);
}

cudaError_t launch_tree_fwd(const TreeBufs &t, const TreeDims &d, const TreeSched &s,
                            const __nv_bfloat16 *Wl_il, const __nv_bfloat16 *U_il, int grid,
                            const DevStatus *st, cudaStream_t str) {
  // the maps span the allocated Nmax rows (rows past this step's N only feed discarded accumulator
  // rows), so they depend on the workspace alone and are encoded once per workspace, not per step
  struct Key { const void *a, *b, *c; long long E, H, Ep, P2, Nmax, rnn; };  // no padding: compared bytewise
  thread_local Key key{};
  thread_local TreeFwdMaps mp;
  const Key k{t.x_leaf, Wl_il, U_il, d.E, d.H, d.Ep, d.P2, d.Nmax, d.rnn};
  if (memcmp(&k, &key, sizeof k) != 0) {
    const int ngh = d.rnn ? d.H : 5 * d.H;
    bool ok = true;
    if (!d.rnn) {  // the TreeRNN has no leaf GEMM
      ok = make_tmap_bf16(&mp.x_leaf, t.x_leaf, d.E, d.Nmax, d.Ep, 128);
      ok = ok && make_tmap_bf16(&mp.w_leaf, Wl_il, d.E, 3ull * d.H, d.Ep, 48);
    }
    ok = ok && make_tmap_bf16(&mp.stage_h, t.stage_h, 2ull * d.H, d.Nmax, d.P2, 128);
    ok = ok && make_tmap_bf16(&mp.u, U_il, 2ull * d.H, (uint64_t)ngh, d.P2, 80);
    ok = ok && make_tmap_bf16(&mp.stage_h32, t.stage_h, 2ull * d.H, d.Nmax, d.P2, 32);
    if (!ok) { key = Key{}; return cudaErrorInvalidValue; }
    key = k;
  }
  const bool six = tree_smem_fwd(6, d.H) <= 227 * 1024;  // ring depth that fits beside the staging
  const int smem = tree_smem_fwd(six ? 6 : 4, d.H);
  const void *fn = d.rnn ? (six ? (const void *)tree_fwd_kernel<6, true> : (const void *)tree_fwd_kernel<4, true>)
                         : (six ? (const void *)tree_fwd_kernel<6, false> : (const void *)tree_fwd_kernel<4, false>);
  cudaError_t e = set_smem_once(fn, smem);
  if (e != cudaSuccess) return e;
  TreeBufs tt = t;
  TreeDims dd = d;
  TreeSched ss = s;
  void *args[] = {&mp, &tt, &dd, &ss, (void *)&st};
  return coop(fn, grid, smem, args, str);
}

// =============================================================================== cell backward
// The cell backward of one (node, unit) once its dh is final (a node's h feeds only its parent,
// or the classifier for a root) and its dc too (written by the parent's cell backward; 0 for a
// root): rb(dz) into the node's DZ row and dc into both children. rk = irank[n] (>= 0: internal,
// row rk of the internal-node arrays; < 0: leaf at level-0 position -1 - rk); kl / kr = the
// node's children (internal nodes only). TreeRNN: dz = dh (1 - h^2), leaves are frozen.
struct CellIn { float g[5], c, cl, cr, dc; };
// loads only (read-only data through the non-coherent path; dc is written by this kernel's
// earlier levels, so it goes through L2), so a batch of items can have all its loads in flight
template <bool RNN>
JN_DEV void cell_load(const TreeBufs &t, const TreeDims &d, int n, int rk, int u, CellIn &x) {
  const int H = d.H;
  if (rk >= 0) {
    x.c = __ldg(t.c_int + (size_t)rk * H + u);
    if constexpr (!RNN) {
      const float *g = t.gates_int + (size_t)rk * 5 * H + 5 * u;
#pragma unroll
      for (int q = 0; q < 5; ++q) x.g[q] = __ldg(g + q);
      x.cl = __ldg(t.stage_c + (size_t)rk * 2 * H + u);
      x.cr = __ldg(t.stage_c + (size_t)rk * 2 * H + H + u);
      x.dc = __ldcg(t.dc_node + (size_t)n * H + u);
    }
  } else if constexpr (!RNN) {
    const int pos = -1 - rk;
    const float *g = t.gates_leaf + (size_t)pos * 3 * H + 3 * u;
#pragma unroll
    for (int q = 0; q < 3; ++q) x.g[q] = __ldg(g + q);
    x.c = __ldg(t.c_leaf + (size_t)pos * H + u);
    x.dc = __ldcg(t.dc_node + (size_t)n * H + u);
  }
}
template <bool RNN>
JN_DEV void cell_apply(const TreeBufs &t, const TreeDims &d, int rk, int kl, int kr, int u, float dh,
                       const CellIn &x) {
  const int H = d.H;
  if (rk >= 0) {
    if constexpr (RNN) {
      t.DZ_int[(size_t)rk * d.P5 + u] = __float2bfloat16_rn(dh * (1.f - x.c * x.c));
    } else {
      const float ig = x.g[0], fl = x.g[1], fr = x.g[2], og = x.g[3], ug = x.g[4];
      const float tc = tanh_t(x.c);
      const float dout = dh * tc;
      const float dc = x.dc + dh * og * (1.f - tc * tc);
      __nv_bfloat16 *dz = t.DZ_int + (size_t)rk * d.P5 + 5 * u;
      dz[0] = __float2bfloat16_rn(dc * ug * ig * (1.f - ig));
      dz[1] = __float2bfloat16_rn(dc * x.cl * fl * (1.f - fl));
      dz[2] = __float2bfloat16_rn(dc * x.cr * fr * (1.f - fr));
      dz[3] = __float2bfloat16_rn(dout * og * (1.f - og));
      dz[4] = __float2bfloat16_rn(dc * ig * (1.f - ug * ug));
      t.dc_node[(size_t)kl * H + u] = dc * fl;
      t.dc_node[(size_t)kr * H + u] = dc * fr;
    }
  } else if constexpr (!RNN) {
    const int pos = -1 - rk;
    const float ig = x.g[0], og = x.g[1], ug = x.g[2];
    const float tc = tanh_t(x.c);
    const float dc = x.dc + dh * og * (1.f - tc * tc);
    __nv_bfloat16 *dz = t.DZ_leaf + (size_t)pos * d.P3 + 3 * u;
    dz[0] = __float2bfloat16_rn(dc * ug * ig * (1.f - ig));
    dz[1] = __float2bfloat16_rn(dh * tc * og * (1.f - og));
    dz[2] = __float2bfloat16_rn(dc * ig * (1.f - ug * ug));
  }
}
// Four consecutive units u0 .. u0+3 (u0 % 4 == 0, H % 4 == 0: every row and unit group 16-B
// aligned): 16-B loads, 8-/16-B stores.
struct CellIn4 { float4 g[5], c, cl, cr, dc; };
template <bool RNN>
JN_DEV void cell4_load(const TreeBufs &t, const TreeDims &d, int n, int rk, int u0, CellIn4 &x) {
  const int H = d.H;
  if (rk >= 0) {
    x.c = __ldg(reinterpret_cast<const float4 *>(t.c_int + rk * H + u0));
    if constexpr (!RNN) {
      const float4 *g = reinterpret_cast<const float4 *>(t.gates_int + rk * 5 * H + 5 * u0);
#pragma unroll
      for (int q = 0; q < 5; ++q) x.g[q] = __ldg(g + q);
      x.cl = __ldg(reinterpret_cast<const float4 *>(t.stage_c + rk * 2 * H + u0));
      x.cr = __ldg(reinterpret_cast<const float4 *>(t.stage_c + rk * 2 * H + H + u0));
      x.dc = __ldcg(reinterpret_cast<const float4 *>(t.dc_node + n * H + u0));
    }
  } else if constexpr (!RNN) {
    const int pos = -1 - rk;
    const float4 *g = reinterpret_cast<const float4 *>(t.gates_leaf + pos * 3 * H + 3 * u0);
#pragma unroll
    for (int q = 0; q < 3; ++q) x.g[q] = __ldg(g + q);
    x.c = __ldg(reinterpret_cast<const float4 *>(t.c_leaf + pos * H + u0));
    x.dc = __ldcg(reinterpret_cast<const float4 *>(t.dc_node + n * H + u0));
  }
}
JN_DEV float f4(const float4 &v, int i) { return i == 0 ? v.x : i == 1 ? v.y : i == 2 ? v.z : v.w; }
JN_DEV uint32_t pack_bf2(float a, float b) {
  const __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<const uint32_t *>(&h);
}
template <bool RNN>
JN_DEV void cell4_apply(const TreeBufs &t, const TreeDims &d, int rk, int kl, int kr, int u0, const float *dh,
                        const CellIn4 &x) {
  const int H = d.H;
  if (rk >= 0) {
    if constexpr (RNN) {
      float v[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) { const float h = f4(x.c, i); v[i] = dh[i] * (1.f - h * h); }
      *reinterpret_cast<uint2 *>(t.DZ_int + (size_t)rk * d.P5 + u0) = make_uint2(pack_bf2(v[0], v[1]), pack_bf2(v[2], v[3]));
    } else {
      const float *gf = reinterpret_cast<const float *>(x.g);  // 20 gates, 5 per unit
      float dz[20], dcl[4], dcr[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float ig = gf[5 * i], fl = gf[5 * i + 1], fr = gf[5 * i + 2], og = gf[5 * i + 3], ug = gf[5 * i + 4];
        const float tc = tanh_t(f4(x.c, i));
        const float dc = f4(x.dc, i) + dh[i] * og * (1.f - tc * tc);
        dz[5 * i] = dc * ug * ig * (1.f - ig);
        dz[5 * i + 1] = dc * f4(x.cl, i) * fl * (1.f - fl);
        dz[5 * i + 2] = dc * f4(x.cr, i) * fr * (1.f - fr);
        dz[5 * i + 3] = dh[i] * tc * og * (1.f - og);
        dz[5 * i + 4] = dc * ig * (1.f - ug * ug);
        dcl[i] = dc * fl;
        dcr[i] = dc * fr;
      }
      uint2 *o = reinterpret_cast<uint2 *>(t.DZ_int + (size_t)rk * d.P5 + 5 * u0);  // 40 B: 8-B aligned
#pragma unroll
      for (int q = 0; q < 5; ++q) o[q] = make_uint2(pack_bf2(dz[4 * q], dz[4 * q + 1]), pack_bf2(dz[4 * q + 2], dz[4 * q + 3]));
      *reinterpret_cast<float4 *>(t.dc_node + kl * H + u0) = make_float4(dcl[0], dcl[1], dcl[2], dcl[3]);
      *reinterpret_cast<float4 *>(t.dc_node + kr * H + u0) = make_float4(dcr[0], dcr[1], dcr[2], dcr[3]);
    }
  } else if constexpr (!RNN) {
    const int pos = -1 - rk;
    const float *gf = reinterpret_cast<const float *>(x.g);  // 12 gates, 3 per unit
    float dz[12];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float ig = gf[3 * i], og = gf[3 * i + 1], ug = gf[3 * i + 2];
      const float tc = tanh_t(f4(x.c, i));
      const float dc = f4(x.dc, i) + dh[i] * og * (1.f - tc * tc);
      dz[3 * i] = dc * ug * ig * (1.f - ig);
      dz[3 * i + 1] = dh[i] * tc * og * (1.f - og);
      dz[3 * i + 2] = dc * ig * (1.f - ug * ug);
    }
    uint2 *o = reinterpret_cast<uint2 *>(t.DZ_leaf + (size_t)pos * d.P3 + 3 * u0);  // 24 B
#pragma unroll
    for (int q = 0; q < 3; ++q) o[q] = make_uint2(pack_bf2(dz[4 * q], dz[4 * q + 1]), pack_bf2(dz[4 * q + 2], dz[4 * q + 3]));
  }
}

template <bool RNN>
JN_DEV void node_cell_bwd(const TreeBufs &t, const TreeDims &d, int n, int rk, int kl, int kr, int u, float dh) {
  CellIn x;
  cell_load<RNN>(t, d, n, rk, u, x);
  cell_apply<RNN>(t, d, rk, kl, kr, u, dh, x);
}

// =============================================================================== root classifier
// y = rb(h_root) rb(W_c)^T + b_c; loss = mean over trees of xent(y, label) (reading Q6);
// dy = (softmax - onehot) / B; dW_c = sum rb(dy)^T rb(h); db_c = sum rb(dy); dh_root = rb(dy) rb(W_c).
// Multi-block: block j owns trees [8j, 8j + 8) — their logits, softmax, loss rows and root dh —
// and writes its share of dW_c / db_c to root_part[j]; the last block to finish (counter in
// barrier word 32, zeroed by the step init) sums the shares in block order (deterministic).
constexpr int ROOT_TPB = 8;  // trees per block

__global__ void __launch_bounds__(256) tree_root_kernel(TreeBufs t, TreeDims d, TreeSched s, DevStatus *st) {
  pdl_enter();
  const int B = d.B, H = d.H, C = d.C;
  __shared__ float dyr[ROOT_TPB * 8];  // [tree][class] rounded dy (C <= 8)
  __shared__ float ysh[ROOT_TPB * 8];  // logits
  __shared__ int sroot[ROOT_TPB];
  __shared__ bool s_last;
  const int b0 = blockIdx.x * ROOT_TPB, nt = min(ROOT_TPB, B - b0);
  if (st->key != KEY_PASS) {
    for (int tr = threadIdx.x; tr < nt; tr += blockDim.x) t.rowloss[b0 + tr] = 0.f;
    return;
  }
  // logits: one warp per (tree, class) pair, lanes over the hidden units, warp reduction
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int p = wid; p < nt * C; p += nw) {
    const int tr = p / C, c = p - tr * C;
    float acc = 0.f;
    for (int k = lane; k < H; k += 32)
      acc += bf16_round(__ldg(t.root_h + (size_t)(b0 + tr) * H + k)) * bf16_round(__ldg(t.Wc + (size_t)c * H + k));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) ysh[p] = acc + t.bc[c];
  }
  __syncthreads();
  for (int tr = threadIdx.x; tr < nt; tr += blockDim.x) {
    const float *y = ysh + tr * C;
    float m = -INFINITY;
    for (int c = 0; c < C; ++c) m = fmaxf(m, y[c]);
    float sum = 0.f;
    for (int c = 0; c < C; ++c) sum += expf(y[c] - m);
    const float lse = m + logf(sum);
    int lab = t.label[b0 + tr];
    if (lab < 0 || lab >= C) {
      atomicOr(reinterpret_cast<unsigned int *>(&st->runtime_err), 2u);
      lab = 0;
    }
    t.rowloss[b0 + tr] = (lse - y[lab]) / B;
    for (int c = 0; c < C; ++c)
      dyr[tr * C + c] = bf16_round((expf(y[c] - lse) - (c == lab ? 1.f : 0.f)) / B);
    sroot[tr] = t.off[b0 + tr + 1] - 1;
  }
  __syncthreads();
  // this block's share of dW_c = sum_trees rb(dy)^T rb(h_root), db_c = sum_trees rb(dy)
  float *part = t.root_part + (size_t)blockIdx.x * (C * H + C);
  for (int e = threadIdx.x; e < C * H; e += blockDim.x) {
    const int c = e / H, k = e - c * H;
    float acc = 0.f;
    for (int tr = 0; tr < nt; ++tr) acc += dyr[tr * C + c] * bf16_round(__ldg(t.root_h + (size_t)(b0 + tr) * H + k));
    part[e] = acc;
  }
  for (int c = threadIdx.x; c < C; c += blockDim.x) {
    float acc = 0.f;
    for (int tr = 0; tr < nt; ++tr) acc += dyr[tr * C + c];
    part[C * H + c] = acc;
  }
  // dh of each root node (dc of a root = 0) and the root's cell backward: the backward kernel
  // then starts with the top level's dgrad
  const int uq = (H & 3) == 0 ? 4 : 1;  // units per item (16-B vectors when H % 4 == 0)
  for (int e = threadIdx.x; e < nt * (H / uq); e += blockDim.x) {
    const int tr = e / (H / uq), k = (e - tr * (H / uq)) * uq;
    const int root = sroot[tr];
    if (root < 0 || root >= d.N) continue;
    float acc[4] = {0.f, 0.f, 0.f, 0.f};
    for (int c = 0; c < C; ++c)
      for (int i = 0; i < uq; ++i) acc[i] += dyr[tr * C + c] * bf16_round(__ldg(t.Wc + (size_t)c * H + k + i));
    for (int i = 0; i < uq; ++i) t.dc_node[(size_t)root * H + k + i] = 0.f;
    const int rk = s.irank[root];
    const int kl = rk >= 0 && !d.rnn ? t.left[root] : 0, kr = rk >= 0 && !d.rnn ? t.right[root] : 0;
    if (uq == 4) {
      if (d.rnn) { CellIn4 x; cell4_load<true>(t, d, root, rk, k, x); cell4_apply<true>(t, d, rk, kl, kr, k, acc, x); }
      else { CellIn4 x; cell4_load<false>(t, d, root, rk, k, x); cell4_apply<false>(t, d, rk, kl, kr, k, acc, x); }
    } else if (d.rnn) {
      node_cell_bwd<true>(t, d, root, rk, kl, kr, k, acc[0]);
    } else {
      node_cell_bwd<false>(t, d, root, rk, kl, kr, k, acc[0]);
    }
  }
  // the last block sums the shares in block order
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = atomicAdd(t.barrier + 32, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  for (int e = threadIdx.x; e < C * H + C; e += blockDim.x) {
    float acc = 0.f;
    for (int j = 0; j < (int)gridDim.x; ++j) acc += __ldcg(t.root_part + (size_t)j * (C * H + C) + e);
    if (e < C * H) t.gWc[e] = acc;
    else t.gbc[e - C * H] = acc;
  }
  (void)s;
}

cudaError_t launch_tree_root(const TreeBufs &t, const TreeDims &d, const TreeSched &s,
                             DevStatus *st, cudaStream_t str) {
  if (d.C > 8) return cudaErrorInvalidValue;
  {
    const cudaError_t pe_ = launch_pdl(tree_root_kernel, dim3((d.B + ROOT_TPB - 1) / ROOT_TPB), dim3(256), 0, str, t, d, s, st);
    if (pe_ != cudaSuccess) return pe_;
  }
  return cudaGetLastError();
}

// =============================================================================== backward
struct TreeBwdMaps {
  CUtensorMap dz, ut, dz32, ut32;
};

// RES: the CTA keeps its 32-column slice of U^T (all K = 5H chunks, <= 96 KB) resident in shared
// memory for the whole launch and only streams dz per level (the dgrad's B operand does not
// change between levels); else both operands stream through the ring.
constexpr int T_RES_CHUNKS = 24;  // resident K chunks (5H <= 1536)
constexpr int T_RES_NT = 16;  // narrow tiles: 2H / 16 CTAs share each level's fused epilogue

// Per tile row (a parent of the level): its two children, their internal ranks and (internal
// children) the grandchildren that receive dc — loaded while the MMAs run.
struct BwdRowMeta { int ch[2], rk[2], gk[2][2]; };

template <bool RES, bool RNN>
__global__ void __launch_bounds__(TT, 1) tree_bwd_kernel(const __grid_constant__ TreeBwdMaps mp,
                                                         TreeBufs t, TreeDims d, TreeSched s,
                                                         const DevStatus *st) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t *base = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                              ~uintptr_t(1023));
  constexpr int BNT = RES ? T_RES_NT : 64;
  constexpr int BW_STAGES = RES ? T_STAGES : 6;  // streamed B: room for the staged 64-column tile
  Ring rg;
  rg.sA = base;
  rg.sB = base + BW_STAGES * T_ASTAGE;
  uint8_t *after = RES ? rg.sB + T_RES_CHUNKS * T_RES_NT * 128 : rg.sB + BW_STAGES * T_BSTAGE;
  rg.full = reinterpret_cast<uint64_t *>(after);
  rg.empty = rg.full + BW_STAGES;
  rg.tfull = rg.empty + BW_STAGES;
  uint64_t *bres_bar = rg.tfull + 1;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bres_bar + 1);
  rg.zst = reinterpret_cast<float *>(after + 256);
  BwdRowMeta *meta = reinterpret_cast<BwdRowMeta *>(rg.zst + 128 * (BNT + 1));
  const int warp = threadIdx.x >> 5;
  const int H = d.H;
  const int NGH = RNN ? H : 5 * H;  // K of the dgrad (dz width)
  if (st->key != KEY_PASS) return;  // assumption failed: skip (uniform across CTAs)
  const int res_ntile = (2 * H + T_RES_NT - 1) / T_RES_NT;
  const int res_groups = gridDim.x / res_ntile;
  if (RES) {
    rg.sBres = rg.sB;
    rg.bres_bar = bres_bar;
    rg.bres_groups = res_groups;
    rg.bres_nn = (int)blockIdx.x < res_groups * res_ntile ? (int)blockIdx.x % res_ntile : -1;
  }
  if (threadIdx.x == 128) {
    for (int i = 0; i < BW_STAGES; ++i) { mbar_init(&rg.full[i], 1); mbar_init(&rg.empty[i], 1); }
    mbar_init(rg.tfull, T_NMW);
    mbar_init(bres_bar, 1);
    fence_barrier_init();
    if (RES && rg.bres_nn >= 0) {  // this CTA's slice of U^T, every K chunk, once
      const int nk = (NGH + 63) / 64;
      mbar_expect_tx(bres_bar, nk * T_RES_NT * 128);
      for (int c = 0; c < nk; ++c)
        tma_load_2d(rg.sB + c * T_RES_NT * 128, &mp.ut32, bres_bar, c * 64, rg.bres_nn * T_RES_NT);
    }
  }
  if (warp == 5) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  rg.tmem = *tmem_slot;
  rg.q = 0;
  rg.tiles = 0;
  const int L = s.meta[0], n0 = s.meta[2], nint = s.meta[3];
  const int gt = blockIdx.x * blockDim.x + threadIdx.x, gs = gridDim.x * blockDim.x;
  // Top-down over the internal levels. The dz rows of level l are complete when its turn comes:
  // the roots' by the classifier kernel, every other node's by its parent's level (higher).
  // Per level: [dh_l ; dh_r] = rb(dz) U lands per tile column, and since a
  // child's h feeds only its parent, that column of the child's dh is final — the epilogue runs
  // the child's cell backward right there (its DZ row, its children's dc; leaves too).
  // Per-level arrival counters instead of a grid barrier per level (as the forward): only the CTAs
  // with tiles at a level take part; each waits for the previous (higher) level's workers, then
  // arrives on its level's counter. A node's dz row / dc come from its parent's / grandparent's
  // level, which is higher still: the chain of release / acquire pairs orders those writes too.
  const int ntile_nb = RES ? res_ntile : (2 * H + BNT - 1) / BNT;
  auto workers = [&](int l) {
    const int mt = (s.lvl_off[l + 1] - s.lvl_off[l] + 127) / 128;
    return RES ? min(mt, res_groups) * res_ntile : min((int)gridDim.x, mt * ntile_nb);
  };
  for (int l = L - 1; l >= 1; --l) {
    const int p0 = s.lvl_off[l], cnt = s.lvl_off[l + 1] - p0, r0 = p0 - s.lvl_off[1];
    if ((int)blockIdx.x >= workers(l)) continue;
    if (l < L - 1) {
      if (threadIdx.x == 0) {
        const unsigned int target = (unsigned)workers(l + 1);
        unsigned int v;
        do {
          asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(t.bwd_lvl + (l + 1) * 32) : "memory");
        } while (v < target);
      }
      __syncthreads();
      fence_proxy_async_global();
    }
    tile_loop<BNT, 2, BW_STAGES>(rg, &mp.dz, &mp.ut, r0, cnt, 2 * H, NGH, [&](int row, int) {
      if (row >= 0) {
        BwdRowMeta m;
        const int n = s.order[p0 + row];
        m.ch[0] = t.left[n];
        m.ch[1] = t.right[n];
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          m.rk[c] = s.irank[m.ch[c]];
          m.gk[c][0] = m.rk[c] >= 0 && !RNN ? t.left[m.ch[c]] : 0;
          m.gk[c][1] = m.rk[c] >= 0 && !RNN ? t.right[m.ch[c]] : 0;
        }
        meta[threadIdx.x] = m;
      }
      return 0;
    }, [&](int, int nrows, int col0) {
      // every warp of the CTA over the tile's (row, 4-column) items, IB per thread with all
      // their loads issued before any store; scalar items when H % 4 != 0
      constexpr int IB = 2;
      const int nth = blockDim.x;
      if ((H & 3) == 0) {
        constexpr int NQ = BNT / 4;
        const int items = nrows * NQ;
        for (int i0 = threadIdx.x; i0 < items; i0 += nth * IB) {
          CellIn4 x[IB];
          int rl[IB], k[IB];
#pragma unroll
          for (int b = 0; b < IB; ++b) {
            const int i = i0 + nth * b;
            rl[b] = i / NQ;
            k[b] = col0 + 4 * (i - rl[b] * NQ);
            if (i < items && k[b] < 2 * H) {
              const int side = k[b] >= H ? 1 : 0;
              const BwdRowMeta &m = meta[rl[b]];
              cell4_load<RNN>(t, d, m.ch[side], m.rk[side], k[b] - side * H, x[b]);
            }
          }
#pragma unroll
          for (int b = 0; b < IB; ++b) {
            if (i0 + nth * b < items && k[b] < 2 * H) {
              const int side = k[b] >= H ? 1 : 0;
              const BwdRowMeta &m = meta[rl[b]];
              cell4_apply<RNN>(t, d, m.rk[side], m.gk[side][0], m.gk[side][1], k[b] - side * H,
                               rg.zst + rl[b] * (BNT + 1) + (k[b] - col0), x[b]);
            }
          }
        }
      } else {
        const int items = nrows * BNT;
        for (int i = threadIdx.x; i < items; i += nth) {
          const int rl = i / BNT, j = i - rl * BNT, k = col0 + j;
          if (k >= 2 * H) continue;
          const int side = k >= H ? 1 : 0;
          const BwdRowMeta &m = meta[rl];
          node_cell_bwd<RNN>(t, d, m.ch[side], m.rk[side], m.gk[side][0], m.gk[side][1], k - side * H,
                             rg.zst[rl * (BNT + 1) + j]);
        }
      }
    }, (NGH + 63) / 64 >= 16 ? (RES ? 4 : 3) : ((NGH + 63) / 64 >= 8 ? 2 : 1),  // a fixed warp per stage
       t.dbg ? t.dbg + 3 * 256 * 256 * 2 + ((size_t)l * 256 + blockIdx.x) * 4 : nullptr, &mp.dz32);
    fence_proxy_async_global();  // the children's DZ rows feed the next level's TMA loads
    __syncthreads();  // every thread's stores of the level precede the release (bar.sync cumulativity)
    if (threadIdx.x == 0) asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(t.bwd_lvl + l * 32) : "memory");
  }
  // zero the dz rows of the last partial 64-row K chunk of the wgrad GEMMs
  for (long long e = gt; e < (long long)(((nint + 63) & ~63) - nint) * d.P5; e += gs)
    t.DZ_int[(size_t)nint * d.P5 + e] = __float2bfloat16_rn(0.f);
  if constexpr (!RNN)
    for (long long e = gt; e < (long long)(((n0 + 63) & ~63) - n0) * d.P3; e += gs)
      t.DZ_leaf[(size_t)n0 * d.P3 + e] = __float2bfloat16_rn(0.f);
  tc_fence_before();
  __syncthreads();
  if (warp == 5) tmem_dealloc(rg.tmem, 512);
  (void)st;
}

cudaError_t launch_tree_bwd(const TreeBufs &t, const TreeDims &d, const TreeSched &s,
                            const __nv_bfloat16 *UT_il, int grid, const DevStatus *st,
                            cudaStream_t str) {
  struct Key { const void *a, *b; long long H, P5, Nmax; };  // once per workspace (see the forward)
  thread_local Key key{};
  thread_local TreeBwdMaps mp;
  const uint64_t ngh = d.rnn ? (uint64_t)d.H : 5ull * d.H;
  const Key k{t.DZ_int, UT_il, d.H, d.P5, d.Nmax + ((long long)d.rnn << 40)};
  if (memcmp(&k, &key, sizeof k) != 0) {
    bool ok = make_tmap_bf16(&mp.dz, t.DZ_int, ngh, d.Nmax, d.P5, 128);
    ok = ok && make_tmap_bf16(&mp.ut, UT_il, ngh, 2ull * d.H, d.P5, 64);
    ok = ok && make_tmap_bf16(&mp.dz32, t.DZ_int, ngh, d.Nmax, d.P5, 32);
    ok = ok && make_tmap_bf16(&mp.ut32, UT_il, ngh, 2ull * d.H, d.P5, T_RES_NT);
    if (!ok) { key = Key{}; return cudaErrorInvalidValue; }
    key = k;
  }
  const bool res = ((int)ngh + 63) / 64 <= T_RES_CHUNKS && grid >= (2 * d.H + T_RES_NT - 1) / T_RES_NT;
  const int stage = 256 + 128 * ((res ? T_RES_NT : 64) + 1) * 4 + 128 * (int)sizeof(BwdRowMeta);
  const int smem = 1024 + (res ? T_STAGES * T_ASTAGE + T_RES_CHUNKS * T_RES_NT * 128 : 6 * (T_ASTAGE + T_BSTAGE)) + stage;
  const void *fn = d.rnn ? (res ? (const void *)tree_bwd_kernel<true, true> : (const void *)tree_bwd_kernel<false, true>)
                         : (res ? (const void *)tree_bwd_kernel<true, false> : (const void *)tree_bwd_kernel<false, false>);
  cudaError_t e = set_smem_once(fn, smem);
  if (e != cudaSuccess) return e;
  TreeBufs tt = t;
  TreeDims dd = d;
  TreeSched ss = s;
  void *args[] = {&mp, &tt, &dd, &ss, (void *)&st};
  return coop(fn, grid, smem, args, str);
}

// =============================================================================== casts
__global__ void cast_il_kernel(const float *src, int H, int ng, int cols, __nv_bfloat16 *dst, int ld) {
  // one block-stride loop per destination row (32-bit index math: a weight has < 2^31 elements)
  const int R = ng * H;
  for (int ri = blockIdx.x; ri < R; ri += gridDim.x) {
    const int rc = (ri % ng) * H + ri / ng;
    const float *sr = src + (size_t)rc * cols;
    __nv_bfloat16 *dr = dst + (size_t)ri * ld;
    for (int k = threadIdx.x; k < ld; k += blockDim.x) dr[k] = __float2bfloat16_rn(k < cols ? sr[k] : 0.f);
  }
}
cudaError_t launch_cast_il(const float *src, int H, int ng, int cols, __nv_bfloat16 *dst, int ld,
                           cudaStream_t s) {
  cast_il_kernel<<<min(ng * H, 16 * 148), 256, 0, s>>>(src, H, ng, cols, dst, ld);
  return cudaGetLastError();
}
// dst[k][ri] = rb(src[rc][k]),  ri = ng*u + g <-> rc = g*H + u
__global__ void cast_il_T_kernel(const float *src, int H, int ng, int cols, __nv_bfloat16 *dst, int ld) {
  __shared__ float tile[32][33];
  const int ri0 = blockIdx.x * 32, k0 = blockIdx.y * 32;
  const int R = ng * H;
  for (int i = threadIdx.y; i < 32; i += 8) {
    const int ri = ri0 + i, k = k0 + threadIdx.x;
    tile[i][threadIdx.x] = (ri < R && k < cols) ? src[(size_t)((ri % ng) * H + ri / ng) * cols + k] : 0.f;
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += 8) {
    const int k = k0 + i, ri = ri0 + threadIdx.x;
    if (k < cols && ri < ld) dst[(size_t)k * ld + ri] = __float2bfloat16_rn(ri < R ? tile[threadIdx.x][i] : 0.f);
  }
}
cudaError_t launch_cast_il_T(const float *src, int H, int ng, int cols, __nv_bfloat16 *dst, int ld,
                             cudaStream_t s) {
  dim3 grid((ld + 31) / 32, (cols + 31) / 32);
  cast_il_T_kernel<<<grid, dim3(32, 8), 0, s>>>(src, H, ng, cols, dst, ld);
  return cudaGetLastError();
}

// The step's three operand copies in one launch: blocks [0, nl) cast W_leaf rows (interleaved by
// 3), [nl, nl + nu) cast U rows (interleaved by 5), the rest transpose 32 x 32 tiles of U into U^T.
__global__ void __launch_bounds__(256) tree_cast3_kernel(const float *Wl, __nv_bfloat16 *Wl_il, int ldw,
                                                         const float *U, __nv_bfloat16 *U_il, int ldu,
                                                         __nv_bfloat16 *UT_il, int ldut, int H, int E) {
  pdl_enter();
  __shared__ float tile[32][33];
  const int nl = 3 * H, nu = 5 * H;
  int bx = blockIdx.x;
  if (bx < nl + nu) {  // one destination row per block
    const bool leaf = bx < nl;
    const int ng = leaf ? 3 : 5, cols = leaf ? E : 2 * H, ld = leaf ? ldw : ldu;
    const int ri = leaf ? bx : bx - nl;
    const int rc = (ri % ng) * H + ri / ng;
    const float *sr = (leaf ? Wl : U) + (size_t)rc * cols;
    __nv_bfloat16 *dr = (leaf ? Wl_il : U_il) + (size_t)ri * ld;
    for (int k = threadIdx.x; k < ld; k += blockDim.x) dr[k] = __float2bfloat16_rn(k < cols ? sr[k] : 0.f);
    return;
  }
  bx -= nl + nu;  // transpose tile: dst[k][ri] = rb(U[rc][k]), ri = 5u + g <-> rc = g H + u
  const int ntr = (ldut + 31) / 32;
  const int ri0 = (bx % ntr) * 32, k0 = (bx / ntr) * 32, cols = 2 * H;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  for (int i = ty; i < 32; i += 8) {
    const int ri = ri0 + i, k = k0 + tx;
    tile[i][tx] = (ri < nu && k < cols) ? U[(size_t)((ri % 5) * H + ri / 5) * cols + k] : 0.f;
  }
  __syncthreads();
  for (int i = ty; i < 32; i += 8) {
    const int k = k0 + i, ri = ri0 + tx;
    if (k < cols && ri < ldut) UT_il[(size_t)k * ldut + ri] = __float2bfloat16_rn(ri < nu ? tile[tx][i] : 0.f);
  }
}
cudaError_t launch_tree_cast3(const float *Wl, __nv_bfloat16 *Wl_il, int ldw, const float *U,
                              __nv_bfloat16 *U_il, int ldu, __nv_bfloat16 *UT_il, int ldut, int H, int E,
                              cudaStream_t s) {
  const int tiles = ((ldut + 31) / 32) * ((2 * H + 31) / 32);
  {
    const cudaError_t pe_ = launch_pdl(tree_cast3_kernel, dim3(8 * H + tiles), dim3(256), 0, s, Wl, Wl_il, ldw, U, U_il, ldu, UT_il, ldut, H, E);
    if (pe_ != cudaSuccess) return pe_;
  }
  return cudaGetLastError();
}

}  // namespace jk
