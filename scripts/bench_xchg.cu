// Microbenchmark: per-step all-gather + synchronisation floor of a recurrent layer (one h block
// shared by every CTA of the layer each step), comparing exchange mechanisms on sm_100a.
//   V0 flags : global slice write + one release flag per CTA (one 128-B line each) + poll all +
//              acquire fence + bulk load of the whole block (current lm_rec.cu design)
//   V1 count : global slice write + red.release.gpu.add on a per-step counter + poll one word
//   V2 sync0 : V0 without data (flag all-to-all only)
//   V3 mcast : thread-block cluster; slice written to global, then ONE multicast bulk copy of the
//              slice into every cluster CTA's smem, completion = mbarrier complete_tx (no flags)
//   V4 dsst  : cluster; slice pushed with st.shared::cluster.v4 to every peer, then a remote
//              release-arrive on each peer's mbarrier
//   V5 dsbulk: cluster; slice staged in own smem, cp.async.bulk smem->peer smem per peer
//   G5 dpoll : grid; no flags and no fences: every word of the slice carries the step number and
//              the consumers load the whole block with relaxed vector loads, re-loading any
//              granule that still holds an older value (the data is its own flag)
//   G6 dpoll1: G5, but warp 0 first polls one word per producer slice before the full load
//   G7 bpoll : no flags and no fences: the consumer bulk-copies the block speculatively right
//              after writing its own slice, every thread checks the words it owns in shared
//              memory, and pieces holding an older step's words are copied again until clean
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/bx.bin scripts/bench_xchg.cu
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t s32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void bar_init(uint64_t *b, unsigned n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(s32(b)), "r"(n));
}
__device__ __forceinline__ void bar_expect(uint64_t *b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bar_wait(uint64_t *b, unsigned par) {
  asm volatile("{\n\t.reg .pred p;\n\tW%=:\n\tmbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n\t@!p bra W%=;\n\t}" ::"r"(s32(b)),
               "r"(par) : "memory");
}
__device__ __forceinline__ uint32_t crank() { uint32_t r; asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r)); return r; }
__device__ __forceinline__ uint32_t cnum() { uint32_t r; asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r)); return r; }
__device__ __forceinline__ uint32_t mapa(uint32_t a, uint32_t r) {
  uint32_t o; asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(o) : "r"(a), "r"(r)); return o;
}
__device__ __forceinline__ void csync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t;
}

constexpr int FS = 32;  // flag stride (words): one 128-B line per flag

// ----------------------------------------------------------------------------- grid variants
template <int MODE>
__global__ void k_grid(uint8_t *xbuf, unsigned *flags, int steps, int slice, unsigned long long *out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ __align__(8) uint64_t bar;
  const int G = gridDim.x;
  if (threadIdx.x == 0) { bar_init(&bar, 1); asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
  __syncthreads();
  unsigned long long t0 = 0;
  const size_t blk = (size_t)G * slice;
  for (int t = 0; t < steps; ++t) {
    if (t == 8 && threadIdx.x == 0) t0 = gtime();
    if (MODE != 2) {
      uint8_t *dst = xbuf + (size_t)(t % 64) * blk + (size_t)blockIdx.x * slice;
      for (int o = threadIdx.x * 16; o < slice; o += blockDim.x * 16)
        *reinterpret_cast<uint4 *>(dst + o) = make_uint4(t, t, t, t);
      asm volatile("fence.proxy.async.global;" ::: "memory");
    }
    if (MODE == 4) {  // every warp releases its own writes: no CTA barrier before the flag
      __syncwarp();
      if ((threadIdx.x & 31) == 0) asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(flags + blockIdx.x * FS), "r"(1) : "memory");
    } else {
      __syncthreads();
      if (threadIdx.x == 0) {
        if (MODE == 1) asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(flags + (t % 64) * FS), "r"(1) : "memory");
        else asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(flags + blockIdx.x * FS), "r"(t + 1) : "memory");
      }
    }
    if (threadIdx.x < 32) {
      if (MODE == 3 || MODE == 4) {
        const unsigned need = MODE == 4 ? 4u * (unsigned)(t + 1) : (unsigned)(t + 1);
        for (int c = threadIdx.x; c < G; c += 32) {
          unsigned x;
          do { asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(x) : "l"(flags + c * FS) : "memory"); } while (x < need);
        }
        __syncwarp();
      } else if (MODE == 1) {
        if (threadIdx.x == 0) {
          unsigned x;
          const unsigned tgt = (unsigned)G * (unsigned)(t / 64 + 1);
          do { asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(x) : "l"(flags + (t % 64) * FS) : "memory"); } while (x < tgt);
        }
        __syncwarp();
      } else {
        for (int c = threadIdx.x; c < G; c += 32) {
          unsigned x;
          do { asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(x) : "l"(flags + c * FS) : "memory"); } while (x < (unsigned)t + 1);
        }
        __syncwarp();
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
      }
      asm volatile("fence.proxy.async.global;" ::: "memory");
      if (MODE != 2 && threadIdx.x == 0) {
        const uint32_t bytes = (uint32_t)blk;
        bar_expect(&bar, bytes);
        const uint8_t *src = xbuf + (size_t)(t % 64) * blk;
        for (uint32_t o = 0; o < bytes; o += 32768) {
          const uint32_t n = bytes - o < 32768 ? bytes - o : 32768;
          asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(s32(sm + o)),
                       "l"(src + o), "r"(n), "r"(s32(&bar)) : "memory");
        }
        bar_wait(&bar, t & 1);
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) out[blockIdx.x] = (gtime() - t0) / (steps - 8);
}


// ----------------------------------------------------------------------------- data-as-flag
template <int MODE>
__global__ void k_dpoll(uint8_t *xbuf, int steps, int slice, unsigned long long *out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  const int G = gridDim.x;
  unsigned long long t0 = 0;
  const size_t blk = (size_t)G * slice;
  for (int t = 0; t < steps; ++t) {
    if (t == 8 && threadIdx.x == 0) t0 = gtime();
    const unsigned tag = (unsigned)t + 1u;
    uint8_t *base = xbuf + (size_t)(t % 64) * blk;
    uint8_t *dst = base + (size_t)blockIdx.x * slice;
    for (int o = threadIdx.x * 16; o < slice; o += blockDim.x * 16)
      *reinterpret_cast<uint4 *>(dst + o) = make_uint4(tag, tag, tag, tag);
    if (MODE == 6 && threadIdx.x < 32) {
      for (int c = threadIdx.x; c < G; c += 32) {
        unsigned x;
        do { asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(x) : "l"(base + (size_t)c * slice + slice - 4) : "memory"); } while (x != tag);
      }
    }
    if (MODE == 6) __syncthreads();
    constexpr int NB = 8;
    for (size_t o0 = (size_t)threadIdx.x * 16; o0 < blk; o0 += (size_t)blockDim.x * 16 * NB) {
      uint4 v[NB];
#pragma unroll
      for (int k = 0; k < NB; ++k) {
        const size_t o = o0 + (size_t)k * blockDim.x * 16;
        if (o < blk)
          asm volatile("ld.relaxed.gpu.global.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v[k].x), "=r"(v[k].y), "=r"(v[k].z), "=r"(v[k].w) : "l"(base + o) : "memory");
      }
#pragma unroll
      for (int k = 0; k < NB; ++k) {
        const size_t o = o0 + (size_t)k * blockDim.x * 16;
        if (o >= blk) continue;
        while (v[k].x != tag || v[k].y != tag || v[k].z != tag || v[k].w != tag)
          asm volatile("ld.relaxed.gpu.global.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v[k].x), "=r"(v[k].y), "=r"(v[k].z), "=r"(v[k].w) : "l"(base + o) : "memory");
        *reinterpret_cast<uint4 *>(sm + o) = v[k];
      }
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
  }
  if (threadIdx.x == 0) out[blockIdx.x] = (gtime() - t0) / (steps - 8);
}


// bulk-copy speculation: pieces of PB bytes; a piece is clean when none of its words holds an
// older tag (every word of step t's block carries t + 1)
template <int PB>
__global__ void k_bpoll(uint8_t *xbuf, int steps, int slice, unsigned long long *out, unsigned *retries) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ __align__(8) uint64_t bar;
  __shared__ int s_bad[512];
  __shared__ int s_nbad;
  const int G = gridDim.x;
  if (threadIdx.x == 0) { bar_init(&bar, 1); asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
  __syncthreads();
  unsigned long long t0 = 0;
  unsigned nretry = 0;
  uint32_t phase = 0;
  const size_t blk = (size_t)G * slice;
  const int npc = (int)((blk + PB - 1) / PB);
  for (int t = 0; t < steps; ++t) {
    if (t == 8 && threadIdx.x == 0) t0 = gtime();
    const unsigned tag = (unsigned)t + 1u;
    uint8_t *base = xbuf + (size_t)(t % 64) * blk;
    uint8_t *dst = base + (size_t)blockIdx.x * slice;
    for (int o = threadIdx.x * 16; o < slice; o += blockDim.x * 16)
      *reinterpret_cast<uint4 *>(dst + o) = make_uint4(tag, tag, tag, tag);
    // first round: every piece
    if (threadIdx.x == 0) { s_nbad = npc; }
    for (int i = threadIdx.x; i < npc; i += blockDim.x) s_bad[i] = i;
    __syncthreads();
    while (true) {
      const int nb = s_nbad;
      if (nb == 0) break;
      if (threadIdx.x == 0) {
        asm volatile("fence.proxy.async.global;" ::: "memory");
        uint32_t bytes = 0;
        for (int i = 0; i < nb; ++i) {
          const size_t o = (size_t)s_bad[i] * PB;
          bytes += (uint32_t)min((size_t)PB, blk - o);
        }
        bar_expect(&bar, bytes);
        for (int i = 0; i < nb; ++i) {
          const size_t o = (size_t)s_bad[i] * PB;
          const uint32_t n = (uint32_t)min((size_t)PB, blk - o);
          asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(s32(sm + o)),
                       "l"(base + o), "r"(n), "r"(s32(&bar)) : "memory");
        }
      }
      bar_wait(&bar, phase & 1);
      ++phase;
      __syncthreads();
      if (threadIdx.x == 0) s_nbad = 0;
      __syncthreads();
      // verify: thread handles words of the re-copied pieces
      for (int i = 0; i < nb; ++i) {
        const size_t o = (size_t)s_bad[i] * PB;
        const int n = (int)min((size_t)PB, blk - o);
        bool bad = false;
        for (int w = threadIdx.x * 16; w < n; w += blockDim.x * 16) {
          const uint4 v = *reinterpret_cast<const uint4 *>(sm + o + w);
          bad |= v.x != tag || v.y != tag || v.z != tag || v.w != tag;
        }
        if (__syncthreads_or(bad)) {
          if (threadIdx.x == 0) { s_bad[s_nbad++] = s_bad[i]; }
        }
      }
      __syncthreads();
      if (s_nbad && threadIdx.x == 0) ++nretry;
      __syncthreads();
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) { out[blockIdx.x] = (gtime() - t0) / (steps - 8); retries[blockIdx.x] = nretry; }
}

// ----------------------------------------------------------------------------- cluster variants
template <int MODE>
__global__ void k_clu(uint8_t *xbuf, int steps, int slice, unsigned long long *out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ __align__(8) uint64_t bar[2];
  const uint32_t cr = crank(), cn = cnum();
  const size_t blk = (size_t)cn * slice;
  uint8_t *buf0 = sm;                 // two receive buffers of blk bytes
  uint8_t *stage = sm + 2 * blk;      // V5 staging
  if (threadIdx.x == 0) {
    bar_init(&bar[0], MODE == 4 ? cn : 1);
    bar_init(&bar[1], MODE == 4 ? cn : 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  csync();
  unsigned long long t0 = 0;
  const int cid = blockIdx.x / cn;
  for (int t = 0; t < steps; ++t) {
    if (t == 8 && threadIdx.x == 0) t0 = gtime();
    const int s = t & 1;
    if (threadIdx.x == 0 && MODE != 4) bar_expect(&bar[s], (unsigned)blk);
    if (MODE == 3) {
      uint8_t *dst = xbuf + ((size_t)cid * 64 + (t % 64)) * blk + (size_t)cr * slice;
      for (int o = threadIdx.x * 16; o < slice; o += blockDim.x * 16)
        *reinterpret_cast<uint4 *>(dst + o) = make_uint4(t, t, t, t);
      asm volatile("fence.proxy.async.global;" ::: "memory");
      __syncthreads();
      if (threadIdx.x == 0) {
        const uint16_t mask = (uint16_t)((1u << cn) - 1);
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1], %2, [%3], %4;" ::"r"(
                         s32(buf0 + s * blk + cr * slice)),
                     "l"(dst), "r"((uint32_t)slice), "r"(s32(&bar[s])), "h"(mask) : "memory");
      }
    } else if (MODE == 4) {
      for (uint32_t p = 0; p < cn; ++p) {
        const uint32_t rb = mapa(s32(buf0 + s * blk + cr * slice), p);
        for (int o = threadIdx.x * 16; o < slice; o += blockDim.x * 16)
          asm volatile("st.shared::cluster.v4.u32 [%0], {%1, %1, %1, %1};" ::"r"(rb + o), "r"(t) : "memory");
      }
      __syncthreads();
      if (threadIdx.x < cn) {
        const uint32_t rbar = mapa(s32(&bar[s]), threadIdx.x);
        asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(rbar) : "memory");
      }
    } else {  // MODE 5
      for (int o = threadIdx.x * 16; o < slice; o += blockDim.x * 16)
        *reinterpret_cast<uint4 *>(stage + s * slice + o) = make_uint4(t, t, t, t);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncthreads();
      if (threadIdx.x < cn) {
        const uint32_t p = threadIdx.x;
        const uint32_t rdst = mapa(s32(buf0 + s * blk + cr * slice), p);
        const uint32_t rbar = mapa(s32(&bar[s]), p);
        asm volatile("cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(rdst),
                     "r"(s32(stage + s * slice)), "r"((uint32_t)slice), "r"(rbar) : "memory");
      }
    }
    if (threadIdx.x == 0) bar_wait(&bar[s], (t >> 1) & 1);
    __syncthreads();
  }
  csync();
  if (threadIdx.x == 0) out[blockIdx.x] = (gtime() - t0) / (steps - 8);
}

static void report(const char *name, int G, int cs, int slice, unsigned long long *d, cudaError_t e) {
  std::vector<unsigned long long> h(G);
  cudaMemcpy(h.data(), d, G * 8, cudaMemcpyDeviceToHost);
  std::sort(h.begin(), h.end());
  printf("%-7s G=%3d cluster=%2d slice=%6d block=%7d : med %6llu max %6llu ns/step (%s)\n", name, G, cs, slice, cs ? cs * slice : G * slice,
         h[G / 2], h[G - 1], cudaGetErrorString(e));
}

int main() {
  uint8_t *xbuf;
  unsigned *flags;
  unsigned long long *out;
  const int steps = 400;
  cudaMalloc(&xbuf, 1 << 30);
  cudaMalloc(&flags, 1 << 20);
  cudaMalloc(&out, 1024 * 8);
  void *gf[] = {(void *)k_grid<0>, (void *)k_grid<1>, (void *)k_grid<2>, (void *)k_grid<3>, (void *)k_grid<4>};
  const char *gn[] = {"flags", "count", "sync0", "acqpoll", "warprel"};
  for (auto f : gf) cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 << 10);
  if (getenv("BX_BPOLL")) {
    unsigned *retries;
    cudaMalloc(&retries, 1024 * 4);
    cudaFuncSetAttribute(k_bpoll<8192>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 << 10);
    cudaFuncSetAttribute(k_bpoll<32768>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 << 10);
    cudaFuncSetAttribute(gf[3], cudaFuncAttributeMaxDynamicSharedMemorySize, 200 << 10);
    for (int G : {41, 82})
      for (int slice : {2048}) {
        for (int m = 0; m < 3; ++m) {
          cudaMemset(flags, 0, 1 << 20);
          cudaMemset(xbuf, 0, 1 << 30);
          int st = steps, sl = slice;
          void *args[] = {&xbuf, &flags, &st, &sl, &out};
          void *args2[] = {&xbuf, &st, &sl, &out, &retries};
          if (m == 0) cudaLaunchCooperativeKernel(gf[3], G, 128, args, 200 << 10, 0);
          else if (m == 1) cudaLaunchCooperativeKernel((void *)k_bpoll<8192>, G, 128, args2, 200 << 10, 0);
          else cudaLaunchCooperativeKernel((void *)k_bpoll<32768>, G, 128, args2, 200 << 10, 0);
          cudaError_t e = cudaDeviceSynchronize();
          const char *nm[] = {"acqpoll", "bpoll8K", "bpoll32K"};
          report(nm[m], G, 0, slice, out, e);
          if (m) {
            std::vector<unsigned> r(G);
            cudaMemcpy(r.data(), retries, G * 4, cudaMemcpyDeviceToHost);
            unsigned long long tot = 0;
            for (unsigned x : r) tot += x;
            printf("        retries per CTA-step: %.3f\n", (double)tot / G / steps);
          }
        }
      }
    return 0;
  }
  if (getenv("BX_DPOLL")) {
    void *df[] = {(void *)k_dpoll<5>, (void *)k_dpoll<6>};
    const char *dn[] = {"dpoll", "dpoll1"};
    for (auto f : df) cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 << 10);
    for (int G : {41, 82, 123})
      for (int slice : {2048}) {
        for (int m = 0; m < 3; ++m) {
          cudaMemset(flags, 0, 1 << 20);
          cudaMemset(xbuf, 0, 1 << 30);
          int st = steps, sl = slice;
          void *args[] = {&xbuf, &flags, &st, &sl, &out};
          void *args2[] = {&xbuf, &st, &sl, &out};
          for (int th : {128, 256}) {
            if (m == 0) { if (th == 256) continue; cudaLaunchCooperativeKernel(gf[3], G, th, args, 200 << 10, 0); }
            else cudaLaunchCooperativeKernel(df[m - 1], G, th, args2, 200 << 10, 0);
            cudaError_t e = cudaDeviceSynchronize();
            char nm[32];
            snprintf(nm, sizeof nm, "%s/%d", m == 0 ? "acqpoll" : dn[m - 1], th);
            report(nm, G, 0, slice, out, e);
          }
        }
      }
    return 0;
  }
  if (getenv("BX_GRID_ONLY")) {
    for (int G : {41, 82, 123})
      for (int slice : {2048}) {
        for (int m = 0; m < 5; ++m) {
          cudaMemset(flags, 0, 1 << 20);
          int st = steps, sl = slice;
          void *args[] = {&xbuf, &flags, &st, &sl, &out};
          cudaLaunchCooperativeKernel(gf[m], G, 128, args, 200 << 10, 0);
          cudaError_t e = cudaDeviceSynchronize();
          report(gn[m], G, 0, slice, out, e);
        }
      }
    return 0;
  }
  for (int G : {21, 41, 82, 123})
    for (int slice : {2048, 5376}) {
      if ((size_t)G * slice > 200000) continue;
      for (int m = 0; m < 5; ++m) {
        cudaMemset(flags, 0, 1 << 20);
        int st = steps, sl = slice;
        void *args[] = {&xbuf, &flags, &st, &sl, &out};
        cudaLaunchCooperativeKernel(gf[m], G, 128, args, 200 << 10, 0);
        cudaError_t e = cudaDeviceSynchronize();
        report(gn[m], G, 0, slice, out, e);
      }
    }
  void *cf[] = {(void *)k_clu<3>, (void *)k_clu<4>, (void *)k_clu<5>};
  const char *cnm[] = {"mcast", "dsst", "dsbulk"};
  for (auto f : cf) {
    cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 << 10);
    cudaFuncSetAttribute(f, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  }
  for (int cs : {4, 8, 12, 16})
    for (int slice : {2048, 5376, 10752}) {
      if ((size_t)cs * slice * 2 + 2 * slice > 220 * 1024) continue;
      for (int ncl : {1, 4, 8}) {
        for (int m = 0; m < 3; ++m) {
          cudaLaunchConfig_t cfg = {};
          cfg.gridDim = dim3(cs * ncl);
          cfg.blockDim = dim3(128);
          cfg.dynamicSmemBytes = 220 << 10;
          cudaLaunchAttribute at[1];
          at[0].id = cudaLaunchAttributeClusterDimension;
          at[0].val.clusterDim.x = cs;
          at[0].val.clusterDim.y = 1;
          at[0].val.clusterDim.z = 1;
          cfg.attrs = at;
          cfg.numAttrs = 1;
          int mx = 0;
          cudaOccupancyMaxActiveClusters(&mx, cf[m], &cfg);
          if (mx < ncl) { printf("%-7s cluster=%d x%d: only %d clusters co-resident, skip\n", cnm[m], cs, ncl, mx); continue; }
          cudaError_t e;
          if (m == 0) e = cudaLaunchKernelEx(&cfg, k_clu<3>, xbuf, steps, slice, out);
          else if (m == 1) e = cudaLaunchKernelEx(&cfg, k_clu<4>, xbuf, steps, slice, out);
          else e = cudaLaunchKernelEx(&cfg, k_clu<5>, xbuf, steps, slice, out);
          if (e == cudaSuccess) e = cudaDeviceSynchronize();
          char nm[32];
          snprintf(nm, sizeof nm, "%s/%d", cnm[m], ncl);
          report(nm, cs * ncl, cs, slice, out, e);
        }
      }
    }
  return 0;
}
