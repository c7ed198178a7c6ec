// Microbenchmark: back-to-back tcgen05.mma (kind::f16, bf16 in, fp32 accumulate into one TMEM
// tile) issue/execution rate for the small shapes of the recurrent kernels, SS mode (A and B in
// shared memory) and TS mode (A in TMEM). One CTA, one issuing thread, clock64 timing.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_1812_01329_b200/csrc -o scripts/bm.bin scripts/bench_mma.cu
#include <cstdio>
#include "common.cuh"
using namespace jk;

__device__ __forceinline__ void umma_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem_d),
      "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(acc));
}

template <int M, int N, bool TS, bool UNI, int NACC>
__global__ void k_mma(int nmma, int reps, int nacc, long long *out) {
  extern __shared__ uint8_t smraw[];
  uint8_t *sm = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smraw) + 1023) & ~uintptr_t(1023));
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t slot;
  // A: 128 rows x 64 KB region (chunks of 128 rows x 128 B = 16 KB), B: N rows chunks
  uint8_t *sA = sm, *sB = sm + 65536;
  for (int i = threadIdx.x; i < 65536 / 4 + 65536 / 4; i += blockDim.x) reinterpret_cast<uint32_t *>(sm)[i] = 0x3f803f80u;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  if (threadIdx.x < 32) tmem_alloc(&slot, 512);
  fence_proxy_async_shared();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  constexpr uint32_t idesc = umma_idesc_bf16(M, N, 0, 0);
  long long t0 = 0, t1 = 0;
  if (UNI && NACC > 100) {  // NACC-100 warps issue concurrently, each into its own accumulator
    const int nw = NACC - 100, w = threadIdx.x >> 5;
    __shared__ __align__(8) uint64_t bars[8];
    if (threadIdx.x < nw) { mbar_init(&bars[threadIdx.x], 1); }
    fence_barrier_init();
    __syncthreads();
    if (w < nw) {
      const uint32_t a0 = smem_u32(sA), b0 = smem_u32(sB);
      const uint32_t d = tmem + (uint32_t)(w * N);
      for (int r = 0; r < reps; ++r) {
        __syncwarp();
        if (r == 1) t0 = clock64();
        for (int i = 0; i < nmma / nw; ++i) {
          const uint32_t off = (uint32_t)(((i >> 2) & 3) * 16384 + (i & 3) * 32);
          uint32_t pred;
          asm volatile("{\n\t.reg .pred p;\n\telect.sync _|p, 0xffffffff;\n\tselp.u32 %0, 1, 0, p;\n\t}" : "=r"(pred));
          if (pred) umma_bf16(d, umma_desc_sw128(a0 + off, 16, 1024), umma_desc_sw128(b0 + off, 16, 1024), idesc, i > 0);
          __syncwarp();
        }
        if ((threadIdx.x & 31) == 0) umma_commit(&bars[w]);
        mbar_wait(&bars[w], r & 1);
      }
      t1 = clock64();
      if (threadIdx.x == 0) out[0] = (t1 - t0) / (reps - 1);
    }
  } else if (UNI) {  // whole warp 0 runs the loop (warp-uniform values), one elected lane issues
    if (threadIdx.x < 32) {
      const uint32_t a0 = smem_u32(sA), b0 = smem_u32(sB);
      for (int r = 0; r < reps; ++r) {
        if (r == 1) t0 = clock64();
#pragma unroll 4
        for (int i = 0; i < nmma; ++i) {
          const uint32_t off = (uint32_t)(((i >> 2) & 3) * 16384 + (i & 3) * 32);
          const uint32_t d = tmem + 256 + (uint32_t)((i & (NACC - 1)) * N);
          uint32_t pred;
          asm volatile("{\n\t.reg .pred p;\n\telect.sync _|p, 0xffffffff;\n\tselp.u32 %0, 1, 0, p;\n\t}" : "=r"(pred));
          if (pred) {
            if (TS) umma_ts(d, tmem + (uint32_t)((i & 31) * 8), umma_desc_sw128(b0 + off, 16, 1024), idesc, i >= NACC);
            else umma_bf16(d, umma_desc_sw128(a0 + off, 16, 1024), umma_desc_sw128(b0 + off, 16, 1024), idesc, i >= NACC);
          }
          __syncwarp();
        }
        if (threadIdx.x == 0) umma_commit(&bar);
        mbar_wait(&bar, r & 1);
      }
      t1 = clock64();
      if (threadIdx.x == 0) out[0] = (t1 - t0) / (reps - 1);
    }
  } else if (threadIdx.x == 0) {
    for (int r = 0; r < reps; ++r) {
      if (r == 1) t0 = clock64();
      for (int i = 0; i < nmma; ++i) {
        const int c = (i >> 2) & 3, kk = i & 3;  // cycle through 4 chunks of 64 K
        const uint32_t b = smem_u32(sB + c * 16384 + kk * 32);
        const int ac = i % nacc;  // independent accumulators, round robin
        const uint32_t d = tmem + 256 + (uint32_t)(ac * N);
        if (TS) {
          umma_ts(d, tmem + (uint32_t)((i & 31) * 8), umma_desc_sw128(b, 16, 1024), idesc, i >= nacc);
        } else {
          const uint32_t a = smem_u32(sA + c * 16384 + kk * 32);
          umma_bf16(d, umma_desc_sw128(a, 16, 1024), umma_desc_sw128(b, 16, 1024), idesc, i >= nacc);
        }
      }
      umma_commit(&bar);
      mbar_wait(&bar, r & 1);
    }
    t1 = clock64();
    out[0] = (t1 - t0) / (reps - 1);
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) tmem_dealloc(tmem, 512);
}

template <int M, int N, bool TS, bool UNI = false, int NACC = 1>
void run(const char *name, int nacc) {
  long long *d, h;
  cudaMalloc(&d, 8);
  auto f = k_mma<M, N, TS, UNI, NACC>;
  cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 << 10);
  for (int n : {16, 44, 164}) {
    f<<<1, 128, 160 << 10>>>(n, 20, nacc, d);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("%-3s M=%3d N=%3d nacc=%d nmma=%3d : %7lld cyc total, %6.1f cyc/mma (%s)\n", name, M, N, nacc, n, h,
           (double)h / n, cudaGetErrorString(e));
    if (e != cudaSuccess) exit(1);
  }
  cudaFree(d);
}

int main(int argc, char **argv) {
  const int M = atoi(argv[1]), N = atoi(argv[2]), ts = atoi(argv[3]), nacc = atoi(argv[4]);
#define R(m, n, t) if (M == m && N == n && ts == t) run<m, n, t>(t ? "TS" : "SS", nacc);
  R(128, 16, 0) R(128, 32, 0) R(128, 64, 0) R(128, 128, 0) R(128, 256, 0) R(64, 16, 0) R(64, 64, 0)
  R(128, 16, 1) R(128, 64, 1) R(128, 128, 1) R(64, 64, 1)
  if (ts == 2) {  // uniform-warp issue variants
    if (N == 256) { run<128, 256, false, true, 1>("US", 1); run<64, 256, false, true, 1>("US", 1); run<128, 256, true, true, 1>("UT", 1); }
    if (N == 64) { run<128, 64, false, true, 101>("MW1", 1); run<128, 64, false, true, 102>("MW2", 2); run<128, 64, false, true, 104>("MW4", 4); }
    if (N == 16) { run<128, 16, false, true, 104>("MW4", 4); run<64, 16, false, true, 104>("MW4", 4); run<64, 16, false, true, 102>("MW2", 2); }
    if (N == 32) { run<128, 32, false, true, 104>("MW4", 4); run<64, 32, false, true, 104>("MW4", 4); }
    if (N == 8) { run<64, 8, false, true, 1>("US", 1); run<64, 64, false, true, 1>("US", 1); run<64, 64, true, true, 1>("UT", 1); run<128, 32, false, true, 1>("US", 1); run<128, 128, false, true, 1>("US", 1);}
  }
  return 0;
}
