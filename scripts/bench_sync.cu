// Microbenchmark: the per-step synchronisation floor of the persistent recurrent kernels.
// G CTAs (co-resident) run STEPS steps; each step every CTA writes its slice (W bytes) of a fresh
// exchange block, publishes a release flag, waits for all G flags, and (optionally) bulk-loads the
// whole block (G*W bytes) into shared memory. Reports ns per step for several variants.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/bs.bin scripts/bench_sync.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t s32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int MODE>  // 0: flags only, 1: + write slice, 2: + write + bulk load, 3: + write + bulk, acq per lane
__global__ void k_sync(uint8_t *xbuf, unsigned *flags, int steps, int slice, unsigned long long *out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ __align__(8) uint64_t bar;
  const int G = gridDim.x;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  unsigned long long t0 = 0, t1;
  const size_t blk = (size_t)G * slice;
  for (int t = 0; t < steps; ++t) {
    if (t == 8 && threadIdx.x == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    if (MODE >= 1) {  // write my slice of block t (128 threads x 16 B strided)
      uint8_t *dst = xbuf + (size_t)t * blk + (size_t)blockIdx.x * slice;
      for (int o = threadIdx.x * 16; o < slice; o += blockDim.x * 16)
        *reinterpret_cast<uint4 *>(dst + o) = make_uint4(t, t, t, t);
      asm volatile("fence.proxy.async.global;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(flags + blockIdx.x), "r"(t + 1) : "memory");
    if (threadIdx.x < 32) {
      for (int c = threadIdx.x; c < G; c += 32) {
        unsigned x;
        do { asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(x) : "l"(flags + c) : "memory"); } while (x < (unsigned)t + 1);
      }
      __syncwarp();
      asm volatile("fence.acq_rel.gpu;" ::: "memory");
      asm volatile("fence.proxy.async.global;" ::: "memory");
      if (MODE >= 2 && threadIdx.x == 0) {
        const uint32_t bytes = (uint32_t)blk;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s32(&bar)), "r"(bytes) : "memory");
        const uint8_t *src = xbuf + (size_t)t * blk;
        for (uint32_t o = 0; o < bytes; o += 49152) {
          const uint32_t n = bytes - o < 49152 ? bytes - o : 49152;
          asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(s32(sm + o)),
                       "l"(src + o), "r"(n), "r"(s32(&bar)) : "memory");
        }
        asm volatile("{\n\t.reg .pred p;\n\tW:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W;\n\t}" ::"r"(s32(&bar)),
                     "r"(t & 1) : "memory");
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    out[blockIdx.x] = (t1 - t0) / (steps - 8);
  }
}

int main() {
  uint8_t *xbuf;
  unsigned *flags;
  unsigned long long *out, h[148];
  const int steps = 200;
  cudaMalloc(&xbuf, 512 << 20);
  cudaMalloc(&flags, 4096);
  cudaMalloc(&out, 148 * 8);
  void *fns[] = {(void *)k_sync<0>, (void *)k_sync<1>, (void *)k_sync<2>};
  for (auto f : fns) cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 << 10);
  for (int G : {11, 41, 82, 148})
    for (int slice : {2048, 8192}) {
      if ((size_t)G * slice > 190000) continue;
      for (int m = 0; m < 3; ++m) {
        cudaMemset(flags, 0, 4096);
        int st = steps, sl = slice;
        void *args[] = {&xbuf, &flags, &st, &sl, &out};
        cudaLaunchCooperativeKernel(fns[m], G, 128, args, 200 << 10, 0);
        cudaError_t e = cudaDeviceSynchronize();
        cudaMemcpy(h, out, G * 8, cudaMemcpyDeviceToHost);
        unsigned long long mx = 0;
        for (int i = 0; i < G; ++i) mx = h[i] > mx ? h[i] : mx;
        printf("G=%3d slice=%5d block=%7d mode=%d : %6llu ns/step (%s)\n", G, slice, G * slice, m, mx, cudaGetErrorString(e));
      }
    }
  return 0;
}
