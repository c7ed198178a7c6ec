// Microbenchmark: how fast can G CTAs (one per SM) pull the same / distinct S-byte block from L2
// into shared memory with cp.async.bulk, for various op sizes? Mimics one recurrent step.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/bb scripts/bench_bulk.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t s32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void k_bulk(const uint8_t *src, size_t per_cta_stride, int bytes, int op_bytes, int reps,
                       unsigned long long *out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  unsigned long long t0 = 0, t1 = 0;
  if (threadIdx.x == 0) {
    const uint8_t *s = src + per_cta_stride * blockIdx.x;
    for (int r = 0; r < reps; ++r) {
      if (r == 1) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s32(&bar)), "r"(bytes) : "memory");
      for (int o = 0; o < bytes; o += op_bytes) {
        const int n = min(op_bytes, bytes - o);
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                s32(sm + o)),
            "l"(s + o), "r"(n), "r"(s32(&bar))
            : "memory");
      }
      asm volatile(
          "{\n\t.reg .pred p;\n\tW:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W;\n\t}" ::"r"(
              s32(&bar)),
          "r"(r & 1)
          : "memory");
    }
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    out[blockIdx.x] = (t1 - t0) / (reps - 1);
  }
}

// 128 threads, 16-B vector loads -> st.shared (generic path)
__global__ void k_ldg(const uint8_t *src, size_t per_cta_stride, int bytes, int reps, unsigned long long *out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  unsigned long long t0 = 0, t1 = 0;
  const uint8_t *s = src + per_cta_stride * blockIdx.x;
  for (int r = 0; r < reps; ++r) {
    if (r == 1) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    for (int o = threadIdx.x * 16; o < bytes; o += blockDim.x * 16) {
      uint4 v;
      asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(s + o));
      *reinterpret_cast<uint4 *>(sm + o) = v;
    }
    __syncthreads();
  }
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
  if (threadIdx.x == 0) out[blockIdx.x] = (t1 - t0) / (reps - 1);
}

int main() {
  const int G = 41;
  uint8_t *src;
  cudaMalloc(&src, 64 << 20);
  cudaMemset(src, 1, 64 << 20);
  unsigned long long *out, h[148];
  cudaMalloc(&out, 148 * 8);
  cudaFuncSetAttribute(k_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 << 10);
  cudaFuncSetAttribute(k_ldg, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 << 10);
  const int sizes[] = {90112, 172032};
  const int ops[] = {8192, 16384, 49152, 172032};
  for (int grid : {1, 41, 82, 148})
    for (int bytes : sizes)
      for (int same = 0; same < 2; ++same) {
        for (int op : ops) {
          if (op > bytes && op != ops[3]) continue;
          k_bulk<<<grid, 32, 200 << 10>>>(src, same ? 0 : (size_t)bytes, bytes, op, 20, out);
          cudaDeviceSynchronize();
          cudaMemcpy(h, out, grid * 8, cudaMemcpyDeviceToHost);
          unsigned long long mx = 0, sum = 0;
          for (int i = 0; i < grid; ++i) { mx = h[i] > mx ? h[i] : mx; sum += h[i]; }
          printf("bulk grid=%3d bytes=%6d %s op=%6d : avg %6.0f ns max %6llu ns  (%.1f GB/s per SM)\n", grid, bytes,
                 same ? "same" : "dist", op, (double)sum / grid, mx, bytes / ((double)sum / grid));
        }
        for (int thr : {128, 256, 512}) {
          k_ldg<<<grid, thr, 200 << 10>>>(src, same ? 0 : (size_t)bytes, bytes, 20, out);
          cudaDeviceSynchronize();
          cudaMemcpy(h, out, grid * 8, cudaMemcpyDeviceToHost);
          unsigned long long mx = 0, sum = 0;
          for (int i = 0; i < grid; ++i) { mx = h[i] > mx ? h[i] : mx; sum += h[i]; }
          printf("ldg  grid=%3d bytes=%6d %s thr=%4d : avg %6.0f ns max %6llu ns  (%.1f GB/s per SM)\n", grid, bytes,
                 same ? "same" : "dist", thr, (double)sum / grid, mx, bytes / ((double)sum / grid));
        }
      }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
