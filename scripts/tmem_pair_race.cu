// Minimal CTA-pair TMEM allocation (tcgen05.alloc.cta_group::2) under compute-sanitizer
// racecheck: does the tool report the allocator's own shared-memory traffic as a hazard?
// nvcc -gencode arch=compute_100a,code=sm_100a -o tmem_pair_race tmem_pair_race.cu
#include <cstdio>
#include <cstdint>
__device__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__global__ void __cluster_dims__(2, 1, 1) k(int *out) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&slot)), "r"(512) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("barrier.cluster.arrive.release.aligned; barrier.cluster.wait.acquire.aligned;" ::: "memory");
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t t = slot;
  if (threadIdx.x == 0) out[blockIdx.x] = (int)t;
  asm volatile("barrier.cluster.arrive.release.aligned; barrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(t), "r"(512) : "memory");
}
int main() {
  int *d;
  cudaMalloc(&d, 8 * sizeof(int));
  k<<<4, 192>>>(d);
  cudaError_t e = cudaDeviceSynchronize();
  int h[4];
  cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
  printf("%s tmem %d %d %d %d\n", cudaGetErrorString(e), h[0], h[1], h[2], h[3]);
  return 0;
}
