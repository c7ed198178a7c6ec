// Microbenchmark: how fast ONE thread can issue tcgen05.mma (kind::f16) depending on how the
// instruction's operands are produced. Variants (one CTA, clock64 around n MMAs + commit/wait):
//   0  descriptors rebuilt per MMA from the shared-memory address (the recurrent kernels' style)
//   1  descriptors built once, advanced with 64-bit adds (+2 = 32 B per K=16 step), 1 MMA per asm
//   2  four MMAs per asm statement, descriptor offsets added inside the asm block
//   3  as 2, issued by the lane elect.sync picked (warp-uniform predicate) instead of threadIdx.x == 0
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_1812_01329_b200/csrc -o /tmp/bmi scripts/bench_mma_issue.cu
#include <cstdio>
#include <cstdlib>
#include "common.cuh"
using namespace jk;

JN_DEV void mma4(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t.reg .b64 a1, a2, a3, b1, b2, b3;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "add.s64 a1, %1, 2;\n\tadd.s64 a2, %1, 4;\n\tadd.s64 a3, %1, 6;\n\t"
      "add.s64 b1, %2, 2;\n\tadd.s64 b2, %2, 4;\n\tadd.s64 b3, %2, 6;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], a1, b1, %3, 1;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], a2, b2, %3, 1;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], a3, b3, %3, 1;\n\t}" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}

template <int M, int N, int V>
__global__ void k_issue(int nmma, int reps, long long *out) {
  extern __shared__ uint8_t smraw[];
  uint8_t *sm = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smraw) + 1023) & ~uintptr_t(1023));
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t slot;
  uint8_t *sA = sm, *sB = sm + 65536;
  for (int i = threadIdx.x; i < 65536 / 2; i += blockDim.x) reinterpret_cast<uint32_t *>(sm)[i] = 0x3f803f80u;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  if (threadIdx.x < 32) tmem_alloc(&slot, 512);
  fence_proxy_async_shared();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  constexpr uint32_t idesc = umma_idesc_bf16(M, N, 0, 0);
  uint32_t elected = 0;
  if (V == 3 && threadIdx.x < 32)
    asm volatile("{\n\t.reg .pred p;\n\telect.sync _|p, 0xffffffff;\n\tselp.u32 %0, 1, 0, p;\n\t}" : "=r"(elected));
  if (V == 3 ? elected != 0 : threadIdx.x == 0) {
    long long t0 = 0;
    const uint64_t da = umma_desc_sw128(smem_u32(sA), 16, 1024), db = umma_desc_sw128(smem_u32(sB), 16, 1024);
    for (int r = 0; r < reps; ++r) {
      if (r == 1) t0 = clock64();
      if (V == 0) {
        for (int i = 0; i < nmma; ++i) {
          const int c = (i >> 2) & 3, kk = i & 3;
          umma_bf16(tmem, umma_desc_sw128(smem_u32(sA + c * 16384 + kk * 32), 16, 1024),
                    umma_desc_sw128(smem_u32(sB + c * 16384 + kk * 32), 16, 1024), idesc, i > 0);
        }
      } else if (V == 1) {
        for (int i = 0; i < nmma; ++i) {
          const uint64_t o = (uint64_t)(((i >> 2) & 3) * 1024 + (i & 3) * 2);
          umma_bf16(tmem, da + o, db + o, idesc, i > 0);
        }
      } else {
        for (int i = 0; i < nmma; i += 4) {
          const uint64_t o = (uint64_t)(((i >> 2) & 3) * 1024);
          mma4(tmem, da + o, db + o, idesc, i > 0);
        }
      }
      umma_commit(&bar);
      mbar_wait(&bar, r & 1);
    }
    out[0] = (clock64() - t0) / (reps - 1);
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) tmem_dealloc(tmem, 512);
}

template <int M, int N, int V>
void run() {
  long long *d, h;
  cudaMalloc(&d, 8);
  auto f = k_issue<M, N, V>;
  cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 << 10);
  for (int n : {16, 44, 160}) {
    f<<<1, 128, 160 << 10>>>(n, 20, d);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("V%d M=%3d N=%3d nmma=%3d : %7lld cyc, %6.1f cyc/mma (%s)\n", V, M, N, n, h, (double)h / n,
           cudaGetErrorString(e));
    if (e != cudaSuccess) exit(1);
  }
  cudaFree(d);
}

int main() {
  run<64, 64, 0>(); run<64, 64, 1>(); run<64, 64, 2>();
  run<128, 64, 0>(); run<128, 64, 1>(); run<128, 64, 2>();
  run<128, 128, 1>(); run<128, 128, 2>();
  run<128, 256, 1>(); run<128, 256, 2>();
  run<64, 32, 2>(); run<64, 128, 2>();
  run<64, 64, 3>(); run<128, 64, 3>(); run<128, 256, 3>();
  return 0;
}
