// fused_ar.h — host interface of the fused gradient reduction (NEXT-3): NCCL-owned symmetric
// windows for the gradient arena and the per-tile flags, descriptors for the GEMM epilogue,
// the null-step participant and the pre-commit wait (fused_ar.cu).
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>

#include "../../include/janus.h"
#include "gemm_tc.h"

namespace jk {

constexpr int FUSED_MAX_GEMMS = 8;

struct FusedArena {
  void *arena = nullptr, *flags = nullptr;  // ncclMemAlloc'd (NCCL-owned, like NCCL's own buffers)
  void *win = nullptr, *fwin = nullptr;     // ncclWindow_t of each
  size_t arena_bytes = 0, flag_bytes = 0;
  int nranks = 1, rank = 0;
  unsigned epoch = 0;                       // steps issued through this arena
};

// Tile geometry of one GEMM of the fused group (as gemm_group_tiling reports it)
struct FusedGeom {
  int M = 0, N = 0, ldc = 0, mblocks = 0, nblocks = 0, bn = 0;
  __host__ __device__ int tiles() const { return mblocks * nblocks; }
};

janus_status fused_ar_init(FusedArena &fa, void *comm, int world_size, size_t arena_bytes, size_t flag_bytes);
void fused_ar_destroy(FusedArena &fa, void *comm);
// descriptor of a GEMM whose C is at byte c_off of the arena and whose tiles' flags start at
// tile index tile_base of the flag window
FusedReduce fused_descriptor(const FusedArena &fa, size_t c_off, size_t tile_base, unsigned epoch);
cudaError_t launch_fused_null(const FusedReduce *fr, const FusedGeom *geo, int ng, cudaStream_t st);
cudaError_t launch_fused_wait(const FusedReduce &f0, int tiles, cudaStream_t st);

}  // namespace jk
