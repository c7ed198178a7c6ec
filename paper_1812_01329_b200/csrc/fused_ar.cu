// fused_ar.cu — host side of the fused gradient reduction (NEXT-3; gemm_tc.h FusedReduce,
// fused_ar.cuh): NCCL symmetric windows for the gradient arena and the tile flags, the
// null-step participant kernel and the wait that precedes the commit.
#include <nccl.h>
#include <nccl_device.h>
#include <stdlib.h>

#include "fused_ar.cuh"
#include "fused_ar.h"

namespace jk {

static size_t r4k(size_t x) { return (x + 4095) & ~size_t(4095); }

janus_status fused_ar_init(FusedArena &fa, void *comm, int world_size, size_t arena_bytes, size_t flag_bytes) {
  if (fa.arena) return JANUS_OK;
  ncclComm_t c = static_cast<ncclComm_t>(comm);
  const ncclTeam_t lsa = ncclTeamLsa(c);
  if (lsa.nRanks != world_size) return JANUS_ERR_UNSUPPORTED;  // one node: every rank load/store accessible
  fa.nranks = lsa.nRanks;
  fa.rank = lsa.rank;
  fa.arena_bytes = r4k(arena_bytes);
  fa.flag_bytes = r4k(flag_bytes);
  ncclWindow_t w = nullptr, fw = nullptr;
  if (ncclMemAlloc(&fa.arena, fa.arena_bytes) != ncclSuccess ||
      ncclCommWindowRegister(c, fa.arena, fa.arena_bytes, &w, NCCL_WIN_COLL_SYMMETRIC) != ncclSuccess ||
      ncclMemAlloc(&fa.flags, fa.flag_bytes) != ncclSuccess ||
      ncclCommWindowRegister(c, fa.flags, fa.flag_bytes, &fw, NCCL_WIN_COLL_SYMMETRIC) != ncclSuccess)
    return JANUS_ERR_NCCL;
  fa.win = w;
  fa.fwin = fw;
  if (cudaMemset(fa.flags, 0, fa.flag_bytes) != cudaSuccess || cudaMemset(fa.arena, 0, fa.arena_bytes) != cudaSuccess ||
      cudaDeviceSynchronize() != cudaSuccess)
    return JANUS_ERR_CUDA;
  return JANUS_OK;
}

void fused_ar_destroy(FusedArena &fa, void *comm) {
  ncclComm_t c = static_cast<ncclComm_t>(comm);
  if (fa.win) ncclCommWindowDeregister(c, static_cast<ncclWindow_t>(fa.win));
  if (fa.fwin) ncclCommWindowDeregister(c, static_cast<ncclWindow_t>(fa.fwin));
  if (fa.arena) ncclMemFree(fa.arena);
  if (fa.flags) ncclMemFree(fa.flags);
  fa = FusedArena();
}

FusedReduce fused_descriptor(const FusedArena &fa, size_t c_off, size_t tile_base, unsigned epoch) {
  FusedReduce f;
  f.win = fa.win;
  f.c_off = c_off;
  f.fwin = fa.fwin;
  f.flag_off = tile_base * 8;
  f.nranks = fa.nranks;
  f.rank = fa.rank;
  f.epoch = epoch;
  const char *e = getenv("JANUS_FUSED_FORCE_PULL");  // test hook: exercise the data path on one rank
  f.force_pull = e && e[0] == '1';
  return f;
}

// A rank whose step does not run (dispatch miss / invalid arguments) still takes its part in
// every tile's protocol — it publishes its (stale) tiles and reduces the tiles it owns — so no
// owner waits forever; the agreement then aborts the step on every rank.
struct FusedNullArgs {
  FusedReduce fr[FUSED_MAX_GEMMS];
  FusedGeom geo[FUSED_MAX_GEMMS];
  int ng;
};
__global__ void __launch_bounds__(128) fused_null_kernel(FusedNullArgs a) {
  int b = blockIdx.x, g = 0;
  while (g + 1 < a.ng && b >= a.geo[g].tiles()) { b -= a.geo[g].tiles(); ++g; }
  const FusedGeom &ge = a.geo[g];
  const int mb = b % ge.mblocks, nb = b / ge.mblocks;
  fr_tile(a.fr[g], b, mb * 128, nb * ge.bn, ge.bn, ge.M, ge.N, ge.ldc, threadIdx.x);
}
cudaError_t launch_fused_null(const FusedReduce *fr, const FusedGeom *geo, int ng, cudaStream_t st) {
  if (ng > FUSED_MAX_GEMMS) return cudaErrorInvalidValue;
  FusedNullArgs a{};
  int tiles = 0;
  for (int g = 0; g < ng; ++g) { a.fr[g] = fr[g]; a.geo[g] = geo[g]; tiles += geo[g].tiles(); }
  a.ng = ng;
  fused_null_kernel<<<tiles, 128, 0, st>>>(a);
  return cudaGetLastError();
}

// every tile of this step reduced (its owner stored `epoch` into this rank's reduced flag)
__global__ void fused_wait_kernel(FusedReduce f, int tiles) {
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < tiles; t += gridDim.x * blockDim.x) {
    const unsigned *p = fr_flag(f, f.rank, t, 1);
    unsigned v;
    do {
      asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    } while (v < f.epoch);
  }
}
cudaError_t launch_fused_wait(const FusedReduce &f0, int tiles, cudaStream_t st) {
  FusedReduce f = f0;
  f.flag_off = 0;  // the group's flags start at the window base
  fused_wait_kernel<<<(tiles + 255) / 256, 256, 0, st>>>(f, tiles);
  return cudaGetLastError();
}

}  // namespace jk
