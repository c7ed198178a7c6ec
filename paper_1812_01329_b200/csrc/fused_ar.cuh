// fused_ar.cuh — the per-tile protocol of the fused gradient reduction (NEXT-3, gemm_tc.h
// FusedReduce): run by the 128 epilogue threads of the weight-gradient GEMM right after a tile is
// written, and by the null-step participant kernel of a rank that runs no GEMM (host_dp.cpp).
// Peer memory is addressed through NCCL's device API (symmetric windows, load/store accessible
// over NVLink); ordering across GPUs uses system-scope release / acquire.
#pragma once
#include <nccl.h>
#include <nccl_device.h>

#include "common.cuh"
#include "gemm_tc.h"

namespace jk {

JN_DEV unsigned *fr_flag(const FusedReduce &f, int peer, int tile, int which) {
  return static_cast<unsigned *>(
      ncclGetLsaPointer(static_cast<ncclWindow_t>(f.fwin), f.flag_off + ((size_t)tile * 2 + which) * 4, peer));
}
JN_DEV float *fr_c(const FusedReduce &f, int peer) {
  return static_cast<float *>(ncclGetLsaPointer(static_cast<ncclWindow_t>(f.win), f.c_off, peer));
}
JN_DEV void fr_bar() { asm volatile("bar.sync 1, 128;" ::: "memory"); }

// Tile `tile` = rows [m0, m0 + 128) x columns [n0, n0 + bn) of an M x N matrix C (pitch ldc
// floats); this rank's tile is already written (its TMA stores completed). t = 0..127 is the
// calling thread's index among the 128 participants (row m0 + t).
JN_DEV void fr_tile(const FusedReduce &f, int tile, int m0, int n0, int bn, int M, int N, int ldc, int t) {
  const int owner = tile % f.nranks;
  fr_bar();  // every participant's stores of the tile precede the release below (cumulativity)
  if (t == 0) {  // publish: my tile is written
    asm volatile("fence.acq_rel.sys;" ::: "memory");
    asm volatile("red.release.sys.global.add.u32 [%0], 1;" ::"l"(fr_flag(f, owner, tile, 0)) : "memory");
  }
  if (owner != f.rank) return;  // uniform over the 128 threads
  if (f.nranks == 1 && !f.force_pull) {  // the sum of one rank's tile is the tile, already in place
    if (t == 0) asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(fr_flag(f, 0, tile, 1)), "r"(f.epoch) : "memory");
    return;
  }
  if (t == 0) {  // every rank's tile t has been published
    const unsigned need = f.epoch * (unsigned)f.nranks;
    const unsigned *rd = fr_flag(f, f.rank, tile, 0);
    unsigned v;
    do {
      asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(rd) : "memory");
    } while (v < need);
  }
  fr_bar();
  const int m = m0 + t;
  if (m < M) {
    const int n1 = min(N, n0 + bn);
    const size_t ro = (size_t)m * ldc;
    const bool v4 = (ldc & 3) == 0 && (n0 & 3) == 0;
    int c = n0;
    if (v4) {
      for (; c + 3 < n1; c += 4) {
        float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
        for (int p = 0; p < f.nranks; ++p) {  // rank order: the same sum on every rank
          const float4 x = __ldcv(reinterpret_cast<const float4 *>(fr_c(f, p) + ro + c));
          s.x += x.x; s.y += x.y; s.z += x.z; s.w += x.w;
        }
        for (int p = 0; p < f.nranks; ++p) *reinterpret_cast<float4 *>(fr_c(f, p) + ro + c) = s;
      }
    }
    for (; c < n1; ++c) {
      float s = 0.f;
      for (int p = 0; p < f.nranks; ++p) s += __ldcv(fr_c(f, p) + ro + c);
      for (int p = 0; p < f.nranks; ++p) fr_c(f, p)[ro + c] = s;
    }
  }
  fr_bar();  // every thread's pushes precede the releases (cumulativity through the barrier)
  if (t == 0) {
    asm volatile("fence.acq_rel.sys;" ::: "memory");
    for (int p = 0; p < f.nranks; ++p)
      asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(fr_flag(f, p, tile, 1)), "r"(f.epoch) : "memory");
  }
}

}  // namespace jk
