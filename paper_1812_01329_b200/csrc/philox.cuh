// philox.cuh — Philox4x32-10 (Salmon, Moraes, Dror, Shaw, SC'11) on the device: the counter-based
// generator of the dropout masks (reading R14: element (r, j) of dropout site s keeps iff word
// j mod 4 of Philox(counter = (j / 4, r, s, 0), key) >= floor(p * 2^32)). Stateless: any thread
// regenerates any mask word, so the forward and the backward draw the same mask without storing it.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace jk {

__device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint2 k) {
  constexpr uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u, W0 = 0x9E3779B9u, W1 = 0xBB67AE85u;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r) { k.x += W0; k.y += W1; }
    const uint32_t hi0 = __umulhi(M0, c.x), lo0 = M0 * c.x;
    const uint32_t hi1 = __umulhi(M1, c.z), lo1 = M1 * c.z;
    c = make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
  }
  return c;
}

// keep flags of columns 4 q .. 4 q + 3 of global row r at dropout site s
__device__ __forceinline__ uint4 dropout_words(uint2 key, int site, int r, int q) {
  return philox4x32_10(make_uint4((uint32_t)q, (uint32_t)r, (uint32_t)site, 0u), key);
}

}  // namespace jk
