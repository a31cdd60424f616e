// Philox4x64-10 counter-based generator (Salmon et al., SC'11), device side.
// R24: key = (seed, round), counter = (global_row, stream, 0, 0);
// u = (first 64-bit output >> 11) * 2^-53 in [0, 1).  Streams: 0 sampling (Alg. 7),
// 1 sketch row sample (R2).  Keying by global row makes every draw independent of the
// page size and of the number of GPUs.
#pragma once
#include <stdint.h>

namespace oocgb {

__device__ __forceinline__ uint64_t philox4x64_10_first(uint64_t c0, uint64_t c1, uint64_t c2,
                                                        uint64_t c3, uint64_t k0, uint64_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint64_t M0 = 0xD2E7470EE14C6C93ull, M1 = 0xCA5A826395121157ull;
    uint64_t lo0 = M0 * c0, hi0 = __umul64hi(M0, c0);
    uint64_t lo1 = M1 * c2, hi1 = __umul64hi(M1, c2);
    uint64_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
    c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
    k0 += 0x9E3779B97F4A7C15ull;
    k1 += 0xBB67AE8584CAA73Bull;
  }
  return c0;
}

__device__ __forceinline__ double philox_uniform(uint64_t seed, uint64_t round, uint64_t row,
                                                 uint64_t stream) {
  uint64_t x = philox4x64_10_first(row, stream, 0, 0, seed, round);
  return (double)(x >> 11) * 0x1.0p-53;
}

}  // namespace oocgb
