// philox.cuh -- Philox-4x32-10 (Salmon, Moraes, Dror, Shaw, SC'11), device side.
//
// Counter-based: the draw for (pulse, subray, voxel) is a pure function of
// its counter, so transmission decisions (Eq. 6) are
// reproducible at any thread count, batch split or launch shape -- the
// property the paper could only get single-threaded.
// Key = (seed_lo, seed_hi), counter = (pulse_lo, pulse_hi, subray, voxel id);
// u = (x0 >> 8) * 2^-24 (R18, R19).
#pragma once
#include <stdint.h>

namespace helios {

__device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint2 k) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t hi0 = __umulhi(0xD2511F53u, c.x), lo0 = 0xD2511F53u * c.x;
    const uint32_t hi1 = __umulhi(0xCD9E8D57u, c.z), lo1 = 0xCD9E8D57u * c.z;
    c = make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
    k.x += 0x9E3779B9u;
    k.y += 0xBB67AE85u;
  }
  return c;
}

__device__ __forceinline__ double transmission_u(uint64_t seed, uint64_t pulse, uint32_t subray,
                                                 uint32_t voxel) {
  uint4 x = philox4x32_10(make_uint4((uint32_t)pulse, (uint32_t)(pulse >> 32), subray, voxel),
                          make_uint2((uint32_t)seed, (uint32_t)(seed >> 32)));
  return (double)(x.x >> 8) * (1.0 / 16777216.0);
}

// Ranging error (R29): standard normal for return number j (1-based)
// of pulse p.  Key = (seed_lo, seed_hi ^ 1) -- stream tag 1, disjoint from the
// transmission stream -- counter (p_lo, p_hi, j, 0); Box-Muller on
// u1 = ((x0 >> 8) + 1) 2^-24 in (0, 1] and u2 = (x1 >> 8) 2^-24.
__device__ __forceinline__ double range_noise(uint64_t seed, uint64_t pulse, uint32_t j) {
  const uint4 x = philox4x32_10(make_uint4((uint32_t)pulse, (uint32_t)(pulse >> 32), j, 0u),
                                make_uint2((uint32_t)seed, (uint32_t)(seed >> 32) ^ 1u));
  const double u1 = (double)((x.x >> 8) + 1u) * (1.0 / 16777216.0);
  const double u2 = (double)(x.y >> 8) * (1.0 / 16777216.0);
  return sqrt(-2.0 * log(u1)) * cos(2.0 * 3.14159265358979323846 * u2);
}

}  // namespace helios
