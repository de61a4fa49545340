// numpy's Philox4x64-10 bit generator (Random123), counter-based: draw #i of
// np.random.Generator(np.random.Philox(key=[seed, counter])).random() is
// (word (i mod 4) of block (i / 4 + 1)) >> 11, times 2^-53.  Shared by the
// stochastic-rounding kernels (hlq_stochastic.cu, hlq_baselines.cu).
#pragma once
#include <cstdint>

namespace hlq {
namespace dev {

constexpr uint64_t kPhM0 = 0xD2E7470EE14C6C93ull, kPhM1 = 0xCA5A826395121157ull;
constexpr uint64_t kPhW0 = 0x9E3779B97F4A7C15ull, kPhW1 = 0xBB67AE8584CAA73Bull;

__device__ __forceinline__ void philox4x64_10(uint64_t (&c)[4], uint64_t k0, uint64_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r) { k0 += kPhW0; k1 += kPhW1; }
    const uint64_t hi0 = __umul64hi(kPhM0, c[0]), lo0 = kPhM0 * c[0];
    const uint64_t hi1 = __umul64hi(kPhM1, c[2]), lo1 = kPhM1 * c[2];
    const uint64_t n0 = hi1 ^ c[1] ^ k0, n2 = hi0 ^ c[3] ^ k1;
    c[0] = n0; c[1] = lo1; c[2] = n2; c[3] = lo0;
  }
}

// draws idx0 .. idx0+3 (idx0 % 4 == 0): one Philox block
__device__ __forceinline__ void philox_u01_x4(uint64_t k0, uint64_t k1, uint64_t idx0, double (&u)[4]) {
  uint64_t c[4] = {(idx0 >> 2) + 1, 0, 0, 0};
  philox4x64_10(c, k0, k1);
#pragma unroll
  for (int i = 0; i < 4; ++i) u[i] = double(c[i] >> 11) * 0x1p-53;
}
__device__ __forceinline__ double philox_u01(uint64_t k0, uint64_t k1, uint64_t idx) {
  uint64_t c[4] = {(idx >> 2) + 1, 0, 0, 0};
  philox4x64_10(c, k0, k1);
  const uint64_t x = (idx & 3) == 0 ? c[0] : (idx & 3) == 1 ? c[1] : (idx & 3) == 2 ? c[2] : c[3];
  return double(x >> 11) * 0x1p-53;
}

}  // namespace dev
}  // namespace hlq
