// Device-side counter-based Philox4x32-10 (Salmon et al., SC'11), the RNG the
// north star fixes for the epoch permutation ("a counter-based Philox stream
// specified once and implemented separately in both oracle and GPU code").
// Written independently of oracle/pp_oracle.c.  The oracle's Philox, unit-key
// layout and generator words are pinned against cuRAND's curand_Philox4x32_10 on
// device (tests/test_gpu_curand_pins.py); this implementation is compared with the
// oracle through every permutation and synthetic-fill parity test.
#pragma once
#include <cstdint>

namespace ppl {

// Philox multipliers and Weyl key increments (published constants).
constexpr uint32_t kPhiloxM0 = 0xD2511F53u;
constexpr uint32_t kPhiloxM1 = 0xCD9E8D57u;
constexpr uint32_t kPhiloxW0 = 0x9E3779B9u;
constexpr uint32_t kPhiloxW1 = 0xBB67AE85u;

__device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint2 k) {
#pragma unroll
  for (int i = 0; i < 10; ++i) {
    const uint32_t hi0 = __umulhi(kPhiloxM0, c.x);
    const uint32_t lo0 = kPhiloxM0 * c.x;
    const uint32_t hi1 = __umulhi(kPhiloxM1, c.z);
    const uint32_t lo1 = kPhiloxM1 * c.z;
    c = make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
    k.x += kPhiloxW0;  // the bump after the 10th round is never used
    k.y += kPhiloxW1;
  }
  return c;
}

// Sort key of shuffle unit u (row for SGD-RR, chunk for chunk reshuffling):
// ctr = (u_lo, u_hi, 0, 0), key = (seed_lo, seed_hi), key64 = (y0 << 32) | y1.
__device__ __forceinline__ uint64_t unit_sort_key(uint64_t seed, uint64_t u) {
  const uint4 y = philox4x32_10(make_uint4(static_cast<uint32_t>(u), static_cast<uint32_t>(u >> 32), 0u, 0u),
                                make_uint2(static_cast<uint32_t>(seed), static_cast<uint32_t>(seed >> 32)));
  return (static_cast<uint64_t>(y.x) << 32) | y.y;
}

// Synthetic-feature word: word (f & 3) of
// Philox(ctr = (v_lo, v_hi, (k << 16) | (f >> 2), 'PPGF'), key = data_seed).
__device__ __forceinline__ uint4 synth_block(uint64_t data_seed, uint64_t v, uint32_t k, uint32_t f4) {
  return philox4x32_10(make_uint4(static_cast<uint32_t>(v), static_cast<uint32_t>(v >> 32), (k << 16) | f4, 0x50504746u),
                       make_uint2(static_cast<uint32_t>(data_seed), static_cast<uint32_t>(data_seed >> 32)));
}

}  // namespace ppl
