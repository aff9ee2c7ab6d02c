// lora_philox.cuh -- LoRA-dropout keep mask on the device (Listing 3
// LORA_DROPOUT; reading R7).
//
// Counter-based, so the backward regenerates the forward's mask instead of
// storing it:  for element (t, k) of a [T, n] adapter input,
//   (w0, w1, w2, w3) = Philox4x32-10(counter = (k / 4, t, offset_lo, offset_hi),
//                                    key     = (seed_lo, seed_hi))
//   keep(t, k)       = w_{k mod 4} >= thr,   thr = floor(p * 2^32).
// One Philox block gives the keep bits of 4 consecutive columns.
#pragma once
#include <cstdint>

#include "lora_kernels.h"   // DropoutParams

namespace lora_sm100 {

__device__ __forceinline__ void philox4x32_10(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3, uint32_t k0,
                                              uint32_t k1, uint32_t (&out)[4]) {
#pragma unroll
    for (int round = 0; round < 10; ++round) {
        if (round > 0) {
            k0 += 0x9E3779B9u;
            k1 += 0xBB67AE85u;
        }
        const uint32_t lo0 = 0xD2511F53u * c0, hi0 = __umulhi(0xD2511F53u, c0);
        const uint32_t lo1 = 0xCD9E8D57u * c2, hi1 = __umulhi(0xCD9E8D57u, c2);
        const uint32_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
        c0 = n0;
        c1 = lo1;
        c2 = n2;
        c3 = lo0;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

// keep bits of columns 4*k4 .. 4*k4+3 of row t (bit i = column 4*k4 + i)
__device__ __forceinline__ uint32_t dropout_keep4(const DropoutParams& d, int64_t t, int64_t k4) {
    uint32_t w[4];
    philox4x32_10(static_cast<uint32_t>(k4), static_cast<uint32_t>(t), static_cast<uint32_t>(d.offset),
                  static_cast<uint32_t>(d.offset >> 32), static_cast<uint32_t>(d.seed),
                  static_cast<uint32_t>(d.seed >> 32), w);
    return (w[0] >= d.thr ? 1u : 0u) | (w[1] >= d.thr ? 2u : 0u) | (w[2] >= d.thr ? 4u : 0u) |
           (w[3] >= d.thr ? 8u : 0u);
}

}  // namespace lora_sm100
