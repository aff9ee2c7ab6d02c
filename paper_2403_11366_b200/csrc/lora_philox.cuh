// lora_philox.cuh -- LoRA-dropout keep mask on the device (Listing 3
// LORA_DROPOUT; reading R7).
//
// Counter-based, so the backward can regenerate the forward's mask instead of
// storing it:  for element (t, k) of a [T, n] adapter input,
//   (w0, w1, w2, w3) = Philox4x32-10(counter = (k / 8, t, offset_lo, offset_hi),
//                                    key     = (seed_lo, seed_hi))
//   u(t, k)          = (w_{(k mod 8) / 2} >> 16 (k mod 2)) & 0xFFFF
//   keep(t, k)       = u(t, k) >= thr,   thr = floor(p * 2^16).
// One Philox block gives the keep bits of 8 consecutive columns (R7).
// Also here: the K0 helpers shared with the forward/backward dropout kernels
// (masking of a 16-byte group of x, keep-bit packing, mma.sync m16n8k16).
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

// keep bits of columns 8*k8 .. 8*k8+7 of row t (bit i = column 8*k8 + i): one
// Philox block gives eight 16-bit draws, draw i = half (i % 2) of word i / 2
__device__ __forceinline__ uint32_t dropout_keep8(const DropoutParams& d, int64_t t, int64_t k8) {
    uint32_t w[4];
    philox4x32_10(static_cast<uint32_t>(k8 + d.col0 / 8), static_cast<uint32_t>(t + d.row0), static_cast<uint32_t>(d.offset),
                  static_cast<uint32_t>(d.offset >> 32), static_cast<uint32_t>(d.seed),
                  static_cast<uint32_t>(d.seed >> 32), w);
    uint32_t keep = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) keep |= (((w[i >> 1] >> (16 * (i & 1))) & 0xFFFFu) >= d.thr ? 1u : 0u) << i;
    return keep;
}

// The same generator with the round keys and offset words prepared on the host
// (PhiloxKeys): w = Philox4x32-10(counter (c0, c1, K.c2, K.c3), key (seed)).
__device__ __forceinline__ void philox4x32_10_keys(uint32_t c0, uint32_t c1, const PhiloxKeys& K,
                                                   uint32_t (&out)[4]) {
    uint32_t c2 = K.c2, c3 = K.c3;
#pragma unroll
    for (int round = 0; round < 10; ++round) {
        const uint32_t lo0 = 0xD2511F53u * c0, hi0 = __umulhi(0xD2511F53u, c0);
        const uint32_t lo1 = 0xCD9E8D57u * c2, hi1 = __umulhi(0xCD9E8D57u, c2);
        const uint32_t n0 = hi1 ^ c1 ^ K.k0[round], n2 = hi0 ^ c3 ^ K.k1[round];
        c0 = n0;
        c1 = lo1;
        c2 = n2;
        c3 = lo0;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

// Keep masks of the two 16-bit draws of one Philox word: 0xFFFF in each half
// whose draw u satisfies u >= thr (thr2 = thr in both halves).  SWAR unsigned
// compare without a borrow between the halves: t's top bit per half = (u & 0x7FFF)
// >= (thr & 0x7FFF); u >= thr = (u_H & ~thr_H) | (~(u_H ^ thr_H) & t_H); prmt then
// replicates each half's top bit over the half.
__device__ __forceinline__ uint32_t keep_mask_word(uint32_t w, uint32_t thr2) {
    const uint32_t t = (w | 0x80008000u) - (thr2 & 0x7FFF7FFFu);
    const uint32_t ge = (w & ~thr2) | (~(w ^ thr2) & t);
    uint32_t m;
    asm("prmt.b32 %0, %1, 0, 0xBB99;" : "=r"(m) : "r"(ge));
    return m;
}

// x word i (elements 8 k8 + 2i, 2i + 1 of a row) masked by member M's draws:
// one Philox block (counter (k8, t)) gives the 16-bit draws of the 8 elements.
__device__ __forceinline__ uint4 masked8(const uint4& u, const PhiloxKeys& K, uint32_t k8, uint32_t t,
                                         uint32_t (&w)[4]) {
    philox4x32_10_keys(k8 + K.k8_base, t + K.t_base, K, w);
#pragma unroll
    for (int i = 0; i < 4; ++i) w[i] = keep_mask_word(w[i], K.thr2);
    return make_uint4(u.x & w[0], u.y & w[1], u.z & w[2], u.w & w[3]);
}

// keep bits of the 8 elements (bit e = element e) from the 4 mask words, and back
__device__ __forceinline__ uint32_t keep8_of(const uint32_t (&w)[4]) {
    uint32_t keep = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) keep |= ((w[i] >> 15) & 1u) << (2 * i) | ((w[i] >> 31) << (2 * i + 1));
    return keep;
}
__device__ __forceinline__ uint4 masked8_bits(const uint4& u, uint32_t keep) {
    uint32_t m[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) m[i] = ((keep >> (2 * i)) & 1u) * 0x0000FFFFu | ((keep >> (2 * i + 1)) & 1u) * 0xFFFF0000u;
    return make_uint4(u.x & m[0], u.y & m[1], u.z & m[2], u.w & m[3]);
}

__device__ __forceinline__ void mma_bf16_16816(float (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                               uint32_t b0, uint32_t b1) {
    asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
                 "{%0,%1,%2,%3};"
                 : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
                 : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

}  // namespace lora_sm100
