// lora_dropout.cu -- LoRA dropout (Listing 3 LORA_DROPOUT = 0.05, PAPER.md:82;
// DESIGN.md reading R7: inverted dropout on the adapter input only; the
// frozen path W0 x never sees it).  With keep mask M and q = 1 / (1 - p):
//   h   = q (M . x) A^T                     (K0, replaces K1's in-MMA h)
//   dX  = G W0 + q M . (gh A)               (K2 dropout mode, lora_gemm.cu)
//   dA  = q gh^T (M . x)                    (K3 on xm = M . x)
// K0 here: streams x once (16-byte loads), draws the keep bits from Philox
// (lora_philox.cuh) and writes any of: h in fp32, xm = M . x in bf16 (exact:
// zeroing only) and the packed keep bits the dX epilogue reads.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>

#include "lora_kernels.h"
#include "lora_philox.cuh"

namespace lora_sm100 {

typedef __nv_bfloat16 bf16;

namespace {

__device__ __forceinline__ void unpack8(const uint4& u, float (&f)[8]) {
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const float2 t = __bfloat1622float2(h[i]);
        f[2 * i] = t.x;
        f[2 * i + 1] = t.y;
    }
}

// RB: register rank bucket (>= r).  A block of 8 warps covers 8 / SPLIT token
// rows; the SPLIT warps of a row take contiguous column ranges (more warps in
// flight than one-warp-per-row at small T), and their partial h sums are
// combined in warp order through shared memory (deterministic).  Each lane
// handles 8 consecutive columns per step: one 16-byte load of x, one Philox
// block for the 8 keep bits.  Outputs (any may be null):
//   h [T, r] = q (M . x) A^T     xm [T, n] = M . x (bf16, exact)
//   bits [T, ceil(n/32)] uint32: bit c of word w = keep(t, 32 w + c)
template <int RB, int SPLIT>
__global__ void __launch_bounds__(256) dropout_input_kernel(const bf16* __restrict__ x, int64_t T, int64_t n,
                                                            const bf16* __restrict__ a, int r, DropoutParams d,
                                                            float* __restrict__ h, bf16* __restrict__ xm,
                                                            uint32_t* __restrict__ bits) {
    __shared__ float part[8][RB];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t t = static_cast<int64_t>(blockIdx.x) * (8 / SPLIT) + warp / SPLIT;
    const int sub = warp % SPLIT;
    const int64_t chunk = ((n + SPLIT * 256 - 1) / (SPLIT * 256)) * 256;   // columns per warp, multiple of 256
    const int64_t k_lo = sub * chunk, k_hi = k_lo + chunk < n ? k_lo + chunk : n;
    const int64_t nw = (n + 31) / 32;
    float acc[RB];
#pragma unroll
    for (int j = 0; j < RB; ++j) acc[j] = 0.0f;
    if (t < T) {
        const bf16* xr = x + t * n;
        for (int64_t k0 = k_lo; k0 < k_hi; k0 += 256) {
            const int64_t k = k0 + lane * 8;
            const bool ok = k < k_hi;
            uint4 u = make_uint4(0, 0, 0, 0);
            uint32_t keep = 0;
            if (ok) {
                u = __ldg(reinterpret_cast<const uint4*>(xr + k));
                keep = dropout_keep8(d, t, k / 8);   // (k % 8 == 0: one Philox block)
            }
            if (bits) {
                // 4 lanes = 32 consecutive columns = one mask word
                uint32_t w = keep << (8 * (lane & 3));
                w |= __shfl_xor_sync(0xffffffffu, w, 1);
                w |= __shfl_xor_sync(0xffffffffu, w, 2);
                if ((lane & 3) == 0 && k < k_hi) bits[t * nw + k / 32] = w;
            }
            if (!ok) continue;
            if (xm) {
                const uint32_t wv[4] = {u.x, u.y, u.z, u.w};
                uint32_t o[4];
#pragma unroll
                for (int i = 0; i < 4; ++i)
                    o[i] = (wv[i] & ((keep >> (2 * i)) & 1u ? 0x0000FFFFu : 0u)) |
                           (wv[i] & ((keep >> (2 * i + 1)) & 1u ? 0xFFFF0000u : 0u));
                *reinterpret_cast<uint4*>(xm + t * n + k) = make_uint4(o[0], o[1], o[2], o[3]);
            }
            if (h) {
                float xv[8];
                unpack8(u, xv);
#pragma unroll
                for (int c = 0; c < 8; ++c) xv[c] = (keep >> c) & 1u ? xv[c] : 0.0f;
#pragma unroll
                for (int j = 0; j < RB; ++j) {
                    if (j < r) {
                        float av[8];
                        unpack8(__ldg(reinterpret_cast<const uint4*>(a + static_cast<int64_t>(j) * n + k)), av);
#pragma unroll
                        for (int c = 0; c < 8; ++c) acc[j] = fmaf(xv[c], av[c], acc[j]);
                    }
                }
            }
        }
    }
    if (!h) return;
#pragma unroll
    for (int j = 0; j < RB; ++j)
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc[j] += __shfl_xor_sync(0xffffffffu, acc[j], o);
    if (lane == 0) {
#pragma unroll
        for (int j = 0; j < RB; ++j) part[warp][j] = acc[j];
    }
    __syncthreads();
    if (sub == 0 && lane == 0 && t < T) {
#pragma unroll
        for (int j = 0; j < RB; ++j) {
            if (j < r) {
                float v = part[warp][j];
                for (int q = 1; q < SPLIT; ++q) v += part[warp + q][j];
                h[t * r + j] = d.q * v;
            }
        }
    }
}

__global__ void dropout_mask_kernel(int64_t T, int64_t n, DropoutParams d, uint8_t* __restrict__ mask) {
    const int64_t n8 = (n + 7) / 8;
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < T * n8; i += stride) {
        const int64_t t = i / n8, k8 = i - t * n8;
        const uint32_t keep = dropout_keep8(d, t, k8);
#pragma unroll
        for (int c = 0; c < 8; ++c)
            if (k8 * 8 + c < n) mask[t * n + k8 * 8 + c] = (keep >> c) & 1u;
    }
}

}  // namespace

template <int RB>
static void launch_input_rb(const bf16* x, int64_t T, int64_t n, const bf16* a, int r, const DropoutParams& d,
                            float* h, bf16* xm, uint32_t* bits, int num_sms, cudaStream_t stream) {
    // SPLIT warps per row: pick the split whose grid fills its last wave best (at
    // cfg2, T = 2048: SPLIT 2 gave 512 CTAs = 1.15 waves of 3 CTAs / SM and ran
    // at ~50% of its issue rate; SPLIT 8 gives 2048 CTAs = 4.6 waves)
    static int per_sm[3] = {0, 0, 0};
    if (!per_sm[0]) {
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm[0], dropout_input_kernel<RB, 1>, 256, 0);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm[1], dropout_input_kernel<RB, 2>, 256, 0);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm[2], dropout_input_kernel<RB, 8>, 256, 0);
        for (int i = 0; i < 3; ++i) per_sm[i] = per_sm[i] > 0 ? per_sm[i] : 1;
    }
    const int splits[3] = {1, 2, 8};
    int best = 0;
    double best_eff = -1.0;
    for (int i = 0; i < 3; ++i) {
        if (splits[i] > 1 && n <= 256 * (splits[i] / 2)) continue;   // a warp needs >= one 256-column step
        const double blocks = static_cast<double>((T + 8 / splits[i] - 1) / (8 / splits[i]));
        const double waves = blocks / (static_cast<double>(num_sms) * per_sm[i]);
        const double eff = waves / std::ceil(waves);
        if (eff > best_eff + 0.02) { best_eff = eff; best = i; }
    }
    if (best == 0) {
        dropout_input_kernel<RB, 1><<<static_cast<unsigned>((T + 7) / 8), 256, 0, stream>>>(x, T, n, a, r, d, h, xm,
                                                                                          bits);
    } else if (best == 1) {
        dropout_input_kernel<RB, 2><<<static_cast<unsigned>((T + 3) / 4), 256, 0, stream>>>(x, T, n, a, r, d, h, xm,
                                                                                          bits);
    } else {
        dropout_input_kernel<RB, 8><<<static_cast<unsigned>(T), 256, 0, stream>>>(x, T, n, a, r, d, h, xm, bits);
    }
}

cudaError_t launch_dropout_input(const bf16* x, int64_t T, int64_t n, const bf16* a, int r, const DropoutParams& d,
                                 float* h, bf16* xm, uint32_t* bits, int num_sms, cudaStream_t stream) {
    if (T <= 0 || (!h && !xm && !bits)) return cudaSuccess;
    if (r <= 4) launch_input_rb<4>(x, T, n, a, r, d, h, xm, bits, num_sms, stream);
    else if (r <= 8) launch_input_rb<8>(x, T, n, a, r, d, h, xm, bits, num_sms, stream);
    else if (r <= 16) launch_input_rb<16>(x, T, n, a, r, d, h, xm, bits, num_sms, stream);
    else if (r <= 32) launch_input_rb<32>(x, T, n, a, r, d, h, xm, bits, num_sms, stream);
    else launch_input_rb<64>(x, T, n, a, r, d, h, xm, bits, num_sms, stream);
    return cudaGetLastError();
}

// the members of a group one launch each (a grouped kernel indexing the members
// dynamically measured 1.5x slower per member, dropout path)
cudaError_t launch_dropout_input_group(const DropoutGroup& G, int num_sms, cudaStream_t stream) {
    for (int g = 0; g < G.count; ++g) {
        const DropoutMember& M = G.m[g];
        cudaError_t e = launch_dropout_input(G.x, G.T, G.n, M.a, M.r, M.drop, M.h, M.xm, M.bits, num_sms, stream);
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

cudaError_t launch_dropout_mask(int64_t T, int64_t n, const DropoutParams& d, uint8_t* mask, int num_sms,
                                cudaStream_t stream) {
    if (T <= 0) return cudaSuccess;
    dropout_mask_kernel<<<num_sms * 4, 256, 0, stream>>>(T, n, d, mask);
    return cudaGetLastError();
}

}  // namespace lora_sm100
