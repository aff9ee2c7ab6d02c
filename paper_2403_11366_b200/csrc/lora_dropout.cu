// lora_dropout.cu -- LoRA dropout (Listing 3 LORA_DROPOUT = 0.05, PAPER.md:82;
// DESIGN.md reading R9: inverted dropout on the adapter input only; the
// frozen path W0 x never sees it).  With keep mask M and q = 1 / (1 - p):
//   h   = q (M . x) A^T                     (K0, replaces K1's in-MMA h)
//   dX  = G W0 + q M . (gh A)               (K2 dropout mode, lora_gemm.cu)
//   dA  = q gh^T (M . x)                    (K3 on xm = M . x)
// K0 here: one warp per token row, 16-byte loads of x, the row's keep bits
// from Philox (lora_philox.cuh), h in fp32 and/or xm = M . x in bf16 (exact:
// zeroing only), streaming x once.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

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

// RB: register rank bucket (>= r)
template <int RB>
__global__ void __launch_bounds__(256) dropout_input_kernel(const bf16* __restrict__ x, int64_t T, int64_t n,
                                                            const bf16* __restrict__ a, int r, DropoutParams d,
                                                            float* __restrict__ h, bf16* __restrict__ xm) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t t = static_cast<int64_t>(blockIdx.x) * 8 + warp;
    if (t >= T) return;
    float acc[RB];
#pragma unroll
    for (int j = 0; j < RB; ++j) acc[j] = 0.0f;
    const bf16* xr = x + t * n;
    for (int64_t k = lane * 8; k < n; k += 256) {
        const uint4 u = __ldg(reinterpret_cast<const uint4*>(xr + k));
        const uint32_t keep = dropout_keep4(d, t, k / 4) | (dropout_keep4(d, t, k / 4 + 1) << 4);
        if (xm) {
            const uint32_t w[4] = {u.x, u.y, u.z, u.w};
            uint32_t o[4];
#pragma unroll
            for (int i = 0; i < 4; ++i)
                o[i] = (w[i] & ((keep >> (2 * i)) & 1u ? 0x0000FFFFu : 0u)) |
                       (w[i] & ((keep >> (2 * i + 1)) & 1u ? 0xFFFF0000u : 0u));
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
    if (!h) return;
#pragma unroll
    for (int j = 0; j < RB; ++j)
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc[j] += __shfl_xor_sync(0xffffffffu, acc[j], o);
    if (lane == 0) {
#pragma unroll
        for (int j = 0; j < RB; ++j)
            if (j < r) h[t * r + j] = d.q * acc[j];
    }
}

__global__ void dropout_mask_kernel(int64_t T, int64_t n, DropoutParams d, uint8_t* __restrict__ mask) {
    const int64_t n4 = (n + 3) / 4;
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < T * n4; i += stride) {
        const int64_t t = i / n4, k4 = i - t * n4;
        const uint32_t keep = dropout_keep4(d, t, k4);
#pragma unroll
        for (int c = 0; c < 4; ++c)
            if (k4 * 4 + c < n) mask[t * n + k4 * 4 + c] = (keep >> c) & 1u;
    }
}

}  // namespace

cudaError_t launch_dropout_input(const bf16* x, int64_t T, int64_t n, const bf16* a, int r, const DropoutParams& d,
                                 float* h, bf16* xm, cudaStream_t stream) {
    if (T <= 0 || (!h && !xm)) return cudaSuccess;
    const dim3 grid(static_cast<unsigned>((T + 7) / 8));
    if (r <= 4) dropout_input_kernel<4><<<grid, 256, 0, stream>>>(x, T, n, a, r, d, h, xm);
    else if (r <= 8) dropout_input_kernel<8><<<grid, 256, 0, stream>>>(x, T, n, a, r, d, h, xm);
    else if (r <= 16) dropout_input_kernel<16><<<grid, 256, 0, stream>>>(x, T, n, a, r, d, h, xm);
    else if (r <= 32) dropout_input_kernel<32><<<grid, 256, 0, stream>>>(x, T, n, a, r, d, h, xm);
    else dropout_input_kernel<64><<<grid, 256, 0, stream>>>(x, T, n, a, r, d, h, xm);
    return cudaGetLastError();
}

cudaError_t launch_dropout_mask(int64_t T, int64_t n, const DropoutParams& d, uint8_t* mask, int num_sms,
                                cudaStream_t stream) {
    if (T <= 0) return cudaSuccess;
    dropout_mask_kernel<<<num_sms * 4, 256, 0, stream>>>(T, n, d, mask);
    return cudaGetLastError();
}

}  // namespace lora_sm100
