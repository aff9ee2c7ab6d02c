// lora_grad.cu -- K3, the two trainable gradients of the LoRA linear
// ("B and A are the trainable weights"):
//     dA[j, k] = sum_t gh[t, j] x[t, k]          gh = s dY B   (from K2)
//     dB[i, j] = s sum_t dY[t, i] h[t, j]        h  = x A^T    (from K1)
// Both are rank-r reductions over all T tokens: 2 T r (n + m) FLOPs reading
// the T x (n + m) bf16 activations once, so they are HBM/FMA-bound and run on
// the CUDA cores.  One CTA owns a 32-column strip of dA (columns of x) or of
// dB (columns of dY) for ALL tokens and writes the final values itself: no
// token split, no partial-sum buffer, no second pass, and a fixed summation
// order (deterministic).  x / dY are read with 16-byte coalesced loads
// (4 lanes x 16 B = one 64 B row segment, 8 rows per warp instruction); the
// fp32 coefficient rows (gh or h) are staged through shared memory.
// Also B6, the adapter pack used only when r % 8 != 0.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "lora_kernels.h"

namespace lora_sm100 {

typedef __nv_bfloat16 bf16;

// ------------------------------------------------------------------ B6
// b8[i, j] = j < r ? B[i, j] : 0, [m, r8], r8 = roundup(r, 8): the 16-byte row
//   pitch TMA needs (forward tail operand, only when r % 8 != 0);
// bt[j, i] = B[i, j], [r, m]: K-major operand of the dX kernel's dY B MMA.
__global__ void pack_b_kernel(const bf16* __restrict__ b, int64_t m, int r, int r8, bf16* __restrict__ b8,
                              bf16* __restrict__ bt) {
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    const int64_t t0 = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const bf16 zero = __float2bfloat16(0.0f);
    if (b8)
        for (int64_t idx = t0; idx < m * r8; idx += stride) {
            const int64_t i = idx / r8;
            const int j = static_cast<int>(idx - i * r8);
            b8[idx] = j < r ? b[i * r + j] : zero;
        }
    if (bt)
        for (int64_t idx = t0; idx < static_cast<int64_t>(r) * m; idx += stride) {
            const int64_t j = idx / m, i = idx - j * m;
            bt[idx] = b[i * r + j];
        }
}

cudaError_t launch_pack_b(const bf16* b, int64_t m, int r, bf16* b8, bf16* bt, int num_sms, cudaStream_t stream) {
    const int r8 = (r + 7) / 8 * 8;
    const int64_t work = m * r8;
    const int blocks = static_cast<int>(std::min<int64_t>((work + 255) / 256, 4LL * num_sms));
    pack_b_kernel<<<blocks, 256, 0, stream>>>(b, m, r, r8, b8, bt);
    return cudaGetLastError();
}

// ------------------------------------------------------------------ K3
struct GradArgs {
    const bf16* x;     // [T, n]
    const float* gh;   // [T, r]   (dA coefficients, already scaled by s)
    const bf16* dy;    // [T, m]
    const float* h;    // [T, r]   (dB coefficients, unscaled)
    float* da;         // [r, n] or null
    float* db;         // [m, r] or null
    int64_t T, n, m;
    int r;
    int strips_a;      // CTAs [0, strips_a) own dA strips, the rest dB strips
    float scale_b;     // s
    int accumulate;
};

constexpr int kStrip = 32;        // columns per CTA
constexpr int kWarps = 8;

__device__ __forceinline__ void bf16x8_to_f32(const uint4& u, float (&f)[8]) {
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const float2 t = __bfloat1622float2(h[i]);
        f[2 * i] = t.x;
        f[2 * i + 1] = t.y;
    }
}

template <int CPT>
struct Vec;
template <>
struct Vec<8> {
    using T = uint4;
    __device__ static void cvt(const T& u, float (&f)[8]) { bf16x8_to_f32(u, f); }
};
template <>
struct Vec<4> {
    using T = uint2;
    __device__ static void cvt(const T& u, float (&f)[4]) {
        const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
        const float2 a = __bfloat1622float2(h[0]), b = __bfloat1622float2(h[1]);
        f[0] = a.x; f[1] = a.y; f[2] = b.x; f[3] = b.y;
    }
};
template <>
struct Vec<2> {
    using T = uint32_t;
    __device__ static void cvt(const T& u, float (&f)[2]) {
        const float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u));
        f[0] = a.x; f[1] = a.y;
    }
};

// RB: register rank bucket (>= r, multiple of 4); CPT: columns per lane.
template <int RB, int CPT, int MINB>
__global__ void __launch_bounds__(256, MINB) grad_strip_kernel(const GradArgs g) {
    constexpr int LPR = kStrip / CPT;            // lanes per row (4, 8, 16)
    constexpr int RPW = 32 / LPR;                // rows per warp instruction (8, 4, 2)
    constexpr int RPI = RPW * kWarps;            // rows per CTA iteration
    constexpr int CHUNK = 16384 / RB;            // staged coefficient rows (64 KiB)
    constexpr int U = 8;                         // loads in flight per lane
    using VT = typename Vec<CPT>::T;
    extern __shared__ float4 smem_f4[];
    float* s_coef = reinterpret_cast<float*>(smem_f4);   // [CHUNK][RB], later the reduction buffer

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int rs = lane / LPR, cc = lane % LPR;
    const bool is_a = static_cast<int>(blockIdx.x) < g.strips_a;
    const bf16* X = is_a ? g.x : g.dy;
    const float* coef = is_a ? g.gh : g.h;
    const int64_t ncols = is_a ? g.n : g.m;
    const int64_t cs = static_cast<int64_t>(is_a ? blockIdx.x : blockIdx.x - g.strips_a) * kStrip;
    const int64_t c0 = cs + cc * CPT;
    const bool col_ok = c0 < ncols;              // ncols % 8 == 0 and CPT | 8
    const int r = g.r;
    const int64_t T = g.T;

    float acc[CPT][RB];
#pragma unroll
    for (int c = 0; c < CPT; ++c)
#pragma unroll
        for (int j = 0; j < RB; ++j) acc[c][j] = 0.0f;

    for (int64_t tb = 0; tb < T; tb += CHUNK) {
        const int nrow = static_cast<int>((T - tb) < CHUNK ? (T - tb) : CHUNK);
        __syncthreads();
        if (r == RB) {
            // contiguous [nrow, r] fp32 block: 16-byte cp.async, all in flight at once
            const float* src = coef + tb * r;
            const int n16 = nrow * RB / 4;
            for (int q = threadIdx.x; q < n16; q += 256)
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;"
                             ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(s_coef + 4 * q))),
                               "l"(src + 4 * q) : "memory");
            asm volatile("cp.async.wait_all;" ::: "memory");
        } else {
            for (int idx = threadIdx.x; idx < nrow * RB; idx += 256) {
                const int rr = idx / RB, j = idx - rr * RB;
                s_coef[idx] = j < r ? coef[(tb + rr) * r + j] : 0.0f;
            }
        }
        __syncthreads();
        if (col_ok) {
            const bf16* xp = X + tb * ncols + c0;
            // row rr = it * RPI + warp * RPW + rs
            for (int base = warp * RPW + rs; base < nrow; base += U * RPI) {
                VT v[U];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int rr = base + u * RPI;
                    if (rr < nrow) v[u] = __ldg(reinterpret_cast<const VT*>(xp + static_cast<int64_t>(rr) * ncols));
                }
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int rr = base + u * RPI;
                    if (rr < nrow) {
                        float xv[CPT];
                        Vec<CPT>::cvt(v[u], xv);
                        const float4* cr = reinterpret_cast<const float4*>(s_coef + rr * RB);
#pragma unroll
                        for (int j4 = 0; j4 < RB / 4; ++j4) {
                            const float4 cj = cr[j4];
#pragma unroll
                            for (int c = 0; c < CPT; ++c) {
                                acc[c][4 * j4 + 0] = fmaf(xv[c], cj.x, acc[c][4 * j4 + 0]);
                                acc[c][4 * j4 + 1] = fmaf(xv[c], cj.y, acc[c][4 * j4 + 1]);
                                acc[c][4 * j4 + 2] = fmaf(xv[c], cj.z, acc[c][4 * j4 + 2]);
                                acc[c][4 * j4 + 3] = fmaf(xv[c], cj.w, acc[c][4 * j4 + 3]);
                            }
                        }
                    }
                }
            }
        }
    }

    // (1) within the warp: lanes with the same column chunk (xor over the row bits)
#pragma unroll
    for (int off = LPR; off < 32; off <<= 1)
#pragma unroll
        for (int c = 0; c < CPT; ++c)
#pragma unroll
            for (int j = 0; j < RB; ++j) acc[c][j] += __shfl_xor_sync(0xffffffffu, acc[c][j], off);
    // (2) across warps, in warp order: red[w][j][col]
    __syncthreads();
    float* red = s_coef;
    if (rs == 0) {
#pragma unroll
        for (int j = 0; j < RB; ++j)
#pragma unroll
            for (int c = 0; c < CPT; ++c) red[(warp * RB + j) * kStrip + cc * CPT + c] = acc[c][j];
    }
    __syncthreads();
    for (int o = threadIdx.x; o < RB * kStrip; o += 256) {
        const int j = o / kStrip, col = o - j * kStrip;
        if (j >= r || cs + col >= ncols) continue;
        float s = 0.0f;
#pragma unroll
        for (int w = 0; w < kWarps; ++w) s += red[(w * RB + j) * kStrip + col];
        if (is_a) {
            float* d = g.da + static_cast<int64_t>(j) * ncols + cs + col;
            *d = g.accumulate ? *d + s : s;
        } else {
            const float v = g.scale_b * s;
            float* d = g.db + (cs + col) * r + j;
            *d = g.accumulate ? *d + v : v;
        }
    }
}

template <int RB, int CPT, int MINB>
static cudaError_t launch_strip(int grid, const GradArgs& g, cudaStream_t stream) {
    const int smem = 16384 * static_cast<int>(sizeof(float));
    auto kern = grad_strip_kernel<RB, CPT, MINB>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    kern<<<grid, 256, smem, stream>>>(g);
    return cudaGetLastError();
}

cudaError_t launch_grad_reduce(int64_t T, int64_t n, int64_t m, int r, float scale, const bf16* x,
                               const float* gh, const bf16* dy, const float* h, float* da, float* db,
                               int accumulate, cudaStream_t stream, int* launches) {
    GradArgs g;
    g.x = x; g.gh = gh; g.dy = dy; g.h = h; g.da = da; g.db = db;
    g.T = T; g.n = n; g.m = m; g.r = r; g.scale_b = scale; g.accumulate = accumulate;
    const int sa = da ? static_cast<int>((n + kStrip - 1) / kStrip) : 0;
    const int sb = db ? static_cast<int>((m + kStrip - 1) / kStrip) : 0;
    g.strips_a = sa;
    if (sa + sb == 0) return cudaSuccess;
    cudaError_t e;
    if (r <= 4) e = launch_strip<4, 8, 2>(sa + sb, g, stream);
    else if (r <= 8) e = launch_strip<8, 8, 2>(sa + sb, g, stream);
    else if (r <= 16) e = launch_strip<16, 4, 2>(sa + sb, g, stream);
    else if (r <= 32) e = launch_strip<32, 2, 2>(sa + sb, g, stream);
    else e = launch_strip<64, 2, 1>(sa + sb, g, stream);
    if (e == cudaSuccess && launches) ++*launches;
    return e;
}

}  // namespace lora_sm100
