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
#include <cooperative_groups.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "lora_kernels.h"
#include "sm100_ptx.cuh"

namespace lora_sm100 {

typedef __nv_bfloat16 bf16;

__device__ __forceinline__ void bf16x8_to_f32(const uint4& u, float (&f)[8]) {
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const float2 t = __bfloat1622float2(h[i]);
        f[2 * i] = t.x;
        f[2 * i + 1] = t.y;
    }
}

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

// ------------------------------------------------------------------ K2a
// gh[t, j] = s * sum_i dY[t, i] B[i, j]  (A5's "dY B" term).
// One warp per token row; lanes stride the row with 16-byte dY loads; B rows
// (r bf16 each, L1/L2-resident: B is m x r) are read as 16-byte vectors when
// r % 8 == 0.  Fixed per-lane order + xor-shuffle tree: deterministic.
template <int RB>
__global__ void __launch_bounds__(256) gh_kernel(const bf16* __restrict__ dy, const bf16* __restrict__ b,
                                                 int64_t T, int64_t m, int r, float s, float* __restrict__ gh) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t row = static_cast<int64_t>(blockIdx.x) * 8 + warp;
    if (row >= T) return;
    float acc[RB];
#pragma unroll
    for (int j = 0; j < RB; ++j) acc[j] = 0.0f;
    const bf16* dr = dy + row * m;
    const bool vec = (r % 8) == 0;
    for (int64_t k = lane * 8; k < m; k += 256) {
        float dv[8];
        bf16x8_to_f32(__ldg(reinterpret_cast<const uint4*>(dr + k)), dv);
#pragma unroll
        for (int c = 0; c < 8; ++c) {
            const bf16* br = b + (k + c) * r;
            if (vec) {
#pragma unroll
                for (int j8 = 0; j8 < (RB + 7) / 8; ++j8) {
                    if (8 * j8 < r) {
                        float bv[8];
                        bf16x8_to_f32(__ldg(reinterpret_cast<const uint4*>(br + 8 * j8)), bv);
#pragma unroll
                        for (int e = 0; e < 8; ++e)
                            if (8 * j8 + e < RB) acc[8 * j8 + e] = fmaf(dv[c], bv[e], acc[8 * j8 + e]);
                    }
                }
            } else {
#pragma unroll
                for (int j = 0; j < RB; ++j)
                    if (j < r) acc[j] = fmaf(dv[c], __bfloat162float(br[j]), acc[j]);
            }
        }
    }
#pragma unroll
    for (int j = 0; j < RB; ++j)
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc[j] += __shfl_xor_sync(0xffffffffu, acc[j], o);
    if (lane == 0) {
#pragma unroll
        for (int j = 0; j < RB; ++j)
            if (j < r) gh[row * r + j] = s * acc[j];
    }
}

// v2: one warp per token row, 8 rows per CTA; B is staged chunk by chunk in
// shared memory TRANSPOSED to fp32 Bt[j][i] (conflict-free 32-byte reads per
// lane), and each lane keeps all 16-byte dY loads of a chunk in flight at once.
template <int RB>
__global__ void __launch_bounds__(256) gh_kernel_v2(const bf16* __restrict__ dy, const bf16* __restrict__ b,
                                                    int64_t T, int64_t m, int r, float s, float* __restrict__ gh) {
    constexpr int C = 16384 / RB;               // staged B rows (columns of dY) per chunk
    constexpr int G = C / 256;                  // 8-column groups per lane per chunk
    extern __shared__ float4 smem_gh[];
    float* bt = reinterpret_cast<float*>(smem_gh);   // [RB][C]
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t row = static_cast<int64_t>(blockIdx.x) * 8 + warp;
    const bool row_ok = row < T;
    float acc[RB];
#pragma unroll
    for (int j = 0; j < RB; ++j) acc[j] = 0.0f;
    const bf16* dr = dy + (row_ok ? row : 0) * m;
    for (int64_t i0 = 0; i0 < m; i0 += C) {
        const int ci = static_cast<int>((m - i0) < C ? (m - i0) : C);   // multiple of 8
        // issue this chunk's dY loads before staging B (they are independent)
        uint4 v[G];
#pragma unroll
        for (int g = 0; g < G; ++g) {
            const int c = (g * 32 + lane) * 8;
            v[g] = (row_ok && c < ci) ? __ldg(reinterpret_cast<const uint4*>(dr + i0 + c)) : make_uint4(0, 0, 0, 0);
        }
        __syncthreads();
        if ((r & 7) == 0) {
            // 16-byte vectors of the contiguous [ci, r] block of B, all loads in flight
            // first (C * RB / 8 / 256 == 8 per thread), then a transposing scatter
            constexpr int NV = C * RB / 8 / 256;
            const int nvec = ci * r / 8;
            const uint4* src = reinterpret_cast<const uint4*>(b + i0 * r);
            uint4 bv[NV];
#pragma unroll
            for (int q = 0; q < NV; ++q) {
                const int vq = threadIdx.x + 256 * q;
                if (vq < nvec) bv[q] = __ldg(src + vq);
            }
#pragma unroll
            for (int q = 0; q < NV; ++q) {
                const int vq = threadIdx.x + 256 * q;
                if (vq < nvec) {
                    const int i = (8 * vq) / r, j0 = (8 * vq) - i * r;
                    float f[8];
                    bf16x8_to_f32(bv[q], f);
#pragma unroll
                    for (int e = 0; e < 8; ++e) bt[(j0 + e) * C + i] = f[e];
                }
            }
            if (i0 == 0)   // rows r..RB-1 of bt stay zero for the whole kernel
                for (int idx = threadIdx.x; idx < (RB - r) * C; idx += 256) bt[r * C + idx] = 0.0f;
        } else {
            for (int idx = threadIdx.x; idx < ci * RB; idx += 256) {
                const int i = idx / RB, j = idx - i * RB;
                bt[j * C + i] = j < r ? __bfloat162float(b[(i0 + i) * r + j]) : 0.0f;
            }
        }
        __syncthreads();
#pragma unroll
        for (int g = 0; g < G; ++g) {
            const int c = (g * 32 + lane) * 8;
            if (c < ci) {
                float dv[8];
                bf16x8_to_f32(v[g], dv);
#pragma unroll
                for (int j = 0; j < RB; ++j) {
                    const float4 b0 = *reinterpret_cast<const float4*>(bt + j * C + c);
                    const float4 b1 = *reinterpret_cast<const float4*>(bt + j * C + c + 4);
                    float t = acc[j];
                    t = fmaf(dv[0], b0.x, t); t = fmaf(dv[1], b0.y, t);
                    t = fmaf(dv[2], b0.z, t); t = fmaf(dv[3], b0.w, t);
                    t = fmaf(dv[4], b1.x, t); t = fmaf(dv[5], b1.y, t);
                    t = fmaf(dv[6], b1.z, t); t = fmaf(dv[7], b1.w, t);
                    acc[j] = t;
                }
            }
        }
    }
#pragma unroll
    for (int j = 0; j < RB; ++j)
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc[j] += __shfl_xor_sync(0xffffffffu, acc[j], o);
    if (lane == 0 && row_ok) {
#pragma unroll
        for (int j = 0; j < RB; ++j)
            if (j < r) gh[row * r + j] = s * acc[j];
    }
}

template <int RB>
static cudaError_t launch_gh_rb(const bf16* dy, const bf16* b, int64_t T, int64_t m, int r, float s, float* gh,
                                cudaStream_t stream) {
    const int smem = 16384 * 4;
    auto kern = gh_kernel_v2<RB>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    kern<<<static_cast<unsigned>((T + 7) / 8), 256, smem, stream>>>(dy, b, T, m, r, s, gh);
    return cudaGetLastError();
}

cudaError_t launch_gh(const bf16* dy, const bf16* b, int64_t T, int64_t m, int r, float s, float* gh,
                      cudaStream_t stream) {
    if (T <= 0) return cudaSuccess;
    if (getenv("LORA_GH_V1")) {
        const unsigned blocks = static_cast<unsigned>((T + 7) / 8);
        if (r <= 8) gh_kernel<8><<<blocks, 256, 0, stream>>>(dy, b, T, m, r, s, gh);
        else gh_kernel<64><<<blocks, 256, 0, stream>>>(dy, b, T, m, r, s, gh);
        return cudaGetLastError();
    }
    if (r <= 4) return launch_gh_rb<4>(dy, b, T, m, r, s, gh, stream);
    if (r <= 8) return launch_gh_rb<8>(dy, b, T, m, r, s, gh, stream);
    if (r <= 16) return launch_gh_rb<16>(dy, b, T, m, r, s, gh, stream);
    if (r <= 32) return launch_gh_rb<32>(dy, b, T, m, r, s, gh, stream);
    return launch_gh_rb<64>(dy, b, T, m, r, s, gh, stream);
}

// ------------------------------------------------------------------ K3

#ifndef LORA_K3_STRIP
#define LORA_K3_STRIP 32
#endif
constexpr int kStrip = LORA_K3_STRIP;   // columns per CTA
int grad_strip_cols() { return kStrip; }
constexpr int kWarps = 8;

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

// ---- K3 with a TMA ring (r % 4 == 0): one producer thread streams 64-row
// tiles of the strip ([64 x 32] bf16 of x or dY plus the matching [64 x r]
// fp32 coefficient rows) through an mbarrier ring, so the 8 compute warps
// never wait on a global load; same ownership, order and reduction as above.
constexpr int kTmaRows = 64;

template <int RB, int CPT, int STAGES>
__global__ void __launch_bounds__(288, (RB >= 64 ? 1 : 2)) grad_strip_tma_kernel(const __grid_constant__ CUtensorMap tm_x,
                                                               const __grid_constant__ CUtensorMap tm_dy,
                                                               const __grid_constant__ CUtensorMap tm_gh,
                                                               const __grid_constant__ CUtensorMap tm_h,
                                                               const GradArgs g) {
    constexpr int LPR = kStrip / CPT;            // lanes per row
    constexpr int RPW = 32 / LPR;                // rows per warp instruction
    constexpr int X_BYTES = kTmaRows * kStrip * 2;
    constexpr int C_BYTES = kTmaRows * RB * 4;   // r <= RB; box inner = r
    constexpr int STAGE = X_BYTES + C_BYTES;
    extern __shared__ __align__(128) uint8_t smem_g[];
    uint8_t* ring = smem_g;
    uint64_t* full = reinterpret_cast<uint64_t*>(ring + STAGES * STAGE);
    uint64_t* empty = full + STAGES;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const bool is_a = static_cast<int>(blockIdx.x) < g.strips_a;
    const int64_t ncols = is_a ? g.n : g.m;
    const int64_t cs = static_cast<int64_t>(is_a ? blockIdx.x : blockIdx.x - g.strips_a) * kStrip;
    const int r = g.r;
    const int n_it = static_cast<int>((g.T + kTmaRows - 1) / kTmaRows);
    const uint32_t stage_tx = static_cast<uint32_t>(X_BYTES + kTmaRows * r * 4);

    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], kWarps);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    float acc[CPT][RB];
#pragma unroll
    for (int c = 0; c < CPT; ++c)
#pragma unroll
        for (int j = 0; j < RB; ++j) acc[c][j] = 0.0f;

    if (warp == kWarps) {
        // ---------------- producer ----------------
        if (lane == 0) {
            const CUtensorMap* mx = is_a ? &tm_x : &tm_dy;
            const CUtensorMap* mc = is_a ? &tm_gh : &tm_h;
            for (int it = 0; it < n_it; ++it) {
                const int s = it % STAGES;
                const uint32_t ph = (it / STAGES) & 1;
                mbar_wait(&empty[s], ph ^ 1);
                mbar_arrive_expect_tx(&full[s], stage_tx);
                uint8_t* dst = ring + s * STAGE;
                tma_load_2d(dst, mx, static_cast<int32_t>(cs), it * kTmaRows, &full[s]);
                tma_load_2d(dst + X_BYTES, mc, 0, it * kTmaRows, &full[s]);
            }
        }
    } else {
        // ---------------- 8 compute warps ----------------
        const int rs = lane / LPR, cc = lane % LPR;
        const bool col_ok = cs + cc * CPT < ncols;
        using VT = typename Vec<CPT>::T;
        for (int it = 0; it < n_it; ++it) {
            const int s = it % STAGES;
            const uint32_t ph = (it / STAGES) & 1;
            mbar_wait(&full[s], ph);
            const uint8_t* xs = ring + s * STAGE;
            const float* cf = reinterpret_cast<const float*>(xs + X_BYTES);
            if (col_ok) {
#pragma unroll
                for (int p = 0; p < kTmaRows / (RPW * kWarps); ++p) {
                    const int rr = p * RPW * kWarps + warp * RPW + rs;
                    float xv[CPT];
                    Vec<CPT>::cvt(*reinterpret_cast<const VT*>(xs + rr * (kStrip * 2) + cc * CPT * 2), xv);
                    const float4* cr = reinterpret_cast<const float4*>(cf + rr * r);
#pragma unroll
                    for (int j4 = 0; j4 < RB / 4; ++j4) {
                        if (4 * j4 < r) {
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
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[s]);
        }
        // (1) within the warp: lanes with the same column chunk (xor over the row bits)
#pragma unroll
        for (int off = LPR; off < 32; off <<= 1)
#pragma unroll
            for (int c = 0; c < CPT; ++c)
#pragma unroll
                for (int j = 0; j < RB; ++j) acc[c][j] += __shfl_xor_sync(0xffffffffu, acc[c][j], off);
    }
    // (2) across the 8 compute warps in warp order: red[w][j][col] (reuses the ring)
    __syncthreads();
    float* red = reinterpret_cast<float*>(smem_g);
    if (warp < kWarps && lane < LPR) {
#pragma unroll
        for (int j = 0; j < RB; ++j)
#pragma unroll
            for (int c = 0; c < CPT; ++c) red[(warp * RB + j) * kStrip + lane * CPT + c] = acc[c][j];
    }
    __syncthreads();
    for (int o = threadIdx.x; o < RB * kStrip; o += blockDim.x) {
        const int j = o / kStrip, col = o - j * kStrip;
        if (j >= r || cs + col >= ncols) continue;
        float sum = 0.0f;
#pragma unroll
        for (int w = 0; w < kWarps; ++w) sum += red[(w * RB + j) * kStrip + col];
        if (is_a) {
            float* d = g.da + static_cast<int64_t>(j) * ncols + cs + col;
            *d = g.accumulate ? *d + sum : sum;
        } else {
            const float v = g.scale_b * sum;
            float* d = g.db + (cs + col) * r + j;
            *d = g.accumulate ? *d + v : v;
        }
    }
}

template <int RB, int CPT>
static cudaError_t launch_strip_tma(int grid, const GradMaps& maps, const GradArgs& g, cudaStream_t stream) {
    constexpr int STAGE = kTmaRows * kStrip * 2 + kTmaRows * RB * 4;
    constexpr int STAGES = (96 * 1024 / STAGE) < 8 ? (96 * 1024 / STAGE) : 8;
    int smem = STAGES * STAGE + 2 * STAGES * 8;
    const int red_bytes = kWarps * RB * kStrip * 4;
    if (smem < red_bytes) smem = red_bytes;
    auto kern = grad_strip_tma_kernel<RB, CPT, STAGES>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    kern<<<grid, 288, smem, stream>>>(maps.x, maps.dy, maps.gh, maps.h, g);
    return cudaGetLastError();
}

cudaError_t launch_grad_reduce_tma(const GradMaps& maps, int64_t T, int64_t n, int64_t m, int r, float scale,
                                   float* da, float* db, int accumulate, cudaStream_t stream, int* launches) {
    GradArgs g = {};
    g.da = da; g.db = db;
    g.T = T; g.n = n; g.m = m; g.r = r; g.scale_b = scale; g.accumulate = accumulate;
    const int sa = da ? static_cast<int>((n + kStrip - 1) / kStrip) : 0;
    const int sb = db ? static_cast<int>((m + kStrip - 1) / kStrip) : 0;
    g.strips_a = sa;
    if (sa + sb == 0) return cudaSuccess;
    cudaError_t e;
    if (r <= 4) e = launch_strip_tma<4, 8>(sa + sb, maps, g, stream);
    else if (r <= 8) e = launch_strip_tma<8, 8>(sa + sb, maps, g, stream);
    else if (r <= 16) e = launch_strip_tma<16, 4>(sa + sb, maps, g, stream);
    else if (r <= 32) e = launch_strip_tma<32, 2>(sa + sb, maps, g, stream);
    else e = launch_strip_tma<64, 2>(sa + sb, maps, g, stream);
    if (e == cudaSuccess && launches) ++*launches;
    return e;
}

template <int CPT>
__device__ __forceinline__ void cp_async_vec(void* dst_smem, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], %2;"
                 ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(dst_smem))), "l"(src), "n"(CPT * 2)
                 : "memory");
}

// ---- K3 v3 (default): column blocks of 32*CPT columns (one warp instruction
// reads a full 512-byte row segment for CPT = 8) with the T tokens split
// across a cluster of kCS CTAs.  Each CTA reduces its rows (8 warps, fixed
// order, through shared memory); rank 0 then sums the kCS partials over
// distributed shared memory in rank order and writes the final dA / dB:
// one launch, no global partials, deterministic.
constexpr int kCS = 8;

template <int RB, int CPT>
__global__ void __launch_bounds__(256, (RB >= 64 ? 1 : 2)) grad_cluster_kernel(const __grid_constant__ GradGroup G) {
    // problem of this column block (grouped launch): blocks [block_start[p], block_start[p+1])
    int prob = 0;
    while (prob + 1 < G.count && static_cast<int>(blockIdx.x) >= G.block_start[prob + 1]) ++prob;
    const GradArgs& g = G.g[prob];
    const int blocks_a = G.blocks_a[prob];
    const int local_block = static_cast<int>(blockIdx.x) - G.block_start[prob];
    constexpr int CB = 32 * CPT;                 // columns per CTA
    constexpr int D = 16;                        // row segments in flight per warp
    constexpr int CHUNK = 8192 / RB;             // staged coefficient rows (32 KiB)
    using VT = typename Vec<CPT>::T;
    namespace cg = cooperative_groups;
    cg::cluster_group cluster = cg::this_cluster();
    extern __shared__ float4 smem_c[];
    float* s_coef = reinterpret_cast<float*>(smem_c);        // [CHUNK][RB]
    float* red = s_coef + CHUNK * RB;                          // [8 warps][RB][CB]
    float* part = red;                                         // [RB][CB] (reuses red[0])
    // [8 warps][D][32 lanes] x VT; aliases `red`, which is only used after the
    // row loop (the launcher sizes the region for the larger of the two)
    uint8_t* ring = reinterpret_cast<uint8_t*>(red);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int rank = static_cast<int>(cluster.block_rank());
    const bool is_a = local_block < blocks_a;
    const bf16* X = is_a ? g.x : g.dy;
    const float* coef = is_a ? g.gh : g.h;
    const int64_t ncols = is_a ? g.n : g.m;
    const int64_t cb0 = static_cast<int64_t>(is_a ? local_block : local_block - blocks_a) * CB;
    const int64_t c0 = cb0 + lane * CPT;
    const bool col_ok = c0 < ncols;
    const int r = g.r;
    int64_t rpc = (g.T + kCS - 1) / kCS;
    rpc = (rpc + 7) / 8 * 8;
    const int64_t t_begin = rank * rpc;
    const int64_t t_end = (g.T < t_begin + rpc) ? g.T : t_begin + rpc;
    griddep_wait();                       // programmatic dependent launch (see lora_gemm.cu)
    if (threadIdx.x == 0) griddep_launch_dependents();

    float acc[CPT][RB];
#pragma unroll
    for (int c = 0; c < CPT; ++c)
#pragma unroll
        for (int j = 0; j < RB; ++j) acc[c][j] = 0.0f;

    for (int64_t tb = t_begin; tb < t_end; tb += CHUNK) {
        const int nrow = static_cast<int>((t_end - tb) < CHUNK ? (t_end - tb) : CHUNK);
        __syncthreads();
        if (r == RB) {
            const float* src = coef + tb * r;
            for (int q = threadIdx.x; q < nrow * RB / 4; q += 256)
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;"
                             ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(s_coef + 4 * q))),
                               "l"(src + 4 * q) : "memory");
        } else {
            for (int idx = threadIdx.x; idx < nrow * RB; idx += 256) {
                const int rr = idx / RB, j = idx - rr * RB;
                s_coef[idx] = j < r ? coef[(tb + rr) * r + j] : 0.0f;
            }
        }
        asm volatile("cp.async.commit_group;" ::: "memory");   // group: the coefficients
        // each warp streams its rows (warp, warp+8, ...) through its own D-slot
        // cp.async ring: D row segments in flight per warp without registers;
        // a lane only ever reads back the bytes it copied itself
        const bf16* xp = X + tb * ncols + c0;
        VT* my_ring = reinterpret_cast<VT*>(ring) + (warp * D) * 32 + lane;   // slot k at my_ring[k * 32]
        const int n_i = (nrow - warp + 7) / 8;
#pragma unroll
        for (int i = 0; i < D; ++i) {
            const int rr = warp + 8 * i;
            if (col_ok && i < n_i)
                cp_async_vec<CPT>(my_ring + i * 32, xp + static_cast<int64_t>(rr) * ncols);
            asm volatile("cp.async.commit_group;" ::: "memory");
        }
        asm volatile("cp.async.wait_group %0;" ::"n"(D) : "memory");  // coefficients landed
        __syncthreads();
        for (int i = 0; i < n_i; ++i) {
            asm volatile("cp.async.wait_group %0;" ::"n"(D - 1) : "memory");
            const int rr = warp + 8 * i;
            const int slot = i % D;
            if (col_ok) {
                float xv[CPT];
                Vec<CPT>::cvt(my_ring[slot * 32], xv);
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
                if (i + D < n_i)
                    cp_async_vec<CPT>(my_ring + slot * 32, xp + static_cast<int64_t>(rr + 8 * D) * ncols);
            }
            asm volatile("cp.async.commit_group;" ::: "memory");
        }
        asm volatile("cp.async.wait_all;" ::: "memory");
    }
    // (1) the 8 warps of this CTA, in warp order
    __syncthreads();
#pragma unroll
    for (int j = 0; j < RB; ++j)
#pragma unroll
        for (int c = 0; c < CPT; ++c) red[(warp * RB + j) * CB + lane * CPT + c] = acc[c][j];
    __syncthreads();
    for (int o = threadIdx.x; o < RB * CB; o += 256) {
        float sum = 0.0f;
#pragma unroll
        for (int w = 0; w < kWarps; ++w) sum += red[w * RB * CB + o];
        part[o] = sum;  // part aliases red[0][*]: each o is read (by this thread) before it is written
    }
    // (2) the kCS CTAs of the cluster, in rank order, by rank 0 over DSMEM
    cluster.sync();
    if (rank == 0) {
        for (int o = threadIdx.x; o < RB * CB; o += 256) {
            const int j = o / CB, col = o - j * CB;
            if (j >= r || cb0 + col >= ncols) continue;
            float sum = 0.0f;
            for (int q = 0; q < kCS; ++q) sum += cluster.map_shared_rank(part, q)[o];
            if (is_a) {
                float* d = g.da + static_cast<int64_t>(j) * ncols + cb0 + col;
                *d = g.accumulate ? *d + sum : sum;
            } else {
                const float val = g.scale_b * sum;
                float* d = g.db + (cb0 + col) * r + j;
                *d = g.accumulate ? *d + val : val;
            }
        }
    }
    cluster.sync();
}

template <int RB, int CPT>
static cudaError_t launch_cluster_rb(GradGroup& G, cudaStream_t stream) {
    constexpr int CB = 32 * CPT;
    int blocks = 0;
    for (int p = 0; p < G.count; ++p) {
        const GradArgs& g = G.g[p];
        const int ba = g.da ? static_cast<int>((g.n + CB - 1) / CB) : 0;
        const int bb = g.db ? static_cast<int>((g.m + CB - 1) / CB) : 0;
        G.block_start[p] = blocks;
        G.blocks_a[p] = ba;
        blocks += ba + bb;
    }
    G.block_start[G.count] = blocks;
    if (blocks == 0) return cudaSuccess;
    const int red_bytes = kWarps * RB * CB * 4, ring_bytes = kWarps * 16 * 32 * CPT * 2;
    const int smem = 8192 * 4 + (red_bytes > ring_bytes ? red_bytes : ring_bytes);
    auto kern = grad_cluster_kernel<RB, CPT>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(blocks, kCS);
    cfg.blockDim = dim3(256);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 1;
    attr[0].val.clusterDim.y = kCS;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 2;
    e = cudaLaunchKernelEx(&cfg, kern, G);
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

int grad_rank_bucket(int r) { return r <= 4 ? 4 : r <= 8 ? 8 : r <= 16 ? 16 : r <= 32 ? 32 : 64; }

GradArgs make_grad_args(int64_t T, int64_t n, int64_t m, int r, float scale, const bf16* x, const float* gh,
                        const bf16* dy, const float* h, float* da, float* db, int accumulate) {
    GradArgs g = {};
    g.x = x; g.gh = gh; g.dy = dy; g.h = h; g.da = da; g.db = db;
    g.T = T; g.n = n; g.m = m; g.r = r; g.scale_b = scale; g.accumulate = accumulate;
    g.scale_a = 1.0f;
    return g;
}

cudaError_t launch_grad_reduce_cluster_group(GradGroup& G, cudaStream_t stream, int* launches) {
    if (G.count < 1 || G.count > kMaxGroup) return cudaErrorInvalidValue;
    const int rb = grad_rank_bucket(G.g[0].r);
    for (int p = 1; p < G.count; ++p)
        if (grad_rank_bucket(G.g[p].r) != rb) return cudaErrorInvalidValue;
    cudaError_t e;
    switch (rb) {
        case 4: e = launch_cluster_rb<4, 8>(G, stream); break;
        case 8: e = launch_cluster_rb<8, 8>(G, stream); break;
        case 16: e = launch_cluster_rb<16, 4>(G, stream); break;
        case 32: e = launch_cluster_rb<32, 2>(G, stream); break;
        default: e = launch_cluster_rb<64, 2>(G, stream); break;
    }
    if (e == cudaSuccess && launches && G.block_start[G.count] > 0) ++*launches;
    return e;
}

cudaError_t launch_grad_reduce_cluster(int64_t T, int64_t n, int64_t m, int r, float scale, const bf16* x,
                                       const float* gh, const bf16* dy, const float* h, float* da, float* db,
                                       int accumulate, cudaStream_t stream, int* launches) {
    if (!da && !db) return cudaSuccess;
    static thread_local GradGroup G;
    G.count = 1;
    G.g[0] = make_grad_args(T, n, m, r, scale, x, gh, dy, h, da, db, accumulate);
    return launch_grad_reduce_cluster_group(G, stream, launches);
}

template <int RB, int CPT, int MINB>
static cudaError_t launch_strip(int grid, const GradArgs& g, cudaStream_t stream) {
    const int smem = static_cast<int>(sizeof(float)) * (16384 > kWarps * RB * kStrip ? 16384 : kWarps * RB * kStrip);
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
