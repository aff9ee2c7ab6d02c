// lora_aux.cu -- the CUDA-core kernels of the LoRA hot path (sm_100a):
//   B6  pack        : padded / transposed copies of the adapters for TMA
//   K3  grad reduce : dA = gh^T x and dB = s dY^T h (the two
//                     trainable gradients), column-strip ownership, 16-byte
//                     coalesced loads, fixed-order warp/CTA reductions
//   K3a rowproj     : h = x A^T or gh = s dY B for the NULL-h / NULL-dx paths
//   K4  merge       : W' = bf16(W0 + s B A) (Eq. 1 line 2)
// These steps are skinny (rank r <= 64) and bandwidth-bound, so they run on
// the CUDA cores ("Kernels").
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "lora_kernels.h"

namespace lora_sm100 {

typedef __nv_bfloat16 bf16;

// ------------------------------------------------------------------ helpers
__device__ __forceinline__ void bf16x8_to_f32(const uint4& u, float (&f)[8]) {
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        float2 t = __bfloat1622float2(h[i]);
        f[2 * i] = t.x;
        f[2 * i + 1] = t.y;
    }
}

template <int CPT>
__device__ __forceinline__ void load_bf16_vec(const bf16* p, float (&f)[CPT]) {
    if constexpr (CPT == 8) {
        uint4 u = __ldg(reinterpret_cast<const uint4*>(p));
        bf16x8_to_f32(u, f);
    } else if constexpr (CPT == 4) {
        uint2 u = __ldg(reinterpret_cast<const uint2*>(p));
        const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
        float2 a = __bfloat1622float2(h[0]), b = __bfloat1622float2(h[1]);
        f[0] = a.x; f[1] = a.y; f[2] = b.x; f[3] = b.y;
    } else {
        uint32_t u = __ldg(reinterpret_cast<const unsigned int*>(p));
        float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u));
        f[0] = a.x; f[1] = a.y;
    }
}

static int rank_bucket(int r) { return r <= 4 ? 4 : r <= 8 ? 8 : r <= 16 ? 16 : r <= 32 ? 32 : 64; }
static int cols_per_thread(int rb) { return rb <= 16 ? 8 : (rb == 32 ? 4 : 2); }

// ------------------------------------------------------------------ B6 pack
__global__ void pack_kernel(const bf16* __restrict__ a, const bf16* __restrict__ b, int64_t n,
                            int64_t m, int r, int r_pad, bf16* __restrict__ bpad,
                            bf16* __restrict__ bt, bf16* __restrict__ at) {
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    const int64_t t0 = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const bf16 zero = __float2bfloat16(0.0f);
    if (bpad)
        for (int64_t idx = t0; idx < m * r_pad; idx += stride) {
            const int64_t i = idx / r_pad;
            const int j = static_cast<int>(idx - i * r_pad);
            bpad[idx] = j < r ? b[i * r + j] : zero;
        }
    if (bt)
        for (int64_t idx = t0; idx < static_cast<int64_t>(r) * m; idx += stride) {
            const int64_t j = idx / m, i = idx - j * m;
            bt[idx] = b[i * r + j];
        }
    if (at)
        for (int64_t idx = t0; idx < n * r_pad; idx += stride) {
            const int64_t k = idx / r_pad;
            const int j = static_cast<int>(idx - k * r_pad);
            at[idx] = j < r ? a[static_cast<int64_t>(j) * n + k] : zero;
        }
}

cudaError_t launch_pack(const bf16* a, const bf16* b, int64_t n, int64_t m, int r, int r_pad,
                        bf16* bpad, bf16* bt, bf16* at, int num_sms, cudaStream_t stream) {
    int64_t work = 0;
    if (bpad) work = std::max<int64_t>(work, m * r_pad);
    if (bt) work = std::max<int64_t>(work, static_cast<int64_t>(r) * m);
    if (at) work = std::max<int64_t>(work, n * r_pad);
    if (work == 0) return cudaSuccess;
    const int threads = 256;
    int64_t blocks = (work + threads - 1) / threads;
    blocks = std::min<int64_t>(blocks, 4LL * num_sms);
    pack_kernel<<<static_cast<int>(blocks), threads, 0, stream>>>(a, b, n, m, r, r_pad, bpad, bt, at);
    return cudaGetLastError();
}

// ------------------------------------------------------------------ K3
struct GradArgs {
    const bf16* x;     // [T, n]
    const float* gh;   // [T, r]
    const bf16* dy;    // [T, m]
    const float* h;    // [T, r]
    int64_t T, n, m;
    int r;
    int strips_a, rows_per_chunk;
    float* part_a;     // [chunks, r, n]
    float* part_b;     // [chunks, r, m]
};

constexpr int kSubRows = 64;

// partial[chunk, j, c] = sum_{t in chunk} coef[t, j] * X[t, c]
// blockIdx.x: column strip (dA strips first, then dB strips); blockIdx.y: token chunk.
template <int RB, int CPT>
__global__ void __launch_bounds__(256) grad_partial_kernel(const GradArgs g) {
    constexpr int CPS = 32 * CPT;
    extern __shared__ float4 smem_f4[];
    float* s_coef = reinterpret_cast<float*>(smem_f4);   // [kSubRows][RB]
    float* s_red = s_coef + kSubRows * RB;                // [4][RB][CPS]
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const bool is_a = static_cast<int>(blockIdx.x) < g.strips_a;
    const bf16* X = is_a ? g.x : g.dy;
    const float* coef = is_a ? g.gh : g.h;
    const int64_t ncols = is_a ? g.n : g.m;
    const int strip = is_a ? blockIdx.x : blockIdx.x - g.strips_a;
    const int64_t c0 = static_cast<int64_t>(strip) * CPS + lane * CPT;
    const bool col_ok = c0 < ncols;  // ncols % 8 == 0 and CPT | 8 -> whole vector in range
    const int64_t t_begin = static_cast<int64_t>(blockIdx.y) * g.rows_per_chunk;
    const int64_t t_end = (g.T < t_begin + g.rows_per_chunk) ? g.T : t_begin + g.rows_per_chunk;
    const int r = g.r;

    float acc[CPT][RB];
#pragma unroll
    for (int c = 0; c < CPT; ++c)
#pragma unroll
        for (int j = 0; j < RB; ++j) acc[c][j] = 0.0f;

    for (int64_t tb = t_begin; tb < t_end; tb += kSubRows) {
        const int nrow = static_cast<int>((t_end - tb) < kSubRows ? (t_end - tb) : kSubRows);
        __syncthreads();
        for (int idx = threadIdx.x; idx < kSubRows * RB; idx += 256) {
            const int rr = idx / RB, j = idx - rr * RB;
            s_coef[idx] = (rr < nrow && j < r) ? coef[(tb + rr) * r + j] : 0.0f;
        }
        __syncthreads();
        if (col_ok) {
            const bf16* xp = X + tb * ncols + c0;
#pragma unroll 4
            for (int rr = warp; rr < nrow; rr += 8) {
                float xv[CPT];
                load_bf16_vec<CPT>(xp + static_cast<int64_t>(rr) * ncols, xv);
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

    // fixed-order cross-warp tree: ((w0+w4)+(w2+w6)) + ((w1+w5)+(w3+w7))
    auto put = [&](int slot) {
#pragma unroll
        for (int j = 0; j < RB; ++j)
#pragma unroll
            for (int c = 0; c < CPT; ++c) s_red[(slot * RB + j) * CPS + lane * CPT + c] = acc[c][j];
    };
    auto add = [&](int slot) {
#pragma unroll
        for (int j = 0; j < RB; ++j)
#pragma unroll
            for (int c = 0; c < CPT; ++c) acc[c][j] += s_red[(slot * RB + j) * CPS + lane * CPT + c];
    };
    __syncthreads();
    if (warp >= 4) put(warp - 4);
    __syncthreads();
    if (warp < 4) add(warp);
    __syncthreads();
    if (warp >= 2 && warp < 4) put(warp - 2);
    __syncthreads();
    if (warp < 2) add(warp);
    __syncthreads();
    if (warp == 1) put(0);
    __syncthreads();
    if (warp == 0 && col_ok) {
        add(0);
        float* part = is_a ? g.part_a : g.part_b;
        const int64_t base = static_cast<int64_t>(blockIdx.y) * r;
#pragma unroll
        for (int j = 0; j < RB; ++j) {
            if (j < r) {
                float* dst = part + (base + j) * ncols + c0;
#pragma unroll
                for (int c = 0; c < CPT; ++c) dst[c] = acc[c][j];
            }
        }
    }
}

// dA[j,k] = sum_chunk part_a;  dB[i,j] = scale * sum_chunk part_b (chunk order fixed)
__global__ void grad_finalize_kernel(const float* __restrict__ part_a, const float* __restrict__ part_b,
                                     int chunks, int r, int64_t n, int64_t m, float scale_b,
                                     float* __restrict__ da, float* __restrict__ db, int accumulate) {
    const int64_t na = da ? static_cast<int64_t>(r) * n : 0;
    const int64_t nb = db ? static_cast<int64_t>(r) * m : 0;
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; idx < na + nb;
         idx += stride) {
        if (idx < na) {
            float s = 0.0f;
            for (int c = 0; c < chunks; ++c) s += part_a[static_cast<int64_t>(c) * r * n + idx];
            da[idx] = accumulate ? da[idx] + s : s;  // idx = j * n + k
        } else {
            const int64_t q = idx - na;              // q = j * m + i
            const int64_t j = q / m, i = q - j * m;
            float s = 0.0f;
            for (int c = 0; c < chunks; ++c) s += part_b[static_cast<int64_t>(c) * r * m + q];
            const float v = scale_b * s;
            float* d = db + i * r + j;
            *d = accumulate ? *d + v : v;
        }
    }
}

GradReducePlan plan_grad_reduce(int64_t T, int64_t n, int64_t m, int r, int num_sms) {
    GradReducePlan pl{};
    pl.r_bucket = rank_bucket(r);
    pl.cols_per_strip = 32 * cols_per_thread(pl.r_bucket);
    pl.strips_a = static_cast<int>((n + pl.cols_per_strip - 1) / pl.cols_per_strip);
    pl.strips_b = static_cast<int>((m + pl.cols_per_strip - 1) / pl.cols_per_strip);
    const int strips = pl.strips_a + pl.strips_b;
    const int64_t target = 2LL * num_sms;
    int64_t chunks = (target + strips - 1) / strips;
    const int64_t max_chunks = std::max<int64_t>(1, (T + 31) / 32);  // >= 32 rows per chunk
    chunks = std::max<int64_t>(1, std::min(chunks, max_chunks));
    int64_t rows = (T + chunks - 1) / chunks;
    rows = std::max<int64_t>(8, (rows + 7) / 8 * 8);
    pl.rows_per_chunk = static_cast<int>(rows);
    pl.chunks = static_cast<int>(std::max<int64_t>(1, (T + rows - 1) / rows));
    return pl;
}

size_t grad_reduce_partial_bytes(const GradReducePlan& pl, int64_t n, int64_t m, int r) {
    return static_cast<size_t>(pl.chunks) * r * (n + m) * sizeof(float);
}

template <int RB, int CPT>
static cudaError_t launch_partial(dim3 grid, const GradArgs& g, cudaStream_t stream) {
    const size_t smem = (kSubRows * RB + 4 * RB * 32 * CPT) * sizeof(float);
    auto kern = grad_partial_kernel<RB, CPT>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    kern<<<grid, 256, smem, stream>>>(g);
    return cudaGetLastError();
}

cudaError_t launch_grad_reduce(const GradReducePlan& pl, int64_t T, int64_t n, int64_t m, int r,
                               float scale, const bf16* x, const float* gh, const bf16* dy,
                               const float* h, float* partials, float* da, float* db,
                               int accumulate, cudaStream_t stream, int* launches) {
    GradArgs g;
    g.x = x; g.gh = gh; g.dy = dy; g.h = h;
    g.T = T; g.n = n; g.m = m; g.r = r;
    g.rows_per_chunk = pl.rows_per_chunk;
    g.part_a = partials;
    g.part_b = partials + static_cast<int64_t>(pl.chunks) * r * n;
    // strips of gradients that were not requested are dropped from the grid
    const int sa = da ? pl.strips_a : 0;
    const int sb = db ? pl.strips_b : 0;
    if (sa + sb == 0) return cudaSuccess;
    g.strips_a = sa;
    if (!da) { g.x = dy; g.gh = h; }  // keep pointers valid; only dB strips exist
    dim3 grid(sa + sb, pl.chunks);
    cudaError_t e;
    switch (pl.r_bucket) {
        case 4: e = launch_partial<4, 8>(grid, g, stream); break;
        case 8: e = launch_partial<8, 8>(grid, g, stream); break;
        case 16: e = launch_partial<16, 8>(grid, g, stream); break;
        case 32: e = launch_partial<32, 4>(grid, g, stream); break;
        default: e = launch_partial<64, 2>(grid, g, stream); break;
    }
    if (e != cudaSuccess) return e;
    if (launches) ++*launches;
    const int64_t work = (da ? static_cast<int64_t>(r) * n : 0) + (db ? static_cast<int64_t>(r) * m : 0);
    const int blocks = static_cast<int>(std::min<int64_t>((work + 255) / 256, 1024));
    grad_finalize_kernel<<<blocks, 256, 0, stream>>>(g.part_a, g.part_b, pl.chunks, r, n, m, scale,
                                                     da, db, accumulate);
    if (launches) ++*launches;
    return cudaGetLastError();
}

// ------------------------------------------------------------------ K3a
template <int RB>
__global__ void __launch_bounds__(256) rowproj_kernel(const bf16* __restrict__ X, int64_t T, int64_t K,
                                                      const bf16* __restrict__ P, int r, float scale,
                                                      float* __restrict__ out) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t row = static_cast<int64_t>(blockIdx.x) * 8 + warp;
    if (row >= T) return;
    float acc[RB];
#pragma unroll
    for (int j = 0; j < RB; ++j) acc[j] = 0.0f;
    const bf16* xr = X + row * K;
    for (int64_t k = lane * 8; k < K; k += 256) {
        float xv[8];
        load_bf16_vec<8>(xr + k, xv);
#pragma unroll
        for (int j = 0; j < RB; ++j) {
            if (j < r) {
                float pv[8];
                load_bf16_vec<8>(P + static_cast<int64_t>(j) * K + k, pv);
#pragma unroll
                for (int c = 0; c < 8; ++c) acc[j] = fmaf(xv[c], pv[c], acc[j]);
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
            if (j < r) out[row * r + j] = scale * acc[j];
    }
}

cudaError_t launch_rowproj(const bf16* X, int64_t T, int64_t K, const bf16* P, int r, float scale,
                           float* out, cudaStream_t stream) {
    if (T <= 0) return cudaSuccess;
    const unsigned blocks = static_cast<unsigned>((T + 7) / 8);
    switch (rank_bucket(r)) {
        case 4: rowproj_kernel<4><<<blocks, 256, 0, stream>>>(X, T, K, P, r, scale, out); break;
        case 8: rowproj_kernel<8><<<blocks, 256, 0, stream>>>(X, T, K, P, r, scale, out); break;
        case 16: rowproj_kernel<16><<<blocks, 256, 0, stream>>>(X, T, K, P, r, scale, out); break;
        case 32: rowproj_kernel<32><<<blocks, 256, 0, stream>>>(X, T, K, P, r, scale, out); break;
        default: rowproj_kernel<64><<<blocks, 256, 0, stream>>>(X, T, K, P, r, scale, out); break;
    }
    return cudaGetLastError();
}

// ------------------------------------------------------------------ K4 merge
// 64 rows x 256 columns per CTA; A[:, k0:k0+256] and B[i0:i0+64, :] staged in
// shared memory as fp32; each thread owns 8 consecutive columns (16-byte IO).
template <int RB>
__global__ void __launch_bounds__(256) merge_kernel(const bf16* __restrict__ w0, const bf16* __restrict__ a,
                                                    const bf16* __restrict__ b, int64_t n, int64_t m, int r,
                                                    float s, bf16* __restrict__ w_out) {
    extern __shared__ float4 smem_f4[];
    float* sA = reinterpret_cast<float*>(smem_f4);  // [RB][256]
    float* sB = sA + RB * 256;                       // [64][RB]
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t k0 = static_cast<int64_t>(blockIdx.x) * 256;
    const int64_t i0 = static_cast<int64_t>(blockIdx.y) * 64;
    for (int idx = threadIdx.x; idx < RB * 256; idx += 256) {
        const int j = idx >> 8, kk = idx & 255;
        sA[idx] = (j < r && k0 + kk < n) ? __bfloat162float(a[static_cast<int64_t>(j) * n + k0 + kk]) : 0.0f;
    }
    for (int idx = threadIdx.x; idx < 64 * RB; idx += 256) {
        const int ii = idx / RB, j = idx - ii * RB;
        sB[idx] = (j < r && i0 + ii < m) ? __bfloat162float(b[(i0 + ii) * r + j]) : 0.0f;
    }
    __syncthreads();
    const int kc = lane * 8;
    if (k0 + kc >= n) return;
#pragma unroll 1
    for (int q = 0; q < 8; ++q) {
        const int ii = warp + 8 * q;
        const int64_t i = i0 + ii;
        if (i >= m) break;
        const int64_t off = i * n + k0 + kc;
        float wv[8];
        load_bf16_vec<8>(w0 + off, wv);
        float ba[8];
#pragma unroll
        for (int c = 0; c < 8; ++c) ba[c] = 0.0f;
#pragma unroll
        for (int j = 0; j < RB; ++j) {
            const float bij = sB[ii * RB + j];
            const float4 a0 = *reinterpret_cast<const float4*>(sA + j * 256 + kc);
            const float4 a1 = *reinterpret_cast<const float4*>(sA + j * 256 + kc + 4);
            ba[0] = fmaf(bij, a0.x, ba[0]); ba[1] = fmaf(bij, a0.y, ba[1]);
            ba[2] = fmaf(bij, a0.z, ba[2]); ba[3] = fmaf(bij, a0.w, ba[3]);
            ba[4] = fmaf(bij, a1.x, ba[4]); ba[5] = fmaf(bij, a1.y, ba[5]);
            ba[6] = fmaf(bij, a1.z, ba[6]); ba[7] = fmaf(bij, a1.w, ba[7]);
        }
        uint4 o;
        __nv_bfloat162 p0 = __floats2bfloat162_rn(wv[0] + s * ba[0], wv[1] + s * ba[1]);
        __nv_bfloat162 p1 = __floats2bfloat162_rn(wv[2] + s * ba[2], wv[3] + s * ba[3]);
        __nv_bfloat162 p2 = __floats2bfloat162_rn(wv[4] + s * ba[4], wv[5] + s * ba[5]);
        __nv_bfloat162 p3 = __floats2bfloat162_rn(wv[6] + s * ba[6], wv[7] + s * ba[7]);
        o.x = *reinterpret_cast<uint32_t*>(&p0);
        o.y = *reinterpret_cast<uint32_t*>(&p1);
        o.z = *reinterpret_cast<uint32_t*>(&p2);
        o.w = *reinterpret_cast<uint32_t*>(&p3);
        *reinterpret_cast<uint4*>(w_out + off) = o;
    }
}

template <int RB>
static cudaError_t launch_merge_rb(const bf16* w0, const bf16* a, const bf16* b, int64_t n, int64_t m,
                                   int r, float s, bf16* w_out, cudaStream_t stream) {
    const size_t smem = (RB * 256 + 64 * RB) * sizeof(float);
    auto kern = merge_kernel<RB>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    dim3 grid(static_cast<unsigned>((n + 255) / 256), static_cast<unsigned>((m + 63) / 64));
    kern<<<grid, 256, smem, stream>>>(w0, a, b, n, m, r, s, w_out);
    return cudaGetLastError();
}

cudaError_t launch_merge(const bf16* w0, const bf16* a, const bf16* b, int64_t n, int64_t m, int r,
                         float s, bf16* w_out, cudaStream_t stream) {
    switch (rank_bucket(r)) {
        case 4: return launch_merge_rb<4>(w0, a, b, n, m, r, s, w_out, stream);
        case 8: return launch_merge_rb<8>(w0, a, b, n, m, r, s, w_out, stream);
        case 16: return launch_merge_rb<16>(w0, a, b, n, m, r, s, w_out, stream);
        case 32: return launch_merge_rb<32>(w0, a, b, n, m, r, s, w_out, stream);
        default: return launch_merge_rb<64>(w0, a, b, n, m, r, s, w_out, stream);
    }
}

__global__ void add_f32_kernel(float* __restrict__ dst, const float* __restrict__ src, int64_t count) {
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < count; i += stride)
        dst[i] += src[i];
}

cudaError_t launch_add_f32(float* dst, const float* src, int64_t count, cudaStream_t stream) {
    if (count <= 0) return cudaSuccess;
    const int blocks = static_cast<int>(std::min<int64_t>((count + 255) / 256, 1024));
    add_f32_kernel<<<blocks, 256, 0, stream>>>(dst, src, count);
    return cudaGetLastError();
}

cudaError_t launch_fill_zero(float* p, int64_t count, cudaStream_t stream) {
    if (!p || count <= 0) return cudaSuccess;
    return cudaMemsetAsync(p, 0, static_cast<size_t>(count) * sizeof(float), stream);
}

}  // namespace lora_sm100
