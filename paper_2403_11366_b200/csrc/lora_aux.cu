// lora_aux.cu -- the CUDA-core kernels of the LoRA path (sm_100a):
//   K4  merge       : W' = bf16(W0 + s B A) (Eq. 1 line 2)
//   N3  adam        : one bias-corrected Adam step for the adapters
//   helpers         : fp32 add (TP gradient accumulation), zero fill
// All are bandwidth-bound elementwise work ("Kernels").
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <cstring>

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

// two fp32 FMAs in one instruction (sm_100 FFMA2), each rounded to nearest
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
    uint64_t d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;"
        : "=l"(d)
        : "l"(*reinterpret_cast<const uint64_t*>(&a)), "l"(*reinterpret_cast<const uint64_t*>(&b)),
          "l"(*reinterpret_cast<const uint64_t*>(&c)));
    return *reinterpret_cast<const float2*>(&d);
}

// LORA_MERGE=oneshot: the one-shot merge kernel (comparison)
static bool merge_one_shot() {
    const char* v = getenv("LORA_MERGE");
    return v && !strcmp(v, "oneshot");
}

static int rank_bucket(int r) { return r <= 4 ? 4 : r <= 8 ? 8 : r <= 16 ? 16 : r <= 32 ? 32 : 64; }

// ------------------------------------------------------------------ K4 merge
// 64 rows x 256 columns per CTA; A[:, k0:k0+256] and B[i0:i0+64, :] staged in
// shared memory as fp32; each thread owns 8 consecutive columns (16-byte IO)
// of 8 rows.  Two CTAs per SM (128 registers: the 8 in-flight W0 rows spill a
// few bytes while the products run; measured faster than 1 CTA per SM).
template <int RB>
__global__ void __launch_bounds__(256, 2) merge_kernel(const bf16* __restrict__ w0, const bf16* __restrict__ a,
                                                    const bf16* __restrict__ b, int64_t n, int64_t m, int r,
                                                    float s, bf16* __restrict__ w_out) {
    extern __shared__ float4 smem_f4[];
    float* sA = reinterpret_cast<float*>(smem_f4);  // [RB][256]
    float* sB = sA + RB * 256;                       // [64][RB]
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t k0 = static_cast<int64_t>(blockIdx.x) * 256;
    const int64_t i0 = static_cast<int64_t>(blockIdx.y) * 64;
    const int kc = lane * 8;
    const bool col_ok = k0 + kc < n;
    // this thread's 8 rows of W0 (16-byte loads) go in flight FIRST: their HBM
    // latency overlaps the A / B staging below instead of following it
    uint4 wraw[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
        const int64_t i = i0 + warp + 8 * q;
        wraw[q] = (col_ok && i < m) ? __ldg(reinterpret_cast<const uint4*>(w0 + i * n + k0 + kc))
                                    : make_uint4(0, 0, 0, 0);
    }
    for (int idx = threadIdx.x; idx < RB * 32; idx += 256) {   // 8 columns per thread (n % 8 == 0)
        const int j = idx >> 5, kk = (idx & 31) * 8;
        float f[8];
        if (j < r && k0 + kk < n) {
            bf16x8_to_f32(__ldg(reinterpret_cast<const uint4*>(a + static_cast<int64_t>(j) * n + k0 + kk)), f);
        } else {
#pragma unroll
            for (int c = 0; c < 8; ++c) f[c] = 0.0f;
        }
        *reinterpret_cast<float4*>(sA + j * 256 + kk) = make_float4(f[0], f[1], f[2], f[3]);
        *reinterpret_cast<float4*>(sA + j * 256 + kk + 4) = make_float4(f[4], f[5], f[6], f[7]);
    }
    for (int idx = threadIdx.x; idx < 64 * RB; idx += 256) {
        const int ii = idx / RB, j = idx - ii * RB;
        sB[idx] = (j < r && i0 + ii < m) ? __bfloat162float(b[(i0 + ii) * r + j]) : 0.0f;
    }
    __syncthreads();
    if (!col_ok) return;
    // The kernel is issue-bound, not HBM-bound, when every row re-reads A from
    // shared memory and runs scalar FMAs: here A[j, kc..kc+8] is read once per j
    // for all 8 rows, and the products run as packed FFMA2 (two fp32 FMAs per
    // instruction, round-to-nearest each -- the same arithmetic, j ascending).
    float2 acc[8][4];
#pragma unroll
    for (int q = 0; q < 8; ++q)
#pragma unroll
        for (int c = 0; c < 4; ++c) acc[q][c] = make_float2(0.0f, 0.0f);
#pragma unroll
    for (int j = 0; j < RB; ++j) {
        if (j >= r) break;   // (uniform)
        const float4 a0 = *reinterpret_cast<const float4*>(sA + j * 256 + kc);
        const float4 a1 = *reinterpret_cast<const float4*>(sA + j * 256 + kc + 4);
        const float2 av[4] = {make_float2(a0.x, a0.y), make_float2(a0.z, a0.w), make_float2(a1.x, a1.y),
                              make_float2(a1.z, a1.w)};
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const float bij = sB[(warp + 8 * q) * RB + j];
            const float2 bb = make_float2(bij, bij);
#pragma unroll
            for (int c = 0; c < 4; ++c) acc[q][c] = ffma2(bb, av[c], acc[q][c]);
        }
    }
    const float2 ss = make_float2(s, s);
#pragma unroll
    for (int q = 0; q < 8; ++q) {
        const int64_t i = i0 + warp + 8 * q;
        if (i >= m) break;
        float wv[8];
        bf16x8_to_f32(wraw[q], wv);
        uint32_t o[4];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            const float2 r2 = ffma2(ss, acc[q][c], make_float2(wv[2 * c], wv[2 * c + 1]));   // W0 + s (B A)
            const __nv_bfloat162 p2 = __floats2bfloat162_rn(r2.x, r2.y);
            o[c] = *reinterpret_cast<const uint32_t*>(&p2);
        }
        *reinterpret_cast<uint4*>(w_out + i * n + k0 + kc) = make_uint4(o[0], o[1], o[2], o[3]);
    }
}

// Pipelined K4: a persistent CTA walks a contiguous range of 64 x 256 tiles
// (column-block major, so A[:, k0:k0+256] is re-staged only when the column
// block changes); the W0 tile and B's 64 rows of tile i+1 are in flight
// (cp.async, double-buffered in shared memory) while tile i is computed and
// stored -- the one-shot kernel above loaded, computed and stored in waves.
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool ok) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(smem))),
                 "l"(gmem), "r"(ok ? 16 : 0) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }

#ifndef LORA_MERGE_ROWS
#define LORA_MERGE_ROWS 64
#endif
constexpr int kMergeTR = LORA_MERGE_ROWS;      // tile rows (8 warps x kMergeTR / 8 rows each)
constexpr int kMergeQ = kMergeTR / 8;
template <int RB>
__global__ void __launch_bounds__(256, 2) merge_pipe_kernel(const bf16* __restrict__ w0, const bf16* __restrict__ a,
                                                            const bf16* __restrict__ b, int64_t n, int64_t m, int r,
                                                            float s, bf16* __restrict__ w_out, int64_t ntiles,
                                                            int64_t per_cta) {
    extern __shared__ uint4 smem_u4[];
    bf16* sW = reinterpret_cast<bf16*>(smem_u4);          // [2][TR][256]
    bf16* sBh = sW + 2 * kMergeTR * 256;                   // [2][TR * RB]
    float* sA = reinterpret_cast<float*>(sBh + 2 * kMergeTR * RB);   // [RB][256]
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int kc = lane * 8;
    const int64_t nrb = (m + kMergeTR - 1) / kMergeTR;
    const int64_t t_begin = static_cast<int64_t>(blockIdx.x) * per_cta;
    const int64_t t_end = t_begin + per_cta < ntiles ? t_begin + per_cta : ntiles;
    if (t_begin >= t_end) return;
    auto issue = [&](int64_t tile, int buf) {
        const int64_t cb = tile / nrb, rb = tile - (tile / nrb) * nrb;
        const int64_t k0 = cb * 256, i0 = rb * kMergeTR;
        const bool col_ok = k0 + kc < n;
#pragma unroll
        for (int q = 0; q < kMergeQ; ++q) {
            const int64_t i = i0 + warp + 8 * q;
            const bool ok = col_ok && i < m;
            cp_async16(sW + (buf * kMergeTR + warp + 8 * q) * 256 + kc, ok ? w0 + i * n + k0 + kc : w0, ok);
        }
        // B rows i0 .. i0 + 63 are one contiguous run of 64 r bf16 (16-byte chunks, r % 8 == 0 here)
        const int64_t rows = m - i0 < kMergeTR ? m - i0 : kMergeTR;
        const int chunks = static_cast<int>(rows * r / 8);
        for (int c = threadIdx.x; c < kMergeTR * RB / 8; c += 256)
            cp_async16(sBh + buf * kMergeTR * RB + c * 8, c < chunks ? b + i0 * r + c * 8 : b, c < chunks);
        cp_async_commit();
    };
    issue(t_begin, 0);
    int64_t cb_staged = -1;
    for (int64_t t = t_begin; t < t_end; ++t) {
        const int buf = static_cast<int>((t - t_begin) & 1);
        const int64_t cb = t / nrb, rb = t - cb * nrb;
        const int64_t k0 = cb * 256, i0 = rb * kMergeTR;
        if (cb != cb_staged) {   // A[:, k0:k0+256] as fp32 (previous tile's readers are past the barrier)
            for (int idx = threadIdx.x; idx < RB * 32; idx += 256) {
                const int j = idx >> 5, kk = (idx & 31) * 8;
                float f[8];
                if (j < r && k0 + kk < n) {
                    bf16x8_to_f32(__ldg(reinterpret_cast<const uint4*>(a + static_cast<int64_t>(j) * n + k0 + kk)), f);
                } else {
#pragma unroll
                    for (int c = 0; c < 8; ++c) f[c] = 0.0f;
                }
                *reinterpret_cast<float4*>(sA + j * 256 + kk) = make_float4(f[0], f[1], f[2], f[3]);
                *reinterpret_cast<float4*>(sA + j * 256 + kk + 4) = make_float4(f[4], f[5], f[6], f[7]);
            }
            cb_staged = cb;
        }
        if (t + 1 < t_end) issue(t + 1, buf ^ 1);
        else cp_async_commit();   // (empty group: wait_group 1 below then covers tile t)
        cp_async_wait1();
        __syncthreads();
        if (k0 + kc < n) {
            float2 acc[kMergeQ][4];
#pragma unroll
            for (int q = 0; q < kMergeQ; ++q)
#pragma unroll
                for (int c = 0; c < 4; ++c) acc[q][c] = make_float2(0.0f, 0.0f);
            const bf16* bsm = sBh + buf * kMergeTR * RB;
#pragma unroll
            for (int j = 0; j < RB; ++j) {
                if (j >= r) break;   // (uniform)
                const float4 a0 = *reinterpret_cast<const float4*>(sA + j * 256 + kc);
                const float4 a1 = *reinterpret_cast<const float4*>(sA + j * 256 + kc + 4);
                const float2 av[4] = {make_float2(a0.x, a0.y), make_float2(a0.z, a0.w), make_float2(a1.x, a1.y),
                                      make_float2(a1.z, a1.w)};
#pragma unroll
                for (int q = 0; q < kMergeQ; ++q) {
                    const float bij = __bfloat162float(bsm[(warp + 8 * q) * r + j]);
                    const float2 bb = make_float2(bij, bij);
#pragma unroll
                    for (int c = 0; c < 4; ++c) acc[q][c] = ffma2(bb, av[c], acc[q][c]);
                }
            }
            const float2 ss = make_float2(s, s);
#pragma unroll
            for (int q = 0; q < kMergeQ; ++q) {
                const int64_t i = i0 + warp + 8 * q;
                if (i >= m) break;
                float wv[8];
                bf16x8_to_f32(*reinterpret_cast<const uint4*>(sW + (buf * kMergeTR + warp + 8 * q) * 256 + kc), wv);
                uint32_t o[4];
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    const float2 r2 = ffma2(ss, acc[q][c], make_float2(wv[2 * c], wv[2 * c + 1]));
                    const __nv_bfloat162 p2 = __floats2bfloat162_rn(r2.x, r2.y);
                    o[c] = *reinterpret_cast<const uint32_t*>(&p2);
                }
                *reinterpret_cast<uint4*>(w_out + i * n + k0 + kc) = make_uint4(o[0], o[1], o[2], o[3]);
            }
        }
        __syncthreads();   // buffer `buf` and sA are free for the next issue / staging
    }
}

template <int RB>
static cudaError_t launch_merge_rb(const bf16* w0, const bf16* a, const bf16* b, int64_t n, int64_t m,
                                   int r, float s, bf16* w_out, cudaStream_t stream) {
    cudaError_t e;
    if (r % 8 == 0 && !merge_one_shot()) {   // pipelined (B rows as 16-byte chunks need r % 8 == 0)
        const size_t smem = 2 * kMergeTR * 256 * 2 + 2 * kMergeTR * RB * 2 + RB * 256 * 4;
        auto kern = merge_pipe_kernel<RB>;
        if ((e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem))) !=
            cudaSuccess)
            return e;
        int dev = 0, sms = 148, per_sm = 1;
        if ((e = cudaGetDevice(&dev)) != cudaSuccess) return e;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 256, smem);
        if (per_sm < 1) per_sm = 1;
        const int64_t ntiles = ((n + 255) / 256) * ((m + kMergeTR - 1) / kMergeTR);
        const int64_t ctas = std::min<int64_t>(ntiles, int64_t(sms) * per_sm);
        const int64_t per_cta = (ntiles + ctas - 1) / ctas;
        kern<<<static_cast<unsigned>((ntiles + per_cta - 1) / per_cta), 256, smem, stream>>>(w0, a, b, n, m, r, s,
                                                                                           w_out, ntiles, per_cta);
        return cudaGetLastError();
    }
    const size_t smem = (RB * 256 + 64 * RB) * sizeof(float);
    auto kern = merge_kernel<RB>;
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
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

// ------------------------------------------------------------------ N3: adapter update
// One bias-corrected Adam step (Kingma & Ba 2015, Alg. 1) for
// all adapter tensors of a model in ONE launch: 4 elements per thread (16-byte
// fp32 loads of grad / m / v / master, 8-byte bf16 param), grid-stride over the
// concatenated element range.  fp32 arithmetic; the bf16 param the fused
// kernels read is RNE(master).
__global__ void __launch_bounds__(256) adam_kernel(const __grid_constant__ AdamGroup G) {
    const int64_t total4 = G.start4[G.count];
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    int ti = 0;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < total4; i += stride) {
        while (i >= G.start4[ti + 1]) ++ti;   // i only grows: the tensor index only moves forward
        const AdamTensor& t = G.t[ti];
        const int64_t e = (i - G.start4[ti]) * 4;
        const float4 g = *reinterpret_cast<const float4*>(t.grad + e);
        float4 m = *reinterpret_cast<const float4*>(t.m + e);
        float4 v = *reinterpret_cast<const float4*>(t.v + e);
        float th[4];
        if (t.master) {
            const float4 w = *reinterpret_cast<const float4*>(t.master + e);
            th[0] = w.x; th[1] = w.y; th[2] = w.z; th[3] = w.w;
        } else {
            const uint2 u = *reinterpret_cast<const uint2*>(t.param + e);
            const float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.x));
            const float2 b = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.y));
            th[0] = a.x; th[1] = a.y; th[2] = b.x; th[3] = b.y;
        }
        float* mp = &m.x;
        float* vp = &v.x;
        const float* gp = &g.x;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            mp[c] = G.b1 * mp[c] + (1.0f - G.b1) * gp[c];
            vp[c] = G.b2 * vp[c] + (1.0f - G.b2) * gp[c] * gp[c];
            const float m_hat = mp[c] / G.bc1;
            const float v_hat = vp[c] / G.bc2;
            th[c] = th[c] - G.lr * m_hat / (sqrtf(v_hat) + G.eps);
        }
        *reinterpret_cast<float4*>(t.m + e) = m;
        *reinterpret_cast<float4*>(t.v + e) = v;
        if (t.master) *reinterpret_cast<float4*>(t.master + e) = make_float4(th[0], th[1], th[2], th[3]);
        const __nv_bfloat162 p0 = __floats2bfloat162_rn(th[0], th[1]);
        const __nv_bfloat162 p1 = __floats2bfloat162_rn(th[2], th[3]);
        *reinterpret_cast<uint2*>(t.param + e) =
            make_uint2(*reinterpret_cast<const uint32_t*>(&p0), *reinterpret_cast<const uint32_t*>(&p1));
    }
}

cudaError_t launch_adam(AdamGroup& G, int num_sms, cudaStream_t stream) {
    if (G.count < 1 || G.count > kMaxAdamTensors) return cudaErrorInvalidValue;
    int64_t total4 = 0;
    for (int i = 0; i < G.count; ++i) {
        G.start4[i] = total4;
        total4 += G.t[i].numel / 4;
    }
    G.start4[G.count] = total4;
    if (total4 == 0) return cudaSuccess;
    const int64_t blocks = std::min<int64_t>((total4 + 255) / 256, static_cast<int64_t>(num_sms) * 8);
    adam_kernel<<<static_cast<unsigned>(blocks), 256, 0, stream>>>(G);
    return cudaGetLastError();
}

// dst = RNE_bf16(sum_g src_g), fp32 accumulation in g order (TP column group: the
// members' dX partials w.r.t. their shared input); 8 elements per thread
__global__ void __launch_bounds__(256) sum_bf16_kernel(const __grid_constant__ SumBf16Args A) {
    const int64_t n8 = A.count / 8;
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n8; i += stride) {
        float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
        for (int g = 0; g < A.n; ++g) {
            float f[8];
            bf16x8_to_f32(__ldg(reinterpret_cast<const uint4*>(A.src[g]) + i), f);
#pragma unroll
            for (int c = 0; c < 8; ++c) acc[c] += f[c];
        }
        uint4 o;
        __nv_bfloat162 p0 = __floats2bfloat162_rn(acc[0], acc[1]), p1 = __floats2bfloat162_rn(acc[2], acc[3]);
        __nv_bfloat162 p2 = __floats2bfloat162_rn(acc[4], acc[5]), p3 = __floats2bfloat162_rn(acc[6], acc[7]);
        o.x = *reinterpret_cast<uint32_t*>(&p0);
        o.y = *reinterpret_cast<uint32_t*>(&p1);
        o.z = *reinterpret_cast<uint32_t*>(&p2);
        o.w = *reinterpret_cast<uint32_t*>(&p3);
        reinterpret_cast<uint4*>(A.dst)[i] = o;
    }
}

cudaError_t launch_sum_bf16(const SumBf16Args& A, int num_sms, cudaStream_t stream) {
    if (A.n < 1 || A.n > kMaxGroup || A.count % 8 != 0) return cudaErrorInvalidValue;
    if (A.count == 0) return cudaSuccess;
    const int64_t blocks = std::min<int64_t>((A.count / 8 + 255) / 256, static_cast<int64_t>(num_sms) * 8);
    sum_bf16_kernel<<<static_cast<unsigned>(blocks), 256, 0, stream>>>(A);
    return cudaGetLastError();
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
