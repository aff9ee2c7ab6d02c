// lora_layer.cu -- the non-LoRA pieces of a Llama-2 decoder layer (SURVEY.md
// 8(f) N4: "full Llama-2 decoder-layer train step ... RMSNorm, RoPE, SwiGLU";
// JORA builds on a Llama-2 implementation -- and :195, the
// long-sequence RAFT setting).  All are HBM-bound row / element kernels with
// 16-byte IO and fp32 math; bf16 in and out.  The attention itself is the cuDNN
// SDPA library call, the seven projections are the LoRA linears.
//
//   RMSNorm   x2 = x (+ res)            (bf16 residual add, written when res)
//             rstd = 1 / sqrt(mean(x2^2) + eps)
//             y  = bf16(g * (x2 * rstd))
//   bwd       xh = x2 * rstd,  gy = g * dy
//             dx = bf16(dres + rstd * (gy - xh * mean(xh * gy)))   (g frozen: no dg)
//   RoPE      per head, pairs (i, i + D/2) ("rotate_half"), angle t * theta^(-2i/D):
//             (a, b) -> (a cos - b sin, b cos + a sin); bwd: the inverse rotation
//   SwiGLU    a = bf16(silu(gate) * up)
//   bwd       d_gate = bf16(da * up * silu'(gate)), d_up = bf16(da * silu(gate))
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "lora_kernels.h"

namespace lora_sm100 {

namespace {

__device__ __forceinline__ void unpack8(const uint4& u, float (&f)[8]) {
    const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        f[2 * i] = __uint_as_float(w[i] << 16);
        f[2 * i + 1] = __uint_as_float(w[i] & 0xFFFF0000u);
    }
}
__device__ __forceinline__ uint32_t pack2(float lo, float hi) {
    const __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
    return *reinterpret_cast<const uint32_t*>(&v);
}
__device__ __forceinline__ uint4 pack8(const float (&f)[8]) {
    return make_uint4(pack2(f[0], f[1]), pack2(f[2], f[3]), pack2(f[4], f[5]), pack2(f[6], f[7]));
}

constexpr int kRowThreads = 128;
constexpr int kMaxVec = 8;   // up to 8 x 16 bytes per thread: d <= 128 * 64 = 8192

// block-wide sum over 128 threads (fixed order: warp shuffles, then warp 0..3)
__device__ __forceinline__ float block_sum(float v, float* red) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int w = threadIdx.x >> 5;
    __syncthreads();
    if ((threadIdx.x & 31) == 0) red[w] = v;
    __syncthreads();
    return (red[0] + red[1]) + (red[2] + red[3]);
}

// one CTA of 128 threads per row; thread i owns 16-byte vectors i, i + 128, ...
// (NV of them: the register arrays are sized for the row, not for the largest d)
template <int NV>
__global__ void __launch_bounds__(kRowThreads) rmsnorm_fwd_kernel(const __nv_bfloat16* __restrict__ x,
                                                                  const __nv_bfloat16* __restrict__ res,
                                                                  const __nv_bfloat16* __restrict__ g, int64_t T,
                                                                  int d, float eps, __nv_bfloat16* __restrict__ y,
                                                                  __nv_bfloat16* __restrict__ x2_out,
                                                                  float* __restrict__ rstd_out) {
    __shared__ float red[4];
    const int64_t t = blockIdx.x;
    if (t >= T) return;
    const int nv = d / 8;
    float v[NV][8];
    float ss = 0.0f;
#pragma unroll
    for (int j = 0; j < NV; ++j) {
        const int c = threadIdx.x + j * kRowThreads;
        if (c >= nv) break;
        unpack8(*reinterpret_cast<const uint4*>(x + t * d + 8 * c), v[j]);
        if (res) {
            float rv[8];
            unpack8(*reinterpret_cast<const uint4*>(res + t * d + 8 * c), rv);
#pragma unroll
            for (int e = 0; e < 8; ++e) v[j][e] += rv[e];
            const uint4 o = pack8(v[j]);                 // the residual stream is bf16
            unpack8(o, v[j]);
            if (x2_out) *reinterpret_cast<uint4*>(x2_out + t * d + 8 * c) = o;
        }
#pragma unroll
        for (int e = 0; e < 8; ++e) ss = fmaf(v[j][e], v[j][e], ss);
    }
    const float rstd = rsqrtf(block_sum(ss, red) / static_cast<float>(d) + eps);
    if (threadIdx.x == 0 && rstd_out) rstd_out[t] = rstd;
#pragma unroll
    for (int j = 0; j < NV; ++j) {
        const int c = threadIdx.x + j * kRowThreads;
        if (c >= nv) break;
        float gv[8], o[8];
        unpack8(*reinterpret_cast<const uint4*>(g + 8 * c), gv);
#pragma unroll
        for (int e = 0; e < 8; ++e) o[e] = gv[e] * (v[j][e] * rstd);
        *reinterpret_cast<uint4*>(y + t * d + 8 * c) = pack8(o);
    }
}

template <int NV>
__global__ void __launch_bounds__(kRowThreads) rmsnorm_bwd_kernel(const __nv_bfloat16* __restrict__ dy,
                                                                  const __nv_bfloat16* __restrict__ x2,
                                                                  const __nv_bfloat16* __restrict__ g,
                                                                  const float* __restrict__ rstd_in,
                                                                  const __nv_bfloat16* __restrict__ dres, int64_t T,
                                                                  int d, __nv_bfloat16* __restrict__ dx) {
    __shared__ float red[4];
    const int64_t t = blockIdx.x;
    if (t >= T) return;
    const int nv = d / 8;
    const float rstd = rstd_in[t];
    float xh[NV][8], gy[NV][8];
    float dot = 0.0f;
#pragma unroll
    for (int j = 0; j < NV; ++j) {
        const int c = threadIdx.x + j * kRowThreads;
        if (c >= nv) break;
        float dv[8], gv[8];
        unpack8(*reinterpret_cast<const uint4*>(x2 + t * d + 8 * c), xh[j]);
        unpack8(*reinterpret_cast<const uint4*>(dy + t * d + 8 * c), dv);
        unpack8(*reinterpret_cast<const uint4*>(g + 8 * c), gv);
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            xh[j][e] *= rstd;
            gy[j][e] = gv[e] * dv[e];
            dot = fmaf(xh[j][e], gy[j][e], dot);
        }
    }
    const float mean = block_sum(dot, red) / static_cast<float>(d);
#pragma unroll
    for (int j = 0; j < NV; ++j) {
        const int c = threadIdx.x + j * kRowThreads;
        if (c >= nv) break;
        float o[8], rv[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
        if (dres) unpack8(*reinterpret_cast<const uint4*>(dres + t * d + 8 * c), rv);
#pragma unroll
        for (int e = 0; e < 8; ++e) o[e] = rv[e] + rstd * (gy[j][e] - xh[j][e] * mean);
        *reinterpret_cast<uint4*>(dx + t * d + 8 * c) = pack8(o);
    }
}

// RoPE in place on [T, heads * D] (row stride ld elements): thread -> (t, 8 pairs,
// a group of kRopeHeads heads) -- the angles depend on (t, pair) only, so each
// thread evaluates its 8 sincos once for kRopeHeads heads (sincosf per element
// measured compute-bound: 25 us per 32 MB call at 7B, T = 4096)
constexpr int kRopeHeads = 4;
__global__ void __launch_bounds__(256) rope_kernel(__nv_bfloat16* __restrict__ q, int64_t T, int heads, int D,
                                                   int64_t ld, int64_t pos0, float theta, float sign) {
    const int half = D / 2, pv = half / 8;   // 16-byte vectors per half-head
    const int hg = (heads + kRopeHeads - 1) / kRopeHeads;
    const int64_t total = T * hg * pv;
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    const float l2t = log2f(theta);
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < total; i += stride) {
        const int64_t t = i / (hg * pv);
        const int rem = static_cast<int>(i - t * hg * pv);
        const int g = rem / pv, v = rem - (rem / pv) * pv;
        const float pos = static_cast<float>(pos0 + t);
        float cs[8], sn[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            const int ii = 8 * v + e;                                      // pair index i < D / 2
            const float inv_freq = exp2f(-l2t * (2.0f * ii) / static_cast<float>(D));
            sincosf(pos * inv_freq, &sn[e], &cs[e]);
            sn[e] *= sign;
        }
        __nv_bfloat16* row = q + t * ld + 8 * v;
#pragma unroll
        for (int hh = 0; hh < kRopeHeads; ++hh) {
            const int h = g * kRopeHeads + hh;
            if (h >= heads) break;
            __nv_bfloat16* base = row + static_cast<int64_t>(h) * D;
            float a[8], b[8], oa[8], ob[8];
            unpack8(*reinterpret_cast<const uint4*>(base), a);
            unpack8(*reinterpret_cast<const uint4*>(base + half), b);
#pragma unroll
            for (int e = 0; e < 8; ++e) {
                oa[e] = a[e] * cs[e] - b[e] * sn[e];
                ob[e] = b[e] * cs[e] + a[e] * sn[e];
            }
            *reinterpret_cast<uint4*>(base) = pack8(oa);
            *reinterpret_cast<uint4*>(base + half) = pack8(ob);
        }
    }
}

__device__ __forceinline__ float sigmoidf(float x) { return 1.0f / (1.0f + __expf(-x)); }

__global__ void __launch_bounds__(256) swiglu_fwd_kernel(const __nv_bfloat16* __restrict__ gate,
                                                         const __nv_bfloat16* __restrict__ up, int64_t n8,
                                                         __nv_bfloat16* __restrict__ out) {
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n8; i += stride) {
        float gv[8], uv[8], o[8];
        unpack8(reinterpret_cast<const uint4*>(gate)[i], gv);
        unpack8(reinterpret_cast<const uint4*>(up)[i], uv);
#pragma unroll
        for (int e = 0; e < 8; ++e) o[e] = gv[e] * sigmoidf(gv[e]) * uv[e];
        reinterpret_cast<uint4*>(out)[i] = pack8(o);
    }
}

__global__ void __launch_bounds__(256) swiglu_bwd_kernel(const __nv_bfloat16* __restrict__ gate,
                                                         const __nv_bfloat16* __restrict__ up,
                                                         const __nv_bfloat16* __restrict__ da, int64_t n8,
                                                         __nv_bfloat16* __restrict__ dgate,
                                                         __nv_bfloat16* __restrict__ dup) {
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n8; i += stride) {
        float gv[8], uv[8], dv[8], dg[8], du[8];
        unpack8(reinterpret_cast<const uint4*>(gate)[i], gv);
        unpack8(reinterpret_cast<const uint4*>(up)[i], uv);
        unpack8(reinterpret_cast<const uint4*>(da)[i], dv);
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            const float sg = sigmoidf(gv[e]);
            const float silu = gv[e] * sg;
            du[e] = dv[e] * silu;
            dg[e] = dv[e] * uv[e] * (sg * (1.0f + gv[e] * (1.0f - sg)));
        }
        reinterpret_cast<uint4*>(dgate)[i] = pack8(dg);
        reinterpret_cast<uint4*>(dup)[i] = pack8(du);
    }
}

int grid_for(int64_t n, int num_sms) {
    const int64_t b = (n + 255) / 256;
    const int64_t cap = static_cast<int64_t>(num_sms) * 8;
    return static_cast<int>(b < cap ? (b > 0 ? b : 1) : cap);
}

}  // namespace

cudaError_t launch_rmsnorm_fwd(const __nv_bfloat16* x, const __nv_bfloat16* res, const __nv_bfloat16* g, int64_t T,
                               int d, float eps, __nv_bfloat16* y, __nv_bfloat16* x2_out, float* rstd,
                               cudaStream_t stream) {
    if (T <= 0) return cudaSuccess;
    if (d % 8 != 0 || d > kRowThreads * kMaxVec * 8) return cudaErrorInvalidValue;
    const int nv = (d / 8 + kRowThreads - 1) / kRowThreads;
    const unsigned grid = static_cast<unsigned>(T);
    if (nv <= 1) rmsnorm_fwd_kernel<1><<<grid, kRowThreads, 0, stream>>>(x, res, g, T, d, eps, y, x2_out, rstd);
    else if (nv <= 2) rmsnorm_fwd_kernel<2><<<grid, kRowThreads, 0, stream>>>(x, res, g, T, d, eps, y, x2_out, rstd);
    else if (nv <= 4) rmsnorm_fwd_kernel<4><<<grid, kRowThreads, 0, stream>>>(x, res, g, T, d, eps, y, x2_out, rstd);
    else rmsnorm_fwd_kernel<8><<<grid, kRowThreads, 0, stream>>>(x, res, g, T, d, eps, y, x2_out, rstd);
    return cudaGetLastError();
}

cudaError_t launch_rmsnorm_bwd(const __nv_bfloat16* dy, const __nv_bfloat16* x2, const __nv_bfloat16* g,
                               const float* rstd, const __nv_bfloat16* dres, int64_t T, int d, __nv_bfloat16* dx,
                               cudaStream_t stream) {
    if (T <= 0) return cudaSuccess;
    if (d % 8 != 0 || d > kRowThreads * kMaxVec * 8) return cudaErrorInvalidValue;
    const int nv = (d / 8 + kRowThreads - 1) / kRowThreads;
    const unsigned grid = static_cast<unsigned>(T);
    if (nv <= 1) rmsnorm_bwd_kernel<1><<<grid, kRowThreads, 0, stream>>>(dy, x2, g, rstd, dres, T, d, dx);
    else if (nv <= 2) rmsnorm_bwd_kernel<2><<<grid, kRowThreads, 0, stream>>>(dy, x2, g, rstd, dres, T, d, dx);
    else if (nv <= 4) rmsnorm_bwd_kernel<4><<<grid, kRowThreads, 0, stream>>>(dy, x2, g, rstd, dres, T, d, dx);
    else rmsnorm_bwd_kernel<8><<<grid, kRowThreads, 0, stream>>>(dy, x2, g, rstd, dres, T, d, dx);
    return cudaGetLastError();
}

cudaError_t launch_rope(__nv_bfloat16* q, int64_t T, int heads, int D, int64_t ld, int64_t pos0, float theta,
                        int inverse, int num_sms, cudaStream_t stream) {
    if (T <= 0 || heads <= 0) return cudaSuccess;
    if (D % 16 != 0) return cudaErrorInvalidValue;
    rope_kernel<<<grid_for(T * ((heads + kRopeHeads - 1) / kRopeHeads) * (D / 16), num_sms), 256, 0, stream>>>(
        q, T, heads, D, ld, pos0, theta, inverse ? -1.0f : 1.0f);
    return cudaGetLastError();
}

cudaError_t launch_swiglu_fwd(const __nv_bfloat16* gate, const __nv_bfloat16* up, int64_t count, __nv_bfloat16* out,
                              int num_sms, cudaStream_t stream) {
    if (count <= 0) return cudaSuccess;
    if (count % 8 != 0) return cudaErrorInvalidValue;
    swiglu_fwd_kernel<<<grid_for(count / 8, num_sms), 256, 0, stream>>>(gate, up, count / 8, out);
    return cudaGetLastError();
}

cudaError_t launch_swiglu_bwd(const __nv_bfloat16* gate, const __nv_bfloat16* up, const __nv_bfloat16* da,
                              int64_t count, __nv_bfloat16* dgate, __nv_bfloat16* dup, int num_sms,
                              cudaStream_t stream) {
    if (count <= 0) return cudaSuccess;
    if (count % 8 != 0) return cudaErrorInvalidValue;
    swiglu_bwd_kernel<<<grid_for(count / 8, num_sms), 256, 0, stream>>>(gate, up, da, count / 8, dgate, dup);
    return cudaGetLastError();
}

}  // namespace lora_sm100

// ============================================================ C ABI
#include "lora_internal.h"

using namespace lora_host;

namespace {
bool al16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }
int sms_now() {
    int dev = 0, sms = 148;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return sms;
}
lora_status launched(cudaError_t e, const char* what) {
    if (e == cudaErrorInvalidValue) return fail(LORA_ERR_SHAPE, "%s: unsupported shape", what);
    if (e != cudaSuccess) return cuda_fail(e, what);
    set_launches(1);
    return LORA_OK;
}
}  // namespace

extern "C" {

lora_status lora_rmsnorm_fwd(int64_t tokens, int64_t dim, float eps, const void* x, const void* res, const void* g,
                             void* y, void* x2_out, float* rstd, void* stream) {
    set_launches(0);
    if (tokens < 0 || dim < 8 || dim % 8 || dim > 8192)
        return fail(LORA_ERR_SHAPE, "lora_rmsnorm_fwd: tokens %lld, dim %lld (dim %% 8 == 0, 8..8192)",
                    static_cast<long long>(tokens), static_cast<long long>(dim));
    if (!x || !g || !y || !rstd || (x2_out && !res))
        return fail(LORA_ERR_INVALID, "lora_rmsnorm_fwd: x, g, y, rstd must be non-NULL (x2_out needs res)");
    const void* ps[] = {x, res, g, y, x2_out};
    for (const void* p : ps)
        if (p && !al16(p)) return fail(LORA_ERR_ALIGN, "lora_rmsnorm_fwd: %p is not 16-byte aligned", p);
    return launched(lora_sm100::launch_rmsnorm_fwd(
                        static_cast<const __nv_bfloat16*>(x), static_cast<const __nv_bfloat16*>(res),
                        static_cast<const __nv_bfloat16*>(g), tokens, static_cast<int>(dim), eps,
                        static_cast<__nv_bfloat16*>(y), static_cast<__nv_bfloat16*>(x2_out), rstd,
                        static_cast<cudaStream_t>(stream)),
                    "lora_rmsnorm_fwd");
}

lora_status lora_rmsnorm_bwd(int64_t tokens, int64_t dim, const void* dy, const void* x2, const void* g,
                             const float* rstd, const void* dres, void* dx, void* stream) {
    set_launches(0);
    if (tokens < 0 || dim < 8 || dim % 8 || dim > 8192)
        return fail(LORA_ERR_SHAPE, "lora_rmsnorm_bwd: tokens %lld, dim %lld (dim %% 8 == 0, 8..8192)",
                    static_cast<long long>(tokens), static_cast<long long>(dim));
    if (!dy || !x2 || !g || !rstd || !dx) return fail(LORA_ERR_INVALID, "lora_rmsnorm_bwd: NULL argument");
    const void* ps[] = {dy, x2, g, dres, dx};
    for (const void* p : ps)
        if (p && !al16(p)) return fail(LORA_ERR_ALIGN, "lora_rmsnorm_bwd: %p is not 16-byte aligned", p);
    return launched(lora_sm100::launch_rmsnorm_bwd(
                        static_cast<const __nv_bfloat16*>(dy), static_cast<const __nv_bfloat16*>(x2),
                        static_cast<const __nv_bfloat16*>(g), rstd, static_cast<const __nv_bfloat16*>(dres), tokens,
                        static_cast<int>(dim), static_cast<__nv_bfloat16*>(dx), static_cast<cudaStream_t>(stream)),
                    "lora_rmsnorm_bwd");
}

lora_status lora_rope(int64_t tokens, int heads, int head_dim, int64_t ld, int64_t pos0, float theta, int inverse,
                      void* q, void* stream) {
    set_launches(0);
    if (tokens < 0 || heads < 0 || head_dim < 16 || head_dim % 16 || ld < int64_t(heads) * head_dim || ld % 8)
        return fail(LORA_ERR_SHAPE, "lora_rope: heads %d, head_dim %d (multiple of 16), ld %lld", heads, head_dim,
                    static_cast<long long>(ld));
    if (!q && tokens * heads > 0) return fail(LORA_ERR_INVALID, "lora_rope: q is NULL");
    if (q && !al16(q)) return fail(LORA_ERR_ALIGN, "lora_rope: q is not 16-byte aligned");
    return launched(lora_sm100::launch_rope(static_cast<__nv_bfloat16*>(q), tokens, heads, head_dim, ld, pos0, theta,
                                            inverse, sms_now(), static_cast<cudaStream_t>(stream)),
                    "lora_rope");
}

lora_status lora_swiglu_fwd(int64_t count, const void* gate, const void* up, void* out, void* stream) {
    set_launches(0);
    if (count < 0 || count % 8) return fail(LORA_ERR_SHAPE, "lora_swiglu_fwd: count %% 8 != 0");
    if (count && (!gate || !up || !out)) return fail(LORA_ERR_INVALID, "lora_swiglu_fwd: NULL argument");
    if (count && (!al16(gate) || !al16(up) || !al16(out)))
        return fail(LORA_ERR_ALIGN, "lora_swiglu_fwd: pointers must be 16-byte aligned");
    return launched(lora_sm100::launch_swiglu_fwd(static_cast<const __nv_bfloat16*>(gate),
                                                  static_cast<const __nv_bfloat16*>(up), count,
                                                  static_cast<__nv_bfloat16*>(out), sms_now(),
                                                  static_cast<cudaStream_t>(stream)),
                    "lora_swiglu_fwd");
}

lora_status lora_swiglu_bwd(int64_t count, const void* gate, const void* up, const void* da, void* dgate, void* dup,
                            void* stream) {
    set_launches(0);
    if (count < 0 || count % 8) return fail(LORA_ERR_SHAPE, "lora_swiglu_bwd: count %% 8 != 0");
    if (count && (!gate || !up || !da || !dgate || !dup)) return fail(LORA_ERR_INVALID, "lora_swiglu_bwd: NULL argument");
    const void* ps[] = {gate, up, da, dgate, dup};
    for (const void* p : ps)
        if (count && !al16(p)) return fail(LORA_ERR_ALIGN, "lora_swiglu_bwd: pointers must be 16-byte aligned");
    return launched(lora_sm100::launch_swiglu_bwd(
                        static_cast<const __nv_bfloat16*>(gate), static_cast<const __nv_bfloat16*>(up),
                        static_cast<const __nv_bfloat16*>(da), count, static_cast<__nv_bfloat16*>(dgate),
                        static_cast<__nv_bfloat16*>(dup), sms_now(), static_cast<cudaStream_t>(stream)),
                    "lora_swiglu_bwd");
}

}  // extern "C"

extern "C" lora_status lora_sum_bf16(int64_t count, int n, const void* const* srcs, void* dst, void* stream) {
    set_launches(0);
    if (count < 0 || count % 8 || n < 1 || n > lora_sm100::kMaxGroup)
        return fail(LORA_ERR_SHAPE, "lora_sum_bf16: count %% 8 == 0 and 1 <= n <= %d", lora_sm100::kMaxGroup);
    if (count == 0) return LORA_OK;
    if (!srcs || !dst) return fail(LORA_ERR_INVALID, "lora_sum_bf16: NULL argument");
    lora_sm100::SumBf16Args A;
    A.n = n;
    A.count = count;
    A.dst = static_cast<__nv_bfloat16*>(dst);
    if (!al16(dst)) return fail(LORA_ERR_ALIGN, "lora_sum_bf16: dst is not 16-byte aligned");
    for (int i = 0; i < n; ++i) {
        if (!srcs[i] || !al16(srcs[i])) return fail(LORA_ERR_ALIGN, "lora_sum_bf16: source %d NULL or unaligned", i);
        A.src[i] = static_cast<const __nv_bfloat16*>(srcs[i]);
    }
    return launched(lora_sm100::launch_sum_bf16(A, sms_now(), static_cast<cudaStream_t>(stream)), "lora_sum_bf16");
}
