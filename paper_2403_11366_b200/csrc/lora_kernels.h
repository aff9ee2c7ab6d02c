// lora_kernels.h -- internal interface between the C-ABI host layer
// (lora_api.cpp) and the sm_100a kernels.  Not part of the public ABI.
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace lora_sm100 {

enum : int { kModeFwd = 0, kModeDx = 1 };

struct FusedGemmParams {
    int64_t T;                    // token rows
    int64_t K;                    // reduction extent (n fwd, m dx)
    int64_t N_out;                // output columns (m fwd, n dx)
    int r;                        // LoRA rank
    float scale;                  // s = alpha / r
    const __nv_bfloat16* bias;    // fwd only; may be null
    __nv_bfloat16* out;           // y or dx, [T, N_out]
    float* side_out;              // fwd: h [T, r] (unscaled); dx: gh [T, r] = s dY B; may be null
};

struct FusedGemmMaps {
    CUtensorMap act, w, nar, tail;
};

// K1 / K2.  r_pad in {16, 32, 64}; tiles are 128 x (256 - r_pad).
int fused_gemm_block_n(int r_pad);
cudaError_t launch_fused_gemm(int mode, int r_pad, const FusedGemmMaps& maps,
                              const FusedGemmParams& p, int num_sms, cudaStream_t stream);

// B6: adapter pack.  Any output pointer may be null (skipped).
//   bpad [m, r_pad] = B zero-padded      (fwd tail operand, K-major)
//   bt   [r, m]     = B^T                (dx narrow operand, K-major)
//   at   [n, r_pad] = A^T zero-padded    (dx tail operand, K-major)
cudaError_t launch_pack(const __nv_bfloat16* a, const __nv_bfloat16* b, int64_t n, int64_t m,
                        int r, int r_pad, __nv_bfloat16* bpad, __nv_bfloat16* bt,
                        __nv_bfloat16* at, int num_sms, cudaStream_t stream);

// K3: dA = gh^T x, dB = s dY^T h.  Column-strip partial sums over token
// chunks (fixed order) + a finalize pass; deterministic.
struct GradReducePlan {
    int r_bucket;        // register tile rank (4, 8, 16, 32, 64)
    int cols_per_strip;  // 32 * columns-per-thread
    int strips_a, strips_b;
    int chunks;          // token chunks
    int rows_per_chunk;
};
GradReducePlan plan_grad_reduce(int64_t T, int64_t n, int64_t m, int r, int num_sms);
size_t grad_reduce_partial_bytes(const GradReducePlan& pl, int64_t n, int64_t m, int r);
cudaError_t launch_grad_reduce(const GradReducePlan& pl, int64_t T, int64_t n, int64_t m, int r,
                               float scale, const __nv_bfloat16* x, const float* gh,
                               const __nv_bfloat16* dy, const float* h, float* partials,
                               float* da, float* db, int accumulate, cudaStream_t stream,
                               int* launches);

// K3a: out[t, j] = scale * sum_k X[t, k] P[j, k]   (h when not saved; gh when dx is skipped)
cudaError_t launch_rowproj(const __nv_bfloat16* X, int64_t T, int64_t K, const __nv_bfloat16* P,
                           int r, float scale, float* out, cudaStream_t stream);

// K4: w_out = bf16(W0 + s * B A)
cudaError_t launch_merge(const __nv_bfloat16* w0, const __nv_bfloat16* a, const __nv_bfloat16* b,
                         int64_t n, int64_t m, int r, float scale, __nv_bfloat16* w_out,
                         cudaStream_t stream);

// dst += src (fp32), used by the TP backward when accumulating reduced grads
cudaError_t launch_add_f32(float* dst, const float* src, int64_t count, cudaStream_t stream);

// zero-fill helper for degenerate (T == 0) gradients
cudaError_t launch_fill_zero(float* p, int64_t count, cudaStream_t stream);

}  // namespace lora_sm100
