// lora_dropout.cu -- LoRA dropout (Listing 3 LORA_DROPOUT = 0.05, PAPER.md:82;
// DESIGN.md reading R7: inverted dropout on the adapter input only; the
// frozen path W0 x never sees it).  With keep mask M and q = 1 / (1 - p):
//   h   = q (M . x) A^T                     (K0, replaces K1's in-MMA h)
//   dX  = G W0 + q M . (gh A)               (K2 dropout mode, lora_gemm.cu)
//   dA  = q gh^T (M . x)                    (K3 on xm = M . x)
// K0 here, for a group of linears sharing x (each its own mask), x read once:
// the forward's h of every member (masked products on mma.sync, one launch) --
// which also writes M . x and the packed keep bits when the caller keeps them
// (lora_dropout.masked_x / keep_bits) -- and, for a backward without them, the
// masked input xm = M . x in bf16 (exact: zeroing only) plus the keep bits the dX
// epilogue reads (one streaming launch).  Keep bits drawn from Philox with the
// round keys prepared on the host (lora_philox.cuh).
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>

#include "lora_kernels.h"
#include "lora_philox.cuh"

namespace lora_sm100 {

typedef __nv_bfloat16 bf16;

namespace {

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


// ------------------------------------------------------------------ K0 (grouped)
// Forward K0 of a group of linears sharing x: h_g = q_g (M_g . x) A_g^T for every
// member g, x streamed from HBM once.  The masked products run on the tensor
// cores (mma.sync m16n8k16, bf16 in, fp32 accumulate): one warp = 16 token rows
// x a k range; lane (g4 = lane / 4, c4 = lane % 4) loads x[row][k0 + 8 c4 .. + 7]
// of rows g4 and g4 + 8 (16-byte loads, the 8 columns of one Philox block), so
// each lane draws exactly its own two Philox blocks per 32 columns.  Within a
// 32-column step the columns are permuted consistently for x and A (MMA 1 takes
// columns 8 c4 + 0..3, MMA 2 columns 8 c4 + 4..7 of every lane): the same dot
// products, no shuffles.  The warps of a CTA split n; their fp32 partials are
// summed in warp order through shared memory (deterministic), then scaled by q.
// NT = n8 tiles per member (r8 / 8); at most MPC <= 8 / NT members per launch
// (the launcher splits larger groups), indexed statically so that the Philox
// round keys are constant operands.
template <int NT, int MPC>   // MPC: members per launch (MPC * NT <= 8)
__global__ void __launch_bounds__(512) dropout_h_group_kernel(const __grid_constant__ DropoutGroup G) {
    extern __shared__ float red[];       // [warps][16][MPC * NT * 8]
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int W = blockDim.x >> 5;
    const int g4 = lane >> 2, c4 = lane & 3;
    const int mcount = G.count;
    const int64_t t0 = static_cast<int64_t>(blockIdx.x) * 16;
    const int64_t rA = t0 + g4, rB = t0 + g4 + 8;
    const int64_t n = G.n;
    const int64_t kc = (n + 32 * W - 1) / (32 * W) * 32;   // columns per warp, multiple of 32
    const int64_t k_lo = warp * kc, k_hi = k_lo + kc < n ? k_lo + kc : n;
    float acc[MPC * NT][4];
#pragma unroll
    for (int s = 0; s < MPC * NT; ++s) acc[s][0] = acc[s][1] = acc[s][2] = acc[s][3] = 0.0f;
    const bf16* xa = G.x + rA * n;
    const bf16* xb = G.x + rB * n;
    const bool okA = rA < G.T, okB = rB < G.T;
    constexpr int U = 4;   // 32-column steps whose x loads are in flight together
    for (int64_t kb = k_lo; kb < k_hi; kb += 32 * U) {
        uint4 ua[U], ub[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t k = kb + 32 * u + 8 * c4;
            ua[u] = ub[u] = make_uint4(0, 0, 0, 0);
            if (k < k_hi && okA) ua[u] = __ldg(reinterpret_cast<const uint4*>(xa + k));
            if (k < k_hi && okB) ub[u] = __ldg(reinterpret_cast<const uint4*>(xb + k));
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t k = kb + 32 * u + 8 * c4;
            if (kb + 32 * u >= k_hi) break;   // (warp-uniform)
            const bool kok = k < k_hi;
            const uint32_t k8 = static_cast<uint32_t>(k / 8);
#pragma unroll
            for (int mi = 0; mi < MPC; ++mi) {
                if (mi >= mcount) break;
                const DropoutMember& M = G.m[mi];
                uint32_t wa[4], wb[4];
                const uint4 xa4 = masked8(ua[u], M.keys, k8, static_cast<uint32_t>(rA), wa);
                const uint4 xb4 = masked8(ub[u], M.keys, k8, static_cast<uint32_t>(rB), wb);
                if (M.xm && kok) {   // M . x for the backward's dA (lora_dropout.masked_x)
                    if (okA) *reinterpret_cast<uint4*>(M.xm + rA * n + k) = xa4;
                    if (okB) *reinterpret_cast<uint4*>(M.xm + rB * n + k) = xb4;
                }
                if (M.bits) {   // keep the mask for the backward (lora_dropout.keep_bits)
                    // the quad's four lanes hold the 32 columns of this step: one word per row
                    uint32_t ba = kok ? keep8_of(wa) << (8 * c4) : 0u, bb = kok ? keep8_of(wb) << (8 * c4) : 0u;
                    ba |= __shfl_xor_sync(0xffffffffu, ba, 1);
                    bb |= __shfl_xor_sync(0xffffffffu, bb, 1);
                    ba |= __shfl_xor_sync(0xffffffffu, ba, 2);
                    bb |= __shfl_xor_sync(0xffffffffu, bb, 2);
                    const int64_t nw = (n + 31) / 32, wcol = (kb + 32 * u) / 32;
                    if (c4 == 0 && okA) M.bits[rA * nw + wcol] = ba;
                    if (c4 == 1 && okB) M.bits[rB * nw + wcol] = bb;
                }
#pragma unroll
                for (int nt = 0; nt < NT; ++nt) {
                    const int j = nt * 8 + g4;
                    uint4 bw = make_uint4(0, 0, 0, 0);
                    if (kok && j < M.r)
                        bw = __ldg(reinterpret_cast<const uint4*>(M.a + static_cast<int64_t>(j) * n + k));
                    mma_bf16_16816(acc[mi * NT + nt], xa4.x, xb4.x, xa4.y, xb4.y, bw.x, bw.y);
                    mma_bf16_16816(acc[mi * NT + nt], xa4.z, xb4.z, xa4.w, xb4.w, bw.z, bw.w);
                }
            }
        }
    }
    // partials -> shared memory: red[warp][row][member * NT * 8 + column]
    constexpr int RC = MPC * NT * 8;
    float* mine = red + warp * 16 * RC;
#pragma unroll
    for (int s = 0; s < MPC * NT; ++s) {
        const int col = s * 8 + 2 * c4;
        mine[g4 * RC + col] = acc[s][0];
        mine[g4 * RC + col + 1] = acc[s][1];
        mine[(g4 + 8) * RC + col] = acc[s][2];
        mine[(g4 + 8) * RC + col + 1] = acc[s][3];
    }
    __syncthreads();
    for (int e = threadIdx.x; e < 16 * RC; e += blockDim.x) {
        const int row = e / RC, col = e - row * RC;
        const int mi = col / (NT * 8), j = col - mi * NT * 8;
        if (mi >= mcount) continue;
        const DropoutMember& M = G.m[mi];
        const int64_t t = t0 + row;
        if (j >= M.r || t >= G.T || M.h == nullptr) continue;
        float v = red[e];
        for (int w = 1; w < W; ++w) v += red[w * 16 * RC + e];
        M.h[t * M.r + j] = M.drop.q * v;
    }
}

// Backward K0 of a group sharing x: for every member g, xm_g = M_g . x (bf16,
// exact) and the packed keep bits (the dX epilogue's), x streamed once.  One
// lane = 8 consecutive columns (one 16-byte load, one Philox block per member);
// a warp covers 256 consecutive columns of a row.  Members' outputs may be null.
__global__ void __launch_bounds__(256) dropout_apply_group_kernel(const __grid_constant__ DropoutGroup G) {
    const int lane = threadIdx.x & 31;
    const uint32_t n8 = static_cast<uint32_t>(G.n / 8);   // (n % 8 == 0)
    const uint32_t warps_per_row = (n8 + 31) / 32;
    const int64_t nw = (G.n + 31) / 32;
    const int64_t total = G.T * warps_per_row;
    const int64_t gw = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int64_t stride = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
    for (int64_t wi = gw; wi < total; wi += stride) {
        const int64_t t = wi / warps_per_row;
        const uint32_t k8 = static_cast<uint32_t>(wi - t * warps_per_row) * 32 + lane;
        const bool ok = k8 < n8;
        uint4 u = make_uint4(0, 0, 0, 0);
        if (ok) u = __ldg(reinterpret_cast<const uint4*>(G.x + t * G.n + 8 * static_cast<int64_t>(k8)));
#pragma unroll
        for (int mi = 0; mi < kMaxGroup; ++mi) {
            if (mi >= G.count) break;
            const DropoutMember& M = G.m[mi];
            uint4 xm;
            uint32_t keep;
            if (M.bits_in) {   // the forward's keep bits: nothing drawn
                keep = ok ? (M.bits_in[t * nw + k8 / 4] >> (8 * (k8 & 3))) & 0xFFu : 0u;
                xm = masked8_bits(u, keep);
            } else {
                uint32_t w[4];
                xm = masked8(u, M.keys, k8, static_cast<uint32_t>(t), w);
                keep = ok ? keep8_of(w) : 0u;
            }
            if (M.bits) {
                uint32_t b = keep << (8 * (lane & 3));
                b |= __shfl_xor_sync(0xffffffffu, b, 1);
                b |= __shfl_xor_sync(0xffffffffu, b, 2);
                if ((lane & 3) == 0 && ok) M.bits[t * nw + k8 / 4] = b;
            }
            if (M.xm && ok) *reinterpret_cast<uint4*>(M.xm + t * G.n + 8 * static_cast<int64_t>(k8)) = xm;
        }
    }
}

}  // namespace

// K0 of a group of linears sharing x: the forward products (h) in one
// tensor-core launch, the backward's masked input and keep bits in one
// streaming launch; x is read once per launch for all members.
static PhiloxKeys philox_keys(const DropoutParams& d) {
    PhiloxKeys K;
    uint32_t k0 = static_cast<uint32_t>(d.seed), k1 = static_cast<uint32_t>(d.seed >> 32);
    for (int r = 0; r < 10; ++r) {
        K.k0[r] = k0;
        K.k1[r] = k1;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    K.c2 = static_cast<uint32_t>(d.offset);
    K.c3 = static_cast<uint32_t>(d.offset >> 32);
    K.thr2 = d.thr | (d.thr << 16);
    K.k8_base = static_cast<uint32_t>(d.col0 / 8);
    K.t_base = static_cast<uint32_t>(d.row0);
    return K;
}

template <int NT, int MPC>
static cudaError_t launch_h_chunk(const DropoutGroup& C, int num_sms, cudaStream_t stream) {
    // warps per CTA: 16 while the token groups alone leave SMs idle, else 8
    const int64_t groups = (C.T + 15) / 16;
    const int W = groups < 2LL * num_sms ? 16 : 8;   // (32 warps at 64 registers measured slower)
    const size_t smem = static_cast<size_t>(W) * 16 * MPC * NT * 8 * sizeof(float);
    static bool attr_set = false;
    if (!attr_set) {
        cudaError_t e = cudaFuncSetAttribute(dropout_h_group_kernel<NT, MPC>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, 128 * 1024);
        if (e != cudaSuccess) return e;
        attr_set = true;
    }
    dropout_h_group_kernel<NT, MPC><<<static_cast<unsigned>(groups), 32 * W, smem, stream>>>(C);
    return cudaGetLastError();
}

template <int NT>
static cudaError_t launch_h_group(const DropoutGroup& G, int num_sms, cudaStream_t stream, int* launches) {
    constexpr int MAXM = 8 / NT;
    for (int m0 = 0; m0 < G.count; m0 += MAXM) {   // at most MAXM members per launch
        DropoutGroup C = G;
        C.count = G.count - m0 < MAXM ? G.count - m0 : MAXM;
        for (int i = 0; i < C.count; ++i) C.m[i] = G.m[m0 + i];
        cudaError_t e;
        if (C.count == 1) e = launch_h_chunk<NT, 1>(C, num_sms, stream);
        else if (C.count == 2 && MAXM >= 2) e = launch_h_chunk<NT, (MAXM >= 2 ? 2 : 1)>(C, num_sms, stream);
        else if (C.count <= 4 && MAXM >= 4) e = launch_h_chunk<NT, (MAXM >= 4 ? 4 : 1)>(C, num_sms, stream);
        else e = launch_h_chunk<NT, MAXM>(C, num_sms, stream);
        if (e != cudaSuccess) return e;
        ++*launches;
    }
    return cudaSuccess;
}

cudaError_t launch_dropout_input_group(const DropoutGroup& G0, int num_sms, cudaStream_t stream, int* launches) {
    if (G0.count < 1 || G0.T <= 0) return cudaSuccess;
    DropoutGroup G = G0;
    bool need_h = false, need_apply = false;
    int rmax = 1;
    for (int g = 0; g < G.count; ++g) {
        G.m[g].keys = philox_keys(G.m[g].drop);
        need_h = need_h || G.m[g].h != nullptr;
        // (keep bits / masked input with h: the h kernel writes them, unless the apply
        // kernel runs anyway)
        need_apply = need_apply || (G.m[g].h == nullptr && (G.m[g].xm != nullptr || G.m[g].bits != nullptr));
        rmax = G.m[g].r > rmax ? G.m[g].r : rmax;
    }
    cudaError_t e = cudaSuccess;
    if (need_h) {
        DropoutGroup H = G;   // (keep bits and M . x, when wanted, come from the apply kernel below)
        if (need_apply)
            for (int g = 0; g < H.count; ++g) {
                H.m[g].bits = nullptr;
                H.m[g].xm = nullptr;
            }
        if (rmax <= 8) e = launch_h_group<1>(H, num_sms, stream, launches);
        else if (rmax <= 16) e = launch_h_group<2>(H, num_sms, stream, launches);
        else if (rmax <= 32) e = launch_h_group<4>(H, num_sms, stream, launches);
        else e = launch_h_group<8>(H, num_sms, stream, launches);
        if (e != cudaSuccess) return e;
    }
    if (need_apply) {
        const int64_t warps = G.T * ((G.n / 8 + 31) / 32);
        int64_t blocks = (warps + 7) / 8;
        const int64_t cap = static_cast<int64_t>(num_sms) * 8;
        blocks = blocks < cap ? blocks : cap;
        dropout_apply_group_kernel<<<static_cast<unsigned>(blocks), 256, 0, stream>>>(G);
        e = cudaGetLastError();
        ++*launches;
    }
    return e;
}

cudaError_t launch_dropout_mask(int64_t T, int64_t n, const DropoutParams& d, uint8_t* mask, int num_sms,
                                cudaStream_t stream) {
    if (T <= 0) return cudaSuccess;
    dropout_mask_kernel<<<num_sms * 4, 256, 0, stream>>>(T, n, d, mask);
    return cudaGetLastError();
}

}  // namespace lora_sm100
