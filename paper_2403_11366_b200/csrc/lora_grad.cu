// lora_grad.cu -- the CUDA-core K3 (kept as the comparison baseline for the
// tensor-core K3 of lora_grad_mma.cu; selected with LORA_K3=cluster) and B6.
// K3 computes the two trainable gradients of the LoRA linear (PAPER.md:111,
// "B and A are the trainable weights"):
//     dA[j, k] = sum_t gh[t, j] x[t, k]          gh = s dY B   (from K2)
//     dB[i, j] = s sum_t dY[t, i] h[t, j]        h  = x A^T    (from K1)
// as rank-r FMA reductions over all T tokens: column blocks of 32*CPT columns
// with the tokens split over a cluster of 8 CTAs and a DSMEM reduction in rank
// order (deterministic).  At 2r FMAs per activation byte this is FMA-bound on
// the CUDA cores once r >= 16 -- the reason the default K3 runs on tcgen05.
// B6: the adapter pack (B zero-padded to 8 columns, or B^T).
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
                              bf16* __restrict__ bt, const float* __restrict__ coef, bf16* __restrict__ cs,
                              int64_t T, int64_t t_pad) {
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    const int64_t t0 = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const bf16 zero = __float2bfloat16(0.0f);
    if (coef)   // K3's exact hi / mid / lo split of coef [T, r] (r == r8): cs [3 r8, t_pad]
        for (int64_t idx = t0; idx < T * r; idx += stride) {
            const int64_t t = idx / r;
            const int k = static_cast<int>(idx - t * r);
            const float v = coef[idx];
            const bf16 hi = __float2bfloat16_rn(v);
            const float r0 = v - __bfloat162float(hi);
            const bf16 md = __float2bfloat16_rn(r0);
            cs[static_cast<int64_t>(k) * t_pad + t] = hi;
            cs[static_cast<int64_t>(r8 + k) * t_pad + t] = md;
            cs[static_cast<int64_t>(2 * r8 + k) * t_pad + t] = __float2bfloat16_rn(r0 - __bfloat162float(md));
        }
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

cudaError_t launch_pack_b(const bf16* b, int64_t m, int r, bf16* b8, bf16* bt, int num_sms, cudaStream_t stream,
                          const float* coef, bf16* cs, int64_t T, int64_t t_pad) {
    const int r8 = (r + 7) / 8 * 8;
    if (coef && r != r8) return cudaErrorInvalidValue;   // no pad rows are written
    const int64_t work = std::max<int64_t>(m * r8, coef ? T * r : 0);
    const int blocks = static_cast<int>(std::min<int64_t>((work + 255) / 256, 4LL * num_sms));
    pack_b_kernel<<<blocks, 256, 0, stream>>>(b, m, r, r8, b8, bt, coef, cs, T, t_pad);
    return cudaGetLastError();
}

// ------------------------------------------------------------------ K3

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
                *d = (g.accumulate & kAccA) ? *d + sum : sum;
            } else {
                const float val = g.scale_b * sum;
                float* d = g.db + (cb0 + col) * r + j;
                *d = (g.accumulate & kAccB) ? *d + val : val;
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

// (lazy loading: see preload_gemm_kernels in lora_gemm.cu)
cudaError_t preload_grad_kernels() {
    cudaFuncAttributes a;
    return cudaFuncGetAttributes(&a, (const void*)pack_b_kernel);
}

}  // namespace lora_sm100
