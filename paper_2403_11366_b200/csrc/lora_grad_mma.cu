// lora_grad_mma.cu -- K3 on the tensor cores: the two trainable gradients of
// the LoRA linear ("B and A are the trainable weights"),
//     dA^T[k, j] = sum_t x[t, k]  gh[t, j]       gh = s dY B   (from K2)
//     dB  [i, j] = s sum_t dY[t, i] h[t, j]       h  = x A^T    (from K1)
// Both have the same shape: O[c, q] = scale * sum_t X[t, c] C[t, q] with X a
// bf16 activation [T, N] (x or dY) and C an fp32 coefficient matrix [T, r].
// At 2 r FMAs per activation byte they are FMA-bound on the CUDA cores once
// r >= 16 (2 T r (n + m) FMAs vs 148 SMs x 128 FMA/clk), but tiny for the
// tensor cores; on tcgen05 the kernel is bound by reading X from HBM once.
//
// K3s (split pre-pass): Cs [3 r8, T_pad] bf16 = the fp32 coefficients as
//   three bf16 rows hi + mid + lo (8 + 8 + 8 significand bits: C is
//   represented exactly, so every tensor-core product is exact and only the
//   fp32 accumulation rounds, as on the CUDA cores), token-contiguous, i.e.
//   the K-major B operand of the MMA below.  Done once per coefficient
//   matrix instead of once per column tile.
// K3 (one CTA = kGradMmaCols = 128 X columns x one token slice; 256 = two M tiles
// sharing Cs is a compile-time option, measured slower: half the CTAs):
//   MMA   D[c, q] += X^T[c, t] Cs[q, t]     M = 128 columns (two MMAs sharing the Cs
//         operand per k-step), N = q_pad, K = 16.
//         A operand = the X tile exactly as TMA lands it ([64 tokens][64
//         columns] SWIZZLE_128B boxes, read MN-major: no transpose pass).
//         Several coefficient SETS sharing one X (dA of q/k/v all read x) are
//         stacked along N, so x is read once for all of them.
//   split when there are too few column tiles to fill the GPU the tokens are
//         split over a cluster of S CTAs; each CTA drains its TMEM partial
//         into shared memory and the cluster sums the S partials over DSMEM
//         in rank order: deterministic, no atomics, no global partial buffer.
//         With S = 1 the epilogue stores straight from TMEM.
// Warp roles (192 threads): warp 0 TMA producer, warp 1 MMA issuer + TMEM
// owner, warps 2..5 epilogue (one TMEM lane quarter each); all six reduce.
#include <cooperative_groups.h>
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>

#include "lora_kernels.h"
#include "sm100_ptx.cuh"

namespace lora_sm100 {

namespace {

constexpr int KB = 64;              // tokens per k-block (one 128-byte SW128 row of Cs)
constexpr int MT = kGradMmaCols / 128;   // M = 128 MMAs per k-step (one per 128 X columns)
constexpr int X_BOX = 64 * KB * 2;       // one [64 tokens][64 columns] bf16 box = 8 KiB
constexpr int X_BYTES = 2 * MT * X_BOX;  // kGradMmaCols columns per CTA
constexpr int ACC_STRIDE = 256;          // TMEM columns between the MT accumulators
constexpr int THREADS = 192;
constexpr int PA = kGradMmaCols + 4;   // dA partial row stride (floats)
constexpr int SMEM_CTA_MAX = 227 * 1024;
constexpr int SMEM_SM = 228 * 1024;
constexpr int MAX_STAGES = 8;

__device__ __forceinline__ void tmem_ld_32x32b_x8(uint32_t taddr, uint32_t (&v)[8]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
                   "=r"(v[7])
                 : "r"(taddr));
}
__device__ __forceinline__ void tmem_alloc_n(uint32_t* dst, uint32_t ncols) {   // whole warp
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst)),
                 "r"(ncols) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc_n(uint32_t taddr, uint32_t ncols) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}

// dB partials: [kGradMmaCols columns][r4 + 4] floats; dA partials: [r][PA]
__device__ __host__ __forceinline__ int partial_floats(const GradMmaSet& st) {
    return st.stride_col == 1 ? st.r * PA : kGradMmaCols * ((st.r + 3) / 4 * 4 + 4);
}

}  // namespace

#ifdef LORA_PROBE_K3
// timing experiment only: per-CTA globaltimer stamps (0 entry, 1 setup done,
// 2 main loop done, 3 partial written, 4 reduction done, 5 exit) and, at
// lora_k3_probe_host[0..1], a one-thread stamp kernel right before / after the launch
constexpr int kProbeSlots = 6;
__device__ unsigned long long lora_k3_probe[16384 * kProbeSlots + 2];
extern "C" int lora_probe_k3_read(unsigned long long* host, int n) {   // read, then clear
    cudaError_t e = cudaMemcpyFromSymbol(host, lora_k3_probe, sizeof(unsigned long long) * n);
    void* p = nullptr;
    if (e == cudaSuccess) e = cudaGetSymbolAddress(&p, lora_k3_probe);
    if (e == cudaSuccess) e = cudaMemset(p, 0, sizeof(lora_k3_probe));
    return static_cast<int>(e);
}
__global__ void k3_probe_stamp_kernel(int slot) { lora_k3_probe[16384 * kProbeSlots + slot] = globaltimer_ns(); }
#define K3_STAMP(i)                                                                                   \
    do {                                                                                              \
        if (threadIdx.x == 64)                                                                        \
            lora_k3_probe[(blockIdx.x * gridDim.y + blockIdx.y) * kProbeSlots + (i)] = globaltimer_ns(); \
    } while (0)
#else
#define K3_STAMP(i) do {} while (0)
#endif

// ------------------------------------------------------------------ K3s
// grid (T_pad / 64, sets); block 256: stage the [64, r] fp32 chunk (contiguous)
// in shared memory, then write the three bf16 rows per coefficient.
__global__ void __launch_bounds__(256) coef_split_kernel(const __grid_constant__ CoefSplitGroup G) {
    __shared__ float chunk[64 * 64];
    const CoefSplitArgs& a = G.s[blockIdx.y];
    const int64_t t0 = static_cast<int64_t>(blockIdx.x) * 64;
    if (t0 >= a.T_pad) return;
    const int rows = a.T - t0 < 64 ? (a.T - t0 > 0 ? static_cast<int>(a.T - t0) : 0) : 64;
    for (int i = threadIdx.x; i < rows * a.r; i += 256) chunk[i] = a.coef[t0 * a.r + i];
    __syncthreads();
    // thread -> (coefficient k, token pair): two tokens per 32-bit store
    for (int e = threadIdx.x; e < a.r8 * 32; e += 256) {
        const int k = e / 32, tp = (e % 32) * 2;
        uint32_t hv[2], mv[2], lv[2];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            const int t = tp + u;
            const float v = (k < a.r && t < rows) ? chunk[t * a.r + k] : 0.0f;
            const __nv_bfloat16 h = __float2bfloat16_rn(v);
            const float r0 = v - __bfloat162float(h);
            const __nv_bfloat16 md = __float2bfloat16_rn(r0);
            const __nv_bfloat16 l = __float2bfloat16_rn(r0 - __bfloat162float(md));
            hv[u] = __bfloat16_as_ushort(h);
            mv[u] = __bfloat16_as_ushort(md);
            lv[u] = __bfloat16_as_ushort(l);
        }
        __nv_bfloat16* base = a.cs + t0 + tp;
        *reinterpret_cast<uint32_t*>(base + static_cast<int64_t>(k) * a.T_pad) = hv[0] | (hv[1] << 16);
        *reinterpret_cast<uint32_t*>(base + static_cast<int64_t>(a.r8 + k) * a.T_pad) = mv[0] | (mv[1] << 16);
        *reinterpret_cast<uint32_t*>(base + static_cast<int64_t>(2 * a.r8 + k) * a.T_pad) = lv[0] | (lv[1] << 16);
    }
}

cudaError_t launch_coef_split(const CoefSplitGroup& G, cudaStream_t stream) {
    if (G.count < 1 || G.count > kMaxGradSetsTotal) return cudaErrorInvalidValue;
    int64_t tp = 0;
    for (int i = 0; i < G.count; ++i) {
        if (G.s[i].r < 1 || G.s[i].r > 64 || G.s[i].T_pad % 64 != 0) return cudaErrorInvalidValue;
        tp = G.s[i].T_pad > tp ? G.s[i].T_pad : tp;
    }
    if (tp == 0) return cudaSuccess;
    coef_split_kernel<<<dim3(static_cast<unsigned>(tp / 64), G.count), 256, 0, stream>>>(G);
    return cudaGetLastError();
}

// exact 3-way bf16 split of v (hi + mid + lo == v) into K3's coefficient layout
__device__ __forceinline__ void split3_store(const GradMmaSet& st, int k, int64_t c, float v) {
    const __nv_bfloat16 hi = __float2bfloat16_rn(v);
    const float r0 = v - __bfloat162float(hi);
    const __nv_bfloat16 md = __float2bfloat16_rn(r0);
    const __nv_bfloat16 lo = __float2bfloat16_rn(r0 - __bfloat162float(md));
    st.cs_out[static_cast<int64_t>(k) * st.cs_t_pad + c] = hi;
    st.cs_out[static_cast<int64_t>(st.r8 + k) * st.cs_t_pad + c] = md;
    st.cs_out[static_cast<int64_t>(2 * st.r8 + k) * st.cs_t_pad + c] = lo;
}

// ------------------------------------------------------------------ K3
// Launch epilogue of every K3 CTA: wait until the preceding grid (K2, when K3
// was launched overlapping it) has completed -- so stream order stays
// transitive for the kernels after K3 -- then the last CTA out zeroes the K2
// flags this launch waited on (self-cleaning sync pool, lora_kernels.h).
__device__ __forceinline__ void k3_exit(const GradMmaGroup& G) {
    K3_STAMP(5);
    if (G.done == nullptr || threadIdx.x != 0) {
        griddep_wait();
        return;
    }
    const unsigned long long ctas = static_cast<unsigned long long>(gridDim.x) * gridDim.y;
    const bool last = atom_add_acq_rel_u64(G.done, 1ull) == ctas - 1;
    griddep_wait();   // K2 complete: no tile of it still reads the flags
    if (!last) return;
    for (int jb = 0; jb < G.njobs; ++jb)
        for (int j = 0; j < G.job[jb].nsets; ++j) {
            const GradMmaSet& st = G.set[G.job[jb].set0 + j];
            for (int f = 0; f < st.wait_n; ++f) const_cast<uint64_t*>(st.wait_flags)[f] = 0;
        }
    *G.done = 0;   // (visible to the next launch: kernel boundary)
}

__global__ void __launch_bounds__(THREADS, 1) grad_mma_kernel(const __grid_constant__ GradMmaGroup G) {
    namespace cg = cooperative_groups;
    cg::cluster_group cluster = cg::this_cluster();
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const int stages = G.stages;
    const int stage_bytes = G.stage_bytes;
    // stage s: [X 16 KiB][Cs operand: q_pad rows x 128 bytes]
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + G.region_bytes);
    uint64_t* empty = full + MAX_STAGES;
    uint64_t* tmem_full = empty + MAX_STAGES;
    uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(tmem_full + 1);
    float* partial = reinterpret_cast<float*>(smem);   // S > 1: reuses the ring after the main loop
    K3_STAMP(0);

    const int tile = static_cast<int>(blockIdx.x);
    int jb = 0;
    while (jb + 1 < G.njobs && tile >= G.tile_start[jb + 1]) ++jb;
    const GradMmaJob& J = G.job[jb];
    const int64_t col0 = static_cast<int64_t>(tile - G.tile_start[jb]) * kGradMmaCols;
    const int S = G.S;
    const int rank = S > 1 ? static_cast<int>(cluster.block_rank()) : 0;
    const int kb_total = static_cast<int>((J.T + KB - 1) / KB);
    const int kps = (kb_total + S - 1) / S;
    const int kb0 = rank * kps;
    const int nkb = kb0 < kb_total ? (kb_total - kb0 < kps ? kb_total - kb0 : kps) : 0;
    int nbox = 0;                        // 64-column boxes (K-major: 64-row boxes) holding real data
    while (nbox < 2 * MT && col0 + 64 * nbox < J.N) ++nbox;
    const int q_pad = J.q_pad;
    const int q_used = J.q_used;
    const uint32_t warp = warp_id(), lane = lane_id();

    if (warp == 0 && lane == 0) {
        tma_prefetch_desc(&G.xmap[jb]);
        for (int j = 0; j < J.nsets; ++j) tma_prefetch_desc(&G.csmap[J.set0 + j]);
    }
    if (warp == 1) {
        if (lane == 0) {
            for (int s = 0; s < stages; ++s) {
                mbar_init(&full[s], 1);
                mbar_init(&empty[s], 1);
            }
            mbar_init(tmem_full, 1);
            fence_mbar_init();
        }
        __syncwarp();
        tmem_alloc_n(tmem_holder, G.tmem_cols);
    }
    if (warp >= 2 && q_pad > q_used) {
        // Cs rows [q_used, q_pad) pad N to a multiple of 16: zero once (TMA never writes them)
        const int pr = (q_pad - q_used) * 8;   // 16-byte chunks per stage
        for (int e = static_cast<int>(threadIdx.x) - 64; e < pr * stages; e += 128) {
            const int s = e / pr, rc = e - s * pr;
            *reinterpret_cast<uint4*>(smem + s * stage_bytes + X_BYTES +
                                      swizzled_offset(q_used + rc / 8, rc % 8, 128)) = make_uint4(0, 0, 0, 0);
        }
        fence_proxy_async_smem();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_holder;
    K3_STAMP(1);

    if (warp == 0) {
        // coefficients produced by a still-running K2: the whole warp polls its row-block
        // flags (32 relaxed loads in flight, not one acquire round trip per flag), then
        // one fence makes the observed release stores an acquire for this thread's TMA
        for (int j = 0; j < J.nsets; ++j) {
            const GradMmaSet& st = G.set[J.set0 + j];
            for (int f0 = 0; f0 < st.wait_n; f0 += 32) {
                const int f = f0 + static_cast<int>(lane);
                const uint64_t t_start = globaltimer_ns();
                while (!__all_sync(0xffffffffu, f >= st.wait_n || ld_relaxed_u64(st.wait_flags + f) == 1ull)) {
                    __nanosleep(128);
                    if (globaltimer_ns() - t_start > kWaitTimeoutNs) {
                        if (lane == 0) printf("lora K3: coefficient flag wait timed out (set %d)\n", J.set0 + j);
                        __trap();
                    }
                }
            }
        }
        fence_acq_rel_gpu();   // each lane: acquire of the flags it observed
        __syncwarp();          // ... ordered before lane 0's TMA issue below
        // ---------------- TMA producer: X boxes [64 tokens][64 columns] + Cs boxes [3 r8 rows][64 tokens]
        if (lane == 0) {
            uint32_t tx = nbox * X_BOX;
            for (int j = 0; j < J.nsets; ++j) tx += G.set[J.set0 + j].nsplit * G.set[J.set0 + j].r8 * 128;
            const uint64_t pol = l2_policy_evict_first();
            fence_proxy_async_global();
            for (int i = 0, s = 0, ph = 0; i < nkb; ++i) {
                mbar_wait(&empty[s], ph ^ 1);
                uint8_t* sx = smem + s * stage_bytes;
                mbar_arrive_expect_tx(&full[s], tx);
                const int t0 = (kb0 + i) * KB;
                for (int b = 0; b < nbox; ++b) {
                    if (J.a_kmajor)   // rows col0 + 64 b .. of X [N, T], reduction columns t0 ..
                        tma_load_2d_hint(sx + b * X_BOX, &G.xmap[jb], t0, static_cast<int32_t>(col0 + 64 * b),
                                         &full[s], pol);
                    else              // columns col0 + 64 b .. of X [T, N], reduction rows t0 ..
                        tma_load_2d_hint(sx + b * X_BOX, &G.xmap[jb], static_cast<int32_t>(col0 + 64 * b), t0,
                                         &full[s], pol);
                }
                for (int j = 0; j < J.nsets; ++j)
                    tma_load_2d(sx + X_BYTES + G.set[J.set0 + j].row0 * 128, &G.csmap[J.set0 + j], t0, 0,
                                &full[s]);
                if (++s == stages) { s = 0; ph ^= 1; }
            }
        }
    } else if (warp == 1) {
        // ---------------- MMA issuer
        if (lane == 0) {
            const uint32_t idesc = make_idesc_bf16(128, static_cast<uint32_t>(q_pad), J.a_kmajor ? 0u : 1u, 0);
            for (int i = 0, s = 0, ph = 0; i < nkb; ++i) {
                mbar_wait(&full[s], ph);
                tc_fence_after();
                const uint32_t sx = smem_u32(smem + s * stage_bytes);
#pragma unroll
                for (int kk = 0; kk < KB / 16; ++kk) {
                    // MN-major X^T: two 64-column boxes, LBO = box stride, SBO = 8 tokens;
                    // K-major X: 128 rows of 128 bytes, SBO = 8 rows.  Cs: K-major SW128
                    const uint64_t b_desc = make_smem_desc(sx + X_BYTES + kk * 32, 16, 1024, kLayoutSW128);
#pragma unroll
                    for (int mt = 0; mt < MT; ++mt) {
                        if (2 * mt >= nbox) break;
                        const uint32_t sa = sx + mt * 2 * X_BOX;
                        const uint64_t a_desc = J.a_kmajor
                            ? make_smem_desc(sa + kk * 32, 16, 1024, kLayoutSW128)
                            : make_smem_desc(sa + kk * 16 * 128, X_BOX, 1024, kLayoutSW128);
                        umma_f16(tmem_base + mt * ACC_STRIDE, a_desc, b_desc, idesc, (i > 0 || kk > 0) ? 1u : 0u);
                    }
                }
                umma_commit(&empty[s]);
                if (++s == stages) { s = 0; ph ^= 1; }
            }
            if (nkb > 0) umma_commit(tmem_full); else mbar_arrive(tmem_full);
        }
    } else {
        // ---------------- epilogue: TMEM -> (hi + mid + lo) -> global (S = 1) or partial (S > 1)
        mbar_wait(tmem_full, 0);
        tc_fence_after();
        K3_STAMP(2);
        const int lq = static_cast<int>(warp & 3);          // TMEM lane quarter of this warp
        for (int mt = 0; mt < MT; ++mt) {
        const int cl = mt * 128 + lq * 32 + static_cast<int>(lane);   // column within the tile
        const bool col_ok = col0 + cl < J.N;
        const bool live = nkb > 0 && 2 * mt < nbox;          // warp-uniform
        const uint32_t tbase = tmem_base + (static_cast<uint32_t>(lq * 32) << 16) + mt * ACC_STRIDE;
        int poff = 0;
        for (int j = 0; j < J.nsets; ++j) {
            const GradMmaSet& st = G.set[J.set0 + j];
            const int r4p = (st.r + 3) / 4 * 4 + 4;
            for (int k0 = 0; k0 < st.r8; k0 += 8) {
                uint32_t h[8], md[8], l[8];
                if (live) {
                    tmem_ld_32x32b_x8(tbase + st.row0 + k0, h);
                    if (st.nsplit == 3) {
                        tmem_ld_32x32b_x8(tbase + st.row0 + st.r8 + k0, md);
                        tmem_ld_32x32b_x8(tbase + st.row0 + 2 * st.r8 + k0, l);
                    } else {
#pragma unroll
                        for (int u = 0; u < 8; ++u) md[u] = l[u] = 0u;
                    }
                    tmem_ld_wait();
                }
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const int k = k0 + u;
                    if (k >= st.r) break;
                    const float v = live
                        ? (__uint_as_float(h[u]) + __uint_as_float(md[u])) + __uint_as_float(l[u]) : 0.0f;
                    if (S == 1) {
                        if (col_ok) {
                            float* dst = st.out + (col0 + cl) * st.stride_col + static_cast<int64_t>(k) * st.stride_k;
                            *dst = st.accumulate ? *dst + st.scale * v : st.scale * v;
                            if (st.cs_out) split3_store(st, k, col0 + cl, st.scale * v);
                        }
                    } else if (st.stride_col == 1) {
                        partial[poff + k * PA + cl] = v;
                    } else {
                        partial[poff + cl * r4p + k] = v;
                    }
                }
            }
            poff += partial_floats(st);
        }
        }
    }
    tc_fence_before();
    if (warp == 2) K3_STAMP(3);
    if (S == 1) {
        __syncthreads();
        if (warp == 1) {
            tc_fence_after();
            tmem_dealloc_n(tmem_base, G.tmem_cols);
        }
        K3_STAMP(4);
        k3_exit(G);
        return;
    }
    cluster.sync();   // all partials of the cluster written (release / acquire)
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc_n(tmem_base, G.tmem_cols);
    }

    // ---------------- cluster reduction in rank order; rank q owns a 1/S share
    int poff = 0;
    for (int j = 0; j < J.nsets; ++j) {
        const GradMmaSet& st = G.set[J.set0 + j];
        const bool is_a = st.stride_col == 1;           // dA^T: O[c, k] at out[k * N + c]
        const int r4p = (st.r + 3) / 4 * 4 + 4;
        const bool vec = is_a || st.r % 4 == 0;
        const int inner = is_a ? kGradMmaCols : st.r;   // output-contiguous extent
        const int outer = is_a ? st.r : kGradMmaCols;
        const int ld = is_a ? PA : r4p;
        const int U = vec ? outer * (inner / 4) : outer * inner;
        const int per = (U + S - 1) / S;
        const int u0 = rank * per;
        const int u1 = u0 + per < U ? u0 + per : U;
        for (int u = u0 + static_cast<int>(threadIdx.x); u < u1; u += THREADS) {
            int o, in;
            if (vec) { o = u / (inner / 4); in = (u - o * (inner / 4)) * 4; }
            else { o = u / inner; in = u - o * inner; }
            const int c = is_a ? in : o, k = is_a ? o : in;
            if (col0 + c >= J.N) continue;
            const int off = poff + o * ld + in;
            float* dst = st.out + (col0 + c) * st.stride_col + static_cast<int64_t>(k) * st.stride_k;
            if (vec) {
                float4 v[8];
#pragma unroll
                for (int q = 0; q < 8; ++q)
                    if (q < S) v[q] = *reinterpret_cast<const float4*>(cluster.map_shared_rank(partial + off, q));
                float4 sum = v[0];
#pragma unroll
                for (int q = 1; q < 8; ++q)
                    if (q < S) { sum.x += v[q].x; sum.y += v[q].y; sum.z += v[q].z; sum.w += v[q].w; }
                sum.x *= st.scale; sum.y *= st.scale; sum.z *= st.scale; sum.w *= st.scale;
                if (st.cs_out) {   // (row projections: never accumulate); 4 columns (dA^T) or 4 ranks
                    const float sv[4] = {sum.x, sum.y, sum.z, sum.w};
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        if (is_a) split3_store(st, k, col0 + c + i, sv[i]);
                        else split3_store(st, k + i, col0 + c, sv[i]);
                    }
                }
                float4* d4 = reinterpret_cast<float4*>(dst);
                if (st.accumulate) {
                    const float4 o4 = *d4;
                    sum.x += o4.x; sum.y += o4.y; sum.z += o4.z; sum.w += o4.w;
                }
                *d4 = sum;
            } else {
                float v[8];
#pragma unroll
                for (int q = 0; q < 8; ++q)
                    if (q < S) v[q] = *cluster.map_shared_rank(partial + off, q);
                float sum = v[0];
#pragma unroll
                for (int q = 1; q < 8; ++q)
                    if (q < S) sum += v[q];
                sum *= st.scale;
                if (st.cs_out) split3_store(st, k, col0 + c, sum);
                *dst = st.accumulate ? *dst + sum : sum;
            }
        }
        poff += partial_floats(st);
    }
    K3_STAMP(4);
    cluster.sync();   // peers may still read this CTA's partial
    k3_exit(G);
}

// Token split S (cluster size): minimise waves x (k-blocks per CTA + a fixed
// cost of ~6 k-blocks for prologue, epilogue and reduction); ties -> smaller S.
// slots[S] = CTAs of cluster size S that can be co-resident (cluster
// placement within GPCs makes this smaller than CTAs-per-SM x SMs for S > 1).
// K3 / K2 overlap on by default; LORA_K3_OVERLAP=0 launches K3 in plain stream order.
bool k3_overlap_enabled() {
    static const bool on = [] {
        const char* v = getenv("LORA_K3_OVERLAP");
        return !(v && v[0] == '0');
    }();
    return on;
}

int grad_mma_cluster_size(int tiles, int kb_total, const int* slots) {
    int best = 1;
    long best_cost = -1;
    for (int S = 1; S <= 8 && S <= kb_total; ++S) {
        if (slots[S] <= 0) continue;
        const long waves = (static_cast<long>(tiles) * S + slots[S] - 1) / slots[S];
        const long cost = waves * ((kb_total + S - 1) / S + 6);
        if (best_cost < 0 || cost < best_cost) { best_cost = cost; best = S; }
    }
    return best;
}

cudaError_t launch_grad_mma(GradMmaGroup& G, int num_sms, cudaStream_t stream, bool overlap_prev) {
    if (G.njobs < 1 || G.njobs > kMaxGradJobs) return cudaErrorInvalidValue;
    int tiles = 0, qmax = 16, pmax = 0, kb_max = 1;
    for (int jb = 0; jb < G.njobs; ++jb) {
        GradMmaJob& J = G.job[jb];
        if (J.q_pad < 16 || J.q_pad > 256 || J.q_pad % 16 != 0 || J.q_used > J.q_pad) return cudaErrorInvalidValue;
        G.tile_start[jb] = tiles;
        tiles += static_cast<int>((J.N + kGradMmaCols - 1) / kGradMmaCols);
        qmax = J.q_pad > qmax ? J.q_pad : qmax;
        int pf = 0;
        for (int j = 0; j < J.nsets; ++j) pf += partial_floats(G.set[J.set0 + j]);
        pmax = pf > pmax ? pf : pmax;
        const int kb = static_cast<int>((J.T + KB - 1) / KB);
        kb_max = kb > kb_max ? kb : kb_max;
    }
    G.tile_start[G.njobs] = tiles;
    if (tiles == 0) return cudaSuccess;
    G.stage_bytes = X_BYTES + (qmax * 128 + 1023) / 1024 * 1024;
    G.tmem_cols = 32;
    while (G.tmem_cols < qmax) G.tmem_cols *= 2;
    if (MT == 2) G.tmem_cols = 512;   // two accumulators at columns 0 and 256 (one CTA per SM)
    const int fixed = 1024 /* barriers */ + 1024 /* alignment */;
    // two CTAs per SM when at least 3 stages fit in half the shared memory (and TMEM allows)
    int per_sm = MT == 1 ? 2 : 1;
    int stages = per_sm == 2 ? (SMEM_SM / 2 - 1024 - fixed) / G.stage_bytes : 0;
#ifdef LORA_K3_ONE_PER_SM
    stages = 0;   // experiment: one CTA per SM, deep ring
#endif
    if (stages < 3) {
        per_sm = 1;
        stages = (SMEM_CTA_MAX - fixed) / G.stage_bytes;
    }
    stages = stages > MAX_STAGES ? MAX_STAGES : stages;
#ifdef LORA_K3_STAGES
    stages = stages > LORA_K3_STAGES ? LORA_K3_STAGES : stages;
#endif
    if (stages < 2) return cudaErrorInvalidValue;
    G.stages = stages;
    int region = stages * G.stage_bytes;
    region = region > pmax * 4 ? region : pmax * 4;   // (the partial only matters for S > 1)
    G.region_bytes = (region + 1023) / 1024 * 1024;
    if (G.region_bytes + fixed > SMEM_CTA_MAX) return cudaErrorInvalidValue;
    const int smem = G.region_bytes + fixed;
    cudaError_t e = cudaFuncSetAttribute(grad_mma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    if (smem > SMEM_SM / 2 - 1024) per_sm = 1;
    cudaLaunchConfig_t cfg = {};
    cfg.blockDim = dim3(THREADS);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    // co-resident CTAs per cluster size (cached per smem size and device)
    static thread_local int cache_smem = -1, cache_dev = -1, slots[9];
    int dev = 0;
    if ((e = cudaGetDevice(&dev)) != cudaSuccess) return e;
    if (cache_smem != smem || cache_dev != dev) {
        slots[0] = 0;
        slots[1] = per_sm * num_sms;
        for (int S = 2; S <= 8; ++S) {
            attr[0].val.clusterDim.y = S;
            cfg.gridDim = dim3(1, S);
            int nc = 0;
            if (cudaOccupancyMaxActiveClusters(&nc, grad_mma_kernel, &cfg) != cudaSuccess) {
                cudaGetLastError();
                nc = 0;
            }
            slots[S] = nc * S;
        }
        // measured on B200: CTA pairs pack two per SM like single CTAs (the
        // occupancy query reports one); S >= 3 clusters do not (query kept)
        slots[2] = slots[2] > slots[1] ? slots[2] : slots[1];
        cache_smem = smem;
        cache_dev = dev;
    }
    G.S = grad_mma_cluster_size(tiles, kb_max, slots);
    // Overlapping K2's last wave (programmatic stream serialization), short token
    // ranges and enough column tiles for most SMs: no token split.  Measured at cfg2
    // (96 tiles, 32 k-blocks; graph-replayed step, profiles/r02/k3_split.txt): S = 1
    // 0.2019 ms per step vs 0.2101 for the cost model's S = 2 -- one-CTA jobs start
    // on the SMs K2's finished pairs free and hide under its tail, although K3 alone
    // takes longer (29 vs 23 us); at cfg3 (64 k-blocks) S = 1 was slower (2.351 vs 2.335).
    if (overlap_prev && k3_overlap_enabled() && kb_max <= 32 && tiles * 10 >= num_sms * 6) G.S = 1;
    if (const char* fs = getenv("LORA_K3_S")) {   // tests / experiments: force the token split
        const int v = atoi(fs);
        if (v >= 1 && v <= 8) G.S = v;
    }
    cfg.gridDim = dim3(tiles, G.S);
    attr[0].val.clusterDim.y = G.S;
    cudaLaunchAttribute attrs[2] = {attr[0], {}};
    attrs[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attrs[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attrs;
    cfg.numAttrs = overlap_prev && k3_overlap_enabled() ? 2 : 1;
#ifdef LORA_PROBE_K3
    k3_probe_stamp_kernel<<<1, 1, 0, stream>>>(0);
#endif
    e = cudaLaunchKernelEx(&cfg, grad_mma_kernel, G);
    if (e != cudaSuccess) return e;
#ifdef LORA_PROBE_K3
    k3_probe_stamp_kernel<<<1, 1, 0, stream>>>(1);
#endif
    return cudaGetLastError();
}

// (lazy loading: see preload_gemm_kernels in lora_gemm.cu)
cudaError_t preload_grad_mma_kernels() {
    cudaFuncAttributes a;
    cudaError_t e = cudaFuncGetAttributes(&a, (const void*)coef_split_kernel);
    return e != cudaSuccess ? e : cudaFuncGetAttributes(&a, (const void*)grad_mma_kernel);
}

}  // namespace lora_sm100
