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
// Mapping (one CTA = 256 X columns x one token slice):
//   MMA   D[c, q] += X^T[c, t] Cs[q, t]     M = 128 columns (two MMAs per
//         k-step for the CTA's 256 columns), N = q_pad, K = 16 tokens.
//         A operand = the X tile exactly as TMA lands it ([64 tokens][64
//         columns] SWIZZLE_128B boxes, read MN-major: no transpose pass).
//   Cs    the fp32 coefficients split into three bf16 rows hi + mid + lo
//         (8 + 8 + 8 significand bits: C is represented exactly, so every
//         product is exact and only the fp32 accumulation rounds, as on the
//         CUDA cores; x and dY are exact bf16), written K-major SW128 by four
//         converter warps; several coefficient SETS sharing one X (dA of the
//         q/k/v projections all read x) are stacked along N, so x is read once
//         for all of them.
//   split the tokens are split over a cluster of S CTAs (same columns); each
//         CTA drains its TMEM partial into shared memory and the cluster sums
//         the S partials over DSMEM in rank order: deterministic, no atomics,
//         no global partial buffer, final values (or +=) written once.
// Warp roles (192 threads): warp 0 TMA producer, warp 1 MMA issuer + TMEM
// owner, warps 2..5 coefficient converters, then epilogue; all six reduce.
#include <cooperative_groups.h>
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "lora_kernels.h"
#include "sm100_ptx.cuh"

namespace lora_sm100 {

namespace {

constexpr int KB = 64;              // tokens per k-block (one 128-byte SW128 row of the Cs operand)
constexpr int X_BOX = 64 * KB * 2;  // one [64 tokens][64 columns] bf16 box = 8 KiB
constexpr int X_BYTES = 4 * X_BOX;  // 256 columns per CTA
constexpr int THREADS = 192;
constexpr int PST = kGradMmaCols + 1;  // partial row stride (floats): conflict-free in both orders
constexpr int SMEM_LIMIT = 227 * 1024;
constexpr int MAX_STAGES = 6;

__device__ __forceinline__ void tmem_ld_32x32b_x8(uint32_t taddr, uint32_t (&v)[8]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
                   "=r"(v[7])
                 : "r"(taddr));
}

// 8 fp32 -> three 16-byte chunks of bf16: hi = RNE(v), mid = RNE(v - hi),
// lo = RNE(v - hi - mid).  Both differences are exact in fp32 (Sterbenz), and
// v - hi - mid has at most 8 significant bits left, so hi + mid + lo == v.
__device__ __forceinline__ void split8(const float (&v)[8], uint4& hi, uint4& mid, uint4& lo) {
    uint32_t h[4], md[4], l[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const __nv_bfloat162 hv = __floats2bfloat162_rn(v[2 * i], v[2 * i + 1]);
        const float2 hf = __bfloat1622float2(hv);
        const float r0 = v[2 * i] - hf.x, r1 = v[2 * i + 1] - hf.y;
        const __nv_bfloat162 mv = __floats2bfloat162_rn(r0, r1);
        const float2 mf = __bfloat1622float2(mv);
        const __nv_bfloat162 lv = __floats2bfloat162_rn(r0 - mf.x, r1 - mf.y);
        h[i] = *reinterpret_cast<const uint32_t*>(&hv);
        md[i] = *reinterpret_cast<const uint32_t*>(&mv);
        l[i] = *reinterpret_cast<const uint32_t*>(&lv);
    }
    hi = make_uint4(h[0], h[1], h[2], h[3]);
    mid = make_uint4(md[0], md[1], md[2], md[3]);
    lo = make_uint4(l[0], l[1], l[2], l[3]);
}

// 1-D bulk copy global -> shared (16-byte multiple), completes on `bar`
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

}  // namespace

__global__ void __launch_bounds__(THREADS, 1) grad_mma_kernel(const __grid_constant__ GradMmaGroup G) {
    namespace cg = cooperative_groups;
    cg::cluster_group cluster = cg::this_cluster();
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const int stages = G.stages;
    const int stage_bytes = G.stage_bytes;
    // stage s: [X 32 KiB][Cs operand, cs_bytes][fp32 coefficient staging, 256 r bytes per set]
    uint64_t* loaded = reinterpret_cast<uint64_t*>(smem + G.region_bytes);   // X + coefficients landed
    uint64_t* full = loaded + MAX_STAGES;                                    // Cs operand written
    uint64_t* empty = full + MAX_STAGES;                                     // MMAs of the stage done
    uint64_t* tmem_full = empty + MAX_STAGES;
    uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(tmem_full + 1);
    float* partial = reinterpret_cast<float*>(smem);   // reuses the ring after the main loop

    const int tile = static_cast<int>(blockIdx.x);
    int jb = 0;
    while (jb + 1 < G.njobs && tile >= G.tile_start[jb + 1]) ++jb;
    const GradMmaJob& J = G.job[jb];
    const int64_t col0 = static_cast<int64_t>(tile - G.tile_start[jb]) * kGradMmaCols;
    const int S = G.S;
    const int rank = static_cast<int>(cluster.block_rank());
    const int kb_total = static_cast<int>((J.T + KB - 1) / KB);
    const int kps = (kb_total + S - 1) / S;
    const int kb0 = rank * kps;
    const int nkb = kb0 < kb_total ? (kb_total - kb0 < kps ? kb_total - kb0 : kps) : 0;
    const bool two = col0 + 128 < J.N;   // the second M = 128 half holds real columns
    const int q_pad = J.q_pad;
    const uint32_t warp = warp_id(), lane = lane_id();

    if (warp == 0 && lane == 0) tma_prefetch_desc(&J.x);
    if (warp == 1) {
        if (lane == 0) {
            for (int s = 0; s < stages; ++s) {
                mbar_init(&loaded[s], 1);     // producer (expect_tx)
                mbar_init(&full[s], 4);       // 4 converter warps
                mbar_init(&empty[s], 1);
            }
            mbar_init(tmem_full, 1);
            fence_mbar_init();
        }
        __syncwarp();
        tmem_alloc<512>(tmem_holder);
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_holder;

    if (warp == 0) {
        // ---------------- producer: X boxes [64 tokens][64 columns] (TMA) and the
        // k-block's fp32 coefficient rows of every set (contiguous: 1-D bulk copy)
        if (lane == 0) {
            const int nbox = two ? 4 : 2;
            const uint64_t pol = l2_policy_evict_first();
            for (int i = 0, s = 0, ph = 0; i < nkb; ++i) {
                mbar_wait(&empty[s], ph ^ 1);
                uint8_t* sx = smem + s * stage_bytes;
                uint8_t* sstg = sx + X_BYTES + G.cs_bytes;
                const int t0 = (kb0 + i) * KB;
                const int64_t rows = J.T - t0 < KB ? J.T - t0 : KB;
                uint32_t tx = nbox * X_BOX;
                for (int j = 0; j < J.nsets; ++j)
                    tx += static_cast<uint32_t>((rows * J.set[j].r * 4 + 15) / 16 * 16);
                mbar_arrive_expect_tx(&loaded[s], tx);
                for (int b = 0; b < nbox; ++b)
                    tma_load_2d_hint(sx + b * X_BOX, &J.x, static_cast<int32_t>(col0 + 64 * b), t0, &loaded[s],
                                     pol);
                // (the last k-block may round up past T * r floats by < 16 bytes: same 16-byte granule)
                for (int j = 0, off = 0; j < J.nsets; off += 256 * J.set[j].r, ++j)
                    bulk_load(sstg + off, J.set[j].coef + static_cast<int64_t>(t0) * J.set[j].r,
                              static_cast<uint32_t>((rows * J.set[j].r * 4 + 15) / 16 * 16), &loaded[s]);
                if (++s == stages) { s = 0; ph ^= 1; }
            }
        }
    } else if (warp == 1) {
        // ---------------- MMA issuer
        if (lane == 0) {
            const uint32_t idesc = make_idesc_bf16(128, static_cast<uint32_t>(q_pad), 1, 0);
            for (int i = 0, s = 0, ph = 0; i < nkb; ++i) {
                mbar_wait(&loaded[s], ph);
                mbar_wait(&full[s], ph);
                tc_fence_after();
                const uint32_t sx = smem_u32(smem + s * stage_bytes);
                const uint32_t sc = sx + X_BYTES;
#pragma unroll
                for (int kk = 0; kk < KB / 16; ++kk) {
                    const uint64_t b_desc = make_smem_desc(sc + kk * 32, 16, 1024, kLayoutSW128);
                    const uint32_t acc = (i > 0 || kk > 0) ? 1u : 0u;
                    // X^T: two 64-column boxes per M = 128 half, LBO = box stride, SBO = 8 tokens
                    umma_f16(tmem_base, make_smem_desc(sx + kk * 16 * 128, X_BOX, 1024, kLayoutSW128), b_desc,
                             idesc, acc);
                    if (two)
                        umma_f16(tmem_base + 256, make_smem_desc(sx + 2 * X_BOX + kk * 16 * 128, X_BOX, 1024,
                                                                 kLayoutSW128),
                                 b_desc, idesc, acc);
                }
                umma_commit(&empty[s]);
                if (++s == stages) { s = 0; ph ^= 1; }
            }
            if (nkb > 0) umma_commit(tmem_full); else mbar_arrive(tmem_full);
        }
    } else {
        // ---------------- converters: Cs[q, t] rows (hi / mid / lo at row0 + {0, 1, 2} r8 + k)
        const int ct = static_cast<int>(threadIdx.x) - 64;   // 0..127
        int k8 = 0;                                          // sum of r8 over the sets
        for (int j = 0; j < J.nsets; ++j) k8 += J.set[j].r8;
        const int tasks = k8 * (KB / 8);
        // rows [3 k8, q_pad) pad N to a multiple of 16: zero once (the ring never overwrites them)
        for (int e = ct; e < (q_pad - 3 * k8) * (KB / 8) * stages; e += 128) {
            const int s = e / ((q_pad - 3 * k8) * (KB / 8));
            const int rc = e - s * ((q_pad - 3 * k8) * (KB / 8));
            *reinterpret_cast<uint4*>(smem + s * stage_bytes + X_BYTES +
                                      swizzled_offset(3 * k8 + rc / (KB / 8), rc % (KB / 8), 128)) =
                make_uint4(0, 0, 0, 0);
        }
        for (int i = 0, s = 0, ph = 0; i < nkb; ++i) {
            mbar_wait(&loaded[s], ph);   // (the producer waited for this stage's MMAs before refilling)
            uint8_t* sc = smem + s * stage_bytes + X_BYTES;
            const float* sstg = reinterpret_cast<const float*>(sc + G.cs_bytes);
            const int64_t t0 = static_cast<int64_t>(kb0 + i) * KB;
            for (int e = ct; e < tasks; e += 128) {
                const int c = e / k8;          // 8-token chunk
                int kk = e - c * k8;           // index into the stacked sets
                int j = 0, off = 0;
                while (kk >= J.set[j].r8) { kk -= J.set[j].r8; off += 64 * J.set[j].r; ++j; }
                const GradMmaSet& st = J.set[j];
                float v[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const int tl = c * 8 + u;
                    v[u] = (kk < st.r && t0 + tl < J.T) ? sstg[off + tl * st.r + kk] : 0.0f;
                }
                uint4 hi, mid, lo;
                split8(v, hi, mid, lo);
                *reinterpret_cast<uint4*>(sc + swizzled_offset(st.row0 + kk, c, 128)) = hi;
                *reinterpret_cast<uint4*>(sc + swizzled_offset(st.row0 + st.r8 + kk, c, 128)) = mid;
                *reinterpret_cast<uint4*>(sc + swizzled_offset(st.row0 + 2 * st.r8 + kk, c, 128)) = lo;
            }
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) mbar_arrive(&full[s]);
            if (++s == stages) { s = 0; ph ^= 1; }
        }
        // ---------------- epilogue: TMEM -> partial[kbase + k][column] (hi + mid + lo)
        mbar_wait(tmem_full, 0);
        tc_fence_after();
        const int lq = static_cast<int>(warp & 3);          // TMEM lane quarter of this warp
        for (int mt = 0; mt < 2; ++mt) {
            const int cl = mt * 128 + lq * 32 + static_cast<int>(lane);
            const uint32_t tbase = tmem_base + (static_cast<uint32_t>(lq * 32) << 16) + mt * 256;
            int kbase = 0;
            for (int j = 0; j < J.nsets; ++j) {
                const GradMmaSet& st = J.set[j];
                for (int k0 = 0; k0 < st.r8; k0 += 8) {
                    uint32_t h[8], md[8], l[8];
                    const bool live = nkb > 0 && (mt == 0 || two);
                    if (live) {   // warp-uniform
                        tmem_ld_32x32b_x8(tbase + st.row0 + k0, h);
                        tmem_ld_32x32b_x8(tbase + st.row0 + st.r8 + k0, md);
                        tmem_ld_32x32b_x8(tbase + st.row0 + 2 * st.r8 + k0, l);
                        tmem_ld_wait();
                    }
#pragma unroll
                    for (int u = 0; u < 8; ++u)
                        if (k0 + u < st.r)
                            partial[(kbase + k0 + u) * PST + cl] =
                                live ? (__uint_as_float(h[u]) + __uint_as_float(md[u])) + __uint_as_float(l[u])
                                     : 0.0f;
                }
                kbase += st.r;
            }
        }
    }
    tc_fence_before();
    cluster.sync();   // all partials of the cluster written (release / acquire)
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc<512>(tmem_base);
    }

    // ---------------- cluster reduction in rank order; rank q owns a 1/S share
    int kbase = 0;
    for (int j = 0; j < J.nsets; ++j) {
        const GradMmaSet& st = J.set[j];
        const int E = st.r * kGradMmaCols;
        const int per = (E + S - 1) / S;
        const int e0 = rank * per;
        const int e1 = e0 + per < E ? e0 + per : E;
        const bool col_fast = st.stride_col == 1;   // dA^T: store O[c, q] at out[q * N + c]
        for (int e = e0 + static_cast<int>(threadIdx.x); e < e1; e += THREADS) {
            int k, c;
            if (col_fast) { k = e / kGradMmaCols; c = e - k * kGradMmaCols; }
            else { c = e / st.r; k = e - c * st.r; }
            if (col0 + c >= J.N) continue;
            const int o = (kbase + k) * PST + c;
            float sum = 0.0f;
            for (int q = 0; q < S; ++q) sum += cluster.map_shared_rank(partial, q)[o];
            sum *= st.scale;
            float* dst = st.out + (col0 + c) * st.stride_col + static_cast<int64_t>(k) * st.stride_k;
            *dst = st.accumulate ? *dst + sum : sum;
        }
        kbase += st.r;
    }
    cluster.sync();   // peers may still read this CTA's partial
}

int grad_mma_cluster_size(int tiles, int kb_total, int num_sms) {
    // minimise waves / S (per-CTA work ~ 1 / S); ties -> smaller S
    int best = 1;
    double best_cost = 1e30;
    for (int S = 1; S <= 8 && S <= kb_total; ++S) {
        const int waves = (tiles * S + num_sms - 1) / num_sms;
        const double cost = static_cast<double>(waves) / S + 1e-3 * S;
        if (cost < best_cost - 1e-9) { best_cost = cost; best = S; }
    }
    return best;
}

cudaError_t launch_grad_mma(GradMmaGroup& G, int num_sms, cudaStream_t stream) {
    if (G.njobs < 1 || G.njobs > kMaxGradJobs) return cudaErrorInvalidValue;
    int tiles = 0, qmax = 16, rsum_max = 0, kb_max = 1;
    for (int jb = 0; jb < G.njobs; ++jb) {
        const GradMmaJob& J = G.job[jb];
        if (J.q_pad < 16 || J.q_pad > 256 || J.q_pad % 16 != 0) return cudaErrorInvalidValue;
        G.tile_start[jb] = tiles;
        tiles += static_cast<int>((J.N + kGradMmaCols - 1) / kGradMmaCols);
        qmax = J.q_pad > qmax ? J.q_pad : qmax;
        int rs = 0;
        for (int j = 0; j < J.nsets; ++j) rs += J.set[j].r;
        rsum_max = rs > rsum_max ? rs : rsum_max;
        const int kb = static_cast<int>((J.T + KB - 1) / KB);
        kb_max = kb > kb_max ? kb : kb_max;
    }
    G.tile_start[G.njobs] = tiles;
    if (tiles == 0) return cudaSuccess;
    G.cs_bytes = (qmax * 128 + 1023) / 1024 * 1024;
    G.stage_bytes = X_BYTES + G.cs_bytes + (rsum_max * 256 + 1023) / 1024 * 1024;
    const int partial_bytes = rsum_max * PST * 4;
    const int fixed = 1024 /* barriers */ + 1024 /* alignment */;
    int stages = (SMEM_LIMIT - fixed) / G.stage_bytes;
    stages = stages > MAX_STAGES ? MAX_STAGES : stages;
    if (stages < 2) return cudaErrorInvalidValue;
    G.stages = stages;
    int region = stages * G.stage_bytes;
    region = region > partial_bytes ? region : partial_bytes;
    G.region_bytes = (region + 1023) / 1024 * 1024;
    if (G.region_bytes + fixed > SMEM_LIMIT) return cudaErrorInvalidValue;
    G.S = grad_mma_cluster_size(tiles, kb_max, num_sms);
    const int smem = G.region_bytes + fixed;
    cudaError_t e = cudaFuncSetAttribute(grad_mma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    if (G.S > 8) return cudaErrorInvalidValue;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(tiles, G.S);
    cfg.blockDim = dim3(THREADS);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 1;
    attr[0].val.clusterDim.y = G.S;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    e = cudaLaunchKernelEx(&cfg, grad_mma_kernel, G);
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

}  // namespace lora_sm100
