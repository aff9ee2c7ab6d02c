// lora_merge_mma.cu -- K4 merge on the tensor cores (sm_100a):
//     W' = bf16(W0 + s (B A))        Eq. 1 line 2, R14
//
// B A is a dense contraction with K = r.  On the CUDA cores it costs r FMAs
// per output element: at r = 8 the 32 M elements of a 4096^2 projection need
// 268 M FMAs = 7.4 us of perfectly issued FFMA2 on 148 SMs, against a 10.3 us
// HBM floor (4 m n bytes); at r = 16 (45 M elements, 11008 x 4096) 20 us
// against 14 us -- the CUDA-core kernel is issue-bound, not HBM-bound.  Here
// one tcgen05.mma per 16 of r puts (B A) for a 128 x 64 tile into TMEM, and
// the CUDA cores only add W0, scale and round.
//
// Persistent, one CTA per SM, 10 warps (producer and MMA issuer on the two highest
// warp ids, which the warp schedulers favour over the busy epilogue warps):
//   warp 8     TMA producer: W0 tile [128 x 64] (one SW128 box), B rows
//              [128 x r_pad] (K-major), A [r_pad x 64] (MN-major SW128) -> an
//              up to 8-deep ring (small tiles: more bytes in flight per SM)
//   warp 9     MMA issuer: D[i, k] = sum_j B[i, j] A[j, k], r_pad / 16 MMAs
//              (M = 128, N = 64) into one of two TMEM accumulators
//   warps 0-7  epilogue: two warps per TMEM lane quarter (32 columns each; one
//              warp per SM sub-partition left the drain latency-bound), row i
//              per thread: tcgen05.ld, out = fma(s, D, W0) with
//              W0 read from the stage, RNE bf16 written back IN PLACE into the
//              W0 box, then one thread TMA-stores the box (bulk group) and
//              frees the stage once the store has read it.
// Traffic: W0 read once, W' written once (TMA, full lines); A and B are tiny
// and L2-resident.  In-place (w_out == w0) is safe: a tile's store is issued
// only after its own load has landed, and tiles are disjoint.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>

#include "lora_kernels.h"
#include "sm100_ptx.cuh"

namespace lora_sm100 {

namespace {

#ifndef LORA_MERGE_CTAS_PER_SM
#define LORA_MERGE_CTAS_PER_SM 1
#endif
constexpr int kMBM = 128;          // W0 rows per tile (UMMA M)
constexpr int kMThreads = 320;   // producer, MMA, 8 epilogue warps
constexpr int kMSmemLimit = 227 * 1024;

template <int R_PAD, int BN>
struct MergeCfg {
    static constexpr int NBOX = BN / 64;                         // [128 x 64] SW128 boxes per tile
    static constexpr int W_BYTES = kMBM * BN * 2;
    static constexpr int BROW = R_PAD * 2;                       // B row bytes in smem (32 / 64 / 128)
    static constexpr int B_BYTES = kMBM * BROW;                  // B rows, K-major
    static constexpr int A_BYTES = NBOX * R_PAD * 128;           // A, 64-column MN-major blocks
    static constexpr int STAGE_BYTES = W_BYTES + B_BYTES + A_BYTES;
    // LORA_MERGE_CTAS_PER_SM CTAs per SM share the shared memory (experiment: 1 or 2)
    static constexpr int HALF_SM = (228 * 1024) / 2 - 1024;
    static constexpr int CTAS = (LORA_MERGE_CTAS_PER_SM == 2 && 2 * STAGE_BYTES + 2048 <= HALF_SM) ? 2 : 1;
    static constexpr int SMEM_AVAIL = CTAS == 1 ? kMSmemLimit : HALF_SM;
    static constexpr int STAGES = (SMEM_AVAIL - 2048) / STAGE_BYTES > 8 ? 8 : (SMEM_AVAIL - 2048) / STAGE_BYTES;
    static constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 /* barriers */ + 1024 /* alignment */;
    static constexpr uint32_t B_LAYOUT = BROW == 32 ? kLayoutSW32 : (BROW == 64 ? kLayoutSW64 : kLayoutSW128);
    static_assert(STAGES >= 2, "shared memory budget");
};

template <int R_PAD, int BN>
__global__ void __launch_bounds__(kMThreads, MergeCfg<R_PAD, BN>::CTAS) merge_mma_kernel(const __grid_constant__ MergeMaps mp, int64_t m,
                                                                int64_t n, float s) {
    using C = MergeCfg<R_PAD, BN>;
    constexpr int kMBN = BN;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::STAGES * C::STAGE_BYTES);
    uint64_t* full = bars;
    uint64_t* empty = bars + C::STAGES;
    uint64_t* tmem_full = bars + 2 * C::STAGES;
    uint64_t* tmem_empty = tmem_full + 2;
    uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(tmem_empty + 2);

    const uint32_t warp = warp_id(), lane = lane_id();
    // the producer and the MMA issuer take the highest warp ids (the warp schedulers
    // favour them over the eight busy epilogue warps): epilogue 0..7, producer 8, MMA 9
    constexpr uint32_t W_PROD = 8, W_MMA = 9;
    const int64_t nrb = (m + kMBM - 1) / kMBM, ncb = (n + kMBN - 1) / kMBN;
    const int64_t ntiles = nrb * ncb;

    if (warp == W_PROD && lane == 0) {
        tma_prefetch_desc(&mp.w);
        tma_prefetch_desc(&mp.out);
        tma_prefetch_desc(&mp.b);
        tma_prefetch_desc(&mp.a);
    }
    if (warp == W_MMA && lane == 0) {
        for (int i = 0; i < C::STAGES; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&tmem_full[i], 1);
            mbar_init(&tmem_empty[i], 8);   // one arrive per epilogue warp
        }
        fence_mbar_init();
    }
    if (warp == 0) tmem_alloc<2 * kMBN>(tmem_holder);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_holder;

    if (warp == W_PROD) {
        // ===================== TMA producer =====================
        if (elect_one()) {
            const uint64_t pol_stream = l2_policy_evict_first();
            uint32_t stage = 0, phase = 0;
            for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
                const int i0 = static_cast<int>((t / ncb) * kMBM), k0 = static_cast<int>((t % ncb) * kMBN);
                mbar_wait(&empty[stage], phase ^ 1);
                uint8_t* sW = smem + stage * C::STAGE_BYTES;
                uint8_t* sB = sW + C::W_BYTES;
                uint8_t* sA = sB + C::B_BYTES;
                mbar_arrive_expect_tx(&full[stage], C::STAGE_BYTES);
#pragma unroll
                for (int q = 0; q < C::NBOX; ++q)
                    tma_load_2d_hint(sW + q * (kMBM * 128), &mp.w, k0 + 64 * q, i0, &full[stage], pol_stream);
                tma_load_2d(sB, &mp.b, 0, i0, &full[stage]);
#pragma unroll
                for (int q = 0; q < C::NBOX; ++q) tma_load_2d(sA + q * (R_PAD * 128), &mp.a, k0 + 64 * q, 0, &full[stage]);
                if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
            }
        }
    } else if (warp == W_MMA) {
        // ===================== MMA issuer =====================
        if (elect_one()) {
            constexpr uint32_t idesc = make_idesc_bf16(kMBM, kMBN, 0, 1);
            uint32_t stage = 0, phase = 0, tl = 0;
            for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++tl) {
                const uint32_t acc = tl & 1, acc_phase = (tl >> 1) & 1;
                mbar_wait(&tmem_empty[acc], acc_phase ^ 1);
                mbar_wait(&full[stage], phase);
                tc_fence_after();
                const uint32_t b_addr = smem_u32(smem + stage * C::STAGE_BYTES + C::W_BYTES);
                const uint32_t a_addr = b_addr + C::B_BYTES;
#pragma unroll
                for (int kk = 0; kk < R_PAD / 16; ++kk) {
                    // MMA A operand: B rows [128 x r_pad] K-major (swizzle = row size)
                    const uint64_t a_desc = make_smem_desc(b_addr + kk * 32, 16, 8 * C::BROW, C::B_LAYOUT);
                    // MMA B operand: A [r_pad x 128] MN-major, 64-column blocks at LBO = r_pad * 128
                    const uint64_t b_desc = make_smem_desc(a_addr + kk * (16 * 128), R_PAD * 128, 1024,
                                                           kLayoutSW128);
                    umma_f16(tmem_base + acc * kMBN, a_desc, b_desc, idesc, kk > 0 ? 1u : 0u);
                }
                umma_commit(&tmem_full[acc]);
                if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
            }
        }
    } else {
        // ===================== epilogue (warps 0..7) =====================
        const uint32_t quarter = warp & 3;            // TMEM lane quarter this warp may access
        const uint32_t half = warp >> 2;              // this warp's columns: [CW half, CW half + CW)
        constexpr int CW = BN / 2;
        const uint32_t row_local = quarter * 32 + lane;
        const bool storer = (warp == 0 && lane == 0);
        const uint64_t pol_stream = l2_policy_evict_first();
        uint32_t stage = 0, phase = 0, tl = 0;
        int prev_stage = -1;
        const float2 ss = make_float2(s, s);
        for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++tl) {
            const int i0 = static_cast<int>((t / ncb) * kMBM), k0 = static_cast<int>((t % ncb) * kMBN);
            const uint32_t acc = tl & 1, acc_phase = (tl >> 1) & 1;
            mbar_wait(&full[stage], phase);          // W0 tile landed (TMA writes visible here)
            mbar_wait(&tmem_full[acc], acc_phase);   // B A in TMEM
            tc_fence_after();
            uint8_t* box = smem + stage * C::STAGE_BYTES + ((half * CW) / 64) * (kMBM * 128);
            const uint32_t ch0 = ((half * CW) % 64) / 8;   // first 16-byte chunk of the row in that box
            const uint32_t tbase = tmem_base + ((quarter * 32) << 16) + acc * kMBN + half * CW;
            uint32_t v[CW / 32][32];
#pragma unroll
            for (int q = 0; q < CW / 32; ++q) tmem_ld_32x32b_x32(tbase + 32 * q, v[q]);
            tmem_ld_wait();
#pragma unroll
            for (int ch = 0; ch < CW / 8; ++ch) {   // columns half CW + 8 ch .. + 7
                uint4* p = reinterpret_cast<uint4*>(box + swizzled_offset(row_local, ch0 + ch, 128));
                const uint4 w = *p;
                const uint32_t wv[4] = {w.x, w.y, w.z, w.w};
                uint32_t o[4];
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    // bf16 pair -> fp32 pair (the bf16 bits are the high halves)
                    const float2 w2 = make_float2(__uint_as_float(wv[e] << 16), __uint_as_float(wv[e] & 0xFFFF0000u));
                    const float2 d2 = make_float2(__uint_as_float(v[ch >> 2][(ch & 3) * 8 + 2 * e]),
                                                  __uint_as_float(v[ch >> 2][(ch & 3) * 8 + 2 * e + 1]));
                    const float2 r2 = ffma2(ss, d2, w2);   // W0 + s (B A), one rounding each
                    o[e] = pack_bf16x2(r2.x, r2.y);
                }
                *p = make_uint4(o[0], o[1], o[2], o[3]);
            }
            // the accumulator is free once every epilogue warp's tcgen05.ld completed
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&tmem_empty[acc]);
            // W' tile complete in the stage: make the generic writes visible to TMA, store
            fence_proxy_async_smem();
            named_bar_sync(1, 256);
            if (storer) {
                uint8_t* sW = smem + stage * C::STAGE_BYTES;
#pragma unroll
                for (int q = 0; q < C::NBOX; ++q) tma_store_2d_hint(&mp.out, sW + q * (kMBM * 128), k0 + 64 * q, i0, pol_stream);
                bulk_commit_group();
                // the previous tile's store has read its stage: give that stage back
                if (prev_stage >= 0) {
                    bulk_wait_group_read<1>();
                    mbar_arrive(&empty[prev_stage]);
                }
                prev_stage = static_cast<int>(stage);
            }
            if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
        }
        if (storer) bulk_wait_group<0>();   // every store performed before the CTA exits
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        tmem_dealloc<2 * kMBN>(tmem_base);
    }
}

template <int R_PAD, int BN>
cudaError_t launch_rp(const MergeMaps& maps, int64_t m, int64_t n, float s, int num_sms, cudaStream_t stream) {
    using C = MergeCfg<R_PAD, BN>;
    auto kern = merge_mma_kernel<R_PAD, BN>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM_BYTES);
    if (e != cudaSuccess) return e;
    const int64_t ntiles = ((m + kMBM - 1) / kMBM) * ((n + BN - 1) / BN);
    const int64_t slots = static_cast<int64_t>(num_sms) * C::CTAS;
    const int grid = static_cast<int>(ntiles < slots ? ntiles : slots);
    if (grid <= 0) return cudaSuccess;
    kern<<<grid, kMThreads, C::SMEM_BYTES, stream>>>(maps, m, n, s);
    return cudaGetLastError();
}

// tile width: LORA_MERGE_BN=64 | 128 (default 128)
int merge_bn() {
    const char* v = getenv("LORA_MERGE_BN");
    return (v && atoi(v) == 64) ? 64 : 128;
}

}  // namespace

cudaError_t launch_merge_mma(const MergeMaps& maps, int r_pad, int64_t m, int64_t n, float s, int num_sms,
                             cudaStream_t stream) {
    const bool w = merge_bn() == 128;
    switch (r_pad) {
        case 16: return w ? launch_rp<16, 128>(maps, m, n, s, num_sms, stream) : launch_rp<16, 64>(maps, m, n, s, num_sms, stream);
        case 32: return w ? launch_rp<32, 128>(maps, m, n, s, num_sms, stream) : launch_rp<32, 64>(maps, m, n, s, num_sms, stream);
        case 64: return w ? launch_rp<64, 128>(maps, m, n, s, num_sms, stream) : launch_rp<64, 64>(maps, m, n, s, num_sms, stream);
    }
    return cudaErrorInvalidValue;
}

}  // namespace lora_sm100
