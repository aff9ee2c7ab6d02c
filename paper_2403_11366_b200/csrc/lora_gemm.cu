// lora_gemm.cu -- fused LoRA-linear tensor-core kernels for sm_100a (B200).
//
// K1 (MODE_FWD), Eq. 1 line 1 in row-vector form:
//     acc  = x W0^T            (base GEMM, tcgen05, fp32 accumulator in TMEM)
//     h    = x A^T             (same pass: A's r_pad rows are appended to the
//                               W0 tile, so ONE 256-column MMA per k-step
//                               produces BN = 256 - r_pad output columns and
//                               the r_pad columns of h)
//     y    = bf16(acc + bf16(s h) B^T + b0)   (epilogue: a K = r_pad "tail"
//                               MMA adds the low-rank update into the same
//                               TMEM accumulator, then one RNE to bf16)
// K2 (MODE_DX), the input gradient of Eq. 1 (W0 frozen):
//     acc  = dY W0             (W0 [m, n] read as an MN-major B operand: no
//                               transposed weight copy)
//     gh   = s dY B            (same pass, but only in the FIRST column tile of
//                               each row block: that tile is 128 columns wide
//                               and runs an extra narrow MMA on B [m, r] into
//                               TMEM columns 128.., publishes gh to global and
//                               raises a per-row-block flag; the other tiles are
//                               256 wide -- 128-byte-aligned MN-major W0 boxes --
//                               and wait for the flag before their tail)
//     dX   = bf16(acc + bf16(gh) A)  (epilogue tail MMA)
// K2 dropout mode (MODE_DX_DROP, LoRA dropout, R7):
//     dX   = bf16(acc + q M . (gh A))  -- the mask is per output element, so
//                               no tail MMA: the epilogue applies gh A on the
//                               CUDA cores from the A tile in shared memory
//                               and the keep bits K0 packed (32 per word)
// K1 with dropout: h = q (M . x) A^T comes from K0 (p.h_in) instead of TMEM.
//
// Structure (persistent over output tiles, 6 warps per CTA; the producer and
// the MMA issuer have the highest warp ids, which the warp schedulers favour):
//   warps 0..3 : epilogue (tcgen05.ld from TMEM, side output h / gh, tail
//                MMA, bf16 conversion, global stores); warp 0 owns TMEM
//   (dX dropout mode, r_pad 16: warps 4..7 drain the upper half of each tile)
//   warp 4(+4) : TMA producer (cp.async.bulk.tensor, SWIZZLE_128B, an
//                STAGES-deep shared-memory ring guarded by mbarriers)
//   warp 5(+4) : tcgen05.mma issuer (one elected thread)
// TMEM holds two 256-column fp32 accumulators (512 columns), so the epilogue
// of tile i overlaps the main loop of tile i+1.
//
// CG = 2 runs the same pipeline on a CTA pair (cluster of 2 on one TPC) with
// tcgen05.mma.cta_group::2: a 256-row tile, each CTA stages its own 128 rows
// of the activation and HALF of the B operand, the leader CTA issues the
// MMAs for both, and both CTAs drain their own TMEM.  Per SM this halves the
// B-operand bytes per k-step (32 KiB instead of 48 KiB), which buys a deeper
// TMA ring for the same shared memory.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <mutex>
#include <vector>

#include "lora_kernels.h"
#include "sm100_ptx.cuh"

namespace lora_sm100 {

constexpr int BM = 128;            // rows per CTA (UMMA M per CTA)
constexpr int BK = 64;             // k-block: 64 bf16 = one 128-byte swizzle row
constexpr int UMMA_K = 16;         // K per tcgen05.mma kind::f16
constexpr int NT = 256;            // TMEM columns per accumulator buffer
constexpr int NUM_THREADS = 192;   // 6 warps
// dX dropout mode (r_pad 16): 4 more epilogue warps drain the upper half of every
// tile's columns (the CUDA-core q M . (gh A) term doubles the drain; registers
// allow the extra warps only at r_pad 16)
template <int MODE, int R_PAD>
struct EpiHelpers {
    static constexpr int WARPS = (MODE == kModeDxDrop && R_PAD == 16) ? 4 : 0;
    static constexpr int THREADS = NUM_THREADS + 32 * WARPS;
};
constexpr int SMEM_LIMIT = 227 * 1024;
constexpr int DX_BN0 = 128;        // dx: width of the first (gh-producing) column tile

__host__ __device__ constexpr int round_up(int v, int a) { return (v + a - 1) / a * a; }
__host__ __device__ constexpr int cmin(int a, int b) { return a < b ? a : b; }
__host__ __device__ constexpr int cmax(int a, int b) { return a > b ? a : b; }

#ifndef LORA_STAGES_CAP
#define LORA_STAGES_CAP 8
#endif
#ifndef LORA_DROP_FHFMA  // 0: the dropout dX epilogue widens A to fp32 and uses FFMA2 (comparison)
#define LORA_DROP_FHFMA 1
#endif
#ifndef LORA_TMA_STORE   // 0: the epilogue stores y / dX with per-thread 16-byte stores (comparison)
#define LORA_TMA_STORE 1
#endif

template <int MODE, int R_PAD, int CG>
struct GemmCfg {
    // fwd: BN + r_pad = 256 (h shares the accumulator); dx: 256 (gh in the first tile)
    static constexpr int BN = (MODE == kModeFwd) ? NT - R_PAD : NT;
    static constexpr int BNH = BN / CG;                           // B-operand columns per CTA
    static constexpr int A_BYTES = BM * BK * 2;                   // activation tile (16 KiB)
    static constexpr int NBH = (BNH + 63) / 64;                   // dx: MN-major W0 64-col blocks per CTA
    static constexpr int B_BYTES = (MODE == kModeFwd) ? (NT / CG) * BK * 2 : NBH * 64 * BK * 2;
    // dx narrow operand (first column tile only): B [m, r] rows k0..k0+63, NAR columns
    // split over the pair; MN-major, swizzle = NAR_H * 2 bytes (32 / 64 / 128)
    static constexpr int NAR = (MODE == kModeFwd) ? 0 : (CG == 2 ? cmax(32, R_PAD) : R_PAD);
    static constexpr int NAR_H = NAR / CG;
    static constexpr int NAR_BYTES = BK * NAR_H * 2;
    static constexpr uint32_t NAR_LAYOUT =
        NAR_H * 2 == 32 ? kLayoutSW32 : (NAR_H * 2 == 64 ? kLayoutSW64 : kLayoutSW128);
    static constexpr int STAGE_BYTES = A_BYTES + B_BYTES + NAR_BYTES;
    static constexpr int TAIL_ROW = R_PAD * 2;                    // 32 / 64 / 128 bytes
    static constexpr uint32_t TAIL_LAYOUT =
        TAIL_ROW == 32 ? kLayoutSW32 : (TAIL_ROW == 64 ? kLayoutSW64 : kLayoutSW128);
    // tail B operand per CTA: fwd = B rows [BNH x R_PAD] K-major (swizzle = row size);
    //                         dx  = A [R_PAD x NBH*64] MN-major, 64-column SW128 blocks
    // (dx dropout mode: each CTA holds A for the FULL tile width -- its epilogue applies it on the CUDA cores)
    static constexpr int TAILB_BYTES = (MODE == kModeFwd) ? BNH * TAIL_ROW
                                                          : (MODE == kModeDxDrop ? NT / 64 : NBH) * R_PAD * 128;
    static constexpr int SH_BYTES = BM * TAIL_ROW;                // bf16(s h) / bf16(gh) tile
    static constexpr int BAR_BYTES = 1024;
    static constexpr int TAIL_BUFS = (MODE == kModeDxDrop) ? 2 : 1;   // dropout: double-buffered A tile
    static constexpr int FIXED0 = TAIL_BUFS * round_up(TAILB_BYTES, 1024) + round_up(SH_BYTES, 1024) +
                                  BAR_BYTES + 1024 /* alignment slack */;
    // TMA-store epilogue: 8 KiB staging buffers ([128 rows][32 columns] bf16, SW64),
    // two when they cost no pipeline stage, else one, else none (per-thread stores)
    static constexpr int STG_BYTES = BM * 32 * 2;
    static constexpr int STAGES0 = cmin(LORA_STAGES_CAP, (SMEM_LIMIT - FIXED0) / STAGE_BYTES);
    static constexpr int STG_BUFS = !LORA_TMA_STORE ? 0
        : (cmin(LORA_STAGES_CAP, (SMEM_LIMIT - FIXED0 - 2 * STG_BYTES) / STAGE_BYTES) == STAGES0 ? 2
        : (cmin(LORA_STAGES_CAP, (SMEM_LIMIT - FIXED0 - STG_BYTES) / STAGE_BYTES) == STAGES0 ? 1 : 0));
    static constexpr bool STORE_TMA = STG_BUFS > 0;
    static constexpr int FIXED = FIXED0 + STG_BUFS * STG_BYTES;
    static constexpr int STAGES = cmin(LORA_STAGES_CAP, (SMEM_LIMIT - FIXED) / STAGE_BYTES);
    static constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + FIXED;
    static_assert(STAGES >= 2, "shared memory budget");
    // stream-K owners stage a contributor's partial in the idle ring (else: no stream-K)
    static constexpr bool SK_OK = STAGES * STAGE_BYTES >= kPartialFloatsPerCta * 4;
    static_assert(BN % 16 == 0 && BN >= 16 && BN <= 256, "UMMA N");
    static_assert(CG == 1 || (BN > 128 && R_PAD % 16 == 0), "2-CTA split");
    static_assert(MODE == kModeFwd || DX_BN0 + NAR <= NT, "gh columns fit next to the first tile");
};

// Column tiling.  fwd: uniform BN-wide tiles.  dx: tile 0 is DX_BN0 wide (and
// computes gh), tiles 1.. are BN wide starting at DX_BN0 (so every 64-column
// W0 / A box starts 128-byte aligned).
template <int MODE, int BN>
struct ColTiles {
    __device__ static int count(int64_t n_out) {
        if (MODE == kModeFwd) return static_cast<int>((n_out + BN - 1) / BN);
        return n_out <= DX_BN0 ? 1 : 1 + static_cast<int>((n_out - DX_BN0 + BN - 1) / BN);
    }
    __device__ static int start(int n_blk) {
        if (MODE == kModeFwd) return n_blk * BN;
        return n_blk == 0 ? 0 : DX_BN0 + (n_blk - 1) * BN;
    }
    // dx: the last tile is only as wide as the columns left (rounded up to 128, so each
    // CTA of a pair still holds whole 64-column blocks): its MMAs run at N = 128, not 256
    __device__ static int width(int n_blk, int64_t n_out) {
        if (MODE == kModeFwd) return BN;
        if (n_blk == 0) return DX_BN0;
        const int64_t left = (n_out - start(n_blk) + 127) / 128 * 128;
        return left < BN ? static_cast<int>(left) : BN;
    }
};

// 2-CTA helpers ---------------------------------------------------------------
__device__ __forceinline__ uint32_t cluster_ctarank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// arrive on the barrier at the same shared-memory offset in CTA `cta` of the cluster
__device__ __forceinline__ void mbar_arrive_cluster(uint64_t* bar, uint32_t cta) {
    asm volatile(
        "{\n\t.reg .b32 ra;\n\t"
        "mapa.shared::cluster.u32 ra, %0, %1;\n\t"
        "mbarrier.arrive.release.cluster.shared::cluster.b64 _, [ra];\n\t}\n"
        ::"r"(smem_u32(bar)), "r"(cta) : "memory");
}
template <int CG>
__device__ __forceinline__ void tma_load(void* dst, const CUtensorMap* map, int32_t c0, int32_t c1, uint64_t* bar) {
    if constexpr (CG == 1) {
        tma_load_2d(dst, map, c0, c1, bar);
    } else {
        // both CTAs complete their bytes on the LEADER's barrier (peer bit cleared)
        asm volatile(
            "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
            " [%0], [%1, {%2, %3}], [%4];"
            ::"r"(smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1),
              "r"(smem_u32(bar) & 0xFEFFFFFFu)
            : "memory");
    }
}
template <int CG>
__device__ __forceinline__ void umma(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    if constexpr (CG == 1) {
        umma_f16(d, a, b, idesc, acc);
    } else {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "setp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}\n"
            ::"r"(d), "l"(a), "l"(b), "r"(idesc), "r"(acc) : "memory");
    }
}
// commit this thread's outstanding tcgen05 ops to `bar` (CG = 2: in both CTAs)
template <int CG>
__device__ __forceinline__ void commit(uint64_t* bar) {
    if constexpr (CG == 1) {
        umma_commit(bar);
    } else {
        asm volatile(
            "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
            ::"r"(smem_u32(bar)), "h"(static_cast<uint16_t>(3)) : "memory");
    }
}
template <int CG>
__device__ __forceinline__ void tmem_alloc_cg(uint32_t* dst) {
    if constexpr (CG == 1) {
        tmem_alloc<512>(dst);
    } else {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(dst))
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    }
}
template <int CG>
__device__ __forceinline__ void tmem_dealloc_cg(uint32_t taddr) {
    if constexpr (CG == 1) {
        tmem_dealloc<512>(taddr);
    } else {
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(taddr) : "memory");
    }
}

// Tile `tile` of a group -> (problem g, row block, column block, k-blocks).
struct TileRef {
    int g, t_blk, n_blk, num_k_blks;
};
template <int TM>
__device__ __forceinline__ TileRef decode_tile(const FusedGemmGroup& grp, int tile) {
    int g = 0;
    while (g + 1 < grp.count && tile >= grp.tile_start[g + 1]) ++g;
    const FusedGemmParams& p = grp.p[g];
    const int local = tile - grp.tile_start[g];
    const int num_t_blks = static_cast<int>((p.T + TM - 1) / TM);
    TileRef t;
    t.g = g;
    t.n_blk = local / num_t_blks;
    t.t_blk = local - t.n_blk * num_t_blks;
    t.num_k_blks = static_cast<int>((p.K + BK - 1) / BK);
    return t;
}

// Rank-r rows of a row-major fp32 [T, r] array (h saved by the forward) for the
// 32 token rows row0 .. row0+31 of a warp: lane L receives row row0+L.  A plain
// per-lane row read strides the warp by 4r bytes (one sector per value); here the
// warp reads its 32 r contiguous floats with coalesced 16-byte loads (r % 4 == 0,
// r <= 16: at most 4 rounds) and transposes them with shuffles -- the register
// component (j % 4) is uniform across lanes, only the source lane and round vary.
template <int R_PAD>
__device__ __forceinline__ void warp_load_rows(const float* base, int64_t row0, int64_t T, int r, uint32_t lane,
                                               float (&hv)[R_PAD]) {
    if (r % 4 == 0 && r <= 16) {
        const int64_t nvalid = (T - row0) * r;   // floats of this warp block inside the array
        const float4* b4 = reinterpret_cast<const float4*>(base + row0 * r);
        float4 v[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int64_t idx = lane + 32 * i;
            v[i] = (i < r / 4 && idx * 4 < nvalid) ? b4[idx] : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int j = 0; j < R_PAD; ++j) {
            if (j >= 16) { hv[j] = 0.0f; continue; }
            const int f4 = static_cast<int>(lane) * (r / 4) + j / 4;
            const int src = f4 & 31, rnd = f4 >> 5;
            float val = 0.0f;
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                if (i >= r / 4) break;   // (warp-uniform)
                const float c = (j & 3) == 0 ? v[i].x : (j & 3) == 1 ? v[i].y : (j & 3) == 2 ? v[i].z : v[i].w;
                const float t = __shfl_sync(0xffffffffu, c, src);
                if (rnd == i) val = t;
            }
            hv[j] = j < r ? val : 0.0f;
        }
        return;
    }
    const int64_t row = row0 + lane;
#pragma unroll
    for (int j = 0; j < R_PAD; ++j) hv[j] = (j < r && row < T) ? base[row * r + j] : 0.0f;
}
// The transpose of warp_load_rows: lane L holds row row0+L's values; the warp
// stores its 32 r floats with coalesced 16-byte stores (r % 4 == 0, r <= 16).
template <int R_PAD>
__device__ __forceinline__ void warp_store_rows(float* base, int64_t row0, int64_t T, int r, uint32_t lane,
                                                const float (&hv)[R_PAD]) {
    if (r % 4 == 0 && r <= 16) {
        const int64_t nvalid = (T - row0) * r;
        float4* b4 = reinterpret_cast<float4*>(base + row0 * r);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            if (i >= r / 4) break;   // (warp-uniform)
            const int q = static_cast<int>(lane) + 32 * i;   // float4 index in the warp block
            const int srow = (4 * q) / r, g = ((4 * q) % r) / 4;   // source lane, column group
            float o[4];
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                float val = 0.0f;
#pragma unroll
                for (int gg = 0; gg < 4; ++gg) {
                    if (4 * gg + c >= R_PAD || gg >= r / 4) break;
                    const float t = __shfl_sync(0xffffffffu, hv[4 * gg + c], srow);
                    if (g == gg) val = t;
                }
                o[c] = val;
            }
            if (static_cast<int64_t>(q) * 4 < nvalid) b4[q] = make_float4(o[0], o[1], o[2], o[3]);
        }
        return;
    }
    const int64_t row = row0 + lane;
    if (row < T) {
#pragma unroll
        for (int j = 0; j < R_PAD; ++j)
            if (j < r) base[row * r + j] = hv[j];
    }
}

#ifdef LORA_PROBE_SK
__device__ unsigned int g_probe_n;
__device__ unsigned long long g_probe_buf[4 * 4096];
#endif

// ---------------------------------------------------------------- schedule
// One unit of a pair's work: k-blocks [kb0, kb1) of tile (g, t_blk, n_blk).
enum : int { kUnitFull = 0, kUnitOwner = 1, kUnitPart = 2 };
struct Unit {
    int g, t_blk, n_blk, kb0, kb1, kbt, role;
    int64_t a;   // stream-K: cost offset of the tile on the body line
    int w;       // stream-K: cost of one k-block of the tile (width / 128)
};

template <int MODE, int CG>
struct Sched {
    // tail tile i -> unit skeleton (tile coordinates, cost line offset, cost per k-block)
    __device__ static Unit tail_unit(const FusedGemmGroup& grp, int i) {
        const TileRef tr = decode_tile<BM * CG>(grp, grp.sk.D + i);
        Unit u;
        u.g = tr.g; u.t_blk = tr.t_blk; u.n_blk = tr.n_blk; u.kbt = tr.num_k_blks;
        u.a = grp.sk.prefix[i];
        u.w = (grp.sk.prefix[i + 1] - grp.sk.prefix[i]) / tr.num_k_blks;
        u.kb0 = u.kb1 = 0;
        u.role = kUnitFull;
        return u;
    }
    // the tail tile containing cost offset x (binary search on the prefix)
    __device__ static int tail_find(const StreamKSched& sk, int x) {
        int lo = 0, hi = sk.ntail - 1;
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (sk.prefix[mid] <= x) lo = mid; else hi = mid - 1;
        }
        return lo;
    }
    // k-block range of tail tile `u` that pair q holds
    __device__ static void seg(const StreamKSched& sk, const Unit& u, int q, int* kb0, int* kb1) {
        const int64_t lo = sk.S[q] > u.a ? sk.S[q] - u.a : 0;
        const int64_t hi = static_cast<int64_t>(sk.S[q + 1]) - u.a;
        int b = static_cast<int>((lo + u.w - 1) / u.w);
        int e = hi <= 0 ? 0 : static_cast<int>((hi + u.w - 1) / u.w);
        *kb0 = b < u.kbt ? b : u.kbt;
        *kb1 = e < u.kbt ? e : u.kbt;
    }
};

// Iterates pair q's units; every warp role walks the same sequence.  Order:
// its dx gh tiles, then its split-off tail segment (a partial for another
// pair: short, never waits, and its fp32 drain hides under the next mainloop),
// then its other data-parallel tiles, then the rest of its tail range (which
// ends with the segment it owns, if any).
template <int MODE, int CG, int BN>
struct UnitIter {
    using SC = Sched<MODE, CG>;
    const FusedGemmGroup& grp;
    int q, npairs, jA, jB, phase;
    int x;                 // stream-K tail cursor
    __device__ UnitIter(const FusedGemmGroup& gr, int pair, int np)
        : grp(gr), q(pair), npairs(np), jA(pair), jB(pair), phase(0) {
        x = grp.sk.enabled ? grp.sk.S[pair] : 0;
    }
    __device__ void dp_unit(Unit& u, int tile) {
        const TileRef tr = decode_tile<BM * CG>(grp, tile);
        u.g = tr.g; u.t_blk = tr.t_blk; u.n_blk = tr.n_blk;
        u.kb0 = 0; u.kb1 = u.kbt = tr.num_k_blks; u.role = kUnitFull; u.a = 0; u.w = 0;
    }
    // first non-empty tail unit at or after x (does not advance x)
    __device__ bool tail_peek(Unit& u, int& x_next) {
        int xx = x;
        while (xx < grp.sk.S[q + 1]) {
            const int i = SC::tail_find(grp.sk, xx);
            u = SC::tail_unit(grp, i);
            SC::seg(grp.sk, u, q, &u.kb0, &u.kb1);
            xx = grp.sk.prefix[i + 1];
            if (u.kb1 <= u.kb0) continue;
            u.role = u.kb0 > 0 ? kUnitPart : (u.kb1 < u.kbt ? kUnitOwner : kUnitFull);
            x_next = xx;
            return true;
        }
        x_next = xx;
        return false;
    }
    __device__ bool next(Unit& u) {
        if (!grp.sk.enabled) {
            if (jB >= grp.tile_start[grp.count]) return false;
            dp_unit(u, jB);
            jB += npairs;
            return true;
        }
        const int D = grp.sk.D;
        if (phase == 0) {   // gh tiles (dx) of the data-parallel part
            while (MODE != kModeFwd && jA < D) {
                const int t = jA;
                jA += npairs;
                dp_unit(u, t);
                if (u.n_blk == 0) return true;
            }
            phase = 1;
        }
        if (phase == 1) {   // the split-off segment of the tail, first
            phase = 2;
            int xn;
            if (tail_peek(u, xn) && u.role == kUnitPart) {
                x = xn;
                return true;
            }
        }
        if (phase == 2) {   // the other data-parallel tiles
            while (jB < D) {
                const int t = jB;
                jB += npairs;
                dp_unit(u, t);
                if (MODE == kModeFwd || u.n_blk != 0) return true;
            }
            phase = 3;
        }
        int xn;
        if (!tail_peek(u, xn)) return false;
        x = xn;
        return true;
    }
};

// Dropout dX epilogue term of one row and 16 columns: lo[e] = sum_j bf16(q gh_j) A[j, c + e]
// with FHFMA.BF16 (fp32 accumulate, A straight from its bf16 halves in the MN-major SW128
// A tile `blk`, chunk ch of its 128-byte rows)
template <int R_PAD>
__device__ __forceinline__ void drop_term16(const uint32_t (&gq)[R_PAD], const uint8_t* blk, uint32_t ch, int r,
                                            float (&lo)[16]) {
#pragma unroll
    for (int e = 0; e < 16; ++e) lo[e] = 0.0f;
#pragma unroll
    for (int j = 0; j < R_PAD; ++j) {
#ifdef LORA_PROBE_DROP_NOFMA
        break;   // timing experiment only: no q M . (gh A) term
#endif
        if (j >= r) break;   // (uniform) rows r..r_pad-1 of A are zero
        const uint4 a0 = *reinterpret_cast<const uint4*>(blk + swizzled_offset(j, ch, 128));
        const uint4 a1 = *reinterpret_cast<const uint4*>(blk + swizzled_offset(j, ch + 1, 128));
        const uint32_t aw[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
#pragma unroll
        for (int e = 0; e < 8; ++e) fma_bf16_pair(gq[j], aw[e], lo[2 * e], lo[2 * e + 1]);
    }
}

// Maps per problem g (grp.maps[g]):
//   act  x or dY [T, K]          w   W0 [m, n] (fwd CG=2: 128-row box)
//   w2   fwd CG=2: W0 box of BN-128 rows
//   nar  fwd: A [r,n]; dx: B [m,r8]          tail  fwd: B [m,r8]; dx: A [r,n]
template <int MODE, int R_PAD, int CG>
__global__ void __launch_bounds__(EpiHelpers<MODE, R_PAD>::THREADS, 1)
lora_fused_gemm_kernel(const __grid_constant__ FusedGemmGroup grp) {
    using C = GemmCfg<MODE, R_PAD, CG>;
    using Cols = ColTiles<MODE, C::BN>;
    constexpr int BN = C::BN;
    constexpr int TM = BM * CG;                    // rows per tile

    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* stage_base = smem;
    uint8_t* s_tailb = smem + C::STAGES * C::STAGE_BYTES;
    uint8_t* s_h = s_tailb + C::TAIL_BUFS * round_up(C::TAILB_BYTES, 1024);
    uint8_t* s_stg = s_h + round_up(C::SH_BYTES, 1024);            // TMA-store staging (STG_BUFS x 8 KiB)
    uint64_t* bars = reinterpret_cast<uint64_t*>(s_stg + C::STG_BUFS * C::STG_BYTES);
    uint64_t* full = bars;
    uint64_t* empty = bars + C::STAGES;
    uint64_t* tmem_full = bars + 2 * C::STAGES;
    uint64_t* tmem_empty = tmem_full + 2;
    uint64_t* tailop_full = tmem_empty + 2;
    uint64_t* tailop_empty = tailop_full + 1;
    uint64_t* tail_done = tailop_empty + 1;
    uint64_t* sh_full = tail_done + 1;             // CG = 2: peer's s_h tile written
    uint64_t* tailop2_full = sh_full + 1;          // dx dropout mode: second A-tile buffer
    uint64_t* tailop2_empty = tailop2_full + 1;
    uint64_t* part_full = tailop2_empty + 1;       // stream-K owner: first contributor's partial in the ring
    uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(part_full + 1);

    const uint32_t crank = (CG == 2) ? cluster_ctarank() : 0;
    const bool leader = crank == 0;
    const int pair = static_cast<int>(blockIdx.x) / CG;
    const int npairs = static_cast<int>(gridDim.x) / CG;
    const uint32_t warp = warp_id();
    const uint32_t lane = lane_id();

    // Warp roles.  The SM sub-partition's scheduler favours the highest warp id among
    // eligible warps, so the TMA producer and the MMA issuer take the two HIGHEST ids
    // (no epilogue warp -- all of them busy on the CUDA cores in the dropout dX mode --
    // can delay an MMA issue or a TMA refill): epilogue warps 0..3 (TMEM lane quarter =
    // warp & 3), drain helpers 4..4+H-1 (dropout dX), producer 4+H, MMA issuer 5+H.
    constexpr uint32_t kHelp = EpiHelpers<MODE, R_PAD>::WARPS;
    constexpr uint32_t W_PROD = 4 + kHelp, W_MMA = 5 + kHelp;
    if (warp == W_PROD && lane < static_cast<uint32_t>(grp.count)) {
        const FusedGemmMaps& mp = grp.maps[lane];
        tma_prefetch_desc(&mp.act);
        tma_prefetch_desc(&mp.w);
        if (MODE == kModeFwd && CG == 2) tma_prefetch_desc(&mp.w2);
        tma_prefetch_desc(&mp.nar);
        tma_prefetch_desc(&mp.tail);
        if (C::STORE_TMA) {
            tma_prefetch_desc(&mp.out32);
            tma_prefetch_desc(&mp.out16);
        }
    }
    if (warp == W_MMA && lane == 0) {
        for (int s = 0; s < C::STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&tmem_full[a], 1);
            mbar_init(&tmem_empty[a], 4 * CG);  // one arrive per epilogue warp of the pair
        }
        mbar_init(tailop_full, 1);
        mbar_init(tailop_empty, 1);
        mbar_init(tailop2_full, 1);
        mbar_init(tailop2_empty, 1);
        mbar_init(tail_done, 1);
        mbar_init(sh_full, 1);
        mbar_init(part_full, 1);
        fence_mbar_init();
    }
    if (warp == 0) tmem_alloc_cg<CG>(tmem_holder);
    tc_fence_before();
    if constexpr (CG == 2) cluster_sync(); else __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_holder;
    // Programmatic dependent launch: everything above (barrier init, TMEM
    // allocation, descriptor prefetch) overlapped the previous kernel's tail;
    // no global memory is touched before the previous grid has completed.
    griddep_wait();
    if (threadIdx.x == 0) griddep_launch_dependents();
#if defined(LORA_PROBE_CLOCK) || defined(LORA_PROBE_SK)
    const long long probe_c0 = clock64();
    const uint64_t probe_t0 = globaltimer_ns();
    (void)probe_c0;
#endif

    if (warp == W_PROD) {
        // ===================== TMA producer (both CTAs) =====================
        if (elect_one()) {
            const uint64_t pol_w = l2_policy_evict_last();
            uint32_t stage = 0, phase = 0, tl = 0, tt = 0;
            UnitIter<MODE, CG, BN> it(grp, pair, npairs);
            Unit un;
            for (; it.next(un); ++tl) {
                const FusedGemmMaps& mp = grp.maps[un.g];
                const int n_blk = un.n_blk;
                const int t_blk = un.t_blk;
                const int t0 = t_blk * TM + static_cast<int>(crank) * BM;
                const int n0 = Cols::start(n_blk);
                const int wh = Cols::width(n_blk, grp.p[un.g].N_out) / CG;   // this CTA's B-operand columns
                const int nh0 = n0 + static_cast<int>(crank) * wh;
                const int nb = (wh + 63) / 64;                          // dx: 64-column W0 / A blocks
                const bool gh_tile = (MODE != kModeFwd) && n_blk == 0;
                const uint32_t stage_tx = (MODE == kModeFwd)
                    ? static_cast<uint32_t>(C::STAGE_BYTES)
                    : static_cast<uint32_t>(C::A_BYTES + nb * 64 * BK * 2 + (gh_tile ? C::NAR_BYTES : 0));
                for (int kb = un.kb0; kb < un.kb1; ++kb) {
                    mbar_wait(&empty[stage], phase ^ 1);
                    uint8_t* sA = stage_base + stage * C::STAGE_BYTES;
                    uint8_t* sB = sA + C::A_BYTES;
#ifdef LORA_PROBE_NO_REFILL
                    // timing experiment only: after the first fill the MMAs re-read stale tiles
                    if (tl > 0 || kb >= C::STAGES) {
                        if (leader) mbar_arrive(&full[stage]);
                        if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
                        continue;
                    }
#endif
                    if (leader) mbar_arrive_expect_tx(&full[stage], CG * stage_tx);
                    const int k0 = kb * BK;
                    tma_load<CG>(sA, &mp.act, k0, t0, &full[stage]);
                    if constexpr (MODE == kModeFwd) {
                        if (CG == 1) {
                            tma_load_2d_hint(sB, &mp.w, k0, n0, &full[stage], pol_w);       // W0 rows
                            tma_load<CG>(sB + BN * 128, &mp.nar, k0, 0, &full[stage]);        // A rows
                        } else if (crank == 0) {
                            tma_load<CG>(sB, &mp.w, k0, n0, &full[stage]);                    // W0 rows 0..127
                        } else {
                            tma_load<CG>(sB, &mp.w2, k0, n0 + 128, &full[stage]);             // W0 rows 128..BN-1
                            tma_load<CG>(sB + (BN - 128) * 128, &mp.nar, k0, 0, &full[stage]); // A rows
                        }
                    } else {
                        for (int j = 0; j < nb; ++j)
                            tma_load<CG>(sB + j * (64 * 128), &mp.w, nh0 + 64 * j, k0, &full[stage]);
                        if (gh_tile)   // B rows k0..k0+63, this CTA's NAR_H columns
                            tma_load<CG>(sB + C::B_BYTES, &mp.nar, static_cast<int>(crank) * C::NAR_H, k0,
                                         &full[stage]);
                    }
                    if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
                }
                // tail operand for this tile: fwd B rows; dx A columns (this CTA's half).
                // Stream-K partial segments have no tail (the owner adds the LoRA term).
                if (un.role == kUnitPart) continue;
                if constexpr (MODE != kModeDxDrop) mbar_wait(tailop_empty, (tt & 1) ^ 1);
                if constexpr (MODE == kModeFwd) {
                    if (leader) mbar_arrive_expect_tx(tailop_full, CG * C::TAILB_BYTES);
                    tma_load<CG>(s_tailb, &mp.tail, 0, nh0, tailop_full);
                } else if constexpr (MODE == kModeDxDrop) {
                    // every CTA: A columns of the whole tile width, on its own barrier, into
                    // buffer tt & 1 (the epilogue holds a buffer for its whole drain)
                    uint64_t* tf = (tt & 1) ? tailop2_full : tailop_full;
                    mbar_wait((tt & 1) ? tailop2_empty : tailop_empty, ((tt >> 1) & 1) ^ 1);
                    uint8_t* tb = s_tailb + (tt & 1) * round_up(C::TAILB_BYTES, 1024);
                    const int nbf = (Cols::width(n_blk, grp.p[un.g].N_out) + 63) / 64;
                    mbar_arrive_expect_tx(tf, nbf * R_PAD * 128);
                    for (int j = 0; j < nbf; ++j)
                        tma_load_2d(tb + j * (R_PAD * 128), &mp.tail, n0 + 64 * j, 0, tf);
                } else {
                    if (leader) mbar_arrive_expect_tx(tailop_full, CG * nb * R_PAD * 128);
                    for (int j = 0; j < nb; ++j)
                        tma_load<CG>(s_tailb + j * (R_PAD * 128), &mp.tail, nh0 + 64 * j, 0, tailop_full);
                }
                ++tt;
            }
        }
    } else if (warp == W_MMA) {
        // ===================== MMA issuer (leader CTA) =====================
        if (leader && elect_one()) {
            constexpr uint32_t idesc_fwd = make_idesc_bf16(TM, NT, 0, 0);
            constexpr uint32_t idesc_nar = make_idesc_bf16(TM, C::NAR > 0 ? C::NAR : 16, 0, 1);
            uint32_t stage = 0, phase = 0, tl = 0;
            UnitIter<MODE, CG, BN> it(grp, pair, npairs);
            Unit un;
            for (; it.next(un); ++tl) {
                const int n_blk = un.n_blk;
                const bool gh_tile = (MODE != kModeFwd) && n_blk == 0;
                const uint32_t idesc_main = (MODE == kModeFwd)
                    ? idesc_fwd
                    : make_idesc_bf16(TM, static_cast<uint32_t>(Cols::width(n_blk, grp.p[un.g].N_out)), 0, 1);
                const uint32_t acc = tl & 1;
                const uint32_t acc_phase = (tl >> 1) & 1;
                mbar_wait<CG == 2>(&tmem_empty[acc], acc_phase ^ 1);
                tc_fence_after();
                const uint32_t d_tmem = tmem_base + acc * NT;
                for (int kb = un.kb0; kb < un.kb1; ++kb) {
                    mbar_wait(&full[stage], phase);
                    tc_fence_after();
                    const uint32_t a_addr = smem_u32(stage_base + stage * C::STAGE_BYTES);
                    const uint32_t b_addr = a_addr + C::A_BYTES;
#pragma unroll
                    for (int kk = 0; kk < BK / UMMA_K; ++kk) {
                        const uint32_t accum = (kb != un.kb0 || kk != 0) ? 1u : 0u;
                        const uint64_t a_desc = make_smem_desc(a_addr + kk * 32, 16, 1024, kLayoutSW128);
                        if constexpr (MODE == kModeFwd) {
                            // [W0 rows ; A rows] as one K-major N = 256 operand
                            const uint64_t b_desc = make_smem_desc(b_addr + kk * 32, 16, 1024, kLayoutSW128);
                            umma<CG>(d_tmem, a_desc, b_desc, idesc_main, accum);
                        } else {
                            // W0 MN-major: 64-column blocks at LBO = 8 KiB, 8-row k groups at SBO = 1 KiB
                            const uint64_t b_desc = make_smem_desc(b_addr + kk * (UMMA_K * 128), 64 * 128,
                                                                   1024, kLayoutSW128);
                            umma<CG>(d_tmem, a_desc, b_desc, idesc_main, accum);
                            if (gh_tile) {
                                // dY B: one MN-major atom of NAR_H columns per CTA, SBO = 8 rows
                                const uint64_t n_desc = make_smem_desc(
                                    b_addr + C::B_BYTES + kk * (UMMA_K * C::NAR_H * 2), 16, 8 * C::NAR_H * 2,
                                    C::NAR_LAYOUT);
                                umma<CG>(d_tmem + DX_BN0, a_desc, n_desc, idesc_nar, accum);
                            }
                        }
                    }
                    commit<CG>(&empty[stage]);  // frees the smem slot(s) when these MMAs finish
                    if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
                }
                commit<CG>(&tmem_full[acc]);
            }
        }
    } else if (warp >= 4) {
        // ===================== dropout dX drain helpers (warps 4..7, both CTAs) =====================
        // Same rows as epilogue warp (warp - 4) (same TMEM lane quarter); per tile: the row's
        // gh (TMEM for the gh tile, else the published split rows), bf16(q gh), then the
        // upper half of the tile's 16-column chunks; a 256-thread barrier with the epilogue
        // warps releases the A tile and the accumulator.  (Stream-K off: the schedule only.)
        if constexpr (EpiHelpers<MODE, R_PAD>::WARPS > 0 && !C::STORE_TMA) {
            if (!grp.sk.enabled) {
                const uint32_t quarter = warp & 3;
                const uint32_t row_local = quarter * 32 + lane;
                uint32_t tl = 0, tt = 0;
                UnitIter<MODE, CG, BN> it(grp, pair, npairs);
                Unit un;
                for (; it.next(un); ++tl, ++tt) {
                    const FusedGemmParams& p = grp.p[un.g];
                    const int n_blk = un.n_blk;
                    const int t_blk = un.t_blk;
                    const int64_t row = static_cast<int64_t>(t_blk) * TM + crank * BM + row_local;
                    const int n0 = Cols::start(n_blk);
                    const int width = Cols::width(n_blk, p.N_out);
                    const uint32_t acc = tl & 1;
                    mbar_wait(&tmem_full[acc], (tl >> 1) & 1);
                    tc_fence_after();
                    const uint32_t tbase = tmem_base + ((quarter * 32) << 16) + acc * NT;
                    float hv[R_PAD];
                    if (n_blk == 0) {
#pragma unroll
                        for (int c = 0; c < R_PAD / 16; ++c) {
                            uint32_t v[16];
                            tmem_ld_32x32b_x16(tbase + DX_BN0 + 16 * c, v);
                            tmem_ld_wait();
#pragma unroll
                            for (int e = 0; e < 16; ++e) hv[16 * c + e] = p.scale * __uint_as_float(v[e]);
                        }
                    } else {
                        const uint64_t* flag = p.flags + static_cast<int64_t>(t_blk) * CG + crank;
                        const uint64_t t_start = globaltimer_ns();
                        while (ld_acquire_u64(flag) != p.epoch) {
                            __nanosleep(64);
                            if (globaltimer_ns() - t_start > kWaitTimeoutNs) {
                                printf("lora dX kernel: gh flag wait timed out (row block %d)\n", t_blk);
                                __trap();
                            }
                        }
                        const int r8 = (p.r + 7) / 8 * 8;
#pragma unroll
                        for (int j = 0; j < R_PAD; ++j) {
                            float v = 0.0f;
                            if (j < p.r && row < p.T) {
                                const __nv_bfloat16* c = p.cs_gh + static_cast<int64_t>(j) * p.t_pad + row;
                                v = (__bfloat162float(c[0]) + __bfloat162float(c[static_cast<int64_t>(r8) * p.t_pad])) +
                                    __bfloat162float(c[static_cast<int64_t>(2 * r8) * p.t_pad]);
                            }
                            hv[j] = v;
                        }
                    }
                    uint32_t gq[R_PAD];
#pragma unroll
                    for (int j = 0; j < R_PAD; ++j)
                        gq[j] = static_cast<uint32_t>(__bfloat16_as_ushort(__float2bfloat16_rn(p.drop.q * hv[j])));
                    mbar_wait((tt & 1) ? tailop2_full : tailop_full, (tt >> 1) & 1);
                    const bool row_ok = row < p.T;
                    __nv_bfloat16* out_row = p.out + row * p.N_out;
                    const int nc = width / 16, c_split = (nc + 1) / 2;
                    const int64_t nw = (p.N_out + 31) / 32;
#pragma unroll 1
                    for (int c = c_split; c < nc; ++c) {
                        uint32_t v[16];
                        tmem_ld_32x32b_x16(tbase + 16 * c, v);
                        tmem_ld_wait();
                        const int64_t col = n0 + 16 * c;
                        if (!(row_ok && col < p.N_out)) continue;   // (after the warp-wide TMEM load)
                        const uint32_t kword = p.drop_bits[row * nw + col / 32];
                        float f[16];
#pragma unroll
                        for (int e = 0; e < 16; ++e) f[e] = __uint_as_float(v[e]);
                        const int lc = 16 * c;
                        const uint8_t* blk = s_tailb + (tt & 1) * round_up(C::TAILB_BYTES, 1024) +
                                             (lc / 64) * (R_PAD * 128);
                        const uint32_t ch = static_cast<uint32_t>((lc % 64) / 8);
                        float lo[16];
                        drop_term16<R_PAD>(gq, blk, ch, p.r, lo);
                        const uint32_t keep = (kword >> ((c & 1) * 16)) & 0xFFFFu;
#pragma unroll
                        for (int e = 0; e < 16; ++e)
                            if ((keep >> e) & 1u) f[e] += lo[e];
                        uint4 q0, q1;
                        q0.x = pack_bf16x2(f[0], f[1]);   q0.y = pack_bf16x2(f[2], f[3]);
                        q0.z = pack_bf16x2(f[4], f[5]);   q0.w = pack_bf16x2(f[6], f[7]);
                        q1.x = pack_bf16x2(f[8], f[9]);   q1.y = pack_bf16x2(f[10], f[11]);
                        q1.z = pack_bf16x2(f[12], f[13]); q1.w = pack_bf16x2(f[14], f[15]);
                        *reinterpret_cast<uint4*>(out_row + col) = q0;
                        if (col + 8 < p.N_out) *reinterpret_cast<uint4*>(out_row + col + 8) = q1;
                    }
                    if (p.unit_flags != nullptr) __threadfence_system();
                    tc_fence_before();
                    named_bar_sync(2, 32 * (4 + EpiHelpers<MODE, R_PAD>::WARPS));   // with the epilogue warps
                }
            }
        }
    } else {
        // ===================== epilogue (warps 0..3, both CTAs) =====================
        const uint32_t ew = warp;                // epilogue warp index 0..3
        const uint32_t quarter = warp & 3;       // TMEM lane quarter this warp may access
        const uint32_t row_local = quarter * 32 + lane;
        constexpr uint32_t idesc_tail_fwd = make_idesc_bf16(TM, BN, 0, 0);
        constexpr uint32_t tail_sbo = 8 * C::TAIL_ROW;
        uint32_t tl = 0, tt = 0;
        UnitIter<MODE, CG, BN> it(grp, pair, npairs);
        Unit un;
        for (; it.next(un); ++tl) {
            const FusedGemmParams& p = grp.p[un.g];
            const int n_blk = un.n_blk;
            const int t_blk = un.t_blk;
            const int64_t row = static_cast<int64_t>(t_blk) * TM + crank * BM + row_local;
            const int n0 = Cols::start(n_blk);
            const int width = Cols::width(n_blk, p.N_out);
            const bool gh_tile = (MODE != kModeFwd) && n_blk == 0;
            const uint32_t acc = tl & 1;
            const uint32_t acc_phase = (tl >> 1) & 1;
            mbar_wait(&tmem_full[acc], acc_phase);
            tc_fence_after();
#ifdef LORA_PROBE_SK
            const uint64_t probe_u0 = globaltimer_ns();
#endif
            const uint32_t tbase = tmem_base + ((quarter * 32) << 16) + acc * NT;
            // stream-K partial slots: [chunk of 16 columns][128 rows][16] fp32 per CTA
            constexpr int ACC_COLS = NT;   // fwd: BN output + r_pad h columns
            auto slot_of = [&](int q) {
                return grp.sk.partial + static_cast<int64_t>(q * CG + static_cast<int>(crank)) * kPartialFloatsPerCta;
            };
            if (un.role == kUnitPart) {
                // (P) a split-off segment: raw fp32 accumulator -> this pair's slot, then publish
                float* slot = slot_of(pair);
                const int ncol = (MODE == kModeFwd) ? ACC_COLS : width;
#pragma unroll 1
                for (int c = 0; c < ncol / 16; ++c) {
                    uint32_t v[16];
                    tmem_ld_32x32b_x16(tbase + 16 * c, v);
                    tmem_ld_wait();
                    // [chunk][4 float4 groups][128 rows] float4: a warp stores 512 contiguous bytes
                    float4* dst = reinterpret_cast<float4*>(slot) + static_cast<int64_t>(c) * 512 + row_local;
#pragma unroll
                    for (int e = 0; e < 4; ++e)
                        dst[e * 128] = make_float4(__uint_as_float(v[4 * e]), __uint_as_float(v[4 * e + 1]),
                                                   __uint_as_float(v[4 * e + 2]), __uint_as_float(v[4 * e + 3]));
                }
                tc_fence_before();
                __threadfence();
                named_bar_sync(1, 128);
                if (ew == 0 && lane == 0) st_release_u64(grp.sk.pflags + pair * CG + crank, 1ull);
#ifdef LORA_PROBE_SK
                if (ew == 0 && lane == 0 && crank == 0) {
                    const unsigned i = atomicAdd(&g_probe_n, 1u);
                    if (i < 4096) {
                        unsigned long long* r = g_probe_buf + 4 * i;
                        r[0] = (static_cast<unsigned long long>(pair) << 32) | (tl << 8) | static_cast<unsigned>(un.role);
                        r[1] = (static_cast<unsigned long long>(un.kb0) << 32) | static_cast<unsigned>(un.kb1);
                        r[2] = probe_u0 - probe_t0;
                        r[3] = globaltimer_ns() - probe_t0;
                    }
                }
#endif
                __syncwarp();
                if (lane == 0) {
                    if (CG == 1) mbar_arrive(&tmem_empty[acc]);
                    else mbar_arrive_cluster(&tmem_empty[acc], 0);
                }
                continue;
            }
            // owner of a split tile: the pairs after this one hold its other k-blocks.  Its
            // segment is this pair's LAST unit, so the stage ring is idle: each contributor's
            // partial in turn is bulk-copied into it and added into the TMEM accumulator
            // (tcgen05.ld / st), in pair order, before anything reads the accumulator.
            if (un.role == kUnitOwner) {
                int cq[4];
                int ncq = 0;
                const int64_t b_end = un.a + static_cast<int64_t>(un.kbt) * un.w;
                for (int q = pair + 1; q < npairs && grp.sk.S[q] < b_end; ++q) {
                    int k0, k1;
                    Sched<MODE, CG>::seg(grp.sk, un, q, &k0, &k1);
                    if (k1 <= k0) continue;
                    if (ncq == 4) __trap();   // planner bound: a tail tile spans at most 5 pairs
                    cq[ncq++] = q;
                }
                const int ncol = (MODE == kModeFwd) ? ACC_COLS : width;
                for (int i = 0; i < ncq; ++i) {
                    if (ew == 0 && lane == 0) {
                        uint64_t* f = grp.sk.pflags + cq[i] * CG + crank;
                        const uint64_t t_start = globaltimer_ns();
                        while (ld_acquire_u64(f) != 1ull) {
                            __nanosleep(64);
                            if (globaltimer_ns() - t_start > kWaitTimeoutNs) {
                                printf("lora fused GEMM: stream-K partial wait timed out (pair %d <- %d)\n", pair,
                                       cq[i]);
                                __trap();
                            }
                        }
                        *f = 0;   // consumed (self-cleaning)
                        fence_proxy_async_global();
                        fence_proxy_async_smem();   // our earlier generic reads of the ring come first
                        const uint32_t bytes = static_cast<uint32_t>(ncol * 512);
                        mbar_arrive_expect_tx(part_full, bytes);
                        const float* src = slot_of(cq[i]);
                        for (uint32_t off = 0; off < bytes; off += 32768u)
                            bulk_load_1d(stage_base + off, src + off / 4, bytes - off < 32768u ? bytes - off : 32768u,
                                         part_full);
                    }
                    mbar_wait(part_full, static_cast<uint32_t>(i & 1));
                    const float4* s4 = reinterpret_cast<const float4*>(stage_base) + row_local;
#pragma unroll 1
                    for (int c = 0; c < ncol / 16; ++c) {
                        uint32_t v[16];
                        tmem_ld_32x32b_x16(tbase + 16 * c, v);
                        tmem_ld_wait();
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            const float4 t4 = s4[(c * 4 + e) * 128];
                            v[4 * e] = __float_as_uint(__uint_as_float(v[4 * e]) + t4.x);
                            v[4 * e + 1] = __float_as_uint(__uint_as_float(v[4 * e + 1]) + t4.y);
                            v[4 * e + 2] = __float_as_uint(__uint_as_float(v[4 * e + 2]) + t4.z);
                            v[4 * e + 3] = __float_as_uint(__uint_as_float(v[4 * e + 3]) + t4.w);
                        }
                        tmem_st_32x32b_x16(tbase + 16 * c, v);
                    }
                    tmem_st_wait();
                    tc_fence_before();
                    named_bar_sync(1, 128);   // ring free for the next contributor; TMEM updated
                    tc_fence_after();
                }
            }
            // (1) the r_pad low-rank values of this row
            float hv[R_PAD];
            if (MODE == kModeFwd && p.h_in != nullptr) {
                // fwd with dropout: h = q (M . x) A^T precomputed by K0 (the MMA's x A^T columns are unused)
#pragma unroll
                for (int j = 0; j < R_PAD; ++j) hv[j] = (j < p.r && row < p.T) ? p.h_in[row * p.r + j] : 0.0f;
            } else if (MODE == kModeFwd || gh_tile) {
                // fwd: h = x A^T in TMEM columns [BN, BN + r_pad); dx first tile: dY B in [128, ..)
                const uint32_t col0 = (MODE == kModeFwd) ? BN : DX_BN0;
#pragma unroll
                for (int c = 0; c < R_PAD / 16; ++c) {
                    uint32_t v[16];
                    tmem_ld_32x32b_x16(tbase + col0 + 16 * c, v);
                    tmem_ld_wait();
#pragma unroll
                    for (int e = 0; e < 16; ++e) hv[16 * c + e] = __uint_as_float(v[e]);
                }
                if (MODE != kModeFwd) {
#pragma unroll
                    for (int j = 0; j < R_PAD; ++j) hv[j] *= p.scale;     // gh = s (dY B)
                }
                // (2) side output: fwd h (for dB); dx fp32 gh only for the CUDA-core K3
                float* side = (MODE == kModeFwd) ? p.side_out : p.gh;
                if (side != nullptr && (MODE != kModeFwd || n_blk == 0))   // (warp-uniform)
                    warp_store_rows<R_PAD>(side, row - lane, p.T, p.r, lane, hv);
                if (MODE != kModeFwd && row < p.T) {
                    // K3's B operand: exact hi / mid / lo bf16 split of gh (and of the saved h),
                    // token-contiguous rows of cs [3 r8, t_pad] (saves K3s a pass)
                    const int r8 = (p.r + 7) / 8 * 8;
                    auto split_store = [&](__nv_bfloat16* cs, int k, float v) {
                        const __nv_bfloat16 hi = __float2bfloat16_rn(v);
                        const float r0 = v - __bfloat162float(hi);
                        const __nv_bfloat16 md = __float2bfloat16_rn(r0);
                        const __nv_bfloat16 lo = __float2bfloat16_rn(r0 - __bfloat162float(md));
                        cs[static_cast<int64_t>(k) * p.t_pad + row] = hi;
                        cs[static_cast<int64_t>(r8 + k) * p.t_pad + row] = md;
                        cs[static_cast<int64_t>(2 * r8 + k) * p.t_pad + row] = lo;
                    };
                    if (p.cs_gh != nullptr) {
                        if (p.cs_gh_rows == 3) {
#pragma unroll
                            for (int k = 0; k < R_PAD; ++k)
                                if (k < r8) split_store(p.cs_gh, k, k < p.r ? hv[k] : 0.0f);
                        } else {   // hi = bf16(gh) only: what the other tiles' tail MMA needs
#pragma unroll
                            for (int k = 0; k < R_PAD; ++k)
                                if (k < p.r) p.cs_gh[static_cast<int64_t>(k) * p.t_pad + row] = __float2bfloat16_rn(hv[k]);
                        }
                    }
                }
                if (MODE != kModeFwd && p.cs_h != nullptr) {   // (warp-uniform; rows >= T read as 0)
                    float hs[R_PAD];
                    warp_load_rows<R_PAD>(p.h_split_src, row - lane, p.T, p.r, lane, hs);
                    if (row < p.T) {
                        const int r8 = (p.r + 7) / 8 * 8;
#pragma unroll
                        for (int k = 0; k < R_PAD; ++k) {
                            if (k >= r8) break;
                            const float v = hs[k];
                            const __nv_bfloat16 hi = __float2bfloat16_rn(v);
                            const float r0 = v - __bfloat162float(hi);
                            const __nv_bfloat16 md = __float2bfloat16_rn(r0);
                            const __nv_bfloat16 lo = __float2bfloat16_rn(r0 - __bfloat162float(md));
                            p.cs_h[static_cast<int64_t>(k) * p.t_pad + row] = hi;
                            p.cs_h[static_cast<int64_t>(r8 + k) * p.t_pad + row] = md;
                            p.cs_h[static_cast<int64_t>(2 * r8 + k) * p.t_pad + row] = lo;
                        }
                    }
                }
                if (MODE != kModeFwd) {
                    // publish: every thread's gh stores, then one release of the flag
                    __threadfence();
                    named_bar_sync(1, 128);
                    if (ew == 0 && lane == 0)
                        st_release_u64(p.flags + static_cast<int64_t>(t_blk) * CG + crank, p.epoch);
                }
            } else {
                // dx, later tiles: wait for this row block's gh, then read it
                const uint64_t* flag = p.flags + static_cast<int64_t>(t_blk) * CG + crank;
                if (ld_acquire_u64(flag) != p.epoch) {
                    const uint64_t t_start = globaltimer_ns();
                    while (ld_acquire_u64(flag) != p.epoch) {
                        __nanosleep(64);
                        if (globaltimer_ns() - t_start > kWaitTimeoutNs) {
                            printf("lora dX kernel: gh flag wait timed out (row block %d)\n", t_blk);
                            __trap();
                        }
                    }
                }
                // gh of this row from the gh tile's token-contiguous split rows: one coalesced
                // 64-byte load per rank index per warp (bf16(gh) = hi; dropout: hi + mid + lo,
                // exactly the fp32 gh)
                const int r8 = (p.r + 7) / 8 * 8;
#pragma unroll
                for (int j = 0; j < R_PAD; ++j) {
                    float v = 0.0f;
                    if (j < p.r && row < p.T) {
                        const __nv_bfloat16* c = p.cs_gh + static_cast<int64_t>(j) * p.t_pad + row;
                        v = __bfloat162float(c[0]);
                        if (MODE == kModeDxDrop)
                            v = (v + __bfloat162float(c[static_cast<int64_t>(r8) * p.t_pad])) +
                                __bfloat162float(c[static_cast<int64_t>(2 * r8) * p.t_pad]);
                    }
                    hv[j] = v;
                }
            }
#if LORA_DROP_FHFMA
            uint32_t gq[(MODE == kModeDxDrop) ? R_PAD : 1];   // bf16(q gh_j) in the low half
            if constexpr (MODE == kModeDxDrop) {
#pragma unroll
                for (int j = 0; j < R_PAD; ++j)
                    gq[j] = static_cast<uint32_t>(__bfloat16_as_ushort(__float2bfloat16_rn(p.drop.q * hv[j])));
            }
#endif
            if constexpr (MODE == kModeDxDrop) {
                // dropout: no tail MMA -- the epilogue adds q M . (gh A) itself (step 5)
                mbar_wait((tt & 1) ? tailop2_full : tailop_full, (tt >> 1) & 1);
            } else {
            // (3) bf16(s h) / bf16(gh) -> swizzled K-major smem tile (tail MMA A operand)
            const float op_scale = (MODE == kModeFwd) ? p.scale : 1.0f;
#pragma unroll
            for (int c = 0; c < R_PAD / 8; ++c) {
                uint4 q;
                q.x = pack_bf16x2(op_scale * hv[8 * c + 0], op_scale * hv[8 * c + 1]);
                q.y = pack_bf16x2(op_scale * hv[8 * c + 2], op_scale * hv[8 * c + 3]);
                q.z = pack_bf16x2(op_scale * hv[8 * c + 4], op_scale * hv[8 * c + 5]);
                q.w = pack_bf16x2(op_scale * hv[8 * c + 6], op_scale * hv[8 * c + 7]);
                *reinterpret_cast<uint4*>(s_h + swizzled_offset(row_local, c, C::TAIL_ROW)) = q;
            }
            fence_proxy_async_smem();
            named_bar_sync(1, 128);
            // (4) tail MMA: acc[:, 0:width] += s_h (rows x r_pad) * tail_tile (width x r_pad)^T
            if (ew == 0 && lane == 0) {
                if (CG == 2 && !leader) {
                    mbar_arrive_cluster(sh_full, 0);      // our half of s_h is ready
                } else {
                    if (CG == 2) mbar_wait<true>(sh_full, tt & 1);
                    mbar_wait(tailop_full, tt & 1);
                    tc_fence_after();
                    const uint32_t h_addr = smem_u32(s_h);
                    const uint32_t t_addr = smem_u32(s_tailb);
                    const uint32_t idesc_tail = (MODE == kModeFwd)
                        ? idesc_tail_fwd : make_idesc_bf16(TM, static_cast<uint32_t>(width), 0, 1);
#ifndef LORA_PROBE_NO_TAIL
#pragma unroll
                    for (int kk = 0; kk < R_PAD / UMMA_K; ++kk) {
                        const uint64_t a_desc = make_smem_desc(h_addr + kk * 32, 16, tail_sbo, C::TAIL_LAYOUT);
                        uint64_t b_desc;
                        if constexpr (MODE == kModeFwd) {
                            b_desc = make_smem_desc(t_addr + kk * 32, 16, tail_sbo, C::TAIL_LAYOUT);
                        } else {
                            // A [R_PAD rows j, 64-col blocks of k] MN-major: LBO = block stride
                            b_desc = make_smem_desc(t_addr + kk * (UMMA_K * 128), R_PAD * 128, 1024,
                                                    kLayoutSW128);
                        }
                        umma<CG>(tmem_base + acc * NT, a_desc, b_desc, idesc_tail, 1u);
                    }
#endif
                    commit<CG>(tail_done);
                }
            }
            mbar_wait(tail_done, tt & 1);
            tc_fence_after();
            if (ew == 0 && lane == 0) mbar_arrive(tailop_empty);
            }

            // (5) drain: acc -> (+ b0) -> bf16 (RNE) -> global
            const bool row_ok = row < p.T;
            __nv_bfloat16* out_row = p.out + row * p.N_out;
            // dx dropout mode: this row's keep bits for the whole tile, loaded once up front
            // (one global round trip instead of one per 16-column chunk)
            uint32_t kw[(MODE == kModeDxDrop) ? NT / 32 : 1];
            if constexpr (MODE == kModeDxDrop) {
                const int64_t nw = (p.N_out + 31) / 32;
#pragma unroll
                for (int w = 0; w < NT / 32; ++w)
                    kw[w] = (row_ok && n0 / 32 + w < nw && 32 * w < width) ? p.drop_bits[row * nw + n0 / 32 + w] : 0u;
            }
            const bool storer = (ew == 0 && lane == 0);
            const int64_t row0 = static_cast<int64_t>(t_blk) * TM + crank * BM;   // this CTA's first row
            // (dropout dX with helper warps: this group drains the lower half of the chunks)
            constexpr bool kHelp = EpiHelpers<MODE, R_PAD>::WARPS > 0 && !C::STORE_TMA;
            const bool helped = kHelp && !grp.sk.enabled;
            const int c_end = helped ? (width / 16 + 1) / 2 : width / 16;
#pragma unroll 1
            for (int c = 0; c < c_end; ++c) {
                uint32_t v[16];
                tmem_ld_32x32b_x16(tbase + 16 * c, v);
                tmem_ld_wait();
                const int64_t col = n0 + 16 * c;
#ifdef LORA_PROBE_NO_STORE
                if (false) {
#else
                if (C::STORE_TMA || (row_ok && col < p.N_out)) {
#endif
                    float f[16];
#pragma unroll
                    for (int e = 0; e < 16; ++e) f[e] = __uint_as_float(v[e]);
                    if (MODE == kModeFwd && p.bias != nullptr) {
#pragma unroll
                        for (int e = 0; e < 16; ++e)
                            if (col + e < p.N_out) f[e] += __bfloat162float(p.bias[col + e]);   // (bias [m])
                    }
                    if constexpr (MODE == kModeDxDrop) {
                        // f += q M . (gh A): A columns of this chunk from the MN-major SW128 tile
                        const int lc = 16 * c;
                        const uint8_t* blk = s_tailb + (tt & 1) * round_up(C::TAILB_BYTES, 1024) +
                                             (lc / 64) * (R_PAD * 128);
                        const uint32_t ch = static_cast<uint32_t>((lc % 64) / 8);
#if LORA_DROP_FHFMA
                        // mixed-precision FMA (FHFMA.BF16: fp32 += bf16 x bf16, the A element taken
                        // straight from its bf16 half -- no widening instructions) with the operand
                        // gq_j = bf16(q gh_j), the same rounding of gh as the plain path's tail MMA
                        float lo[16];
                        drop_term16<R_PAD>(gq, blk, ch, p.r, lo);
                        const float qs = 1.0f;   // (q is inside gq)
#else
                        // packed FFMA2 (two fp32 FMAs per instruction, same order and rounding)
                        float2 lo2[8];
#pragma unroll
                        for (int e = 0; e < 8; ++e) lo2[e] = make_float2(0.0f, 0.0f);
#pragma unroll
                        for (int j = 0; j < R_PAD; ++j) {
#ifdef LORA_PROBE_DROP_NOFMA
                            break;   // timing experiment only: no q M . (gh A) term
#endif
                            if (j >= p.r) break;   // (uniform) rows r..r_pad-1 of A are zero
                            const uint4 a0 = *reinterpret_cast<const uint4*>(blk + swizzled_offset(j, ch, 128));
                            const uint4 a1 = *reinterpret_cast<const uint4*>(blk + swizzled_offset(j, ch + 1, 128));
                            const uint32_t aw[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
                            const float2 hh = make_float2(hv[j], hv[j]);
#pragma unroll
                            for (int e = 0; e < 8; ++e) {
                                // bf16 pair -> fp32 pair: the bf16 bits are the high halves
                                const float2 av = make_float2(__uint_as_float(aw[e] << 16),
                                                              __uint_as_float(aw[e] & 0xFFFF0000u));
                                lo2[e] = ffma2(hh, av, lo2[e]);
                            }
                        }
                        float lo[16];
#pragma unroll
                        for (int e = 0; e < 8; ++e) {
                            lo[2 * e] = lo2[e].x;
                            lo[2 * e + 1] = lo2[e].y;
                        }
                        const float qs = p.drop.q;
#endif
                        // keep bits of the 16 columns, packed by K0 (32 per word; col % 16 == 0)
                        const uint32_t keep = (kw[c >> 1] >> ((c & 1) * 16)) & 0xFFFFu;
#pragma unroll
                        for (int e = 0; e < 16; ++e)
                            if ((keep >> e) & 1u) f[e] = fmaf(qs, lo[e], f[e]);
                    }
                    uint4 q0, q1;
                    q0.x = pack_bf16x2(f[0], f[1]);   q0.y = pack_bf16x2(f[2], f[3]);
                    q0.z = pack_bf16x2(f[4], f[5]);   q0.w = pack_bf16x2(f[6], f[7]);
                    q1.x = pack_bf16x2(f[8], f[9]);   q1.y = pack_bf16x2(f[10], f[11]);
                    q1.z = pack_bf16x2(f[12], f[13]); q1.w = pack_bf16x2(f[14], f[15]);
                    if constexpr (C::STORE_TMA) {
                        // TMA-store epilogue: 32-column blocks (16 for a tile's odd tail: fwd
                        // tiles are 256 - r_pad wide) staged swizzled in shared memory, then ONE
                        // bulk tensor store per block by one thread; rows >= T and columns
                        // >= N_out are clipped by the store
                        const int blk = c >> 1, half = c & 1;
                        const bool tail16 = (c == width / 16 - 1) && !half;   // a lone 16-column block
                        const int buf = blk % C::STG_BUFS;
                        uint8_t* sb = s_stg + buf * C::STG_BYTES;
                        if (!half) {
                            // the store issued STG_BUFS blocks ago has read this buffer
                            if (storer) bulk_wait_group_read<C::STG_BUFS - 1>();
                            named_bar_sync(1, 128);
                        }
                        if (tail16) {   // [128 rows][32 B], SW32
                            *reinterpret_cast<uint4*>(sb + swizzled_offset(row_local, 0, 32)) = q0;
                            *reinterpret_cast<uint4*>(sb + swizzled_offset(row_local, 1, 32)) = q1;
                        } else {        // [128 rows][64 B], SW64
                            *reinterpret_cast<uint4*>(sb + swizzled_offset(row_local, 2 * half, 64)) = q0;
                            *reinterpret_cast<uint4*>(sb + swizzled_offset(row_local, 2 * half + 1, 64)) = q1;
                        }
                        if (half || tail16) {
                            fence_proxy_async_smem();
                            named_bar_sync(1, 128);
                            if (storer) {
                                const FusedGemmMaps& om = grp.maps[un.g];
                                tma_store_2d(tail16 ? &om.out16 : &om.out32, sb,
                                             static_cast<int32_t>(n0 + 32 * blk), static_cast<int32_t>(row0));
                                bulk_commit_group();
                            }
                        }
                    } else {
                        *reinterpret_cast<uint4*>(out_row + col) = q0;               // N_out % 8 == 0
                        if (col + 8 < p.N_out) *reinterpret_cast<uint4*>(out_row + col + 8) = q1;
                    }
                }
            }
            if constexpr (MODE == kModeDxDrop) {
                // every epilogue (and helper) warp is done with the A tile (and the accumulator)
                if (helped) {
                    tc_fence_before();
                    named_bar_sync(2, 32 * (4 + EpiHelpers<MODE, R_PAD>::WARPS));
                    tc_fence_after();
                } else {
                    named_bar_sync(1, 128);
                }
                if (ew == 0 && lane == 0) mbar_arrive((tt & 1) ? tailop2_empty : tailop_empty);
            }
            if (p.unit_flags != nullptr) {
                // comm-fused epilogue: this CTA's 128 rows of the tile are stored -- publish
                // them to the ranks' reducers (lora_symm.cu) with one system-scope release
                if (C::STORE_TMA && storer) bulk_wait_group<0>();   // the bulk stores have landed
                __threadfence_system();
                named_bar_sync(1, 128);
                const int64_t nrow128 = (p.T + BM - 1) / BM;
                const int64_t row128 = static_cast<int64_t>(t_blk) * CG + crank;
                if (ew == 0 && lane == 0 && row128 < nrow128)   // (a pair's second CTA past T has no rows)
                    st_release_sys_u32(p.unit_flags + n_blk * nrow128 + row128, 1u);
            }
            ++tt;
#ifdef LORA_PROBE_SK
            if (ew == 0 && lane == 0 && crank == 0) {
                const unsigned i = atomicAdd(&g_probe_n, 1u);
                if (i < 4096) {
                    unsigned long long* r = g_probe_buf + 4 * i;
                    r[0] = (static_cast<unsigned long long>(pair) << 32) | (tl << 8) | static_cast<unsigned>(un.role);
                    r[1] = (static_cast<unsigned long long>(un.kb0) << 32) | static_cast<unsigned>(un.kb1);
                    r[2] = probe_u0 - probe_t0;
                    r[3] = globaltimer_ns() - probe_t0;
                }
            }
#endif
            tc_fence_before();
            __syncwarp();
            if (lane == 0) {
                if (CG == 1) mbar_arrive(&tmem_empty[acc]);
                else mbar_arrive_cluster(&tmem_empty[acc], 0);  // the leader's MMA warp waits on it
            }
        }
    }

    if (C::STORE_TMA && warp == 0 && lane == 0) bulk_wait_group<0>();   // every y / dX store performed
    tc_fence_before();
    if constexpr (CG == 2) cluster_sync(); else __syncthreads();
#ifdef LORA_PROBE_CLOCK
    if (threadIdx.x == 0 && (blockIdx.x == 0 || blockIdx.x == gridDim.x - 1))
        printf("PROBE_CLOCK mode=%d block=%d cycles=%lld ns=%llu\n", MODE, blockIdx.x, clock64() - probe_c0,
               (unsigned long long)(globaltimer_ns() - probe_t0));
#endif
    if (warp == 0) {
        tc_fence_after();
        tmem_dealloc_cg<CG>(tmem_base);
    }
    // self-cleaning gh flags: every CTA is past its last flag wait; the last one
    // out zeroes the flags no K3 will wait on, and the counter
    if (MODE != kModeFwd && grp.done != nullptr && threadIdx.x == 0) {
        if (atom_add_acq_rel_u64(grp.done, 1ull) == static_cast<unsigned long long>(gridDim.x) - 1) {
            for (int g = 0; g < grp.count; ++g)
                if (grp.p[g].reset_flags)
                    for (int i = 0; i < grp.p[g].nflags; ++i) grp.p[g].flags[i] = 0;
            *grp.done = 0;   // (visible to the next launch: kernel boundary)
        }
    }
}

// ----------------------------------------------------------------------------
// sync pool (see lora_kernels.h)
// ----------------------------------------------------------------------------
constexpr int kSyncPoolWords = 1 << 18;   // 2 MiB of device memory
constexpr int kSyncPoolRing = 1 << 17;    // [0, ring): eager calls, recycled; [ring, end): captured graphs
__device__ unsigned long long g_sync_pool[kSyncPoolWords];

namespace {
// Captured-graph region: first-fit free list of [offset, offset + len) word
// ranges.  A range handed to a capturing stream is owned by that graph through
// a cudaUserObject whose destructor (run by the CUDA runtime when the graph and
// every executable instantiated from it are destroyed) returns it here -- so
// re-capturing graphs for the life of a process never exhausts the region.
// The words are zero when returned: every protocol resets its words before its
// launch chain ends.
struct CapturePool {
    std::mutex mu;
    std::vector<std::pair<int, int>> free_list[64];   // per device: sorted, coalesced
    bool init[64] = {};
};
CapturePool& cap_pool() {
    static CapturePool* p = new CapturePool();   // never destroyed: destructors may run at exit
    return *p;
}
struct CapturedRange {
    int dev, off, len;
};
void CUDART_CB release_captured(void* ptr) {
    CapturedRange* r = static_cast<CapturedRange*>(ptr);
    CapturePool& P = cap_pool();
    {
        std::lock_guard<std::mutex> lk(P.mu);
        auto& fl = P.free_list[r->dev];
        auto it = std::lower_bound(fl.begin(), fl.end(), std::make_pair(r->off, 0));
        it = fl.insert(it, {r->off, r->len});
        // coalesce with the neighbours
        if (it + 1 != fl.end() && it->first + it->second == (it + 1)->first) {
            it->second += (it + 1)->second;
            fl.erase(it + 1);
        }
        if (it != fl.begin() && (it - 1)->first + (it - 1)->second == it->first) {
            (it - 1)->second += it->second;
            fl.erase(it);
        }
    }
    delete r;
}
}  // namespace

int sync_pool_captured_free_words(int dev) {
    CapturePool& P = cap_pool();
    std::lock_guard<std::mutex> lk(P.mu);
    if (dev < 0 || dev >= 64) return 0;
    if (!P.init[dev]) return kSyncPoolWords - kSyncPoolRing;
    int n = 0;
    for (const auto& f : P.free_list[dev]) n += f.second;
    return n;
}

unsigned long long* sync_pool_alloc(int words, cudaStream_t stream) {
    static std::mutex mu;
    static unsigned long long* base[64] = {};
    static int ring_next[64] = {};
    if (words <= 0 || words > 4096) return nullptr;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return nullptr;
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    cudaGraph_t graph = nullptr;
    if (cudaStreamGetCaptureInfo(stream, &cs, nullptr, &graph) != cudaSuccess) return nullptr;
    const int w = (words + 7) / 8 * 8;   // 64-byte granules
    {
        std::lock_guard<std::mutex> lk(mu);
        if (base[dev] == nullptr) {
            void* p = nullptr;
            if (cudaGetSymbolAddress(&p, g_sync_pool) != cudaSuccess) return nullptr;
            base[dev] = static_cast<unsigned long long*>(p);
        }
    }
    if (cs != cudaStreamCaptureStatusNone) {
        if (graph == nullptr) return nullptr;
        CapturePool& P = cap_pool();
        int off = -1;
        {
            std::lock_guard<std::mutex> lk(P.mu);
            auto& fl = P.free_list[dev];
            if (!P.init[dev]) {
                fl.push_back({kSyncPoolRing, kSyncPoolWords - kSyncPoolRing});
                P.init[dev] = true;
            }
            for (auto it = fl.begin(); it != fl.end(); ++it) {
                if (it->second < w) continue;
                off = it->first;
                it->first += w;
                it->second -= w;
                if (it->second == 0) fl.erase(it);
                break;
            }
        }
        if (off < 0) return nullptr;   // every captured word is held by a live graph
        CapturedRange* r = new CapturedRange{dev, off, w};
        cudaUserObject_t obj;
        if (cudaUserObjectCreate(&obj, r, release_captured, 1, cudaUserObjectNoDestructorSync) != cudaSuccess) {
            release_captured(r);
            return nullptr;
        }
        if (cudaGraphRetainUserObject(graph, obj, 1, cudaGraphUserObjectMove) != cudaSuccess) {
            cudaUserObjectRelease(obj, 1);   // runs release_captured
            return nullptr;
        }
        return base[dev] + off;
    }
    // eager calls: a recycled ring.  A word is reused only after 2^17 words of later
    // eager allocations on this device -- thousands of calls -- by which time the
    // launch chain that used it has long completed (its stream had to run them).
    std::lock_guard<std::mutex> lk(mu);
    if (ring_next[dev] + w > kSyncPoolRing) ring_next[dev] = 0;
    unsigned long long* r = base[dev] + ring_next[dev];
    ring_next[dev] += w;
    return r;
}

// ----------------------------------------------------------------------------
// host side
// ----------------------------------------------------------------------------

static int64_t col_tiles_host(int mode, int r_pad, int64_t n_out) {
    if (mode == kModeFwd) {
        const int bn = NT - r_pad;
        return (n_out + bn - 1) / bn;
    }
    return n_out <= DX_BN0 ? 1 : 1 + (n_out - DX_BN0 + NT - 1) / NT;
}

// The stream-K tail is opt-in (LORA_STREAMK=1, read per call): measured on B200
// it does not beat the data-parallel schedule ("K1/K2 schedule"),
// because every split exposes one more fused epilogue (5-10 us for a dX tile)
// that the two TMEM accumulators otherwise hide under the next mainloop.
static bool coop_enabled() {
    static const bool on = [] {
        const char* s = getenv("LORA_COOP");
        return !(s && s[0] == '0');
    }();
    return on;
}

static bool streamk_enabled() {
    const char* v = getenv("LORA_STREAMK");
    return v && v[0] == '1';
}

size_t fused_gemm_partial_bytes(int64_t T, int64_t N_out) {
    // worth a stream-K schedule only when the launch has at least a wave of tiles
    if (!streamk_enabled()) return 0;
    const int64_t tiles = ((T + 255) / 256) * ((N_out + 255) / 256);
    return tiles >= 32 ? size_t(kMaxPairs) * kPartialFloatsPerCta * sizeof(float) : 0;
}

// Host side of the schedule (lora_kernels.h, StreamKSched).
template <int MODE, int R_PAD, int CG>
static cudaError_t plan_stream_k(FusedGemmGroup& grp, int npairs, cudaStream_t stream) {
    using C = GemmCfg<MODE, R_PAD, CG>;
    StreamKSched& sk = grp.sk;
    sk.enabled = 0;
    sk.partial = grp.p[0].sk_partial;
    sk.pflags = nullptr;
    const int W = grp.tile_start[grp.count];
    if (!C::SK_OK || !streamk_enabled() || sk.partial == nullptr || npairs < 2 || npairs > kMaxPairs || W <= npairs)
        return cudaSuccess;
    const int TM = BM * CG;
    // per-tile cost in tile order (decode_tile): k-blocks x width / 128 (fwd: always N = 256)
    std::vector<int> cost(W), is_gh(W, 0);
    for (int g = 0; g < grp.count; ++g) {
        const FusedGemmParams& p = grp.p[g];
        const int ntb = static_cast<int>((p.T + TM - 1) / TM), kb = static_cast<int>((p.K + BK - 1) / BK);
        const int nc = static_cast<int>(col_tiles_host(MODE, R_PAD, p.N_out));
        for (int nb = 0; nb < nc; ++nb) {
            int w = 2;
            if (MODE != kModeFwd) {
                const int64_t start = nb == 0 ? 0 : DX_BN0 + int64_t(nb - 1) * C::BN;
                const int64_t width = nb == 0 ? DX_BN0 : std::min<int64_t>(C::BN, (p.N_out - start + 127) / 128 * 128);
                w = static_cast<int>(width / 128);
            }
            for (int t = 0; t < ntb; ++t) {
                cost[grp.tile_start[g] + nb * ntb + t] = kb * w;
                is_gh[grp.tile_start[g] + nb * ntb + t] = MODE != kModeFwd && nb == 0;
            }
        }
    }
    // the tail = the last partial round of the data-parallel order
    int D = W - W % npairs;
    if (D == W) D = W - npairs;   // full rounds only: split the last one if loads are uneven
    for (int i = D; i < W; ++i)
        if (is_gh[i]) return cudaSuccess;   // a gh tile must not be split: keep data-parallel
    std::vector<int64_t> load(npairs, 0);
    for (int i = 0; i < D; ++i) load[i % npairs] += cost[i];
    std::vector<int64_t> dp = load;
    for (int i = D; i < W; ++i) dp[i % npairs] += cost[i];
    int64_t tail = 0;
    for (int i = D; i < W; ++i) tail += cost[i];
    // smallest common finish time that absorbs the tail
    int64_t lo = *std::max_element(load.begin(), load.end()), hi = lo + tail;
    while (lo < hi) {
        const int64_t mid = (lo + hi) / 2;
        int64_t cap = 0;
        for (int q = 0; q < npairs; ++q) cap += mid > load[q] ? mid - load[q] : 0;
        if (cap >= tail) hi = mid; else lo = mid + 1;
    }
    const int64_t finish = lo;
    const int64_t dp_finish = *std::max_element(dp.begin(), dp.end());
    if (finish * 100 > dp_finish * 97) return cudaSuccess;   // < 3% to gain: keep data-parallel
    if (tail > (1 << 30)) return cudaSuccess;
    sk.D = D;
    sk.ntail = W - D;
    sk.prefix[0] = 0;
    for (int i = 0; i < sk.ntail; ++i) sk.prefix[i + 1] = sk.prefix[i] + cost[D + i];
    sk.S[0] = 0;
    for (int q = 0; q < npairs; ++q) {
        const int64_t b = finish > load[q] ? finish - load[q] : 0;
        sk.S[q + 1] = static_cast<int>(std::min<int64_t>(tail, sk.S[q] + b));
    }
    sk.S[npairs] = static_cast<int>(tail);
    // the kernel's owner handles at most 4 contributors per split tile
    for (int i = 0; i < sk.ntail; ++i) {
        const int64_t a = sk.prefix[i], b = sk.prefix[i + 1];
        int holders = 0;
        for (int q = 0; q < npairs; ++q)
            if (sk.S[q] < b && sk.S[q + 1] > a) ++holders;
        if (holders > 5) return cudaSuccess;   // (S stays unused: sk.enabled == 0)
    }
    sk.pflags = reinterpret_cast<uint64_t*>(sync_pool_alloc(npairs * CG, stream));
    if (sk.pflags == nullptr) return cudaErrorMemoryAllocation;
    sk.enabled = 1;
    return cudaSuccess;
}

template <int MODE, int R_PAD, int CG>
static cudaError_t launch_impl(FusedGemmGroup& grp, int num_sms, cudaStream_t stream) {
    using C = GemmCfg<MODE, R_PAD, CG>;
    auto kern = lora_fused_gemm_kernel<MODE, R_PAD, CG>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM_BYTES);
    if (e != cudaSuccess) return e;
    if (grp.count < 1 || grp.count > kMaxGroup) return cudaErrorInvalidValue;
    int64_t tiles = 0;
    for (int g = 0; g < grp.count; ++g) {
        grp.tile_start[g] = static_cast<int>(tiles);
        const FusedGemmParams& p = grp.p[g];
        tiles += ((p.T + BM * CG - 1) / (BM * CG)) * col_tiles_host(MODE, R_PAD, p.N_out);
    }
    grp.tile_start[grp.count] = static_cast<int>(tiles);
    grp.done = nullptr;
    bool any_reset = false;
    for (int g = 0; g < grp.count; ++g) any_reset = any_reset || (MODE != kModeFwd && grp.p[g].reset_flags);
    if (any_reset) {   // someone must zero the flags at the end (no K3 waits on them)
        grp.done = sync_pool_alloc(1, stream);
        if (grp.done == nullptr) return cudaErrorMemoryAllocation;
    }
    const int64_t units = num_sms / CG;
    const int grid = static_cast<int>((tiles < units ? tiles : units) * CG);
    if (grid <= 0) return cudaSuccess;
    if ((e = plan_stream_k<MODE, R_PAD, CG>(grp, grid / CG, stream)) != cudaSuccess) return e;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(EpiHelpers<MODE, R_PAD>::THREADS);
    cfg.dynamicSmemBytes = C::SMEM_BYTES;
    cfg.stream = stream;
    cudaLaunchAttribute attr[3];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CG;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    // CTAs that wait on flags other CTAs of the SAME grid raise (dX gh tiles,
    // stream-K partials) need those producers resident: a cooperative launch
    // guarantees the whole (persistent, <= 1 CTA per SM) grid is co-resident even
    // when kernels on other streams hold SMs (LORA_COOP=0 turns it off)
    attr[2].id = cudaLaunchAttributeCooperative;
    attr[2].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = ((MODE != kModeFwd || grp.sk.enabled) && coop_enabled() && !grp.no_coop) ? 3 : 2;
    e = cudaLaunchKernelEx(&cfg, kern, grp);
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

int fused_gemm_block_n(int mode, int r_pad) { return mode == kModeFwd ? NT - r_pad : NT; }

template <int CG>
static const void* gemm_fn(int mode, int r_pad) {
    switch (mode * 100 + r_pad) {
        case 16: return (const void*)lora_fused_gemm_kernel<kModeFwd, 16, CG>;
        case 32: return (const void*)lora_fused_gemm_kernel<kModeFwd, 32, CG>;
        case 64: return (const void*)lora_fused_gemm_kernel<kModeFwd, 64, CG>;
        case 116: return (const void*)lora_fused_gemm_kernel<kModeDx, 16, CG>;
        case 132: return (const void*)lora_fused_gemm_kernel<kModeDx, 32, CG>;
        case 164: return (const void*)lora_fused_gemm_kernel<kModeDx, 64, CG>;
        case 216: return (const void*)lora_fused_gemm_kernel<kModeDxDrop, 16, CG>;
        case 232: return (const void*)lora_fused_gemm_kernel<kModeDxDrop, 32, CG>;
        case 264: return (const void*)lora_fused_gemm_kernel<kModeDxDrop, 64, CG>;
    }
    return nullptr;
}

int fused_gemm_regs(int mode, int r_pad, int cta_group) {
    const void* f = cta_group == 2 ? gemm_fn<2>(mode, r_pad) : gemm_fn<1>(mode, r_pad);
    cudaFuncAttributes fa;
    if (!f || cudaFuncGetAttributes(&fa, f) != cudaSuccess) return 255;
    return fa.numRegs;
}

// Column tiles of a fused-GEMM output as the kernel walks them (ColTiles):
// starts[0 .. count] with starts[count] = n_out; returns count (or -1 > max).
int fused_gemm_col_tiles(int mode, int r_pad, int64_t n_out, int* starts, int max) {
    const int64_t count = col_tiles_host(mode, r_pad, n_out);
    if (count > max) return -1;
    for (int64_t c = 0; c < count; ++c) {
        int64_t st;
        if (mode == kModeFwd) st = c * (NT - r_pad);
        else st = c == 0 ? 0 : DX_BN0 + (c - 1) * NT;
        starts[c] = static_cast<int>(st);
    }
    starts[count] = static_cast<int>(n_out);
    return static_cast<int>(count);
}

// On by default since round 2 (cfg2 step replayed as a CUDA graph, alternating
// runs on one box: 199.6-199.7 vs 201.3-201.4 us; cfg3 within its power-cap
// noise; every GPU test passes either way -- round 1's kernels had measured 6%
// slower); LORA_PDL=0 turns it off.
bool pdl_enabled() {
    static const bool on = [] {
        const char* s = getenv("LORA_PDL");
        return !(s && s[0] == '0');
    }();
    return on;
}

int fused_gemm_narrow_cols(int r_pad, int cta_group) {
    const int nar = cta_group == 2 ? (r_pad > 32 ? r_pad : 32) : r_pad;
    return nar / cta_group;
}

int64_t fused_gemm_row_blocks(int64_t T, int cta_group) { return (T + BM * cta_group - 1) / (BM * cta_group); }

template <int CG>
static cudaError_t dispatch(int mode, int r_pad, FusedGemmGroup& grp, int num_sms, cudaStream_t stream) {
    if (mode == kModeFwd) {
        switch (r_pad) {
            case 16: return launch_impl<kModeFwd, 16, CG>(grp, num_sms, stream);
            case 32: return launch_impl<kModeFwd, 32, CG>(grp, num_sms, stream);
            case 64: return launch_impl<kModeFwd, 64, CG>(grp, num_sms, stream);
        }
    } else if (mode == kModeDx) {
        switch (r_pad) {
            case 16: return launch_impl<kModeDx, 16, CG>(grp, num_sms, stream);
            case 32: return launch_impl<kModeDx, 32, CG>(grp, num_sms, stream);
            case 64: return launch_impl<kModeDx, 64, CG>(grp, num_sms, stream);
        }
    } else if (mode == kModeDxDrop) {
        switch (r_pad) {
            case 16: return launch_impl<kModeDxDrop, 16, CG>(grp, num_sms, stream);
            case 32: return launch_impl<kModeDxDrop, 32, CG>(grp, num_sms, stream);
            case 64: return launch_impl<kModeDxDrop, 64, CG>(grp, num_sms, stream);
        }
    }
    return cudaErrorInvalidValue;
}

cudaError_t launch_fused_gemm_group(int mode, int r_pad, int cta_group, FusedGemmGroup& grp, int num_sms,
                                    cudaStream_t stream) {
    return cta_group == 2 ? dispatch<2>(mode, r_pad, grp, num_sms, stream)
                          : dispatch<1>(mode, r_pad, grp, num_sms, stream);
}

cudaError_t launch_fused_gemm(int mode, int r_pad, int cta_group, const FusedGemmMaps& maps,
                              const FusedGemmParams& p, int num_sms, cudaStream_t stream) {
    static thread_local FusedGemmGroup grp;   // ~6 KiB: keep it off the stack
    grp.count = 1;
    grp.no_coop = 0;
    grp.maps[0] = maps;
    grp.p[0] = p;
    return launch_fused_gemm_group(mode, r_pad, cta_group, grp, num_sms, stream);
}


// Lazy module loading (the CUDA 12 default) loads a kernel at its first launch,
// and that load waits for the device to drain.  A kernel that spins on another
// one's output (the comm-fused reducer, lora_symm.cu) must therefore never be
// running while the kernel it waits for is launched for the first time:
// preload_*() loads every kernel of a file up front (cudaFuncGetAttributes).
template <int CG>
static cudaError_t preload_cg() {
    cudaFuncAttributes a;
    const void* ks[] = {
        (const void*)lora_fused_gemm_kernel<kModeFwd, 16, CG>, (const void*)lora_fused_gemm_kernel<kModeFwd, 32, CG>,
        (const void*)lora_fused_gemm_kernel<kModeFwd, 64, CG>, (const void*)lora_fused_gemm_kernel<kModeDx, 16, CG>,
        (const void*)lora_fused_gemm_kernel<kModeDx, 32, CG>, (const void*)lora_fused_gemm_kernel<kModeDx, 64, CG>,
        (const void*)lora_fused_gemm_kernel<kModeDxDrop, 16, CG>,
        (const void*)lora_fused_gemm_kernel<kModeDxDrop, 32, CG>,
        (const void*)lora_fused_gemm_kernel<kModeDxDrop, 64, CG>};
    for (const void* k : ks) {
        cudaError_t e = cudaFuncGetAttributes(&a, k);
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}
cudaError_t preload_gemm_kernels() {
    cudaError_t e = preload_cg<1>();
    return e != cudaSuccess ? e : preload_cg<2>();
}

}  // namespace lora_sm100

#ifdef LORA_PROBE_SK
// experiment only: copy and reset the unit timeline (pair<<32 | unit<<8 | role, kb0<<32 | kb1, t_mma_done, t_end)
extern "C" int lora_probe_sk_dump(unsigned long long* host, int max_rows) {
    unsigned n = 0;
    cudaMemcpyFromSymbol(&n, lora_sm100::g_probe_n, sizeof(n));
    if (n > 4096) n = 4096;
    if (static_cast<int>(n) > max_rows) n = max_rows;
    cudaMemcpyFromSymbol(host, lora_sm100::g_probe_buf, n * 4 * sizeof(unsigned long long));
    const unsigned z = 0;
    cudaMemcpyToSymbol(lora_sm100::g_probe_n, &z, sizeof(z));
    return static_cast<int>(n);
}
#endif
