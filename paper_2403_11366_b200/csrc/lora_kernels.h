// lora_kernels.h -- internal interface between the C-ABI host layer
// (lora_api.cpp) and the sm_100a kernels.  Not part of the public ABI.
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace lora_sm100 {

enum : int { kModeFwd = 0, kModeDx = 1, kModeDxDrop = 2 };

// Programmatic dependent launch for the step's kernels (LORA_PDL=1; off by default).
bool pdl_enabled();
bool k3_overlap_enabled();   // LORA_K3_OVERLAP (default on)

// LoRA dropout (lora_philox.cuh): keep(t, k) = 16-bit draw (k % 8) of Philox4x32-10((k/8, t, offset), seed) >= thr
struct DropoutParams {
    uint64_t seed, offset;
    uint32_t thr;    // floor(p * 2^16); 0 = keep everything
    float q;         // 1 / (1 - p)
    uint32_t* keep_bits;   // caller's keep-mask buffer (lora_dropout.keep_bits) or null
    __nv_bfloat16* masked_x;   // caller's M . x buffer (lora_dropout.masked_x) or null
    int64_t row0, col0;    // position of this call's input in the full one (col0 % 8 == 0)
};

// Philox4x32-10 of one member, prepared on the host (launch_dropout_input_group):
// the ten round keys and the counter's offset words, so the device rounds take
// them as constant operands; thr2 = thr in both 16-bit halves
struct PhiloxKeys {
    uint32_t k0[10], k1[10];
    uint32_t c2, c3;
    uint32_t thr2;
    uint32_t k8_base, t_base;   // counter words c0 = k / 8 + k8_base, c1 = t + t_base (col0 / 8, row0)
};

struct FusedGemmParams {
    int64_t T;                    // token rows
    int64_t K;                    // reduction extent (n fwd, m dx)
    int64_t N_out;                // output columns (m fwd, n dx)
    int r;                        // LoRA rank
    float scale;                  // s = alpha / r
    const __nv_bfloat16* bias;    // fwd only; may be null
    __nv_bfloat16* out;           // y or dx, [T, N_out]
    float* side_out;              // fwd: h [T, r] (unscaled), may be null
    float* gh;                    // dx: gh [T, r] fp32 = s dY B for the CUDA-core K3 (LORA_K3=cluster), or null
    uint64_t* flags;              // dx: one per (row block, CTA of the pair), sync pool: 1 = gh published
    uint64_t epoch;               // dx: value a published flag holds (1)
    int nflags;                   // dx: row blocks x CTAs per pair
    int reset_flags;              // dx: 1 = this launch's last CTA zeroes the flags (no K3 waits on them)
    const float* h_in;            // fwd with dropout: h [T, r] precomputed by K0 (else null: h from the MMA)
    DropoutParams drop;           // dx dropout mode: dX += q M . (gh A) in the epilogue
    const uint32_t* drop_bits;    // dx dropout mode: keep bits [T, ceil(N_out/32)] from K0
    // dx: K3's split coefficients written by the gh tile (else null): cs_gh <- gh,
    // cs_h <- h_split_src; [3 r8, t_pad] bf16 hi / mid / lo rows (see K3s).
    // cs_gh is also how the other column tiles of a row block read gh: token-
    // contiguous rows, so a warp's 32 rows are one coalesced 64-byte load per rank
    // index.  cs_gh_rows = 1 writes only hi = bf16(gh) (all the tail MMA needs),
    // 3 the full split (dA wants it; dropout mode rebuilds fp32 gh = hi + mid + lo).
    __nv_bfloat16* cs_gh;
    int cs_gh_rows;
    __nv_bfloat16* cs_h;
    const float* h_split_src;
    int64_t t_pad;
    float* sk_partial;            // stream-K partial slots in this problem's workspace (group: p[0]'s), or null
    // comm-fused epilogue (lora_symm.cu): after the 128-row half of an
    // output tile is stored, one release store (system scope: peers read it over
    // NVLink) sets unit_flags[n_blk * ceil(T / 128) + row128] = 1; null = off
    uint32_t* unit_flags;
};

struct FusedGemmMaps {
    CUtensorMap act, w, w2, nar, tail;
    CUtensorMap out32, out16;   // the output (y / dX) for the TMA-store epilogue: boxes [128 x 32] SW64, [128 x 16] SW32
};

// Schedule of a fused-GEMM launch.  Tiles in
// tile order [0, D) run data-parallel (pair q takes q, q + P, ...): the pairs
// move through the W0 column blocks in lock-step rounds, so concurrent tiles
// share their x / W0 k-blocks in L2.  The last partial round [D, W) would
// leave pairs idle; its work is split over ALL pairs ("stream-K tail"): cost
// units = one 64-deep k-block of a 128-column slab (a 256-wide tile k-block
// costs 2), tail tile i occupies [prefix[i], prefix[i+1]) of one cost line,
// and pair q takes [S[q], S[q+1]), sized so every pair's total is equal.  A
// tile cut by a range boundary is finished by the pair holding its k-block 0
// (the owner); the pairs holding the rest write fp32 partial accumulators to
// `partial` (one slot per CTA: only a pair's first tail segment can start
// mid-tile) and raise pflags; the owner adds them in pair order --
// deterministic for a given launch shape.  dx gh tiles (column tile 0) are
// never in the tail.
constexpr int kMaxPairs = 148;
constexpr int kPartialFloatsPerCta = 128 * 256;   // one CTA's 128 x 256 fp32 accumulator
struct StreamKSched {
    int enabled;                   // 0: data-parallel over all tiles
    int D;                         // first tail tile
    int ntail;                     // tail tiles (<= kMaxPairs)
    int prefix[kMaxPairs + 1];     // tail cost prefix
    int S[kMaxPairs + 1];          // tail cost range of pair q
    float* partial;                // [P * CTAs per pair][kPartialFloatsPerCta] (caller workspace)
    uint64_t* pflags;              // [P * CTAs per pair] sync pool: 1 = slot written; the owner zeroes it
};

// A group of independent LoRA linears (same rank bucket) processed by ONE
// persistent launch: the tiles of problem g occupy [tile_start[g], tile_start[g+1]).
constexpr int kMaxGroup = 8;
struct FusedGemmGroup {
    FusedGemmMaps maps[kMaxGroup];
    FusedGemmParams p[kMaxGroup];
    int tile_start[kMaxGroup + 1];
    int count;
    unsigned long long* done;     // dx: sync-pool launch counter (last CTA out resets flags), or null
    int no_coop;                  // 1: never a cooperative launch (the comm-fused path: a cooperative grid
                                  // waits for the co-resident reducer it feeds -- lora_symm.cu)
    StreamKSched sk;              // filled in by the launcher
};
// bytes of stream-K partial workspace a fused-GEMM launch may use (0: none)
size_t fused_gemm_partial_bytes(int64_t T, int64_t N_out);

// Device-side synchronisation words (K2's gh flags, launch done-counters): a
// static __device__ pool, zero when the module loads.  Every protocol that
// uses it returns its words to zero before its launch chain ends (the last
// consumer resets), so no host memset is needed and captured CUDA graphs
// replay correctly.  Eager calls take words from a recycled ring; calls made
// while `stream` is capturing get words of their own, owned by the capturing
// graph (a cudaUserObject returns them when the graph is destroyed).
// Returns null when the pool is exhausted (capture) or on a CUDA error.
unsigned long long* sync_pool_alloc(int words, cudaStream_t stream);
// words of the captured-graph region currently free on device `dev` (a graph's
// words return when the graph and its executables are destroyed)
int sync_pool_captured_free_words(int dev);

// K1 / K2.  r_pad in {16, 32, 64}; tiles are (128 * cta_group) x (256 - r_pad).
// cta_group = 2 runs on CTA pairs (tcgen05 cta_group::2); the TMA boxes of
// `maps` must match (see lora_api.cpp).
int fused_gemm_block_n(int mode, int r_pad);
int fused_gemm_narrow_cols(int r_pad, int cta_group);     // dx: B columns per CTA (TMA box inner)
int64_t fused_gemm_row_blocks(int64_t T, int cta_group);  // dx: flags needed = row blocks * cta_group
cudaError_t launch_fused_gemm(int mode, int r_pad, int cta_group, const FusedGemmMaps& maps,
                              const FusedGemmParams& p, int num_sms, cudaStream_t stream);
// grouped variant: `grp.count` problems, tile_start filled in by the launcher
cudaError_t launch_fused_gemm_group(int mode, int r_pad, int cta_group, FusedGemmGroup& grp, int num_sms,
                                    cudaStream_t stream);

// B6: b8 [m, roundup(r, 8)] = B zero-padded (fwd, only when r % 8 != 0: TMA
// row pitch must be a multiple of 16 bytes); bt [r, m] = B^T (dx narrow
// operand, K-major).  Either output may be null.
cudaError_t launch_pack_b(const __nv_bfloat16* b, int64_t m, int r, __nv_bfloat16* b8, __nv_bfloat16* bt,
                          int num_sms, cudaStream_t stream, const float* coef = nullptr,
                          __nv_bfloat16* cs = nullptr, int64_t T = 0, int64_t t_pad = 0);
// (coef != null, r % 8 == 0: the same launch also writes K3's exact split of coef [T, r]
//  into cs [3 r, t_pad] -- the dX-free backward's h, saving the K3s pass)



enum : int { kAccA = 1, kAccB = 2 };   // GradArgs::accumulate bits

struct GradArgs {
    const __nv_bfloat16* x;   // [T, n]
    const float* gh;          // [T, r]   (dA coefficients, already scaled by s)
    const __nv_bfloat16* dy;  // [T, m]
    const float* h;           // [T, r]   (dB coefficients, unscaled)
    float* da;                // [r, n] or null
    float* db;                // [m, r] or null
    int64_t T, n, m;
    int r;
    float scale_b;            // s
    int accumulate;           // bit mask: kAccA adds into da, kAccB adds into db (else overwrite)
    __nv_bfloat16* cs_a;      // tensor-core K3: split gh [3 r8, T_pad] (workspace)
    __nv_bfloat16* cs_b;      // tensor-core K3: split h  [3 r8, T_pad] (workspace)
    float scale_a;            // dA multiplier (1, or q = 1/(1-p) when x is the dropout-masked M . x)
    int cs_a_ready, cs_b_ready;   // split already written (by K2 or a row projection): no K3s work for that set
    int cs_a_k2, cs_b_k2;         // ... written by THIS backward's K2, which raises k2_flags per row block
                                  // (only those sets wait on the flags; a row projection's split is
                                  // ordered by the stream and K2 may already have reset its flags)
    const uint64_t* k2_flags;     // K2's per-row-block flags (value 1 once cs_* are written), or null
    int k2_nflags;
};
// several problems of the same rank bucket in one K3 launch
struct GradGroup {
    GradArgs g[kMaxGroup];
    int block_start[kMaxGroup + 1];
    int blocks_a[kMaxGroup];
    int count;
};
// K3 on the tensor cores (default): O[c, q] = scale * sum_t X[t, c] C[t, q].
// A JOB is one bf16 activation X [T, N] (xmap: box {64 columns, 64 tokens},
// SWIZZLE_128B) with the coefficient SETS stacked along the MMA N dimension:
// set j occupies B-operand rows [row0, row0 + 3 r8) (hi, mid, lo), loaded by
// TMA from its split array Cs [3 r8, T_pad] bf16 (csmap: box {64 tokens,
// 3 r8 rows}, SWIZZLE_128B) that K3s wrote.
#ifndef LORA_K3_COLS
#define LORA_K3_COLS 128
#endif
constexpr int kGradMmaCols = LORA_K3_COLS;   // X columns per CTA (one M = 128 MMA per 128)
constexpr int kMaxGradJobs = 16;
constexpr int kMaxGradSetsTotal = 16;
struct GradMmaSet {
    float* out;                 // O[c, k] at out[c * stride_col + k * stride_k]
    int64_t stride_col, stride_k;
    int r, r8, row0, accumulate;
    float scale;
    int nsplit;                 // 3: rows hi / mid / lo of an fp32 coefficient (K3s); 1: a bf16 operand as is
    // the dX kernel (K2) of the same backward writes this set's split coefficients
    // and raises wait_flags[0 .. wait_n) to 1 per row block: K3 waits on them before
    // its first coefficient load (lets K3 start while K2 is still running; else null)
    const uint64_t* wait_flags;
    int wait_n;
    // optional (row projections): also write the exact hi / mid / lo bf16 split of
    // scale * O[c, k] to cs_out [3 r8, cs_t_pad] (K3's coefficient operand; rows
    // k < r only -- used when r == r8, so no pad rows exist)
    __nv_bfloat16* cs_out;
    int64_t cs_t_pad;
};
struct GradMmaJob {
    int64_t T, N;               // T: reduction extent (k-blocks of 64), N: output extent (MMA M, 128 per CTA)
    int set0, nsets;            // sets [set0, set0 + nsets) of the group
    int q_used, q_pad;          // q_used = sum nsplit r8; q_pad = roundup(q_used, 16) (MMA N, <= 256)
    int a_kmajor;               // 0: X [T, N] read MN-major (dA, dB); 1: X [N, T] read K-major (row projections)
};
struct GradMmaGroup {
    CUtensorMap xmap[kMaxGradJobs];
    CUtensorMap csmap[kMaxGradSetsTotal];
    GradMmaSet set[kMaxGradSetsTotal];
    unsigned long long* done;   // sync-pool launch counter: the last CTA out zeroes every set's wait_flags
    GradMmaJob job[kMaxGradJobs];
    int tile_start[kMaxGradJobs + 1];
    int njobs;
    // filled in by launch_grad_mma
    int S, stages, stage_bytes, region_bytes, tmem_cols;
};
// overlap_prev: launch with programmatic stream serialization, so K3's CTAs
// fill the SMs the preceding K2 frees in its last wave; only legal when every
// set that K2 produces carries wait_flags and nothing else runs in between.
cudaError_t launch_grad_mma(GradMmaGroup& G, int num_sms, cudaStream_t stream, bool overlap_prev = false);
int grad_mma_cluster_size(int tiles, int kb_total, const int* slots /* [9], by cluster size */);

// K3s: cs [3 r8, T_pad] bf16 = exact hi / mid / lo split of coef [T, r] fp32
// (rows k, r8 + k, 2 r8 + k; zero for k >= r and tokens >= T).
struct CoefSplitArgs {
    const float* coef;
    __nv_bfloat16* cs;
    int64_t T, T_pad;
    int r, r8;
};
struct CoefSplitGroup {
    CoefSplitArgs s[kMaxGradSetsTotal];
    int count;
};
cudaError_t launch_coef_split(const CoefSplitGroup& G, cudaStream_t stream);

GradArgs make_grad_args(int64_t T, int64_t n, int64_t m, int r, float scale, const __nv_bfloat16* x,
                        const float* gh, const __nv_bfloat16* dy, const float* h, float* da, float* db,
                        int accumulate);
int grad_rank_bucket(int r);
cudaError_t launch_grad_reduce_cluster_group(GradGroup& G, cudaStream_t stream, int* launches);

// CUDA-core K3 (LORA_K3=cluster): T split over a cluster of 8 CTAs, DSMEM reduction in rank order.
cudaError_t launch_grad_reduce_cluster(int64_t T, int64_t n, int64_t m, int r, float scale,
                                       const __nv_bfloat16* x, const float* gh, const __nv_bfloat16* dy,
                                       const float* h, float* da, float* db, int accumulate,
                                       cudaStream_t stream, int* launches);
// K4: w_out = bf16(W0 + s * B A)
cudaError_t launch_merge(const __nv_bfloat16* w0, const __nv_bfloat16* a, const __nv_bfloat16* b,
                         int64_t n, int64_t m, int r, float scale, __nv_bfloat16* w_out,
                         cudaStream_t stream);

// column tiles of a fused-GEMM output (lora_gemm.cu ColTiles): starts[0..count], starts[count] = n_out
int fused_gemm_col_tiles(int mode, int r_pad, int64_t n_out, int* starts, int max);

// Comm-fused epilogue reducer (lora_symm.cu): sums the 128-row
// output units the fused GEMMs of every rank (and every member of a group)
// published into their symmetric partial regions, in (rank, member) order in
// fp32, rounds once to bf16 and stores the result into every rank's output
// region.  Unit u (flag index n_blk * nrow128 + row128) is reduced by rank u % N.
constexpr int kSymmMaxRanks = 8;
constexpr int kSymmMaxColTiles = 256;
struct SymmReduceArgs {
    int nranks, rank, nsrc;
    int nrow128, ncol_tiles, units;
    int64_t T, ncols, ld;
    int col_start[kSymmMaxColTiles + 1];
    const __nv_bfloat16* part[kSymmMaxRanks][kMaxGroup];
    uint32_t* flags[kSymmMaxRanks];      // rank r's unit flags, [member][units]
    __nv_bfloat16* out[kSymmMaxRanks];
    uint32_t* done[kSymmMaxRanks];       // rank r's launch counter
};
cudaError_t launch_symm_reduce(const SymmReduceArgs& A, int ctas, int variant, cudaStream_t stream);
// which reducer variant fits next to one CTA of the GEMM (regs per thread, warps):
// 0 (fat), 1 (lean), or -1 (none: the reducer must run after the GEMM)
cudaError_t symm_reducer_plan(int gemm_regs, int gemm_warps, int* variant);
// registers per thread of the fused-GEMM instantiation (mode, r_pad, CTA group)
int fused_gemm_regs(int mode, int r_pad, int cta_group);
// load every kernel the fused TP paths launch while a reducer may be spinning (lazy
// module loading would otherwise load them at first launch, which waits for the
// device to drain -- i.e. for the spinning reducer: a deadlock)
cudaError_t preload_gemm_kernels();
cudaError_t preload_grad_kernels();
cudaError_t preload_grad_mma_kernels();

// K4 on the tensor cores (lora_merge_mma.cu; r % 8 == 0, r <= 64): TMA maps of
// W0 [m, n] and W' [m, n] (box 64 x 128, SW128), B [m, r] (box r_pad x 128,
// swizzle 2 r_pad bytes), A [r, n] (box 64 x r_pad, SW128)
struct MergeMaps {
    CUtensorMap w, out, b, a;
};
cudaError_t launch_merge_mma(const MergeMaps& maps, int r_pad, int64_t m, int64_t n, float s, int num_sms,
                             cudaStream_t stream);

// decoder-layer pieces (lora_layer.cu)
cudaError_t launch_rmsnorm_fwd(const __nv_bfloat16* x, const __nv_bfloat16* res, const __nv_bfloat16* g, int64_t T,
                               int d, float eps, __nv_bfloat16* y, __nv_bfloat16* x2_out, float* rstd,
                               cudaStream_t stream);
cudaError_t launch_rmsnorm_bwd(const __nv_bfloat16* dy, const __nv_bfloat16* x2, const __nv_bfloat16* g,
                               const float* rstd, const __nv_bfloat16* dres, int64_t T, int d, __nv_bfloat16* dx,
                               cudaStream_t stream);
cudaError_t launch_rope(__nv_bfloat16* q, int64_t T, int heads, int D, int64_t ld, int64_t pos0, float theta,
                        int inverse, int num_sms, cudaStream_t stream);
cudaError_t launch_swiglu_fwd(const __nv_bfloat16* gate, const __nv_bfloat16* up, int64_t count, __nv_bfloat16* out,
                              int num_sms, cudaStream_t stream);
cudaError_t launch_swiglu_bwd(const __nv_bfloat16* gate, const __nv_bfloat16* up, const __nv_bfloat16* da,
                              int64_t count, __nv_bfloat16* dgate, __nv_bfloat16* dup, int num_sms,
                              cudaStream_t stream);

// N3: one Adam step for up to kMaxAdamTensors adapter tensors (numel % 4 == 0)
constexpr int kMaxAdamTensors = 64;
struct AdamTensor {
    __nv_bfloat16* param;
    float* master;      // may be null
    const float* grad;
    float* m;
    float* v;
    int64_t numel;
};
struct AdamGroup {
    AdamTensor t[kMaxAdamTensors];
    int64_t start4[kMaxAdamTensors + 1];   // filled in by launch_adam
    int count;
    float lr, b1, b2, eps, bc1, bc2;        // bc = 1 - beta^t
};
cudaError_t launch_adam(AdamGroup& G, int num_sms, cudaStream_t stream);

// dst = RNE_bf16(sum of n bf16 tensors of `count` elements, count % 8 == 0), fp32 accumulation
struct SumBf16Args {
    const __nv_bfloat16* src[kMaxGroup];
    __nv_bfloat16* dst;
    int64_t count;
    int n;
};
cudaError_t launch_sum_bf16(const SumBf16Args& A, int num_sms, cudaStream_t stream);

// dst += src (fp32), used by the TP backward when accumulating reduced grads
cudaError_t launch_add_f32(float* dst, const float* src, int64_t count, cudaStream_t stream);

// K0 (dropout): h = q (M . x) A^T [T, r] fp32, xm = M . x [T, n] bf16 and the keep bits
// [T, ceil(n/32)] uint32 (bit c of word w = keep(t, 32 w + c)); any output may be null
// K0 for several linears that share x (each its own mask and outputs), one launch
struct DropoutMember {
    const __nv_bfloat16* a;
    int r;
    DropoutParams drop;
    float* h;
    __nv_bfloat16* xm;
    uint32_t* bits;          // keep bits out (fwd: the caller's buffer; bwd: K2's)
    const uint32_t* bits_in; // bwd: the forward's keep bits -- read instead of drawn
    PhiloxKeys keys;         // (filled by the launcher from drop)
};
struct DropoutGroup {
    const __nv_bfloat16* x;
    int64_t T, n;
    int count;
    DropoutMember m[kMaxGroup];
};
cudaError_t launch_dropout_input_group(const DropoutGroup& G, int num_sms, cudaStream_t stream, int* launches);
// keep mask M [T, n] uint8 (for lora_dropout_mask)
cudaError_t launch_dropout_mask(int64_t T, int64_t n, const DropoutParams& d, uint8_t* mask, int num_sms,
                                cudaStream_t stream);

// zero-fill helper for degenerate (T == 0) gradients
cudaError_t launch_fill_zero(float* p, int64_t count, cudaStream_t stream);

}  // namespace lora_sm100
