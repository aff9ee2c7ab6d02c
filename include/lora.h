/*
 * include/lora.h -- C ABI of liblora.so: the B200 (sm_100a) hot path of JORA
 * (arXiv 2403.11366), the LoRA-adapted projection and its backward.
 *
 * The operation (PAPER.md = the paper text, /root/reference/PAPER.md):
 *   PAPER.md:109 (Sec. 3): frozen W0 in R^{m x n}, trainable A in R^{r x n},
 *     B in R^{m x r}, r << m, n; W0 x + b0 is tuned to W0 x + b0 + B A x.
 *   PAPER.md:115-120 (Eq. 1): Output = W0 x + b0 + B A x = (W0 + B A) x + b0.
 *   only A and B are trained (no gradient for W0, b0).
 *   PAPER.md:80-81 (Listing 3): LORA_R, LORA_ALPHA -> s = alpha / r.
 * Row-vector orientation used here (R1), for T tokens:
 *   forward : h = x A^T [T,r];  y = x W0^T + s h B^T (+ b0)          [T,m]
 *   backward: gh = s dy B [T,r]; dx = dy W0 + gh A [T,n];
 *             dA = gh^T x [r,n]; dB = s dy^T h [m,r]
 *   merge   : W' = W0 + s B A [m,n]   (Eq. 1 line 2; PAPER.md:92-106 export)
 *
 * Conventions for every call:
 *   - Tensor pointers are DEVICE pointers to row-major, contiguous tensors.
 *     "bf16" tensors hold IEEE bfloat16 values (2 bytes each); fp32 tensors
 *     hold float.  The caller owns all memory; the library never allocates
 *     device memory inside a call (scratch comes from `workspace`, whose
 *     contents need no initialisation).  Cross-CTA / cross-kernel flags live
 *     in a 2 MiB static device pool inside liblora.so (zero at load, returned
 *     to zero by every launch chain that uses it), so calls may be captured
 *     into CUDA graphs and replayed with new inputs; words taken during a
 *     capture belong to that graph until it is destroyed.
 *   - *_workspace_bytes() depend only on the dims -- and on the experimental
 *     environment switch LORA_STREAMK=1 (stream-K tail schedule), which adds
 *     148 fp32 128x256 partial slots (18.9 MB) for launches of >= 32 tiles:
 *     query the size in the same environment the calls run in.
 *   - Every device pointer must be 16-byte aligned.  d_in and d_out must be
 *     multiples of 8 (so bf16 rows are 16-byte multiples, as TMA requires);
 *     1 <= rank <= 64; tokens >= 0.  Violations -> LORA_ERR_SHAPE /
 *     LORA_ERR_ALIGN / LORA_ERR_UNSUPPORTED, returned before anything is
 *     launched and with no output written.
 *   - `stream` is a cudaStream_t (NULL = legacy default stream).  All work
 *     is enqueued asynchronously on it; asynchronous faults surface at the
 *     caller's synchronisation.  A failed launch returns LORA_ERR_CUDA.
 *   - Outputs must not alias inputs (the one exception: lora_merge with
 *     w_out == w0, an explicit in-place merge).
 *   - lora_last_error() returns a thread-local, human-readable description of
 *     the last failure (names the offending shapes / pointers).
 *   - y and dx are rounded once to bf16 (round-to-nearest-even); h, gh, dA,
 *     dB are fp32; all products accumulate in fp32 (R4, R5).
 */
#ifndef LORA_B200_H_
#define LORA_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    LORA_OK = 0,
    LORA_ERR_INVALID = 1,     /* NULL required pointer, bad enum, bad comm */
    LORA_ERR_SHAPE = 2,       /* non-positive / non-multiple-of-8 dims, shard mismatch */
    LORA_ERR_ALIGN = 3,       /* a pointer is not 16-byte aligned */
    LORA_ERR_UNSUPPORTED = 4, /* rank > 64, device is not sm_100 */
    LORA_ERR_CUDA = 5,        /* CUDA runtime/driver failure */
    LORA_ERR_NCCL = 6,        /* NCCL failure */
    LORA_ERR_WORKSPACE = 7    /* workspace NULL or smaller than *_workspace_bytes() */
} lora_status;

/* One LoRA linear.  tokens = T (batch x seq), d_in = n, d_out = m, rank = r,
 * alpha = the LoRA alpha of Listing 3; s = alpha / rank is
 * computed in fp32. */
typedef struct {
    int64_t tokens;
    int64_t d_in;
    int64_t d_out;
    int32_t rank;
    float alpha;
} lora_dims;

/* Bytes of device scratch lora_linear_fwd needs for `dims` (O(d_out * 64)). */
size_t lora_linear_fwd_workspace_bytes(const lora_dims* dims);

/*
 * Forward, Eq. 1 line 1:  y = x W0^T + s (x A^T) B^T (+ bias)
 *   x    [T, n] bf16     w0 [m, n] bf16     a [r, n] bf16     b [m, r] bf16
 *   bias [m] bf16 or NULL (Llama-2 projections have none)
 *   y    [T, m] bf16 (out)
 *   h_out [T, r] fp32 (out, optional): h = x A^T, unscaled, saved for the
 *         backward (dB = s dy^T h); NULL skips the store.
 * One fused launch computes x W0^T and x A^T in the same tensor-core pass and
 * adds (s h) B^T in its epilogue (kernel K1).
 */
lora_status lora_linear_fwd(const lora_dims* dims, const void* x, const void* w0,
                            const void* a, const void* b, const void* bias,
                            void* y, float* h_out,
                            void* workspace, size_t workspace_bytes, void* stream);

/* Bytes of device scratch lora_linear_bwd needs for `dims`. */
size_t lora_linear_bwd_workspace_bytes(const lora_dims* dims);

/*
 * Backward of Eq. 1 for trainable A, B and frozen W0, b0:
 *   dy      [T, m] bf16      upstream gradient
 *   h_saved [T, r] fp32      h from lora_linear_fwd, or NULL (recomputed)
 *   dx      [T, n] bf16 out  dy W0 + gh A, or NULL (input grad not needed)
 *   da      [r, n] fp32 out  gh^T x            (NULL skips)
 *   db      [m, r] fp32 out  s dy^T h          (NULL skips)
 *   accumulate: 0 overwrite da/db, 1 add into them (gradient accumulation).
 * No gradient for W0 or bias is produced (frozen base).
 */
lora_status lora_linear_bwd(const lora_dims* dims, const void* x, const void* w0,
                            const void* a, const void* b, const float* h_saved,
                            const void* dy, void* dx, float* da, float* db,
                            int accumulate,
                            void* workspace, size_t workspace_bytes, void* stream);

/*
 * Merge for export, Eq. 1 line 2 (script PAPER.md:92-106):
 *   w_out[i,k] = RNE_bf16( W0[i,k] + s * sum_j B[i,j] A[j,k] ), fp32 math.
 * dims->tokens is ignored.  w_out == w0 performs the merge in place;
 * otherwise w_out must not overlap any input.  The bias is unaffected.
 */
lora_status lora_merge(const lora_dims* dims, const void* w0, const void* a,
                       const void* b, void* w_out, void* stream);

/* ---------------- Adapter update ----------------------------
 * One bias-corrected Adam step (Kingma & Ba, ICLR 2015, Algorithm 1; the paper
 * names no optimizer) for up to LORA_ADAM_MAX_TENSORS
 * adapter tensors (every A and B of a model) in ONE launch, fp32 arithmetic:
 *   m <- b1 m + (1-b1) g;  v <- b2 v + (1-b2) g^2
 *   theta <- theta - lr (m / (1-b1^step)) / (sqrt(v / (1-b2^step)) + eps)
 *   param <- RNE_bf16(theta)      (the bf16 A / B the fused kernels read)
 * theta is `master` (fp32 master weights) when non-NULL, else `param` itself.
 * grad is the dA / dB of lora_linear_bwd (after any TP all-reduce).  numel must
 * be a multiple of 4 (A [r,n], B [m,r] with n, m multiples of 8 always are);
 * pointers 16-byte aligned; step >= 1; lr >= 0; 0 <= beta < 1; eps >= 0.
 * Only adapters have optimizer state; W0 is never touched. */
#define LORA_ADAM_MAX_TENSORS 64
typedef struct {
    void* param;          /* bf16 [numel], updated */
    float* master;        /* fp32 [numel] master weights, updated; or NULL */
    const float* grad;    /* fp32 [numel] */
    float* m;             /* fp32 [numel] first moment, updated */
    float* v;             /* fp32 [numel] second moment, updated */
    int64_t numel;
} lora_adam_tensor;
typedef struct {
    float lr, beta1, beta2, eps;
} lora_adam_hparams;
lora_status lora_adam_step(int count, const lora_adam_tensor* tensors, const lora_adam_hparams* hparams,
                           int64_t step, void* stream);

/* ---------------- LoRA dropout (Listing 3 LORA_DROPOUT = 0.05) ----
 * Inverted dropout on the ADAPTER input only (reading R7; the frozen
 * path W0 x never sees it).  Keep mask M[t,k] in {0,1}, q = 1 / (1 - p):
 *   y  = x W0^T + s (q (M . x) A^T) B^T (+ bias),   h = q (M . x) A^T
 *   dX = dy W0 + q M . (gh A),   dA = q gh^T (M . x),   dB = s dy^T h
 * M is a pure function of (t, k, seed, offset, p) -- Philox4x32-10 with
 * counter (k/8, t, offset_lo, offset_hi) and key (seed_lo, seed_hi) gives eight
 * 16-bit draws u = (word (k%8)/2 >> 16 (k%2)) & 0xFFFF; element (t, k) is kept
 * iff u >= floor(p * 2^16) (p resolved to 2^-16) -- so the backward, given
 * the same lora_dropout, regenerates the forward's mask (nothing needs to be
 * stored).  Optionally the caller keeps the mask instead: keep_bits, a device
 * buffer of tokens x ceil(d_in / 32) uint32 (bit c of word w of row t =
 * M[t, 32 w + c]; 16-byte aligned; owned by the caller), is WRITTEN by the
 * forward calls and READ by the backward calls (which then draw nothing: the
 * buffer must hold the bits the forward wrote with the same p, seed, offset).
 * NULL: the backward redraws.  T n / 8 bytes per linear (1 MB at 2048 x 4096).
 * Likewise masked_x, a device buffer of tokens x d_in bf16 (16-byte aligned):
 * the forward writes M . x there (exact: zeroing only) and the backward reads
 * it for dA instead of masking x again (2 T n bytes per linear, what a framework
 * saves for the adapter's backward anyway).  With both buffers and h_saved the
 * backward draws and masks nothing.  Both are untouched when p = 0.
 * A shard or token slice of a larger input (TP row mode shards x on d_in) passes
 * its position (row_offset, col_offset) so every shard draws its part of the one
 * mask of the full input; keep_bits / masked_x then have the local shape.
 * Use a fresh offset (or seed) per step and per linear.  p = 0 gives exactly
 * the plain calls.  p must be in [0, 1) (LORA_ERR_INVALID otherwise). */
typedef struct {
    float p;          /* drop probability */
    uint64_t seed;    /* Philox key */
    uint64_t offset;  /* Philox counter high words: a stream per (step, linear) */
    uint32_t* keep_bits;  /* optional: [tokens, ceil(d_in/32)] keep mask, fwd writes / bwd reads */
    void* masked_x;       /* optional: [tokens, d_in] bf16 M . x, fwd writes / bwd reads */
    int64_t row_offset;   /* where this call's x sits in the full adapter input: element (t, k) */
    int64_t col_offset;   /*   draws the mask of (t + row_offset, k + col_offset); >= 0,
                             col_offset % 8 == 0 (tensor-parallel shards, token slices; 0 = whole) */
} lora_dropout;

/* As lora_linear_fwd, plus one launch (K0: h from the masked input). */
size_t lora_linear_fwd_dropout_workspace_bytes(const lora_dims* dims);
lora_status lora_linear_fwd_dropout(const lora_dims* dims, const lora_dropout* dropout,
                                    const void* x, const void* w0, const void* a, const void* b,
                                    const void* bias, void* y, float* h_out,
                                    void* workspace, size_t workspace_bytes, void* stream);
/* As lora_linear_bwd (h_saved must come from lora_linear_fwd_dropout with the
 * same dropout, or NULL); the workspace also holds M . x [T, n] bf16. */
size_t lora_linear_bwd_dropout_workspace_bytes(const lora_dims* dims);
lora_status lora_linear_bwd_dropout(const lora_dims* dims, const lora_dropout* dropout,
                                    const void* x, const void* w0, const void* a, const void* b,
                                    const float* h_saved, const void* dy, void* dx, float* da, float* db,
                                    int accumulate, void* workspace, size_t workspace_bytes, void* stream);
/* The keep mask M [tokens, d_in] (uint8 0/1, device memory) the calls above use. */
lora_status lora_dropout_mask(int64_t tokens, int64_t d_in, const lora_dropout* dropout, uint8_t* mask,
                              void* stream);

/* ---------------- Grouped calls: several independent LoRA linears ----------
 * Equivalent to `count` single calls -- y, h and dX bitwise identical; dA and
 * dB identical up to fp32 re-association (the dA/dB kernel's token split is
 * chosen for the whole launch, so a group may sum the token partials in
 * other chunks than a single call; repeated calls are bitwise reproducible) --
 * but the fused tensor-core GEMMs of all problems whose rank falls in the same
 * 16/32/64 bucket (and with the same T > 128 or not) run as ONE persistent
 * launch, which removes per-launch prologue / tail time.  Typical use: the
 * projections that share an input (q, k, v; gate, up).  Problems must not
 * alias each other's outputs.  Workspace: the *_grouped_workspace_bytes()
 * of the same dims array (problem g uses its own slice). */
#define LORA_MAX_GROUP 8
typedef struct {
    const void* x; const void* w0; const void* a; const void* b; const void* bias;  /* as lora_linear_fwd */
    void* y; float* h_out;
} lora_fwd_problem;
typedef struct {
    const void* x; const void* w0; const void* a; const void* b; const float* h_saved;  /* as lora_linear_bwd */
    const void* dy; void* dx; float* da; float* db;
} lora_bwd_problem;

size_t lora_linear_fwd_grouped_workspace_bytes(int count, const lora_dims* dims);
lora_status lora_linear_fwd_grouped(int count, const lora_dims* dims, const lora_fwd_problem* problems,
                                    void* workspace, size_t workspace_bytes, void* stream);
size_t lora_linear_bwd_grouped_workspace_bytes(int count, const lora_dims* dims);
lora_status lora_linear_bwd_grouped(int count, const lora_dims* dims, const lora_bwd_problem* problems,
                                    int accumulate, void* workspace, size_t workspace_bytes, void* stream);

/* Grouped calls with LoRA dropout (Listing 3 LORA_DROPOUT; R7): one
 * lora_dropout per problem (each linear draws its own mask: its own seed /
 * offset); p must be > 0 for all problems or for none (one dX kernel mode per
 * group).  Same semantics as `count` lora_linear_{fwd,bwd}_dropout calls, with
 * the fused GEMMs of the group in one launch. */
size_t lora_linear_fwd_grouped_dropout_workspace_bytes(int count, const lora_dims* dims);
size_t lora_linear_bwd_grouped_dropout_workspace_bytes(int count, const lora_dims* dims);
lora_status lora_linear_fwd_grouped_dropout(int count, const lora_dims* dims, const lora_dropout* dropouts,
                                            const lora_fwd_problem* problems, void* workspace, size_t workspace_bytes,
                                            void* stream);
lora_status lora_linear_bwd_grouped_dropout(int count, const lora_dims* dims, const lora_dropout* dropouts,
                                            const lora_bwd_problem* problems, int accumulate, void* workspace,
                                            size_t workspace_bytes, void* stream);

const char* lora_status_string(lora_status status);
const char* lora_last_error(void);

/* Library / device information.  lora_device_check returns LORA_OK if the
 * current CUDA device is sm_100 (B200), LORA_ERR_UNSUPPORTED otherwise. */
int lora_version(void);
lora_status lora_device_check(void);

/* Number of kernel launches the last fwd / bwd / merge call on this thread
 * enqueued (for the bench's gpu_launches accounting). */
int lora_last_launch_count(void);

/* Free words (8 bytes each) of the sync-pool region that calls made during CUDA
 * graph capture draw from (131072 words per device).  Each captured backward
 * takes ~16-80 words for its cross-CTA flags; they belong to the capturing
 * graph and are returned when that graph and every executable instantiated
 * from it are destroyed, so re-capturing never exhausts the region.  A capture
 * that finds the region full (too many LIVE graphs) fails with LORA_ERR_CUDA.
 * Diagnostics for tests; -1 if no CUDA device is current. */
int lora_captured_sync_words_free(void);

/* Measurement hook (bench.py's in-step roofline of the dX kernel): the next
 * backward call on this thread (lora_linear_bwd, lora_linear_bwd_grouped, or
 * the TP backward calls) records events[0] / events[1] (cudaEvent_t, may be
 * NULL) on its stream right before / after the fused dX kernel (K2) launch and
 * events[2] / events[3] around the dA / dB kernel (K3).  One-shot: cleared when
 * that call returns.  Recording between K2 and K3 stops K3 from starting in
 * K2's last wave, so these events time each kernel on its own. */
lora_status lora_profile_next_bwd(void* const events[4]);

/* ---------------- Tensor parallelism (R10-R13) ------
 * One process per GPU.  COLUMN: W0 and B sharded on d_out, A replicated;
 * ROW: W0 and A sharded on d_in, B replicated.  `local` holds the LOCAL shard
 * dims (column: d_out / N; row: d_in / N).  Collectives are NCCL all-reduces
 * (sum) over NVLink on `stream`:
 *   COLUMN fwd: none.             COLUMN bwd: dx (bf16), dA (fp32).
 *   ROW    fwd: y (bf16).         ROW    bwd: dB (fp32).
 * The LoRA-gradient all-reduce is a SUM with no 1/N (R12); pass
 * reduce_lora_grads = 0 to leave it to a bucketed lora_allreduce call. */
typedef struct lora_comm lora_comm;
typedef enum { LORA_TP_COLUMN = 0, LORA_TP_ROW = 1 } lora_tp_mode;
typedef enum { LORA_DT_F32 = 0, LORA_DT_BF16 = 1 } lora_dtype;

#define LORA_COMM_ID_BYTES 128
lora_status lora_comm_unique_id(uint8_t id[LORA_COMM_ID_BYTES]);
lora_status lora_comm_init(int nranks, int rank, const uint8_t id[LORA_COMM_ID_BYTES],
                           lora_comm** out);
lora_status lora_comm_destroy(lora_comm* comm);
int lora_comm_size(const lora_comm* comm);
int lora_comm_rank(const lora_comm* comm);

/* In-place sum all-reduce of `count` elements of `dtype`. */
lora_status lora_allreduce(lora_comm* comm, void* buf, size_t count, lora_dtype dtype,
                           void* stream);

/* Row mode: only rank 0 adds the bias (it is not sharded).  Row mode with
 * N > 1 and T >= 4096 runs in 4 token slices (multiples of 256 rows; LORA_TP_CHUNKS=k
 * overrides): slice i's y all-reduce runs on the communicator's side stream while
 * the GEMM of slice i + 1 runs on `stream` (joined before return).  y and h are
 * the same as unsliced, bit for bit (rows are independent). */
lora_status lora_tp_linear_fwd(lora_comm* comm, lora_tp_mode mode, const lora_dims* local,
                               const void* x, const void* w0, const void* a, const void* b,
                               const void* bias, void* y, float* h_out,
                               void* workspace, size_t workspace_bytes, void* stream);

/* Workspace for lora_tp_linear_bwd: lora_linear_bwd_workspace_bytes(local)
 * plus fp32 scratch for the reduced partial gradient. */
size_t lora_tp_linear_bwd_workspace_bytes(const lora_dims* local);

lora_status lora_tp_linear_bwd(lora_comm* comm, lora_tp_mode mode, const lora_dims* local,
                               const void* x, const void* w0, const void* a, const void* b,
                               const float* h_saved, const void* dy, void* dx,
                               float* da, float* db, int accumulate, int reduce_lora_grads,
                               void* workspace, size_t workspace_bytes, void* stream);

/* Tensor-parallel calls with LoRA dropout (Listing 3; R7).
 * `dropout` describes the FULL adapter input's mask (p, seed, offset, row/col
 * offsets of the full input, usually 0); ROW mode adds rank * local->d_in to its
 * col_offset (x is sharded on d_in), so the shards' masks are the slices of one
 * mask and the all-reduced result equals the unsharded dropout call.  keep_bits /
 * masked_x, if given, are LOCAL buffers ([T, ceil(local d_in / 32)], [T, local
 * d_in]).  Otherwise as lora_tp_linear_fwd / lora_tp_linear_bwd (workspaces: the
 * *_dropout_workspace_bytes of the local dims, plus the bwd scratch). */
size_t lora_tp_linear_bwd_dropout_workspace_bytes(const lora_dims* local);
lora_status lora_tp_linear_fwd_dropout(lora_comm* comm, lora_tp_mode mode, const lora_dims* local,
                                       const lora_dropout* dropout, const void* x, const void* w0, const void* a,
                                       const void* b, const void* bias, void* y, float* h_out,
                                       void* workspace, size_t workspace_bytes, void* stream);
lora_status lora_tp_linear_bwd_dropout(lora_comm* comm, lora_tp_mode mode, const lora_dims* local,
                                       const lora_dropout* dropout, const void* x, const void* w0, const void* a,
                                       const void* b, const float* h_saved, const void* dy, void* dx,
                                       float* da, float* db, int accumulate, int reduce_lora_grads,
                                       void* workspace, size_t workspace_bytes, void* stream);

/* Tensor-parallel backward of a COLUMN-parallel group of linears that read the
 * SAME input x (q, k, v or gate, up): the grouped local backward
 * (one fused dX launch, one dA/dB launch), then the members' dX partials summed
 * into dx_sum [T, d_in] bf16 (fp32 accumulation, one RNE) -- the gradient w.r.t.
 * the shared input -- and ONE all-reduce of dx_sum instead of one per member;
 * the members' partial dA are all-reduced in one NCCL group.  problems[g].x must
 * all be the same pointer; problems[g].dx are the members' own partials (kept);
 * dx_sum may be NULL (no dX wanted).  dB stays local (column mode).
 * accumulate with reduce_lora_grads is rejected (LORA_ERR_UNSUPPORTED: accumulate
 * locally with reduce_lora_grads = 0, then lora_allreduce the sums).  Workspace: lora_linear_bwd_grouped_workspace_bytes. */
size_t lora_tp_linear_bwd_column_group_workspace_bytes(int count, const lora_dims* local);
lora_status lora_tp_linear_bwd_column_group(lora_comm* comm, int count, const lora_dims* local,
                                            const lora_bwd_problem* problems, void* dx_sum, int accumulate,
                                            int reduce_lora_grads, void* workspace, size_t workspace_bytes,
                                            void* stream);

/* The column-group backward with LoRA dropout: one lora_dropout per problem (each
 * member's own mask of the replicated input; p > 0 for all or none), the same
 * forward masks (lora_linear_fwd_grouped_dropout or the TP calls).  Workspace:
 * lora_tp_linear_bwd_column_group_dropout_workspace_bytes. */
size_t lora_tp_linear_bwd_column_group_dropout_workspace_bytes(int count, const lora_dims* local);
lora_status lora_tp_linear_bwd_column_group_dropout(lora_comm* comm, int count, const lora_dims* local,
                                                    const lora_dropout* dropouts, const lora_bwd_problem* problems,
                                                    void* dx_sum, int accumulate, int reduce_lora_grads,
                                                    void* workspace, size_t workspace_bytes, void* stream);

/* ---------------- Comm-fused epilogues over peer memory ----
 * PAPER.md:199 blames the multi-GPU slowdown on "cross-GPU communication
 * overhead"; these calls fuse the two activation all-reduces of the TP linear
 * with the GEMM that produces them.  Each rank's fused GEMM writes its partial
 * output into a SYMMETRIC buffer and publishes every 128-row tile half as soon as
 * it is stored; a reducer kernel on a side stream (forked from and joined back to
 * `stream`) sums each published unit it owns (unit u -> rank u % N) over ranks
 * (and group members) in fp32, in rank order, rounds once to bf16 and stores it
 * into EVERY rank's output region with peer stores, while the GEMM computes
 * the next tiles.  All ranks end with bitwise identical results.
 *
 * lora_symm: one per rank, created with the same data_bytes everywhere
 * (device memory allocated by the library: [256 KiB control | data]); peers
 * are mapped with CUDA IPC (lora_symm_ipc_handle on every rank, all-gather the
 * handles, lora_symm_connect) or, to run the protocol on ONE GPU,
 * lora_symm_connect_local joins N buffers of this process as N virtual ranks
 * (each call then runs on its own stream).  Regions are given as byte offsets
 * into the data region (lora_symm_ptr): 16-byte aligned, inside it, disjoint.
 * One fused call at a time per lora_symm (calls on one stream are ordered).
 * The output region holds the result until the next fused call that writes it.
 * Errors: LORA_ERR_INVALID (not connected, wrong device, overlap),
 * LORA_ERR_SHAPE (region outside the buffer), LORA_ERR_ALIGN, LORA_ERR_CUDA. */
typedef struct lora_symm lora_symm;
#define LORA_SYMM_HANDLE_BYTES 64
lora_status lora_symm_create(size_t data_bytes, lora_symm** out);
lora_status lora_symm_ipc_handle(const lora_symm* symm, uint8_t handle[LORA_SYMM_HANDLE_BYTES]);
/* handles: nranks x LORA_SYMM_HANDLE_BYTES, rank order (this rank's own is ignored). */
lora_status lora_symm_connect(lora_symm* symm, int nranks, int rank, const uint8_t* handles);
lora_status lora_symm_connect_local(int nranks, lora_symm* const* group);
void* lora_symm_ptr(const lora_symm* symm);        /* this rank's data region (device) */
size_t lora_symm_bytes(const lora_symm* symm);
/* Where the last fused call's reducer ran (diagnostics): 1 co-resident with the
 * GEMM (overlapping it), 2 after the GEMM (no reducer variant fits next to that
 * GEMM's registers), 3 virtual ranks (GEMMs capped to SMs - 16, reducers on the
 * rest); 0 before any call. */
int lora_symm_last_placement(const lora_symm* symm);
lora_status lora_symm_destroy(lora_symm* symm);

/* ROW-parallel forward (o, down) with the y all-reduce fused into the GEMM:
 * the partial x_i W0_i^T + s (x_i A_i^T) B^T (+ bias on rank 0) goes to
 * [part_offset, + T d_out 2) of the data region, the reduced y [T, d_out] bf16
 * to [y_offset, ...) on every rank.  Other arguments as lora_tp_linear_fwd. */
lora_status lora_tp_linear_fwd_fused(lora_symm* symm, const lora_dims* local, const void* x, const void* w0,
                                     const void* a, const void* b, const void* bias, size_t part_offset,
                                     size_t y_offset, float* h_out, void* workspace, size_t workspace_bytes,
                                     void* stream);
/* COLUMN-parallel group backward (q/k/v, gate/up sharing x) with the dX
 * all-reduce fused into the grouped dX GEMM: member g's partial goes to
 * [part_offset + g T d_in 2, ...), the gradient w.r.t. the shared input,
 * sum over ranks and members, to [dx_offset, + T d_in 2) on every rank.
 * problems[g].dx must be NULL.  dA partials are all-reduced over `comm` (NCCL)
 * when reduce_lora_grads (comm may be NULL otherwise); dB stays local.
 * Workspace: lora_linear_bwd_grouped_workspace_bytes. */
lora_status lora_tp_linear_bwd_column_group_fused(lora_symm* symm, lora_comm* comm, int count,
                                                  const lora_dims* local, const lora_bwd_problem* problems,
                                                  size_t part_offset, size_t dx_offset, int reduce_lora_grads,
                                                  void* workspace, size_t workspace_bytes, void* stream);

/* ---------------- Merged-weight export ------------------
 * PAPER.md:86-106 (Listing 4, huggingface_merger.py): the fine-tuned LoRA
 * factors are folded into the base weights, W' = bf16(W0 + s B A) (Eq. 1 line 2,
 * PAPER.md:118), and the model is saved in a Hugging Face-loadable format.  The
 * file is safetensors: u64 little-endian header length, JSON header
 * {name: {"dtype", "shape", "data_offsets"}, "__metadata__": {"format": "pt"}}
 * padded with spaces to 8 bytes, then the raw tensors in order.
 *
 * lora_write_safetensors: HOST tensors, written as they are (CPU only).
 * lora_export_merged: DEVICE tensors; an entry with a and b non-NULL is merged on
 * the GPU (lora_merge: tensor cores; dims give d_out x d_in, rank, alpha; written
 * as BF16 [d_out, d_in]), an entry with a == b == NULL is copied as it is (dtype,
 * ndim, shape as given; w0 = the tensor).  The call allocates one device and one
 * pinned host staging buffer of the largest entry, synchronizes `stream` per
 * entry, and writes `path` (overwritten).  Names are the caller's (e.g.
 * "model.layers.0.self_attn.q_proj.weight").  Errors: LORA_ERR_INVALID (NULL
 * pointers, unwritable path), LORA_ERR_SHAPE, LORA_ERR_CUDA; a failed call may
 * leave a partial file. */
typedef struct {
    const char* name;
    int dtype;               /* lora_dtype */
    int ndim;                /* 1..4 */
    int64_t shape[4];
    const void* data;        /* host */
} lora_host_tensor;
typedef struct {
    const char* name;
    const void* w0;          /* device: the base weight (or the tensor itself) */
    const void* a;           /* device [rank, d_in] bf16, or NULL */
    const void* b;           /* device [d_out, rank] bf16, or NULL */
    lora_dims dims;          /* merged entries: d_out, d_in, rank, alpha (tokens ignored) */
    int dtype, ndim;         /* unmerged entries */
    int64_t shape[4];
} lora_export_tensor;
lora_status lora_write_safetensors(const char* path, int count, const lora_host_tensor* tensors);
lora_status lora_export_merged(const char* path, int count, const lora_export_tensor* tensors, void* stream);

/* ---------------- Decoder-layer pieces -------------------
 * The Llama-2 decoder layer (JORA builds on a Llama-2
 * implementation; :195 the long-sequence RAFT setting) around the seven LoRA
 * linears: RMSNorm, rotary position embedding, SwiGLU.  Device pointers, bf16
 * row-major, 16-byte aligned; fp32 math, one RNE per output.  The attention is
 * a library call (cuDNN SDPA) made by the Python layer.
 *
 * lora_rmsnorm_fwd: x2 = x + res (bf16; res may be NULL -> x2 = x; written to
 *   x2_out if non-NULL), rstd[t] = 1/sqrt(mean_k x2[t,k]^2 + eps) (fp32 [T]),
 *   y = g * (x2 * rstd).  dim % 8 == 0, 8 <= dim <= 8192.
 * lora_rmsnorm_bwd: dx = dres + rstd * (g.dy - xh * mean(xh * g.dy)),
 *   xh = x2 * rstd (g frozen: no dg; dres may be NULL).
 * lora_rope: in place on q [T, ld] (heads x head_dim used per row), pair
 *   (i, i + head_dim/2) of a head rotated by angle (pos0 + t) * theta^(-2i/head_dim);
 *   inverse = 1 applies the transposed rotation (the backward).
 * lora_swiglu_fwd: out = silu(gate) * up, count elements.
 * lora_swiglu_bwd: dgate = da * up * silu'(gate), dup = da * silu(gate). */
lora_status lora_rmsnorm_fwd(int64_t tokens, int64_t dim, float eps, const void* x, const void* res, const void* g,
                             void* y, void* x2_out, float* rstd, void* stream);
lora_status lora_rmsnorm_bwd(int64_t tokens, int64_t dim, const void* dy, const void* x2, const void* g,
                             const float* rstd, const void* dres, void* dx, void* stream);
lora_status lora_rope(int64_t tokens, int heads, int head_dim, int64_t ld, int64_t pos0, float theta, int inverse,
                      void* q, void* stream);
lora_status lora_swiglu_fwd(int64_t count, const void* gate, const void* up, void* out, void* stream);
lora_status lora_swiglu_bwd(int64_t count, const void* gate, const void* up, const void* da, void* dgate, void* dup,
                            void* stream);
/* dst = bf16(sum_i srcs[i]) over `count` elements (fp32 accumulation in i order,
 * one RNE; 1 <= n <= LORA_MAX_GROUP; dst may alias srcs[0]): residual adds and the
 * members' dX partials of a group sharing an input. */
lora_status lora_sum_bf16(int64_t count, int n, const void* const* srcs, void* dst, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* LORA_B200_H_ */
