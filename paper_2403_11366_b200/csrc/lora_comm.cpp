// lora_comm.cpp -- tensor-parallel LoRA linear over NCCL (NVLink 5 / NVSwitch).
//
// "JORA parallelizes all parameters ... Projection and
// Embedding layers are sharded on the non-sequential dimension."  Read as
// Megatron column/row parallelism inside the block (R10); A/B are
// sharded with the side of W0 they touch, the other factor is replicated
// (R11); partial results are SUMMED with no 1/N (R12).
//   COLUMN (q, k, v, gate, up): W0, B split on d_out; A replicated.
//     fwd  y_local = lora_fwd(local)                       -- no collective
//     bwd  dx = sum_ranks(dY_i W0_i + gh_i A)   all-reduce bf16 [T, n]
//          dA = sum_ranks(gh_i^T x)             all-reduce fp32 [r, n]
//          dB_i = s dY_i^T h                    local
//   ROW (o, down): W0, A split on d_in; B replicated.
//     fwd  y = sum_ranks(x_i W0_i^T + s (x_i A_i^T) B^T)   all-reduce bf16 [T, m]
//     bwd  dx_i, dA_i local; dB = sum_ranks(s dY^T h_i)   all-reduce fp32 [m, r]
// NCCL is resolved with dlopen at lora_comm_init, so single-GPU use of
// liblora.so never needs libnccl.
#include <dlfcn.h>
#include <nccl.h>

#include <cstdlib>
#include <cstring>

#include "lora_internal.h"
#include "lora_kernels.h"

using namespace lora_host;

namespace {

struct NcclApi {
    ncclResult_t (*GetUniqueId)(ncclUniqueId*);
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int);
    ncclResult_t (*CommDestroy)(ncclComm_t);
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t);
    const char* (*GetErrorString)(ncclResult_t);
    ncclResult_t (*GroupStart)();   // optional: batches several collectives into one launch
    ncclResult_t (*GroupEnd)();
    bool ok = false;
};

NcclApi* nccl() {
    static NcclApi api;
    static bool tried = false;
    if (tried) return api.ok ? &api : nullptr;
    tried = true;
    const char* cands[] = {getenv("LORA_NCCL_LIB"), "libnccl.so.2", "libnccl.so"};
    void* h = nullptr;
    for (const char* c : cands) {
        if (!c || !*c) continue;
        h = dlopen(c, RTLD_NOW | RTLD_GLOBAL);
        if (h) break;
    }
    if (!h) return nullptr;
    api.GetUniqueId = reinterpret_cast<decltype(api.GetUniqueId)>(dlsym(h, "ncclGetUniqueId"));
    api.CommInitRank = reinterpret_cast<decltype(api.CommInitRank)>(dlsym(h, "ncclCommInitRank"));
    api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(dlsym(h, "ncclCommDestroy"));
    api.AllReduce = reinterpret_cast<decltype(api.AllReduce)>(dlsym(h, "ncclAllReduce"));
    api.GetErrorString = reinterpret_cast<decltype(api.GetErrorString)>(dlsym(h, "ncclGetErrorString"));
    api.GroupStart = reinterpret_cast<decltype(api.GroupStart)>(dlsym(h, "ncclGroupStart"));
    api.GroupEnd = reinterpret_cast<decltype(api.GroupEnd)>(dlsym(h, "ncclGroupEnd"));
    api.ok = api.GetUniqueId && api.CommInitRank && api.CommDestroy && api.AllReduce && api.GetErrorString;
    return api.ok ? &api : nullptr;
}

lora_status nccl_fail(NcclApi* api, ncclResult_t r, const char* what) {
    return fail(LORA_ERR_NCCL, "%s: %s", what, api ? api->GetErrorString(r) : "NCCL unavailable");
}

size_t align256(size_t v) { return (v + 255) & ~size_t(255); }

}  // namespace

struct lora_comm {
    ncclComm_t comm;
    int nranks;
    int rank;
    // side stream + fork / join events: the column group's dX sum and all-reduce
    // run there, concurrently with the dA / dB kernel (created with the comm)
    cudaStream_t side = nullptr;
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
};

static_assert(sizeof(ncclUniqueId) == LORA_COMM_ID_BYTES, "NCCL unique id size");

// Token slices of the ROW-parallel forward (compute / all-reduce overlap): 4 when
// there is a peer to talk to and every slice keeps at least 1024 tokens (4 row
// blocks of 256: the GEMM of a slice still fills the GPU at the 8-way shard
// widths), else 1 -- at N = 1 the all-reduce is free and slicing only costs
// (cfg3 at N = 1: 2.40 -> 2.60 ms per step); LORA_TP_CHUNKS overrides.
static int tp_fwd_chunks(int64_t T, int nranks) {
    if (const char* v = getenv("LORA_TP_CHUNKS")) {
        const int k = atoi(v);
        return k >= 1 && k <= 64 ? k : 1;
    }
    return (nranks > 1 && T >= 4096) ? 4 : 1;
}

static lora_status allreduce_impl(lora_comm* c, void* buf, size_t count, lora_dtype dt, cudaStream_t st) {
    NcclApi* api = nccl();
    if (!api) return fail(LORA_ERR_NCCL, "libnccl could not be loaded (set LORA_NCCL_LIB)");
    if (count == 0) return LORA_OK;
    // (nranks == 1 still issues the collective: the single-rank path runs -- and is
    // graph-captured / timed -- exactly as at N > 1; NCCL's 1-rank all-reduce is a copy)
    ncclResult_t r = api->AllReduce(buf, buf, count, dt == LORA_DT_F32 ? ncclFloat32 : ncclBfloat16, ncclSum,
                                    c->comm, st);
    if (r != ncclSuccess) return nccl_fail(api, r, "ncclAllReduce");
    return LORA_OK;
}

extern "C" {

lora_status lora_comm_unique_id(uint8_t id[LORA_COMM_ID_BYTES]) {
    if (!id) return fail(LORA_ERR_INVALID, "id is NULL");
    NcclApi* api = nccl();
    if (!api) return fail(LORA_ERR_NCCL, "libnccl could not be loaded (set LORA_NCCL_LIB)");
    ncclUniqueId u;
    ncclResult_t r = api->GetUniqueId(&u);
    if (r != ncclSuccess) return nccl_fail(api, r, "ncclGetUniqueId");
    memcpy(id, &u, sizeof u);
    return LORA_OK;
}

lora_status lora_comm_init(int nranks, int rank, const uint8_t id[LORA_COMM_ID_BYTES], lora_comm** out) {
    if (!out || !id) return fail(LORA_ERR_INVALID, "lora_comm_init: NULL argument");
    if (nranks < 1 || rank < 0 || rank >= nranks)
        return fail(LORA_ERR_INVALID, "lora_comm_init: rank %d / nranks %d invalid", rank, nranks);
    NcclApi* api = nccl();
    if (!api) return fail(LORA_ERR_NCCL, "libnccl could not be loaded (set LORA_NCCL_LIB)");
    // the fused kernels must not be lazily loaded at a first launch that lands next to an
    // NCCL kernel waiting for a peer (the load would wait for that kernel)
    lora_status ps = preload_kernels();
    if (ps != LORA_OK) return ps;
    ncclUniqueId u;
    memcpy(&u, id, sizeof u);
    lora_comm* c = new lora_comm();
    c->nranks = nranks;
    c->rank = rank;
    ncclResult_t r = api->CommInitRank(&c->comm, nranks, u, rank);
    if (r != ncclSuccess) {
        delete c;
        return nccl_fail(api, r, "ncclCommInitRank");
    }
    // (no side stream -> the column group runs its collectives in stream order)
    if (cudaStreamCreateWithFlags(&c->side, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming) != cudaSuccess) {
        cudaGetLastError();
        if (c->ev_fork) cudaEventDestroy(c->ev_fork);
        if (c->side) cudaStreamDestroy(c->side);
        c->side = nullptr;
        c->ev_fork = c->ev_join = nullptr;
    }
    *out = c;
    return LORA_OK;
}

lora_status lora_comm_destroy(lora_comm* c) {
    if (!c) return LORA_OK;
    NcclApi* api = nccl();
    if (api) api->CommDestroy(c->comm);
    if (c->ev_join) cudaEventDestroy(c->ev_join);
    if (c->ev_fork) cudaEventDestroy(c->ev_fork);
    if (c->side) cudaStreamDestroy(c->side);
    delete c;
    return LORA_OK;
}

int lora_comm_size(const lora_comm* c) { return c ? c->nranks : 0; }
int lora_comm_rank(const lora_comm* c) { return c ? c->rank : -1; }

lora_status lora_allreduce(lora_comm* c, void* buf, size_t count, lora_dtype dt, void* stream) {
    if (!c) return fail(LORA_ERR_INVALID, "lora_allreduce: comm is NULL");
    if (dt != LORA_DT_F32 && dt != LORA_DT_BF16) return fail(LORA_ERR_INVALID, "lora_allreduce: bad dtype");
    if (count && !buf) return fail(LORA_ERR_INVALID, "lora_allreduce: buf is NULL");
    return allreduce_impl(c, buf, count, dt, static_cast<cudaStream_t>(stream));
}

size_t lora_tp_linear_bwd_workspace_bytes(const lora_dims* local) {
    const size_t base = bwd_workspace(local);
    if (!base) return 0;
    const size_t scratch = size_t(local->rank) * (local->d_in > local->d_out ? local->d_in : local->d_out) * 4;
    return base + align256(scratch);
}

// drop: LoRA dropout of the FULL input (null: none); row mode shifts its column
// offset to this rank's shard, the token slices shift its row offset and the
// kept-mask pointers
static lora_status tp_fwd(lora_comm* c, lora_tp_mode mode, const lora_dims* local, const void* x,
                          const void* w0, const void* a, const void* b, const void* bias, void* y,
                          float* h_out, void* workspace, size_t workspace_bytes, void* stream,
                          const lora_sm100::DropoutParams* drop0) {
    int launches = 0;
    if (!c) return fail(LORA_ERR_INVALID, "lora_tp_linear_fwd: comm is NULL");
    if (mode != LORA_TP_COLUMN && mode != LORA_TP_ROW) return fail(LORA_ERR_INVALID, "bad TP mode");
    lora_sm100::DropoutParams dshard;
    const lora_sm100::DropoutParams* drop = nullptr;
    if (drop0) {
        dshard = *drop0;
        if (mode == LORA_TP_ROW) dshard.col0 += static_cast<int64_t>(c->rank) * local->d_in;
        drop = &dshard;
    }
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    // row mode: the (unsharded) bias is added once, by rank 0
    const void* b0 = (mode == LORA_TP_ROW && c->rank != 0) ? nullptr : bias;
    const int chunks = mode == LORA_TP_ROW ? tp_fwd_chunks(local->tokens, c->nranks) : 1;
    if (chunks <= 1 || !c->side) {
        lora_status s = fwd_impl(local, x, w0, a, b, b0, y, h_out, workspace, workspace_bytes, st, &launches, nullptr,
                                 drop);
        set_launches(launches);
        if (s != LORA_OK || mode == LORA_TP_COLUMN) return s;
        return allreduce_impl(c, y, size_t(local->tokens) * local->d_out, LORA_DT_BF16, st);
    }
    // ROW mode, T-chunked (compute / comm overlap): the rows of y
    // depend only on their own tokens (Eq. 1 is row-wise in x), so the forward runs
    // as `chunks` launches over token slices of 256-row multiples; the all-reduce
    // of slice i runs on the communicator's side stream while the GEMM of slice
    // i + 1 runs on `stream`.  Every rank enqueues the same collectives in the
    // same order; the caller's stream joins the side stream at the end.
    lora_status s = fwd_impl(local, x, w0, a, b, b0, y, h_out, workspace, workspace_bytes, st, &launches, nullptr,
                             drop, true);   // validate the whole problem first
    if (s != LORA_OK) return s;
    const int64_t T = local->tokens, n = local->d_in, m = local->d_out;
    const int r = local->rank;
    const int64_t tc = ((T + chunks - 1) / chunks + 255) / 256 * 256;
    for (int64_t t0 = 0; t0 < T && s == LORA_OK; t0 += tc) {
        lora_dims dc = *local;
        dc.tokens = (T - t0) < tc ? (T - t0) : tc;
        lora_sm100::DropoutParams dslice;
        if (drop) {   // this slice's rows of the one mask (and of the kept buffers)
            dslice = *drop;
            dslice.row0 += t0;
            if (dslice.keep_bits) dslice.keep_bits += t0 * ((n + 31) / 32);
            if (dslice.masked_x) dslice.masked_x += t0 * n;
        }
        s = fwd_impl(&dc, static_cast<const uint8_t*>(x) + t0 * n * 2, w0, a, b, b0,
                     static_cast<uint8_t*>(y) + t0 * m * 2, h_out ? h_out + t0 * r : nullptr, workspace,
                     workspace_bytes, st, &launches, nullptr, drop ? &dslice : nullptr);
        if (s != LORA_OK) break;
        cudaError_t e = cudaEventRecord(c->ev_fork, st);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(c->side, c->ev_fork, 0);
        if (e != cudaSuccess) { s = cuda_fail(e, "row forward: fork the slice all-reduce"); break; }
        s = allreduce_impl(c, static_cast<uint8_t*>(y) + t0 * m * 2, size_t(dc.tokens) * m, LORA_DT_BF16, c->side);
    }
    cudaError_t e = cudaEventRecord(c->ev_join, c->side);   // (also on failure: no dangling fork)
    if (e == cudaSuccess) e = cudaStreamWaitEvent(st, c->ev_join, 0);
    set_launches(launches);
    if (s == LORA_OK && e != cudaSuccess) s = cuda_fail(e, "row forward: join the side stream");
    return s;
}

lora_status lora_tp_linear_fwd(lora_comm* c, lora_tp_mode mode, const lora_dims* local, const void* x,
                               const void* w0, const void* a, const void* b, const void* bias, void* y,
                               float* h_out, void* workspace, size_t workspace_bytes, void* stream) {
    return tp_fwd(c, mode, local, x, w0, a, b, bias, y, h_out, workspace, workspace_bytes, stream, nullptr);
}

lora_status lora_tp_linear_fwd_dropout(lora_comm* c, lora_tp_mode mode, const lora_dims* local,
                                       const lora_dropout* dropout, const void* x, const void* w0, const void* a,
                                       const void* b, const void* bias, void* y, float* h_out, void* workspace,
                                       size_t workspace_bytes, void* stream) {
    lora_sm100::DropoutParams dp;
    lora_status st = dropout_params(dropout, &dp);
    if (st != LORA_OK) return st;
    return tp_fwd(c, mode, local, x, w0, a, b, bias, y, h_out, workspace, workspace_bytes, stream,
                  dp.thr > 0 ? &dp : nullptr);
}

static lora_status tp_bwd(lora_comm* c, lora_tp_mode mode, const lora_dims* local, const void* x,
                          const void* w0, const void* a, const void* b, const float* h_saved,
                          const void* dy, void* dx, float* da, float* db, int accumulate,
                          int reduce_lora_grads, void* workspace, size_t workspace_bytes, void* stream,
                          const lora_sm100::DropoutParams* drop0) {
    int launches = 0;
    ProfGuard pg;
    if (!c) return fail(LORA_ERR_INVALID, "lora_tp_linear_bwd: comm is NULL");
    if (mode != LORA_TP_COLUMN && mode != LORA_TP_ROW) return fail(LORA_ERR_INVALID, "bad TP mode");
    lora_status s = check_dims(local, true);
    if (s != LORA_OK) return s;
    lora_sm100::DropoutParams dshard;
    const lora_sm100::DropoutParams* drop = nullptr;
    if (drop0) {   // row mode: this rank's columns of the one mask
        dshard = *drop0;
        if (mode == LORA_TP_ROW) dshard.col0 += static_cast<int64_t>(c->rank) * local->d_in;
        drop = &dshard;
    }
    const size_t need = drop0 ? lora_tp_linear_bwd_dropout_workspace_bytes(local)
                              : lora_tp_linear_bwd_workspace_bytes(local);
    if (!workspace || workspace_bytes < need)
        return fail(LORA_ERR_WORKSPACE, "lora_tp_linear_bwd: workspace %zu < required %zu", workspace_bytes, need);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const size_t base = drop0 ? bwd_workspace_dropout(local) : bwd_workspace(local);
    float* scratch = reinterpret_cast<float*>(static_cast<uint8_t*>(workspace) + base);
    // the gradient that is a partial sum on this rank
    float* partial_grad = (mode == LORA_TP_COLUMN) ? da : db;
    const size_t pcount = (mode == LORA_TP_COLUMN) ? size_t(local->rank) * local->d_in
                                                   : size_t(local->d_out) * local->rank;
    if (accumulate != 0 && accumulate != 1) return fail(LORA_ERR_INVALID, "accumulate must be 0 or 1");
    // accumulate + reduce: the partial gradient of THIS step is written to scratch
    // (overwrite), all-reduced, then added into the caller's buffer; the other
    // gradient is local and accumulates directly -- in the same single backward
    // (per-gradient accumulate bits), so nothing is computed twice.
    const bool via_scratch = reduce_lora_grads && accumulate && partial_grad;   // (also at N = 1: same path)
    float* da_out = (via_scratch && mode == LORA_TP_COLUMN) ? scratch : da;
    float* db_out = (via_scratch && mode == LORA_TP_ROW) ? scratch : db;
    int acc = accumulate ? lora_sm100::kAccA | lora_sm100::kAccB : 0;
    if (via_scratch) acc = (mode == LORA_TP_COLUMN) ? lora_sm100::kAccB : lora_sm100::kAccA;
    // bwd_impl sees a workspace that excludes the scratch tail
    s = bwd_impl(local, x, w0, a, b, h_saved, dy, dx, da_out, db_out, acc, workspace, base, st, &launches, nullptr, 3,
                 drop);
    if (s != LORA_OK) {
        set_launches(launches);
        return s;
    }
    if (mode == LORA_TP_COLUMN && dx) {
        s = allreduce_impl(c, dx, size_t(local->tokens) * local->d_in, LORA_DT_BF16, st);
        if (s != LORA_OK) return s;
    }
    if (reduce_lora_grads && partial_grad) {
        float* red = via_scratch ? scratch : partial_grad;
        s = allreduce_impl(c, red, pcount, LORA_DT_F32, st);
        if (s != LORA_OK) return s;
        if (via_scratch) {
            cudaError_t e = lora_sm100::launch_add_f32(partial_grad, scratch, static_cast<int64_t>(pcount), st);
            if (e != cudaSuccess) return cuda_fail(e, "grad accumulate launch");
            ++launches;
        }
    }
    set_launches(launches);
    return LORA_OK;
}

lora_status lora_tp_linear_bwd(lora_comm* c, lora_tp_mode mode, const lora_dims* local, const void* x,
                               const void* w0, const void* a, const void* b, const float* h_saved,
                               const void* dy, void* dx, float* da, float* db, int accumulate,
                               int reduce_lora_grads, void* workspace, size_t workspace_bytes, void* stream) {
    return tp_bwd(c, mode, local, x, w0, a, b, h_saved, dy, dx, da, db, accumulate, reduce_lora_grads, workspace,
                  workspace_bytes, stream, nullptr);
}

size_t lora_tp_linear_bwd_dropout_workspace_bytes(const lora_dims* local) {
    const size_t base = bwd_workspace_dropout(local);
    if (!base) return 0;
    const size_t scratch = size_t(local->rank) * (local->d_in > local->d_out ? local->d_in : local->d_out) * 4;
    return base + align256(scratch);
}

lora_status lora_tp_linear_bwd_dropout(lora_comm* c, lora_tp_mode mode, const lora_dims* local,
                                       const lora_dropout* dropout, const void* x, const void* w0, const void* a,
                                       const void* b, const float* h_saved, const void* dy, void* dx, float* da,
                                       float* db, int accumulate, int reduce_lora_grads, void* workspace,
                                       size_t workspace_bytes, void* stream) {
    lora_sm100::DropoutParams dp;
    lora_status st = dropout_params(dropout, &dp);
    if (st != LORA_OK) return st;
    return tp_bwd(c, mode, local, x, w0, a, b, h_saved, dy, dx, da, db, accumulate, reduce_lora_grads, workspace,
                  workspace_bytes, stream, dp.thr > 0 ? &dp : nullptr);
}

size_t lora_tp_linear_bwd_column_group_workspace_bytes(int count, const lora_dims* local) {
    return lora_linear_bwd_grouped_workspace_bytes(count, local);
}

static lora_status tp_bwd_column_group(lora_comm* c, int count, const lora_dims* local,
                                       const lora_bwd_problem* problems, void* dx_sum, int accumulate,
                                       int reduce_lora_grads, void* workspace, size_t workspace_bytes,
                                       void* stream, const lora_sm100::DropoutParams* drops) {
    ProfGuard pg;
    if (!c) return fail(LORA_ERR_INVALID, "lora_tp_linear_bwd_column_group: comm is NULL");
    if (count < 1 || count > LORA_MAX_GROUP || !local || !problems)
        return fail(LORA_ERR_INVALID, "lora_tp_linear_bwd_column_group: need 1..%d problems", LORA_MAX_GROUP);
    if (accumulate && reduce_lora_grads)
        return fail(LORA_ERR_UNSUPPORTED, "lora_tp_linear_bwd_column_group: accumulate with reduce_lora_grads "
                                          "(accumulate locally, then lora_allreduce the sums)");
    for (int g = 0; g < count; ++g) {
        if (local[g].tokens != local[0].tokens || local[g].d_in != local[0].d_in || problems[g].x != problems[0].x)
            return fail(LORA_ERR_INVALID, "lora_tp_linear_bwd_column_group: problem %d does not share problem 0's "
                                          "input x [T, d_in]", g);
        if (dx_sum && !problems[g].dx)
            return fail(LORA_ERR_INVALID, "lora_tp_linear_bwd_column_group: problem %d needs a dx buffer (the "
                                          "members' partials are summed into dx_sum)", g);
    }
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    // (1) the grouped local backward: one fused K2 launch, one K3 launch.  Right after
    // K2 is enqueued, (2) + (3) are forked onto the comm's side stream: the dX sum and
    // its all-reduce need only K2's outputs, so they overlap K3 (SURVEY.md 8(e):
    // "schedule the independent backward pieces concurrently"); joined before (4).
    struct Fork {
        lora_comm* c;
        int count;
        const lora_dims* local;
        const lora_bwd_problem* problems;
        void* dx_sum;
        cudaStream_t st;
        bool forked;
    } fk = {c, count, local, problems, dx_sum, st, false};
    auto dx_sum_and_reduce = [](void* ctx, int* launches) -> lora_status {
        Fork& f = *static_cast<Fork*>(ctx);
        const int64_t T = f.local[0].tokens, n = f.local[0].d_in;
        if (!f.dx_sum || T <= 0) return LORA_OK;
        cudaStream_t ss = f.st;
        if (f.c->side) {
            cudaError_t e = cudaEventRecord(f.c->ev_fork, f.st);
            if (e == cudaSuccess) e = cudaStreamWaitEvent(f.c->side, f.c->ev_fork, 0);
            if (e != cudaSuccess) return cuda_fail(e, "column group: fork onto the side stream");
            ss = f.c->side;
            f.forked = true;
        }
        // (2) dX w.r.t. the shared input: the members' partials summed (fp32, one RNE)
        lora_sm100::SumBf16Args A;
        A.n = f.count;
        A.count = T * n;
        A.dst = static_cast<__nv_bfloat16*>(f.dx_sum);
        for (int g = 0; g < f.count; ++g) A.src[g] = static_cast<const __nv_bfloat16*>(f.problems[g].dx);
        int dev = 0, sms = 148;
        if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaError_t e = lora_sm100::launch_sum_bf16(A, sms, ss);
        if (e != cudaSuccess) return cuda_fail(e, "dX sum launch");
        ++*launches;
        // (3) ONE all-reduce of the summed dX (q, k, v fused)
        lora_status s = allreduce_impl(f.c, f.dx_sum, size_t(T) * n, LORA_DT_BF16, ss);
        if (s != LORA_OK) return s;
        if (f.forked && (e = cudaEventRecord(f.c->ev_join, ss)) != cudaSuccess)
            return cuda_fail(e, "column group: side stream join event");
        return LORA_OK;
    };
    lora_status s = bwd_grouped_impl(count, local, problems, accumulate, workspace, workspace_bytes, stream,
                                     dx_sum_and_reduce, &fk, nullptr, nullptr, drops);
    int launches = get_launches();
    if (fk.forked) {   // join (also on failure: never leave the side stream dangling in a capture)
        cudaError_t e = cudaStreamWaitEvent(st, c->ev_join, 0);
        if (s == LORA_OK && e != cudaSuccess) s = cuda_fail(e, "column group: join the side stream");
    }
    if (s != LORA_OK) return s;
    // (4) the partial dA of every member, batched into one NCCL group
    if (reduce_lora_grads) {
        NcclApi* api = nccl();
        if (!api) return fail(LORA_ERR_NCCL, "libnccl could not be loaded (set LORA_NCCL_LIB)");
        if (api->GroupStart) api->GroupStart();
        for (int g = 0; g < count && s == LORA_OK; ++g)
            if (problems[g].da) s = allreduce_impl(c, problems[g].da, size_t(local[g].rank) * local[g].d_in,
                                                   LORA_DT_F32, st);
        if (api->GroupEnd) {
            ncclResult_t r = api->GroupEnd();
            if (s == LORA_OK && r != ncclSuccess) s = nccl_fail(api, r, "ncclGroupEnd");
        }
        if (s != LORA_OK) return s;
    }
    set_launches(launches);
    return LORA_OK;
}

lora_status lora_tp_linear_bwd_column_group(lora_comm* c, int count, const lora_dims* local,
                                            const lora_bwd_problem* problems, void* dx_sum, int accumulate,
                                            int reduce_lora_grads, void* workspace, size_t workspace_bytes,
                                            void* stream) {
    return tp_bwd_column_group(c, count, local, problems, dx_sum, accumulate, reduce_lora_grads, workspace,
                               workspace_bytes, stream, nullptr);
}

size_t lora_tp_linear_bwd_column_group_dropout_workspace_bytes(int count, const lora_dims* local) {
    return lora_linear_bwd_grouped_dropout_workspace_bytes(count, local);
}

lora_status lora_tp_linear_bwd_column_group_dropout(lora_comm* c, int count, const lora_dims* local,
                                                    const lora_dropout* dropouts, const lora_bwd_problem* problems,
                                                    void* dx_sum, int accumulate, int reduce_lora_grads,
                                                    void* workspace, size_t workspace_bytes, void* stream) {
    if (count < 1 || count > LORA_MAX_GROUP || !dropouts)
        return fail(LORA_ERR_INVALID, "lora_tp_linear_bwd_column_group_dropout: need 1..%d problems and their "
                                      "dropouts", LORA_MAX_GROUP);
    lora_sm100::DropoutParams dp[LORA_MAX_GROUP];
    int dropping = 0;
    for (int g = 0; g < count; ++g) {
        lora_status st = dropout_params(&dropouts[g], &dp[g]);
        if (st != LORA_OK) return st;
        dropping += dp[g].thr > 0 ? 1 : 0;
    }
    if (dropping != 0 && dropping != count)
        return fail(LORA_ERR_INVALID, "lora_tp_linear_bwd_column_group_dropout: p must be > 0 for all problems "
                                      "or for none");
    // (COLUMN mode: x is replicated, every rank draws the full mask -- no offset)
    return tp_bwd_column_group(c, count, local, problems, dx_sum, accumulate, reduce_lora_grads, workspace,
                               workspace_bytes, stream, dropping ? dp : nullptr);
}

}  // extern "C"
