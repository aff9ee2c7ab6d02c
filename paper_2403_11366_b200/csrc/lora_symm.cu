// lora_symm.cu -- comm-fused epilogues over peer memory.
//
// PAPER.md:199 attributes JORA's multi-GPU slowdown to "cross-GPU
// communication overhead".  The two activation all-reduces of the tensor-
// parallel LoRA linear (row-parallel y, column-parallel dX; PAPER.md:122,
// DESIGN.md R10-R12) are fused with the kernels that produce them:
//
//   producer  the fused GEMM (K1 / K2) of every rank writes its partial output
//             into its SYMMETRIC buffer and, as soon as the 128 rows of a tile
//             half are stored, raises that unit's flag (release, system scope);
//   reducer   a small kernel launched on a side stream just before the GEMM
//             (co-resident with it: no shared memory, few registers) owns the
//             units u with u % N == rank; for each, in production order, it
//             waits for the N (x members) flags, loads the partial tiles from
//             every rank's buffer (peer loads over NVLink), sums them in
//             (rank, member) order in fp32, rounds ONCE to bf16 and stores the
//             result into every rank's output region (peer stores) -- so the
//             reduction of tile i overlaps the GEMM of tiles i+1.. and NVLink
//             carries (N-1)/N of the bytes in each direction (push, not pull).
//             It resets the flags it consumed, then counts itself in on every
//             rank's launch counter; the kernel ends when all N x CTAs have, so
//             the caller's stream (joined to the side stream) sees the whole
//             reduced output.
// Every value is summed exactly once by one rank, so all ranks hold bitwise
// identical results and repeat runs are bitwise equal (R13), with
// fewer roundings than a bf16 ring all-reduce.
//
// Peers are mapped with CUDA IPC (one process per GPU) or, for the single-GPU
// test of the protocol, are the buffers of N "virtual ranks" on one device in
// one process (lora_symm_connect_local).  NVLS multicast (multimem.ld_reduce)
// would replace the N peer loads by one; the round's one-GPU boxes cannot create
// a multicast object (profiles/r02/nvls_probe.txt), so it is not built.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <cstring>

#include "lora_internal.h"
#include "lora_kernels.h"
#include "sm100_ptx.cuh"

namespace lora_sm100 {

__device__ __forceinline__ uint4 ld_cg_u4(const void* p) {
    uint4 v;
    asm volatile("ld.global.cg.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p) : "memory");
    return v;
}

// KV 16-byte vectors per thread per round; MINB = CTAs per SM the launch bounds
// assume, which caps the registers (65536 / (128 MINB)): KV 4 <= 128, KV 2 <= 80
template <int KV, int MINB>
__global__ void __launch_bounds__(128, MINB) symm_reduce_kernel(const __grid_constant__ SymmReduceArgs A) {
    const int N = A.nranks, G = A.nsrc;
    const int nwait = N * G;
    for (int64_t k = blockIdx.x;; k += gridDim.x) {
        const int64_t u = A.rank + static_cast<int64_t>(N) * k;
        if (u >= A.units) break;
        const int nb = static_cast<int>(u / A.nrow128);
        const int64_t r0 = (u - static_cast<int64_t>(nb) * A.nrow128) * 128;
        const int64_t c0 = A.col_start[nb];
        const int64_t c1 = A.col_start[nb + 1] < A.ncols ? A.col_start[nb + 1] : A.ncols;
        const int rows = static_cast<int>(A.T - r0 < 128 ? A.T - r0 : 128);
        const int nv = static_cast<int>((c1 - c0) / 8);
        if (static_cast<int>(threadIdx.x) < nwait) {
            const int r = threadIdx.x / G, g = threadIdx.x - (threadIdx.x / G) * G;
            const uint32_t* f = A.flags[r] + static_cast<int64_t>(g) * A.units + u;
            if (ld_acquire_sys_u32(f) == 0u) {
                const uint64_t t0 = globaltimer_ns();
                while (ld_acquire_sys_u32(f) == 0u) {
                    __nanosleep(256);
                    if (globaltimer_ns() - t0 > kWaitTimeoutNs) {
                        printf("lora symm reduce: unit %lld of rank %d member %d never published\n",
                               static_cast<long long>(u), r, g);
                        __trap();
                    }
                }
            }
        }
        __syncthreads();
        // kV vectors (16 bytes) per thread per round, their loads for kSrc sources at a
        // time all in flight before any is consumed: the reduction is latency-bound (peer
        // loads), and the CTA must stay small enough to sit next to the GEMM's
        constexpr int kV = KV, kSrc = 2;
        const int total = rows * nv;
        for (int i0 = threadIdx.x; i0 < total; i0 += kV * blockDim.x) {
            int64_t off[kV];
            bool ok[kV];
#pragma unroll
            for (int v = 0; v < kV; ++v) {
                const int i = i0 + v * blockDim.x;
                ok[v] = i < total;
                const int row = ok[v] ? i / nv : 0, cv = ok[v] ? i - (i / nv) * nv : 0;
                off[v] = (r0 + row) * A.ld + c0 + 8 * cv;
            }
            float acc[kV][8];
#pragma unroll
            for (int v = 0; v < kV; ++v)
#pragma unroll
                for (int e = 0; e < 8; ++e) acc[v][e] = 0.0f;
            for (int s0 = 0; s0 < nwait; s0 += kSrc) {   // (rank, member) order
                uint4 q[kSrc][kV];
#pragma unroll
                for (int j = 0; j < kSrc; ++j) {
                    const int sj = s0 + j;
                    const __nv_bfloat16* src = sj < nwait ? A.part[sj / G][sj - (sj / G) * G] : nullptr;
#pragma unroll
                    for (int v = 0; v < kV; ++v)
                        q[j][v] = (src != nullptr && ok[v]) ? ld_cg_u4(src + off[v]) : make_uint4(0, 0, 0, 0);
                }
#pragma unroll
                for (int j = 0; j < kSrc; ++j) {
                    if (s0 + j >= nwait) break;
#pragma unroll
                    for (int v = 0; v < kV; ++v) {
                        const uint32_t w[4] = {q[j][v].x, q[j][v].y, q[j][v].z, q[j][v].w};
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            acc[v][2 * e] += __uint_as_float(w[e] << 16);
                            acc[v][2 * e + 1] += __uint_as_float(w[e] & 0xFFFF0000u);
                        }
                    }
                }
            }
#pragma unroll
            for (int v = 0; v < kV; ++v) {
                if (!ok[v]) continue;
                const uint4 o = make_uint4(pack_bf16x2(acc[v][0], acc[v][1]), pack_bf16x2(acc[v][2], acc[v][3]),
                                           pack_bf16x2(acc[v][4], acc[v][5]), pack_bf16x2(acc[v][6], acc[v][7]));
                for (int r = 0; r < N; ++r) *reinterpret_cast<uint4*>(A.out[r] + off[v]) = o;
            }
        }
        __syncthreads();   // every read of this unit's partials is done: its flags may be reused
        if (static_cast<int>(threadIdx.x) < nwait) {
            const int r = threadIdx.x / G, g = threadIdx.x - (threadIdx.x / G) * G;
            st_relaxed_sys_u32(A.flags[r] + static_cast<int64_t>(g) * A.units + u, 0u);
        }
    }
    // this CTA's output stores (and flag resets) before its arrival on every rank
    __threadfence_system();
    __syncthreads();
    if (static_cast<int>(threadIdx.x) < N) red_release_sys_add_u32(A.done[threadIdx.x], 1u);
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        // the launch ends only when every CTA of every rank has stored its units here
        const uint32_t want = static_cast<uint32_t>(N) * gridDim.x;
        const uint64_t t0 = globaltimer_ns();
        while (ld_acquire_sys_u32(A.done[A.rank]) != want) {
            __nanosleep(256);
            if (globaltimer_ns() - t0 > kWaitTimeoutNs) {
                printf("lora symm reduce: rank %d saw %u of %u reducer CTAs\n", A.rank,
                       ld_acquire_sys_u32(A.done[A.rank]), want);
                __trap();
            }
        }
        // (no peer counts in again before this rank's next fused GEMM has run, which is
        // stream-ordered after this kernel)
        st_relaxed_sys_u32(A.done[A.rank], 0u);
    }
}

// Register footprint per SM sub-partition (16 Ki registers each) when one CTA of a
// kernel with `warps` warps and `regs` registers per thread is resident: warp w
// sits on sub-partition w % 4, registers are allocated per warp in units of 8 per
// thread.  Returns the largest per-sub-partition use.
static int smsp_regs(int warps, int regs) {
    const int per_warp = (regs + 7) / 8 * 8 * 32;
    return ((warps + 3) / 4) * per_warp;
}

cudaError_t symm_reducer_plan(int gemm_regs, int gemm_warps, int* variant) {
    cudaFuncAttributes fa;
    const int budget = 16384 - smsp_regs(gemm_warps, gemm_regs);
    const void* ks[2] = {(const void*)symm_reduce_kernel<4, 4>, (const void*)symm_reduce_kernel<2, 6>};
    for (int v = 0; v < 2; ++v) {
        cudaError_t e = cudaFuncGetAttributes(&fa, ks[v]);
        if (e != cudaSuccess) return e;
        if (smsp_regs(4, fa.numRegs) <= budget) {   // 4 warps: one per sub-partition
            *variant = v;
            return cudaSuccess;
        }
    }
    *variant = -1;   // no reducer fits next to this GEMM: run it after the GEMM
    return cudaSuccess;
}

cudaError_t launch_symm_reduce(const SymmReduceArgs& A, int ctas, int variant, cudaStream_t stream) {
    if (A.nranks < 1 || A.nranks > kSymmMaxRanks || A.nsrc < 1 || A.nsrc > kMaxGroup || ctas < 1)
        return cudaErrorInvalidValue;
    // The reducer co-resides with the fused GEMM (~200 KiB of shared memory per SM;
    // tools/probe/coresid.cu): ask for a shared-memory-heavy carveout so an SM that
    // hosts a reducer CTA stays configured for a GEMM CTA next to it.
    static bool attr_set = false;
    if (!attr_set) {
        cudaError_t e = cudaFuncSetAttribute(symm_reduce_kernel<4, 4>, cudaFuncAttributePreferredSharedMemoryCarveout,
                                             cudaSharedmemCarveoutMaxShared);
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(symm_reduce_kernel<2, 6>, cudaFuncAttributePreferredSharedMemoryCarveout,
                                     cudaSharedmemCarveoutMaxShared);
        if (e != cudaSuccess) return e;
        attr_set = true;
    }
    if (variant == 1) symm_reduce_kernel<2, 6><<<ctas, 128, 0, stream>>>(A);
    else symm_reduce_kernel<4, 4><<<ctas, 128, 0, stream>>>(A);
    return cudaGetLastError();
}

}  // namespace lora_sm100

// =============================================================================
// host side: the symmetric buffer and the fused tensor-parallel entry points
// =============================================================================
using namespace lora_host;
using namespace lora_sm100;

namespace {
constexpr size_t kCtlBytes = 256 * 1024;      // launch counter + unit flags, ahead of the data region
constexpr size_t kFlagsOff = 1024;
constexpr size_t kMaxFlags = (kCtlBytes - kFlagsOff) / 4;
}  // namespace

struct lora_symm {
    int dev = -1;
    size_t data_bytes = 0;
    uint8_t* base = nullptr;                    // this rank: [control | data], owned
    int nranks = 0, rank = 0;                   // 0 until connected
    uint8_t* peer[kSymmMaxRanks] = {};          // every rank's base (peer[rank] == base)
    bool opened[kSymmMaxRanks] = {};            // IPC mappings to close
    bool local = false;                         // virtual ranks of one process on one GPU
    int last_mode = 0;                          // last reducer placement: 1 co-resident, 2 after the GEMM, 3 split SMs
    cudaStream_t side = nullptr;
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
};

namespace lora_host {
// Load every kernel that can be launched while a kernel spinning on another
// one's output is resident -- the comm-fused reducer, or NCCL collectives waiting
// for peers (lora_kernels.h, preload_*): once per device.
lora_status preload_kernels() {
    static bool done[64] = {};
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
    if (dev < 0 || dev >= 64 || done[dev]) return LORA_OK;
    cudaFuncAttributes fa;
    if ((e = preload_gemm_kernels()) != cudaSuccess || (e = preload_grad_kernels()) != cudaSuccess ||
        (e = preload_grad_mma_kernels()) != cudaSuccess ||
        (e = cudaFuncGetAttributes(&fa, (const void*)symm_reduce_kernel<4, 4>)) != cudaSuccess ||
        (e = cudaFuncGetAttributes(&fa, (const void*)symm_reduce_kernel<2, 6>)) != cudaSuccess)
        return cuda_fail(e, "kernel preload");
    done[dev] = true;
    return LORA_OK;
}
}  // namespace lora_host

static lora_status symm_check(const lora_symm* s, const char* fn) {
    if (!s) return fail(LORA_ERR_INVALID, "%s: symm is NULL", fn);
    if (s->nranks < 1) return fail(LORA_ERR_INVALID, "%s: symm is not connected (lora_symm_connect*)", fn);
    int dev = -1;
    cudaGetDevice(&dev);
    if (dev != s->dev) return fail(LORA_ERR_INVALID, "%s: current device %d is not the symm's device %d", fn, dev,
                                   s->dev);
    return LORA_OK;
}

static lora_status region_check(const lora_symm* s, size_t off, size_t bytes, const char* what, const char* fn) {
    if (off % 16 != 0) return fail(LORA_ERR_ALIGN, "%s: %s offset %zu is not 16-byte aligned", fn, what, off);
    if (off > s->data_bytes || bytes > s->data_bytes - off)
        return fail(LORA_ERR_SHAPE, "%s: %s [%zu, %zu) exceeds the symmetric data region (%zu bytes)", fn, what, off,
                    off + bytes, s->data_bytes);
    return LORA_OK;
}

// reducer arguments for G members whose partials are at part_off + g * part_stride
static lora_status make_reduce_args(const lora_symm* s, int mode, int rp, int64_t T, int64_t ncols, int G,
                                    size_t part_off, size_t part_stride, size_t out_off, SymmReduceArgs* A,
                                    const char* fn) {
    memset(A, 0, sizeof(*A));
    A->nranks = s->nranks;
    A->rank = s->rank;
    A->nsrc = G;
    A->T = T;
    A->ncols = ncols;
    A->ld = ncols;
    A->nrow128 = static_cast<int>((T + 127) / 128);
    A->ncol_tiles = fused_gemm_col_tiles(mode, rp, ncols, A->col_start, kSymmMaxColTiles);
    if (A->ncol_tiles < 0) return fail(LORA_ERR_UNSUPPORTED, "%s: %lld output columns need too many tiles", fn,
                                       static_cast<long long>(ncols));
    A->units = A->ncol_tiles * A->nrow128;
    if (static_cast<size_t>(A->units) * G > kMaxFlags)
        return fail(LORA_ERR_UNSUPPORTED, "%s: %d units x %d members exceed the %zu unit flags", fn, A->units, G,
                    kMaxFlags);
    for (int r = 0; r < s->nranks; ++r) {
        uint8_t* b = s->peer[r];
        for (int g = 0; g < G; ++g)
            A->part[r][g] = reinterpret_cast<const __nv_bfloat16*>(b + kCtlBytes + part_off + g * part_stride);
        A->flags[r] = reinterpret_cast<uint32_t*>(b + kFlagsOff);
        A->out[r] = reinterpret_cast<__nv_bfloat16*>(b + kCtlBytes + out_off);
        A->done[r] = reinterpret_cast<uint32_t*>(b);
    }
    return LORA_OK;
}

// Placement (the GEMM's persistent CTAs own fixed tiles the reducer waits for, so
// no reducer CTA may ever keep a GEMM CTA from being placed -- that deadlocks):
//  * one rank per GPU: if a reducer variant fits next to one GEMM CTA on EVERY SM
//    (per sub-partition register budget, symm_reducer_plan: the fused dX kernel
//    has 6 warps of up to 254 registers, sub-partitions 0 / 1 carry two of them),
//    the reducer runs co-resident, one CTA per SM at most, overlapping the GEMM;
//    otherwise it runs after the GEMM (no overlap, no risk);
//  * virtual ranks on one GPU (connect_local): the ranks' GEMMs run one after the
//    other and every rank's reducer waits for all of them, so the SMs are split
//    instead: the GEMMs are capped at (SMs - 16) / 2 CTA pairs and the N reducers
//    share 8 CTAs (at most 8 SMs / TPCs, while 8 TPCs are left free).
constexpr int kLocalReducerCtas = 8;
constexpr int kLocalReservedSms = 2 * kLocalReducerCtas;

static int reducer_ctas(const SymmReduceArgs& A, int num_sms, bool local, bool coresident) {
    const int owned = (A.units + A.nranks - 1) / A.nranks;
    int cap = local ? (kLocalReducerCtas / A.nranks > 0 ? kLocalReducerCtas / A.nranks : 1)
                    : (coresident ? num_sms : 2 * num_sms);
    return owned < cap ? (owned > 0 ? owned : 1) : cap;
}

// fork the side stream off `st`, launch the reducer there
// The side stream must not wait for the GEMM (the reducer runs next to it): the
// fork event is recorded on `st` BEFORE the GEMM (record_fork), the reducer is
// launched after the GEMM has been enqueued.
static lora_status record_fork(lora_symm* s, cudaStream_t st) {
    cudaError_t e = cudaEventRecord(s->ev_fork, st);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(s->side, s->ev_fork, 0);
    return e == cudaSuccess ? LORA_OK : cuda_fail(e, "symm: fork the reducer stream");
}

// Called right after the GEMM (registers per thread `gemm_regs`) was enqueued on `st`
// (the fork event was recorded before it).
static lora_status fork_reducer(lora_symm* s, const SymmReduceArgs& A, cudaStream_t st, int* launches,
                                int gemm_regs) {
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, s->dev);
    int variant = 0;
    cudaError_t e = cudaSuccess;
    if (!s->local) {
        if ((e = symm_reducer_plan(gemm_regs, 6, &variant)) != cudaSuccess) return cuda_fail(e, "symm reducer plan");
        if (variant < 0) {   // nothing fits next to this GEMM: reduce after it
            if ((e = cudaEventRecord(s->ev_fork, st)) == cudaSuccess) e = cudaStreamWaitEvent(s->side, s->ev_fork, 0);
            if (e != cudaSuccess) return cuda_fail(e, "symm: order the reducer after the GEMM");
            variant = 0;
            s->last_mode = 2;
        } else {
            s->last_mode = 1;
        }
    } else {
        s->last_mode = 3;
    }
    if ((e = launch_symm_reduce(A, reducer_ctas(A, sms, s->local, s->last_mode == 1), variant, s->side)) !=
        cudaSuccess)
        return cuda_fail(e, "symm reduce launch");
    ++*launches;
    return LORA_OK;
}

static int max_gemm_regs(const GemmCollector& col, int mode) {
    int r = 0;
    for (int g = 0; g < col.count; ++g) {
        const int v = fused_gemm_regs(mode, col.rp[g], col.cg[g]);
        r = v > r ? v : r;
    }
    return r;
}

static int local_gemm_sms(const lora_symm* s) {
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, s->dev);
    return sms - kLocalReservedSms;
}

static lora_status join_reducer(lora_symm* s, cudaStream_t st) {
    cudaError_t e = cudaEventRecord(s->ev_join, s->side);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(st, s->ev_join, 0);
    return e == cudaSuccess ? LORA_OK : cuda_fail(e, "symm: join the reducer stream");
}

extern "C" {

lora_status lora_symm_create(size_t data_bytes, lora_symm** out) {
    if (!out) return fail(LORA_ERR_INVALID, "lora_symm_create: out is NULL");
    *out = nullptr;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return cuda_fail(e, "lora_symm_create: cudaGetDevice");
    // every kernel a fused call launches next to a spinning reducer is loaded now
    // (lora_kernels.h: lazy loading would stall those launches behind the reducer)
    lora_status ps = preload_kernels();
    if (ps != LORA_OK) return ps;
    lora_symm* s = new lora_symm();
    s->dev = dev;
    s->data_bytes = (data_bytes + 255) / 256 * 256;
    void* p = nullptr;
    if ((e = cudaMalloc(&p, kCtlBytes + s->data_bytes)) != cudaSuccess) {
        delete s;
        return cuda_fail(e, "lora_symm_create: cudaMalloc");
    }
    s->base = static_cast<uint8_t*>(p);
    if ((e = cudaMemset(p, 0, kCtlBytes + s->data_bytes)) != cudaSuccess ||
        (e = cudaDeviceSynchronize()) != cudaSuccess ||
        (e = cudaStreamCreateWithFlags(&s->side, cudaStreamNonBlocking)) != cudaSuccess ||
        (e = cudaEventCreateWithFlags(&s->ev_fork, cudaEventDisableTiming)) != cudaSuccess ||
        (e = cudaEventCreateWithFlags(&s->ev_join, cudaEventDisableTiming)) != cudaSuccess) {
        lora_symm_destroy(s);
        return cuda_fail(e, "lora_symm_create");
    }
    *out = s;
    return LORA_OK;
}

lora_status lora_symm_ipc_handle(const lora_symm* s, uint8_t handle[LORA_SYMM_HANDLE_BYTES]) {
    if (!s || !handle) return fail(LORA_ERR_INVALID, "lora_symm_ipc_handle: NULL argument");
    static_assert(sizeof(cudaIpcMemHandle_t) == LORA_SYMM_HANDLE_BYTES, "IPC handle size");
    cudaIpcMemHandle_t h;
    cudaError_t e = cudaIpcGetMemHandle(&h, s->base);
    if (e != cudaSuccess) return cuda_fail(e, "cudaIpcGetMemHandle");
    memcpy(handle, &h, sizeof h);
    return LORA_OK;
}

lora_status lora_symm_connect(lora_symm* s, int nranks, int rank, const uint8_t* handles) {
    if (!s || !handles) return fail(LORA_ERR_INVALID, "lora_symm_connect: NULL argument");
    if (nranks < 1 || nranks > kSymmMaxRanks || rank < 0 || rank >= nranks)
        return fail(LORA_ERR_INVALID, "lora_symm_connect: rank %d / nranks %d (1..%d ranks)", rank, nranks,
                    kSymmMaxRanks);
    if (s->nranks) return fail(LORA_ERR_INVALID, "lora_symm_connect: already connected");
    for (int r = 0; r < nranks; ++r) {
        if (r == rank) {
            s->peer[r] = s->base;
            continue;
        }
        cudaIpcMemHandle_t h;
        memcpy(&h, handles + size_t(r) * LORA_SYMM_HANDLE_BYTES, sizeof h);
        void* p = nullptr;
        cudaError_t e = cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess);
        if (e != cudaSuccess) {
            for (int q = 0; q < r; ++q)
                if (s->opened[q]) cudaIpcCloseMemHandle(s->peer[q]);
            memset(s->peer, 0, sizeof s->peer);
            memset(s->opened, 0, sizeof s->opened);
            return cuda_fail(e, "cudaIpcOpenMemHandle (peer symmetric buffer)");
        }
        s->peer[r] = static_cast<uint8_t*>(p);
        s->opened[r] = true;
    }
    s->nranks = nranks;
    s->rank = rank;
    return LORA_OK;
}

lora_status lora_symm_connect_local(int nranks, lora_symm* const* group) {
    if (!group || nranks < 1 || nranks > kSymmMaxRanks)
        return fail(LORA_ERR_INVALID, "lora_symm_connect_local: need 1..%d buffers", kSymmMaxRanks);
    for (int r = 0; r < nranks; ++r) {
        if (!group[r] || group[r]->nranks) return fail(LORA_ERR_INVALID, "lora_symm_connect_local: buffer %d is NULL "
                                                                        "or already connected", r);
        if (group[r]->dev != group[0]->dev || group[r]->data_bytes != group[0]->data_bytes)
            return fail(LORA_ERR_INVALID, "lora_symm_connect_local: buffers differ in device or size");
    }
    for (int r = 0; r < nranks; ++r) {
        for (int q = 0; q < nranks; ++q) group[r]->peer[q] = group[q]->base;
        group[r]->nranks = nranks;
        group[r]->rank = r;
        group[r]->local = true;
    }
    return LORA_OK;
}

void* lora_symm_ptr(const lora_symm* s) { return s ? s->base + kCtlBytes : nullptr; }
int lora_symm_last_placement(const lora_symm* s) { return s ? s->last_mode : 0; }
size_t lora_symm_bytes(const lora_symm* s) { return s ? s->data_bytes : 0; }

lora_status lora_symm_destroy(lora_symm* s) {
    if (!s) return LORA_OK;
    int cur = -1;
    cudaGetDevice(&cur);
    if (s->dev >= 0) cudaSetDevice(s->dev);
    if (s->side) cudaStreamSynchronize(s->side);
    for (int r = 0; r < kSymmMaxRanks; ++r)
        if (s->opened[r]) cudaIpcCloseMemHandle(s->peer[r]);
    if (s->ev_join) cudaEventDestroy(s->ev_join);
    if (s->ev_fork) cudaEventDestroy(s->ev_fork);
    if (s->side) cudaStreamDestroy(s->side);
    if (s->base) cudaFree(s->base);
    if (cur >= 0) cudaSetDevice(cur);
    delete s;
    return LORA_OK;
}

lora_status lora_tp_linear_fwd_fused(lora_symm* s, const lora_dims* local, const void* x, const void* w0,
                                     const void* a, const void* b, const void* bias, size_t part_offset,
                                     size_t y_offset, float* h_out, void* workspace, size_t workspace_bytes,
                                     void* stream) {
    static const char* fn = "lora_tp_linear_fwd_fused";
    int launches = 0;
    lora_status st = symm_check(s, fn);
    if (st != LORA_OK) return st;
    if ((st = check_dims(local, true)) != LORA_OK) return st;
    const int64_t T = local->tokens, m = local->d_out;
    const size_t yb = size_t(T) * m * 2;
    if ((st = region_check(s, part_offset, yb, "partial", fn)) != LORA_OK) return st;
    if ((st = region_check(s, y_offset, yb, "y", fn)) != LORA_OK) return st;
    if (part_offset < y_offset + yb && y_offset < part_offset + yb)
        return fail(LORA_ERR_INVALID, "%s: the partial and y regions overlap", fn);
    cudaStream_t cs = static_cast<cudaStream_t>(stream);
    void* part = s->base + kCtlBytes + part_offset;
    const void* b0 = s->rank == 0 ? bias : nullptr;   // the unsharded bias is added once
    GemmCollector col;
    if ((st = fwd_impl(local, x, w0, a, b, b0, part, h_out, workspace, workspace_bytes, cs, &launches, nullptr,
                       nullptr, true)) != LORA_OK)
        return st;
    if (T == 0) return LORA_OK;
    SymmReduceArgs A;
    const int rp = r_pad_of(local->rank);
    if ((st = make_reduce_args(s, kModeFwd, rp, T, m, 1, part_offset, 0, y_offset, &A, fn)) != LORA_OK) return st;
    if ((st = fwd_impl(local, x, w0, a, b, b0, part, h_out, workspace, workspace_bytes, cs, &launches, &col)) !=
        LORA_OK) {
        set_launches(launches);
        return st;
    }
    if ((st = record_fork(s, cs)) != LORA_OK) return st;
    for (int g = 0; g < col.count; ++g) {
        col.p[g].unit_flags = reinterpret_cast<uint32_t*>(s->base + kFlagsOff);
        col.p[g].sk_partial = nullptr;
    }
    if (s->local) col.max_sms = local_gemm_sms(s);
    // the GEMM is enqueued before the reducer (see reducer_ctas for the placement rules)
    if ((st = launch_collected(kModeFwd, col, cs, &launches)) != LORA_OK) {
        set_launches(launches);
        return st;
    }
    if ((st = fork_reducer(s, A, cs, &launches, max_gemm_regs(col, kModeFwd))) != LORA_OK) return st;
    st = join_reducer(s, cs);
    set_launches(launches);
    return st;
}

lora_status lora_tp_linear_bwd_column_group_fused(lora_symm* s, lora_comm* comm, int count, const lora_dims* local,
                                                  const lora_bwd_problem* problems, size_t part_offset,
                                                  size_t dx_offset, int reduce_lora_grads, void* workspace,
                                                  size_t workspace_bytes, void* stream) {
    static const char* fn = "lora_tp_linear_bwd_column_group_fused";
    lora_status st = symm_check(s, fn);
    if (st != LORA_OK) return st;
    if (count < 1 || count > LORA_MAX_GROUP || !local || !problems)
        return fail(LORA_ERR_INVALID, "%s: need 1..%d problems", fn, LORA_MAX_GROUP);
    if (reduce_lora_grads && !comm) return fail(LORA_ERR_INVALID, "%s: reduce_lora_grads needs a lora_comm", fn);
    for (int g = 0; g < count; ++g) {
        if ((st = check_dims(&local[g], true)) != LORA_OK) return st;
        if (local[g].tokens != local[0].tokens || local[g].d_in != local[0].d_in || problems[g].x != problems[0].x)
            return fail(LORA_ERR_INVALID, "%s: problem %d does not share problem 0's input x [T, d_in]", fn, g);
        if (problems[g].dx)
            return fail(LORA_ERR_INVALID, "%s: problems[%d].dx must be NULL (the members' dX partials live in the "
                                          "symmetric buffer)", fn, g);
    }
    const int64_t T = local[0].tokens, n = local[0].d_in;
    const size_t xb = size_t(T) * n * 2;
    if ((st = region_check(s, part_offset, xb * count, "partials", fn)) != LORA_OK) return st;
    if ((st = region_check(s, dx_offset, xb, "dx", fn)) != LORA_OK) return st;
    if (part_offset < dx_offset + xb && dx_offset < part_offset + xb * count)
        return fail(LORA_ERR_INVALID, "%s: the partial and dx regions overlap", fn);
    cudaStream_t cs = static_cast<cudaStream_t>(stream);
    lora_bwd_problem probs[LORA_MAX_GROUP];
    for (int g = 0; g < count; ++g) {
        probs[g] = problems[g];
        probs[g].dx = s->base + kCtlBytes + part_offset + g * xb;   // member g's dX partial
    }
    SymmReduceArgs A;
    if ((st = make_reduce_args(s, kModeDx, 16, T, n, count, part_offset, xb, dx_offset, &A, fn)) != LORA_OK)
        return st;
    struct Ctx {
        lora_symm* s;
        const SymmReduceArgs* A;
        cudaStream_t cs;
        bool forked;
        int gemm_regs;
    } ctx = {s, &A, cs, false, 255};
    // right before the grouped dX kernel: every member publishes its units, and the
    // side stream forks off here; right after K2 is enqueued the reducer is launched
    // (GEMM first: see lora_tp_linear_fwd_fused) and sums the units over members and
    // ranks while K2 runs; K3 follows on `cs`
    auto before_k2 = [](void* c, GemmCollector* col, int* launches) -> lora_status {
        (void)launches;
        Ctx& k = *static_cast<Ctx*>(c);
        for (int g = 0; g < col->count; ++g) {
            col->p[g].unit_flags = reinterpret_cast<uint32_t*>(k.s->base + kFlagsOff) + int64_t(g) * k.A->units;
            col->p[g].sk_partial = nullptr;
        }
        // a cooperative dX launch would wait for the resident reducer, which waits for it
        col->no_coop = true;
        if (k.s->local) col->max_sms = local_gemm_sms(k.s);
        k.gemm_regs = max_gemm_regs(*col, kModeDx);
        lora_status r = record_fork(k.s, k.cs);
        k.forked = r == LORA_OK;
        return r;
    };
    auto after_k2 = [](void* c, int* launches) -> lora_status {
        Ctx& k = *static_cast<Ctx*>(c);
        return fork_reducer(k.s, *k.A, k.cs, launches, k.gemm_regs);
    };
    st = bwd_grouped_impl(count, local, probs, 0, workspace, workspace_bytes, stream, after_k2, &ctx, before_k2,
                          &ctx);
    int launches = get_launches();
    if (ctx.forked) {
        const lora_status sj = join_reducer(s, cs);
        if (st == LORA_OK) st = sj;
    }
    if (st != LORA_OK) return st;
    if (reduce_lora_grads) {   // the members' partial dA (small, fp32): one NCCL group
        for (int g = 0; g < count && st == LORA_OK; ++g)
            if (problems[g].da)
                st = lora_allreduce(comm, problems[g].da, size_t(local[g].rank) * local[g].d_in, LORA_DT_F32, stream);
        if (st != LORA_OK) return st;
    }
    set_launches(launches);
    return LORA_OK;
}

}  // extern "C"
