// lora_api.cpp -- C ABI of liblora.so (see include/lora.h for the contract).
//
// Validation is synchronous and complete before anything is enqueued; every
// compute step runs in the sm_100a kernels of lora_gemm.cu / lora_aux.cu.
// There is no CPU fallback: a missing or non-sm_100 device is an error.
#include "lora.h"

#include <cuda.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <atomic>
#include <chrono>
#include <cstdlib>
#include <mutex>
#include <string>

#include "lora_internal.h"
#include "lora_kernels.h"

using namespace lora_sm100;

namespace lora_host {

static thread_local std::string g_last_error;
static thread_local int g_last_launches = 0;
// lora_profile_next_bwd: CUDA events recorded around the dX kernel (0, 1) and the
// dA / dB kernel (2, 3) of the next backward call on this thread (one-shot)
static thread_local void* g_prof_events[4] = {};

void prof_record(int i, cudaStream_t stream) {
    if (g_prof_events[i]) cudaEventRecord(static_cast<cudaEvent_t>(g_prof_events[i]), stream);
}
void prof_clear() {
    for (auto& e : g_prof_events) e = nullptr;
}

lora_status fail(lora_status st, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_last_error = buf;
    return st;
}

void set_launches(int n) { g_last_launches = n; }
int get_launches() { return g_last_launches; }

lora_status cuda_fail(cudaError_t e, const char* what) {
    return fail(LORA_ERR_CUDA, "%s: %s (%s)", what, cudaGetErrorName(e), cudaGetErrorString(e));
}

// ------------------------------------------------------------ device info
struct DevInfo {
    int sms = 0;
    int major = 0, minor = 0;
    bool ok = false;
};

static lora_status device_info(DevInfo* out) {
    static std::mutex mu;
    static DevInfo cache[64];
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
    if (dev < 0 || dev >= 64) return fail(LORA_ERR_CUDA, "device ordinal %d out of range", dev);
    std::lock_guard<std::mutex> lk(mu);
    if (!cache[dev].ok) {
        DevInfo d;
        if ((e = cudaDeviceGetAttribute(&d.sms, cudaDevAttrMultiProcessorCount, dev)) != cudaSuccess)
            return cuda_fail(e, "cudaDeviceGetAttribute(SM count)");
        cudaDeviceGetAttribute(&d.major, cudaDevAttrComputeCapabilityMajor, dev);
        cudaDeviceGetAttribute(&d.minor, cudaDevAttrComputeCapabilityMinor, dev);
        d.ok = true;
        cache[dev] = d;
    }
    *out = cache[dev];
    if (!(out->major == 10 && out->minor == 0))
        return fail(LORA_ERR_UNSUPPORTED, "device %d is sm_%d%d; liblora.so is built for sm_100a (B200)",
                    dev, out->major, out->minor);
    return LORA_OK;
}

// ------------------------------------------------------------ TMA descriptors
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                                  CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                                  CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
    static EncodeTiledFn fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeTiledFn>(p);
    });
    return fn;
}

// 2-D bf16 tensor [outer, inner] (row-major, row pitch row_bytes), box
// [box_outer, box_inner].  Out-of-bounds box elements read as zero.
static lora_status encode_2d(CUtensorMap* map, const void* ptr, uint64_t inner, uint64_t outer,
                             uint64_t row_bytes, uint32_t box_inner, uint32_t box_outer, int swizzle_bytes,
                             const char* name, CUtensorMapDataType dtype = CU_TENSOR_MAP_DATA_TYPE_BFLOAT16) {
    EncodeTiledFn fn = encode_fn();
    if (!fn) return fail(LORA_ERR_CUDA, "cuTensorMapEncodeTiled unavailable (driver too old?)");
    cuuint64_t dims[2] = {inner, outer};
    cuuint64_t strides[1] = {row_bytes};
    cuuint32_t box[2] = {box_inner, box_outer};
    cuuint32_t estr[2] = {1, 1};
    CUtensorMapSwizzle sw = swizzle_bytes == 128 ? CU_TENSOR_MAP_SWIZZLE_128B
                            : swizzle_bytes == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
                            : swizzle_bytes == 32 ? CU_TENSOR_MAP_SWIZZLE_32B
                                                  : CU_TENSOR_MAP_SWIZZLE_NONE;
    CUresult r = fn(map, dtype, 2, const_cast<void*>(ptr), dims, strides, box, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS)
        return fail(LORA_ERR_CUDA, "cuTensorMapEncodeTiled(%s: %llu x %llu, box %u x %u) failed: %d", name,
                    (unsigned long long)outer, (unsigned long long)inner, box_outer, box_inner, (int)r);
    return LORA_OK;
}

// ------------------------------------------------------------ validation
static bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

static bool overlap(const void* a, size_t na, const void* b, size_t nb) {
    if (!a || !b || na == 0 || nb == 0) return false;
    const uintptr_t a0 = reinterpret_cast<uintptr_t>(a), b0 = reinterpret_cast<uintptr_t>(b);
    return a0 < b0 + nb && b0 < a0 + na;
}

lora_status check_dims(const lora_dims* d, bool need_tokens) {
    if (!d) return fail(LORA_ERR_INVALID, "dims is NULL");
    if (need_tokens && d->tokens < 0)
        return fail(LORA_ERR_SHAPE, "tokens = %lld must be >= 0", (long long)d->tokens);
    if (d->d_in < 8 || d->d_in % 8 != 0)
        return fail(LORA_ERR_SHAPE, "d_in = %lld must be a positive multiple of 8", (long long)d->d_in);
    if (d->d_out < 8 || d->d_out % 8 != 0)
        return fail(LORA_ERR_SHAPE, "d_out = %lld must be a positive multiple of 8", (long long)d->d_out);
    if (d->rank < 1) return fail(LORA_ERR_SHAPE, "rank = %d must be >= 1", d->rank);
    if (d->rank > 64) return fail(LORA_ERR_UNSUPPORTED, "rank = %d > 64 is not supported", d->rank);
    if (d->d_in > (int64_t(1) << 31) || d->d_out > (int64_t(1) << 31) || d->tokens > (int64_t(1) << 31))
        return fail(LORA_ERR_UNSUPPORTED, "dimension exceeds 2^31");
    if (!std::isfinite(d->alpha)) return fail(LORA_ERR_INVALID, "alpha is not finite");
    return LORA_OK;
}

int r_pad_of(int r) { return r <= 16 ? 16 : (r <= 32 ? 32 : 64); }

static size_t align256(size_t v) { return (v + 255) & ~size_t(255); }

int r8_of(int r) { return (r + 7) / 8 * 8; }

// CTA pairs (256-row tiles) once there are more than 128 tokens; the
// LORA_CTA_GROUP environment variable (1 or 2) overrides, for experiments.
static int cta_group_for(int64_t T) {
    static const int forced = [] {
        const char* s = getenv("LORA_CTA_GROUP");
        return s ? atoi(s) : 0;
    }();
    if (forced == 1 || forced == 2) return forced;
    return T > 128 ? 2 : 1;
}

// Forward workspace: B8 (B zero-padded to a multiple of 8 columns), used only
// when r % 8 != 0 (sized unconditionally so it depends on dims alone).
// Both also hold the fused GEMM's stream-K partial slots when the problem is
// large enough to get a stream-K schedule (fused_gemm_partial_bytes).
struct FwdWs {
    size_t b8, h, partial, partial_bytes, total;
};
static FwdWs fwd_ws(const lora_dims* d, bool dropout = false) {
    FwdWs w;
    w.b8 = 0;
    w.h = align256(size_t(d->d_out) * r8_of(d->rank) * 2);
    w.total = w.h;
    if (dropout) w.total += align256(size_t(d->tokens > 0 ? d->tokens : 0) * d->rank * 4);   // K0's h
    w.partial = w.total;
    w.partial_bytes = fused_gemm_partial_bytes(d->tokens > 0 ? d->tokens : 0, d->d_out);
    w.total += align256(w.partial_bytes);
    return w;
}

// Backward workspace: B^T [r, m], gh [T, r] fp32, h [T, r] fp32 (when not saved).
struct BwdWs {
    size_t b8, gh, h, cs_a, cs_b, xm, bits, partial, partial_bytes, total;
};
static BwdWs bwd_ws(const lora_dims* d, bool dropout = false) {
    BwdWs w;
    const int64_t T = d->tokens > 0 ? d->tokens : 0;
    const int r = d->rank;
    size_t off = 0;
    w.b8 = off; off += align256(size_t(d->d_out) * r8_of(r) * 2);    // only used when r % 8 != 0
    w.gh = off; off += align256(size_t(T) * r * 4);
    w.h = off; off += align256(size_t(T) * r * 4);
    const size_t cs = align256(size_t(3 * r8_of(r)) * size_t((T + 63) / 64 * 64) * 2);
    w.cs_a = off; off += cs;                                         // K3s: split gh
    w.cs_b = off; off += cs;                                         // K3s: split h
    w.xm = off;                                                      // dropout: M . x [T, n] bf16
    if (dropout) off += align256(size_t(T) * size_t(d->d_in) * 2);
    w.bits = off;                                                    // dropout: keep bits [T, ceil(n/32)]
    if (dropout) off += align256(size_t(T) * size_t((d->d_in + 31) / 32) * 4);
    w.partial = off;                                                 // stream-K partials of the dX kernel
    w.partial_bytes = fused_gemm_partial_bytes(T, d->d_in);
    off += align256(w.partial_bytes);
    w.total = off;
    return w;
}

// The dX kernel's per-row-block gh flags live in the self-cleaning device sync
// pool (lora_kernels.h): the gh tile raises them to 1 and the last consumer
// (K2's last CTA, or K3's when K3 waits on them) zeroes them again, so a
// captured CUDA graph replays correctly -- a per-call flag value baked into the
// kernel parameters would already be set by the previous replay.
static constexpr uint64_t kFlagSet = 1;

static lora_status collect(GemmCollector* col, const FusedGemmMaps& maps, const FusedGemmParams& p, int rp, int cg);
static lora_status queue_k0(GemmCollector* col, const void* x, int64_t T, int64_t n, const DropoutMember& m);

// ------------------------------------------------------------ forward
lora_status fwd_impl(const lora_dims* d, const void* x, const void* w0, const void* a, const void* b,
                     const void* bias, void* y, float* h_out, void* ws, size_t ws_bytes,
                     cudaStream_t stream, int* launches, GemmCollector* col, const DropoutParams* drop,
                     bool validate_only) {
    lora_status st = check_dims(d, true);
    if (st != LORA_OK) return st;
    const int64_t T = d->tokens, n = d->d_in, m = d->d_out;
    const int r = d->rank;
    if (!w0 || !a || !b || (T > 0 && (!x || !y)))
        return fail(LORA_ERR_INVALID, "lora_linear_fwd: x, w0, a, b, y must be non-NULL");
    const void* ptrs[] = {x, w0, a, b, bias, y, h_out, ws};
    const char* names[] = {"x", "w0", "a", "b", "bias", "y", "h_out", "workspace"};
    for (int i = 0; i < 8; ++i)
        if (ptrs[i] && !aligned16(ptrs[i]))
            return fail(LORA_ERR_ALIGN, "lora_linear_fwd: %s = %p is not 16-byte aligned", names[i], ptrs[i]);
    const FwdWs W = fwd_ws(d, drop != nullptr);
    if (!ws || ws_bytes < W.total)
        return fail(LORA_ERR_WORKSPACE, "lora_linear_fwd: workspace %zu bytes < required %zu", ws ? ws_bytes : 0,
                    W.total);
    const size_t yb = size_t(T) * m * 2, hb = h_out ? size_t(T) * r * 4 : 0;
    const void* ins[] = {x, w0, a, b, bias};
    const size_t inb[] = {size_t(T) * n * 2, size_t(m) * n * 2, size_t(r) * n * 2, size_t(m) * r * 2,
                          bias ? size_t(m) * 2 : 0};
    for (int i = 0; i < 5; ++i) {
        if (overlap(y, yb, ins[i], inb[i]) || overlap(h_out, hb, ins[i], inb[i]) ||
            overlap(ws, W.total, ins[i], inb[i]))
            return fail(LORA_ERR_INVALID, "lora_linear_fwd: an output/workspace overlaps input %s", names[i]);
    }
    if (overlap(y, yb, h_out, hb)) return fail(LORA_ERR_INVALID, "lora_linear_fwd: y overlaps h_out");
    DevInfo dev;
    if ((st = device_info(&dev)) != LORA_OK) return st;
    if (T == 0 || validate_only) return LORA_OK;

    const int rp = r_pad_of(r);
    const int r8 = r8_of(r);
    const int BN = fused_gemm_block_n(kModeFwd, rp);
    // B is read by TMA with its own row pitch when r % 8 == 0; otherwise a
    // zero-padded copy B8 [m, r8] is made first (B6).
    const void* bsrc = b;
    if (r != r8) {
        auto* b8 = reinterpret_cast<__nv_bfloat16*>(static_cast<uint8_t*>(ws) + W.b8);
        cudaError_t e = launch_pack_b(static_cast<const __nv_bfloat16*>(b), m, r, b8, nullptr, dev.sms, stream);
        if (e != cudaSuccess) return cuda_fail(e, "pack launch");
        ++*launches;
        bsrc = b8;
    }
    FusedGemmMaps maps;
    const int cg = cta_group_for(T);
    if ((st = encode_2d(&maps.act, x, n, T, n * 2, 64, 128, 128, "x")) != LORA_OK) return st;
    // W0 rows of the [W0 ; A] B-operand tile: CTA pair splits it 128 / (BN - 128) + A rows
    if ((st = encode_2d(&maps.w, w0, n, m, n * 2, 64, cg == 2 ? 128 : BN, 128, "w0")) != LORA_OK) return st;
    maps.w2 = maps.w;
    if (cg == 2 && (st = encode_2d(&maps.w2, w0, n, m, n * 2, 64, BN - 128, 128, "w0")) != LORA_OK) return st;
    if ((st = encode_2d(&maps.nar, a, n, r, n * 2, 64, rp, 128, "a")) != LORA_OK) return st;
    if ((st = encode_2d(&maps.tail, bsrc, r8, m, r8 * 2, rp, BN / cg, rp * 2, "b")) != LORA_OK) return st;
    // the TMA-store epilogue's output maps: y [T, m], boxes [128 x 32] SW64 and [128 x 16] SW32
    if ((st = encode_2d(&maps.out32, y, m, T, m * 2, 32, 128, 64, "y")) != LORA_OK) return st;
    if ((st = encode_2d(&maps.out16, y, m, T, m * 2, 16, 128, 32, "y")) != LORA_OK) return st;
    FusedGemmParams p;
    p.T = T; p.K = n; p.N_out = m; p.r = r;
    p.scale = d->alpha / static_cast<float>(r);
    p.bias = static_cast<const __nv_bfloat16*>(bias);
    p.out = static_cast<__nv_bfloat16*>(y);
    p.side_out = h_out;
    p.gh = nullptr;
    p.flags = nullptr;
    p.epoch = 0;
    p.nflags = 0;
    p.reset_flags = 0;
    p.h_in = nullptr;
    p.drop = DropoutParams{};
    p.drop_bits = nullptr;
    p.cs_gh = p.cs_h = nullptr;
    p.cs_gh_rows = 0;
    p.h_split_src = nullptr;
    p.t_pad = 0;
    p.sk_partial = W.partial_bytes ? reinterpret_cast<float*>(static_cast<uint8_t*>(ws) + W.partial) : nullptr;
    p.unit_flags = nullptr;
    if (drop && drop->thr > 0) {
        // LoRA dropout: K0 computes h = q (M . x) A^T; K1 takes it instead of its in-MMA
        // x A^T -- K0 is queued (grouped: one launch for every member sharing x) and K1
        // overlaps it (programmatic stream serialization; its epilogue waits for K0)
        float* hd = h_out ? h_out : reinterpret_cast<float*>(static_cast<uint8_t*>(ws) + W.h);
        p.h_in = hd;
        p.side_out = nullptr;
        const DropoutMember mem{static_cast<const __nv_bfloat16*>(a), r, *drop, hd, drop->masked_x,
                                drop->keep_bits, nullptr, {}};
        if (col) {
            if ((st = queue_k0(col, x, T, n, mem)) != LORA_OK) return st;
            return collect(col, maps, p, rp, cg);
        }
        GemmCollector one;
        if ((st = queue_k0(&one, x, T, n, mem)) != LORA_OK) return st;
        if ((st = collect(&one, maps, p, rp, cg)) != LORA_OK) return st;
        if ((st = launch_collected_k0(one, stream, launches)) != LORA_OK) return st;
        return launch_collected(kModeFwd, one, stream, launches);
    }
    if (col) return collect(col, maps, p, rp, cg);
    cudaError_t e = launch_fused_gemm(kModeFwd, rp, cg, maps, p, dev.sms, stream);
    if (e != cudaSuccess) return cuda_fail(e, "fused forward launch");
    ++*launches;
    return LORA_OK;
}

// K3 implementation: "mma" (default, tensor cores) or the CUDA-core
// comparison kernel "cluster" (LORA_K3=cluster).
enum K3Mode { kK3Mma, kK3Cluster };
static K3Mode k3_mode() {
    const char* v = getenv("LORA_K3");
    return v && !strcmp(v, "cluster") ? kK3Cluster : kK3Mma;
}

// K3 on the tensor cores for `count` problems: one dA set (X = x, C = gh) and
// one dB set (X = dY, C = h, scale s) per problem; dA sets of problems that
// share x (same pointer and shape) are stacked into one job, so x is read once.
// Two launches: K3s (split every coefficient matrix once) and K3.
static int64_t t_pad_of(int64_t T) { return (T + 63) / 64 * 64; }

static lora_status launch_k3_mma(const GradArgs* pr, int count, cudaStream_t stream, int* launches) {
    DevInfo dev;
    lora_status st = device_info(&dev);
    if (st != LORA_OK) return st;
    if (count > kMaxGroup) return fail(LORA_ERR_UNSUPPORTED, "too many problems for one K3 launch");
    static thread_local GradMmaGroup G;
    static thread_local CoefSplitGroup SG;
    struct Pending {
        const void* X;
        int64_t T, N;
        const float* coef;
        __nv_bfloat16* cs;
        bool ready;          // cs already written (by K2's gh tile)
        GradMmaSet set;
    } sets[kMaxGradSetsTotal];
    int ns = 0;
    for (int i = 0; i < count; ++i) {
        const GradArgs& g = pr[i];
        const int r8 = (g.r + 7) / 8 * 8;
        if (g.da) {
            GradMmaSet s = {g.da, 1, g.n, g.r, r8, 0, (g.accumulate & kAccA) ? 1 : 0, g.scale_a, 3, nullptr, 0};
            if (g.cs_a_k2 && g.k2_flags) { s.wait_flags = g.k2_flags; s.wait_n = g.k2_nflags; }
            sets[ns++] = {g.x, g.T, g.n, g.gh, g.cs_a, g.cs_a_ready != 0, s};
        }
        if (g.db) {
            GradMmaSet s = {g.db, g.r, 1, g.r, r8, 0, (g.accumulate & kAccB) ? 1 : 0, g.scale_b, 3, nullptr, 0};
            if (g.cs_b_k2 && g.k2_flags) { s.wait_flags = g.k2_flags; s.wait_n = g.k2_nflags; }
            sets[ns++] = {g.dy, g.T, g.m, g.h, g.cs_b, g.cs_b_ready != 0, s};
        }
    }
    if (ns == 0) return LORA_OK;
    // group the sets into jobs: same activation (pointer, T, N), at most 256 B-operand rows
    int job_of[kMaxGradSetsTotal];
    int used[kMaxGradJobs];
    int nj = 0;
    const void* jx[kMaxGradJobs];
    for (int i = 0; i < ns; ++i) {
        job_of[i] = -1;
        for (int j = 0; j < nj; ++j)
            if (jx[j] == sets[i].X && G.job[j].T == sets[i].T && G.job[j].N == sets[i].N &&
                used[j] + 3 * sets[i].set.r8 <= 256) {
                job_of[i] = j;
                break;
            }
        if (job_of[i] < 0) {
            GradMmaJob& J = G.job[nj];
            J.T = sets[i].T; J.N = sets[i].N; J.nsets = 0; J.a_kmajor = 0;
            jx[nj] = sets[i].X;
            used[nj] = 0;
            job_of[i] = nj++;
        }
        used[job_of[i]] += 3 * sets[i].set.r8;
    }
    // sets in job order (each job's sets contiguous), row offsets, maps
    int k = 0;
    SG.count = 0;
    for (int j = 0; j < nj; ++j) {
        GradMmaJob& J = G.job[j];
        J.set0 = k;
        J.nsets = 0;
        int row = 0;
        for (int i = 0; i < ns; ++i) {
            if (job_of[i] != j) continue;
            GradMmaSet s = sets[i].set;
            s.row0 = row;
            row += 3 * s.r8;
            G.set[k] = s;
            const int64_t tp = t_pad_of(sets[i].T);
            // inner extent T (not T_pad): TMA zero-fills the token tail, so the pad is never read
            if ((st = encode_2d(&G.csmap[k], sets[i].cs, sets[i].T, 3 * s.r8, tp * 2, 64, 3 * s.r8, 128,
                                "K3 split coefficients")) != LORA_OK)
                return st;
            if (!sets[i].ready) SG.s[SG.count++] = {sets[i].coef, sets[i].cs, sets[i].T, tp, s.r, s.r8};
            ++k;
            ++J.nsets;
        }
        J.q_used = row;
        J.q_pad = (row + 15) / 16 * 16;
        if ((st = encode_2d(&G.xmap[j], jx[j], J.N, J.T, J.N * 2, 64, 64, 128, "K3 activation")) != LORA_OK)
            return st;
    }
    G.njobs = nj;
    cudaError_t e;
    if (SG.count > 0) {   // coefficient matrices K2 did not already split
        if ((e = launch_coef_split(SG, stream)) != cudaSuccess) return cuda_fail(e, "K3s (coefficient split) launch");
        ++*launches;
    }
    // every coefficient set comes straight from the K2 launched just before (no K3s
    // in between): K3 may start on the SMs K2 frees and wait on K2's flags instead
    bool overlap = SG.count == 0, waits = false;
    for (int i = 0; i < k; ++i) {
        overlap = overlap && G.set[i].wait_flags != nullptr;
        waits = waits || G.set[i].wait_flags != nullptr;
    }
    G.done = nullptr;
    prof_record(2, stream);
    if (waits && (G.done = sync_pool_alloc(1, stream)) == nullptr)
        e = cudaErrorMemoryAllocation;
    else
        e = launch_grad_mma(G, dev.sms, stream, overlap);
    prof_record(3, stream);
    if (e != cudaSuccess) {
        for (int i = 0; i < k; ++i)   // leave no raised flag behind in the pool
            if (G.set[i].wait_flags)
                cudaMemsetAsync(const_cast<uint64_t*>(G.set[i].wait_flags), 0, size_t(G.set[i].wait_n) * 8, stream);
        return cuda_fail(e, "K3 (tensor-core dA / dB) launch");
    }
    ++*launches;
    return LORA_OK;
}

// Row projection on the tensor cores: out[t, j] = scale * sum_k X[t, k] P[j, k] for
// X [T, K] bf16 and P [r, K] bf16 (K-contiguous rows: A itself, or B^T) -- the K3
// kernel with X read K-major and P as a single (unsplit, already bf16) coefficient set.
// Used for gh = s dY B when dX is not requested and for h = x A^T when h was not saved.
static lora_status launch_rowproj_mma(const void* X, int64_t T, int64_t K, const void* P, int r, float scale,
                                      float* out, cudaStream_t stream, int* launches,
                                      __nv_bfloat16* cs_out = nullptr /* also K3's split, r % 8 == 0 */) {
    DevInfo dev;
    lora_status st = device_info(&dev);
    if (st != LORA_OK) return st;
    static thread_local GradMmaGroup G;
    const int r8 = (r + 7) / 8 * 8;
    GradMmaJob& J = G.job[0];
    J.T = K; J.N = T; J.set0 = 0; J.nsets = 1; J.q_used = r8; J.q_pad = (r8 + 15) / 16 * 16; J.a_kmajor = 1;
    G.set[0] = GradMmaSet{out, r, 1, r, r8, 0, 0, scale, 1};
    G.set[0].cs_out = (cs_out && r == r8) ? cs_out : nullptr;
    G.set[0].cs_t_pad = t_pad_of(T);
    if ((st = encode_2d(&G.xmap[0], X, K, T, K * 2, 64, 64, 128, "row-projection activation")) != LORA_OK) return st;
    // P rows r..r8-1 are out of bounds: TMA zero-fills them
    if ((st = encode_2d(&G.csmap[0], P, K, r, K * 2, 64, r8, 128, "row-projection operand")) != LORA_OK) return st;
    G.njobs = 1;
    cudaError_t e = launch_grad_mma(G, dev.sms, stream);
    if (e != cudaSuccess) return cuda_fail(e, "row projection (tensor cores) launch");
    ++*launches;
    return LORA_OK;
}

lora_status launch_collected_k3(GemmCollector& col, cudaStream_t stream, int* launches) {
    if (k3_mode() == kK3Mma) {
        lora_status st = launch_k3_mma(col.k3, col.k3_count, stream, launches);
        col.k3_count = 0;
        return st;
    }
    static thread_local GradGroup G;
    bool done[kMaxGroup] = {};
    prof_record(2, stream);
    for (int i = 0; i < col.k3_count; ++i) {
        if (done[i]) continue;
        G.count = 0;
        for (int j = i; j < col.k3_count; ++j) {
            if (done[j] || grad_rank_bucket(col.k3[j].r) != grad_rank_bucket(col.k3[i].r)) continue;
            G.g[G.count++] = col.k3[j];
            done[j] = true;
        }
        cudaError_t e = launch_grad_reduce_cluster_group(G, stream, launches);
        if (e != cudaSuccess) return cuda_fail(e, "grouped grad reduce launch");
    }
    prof_record(3, stream);
    col.k3_count = 0;
    return LORA_OK;
}

static lora_status collect(GemmCollector* col, const FusedGemmMaps& maps, const FusedGemmParams& p, int rp, int cg) {
    if (col->count >= kMaxGroup) return fail(LORA_ERR_UNSUPPORTED, "more than %d grouped problems", kMaxGroup);
    col->maps[col->count] = maps;
    col->p[col->count] = p;
    col->rp[col->count] = rp;
    col->cg[col->count] = cg;
    ++col->count;
    return LORA_OK;
}

lora_status launch_collected(int mode, GemmCollector& col, cudaStream_t stream, int* launches) {
    if (col.count == 0) return LORA_OK;
    DevInfo dev;
    lora_status st = device_info(&dev);
    if (st != LORA_OK) return st;
    static thread_local FusedGemmGroup grp;
    bool done[kMaxGroup] = {};
    for (int i = 0; i < col.count; ++i) {
        if (done[i]) continue;
        grp.count = 0;
        grp.no_coop = col.no_coop ? 1 : 0;
        for (int j = i; j < col.count; ++j) {
            if (done[j] || col.rp[j] != col.rp[i] || col.cg[j] != col.cg[i]) continue;
            grp.maps[grp.count] = col.maps[j];
            grp.p[grp.count] = col.p[j];
            ++grp.count;
            done[j] = true;
        }
        const int sms = (col.max_sms > 0 && col.max_sms < dev.sms) ? col.max_sms : dev.sms;
        cudaError_t e = launch_fused_gemm_group(mode, col.rp[i], col.cg[i], grp, sms, stream);
        if (e != cudaSuccess) return cuda_fail(e, "grouped fused GEMM launch");
        ++*launches;
    }
    return LORA_OK;
}

// K0 of the collected problems (members sharing x, each its own mask), in
// stream order right before the fused GEMMs: the forward's h products of all
// members in one tensor-core launch, the backward's masked inputs and keep bits
// in one streaming launch (lora_dropout.cu).  Measured and dropped (DESIGN.md
// dropout path): the fused GEMM launched with programmatic stream serialization
// to overlap K0 -- K0 fills every SM and cannot share them with the GEMM's CTAs.
lora_status launch_collected_k0(GemmCollector& col, cudaStream_t stream, int* launches) {
    if (col.k0.count == 0) return LORA_OK;
    DevInfo dev;
    lora_status st = device_info(&dev);
    if (st != LORA_OK) return st;
    cudaError_t e = launch_dropout_input_group(col.k0, dev.sms, stream, launches);
    if (e != cudaSuccess) return cuda_fail(e, "dropout K0 launch");
    col.k0.count = 0;
    return LORA_OK;
}

// queue K0 work for `col` (one grouped launch later); members must share x
static lora_status queue_k0(GemmCollector* col, const void* x, int64_t T, int64_t n, const DropoutMember& m) {
    if (col->k0.count > 0 && (col->k0.x != x || col->k0.T != T || col->k0.n != n))
        return fail(LORA_ERR_UNSUPPORTED, "grouped LoRA dropout: the problems must share the input x");
    if (col->k0.count >= kMaxGroup) return fail(LORA_ERR_UNSUPPORTED, "more than %d grouped problems", kMaxGroup);
    col->k0.x = static_cast<const __nv_bfloat16*>(x);
    col->k0.T = T;
    col->k0.n = n;
    col->k0.m[col->k0.count++] = m;
    return LORA_OK;
}

// ------------------------------------------------------------ backward
lora_status bwd_impl(const lora_dims* d, const void* x, const void* w0, const void* a, const void* b,
                     const float* h_saved, const void* dy, void* dx, float* da, float* db, int accumulate,
                     void* ws, size_t ws_bytes, cudaStream_t stream, int* launches, GemmCollector* col,
                     int stages, const DropoutParams* drop) {
    lora_status st = check_dims(d, true);
    if (st != LORA_OK) return st;
    const int64_t T = d->tokens, n = d->d_in, m = d->d_out;
    const int r = d->rank;
    if (!w0 || !a || !b || (T > 0 && (!x || !dy)))
        return fail(LORA_ERR_INVALID, "lora_linear_bwd: x, w0, a, b, dy must be non-NULL");
    if (accumulate < 0 || accumulate > (kAccA | kAccB)) return fail(LORA_ERR_INVALID, "accumulate must be 0 or 1");
    const void* ptrs[] = {x, w0, a, b, h_saved, dy, dx, da, db, ws};
    const char* names[] = {"x", "w0", "a", "b", "h_saved", "dy", "dx", "da", "db", "workspace"};
    for (int i = 0; i < 10; ++i)
        if (ptrs[i] && !aligned16(ptrs[i]))
            return fail(LORA_ERR_ALIGN, "lora_linear_bwd: %s = %p is not 16-byte aligned", names[i], ptrs[i]);
    const bool dropping = drop && drop->thr > 0;
    const BwdWs W = bwd_ws(d, drop != nullptr);
    if (!ws || ws_bytes < W.total)
        return fail(LORA_ERR_WORKSPACE, "lora_linear_bwd: workspace %zu bytes < required %zu", ws ? ws_bytes : 0,
                    W.total);
    const void* ins[] = {x, w0, a, b, h_saved, dy};
    const size_t inb[] = {size_t(T) * n * 2, size_t(m) * n * 2, size_t(r) * n * 2, size_t(m) * r * 2,
                          h_saved ? size_t(T) * r * 4 : 0, size_t(T) * m * 2};
    const void* outs[] = {dx, da, db, ws};
    const size_t outb[] = {dx ? size_t(T) * n * 2 : 0, da ? size_t(r) * n * 4 : 0, db ? size_t(m) * r * 4 : 0,
                           W.total};
    for (int o = 0; o < 4; ++o) {
        for (int i = 0; i < 6; ++i)
            if (overlap(outs[o], outb[o], ins[i], inb[i]))
                return fail(LORA_ERR_INVALID, "lora_linear_bwd: output %s overlaps input %s",
                            o == 3 ? "workspace" : names[6 + o], names[i]);
        for (int o2 = o + 1; o2 < 4; ++o2)
            if (overlap(outs[o], outb[o], outs[o2], outb[o2]))
                return fail(LORA_ERR_INVALID, "lora_linear_bwd: outputs overlap each other");
    }
    DevInfo dev;
    if ((st = device_info(&dev)) != LORA_OK) return st;
    if (stages & kStageValidate) return LORA_OK;
    cudaError_t e;
    if (T == 0) {
        if (stages & 1) {
            if (!(accumulate & kAccA) && (e = launch_fill_zero(da, int64_t(r) * n, stream)) != cudaSuccess)
                return cuda_fail(e, "memset dA");
            if (!(accumulate & kAccB) && (e = launch_fill_zero(db, int64_t(m) * r, stream)) != cudaSuccess)
                return cuda_fail(e, "memset dB");
        }
        return LORA_OK;
    }
    const float s = d->alpha / static_cast<float>(r);
    const int rp = r_pad_of(r);
    const int r8 = r8_of(r);
    uint8_t* wsb = static_cast<uint8_t*>(ws);
    float* gh = reinterpret_cast<float*>(wsb + W.gh);
    float* hbuf = reinterpret_cast<float*>(wsb + W.h);
    const auto* xa = static_cast<const __nv_bfloat16*>(x);
    const auto* aa = static_cast<const __nv_bfloat16*>(a);
    const auto* dya = static_cast<const __nv_bfloat16*>(dy);
    const bool need_gh = dx || da;
    const bool need_h = db && !h_saved;
    const uint64_t* k2_flags = nullptr;   // this problem's K2 gh flags (stage 1; grouped stage 2: from col)
    bool gh_split = false, h_split = false;   // a row projection already wrote K3's split of gh / h

    // M . x for dA: the forward's (lora_dropout.masked_x) when the caller kept it, else K0 writes it
    auto* xm = (drop && drop->masked_x) ? drop->masked_x : reinterpret_cast<__nv_bfloat16*>(wsb + W.xm);
    GemmCollector one;                      // single calls: K0 + K2 through a local collector
    GemmCollector* k0col = col ? col : &one;
    if (dropping && (stages & 1)) {
        // K0: keep bits for K2's epilogue, M . x for dA, h = q (M . x) A^T when not saved -- one
        // pass over x, queued (grouped: one launch for the members sharing x) right before K2,
        // which overlaps it and waits for it in its epilogue only
        // (the caller's keep_bits from the forward: read, nothing drawn except for a recomputed h)
        const DropoutMember mem{static_cast<const __nv_bfloat16*>(a), r, *drop, need_h ? hbuf : nullptr,
                                (da && !drop->masked_x) ? xm : nullptr,
                                (dx && !drop->keep_bits) ? reinterpret_cast<uint32_t*>(wsb + W.bits) : nullptr,
                                drop->keep_bits, {}};
        if ((st = queue_k0(k0col, x, T, n, mem)) != LORA_OK) return st;
        if (!col && !dx && (st = launch_collected_k0(one, stream, launches)) != LORA_OK) return st;
    }
    if (dx && (stages & 1)) {
        // K2 computes gh = s dY B itself (first column tile of each row block)
        const __nv_bfloat16* bsrc = static_cast<const __nv_bfloat16*>(b);
        if (r != r8) {   // B rows of 2r bytes are not TMA-legal: B6 pads them to r8
            auto* b8 = reinterpret_cast<__nv_bfloat16*>(wsb + W.b8);
            if ((e = launch_pack_b(bsrc, m, r, b8, nullptr, dev.sms, stream)) != cudaSuccess)
                return cuda_fail(e, "pack launch");
            ++*launches;
            bsrc = b8;
        }
        FusedGemmMaps maps;
        const int cg = cta_group_for(T);
        const int nar_h = fused_gemm_narrow_cols(rp, cg);
        if ((st = encode_2d(&maps.act, dy, m, T, m * 2, 64, 128, 128, "dy")) != LORA_OK) return st;
        if ((st = encode_2d(&maps.w, w0, n, m, n * 2, 64, 64, 128, "w0")) != LORA_OK) return st;
        maps.w2 = maps.w;
        if ((st = encode_2d(&maps.nar, bsrc, r8, m, r8 * 2, nar_h, 64, nar_h * 2, "b")) != LORA_OK) return st;
        if ((st = encode_2d(&maps.tail, a, n, r, n * 2, 64, rp, 128, "a")) != LORA_OK) return st;
        if ((st = encode_2d(&maps.out32, dx, n, T, n * 2, 32, 128, 64, "dx")) != LORA_OK) return st;
        if ((st = encode_2d(&maps.out16, dx, n, T, n * 2, 16, 128, 32, "dx")) != LORA_OK) return st;
        FusedGemmParams p;
        p.T = T; p.K = m; p.N_out = n; p.r = r; p.scale = s;
        p.bias = nullptr;
        p.out = static_cast<__nv_bfloat16*>(dx);
        p.side_out = nullptr;
        p.epoch = kFlagSet;
        p.nflags = static_cast<int>(fused_gemm_row_blocks(T, cg) * cg);
        p.flags = p.nflags > 0 ? reinterpret_cast<uint64_t*>(sync_pool_alloc(p.nflags, stream)) : nullptr;
        if (p.nflags > 0 && p.flags == nullptr)
            return fail(LORA_ERR_CUDA, "dX kernel: device sync pool exhausted or unavailable");
        // K3 (tensor cores) waits on these flags and zeroes them when it reads a
        // coefficient split this K2 writes; otherwise K2's last CTA does
        const bool k3_waits = k3_mode() == kK3Mma &&
                              (da != nullptr || (db != nullptr && (h_saved != nullptr || (dropping && need_h))));
        p.reset_flags = k3_waits ? 0 : 1;
        k2_flags = p.flags;
        p.h_in = nullptr;
        p.drop = dropping ? *drop : DropoutParams{};
        p.drop_bits = !dropping ? nullptr
                      : drop->keep_bits ? drop->keep_bits : reinterpret_cast<const uint32_t*>(wsb + W.bits);
        // the gh tile also writes K3's split coefficients (gh; h when it already exists)
        p.t_pad = t_pad_of(T);
        p.sk_partial = W.partial_bytes ? reinterpret_cast<float*>(wsb + W.partial) : nullptr;
        p.unit_flags = nullptr;
        // the gh tile publishes gh to the other tiles through cs_a (hi rows; the full
        // split when dA -- or the dropout epilogue's fp32 gh -- needs it)
        p.cs_gh = reinterpret_cast<__nv_bfloat16*>(wsb + W.cs_a);
        p.cs_gh_rows = (da || dropping) ? 3 : 1;
        p.gh = k3_mode() == kK3Cluster ? gh : nullptr;   // fp32 gh: only the CUDA-core K3 reads it
        p.h_split_src = h_saved ? h_saved : (dropping && need_h ? hbuf : nullptr);
        p.cs_h = db && p.h_split_src ? reinterpret_cast<__nv_bfloat16*>(wsb + W.cs_b) : nullptr;
        if (col) {
            if ((st = collect(col, maps, p, rp, cg)) != LORA_OK) return st;
        } else if (dropping) {
            // dropout: the epilogue applies q M . (gh A) itself (no tail MMA); K0 right before
            if ((st = collect(&one, maps, p, rp, cg)) != LORA_OK) return st;
            if ((st = launch_collected_k0(one, stream, launches)) != LORA_OK) return st;
            prof_record(0, stream);
            st = launch_collected(kModeDxDrop, one, stream, launches);
            prof_record(1, stream);
            if (st != LORA_OK) return st;
        } else {
            prof_record(0, stream);
            e = launch_fused_gemm(kModeDx, rp, cg, maps, p, dev.sms, stream);
            prof_record(1, stream);
            if (e != cudaSuccess) return cuda_fail(e, "fused dX launch");
            ++*launches;
        }
    }
    if (!(stages & 2)) return LORA_OK;
    if (!dx && da) {
        // K2a: gh = s dY B [T, r] fp32 for dA when the input gradient is not requested --
        // B^T [r, m] (B6, into the unused B8 slot) then the tensor-core row projection
        auto* bt = reinterpret_cast<__nv_bfloat16*>(wsb + W.b8);
        // the same launch splits the saved h for K3's dB when it can (no K3s pass)
        h_split = db && h_saved && r % 8 == 0 && k3_mode() == kK3Mma && !dropping;
        if ((e = launch_pack_b(static_cast<const __nv_bfloat16*>(b), m, r, nullptr, bt, dev.sms, stream,
                               h_split ? h_saved : nullptr,
                               h_split ? reinterpret_cast<__nv_bfloat16*>(wsb + W.cs_b) : nullptr, T,
                               t_pad_of(T))) != cudaSuccess)
            return cuda_fail(e, "B^T pack launch");
        ++*launches;
        // (r % 8 == 0: it also writes K3's split of gh -- no K3s pass)
        gh_split = r % 8 == 0 && k3_mode() == kK3Mma;
        if ((st = launch_rowproj_mma(dya, T, m, bt, r, s, gh, stream, launches,
                                     gh_split ? reinterpret_cast<__nv_bfloat16*>(wsb + W.cs_a) : nullptr)) != LORA_OK)
            return st;
    }
    const float* hsrc = h_saved;
    const __nv_bfloat16* xk3 = xa;   // K3's dA activation: x, or M . x under dropout
    float scale_a = 1.0f;
    if (dropping) {   // K0 (above) wrote M . x and, if needed, h
        if (need_h) hsrc = hbuf;
        xk3 = xm;
        scale_a = drop->q;
    } else if (need_h) {
        // K3a: h = x A^T recomputed on the tensor cores (A [r, n] is already K-contiguous);
        // r % 8 == 0: it also writes K3's split of h (no K3s pass)
        h_split = r % 8 == 0 && k3_mode() == kK3Mma;
        if ((st = launch_rowproj_mma(xa, T, n, aa, r, 1.0f, hbuf, stream, launches,
                                     h_split ? reinterpret_cast<__nv_bfloat16*>(wsb + W.cs_b) : nullptr)) != LORA_OK)
            return st;
        hsrc = hbuf;
    }
    if (da || db) {
        const K3Mode k3 = k3_mode();
        if (dropping && k3 != kK3Mma) return fail(LORA_ERR_UNSUPPORTED, "LoRA dropout needs the default K3");
        GradArgs g = make_grad_args(T, n, m, r, s, xk3, gh, dya, hsrc, da, db, accumulate);
        g.scale_a = scale_a;
        g.cs_a = reinterpret_cast<__nv_bfloat16*>(wsb + W.cs_a);
        g.cs_b = reinterpret_cast<__nv_bfloat16*>(wsb + W.cs_b);
        // who wrote K3's split coefficients: K2 (then K3 waits on K2's per-row-block flags)
        // or a row projection / pack launched after K2 in stream order (no wait: K2 may
        // already have reset its flags -- they are only kept for K3 when k3_waits)
        g.cs_a_k2 = dx != nullptr;
        g.cs_b_k2 = dx != nullptr && (h_saved != nullptr || (dropping && need_h));
        g.cs_a_ready = g.cs_a_k2 || gh_split;                             // K2 / K2a split gh
        g.cs_b_ready = g.cs_b_k2 || h_split;                              // K2 / B6 / K3a split h
        if (dx && !k2_flags && col) {   // grouped: stage 1 collected this problem's K2
            for (int i = 0; i < col->count; ++i)
                if (col->p[i].out == dx) k2_flags = col->p[i].flags;
        }
        if (dx) {   // K2 raises these once a row block's split coefficients are written
            if (!k2_flags && T > 0) return fail(LORA_ERR_INVALID, "lora_linear_bwd: internal: dX kernel flags not found");
            g.k2_flags = k2_flags;
            g.k2_nflags = static_cast<int>(fused_gemm_row_blocks(T, cta_group_for(T)) * cta_group_for(T));
        }
        if (col) {   // grouped backward: one K3 launch for the whole group
            if (col->k3_count >= kMaxGroup) return fail(LORA_ERR_UNSUPPORTED, "too many grouped problems");
            col->k3[col->k3_count++] = g;
            return LORA_OK;
        }
        if (k3 == kK3Mma) return launch_k3_mma(&g, 1, stream, launches);
        e = launch_grad_reduce_cluster(T, n, m, r, s, xk3, gh, dya, hsrc, da, db, accumulate, stream, launches);
        if (e != cudaSuccess) return cuda_fail(e, "grad reduce launch");
    }
    return LORA_OK;
}

lora_status merge_impl(const lora_dims* d, const void* w0, const void* a, const void* b, void* w_out,
                       cudaStream_t stream, int* launches) {
    lora_status st = check_dims(d, false);
    if (st != LORA_OK) return st;
    const int64_t n = d->d_in, m = d->d_out;
    const int r = d->rank;
    if (!w0 || !a || !b || !w_out) return fail(LORA_ERR_INVALID, "lora_merge: w0, a, b, w_out must be non-NULL");
    const void* ptrs[] = {w0, a, b, w_out};
    const char* names[] = {"w0", "a", "b", "w_out"};
    for (int i = 0; i < 4; ++i)
        if (!aligned16(ptrs[i]))
            return fail(LORA_ERR_ALIGN, "lora_merge: %s = %p is not 16-byte aligned", names[i], ptrs[i]);
    const size_t wb = size_t(m) * n * 2;
    if (w_out != w0 && overlap(w_out, wb, w0, wb))
        return fail(LORA_ERR_INVALID, "lora_merge: w_out partially overlaps w0 (only w_out == w0 is allowed)");
    if (overlap(w_out, wb, a, size_t(r) * n * 2) || overlap(w_out, wb, b, size_t(m) * r * 2))
        return fail(LORA_ERR_INVALID, "lora_merge: w_out overlaps a or b");
    DevInfo dev;
    if ((st = device_info(&dev)) != LORA_OK) return st;
    const float s = d->alpha / static_cast<float>(r);
    const char* mv = getenv("LORA_MERGE");
    if (r % 8 == 0 && r <= 64 && !(mv && (!strcmp(mv, "cuda") || !strcmp(mv, "oneshot")))) {
        // tensor cores (lora_merge_mma.cu): B's rows are 16-byte multiples, so B is a TMA operand as is
        const int rp = r <= 16 ? 16 : (r <= 32 ? 32 : 64);
        MergeMaps maps;
        if ((st = encode_2d(&maps.w, w0, n, m, n * 2, 64, 128, 128, "w0")) != LORA_OK) return st;
        if ((st = encode_2d(&maps.out, w_out, n, m, n * 2, 64, 128, 128, "w_out")) != LORA_OK) return st;
        if ((st = encode_2d(&maps.b, b, r, m, r * 2, rp, 128, rp * 2, "b")) != LORA_OK) return st;
        if ((st = encode_2d(&maps.a, a, n, r, n * 2, 64, rp, 128, "a")) != LORA_OK) return st;
        cudaError_t e = launch_merge_mma(maps, rp, m, n, s, dev.sms, stream);
        if (e != cudaSuccess) return cuda_fail(e, "merge launch");
        ++*launches;
        return LORA_OK;
    }
    cudaError_t e = launch_merge(static_cast<const __nv_bfloat16*>(w0), static_cast<const __nv_bfloat16*>(a),
                                 static_cast<const __nv_bfloat16*>(b), n, m, r, d->alpha / static_cast<float>(r),
                                 static_cast<__nv_bfloat16*>(w_out), stream);
    if (e != cudaSuccess) return cuda_fail(e, "merge launch");
    ++*launches;
    return LORA_OK;
}

size_t fwd_workspace(const lora_dims* d) { return check_dims(d, true) == LORA_OK ? fwd_ws(d).total : 0; }
size_t bwd_workspace(const lora_dims* d) { return check_dims(d, true) == LORA_OK ? bwd_ws(d).total : 0; }
size_t fwd_workspace_dropout(const lora_dims* d) {
    return check_dims(d, true) == LORA_OK ? fwd_ws(d, true).total : 0;
}
size_t bwd_workspace_dropout(const lora_dims* d) {
    return check_dims(d, true) == LORA_OK ? bwd_ws(d, true).total : 0;
}

// lora_dropout -> kernel parameters (threshold floor(p 2^16) computed in fp64, as the oracle does)
lora_status dropout_params(const lora_dropout* dr, DropoutParams* out) {
    if (!dr) return fail(LORA_ERR_INVALID, "dropout is NULL");
    if (!(dr->p >= 0.0f && dr->p < 1.0f))
        return fail(LORA_ERR_INVALID, "dropout p = %g must be in [0, 1)", static_cast<double>(dr->p));
    out->seed = dr->seed;
    out->offset = dr->offset;
    out->thr = static_cast<uint32_t>(static_cast<double>(dr->p) * 65536.0);   // 16-bit draws (R7)
    out->q = 1.0f / (1.0f - dr->p);
    out->keep_bits = dr->keep_bits;
    out->masked_x = static_cast<__nv_bfloat16*>(dr->masked_x);
    if (dr->row_offset < 0 || dr->col_offset < 0 || dr->col_offset % 8 != 0 || dr->row_offset > 0xFFFFFFFFll ||
        dr->col_offset > 0x7FFFFFFF8ll)
        return fail(LORA_ERR_INVALID, "dropout row_offset = %lld / col_offset = %lld: need >= 0 and col_offset %% 8 == 0",
                    static_cast<long long>(dr->row_offset), static_cast<long long>(dr->col_offset));
    out->row0 = dr->row_offset;
    out->col0 = dr->col_offset;
    if (dr->keep_bits && !aligned16(dr->keep_bits))
        return fail(LORA_ERR_ALIGN, "dropout keep_bits = %p is not 16-byte aligned", static_cast<void*>(dr->keep_bits));
    if (dr->masked_x && !aligned16(dr->masked_x))
        return fail(LORA_ERR_ALIGN, "dropout masked_x = %p is not 16-byte aligned", dr->masked_x);
    return LORA_OK;
}

}  // namespace lora_host

// ============================================================ C ABI
using namespace lora_host;

extern "C" {

size_t lora_linear_fwd_workspace_bytes(const lora_dims* dims) { return fwd_workspace(dims); }
size_t lora_linear_bwd_workspace_bytes(const lora_dims* dims) { return bwd_workspace(dims); }

lora_status lora_linear_fwd(const lora_dims* dims, const void* x, const void* w0, const void* a, const void* b,
                            const void* bias, void* y, float* h_out, void* workspace, size_t workspace_bytes,
                            void* stream) {
    int launches = 0;
    lora_status st = fwd_impl(dims, x, w0, a, b, bias, y, h_out, workspace, workspace_bytes,
                              static_cast<cudaStream_t>(stream), &launches);
    set_launches(launches);
    return st;
}

lora_status lora_linear_bwd(const lora_dims* dims, const void* x, const void* w0, const void* a, const void* b,
                            const float* h_saved, const void* dy, void* dx, float* da, float* db, int accumulate,
                            void* workspace, size_t workspace_bytes, void* stream) {
    int launches = 0;
    if (accumulate != 0 && accumulate != 1) return fail(LORA_ERR_INVALID, "accumulate must be 0 or 1");
    lora_status st = bwd_impl(dims, x, w0, a, b, h_saved, dy, dx, da, db, accumulate ? kAccA | kAccB : 0,
                              workspace, workspace_bytes,
                              static_cast<cudaStream_t>(stream), &launches);
    prof_clear();
    set_launches(launches);
    return st;
}

size_t lora_linear_fwd_dropout_workspace_bytes(const lora_dims* dims) { return fwd_workspace_dropout(dims); }
size_t lora_linear_bwd_dropout_workspace_bytes(const lora_dims* dims) { return bwd_workspace_dropout(dims); }

lora_status lora_linear_fwd_dropout(const lora_dims* dims, const lora_dropout* dropout, const void* x, const void* w0,
                                    const void* a, const void* b, const void* bias, void* y, float* h_out,
                                    void* workspace, size_t workspace_bytes, void* stream) {
    int launches = 0;
    DropoutParams dp;
    lora_status st = dropout_params(dropout, &dp);
    if (st == LORA_OK)
        st = fwd_impl(dims, x, w0, a, b, bias, y, h_out, workspace, workspace_bytes, static_cast<cudaStream_t>(stream),
                      &launches, nullptr, &dp);
    set_launches(launches);
    return st;
}

lora_status lora_linear_bwd_dropout(const lora_dims* dims, const lora_dropout* dropout, const void* x, const void* w0,
                                    const void* a, const void* b, const float* h_saved, const void* dy, void* dx,
                                    float* da, float* db, int accumulate, void* workspace, size_t workspace_bytes,
                                    void* stream) {
    int launches = 0;
    ProfGuard pg;
    DropoutParams dp;
    lora_status st = dropout_params(dropout, &dp);
    if (st == LORA_OK && accumulate != 0 && accumulate != 1)
        st = fail(LORA_ERR_INVALID, "accumulate must be 0 or 1");
    if (st == LORA_OK)
        st = bwd_impl(dims, x, w0, a, b, h_saved, dy, dx, da, db, accumulate ? kAccA | kAccB : 0, workspace,
                      workspace_bytes,
                      static_cast<cudaStream_t>(stream), &launches, nullptr, 3, &dp);
    set_launches(launches);
    return st;
}

lora_status lora_dropout_mask(int64_t tokens, int64_t d_in, const lora_dropout* dropout, uint8_t* mask, void* stream) {
    int launches = 0;
    DropoutParams dp;
    lora_status st = dropout_params(dropout, &dp);
    if (st == LORA_OK && (tokens < 0 || d_in < 1)) st = fail(LORA_ERR_SHAPE, "mask shape %lld x %lld", (long long)tokens,
                                                             (long long)d_in);
    if (st == LORA_OK && tokens > 0 && !mask) st = fail(LORA_ERR_INVALID, "mask is NULL");
    DevInfo dev;
    if (st == LORA_OK) st = device_info(&dev);
    if (st == LORA_OK && tokens > 0) {
        cudaError_t e = launch_dropout_mask(tokens, d_in, dp, mask, dev.sms, static_cast<cudaStream_t>(stream));
        if (e != cudaSuccess) st = cuda_fail(e, "dropout mask launch");
        else ++launches;
    }
    set_launches(launches);
    return st;
}

lora_status lora_adam_step(int count, const lora_adam_tensor* tensors, const lora_adam_hparams* hp, int64_t step,
                           void* stream) {
    set_launches(0);
    if (count < 1 || count > LORA_ADAM_MAX_TENSORS || !tensors || !hp)
        return fail(LORA_ERR_INVALID, "lora_adam_step: need 1..%d tensors and hparams", LORA_ADAM_MAX_TENSORS);
    if (step < 1) return fail(LORA_ERR_INVALID, "lora_adam_step: step = %lld must be >= 1", (long long)step);
    if (!(hp->lr >= 0.0f) || !(hp->beta1 >= 0.0f && hp->beta1 < 1.0f) || !(hp->beta2 >= 0.0f && hp->beta2 < 1.0f) ||
        !(hp->eps >= 0.0f))
        return fail(LORA_ERR_INVALID, "lora_adam_step: lr >= 0, 0 <= beta < 1, eps >= 0 required");
    static thread_local AdamGroup G;
    G.count = count;
    for (int i = 0; i < count; ++i) {
        const lora_adam_tensor& t = tensors[i];
        if (t.numel < 0 || t.numel % 4 != 0)
            return fail(LORA_ERR_SHAPE, "lora_adam_step: tensor %d numel = %lld must be a multiple of 4", i,
                        (long long)t.numel);
        if (t.numel > 0 && (!t.param || !t.grad || !t.m || !t.v))
            return fail(LORA_ERR_INVALID, "lora_adam_step: tensor %d has a NULL param / grad / m / v", i);
        const void* ptrs[] = {t.param, t.master, t.grad, t.m, t.v};
        for (const void* q : ptrs)
            if (q && !aligned16(q)) return fail(LORA_ERR_ALIGN, "lora_adam_step: tensor %d pointer %p", i, q);
        G.t[i] = {static_cast<__nv_bfloat16*>(t.param), t.master, t.grad, t.m, t.v, t.numel};
    }
    G.lr = hp->lr;
    G.b1 = hp->beta1;
    G.b2 = hp->beta2;
    G.eps = hp->eps;
    G.bc1 = static_cast<float>(1.0 - std::pow(static_cast<double>(hp->beta1), static_cast<double>(step)));
    G.bc2 = static_cast<float>(1.0 - std::pow(static_cast<double>(hp->beta2), static_cast<double>(step)));
    DevInfo dev;
    lora_status st = device_info(&dev);
    if (st != LORA_OK) return st;
    cudaError_t e = launch_adam(G, dev.sms, static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail(e, "adam launch");
    set_launches(1);
    return LORA_OK;
}

lora_status lora_merge(const lora_dims* dims, const void* w0, const void* a, const void* b, void* w_out,
                       void* stream) {
    int launches = 0;
    lora_status st = merge_impl(dims, w0, a, b, w_out, static_cast<cudaStream_t>(stream), &launches);
    set_launches(launches);
    return st;
}

// ---------------------------------------------------------------- grouped
static size_t ws_align(size_t v) { return (v + 255) & ~size_t(255); }

static lora_status check_group(int count, const lora_dims* dims, const void* probs, const char* fn) {
    if (count < 1 || count > LORA_MAX_GROUP)
        return fail(LORA_ERR_INVALID, "%s: count = %d must be in [1, %d]", fn, count, LORA_MAX_GROUP);
    if (!dims || !probs) return fail(LORA_ERR_INVALID, "%s: dims / problems is NULL", fn);
    return LORA_OK;
}

static size_t fwd_grouped_ws(int count, const lora_dims* dims, bool dropout) {
    if (count < 1 || count > LORA_MAX_GROUP || !dims) return 0;
    size_t total = 0;
    for (int g = 0; g < count; ++g) {
        const size_t w = dropout ? fwd_workspace_dropout(&dims[g]) : fwd_workspace(&dims[g]);
        if (!w) return 0;
        total += ws_align(w);
    }
    return total;
}
static size_t bwd_grouped_ws(int count, const lora_dims* dims, bool dropout) {
    if (count < 1 || count > LORA_MAX_GROUP || !dims) return 0;
    size_t total = 0;
    for (int g = 0; g < count; ++g) {
        const size_t w = dropout ? bwd_workspace_dropout(&dims[g]) : bwd_workspace(&dims[g]);
        if (!w) return 0;
        total += ws_align(w);
    }
    return total;
}

size_t lora_linear_fwd_grouped_workspace_bytes(int count, const lora_dims* dims) {
    return fwd_grouped_ws(count, dims, false);
}
size_t lora_linear_bwd_grouped_workspace_bytes(int count, const lora_dims* dims) {
    return bwd_grouped_ws(count, dims, false);
}
size_t lora_linear_fwd_grouped_dropout_workspace_bytes(int count, const lora_dims* dims) {
    return fwd_grouped_ws(count, dims, true);
}
size_t lora_linear_bwd_grouped_dropout_workspace_bytes(int count, const lora_dims* dims) {
    return bwd_grouped_ws(count, dims, true);
}

// drops: per-problem dropout or NULL (no dropout)
static lora_status fwd_grouped_impl(int count, const lora_dims* dims, const DropoutParams* drops,
                                    const lora_fwd_problem* probs, void* workspace, size_t workspace_bytes,
                                    void* stream, const char* fn) {
    int launches = 0;
    lora_status st = check_group(count, dims, probs, fn);
    if (st != LORA_OK) return st;
    const size_t need = fwd_grouped_ws(count, dims, drops != nullptr);
    if (!need) return fail(LORA_ERR_SHAPE, "%s: invalid dims", fn);
    if (!workspace || workspace_bytes < need)
        return fail(LORA_ERR_WORKSPACE, "%s: workspace %zu < required %zu", fn, workspace_bytes, need);
    cudaStream_t st_ = static_cast<cudaStream_t>(stream);
    GemmCollector col;
    for (int pass = 0; pass < 2; ++pass) {   // pass 0: validation of every problem before anything is enqueued
        size_t off = 0;
        for (int g = 0; g < count; ++g) {
            const lora_fwd_problem& pr = probs[g];
            const size_t wg = ws_align(drops ? fwd_workspace_dropout(&dims[g]) : fwd_workspace(&dims[g]));
            st = fwd_impl(&dims[g], pr.x, pr.w0, pr.a, pr.b, pr.bias, pr.y, pr.h_out,
                          static_cast<uint8_t*>(workspace) + off, wg, st_, &launches, &col,
                          drops ? &drops[g] : nullptr, pass == 0);
            if (st != LORA_OK) { set_launches(pass ? launches : 0); return st; }
            off += wg;
        }
    }
    if ((st = launch_collected_k0(col, st_, &launches)) != LORA_OK) { set_launches(launches); return st; }
    st = launch_collected(kModeFwd, col, st_, &launches);
    set_launches(launches);
    return st;
}

lora_status lora_linear_fwd_grouped(int count, const lora_dims* dims, const lora_fwd_problem* probs,
                                    void* workspace, size_t workspace_bytes, void* stream) {
    return fwd_grouped_impl(count, dims, nullptr, probs, workspace, workspace_bytes, stream,
                            "lora_linear_fwd_grouped");
}

static lora_status group_dropouts(int count, const lora_dropout* dropouts, DropoutParams* dp, const char* fn) {
    if (!dropouts) return fail(LORA_ERR_INVALID, "%s: dropouts is NULL", fn);
    if (count < 1 || count > LORA_MAX_GROUP) return fail(LORA_ERR_INVALID, "%s: count = %d", fn, count);
    for (int g = 0; g < count; ++g) {
        lora_status st = dropout_params(&dropouts[g], &dp[g]);
        if (st != LORA_OK) return st;
        if ((dp[g].thr > 0) != (dp[0].thr > 0))
            return fail(LORA_ERR_UNSUPPORTED, "%s: problems %d and 0 disagree on p > 0 (one dX kernel mode per group)",
                        fn, g);
    }
    return LORA_OK;
}

lora_status lora_linear_fwd_grouped_dropout(int count, const lora_dims* dims, const lora_dropout* dropouts,
                                            const lora_fwd_problem* probs, void* workspace, size_t workspace_bytes,
                                            void* stream) {
    DropoutParams dp[LORA_MAX_GROUP];
    lora_status st = group_dropouts(count, dropouts, dp, "lora_linear_fwd_grouped_dropout");
    if (st != LORA_OK) return st;
    return fwd_grouped_impl(count, dims, dp, probs, workspace, workspace_bytes, stream,
                            "lora_linear_fwd_grouped_dropout");
}

lora_status lora_linear_bwd_grouped_dropout(int count, const lora_dims* dims, const lora_dropout* dropouts,
                                            const lora_bwd_problem* probs, int accumulate, void* workspace,
                                            size_t workspace_bytes, void* stream) {
    DropoutParams dp[LORA_MAX_GROUP];
    lora_status st = group_dropouts(count, dropouts, dp, "lora_linear_bwd_grouped_dropout");
    if (st == LORA_OK)
        st = lora_host::bwd_grouped_impl(count, dims, probs, accumulate, workspace, workspace_bytes, stream, nullptr,
                                         nullptr, nullptr, nullptr, dp);
    lora_host::prof_clear();
    return st;
}

lora_status lora_linear_bwd_grouped(int count, const lora_dims* dims, const lora_bwd_problem* probs, int accumulate,
                                    void* workspace, size_t workspace_bytes, void* stream) {
    const lora_status st = lora_host::bwd_grouped_impl(count, dims, probs, accumulate, workspace, workspace_bytes,
                                                       stream, nullptr, nullptr);
    lora_host::prof_clear();
    return st;
}

}  // extern "C"

namespace lora_host {

lora_status bwd_grouped_impl(int count, const lora_dims* dims, const lora_bwd_problem* probs, int accumulate,
                             void* workspace, size_t workspace_bytes, void* stream,
                             lora_status (*after_k2)(void* ctx, int* launches), void* ctx,
                             lora_status (*before_k2)(void* bctx, GemmCollector* col, int* launches), void* bctx,
                             const DropoutParams* drops) {
    int launches = 0;
    lora_status st = check_group(count, dims, probs, "lora_linear_bwd_grouped");
    if (st != LORA_OK) return st;
    const size_t need = bwd_grouped_ws(count, dims, drops != nullptr);
    if (!need) return fail(LORA_ERR_SHAPE, "lora_linear_bwd_grouped: invalid dims");
    if (!workspace || workspace_bytes < need)
        return fail(LORA_ERR_WORKSPACE, "lora_linear_bwd_grouped: workspace %zu < required %zu", workspace_bytes,
                    need);
    if (accumulate != 0 && accumulate != 1) return fail(LORA_ERR_INVALID, "accumulate must be 0 or 1");
    const int acc = accumulate ? kAccA | kAccB : 0;
    cudaStream_t st_ = static_cast<cudaStream_t>(stream);
    GemmCollector col;
    // validation of EVERY problem before anything is enqueued (include/lora.h)
    {
        size_t off = 0;
        for (int g = 0; g < count; ++g) {
            const lora_bwd_problem& pr = probs[g];
            const size_t wg = ws_align(drops ? bwd_workspace_dropout(&dims[g]) : bwd_workspace(&dims[g]));
            st = bwd_impl(&dims[g], pr.x, pr.w0, pr.a, pr.b, pr.h_saved, pr.dy, pr.dx, pr.da, pr.db, acc,
                          static_cast<uint8_t*>(workspace) + off, wg, st_, &launches, &col, kStageValidate,
                          drops ? &drops[g] : nullptr);
            if (st != LORA_OK) { set_launches(0); return st; }
            off += wg;
        }
    }
    for (int stage = 1; stage <= 2; ++stage) {
        size_t off = 0;
        for (int g = 0; g < count; ++g) {
            const lora_bwd_problem& pr = probs[g];
            const size_t wg = ws_align(drops ? bwd_workspace_dropout(&dims[g]) : bwd_workspace(&dims[g]));
            st = bwd_impl(&dims[g], pr.x, pr.w0, pr.a, pr.b, pr.h_saved, pr.dy, pr.dx, pr.da, pr.db, acc,
                          static_cast<uint8_t*>(workspace) + off, wg, st_, &launches, &col, stage,
                          drops ? &drops[g] : nullptr);
            if (st != LORA_OK) { set_launches(launches); return st; }
            off += wg;
        }
        if (stage == 1 && before_k2 && (st = before_k2(bctx, &col, &launches)) != LORA_OK) {
            set_launches(launches);
            return st;
        }
        if (stage == 1) {
            if ((st = launch_collected_k0(col, st_, &launches)) != LORA_OK) {
                set_launches(launches);
                return st;
            }
            prof_record(0, st_);
            st = launch_collected(drops && drops[0].thr > 0 ? kModeDxDrop : kModeDx, col, st_, &launches);
            prof_record(1, st_);
            if (st != LORA_OK) {
                set_launches(launches);
                return st;
            }
        }
        // work that needs only the dX kernel's outputs (the TP column group forks its dX
        // sum and all-reduce here, so they overlap the dA / dB kernel below)
        if (stage == 1 && after_k2 && (st = after_k2(ctx, &launches)) != LORA_OK) {
            set_launches(launches);
            return st;
        }
    }
    st = launch_collected_k3(col, st_, &launches);
    set_launches(launches);
    return st;
}

}  // namespace lora_host

extern "C" {

const char* lora_status_string(lora_status s) {
    switch (s) {
        case LORA_OK: return "LORA_OK";
        case LORA_ERR_INVALID: return "LORA_ERR_INVALID";
        case LORA_ERR_SHAPE: return "LORA_ERR_SHAPE";
        case LORA_ERR_ALIGN: return "LORA_ERR_ALIGN";
        case LORA_ERR_UNSUPPORTED: return "LORA_ERR_UNSUPPORTED";
        case LORA_ERR_CUDA: return "LORA_ERR_CUDA";
        case LORA_ERR_NCCL: return "LORA_ERR_NCCL";
        case LORA_ERR_WORKSPACE: return "LORA_ERR_WORKSPACE";
    }
    return "LORA_ERR_UNKNOWN";
}

const char* lora_last_error(void) { return g_last_error.c_str(); }

int lora_version(void) { return 100; }

lora_status lora_device_check(void) {
    DevInfo d;
    return device_info(&d);
}

int lora_last_launch_count(void) { return get_launches(); }

lora_status lora_profile_next_bwd(void* const events[4]) {
    for (int i = 0; i < 4; ++i) g_prof_events[i] = events ? events[i] : nullptr;
    return LORA_OK;
}

int lora_captured_sync_words_free(void) {
    int dev = -1;
    if (cudaGetDevice(&dev) != cudaSuccess) return -1;
    return sync_pool_captured_free_words(dev);
}

}  // extern "C"
