// lora_internal.h -- shared host-side helpers of liblora.so (not public ABI).
#pragma once
#include <cuda_runtime.h>

#include "lora.h"
#include "lora_kernels.h"

namespace lora_host {

lora_status fail(lora_status st, const char* fmt, ...);
lora_status cuda_fail(cudaError_t e, const char* what);
lora_status check_dims(const lora_dims* d, bool need_tokens);
void set_launches(int n);
void prof_record(int i, cudaStream_t stream);   // lora_profile_next_bwd events
void prof_clear();
struct ProfGuard {   // one-shot lora_profile_next_bwd events end with the public call
    ~ProfGuard() { prof_clear(); }
};
int get_launches();

// lora_linear_bwd_grouped with a hook run right after the grouped dX kernel is
// enqueued (before the dA / dB kernel): after_k2(ctx, &launches) may enqueue
// work that depends only on the members' dX (the TP column group's dX sum and
// all-reduce, on a side stream).
// before_k2(bctx, &col, &launches) runs right before the grouped dX kernel is
// launched: it may edit the collected K2 parameters (the comm-fused epilogue sets
// unit flags) and enqueue work that must precede K2 (the fused reducer's fork).
struct GemmCollector;
lora_status bwd_grouped_impl(int count, const lora_dims* dims, const lora_bwd_problem* probs, int accumulate,
                             void* workspace, size_t workspace_bytes, void* stream,
                             lora_status (*after_k2)(void* ctx, int* launches), void* ctx,
                             lora_status (*before_k2)(void* bctx, GemmCollector* col, int* launches) = nullptr,
                             void* bctx = nullptr, const lora_sm100::DropoutParams* drops = nullptr);
int r_pad_of(int r);
lora_status merge_impl(const lora_dims* d, const void* w0, const void* a, const void* b, void* w_out,
                       cudaStream_t stream, int* launches);
// load the kernels launched next to spinning kernels (reducer, NCCL) -- lora_symm.cu
lora_status preload_kernels();

// Fused-GEMM problems gathered by the grouped entry points (launched together).
struct GemmCollector {
    int count = 0;
    lora_sm100::FusedGemmMaps maps[lora_sm100::kMaxGroup];
    lora_sm100::FusedGemmParams p[lora_sm100::kMaxGroup];
    int rp[lora_sm100::kMaxGroup];
    int cg[lora_sm100::kMaxGroup];
    bool no_coop = false;   // launch the fused GEMMs non-cooperatively (comm-fused path)
    // LoRA dropout: the K0 work of the collected problems, launched right before the
    // fused GEMMs (launch_collected_k0)
    lora_sm100::DropoutGroup k0{};
    int max_sms = 0;        // > 0: the fused GEMMs use at most this many SMs (comm-fused path, virtual ranks)
    // K3 (dA, dB) problems of the grouped backward, launched together at the end
    int k3_count = 0;
    lora_sm100::GradArgs k3[lora_sm100::kMaxGroup];
};

// col != nullptr: the fused GEMM is appended to `col` instead of launched.
// bwd stages: bit 0 = validation, pack, K2 (launch or collect);
//             bit 1 = everything after K2 (gh pre-pass, h recompute, K3).
lora_status fwd_impl(const lora_dims* d, const void* x, const void* w0, const void* a, const void* b,
                     const void* bias, void* y, float* h_out, void* ws, size_t ws_bytes,
                     cudaStream_t stream, int* launches, GemmCollector* col = nullptr,
                     const lora_sm100::DropoutParams* drop = nullptr, bool validate_only = false);
// bwd stage bit 2: validate the arguments only (the grouped calls check every
// problem before enqueueing anything); accumulate is a lora_sm100::kAccA | kAccB mask
constexpr int kStageValidate = 4;
lora_status bwd_impl(const lora_dims* d, const void* x, const void* w0, const void* a, const void* b,
                     const float* h_saved, const void* dy, void* dx, float* da, float* db, int accumulate,
                     void* ws, size_t ws_bytes, cudaStream_t stream, int* launches,
                     GemmCollector* col = nullptr, int stages = 3,
                     const lora_sm100::DropoutParams* drop = nullptr);
size_t fwd_workspace_dropout(const lora_dims* d);
// lora_dropout -> kernel parameters (validates p, alignment of the kept buffers, offsets)
lora_status dropout_params(const lora_dropout* dr, lora_sm100::DropoutParams* out);
size_t bwd_workspace_dropout(const lora_dims* d);
// launch the collected problems, one grouped launch per (r_pad, CTA group) class
lora_status launch_collected(int mode, GemmCollector& col, cudaStream_t stream, int* launches);
// launch the collected K0 work (if any)
lora_status launch_collected_k0(GemmCollector& col, cudaStream_t stream, int* launches);
// launch the collected K3 problems, one launch per rank bucket
lora_status launch_collected_k3(GemmCollector& col, cudaStream_t stream, int* launches);
size_t fwd_workspace(const lora_dims* d);
size_t bwd_workspace(const lora_dims* d);

}  // namespace lora_host
