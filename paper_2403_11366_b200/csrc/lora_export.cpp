// lora_export.cpp -- merged-weight export in the Hugging Face safetensors format
// (Listing 4 "huggingface_merger.py
// HUGGINGFACE_PATH JAX_PATH SAVE_PATH": the fine-tuned LoRA factors are folded
// into the base weights, W' = W0 + s B A (Eq. 1 line 2), and the
// model is saved where Hugging Face-compatible libraries can load it).
//
// lora_export_merged: every entry with adapters is merged on the GPU by the
// tensor-core K4 (lora_merge), copied to pinned host memory and streamed into
// the file; entries without adapters are written as they are.  The file layout
// is safetensors: u64 little-endian header length, a JSON header
// {name: {"dtype", "shape", "data_offsets": [begin, end)}, "__metadata__": ...}
// padded with spaces to a multiple of 8 bytes, then the raw tensor bytes in
// header order.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "lora_internal.h"

using namespace lora_host;

namespace {

const char* dtype_name(int dt) {
    switch (dt) {
        case LORA_DT_F32: return "F32";
        case LORA_DT_BF16: return "BF16";
    }
    return nullptr;
}
size_t dtype_size(int dt) { return dt == LORA_DT_F32 ? 4 : 2; }

std::string json_escape(const char* s) {
    std::string o;
    for (; *s; ++s) {
        const unsigned char c = static_cast<unsigned char>(*s);
        if (c == '"' || c == '\\') { o += '\\'; o += static_cast<char>(c); }
        else if (c < 0x20) { char b[8]; snprintf(b, sizeof b, "\\u%04x", c); o += b; }
        else o += static_cast<char>(c);
    }
    return o;
}

struct Entry {
    std::string name;
    int dtype;
    int ndim;
    int64_t shape[4];
    size_t bytes;
};

// header JSON for `entries` (in order), padded with spaces to a multiple of 8
lora_status build_header(const std::vector<Entry>& entries, std::string* out) {
    std::string h = "{\"__metadata__\":{\"format\":\"pt\",\"producer\":\"liblora lora_export_merged\"}";
    size_t off = 0;
    for (const Entry& e : entries) {
        h += ",\"" + json_escape(e.name.c_str()) + "\":{\"dtype\":\"" + dtype_name(e.dtype) + "\",\"shape\":[";
        for (int d = 0; d < e.ndim; ++d) h += (d ? "," : "") + std::to_string(e.shape[d]);
        h += "],\"data_offsets\":[" + std::to_string(off) + "," + std::to_string(off + e.bytes) + "]}";
        off += e.bytes;
    }
    h += "}";
    while (h.size() % 8) h += ' ';
    *out = h;
    return LORA_OK;
}

lora_status check_entry(const char* name, int dtype, int ndim, const int64_t* shape, const char* fn, Entry* e) {
    if (!name || !*name) return fail(LORA_ERR_INVALID, "%s: tensor name is empty", fn);
    if (!dtype_name(dtype)) return fail(LORA_ERR_INVALID, "%s: %s: dtype %d (LORA_DT_F32 / LORA_DT_BF16)", fn, name, dtype);
    if (ndim < 1 || ndim > 4) return fail(LORA_ERR_SHAPE, "%s: %s: ndim %d (1..4)", fn, name, ndim);
    e->name = name;
    e->dtype = dtype;
    e->ndim = ndim;
    size_t n = 1;
    for (int d = 0; d < ndim; ++d) {
        if (shape[d] < 0) return fail(LORA_ERR_SHAPE, "%s: %s: negative extent", fn, name);
        e->shape[d] = shape[d];
        n *= static_cast<size_t>(shape[d]);
    }
    e->bytes = n * dtype_size(dtype);
    return LORA_OK;
}

struct File {
    FILE* f = nullptr;
    ~File() { if (f) fclose(f); }
};

lora_status write_all(FILE* f, const void* p, size_t n, const char* path) {
    if (n && fwrite(p, 1, n, f) != n) return fail(LORA_ERR_INVALID, "write to %s failed", path);
    return LORA_OK;
}

}  // namespace

extern "C" {

lora_status lora_write_safetensors(const char* path, int count, const lora_host_tensor* tensors) {
    static const char* fn = "lora_write_safetensors";
    if (!path || count < 0 || (count && !tensors)) return fail(LORA_ERR_INVALID, "%s: NULL argument", fn);
    std::vector<Entry> es(count);
    for (int i = 0; i < count; ++i) {
        lora_status st = check_entry(tensors[i].name, tensors[i].dtype, tensors[i].ndim, tensors[i].shape, fn, &es[i]);
        if (st != LORA_OK) return st;
        if (es[i].bytes && !tensors[i].data) return fail(LORA_ERR_INVALID, "%s: %s: data is NULL", fn, tensors[i].name);
    }
    std::string h;
    build_header(es, &h);
    File F;
    if (!(F.f = fopen(path, "wb"))) return fail(LORA_ERR_INVALID, "%s: cannot open %s for writing", fn, path);
    const uint64_t hl = h.size();
    uint8_t le[8];
    for (int b = 0; b < 8; ++b) le[b] = static_cast<uint8_t>(hl >> (8 * b));
    lora_status st = write_all(F.f, le, 8, path);
    if (st == LORA_OK) st = write_all(F.f, h.data(), h.size(), path);
    for (int i = 0; i < count && st == LORA_OK; ++i) st = write_all(F.f, tensors[i].data, es[i].bytes, path);
    return st;
}

lora_status lora_export_merged(const char* path, int count, const lora_export_tensor* tensors, void* stream) {
    static const char* fn = "lora_export_merged";
    if (!path || count < 0 || (count && !tensors)) return fail(LORA_ERR_INVALID, "%s: NULL argument", fn);
    std::vector<Entry> es(count);
    size_t stage = 0;
    for (int i = 0; i < count; ++i) {
        const lora_export_tensor& t = tensors[i];
        const bool merge = t.a || t.b;
        if (merge) {
            if (!t.a || !t.b || !t.w0) return fail(LORA_ERR_INVALID, "%s: %s: a merged entry needs w0, a and b", fn,
                                                   t.name ? t.name : "?");
            const int64_t shape[2] = {t.dims.d_out, t.dims.d_in};
            lora_status st = check_entry(t.name, LORA_DT_BF16, 2, shape, fn, &es[i]);
            if (st != LORA_OK) return st;
            if ((st = check_dims(&t.dims, false)) != LORA_OK) return st;
        } else {
            lora_status st = check_entry(t.name, t.dtype, t.ndim, t.shape, fn, &es[i]);
            if (st != LORA_OK) return st;
            if (es[i].bytes && !t.w0) return fail(LORA_ERR_INVALID, "%s: %s: w0 (the tensor) is NULL", fn, t.name);
        }
        stage = es[i].bytes > stage ? es[i].bytes : stage;
    }
    cudaStream_t st_ = static_cast<cudaStream_t>(stream);
    void* dbuf = nullptr;
    void* hbuf = nullptr;
    cudaError_t e = cudaSuccess;
    if (stage) {
        if ((e = cudaMalloc(&dbuf, stage)) != cudaSuccess) return cuda_fail(e, "lora_export_merged: staging buffer");
        if ((e = cudaMallocHost(&hbuf, stage)) != cudaSuccess) {
            cudaFree(dbuf);
            return cuda_fail(e, "lora_export_merged: pinned host buffer");
        }
    }
    struct Free {
        void *d, *h;
        ~Free() { if (d) cudaFree(d); if (h) cudaFreeHost(h); }
    } fr{dbuf, hbuf};
    std::string h;
    build_header(es, &h);
    File F;
    if (!(F.f = fopen(path, "wb"))) return fail(LORA_ERR_INVALID, "%s: cannot open %s for writing", fn, path);
    const uint64_t hl = h.size();
    uint8_t le[8];
    for (int b = 0; b < 8; ++b) le[b] = static_cast<uint8_t>(hl >> (8 * b));
    lora_status st = write_all(F.f, le, 8, path);
    if (st == LORA_OK) st = write_all(F.f, h.data(), h.size(), path);
    for (int i = 0; i < count && st == LORA_OK; ++i) {
        const lora_export_tensor& t = tensors[i];
        if (!es[i].bytes) continue;
        const void* src = t.w0;
        if (t.a) {   // W' = bf16(W0 + s B A) on the tensor cores, into the staging buffer
            int launches = 0;
            if ((st = merge_impl(&t.dims, t.w0, t.a, t.b, dbuf, st_, &launches)) != LORA_OK) break;
            src = dbuf;
        }
        if ((e = cudaMemcpyAsync(hbuf, src, es[i].bytes, cudaMemcpyDeviceToHost, st_)) != cudaSuccess ||
            (e = cudaStreamSynchronize(st_)) != cudaSuccess) {
            st = cuda_fail(e, "lora_export_merged: copy to host");
            break;
        }
        st = write_all(F.f, hbuf, es[i].bytes, path);
    }
    return st;
}

}  // extern "C"
