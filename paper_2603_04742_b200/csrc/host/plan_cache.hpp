// plan_cache.hpp -- per-context cache of cloud plans keyed by chunk shapes.
//
// A cloud plan (cloud_plan.hpp) depends only on the chunk shapes the cloud
// receives as ChunkShapeMeta (protocol.cpp:113-116): every chunk's (h, k) and
// the slice it belongs to.  Repeated evaluations over matrices with the same
// sparsity structure reuse the plan, its ciphertext buffers and, from the
// second use on, its captured CUDA graph.  Encryption still runs every call:
// only the launch sequence and the buffers are reused, never a result.
// Internal to the library (the C-ABI is unchanged); implemented in capi.cpp.
#pragma once

#include <cstdint>
#include <vector>

#include "spmvgpu.h"

namespace spmv::detail {

struct PlanLease {
    std::vector<std::uint64_t> key;
    std::vector<spmvgpu_ct> a, b, out;
    spmvgpu_plan* plan = nullptr;
    bool captured = false;
    std::uint64_t uses = 0;
    // whole-evaluation pipeline (CloudPlan::capture_pipeline): pinned image and
    // result buffers at fixed addresses, and the image layout it was captured for
    unsigned char* pimg = nullptr;
    std::size_t pimg_cap = 0;
    unsigned char* pout = nullptr;
    std::size_t pout_cap = 0;
    std::vector<std::size_t> pkey;
};

// Moves a cached lease for `key` into `out` and returns true, or returns false.
bool plan_cache_take(spmvgpu_ctx* ctx, const std::vector<std::uint64_t>& key, PlanLease& out);
// Hands a lease back (the cache owns it from now on and may evict it).
void plan_cache_give(spmvgpu_ctx* ctx, PlanLease&& lease);
// Frees a lease's plan and ciphertexts.
void plan_lease_free(spmvgpu_ctx* ctx, PlanLease& lease);

// Client upload image in pinned host memory, laid out like spmvgpu_encrypt_cssc's
// arrays (BatchedSpmv writes it directly; the descriptors are correct by
// construction, so this internal path skips the C-ABI's validation).
struct ClientImage {
    unsigned char* p = nullptr;
    std::size_t cap = 0;
    std::size_t o_ci = 0, o_va = 0, o_v = 0, o_rows = 0, o_rpre = 0, o_sl = 0, o_cols = 0, o_st = 0, o_out = 0,
                bytes = 0;
    std::size_t nnz = 0, vec_len = 0, n_rows = 0, n_slices = 0, n_cols = 0;
    int items = 0;
    int ci_w = 8, va_w = 8, v_w = 8;  // element widths (cssc::CsscLayout)
};
ClientImage client_image_layout(std::size_t nnz, std::size_t vec_len, std::size_t n_rows, std::size_t n_slices,
                                std::size_t n_cols, int items, int ci_w = 8, int va_w = 8,
                                int v_w = 8);  // offsets only, p = nullptr
ClientImage client_image_take(spmvgpu_ctx* ctx, std::size_t nnz, std::size_t vec_len, std::size_t n_rows,
                              std::size_t n_slices, std::size_t n_cols, int items, int ci_w = 8, int va_w = 8,
                              int v_w = 8);
void client_image_give(spmvgpu_ctx* ctx, ClientImage& img);
// fills the stream ids and output handles, uploads, packs and encrypts
void client_image_encrypt(spmvgpu_ctx* ctx, ClientImage& img, const spmvgpu_ct* out);
// writes fresh stream ids and the output handles into an image at `p` laid out as `img`
void client_image_fill(spmvgpu_ctx* ctx, unsigned char* p, const ClientImage& img, const spmvgpu_ct* out);
// the image layout a pipeline depends on
std::vector<std::size_t> client_image_key(const ClientImage& img);
// (re)captures the lease's whole-evaluation graph for images laid out as `img`
// (allocates the lease's pinned image/result buffers); then runs it and waits
void pipeline_prepare(spmvgpu_ctx* ctx, PlanLease& lease, const ClientImage& img);
// at the start of a batch call: enqueue the early encryption graph of the
// last pipeline run's plan with the stream ids the call will assign next, so
// it overlaps the host's packing; pipeline_run skips it if the call uses that
// plan and those ids, and runs it otherwise
void pipeline_speculate(spmvgpu_ctx* ctx);
void pipeline_run(spmvgpu_ctx* ctx, PlanLease& lease);
bool pipeline_ready(const PlanLease& lease, const ClientImage& img);
// after pipeline_run: result r's decrypted slots [0, rows) as u32 (slots past
// rows are zero) and its rounding deviation
struct PipelineResult {
    const std::uint32_t* slots;
    int rows;
    unsigned long long maxdev;
};
PipelineResult pipeline_result(const PlanLease& lease, int r);
std::size_t pipeline_out_bytes(const PlanLease& lease);  // bytes one pipeline run downloads

}  // namespace spmv::detail
