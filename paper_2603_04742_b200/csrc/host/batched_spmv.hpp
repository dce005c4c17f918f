// batched_spmv.hpp -- the GPU evaluation of spmv_partitioned over one or more
// matrices: every slice's pack (Client A/B, host), one batched encryption,
// one cloud plan over all chunks (device), one batched decryption, then the
// reference's per-slice bookkeeping (ledger, transcript, model noise) so each
// matrix's SpmvResult equals its own reference run (protocol.cpp:74-176).
#pragma once

#include <cstdint>
#include <span>
#include <vector>

#include "host/plan_cache.hpp"
#include "spmv/protocol.hpp"
#include "spmvgpu.h"

namespace spmv::detail {

class BatchedSpmv {
public:
    BatchedSpmv(spmvgpu_ctx* ctx, const HeParams& hp, std::span<const CsrMatrix> ms,
                std::span<const std::vector<std::int64_t>> vs, std::size_t chunk_size,
                PartyRole key_holder, bool partition = true);
    ~BatchedSpmv();
    BatchedSpmv(const BatchedSpmv&) = delete;
    BatchedSpmv& operator=(const BatchedSpmv&) = delete;

    void encrypt();               // Client A + Client B: one batched encrypt
    void cloud(bool use_graph);   // enqueue the cloud plan (no host sync)
    std::vector<SpmvResult> finish();  // key holder: decrypt, unpermute, bookkeeping

    spmvgpu_plan* plan() const { return lease_.plan; }
    std::uint64_t h2d_bytes() const { return h2d_; }
    std::uint64_t d2h_bytes() const { return d2h_; }
    std::size_t total_chunks() const { return r_.size(); }

private:
    struct Slice {
        std::size_t mat = 0;
        std::size_t rows = 0;
        ChunkSet cs;
        std::size_t first_chunk = 0;  // global chunk index
        int result = -1;              // result ciphertext index, -1 when no chunks
    };
    void ensure_plan();

    spmvgpu_ctx* ctx_;
    HeParams hp_;
    PartyRole kh_;
    std::size_t nmat_;
    std::vector<std::size_t> rows_of_;
    std::vector<Slice> slices_;
    std::vector<std::int64_t> vals_;   // A flats then B segments
    std::vector<std::uint64_t> offs_;
    std::vector<std::uint64_t> r_, c_;
    std::vector<std::uint32_t> slice_id_;
    std::size_t n_out_ = 0;
    PlanLease lease_;
    bool done_ = false;  // plan + ciphertext buffers, from / back to the context's plan cache
    std::uint64_t h2d_ = 0, d2h_ = 0;
};

}  // namespace spmv::detail
