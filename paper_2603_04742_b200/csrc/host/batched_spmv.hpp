// batched_spmv.hpp -- the GPU evaluation of spmv_partitioned over one or more
// matrices: the CSSC shapes of every slice on the host (row-length counting
// sort and chunk boundaries only), Client A + B's packing and encryption in
// one device pass (spmvgpu_encrypt_cssc), one cloud plan over all chunks, one
// batched decryption, then the reference's per-slice bookkeeping (ledger,
// transcript, model noise) so each matrix's SpmvResult equals its own
// reference run (protocol.cpp:74-176).
#pragma once

#include <cstdint>
#include <memory>
#include <utility>
#include <exception>
#include <span>
#include <vector>

#include "host/plan_cache.hpp"
#include "spmv/protocol.hpp"
#include "spmvgpu.h"

namespace spmv::detail {

// Borrowed CSR arrays (a CsrMatrix or a C-ABI cssc_csr); read only while the
// BatchedSpmv is constructed.
struct CsrView {
    std::size_t rows = 0, cols = 0, nnz = 0;
    const std::uint64_t* row_ptrs = nullptr;     // rows + 1
    const std::uint64_t* col_indices = nullptr;  // nnz
    const std::int64_t* values = nullptr;        // nnz
    const std::int64_t* vec = nullptr;           // cols
};
CsrView view_of(const CsrMatrix& m, std::span<const std::int64_t> v);

class BatchedSpmv {
public:
    // rank/world: evaluate only the chunks g with g % world == rank (SURVEY 8(e):
    // chunks split across GPUs); the per-slice partial results are summed
    // across ranks from result_words() and decrypted with finish_words()
    BatchedSpmv(spmvgpu_ctx* ctx, const HeParams& hp, std::span<const CsrView> ms, std::size_t chunk_size,
                PartyRole key_holder, bool partition = true, int rank = 0, int world = 1);
    ~BatchedSpmv();
    BatchedSpmv(const BatchedSpmv&) = delete;
    BatchedSpmv& operator=(const BatchedSpmv&) = delete;

    void encrypt();               // Client A + Client B: pack + encrypt on the device
    void cloud(bool use_graph);   // enqueue the cloud plan (no host sync)
    std::vector<SpmvResult> finish();  // key holder: decrypt, unpermute, bookkeeping
    // encrypt + cloud + finish; from a plan's second use on, one graph launch
    // out_values (optional, one caller buffer of rows_i entries per matrix):
    // the decrypted rows are written there directly and the results' `values`
    // stay empty (the C-ABI batch path; saves a copy of every row)
    std::vector<SpmvResult> run_all(std::int64_t* const* out_values = nullptr);
    // this rank's per-slice result ciphertext words (zeros for slices it holds
    // no chunk of), [results][ct words]; and the decryption of summed words
    std::vector<std::uint64_t> result_words();
    std::vector<SpmvResult> finish_words(const std::uint64_t* words);
    // the same with the words in device memory (the ranks' buffers summed by an
    // NCCL all-reduce): result_words_dev copies this rank's partial results
    // into `dev` (zeros for slices it holds none of) and waits; finish_words_dev
    // folds `dev` mod q_j in place on the device, then decrypts
    void result_words_dev(std::uint64_t* dev);
    std::vector<SpmvResult> finish_words_dev(std::uint64_t* dev);
    std::size_t result_count() const { return n_out_; }

    spmvgpu_plan* plan() const { return lease_.plan; }
    std::uint64_t h2d_bytes() const { return h2d_; }
    std::uint64_t d2h_bytes() const { return d2h_; }
    std::size_t total_chunks() const { return r_.size(); }
    std::size_t local_chunks() const { return dr_.size(); }

private:
    struct Slice {
        std::size_t mat = 0;
        std::size_t rows = 0;
        std::vector<std::size_t> row_map;  // CSSC row order (rm, sparse.cpp:79-117)
        std::size_t first_chunk = 0;       // global chunk index
        std::size_t n_ct = 0;
        int result = -1;                   // result ciphertext index, -1 when no chunks
    };
    struct SliceJob {  // rows [r0, r1) of matrix `mat`
        std::size_t mat = 0, r0 = 0, r1 = 0;
        std::int64_t nz_base = 0, vec_base = 0;
    };
    struct SliceShape {  // one slice's CSSC shapes, chunk indices and slice id local
        std::size_t mat = 0, rows = 0;
        std::int32_t vec_base = 0;
        std::vector<std::size_t> row_map;
        std::vector<std::int32_t> rowrec, colrec;
        std::vector<std::uint64_t> r, c;
        std::exception_ptr err;
    };
    void shape_slice(const CsrView& m, const SliceJob& job, std::size_t budget, SliceShape& out) const;
    // slice metadata (takes the shape's row map), chunk shapes and slice
    // record; the row / column records are placed into the image by the
    // caller (col_base = the slice's first column record)
    void append_slice(SliceShape& s, std::size_t col_base);
    void ensure_plan();
    std::vector<SpmvResult> decrypt_and_report(const std::vector<spmvgpu_ct>& outs);
    // one result's decrypted slots: u64 (decrypt) or u32 (pipeline download);
    // slots at and past `count` are zero
    struct SlotSource {
        const std::uint64_t* u64 = nullptr;
        const std::uint32_t* u32 = nullptr;
        std::size_t count = 0;
    };
    std::vector<SpmvResult> report(const std::vector<SlotSource>& slots, const std::vector<std::int32_t>& measured,
                                   std::int64_t* const* out_values = nullptr);

    spmvgpu_ctx* ctx_;
    HeParams hp_;
    PartyRole kh_;
    std::size_t nmat_;
    std::vector<std::size_t> rows_of_;
    std::vector<Slice> slices_;
    // slice records {first column record, vector base} (the image's slice table)
    std::vector<std::int32_t> slicerec_;
    ClientImage img_;
    bool img_borrowed_ = false;  // img_.p is the cached pipeline's pinned buffer
    bool encrypted_ = false;
    std::vector<std::uint64_t> r_, c_;
    std::vector<std::uint32_t> slice_id_;
    std::size_t n_out_ = 0;
    // this rank's share: local chunk shapes, local result ids, global -> local result
    int rank_ = 0, world_ = 1;
    std::vector<std::uint64_t> dr_, dc_;
    std::vector<std::uint32_t> dslice_;
    std::vector<int> res_local_;
    std::size_t n_dout_ = 0;
    PlanLease lease_;  // plan + ciphertext buffers, from / back to the context's plan cache
    bool done_ = false;
    std::uint64_t h2d_ = 0, d2h_ = 0;
};

}  // namespace spmv::detail
