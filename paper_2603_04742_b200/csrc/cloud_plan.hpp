// cloud_plan.hpp -- the batched cloud phase of the encrypted CSSC SpMV.
//
// Lowers the reference's per-chunk loop (protocol.cpp:121-140:
// multiply -> intra_chunk_sum -> inter_chunk_sum) over every chunk of every
// slice (and every matrix of a batch) into a fixed launch sequence:
//   1. one batched ct x ct multiply + relinearisation over all chunks;
//   2. level l = 0..depth-1 of the rotate-and-add trees (rotation_schedule,
//      aggregate.cpp:19-34): every chunk with more than l doubling steps does
//      acc <- acc + rot(acc, offset) [+ a hoisted odd-step rotation of the
//      product] in one fused key-switch launch group; level 0 also rotates the
//      products for all odd steps (they never depend on the accumulator), so
//      the depth is numBits(c) - 1 instead of numBits(c) + popcount(c) - 2
//      (chunks are ordered by descending depth: level l is an item prefix);
//   3. one masked, segmented accumulation of all folded chunks into one
//      result ciphertext per slice (inter_chunk_sum, aggregate.cpp:55-74).
// The sequence is fixed at plan time and can be captured as a CUDA graph.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <vector>

#include "bfv_context.hpp"

namespace cssc {

struct PlanStats {
    uint64_t chunks = 0, slices = 0, levels = 0, kernels = 0, limb_ntts = 0;
    uint64_t rotations = 0, distinct_keys = 0;
    uint64_t hbm_bytes = 0, key_bytes = 0;
    uint64_t relin_folded = 0;  // 1: rotated chunks' relinearisation folded into level 0
};

// one launch group of the plan, timed by profile()
struct PhaseTiming {
    std::string name;
    double us = 0;
    uint64_t items = 0, bytes = 0, limb_ntts = 0;  // compulsory HBM bytes, limb NTTs
    uint64_t sources = 0;    // distinct key-switch sources (hoisted level 0: the products)
    uint64_t acc_items = 0;  // key switches accumulated (odd steps fold into their doubling step's ModDown)
    uint64_t mac_terms = 0;  // key products summed (folded level 0: relin + z1 and z2 rotations)
};

// one kernel launch of the plan, timed by profile_kernels()
struct KernelTiming {
    std::string name;
    int group = 0;  // index into profile()'s launch groups
    double us = 0;  // mean over the replays
};

class CloudPlan {
public:
    // a/b: per-chunk input ciphertexts; out: one result ciphertext per slice
    CloudPlan(GpuContext& ctx, const std::vector<uint64_t>& r, const std::vector<uint64_t>& c,
              const std::vector<uint32_t>& slice, int n_slices, const std::vector<const u64*>& a,
              const std::vector<const u64*>& b, const std::vector<u64*>& out);
    ~CloudPlan();
    void run();      // enqueue (graph replay when captured)
    void capture();  // record a CUDA graph of run()
    // one graph replay with event nodes between launch groups (multiply+relin,
    // each rotate level, the level-0 add, the mask accumulation)
    std::vector<PhaseTiming> profile();
    // `reps` graph replays with an event node after every kernel launch; L2 is
    // flushed (a `flush_bytes` device memset) before each replay
    std::vector<KernelTiming> profile_kernels(int reps, size_t flush_bytes);
    // The whole evaluation as one graph: upload of the client image `img`
    // (pinned, fixed address), device pack + encryption into the plan's input
    // ciphertexts, the cloud plan, decryption of the results and the download
    // of slots + noise deviations into `out` (pinned).  Plan-owned workspaces.
    // Two graphs: the early one is the encryption's message-independent branch
    // (upload of the image's stream ids and output handles, u, pk u), the main
    // one everything else.  run_early() may be enqueued before the host has
    // built the image's CSR part (the ids must already be in place);
    // run_pipeline(early_done) enqueues the early graph too unless it ran.
    void capture_pipeline(const unsigned char* img, const CsscLayout& lay, unsigned char* out);
    void run_early();
    void run_pipeline(bool early_done = false);  // enqueue (no sync)
    bool has_pipeline() const { return pexec_ != nullptr; }
    int results() const { return ns_; }
    // pipeline download layout: result s's first rows_[s] slots as u32 at
    // out_off()[s] (in u32 units), then one u64 rounding deviation per result
    // at byte offset maxdev_off(); slots past the tallest chunk of a slice are
    // masked to zero and not downloaded
    const std::vector<size_t>& out_off() const { return out_off_; }
    const std::vector<int>& out_rows() const { return rows_; }
    size_t maxdev_off() const { return maxdev_off_; }
    size_t pipeline_out_bytes() const { return maxdev_off_ + 8 * (size_t)ns_; }
    const PlanStats& stats() const { return stats_; }

private:
    // dec_d: the pipeline's decrypting tail (fused path): the mask step writes
    // d = c0 + c1 s per slice into dec_d ([ns][L][N]) instead of the result cts
    // enc: the inputs still need the encryption's finishing step (pipeline)
    void record(std::vector<cudaEvent_t>* marks = nullptr, u64* dec_d = nullptr, const EncIn* enc = nullptr);
    template <class T>
    T* put(const std::vector<T>& v);

    GpuContext& ctx_;
    int n_ = 0, ns_ = 0;
    std::vector<int> rows_;        // per result: tallest chunk height
    std::vector<size_t> out_off_;  // per result: u32 offset in the download
    size_t maxdev_off_ = 0;
    DevBuf pgather_;               // device copy of {rows, out_off}
    const int* ORDER_ = nullptr;   // multiply item k -> chunk (depth order), device
    PlanStats stats_;
    DevBuf prod_, acc0_, acc1_, rp_;  // rp_: hoisted odd-step rotations of the products
    DevBuf T_, Z_, D2_, DX_, ACC_, MT_, MASKS_;
    DevBuf arena_;                        // device pointer / index arrays (one block)
    std::vector<unsigned char> stage_;    // host staging of arena_
    // device arrays
    const u64* const* A_ = nullptr;
    const u64* const* B_ = nullptr;
    u64* const* PROD_ = nullptr;
    const u64* const* RLK_ = nullptr;
    struct Level {
        int items;      // tail items (one INTT + ModDown each): the doubling steps
        int acc_items;  // key switches accumulated: + level 0's odd steps
        const u64* const* src;
        const u64* const* base;
        u64* const* out;
        const u64* const* key;
        const u32* ginv;
        const u64* const* extra;  // fused add of a hoisted odd-step rotation (nullable)
        const int* pair;          // level 0: D_1 items merging their O_1 rotation (nullable)
        const u64* const* ysrc;   // hoisted ModUp factors of each source's c1 (KsY; nullable)
        u64* const* yout;         // ... of each output's c1 when a later level rotates it
        int keys;                  // distinct switching keys of the level
        // level 0 hoisted: every rotation of a product shares its ModUp + NTT
        int hsrc = 0;                      // products (0: not hoisted)
        const u64* const* hprod = nullptr;  // per product: its ciphertext
        const u64* const* hy = nullptr;     // per product: KsY factors of c1
        int hterm = 1;                      // MAC terms per item
        int mac_terms = 0;                  // key products summed over the level's items
        const int* hidx = nullptr;          // [item][hterm] source index (-1: none)
        const u32* gel = nullptr;           // [item][hterm] Galois element (1: identity)
        const u64* const* hkey = nullptr;   // [item][hterm] switching key
        const int* horder = nullptr;        // K2h launch order (by Galois element)
        const u64* const* xacc = nullptr;   // per tail item: an odd step's accumulators (nullable)
        int odd_n = 0;                      // level 0: odd steps whose c0 term goes to rp slots
        const u64* const* odd_src = nullptr;
        const u32* odd_ginv = nullptr;
        u64* const* odd_out = nullptr;
        // fold mode: c0 terms summed into EXTRA slots (level 0 writes them, later levels add)
        int asum_n = 0;
        u64* const* asum_out = nullptr;
        const u64* const* asum_src = nullptr;  // [item][3]
        const u32* asum_gi = nullptr;           // [item][3] inverse Galois elements (0: none)
        bool asum_acc = false;
    };
    std::vector<Level> levels_;
    const u64* const* FINAL_ = nullptr;
    u64* const* OUT_ = nullptr;
    const int* slice_off_ = nullptr;
    const int* slice_items_ = nullptr;
    const int* item_mask_ = nullptr;
    int n_masks_ = 0;
    cudaGraph_t graph_ = nullptr;
    cudaGraphExec_t exec_ = nullptr;
    DevBuf pup_, pU_, pCM_, pX_, pM_, pslots_, pE_;  // pipeline workspaces
    DevBuf prodY_, accY0_, accY1_, D2Y_;            // hoisted ModUp factors (KsY)
    u64* const* PRODY_ = nullptr;
    bool fold_ = false;  // relinearisation folded into level 0 (rotated chunks' products stay unrelinearised)
    int nd_ = 0;         // chunks with at least one doubling step (items 0 .. nd_-1)
    cudaGraphExec_t pexec_ = nullptr, eexec_ = nullptr;
    cudaEvent_t ev_early_ = nullptr, ev_fork_ = nullptr;  // early graph on the side stream
    std::vector<cudaEvent_t> pmarks_;  // CSSC_PIPE_PROFILE=1: phase marks inside the pipeline graph
};

}  // namespace cssc
