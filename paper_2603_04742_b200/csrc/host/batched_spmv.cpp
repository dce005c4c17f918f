// batched_spmv.cpp -- see batched_spmv.hpp.
#include "batched_spmv.hpp"

#include <algorithm>
#include <stdexcept>
#include <string>

#include "spmv/gpu_backend.hpp"

namespace spmv::detail {

namespace {

std::uint64_t column_index_bytes(const ChunkSet& cs) {
    std::uint64_t b = 4;  // chunk count, then an (h, k) header and 4-byte indices per chunk
    for (const Chunk& c : cs.chunks) b += 8 + 4 * static_cast<std::uint64_t>(c.colidx_flat.size());
    return b;
}

int lowered(int b, int c) { return std::max(0, b - c); }

}  // namespace

BatchedSpmv::BatchedSpmv(spmvgpu_ctx* ctx, const HeParams& hp, std::span<const CsrMatrix> ms,
                         std::span<const std::vector<std::int64_t>> vs, std::size_t chunk_size,
                         PartyRole key_holder, bool partition)
    : ctx_(ctx), hp_(hp), kh_(key_holder), nmat_(ms.size()) {
    if (ms.size() != vs.size()) throw DimensionMismatchError("spmv_batch: matrices and vectors differ in count");
    std::vector<std::int64_t> b_vals;
    for (std::size_t mi = 0; mi < ms.size(); ++mi) {
        const CsrMatrix& m = ms[mi];
        const auto& v = vs[mi];
        if (m.cols != v.size())
            throw DimensionMismatchError("spmv_partitioned: vector length does not match columns");
        rows_of_.push_back(m.rows);
        // spmv_partitioned slices rows by chunk_size; plain spmv keeps one slice
        std::vector<CsrMatrix> parts = partition ? partition_rows(m, chunk_size) : std::vector<CsrMatrix>{m};
        for (CsrMatrix& part : parts) {
            // per-slice checks in the reference's order (protocol.cpp:80-90)
            if (chunk_size == 0 || chunk_size > hp_.slot_count)
                throw std::invalid_argument("spmv: chunk_size must be in [1, slot_count]");
            Slice s;
            s.mat = mi;
            s.rows = part.rows;
            s.cs = generate_chunks(csr_to_cssc(part), chunk_size);
            const ReorgVector rv = reorg_vector(v, s.cs);
            s.first_chunk = r_.size();
            for (std::size_t i = 0; i < s.cs.n_ct(); ++i) {
                r_.push_back(s.cs.r_list[i]);
                c_.push_back(s.cs.c_list[i]);
            }
            if (s.cs.n_ct()) {
                s.result = static_cast<int>(n_out_++);
            }
            for (std::size_t i = 0; i < s.cs.n_ct(); ++i) slice_id_.push_back(static_cast<std::uint32_t>(s.result));
            for (const auto& seg : rv.segments) b_vals.insert(b_vals.end(), seg.begin(), seg.end());
            slices_.push_back(std::move(s));
        }
    }
    // encryption inputs: [A flats of all chunks][B segments of all chunks]
    const std::size_t n = r_.size();
    offs_.assign(2 * n + 1, 0);
    std::size_t k = 0;
    for (int half = 0; half < 2; ++half)
        for (const Slice& s : slices_)
            for (const Chunk& ch : s.cs.chunks) {
                if (half == 0) vals_.insert(vals_.end(), ch.value_flat.begin(), ch.value_flat.end());
                offs_[k + 1] = offs_[k] + ch.value_flat.size();
                ++k;
            }
    vals_.insert(vals_.end(), b_vals.begin(), b_vals.end());
    if (!n) return;
    // the cloud's view of the job: chunk shapes and slice ids (ChunkShapeMeta)
    std::vector<std::uint64_t> key{n, n_out_};
    key.insert(key.end(), r_.begin(), r_.end());
    key.insert(key.end(), c_.begin(), c_.end());
    key.insert(key.end(), slice_id_.begin(), slice_id_.end());
    if (plan_cache_take(ctx_, key, lease_)) return;
    lease_.key = std::move(key);
    lease_.a.assign(n, 0);
    lease_.b.assign(n, 0);
    lease_.out.assign(n_out_, 0);
    try {
        check_status(spmvgpu_ct_alloc(ctx_, n, lease_.a.data()));
        check_status(spmvgpu_ct_alloc(ctx_, n, lease_.b.data()));
        check_status(spmvgpu_ct_alloc(ctx_, n_out_, lease_.out.data()));
    } catch (...) {
        plan_lease_free(ctx_, lease_);
        throw;
    }
}

BatchedSpmv::~BatchedSpmv() {
    if (lease_.key.empty()) return;
    if (done_)
        plan_cache_give(ctx_, std::move(lease_));
    else  // an evaluation that did not complete: do not keep its buffers
        plan_lease_free(ctx_, lease_);
}

void BatchedSpmv::encrypt() {
    const std::size_t n = r_.size();
    if (!n) return;
    std::vector<spmvgpu_ct> all(lease_.a);
    all.insert(all.end(), lease_.b.begin(), lease_.b.end());
    check_status(spmvgpu_encrypt(ctx_, vals_.data(), offs_.data(), nullptr, all.data(), 2 * n));
    h2d_ = sizeof(std::int64_t) * vals_.size() + sizeof(std::uint64_t) * offs_.size();
}

void BatchedSpmv::ensure_plan() {
    if (lease_.plan || r_.empty()) return;
    check_status(spmvgpu_plan_create(ctx_, r_.size(), r_.data(), c_.data(), slice_id_.data(), n_out_,
                                     lease_.a.data(), lease_.b.data(), lease_.out.data(), &lease_.plan));
}

void BatchedSpmv::cloud(bool use_graph) {
    if (r_.empty()) return;
    ensure_plan();
    // a plan seen before is worth a graph: capture on its second use
    if ((use_graph || lease_.uses > 0) && !lease_.captured) {
        check_status(spmvgpu_plan_capture(lease_.plan));
        lease_.captured = true;
    }
    check_status(spmvgpu_plan_run(lease_.plan));
    ++lease_.uses;
}

std::vector<SpmvResult> BatchedSpmv::finish() {
    const std::size_t S = hp_.slot_count;
    std::vector<std::uint64_t> slots(n_out_ * S);
    std::vector<std::int32_t> measured(n_out_, 0);
    if (n_out_)
        check_status(spmvgpu_decrypt(ctx_, lease_.out.data(), n_out_, slots.data(), measured.data()));
    else
        check_status(spmvgpu_sync(ctx_));
    done_ = true;
    d2h_ = sizeof(std::uint64_t) * slots.size();

    const NoiseModel& nm = hp_.noise;
    std::vector<SpmvResult> res(nmat_);
    for (std::size_t mi = 0; mi < nmat_; ++mi) {
        res[mi].message_ledger.key_holder = kh_;
        res[mi].noise_budget_remaining_bits = nm.initial_budget_bits;
        res[mi].values.reserve(rows_of_[mi]);
    }
    for (const Slice& s : slices_) {
        SpmvResult& R = res[s.mat];
        const std::size_t n_ct = s.cs.n_ct();
        // ledger identities of one slice (protocol.cpp:99-136)
        OpLedger led;
        led.n_enc = 2 * n_ct;
        led.n_mult_cc = n_ct;
        led.n_mult_cp = n_ct;
        std::uint64_t rot = 0;
        for (std::size_t i = 0; i < n_ct; ++i) rot += rotation_schedule(s.cs.r_list[i], s.cs.c_list[i]).size();
        led.n_rot = rot;
        led.n_add = rot + n_ct;
        led.n_dec = n_ct ? 1 : 0;
        R.op_ledger += led;
        R.n_ct += n_ct;
        // transcript (protocol.cpp:104-134)
        auto& msgs = R.message_ledger.messages;
        msgs.push_back({PartyRole::ClientA, PartyRole::Cloud, MessageKind::CiphertextBatch,
                        ciphertext_batch_bytes(hp_, n_ct), n_ct});
        msgs.push_back({PartyRole::ClientA, PartyRole::ClientB, MessageKind::ColumnIndexPlain,
                        column_index_bytes(s.cs), 0});
        msgs.push_back({PartyRole::ClientA, PartyRole::Cloud, MessageKind::ChunkShapeMeta,
                        4 + 8 * static_cast<std::uint64_t>(n_ct), 0});
        msgs.push_back({PartyRole::ClientB, PartyRole::Cloud, MessageKind::CiphertextBatch,
                        ciphertext_batch_bytes(hp_, n_ct), n_ct});
        // model noise, replaying the backend's budget arithmetic
        int slice_noise = nm.initial_budget_bits;
        std::vector<std::int64_t> vals(s.rows, 0);
        if (n_ct) {
            msgs.push_back({PartyRole::Cloud, kh_, MessageKind::ResultCiphertext, ciphertext_batch_bytes(hp_, 1), 1});
            int res_b = nm.initial_budget_bits;
            for (std::size_t i = 0; i < n_ct; ++i) {
                const int prod_b = lowered(nm.initial_budget_bits, nm.cost_ct_ct_mult_bits);
                int acc_b = prod_b;
                for (const RotStep& st : rotation_schedule(s.cs.r_list[i], s.cs.c_list[i])) {
                    const int rot_b = lowered(st.from_accumulator ? acc_b : prod_b, nm.cost_rot_bits);
                    acc_b = lowered(std::min(acc_b, rot_b), nm.cost_add_bits);
                }
                res_b = lowered(std::min(res_b, lowered(acc_b, nm.cost_ct_pt_mult_bits)), nm.cost_add_bits);
            }
            slice_noise = res_b;
            if (res_b <= 0)
                throw NoiseExhaustedError("decrypt: noise budget exhausted (slice result)");
            const std::uint64_t* sl = slots.data() + static_cast<std::size_t>(s.result) * S;
            for (std::size_t idx = 0; idx < s.rows; ++idx)
                vals[s.cs.row_map[idx]] = idx < S ? to_signed(sl[idx], hp_.plaintext_modulus) : 0;
            const int meas = measured[static_cast<std::size_t>(s.result)];
            R.measured_noise_budget_bits =
                R.measured_noise_budget_bits < 0 ? meas : std::min(R.measured_noise_budget_bits, meas);
        }
        R.values.insert(R.values.end(), vals.begin(), vals.end());
        R.noise_budget_remaining_bits = std::min(R.noise_budget_remaining_bits, slice_noise);
    }
    return res;
}

}  // namespace spmv::detail
