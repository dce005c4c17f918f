// diagonal.cpp -- the diagonal-method baseline (reference proj/src/diagonal.cpp:10-115).
//
// extract_diagonals and the generic diag_spmv restate the reference over any
// HeBackend.  With a GpuBfvBackend the same computation runs batched through
// the C-ABI: all diagonal and vector encryptions in one call, the n_diag
// rotations of the vector ciphertext as one key-switch launch group, the
// n_diag products as one multiply group, and the accumulation as one
// summation launch, in groups of kGroup diagonals to bound memory.  Ledger,
// transcript and model noise are the reference's.
#include "spmv/diagonal.hpp"

#include <algorithm>
#include <string>

#include "spmv/gpu_backend.hpp"

namespace spmv {

DiagPlan extract_diagonals(const CsrMatrix& m) {
    if (m.rows != m.cols)
        throw NonSquareError("extract_diagonals: matrix is " + std::to_string(m.rows) + "x" +
                             std::to_string(m.cols) + "; the diagonal method needs square input");
    const std::size_t n = m.rows;
    DiagPlan plan;
    plan.n = n;
    std::vector<int> slot(n, -1);  // offset -> index into by_offset
    std::vector<std::vector<std::int64_t>> by_offset;
    std::vector<std::size_t> offs;
    for (std::size_t i = 0; i < n; ++i)
        for (std::size_t k = m.row_ptrs[i]; k < m.row_ptrs[i + 1]; ++k) {
            const std::size_t d = (m.col_indices[k] + n - i) % n;
            if (slot[d] < 0) {
                slot[d] = static_cast<int>(by_offset.size());
                by_offset.emplace_back(n, 0);
                offs.push_back(d);
            }
            by_offset[static_cast<std::size_t>(slot[d])][i] = m.values[k];
        }
    // ascending offsets, as the reference lists them
    std::vector<std::size_t> order(offs.size());
    for (std::size_t i = 0; i < order.size(); ++i) order[i] = i;
    std::sort(order.begin(), order.end(), [&](std::size_t a, std::size_t b) { return offs[a] < offs[b]; });
    for (std::size_t i : order) {
        plan.offsets.push_back(offs[i]);
        plan.vectors.push_back(std::move(by_offset[i]));
    }
    return plan;
}

namespace {

int lowered(int b, int c) { return std::max(0, b - c); }

constexpr std::size_t kGroup = 256;  // diagonals per device launch group

// Batched device evaluation; returns the decrypted slots of the accumulator.
SlotVector diag_cloud_gpu(const GpuBfvBackend& be, const DiagPlan& plan, const std::vector<std::int64_t>& packed,
                          int* measured) {
    spmvgpu_ctx* ctx = be.context();
    const std::size_t n_diag = plan.offsets.size();
    std::vector<spmvgpu_ct> partial;
    std::vector<spmvgpu_ct> live;
    auto release = [&](std::vector<spmvgpu_ct>& v) {
        if (!v.empty()) spmvgpu_ct_free(ctx, v.data(), v.size());
        v.clear();
    };
    try {
        for (std::size_t g0 = 0; g0 < n_diag; g0 += kGroup) {
            const std::size_t g = std::min(kGroup, n_diag - g0);
            // Client A (diagonals of this group) + Client B (the vector, once per group)
            std::vector<std::int64_t> vals;
            std::vector<std::uint64_t> offs{0};
            for (std::size_t k = g0; k < g0 + g; ++k) {
                vals.insert(vals.end(), plan.vectors[k].begin(), plan.vectors[k].end());
                offs.push_back(vals.size());
            }
            vals.insert(vals.end(), packed.begin(), packed.end());
            offs.push_back(vals.size());
            live.assign(3 * g + 1, 0);
            check_status(spmvgpu_ct_alloc(ctx, live.size(), live.data()));
            const spmvgpu_ct* cd = live.data();          // g diagonal cts
            const spmvgpu_ct cv = live[g];               // vector ct
            const spmvgpu_ct* rot = live.data() + g + 1;  // g rotated vectors
            const spmvgpu_ct* prod = rot + g;            // g products
            check_status(spmvgpu_encrypt(ctx, vals.data(), offs.data(), nullptr, live.data(), g + 1));
            // Cloud: rotate, multiply, accumulate
            const std::vector<spmvgpu_ct> src(g, cv);
            std::vector<std::int64_t> steps(g);
            for (std::size_t k = 0; k < g; ++k) steps[k] = static_cast<std::int64_t>(plan.offsets[g0 + k]);
            check_status(spmvgpu_rotate(ctx, src.data(), steps.data(), rot, g));
            check_status(spmvgpu_mul_relin(ctx, cd, rot, prod, g));
            spmvgpu_ct acc = 0;
            check_status(spmvgpu_ct_alloc(ctx, 1, &acc));
            partial.push_back(acc);
            check_status(spmvgpu_sum(ctx, prod, g, acc));
            release(live);
        }
        spmvgpu_ct total = partial[0];
        if (partial.size() > 1) {
            check_status(spmvgpu_ct_alloc(ctx, 1, &total));
            live.push_back(total);
            check_status(spmvgpu_sum(ctx, partial.data(), partial.size(), total));
        }
        std::uint64_t n = 0, slots = 0, ctw = 0, kw = 0;
        int dnum = 0;
        check_status(spmvgpu_ctx_sizes(ctx, &n, &slots, &ctw, &kw, &dnum));
        SlotVector out(slots, 0);
        std::int32_t meas = 0;
        check_status(spmvgpu_decrypt(ctx, &total, 1, out.data(), &meas));
        *measured = meas;
        release(live);
        release(partial);
        return out;
    } catch (...) {
        release(live);
        release(partial);
        throw;
    }
}

}  // namespace

SpmvResult diag_spmv(const HeBackend& be, const CsrMatrix& m, std::span<const std::int64_t> v,
                     PartyRole key_holder) {
    const HeParams& params = be.params();
    if (m.cols != v.size())
        throw DimensionMismatchError("diag_spmv: vector length does not match matrix columns");
    const DiagPlan plan = extract_diagonals(m);
    const std::size_t n = plan.n;
    if (n > params.slot_count) throw OverLengthError("diag_spmv: matrix order exceeds slot count");
    const bool duplicated = 2 * n <= params.slot_count;
    if (!duplicated && n != params.slot_count)
        throw OverLengthError("diag_spmv: order " + std::to_string(n) +
                              " needs the duplicated vector layout, which requires 2n <= slot_count "
                              "(or n == slot_count)");

    SpmvResult res;
    res.message_ledger.key_holder = key_holder;
    OpLedger& ops = res.op_ledger;
    MessageLedger& msgs = res.message_ledger;
    const std::size_t n_diag = plan.offsets.size();
    res.n_ct = n_diag;
    std::vector<std::int64_t> packed(v.begin(), v.end());
    if (duplicated) packed.insert(packed.end(), v.begin(), v.end());

    const auto* gpu = dynamic_cast<const GpuBfvBackend*>(&be);
    if (gpu) {
        const NoiseModel& nm = params.noise;
        ops.n_enc += n_diag + 1;
        msgs.append({PartyRole::ClientA, PartyRole::Cloud, MessageKind::CiphertextBatch,
                     ciphertext_batch_bytes(params, n_diag), n_diag});
        msgs.append({PartyRole::ClientB, PartyRole::Cloud, MessageKind::CiphertextBatch,
                     ciphertext_batch_bytes(params, 1), 1});
        if (n_diag == 0) {
            res.noise_budget_remaining_bits = nm.initial_budget_bits;
            res.values.assign(n, 0);
            return res;
        }
        // model noise exactly as the op-by-op evaluation would track it
        const int rot_b = lowered(nm.initial_budget_bits, nm.cost_rot_bits);
        const int prod_b = lowered(std::min(nm.initial_budget_bits, rot_b), nm.cost_ct_ct_mult_bits);
        int acc_b = nm.initial_budget_bits;
        for (std::size_t k = 0; k < n_diag; ++k) acc_b = lowered(std::min(acc_b, prod_b), nm.cost_add_bits);
        ops.n_rot += n_diag;
        ops.n_mult_cc += n_diag;
        ops.n_add += n_diag;
        msgs.append({PartyRole::Cloud, key_holder, MessageKind::ResultCiphertext, ciphertext_batch_bytes(params, 1), 1});
        if (acc_b <= 0) throw NoiseExhaustedError("decrypt: noise budget exhausted");
        int measured = -1;
        const SlotVector slots = diag_cloud_gpu(*gpu, plan, packed, &measured);
        if (measured <= 0)  // the real BFV check: the result would decrypt to wrong values
            throw NoiseExhaustedError("decrypt: measured invariant-noise budget exhausted");
        ops.n_dec += 1;
        res.noise_budget_remaining_bits = acc_b;
        res.measured_noise_budget_bits = measured;
        res.values.resize(n);
        for (std::size_t i = 0; i < n; ++i) res.values[i] = to_signed(slots[i], params.plaintext_modulus);
        return res;
    }

    // generic backend: one call per homomorphic operation, as the reference
    std::vector<Ciphertext> ct_diags;
    ct_diags.reserve(n_diag);
    for (const auto& diag : plan.vectors) ct_diags.push_back(be.encrypt(be.encode(diag), ops));
    msgs.append({PartyRole::ClientA, PartyRole::Cloud, MessageKind::CiphertextBatch,
                 ciphertext_batch_bytes(params, n_diag), n_diag});
    const Ciphertext ct_v = be.encrypt(be.encode(packed), ops);
    msgs.append({PartyRole::ClientB, PartyRole::Cloud, MessageKind::CiphertextBatch, ciphertext_batch_bytes(params, 1), 1});
    if (n_diag == 0) {
        res.noise_budget_remaining_bits = params.noise.initial_budget_bits;
        res.values.assign(n, 0);
        return res;
    }
    Ciphertext acc = be.zero_ciphertext();
    for (std::size_t k = 0; k < n_diag; ++k) {
        const Ciphertext rotated = be.rotate(ct_v, static_cast<std::int64_t>(plan.offsets[k]), ops);
        acc = be.add(acc, be.multiply(ct_diags[k], rotated, ops), ops);
    }
    msgs.append({PartyRole::Cloud, key_holder, MessageKind::ResultCiphertext, ciphertext_batch_bytes(params, 1), 1});
    const SlotVector slots = be.decrypt(acc, ops);
    res.noise_budget_remaining_bits = acc.noise_budget_bits;
    res.values.resize(n);
    for (std::size_t i = 0; i < n; ++i) res.values[i] = to_signed(slots[i], params.plaintext_modulus);
    return res;
}

ComparisonReport compare_ledgers(const OpLedger& ours, const OpLedger& baseline, const CostTable& costs) {
    ComparisonReport r;
    r.ours = ours;
    r.baseline = baseline;
    r.ours_ms = estimate_time_ms(ours, costs);
    r.baseline_ms = estimate_time_ms(baseline, costs);
    r.time_ratio = r.ours_ms > 0.0 ? r.baseline_ms / r.ours_ms : 0.0;
    return r;
}

}  // namespace spmv
