// protocol.cpp -- the three-party encrypted SpMV round (reference
// protocol.cpp:16-202).  spmv()/spmv_partitioned() keep the reference's
// signatures; with a GpuBfvBackend they run the batched device plan
// (batched_spmv.cpp), with any other HeBackend the op-by-op loop below.
#include "spmv/protocol.hpp"

#include <algorithm>
#include <cmath>

#include "batched_spmv.hpp"
#include "spmv/gpu_backend.hpp"

namespace spmv {

std::string to_string(PartyRole p) {
    switch (p) {
        case PartyRole::ClientA: return "A";
        case PartyRole::ClientB: return "B";
        case PartyRole::Cloud: return "Cloud";
    }
    return "?";
}

std::string to_string(MessageKind k) {
    switch (k) {
        case MessageKind::CiphertextBatch: return "ciphertext_batch";
        case MessageKind::ColumnIndexPlain: return "column_index_plain";
        case MessageKind::ChunkShapeMeta: return "chunk_shape_meta";
        case MessageKind::ResultCiphertext: return "result_ciphertext";
        case MessageKind::PlaintextValues: return "plaintext_values";
    }
    return "?";
}

std::uint64_t MessageLedger::bytes_between(PartyRole from, PartyRole to) const {
    std::uint64_t sum = 0;
    for (const Message& m : messages)
        if (m.from == from && m.to == to) sum += m.payload_bytes;
    return sum;
}

std::size_t MessageLedger::ciphertexts_between(PartyRole from, PartyRole to) const {
    std::size_t sum = 0;
    for (const Message& m : messages)
        if (m.from == from && m.to == to) sum += m.ciphertext_count;
    return sum;
}

std::uint64_t ciphertext_batch_bytes(const HeParams& params, std::size_t count) {
    return static_cast<std::uint64_t>(std::llround(static_cast<double>(count) * params.ciphertext_size_mb * 1048576.0));
}

namespace {

std::uint64_t colidx_bytes(const ChunkSet& cs) {
    std::uint64_t b = 4;
    for (const Chunk& c : cs.chunks) b += 8 + 4 * static_cast<std::uint64_t>(c.colidx_flat.size());
    return b;
}

// Reference semantics, one HeBackend call per homomorphic operation.
SpmvResult spmv_generic(const HeBackend& be, const CsrMatrix& m, std::span<const std::int64_t> v,
                        std::size_t chunk_size, PartyRole key_holder) {
    const HeParams& hp = be.params();
    SpmvResult res;
    res.message_ledger.key_holder = key_holder;
    OpLedger& ops = res.op_ledger;
    auto& msgs = res.message_ledger;
    const ChunkSet cs = generate_chunks(csr_to_cssc(m), chunk_size);
    const std::size_t n_ct = cs.n_ct();
    res.n_ct = n_ct;
    std::vector<Ciphertext> A, B;
    for (const Chunk& ch : cs.chunks) A.push_back(be.encrypt(be.encode(ch.value_flat), ops));
    msgs.append({PartyRole::ClientA, PartyRole::Cloud, MessageKind::CiphertextBatch, ciphertext_batch_bytes(hp, n_ct), n_ct});
    msgs.append({PartyRole::ClientA, PartyRole::ClientB, MessageKind::ColumnIndexPlain, colidx_bytes(cs), 0});
    msgs.append({PartyRole::ClientA, PartyRole::Cloud, MessageKind::ChunkShapeMeta, 4 + 8 * static_cast<std::uint64_t>(n_ct), 0});
    for (const auto& seg : reorg_vector(v, cs).segments) B.push_back(be.encrypt(be.encode(seg), ops));
    msgs.append({PartyRole::ClientB, PartyRole::Cloud, MessageKind::CiphertextBatch, ciphertext_batch_bytes(hp, n_ct), n_ct});
    SlotVector slots(hp.slot_count, 0);
    res.noise_budget_remaining_bits = hp.noise.initial_budget_bits;
    if (n_ct) {
        std::vector<Ciphertext> parts;
        for (std::size_t i = 0; i < n_ct; ++i)
            parts.push_back(intra_chunk_sum(be, be.multiply(A[i], B[i], ops), cs.r_list[i], cs.c_list[i], ops));
        const Ciphertext out = inter_chunk_sum(be, parts, cs.r_list, ops);
        msgs.append({PartyRole::Cloud, key_holder, MessageKind::ResultCiphertext, ciphertext_batch_bytes(hp, 1), 1});
        slots = be.decrypt(out, ops);
        res.noise_budget_remaining_bits = out.noise_budget_bits;
    }
    res.values.assign(m.rows, 0);
    for (std::size_t p = 0; p < m.rows; ++p)
        res.values[cs.row_map[p]] = p < slots.size() ? to_signed(slots[p], hp.plaintext_modulus) : 0;
    return res;
}

}  // namespace

SpmvResult spmv(const HeBackend& be, const CsrMatrix& m, std::span<const std::int64_t> v,
                std::size_t chunk_size, PartyRole key_holder) {
    if (m.cols != v.size())
        throw DimensionMismatchError("spmv: vector length " + std::to_string(v.size()) +
                                     " does not match matrix column count " + std::to_string(m.cols));
    if (chunk_size == 0 || chunk_size > be.params().slot_count)
        throw std::invalid_argument("spmv: chunk_size must be in [1, slot_count]");
    if (const auto* gpu = dynamic_cast<const GpuBfvBackend*>(&be)) {
        // a single slice of the batched path: no row partitioning here
        const detail::CsrView w = detail::view_of(m, v);
        detail::BatchedSpmv job(gpu->context(), gpu->params(), std::span<const detail::CsrView>(&w, 1), chunk_size,
                                key_holder, /*partition=*/false);
        return std::move(job.run_all()[0]);
    }
    return spmv_generic(be, m, v, chunk_size, key_holder);
}

std::vector<SpmvResult> spmv_batch(const HeBackend& be, std::span<const CsrMatrix> ms,
                                   std::span<const std::vector<std::int64_t>> vs, std::size_t chunk_size,
                                   PartyRole key_holder) {
    if (const auto* gpu = dynamic_cast<const GpuBfvBackend*>(&be)) {
        if (ms.size() != vs.size()) throw DimensionMismatchError("spmv_batch: matrices and vectors differ in count");
        std::vector<detail::CsrView> w;
        for (std::size_t i = 0; i < ms.size(); ++i) w.push_back(detail::view_of(ms[i], vs[i]));
        detail::BatchedSpmv job(gpu->context(), gpu->params(), w, chunk_size, key_holder);
        return job.run_all();
    }
    std::vector<SpmvResult> out;
    for (std::size_t i = 0; i < ms.size(); ++i) out.push_back(spmv_partitioned(be, ms[i], vs[i], chunk_size, key_holder));
    return out;
}

SpmvResult spmv_partitioned(const HeBackend& be, const CsrMatrix& m, std::span<const std::int64_t> v,
                            std::size_t chunk_size, PartyRole key_holder) {
    if (m.cols != v.size()) throw DimensionMismatchError("spmv_partitioned: vector length does not match columns");
    if (const auto* gpu = dynamic_cast<const GpuBfvBackend*>(&be)) {
        const detail::CsrView w = detail::view_of(m, v);
        detail::BatchedSpmv job(gpu->context(), gpu->params(), std::span<const detail::CsrView>(&w, 1), chunk_size,
                                key_holder);
        return std::move(job.run_all()[0]);
    }
    SpmvResult merged;
    merged.message_ledger.key_holder = key_holder;
    merged.noise_budget_remaining_bits = be.params().noise.initial_budget_bits;
    for (const CsrMatrix& slice : partition_rows(m, chunk_size)) {
        SpmvResult part = spmv(be, slice, v, chunk_size, key_holder);
        merged.values.insert(merged.values.end(), part.values.begin(), part.values.end());
        merged.op_ledger += part.op_ledger;
        merged.message_ledger.messages.insert(merged.message_ledger.messages.end(),
                                              part.message_ledger.messages.begin(), part.message_ledger.messages.end());
        merged.n_ct += part.n_ct;
        merged.noise_budget_remaining_bits = std::min(merged.noise_budget_remaining_bits, part.noise_budget_remaining_bits);
    }
    return merged;
}

AuditReport audit_leakage(const MessageLedger& ledger) {
    AuditReport rep;
    for (std::size_t i = 0; i < ledger.messages.size(); ++i) {
        const Message& m = ledger.messages[i];
        const std::string at = "message #" + std::to_string(i) + " (" + to_string(m.from) + " -> " +
                               to_string(m.to) + ", " + to_string(m.kind) + ")";
        if (m.to == PartyRole::Cloud && m.kind != MessageKind::CiphertextBatch && m.kind != MessageKind::ChunkShapeMeta)
            rep.violations.push_back(at + ": the cloud may receive only ciphertext batches and chunk-shape metadata");
        if (m.kind == MessageKind::ColumnIndexPlain && !(m.from == PartyRole::ClientA && m.to == PartyRole::ClientB))
            rep.violations.push_back(at + ": plaintext column indices may flow only from A to B");
        if (m.kind == MessageKind::PlaintextValues && m.to != ledger.key_holder)
            rep.violations.push_back(at + ": plaintext values delivered to " + to_string(m.to) +
                                     ", but the key holder is " + to_string(ledger.key_holder));
    }
    rep.passed = rep.violations.empty();
    return rep;
}

}  // namespace spmv
