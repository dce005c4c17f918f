// ref_shim.cpp -- C-ABI shim over the UNMODIFIED reference library
// (/root/reference/proj/src/*.cpp, compiled in place by oracle/Makefile into
// oracle/_ref/libspmv_ref.so).  TEST / BASELINE INFRASTRUCTURE ONLY: it lets
// Python tests and bench.py's reference arm call the reference's own
// spmv_partitioned with its SimBackend, its synthetic generators and its
// aggregation plan.  Nothing in the product links it.
//
// Reference entry points wrapped here:
//   spmv_partitioned      proj/src/protocol.cpp:155-176
//   SimBackend            proj/include/spmv/he.hpp:119-139
//   random_sparse_csr     proj/src/synthetic.cpp:32-72
//   random_vector         proj/src/synthetic.cpp:74-86
//   rotation_schedule     proj/src/aggregate.cpp:19-34
//   csr_to_cssc           proj/src/sparse.cpp:79-117
//   generate_chunks       proj/src/chunk.cpp:10-50
//   diag_spmv             proj/src/diagonal.cpp:44-104
//   spmv convert JSON     proj/tools/spmv_main.cpp:39-58 (csr_to_cssc,
//                         validate_cssc, ordered_json dump(2); needs the
//                         nlohmann/json header the CLI uses)
//   cloud section         proj/src/protocol.cpp:121-134 (multiply,
//                         intra_chunk_sum, inter_chunk_sum on the prepared
//                         client ciphertexts of every row slice)
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <memory>
#include <string>
#include <vector>

#include "spmv/aggregate.hpp"
#include "spmv/chunk.hpp"
#include "spmv/diagonal.hpp"
#include "spmv/he.hpp"
#include "spmv/protocol.hpp"
#include "spmv/reorg.hpp"
#include "spmv/sparse.hpp"
#include "spmv/synthetic.hpp"

#if __has_include(<nlohmann/json.hpp>)
#include <nlohmann/json.hpp>
#define REF_HAVE_JSON 1
#endif

namespace {
thread_local std::string g_err;

spmv::CsrMatrix make_csr(uint64_t rows, uint64_t cols, const int64_t* rp, const int64_t* ci,
                         const int64_t* va) {
    spmv::CsrMatrix m;
    m.rows = rows;
    m.cols = cols;
    m.row_ptrs.assign(rp, rp + rows + 1);
    const size_t nnz = static_cast<size_t>(rp[rows]);
    m.col_indices.assign(ci, ci + nnz);
    m.values.assign(va, va + nnz);
    return m;
}

int classify(const std::exception& e) {
    g_err = e.what();
    if (dynamic_cast<const spmv::ColumnTooTallError*>(&e)) return -1;
    if (dynamic_cast<const spmv::DimensionMismatchError*>(&e)) return -2;
    if (dynamic_cast<const std::invalid_argument*>(&e)) return -3;
    if (dynamic_cast<const spmv::OverLengthError*>(&e)) return -4;
    return -9;
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// Full protocol on the reference SimBackend.  ledger6 = {cc,cp,rot,add,enc,dec};
// msgs: 5 int64 per message (from,to,kind,bytes,count).  Returns n_ct (>= 0)
// or a negative error class.
int64_t ref_spmv_partitioned(uint64_t slot_count, uint64_t t, double ct_mb, const int* noise5,
                             uint64_t rows, uint64_t cols, const int64_t* rp, const int64_t* ci,
                             const int64_t* va, const int64_t* v, uint64_t vlen, uint64_t chunk,
                             int key_holder, int64_t* out_vals, uint64_t* ledger6,
                             int64_t* msgs, uint64_t* nmsgs, uint64_t msg_cap, int* noise_out) {
    try {
        spmv::HeParams p;
        p.slot_count = slot_count;
        p.plaintext_modulus = t;
        p.ciphertext_size_mb = ct_mb;
        p.noise = {noise5[0], noise5[1], noise5[2], noise5[3], noise5[4]};
        spmv::SimBackend be(p);
        const spmv::CsrMatrix m = make_csr(rows, cols, rp, ci, va);
        const std::vector<int64_t> vv(v, v + vlen);
        auto kh = static_cast<spmv::PartyRole>(key_holder);
        spmv::SpmvResult r = spmv::spmv_partitioned(be, m, vv, chunk, kh);
        std::memcpy(out_vals, r.values.data(), sizeof(int64_t) * r.values.size());
        const auto& L = r.op_ledger;
        const uint64_t led[6] = {L.n_mult_cc, L.n_mult_cp, L.n_rot, L.n_add, L.n_enc, L.n_dec};
        std::memcpy(ledger6, led, sizeof led);
        const auto& ms = r.message_ledger.messages;
        *nmsgs = ms.size();
        for (size_t i = 0; i < ms.size() && i < msg_cap; ++i) {
            msgs[5 * i + 0] = static_cast<int64_t>(ms[i].from);
            msgs[5 * i + 1] = static_cast<int64_t>(ms[i].to);
            msgs[5 * i + 2] = static_cast<int64_t>(ms[i].kind);
            msgs[5 * i + 3] = static_cast<int64_t>(ms[i].payload_bytes);
            msgs[5 * i + 4] = static_cast<int64_t>(ms[i].ciphertext_count);
        }
        *noise_out = r.noise_budget_remaining_bits;
        return static_cast<int64_t>(r.n_ct);
    } catch (const std::exception& e) {
        return classify(e);
    }
}

// The diagonal-method baseline on the reference SimBackend; same outputs as
// ref_spmv_partitioned (returns the number of diagonal ciphertexts).
int64_t ref_diag_spmv(uint64_t slot_count, uint64_t t, double ct_mb, const int* noise5, uint64_t rows,
                      uint64_t cols, const int64_t* rp, const int64_t* ci, const int64_t* va, const int64_t* v,
                      uint64_t vlen, int key_holder, int64_t* out_vals, uint64_t* ledger6, int64_t* msgs,
                      uint64_t* nmsgs, uint64_t msg_cap, int* noise_out) {
    try {
        spmv::HeParams p;
        p.slot_count = slot_count;
        p.plaintext_modulus = t;
        p.ciphertext_size_mb = ct_mb;
        p.noise = {noise5[0], noise5[1], noise5[2], noise5[3], noise5[4]};
        spmv::SimBackend be(p);
        const spmv::CsrMatrix m = make_csr(rows, cols, rp, ci, va);
        const std::vector<int64_t> vv(v, v + vlen);
        spmv::SpmvResult r = spmv::diag_spmv(be, m, vv, static_cast<spmv::PartyRole>(key_holder));
        std::memcpy(out_vals, r.values.data(), sizeof(int64_t) * r.values.size());
        const auto& L = r.op_ledger;
        const uint64_t led[6] = {L.n_mult_cc, L.n_mult_cp, L.n_rot, L.n_add, L.n_enc, L.n_dec};
        std::memcpy(ledger6, led, sizeof led);
        const auto& ms = r.message_ledger.messages;
        *nmsgs = ms.size();
        for (size_t i = 0; i < ms.size() && i < msg_cap; ++i) {
            msgs[5 * i + 0] = static_cast<int64_t>(ms[i].from);
            msgs[5 * i + 1] = static_cast<int64_t>(ms[i].to);
            msgs[5 * i + 2] = static_cast<int64_t>(ms[i].kind);
            msgs[5 * i + 3] = static_cast<int64_t>(ms[i].payload_bytes);
            msgs[5 * i + 4] = static_cast<int64_t>(ms[i].ciphertext_count);
        }
        *noise_out = r.noise_budget_remaining_bits;
        return static_cast<int64_t>(r.n_ct);
    } catch (const std::exception& e) {
        if (dynamic_cast<const spmv::NonSquareError*>(&e)) {
            g_err = e.what();
            return -5;
        }
        return classify(e);
    }
}

// Timing helper for the reference arm: runs spmv_partitioned `reps` times
// and returns the best wall time in ms (steady_clock, like the reference's
// own acceptance timing, acceptance_main.cpp:58-60).
double ref_time_spmv_partitioned(uint64_t slot_count, uint64_t t, uint64_t rows, uint64_t cols,
                                 const int64_t* rp, const int64_t* ci, const int64_t* va,
                                 const int64_t* v, uint64_t chunk, int reps) {
    spmv::HeParams p;
    p.slot_count = slot_count;
    p.plaintext_modulus = t;
    spmv::SimBackend be(p);
    const spmv::CsrMatrix m = make_csr(rows, cols, rp, ci, va);
    const std::vector<int64_t> vv(v, v + cols);
    double best = 1e300;
    for (int i = 0; i < reps; ++i) {
        auto t0 = std::chrono::steady_clock::now();
        spmv::SpmvResult r = spmv::spmv_partitioned(be, m, vv, chunk);
        auto t1 = std::chrono::steady_clock::now();
        (void)r;
        double ms = std::chrono::duration<double, std::milli>(t1 - t0).count();
        if (ms < best) best = ms;
    }
    return best;
}

// random_sparse_csr: returns nnz; buffers rp (rows+1), ci/va (nnz)
int64_t ref_random_sparse_csr(uint64_t rows, uint64_t cols, uint64_t nnz, uint64_t seed,
                              int64_t lo, int64_t hi, int64_t* rp, int64_t* ci, int64_t* va) {
    try {
        spmv::CsrMatrix m = spmv::random_sparse_csr(rows, cols, nnz, seed, lo, hi);
        for (size_t i = 0; i <= rows; ++i) rp[i] = static_cast<int64_t>(m.row_ptrs[i]);
        for (size_t k = 0; k < m.nnz(); ++k) {
            ci[k] = static_cast<int64_t>(m.col_indices[k]);
            va[k] = m.values[k];
        }
        return static_cast<int64_t>(m.nnz());
    } catch (const std::exception& e) {
        return classify(e);
    }
}

void ref_random_vector(uint64_t len, uint64_t seed, int64_t lo, int64_t hi, int64_t* out) {
    auto v = spmv::random_vector(len, seed, lo, hi);
    std::memcpy(out, v.data(), sizeof(int64_t) * len);
}

int ref_rotation_schedule(uint64_t rows, uint64_t cols, uint64_t* offsets, int* from_acc) {
    try {
        auto s = spmv::rotation_schedule(rows, cols);
        for (size_t i = 0; i < s.size(); ++i) {
            offsets[i] = s[i].offset;
            from_acc[i] = s[i].from_accumulator ? 1 : 0;
        }
        return static_cast<int>(s.size());
    } catch (const std::exception& e) {
        return classify(e);
    }
}

// csr -> cssc -> chunks; returns n_ct; r/c lists and flats (sum r*c entries),
// row_map (rows entries).  Sizes first: call with null buffers to get
// n_ct and *flat_total.
int64_t ref_chunks(uint64_t rows, uint64_t cols, const int64_t* rp, const int64_t* ci,
                   const int64_t* va, uint64_t budget, int64_t* r_list, int64_t* c_list,
                   int64_t* vflat, int64_t* cflat, int64_t* row_map, uint64_t* flat_total) {
    try {
        const spmv::CsrMatrix m = make_csr(rows, cols, rp, ci, va);
        const spmv::ChunkSet cs = spmv::generate_chunks(spmv::csr_to_cssc(m), budget);
        uint64_t tot = 0;
        for (const auto& c : cs.chunks) tot += c.value_flat.size();
        *flat_total = tot;
        if (r_list) {
            uint64_t off = 0;
            for (size_t i = 0; i < cs.n_ct(); ++i) {
                r_list[i] = static_cast<int64_t>(cs.r_list[i]);
                c_list[i] = static_cast<int64_t>(cs.c_list[i]);
                const auto& c = cs.chunks[i];
                std::memcpy(vflat + off, c.value_flat.data(), 8 * c.value_flat.size());
                std::memcpy(cflat + off, c.colidx_flat.data(), 8 * c.colidx_flat.size());
                off += c.value_flat.size();
            }
            for (size_t i = 0; i < rows; ++i) row_map[i] = static_cast<int64_t>(cs.row_map[i]);
        }
        return static_cast<int64_t>(cs.n_ct());
    } catch (const std::exception& e) {
        return classify(e);
    }
}

// csr_to_cssc of the reference: sizes first (null arrays), then va/ci/rm/cp
int64_t ref_csr_to_cssc(uint64_t rows, uint64_t cols, const int64_t* rp, const int64_t* ci, const int64_t* va,
                        int64_t* out_va, int64_t* out_ci, int64_t* out_rm, int64_t* out_cp, uint64_t* aligned) {
    try {
        const spmv::CsscMatrix c = spmv::csr_to_cssc(make_csr(rows, cols, rp, ci, va));
        *aligned = c.aligned_cols();
        if (out_va) {
            for (size_t k = 0; k < c.va.size(); ++k) out_va[k] = c.va[k], out_ci[k] = static_cast<int64_t>(c.ci[k]);
            for (size_t k = 0; k < c.rm.size(); ++k) out_rm[k] = static_cast<int64_t>(c.rm[k]);
            for (size_t k = 0; k < c.cp.size(); ++k) out_cp[k] = static_cast<int64_t>(c.cp[k]);
        }
        return static_cast<int64_t>(c.nnz());
    } catch (const std::exception& e) {
        return classify(e);
    }
}

// the text `spmv convert` writes (tools/spmv_main.cpp:50-54): length, then bytes
int64_t ref_cssc_json(uint64_t rows, uint64_t cols, const int64_t* rp, const int64_t* ci, const int64_t* va,
                      char* out, uint64_t cap) {
#ifdef REF_HAVE_JSON
    try {
        const spmv::CsscMatrix cssc = spmv::csr_to_cssc(make_csr(rows, cols, rp, ci, va));
        using ordered_json = nlohmann::ordered_json;
        ordered_json j{
            {"rows", cssc.rows}, {"cols", cssc.cols}, {"va", cssc.va},
            {"ci", cssc.ci},     {"rm", cssc.rm},     {"cp", cssc.cp},
        };
        const std::string text = j.dump(2) + "\n";
        if (out && cap >= text.size()) std::memcpy(out, text.data(), text.size());
        return static_cast<int64_t>(text.size());
    } catch (const std::exception& e) {
        return classify(e);
    }
#else
    (void)rows, (void)cols, (void)rp, (void)ci, (void)va, (void)out, (void)cap;
    g_err = "built without nlohmann/json";
    return -8;
#endif
}

// ---- cloud-section probe (bench.py --impl reference `value`) ----
// ref_cloud_prepare runs the client phases of spmv() for every row slice
// (partition_rows, csr_to_cssc, generate_chunks, reorg_vector, encode +
// encrypt; protocol.cpp:94-119, :164) once; ref_cloud_run then replays only
// the cloud section (protocol.cpp:121-134) with the reference's own
// functions and returns its wall time in ms.
struct RefCloud {
    spmv::SimBackend be;
    struct Slice {
        std::vector<spmv::Ciphertext> a, b;
        std::vector<std::size_t> r, c;
    };
    std::vector<Slice> slices;
    explicit RefCloud(const spmv::HeParams& p) : be(p) {}
};

void* ref_cloud_prepare(uint64_t slot_count, uint64_t t, uint64_t rows, uint64_t cols, const int64_t* rp,
                        const int64_t* ci, const int64_t* va, const int64_t* v, uint64_t chunk) {
    try {
        spmv::HeParams p;
        p.slot_count = slot_count;
        p.plaintext_modulus = t;
        auto h = std::make_unique<RefCloud>(p);
        const spmv::CsrMatrix m = make_csr(rows, cols, rp, ci, va);
        const std::vector<int64_t> vv(v, v + cols);
        spmv::OpLedger ops;
        for (const spmv::CsrMatrix& slice : spmv::partition_rows(m, chunk)) {
            const spmv::ChunkSet cs = spmv::generate_chunks(spmv::csr_to_cssc(slice), chunk);
            const spmv::ReorgVector rv = spmv::reorg_vector(vv, cs);
            RefCloud::Slice s;
            for (const auto& c : cs.chunks) s.a.push_back(h->be.encrypt(h->be.encode(c.value_flat), ops));
            for (const auto& seg : rv.segments) s.b.push_back(h->be.encrypt(h->be.encode(seg), ops));
            s.r = cs.r_list;
            s.c = cs.c_list;
            h->slices.push_back(std::move(s));
        }
        return h.release();
    } catch (const std::exception& e) {
        classify(e);
        return nullptr;
    }
}

double ref_cloud_run(void* handle) {
    auto* h = static_cast<RefCloud*>(handle);
    spmv::OpLedger ops;
    const auto t0 = std::chrono::steady_clock::now();
    for (const auto& s : h->slices) {
        if (s.a.empty()) continue;
        std::vector<spmv::Ciphertext> parts;
        parts.reserve(s.a.size());
        for (std::size_t i = 0; i < s.a.size(); ++i) {
            spmv::Ciphertext product = h->be.multiply(s.a[i], s.b[i], ops);
            parts.push_back(spmv::intra_chunk_sum(h->be, product, s.r[i], s.c[i], ops));
        }
        spmv::Ciphertext res = spmv::inter_chunk_sum(h->be, parts, s.r, ops);
        (void)res;
    }
    const auto t1 = std::chrono::steady_clock::now();
    return std::chrono::duration<double, std::milli>(t1 - t0).count();
}

void ref_cloud_free(void* handle) { delete static_cast<RefCloud*>(handle); }

}  // extern "C"
