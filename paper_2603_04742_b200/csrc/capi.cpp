// capi.cpp -- the extern "C" boundary (include/spmvgpu.h).
// Device-side entry points (spmvgpu_*) wrap GpuContext / CloudPlan; the
// protocol front door (cssc_*) wraps the host C++ spmv layer, which itself
// talks to the device only through spmvgpu_*.  No exception crosses the ABI.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <list>
#include <memory>
#include <mutex>
#include <new>
#include <stdexcept>
#include <string>

#include <sys/random.h>

#include "bfv_context.hpp"
#include "cloud_plan.hpp"
#include "host/batched_spmv.hpp"
#include "host/plan_cache.hpp"
#include "spmv/diagonal.hpp"
#include "spmv/gpu_backend.hpp"
#include "spmvgpu.h"

struct spmvgpu_ctx {
    std::unique_ptr<cssc::GpuContext> g;
    spmvgpu_params p;
    spmv::HeParams hp;
    // plan cache (host/plan_cache.hpp), most recently returned first
    std::mutex plans_mu;
    std::list<spmv::detail::PlanLease> plans;
    std::size_t plan_capacity = 4;
    // one host thread at a time per context (the reference's backends may be
    // shared across threads); recursive: the protocol layer calls
    // back into the C-ABI
    std::recursive_mutex api_mu;
    // early encryption (pipeline_speculate): the chunk-shape key of the last
    // pipeline run, and within one call the plan whose early graph was
    // enqueued with stream ids from spec_id0
    std::vector<std::uint64_t> spec_key;
    spmvgpu_plan* spec_plan = nullptr;
    std::uint64_t spec_id0 = 0;
    ~spmvgpu_ctx();
};

struct spmvgpu_plan {
    spmvgpu_ctx* ctx;
    std::unique_ptr<cssc::CloudPlan> plan;
};

struct cssc_job {
    spmvgpu_ctx* ctx;
    std::unique_ptr<spmv::detail::BatchedSpmv> job;
};

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
    g_err = msg;
    return code;
}

template <class F>
int guard(F&& f) {
    try {
        f();
        return SPMVGPU_OK;
    } catch (const spmv::OverLengthError& e) {
        return fail(SPMVGPU_ERR_OVER_LENGTH, e.what());
    } catch (const std::length_error& e) {
        return fail(SPMVGPU_ERR_OVER_LENGTH, e.what());
    } catch (const spmv::NoiseExhaustedError& e) {
        return fail(SPMVGPU_ERR_NOISE_EXHAUSTED, e.what());
    } catch (const spmv::DimensionMismatchError& e) {
        return fail(SPMVGPU_ERR_DIMENSION, e.what());
    } catch (const spmv::ColumnTooTallError& e) {
        return fail(SPMVGPU_ERR_COLUMN_TOO_TALL, e.what());
    } catch (const spmv::IndexOutOfRangeError& e) {
        return fail(SPMVGPU_ERR_INDEX_RANGE, e.what());
    } catch (const spmv::DuplicateEntryError& e) {
        return fail(SPMVGPU_ERR_DUPLICATE, e.what());
    } catch (const spmv::NonSquareError& e) {
        return fail(SPMVGPU_ERR_NON_SQUARE, e.what());
    } catch (const spmv::ParseError& e) {
        return fail(SPMVGPU_ERR_PARSE, e.what());
    } catch (const std::invalid_argument& e) {
        return fail(SPMVGPU_ERR_INVALID_ARGUMENT, e.what());
    } catch (const std::bad_alloc&) {
        return fail(SPMVGPU_ERR_INTERNAL, "host allocation failed");
    } catch (const std::exception& e) {
        const std::string w = e.what();
        return fail(w.find("cuda") != std::string::npos || w.find("CUDA") != std::string::npos ||
                            w.find("kernel") != std::string::npos
                        ? SPMVGPU_ERR_CUDA
                        : SPMVGPU_ERR_INTERNAL,
                    w);
    }
}

std::unique_lock<std::recursive_mutex> api_lock(const spmvgpu_ctx* c) {
    if (!c) throw std::invalid_argument("null context");
    return std::unique_lock<std::recursive_mutex>(const_cast<spmvgpu_ctx*>(c)->api_mu);
}

cssc::GpuContext& G(spmvgpu_ctx* c) {
    if (!c || !c->g) throw std::invalid_argument("null context");
    return *c->g;
}

using cssc::u64;

std::vector<const u64*> cptrs(const spmvgpu_ct* h, size_t n) {
    std::vector<const u64*> v(n);
    for (size_t i = 0; i < n; ++i) {
        if (!h[i]) throw std::invalid_argument("null ciphertext handle");
        v[i] = reinterpret_cast<const u64*>(h[i]);
    }
    return v;
}
std::vector<u64*> mptrs(const spmvgpu_ct* h, size_t n) {
    std::vector<u64*> v(n);
    for (size_t i = 0; i < n; ++i) {
        if (!h[i]) throw std::invalid_argument("null ciphertext handle");
        v[i] = reinterpret_cast<u64*>(h[i]);
    }
    return v;
}

// C-ABI CSR -> borrowed view (BatchedSpmv validates row pointers and columns)
spmv::detail::CsrView view_of(const cssc_csr& m, const int64_t* v, uint64_t vlen) {
    if (vlen != m.cols)  // reference protocol.cpp:77-81
        throw spmv::DimensionMismatchError("spmv: vector length " + std::to_string(vlen) +
                                           " does not match matrix column count " + std::to_string(m.cols));
    if (m.rows && (!m.row_ptrs || (m.row_ptrs[m.rows] && (!m.col_indices || !m.values))))
        throw std::invalid_argument("csr: null array");
    if (m.cols && !v) throw std::invalid_argument("null vector");
    if (m.rows && m.row_ptrs[0] != 0) throw std::invalid_argument("csr: row_ptrs[0] must be 0");
    spmv::detail::CsrView w;
    w.rows = m.rows;
    w.cols = m.cols;
    w.nnz = m.rows ? static_cast<size_t>(m.row_ptrs[m.rows]) : 0;
    static const std::uint64_t zero = 0;
    w.row_ptrs = m.rows ? reinterpret_cast<const std::uint64_t*>(m.row_ptrs) : &zero;
    w.col_indices = reinterpret_cast<const std::uint64_t*>(m.col_indices);
    w.values = m.values;
    w.vec = v;
    return w;
}

spmv::CsrMatrix to_csr(const cssc_csr& m) {
    spmv::CsrMatrix out;
    out.rows = m.rows;
    out.cols = m.cols;
    out.row_ptrs.assign(m.row_ptrs, m.row_ptrs + m.rows + 1);
    const size_t nnz = m.rows ? static_cast<size_t>(m.row_ptrs[m.rows]) : 0;
    if (m.rows && m.row_ptrs[0] != 0) throw std::invalid_argument("csr: row_ptrs[0] must be 0");
    out.col_indices.assign(m.col_indices, m.col_indices + nnz);
    out.values.assign(m.values, m.values + nnz);
    for (size_t c : out.col_indices)
        if (c >= m.cols) throw spmv::IndexOutOfRangeError("csr: column index out of range");
    return out;
}

void fill_result(const spmv::SpmvResult& r, int64_t* values, cssc_result* res, cssc_message* msgs,
                 uint64_t cap) {
    if (values && !r.values.empty()) std::memcpy(values, r.values.data(), sizeof(int64_t) * r.values.size());
    if (res) {
        res->ledger = {r.op_ledger.n_mult_cc, r.op_ledger.n_mult_cp, r.op_ledger.n_rot,
                       r.op_ledger.n_add,     r.op_ledger.n_enc,     r.op_ledger.n_dec};
        res->n_ct = r.n_ct;
        res->noise_model_bits = r.noise_budget_remaining_bits;
        res->noise_measured_bits = r.measured_noise_budget_bits;
        res->n_messages = r.message_ledger.messages.size();
    }
    if (msgs)
        for (size_t i = 0; i < r.message_ledger.messages.size() && i < cap; ++i) {
            const auto& m = r.message_ledger.messages[i];
            msgs[i] = {static_cast<int64_t>(m.from), static_cast<int64_t>(m.to), static_cast<int64_t>(m.kind),
                       static_cast<int64_t>(m.payload_bytes), static_cast<int64_t>(m.ciphertext_count)};
        }
}

}  // namespace

namespace spmv::detail {

bool plan_cache_take(spmvgpu_ctx* ctx, const std::vector<std::uint64_t>& key, PlanLease& out) {
    std::lock_guard<std::mutex> g(ctx->plans_mu);
    for (auto it = ctx->plans.begin(); it != ctx->plans.end(); ++it)
        if (it->key == key) {
            out = std::move(*it);
            ctx->plans.erase(it);
            return true;
        }
    return false;
}

void plan_lease_free(spmvgpu_ctx* ctx, PlanLease& l) {
    // a speculative early graph of this plan may still run on the side stream
    if (l.plan && ctx->g) ctx->g->synchronize_side();
    if (l.plan) spmvgpu_plan_destroy(l.plan);
    l.plan = nullptr;
    if (ctx->g) {
        if (l.pimg) ctx->g->pinned_give(l.pimg, l.pimg_cap);
        if (l.pout) ctx->g->pinned_give(l.pout, l.pout_cap);
    }
    l.pimg = l.pout = nullptr;
    l.pkey.clear();
    for (auto* v : {&l.a, &l.b, &l.out}) {
        if (!v->empty()) spmvgpu_ct_free(ctx, v->data(), v->size());
        v->clear();
    }
    l.key.clear();
}

void plan_cache_give(spmvgpu_ctx* ctx, PlanLease&& lease) {
    std::list<PlanLease> evicted;
    {
        std::lock_guard<std::mutex> g(ctx->plans_mu);
        ctx->plans.push_front(std::move(lease));
        while (ctx->plans.size() > ctx->plan_capacity) {
            evicted.splice(evicted.end(), ctx->plans, std::prev(ctx->plans.end()));
        }
    }
    for (auto& l : evicted) plan_lease_free(ctx, l);
}

}  // namespace spmv::detail

namespace spmv::detail {

ClientImage client_image_layout(std::size_t nnz, std::size_t vec_len, std::size_t n_rows, std::size_t n_slices,
                                std::size_t n_cols, int items, int ci_w, int va_w, int v_w) {
    const cssc::CsscLayout l = cssc::CsscLayout::make(nnz, vec_len, n_rows, n_slices, n_cols, items, ci_w, va_w, v_w);
    ClientImage img;
    img.ci_w = ci_w;
    img.va_w = va_w;
    img.v_w = v_w;
    img.o_ci = l.o_ci;
    img.o_va = l.o_va;
    img.o_v = l.o_v;
    img.o_rows = l.o_rows;
    img.o_rpre = l.o_rpre;
    img.o_sl = l.o_sl;
    img.o_cols = l.o_cols;
    img.o_st = l.o_st;
    img.o_out = l.o_out;
    img.bytes = l.bytes;
    img.nnz = nnz;
    img.vec_len = vec_len;
    img.n_rows = n_rows;
    img.n_slices = n_slices;
    img.n_cols = n_cols;
    img.items = items;
    return img;
}

ClientImage client_image_take(spmvgpu_ctx* ctx, std::size_t nnz, std::size_t vec_len, std::size_t n_rows,
                              std::size_t n_slices, std::size_t n_cols, int items, int ci_w, int va_w, int v_w) {
    ClientImage img = client_image_layout(nnz, vec_len, n_rows, n_slices, n_cols, items, ci_w, va_w, v_w);
    img.p = ctx->g->pinned_take(img.bytes, &img.cap);
    return img;
}

void client_image_give(spmvgpu_ctx* ctx, ClientImage& img) {
    if (img.p) ctx->g->pinned_give(img.p, img.cap);
    img.p = nullptr;
}

void client_image_fill(spmvgpu_ctx* ctx, unsigned char* p, const ClientImage& img, const spmvgpu_ct* out) {
    auto& g = *ctx->g;
    auto* st = reinterpret_cast<std::uint64_t*>(p + img.o_st);
    for (int i = 0; i < img.items; ++i) st[i] = g.next_stream_id();
    std::memcpy(p + img.o_out, out, sizeof(spmvgpu_ct) * (std::size_t)img.items);
}

std::vector<std::size_t> client_image_key(const ClientImage& img) {
    return {img.bytes, img.nnz, img.vec_len, img.n_rows, img.n_slices, img.n_cols, (std::size_t)img.items,
            (std::size_t)img.ci_w, (std::size_t)img.va_w, (std::size_t)img.v_w};
}

static cssc::CsscLayout layout_of(const ClientImage& img) {
    cssc::CsscLayout l;
    l.o_ci = img.o_ci;
    l.o_va = img.o_va;
    l.o_v = img.o_v;
    l.o_rows = img.o_rows;
    l.o_rpre = img.o_rpre;
    l.o_sl = img.o_sl;
    l.o_cols = img.o_cols;
    l.o_st = img.o_st;
    l.o_out = img.o_out;
    l.bytes = img.bytes;
    l.nnz = img.nnz;
    l.entries = img.nnz;  // BatchedSpmv's rows partition the nonzeros
    l.vec_len = img.vec_len;
    l.n_rows = img.n_rows;
    l.n_slices = img.n_slices;
    l.n_cols = img.n_cols;
    l.items = img.items;
    l.ci_w = img.ci_w;
    l.va_w = img.va_w;
    l.v_w = img.v_w;
    return l;
}

bool pipeline_ready(const PlanLease& lease, const ClientImage& img) {
    return lease.plan && lease.plan->plan->has_pipeline() && lease.pimg && lease.pkey == client_image_key(img);
}

static ClientImage layout_of_key(const std::vector<std::size_t>& k) {
    return client_image_layout(k[1], k[2], k[3], k[4], k[5], static_cast<int>(k[6]), static_cast<int>(k[7]),
                               static_cast<int>(k[8]), static_cast<int>(k[9]));
}

void pipeline_speculate(spmvgpu_ctx* ctx) {
    ctx->spec_plan = nullptr;
    if (ctx->spec_key.empty() || !ctx->g) return;
    std::lock_guard<std::mutex> lk(ctx->plans_mu);
    for (PlanLease& l : ctx->plans) {
        if (l.key != ctx->spec_key) continue;
        if (!l.plan || !l.plan->plan->has_pipeline() || !l.pimg || l.pkey.size() != 10) return;
        const ClientImage lay = layout_of_key(l.pkey);
        if (l.a.size() + l.b.size() != static_cast<std::size_t>(lay.items)) return;
        // the ids and output handles exactly as client_image_fill will write them
        const std::uint64_t id0 = ctx->g->peek_stream_id();
        auto* st = reinterpret_cast<std::uint64_t*>(l.pimg + lay.o_st);
        for (int i = 0; i < lay.items; ++i) st[i] = id0 + static_cast<std::uint64_t>(i);
        unsigned char* o = l.pimg + lay.o_out;
        std::memcpy(o, l.a.data(), sizeof(spmvgpu_ct) * l.a.size());
        std::memcpy(o + sizeof(spmvgpu_ct) * l.a.size(), l.b.data(), sizeof(spmvgpu_ct) * l.b.size());
        l.plan->plan->run_early();
        ctx->spec_plan = l.plan;
        ctx->spec_id0 = id0;
        return;
    }
}

void pipeline_prepare(spmvgpu_ctx* ctx, PlanLease& lease, const ClientImage& img) {
    auto& g = *ctx->g;
    ctx->spec_plan = nullptr;  // a re-capture invalidates an early graph already enqueued
    g.synchronize_side();      // ... which must not run while its workspaces are replaced
    if (!lease.plan) throw std::logic_error("pipeline: no plan");
    const std::size_t out_bytes = lease.plan->plan->pipeline_out_bytes();
    if (!lease.pimg || lease.pimg_cap < img.bytes) {
        if (lease.pimg) g.pinned_give(lease.pimg, lease.pimg_cap);
        lease.pimg = nullptr;
        lease.pimg = g.pinned_take(img.bytes, &lease.pimg_cap);
    }
    if (!lease.pout || lease.pout_cap < out_bytes) {
        if (lease.pout) g.pinned_give(lease.pout, lease.pout_cap);
        lease.pout = nullptr;
        lease.pout = g.pinned_take(out_bytes, &lease.pout_cap);
    }
    lease.pkey.clear();
    lease.plan->plan->capture_pipeline(lease.pimg, layout_of(img), lease.pout);
    lease.pkey = client_image_key(img);
}

std::size_t pipeline_out_bytes(const PlanLease& lease) { return lease.plan->plan->pipeline_out_bytes(); }

PipelineResult pipeline_result(const PlanLease& lease, int r) {
    const auto& pl = *lease.plan->plan;
    const auto* md = reinterpret_cast<const unsigned long long*>(lease.pout + pl.maxdev_off());
    return {reinterpret_cast<const std::uint32_t*>(lease.pout) + pl.out_off()[r], pl.out_rows()[r], md[r]};
}

void pipeline_run(spmvgpu_ctx* ctx, PlanLease& lease) {
    // the early graph already ran iff pipeline_speculate enqueued it for this
    // plan with the ids client_image_fill has just written
    const ClientImage lay = layout_of_key(lease.pkey);
    const auto id0 = *reinterpret_cast<const std::uint64_t*>(lease.pimg + lay.o_st);
    const bool early = ctx->spec_plan == lease.plan && ctx->spec_id0 == id0;
    ctx->spec_plan = nullptr;
    lease.plan->plan->run_pipeline(early);
    ctx->g->synchronize();
    ctx->g->synchronize_side();  // done already unless another plan's speculative graph is still running
    ctx->spec_key = lease.key;
}

void client_image_encrypt(spmvgpu_ctx* ctx, ClientImage& img, const spmvgpu_ct* out) {
    auto& g = *ctx->g;
    client_image_fill(ctx, img.p, img, out);
    cssc::CsscLayout l;
    l.o_ci = img.o_ci;
    l.o_va = img.o_va;
    l.o_v = img.o_v;
    l.o_rows = img.o_rows;
    l.o_rpre = img.o_rpre;
    l.o_sl = img.o_sl;
    l.o_cols = img.o_cols;
    l.o_st = img.o_st;
    l.o_out = img.o_out;
    l.bytes = img.bytes;
    l.nnz = img.nnz;
    l.entries = img.nnz;  // BatchedSpmv's rows partition the nonzeros
    l.vec_len = img.vec_len;
    l.n_rows = img.n_rows;
    l.n_slices = img.n_slices;
    l.n_cols = img.n_cols;
    l.items = img.items;
    l.ci_w = img.ci_w;
    l.va_w = img.va_w;
    l.v_w = img.v_w;
    g.encrypt_cssc_image(img.p, l);
}

}  // namespace spmv::detail

spmvgpu_ctx::~spmvgpu_ctx() {
    if (g) {
        for (auto& l : plans) spmv::detail::plan_lease_free(this, l);
        plans.clear();
    }
}

extern "C" {

const char* spmvgpu_last_error(void) { return g_err.c_str(); }

void spmvgpu_default_params(int logn, spmvgpu_params* p) {
    std::memset(p, 0, sizeof *p);
    p->logn = logn;
    // Q just large enough for the path's depth (1 ct x ct + 1 ct x pt + a
    // rotate-and-add tree of up to 14 doublings) with a wide margin: the
    // invariant-noise budget left after the deepest tree (1 x S chunk) is ~30
    // bits at N = 2^13 / 2^14 and ~140 bits at 2^15.  One
    // key-switching digit (alpha = L, K = L: P >= Q), so a key switch is one
    // ModUp of c1 and L + K limb NTTs each way.
    if (logn <= 13) {  // N = 8192: 4 x 54 = 216 <= 218 (128-bit security), 4 primes
        p->L = 2, p->K = 2, p->alpha = 2, p->qbits = 54, p->pbits = 54;
    } else if (logn == 14) {  // N = 16384: 4 x 58 = 232 <= 438, 4 primes
        p->L = 2, p->K = 2, p->alpha = 2, p->qbits = 58, p->pbits = 58;
    } else {  // N = 32768: 8 x 58 = 464 <= 881, 8 primes
        p->L = 4, p->K = 4, p->alpha = 4, p->qbits = 58, p->pbits = 58;
    }
    p->t = 65537;
    p->seed = 0;  // 0: 256-bit ChaCha key + stream-id base from OS entropy
    p->device = 0;
    p->ciphertext_size_mb = 0.52;
    p->noise_initial = 146;
    p->noise_ct_ct = 33;
    p->noise_ct_pt = 26;
    p->noise_add = 0;
    p->noise_rot = 0;
}

int spmvgpu_ctx_create(const spmvgpu_params* p, spmvgpu_ctx** out) {
    return guard([&] {
        if (!p || !out) throw std::invalid_argument("null argument");
        cssc::RnsConfig cfg;
        cfg.logn = p->logn;
        cfg.L = p->L;
        cfg.K = p->K;
        cfg.alpha = p->alpha;
        cfg.qbits = p->qbits;
        cfg.pbits = p->pbits;
        cfg.t = p->t;
        cfg.seed = p->seed;
        uint64_t stream_base = 1;
        if (p->seed) {  // deterministic key (tests, KATs; oracle/bfv_oracle.c restates it)
            cfg.key = cssc::seed_key(p->seed);
        } else {  // production default: 256-bit key and a random stream-id base
            unsigned char rnd[40];
            size_t got = 0;
            while (got < sizeof rnd) {
                const ssize_t r = getrandom(rnd + got, sizeof rnd - got, 0);
                if (r <= 0) throw std::runtime_error("getrandom failed: no OS entropy for the key");
                got += static_cast<size_t>(r);
            }
            std::memcpy(cfg.key.w, rnd, 32);
            std::memcpy(&stream_base, rnd + 32, 8);
            stream_base = (stream_base >> 2) | 1;  // leave headroom below 2^64
        }
        auto c = std::make_unique<spmvgpu_ctx>();
        c->p = *p;
        c->hp.slot_count = (size_t)1 << (p->logn - 1);
        c->hp.plaintext_modulus = p->t;
        c->hp.ciphertext_size_mb = p->ciphertext_size_mb > 0 ? p->ciphertext_size_mb : 0.52;
        c->hp.noise = {p->noise_initial, p->noise_ct_ct, p->noise_ct_pt, p->noise_add, p->noise_rot};
        c->hp.validate();
        c->g = std::make_unique<cssc::GpuContext>(cfg, p->device);
        c->g->set_stream_base(stream_base);
        *out = c.release();
    });
}

void spmvgpu_ctx_destroy(spmvgpu_ctx* c) { delete c; }


int spmvgpu_ctx_primes(const spmvgpu_ctx* c, uint64_t* primes, int cap, int* count) {
    return guard([&] { auto lk_ = api_lock(c);
        const auto& P = const_cast<spmvgpu_ctx*>(c)->g->params();
        *count = P.np;
        for (int i = 0; i < P.np && i < cap; ++i) primes[i] = P.primes[i];
    });
}

int spmvgpu_ctx_sizes(const spmvgpu_ctx* c, uint64_t* n, uint64_t* slots, uint64_t* ct_words,
                      uint64_t* ksk_words, int* dnum) {
    return guard([&] { auto lk_ = api_lock(c);
        auto& g = G(const_cast<spmvgpu_ctx*>(c));
        if (n) *n = g.n();
        if (slots) *slots = g.params().S;
        if (ct_words) *ct_words = g.ct_words();
        if (ksk_words) *ksk_words = g.ksk_words();
        if (dnum) *dnum = g.params().dnum;
    });
}

int spmvgpu_sync(spmvgpu_ctx* c) { return guard([&] { auto lk_ = api_lock(c); G(c).synchronize(); }); }
int spmvgpu_set_option(spmvgpu_ctx* c, const char* name, int64_t value) {
    return guard([&] { auto lk_ = api_lock(c);
        const std::string n = name ? name : "";
        if (n == "fused_key_switch") {
            G(c).set_fused_key_switch(value != 0);
        } else if (n == "forked_encrypt") {
            G(c).set_forked_encrypt(value != 0);
        } else if (n == "pipeline_fuse") {
            if (value < 0 || value > 3) throw std::invalid_argument("pipeline_fuse: 0..3");
            G(c).set_pipe_fuse(static_cast<int>(value));
            std::list<spmv::detail::PlanLease> evicted;  // cached graphs bake the old choice in
            {
                std::lock_guard<std::mutex> g(c->plans_mu);
                evicted.splice(evicted.end(), c->plans);
            }
            for (auto& l : evicted) spmv::detail::plan_lease_free(c, l);
        } else if (n == "stream_base") {
            if (value <= 0) throw std::invalid_argument("stream_base: must be positive");
            G(c).set_stream_base(static_cast<uint64_t>(value));
        } else if (n == "plan_cache") {
            if (value < 0) throw std::invalid_argument("plan_cache: capacity must be >= 0");
            std::list<spmv::detail::PlanLease> evicted;
            {
                std::lock_guard<std::mutex> g(c->plans_mu);
                c->plan_capacity = static_cast<std::size_t>(value);
                while (c->plans.size() > c->plan_capacity)
                    evicted.splice(evicted.end(), c->plans, std::prev(c->plans.end()));
            }
            for (auto& l : evicted) spmv::detail::plan_lease_free(c, l);
        }
        else
            throw std::invalid_argument("unknown option: " + n);
    });
}
void* spmvgpu_stream(spmvgpu_ctx* c) { return c && c->g ? (void*)c->g->stream() : nullptr; }

int spmvgpu_galois_keys(spmvgpu_ctx* c, const int64_t* steps, size_t n) {
    return guard([&] { auto lk_ = api_lock(c); G(c).ensure_galois_keys(std::vector<int64_t>(steps, steps + n)); });
}
uint32_t spmvgpu_galois_element(const spmvgpu_ctx* c, int64_t step) {
    return cssc::galois_element(step, const_cast<spmvgpu_ctx*>(c)->g->n());
}
int spmvgpu_download_sk(spmvgpu_ctx* c, int64_t* out) { return guard([&] { auto lk_ = api_lock(c); G(c).download_sk(out); }); }
int spmvgpu_download_pk(spmvgpu_ctx* c, uint64_t* out) { return guard([&] { auto lk_ = api_lock(c); G(c).download_pk_coef(out); }); }
int spmvgpu_download_ksk(spmvgpu_ctx* c, uint32_t which, uint64_t* out) {
    return guard([&] { auto lk_ = api_lock(c); G(c).download_key_coef(which, out); });
}

int spmvgpu_ct_alloc(spmvgpu_ctx* c, size_t count, spmvgpu_ct* out) {
    return guard([&] { auto lk_ = api_lock(c);
        auto& g = G(c);
        for (size_t i = 0; i < count; ++i) out[i] = reinterpret_cast<spmvgpu_ct>(g.pool().alloc(sizeof(u64) * g.ct_words()));
    });
}
int spmvgpu_ct_free(spmvgpu_ctx* c, const spmvgpu_ct* cts, size_t count) {
    return guard([&] { auto lk_ = api_lock(c);
        auto& g = G(c);
        for (size_t i = 0; i < count; ++i)
            if (cts[i]) g.pool().release(reinterpret_cast<void*>(cts[i]), sizeof(u64) * g.ct_words());
    });
}
int spmvgpu_ct_upload(spmvgpu_ctx* c, spmvgpu_ct ct, const uint64_t* words) {
    return guard([&] { auto lk_ = api_lock(c);
        auto& g = G(c);
        cssc::cuda_check(cudaMemcpyAsync(reinterpret_cast<void*>(ct), words, sizeof(u64) * g.ct_words(),
                                         cudaMemcpyHostToDevice, g.stream()), "ct upload");
        g.synchronize();
    });
}
int spmvgpu_ct_download(spmvgpu_ctx* c, spmvgpu_ct ct, uint64_t* words) {
    return guard([&] { auto lk_ = api_lock(c);
        auto& g = G(c);
        cssc::cuda_check(cudaMemcpyAsync(words, reinterpret_cast<void*>(ct), sizeof(u64) * g.ct_words(),
                                         cudaMemcpyDeviceToHost, g.stream()), "ct download");
        g.synchronize();
    });
}

// ---------------------------------------------------------------- wire format
// [magic "CSW1"][logn u8][L u8][0 u16][FNV-1a of the Q primes, u64] then, for
// poly 0..1 and limb j < L, the N residues of q_j at bitlen(q_j) bits each,
// one little-endian bit stream (a real serialized size in place
// of the reference's 0.52 MB pricing, protocol.cpp:51-54).
namespace {
constexpr size_t kWireHeader = 16;

uint64_t q_fingerprint(const cssc::RnsParams& P) {
    uint64_t h = 1469598103934665603ULL;
    for (int j = 0; j < P.cfg.L; ++j)
        for (int b = 0; b < 8; ++b) {
            h ^= (P.primes[j] >> (8 * b)) & 0xff;
            h *= 1099511628211ULL;
        }
    return h;
}
int bitlen(uint64_t q) { return 64 - __builtin_clzll(q); }
size_t wire_bytes(const cssc::RnsParams& P) {
    uint64_t bits = 0;
    for (int j = 0; j < P.cfg.L; ++j) bits += (uint64_t)bitlen(P.primes[j]);
    return kWireHeader + (size_t)((2 * (uint64_t)P.n * bits + 7) / 8);
}
}  // namespace

int spmvgpu_ct_wire_size(spmvgpu_ctx* c, size_t* bytes) {
    return guard([&] { auto lk_ = api_lock(c);
        if (!bytes) throw std::invalid_argument("null argument");
        *bytes = wire_bytes(G(c).params());
    });
}

int spmvgpu_ct_serialize(spmvgpu_ctx* c, spmvgpu_ct ct, uint8_t* buf, size_t cap, size_t* written) {
    return guard([&] { auto lk_ = api_lock(c);
        auto& g = G(c);
        const auto& P = g.params();
        const size_t need = wire_bytes(P);
        if (!buf || cap < need) throw std::length_error("serialize: buffer smaller than the wire size");
        if (!ct) throw std::invalid_argument("null ciphertext handle");
        std::vector<u64> w(g.ct_words());
        cssc::cuda_check(cudaMemcpyAsync(w.data(), reinterpret_cast<void*>(ct), sizeof(u64) * w.size(),
                                         cudaMemcpyDeviceToHost, g.stream()), "ct download");
        g.synchronize();
        std::memset(buf, 0, need);
        std::memcpy(buf, "CSW1", 4);
        buf[4] = (uint8_t)P.cfg.logn;
        buf[5] = (uint8_t)P.cfg.L;
        const uint64_t fp = q_fingerprint(P);
        std::memcpy(buf + 8, &fp, 8);
        uint64_t bitpos = 0;
        uint8_t* out = buf + kWireHeader;
        for (int p = 0; p < 2; ++p)
            for (int j = 0; j < P.cfg.L; ++j) {
                const int nb = bitlen(P.primes[j]);
                const u64* src = w.data() + ((size_t)p * P.cfg.L + j) * P.n;
                for (int k = 0; k < P.n; ++k) {
                    u64 v = src[k];
                    if (v >= P.primes[j]) throw std::runtime_error("serialize: non-canonical residue");
                    for (int b = 0; b < nb;) {  // write nb bits, byte-aligned chunks
                        const int off = (int)(bitpos & 7), take = std::min(8 - off, nb - b);
                        out[bitpos >> 3] |= (uint8_t)((v & ((1u << take) - 1)) << off);
                        v >>= take;
                        b += take;
                        bitpos += (uint64_t)take;
                    }
                }
            }
        if (written) *written = need;
    });
}

int spmvgpu_ct_deserialize(spmvgpu_ctx* c, const uint8_t* buf, size_t len, spmvgpu_ct ct) {
    return guard([&] { auto lk_ = api_lock(c);
        auto& g = G(c);
        const auto& P = g.params();
        if (!buf || !ct) throw std::invalid_argument("null argument");
        if (len != wire_bytes(P)) throw std::invalid_argument("deserialize: wrong length for these parameters");
        uint64_t fp = 0;
        std::memcpy(&fp, buf + 8, 8);
        if (std::memcmp(buf, "CSW1", 4) != 0 || buf[4] != P.cfg.logn || buf[5] != P.cfg.L || fp != q_fingerprint(P))
            throw std::invalid_argument("deserialize: header does not match this context");
        std::vector<u64> w(g.ct_words());
        uint64_t bitpos = 0;
        const uint8_t* in = buf + kWireHeader;
        for (int p = 0; p < 2; ++p)
            for (int j = 0; j < P.cfg.L; ++j) {
                const int nb = bitlen(P.primes[j]);
                u64* dst = w.data() + ((size_t)p * P.cfg.L + j) * P.n;
                for (int k = 0; k < P.n; ++k) {
                    u64 v = 0;
                    for (int b = 0; b < nb;) {
                        const int off = (int)(bitpos & 7), take = std::min(8 - off, nb - b);
                        v |= (u64)((in[bitpos >> 3] >> off) & ((1u << take) - 1)) << b;
                        b += take;
                        bitpos += (uint64_t)take;
                    }
                    if (v >= P.primes[j]) throw std::invalid_argument("deserialize: residue out of range");
                    dst[k] = v;
                }
            }
        cssc::cuda_check(cudaMemcpyAsync(reinterpret_cast<void*>(ct), w.data(), sizeof(u64) * w.size(),
                                         cudaMemcpyHostToDevice, g.stream()), "ct upload");
        g.synchronize();
    });
}

int spmvgpu_encrypt(spmvgpu_ctx* c, const int64_t* vals, const uint64_t* offsets, const uint64_t* streams,
                    const spmvgpu_ct* out, size_t n) {
    return guard([&] { auto lk_ = api_lock(c);
        auto& g = G(c);
        std::vector<u64> st(n);
        for (size_t i = 0; i < n; ++i) st[i] = streams && streams[i] ? streams[i] : g.next_stream_id();
        g.encrypt(vals, offsets, st.data(), mptrs(out, n));
    });
}
int spmvgpu_encrypt_cssc(spmvgpu_ctx* c, const int64_t* col_indices, const int64_t* values, uint64_t nnz,
                         const int64_t* vec, uint64_t vec_len, const int32_t* rows, uint64_t n_rows,
                         const int32_t* slices, uint64_t n_slices, const int32_t* cols, uint64_t n_cols,
                         const spmvgpu_ct* out, size_t n_chunks) {
    return guard([&] { auto lk_ = api_lock(c);
        auto& g = G(c);
        // descriptor validation: the kernel trusts every index it reads
        const uint64_t S = g.params().S;
        for (uint64_t k = 0; k < n_cols; ++k) {
            const int32_t* cr = cols + 4 * k;
            if (cr[0] < -1 || cr[0] >= (int64_t)n_chunks || cr[1] < 0 || cr[2] <= 0 ||
                ((uint64_t)cr[1] + 1) * (uint64_t)cr[2] > S)
                throw std::invalid_argument("encrypt_cssc: column record out of range");
        }
        for (uint64_t s = 0; s < n_slices; ++s)
            if (slices[2 * s] < 0 || slices[2 * s + 1] < 0 || (uint64_t)slices[2 * s + 1] > vec_len)
                throw std::invalid_argument("encrypt_cssc: slice record out of range");
        for (uint64_t r = 0; r < n_rows; ++r) {
            const int32_t* rec = rows + 4 * r;
            if (rec[0] < 0 || rec[1] < 0 || (uint64_t)rec[0] + (uint64_t)rec[1] > nnz || rec[2] < 0 ||
                rec[3] < 0 || (uint64_t)rec[3] >= n_slices)
                throw std::invalid_argument("encrypt_cssc: row record out of range");
            const int32_t* sl = slices + 2 * rec[3];
            if ((uint64_t)sl[0] + (uint64_t)rec[1] > n_cols)
                throw std::invalid_argument("encrypt_cssc: row longer than its slice's aligned columns");
            const uint64_t vroom = vec_len - (uint64_t)sl[1];
            for (int32_t j = 0; j < rec[1]; ++j) {
                if (rec[2] >= cols[4 * (sl[0] + j) + 2])
                    throw std::invalid_argument("encrypt_cssc: row position beyond its chunk height");
                if ((uint64_t)col_indices[rec[0] + j] >= vroom)
                    throw spmv::IndexOutOfRangeError("encrypt_cssc: column index outside the vector");
            }
        }
        g.encrypt_cssc(col_indices, values, nnz, vec, vec_len, rows, n_rows, slices, n_slices, cols, n_cols,
                       mptrs(out, 2 * n_chunks));
    });
}
int spmvgpu_decrypt(spmvgpu_ctx* c, const spmvgpu_ct* cts, size_t n, uint64_t* slots, int32_t* budgets) {
    return guard([&] { auto lk_ = api_lock(c);
        std::vector<int> b(n);
        G(c).decrypt(cptrs(cts, n), slots, b.data());
        if (budgets)
            for (size_t i = 0; i < n; ++i) budgets[i] = b[i];
    });
}
int spmvgpu_add(spmvgpu_ctx* c, const spmvgpu_ct* a, const spmvgpu_ct* b, const spmvgpu_ct* out, size_t n) {
    return guard([&] { auto lk_ = api_lock(c); G(c).add(cptrs(a, n), cptrs(b, n), mptrs(out, n)); });
}
int spmvgpu_sum(spmvgpu_ctx* c, const spmvgpu_ct* cts, size_t n, spmvgpu_ct out) {
    return guard([&] { auto lk_ = api_lock(c);
        if (!out) throw std::invalid_argument("null output ciphertext");
        G(c).sum(cptrs(cts, n), reinterpret_cast<u64*>(out));
    });
}
int spmvgpu_mul_relin(spmvgpu_ctx* c, const spmvgpu_ct* a, const spmvgpu_ct* b, const spmvgpu_ct* out,
                      size_t n) {
    return guard([&] { auto lk_ = api_lock(c); G(c).mul_relin(cptrs(a, n), cptrs(b, n), mptrs(out, n)); });
}
int spmvgpu_rotate(spmvgpu_ctx* c, const spmvgpu_ct* src, const int64_t* steps, const spmvgpu_ct* out,
                   size_t n) {
    return guard([&] { auto lk_ = api_lock(c);
        G(c).rotate(cptrs(src, n), std::vector<int64_t>(steps, steps + n), std::vector<const u64*>(n, nullptr),
                    mptrs(out, n));
    });
}
int spmvgpu_rotate_add(spmvgpu_ctx* c, const spmvgpu_ct* acc, const spmvgpu_ct* src, const int64_t* steps,
                       const spmvgpu_ct* out, size_t n) {
    return guard([&] { auto lk_ = api_lock(c);
        auto o = mptrs(out, n);
        auto s = cptrs(src, n);
        for (size_t i = 0; i < n; ++i)
            if ((const u64*)o[i] == s[i]) throw std::invalid_argument("rotate_add: out must not alias src");
        G(c).rotate(s, std::vector<int64_t>(steps, steps + n), cptrs(acc, n), o);
    });
}
int spmvgpu_mul_plain(spmvgpu_ctx* c, const spmvgpu_ct* a, const int64_t* vals, const uint64_t* offsets,
                      const spmvgpu_ct* out, size_t n) {
    return guard([&] { auto lk_ = api_lock(c); G(c).mul_plain(cptrs(a, n), vals, offsets, mptrs(out, n)); });
}
int spmvgpu_ntt(spmvgpu_ctx* c, int prime_index, uint64_t* data, size_t limbs, int inverse) {
    return guard([&] { auto lk_ = api_lock(c);
        auto& g = G(c);
        if (prime_index < 0 || prime_index >= g.params().np) throw std::invalid_argument("prime index");
        g.ntt_host(prime_index, data, (int)limbs, inverse != 0);
    });
}

int spmvgpu_plan_create(spmvgpu_ctx* c, size_t n_chunks, const uint64_t* r, const uint64_t* cols,
                        const uint32_t* slice, size_t n_slices, const spmvgpu_ct* a_cts, const spmvgpu_ct* b_cts,
                        const spmvgpu_ct* out_cts, spmvgpu_plan** out) {
    return guard([&] { auto lk_ = api_lock(c);
        auto p = std::make_unique<spmvgpu_plan>();
        p->ctx = c;
        p->plan = std::make_unique<cssc::CloudPlan>(
            G(c), std::vector<uint64_t>(r, r + n_chunks), std::vector<uint64_t>(cols, cols + n_chunks),
            std::vector<uint32_t>(slice, slice + n_chunks), (int)n_slices, cptrs(a_cts, n_chunks),
            cptrs(b_cts, n_chunks), mptrs(out_cts, n_slices));
        *out = p.release();
    });
}
int spmvgpu_plan_run(spmvgpu_plan* p) { return guard([&] { auto lk_ = api_lock(p ? p->ctx : nullptr); p->plan->run(); }); }
int spmvgpu_plan_capture(spmvgpu_plan* p) { return guard([&] { auto lk_ = api_lock(p ? p->ctx : nullptr); p->plan->capture(); }); }
int spmvgpu_plan_stats_get(const spmvgpu_plan* p, spmvgpu_plan_stats* o) {
    return guard([&] { auto lk_ = api_lock(p ? p->ctx : nullptr);
        const auto& s = p->plan->stats();
        o->chunks = s.chunks;
        o->slices = s.slices;
        o->levels = s.levels;
        o->kernels_per_run = s.kernels;
        o->limb_ntts_per_run = s.limb_ntts;
        o->rotations = s.rotations;
        o->distinct_keys = s.distinct_keys;
        o->hbm_bytes_algorithmic = s.hbm_bytes;
        o->key_bytes_per_run = s.key_bytes;
        o->relin_folded = s.relin_folded;
    });
}
int spmvgpu_plan_profile(spmvgpu_plan* p, spmvgpu_phase* phases, int cap, int* count) {
    return guard([&] { auto lk_ = api_lock(p ? p->ctx : nullptr);
        if (!p || !count) throw std::invalid_argument("null argument");
        const auto ph = p->plan->profile();
        *count = (int)ph.size();
        for (int i = 0; i < (int)ph.size() && i < cap; ++i) {
            std::memset(&phases[i], 0, sizeof phases[i]);
            std::strncpy(phases[i].name, ph[i].name.c_str(), sizeof phases[i].name - 1);
            phases[i].us = ph[i].us;
            phases[i].items = ph[i].items;
            phases[i].bytes = ph[i].bytes;
            phases[i].limb_ntts = ph[i].limb_ntts;
            phases[i].sources = ph[i].sources;
            phases[i].acc_items = ph[i].acc_items;
            phases[i].mac_terms = ph[i].mac_terms;
        }
    });
}
int spmvgpu_plan_profile_kernels(spmvgpu_plan* p, int reps, uint64_t flush_bytes, spmvgpu_kernel_timing* out,
                                 int cap, int* count) {
    return guard([&] { auto lk_ = api_lock(p ? p->ctx : nullptr);
        if (!p || !count) throw std::invalid_argument("null argument");
        const auto kt = p->plan->profile_kernels(reps, flush_bytes);
        *count = (int)kt.size();
        for (int i = 0; i < (int)kt.size() && i < cap; ++i) {
            std::memset(&out[i], 0, sizeof out[i]);
            std::strncpy(out[i].name, kt[i].name.c_str(), sizeof out[i].name - 1);
            out[i].group = kt[i].group;
            out[i].us = kt[i].us;
        }
    });
}
void spmvgpu_plan_destroy(spmvgpu_plan* p) { delete p; }

// ---------------------------------------------------------------- protocol front door
int cssc_spmv_partitioned(spmvgpu_ctx* c, const cssc_csr* m, const int64_t* v, uint64_t vlen,
                          uint64_t chunk_size, int key_holder, int64_t* values, cssc_result* res,
                          cssc_message* msgs, uint64_t msg_cap) {
    return guard([&] { auto lk_ = api_lock(c);
        spmv::GpuBfvBackend be(c->hp, c);
        const spmv::CsrMatrix mm = to_csr(*m);
        const std::vector<int64_t> vv(v, v + vlen);
        const auto r = spmv::spmv_partitioned(be, mm, vv, chunk_size, static_cast<spmv::PartyRole>(key_holder));
        fill_result(r, values, res, msgs, msg_cap);
    });
}

int cssc_spmv(spmvgpu_ctx* c, const cssc_csr* m, const int64_t* v, uint64_t vlen, uint64_t chunk_size,
              int key_holder, int64_t* values, cssc_result* res, cssc_message* msgs, uint64_t msg_cap) {
    return guard([&] { auto lk_ = api_lock(c);
        spmv::GpuBfvBackend be(c->hp, c);
        const spmv::CsrMatrix mm = to_csr(*m);
        const std::vector<int64_t> vv(v, v + vlen);
        const auto r = spmv::spmv(be, mm, vv, chunk_size, static_cast<spmv::PartyRole>(key_holder));
        fill_result(r, values, res, msgs, msg_cap);
    });
}

int cssc_diag_spmv(spmvgpu_ctx* c, const cssc_csr* m, const int64_t* v, uint64_t vlen, int key_holder,
                   int64_t* values, cssc_result* res, cssc_message* msgs, uint64_t msg_cap) {
    return guard([&] { auto lk_ = api_lock(c);
        spmv::GpuBfvBackend be(c->hp, c);
        const spmv::CsrMatrix mm = to_csr(*m);
        const std::vector<int64_t> vv(v, v + vlen);
        const auto r = spmv::diag_spmv(be, mm, vv, static_cast<spmv::PartyRole>(key_holder));
        fill_result(r, values, res, msgs, msg_cap);
    });
}

int cssc_spmv_batch(spmvgpu_ctx* c, const cssc_csr* ms, const int64_t* const* vs, const uint64_t* vlens, size_t nmat,
                    uint64_t chunk_size, int key_holder, int64_t* const* values, cssc_result* res) {
    return guard([&] { auto lk_ = api_lock(c);
        G(c);
        static const bool trace = std::getenv("CSSC_TRACE_E2E") != nullptr;
        const auto t0 = std::chrono::steady_clock::now();
        // the previous call's plan: its early encryption graph runs while the
        // host packs (used only if this call's chunk shapes select that plan)
        static const bool spec = std::getenv("CSSC_NO_EARLY_ENC") == nullptr;
        if (spec && !c->spec_plan) spmv::detail::pipeline_speculate(c);  // unless cssc_speculate did
        const auto t0s = std::chrono::steady_clock::now();
        if (nmat && (!ms || !vs || !vlens)) throw std::invalid_argument("null argument");
        std::vector<spmv::detail::CsrView> w;
        for (size_t i = 0; i < nmat; ++i) w.push_back(view_of(ms[i], vs[i], vlens[i]));
        spmv::detail::BatchedSpmv job(c, c->hp, w, chunk_size, static_cast<spmv::PartyRole>(key_holder));
        const auto t1 = std::chrono::steady_clock::now();
        const auto r = job.run_all(values);
        const auto t2 = std::chrono::steady_clock::now();
        for (size_t i = 0; i < nmat; ++i) fill_result(r[i], values ? values[i] : nullptr, res ? res + i : nullptr, nullptr, 0);
        if (trace) {
            const auto t3 = std::chrono::steady_clock::now();
            auto us = [](auto a, auto b) { return std::chrono::duration<double, std::micro>(b - a).count(); };
            std::fprintf(stderr, "e2e-trace speculate %.1f pack %.1f run %.1f fill %.1f us\n", us(t0, t0s),
                         us(t0s, t1), us(t1, t2), us(t2, t3));
        }
    });
}

int cssc_speculate(spmvgpu_ctx* c) {
    return guard([&] { auto lk_ = api_lock(c);
        G(c);
        static const bool spec = std::getenv("CSSC_NO_EARLY_ENC") == nullptr;
        if (spec) spmv::detail::pipeline_speculate(c);
    });
}

int cssc_job_create_shard(spmvgpu_ctx* c, const cssc_csr* ms, const int64_t* const* vs, const uint64_t* vlens,
                          size_t nmat, uint64_t chunk_size, int rank, int world, cssc_job** out) {
    return guard([&] { auto lk_ = api_lock(c);
        auto j = std::make_unique<cssc_job>();
        j->ctx = c;
        G(c);
        if (nmat && (!ms || !vs || !vlens)) throw std::invalid_argument("null argument");
        std::vector<spmv::detail::CsrView> w;
        for (size_t i = 0; i < nmat; ++i) w.push_back(view_of(ms[i], vs[i], vlens[i]));
        j->job = std::make_unique<spmv::detail::BatchedSpmv>(c, c->hp, w, chunk_size, spmv::PartyRole::ClientA,
                                                             true, rank, world);
        *out = j.release();
    });
}
int cssc_job_create(spmvgpu_ctx* c, const cssc_csr* ms, const int64_t* const* vs, const uint64_t* vlens, size_t nmat,
                    uint64_t chunk_size, cssc_job** out) {
    return cssc_job_create_shard(c, ms, vs, vlens, nmat, chunk_size, 0, 1, out);
}
int cssc_job_result_words(cssc_job* j, uint64_t* words, uint64_t cap_words, uint64_t* n_results) {
    return guard([&] { auto lk_ = api_lock(j ? j->ctx : nullptr);
        if (!j || !n_results) throw std::invalid_argument("null argument");
        *n_results = j->job->result_count();
        if (!words) return;
        const auto w = j->job->result_words();
        if (cap_words < w.size()) throw std::length_error("result_words: buffer too small");
        std::memcpy(words, w.data(), sizeof(uint64_t) * w.size());
    });
}
int cssc_job_finish_words(cssc_job* j, const uint64_t* words, int64_t* const* values, cssc_result* res) {
    return guard([&] { auto lk_ = api_lock(j ? j->ctx : nullptr);
        if (!j || (!words && j->job->result_count())) throw std::invalid_argument("null argument");
        const auto r = j->job->finish_words(words);
        for (size_t i = 0; i < r.size(); ++i) fill_result(r[i], values ? values[i] : nullptr, res ? res + i : nullptr, nullptr, 0);
    });
}
int cssc_job_result_words_dev(cssc_job* j, uint64_t* dev_words, uint64_t cap_words, uint64_t* n_results) {
    return guard([&] { auto lk_ = api_lock(j ? j->ctx : nullptr);
        if (!j || !n_results) throw std::invalid_argument("null argument");
        *n_results = j->job->result_count();
        if (!dev_words) return;
        if (cap_words < *n_results * G(j->ctx).ct_words()) throw std::length_error("result_words_dev: buffer too small");
        j->job->result_words_dev(dev_words);
    });
}
int cssc_job_finish_words_dev(cssc_job* j, uint64_t* dev_words, int64_t* const* values, cssc_result* res) {
    return guard([&] { auto lk_ = api_lock(j ? j->ctx : nullptr);
        if (!j || (!dev_words && j->job->result_count())) throw std::invalid_argument("null argument");
        const auto r = j->job->finish_words_dev(dev_words);
        for (size_t i = 0; i < r.size(); ++i) fill_result(r[i], values ? values[i] : nullptr, res ? res + i : nullptr, nullptr, 0);
    });
}
int spmvgpu_fold_mod(spmvgpu_ctx* c, uint64_t* dev_words, uint64_t n_cts) {
    return guard([&] { auto lk_ = api_lock(c);
        auto& g = G(c);
        cssc::launch_fold_mod(g.dconsts(), g.params(), dev_words, (int)n_cts, g.stream());
        g.synchronize();
    });
}
int cssc_job_encrypt(cssc_job* j) { return guard([&] { auto lk_ = api_lock(j ? j->ctx : nullptr); j->job->encrypt(); }); }
int cssc_job_cloud(cssc_job* j, int use_graph) { return guard([&] { auto lk_ = api_lock(j ? j->ctx : nullptr); j->job->cloud(use_graph != 0); }); }
int cssc_job_cloud_timed(cssc_job* j, int use_graph, void* ev_start, void* ev_stop) {
    return guard([&] { auto lk_ = api_lock(j ? j->ctx : nullptr);
        if (!j || !ev_start || !ev_stop) throw std::invalid_argument("null argument");
        cudaStream_t st = j->ctx->g->stream();
        cssc::cuda_check(cudaEventRecord(static_cast<cudaEvent_t>(ev_start), st), "event record");
        j->job->cloud(use_graph != 0);
        cssc::cuda_check(cudaEventRecord(static_cast<cudaEvent_t>(ev_stop), st), "event record");
    });
}
int cssc_job_finish(cssc_job* j, int64_t* const* values, cssc_result* res) {
    return guard([&] { auto lk_ = api_lock(j ? j->ctx : nullptr);
        const auto r = j->job->finish();
        for (size_t i = 0; i < r.size(); ++i) fill_result(r[i], values ? values[i] : nullptr, res ? res + i : nullptr, nullptr, 0);
    });
}
int cssc_job_run(cssc_job* j, int64_t* const* values, cssc_result* res) {
    return guard([&] { auto lk_ = api_lock(j ? j->ctx : nullptr);
        const auto r = j->job->run_all(values);
        for (size_t i = 0; i < r.size(); ++i) fill_result(r[i], values ? values[i] : nullptr, res ? res + i : nullptr, nullptr, 0);
    });
}
int cssc_job_plan_stats(const cssc_job* j, spmvgpu_plan_stats* out) {
    return guard([&] { auto lk_ = api_lock(j ? j->ctx : nullptr);
        std::memset(out, 0, sizeof *out);
        if (j->job->plan()) spmvgpu_plan_stats_get(j->job->plan(), out);
    });
}
int cssc_job_profile(cssc_job* j, spmvgpu_phase* phases, int cap, int* count) {
    return guard([&] { auto lk_ = api_lock(j ? j->ctx : nullptr);
        if (!j || !j->job->plan()) throw std::invalid_argument("job has no plan yet (run cloud first)");
        const int st = spmvgpu_plan_profile(j->job->plan(), phases, cap, count);
        if (st != SPMVGPU_OK) throw std::runtime_error(g_err);
    });
}
int cssc_job_profile_kernels(cssc_job* j, int reps, uint64_t flush_bytes, spmvgpu_kernel_timing* out, int cap,
                             int* count) {
    return guard([&] { auto lk_ = api_lock(j ? j->ctx : nullptr);
        if (!j || !j->job->plan()) throw std::invalid_argument("job has no plan yet (run cloud first)");
        const int st = spmvgpu_plan_profile_kernels(j->job->plan(), reps, flush_bytes, out, cap, count);
        if (st != SPMVGPU_OK) throw std::runtime_error(g_err);
    });
}
int cssc_job_input_bytes(const cssc_job* j, uint64_t* h2d, uint64_t* d2h) {
    return guard([&] { auto lk_ = api_lock(j ? j->ctx : nullptr);
        *h2d = j->job->h2d_bytes();
        *d2h = j->job->d2h_bytes();
    });
}
void cssc_job_destroy(cssc_job* j) { delete j; }

int64_t cssc_pack_chunks(const cssc_csr* m, uint64_t budget, int64_t* r_list, int64_t* c_list, int64_t* vflat,
                         int64_t* cflat, int64_t* row_map, uint64_t* flat_total) {
    int64_t n = 0;
    const int st = guard([&] {
        const auto cs = spmv::generate_chunks(spmv::csr_to_cssc(to_csr(*m)), budget);
        uint64_t tot = 0;
        for (const auto& ch : cs.chunks) tot += ch.value_flat.size();
        *flat_total = tot;
        if (r_list) {
            uint64_t off = 0;
            for (size_t i = 0; i < cs.n_ct(); ++i) {
                r_list[i] = (int64_t)cs.r_list[i];
                c_list[i] = (int64_t)cs.c_list[i];
                std::memcpy(vflat + off, cs.chunks[i].value_flat.data(), 8 * cs.chunks[i].value_flat.size());
                std::memcpy(cflat + off, cs.chunks[i].colidx_flat.data(), 8 * cs.chunks[i].colidx_flat.size());
                off += cs.chunks[i].value_flat.size();
            }
            for (size_t i = 0; i < cs.row_map.size(); ++i) row_map[i] = (int64_t)cs.row_map[i];
        }
        n = (int64_t)cs.n_ct();
    });
    return st == SPMVGPU_OK ? n : st;
}

int cssc_rotation_schedule(uint64_t rows, uint64_t cols, uint64_t* offsets, int32_t* from_acc) {
    int n = 0;
    const int st = guard([&] {
        const auto s = spmv::rotation_schedule(rows, cols);
        for (size_t i = 0; i < s.size(); ++i) {
            if (offsets) offsets[i] = s[i].offset;
            if (from_acc) from_acc[i] = s[i].from_accumulator ? 1 : 0;
        }
        n = (int)s.size();
    });
    return st == SPMVGPU_OK ? n : st;
}

static spmv::CsscMatrix converted(const cssc_csr* m) {
    if (!m) throw std::invalid_argument("null matrix");
    spmv::CsscMatrix c = spmv::csr_to_cssc(to_csr(*m));
    const auto bad = spmv::validate_cssc(c);
    if (!bad.empty()) throw std::runtime_error("conversion produced an invalid structure: " + bad.front());
    return c;
}
int cssc_convert_binary(const cssc_csr* m, uint8_t* buf, uint64_t cap, uint64_t* written) {
    return guard([&] {
        if (!written) throw std::invalid_argument("null argument");
        const auto bytes = spmv::cssc_to_bytes(converted(m));
        *written = bytes.size();
        if (!buf) return;
        if (cap < bytes.size()) throw std::length_error("convert: buffer too small");
        std::memcpy(buf, bytes.data(), bytes.size());
    });
}
int cssc_convert_json(const cssc_csr* m, char* buf, uint64_t cap, uint64_t* written) {
    return guard([&] {
        if (!written) throw std::invalid_argument("null argument");
        const std::string j = spmv::cssc_to_json(converted(m));
        *written = j.size();
        if (!buf) return;
        if (cap < j.size()) throw std::length_error("convert: buffer too small");
        std::memcpy(buf, j.data(), j.size());
    });
}
int cssc_load_binary(const uint8_t* buf, uint64_t len, uint64_t* rows, uint64_t* cols, uint64_t* nnz,
                     uint64_t* aligned_cols, int64_t* va, uint64_t* ci, uint64_t* rm, uint64_t* cp) {
    return guard([&] {
        if (!buf || !rows || !cols || !nnz || !aligned_cols) throw std::invalid_argument("null argument");
        const spmv::CsscMatrix c = spmv::cssc_from_bytes(std::span<const uint8_t>(buf, len));
        *rows = c.rows;
        *cols = c.cols;
        *nnz = c.nnz();
        *aligned_cols = c.aligned_cols();
        if (va && !c.va.empty()) std::memcpy(va, c.va.data(), 8 * c.va.size());
        if (ci) for (size_t k = 0; k < c.ci.size(); ++k) ci[k] = c.ci[k];
        if (rm) for (size_t k = 0; k < c.rm.size(); ++k) rm[k] = c.rm[k];
        if (cp) for (size_t k = 0; k < c.cp.size(); ++k) cp[k] = c.cp[k];
    });
}

}  // extern "C"

extern "C" {

int spmvgpu_probe_ntt(spmvgpu_ctx* c, size_t limbs, int inverse, int reps, double* us_per_launch) {
    return guard([&] { auto lk_ = api_lock(c);
        auto& g = G(c);
        const auto& P = g.params();
        cssc::DevBuf buf(&g.pool(), sizeof(u64) * limbs * P.n);
        cssc::cuda_check(cudaMemsetAsync(buf.words(), 0, buf.bytes(), g.stream()), "memset");
        std::vector<int> pidx;
        for (int j = 0; j < P.cfg.L; ++j) pidx.push_back(j);
        // `limbs` CTAs as (limbs / L) items of L limbs, primes cycling over Q
        const cssc::NttJob job = g.job(buf.words(), buf.words(), P.cfg.L, pidx);
        const int items = (int)std::max<size_t>(1, limbs / P.cfg.L);
        cssc::launch_ntt(g.dconsts(), P.cfg.logn, inverse != 0, job, items, g.stream());
        g.synchronize();
        cudaEvent_t a = nullptr, b = nullptr;
        cssc::cuda_check(cudaEventCreate(&a), "event");
        cssc::cuda_check(cudaEventCreate(&b), "event");
        cssc::cuda_check(cudaEventRecord(a, g.stream()), "event record");
        for (int r = 0; r < reps; ++r) cssc::launch_ntt(g.dconsts(), P.cfg.logn, inverse != 0, job, items, g.stream());
        cssc::cuda_check(cudaEventRecord(b, g.stream()), "event record");
        cssc::cuda_check(cudaEventSynchronize(b), "probe ntt");
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        cudaEventDestroy(a);
        cudaEventDestroy(b);
        *us_per_launch = 1e3 * ms / reps;
    });
}

int spmvgpu_probe_butterfly_peak(spmvgpu_ctx* c, double* bps) {
    return guard([&] { auto lk_ = api_lock(c);
        auto& g = G(c);
        const auto& P = g.params();
        const u64 q = P.primes[0], w = P.tw_fwd[0][2], wsh = P.tw_fwd[0][3];
        *bps = cssc::probe_butterfly_peak(nullptr, q, w, wsh, g.stream());
    });
}

}  // extern "C"
