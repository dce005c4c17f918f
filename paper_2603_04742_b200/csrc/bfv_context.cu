// bfv_context.cu -- see bfv_context.hpp.
#include "bfv_context.hpp"

#include <algorithm>
#include <climits>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>

namespace cssc {

void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}

// ------------------------------------------------------------------ pool
DevicePool::~DevicePool() { trim(); }

void* DevicePool::alloc(size_t bytes) {
    {
        std::lock_guard<std::mutex> g(mu_);
        auto it = free_.find(bytes);
        if (it != free_.end()) {
            void* p = it->second;
            free_.erase(it);
            return p;
        }
    }
    void* p = nullptr;
    cudaError_t e = cudaMalloc(&p, bytes);
    if (e != cudaSuccess) {
        cudaGetLastError();
        trim();
        cuda_check(cudaMalloc(&p, bytes), "cudaMalloc");
    }
    return p;
}

void DevicePool::release(void* p, size_t bytes) {
    std::lock_guard<std::mutex> g(mu_);
    free_.emplace(bytes, p);
}

void DevicePool::trim() {
    std::lock_guard<std::mutex> g(mu_);
    for (auto& kv : free_) cudaFree(kv.second);
    free_.clear();
}

DevBuf::DevBuf(DevicePool* pool, size_t bytes) : pool_(pool), bytes_(bytes) {
    ptr_ = bytes ? pool->alloc(bytes) : nullptr;
}
DevBuf::~DevBuf() {
    if (ptr_) pool_->release(ptr_, bytes_);
}
DevBuf::DevBuf(DevBuf&& o) noexcept : pool_(o.pool_), ptr_(o.ptr_), bytes_(o.bytes_) {
    o.ptr_ = nullptr;
    o.bytes_ = 0;
}
DevBuf& DevBuf::operator=(DevBuf&& o) noexcept {
    if (this != &o) {
        if (ptr_) pool_->release(ptr_, bytes_);
        pool_ = o.pool_;
        ptr_ = o.ptr_;
        bytes_ = o.bytes_;
        o.ptr_ = nullptr;
        o.bytes_ = 0;
    }
    return *this;
}
void DevBuf::ensure(DevicePool* pool, size_t bytes) {
    if (bytes <= bytes_) return;
    // all work is ordered on the context stream, so releasing to the pool is safe
    if (ptr_) pool_->release(ptr_, bytes_);
    pool_ = pool;
    ptr_ = pool->alloc(bytes);
    bytes_ = bytes;
}

// ------------------------------------------------------------------ context
GpuContext::GpuContext(const RnsConfig& cfg, int device) : P_(cfg), device_(device) {
    cuda_check(cudaSetDevice(device), "cudaSetDevice");
    cuda_check(cudaStreamCreateWithFlags(&st_, cudaStreamNonBlocking), "stream");
    cuda_check(cudaStreamCreateWithFlags(&st2_, cudaStreamNonBlocking), "stream");
    cuda_check(cudaEventCreateWithFlags(&ev_fork_, cudaEventDisableTiming), "event");
    cuda_check(cudaEventCreateWithFlags(&ev_join_, cudaEventDisableTiming), "event");
    cuda_check(cudaEventCreateWithFlags(&ev_upload_, cudaEventDisableTiming), "event");
    DevConsts host = P_.host;
    const size_t tw_bytes = sizeof(u64) * 2 * (size_t)P_.n;
    for (int i = 0; i < P_.np; ++i) {
        DevBuf f(&pool_, tw_bytes), v(&pool_, tw_bytes);
        cuda_check(cudaMemcpy(f.words(), P_.tw_fwd[i].data(), tw_bytes, cudaMemcpyHostToDevice), "tw");
        cuda_check(cudaMemcpy(v.words(), P_.tw_inv[i].data(), tw_bytes, cudaMemcpyHostToDevice), "tw");
        host.tw[i].fwd = f.words();
        host.tw[i].inv = v.words();
        tables_.push_back(std::move(f));
        tables_.push_back(std::move(v));
    }
    pos0_ = DevBuf(&pool_, sizeof(u32) * P_.S);
    cuda_check(cudaMemcpy(pos0_.as<u32>(), P_.pos0.data(), sizeof(u32) * P_.S, cudaMemcpyHostToDevice),
               "pos0");
    host.pos0 = pos0_.as<u32>();
    cuda_check(cudaMalloc(&dc_, sizeof(DevConsts)), "consts");
    cuda_check(cudaMemcpy(dc_, &host, sizeof(DevConsts), cudaMemcpyHostToDevice), "consts");
    keygen();
    synchronize();
}

GpuContext::~GpuContext() {
    if (st_) cudaStreamSynchronize(st_);
    if (stage_ev_) cudaEventDestroy(stage_ev_);
    if (stage_) cudaFreeHost(stage_);
    for (auto& kv : pinned_free_) cudaFreeHost(kv.second);
    // buffers release into pool_; pool_ destructor frees device memory
    gk_.clear();
    gk2_.clear();
    if (dc_) cudaFree(dc_);
    if (ev_fork_) cudaEventDestroy(ev_fork_);
    if (ev_join_) cudaEventDestroy(ev_join_);
    if (ev_upload_) cudaEventDestroy(ev_upload_);
    if (st2_) cudaStreamDestroy(st2_);
    if (st_) cudaStreamDestroy(st_);
}

void GpuContext::synchronize() { cuda_check(cudaStreamSynchronize(st_), "stream sync"); }

void* GpuContext::upload_bytes(const void* src, size_t bytes, int slot) {
    ensure_ws(scratch_[slot], std::max<size_t>(bytes, 256));
    if (bytes)
        cuda_check(cudaMemcpyAsync(scratch_[slot].as<void>(), src, bytes, cudaMemcpyHostToDevice, st_),
                   "upload");
    return scratch_[slot].as<void>();
}

unsigned char* GpuContext::stage_host(size_t bytes) {
    if (stage_ev_) cuda_check(cudaEventSynchronize(stage_ev_), "staging wait");
    if (bytes > stage_bytes_) {
        if (stage_) cuda_check(cudaFreeHost(stage_), "cudaFreeHost");
        stage_ = nullptr;
        const size_t cap = std::max<size_t>(bytes + bytes / 2, 1 << 20);
        cuda_check(cudaHostAlloc(reinterpret_cast<void**>(&stage_), cap, cudaHostAllocDefault), "cudaHostAlloc");
        stage_bytes_ = cap;
    }
    if (!stage_ev_) cuda_check(cudaEventCreateWithFlags(&stage_ev_, cudaEventDisableTiming), "event");
    return stage_;
}

void* GpuContext::stage_upload(size_t bytes, int slot) {
    ensure_ws(scratch_[slot], std::max<size_t>(bytes, 256));
    cuda_check(cudaMemcpyAsync(scratch_[slot].as<void>(), stage_, bytes, cudaMemcpyHostToDevice, st_), "upload");
    cuda_check(cudaEventRecord(stage_ev_, st_), "event");
    return scratch_[slot].as<void>();
}

template <class T>
T* GpuContext::upload_ptrs(const std::vector<T>& v, int slot) {
    return static_cast<T*>(upload_bytes(v.data(), sizeof(T) * v.size(), slot));
}

NttJob GpuContext::job(const u64* src, u64* dst, int limbs, const std::vector<int>& pidx) const {
    NttJob j;
    std::memset(j.pidx, 0, sizeof j.pidx);
    j.src = src;
    j.dst = dst;
    j.limbs = limbs;
    if (limbs > MAX_JOB_LIMBS || limbs < 1) throw std::invalid_argument("NTT job limb count out of range");
    for (int p : pidx)
        if (p < 0 || p >= P_.np) throw std::invalid_argument("NTT job prime index out of range");
    for (int i = 0; i < limbs; ++i) j.pidx[i] = (signed char)pidx[i % pidx.size()];
    return j;
}

static std::vector<int> range_idx(int lo, int hi) {
    std::vector<int> v;
    for (int i = lo; i < hi; ++i) v.push_back(i);
    return v;
}

// ------------------------------------------------------------------ keys
void GpuContext::keygen() {
    const int n = P_.n, L = P_.cfg.L, LK = L + P_.cfg.K, logn = P_.cfg.logn;
    const SeedKey seed = P_.cfg.key;
    s_small_ = DevBuf(&pool_, sizeof(int64_t) * n);
    launch_sample_small(logn, seed, DOM_SK, 0, 0, s_small_.as<int64_t>(), st_);
    s_ntt_ = DevBuf(&pool_, sizeof(u64) * (size_t)LK * n);
    launch_lift_small(dc_, logn, s_small_.as<int64_t>(), LK, 0, s_ntt_.words(), st_);
    launch_ntt(dc_, logn, false, job(s_ntt_.words(), s_ntt_.words(), LK, range_idx(0, LK)), 1, st_);

    // public key over Q: pk1 = a, pk0 = -(a s + e)
    pk_ = DevBuf(&pool_, sizeof(u64) * 2 * (size_t)L * n);
    u64* pk0 = pk_.words();
    u64* pk1 = pk_.words() + (size_t)L * n;
    launch_sample_uniform(dc_, logn, seed, DOM_PK_A, 0, 0, L, 0, pk1, st_);
    launch_ntt(dc_, logn, false, job(pk1, pk1, L, range_idx(0, L)), 1, st_);
    DevBuf e_small(&pool_, sizeof(int64_t) * n), E(&pool_, sizeof(u64) * (size_t)L * n);
    launch_sample_small(logn, seed, DOM_PK_E, 0, 1, e_small.as<int64_t>(), st_);
    launch_lift_small(dc_, logn, e_small.as<int64_t>(), L, 0, E.words(), st_);
    launch_ntt(dc_, logn, false, job(E.words(), E.words(), L, range_idx(0, L)), 1, st_);
    launch_key_combine(dc_, logn, L, pk1, E.words(), s_ntt_.words(), nullptr, 0, 0, pk0, st_);

    // Shoup companions of the fixed multipliers of encryption (pk) and decryption (s)
    pk_sh_ = DevBuf(&pool_, sizeof(u64) * 2 * (size_t)L * n);
    launch_shoup_companions(dc_, pk_.words(), pk_sh_.words(), L, n, 2, st_);
    s_sh_ = DevBuf(&pool_, sizeof(u64) * (size_t)L * n);
    launch_shoup_companions(dc_, s_ntt_.words(), s_sh_.words(), L, n, 1, st_);

    // relinearisation key: target s^2
    DevBuf s2(&pool_, sizeof(u64) * (size_t)LK * n);
    launch_square(dc_, logn, LK, s_ntt_.words(), s2.words(), st_);
    rlk_ = gen_ksk(0, s2.words());
    synchronize();
}

DevBuf GpuContext::gen_ksk(u64 keyid, const u64* sp_ntt) {
    const int n = P_.n, L = P_.cfg.L, LK = L + P_.cfg.K, logn = P_.cfg.logn;
    const SeedKey seed = P_.cfg.key;
    // [dnum][2][L+K][N] key words, then their Shoup companions (the fused MAC)
    DevBuf key(&pool_, sizeof(u64) * 2 * ksk_words());
    DevBuf e_small(&pool_, sizeof(int64_t) * n), E(&pool_, sizeof(u64) * (size_t)LK * n);
    for (int d = 0; d < P_.dnum; ++d) {
        u64* k0 = key.words() + ((size_t)d * 2 + 0) * LK * n;
        u64* k1 = key.words() + ((size_t)d * 2 + 1) * LK * n;
        launch_sample_uniform(dc_, logn, seed, DOM_KSK_A, d, keyid, LK, 0, k1, st_);
        launch_ntt(dc_, logn, false, job(k1, k1, LK, range_idx(0, LK)), 1, st_);
        launch_sample_small(logn, seed, DOM_KSK_E | ((u32)d << 16), keyid, 1, e_small.as<int64_t>(), st_);
        launch_lift_small(dc_, logn, e_small.as<int64_t>(), LK, 0, E.words(), st_);
        launch_ntt(dc_, logn, false, job(E.words(), E.words(), LK, range_idx(0, LK)), 1, st_);
        const int lo = d * P_.cfg.alpha, hi = std::min(lo + P_.cfg.alpha, L);
        launch_key_combine(dc_, logn, LK, k1, E.words(), s_ntt_.words(), sp_ntt, lo, hi, k0, st_);
    }
    launch_shoup_companions(dc_, key.words(), key.words() + ksk_words(), LK, n, 2 * P_.dnum, st_);
    return key;
}

const u64* GpuContext::galois_key(u32 g) {
    std::lock_guard<std::mutex> lk(mu_);
    auto it = gk_.find(g);
    if (it != gk_.end()) return it->second.words();
    const int n = P_.n, LK = P_.cfg.L + P_.cfg.K, logn = P_.cfg.logn;
    DevBuf sg(&pool_, sizeof(int64_t) * n), sp(&pool_, sizeof(u64) * (size_t)LK * n);
    launch_automorph_small(logn, g, s_small_.as<int64_t>(), sg.as<int64_t>(), st_);
    launch_lift_small(dc_, logn, sg.as<int64_t>(), LK, 0, sp.words(), st_);
    launch_ntt(dc_, logn, false, job(sp.words(), sp.words(), LK, range_idx(0, LK)), 1, st_);
    DevBuf key = gen_ksk(g, sp.words());
    const u64* p = key.words();
    gk_.emplace(g, std::move(key));
    return p;
}

const u64* GpuContext::galois_key_sq(u32 g) {
    std::lock_guard<std::mutex> lk(mu_);
    auto it = gk2_.find(g);
    if (it != gk2_.end()) return it->second.words();
    const int n = P_.n, LK = P_.cfg.L + P_.cfg.K, logn = P_.cfg.logn;
    DevBuf sg(&pool_, sizeof(int64_t) * n), sp(&pool_, sizeof(u64) * (size_t)LK * n),
        sp2(&pool_, sizeof(u64) * (size_t)LK * n);
    launch_automorph_small(logn, g, s_small_.as<int64_t>(), sg.as<int64_t>(), st_);
    launch_lift_small(dc_, logn, sg.as<int64_t>(), LK, 0, sp.words(), st_);
    launch_ntt(dc_, logn, false, job(sp.words(), sp.words(), LK, range_idx(0, LK)), 1, st_);
    launch_square(dc_, logn, LK, sp.words(), sp2.words(), st_);
    DevBuf key = gen_ksk(((u64)1 << 32) | g, sp2.words());
    const u64* p = key.words();
    gk2_.emplace(g, std::move(key));
    return p;
}

void GpuContext::ensure_galois_keys(const std::vector<int64_t>& steps) {
    for (int64_t k : steps) {
        const u32 g = galois_element(k, P_.n);
        if (g != 1) galois_key(g);
    }
}

void GpuContext::download_sk(int64_t* out) {
    synchronize();
    cuda_check(cudaMemcpy(out, s_small_.as<int64_t>(), sizeof(int64_t) * P_.n, cudaMemcpyDeviceToHost), "sk");
}

void GpuContext::download_pk_coef(u64* out) {
    const int L = P_.cfg.L;
    DevBuf tmp(&pool_, sizeof(u64) * 2 * (size_t)L * P_.n);
    launch_ntt(dc_, P_.cfg.logn, true, job(pk_.words(), tmp.words(), 2 * L, range_idx(0, L)), 1, st_);
    synchronize();
    cuda_check(cudaMemcpy(out, tmp.words(), tmp.bytes(), cudaMemcpyDeviceToHost), "pk");
}

void GpuContext::download_key_coef(u32 which, u64* out) {
    const int LK = P_.cfg.L + P_.cfg.K;
    const u64* key = which == 0 ? rlk_.words() : galois_key(which);
    DevBuf tmp(&pool_, sizeof(u64) * ksk_words());
    launch_ntt(dc_, P_.cfg.logn, true, job(key, tmp.words(), 2 * P_.dnum * LK, range_idx(0, LK)), 1,
               st_);
    synchronize();
    cuda_check(cudaMemcpy(out, tmp.words(), tmp.bytes(), cudaMemcpyDeviceToHost), "ksk");
}

// ------------------------------------------------------------------ encrypt / decrypt
void GpuContext::encrypt(const int64_t* vals, const u64* offs, const u64* streams,
                         const std::vector<u64*>& out) {
    const int items = (int)out.size();
    if (!items) return;
    for (int i = 0; i < items; ++i)
        if (offs[i + 1] - offs[i] > (u64)P_.S) throw std::length_error("encode: values exceed slot count");
    auto* dv = static_cast<int64_t*>(upload_bytes(vals, sizeof(int64_t) * offs[items], 0));
    auto* doff = static_cast<u64*>(upload_bytes(offs, sizeof(u64) * (items + 1), 1));
    auto* dst = static_cast<u64*>(upload_bytes(streams, sizeof(u64) * items, 2));
    auto* dout = upload_ptrs(out, 3);
    encrypt_dev(dv, doff, dst, dout, items);
}

void GpuContext::encrypt_dev(const int64_t* d_vals, const u64* d_offs, const u64* d_streams,
                             u64* const* d_out, int items) {
    u64* CM = enc_workspace(items);
    launch_encode_scatter(dc_, P_, d_vals, d_offs, CM + (size_t)2 * P_.cfg.L * P_.n, items, st_, cm_stride());
    encrypt_encoded(d_streams, d_out, items);
}

u64* GpuContext::enc_workspace(int items) {
    ensure_ws(wsU_, sizeof(u64) * (size_t)items * P_.cfg.L * P_.n);
    ensure_ws(wsC_, sizeof(u64) * (size_t)items * cm_stride());
    return wsC_.words();
}

CsscLayout CsscLayout::make(size_t nnz, size_t vec_len, size_t n_rows, size_t n_slices, size_t n_cols, int items,
                            int ci_w, int va_w, int v_w) {
    if ((ci_w != 2 && ci_w != 4 && ci_w != 8) || (va_w != 1 && va_w != 8) || (v_w != 1 && v_w != 8))
        throw std::invalid_argument("client image: unsupported element width");
    CsscLayout l;
    l.ci_w = ci_w;
    l.va_w = va_w;
    l.v_w = v_w;
    size_t off = 0;
    auto place = [&](size_t b) {
        const size_t o = off;
        off += (b + 15) & ~size_t(15);
        return o;
    };
    l.o_ci = place((size_t)ci_w * nnz);
    l.o_va = place((size_t)va_w * nnz);
    l.o_v = place((size_t)v_w * vec_len);
    l.o_rows = place(16 * n_rows);
    l.o_rpre = place(4 * (n_rows + 1));  // exclusive prefix of the row lengths (+ total)
    l.o_sl = place(8 * n_slices);
    l.o_cols = place(16 * n_cols);
    l.o_st = place(8 * (size_t)items);
    l.o_out = place(8 * (size_t)items);
    l.bytes = off;
    l.nnz = nnz;
    l.entries = nnz;
    l.vec_len = vec_len;
    l.n_rows = n_rows;
    l.n_slices = n_slices;
    l.n_cols = n_cols;
    l.items = items;
    return l;
}

unsigned char* GpuContext::pinned_take(size_t bytes, size_t* cap) {
    {
        std::lock_guard<std::mutex> g(mu_);
        auto it = pinned_free_.lower_bound(bytes);
        if (it != pinned_free_.end() && it->first <= 2 * bytes + (1 << 20)) {
            unsigned char* p = it->second;
            *cap = it->first;
            pinned_free_.erase(it);
            return p;
        }
    }
    const size_t c = std::max<size_t>(bytes, 1 << 16);
    unsigned char* p = nullptr;
    cuda_check(cudaHostAlloc(reinterpret_cast<void**>(&p), c, cudaHostAllocDefault), "cudaHostAlloc");
    *cap = c;
    return p;
}

void GpuContext::pinned_give(unsigned char* p, size_t cap) {
    if (!p) return;
    std::lock_guard<std::mutex> g(mu_);
    pinned_free_.emplace(cap, p);
}

void GpuContext::encrypt_cssc(const int64_t* ci, const int64_t* va, size_t nnz, const int64_t* vec,
                              size_t vec_len, const int32_t* rows, size_t n_rows, const int32_t* slices,
                              size_t n_slices, const int32_t* cols, size_t n_cols, const std::vector<u64*>& out) {
    const int items = (int)out.size();
    if (!items) return;
    if (items % 2) throw std::invalid_argument("encrypt_cssc: expects value and vector chunks in pairs");
    if (nnz > (size_t)INT32_MAX || vec_len > (size_t)INT32_MAX || n_rows > (size_t)INT32_MAX)
        throw std::length_error("encrypt_cssc: batch too large for 32-bit descriptors");
    CsscLayout lay = CsscLayout::make(nnz, vec_len, n_rows, n_slices, n_cols, items);
    unsigned char* h = stage_host(lay.bytes);
    {
        auto* pre = reinterpret_cast<int32_t*>(h + lay.o_rpre);
        int64_t acc = 0;
        for (size_t r = 0; r < n_rows; ++r) {
            pre[r] = (int32_t)acc;
            acc += rows[4 * r + 1];
            if (acc > INT32_MAX) throw std::length_error("encrypt_cssc: row entries exceed 2^31");
        }
        pre[n_rows] = (int32_t)acc;
        lay.entries = (size_t)acc;
    }
    std::memcpy(h + lay.o_ci, ci, 8 * nnz);
    std::memcpy(h + lay.o_va, va, 8 * nnz);
    std::memcpy(h + lay.o_v, vec, 8 * vec_len);
    std::memcpy(h + lay.o_rows, rows, 16 * n_rows);
    std::memcpy(h + lay.o_sl, slices, 8 * n_slices);
    std::memcpy(h + lay.o_cols, cols, 16 * n_cols);
    auto* hs = reinterpret_cast<u64*>(h + lay.o_st);
    for (int i = 0; i < items; ++i) hs[i] = next_stream_id();
    std::memcpy(h + lay.o_out, out.data(), 8 * (size_t)items);
    encrypt_cssc_image(h, lay);
}

void GpuContext::encrypt_cssc_image(const unsigned char* img, const CsscLayout& lay, const ClientWs* ws,
                                    EncIn* defer, int part, cudaEvent_t early_ev) {
    const int items = lay.items;
    if (!items) return;
    unsigned char* d;
    u64 *U, *CM;
    if (ws) {
        encrypt_cssc_forked(img, lay, *ws, defer, part, early_ev);
        return;
    } else if (forked_enc_) {
        ensure_ws(scratch_[0], std::max<size_t>(lay.bytes, 256));
        ClientWs w;
        w.up = scratch_[0].as<unsigned char>();
        w.CM = enc_workspace(items);
        w.U = wsU_.words();
        encrypt_cssc_forked(img, lay, w);
        if (img == stage_) cuda_check(cudaEventRecord(stage_ev_, st_), "event");
        return;
    } else {
        ensure_ws(scratch_[0], std::max<size_t>(lay.bytes, 256));
        d = scratch_[0].as<unsigned char>();
        CM = enc_workspace(items);
        U = wsU_.words();
    }
    cuda_check(cudaMemcpyAsync(d, img, lay.bytes, cudaMemcpyHostToDevice, st_), "upload");
    if (img == stage_) cuda_check(cudaEventRecord(stage_ev_, st_), "event");  // staging reusable after this
    launch_pack_cssc(dc_, P_, d + lay.o_ci, d + lay.o_va, d + lay.o_v, lay.ci_w, lay.va_w, lay.v_w,
                     reinterpret_cast<const int4*>(d + lay.o_rows), reinterpret_cast<const int*>(d + lay.o_rpre),
                     (int)lay.n_rows, (long)lay.entries,
                     reinterpret_cast<const int2*>(d + lay.o_sl), reinterpret_cast<const int4*>(d + lay.o_cols),
                     items / 2, CM + (size_t)2 * P_.cfg.L * P_.n, cm_stride(), st_);
    encrypt_encoded(reinterpret_cast<const u64*>(d + lay.o_st), reinterpret_cast<u64* const*>(d + lay.o_out), items,
                    U, CM);
}

// The pipeline's encryption as two graph branches (captured from st_ and
// st2_): the ciphertext randomness depends only on (seed, stream id), so
//   st_ : stream ids + output pointers (16 B per item) -> sample u -> NTT(u)
//         -> x pk + inverse block phase -> inverse columns      (c0', c1')
//   st2_: CSR image -> device CSSC pack -> inverse NTT of the messages mod t
// run side by side, joined by the finishing kernel (+ e0 + Delta m, + e1).
// CM is [item][2L][N] followed by the messages [item][N]; same words as the
// staged path.
void GpuContext::encrypt_cssc_forked(const unsigned char* img, const CsscLayout& lay, const ClientWs& ws,
                                     EncIn* defer, int part, cudaEvent_t early_ev) {
    const int items = lay.items, L = P_.cfg.L, logn = P_.cfg.logn;
    const size_t n = (size_t)P_.n;
    unsigned char* d = ws.up;
    u64* CM = ws.CM;
    u64* MSG = CM + (size_t)items * 2 * L * n;
    const auto* streams = reinterpret_cast<const u64*>(d + lay.o_st);
    // branch A: stream ids and output pointers, then the message-independent encryption
    auto branch_a = [&] {
        cuda_check(cudaMemcpyAsync(d + lay.o_st, img + lay.o_st, lay.bytes - lay.o_st, cudaMemcpyHostToDevice, st_),
                   "upload");
        if (part == 1 && ws.E) cuda_check(cudaEventRecord(ev_upload_, st_), "ids uploaded");
        launch_enc_sample_u(dc_, P_, P_.cfg.key, streams, ws.U, items, st_);
        launch_ntt_phase(dc_, logn, false, true, job(ws.U, ws.U, L, range_idx(0, L)), items, st_);
        launch_blocks_mul_inv(dc_, P_, ws.U, pk_.words(), 2, CM, (size_t)2 * L * n, nullptr, 0, 0, items, st_,
                              pk_sh_.words());
        std::vector<int> pidx = range_idx(0, L);
        pidx.insert(pidx.end(), pidx.begin(), pidx.end());
        launch_ntt_phase(dc_, logn, true, true, job(CM, CM, 2 * L, pidx), items, st_);
    };
    if (part == 1) {  // branch A alone (the pipeline's early graph), the e draws beside it
        branch_a();
        if (ws.E) {
            cuda_check(cudaStreamWaitEvent(st2_, ev_upload_, 0), "ids");
            launch_enc_sample_e(dc_, P_, P_.cfg.key, streams, ws.E, items, st2_);
            cuda_check(cudaEventRecord(ev_join_, st2_), "join");
            cuda_check(cudaStreamWaitEvent(st_, ev_join_, 0), "join");
        }
        return;
    }
    cudaStream_t sb = part == 2 ? st_ : st2_;
    if (part != 2) {
        cuda_check(cudaEventRecord(ev_fork_, st_), "fork");
        cuda_check(cudaStreamWaitEvent(st2_, ev_fork_, 0), "fork");
    }
    // branch B: the CSR image, packing, message INTT
    cuda_check(cudaMemcpyAsync(d, img, lay.o_st, cudaMemcpyHostToDevice, sb), "upload");
    launch_pack_cssc(dc_, P_, d + lay.o_ci, d + lay.o_va, d + lay.o_v, lay.ci_w, lay.va_w, lay.v_w,
                     reinterpret_cast<const int4*>(d + lay.o_rows), reinterpret_cast<const int*>(d + lay.o_rpre),
                     (int)lay.n_rows, (long)lay.entries,
                     reinterpret_cast<const int2*>(d + lay.o_sl), reinterpret_cast<const int4*>(d + lay.o_cols),
                     items / 2, MSG, n, sb);
    launch_ntt(dc_, logn, true, job(MSG, MSG, 1, {P_.t_index()}), items, sb);
    if (part != 2) {
        cuda_check(cudaEventRecord(ev_join_, st2_), "join");
        branch_a();
        cuda_check(cudaStreamWaitEvent(st_, ev_join_, 0), "join");
    } else if (early_ev) {  // branch A ran as the early graph on the side stream
        cuda_check(cudaStreamWaitEvent(st_, early_ev, cudaEventWaitExternal), "join early");
    }
    if (defer) {
        *defer = EncIn{P_.cfg.key, streams, CM, (size_t)2 * L * n, MSG, n,
                       reinterpret_cast<u64* const*>(d + lay.o_out), items / 2, nullptr,
                       part == 2 ? ws.E : nullptr};
        stats_.kernels += 7;
    } else {
        launch_enc_finish(dc_, P_, P_.cfg.key, streams, CM, reinterpret_cast<u64* const*>(d + lay.o_out), items,
                          st_, MSG, (size_t)2 * L * n, n, part == 2 ? ws.E : nullptr);
        stats_.kernels += 8;
    }
    stats_.limb_ntts += (u64)items * (1 + 3 * L);
}

// CM = wsC_[item][2L+1][N] holds the encoded messages in limb 2L on entry;
// the inverse NTT of the message (mod t) rides in the same launch as the
// inverse NTT of pk * u (limbs 0 .. 2L-1).
void GpuContext::encrypt_encoded(const u64* d_streams, u64* const* d_out, int items, u64* U, u64* CM) {
    const int L = P_.cfg.L, logn = P_.cfg.logn;
    if (!U) U = wsU_.words();
    if (!CM) CM = wsC_.words();
    launch_enc_sample_u(dc_, P_, P_.cfg.key, d_streams, U, items, st_);
    std::vector<int> pidx = range_idx(0, L);
    pidx.insert(pidx.end(), pidx.begin(), pidx.end());
    pidx.push_back(P_.t_index());
    if (fused_ks_) {  // NTT(u) column phase; block phase x pk + inverse block phase (+ message); columns
        launch_ntt_phase(dc_, logn, false, true, job(U, U, L, range_idx(0, L)), items, st_);
        launch_blocks_mul_inv(dc_, P_, U, pk_.words(), 2, CM, cm_stride(), CM, 2 * L, P_.t_index(), items, st_,
                              pk_sh_.words());
        launch_ntt_phase(dc_, logn, true, true, job(CM, CM, 2 * L + 1, pidx), items, st_);
        stats_.kernels += 5;
    } else {
        launch_ntt(dc_, logn, false, job(U, U, L, range_idx(0, L)), items, st_);
        launch_enc_pk(dc_, P_, pk_.words(), U, CM, items, st_);
        launch_ntt(dc_, logn, true, job(CM, CM, 2 * L + 1, pidx), items, st_);
        stats_.kernels += 7;
    }
    launch_enc_finish(dc_, P_, P_.cfg.key, d_streams, CM, d_out, items, st_);
    stats_.limb_ntts += (u64)items * (1 + 3 * L);
}

void GpuContext::decrypt(const std::vector<const u64*>& cts, u64* slots_host, int* budgets) {
    const int items = (int)cts.size();
    if (!items) return;
    const int n = P_.n, L = P_.cfg.L, logn = P_.cfg.logn;
    ensure_ws(wsX_, sizeof(u64) * (size_t)items * L * n);
    ensure_ws(wsM_, sizeof(u64) * (size_t)items * n);
    ensure_ws(wsU_, sizeof(u64) * (size_t)items * (n / 2) + 8 * (size_t)items + 64);
    // one pinned block: ct pointers up, slots + noise deviations down (async copies)
    const size_t down = sizeof(u64) * (size_t)items * (n / 2) + 8 * (size_t)items;
    size_t pcap = 0;
    unsigned char* pin = pinned_take(8 * (size_t)items + down, &pcap);
    std::memcpy(pin, cts.data(), 8 * (size_t)items);
    ensure_ws(scratch_[0], std::max<size_t>(8 * (size_t)items, 256));
    auto* dct = scratch_[0].as<const u64*>();
    cuda_check(cudaMemcpyAsync(scratch_[0].as<void>(), pin, 8 * (size_t)items, cudaMemcpyHostToDevice, st_),
               "upload");
    u64* slots_dev = wsU_.words();
    auto* maxdev = reinterpret_cast<unsigned long long*>(wsU_.words() + (size_t)items * (n / 2));
    decrypt_dev(dct, items, wsX_.words(), wsM_.words(), slots_dev, maxdev);
    unsigned char* back = pin + 8 * (size_t)items;
    cuda_check(cudaMemcpyAsync(back, slots_dev, down, cudaMemcpyDeviceToHost, st_), "slots");
    try {
        synchronize();
    } catch (...) {
        pinned_give(pin, pcap);
        throw;
    }
    std::memcpy(slots_host, back, sizeof(u64) * (size_t)items * (n / 2));
    const auto* md = reinterpret_cast<const unsigned long long*>(back + sizeof(u64) * (size_t)items * (n / 2));
    for (int i = 0; i < items; ++i) {
        const int bl = md[i] ? 64 - __builtin_clzll(md[i]) : 0;
        if (budgets) budgets[i] = std::max(0, 63 - bl);
    }
    pinned_give(pin, pcap);
}

void GpuContext::decrypt_dev(const u64* const* dct, int items, u64* X, u64* M, u64* slots_dev,
                             unsigned long long* maxdev) {
    const int n = P_.n, L = P_.cfg.L, logn = P_.cfg.logn;
    NttJob j = job(nullptr, X, L, range_idx(0, L));
    j.src_items = dct;
    j.src_limb_offset = L;
    if (fused_ks_) {  // column phase of c1; block phase x s + inverse block phase; inverse columns
        launch_ntt_phase(dc_, logn, false, true, j, items, st_);
        launch_blocks_mul_inv(dc_, P_, X, s_ntt_.words(), 1, X, (size_t)L * n, nullptr, 0, 0, items, st_,
                              s_sh_.words());
        launch_ntt_phase(dc_, logn, true, true, job(X, X, L, range_idx(0, L)), items, st_);
    } else {
        launch_ntt(dc_, logn, false, j, items, st_);
        launch_mul_s(dc_, P_, X, s_ntt_.words(), items, st_);
        launch_ntt(dc_, logn, true, job(X, X, L, range_idx(0, L)), items, st_);
    }
    launch_dec_scale(dc_, P_, dct, X, M, maxdev, items, st_);
    launch_ntt(dc_, logn, false, job(M, M, 1, {P_.t_index()}), items, st_);
    if (slots_dev) launch_decode_gather(dc_, P_, M, slots_dev, items, st_);
    stats_.kernels += 7;
    stats_.limb_ntts += (u64)items * (2 * L + 1);
}

// ------------------------------------------------------------------ ct ops
void GpuContext::sum(const std::vector<const u64*>& a, u64* out) {
    if (a.empty()) {
        cuda_check(cudaMemsetAsync(out, 0, sizeof(u64) * ct_words(), st_), "zero");
        return;
    }
    for (const u64* p : a)
        if (p == out) throw std::invalid_argument("sum: output aliases an input");
    launch_sum_items(dc_, P_, upload_ptrs(a, 0), (int)a.size(), out, st_);
    stats_.kernels += 1;
}

void GpuContext::add(const std::vector<const u64*>& a, const std::vector<const u64*>& b,
                     const std::vector<u64*>& out) {
    const int items = (int)out.size();
    if (!items) return;
    launch_add(dc_, P_, upload_ptrs(a, 0), upload_ptrs(b, 1), upload_ptrs(out, 2), items, st_);
    stats_.kernels += 1;
}

void GpuContext::mul_relin_dev(const u64* const* A, const u64* const* B, u64* const* OUT,
                               int items, u64* T, u64* Z, u64* D2, u64* DX, u64* ACC,
                               const u64* const* RLK, const EncIn* enc, u64* D2Y, u64* const* YOUT,
                               int relin_lo, u64* const* Y1) {
    const int L = P_.cfg.L, K = P_.cfg.K, LK = L + K, M = P_.mul_limbs(), logn = P_.cfg.logn;
    std::vector<int> pm;
    for (int j = 0; j < M; ++j) pm.push_back(j < L ? j : K + j);
    bool lazy_z = false;
    if (enc)
        launch_mul_extend_enc(dc_, P_, *enc, T, items, st_);
    else
        launch_mul_extend(dc_, P_, A, B, T, items, st_);
    kmark(enc ? "k_mul_extend_enc" : "k_mul_extend_k", st_);
    if (fused_ks_) {  // column phase, fused blocks + tensor + inverse blocks, column phase
        launch_ntt_phase(dc_, logn, false, true, job(T, T, 4 * M, pm), items, st_);
        kmark("k_ntt_cols fwd (multiply)", st_);
        launch_mul_blocks_tensor(dc_, P_, T, Z, items, st_);
        kmark("k_mul_blocks_tensor", st_);
        NttJob jz = job(Z, Z, 3 * M, pm);
        jz.lazy_out = fixed_rns_shape(P_) ? 1 : 0;  // the fixed-shape scale folds N^-1 into its constants
        launch_ntt_phase(dc_, logn, true, true, jz, items, st_);
        lazy_z = jz.lazy_out != 0;
        kmark("k_ntt_cols inv (multiply)", st_);
    } else {
        launch_ntt(dc_, logn, false, job(T, T, 4 * M, pm), items, st_);
        launch_mul_tensor(dc_, P_, T, Z, items, st_);
        launch_ntt(dc_, logn, true, job(Z, Z, 3 * M, pm), items, st_);
    }
    launch_mul_scale(dc_, P_, Z, OUT, D2, items, st_, fused_ks_ ? D2Y : nullptr, lazy_z, fused_ks_ ? Y1 : nullptr);
    kmark("k_mul_scale_k", st_);
    if (relin_lo < 0 || relin_lo > items) throw std::invalid_argument("mul_relin: relin range");
    const int nr = items - relin_lo;  // relinearised items, from relin_lo on
    if (nr == 0) {
        stats_.kernels += 5;
    } else if (fused_ks_) {
        KsY ky;
        ky.srcc = D2Y ? D2Y + (size_t)relin_lo * L * P_.n : nullptr;
        ky.out = YOUT ? YOUT + relin_lo : nullptr;
        launch_ks_fused(dc_, P_, nullptr, D2 + (size_t)relin_lo * L * P_.n, 0, nullptr, RLK + relin_lo,
                        reinterpret_cast<const u64* const*>(OUT + relin_lo), nullptr, OUT + relin_lo, DX, ACC, nr,
                        st_, nullptr, nullptr, ky);
        stats_.kernels += 9;
    } else {
        if (relin_lo) throw std::invalid_argument("mul_relin: folded relinearisation needs the fused key switch");
        launch_ks_modup_contig(dc_, P_, D2, DX, items, st_);
        launch_ntt(dc_, logn, false, job(DX, DX, P_.dnum * LK, range_idx(0, LK)), items, st_);
        launch_ks_inner(dc_, P_, DX, RLK, ACC, items, st_);
        launch_ntt(dc_, logn, true, job(ACC, ACC, 2 * LK, range_idx(0, LK)), items, st_);
        launch_ks_moddown(dc_, P_, ACC, reinterpret_cast<const u64* const*>(OUT), nullptr, nullptr, OUT,
                          items, st_);
        stats_.kernels += 10;
    }
    stats_.limb_ntts += (u64)items * (7 * M + P_.dnum * LK + 2 * LK);
}

void GpuContext::mul_relin(const std::vector<const u64*>& a, const std::vector<const u64*>& b,
                           const std::vector<u64*>& out) {
    const int items = (int)out.size();
    if (!items) return;
    ensure_ws(wsT_, sizeof(u64) * items * mul_T_words());
    ensure_ws(wsZ_, sizeof(u64) * items * mul_Z_words());
    ensure_ws(wsD2_, sizeof(u64) * items * poly_words());
    ensure_ws(wsDX_, sizeof(u64) * items * dx_words());
    ensure_ws(wsACC_, sizeof(u64) * items * ksacc_words());
    std::vector<const u64*> rlk(items, rlk_.words());
    mul_relin_dev(upload_ptrs(a, 0), upload_ptrs(b, 1), upload_ptrs(out, 2), items, wsT_.words(),
                  wsZ_.words(), wsD2_.words(), wsDX_.words(), wsACC_.words(), upload_ptrs(rlk, 3));
}

void GpuContext::rotate_dev(const u64* const* SRC, const u32* ginv, const u64* const* KEY,
                            const u64* const* BASE, u64* const* OUT, int items, u64* DX, u64* ACC,
                            const u64* const* EXTRA, const int* PAIR, const KsY& ky) {
    const int LK = P_.cfg.L + P_.cfg.K, logn = P_.cfg.logn;
    if (fused_ks_) {
        launch_ks_fused(dc_, P_, SRC, nullptr, 1, ginv, KEY, BASE, SRC, OUT, DX, ACC, items, st_, EXTRA, PAIR, ky);
        stats_.kernels += 4;
    } else {
        launch_ks_modup(dc_, P_, SRC, 1, ginv, DX, items, st_);
        launch_ntt(dc_, logn, false, job(DX, DX, P_.dnum * LK, range_idx(0, LK)), items, st_);
        launch_ks_inner(dc_, P_, DX, KEY, ACC, items, st_);
        launch_ntt(dc_, logn, true, job(ACC, ACC, 2 * LK, range_idx(0, LK)), items, st_);
        launch_ks_moddown(dc_, P_, ACC, BASE, SRC, ginv, OUT, items, st_, EXTRA, PAIR);
        stats_.kernels += 7;
    }
    stats_.limb_ntts += (u64)items * (P_.dnum * LK + 2 * LK);
}

static u32 inverse_galois(u32 g, int n) {
    const u64 two_n = 2 * (u64)n;
    u64 r = 1, b = g;
    for (u64 e = (u64)n - 1; e; e >>= 1) {
        if (e & 1) r = r * b % two_n;
        b = b * b % two_n;
    }
    return (u32)r;
}

void GpuContext::rotate(const std::vector<const u64*>& src, const std::vector<int64_t>& k,
                        const std::vector<const u64*>& base, const std::vector<u64*>& out) {
    const int items = (int)out.size();
    std::vector<const u64*> rs, rb, keys, ia, ib;
    std::vector<u64*> ro, io;
    std::vector<u32> gi;
    bool any_base = false;
    for (int i = 0; i < items; ++i) any_base |= base[i] != nullptr;
    for (int i = 0; i < items; ++i) {
        const u32 g = galois_element(k[i], P_.n);
        if (g == 1) {
            if (base[i]) {
                ia.push_back(base[i]);
                ib.push_back(src[i]);
                io.push_back(out[i]);
            } else if (out[i] != src[i]) {
                cuda_check(cudaMemcpyAsync(out[i], src[i], sizeof(u64) * ct_words(),
                                           cudaMemcpyDeviceToDevice, st_), "copy");
            }
            continue;
        }
        rs.push_back(src[i]);
        rb.push_back(base[i]);
        keys.push_back(galois_key(g));
        gi.push_back(inverse_galois(g, P_.n));
        ro.push_back(out[i]);
    }
    const int r = (int)ro.size();
    if (r) {
        if (any_base)
            for (auto& p : rb)
                if (!p) throw std::invalid_argument("rotate: mixed base/no-base batch");
        ensure_ws(wsDX_, sizeof(u64) * r * dx_words());
        ensure_ws(wsACC_, sizeof(u64) * r * ksacc_words());
        rotate_dev(upload_ptrs(rs, 0), upload_ptrs(gi, 1), upload_ptrs(keys, 2),
                   any_base ? upload_ptrs(rb, 3) : nullptr, upload_ptrs(ro, 4), r, wsDX_.words(),
                   wsACC_.words());
    }
    if (!io.empty()) add(ia, ib, io);
}

void GpuContext::mul_plain(const std::vector<const u64*>& a, const int64_t* vals,
                           const u64* offs, const std::vector<u64*>& out) {
    const int items = (int)out.size();
    if (!items) return;
    const int n = P_.n, L = P_.cfg.L, logn = P_.cfg.logn;
    for (int i = 0; i < items; ++i)
        if (offs[i + 1] - offs[i] > (u64)P_.S) throw std::length_error("encode: values exceed slot count");
    ensure_ws(wsM_, sizeof(u64) * (size_t)items * n);
    ensure_ws(wsPT_, sizeof(u64) * (size_t)items * L * n);
    ensure_ws(wsX_, sizeof(u64) * (size_t)items * 2 * L * n);
    auto* dv = static_cast<int64_t*>(upload_bytes(vals, sizeof(int64_t) * offs[items], 0));
    auto* doff = static_cast<u64*>(upload_bytes(offs, sizeof(u64) * (items + 1), 1));
    launch_encode_scatter(dc_, P_, dv, doff, wsM_.words(), items, st_);
    launch_ntt(dc_, logn, true, job(wsM_.words(), wsM_.words(), 1, {P_.t_index()}), items, st_);
    launch_plain_lift(dc_, P_, wsM_.words(), wsPT_.words(), items, st_);
    launch_ntt(dc_, logn, false, job(wsPT_.words(), wsPT_.words(), L, range_idx(0, L)), items, st_);
    NttJob j = job(nullptr, wsX_.words(), 2 * L, range_idx(0, L));
    j.src_items = upload_ptrs(a, 2);
    launch_ntt(dc_, logn, false, j, items, st_);
    launch_pointwise_plain(dc_, P_, wsX_.words(), wsPT_.words(), items, 2, st_);
    launch_ntt(dc_, logn, true, job(wsX_.words(), wsX_.words(), 2 * L, range_idx(0, L)), items, st_);
    for (int i = 0; i < items; ++i)
        cuda_check(cudaMemcpyAsync(out[i], wsX_.words() + (size_t)i * ct_words(), sizeof(u64) * ct_words(),
                                   cudaMemcpyDeviceToDevice, st_), "copy");
    stats_.kernels += 7;
}

void GpuContext::encode_masks(const std::vector<int>& ones_len, u64* MASKS) {
    const int m = (int)ones_len.size();
    if (!m) return;
    const int n = P_.n, L = P_.cfg.L, logn = P_.cfg.logn;
    std::vector<u64> offs(m + 1, 0);
    for (int i = 0; i < m; ++i) {
        if (ones_len[i] > P_.S) throw std::length_error("mask longer than slot count");
        offs[i + 1] = offs[i] + (u64)ones_len[i];
    }
    std::vector<int64_t> vals(std::max<u64>(offs[m], 1), 1);
    ensure_ws(wsM_, sizeof(u64) * (size_t)m * n);
    auto* dv = static_cast<int64_t*>(upload_bytes(vals.data(), sizeof(int64_t) * vals.size(), 0));
    auto* doff = static_cast<u64*>(upload_bytes(offs.data(), sizeof(u64) * offs.size(), 1));
    launch_encode_scatter(dc_, P_, dv, doff, wsM_.words(), m, st_);
    launch_ntt(dc_, logn, true, job(wsM_.words(), wsM_.words(), 1, {P_.t_index()}), m, st_);
    launch_plain_lift(dc_, P_, wsM_.words(), MASKS, m, st_);
    launch_ntt(dc_, logn, false, job(MASKS, MASKS, L, range_idx(0, L)), m, st_);
}

void GpuContext::ntt_host(int prime_index, u64* data, int limbs, bool inverse) {
    const int n = P_.n;
    DevBuf buf(&pool_, sizeof(u64) * (size_t)limbs * n);
    cuda_check(cudaMemcpyAsync(buf.words(), data, buf.bytes(), cudaMemcpyHostToDevice, st_), "ntt in");
    launch_ntt(dc_, P_.cfg.logn, inverse, job(buf.words(), buf.words(), 1, {prime_index}), limbs, st_);
    cuda_check(cudaMemcpyAsync(data, buf.words(), buf.bytes(), cudaMemcpyDeviceToHost, st_), "ntt out");
    synchronize();
}

template const u64** GpuContext::upload_ptrs<const u64*>(const std::vector<const u64*>&, int);
template u64** GpuContext::upload_ptrs<u64*>(const std::vector<u64*>&, int);
template u32* GpuContext::upload_ptrs<u32>(const std::vector<u32>&, int);

}  // namespace cssc
