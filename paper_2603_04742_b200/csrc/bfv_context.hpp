// bfv_context.hpp -- device-resident RNS-BFV context: parameters, keys,
// ciphertext memory and the batched homomorphic operations.  Host C++ only
// orchestrates; every arithmetic step is a kernel in bfv_kernels.cu.
#pragma once
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <map>
#include <memory>
#include <mutex>
#include <vector>

#include "bfv_kernels.cuh"
#include "rns_params.hpp"

namespace cssc {

void cuda_check(cudaError_t e, const char* what);

// Size-bucketed caching allocator (all ciphertexts of a context share a size).
class DevicePool {
public:
    ~DevicePool();
    void* alloc(size_t bytes);
    void release(void* p, size_t bytes);
    void trim();

private:
    std::mutex mu_;
    std::multimap<size_t, void*> free_;
};

// RAII device buffer backed by a pool
class DevBuf {
public:
    DevBuf() = default;
    DevBuf(DevicePool* pool, size_t bytes);
    ~DevBuf();
    DevBuf(DevBuf&& o) noexcept;
    DevBuf& operator=(DevBuf&& o) noexcept;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    template <class T>
    T* as() const { return static_cast<T*>(ptr_); }
    u64* words() const { return static_cast<u64*>(ptr_); }
    size_t bytes() const { return bytes_; }
    bool empty() const { return ptr_ == nullptr; }
    void ensure(DevicePool* pool, size_t bytes);  // grow (contents discarded)

private:
    DevicePool* pool_ = nullptr;
    void* ptr_ = nullptr;
    size_t bytes_ = 0;
};

// Counts what one batched call launched (for bench accounting).
struct LaunchStats {
    uint64_t kernels = 0;
    uint64_t limb_ntts = 0;
};

// Byte offsets of the arrays in one client upload image (see encrypt_cssc).
struct CsscLayout {
    size_t o_ci = 0, o_va = 0, o_v = 0, o_rows = 0, o_rpre = 0, o_sl = 0, o_cols = 0, o_st = 0, o_out = 0, bytes = 0;
    size_t nnz = 0, vec_len = 0, n_rows = 0, n_slices = 0, n_cols = 0;
    size_t entries = 0;  // sum of the row lengths (= nnz for CSR-derived rows): one pack thread each
    int items = 0;  // 2 * chunks
    // element widths in bytes: column indices 2 / 4 / 8 (unsigned), values and
    // vector entries 1 / 8 (signed) -- the compact forms when every entry fits
    int ci_w = 8, va_w = 8, v_w = 8;
    static CsscLayout make(size_t nnz, size_t vec_len, size_t n_rows, size_t n_slices, size_t n_cols, int items,
                           int ci_w = 8, int va_w = 8, int v_w = 8);
};

// Device buffers of a client pass owned by its caller (a cached pipeline), so
// that a captured graph never points into the context's growable workspaces.
struct ClientWs {
    unsigned char* up = nullptr;  // upload image
    u64* U = nullptr;             // [items][L][N] encryption u
    u64* CM = nullptr;            // [items][2L+1][N] encryption accumulators + message
    u64* X = nullptr;             // [results][L][N] decryption c1*s
    u64* M = nullptr;             // [results][N] decoded message
    u64* slots = nullptr;         // [results][S] slots, then [results] noise deviations
    int8_t* E = nullptr;          // [items][2][N] pre-drawn e (early graph; null: drawn in the finish)
};

class GpuContext {
public:
    explicit GpuContext(const RnsConfig& cfg, int device = 0);
    ~GpuContext();

    const RnsParams& params() const { return P_; }
    const DevConsts* dconsts() const { return dc_; }
    cudaStream_t stream() const { return st_; }
    DevicePool& pool() { return pool_; }
    int n() const { return P_.n; }
    int L() const { return P_.cfg.L; }
    size_t ct_words() const { return (size_t)2 * P_.cfg.L * P_.n; }
    size_t ksk_words() const { return (size_t)P_.dnum * 2 * (P_.cfg.L + P_.cfg.K) * P_.n; }
    uint64_t next_stream_id() { return stream_counter_.fetch_add(1); }
    // first stream id the counter hands out (ids name the encryption
    // randomness under the context key: two contexts sharing a key must use
    // disjoint id ranges)
    void set_stream_base(uint64_t b) { stream_counter_.store(b); }
    LaunchStats& stats() { return stats_; }
    // fused 3-kernel key switch (default) or the 7-launch reference pipeline
    void set_fused_key_switch(bool on) { fused_ks_ = on; }
    bool fused_key_switch() const { return fused_ks_; }
    void set_forked_encrypt(bool on) { forked_enc_ = on; }
    // whole-evaluation graph fusions across the party boundary (bit 0: the
    // encryption's finish inside the multiply's extension, bit 1: the
    // decryption inside the mask step); 0 = party-separated (default)
    void set_pipe_fuse(int mask) { pipe_fuse_ = mask & 3; }
    int pipe_fuse() const { return pipe_fuse_; }

    // keys (NTT form on device)
    const u64* relin_key() const { return rlk_.words(); }
    const u64* galois_key(u32 g);                 // generated on first use
    // key for target phi_g(s)^2 (key id 2^32 | g): rotates the s^2 component of
    // an unrelinearised product (the plan's folded level 0)
    const u64* galois_key_sq(u32 g);
    void ensure_galois_keys(const std::vector<int64_t>& steps);
    size_t galois_key_count() const { return gk_.size(); }
    const u64* s_ntt() const { return s_ntt_.words(); }
    const u64* pk() const { return pk_.words(); }
    void download_sk(int64_t* out);
    void download_pk_coef(u64* out);               // canonical coefficient form
    void download_key_coef(u32 which, u64* out);   // 0 = relin, else Galois element

    // ---- batched operations; all pointers are device pointers ----
    // item i encodes vals[offs[i] .. offs[i+1]) (host arrays); streams: encryption stream ids
    void encrypt(const int64_t* vals, const u64* offs, const u64* streams,
                 const std::vector<u64*>& out);
    // same with device-resident arrays
    void encrypt_dev(const int64_t* d_vals, const u64* d_offs, const u64* d_streams,
                     u64* const* d_out, int items);
    // Client A + Client B on the device: scatter CSR rows into the CSSC chunk
    // plaintexts (value chunks then vector chunks) and encrypt them; host arrays
    // go up in one pinned upload.  Layout of the descriptors: spmvgpu_encrypt_cssc.
    void encrypt_cssc(const int64_t* ci, const int64_t* va, size_t nnz, const int64_t* vec, size_t vec_len,
                      const int32_t* rows, size_t n_rows, const int32_t* slices, size_t n_slices,
                      const int32_t* cols, size_t n_cols, const std::vector<u64*>& out);
    // the same from an image already laid out in pinned host memory (trusted
    // descriptors: the caller built them); the image must stay alive until the
    // stream has consumed it
    // defer (pipeline, fused path): skip the finishing kernel and describe its
    // inputs instead; the multiply's extension (launch_mul_extend_enc) finishes
    // part (pipeline capture): 0 both branches, 1 only the message-independent
    // branch (ids + output handles upload, u, pk u), 2 only the image branch
    // and the join (part 1 must have run before on the same stream)
    // early_ev (part 2): the early graph's completion event, waited on
    // (external event wait) before the join
    void encrypt_cssc_image(const unsigned char* img, const CsscLayout& lay, const ClientWs* ws = nullptr,
                            EncIn* defer = nullptr, int part = 0, cudaEvent_t early_ev = nullptr);
    cudaStream_t side_stream() const { return st2_; }
    uint64_t peek_stream_id() const { return stream_counter_.load(); }
    // pinned host buffers, pooled by capacity
    unsigned char* pinned_take(size_t bytes, size_t* cap);
    void pinned_give(unsigned char* p, size_t cap);
    void decrypt(const std::vector<const u64*>& cts, u64* slots_host, int* budgets);
    // capture-safe device part of decrypt: slots_dev[items][S], maxdev[items]
    // (zeroed here) from the device pointer array dct
    void decrypt_dev(const u64* const* dct, int items, u64* X, u64* M, u64* slots_dev, unsigned long long* maxdev);
    void add(const std::vector<const u64*>& a, const std::vector<const u64*>& b,
             const std::vector<u64*>& out);
    void mul_relin(const std::vector<const u64*>& a, const std::vector<const u64*>& b,
                   const std::vector<u64*>& out);
    // out = a_0 + a_1 + ... (out may not alias an input)
    void sum(const std::vector<const u64*>& a, u64* out);
    // out_i = (base_i ? base_i : 0) + rot(src_i, k_i)
    void rotate(const std::vector<const u64*>& src, const std::vector<int64_t>& k,
                const std::vector<const u64*>& base, const std::vector<u64*>& out);
    // out_i = a_i * encode(vals_i)
    void mul_plain(const std::vector<const u64*>& a, const int64_t* vals, const u64* offs,
                   const std::vector<u64*>& out);
    // KAT helpers
    void ntt_host(int prime_index, u64* data, int limbs, bool inverse);
    void synchronize();
    // the side stream (an early encryption graph may run there, pipeline_speculate)
    void synchronize_side() { cuda_check(cudaStreamSynchronize(st2_), "side stream sync"); }

    // building blocks reused by the batched cloud plan (pointer arrays on device)
    // enc: A and B are still to be finished from a deferred encryption (EncIn)
    // D2Y / YOUT (fused key switch, fixed shapes): the ModUp factors of c2 and
    // of the products' c1 (KsY)
    // relin_lo > 0: items [0, relin_lo) stay unrelinearised (OUT = (z0, z1), D2 =
    // z2, D2Y its ModUp factors, Y1 those of z1: the plan folds their
    // relinearisation into level 0); items [relin_lo, items) are relinearised
    void mul_relin_dev(const u64* const* A, const u64* const* B, u64* const* OUT, int items,
                       u64* T, u64* Z, u64* D2, u64* DX, u64* ACC, const u64* const* RLK,
                       const EncIn* enc = nullptr, u64* D2Y = nullptr, u64* const* YOUT = nullptr,
                       int relin_lo = 0, u64* const* Y1 = nullptr);
    // OUT = BASE + EXTRA + rot(SRC) (BASE / EXTRA per-item nullable); PAIR (nullable):
    // PAIR[i] = j >= 0 also adds item j's rotation into OUT[i] (PAIR[j] = -3 - i;
    // the two items' CTAs split the limbs)
    void rotate_dev(const u64* const* SRC, const u32* ginv, const u64* const* KEY,
                    const u64* const* BASE, u64* const* OUT, int items, u64* DX, u64* ACC,
                    const u64* const* EXTRA = nullptr, const int* PAIR = nullptr, const KsY& ky = KsY{});
    void encode_masks(const std::vector<int>& ones_len, u64* MASKS);  // NTT form [m][L][N]
    NttJob job(const u64* src, u64* dst, int limbs, const std::vector<int>& pidx) const;

    // workspace sizing (words per item)
    size_t mul_T_words() const { return (size_t)4 * (P_.cfg.L + P_.nB) * P_.n; }
    size_t mul_Z_words() const { return (size_t)3 * (P_.cfg.L + P_.nB) * P_.n; }
    size_t dx_words() const { return (size_t)P_.dnum * (P_.cfg.L + P_.cfg.K) * P_.n; }
    size_t ksacc_words() const { return (size_t)2 * (P_.cfg.L + P_.cfg.K) * P_.n; }
    size_t poly_words() const { return (size_t)P_.cfg.L * P_.n; }
    size_t cm_stride() const { return (size_t)(2 * P_.cfg.L + 1) * P_.n; }  // encryption CM item stride

    // scratch pointer arrays (stream-ordered reuse)
    template <class T>
    T* upload_ptrs(const std::vector<T>& v, int slot);
    void* upload_bytes(const void* src, size_t bytes, int slot);

private:
    void keygen();
    // encryption of the encoded messages staged in limb 2L of the CM workspace
    void encrypt_encoded(const u64* d_streams, u64* const* d_out, int items, u64* U = nullptr, u64* CM = nullptr);
    u64* enc_workspace(int items);  // wsU_ + wsC_ (CM layout), returns CM
    // pinned host staging buffer, reusable once its previous upload completed
    unsigned char* stage_host(size_t bytes);
    void* stage_upload(size_t bytes, int slot);
    DevBuf gen_ksk(u64 keyid, const u64* sp_ntt);
    void encrypt_cssc_forked(const unsigned char* img, const CsscLayout& lay, const ClientWs& ws,
                             EncIn* defer = nullptr, int part = 0, cudaEvent_t early_ev = nullptr);
    void ensure_ws(DevBuf& b, size_t bytes) { b.ensure(&pool_, bytes); }

    RnsParams P_;
    int device_ = 0;
    cudaStream_t st_ = nullptr;
    DevicePool pool_;
    DevConsts* dc_ = nullptr;
    std::vector<DevBuf> tables_;
    DevBuf pos0_;
    DevBuf s_small_, s_ntt_, pk_, rlk_;
    std::map<u32, DevBuf> gk_, gk2_;
    DevBuf pk_sh_, s_sh_;  // Shoup companions of pk and of s's Q limbs
    std::atomic<uint64_t> stream_counter_{1};
    LaunchStats stats_;
    bool fused_ks_ = true;
    bool forked_enc_ = false;
    int pipe_fuse_ = 0;
    // workspaces for ad-hoc batched calls
    DevBuf wsT_, wsZ_, wsD2_, wsDX_, wsACC_, wsM_, wsX_, wsU_, wsC_, wsPT_;
    DevBuf scratch_[8];
    std::multimap<size_t, unsigned char*> pinned_free_;
    unsigned char* stage_ = nullptr;  // pinned
    size_t stage_bytes_ = 0;
    cudaEvent_t stage_ev_ = nullptr;
    // side stream + fork/join events: the pipeline's encryption runs its
    // message-independent part beside the upload and packing
    cudaStream_t st2_ = nullptr;
    cudaEvent_t ev_fork_ = nullptr, ev_join_ = nullptr, ev_upload_ = nullptr;
    std::mutex mu_;
};

}  // namespace cssc
