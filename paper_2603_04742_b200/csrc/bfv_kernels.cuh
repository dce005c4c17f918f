// bfv_kernels.cuh -- launch wrappers for the sm_100a RNS-BFV kernels.
//
// Every wrapper processes a whole batch (all chunks x all RNS limbs) in one
// launch.  Per-item operands are passed as device arrays of pointers so that
// ciphertexts can live anywhere in the context's arena; temporaries are
// contiguous [item][poly][limb][N].
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

#include "rns_params.hpp"

namespace cssc {

constexpr int MAX_JOB_LIMBS = 128;  // 4 * (2L + 1) = 68 at L = 8 (ring 2^15)

struct NttJob {
    const u64* src = nullptr;               // contiguous [items][limbs][N] (if src_items null)
    const u64* const* src_items = nullptr;  // per-item base pointers, each [limbs][N]
    int src_limb_offset = 0;                // skip this many limbs of each src item
    u64* dst = nullptr;                     // contiguous [items][limbs][N] (if dst_items null)
    u64* const* dst_items = nullptr;        // per-item base pointers, each [limbs][N]
    int limbs = 0;                          // limbs per item
    signed char pidx[MAX_JOB_LIMBS];        // global prime index of limb j
    // inverse column phase only: skip the final x N^-1, outputs lazy in [0, 2q);
    // set when the consumer (k_mul_scale_k, k_ks_moddown_k) folds N^-1 into its
    // constants (same canonical results, one Shoup product less per coefficient)
    int lazy_out = 0;
    // inverse column phase only: per item (nullable entries) an addend with the
    // layout of the input, added to it first (lazy inputs < 2q, sum reduced to
    // < 2q): the key-switch accumulators of an odd step folded into its
    // doubling step's INTT + ModDown
    const u64* const* add_items = nullptr;
};

// sampler domains (nonce word 0 = dom | limb << 8 | digit << 16)
enum SampleDomain : u32 {
    DOM_SK = 1,
    DOM_PK_A = 2,
    DOM_PK_E = 3,
    DOM_KSK_A = 4,
    DOM_KSK_E = 5,
    DOM_ENC_U = 6,
    DOM_ENC_E0 = 7,
    DOM_ENC_E1 = 8,
};

void cuda_check(cudaError_t e, const char* what);

// Opt kernel `fn` into `bytes` of dynamic shared memory on the CURRENT device.
// The attribute is per device, so the record is keyed by (kernel, device) and
// guarded by a mutex (several contexts / devices / threads in one process).
void smem_optin(const void* fn, int bytes);
template <class F>
inline void smem_optin_k(F* fn, int bytes) {
    smem_optin(reinterpret_cast<const void*>(fn), bytes);
}

// Kernel-level timing marks (bench.py's per-kernel profile): when a mark list
// is installed for this thread, every launch site records an external event
// labelled with its kernel after the launch (an event node under capture).
struct KernelMark {
    const char* name;
    cudaEvent_t ev;
};
void kmarks_install(std::vector<KernelMark>* marks);  // nullptr: off
void kmark(const char* name, cudaStream_t st);

// column-tile width policy shared by the column-phase kernels (ctas16 = CTAs at 16 columns)
bool cols_use_ln8(long ctas16, bool allowed);
bool cols_use_ln4(long ctas16, bool allowed);
// block-phase kernels (K2, mask): 8-block tiles when the 16-block launch has
// fewer than CSSC_BLOCKS_LN8_MAX CTAs (default 2 x 148); CSSC_BLOCKS_LN=8|16 forces
bool blocks_use_ln8(long ctas16);
void launch_ntt(const DevConsts* dc, int logn, bool inverse, const NttJob& job, int items,
                cudaStream_t st);
// a single phase of the two-phase NTT (cols = column phase, else block phase)
void launch_ntt_phase(const DevConsts* dc, int logn, bool inverse, bool cols, const NttJob& job,
                      int items, cudaStream_t st);
size_t ntt_smem_bytes(int logn);

// ct x ct
// pipeline: the encryption's finish (e, Delta m) fused into the base extension
// Hoisted ModUp factors: y_i = [x_i (Q_d / q_i)^-1]_{q_i} of a ciphertext's c1
// (the key switch's source), written by the kernel that produces c1 (ModDown,
// the multiply's scale) so K1 reads y instead of recomputing it per target.
struct KsY {
    const u64* const* src = nullptr;  // per item: y of the source's c1 [L][N] (null: compute from x)
    const u64* srcc = nullptr;        // contiguous variant ([item][L][N])
    u64* const* out = nullptr;        // per item (nullable entries): y of the output's c1
};

struct EncIn {
    SeedKey seed;
    const u64* streams;  // per encryption item (a chunks, then b chunks)
    const u64* CM;       // pk u after the inverse NTT, [item][2L][N] (cstride words apart)
    size_t cstride;
    const u64* MSG;      // encoded messages mod t, mstride words apart
    size_t mstride;
    u64* const* OUT;     // ciphertext of each encryption item
    int n_chunks;
    const int* order;    // multiply item -> chunk (the plan's depth order); null = identity
    const int8_t* E;     // pre-drawn e: [item][2][N] (k_enc_sample_e); null = draw in place
};
bool fixed_rns_shape(const RnsParams& P);  // one of the compiled (L, K, alpha) shapes
void launch_mul_extend_enc(const DevConsts* dc, const RnsParams& P, const EncIn& in, u64* T, int items,
                           cudaStream_t st);
void launch_mul_extend(const DevConsts* dc, const RnsParams& P, const u64* const* A,
                       const u64* const* B, u64* T, int items, cudaStream_t st);
// fused forward block phase + mask multiply-accumulate + inverse block phase
// (mul_fused.cu); OUT[s] receives the slice sums before the inverse column phase
// the pipeline's decrypting mask step: D[slice][L][N] = c0 + c1 s (see mul_fused.cu)
void launch_mask_dec_blocks(const DevConsts* dc, const RnsParams& P, const u64* MT, const int* slice_off,
                            const int* slice_items, const int* item_mask, const u64* MASKS, const u64* S_NTT,
                            u64* D, int slices, cudaStream_t st);
// D -> inverse column phase -> t/Q scale + decode NTT mod t -> slots (maxdev per item)
void launch_decrypt_ntt(const DevConsts* dc, const RnsParams& P, u64* D, u64* M, u64* slots,
                        unsigned long long* maxdev, int items, cudaStream_t st);
void launch_mask_blocks(const DevConsts* dc, const RnsParams& P, const u64* MT, const int* slice_off,
                        const int* slice_items, const int* item_mask, const u64* MASKS, u64* const* OUT,
                        int slices, cudaStream_t st);
// block phase x NTT-form multipliers (pk or s) + inverse block phase, limb-wise
// (mul_fused.cu); OUT limb p*L+j of item i at OUT + i*out_stride; XTRA: an extra
// limb run through the inverse block phase in place (prime index xprime)
void launch_blocks_mul_inv(const DevConsts* dc, const RnsParams& P, const u64* IN, const u64* MUL, int nmul,
                           u64* OUT, size_t out_stride, u64* XTRA, int xlimb, int xprime, int items,
                           cudaStream_t st, const u64* MULSH = nullptr);
// fused forward block phase + tensor + inverse block phase (mul_fused.cu)
void launch_mul_blocks_tensor(const DevConsts* dc, const RnsParams& P, const u64* T, u64* Z, int items,
                              cudaStream_t st);
void launch_mul_tensor(const DevConsts* dc, const RnsParams& P, const u64* T, u64* Z, int items,
                       cudaStream_t st);
// lazy_in: Z is the unscaled, lazy inverse column output (NttJob::lazy_out)
// Y1 (per item nullable): ModUp factors of z1 (the product's c1 when it is
// key-switched without relinearisation)
void launch_mul_scale(const DevConsts* dc, const RnsParams& P, const u64* Z, u64* const* OUT,
                      u64* D2, int items, cudaStream_t st, u64* D2Y = nullptr, bool lazy_in = false,
                      u64* const* Y1 = nullptr);

// hybrid key switching
void launch_ks_modup(const DevConsts* dc, const RnsParams& P, const u64* const* SRC, int src_poly,
                     const u32* ginv, u64* DX, int items, cudaStream_t st);
void launch_ks_modup_contig(const DevConsts* dc, const RnsParams& P, const u64* SRC, u64* DX,
                            int items, cudaStream_t st);
void launch_ks_inner(const DevConsts* dc, const RnsParams& P, const u64* DX,
                     const u64* const* KEY, u64* ACC, int items, cudaStream_t st);
// OUT[p] = BASE[p] (same index, optional) + (p==0 ? phi_g(RSRC[0]) : 0) (optional)
//          + ModDown(ACC[p])
// the key switch's inverse column phase + ModDown in one launch (fixed shapes
// L = K = 2 at N = 2^13 / 2^14); false: not applicable, use the two kernels
bool ks_cols_moddown_applies(const RnsParams& P, int items);
// XACC (nullable, per item nullable): accumulators added before the shared INTT + ModDown
bool launch_ks_cols_moddown(const DevConsts* dc, const RnsParams& P, const u64* ACC, const u64* const* BASE,
                            const u64* const* RSRC, const u32* ginv, u64* const* OUT, int items, cudaStream_t st,
                            const u64* const* EXTRA, const int* PAIR, u64* const* YOUT,
                            const u64* const* XACC = nullptr);
void launch_acc_add(const DevConsts* dc, const RnsParams& P, u64* ACC, const u64* const* XACC, int items,
                    cudaStream_t st);
// OUT[i].c0 (=|+=) sum_t phi(SRC[i*3+t].c0) with inverse Galois elements GI[i*3+t] (0: none)
void launch_automorph_sum(const DevConsts* dc, const RnsParams& P, u64* const* OUT, const u64* const* SRC,
                          const u32* GI, bool accumulate, int items, cudaStream_t st);
void launch_automorph_c0(const DevConsts* dc, const RnsParams& P, const u64* const* SRC, const u32* ginv,
                         u64* const* OUT, int items, cudaStream_t st);
void launch_ks_moddown(const DevConsts* dc, const RnsParams& P, const u64* ACC,
                       const u64* const* BASE, const u64* const* RSRC, const u32* ginv,
                       u64* const* OUT, int items, cudaStream_t st, const u64* const* EXTRA = nullptr,
                       const int* PAIR = nullptr, u64* const* YOUT = nullptr, bool lazy_in = false);

// masks / plaintext products
void launch_mask_accum(const DevConsts* dc, const RnsParams& P, const u64* MT,
                       const int* slice_off, const int* slice_items, const int* item_mask,
                       const u64* MASKS, u64* RES, int slices, cudaStream_t st);
void launch_pointwise_plain(const DevConsts* dc, const RnsParams& P, u64* X, const u64* PT,
                            int items, int polys, cudaStream_t st);

// encoding / encryption / decryption
// item i encodes vals[offs[i] .. offs[i+1]) (at most S values)
// CSR rows -> CSSC chunk plaintexts (value chunks [0, n_chunks), vector
// chunks [n_chunks, 2 n_chunks)), slot layout applied; see spmvgpu_encrypt_cssc
// CI / VA / V: column indices (unsigned, ci_w = 2 / 4 / 8 bytes), values and
// vector entries (signed, va_w / v_w = 1 / 8 bytes) of the client image
void launch_pack_cssc(const DevConsts* dc, const RnsParams& P, const void* CI, const void* VA, const void* V,
                      int ci_w, int va_w, int v_w, const int4* rows, const int* rpre, int n_rows, long entries,
                      const int2* slices, const int4* cols, int n_chunks, u64* M, size_t mstride, cudaStream_t st);
void launch_encode_scatter(const DevConsts* dc, const RnsParams& P, const int64_t* vals,
                           const u64* offs, u64* M, int items, cudaStream_t st, size_t mstride = 0);
void launch_plain_lift(const DevConsts* dc, const RnsParams& P, const u64* M, u64* PT, int items,
                       cudaStream_t st);
// E[item][poly][N] = the CBD e draws of k_enc_finish (|e| <= 21, as int8)
void launch_enc_sample_e(const DevConsts* dc, const RnsParams& P, SeedKey seed, const u64* streams, int8_t* E,
                         int items, cudaStream_t st);
void launch_enc_sample_u(const DevConsts* dc, const RnsParams& P, SeedKey seed, const u64* streams,
                         u64* U, int items, cudaStream_t st);
void launch_enc_pk(const DevConsts* dc, const RnsParams& P, const u64* PK, const u64* U, u64* C,
                   int items, cudaStream_t st);
// CM[item][2L+1][N]: c0 (L limbs), c1 (L limbs), then the message (coef form mod t);
// or, with MSG set, CM items cstride words apart and the messages in MSG
// (mstride words apart)
void launch_enc_finish(const DevConsts* dc, const RnsParams& P, SeedKey seed, const u64* streams,
                       const u64* CM, u64* const* OUT, int items, cudaStream_t st, const u64* MSG = nullptr,
                       size_t cstride = 0, size_t mstride = 0, const int8_t* E = nullptr);
void launch_mul_s(const DevConsts* dc, const RnsParams& P, u64* X, const u64* S_NTT, int items,
                  cudaStream_t st);
void launch_dec_scale(const DevConsts* dc, const RnsParams& P, const u64* const* CT,
                      const u64* X, u64* M, unsigned long long* maxdev, int items,
                      cudaStream_t st);
// slots [0, rows[r]) of result r as u32 at out + off[r] (the pipeline's compact download)
void launch_decode_rows(const DevConsts* dc, const RnsParams& P, const u64* M, u32* out, const int* rows,
                        const int* off, int max_rows, int items, cudaStream_t st);
void launch_decode_gather(const DevConsts* dc, const RnsParams& P, const u64* M, u64* slots,
                          int items, cudaStream_t st);

// keys
void launch_sample_small(int logn, SeedKey seed, u32 dom, u64 id, int kind /*0 ternary,1 cbd*/,
                         int64_t* out, cudaStream_t st);
void launch_sample_uniform(const DevConsts* dc, int logn, SeedKey seed, u32 dom, int digit, u64 id,
                           int limbs, int limb0, u64* out, cudaStream_t st);
void launch_lift_small(const DevConsts* dc, int logn, const int64_t* s, int limbs, int limb0,
                       u64* out, cudaStream_t st);
void launch_automorph_small(int logn, u32 g, const int64_t* in, int64_t* out, cudaStream_t st);
// out = -(A*S + E) [+ P_q * SP on the digit's limbs]; all NTT form over limbs [0, limbs)
// Shoup companions floor(w 2^64 / q_j) of `polys` polynomials over the L+K key primes
void launch_shoup_companions(const DevConsts* dc, const u64* W, u64* WS, int LK, int n, int polys,
                             cudaStream_t st);
void launch_key_combine(const DevConsts* dc, int logn, int limbs, const u64* A, const u64* E,
                        const u64* S, const u64* SP, int digit_lo, int digit_hi, u64* out,
                        cudaStream_t st);
void launch_square(const DevConsts* dc, int logn, int limbs, const u64* S, u64* out,
                   cudaStream_t st);

// generic ct ops
void launch_sum_items(const DevConsts* dc, const RnsParams& P, const u64* const* A, int count, u64* OUT,
                      cudaStream_t st);
void launch_add(const DevConsts* dc, const RnsParams& P, const u64* const* A,
                const u64* const* B, u64* const* OUT, int items, cudaStream_t st);
// SURVEY 8(e) chunk split: W = [results][2][L][N] sums of the ranks' partial
// result words (each < q_j, at most 16 ranks: < 2^62) -> residues mod q_j, in place
void launch_fold_mod(const DevConsts* dc, const RnsParams& P, u64* W, int results, cudaStream_t st);


}  // namespace cssc

namespace cssc {
// register-resident lazy-Shoup butterfly peak (butterflies / s)
double probe_butterfly_peak(const DevConsts* unused, u64 q, u64 w, u64 wsh, cudaStream_t st);
}  // namespace cssc

namespace cssc {
// Fused hybrid key switch (ks_fused.cu): OUT[p] = BASE[p] + (p==0 ? phi_g(RSRC.c0) : 0)
// + KeySwitch(phi_g(SRC poly src_poly)) with per-item keys; SRC == nullptr reads the
// contiguous [item][L][N] polynomials at SRCC instead.  DX / ACC are workspaces.
// ModUp + NTT + key product + INTT of a key switch as one cluster kernel
// (ks_cluster.cu); false when the shape has no cluster specialisation
bool launch_ks_cluster(const DevConsts* dc, const RnsParams& P, const u64* const* SRC, const u64* SRCC,
                       int src_poly, const u32* ginv, const u64* const* KEY, u64* ACC, int items, cudaStream_t st);
// Hoisted key switches of shared sources (level 0): every source polynomial
// gets one ModUp + forward NTT (H); item i's accumulators are the sum over its
// `nterm` terms t of H[hidx[i*nterm+t]] permuted by gel[...] (1: identity)
// times key[i*nterm+t] (hidx < 0: no term)
struct HoistedKs {
    int nsrc = 0;
    const u64* const* src = nullptr;   // per source: the ciphertext holding it
    int src_poly = 1;                  // ... as polynomial src_poly of that ciphertext
    const u64* const* ysrc = nullptr;  // per source: its ModUp factors y (KsY), nullable
    int nterm = 1;
    const int* hidx = nullptr;         // [item][nterm] source index
    const u32* gel = nullptr;          // [item][nterm] Galois element
    const int* order = nullptr;        // launch order of the items (nullable)
};

// A batched key switch in two phases, so that the accumulators of several key
// switches can be summed before one shared INTT + ModDown (the plan's odd steps):
// accumulate ACC[item] (phi_g(ModUp(SRC[item].c1)) x KEY[item]; hk: hoisted
// sources), then finish (XACC[item] added, INTT, ModDown, + BASE + EXTRA +
// phi_g(RSRC.c0), KsY factors of c1 into YOUT).  The domain of ACC between
// the two depends on the path.
enum class KsAccDomain { BlockInv, Coeff, Ntt };
KsAccDomain launch_ks_accumulate(const DevConsts* dc, const RnsParams& P, bool fused, const u64* const* SRC,
                                 const u32* ginv, const u64* const* KEY, u64* DX, u64* ACC, int items,
                                 cudaStream_t st, const KsY& ky, const HoistedKs* hk = nullptr);
void launch_ks_finish(const DevConsts* dc, const RnsParams& P, KsAccDomain dom, const u64* const* BASE,
                      const u64* const* RSRC, const u32* ginv, u64* const* OUT, u64* ACC, int items, cudaStream_t st,
                      const u64* const* EXTRA, u64* const* YOUT, const u64* const* XACC);
void launch_ks_fused(const DevConsts* dc, const RnsParams& P, const u64* const* SRC, const u64* SRCC,
                     int src_poly, const u32* ginv, const u64* const* KEY, const u64* const* BASE,
                     const u64* const* RSRC, u64* const* OUT, u64* DX, u64* ACC, int items, cudaStream_t st,
                     const u64* const* EXTRA = nullptr, const int* PAIR = nullptr, const KsY& ky = KsY{});
}  // namespace cssc
