// ks_fused.cu -- hybrid key switching fused around the two-phase NTT.
//
//   K1 k_ks_modup_cols   : automorphism gather + ModUp (E3) of one digit into
//                          one target limb, then the NTT column phase, per
//                          column tile                    -> DX (lazy, [0,4q))
//   K2 k_ks_blocks_inner : for every digit: NTT block phase of DX, multiply by
//                          the switching-key tiles and accumulate (both key
//                          polynomials); then the INTT block phase of both
//                          accumulators                    -> ACC (lazy, [0,2q))
//   then the column-phase INTT of ACC (standard kernel, full occupancy) and
//   the elementwise ModDown (E4) with the fused adds
//                          out = base + phi_g(rsrc.c0) + ModDown(acc)
// replacing ModUp, NTT x2, inner product, INTT x2 and ModDown (7 launches)
// by 4 launches with two fewer full passes over the digit/accumulator
// buffers.  Same integer formulas as bfv_kernels.cu / the oracle, so the
// outputs are bit-identical.
#include <stdexcept>
#include <string>
#include <type_traits>

#include "bfv_kernels.cuh"
#include "ntt.cuh"

namespace cssc {

#define KS_CHECK()                                                                              \
    do {                                                                                        \
        cudaError_t e_ = cudaGetLastError();                                                    \
        if (e_ != cudaSuccess) throw std::runtime_error(std::string("ks launch: ") + cudaGetErrorString(e_)); \
    } while (0)

__device__ __forceinline__ int ks_automorph(u32 ginv, int k, int n, bool& neg) {
    if (ginv == 0) {
        neg = false;
        return k;
    }
    const u32 i0 = (u32)(((unsigned long long)ginv * (unsigned)k) & (unsigned long long)(2 * n - 1));
    neg = i0 >= (u32)n;
    return neg ? (int)(i0 - n) : (int)i0;
}

template <int LOGN>
__device__ __forceinline__ void load_col_twiddles(u64* tws, const u64* tw) {
    using G = Ntt2<LOGN>;
    for (int i = threadIdx.x; i < G::R1; i += blockDim.x) {
        const ulonglong2 w = __ldg(reinterpret_cast<const ulonglong2*>(tw) + i);
        tws[2 * i] = w.x;
        tws[2 * i + 1] = w.y;
    }
}

// ---------------------------------------------------------------------------
// K1: ModUp + NTT column phase
// ---------------------------------------------------------------------------
// LN columns per CTA: 16, or 8 when the launch would not fill the GPU
template <int LOGN, int LT, int KT, int AT, int LN = 16>
__global__ void __launch_bounds__(Ntt2<LOGN>::TC, 256 / Ntt2<LOGN>::TC * 3) k_ks_modup_cols(const DevConsts* __restrict__ dc, const u64* const* SRC,
                                                       const u64* SRCC, int src_poly, const u32* ginv, u64* DX,
                                                       const u64* const* YS, const u64* YSC) {
    using G = Ntt2<LOGN>;
    constexpr int CTAS = G::R2 / LN;
    extern __shared__ u64 smem[];
    u64* tile = smem;
    u64* tws = smem + LN * G::R1;
    const int L = LT ? LT : dc->L, K = KT ? KT : dc->K, LK = L + K;
    const int alpha = AT ? AT : dc->alpha, dnum = (L + alpha - 1) / alpha;
    int bid = blockIdx.x;
    const int tileid = bid % CTAS;
    bid /= CTAS;
    const int j = bid % LK;
    bid /= LK;
    const int dg = bid % dnum;
    const int item = bid / dnum;
    const int lo = dg * alpha, hi = min(lo + alpha, L);
    const u64* src = SRC ? SRC[item] + (size_t)src_poly * L * G::N : SRCC + (size_t)item * L * G::N;
    // hoisted ModUp factors y_i of the source (KsY), when its producer wrote them
    const u64* ysrc = YS ? YS[item] : (YSC ? YSC + (size_t)item * L * G::N : nullptr);
    const u32 gi = ginv ? ginv[item] : 0u;
    const u64 m = dc->mod[j].q;
    const bool own = j >= lo && j < hi;
    const int col0 = tileid * LN;
    load_col_twiddles<LOGN>(tws, dc->tw[j].fwd);
    constexpr int PER = G::R1 * LN / G::TC;  // elements per thread
#pragma unroll 8
    for (int r = 0; r < PER; ++r) {
        const int e = threadIdx.x + G::TC * r, c = e / LN, jl = e % LN;
        bool neg;
        const int idx = ks_automorph(gi, col0 + jl + G::R2 * c, G::N, neg);
        u64 v;
        if (own) {
            const u64 x = __ldg(src + (size_t)j * G::N + idx);
            v = neg ? neg_mod(x, m) : x;
        } else {
            v = 0;
#pragma unroll
            for (int i = lo; i < (AT ? lo + AT : hi); ++i) {
                if (AT && i >= hi) break;
                const u64 qi = dc->mod[i].q;
                u64 y;
                if (ysrc) {  // hoisted factors of the source (un-rotated)
                    y = __ldg(ysrc + (size_t)i * G::N + idx);
                } else {
                    const u64 x = __ldg(src + (size_t)i * G::N + idx);
                    y = shoup_q(x, dc->dig_hat_inv[i], dc->dig_hat_inv_sh[i], qi);
                }
                v += shoup_lazy_q(y, dc->dig_hat[i][j], dc->dig_hat_sh[i][j], m);  // alpha <= 16 terms < 2m
            }
            // phi_g(ModUp(x)): the automorphism's sign applies to the converted limb (DESIGN 2.9)
            v = reduce_small_quot_q(v, dc->mod[j]);
            v = neg ? neg_mod(v, m) : v;
        }
        tile[c * LN + jl] = v;
    }
    __syncthreads();
    auto addr = [](int l, int pos) { return pos * LN + l; };
    auto twf = [&](int sl, int, int blk) {
        const int k = (1 << sl) + blk;
        return make_ulonglong2(tws[2 * k], tws[2 * k + 1]);
    };
    line_ntt_v<G::A, 0, false, (LN >= 8 ? 3 : 2), LN>(tile, SpecQ{m}, addr, twf, whole_cta());  // radix-8: 3 CTAs/SM
    u64* dst = DX + (((size_t)item * dnum + dg) * LK + j) * G::N;
    constexpr int SEG = LN / 2;
#pragma unroll
    for (int r = 0; r < G::R1 * SEG / G::TC; ++r) {
        const int i = threadIdx.x + G::TC * r, c = i / SEG, h = i % SEG;
        *reinterpret_cast<ulonglong2*>(dst + (size_t)c * G::R2 + col0 + 2 * h) =
            make_ulonglong2(tile[c * LN + 2 * h], tile[c * LN + 2 * h + 1]);
    }
}

// K1 over all target limbs of a digit (fixed RNS shapes): one CTA per (item,
// digit, tile of LC columns) holds the LC columns of every one of the L+K
// target limbs (16 lines = (L+K) x LC).  Each coefficient of phi_g(source)
// is gathered once per digit prime -- the alpha hoisted factors y_i -- and
// feeds every target limb: the digit's own limbs x_i = y_i [Q_d/q_i]_{q_i}
// (one Shoup product, the same canonical word as gathering x_i), the others
// the ModUp sum.  The per-limb kernel above gathers each coefficient once
// per target limb (x_i for own limbs, all y_i for each other limb: 6 loads
// per coefficient at L = K = 2 instead of 2); K1 stalls on those gathers
// (long scoreboard, profiles/r02_ncu_c5_*).
template <int LOGN, int LT, int KT, int AT, int LC>
__global__ void __launch_bounds__(Ntt2<LOGN>::TC, 256 / Ntt2<LOGN>::TC * 3)
    k_ks_modup_all(const DevConsts* __restrict__ dc, const u64* const* SRC, const u64* SRCC, int src_poly,
                   const u32* ginv, u64* DX, const u64* const* YS, const u64* YSC) {
    using G = Ntt2<LOGN>;
    constexpr int LK = LT + KT, VL = LK * LC, DN = (LT + AT - 1) / AT;
    static_assert(LT > 0 && VL <= 16 && G::TC % VL == 0, "fixed shapes with at most 16 lines");
    constexpr int CT = G::R2 / LC;
    constexpr int TWS = 2 * G::R1 + 2;  // per-limb twiddle stride (16 B pad: limbs on distinct banks)
    extern __shared__ u64 smem[];
    u64* tile = smem;                   // [R1][VL], line = limb * LC + column
    u64* tws = smem + VL * G::R1;       // [LK][TWS]
    int bid = blockIdx.x;
    const int tileid = bid % CT;
    bid /= CT;
    const int dg = bid % DN;
    const int item = bid / DN;
    const int lo = dg * AT, hi = lo + AT < LT ? lo + AT : LT;
    const u64* src = SRC ? SRC[item] + (size_t)src_poly * LT * G::N : SRCC + (size_t)item * LT * G::N;
    const u64* ysrc = YS ? YS[item] : (YSC ? YSC + (size_t)item * LT * G::N : nullptr);
    const u32 gi = ginv ? ginv[item] : 0u;
    const int col0 = tileid * LC;
    for (int i = threadIdx.x; i < LK * G::R1; i += G::TC) {
        const int jj = i / G::R1, k = i % G::R1;
        const ulonglong2 w = __ldg(reinterpret_cast<const ulonglong2*>(dc->tw[jj].fwd) + k);
        *reinterpret_cast<ulonglong2*>(tws + jj * TWS + 2 * k) = w;
    }
    constexpr int PER = G::R1 * LC / G::TC;
    static_assert(PER >= 1, "column tile smaller than the CTA");
#pragma unroll
    for (int r = 0; r < PER; ++r) {
        const int e = threadIdx.x + G::TC * r, c = e / LC, jl = e % LC;
        bool neg;
        const int idx = ks_automorph(gi, col0 + jl + G::R2 * c, G::N, neg);
        u64 x[AT], y[AT];
#pragma unroll
        for (int a = 0; a < AT; ++a) {
            const int i = lo + a;
            if (i >= hi) break;
            const u64 qi = dc->mod[i].q;
            if (ysrc) {  // hoisted factors of the un-rotated source; x_i = y_i [Q_d/q_i]_{q_i}
                y[a] = __ldg(ysrc + (size_t)i * G::N + idx);
                x[a] = shoup_q(y[a], dc->dig_hat[i][i], dc->dig_hat_sh[i][i], qi);
            } else {
                x[a] = __ldg(src + (size_t)i * G::N + idx);
                y[a] = shoup_q(x[a], dc->dig_hat_inv[i], dc->dig_hat_inv_sh[i], qi);
            }
        }
#pragma unroll
        for (int j = 0; j < LK; ++j) {
            u64 v;
            if (j >= lo && j < hi) {
                v = x[j - lo];
            } else {
                v = 0;
#pragma unroll
                for (int a = 0; a < AT; ++a) {
                    const int i = lo + a;
                    if (i >= hi) break;
                    v += shoup_lazy_q(y[a], dc->dig_hat[i][j], dc->dig_hat_sh[i][j], dc->mod[j].q);
                }
                v = reduce_small_quot_q(v, dc->mod[j]);
            }
            // phi_g(ModUp(x)): the automorphism's sign on every target limb (DESIGN 2.9)
            tile[c * VL + j * LC + jl] = neg ? neg_mod(v, dc->mod[j].q) : v;
        }
    }
    __syncthreads();
    // every thread keeps one line (tid % VL) in every pass: its modulus and
    // twiddle row are per-thread constants
    const int myl = threadIdx.x % VL;
    const u64 myq = dc->mod[myl / LC].q;
    const u64* mytw = tws + (myl / LC) * TWS;
    auto addr = [](int l, int pos) { return pos * VL + l; };
    auto twf = [&](int sl, int, int blk) {
        const int k = (1 << sl) + blk;
        return *reinterpret_cast<const ulonglong2*>(mytw + 2 * k);
    };
    line_ntt_v<G::A, 0, false, 3, VL>(tile, SpecQ{myq}, addr, twf, whole_cta());
    u64* dst = DX + ((size_t)item * DN + dg) * LK * G::N;
    constexpr int SEG = LC / 2;
    static_assert(LC % 2 == 0, "pairs of columns per store");
#pragma unroll
    for (int r = 0; r < G::R1 * LK * SEG / G::TC; ++r) {
        const int i = threadIdx.x + G::TC * r, h = i % SEG, j = (i / SEG) % LK, c = i / (SEG * LK);
        *reinterpret_cast<ulonglong2*>(dst + (size_t)j * G::N + (size_t)c * G::R2 + col0 + 2 * h) =
            make_ulonglong2(tile[c * VL + j * LC + 2 * h], tile[c * VL + j * LC + 2 * h + 1]);
    }
}

template <int LT, int KT>
constexpr int modup_all_lc() { return 16 / (LT + KT) >= 2 ? 16 / (LT + KT) : 0; }

// Used for launches whose 16-column CTAs fill a wave (default, =2); =1 also
// below that with 8 lines per CTA (measured 1-2 % slower at C1-C3 than the
// per-limb 4/8-column tiles there); =0 keeps the per-limb K1 everywhere.
static int k1_all_mode() {
    static const int mode = [] {
        const char* e = std::getenv("CSSC_K1_ALL");
        return e ? std::atoi(e) : 2;
    }();
    return mode;
}

// ---------------------------------------------------------------------------
// K2: NTT block phase + key inner product + INTT block phase
// ---------------------------------------------------------------------------
// Two 128-thread groups with named barriers: the dnum digit tiles are
// transformed two at a time, and the two accumulators' inverse transforms run
// concurrently, so a CTA's serial chain is ceil(dnum/2) + 1 tile transforms.
constexpr int kKsGroups = 2, kKsGroupThreads = 128;
// Key MAC: lazy sums.  Every Shoup product is < 2q and q < 2^58, so 15 of them
// stay below 2^(k+5), reduce_small_quot_q's domain: one reduction per sum
// instead of two conditional subtractions per term (CSSC_LAZY_MAC=0: the eager form).
#ifndef CSSC_LAZY_MAC
#define CSSC_LAZY_MAC 1
#endif
constexpr int kLazyMacTerms = 15;
__device__ __forceinline__ void mac_term(u64& a, u64 w, u64 k, u64 ksh, u64 q) {
#if CSSC_LAZY_MAC
    a += shoup_lazy_q(w, k, ksh, q);
#else
    a = add_mod(a, shoup_q(w, k, ksh, q), q);
#endif
}
__device__ __forceinline__ u64 mac_reduce(u64 a, const Modulus& md) {
#if CSSC_LAZY_MAC
    return reduce_small_quot_q(a, md);
#else
    return a;
#endif
}
template <int LOGN>
constexpr bool ks_keys_tma() { return LOGN <= 14; }

template <int LOGN, int LT, int KT, int AT, int LN = 16>
__global__ void __launch_bounds__(kKsGroups * kKsGroupThreads) k_ks_blocks_inner(const DevConsts* __restrict__ dc,
                                                                               const u64* __restrict__ DX,
                                                                               const u64* const* KEY,
                                                                               u64* __restrict__ ACC) {
    using G = Ntt2<LOGN>;
    extern __shared__ u64 smem[];
    constexpr int PITCH = G::PITCH;
    constexpr int TW = LN * PITCH;
    constexpr int T = kKsGroups * kKsGroupThreads;
    constexpr int PER = LN * G::R2 / T;  // elements per thread
    // 8-block tiles (small launches): radix-4 passes keep all 128 threads of a
    // group busy (radix-8 would leave half idle) and halve each thread's chain
    constexpr int KMR = LN >= 16 ? 4 : 2;
    constexpr int CTAS = G::R1 / LN;
    static_assert(PER >= 1, "tile smaller than the CTA");
    const int L = LT ? LT : dc->L, K = KT ? KT : dc->K, LK = L + K;
    const int alpha = AT ? AT : dc->alpha, dnum = (L + alpha - 1) / alpha;
    u64* work = smem;               // dnum digit tiles; then acc0 in tile 0, acc1 in tile 1
    u64* tws = smem + (dnum < 2 ? 2 : dnum) * TW;
    constexpr int KT_W = LN * G::R2;  // words of one key tile (contiguous in HBM)
    // key tiles by TMA into smem at 2^14 and below; at 2^15 they would cost the
    // second CTA per SM, so the MAC reads them straight from HBM there
    constexpr bool KTMA = ks_keys_tma<LOGN>();
    u64* keys = tws + 2 * btw_entries<LOGN, LN>();  // [dnum][2][KT_W]
    auto* bar = reinterpret_cast<unsigned long long*>(keys + (KTMA ? (size_t)dnum * 2 * KT_W : 0));
    int bid = blockIdx.x;
    const int tileid = bid % CTAS;
    bid /= CTAS;
    const int j = bid % LK;
    const int item = bid / LK;
    const Modulus md = dc->mod[j];
    const u64 q = md.q;
    const int blk0 = tileid * LN;
    const size_t base = (size_t)blk0 * G::R2;
    const u64* key = KEY[item];
    const size_t PL = (size_t)LK * G::N;
    const size_t KW = (size_t)dnum * 2 * PL;  // key words; their Shoup companions follow
    const int grp = threadIdx.x / kKsGroupThreads;
    const ThreadGroup tg = cta_slice(grp, kKsGroups);
    // element x = threadIdx.x + T r of the tile (line x >> B, column x & (R2-1)):
    // consecutive lanes touch consecutive words in HBM and in smem (conflict free)
    auto saddr = [](int x) { return (x >> G::B) * PITCH + (x & (G::R2 - 1)); };
    auto addr = [](int l, int pos) { return l * PITCH + pos; };
    auto twf = [&](int sl, int l, int blk) { return block_tw<LOGN, LN>(tws, sl, l, blk); };
    // the key tiles of every digit and both polynomials: TMA bulk copies issued
    // first, landing while the digits are transformed
    if (KTMA && threadIdx.x == 0) {
        mbar_init(bar, 1);
        mbar_expect_tx(bar, (unsigned)(dnum * 2 * KT_W * 8));
        for (int dg = 0; dg < dnum; ++dg)
            for (int p = 0; p < 2; ++p)
                bulk_g2s(keys + (size_t)(dg * 2 + p) * KT_W, key + ((size_t)dg * 2 + p) * PL + (size_t)j * G::N + base,
                         KT_W * 8, bar);
    }
    load_block_twiddles<LOGN, LN>(tws, dc->tw[j].fwd, blk0);
    for (int dg = 0; dg < dnum; ++dg) {
        const u64* d = DX + (((size_t)item * dnum + dg) * LK + j) * G::N + base;
#pragma unroll
        for (int r = 0; r < PER; ++r) {
            const int x = threadIdx.x + T * r;
            cp_async8(work + dg * TW + saddr(x), d + x);
        }
    }
    cp_async_wait_all();
    __syncthreads();
#pragma unroll 1
    for (int dg = grp; dg < dnum; dg += kKsGroups)
        line_ntt_v<G::B, 0, false, KMR, LN>(work + dg * TW, SpecQ{q}, addr, twf, tg);
    __syncthreads();
    // inner product with both key polynomials (tiles in smem once the TMA
    // transaction completes); every position is read (all digits) and then
    // overwritten by one thread
    if (KTMA) mbar_wait(bar, 0);
#pragma unroll
    for (int r = 0; r < PER; ++r) {
        const int x = threadIdx.x + T * r, s0 = saddr(x);
        u64 a0 = 0, a1 = 0;
        int pend = 0;
        for (int dg = 0; dg < dnum; ++dg) {
            if (pend == kLazyMacTerms) {
                a0 = mac_reduce(a0, md);
                a1 = mac_reduce(a1, md);
                pend = 1;
            }
            ++pend;
            const u64 w = work[dg * TW + s0];
            u64 k0, k1;
            const size_t ko = ((size_t)dg * 2) * PL + (size_t)j * G::N + base + x;
            if (KTMA) {
                k0 = keys[(size_t)(dg * 2) * KT_W + x];
                k1 = keys[(size_t)(dg * 2 + 1) * KT_W + x];
            } else {
                k0 = __ldg(key + ko);
                k1 = __ldg(key + ko + PL);
            }
            // the key's Shoup companions (stored after the key words, KW apart):
            // a constant-operand product instead of a Barrett reduction
            const u64 s0 = __ldg(key + KW + ko), s1 = __ldg(key + KW + ko + PL);
            mac_term(a0, w, k0, s0, q);
            mac_term(a1, w, k1, s1, q);
        }
        work[s0] = mac_reduce(a0, md);
        work[TW + s0] = mac_reduce(a1, md);
    }
    __syncthreads();
    load_block_twiddles<LOGN, LN>(tws, dc->tw[j].inv, blk0);
    cp_async_wait_all();
    __syncthreads();
    line_ntt_v<G::B, 0, true, KMR, LN>(work + grp * TW, SpecQ{q}, addr, twf, tg);  // group p: accumulator p
    __syncthreads();
#pragma unroll
    for (int p = 0; p < 2; ++p) {
        u64* dst = ACC + (((size_t)item * 2 + p) * LK + j) * G::N + base;
#pragma unroll
        for (int r = 0; r < PER; ++r) {
            const int x = threadIdx.x + T * r;
            dst[x] = work[p * TW + saddr(x)];
        }
    }
}

// ---------------------------------------------------------------------------
// K2h: hoisted rotations (level 0).  Every rotation of one source shares
// H = NTT(ModUp(c1)) (K1 without the automorphism + the forward block phase,
// once per source); a rotation by g reads H in the NTT domain permuted by g
// (position p holds a(psi^(2 brv(p) + 1)), so NTT(phi_g a)[p] = NTT(a)[p'] with
// 2 brv(p') + 1 = g (2 brv(p) + 1) mod 2N), then the key MAC and the inverse
// block phase of both accumulators as K2.  The words equal the unhoisted key
// switch (phi_g(ModUp(c1)), DESIGN 2.9); a second rotation of the same source
// costs no ModUp and no forward transform.
// ---------------------------------------------------------------------------
template <int LOGN>
__device__ __forceinline__ int ntt_perm(u32 g, int p) {
    constexpr u32 TWO_N_MASK = 2u * (1u << LOGN) - 1u;
    const u32 e = 2u * (__brev((u32)p) >> (32 - LOGN)) + 1u;
    const u32 e2 = (g * e) & TWO_N_MASK;
    return (int)(__brev((e2 - 1u) >> 1) >> (32 - LOGN));
}

template <int LOGN, int LT, int KT, int AT, int LN = 16>
__global__ void __launch_bounds__(kKsGroups * kKsGroupThreads) k_ks_blocks_gather(const DevConsts* __restrict__ dc,
                                                                                const u64* __restrict__ H,
                                                                                const int* __restrict__ HIDX,
                                                                                const u32* __restrict__ GEL,
                                                                                const u64* const* KEY, int nterm,
                                                                                const int* __restrict__ ORDER,
                                                                                u64* __restrict__ ACC) {
    using G = Ntt2<LOGN>;
    extern __shared__ u64 smem[];
    constexpr int PITCH = G::PITCH;
    constexpr int TW = LN * PITCH;
    constexpr int T = kKsGroups * kKsGroupThreads;
    constexpr int PER = LN * G::R2 / T;
    constexpr int KMR = LN >= 16 ? 4 : 2;
    constexpr int CTAS = G::R1 / LN;
    static_assert(PER >= 1, "tile smaller than the CTA");
    const int L = LT ? LT : dc->L, K = KT ? KT : dc->K, LK = L + K;
    const int alpha = AT ? AT : dc->alpha, dnum = (L + alpha - 1) / alpha;
    u64* work = smem;  // acc0 in tile 0, acc1 in tile 1
    u64* tws = smem + 2 * TW;
    int bid = blockIdx.x;
    const int tileid = bid % CTAS;
    bid /= CTAS;
    const int j = bid % LK;
    // ORDER: items sharing switching keys run back to back (the keys stay in L2)
    const int item = ORDER ? ORDER[bid / LK] : bid / LK;
    const Modulus md = dc->mod[j];
    const u64 q = md.q;
    const int blk0 = tileid * LN;
    const size_t base = (size_t)blk0 * G::R2;
    const size_t PL = (size_t)LK * G::N;
    const size_t KW = (size_t)dnum * 2 * PL;  // key words; their Shoup companions follow
    const int grp = threadIdx.x / kKsGroupThreads;
    const ThreadGroup tg = cta_slice(grp, kKsGroups);
    auto saddr = [](int x) { return (x >> G::B) * PITCH + (x & (G::R2 - 1)); };
    auto addr = [](int l, int pos) { return l * PITCH + pos; };
    auto twf = [&](int sl, int l, int blk) { return block_tw<LOGN, LN>(tws, sl, l, blk); };
    load_block_twiddles<LOGN, LN>(tws, dc->tw[j].inv, blk0);
    u64 a0[PER], a1[PER];
#pragma unroll
    for (int r = 0; r < PER; ++r) a0[r] = a1[r] = 0;
    // lazy sums (see K2): at most kLazyMacTerms products < 2q between reductions
    int pend = 0;
    for (int t = 0; t < nterm; ++t) {
        const int hi = HIDX[item * nterm + t];
        if (hi < 0) continue;
        const u64* h = H + (size_t)hi * dnum * PL + (size_t)j * G::N;
        const u32 g = GEL[item * nterm + t];
        const u64* key = KEY[item * nterm + t];
        for (int dg = 0; dg < dnum; ++dg) {
            // every load of the term first (gathered digit, both key words and
            // their companions for all PER elements), then the products
            u64 w[PER], k0[PER], k1[PER], c0[PER], c1[PER];
            if (pend == kLazyMacTerms) {
#pragma unroll
                for (int r = 0; r < PER; ++r) {
                    a0[r] = mac_reduce(a0[r], md);
                    a1[r] = mac_reduce(a1[r], md);
                }
                pend = 1;
            }
            ++pend;
#pragma unroll
            for (int r = 0; r < PER; ++r) {
                const int x = threadIdx.x + T * r;
                const size_t ko = ((size_t)dg * 2) * PL + (size_t)j * G::N + base + x;
                w[r] = __ldg(h + (size_t)dg * PL + ntt_perm<LOGN>(g, (int)base + x));
                k0[r] = __ldg(key + ko);
                k1[r] = __ldg(key + ko + PL);
                c0[r] = __ldg(key + KW + ko);
                c1[r] = __ldg(key + KW + ko + PL);
            }
#pragma unroll
            for (int r = 0; r < PER; ++r) {
                mac_term(a0[r], w[r], k0[r], c0[r], q);
                mac_term(a1[r], w[r], k1[r], c1[r], q);
            }
        }
    }
#pragma unroll
    for (int r = 0; r < PER; ++r) {
        const int s0 = saddr(threadIdx.x + T * r);
        work[s0] = mac_reduce(a0[r], md);
        work[TW + s0] = mac_reduce(a1[r], md);
    }
    cp_async_wait_all();
    __syncthreads();
    line_ntt_v<G::B, 0, true, KMR, LN>(work + grp * TW, SpecQ{q}, addr, twf, tg);  // group p: accumulator p
    __syncthreads();
#pragma unroll
    for (int p = 0; p < 2; ++p) {
        u64* dst = ACC + (((size_t)item * 2 + p) * LK + j) * G::N + base;
#pragma unroll
        for (int r = 0; r < PER; ++r) {
            const int x = threadIdx.x + T * r;
            dst[x] = work[p * TW + saddr(x)];
        }
    }
}

// ---------------------------------------------------------------------------
// launch
// ---------------------------------------------------------------------------
template <class F>
static void ks_dispatch_shape(const RnsParams& P, F&& f) {
    const auto& c = P.cfg;
    using std::integral_constant;
    if (c.L == 2 && c.K == 2 && c.alpha == 2)
        f(integral_constant<int, 2>{}, integral_constant<int, 2>{}, integral_constant<int, 2>{});
    else if (c.L == 4 && c.K == 4 && c.alpha == 4)
        f(integral_constant<int, 4>{}, integral_constant<int, 4>{}, integral_constant<int, 4>{});
    else
        f(integral_constant<int, 0>{}, integral_constant<int, 0>{}, integral_constant<int, 0>{});
}

// K1 (ModUp + column phase) of `items` sources into DX: the all-limbs kernel
// for launches of a wave or more, per-limb 16/8/4-column tiles below
template <int LOGN, int LT, int KT, int AT>
static void launch_k1(const DevConsts* dc, const RnsParams& P, const u64* const* SRC, const u64* SRCC, int src_poly,
                      const u32* ginv, u64* DX, int items, cudaStream_t st, const KsY& ky) {
    using G = Ntt2<LOGN>;
    const int LK = P.cfg.L + P.cfg.K, dnum = P.dnum;
    const int smem1 = G::SMEM_C;
    smem_optin_k(k_ks_modup_cols<LOGN, LT, KT, AT>, smem1);
    bool k1_done = false;
    constexpr int LCA = LT ? modup_all_lc<LT, KT>() : 0;
    constexpr bool HALF = LCA >= 4 && G::R1 * LCA / 2 >= G::TC && (G::R1 * LCA / 4 * (LT + KT)) % G::TC == 0;
    if constexpr (LCA >= 2 && G::R1 * LCA >= G::TC && (G::R1 * LCA / 2 * (LT + KT)) % G::TC == 0) {
        const bool small = cols_use_ln8((long)items * dnum * LK * G::CTAS_C, G::R1 * 4 >= G::TC);
        if (k1_all_mode() != 0 && (!small || (HALF && k1_all_mode() == 1))) {
            // 16 lines, or 8 (half the columns per CTA) when the launch would not fill the GPU
            constexpr int VL = (LT + KT) * LCA;
            auto go = [&](auto lc_) {
                constexpr int LC = decltype(lc_)::value;
                const int smemA = (VL / (LCA / LC) * G::R1 + (LT + KT) * (2 * G::R1 + 2)) * 8;
                smem_optin_k(k_ks_modup_all<LOGN, LT, KT, AT, LC>, smemA);
                k_ks_modup_all<LOGN, LT, KT, AT, LC><<<items * dnum * (G::R2 / LC), G::TC, smemA, st>>>(
                    dc, SRC, SRCC, src_poly, ginv, DX, ky.src, ky.srcc);
            };
            if constexpr (HALF)
                if (small) {
                    go(std::integral_constant<int, LCA / 2>{});
                    k1_done = true;
                }
            if (!k1_done)
                go(std::integral_constant<int, LCA>{});
            k1_done = true;
        }
    }
    if (k1_done) {
    } else if (cols_use_ln4((long)items * dnum * LK * G::CTAS_C, G::R1 >= G::TC)) {  // 4-column tiles
        constexpr int LN = 4;
        k_ks_modup_cols<LOGN, LT, KT, AT, LN><<<items * dnum * LK * (G::R2 / LN), G::TC,
                                                (LN * G::R1 + 2 * G::R1) * 8, st>>>(dc, SRC, SRCC, src_poly, ginv, DX, ky.src, ky.srcc);
    } else if (cols_use_ln8((long)items * dnum * LK * G::CTAS_C, G::R1 * 4 >= G::TC)) {  // 8-column tiles
        constexpr int LN = 8;
        k_ks_modup_cols<LOGN, LT, KT, AT, LN><<<items * dnum * LK * (G::R2 / LN), G::TC,
                                                (LN * G::R1 + 2 * G::R1) * 8, st>>>(dc, SRC, SRCC, src_poly, ginv, DX, ky.src, ky.srcc);
    } else {
        k_ks_modup_cols<LOGN, LT, KT, AT><<<items * dnum * LK * G::CTAS_C, G::TC, smem1, st>>>(dc, SRC, SRCC,
                                                                                          src_poly, ginv, DX, ky.src,
                                                                                          ky.srcc);
    }
    KS_CHECK();
    kmark("k_ks_modup_cols (K1)", st);
}

// inverse column phase of ACC + ModDown + base + extra + phi_g(rsrc.c0); XACC
// (nullable): other key switches' accumulators added before the shared INTT +
// ModDown (inside the fused inverse-cols + ModDown kernel, else one add pass)
template <int LOGN, int LT>
static void launch_ks_tail(const DevConsts* dc, const RnsParams& P, const u64* const* BASE, const u64* const* RSRC,
                           const u32* ginv, u64* const* OUT, u64* ACC, int items, cudaStream_t st,
                           const u64* const* EXTRA, const int* PAIR, u64* const* YOUT,
                           const u64* const* XACC = nullptr) {
    const int LK = P.cfg.L + P.cfg.K;
    NttJob j;
    for (int i = 0; i < MAX_JOB_LIMBS; ++i) j.pidx[i] = (signed char)(i % LK);
    j.src = ACC;
    j.dst = ACC;
    j.limbs = 2 * LK;
    if (launch_ks_cols_moddown(dc, P, ACC, BASE, RSRC, ginv, OUT, items, st, EXTRA, PAIR, YOUT, XACC)) {
        kmark("k_ks_cols_moddown (inv cols + ModDown)", st);
        return;
    }
    j.add_items = XACC;           // folded into the inverse column phase's tile load
    j.lazy_out = LT > 0 ? 1 : 0;  // the fixed-shape ModDown folds N^-1 into its constants
    launch_ntt_phase(dc, LOGN, /*inverse=*/true, /*cols=*/true, j, items, st);
    kmark("k_ntt_cols inv (key switch)", st);
    launch_ks_moddown(dc, P, ACC, BASE, RSRC, ginv, OUT, items, st, EXTRA, PAIR, YOUT, j.lazy_out != 0);
    kmark("k_ks_moddown_k", st);
}

// accumulate phase: ACC[item] = the key products of phi_g(ModUp(c1)), in the
// domain the tail expects; returns true when the cluster kernel produced them
// (coefficient domain: ModDown only)
template <int LOGN, int LT, int KT, int AT>
static bool ks_accumulate_t(const DevConsts* dc, const RnsParams& P, const u64* const* SRC, const u64* SRCC,
                            int src_poly, const u32* ginv, const u64* const* KEY, u64* DX, u64* ACC, int items,
                            cudaStream_t st, const KsY& ky) {
    using G = Ntt2<LOGN>;
    if (launch_ks_cluster(dc, P, SRC, SRCC, src_poly, ginv, KEY, ACC, items, st)) return true;
    const int L = P.cfg.L, K = P.cfg.K, LK = L + K, dnum = P.dnum;
    constexpr int KTM = ks_keys_tma<LOGN>() ? 1 : 0;
    const int smem2 =
        ((dnum < 2 ? 2 : dnum) * G::LINES * G::PITCH + 2 * G::TWB + KTM * dnum * 2 * G::LINES * G::R2) * 8 + 16;
    const int smem2h =
        ((dnum < 2 ? 2 : dnum) * 8 * G::PITCH + 2 * btw_entries<LOGN, 8>() + KTM * dnum * 2 * 8 * G::R2) * 8 + 16;
    if (smem2 > 200 * 1024)
        throw std::invalid_argument("key switch: too many digits for the fused kernel; set fused_key_switch 0");
    smem_optin_k(k_ks_blocks_inner<LOGN, LT, KT, AT>, smem2);
    smem_optin_k(k_ks_blocks_inner<LOGN, LT, KT, AT, 8>, smem2h);
    launch_k1<LOGN, LT, KT, AT>(dc, P, SRC, SRCC, src_poly, ginv, DX, items, st, ky);
    constexpr int T2 = kKsGroups * kKsGroupThreads;
    if (blocks_use_ln8((long)items * LK * G::CTAS_B) && 8 * G::R2 >= T2)  // small launch: 8-block tiles
        k_ks_blocks_inner<LOGN, LT, KT, AT, 8><<<items * LK * (G::R1 / 8), T2, smem2h, st>>>(dc, DX, KEY, ACC);
    else
        k_ks_blocks_inner<LOGN, LT, KT, AT><<<items * LK * G::CTAS_B, T2, smem2, st>>>(dc, DX, KEY, ACC);
    KS_CHECK();
    kmark("k_ks_blocks_inner (K2)", st);
    return false;
}

template <int LOGN, int LT, int KT, int AT>
static void ks_fused_t(const DevConsts* dc, const RnsParams& P, const u64* const* SRC, const u64* SRCC,
                       int src_poly, const u32* ginv, const u64* const* KEY, const u64* const* BASE,
                       const u64* const* RSRC, u64* const* OUT, u64* DX, u64* ACC, int items, cudaStream_t st,
                       const u64* const* EXTRA, const int* PAIR, const KsY& ky) {
    if (ks_accumulate_t<LOGN, LT, KT, AT>(dc, P, SRC, SRCC, src_poly, ginv, KEY, DX, ACC, items, st, ky)) {
        launch_ks_moddown(dc, P, ACC, BASE, RSRC, ginv, OUT, items, st, EXTRA, PAIR, ky.out);
        return;
    }
    launch_ks_tail<LOGN, LT>(dc, P, BASE, RSRC, ginv, OUT, ACC, items, st, EXTRA, PAIR, ky.out);
}

// Hoisted accumulate: K1 (no automorphism) + the forward block phase of every
// source once (H in DX), then K2h per rotation into ACC
template <int LOGN, int LT, int KT, int AT>
static void ks_hoisted_acc_t(const DevConsts* dc, const RnsParams& P, const HoistedKs& hk, const u64* const* KEY,
                             u64* DX, u64* ACC, int items, cudaStream_t st) {
    using G = Ntt2<LOGN>;
    const int LK = P.cfg.L + P.cfg.K, dnum = P.dnum;
    KsY ky;
    ky.src = hk.ysrc;
    launch_k1<LOGN, LT, KT, AT>(dc, P, hk.src, nullptr, hk.src_poly, nullptr, DX, hk.nsrc, st, ky);
    NttJob jb;
    for (int i = 0; i < MAX_JOB_LIMBS; ++i) jb.pidx[i] = (signed char)(i % LK);
    jb.src = DX;
    jb.dst = DX;
    jb.limbs = dnum * LK;
    launch_ntt_phase(dc, LOGN, /*inverse=*/false, /*cols=*/false, jb, hk.nsrc, st);
    kmark("k_ntt_blocks fwd (hoisted ModUp)", st);
    constexpr int T2 = kKsGroups * kKsGroupThreads;
    if (blocks_use_ln8((long)items * LK * G::CTAS_B) && 8 * G::R2 >= T2) {
        const int sm = (2 * 8 * G::PITCH + 2 * btw_entries<LOGN, 8>()) * 8;
        smem_optin_k(k_ks_blocks_gather<LOGN, LT, KT, AT, 8>, sm);
        k_ks_blocks_gather<LOGN, LT, KT, AT, 8><<<items * LK * (G::R1 / 8), T2, sm, st>>>(dc, DX, hk.hidx, hk.gel,
                                                                                        KEY, hk.nterm, hk.order, ACC);
    } else {
        const int sm = (2 * G::LINES * G::PITCH + 2 * G::TWB) * 8;
        smem_optin_k(k_ks_blocks_gather<LOGN, LT, KT, AT>, sm);
        k_ks_blocks_gather<LOGN, LT, KT, AT><<<items * LK * G::CTAS_B, T2, sm, st>>>(dc, DX, hk.hidx, hk.gel, KEY,
                                                                                     hk.nterm, hk.order, ACC);
    }
    KS_CHECK();
    kmark("k_ks_blocks_gather (K2h)", st);
}

template <int LOGN>
static void ks_fused_logn(const DevConsts* dc, const RnsParams& P, const u64* const* SRC, const u64* SRCC,
                          int src_poly, const u32* ginv, const u64* const* KEY, const u64* const* BASE,
                          const u64* const* RSRC, u64* const* OUT, u64* DX, u64* ACC, int items, cudaStream_t st,
                       const u64* const* EXTRA, const int* PAIR, const KsY& ky) {
    ks_dispatch_shape(P, [&](auto l_, auto k_, auto a_) {
        ks_fused_t<LOGN, decltype(l_)::value, decltype(k_)::value, decltype(a_)::value>(
            dc, P, SRC, SRCC, src_poly, ginv, KEY, BASE, RSRC, OUT, DX, ACC, items, st, EXTRA, PAIR, ky);
    });
}

template <class F>
static void logn_dispatch(int logn, F&& f) {
    switch (logn) {
        case 10: f(std::integral_constant<int, 10>{}); break;
        case 11: f(std::integral_constant<int, 11>{}); break;
        case 12: f(std::integral_constant<int, 12>{}); break;
        case 13: f(std::integral_constant<int, 13>{}); break;
        case 14: f(std::integral_constant<int, 14>{}); break;
        case 15: f(std::integral_constant<int, 15>{}); break;
        default: throw std::invalid_argument("key switch: unsupported logn");
    }
}

KsAccDomain launch_ks_accumulate(const DevConsts* dc, const RnsParams& P, bool fused, const u64* const* SRC,
                                 const u32* ginv, const u64* const* KEY, u64* DX, u64* ACC, int items,
                                 cudaStream_t st, const KsY& ky, const HoistedKs* hk) {
    if (!items) return KsAccDomain::BlockInv;
    if (!fused) {  // ModUp, NTT, inner product: the NTT domain
        const int LK = P.cfg.L + P.cfg.K;
        launch_ks_modup(dc, P, SRC, 1, ginv, DX, items, st);
        NttJob j;
        for (int i = 0; i < MAX_JOB_LIMBS; ++i) j.pidx[i] = (signed char)(i % LK);
        j.src = DX;
        j.dst = DX;
        j.limbs = P.dnum * LK;
        launch_ntt(dc, P.cfg.logn, false, j, items, st);
        launch_ks_inner(dc, P, DX, KEY, ACC, items, st);
        return KsAccDomain::Ntt;
    }
    KsAccDomain dom = KsAccDomain::BlockInv;
    logn_dispatch(P.cfg.logn, [&](auto lg_) {
        constexpr int LG = decltype(lg_)::value;
        ks_dispatch_shape(P, [&](auto l_, auto k_, auto a_) {
            constexpr int LT = decltype(l_)::value, KT = decltype(k_)::value, AT = decltype(a_)::value;
            if (hk)
                ks_hoisted_acc_t<LG, LT, KT, AT>(dc, P, *hk, KEY, DX, ACC, items, st);
            else if (ks_accumulate_t<LG, LT, KT, AT>(dc, P, SRC, nullptr, 1, ginv, KEY, DX, ACC, items, st, ky))
                dom = KsAccDomain::Coeff;
        });
    });
    return dom;
}

void launch_ks_finish(const DevConsts* dc, const RnsParams& P, KsAccDomain dom, const u64* const* BASE,
                      const u64* const* RSRC, const u32* ginv, u64* const* OUT, u64* ACC, int items, cudaStream_t st,
                      const u64* const* EXTRA, u64* const* YOUT, const u64* const* XACC) {
    if (!items) return;
    if (dom == KsAccDomain::Coeff) {
        launch_acc_add(dc, P, ACC, XACC, items, st);
        launch_ks_moddown(dc, P, ACC, BASE, RSRC, ginv, OUT, items, st, EXTRA, nullptr, YOUT);
        return;
    }
    if (dom == KsAccDomain::Ntt) {
        const int LK = P.cfg.L + P.cfg.K;
        launch_acc_add(dc, P, ACC, XACC, items, st);
        NttJob j;
        for (int i = 0; i < MAX_JOB_LIMBS; ++i) j.pidx[i] = (signed char)(i % LK);
        j.src = ACC;
        j.dst = ACC;
        j.limbs = 2 * LK;
        launch_ntt(dc, P.cfg.logn, true, j, items, st);
        launch_ks_moddown(dc, P, ACC, BASE, RSRC, ginv, OUT, items, st, EXTRA, nullptr, YOUT);
        return;
    }
    logn_dispatch(P.cfg.logn, [&](auto lg_) {
        constexpr int LG = decltype(lg_)::value;
        ks_dispatch_shape(P, [&](auto l_, auto, auto) {
            launch_ks_tail<LG, decltype(l_)::value>(dc, P, BASE, RSRC, ginv, OUT, ACC, items, st, EXTRA, nullptr, YOUT,
                                                    XACC);
        });
    });
}

void launch_ks_fused(const DevConsts* dc, const RnsParams& P, const u64* const* SRC, const u64* SRCC,
                     int src_poly, const u32* ginv, const u64* const* KEY, const u64* const* BASE,
                     const u64* const* RSRC, u64* const* OUT, u64* DX, u64* ACC, int items, cudaStream_t st,
                       const u64* const* EXTRA, const int* PAIR, const KsY& ky) {
    if (!items) return;
    switch (P.cfg.logn) {
        case 10: ks_fused_logn<10>(dc, P, SRC, SRCC, src_poly, ginv, KEY, BASE, RSRC, OUT, DX, ACC, items, st, EXTRA, PAIR, ky); break;
        case 11: ks_fused_logn<11>(dc, P, SRC, SRCC, src_poly, ginv, KEY, BASE, RSRC, OUT, DX, ACC, items, st, EXTRA, PAIR, ky); break;
        case 12: ks_fused_logn<12>(dc, P, SRC, SRCC, src_poly, ginv, KEY, BASE, RSRC, OUT, DX, ACC, items, st, EXTRA, PAIR, ky); break;
        case 13: ks_fused_logn<13>(dc, P, SRC, SRCC, src_poly, ginv, KEY, BASE, RSRC, OUT, DX, ACC, items, st, EXTRA, PAIR, ky); break;
        case 14: ks_fused_logn<14>(dc, P, SRC, SRCC, src_poly, ginv, KEY, BASE, RSRC, OUT, DX, ACC, items, st, EXTRA, PAIR, ky); break;
        case 15: ks_fused_logn<15>(dc, P, SRC, SRCC, src_poly, ginv, KEY, BASE, RSRC, OUT, DX, ACC, items, st, EXTRA, PAIR, ky); break;
        default: throw std::invalid_argument("key switch: unsupported logn");
    }
}

}  // namespace cssc
