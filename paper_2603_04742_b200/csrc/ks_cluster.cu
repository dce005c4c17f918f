// ks_cluster.cu -- the key switch's ModUp + NTT + key product + INTT as one
// thread-block-cluster kernel: the two NTT phases exchange their tiles through
// distributed shared memory instead of HBM.
//
// One cluster of CL = R2/16 CTAs owns one target limb j of one item.  CTA c
// holds columns [16c, 16c+16) in the column phase and rows [c*RB, (c+1)*RB)
// (RB = R1/CL blocks) in the block phase:
//   for each digit:  ModUp (E3, with the automorphism gather) of its 16 columns
//                    -> column-phase NTT -> cluster barrier -> transpose: read
//                    its RB rows from every CTA's column tile (DSMEM) -> block-
//                    phase NTT -> multiply by both key tiles, accumulate
//   then:            block-phase INTT of both accumulators -> cluster barrier
//                    -> transpose back (DSMEM) -> column-phase INTT, x N^-1
//                    -> ACC[item][2][L+K][N] in coefficient form (for ModDown)
// It replaces K1, K2 and the inverse column launch (three launches, and the
// DX and middle-domain ACC round trips through HBM).  Same integer formulas as
// the other paths, so the words are identical.
#include <cooperative_groups.h>

#include <cstdlib>
#include <stdexcept>
#include <string>

#include "bfv_kernels.cuh"
#include "ntt.cuh"

namespace cg = cooperative_groups;

namespace cssc {

namespace {

__device__ __forceinline__ int cl_automorph(u32 ginv, int k, int n, bool& neg) {
    if (ginv == 0) {
        neg = false;
        return k;
    }
    const u32 i0 = (u32)(((unsigned long long)ginv * (unsigned)k) & (unsigned long long)(2 * n - 1));
    neg = i0 >= (u32)n;
    return neg ? (int)(i0 - n) : (int)i0;
}

template <int LOGN>
struct KsCl {
    using G = Ntt2<LOGN>;
    static constexpr int CL = G::R2 / 16;       // CTAs per cluster (one limb)
    static constexpr int RB = G::R1 / CL;       // block-phase rows per CTA
    static constexpr int T = 512;               // threads per CTA
    static constexpr int CT = 16 * G::R1;       // column tile words
    static constexpr int BT = RB * G::PITCH;    // block tile words
    static constexpr int SMEM_WORDS = 2 * CT + 3 * BT + 4 * G::R1;
    static constexpr int SMEM = SMEM_WORDS * 8;
};

}  // namespace

template <int LOGN, int LT, int KT, int AT>
__global__ void __cluster_dims__(KsCl<LOGN>::CL, 1, 1) __launch_bounds__(KsCl<LOGN>::T, 1)
    k_ks_cluster(const DevConsts* __restrict__ dc, const u64* const* SRC, const u64* SRCC, int src_poly,
                 const u32* ginv, const u64* const* KEY, u64* __restrict__ ACC) {
    using G = Ntt2<LOGN>;
    using C = KsCl<LOGN>;
    constexpr int L = LT, K = KT, LK = L + K, alpha = AT, dnum = (L + alpha - 1) / alpha;
    constexpr int T = C::T, RB = C::RB, PITCH = G::PITCH;
    extern __shared__ u64 smem[];
    u64* ct = smem;                  // column tile [R1][16]: digits, then accumulator 0
    u64* ct1 = smem + C::CT;         // column tile of accumulator 1
    u64* bt = ct1 + C::CT;           // block tile [RB][PITCH] of the current digit
    u64* b0 = bt + C::BT;            // accumulators in the block domain
    u64* b1 = b0 + C::BT;
    u64* twf_s = b1 + C::BT;         // column twiddles: forward R1 pairs
    u64* twi_s = twf_s + 2 * G::R1;  // inverse R1 pairs
    cg::cluster_group cluster = cg::this_cluster();
    const int rank = (int)cluster.block_rank();
    const int limb_task = blockIdx.x / C::CL;
    const int j = limb_task % LK;
    const int item = limb_task / LK;
    const Modulus md = dc->mod[j];
    const u64 q = md.q;
    const u64* src = SRC ? SRC[item] + (size_t)src_poly * L * G::N : SRCC + (size_t)item * L * G::N;
    const u32 gi = ginv ? ginv[item] : 0u;
    const u64* key = KEY[item];
    const size_t PL = (size_t)LK * G::N;
    const int col0 = rank * 16;
    const int row0 = rank * RB;
    for (int i = threadIdx.x; i < G::R1; i += T) {
        cp_async16(twf_s + 2 * i, dc->tw[j].fwd + 2 * i);
        cp_async16(twi_s + 2 * i, dc->tw[j].inv + 2 * i);
    }
    cp_async_wait_all();
    __syncthreads();
    auto addr_c = [](int l, int pos) { return pos * 16 + l; };
    auto tw_cf = [&](int sl, int, int blk) {
        const int k = (1 << sl) + blk;
        return make_ulonglong2(twf_s[2 * k], twf_s[2 * k + 1]);
    };
    auto tw_ci = [&](int sl, int, int blk) {
        const int k = (1 << sl) + blk;
        return make_ulonglong2(twi_s[2 * k], twi_s[2 * k + 1]);
    };
    auto addr_b = [](int l, int pos) { return l * PITCH + pos; };
    const ulonglong2* twb_f = reinterpret_cast<const ulonglong2*>(dc->tw[j].fwd);
    const ulonglong2* twb_i = reinterpret_cast<const ulonglong2*>(dc->tw[j].inv);
    // block-phase twiddles straight from the (L2-resident) table: W[2^(A+s) + blk_g 2^s + b]
    auto tw_bf = [&](int sl, int l, int blk) { return __ldg(twb_f + (1 << (G::A + sl)) + ((row0 + l) << sl) + blk); };
    auto tw_bi = [&](int sl, int l, int blk) { return __ldg(twb_i + (1 << (G::A + sl)) + ((row0 + l) << sl) + blk); };

#pragma unroll 1
    for (int dg = 0; dg < dnum; ++dg) {
        const int lo = dg * alpha, hi = lo + alpha < L ? lo + alpha : L;
        const bool own = j >= lo && j < hi;
        if (dg) cluster.sync();  // every CTA finished reading the previous digit's column tile
        // ModUp of this CTA's 16 columns (E3), automorphism gather
#pragma unroll 4
        for (int r = 0; r < G::R1 * 16 / T; ++r) {
            const int e = threadIdx.x + T * r, c = e >> 4, jl = e & 15;
            bool neg;
            const int idx = cl_automorph(gi, col0 + jl + G::R2 * c, G::N, neg);
            u64 v;
            if (own) {
                const u64 x = __ldg(src + (size_t)j * G::N + idx);
                v = neg ? neg_mod(x, q) : x;
            } else {
                v = 0;
#pragma unroll
                for (int i = lo; i < lo + alpha; ++i) {
                    if (i >= hi) break;
                    const u64 qi = dc->mod[i].q;
                    const u64 x = __ldg(src + (size_t)i * G::N + idx);
                    const u64 y = shoup(x, dc->dig_hat_inv[i], dc->dig_hat_inv_sh[i], qi);
                    v += shoup_lazy(y, dc->dig_hat[i][j], dc->dig_hat_sh[i][j], q);
                }
                v = reduce_small_quot(v, md);
                v = neg ? neg_mod(v, q) : v;  // phi_g(ModUp(x)) (DESIGN 2.9)
            }
            ct[c * 16 + jl] = v;
        }
        __syncthreads();
        line_ntt_v<G::A, 0, false, 3, 16>(ct, ConstQ{q}, addr_c, tw_cf, whole_cta());
        cluster.sync();  // all column tiles of the limb complete
        // transpose: rows [row0, row0 + RB) x all R2 columns, from every CTA (DSMEM)
#pragma unroll 4
        for (int r = 0; r < RB * G::R2 / T; ++r) {
            const int e = threadIdx.x + T * r, rr = e / G::R2, col = e % G::R2;
            const u64* remote = cluster.map_shared_rank(ct, col >> 4);
            bt[rr * PITCH + col] = remote[(row0 + rr) * 16 + (col & 15)];
        }
        __syncthreads();
        line_ntt_v<G::B, 0, false, 3, RB>(bt, ConstQ{q}, addr_b, tw_bf, whole_cta());
        // key product: element (rr, col) is NTT index (row0 + rr) * R2 + col
        const u64* k0 = key + ((size_t)dg * 2 + 0) * PL + (size_t)j * G::N + (size_t)row0 * G::R2;
        const u64* k1 = key + ((size_t)dg * 2 + 1) * PL + (size_t)j * G::N + (size_t)row0 * G::R2;
#pragma unroll 4
        for (int r = 0; r < RB * G::R2 / T; ++r) {
            const int e = threadIdx.x + T * r, s0 = (e / G::R2) * PITCH + (e % G::R2);
            const u64 w = bt[s0];
            const u64 p0 = mul_mod(w, __ldg(k0 + e), md), p1 = mul_mod(w, __ldg(k1 + e), md);
            b0[s0] = dg ? add_mod(b0[s0], p0, q) : p0;
            b1[s0] = dg ? add_mod(b1[s0], p1, q) : p1;
        }
        __syncthreads();
    }
    // inverse block phase of both accumulators, concurrently on two thread groups
    {
        const int grp = threadIdx.x / (T / 2);
        line_ntt_v<G::B, 0, true, 3, RB>(grp ? b1 : b0, ConstQ{q}, addr_b, tw_bi, cta_slice(grp, 2));
    }
    cluster.sync();  // all block tiles complete (and every digit column tile consumed)
    // transpose back: this CTA's 16 columns x all R1 rows, from every CTA's block tiles
#pragma unroll 4
    for (int r = 0; r < G::R1 * 16 / T; ++r) {
        const int e = threadIdx.x + T * r, row = e >> 4, l = e & 15;
        const int owner = row / RB, rr = row - owner * RB;
        const u64* r0 = cluster.map_shared_rank(b0, owner);
        const u64* r1 = cluster.map_shared_rank(b1, owner);
        ct[row * 16 + l] = r0[rr * PITCH + col0 + l];
        ct1[row * 16 + l] = r1[rr * PITCH + col0 + l];
    }
    cluster.sync();  // nobody reads this CTA's block tiles any more
    {
        const int grp = threadIdx.x / (T / 2);
        line_ntt_v<G::A, 0, true, 3, 16>(grp ? ct1 : ct, ConstQ{q}, addr_c, tw_ci, cta_slice(grp, 2));
    }
    __syncthreads();
    const u64 ni = dc->ninv[j], nish = dc->ninv_sh[j];
#pragma unroll
    for (int p = 0; p < 2; ++p) {
        const u64* tile = p ? ct1 : ct;
        u64* dst = ACC + (((size_t)item * 2 + p) * LK + j) * G::N;
#pragma unroll 4
        for (int r = 0; r < G::R1 * 8 / T; ++r) {
            const int i = threadIdx.x + T * r, c = i >> 3, h = i & 7;
            const u64 a0 = shoup(tile[c * 16 + 2 * h], ni, nish, q), a1 = shoup(tile[c * 16 + 2 * h + 1], ni, nish, q);
            *reinterpret_cast<ulonglong2*>(dst + (size_t)c * G::R2 + col0 + 2 * h) = make_ulonglong2(a0, a1);
        }
    }
}

template <int LOGN, int LT, int KT, int AT>
static bool ks_cluster_t(const DevConsts* dc, const u64* const* SRC, const u64* SRCC, int src_poly, const u32* ginv,
                         const u64* const* KEY, u64* ACC, int items, cudaStream_t st) {
    using C = KsCl<LOGN>;
    if constexpr (LT == 0 || C::CL < 2 || C::CL > 8 || (C::RB * Ntt2<LOGN>::R2) % C::T != 0) {
        return false;
    } else {
        try {
            smem_optin_k(k_ks_cluster<LOGN, LT, KT, AT>, C::SMEM);
        } catch (const std::exception&) {
            cudaGetLastError();
            return false;
        }
        const int LK = LT + KT;
        k_ks_cluster<LOGN, LT, KT, AT><<<items * LK * C::CL, C::T, C::SMEM, st>>>(dc, SRC, SRCC, src_poly, ginv, KEY,
                                                                                  ACC);
        const cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) throw std::runtime_error(std::string("ks cluster launch: ") + cudaGetErrorString(e));
        return true;
    }
}

bool launch_ks_cluster(const DevConsts* dc, const RnsParams& P, const u64* const* SRC, const u64* SRCC,
                       int src_poly, const u32* ginv, const u64* const* KEY, u64* ACC, int items, cudaStream_t st) {
    static const int enabled = [] {
        const char* e = std::getenv("CSSC_KS_CLUSTER");
        return e ? std::atoi(e) : 0;  // opt-in: slower than K1+K2 (DESIGN 9)
    }();
    if (!enabled || !items) return false;
    const auto& c = P.cfg;
#define CSSC_KSC(LG, L_, K_, A_) \
    if (c.logn == LG && c.L == L_ && c.K == K_ && c.alpha == A_) \
        return ks_cluster_t<LG, L_, K_, A_>(dc, SRC, SRCC, src_poly, ginv, KEY, ACC, items, st);
    CSSC_KSC(13, 2, 2, 2)
    CSSC_KSC(14, 2, 2, 2)
    CSSC_KSC(15, 4, 4, 4)
#undef CSSC_KSC
    return false;
}

}  // namespace cssc
