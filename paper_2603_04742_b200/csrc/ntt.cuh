// ntt.cuh -- batched negacyclic NTT / INTT for RNS limbs on sm_100a.
//
// Convention (shared with DESIGN.md "Arithmetic spec" and the CPU oracle):
// forward Cooley-Tukey with the psi-power table W[k] = psi^bitrev(k); output
// position p holds a(psi^(2*bitrev(p)+1)).  Inverse Gentleman-Sande with
// psi^-bitrev(k), then a multiplication by N^-1.  Outputs are canonical, so
// any correct NTT agrees word for word with the oracle.
//
// Two-phase ("columns, then blocks") structure, N = R1 * R2:
//   phase C: stages 0..A-1 act on the R2 strided columns {j + R2*c}; their
//            twiddles are W[1 .. R1), shared by every column -> staged in smem;
//   phase B: stages A..logN-1 act on the R1 contiguous blocks {b*R2 + c}.
// A CTA owns LN lines (16 columns or blocks; 8 when a launch is too small to
// fill the GPU): a small tile (8-32 KB), so several CTAs share an SM and one
// limb is spread over R/LN CTAs -- the machine stays busy even for a single
// ciphertext.  Inside a tile each thread runs radix-2^r butterfly groups in
// registers (radix-8 in the column phase, to stay at 80 registers and 3 CTAs
// per SM); lane % LN picks the line, which keeps the passes bank-conflict free
// (column tiles have stride 1 across lines, block tiles an odd stride R2+1).
// Lazy reduction: the forward transform needs no correction at all for
// q < 2^58 (values stay < 31q, reduced once at the end), the inverse keeps
// [0, 2q) with one conditional subtraction per butterfly.
#pragma once
#include "modarith.cuh"
#include "rns_params.hpp"

namespace cssc {

#ifndef CSSC_PTX_ADD
#define CSSC_PTX_ADD 1
#endif
#if CSSC_PTX_ADD
#define NTT_ADD(a, b) add64(a, b)
#define NTT_SUBADD(a, b, c) sub_add64(a, b, c)
#else
#define NTT_ADD(a, b) ((a) + (b))
#define NTT_SUBADD(a, b, c) ((a) - (b) + (c))
#endif

template <int LOGN>
struct Ntt2 {
    // block phase: 6 stages (7 at 2^15) so its twiddles fit next to the tile
    static constexpr int B = LOGN >= 15 ? 7 : (LOGN >= 12 ? 6 : LOGN / 2);
    static constexpr int A = LOGN - B;        // column-phase stages
    static constexpr int R1 = 1 << A;         // column length
    static constexpr int R2 = 1 << B;         // block length / number of columns
    static constexpr int N = 1 << LOGN;
    static constexpr int THREADS = 128;        // block-phase CTAs
    static constexpr int TC = R1 >= 256 ? 256 : 128;  // column-phase CTAs: one radix group per thread
    static constexpr int LINES = 16;
    static constexpr int CTAS_C = R2 / LINES;  // column-phase CTAs per limb
    static constexpr int CTAS_B = R1 / LINES;  // block-phase CTAs per limb
    static constexpr int PITCH = R2 + 1;       // odd block-tile pitch (conflict free)
    // block-phase twiddles of one tile: stage s holds 16 lines x 2^s entries
    // with an odd line stride (1 at s = 0, 2^s + 1 after) -> conflict-free LDS.128
    __host__ __device__ static constexpr int tw_stride(int s) { return s == 0 ? 1 : (1 << s) + 1; }
    __host__ __device__ static constexpr int tw_off(int s) { return s == 0 ? 0 : LINES * ((1 << s) + s - 2); }
    static constexpr int TWB = LINES * ((1 << B) + B - 2);  // = tw_off(B) entries
    static constexpr int SMEM_C = (LINES * R1 + 2 * R1) * 8;
    static constexpr int SMEM_B = (2 * LINES * PITCH + 2 * TWB) * 8;  // 2 tile buffers + twiddles
};

// Ampere-style async global->smem copies (LDGSTS): the tile and twiddle loads
// of a CTA are all in flight at once without register staging.
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }

// TMA 1D bulk copies (global -> shared) completing on an mbarrier
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
                 ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned phase) {
    asm volatile(
        "{\n .reg .pred p;\n"
        "WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}\n" ::"r"(
            smem_u32(bar)),
        "r"(phase)
        : "memory");
}

// Block-phase twiddle layout for tiles of LN blocks: stage s holds LN lines x
// 2^s entries with an odd line stride (conflict-free LDS.128).
template <int LN>
__host__ __device__ constexpr int btw_off(int s) { return s == 0 ? 0 : LN * ((1 << s) + s - 2); }
template <int LOGN, int LN>
constexpr int btw_entries() { return LN * ((1 << Ntt2<LOGN>::B) + Ntt2<LOGN>::B - 2); }

// Stage the block-phase twiddles of blocks [blk0, blk0 + LN) into smem:
// stage s needs W[2^(A+s) + (blk0 + l) * 2^s + blk], contiguous over (l, blk).
template <int LOGN, int LN = 16>
__device__ __forceinline__ void load_block_twiddles(u64* tws, const u64* table, int blk0) {
    using G = Ntt2<LOGN>;
    const ulonglong2* t2 = reinterpret_cast<const ulonglong2*>(table);
#pragma unroll
    for (int s = 0; s < G::B; ++s) {
        const int cnt = LN << s;
        const int gbase = (1 << (G::A + s)) + (blk0 << s);
        for (int i = threadIdx.x; i < cnt; i += blockDim.x) {
            const int l = i >> s, blk = i & ((1 << s) - 1);
            const int e = btw_off<LN>(s) + l * G::tw_stride(s) + blk;
            cp_async16(tws + 2 * e, t2 + gbase + i);
        }
    }
}

template <int LOGN, int LN = 16>
__device__ __forceinline__ ulonglong2 block_tw(const u64* tws, int s, int l, int blk) {
    using G = Ntt2<LOGN>;
    return *reinterpret_cast<const ulonglong2*>(tws + 2 * (btw_off<LN>(s) + l * G::tw_stride(s) + blk));
}

// A set of threads working on one tile: the whole CTA (__syncthreads) or a
// warp-aligned group of it with its own named barrier, so that several tiles
// of one CTA are transformed concurrently (fused kernels with many tiles per
// CTA would otherwise run them one after another).
struct ThreadGroup {
    int tid, nthreads, bar;  // bar < 0: the whole CTA
    __device__ __forceinline__ void sync() const {
        if (bar < 0)
            __syncthreads();
        else
            asm volatile("bar.sync %0, %1;\n" ::"r"(bar), "r"(nthreads) : "memory");
    }
};
__device__ __forceinline__ ThreadGroup whole_cta() { return ThreadGroup{(int)threadIdx.x, (int)blockDim.x, -1}; }
// group g of `groups` equal warp-aligned slices of the CTA (named barrier g + 1)
__device__ __forceinline__ ThreadGroup cta_slice(int g, int groups) {
    const int n = (int)blockDim.x / groups;
    return ThreadGroup{(int)threadIdx.x - g * n, n, g + 1};
}

// the modulus of every line of a tile (one prime per tile)
struct ConstQ {
    static constexpr bool kSpecial = false;
    u64 q;
    __device__ __forceinline__ u64 operator()(int) const { return q; }
};
// the same for a ciphertext prime (= 1 mod 2^32): butterflies use shoup_lazy_q
struct SpecQ {
    static constexpr bool kSpecial = true;
    u64 q;
    __device__ __forceinline__ u64 operator()(int) const { return q; }
};
template <class QF>
__device__ __forceinline__ u64 shoup_lazy_of(u64 a, u64 w, u64 wsh, u64 q) {
    if constexpr (QF::kSpecial)
        return shoup_lazy_q(a, w, wsh, q);
    else
        return shoup_lazy(a, w, wsh, q);
}

// One radix-2^R pass over local stages [S0L, S0L+R) of VL lines of length 2^RB.
// addr(l, pos): smem word of element pos of line l.  tw(sl, l, blk): twiddle
// (w, w_shoup) of local stage sl for line l and line-local butterfly block blk.
// qf(l): the modulus of line l (lines of several limbs in one tile).
template <int RB, int S0L, int R, bool INV, int VL, class QF, class Addr, class Tw>
__device__ __forceinline__ void line_pass(u64* s, QF qf, Addr addr, Tw tw, const ThreadGroup& tg) {
    constexpr int E = 1 << R;
    constexpr int TL = 1 << (RB - S0L - R);
    constexpr int LOG_TL = RB - S0L - R;
    constexpr int G = VL * (1 << (RB - R));
#pragma unroll 1
    for (int gi = tg.tid; gi < G; gi += tg.nthreads) {
        const int l = gi % VL;
        const int g = gi / VL;
        const u64 q = qf(l);
        const u64 two_q = 2 * q;
        const int blk = g >> LOG_TL;
        const int off = g & (TL - 1);
        const int base = (blk << (RB - S0L)) + off;
        u64 v[E];
#pragma unroll
        for (int k = 0; k < E; ++k) v[k] = s[addr(l, base + k * TL)];
        if (!INV) {
#pragma unroll
            for (int u = 0; u < R; ++u) {
                const int h = 1 << (R - 1 - u);
#pragma unroll
                for (int k = 0; k < E; ++k) {
                    if (k & h) continue;
                    // no correction: y < 2q, so each stage adds < 2q to the bound;
                    // a whole forward transform from < q stays < 31q < 2^64 for
                    // q < 2^58 (enforced by RnsParams) and is reduced once at the end
                    const ulonglong2 w = tw(S0L + u, l, (blk << u) + (k >> (R - u)));
                    const u64 x = v[k];
                    const u64 y = shoup_lazy_of<QF>(v[k + h], w.x, w.y, q);
                    v[k] = NTT_ADD(x, y);
                    v[k + h] = NTT_SUBADD(x, y, two_q);
                }
            }
        } else {
#pragma unroll
            for (int u = R - 1; u >= 0; --u) {
                const int h = 1 << (R - 1 - u);
#pragma unroll
                for (int k = 0; k < E; ++k) {
                    if (k & h) continue;
                    const ulonglong2 w = tw(S0L + u, l, (blk << u) + (k >> (R - u)));
                    const u64 x = v[k], y = v[k + h];
                    u64 sm = NTT_ADD(x, y);
                    sm = sm >= two_q ? sm - two_q : sm;
                    v[k] = sm;
                    v[k + h] = shoup_lazy_of<QF>(NTT_SUBADD(x, y, two_q), w.x, w.y, q);
                }
            }
        }
#pragma unroll
        for (int k = 0; k < E; ++k) s[addr(l, base + k * TL)] = v[k];
    }
}

// all passes of a line transform (radix-16 passes, remainder last); inverse
// runs the passes in reverse order.
// MAXR caps the pass radix (3: radix-8 passes, fewer live registers).
template <int RB, int S0L, bool INV, int MAXR, int VL, class QF, class Addr, class Tw>
__device__ __forceinline__ void line_ntt_v(u64* s, QF qf, Addr addr, Tw tw, const ThreadGroup& tg) {
    if constexpr (S0L < RB) {
        // pass radix: 6 -> 3+3, 9 -> 3+3+3, 5 -> 3+2, otherwise 4s then the rest
        constexpr int REM = RB - S0L;
        constexpr int R0 = (REM == 6 || REM == 9 || REM == 5) ? 3 : (REM >= 4 ? 4 : REM);
        constexpr int R = R0 < MAXR ? R0 : MAXR;
        if (!INV) {
            line_pass<RB, S0L, R, false, VL>(s, qf, addr, tw, tg);
            tg.sync();
            line_ntt_v<RB, S0L + R, false, MAXR, VL>(s, qf, addr, tw, tg);
        } else {
            line_ntt_v<RB, S0L + R, true, MAXR, VL>(s, qf, addr, tw, tg);
            line_pass<RB, S0L, R, true, VL>(s, qf, addr, tw, tg);
            tg.sync();
        }
    }
}
// 16 lines of one prime
template <int RB, int S0L, bool INV, int MAXR = 4, class Addr, class Tw>
__device__ __forceinline__ void line_ntt(u64* s, u64 q, Addr addr, Tw tw, const ThreadGroup& tg) {
    line_ntt_v<RB, S0L, INV, MAXR, 16>(s, ConstQ{q}, addr, tw, tg);
}
// the whole CTA on one tile
template <int RB, int S0L, bool INV, int MAXR = 4, class Addr, class Tw>
__device__ __forceinline__ void line_ntt(u64* s, u64 q, Addr addr, Tw tw) {
    line_ntt<RB, S0L, INV, MAXR>(s, q, addr, tw, whole_cta());
}
// the whole CTA on 16 lines of one ciphertext prime
template <int RB, int S0L, bool INV, int MAXR = 4, class Addr, class Tw>
__device__ __forceinline__ void line_ntt_q(u64* s, u64 q, Addr addr, Tw tw) {
    line_ntt_v<RB, S0L, INV, MAXR, 16>(s, SpecQ{q}, addr, tw, whole_cta());
}

}  // namespace cssc
