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
// A CTA owns 16 lines (16 columns or 16 blocks): a small tile (16-32 KB), so
// several CTAs share an SM and one limb is spread over R/16 CTAs -- this keeps
// the machine busy even for a single ciphertext.  Inside a tile each thread
// runs radix-16 (then radix-2^r) butterfly groups in registers; lane%16 picks
// the line, which makes every pass bank-conflict free (column tiles have
// stride 1 across lines, block tiles an odd stride R2+1).  Harvey lazy
// reduction: [0, 4q) forward, [0, 2q) inverse, canonical at the end.
#pragma once
#include "modarith.cuh"
#include "rns_params.hpp"

namespace cssc {

template <int LOGN>
struct Ntt2 {
    static constexpr int A = (LOGN + 1) / 2;  // column-phase stages
    static constexpr int B = LOGN - A;        // block-phase stages
    static constexpr int R1 = 1 << A;         // column length
    static constexpr int R2 = 1 << B;         // block length / number of columns
    static constexpr int N = 1 << LOGN;
    static constexpr int THREADS = 128;
    static constexpr int LINES = 16;
    static constexpr int CTAS_C = R2 / LINES;  // column-phase CTAs per limb
    static constexpr int CTAS_B = R1 / LINES;  // block-phase CTAs per limb
    static constexpr int SMEM_C = (LINES * R1 + 2 * R1) * 8;
    static constexpr int SMEM_B = (LINES * (R2 + 1)) * 8;
};

// One radix-2^R pass over local stages [S0L, S0L+R) of 16 lines of length 2^RB.
// addr(l, pos): smem word of element pos of line l.  tw(sl, l, blk): twiddle
// (w, w_shoup) of local stage sl for line l and line-local butterfly block blk.
template <int RB, int S0L, int R, bool INV, class Addr, class Tw>
__device__ __forceinline__ void line_pass(u64* s, u64 q, Addr addr, Tw tw) {
    constexpr int E = 1 << R;
    constexpr int TL = 1 << (RB - S0L - R);
    constexpr int LOG_TL = RB - S0L - R;
    constexpr int G = 16 * (1 << (RB - R));
    const u64 two_q = 2 * q;
    for (int gi = threadIdx.x; gi < G; gi += 128) {
        const int l = gi & 15;
        const int g = gi >> 4;
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
                    const ulonglong2 w = tw(S0L + u, l, (blk << u) + (k >> (R - u)));
                    u64 x = v[k];
                    x = x >= two_q ? x - two_q : x;
                    const u64 y = shoup_lazy(v[k + h], w.x, w.y, q);
                    v[k] = x + y;
                    v[k + h] = x - y + two_q;
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
                    u64 sm = x + y;
                    sm = sm >= two_q ? sm - two_q : sm;
                    v[k] = sm;
                    v[k + h] = shoup_lazy(x - y + two_q, w.x, w.y, q);
                }
            }
        }
#pragma unroll
        for (int k = 0; k < E; ++k) s[addr(l, base + k * TL)] = v[k];
    }
}

// all passes of a line transform (radix-16 passes, remainder last); inverse
// runs the passes in reverse order.
template <int RB, int S0L, bool INV, class Addr, class Tw>
__device__ __forceinline__ void line_ntt(u64* s, u64 q, Addr addr, Tw tw) {
    if constexpr (S0L < RB) {
        constexpr int R = (RB - S0L) >= 4 ? 4 : (RB - S0L);
        if (!INV) {
            line_pass<RB, S0L, R, false>(s, q, addr, tw);
            __syncthreads();
            line_ntt<RB, S0L + R, false>(s, q, addr, tw);
        } else {
            line_ntt<RB, S0L + R, true>(s, q, addr, tw);
            line_pass<RB, S0L, R, true>(s, q, addr, tw);
            __syncthreads();
        }
    }
}

}  // namespace cssc
