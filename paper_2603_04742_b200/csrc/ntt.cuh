// ntt.cuh -- CTA-level negacyclic NTT / INTT for one RNS limb held in shared
// memory (sm_100a).
//
// Convention (shared with DESIGN.md "Arithmetic spec"): forward Cooley-Tukey
// with the psi-power table W[k] = psi^bitrev(k); output position p holds
// a(psi^(2*bitrev(p)+1)).  Inverse Gentleman-Sande with psi^-bitrev(k), then
// a multiplication by N^-1.  Outputs are canonical, so any correct NTT agrees
// word for word with the CPU oracle.
//
// Structure: the log2(N) butterfly stages are grouped into passes of R <= 4
// stages.  In a pass every thread owns groups of 2^R elements spaced
// t_last = N >> (s0 + R) apart, which are closed under those R stages, so
// the butterflies of a pass run entirely in registers (radix-16).  Between
// passes the limb lives in shared memory with an XOR swizzle
// (x ^ ((x >> 4) & 15)) that keeps every pass's 8-byte accesses bank-conflict
// free.  Harvey lazy reduction keeps values in [0, 4q) (forward) and
// [0, 2q) (inverse) between stages; twiddles use Shoup multiplication.
#pragma once
#include "modarith.cuh"
#include "rns_params.hpp"

namespace cssc {

__device__ __forceinline__ int swz(int x) { return x ^ ((x >> 4) & 15); }

template <int LOGN>
struct NttGeom {
    static constexpr int N = 1 << LOGN;
    static constexpr int THREADS = (N / 16) >= 512 ? 512 : ((N / 16) < 32 ? 32 : N / 16);
    static constexpr int SMEM = N * 8;
};

__device__ __forceinline__ ulonglong2 ldg_tw(const u64* tw, int k) {
    return __ldg(reinterpret_cast<const ulonglong2*>(tw) + k);
}

template <int LOGN, int S0, int R>
__device__ __forceinline__ void fwd_pass(u64* s, const u64* tw, u64 q) {
    constexpr int N = 1 << LOGN;
    constexpr int G = N >> R;
    constexpr int TL = N >> (S0 + R);  // t_last
    constexpr int LOG_TL = LOGN - S0 - R;
    constexpr int E = 1 << R;
    const u64 two_q = 2 * q;
    for (int g = threadIdx.x; g < G; g += blockDim.x) {
        const int blk = g >> LOG_TL;
        const int off = g & (TL - 1);
        const int base = (blk << (LOGN - S0)) + off;
        u64 v[E];
#pragma unroll
        for (int c = 0; c < E; ++c) v[c] = s[swz(base + c * TL)];
#pragma unroll
        for (int u = 0; u < R; ++u) {
            const int h = 1 << (R - 1 - u);
#pragma unroll
            for (int c = 0; c < E; ++c) {
                if (c & h) continue;
                const ulonglong2 w = ldg_tw(tw, (1 << (S0 + u)) + (blk << u) + (c >> (R - u)));
                u64 x = v[c];
                x = x >= two_q ? x - two_q : x;
                const u64 y = shoup_lazy(v[c + h], w.x, w.y, q);
                v[c] = x + y;
                v[c + h] = x - y + two_q;
            }
        }
#pragma unroll
        for (int c = 0; c < E; ++c) s[swz(base + c * TL)] = v[c];
    }
}

template <int LOGN, int S0, int R>
__device__ __forceinline__ void inv_pass(u64* s, const u64* tw, u64 q) {
    constexpr int N = 1 << LOGN;
    constexpr int G = N >> R;
    constexpr int TL = N >> (S0 + R);
    constexpr int LOG_TL = LOGN - S0 - R;
    constexpr int E = 1 << R;
    const u64 two_q = 2 * q;
    for (int g = threadIdx.x; g < G; g += blockDim.x) {
        const int blk = g >> LOG_TL;
        const int off = g & (TL - 1);
        const int base = (blk << (LOGN - S0)) + off;
        u64 v[E];
#pragma unroll
        for (int c = 0; c < E; ++c) v[c] = s[swz(base + c * TL)];
#pragma unroll
        for (int u = R - 1; u >= 0; --u) {
            const int h = 1 << (R - 1 - u);
#pragma unroll
            for (int c = 0; c < E; ++c) {
                if (c & h) continue;
                const ulonglong2 w = ldg_tw(tw, (1 << (S0 + u)) + (blk << u) + (c >> (R - u)));
                const u64 x = v[c], y = v[c + h];
                u64 sm = x + y;
                sm = sm >= two_q ? sm - two_q : sm;
                v[c] = sm;
                v[c + h] = shoup_lazy(x - y + two_q, w.x, w.y, q);
            }
        }
#pragma unroll
        for (int c = 0; c < E; ++c) s[swz(base + c * TL)] = v[c];
    }
}

template <int LOGN, int S0>
__device__ __forceinline__ void fwd_passes(u64* s, const u64* tw, u64 q) {
    if constexpr (S0 < LOGN) {
        constexpr int R = (LOGN - S0) >= 4 ? 4 : (LOGN - S0);
        fwd_pass<LOGN, S0, R>(s, tw, q);
        __syncthreads();
        fwd_passes<LOGN, S0 + R>(s, tw, q);
    }
}

template <int LOGN, int S0>
__device__ __forceinline__ void inv_passes(u64* s, const u64* tw, u64 q) {
    if constexpr (S0 < LOGN) {
        constexpr int R = (LOGN - S0) >= 4 ? 4 : (LOGN - S0);
        inv_passes<LOGN, S0 + R>(s, tw, q);
        inv_pass<LOGN, S0, R>(s, tw, q);
        __syncthreads();
    }
}

// In-place forward NTT of the smem limb; output in [0, 4q) (lazy).
template <int LOGN>
__device__ __forceinline__ void ntt_fwd_smem(u64* s, const DevConsts* dc, int prime) {
    fwd_passes<LOGN, 0>(s, dc->tw[prime].fwd, dc->mod[prime].q);
}

// In-place inverse NTT WITHOUT the final N^-1 scaling; output in [0, 2q).
template <int LOGN>
__device__ __forceinline__ void ntt_inv_smem(u64* s, const DevConsts* dc, int prime) {
    inv_passes<LOGN, 0>(s, dc->tw[prime].inv, dc->mod[prime].q);
}

// ---- limb transfer helpers (global <-> swizzled smem, 16-byte vectors) ----

template <int LOGN>
__device__ __forceinline__ void load_limb(u64* s, const u64* __restrict__ g) {
    constexpr int N = 1 << LOGN;
    const ulonglong2* g2 = reinterpret_cast<const ulonglong2*>(g);
    for (int i = threadIdx.x; i < N / 2; i += blockDim.x) {
        const ulonglong2 v = g2[i];
        s[swz(2 * i)] = v.x;
        s[swz(2 * i + 1)] = v.y;
    }
}

// forward output: [0,4q) -> canonical
template <int LOGN>
__device__ __forceinline__ void store_limb_fwd(u64* __restrict__ g, const u64* s, u64 q) {
    constexpr int N = 1 << LOGN;
    ulonglong2* g2 = reinterpret_cast<ulonglong2*>(g);
    const u64 two_q = 2 * q;
    for (int i = threadIdx.x; i < N / 2; i += blockDim.x) {
        u64 a = s[swz(2 * i)], b = s[swz(2 * i + 1)];
        a = a >= two_q ? a - two_q : a;
        a = a >= q ? a - q : a;
        b = b >= two_q ? b - two_q : b;
        b = b >= q ? b - q : b;
        g2[i] = make_ulonglong2(a, b);
    }
}

// inverse output: [0,2q) times N^-1 -> canonical
template <int LOGN>
__device__ __forceinline__ void store_limb_inv(u64* __restrict__ g, const u64* s, u64 q, u64 ninv,
                                               u64 ninv_sh) {
    constexpr int N = 1 << LOGN;
    ulonglong2* g2 = reinterpret_cast<ulonglong2*>(g);
    for (int i = threadIdx.x; i < N / 2; i += blockDim.x) {
        const u64 a = shoup(s[swz(2 * i)], ninv, ninv_sh, q);
        const u64 b = shoup(s[swz(2 * i + 1)], ninv, ninv_sh, q);
        g2[i] = make_ulonglong2(a, b);
    }
}

}  // namespace cssc
