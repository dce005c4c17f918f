// rns_params.hpp -- RNS-BFV parameter derivation (host side).
//
// Prime chains, NTT twiddle tables, slot maps and every basis-conversion
// constant, computed once per context and uploaded as a DevConsts block.
// The choices here (prime order, psi selection, slot <-> evaluation-point
// map) are the parameter spec of DESIGN.md "Arithmetic spec"; they decide the
// ciphertext words, so they are fixed, deterministic functions of
// (logn, L, K, alpha, qbits, pbits, t).
#pragma once
#include <cstdint>
#include <vector>

#include "modarith.cuh"

namespace cssc {

constexpr int MAXL = 16;  // max data / special primes
constexpr int MAXB = MAXL + 1;
constexpr int MAXP = 56;  // Q + P + B + t

// ChaCha20 key of every sampled polynomial (keys, encryptions).  A nonzero
// 64-bit seed gives the deterministic key (seed_lo, seed_hi, 6 fixed words)
// that oracle/bfv_oracle.c restates (tests, KATs); seed 0 asks the context for
// 256 bits of OS entropy (getrandom) instead.
struct SeedKey {
    uint32_t w[8];
};
inline SeedKey seed_key(u64 seed) {
    return SeedKey{{(uint32_t)seed, (uint32_t)(seed >> 32), 0x63737363u, 0x2d68652du, 0x62323030u, 0x2d707267u,
                    0x6b657973u, 0x00000001u}};
}

struct RnsConfig {
    int logn = 14;
    int L = 4;       // data primes (ciphertext modulus Q)
    int K = 2;       // special primes (key-switching modulus P)
    int alpha = 2;   // primes per key-switching digit; dnum = ceil(L / alpha)
    int qbits = 60;
    int pbits = 60;
    u64 t = 65537;
    u64 seed = 1;
    SeedKey key = seed_key(1);
};

// exact centred basis extension X -> Y (E1), all constants in Shoup form
struct ExtConsts {
    int nx = 0, ny = 0;
    int xi[MAXB];             // global prime index of x_i
    int yi[MAXB];             // global prime index of y_j
    u64 xhat_inv[MAXB], xhat_inv_sh[MAXB];
    u64 R1[MAXB], R0[MAXB];   // floor(2^128 / x_i)
    u64 xhat_y[MAXB][MAXB], xhat_y_sh[MAXB][MAXB];
    u64 X_y[MAXB], X_y_sh[MAXB];
};

struct TwiddlePtrs {
    const u64* fwd;  // [N] pairs (w, w_shoup) interleaved: 2N words
    const u64* inv;
};

// POD block uploaded to device memory; kernels take a const pointer to it.
struct DevConsts {
    int n, logn, L, K, nB, dnum, alpha, np;
    u64 t;
    Modulus mod[MAXP];
    TwiddlePtrs tw[MAXP];
    u64 ninv[MAXP], ninv_sh[MAXP];
    ExtConsts extQB, extBQ;
    ExtConsts extQR, extRQ;  // over-Q multiply: R = b_0 .. b_{L-1} (E1 both ways)
    // t/Q scale-and-round (E2 / E5)
    u64 QhatInv[MAXL], QhatInv_sh[MAXL];
    u64 T1[MAXL], T0[MAXL];
    u64 QhatB[MAXL][MAXB], QhatB_sh[MAXL][MAXB];
    u64 QinvB[MAXB], QinvB_sh[MAXB];
    u64 tB[MAXB], tB_sh[MAXB];
    u64 delta[MAXL], delta_sh[MAXL];
    // hybrid key switching (E3 / E4)
    u64 dig_hat_inv[MAXL], dig_hat_inv_sh[MAXL];
    u64 dig_hat[MAXL][2 * MAXL], dig_hat_sh[MAXL][2 * MAXL];
    u64 P_q[MAXL], P_q_sh[MAXL];
    u64 Pinv_q[MAXL], Pinv_q_sh[MAXL];
    u64 phat_inv[MAXL], phat_inv_sh[MAXL];
    u64 phat_q[MAXL][MAXL], phat_q_sh[MAXL][MAXL];
    const u32* pos0;  // slot j -> NTT position (row 0), S entries
};

struct RnsParams {
    RnsConfig cfg;
    int n = 0, S = 0, dnum = 0, nB = 0, np = 0;
    std::vector<u64> primes;  // Q | P | B | t
    std::vector<u64> psi;
    std::vector<std::vector<u64>> tw_fwd, tw_inv;  // interleaved (w, wsh)
    std::vector<u32> pos0;
    DevConsts host;  // filled except device pointers

    // The multiply runs over Q u R (R = the first L primes of B; E6-E8,
    // 2L limbs) for the shapes with specialised kernels, over Q u B (HPS,
    // 2L + 1 limbs) otherwise; oracle/bfv_oracle.c applies the same rule.
    bool overq = false;
    int mul_limbs() const { return overq ? 2 * cfg.L : cfg.L + nB; }

    explicit RnsParams(const RnsConfig& c);
    int q_index(int j) const { return j; }
    int p_index(int k) const { return cfg.L + k; }
    int b_index(int j) const { return cfg.L + cfg.K + j; }
    int t_index() const { return np - 1; }
};

// helpers shared by host code
u64 pow_mod_host(u64 a, u64 e, u64 q);
u64 inv_mod_host(u64 a, u64 q);
u64 shoup_factor(u64 w, u64 q);
bool is_prime_u64(u64 n);
u32 galois_element(int64_t k, int n);

}  // namespace cssc
