// rns_params.cpp -- see rns_params.hpp.
#include "rns_params.hpp"

#include <algorithm>
#include <stdexcept>
#include <string>

namespace cssc {

using u128 = unsigned __int128;

static u64 mulm(u64 a, u64 b, u64 q) { return (u64)((u128)a * b % q); }

u64 pow_mod_host(u64 a, u64 e, u64 q) {
    u64 r = 1 % q;
    a %= q;
    for (; e; e >>= 1) {
        if (e & 1) r = mulm(r, a, q);
        a = mulm(a, a, q);
    }
    return r;
}

u64 inv_mod_host(u64 a, u64 q) { return pow_mod_host(a, q - 2, q); }

u64 shoup_factor(u64 w, u64 q) { return (u64)(((u128)w << 64) / q); }

bool is_prime_u64(u64 n) {
    if (n < 2) return false;
    const u64 bases[] = {2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37};
    for (u64 p : bases)
        if (n % p == 0) return n == p;
    u64 d = n - 1;
    int r = 0;
    while (!(d & 1)) {
        d >>= 1;
        ++r;
    }
    for (u64 a : bases) {
        u64 x = pow_mod_host(a, d, n);
        if (x == 1 || x == n - 1) continue;
        bool witness = true;
        for (int i = 1; i < r && witness; ++i) {
            x = mulm(x, x, n);
            if (x == n - 1) witness = false;
        }
        if (witness) return false;
    }
    return true;
}

// Galois element of a left row-rotation by k over S = N/2 slots: 3^(k mod S) mod 2N.
u32 galois_element(int64_t k, int n) {
    const int64_t S = n / 2;
    int64_t r = ((k % S) + S) % S;
    return (u32)pow_mod_host(3, (u64)r, 2 * (u64)n);
}

namespace {

unsigned reverse_bits(unsigned x, int bits) {
    unsigned r = 0;
    for (int i = 0; i < bits; ++i, x >>= 1) r = (r << 1) | (x & 1u);
    return r;
}

// Largest primes below 2^bits with p = 1 mod 2^32 (hence = 1 mod 2N for every
// ring here), skipping `taken`: q = h 2^32 + 1 makes the quotient correction
// qh * q of every Shoup product one 32-bit multiply (modarith.cuh, shoup_lazy_q).
void pick_primes(int bits, u64 two_n, int count, std::vector<u64>& out) {
    const u64 top = (1ull << bits) - 1;
    two_n = std::max<u64>(two_n, 1ull << 32);
    u64 cand = (top - 1) / two_n * two_n + 1;
    int got = 0;
    while (got < count) {
        if (std::find(out.begin(), out.end(), cand) == out.end() && is_prime_u64(cand)) {
            out.push_back(cand);
            ++got;
        }
        cand -= two_n;
    }
}

// psi: first generator candidate g = 2, 3, ... whose (q-1)/2N power has order 2N.
u64 root_of_unity(u64 q, u64 two_n) {
    for (u64 g = 2;; ++g) {
        u64 x = pow_mod_host(g, (q - 1) / two_n, q);
        if (pow_mod_host(x, two_n / 2, q) == q - 1) return x;
    }
}

void floor_pow128_div(u64 q, u64& hi, u64& lo, u64& rem) {
    u128 all = ~(u128)0;
    u128 quo = all / q;
    u128 r = all % q + 1;
    if (r == q) {
        quo += 1;
        r = 0;
    }
    hi = (u64)(quo >> 64);
    lo = (u64)quo;
    rem = (u64)r;
}

u64 prod_mod(const std::vector<u64>& ps, int skip, u64 m) {
    u64 acc = 1 % m;
    for (int i = 0; i < (int)ps.size(); ++i)
        if (i != skip) acc = mulm(acc, ps[i] % m, m);
    return acc;
}

void fill_ext(ExtConsts& e, const std::vector<u64>& X, const std::vector<int>& xi,
              const std::vector<u64>& Y, const std::vector<int>& yi) {
    e.nx = (int)X.size();
    e.ny = (int)Y.size();
    for (int i = 0; i < e.nx; ++i) {
        e.xi[i] = xi[i];
        e.xhat_inv[i] = inv_mod_host(prod_mod(X, i, X[i]), X[i]);
        e.xhat_inv_sh[i] = shoup_factor(e.xhat_inv[i], X[i]);
        u64 rem;
        floor_pow128_div(X[i], e.R1[i], e.R0[i], rem);
        for (int j = 0; j < e.ny; ++j) {
            e.xhat_y[i][j] = prod_mod(X, i, Y[j]);
            e.xhat_y_sh[i][j] = shoup_factor(e.xhat_y[i][j], Y[j]);
        }
    }
    for (int j = 0; j < e.ny; ++j) {
        e.yi[j] = yi[j];
        e.X_y[j] = prod_mod(X, -1, Y[j]);
        e.X_y_sh[j] = shoup_factor(e.X_y[j], Y[j]);
    }
}

}  // namespace

RnsParams::RnsParams(const RnsConfig& c) : cfg(c), host{} {
    if (c.logn < 4 || c.logn > 15) throw std::invalid_argument("logn must be in [4, 15]");
    // L + 1 <= 16 auxiliary terms keep the lazy basis-conversion sums below 32 q
    if (c.L < 1 || c.L > MAXL - 1 || c.K < 1 || c.K > MAXL || c.alpha < 1 || c.alpha > c.L)
        throw std::invalid_argument("prime counts out of range");
    if (c.qbits < 44 || c.qbits > 58 || c.pbits < 44 || c.pbits > 58)
        // <= 58 bits: 64q headroom lets the forward NTT skip per-butterfly corrections
        throw std::invalid_argument("prime bit sizes must be in [44, 58]");
    n = 1 << c.logn;
    S = n / 2;
    const u64 two_n = 2 * (u64)n;
    if (!is_prime_u64(c.t) || (c.t - 1) % two_n != 0)
        throw std::invalid_argument("plaintext modulus must be a prime = 1 mod 2N for batching");
    dnum = (c.L + c.alpha - 1) / c.alpha;
    nB = c.L + 1;
    if (c.K < c.alpha) {
        // P must dominate every digit for the key-switching noise to stay small
        throw std::invalid_argument("need K >= alpha special primes");
    }
    pick_primes(c.qbits, two_n, c.L, primes);
    pick_primes(c.pbits, two_n, c.K, primes);
    pick_primes(58, two_n, nB, primes);
    primes.push_back(c.t);
    np = (int)primes.size();
    if (np > MAXP) throw std::invalid_argument("too many primes");

    DevConsts& d = host;
    d.n = n;
    d.logn = c.logn;
    d.L = c.L;
    d.K = c.K;
    d.nB = nB;
    d.dnum = dnum;
    d.alpha = c.alpha;
    d.np = np;
    d.t = c.t;

    psi.resize(np);
    tw_fwd.resize(np);
    tw_inv.resize(np);
    for (int i = 0; i < np; ++i) {
        const u64 q = primes[i];
        u64 rem;
        d.mod[i].q = q;
        floor_pow128_div(q, d.mod[i].mu1, d.mod[i].mu0, rem);
        const int k = 64 - __builtin_clzll(q);
        if (k < 7 || k > 62) throw std::invalid_argument("modulus bit length out of range");
        d.mod[i].mub = (u64)(((unsigned __int128)1 << (k + 63)) / q);
        d.mod[i].sh = (u32)(k - 1);
        d.mod[i].mus = (u32)(((unsigned __int128)1 << (k + 20)) / q);
        psi[i] = root_of_unity(q, two_n);
        const u64 psi_inv = inv_mod_host(psi[i], q);
        tw_fwd[i].resize(2 * (size_t)n);
        tw_inv[i].resize(2 * (size_t)n);
        // W[k] = psi^bitrev(k), Winv[k] = psi^-bitrev(k)
        std::vector<u64> pw(n), pwi(n);
        pw[0] = pwi[0] = 1;
        for (int k = 1; k < n; ++k) {
            pw[k] = mulm(pw[k - 1], psi[i], q);
            pwi[k] = mulm(pwi[k - 1], psi_inv, q);
        }
        for (int k = 0; k < n; ++k) {
            unsigned e = reverse_bits((unsigned)k, c.logn);
            tw_fwd[i][2 * k] = pw[e];
            tw_fwd[i][2 * k + 1] = shoup_factor(pw[e], q);
            tw_inv[i][2 * k] = pwi[e];
            tw_inv[i][2 * k + 1] = shoup_factor(pwi[e], q);
        }
        d.ninv[i] = inv_mod_host((u64)n % q, q);
        d.ninv_sh[i] = shoup_factor(d.ninv[i], q);
    }

    // slot map: slot j <-> psi_t^(3^j)  at NTT position bitrev((3^j - 1) / 2)
    pos0.resize(S);
    u64 e = 1;
    for (int j = 0; j < S; ++j) {
        pos0[j] = reverse_bits((unsigned)((e - 1) / 2), c.logn);
        e = e * 3 % two_n;
    }

    const int L = c.L, K = c.K;
    std::vector<u64> Q(primes.begin(), primes.begin() + L);
    std::vector<u64> P(primes.begin() + L, primes.begin() + L + K);
    std::vector<u64> B(primes.begin() + L + K, primes.begin() + L + K + nB);
    std::vector<int> qi(L), bi(nB);
    for (int j = 0; j < L; ++j) qi[j] = j;
    for (int j = 0; j < nB; ++j) bi[j] = L + K + j;
    fill_ext(d.extQB, Q, qi, B, bi);
    fill_ext(d.extBQ, B, bi, Q, qi);
    overq = (L == 2 && K == 2 && c.alpha == 2) || (L == 4 && K == 4 && c.alpha == 4);
    {
        std::vector<u64> R(B.begin(), B.begin() + L);
        std::vector<int> ri(bi.begin(), bi.begin() + L);
        fill_ext(d.extQR, Q, qi, R, ri);
        fill_ext(d.extRQ, R, ri, Q, qi);
    }

    const u64 t = c.t;
    for (int i = 0; i < L; ++i) {
        d.QhatInv[i] = d.extQB.xhat_inv[i];
        d.QhatInv_sh[i] = d.extQB.xhat_inv_sh[i];
        u64 R1, R0, rem;
        floor_pow128_div(Q[i], R1, R0, rem);
        u128 R = ((u128)R1 << 64) | R0;
        u128 T = R * t + ((u128)rem * t) / Q[i];
        d.T1[i] = (u64)(T >> 64);
        d.T0[i] = (u64)T;
        for (int j = 0; j < nB; ++j) {
            d.QhatB[i][j] = d.extQB.xhat_y[i][j];
            d.QhatB_sh[i][j] = d.extQB.xhat_y_sh[i][j];
        }
    }
    for (int j = 0; j < nB; ++j) {
        d.QinvB[j] = inv_mod_host(d.extQB.X_y[j], B[j]);
        d.QinvB_sh[j] = shoup_factor(d.QinvB[j], B[j]);
        d.tB[j] = t % B[j];
        d.tB_sh[j] = shoup_factor(d.tB[j], B[j]);
    }
    const u64 Q_mod_t = prod_mod(Q, -1, t);
    for (int j = 0; j < L; ++j) {
        // floor(Q/t) mod q_j = (0 - [Q]_t) * t^-1  (Q = 0 mod q_j)
        u64 neg = (Q[j] - Q_mod_t % Q[j]) % Q[j];
        d.delta[j] = mulm(neg, inv_mod_host(t % Q[j], Q[j]), Q[j]);
        d.delta_sh[j] = shoup_factor(d.delta[j], Q[j]);
    }
    // key switching digits
    std::vector<u64> QP(primes.begin(), primes.begin() + L + K);
    for (int i = 0; i < L; ++i) {
        const int dg = i / c.alpha, lo = dg * c.alpha, hi = std::min(lo + c.alpha, L);
        std::vector<u64> digit(Q.begin() + lo, Q.begin() + hi);
        const int self = i - lo;
        d.dig_hat_inv[i] = inv_mod_host(prod_mod(digit, self, Q[i]), Q[i]);
        d.dig_hat_inv_sh[i] = shoup_factor(d.dig_hat_inv[i], Q[i]);
        for (int j = 0; j < L + K; ++j) {
            d.dig_hat[i][j] = prod_mod(digit, self, QP[j]);
            d.dig_hat_sh[i][j] = shoup_factor(d.dig_hat[i][j], QP[j]);
        }
    }
    for (int j = 0; j < L; ++j) {
        d.P_q[j] = prod_mod(P, -1, Q[j]);
        d.P_q_sh[j] = shoup_factor(d.P_q[j], Q[j]);
        d.Pinv_q[j] = inv_mod_host(d.P_q[j], Q[j]);
        d.Pinv_q_sh[j] = shoup_factor(d.Pinv_q[j], Q[j]);
    }
    for (int k = 0; k < K; ++k) {
        d.phat_inv[k] = inv_mod_host(prod_mod(P, k, P[k]), P[k]);
        d.phat_inv_sh[k] = shoup_factor(d.phat_inv[k], P[k]);
        for (int j = 0; j < L; ++j) {
            d.phat_q[k][j] = prod_mod(P, k, Q[j]);
            d.phat_q_sh[k][j] = shoup_factor(d.phat_q[k][j], Q[j]);
        }
    }
}

}  // namespace cssc
