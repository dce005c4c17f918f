// Host check of the device modular arithmetic (csrc/modarith.cuh is
// host-compilable): barrett()/mul_mod() against __int128 arithmetic over
// random and boundary operands for moduli of every bit length the library
// admits (t = 65537 up to 62-bit), including the lazy a < 2^63 inputs.
#include <cstdio>
#include <random>

#include "modarith.cuh"

using namespace cssc;

static Modulus make(u64 q) {
    Modulus m{};
    m.q = q;
    const int k = 64 - __builtin_clzll(q);
    m.mub = (u64)(((unsigned __int128)1 << (k + 63)) / q);
    m.sh = (u32)(k - 1);
    m.mus = (u32)(((unsigned __int128)1 << (k + 20)) / q);
    return m;
}

int main() {
    std::mt19937_64 rng(12345);
    const u64 fixed[] = {65537ULL, (1ULL << 30) - 35, (1ULL << 54) - 33, (1ULL << 58) - 27,
                         (1ULL << 57) + 29, (1ULL << 60) - 93, (1ULL << 62) - 57, 67ULL};
    long bad = 0, n = 0;
    for (int trial = 0; trial < 64; ++trial) {
        u64 q;
        if (trial < 8) {
            q = fixed[trial];
        } else {
            const int k = 17 + (int)(rng() % 46);  // 17 .. 62 bits
            q = (rng() >> (64 - k)) | (1ULL << (k - 1)) | 1ULL;
            if ((q & (q - 1)) == 0) q += 2;
        }
        const Modulus m = make(q);
        auto check = [&](u64 a, u64 b) {
            const unsigned __int128 z = (unsigned __int128)a * b;
            const u64 want = (u64)(z % q);
            const u64 got = mul_mod(a, b, m);
            ++n;
            if (got != want) {
                if (bad < 10) std::printf("q=%llu a=%llu b=%llu got %llu want %llu\n", (unsigned long long)q,
                                          (unsigned long long)a, (unsigned long long)b, (unsigned long long)got,
                                          (unsigned long long)want);
                ++bad;
            }
        };
        // reduce_small_quot: every a < 2^(k+5)
        const int kq = 64 - __builtin_clzll(q);
        if (kq >= 7 && kq <= 58) {
            const u64 lim = 1ULL << (kq + 5);
            for (u64 a : {(u64)0, q - 1, q, 2 * q - 1, 31 * q - 1, lim - 1}) {
                if (a >= lim) continue;
                ++n;
                if (reduce_small_quot(a, m) != a % q) ++bad;
            }
            for (int i = 0; i < 100000; ++i) {
                const u64 a = rng() % lim;
                ++n;
                if (reduce_small_quot(a, m) != a % q) {
                    if (bad < 10) std::printf("small q=%llu a=%llu\n", (unsigned long long)q, (unsigned long long)a);
                    ++bad;
                }
            }
        }
        const u64 amax = (1ULL << 63) - 1;
        for (u64 a : {(u64)0, (u64)1, q - 1, q, 2 * q - 1, 4 * q - 1, amax, amax - q})
            for (u64 b : {(u64)0, (u64)1, q - 1, q / 2})
                if ((unsigned __int128)a * b < ((unsigned __int128)1 << (64 - __builtin_clzll(q) + 63))) check(a, b);
        for (int i = 0; i < 200000; ++i) {
            const u64 b = rng() % q;
            u64 a = rng();
            if (i & 1) a %= q;              // canonical
            else if ((i & 2) && q < (1ULL << 59)) a %= 31 * q;  // lazy NTT outputs
            else a >>= 1;                    // anything below 2^63
            if ((unsigned __int128)a * b < ((unsigned __int128)1 << (64 - __builtin_clzll(q) + 63))) check(a, b);
        }
    }
    // the key MAC's lazy sums (ks_fused.cu mac_term / mac_reduce): 15 lazy Shoup
    // products (< 2q each, any 64-bit first factor) summed without reduction,
    // then one reduce_small_quot_q, for ciphertext moduli q = 1 mod 2^32
    for (int k = 44; k <= 58; ++k) {
        for (int trial = 0; trial < 4; ++trial) {
            const u64 q = (((rng() >> (64 - (k - 32))) | (1ULL << (k - 33))) << 32) | 1ULL;
            const Modulus m = make(q);
            for (int rep = 0; rep < 2000; ++rep) {
                u64 acc = 0;
                unsigned __int128 want = 0;
                for (int t = 0; t < 15; ++t) {
                    const u64 key = rep == 0 ? q - 1 : rng() % q;
                    const u64 w = rep == 0 ? ~0ULL : ((t & 1) ? rng() % q : rng());
                    const u64 ksh = (u64)((((unsigned __int128)key) << 64) / q);
                    const u64 term = shoup_lazy_q(w, key, ksh, q);
                    if (term >= 2 * q) ++bad;
                    acc += term;
                    want += (unsigned __int128)w % q * key % q;
                }
                ++n;
                if (acc >= (1ULL << (k + 5)) || reduce_small_quot_q(acc, m) != (u64)(want % q)) {
                    if (bad < 10) std::printf("lazy mac q=%llu\n", (unsigned long long)q);
                    ++bad;
                }
            }
        }
    }
    std::printf("%ld / %ld mismatches\n", bad, n);
    return bad ? 1 : 0;
}
