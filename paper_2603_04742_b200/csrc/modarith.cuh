// modarith.cuh -- 64-bit modular arithmetic for the RNS-BFV kernels (sm_100a).
//
// All primes are < 2^62 so lazy values in [0, 4q) fit a u64.  Constant
// multiplications (NTT twiddles, basis-conversion constants) use Shoup's
// precomputed quotient (3 u64 multiplies); variable x variable products use a
// Barrett reduction of the 128-bit product with mu = floor(2^128 / q).
// Results are always canonical in [0, q) unless the name says "lazy", so the
// outputs are independent of the reduction strategy.
#pragma once
#include <cstdint>

#ifdef __CUDACC__
#define CSSC_HD __host__ __device__ __forceinline__
#else
#define CSSC_HD inline
#endif

namespace cssc {

using u64 = std::uint64_t;
using u32 = std::uint32_t;

CSSC_HD u64 umulhi(u64 a, u64 b) {
#ifdef __CUDA_ARCH__
    return __umul64hi(a, b);
#else
    return (u64)(((unsigned __int128)a * b) >> 64);
#endif
}

// 64-bit add / a - b + c through explicit 32-bit carry chains (PTX add.cc /
// addc): keeps the high halves on the ALU pipe (IADD3.X) where ptxas would
// otherwise pick IMAD.X, which competes with the products for the FMA pipe
CSSC_HD u64 add64(u64 a, u64 b) {
#ifdef __CUDA_ARCH__
    unsigned lo, hi;
    asm("add.cc.u32 %0, %2, %3;\n\taddc.u32 %1, %4, %5;"
        : "=r"(lo), "=r"(hi)
        : "r"((unsigned)a), "r"((unsigned)b), "r"((unsigned)(a >> 32)), "r"((unsigned)(b >> 32)));
    return ((u64)hi << 32) | lo;
#else
    return a + b;
#endif
}
CSSC_HD u64 sub_add64(u64 a, u64 b, u64 c) {  // a - b + c
#ifdef __CUDA_ARCH__
    unsigned lo, hi;
    asm("sub.cc.u32 %0, %2, %3;\n\tsubc.u32 %1, %4, %5;"
        : "=r"(lo), "=r"(hi)
        : "r"((unsigned)a), "r"((unsigned)b), "r"((unsigned)(a >> 32)), "r"((unsigned)(b >> 32)));
    return add64(((u64)hi << 32) | lo, c);
#else
    return a - b + c;
#endif
}

CSSC_HD u64 add_mod(u64 a, u64 b, u64 q) {
    u64 s = a + b;
    return s >= q ? s - q : s;
}
CSSC_HD u64 sub_mod(u64 a, u64 b, u64 q) { return a >= b ? a - b : a + q - b; }
CSSC_HD u64 neg_mod(u64 a, u64 q) { return a ? q - a : 0; }

// a * w mod q in [0, 2q) for any a < 2^64, w < q, wsh = floor(w * 2^64 / q)
// -q mod 2^64, opaque to the optimiser: a*w + qh*(-q) then compiles to
// multiply-adds (IMAD.WIDE.U32 with a 64-bit addend) instead of a negated
// product and a separate 64-bit subtraction (two IMAD.X on the FMA pipe)
CSSC_HD u64 neg_opaque(u64 q) {
    u64 nq = 0 - q;
#ifdef __CUDA_ARCH__
    asm("" : "+l"(nq));
#endif
    return nq;
}
#ifndef CSSC_SHOUP_VARIANT
#define CSSC_SHOUP_VARIANT 2
#endif
CSSC_HD u64 shoup_lazy(u64 a, u64 w, u64 wsh, u64 q) {
    const u64 qh = umulhi(a, wsh);
#if CSSC_SHOUP_VARIANT == 0
    return a * w - qh * q;
#elif CSSC_SHOUP_VARIANT == 1
    return a * w + qh * neg_opaque(q);
#elif defined(__CUDA_ARCH__)
    // low 64 bits of a*w + qh*(-q) as explicit 32-bit multiply-add chains:
    // two IMAD.WIDE.U32 (the second taking the first as its 64-bit addend)
    // and four IMAD into the high word, no separate 64-bit adds
    const u64 nq = 0 - q;
    u64 r;
    asm("{\n\t.reg .u32 a0, a1, w0, w1, h0, h1, n0, n1, th;\n\t.reg .u64 t;\n\t"
        "mov.b64 {a0, a1}, %1;\n\tmov.b64 {w0, w1}, %2;\n\t"
        "mov.b64 {h0, h1}, %3;\n\tmov.b64 {n0, n1}, %4;\n\t"
        "mul.wide.u32 t, a0, w0;\n\t"
        "mov.b64 {w0, th}, t;\n\t"
        "mad.lo.u32 th, a0, w1, th;\n\t"
        "mad.lo.u32 th, a1, %5, th;\n\t"
        "mov.b64 t, {w0, th};\n\t"
        "mad.wide.u32 %0, h0, n0, t;\n\t"
        "mov.b64 {w0, th}, %0;\n\t"
        "mad.lo.u32 th, h0, n1, th;\n\t"
        "mad.lo.u32 th, h1, n0, th;\n\t"
        "mov.b64 %0, {w0, th};\n\t}"
        : "=l"(r)
        : "l"(a), "l"(w), "l"(qh), "l"(nq), "r"((unsigned)w));
    return r;
#else
    return a * w - qh * q;
#endif
}
CSSC_HD u64 shoup(u64 a, u64 w, u64 wsh, u64 q) {
    u64 r = shoup_lazy(a, w, wsh, q);
    return r >= q ? r - q : r;
}

// The same product for the ciphertext primes.  Every prime of Q, P and the
// multiply's extension base is chosen = 1 mod 2^32 (rns_params.cpp,
// pick_primes): q = h 2^32 + 1, so qh * q mod 2^64 = qh + ((lo32(qh) * h) << 32)
// and the low words of a*w - qh*q cost one IMAD.WIDE.U32 + three IMAD and a
// 64-bit subtraction on the ALU pipe (IADD3 / IADD3.X) instead of two
// IMAD.WIDE.U32 + four IMAD: 8 instead of 10 FMA-pipe operations per product.
// Same value as shoup_lazy for such q (both are a*w - qh*q mod 2^64); the
// plaintext modulus t is not of this form and keeps shoup_lazy.
#ifndef CSSC_Q32
#define CSSC_Q32 1
#endif
CSSC_HD u64 shoup_lazy_q(u64 a, u64 w, u64 wsh, u64 q) {
#if CSSC_Q32 && defined(__CUDA_ARCH__)
    const u64 qh = umulhi(a, wsh);
    const unsigned nh = 0u - (unsigned)(q >> 32);
    u64 r;
    asm("{\n\t.reg .u32 a0, a1, w0, w1, h0, h1, tl, th;\n\t.reg .u64 t;\n\t"
        "mov.b64 {a0, a1}, %1;\n\tmov.b64 {w0, w1}, %2;\n\t"
        "mov.b64 {h0, h1}, %3;\n\t"
        "mul.wide.u32 t, a0, w0;\n\t"
        "mov.b64 {tl, th}, t;\n\t"
        "mad.lo.u32 th, a0, w1, th;\n\t"
        "mad.lo.u32 th, a1, w0, th;\n\t"
        "mad.lo.u32 th, h0, %4, th;\n\t"
        "sub.cc.u32 tl, tl, h0;\n\t"
        "subc.u32 th, th, h1;\n\t"
        "mov.b64 %0, {tl, th};\n\t}"
        : "=l"(r)
        : "l"(a), "l"(w), "l"(qh), "r"(nh));
    return r;
#else
    return shoup_lazy(a, w, wsh, q);
#endif
}
CSSC_HD u64 shoup_q(u64 a, u64 w, u64 wsh, u64 q) {
    u64 r = shoup_lazy_q(a, w, wsh, q);
    return r >= q ? r - q : r;
}

// (z1 * 2^64 + z0) mod q for z1 < q; mu = floor(2^128 / q) = mu1 * 2^64 + mu0.
// The quotient estimate is at most 2 short, hence two conditional subtractions.
CSSC_HD u64 reduce128(u64 z1, u64 z0, u64 q, u64 mu1, u64 mu0) {
    u64 a_hi = umulhi(z0, mu0);
    u64 b_lo = z0 * mu1, b_hi = umulhi(z0, mu1);
    u64 c_lo = z1 * mu0, c_hi = umulhi(z1, mu0);
    u64 s = a_hi + b_lo;
    u64 carry = s < a_hi;
    u64 s2 = s + c_lo;
    carry += s2 < s;
    u64 qhat = z1 * mu1 + b_hi + c_hi + carry;
    u64 r = z0 - qhat * q;
    if (r >= q) r -= q;
    if (r >= q) r -= q;
    return r;
}

CSSC_HD u64 mul_mod(u64 a, u64 b, u64 q, u64 mu1, u64 mu0) {
    return reduce128(umulhi(a, b), a * b, q, mu1, mu0);
}

// Per-prime constants needed inside kernels.
struct Modulus {
    u64 q;
    u64 mu1, mu0;  // floor(2^128 / q)
    u64 mub;       // floor(2^(k+63) / q), k = bit length of q (< 2^64 as q is not a power of 2)
    u32 sh;        // k - 1
    u32 mus;       // floor(2^(k+20) / q) < 2^21
};

// Barrett reduction of z = z1 * 2^64 + z0 < 2^(k+63) (HAC 14.42 with the
// quotient scaled so one high product gives it): x = floor(z / 2^(k-1)) < 2^64,
// qhat = hi64(x * mub).  With z = x 2^(k-1) + zl and mub = 2^(k+63)/q - e,
// z/q - x mub/2^64 = zl/q + x e/2^64 < 2, so floor(z/q) - 2 <= qhat <= floor(z/q)
// and z - qhat q lies in [0, 3q): two conditional subtractions.  Needs k <= 63;
// covers a * b for any a < 2^63 and b < q (lazy NTT outputs < 31q included).
CSSC_HD u64 barrett(u64 z1, u64 z0, const Modulus& m) {
    const u64 x = (z0 >> m.sh) | (z1 << (64 - m.sh));
    const u64 qh = umulhi(x, m.mub);
    u64 r = z0 - qh * m.q;
    r = r >= m.q ? r - m.q : r;
    return r >= m.q ? r - m.q : r;
}

CSSC_HD u64 mul_mod(u64 a, u64 b, const Modulus& m) { return barrett(umulhi(a, b), a * b, m); }

// z - qh * q mod 2^64 for a ciphertext prime q = h 2^32 + 1 (see shoup_lazy_q):
// one IMAD into the high word and a 64-bit subtraction on the ALU pipe
CSSC_HD u64 sub_qh_q(u64 z, u64 qh, u64 q) {
#if CSSC_Q32 && defined(__CUDA_ARCH__)
    const unsigned nh = 0u - (unsigned)(q >> 32);
    u64 r;
    asm("{\n\t.reg .u32 zl, zh, h0, h1;\n\t"
        "mov.b64 {zl, zh}, %1;\n\tmov.b64 {h0, h1}, %2;\n\t"
        "mad.lo.u32 zh, h0, %3, zh;\n\t"
        "sub.cc.u32 zl, zl, h0;\n\t"
        "subc.u32 zh, zh, h1;\n\t"
        "mov.b64 %0, {zl, zh};\n\t}"
        : "=l"(r)
        : "l"(z), "l"(qh), "r"(nh));
    return r;
#else
    return z - qh * q;
#endif
}
// barrett / mul_mod for a ciphertext prime (same value)
CSSC_HD u64 barrett_q(u64 z1, u64 z0, const Modulus& m) {
    const u64 x = (z0 >> m.sh) | (z1 << (64 - m.sh));
    const u64 qh = umulhi(x, m.mub);
    u64 r = sub_qh_q(z0, qh, m.q);
    r = r >= m.q ? r - m.q : r;
    return r >= m.q ? r - m.q : r;
}
CSSC_HD u64 mul_mod_q(u64 a, u64 b, const Modulus& m) { return barrett_q(umulhi(a, b), a * b, m); }

// Exact dot products for the basis conversions: sum_i y_i * w_i mod p with
// every y_i < 2^58 (canonical residues) and constant w_i < p <= 2^58.  Both
// factors are split into 29-bit halves and each term is three 32x32->64
// multiply-adds (IMAD.WIDE.U32 with the 64-bit addend, Karatsuba middle term
// (y0 + y1)(w0 + w1)) into three u64 column sums, instead of a Shoup product
// (six IMAD.WIDE + four IMAD); the sum S = a0 + mid 2^29 + ah 2^58, mid =
// am - a0 - ah, is reduced once by the Barrett step above.  Bounds for up to
// 15 terms: a0, ah < 2^62, am < 15 * 2^60 < 2^64, S < 2^(k+62) < 2^(k+63),
// k = bit length of p >= 30.  The result is canonical, hence identical to any
// other exact reduction.
struct Dot29 {
    u64 a0 = 0, am = 0, ah = 0;
};
struct W29 {
    u32 lo, hi, sum;  // w = hi 2^29 + lo, sum = lo + hi
};
constexpr u32 kMask29 = (1u << 29) - 1;
CSSC_HD void dot29_mac(Dot29& d, u64 y, const W29& w) {
    const u32 y0 = (u32)y & kMask29, y1 = (u32)(y >> 29);
    d.a0 += (u64)y0 * w.lo;
    d.ah += (u64)y1 * w.hi;
    d.am += (u64)(y0 + y1) * w.sum;
}
// a small multiplier (y < 2^29) times w
CSSC_HD void dot29_mac_small(Dot29& d, u32 y, const W29& w) {
    d.a0 += (u64)y * w.lo;
    d.am += (u64)y * w.sum;
}
// a variable product a * b (both canonical, < 2^58) into the same column sums:
// three IMAD.WIDE.U32 instead of the 64 x 64 -> 128 product of mul_mod
CSSC_HD void dot29_mac_var(Dot29& d, u64 a, u64 b) {
    const u32 a0 = (u32)a & kMask29, a1 = (u32)(a >> 29);
    const u32 b0 = (u32)b & kMask29, b1 = (u32)(b >> 29);
    d.a0 += (u64)a0 * b0;
    d.ah += (u64)a1 * b1;
    d.am += (u64)(a0 + a1) * (b0 + b1);
}
CSSC_HD u64 dot29_reduce(const Dot29& d, const Modulus& m) {
    const u64 mid = d.am - d.a0 - d.ah;
    const u64 t = mid << 29, u = d.ah << 58;
    const u64 lo = d.a0 + t;
    u64 hi = (mid >> 35) + (d.ah >> 6) + (lo < t);
    const u64 lo2 = lo + u;
    hi += lo2 < u;
    return barrett(hi, lo2, m);
}
CSSC_HD u64 dot29_reduce_q(const Dot29& d, const Modulus& m) {  // m a ciphertext prime
    const u64 mid = d.am - d.a0 - d.ah;
    const u64 t = mid << 29, u = d.ah << 58;
    const u64 lo = d.a0 + t;
    u64 hi = (mid >> 35) + (d.ah >> 6) + (lo < t);
    const u64 lo2 = lo + u;
    hi += lo2 < u;
    return barrett_q(hi, lo2, m);
}
inline W29 split29(u64 w) {
    const u32 lo = (u32)(w & kMask29), hi = (u32)(w >> 29);
    return W29{lo, hi, lo + hi};
}

// a mod q for a < 2^(k+5) (a lazy forward-NTT output < 31q, say), k >= 7: the
// quotient is < 32, so 11 leading bits of a and a 21-bit scaled inverse give
// it in one 32-bit multiply.  a = x 2^(k-6) + al with al < 2^(k-6) < q/32 and
// mus = 2^(k+20)/q - e: a/q - x mus/2^26 = al/q + x e/2^26 < 1/32 + 2^-15, so
// the estimate is exact or one short -> one conditional subtraction.
CSSC_HD u64 reduce_small_quot(u64 a, const Modulus& m) {
    const u32 x = (u32)(a >> (m.sh - 5));
    const u32 qh = (x * m.mus) >> 26;
    const u64 r = a - (u64)qh * m.q;
    return r >= m.q ? r - m.q : r;
}
CSSC_HD u64 reduce_small_quot_q(u64 a, const Modulus& m) {  // m a ciphertext prime
    const u32 x = (u32)(a >> (m.sh - 5));
    const u32 qh = (x * m.mus) >> 26;
    const u64 r = sub_qh_q(a, (u64)qh, m.q);
    return r >= m.q ? r - m.q : r;
}
CSSC_HD u64 reduce64(u64 a, const Modulus& m) { return reduce128(0, a, m.q, m.mu1, m.mu0); }

// Fixed-point fraction floor(y * 2^64 / x) ~ y*R1 + hi(y*R0), R = floor(2^128/x):
// the integer formula shared with the oracle (E1).
CSSC_HD u64 frac64(u64 y, u64 R1, u64 R0) { return y * R1 + umulhi(y, R0); }

}  // namespace cssc
