/*
 * bfv_oracle.c -- CPU restatement of the RNS-BFV arithmetic (word-level
 * oracle "L2").  TEST INFRASTRUCTURE ONLY: see bfv_oracle.h.
 *
 * Deliberately plain: exact unsigned __int128 '%' for every modular product,
 * textbook loops, one coefficient at a time.  The only non-canonical integer
 * steps -- the fixed-point rounding terms of the exact basis extension (E1),
 * the t/Q scale-and-round (E2) and the decryption rounding (E5) -- follow the
 * formulas in DESIGN.md "Arithmetic spec" literally, because the CUDA path
 * must reproduce them bit for bit.
 *
 * Reference anchors (semantics being made real):
 *   encode/encrypt/decrypt        proj/src/he.cpp:64-91
 *   add / multiply / mult_plain   proj/src/he.cpp:93-136
 *   rotate (cyclic left by k)     proj/src/he.cpp:138-148, he.hpp:108-110
 *   slot_count = S = N/2          SURVEY.md section 0.4 (BFV row rotation)
 */
#include "bfv_oracle.h"

#include <pthread.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

typedef unsigned __int128 u128;
typedef uint64_t u64;

#define MAXP 40

/* ------------------------------------------------------------------ */
/* scalar modular arithmetic                                           */
/* ------------------------------------------------------------------ */
static inline u64 mulm(u64 a, u64 b, u64 q) { return (u64)(((u128)a * b) % q); }
static inline u64 addm(u64 a, u64 b, u64 q) { u64 s = a + b; return s >= q ? s - q : s; }
static inline u64 subm(u64 a, u64 b, u64 q) { return a >= b ? a - b : a + q - b; }
static u64 powm(u64 a, u64 e, u64 q) {
    u64 r = 1 % q;
    a %= q;
    while (e) {
        if (e & 1) r = mulm(r, a, q);
        a = mulm(a, a, q);
        e >>= 1;
    }
    return r;
}
static u64 invm(u64 a, u64 q) { return powm(a, q - 2, q); }
static inline u64 mulhi(u64 a, u64 b) { return (u64)(((u128)a * b) >> 64); }

static int is_prime(u64 n) {
    if (n < 2) return 0;
    static const u64 small[] = {2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37};
    for (int i = 0; i < 12; i++) {
        if (n % small[i] == 0) return n == small[i];
    }
    u64 d = n - 1;
    int r = 0;
    while ((d & 1) == 0) { d >>= 1; r++; }
    for (int i = 0; i < 12; i++) {
        u64 x = powm(small[i], d, n);
        if (x == 1 || x == n - 1) continue;
        int comp = 1;
        for (int j = 1; j < r; j++) {
            x = mulm(x, x, n);
            if (x == n - 1) { comp = 0; break; }
        }
        if (comp) return 0;
    }
    return 1;
}

static unsigned bitrev(unsigned x, int bits) {
    unsigned r = 0;
    for (int i = 0; i < bits; i++) { r = (r << 1) | (x & 1); x >>= 1; }
    return r;
}

/* ------------------------------------------------------------------ */
/* ChaCha20 block function (RFC 8439 section 2.3) as the counter-mode   */
/* sampler.  key = (seed_lo, seed_hi, 6 fixed words), nonce = stream.   */
/* ------------------------------------------------------------------ */
#define ROTL32(v, n) (((v) << (n)) | ((v) >> (32 - (n))))
#define QR(a, b, c, d)                 \
    a += b; d ^= a; d = ROTL32(d, 16); \
    c += d; b ^= c; b = ROTL32(b, 12); \
    a += b; d ^= a; d = ROTL32(d, 8);  \
    c += d; b ^= c; b = ROTL32(b, 7);

static void chacha_block(u64 seed, uint32_t ctr, uint32_t n0, uint32_t n1, uint32_t n2,
                         uint32_t out[16]) {
    uint32_t s[16] = {0x61707865u, 0x3320646eu, 0x79622d32u, 0x6b206574u,
                      (uint32_t)seed, (uint32_t)(seed >> 32), 0x63737363u, 0x2d68652du,
                      0x62323030u, 0x2d707267u, 0x6b657973u, 0x00000001u,
                      ctr, n0, n1, n2};
    uint32_t x[16];
    memcpy(x, s, sizeof x);
    for (int i = 0; i < 10; i++) {
        QR(x[0], x[4], x[8], x[12]);
        QR(x[1], x[5], x[9], x[13]);
        QR(x[2], x[6], x[10], x[14]);
        QR(x[3], x[7], x[11], x[15]);
        QR(x[0], x[5], x[10], x[15]);
        QR(x[1], x[6], x[11], x[12]);
        QR(x[2], x[7], x[8], x[13]);
        QR(x[3], x[4], x[9], x[14]);
    }
    for (int i = 0; i < 16; i++) out[i] = x[i] + s[i];
}

u64 bfvo_chacha_word(u64 seed, uint32_t n0, uint32_t n1, uint32_t n2, u64 index) {
    uint32_t blk[16];
    chacha_block(seed, (uint32_t)(index >> 3), n0, n1, n2, blk);
    unsigned w = (unsigned)(index & 7);
    return (u64)blk[2 * w] | ((u64)blk[2 * w + 1] << 32);
}

/* sampling domains (nonce word 0 = domain | limb << 8 | digit << 16) */
enum { DOM_SK = 1, DOM_PK_A = 2, DOM_PK_E = 3, DOM_KSK_A = 4, DOM_KSK_E = 5,
       DOM_ENC_U = 6, DOM_ENC_E0 = 7, DOM_ENC_E1 = 8 };

static inline uint32_t nonce0(int dom, int limb, int digit) {
    return (uint32_t)dom | ((uint32_t)limb << 8) | ((uint32_t)digit << 16);
}

/* uniform residue: (w[2k] * 2^64 + w[2k+1]) mod q */
static void sample_uniform(u64 seed, uint32_t n0, u64 id, int n, u64 q, u64* out) {
    for (int k = 0; k < n; k++) {
        u64 hi = bfvo_chacha_word(seed, n0, (uint32_t)id, (uint32_t)(id >> 32), 2 * (u64)k);
        u64 lo = bfvo_chacha_word(seed, n0, (uint32_t)id, (uint32_t)(id >> 32), 2 * (u64)k + 1);
        out[k] = (u64)((((u128)hi << 64) | lo) % q);
    }
}
/* ternary {-1,0,1}: (w[k] mod 3) - 1 */
static void sample_ternary(u64 seed, uint32_t n0, u64 id, int n, int64_t* out) {
    for (int k = 0; k < n; k++) {
        u64 w = bfvo_chacha_word(seed, n0, (uint32_t)id, (uint32_t)(id >> 32), (u64)k);
        out[k] = (int64_t)(w % 3) - 1;
    }
}
/* centered binomial eta=21: popc(w & (2^21-1)) - popc((w>>21) & (2^21-1)) */
static void sample_cbd(u64 seed, uint32_t n0, u64 id, int n, int64_t* out) {
    for (int k = 0; k < n; k++) {
        u64 w = bfvo_chacha_word(seed, n0, (uint32_t)id, (uint32_t)(id >> 32), (u64)k);
        out[k] = (int64_t)__builtin_popcountll(w & 0x1FFFFFull) -
                 (int64_t)__builtin_popcountll((w >> 21) & 0x1FFFFFull);
    }
}

/* ------------------------------------------------------------------ */
/* context                                                             */
/* ------------------------------------------------------------------ */
typedef struct {
    /* exact centred extension X -> Y (E1) */
    int nx, ny;
    const u64* xq;
    const u64* yq;
    u64 xhat_inv[MAXP];       /* [(X/x_i)^-1]_{x_i} */
    u64 R1[MAXP], R0[MAXP];   /* floor(2^128 / x_i) */
    u64 xhat_y[MAXP][MAXP];   /* [X/x_i]_{y_j} */
    u64 X_y[MAXP];            /* [X]_{y_j} */
} ext_t;

typedef struct {
    uint32_t g;
    u64* key; /* NTT form [dnum][2][L+K][N] */
} gkey_t;

struct bfvo_ctx {
    int logn, n, L, K, alpha, dnum, nB;
    u64 t, seed;
    int np;              /* L + K + nB + 1 (last = t) */
    u64 q[MAXP];
    u64 psi[MAXP];
    u64* W[MAXP];
    u64* Winv[MAXP];
    u64 ninv[MAXP];
    unsigned* pos0;      /* slot -> NTT position (row 0) */
    unsigned* pos1;      /* row 1 */
    /* keys */
    int64_t* s;          /* coef, N */
    u64* s_ntt;          /* [L+K][N] */
    u64* pk;             /* NTT [2][L][N] */
    u64* rlk;            /* NTT [dnum][2][L+K][N] */
    gkey_t* gk;
    int ngk, capgk;
    gkey_t* gk2;         /* keys for target phi_g(s)^2 (rotations of a 3-component product) */
    int ngk2, capgk2;
    /* constants */
    ext_t extQB, extBQ;
    u64 QhatInv[MAXP];          /* [(Q/q_i)^-1]_{q_i} */
    u64 T1[MAXP], T0[MAXP];     /* floor(t * 2^128 / q_i) */
    u64 QhatB[MAXP][MAXP];      /* [Q/q_i]_{b_j} */
    u64 QinvB[MAXP];            /* [Q^-1]_{b_j} */
    u64 delta[MAXP];            /* [floor(Q/t)]_{q_j} */
    /* hybrid key switching */
    u64 dig_hat_inv[MAXP];      /* per data prime i: [(Q_d/q_i)^-1]_{q_i}, d = digit of i */
    u64 dig_hat[MAXP][MAXP];    /* [Q_d/q_i]_{m_j}  (i data prime, j in Q u P) */
    u64 P_q[MAXP];              /* [P]_{q_j} */
    u64 Pinv_q[MAXP];           /* [P^-1]_{q_j} */
    u64 phat_inv[MAXP];         /* [(P/p_k)^-1]_{p_k} */
    u64 phat_q[MAXP][MAXP];     /* [P/p_k]_{q_j} */
    /* the over-Q multiply (fixed shapes, E6-E8): R = first L primes of B */
    int overq;
    ext_t extQR, extRQ;
    u64 QR_theta[MAXP];         /* floor(2^64 [R]_{q_i} / q_i) */
    u64 QR_omega[MAXP][MAXP];   /* [floor(R / q_i)]_{r_k} */
    u64 TR1[MAXP], TR0[MAXP];   /* floor(t 2^128 / r_k) */
    u64 tRinv_q[MAXP];          /* [t R^-1]_{q_j} */
    u64 tRinvRhat_q[MAXP][MAXP];/* [-t R^-1 (R / r_k)]_{q_j} */
};

static void floor_2_128_div(u64 q, u64* hi, u64* lo, u64* rem) {
    /* 2^128 = R*q + rem */
    u128 m = ~(u128)0; /* 2^128 - 1 */
    u128 R = m / q;
    u128 r = m % q;
    r += 1;
    if (r == q) { R += 1; r = 0; }
    *hi = (u64)(R >> 64);
    *lo = (u64)R;
    if (rem) *rem = (u64)r;
}

static void gen_primes(int bits, u64 twoN, int count, u64* out, const u64* used, int nused) {
    u64 top = (bits >= 64) ? ~0ull : ((1ull << bits) - 1);
    /* the product's rule: primes = 1 mod 2^32, largest first */
    if (twoN < (1ull << 32)) twoN = 1ull << 32;
    u64 cand = (top - 1) / twoN * twoN + 1;
    int got = 0;
    while (got < count) {
        int dup = 0;
        for (int i = 0; i < nused; i++) if (used[i] == cand) dup = 1;
        for (int i = 0; i < got; i++) if (out[i] == cand) dup = 1;
        if (!dup && is_prime(cand)) out[got++] = cand;
        cand -= twoN;
    }
}

/* first g = 2,3,... whose (q-1)/2N power has order exactly 2N */
static u64 find_psi(u64 q, u64 twoN) {
    for (u64 g = 2;; g++) {
        u64 x = powm(g, (q - 1) / twoN, q);
        if (powm(x, twoN / 2, q) == q - 1) return x;
    }
}

static void setup_ext(ext_t* e, const u64* xq, int nx, const u64* yq, int ny) {
    e->nx = nx; e->ny = ny; e->xq = xq; e->yq = yq;
    for (int i = 0; i < nx; i++) {
        u64 h = 1;
        for (int k = 0; k < nx; k++) if (k != i) h = mulm(h, xq[k] % xq[i], xq[i]);
        e->xhat_inv[i] = invm(h, xq[i]);
        floor_2_128_div(xq[i], &e->R1[i], &e->R0[i], NULL);
        for (int j = 0; j < ny; j++) {
            u64 hy = 1;
            for (int k = 0; k < nx; k++) if (k != i) hy = mulm(hy, xq[k] % yq[j], yq[j]);
            e->xhat_y[i][j] = hy;
        }
    }
    for (int j = 0; j < ny; j++) {
        u64 X = 1;
        for (int k = 0; k < nx; k++) X = mulm(X, xq[k] % yq[j], yq[j]);
        e->X_y[j] = X;
    }
}

/* E1: exact centred extension of one coefficient */
static void ext_coeff(const ext_t* e, const u64* x, u64* out) {
    u64 y[MAXP];
    u128 S = 0;
    for (int i = 0; i < e->nx; i++) {
        y[i] = mulm(x[i], e->xhat_inv[i], e->xq[i]);
        u64 F = y[i] * e->R1[i] + mulhi(y[i], e->R0[i]);
        S += F;
    }
    u64 v = (u64)((S + ((u128)1 << 63)) >> 64);
    for (int j = 0; j < e->ny; j++) {
        u64 p = e->yq[j];
        u64 acc = 0;
        for (int i = 0; i < e->nx; i++) acc = addm(acc, mulm(y[i] % p, e->xhat_y[i][j], p), p);
        out[j] = subm(acc, mulm(v % p, e->X_y[j], p), p);
    }
}

static void ntt_tables(bfvo_ctx* c, int i) {
    u64 q = c->q[i];
    int n = c->n;
    c->psi[i] = find_psi(q, 2 * (u64)n);
    c->W[i] = (u64*)malloc(sizeof(u64) * n);
    c->Winv[i] = (u64*)malloc(sizeof(u64) * n);
    u64 psiinv = invm(c->psi[i], q);
    for (int k = 0; k < n; k++) {
        unsigned e = bitrev((unsigned)k, c->logn);
        c->W[i][k] = powm(c->psi[i], e, q);
        c->Winv[i][k] = powm(psiinv, e, q);
    }
    c->ninv[i] = invm((u64)n % q, q);
}

void bfvo_ntt(const bfvo_ctx* c, int pi, u64* a) {
    u64 q = c->q[pi];
    int n = c->n;
    int t = n;
    for (int m = 1; m < n; m <<= 1) {
        t >>= 1;
        for (int i = 0; i < m; i++) {
            int j1 = 2 * i * t;
            u64 S = c->W[pi][m + i];
            for (int j = j1; j < j1 + t; j++) {
                u64 U = a[j], V = mulm(a[j + t], S, q);
                a[j] = addm(U, V, q);
                a[j + t] = subm(U, V, q);
            }
        }
    }
}

void bfvo_intt(const bfvo_ctx* c, int pi, u64* a) {
    u64 q = c->q[pi];
    int n = c->n;
    int t = 1;
    for (int m = n; m > 1; m >>= 1) {
        int h = m >> 1, j1 = 0;
        for (int i = 0; i < h; i++) {
            u64 S = c->Winv[pi][h + i];
            for (int j = j1; j < j1 + t; j++) {
                u64 U = a[j], V = a[j + t];
                a[j] = addm(U, V, q);
                a[j + t] = mulm(subm(U, V, q), S, q);
            }
            j1 += 2 * t;
        }
        t <<= 1;
    }
    for (int j = 0; j < n; j++) a[j] = mulm(a[j], c->ninv[pi], q);
}

/* signed small polynomial -> residues mod q */
static void lift_small(const int64_t* s, int n, u64 q, u64* out) {
    for (int k = 0; k < n; k++) out[k] = s[k] >= 0 ? (u64)s[k] % q : q - ((u64)(-s[k]) % q);
}

static void automorph_limb(int n, u64 q, uint32_t g, const u64* in, u64* out) {
    /* gather form: out[k] = +- in[i0] with i0 = g^-1 * k mod 2N */
    u64 twoN = 2 * (u64)n;
    /* g^-1 mod 2N: g odd; g^(N-1) is the inverse in (Z/2N)^* of order | N */
    u64 ginv = 1, base = g, e = (u64)n - 1;
    while (e) { if (e & 1) ginv = ginv * base % twoN; base = base * base % twoN; e >>= 1; }
    for (int k = 0; k < n; k++) {
        u64 i0 = ginv * (u64)k % twoN;
        if (i0 < (u64)n) out[k] = in[i0];
        else { u64 v = in[i0 - n]; out[k] = v ? q - v : 0; }
    }
}

void bfvo_automorph(const bfvo_ctx* c, uint32_t g, const u64* in, u64* out, int limbs) {
    for (int j = 0; j < limbs; j++)
        automorph_limb(c->n, c->q[j], g, in + (size_t)j * c->n, out + (size_t)j * c->n);
}

uint32_t bfvo_galois_elt(const bfvo_ctx* c, int64_t k) {
    int64_t S = c->n / 2;
    int64_t r = ((k % S) + S) % S;
    u64 twoN = 2 * (u64)c->n, g = 1;
    for (int64_t i = 0; i < r; i++) g = g * 3 % twoN;
    return (uint32_t)g;
}

/* ksk generation for target s' (NTT form over Q u P, [L+K][N]) */
static u64* gen_ksk(bfvo_ctx* c, u64 keyid, const u64* sp_ntt) {
    int n = c->n, LK = c->L + c->K;
    u64* key = (u64*)calloc((size_t)c->dnum * 2 * LK * n, sizeof(u64));
    int64_t* e = (int64_t*)malloc(sizeof(int64_t) * n);
    u64* tmp = (u64*)malloc(sizeof(u64) * n);
    for (int d = 0; d < c->dnum; d++) {
        sample_cbd(c->seed, nonce0(DOM_KSK_E, 0, d), keyid, n, e);
        for (int j = 0; j < LK; j++) {
            u64 q = c->q[j];
            u64* k0 = key + (((size_t)d * 2 + 0) * LK + j) * n;
            u64* k1 = key + (((size_t)d * 2 + 1) * LK + j) * n;
            sample_uniform(c->seed, nonce0(DOM_KSK_A, j, d), keyid, n, q, k1);
            bfvo_ntt(c, j, k1);
            lift_small(e, n, q, tmp);
            bfvo_ntt(c, j, tmp);
            int in_digit = (j < c->L) && (j / c->alpha == d);
            for (int k = 0; k < n; k++) {
                u64 v = addm(mulm(k1[k], c->s_ntt[(size_t)j * n + k], q), tmp[k], q);
                v = subm(0, v, q);
                if (in_digit) v = addm(v, mulm(c->P_q[j], sp_ntt[(size_t)j * n + k], q), q);
                k0[k] = v;
            }
        }
    }
    free(e);
    free(tmp);
    return key;
}

bfvo_ctx* bfvo_create(int logn, int L, int K, int alpha, int qbits, int pbits, u64 t, u64 seed) {
    bfvo_ctx* c = (bfvo_ctx*)calloc(1, sizeof(bfvo_ctx));
    c->logn = logn; c->n = 1 << logn; c->L = L; c->K = K; c->alpha = alpha;
    c->dnum = (L + alpha - 1) / alpha; c->nB = L + 1; c->t = t; c->seed = seed;
    int n = c->n;
    u64 twoN = 2 * (u64)n;
    gen_primes(qbits, twoN, L, c->q, NULL, 0);
    gen_primes(pbits, twoN, K, c->q + L, c->q, L);
    gen_primes(58, twoN, c->nB, c->q + L + K, c->q, L + K);
    c->np = L + K + c->nB + 1;
    c->q[c->np - 1] = t;
    for (int i = 0; i < c->np; i++) ntt_tables(c, i);

    /* slot maps: slot j <-> exponent 3^j (row 0), -3^j (row 1) */
    int S = n / 2;
    c->pos0 = (unsigned*)malloc(sizeof(unsigned) * S);
    c->pos1 = (unsigned*)malloc(sizeof(unsigned) * S);
    u64 e = 1;
    for (int j = 0; j < S; j++) {
        c->pos0[j] = bitrev((unsigned)((e - 1) / 2), logn);
        u64 e1 = twoN - e;
        c->pos1[j] = bitrev((unsigned)((e1 - 1) / 2), logn);
        e = e * 3 % twoN;
    }

    /* constants */
    const u64* Q = c->q;
    const u64* B = c->q + L + K;
    setup_ext(&c->extQB, Q, L, B, c->nB);
    setup_ext(&c->extBQ, B, c->nB, Q, L);
    for (int i = 0; i < L; i++) {
        c->QhatInv[i] = c->extQB.xhat_inv[i];
        u64 R1, R0, rem;
        floor_2_128_div(Q[i], &R1, &R0, &rem);
        u128 R = ((u128)R1 << 64) | R0;
        u128 T = R * t + ((u128)rem * t) / Q[i];
        c->T1[i] = (u64)(T >> 64);
        c->T0[i] = (u64)T;
        for (int j = 0; j < c->nB; j++) c->QhatB[i][j] = c->extQB.xhat_y[i][j];
    }
    for (int j = 0; j < c->nB; j++) c->QinvB[j] = invm(c->extQB.X_y[j], B[j]);
    {
        u64 Qt = 1;
        for (int i = 0; i < L; i++) Qt = mulm(Qt, Q[i] % t, t);
        for (int j = 0; j < L; j++) {
            /* floor(Q/t) = (Q - [Q]_t) / t ; [Q]_{q_j} = 0 */
            c->delta[j] = mulm(subm(0, Qt % Q[j], Q[j]), invm(t % Q[j], Q[j]), Q[j]);
        }
    }
    int LK = L + K;
    for (int i = 0; i < L; i++) {
        int d = i / alpha, lo = d * alpha, hi = lo + alpha < L ? lo + alpha : L;
        u64 h = 1;
        for (int k = lo; k < hi; k++) if (k != i) h = mulm(h, Q[k] % Q[i], Q[i]);
        c->dig_hat_inv[i] = invm(h, Q[i]);
        for (int j = 0; j < LK; j++) {
            u64 hm = 1;
            for (int k = lo; k < hi; k++) if (k != i) hm = mulm(hm, Q[k] % c->q[j], c->q[j]);
            c->dig_hat[i][j] = hm;
        }
    }
    for (int j = 0; j < L; j++) {
        u64 P = 1;
        for (int k = 0; k < K; k++) P = mulm(P, c->q[L + k] % Q[j], Q[j]);
        c->P_q[j] = P;
        c->Pinv_q[j] = invm(P, Q[j]);
    }
    for (int k = 0; k < K; k++) {
        u64 pk = c->q[L + k], h = 1;
        for (int m = 0; m < K; m++) if (m != k) h = mulm(h, c->q[L + m] % pk, pk);
        c->phat_inv[k] = invm(h, pk);
        for (int j = 0; j < L; j++) {
            u64 hq = 1;
            for (int m = 0; m < K; m++) if (m != k) hq = mulm(hq, c->q[L + m] % Q[j], Q[j]);
            c->phat_q[k][j] = hq;
        }
    }

    /* over-Q multiply: the shapes with specialised GPU kernels use it (E6-E8) */
    c->overq = (L == 2 && K == 2 && alpha == 2) || (L == 4 && K == 4 && alpha == 4);
    {
        const u64* R = B; /* r_k = b_k, k < L */
        setup_ext(&c->extQR, Q, L, R, L);
        setup_ext(&c->extRQ, R, L, Q, L);
        for (int i = 0; i < L; i++) {
            u64 Rq = 1;
            for (int k = 0; k < L; k++) Rq = mulm(Rq, R[k] % Q[i], Q[i]);
            c->QR_theta[i] = (u64)(((u128)Rq << 64) / Q[i]);
            for (int k = 0; k < L; k++) /* floor(R/q_i) = (R - [R]_{q_i}) / q_i, R = 0 mod r_k */
                c->QR_omega[i][k] = mulm(subm(0, Rq % R[k], R[k]), invm(Q[i] % R[k], R[k]), R[k]);
        }
        for (int k = 0; k < L; k++) {
            u64 R1, R0, rem;
            floor_2_128_div(R[k], &R1, &R0, &rem);
            u128 Rr = ((u128)R1 << 64) | R0;
            u128 T = Rr * t + ((u128)rem * t) / R[k];
            c->TR1[k] = (u64)(T >> 64);
            c->TR0[k] = (u64)T;
        }
        for (int j = 0; j < L; j++) {
            u64 Rq = 1;
            for (int k = 0; k < L; k++) Rq = mulm(Rq, R[k] % Q[j], Q[j]);
            u64 tRinv = mulm(t % Q[j], invm(Rq, Q[j]), Q[j]);
            c->tRinv_q[j] = tRinv;
            for (int k = 0; k < L; k++) {
                u64 hk = 1;
                for (int m = 0; m < L; m++) if (m != k) hk = mulm(hk, R[m] % Q[j], Q[j]);
                c->tRinvRhat_q[k][j] = subm(0, mulm(tRinv, hk, Q[j]), Q[j]);
            }
        }
    }

    /* secret key, public key, relinearisation key */
    c->s = (int64_t*)malloc(sizeof(int64_t) * n);
    sample_ternary(seed, nonce0(DOM_SK, 0, 0), 0, n, c->s);
    c->s_ntt = (u64*)malloc(sizeof(u64) * (size_t)LK * n);
    for (int j = 0; j < LK; j++) {
        lift_small(c->s, n, c->q[j], c->s_ntt + (size_t)j * n);
        bfvo_ntt(c, j, c->s_ntt + (size_t)j * n);
    }
    c->pk = (u64*)malloc(sizeof(u64) * 2 * (size_t)L * n);
    {
        int64_t* e0 = (int64_t*)malloc(sizeof(int64_t) * n);
        u64* tmp = (u64*)malloc(sizeof(u64) * n);
        sample_cbd(seed, nonce0(DOM_PK_E, 0, 0), 0, n, e0);
        for (int j = 0; j < L; j++) {
            u64 q = Q[j];
            u64* p0 = c->pk + (size_t)j * n;
            u64* p1 = c->pk + ((size_t)L + j) * n;
            sample_uniform(seed, nonce0(DOM_PK_A, j, 0), 0, n, q, p1);
            bfvo_ntt(c, j, p1);
            lift_small(e0, n, q, tmp);
            bfvo_ntt(c, j, tmp);
            for (int k = 0; k < n; k++)
                p0[k] = subm(0, addm(mulm(p1[k], c->s_ntt[(size_t)j * n + k], q), tmp[k], q), q);
        }
        free(e0);
        free(tmp);
    }
    {
        u64* s2 = (u64*)malloc(sizeof(u64) * (size_t)LK * n);
        for (int j = 0; j < LK; j++)
            for (int k = 0; k < n; k++) {
                u64 v = c->s_ntt[(size_t)j * n + k];
                s2[(size_t)j * n + k] = mulm(v, v, c->q[j]);
            }
        c->rlk = gen_ksk(c, 0, s2);
        free(s2);
    }
    return c;
}

void bfvo_destroy(bfvo_ctx* c) {
    if (!c) return;
    for (int i = 0; i < c->np; i++) { free(c->W[i]); free(c->Winv[i]); }
    free(c->pos0); free(c->pos1); free(c->s); free(c->s_ntt); free(c->pk); free(c->rlk);
    for (int i = 0; i < c->ngk; i++) free(c->gk[i].key);
    free(c->gk);
    for (int i = 0; i < c->ngk2; i++) free(c->gk2[i].key);
    free(c->gk2);
    free(c);
}

int bfvo_primes(const bfvo_ctx* c, u64* out) {
    for (int i = 0; i < c->np; i++) out[i] = c->q[i];
    return c->np;
}
u64 bfvo_psi(const bfvo_ctx* c, int i) { return c->psi[i]; }

void bfvo_add_galois_key(bfvo_ctx* c, uint32_t g) {
    for (int i = 0; i < c->ngk; i++) if (c->gk[i].g == g) return;
    int n = c->n, LK = c->L + c->K;
    u64* sp = (u64*)malloc(sizeof(u64) * (size_t)LK * n);
    u64* tmp = (u64*)malloc(sizeof(u64) * n);
    for (int j = 0; j < LK; j++) {
        lift_small(c->s, n, c->q[j], tmp);
        automorph_limb(n, c->q[j], g, tmp, sp + (size_t)j * n);
        bfvo_ntt(c, j, sp + (size_t)j * n);
    }
    if (c->ngk == c->capgk) {
        c->capgk = c->capgk ? 2 * c->capgk : 8;
        c->gk = (gkey_t*)realloc(c->gk, sizeof(gkey_t) * c->capgk);
    }
    c->gk[c->ngk].g = g;
    c->gk[c->ngk].key = gen_ksk(c, g, sp);
    c->ngk++;
    free(sp);
    free(tmp);
}

/* switching key for target phi_g(s)^2 = phi_g(s^2): rotates the s^2 component
 * of an unrelinearised product (key id 2^32 | g) */
/* the key caches are shared by the tests' parallel per-chunk evaluations */
static pthread_mutex_t key_mu = PTHREAD_MUTEX_INITIALIZER;

static const u64* find_key_sq_locked(bfvo_ctx* c, uint32_t g);
static const u64* find_key_sq(bfvo_ctx* c, uint32_t g) {
    pthread_mutex_lock(&key_mu);
    const u64* k = find_key_sq_locked(c, g);
    pthread_mutex_unlock(&key_mu);
    return k;
}

static const u64* find_key_sq_locked(bfvo_ctx* c, uint32_t g) {
    for (int i = 0; i < c->ngk2; i++) if (c->gk2[i].g == g) return c->gk2[i].key;
    int n = c->n, LK = c->L + c->K;
    u64* sp = (u64*)malloc(sizeof(u64) * (size_t)LK * n);
    u64* tmp = (u64*)malloc(sizeof(u64) * n);
    for (int j = 0; j < LK; j++) {
        u64* sj = sp + (size_t)j * n;
        lift_small(c->s, n, c->q[j], tmp);
        automorph_limb(n, c->q[j], g, tmp, sj);
        bfvo_ntt(c, j, sj);
        for (int k = 0; k < n; k++) sj[k] = mulm(sj[k], sj[k], c->q[j]);
    }
    if (c->ngk2 == c->capgk2) {
        c->capgk2 = c->capgk2 ? 2 * c->capgk2 : 8;
        c->gk2 = (gkey_t*)realloc(c->gk2, sizeof(gkey_t) * c->capgk2);
    }
    c->gk2[c->ngk2].g = g;
    c->gk2[c->ngk2].key = gen_ksk(c, ((u64)1 << 32) | g, sp);
    free(sp);
    free(tmp);
    return c->gk2[c->ngk2++].key;
}

void bfvo_add_galois_key_sq(bfvo_ctx* c, uint32_t g) { (void)find_key_sq(c, g); }

int bfvo_get_ksk_sq(bfvo_ctx* c, uint32_t g, u64* out) {
    const u64* key = find_key_sq(c, g);
    memcpy(out, key, sizeof(u64) * (size_t)c->dnum * 2 * (c->L + c->K) * c->n);
    return 0;
}

static const u64* find_key(bfvo_ctx* c, uint32_t which) {
    if (which == 0) return c->rlk;
    pthread_mutex_lock(&key_mu);
    bfvo_add_galois_key(c, which);
    const u64* k = NULL;
    for (int i = 0; i < c->ngk; i++) if (c->gk[i].g == which) k = c->gk[i].key;
    pthread_mutex_unlock(&key_mu);
    return k;
}

void bfvo_get_sk(const bfvo_ctx* c, int64_t* s) { memcpy(s, c->s, sizeof(int64_t) * c->n); }

void bfvo_get_pk(const bfvo_ctx* c, u64* out) {
    int n = c->n;
    memcpy(out, c->pk, sizeof(u64) * 2 * (size_t)c->L * n);
    for (int p = 0; p < 2; p++)
        for (int j = 0; j < c->L; j++) bfvo_intt(c, j, out + ((size_t)p * c->L + j) * n);
}

int bfvo_get_ksk(bfvo_ctx* c, uint32_t which, u64* out) {
    const u64* key = find_key(c, which);
    if (!key) return -1;
    int n = c->n, LK = c->L + c->K;
    size_t total = (size_t)c->dnum * 2 * LK * n;
    memcpy(out, key, sizeof(u64) * total);
    for (int d = 0; d < c->dnum; d++)
        for (int p = 0; p < 2; p++)
            for (int j = 0; j < LK; j++) bfvo_intt(c, j, out + (((size_t)d * 2 + p) * LK + j) * n);
    return 0;
}

/* ------------------------------------------------------------------ */
/* encoding                                                            */
/* ------------------------------------------------------------------ */
int bfvo_encode(const bfvo_ctx* c, const int64_t* vals, size_t nv, u64* m) {
    int n = c->n, S = n / 2, ti = c->np - 1;
    u64 t = c->t;
    if (nv > (size_t)S) return -1;
    memset(m, 0, sizeof(u64) * n);
    for (size_t j = 0; j < nv; j++) {
        int64_t v = vals[j] % (int64_t)t;
        if (v < 0) v += (int64_t)t;
        m[c->pos0[j]] = (u64)v;
    }
    bfvo_intt(c, ti, m);
    return 0;
}

void bfvo_decode(const bfvo_ctx* c, const u64* m, u64* slots) {
    int n = c->n, S = n / 2, ti = c->np - 1;
    u64* tmp = (u64*)malloc(sizeof(u64) * n);
    memcpy(tmp, m, sizeof(u64) * n);
    bfvo_ntt(c, ti, tmp);
    for (int j = 0; j < S; j++) slots[j] = tmp[c->pos0[j]];
    free(tmp);
}

/* ------------------------------------------------------------------ */
/* encrypt / decrypt                                                   */
/* ------------------------------------------------------------------ */
void bfvo_encrypt(const bfvo_ctx* c, const u64* m, u64 stream, u64* ct) {
    int n = c->n, L = c->L;
    int64_t* u = (int64_t*)malloc(sizeof(int64_t) * n);
    int64_t* e0 = (int64_t*)malloc(sizeof(int64_t) * n);
    int64_t* e1 = (int64_t*)malloc(sizeof(int64_t) * n);
    u64* un = (u64*)malloc(sizeof(u64) * n);
    sample_ternary(c->seed, nonce0(DOM_ENC_U, 0, 0), stream, n, u);
    sample_cbd(c->seed, nonce0(DOM_ENC_E0, 0, 0), stream, n, e0);
    sample_cbd(c->seed, nonce0(DOM_ENC_E1, 0, 0), stream, n, e1);
    for (int j = 0; j < L; j++) {
        u64 q = c->q[j];
        lift_small(u, n, q, un);
        bfvo_ntt(c, j, un);
        u64* c0 = ct + (size_t)j * n;
        u64* c1 = ct + ((size_t)L + j) * n;
        const u64* p0 = c->pk + (size_t)j * n;
        const u64* p1 = c->pk + ((size_t)L + j) * n;
        for (int k = 0; k < n; k++) {
            c0[k] = mulm(p0[k], un[k], q);
            c1[k] = mulm(p1[k], un[k], q);
        }
        bfvo_intt(c, j, c0);
        bfvo_intt(c, j, c1);
        for (int k = 0; k < n; k++) {
            u64 ee0 = e0[k] >= 0 ? (u64)e0[k] : q - (u64)(-e0[k]);
            u64 ee1 = e1[k] >= 0 ? (u64)e1[k] : q - (u64)(-e1[k]);
            c0[k] = addm(addm(c0[k], ee0, q), mulm(c->delta[j], m[k] % q, q), q);
            c1[k] = addm(c1[k], ee1, q);
        }
    }
    free(u); free(e0); free(e1); free(un);
}

/* E5: m = round(t/Q * x) mod t, x given by Q residues; returns dev (signed, 2^-64 units) */
static u64 scale_round_t(const bfvo_ctx* c, const u64* x, int64_t* dev) {
    u128 S = 0;
    for (int i = 0; i < c->L; i++) {
        u64 xi = mulm(x[i], c->QhatInv[i], c->q[i]);
        u128 G = (u128)xi * c->T1[i] + mulhi(xi, c->T0[i]);
        S += G;
    }
    u128 Sr = S + ((u128)1 << 63);
    u64 r = (u64)(Sr >> 64);
    u64 frac = (u64)S;
    if (dev) *dev = (int64_t)frac; /* two's complement: frac - 2^64 when >= 2^63 */
    return r % c->t;
}

int bfvo_decrypt(const bfvo_ctx* c, const u64* ct, u64* m) {
    int n = c->n, L = c->L;
    u64* x = (u64*)malloc(sizeof(u64) * (size_t)L * n);
    for (int j = 0; j < L; j++) {
        u64 q = c->q[j];
        u64* xj = x + (size_t)j * n;
        memcpy(xj, ct + ((size_t)L + j) * n, sizeof(u64) * n);
        bfvo_ntt(c, j, xj);
        for (int k = 0; k < n; k++) xj[k] = mulm(xj[k], c->s_ntt[(size_t)j * n + k], q);
        bfvo_intt(c, j, xj);
        for (int k = 0; k < n; k++) xj[k] = addm(xj[k], ct[(size_t)j * n + k], q);
    }
    u64 maxdev = 0;
    u64 col[MAXP];
    for (int k = 0; k < n; k++) {
        for (int j = 0; j < L; j++) col[j] = x[(size_t)j * n + k];
        int64_t d;
        m[k] = scale_round_t(c, col, &d);
        u64 ad = d < 0 ? (u64)0 - (u64)d : (u64)d;
        if (ad > maxdev) maxdev = ad;
    }
    free(x);
    int bl = maxdev ? 64 - __builtin_clzll(maxdev) : 0;
    int budget = 63 - bl;
    return budget < 0 ? 0 : budget;
}

/* ------------------------------------------------------------------ */
/* homomorphic operations                                              */
/* ------------------------------------------------------------------ */
void bfvo_add(const bfvo_ctx* c, const u64* a, const u64* b, u64* out) {
    int n = c->n;
    for (int p = 0; p < 2; p++)
        for (int j = 0; j < c->L; j++) {
            size_t o = ((size_t)p * c->L + j) * n;
            for (int k = 0; k < n; k++) out[o + k] = addm(a[o + k], b[o + k], c->q[j]);
        }
}

void bfvo_mul_plain(const bfvo_ctx* c, const u64* a, const u64* m, u64* out) {
    int n = c->n, L = c->L;
    u64* pm = (u64*)malloc(sizeof(u64) * n);
    u64 t = c->t;
    for (int j = 0; j < L; j++) {
        u64 q = c->q[j];
        for (int k = 0; k < n; k++) pm[k] = m[k] <= t / 2 ? m[k] % q : q - (t - m[k]);
        bfvo_ntt(c, j, pm);
        for (int p = 0; p < 2; p++) {
            size_t o = ((size_t)p * L + j) * n;
            memcpy(out + o, a + o, sizeof(u64) * n);
            bfvo_ntt(c, j, out + o);
            for (int k = 0; k < n; k++) out[o + k] = mulm(out[o + k], pm[k], q);
            bfvo_intt(c, j, out + o);
        }
    }
    free(pm);
}

/* hybrid key switch of d (coef form over Q) with key (NTT form) */
/* Hybrid key switch of d (E3/E4).  A rotation passes its Galois element g
 * and the UN-rotated c1: ModUp runs on d and the automorphism is applied to
 * every ModUp'd limb afterwards, phi_g(ModUp(d)), so rotations
 * of one source by several g share one ModUp (and its NTT) word for word. */
/* key-switch accumulation: acc0/acc1 (NTT domain over Q u P) += the inner
 * products of phi_g(ModUp(d)) with the key */
static void ks_accumulate(const bfvo_ctx* c, const u64* key, const u64* d, uint32_t g, u64* acc0, u64* acc1) {
    int n = c->n, L = c->L, K = c->K, LK = L + K;
    u64* D = (u64*)malloc(sizeof(u64) * n);
    u64* Dg = (u64*)malloc(sizeof(u64) * n);
    for (int dg = 0; dg < c->dnum; dg++) {
        int lo = dg * c->alpha, hi = lo + c->alpha < L ? lo + c->alpha : L;
        for (int j = 0; j < LK; j++) {
            u64 mj = c->q[j];
            if (j >= lo && j < hi) {
                memcpy(D, d + (size_t)j * n, sizeof(u64) * n);
            } else {
                for (int k = 0; k < n; k++) {
                    u64 acc = 0;
                    for (int i = lo; i < hi; i++) {
                        u64 y = mulm(d[(size_t)i * n + k], c->dig_hat_inv[i], c->q[i]);
                        acc = addm(acc, mulm(y % mj, c->dig_hat[i][j], mj), mj);
                    }
                    D[k] = acc;
                }
            }
            if (g != 1) {
                automorph_limb(n, mj, g, D, Dg);
                memcpy(D, Dg, sizeof(u64) * n);
            }
            bfvo_ntt(c, j, D);
            const u64* k0 = key + (((size_t)dg * 2 + 0) * LK + j) * n;
            const u64* k1 = key + (((size_t)dg * 2 + 1) * LK + j) * n;
            for (int k = 0; k < n; k++) {
                acc0[(size_t)j * n + k] = addm(acc0[(size_t)j * n + k], mulm(D[k], k0[k], mj), mj);
                acc1[(size_t)j * n + k] = addm(acc1[(size_t)j * n + k], mulm(D[k], k1[k], mj), mj);
            }
        }
    }
    free(D); free(Dg);
    (void)K;
}

/* INTT of the accumulators and ModDown (E4) into ks0/ks1 over Q */
static void ks_finish(const bfvo_ctx* c, u64* acc0, u64* acc1, u64* ks0, u64* ks1) {
    int n = c->n, L = c->L, K = c->K, LK = L + K;
    for (int j = 0; j < LK; j++) {
        bfvo_intt(c, j, acc0 + (size_t)j * n);
        bfvo_intt(c, j, acc1 + (size_t)j * n);
    }
    for (int p = 0; p < 2; p++) {
        u64* acc = p ? acc1 : acc0;
        u64* out = p ? ks1 : ks0;
        for (int k = 0; k < n; k++) {
            u64 y[MAXP];
            for (int kk = 0; kk < K; kk++)
                y[kk] = mulm(acc[(size_t)(L + kk) * n + k], c->phat_inv[kk], c->q[L + kk]);
            for (int j = 0; j < L; j++) {
                u64 q = c->q[j], cj = 0;
                for (int kk = 0; kk < K; kk++) cj = addm(cj, mulm(y[kk] % q, c->phat_q[kk][j], q), q);
                out[(size_t)j * n + k] = mulm(subm(acc[(size_t)j * n + k], cj, q), c->Pinv_q[j], q);
            }
        }
    }
}

static void key_switch_g(const bfvo_ctx* c, const u64* key, const u64* d, uint32_t g, u64* ks0, u64* ks1) {
    int n = c->n, LK = c->L + c->K;
    u64* acc0 = (u64*)calloc((size_t)LK * n, sizeof(u64));
    u64* acc1 = (u64*)calloc((size_t)LK * n, sizeof(u64));
    ks_accumulate(c, key, d, g, acc0, acc1);
    ks_finish(c, acc0, acc1, ks0, ks1);
    free(acc0); free(acc1);
}

static void key_switch(const bfvo_ctx* c, const u64* key, const u64* d, u64* ks0, u64* ks1) {
    key_switch_g(c, key, d, 1, ks0, ks1);
}

int bfvo_key_switch(bfvo_ctx* c, uint32_t which, const u64* d, u64* ks0, u64* ks1) {
    const u64* key = find_key(c, which);
    if (!key) return -1;
    key_switch(c, key, d, ks0, ks1);
    return 0;
}

/* E6: b'' = round(R b / Q) mod r_k for one coefficient (b by its Q residues):
 * R b / Q = sum_i y_i R / q_i - v R with y_i = [b_i (Q/q_i)^-1]_{q_i}; mod r_k the
 * v R term vanishes and R/q_i = floor(R/q_i) + [R]_{q_i}/q_i, so
 * b''_k = sum_i y_i [floor(R/q_i)]_{r_k} + round(sum_i y_i theta_i), the
 * rounding term in 64-bit fixed point (theta_i = floor(2^64 [R]_{q_i} / q_i)). */
static void scale_q_to_r(const bfvo_ctx* c, const u64* x, u64* out) {
    const u64* R = c->q + c->L + c->K;
    u64 y[MAXP];
    u128 S = 0;
    for (int i = 0; i < c->L; i++) {
        y[i] = mulm(x[i], c->extQR.xhat_inv[i], c->q[i]);
        S += (u128)y[i] * c->QR_theta[i];
    }
    u64 rnd = (u64)((S + ((u128)1 << 63)) >> 64);
    for (int k = 0; k < c->L; k++) {
        u64 acc = rnd % R[k];
        for (int i = 0; i < c->L; i++) acc = addm(acc, mulm(y[i] % R[k], c->QR_omega[i][k], R[k]), R[k]);
        out[k] = acc;
    }
}

/* E8: round(t z / R) mod q_j from the Q u R residues of z (any representative
 * mod QR: t z / R is then fixed mod tQ, so mod Q the wrap is harmless).  With
 * z_R = sum_k y_k R/r_k - v R (y_k = [z_k (R/r_k)^-1]_{r_k}) and z = z_R + R u,
 * round(t z / R) = t u + round(sum_k t y_k / r_k) - t v, and mod q_j the v terms
 * cancel: [t R^-1] z_j + sum_k y_k [-t R^-1 R/r_k] + round(sum_k t y_k / r_k),
 * the rounding term in the fixed point of E2 (floor(t 2^128 / r_k)). */
static void scale_r_to_q(const bfvo_ctx* c, const u64* zq, const u64* zr, u64* out) {
    const u64* R = c->q + c->L + c->K;
    u64 y[MAXP];
    u128 S = 0;
    for (int k = 0; k < c->L; k++) {
        y[k] = mulm(zr[k], c->extRQ.xhat_inv[k], R[k]);
        S += (u128)y[k] * c->TR1[k] + mulhi(y[k], c->TR0[k]);
    }
    u64 rnd = (u64)((S + ((u128)1 << 63)) >> 64);
    for (int j = 0; j < c->L; j++) {
        u64 q = c->q[j];
        u64 acc = addm(mulm(zq[j], c->tRinv_q[j], q), rnd % q, q);
        for (int k = 0; k < c->L; k++) acc = addm(acc, mulm(y[k] % q, c->tRinvRhat_q[k][j], q), q);
        out[j] = acc;
    }
}

/* the over-Q multiply (Kim-Polyakov-Zucca's HPS-over-Q): a extended Q -> R
 * (E1), b scaled to R (E6) and extended R -> Q (E1), tensor over Q u R
 * (2L limbs instead of 2L+1), round(t z / R) to Q (E8) */
static void mul_tensor_overq(const bfvo_ctx* c, const u64* a, const u64* b, u64* out3) {
    int n = c->n, L = c->L, M = 2 * L;
    int pidx[MAXP];
    for (int j = 0; j < L; j++) pidx[j] = j;
    for (int j = 0; j < L; j++) pidx[L + j] = L + c->K + j;
    u64* ext[4];
    const u64* src[4] = {a, a + (size_t)L * n, b, b + (size_t)L * n};
    u64 col[MAXP], o[MAXP], br[MAXP];
    for (int p = 0; p < 4; p++) {
        ext[p] = (u64*)malloc(sizeof(u64) * (size_t)M * n);
        for (int k = 0; k < n; k++) {
            for (int j = 0; j < L; j++) col[j] = src[p][(size_t)j * n + k];
            if (p < 2) {
                ext_coeff(&c->extQR, col, o);
                for (int j = 0; j < L; j++) {
                    ext[p][(size_t)j * n + k] = col[j];
                    ext[p][(size_t)(L + j) * n + k] = o[j];
                }
            } else {
                scale_q_to_r(c, col, br);
                ext_coeff(&c->extRQ, br, o);
                for (int j = 0; j < L; j++) {
                    ext[p][(size_t)j * n + k] = o[j];
                    ext[p][(size_t)(L + j) * n + k] = br[j];
                }
            }
        }
        for (int j = 0; j < M; j++) bfvo_ntt(c, pidx[j], ext[p] + (size_t)j * n);
    }
    u64* z[3];
    for (int r = 0; r < 3; r++) z[r] = (u64*)malloc(sizeof(u64) * (size_t)M * n);
    for (int j = 0; j < M; j++) {
        u64 q = c->q[pidx[j]];
        for (int k = 0; k < n; k++) {
            size_t x = (size_t)j * n + k;
            z[0][x] = mulm(ext[0][x], ext[2][x], q);
            z[1][x] = addm(mulm(ext[0][x], ext[3][x], q), mulm(ext[1][x], ext[2][x], q), q);
            z[2][x] = mulm(ext[1][x], ext[3][x], q);
        }
    }
    for (int r = 0; r < 3; r++)
        for (int j = 0; j < M; j++) bfvo_intt(c, pidx[j], z[r] + (size_t)j * n);
    u64 zq[MAXP], zr[MAXP];
    for (int r = 0; r < 3; r++)
        for (int k = 0; k < n; k++) {
            for (int j = 0; j < L; j++) {
                zq[j] = z[r][(size_t)j * n + k];
                zr[j] = z[r][(size_t)(L + j) * n + k];
            }
            scale_r_to_q(c, zq, zr, o);
            for (int j = 0; j < L; j++) out3[((size_t)r * L + j) * n + k] = o[j];
        }
    for (int p = 0; p < 4; p++) free(ext[p]);
    for (int r = 0; r < 3; r++) free(z[r]);
}

int bfvo_mul_overq(const bfvo_ctx* c) { return c->overq; }

void bfvo_mul_tensor(const bfvo_ctx* c, const u64* a, const u64* b, u64* out3) {
    if (c->overq) {
        mul_tensor_overq(c, a, b, out3);
        return;
    }
    int n = c->n, L = c->L, nB = c->nB, M = L + nB;
    /* basis Q u B: limb index 0..L-1 -> q[0..L-1]; L..L+nB-1 -> q[L+K ..] */
    int pidx[MAXP];
    for (int j = 0; j < L; j++) pidx[j] = j;
    for (int j = 0; j < nB; j++) pidx[L + j] = L + c->K + j;
    u64* ext[4];
    const u64* src[4] = {a, a + (size_t)L * n, b, b + (size_t)L * n};
    u64 col[MAXP], o[MAXP];
    for (int p = 0; p < 4; p++) {
        ext[p] = (u64*)malloc(sizeof(u64) * (size_t)M * n);
        memcpy(ext[p], src[p], sizeof(u64) * (size_t)L * n);
        for (int k = 0; k < n; k++) {
            for (int j = 0; j < L; j++) col[j] = src[p][(size_t)j * n + k];
            ext_coeff(&c->extQB, col, o);
            for (int j = 0; j < nB; j++) ext[p][(size_t)(L + j) * n + k] = o[j];
        }
        for (int j = 0; j < M; j++) bfvo_ntt(c, pidx[j], ext[p] + (size_t)j * n);
    }
    u64* z[3];
    for (int r = 0; r < 3; r++) z[r] = (u64*)malloc(sizeof(u64) * (size_t)M * n);
    for (int j = 0; j < M; j++) {
        u64 q = c->q[pidx[j]];
        for (int k = 0; k < n; k++) {
            size_t x = (size_t)j * n + k;
            z[0][x] = mulm(ext[0][x], ext[2][x], q);
            z[1][x] = addm(mulm(ext[0][x], ext[3][x], q), mulm(ext[1][x], ext[2][x], q), q);
            z[2][x] = mulm(ext[1][x], ext[3][x], q);
        }
    }
    for (int r = 0; r < 3; r++)
        for (int j = 0; j < M; j++) bfvo_intt(c, pidx[j], z[r] + (size_t)j * n);
    /* E2: w = round(t z / Q) in B, then exact extension B -> Q */
    const u64* B = c->q + L + c->K;
    u64 w[MAXP];
    for (int r = 0; r < 3; r++) {
        for (int k = 0; k < n; k++) {
            u64 xi[MAXP];
            u128 S = 0;
            for (int i = 0; i < L; i++) {
                xi[i] = mulm(z[r][(size_t)i * n + k], c->QhatInv[i], c->q[i]);
                S += (u128)xi[i] * c->T1[i] + mulhi(xi[i], c->T0[i]);
            }
            u64 rr = (u64)((S + ((u128)1 << 63)) >> 64);
            for (int j = 0; j < nB; j++) {
                u64 bj = B[j], acc = 0;
                for (int i = 0; i < L; i++) acc = addm(acc, mulm(xi[i] % bj, c->QhatB[i][j], bj), bj);
                u64 alpha = mulm(subm(acc, z[r][(size_t)(L + j) * n + k], bj), c->QinvB[j], bj);
                w[j] = subm(rr % bj, mulm(c->t % bj, alpha, bj), bj);
            }
            ext_coeff(&c->extBQ, w, o);
            for (int j = 0; j < L; j++) out3[((size_t)r * L + j) * n + k] = o[j];
        }
    }
    for (int p = 0; p < 4; p++) free(ext[p]);
    for (int r = 0; r < 3; r++) free(z[r]);
}

/* relinearisation of a tensor z ([3][L][N]) */
void bfvo_mul_relin_z(bfvo_ctx* c, const u64* z, u64* out) {
    int n = c->n, L = c->L;
    u64* ks0 = (u64*)malloc(sizeof(u64) * (size_t)L * n);
    u64* ks1 = (u64*)malloc(sizeof(u64) * (size_t)L * n);
    key_switch(c, c->rlk, z + 2 * (size_t)L * n, ks0, ks1);
    for (int j = 0; j < L; j++)
        for (int k = 0; k < n; k++) {
            size_t x = (size_t)j * n + k;
            out[x] = addm(z[x], ks0[x], c->q[j]);
            out[(size_t)L * n + x] = addm(z[(size_t)L * n + x], ks1[x], c->q[j]);
        }
    free(ks0); free(ks1);
}

void bfvo_mul_relin(bfvo_ctx* c, const u64* a, const u64* b, u64* out) {
    int n = c->n, L = c->L;
    u64* z = (u64*)malloc(sizeof(u64) * 3 * (size_t)L * n);
    bfvo_mul_tensor(c, a, b, z);
    u64* ks0 = (u64*)malloc(sizeof(u64) * (size_t)L * n);
    u64* ks1 = (u64*)malloc(sizeof(u64) * (size_t)L * n);
    key_switch(c, c->rlk, z + 2 * (size_t)L * n, ks0, ks1);
    for (int j = 0; j < L; j++)
        for (int k = 0; k < n; k++) {
            size_t x = (size_t)j * n + k;
            out[x] = addm(z[x], ks0[x], c->q[j]);
            out[(size_t)L * n + x] = addm(z[(size_t)L * n + x], ks1[x], c->q[j]);
        }
    free(z); free(ks0); free(ks1);
}

void bfvo_rotate(bfvo_ctx* c, const u64* a, int64_t k, u64* out) {
    int n = c->n, L = c->L;
    uint32_t g = bfvo_galois_elt(c, k);
    if (g == 1) { memcpy(out, a, sizeof(u64) * 2 * (size_t)L * n); return; }
    const u64* key = find_key(c, g);
    u64* c0 = (u64*)malloc(sizeof(u64) * (size_t)L * n);
    bfvo_automorph(c, g, a, c0, L);
    u64* ks0 = (u64*)malloc(sizeof(u64) * (size_t)L * n);
    key_switch_g(c, key, a + (size_t)L * n, g, ks0, out + (size_t)L * n);
    for (int j = 0; j < L; j++)
        for (int x = 0; x < n; x++) {
            size_t i = (size_t)j * n + x;
            out[i] = addm(c0[i], ks0[i], c->q[j]);
        }
    free(c0); free(ks0);
}

/* acc + rot(acc, k1) + rot(src, k2) with ONE ModDown: the two key switches'
 * accumulators are summed over Q u P before INTT + ModDown (a doubling step
 * and the odd step right after it in the batched plan) */
int bfvo_rotate2_add(bfvo_ctx* c, const u64* acc, const u64* src, int64_t k1, int64_t k2, u64* out) {
    int n = c->n, L = c->L, LK = L + c->K;
    uint32_t g1 = bfvo_galois_elt(c, k1), g2 = bfvo_galois_elt(c, k2);
    if (g1 == 1 || g2 == 1) return -2;
    const u64* key1 = find_key(c, g1);
    const u64* key2 = find_key(c, g2);
    if (!key1 || !key2) return -1;
    u64* a0 = (u64*)calloc((size_t)LK * n, sizeof(u64));
    u64* a1 = (u64*)calloc((size_t)LK * n, sizeof(u64));
    ks_accumulate(c, key1, acc + (size_t)L * n, g1, a0, a1);
    ks_accumulate(c, key2, src + (size_t)L * n, g2, a0, a1);
    u64* ks0 = (u64*)malloc(sizeof(u64) * (size_t)L * n);
    u64* ks1 = (u64*)malloc(sizeof(u64) * (size_t)L * n);
    ks_finish(c, a0, a1, ks0, ks1);
    u64* r1 = (u64*)malloc(sizeof(u64) * (size_t)L * n);
    u64* r2 = (u64*)malloc(sizeof(u64) * (size_t)L * n);
    bfvo_automorph(c, g1, acc, r1, L);
    bfvo_automorph(c, g2, src, r2, L);
    for (int j = 0; j < L; j++)
        for (int x = 0; x < n; x++) {
            size_t i = (size_t)j * n + x;
            u64 q = c->q[j];
            out[i] = addm(addm(addm(acc[i], r1[i], q), r2[i], q), ks0[i], q);
            out[(size_t)L * n + i] = addm(acc[(size_t)L * n + i], ks1[i], q);
        }
    free(a0); free(a1); free(ks0); free(ks1); free(r1); free(r2);
    return 0;
}

/* intra_chunk_sum of one chunk as the batched plan evaluates it (aggregate.cpp
 * semantics), from the product's tensor z = (z0, z1, z2)
 * ([3][L][N]) and the rotation schedule:
 *   fold_relin = 0: p = relin(z); then every doubling step D_a and the odd
 *     step O_a right after it share one ModDown (rotate2_add), a lone D_a is
 *     rotate + add;
 *   fold_relin = 1 (the plan with hoisted level 0): with a schedule, p is never
 *     relinearised on its own: level 0 sums the relinearisation of z2 and the
 *     key switches of phi_g(z1) (key for phi_g(s)) and phi_g(z2) (key for
 *     phi_g(s)^2) of D_1 (and O_1) into one ModDown; a later odd step O_a adds
 *     its two z key switches and phi_O(z0) into D_a's ModDown.
 * Without a schedule the result is relin(z). */
int bfvo_plan_fold(bfvo_ctx* c, const u64* z, int nsteps, const int64_t* offs, const int* from_acc, int fold_relin,
                   u64* out) {
    int n = c->n, L = c->L, LK = L + c->K;
    size_t cw = (size_t)L * n, aw = (size_t)LK * n;
    const u64 *z0 = z, *z1 = z + cw, *z2 = z + 2 * cw;
    u64* a0 = (u64*)calloc(aw, sizeof(u64));
    u64* a1 = (u64*)calloc(aw, sizeof(u64));
    u64* k0 = (u64*)malloc(sizeof(u64) * cw);
    u64* k1 = (u64*)malloc(sizeof(u64) * cw);
    u64* r = (u64*)malloc(sizeof(u64) * cw);
    u64* acc = (u64*)malloc(sizeof(u64) * 2 * cw);
    u64* nx = (u64*)malloc(sizeof(u64) * 2 * cw);
    int i = 0;
    if (!fold_relin || nsteps == 0) {
        bfvo_mul_relin_z(c, z, acc);
    } else {
        /* level 0: relin + D_1 (+ O_1) of the unrelinearised product */
        uint32_t gd = bfvo_galois_elt(c, offs[0]);
        ks_accumulate(c, c->rlk, z2, 1, a0, a1);
        ks_accumulate(c, find_key(c, gd), z1, gd, a0, a1);
        ks_accumulate(c, find_key_sq(c, gd), z2, gd, a0, a1);
        memcpy(acc, z, sizeof(u64) * 2 * cw);
        bfvo_automorph(c, gd, z0, r, L);
        for (size_t x = 0; x < cw; x++) acc[x] = addm(acc[x], r[x], c->q[x / n]);
        i = 1;
        if (nsteps > 1 && !from_acc[1]) {
            uint32_t go = bfvo_galois_elt(c, offs[1]);
            ks_accumulate(c, find_key(c, go), z1, go, a0, a1);
            ks_accumulate(c, find_key_sq(c, go), z2, go, a0, a1);
            bfvo_automorph(c, go, z0, r, L);
            for (size_t x = 0; x < cw; x++) acc[x] = addm(acc[x], r[x], c->q[x / n]);
            i = 2;
        }
        ks_finish(c, a0, a1, k0, k1);
        for (size_t x = 0; x < cw; x++) {
            acc[x] = addm(acc[x], k0[x], c->q[x / n]);
            acc[cw + x] = addm(acc[cw + x], k1[x], c->q[x / n]);
        }
    }
    /* p = relin(z) when the odd steps need it in the unfolded form */
    u64* p = NULL;
    if (!fold_relin) {
        p = (u64*)malloc(sizeof(u64) * 2 * cw);
        bfvo_mul_relin_z(c, z, p);
    }
    int64_t S = n / 2;
    while (i < nsteps) {
        if (!from_acc[i]) { free(a0); free(a1); free(k0); free(k1); free(r); free(acc); free(nx); free(p); return -3; }
        /* fold_relin = 2: two doubling steps D_{a+1}, D_{a+2} (with their odd
         * steps) in one key-switch stage: acc + R(acc, d1) + R(acc, d2) +
         * R(acc, d1 + d2) + R(p, o1) + R(p, o1 + d2) + R(p, o2), one ModDown;
         * merged only when no combined offset is 0 mod S (plan_stage_merge) */
        if (fold_relin == 2) {
            int i2 = i + 1 + (i + 1 < nsteps && !from_acc[i + 1]);  /* index of D_{a+2} */
            if (i2 < nsteps && from_acc[i2]) {
                int64_t d1 = offs[i], d2 = offs[i2];
                int has_o1 = i2 == i + 2, has_o2 = i2 + 1 < nsteps && !from_acc[i2 + 1];
                int64_t o1 = has_o1 ? offs[i + 1] : 0, o2 = has_o2 ? offs[i2 + 1] : 0;
                int ok = (d1 + d2) % S != 0 && (!has_o1 || (o1 + d2) % S != 0);
                if (ok) {
                    int64_t aoff[3] = {d1, d2, d1 + d2};
                    int64_t zoff[3];
                    int nz = 0;
                    if (has_o1) { zoff[nz++] = o1; zoff[nz++] = o1 + d2; }
                    if (has_o2) zoff[nz++] = o2;
                    memset(a0, 0, sizeof(u64) * aw);
                    memset(a1, 0, sizeof(u64) * aw);
                    memcpy(nx, acc, sizeof(u64) * 2 * cw);
                    for (int t = 0; t < 3; t++) {
                        uint32_t g = bfvo_galois_elt(c, aoff[t]);
                        ks_accumulate(c, find_key(c, g), acc + cw, g, a0, a1);
                        bfvo_automorph(c, g, acc, r, L);
                        for (size_t x = 0; x < cw; x++) nx[x] = addm(nx[x], r[x], c->q[x / n]);
                    }
                    for (int t = 0; t < nz; t++) {
                        uint32_t g = bfvo_galois_elt(c, zoff[t]);
                        ks_accumulate(c, find_key(c, g), z1, g, a0, a1);
                        ks_accumulate(c, find_key_sq(c, g), z2, g, a0, a1);
                        bfvo_automorph(c, g, z0, r, L);
                        for (size_t x = 0; x < cw; x++) nx[x] = addm(nx[x], r[x], c->q[x / n]);
                    }
                    ks_finish(c, a0, a1, k0, k1);
                    for (size_t x = 0; x < cw; x++) {
                        nx[x] = addm(nx[x], k0[x], c->q[x / n]);
                        nx[cw + x] = addm(nx[cw + x], k1[x], c->q[x / n]);
                    }
                    memcpy(acc, nx, sizeof(u64) * 2 * cw);
                    i = i2 + 1 + has_o2;
                    continue;
                }
            }
        }
        uint32_t gd = bfvo_galois_elt(c, offs[i]);
        memset(a0, 0, sizeof(u64) * aw);
        memset(a1, 0, sizeof(u64) * aw);
        ks_accumulate(c, find_key(c, gd), acc + cw, gd, a0, a1);
        memcpy(nx, acc, sizeof(u64) * 2 * cw);
        bfvo_automorph(c, gd, acc, r, L);
        for (size_t x = 0; x < cw; x++) nx[x] = addm(nx[x], r[x], c->q[x / n]);
        if (i + 1 < nsteps && !from_acc[i + 1]) {
            uint32_t go = bfvo_galois_elt(c, offs[i + 1]);
            if (fold_relin) {
                ks_accumulate(c, find_key(c, go), z1, go, a0, a1);
                ks_accumulate(c, find_key_sq(c, go), z2, go, a0, a1);
                bfvo_automorph(c, go, z0, r, L);
            } else {
                ks_accumulate(c, find_key(c, go), p + cw, go, a0, a1);
                bfvo_automorph(c, go, p, r, L);
            }
            for (size_t x = 0; x < cw; x++) nx[x] = addm(nx[x], r[x], c->q[x / n]);
            i += 2;
        } else {
            i += 1;
        }
        ks_finish(c, a0, a1, k0, k1);
        for (size_t x = 0; x < cw; x++) {
            nx[x] = addm(nx[x], k0[x], c->q[x / n]);
            nx[cw + x] = addm(nx[cw + x], k1[x], c->q[x / n]);
        }
        memcpy(acc, nx, sizeof(u64) * 2 * cw);
    }
    memcpy(out, acc, sizeof(u64) * 2 * cw);
    free(a0); free(a1); free(k0); free(k1); free(r); free(acc); free(nx); free(p);
    return 0;
}

/* RFC 8439 section 2.3 block function with an arbitrary key / nonce, for the
 * known-answer test of the sampler's core (tests/test_oracle_bfv.py). */
void bfvo_chacha_block_raw(const uint32_t key[8], uint32_t counter, const uint32_t nonce[3],
                           uint32_t out[16]) {
    uint32_t s[16] = {0x61707865u, 0x3320646eu, 0x79622d32u, 0x6b206574u,
                      key[0], key[1], key[2], key[3], key[4], key[5], key[6], key[7],
                      counter, nonce[0], nonce[1], nonce[2]};
    uint32_t x[16];
    memcpy(x, s, sizeof x);
    for (int i = 0; i < 10; i++) {
        QR(x[0], x[4], x[8], x[12]);
        QR(x[1], x[5], x[9], x[13]);
        QR(x[2], x[6], x[10], x[14]);
        QR(x[3], x[7], x[11], x[15]);
        QR(x[0], x[5], x[10], x[15]);
        QR(x[1], x[6], x[11], x[12]);
        QR(x[2], x[7], x[8], x[13]);
        QR(x[3], x[4], x[9], x[14]);
    }
    for (int i = 0; i < 16; i++) out[i] = x[i] + s[i];
}
