/*
 * bfv_oracle.h -- CPU word-level oracle ("L2") for the RNS-BFV arithmetic
 * behind the encrypted CSSC SpMV cloud phase.
 *
 * TEST INFRASTRUCTURE ONLY. Nothing in the product (paper_2603_04742_b200/)
 * links, loads or calls this code; only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline leg may use it, and only as the checker.
 *
 * The reference (/root/reference/proj) ships a slot-vector simulator
 * (proj/src/he.cpp:64-153) and no lattice arithmetic at all (he.hpp:82-85,
 * SPEC.md:9), so the ciphertext-word semantics below are restated from the
 * public RNS-BFV literature (Fan-Vercauteren BFV; Halevi-Polyakov-Shoup RNS
 * scale-and-round; hybrid key switching with digit decomposition) and pinned
 * by the known-answer tests in tests/test_oracle_bfv.py.  Decryptions are
 * pinned to the reference simulator (oracle/_ref) slot for slot.
 * At the ciphertext-word level parity is therefore UNPINNED by the reference
 * (SURVEY 8(c)): the words are self-consistent with these KATs, not with a
 * reference output.
 *
 * Every integer formula that is not a canonical modular identity (the
 * fixed-point rounding terms of the exact basis extension and of the t/Q
 * scaling) is spelled out in DESIGN.md section "Arithmetic spec"; the CUDA
 * path implements the identical integer formulas, so ciphertext words match
 * bit for bit.
 */
#ifndef CSSC_BFV_ORACLE_H
#define CSSC_BFV_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct bfvo_ctx bfvo_ctx;

/* logn: ring degree N = 2^logn.  L data primes (qbits), K special primes
 * (pbits), digit size alpha (dnum = ceil(L/alpha)), plaintext modulus t
 * (prime, t = 1 mod 2N), seed for every sampled polynomial. */
bfvo_ctx* bfvo_create(int logn, int L, int K, int alpha, int qbits, int pbits,
                      uint64_t t, uint64_t seed);
void bfvo_destroy(bfvo_ctx* c);

/* primes in order Q (L) | P (K) | B (L+1 aux primes of the multiplication);
 * returns the count. */
int bfvo_primes(const bfvo_ctx* c, uint64_t* out);
uint64_t bfvo_psi(const bfvo_ctx* c, int prime_index); /* index L+K+L+1 = t */

/* Low-level KATs: negacyclic NTT of one limb in the repo's convention
 * (output position p holds a(psi^(2*bitrev(p)+1))). */
void bfvo_ntt(const bfvo_ctx* c, int prime_index, uint64_t* a);
void bfvo_intt(const bfvo_ctx* c, int prime_index, uint64_t* a);
void bfvo_chacha_block_raw(const uint32_t key[8], uint32_t counter, const uint32_t nonce[3],
                           uint32_t out[16]);
uint64_t bfvo_chacha_word(uint64_t seed, uint32_t n0, uint32_t n1, uint32_t n2,
                          uint64_t index);

/* Keys (deterministic from seed).  Galois keys are generated on demand. */
void bfvo_add_galois_key(bfvo_ctx* c, uint32_t galois_elt);
uint32_t bfvo_galois_elt(const bfvo_ctx* c, int64_t k);
/* canonical (coefficient-form, fully reduced) key material for comparisons */
void bfvo_get_sk(const bfvo_ctx* c, int64_t* s);                 /* N */
void bfvo_get_pk(const bfvo_ctx* c, uint64_t* out);              /* 2*L*N */
/* which = 0: relinearisation key, else the Galois key for element `which` */
int bfvo_get_ksk(bfvo_ctx* c, uint32_t which, uint64_t* out);    /* dnum*2*(L+K)*N */

/* Batch encoding mod t (S = N/2 slots, BFV row 0; row 1 zero). */
int bfvo_encode(const bfvo_ctx* c, const int64_t* vals, size_t n, uint64_t* m);
void bfvo_decode(const bfvo_ctx* c, const uint64_t* m, uint64_t* slots /* S */);

/* Ciphertexts are uint64 [2][L][N], coefficient form, residues in [0,q). */
void bfvo_encrypt(const bfvo_ctx* c, const uint64_t* m, uint64_t stream, uint64_t* ct);
/* returns the measured invariant-noise budget in bits (fixed-point estimate) */
int bfvo_decrypt(const bfvo_ctx* c, const uint64_t* ct, uint64_t* m);
void bfvo_add(const bfvo_ctx* c, const uint64_t* a, const uint64_t* b, uint64_t* out);
void bfvo_mul_relin(bfvo_ctx* c, const uint64_t* a, const uint64_t* b, uint64_t* out);
/* multiply without relinearisation: out is [3][L][N] */
void bfvo_mul_tensor(const bfvo_ctx* c, const uint64_t* a, const uint64_t* b, uint64_t* out3);
/* 1: the context multiplies over Q u R (2L limbs, E6-E8), 0: over Q u B (HPS, 2L+1) */
int bfvo_mul_overq(const bfvo_ctx* c);
void bfvo_rotate(bfvo_ctx* c, const uint64_t* a, int64_t k, uint64_t* out);
/* acc + rot(acc, k1) + rot(src, k2), the two key switches sharing one ModDown
 * (the batched plan's doubling step fused with the odd step after it) */
void bfvo_mul_relin_z(bfvo_ctx* c, const uint64_t* z, uint64_t* out);
void bfvo_add_galois_key_sq(bfvo_ctx* c, uint32_t g); /* not thread safe: call before parallel use */
int bfvo_get_ksk_sq(bfvo_ctx* c, uint32_t g, uint64_t* out);
/* intra_chunk_sum of one chunk from the product's tensor z ([3][L][N]) as the
 * batched plan evaluates it; fold_relin: 1 relinearisation folded into level 0,
 * 2 also two doubling steps per key-switch stage after level 0 */
int bfvo_plan_fold(bfvo_ctx* c, const uint64_t* z, int nsteps, const int64_t* offs, const int* from_acc,
                   int fold_relin, uint64_t* out);
int bfvo_rotate2_add(bfvo_ctx* c, const uint64_t* acc, const uint64_t* src, int64_t k1, int64_t k2, uint64_t* out);
/* plaintext multiply by a coefficient-form plaintext m (mod t) */
void bfvo_mul_plain(const bfvo_ctx* c, const uint64_t* a, const uint64_t* m, uint64_t* out);
/* key switch of one Q polynomial d (coef form) with the given key id */
int bfvo_key_switch(bfvo_ctx* c, uint32_t which, const uint64_t* d, uint64_t* ks0, uint64_t* ks1);
/* Galois automorphism X -> X^g on L limbs of one polynomial */
void bfvo_automorph(const bfvo_ctx* c, uint32_t g, const uint64_t* in, uint64_t* out, int limbs);

#ifdef __cplusplus
}
#endif
#endif
