/*
 * sim_oracle.c -- plain-C restatement of the reference's encrypted-SpMV path
 * at the slot level ("L1"): SimBackend semantics, CSSC build, greedy
 * chunker, row partitioner, vector reorganisation, rotate-and-add schedule,
 * masked inter-chunk stacking, and the three-party transcript pricing.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline leg may call it, and only as the checker.  It is
 * pinned against the reference's own golden vectors (tests/test_oracle_sim.py)
 * and against the reference library itself built from /root/reference into
 * oracle/_ref (see tests/golden/ and tests/test_oracle_ref.py).
 *
 * Each function names the reference lines it restates.
 */
#include <stddef.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>

typedef uint64_t u64;
typedef int64_t i64;

/* he.cpp:42-56 */
i64 simo_to_signed(u64 r, u64 t) { return r <= t / 2 ? (i64)r : (i64)r - (i64)t; }
u64 simo_to_residue(i64 v, u64 t) {
    i64 m = (i64)t, r = v % m;
    if (r < 0) r += m;
    return (u64)r;
}

/* aggregate.cpp:12-34: writes (offset, from_acc) pairs; returns step count */
int simo_rotation_schedule(u64 rows, u64 cols, u64* offsets, int* from_acc) {
    if (rows == 0 || cols == 0) return -1;
    int nb = 64 - __builtin_clzll(cols);
    u64 e = 1;
    int k = 0;
    for (int j = nb - 2; j >= 0; --j) {
        if (offsets) { offsets[k] = e * rows; from_acc[k] = 1; }
        k++;
        e *= 2;
        if ((cols >> j) & 1u) {
            if (offsets) { offsets[k] = e * rows; from_acc[k] = 0; }
            k++;
            e += 1;
        }
    }
    return k;
}

/* sparse.cpp:79-117.  rm/cp/va/ci are caller buffers (rows, max_nnz+1, nnz, nnz).
 * returns L = number of aligned columns. */
typedef struct { size_t idx; size_t key; } pair_t;
static int cmp_desc_stable(const void* a, const void* b) {
    const pair_t* x = (const pair_t*)a;
    const pair_t* y = (const pair_t*)b;
    if (x->key != y->key) return x->key > y->key ? -1 : 1;
    return x->idx < y->idx ? -1 : (x->idx > y->idx);
}
i64 simo_csr_to_cssc(u64 rows, const i64* row_ptrs, const i64* col_idx, const i64* vals,
                     i64* rm, i64* cp, i64* va, i64* ci) {
    pair_t* pr = (pair_t*)malloc(sizeof(pair_t) * (rows ? rows : 1));
    size_t maxn = 0;
    for (size_t i = 0; i < rows; i++) {
        pr[i].idx = i;
        pr[i].key = (size_t)(row_ptrs[i + 1] - row_ptrs[i]);
        if (pr[i].key > maxn) maxn = pr[i].key;
    }
    qsort(pr, rows, sizeof(pair_t), cmp_desc_stable); /* (key desc, idx asc) == stable */
    for (size_t p = 0; p < rows; p++) rm[p] = (i64)pr[p].idx;
    size_t w = 0;
    for (size_t j = 0; j < maxn; j++) {
        cp[j] = (i64)w;
        for (size_t p = 0; p < rows; p++) {
            size_t i = pr[p].idx;
            if (j < pr[p].key) {
                size_t k = (size_t)row_ptrs[i] + j;
                va[w] = vals[k];
                ci[w] = col_idx[k];
                w++;
            } else {
                break; /* sorted descending: no later row is longer */
            }
        }
    }
    cp[maxn] = (i64)w;
    free(pr);
    return (i64)maxn;
}

/* chunk.cpp:10-50.  Fills r_list/c_list and the flats (column-major, 0/-1
 * padding); returns n_ct, or -1 when a column is taller than the budget
 * (ColumnTooTallError). flat buffers must hold sum(r*c) entries. */
i64 simo_generate_chunks(i64 L, const i64* cp, const i64* va, const i64* ci, u64 budget,
                         i64* r_list, i64* c_list, i64* flat_off, i64* vflat, i64* cflat) {
    for (i64 j = 0; j < L; j++)
        if ((u64)(cp[j + 1] - cp[j]) > budget) return -1;
    i64 i = 0, n = 0, off = 0;
    while (i < L) {
        u64 h = (u64)(cp[i + 1] - cp[i]);
        u64 cols = 0;
        if (flat_off) flat_off[n] = off;
        while (i < L && h * (cols + 1) <= budget) {
            u64 height = (u64)(cp[i + 1] - cp[i]);
            for (i64 x = cp[i]; x < cp[i + 1]; x++) {
                if (vflat) { vflat[off] = va[x]; cflat[off] = ci[x]; }
                off++;
            }
            for (u64 pad = height; pad < h; pad++) {
                if (vflat) { vflat[off] = 0; cflat[off] = -1; }
                off++;
            }
            cols++;
            i++;
        }
        if (r_list) { r_list[n] = (i64)h; c_list[n] = (i64)cols; }
        n++;
    }
    if (flat_off) flat_off[n] = off;
    return n;
}

/* ------------------------------------------------------------------ */
/* SimBackend slot arithmetic (he.cpp:93-148) on S-slot vectors          */
/* ------------------------------------------------------------------ */
typedef struct {
    u64 n_mult_cc, n_mult_cp, n_rot, n_add, n_enc, n_dec;
} ledger_t;

static void v_add(u64* o, const u64* a, const u64* b, size_t S, u64 t) {
    for (size_t i = 0; i < S; i++) o[i] = (a[i] + b[i]) % t;
}
static void v_mul(u64* o, const u64* a, const u64* b, size_t S, u64 t) {
    for (size_t i = 0; i < S; i++) o[i] = (u64)(((unsigned __int128)a[i] * b[i]) % t);
}
static void v_rot(u64* o, const u64* a, i64 k, size_t S) {
    i64 n = (i64)S;
    size_t sh = (size_t)(((k % n) + n) % n);
    for (size_t i = 0; i < S; i++) o[i] = a[(i + sh) % S];
}

/* Message record: from, to, kind, payload_bytes, ciphertext_count
 * (roles A=0 B=1 Cloud=2; kinds as protocol.hpp:25-31) */
typedef struct { i64 from, to, kind, bytes, count; } msg_t;

static u64 batch_bytes(double mb, size_t count) {
    return (u64)llround((double)count * mb * 1048576.0);
}

typedef struct {
    size_t S;
    u64 t;
    double ct_mb;
    int init_budget, cost_cc, cost_cp, cost_add, cost_rot;
} simparams_t;

static int lowered(int b, int c) { return b - c > 0 ? b - c : 0; }

/* protocol.cpp:74-153 for one slice; appends messages; returns n_ct or
 * -1 (ColumnTooTall) / -2 (dimension) / -3 (chunk size) */
static i64 spmv_slice(const simparams_t* P, u64 rows, const i64* rp, const i64* cix,
                      const i64* vals, const i64* v, size_t chunk, int key_holder, i64* out_vals,
                      ledger_t* led, msg_t* msgs, size_t* nmsg, int* noise) {
    if (chunk == 0 || chunk > P->S) return -3;
    size_t nnz = (size_t)rp[rows];
    i64* rm = (i64*)malloc(sizeof(i64) * (rows + 1));
    i64 maxn = 0;
    for (u64 i = 0; i < rows; i++) if (rp[i + 1] - rp[i] > maxn) maxn = rp[i + 1] - rp[i];
    i64* cp = (i64*)malloc(sizeof(i64) * (maxn + 2));
    i64* va = (i64*)malloc(sizeof(i64) * (nnz + 1));
    i64* ci = (i64*)malloc(sizeof(i64) * (nnz + 1));
    i64 L = simo_csr_to_cssc(rows, rp, cix, vals, rm, cp, va, ci);
    i64 nct = simo_generate_chunks(L, cp, va, ci, chunk, NULL, NULL, NULL, NULL, NULL);
    if (nct < 0) { free(rm); free(cp); free(va); free(ci); return -1; }
    i64* rl = (i64*)malloc(sizeof(i64) * (nct + 1));
    i64* cl = (i64*)malloc(sizeof(i64) * (nct + 1));
    i64* fo = (i64*)malloc(sizeof(i64) * (nct + 2));
    i64 tot = 0;
    simo_generate_chunks(L, cp, va, ci, chunk, rl, cl, fo, NULL, NULL);
    tot = fo[nct];
    i64* vf = (i64*)malloc(sizeof(i64) * (tot + 1));
    i64* cf = (i64*)malloc(sizeof(i64) * (tot + 1));
    simo_generate_chunks(L, cp, va, ci, chunk, rl, cl, fo, vf, cf);

    size_t S = P->S;
    u64 t = P->t;
    /* Client A: encode + encrypt chunk values (he.cpp:64-82) */
    u64* A = (u64*)calloc((size_t)nct * S + 1, sizeof(u64));
    u64* Bv = (u64*)calloc((size_t)nct * S + 1, sizeof(u64));
    for (i64 c = 0; c < nct; c++)
        for (i64 x = fo[c]; x < fo[c + 1]; x++) A[(size_t)c * S + (size_t)(x - fo[c])] = simo_to_residue(vf[x], t);
    led->n_enc += (u64)nct;
    u64 cib = 4;
    for (i64 c = 0; c < nct; c++) cib += 8 + 4 * (u64)(fo[c + 1] - fo[c]);
    msgs[(*nmsg)++] = (msg_t){0, 2, 0, (i64)batch_bytes(P->ct_mb, (size_t)nct), nct};
    msgs[(*nmsg)++] = (msg_t){0, 1, 1, (i64)cib, 0};
    msgs[(*nmsg)++] = (msg_t){0, 2, 2, (i64)(4 + 8 * (u64)nct), 0};
    /* Client B: reorg_vector (reorg.cpp:10-34) + encrypt */
    for (i64 c = 0; c < nct; c++)
        for (i64 x = fo[c]; x < fo[c + 1]; x++) {
            i64 idx = cf[x];
            Bv[(size_t)c * S + (size_t)(x - fo[c])] = idx < 0 ? 0 : simo_to_residue(v[idx], t);
        }
    led->n_enc += (u64)nct;
    msgs[(*nmsg)++] = (msg_t){1, 2, 0, (i64)batch_bytes(P->ct_mb, (size_t)nct), nct};

    u64* res = (u64*)calloc(S, sizeof(u64));
    if (nct > 0) {
        u64* prod = (u64*)malloc(sizeof(u64) * S);
        u64* acc = (u64*)malloc(sizeof(u64) * S);
        u64* tmp = (u64*)malloc(sizeof(u64) * S);
        u64* mask = (u64*)malloc(sizeof(u64) * S);
        u64 offs[160];
        int fa[160];
        int res_b = P->init_budget; /* zero_ciphertext() carries the initial budget */
        for (i64 c = 0; c < nct; c++) {
            v_mul(prod, A + (size_t)c * S, Bv + (size_t)c * S, S, t);
            led->n_mult_cc++;
            int prod_b = lowered(P->init_budget, P->cost_cc);
            /* intra_chunk_sum (aggregate.cpp:36-48) */
            memcpy(acc, prod, sizeof(u64) * S);
            int acc_b = prod_b;
            int ns = simo_rotation_schedule((u64)rl[c], (u64)cl[c], offs, fa);
            for (int s = 0; s < ns; s++) {
                v_rot(tmp, fa[s] ? acc : prod, (i64)offs[s], S);
                int rot_b = lowered(fa[s] ? acc_b : prod_b, P->cost_rot);
                led->n_rot++;
                v_add(acc, acc, tmp, S, t);
                acc_b = lowered(acc_b < rot_b ? acc_b : rot_b, P->cost_add);
                led->n_add++;
            }
            /* inter_chunk_sum (aggregate.cpp:55-74) */
            for (size_t i = 0; i < S; i++) mask[i] = i < (size_t)rl[c] ? 1 % t : 0;
            v_mul(tmp, acc, mask, S, t);
            int masked_b = lowered(acc_b, P->cost_cp);
            led->n_mult_cp++;
            v_add(res, res, tmp, S, t);
            res_b = lowered(res_b < masked_b ? res_b : masked_b, P->cost_add);
            led->n_add++;
        }
        msgs[(*nmsg)++] = (msg_t){2, key_holder, 3, (i64)batch_bytes(P->ct_mb, 1), 1};
        led->n_dec++;
        *noise = res_b;
        free(prod); free(acc); free(tmp); free(mask);
    } else {
        *noise = P->init_budget;
    }
    for (u64 idx = 0; idx < rows; idx++) {
        i64 val = idx < S ? simo_to_signed(res[idx], t) : 0;
        out_vals[rm[idx]] = val;
    }
    free(rm); free(cp); free(va); free(ci); free(rl); free(cl); free(fo); free(vf); free(cf);
    free(A); free(Bv); free(res);
    return nct;
}

/* protocol.cpp:155-176.  msgs must hold 5 * ceil(rows/chunk) records.
 * ledger6 = {cc, cp, rot, add, enc, dec}.  Returns total n_ct or < 0. */
i64 simo_spmv_partitioned(u64 S, u64 t, double ct_mb, const int* noise5, u64 rows, u64 cols,
                          const i64* rp, const i64* cix, const i64* vals, const i64* v,
                          u64 vlen, u64 chunk, int key_holder, i64* out_vals, u64* ledger6,
                          i64* msgs_out, u64* nmsgs, int* noise_out) {
    if (vlen != cols) return -2;
    if (chunk == 0) return -3;
    simparams_t P = {S, t, ct_mb, noise5[0], noise5[1], noise5[2], noise5[3], noise5[4]};
    ledger_t led = {0, 0, 0, 0, 0, 0};
    size_t nmsg = 0;
    msg_t* msgs = (msg_t*)msgs_out;
    int noise = P.init_budget;
    i64 total = 0;
    for (u64 start = 0; start < rows; start += chunk) {
        u64 end = start + chunk < rows ? start + chunk : rows;
        u64 sr = end - start;
        i64 base = rp[start];
        i64* srp = (i64*)malloc(sizeof(i64) * (sr + 1));
        for (u64 i = 0; i <= sr; i++) srp[i] = rp[start + i] - base;
        int nz;
        i64 r = spmv_slice(&P, sr, srp, cix + base, vals + base, v, chunk, key_holder,
                           out_vals + start, &led, msgs, &nmsg, &nz);
        free(srp);
        if (r < 0) return r;
        total += r;
        if (nz < noise) noise = nz;
    }
    ledger6[0] = led.n_mult_cc; ledger6[1] = led.n_mult_cp; ledger6[2] = led.n_rot;
    ledger6[3] = led.n_add; ledger6[4] = led.n_enc; ledger6[5] = led.n_dec;
    *nmsgs = nmsg;
    *noise_out = noise;
    return total;
}

/* SimBackend rotate on a raw slot vector (he.cpp:138-148), for golden tests */
void simo_rotate(const u64* a, i64 k, u64 S, u64* out) { v_rot(out, a, k, S); }
