/*
 * spmvgpu.h -- C-ABI of the B200-native RNS-BFV backend for the CSSC
 * encrypted-SpMV cloud phase.  Plain pointers and sizes only; no exceptions
 * cross this boundary: every call returns SPMVGPU_OK or a negative status and
 * leaves a thread-local message for spmvgpu_last_error().
 *
 * What each group replaces in the reference (/root/reference/proj):
 *   context + keys     HeParams / SimBackend ctor      include/spmv/he.hpp:35-43, 119-139
 *   ciphertext arena   Ciphertext value type           include/spmv/he.hpp:51-55
 *   encrypt/decrypt    HeBackend::encode/encrypt/decrypt  include/spmv/he.hpp:95-100
 *   add/mul/rotate     HeBackend::add/multiply/multiply_plain/rotate  he.hpp:102-110
 *   cloud plan         the cloud loop of spmv()          src/protocol.cpp:121-140
 *                      + intra_chunk_sum / inter_chunk_sum  src/aggregate.cpp:36-74
 *   cssc_spmv_*        spmv / spmv_partitioned          include/spmv/protocol.hpp:62-71
 *   cssc_pack_*        csr_to_cssc / generate_chunks / partition_rows / reorg_vector
 *                      include/spmv/sparse.hpp:68, chunk.hpp:30-35, reorg.hpp:21
 */
#ifndef SPMVGPU_H
#define SPMVGPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes; the C++ adapter maps them back to the reference's exception
 * types (include/spmv/errors.hpp:13-66) */
enum {
    SPMVGPU_OK = 0,
    SPMVGPU_ERR_INVALID_ARGUMENT = -1,  /* std::invalid_argument */
    SPMVGPU_ERR_OVER_LENGTH = -2,       /* OverLengthError */
    SPMVGPU_ERR_NOISE_EXHAUSTED = -3,   /* NoiseExhaustedError */
    SPMVGPU_ERR_DIMENSION = -4,         /* DimensionMismatchError */
    SPMVGPU_ERR_COLUMN_TOO_TALL = -5,   /* ColumnTooTallError */
    SPMVGPU_ERR_INDEX_RANGE = -6,       /* IndexOutOfRangeError */
    SPMVGPU_ERR_DUPLICATE = -7,         /* DuplicateEntryError */
    SPMVGPU_ERR_CUDA = -8,
    SPMVGPU_ERR_INTERNAL = -9,
    SPMVGPU_ERR_NON_SQUARE = -10,       /* NonSquareError (diagonal method) */
    SPMVGPU_ERR_PARSE = -11             /* ParseError (malformed CSSC buffer) */
};

typedef struct spmvgpu_ctx spmvgpu_ctx;
typedef struct spmvgpu_plan spmvgpu_plan;
typedef uint64_t spmvgpu_ct; /* opaque device ciphertext handle */

typedef struct {
    int logn;        /* ring degree N = 2^logn; slots per BFV row S = N/2 */
    int L;           /* data primes (ciphertext modulus Q) */
    int K;           /* special primes (key switching modulus P) */
    int alpha;       /* primes per key-switching digit */
    int qbits, pbits;
    uint64_t t;      /* plaintext modulus, prime, t = 1 mod 2N */
    uint64_t seed;   /* 0 (default): a 256-bit ChaCha20 key and a random stream-id base
                      * from OS entropy; nonzero: the deterministic key (seed_lo, seed_hi,
                      * 6 fixed words) and stream ids from 1 (tests / known answers) */
    int device;
    /* reference HeParams fields kept for API parity (he.hpp:24-43) */
    double ciphertext_size_mb;
    int noise_initial, noise_ct_ct, noise_ct_pt, noise_add, noise_rot;
} spmvgpu_params;

const char* spmvgpu_last_error(void);
void spmvgpu_default_params(int logn, spmvgpu_params* out);

int spmvgpu_ctx_create(const spmvgpu_params* p, spmvgpu_ctx** out);
void spmvgpu_ctx_destroy(spmvgpu_ctx* c);
/* primes (Q | P | B | t) and basic sizes */
int spmvgpu_ctx_primes(const spmvgpu_ctx* c, uint64_t* primes, int cap, int* count);
int spmvgpu_ctx_sizes(const spmvgpu_ctx* c, uint64_t* n, uint64_t* slots, uint64_t* ct_words,
                      uint64_t* ksk_words, int* dnum);
int spmvgpu_sync(spmvgpu_ctx* c);
/* tuning switches: "fused_key_switch" (1 = 3-kernel fused key switch, default;
 * 0 = the 7-launch ModUp / NTT / inner product / INTT / ModDown pipeline);
 * "plan_cache" (how many cloud plans, keyed by chunk shapes, cssc_spmv_* and
 * cssc_job_* keep for reuse with their buffers and CUDA graph; default 4, 0 = off);
 * "forked_encrypt" (spmvgpu_encrypt_cssc as two concurrent branches, upload +
 * pack beside the message-independent encryption, as the cached whole-
 * evaluation graph always does; same words; default 0);
 * "pipeline_fuse" (the cached whole-evaluation graph of cssc_spmv_batch /
 * cssc_job_run: 0 = party-separated, default: the clients' encryption writes
 * the input ciphertexts, the cloud writes the result ciphertexts, the key
 * holder decrypts them; bit 0 fuses the encryption's finish into the cloud's
 * multiply, bit 1 the decryption into the cloud's mask step; evicts cached
 * plans);
 * "stream_base" (the next stream id spmvgpu_encrypt / the pipeline hand out
 * when streams = NULL; contexts sharing a key -- the ranks of a chunk split --
 * must use disjoint ranges) */
int spmvgpu_set_option(spmvgpu_ctx* c, const char* name, int64_t value);
/* opaque CUDA stream the context works on (cudaStream_t) */
void* spmvgpu_stream(spmvgpu_ctx* c);

/* keys: generated on the device from the seed; download in canonical
 * coefficient form for word-level parity checks */
int spmvgpu_galois_keys(spmvgpu_ctx* c, const int64_t* steps, size_t n);
uint32_t spmvgpu_galois_element(const spmvgpu_ctx* c, int64_t step);
int spmvgpu_download_sk(spmvgpu_ctx* c, int64_t* out);
int spmvgpu_download_pk(spmvgpu_ctx* c, uint64_t* out);
int spmvgpu_download_ksk(spmvgpu_ctx* c, uint32_t which, uint64_t* out); /* 0 = relin */

/* ciphertext arena: [2][L][N] uint64 words, coefficient form */
int spmvgpu_ct_alloc(spmvgpu_ctx* c, size_t count, spmvgpu_ct* out);
int spmvgpu_ct_free(spmvgpu_ctx* c, const spmvgpu_ct* cts, size_t count);
int spmvgpu_ct_upload(spmvgpu_ctx* c, spmvgpu_ct ct, const uint64_t* words);
int spmvgpu_ct_download(spmvgpu_ctx* c, spmvgpu_ct ct, uint64_t* words);
/* wire format (in place of protocol.cpp:51-54's 0.52 MB price):
 * 16-byte header (magic, logn, L, fingerprint of Q) + every residue of q_j at
 * bitlen(q_j) bits.  Deserialisation rejects foreign headers and residues >= q_j. */
int spmvgpu_ct_wire_size(spmvgpu_ctx* c, size_t* bytes);
int spmvgpu_ct_serialize(spmvgpu_ctx* c, spmvgpu_ct ct, uint8_t* buf, size_t cap, size_t* written);
int spmvgpu_ct_deserialize(spmvgpu_ctx* c, const uint8_t* buf, size_t len, spmvgpu_ct ct);

/* batched encode+encrypt: item i encodes vals[offsets[i] .. offsets[i+1]) into
 * row 0 of the slots with encryption stream streams[i] (0 = next fresh id;
 * streams may be NULL) */
int spmvgpu_encrypt(spmvgpu_ctx* c, const int64_t* vals, const uint64_t* offsets,
                    const uint64_t* streams, const spmvgpu_ct* out, size_t n);
/* Client A + Client B fused on the device (replaces the host chain of
 * reference sparse.cpp:79-117 csr_to_cssc, chunk.cpp:10-52 generate_chunks,
 * reorg.cpp:10-34 reorg_vector and he.cpp encode/encrypt per chunk): scatters
 * CSR entries straight into the CSSC chunk plaintexts and encrypts them.
 *   col_indices/values: nnz entries (all matrices back to back);
 *   vec: vec_len entries (all vectors back to back);
 *   rows: n_rows x {nz_begin, len, pos, slice}: every non-empty row of every
 *         slice, pos = its place in the slice's descending-length order;
 *   slices: n_slices x {col_base, vec_base};
 *   cols: n_cols x {chunk, k, h, 0}: aligned column j of a slice is record
 *         col_base + j, slot k*h + pos of chunk `chunk` (height h); chunk -1
 *         drops the column's entries (a chunk another GPU evaluates).
 * Entry j of a row lands in out[chunk] (value) and out[n_chunks + chunk]
 * (vec[vec_base + col]); all other slots are 0.  Stream ids as for
 * spmvgpu_encrypt with streams = NULL.  Every index is validated. */
int spmvgpu_encrypt_cssc(spmvgpu_ctx* c, const int64_t* col_indices, const int64_t* values, uint64_t nnz,
                         const int64_t* vec, uint64_t vec_len, const int32_t* rows, uint64_t n_rows,
                         const int32_t* slices, uint64_t n_slices, const int32_t* cols, uint64_t n_cols,
                         const spmvgpu_ct* out, size_t n_chunks);
/* batched decrypt+decode: slots is n x S residues mod t; budgets = measured
 * invariant-noise budget (bits, saturates near 60) */
int spmvgpu_decrypt(spmvgpu_ctx* c, const spmvgpu_ct* cts, size_t n, uint64_t* slots,
                    int32_t* budgets);
int spmvgpu_add(spmvgpu_ctx* c, const spmvgpu_ct* a, const spmvgpu_ct* b, const spmvgpu_ct* out,
                size_t n);
int spmvgpu_mul_relin(spmvgpu_ctx* c, const spmvgpu_ct* a, const spmvgpu_ct* b,
                      const spmvgpu_ct* out, size_t n);
/* out = cts[0] + ... + cts[n-1] in one launch (n = 0: the zero ciphertext) */
int spmvgpu_sum(spmvgpu_ctx* c, const spmvgpu_ct* cts, size_t n, spmvgpu_ct out);
/* out_i = rot(src_i, steps_i) (cyclic left over S slots, negative = right) */
int spmvgpu_rotate(spmvgpu_ctx* c, const spmvgpu_ct* src, const int64_t* steps,
                   const spmvgpu_ct* out, size_t n);
/* out_i = acc_i + rot(src_i, steps_i): the fused rotate-and-add tree step */
int spmvgpu_rotate_add(spmvgpu_ctx* c, const spmvgpu_ct* acc, const spmvgpu_ct* src,
                       const int64_t* steps, const spmvgpu_ct* out, size_t n);
/* out_i = a_i * encode(vals[offsets[i] .. offsets[i+1])) */
int spmvgpu_mul_plain(spmvgpu_ctx* c, const spmvgpu_ct* a, const int64_t* vals,
                      const uint64_t* offsets, const spmvgpu_ct* out, size_t n);
/* KAT: in-place forward/inverse NTT of `limbs` host limbs modulo prime index */
int spmvgpu_ntt(spmvgpu_ctx* c, int prime_index, uint64_t* data, size_t limbs, int inverse);

/* roofline probes, timed with CUDA events on the context stream:
 * average device time (us) of one batched NTT launch over `limbs` device limbs
 * (the kernel the cloud plan launches), and the register-resident peak of the
 * identical lazy Shoup butterfly sequence (butterflies per second). */
int spmvgpu_probe_ntt(spmvgpu_ctx* c, size_t limbs, int inverse, int reps, double* us_per_launch);
int spmvgpu_probe_butterfly_peak(spmvgpu_ctx* c, double* butterflies_per_s);

/* ---- the batched cloud phase: every chunk of every slice in shared launches ----
 * chunk i: product of a_cts[i] and b_cts[i], folded by rotation_schedule(r_i, c_i),
 * masked to its first r_i slots and accumulated into out_cts[slice_i]. */
int spmvgpu_plan_create(spmvgpu_ctx* c, size_t n_chunks, const uint64_t* r, const uint64_t* cols,
                        const uint32_t* slice, size_t n_slices, const spmvgpu_ct* a_cts,
                        const spmvgpu_ct* b_cts, const spmvgpu_ct* out_cts, spmvgpu_plan** out);
int spmvgpu_plan_run(spmvgpu_plan* p);         /* enqueue on the context stream */
int spmvgpu_plan_capture(spmvgpu_plan* p);     /* record a CUDA graph; later runs replay it */
typedef struct {
    uint64_t chunks, slices, levels, kernels_per_run, limb_ntts_per_run;
    uint64_t rotations, distinct_keys;
    uint64_t hbm_bytes_algorithmic; /* compulsory bytes per run (SURVEY 8(d) formulas) */
    uint64_t key_bytes_per_run;
    uint64_t relin_folded; /* 1: the rotated chunks' relinearisation shares level 0's ModDown (DESIGN 2.9) */
} spmvgpu_plan_stats;
int spmvgpu_plan_stats_get(const spmvgpu_plan* p, spmvgpu_plan_stats* out);
/* one CUDA-graph replay of the plan with event nodes between launch groups
 * (multiply+relin, each rotate level, the level-0 add, mask accumulate; the
 * L2 is left as the caller left it): device time per group, its
 * compulsory HBM bytes (SURVEY 8(d) op table) and limb NTTs; *count = groups */
typedef struct {
    char name[32];
    double us;
    uint64_t items, bytes, limb_ntts;
    uint64_t sources;   /* distinct key-switch sources (< items when a level's ModUp is hoisted) */
    uint64_t acc_items; /* key switches accumulated (> items: odd steps share their doubling step's ModDown) */
    uint64_t mac_terms; /* key products summed (folded level 0: relinearisation + rotations of z1 and z2) */
} spmvgpu_phase;
int spmvgpu_plan_profile(spmvgpu_plan* p, spmvgpu_phase* phases, int cap, int* count);
/* per kernel launch of the plan: `reps` graph replays, each after an L2 flush
 * (a memset of flush_bytes), with an event node after every launch; mean us
 * per launch, its kernel name and the launch group it belongs to (the index
 * into spmvgpu_plan_profile's groups); *count = launches */
typedef struct {
    char name[48];
    int32_t group;
    double us;
} spmvgpu_kernel_timing;
int spmvgpu_plan_profile_kernels(spmvgpu_plan* p, int reps, uint64_t flush_bytes, spmvgpu_kernel_timing* out,
                                 int cap, int* count);
void spmvgpu_plan_destroy(spmvgpu_plan* p);

/* ---- protocol level (host C++ above the device ABI) ---- */
typedef struct {
    uint64_t n_mult_cc, n_mult_cp, n_rot, n_add, n_enc, n_dec;
} cssc_ledger;
typedef struct {
    int64_t from, to, kind, payload_bytes, ciphertext_count;
} cssc_message; /* roles A=0 B=1 Cloud=2; kinds per protocol.hpp:25-31 */
typedef struct {
    uint64_t rows, cols;
    const int64_t* row_ptrs;    /* rows + 1 */
    const int64_t* col_indices; /* nnz */
    const int64_t* values;      /* nnz */
} cssc_csr;
typedef struct {
    cssc_ledger ledger;
    uint64_t n_ct;
    int32_t noise_model_bits;     /* reference model counter (87 with >= 1 chunk) */
    int32_t noise_measured_bits;  /* min measured BFV budget over slices */
    uint64_t n_messages;
} cssc_result;

/* spmv on the GPU backend (reference protocol.cpp:74-153): one slice, every row
 * in one chunk set (rows <= slot budget, else ColumnTooTallError) */
int cssc_spmv(spmvgpu_ctx* c, const cssc_csr* m, const int64_t* v, uint64_t vlen, uint64_t chunk_size,
              int key_holder, int64_t* values, cssc_result* res, cssc_message* msgs, uint64_t msg_cap);
/* spmv_partitioned on the GPU backend: values (rows) in original row order */
int cssc_spmv_partitioned(spmvgpu_ctx* c, const cssc_csr* m, const int64_t* v, uint64_t vlen,
                          uint64_t chunk_size, int key_holder, int64_t* values,
                          cssc_result* res, cssc_message* msgs, uint64_t msg_cap);
/* the diagonal-method baseline (reference diagonal.cpp:56-104) on the GPU
 * backend: square matrices, n <= slots/2 (or n == slots); values has n rows */
int cssc_diag_spmv(spmvgpu_ctx* c, const cssc_csr* m, const int64_t* v, uint64_t vlen, int key_holder,
                   int64_t* values, cssc_result* res, cssc_message* msgs, uint64_t msg_cap);
/* several independent matrices in shared launches (BASELINE config 5) */
/* vlens[i] = length of vs[i]; != ms[i].cols raises DimensionMismatchError */
int cssc_spmv_batch(spmvgpu_ctx* c, const cssc_csr* ms, const int64_t* const* vs, const uint64_t* vlens, size_t nmat,
                    uint64_t chunk_size, int key_holder, int64_t* const* values,
                    cssc_result* res);
/* optional, before marshalling a cssc_spmv_batch call: enqueue the early
 * (message-independent) encryption graph of the previous call's plan with the
 * stream ids the next call will assign, so the device starts while the host
 * still prepares the call; cssc_spmv_batch does it itself otherwise, and
 * re-runs it when the next call selects another plan */
int cssc_speculate(spmvgpu_ctx* c);

/* staged form for benchmarking: pack + encrypt once, run the cloud phase many
 * times from device-resident ciphertexts, then decrypt */
typedef struct cssc_job cssc_job;
int cssc_job_create(spmvgpu_ctx* c, const cssc_csr* ms, const int64_t* const* vs, const uint64_t* vlens, size_t nmat,
                    uint64_t chunk_size, cssc_job** out);
/* SURVEY 8(e) chunk split: this GPU evaluates the chunks g with g % world == rank;
 * cssc_job_result_words gives its per-slice partial results ([results][ct words],
 * zeros where it holds no chunk of a slice; words = NULL: count only), the caller
 * sums them across GPUs (mod q_j per limb), and cssc_job_finish_words decrypts */
int cssc_job_create_shard(spmvgpu_ctx* c, const cssc_csr* ms, const int64_t* const* vs, const uint64_t* vlens, size_t nmat,
                          uint64_t chunk_size, int rank, int world, cssc_job** out);
int cssc_job_result_words(cssc_job* j, uint64_t* words, uint64_t cap_words, uint64_t* n_results);
int cssc_job_finish_words(cssc_job* j, const uint64_t* words, int64_t* const* values, cssc_result* res);
/* the same with the words in DEVICE memory of the context's GPU, for an
 * all-reduce that stays on the device (NCCL over NVLink): result_words_dev
 * copies this rank's partials into dev_words ([results][ct words]) and waits;
 * finish_words_dev folds the summed words mod q_j in place (spmvgpu_fold_mod)
 * and decrypts */
int cssc_job_result_words_dev(cssc_job* j, uint64_t* dev_words, uint64_t cap_words, uint64_t* n_results);
int cssc_job_finish_words_dev(cssc_job* j, uint64_t* dev_words, int64_t* const* values, cssc_result* res);
/* device words [n_cts][2][L][N], each a sum of <= 16 residues < q_j: reduce mod q_j in place */
int spmvgpu_fold_mod(spmvgpu_ctx* c, uint64_t* dev_words, uint64_t n_cts);
int cssc_job_encrypt(cssc_job* j);            /* client phase: encode + encrypt on device */
int cssc_job_cloud(cssc_job* j, int use_graph); /* cloud phase, enqueued (no sync) */
/* the same between two caller-created cudaEvent_t records on the context
 * stream, both issued inside this call (no host gap inside the bracket) */
int cssc_job_cloud_timed(cssc_job* j, int use_graph, void* ev_start, void* ev_stop);
int cssc_job_finish(cssc_job* j, int64_t* const* values, cssc_result* res); /* decrypt */
/* encrypt + cloud + decrypt in one call (what cssc_spmv_batch runs): from the
 * second job over a chunk-shape structure, one cached graph launch */
int cssc_job_run(cssc_job* j, int64_t* const* values, cssc_result* res);
int cssc_job_plan_stats(const cssc_job* j, spmvgpu_plan_stats* out);
int cssc_job_profile(cssc_job* j, spmvgpu_phase* phases, int cap, int* count); /* see spmvgpu_plan_profile */
int cssc_job_profile_kernels(cssc_job* j, int reps, uint64_t flush_bytes, spmvgpu_kernel_timing* out, int cap,
                             int* count); /* see spmvgpu_plan_profile_kernels */
int cssc_job_input_bytes(const cssc_job* j, uint64_t* h2d, uint64_t* d2h);
void cssc_job_destroy(cssc_job* j);

/* host pack helpers (reference algorithms, exposed for parity tests) */
int64_t cssc_pack_chunks(const cssc_csr* m, uint64_t budget, int64_t* r_list, int64_t* c_list,
                         int64_t* vflat, int64_t* cflat, int64_t* row_map, uint64_t* flat_total);
int cssc_rotation_schedule(uint64_t rows, uint64_t cols, uint64_t* offsets, int32_t* from_acc);
/* CSSC persistence, in place of `spmv convert` (reference
 * tools/spmv_main.cpp:39-58): csr_to_cssc + validate_cssc, then the compact
 * binary form (buf NULL: size only) or the reference's JSON text (same bytes
 * as its ordered_json dump(2)); cssc_load_binary returns the CSSC arrays
 * (va, ci, rm, cp; NULL arrays: sizes only) and raises ParseError on a
 * malformed buffer */
int cssc_convert_binary(const cssc_csr* m, uint8_t* buf, uint64_t cap, uint64_t* written);
int cssc_convert_json(const cssc_csr* m, char* buf, uint64_t cap, uint64_t* written);
int cssc_load_binary(const uint8_t* buf, uint64_t len, uint64_t* rows, uint64_t* cols, uint64_t* nnz,
                     uint64_t* aligned_cols, int64_t* va, uint64_t* ci, uint64_t* rm, uint64_t* cp);

#ifdef __cplusplus
}
#endif
#endif
