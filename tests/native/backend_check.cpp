// backend_check.cpp -- the drop-in boundary exercised from C++, the way a
// reference user would: include spmv/*.hpp, link libcssc_he.so, construct
// spmv::GpuBfvBackend and call every HeBackend virtual (he.hpp:86-115) plus
// the reference's op-by-op aggregation (aggregate.cpp:36-74) over it.
//
// The cases restate the reference's own unit tests
// (/root/reference/proj/tests/test_he.cpp:28-207) at the GPU backend's
// parameters: slot_count = N/2 = 2048, t = 65537.  Checks that need an
// independent oracle (ciphertext words vs oracle/bfv_oracle.c, values and
// ledger vs the compiled reference) are done by tests/test_gpu_backend_cpp.py
// from what this program writes: `words <name> <file>` (raw uint64 ciphertext
// words), `ledger <name> cc cp rot add enc dec`, `slots <name> v0 v1 ...`.
//
// usage: backend_check <out_dir> ; exit code = number of failed checks
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

#include "spmv/aggregate.hpp"
#include "spmv/gpu_backend.hpp"
#include "spmv/protocol.hpp"

using namespace spmv;

static int failures = 0;
#define CHECK(x)                                                                 \
    do {                                                                         \
        if (!(x)) {                                                              \
            std::fprintf(stderr, "FAIL %s:%d: %s\n", __FILE__, __LINE__, #x);    \
            ++failures;                                                          \
        }                                                                        \
    } while (0)
#define CHECK_THROWS_AS(expr, T)                                                 \
    do {                                                                         \
        bool caught_ = false;                                                    \
        try {                                                                    \
            (void)(expr);                                                        \
        } catch (const T&) {                                                     \
            caught_ = true;                                                      \
        } catch (const std::exception& e_) {                                     \
            std::fprintf(stderr, "  other exception: %s\n", e_.what());          \
        }                                                                        \
        if (!caught_) {                                                          \
            std::fprintf(stderr, "FAIL %s:%d: %s throws %s\n", __FILE__, __LINE__, #expr, #T); \
            ++failures;                                                          \
        }                                                                        \
    } while (0)

static std::string g_out;
static constexpr std::uint64_t kT = 65537;
static constexpr std::size_t kS = 2048;  // slot_count = N/2, N = 4096

static HeParams params(NoiseModel nm = {}) {
    HeParams p;
    p.slot_count = kS;
    p.plaintext_modulus = kT;
    p.noise = nm;
    return p;
}

static GpuBfvOptions seeded(std::uint64_t seed) {
    GpuBfvOptions o;
    o.seed = seed;  // deterministic key: oracle/bfv_oracle.c restates it
    return o;
}

static void dump_words(const GpuBfvBackend& be, const char* name, const Ciphertext& ct) {
    std::uint64_t n = 0, slots = 0, ctw = 0, kw = 0;
    int dnum = 0;
    check_status(spmvgpu_ctx_sizes(be.context(), &n, &slots, &ctw, &kw, &dnum));
    std::vector<std::uint64_t> w(ctw);
    check_status(spmvgpu_ct_download(be.context(), be.handle(ct), w.data()));
    const std::string path = g_out + "/" + name + ".u64";
    FILE* f = std::fopen(path.c_str(), "wb");
    if (!f) throw std::runtime_error("cannot write " + path);
    std::fwrite(w.data(), 8, w.size(), f);
    std::fclose(f);
    std::printf("words %s %s\n", name, path.c_str());
}

static void print_ledger(const char* name, const OpLedger& l) {
    std::printf("ledger %s %llu %llu %llu %llu %llu %llu\n", name, (unsigned long long)l.n_mult_cc,
                (unsigned long long)l.n_mult_cp, (unsigned long long)l.n_rot, (unsigned long long)l.n_add,
                (unsigned long long)l.n_enc, (unsigned long long)l.n_dec);
}

static void print_slots(const char* name, const SlotVector& s, std::size_t k) {
    std::printf("slots %s", name);
    for (std::size_t i = 0; i < k && i < s.size(); ++i) std::printf(" %llu", (unsigned long long)s[i]);
    std::printf("\n");
}

static SlotVector padded(std::initializer_list<std::uint64_t> xs) {
    SlotVector v(kS, 0);
    std::size_t i = 0;
    for (auto x : xs) v[i++] = x;
    return v;
}

// test_he.cpp:28-48
static void encode_cases() {
    GpuBfvBackend be(params(), seeded(3));
    const std::int64_t input[] = {1, 2, 3};
    CHECK(be.encode(input).slots == padded({1, 2, 3}));
    const std::int64_t negative[] = {-1};
    CHECK(be.encode(negative).slots[0] == kT - 1);
    const std::int64_t wrap[] = {65537, 65538, -65538};
    const Plaintext w = be.encode(wrap);
    CHECK(w.slots[0] == 0 && w.slots[1] == 1 && w.slots[2] == kT - 1);
    const std::vector<std::int64_t> too_long(kS + 1, 1);
    CHECK_THROWS_AS(be.encode(too_long), OverLengthError);
    CHECK(to_signed(0, kT) == 0 && to_signed(32768, kT) == 32768 && to_signed(32769, kT) == -32768);
    CHECK(to_signed(65536, kT) == -1 && to_residue(-1, kT) == 65536);
}

// test_he.cpp:65-129 (budgets are the model counter; decrypt also checks the measured budget)
static void budget_cases() {
    GpuBfvBackend be(params(), seeded(4));
    OpLedger ledger;
    const std::int64_t five[] = {5};
    Ciphertext a = be.encrypt(be.encode(five), ledger);
    Ciphertext b = be.encrypt(be.encode(five), ledger);
    CHECK(a.noise_budget_bits == 146);
    CHECK(a.id != b.id);
    CHECK(ledger.n_enc == 2);
    CHECK(be.decrypt(a, ledger)[0] == 5);
    CHECK(ledger.n_dec == 1);

    const std::int64_t two[] = {2};
    Ciphertext ct = be.encrypt(be.encode(two), ledger);
    for (int i = 0; i < 5; ++i) ct = be.multiply(ct, ct, ledger);
    CHECK(ct.noise_budget_bits == 0);
    CHECK_THROWS_AS(be.decrypt(ct, ledger), NoiseExhaustedError);

    const std::int64_t three[] = {3};
    Ciphertext c3 = be.encrypt(be.encode(three), ledger);
    c3 = be.multiply(c3, c3, ledger);
    CHECK(c3.noise_budget_bits == 113);
    c3 = be.multiply_plain(c3, be.encode(three), ledger);
    CHECK(c3.noise_budget_bits == 87);
    CHECK(be.decrypt(c3, ledger)[0] == 27);

    const int model_cc[] = {146, 113, 80, 47, 14, 0, 0};
    const int model_cp[] = {146, 120, 94, 68, 42, 16, 0};
    const std::int64_t one[] = {1};
    Ciphertext cc = be.encrypt(be.encode(one), ledger);
    Ciphertext cp = be.encrypt(be.encode(one), ledger);
    const Plaintext pt_one = be.encode(one);
    for (int k = 0; k <= 6; ++k) {
        CHECK(cc.noise_budget_bits == model_cc[k]);
        CHECK(cp.noise_budget_bits == model_cp[k]);
        cc = be.multiply(cc, cc, ledger);
        cp = be.multiply_plain(cp, pt_one, ledger);
    }
}

// the real BFV budget behind the model: with a model that never
// runs out, repeated squaring must end in NoiseExhaustedError from the
// measured budget, and every decryption before that must be right; a
// ciphertext of random words has no budget at all
static void measured_noise_cases() {
    GpuBfvBackend be(params(NoiseModel{146, 0, 0, 0, 0}), seeded(5));
    OpLedger ledger;
    const std::int64_t two[] = {2};
    Ciphertext ct = be.encrypt(be.encode(two), ledger);
    std::uint64_t want = 2;
    int squarings = 0, last_budget = be.measured_noise_budget(ct);
    std::printf("measured fresh %d\n", last_budget);
    bool exhausted = false;
    for (; squarings < 8 && !exhausted; ++squarings) {
        ct = be.multiply(ct, ct, ledger);
        want = want * want % kT;
        const int b = be.measured_noise_budget(ct);
        std::printf("measured after %d squarings %d\n", squarings + 1, b);
        if (b > 0) {
            CHECK(be.decrypt(ct, ledger)[0] == want);
            CHECK(b < last_budget);
            last_budget = b;
        } else {
            CHECK_THROWS_AS(be.decrypt(ct, ledger), NoiseExhaustedError);
            exhausted = true;
        }
    }
    CHECK(exhausted);
    CHECK(ct.noise_budget_bits == 146);  // the model alone would not have caught it

    Ciphertext garbage = be.zero_ciphertext();
    std::uint64_t n = 0, slots = 0, ctw = 0, kw = 0;
    int dnum = 0;
    check_status(spmvgpu_ctx_sizes(be.context(), &n, &slots, &ctw, &kw, &dnum));
    std::vector<std::uint64_t> primes(64);
    int np = 0;
    check_status(spmvgpu_ctx_primes(be.context(), primes.data(), 64, &np));
    std::vector<std::uint64_t> w(ctw);
    std::mt19937_64 rng(99);
    const std::size_t L = ctw / (2 * n);
    for (std::size_t i = 0; i < ctw; ++i) w[i] = rng() % primes[(i / n) % L];
    check_status(spmvgpu_ct_upload(be.context(), be.handle(garbage), w.data()));
    CHECK_THROWS_AS(be.decrypt(garbage, ledger), NoiseExhaustedError);
}

// test_he.cpp:134-207
static void op_cases() {
    GpuBfvBackend be(params(), seeded(6));
    OpLedger ledger;
    const std::int64_t xs[] = {1, 2, 3, 4};
    const std::int64_t ys[] = {6, 6, 6, 6};
    Ciphertext a = be.encrypt(be.encode(xs), ledger);
    Ciphertext b = be.encrypt(be.encode(ys), ledger);
    CHECK(be.decrypt(be.add(a, b, ledger), ledger) == padded({7, 8, 9, 10}));
    CHECK(be.decrypt(be.multiply(a, b, ledger), ledger) == padded({6, 12, 18, 24}));
    CHECK(be.decrypt(be.multiply_plain(a, be.encode(ys), ledger), ledger) == padded({6, 12, 18, 24}));
    CHECK(ledger.n_add == 1 && ledger.n_mult_cc == 1 && ledger.n_mult_cp == 1);

    // rotation is cyclic to the left over the S slots, negative goes right
    OpLedger rl;
    Ciphertext ct = be.encrypt(be.encode(xs), rl);
    SlotVector left(kS, 0), right(kS, 0);
    for (std::size_t i = 0; i < 4; ++i) {
        left[(i + kS - 1) % kS] = static_cast<std::uint64_t>(xs[i]);
        right[(i + 1) % kS] = static_cast<std::uint64_t>(xs[i]);
    }
    CHECK(be.decrypt(be.rotate(ct, 1, rl), rl) == left);
    CHECK(be.decrypt(be.rotate(ct, -1, rl), rl) == right);
    CHECK(be.decrypt(be.rotate(ct, 0, rl), rl) == padded({1, 2, 3, 4}));
    CHECK(be.decrypt(be.rotate(ct, kS, rl), rl) == padded({1, 2, 3, 4}));
    CHECK(be.decrypt(be.rotate(ct, kS + 1, rl), rl) == left);
    Ciphertext back = be.rotate(be.rotate(ct, 3, rl), kS - 3, rl);
    CHECK(be.decrypt(back, rl) == padded({1, 2, 3, 4}));
    CHECK(rl.n_rot == 7);

    // adds and rotations do not consume the model budget
    const std::int64_t one_two[] = {1, 2};
    Ciphertext acc = be.encrypt(be.encode(one_two), ledger);
    for (int i = 0; i < 50; ++i) acc = be.add(be.rotate(acc, 1, ledger), acc, ledger);
    CHECK(acc.noise_budget_bits == 146);

    // the ledger counts every call and resets explicitly
    OpLedger l2;
    const std::int64_t x1[] = {1};
    Ciphertext p = be.encrypt(be.encode(x1), l2);
    Ciphertext q = be.encrypt(be.encode(x1), l2);
    be.add(p, q, l2);
    be.multiply(p, q, l2);
    be.multiply_plain(p, be.encode(x1), l2);
    be.rotate(p, 2, l2);
    be.decrypt(p, l2);
    CHECK((l2 == OpLedger{1, 1, 1, 1, 2, 1}));
    print_ledger("op_calls", l2);
    l2.reset();
    CHECK(l2 == OpLedger{});

    // the zero ciphertext is a neutral accumulator and not ledgered
    OpLedger l3;
    Ciphertext zero = be.zero_ciphertext();
    CHECK(l3.n_enc == 0);
    const std::int64_t z4[] = {9, 8, 7, 6};
    Ciphertext c4 = be.encrypt(be.encode(z4), l3);
    CHECK(be.decrypt(be.add(zero, c4, l3), l3) == padded({9, 8, 7, 6}));
}

// aggregate.cpp:36-74 op by op over the GPU backend; the ciphertext words go
// to the oracle comparison.  Encryption stream ids of this context: 1, 2, ...
static void aggregate_cases() {
    GpuBfvBackend be(params(), seeded(11));
    OpLedger ledger;
    // chunk 0: r = 3, c = 5; chunk 1: r = 7, c = 2 (flat column-major blocks)
    const std::size_t r0 = 3, c0 = 5, r1 = 7, c1 = 2;
    std::vector<std::int64_t> a0(r0 * c0), b0(r0 * c0), a1(r1 * c1), b1(r1 * c1);
    for (std::size_t i = 0; i < a0.size(); ++i) a0[i] = (std::int64_t)(i % 17) - 8, b0[i] = (std::int64_t)(i % 13) - 6;
    for (std::size_t i = 0; i < a1.size(); ++i) a1[i] = (std::int64_t)(i % 11) - 5, b1[i] = (std::int64_t)(i % 7) - 3;
    Ciphertext ca0 = be.encrypt(be.encode(a0), ledger);  // stream 1
    Ciphertext cb0 = be.encrypt(be.encode(b0), ledger);  // stream 2
    Ciphertext ca1 = be.encrypt(be.encode(a1), ledger);  // stream 3
    Ciphertext cb1 = be.encrypt(be.encode(b1), ledger);  // stream 4
    Ciphertext p0 = be.multiply(ca0, cb0, ledger);
    Ciphertext p1 = be.multiply(ca1, cb1, ledger);
    Ciphertext s0 = intra_chunk_sum(be, p0, r0, c0, ledger);
    Ciphertext s1 = intra_chunk_sum(be, p1, r1, c1, ledger);
    const Ciphertext parts[] = {s0, s1};
    const std::size_t rl[] = {r0, r1};
    Ciphertext res = inter_chunk_sum(be, parts, rl, ledger);
    dump_words(be, "agg_a0", ca0);
    dump_words(be, "agg_p0", p0);
    dump_words(be, "agg_s0", s0);
    dump_words(be, "agg_s1", s1);
    dump_words(be, "agg_res", res);
    const SlotVector out = be.decrypt(res, ledger);
    print_ledger("aggregate", ledger);
    print_slots("aggregate", out, 16);
    // block sums (test_util.hpp:44-53): row i of a chunk = sum over its columns
    SlotVector want(kS, 0);
    for (std::size_t i = 0; i < r0; ++i) {
        std::int64_t acc = 0;
        for (std::size_t k = 0; k < c0; ++k) acc += a0[k * r0 + i] * b0[k * r0 + i];
        want[i] = to_residue(acc, kT);
    }
    for (std::size_t i = 0; i < r1; ++i) {
        std::int64_t acc = 0;
        for (std::size_t k = 0; k < c1; ++k) acc += a1[k * r1 + i] * b1[k * r1 + i];
        want[i] = (want[i] + to_residue(acc, kT)) % kT;
    }
    CHECK(out == want);
    CHECK(res.noise_budget_bits == 87);
}

// the protocol front door from C++ (protocol.hpp:62-71) on the same backend type
static void protocol_cases() {
    GpuBfvBackend be(params(), seeded(12));
    CsrMatrix m;
    m.rows = 5;
    m.cols = 4;
    m.row_ptrs = {0, 2, 2, 5, 6, 7};
    m.col_indices = {0, 3, 0, 1, 2, 1, 3};
    m.values = {3, -2, 1, 4, -5, 7, 8};
    const std::vector<std::int64_t> v = {2, -1, 3, 5};
    const SpmvResult r = spmv_partitioned(be, m, v, kS);
    const std::vector<std::int64_t> want = {6 - 10, 0, 2 - 4 - 15, -7, 40};
    CHECK(r.values == want);
    CHECK(r.noise_budget_remaining_bits == 87);
    CHECK(r.measured_noise_budget_bits > 0);
    print_ledger("protocol", r.op_ledger);
    const std::vector<std::int64_t> short_v = {1, 2, 3};
    CHECK_THROWS_AS(spmv_partitioned(be, m, short_v, kS), DimensionMismatchError);
}

// a Ciphertext may outlive the backend that made it (it shares the context)
static void lifetime_cases() {
    Ciphertext keep;
    {
        GpuBfvBackend be(params(), seeded(13));
        OpLedger l;
        const std::int64_t xs[] = {4, 5};
        keep = be.encrypt(be.encode(xs), l);
    }
    CHECK(keep.payload != nullptr);
    keep = Ciphertext{};  // frees the device ciphertext, then the context
    std::printf("lifetime ok\n");
}

int main(int argc, char** argv) {
    g_out = argc > 1 ? argv[1] : ".";
    try {
        encode_cases();
        budget_cases();
        measured_noise_cases();
        op_cases();
        aggregate_cases();
        protocol_cases();
        lifetime_cases();
    } catch (const std::exception& e) {
        std::fprintf(stderr, "FAIL uncaught: %s\n", e.what());
        ++failures;
    }
    std::printf("failures %d\n", failures);
    return failures;
}
