// gpu_backend.cpp -- HeBackend adapter over the spmvgpu_* C-ABI.
// Virtual-for-virtual replacement of the reference SimBackend
// (proj/src/he.cpp:58-153): same ledger increments, same model-noise
// arithmetic, same exceptions; the payload is a device RNS-BFV ciphertext.
#include <atomic>
#include <bit>
#include <stdexcept>
#include <string>

#include "spmv/gpu_backend.hpp"

namespace spmv {

struct DeviceCiphertext {
    std::shared_ptr<spmvgpu_ctx> ctx;  // keeps the context alive while this ciphertext exists
    spmvgpu_ct h = 0;
    ~DeviceCiphertext() {
        if (ctx && h) spmvgpu_ct_free(ctx.get(), &h, 1);
    }
};

[[noreturn]] void throw_status(int status) {
    const std::string msg = spmvgpu_last_error();
    switch (status) {
        case SPMVGPU_ERR_INVALID_ARGUMENT: throw std::invalid_argument(msg);
        case SPMVGPU_ERR_OVER_LENGTH: throw OverLengthError(msg);
        case SPMVGPU_ERR_NOISE_EXHAUSTED: throw NoiseExhaustedError(msg);
        case SPMVGPU_ERR_DIMENSION: throw DimensionMismatchError(msg);
        case SPMVGPU_ERR_COLUMN_TOO_TALL: throw ColumnTooTallError(msg);
        case SPMVGPU_ERR_INDEX_RANGE: throw IndexOutOfRangeError(msg);
        case SPMVGPU_ERR_DUPLICATE: throw DuplicateEntryError(msg);
        case SPMVGPU_ERR_NON_SQUARE: throw NonSquareError(msg);
        default: throw std::runtime_error("spmvgpu: " + msg);
    }
}

namespace {
int lowered(int b, int c) { return b - c > 0 ? b - c : 0; }
}  // namespace

GpuBfvBackend::GpuBfvBackend(HeParams params, GpuBfvOptions opt) : params_(params) {
    params_.validate();
    int logn = opt.logn;
    if (logn == 0) {
        if (!std::has_single_bit(params_.slot_count))
            throw std::invalid_argument("GpuBfvBackend: slot_count must be a power of two (one BFV row of N/2 slots)");
        logn = std::bit_width(params_.slot_count);  // N = 2 * slot_count
    }
    spmvgpu_params p;
    spmvgpu_default_params(logn, &p);
    if (opt.L) p.L = opt.L;
    if (opt.K) p.K = opt.K;
    if (opt.alpha) p.alpha = opt.alpha;
    if (opt.qbits) p.qbits = opt.qbits;
    if (opt.pbits) p.pbits = opt.pbits;
    p.t = params_.plaintext_modulus;
    p.seed = opt.seed;
    p.device = opt.device;
    p.ciphertext_size_mb = params_.ciphertext_size_mb;
    p.noise_initial = params_.noise.initial_budget_bits;
    p.noise_ct_ct = params_.noise.cost_ct_ct_mult_bits;
    p.noise_ct_pt = params_.noise.cost_ct_pt_mult_bits;
    p.noise_add = params_.noise.cost_add_bits;
    p.noise_rot = params_.noise.cost_rot_bits;
    if ((std::size_t{1} << (logn - 1)) != params_.slot_count)
        throw std::invalid_argument("GpuBfvBackend: slot_count must equal N/2");
    spmvgpu_ctx* raw = nullptr;
    check_status(spmvgpu_ctx_create(&p, &raw));
    ctx_ = std::shared_ptr<spmvgpu_ctx>(raw, [](spmvgpu_ctx* c) { spmvgpu_ctx_destroy(c); });
}

// a view: the caller owns the context and keeps it alive
GpuBfvBackend::GpuBfvBackend(HeParams params, spmvgpu_ctx* ctx)
    : params_(params), ctx_(ctx, [](spmvgpu_ctx*) {}) {
    params_.validate();
}

GpuBfvBackend::~GpuBfvBackend() = default;

std::shared_ptr<DeviceCiphertext> GpuBfvBackend::fresh() const {
    auto d = std::make_shared<DeviceCiphertext>();
    check_status(spmvgpu_ct_alloc(ctx_.get(), 1, &d->h));
    d->ctx = ctx_;
    return d;
}

Ciphertext GpuBfvBackend::wrap(std::shared_ptr<DeviceCiphertext> d, int budget) const {
    static std::atomic<std::uint64_t> next_id{1};
    return Ciphertext{std::move(d), budget, next_id.fetch_add(1)};
}

spmvgpu_ct GpuBfvBackend::handle(const Ciphertext& ct) const {
    if (!ct.payload) throw std::invalid_argument("GpuBfvBackend: empty ciphertext");
    return ct.payload->h;
}

Plaintext GpuBfvBackend::encode(std::span<const std::int64_t> values) const {
    if (values.size() > params_.slot_count)
        throw OverLengthError("encode: " + std::to_string(values.size()) + " values exceed " +
                              std::to_string(params_.slot_count) + " slots");
    Plaintext pt;
    pt.slots.assign(params_.slot_count, 0);
    for (std::size_t i = 0; i < values.size(); ++i) pt.slots[i] = to_residue(values[i], params_.plaintext_modulus);
    return pt;
}

Ciphertext GpuBfvBackend::encrypt(const Plaintext& pt, OpLedger& ledger) const {
    if (pt.slots.size() != params_.slot_count)
        throw DimensionMismatchError("encrypt: plaintext slot count does not match parameters");
    std::vector<std::int64_t> vals(pt.slots.begin(), pt.slots.end());
    const std::uint64_t offs[2] = {0, vals.size()};
    auto out = fresh();
    check_status(spmvgpu_encrypt(ctx_.get(), vals.data(), offs, nullptr, &out->h, 1));
    ledger.n_enc += 1;
    return wrap(std::move(out), params_.noise.initial_budget_bits);
}

SlotVector GpuBfvBackend::decrypt(const Ciphertext& ct, OpLedger& ledger) const {
    if (ct.noise_budget_bits <= 0)
        throw NoiseExhaustedError("decrypt: noise budget exhausted (ciphertext id " + std::to_string(ct.id) + ")");
    SlotVector slots(params_.slot_count);
    const spmvgpu_ct h = handle(ct);
    std::int32_t measured = 0;
    check_status(spmvgpu_decrypt(ctx_.get(), &h, 1, slots.data(), &measured));
    // the real BFV check behind the model counter: no invariant-noise
    // budget left means the slots below are not the plaintext
    if (measured <= 0)
        throw NoiseExhaustedError("decrypt: measured invariant-noise budget exhausted (ciphertext id " +
                                  std::to_string(ct.id) + ")");
    ledger.n_dec += 1;
    return slots;
}

int GpuBfvBackend::measured_noise_budget(const Ciphertext& ct) const {
    SlotVector slots(params_.slot_count);
    const spmvgpu_ct h = handle(ct);
    std::int32_t measured = 0;
    check_status(spmvgpu_decrypt(ctx_.get(), &h, 1, slots.data(), &measured));
    return measured;
}

Ciphertext GpuBfvBackend::add(const Ciphertext& a, const Ciphertext& b, OpLedger& ledger) const {
    const spmvgpu_ct x = handle(a), y = handle(b);
    auto o = fresh();
    check_status(spmvgpu_add(ctx_.get(), &x, &y, &o->h, 1));
    ledger.n_add += 1;
    return wrap(std::move(o), lowered(std::min(a.noise_budget_bits, b.noise_budget_bits), params_.noise.cost_add_bits));
}

Ciphertext GpuBfvBackend::multiply(const Ciphertext& a, const Ciphertext& b, OpLedger& ledger) const {
    const spmvgpu_ct x = handle(a), y = handle(b);
    auto o = fresh();
    check_status(spmvgpu_mul_relin(ctx_.get(), &x, &y, &o->h, 1));
    ledger.n_mult_cc += 1;
    return wrap(std::move(o), lowered(std::min(a.noise_budget_bits, b.noise_budget_bits), params_.noise.cost_ct_ct_mult_bits));
}

Ciphertext GpuBfvBackend::multiply_plain(const Ciphertext& a, const Plaintext& b, OpLedger& ledger) const {
    if (b.slots.size() != params_.slot_count) throw DimensionMismatchError("multiply_plain: slot counts differ");
    std::vector<std::int64_t> vals(b.slots.begin(), b.slots.end());
    const std::uint64_t offs[2] = {0, vals.size()};
    const spmvgpu_ct x = handle(a);
    auto o = fresh();
    check_status(spmvgpu_mul_plain(ctx_.get(), &x, vals.data(), offs, &o->h, 1));
    ledger.n_mult_cp += 1;
    return wrap(std::move(o), lowered(a.noise_budget_bits, params_.noise.cost_ct_pt_mult_bits));
}

Ciphertext GpuBfvBackend::rotate(const Ciphertext& a, std::int64_t k, OpLedger& ledger) const {
    const spmvgpu_ct x = handle(a);
    auto o = fresh();
    check_status(spmvgpu_rotate(ctx_.get(), &x, &k, &o->h, 1));
    ledger.n_rot += 1;
    return wrap(std::move(o), lowered(a.noise_budget_bits, params_.noise.cost_rot_bits));
}

Ciphertext GpuBfvBackend::zero_ciphertext() const {
    std::uint64_t n = 0, slots = 0, ctw = 0, kw = 0;
    int dnum = 0;
    check_status(spmvgpu_ctx_sizes(ctx_.get(), &n, &slots, &ctw, &kw, &dnum));
    const std::vector<std::uint64_t> zeros(ctw, 0);
    auto o = fresh();
    check_status(spmvgpu_ct_upload(ctx_.get(), o->h, zeros.data()));
    return wrap(std::move(o), params_.noise.initial_budget_bits);
}

}  // namespace spmv
