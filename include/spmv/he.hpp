// spmv/he.hpp -- homomorphic-encryption backend contract.
//
// API-compatible with the reference's plugin boundary
// (proj/include/spmv/he.hpp:14-146): same value types, ledger and virtual
// interface, so protocol code written against HeBackend runs unchanged.  The
// one deliberate difference is Ciphertext::payload, which the reference
// documents as simulator-internal (he.hpp:49-50): here it is an opaque handle
// to a device-resident RNS-BFV ciphertext (see spmv/gpu_backend.hpp).
#pragma once

#include <cstdint>
#include <memory>
#include <span>
#include <vector>

#include "spmv/errors.hpp"

namespace spmv {

using SlotVector = std::vector<std::uint64_t>;

// Linear noise-budget model kept for API parity (reference he.hpp:24-30):
// each op subtracts a fixed cost, floored at zero.  The GPU backend also
// reports the measured BFV invariant-noise budget separately.
struct NoiseModel {
    int initial_budget_bits = 146;
    int cost_ct_ct_mult_bits = 33;
    int cost_ct_pt_mult_bits = 26;
    int cost_add_bits = 0;
    int cost_rot_bits = 0;
};

struct HeParams {
    std::size_t slot_count = 8192;
    std::uint64_t plaintext_modulus = 65537;
    double ciphertext_size_mb = 0.52;  // prices transcript messages only
    NoiseModel noise;

    void validate() const;  // std::invalid_argument on nonsense
};

struct Plaintext {
    SlotVector slots;
};

// Device ciphertext handle; defined by the backend that created it.
struct DeviceCiphertext;

struct Ciphertext {
    std::shared_ptr<const DeviceCiphertext> payload;
    int noise_budget_bits = 0;  // model counter
    std::uint64_t id = 0;
};

struct OpLedger {
    std::uint64_t n_mult_cc = 0;
    std::uint64_t n_mult_cp = 0;
    std::uint64_t n_rot = 0;
    std::uint64_t n_add = 0;
    std::uint64_t n_enc = 0;
    std::uint64_t n_dec = 0;

    void reset() { *this = OpLedger{}; }
    OpLedger& operator+=(const OpLedger& o) {
        n_mult_cc += o.n_mult_cc;
        n_mult_cp += o.n_mult_cp;
        n_rot += o.n_rot;
        n_add += o.n_add;
        n_enc += o.n_enc;
        n_dec += o.n_dec;
        return *this;
    }
    bool operator==(const OpLedger&) const = default;
};

class HeBackend {
public:
    virtual ~HeBackend() = default;
    virtual const HeParams& params() const = 0;
    // residues mod t, zero-padded to slot_count; OverLengthError if too long
    virtual Plaintext encode(std::span<const std::int64_t> values) const = 0;
    virtual Ciphertext encrypt(const Plaintext& pt, OpLedger& ledger) const = 0;
    // NoiseExhaustedError once the budget is gone
    virtual SlotVector decrypt(const Ciphertext& ct, OpLedger& ledger) const = 0;
    virtual Ciphertext add(const Ciphertext& a, const Ciphertext& b, OpLedger& ledger) const = 0;
    virtual Ciphertext multiply(const Ciphertext& a, const Ciphertext& b,
                                OpLedger& ledger) const = 0;
    virtual Ciphertext multiply_plain(const Ciphertext& a, const Plaintext& b,
                                      OpLedger& ledger) const = 0;
    // cyclic left rotation by k (negative = right), k taken mod slot_count
    virtual Ciphertext rotate(const Ciphertext& a, std::int64_t k, OpLedger& ledger) const = 0;
    // transparent all-zero accumulator; not an encryption, not ledgered
    virtual Ciphertext zero_ciphertext() const = 0;
};

// centred representative in [-(t-1)/2, t/2]
std::int64_t to_signed(std::uint64_t residue, std::uint64_t modulus);
std::uint64_t to_residue(std::int64_t value, std::uint64_t modulus);

}  // namespace spmv
