// he.cpp -- HeParams validation and residue helpers (reference he.cpp:23-56).
#include "spmv/he.hpp"

#include <stdexcept>

namespace spmv {

void HeParams::validate() const {
    if (slot_count == 0) throw std::invalid_argument("slot_count must be positive");
    if (plaintext_modulus < 2) throw std::invalid_argument("plaintext_modulus must be at least 2");
    if (!(ciphertext_size_mb > 0.0)) throw std::invalid_argument("ciphertext_size_mb must be positive");
    if (noise.initial_budget_bits <= 0)
        throw std::invalid_argument("initial noise budget must be positive");
    if (noise.cost_ct_ct_mult_bits < 0 || noise.cost_ct_pt_mult_bits < 0 || noise.cost_add_bits < 0 ||
        noise.cost_rot_bits < 0)
        throw std::invalid_argument("noise costs must be non-negative");
}

std::int64_t to_signed(std::uint64_t residue, std::uint64_t modulus) {
    const auto r = static_cast<std::int64_t>(residue);
    return residue <= modulus / 2 ? r : r - static_cast<std::int64_t>(modulus);
}

std::uint64_t to_residue(std::int64_t value, std::uint64_t modulus) {
    const auto m = static_cast<std::int64_t>(modulus);
    const std::int64_t r = value % m;
    return static_cast<std::uint64_t>(r < 0 ? r + m : r);
}

}  // namespace spmv
