// spmv/aggregate.hpp -- rotate-and-add folding and masked stacking.
// API-compatible with the reference (proj/include/spmv/aggregate.hpp:14-54).
#pragma once

#include <cstdint>
#include <span>
#include <vector>

#include "spmv/he.hpp"

namespace spmv {

int num_bits(std::size_t c);

struct RotStep {
    std::size_t offset = 0;
    bool from_accumulator = true;  // else: rotate the untouched product
    bool operator==(const RotStep&) const = default;
};

// numBits(cols) + popcount(cols) - 2 steps, offsets multiples of rows
std::vector<RotStep> rotation_schedule(std::size_t rows, std::size_t cols);

Ciphertext intra_chunk_sum(const HeBackend& be, const Ciphertext& ct, std::size_t rows,
                           std::size_t cols, OpLedger& ledger);

struct MaskSpec {
    std::size_t ones_len = 0;
};

Plaintext mask_plaintext(const HeBackend& be, const MaskSpec& spec);

Ciphertext inter_chunk_sum(const HeBackend& be, std::span<const Ciphertext> parts,
                           std::span<const std::size_t> r_list, OpLedger& ledger);

}  // namespace spmv
