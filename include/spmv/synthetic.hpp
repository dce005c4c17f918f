// spmv/synthetic.hpp -- seeded matrix / vector generators.
// random_sparse_csr / random_vector reproduce the reference's streams
// (proj/src/synthetic.cpp:32-86) bit for bit; the rest build the BASELINE.json
// config shapes.
#pragma once

#include <cstdint>
#include <random>
#include <vector>

#include "spmv/sparse.hpp"

namespace spmv {

inline std::uint64_t bounded_draw(std::mt19937_64& rng, std::uint64_t n) { return rng() % n; }

CsrMatrix random_sparse_csr(std::size_t rows, std::size_t cols, std::size_t nnz,
                            std::uint64_t seed, std::int64_t value_min = -100,
                            std::int64_t value_max = 100);
std::vector<std::int64_t> random_vector(std::size_t length, std::uint64_t seed,
                                        std::int64_t value_min = -100,
                                        std::int64_t value_max = 100);
// like random_vector but rejects 0 (BASELINE: values in [-8,8] excluding 0)
std::vector<std::int64_t> random_nonzero_vector(std::size_t length, std::uint64_t seed,
                                                std::int64_t value_min, std::int64_t value_max);
// Zipf(exponent) row degrees rescaled to mean_degree, hub-biased columns floor(n u^3)
CsrMatrix power_law_csr(std::size_t n, double mean_degree, double exponent, std::uint64_t seed,
                        std::int64_t value_min, std::int64_t value_max);
// side^3 grid, 27-point stencil (all in-grid neighbours incl. self)
CsrMatrix stencil27_csr(std::size_t side, std::uint64_t seed, std::int64_t value_min,
                        std::int64_t value_max);

}  // namespace spmv
