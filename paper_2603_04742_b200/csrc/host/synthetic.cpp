// synthetic.cpp -- seeded generators.
// random_sparse_csr / random_vector follow the reference's draw order exactly
// (proj/src/synthetic.cpp:32-86) so C1/C2/C5 matrices are bit-identical to the
// reference's; power_law_csr and stencil27_csr build BASELINE configs 3 and 4
// (SURVEY.md 8(d)).  Only integer PRNG bits are used (no std:: distributions).
#include <algorithm>
#include <cmath>
#include <numeric>
#include <stdexcept>
#include <unordered_set>

#include "spmv/synthetic.hpp"

namespace spmv {

namespace {

std::int64_t nonzero_draw(std::mt19937_64& rng, std::int64_t lo, std::int64_t hi) {
    if (lo > hi) throw std::invalid_argument("draw_value: empty range");
    if (lo == 0 && hi == 0) throw std::invalid_argument("draw_value: range holds only zero");
    const auto span = static_cast<std::uint64_t>(hi - lo) + 1;
    for (;;) {
        const std::int64_t v = lo + static_cast<std::int64_t>(bounded_draw(rng, span));
        if (v != 0) return v;
    }
}

double unit_draw(std::mt19937_64& rng) { return static_cast<double>(rng() >> 11) * 0x1.0p-53; }

}  // namespace

CsrMatrix random_sparse_csr(std::size_t rows, std::size_t cols, std::size_t nnz, std::uint64_t seed,
                            std::int64_t value_min, std::int64_t value_max) {
    const std::size_t cells = rows * cols;
    if (nnz > cells) throw std::invalid_argument("random_sparse_csr: nnz exceeds rows * cols");
    std::mt19937_64 rng(seed);
    std::vector<std::uint64_t> cell_of;
    cell_of.reserve(nnz);
    if (2 * nnz >= cells) {
        std::vector<std::uint64_t> pool(cells);
        std::iota(pool.begin(), pool.end(), std::uint64_t{0});
        for (std::size_t i = 0; i < nnz; ++i) {
            std::swap(pool[i], pool[i + static_cast<std::size_t>(bounded_draw(rng, cells - i))]);
            cell_of.push_back(pool[i]);
        }
    } else {
        std::unordered_set<std::uint64_t> used;
        used.reserve(2 * nnz);
        while (cell_of.size() < nnz) {
            const std::uint64_t c = bounded_draw(rng, cells);
            if (used.insert(c).second) cell_of.push_back(c);
        }
    }
    CooMatrix coo;
    coo.rows = rows;
    coo.cols = cols;
    coo.entries.reserve(nnz);
    for (std::uint64_t c : cell_of)
        coo.entries.push_back({static_cast<std::size_t>(c / cols), static_cast<std::size_t>(c % cols),
                               nonzero_draw(rng, value_min, value_max)});
    return coo_to_csr(coo);
}

std::vector<std::int64_t> random_vector(std::size_t length, std::uint64_t seed, std::int64_t value_min,
                                        std::int64_t value_max) {
    if (value_min > value_max) throw std::invalid_argument("random_vector: empty range");
    std::mt19937_64 rng(seed ^ 0x9e3779b97f4a7c15ULL);
    const auto span = static_cast<std::uint64_t>(value_max - value_min) + 1;
    std::vector<std::int64_t> v(length);
    for (auto& x : v) x = value_min + static_cast<std::int64_t>(bounded_draw(rng, span));
    return v;
}

std::vector<std::int64_t> random_nonzero_vector(std::size_t length, std::uint64_t seed,
                                                std::int64_t value_min, std::int64_t value_max) {
    std::mt19937_64 rng(seed ^ 0x9e3779b97f4a7c15ULL);
    std::vector<std::int64_t> v(length);
    for (auto& x : v) x = nonzero_draw(rng, value_min, value_max);
    return v;
}

CsrMatrix power_law_csr(std::size_t n, double mean_degree, double exponent, std::uint64_t seed,
                        std::int64_t value_min, std::int64_t value_max) {
    if (n == 0) return CsrMatrix{0, 0, {}, {}, {0}};
    std::mt19937_64 rng(seed);
    // Zipf(exponent) on {1..n} by inverse CDF
    std::vector<double> cdf(n);
    double acc = 0.0;
    for (std::size_t k = 1; k <= n; ++k) cdf[k - 1] = (acc += std::pow(static_cast<double>(k), -exponent));
    for (double& c : cdf) c /= acc;
    std::vector<double> raw(n);
    double total = 0.0;
    for (std::size_t i = 0; i < n; ++i) {
        const double u = unit_draw(rng);
        raw[i] = static_cast<double>(std::lower_bound(cdf.begin(), cdf.end(), u) - cdf.begin() + 1);
        total += raw[i];
    }
    const double scale = mean_degree * static_cast<double>(n) / total;
    CsrMatrix m;
    m.rows = m.cols = n;
    m.row_ptrs.assign(n + 1, 0);
    std::vector<std::size_t> cols_row;
    std::unordered_set<std::size_t> seen;
    for (std::size_t i = 0; i < n; ++i) {
        const auto want = static_cast<std::size_t>(
            std::clamp<double>(std::llround(raw[i] * scale), 1.0, static_cast<double>(n)));
        cols_row.clear();
        seen.clear();
        while (cols_row.size() < want) {
            const double u = unit_draw(rng);
            const auto c = std::min(n - 1, static_cast<std::size_t>(static_cast<double>(n) * u * u * u));
            if (seen.insert(c).second) cols_row.push_back(c);
        }
        std::sort(cols_row.begin(), cols_row.end());
        for (std::size_t c : cols_row) {
            m.col_indices.push_back(c);
            m.values.push_back(nonzero_draw(rng, value_min, value_max));
        }
        m.row_ptrs[i + 1] = m.values.size();
    }
    return m;
}

CsrMatrix stencil27_csr(std::size_t side, std::uint64_t seed, std::int64_t value_min,
                        std::int64_t value_max) {
    std::mt19937_64 rng(seed);
    const std::size_t n = side * side * side;
    CsrMatrix m;
    m.rows = m.cols = n;
    m.row_ptrs.assign(n + 1, 0);
    auto in = [&](std::ptrdiff_t a) { return a >= 0 && a < static_cast<std::ptrdiff_t>(side); };
    for (std::size_t x = 0; x < side; ++x)
        for (std::size_t y = 0; y < side; ++y)
            for (std::size_t z = 0; z < side; ++z) {
                const std::size_t row = (x * side + y) * side + z;
                for (int dx = -1; dx <= 1; ++dx)
                    for (int dy = -1; dy <= 1; ++dy)
                        for (int dz = -1; dz <= 1; ++dz) {
                            const auto nx = static_cast<std::ptrdiff_t>(x) + dx;
                            const auto ny = static_cast<std::ptrdiff_t>(y) + dy;
                            const auto nz = static_cast<std::ptrdiff_t>(z) + dz;
                            if (!in(nx) || !in(ny) || !in(nz)) continue;
                            m.col_indices.push_back(static_cast<std::size_t>((nx * static_cast<std::ptrdiff_t>(side) + ny) *
                                                                                 static_cast<std::ptrdiff_t>(side) +
                                                                             nz));
                            m.values.push_back(nonzero_draw(rng, value_min, value_max));
                        }
                m.row_ptrs[row + 1] = m.values.size();
            }
    return m;
}

}  // namespace spmv
