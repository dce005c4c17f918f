// cost.cpp -- see spmv/cost.hpp (reference proj/src/cost.cpp:8-28).
#include "spmv/cost.hpp"

namespace spmv {

namespace {
double d(std::uint64_t x) { return static_cast<double>(x); }
}  // namespace

double estimate_cloud_time_ms(const OpLedger& l, const CostTable& c) {
    return d(l.n_mult_cc) * c.mult_cc_ms + d(l.n_mult_cp) * c.mult_cp_ms + d(l.n_rot) * c.rot_ms +
           d(l.n_add) * c.add_ms;
}

double estimate_time_ms(const OpLedger& l, const CostTable& c) {
    return estimate_cloud_time_ms(l, c) + d(l.n_enc) * c.enc_ms + d(l.n_dec) * c.dec_ms;
}

double estimate_memory_mb(const OpLedger& l, const HeParams& p) {
    return d(l.n_enc + l.n_add + l.n_mult_cc + l.n_mult_cp + l.n_rot) * p.ciphertext_size_mb;
}

}  // namespace spmv
