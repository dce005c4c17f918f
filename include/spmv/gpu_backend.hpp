// spmv/gpu_backend.hpp -- HeBackend over the B200 RNS-BFV device path.
//
// Drop-in for the reference's SimBackend (proj/include/spmv/he.hpp:119-139):
// same virtual interface, same ledger and model-noise semantics, but every
// ciphertext is a real RNS-BFV ciphertext resident in HBM and every operation
// runs as sm_100a kernels through the C-ABI in spmvgpu.h.  slot_count must be
// N/2 (one BFV row).  spmv()/spmv_partitioned() detect this
// backend and run the batched cloud plan instead of op-by-op calls.
#pragma once

#include <cstdint>
#include <memory>

#include "spmv/he.hpp"
#include "spmvgpu.h"

namespace spmv {

struct GpuBfvOptions {
    int logn = 0;        // 0: derive from slot_count (N = 2 * slot_count)
    int L = 0, K = 0, alpha = 0, qbits = 0, pbits = 0;  // 0: defaults for N
    std::uint64_t seed = 0;  // 0: 256-bit key from OS entropy; nonzero: deterministic (tests)
    int device = 0;
};

class GpuBfvBackend final : public HeBackend {
public:
    explicit GpuBfvBackend(HeParams params, GpuBfvOptions opt = {});
    // non-owning view over an existing context (used by the C-ABI front door)
    GpuBfvBackend(HeParams params, spmvgpu_ctx* ctx);
    ~GpuBfvBackend() override;

    const HeParams& params() const override { return params_; }
    Plaintext encode(std::span<const std::int64_t> values) const override;
    Ciphertext encrypt(const Plaintext& pt, OpLedger& ledger) const override;
    SlotVector decrypt(const Ciphertext& ct, OpLedger& ledger) const override;
    Ciphertext add(const Ciphertext& a, const Ciphertext& b, OpLedger& ledger) const override;
    Ciphertext multiply(const Ciphertext& a, const Ciphertext& b, OpLedger& ledger) const override;
    Ciphertext multiply_plain(const Ciphertext& a, const Plaintext& b,
                              OpLedger& ledger) const override;
    Ciphertext rotate(const Ciphertext& a, std::int64_t k, OpLedger& ledger) const override;
    Ciphertext zero_ciphertext() const override;

    // measured invariant-noise budget of a ciphertext (decrypts it)
    int measured_noise_budget(const Ciphertext& ct) const;
    spmvgpu_ctx* context() const { return ctx_.get(); }
    spmvgpu_ct handle(const Ciphertext& ct) const;

private:
    // a fresh device ciphertext, owned (freed on every exit path) before the
    // operation that fills it runs
    std::shared_ptr<DeviceCiphertext> fresh() const;
    Ciphertext wrap(std::shared_ptr<DeviceCiphertext> d, int budget) const;
    HeParams params_;
    // shared with every DeviceCiphertext this backend creates: an owned
    // context lives until the backend and its last ciphertext are gone
    std::shared_ptr<spmvgpu_ctx> ctx_;
};

// map a C-ABI status to the reference exception types
[[noreturn]] void throw_status(int status);
inline void check_status(int status) {
    if (status != SPMVGPU_OK) throw_status(status);
}

}  // namespace spmv
