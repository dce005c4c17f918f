// host_pool.hpp -- a small process-wide worker pool for the client-side host
// passes of large batches (CSR validation, the pinned upload image).  The
// caller participates; one run at a time; the first exception is rethrown in
// the caller.  Small inputs should not use it (a run costs a few µs).
#pragma once

#include <atomic>
#include <condition_variable>
#include <cstddef>
#include <exception>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

namespace spmv::detail {

class HostPool {
public:
    static HostPool& get();
    // fn(i) for every i in [0, n), spread over the workers and the caller
    void run(std::size_t n, const std::function<void(std::size_t)>& fn);
    std::size_t threads() const { return workers_.size() + 1; }

private:
    explicit HostPool(unsigned workers);
    void loop();
    void drain();

    std::vector<std::thread> workers_;
    std::mutex run_mu_;  // one run at a time
    std::mutex mu_;
    std::condition_variable cv_, done_cv_;
    const std::function<void(std::size_t)>* fn_ = nullptr;
    std::size_t n_ = 0;
    std::atomic<std::size_t> next_{0};
    std::size_t active_ = 0;
    unsigned gen_ = 0;
    std::exception_ptr err_;
};

}  // namespace spmv::detail
