// host_pool.cpp -- see host_pool.hpp.
#include "host/host_pool.hpp"

#include <algorithm>
#include <cstdlib>

namespace spmv::detail {

HostPool& HostPool::get() {
    // never destroyed: idle workers simply end with the process
    static HostPool* pool = [] {
        unsigned w = std::min(15u, std::max(1u, std::thread::hardware_concurrency()) - 1);
        if (const char* e = std::getenv("CSSC_HOST_THREADS")) w = static_cast<unsigned>(std::max(1, std::atoi(e)) - 1);
        return new HostPool(w);
    }();
    return *pool;
}

HostPool::HostPool(unsigned workers) {
    for (unsigned i = 0; i < workers; ++i) workers_.emplace_back([this] { loop(); });
    for (auto& t : workers_) t.detach();
}

void HostPool::drain() {
    for (std::size_t i; (i = next_.fetch_add(1)) < n_;) {
        try {
            (*fn_)(i);
        } catch (...) {
            std::lock_guard<std::mutex> g(mu_);
            if (!err_) err_ = std::current_exception();
        }
    }
}

void HostPool::loop() {
    unsigned seen = 0;
    for (;;) {
        {
            std::unique_lock<std::mutex> lk(mu_);
            cv_.wait(lk, [&] { return gen_ != seen; });
            seen = gen_;
        }
        drain();
        std::lock_guard<std::mutex> g(mu_);
        if (--active_ == 0) done_cv_.notify_one();
    }
}

void HostPool::run(std::size_t n, const std::function<void(std::size_t)>& fn) {
    if (n == 0) return;
    std::lock_guard<std::mutex> one(run_mu_);
    if (workers_.empty() || n == 1) {
        for (std::size_t i = 0; i < n; ++i) fn(i);
        return;
    }
    {
        std::lock_guard<std::mutex> g(mu_);
        fn_ = &fn;
        n_ = n;
        next_.store(0);
        active_ = workers_.size();
        err_ = nullptr;
        ++gen_;
    }
    cv_.notify_all();
    drain();
    std::unique_lock<std::mutex> lk(mu_);
    done_cv_.wait(lk, [&] { return active_ == 0; });
    fn_ = nullptr;
    if (err_) std::rethrow_exception(err_);
}

}  // namespace spmv::detail
