// Shared host-side helpers: error plumbing for the C ABI and a small
// deterministic parallel-for. Errors are C++ exceptions internally (the same
// types the reference throws) and become psc_status codes at the boundary.
#pragma once

#include <algorithm>
#include <atomic>
#include <cstdint>
#include <functional>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "psc_b200.h"

namespace pscb {

// CUDA or allocation failures that have no reference exception type.
struct CudaError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

void set_last_error(const std::string& msg);

template <class F>
psc_status guarded(F&& f) {
    try {
        f();
        return PSC_OK;
    } catch (const std::invalid_argument& e) {
        set_last_error(e.what());
        return PSC_ERR_INVALID_ARGUMENT;
    } catch (const std::logic_error& e) {
        set_last_error(e.what());
        return PSC_ERR_LOGIC;
    } catch (const CudaError& e) {
        set_last_error(e.what());
        return PSC_ERR_CUDA;
    } catch (const std::bad_alloc&) {
        set_last_error("out of host memory");
        return PSC_ERR_NOMEM;
    } catch (const std::exception& e) {
        set_last_error(e.what());
        return PSC_ERR_INTERNAL;
    }
}

inline void require(bool ok, const std::string& what) {
    if (!ok) throw std::invalid_argument(what);
}

inline int hw_threads(int requested) {
    if (requested > 0) return requested;
    unsigned hw = std::thread::hardware_concurrency();
    return hw == 0 ? 1 : static_cast<int>(hw);
}

// Runs fn(task) for task in [0, n_tasks) on up to `threads` threads with
// dynamic claiming. Callers write results into per-task slots, so output
// never depends on the thread count.
inline void parallel_for(int64_t n_tasks, int threads, const std::function<void(int64_t)>& fn) {
    threads = static_cast<int>(std::min<int64_t>(std::max(1, threads), std::max<int64_t>(1, n_tasks)));
    if (threads <= 1) {
        for (int64_t i = 0; i < n_tasks; ++i) fn(i);
        return;
    }
    std::atomic<int64_t> next{0};
    std::exception_ptr err;
    std::atomic<bool> failed{false};
    auto body = [&] {
        while (!failed.load(std::memory_order_relaxed)) {
            int64_t i = next.fetch_add(1, std::memory_order_relaxed);
            if (i >= n_tasks) break;
            try {
                fn(i);
            } catch (...) {
                if (!failed.exchange(true)) err = std::current_exception();
            }
        }
    };
    std::vector<std::thread> pool;
    pool.reserve(threads - 1);
    for (int t = 1; t < threads; ++t) pool.emplace_back(body);
    body();
    for (auto& th : pool) th.join();
    if (err) std::rethrow_exception(err);
}

}  // namespace pscb
