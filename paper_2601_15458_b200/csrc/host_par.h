// Host-side data parallelism for the per-item host work around the kernels
// (input validation, result assembly): static chunks on the persistent host
// pool (host_pack.h), 4 per pool thread. Exceptions from a chunk are
// rethrown on the calling thread (the first one wins), as
// divmsa::parallel_for does (parallel.cpp:111-139).
#pragma once

#include <algorithm>
#include <cstdint>
#include <exception>
#include <mutex>
#include <thread>
#include <vector>

#include "host_pack.h"

namespace dm {

template <class F>
void host_parallel_for(uint64_t n, uint64_t min_chunk, F&& f) {
    const uint64_t hw = std::max(1u, host_pool_threads());
    const uint64_t nt = std::min<uint64_t>(hw * 4, (n + min_chunk - 1) / std::max<uint64_t>(min_chunk, 1));
    if (nt <= 1) {
        for (uint64_t i = 0; i < n; ++i) f(i);
        return;
    }
    // static chunks on the persistent host pool (no thread start-up per call)
    std::exception_ptr err;
    std::mutex mu;
    host_pool_run(nt, [&](uint64_t t) {
        const uint64_t lo = n * t / nt, hi = n * (t + 1) / nt;
        try {
            for (uint64_t i = lo; i < hi; ++i) f(i);
        } catch (...) {
            std::lock_guard<std::mutex> g(mu);
            if (!err) err = std::current_exception();
        }
    });
    if (err) std::rethrow_exception(err);
}

}  // namespace dm
