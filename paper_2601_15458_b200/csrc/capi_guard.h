// Exception -> status-code mapping shared by the C ABI translation units.
#pragma once

#include <new>
#include <utility>
#include <string>

#include "dm_internal.h"

namespace dm {

std::string& last_error();  // thread-local, defined in capi.cpp

template <class F>
int guard(F&& f) {
    try {
        f();
        return DM_OK;
    } catch (const invalid_argument& e) {
        last_error() = e.what();
        return DM_EINVAL;
    } catch (const cuda_error& e) {
        last_error() = e.what();
        return DM_ECUDA;
    } catch (const std::bad_alloc&) {
        last_error() = "out of memory";
        return DM_ENOMEM;
    } catch (const std::exception& e) {
        last_error() = e.what();
        return DM_ERUNTIME;
    }
}

// guard() holding the context's lock (null ctx: no lock; the body reports it),
// with the context's device current on this host thread (a process may hold
// contexts on several GPUs, and the calling thread's current device is the
// caller's business).
template <class F>
int guard(dm_ctx* ctx, F&& f) {
    if (!ctx) return guard(std::forward<F>(f));
    std::lock_guard<std::recursive_mutex> lk(ctx->mu);
    return guard([&] {
        DM_CUDA(cudaSetDevice(ctx->device));
        f();
    });
}

inline void require(bool ok, const char* msg) {
    if (!ok) throw invalid_argument(msg);
}

}  // namespace dm
