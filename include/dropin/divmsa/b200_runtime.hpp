// Shared plumbing of the GPU drop-in headers (include/dropin/divmsa/*.hpp):
// the process-wide libdmb200 context, status -> exception mapping and the
// per-call sequence upload. Not a reference header; the four drop-ins
// (distance.hpp, pairwise.hpp, cluster_tree.hpp, msa_merge.hpp) include it.
#pragma once

#include <cstdint>
#include <cstdlib>
#include <memory>
#include <mutex>
#include <span>
#include <stdexcept>
#include <string>
#include <string_view>
#include <vector>

#include "dm_b200.h"

namespace divmsa::b200 {

/// DM_EINVAL -> std::invalid_argument, anything else -> std::runtime_error,
/// with the library's message (which is the reference's message text).
inline void check(int rc) {
    if (rc == DM_OK) return;
    const std::string msg = dm_last_error();
    if (rc == DM_EINVAL) throw std::invalid_argument(msg);
    throw std::runtime_error(msg);
}

/// One context per process, on device DM_DEVICE (default 0), created on first
/// use. The library serialises calls on a context, so every pool thread of
/// the reference may call in concurrently.
inline dm_ctx* ctx() {
    static std::once_flag once;
    static dm_ctx* c = nullptr;
    std::call_once(once, [] {
        const char* d = std::getenv("DM_DEVICE");
        check(dm_ctx_create(d ? std::atoi(d) : 0, &c));
    });
    return c;
}

struct SeqsetDeleter {
    void operator()(dm_seqset* s) const { dm_seqset_destroy(s); }
};
using Seqset = std::unique_ptr<dm_seqset, SeqsetDeleter>;

/// Packs the views into one buffer + offsets and builds the device sequence set.
inline Seqset upload(std::span<const std::string_view> seqs) {
    std::string data;
    std::vector<std::uint64_t> off(seqs.size() + 1, 0);
    std::size_t total = 0;
    for (auto s : seqs) total += s.size();
    data.reserve(total);
    for (std::size_t i = 0; i < seqs.size(); ++i) {
        data.append(seqs[i]);
        off[i + 1] = data.size();
    }
    dm_seqset* s = nullptr;
    check(dm_seqset_create(ctx(), data.data(), off.data(), static_cast<std::uint32_t>(seqs.size()), &s));
    return Seqset(s);
}

}  // namespace divmsa::b200
