// 2-bit packing of nucleotide chunks for the streamed upload (host_pack.h).
#include "host_pack.h"

#include <immintrin.h>

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <thread>
#include <vector>

namespace dm {
namespace {

// Persistent workers woken per run(); tasks are claimed from an atomic
// counter, so uneven tasks balance themselves.
class HostPool {
public:
    HostPool() {
        unsigned hw = std::max(1u, std::thread::hardware_concurrency());
        if (const char* env = std::getenv("DM_HOST_THREADS")) hw = std::max(1, std::atoi(env));
        nthreads_ = hw;
        for (unsigned t = 1; t < hw; ++t) workers_.emplace_back([this] { loop(); });
    }
    ~HostPool() {
        {
            std::lock_guard<std::mutex> g(mu_);
            stop_ = true;
        }
        cv_.notify_all();
        for (auto& w : workers_) w.join();
    }
    unsigned threads() const { return nthreads_; }

    void run(uint64_t ntasks, const std::function<void(uint64_t)>& f) {
        if (ntasks == 0) return;
        std::lock_guard<std::mutex> serial(run_mu_);
        if (workers_.empty() || ntasks == 1) {
            for (uint64_t i = 0; i < ntasks; ++i) f(i);
            return;
        }
        {
            std::lock_guard<std::mutex> g(mu_);
            f_ = &f;
            ntasks_ = ntasks;
            next_.store(0);
            pending_ = (unsigned)workers_.size();
            ++gen_;
        }
        cv_.notify_all();
        work();
        std::unique_lock<std::mutex> g(mu_);
        done_cv_.wait(g, [this] { return pending_ == 0; });
        f_ = nullptr;
    }

private:
    void work() {
        for (uint64_t i; (i = next_.fetch_add(1)) < ntasks_;) (*f_)(i);
    }
    void loop() {
        uint64_t seen = 0;
        for (;;) {
            {
                std::unique_lock<std::mutex> g(mu_);
                cv_.wait(g, [&] { return stop_ || gen_ != seen; });
                if (stop_) return;
                seen = gen_;
            }
            work();
            std::lock_guard<std::mutex> g(mu_);
            if (--pending_ == 0) done_cv_.notify_one();
        }
    }

    unsigned nthreads_ = 1;
    std::vector<std::thread> workers_;
    std::mutex mu_, run_mu_;
    std::condition_variable cv_, done_cv_;
    const std::function<void(uint64_t)>* f_ = nullptr;
    uint64_t ntasks_ = 0, gen_ = 0;
    std::atomic<uint64_t> next_{0};
    unsigned pending_ = 0;
    bool stop_ = false;
};

HostPool& pool() {
    static HostPool p;
    return p;
}

// code = ((c >> 1) ^ (c >> 2)) & 3 maps A C G T (0x41 0x43 0x47 0x54) to
// 0 1 2 3; a byte is valid iff "ACGT"[code] gives it back.
inline bool pack_scalar(const uint8_t* s, uint64_t n, uint8_t* d) {
    static const uint8_t back[4] = {'A', 'C', 'G', 'T'};
    for (uint64_t i = 0; i < n; i += 4) {
        uint8_t v = 0;
        for (uint64_t k = 0; k < 4 && i + k < n; ++k) {
            const uint8_t c = s[i + k];
            const uint8_t code = ((c >> 1) ^ (c >> 2)) & 3;
            if (back[code] != c) return false;
            v |= (uint8_t)(code << (2 * k));
        }
        d[i / 4] = v;
    }
    return true;
}

// 128 residues -> 32 bytes: per 32-residue vector, codes by shift/xor,
// validity by PSHUFB lookup, 4 codes per byte by two multiply-adds; four
// vectors are narrowed with PACKUS and put back in order by one lane
// permute. Streaming store when the caller's destination allows it (the copy
// engine reads the bytes next, not this core).
__attribute__((target("avx2"))) inline bool block128_avx2(const uint8_t* s, uint8_t* d, bool stream) {
    const __m256i three = _mm256_set1_epi8(3);
    const __m256i lut = _mm256_setr_epi8('A', 'C', 'G', 'T', 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0,
                                         'A', 'C', 'G', 'T', 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0);
    const __m256i w14 = _mm256_set1_epi16(0x0401);       // k0 + 4 k1
    const __m256i w116 = _mm256_set1_epi32(0x00100001);  // p0 + 16 p1
    const __m256i order = _mm256_setr_epi32(0, 4, 1, 5, 2, 6, 3, 7);
    __m256i bad = _mm256_setzero_si256(), p[4];
#pragma GCC unroll 4
    for (int u = 0; u < 4; ++u) {
        const __m256i x = _mm256_loadu_si256((const __m256i*)(s + 32 * u));
        const __m256i k = _mm256_and_si256(_mm256_xor_si256(_mm256_srli_epi16(x, 1), _mm256_srli_epi16(x, 2)), three);
        bad = _mm256_or_si256(bad, _mm256_xor_si256(_mm256_shuffle_epi8(lut, k), x));
        p[u] = _mm256_madd_epi16(_mm256_maddubs_epi16(k, w14), w116);  // one byte per dword
    }
    const __m256i q = _mm256_packus_epi16(_mm256_packus_epi32(p[0], p[1]), _mm256_packus_epi32(p[2], p[3]));
    const __m256i r = _mm256_permutevar8x32_epi32(q, order);
    if (stream) _mm256_stream_si256((__m256i*)d, r);
    else _mm256_storeu_si256((__m256i*)d, r);
    return _mm256_testz_si256(bad, bad);
}

// The last < 128 residues of a sequence in place: 128 bytes are read from s
// (the caller guarantees they are readable), those at rem and beyond count
// as 'A'; 32 bytes are written.
__attribute__((target("avx2"))) inline bool tail_avx2(const uint8_t* s, uint64_t rem, uint8_t* d) {
    alignas(32) uint8_t buf[128];
    const __m256i A = _mm256_set1_epi8('A');
    const __m256i idx0 = _mm256_setr_epi8(0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15, 16, 17, 18, 19, 20, 21,
                                          22, 23, 24, 25, 26, 27, 28, 29, 30, 31);
    const __m256i lim = _mm256_set1_epi8((char)rem);  // rem < 128: signed compare is exact
#pragma GCC unroll 4
    for (int u = 0; u < 4; ++u) {
        const __m256i idx = _mm256_add_epi8(idx0, _mm256_set1_epi8((char)(32 * u)));
        const __m256i keep = _mm256_cmpgt_epi8(lim, idx);  // idx < rem
        const __m256i x = _mm256_loadu_si256((const __m256i*)(s + 32 * u));
        _mm256_store_si256((__m256i*)(buf + 32 * u), _mm256_blendv_epi8(A, x, keep));
    }
    return block128_avx2(buf, d, true);
}

__attribute__((target("avx2"))) bool pack_avx2(const uint8_t* s, uint64_t n, uint8_t* d) {
    const bool aligned = ((uintptr_t)d & 31) == 0;
    uint64_t i = 0;
    for (; i + 128 <= n; i += 128)
        if (!block128_avx2(s + i, d + i / 4, aligned)) {
            _mm_sfence();
            return false;
        }
    _mm_sfence();
    return pack_scalar(s + i, n - i, d + i / 4);
}

// One sequence into its code_bytes(L, 2) region (32 B per started block of
// 128 residues, zero past the end), every block with one aligned streaming
// store. The tail block reads 128 bytes in place (past the sequence, into
// the next one) unless that would cross src_end; then it goes through a
// buffer, so nothing past the input is read.
template <bool AVX>
inline bool pack_seq(const uint8_t* s, uint64_t L, uint8_t* d, const uint8_t* src_end) {
    uint64_t i = 0;
    for (; i + 128 <= L; i += 128) {
        bool ok;
        if constexpr (AVX) ok = block128_avx2(s + i, d + i / 4, true);
        else ok = pack_scalar(s + i, 128, d + i / 4);
        if (!ok) return false;
    }
    const uint64_t rem = L - i;
    if (rem == 0) return true;
    if constexpr (AVX) {
        if (s + i + 128 <= src_end) return tail_avx2(s + i, rem, d + i / 4);
    }
    alignas(32) uint8_t tail[128];
    std::memset(tail, 'A', sizeof(tail));
    std::memcpy(tail, s + i, rem);
    if constexpr (AVX) return block128_avx2(tail, d + i / 4, true);
    else return pack_scalar(tail, 128, d + i / 4);
}

__attribute__((target("avx2"))) bool pack_seqs_avx2(const uint8_t* data, const uint64_t* offs, uint64_t lo,
                                                      uint64_t hi, uint8_t* d, const uint8_t* src_end) {
    bool ok = true;
    for (uint64_t k = lo; k < hi && ok; ++k) {
        const uint64_t L = offs[k + 1] - offs[k];
        ok = pack_seq<true>(data + offs[k], L, d, src_end);
        d += ((L + 127) >> 7) << 5;
    }
    _mm_sfence();
    return ok;
}

bool pack_seqs_scalar(const uint8_t* data, const uint64_t* offs, uint64_t lo, uint64_t hi, uint8_t* d) {
    for (uint64_t k = lo; k < hi; ++k) {
        const uint64_t L = offs[k + 1] - offs[k];
        if (!pack_seq<false>(data + offs[k], L, d, nullptr)) return false;
        d += ((L + 127) >> 7) << 5;
    }
    return true;
}

bool have_avx2() {
    static const bool v = __builtin_cpu_supports("avx2");
    return v;
}

}  // namespace

void host_pool_run(uint64_t ntasks, const std::function<void(uint64_t)>& f) { pool().run(ntasks, f); }
unsigned host_pool_threads() { return pool().threads(); }

bool pack_acgt_serial(const uint8_t* src, uint64_t n, uint8_t* dst) {
    return have_avx2() ? pack_avx2(src, n, dst) : pack_scalar(src, n, dst);
}

bool pack_acgt_seqs(const char* data, const uint64_t* offs, uint64_t n, uint8_t* dst, uint64_t* bytes) {
    // sequences per task: >= 4 tasks per pool thread (balance), >= 256 (overhead)
    const uint64_t per = std::max<uint64_t>(256, (n + 4 * host_pool_threads() - 1) / (4 * host_pool_threads()));
    const uint64_t ntasks = (n + per - 1) / per;
    std::vector<uint64_t> base(ntasks + 1, 0);
    host_pool_run(ntasks, [&](uint64_t t) {
        uint64_t sum = 0;
        for (uint64_t k = t * per, e = std::min(n, k + per); k < e; ++k) sum += ((offs[k + 1] - offs[k] + 127) >> 7) << 5;
        base[t + 1] = sum;
    });
    for (uint64_t t = 0; t < ntasks; ++t) base[t + 1] += base[t];
    *bytes = base[ntasks];
    std::atomic<bool> bad{false};
    const uint8_t* d8 = reinterpret_cast<const uint8_t*>(data);
    const bool avx = have_avx2();
    host_pool_run(ntasks, [&](uint64_t t) {
        if (bad.load(std::memory_order_relaxed)) return;
        const uint64_t lo = t * per, hi = std::min(n, lo + per);
        const bool ok = avx ? pack_seqs_avx2(d8, offs, lo, hi, dst + base[t], d8 + offs[n])
                            : pack_seqs_scalar(d8, offs, lo, hi, dst + base[t]);
        if (!ok) bad.store(true, std::memory_order_relaxed);
    });
    return !bad.load();
}

bool pack_acgt(const uint8_t* src, uint64_t n, uint8_t* dst) {
    constexpr uint64_t piece = 1ull << 20;  // residues per task (multiple of 128)
    const uint64_t ntasks = (n + piece - 1) / piece;
    std::atomic<bool> bad{false};
    host_pool_run(ntasks, [&](uint64_t t) {
        if (bad.load(std::memory_order_relaxed)) return;
        const uint64_t lo = t * piece, len = std::min(piece, n - lo);
        if (!pack_acgt_serial(src + lo, len, dst + lo / 4)) bad.store(true, std::memory_order_relaxed);
    });
    return !bad.load();
}

}  // namespace dm
