// Device-resident sequence store: raw residues, a dense
// re-coding of the residues for the distance engine (2 bits per residue when
// at most 4 symbols occur, else a byte; layout code_bytes()), and
// per-sequence bit-plane profiles.
//
// Levenshtein compares raw bytes (distance.cpp:40 `ai != b[j]`),
// so the code map is a bijection over the bytes that actually occur: S
// distinct bytes get codes 0..S-1 and the distance engine works on
// NP = 2 (S <= 4, e.g. ACGT), 5 (S <= 32, proteins) or 8 bit-planes.
//
// Plane layout: sequence i owns blocks [blk_off[i], blk_off[i] + ceil(len/64));
// block b holds NP 64-bit words, word k bit t = bit k of code(residue 64b+t).
// Residues past the end of the sequence are zero (their rows are never read
// by the final count; see lev.cu).
#include <algorithm>
#include <cstring>

#include <cub/cub.cuh>

#include "dm_internal.h"
#include "host_copy.h"

namespace dm {
namespace {

// Byte census: each thread ORs 16 bytes per uint4 into a private 256-bit
// mask (4 x u64 in registers), then one warp-reduced atomicOr per word.
__global__ void census_kernel(const uint8_t* __restrict__ raw, uint64_t nbytes,
                              unsigned long long* __restrict__ present) {
    unsigned long long m0 = 0, m1 = 0, m2 = 0, m3 = 0;
    auto put = [&](uint32_t c) {
        const unsigned long long bit = 1ull << (c & 63);
        const uint32_t q = c >> 6;
        m0 |= q == 0 ? bit : 0ull;
        m1 |= q == 1 ? bit : 0ull;
        m2 |= q == 2 ? bit : 0ull;
        m3 |= q == 3 ? bit : 0ull;
    };
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    const uint64_t head = (16 - ((uintptr_t)raw & 15)) & 15;
    const uint64_t t0 = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t0 < head && t0 < nbytes) put(raw[t0]);
    const uint64_t nvec = nbytes > head ? (nbytes - head) / 16 : 0;
    const uint4* v = reinterpret_cast<const uint4*>(raw + head);
    for (uint64_t i = t0; i < nvec; i += stride) {
        const uint4 x = v[i];
        const uint32_t w[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            put(w[k] & 0xff);
            put((w[k] >> 8) & 0xff);
            put((w[k] >> 16) & 0xff);
            put(w[k] >> 24);
        }
    }
    for (uint64_t i = head + nvec * 16 + t0; i < nbytes; i += stride) put(raw[i]);
    for (int o = 16; o > 0; o >>= 1) {
        m0 |= __shfl_xor_sync(0xffffffffu, m0, o);
        m1 |= __shfl_xor_sync(0xffffffffu, m1, o);
        m2 |= __shfl_xor_sync(0xffffffffu, m2, o);
        m3 |= __shfl_xor_sync(0xffffffffu, m3, o);
    }
    if ((threadIdx.x & 31) == 0) {
        if (m0) atomicOr(&present[0], m0);
        if (m1) atomicOr(&present[1], m1);
        if (m2) atomicOr(&present[2], m2);
        if (m3) atomicOr(&present[3], m3);
    }
}

// One warp per sequence: recode raw bytes into the 16-B aligned code buffer.
__global__ void recode_kernel(const uint8_t* __restrict__ raw, const uint64_t* __restrict__ raw_off,
                              const uint64_t* __restrict__ off, uint32_t n,
                              const uint8_t* __restrict__ lut, uint8_t* __restrict__ codes) {
    __shared__ uint8_t slut[256];
    for (int i = threadIdx.x; i < 256; i += blockDim.x) slut[i] = lut[i];
    __syncthreads();
    const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
    for (uint32_t s = warp; s < n; s += nw) {
        const uint64_t a = raw_off[s], e = raw_off[s + 1], o = off[s];
        for (uint64_t i = a + lane; i < e; i += 32) codes[o + (i - a)] = slut[raw[i]];
    }
}

// 2-bit code layout (<= 4 symbols, code_bytes()): one warp per sequence,
// one lane per 16-residue word; the padding words come out zero, so the code
// buffer needs no memset.
__global__ void recode2_kernel(const uint8_t* __restrict__ raw, const uint64_t* __restrict__ raw_off,
                               const uint64_t* __restrict__ off, uint32_t n,
                               const uint8_t* __restrict__ lut, uint32_t* __restrict__ codes) {
    __shared__ uint8_t slut[256];
    for (int i = threadIdx.x; i < 256; i += blockDim.x) slut[i] = lut[i];
    __syncthreads();
    const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
    for (uint32_t s = warp; s < n; s += nw) {
        const uint64_t a = raw_off[s], e = raw_off[s + 1], o = off[s] >> 2, words = (off[s + 1] >> 2) - o;
        for (uint64_t w = lane; w < words; w += 32) {
            uint32_t v = 0;
#pragma unroll
            for (int k = 0; k < 16; ++k) {
                const uint64_t r = a + w * 16 + k;
                if (r < e) v |= (uint32_t)slut[raw[r]] << (2 * k);
            }
            codes[o + w] = v;
        }
    }
}

// Even bits of x (bits 0, 2, .., 30) gathered into the low 16 bits.
__device__ __forceinline__ uint32_t even_bits(uint32_t x) {
    x &= 0x55555555u;
    x = (x | (x >> 1)) & 0x33333333u;
    x = (x | (x >> 2)) & 0x0f0f0f0fu;
    x = (x | (x >> 4)) & 0x00ff00ffu;
    return (x | (x >> 8)) & 0x0000ffffu;
}

template <int NP>
__global__ void planes_kernel(const uint8_t* __restrict__ codes, const uint64_t* __restrict__ off,
                              const uint32_t* __restrict__ len, const uint64_t* __restrict__ blk,
                              uint32_t n, uint64_t* __restrict__ planes) {
    // one thread per sequence block; sequences located by binary search on blk
    const uint64_t total = blk[n];
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t b = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; b < total; b += stride) {
        uint32_t lo = 0, hi = n;  // largest s with blk[s] <= b
        while (hi - lo > 1) {
            const uint32_t mid = (lo + hi) >> 1;
            if (blk[mid] <= b) lo = mid; else hi = mid;
        }
        // skip empty sequences sharing the same start
        while (lo + 1 < n && blk[lo + 1] <= b) ++lo;
        const uint32_t s = lo;
        const uint64_t local = b - blk[s];
        const uint32_t L = len[s];
        const uint8_t* p = codes + off[s] + local * 64;
        const uint64_t rem = (uint64_t)L - local * 64;
        const int cnt = rem < 64 ? (int)rem : 64;
        uint64_t w[NP];
#pragma unroll
        for (int k = 0; k < NP; ++k) w[k] = 0;
        if constexpr (NP == 2) {
            // 2-bit codes: 64 residues = 4 words; plane k = bit k of every code
            const uint32_t* pw = reinterpret_cast<const uint32_t*>(codes + off[s]) + local * 4;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const uint32_t x = q * 16 < cnt ? pw[q] : 0u;
                w[0] |= (uint64_t)even_bits(x) << (16 * q);
                w[1] |= (uint64_t)even_bits(x >> 1) << (16 * q);
            }
            const uint64_t keep = cnt >= 64 ? ~0ull : ((1ull << cnt) - 1ull);
            planes[b * 2] = w[0] & keep;
            planes[b * 2 + 1] = w[1] & keep;
            continue;
        }
        // codes are 16-B aligned per sequence and zero-padded past the end
        const uint4* pv = reinterpret_cast<const uint4*>(p);
        for (int q = 0; q < (cnt + 15) / 16; ++q) {
            const uint4 x = pv[q];
            const uint32_t ww[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
            for (int k4 = 0; k4 < 16; ++k4) {
                const int t = q * 16 + k4;
                const unsigned c = t < cnt ? (ww[k4 >> 2] >> ((k4 & 3) * 8)) & 0xffu : 0u;
#pragma unroll
                for (int k = 0; k < NP; ++k) w[k] |= (uint64_t)((c >> k) & 1u) << t;
            }
        }
#pragma unroll
        for (int k = 0; k < NP; ++k) planes[b * NP + k] = w[k];
    }
}

// Per-sequence metadata from absolute device offsets (streamed batches):
// relative raw offsets, lengths and the padded sizes the two scans turn into
// code offsets (code_bytes() layout) and first plane block.
__global__ void meta_kernel(const uint64_t* __restrict__ offs, uint32_t n, int planes, uint64_t* __restrict__ raw_off,
                            uint32_t* __restrict__ len, uint64_t* __restrict__ code_sz,
                            uint64_t* __restrict__ blk_sz) {
    const uint64_t base = offs[0];
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i <= n; i += gridDim.x * blockDim.x) {
        raw_off[i] = offs[i] - base;
        if (i < n) {
            const uint64_t L = offs[i + 1] - offs[i];
            len[i] = (uint32_t)L;
            code_sz[i] = code_bytes(L, planes);
            blk_sz[i] = (L + 63) / 64;
        } else {
            code_sz[i] = 0;
            blk_sz[i] = 0;
        }
    }
}

// Dense code map from the census mask: code(c) = #present bytes below c.
__global__ void lut_kernel(const unsigned int* __restrict__ present, uint8_t* __restrict__ lut) {
    const int c = threadIdx.x;
    int below = 0;
    for (int w = 0; w < (c >> 5); ++w) below += __popc(present[w]);
    below += __popc(present[c >> 5] & ((1u << (c & 31)) - 1u));
    lut[c] = (present[c >> 5] >> (c & 31)) & 1u ? (uint8_t)below : 0;
}

// Fixed code map of an all-A/C/G/T set: A0 C1 G2 T3.
__global__ void acgt_lut_kernel(uint8_t* __restrict__ lut) {
    const int c = threadIdx.x;
    lut[c] = c == 'C' ? 1 : (c == 'G' ? 2 : (c == 'T' ? 3 : 0));
}

}  // namespace

dm_seqset* seqset_create_device(dm_ctx* ctx, const uint8_t* d_raw, const uint64_t* d_offs,
                                const uint64_t* h_offs, uint32_t n, bool acgt, const uint8_t* d_codes_given) {
    auto* s = new dm_seqset;
    s->ctx = ctx;
    s->n = n;
    s->owns_raw = false;
    s->d_raw = const_cast<uint8_t*>(d_raw);
    try {
        if (d_codes_given && !acgt) throw invalid_argument("given codes need a known A/C/G/T alphabet");
        const uint64_t nbytes = h_offs[n] - h_offs[0];
        cudaStream_t st = ctx->stream;
        // alphabet: known (packed A/C/G/T chunk) or from the device census (one host sync)
        uint8_t* d_lut = (uint8_t*)ctx->aux2.get(256);
        if (acgt) {
            acgt_lut_kernel<<<1, 256, 0, st>>>(d_lut);
            DM_CUDA(cudaGetLastError());
            int k = 0;
            for (int c : {'A', 'C', 'G', 'T'}) {
                s->code_of[c] = (uint8_t)k++;
                s->present[c] = true;
            }
            s->nsym = 4;
            s->planes = 2;
        } else {
            unsigned int* d_present = ctx->aux.as<unsigned int>(8);
            DM_CUDA(cudaMemsetAsync(d_present, 0, 32, st));
            if (nbytes) {
                const int grid = (int)std::min<uint64_t>((nbytes + 4095) / 4096, (uint64_t)ctx->sm_count * 16);
                census_kernel<<<std::max(grid, 1), 256, 0, st>>>(d_raw, nbytes,
                                                                 reinterpret_cast<unsigned long long*>(d_present));
                DM_CUDA(cudaGetLastError());
            }
            lut_kernel<<<1, 256, 0, st>>>(d_present, d_lut);
            DM_CUDA(cudaGetLastError());
            unsigned int present[8];
            DM_CUDA(cudaMemcpyAsync(present, d_present, 32, cudaMemcpyDeviceToHost, st));
            DM_CUDA(cudaStreamSynchronize(st));
            int nsym = 0;
            for (int c = 0; c < 256; ++c)
                if (present[c >> 5] & (1u << (c & 31))) {
                    s->code_of[c] = (uint8_t)nsym++;
                    s->present[c] = true;
                }
            s->nsym = nsym;
            s->planes = nsym <= 4 ? 2 : (nsym <= 32 ? 5 : 8);
        }
        uint64_t o = 0, b = 0;
        for (uint32_t i = 0; i < n; ++i) {
            const uint64_t L = h_offs[i + 1] - h_offs[i];
            if (L > 0xffffffffull) throw invalid_argument("sequence longer than 2^32-1 residues");
            o += code_bytes(L, s->planes);
            b += (L + 63) / 64;
        }
        s->total_blocks = b;
        // device arrays from the context's scratch: no pool traffic per chunk
        s->owns_meta = false;
        const size_t a8 = ((size_t)(n + 1) * 8 + 255) & ~size_t(255), a4 = ((size_t)n * 4 + 259) & ~size_t(255);
        char* meta = (char*)ctx->ss_meta.get(3 * a8 + a4);
        s->d_raw_off = (uint64_t*)meta;
        s->d_off = (uint64_t*)(meta + a8);
        s->d_blk = (uint64_t*)(meta + 2 * a8);
        s->d_len = (uint32_t*)(meta + 3 * a8);
        size_t cub_b = 0;
        DM_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, cub_b, (uint64_t*)nullptr, (uint64_t*)nullptr, (int)n + 1, st));
        const size_t sz_b = ((size_t)(n + 1) * 8 + 255) & ~size_t(255);
        char* scratch = (char*)ctx->aux3.get(2 * sz_b + cub_b + 256);
        uint64_t* code_sz = (uint64_t*)scratch;
        uint64_t* blk_sz = (uint64_t*)(scratch + sz_b);
        void* cub_tmp = scratch + 2 * sz_b;
        const int mgrid = (int)std::min<uint64_t>((n + 256) / 256, (uint64_t)ctx->sm_count * 8);
        meta_kernel<<<std::max(mgrid, 1), 256, 0, st>>>(d_offs, n, s->planes, s->d_raw_off, s->d_len, code_sz, blk_sz);
        DM_CUDA(cudaGetLastError());
        DM_CUDA(cub::DeviceScan::ExclusiveSum(cub_tmp, cub_b, code_sz, s->d_off, (int)n + 1, st));
        DM_CUDA(cub::DeviceScan::ExclusiveSum(cub_tmp, cub_b, blk_sz, s->d_blk, (int)n + 1, st));

        s->d_planes = ctx->ss_planes.as<uint64_t>(std::max<uint64_t>(b, 1) * s->planes);
        if (d_codes_given) {
            s->d_raw = nullptr;  // the residues arrived as codes; there are no raw bytes
            s->d_codes = const_cast<uint8_t*>(d_codes_given);
        } else {
            s->d_codes = (uint8_t*)ctx->ss_codes.get(o + 16);
            const int grid = (int)std::min<uint64_t>((n + 7) / 8, (uint64_t)ctx->sm_count * 16);
            if (s->planes == 2) {
                if (n)
                    recode2_kernel<<<grid, 256, 0, st>>>(d_raw, s->d_raw_off, s->d_off, n, d_lut,
                                                         reinterpret_cast<uint32_t*>(s->d_codes));
            } else {
                DM_CUDA(cudaMemsetAsync(s->d_codes, 0, o + 16, st));
                if (n) recode_kernel<<<grid, 256, 0, st>>>(d_raw, s->d_raw_off, s->d_off, n, d_lut, s->d_codes);
            }
            DM_CUDA(cudaGetLastError());
        }
        if (b) {
            const int grid = (int)std::min<uint64_t>((b + 255) / 256, (uint64_t)ctx->sm_count * 16);
            if (s->planes == 2)
                planes_kernel<2><<<grid, 256, 0, st>>>(s->d_codes, s->d_off, s->d_len, s->d_blk, n, s->d_planes);
            else if (s->planes == 5)
                planes_kernel<5><<<grid, 256, 0, st>>>(s->d_codes, s->d_off, s->d_len, s->d_blk, n, s->d_planes);
            else
                planes_kernel<8><<<grid, 256, 0, st>>>(s->d_codes, s->d_off, s->d_len, s->d_blk, n, s->d_planes);
            DM_CUDA(cudaGetLastError());
        }
        ctx->launches += 7;
    } catch (...) {
        delete s;
        throw;
    }
    return s;
}

dm_seqset* seqset_create(dm_ctx* ctx, const char* data, const uint64_t* offsets, uint32_t n,
                         const uint8_t* d_raw_given) {
    auto* s = new dm_seqset;
    s->ctx = ctx;
    s->n = n;
    try {
        s->len.resize(n);
        s->off.resize(n + 1);
        s->blk_off.resize(n + 1);
        uint64_t o = 0, b = 0;
        for (uint32_t i = 0; i < n; ++i) {
            if (offsets[i + 1] < offsets[i]) throw invalid_argument("sequence offsets must be non-decreasing");
            const uint64_t L = offsets[i + 1] - offsets[i];
            if (L > 0xffffffffull) throw invalid_argument("sequence longer than 2^32-1 residues");
            s->len[i] = (uint32_t)L;
            s->blk_off[i] = b;
            b += (L + 63) / 64;
        }
        s->blk_off[n] = b;
        s->total_blocks = b;
        s->raw_off.assign(offsets, offsets + n + 1);
        const uint64_t base = offsets[0];
        const uint64_t nbytes = offsets[n] - base;
        cudaStream_t st = ctx->stream;

        uint8_t* d_raw = nullptr;
        uint64_t* d_raw_off = nullptr;
        if (d_raw_given) {  // bytes already on the device (streamed batches); not owned
            d_raw = const_cast<uint8_t*>(d_raw_given);
            s->owns_raw = false;
        } else {
            DM_CUDA(cudaMallocAsync(&d_raw, nbytes + 16, st));
        }
        DM_CUDA(cudaMallocAsync(&d_raw_off, (n + 1) * sizeof(uint64_t), st));
        s->d_raw = d_raw;
        s->d_raw_off = d_raw_off;
        std::vector<uint64_t> rel(n + 1);
        for (uint32_t i = 0; i <= n; ++i) rel[i] = offsets[i] - base;
        if (nbytes && !d_raw_given) upload_host(ctx, d_raw, data + base, nbytes, st);
        DM_CUDA(cudaMemcpyAsync(d_raw_off, rel.data(), (n + 1) * 8, cudaMemcpyHostToDevice, st));
        s->raw_off = rel;

        unsigned int* d_present = ctx->aux.as<unsigned int>(8);
        DM_CUDA(cudaMemsetAsync(d_present, 0, 32, st));
        if (nbytes) {
            const int grid = (int)std::min<uint64_t>((nbytes + 4095) / 4096, (uint64_t)ctx->sm_count * 16);
            census_kernel<<<std::max(grid, 1), 256, 0, st>>>(d_raw, nbytes,
                                                             reinterpret_cast<unsigned long long*>(d_present));
            DM_CUDA(cudaGetLastError());
            trace_bytes("census_kernel", nbytes, 0);
        }
        unsigned int present[8];
        DM_CUDA(cudaMemcpyAsync(present, d_present, 32, cudaMemcpyDeviceToHost, st));
        DM_CUDA(cudaStreamSynchronize(st));
        uint8_t lut[256] = {};
        int nsym = 0;
        for (int c = 0; c < 256; ++c)
            if (present[c >> 5] & (1u << (c & 31))) {
                lut[c] = (uint8_t)nsym++;
                s->present[c] = true;
            }
        std::memcpy(s->code_of, lut, 256);
        s->nsym = nsym;
        s->planes = nsym <= 4 ? 2 : (nsym <= 32 ? 5 : 8);
        for (uint32_t i = 0; i < n; ++i) {
            s->off[i] = o;
            o += code_bytes(s->len[i], s->planes);
        }
        s->off[n] = o;

        DM_CUDA(cudaMallocAsync(&s->d_codes, o + 16, st));
        DM_CUDA(cudaMallocAsync(&s->d_off, (n + 1) * sizeof(uint64_t), st));
        DM_CUDA(cudaMallocAsync(&s->d_len, std::max<size_t>(n, 1) * sizeof(uint32_t), st));
        DM_CUDA(cudaMallocAsync(&s->d_blk, (n + 1) * sizeof(uint64_t), st));
        DM_CUDA(cudaMallocAsync(&s->d_planes, std::max<uint64_t>(b, 1) * s->planes * sizeof(uint64_t), st));
        if (s->planes != 2) DM_CUDA(cudaMemsetAsync(s->d_codes, 0, o + 16, st));
        DM_CUDA(cudaMemcpyAsync(s->d_off, s->off.data(), (n + 1) * 8, cudaMemcpyHostToDevice, st));
        if (n) DM_CUDA(cudaMemcpyAsync(s->d_len, s->len.data(), n * 4, cudaMemcpyHostToDevice, st));
        DM_CUDA(cudaMemcpyAsync(s->d_blk, s->blk_off.data(), (n + 1) * 8, cudaMemcpyHostToDevice, st));
        uint8_t* d_lut = (uint8_t*)ctx->aux2.get(256);
        DM_CUDA(cudaMemcpyAsync(d_lut, lut, 256, cudaMemcpyHostToDevice, st));
        if (n) {
            const int grid = (int)std::min<uint64_t>((n + 7) / 8, (uint64_t)ctx->sm_count * 16);
            if (s->planes == 2)
                recode2_kernel<<<grid, 256, 0, st>>>(d_raw, d_raw_off, s->d_off, n, d_lut,
                                                     reinterpret_cast<uint32_t*>(s->d_codes));
            else
                recode_kernel<<<grid, 256, 0, st>>>(d_raw, d_raw_off, s->d_off, n, d_lut, s->d_codes);
            DM_CUDA(cudaGetLastError());
            trace_bytes(s->planes == 2 ? "recode2_kernel" : "recode_kernel", nbytes, o);
        }
        if (b) {
            const int grid = (int)std::min<uint64_t>((b + 255) / 256, (uint64_t)ctx->sm_count * 16);
            if (s->planes == 2)
                planes_kernel<2><<<grid, 256, 0, st>>>(s->d_codes, s->d_off, s->d_len, s->d_blk, n, s->d_planes);
            else if (s->planes == 5)
                planes_kernel<5><<<grid, 256, 0, st>>>(s->d_codes, s->d_off, s->d_len, s->d_blk, n, s->d_planes);
            else
                planes_kernel<8><<<grid, 256, 0, st>>>(s->d_codes, s->d_off, s->d_len, s->d_blk, n, s->d_planes);
            DM_CUDA(cudaGetLastError());
            trace_bytes("planes_kernel", o, b * s->planes * 8);
        }
        ctx->launches += 3;
        DM_CUDA(cudaStreamSynchronize(st));
    } catch (...) {
        delete s;
        throw;
    }
    return s;
}

}  // namespace dm

dm_seqset::~dm_seqset() {
    if (d_raw && owns_raw) cudaFreeAsync(d_raw, ctx->stream);
    if (!owns_meta) return;
    if (d_raw_off) cudaFreeAsync(d_raw_off, ctx->stream);
    if (d_codes) cudaFreeAsync(d_codes, ctx->stream);
    if (d_off) cudaFreeAsync(d_off, ctx->stream);
    if (d_len) cudaFreeAsync(d_len, ctx->stream);
    if (d_blk) cudaFreeAsync(d_blk, ctx->stream);
    if (d_planes) cudaFreeAsync(d_planes, ctx->stream);
}
