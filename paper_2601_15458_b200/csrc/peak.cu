// INT32 lane-op peak microbenchmark: the denominator of the
// distance/alignment rooflines. MEASURED_PEAKS.json carries only HBM and
// bf16, so the integer peak is measured on the box, at the clocks of the run.
//
// mode 0: independent LOP3 chains            (ALU pipe only)
// mode 1: independent IMAD chains            (FMA pipe only)
// mode 2: LOP3 chains interleaved with IMAD  (ALU + FMA pipes, dual issue)
// Each chain step is exactly one SASS instruction (inline PTX lop3 / mad.lo);
// 8 chains per thread give ILP well past the 4-cycle latency.
#include "dm_internal.h"

namespace dm {
namespace {

template <int MODE>
__global__ void __launch_bounds__(256) int_peak_kernel(uint32_t* out, int iters, uint32_t seed) {
    uint32_t a[8], b = seed * 2654435761u + threadIdx.x, c = seed ^ (blockIdx.x * 7919u);
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = threadIdx.x * (k + 3) + seed;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 16; ++u) {
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                if (MODE == 0 || (MODE == 2 && (k & 1) == 0)) {
                    asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(a[k]) : "r"(b), "r"(c));
                } else {
                    asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(a[k]) : "r"(b | 1u), "r"(c));
                }
            }
        }
        b += 0x9e3779b9u;
        c ^= b;
    }
    uint32_t r = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) r ^= a[k];
    if (r == 0x12345678u) out[0] = r;  // keep the chains alive
}

}  // namespace

double int32_peak(dm_ctx* ctx, int mode) {
    const int iters = 4096;
    const int blocks = ctx->sm_count * 8;  // 2048 threads / SM resident
    uint32_t* d = ctx->aux.as<uint32_t>(4);
    auto launch = [&] {
        if (mode == 0) int_peak_kernel<0><<<blocks, 256, 0, ctx->stream>>>(d, iters, 1u);
        else if (mode == 1) int_peak_kernel<1><<<blocks, 256, 0, ctx->stream>>>(d, iters, 1u);
        else int_peak_kernel<2><<<blocks, 256, 0, ctx->stream>>>(d, iters, 1u);
    };
    launch();  // warm-up
    DM_CUDA(cudaGetLastError());
    DM_CUDA(cudaEventRecord(ctx->ev0, ctx->stream));
    const int reps = 5;
    for (int r = 0; r < reps; ++r) launch();
    DM_CUDA(cudaEventRecord(ctx->ev1, ctx->stream));
    DM_CUDA(cudaEventSynchronize(ctx->ev1));
    float ms = 0;
    DM_CUDA(cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1));
    // lane-ops: threads * iters * 16 unroll * 8 chains, one instruction each
    const double ops = (double)blocks * 256 * iters * 16.0 * 8.0 * reps;
    return ops / (ms * 1e-3);
}

}  // namespace dm

