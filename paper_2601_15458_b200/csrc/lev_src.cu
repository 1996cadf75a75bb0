// Distance-kernel instances for host-planned streamed chunks (stream.cu):
// <= 4 residue symbols, pattern match masks split out of the 2-bit codes
// (kSrcCodes, host-packed chunks) or of the caller's A/C/G/T bytes
// (kSrcRaw, chunks uploaded as given), so no device-side preparation runs
// between a chunk's upload and its kernels. Kept apart from lev.cu so the
// two instance sets compile in parallel.
#include "lev_kernel.cuh"

namespace dm {

void lev_launch_bucket_src(int src, int w, const LevArgs& a, int sm_count, cudaStream_t st) {
    if (src == kSrcCodes) dispatch_w<2, 1, kSrcCodes>(w, a, sm_count, st);
    else if (src == kSrcRaw) dispatch_w<2, 1, kSrcRaw>(w, a, sm_count, st);
    else throw runtime_error("internal error: unknown distance-kernel source");
}

void lev_warm_src() {
    warm_np<2, 1, kSrcCodes>();
    warm_np<2, 1, kSrcRaw>();
}

}  // namespace dm
