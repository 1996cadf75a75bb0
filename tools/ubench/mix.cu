// Ceiling of the distance kernel's per-word instruction mix on one B200:
// the K1 word update (LDS match mask, 6 LOP3, carry-chained add, IMAD Ph,
// two 1-bit shifts) over W = 16 words per column, no shuffles, no text loads,
// no bounds checks, 24 warps per SM as in lev_kernel<2,16>. Variants compare
// shift forms (IMAD.WIDE+IMAD, funnel, carry-chained add — the one K1 uses)
// and Ph as IMAD vs LOP3; results in profiles/r01_ubench_mix.txt.
// Prints cells/s; the real kernel's number divided by this one is the share
// of the mix's ceiling it reaches.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#include "../../paper_2601_15458_b200/csrc/lev_chains.h"

constexpr int W = 16;

__device__ __forceinline__ uint32_t imad(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d;
  asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}
template <int LUT>
__device__ __forceinline__ uint32_t lop3(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d;
  asm("lop3.b32 %0, %1, %2, %3, %4;" : "=r"(d) : "r"(a), "r"(b), "r"(c), "n"(LUT));
  return d;
}
__device__ __forceinline__ uint32_t shl1(uint32_t (&v)[W], uint32_t cin, uint32_t two, uint32_t one) {
  uint32_t carry = cin;
#pragma unroll
  for (int w = 0; w < W; ++w) {
    uint32_t lo, hi;
    asm("{\n\t.reg .u64 t;\n\tmul.wide.u32 t, %2, %3;\n\tmov.b64 {%0, %1}, t;\n\t}" : "=r"(lo), "=r"(hi) : "r"(v[w]), "r"(two));
    v[w] = imad(lo, one, carry);
    carry = hi;
  }
  return carry;
}

// shift variants: 0 IMAD.WIDE + IMAD (FMA pipe), 1 funnel shift (SHF), 2 add-with-carry chain
template <int SV>
__device__ __forceinline__ uint32_t shl1v(uint32_t (&v)[W], uint32_t cin, uint32_t two, uint32_t one) {
  if constexpr (SV == 0) return shl1(v, cin, two, one);
  if constexpr (SV == 1) {
    const uint32_t out = v[W - 1] >> 31;
#pragma unroll
    for (int w = W - 1; w > 0; --w) v[w] = __funnelshift_l(v[w - 1], v[w], 1);
    v[0] = (v[0] << 1) | cin;
    return out;
  }
  if constexpr (SV == 3) {  // FMA pipe: word w = v[w] * 2 + hi(v[w-1] * 2) (IMAD + IMAD.HI)
    uint32_t out;
    asm("mul.hi.u32 %0, %1, %2;" : "=r"(out) : "r"(v[W - 1]), "r"(two));
#pragma unroll
    for (int w = W - 1; w > 0; --w) {
      uint32_t h;
      asm("mul.hi.u32 %0, %1, %2;" : "=r"(h) : "r"(v[w - 1]), "r"(two));
      v[w] = imad(v[w], two, h);
    }
    v[0] = imad(v[0], two, cin);
    return out;
  }
  if constexpr (SV == 2) {
    uint32_t out;
    uint32_t t[W];
#pragma unroll
    for (int w = 0; w < W; ++w) t[w] = v[w];
    dm::Chain<W>::add(v, t, t);  // v = t + t (carry across words)
    out = t[W - 1] >> 31;
    v[0] |= cin;
    return out;
  }
  return 0;
}

template <int ILP, int MINB, int SV = 0, int PH = 0, int SVM = SV>
__global__ void __launch_bounds__(256, MINB) mix(uint32_t* out, int cols, uint32_t one) {
  extern __shared__ uint32_t tab[];
  for (int i = threadIdx.x; i < 4 * W * 256; i += 256) tab[i] = i * 2654435761u;
  __syncthreads();
  const uint32_t two = one + one;
  uint32_t PvA[ILP][W], MvA[ILP][W];
  uint32_t hpA[ILP], hmA[ILP], cA[ILP];
#pragma unroll
  for (int q = 0; q < ILP; ++q) {
#pragma unroll
    for (int w = 0; w < W; ++w) { PvA[q][w] = ~0u; MvA[q][w] = 0; }
    hpA[q] = 1; hmA[q] = 0; cA[q] = (threadIdx.x + q) & 3;
  }
  for (int s = 0; s < cols; ++s) {
#pragma unroll
  for (int q = 0; q < ILP; ++q) {
    uint32_t (&Pv)[W] = PvA[q];
    uint32_t (&Mv)[W] = MvA[q];
    uint32_t& hp = hpA[q];
    uint32_t& hm = hmA[q];
    uint32_t& c = cA[q];
    uint32_t X[W], S[W], Ph[W], Mh[W], Xv[W];
#pragma unroll
    for (int w = 0; w < W; ++w) {
      const uint32_t e = tab[(c * W + w) * 256 + threadIdx.x];
      Xv[w] = e | Mv[w];
      X[w] = w == 0 ? lop3<0xA8>(e, hm, Pv[w]) : (e & Pv[w]);
    }
    dm::Chain<W>::add(S, X, Pv);
#pragma unroll
    for (int w = 0; w < W; ++w) {
      Mh[w] = lop3<0xBA>(Pv[w], S[w], X[w]);
      if constexpr (PH == 0) Ph[w] = imad(lop3<0x01>(S[w], Pv[w], Xv[w]), one, Mv[w]);
      else Ph[w] = lop3<0xF1>(Mv[w], S[w], Pv[w] | Xv[w]);
    }
    const uint32_t hpo = shl1v<SV>(Ph, hp, two, one);
    const uint32_t hmo = shl1v<SVM>(Mh, hm, two, one);
#pragma unroll
    for (int w = 0; w < W; ++w) {
      Pv[w] = lop3<0xF1>(Mh[w], Xv[w], Ph[w]);
      Mv[w] = Ph[w] & Xv[w];
    }
    hp = hpo & 1u;
    hm = hmo & 1u;
    c = (c + hp + s) & 3u;
  }
  }
  uint32_t r = 0;
#pragma unroll
  for (int q = 0; q < ILP; ++q)
#pragma unroll
    for (int w = 0; w < W; ++w) r += __popc(PvA[q][w]) - __popc(MvA[q][w]);
  if (r == (uint32_t)cols * 977u + one) out[0] = r;  // runtime-opaque: keeps the work live
}

template <int ILP, int MINB, int SV = 0, int PH = 0, int SVM = SV>
void run(uint32_t* d, int sms) {
  const int smem = 4 * W * 256 * 4;
  cudaFuncSetAttribute(mix<ILP, MINB, SV, PH, SVM>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, mix<ILP, MINB, SV, PH, SVM>, 256, smem);
  const int cols = 4096, blocks = sms * occ;
  mix<ILP, MINB, SV, PH, SVM><<<blocks, 256, smem>>>(d, 64, 1u);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  mix<ILP, MINB, SV, PH, SVM><<<blocks, 256, smem>>>(d, cols, 1u);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) {
    printf("CUDA error: %s\n", cudaGetErrorString(err));
    return;
  }
  const double cells = (double)blocks * 256 * cols * W * 32 * ILP;
  const char* nm[] = {"IMAD.WIDE", "funnel", "add-chain", "IMAD+IMAD.HI"};
  printf("ILP %d, blocks/SM %d, shifts Ph %s / Mh %s, Ph %s: %.1f TCUPS for the bare per-word mix (W=%d)\n", ILP,
         occ, nm[SV], nm[SVM], PH == 0 ? "IMAD" : "LOP3",
         cells / (ms * 1e-3) / 1e12, W);
}

int main() {
  uint32_t* d;
  cudaMalloc(&d, 64);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<1, 3>(d, sms);
  run<1, 3, 2>(d, sms);
  run<1, 3, 2, 1>(d, sms);
  run<1, 3, 2, 0, 0>(d, sms);
  run<1, 3, 0, 0, 2>(d, sms);
  run<1, 3, 2, 0, 1>(d, sms);
  run<1, 3, 1, 0, 2>(d, sms);
  run<2, 2, 2>(d, sms);
  run<1, 3, 3, 0, 2>(d, sms);
  run<1, 3, 2, 0, 3>(d, sms);
  run<1, 3, 3, 0, 3>(d, sms);
  run<1, 3, 3, 0, 1>(d, sms);
  return 0;
}
