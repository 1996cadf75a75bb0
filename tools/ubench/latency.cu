// Dependent-chain latency (cycles per op) of integer / DPX instructions on one warp.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int MODE>
__global__ void lat(uint32_t* out, uint32_t seed, long long* cyc) {
  uint32_t a = seed + threadIdx.x, b = seed * 3u, c = seed ^ 0x1234u;
  long long t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 1024; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      if (MODE == 0) asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(a) : "r"(b), "r"(c));
      if (MODE == 1) asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(a) : "r"(b | 1u), "r"(c));
      if (MODE == 2) a = (uint32_t)__viaddmax_s32((int)a, (int)b, (int)c);
      if (MODE == 3) a = __viaddmax_s16x2(a, b, c);
      if (MODE == 4) a = (uint32_t)__vimax3_s32((int)a, (int)b, (int)c);
      if (MODE == 5) a = __vimax3_s16x2(a, b, c);
      if (MODE == 6) a = __byte_perm(a, b, 0x5410);
      if (MODE == 7) asm volatile("shfl.sync.up.b32 %0, %0, 1, 0, -1;" : "+r"(a));
    }
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[MODE] = t1 - t0;
  if (a == 0x12345678u) out[0] = a;
}

int main() {
  uint32_t* d; long long* c; cudaMalloc(&d, 64); cudaMalloc(&c, 8 * sizeof(long long));
  lat<0><<<1, 32>>>(d, 1, c); lat<1><<<1, 32>>>(d, 1, c); lat<2><<<1, 32>>>(d, 1, c); lat<3><<<1, 32>>>(d, 1, c);
  lat<4><<<1, 32>>>(d, 1, c); lat<5><<<1, 32>>>(d, 1, c); lat<6><<<1, 32>>>(d, 1, c); lat<7><<<1, 32>>>(d, 1, c);
  long long h[8]; cudaMemcpy(h, c, sizeof(h), cudaMemcpyDeviceToHost);
  const char* nm[] = {"LOP3", "IMAD", "VIADDMNMX", "VIADDMNMX.S16x2", "VIMNMX3", "VIMNMX3.S16x2", "PRMT", "SHFL.UP"};
  for (int i = 0; i < 8; ++i) printf("%-16s %.2f cycles/op\n", nm[i], h[i] / (1024.0 * 16));
  return 0;
}
