// Host side of the compressed upload of streamed pair batches: nucleotide
// chunks (bytes A, C, G, T only) cross PCIe as 2-bit codes, a quarter of the
// bytes, and are expanded back to the identical residue bytes on the device
// (stream.cu). Packing runs on a persistent pool of host threads.
#pragma once

#include <cstdint>
#include <functional>

namespace dm {

// Run f(0..ntasks-1) on the process-wide host pool (the calling thread
// helps); returns when every task is done. Calls are serialised.
void host_pool_run(uint64_t ntasks, const std::function<void(uint64_t)>& f);
unsigned host_pool_threads();

// Residue j of src -> bits 2(j%4)..2(j%4)+1 of dst[j/4], codes A0 C1 G2 T3;
// the last byte is zero-padded. Returns false (dst unspecified) as soon as a
// byte other than 'A', 'C', 'G', 'T' is seen. Multithreaded.
bool pack_acgt(const uint8_t* src, uint64_t n, uint8_t* dst);

// Sequences offs[0..n] of data (absolute offsets) packed one by one into the
// 2-bit code layout of a sequence set (code_bytes(L, 2) bytes each: 32 B per
// started 128-residue block, zero-padded), i.e. the device code buffer
// itself; dst must be 32-B aligned; *bytes = its size. False (dst
// unspecified) if a byte is not A/C/G/T. Multithreaded.
bool pack_acgt_seqs(const char* data, const uint64_t* offs, uint64_t n, uint8_t* dst, uint64_t* bytes);

// Single-threaded kernel of pack_acgt over [src, src+n) (n % 4 == 0 except
// for the last piece); exposed for tests.
bool pack_acgt_serial(const uint8_t* src, uint64_t n, uint8_t* dst);

}  // namespace dm
