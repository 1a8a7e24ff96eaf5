/*
 * include/gcr_synth.h -- C-ABI of libgcr_synth.so: the seeded synthetic-input
 * generator shared by the GPU tests, the bench and smoke() (DESIGN.md §6,
 * "input recipe").  HARNESS, not part of the snapshot method: it holds none of
 * the method's arithmetic (no CRC, no classification, no packing).  The CPU
 * twin is paper_2502_16631_b200/synth.py; both implement the same
 * counter-based generator, so CPU and GPU bytes are identical.
 *
 * Word i (u64, little-endian) of an allocation with key k under seed s is
 * derived from r = splitmix64(s ^ (k << 40) ^ i) according to `kind`:
 *   0 RANDOM       r
 *   1 F32_WEIGHT   per 32-bit half b: sign(b) | (118 + ((b>>23)&3)) << 23 | b & 0x7FFFFF
 *                  (|w| in [2^-9, 2^-5): random-init weights)
 *   2 F32_CONST    both halves = const_bits (e.g. 0x3F800000 = 1.0f, LayerNorm gamma)
 *   3 ZERO         0 (biases, LayerNorm beta, step-0 optimizer state)
 *   4 F32_M        sign(b) | (113 + ((b>>23)&3)) << 23 | mantissa  (Adam m, [2^-14, 2^-10))
 *   5 F32_V        (103 + ((b>>23)&3)) << 23 | mantissa            (Adam v > 0, [2^-24, 2^-20))
 *   6 BF16_WEIGHT  per 16-bit quarter h: sign(h) | (118 + ((h>>7)&3)) << 7 | h & 0x7F
 */
#ifndef GCR_SYNTH_H
#define GCR_SYNTH_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

/* Fill [dptr, dptr+bytes) (device memory, bytes % 8 == 0) asynchronously on
 * cuda_stream.  Returns 0, or a cudaError_t value. */
int gsy_fill(uint64_t dptr, uint64_t bytes, uint64_t seed, uint32_t key, uint32_t kind,
             uint32_t const_bits, void *cuda_stream);

/* XOR the u32 at dptr with x (one mutation: the page becomes dirty).  Async. */
int gsy_xor_u32(uint64_t dptr, uint32_t x, void *cuda_stream);

/* n mutations at once: dptrs[i] ^= xs[i] (host arrays, copied; synchronous
 * with respect to the host arrays, asynchronous on cuda_stream otherwise). */
int gsy_xor_u32_batch(const uint64_t *dptrs, const uint32_t *xs, uint64_t n, void *cuda_stream);

/* Fault-injection helpers for the lock-timeout test: a mapped pinned flag and
 * a kernel that spins on `cuda_stream` until the flag becomes non-zero. */
int gsy_flag_alloc(uint64_t *host_ptr, uint64_t *dev_ptr);
int gsy_flag_set(uint64_t host_ptr, uint32_t value);
int gsy_flag_free(uint64_t host_ptr);
int gsy_spin_until_flag(uint64_t dev_flag, void *cuda_stream);

#ifdef __cplusplus
}
#endif
#endif
