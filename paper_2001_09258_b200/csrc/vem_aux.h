/* vem auxiliary device utilities for the BENCH and the TESTS -- not part of
 * the reference-facing C ABI (include/vem.h) and never on the math path.
 *
 *  - vem_aux_fill: the config-input generator of paper_2001_09258_b200/inputs.py
 *    evaluated on the device (same recipe, same global element index, same
 *    bits), so bench.py can create 2^28..2^31-element config arrays in HBM
 *    without shipping them over PCIe, and the parity tests can check them
 *    against the host generator's checksums;
 *  - vem_aux_checksum: position-keyed additive 64-bit checksums of an array,
 *    per 2^log2chunk-element chunk of the GLOBAL index space:
 *      C[c] = sum_{i in chunk c} fmix64(bits(v_i) ^ (i * 0x9E3779B97F4A7C15))  mod 2^64
 *    Additive, so the partial sums of any set of shards (arbitrary
 *    boundaries) add up to the checksum of the whole array -- the property
 *    the sharded bench and the shard-invariance tests rely on.  The host
 *    twins live in oracle/vem_gen_host.c (C, OpenMP) and inputs.py (numpy).
 */
#ifndef VEM_AUX_H
#define VEM_AUX_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  uint64_t seed;      /* value stream */
  uint64_t spec_seed; /* special-value overlay streams (config 5) */
  double a, b;        /* uniform: [a, b); log-uniform: log2 bounds */
  int32_t kind;       /* 0 uniform, 1 log-uniform */
  int32_t sign;       /* 1: random sign from stream seed ^ 0x5151 */
  int32_t specials;   /* 1: 1 % special-value overlay */
  int32_t f32;        /* 1: binary32 output */
} vem_recipe;

/* out[j] = element (offset + j) of the recipe's array, j < n.  Async on s. */
int vem_aux_fill(const vem_recipe* r, void* out, size_t n, uint64_t offset, void* stream);

/* Adds the checksum contributions of p[0..n) (global indices offset..) into
 * sums[c - (offset >> log2chunk)] for every chunk c the range touches (sums
 * is a device array the caller zeroes).  elem_bytes 4 or 8.  Async on s. */
int vem_aux_checksum(const void* p, size_t n, int elem_bytes, uint64_t offset, int log2chunk,
                     unsigned long long* sums, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* VEM_AUX_H */
