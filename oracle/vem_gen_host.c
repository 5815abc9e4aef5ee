/* TEST INFRASTRUCTURE ONLY -- host twin (C, OpenMP) of the config-input
 * generator and the chunk checksums (paper_2001_09258_b200/inputs.py spec,
 * device twin csrc/vem_aux.cu).  Used by tools/make_config_digests.py to
 * evaluate the CPU oracle over the FULL BASELINE config arrays (2^24..2^31
 * elements) in bounded memory, and pinned bit-for-bit against the numpy
 * generator by tests/test_config_inputs.py.  Compiled with
 * -ffp-contract=off: every operation is the rounded IEEE basic operation the
 * other two twins perform, in the same order. */
#include <math.h>
#include <stddef.h>
#include <stdint.h>
#include <string.h>

#include "../paper_2001_09258_b200/csrc/vem_aux.h"

static const uint64_t kGolden = 0x9E3779B97F4A7C15ull;

static inline uint64_t fmix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
static inline uint64_t sm64(uint64_t seed, uint64_t i) { return fmix64(seed + (i + 1) * kGolden); }
static inline double unit(uint64_t seed, uint64_t i) { return (double)(sm64(seed, i) >> 11) * 0x1p-53; }
static inline double from_bits(uint64_t b) {
  double d;
  memcpy(&d, &b, 8);
  return d;
}

static const double kExp2C[14] = {0x1.0000000000000p+0,  0x1.62e42fefa39efp-1,  0x1.ebfbdff82c58fp-3,
                                  0x1.c6b08d704a0c0p-5,  0x1.3b2ab6fba4e77p-7,  0x1.5d87fe78a6731p-10,
                                  0x1.430912f86c787p-13, 0x1.ffcbfc588b0c7p-17, 0x1.62c0223a5c824p-20,
                                  0x1.b5253d395e7c4p-24, 0x1.e4cf5158b8ecap-28, 0x1.e8cac7351bb25p-32,
                                  0x1.c3bd650fc2986p-36, 0x1.816193166d0f9p-40};

static inline double exp2_repro(double L) {
  const double k = floor(L);
  const double f = L - k;
  double p = kExp2C[13];
  for (int j = 12; j >= 0; j--) p = p * f + kExp2C[j];
  return p * from_bits((uint64_t)((int64_t)k + 1023) << 52);
}

static double element(const vem_recipe* r, uint64_t i) {
  const double u = unit(r->seed, i);
  double v = r->a + (r->b - r->a) * u;
  if (r->kind == 1) {
    v = exp2_repro(v);
    if (r->f32) v = fmin(fmax(v, 0x1p-126), 0x1.fffffep+127);
  }
  if (r->sign && (sm64(r->seed ^ 0x5151ull, i) >> 63)) v = -v;
  if (r->specials) {
    const uint64_t ss = r->spec_seed;
    if (unit(ss ^ 0xC0FFEEull, i) < 0.01) {
      const int which = (int)(sm64(ss ^ 0xBEEFull, i) % 9ull);
      static const uint64_t sp[9] = {0x0ull, 0x8000000000000000ull, 0x7ff0000000000000ull, 0xfff0000000000000ull,
                                     0x7ff8000000000000ull, 0x1ull, 0x0ull, 0x7fefffffffffffffull,
                                     0xffefffffffffffffull};
      v = which == 6 ? from_bits((sm64(ss ^ 0xD00Dull, i) & ((1ull << 52) - 1)) | 1ull) : from_bits(sp[which]);
    }
  }
  return v;
}

void vg_fill(const vem_recipe* r, void* out, size_t n, uint64_t offset) {
  if (r->f32) {
    float* o = (float*)out;
#pragma omp parallel for schedule(static)
    for (size_t j = 0; j < n; j++) o[j] = (float)element(r, offset + j);
  } else {
    double* o = (double*)out;
#pragma omp parallel for schedule(static)
    for (size_t j = 0; j < n; j++) o[j] = element(r, offset + j);
  }
}

/* sums[c - (offset >> log2chunk)] += chunk contributions of p[0..n) */
void vg_checksum(const void* p, size_t n, int elem_bytes, uint64_t offset, int log2chunk, uint64_t* sums) {
  const uint64_t c0 = offset >> log2chunk;
  size_t j = 0;
  while (j < n) {
    const uint64_t g = offset + j;
    const uint64_t c = g >> log2chunk;
    const uint64_t end = (c + 1) << log2chunk;
    const size_t m = (size_t)((end - g) < (n - j) ? (end - g) : (n - j));
    uint64_t acc = 0;
    if (elem_bytes == 8) {
      const uint64_t* q = (const uint64_t*)p + j;
#pragma omp parallel for schedule(static) reduction(+ : acc)
      for (size_t k = 0; k < m; k++) acc += fmix64(q[k] ^ ((g + k) * kGolden));
    } else {
      const uint32_t* q = (const uint32_t*)p + j;
#pragma omp parallel for schedule(static) reduction(+ : acc)
      for (size_t k = 0; k < m; k++) acc += fmix64((uint64_t)q[k] ^ ((g + k) * kGolden));
    }
    sums[c - c0] += acc;
    j += m;
  }
}
