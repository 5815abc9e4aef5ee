/* Exhaustive margin check for the binary32 integer Payne-Hanek table
 * (tools/genphtable.py, csrc/vem_ph_tables.h): for every exponent entry and
 * every 24-bit mantissa M in [2^23, 2^24), forms p = M*W(E) mod 2^128 and the
 * signed fraction s = p << 2 (value s/2^128 in [-1/2, 1/2)), and reports the
 * largest number of leading zeros of |s|.  The kernels (csrc/vem_math.cuh
 * ph_f) rely on that being <= 29 (the leading one lies in the top 32-bit word).
 * Build/run:  gcc -O2 -I paper_2001_09258_b200/csrc tools/phf_margin.c -o /tmp/phf_margin && /tmp/phf_margin
 * (~3 s).  Measured: worst 29 leading zeros (E = 11, M = 10741887). */
#include <stdint.h>
#include <stdio.h>

#include "vem_ph_tables.h"

static const uint32_t W[4 * VEM_PH_F_ENTRIES] = {VEM_PH_F_INIT};

int main(void) {
  int worst = 0;
  for (int e = 0; e < VEM_PH_F_ENTRIES; e++) {
    const uint32_t* w = W + 4 * e;
    unsigned __int128 wv = ((unsigned __int128)(((uint64_t)w[3] << 32) | w[2]) << 64) | (((uint64_t)w[1] << 32) | w[0]);
    int elz = 0;
    uint32_t wm = 0;
    for (uint32_t M = 1u << 23; M < (1u << 24); M++) {
      unsigned __int128 s = (wv * M) << 2;
      if ((int64_t)(uint64_t)(s >> 64) < 0) s = ~s;
      uint32_t s3 = (uint32_t)(s >> 96);
      int lz = s3 ? __builtin_clz(s3) : 32;
      if (lz > elz) { elz = lz; wm = M; }
    }
    if (elz > worst) {
      worst = elz;
      printf("E=%d: %d leading zeros (M=%u)\n", e + VEM_PH_F_EMIN, elz, wm);
    }
  }
  printf("worst %d (need <= 29)\n", worst);
  return worst <= 29 ? 0 : 1;
}
