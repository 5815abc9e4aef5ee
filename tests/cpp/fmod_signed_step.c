/* CPU model of the device fmod schedule (vem_kernels.cu fmod_pend_setup /
 * fmod_stepn50 / fmod_pend_finish; vem_math.cuh fmod_stepn_rs): signed
 * remainders, Q = rint(rs * RN(1/md)), V = fma(-Q, md, rs), one r < 0 fix-up
 * at the end.  Test infrastructure: checks every step's invariant (|V| <= md,
 * V exact: rs - Q md == V in binary128) and the result against glibc fmod.
 * Build: gcc -O2 -ffp-contract=off fmod_signed_step.c -lm -lquadmath */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static uint64_t sm64(uint64_t *s) {
  uint64_t z = (*s += 0x9e3779b97f4a7c15ull);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}
static double from_bits(uint64_t b) { double d; memcpy(&d, &b, 8); return d; }
static uint64_t to_bits(double d) { uint64_t b; memcpy(&b, &d, 8); return b; }

static long bad_steps, max_steps;

static double step(double rs, double md, double rmd) {
  double q = rint(rs * rmd);
  double v = fma(-q, md, rs);
  /* exactness: rs - q md computed in binary128 (113 bits hold the 106-bit product) */
  __float128 ex = (__float128)rs - (__float128)q * (__float128)md;
  if ((__float128)v != ex || fabs(v) > md) bad_steps++;
  return v;
}

/* |x| > |y| > 0, finite */
static double model(double x, double y) {
  double n = fabs(x), d = fabs(y);
  int en, ed;
  double mn = frexp(n, &en) * 2.0, md = frexp(d, &ed) * 2.0; /* [1, 2) */
  en--, ed--;
  int E = en - ed;
  double rmd = 1.0 / md;
  int steps = E == 0 ? 0 : (E - 1) / 50;
  double r = step(ldexp(mn, E - 50 * steps), md, rmd);
  double rmd50 = rmd * 0x1p50;
  for (int k = 0; k < steps; k++) {
    double q = rint(r * rmd50);
    double rs = r * 0x1p50;
    if (q != rint(rs * rmd)) bad_steps++; /* r*rmd50 == rs*rmd */
    r = step(rs, md, rmd);
  }
  if (steps > max_steps) max_steps = steps;
  if (r < 0.0) r += md;
  return copysign(ldexp(r, ed), x);
}

int main(int argc, char **argv) {
  long n = argc > 1 ? atol(argv[1]) : 2000000;
  uint64_t s = 0x5EEF0F00ull;
  long mism = 0, pend = 0;
  for (long i = 0; i < n; i++) {
    double x, y;
    int mode = (int)(i % 4);
    if (mode == 0) { /* random bit patterns */
      x = from_bits(sm64(&s));
      y = from_bits(sm64(&s));
    } else if (mode == 1) { /* config-4-like: log-uniform magnitudes */
      double u = (sm64(&s) >> 11) * 0x1p-53, v = (sm64(&s) >> 11) * 0x1p-53;
      x = pow(10.0, -300.0 + 600.0 * u);
      y = pow(10.0, -300.0 + 600.0 * v);
      if (sm64(&s) & 1) x = -x;
      if (sm64(&s) & 1) y = -y;
    } else if (mode == 2) { /* worst divisor mantissas: md near 1 and near 2 */
      uint64_t m = sm64(&s);
      y = from_bits((to_bits(1.0 + (m & 1 ? 0x1p-52 * (m >> 60) : 1.0 - 0x1p-52 * (1 + (m >> 60))))) +
                    ((uint64_t)((sm64(&s) % 1900)) << 52) - (950ull << 52));
      x = from_bits((sm64(&s) & 0x000fffffffffffffull) | ((uint64_t)(1 + sm64(&s) % 2046) << 52));
    } else { /* subnormal operands */
      x = from_bits(sm64(&s) >> (sm64(&s) % 12));
      y = from_bits(sm64(&s) >> (12 + sm64(&s) % 52));
    }
    if (!isfinite(x) || !isfinite(y) || y == 0.0 || !(fabs(x) > fabs(y))) continue;
    pend++;
    double a = model(x, y), b = fmod(x, y);
    if (to_bits(a) != to_bits(b)) {
      if (mism < 5) printf("mismatch x=%a y=%a model=%a glibc=%a\n", x, y, a, b);
      mism++;
    }
  }
  printf("pending=%ld mismatches=%ld bad_steps=%ld max_steps=%ld\n", pend, mism, bad_steps, max_steps);
  return (mism || bad_steps) ? 1 : 0;
}
