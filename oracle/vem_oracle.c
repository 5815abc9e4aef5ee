/* TEST INFRASTRUCTURE ONLY -- the CPU oracle.
 *
 * A plain-C restatement of the batched elementwise math path, used solely by
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference leg, as the checker.  The product (libvem.so, CUDA sm_100a) never
 * links or calls anything here, and there is no CPU fallback in the product.
 *
 * Every function follows the same operation order as the CUDA kernel of the
 * same name, so GPU results must be BIT-IDENTICAL to this file (the
 * "deterministic variant" of the north star).  Independently of that, each
 * function is checked against MPFR 4.2.1 for its ULP bound (tests/), and:
 *   - the reduction (cw1 / cw2 / ph / trig_reduce) is checked bit-for-bit
 *     against the reference's own code compiled from /root/reference
 *     (oracle/_ref, see ref_build.py): reduction.hpp:147-212, ddarith.hpp;
 *   - fmod is checked bit-for-bit against glibc fmod/fmodf (exact);
 *   - the Payne-Hanek table digests are pinned (tests/golden).
 *
 * Build: gcc -O2 -ffp-contract=off -mfma -fopenmp (oracle/Makefile).
 * Contraction MUST stay off: every fused op below is an explicit fma().
 *
 * Citations: backend.hpp / ddarith.hpp / reduction.hpp / constants.hpp are
 * /root/reference/proj/core/include/vem/; SPEC.md / PAPER.md at the root of
 * /root/reference.
 */
#include <math.h>
#include <stdint.h>
#include <stddef.h>
#include <string.h>

#include "vem_coeffs.h"
#include "vem_ph_tables.h"
#include "vem_log_tables.h"

typedef struct { double hi, lo; } dd_t;

/* ------------------------------------------------------------------ bits */
static inline uint64_t bits_d(double x) { uint64_t u; memcpy(&u, &x, 8); return u; }
static inline double from_bits_d(uint64_t u) { double x; memcpy(&x, &u, 8); return x; }
static inline uint32_t bits_f(float x) { uint32_t u; memcpy(&u, &x, 4); return u; }
static inline float from_bits_f(uint32_t u) { float x; memcpy(&x, &u, 4); return x; }

#define CANON_NAN_D 0x7ff8000000000000ull
#define CANON_NAN_F 0x7fc00000u
static inline double canon_d(double y) { return (y != y) ? from_bits_d(CANON_NAN_D) : y; }
static inline float canon_f(float y) { return (y != y) ? from_bits_f(CANON_NAN_F) : y; }

/* constants.hpp:14-58 (values reused; they are the reference's frozen limbs) */
#define K_PIO2_QD0 0x1.921fb54442d18p+0
#define K_PIO2_QD1 0x1.1a62633145c07p-54
#define K_PIO2_QD2 -0x1.f1976b7ed8fbcp-110
#define K_PIO2_QD3 0x1.4cf98e804177dp-164
#define K_TWO_OVER_PI 0x1.45f306dc9c883p-1
#define K_CW1_P0 0x1.921fb54442d20p+0
#define K_CW1_T1 -0x1.ee59d9cceba40p-50
#define K_CW1_T2 0x1.b839a252049c1p-104
#define K_CW2_A 0x1.921fb58000000p+0
#define K_CW2_B -0x1.dde9740000000p-27
#define K_CW2_C 0x1.1a62630000000p-54
#define K_CW2_D1 0x1.8a2e03707344ap-81
#define K_CW2_D2 0x1.024e088a67cc7p-135
#define K_INV_LN2 0x1.71547652b82fep+0
#define K_EXP_L1 0x1.62e42fefa3800p-1
#define K_EXP_L2 0x1.ef35793c76730p-45
#define K_LN2_HI 0x1.62e42fefa39efp-1
#define K_LN2_LO 0x1.abc9e3b39803fp-56
#define K_EXP_OVF 0x1.62e42fefa39efp+9
#define K_EXP_UNF -0x1.74910d52d3051p+9
#define K_CW1_MAX 15.0
#define K_CW2_MAX 1e14
#define K_FOUR_THIRDS 0x1.5555555555555p+0

static const double PH_D[4 * VEM_PH_D_ENTRIES] = {VEM_PH_D_INIT};
static const uint64_t PH_DI[4 * VEM_PH_DI_ENTRIES] = {VEM_PH_DI_INIT};
static const double LOGT_INVC[256] = {VEM_LOGT_INVC_INIT};
static const double LOGT_HI[256] = {VEM_LOGT_HI_INIT};
static const double LOGT_LO[256] = {VEM_LOGT_LO_INIT};
static const double EXPT_HI[128] = {VEM_EXPT_HI_INIT};
static const double EXPT_LO[128] = {VEM_EXPT_LO_INIT};
static const double LOGTF_HI[256] = {VEM_LOGTF_HI_INIT};
static const float LOGTF_INVC[256] = {VEM_LOGTF_INVC_INIT};

/* ------------------------------------------- primitives (backend.hpp) */
/* backend.hpp:47-52 round_ta: nearest integer, ties away from zero */
static inline double round_ta(double x) {
  double t = trunc(x);
  double f = x - t;
  double up = t + (x < 0 ? -1.0 : 1.0);
  return (f >= 0.5 || f <= -0.5) ? up : t;
}
/* backend.hpp:133-138 ldexp2 (two half-step power-of-two multiplies) */
static inline double pow2_bits(int64_t e) { return from_bits_d((uint64_t)(e + 1023) << 52); }
static inline double ldexp2(double x, int64_t e) {
  e = e > 2046 ? 2046 : (e < -2044 ? -2044 : e);
  int64_t h = e >> 1;
  return (x * pow2_bits(h)) * pow2_bits(e - h);
}
/* backend.hpp:381-384 mulsign */
static inline double mulsign(double x, double s) {
  return from_bits_d(bits_d(x) ^ (bits_d(s) & 0x8000000000000000ull));
}
static inline double copysign_b(double m, double s) {
  return from_bits_d((bits_d(m) & 0x7fffffffffffffffull) | (bits_d(s) & 0x8000000000000000ull));
}
static inline double neg_if(double y, int c) {
  return from_bits_d(bits_d(y) ^ ((uint64_t)(c != 0) << 63));
}
/* nearest integer of a*b by one fma against 1.5*2^52 (ties-to-even of the
 * exactly rounded product+shift); |a*b| < 2^31.  k = the low word. */
#define K_SHIFT 0x1.8p52
static inline double rint_fma(double a, double b, int32_t* k) {
  double u = fma(a, b, K_SHIFT);
  *k = (int32_t)(uint32_t)bits_d(u);
  return u - K_SHIFT;
}
/* backend.hpp:418-423 toward_zero for positive finite x */
static inline double toward0_pos(double x) { return from_bits_d(bits_d(x) - 1); }

/* ------------------------------------------------- DD (ddarith.hpp) */
static inline dd_t two_sum(double a, double b) { /* ddarith.hpp:29-35 */
  double s = a + b, v = s - a;
  dd_t r = {s, (a - (s - v)) + (b - v)};
  return r;
}
static inline dd_t two_sum_fast(double a, double b) { /* ddarith.hpp:39-44 */
  double s = a + b;
  dd_t r = {s, b - (s - a)};
  return r;
}
static inline dd_t two_prod(double a, double b) { /* ddarith.hpp:51-56 (FMA) */
  double p = a * b;
  dd_t r = {p, fma(a, b, -p)};
  return r;
}
static inline dd_t dd_add2(dd_t x, dd_t y) { /* ddarith.hpp:111-117 */
  double s = x.hi + y.hi, v = s - x.hi;
  double e = (x.hi - (s - v)) + (y.hi - v);
  dd_t r = {s, e + (x.lo + y.lo)};
  return r;
}
static inline dd_t dd_add2_d(dd_t x, double y) { /* ddarith.hpp:120-126 */
  double s = x.hi + y, v = s - x.hi;
  double e = (x.hi - (s - v)) + (y - v);
  dd_t r = {s, e + x.lo};
  return r;
}
static inline dd_t dd_mul(dd_t x, dd_t y) { /* ddarith.hpp:163-170 (FMA) */
  double p = x.hi * y.hi;
  double e = fma(x.hi, y.hi, -p);
  e = fma(x.hi, y.lo, e);
  e = fma(x.lo, y.hi, e);
  dd_t r = {p, e};
  return r;
}
static inline dd_t dd_mul_d(dd_t x, double y) { /* ddarith.hpp:178-184 (FMA) */
  double p = x.hi * y;
  double e = fma(x.hi, y, -p);
  e = fma(x.lo, y, e);
  dd_t r = {p, e};
  return r;
}
static inline dd_t dd_squ(dd_t x) { /* ddarith.hpp:197-203 (FMA) */
  double p = x.hi * x.hi;
  double e = fma(x.hi, x.hi, -p);
  e = fma(x.hi + x.hi, x.lo, e);
  dd_t r = {p, e};
  return r;
}
static inline dd_t dd_div(dd_t x, dd_t y) { /* ddarith.hpp:220-228 (FMA) */
  double t = 1.0 / y.hi;
  double q = x.hi * t;
  double u = fma(t, x.hi, -q);
  double v = fma(y.lo, -t, fma(y.hi, -t, 1.0));
  dd_t r = {q, fma(q, v, fma(x.lo, t, u))};
  return r;
}
static inline dd_t dd_normalize(dd_t x) { return two_sum_fast(x.hi, x.lo); } /* ddarith.hpp:103 */

/* Polynomial evaluation: Horner, c[0] + x*(c[1] + x*(...)).  The paper uses
 * Estrin's scheme to cut FMA latency on out-of-order CPUs;
 * on the GPU the kernels are throughput-bound with thousands of independent
 * lanes in flight, and Horner issues the fewest instructions (n-1 FMAs, one
 * constant-bank operand each, no power precomputation).  The CUDA kernels
 * (vem_math.cuh: poly) use the identical order. */
static inline double poly(const double* c, int n, double x) {
  double acc = c[n - 1];
  for (int i = n - 2; i >= 0; i--) acc = fma(acc, x, c[i]);
  return acc;
}

/* ============================================ trig reduction (f64) */
typedef struct { double hi, lo; int q; } red_t;

/* reduction.hpp:148-159 -- Cody-Waite level 1, |x| <= 15 */
static red_t cw1(double x) {
  double qd = round_ta(x * K_TWO_OVER_PI);
  double r0 = fma(qd, -K_CW1_P0, x);
  dd_t tail = two_prod(qd, -K_CW1_T1);
  tail.lo = fma(qd, -K_CW1_T2, tail.lo);
  dd_t r0d = {r0, 0.0};
  dd_t r = dd_normalize(dd_add2(r0d, tail));
  red_t o = {r.hi, r.lo, (int)((int64_t)qd & 3)};
  return o;
}

/* reduction.hpp:163-178 -- Cody-Waite level 2, |x| <= 1e14 */
static red_t cw2(double x) {
  double t = x * K_TWO_OVER_PI;
  double qh = trunc(t * 0x1p-24);
  qh = qh * 0x1p24;
  double ql = round_ta(t - qh);
  double r = x;
  r = fma(qh, -K_CW2_A, r);
  r = fma(ql, -K_CW2_A, r);
  r = fma(qh, -K_CW2_B, r);
  r = fma(ql, -K_CW2_B, r);
  dd_t rd = {r, 0.0};
  dd_t acc = dd_add2(rd, two_prod(qh, -K_CW2_C));
  acc = dd_add2(acc, two_prod(ql, -K_CW2_C));
  double qs = qh + ql;
  dd_t dtail = two_prod(qs, -K_CW2_D1);
  dtail.lo = fma(qs, -K_CW2_D2, dtail.lo);
  acc = dd_add2(acc, dtail);
  acc = dd_normalize(acc);
  red_t o = {acc.hi, acc.lo, (int)((int64_t)ql & 3)};
  return o;
}

/* reduction.hpp:35-43 rfrac with quadrant accumulation */
static inline dd_t rfrac_q(dd_t a, int64_t* q) {
  double rh = round_ta(a.hi);
  a.hi = a.hi - rh;
  *q += (int64_t)rh;
  double rl = round_ta(a.lo);
  a.lo = a.lo - rl;
  *q += (int64_t)rl;
  return a;
}

/* reduction.hpp:89-137 Payne-Hanek, REPAIRED:
 * mod-4 table (tools/genphtable.py) + two_sum renormalisation after each
 * rfrac.  Non-finite x are computed on a sanitised 0 and replaced by NaN at
 * the end (the reference's `bad` select, reduction.hpp:131-135). */
static red_t ph(double x_in) {
  int bad = !(fabs(x_in) <= 1.7976931348623157e308);
  double x = bad ? 0.0 : x_in;
  double a = fabs(x);
  int64_t er = (int64_t)((bits_d(a) >> 52) & 0x7ff);
  int64_t idx = er - 1023;
  idx = (0 > idx) ? 0 : idx;
  idx = (idx > 1023) ? 1023 : idx;
  double m = ldexp2(a, 52 - idx);
  const double* f = PH_D + (idx << 2);
  int64_t q = 0;
  dd_t u = two_prod(m, f[0]);
  u = rfrac_q(u, &q);
  u = two_sum(u.hi, u.lo);
  u = dd_add2(u, two_prod(m, f[1]));
  u = rfrac_q(u, &q);
  u = two_sum(u.hi, u.lo);
  u = dd_add2(u, two_prod(m, f[2]));
  u = rfrac_q(u, &q);
  u = two_sum(u.hi, u.lo);
  u = dd_add2(u, two_prod(m, f[3]));
  double qv = round_ta(u.hi + u.lo);
  u.hi = u.hi - qv;
  q += (int64_t)qv;
  double ql = round_ta(u.lo);
  u.lo = u.lo - ql;
  q += (int64_t)ql;
  u = dd_normalize(u);
  /* reduction.hpp:57-69 mul_pio2_qd */
  double p = u.hi * K_PIO2_QD0;
  double e = fma(u.hi, K_PIO2_QD0, -p);
  e = fma(u.hi, K_PIO2_QD1, e);
  e = fma(u.lo, K_PIO2_QD0, e);
  e = fma(u.hi, K_PIO2_QD2, e);
  e = fma(u.lo, K_PIO2_QD1, e);
  e = fma(u.hi, K_PIO2_QD3, e);
  e = fma(u.lo, K_PIO2_QD2, e);
  double rh = mulsign(p, x), rl = mulsign(e, x);
  if (x < 0.0) q = 0 - q;
  red_t o;
  if (bad) {
    o.hi = from_bits_d(CANON_NAN_D);
    o.lo = from_bits_d(CANON_NAN_D);
    o.q = 0;
  } else {
    o.hi = rh;
    o.lo = rl;
    o.q = (int)(q & 3);
  }
  return o;
}

/* Integer Payne-Hanek for binary64 (own design; SURVEY.md §8(a) a9 allows
 * "an own design validated to 2^-60 abs"; the function kernels use it, the
 * reference algorithm above stays the parity anchor of vem_ph_reduce_d).
 * |x| = M 2^E, M in [2^52, 2^53): P = M W(E) mod 2^192 with
 * W(E) = floor((2^E 2/pi mod 4) 2^190) (tools/genphtable.py) is x 2/pi mod 4
 * in units of 2^-190, short by less than M units (2^-137).  Adding half a
 * unit of the quadrant (2^189) and taking the top two bits gives
 * q = round(x 2/pi) mod 4.  The centred fraction F = frac - [frac >= 1/2]
 * is summed from P's 32-bit words p5 (30 fraction bits) .. p1 as doubles
 * (each exact) with fast two-sums: every partial sum is 0 or at least 2^-63
 * in magnitude, because binary64 never comes closer than ~2^-61 (relative)
 * to a multiple of pi/2, so every step is exact and only the error terms'
 * sum rounds (~2^-104 relative).  r = F (pi/2) as p + e with pi/2 = C0 + C1
 * and the sign of x folded into the constants.  r keeps >= 70 correct bits
 * (tests check it against mpmath, worst cases included).  |x| < 1/2: r = x,
 * q = 0; non-finite x: NaN. */
static red_t ph_int192(double x) {
  const uint64_t b = bits_d(x), ab = b & 0x7fffffffffffffffull;
  red_t o;
  if (ab >= 0x7ff0000000000000ull) {
    o.hi = from_bits_d(CANON_NAN_D);
    o.lo = from_bits_d(CANON_NAN_D);
    o.q = 0;
    return o;
  }
  const int ue = (int)(ab >> 52) - 1023;
  if (ue < VEM_PH_DI_UEMIN) {
    o.hi = x;
    o.lo = 0.0;
    o.q = 0;
    return o;
  }
  const uint64_t M = (ab & 0x000fffffffffffffull) | 0x0010000000000000ull;
  const uint64_t* w = PH_DI + 4 * (ue - VEM_PH_DI_UEMIN);
  const unsigned __int128 t0 = (unsigned __int128)M * w[0];
  const unsigned __int128 t1 = (unsigned __int128)M * w[1];
  const uint64_t P0 = (uint64_t)t0;
  const uint64_t h0 = (uint64_t)(t0 >> 64), l1 = (uint64_t)t1, h1 = (uint64_t)(t1 >> 64);
  const uint64_t P1 = h0 + l1;
  const uint64_t P2 = M * w[2] + h1 + (uint64_t)(P1 < l1);
  const uint32_t p5 = (uint32_t)(P2 >> 32), p4 = (uint32_t)P2;
  const uint32_t p3 = (uint32_t)(P1 >> 32), p2 = (uint32_t)P1, p1 = (uint32_t)(P0 >> 32);
  int q = (int)((p5 + 0x20000000u) >> 30);
  const uint32_t f5 = p5 & 0x3fffffffu;
  const double s0 = fma((double)f5, 0x1p-30, -(double)(f5 >> 29));
  double t = (double)p4 * 0x1p-62;
  const double s1 = s0 + t;
  double e = t - (s1 - s0);
  t = (double)p3 * 0x1p-94;
  const double s2 = s1 + t;
  e = e + (t - (s2 - s1));
  t = (double)p2 * 0x1p-126;
  const double s3 = s2 + t;
  e = e + (t - (s3 - s2));
  t = (double)p1 * 0x1p-158;
  const double s4 = s3 + t;
  e = e + (t - (s4 - s3));
  const double fh = s4 + e;
  const double fl = e - (fh - s4);
  const double c0 = (b >> 63) ? -K_PIO2_QD0 : K_PIO2_QD0;
  const double c1 = (b >> 63) ? -K_PIO2_QD1 : K_PIO2_QD1;
  const double p = fh * c0;
  double ee = fma(fh, c0, -p);
  ee = fma(fh, c1, ee);
  ee = fma(fl, c0, ee);
  if (b >> 63) q = -q;
  o.hi = p;
  o.lo = ee;
  o.q = q & 3;
  return o;
}

/* Two-level integer Payne-Hanek (the functions' binary64 reduction).
 * Fast level: the top 128 bits of the 192-bit window, P = M * W128 mod 2^128
 * (quadrant units: LSB 2^-126); the fraction's 126 bits are cut into three
 * exactly convertible chunks c0 (53 bits, centred in integer arithmetic),
 * c1 (53), c2 (20) and summed with one Fast2Sum (|c0| is 0 or >= 1 > c1 in
 * units of 2^-53).  The missing M * w[0] term is < 2^-73 quadrant units, so
 * whenever |F| >= 2^-11 the result is within 2^-62 relative; otherwise
 * (probability ~2^-10 for random arguments) the full 192-bit form ph_int192
 * recomputes it.  The GPU kernels (vem_math.cuh ph_int) perform the same
 * operations in the same order. */
static red_t ph_int(double x) {
  const uint64_t b = bits_d(x), ab = b & 0x7fffffffffffffffull;
  const int ue = (int)(ab >> 52) - 1023;
  if (ab >= 0x7ff0000000000000ull || ue < VEM_PH_DI_UEMIN) return ph_int192(x);
  const uint64_t M = (ab & 0x000fffffffffffffull) | 0x0010000000000000ull;
  const uint64_t* w = PH_DI + 4 * (ue - VEM_PH_DI_UEMIN);
  const unsigned __int128 u = (unsigned __int128)M * w[1];
  const uint64_t T0 = (uint64_t)u;
  const uint64_t T1 = M * w[2] + (uint64_t)(u >> 64);
  const uint32_t t3 = (uint32_t)(T1 >> 32), t2 = (uint32_t)T1, t1 = (uint32_t)(T0 >> 32);
  int q = (int)((t3 + 0x20000000u) >> 30);
  const uint32_t f = t3 & 0x3fffffffu;
  /* fraction bits below 2^-73 are noise (the dropped M*w0 term): two chunks,
   * 53 bits centred + the next 32 (weights down to 2^-85), units of 2^-53 */
  const int64_t c0 = (int64_t)(((uint64_t)f << 23) | (t2 >> 9)) - ((f >> 29) ? (1ll << 53) : 0);
  const uint32_t c1 = (t2 << 23) | (t1 >> 9);
  const double S0 = (double)c0;
  const double tb = (double)c1 * 0x1p-32;
  const double fh = S0 + tb;           /* |S0| is 0 or >= 1 > tb: Fast2Sum, exact pair */
  const double fl = tb - (fh - S0);
  if (fabs(fh) < 0x1p42) return ph_int192(x);
  const double c0p = (b >> 63) ? -K_PIO2_QD0 * 0x1p-53 : K_PIO2_QD0 * 0x1p-53;
  const double c1p = (b >> 63) ? -K_PIO2_QD1 * 0x1p-53 : K_PIO2_QD1 * 0x1p-53;
  const double p = fh * c0p;
  double ee = fma(fh, c0p, -p);
  ee = fma(fh, c1p, ee);
  ee = fma(fl, c0p, ee);
  if (b >> 63) q = -q;
  red_t o;
  o.hi = p;
  o.lo = ee;
  o.q = q & 3;
  return o;
}

/* reduction.hpp:189-206, deterministic policy, per lane */
static red_t trig_reduce(double x) {
  double ax = fabs(x);
  if (ax <= K_CW1_MAX) return cw1(x);
  if (ax <= K_CW2_MAX) return cw2(x);
  return ph(x);
}

/* the functions' selector: CW1 / CW2 (the reference's, bit for bit) and the
 * integer Payne-Hanek above for |x| > 1e14 */
static red_t trig_reduce_fn(double x) {
  double ax = fabs(x);
  if (ax <= K_CW1_MAX) return cw1(x);
  if (ax <= K_CW2_MAX) return cw2(x);
  return ph_int(x);
}

/* ======================================================= f64 kernels */
static const double C_SIN_D[] = VEM_SIN_D_ARR;
static const double C_COS_D[] = VEM_COS_D_ARR;
static const double C_TAN_D[] = VEM_TAN_D_ARR;
static const double C_ATAN_D[] = VEM_ATAN_D_ARR;
static const double C_EXP_D[] = VEM_EXP_D_ARR;
static const double C_EXP_D_U35[] = VEM_EXP_D_U35_ARR;

/* sin/cos core on the reduced argument r = rh + rl, |r| <= 0.80, using a
 * per-lane SELECTED polynomial (sin form for even effective quadrant, cos
 * form for odd) -- branch-free on the GPU (SPEC.md:470 leaves the cos
 * recipe open).  `cosform` picks the cos polynomial. */
static double sincos_core_d(double rh, double rl, int cosform) {
  double c[VEM_SIN_D_N];
  for (int i = 0; i < VEM_SIN_D_N; i++) c[i] = cosform ? C_COS_D[i] : C_SIN_D[i];
  double z = rh * rh;
  double P = poly(c, VEM_SIN_D_N, z);
  /* sin form: rh + (rl - rl*z/2 + rh*z*P) */
  double As = rh, Bs = 0.0, Ms = rh * z, Ts = fma(-0.5 * z, rl, rl);
  /* cos form: w + (((1-w) - z/2) + (z^2*P - (zl/2 + rh*rl))), w = 1 - z/2 */
  double zl = fma(rh, rh, -z);
  double hz = 0.5 * z;
  double w = 1.0 - hz;
  double Ac = w, Bc = (1.0 - w) - hz, Mc = z * z, Tc = -fma(0.5, zl, rh * rl);
  double A = cosform ? Ac : As, B = cosform ? Bc : Bs, M = cosform ? Mc : Ms, T = cosform ? Tc : Ts;
  return A + (B + fma(M, P, T));
}

double vo_sin_d_u10(double x) {
  red_t r = trig_reduce_fn(x);
  double y = sincos_core_d(r.hi, r.lo, r.q & 1);
  y = neg_if(y, r.q & 2);
  y = (x == 0.0) ? x : y;
  return canon_d(y);
}
double vo_cos_d_u10(double x) {
  red_t r = trig_reduce_fn(x);
  double y = sincos_core_d(r.hi, r.lo, (r.q & 1) ^ 1);
  y = neg_if(y, (r.q + 1) & 2);
  return canon_d(y);
}
double vo_sin_d_u10_ph(double x) {
  red_t r = ph_int(x);
  double y = sincos_core_d(r.hi, r.lo, r.q & 1);
  y = neg_if(y, r.q & 2);
  y = (x == 0.0) ? x : y;
  return canon_d(y);
}
double vo_cos_d_u10_ph(double x) {
  red_t r = ph_int(x);
  double y = sincos_core_d(r.hi, r.lo, (r.q & 1) ^ 1);
  y = neg_if(y, (r.q + 1) & 2);
  return canon_d(y);
}

/* tan: half-angle: t = tan(r/2), tan r = 2t/(1-t^2),
 * -cot r = -(1-t^2)/(2t); one DD division for both quadrant parities. */
static double tan_core_d(double rh, double rl, int odd) {
  double hh = rh * 0.5, hl = rl * 0.5;
  double z = hh * hh;
  double P = poly(C_TAN_D, VEM_TAN_D_N, z);
  double corr = fma(hh * z, P, fma(hl, z, hl));
  dd_t t = two_sum_fast(hh, corr);
  dd_t t2 = dd_squ(t);
  dd_t den = two_sum(1.0, -t2.hi);
  den.lo = den.lo - t2.lo;
  dd_t num = {t.hi * 2.0, t.lo * 2.0};
  dd_t X, Y;
  if (odd) {
    X.hi = -den.hi; X.lo = -den.lo; Y = num;
  } else {
    X = num; Y = den;
  }
  dd_t q = dd_div(X, Y);
  return q.hi + q.lo;
}
double vo_tan_d_u10(double x) {
  red_t r = trig_reduce_fn(x);
  double y = tan_core_d(r.hi, r.lo, r.q & 1);
  y = (fabs(x) < 0x1p-27) ? x : y;
  return canon_d(y);
}
double vo_tan_d_u10_ph(double x) {
  red_t r = ph_int(x);
  double y = tan_core_d(r.hi, r.lo, r.q & 1);
  y = (fabs(x) < 0x1p-27) ? x : y;
  return canon_d(y);
}

/* atan (restructured for one division): fold |x| into
 * |b| <= tan(pi/8) with b = x, (x-1)/(x+1) or -1/x (offsets 0, pi/4, pi/2),
 * one DD division (ddarith.hpp:220-228) covers all three cases, 12-term odd
 * polynomial, offset added in DD.  The paper's single 1/x fold with a
 * 20-term polynomial on [0,1] measured 1.29 ulp with a binary64 assembly;
 * see DESIGN.md §4. */
#define K_TAN_PI8 0x1.a827999fcef32p-2
#define K_TAN_3PI8 0x1.3504f333f9de6p+1
#define K_PIO4_HI 0x1.921fb54442d18p-1
#define K_PIO4_LO 0x1.1a62633145c07p-55
double vo_atan_d_u10(double x) {
  double a = fabs(x);
  int c1 = a > K_TAN_PI8;
  int c2 = a > K_TAN_3PI8;
  dd_t ns = two_sum(a, -1.0), ds = two_sum(a, 1.0);
  dd_t nn, dn;
  nn.hi = c2 ? -1.0 : (c1 ? ns.hi : a);
  nn.lo = c2 ? 0.0 : (c1 ? ns.lo : 0.0);
  /* |x| >= 2^60 gives RN(pi/2 - 1/|x|) = pi/2 exactly like |x| = 2^60, and
   * keeps 1/|x| normal (a subnormal reciprocal takes the GPU division's
   * slow path) */
  dn.hi = c2 ? fmin(a, 0x1p60) : (c1 ? ds.hi : 1.0);
  dn.lo = c2 ? 0.0 : (c1 ? ds.lo : 0.0);
  dd_t b = dd_div(nn, dn);
  double z = b.hi * b.hi;
  double P = poly(C_ATAN_D, VEM_ATAN_D_N, z);
  double corr = fma(b.hi * z, P, fma(-b.lo, z, b.lo));
  double offh = c2 ? K_PIO2_QD0 : (c1 ? K_PIO4_HI : 0.0);
  double offl = c2 ? K_PIO2_QD1 : (c1 ? K_PIO4_LO : 0.0);
  dd_t s = two_sum(offh, b.hi);
  double y = s.hi + (s.lo + (offl + corr));
  y = (a == INFINITY) ? K_PIO2_QD0 : y;
  y = copysign_b(y, x);
  return canon_d(y);
}

/* exp: k = rint(x/ln2), r = x - k*L1 - k*L2
 * (constants.hpp:44-46), 13-term polynomial (u10) / 12-term (u35), no DD
 * (SPEC.md:406).  Fast path |x| < 708: the result is normal, so 2^k is applied
 * by adding k to the exponent field (== ldexp2, exact).  Slow path: ldexp2
 * (backend.hpp:133-138, single rounding into subnormals) and saturation
 * (constants.hpp:53-54); NaN in, canonical NaN out. */
#define EXP_FAST_HI 0x40862000u /* |x| < 708 */
static inline double exp_poly_d(double xs, const double* c, int n, int u10, int32_t* k_out) {
  double kd = rint_fma(xs, K_INV_LN2, k_out);
  double r1 = fma(kd, -K_EXP_L1, xs);
  double r = fma(kd, -K_EXP_L2, r1);
  double P = poly(c, n, r);
  double y;
  if (u10) {
    double rl = fma(-kd, K_EXP_L2, r1 - r);
    double s = 1.0 + r;
    double se = (1.0 - s) + r;
    y = s + (se + fma(r * r, P, rl));
  } else {
    y = 1.0 + fma(r * r, P, r);
  }
  return y;
}
static double exp_core_d(double x, const double* c, int n, int u10) {
  uint32_t hx = (uint32_t)(bits_d(x) >> 32) & 0x7fffffffu;
  int32_t k;
  if (hx < EXP_FAST_HI) {
    double y = exp_poly_d(x, c, n, u10, &k);
    return from_bits_d(bits_d(y) + ((uint64_t)(int64_t)k << 52));
  }
  if (x > K_EXP_OVF) return INFINITY;       /* saturation, constants.hpp:53-54 */
  if (x < K_EXP_UNF) return 0.0;
  if (x != x) return from_bits_d(CANON_NAN_D);
  double y = exp_poly_d(x, c, n, u10, &k);  /* 708 <= |x|: ldexp2 rounds once */
  return ldexp2(y, (int64_t)k);
}
double vo_exp_d_u10(double x) { return exp_core_d(x, C_EXP_D, VEM_EXP_D_N, 1); }
double vo_exp_d_u35(double x) { return exp_core_d(x, C_EXP_D_U35, VEM_EXP_D_U35_N, 0); }

/* ---- table-driven log / exp cores (tools/genlogtables.py)
 * a = 2^E * m, m in [0.75, 1.5) (the paper's split, so
 * x near 1 has E = 0 and no cancellation); idx = top 8 bits of
 * bits(m) - bits(0.75); r = m*invc - 1 formed exactly as rh + rl (two_prod,
 * Sterbenz), |r| <= 2^-8; log(a) = E*ln2 + logc + log1p(r).  No division. */
#define LN2_H42 VEM_LN2_H42
#define LN2_T42 VEM_LN2_T42
static const double C_LOG1P_D[] = VEM_LOG1P_D_ARR;
static const double C_LOG1P_D_U35[] = VEM_LOG1P_D_U35_ARR;
static const double C_EXPJ_D[] = VEM_EXPJ_D_ARR;
static const double C_LOG1P_F[] = VEM_LOG1P_F_ARR;
static const double C_LOG1P_F_U35[] = VEM_LOG1P_F_U35_ARR;

typedef struct { double rh, rl, E, logc_hi, logc_lo; } logred_t;

/* a: positive normal finite binary64 */
static inline logred_t log_reduce(double a, double Eadj) {
  uint64_t ix = bits_d(a);
  uint64_t tmp = ix - 0x3fe8000000000000ull;
  int64_t k = (int64_t)tmp >> 52;
  int idx = (int)((tmp >> 44) & 255u);
  double m = from_bits_d(ix - ((uint64_t)k << 52));
  double invc = LOGT_INVC[idx];
  double p = m * invc;
  logred_t o;
  o.rl = fma(m, invc, -p);
  o.rh = p - 1.0;
  o.E = (double)(int32_t)k + Eadj;
  o.logc_hi = LOGT_HI[idx];
  o.logc_lo = LOGT_LO[idx];
  return o;
}

/* log1p(rh + rl) as DD: rh - rh^2/2 (exact: p2 = -z/2, its error -ez/2 with
 * ez = fma(rh, rh, -z)) + rh^3 Q(rh) + rl(1 - rh), the low terms fused */
static inline dd_t log1p_dd(double rh, double rl, const double* c, int n) {
  double z = rh * rh;
  double Q = poly(c, n, rh);
  double p2 = -0.5 * z;
  double ez = fma(rh, rh, -z);
  double lo = fma(-0.5, ez, fma(rh * z, Q, fma(-rl, rh, rl)));
  dd_t S = two_sum_fast(rh, p2);
  S.lo = S.lo + lo;
  return S;
}

/* E*ln2 + logc as DD: E*LN2_H42 (exact for |E| < 2^11) and logc_hi are both
 * on the 2^-42 grid below 2^10, so their sum is exact (tools/genlogtables.py) */
static inline dd_t eln2_logc(const logred_t* g) {
  double eh = g->E * LN2_H42;
  dd_t H = {eh + g->logc_hi, fma(g->E, LN2_T42, g->logc_lo)};
  return H;
}

static double log_fast_d(double a, double Eadj, int u10) {
  logred_t g = log_reduce(a, Eadj);
  dd_t H = eln2_logc(&g);
  dd_t L;
  if (u10) {
    /* the 5-term set (2^-64.2): the 6-term one (2^-71.6) is for pow's double-double log */
    L = log1p_dd(g.rh, g.rl, C_LOG1P_D_U35, VEM_LOG1P_D_U35_N);
  } else {
    double z = g.rh * g.rh;
    double Q = poly(C_LOG1P_D_U35, VEM_LOG1P_D_U35_N, g.rh);
    L.hi = g.rh;
    L.lo = fma(z, fma(g.rh, Q, -0.5), g.rl);
  }
  dd_t T = two_sum(H.hi, L.hi);
  return T.hi + (T.lo + (H.lo + L.lo));
}

/* log: fast path for positive normal finite x; slow path: subnormals (x 2^64,
 * PAPER.md:797-803), 0 -> -inf, <0 -> NaN, inf, NaN. */
static double log_core_d(double x, int u10) {
  uint64_t ix = bits_d(x);
  if (ix - 0x0010000000000000ull < 0x7fe0000000000000ull) return log_fast_d(x, 0.0, u10);
  if (x > 0.0 && x < 0x1p-1022) return log_fast_d(x * 0x1p64, -64.0, u10);
  if (x == 0.0) return -INFINITY;
  if (x == INFINITY) return x;
  return from_bits_d(CANON_NAN_D); /* negative or NaN */
}
double vo_log_d_u10(double x) { return log_core_d(x, 1); }
double vo_log_d_u35(double x) { return log_core_d(x, 0); }

/* pow internals: log as a double-double (rel. err ~2^-70) */
static inline dd_t log_dd(double a, double Eadj, const double* c, int n) {
  logred_t g = log_reduce(a, Eadj);
  dd_t H = eln2_logc(&g);
  dd_t L = log1p_dd(g.rh, g.rl, c, n);
  /* |H.hi| >= |L.hi| or H.hi == 0 (E != 0: |H| > ln2 - 0.41; E = 0: |logc|
   * exceeds the interval half-width except c = 1 where logc = 0) */
  dd_t S = two_sum_fast(H.hi, L.hi);
  S.lo = S.lo + (H.lo + L.lo);
  return S;
}

/* exp of a double-double t with a 128-entry 2^(i/128) table (EXPT):
 * k = rint(t*128/ln2), r = t - k*ln2/128 (3-part constant), |r| <= ln2/256,
 * exp(t) = 2^(k>>7) * T[k&127] * (1 + em1(r)).  |th| < 708: normal result,
 * exponent-field scaling; otherwise saturation / ldexp2. */
static double exp_dd(dd_t t) {
  double th = t.hi, tl = t.lo;
  uint32_t hx = (uint32_t)(bits_d(th) >> 32) & 0x7fffffffu;
  int fast = hx < EXP_FAST_HI;
  if (!fast) {
    int ok = (th >= -760.0) && (th <= 720.0);
    th = ok ? th : 0.0;
    tl = ok ? tl : 0.0;
  }
  int32_t k;
  double kd = rint_fma(th, VEM_EXPJ_INV, &k);
  double r1 = fma(kd, -VEM_EXPJ_L1, th);
  double r2 = fma(kd, -VEM_EXPJ_L2, tl);
  /* |r2| <~ 2^-26, |r| <= ln2/256: the rounding error of this sum is below
   * 2^-61.5, i.e. 0.003 ulp of the result -- not worth a two-sum and the two
   * operations that would carry it (round 2; the result moved by at most that) */
  double r = r1 + r2;
  double z = r * r;
  double Q = poly(C_EXPJ_D, VEM_EXPJ_D_N, r);
  double s2 = z * fma(r, Q, 0.5);
  double Th = EXPT_HI[k & 127], Tl = EXPT_LO[k & 127];
  double u = fma(Th, r, fma(Th, s2, Tl));
  double R = Th + u;
  int32_t e = k >> 7;
  if (fast) return from_bits_d(bits_d(R) + ((uint64_t)(int64_t)e << 52));
  double y = ldexp2(R, (int64_t)e);
  y = (t.hi > K_EXP_OVF) ? INFINITY : y;
  y = (t.hi < K_EXP_UNF) ? 0.0 : y;
  return y;
}

/* C99 Annex F pow special cases. */
static inline int is_int_d(double y) { return (fabs(y) < INFINITY) && (trunc(y) == y); }
static inline int is_odd_d(double y) {
  return is_int_d(y) && (fabs(y) < 0x1p53) && (trunc(y * 0.5) * 2.0 != y);
}

/* pow = exp(y * log|x|).  Fast path: x positive normal
 * finite, y finite nonzero -- no special-case logic at all.  Slow path:
 * subnormal/negative x and every C99 special value. */
static double pow_core_d(double x, double y, const double* cl, int nl) {
  uint32_t hx = (uint32_t)(bits_d(x) >> 32);
  uint32_t hy = (uint32_t)(bits_d(y) >> 32) & 0x7fffffffu, ly = (uint32_t)bits_d(y);
  int fx = ((hx & 0x7fffffffu) - 0x00100000u) < 0x7fe00000u; /* x normal finite */
  int fy = (hy < 0x7ff00000u) && ((hy | ly) != 0u);           /* y finite, nonzero */
  if (fx && fy) {
    double R = exp_dd(dd_mul_d(log_dd(fabs(x), 0.0, cl, nl), y));
    if (x < 0.0) R = is_int_d(y) ? (is_odd_d(y) ? -R : R) : from_bits_d(CANON_NAN_D);
    return R;
  }
  double ax = fabs(x);
  int fin = (ax > 0.0) && (ax < INFINITY) && (fabs(y) < INFINITY);
  double R = 1.0;
  if (fin) {
    int sub = ax < 0x1p-1022;
    R = exp_dd(dd_mul_d(log_dd(sub ? ax * 0x1p64 : ax, sub ? -64.0 : 0.0, cl, nl), y));
  }
  int yint = is_int_d(y), yodd = is_odd_d(y);
  double res = (x < 0.0 && yodd) ? -R : R;
  res = (x < 0.0 && !yint && fabs(y) < INFINITY) ? from_bits_d(CANON_NAN_D) : res;
  if (x == 0.0) {
    if (y < 0.0) res = yodd ? copysign_b(INFINITY, x) : INFINITY;
    else res = yodd ? x : 0.0;
  }
  if (ax == INFINITY) {
    if (y < 0.0) res = (yodd && x < 0.0) ? -0.0 : 0.0;
    else res = (yodd && x < 0.0) ? -INFINITY : INFINITY;
  }
  if (fabs(y) == INFINITY) {
    if (ax == 1.0) res = 1.0;
    else res = ((ax < 1.0) == (y < 0.0)) ? INFINITY : 0.0;
  }
  if (x != x || y != y) res = from_bits_d(CANON_NAN_D);
  if (y == 0.0 || x == 1.0) res = 1.0;
  return res;
}
double vo_pow_d_u10(double x, double y) { return pow_core_d(x, y, C_LOG1P_D, VEM_LOG1P_D_N); }
double vo_pow_d_u35(double x, double y) { return pow_core_d(x, y, C_LOG1P_D_U35, VEM_LOG1P_D_U35_N); }

/* fmod -- exact remainder by FP long division (Alg. 1, PAPER.md:958-975,
 * 1445-1469), restated on normalised mantissas so the quotient ratio never
 * overflows (SLEEF/the paper return NaN when |x/y| > DBL_MAX, SURVEY.md §0
 * item 6):  n = mn*2^en, d = md*2^ed with mn, md in [1,2) (exact, subnormals
 * via clz), E = en - ed, and n mod d = 2^ed * ((mn * 2^E) mod md).  Each step
 * shifts the running remainder r in [0, md) left by s = min(E, 50) bits and
 * removes Q*md, Q = trunc(toward0(r*2^s * toward0(1/md))), which
 * is floor or floor-1 of the true quotient (< 2^51); the off-by-one is resolved
 * exactly with two candidate remainders.  One division per call; the loop runs
 * ceil(E/50) times.  Exact, hence bit-identical to glibc fmod. */
static inline int64_t ilogb_pos(double x) { /* x > 0 finite, subnormals exact */
  uint64_t b = bits_d(x);
  int64_t e = (int64_t)(b >> 52);
  if (e != 0) return e - 1023;
  return (int64_t)(63 - __builtin_clzll(b)) - 1074;
}
/* x > 0 finite with ilogb e: x * 2^-e in [1, 2), exactly (bit manipulation) */
static inline double mant_1_2(double x, int64_t e) {
  uint64_t b = bits_d(x);
  uint64_t m = (e >= -1022) ? (b & 0x000fffffffffffffull) : ((b << (-1022 - e)) & 0x000fffffffffffffull);
  return from_bits_d(m | 0x3ff0000000000000ull);
}
/* one long-division step of width s (1 <= s <= 50); r > 0 */
static inline double fmod_step(double r, int s, double md, double rmd) {
  double rs = r * pow2_bits(s);
  double Q = trunc(toward0_pos(rs * rmd));
  double Q2 = Q + 1.0;
  double p1 = Q * md, e1 = fma(Q, md, -p1);
  double V1 = (rs - p1) - e1;
  double p2 = Q2 * md, e2 = fma(Q2, md, -p2);
  double V2 = (rs - p2) - e2;
  return (V2 >= 0.0) ? V2 : V1;
}
static _Thread_local int g_fmod_steps; /* iteration counter for vo_fmod_d_iters */
static double fmod_core(double x, double y) {
  double n = fabs(x), d = fabs(y);
  if (x != x || y != y || !(n < INFINITY) || d == 0.0) return from_bits_d(CANON_NAN_D);
  if (d == INFINITY || n < d) return x;
  int64_t en = ilogb_pos(n), ed = ilogb_pos(d);
  double mn = mant_1_2(n, en), md = mant_1_2(d, ed);
  int64_t E = en - ed;
  double rmd = toward0_pos(1.0 / md);
  double r = (E == 0) ? mn - md : mn;
  while (E > 0 && r != 0.0) {
    int s = E > 50 ? 50 : (int)E;
    E -= s;
    r = fmod_step(r, s, md, rmd);
    g_fmod_steps++;
  }
  return copysign_b(ldexp2(r, ed), x);
}
double vo_fmod_d(double x, double y) { return fmod_core(x, y); }

/* ================================ f32 kernels (binary64 internals) */
static const double C_SIN_F[] = VEM_SIN_F_ARR;
static const double C_COS_F[] = VEM_COS_F_ARR;
static const double C_TAN_F[] = VEM_TAN_F_ARR;
static const double C_EXP_F[] = VEM_EXP_F_ARR;
static const double C_EXP_F_U35[] = VEM_EXP_F_U35_ARR;

/* f32 Payne-Hanek in binary64 limbs (new; the reference is double-only).
 * |x| = M*2^S, M in [2^23, 2^24); the table (tools/genphtable.py) holds
 * V(S) = (2^S * 2/pi) mod 4 as three limbs t0 (29 bits, weights 2^1..2^-27),
 * t1 (29 bits, ..2^-56), t2 (53 bits, ..2^-109), each divided by 2^S, so with
 * xd = (double)x:  p0 = xd*t0 = M*a0 is exact (53 bits), n = rint(p0 + xd*t1)
 * by the 1.5*2^52 shift (its low word carries the quadrant, two's complement
 * for x < 0; M*a1 < 2^-3 must take part, or |f| could reach 5/8),
 * f0 = p0 - n exact, and f = fma(xd, t2, fma(xd, t1, f0)) is the
 * centred fraction of x*2/pi: the inner fma is exact whenever its result is
 * below 2^-3 (the cancellation case), so f is within 2^-52 relative + 2^-85
 * absolute (smallest |f| over all binary32: ~2^-30).  r = f * pi/2.
 * Exponents below 2^25 use entry 0 (plain 2/pi split), so tiny x need no
 * special case: r = x(1 + O(2^-52)).  Inf/NaN give NaN (inf - inf).  Every
 * f32 trig lane takes this path (no selector, no divergence). */
typedef struct { double r; int q; } redf_t;
static const double PH_F[4 * VEM_PH_F_ENTRIES] = {VEM_PH_F_INIT};
static redf_t ph_f(float xf) {
  uint32_t fe = (bits_f(xf) >> 23) & 0xffu;
  uint32_t idx = (fe > VEM_PH_F_FE0 ? fe : VEM_PH_F_FE0) - VEM_PH_F_FE0;
  const double* t = PH_F + 4 * idx;
  double xd = (double)xf;
  double p0 = xd * t[0];
  double n = fma(xd, t[1], p0) + 0x1.8p52; /* rint of the two-limb product: |f| <= 1/2 + 2^-31 */
  double f0 = p0 - (n - 0x1.8p52);
  double f = fma(xd, t[2], fma(xd, t[1], f0));
  redf_t o;
  o.r = f * 0x1.921fb54442d18p+0;
  o.q = (int)((uint32_t)bits_d(n) & 3u);
  return o;
}

static double sincos_core_f(double r, int cosform) {
  /* sin: r (1 + z S(z)) (a product: -0 stays -0);  cos: 1 + z (-1/2 + z C(z)) */
  double z = r * r;
  if (cosform) {
    double c[5] = {-0.5, C_COS_F[0], C_COS_F[1], C_COS_F[2], C_COS_F[3]};
    return fma(z, poly(c, 5, z), 1.0);
  }
  return r * fma(z, poly(C_SIN_F, 4, z), 1.0);
}

float vo_sin_f_u10(float x) {
  redf_t r = ph_f(x);
  double y = sincos_core_f(r.r, r.q & 1);
  y = neg_if(y, r.q & 2);
  float o = (float)y;
  o = (x == 0.0f) ? x : o;
  return canon_f(isinf(x) ? (float)NAN : (x != x ? x : o));
}
float vo_cos_f_u10(float x) {
  redf_t r = ph_f(x);
  double y = sincos_core_f(r.r, (r.q & 1) ^ 1);
  y = neg_if(y, (r.q + 1) & 2);
  float o = (float)y;
  return canon_f(isinf(x) ? (float)NAN : (x != x ? x : o));
}
float vo_tan_f_u10(float x) {
  redf_t r = ph_f(x);
  double z = r.r * r.r;
  double P = poly(C_TAN_F, VEM_TAN_F_N, z);
  double t = fma(r.r * z, P, r.r);
  /* -cot, branch-free: 1/|t| from a binary32 magic-constant seed (rel. error
   * <= 0.051), three binary32 Newton steps (<= 2^-23.9 measured bound 6e-8) and
   * one binary64 Newton step (<= 2^-47): far below the final binary32
   * rounding.  |t| >= 2^-31 for an odd quadrant: every binary32 value normal. */
  double ta = fabs(t);
  float tf = (float)ta;
  float yf = from_bits_f(0x7EF311C7u - bits_f(tf));
  for (int i = 0; i < 3; i++) yf = fmaf(yf, fmaf(-tf, yf, 1.0f), yf);
  double y0 = (double)yf;
  double y1 = fma(y0, fma(-ta, y0, 1.0), y0);
  double y = (r.q & 1) ? (t < 0.0 ? y1 : -y1) : t;
  float o = (float)y;
  o = (x == 0.0f) ? x : o;
  return canon_f(isinf(x) ? (float)NAN : (x != x ? x : o));
}

static float exp_core_f(float x, const double* c, int n) {
  float xc = fminf(fmaxf(x, -150.0f), 130.0f);
  double xd = (double)xc;
  int32_t k;
  double kd = rint_fma(xd, K_INV_LN2, &k);
  double r = fma(kd, -K_EXP_L1, xd);
  r = fma(kd, -K_EXP_L2, r);
  double P = poly(c, n, r);
  double y = fma(r, P, 1.0);
  y = from_bits_d(bits_d(y) + ((uint64_t)(int64_t)k << 52)); /* |k| <= 217: normal */
  float o = (float)y;
  return canon_f((x != x) ? x : o);
}
float vo_exp_f_u10(float x) { return exp_core_f(x, C_EXP_F, VEM_EXP_F_N); }
float vo_exp_f_u35(float x) { return exp_core_f(x, C_EXP_F_U35, VEM_EXP_F_U35_N); }

/* f32 log in binary64 with the same 256-entry table: r = m*invc - 1 by one
 * fma (its rounding is far below binary32 resolution), log1p(r) = r + r^2 Q(r).
 * Every positive finite binary32 (incl. subnormals) is a normal binary64. */
static inline double log_f_internal(double a, const double* c, int n) {
  uint64_t ix = bits_d(a);
  uint64_t tmp = ix - 0x3fe8000000000000ull;
  int64_t k = (int64_t)tmp >> 52;
  int idx = (int)((tmp >> 44) & 255u);
  double m = from_bits_d(ix - ((uint64_t)k << 52));
  double r = fma(m, (double)LOGTF_INVC[idx], -1.0); /* exact: 24 x 24 bits */
  double Q = poly(c, n, r);
  double L = fma(r * r, Q, r);
  return fma((double)(int32_t)k, K_LN2_HI, LOGTF_HI[idx] + L);
}
static float log_core_f(float x, const double* c, int n) {
  uint32_t ux = bits_f(x);
  if (ux - 1u < 0x7f7fffffu) return (float)log_f_internal((double)x, c, n);
  if (x == 0.0f) return -INFINITY;
  if (x == INFINITY) return x;
  return from_bits_f(CANON_NAN_F);
}
float vo_log_f_u10(float x) { return log_core_f(x, C_LOG1P_F, VEM_LOG1P_F_N); }
float vo_log_f_u35(float x) { return log_core_f(x, C_LOG1P_F_U35, VEM_LOG1P_F_U35_N); }

static inline int is_int_f(float y) { return (fabsf(y) < INFINITY) && (truncf(y) == y); }
static inline int is_odd_f(float y) {
  return is_int_f(y) && (fabsf(y) < 0x1p24f) && (truncf(y * 0.5f) * 2.0f != y);
}
/* exp(t) for the f32 pow, |t| <= 200: EXPT hi limb x (1 + r + r^2/2 + r^3/6) */
static inline double exp_f_internal(double t) {
  int32_t k;
  double kd = rint_fma(t, VEM_EXPJ_INV, &k);
  double r = fma(kd, -VEM_EXPJ_L1, t);
  r = fma(kd, -VEM_EXPJ_L2, r);
  double p = fma(r * r, fma(r, 0x1.5555555555555p-3, 0.5), r);
  double T = EXPT_HI[k & 127];
  double R = fma(T, p, T);
  return from_bits_d(bits_d(R) + ((uint64_t)(int64_t)(k >> 7) << 52));
}
static float pow_core_f(float x, float y, const double* cl, int nl) {
  uint32_t ux = bits_f(x), uy = bits_f(y);
  int fx = (ux - 1u) < 0x7f7fffffu;             /* x in (0, inf) */
  int fy = ((uy & 0x7fffffffu) - 1u) < 0x7f7fffffu; /* y finite, != 0 */
  if (fx && fy) {
    double t = (double)y * log_f_internal((double)x, cl, nl);
    if (((uint32_t)(bits_d(t) >> 32) & 0x7fffffffu) >= 0x40690000u) t = (t > 0.0) ? 200.0 : -200.0;
    return (float)exp_f_internal(t);
  }
  float ax = fabsf(x);
  int fin = (ax > 0.0f) && (ax < INFINITY) && (fabsf(y) < INFINITY);
  float Rf = 1.0f;
  if (fin) {
    double t = (double)y * log_f_internal((double)ax, cl, nl);
    t = fmin(fmax(t, -200.0), 200.0);
    Rf = (float)exp_f_internal(t);
  }
  int yint = is_int_f(y), yodd = is_odd_f(y);
  float res = (x < 0.0f && yodd) ? -Rf : Rf;
  res = (x < 0.0f && !yint && fabsf(y) < INFINITY) ? from_bits_f(CANON_NAN_F) : res;
  if (x == 0.0f) {
    if (y < 0.0f) res = yodd ? copysignf(INFINITY, x) : INFINITY;
    else res = yodd ? x : 0.0f;
  }
  if (ax == INFINITY) {
    if (y < 0.0f) res = (yodd && x < 0.0f) ? -0.0f : 0.0f;
    else res = (yodd && x < 0.0f) ? -INFINITY : INFINITY;
  }
  if (fabsf(y) == INFINITY) {
    if (ax == 1.0f) res = 1.0f;
    else res = ((ax < 1.0f) == (y < 0.0f)) ? INFINITY : 0.0f;
  }
  if (x != x || y != y) res = from_bits_f(CANON_NAN_F);
  if (y == 0.0f || x == 1.0f) res = 1.0f;
  return res;
}
float vo_pow_f_u10(float x, float y) { return pow_core_f(x, y, C_LOG1P_F, VEM_LOG1P_F_N); }
float vo_pow_f_u35(float x, float y) { return pow_core_f(x, y, C_LOG1P_F_U35, VEM_LOG1P_F_U35_N); }

float vo_fmod_f(float x, float y) {
  /* fmodf(x,y) == (float)fmod((double)x,(double)y) exactly: the remainder is
   * representable in binary32. NaN canonicalised in the float domain. */
  double r = fmod_core((double)x, (double)y);
  return canon_f((float)r);
}

/* ============================ SURVEY §8(f).1: fdim, atan2, asin/acos, u35
 * trig/atan (u35 recipe: "same reductions with shorter
 * polynomials and single-double reconstruction", SPEC.md DESIGN DECISIONS).
 * Float32 versions evaluate the binary64 routine and round once. */
static const double C_ASIN_D[] = VEM_ASIN_D_ARR;
static const double C_ASIN_D_U35[] = VEM_ASIN_D_U35_ARR;
static const double C_SIN_D_U35[] = VEM_SIN_D_U35_ARR;
static const double C_COS_D_U35[] = VEM_COS_D_U35_ARR;
static const double C_ATAN_D_U35[] = VEM_ATAN_D_U35_ARR;
#define K_PI_HI 0x1.921fb54442d18p+1
#define K_PI_LO 0x1.1a62633145c07p-53
#define K_3PIO4_HI 0x1.2d97c7f3321d2p+1
#define K_3PIO4_LO 0x1.a79394c9e8a0ap-54

/* fdim: x - y if x > y, +0 otherwise; NaN if either is */
double vo_fdim_d(double x, double y) {
  double r = (x > y) ? x - y : 0.0;
  return (x != x || y != y) ? from_bits_d(CANON_NAN_D) : r;
}
float vo_fdim_f(float x, float y) {
  float r = (x > y) ? x - y : 0.0f;
  return (x != x || y != y) ? from_bits_f(CANON_NAN_F) : r;
}

/* u35 sin/cos/tan: the u10 reduction, r = hi part only */
static double sincos_core_d_u35(double r, int cosform) {
  double z = r * r;
  if (cosform) {
    double P = poly(C_COS_D_U35, VEM_COS_D_U35_N, z);
    return fma(z, fma(z, P, -0.5), 1.0);
  }
  double P = poly(C_SIN_D_U35, VEM_SIN_D_U35_N, z);
  return fma(r * z, P, r);
}
double vo_sin_d_u35(double x) {
  red_t r = trig_reduce_fn(x);
  double y = sincos_core_d_u35(r.hi, r.q & 1);
  y = neg_if(y, r.q & 2);
  y = (x == 0.0) ? x : y;
  return canon_d(y);
}
double vo_cos_d_u35(double x) {
  red_t r = trig_reduce_fn(x);
  double y = sincos_core_d_u35(r.hi, (r.q & 1) ^ 1);
  y = neg_if(y, (r.q + 1) & 2);
  return canon_d(y);
}
/* tan u35: half angle with the u10 polynomial and the reduction's low
 * part folded in, one binary64 division for both quadrant parities */
static double tan_core_d_u35(double rh, double rl, int odd) {
  double h = rh * 0.5, hl = rl * 0.5;
  double z = h * h;
  double P = poly(C_TAN_D, VEM_TAN_D_N, z);
  double t = h + fma(h * z, P, hl);
  double num = t + t;
  double den = fma(-t, t, 1.0);
  double X = odd ? -den : num, Y = odd ? num : den;
  return X / Y;
}
double vo_tan_d_u35(double x) {
  red_t r = trig_reduce_fn(x);
  double y = tan_core_d_u35(r.hi, r.lo, r.q & 1);
  y = (fabs(x) < 0x1p-27) ? x : y;
  return canon_d(y);
}
/* atan u35: the u10 fold with binary64 division, no DD */
double vo_atan_d_u35(double x) {
  double a = fabs(x);
  int c1 = a > K_TAN_PI8;
  int c2 = a > K_TAN_3PI8;
  double nn = c2 ? -1.0 : (c1 ? a - 1.0 : a);
  double dn = c2 ? fmin(a, 0x1p60) : (c1 ? a + 1.0 : 1.0);  /* see vo_atan_d_u10 */
  double b = nn / dn;
  double z = b * b;
  double P = poly(C_ATAN_D_U35, VEM_ATAN_D_U35_N, z);
  double off = c2 ? K_PIO2_QD0 : (c1 ? K_PIO4_HI : 0.0);
  double y = off + fma(b * z, P, b);
  y = copysign_b(y, x);
  return canon_d(y);
}

/* asin / acos (§5.3): |x| <= 1/2 directly,
 * asin t = t + t z P(z), z = t^2; |x| > 1/2 by asin|x| = pi/2 - 2 asin(s),
 * s = sqrt(z), z = (1-|x|)/2 exact.  u10 carries sqrt's rounding error as
 * sl = (z - s^2)/(2s) (z - s^2 exact by FMA) and adds pi/2 in DD. */
typedef struct { double a, z, s, sl, u; int big; } asin_parts_t;
static asin_parts_t asin_parts(double x, const double* c, int n, int u10) {
  asin_parts_t o;
  o.a = fabs(x);
  o.big = o.a > 0.5;
  o.z = o.big ? (1.0 - o.a) * 0.5 : o.a * o.a;
  o.s = sqrt(o.z);
  double t = o.big ? o.s : o.a;
  double P = poly(c, n, o.z);
  o.u = (t * o.z) * P;
  o.sl = 0.0;
  if (u10) {
    double e = fma(-o.s, o.s, o.z);
    o.sl = (o.z == 0.0) ? 0.0 : e / (o.s + o.s);
  }
  return o;
}
double vo_asin_d_u10(double x) {
  asin_parts_t p = asin_parts(x, C_ASIN_D, VEM_ASIN_D_N, 1);
  dd_t h = two_sum(K_PIO2_QD0, -2.0 * p.s);
  double yb = h.hi + (h.lo + (K_PIO2_QD1 - 2.0 * (p.sl + p.u)));
  double y = p.big ? yb : p.a + p.u;
  y = (p.a > 1.0) ? from_bits_d(CANON_NAN_D) : y;
  return canon_d(copysign_b(y, x));
}
double vo_asin_d_u35(double x) {
  asin_parts_t p = asin_parts(x, C_ASIN_D_U35, VEM_ASIN_D_U35_N, 0);
  double yb = (K_PIO2_QD0 - 2.0 * p.s) + (K_PIO2_QD1 - 2.0 * p.u);
  double y = p.big ? yb : p.a + p.u;
  y = (p.a > 1.0) ? from_bits_d(CANON_NAN_D) : y;
  return canon_d(copysign_b(y, x));
}
double vo_acos_d_u10(double x) {
  asin_parts_t p = asin_parts(x, C_ASIN_D, VEM_ASIN_D_N, 1);
  /* |x| <= 1/2: pi/2 - asin x;  x > 1/2: 2 asin s;  x < -1/2: pi - 2 asin s */
  double us = copysign_b(p.u, x);
  dd_t hs = two_sum(K_PIO2_QD0, -x);
  double ys = hs.hi + (hs.lo + (K_PIO2_QD1 - us));
  double yp = 2.0 * p.s + 2.0 * (p.sl + p.u);
  dd_t hn = two_sum(K_PI_HI, -2.0 * p.s);
  double yn = hn.hi + (hn.lo + (K_PI_LO - 2.0 * (p.sl + p.u)));
  double y = p.big ? (x > 0.0 ? yp : yn) : ys;
  y = (p.a > 1.0) ? from_bits_d(CANON_NAN_D) : y;
  return canon_d(y);
}
double vo_acos_d_u35(double x) {
  asin_parts_t p = asin_parts(x, C_ASIN_D_U35, VEM_ASIN_D_U35_N, 0);
  double us = copysign_b(p.u, x);
  double ys = (K_PIO2_QD0 - x) + (K_PIO2_QD1 - us);
  double yp = 2.0 * (p.s + p.u);
  double yn = (K_PI_HI - 2.0 * p.s) + (K_PI_LO - 2.0 * p.u);
  double y = p.big ? (x > 0.0 ? yp : yn) : ys;
  y = (p.a > 1.0) ? from_bits_d(CANON_NAN_D) : y;
  return canon_d(y);
}

/* atan2: num = min(|x|,|y|), den = max(|x|,|y|) (scaled
 * by a common power of two away from overflow / reciprocal underflow), the
 * atan fold of num/den -- b = num/den or (num-den)/(num+den), one DD
 * division -- then result = C + sigma * atan(b) with C in {0, pi/4, pi/2,
 * 3pi/4, pi} (DD) and sigma = +-1 by (|y| > |x|, x < 0, fold), sign of y.
 * C99 Annex F.9.1.4 special cases selected at the end. */
static double atan2_special(double y, double x, double g) {
  double ax = fabs(x), ay = fabs(y);
  double r = g;
  if (ax == INFINITY) r = (ay == INFINITY) ? (x > 0.0 ? K_PIO4_HI : K_3PIO4_HI) : (x > 0.0 ? 0.0 : K_PI_HI);
  else if (ay == INFINITY) r = K_PIO2_QD0;
  if (x == 0.0) r = (y == 0.0) ? ((bits_d(x) >> 63) ? K_PI_HI : 0.0) : K_PIO2_QD0;
  else if (y == 0.0) r = (x > 0.0) ? 0.0 : K_PI_HI;
  r = copysign_b(r, y);
  return (x != x || y != y) ? from_bits_d(CANON_NAN_D) : r;
}
typedef struct { double num, den, ch, cl; int c1, sig; } atan2_parts_t;
static atan2_parts_t atan2_parts(double y, double x) {
  atan2_parts_t o;
  double ax = fabs(x), ay = fabs(y);
  int swap = ay > ax;
  double num = swap ? ax : ay, den = swap ? ay : ax;
  double sc = den >= 0x1p1000 ? 0x1p-100 : (den < 0x1p-900 ? 0x1p100 : 1.0);
  o.num = num * sc;
  o.den = den * sc;
  o.c1 = o.num > K_TAN_PI8 * o.den;
  int neg = x < 0.0;
  /* C = (neg ? pi : 0) + (swap ? (neg ? -pi/2 : pi/2) : 0) + s * (c1 ? pi/4 : 0) */
  int q = (neg ? 4 : 0) + (swap ? (neg ? -2 : 2) : 0);   /* multiples of pi/4 */
  o.sig = (swap != neg) ? -1 : 1;
  q += o.c1 ? o.sig : 0;
  o.ch = q == 0 ? 0.0 : (q == 1 ? K_PIO4_HI : (q == 2 ? K_PIO2_QD0 : (q == 3 ? K_3PIO4_HI : K_PI_HI)));
  o.cl = q == 0 ? 0.0 : (q == 1 ? K_PIO4_LO : (q == 2 ? K_PIO2_QD1 : (q == 3 ? K_3PIO4_LO : K_PI_LO)));
  return o;
}
double vo_atan2_d_u10(double y, double x) {
  atan2_parts_t p = atan2_parts(y, x);
  dd_t ns = two_sum(p.num, -p.den), ds = two_sum(p.num, p.den);
  dd_t nn = p.c1 ? ns : (dd_t){p.num, 0.0};
  dd_t dn = p.c1 ? ds : (dd_t){p.den, 0.0};
  dd_t b = dd_div(nn, dn);
  double z = b.hi * b.hi;
  double P = poly(C_ATAN_D, VEM_ATAN_D_N, z);
  double corr = fma(b.hi * z, P, fma(-b.lo, z, b.lo));
  double sg = (double)p.sig;
  dd_t s = two_sum(p.ch, sg * b.hi);
  double g = s.hi + (s.lo + (p.cl + sg * corr));
  return canon_d(atan2_special(y, x, copysign_b(g, y)));
}
double vo_atan2_d_u35(double y, double x) {
  atan2_parts_t p = atan2_parts(y, x);
  double nn = p.c1 ? p.num - p.den : p.num;
  double dn = p.c1 ? p.num + p.den : p.den;
  double b = nn * (1.0 / dn);  /* 1/dn normal after scaling; a tiny quotient stays off the division slow path */
  double z = b * b;
  double P = poly(C_ATAN_D_U35, VEM_ATAN_D_U35_N, z);
  double g = p.ch + (double)p.sig * fma(b * z, P, b);
  return canon_d(atan2_special(y, x, copysign_b(g, y)));
}

/* float32: binary64 routine, one rounding */
float vo_atan_f_u10(float x) { return canon_f((float)vo_atan_d_u10((double)x)); }
float vo_atan_f_u35(float x) { return canon_f((float)vo_atan_d_u35((double)x)); }
float vo_asin_f_u10(float x) { return canon_f((float)vo_asin_d_u10((double)x)); }
float vo_asin_f_u35(float x) { return canon_f((float)vo_asin_d_u35((double)x)); }
float vo_acos_f_u10(float x) { return canon_f((float)vo_acos_d_u10((double)x)); }
float vo_acos_f_u35(float x) { return canon_f((float)vo_acos_d_u35((double)x)); }
float vo_atan2_f_u10(float y, float x) { return canon_f((float)vo_atan2_d_u10((double)y, (double)x)); }
float vo_atan2_f_u35(float y, float x) { return canon_f((float)vo_atan2_d_u35((double)y, (double)x)); }

/* ============================================ exported array API */
void vo_ph_int_reduce_d(const double* x, double* hi, double* lo, int* q, size_t n) {
  for (size_t i = 0; i < n; i++) {
    red_t r = ph_int(x[i]);
    hi[i] = r.hi;
    lo[i] = r.lo;
    q[i] = r.q;
  }
}
void vo_trig_reduce_d(const double* x, double* hi, double* lo, int* q, size_t n) {
  for (size_t i = 0; i < n; i++) {
    red_t r = trig_reduce(x[i]);
    hi[i] = r.hi; lo[i] = r.lo; q[i] = r.q;
  }
}
void vo_ph_reduce_d(const double* x, double* hi, double* lo, int* q, size_t n) {
  for (size_t i = 0; i < n; i++) {
    red_t r = ph(x[i]);
    hi[i] = r.hi; lo[i] = r.lo; q[i] = r.q;
  }
}
void vo_cw_reduce_d(const double* x, double* hi, double* lo, int* q, size_t n, int level) {
  for (size_t i = 0; i < n; i++) {
    red_t r = level == 1 ? cw1(x[i]) : cw2(x[i]);
    hi[i] = r.hi; lo[i] = r.lo; q[i] = r.q;
  }
}
void vo_ph_reduce_f(const float* x, double* r, int* q, size_t n) {
  for (size_t i = 0; i < n; i++) {
    redf_t o = ph_f(x[i]);
    r[i] = o.r; q[i] = o.q;
  }
}
const double* vo_ph_table_d(void) { return PH_D; }
const double* vo_ph_table_f(void) { return PH_F; }
double vo_round_ta(double x) { return round_ta(x); }

#define UNARY_ARR(name, T)                                             \
  void name##_arr(const T* x, T* y, size_t n) {                        \
    _Pragma("omp parallel for schedule(static)")                       \
    for (size_t i = 0; i < n; i++) y[i] = name(x[i]);                  \
  }
#define BINARY_ARR(name, T)                                            \
  void name##_arr(const T* x, const T* y2, T* y, size_t n) {           \
    _Pragma("omp parallel for schedule(static)")                       \
    for (size_t i = 0; i < n; i++) y[i] = name(x[i], y2[i]);           \
  }

UNARY_ARR(vo_sin_d_u10, double)
UNARY_ARR(vo_cos_d_u10, double)
UNARY_ARR(vo_tan_d_u10, double)
UNARY_ARR(vo_sin_d_u10_ph, double)
UNARY_ARR(vo_cos_d_u10_ph, double)
UNARY_ARR(vo_tan_d_u10_ph, double)
UNARY_ARR(vo_atan_d_u10, double)
UNARY_ARR(vo_exp_d_u10, double)
UNARY_ARR(vo_exp_d_u35, double)
UNARY_ARR(vo_log_d_u10, double)
UNARY_ARR(vo_log_d_u35, double)
BINARY_ARR(vo_pow_d_u10, double)
BINARY_ARR(vo_pow_d_u35, double)
BINARY_ARR(vo_fmod_d, double)
UNARY_ARR(vo_sin_f_u10, float)
UNARY_ARR(vo_cos_f_u10, float)
UNARY_ARR(vo_tan_f_u10, float)
UNARY_ARR(vo_exp_f_u10, float)
UNARY_ARR(vo_exp_f_u35, float)
UNARY_ARR(vo_log_f_u10, float)
UNARY_ARR(vo_log_f_u35, float)
BINARY_ARR(vo_pow_f_u10, float)
BINARY_ARR(vo_pow_f_u35, float)
BINARY_ARR(vo_fmod_f, float)
UNARY_ARR(vo_sin_d_u35, double)
UNARY_ARR(vo_cos_d_u35, double)
UNARY_ARR(vo_tan_d_u35, double)
UNARY_ARR(vo_atan_d_u35, double)
UNARY_ARR(vo_asin_d_u10, double)
UNARY_ARR(vo_asin_d_u35, double)
UNARY_ARR(vo_acos_d_u10, double)
UNARY_ARR(vo_acos_d_u35, double)
BINARY_ARR(vo_atan2_d_u10, double)
BINARY_ARR(vo_atan2_d_u35, double)
BINARY_ARR(vo_fdim_d, double)
UNARY_ARR(vo_atan_f_u10, float)
UNARY_ARR(vo_atan_f_u35, float)
UNARY_ARR(vo_asin_f_u10, float)
UNARY_ARR(vo_asin_f_u35, float)
UNARY_ARR(vo_acos_f_u10, float)
UNARY_ARR(vo_acos_f_u35, float)
BINARY_ARR(vo_atan2_f_u10, float)
BINARY_ARR(vo_atan2_f_u35, float)
BINARY_ARR(vo_fdim_f, float)

/* fmod iteration count (for the step-curve property) */
int vo_fmod_d_iters(double x, double y) {
  g_fmod_steps = 0;
  (void)fmod_core(x, y);
  return g_fmod_steps;
}

/* debug hooks (tests only) */
void vo_dbg_log_dd(double a, double* hi, double* lo) {
  dd_t r = log_dd(a, 0.0, C_LOG1P_D, VEM_LOG1P_D_N);
  *hi = r.hi; *lo = r.lo;
}
double vo_dbg_exp_dd(double th, double tl) {
  dd_t t = {th, tl};
  return exp_dd(t);
}

/* every f32 trig lane takes the f32 Payne-Hanek path: forced variants alias */
void vo_sin_f_u10_ph_arr(const float* x, float* y, size_t n) { vo_sin_f_u10_arr(x, y, n); }
void vo_cos_f_u10_ph_arr(const float* x, float* y, size_t n) { vo_cos_f_u10_arr(x, y, n); }
void vo_tan_f_u10_ph_arr(const float* x, float* y, size_t n) { vo_tan_f_u10_arr(x, y, n); }
/* f32 u35 trig entry points are the u10 kernels (vem.h §8(f).1 note) */
void vo_sin_f_u35_arr(const float* x, float* y, size_t n) { vo_sin_f_u10_arr(x, y, n); }
void vo_cos_f_u35_arr(const float* x, float* y, size_t n) { vo_cos_f_u10_arr(x, y, n); }
void vo_tan_f_u35_arr(const float* x, float* y, size_t n) { vo_tan_f_u10_arr(x, y, n); }

/* DD operator hooks (tests only): the restated ddarith.hpp operators above,
 * exported so tests/test_oracle_reference.py can pin them bit-for-bit against
 * the reference's own templates (oracle/ref_shim.cpp). */
static inline dd_t dd_recip(double y) { /* ddarith.hpp:243-254 (FMA path) */
  double q = 1.0 / y;
  double e = fma(q, -y, 1.0);
  dd_t r = {q, q * e};
  return r;
}
void vo_dd_add2(double xh, double xl, double yh, double yl, double* h, double* l) {
  dd_t x = {xh, xl}, y = {yh, yl}, r = dd_add2(x, y);
  *h = r.hi; *l = r.lo;
}
void vo_dd_mul(double xh, double xl, double yh, double yl, double* h, double* l) {
  dd_t x = {xh, xl}, y = {yh, yl}, r = dd_mul(x, y);
  *h = r.hi; *l = r.lo;
}
void vo_dd_div(double xh, double xl, double yh, double yl, double* h, double* l) {
  dd_t x = {xh, xl}, y = {yh, yl}, r = dd_div(x, y);
  *h = r.hi; *l = r.lo;
}
void vo_dd_squ(double xh, double xl, double* h, double* l) {
  dd_t x = {xh, xl}, r = dd_squ(x);
  *h = r.hi; *l = r.lo;
}
void vo_dd_recip(double y, double* h, double* l) {
  dd_t r = dd_recip(y);
  *h = r.hi; *l = r.lo;
}
void vo_dd_normalize(double xh, double xl, double* h, double* l) {
  dd_t x = {xh, xl}, r = dd_normalize(x);
  *h = r.hi; *l = r.lo;
}
void vo_two_sum(double a, double b, double* s, double* e) {
  dd_t r = two_sum(a, b);
  *s = r.hi; *e = r.lo;
}
void vo_two_prod(double a, double b, double* p, double* e) {
  dd_t r = two_prod(a, b);
  *p = r.hi; *e = r.lo;
}
