/* TEST INFRASTRUCTURE ONLY -- ULP error against MPFR 4.2.1 (the paper's own
 * accuracy oracle), called through hand-declared
 * prototypes because the image ships libmpfr.so.6 without headers
 * (SURVEY.md Appendix A.4).
 *
 * ULP metric: |actual - exact| / ulp(exact), ulp taken at the
 * binade of the exact (256-bit) result, denormal-aware; both NaN or equal
 * infinities -> 0; a result that must round to +-inf counts 0 only if the
 * actual value is that infinity; any other special mismatch -> +inf.
 */
#include <math.h>
#include <stddef.h>
#include <stdint.h>

typedef struct { long prec; int sign; long exp; void* d; } mpfr_s;
typedef mpfr_s mpfr_t[1];
typedef int rnd_t;
#define RNDN 0

extern void mpfr_init2(mpfr_s*, long);
extern void mpfr_clear(mpfr_s*);
extern int mpfr_set_d(mpfr_s*, double, rnd_t);
extern double mpfr_get_d(const mpfr_s*, rnd_t);
extern int mpfr_sin(mpfr_s*, const mpfr_s*, rnd_t);
extern int mpfr_cos(mpfr_s*, const mpfr_s*, rnd_t);
extern int mpfr_tan(mpfr_s*, const mpfr_s*, rnd_t);
extern int mpfr_atan(mpfr_s*, const mpfr_s*, rnd_t);
extern int mpfr_exp(mpfr_s*, const mpfr_s*, rnd_t);
extern int mpfr_log(mpfr_s*, const mpfr_s*, rnd_t);
extern int mpfr_pow(mpfr_s*, const mpfr_s*, const mpfr_s*, rnd_t);
extern int mpfr_fmod(mpfr_s*, const mpfr_s*, const mpfr_s*, rnd_t);
extern int mpfr_sub_d(mpfr_s*, const mpfr_s*, double, rnd_t);
extern long mpfr_get_exp(const mpfr_s*);
extern int mpfr_mul_2si(mpfr_s*, const mpfr_s*, long, rnd_t);
extern int mpfr_nan_p(const mpfr_s*);
extern int mpfr_inf_p(const mpfr_s*);
extern int mpfr_zero_p(const mpfr_s*);
extern int mpfr_sgn(const mpfr_s*);
extern int mpfr_cmpabs(const mpfr_s*, const mpfr_s*);
extern int mpfr_set_ui_2exp(mpfr_s*, unsigned long, long, rnd_t);
extern int mpfr_abs(mpfr_s*, const mpfr_s*, rnd_t);
extern int mpfr_asin(mpfr_s*, const mpfr_s*, rnd_t);
extern int mpfr_acos(mpfr_s*, const mpfr_s*, rnd_t);
extern int mpfr_atan2(mpfr_s*, const mpfr_s*, const mpfr_s*, rnd_t);
extern int mpfr_dim(mpfr_s*, const mpfr_s*, const mpfr_s*, rnd_t);

enum { F_SIN = 0, F_COS, F_TAN, F_ATAN, F_EXP, F_LOG, F_POW, F_FMOD, F_ASIN, F_ACOS, F_ATAN2, F_FDIM };

#define PREC 320

static void eval(int fn, mpfr_s* r, mpfr_s* a, mpfr_s* b) {
  switch (fn) {
    case F_SIN: mpfr_sin(r, a, RNDN); break;
    case F_COS: mpfr_cos(r, a, RNDN); break;
    case F_TAN: mpfr_tan(r, a, RNDN); break;
    case F_ATAN: mpfr_atan(r, a, RNDN); break;
    case F_EXP: mpfr_exp(r, a, RNDN); break;
    case F_LOG: mpfr_log(r, a, RNDN); break;
    case F_POW: mpfr_pow(r, a, b, RNDN); break;
    case F_FMOD: mpfr_fmod(r, a, b, RNDN); break;
    case F_ASIN: mpfr_asin(r, a, RNDN); break;
    case F_ACOS: mpfr_acos(r, a, RNDN); break;
    case F_ATAN2: mpfr_atan2(r, a, b, RNDN); break;
    case F_FDIM: mpfr_dim(r, a, b, RNDN); break;
  }
}

/* p = precision (53 / 24), emin = minimum normal exponent, emax_plus1 = 1024/128 */
static double ulp_one(int fn, double x, double y, double act, int p, long emin, long emax) {
  mpfr_t a, b, r, d, lim;
  mpfr_init2(a, PREC); mpfr_init2(b, PREC); mpfr_init2(r, PREC); mpfr_init2(d, PREC);
  mpfr_init2(lim, PREC);
  mpfr_set_d(a, x, RNDN);
  mpfr_set_d(b, y, RNDN);
  eval(fn, r, a, b);
  double res;
  if (mpfr_nan_p(r)) {
    res = isnan(act) ? 0.0 : INFINITY;
  } else if (isnan(act)) {
    res = INFINITY;
  } else {
    /* overflow threshold: values >= 2^emax (1 - 2^-(p+1)) round to inf */
    mpfr_set_ui_2exp(lim, (1ul << (p + 1)) - 1, emax - p - 1, RNDN);
    int ovf = mpfr_inf_p(r) || (mpfr_cmpabs(r, lim) >= 0);
    if (ovf) {
      res = (isinf(act) && ((act > 0) == (mpfr_sgn(r) > 0))) ? 0.0 : INFINITY;
    } else if (isinf(act)) {
      res = INFINITY;
    } else {
      long e;
      if (mpfr_zero_p(r)) e = emin;
      else {
        e = mpfr_get_exp(r) - 1; /* |r| in [2^e, 2^(e+1)) */
        if (e < emin) e = emin;
      }
      long ue = e - (p - 1);
      mpfr_sub_d(d, r, act, RNDN);
      mpfr_abs(d, d, RNDN);
      mpfr_mul_2si(d, d, -ue, RNDN);
      res = mpfr_get_d(d, RNDN);
      /* sign of zero: +0 vs -0 for an exact zero result counts as 0 ulp */
    }
  }
  mpfr_clear(a); mpfr_clear(b); mpfr_clear(r); mpfr_clear(d); mpfr_clear(lim);
  return res;
}

void mp_ulp_d(int fn, const double* x, const double* y, const double* act, double* out, size_t n) {
#pragma omp parallel for schedule(dynamic, 256)
  for (size_t i = 0; i < n; i++) out[i] = ulp_one(fn, x[i], y ? y[i] : 0.0, act[i], 53, -1022, 1024);
}

void mp_ulp_f(int fn, const float* x, const float* y, const float* act, double* out, size_t n) {
#pragma omp parallel for schedule(dynamic, 256)
  for (size_t i = 0; i < n; i++)
    out[i] = ulp_one(fn, (double)x[i], y ? (double)y[i] : 0.0, (double)act[i], 24, -126, 128);
}

/* correctly rounded reference value (for golden fixtures) */
void mp_ref_d(int fn, const double* x, const double* y, double* out, size_t n) {
#pragma omp parallel for schedule(dynamic, 256)
  for (size_t i = 0; i < n; i++) {
    mpfr_t a, b, r;
    mpfr_init2(a, PREC); mpfr_init2(b, PREC); mpfr_init2(r, PREC);
    mpfr_set_d(a, x[i], RNDN);
    mpfr_set_d(b, y ? y[i] : 0.0, RNDN);
    eval(fn, r, a, b);
    out[i] = mpfr_get_d(r, RNDN);
    mpfr_clear(a); mpfr_clear(b); mpfr_clear(r);
  }
}
