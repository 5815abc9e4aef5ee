/* BENCH + TEST INFRASTRUCTURE ONLY -- upstream SLEEF 3.8.0 AVX-512 on the
 * host cores, the paper's own library, exported by torch's libtorch_cpu.so
 * (header torch/include/sleef.h).  Timed by bench.py next to the oracle port
 * (the CPU context number of BASELINE.md (C)) and used by
 * tests/test_sleef_crosscheck.py as the <= 1 ulp cross-check of north_star
 * ("within 1 ULP of the reference"); never part of the product.
 * Entry names follow vem's; a name SLEEF lacks returns -1.
 * SLEEF has no u35 exp / pow: those names time the u10 entry (labelled). */
#include <immintrin.h>
#include <omp.h>
#include <stddef.h>
#include <string.h>

__m512d Sleef_sind8_u10avx512f(__m512d);
__m512d Sleef_cosd8_u10avx512f(__m512d);
__m512d Sleef_tand8_u10avx512f(__m512d);
__m512d Sleef_atand8_u10avx512f(__m512d);
__m512d Sleef_sind8_u35avx512f(__m512d);
__m512d Sleef_cosd8_u35avx512f(__m512d);
__m512d Sleef_tand8_u35avx512f(__m512d);
__m512d Sleef_atand8_u35avx512f(__m512d);
__m512d Sleef_expd8_u10avx512f(__m512d);
__m512d Sleef_logd8_u10avx512f(__m512d);
__m512d Sleef_logd8_u35avx512f(__m512d);
__m512d Sleef_powd8_u10avx512f(__m512d, __m512d);
__m512d Sleef_fmodd8_avx512f(__m512d, __m512d);
__m512 Sleef_sinf16_u10avx512f(__m512);
__m512 Sleef_cosf16_u10avx512f(__m512);
__m512 Sleef_tanf16_u10avx512f(__m512);
__m512 Sleef_expf16_u10avx512f(__m512);
__m512 Sleef_logf16_u10avx512f(__m512);
__m512 Sleef_logf16_u35avx512f(__m512);
__m512 Sleef_powf16_u10avx512f(__m512, __m512);
__m512 Sleef_fmodf16_avx512f(__m512, __m512);
__m512d Sleef_asind8_u10avx512f(__m512d);
__m512d Sleef_asind8_u35avx512f(__m512d);
__m512d Sleef_acosd8_u10avx512f(__m512d);
__m512d Sleef_acosd8_u35avx512f(__m512d);
__m512d Sleef_atan2d8_u10avx512f(__m512d, __m512d);
__m512d Sleef_atan2d8_u35avx512f(__m512d, __m512d);
__m512d Sleef_fdimd8_avx512f(__m512d, __m512d);
__m512 Sleef_sinf16_u35avx512f(__m512);
__m512 Sleef_cosf16_u35avx512f(__m512);
__m512 Sleef_tanf16_u35avx512f(__m512);
__m512 Sleef_atanf16_u10avx512f(__m512);
__m512 Sleef_atanf16_u35avx512f(__m512);
__m512 Sleef_asinf16_u10avx512f(__m512);
__m512 Sleef_asinf16_u35avx512f(__m512);
__m512 Sleef_acosf16_u10avx512f(__m512);
__m512 Sleef_acosf16_u35avx512f(__m512);
__m512 Sleef_atan2f16_u10avx512f(__m512, __m512);
__m512 Sleef_atan2f16_u35avx512f(__m512, __m512);
__m512 Sleef_fdimf16_avx512f(__m512, __m512);

typedef __m512d (*ud)(__m512d);
typedef __m512d (*bd)(__m512d, __m512d);
typedef __m512 (*uf)(__m512);
typedef __m512 (*bf)(__m512, __m512);

static void* pick(const char* n, int* kind) {
  /* kind: 0 unary d, 1 binary d, 2 unary f, 3 binary f */
#define M(str, fn, k) if (!strcmp(n, str)) { *kind = k; return (void*)fn; }
  M("sin_d_u10", Sleef_sind8_u10avx512f, 0) M("cos_d_u10", Sleef_cosd8_u10avx512f, 0)
  M("tan_d_u10", Sleef_tand8_u10avx512f, 0) M("sin_d_u10_ph", Sleef_sind8_u10avx512f, 0)
  M("cos_d_u10_ph", Sleef_cosd8_u10avx512f, 0) M("tan_d_u10_ph", Sleef_tand8_u10avx512f, 0)
  M("atan_d_u10", Sleef_atand8_u10avx512f, 0) M("exp_d_u10", Sleef_expd8_u10avx512f, 0)
  M("exp_d_u35", Sleef_expd8_u10avx512f, 0) M("log_d_u10", Sleef_logd8_u10avx512f, 0)
  M("log_d_u35", Sleef_logd8_u35avx512f, 0) M("pow_d_u10", Sleef_powd8_u10avx512f, 1)
  M("pow_d_u35", Sleef_powd8_u10avx512f, 1) M("fmod_d", Sleef_fmodd8_avx512f, 1)
  M("sin_f_u10", Sleef_sinf16_u10avx512f, 2) M("cos_f_u10", Sleef_cosf16_u10avx512f, 2)
  M("tan_f_u10", Sleef_tanf16_u10avx512f, 2) M("sin_f_u10_ph", Sleef_sinf16_u10avx512f, 2)
  M("cos_f_u10_ph", Sleef_cosf16_u10avx512f, 2) M("tan_f_u10_ph", Sleef_tanf16_u10avx512f, 2)
  M("exp_f_u10", Sleef_expf16_u10avx512f, 2) M("exp_f_u35", Sleef_expf16_u10avx512f, 2)
  M("log_f_u10", Sleef_logf16_u10avx512f, 2) M("log_f_u35", Sleef_logf16_u35avx512f, 2)
  M("pow_f_u10", Sleef_powf16_u10avx512f, 3) M("pow_f_u35", Sleef_powf16_u10avx512f, 3)
  M("fmod_f", Sleef_fmodf16_avx512f, 3)
  M("sin_d_u35", Sleef_sind8_u35avx512f, 0) M("cos_d_u35", Sleef_cosd8_u35avx512f, 0)
  M("tan_d_u35", Sleef_tand8_u35avx512f, 0) M("atan_d_u35", Sleef_atand8_u35avx512f, 0)
  M("asin_d_u10", Sleef_asind8_u10avx512f, 0) M("asin_d_u35", Sleef_asind8_u35avx512f, 0)
  M("acos_d_u10", Sleef_acosd8_u10avx512f, 0) M("acos_d_u35", Sleef_acosd8_u35avx512f, 0)
  M("atan2_d_u10", Sleef_atan2d8_u10avx512f, 1) M("atan2_d_u35", Sleef_atan2d8_u35avx512f, 1)
  M("fdim_d", Sleef_fdimd8_avx512f, 1)
  M("sin_f_u35", Sleef_sinf16_u35avx512f, 2) M("cos_f_u35", Sleef_cosf16_u35avx512f, 2)
  M("tan_f_u35", Sleef_tanf16_u35avx512f, 2) M("atan_f_u10", Sleef_atanf16_u10avx512f, 2)
  M("atan_f_u35", Sleef_atanf16_u35avx512f, 2) M("asin_f_u10", Sleef_asinf16_u10avx512f, 2)
  M("asin_f_u35", Sleef_asinf16_u35avx512f, 2) M("acos_f_u10", Sleef_acosf16_u10avx512f, 2)
  M("acos_f_u35", Sleef_acosf16_u35avx512f, 2) M("atan2_f_u10", Sleef_atan2f16_u10avx512f, 3)
  M("atan2_f_u35", Sleef_atan2f16_u35avx512f, 3) M("fdim_f", Sleef_fdimf16_avx512f, 3)
#undef M
  return 0;
}

/* Evaluates over n elements (n a multiple of 16) on `threads` OpenMP threads
 * with static contiguous chunks; returns wall seconds, or -1 if unknown. */
double sleef_run(const char* name, const void* x, const void* y, void* out, size_t n, int threads) {
  int kind = -1;
  void* f = pick(name, &kind);
  if (!f || (n % 16)) return -1.0;
  double t0 = omp_get_wtime();
  if (kind == 0) {
    const double* a = (const double*)x; double* o = (double*)out;
#pragma omp parallel for schedule(static) num_threads(threads)
    for (size_t i = 0; i < n; i += 8) _mm512_storeu_pd(o + i, ((ud)f)(_mm512_loadu_pd(a + i)));
  } else if (kind == 1) {
    const double* a = (const double*)x; const double* b = (const double*)y; double* o = (double*)out;
#pragma omp parallel for schedule(static) num_threads(threads)
    for (size_t i = 0; i < n; i += 8)
      _mm512_storeu_pd(o + i, ((bd)f)(_mm512_loadu_pd(a + i), _mm512_loadu_pd(b + i)));
  } else if (kind == 2) {
    const float* a = (const float*)x; float* o = (float*)out;
#pragma omp parallel for schedule(static) num_threads(threads)
    for (size_t i = 0; i < n; i += 16) _mm512_storeu_ps(o + i, ((uf)f)(_mm512_loadu_ps(a + i)));
  } else {
    const float* a = (const float*)x; const float* b = (const float*)y; float* o = (float*)out;
#pragma omp parallel for schedule(static) num_threads(threads)
    for (size_t i = 0; i < n; i += 16)
      _mm512_storeu_ps(o + i, ((bf)f)(_mm512_loadu_ps(a + i), _mm512_loadu_ps(b + i)));
  }
  return omp_get_wtime() - t0;
}
