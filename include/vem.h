/* vem -- B200-native batched elementwise C99 math (SLEEF-class), C ABI.
 *
 * Drop-in boundary for the reference's per-function, per-precision,
 * per-accuracy kernels.  The reference (/root/reference) specifies them only
 * by name -- "name, name_u35, name_det" -- over one lane
 * vector per call (backend.hpp:294-305 Vd<B>; SLEEF's own boundary is one
 * vector register per call).  The B200 boundary is one
 * device ARRAY per call:
 *
 *   unary :  int vem_<fn>_<d|f>_<acc>(const T* x, T* y, size_t n, vem_stream_t s)
 *   binary:  int vem_<fn>_<d|f>_<acc>(const T* x, const T* y2, T* out, size_t n, vem_stream_t s)
 *
 *  - pointers are caller-owned DEVICE buffers (in-place allowed), no
 *    allocation on the call path, asynchronous on stream `s` (NULL = legacy
 *    default stream);
 *  - return 0 or a cudaError_t code (launch/configuration errors only); math
 *    errors stay in-band exactly as in the reference: NaN/Inf, no errno, no FP
 *    exceptions; NaN results are the
 *    canonical quiet NaN (0x7ff8000000000000 / 0x7fc00000);
 *  - reentrant from any host thread, on any device (launch state is cached
 *    per device); the Payne-Hanek tables are device constants (replace the
 *    lazy singleton ph_table(), ph_table.cpp:182-185) staged per CTA into
 *    shared memory in bank-conflict-aware layouts (the binary32 limbs
 *    replicated per bank group, the binary64 window words as two 8-byte
 *    arrays); the binary64 selector kernels (sin/cos/tan_d) stage theirs
 *    lazily, when a CTA first meets an argument above 1e14;
 *  - results are bit-identical to the deterministic CPU oracle (oracle/).
 *
 * Accuracy: *_u10 <= 1.0 ulp, *_u35 <= 3.5 ulp (vs MPFR), fmod exact.
 * Each entry below cites the reference item it replaces.
 */
#ifndef VEM_H
#define VEM_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef void* vem_stream_t; /* a cudaStream_t */

/* ---- float64 -------------------------------------------------------- */
/* sin/cos: SPEC.md:362-370; reduction reduction.hpp:189 */
int vem_sin_d_u10(const double* x, double* y, size_t n, vem_stream_t s);
int vem_cos_d_u10(const double* x, double* y, size_t n, vem_stream_t s);
/* tan: SPEC.md:371-379 */
int vem_tan_d_u10(const double* x, double* y, size_t n, vem_stream_t s);
/* forced Payne-Hanek variants (config 3: every lane takes
 * payne_hanek_reduce, reduction.hpp:89; valid for all finite x) */
int vem_sin_d_u10_ph(const double* x, double* y, size_t n, vem_stream_t s);
int vem_cos_d_u10_ph(const double* x, double* y, size_t n, vem_stream_t s);
int vem_tan_d_u10_ph(const double* x, double* y, size_t n, vem_stream_t s);
/* atan: SPEC.md:388-395 */
int vem_atan_d_u10(const double* x, double* y, size_t n, vem_stream_t s);
/* exp: SPEC.md:404-411, constants.hpp:42-54 */
int vem_exp_d_u10(const double* x, double* y, size_t n, vem_stream_t s);
int vem_exp_d_u35(const double* x, double* y, size_t n, vem_stream_t s);
/* log: SPEC.md:396-403, constants.hpp:48-50 */
int vem_log_d_u10(const double* x, double* y, size_t n, vem_stream_t s);
int vem_log_d_u35(const double* x, double* y, size_t n, vem_stream_t s);
/* pow: SPEC.md:412-419 */
int vem_pow_d_u10(const double* x, const double* y2, double* out, size_t n, vem_stream_t s);
int vem_pow_d_u35(const double* x, const double* y2, double* out, size_t n, vem_stream_t s);
/* fmod: Alg. 1 PAPER.md:958-975 (exact) */
int vem_fmod_d(const double* x, const double* y2, double* out, size_t n, vem_stream_t s);

/* ---- float32 (new: the reference is double-only) -------- */
int vem_sin_f_u10(const float* x, float* y, size_t n, vem_stream_t s);
int vem_cos_f_u10(const float* x, float* y, size_t n, vem_stream_t s);
int vem_tan_f_u10(const float* x, float* y, size_t n, vem_stream_t s);
int vem_sin_f_u10_ph(const float* x, float* y, size_t n, vem_stream_t s);
int vem_cos_f_u10_ph(const float* x, float* y, size_t n, vem_stream_t s);
int vem_tan_f_u10_ph(const float* x, float* y, size_t n, vem_stream_t s);
int vem_exp_f_u10(const float* x, float* y, size_t n, vem_stream_t s);
int vem_exp_f_u35(const float* x, float* y, size_t n, vem_stream_t s);
int vem_log_f_u10(const float* x, float* y, size_t n, vem_stream_t s);
int vem_log_f_u35(const float* x, float* y, size_t n, vem_stream_t s);
int vem_pow_f_u10(const float* x, const float* y2, float* out, size_t n, vem_stream_t s);
int vem_pow_f_u35(const float* x, const float* y2, float* out, size_t n, vem_stream_t s);
int vem_fmod_f(const float* x, const float* y2, float* out, size_t n, vem_stream_t s);

/* ---- SURVEY.md §8(f).1 additions ---------------------------------------
 * u35 trig/atan (SPEC.md DESIGN DECISIONS: same reductions, shorter
 * polynomials, single-double reconstruction), asin/acos,
 * atan2(y, x) (x2 = x, first operand = y), fdim
 * (exact).  Float32 variants evaluate binary64 internals;
 * the f32 u35 trig entry points are the u10 kernels (already <= 0.5001 ulp;
 * the reduction dominates their cost). */
int vem_sin_d_u35(const double* x, double* y, size_t n, vem_stream_t s);
int vem_cos_d_u35(const double* x, double* y, size_t n, vem_stream_t s);
int vem_tan_d_u35(const double* x, double* y, size_t n, vem_stream_t s);
int vem_atan_d_u35(const double* x, double* y, size_t n, vem_stream_t s);
int vem_asin_d_u10(const double* x, double* y, size_t n, vem_stream_t s);
int vem_asin_d_u35(const double* x, double* y, size_t n, vem_stream_t s);
int vem_acos_d_u10(const double* x, double* y, size_t n, vem_stream_t s);
int vem_acos_d_u35(const double* x, double* y, size_t n, vem_stream_t s);
int vem_atan2_d_u10(const double* y, const double* x, double* out, size_t n, vem_stream_t s);
int vem_atan2_d_u35(const double* y, const double* x, double* out, size_t n, vem_stream_t s);
int vem_fdim_d(const double* x, const double* y2, double* out, size_t n, vem_stream_t s);
int vem_sin_f_u35(const float* x, float* y, size_t n, vem_stream_t s);
int vem_cos_f_u35(const float* x, float* y, size_t n, vem_stream_t s);
int vem_tan_f_u35(const float* x, float* y, size_t n, vem_stream_t s);
int vem_atan_f_u10(const float* x, float* y, size_t n, vem_stream_t s);
int vem_atan_f_u35(const float* x, float* y, size_t n, vem_stream_t s);
int vem_asin_f_u10(const float* x, float* y, size_t n, vem_stream_t s);
int vem_asin_f_u35(const float* x, float* y, size_t n, vem_stream_t s);
int vem_acos_f_u10(const float* x, float* y, size_t n, vem_stream_t s);
int vem_acos_f_u35(const float* x, float* y, size_t n, vem_stream_t s);
int vem_atan2_f_u10(const float* y, const float* x, float* out, size_t n, vem_stream_t s);
int vem_atan2_f_u35(const float* y, const float* x, float* out, size_t n, vem_stream_t s);
int vem_fdim_f(const float* x, const float* y2, float* out, size_t n, vem_stream_t s);

/* ---- reduction entry points (parity anchors) ------------------------- */
/* trig_reduce<ScalarFmaDet> (reduction.hpp:189-206): r = hi + lo, q = quadrant mod 4 */
int vem_trig_reduce_d(const double* x, double* r_hi, double* r_lo, int* q, size_t n, vem_stream_t s);
/* cody_waite_reduce(x, level) (reduction.hpp:148), level 1 or 2 */
int vem_cw_reduce_d(const double* x, double* r_hi, double* r_lo, int* q, size_t n, int level, vem_stream_t s);
/* payne_hanek_reduce (reduction.hpp:89-137), repaired */
int vem_ph_reduce_d(const double* x, double* r_hi, double* r_lo, int* q, size_t n, vem_stream_t s);
/* float32 Payne-Hanek (binary64 residual) */
int vem_ph_reduce_f(const float* x, double* r, int* q, size_t n, vem_stream_t s);

/* ---- tables / introspection ------------------------------------------ */
/* Copies the repaired f64 Payne-Hanek table (32768 bytes, layout
 * ph_table.hpp:14-15, serialize ph_table.cpp:187-195) to host memory. */
int vem_ph_table_d(unsigned char* out32768);
/* Number of __global__ kernel launches issued by this library so far (for
 * the bench's gpu_launches evidence).  Thread-safe. */
uint64_t vem_launch_count(void);
/* Library version string. */
const char* vem_version(void);

/* FP64 (kind 0) / FP32 (kind 1) FMA pipe throughput microbenchmark on the
 * current device: independent FMA chains, no memory traffic; writes Gop/s. */
int vem_probe_peak(int kind, int iters, double* gops_out);

/* ---- multi-GPU host driver ------------------- */
/* Evaluates function `name` (e.g. "sin_d_u10") over HOST arrays sharded
 * contiguously across `ngpu` devices: one host thread per device, its own
 * stream, H2D + kernel + D2H per shard, no collective on the data path.
 * Returns 0 or a cudaError_t.  `ms_out` (may be NULL) receives the max over
 * devices of the kernel time in milliseconds (CUDA events). */
int vem_run_sharded(const char* name, const void* x, const void* y2, void* out, size_t n, int ngpu,
                    double* ms_out);
/* Same with an explicit device per shard (shard g on devices[g]; a device may
 * appear more than once -- each shard still gets its own host thread and
 * stream).  vem_run_sharded(..., ngpu, ...) == devices {0, 1, ..., ngpu-1}. */
int vem_run_sharded_on(const char* name, const void* x, const void* y2, void* out, size_t n, int ngpu,
                       const int* devices, double* ms_out);

#ifdef __cplusplus
}
#endif

#endif /* VEM_H */
