// vem.hpp -- C++ host mirror of the reference's function interface over the
// C ABI of vem.h (device arrays).
//
// The reference names each kernel `name`, `name_u35`, `name_det`
// and writes them as templates over a lane backend
// (backend.hpp:294-305).  Here the same names are overloads on the element
// type (double / float) taking caller-owned device pointers, so a reference
// user switches
//     vem::Vd<B> y = vem::sin(x);            // one lane vector
// to
//     vem::gpu::sin(x_dev, y_dev, n, stream); // one device array
// Error behaviour matches the reference: math errors are in-band (NaN/Inf),
// the return value only reports CUDA launch/configuration errors (0 = ok).
// The u10 kernels are the deterministic variants (bit-identical to the CPU
// oracle), so name_det == name.
#pragma once

#include <cstddef>

#include "vem.h"

namespace vem {
namespace gpu {

using stream_t = vem_stream_t;

#define VEM_UNARY_PAIR(NAME, DFN, FFN)                                                                \
  inline int NAME(const double* x, double* y, size_t n, stream_t s = nullptr) { return DFN(x, y, n, s); } \
  inline int NAME(const float* x, float* y, size_t n, stream_t s = nullptr) { return FFN(x, y, n, s); }

VEM_UNARY_PAIR(sin, vem_sin_d_u10, vem_sin_f_u10)
VEM_UNARY_PAIR(cos, vem_cos_d_u10, vem_cos_f_u10)
VEM_UNARY_PAIR(tan, vem_tan_d_u10, vem_tan_f_u10)
VEM_UNARY_PAIR(sin_det, vem_sin_d_u10, vem_sin_f_u10)
VEM_UNARY_PAIR(cos_det, vem_cos_d_u10, vem_cos_f_u10)
VEM_UNARY_PAIR(tan_det, vem_tan_d_u10, vem_tan_f_u10)
VEM_UNARY_PAIR(sin_ph, vem_sin_d_u10_ph, vem_sin_f_u10_ph)
VEM_UNARY_PAIR(cos_ph, vem_cos_d_u10_ph, vem_cos_f_u10_ph)
VEM_UNARY_PAIR(tan_ph, vem_tan_d_u10_ph, vem_tan_f_u10_ph)
VEM_UNARY_PAIR(exp, vem_exp_d_u10, vem_exp_f_u10)
VEM_UNARY_PAIR(exp_u35, vem_exp_d_u35, vem_exp_f_u35)
VEM_UNARY_PAIR(exp_det, vem_exp_d_u10, vem_exp_f_u10)
VEM_UNARY_PAIR(log, vem_log_d_u10, vem_log_f_u10)
VEM_UNARY_PAIR(log_u35, vem_log_d_u35, vem_log_f_u35)
VEM_UNARY_PAIR(log_det, vem_log_d_u10, vem_log_f_u10)
VEM_UNARY_PAIR(sin_u35, vem_sin_d_u35, vem_sin_f_u35)
VEM_UNARY_PAIR(cos_u35, vem_cos_d_u35, vem_cos_f_u35)
VEM_UNARY_PAIR(tan_u35, vem_tan_d_u35, vem_tan_f_u35)
VEM_UNARY_PAIR(atan, vem_atan_d_u10, vem_atan_f_u10)
VEM_UNARY_PAIR(atan_u35, vem_atan_d_u35, vem_atan_f_u35)
VEM_UNARY_PAIR(atan_det, vem_atan_d_u10, vem_atan_f_u10)
VEM_UNARY_PAIR(asin, vem_asin_d_u10, vem_asin_f_u10)
VEM_UNARY_PAIR(asin_u35, vem_asin_d_u35, vem_asin_f_u35)
VEM_UNARY_PAIR(asin_det, vem_asin_d_u10, vem_asin_f_u10)
VEM_UNARY_PAIR(acos, vem_acos_d_u10, vem_acos_f_u10)
VEM_UNARY_PAIR(acos_u35, vem_acos_d_u35, vem_acos_f_u35)
VEM_UNARY_PAIR(acos_det, vem_acos_d_u10, vem_acos_f_u10)
#undef VEM_UNARY_PAIR

#define VEM_BINARY_PAIR(NAME, DFN, FFN)                                                                  \
  inline int NAME(const double* x, const double* y, double* o, size_t n, stream_t s = nullptr) {        \
    return DFN(x, y, o, n, s);                                                                          \
  }                                                                                                     \
  inline int NAME(const float* x, const float* y, float* o, size_t n, stream_t s = nullptr) {           \
    return FFN(x, y, o, n, s);                                                                          \
  }
VEM_BINARY_PAIR(pow, vem_pow_d_u10, vem_pow_f_u10)
VEM_BINARY_PAIR(pow_u35, vem_pow_d_u35, vem_pow_f_u35)
VEM_BINARY_PAIR(pow_det, vem_pow_d_u10, vem_pow_f_u10)
VEM_BINARY_PAIR(fmod, vem_fmod_d, vem_fmod_f)
VEM_BINARY_PAIR(fmod_det, vem_fmod_d, vem_fmod_f)
VEM_BINARY_PAIR(atan2, vem_atan2_d_u10, vem_atan2_f_u10)  // atan2(y, x): first operand y
VEM_BINARY_PAIR(atan2_u35, vem_atan2_d_u35, vem_atan2_f_u35)
VEM_BINARY_PAIR(atan2_det, vem_atan2_d_u10, vem_atan2_f_u10)
VEM_BINARY_PAIR(fdim, vem_fdim_d, vem_fdim_f)
VEM_BINARY_PAIR(fdim_det, vem_fdim_d, vem_fdim_f)
#undef VEM_BINARY_PAIR

// reduction.hpp:189 trig_reduce / reduction.hpp:148 cody_waite_reduce /
// reduction.hpp:89 payne_hanek_reduce over device arrays.
inline int trig_reduce(const double* x, double* hi, double* lo, int* q, size_t n, stream_t s = nullptr) {
  return vem_trig_reduce_d(x, hi, lo, q, n, s);
}
inline int cody_waite_reduce(const double* x, int level, double* hi, double* lo, int* q, size_t n,
                             stream_t s = nullptr) {
  return vem_cw_reduce_d(x, hi, lo, q, n, level, s);
}
inline int payne_hanek_reduce(const double* x, double* hi, double* lo, int* q, size_t n, stream_t s = nullptr) {
  return vem_ph_reduce_d(x, hi, lo, q, n, s);
}

}  // namespace gpu
}  // namespace vem
