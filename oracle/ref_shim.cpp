// TEST INFRASTRUCTURE ONLY (oracle/_ref).  extern "C" shim over the
// *reference's own* headers (/root/reference/proj/core, copied into
// oracle/_ref/src/<variant>/ and patched by oracle/ref_build.py) so that the
// reference's reduction and DD code can be called from pytest via ctypes.
//
// Built twice:
//   variant "gcc"      : only the GCC vector_size patch --
//                        the reference's shipped semantics, incl. its defective
//                        Payne-Hanek table (ph_table.cpp:114).
//   variant "repaired" : + ph_table.cpp:114 off-by-one removed and
//                        `u = two_sum(u.hi, u.lo)` after each rfrac in
//                        payne_hanek_reduce (reduction.hpp:108-112); the
//                        mod-4 table is supplied by the caller (deserialize).
// The shim itself contains no math: every call forwards to reference code.
#include <cstdint>
#include <cstring>
#include <vector>

#include "vem/reduction.hpp"

using B = vem::ScalarFmaDet;  // backend.hpp:430, the FMA-deterministic config

namespace {
inline void put(const vem::Reduced<B>& r, double* hi, double* lo, int64_t* q) {
  *hi = r.r.hi.raw;
  *lo = r.r.lo.raw;
  *q = r.q.raw;
}
vem::PayneHanekTable g_user_table;
}  // namespace

extern "C" {

// reduction.hpp:148 (level 1 / level 2)
void ref_cw_reduce(const double* x, double* hi, double* lo, int64_t* q, size_t n, int level) {
  for (size_t i = 0; i < n; i++) put(vem::cody_waite_reduce<B>(vem::Vd<B>{x[i]}, level), hi + i, lo + i, q + i);
}

// reduction.hpp:140 with the process-wide table (ph_table.cpp:182)
void ref_ph_reduce(const double* x, double* hi, double* lo, int64_t* q, size_t n) {
  for (size_t i = 0; i < n; i++) put(vem::payne_hanek_reduce<B>(vem::Vd<B>{x[i]}), hi + i, lo + i, q + i);
}

// reduction.hpp:89 with a caller-supplied serialized table (ph_table.hpp:37-38)
int ref_set_table(const unsigned char* bytes, size_t nbytes) {
  try {
    g_user_table = vem::PayneHanekTable::deserialize(std::vector<unsigned char>(bytes, bytes + nbytes));
  } catch (...) {
    return -1;
  }
  return 0;
}
void ref_ph_reduce_table(const double* x, double* hi, double* lo, int64_t* q, size_t n) {
  for (size_t i = 0; i < n; i++)
    put(vem::payne_hanek_reduce<B>(vem::Vd<B>{x[i]}, g_user_table), hi + i, lo + i, q + i);
}

// reduction.hpp:189 (Det policy, per lane)
void ref_trig_reduce(const double* x, double* hi, double* lo, int64_t* q, size_t n) {
  for (size_t i = 0; i < n; i++) put(vem::trig_reduce<B>(vem::Vd<B>{x[i]}), hi + i, lo + i, q + i);
}

// ph_table.cpp:168 + ph_table.cpp:187 (32768 bytes)
void ref_build_table(unsigned char* out32768) {
  auto v = vem::build_ph_table().serialize();
  std::memcpy(out32768, v.data(), v.size());
}

// ddarith.hpp operators, 2-limb in/out
void ref_two_sum(double a, double b, double* s, double* e) {
  auto r = vem::two_sum<B>(vem::Vd<B>{a}, vem::Vd<B>{b});
  *s = r.hi.raw; *e = r.lo.raw;
}
void ref_two_prod(double a, double b, double* p, double* e) {
  auto r = vem::two_prod<B>(vem::Vd<B>{a}, vem::Vd<B>{b});
  *p = r.hi.raw; *e = r.lo.raw;
}
static vem::Dd<B> mk(double h, double l) { return {vem::Vd<B>{h}, vem::Vd<B>{l}}; }
void ref_dd_add2(double xh, double xl, double yh, double yl, double* h, double* l) {
  auto r = vem::dd_add2<B>(mk(xh, xl), mk(yh, yl));
  *h = r.hi.raw; *l = r.lo.raw;
}
void ref_dd_mul(double xh, double xl, double yh, double yl, double* h, double* l) {
  auto r = vem::dd_mul<B>(mk(xh, xl), mk(yh, yl));
  *h = r.hi.raw; *l = r.lo.raw;
}
void ref_dd_div(double xh, double xl, double yh, double yl, double* h, double* l) {
  auto r = vem::dd_div<B>(mk(xh, xl), mk(yh, yl));
  *h = r.hi.raw; *l = r.lo.raw;
}
void ref_dd_squ(double xh, double xl, double* h, double* l) {
  auto r = vem::dd_squ<B>(mk(xh, xl));
  *h = r.hi.raw; *l = r.lo.raw;
}
void ref_dd_recip(double y, double* h, double* l) {
  auto r = vem::dd_recip<B>(vem::Vd<B>{y});
  *h = r.hi.raw; *l = r.lo.raw;
}
void ref_dd_normalize(double xh, double xl, double* h, double* l) {
  auto r = vem::dd_normalize<B>(mk(xh, xl));
  *h = r.hi.raw; *l = r.lo.raw;
}
double ref_round_nearest(double x) { return vem::round_nearest<B>(vem::Vd<B>{x}).raw; }
double ref_ldexp2(double x, int64_t e) { return vem::ldexp2<B>(vem::Vd<B>{x}, vem::Vl<B>{e}).raw; }

}  // extern "C"
