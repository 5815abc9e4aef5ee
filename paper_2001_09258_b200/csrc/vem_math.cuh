// Per-lane device math for the vem kernels (sm_100a).
//
// One CUDA thread = one lane of the reference's Backend<1, Fma=true, Det=true>
// (backend.hpp:62-144, ScalarFmaDet backend.hpp:430): opmask `select` becomes a
// predicated SEL, `all/any` skips become plain per-lane branches that a warp
// only pays for when its lanes disagree.  Every floating-point operation is
// written out explicitly (the library is compiled with --fmad=false; fused
// operations are explicit fma()), in exactly the order of the CPU oracle
// (oracle/vem_oracle.c), so results are bit-identical to it.
//
// DD arithmetic follows ddarith.hpp (FMA paths); the reduction follows
// reduction.hpp:31-212 with the Payne-Hanek repairs of SURVEY.md §0 item 4.
#pragma once

#include <cstdint>

#include "vem_coeffs.h"
#include "vem_ph_tables.h"
#include "vem_log_tables.h"

namespace vem {

struct dd { double hi, lo; };

// ---------------------------------------------------------------- bits
__device__ __forceinline__ uint64_t bits_d(double x) { return (uint64_t)__double_as_longlong(x); }
__device__ __forceinline__ double from_bits_d(uint64_t u) { return __longlong_as_double((long long)u); }
__device__ __forceinline__ uint32_t bits_f(float x) { return (uint32_t)__float_as_uint(x); }
__device__ __forceinline__ float from_bits_f(uint32_t u) { return __uint_as_float(u); }

constexpr uint64_t kCanonNanD = 0x7ff8000000000000ull;
constexpr uint32_t kCanonNanF = 0x7fc00000u;
__device__ __forceinline__ double canon_d(double y) { return (y != y) ? from_bits_d(kCanonNanD) : y; }
__device__ __forceinline__ float canon_f(float y) { return (y != y) ? from_bits_f(kCanonNanF) : y; }

// constants.hpp:14-58
constexpr double kPio2Qd0 = 0x1.921fb54442d18p+0;
constexpr double kPio2Qd1 = 0x1.1a62633145c07p-54;
constexpr double kPio2Qd2 = -0x1.f1976b7ed8fbcp-110;
constexpr double kPio2Qd3 = 0x1.4cf98e804177dp-164;
constexpr double kTwoOverPi = 0x1.45f306dc9c883p-1;
constexpr double kCw1P0 = 0x1.921fb54442d20p+0;
constexpr double kCw1T1 = -0x1.ee59d9cceba40p-50;
constexpr double kCw1T2 = 0x1.b839a252049c1p-104;
constexpr double kCw2A = 0x1.921fb58000000p+0;
constexpr double kCw2B = -0x1.dde9740000000p-27;
constexpr double kCw2C = 0x1.1a62630000000p-54;
constexpr double kCw2D1 = 0x1.8a2e03707344ap-81;
constexpr double kCw2D2 = 0x1.024e088a67cc7p-135;
constexpr double kInvLn2 = 0x1.71547652b82fep+0;
constexpr double kExpL1 = 0x1.62e42fefa3800p-1;
constexpr double kExpL2 = 0x1.ef35793c76730p-45;
constexpr double kLn2Hi = 0x1.62e42fefa39efp-1;
constexpr double kLn2Lo = 0x1.abc9e3b39803fp-56;
constexpr double kExpOvf = 0x1.62e42fefa39efp+9;
constexpr double kExpUnf = -0x1.74910d52d3051p+9;
constexpr double kCw1Max = 15.0;
constexpr double kCw2Max = 1e14;
constexpr double kFourThirds = 0x1.5555555555555p+0;
constexpr double kTanPi8 = 0x1.a827999fcef32p-2;
constexpr double kTan3Pi8 = 0x1.3504f333f9de6p+1;
constexpr double kPio4Hi = 0x1.921fb54442d18p-1;
constexpr double kPio4Lo = 0x1.1a62633145c07p-55;
constexpr double kDblMax = 1.7976931348623157e308;
constexpr double kInf = __builtin_huge_val();
constexpr float kInfF = __builtin_huge_valf();


// Constant-bank copies of scalar constants used as DFMA/DMUL operands: a
// c[bank][offset] operand is free, a 64-bit immediate costs two UMOVs per use.
__constant__ double ccShift = 0x1.8p52;
__constant__ double ccInvLn2 = 0x1.71547652b82fep+0;
__constant__ double ccExpL1 = 0x1.62e42fefa3800p-1;
__constant__ double ccExpL2 = 0x1.ef35793c76730p-45;
__constant__ double ccLn2Hi = 0x1.62e42fefa39efp-1;
__constant__ double ccLn2H42 = VEM_LN2_H42;
__constant__ double ccLn2T42 = VEM_LN2_T42;
__constant__ double ccExpjInv = VEM_EXPJ_INV;
__constant__ double ccExpjL1 = VEM_EXPJ_L1;
__constant__ double ccExpjL2 = VEM_EXPJ_L2;
__constant__ double ccPio2Qd0 = 0x1.921fb54442d18p+0;
__constant__ double ccPio2Qd1 = 0x1.1a62633145c07p-54;
__constant__ double ccSixth = 0x1.5555555555555p-3;

// Coefficients live in the constant bank: uniform operands of DFMA.
__constant__ double cSinD[] = VEM_SIN_D_ARR;
__constant__ double cCosD[] = VEM_COS_D_ARR;
__constant__ double cTanD[] = VEM_TAN_D_ARR;
__constant__ double cAtanD[] = VEM_ATAN_D_ARR;
__constant__ double cExpD[] = VEM_EXP_D_ARR;
__constant__ double cExpDU35[] = VEM_EXP_D_U35_ARR;
__constant__ double cSinF[] = VEM_SIN_F_ARR;
__constant__ double cCosF[] = VEM_COS_F_ARR;
__constant__ double cTanF[] = VEM_TAN_F_ARR;
__constant__ double cExpF[] = VEM_EXP_F_ARR;
__constant__ double cExpFU35[] = VEM_EXP_F_U35_ARR;

__constant__ double cLog1pD[] = VEM_LOG1P_D_ARR;
__constant__ double cLog1pDU35[] = VEM_LOG1P_D_U35_ARR;
__constant__ double cExpjD[] = VEM_EXPJ_D_ARR;
__constant__ double cLog1pF[] = VEM_LOG1P_F_ARR;
__constant__ double cLog1pFU35[] = VEM_LOG1P_F_U35_ARR;

// sin | cos coefficient sets, 8-double aligned, staged behind the PH tables so
// a lane fetches its quadrant's set with LDS.128 instead of per-coefficient
// selects (2 distinct addresses per warp, conflict-free).
constexpr int kSinCosCoefN = 16;
__device__ const double gSinCosD[kSinCosCoefN] = {
    VEM_SIN_D_C0, VEM_SIN_D_C1, VEM_SIN_D_C2, VEM_SIN_D_C3, VEM_SIN_D_C4, VEM_SIN_D_C5, 0.0, 0.0,
    VEM_COS_D_C0, VEM_COS_D_C1, VEM_COS_D_C2, VEM_COS_D_C3, VEM_COS_D_C4, VEM_COS_D_C5, 0.0, 0.0};
__device__ const double gSinCosF[kSinCosCoefN] = {
    VEM_SIN_F_C0, VEM_SIN_F_C1, VEM_SIN_F_C2, VEM_SIN_F_C3, 0.0,          0.0, 0.0, 0.0,
    -0.5,         VEM_COS_F_C0, VEM_COS_F_C1, VEM_COS_F_C2, VEM_COS_F_C3, 0.0, 0.0, 0.0};

// u35 sin | cos sets (cos: 5 terms + a zero leading coefficient, so the same
// 6-step Horner gives the 5-term value exactly: fma(0, z, c4) == c4)
__device__ const double gSinCosD35[kSinCosCoefN] = {
    VEM_SIN_D_U35_C0, VEM_SIN_D_U35_C1, VEM_SIN_D_U35_C2, VEM_SIN_D_U35_C3, VEM_SIN_D_U35_C4, VEM_SIN_D_U35_C5,
    0.0, 0.0,
    VEM_COS_D_U35_C0, VEM_COS_D_U35_C1, VEM_COS_D_U35_C2, VEM_COS_D_U35_C3, VEM_COS_D_U35_C4, 0.0, 0.0, 0.0};
__constant__ double cAtanDU35[] = VEM_ATAN_D_U35_ARR;
__constant__ double cAsinD[] = VEM_ASIN_D_ARR;
__constant__ double cAsinDU35[] = VEM_ASIN_D_U35_ARR;

// Payne-Hanek tables (global copy; kernels stage them into shared memory).
__device__ const double gPhD[4 * VEM_PH_D_ENTRIES] = {VEM_PH_D_INIT};
// integer Payne-Hanek table (ph_int): [w0, w1, w2, 0] per exponent
__device__ const unsigned long long gPhDI[4 * VEM_PH_DI_ENTRIES] = {VEM_PH_DI_INIT};
constexpr int kPhDIStaged = 2 * VEM_PH_DI_ENTRIES;  // staged w1 | w2 arrays (doubles; even: 16-byte aligned tail)
__device__ __align__(16) const double gPhF[4 * VEM_PH_F_ENTRIES] = {VEM_PH_F_INIT};
// Staged layout of the binary32 Payne-Hanek table: every lane of a warp reads
// a different entry (the exponents are random), so a plain table costs ~11
// bank-conflict wavefronts per load.  The staged copy is replicated once per
// bank group with a one-group skew between copies -- {t0, t1} as 16-byte
// records in 8 copies (stride 105 records = 1 mod 8), t2 as doubles in 16
// copies (stride 113 = 1 mod 16) -- and lane L reads copy (L - entry) mod 8
// (mod 16), so its bank group is L mod 8 (mod 16): conflict-free, 4 + 2
// wavefronts, the minimum for 24 bytes per lane.
constexpr int kPhFStride01 = VEM_PH_F_ENTRIES + 1, kPhFStride2 = VEM_PH_F_ENTRIES + 9;
static_assert(kPhFStride01 % 8 == 1 && kPhFStride2 % 16 == 1, "skew of one bank group per copy");
constexpr int kPhFT2 = 2 * 8 * kPhFStride01;                 // offset of the t2 copies (doubles)
constexpr int kPhFDoubles = kPhFT2 + 16 * kPhFStride2;       // staged size in doubles
// log / exp tables (tools/genlogtables.py).  Global copy: structure of
// arrays (offsets in doubles below).  Staged shared-memory block: dense
// 16-byte pairs where a lookup needs two values (one LDS.128, no stride
// gaps that would idle half of the banks), dense doubles otherwise:
//   [kSlLogIH + 2 i] {invc, logc_hi}                 i < 256  (f64 log)
//   [kSlLogLo + i]   logc_lo                         i < 256
//   [kSlExp + 2 j]   {2^(j/128) hi, lo}              j < 128  (exp of pow_d)
constexpr int kLtInvc = 0, kLtHi = 256, kLtLo = 512, kLtExpHi = 768, kLtExpLo = 896, kLtfHi = 1024;
constexpr int kLogTabD = 1280;  // global SoA doubles (+ 256 binary32 invc)
constexpr int kSlLogIH = 0, kSlLogLo = 512, kSlExp = 768;
constexpr int kLogTabN = 1024;  // staged doubles (f64 log / pow kernels)
// Replicated staging for the f32 log kernels (layout 1): the lanes of a warp
// read random entries, so the plain 16-byte records cost ~7.5 bank-conflict
// wavefronts per load (the f32 log kernels were shared-memory bound: 70 % of
// the LSU's wavefronts at 0.78 of the HBM roofline).  8 copies of the
// {invc, logc hi} records, one bank group of skew between copies (stride 257
// records = 1 mod 8); lane L reads copy (L - entry) mod 8, so its bank group is
// L mod 8: conflict-free, 4 wavefronts.
constexpr int kRepLogFStride = 257;
constexpr int kRepLogFN = 2 * 8 * kRepLogFStride;  // staged doubles (then 128 doubles 2^(j/128) for pow_f)
__device__ const double gLogExp[kLogTabD] = {VEM_LOGT_INVC_INIT VEM_LOGT_HI_INIT VEM_LOGT_LO_INIT
                                                 VEM_EXPT_HI_INIT VEM_EXPT_LO_INIT VEM_LOGTF_HI_INIT};
__device__ const float gLogTfInvc[256] = {VEM_LOGTF_INVC_INIT};

// ---------------------------------------------------- primitives
// backend.hpp:47-52 round_ta == CUDA round() (ties away from zero) for every
// binary64 input incl. signed zeros; tests/test_gpu_parity.py pins it.
__device__ __forceinline__ double round_ta(double x) { return round(x); }
__device__ __forceinline__ double pow2_bits(int64_t e) { return from_bits_d((uint64_t)(e + 1023) << 52); }
// backend.hpp:133-138
__device__ __forceinline__ double ldexp2(double x, int64_t e) {
  e = e > 2046 ? 2046 : (e < -2044 ? -2044 : e);
  int64_t h = e >> 1;
  return (x * pow2_bits(h)) * pow2_bits(e - h);
}
__device__ __forceinline__ double mulsign(double x, double s) {  // backend.hpp:381-384
  return from_bits_d(bits_d(x) ^ (bits_d(s) & 0x8000000000000000ull));
}
__device__ __forceinline__ double copysign_b(double m, double s) {
  return from_bits_d((bits_d(m) & 0x7fffffffffffffffull) | (bits_d(s) & 0x8000000000000000ull));
}
__device__ __forceinline__ double neg_if(double y, int c) {
  return from_bits_d(bits_d(y) ^ ((uint64_t)(c != 0) << 63));
}
__device__ __forceinline__ double toward0_pos(double x) { return from_bits_d(bits_d(x) - 1); }
// nearest integer of a*b via one fma against 1.5*2^52 (oracle: rint_fma)
constexpr double kShift = 0x1.8p52;
__device__ __forceinline__ double rint_fma(double a, double b, int& k) {
  double u = fma(a, b, ccShift);
  k = __double2loint(u);
  return u - ccShift;
}

// ------------------------------------------------------ DD (ddarith.hpp)
__device__ __forceinline__ dd two_sum(double a, double b) {
  double s = a + b, v = s - a;
  return {s, (a - (s - v)) + (b - v)};
}
__device__ __forceinline__ dd two_sum_fast(double a, double b) {
  double s = a + b;
  return {s, b - (s - a)};
}
__device__ __forceinline__ dd two_prod(double a, double b) {
  double p = a * b;
  return {p, fma(a, b, -p)};
}
__device__ __forceinline__ dd dd_add2(dd x, dd y) {
  double s = x.hi + y.hi, v = s - x.hi;
  double e = (x.hi - (s - v)) + (y.hi - v);
  return {s, e + (x.lo + y.lo)};
}
__device__ __forceinline__ dd dd_add2_d(dd x, double y) {
  double s = x.hi + y, v = s - x.hi;
  double e = (x.hi - (s - v)) + (y - v);
  return {s, e + x.lo};
}
__device__ __forceinline__ dd dd_mul(dd x, dd y) {
  double p = x.hi * y.hi;
  double e = fma(x.hi, y.hi, -p);
  e = fma(x.hi, y.lo, e);
  e = fma(x.lo, y.hi, e);
  return {p, e};
}
__device__ __forceinline__ dd dd_mul_d(dd x, double y) {
  double p = x.hi * y;
  double e = fma(x.hi, y, -p);
  e = fma(x.lo, y, e);
  return {p, e};
}
__device__ __forceinline__ dd dd_squ(dd x) {
  double p = x.hi * x.hi;
  double e = fma(x.hi, x.hi, -p);
  e = fma(x.hi + x.hi, x.lo, e);
  return {p, e};
}
__device__ __forceinline__ dd dd_div(dd x, dd y) {
  double t = __drcp_rn(y.hi);  // == RN(1 / y.hi), without the division routine's slow path
  double q = x.hi * t;
  double u = fma(t, x.hi, -q);
  double v = fma(y.lo, -t, fma(y.hi, -t, 1.0));
  return {q, fma(q, v, fma(x.lo, t, u))};
}
__device__ __forceinline__ dd dd_normalize(dd x) { return two_sum_fast(x.hi, x.lo); }

// Horner, the oracle's order (oracle/vem_oracle.c: poly): n-1 DFMAs, each
// with its coefficient as a constant-bank operand.
template <int N>
__device__ __forceinline__ double poly(const double* c, double x) {
  double acc = c[N - 1];
#pragma unroll
  for (int i = N - 2; i >= 0; i--) acc = fma(acc, x, c[i]);
  return acc;
}
// Same with per-lane selected coefficients (a ? ca[i] : cb[i]).
template <int N>
__device__ __forceinline__ double poly_sel(const double* ca, const double* cb, bool a, double x) {
  double acc = a ? ca[N - 1] : cb[N - 1];
#pragma unroll
  for (int i = N - 2; i >= 0; i--) acc = fma(acc, x, a ? ca[i] : cb[i]);
  return acc;
}

// ===================================================== reduction (f64)
struct red { double hi, lo; int q; };

// reduction.hpp:148-159
__device__ __forceinline__ red cw1(double x) {
  double qd = round_ta(x * kTwoOverPi);
  double r0 = fma(qd, -kCw1P0, x);
  dd tail = two_prod(qd, -kCw1T1);
  tail.lo = fma(qd, -kCw1T2, tail.lo);
  // dd_add2({r0, 0}, tail) without the "+ 0.0": that add only turns a -0
  // tail.lo into +0, which changes no result bit of any caller (the residual
  // lo only enters sums with nonzero terms; tests pin CW1 bit for bit)
  double s = r0 + tail.hi, v = s - r0;
  double e = (r0 - (s - v)) + (tail.hi - v);
  dd r = dd_normalize(dd{s, e + tail.lo});
  return {r.hi, r.lo, (int)qd & 3};  // |qd| <= 10
}

// reduction.hpp:163-178
__device__ __forceinline__ red cw2(double x) {
  double t = x * kTwoOverPi;
  double qh = trunc(t * 0x1p-24);
  qh = qh * 0x1p24;
  double ql = round_ta(t - qh);
  double r = x;
  r = fma(qh, -kCw2A, r);
  r = fma(ql, -kCw2A, r);
  r = fma(qh, -kCw2B, r);
  r = fma(ql, -kCw2B, r);
  dd acc = dd_add2(dd{r, 0.0}, two_prod(qh, -kCw2C));
  acc = dd_add2(acc, two_prod(ql, -kCw2C));
  double qs = qh + ql;
  dd dtail = two_prod(qs, -kCw2D1);
  dtail.lo = fma(qs, -kCw2D2, dtail.lo);
  acc = dd_add2(acc, dtail);
  acc = dd_normalize(acc);
  return {acc.hi, acc.lo, (int)ql & 3};  // |ql| < 2^24
}

// reduction.hpp:35-43
__device__ __forceinline__ dd rfrac_q(dd a, long long& q) {
  double rh = round_ta(a.hi);
  a.hi = a.hi - rh;
  q += (long long)rh;
  double rl = round_ta(a.lo);
  a.lo = a.lo - rl;
  q += (long long)rl;
  return a;
}

// reduction.hpp:89-137, repaired (mod-4 table in `tab`, two_sum renorm).
__device__ __forceinline__ red ph(double x_in, const double* __restrict__ tab) {
  bool bad = !(fabs(x_in) <= kDblMax);
  double x = bad ? 0.0 : x_in;
  double a = fabs(x);
  long long er = (long long)((bits_d(a) >> 52) & 0x7ff);
  long long idx = er - 1023;
  idx = (0 > idx) ? 0 : idx;
  idx = (idx > 1023) ? 1023 : idx;
  double m = ldexp2(a, 52 - idx);
  const double2* f2 = reinterpret_cast<const double2*>(tab + (idx << 2));
  double2 fa = f2[0], fb = f2[1];
  long long q = 0;
  dd u = two_prod(m, fa.x);
  u = rfrac_q(u, q);
  u = two_sum(u.hi, u.lo);
  u = dd_add2(u, two_prod(m, fa.y));
  u = rfrac_q(u, q);
  u = two_sum(u.hi, u.lo);
  u = dd_add2(u, two_prod(m, fb.x));
  u = rfrac_q(u, q);
  u = two_sum(u.hi, u.lo);
  u = dd_add2(u, two_prod(m, fb.y));
  double qv = round_ta(u.hi + u.lo);
  u.hi = u.hi - qv;
  q += (long long)qv;
  double ql = round_ta(u.lo);
  u.lo = u.lo - ql;
  q += (long long)ql;
  u = dd_normalize(u);
  double p = u.hi * kPio2Qd0;  // reduction.hpp:57-69 mul_pio2_qd
  double e = fma(u.hi, kPio2Qd0, -p);
  e = fma(u.hi, kPio2Qd1, e);
  e = fma(u.lo, kPio2Qd0, e);
  e = fma(u.hi, kPio2Qd2, e);
  e = fma(u.lo, kPio2Qd1, e);
  e = fma(u.hi, kPio2Qd3, e);
  e = fma(u.lo, kPio2Qd2, e);
  double rh = mulsign(p, x), rl = mulsign(e, x);
  if (x < 0.0) q = 0 - q;
  red o;
  o.hi = bad ? from_bits_d(kCanonNanD) : rh;
  o.lo = bad ? from_bits_d(kCanonNanD) : rl;
  o.q = bad ? 0 : (int)(q & 3);
  return o;
}

// Integer Payne-Hanek for binary64, full 192-bit window (oracle: ph_int192;
// the slow level of ph_int below, out of line): 53 x 192-bit product mod 2^192 (IMAD.WIDE chains), the quadrant
// from its top two bits, and the centred fraction summed straight from the
// product's 32-bit words as an exact floating-point expansion (each word
// converts exactly; fast two-sums, no leading-zero shifts), then times pi/2
// in double-double with the sign of x folded into the constant.  The
// cascaded double-double form of reduction.hpp:89-137 takes ~90 FP64
// instructions per element; this takes ~30 and a few integer ones.
// Reads the full window (w0, w1, w2) from the global table gPhDI (rare path).
__device__ __noinline__ red ph_int192(double x) {
  const double* __restrict__ tab = reinterpret_cast<const double*>(gPhDI);
  const uint64_t b = bits_d(x), ab = b & 0x7fffffffffffffffull;
  const int ue = (int)(ab >> 52) - 1023;
  const bool small = ue < VEM_PH_DI_UEMIN;
  int idx = ue - VEM_PH_DI_UEMIN;
  idx = small ? 0 : (idx > VEM_PH_DI_ENTRIES - 1 ? VEM_PH_DI_ENTRIES - 1 : idx);
  const uint64_t M = (ab & 0x000fffffffffffffull) | 0x0010000000000000ull;
  const ulonglong2* wt = reinterpret_cast<const ulonglong2*>(tab) + 2 * idx;
  const ulonglong2 w01 = wt[0], w2p = wt[1];
  const uint64_t P0 = M * w01.x, h0 = __umul64hi(M, w01.x);
  const uint64_t l1 = M * w01.y, h1 = __umul64hi(M, w01.y);
  const uint64_t P1 = h0 + l1;
  const uint64_t P2 = M * w2p.x + h1 + (uint64_t)(P1 < l1);
  const uint32_t p5 = (uint32_t)(P2 >> 32), p4 = (uint32_t)P2;
  const uint32_t p3 = (uint32_t)(P1 >> 32), p2 = (uint32_t)P1, p1 = (uint32_t)(P0 >> 32);
  int q = (int)((p5 + 0x20000000u) >> 30);
  const uint32_t f5 = p5 & 0x3fffffffu;
  // centred fraction F = frac - [frac >= 1/2] as an exact expansion: every
  // partial sum is 0 or at least 2^-63 in magnitude (no binary64 is closer
  // than ~2^-61 to a multiple of pi/2), so each fast two-sum is exact
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
  // r = F (pi/2) sign(x), pi/2 = C0 + C1
  const int sx = (int)(uint32_t)(b >> 32) & (int)0x80000000u;
  const double c0 = __hiloint2double(__double2hiint(kPio2Qd0) ^ sx, __double2loint(kPio2Qd0));
  const double c1 = __hiloint2double(__double2hiint(kPio2Qd1) ^ sx, __double2loint(kPio2Qd1));
  const double p = fh * c0;
  double ee = fma(fh, c0, -p);
  ee = fma(fh, c1, ee);
  ee = fma(fl, c0, ee);
  if (b >> 63) q = -q;
  red o;
  // non-finite x: a meaningless r (the functions select the canonical NaN
  // from x itself, as the oracle's NaN r yields)
  o.hi = small ? x : p;
  o.lo = small ? 0.0 : ee;
  o.q = small ? 0 : (q & 3);
  return o;
}

// Two-level integer Payne-Hanek (oracle: ph_int, same operations in the same
// order).  Fast level: M * (top 128 bits of the window) mod 2^128 (one
// 64 x 64 -> 128 product and one low product), the quadrant from the top two
// bits, the top 85 fraction bits (the rest is below the dropped M*w0 term) as
// two exactly convertible chunks (53 bits centred in integer arithmetic, 32)
// summed with one Fast2Sum, times pi/2 in double-double.  Within 2^-62 relative whenever |F| >= 2^-11
// quadrants; below that (~2^-10 of random arguments) ph_int192 recomputes.
// `tab`: the staged copy of the window's top two words as two arrays, w1 at
// [0, ENTRIES) and w2 at [ENTRIES, 2 ENTRIES) (kPhDIStaged doubles).  The
// lanes of a warp read random entries: 8-byte words at an 8-byte stride spread
// over all 16 bank pairs (~5 wavefronts per load), where the 32-byte records
// of gPhDI use 4 of them (~11).
// kAbs: reduce |x| (positive constants, no quadrant negation: 6 instructions
// fewer); the caller folds the sign of x into its result -- every function
// here is exactly odd or even in (r, q), so the values are the same bit for
// bit as with the signed reduction (the oracle's).
template <bool kAbs = false>
__device__ __forceinline__ red ph_int(double x, const double* __restrict__ tab) {
  const uint64_t b = bits_d(x), ab = b & 0x7fffffffffffffffull;
  const int ue = (int)(ab >> 52) - 1023;
  // one unsigned clamp: |x| < 1/2 (negative index) and inf/NaN read the last
  // entry and leave through the rare path / the functions' NaN select
  uint32_t idx = (uint32_t)(ue - VEM_PH_DI_UEMIN);
  idx = idx > VEM_PH_DI_ENTRIES - 1 ? VEM_PH_DI_ENTRIES - 1 : idx;
  const uint64_t M = (ab & 0x000fffffffffffffull) | 0x0010000000000000ull;
  const uint64_t* wt = reinterpret_cast<const uint64_t*>(tab) + idx;
  const uint64_t w1 = wt[0], w2 = wt[VEM_PH_DI_ENTRIES];
  const uint64_t T0 = M * w1;
  const uint64_t T1 = M * w2 + __umul64hi(M, w1);
  const uint32_t t3 = (uint32_t)(T1 >> 32), t2 = (uint32_t)T1, t1 = (uint32_t)(T0 >> 32);
  int q = (int)((t3 + 0x20000000u) >> 30);
  // fraction bits below 2^-73 are noise (the dropped M*w0 term): two chunks,
  // c0 = f : t2[31..9] (f = the 30 fraction bits of t3; 53 bits) minus 2^53
  // when the fraction is >= 1/2 -- i.e. the 53-bit field read as two's
  // complement: its high word is t3 shifted left by 2 (the quadrant bits out)
  // and arithmetically right by 11 -- and c1 = t2[8..0] : t1[31..9] (32 bits,
  // weights down to 2^-85); units of 2^-53
  const int c0hi = (int)(t3 << 2) >> 11;
  const uint32_t c0lo = __funnelshift_l(t2, t3, 23);
  const double S0 = (double)(long long)(((uint64_t)(uint32_t)c0hi << 32) | c0lo);
  // c1 * 2^-32 without a conversion: 2^20 + c1 2^-32 is the double with high word
  // 0x41300000 and low word c1 (exact), minus 2^20 (exact)
  const double tb = __hiloint2double(0x41300000, (int)__funnelshift_l(t1, t2, 23)) - 0x1p20;
  const double fh = S0 + tb;  // |S0| is 0 or >= 1 > tb: Fast2Sum, exact pair
  const double fl = tb - (fh - S0);
  // rare: |F| < 2^-11 quadrants (finite x), or |x| < 1/2 (ph_int192 returns
  // (x, 0, 0)); non-finite x leaves a meaningless r (the functions select
  // the canonical NaN from x itself).  Tests on high words only.
  const uint32_t hab = (uint32_t)(ab >> 32);
  const bool fsmall = ((uint32_t)__double2hiint(fh) & 0x7fffffffu) < 0x42900000u;  // |fh| < 2^42
  // (a non-finite x with a small garbage fraction takes the rare path too: harmless)
  if (hab < 0x3fe00000u || fsmall) return ph_int192(kAbs ? from_bits_d(ab) : x);
  // r = F (pi/2) sign(x) with pi/2 * 2^-53 = C0 + C1 (units of 2^-53 above)
  constexpr double kC0 = kPio2Qd0 * 0x1p-53, kC1 = kPio2Qd1 * 0x1p-53;
  double c0 = kC0, c1 = kC1;
  if constexpr (!kAbs) {
    const int sx = (int)(uint32_t)(b >> 32) & (int)0x80000000u;
    c0 = __hiloint2double(__double2hiint(kC0) ^ sx, __double2loint(kC0));
    c1 = __hiloint2double(__double2hiint(kC1) ^ sx, __double2loint(kC1));
  }
  const double p = fh * c0;
  double ee = fma(fh, c0, -p);
  ee = fma(fh, c1, ee);
  ee = fma(fl, c0, ee);
  if constexpr (!kAbs) {
    if (b >> 63) q = -q;
  }
  red o;
  o.hi = p;
  o.lo = ee;
  o.q = q & 3;
  return o;
}

// |x| < 15 (inside the CW1 range |x| <= 15) from the high word alone
// (15 = 0x402E0000_00000000); |x| == 15 exactly is left to trig_class
__device__ __forceinline__ bool trig_is_cw1(double x) {
  return ((uint32_t)__double2hiint(x) & 0x7fffffffu) < 0x402E0000u;
}
// reduction path class of x: 0 = CW1 (|x| <= 15), 1 = CW2 (<= 1e14), 2 = PH
__device__ __forceinline__ int trig_class(double x) {
  const uint64_t ab = bits_d(x) & 0x7fffffffffffffffull;
  return ab <= 0x402e000000000000ull ? 0 : (ab <= 0x42d6bcc41e900000ull ? 1 : 2);
}

// reduction.hpp:189-206 (deterministic, per lane).  A lane takes only its own
// method; warps whose lanes agree (all warps after the class regrouping in
// the streaming kernel) therefore skip the heavier methods entirely.
__device__ __forceinline__ red trig_reduce(double x, const double* __restrict__ tab) {
  const int c = trig_class(x);
  red r;
  if (c == 0) {
    r = cw1(x);
  } else if (c == 1) {
    r = cw2(x);
  } else {
    r = ph(x, tab);
  }
  return r;
}

// the functions' selector (oracle: trig_reduce_fn): CW1 / CW2 as the
// reference, the integer Payne-Hanek above 1e14; `tab` = the staged window
// words (kPhDIStaged)
__device__ __forceinline__ red trig_reduce_fn(double x, const double* __restrict__ tab) {
  const int c = trig_class(x);
  red r;
  if (c == 0) {
    r = cw1(x);
  } else if (c == 1) {
    r = cw2(x);
  } else {
    r = ph_int(x, tab);
  }
  return r;
}

// ===================================================== f64 functions
// oracle: sincos_core_d (same values; selects hoisted to the inputs of the
// shared operations so the two forms cost one multiply, one final sum)
__device__ __forceinline__ double sincos_core_d(double rh, double rl, int cosform, const double* coef) {
  bool cf = cosform != 0;
  double z = rh * rh;
  const double2* cs = reinterpret_cast<const double2*>(coef + (cf ? 8 : 0));
  const double2 c01 = cs[0], c23 = cs[1], c45 = cs[2];
  double P = fma(fma(fma(fma(fma(c45.y, z, c45.x), z, c23.y), z, c23.x), z, c01.y), z, c01.x);
  double hz = 0.5 * z;
  double M = z * (cf ? z : rh);              // cos: z*z, sin: rh*z
  double Ts = fma(-hz, rl, rl);              // sin: rl - rl*z/2
  double zl = fma(rh, rh, -z);
  double Tc = -fma(0.5, zl, rh * rl);        // cos: -(zl/2 + rh*rl)
  double w = 1.0 - hz;
  double Bc = (1.0 - w) - hz;
  double A = cf ? w : rh, B = cf ? Bc : 0.0, T = cf ? Tc : Ts;
  return A + (B + fma(M, P, T));
}

__device__ __forceinline__ bool is_zero_bits(double x) { return (bits_d(x) << 1) == 0ull; }
__device__ __forceinline__ bool not_finite_bits(double x) {
  return ((uint32_t)__double2hiint(x) & 0x7fffffffu) >= 0x7ff00000u;
}

// Reduction mode: kSel = per-lane selector (reduction.hpp:189-206), kPh =
// Payne-Hanek for every lane (config 3), kCw1 = Cody-Waite level 1 only (the
// kernels use it for warps whose elements are all |x| <= 15, where the
// selector takes that path anyway: same values, no branches).
enum RedMode { kSel = 0, kPh = 1, kCw1 = 2 };
// `tab`: the staged integer Payne-Hanek window words (w1 | w2, kPhDIStaged)
template <int kMode>
__device__ __forceinline__ red reduce_mode(double x, const double* tab) {
  if constexpr (kMode == kPh) return ph_int<true>(x, tab);  // (r, q) of |x|: see odd_sign
  else if constexpr (kMode == kCw1) return cw1(x);
  else return trig_reduce_fn(x, tab);
}
// kPh reduces |x|: the odd functions (sin, tan) flip their result by the sign
// of x, cos needs nothing.  0 for the signed reductions.
template <int kMode>
__device__ __forceinline__ double odd_sign(double y, double x) {
  if constexpr (kMode == kPh)
    return __hiloint2double(__double2hiint(y) ^ (__double2hiint(x) & (int)0x80000000u), __double2loint(y));
  else
    return y;
}

// NaN can only come from a non-finite input: canonicalised by an integer test
// `tab`: Payne-Hanek table (shared or global); `coef`: the sin|cos block
template <int kMode>
__device__ __forceinline__ double sin_d_u10(double x, const double* tab, const double* coef) {
  red r = reduce_mode<kMode>(x, tab);
  double y = sincos_core_d(r.hi, r.lo, r.q & 1, coef);
  y = odd_sign<kMode>(neg_if(y, r.q & 2), x);
  // +-0 -> x; kPh: the reduction of |x| = 0 is (0, 0, 0), the core gives +0 and
  // odd_sign the sign of x: no select needed
  if constexpr (kMode != kPh) y = is_zero_bits(x) ? x : y;
  if constexpr (kMode == kCw1) return y;  // |x| <= 15: finite
  else return not_finite_bits(x) ? from_bits_d(kCanonNanD) : y;
}
template <int kMode>
__device__ __forceinline__ double cos_d_u10(double x, const double* tab, const double* coef) {
  red r = reduce_mode<kMode>(x, tab);
  double y = sincos_core_d(r.hi, r.lo, (r.q & 1) ^ 1, coef);
  y = neg_if(y, (r.q + 1) & 2);
  if constexpr (kMode == kCw1) return y;
  else return not_finite_bits(x) ? from_bits_d(kCanonNanD) : y;
}

__device__ __forceinline__ double tan_core_d(double rh, double rl, int odd) {
  double hh = rh * 0.5, hl = rl * 0.5;
  double z = hh * hh;
  double P = poly<VEM_TAN_D_N>(cTanD, z);
  double corr = fma(hh * z, P, fma(hl, z, hl));
  dd t = two_sum_fast(hh, corr);
  dd t2 = dd_squ(t);
  // |t2| <= tan^2(pi/8) < 1: the fast two-sum gives the same exact pair
  // as the oracle's two_sum, three adds fewer
  dd den = two_sum_fast(1.0, -t2.hi);
  den.lo = den.lo - t2.lo;
  dd num = {t.hi * 2.0, t.lo * 2.0};
  bool o = odd != 0;
  dd X = {o ? -den.hi : num.hi, o ? -den.lo : num.lo};
  dd Y = {o ? num.hi : den.hi, o ? num.lo : den.lo};
  dd q = dd_div(X, Y);
  return q.hi + q.lo;
}
template <int kMode>
__device__ __forceinline__ double tan_d_u10(double x, const double* tab) {
  red r = reduce_mode<kMode>(x, tab);
  double y = odd_sign<kMode>(tan_core_d(r.hi, r.lo, r.q & 1), x);
  y = (fabs(x) < 0x1p-27) ? x : y;
  // finite x never gives a NaN y: the oracle's canon_d(y) is this select
  return not_finite_bits(x) ? from_bits_d(kCanonNanD) : y;
}

__device__ __forceinline__ double atan_d_u10(double x) {
  double a = fabs(x);
  bool c1 = a > kTanPi8;
  bool c2 = a > kTan3Pi8;
  // ns/ds are used for a in (tan(pi/8), tan(3pi/8)]: there a -+ 1 is exact
  // or |a| < 1, and 1 is a multiple of ulp(a), so the fast two-sums with
  // the constant first give the oracle's exact two_sum pairs
  dd ns = two_sum_fast(-1.0, a), ds = two_sum_fast(1.0, a);
  dd nn, dn;
  nn.hi = c2 ? -1.0 : (c1 ? ns.hi : a);
  nn.lo = c2 ? 0.0 : (c1 ? ns.lo : 0.0);
  dn.hi = c2 ? fmin(a, 0x1p60) : (c1 ? ds.hi : 1.0);  // oracle: normal 1/|x|, same result
  dn.lo = c2 ? 0.0 : (c1 ? ds.lo : 0.0);
  dd b = dd_div(nn, dn);
  double z = b.hi * b.hi;
  double P = poly<VEM_ATAN_D_N>(cAtanD, z);
  double corr = fma(b.hi * z, P, fma(-b.lo, z, b.lo));
  double offh = c2 ? kPio2Qd0 : (c1 ? kPio4Hi : 0.0);
  double offl = c2 ? kPio2Qd1 : (c1 ? kPio4Lo : 0.0);
  // offh is 0 or >= pi/4 > tan(pi/8) >= |b|: fast two-sum, same exact pair
  dd s = two_sum_fast(offh, b.hi);
  double y = s.hi + (s.lo + (offl + corr));
  y = (a == kInf) ? kPio2Qd0 : y;
  y = copysign_b(y, x);
  return canon_d(y);
}

constexpr uint32_t kExpFastHi = 0x40862000u;  // |x| < 708

template <int N, bool kU10>
__device__ __forceinline__ double exp_poly_d(double xs, const double* c, int& k_out) {
  double kd = rint_fma(xs, ccInvLn2, k_out);
  double r1 = fma(kd, -ccExpL1, xs);
  double r = fma(kd, -ccExpL2, r1);
  double P = poly<N>(c, r);
  double y;
  if (kU10) {
    double rl = fma(-kd, ccExpL2, r1 - r);
    double s = 1.0 + r;
    double se = (1.0 - s) + r;
    y = s + (se + fma(r * r, P, rl));
  } else {
    y = 1.0 + fma(r * r, P, r);
  }
  return y;
}
// oracle: exp_core_d.  Fast path: exponent-field scaling (result normal).
template <int N, bool kU10>
__device__ __forceinline__ double exp_core_d(double x, const double* c) {
  uint32_t hx = (uint32_t)__double2hiint(x) & 0x7fffffffu;
  int k;
  if (hx < kExpFastHi) {
    double y = exp_poly_d<N, kU10>(x, c, k);
    return __hiloint2double(__double2hiint(y) + (k << 20), __double2loint(y));
  }
  if (x > kExpOvf) return kInf;
  if (x < kExpUnf) return 0.0;
  if (x != x) return from_bits_d(kCanonNanD);
  double y = exp_poly_d<N, kU10>(x, c, k);
  return ldexp2(y, (long long)k);
}
__device__ __forceinline__ double exp_d_u10(double x) { return exp_core_d<VEM_EXP_D_N, true>(x, cExpD); }
__device__ __forceinline__ double exp_d_u35(double x) { return exp_core_d<VEM_EXP_D_U35_N, false>(x, cExpDU35); }

// ---- table-driven log / exp (oracle: log_reduce, log1p_dd, ... ) -------
// `lt` points at the staged LOGT (4 doubles per entry) followed by EXPT.
struct logred { double rh, rl, E, logc_hi, logc_lo; };

// kAdj = false: Eadj is known to be 0 -> E = (double)k (same value; (double)k
// is never -0, so the dropped "+ 0.0" cannot change a bit).
template <bool kAdj = true>
__device__ __forceinline__ logred log_reduce(double a, double Eadj, const double* __restrict__ lt) {
  // bits(a) - bits(0.75): the constant's low word is 0, so everything is on
  // the high word (same k, idx and m as the oracle's 64-bit form); the table
  // offsets are formed in bytes (idx * 16, idx * 8) with one shift and one mask
  const uint32_t hix = (uint32_t)__double2hiint(a);
  const uint32_t t = hix - 0x3fe80000u;
  const int k = (int)t >> 20;
  const uint32_t off16 = (t >> 8) & 0xff0u;  // idx = bits 12..19 of t
  const double m = __hiloint2double((int)(hix - (t & 0xfff00000u)), __double2loint(a));
  const double2 ih =
      *reinterpret_cast<const double2*>(reinterpret_cast<const char*>(lt + kSlLogIH) + off16);  // {invc, hi}
  double invc = ih.x;
  double p = m * invc;
  logred o;
  o.rl = fma(m, invc, -p);
  o.rh = p - 1.0;
  o.E = kAdj ? (double)k + Eadj : (double)k;
  o.logc_hi = ih.y;
  o.logc_lo = *reinterpret_cast<const double*>(reinterpret_cast<const char*>(lt + kSlLogLo) + (off16 >> 1));
  return o;
}

template <int N>
__device__ __forceinline__ dd log1p_dd(double rh, double rl, const double* c) {
  const double z = rh * rh;
  const double Q = poly<N>(c, rh);
  const double p2 = -0.5 * z;  // -rh^2/2, its error -ez/2 (exact)
  const double ez = fma(rh, rh, -z);
  const double lo = fma(-0.5, ez, fma(rh * z, Q, fma(-rl, rh, rl)));
  dd S = two_sum_fast(rh, p2);
  S.lo = S.lo + lo;
  return S;
}

// E ln2_h42 and logc_hi lie on the 2^-42 grid below 2^10: their sum is exact
__device__ __forceinline__ dd eln2_logc(const logred& g) {
  const double eh = g.E * ccLn2H42;
  return dd{eh + g.logc_hi, fma(g.E, ccLn2T42, g.logc_lo)};
}

template <bool kU10, bool kAdj = true>
__device__ __forceinline__ double log_fast_d(double a, double Eadj, const double* lt) {
  logred g = log_reduce<kAdj>(a, Eadj, lt);
  dd H = eln2_logc(g);
  dd L;
  if (kU10) {
    // the 5-term set (2^-64.2): the 6-term one (2^-71.6) is for pow's double-double log
    L = log1p_dd<VEM_LOG1P_D_U35_N>(g.rh, g.rl, cLog1pDU35);
  } else {
    double z = g.rh * g.rh;
    double Q = poly<VEM_LOG1P_D_U35_N>(cLog1pDU35, g.rh);
    L.hi = g.rh;
    L.lo = fma(z, fma(g.rh, Q, -0.5), g.rl);
  }
  // H.hi is 0 or has an exponent >= L.hi's: |E ln2 + log c| >= 0.28 for
  // E != 0, and for E = 0 every nonzero table log c is >= 2.99x the largest
  // |r| of its subinterval (checked over all 256 entries).  The fast
  // two-sum then gives the same exact pair as the oracle's two_sum.
  dd T = two_sum_fast(H.hi, L.hi);
  return T.hi + (T.lo + (H.lo + L.lo));
}

template <bool kU10>
__device__ __forceinline__ double log_core_d(double x, const double* lt) {
  uint64_t ix = bits_d(x);
  if (ix - 0x0010000000000000ull < 0x7fe0000000000000ull) return log_fast_d<kU10>(x, 0.0, lt);
  if (x > 0.0 && x < 0x1p-1022) return log_fast_d<kU10>(x * 0x1p64, -64.0, lt);
  if (x == 0.0) return -kInf;
  if (x == kInf) return x;
  return from_bits_d(kCanonNanD);
}

template <int N, bool kAdj = true>
__device__ __forceinline__ dd log_dd(double a, double Eadj, const double* c, const double* lt) {
  logred g = log_reduce<kAdj>(a, Eadj, lt);
  dd H = eln2_logc(g);
  dd L = log1p_dd<N>(g.rh, g.rl, c);
  dd S = two_sum_fast(H.hi, L.hi);
  S.lo = S.lo + (H.lo + L.lo);
  return S;
}

// shared body of exp_dd (oracle: exp_dd): r = t - k ln2/128, 2^(i/128) table
__device__ __forceinline__ double exp_dd_core(double th, double tl, const double* __restrict__ lt, int& e) {
  int k;
  double kd = rint_fma(th, ccExpjInv, k);
  double r1 = fma(kd, -ccExpjL1, th);
  double r2 = fma(kd, -ccExpjL2, tl);
  // |r2| <~ 2^-26, |r| <= ln2/256: the sum's rounding error is < 2^-61.5 (0.003
  // ulp of the result): no two-sum (oracle: exp_dd, same operations)
  double r = r1 + r2;
  double z = r * r;
  double Q = poly<VEM_EXPJ_D_N>(cExpjD, r);
  double s2 = z * fma(r, Q, 0.5);
  const double2 T2 = reinterpret_cast<const double2*>(lt + kSlExp)[k & 127];
  double Th = T2.x, Tl = T2.y;
  double u = fma(Th, r, fma(Th, s2, Tl));
  e = k >> 7;
  return Th + u;
}
// |th| >= 708: saturation / gradual underflow (rare; kept out of line)
__device__ __noinline__ double exp_dd_slow(dd t, const double* lt) {
  bool ok = (t.hi >= -760.0) && (t.hi <= 720.0);
  double th = ok ? t.hi : 0.0, tl = ok ? t.lo : 0.0;
  int e;
  double R = exp_dd_core(th, tl, lt, e);
  double y = ldexp2(R, (long long)e);
  y = (t.hi > kExpOvf) ? kInf : y;
  y = (t.hi < kExpUnf) ? 0.0 : y;
  return y;
}
__device__ __forceinline__ double exp_dd(dd t, const double* __restrict__ lt) {
  uint32_t hx = (uint32_t)__double2hiint(t.hi) & 0x7fffffffu;
  if (hx >= kExpFastHi) return exp_dd_slow(t, lt);
  int e;
  double R = exp_dd_core(t.hi, t.lo, lt, e);
  return __hiloint2double(__double2hiint(R) + (e << 20), __double2loint(R));
}

__device__ __forceinline__ bool is_int_d(double y) { return (fabs(y) < kInf) && (trunc(y) == y); }
__device__ __forceinline__ bool is_odd_d(double y) {
  return is_int_d(y) && (fabs(y) < 0x1p53) && (trunc(y * 0.5) * 2.0 != y);
}

template <int NL>
__device__ __noinline__ double pow_slow_d(double x, double y, const double* cl, const double* lt) {
  double ax = fabs(x);
  bool fin = (ax > 0.0) && (ax < kInf) && (fabs(y) < kInf);
  double R = 1.0;
  if (fin) {
    bool sub = ax < 0x1p-1022;
    R = exp_dd(dd_mul_d(log_dd<NL>(sub ? ax * 0x1p64 : ax, sub ? -64.0 : 0.0, cl, lt), y), lt);
  }
  bool yint = is_int_d(y), yodd = is_odd_d(y);
  double res = (x < 0.0 && yodd) ? -R : R;
  res = (x < 0.0 && !yint && fabs(y) < kInf) ? from_bits_d(kCanonNanD) : res;
  if (x == 0.0) {
    if (y < 0.0) res = yodd ? copysign_b(kInf, x) : kInf;
    else res = yodd ? x : 0.0;
  }
  if (ax == kInf) {
    if (y < 0.0) res = (yodd && x < 0.0) ? -0.0 : 0.0;
    else res = (yodd && x < 0.0) ? -kInf : kInf;
  }
  if (fabs(y) == kInf) {
    if (ax == 1.0) res = 1.0;
    else res = ((ax < 1.0) == (y < 0.0)) ? kInf : 0.0;
  }
  if (x != x || y != y) res = from_bits_d(kCanonNanD);
  if (y == 0.0 || x == 1.0) res = 1.0;
  return res;
}

// oracle: pow_core_d (fast path without any special-value logic)
template <int NL>
__device__ __forceinline__ double pow_core_d(double x, double y, const double* cl, const double* lt) {
  uint32_t hx = (uint32_t)__double2hiint(x);
  uint32_t hy = (uint32_t)__double2hiint(y) & 0x7fffffffu, ly = (uint32_t)__double2loint(y);
  bool fx = ((hx & 0x7fffffffu) - 0x00100000u) < 0x7fe00000u;
  bool fy = (hy < 0x7ff00000u) && ((hy | ly) != 0u);
  if (fx && fy) {
    double ax = __hiloint2double((int)(hx & 0x7fffffffu), __double2loint(x));
    double R = exp_dd(dd_mul_d(log_dd<NL>(ax, 0.0, cl, lt), y), lt);
    if ((int)hx < 0) R = is_int_d(y) ? (is_odd_d(y) ? -R : R) : from_bits_d(kCanonNanD);
    return R;
  }
  return pow_slow_d<NL>(x, y, cl, lt);
}
__device__ __forceinline__ double pow_d_u10(double x, double y, const double* lt) {
  return pow_core_d<VEM_LOG1P_D_N>(x, y, cLog1pD, lt);
}
__device__ __forceinline__ double pow_d_u35(double x, double y, const double* lt) {
  return pow_core_d<VEM_LOG1P_D_U35_N>(x, y, cLog1pDU35, lt);
}

// fmod: normalised-mantissa FP long division (oracle: fmod_core).  The
// shipped kernels (vem_kernels.cu: k_queue / k_wqueue with FmodQ) triage on
// the operand bits and run fmod_pend_setup / fmod_stepn50 / fmod_pend_finish
// on sorted queue rows; fmod_core is the full per-element function (tails,
// unaligned pointers); the setup / step / finish split below also serves the
// tuning build's work-ring kernel.
__device__ __forceinline__ int ilogb_pos(double x) {
  uint64_t b = bits_d(x);
  int e = (int)(b >> 52);
  return e != 0 ? e - 1023 : (63 - __clzll((long long)b)) - 1074;
}
__device__ __forceinline__ double mant_1_2(double x, int e) {
  uint64_t b = bits_d(x);
  uint64_t m = (e >= -1022) ? (b & 0x000fffffffffffffull) : ((b << (-1022 - e)) & 0x000fffffffffffffull);
  return from_bits_d(m | 0x3ff0000000000000ull);
}
// One long-division step of up to 50 bits: V == r 2^s (mod md), exactly,
// with signed remainders: V = rs - rint(rs * rmd) md, rmd = RN(1/md), and no
// sign fix-up inside the loop (4 FP64 instructions; the round-1 unsigned
// form trunc(RZ(rs rmd + 1)) / fma / compare / add took 8).  With r = b md
// (|b| <= 1 after the first step) and an s-bit step, rs * rmd = (rs/md)(1 +
// e), |e| <= 2^-52 + 2^-106, so |rint(rs*rmd) - rs/md| <= 1/2 + |b| 2^(s-52)
// + tiny: s = 50 keeps |b| <= 1/2 + 1/4 + ... < 1, and the first step (mn /
// md < 2, s0 <= 50) gives |b| <= 1 + 2^-55, i.e. |V| <= md as V and md are
// multiples of 2^-52.  So |V| < 2 is a multiple of 2^-52, representable, and
// the FMA (exact product Q md) is exact at every step.  The final r in (-md,
// md) takes r + md when negative (exact), giving r 2^s mod md in [0, md):
// the exact remainder, equal to the oracle's (vem_oracle.c fmod_step:
// two_prod, 50-bit steps from the top) bit for bit although the steps differ.
// CPU model with a per-step exactness check: tests/cpp/fmod_signed_step.c.
__device__ __forceinline__ double fmod_stepn_rs(double rs, double md, double rmd) {
  return fma(-rint(rs * rmd), md, rs);
}
// 50-bit step on r; rmd50 = rmd 2^50 (exact) so r * rmd50 == rs * rmd and the
// two products are independent.
__device__ __forceinline__ double fmod_stepn50(double r, double md, double rmd50) {
  return fma(-rint(r * rmd50), md, r * 0x1p50);
}
// After setup: r == (mn * 2^s0) mod md (signed) with s0 = E - 50*E50 in [1, 50], and
// E = E50 full 50-bit steps still to go (the kernels' ring holds only
// elements with E > 0).
struct fmod_state {
  double r, md, rmd, x;
  int E, ed;
};
__device__ __forceinline__ double fmod_finish(const fmod_state& st);
// returns true when the element is finished already (result in `res`)
__device__ __forceinline__ bool fmod_setup(double x, double y, fmod_state& st, double& res) {
  double n = fabs(x), d = fabs(y);
  if (x != x || y != y || !(n < kInf) || d == 0.0) {
    res = from_bits_d(kCanonNanD);
    return true;
  }
  if (d == kInf || n < d) {
    res = x;
    return true;
  }
  int en = ilogb_pos(n), ed = ilogb_pos(d);
  double mn = mant_1_2(n, en), md = mant_1_2(d, ed);
  int E = en - ed;
  st.md = md;
  const double rmd = __drcp_rn(md);  // RN(1/md): signed steps (fmod_stepn_rs)
  st.rmd = rmd * 0x1p50;
  st.ed = ed;
  st.x = x;
  if (E == 0) {  // mn >= md: one exact subtraction finishes it
    st.r = mn - md;
    st.E = 0;
    res = copysign_b(ldexp2(st.r, ed), x);
    return true;
  }
  const int E50 = (E - 1) / 50;
  st.r = fmod_stepn_rs(mn * __hiloint2double((1023 + E - 50 * E50) << 20, 0), md, rmd);
  st.E = E50;
  if (E50 == 0) {
    res = fmod_finish(st);
    return true;
  }
  return false;
}
// signed r in (-md, md) -> [0, md), scaled, sign of x
__device__ __forceinline__ double fmod_finish(const fmod_state& st) {
  const double r = st.r < 0.0 ? st.r + st.md : st.r;
  return copysign_b(ldexp2(r, st.ed), st.x);
}
__device__ __forceinline__ double fmod_core(double x, double y) {
  fmod_state st;
  double res;
  if (fmod_setup(x, y, st, res)) return res;
  for (int i = 0; i < st.E; i++) st.r = fmod_stepn50(st.r, st.md, st.rmd);
  return fmod_finish(st);
}
__device__ __forceinline__ double fmod_d(double x, double y) { return fmod_core(x, y); }

// ===================================== f32 functions (binary64 internals)
struct redf { double r; int q; };

// NaN results (inf / NaN arguments: the reduction's inf - inf) -> canonical NaN
__device__ __forceinline__ float fin_f_nan(float o) { return o != o ? from_bits_f(kCanonNanF) : o; }

// oracle/vem_oracle.c ph_f: binary32 Payne-Hanek in three binary64 limbs.
// The table entry for the biased exponent (clamped below at 2^25, where no
// bits above the quadrant need dropping) holds (2^S 2/pi mod 4) / 2^S as t0
// (29 bits), t1 (29 bits), t2 (53 bits): xd*t0 is exact, n = rint(xd*t0 +
// xd*t1) by the 1.5*2^52 shift carries the quadrant in its low word (two's
// complement for x < 0), f0 = xd*t0 - n is exact and two FMAs add the lower
// limbs (the inner one exact in the cancellation case).  8 FP64 instructions, one
// conversion, no integer multiply, no sign / small-argument special cases
// (tiny x: r = x(1 + O(2^-52)); +-0 stays +-0; inf/NaN -> NaN).
__device__ __forceinline__ redf ph_f(float xf, const double* __restrict__ tab) {
  const uint32_t fe = (bits_f(xf) >> 23) & 0xffu;
  const uint32_t idx = (fe > VEM_PH_F_FE0 ? fe : VEM_PH_F_FE0) - VEM_PH_F_FE0;
  const uint32_t sk = threadIdx.x - idx;  // copy = (lane - entry) mod 8 / 16 (kPhFStride*: conflict-free)
  const double2 t01 = reinterpret_cast<const double2*>(tab)[(sk & 7u) * kPhFStride01 + idx];
  const double t2 = tab[kPhFT2 + (sk & 15u) * kPhFStride2 + idx];
  const double xd = (double)xf;
  const double p0 = xd * t01.x;
  const double n = fma(xd, t01.y, p0) + 0x1.8p52;  // rint of the two-limb product: |f| <= 1/2 + 2^-31
  const double f0 = p0 - (n - 0x1.8p52);
  const double f = fma(xd, t2, fma(xd, t01.y, f0));
  redf o;
  o.r = f * 0x1.921fb54442d18p+0;
  o.q = __double2loint(n) & 3;
  return o;
}

// oracle: sincos_core_f.  Both forms from constant-bank coefficients and a
// per-lane select of the result (cheaper than selecting five coefficients).
// sin as a product r (1 + z S(z)): -0 stays -0 without a select.
__device__ __forceinline__ double sincos_core_f(double r, int cosform, const double* tab) {
  (void)tab;
  const double z = r * r;
  const double Ps = fma(fma(fma(cSinF[3], z, cSinF[2]), z, cSinF[1]), z, cSinF[0]);
  const double Pc = fma(fma(fma(fma(cCosF[3], z, cCosF[2]), z, cCosF[1]), z, cCosF[0]), z, -0.5);
  const double ys = r * fma(z, Ps, 1.0);
  const double yc = fma(z, Pc, 1.0);
  return cosform != 0 ? yc : ys;
}

__device__ __forceinline__ float sin_f_u10(float x, const double* tab) {
  redf r = ph_f(x, tab);
  double y = sincos_core_f(r.r, r.q & 1, tab);
  y = neg_if(y, r.q & 2);
  return fin_f_nan((float)y);
}
__device__ __forceinline__ float cos_f_u10(float x, const double* tab) {
  redf r = ph_f(x, tab);
  double y = sincos_core_f(r.r, (r.q & 1) ^ 1, tab);
  y = neg_if(y, (r.q + 1) & 2);
  return fin_f_nan((float)y);
}
__device__ __forceinline__ float tan_f_u10(float x, const double* tab) {
  redf r = ph_f(x, tab);
  double z = r.r * r.r;
  double P = poly<VEM_TAN_F_N>(cTanF, z);
  double t = fma(r.r * z, P, r.r);
  // -cot, branch-free (the library reciprocals carry a slow-path branch per
  // element, which keeps the compiler from interleaving the elements' chains):
  // 1/|t| from a binary32 magic-constant seed (<= 0.051), three binary32 Newton
  // steps (FP32 pipe, <= 2^-23.9) and one binary64 step (<= 2^-47)
  const double ta = fabs(t);
  const float tf = (float)ta;
  float yf = from_bits_f(0x7EF311C7u - bits_f(tf));
#pragma unroll
  for (int i = 0; i < 3; i++) yf = fmaf(yf, fmaf(-tf, yf, 1.0f), yf);
  const double y0 = (double)yf;
  const double y1 = fma(y0, fma(-ta, y0, 1.0), y0);
  // odd quadrant: -1/t = -sign(t) y1
  const double yo = __hiloint2double(__double2hiint(y1) | (~__double2hiint(t) & (int)0x80000000u), __double2loint(y1));
  double y = (r.q & 1) ? yo : t;
  return fin_f_nan((float)y);
}

template <int N>
__device__ __forceinline__ float exp_core_f(float x, const double* c) {
  float xc = fminf(fmaxf(x, -150.0f), 130.0f);
  double xd = (double)xc;
  int k;
  double kd = rint_fma(xd, ccInvLn2, k);
  double r = fma(kd, -ccExpL1, xd);
  r = fma(kd, -ccExpL2, r);
  double P = poly<N>(c, r);
  double y = fma(r, P, 1.0);
  y = __hiloint2double(__double2hiint(y) + (k << 20), __double2loint(y));
  float o = (float)y;
  return canon_f((x != x) ? x : o);
}
__device__ __forceinline__ float exp_f_u10(float x) { return exp_core_f<VEM_EXP_F_N>(x, cExpF); }
__device__ __forceinline__ float exp_f_u35(float x) { return exp_core_f<VEM_EXP_F_U35_N>(x, cExpFU35); }

// {invc, logc hi} of entry idx from the replicated f32 staging (kRepLogF*,
// kTableLogF: what every f32 log / pow kernel stages)
__device__ __forceinline__ double2 ld_logf(const double* __restrict__ lt, int idx) {
  return reinterpret_cast<const double2*>(lt)[(int)((threadIdx.x - (uint32_t)idx) & 7u) * kRepLogFStride + idx];
}
template <int N>
__device__ __forceinline__ double log_f_internal(double a, const double* c, const double* __restrict__ lt) {
  uint64_t ix = bits_d(a);
  uint64_t tmp = ix - 0x3fe8000000000000ull;
  long long k = (long long)tmp >> 52;
  int idx = (int)((tmp >> 44) & 255u);
  double m = from_bits_d(ix - ((uint64_t)k << 52));
  const double2 ih = ld_logf(lt, idx);  // {invc, hi}
  double r = fma(m, ih.x, -1.0);  // == (double)invc_f32: exact product
  double Q = poly<N>(c, r);
  double L = fma(r * r, Q, r);
  return fma((double)(int)k, ccLn2Hi, ih.y + L);
}
// Same values from the binary32 bits (positive NORMAL x only): bits(0.75f) =
// 0x3f400000 and the 23-bit mantissa offset give the identical k, idx and m
// as the binary64 decomposition above (which shifts them left by 29 bits).
template <int N>
__device__ __forceinline__ double log_f_internal_f(float x, const double* c, const double* __restrict__ lt) {
  uint32_t ux = bits_f(x);
  uint32_t t = ux - 0x3f400000u;
  int k = (int)t >> 23;
  int idx = (int)((t >> 15) & 255u);
  double m = (double)from_bits_f(ux - ((uint32_t)k << 23));
  const double2 ih = ld_logf(lt, idx);
  double r = fma(m, ih.x, -1.0);
  double Q = poly<N>(c, r);
  double L = fma(r * r, Q, r);
  return fma((double)k, ccLn2Hi, ih.y + L);
}
__device__ __forceinline__ bool is_pos_normal_f(float x) { return bits_f(x) - 0x00800000u < 0x7f000000u; }

template <int N>
__device__ __forceinline__ float log_core_f(float x, const double* c, const double* lt) {
  uint32_t ux = bits_f(x);
  if (is_pos_normal_f(x)) return (float)log_f_internal_f<N>(x, c, lt);
  if (ux - 1u < 0x7f7fffffu) return (float)log_f_internal<N>((double)x, c, lt);
  if (x == 0.0f) return -kInfF;
  if (x == kInfF) return x;
  return from_bits_f(kCanonNanF);
}
__device__ __forceinline__ float log_f_u10(float x, const double* lt) { return log_core_f<VEM_LOG1P_F_N>(x, cLog1pF, lt); }
__device__ __forceinline__ float log_f_u35(float x, const double* lt) { return log_core_f<VEM_LOG1P_F_U35_N>(x, cLog1pFU35, lt); }

__device__ __forceinline__ bool is_int_f(float y) { return (fabsf(y) < kInfF) && (truncf(y) == y); }
__device__ __forceinline__ bool is_odd_f(float y) {
  return is_int_f(y) && (fabsf(y) < 0x1p24f) && (truncf(y * 0.5f) * 2.0f != y);
}
__device__ __forceinline__ double exp_f_internal(double t, const double* __restrict__ lt) {
  int k;
  double kd = rint_fma(t, ccExpjInv, k);
  double r = fma(kd, -ccExpjL1, t);
  r = fma(kd, -ccExpjL2, r);
  double p = fma(r * r, fma(r, ccSixth, 0.5), r);
  double T = lt[kRepLogFN + (k & 127)];  // f32 staging (kTableLogF): 2^(j/128) after the replicated log records
  double R = fma(T, p, T);
  return __hiloint2double(__double2hiint(R) + ((k >> 7) << 20), __double2loint(R));
}
template <int NL>
__device__ __noinline__ float pow_slow_f(float x, float y, const double* cl, const double* lt) {
  float ax = fabsf(x);
  bool fin = (ax > 0.0f) && (ax < kInfF) && (fabsf(y) < kInfF);
  float Rf = 1.0f;
  if (fin) {
    double t = (double)y * log_f_internal<NL>((double)ax, cl, lt);
    t = fmin(fmax(t, -200.0), 200.0);
    Rf = (float)exp_f_internal(t, lt);
  }
  bool yint = is_int_f(y), yodd = is_odd_f(y);
  float res = (x < 0.0f && yodd) ? -Rf : Rf;
  res = (x < 0.0f && !yint && fabsf(y) < kInfF) ? from_bits_f(kCanonNanF) : res;
  if (x == 0.0f) {
    if (y < 0.0f) res = yodd ? copysignf(kInfF, x) : kInfF;
    else res = yodd ? x : 0.0f;
  }
  if (ax == kInfF) {
    if (y < 0.0f) res = (yodd && x < 0.0f) ? -0.0f : 0.0f;
    else res = (yodd && x < 0.0f) ? -kInfF : kInfF;
  }
  if (fabsf(y) == kInfF) {
    if (ax == 1.0f) res = 1.0f;
    else res = ((ax < 1.0f) == (y < 0.0f)) ? kInfF : 0.0f;
  }
  if (x != x || y != y) res = from_bits_f(kCanonNanF);
  if (y == 0.0f || x == 1.0f) res = 1.0f;
  return res;
}
template <int NL>
__device__ __forceinline__ float pow_core_f(float x, float y, const double* cl, const double* lt) {
  uint32_t ux = bits_f(x), uy = bits_f(y);
  bool fx = (ux - 1u) < 0x7f7fffffu;
  bool fy = ((uy & 0x7fffffffu) - 1u) < 0x7f7fffffu;
  if (fx && fy) {
    double t = (double)y * (is_pos_normal_f(x) ? log_f_internal_f<NL>(x, cl, lt) : log_f_internal<NL>((double)x, cl, lt));
    if (((uint32_t)__double2hiint(t) & 0x7fffffffu) >= 0x40690000u) t = (t > 0.0) ? 200.0 : -200.0;
    return (float)exp_f_internal(t, lt);
  }
  return pow_slow_f<NL>(x, y, cl, lt);
}
__device__ __forceinline__ float pow_f_u10(float x, float y, const double* lt) {
  return pow_core_f<VEM_LOG1P_F_N>(x, y, cLog1pF, lt);
}
__device__ __forceinline__ float pow_f_u35(float x, float y, const double* lt) {
  return pow_core_f<VEM_LOG1P_F_U35_N>(x, y, cLog1pFU35, lt);
}
__device__ __forceinline__ float fmod_f(float x, float y) {
  double r = fmod_core((double)x, (double)y);
  return canon_f((float)r);
}
// fmodf without a work queue (the shipped vem_fmod_f): binary32 exponent
// gaps are <= 277, i.e. <= 5 signed 50-bit steps (fmod_stepn50), so every
// lane runs the same straight-line body plus a loop whose trip count varies
// by at most 5 across the warp; trivial pairs and specials are selected at
// the end.  |x| and |y| are exact normal binary64 values (subnormal floats
// included), the remainder r 2^ed is exact and a binary32 value, so the
// result equals fmod_f / glibc fmodf bit for bit.
__device__ __forceinline__ float fmod_f_flat(float x, float y) {
  const uint32_t bx = bits_f(x) & 0x7fffffffu, by = bits_f(y) & 0x7fffffffu;
  const bool pend = bx > by && bx < 0x7f800000u && by != 0u;  // |x| > |y| > 0, x finite (so y finite)
  const uint64_t nb = bits_d((double)from_bits_f(pend ? bx : 0x3f800000u));
  const uint64_t db = bits_d((double)from_bits_f(pend ? by : 0x3f800000u));
  const int en = (int)(nb >> 52), ed = (int)(db >> 52);
  const double mn = from_bits_d((nb & 0x000fffffffffffffull) | 0x3ff0000000000000ull);
  const double md = from_bits_d((db & 0x000fffffffffffffull) | 0x3ff0000000000000ull);
  const int E = en - ed;  // 0 when not pending
  const int steps = E == 0 ? 0 : (int)(((uint32_t)(E - 1) * 1311u) >> 16);
  const double rmd = __drcp_rn(md);
  const double rmd50 = rmd * 0x1p50;
  double r = fmod_stepn_rs(mn * __hiloint2double((1023 + E - 50 * steps) << 20, 0), md, rmd);
  // warp-uniform trip count (the largest of the active lanes' counts) with the
  // step predicated per lane: the same iterations as a per-lane loop, without
  // its divergence bookkeeping (BSSY / BSYNC / predicated branch: more
  // instructions per trip than the step's four)
  const int kmax = __reduce_max_sync(__activemask(), steps);
#pragma unroll 1
  for (int k = 0; k < kmax; k++) {
    if (k < steps) r = fmod_stepn50(r, md, rmd50);
  }
  r = r < 0.0 ? r + md : r;
  const float m = (float)(r * __hiloint2double(ed << 20, 0));  // r 2^(ed-1023), exact
  float res = pend ? m : (bx < by ? x : 0.0f);                 // |x| < |y| -> x; |x| == |y| -> 0
  res = from_bits_f((bits_f(res) & 0x7fffffffu) | (bits_f(x) & 0x80000000u));
  const bool nan = bx >= 0x7f800000u || by > 0x7f800000u || by == 0u;
  return nan ? from_bits_f(kCanonNanF) : res;
}
// Branch-free fmodf: the exponent gap E <= 277 is split into exactly six
// signed steps of s_i = floor((E + i) / 6) <= 47 bits (sum E, Hermite), so
// every element runs the same straight-line body and the kernel's elements
// interleave.  Each step: rs = r 2^s_i (exact), V = rs - rint(rs RN(1/md)) md
// with |rint(..) - rs/md| <= 1/2 + 2^-4 |r/md| (fmod_stepn_rs' bound for s <=
// 47), so every step is exact; same result as fmod_f bit for bit.
__device__ __forceinline__ float fmod_f_fixed(float x, float y) {
  const uint32_t bx = bits_f(x) & 0x7fffffffu, by = bits_f(y) & 0x7fffffffu;
  const bool pend = bx > by && bx < 0x7f800000u && by != 0u;
  const uint64_t nb = bits_d((double)from_bits_f(pend ? bx : 0x3f800000u));
  const uint64_t db = bits_d((double)from_bits_f(pend ? by : 0x3f800000u));
  const int en = (int)(nb >> 52), ed = (int)(db >> 52);
  double r = from_bits_d((nb & 0x000fffffffffffffull) | 0x3ff0000000000000ull);
  const double md = from_bits_d((db & 0x000fffffffffffffull) | 0x3ff0000000000000ull);
  const int E = en - ed;  // [0, 277]; 0 when not pending
  const double rmd = __drcp_rn(md);
#pragma unroll
  for (int i = 0; i < 6; i++) {
    const int s = (int)(((uint32_t)(E + i) * 10923u) >> 16);  // (E + i) / 6 for E + i <= 282
    r = fmod_stepn_rs(r * __hiloint2double((1023 + s) << 20, 0), md, rmd);
  }
  r = r < 0.0 ? r + md : r;
  const float m = (float)(r * __hiloint2double(ed << 20, 0));  // r 2^(ed-1023), exact
  float res = pend ? m : (bx < by ? x : 0.0f);
  res = from_bits_f((bits_f(res) & 0x7fffffffu) | (bits_f(x) & 0x80000000u));
  const bool nan = bx >= 0x7f800000u || by > 0x7f800000u || by == 0u;
  return nan ? from_bits_f(kCanonNanF) : res;
}

// ============================ SURVEY §8(f).1 additions (oracle: same names)
// fdim, u35 sin/cos/tan/atan, asin/acos, atan2; float32 through binary64.
constexpr double kPiHi = 0x1.921fb54442d18p+1, kPiLo = 0x1.1a62633145c07p-53;
constexpr double k3Pio4Hi = 0x1.2d97c7f3321d2p+1, k3Pio4Lo = 0x1.a79394c9e8a0ap-54;

__device__ __forceinline__ double fdim_d(double x, double y) {
  double r = (x > y) ? x - y : 0.0;
  return (x != x || y != y) ? from_bits_d(kCanonNanD) : r;
}
__device__ __forceinline__ float fdim_f(float x, float y) {
  float r = (x > y) ? x - y : 0.0f;
  return (x != x || y != y) ? from_bits_f(kCanonNanF) : r;
}

// oracle: sincos_core_d_u35 (per-lane coefficient set from the staged block)
__device__ __forceinline__ double sincos_core_d_u35(double r, int cosform, const double* coef) {
  const bool cf = cosform != 0;
  const double z = r * r;
  const double2* cs = reinterpret_cast<const double2*>(coef + (cf ? 8 : 0));
  const double2 c01 = cs[0], c23 = cs[1], c45 = cs[2];
  const double P = fma(fma(fma(fma(fma(c45.y, z, c45.x), z, c23.y), z, c23.x), z, c01.y), z, c01.x);
  const double A = cf ? z : r * z;
  const double B = cf ? fma(z, P, -0.5) : P;
  const double C = cf ? 1.0 : r;
  return fma(A, B, C);
}
template <int kMode>
__device__ __forceinline__ double sin_d_u35(double x, const double* tab, const double* coef) {
  red r = reduce_mode<kMode>(x, tab);
  double y = sincos_core_d_u35(r.hi, r.q & 1, coef);
  y = odd_sign<kMode>(neg_if(y, r.q & 2), x);
  if constexpr (kMode != kPh) y = is_zero_bits(x) ? x : y;  // (kPh: as sin_d_u10)
  if constexpr (kMode == kCw1) return y;
  else return not_finite_bits(x) ? from_bits_d(kCanonNanD) : y;
}
template <int kMode>
__device__ __forceinline__ double cos_d_u35(double x, const double* tab, const double* coef) {
  red r = reduce_mode<kMode>(x, tab);
  double y = sincos_core_d_u35(r.hi, (r.q & 1) ^ 1, coef);
  y = neg_if(y, (r.q + 1) & 2);
  if constexpr (kMode == kCw1) return y;
  else return not_finite_bits(x) ? from_bits_d(kCanonNanD) : y;
}
__device__ __forceinline__ double tan_core_d_u35(double rh, double rl, int odd) {
  const double h = rh * 0.5, hl = rl * 0.5;
  const double z = h * h;
  const double P = poly<VEM_TAN_D_N>(cTanD, z);
  const double t = h + fma(h * z, P, hl);
  const double num = t + t;
  const double den = fma(-t, t, 1.0);
  const bool o = odd != 0;
  return (o ? -den : num) / (o ? num : den);
}
template <int kMode>
__device__ __forceinline__ double tan_d_u35(double x, const double* tab) {
  red r = reduce_mode<kMode>(x, tab);
  double y = odd_sign<kMode>(tan_core_d_u35(r.hi, r.lo, r.q & 1), x);
  y = (fabs(x) < 0x1p-27) ? x : y;
  return not_finite_bits(x) ? from_bits_d(kCanonNanD) : y;
}
__device__ __forceinline__ double atan_d_u35(double x) {
  const double a = fabs(x);
  const bool c1 = a > kTanPi8;
  const bool c2 = a > kTan3Pi8;
  const double nn = c2 ? -1.0 : (c1 ? a - 1.0 : a);
  const double dn = c2 ? fmin(a, 0x1p60) : (c1 ? a + 1.0 : 1.0);
  const double b = nn / dn;
  const double z = b * b;
  const double P = poly<VEM_ATAN_D_U35_N>(cAtanDU35, z);
  const double off = c2 ? kPio2Qd0 : (c1 ? kPio4Hi : 0.0);
  double y = off + fma(b * z, P, b);
  y = copysign_b(y, x);
  return canon_d(y);
}

// asin / acos (oracle: asin_parts, vo_asin_d_u10, ...)
struct asin_parts { double a, z, s, sl, u; bool big; };
template <int N, bool kU10>
__device__ __forceinline__ asin_parts asin_split(double x, const double* c) {
  asin_parts o;
  o.a = fabs(x);
  o.big = o.a > 0.5;
  o.z = o.big ? (1.0 - o.a) * 0.5 : o.a * o.a;
  o.s = sqrt(o.z);
  const double t = o.big ? o.s : o.a;
  const double P = poly<N>(c, o.z);
  o.u = (t * o.z) * P;
  o.sl = 0.0;
  if (kU10) {
    const double e = fma(-o.s, o.s, o.z);
    o.sl = (o.z == 0.0) ? 0.0 : e / (o.s + o.s);
  }
  return o;
}
__device__ __forceinline__ double asin_d_u10(double x) {
  const asin_parts p = asin_split<VEM_ASIN_D_N, true>(x, cAsinD);
  const dd h = two_sum_fast(kPio2Qd0, -2.0 * p.s);  // 2s <= 1 < pi/2 where used: same exact pair
  const double yb = h.hi + (h.lo + (kPio2Qd1 - 2.0 * (p.sl + p.u)));
  double y = p.big ? yb : p.a + p.u;
  y = (p.a > 1.0) ? from_bits_d(kCanonNanD) : y;
  return canon_d(copysign_b(y, x));
}
__device__ __forceinline__ double asin_d_u35(double x) {
  const asin_parts p = asin_split<VEM_ASIN_D_U35_N, false>(x, cAsinDU35);
  const double yb = (kPio2Qd0 - 2.0 * p.s) + (kPio2Qd1 - 2.0 * p.u);
  double y = p.big ? yb : p.a + p.u;
  y = (p.a > 1.0) ? from_bits_d(kCanonNanD) : y;
  return canon_d(copysign_b(y, x));
}
__device__ __forceinline__ double acos_d_u10(double x) {
  const asin_parts p = asin_split<VEM_ASIN_D_N, true>(x, cAsinD);
  const double us = copysign_b(p.u, x);
  const dd hs = two_sum_fast(kPio2Qd0, -x);  // |x| <= 1 < pi/2 where used
  const double ys = hs.hi + (hs.lo + (kPio2Qd1 - us));
  const double yp = 2.0 * p.s + 2.0 * (p.sl + p.u);
  const dd hn = two_sum_fast(kPiHi, -2.0 * p.s);
  const double yn = hn.hi + (hn.lo + (kPiLo - 2.0 * (p.sl + p.u)));
  double y = p.big ? (x > 0.0 ? yp : yn) : ys;
  y = (p.a > 1.0) ? from_bits_d(kCanonNanD) : y;
  return canon_d(y);
}
__device__ __forceinline__ double acos_d_u35(double x) {
  const asin_parts p = asin_split<VEM_ASIN_D_U35_N, false>(x, cAsinDU35);
  const double us = copysign_b(p.u, x);
  const double ys = (kPio2Qd0 - x) + (kPio2Qd1 - us);
  const double yp = 2.0 * (p.s + p.u);
  const double yn = (kPiHi - 2.0 * p.s) + (kPiLo - 2.0 * p.u);
  double y = p.big ? (x > 0.0 ? yp : yn) : ys;
  y = (p.a > 1.0) ? from_bits_d(kCanonNanD) : y;
  return canon_d(y);
}

// atan2 (oracle: atan2_special, atan2_parts, vo_atan2_d_u10/u35)
__device__ __forceinline__ double atan2_special(double y, double x, double g) {
  const double ax = fabs(x), ay = fabs(y);
  double r = g;
  if (ax == kInf) r = (ay == kInf) ? (x > 0.0 ? kPio4Hi : k3Pio4Hi) : (x > 0.0 ? 0.0 : kPiHi);
  else if (ay == kInf) r = kPio2Qd0;
  if (x == 0.0) r = (y == 0.0) ? (((bits_d(x) >> 63) != 0) ? kPiHi : 0.0) : kPio2Qd0;
  else if (y == 0.0) r = (x > 0.0) ? 0.0 : kPiHi;
  r = copysign_b(r, y);
  return (x != x || y != y) ? from_bits_d(kCanonNanD) : r;
}
struct atan2_parts { double num, den, ch, cl; bool c1; int sig; };
__device__ __forceinline__ atan2_parts atan2_split(double y, double x) {
  atan2_parts o;
  const double ax = fabs(x), ay = fabs(y);
  const bool swap = ay > ax;
  const double num = swap ? ax : ay, den = swap ? ay : ax;
  const double sc = den >= 0x1p1000 ? 0x1p-100 : (den < 0x1p-900 ? 0x1p100 : 1.0);
  o.num = num * sc;
  o.den = den * sc;
  o.c1 = o.num > kTanPi8 * o.den;
  const bool neg = x < 0.0;
  int q = (neg ? 4 : 0) + (swap ? (neg ? -2 : 2) : 0);  // multiples of pi/4
  o.sig = (swap != neg) ? -1 : 1;
  q += o.c1 ? o.sig : 0;
  o.ch = q == 0 ? 0.0 : (q == 1 ? kPio4Hi : (q == 2 ? kPio2Qd0 : (q == 3 ? k3Pio4Hi : kPiHi)));
  o.cl = q == 0 ? 0.0 : (q == 1 ? kPio4Lo : (q == 2 ? kPio2Qd1 : (q == 3 ? k3Pio4Lo : kPiLo)));
  return o;
}
__device__ __forceinline__ double atan2_d_u10(double y, double x) {
  const atan2_parts p = atan2_split(y, x);
  // den >= num >= 0: fast two-sums (den first), same exact pairs
  const dd ns = two_sum_fast(-p.den, p.num), ds = two_sum_fast(p.den, p.num);
  const dd nn = p.c1 ? ns : dd{p.num, 0.0};
  const dd dn = p.c1 ? ds : dd{p.den, 0.0};
  const dd b = dd_div(nn, dn);
  const double z = b.hi * b.hi;
  const double P = poly<VEM_ATAN_D_N>(cAtanD, z);
  const double corr = fma(b.hi * z, P, fma(-b.lo, z, b.lo));
  const double sg = (double)p.sig;
  const dd s = two_sum_fast(p.ch, sg * b.hi);  // p.ch is 0 or >= pi/4 > |b|
  const double g = s.hi + (s.lo + (p.cl + sg * corr));
  return canon_d(atan2_special(y, x, copysign_b(g, y)));
}
__device__ __forceinline__ double atan2_d_u35(double y, double x) {
  const atan2_parts p = atan2_split(y, x);
  const double nn = p.c1 ? p.num - p.den : p.num;
  const double dn = p.c1 ? p.num + p.den : p.den;
  const double b = nn * __drcp_rn(dn);
  const double z = b * b;
  const double P = poly<VEM_ATAN_D_U35_N>(cAtanDU35, z);
  const double g = p.ch + (double)p.sig * fma(b * z, P, b);
  return canon_d(atan2_special(y, x, copysign_b(g, y)));
}

// ============================================ trivial classes (kernels)
// Closed-form results for arguments whose value the full function returns
// without computation -- saturated, special or tiny -- used by k_stream to
// keep such elements out of the computed rows (config 5: 50-97 % of the
// elements).  maybe() is a cheap superset test on the bits; exact() decides
// and gives the result, bit-identical to the full function's (oracle:
// vo_triv_*, tests/test_trivial_classes.py checks every rule against the
// oracle's full functions).
// exp: |x| < 2^-54 -> 1.0; x > ln(DBL_MAX) -> +inf; x < -745.13 -> +0; NaN.
__device__ __forceinline__ bool triv_exp_maybe(double x) {
  const uint32_t h = (uint32_t)__double2hiint(x) & 0x7fffffffu;
  return h >= 0x40862E42u || h < 0x3C900000u;
}
__device__ __forceinline__ bool triv_exp(double x, double& r) {
  const uint32_t h = (uint32_t)__double2hiint(x) & 0x7fffffffu;
  r = h < 0x3C900000u ? 1.0 : (x > kExpOvf ? kInf : (x < kExpUnf ? 0.0 : from_bits_d(kCanonNanD)));
  return h < 0x3C900000u || x > kExpOvf || x < kExpUnf || x != x;
}
// log: negative (incl. -inf, negative NaN bits) -> NaN, +-0 -> -inf, +inf, NaN
__device__ __forceinline__ bool triv_log_maybe(double x) {
  const uint64_t ix = bits_d(x);
  return ix - 0x0000000000000001ull >= 0x7fefffffffffffffull;  // not positive finite nonzero
}
__device__ __forceinline__ bool triv_log(double x, double& r) {
  const uint64_t ix = bits_d(x);
  r = (ix << 1) == 0ull ? -kInf : (ix == 0x7ff0000000000000ull ? kInf : from_bits_d(kCanonNanD));
  return ix - 0x0000000000000001ull >= 0x7fefffffffffffffull;
}
// pow (x, y finite and nonzero, x normal): x < 0 with y not an integer ->
// NaN; x > 0 with |y log x| certainly beyond the saturation thresholds ->
// +inf / +0.  log|x| lies in [e ln2, (e+1) ln2) for x = 2^e m, so
// |y log x| >= |y| m ln2 with m = e (e >= 0) or e + 1 (e < 0), its sign the
// sign of y m: y m > 1025 (710.5 > ln DBL_MAX) -> +inf, y m < -1077
// (-746.5 < -745.14) -> +0.  maybe(): x negative / special / subnormal or
// |e| > 34 (config 2's x in [1e-10, 1e10]: never).
__device__ __forceinline__ bool triv_pow_maybe(double x, double y) {
  (void)y;  // a hint only: large |y| with moderate x is left to the full path
  // x negative (sign bit: a huge unsigned word), special, or 2^e with
  // |e| > 34: one subtract and one compare on the high word
  return (uint32_t)__double2hiint(x) - 0x3DD00000u >= 0x04400000u;
}
__device__ __forceinline__ bool triv_pow(double x, double y, double& r) {
  const uint32_t hx = (uint32_t)__double2hiint(x);
  const uint32_t hy = (uint32_t)__double2hiint(y) & 0x7fffffffu, ly = (uint32_t)__double2loint(y);
  const bool fx = ((hx & 0x7fffffffu) - 0x00100000u) < 0x7fe00000u;  // normal, either sign
  const bool fy = (hy < 0x7ff00000u) && ((hy | ly) != 0u);
  const int e = (int)((hx >> 20) & 0x7ffu) - 1023;
  const double p = y * (double)(e >= 0 ? e : e + 1);
  const bool neg = (int)hx < 0;
  const bool nanr = neg && trunc(y) != y;
  r = nanr ? from_bits_d(kCanonNanD) : (p > 1025.0 ? kInf : 0.0);
  return fx && fy && (nanr || (!neg && (p > 1025.0 || p < -1077.0)));
}
// atan: |x| >= 2^54 (incl. inf) -> +-pi/2 (the double nearest); |x| < 2^-27
// -> x; NaN -> NaN
__device__ __forceinline__ bool triv_atan_maybe(double x) {
  const uint32_t h = (uint32_t)__double2hiint(x) & 0x7fffffffu;
  return h >= 0x43500000u || h < 0x3E400000u;
}
__device__ __forceinline__ bool triv_atan(double x, double& r) {
  const uint32_t h = (uint32_t)__double2hiint(x) & 0x7fffffffu;
  r = x != x ? from_bits_d(kCanonNanD) : (h < 0x3E400000u ? x : copysign_b(kPio2Qd0, x));
  return h >= 0x43500000u || h < 0x3E400000u;
}

// ============================================ split fast paths (kernels)
// Branch-free bodies for the common inputs, returning a nonzero `code` for
// elements they do not finish.  The streaming kernel evaluates a tile's
// elements with these (so the compiler interleaves the independent chains
// of one thread's elements), then passes the flagged ones to the op's
// `slow` hook (vem_kernels.cu), which selects saturated / special results
// inline and calls the full, out-of-line function only for genuinely rare
// inputs (subnormal operands or results, NaN operands of pow, ...).  For
// code 0 each returns exactly the full function's value.
template <int N, bool kU10>
__device__ __forceinline__ double exp_fast_d(double x, const double* c, int& code) {
  code = ((uint32_t)__double2hiint(x) & 0x7fffffffu) >= kExpFastHi ? 1 : 0;
  int k;
  double y = exp_poly_d<N, kU10>(x, c, k);
  return __hiloint2double(__double2hiint(y) + (k << 20), __double2loint(y));
}
// |x| >= 708: overflow / underflow / NaN selected, the gradual-underflow and
// near-overflow bands need the full function (`full` is called only then)
template <class F>
__device__ __forceinline__ double exp_slow_d(double x, F full) {
  if ((x >= kExpUnf) && (x <= kExpOvf)) return full();
  return (x != x) ? from_bits_d(kCanonNanD) : (x > 0.0 ? kInf : 0.0);
}
template <bool kU10>
__device__ __forceinline__ double log_fast_split_d(double x, const double* lt, int& code) {
  code = (bits_d(x) - 0x0010000000000000ull < 0x7fe0000000000000ull) ? 0 : 1;  // positive normal
  return log_fast_d<kU10, false>(x, 0.0, lt);
}
template <class F>
__device__ __forceinline__ double log_slow_d(double x, F full) {
  const uint64_t ix = bits_d(x);
  if (ix - 1ull < 0x000fffffffffffffull) return full();  // positive subnormal
  return (ix << 1) == 0ull ? -kInf : (ix == 0x7ff0000000000000ull ? kInf : from_bits_d(kCanonNanD));
}
// pow code: 0 for a positive normal x with |t| < 708 (t = y log x; y = +-0
// gives t = +-0 and the exact 1.0, inf / NaN y give |t| = inf / NaN and are
// flagged) -- two compares per element; otherwise bit 31 set and the high
// word of t (shifted right by one) below it, from which the slow hook
// rebuilds the classification (saturated / negative base / special operand).
template <int NL>
__device__ __forceinline__ double pow_fast_d(double x, double y, const double* cl, const double* lt, int& code) {
  const uint32_t hx = (uint32_t)__double2hiint(x);
  const double ax = __hiloint2double((int)(hx & 0x7fffffffu), __double2loint(x));
  const dd t = dd_mul_d(log_dd<NL, false>(ax, 0.0, cl, lt), y);
  int e;
  const double R = exp_dd_core(t.hi, t.lo, lt, e);
  const uint32_t th = (uint32_t)__double2hiint(t.hi);
  const bool ok = (hx - 0x00100000u < 0x7fe00000u) && ((th & 0x7fffffffu) < kExpFastHi);
  code = ok ? 0 : (int)((th >> 1) | 0x80000000u);
  return __hiloint2double(__double2hiint(R) + (e << 20), __double2loint(R));
}
// pow of a negative finite base (pow_core_d's rule on R = pow(|x|, y))
__device__ __forceinline__ double pow_neg_fix_d(double R, double y) {
  return is_int_d(y) ? (is_odd_d(y) ? -R : R) : from_bits_d(kCanonNanD);
}
// x in {+-0, +-Inf, NaN} with y finite and nonzero: pow_slow_d's C99 Annex F
// results, selected inline (these are most of the flagged specials; the
// out-of-line call costs the warp ~150 instructions per occurrence)
__device__ __forceinline__ double pow_special_x_d(double x, double y) {
  const bool yodd = is_odd_d(y);
  double res;
  if (x == 0.0) res = (y < 0.0) ? (yodd ? copysign_b(kInf, x) : kInf) : (yodd ? x : 0.0);
  else res = (y < 0.0) ? ((yodd && x < 0.0) ? -0.0 : 0.0) : ((yodd && x < 0.0) ? -kInf : kInf);
  return (x != x) ? from_bits_d(kCanonNanD) : res;
}
// The saturation tests use the high word of t without its last bit, with a
// margin: t in the margin goes to the full function, never to a wrong
// saturation (ln DBL_MAX = 0x40862E42FEFA39EF, -ln(2^-1075) = 0x40874910D52D3052).
template <class F>
__device__ __forceinline__ double pow_slow_split_d(double x, double y, double r, int code, F full) {
  const uint32_t hx = (uint32_t)__double2hiint(x);
  const uint32_t hy = (uint32_t)__double2hiint(y) & 0x7fffffffu, ly = (uint32_t)__double2loint(y);
  const bool fx = ((hx & 0x7fffffffu) - 0x00100000u) < 0x7fe00000u;  // normal, either sign
  const bool fy = (hy < 0x7ff00000u) && ((hy | ly) != 0u);
  if (!(fx && fy)) {
    // x in {+-0, +-Inf, NaN} with an ordinary y: inline; everything else
    // flagged here (subnormal x, special y) needs the full function
    const bool sx = (hx & 0x7fffffffu) >= 0x7ff00000u || is_zero_bits(x);
    if (fy && sx) return pow_special_x_d(x, y);
    return full();
  }
  const uint32_t t2 = (uint32_t)code & 0x3fffffffu;  // |t| high word >> 1
  const bool tneg = ((uint32_t)code & 0x40000000u) != 0u;
  if (t2 >= (kExpFastHi >> 1)) {
    const bool sat = tneg ? (t2 >= (0x40874912u >> 1)) : (t2 >= (0x40862E44u >> 1));
    if (!sat) return full();
    r = tneg ? 0.0 : kInf;
  }
  return ((int)hx < 0) ? pow_neg_fix_d(r, y) : r;
}
template <int N>
__device__ __forceinline__ float log_fast_f(float x, const double* c, const double* lt, int& code) {
  code = is_pos_normal_f(x) ? 0 : 1;
  return (float)log_f_internal_f<N>(x, c, lt);
}
template <int NL>
__device__ __forceinline__ float pow_fast_f(float x, float y, const double* cl, const double* lt, int& code) {
  const uint32_t uy = bits_f(y);
  const bool fy = ((uy & 0x7fffffffu) - 1u) < 0x7f7fffffu;
  const double t = (double)y * log_f_internal_f<NL>(x, cl, lt);
  // |t| >= 200 saturates: left to the full function (a flag instead of the
  // clamp's three selects; the table index below is masked, so a huge or NaN
  // t reads inside the table)
  const bool big = ((uint32_t)__double2hiint(t) & 0x7fffffffu) >= 0x40690000u;
  code = (is_pos_normal_f(x) && fy && !big) ? 0 : 1;
  return (float)exp_f_internal(t, lt);
}

}  // namespace vem
