// vem sm_100a kernels and the C-ABI entry points declared in include/vem.h.
//
// Layout in HBM: plain contiguous arrays of binary64 / binary32, caller-owned.
// Each CTA streams 16-byte vectors (double2 / float4) with cache-streaming
// loads/stores (ld.global.cs / st.global.cs: read-once data, evict-first),
// U independent vectors in flight per thread, over a persistent grid sized to
// (SM count x resident CTAs per SM).  Trig kernels first stage their
// Payne-Hanek table (32 KB f64 / 3 KB f32) into shared memory so the four
// per-lane gathers are shared-memory loads instead of divergent constant-bank
// reads (north star; reduction.hpp:101-104 `gather`).
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <cstring>

#include "../../include/vem.h"
#include "vem_math.cuh"

namespace vem {

static std::atomic<uint64_t> g_launches{0};

enum TableKind { kNoTable = 0, kTableD = 1, kTableF = 2 };

template <int TABLE>
struct TableSize {
  static constexpr int n = TABLE == kTableD ? 4 * VEM_PH_D_ENTRIES : (TABLE == kTableF ? 3 * VEM_PH_F_ENTRIES : 2);
};

template <int TABLE>
__device__ __forceinline__ const double* stage_table(double* stab) {
  if constexpr (TABLE == kNoTable) {
    return nullptr;
  } else {
    const double* src = TABLE == kTableD ? gPhD : gPhF;
    constexpr int n2 = TableSize<TABLE>::n / 2;
    const double2* s2 = reinterpret_cast<const double2*>(src);
    double2* d2 = reinterpret_cast<double2*>(stab);
    for (int i = threadIdx.x; i < n2; i += blockDim.x) d2[i] = __ldg(s2 + i);
    __syncthreads();
    return stab;
  }
}

template <class T> struct Vec16;
template <> struct Vec16<double> { using type = double2; static constexpr int n = 2; };
template <> struct Vec16<float> { using type = float4; static constexpr int n = 4; };

__device__ __forceinline__ double& vget(double2& v, int i) { return i == 0 ? v.x : v.y; }
__device__ __forceinline__ float& vget(float4& v, int i) { return i == 0 ? v.x : (i == 1 ? v.y : (i == 2 ? v.z : v.w)); }

constexpr int kThreads = 256;

// ------------------------------------------------------------ unary kernel
template <class Op, class T, int TABLE, int U, bool VEC>
__global__ void __launch_bounds__(kThreads) k_unary(const T* __restrict__ x, T* __restrict__ y, size_t n) {
  __shared__ __align__(16) double stab[TableSize<TABLE>::n];
  const double* tab = stage_table<TABLE>(stab);
  Op op;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  const size_t tid = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if constexpr (VEC) {
    using V = typename Vec16<T>::type;
    constexpr int W = Vec16<T>::n;
    const size_t nv = n / W;
    const V* xv = reinterpret_cast<const V*>(x);
    V* yv = reinterpret_cast<V*>(y);
    for (size_t i = tid; i < nv; i += stride * U) {
      V v[U];
#pragma unroll
      for (int u = 0; u < U; u++) {
        size_t j = i + u * stride;
        if (j < nv) v[u] = __ldcs(xv + j);
      }
#pragma unroll
      for (int u = 0; u < U; u++) {
        size_t j = i + u * stride;
        if (j < nv) {
          V o;
#pragma unroll
          for (int k = 0; k < W; k++) vget(o, k) = op(vget(v[u], k), tab);
          __stcs(yv + j, o);
        }
      }
    }
    const size_t done = nv * W;
    if (tid < n - done) y[done + tid] = op(x[done + tid], tab);
  } else {
    for (size_t i = tid; i < n; i += stride) y[i] = op(x[i], tab);
  }
}

// ----------------------------------------------------------- binary kernel
template <class Op, class T, int U, bool VEC>
__global__ void __launch_bounds__(kThreads) k_binary(const T* __restrict__ x, const T* __restrict__ y2,
                                                     T* __restrict__ out, size_t n) {
  Op op;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  const size_t tid = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if constexpr (VEC) {
    using V = typename Vec16<T>::type;
    constexpr int W = Vec16<T>::n;
    const size_t nv = n / W;
    const V* xv = reinterpret_cast<const V*>(x);
    const V* yv = reinterpret_cast<const V*>(y2);
    V* ov = reinterpret_cast<V*>(out);
    for (size_t i = tid; i < nv; i += stride * U) {
      V a[U], b[U];
#pragma unroll
      for (int u = 0; u < U; u++) {
        size_t j = i + u * stride;
        if (j < nv) {
          a[u] = __ldcs(xv + j);
          b[u] = __ldcs(yv + j);
        }
      }
#pragma unroll
      for (int u = 0; u < U; u++) {
        size_t j = i + u * stride;
        if (j < nv) {
          V o;
#pragma unroll
          for (int k = 0; k < W; k++) vget(o, k) = op(vget(a[u], k), vget(b[u], k));
          __stcs(ov + j, o);
        }
      }
    }
    const size_t done = nv * W;
    if (tid < n - done) out[done + tid] = op(x[done + tid], y2[done + tid]);
  } else {
    for (size_t i = tid; i < n; i += stride) out[i] = op(x[i], y2[i]);
  }
}

// ------------------------------------------------------------- functors
#define VEM_UNARY_OP(NAME, T, EXPR)                                                   \
  struct NAME {                                                                       \
    __device__ __forceinline__ T operator()(T x, const double* tab) const { return EXPR; } \
  };
VEM_UNARY_OP(OpSinD, double, (sin_d_u10<false>(x, tab)))
VEM_UNARY_OP(OpCosD, double, (cos_d_u10<false>(x, tab)))
VEM_UNARY_OP(OpTanD, double, (tan_d_u10<false>(x, tab)))
VEM_UNARY_OP(OpSinDPh, double, (sin_d_u10<true>(x, tab)))
VEM_UNARY_OP(OpCosDPh, double, (cos_d_u10<true>(x, tab)))
VEM_UNARY_OP(OpTanDPh, double, (tan_d_u10<true>(x, tab)))
VEM_UNARY_OP(OpAtanD, double, ((void)tab, atan_d_u10(x)))
VEM_UNARY_OP(OpExpD, double, ((void)tab, exp_d_u10(x)))
VEM_UNARY_OP(OpExpDU35, double, ((void)tab, exp_d_u35(x)))
VEM_UNARY_OP(OpLogD, double, ((void)tab, log_core_d<true>(x)))
VEM_UNARY_OP(OpLogDU35, double, ((void)tab, log_core_d<false>(x)))
VEM_UNARY_OP(OpSinF, float, (sin_f_u10(x, tab)))
VEM_UNARY_OP(OpCosF, float, (cos_f_u10(x, tab)))
VEM_UNARY_OP(OpTanF, float, (tan_f_u10(x, tab)))
VEM_UNARY_OP(OpExpF, float, ((void)tab, exp_f_u10(x)))
VEM_UNARY_OP(OpExpFU35, float, ((void)tab, exp_f_u35(x)))
VEM_UNARY_OP(OpLogF, float, ((void)tab, log_f_u10(x)))
VEM_UNARY_OP(OpLogFU35, float, ((void)tab, log_f_u35(x)))
#undef VEM_UNARY_OP

#define VEM_BINARY_OP(NAME, T, EXPR)                                              \
  struct NAME {                                                                   \
    __device__ __forceinline__ T operator()(T x, T y) const { return EXPR; }      \
  };
VEM_BINARY_OP(OpPowD, double, pow_d_u10(x, y))
VEM_BINARY_OP(OpPowDU35, double, pow_d_u35(x, y))
VEM_BINARY_OP(OpFmodD, double, fmod_d(x, y))
VEM_BINARY_OP(OpPowF, float, pow_f_u10(x, y))
VEM_BINARY_OP(OpPowFU35, float, pow_f_u35(x, y))
VEM_BINARY_OP(OpFmodF, float, fmod_f(x, y))
#undef VEM_BINARY_OP

// ------------------------------------------------------------- launching
static int num_sms() {
  static int sms = [] {
    int dev = 0, v = 148;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v;
  }();
  return sms;
}

template <class K>
static int occupancy(K kernel) {
  int b = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kernel, kThreads, 0) != cudaSuccess || b < 1) b = 1;
  return b;
}

// Persistent grid: min(work, SMs x resident CTAs per SM); `occ` is cached by
// the caller per kernel instantiation.
static int grid_for(int occ, size_t work_items, int per_thread) {
  size_t need = (work_items + (size_t)kThreads * per_thread - 1) / ((size_t)kThreads * per_thread);
  size_t cap = (size_t)num_sms() * occ;
  size_t g = need < cap ? need : cap;
  return (int)(g < 1 ? 1 : g);
}

static inline bool aligned16(const void* p) { return ((uintptr_t)p & 15u) == 0; }

template <class Op, class T, int TABLE, int U>
static int launch_unary(const T* x, T* y, size_t n, vem_stream_t s) {
  if (n == 0) return 0;
  cudaStream_t st = (cudaStream_t)s;
  if (aligned16(x) && aligned16(y)) {
    auto k = k_unary<Op, T, TABLE, U, true>;
    static const int occ = occupancy(k);
    int g = grid_for(occ, n / Vec16<T>::n + 1, U);
    k<<<g, kThreads, 0, st>>>(x, y, n);
  } else {
    auto k = k_unary<Op, T, TABLE, 1, false>;
    static const int occ = occupancy(k);
    int g = grid_for(occ, n, 1);
    k<<<g, kThreads, 0, st>>>(x, y, n);
  }
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return (int)cudaGetLastError();
}

template <class Op, class T, int U>
static int launch_binary(const T* x, const T* y2, T* out, size_t n, vem_stream_t s) {
  if (n == 0) return 0;
  cudaStream_t st = (cudaStream_t)s;
  if (aligned16(x) && aligned16(y2) && aligned16(out)) {
    auto k = k_binary<Op, T, U, true>;
    static const int occ = occupancy(k);
    int g = grid_for(occ, n / Vec16<T>::n + 1, U);
    k<<<g, kThreads, 0, st>>>(x, y2, out, n);
  } else {
    auto k = k_binary<Op, T, 1, false>;
    static const int occ = occupancy(k);
    int g = grid_for(occ, n, 1);
    k<<<g, kThreads, 0, st>>>(x, y2, out, n);
  }
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return (int)cudaGetLastError();
}

// ---------------------------------------------------- reduction kernels
template <int MODE>  // 0 trig_reduce, 1 cw1, 2 cw2, 3 ph
__global__ void __launch_bounds__(kThreads) k_reduce_d(const double* __restrict__ x, double* hi, double* lo,
                                                       int* q, size_t n) {
  __shared__ __align__(16) double stab[TableSize<kTableD>::n];
  const double* tab = stage_table<kTableD>(stab);
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    double v = x[i];
    red r;
    if (MODE == 0) r = trig_reduce(v, tab);
    else if (MODE == 1) r = cw1(v);
    else if (MODE == 2) r = cw2(v);
    else r = ph(v, tab);
    hi[i] = r.hi;
    lo[i] = r.lo;
    q[i] = r.q;
  }
}

__global__ void __launch_bounds__(kThreads) k_reduce_f(const float* __restrict__ x, double* rr, int* q, size_t n) {
  __shared__ __align__(16) double stab[TableSize<kTableF>::n];
  const double* tab = stage_table<kTableF>(stab);
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    redf r = ph_f(x[i], tab);
    rr[i] = r.r;
    q[i] = r.q;
  }
}

template <int MODE>
static int launch_reduce_d(const double* x, double* hi, double* lo, int* q, size_t n, vem_stream_t s) {
  if (n == 0) return 0;
  auto k = k_reduce_d<MODE>;
  static const int occ = occupancy(k);
  int g = grid_for(occ, n, 1);
  k<<<g, kThreads, 0, (cudaStream_t)s>>>(x, hi, lo, q, n);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return (int)cudaGetLastError();
}

static const double kHostPhD[4 * VEM_PH_D_ENTRIES] = {VEM_PH_D_INIT};

}  // namespace vem

using namespace vem;

// Elements per thread in flight (16-byte vectors): HBM-bound kernels keep 4
// vectors in flight, FP64-pipe-bound ones 2 (register pressure).
extern "C" {

int vem_sin_d_u10(const double* x, double* y, size_t n, vem_stream_t s) { return launch_unary<OpSinD, double, kTableD, 2>(x, y, n, s); }
int vem_cos_d_u10(const double* x, double* y, size_t n, vem_stream_t s) { return launch_unary<OpCosD, double, kTableD, 2>(x, y, n, s); }
int vem_tan_d_u10(const double* x, double* y, size_t n, vem_stream_t s) { return launch_unary<OpTanD, double, kTableD, 2>(x, y, n, s); }
int vem_sin_d_u10_ph(const double* x, double* y, size_t n, vem_stream_t s) { return launch_unary<OpSinDPh, double, kTableD, 1>(x, y, n, s); }
int vem_cos_d_u10_ph(const double* x, double* y, size_t n, vem_stream_t s) { return launch_unary<OpCosDPh, double, kTableD, 1>(x, y, n, s); }
int vem_tan_d_u10_ph(const double* x, double* y, size_t n, vem_stream_t s) { return launch_unary<OpTanDPh, double, kTableD, 1>(x, y, n, s); }
int vem_atan_d_u10(const double* x, double* y, size_t n, vem_stream_t s) { return launch_unary<OpAtanD, double, kNoTable, 2>(x, y, n, s); }
int vem_exp_d_u10(const double* x, double* y, size_t n, vem_stream_t s) { return launch_unary<OpExpD, double, kNoTable, 4>(x, y, n, s); }
int vem_exp_d_u35(const double* x, double* y, size_t n, vem_stream_t s) { return launch_unary<OpExpDU35, double, kNoTable, 4>(x, y, n, s); }
int vem_log_d_u10(const double* x, double* y, size_t n, vem_stream_t s) { return launch_unary<OpLogD, double, kNoTable, 2>(x, y, n, s); }
int vem_log_d_u35(const double* x, double* y, size_t n, vem_stream_t s) { return launch_unary<OpLogDU35, double, kNoTable, 2>(x, y, n, s); }
int vem_pow_d_u10(const double* x, const double* y2, double* o, size_t n, vem_stream_t s) { return launch_binary<OpPowD, double, 1>(x, y2, o, n, s); }
int vem_pow_d_u35(const double* x, const double* y2, double* o, size_t n, vem_stream_t s) { return launch_binary<OpPowDU35, double, 1>(x, y2, o, n, s); }
int vem_fmod_d(const double* x, const double* y2, double* o, size_t n, vem_stream_t s) { return launch_binary<OpFmodD, double, 1>(x, y2, o, n, s); }

int vem_sin_f_u10(const float* x, float* y, size_t n, vem_stream_t s) { return launch_unary<OpSinF, float, kTableF, 1>(x, y, n, s); }
int vem_cos_f_u10(const float* x, float* y, size_t n, vem_stream_t s) { return launch_unary<OpCosF, float, kTableF, 1>(x, y, n, s); }
int vem_tan_f_u10(const float* x, float* y, size_t n, vem_stream_t s) { return launch_unary<OpTanF, float, kTableF, 1>(x, y, n, s); }
// every f32 trig lane takes the f32 Payne-Hanek path: the forced variants are the same kernels
int vem_sin_f_u10_ph(const float* x, float* y, size_t n, vem_stream_t s) { return vem_sin_f_u10(x, y, n, s); }
int vem_cos_f_u10_ph(const float* x, float* y, size_t n, vem_stream_t s) { return vem_cos_f_u10(x, y, n, s); }
int vem_tan_f_u10_ph(const float* x, float* y, size_t n, vem_stream_t s) { return vem_tan_f_u10(x, y, n, s); }
int vem_exp_f_u10(const float* x, float* y, size_t n, vem_stream_t s) { return launch_unary<OpExpF, float, kNoTable, 2>(x, y, n, s); }
int vem_exp_f_u35(const float* x, float* y, size_t n, vem_stream_t s) { return launch_unary<OpExpFU35, float, kNoTable, 2>(x, y, n, s); }
int vem_log_f_u10(const float* x, float* y, size_t n, vem_stream_t s) { return launch_unary<OpLogF, float, kNoTable, 2>(x, y, n, s); }
int vem_log_f_u35(const float* x, float* y, size_t n, vem_stream_t s) { return launch_unary<OpLogFU35, float, kNoTable, 2>(x, y, n, s); }
int vem_pow_f_u10(const float* x, const float* y2, float* o, size_t n, vem_stream_t s) { return launch_binary<OpPowF, float, 1>(x, y2, o, n, s); }
int vem_pow_f_u35(const float* x, const float* y2, float* o, size_t n, vem_stream_t s) { return launch_binary<OpPowFU35, float, 1>(x, y2, o, n, s); }
int vem_fmod_f(const float* x, const float* y2, float* o, size_t n, vem_stream_t s) { return launch_binary<OpFmodF, float, 1>(x, y2, o, n, s); }

int vem_trig_reduce_d(const double* x, double* hi, double* lo, int* q, size_t n, vem_stream_t s) {
  return launch_reduce_d<0>(x, hi, lo, q, n, s);
}
int vem_cw_reduce_d(const double* x, double* hi, double* lo, int* q, size_t n, int level, vem_stream_t s) {
  return level == 1 ? launch_reduce_d<1>(x, hi, lo, q, n, s) : launch_reduce_d<2>(x, hi, lo, q, n, s);
}
int vem_ph_reduce_d(const double* x, double* hi, double* lo, int* q, size_t n, vem_stream_t s) {
  return launch_reduce_d<3>(x, hi, lo, q, n, s);
}
int vem_ph_reduce_f(const float* x, double* r, int* q, size_t n, vem_stream_t s) {
  if (n == 0) return 0;
  static const int occ = occupancy(k_reduce_f);
  int g = grid_for(occ, n, 1);
  k_reduce_f<<<g, kThreads, 0, (cudaStream_t)s>>>(x, r, q, n);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return (int)cudaGetLastError();
}

int vem_ph_table_d(unsigned char* out) {
  std::memcpy(out, kHostPhD, sizeof(kHostPhD));
  return 0;
}
uint64_t vem_launch_count(void) { return g_launches.load(); }
const char* vem_version(void) { return "vem-b200 0.1 (sm_100a)"; }

}  // extern "C"
