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
#include <type_traits>

#include "../../include/vem.h"
#include "vem_math.cuh"
#include "vem_stream.cuh"

namespace vem {

static std::atomic<uint64_t> g_launches{0};

// Checked build (-DVEM_CHECK, build.py --check -> libvem_check.so): device-side
// bounds assertions on every computed shared-memory index of the sorting
// kernels (k_trig, k_queue) and on the queue / list counts; a violation traps
// (the launch fails with cudaErrorLaunchFailure / illegal instruction).  This
// stands in for compute-sanitizer, which is closed on the GPU pool; the
// guard-band tests (tests/test_gpu_guard.py) cover the global side.
#ifdef VEM_CHECK
#define VEM_ASSERT(c) \
  do {                \
    if (!(c)) __trap(); \
  } while (0)
#else
#define VEM_ASSERT(c) ((void)0)
#endif

// kTableDG / kTableDG35 (selector kernels): sin|cos coefficients, then the
// integer Payne-Hanek window words w1 | w2 (kPhDIStaged doubles, 16.4 KB).
// k_trig stages the window lazily -- the first warp of a CTA that meets a
// Payne-Hanek element copies it (stage_ph_lazy) -- so inputs that never leave
// the Cody-Waite range (config 1) pay nothing.
// kTableD: the reference-algorithm PH table (reduction entry points);
// kTableDI: the integer PH window words w1 | w2 (forced-PH kernels) + sin|cos
// coefficients
enum TableKind { kNoTable = 0, kTableD = 1, kTableF = 2, kTableLog = 3, kTableDG = 4, kTableDG35 = 5, kTableDI = 6,
                 kTableLogF = 7 };  // kTableLogF: the f32 log records, replicated per bank group (vem_math.cuh kRepLogF*)

template <int TABLE>
struct TableSize {
  static constexpr int n = TABLE == kTableD   ? 4 * VEM_PH_D_ENTRIES + kSinCosCoefN
                           : TABLE == kTableDI ? kPhDIStaged + kSinCosCoefN
                           : TABLE == kTableF ? kPhFDoubles + kSinCosCoefN
                           : TABLE == kTableLog ? kLogTabN
                           : TABLE == kTableLogF ? kRepLogFN + 128
                           : (TABLE == kTableDG || TABLE == kTableDG35) ? kSinCosCoefN + kPhDIStaged
                                                : 2;
};

// w1 | w2 of the integer Payne-Hanek window, gPhDI records -> two arrays
__device__ __forceinline__ void copy_ph_window(double* dst, int first, int step) {
  unsigned long long* d = reinterpret_cast<unsigned long long*>(dst);
  for (int i = first; i < VEM_PH_DI_ENTRIES; i += step) {
    d[i] = __ldg(gPhDI + 4 * i + 1);
    d[VEM_PH_DI_ENTRIES + i] = __ldg(gPhDI + 4 * i + 2);
  }
}
// Lazy staging for k_trig, called by a converged warp that is about to run
// Payne-Hanek elements.  `ready` is a CTA-shared flag (0 at kernel start).
// Warps that find it clear copy the window themselves (concurrent copies
// write identical values) and set it after a CTA-scope fence; a warp that
// finds it set fences and reads.
__device__ __forceinline__ void stage_ph_lazy(double* dst, volatile int* ready) {
  const int lane = threadIdx.x & 31;
  const int r = __shfl_sync(0xffffffffu, *ready, 0);
  if (r == 0) {
    copy_ph_window(dst, lane, 32);
    __threadfence_block();
    __syncwarp();
    if (lane == 0) *ready = 1;
  } else {
    __threadfence_block();
  }
}

template <int TABLE, bool LAZY_PH = false>
__device__ __forceinline__ const double* stage_table(double* stab) {
  if constexpr (TABLE == kNoTable) {
    return nullptr;
  } else if constexpr (TABLE == kTableDG || TABLE == kTableDG35) {
    if (threadIdx.x < kSinCosCoefN) stab[threadIdx.x] = (TABLE == kTableDG ? gSinCosD : gSinCosD35)[threadIdx.x];
    if constexpr (!LAZY_PH) copy_ph_window(stab + kSinCosCoefN, threadIdx.x, blockDim.x);
    __syncthreads();
    return stab;
  } else {
    if constexpr (TABLE == kTableLog) {  // SoA global -> record layout (vem_math.cuh)
      for (int i = threadIdx.x; i < 256; i += blockDim.x) {
        reinterpret_cast<double2*>(stab + kSlLogIH)[i] = make_double2(gLogExp[kLtInvc + i], gLogExp[kLtHi + i]);
        stab[kSlLogLo + i] = gLogExp[kLtLo + i];
        if (i < 128)
          reinterpret_cast<double2*>(stab + kSlExp)[i] = make_double2(gLogExp[kLtExpHi + i], gLogExp[kLtExpLo + i]);
      }
    } else if constexpr (TABLE == kTableLogF) {
      for (int i = threadIdx.x; i < 8 * 256; i += blockDim.x) {
        const int c = i >> 8, k = i & 255;
        reinterpret_cast<double2*>(stab)[c * kRepLogFStride + k] =
            make_double2((double)__ldg(gLogTfInvc + k), gLogExp[kLtfHi + k]);
      }
      if (threadIdx.x < 128) stab[kRepLogFN + threadIdx.x] = gLogExp[kLtExpHi + threadIdx.x];
    } else if constexpr (TABLE == kTableF) {  // replicated, skewed copies (vem_math.cuh kPhFStride*)
      for (int i = threadIdx.x; i < 16 * VEM_PH_F_ENTRIES; i += blockDim.x) {
        const int c = i / VEM_PH_F_ENTRIES, k = i - c * VEM_PH_F_ENTRIES;
        if (c < 8)
          reinterpret_cast<double2*>(stab)[c * kPhFStride01 + k] = make_double2(gPhF[4 * k], gPhF[4 * k + 1]);
        stab[kPhFT2 + c * kPhFStride2 + k] = gPhF[4 * k + 2];
      }
    } else if constexpr (TABLE == kTableDI) {
      copy_ph_window(stab, threadIdx.x, blockDim.x);
    } else {
      const double* src = gPhD;
      constexpr int n2 = (TableSize<TABLE>::n - kSinCosCoefN) / 2;
      const double2* s2 = reinterpret_cast<const double2*>(src);
      double2* d2 = reinterpret_cast<double2*>(stab);
      for (int i = threadIdx.x; i < n2; i += blockDim.x) d2[i] = __ldg(s2 + i);
    }
    if constexpr (TABLE == kTableD || TABLE == kTableDI || TABLE == kTableF) {  // per-lane sin|cos coefficients
      const double* cs = TABLE == kTableF ? gSinCosF : gSinCosD;
      if (threadIdx.x < kSinCosCoefN) stab[TableSize<TABLE>::n - kSinCosCoefN + threadIdx.x] = cs[threadIdx.x];
    }
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
template <class Op, class T, int TABLE, int U, bool VEC>
__global__ void __launch_bounds__(kThreads) k_binary(const T* __restrict__ x, const T* __restrict__ y2,
                                                     T* __restrict__ out, size_t n) {
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
          for (int k = 0; k < W; k++) vget(o, k) = op(vget(a[u], k), vget(b[u], k), tab);
          __stcs(ov + j, o);
        }
      }
    }
    const size_t done = nv * W;
    if (tid < n - done) out[done + tid] = op(x[done + tid], y2[done + tid], tab);
  } else {
    for (size_t i = tid; i < n; i += stride) out[i] = op(x[i], y2[i], tab);
  }
}

// Ops with a split fast path (vem_math.cuh "split fast paths"): the kernel
// evaluates a tile's elements with Op::fast (branch-free, interleavable)
// and passes the elements it flags to Op::slow.
template <class Op> struct HasFast { static constexpr bool value = false; };
// Ops with trivial-result classes (closed-form results for saturated /
// special / tiny arguments: exp, log, pow, atan; vem_math.cuh "trivial
// classes").  Triv<Op>::maybe is a cheap bit test (false for every argument
// of the configs where nothing saturates, e.g. config 2); Triv<Op>::exact decides
// exactly and gives the result, equal bit for bit to the full function's.
// k_stream compacts the non-trivial elements of a warp into rows when at
// least a quarter of its lanes' first elements may be trivial (config 5:
// 50-97 % of the elements are).
template <class Op> struct Triv { static constexpr bool value = false; };
template <class Op> struct HasTriv { static constexpr bool value = Triv<Op>::value; };
// the full function for rare elements: one out-of-line copy per Op
template <class Op, class T>
__device__ __noinline__ T full_op(T x, const double* tab) { return Op()(x, tab); }
template <class Op, class T>
__device__ __noinline__ T full_op(T x, T y, const double* tab) { return Op()(x, y, tab); }

// one element through the op's fast path and, if flagged, its slow hook (or
// the plain op for ops without a split fast path)
template <class Op, int NIN, class T>
__device__ __forceinline__ T eval_one(const Op& op, T x, T y, const double* tab) {
  if constexpr (HasFast<Op>::value) {
    int code;
    T r;
    if constexpr (NIN == 2) r = op.fast(x, y, tab, code);
    else r = op.fast(x, tab, code);
    if (code) {
      if constexpr (NIN == 2) r = Op::slow(x, y, r, code, tab);
      else r = Op::slow(x, r, code, tab);
    }
    return r;
  } else {
    (void)y;
    if constexpr (NIN == 2) return op(x, y, tab);
    else return op(x, tab);
  }
}

// ------------------------------------------------- TMA-staged streaming
// NIN inputs (1 or 2); tiles of kThreads*VPT 16-byte vectors per input;
// STAGES tiles in flight per CTA (see vem_stream.cuh).  Elements past the
// last full tile are finished by a grid-stride scalar loop in the same launch.
// WREL: release stages per warp (tma::stage_release_last: warps drift, no
// CTA barrier per tile -- for kernels whose warps finish tiles at different
// times, e.g. pow with its slow paths) or with one CTA barrier after which
// thread 0 refills at once (the shortest refill latency, for HBM-bound
// kernels whose bytes in flight are the limit).
template <class Op, class T, int NIN, int TABLE, int VPT, int STAGES, int MINB = 1, bool WREL = false>
__global__ void __launch_bounds__(kThreads, MINB) k_stream(const T* __restrict__ a, const T* __restrict__ b,
                                                           T* __restrict__ out, size_t n) {
  using V = typename Vec16<T>::type;
  constexpr int W = Vec16<T>::n;
  constexpr int TILE_V = kThreads * VPT;
  constexpr uint32_t TILE_BYTES = TILE_V * 16;
  constexpr int TILE_E = TILE_V * W;
  constexpr int NE = VPT * W;  // elements per lane per tile
  constexpr int NW = kThreads / 32;
  extern __shared__ __align__(128) unsigned char dsm[];
  __shared__ uint64_t bars[STAGES];
  __shared__ uint32_t rel[STAGES];
  __shared__ __align__(16) double stab[TableSize<TABLE>::n];
  // trivial-class compaction (HasTriv ops only): per warp a stack of pending
  // non-trivial elements (argument(s) + global element index), carried from
  // tile to tile so that they are evaluated in full rows of 32
  constexpr int kQGrp = NE < 4 ? NE : 4;  // elements per lane pushed between two drains
  constexpr int kQCap = HasTriv<Op>::value ? 32 * kQGrp + 32 : 1;
  __shared__ __align__(16) T s_qx[HasTriv<Op>::value ? NW : 1][kQCap];
  __shared__ __align__(16) T s_qy[HasTriv<Op>::value && NIN == 2 ? NW : 1][kQCap];
  __shared__ uint32_t s_qi[HasTriv<Op>::value ? NW : 1][kQCap];  // (CTA-local tile number) * TILE_E + offset in the tile
  V* buf = reinterpret_cast<V*>(dsm);
  const int tid = threadIdx.x, lane = tid & 31;
  if (tid == 0) {
#pragma unroll
    for (int s = 0; s < STAGES; s++) tma::mbar_init(&bars[s], 1);
    tma::fence_barrier_init();
  }
  if (tid < STAGES) rel[tid] = 0;
  const double* tab = stage_table<TABLE>(stab);  // includes __syncthreads()
  if constexpr (TABLE == kNoTable) __syncthreads();
  tma::griddep_wait();  // inputs / outputs may belong to the previous grid
  tma::griddep_launch_dependents();
  Op op;
  const size_t ntiles = n / TILE_E;
  const size_t G = gridDim.x;
  const size_t my = ntiles > blockIdx.x ? (ntiles - blockIdx.x + G - 1) / G : 0;
  const uint64_t pol = tma::policy_evict_first();
  bool tmode = false;  // HasTriv: this warp compacts trivial elements (decided on its first tile)
  int qn = 0;          // HasTriv: entries on this warp's stack of pending non-trivial elements
  // stack entry -> global element index (entries hold the CTA-local tile number in 32 bits)
  auto qelem = [&](uint32_t q) -> size_t {
    return (blockIdx.x + (size_t)(q / (uint32_t)TILE_E) * G) * (size_t)TILE_E + (q % (uint32_t)TILE_E);
  };
  (void)qelem;
  (void)tmode;
  (void)qn;
  auto issue = [&](int s, size_t tile) {
    tma::mbar_expect_tx(&bars[s], NIN * TILE_BYTES);
    tma::bulk_g2s(buf + (size_t)(s * NIN) * TILE_V, reinterpret_cast<const V*>(a) + tile * TILE_V, TILE_BYTES,
                  &bars[s], pol);
    if constexpr (NIN == 2)
      tma::bulk_g2s(buf + (size_t)(s * NIN + 1) * TILE_V, reinterpret_cast<const V*>(b) + tile * TILE_V,
                    TILE_BYTES, &bars[s], pol);
  };
  if (tid == 0)
    for (int s = 0; s < STAGES && (size_t)s < my; s++) issue(s, blockIdx.x + (size_t)s * G);
  for (size_t j = 0; j < my; j++) {
    const int s = (int)(j % STAGES);
    tma::mbar_wait(&bars[s], (uint32_t)((j / STAGES) & 1));
    V va[VPT], vb[VPT];
#pragma unroll
    for (int v = 0; v < VPT; v++) {
      va[v] = buf[(size_t)(s * NIN) * TILE_V + v * kThreads + tid];
      if constexpr (NIN == 2) vb[v] = buf[(size_t)(s * NIN + 1) * TILE_V + v * kThreads + tid];
    }
    if constexpr (WREL) {  // per-warp stage release (vem_stream.cuh)
      __syncwarp();
      if (lane == 0 && tma::stage_release_last(&rel[s], NW) && j + STAGES < my) {
        tma::fence_proxy_async_smem();
        issue(s, blockIdx.x + (j + STAGES) * G);
      }
    } else {  // stage s fully consumed by the CTA -> refill it
      __syncthreads();
      if (tid == 0 && j + STAGES < my) {
        tma::fence_proxy_async_smem();
        issue(s, blockIdx.x + (j + STAGES) * G);
      }
    }
    V* ov = reinterpret_cast<V*>(out) + (blockIdx.x + j * G) * TILE_V;
    if constexpr (HasTriv<Op>::value) {
      // ---- warps with many trivial elements.  The decision samples each
      // lane's first element (one cheap test per lane and tile, so the dense
      // path below pays ~1 instruction per element).  The mode is decided per
      // warp on its first tile (input arrays are rarely heterogeneous at this
      // scale) so that the dense path carries no per-tile test; in compaction
      // mode every tile re-checks (at least a quarter of the samples).
      // Trivial results are stored at once; the other elements are pushed on
      // the warp's stack and evaluated 32 at a time -- full rows, whatever the
      // tile's share of them (config 5: 4-8 %, i.e. 5-10 per warp and tile:
      // evaluated per tile, the rows ran 5-10 active lanes of 32) -- each
      // result stored to its own element.
      bool m0;
      if constexpr (NIN == 2) m0 = Triv<Op>::maybe(vget(va[0], 0), vget(vb[0], 0));
      else m0 = Triv<Op>::maybe(vget(va[0], 0));
      if (j == 0) tmode = __popc(__ballot_sync(0xffffffffu, m0)) >= 8 && my * (size_t)TILE_E < ((size_t)1 << 32);
      if (tmode && __popc(__ballot_sync(0xffffffffu, m0)) >= 8) {
        T* qx = s_qx[tid >> 5];
        T* qy = NIN == 2 ? s_qy[(tid >> 5) % (NIN == 2 ? NW : 1)] : qx;  // unary: y unused
        uint32_t* qi = s_qi[tid >> 5];
        const uint32_t qbase = (uint32_t)j * (uint32_t)TILE_E;
        uint32_t mn = 0;  // non-trivial
#pragma unroll
        for (int v = 0; v < VPT; v++) {
          V o = va[v];  // a non-trivial element's placeholder: its own argument
#pragma unroll
          for (int k = 0; k < W; k++) {
            bool t;
            if constexpr (NIN == 2) t = Triv<Op>::exact(vget(va[v], k), vget(vb[v], k), vget(o, k));
            else t = Triv<Op>::exact(vget(va[v], k), vget(o, k));
            mn |= (uint32_t)!t << (v * W + k);
          }
          // one coalesced 16-byte store per vector; a non-trivial element's
          // part is a placeholder that the same warp overwrites when it pops the
          // element (the __syncwarp()s between the push and the pop order the
          // two stores; separate narrow stores of the trivial parts measured
          // 15 % slower: partially written sectors)
          __stcs(ov + v * kThreads + tid, o);
        }
#pragma unroll
        for (int g = 0; g < NE; g += kQGrp) {  // push kQGrp elements per lane, then drain full rows
          const uint32_t mg = (mn >> g) & ((1u << kQGrp) - 1u);
          const int cnt = __popc(mg);
          int inc = cnt;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const int t = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += t;
          }
          int p = qn + inc - cnt;
          qn += __shfl_sync(0xffffffffu, inc, 31);
          VEM_ASSERT(qn <= kQCap);
#pragma unroll
          for (int e = g; e < g + kQGrp; e++)
            if ((mn >> e) & 1u) {
              qx[p] = vget(va[e / W], e % W);
              if constexpr (NIN == 2) qy[p] = vget(vb[e / W], e % W);
              qi[p] = qbase + (uint32_t)(((e / W) * kThreads + tid) * W + (e % W));
              p++;
            }
          __syncwarp();
          while (qn >= 32) {  // full rows off the top of the stack; two at a time (independent chains)
            if (qn >= 64) {
              const int ia = qn - 32 + lane, ib = qn - 64 + lane;
              const T ya = eval_one<Op, NIN>(op, qx[ia], qy[ia], tab);
              const T yb = eval_one<Op, NIN>(op, qx[ib], qy[ib], tab);
              __stcs(out + qelem(qi[ia]), ya);
              __stcs(out + qelem(qi[ib]), yb);
              qn -= 64;
            } else {
              const int ia = qn - 32 + lane;
              __stcs(out + qelem(qi[ia]), eval_one<Op, NIN>(op, qx[ia], qy[ia], tab));
              qn -= 32;
            }
          }
          __syncwarp();  // the popped entries are overwritten by the next pushes
        }
        continue;
      }
    }
    if constexpr (HasFast<Op>::value) {
      T res[NE];
      int code[NE];
      int any = 0;
#pragma unroll
      for (int v = 0; v < VPT; v++)
#pragma unroll
        for (int k = 0; k < W; k++) {
          const int e = v * W + k;
          if constexpr (NIN == 2) res[e] = op.fast(vget(va[v], k), vget(vb[v], k), tab, code[e]);
          else res[e] = op.fast(vget(va[v], k), tab, code[e]);
          any |= code[e];
        }
      if (any) {
#pragma unroll
        for (int e = 0; e < NE; e++) {
          const int v = e / W, k = e % W;
          if (code[e]) {
            if constexpr (NIN == 2) res[e] = Op::slow(vget(va[v], k), vget(vb[v], k), res[e], code[e], tab);
            else res[e] = Op::slow(vget(va[v], k), res[e], code[e], tab);
          }
        }
      }
#pragma unroll
      for (int v = 0; v < VPT; v++) {
        V o;
#pragma unroll
        for (int k = 0; k < W; k++) vget(o, k) = res[v * W + k];
        __stcs(ov + v * kThreads + tid, o);
      }
    } else {
#pragma unroll
      for (int v = 0; v < VPT; v++) {
        V o;
#pragma unroll
        for (int k = 0; k < W; k++) {
          if constexpr (NIN == 2) vget(o, k) = op(vget(va[v], k), vget(vb[v], k), tab);
          else vget(o, k) = op(vget(va[v], k), tab);
        }
        __stcs(ov + v * kThreads + tid, o);
      }
    }
  }
  if constexpr (HasTriv<Op>::value) {  // the last, partial row of the warp's stack
    if (lane < qn) {
      const T* qy = NIN == 2 ? s_qy[(tid >> 5) % (NIN == 2 ? NW : 1)] : s_qx[tid >> 5];
      __stcs(out + qelem(s_qi[tid >> 5][lane]), eval_one<Op, NIN>(op, s_qx[tid >> 5][lane], qy[lane], tab));
    }
  }
  // remainder (< one tile)
  const size_t done = ntiles * TILE_E;
  for (size_t i = done + (size_t)blockIdx.x * kThreads + tid; i < n; i += G * kThreads) {
    if constexpr (NIN == 2) out[i] = op(a[i], b[i], tab);
    else out[i] = op(a[i], tab);
  }
}

// ------------------------------------------------ trig selector kernel
// sin / cos / tan f64 (u10, u35) with the reference's per-lane reduction
// selector (reduction.hpp:189-206: Cody-Waite 1 / 2 below 1e14, Payne-Hanek
// above).  TMA pipeline as k_stream, but stages are released per warp
// (tma::stage_release_last): no CTA barrier per tile, warps drift by up to
// STAGES - 1 tiles, so a warp with more Payne-Hanek work does not hold the
// others.  Per tile, every warp (32 x NE elements, NE = 2 VPT <= 8):
//   0. all elements |x| < 15      -> branch-free Cody-Waite-1 bodies from
//      registers (config 1); all elements Payne-Hanek -> branch-free Op::ph
//      bodies (config 3-like inputs through the selector);
//   1. otherwise a class per element from its high word: Payne-Hanek (high
//      word > that of 1e14, incl. Inf/NaN, for which Op::ph returns the
//      canonical NaN like every other path), Cody-Waite (2^-27 <= |x| and
//      high word <= that of 1e14; the per-lane selector decides at the
//      boundary word), trivial (|x| < 2^-27: sin/tan x, cos 1.0, Op::tiny);
//   2. the warp's arguments go to a shared-memory block in slot order (slot
//      = e * 32 + lane; conflict-free), trivial ones already replaced by their
//      result, and one warp scan of the packed per-lane counts
//      (nph << 16 | ncw) builds the list of non-trivial slots (8 bits each),
//      Payne-Hanek slots first;
//   3. full Payne-Hanek rows of the list run Op::ph (two rows interleaved, no
//      divergence); the boundary row and the Cody-Waite rows run the
//      per-lane selector op(); each result overwrites its argument's slot;
//   4. the block is stored in slot order: conflict-free LDS, coalesced
//      16-byte st.global.cs.
// 2.25 KB of scratch per warp and the lazily staged Payne-Hanek window
// (w1 | w2, 16.4 KB): with 2 x 16 KB stages the CTA needs 68 KB, so 3 CTAs
// (24 warps, <= 80 registers) fit.
template <class Op, int TABLE, int VPT, int STAGES, int MINB>
__global__ void __launch_bounds__(kThreads, MINB) k_trig(const double* __restrict__ a, double* __restrict__ out,
                                                         size_t n) {
  using V = double2;
  constexpr int W = 2;
  constexpr int TILE_V = kThreads * VPT;
  constexpr uint32_t TILE_BYTES = TILE_V * 16;
  constexpr int TILE_E = TILE_V * W;
  constexpr int NE = VPT * W;  // elements per lane per tile
  constexpr int WE = 32 * NE;  // elements per warp per tile
  constexpr int NW = kThreads / 32;
  static_assert(WE <= 256, "positions are kept in 8 bits");
  extern __shared__ __align__(128) unsigned char dsm[];
  __shared__ uint64_t bars[STAGES];
  __shared__ uint32_t rel[STAGES];
  __shared__ __align__(16) double stab[TableSize<TABLE>::n];
  __shared__ __align__(16) double s_x[NW][WE];  // per warp: arguments in slot order, then results in place
  __shared__ unsigned char s_i[NW][WE];         // per warp: non-trivial slots, Payne-Hanek first
  V* buf = reinterpret_cast<V*>(dsm);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double* sx = s_x[warp];
  unsigned char* si = s_i[warp];
  if (tid == 0) {
#pragma unroll
    for (int s = 0; s < STAGES; s++) tma::mbar_init(&bars[s], 1);
    tma::fence_barrier_init();
  }
  if (tid < STAGES) rel[tid] = 0;
  __shared__ int s_phready;  // the Payne-Hanek window is staged (stage_ph_lazy)
  if (tid == 0) s_phready = 0;
  bool have_ph = false;      // this warp has seen it staged
  const double* tab = stage_table<TABLE, true>(stab);  // includes __syncthreads()
  tma::griddep_wait();  // inputs / outputs may belong to the previous grid
  tma::griddep_launch_dependents();
  Op op;
  const size_t ntiles = n / TILE_E;
  const size_t G = gridDim.x;
  const size_t my = ntiles > blockIdx.x ? (ntiles - blockIdx.x + G - 1) / G : 0;
  const uint64_t pol = tma::policy_evict_first();
  auto issue = [&](int s, size_t tile) {
    tma::mbar_expect_tx(&bars[s], TILE_BYTES);
    tma::bulk_g2s(buf + (size_t)s * TILE_V, reinterpret_cast<const V*>(a) + tile * TILE_V, TILE_BYTES, &bars[s],
                  pol);
  };
  if (tid == 0)
    for (int s = 0; s < STAGES && (size_t)s < my; s++) issue(s, blockIdx.x + (size_t)s * G);
  for (size_t j = 0; j < my; j++) {
    const int s = (int)(j % STAGES);
    tma::mbar_wait(&bars[s], (uint32_t)((j / STAGES) & 1));
    double xe[NE];
#pragma unroll
    for (int v = 0; v < VPT; v++) {
      const V t = buf[(size_t)s * TILE_V + v * kThreads + tid];
      xe[v * W] = t.x;
      xe[v * W + 1] = t.y;
    }
    __syncwarp();  // the warp's reads of stage s are done -> release it
    if (lane == 0 && tma::stage_release_last(&rel[s], NW) && j + STAGES < my) {
      tma::fence_proxy_async_smem();
      issue(s, blockIdx.x + (j + STAGES) * G);
    }
    V* ov = reinterpret_cast<V*>(out) + (blockIdx.x + j * G) * TILE_V;
    // ---- 0. uniform warps
    bool small = true;
#pragma unroll
    for (int e = 0; e < NE; e++) small = small && Op::is_cw1(xe[e]);
    if (__all_sync(0xffffffffu, small)) {
#pragma unroll
      for (int v = 0; v < VPT; v++) __stcs(ov + v * kThreads + tid, make_double2(op.cw1(xe[v * W], tab),
                                                                                   op.cw1(xe[v * W + 1], tab)));
      continue;
    }
    // ---- 1. classes from the high word (bit e of mph / mcw)
    uint32_t mph = 0, mcw = 0;
#pragma unroll
    for (int e = 0; e < NE; e++) {
      const uint32_t h = (uint32_t)__double2hiint(xe[e]) & 0x7fffffffu;
      mph |= (uint32_t)(h > 0x42D6BCC4u) << e;                        // |x| > 1e14 or non-finite
      mcw |= (uint32_t)(h - 0x3E400000u <= 0x42D6BCC4u - 0x3E400000u) << e;  // 2^-27 <= |x| <~ 1e14
    }
    if (!have_ph) {  // any element the selector may send to Payne-Hanek (boundary word included)
      uint32_t hm = 0;
#pragma unroll
      for (int e = 0; e < NE; e++) hm = max(hm, (uint32_t)__double2hiint(xe[e]) & 0x7fffffffu);
      if (__any_sync(0xffffffffu, hm >= 0x42D6BCC4u)) {
        stage_ph_lazy(stab + kSinCosCoefN, &s_phready);
        have_ph = true;
      }
    }
    if (__all_sync(0xffffffffu, mph == (1u << NE) - 1u)) {
#pragma unroll
      for (int v = 0; v < VPT; v++) {
        const double x0 = xe[v * W], x1 = xe[v * W + 1];
        __stcs(ov + v * kThreads + tid, make_double2(op.ph(x0, tab), op.ph(x1, tab)));
      }
      continue;
    }
    // ---- 2. placement: the arguments in slot order (slot = e * 32 + lane,
    // trivial ones already replaced by their result), plus a list of the
    // non-trivial slots, Payne-Hanek first, from one scan of the packed
    // per-lane counts
    const int cnt = (__popc(mph) << 16) | __popc(mcw);
    int inc = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += t;
    }
    const int tot = __shfl_sync(0xffffffffu, inc, 31);
    const int nph = tot >> 16, nall = nph + (tot & 0xffff);
    const int exc = inc - cnt;
    int pph = exc >> 16;
    int pcw = nph + (exc & 0xffff);
#pragma unroll
    for (int e = 0; e < NE; e++) {
      const bool isph = (mph >> e) & 1u, iscw = (mcw >> e) & 1u;
      const int slot = e * 32 + lane;
      sx[slot] = (isph || iscw) ? xe[e] : Op::tiny(xe[e]);
      VEM_ASSERT(!(isph || iscw) || ((isph ? pph : pcw) < WE && (isph ? pph < nph : pcw < nall)));
      if (isph || iscw) si[isph ? pph : pcw] = (unsigned char)slot;
      pph += isph;
      pcw += iscw;
    }
    __syncwarp();
    // ---- 3. rows over the slot list, results in place
    int r = 0;
#pragma unroll 1
    for (; (r + 2) * 32 <= nph; r += 2) {
      const int sa = si[r * 32 + lane], sb = si[r * 32 + 32 + lane];
      VEM_ASSERT((r + 2) * 32 <= nph && sa < WE && sb < WE);
      const double xa = sx[sa], xb = sx[sb];
      const double ya = op.ph(xa, tab), yb = op.ph(xb, tab);
      sx[sa] = ya;
      sx[sb] = yb;
    }
    if ((r + 1) * 32 <= nph) {
      const int sa = si[r * 32 + lane];
      sx[sa] = op.ph(sx[sa], tab);
      r++;
    }
#pragma unroll 1
    for (; r * 32 < nall; r++) {
      const int i = r * 32 + lane;
      if (i < nall) {
        const int sa = si[i];
        sx[sa] = op(sx[sa], tab);
      }
    }
    __syncwarp();
    // ---- 4. coalesced store straight from the slot-order block
#pragma unroll
    for (int v = 0; v < VPT; v++)
      __stcs(ov + v * kThreads + tid, make_double2(sx[(v * W) * 32 + lane], sx[(v * W + 1) * 32 + lane]));
    __syncwarp();  // the block is rewritten by the next tile
  }
  // remainder (< one tile): per-lane selector; a warp with a Payne-Hanek
  // element stages the window first
  const size_t done = ntiles * TILE_E;
  for (size_t i0 = done + (size_t)blockIdx.x * kThreads + (tid & ~31); i0 < n; i0 += G * kThreads) {
    const size_t i = i0 + lane;
    const double x = i < n ? a[i] : 0.0;
    if (!have_ph && __any_sync(0xffffffffu, ((uint32_t)__double2hiint(x) & 0x7fffffffu) >= 0x42D6BCC4u)) {
      stage_ph_lazy(stab + kSinCosCoefN, &s_phready);
      have_ph = true;
    }
    if (i < n) out[i] = op(x, tab);
  }
}

// ------------------------------------------------------- fmod: step queue
// fmod's cost is data dependent: ceil(E/50) exact 50-bit long-division steps
// (E = exponent gap, config 4 f64: 0 for the half of the pairs with |x| < |y|,
// up to 42 otherwise).  Per TMA tile (TILE_E pairs):
//   1. triage on the operand bits, every element: NaN / Inf / zero divisor /
//      |x| <= |y| are finished at once into the tile's output block in
//      shared memory; the others get a sort key (steps estimated from the
//      biased exponents) and a rank from a shared-memory histogram atomic;
//   2. one warp-level suffix scan of the histogram (every warp redundantly:
//      no extra barrier) gives each key its queue offset, heaviest first;
//      the pending pairs are written to the queue in that order;
//   3. the warps take queue rows of 32 (snake order over the 8 warps for
//      balance): the lanes of a row hold pairs of (nearly) the same step
//      count, so the long division runs converged with no idle lanes;
//      results go back into the output block at their tile slots;
//   4. the output block is stored coalesced (16-byte st.global.cs).
// Per element the math is fmod_pend_setup / fmod_stepn50 / fmod_pend_finish (exact),
// so results are bit-identical to the oracle and to glibc.
// Pending pair (|x| > |y| > 0, both finite) after setup: r == (mn 2^s0) mod md, signed,
// with `steps` full 50-bit steps to go (fmod_stepn50); result = +-(r mod md) 2^ed.
struct fmod_pend {
  double r, md, rmd;  // r signed in (-md, md); rmd = RN(1/md) 2^50
  int steps, ed;
  uint32_t sx;  // sign word of x
};
__device__ __forceinline__ fmod_pend fmod_pend_setup(double x, double y) {
  fmod_pend p;
  const uint32_t hx = (uint32_t)__double2hiint(x), hy = (uint32_t)__double2hiint(y);
  const int bx = (int)((hx >> 20) & 0x7ffu), by = (int)((hy >> 20) & 0x7ffu);
  p.sx = hx & 0x80000000u;
  double mn, md;
  int E;
  if (bx != 0 && by != 0) {  // normal operands: mantissas by bit surgery
    mn = __hiloint2double((int)((hx & 0x000fffffu) | 0x3ff00000u), __double2loint(x));
    md = __hiloint2double((int)((hy & 0x000fffffu) | 0x3ff00000u), __double2loint(y));
    E = bx - by;
    p.ed = by - 1023;
  } else {  // a subnormal operand (rare)
    const double n = fabs(x), d = fabs(y);
    const int en = ilogb_pos(n), ed = ilogb_pos(d);
    mn = mant_1_2(n, en);
    md = mant_1_2(d, ed);
    E = en - ed;
    p.ed = ed;
  }
  p.md = md;
  const double rmd = __drcp_rn(md);  // RN(1/md): the signed step's bound (fmod_stepn_rs)
  p.rmd = rmd * 0x1p50;
  // E >= 0; (E - 1) / 50 for E - 1 in [0, 2100] (and 0 for E = 0)
  p.steps = E == 0 ? 0 : (int)(((uint32_t)(E - 1) * 1311u) >> 16);
  // first step of s0 = E - 50 steps in [1, 50] bits (E = 0: 0 bits, mn - {1,2} md)
  p.r = fmod_stepn_rs(mn * __hiloint2double((1023 + E - 50 * p.steps) << 20, 0), md, rmd);
  return p;
}
__device__ __forceinline__ double fmod_pend_finish(const fmod_pend& p) {
  // signed r in (-md, md) -> [0, md), a multiple of 2^-52: r 2^ed is normal
  // when ed >= -970
  const double r = p.r < 0.0 ? p.r + p.md : p.r;
  const double m = p.ed >= -970 ? r * __hiloint2double((p.ed + 1023) << 20, 0) : ldexp2(r, p.ed);
  return __hiloint2double(__double2hiint(m) | (int)p.sx, __double2loint(m));
}

// Queue ops for fmod (the binary kernel below): triage on the operand bits,
// key = estimated 50-bit steps, exact long division for the queue rows.
template <class T>
struct FmodQ {
  // every slot gets its trivial result (pending slots are overwritten later)
  __device__ static bool triage(T x, T y, T& res, int& key) {
    const T nx = fabs(x), ny = fabs(y);
    const bool nan_res = !(nx < (T)kInf) || !(ny > (T)0);  // x NaN/Inf, y NaN/0
    const bool ret_x = nx < ny;                            // incl. y = +-Inf
    res = ret_x ? x : copysign((T)0, x);                   // |x| == |y| -> +-0
    res = nan_res ? (sizeof(T) == 8 ? (T)from_bits_d(kCanonNanD) : (T)from_bits_f(kCanonNanF)) : res;
    if (nan_res || ret_x || nx == ny) return false;
    uint32_t hx, hy;
    int gap;
    if constexpr (sizeof(T) == 8) {
      hx = (uint32_t)__double2hiint((double)x);
      hy = (uint32_t)__double2hiint((double)y);
      gap = (int)((hx >> 20) & 0x7ffu) - (int)((hy >> 20) & 0x7ffu);
    } else {
      hx = bits_f((float)x);
      hy = bits_f((float)y);
      gap = (int)((hx >> 23) & 0xffu) - (int)((hy >> 23) & 0xffu);
    }
    key = gap <= 0 ? 0 : min((int)(((uint32_t)(gap - 1) * 1311u) >> 16), 63);
    return true;
  }
  __device__ static T eval_full(T x, T y, const double*) {
    if constexpr (sizeof(T) == 8) return fmod_d(x, y);
    else return fmod_f(x, y);
  }
  __device__ static T eval1(T x, T y, const double*) {
    fmod_pend A = fmod_pend_setup((double)x, (double)y);
    // the lanes of a queue row have (nearly) the same step count: four steps
    // per trip keep the loop control off the dependent chain
    int k = A.steps;
#pragma unroll 1
    for (; k >= 4; k -= 4) {
      A.r = fmod_stepn50(A.r, A.md, A.rmd);
      A.r = fmod_stepn50(A.r, A.md, A.rmd);
      A.r = fmod_stepn50(A.r, A.md, A.rmd);
      A.r = fmod_stepn50(A.r, A.md, A.rmd);
    }
#pragma unroll 1
    for (; k > 0; k--) A.r = fmod_stepn50(A.r, A.md, A.rmd);
    return (T)fmod_pend_finish(A);
  }
  __device__ static void eval2(T xa, T ya, T xb, T yb, T& ra, T& rb, const double*) {
    fmod_pend A = fmod_pend_setup((double)xa, (double)ya);
    fmod_pend B = fmod_pend_setup((double)xb, (double)yb);
    // two independent chains interleaved, two steps of each per trip
    int i = min(A.steps, B.steps);
#pragma unroll 1
    for (; i >= 2; i -= 2) {
      A.r = fmod_stepn50(A.r, A.md, A.rmd);
      B.r = fmod_stepn50(B.r, B.md, B.rmd);
      A.r = fmod_stepn50(A.r, A.md, A.rmd);
      B.r = fmod_stepn50(B.r, B.md, B.rmd);
    }
    const int c = min(A.steps, B.steps) - i;
#pragma unroll 1
    for (int k = c; k < A.steps; k++) A.r = fmod_stepn50(A.r, A.md, A.rmd);
#pragma unroll 1
    for (int k = c; k < B.steps; k++) B.r = fmod_stepn50(B.r, B.md, B.rmd);
    ra = (T)fmod_pend_finish(A);
    rb = (T)fmod_pend_finish(B);
  }
};

// ------------------------------------------------ tile work-queue kernel
// For entry points whose per-element cost is data dependent (fmod: step
// count; the trig selector: Cody-Waite 1 / 2 / Payne-Hanek).  Per TMA tile:
//   1. triage: Q::triage finishes trivial elements into the tile's output
//      block in shared memory and gives the others a key (cost class) and a
//      rank from a shared-memory histogram atomic;
//   2. a warp-level suffix scan of the histogram (every warp redundantly: no
//      extra barrier) gives each key its queue offset, heaviest first; the
//      pending elements are written to the queue, which lives in the
//      consumed TMA stage (its refill is issued after step 3);
//   3. warps fetch units of ROWS x 32 queue entries dynamically (heaviest
//      first: list scheduling balances the warps); the lanes of a row hold
//      elements of (nearly) the same cost, so they run converged; ROWS = 2
//      gives each lane two independent chains (Q::eval2);
//   4. the output block is stored coalesced (16-byte st.global.cs).
// Results per element are the op's own (bit-identical to the oracle).
constexpr int kQKeys = 64;

template <class Q, class T, int NIN, int TABLE, int VPT, int STAGES, int MINB, int ROWS, int FETCH = 1>
__global__ void __launch_bounds__(kThreads, MINB) k_queue(const T* __restrict__ a, const T* __restrict__ b,
                                                          T* __restrict__ out, size_t n) {
  using V = typename Vec16<T>::type;
  constexpr int W = Vec16<T>::n;
  constexpr int TILE_V = kThreads * VPT;
  constexpr uint32_t TILE_BYTES = TILE_V * 16;
  constexpr int TILE_E = TILE_V * W;
  constexpr int NE = VPT * W;
  extern __shared__ __align__(128) unsigned char dsm[];
  __shared__ uint64_t bars[STAGES];
  __shared__ __align__(16) double stab[TableSize<TABLE>::n];
  __shared__ __align__(16) T so[TILE_E];  // output block (tile order)
  __shared__ unsigned short qi[TILE_E];
  __shared__ int hist[kQKeys + 1];  // + the unit-fetch counter
  __shared__ int qoff[kThreads / 32][kQKeys];  // per-warp copies of the queue offsets
  V* buf = reinterpret_cast<V*>(dsm);
  const int tid = threadIdx.x, lane = tid & 31;
  if (tid == 0) {
#pragma unroll
    for (int s = 0; s < STAGES; s++) tma::mbar_init(&bars[s], 1);
    tma::fence_barrier_init();
  }
  if (tid <= kQKeys) hist[tid] = 0;
  const double* tab = stage_table<TABLE>(stab);  // includes __syncthreads()
  if constexpr (TABLE == kNoTable) __syncthreads();
  tma::griddep_wait();
  tma::griddep_launch_dependents();
  const size_t ntiles = n / TILE_E;
  const size_t G = gridDim.x;
  const size_t my = ntiles > blockIdx.x ? (ntiles - blockIdx.x + G - 1) / G : 0;
  uint64_t pol = 0;
  auto issue = [&](int s, size_t tile) {
    tma::mbar_expect_tx(&bars[s], NIN * TILE_BYTES);
    tma::bulk_g2s(buf + (size_t)(s * NIN) * TILE_V, reinterpret_cast<const V*>(a) + tile * TILE_V, TILE_BYTES,
                  &bars[s], pol);
    if constexpr (NIN == 2)
      tma::bulk_g2s(buf + (size_t)(s * NIN + 1) * TILE_V, reinterpret_cast<const V*>(b) + tile * TILE_V,
                    TILE_BYTES, &bars[s], pol);
  };
  if (tid == 0) {
    pol = tma::policy_evict_first();
    for (int s = 0; s < STAGES && (size_t)s < my; s++) issue(s, blockIdx.x + (size_t)s * G);
  }
  for (size_t j = 0; j < my; j++) {
    const int s = (int)(j % STAGES);
    tma::mbar_wait(&bars[s], (uint32_t)((j / STAGES) & 1));
    T xe[NE], ye[NE];
#pragma unroll
    for (int v = 0; v < VPT; v++) {
      V va = buf[(size_t)(s * NIN) * TILE_V + v * kThreads + tid];
      V vb;
      if constexpr (NIN == 2) vb = buf[(size_t)(s * NIN + 1) * TILE_V + v * kThreads + tid];
#pragma unroll
      for (int k = 0; k < W; k++) {
        xe[v * W + k] = vget(va, k);
        ye[v * W + k] = NIN == 2 ? vget(vb, k) : (T)0;
      }
    }
    V* ov = reinterpret_cast<V*>(out) + (blockIdx.x + j * G) * TILE_V;
    __syncthreads();  // stage consumed; previous tile's output block stored
    T* qx = reinterpret_cast<T*>(buf + (size_t)(s * NIN) * TILE_V);
    T* qy = reinterpret_cast<T*>(buf + (size_t)(s * NIN + (NIN - 1)) * TILE_V);
    // ---- 1. triage
    int key[NE], rank[NE];
#pragma unroll
    for (int e = 0; e < NE; e++) {
      const int slot = ((e / W) * kThreads + tid) * W + (e % W);
      T res;
      key[e] = -1;
      int k;
      if (Q::triage(xe[e], ye[e], res, k)) {
        key[e] = k;
        rank[e] = (int)tma::smem_atomic_inc(&hist[k]);
      }
      so[slot] = res;
    }
    __syncthreads();
    // ---- 2. queue offsets: suffix scan over keys (heaviest first), per warp
    const int h0 = hist[2 * lane], h1 = hist[2 * lane + 1];
    int suf = h0 + h1;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const int t = __shfl_down_sync(0xffffffffu, suf, off);
      if (lane + off < 32) suf += t;
    }
    const int Qn = __shfl_sync(0xffffffffu, suf, 0);
    const int base_odd = suf - h0 - h1;  // keys > 2*lane+1
    const int base_even = base_odd + h1;
    // this warp's copy of the 64 queue offsets (one LDS per element below
    // instead of two shuffles)
    int* offs = qoff[tid >> 5];
    offs[2 * lane] = base_even;
    offs[2 * lane + 1] = base_odd;
    __syncwarp();
#pragma unroll
    for (int e = 0; e < NE; e++) {
      if (key[e] >= 0) {
        const int pos = offs[key[e]] + rank[e];
        VEM_ASSERT(pos >= 0 && pos < Qn && Qn <= TILE_E);
        qx[pos] = xe[e];
        if constexpr (NIN == 2) qy[pos] = ye[e];
        qi[pos] = (unsigned short)(((e / W) * kThreads + tid) * W + (e % W));
      }
    }
    __syncthreads();
    // ---- 3. queue units, fetched dynamically heaviest first; lanes past the
    // end duplicate the unit's first entry (same cost class, result dropped)
    // (FETCH units per atomic: consecutive units have nearly the same cost)
    const int nunits = (Qn + 32 * ROWS - 1) / (32 * ROWS);
    // FETCH == 0: static snake order over the warps (round k: unit 8k + w
    // for even k, 8k + 7 - w for odd k) -- the units are sorted heaviest
    // first, so consecutive rounds balance; no atomic per unit.
    // FETCH > 0: dynamic fetch of FETCH units per shared-memory atomic.
    constexpr int kNW = kThreads / 32;
    const int wq = tid >> 5;
    for (int u0 = 0, rnd = 0;; rnd++) {
      if constexpr (FETCH == 0) {
        u0 = rnd * kNW + ((rnd & 1) ? kNW - 1 - wq : wq);
      } else {
        if (lane == 0) u0 = (int)tma::smem_atomic_add(&hist[kQKeys], FETCH);
        u0 = __shfl_sync(0xffffffffu, u0, 0);
      }
      if (u0 >= nunits) break;  // (snake: every later round's unit is larger)
#pragma unroll 1
      for (int u = u0; u < u0 + (FETCH == 0 ? 1 : FETCH) && u < nunits; u++) {
        const int p0 = u * 32 * ROWS;
        const int pa = p0 + lane, ca = pa < Qn ? pa : p0;
        if constexpr (ROWS == 1) {
          const T r = Q::eval1(qx[ca], NIN == 2 ? qy[ca] : (T)0, tab);
          VEM_ASSERT(ca >= 0 && ca < Qn && (pa >= Qn || qi[pa] < TILE_E));
          if (pa < Qn) so[qi[pa]] = r;
        } else {
          const int pb = pa + 32, cb = pb < Qn ? pb : p0;
          T ra, rb;
          Q::eval2(qx[ca], NIN == 2 ? qy[ca] : (T)0, qx[cb], NIN == 2 ? qy[cb] : (T)0, ra, rb, tab);
          if (pa < Qn) so[qi[pa]] = ra;
          if (pb < Qn) so[qi[pb]] = rb;
        }
      }
    }
    __syncthreads();
    if (tid <= kQKeys) hist[tid] = 0;  // for the next tile (ranks and fetches consumed)
    if (tid == 0 && j + STAGES < my) {  // the queue's stage is free: refill it
      tma::fence_proxy_async_smem();
      issue(s, blockIdx.x + (j + STAGES) * G);
    }
    // ---- 4. coalesced store of the output block
    const V* sv = reinterpret_cast<const V*>(so);
#pragma unroll
    for (int v = 0; v < VPT; v++) __stcs(ov + v * kThreads + tid, sv[v * kThreads + tid]);
  }
  // remainder (< one tile): the full per-element function
  const size_t done = ntiles * TILE_E;
  for (size_t i = done + (size_t)blockIdx.x * kThreads + tid; i < n; i += G * kThreads)
    out[i] = Q::eval_full(a[i], NIN == 2 ? b[i] : (T)0, tab);
}

#ifdef VEM_TUNE
// ------------------------------------------- warp-private work queue
// (tuning build only: fmod_f shipped it until the straight-line fmod_f_flat)
// Same four steps as k_queue, but every warp owns its chunks (32 x NE
// elements), TMA stages, mbarriers, histogram and queue: no CTA barriers, so
// a warp with a heavy queue never holds the others back.
template <class Q, class T, int NIN, int VPT, int STAGES, int MINB>
__global__ void __launch_bounds__(kThreads, MINB) k_wqueue(const T* __restrict__ a, const T* __restrict__ b,
                                                           T* __restrict__ out, size_t n) {
  using V = typename Vec16<T>::type;
  constexpr int W = Vec16<T>::n;
  constexpr int NW = kThreads / 32;
  constexpr int CH_V = 32 * VPT;  // 16-byte vectors per input per chunk
  constexpr uint32_t CH_BYTES = CH_V * 16;
  constexpr int CH_E = CH_V * W;
  constexpr int NE = VPT * W;
  extern __shared__ __align__(128) unsigned char dsm[];
  __shared__ uint64_t bars[NW][STAGES];
  __shared__ __align__(16) T so_all[NW][CH_E];
  __shared__ unsigned short qi_all[NW][CH_E];
  __shared__ int hist_all[NW][kQKeys];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  V* buf = reinterpret_cast<V*>(dsm) + (size_t)warp * STAGES * NIN * CH_V;
  T* so = so_all[warp];
  unsigned short* qi = qi_all[warp];
  int* hist = hist_all[warp];
  uint64_t* bar = bars[warp];
  if (lane == 0) {
#pragma unroll
    for (int s = 0; s < STAGES; s++) tma::mbar_init(&bar[s], 1);
    tma::fence_barrier_init();
  }
  hist[lane] = 0;
  hist[lane + 32] = 0;
  __syncwarp();
  tma::griddep_wait();
  tma::griddep_launch_dependents();
  const size_t nch = n / CH_E;
  const size_t GW = (size_t)gridDim.x * NW;
  const size_t gw = (size_t)blockIdx.x * NW + warp;
  const size_t my = nch > gw ? (nch - gw + GW - 1) / GW : 0;
  uint64_t pol = 0;
  auto issue = [&](int s, size_t ch) {
    tma::mbar_expect_tx(&bar[s], NIN * CH_BYTES);
    tma::bulk_g2s(buf + (size_t)(s * NIN) * CH_V, reinterpret_cast<const V*>(a) + ch * CH_V, CH_BYTES, &bar[s], pol);
    if constexpr (NIN == 2)
      tma::bulk_g2s(buf + (size_t)(s * NIN + 1) * CH_V, reinterpret_cast<const V*>(b) + ch * CH_V, CH_BYTES, &bar[s],
                    pol);
  };
  if (lane == 0) {
    pol = tma::policy_evict_first();
    for (int s = 0; s < STAGES && (size_t)s < my; s++) issue(s, gw + (size_t)s * GW);
  }
  for (size_t j = 0; j < my; j++) {
    const int s = (int)(j % STAGES);
    tma::mbar_wait(&bar[s], (uint32_t)((j / STAGES) & 1));
    T xe[NE], ye[NE];
#pragma unroll
    for (int v = 0; v < VPT; v++) {
      V va = buf[(size_t)(s * NIN) * CH_V + v * 32 + lane];
      V vb;
      if constexpr (NIN == 2) vb = buf[(size_t)(s * NIN + 1) * CH_V + v * 32 + lane];
#pragma unroll
      for (int k = 0; k < W; k++) {
        xe[v * W + k] = vget(va, k);
        ye[v * W + k] = NIN == 2 ? vget(vb, k) : (T)0;
      }
    }
    __syncwarp();  // stage consumed (it holds the queue until the rows are done)
    T* qx = reinterpret_cast<T*>(buf + (size_t)(s * NIN) * CH_V);
    T* qy = reinterpret_cast<T*>(buf + (size_t)(s * NIN + (NIN - 1)) * CH_V);
    int key[NE], rank[NE];
#pragma unroll
    for (int e = 0; e < NE; e++) {
      const int slot = ((e / W) * 32 + lane) * W + (e % W);
      T res;
      key[e] = -1;
      int k;
      if (Q::triage(xe[e], ye[e], res, k)) {
        key[e] = k;
        rank[e] = atomicAdd(&hist[k], 1);
      }
      so[slot] = res;
    }
    __syncwarp();
    const int h0 = hist[2 * lane], h1 = hist[2 * lane + 1];
    int suf = h0 + h1;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const int t = __shfl_down_sync(0xffffffffu, suf, off);
      if (lane + off < 32) suf += t;
    }
    const int Qn = __shfl_sync(0xffffffffu, suf, 0);
    const int base_odd = suf - h0 - h1;
    const int base_even = base_odd + h1;
    hist[2 * lane] = 0;  // this lane's two counters are read: reset for the next chunk
    hist[2 * lane + 1] = 0;
#pragma unroll
    for (int e = 0; e < NE; e++) {
      const int k = key[e] < 0 ? 0 : key[e];
      const int bo = __shfl_sync(0xffffffffu, base_odd, k >> 1);
      const int be = __shfl_sync(0xffffffffu, base_even, k >> 1);
      if (key[e] >= 0) {
        const int pos = ((k & 1) ? bo : be) + rank[e];
        qx[pos] = xe[e];
        if constexpr (NIN == 2) qy[pos] = ye[e];
        qi[pos] = (unsigned short)(((e / W) * 32 + lane) * W + (e % W));
      }
    }
    __syncwarp();
    // rows in pairs, heaviest first; lanes past the end duplicate entry p0
    for (int p0 = 0; p0 < Qn; p0 += 64) {
      const int pa = p0 + lane, pb = pa + 32;
      const int ca = pa < Qn ? pa : p0, cb = pb < Qn ? pb : p0;
      T ra, rb;
      Q::eval2(qx[ca], NIN == 2 ? qy[ca] : (T)0, qx[cb], NIN == 2 ? qy[cb] : (T)0, ra, rb, nullptr);
      if (pa < Qn) so[qi[pa]] = ra;
      if (pb < Qn) so[qi[pb]] = rb;
    }
    __syncwarp();
    if (lane == 0 && j + STAGES < my) {
      tma::fence_proxy_async_smem();
      issue(s, gw + (j + STAGES) * GW);
    }
    V* ov = reinterpret_cast<V*>(out) + (gw + j * GW) * CH_V;
    const V* sv = reinterpret_cast<const V*>(so);
#pragma unroll
    for (int v = 0; v < VPT; v++) __stcs(ov + v * 32 + lane, sv[v * 32 + lane]);
    __syncwarp();
  }
  const size_t done = nch * CH_E;
  const size_t tg = (size_t)blockIdx.x * kThreads + tid;
  for (size_t i = done + tg; i < n; i += (size_t)gridDim.x * kThreads)
    out[i] = Q::eval_full(a[i], NIN == 2 ? b[i] : (T)0, nullptr);
}

// Work-ring fmod kernel (superseded by the regrouped streaming kernel,
// OpFmodD/OpFmodF below; kept in the tuning build for comparison).
// ------------------------------------------------------------ fmod
// The remainder loop runs ceil(E/50) steps, E = exponent gap of |x| and |y|;
// a plain SIMT loop makes every lane wait for its warp's slowest element
// (config 4: mean ~7 vs warp-max ~30 steps).  Two phases per warp instead:
//   1. setup, uniform over a chunk of 64 elements (coalesced loads, one
//      division each): trivial elements (|x| < |y|, specials, equal
//      exponents) are finished and stored at once; the others are appended,
//      compacted by ballot + prefix popcount, to a per-warp work ring in
//      shared memory (r, md, 1/md, E, ed|sign: 32 B);
//   2. long division: every active lane takes one 50-bit step; whenever at
//      least kRefill lanes are idle they pull the next ring entries.
// So lanes only idle while the ring is empty; per-element math is the
// oracle's (setup / step / finish), hence bit-identical results.
constexpr int kFmodWarps = 4;        // 128-thread CTAs
constexpr int kFmodChunk = 64;       // elements per warp per phase 1
constexpr int kFmodRing = 64;        // ring entries per warp (>= chunk)
constexpr int kRefill = 8;

template <class T, int MINB = 1>
__global__ void __launch_bounds__(kFmodWarps * 32, MINB) k_fmod(const T* __restrict__ a, const T* __restrict__ b,
                                                          T* __restrict__ out, size_t n) {
  __shared__ double s_r[kFmodWarps][kFmodRing], s_md[kFmodWarps][kFmodRing], s_rmd[kFmodWarps][kFmodRing];
  __shared__ int2 s_e[kFmodWarps][kFmodRing];
  __shared__ unsigned long long s_g[kFmodWarps][kFmodRing];
  const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
  const unsigned lt_mask = (1u << lane) - 1u;
  const size_t W = (size_t)gridDim.x * kFmodWarps;
  const size_t w = (size_t)blockIdx.x * kFmodWarps + wl;
  const size_t nch = (n + kFmodChunk - 1) / kFmodChunk;
  const size_t mych = nch > w ? (nch - w + W - 1) / W : 0;
  unsigned head = 0, tail = 0;  // ring consumer / producer counters (warp-uniform)
  fmod_state st = {0.0, 1.0, 1.0, 1.0, 0, 0};
  size_t gi = 0;
  bool active = false;  // stepping
  bool pend = false;    // finished, result not stored yet (stored at the next refill)

  auto step_all = [&]() {
    if (active) {
      st.r = fmod_stepn50(st.r, st.md, st.rmd);
      if (--st.E == 0) {
        active = false;
        pend = true;
      }
    }
  };
  // finishing is deferred into the (divergent) refill block, so the step
  // loop itself carries no per-iteration finish code
  auto refill = [&](bool force) {
    unsigned idle = __ballot_sync(0xffffffffu, !active);
    int nidle = __popc(idle);
    unsigned avail = tail - head;
    if (nidle == 0 || (!force && (nidle < kRefill || avail == 0u))) return;
    unsigned k = head + __popc(idle & lt_mask);
    if (!active) {
      if (pend) {
        __stcs(out + gi, (T)fmod_finish(st));
        pend = false;
      }
      if (k < tail) {
        int sl = (int)(k % kFmodRing);
        st.r = s_r[wl][sl];
        st.md = s_md[wl][sl];
        st.rmd = s_rmd[wl][sl];
        int2 e = s_e[wl][sl];
        st.E = e.x;
        st.ed = e.y >> 1;
        st.x = (e.y & 1) ? -1.0 : 1.0;
        gi = (size_t)s_g[wl][sl];
        active = true;
      }
    }
    head += min((unsigned)nidle, avail);
    __syncwarp();
  };

  for (size_t j = 0; j < mych; j++) {
    // ---- phase 1: setup a chunk, compact the non-trivial elements into the ring
    const size_t base = (w + j * W) * kFmodChunk;
    const size_t valid = min((size_t)kFmodChunk, n - base);
    T xv[kFmodChunk / 32], yv[kFmodChunk / 32];
#pragma unroll
    for (int k = 0; k < kFmodChunk / 32; k++) {
      size_t e = (size_t)(k * 32 + lane);
      xv[k] = e < valid ? __ldcs(a + base + e) : (T)0;
      yv[k] = e < valid ? __ldcs(b + base + e) : (T)1;
    }
#pragma unroll
    for (int k = 0; k < kFmodChunk / 32; k++) {
      size_t e = (size_t)(k * 32 + lane);
      fmod_state s0;
      double res;
      bool in = e < valid;
      bool todo = false;
      if (in) {
        if (fmod_setup((double)xv[k], (double)yv[k], s0, res)) __stcs(out + base + e, (T)res);
        else todo = true;
      }
      unsigned m = __ballot_sync(0xffffffffu, todo);
      if (todo) {
        int sl = (int)((tail + __popc(m & lt_mask)) % kFmodRing);
        s_r[wl][sl] = s0.r;
        s_md[wl][sl] = s0.md;
        s_rmd[wl][sl] = s0.rmd;
        s_e[wl][sl] = make_int2(s0.E, (s0.ed << 1) | (s0.x < 0.0 ? 1 : 0));
        s_g[wl][sl] = (unsigned long long)(base + e);
      }
      tail += __popc(m);
    }
    __syncwarp();
    // ---- phase 2: refill, then step (two per check) until at least kRefill
    // lanes are idle; leave when the ring is empty (next chunk's setup)
    while (true) {
      refill(false);
      if (tail == head) break;
      do {
        step_all();
        step_all();
      } while (__popc(__ballot_sync(0xffffffffu, !active)) < kRefill);
    }
  }
  // ---- drain
  while (__any_sync(0xffffffffu, active)) {
    step_all();
    step_all();
    refill(true);
  }
  if (pend) __stcs(out + gi, (T)fmod_finish(st));
}

#endif  // VEM_TUNE

// ------------------------------------------------------------- functors
#define VEM_UNARY_OP(NAME, T, EXPR)                                                   \
  struct NAME {                                                                       \
    __device__ __forceinline__ T operator()(T x, const double* tab) const { return EXPR; } \
  };
// Trivial trig inputs: |x| < 2^-27 (incl. zeros and subnormals) and non-finite
// x.  For |x| < 2^-27 every sin/tan form returns x exactly and every cos form
// 1.0 (the polynomial terms are below half an ulp: |x|^3/6 < 2^-54 |x|,
// x^2/2 < 2^-55), and the selector's own finals give +-0 -> x / 1.0 and
// Inf/NaN -> the canonical NaN; the GPU parity and digest tests pin this on
// random bit patterns.
__device__ __forceinline__ bool trig_is_trivial(double x) {
  const uint32_t h = (uint32_t)__double2hiint(x) & 0x7fffffffu;
  return h < 0x3E400000u || h >= 0x7ff00000u;
}
#define VEM_TRIG_OP(NAME, FN, ...)                                                       \
  struct NAME {                                                                          \
    __device__ __forceinline__ double operator()(double x, const double* tab) const {   \
      return FN<kSel>(x, tab + kSinCosCoefN __VA_ARGS__);                                 \
    }                                                                                    \
    __device__ __forceinline__ double cw1(double x, const double* tab) const {          \
      return FN<kCw1>(x, tab + kSinCosCoefN __VA_ARGS__);                                 \
    }                                                                                    \
    __device__ __forceinline__ double ph(double x, const double* tab) const {           \
      return FN<kPh>(x, tab + kSinCosCoefN __VA_ARGS__);                                  \
    }                                                                                    \
    __device__ __forceinline__ static bool is_cw1(double x) { return trig_is_cw1(x); } \
    __device__ __forceinline__ static bool is_trivial(double x) { return trig_is_trivial(x); } \
    __device__ static double trivial(double x);                                          \
    __device__ static double tiny(double x);                                             \
  };
// selector variants: `tab` = staged coefficients, then the PH window words
VEM_TRIG_OP(OpSinD, sin_d_u10, , tab)
VEM_TRIG_OP(OpCosD, cos_d_u10, , tab)
VEM_TRIG_OP(OpTanD, tan_d_u10)
VEM_TRIG_OP(OpSinDU35, sin_d_u35, , tab)
VEM_TRIG_OP(OpCosDU35, cos_d_u35, , tab)
VEM_TRIG_OP(OpTanDU35, tan_d_u35)
#undef VEM_TRIG_OP
// TINY: the result for a finite trivial x
#define VEM_TRIG_TINY(NAME, TINY)                                                         \
  __device__ __forceinline__ double NAME::trivial(double x) {                              \
    return ((uint32_t)__double2hiint(x) & 0x7fffffffu) >= 0x7ff00000u ? from_bits_d(kCanonNanD) : (TINY); \
  }                                                                                         \
  __device__ __forceinline__ double NAME::tiny(double x) { return (TINY); }
VEM_TRIG_TINY(OpSinD, x)
VEM_TRIG_TINY(OpCosD, 1.0)
VEM_TRIG_TINY(OpTanD, x)
VEM_TRIG_TINY(OpSinDU35, x)
VEM_TRIG_TINY(OpCosDU35, 1.0)
VEM_TRIG_TINY(OpTanDU35, x)
#undef VEM_TRIG_TINY
VEM_UNARY_OP(OpSinDPh, double, (sin_d_u10<kPh>(x, tab, tab + kPhDIStaged)))
VEM_UNARY_OP(OpCosDPh, double, (cos_d_u10<kPh>(x, tab, tab + kPhDIStaged)))
VEM_UNARY_OP(OpTanDPh, double, (tan_d_u10<kPh>(x, tab)))
VEM_UNARY_OP(OpAtanD, double, ((void)tab, atan_d_u10(x)))
VEM_UNARY_OP(OpAtanDU35, double, ((void)tab, atan_d_u35(x)))
VEM_UNARY_OP(OpAsinD, double, ((void)tab, asin_d_u10(x)))
VEM_UNARY_OP(OpAsinDU35, double, ((void)tab, asin_d_u35(x)))
VEM_UNARY_OP(OpAcosD, double, ((void)tab, acos_d_u10(x)))
VEM_UNARY_OP(OpAcosDU35, double, ((void)tab, acos_d_u35(x)))
VEM_UNARY_OP(OpAtanF, float, ((void)tab, canon_f((float)atan_d_u10((double)x))))
VEM_UNARY_OP(OpAtanFU35, float, ((void)tab, canon_f((float)atan_d_u35((double)x))))
VEM_UNARY_OP(OpAsinF, float, ((void)tab, canon_f((float)asin_d_u10((double)x))))
VEM_UNARY_OP(OpAsinFU35, float, ((void)tab, canon_f((float)asin_d_u35((double)x))))
VEM_UNARY_OP(OpAcosF, float, ((void)tab, canon_f((float)acos_d_u10((double)x))))
VEM_UNARY_OP(OpAcosFU35, float, ((void)tab, canon_f((float)acos_d_u35((double)x))))
// SLOW: value for a flagged element (x, r = fast result, code); `full()`
// is the out-of-line full function
#define VEM_SPLIT_UNARY_OP(NAME, T, EXPR, FAST, SLOW)                                    \
  struct NAME {                                                                          \
    __device__ __forceinline__ T operator()(T x, const double* tab) const { return EXPR; } \
    __device__ __forceinline__ T fast(T x, const double* tab, int& code) const { return FAST; } \
    __device__ __forceinline__ static T slow(T x, T r, int code, const double* tab) {    \
      (void)r;                                                                           \
      (void)code;                                                                        \
      auto full = [&]() { return full_op<NAME>(x, tab); };                               \
      return SLOW;                                                                       \
    }                                                                                    \
  };                                                                                     \
  template <> struct HasFast<NAME> { static constexpr bool value = true; };
VEM_SPLIT_UNARY_OP(OpExpD, double, ((void)tab, exp_d_u10(x)), ((void)tab, (exp_fast_d<VEM_EXP_D_N, true>(x, cExpD, code))),
                   exp_slow_d(x, full))
VEM_SPLIT_UNARY_OP(OpExpDU35, double, ((void)tab, exp_d_u35(x)),
                   ((void)tab, (exp_fast_d<VEM_EXP_D_U35_N, false>(x, cExpDU35, code))), exp_slow_d(x, full))
VEM_SPLIT_UNARY_OP(OpLogD, double, (log_core_d<true>(x, tab)), (log_fast_split_d<true>(x, tab, code)),
                   log_slow_d(x, full))
VEM_SPLIT_UNARY_OP(OpLogDU35, double, (log_core_d<false>(x, tab)), (log_fast_split_d<false>(x, tab, code)),
                   log_slow_d(x, full))
VEM_UNARY_OP(OpSinF, float, (sin_f_u10(x, tab)))
VEM_UNARY_OP(OpCosF, float, (cos_f_u10(x, tab)))
VEM_UNARY_OP(OpTanF, float, (tan_f_u10(x, tab)))
VEM_UNARY_OP(OpExpF, float, ((void)tab, exp_f_u10(x)))
VEM_UNARY_OP(OpExpFU35, float, ((void)tab, exp_f_u35(x)))
// f32 log / pow: the replicated table staging (kTableLogF)
VEM_SPLIT_UNARY_OP(OpLogF, float, (log_f_u10(x, tab)), (log_fast_f<VEM_LOG1P_F_N>(x, cLog1pF, tab, code)), full())
VEM_SPLIT_UNARY_OP(OpLogFU35, float, (log_f_u35(x, tab)),
                   (log_fast_f<VEM_LOG1P_F_U35_N>(x, cLog1pFU35, tab, code)), full())
#undef VEM_UNARY_OP
#undef VEM_SPLIT_UNARY_OP

#define VEM_BINARY_OP(NAME, T, EXPR)                                              \
  struct NAME {                                                                   \
    __device__ __forceinline__ T operator()(T x, T y, const double* tab) const { return EXPR; } \
  };
#define VEM_SPLIT_BINARY_OP(NAME, T, EXPR, FAST, SLOW)                                 \
  struct NAME {                                                                   \
    __device__ __forceinline__ T operator()(T x, T y, const double* tab) const { return EXPR; } \
    __device__ __forceinline__ T fast(T x, T y, const double* tab, int& code) const { return FAST; } \
    __device__ __forceinline__ static T slow(T x, T y, T r, int code, const double* tab) { \
      (void)r;                                                                    \
      (void)code;                                                                 \
      auto full = [&]() { return full_op<NAME>(x, y, tab); };                     \
      return SLOW;                                                                \
    }                                                                             \
  };                                                                              \
  template <> struct HasFast<NAME> { static constexpr bool value = true; };
VEM_SPLIT_BINARY_OP(OpPowD, double, pow_d_u10(x, y, tab), (pow_fast_d<VEM_LOG1P_D_N>(x, y, cLog1pD, tab, code)),
                    pow_slow_split_d(x, y, r, code, full))
VEM_SPLIT_BINARY_OP(OpPowDU35, double, pow_d_u35(x, y, tab),
                    (pow_fast_d<VEM_LOG1P_D_U35_N>(x, y, cLog1pDU35, tab, code)), pow_slow_split_d(x, y, r, code, full))
// fmod functors: operator() is the full function (unaligned pointers, tails);
// the step-class regrouping traits serve only the tuning build's variant 7
// (the shipped entry points use the tile work queue, FmodQ)
struct OpFmodD {
  __device__ __forceinline__ double operator()(double x, double y, const double* tab) const {
    (void)tab;
    return fmod_d(x, y);
  }
};
VEM_SPLIT_BINARY_OP(OpPowF, float, pow_f_u10(x, y, tab), (pow_fast_f<VEM_LOG1P_F_N>(x, y, cLog1pF, tab, code)),
                    full())
VEM_SPLIT_BINARY_OP(OpPowFU35, float, pow_f_u35(x, y, tab),
                    (pow_fast_f<VEM_LOG1P_F_U35_N>(x, y, cLog1pFU35, tab, code)), full())
struct OpFmodF {
  __device__ __forceinline__ float operator()(float x, float y, const double* tab) const {
    (void)tab;
    return fmod_f(x, y);
  }
};
VEM_BINARY_OP(OpAtan2D, double, ((void)tab, atan2_d_u10(x, y)))
VEM_BINARY_OP(OpAtan2DU35, double, ((void)tab, atan2_d_u35(x, y)))
VEM_BINARY_OP(OpFdimD, double, ((void)tab, fdim_d(x, y)))
VEM_BINARY_OP(OpAtan2F, float, ((void)tab, canon_f((float)atan2_d_u10((double)x, (double)y))))
VEM_BINARY_OP(OpAtan2FU35, float, ((void)tab, canon_f((float)atan2_d_u35((double)x, (double)y))))
VEM_BINARY_OP(OpFdimF, float, ((void)tab, fdim_f(x, y)))
#undef VEM_BINARY_OP
#undef VEM_SPLIT_BINARY_OP

// trivial classes (vem_math.cuh triv_*): exp, log, pow, atan (binary64)
struct TrivExpD {
  static constexpr bool value = true;
  __device__ __forceinline__ static bool maybe(double x) { return triv_exp_maybe(x); }
  __device__ __forceinline__ static bool exact(double x, double& r) { return triv_exp(x, r); }
};
struct TrivLogD {
  static constexpr bool value = true;
  __device__ __forceinline__ static bool maybe(double x) { return triv_log_maybe(x); }
  __device__ __forceinline__ static bool exact(double x, double& r) { return triv_log(x, r); }
};
struct TrivPowD {
  static constexpr bool value = true;
  __device__ __forceinline__ static bool maybe(double x, double y) { return triv_pow_maybe(x, y); }
  __device__ __forceinline__ static bool exact(double x, double y, double& r) { return triv_pow(x, y, r); }
};
struct TrivAtanD {
  static constexpr bool value = true;
  __device__ __forceinline__ static bool maybe(double x) { return triv_atan_maybe(x); }
  __device__ __forceinline__ static bool exact(double x, double& r) { return triv_atan(x, r); }
};
// Enabled where the full computation is expensive enough for the compaction
// to pay and the dense path does not lose (A/B, `profiles/r02_ab_triv/`:
// config 5 pow_d_u10 +17 %, atan +5-13 %, config 2 pow_d_u10 unchanged;
// exp -40 %, log -10 % on config 5 -- their fast paths are cheaper than the
// placement and rows -- and pow_d_u35 -3.5 % on config 2 (code layout of
// its dense path), so TrivExpD / TrivLogD stay unused and pow_d_u35 keeps
// the dense path only).
template <> struct Triv<OpPowD> : TrivPowD {};
template <> struct Triv<OpAtanD> : TrivAtanD {};
template <> struct Triv<OpAtanDU35> : TrivAtanD {};

// ------------------------------------------------------------- launching
// Per-device launch state.  The shared-memory opt-in
// (cudaFuncAttributeMaxDynamicSharedMemorySize) and the occupancy figure are
// properties of a kernel ON A DEVICE: they are cached per (instantiation,
// device) and (re)computed the first time a kernel is launched on each device,
// so one process can drive several GPUs (vem_run_sharded, multi-device torch
// programs).  Zero in the cache = not yet initialised on that device.
constexpr int kMaxDevices = 64;
using DevCache = std::atomic<int>[kMaxDevices];

static int current_device() {
  int d = 0;
  if (cudaGetDevice(&d) != cudaSuccess || d < 0) d = 0;
  return d;
}

template <class F>
static int per_device(DevCache& cache, int dev, F init) {
  if (dev >= kMaxDevices) return init();
  int v = cache[dev].load(std::memory_order_acquire);
  if (v == 0) {
    v = init();  // idempotent: two threads racing here compute the same value
    cache[dev].store(v, std::memory_order_release);
  }
  return v;
}

static int num_sms(int dev) {
  static DevCache cache;
  return per_device(cache, dev, [dev] {
    int v = 0;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v < 1) v = 148;
    return v;
  });
}

// resident CTAs per SM of `kernel` with `smem` dynamic bytes on the current
// device (applies the dynamic shared-memory opt-in there first)
template <class K>
static int occupancy(K kernel, int smem = 0) {
  // opt in whenever there is dynamic shared memory: static + dynamic may
  // exceed the 48 KB default even when the dynamic part alone does not
  if (smem > 0) cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  int b = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kernel, kThreads, smem) != cudaSuccess || b < 1) b = 1;
  return b;
}

// Persistent grid: min(work, SMs x resident CTAs per SM).
static int grid_for(int dev, int occ, size_t work_items, int per_thread) {
  size_t need = (work_items + (size_t)kThreads * per_thread - 1) / ((size_t)kThreads * per_thread);
  size_t cap = (size_t)num_sms(dev) * occ;
  size_t g = need < cap ? need : cap;
  return (int)(g < 1 ? 1 : g);
}

static inline bool aligned16(const void* p) { return ((uintptr_t)p & 15u) == 0; }

// Launch with programmatic stream serialization (see tma::griddep_wait): the
// kernel may start while the previous grid in the stream drains.  INVARIANT:
// every kernel launched through launch_pdl executes tma::griddep_wait()
// before its first global-memory access (k_stream, k_queue); only
// kernel-private set-up (mbarrier init, constant-table staging) may precede
// it.  Kernels without that wait (k_unary, k_binary, k_reduce_*) are
// launched with plain <<<>>>.
template <class K, class... Args>
static void launch_pdl(K kernel, int grid, int smem, cudaStream_t st, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = (size_t)smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kernel, args...);
}

template <class Op, class T, int TABLE, int U>
static int launch_unary(const T* x, T* y, size_t n, vem_stream_t s) {
  if (n == 0) return 0;
  cudaStream_t st = (cudaStream_t)s;
  if (aligned16(x) && aligned16(y)) {
    auto k = k_unary<Op, T, TABLE, U, true>;
    static DevCache occ;
    const int dev = current_device();
    int g = grid_for(dev, per_device(occ, dev, [k] { return occupancy(k); }), n / Vec16<T>::n + 1, U);
    k<<<g, kThreads, 0, st>>>(x, y, n);
  } else {
    auto k = k_unary<Op, T, TABLE, 1, false>;
    static DevCache occ;
    const int dev = current_device();
    int g = grid_for(dev, per_device(occ, dev, [k] { return occupancy(k); }), n, 1);
    k<<<g, kThreads, 0, st>>>(x, y, n);
  }
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return (int)cudaGetLastError();
}

template <class Op, class T, int TABLE, int U>
static int launch_binary(const T* x, const T* y2, T* out, size_t n, vem_stream_t s) {
  if (n == 0) return 0;
  cudaStream_t st = (cudaStream_t)s;
  if (aligned16(x) && aligned16(y2) && aligned16(out)) {
    auto k = k_binary<Op, T, TABLE, U, true>;
    static DevCache occ;
    const int dev = current_device();
    int g = grid_for(dev, per_device(occ, dev, [k] { return occupancy(k); }), n / Vec16<T>::n + 1, U);
    k<<<g, kThreads, 0, st>>>(x, y2, out, n);
  } else {
    auto k = k_binary<Op, T, TABLE, 1, false>;
    static DevCache occ;
    const int dev = current_device();
    int g = grid_for(dev, per_device(occ, dev, [k] { return occupancy(k); }), n, 1);
    k<<<g, kThreads, 0, st>>>(x, y2, out, n);
  }
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return (int)cudaGetLastError();
}

template <class Op, class T, int NIN, int TABLE, int VPT, int STAGES, int MINB = 1, bool WREL = false>
static int launch_stream(const T* a, const T* b, T* out, size_t n, vem_stream_t s) {
  if (n == 0) return 0;
  if (!(aligned16(a) && aligned16(out) && (NIN == 1 || aligned16(b)))) {
    if constexpr (NIN == 2) return launch_binary<Op, T, TABLE, 1>(a, b, out, n, s);
    else return launch_unary<Op, T, TABLE, 1>(a, out, n, s);
  }
  auto k = k_stream<Op, T, NIN, TABLE, VPT, STAGES, MINB, WREL>;
  constexpr int smem = STAGES * NIN * kThreads * VPT * 16;
  static DevCache occ_cache;
  const int dev = current_device();
  const int occ = per_device(occ_cache, dev, [k] { return occupancy(k, smem); });
  constexpr size_t tile_e = (size_t)kThreads * VPT * Vec16<T>::n;
  size_t tiles = n / tile_e;
  size_t cap = (size_t)num_sms(dev) * occ;
  size_t g = tiles < cap ? tiles : cap;
  if (g < 1) g = 1;
  launch_pdl(k, (int)g, smem, (cudaStream_t)s, a, b, out, n);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return (int)cudaGetLastError();
}

template <class Op, int TABLE, int VPT, int STAGES, int MINB>
static int launch_trig(const double* a, const double*, double* out, size_t n, vem_stream_t s) {
  if (n == 0) return 0;
  if (!(aligned16(a) && aligned16(out))) return launch_unary<Op, double, TABLE, 1>(a, out, n, s);
  auto k = k_trig<Op, TABLE, VPT, STAGES, MINB>;
  constexpr int smem = STAGES * kThreads * VPT * 16;
  static DevCache occ_cache;
  const int dev = current_device();
  const int occ = per_device(occ_cache, dev, [k] { return occupancy(k, smem); });
  constexpr size_t tile_e = (size_t)kThreads * VPT * 2;
  size_t tiles = n / tile_e;
  size_t cap = (size_t)num_sms(dev) * occ;
  size_t g = tiles < cap ? tiles : cap;
  if (g < 1) g = 1;
  launch_pdl(k, (int)g, smem, (cudaStream_t)s, a, out, n);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return (int)cudaGetLastError();
}

template <class Q, class Op, class T, int NIN, int TABLE, int VPT, int STAGES, int MINB = 1, int ROWS = 1,
          int FETCH = 1>
static int launch_queue(const T* a, const T* b, T* out, size_t n, vem_stream_t s) {
  if (n == 0) return 0;
  if (!(aligned16(a) && aligned16(out) && (NIN == 1 || aligned16(b)))) {
    if constexpr (NIN == 2) return launch_binary<Op, T, TABLE, 1>(a, b, out, n, s);
    else return launch_unary<Op, T, TABLE, 1>(a, out, n, s);
  }
  auto k = k_queue<Q, T, NIN, TABLE, VPT, STAGES, MINB, ROWS, FETCH>;
  constexpr int smem = STAGES * NIN * kThreads * VPT * 16;
  static DevCache occ_cache;
  const int dev = current_device();
  const int occ = per_device(occ_cache, dev, [k] { return occupancy(k, smem); });
  constexpr size_t tile_e = (size_t)kThreads * VPT * Vec16<T>::n;
  size_t tiles = n / tile_e;
  size_t cap = (size_t)num_sms(dev) * occ;
  size_t g = tiles < cap ? tiles : cap;
  if (g < 1) g = 1;
  launch_pdl(k, (int)g, smem, (cudaStream_t)s, a, b, out, n);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return (int)cudaGetLastError();
}
#ifdef VEM_TUNE  // tuning-only launchers (tools/tune.py)
template <class T, int VPT, int STAGES, int MINB = 1>
static int launch_fmod_w(const T* a, const T* b, T* out, size_t n, vem_stream_t s) {
  using OpF = typename std::conditional<sizeof(T) == 8, OpFmodD, OpFmodF>::type;
  if (n == 0) return 0;
  if (!(aligned16(a) && aligned16(out) && aligned16(b))) return launch_binary<OpF, T, kNoTable, 1>(a, b, out, n, s);
  auto k = k_wqueue<FmodQ<T>, T, 2, VPT, STAGES, MINB>;
  constexpr int smem = (kThreads / 32) * STAGES * 2 * 32 * VPT * 16;
  static DevCache occ_cache;
  const int dev = current_device();
  const int occ = per_device(occ_cache, dev, [k] { return occupancy(k, smem); });
  constexpr size_t ch_e = (size_t)32 * VPT * Vec16<T>::n;
  size_t warps = n / ch_e;
  size_t cap = (size_t)num_sms(dev) * occ * (kThreads / 32);
  size_t w = warps < cap ? warps : cap;
  size_t g = (w + kThreads / 32 - 1) / (kThreads / 32);
  if (g < 1) g = 1;
  launch_pdl(k, (int)g, smem, (cudaStream_t)s, a, b, out, n);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return (int)cudaGetLastError();
}
#endif  // VEM_TUNE
template <class T, int VPT, int STAGES, int MINB = 1, int ROWS = 1, int FETCH = 1>
static int launch_fmod_q(const T* a, const T* b, T* out, size_t n, vem_stream_t s) {
  using OpF = typename std::conditional<sizeof(T) == 8, OpFmodD, OpFmodF>::type;
  return launch_queue<FmodQ<T>, OpF, T, 2, kNoTable, VPT, STAGES, MINB, ROWS, FETCH>(a, b, out, n, s);
}

// fmodf as one straight-line streaming body (fmod_f_flat; no work queue)
struct OpFmodFFlat {
  __device__ __forceinline__ float operator()(float x, float y, const double* tab) const {
    (void)tab;
    return fmod_f_flat(x, y);
  }
};
// (A trivial class for fmodf -- everything but |x| > |y| > 0, half of config
// 4's pairs -- through the carry-over stack measured slower, 260 -> 238
// Gelem/s: with half of the elements non-trivial, their scattered 4-byte
// stores cost more than the skipped work; the stack pays for shares of a few
// per cent, as pow's and atan's on config 5.)
#ifdef VEM_TUNE
struct OpFmodFFixed {
  __device__ __forceinline__ float operator()(float x, float y, const double* tab) const {
    (void)tab;
    return fmod_f_fixed(x, y);
  }
};
template <class T, int VPT, int STAGES, int MINB = 1>
static int launch_fmod_fixed(const T* a, const T* b, T* out, size_t n, vem_stream_t s) {
  if constexpr (sizeof(T) == 4) return launch_stream<OpFmodFFixed, float, 2, kNoTable, VPT, STAGES, MINB>(a, b, out, n, s);
  else return launch_fmod_q<double, 2, 2, 1, 1>(a, b, out, n, s);
}
#endif  // VEM_TUNE
template <class T, int VPT, int STAGES, int MINB = 1>
static int launch_fmod_flat(const T* a, const T* b, T* out, size_t n, vem_stream_t s) {
  if constexpr (sizeof(T) == 4) return launch_stream<OpFmodFFlat, float, 2, kNoTable, VPT, STAGES, MINB>(a, b, out, n, s);
  else return launch_fmod_q<double, 2, 2, 1, 1>(a, b, out, n, s);
}

#ifdef VEM_TUNE
template <class T, int MINB = 1>
static int launch_fmod(const T* a, const T* b, T* out, size_t n, vem_stream_t s) {
  if (n == 0) return 0;
  if (!(aligned16(a) && aligned16(b))) {
    if constexpr (sizeof(T) == 8) return launch_binary<OpFmodD, T, kNoTable, 1>(a, b, out, n, s);
    else return launch_binary<OpFmodF, T, kNoTable, 1>(a, b, out, n, s);
  }
  auto k = k_fmod<T, MINB>;
  static DevCache occ_cache;
  const int dev = current_device();
  const int occ = per_device(occ_cache, dev, [k] {
    int bpm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bpm, k, kFmodWarps * 32, 0) != cudaSuccess || bpm < 1)
      bpm = 1;
    return bpm;
  });
  size_t chunks = (n + kFmodChunk - 1) / kFmodChunk;
  size_t warps_cap = (size_t)num_sms(dev) * occ * kFmodWarps;
  size_t warps = chunks < warps_cap ? chunks : warps_cap;
  size_t g = (warps + kFmodWarps - 1) / kFmodWarps;
  k<<<(int)(g < 1 ? 1 : g), kFmodWarps * 32, 0, (cudaStream_t)s>>>(a, b, out, n);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return (int)cudaGetLastError();
}

#endif  // VEM_TUNE

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
  static DevCache occ;
  const int dev = current_device();
  int g = grid_for(dev, per_device(occ, dev, [k] { return occupancy(k); }), n, 1);
  k<<<g, kThreads, 0, (cudaStream_t)s>>>(x, hi, lo, q, n);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return (int)cudaGetLastError();
}

static const double kHostPhD[4 * VEM_PH_D_ENTRIES] = {VEM_PH_D_INIT};

}  // namespace vem

using namespace vem;

// Launch-shape tuning build (-DVEM_TUNE, tools/tune.py): every streaming entry
// point can be switched at run time between (VPT, STAGES) variants.
#ifdef VEM_TUNE
static int g_tune = -1;
extern "C" void vem_tune_set(int v) { g_tune = v; }
template <class Op, class T, int NIN, int TAB, int VPT, int ST, int MINB = 1, bool WREL = false>
static int launch_tuned(const T* a, const T* b, T* o, size_t n, vem_stream_t s) {
  switch (g_tune) {
    case 11: return launch_stream<Op, T, NIN, TAB, VPT, ST, MINB, !WREL>(a, b, o, n, s);
    case 12: return launch_stream<Op, T, NIN, TAB, VPT, ST + 1, MINB, WREL>(a, b, o, n, s);
    case 13: return launch_stream<Op, T, NIN, TAB, VPT, ST + 1, MINB, !WREL>(a, b, o, n, s);
    case 14: return launch_stream<Op, T, NIN, TAB, VPT, ST + 2, MINB, WREL>(a, b, o, n, s);
    case 0: return launch_stream<Op, T, NIN, TAB, 1, 2>(a, b, o, n, s);
    case 1: return launch_stream<Op, T, NIN, TAB, 1, 4>(a, b, o, n, s);
    case 2: return launch_stream<Op, T, NIN, TAB, 2, 2>(a, b, o, n, s);
    case 3: return launch_stream<Op, T, NIN, TAB, 2, 3>(a, b, o, n, s);
    case 4: return launch_stream<Op, T, NIN, TAB, 2, 4>(a, b, o, n, s);
    case 5: return launch_stream<Op, T, NIN, TAB, 4, 2>(a, b, o, n, s);
    case 6: return launch_stream<Op, T, NIN, TAB, VPT, ST, 2>(a, b, o, n, s);
    case 7: return launch_stream<Op, T, NIN, TAB, VPT, ST, 3>(a, b, o, n, s);
    case 8: return launch_stream<Op, T, NIN, TAB, VPT, ST, 4>(a, b, o, n, s);
    case 9: return launch_stream<Op, T, NIN, TAB, 4, 2, 2>(a, b, o, n, s);
    case 10: return launch_stream<Op, T, NIN, TAB, 4, 2, 3>(a, b, o, n, s);
    case 15: return launch_stream<Op, T, NIN, TAB, 2, 2, 3>(a, b, o, n, s);
    case 16: return launch_stream<Op, T, NIN, TAB, 2, 2, 4>(a, b, o, n, s);
    case 17: return launch_stream<Op, T, NIN, TAB, 2, 3, 4>(a, b, o, n, s);
    case 18: return launch_stream<Op, T, NIN, TAB, 1, 2, 6>(a, b, o, n, s);
    case 19: return launch_stream<Op, T, NIN, TAB, 1, 4, 6>(a, b, o, n, s);
    case 20: return launch_stream<Op, T, NIN, TAB, 2, 2, 5>(a, b, o, n, s);
    default: return launch_stream<Op, T, NIN, TAB, VPT, ST, MINB, WREL>(a, b, o, n, s);
  }
}
// fmod without regrouping or queue (every lane loops to its warp's largest
// step count): comparison only
template <class T>
struct OpFmodPlain {
  __device__ __forceinline__ T operator()(T x, T y, const double* tab) const {
    (void)tab;
    if constexpr (sizeof(T) == 8) return fmod_d(x, y);
    else return fmod_f(x, y);
  }
};
template <class Op, int TAB, int VPT, int ST, int MINB>
static int launch_trig_tuned(const double* a, const double* b, double* o, size_t n, vem_stream_t s) {
  switch (g_tune) {
    case 30: return launch_trig<Op, TAB, 4, 3, 3>(a, b, o, n, s);
    case 31: return launch_trig<Op, TAB, 4, 3, 2>(a, b, o, n, s);
    case 32: return launch_trig<Op, TAB, 2, 3, 3>(a, b, o, n, s);
    case 33: return launch_trig<Op, TAB, 2, 4, 3>(a, b, o, n, s);
    case 34: return launch_trig<Op, TAB, 4, 2, 2>(a, b, o, n, s);
    case 35: return launch_trig<Op, TAB, 2, 2, 4>(a, b, o, n, s);
    case 36: return launch_trig<Op, TAB, 4, 4, 2>(a, b, o, n, s);
    default: return launch_trig<Op, TAB, VPT, ST, MINB>(a, b, o, n, s);
  }
}
#define VEM_STREAM launch_tuned
#define VEM_TRIG launch_trig_tuned
template <class T>
static int launch_fmod_tuned(const T* a, const T* b, T* o, size_t n, vem_stream_t s) {
  using OpF = typename std::conditional<sizeof(T) == 8, OpFmodD, OpFmodF>::type;
  switch (g_tune) {
    case 0: return launch_fmod_w<T, 2, 2>(a, b, o, n, s);
    case 1: return launch_fmod_w<T, 4, 2>(a, b, o, n, s);
    case 2: return launch_fmod_w<T, 2, 3>(a, b, o, n, s);
    case 3: return launch_fmod_w<T, 4, 2, 2>(a, b, o, n, s);
    case 4: return launch_fmod_w<T, 2, 2, 3>(a, b, o, n, s);
    case 5: return launch_fmod_q<T, 2, 2, 1, 2>(a, b, o, n, s);
    case 6: return launch_fmod_q<T, 4, 2, 1, 1>(a, b, o, n, s);
    case 9: return launch_stream<OpFmodPlain<T>, T, 2, kNoTable, 2, 2>(a, b, o, n, s);
    case 10: return launch_stream<OpFmodPlain<T>, T, 2, kNoTable, 1, 2>(a, b, o, n, s);
    case 11: return launch_fmod_q<T, 2, 2, 1, 1, 2>(a, b, o, n, s);
    case 12: return launch_fmod_q<T, 2, 2, 1, 1, 4>(a, b, o, n, s);
    case 13: return launch_fmod_q<T, 2, 2, 2, 1, 2>(a, b, o, n, s);
    case 14: return launch_fmod_flat<T, 2, 2>(a, b, o, n, s);
    case 15: return launch_fmod_flat<T, 4, 2>(a, b, o, n, s);
    case 16: return launch_fmod_flat<T, 1, 2>(a, b, o, n, s);
    case 17: return launch_fmod_flat<T, 2, 2, 4>(a, b, o, n, s);
    case 18: return launch_fmod_flat<T, 4, 2, 3>(a, b, o, n, s);
    case 19: return launch_fmod_fixed<T, 2, 2>(a, b, o, n, s);
    case 20: return launch_fmod_fixed<T, 1, 2>(a, b, o, n, s);
    case 21: return launch_fmod_fixed<T, 2, 2, 2>(a, b, o, n, s);
    case 22: return launch_fmod_fixed<T, 1, 4>(a, b, o, n, s);
    case 8: return launch_fmod<T>(a, b, o, n, s);
    case 23: return launch_fmod_q<T, 4, 2, 1, 2>(a, b, o, n, s);
    case 24: return launch_fmod_q<T, 2, 3, 1, 2>(a, b, o, n, s);
    case 25: return launch_fmod_q<T, 2, 2, 2, 2>(a, b, o, n, s);
    case 26: return launch_fmod_q<T, 4, 2, 1, 1>(a, b, o, n, s);
    case 27: return launch_fmod_q<T, 2, 2, 1, 1, 0>(a, b, o, n, s);
    case 28: return launch_fmod_q<T, 2, 2, 1, 2, 0>(a, b, o, n, s);
    default: return launch_fmod_q<T, 2, 2, 1, 1>(a, b, o, n, s);
  }
}
#define VEM_FMOD launch_fmod_tuned
#else
#define VEM_STREAM launch_stream
#define VEM_TRIG launch_trig
#define VEM_FMOD launch_fmod
#endif

// Elements per thread in flight (16-byte vectors): HBM-bound kernels keep 4
// vectors in flight, FP64-pipe-bound ones 2 (register pressure).
extern "C" {

int vem_sin_d_u10(const double* x, double* y, size_t n, vem_stream_t s) { return VEM_TRIG<OpSinD, kTableDG, 4, 2, 3>(x, nullptr, y, n, s); }
int vem_cos_d_u10(const double* x, double* y, size_t n, vem_stream_t s) { return VEM_TRIG<OpCosD, kTableDG, 4, 2, 3>(x, nullptr, y, n, s); }
int vem_tan_d_u10(const double* x, double* y, size_t n, vem_stream_t s) { return VEM_TRIG<OpTanD, kTableDG, 4, 2, 3>(x, nullptr, y, n, s); }
int vem_sin_d_u10_ph(const double* x, double* y, size_t n, vem_stream_t s) { return VEM_STREAM<OpSinDPh, double, 1, kTableDI, 4, 2, 2>(x, nullptr, y, n, s); }
int vem_cos_d_u10_ph(const double* x, double* y, size_t n, vem_stream_t s) { return VEM_STREAM<OpCosDPh, double, 1, kTableDI, 4, 2, 2>(x, nullptr, y, n, s); }
int vem_tan_d_u10_ph(const double* x, double* y, size_t n, vem_stream_t s) { return VEM_STREAM<OpTanDPh, double, 1, kTableDI, 4, 2, 2>(x, nullptr, y, n, s); }
int vem_atan_d_u10(const double* x, double* y, size_t n, vem_stream_t s) { return VEM_STREAM<OpAtanD, double, 1, kNoTable, 2, 2>(x, nullptr, y, n, s); }
int vem_exp_d_u10(const double* x, double* y, size_t n, vem_stream_t s) { return VEM_STREAM<OpExpD, double, 1, kNoTable, 2, 2, 3>(x, nullptr, y, n, s); }
int vem_exp_d_u35(const double* x, double* y, size_t n, vem_stream_t s) { return VEM_STREAM<OpExpDU35, double, 1, kNoTable, 4, 2>(x, nullptr, y, n, s); }
int vem_log_d_u10(const double* x, double* y, size_t n, vem_stream_t s) { return VEM_STREAM<OpLogD, double, 1, kTableLog, 4, 2, 3, true>(x, nullptr, y, n, s); }
int vem_log_d_u35(const double* x, double* y, size_t n, vem_stream_t s) { return VEM_STREAM<OpLogDU35, double, 1, kTableLog, 2, 2, 4>(x, nullptr, y, n, s); }
int vem_pow_d_u10(const double* x, const double* y2, double* o, size_t n, vem_stream_t s) { return VEM_STREAM<OpPowD, double, 2, kTableLog, 2, 2, 3, true>(x, y2, o, n, s); }
int vem_pow_d_u35(const double* x, const double* y2, double* o, size_t n, vem_stream_t s) { return VEM_STREAM<OpPowDU35, double, 2, kTableLog, 2, 2, 3, true>(x, y2, o, n, s); }
int vem_fmod_d(const double* x, const double* y2, double* o, size_t n, vem_stream_t s) {
#ifdef VEM_TUNE
  return VEM_FMOD<double>(x, y2, o, n, s);
#else
  return launch_fmod_q<double, 2, 2, 1, 2, 0>(x, y2, o, n, s);  // two rows per lane, static snake schedule
#endif
}

int vem_sin_f_u10(const float* x, float* y, size_t n, vem_stream_t s) { return VEM_STREAM<OpSinF, float, 1, kTableF, 4, 2>(x, nullptr, y, n, s); }
int vem_cos_f_u10(const float* x, float* y, size_t n, vem_stream_t s) { return VEM_STREAM<OpCosF, float, 1, kTableF, 4, 2>(x, nullptr, y, n, s); }
int vem_tan_f_u10(const float* x, float* y, size_t n, vem_stream_t s) { return VEM_STREAM<OpTanF, float, 1, kTableF, 4, 2, 2>(x, nullptr, y, n, s); }
// every f32 trig lane takes the f32 Payne-Hanek path: the forced variants are the same kernels
int vem_sin_f_u10_ph(const float* x, float* y, size_t n, vem_stream_t s) { return vem_sin_f_u10(x, y, n, s); }
int vem_cos_f_u10_ph(const float* x, float* y, size_t n, vem_stream_t s) { return vem_cos_f_u10(x, y, n, s); }
int vem_tan_f_u10_ph(const float* x, float* y, size_t n, vem_stream_t s) { return vem_tan_f_u10(x, y, n, s); }
int vem_exp_f_u10(const float* x, float* y, size_t n, vem_stream_t s) { return VEM_STREAM<OpExpF, float, 1, kNoTable, 2, 2, 3>(x, nullptr, y, n, s); }
int vem_exp_f_u35(const float* x, float* y, size_t n, vem_stream_t s) { return VEM_STREAM<OpExpFU35, float, 1, kNoTable, 2, 2, 3>(x, nullptr, y, n, s); }
int vem_log_f_u10(const float* x, float* y, size_t n, vem_stream_t s) { return VEM_STREAM<OpLogF, float, 1, kTableLogF, 2, 2>(x, nullptr, y, n, s); }
int vem_log_f_u35(const float* x, float* y, size_t n, vem_stream_t s) { return VEM_STREAM<OpLogFU35, float, 1, kTableLogF, 2, 2>(x, nullptr, y, n, s); }
int vem_pow_f_u10(const float* x, const float* y2, float* o, size_t n, vem_stream_t s) { return VEM_STREAM<OpPowF, float, 2, kTableLogF, 2, 4>(x, y2, o, n, s); }
int vem_pow_f_u35(const float* x, const float* y2, float* o, size_t n, vem_stream_t s) { return VEM_STREAM<OpPowFU35, float, 2, kTableLogF, 2, 4>(x, y2, o, n, s); }
int vem_fmod_f(const float* x, const float* y2, float* o, size_t n, vem_stream_t s) {
#ifdef VEM_TUNE
  return VEM_FMOD<float>(x, y2, o, n, s);
#else
  return launch_fmod_flat<float, 2, 2>(x, y2, o, n, s);
#endif
}

// ---- SURVEY.md §8(f).1 additions
int vem_sin_d_u35(const double* x, double* y, size_t n, vem_stream_t s) { return VEM_TRIG<OpSinDU35, kTableDG35, 4, 2, 3>(x, nullptr, y, n, s); }
int vem_cos_d_u35(const double* x, double* y, size_t n, vem_stream_t s) { return VEM_TRIG<OpCosDU35, kTableDG35, 4, 2, 3>(x, nullptr, y, n, s); }
int vem_tan_d_u35(const double* x, double* y, size_t n, vem_stream_t s) { return VEM_TRIG<OpTanDU35, kTableDG35, 4, 2, 3>(x, nullptr, y, n, s); }
int vem_atan_d_u35(const double* x, double* y, size_t n, vem_stream_t s) { return VEM_STREAM<OpAtanDU35, double, 1, kNoTable, 2, 2>(x, nullptr, y, n, s); }
int vem_asin_d_u10(const double* x, double* y, size_t n, vem_stream_t s) { return VEM_STREAM<OpAsinD, double, 1, kNoTable, 2, 2>(x, nullptr, y, n, s); }
int vem_asin_d_u35(const double* x, double* y, size_t n, vem_stream_t s) { return VEM_STREAM<OpAsinDU35, double, 1, kNoTable, 2, 2>(x, nullptr, y, n, s); }
int vem_acos_d_u10(const double* x, double* y, size_t n, vem_stream_t s) { return VEM_STREAM<OpAcosD, double, 1, kNoTable, 2, 2>(x, nullptr, y, n, s); }
int vem_acos_d_u35(const double* x, double* y, size_t n, vem_stream_t s) { return VEM_STREAM<OpAcosDU35, double, 1, kNoTable, 2, 2>(x, nullptr, y, n, s); }
int vem_atan2_d_u10(const double* y, const double* x, double* o, size_t n, vem_stream_t s) { return VEM_STREAM<OpAtan2D, double, 2, kNoTable, 2, 2>(y, x, o, n, s); }
int vem_atan2_d_u35(const double* y, const double* x, double* o, size_t n, vem_stream_t s) { return VEM_STREAM<OpAtan2DU35, double, 2, kNoTable, 2, 2>(y, x, o, n, s); }
int vem_fdim_d(const double* x, const double* y2, double* o, size_t n, vem_stream_t s) { return VEM_STREAM<OpFdimD, double, 2, kNoTable, 4, 2>(x, y2, o, n, s); }
int vem_sin_f_u35(const float* x, float* y, size_t n, vem_stream_t s) { return vem_sin_f_u10(x, y, n, s); }
int vem_cos_f_u35(const float* x, float* y, size_t n, vem_stream_t s) { return vem_cos_f_u10(x, y, n, s); }
int vem_tan_f_u35(const float* x, float* y, size_t n, vem_stream_t s) { return vem_tan_f_u10(x, y, n, s); }
int vem_atan_f_u10(const float* x, float* y, size_t n, vem_stream_t s) { return VEM_STREAM<OpAtanF, float, 1, kNoTable, 2, 2>(x, nullptr, y, n, s); }
int vem_atan_f_u35(const float* x, float* y, size_t n, vem_stream_t s) { return VEM_STREAM<OpAtanFU35, float, 1, kNoTable, 2, 2>(x, nullptr, y, n, s); }
int vem_asin_f_u10(const float* x, float* y, size_t n, vem_stream_t s) { return VEM_STREAM<OpAsinF, float, 1, kNoTable, 1, 2>(x, nullptr, y, n, s); }
int vem_asin_f_u35(const float* x, float* y, size_t n, vem_stream_t s) { return VEM_STREAM<OpAsinFU35, float, 1, kNoTable, 2, 2>(x, nullptr, y, n, s); }
int vem_acos_f_u10(const float* x, float* y, size_t n, vem_stream_t s) { return VEM_STREAM<OpAcosF, float, 1, kNoTable, 1, 2>(x, nullptr, y, n, s); }
int vem_acos_f_u35(const float* x, float* y, size_t n, vem_stream_t s) { return VEM_STREAM<OpAcosFU35, float, 1, kNoTable, 2, 2>(x, nullptr, y, n, s); }
int vem_atan2_f_u10(const float* y, const float* x, float* o, size_t n, vem_stream_t s) { return VEM_STREAM<OpAtan2F, float, 2, kNoTable, 2, 2>(y, x, o, n, s); }
int vem_atan2_f_u35(const float* y, const float* x, float* o, size_t n, vem_stream_t s) { return VEM_STREAM<OpAtan2FU35, float, 2, kNoTable, 2, 2>(y, x, o, n, s); }
int vem_fdim_f(const float* x, const float* y2, float* o, size_t n, vem_stream_t s) { return VEM_STREAM<OpFdimF, float, 2, kNoTable, 4, 2>(x, y2, o, n, s); }

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
  static DevCache occ;
  const int dev = current_device();
  int g = grid_for(dev, per_device(occ, dev, [] { return occupancy(k_reduce_f); }), n, 1);
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
