// Device twins of the config-input generator and the chunk checksums
// (bench + test infrastructure; see vem_aux.h).  Compiled with --fmad=false
// like the math kernels: the generator's arithmetic must be the exact IEEE
// sequence inputs.py and oracle/vem_gen_host.c perform (mul then add, each
// rounded), so the three produce identical bits.
#include <cuda_runtime.h>

#include <cstdint>

#include "vem_aux.h"

namespace {

constexpr uint64_t kGolden = 0x9E3779B97F4A7C15ull;

__device__ __forceinline__ uint64_t fmix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
// SplitMix64 output #(i+1) of the stream `seed` (inputs.splitmix64)
__device__ __forceinline__ uint64_t sm64(uint64_t seed, uint64_t i) { return fmix64(seed + (i + 1) * kGolden); }
__device__ __forceinline__ double unit(uint64_t seed, uint64_t i) {
  return __dmul_rn((double)(sm64(seed, i) >> 11), 0x1p-53);
}

// (ln 2)^k / k!, k = 0..13 (inputs.EXP2_C)
__constant__ double kExp2C[14] = {0x1.0000000000000p+0,  0x1.62e42fefa39efp-1,  0x1.ebfbdff82c58fp-3,
                                  0x1.c6b08d704a0c0p-5,  0x1.3b2ab6fba4e77p-7,  0x1.5d87fe78a6731p-10,
                                  0x1.430912f86c787p-13, 0x1.ffcbfc588b0c7p-17, 0x1.62c0223a5c824p-20,
                                  0x1.b5253d395e7c4p-24, 0x1.e4cf5158b8ecap-28, 0x1.e8cac7351bb25p-32,
                                  0x1.c3bd650fc2986p-36, 0x1.816193166d0f9p-40};

__device__ __forceinline__ double exp2_repro(double L) {
  const double k = floor(L);
  const double f = __dsub_rn(L, k);  // exact
  double p = kExp2C[13];
#pragma unroll
  for (int j = 12; j >= 0; j--) p = __dadd_rn(__dmul_rn(p, f), kExp2C[j]);
  // p * 2^k, exact for normal results (the recipes keep k in [-1022, 1023])
  return __dmul_rn(p, __longlong_as_double((long long)((int)k + 1023) << 52));
}

__device__ double element(const vem_recipe r, uint64_t i) {
  const double u = unit(r.seed, i);
  double v = __dadd_rn(r.a, __dmul_rn(__dsub_rn(r.b, r.a), u));
  if (r.kind == 1) {
    v = exp2_repro(v);
    if (r.f32) v = fmin(fmax(v, 0x1p-126), 0x1.fffffep+127);
  }
  if (r.sign && (sm64(r.seed ^ 0x5151ull, i) >> 63)) v = -v;
  if (r.specials) {
    const uint64_t ss = r.spec_seed;
    if (unit(ss ^ 0xC0FFEEull, i) < 0.01) {
      const int which = (int)(sm64(ss ^ 0xBEEFull, i) % 9ull);
      const double sp[9] = {0.0, -0.0, __longlong_as_double(0x7ff0000000000000ll),
                            __longlong_as_double((long long)0xfff0000000000000ull),
                            __longlong_as_double(0x7ff8000000000000ll), __longlong_as_double(1ll), 0.0,
                            __longlong_as_double(0x7fefffffffffffffll),
                            __longlong_as_double((long long)0xffefffffffffffffull)};
      v = which == 6 ? __longlong_as_double(
                           (long long)((sm64(ss ^ 0xD00Dull, i) & ((1ull << 52) - 1)) | 1ull))
                     : sp[which];
    }
  }
  return v;
}

__global__ void k_fill(const vem_recipe r, void* out, size_t n, uint64_t offset) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t j = (size_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += stride) {
    const double v = element(r, offset + j);
    if (r.f32) static_cast<float*>(out)[j] = __double2float_rn(v);
    else static_cast<double*>(out)[j] = v;
  }
}

// one launch per chunk segment: every block adds its partial sum into *sum
template <int EB>
__global__ void k_checksum(const void* p, size_t n, uint64_t offset, unsigned long long* sum) {
  uint64_t acc = 0;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t j = (size_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += stride) {
    const uint64_t b = EB == 8 ? (uint64_t)__ldg(static_cast<const unsigned long long*>(p) + j)
                               : (uint64_t)__ldg(static_cast<const unsigned int*>(p) + j);
    acc += fmix64(b ^ ((offset + j) * kGolden));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  __shared__ uint64_t part[32];
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint64_t t = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); w++) t += part[w];
    atomicAdd(sum, (unsigned long long)t);
  }
}

int grid_of(size_t n) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  size_t g = (n + 255) / 256;
  const size_t cap = (size_t)sms * 8;
  return (int)(g < 1 ? 1 : (g < cap ? g : cap));
}

}  // namespace

extern "C" int vem_aux_fill(const vem_recipe* r, void* out, size_t n, uint64_t offset, void* stream) {
  if (!r || (!out && n)) return (int)cudaErrorInvalidValue;
  if (n == 0) return 0;
  k_fill<<<grid_of(n), 256, 0, (cudaStream_t)stream>>>(*r, out, n, offset);
  return (int)cudaGetLastError();
}

extern "C" int vem_aux_checksum(const void* p, size_t n, int elem_bytes, uint64_t offset, int log2chunk,
                                unsigned long long* sums, void* stream) {
  if ((elem_bytes != 4 && elem_bytes != 8) || log2chunk < 0 || log2chunk > 40) return (int)cudaErrorInvalidValue;
  const uint64_t c0 = offset >> log2chunk;
  size_t j = 0;
  while (j < n) {
    const uint64_t g = offset + j;
    const uint64_t c = g >> log2chunk;
    const uint64_t end = (c + 1) << log2chunk;
    const size_t m = (size_t)((end - g) < (n - j) ? (end - g) : (n - j));
    const void* q = static_cast<const char*>(p) + j * (size_t)elem_bytes;
    if (elem_bytes == 8)
      k_checksum<8><<<grid_of(m), 256, 0, (cudaStream_t)stream>>>(q, m, g, sums + (c - c0));
    else
      k_checksum<4><<<grid_of(m), 256, 0, (cudaStream_t)stream>>>(q, m, g, sums + (c - c0));
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return (int)e;
    j += m;
  }
  return 0;
}
