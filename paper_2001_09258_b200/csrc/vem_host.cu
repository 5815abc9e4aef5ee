// Host-side multi-GPU driver above the per-device C ABI (SURVEY.md §3 S5,
// §8(e)): contiguous shards [g*N/G, (g+1)*N/G) of every operand, one host
// thread per device with its own stream and events, no collective on the data
// path.  The host-array entry point for a C++ caller that owns several GPUs
// in one process (tests/cpp/host_abi_test.cpp); bench.py's multi-GPU path is
// one process per GPU under torchrun instead and calls the per-device ABI.
#include <cuda_runtime.h>

#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "../../include/vem.h"

namespace {

typedef int (*unary_d)(const double*, double*, size_t, vem_stream_t);
typedef int (*unary_f)(const float*, float*, size_t, vem_stream_t);
typedef int (*binary_d)(const double*, const double*, double*, size_t, vem_stream_t);
typedef int (*binary_f)(const float*, const float*, float*, size_t, vem_stream_t);

struct Entry {
  const char* name;
  int elem;    // bytes per element
  int binary;  // 1 = two inputs
  void* fn;
};

const Entry kTable[] = {
    {"sin_d_u10", 8, 0, (void*)vem_sin_d_u10},       {"cos_d_u10", 8, 0, (void*)vem_cos_d_u10},
    {"tan_d_u10", 8, 0, (void*)vem_tan_d_u10},       {"sin_d_u10_ph", 8, 0, (void*)vem_sin_d_u10_ph},
    {"cos_d_u10_ph", 8, 0, (void*)vem_cos_d_u10_ph}, {"tan_d_u10_ph", 8, 0, (void*)vem_tan_d_u10_ph},
    {"atan_d_u10", 8, 0, (void*)vem_atan_d_u10},     {"exp_d_u10", 8, 0, (void*)vem_exp_d_u10},
    {"exp_d_u35", 8, 0, (void*)vem_exp_d_u35},       {"log_d_u10", 8, 0, (void*)vem_log_d_u10},
    {"log_d_u35", 8, 0, (void*)vem_log_d_u35},       {"pow_d_u10", 8, 1, (void*)vem_pow_d_u10},
    {"pow_d_u35", 8, 1, (void*)vem_pow_d_u35},       {"fmod_d", 8, 1, (void*)vem_fmod_d},
    {"sin_f_u10", 4, 0, (void*)vem_sin_f_u10},       {"cos_f_u10", 4, 0, (void*)vem_cos_f_u10},
    {"tan_f_u10", 4, 0, (void*)vem_tan_f_u10},       {"sin_f_u10_ph", 4, 0, (void*)vem_sin_f_u10_ph},
    {"cos_f_u10_ph", 4, 0, (void*)vem_cos_f_u10_ph}, {"tan_f_u10_ph", 4, 0, (void*)vem_tan_f_u10_ph},
    {"exp_f_u10", 4, 0, (void*)vem_exp_f_u10},       {"exp_f_u35", 4, 0, (void*)vem_exp_f_u35},
    {"log_f_u10", 4, 0, (void*)vem_log_f_u10},       {"log_f_u35", 4, 0, (void*)vem_log_f_u35},
    {"pow_f_u10", 4, 1, (void*)vem_pow_f_u10},       {"pow_f_u35", 4, 1, (void*)vem_pow_f_u35},
    {"fmod_f", 4, 1, (void*)vem_fmod_f},
    {"sin_d_u35", 8, 0, (void*)vem_sin_d_u35},       {"cos_d_u35", 8, 0, (void*)vem_cos_d_u35},
    {"tan_d_u35", 8, 0, (void*)vem_tan_d_u35},       {"atan_d_u35", 8, 0, (void*)vem_atan_d_u35},
    {"asin_d_u10", 8, 0, (void*)vem_asin_d_u10},     {"asin_d_u35", 8, 0, (void*)vem_asin_d_u35},
    {"acos_d_u10", 8, 0, (void*)vem_acos_d_u10},     {"acos_d_u35", 8, 0, (void*)vem_acos_d_u35},
    {"atan2_d_u10", 8, 1, (void*)vem_atan2_d_u10},   {"atan2_d_u35", 8, 1, (void*)vem_atan2_d_u35},
    {"fdim_d", 8, 1, (void*)vem_fdim_d},
    {"sin_f_u35", 4, 0, (void*)vem_sin_f_u35},       {"cos_f_u35", 4, 0, (void*)vem_cos_f_u35},
    {"tan_f_u35", 4, 0, (void*)vem_tan_f_u35},       {"atan_f_u10", 4, 0, (void*)vem_atan_f_u10},
    {"atan_f_u35", 4, 0, (void*)vem_atan_f_u35},     {"asin_f_u10", 4, 0, (void*)vem_asin_f_u10},
    {"asin_f_u35", 4, 0, (void*)vem_asin_f_u35},     {"acos_f_u10", 4, 0, (void*)vem_acos_f_u10},
    {"acos_f_u35", 4, 0, (void*)vem_acos_f_u35},     {"atan2_f_u10", 4, 1, (void*)vem_atan2_f_u10},
    {"atan2_f_u35", 4, 1, (void*)vem_atan2_f_u35},   {"fdim_f", 4, 1, (void*)vem_fdim_f},
};

const Entry* find(const char* name) {
  for (const Entry& e : kTable)
    if (std::strcmp(e.name, name) == 0) return &e;
  return nullptr;
}

int call(const Entry* e, const void* x, const void* y, void* o, size_t n, cudaStream_t s) {
  if (e->elem == 8) {
    if (e->binary) return ((binary_d)e->fn)((const double*)x, (const double*)y, (double*)o, n, s);
    return ((unary_d)e->fn)((const double*)x, (double*)o, n, s);
  }
  if (e->binary) return ((binary_f)e->fn)((const float*)x, (const float*)y, (float*)o, n, s);
  return ((unary_f)e->fn)((const float*)x, (float*)o, n, s);
}

}  // namespace

extern "C" int vem_run_sharded_on(const char* name, const void* x, const void* y2, void* out, size_t n,
                                  int ngpu, const int* devices, double* ms_out) {
  const Entry* e = find(name);
  if (!e || !devices) return (int)cudaErrorInvalidValue;
  if (e->binary && !y2) return (int)cudaErrorInvalidValue;
  int ndev = 0;
  cudaError_t st = cudaGetDeviceCount(&ndev);
  if (st != cudaSuccess) return (int)st;
  if (ngpu < 1) return (int)cudaErrorInvalidValue;
  for (int g = 0; g < ngpu; g++)
    if (devices[g] < 0 || devices[g] >= ndev) return (int)cudaErrorInvalidDevice;
  std::vector<int> rc(ngpu, 0);
  std::vector<double> ms(ngpu, 0.0);
  std::vector<std::thread> th;
  for (int g = 0; g < ngpu; g++) {
    th.emplace_back([&, g] {
      size_t lo = n * (size_t)g / ngpu, hi = n * (size_t)(g + 1) / ngpu, m = hi - lo;
      size_t bytes = m * e->elem;
      cudaError_t err = cudaSetDevice(devices[g]);
      cudaStream_t s = nullptr;
      void *dx = nullptr, *dy = nullptr, *dout = nullptr;
      cudaEvent_t e0 = nullptr, e1 = nullptr;
      if (err == cudaSuccess) err = cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
      if (err == cudaSuccess && m) err = cudaMalloc(&dx, bytes);
      if (err == cudaSuccess && m && e->binary) err = cudaMalloc(&dy, bytes);
      if (err == cudaSuccess && m) err = cudaMalloc(&dout, bytes);
      if (err == cudaSuccess) err = cudaEventCreate(&e0);
      if (err == cudaSuccess) err = cudaEventCreate(&e1);
      if (err == cudaSuccess && m) err = cudaMemcpyAsync(dx, (const char*)x + lo * e->elem, bytes, cudaMemcpyHostToDevice, s);
      if (err == cudaSuccess && m && e->binary)
        err = cudaMemcpyAsync(dy, (const char*)y2 + lo * e->elem, bytes, cudaMemcpyHostToDevice, s);
      if (err == cudaSuccess) err = cudaEventRecord(e0, s);
      if (err == cudaSuccess && m) err = (cudaError_t)call(e, dx, dy, dout, m, s);
      if (err == cudaSuccess) err = cudaEventRecord(e1, s);
      if (err == cudaSuccess && m) err = cudaMemcpyAsync((char*)out + lo * e->elem, dout, bytes, cudaMemcpyDeviceToHost, s);
      if (err == cudaSuccess) err = cudaStreamSynchronize(s);
      float t = 0.f;
      if (err == cudaSuccess) err = cudaEventElapsedTime(&t, e0, e1);
      ms[g] = t;
      if (dx) cudaFree(dx);
      if (dy) cudaFree(dy);
      if (dout) cudaFree(dout);
      if (e0) cudaEventDestroy(e0);
      if (e1) cudaEventDestroy(e1);
      if (s) cudaStreamDestroy(s);
      rc[g] = (int)err;
    });
  }
  for (auto& t : th) t.join();
  double mx = 0.0;
  for (int g = 0; g < ngpu; g++) {
    if (rc[g]) return rc[g];
    if (ms[g] > mx) mx = ms[g];
  }
  if (ms_out) *ms_out = mx;
  return 0;
}

extern "C" int vem_run_sharded(const char* name, const void* x, const void* y2, void* out, size_t n, int ngpu,
                               double* ms_out) {
  int ndev = 0;
  cudaError_t st = cudaGetDeviceCount(&ndev);
  if (st != cudaSuccess) return (int)st;
  if (ngpu < 1 || ngpu > ndev) return (int)cudaErrorInvalidDevice;
  std::vector<int> devs(ngpu);
  for (int g = 0; g < ngpu; g++) devs[g] = g;
  return vem_run_sharded_on(name, x, y2, out, n, ngpu, devs.data(), ms_out);
}
