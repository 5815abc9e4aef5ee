// C++ host test of the drop-in boundary: include/vem.hpp over libvem.so,
// device buffers via the CUDA runtime, results compared bit-for-bit with the
// CPU oracle (oracle/_build/libvem_oracle.so, loaded with dlopen as the
// checker).  Built and run by tests/test_cpp_host.py on a GPU box.
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <vector>

#include "vem.hpp"

typedef void (*uarr_d)(const double*, double*, size_t);
typedef void (*barr_d)(const double*, const double*, double*, size_t);

int main(int argc, char** argv) {
  if (argc < 2) return 2;
  void* h = dlopen(argv[1], RTLD_NOW);
  if (!h) { std::printf("cannot load oracle %s\n", argv[1]); return 2; }
  const size_t n = (1 << 16) + 3;
  std::vector<double> x(n), y(n), o(n), e(n);
  uint64_t s = 88172645463325252ull;
  for (size_t i = 0; i < n; i++) {
    s ^= s << 13; s ^= s >> 7; s ^= s << 17;
    x[i] = std::ldexp((double)(s >> 11) * 0x1p-53 * 2 - 1, (int)(s % 41) - 20);
    y[i] = (double)((s >> 7) % 61) - 30.0 + 0.25;
  }
  double *dx, *dy, *dout;
  cudaMalloc(&dx, n * 8); cudaMalloc(&dy, n * 8); cudaMalloc(&dout, n * 8);
  cudaMemcpy(dx, x.data(), n * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(dy, y.data(), n * 8, cudaMemcpyHostToDevice);
  int bad = 0;
  struct U { const char* name; int (*f)(const double*, double*, size_t, vem::gpu::stream_t); const char* oname; };
  U us[] = {{"sin", vem::gpu::sin, "vo_sin_d_u10_arr"}, {"cos", vem::gpu::cos, "vo_cos_d_u10_arr"},
            {"tan", vem::gpu::tan, "vo_tan_d_u10_arr"}, {"atan", vem::gpu::atan, "vo_atan_d_u10_arr"},
            {"exp", vem::gpu::exp, "vo_exp_d_u10_arr"}, {"log", vem::gpu::log, "vo_log_d_u10_arr"}};
  for (auto& u : us) {
    if (u.f(dx, dout, n, nullptr) != 0) { std::printf("%s launch failed\n", u.name); return 1; }
    cudaMemcpy(o.data(), dout, n * 8, cudaMemcpyDeviceToHost);
    ((uarr_d)dlsym(h, u.oname))(x.data(), e.data(), n);
    if (std::memcmp(o.data(), e.data(), n * 8) != 0) { std::printf("%s differs\n", u.name); bad++; }
  }
  if (vem::gpu::pow(dx, dy, dout, n) != 0) return 1;
  cudaMemcpy(o.data(), dout, n * 8, cudaMemcpyDeviceToHost);
  ((barr_d)dlsym(h, "vo_pow_d_u10_arr"))(x.data(), y.data(), e.data(), n);
  if (std::memcmp(o.data(), e.data(), n * 8) != 0) { std::printf("pow differs\n"); bad++; }
  if (vem::gpu::fmod(dx, dy, dout, n) != 0) return 1;
  cudaMemcpy(o.data(), dout, n * 8, cudaMemcpyDeviceToHost);
  ((barr_d)dlsym(h, "vo_fmod_d_arr"))(x.data(), y.data(), e.data(), n);
  if (std::memcmp(o.data(), e.data(), n * 8) != 0) { std::printf("fmod differs\n"); bad++; }
  // the host multi-GPU driver on one device (host arrays in/out)
  double ms = 0;
  if (vem_run_sharded("exp_d_u10", x.data(), nullptr, o.data(), n, 1, &ms) != 0) return 1;
  ((uarr_d)dlsym(h, "vo_exp_d_u10_arr"))(x.data(), e.data(), n);
  if (std::memcmp(o.data(), e.data(), n * 8) != 0) { std::printf("run_sharded differs\n"); bad++; }
  // three shards on device 0 from three host threads (ragged boundaries:
  // n = 2^16 + 3 is not a multiple of 3 * 16 bytes), binary entry point
  const int devs[3] = {0, 0, 0};
  if (vem_run_sharded_on("pow_d_u10", x.data(), y.data(), o.data(), n, 3, devs, &ms) != 0) return 1;
  ((barr_d)dlsym(h, "vo_pow_d_u10_arr"))(x.data(), y.data(), e.data(), n);
  if (std::memcmp(o.data(), e.data(), n * 8) != 0) { std::printf("run_sharded_on differs\n"); bad++; }
  cudaFree(dx); cudaFree(dy); cudaFree(dout);
  std::printf("%s: %d mismatching entry points\n", bad ? "FAIL" : "OK", bad);
  return bad ? 1 : 0;
}
