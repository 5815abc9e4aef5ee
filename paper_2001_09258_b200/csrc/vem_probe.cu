// Pipe-peak microbenchmarks for the roofline denominators that
// MEASURED_PEAKS.json does not carry (SURVEY.md §7 hard part (h)): FP64 DFMA
// and FP32 FFMA throughput, independent chains, no memory traffic.
#include <cuda_runtime.h>

#include "../../include/vem.h"

namespace {

template <typename T, int CHAINS>
__global__ void __launch_bounds__(256) k_fma_peak(T* out, int iters, T a, T b) {
  T acc[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; c++) acc[c] = (T)(threadIdx.x + c);
  for (int i = 0; i < iters; i++) {
#pragma unroll
    for (int c = 0; c < CHAINS; c++) acc[c] = fma(acc[c], a, b);
  }
  T s = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; c++) s += acc[c];
  if (s == (T)12345.678) out[0] = s;  // keep the chains alive
}

}  // namespace

extern "C" int vem_probe_peak(int kind, int iters, double* gops_out) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int blocks = sms * 8, threads = 256, chains = 8;
  void* buf = nullptr;
  cudaError_t e = cudaMalloc(&buf, 16);
  if (e != cudaSuccess) return (int)e;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int rep = 0; rep < 4; rep++) {
    cudaEventRecord(e0);
    if (kind == 0)
      k_fma_peak<double, chains><<<blocks, threads>>>((double*)buf, iters, 0.999999, 1e-9);
    else
      k_fma_peak<float, chains><<<blocks, threads>>>((float*)buf, iters, 0.999999f, 1e-9f);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    if (rep > 0 && ms < best) best = ms;
  }
  e = cudaGetLastError();
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(buf);
  if (e != cudaSuccess) return (int)e;
  double ops = (double)blocks * threads * chains * (double)iters;
  if (gops_out) *gops_out = ops / (best * 1e-3) / 1e9;
  return 0;
}
