// probe.cu -- microbenchmarks the roofline needs beside the copy bandwidth
// and bf16 numbers of MEASURED_PEAKS.json (BASELINE.md s.2 asks for the FP64
// rate: every decision of the hot path is taken in fp64, P1):
// sustained DFMA throughput over every SM, and the SM instruction issue rate
// is derived from the clock (bench.py).
#include <cuda_runtime.h>
#include <stdint.h>

#include "internal.cuh"

namespace helios {
namespace {

// 8 independent DFMA chains per thread (enough ILP to fill the fp64 pipe),
// `iters` x 8 FMAs; the result is stored so nothing is optimised away
__global__ void __launch_bounds__(256) k_dfma(double* __restrict__ out, int iters, double y) {
  double x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = 1.0 + 1e-3 * (threadIdx.x + i);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = fma(x[i], y, 1e-9);
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

}  // namespace
}  // namespace helios

extern "C" int helios_util_fp64_fma_tflops(double* tflops, void* stream) {
  if (!tflops) return 1;
  const cudaStream_t s = (cudaStream_t)stream;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int blocks = sms * 8, threads = 256, iters = 1 << 14;
  double* out = nullptr;
  if (helios::dev_alloc((void**)&out, sizeof(double) * blocks * threads, s) != cudaSuccess) {
    cudaGetLastError();
    return 2;
  }
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  helios::k_dfma<<<blocks, threads, 0, s>>>(out, 256, 0.999999);  // warm-up
  cudaEventRecord(e0, s);
  helios::k_dfma<<<blocks, threads, 0, s>>>(out, iters, 0.999999);
  cudaEventRecord(e1, s);
  cudaError_t e = cudaEventSynchronize(e1);
  float ms = 0.f;
  if (e == cudaSuccess) e = cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFreeAsync(out, s);
  cudaStreamSynchronize(s);
  if (e != cudaSuccess || ms <= 0.f) {
    cudaGetLastError();
    return 3;
  }
  const double flops = 2.0 * 8.0 * (double)iters * blocks * threads;
  *tflops = flops / (ms * 1e-3) / 1e12;
  return 0;
}
