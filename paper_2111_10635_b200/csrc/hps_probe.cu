// hps_probe.cu — FP64 pipe microbenchmark used by bench.py for the roofline denominator
// (MEASURED_PEAKS.json carries HBM and bf16 peaks only; the plan evaluator is FP64-bound).
#include "hps_launch.h"
#include <cuda_runtime.h>
#include <cstdint>

namespace {
__global__ void dfma_probe(double* out, int iters) {
  double a0 = threadIdx.x * 1e-3, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3;
  double a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
  const double m = 0.9999999, c = 1e-7;
  for (int i = 0; i < iters; i++) {
#pragma unroll
    for (int j = 0; j < 8; j++) {
      a0 = fma(a0, m, c); a1 = fma(a1, m, c); a2 = fma(a2, m, c); a3 = fma(a3, m, c);
      a4 = fma(a4, m, c); a5 = fma(a5, m, c); a6 = fma(a6, m, c); a7 = fma(a7, m, c);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}

__global__ void ddiv_probe(double* out, int iters) {
  double a0 = 1.0 + threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3;
  const double d = 1.0000001;
  for (int i = 0; i < iters; i++) {
#pragma unroll
    for (int j = 0; j < 8; j++) { a0 = a0 / d; a1 = a1 / d; a2 = a2 / d; a3 = a3 / d; }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3;
}
}  // namespace

extern "C" int hps_probe_fp64(int kind, double* d_out, int blocks, int threads, int iters,
                              void* stream) {
  HPS_COUNT_LAUNCH();
  if (kind == 0)
    dfma_probe<<<blocks, threads, 0, (cudaStream_t)stream>>>(d_out, iters);
  else
    ddiv_probe<<<blocks, threads, 0, (cudaStream_t)stream>>>(d_out, iters);
  return cudaGetLastError() == cudaSuccess ? 0 : 4;
}
