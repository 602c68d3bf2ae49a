// fp64_peak.cu — FP64 FMA-pipe throughput probe (not part of the hot path; used by bench.py to report the measured
// DFMA peak beside the nominal one).  Each thread runs 8 independent DFMA chains; 148·k blocks × 256 threads.
#include <cuda_runtime.h>
#include <stdint.h>

__global__ void __launch_bounds__(256) dfma_loop(double* out, int iters, double a, double b) {
  double x[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) x[j] = threadIdx.x * 1e-7 + j;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) x[j] = fma(x[j], a, b);
  }
  double s = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) s += x[j];
  if (s == 12345.678) out[0] = s;  // keep the chains alive
}

extern "C" int fp64_peak_probe(int blocks_per_sm, int iters, int reps, double* tflops_out, double* ms_out) {
  int dev = 0, sms = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return -1;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  double* out;
  if (cudaMalloc(&out, sizeof(double)) != cudaSuccess) return -1;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int blocks = sms * blocks_per_sm;
  dfma_loop<<<blocks, 256>>>(out, iters, 0.999999, 1e-9);  // warm-up
  cudaEventRecord(e0);
  for (int r = 0; r < reps; ++r) dfma_loop<<<blocks, 256>>>(out, iters, 0.999999, 1e-9);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  const double flops = 2.0 * 8.0 * (double)iters * blocks * 256.0 * reps;
  *tflops_out = flops / (ms * 1e-3) / 1e12;
  *ms_out = ms;
  cudaFree(out);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  return cudaGetLastError() == cudaSuccess ? 0 : -1;
}
