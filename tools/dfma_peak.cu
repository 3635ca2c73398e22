// dfma_peak.cu -- fp64 pipe microbenchmark for the roofline denominator ("measure
// the DFMA peak with a dependent-free DFMA microbenchmark at those clocks").
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/dfma_peak tools/dfma_peak.cu
//   tools/dfma_peak            -> one JSON line: DFMA throughput (independent chains), DFMA latency
//                                 (one dependent chain), SM clock during the run
#include <cstdio>
#include <cuda_runtime.h>

// ILP independent FMA chains per thread; every FMA is 2 flops.
template <int ILP>
__global__ void k_dfma(double* out, int iters, double a, double b) {
  double x[ILP];
#pragma unroll
  for (int k = 0; k < ILP; ++k) x[k] = threadIdx.x * 1e-9 + k;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < ILP; ++k) x[k] = fma(x[k], a, b);
  }
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < ILP; ++k) s += x[k];
  if (s == 1234.5) out[0] = s;   // keeps the chains live
}

// one dependent chain per thread, one warp per SM: cycles per DFMA = latency
__global__ void k_dfma_lat(double* out, long long* cyc, int iters, double a, double b) {
  double x = threadIdx.x * 1e-9;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 16; ++k) x = fma(x, a, b);
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  if (x == 1234.5) out[0] = x;
}

int main() {
  int dev = 0, sms = 0, clk_khz = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev);
  double* out;
  long long* cyc;
  cudaMalloc(&out, 8);
  cudaMalloc(&cyc, sizeof(long long) * 1024);
  const int ILP = 8, threads = 512, blocks = sms * 4, iters = 20000;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int w = 0; w < 3; ++w) k_dfma<ILP><<<blocks, threads>>>(out, iters / 10, 1.0000001, 1e-12);
  cudaEventRecord(e0);
  k_dfma<ILP><<<blocks, threads>>>(out, iters, 1.0000001, 1e-12);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  const double fmas = (double)blocks * threads * iters * ILP;
  const double tflops = 2.0 * fmas / (ms * 1e-3) / 1e12;
  const double per_sm_clk = fmas / (ms * 1e-3) / sms;   // FMAs per second per SM
  k_dfma_lat<<<sms, 32>>>(out, cyc, 1000, 1.0000001, 1e-12);
  long long c = 0;
  cudaMemcpy(&c, cyc, sizeof(long long), cudaMemcpyDeviceToHost);
  const double lat = (double)c / (1000.0 * 16);
  cudaError_t e = cudaGetLastError();
  printf("{\"dfma_tflops\": %.3f, \"dfma_per_sm_per_s\": %.4g, \"ms\": %.3f, \"dfma_latency_cycles\": %.2f, "
         "\"sms\": %d, \"attr_clock_mhz\": %.0f, \"config\": \"%d blocks x %d threads x %d chains x %d iters\", "
         "\"error\": \"%s\"}\n",
         tflops, per_sm_clk, ms, lat, sms, clk_khz / 1000.0, blocks, threads, ILP, iters, cudaGetErrorString(e));
  return e == cudaSuccess ? 0 : 1;
}
