// fp64_peak.cu — measures the FP64 FMA throughput of this GPU (the "alu" roofline denominator of
// the fused heat iteration).  8 independent DFMA chains per thread, full occupancy.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/fp64_peak scripts/fp64_peak.cu && /tmp/fp64_peak
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = fma(x[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += x[i];
  if (s == 12345.678) out[0] = s;   // keep the chains live
}

int main() {
  int dev = 0, nsm = 0, clk = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  double* out;
  cudaMalloc(&out, 8);
  const int threads = 256, blocks = nsm * 8, iters = 1 << 14;
  dfma_kernel<<<blocks, threads>>>(out, 64, 0.999, 1e-3);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    dfma_kernel<<<blocks, threads>>>(out, iters, 0.999, 1e-3);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  const double fma = (double)blocks * threads * iters * 8;
  const double tf = 2.0 * fma / (best * 1e-3) / 1e12;
  printf("{\"fp64_tflops\": %.3f, \"dfma_per_clk_per_sm_at_max_clock\": %.2f, \"sms\": %d, \"max_clock_mhz\": %.0f}\n",
         tf, fma / (best * 1e-3) / nsm / (clk * 1e3), nsm, clk / 1e3);
  return 0;
}
