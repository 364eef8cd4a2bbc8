// FP64 latency / per-warp throughput probe (B200): dependent DFMA chains, K independent chains per
// thread, 1..W warps per SM.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 lat_probe.cu
#include <cstdio>
template <int K>
__global__ void chain(double* out, long long* cyc, int iters, double a, double b) {
  double x[K];
#pragma unroll
  for (int k = 0; k < K; ++k) x[k] = threadIdx.x * 1e-3 + k;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int k = 0; k < K; ++k) x[k] = fma(x[k], a, b);
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int k = 0; k < K; ++k) s += x[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
__global__ void shfl_chain(double* out, long long* cyc, int iters) {
  double x = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) x = __shfl_xor_sync(0xffffffffu, x, 1) + 1.0;
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
template <int K> void run(int warps, double* d, long long* c) {
  const int it = 4096;
  chain<K><<<1, 32 * warps>>>(d, c, it, 0.999, 1e-3);
  long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("K=%d warps=%2d: %.2f cyc per step (per chain step), %.3f DFMA warp-instr/cyc/SM\n", K, warps,
         (double)h / it, (double)K * warps * it / h);
}
int main() {
  double* d; long long* c;
  cudaMalloc(&d, 1 << 20); cudaMalloc(&c, 1 << 12);
  for (int w : {1, 2, 4, 8, 16}) { run<1>(w, d, c); run<2>(w, d, c); run<4>(w, d, c); run<8>(w, d, c); }
  shfl_chain<<<1, 32>>>(d, c, 4096);
  long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("shfl+dadd chain: %.2f cyc per step\n", (double)h / 4096);
  return 0;
}
