// DFMA throughput vs warps per SM and independent chains per thread (uniform second operand), to
// size the thread-per-column DST kernels.  Not part of the product.
#include <cstdio>
#include <cuda_runtime.h>

__constant__ double c_k[8];

template <int CH>
__global__ void dfma_chains(double* out, int iters) {
  double acc[CH];
#pragma unroll
  for (int i = 0; i < CH; ++i) acc[i] = threadIdx.x + i;
  const double x = 1.0 + threadIdx.x * 1e-12;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < CH; ++u) acc[u] = fma(x, c_k[u & 7], acc[u]);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CH; ++i) s += acc[i];
  if (s == 12345.678) out[0] = s;
}

template <int CH>
void run(int sms, int warps_per_sm, double* out) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 8192 * 24 / CH;
  dfma_chains<CH><<<sms, 32 * warps_per_sm>>>(out, 16);
  cudaEventRecord(e0);
  dfma_chains<CH><<<sms, 32 * warps_per_sm>>>(out, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double flops = 2.0 * 32 * (double)iters * CH * warps_per_sm * sms;
  printf("DFMA chains=%2d warps/SM=%2d  %6.2f TFLOP/s\n", CH, warps_per_sm, flops / (ms * 1e-3) / 1e12);
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double k[8] = {0.999, 0.998, 0.997, 0.996, 0.995, 0.994, 0.993, 0.992};
  cudaMemcpyToSymbol(c_k, k, sizeof(k));
  double* out;
  cudaMalloc(&out, 8);
  for (int w : {4, 8, 12, 16, 32}) {
    run<4>(sms, w, out);
    run<8>(sms, w, out);
    run<24>(sms, w, out);
  }
  return 0;
}
