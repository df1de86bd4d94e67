// DMMA.8x8x4 throughput vs warps per SM and independent accumulator chains per warp
// (decides how many warps the DST kernels need).  Not part of the product.
#include <cstdio>
#include <cuda_runtime.h>

template <int CH>
__global__ void dmma_chains(double* out, int iters) {
  double acc[CH][2];
#pragma unroll
  for (int i = 0; i < CH; ++i) acc[i][0] = acc[i][1] = 0;
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < CH; ++u)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(acc[u][0]), "+d"(acc[u][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CH; ++i) s += acc[i][0] + acc[i][1];
  if (s == 12345.678) out[0] = s;
}

template <int CH>
void run(int sms, int warps_per_sm, double* out) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int threads = 32 * warps_per_sm;   // one CTA per SM
  const int iters = 4096 * 18 / CH;
  dmma_chains<CH><<<sms, threads>>>(out, 16);
  cudaEventRecord(e0);
  dmma_chains<CH><<<sms, threads>>>(out, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double flops = 2.0 * 256 * 32.0 / 32 * (double)iters * CH * warps_per_sm * sms;   // 256 MAC per warp-DMMA
  printf("chains=%2d warps/SM=%2d  %6.2f TFLOP/s\n", CH, warps_per_sm, flops / (ms * 1e-3) / 1e12);
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  cudaMalloc(&out, 8);
  for (int w : {4, 8, 12, 16}) {
    run<1>(sms, w, out);
    run<3>(sms, w, out);
    run<6>(sms, w, out);
    run<18>(sms, w, out);
  }
  return 0;
}
