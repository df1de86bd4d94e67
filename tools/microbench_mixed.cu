// Microbenchmark: do DMMA.8x8x4 and DFMA share the fp64 pipe on B200, or do they add up?
// Three kernels with the same launch shape: DFMA only, DMMA only, and a mixed one in which
// every warp interleaves D DMMAs per F DFMAs (independent accumulator chains).  If the two
// units were separate, the mixed kernel would exceed either peak.  Not part of the product.
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); return 1; } } while (0)

__device__ __forceinline__ void dmma884(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d[0]), "+d"(d[1]) : "d"(a), "d"(b));
}

// ND DMMA chains and NF DFMA chains per warp, each advanced once per iteration
template <int ND, int NF>
__global__ void mixed(double* out, int iters, double a, double b) {
  double acc[ND > 0 ? ND : 1][2];
  double x[NF > 0 ? NF : 1];
#pragma unroll
  for (int i = 0; i < (ND > 0 ? ND : 1); ++i) acc[i][0] = acc[i][1] = threadIdx.x;
#pragma unroll
  for (int i = 0; i < (NF > 0 ? NF : 1); ++i) x[i] = threadIdx.x + i;
  const double fa = 1.0 + threadIdx.x * 1e-9, fb = 1.0 - threadIdx.x * 1e-9;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
#pragma unroll
      for (int i = 0; i < ND; ++i) dmma884(acc[i], fa, fb);
#pragma unroll
      for (int i = 0; i < NF; ++i) x[i] = fma(x[i], a, b);
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < ND; ++i) s += acc[i][0] + acc[i][1];
#pragma unroll
  for (int i = 0; i < NF; ++i) s += x[i];
  if (s == 12345.678) out[0] = s;
}

template <int ND, int NF>
int run(int sms, double* out, int warps_per_sm) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int threads = 128, blocks = sms * warps_per_sm / 4, iters = 4000;
  mixed<ND, NF><<<blocks, threads>>>(out, 10, 1.0000001, 1e-9);
  CK(cudaDeviceSynchronize());
  cudaEventRecord(e0);
  mixed<ND, NF><<<blocks, threads>>>(out, iters, 1.0000001, 1e-9);
  cudaEventRecord(e1);
  CK(cudaEventSynchronize(e1));
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double warps = (double)blocks * threads / 32, reps = (double)iters * 4;
  const double fl_d = 2.0 * 256 * ND * reps * warps, fl_f = 2.0 * 32 * NF * reps * warps;
  printf("DMMA chains=%2d DFMA chains=%2d warps/SM=%2d  %.3f ms  DMMA %.2f + DFMA %.2f = %.2f TFLOP/s\n", ND, NF,
         warps_per_sm, ms, fl_d / ms / 1e9, fl_f / ms / 1e9, (fl_d + fl_f) / ms / 1e9);
  return 0;
}

int main() {
  cudaDeviceProp p;
  CK(cudaGetDeviceProperties(&p, 0));
  printf("device %s SMs %d\n", p.name, p.multiProcessorCount);
  double* out;
  CK(cudaMalloc(&out, 8));
  const int sms = p.multiProcessorCount;
  for (int w : {8, 16}) {
    run<4, 0>(sms, out, w);
    run<0, 16>(sms, out, w);
    run<4, 8>(sms, out, w);
    run<4, 16>(sms, out, w);
    run<2, 16>(sms, out, w);
    run<4, 32>(sms, out, w);
    run<1, 16>(sms, out, w);
  }
  return 0;
}
