// Microbenchmark: fp64 pipe peaks on B200 (DFMA vs DMMA.8x8x4) and a plain
// double2 copy, to choose the DST-I transform design ("The
// builder must microbenchmark DFMA and DMMA peaks on the box before choosing the
// transform").  Not part of the product; run via gpurun.
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); return 1; } } while (0)

__global__ void dfma_peak(double* out, int iters, double a, double b) {
  double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
      x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
    }
  }
  double s = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
  if (s == 12345.678) out[0] = s;
}

__device__ __forceinline__ void dmma884(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d[0]), "+d"(d[1]) : "d"(a), "d"(b));
}

__device__ __forceinline__ void dmma1688(double (&d)[4], double a0, double a1, double a2, double a3,
                                         double b0, double b1) {
  asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
               : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3])
               : "d"(a0), "d"(a1), "d"(a2), "d"(a3), "d"(b0), "d"(b1));
}

__global__ void dmma_peak(double* out, int iters) {
  double acc[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) { acc[i][0] = 0; acc[i][1] = 0; }
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 8; ++u) dmma884(acc[u], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += acc[i][0] + acc[i][1];
  if (s == 12345.678) out[0] = s;
}

__global__ void dmma1688_peak(double* out, int iters) {
  double acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i) for (int j = 0; j < 4; ++j) acc[i][j] = 0;
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 4; ++u) dmma1688(acc[u], a, a, a, a, b, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) s += acc[i][0] + acc[i][1] + acc[i][2] + acc[i][3];
  if (s == 12345.678) out[0] = s;
}

__global__ void copy2(const double2* __restrict__ a, double2* __restrict__ b, size_t n) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (; i < n; i += stride) b[i] = a[i];
}

int main() {
  int dev = 0; cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, dev));
  printf("device %s SMs %d L2 %d MB smemOptin %zu\n", p.name, p.multiProcessorCount, p.l2CacheSize >> 20,
         p.sharedMemPerBlockOptin);
  double* out; CK(cudaMalloc(&out, 8));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int sms = p.multiProcessorCount;
  for (int bpsm : {4, 8}) {
    int iters = 20000, blocks = sms * bpsm, threads = 256;
    dfma_peak<<<blocks, threads>>>(out, 10, 1.0000001, 1e-9);
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    dfma_peak<<<blocks, threads>>>(out, iters, 1.0000001, 1e-9);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double fl = 2.0 * 64 * (double)iters * blocks * threads;
    printf("DFMA  blocks/SM=%d  %.2f TFLOP/s (%.3f ms)\n", bpsm, fl / ms / 1e9, ms);
  }
  for (int bpsm : {2, 4, 8}) {
    int iters = 20000, blocks = sms * bpsm, threads = 128;
    dmma_peak<<<blocks, threads>>>(out, 10);
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    dmma_peak<<<blocks, threads>>>(out, iters);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double fl = 2.0 * 256 * 8 * (double)iters * blocks * (threads / 32);
    printf("DMMA m8n8k4  blocks/SM=%d  %.2f TFLOP/s (%.3f ms)\n", bpsm, fl / ms / 1e9, ms);
  }
  for (int bpsm : {2, 4, 8}) {
    int iters = 10000, blocks = sms * bpsm, threads = 128;
    dmma1688_peak<<<blocks, threads>>>(out, 10);
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    dmma1688_peak<<<blocks, threads>>>(out, iters);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double fl = 2.0 * 16 * 8 * 8 * 4 * (double)iters * blocks * (threads / 32);
    printf("DMMA m16n8k8 blocks/SM=%d  %.2f TFLOP/s (%.3f ms)\n", bpsm, fl / ms / 1e9, ms);
  }
  size_t n = (size_t)1 << 28;  // 256M doubles = 2 GiB per buffer
  double2 *a, *b; CK(cudaMalloc(&a, n * 8)); CK(cudaMalloc(&b, n * 8));
  cudaMemset(a, 0, n * 8);
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0);
    copy2<<<sms * 8, 512>>>(a, b, n / 2);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("copy double2: %.1f GB/s\n", 2.0 * n * 8 / ms / 1e6);
  }
  return 0;
}
