// L2-resident streaming bandwidth: in-place read+write of a W MB buffer, repeated (the AP-solve
// passes run on 64 MB chunks that should stay in the 126 MB L2).  Not part of the product.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void rw(double2* __restrict__ a, size_t n, double s) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x, st = (size_t)gridDim.x * blockDim.x;
  for (; i < n; i += st) {
    double2 v = __ldcg(a + i);
    v.x *= s; v.y *= s;
    __stcg(a + i, v);
  }
}
// strided-row variant like the x pass: warp reads 256 B rows 128 KB apart
__global__ void rw_rows(double* __restrict__ a, int nfields, double s) {
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  const int tiles = nfields * 512;
  for (int t = gw; t < tiles; t += nw) {
    const int f = t / 512, c = (t % 512) * 32 + lane;
    double* col = a + (size_t)f * 2097152 + c;
    double v[8];
    for (int r0 = 0; r0 < 128; r0 += 8) {
#pragma unroll
      for (int r = 0; r < 8; ++r) v[r] = __ldcg(col + (size_t)(r0 + r) * 16384);
#pragma unroll
      for (int r = 0; r < 8; ++r) __stcg(col + (size_t)(r0 + r) * 16384, v[r] * s);
    }
  }
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int mb : {16, 32, 64, 96, 256, 4096}) {
    size_t n = (size_t)mb * (1 << 20) / 16;
    double2* a;
    cudaMalloc(&a, n * 16);
    cudaMemset(a, 0, n * 16);
    for (int w = 0; w < 3; ++w) rw<<<sms * 8, 256>>>(a, n, 1.0);
    const int reps = mb >= 1024 ? 3 : 20;
    cudaEventRecord(e0);
    for (int r = 0; r < reps; ++r) rw<<<sms * 8, 256>>>(a, n, 1.0);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("contiguous in-place rw %5d MB: %.2f TB/s (read+write)\n", mb, 2.0 * n * 16 * reps / (ms * 1e-3) / 1e12);
    if (mb == 64) {
      for (int bpsm : {2, 4, 8}) {
        for (int w = 0; w < 3; ++w) rw_rows<<<sms * bpsm, 256>>>((double*)a, 4, 1.0);
        cudaEventRecord(e0);
        for (int r = 0; r < reps; ++r) rw_rows<<<sms * bpsm, 256>>>((double*)a, 4, 1.0);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        printf("  x-pass-like rows, 64 MB, %d x 256 thr/SM: %.2f TB/s, %.1f us per pass\n", bpsm,
               2.0 * n * 16 * reps / (ms * 1e-3) / 1e12, ms * 1e3 / reps);
      }
    }
    cudaFree(a);
  }
  return 0;
}
