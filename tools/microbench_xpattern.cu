// Microbenchmark: HBM read+write throughput of the n = 128 x-pass access pattern (each warp a tile of C
// consecutive columns x 128 rows at a 128 KB row stride, out of place) against a contiguous copy, on
// 64 fields (2 GiB in, 2 GiB out).  Answers whether the x pass's 5.4 TB/s is the pattern's ceiling.
// Not part of the product.
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); return 1; } } while (0)

constexpr int N = 128, NN = N * N;

// warp tile = C columns (C/2 double2 per row) x 128 rows; lanes cover (row, column pair)
template <int C>
__global__ void xpattern_copy(const double2* __restrict__ in, double2* __restrict__ out, int nfields) {
  constexpr int PAIRS = C / 2, ROWS_PER = 32 / PAIRS;   // rows per warp instruction
  const int lane = threadIdx.x & 31;
  const long gw = (blockIdx.x * (long)blockDim.x + threadIdx.x) >> 5, nw = ((long)gridDim.x * blockDim.x) >> 5;
  const long tpf = NN / C, ntiles = (long)nfields * tpf;
  for (long t = gw; t < ntiles; t += nw) {
    const long f = t / tpf, c0 = (t - f * tpf) * C;
    const size_t base = (size_t)f * NN * N + c0;
    double2 v[128 / ROWS_PER];
#pragma unroll
    for (int i = 0; i < 128 / ROWS_PER; ++i) {
      const int r = i * ROWS_PER + lane / PAIRS, cp = lane % PAIRS;
      v[i] = __ldcg(reinterpret_cast<const double2*>(reinterpret_cast<const double*>(in) + base + (size_t)r * NN) + cp);
    }
#pragma unroll
    for (int i = 0; i < 128 / ROWS_PER; ++i) {
      const int r = i * ROWS_PER + lane / PAIRS, cp = lane % PAIRS;
      __stcg(reinterpret_cast<double2*>(reinterpret_cast<double*>(out) + base + (size_t)r * NN) + cp, v[i]);
    }
  }
}

__global__ void contiguous_copy(const double2* __restrict__ in, double2* __restrict__ out, size_t n2) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n2; i += (size_t)gridDim.x * blockDim.x)
    __stcg(out + i, __ldcg(in + i));
}

template <typename F>
float timeit(F&& f) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  f();
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    f();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    best = ms < best ? ms : best;
  }
  return best;
}

int main() {
  cudaDeviceProp p;
  CK(cudaGetDeviceProperties(&p, 0));
  const int sms = p.multiProcessorCount, nf = 64;
  const size_t n = (size_t)nf * NN * N;   // doubles
  double *a, *b;
  CK(cudaMalloc(&a, n * 8));
  CK(cudaMalloc(&b, n * 8));
  CK(cudaMemset(a, 0, n * 8));
  const double gb = 2.0 * n * 8 / 1e9;
  float ms = timeit([&] { contiguous_copy<<<sms * 8, 512>>>((const double2*)a, (double2*)b, n / 2); });
  printf("contiguous copy          %.3f ms  %.0f GB/s\n", ms, gb / ms * 1e3);
  for (int wps : {8, 16, 32}) {
    ms = timeit([&] { xpattern_copy<16><<<sms * wps / 8, 256>>>((const double2*)a, (double2*)b, nf); });
    printf("x pattern C=16 warps/SM=%2d %.3f ms  %.0f GB/s\n", wps, ms, gb / ms * 1e3);
    ms = timeit([&] { xpattern_copy<32><<<sms * wps / 8, 256>>>((const double2*)a, (double2*)b, nf); });
    printf("x pattern C=32 warps/SM=%2d %.3f ms  %.0f GB/s\n", wps, ms, gb / ms * 1e3);
    ms = timeit([&] { xpattern_copy<64><<<sms * wps / 8, 256>>>((const double2*)a, (double2*)b, nf); });
    printf("x pattern C=64 warps/SM=%2d %.3f ms  %.0f GB/s\n", wps, ms, gb / ms * 1e3);
  }
  return 0;
}
