/* A plain-C client of libdpm.so (no Python, no torch): one batched AP solve through the C ABI.
 *
 *   gcc -O2 examples/solve_c.c -Iinclude -I/usr/local/cuda/include -Lpaper_1811_03557_b200 -ldpm \
 *       -L/usr/local/cuda/lib64 -lcudart -Wl,-rpath,$PWD/paper_1811_03557_b200 -lm -o solve_c && ./solve_c 64
 *
 * The right-hand side is a discrete sine eigenfunction, q = (1/dt + λ_a + λ_b + λ_c) S with
 * S(x,y,z) = sin(π a i/(n+1)) sin(π b j/(n+1)) sin(π c k/(n+1)) and λ_m = (4/h²) sin²(π m/(2(n+1))),
 * so the exact solution of (I/dt - Δ_h) u = q with zero Dirichlet data is u = S.
 * Prints the max error and exits 1 if it exceeds 1e-12. */
#include <cuda_runtime.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

#include "dpm.h"

int main(int argc, char** argv) {
  const int n = argc > 1 ? atoi(argv[1]) : 64;
  const double lo = -1.1, hi = 1.1, dt = 1e-3, h = (hi - lo) / (n + 1);
  const int a = 3, b = n / 2, c = n;   /* three modes, including the highest */
  const dpm_grid grid = {n, lo, hi};
  const dpm_domain dom = {DPM_SPHERE, {0.0, 0.0, 0.0}, {1.0, 1.0, 1.0}};
  dpm_ctx* ctx = NULL;
  if (dpm_create(&grid, &dom, 2, dt, DPM_BASIS_CAUCHY, 0, &ctx) != DPM_OK) {
    fprintf(stderr, "dpm_create: %s\n", dpm_last_error(NULL));
    return 2;
  }
  const size_t nn = (size_t)n * n * n;
  double* S = (double*)malloc(nn * sizeof(double));
  double* q = (double*)malloc(nn * sizeof(double));
  const double pi = 3.14159265358979323846;
  const double la = 4.0 / (h * h) * pow(sin(pi * a / (2.0 * (n + 1))), 2);
  const double lb = 4.0 / (h * h) * pow(sin(pi * b / (2.0 * (n + 1))), 2);
  const double lc = 4.0 / (h * h) * pow(sin(pi * c / (2.0 * (n + 1))), 2);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j)
      for (int k = 0; k < n; ++k) {
        const size_t p = ((size_t)i * n + j) * n + k;
        S[p] = sin(pi * a * (i + 1) / (n + 1)) * sin(pi * b * (j + 1) / (n + 1)) * sin(pi * c * (k + 1) / (n + 1));
        q[p] = (1.0 / dt + la + lb + lc) * S[p];
      }
  double *dq = NULL, *du = NULL;
  if (cudaMalloc((void**)&dq, nn * sizeof(double)) != cudaSuccess ||
      cudaMalloc((void**)&du, nn * sizeof(double)) != cudaSuccess) {
    fprintf(stderr, "cudaMalloc failed\n");
    return 2;
  }
  cudaMemcpy(dq, q, nn * sizeof(double), cudaMemcpyHostToDevice);
  if (dpm_aux_solve_batch(ctx, dq, du, 1, NULL) != DPM_OK) {
    fprintf(stderr, "dpm_aux_solve_batch: %s\n", dpm_last_error(ctx));
    return 2;
  }
  cudaMemcpy(q, du, nn * sizeof(double), cudaMemcpyDeviceToHost);
  double err = 0.0;
  for (size_t p = 0; p < nn; ++p) err = fmax(err, fabs(q[p] - S[p]));
  printf("n = %d: max |u - S| = %.3e\n", n, err);
  cudaFree(dq);
  cudaFree(du);
  free(S);
  free(q);
  dpm_destroy(ctx);
  return err <= 1e-12 ? 0 : 1;
}
