// S5 / S8 — least squares for the spectral coefficients of the reduced BEP (QR
// precomputed at Step 2 and recomputed at Step 4b).
//
// Factorization: column equilibration (unit 2-norm columns) then CholeskyQR2:
//   G = A^T A, G = R1^T R1, Q1 = A R1^{-1};  G2 = Q1^T Q1 = R2^T R2, Q = Q1 R2^{-1}; R = R2 R1.
// CholeskyQR2 gives an orthogonal Q to O(eps) when κ(A)^2 eps << 1 (κ of the equilibrated
// BEP ≤ 1.85e4 at cfg1-3), and is built only from GEMM-shaped, fully
// parallel steps plus a small K x K Cholesky.
// Apply: coef = D R^{-1} Q^T g,  u_γ = E coef (extension operator), optional clamp (R17).
#include "dpm_internal.h"

namespace {

constexpr int TB = 256;

__global__ void colnorm_kernel(const double* __restrict__ B, int64_t m, double* scale) {
  const int c = blockIdx.x;
  const double* col = B + (size_t)c * m;
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < m; i += blockDim.x) s += col[i] * col[i];
  __shared__ double red[TB / 32];
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0;
    for (int q = 0; q < TB / 32; ++q) t += red[q];
    scale[c] = t > 0 ? 1.0 / sqrt(t) : 1.0;
  }
}

__global__ void scale_cols_kernel(const double* __restrict__ B, int64_t m, int K, const double* scale, double* A) {
  const long tot = (long)m * K;
  for (long t = blockIdx.x * (long)blockDim.x + threadIdx.x; t < tot; t += (long)gridDim.x * blockDim.x)
    A[t] = B[t] * scale[t / m];
}

// G = A^T A (K x K, col-major), tiled 32x32 over (i, j) with partial sums over row-chunks.
// grid: (ceil(K/32), ceil(K/32), nsplit); atomics combine the row-chunks (G pre-zeroed).
__global__ void gram_kernel(const double* __restrict__ A, int64_t m, int K, double* G, int64_t rows_per_split) {
  const int bi = blockIdx.x * 32, bj = blockIdx.y * 32;
  if (bj < bi) return;   // upper tiles only; mirrored at the end
  const int64_t r0 = blockIdx.z * rows_per_split, r1 = min(m, r0 + rows_per_split);
  __shared__ double sa[32][33], sb[32][33];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;   // 256 threads: ty 0..7
  double acc[4] = {0, 0, 0, 0};
  for (int64_t r = r0; r < r1; r += 32) {
    for (int q = ty; q < 32; q += 8) {
      const int64_t row = r + tx;
      sa[q][tx] = (row < r1 && bi + q < K) ? A[(size_t)(bi + q) * m + row] : 0.0;
      sb[q][tx] = (row < r1 && bj + q < K) ? A[(size_t)(bj + q) * m + row] : 0.0;
    }
    __syncthreads();
#pragma unroll 8
    for (int rr = 0; rr < 32; ++rr) {
      const double b = sb[tx][rr];
#pragma unroll
      for (int u = 0; u < 4; ++u) acc[u] += sa[ty + 8 * u][rr] * b;
    }
    __syncthreads();
  }
  for (int u = 0; u < 4; ++u) {
    const int i = bi + ty + 8 * u, j = bj + tx;
    if (i < K && j < K && j >= i) atomicAdd(G + (size_t)j * K + i, acc[u]);
  }
}

// In-place Cholesky of the upper triangle of G (col-major, G[i + j*K] for i <= j) -> R upper.
// Single CTA (K <= ~1000); right-looking. Sets *fail if a pivot is not positive.
__global__ void cholesky_kernel(double* G, int K, int* fail) {
  __shared__ double piv;
  for (int k = 0; k < K; ++k) {
    if (threadIdx.x == 0) {
      const double d = G[(size_t)k * K + k];
      if (!(d > 0.0)) *fail = 1;
      piv = d > 0.0 ? sqrt(d) : 1.0;
      G[(size_t)k * K + k] = piv;
    }
    __syncthreads();
    for (int j = k + 1 + threadIdx.x; j < K; j += blockDim.x) G[(size_t)j * K + k] /= piv;
    __syncthreads();
    // trailing update: G[i][j] -= R[k][i] R[k][j] for k < i <= j
    const int rem = K - k - 1;
    const long tot = (long)rem * rem;
    for (long t = threadIdx.x; t < tot; t += blockDim.x) {
      const int ii = k + 1 + (int)(t % rem), jj = k + 1 + (int)(t / rem);
      if (ii <= jj) G[(size_t)jj * K + ii] -= G[(size_t)ii * K + k] * G[(size_t)jj * K + k];
    }
    __syncthreads();
  }
  // zero the strict lower triangle
  for (long t = threadIdx.x; t < (long)K * K; t += blockDim.x) {
    const int i = (int)(t % K), j = (int)(t / K);
    if (i > j) G[t] = 0.0;
  }
}

// A <- A R^{-1} row by row: x^T R = a^T  (forward substitution over columns).
__global__ void trsm_rows_kernel(double* A, int64_t m, int K, const double* __restrict__ R) {
  const int64_t row = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (row >= m) return;
  for (int j = 0; j < K; ++j) {
    double v = A[(size_t)j * m + row];
    for (int i = 0; i < j; ++i) v -= A[(size_t)i * m + row] * R[(size_t)j * K + i];
    A[(size_t)j * m + row] = v / R[(size_t)j * K + j];
  }
}

// C = A B for upper-triangular K x K (col-major)
__global__ void trmm_kernel(const double* __restrict__ A, const double* __restrict__ B, double* C, int K) {
  const long t = blockIdx.x * (long)blockDim.x + threadIdx.x;
  if (t >= (long)K * K) return;
  const int i = (int)(t % K), j = (int)(t / K);
  double s = 0.0;
  if (i <= j)
    for (int l = i; l <= j; ++l) s += A[(size_t)l * K + i] * B[(size_t)j * K + l];
  C[t] = s;
}

__global__ void diag_ratio_kernel(const double* R, int K, double* out) {
  double mx = 0, mn = INFINITY;
  for (int i = 0; i < K; ++i) {
    const double d = fabs(R[(size_t)i * K + i]);
    mx = fmax(mx, d);
    mn = fmin(mn, d);
  }
  *out = mx / mn;
}

// z[c + r*K] = Q_c . g_r
__global__ void qtg_kernel(const double* __restrict__ Q, int64_t m, int K, const double* __restrict__ g, int nrhs,
                           double* z) {
  const int c = blockIdx.x, r = blockIdx.y;
  const double* q = Q + (size_t)c * m;
  const double* gr = g + (size_t)r * m;
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < m; i += blockDim.x) s += q[i] * gr[i];
  __shared__ double red[TB / 32];
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0;
    for (int w = 0; w < TB / 32; ++w) t += red[w];
    z[(size_t)r * K + c] = t;
  }
}

// back substitution R x = z (one CTA per rhs), coef = scale .* x
__global__ void backsub_kernel(const double* __restrict__ R, int K, double* z, const double* scale, double* coef) {
  double* zr = z + (size_t)blockIdx.x * K;
  for (int j = K - 1; j >= 0; --j) {
    __syncthreads();
    const double xj = zr[j] / R[(size_t)j * K + j];
    __syncthreads();
    if (threadIdx.x == 0) zr[j] = xj;
    for (int i = threadIdx.x; i < j; i += blockDim.x) zr[i] -= R[(size_t)j * K + i] * xj;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < K; i += blockDim.x) coef[(size_t)blockIdx.x * K + i] = scale[i] * zr[i];
}

__global__ void extend_kernel(const double* __restrict__ E, int64_t ng, int K, const double* __restrict__ coef, int nrhs,
                              int clamp, double* ug) {
  const long tot = (long)ng * nrhs;
  for (long t = blockIdx.x * (long)blockDim.x + threadIdx.x; t < tot; t += (long)gridDim.x * blockDim.x) {
    const int r = (int)(t / ng);
    const long g = t - (long)r * ng;
    const double* cr = coef + (size_t)r * K;
    double s = 0.0;
    for (int c = 0; c < K; ++c) s += E[(size_t)c * ng + g] * cr[c];
    ug[t] = clamp ? fmax(s, 0.0) : s;
  }
}

dpm_status chol_qr_pass(dpm_ctx* ctx, double* A, int64_t m, int K, double* Rout, int* dfail, cudaStream_t s) {
  DPM_CUDA_TRY(ctx, cudaMemsetAsync(Rout, 0, (size_t)K * K * sizeof(double), s));
  const int tiles = (K + 31) / 32;
  const int64_t target_split = std::max<int64_t>(1, (148 * 4) / ((int64_t)tiles * (tiles + 1) / 2));
  const int64_t rps = std::max<int64_t>(32, ((m + target_split - 1) / target_split + 31) / 32 * 32);
  const int nsplit = (int)((m + rps - 1) / rps);
  DPM_COUNT_LAUNCH(1);
  gram_kernel<<<dim3(tiles, tiles, nsplit), TB, 0, s>>>(A, m, K, Rout, rps);
  DPM_COUNT_LAUNCH(1);
  cholesky_kernel<<<1, 1024, 0, s>>>(Rout, K, dfail);
  DPM_COUNT_LAUNCH(1);
  trsm_rows_kernel<<<(m + 127) / 128, 128, 0, s>>>(A, m, K, Rout);
  DPM_CUDA_TRY(ctx, cudaGetLastError());
  return DPM_OK;
}

}  // namespace

dpm_status lsq_factor(dpm_ctx* ctx, const double* B, cudaStream_t s) {
  const int K = ctx->K;
  const int64_t m = ctx->counts[DPM_SET_GAMMA_IN];
  if (K >= m) {
    ctx->err = "K >= |gamma_in|: under-determined BEP";
    return DPM_ERR_RANK;
  }
  if (!ctx->Q) DPM_CUDA_TRY(ctx, cudaMalloc(&ctx->Q, (size_t)m * K * sizeof(double)));
  if (!ctx->R) DPM_CUDA_TRY(ctx, cudaMalloc(&ctx->R, (size_t)K * K * sizeof(double)));
  if (!ctx->colscale) DPM_CUDA_TRY(ctx, cudaMalloc(&ctx->colscale, (size_t)K * sizeof(double)));
  if (!ctx->lsq_ws) DPM_CUDA_TRY(ctx, cudaMalloc(&ctx->lsq_ws, (size_t)(3 * K * K + 2 * 1024 * K + 16) * sizeof(double)));
  double* R1 = ctx->lsq_ws;
  double* R2 = R1 + (size_t)K * K;
  int* dfail = (int*)(R2 + (size_t)K * K);
  double* dcond = (double*)(dfail + 4);
  DPM_CUDA_TRY(ctx, cudaMemsetAsync(dfail, 0, sizeof(int), s));
  DPM_COUNT_LAUNCH(1);
  colnorm_kernel<<<K, TB, 0, s>>>(B, m, ctx->colscale);
  DPM_COUNT_LAUNCH(1);
  scale_cols_kernel<<<148 * 8, TB, 0, s>>>(B, m, K, ctx->colscale, ctx->Q);
  dpm_status st;
  if ((st = chol_qr_pass(ctx, ctx->Q, m, K, R1, dfail, s)) != DPM_OK) return st;
  if ((st = chol_qr_pass(ctx, ctx->Q, m, K, R2, dfail, s)) != DPM_OK) return st;
  DPM_COUNT_LAUNCH(1);
  trmm_kernel<<<(K * K + 255) / 256, 256, 0, s>>>(R2, R1, ctx->R, K);
  DPM_COUNT_LAUNCH(1);
  diag_ratio_kernel<<<1, 1, 0, s>>>(ctx->R, K, dcond);
  DPM_CUDA_TRY(ctx, cudaGetLastError());
  int hfail = 0;
  DPM_CUDA_TRY(ctx, cudaMemcpyAsync(&hfail, dfail, sizeof(int), cudaMemcpyDeviceToHost, s));
  DPM_CUDA_TRY(ctx, cudaMemcpyAsync(&ctx->bep_cond, dcond, sizeof(double), cudaMemcpyDeviceToHost, s));
  DPM_CUDA_TRY(ctx, cudaStreamSynchronize(s));
  if (hfail) {
    ctx->err = "CholeskyQR2 breakdown: BEP numerically rank deficient";
    return DPM_ERR_RANK;
  }
  return DPM_OK;
}

cudaError_t lsq_apply(dpm_ctx* ctx, const double* g, double* coef, double* u_gamma, int nrhs, int clamp,
                      cudaStream_t s) {
  const int K = ctx->K;
  const int64_t m = ctx->counts[DPM_SET_GAMMA_IN], ng = ctx->counts[DPM_SET_GAMMA];
  double* z = ctx->lsq_ws + 2 * (size_t)K * K + 16;
  DPM_COUNT_LAUNCH(1);
  qtg_kernel<<<dim3(K, nrhs), TB, 0, s>>>(ctx->Q, m, K, g, nrhs, z);
  DPM_COUNT_LAUNCH(1);
  backsub_kernel<<<nrhs, 256, 0, s>>>(ctx->R, K, z, ctx->colscale, coef);
  if (u_gamma) {
    const long tot = (long)ng * nrhs;
    DPM_COUNT_LAUNCH(1);
    extend_kernel<<<(int)std::min<long>((tot + TB - 1) / TB, 148 * 16), TB, 0, s>>>(ctx->E, ng, K, coef, nrhs, clamp,
                                                                                 u_gamma);
  }
  return cudaGetLastError();
}
