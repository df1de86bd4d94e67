// S5 / S8 — least squares for the spectral coefficients of the reduced BEP (QR
// precomputed at Step 2 and recomputed at Step 4b).
//
// Factorization: column equilibration (unit 2-norm columns) then CholeskyQR2:
//   G = A^T A, G = R1^T R1, Q1 = A R1^{-1};  G2 = Q1^T Q1 = R2^T R2, Q = Q1 R2^{-1}; R = R2 R1.
// CholeskyQR2 gives an orthogonal Q to O(eps) when κ(A)^2 eps << 1 (κ of the equilibrated
// BEP ≤ 1.85e4 at cfg1-3), and is built only from GEMM-shaped, fully
// parallel steps plus a small K x K Cholesky.
// Apply: coef = M g with M = D R^{-1} Q^T formed once per factorisation (K x |γ_in|; one GEMV per
// solve instead of a K-step back substitution), u_γ = E coef (extension operator),
// optional clamp (R17).
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

// R^{-1} of the upper-triangular K x K R (col-major), one column per thread (back substitution of e_j).
__global__ void rinv_kernel(const double* __restrict__ R, int K, double* __restrict__ Ri) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= K) return;
  double* x = Ri + (size_t)j * K;
  for (int i = K - 1; i > j; --i) x[i] = 0.0;
  for (int i = j; i >= 0; --i) {
    double v = (i == j) ? 1.0 : 0.0;
    for (int k = i + 1; k <= j; ++k) v -= R[(size_t)k * K + i] * x[k];
    x[i] = v / R[(size_t)i * K + i];
  }
}

// M = diag(scale) R^{-1} Q^T  (K x m, row-major), Q col-major m x K (so Q^T rows are contiguous).
// 32x32 output tiles, k-loop over 32-wide panels (R^{-1} upper: panels below the diagonal skipped).
__global__ void lsq_operator_kernel(const double* __restrict__ Ri, const double* __restrict__ Q, const double* scale,
                                    int K, int64_t m, double* __restrict__ M) {
  const int c0 = blockIdx.y * 32;
  const int64_t i0 = (int64_t)blockIdx.x * 32;
  __shared__ double sa[32][33], sb[32][33];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;   // 256 threads: ty 0..7
  double acc[4] = {0, 0, 0, 0};
  for (int k0 = c0 - (c0 % 32); k0 < K; k0 += 32) {
    for (int q = ty; q < 32; q += 8) {
      const int c = c0 + q, k = k0 + tx;
      sa[q][tx] = (c < K && k < K && k >= c) ? Ri[(size_t)k * K + c] : 0.0;   // Ri[c][k]
      const int kk = k0 + q;
      const int64_t i = i0 + tx;
      sb[q][tx] = (kk < K && i < m) ? Q[(size_t)kk * m + i] : 0.0;             // Q^T[kk][i]
    }
    __syncthreads();
#pragma unroll 8
    for (int k = 0; k < 32; ++k) {
      const double b = sb[k][tx];
#pragma unroll
      for (int u = 0; u < 4; ++u) acc[u] += sa[ty + 8 * u][k] * b;
    }
    __syncthreads();
  }
  for (int u = 0; u < 4; ++u) {
    const int c = c0 + ty + 8 * u;
    const int64_t i = i0 + tx;
    if (c < K && i < m) M[(size_t)c * m + i] = scale[c] * acc[u];
  }
}

// coef[r][c] = Σ_i M[c][i] g[r][i]: one 128-thread block per (c, r)
__global__ void lsq_gemv_kernel(const double* __restrict__ M, int64_t m, int K, const double* __restrict__ g, int nrhs,
                                double* __restrict__ coef) {
  const int c = blockIdx.x, r = blockIdx.y;
  const double* a = M + (size_t)c * m;
  const double* b = g + (size_t)r * m;
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < m; i += blockDim.x) s = fma(a[i], b[i], s);
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  __shared__ double red[4];
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) coef[(size_t)r * K + c] = (red[0] + red[1]) + (red[2] + red[3]);
}

// u_γ[r][g] = Σ_c E[c][g] coef[r][c] (optionally clamped at 0, R17): 32 γ points x 8 column slices
// per block, coefficients staged in shared memory.
__global__ void extend2_kernel(const double* __restrict__ E, int64_t ng, int K, const double* __restrict__ coef, int r,
                               int clamp, double* __restrict__ ug) {
  extern __shared__ double sc[];   // K coefficients + 8 x 32 partial sums
  const double* cr = coef + (size_t)r * K;
  for (int c = threadIdx.x; c < K; c += blockDim.x) sc[c] = cr[c];
  double* part = sc + K;
  __syncthreads();
  const int gl = threadIdx.x & 31, sl = threadIdx.x >> 5;
  const int64_t g = (int64_t)blockIdx.x * 32 + gl;
  double s = 0.0;
  if (g < ng)
    for (int c = sl; c < K; c += 8) s = fma(E[(size_t)c * ng + g], sc[c], s);
  part[sl * 32 + gl] = s;
  __syncthreads();
  if (sl == 0 && g < ng) {
    double t = part[gl];
    for (int q = 1; q < 8; ++q) t += part[q * 32 + gl];
    ug[(size_t)r * ng + g] = clamp ? fmax(t, 0.0) : t;
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
  // apply operator M = D R^{-1} Q^T (K x |γ_in|): each LSQ solve is then one GEMV
  if (!ctx->Mlsq) DPM_CUDA_TRY(ctx, cudaMalloc(&ctx->Mlsq, (size_t)m * K * sizeof(double)));
  double* Ri = R1;   // R1 is free after the trmm
  DPM_COUNT_LAUNCH(1);
  rinv_kernel<<<(K + 63) / 64, 64, 0, s>>>(ctx->R, K, Ri);
  DPM_COUNT_LAUNCH(1);
  lsq_operator_kernel<<<dim3((unsigned)((m + 31) / 32), (K + 31) / 32), 256, 0, s>>>(Ri, ctx->Q, ctx->colscale, K, m,
                                                                                      ctx->Mlsq);
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
  DPM_COUNT_LAUNCH(1);
  lsq_gemv_kernel<<<dim3(K, nrhs), 128, 0, s>>>(ctx->Mlsq, m, K, g, nrhs, coef);
  if (u_gamma) return lsq_extend(ctx->E, ng, K, coef, nrhs, clamp, u_gamma, s);
  return cudaGetLastError();
}

// ---- building blocks shared with the octant DD (dd.cu): distributed CholeskyQR2 ----
cudaError_t lsq_gram(const double* A, int64_t m, int K, double* G, cudaStream_t s) {
  cudaError_t e = cudaMemsetAsync(G, 0, (size_t)K * K * sizeof(double), s);
  if (e != cudaSuccess) return e;
  const int tiles = (K + 31) / 32;
  const int64_t target_split = std::max<int64_t>(1, (148 * 4) / ((int64_t)tiles * (tiles + 1) / 2));
  const int64_t rps = std::max<int64_t>(32, ((m + target_split - 1) / target_split + 31) / 32 * 32);
  const int nsplit = (int)std::max<int64_t>(1, (m + rps - 1) / rps);
  DPM_COUNT_LAUNCH(1);
  gram_kernel<<<dim3(tiles, tiles, nsplit), TB, 0, s>>>(A, m, K, G, rps);
  return cudaGetLastError();
}

cudaError_t lsq_cholesky(double* G, int K, int* dfail, cudaStream_t s) {
  DPM_COUNT_LAUNCH(1);
  cholesky_kernel<<<1, 1024, 0, s>>>(G, K, dfail);
  return cudaGetLastError();
}

cudaError_t lsq_trsm_rows(double* A, int64_t m, int K, const double* R, cudaStream_t s) {
  if (m == 0) return cudaSuccess;
  DPM_COUNT_LAUNCH(1);
  trsm_rows_kernel<<<(unsigned)((m + 127) / 128), 128, 0, s>>>(A, m, K, R);
  return cudaGetLastError();
}

cudaError_t lsq_trmm(const double* A, const double* B, double* C, int K, cudaStream_t s) {
  DPM_COUNT_LAUNCH(1);
  trmm_kernel<<<(K * K + 255) / 256, 256, 0, s>>>(A, B, C, K);
  return cudaGetLastError();
}

cudaError_t lsq_scale_cols(const double* B, int64_t m, int K, const double* scale, double* A, cudaStream_t s) {
  DPM_COUNT_LAUNCH(1);
  scale_cols_kernel<<<148 * 8, TB, 0, s>>>(B, m, K, scale, A);
  return cudaGetLastError();
}

// M = diag(scale) R^{-1} Q^T (K x m row-major); Ri_ws: K x K workspace
cudaError_t lsq_build_operator(const double* R, const double* Q, int64_t m, int K, const double* scale, double* M,
                               double* Ri_ws, cudaStream_t s) {
  DPM_COUNT_LAUNCH(1);
  rinv_kernel<<<(K + 63) / 64, 64, 0, s>>>(R, K, Ri_ws);
  if (m == 0) return cudaGetLastError();
  DPM_COUNT_LAUNCH(1);
  lsq_operator_kernel<<<dim3((unsigned)((m + 31) / 32), (K + 31) / 32), 256, 0, s>>>(Ri_ws, Q, scale, K, m, M);
  return cudaGetLastError();
}

cudaError_t lsq_gemv(const double* M, int64_t m, int K, const double* g, int nrhs, double* coef, cudaStream_t s) {
  DPM_COUNT_LAUNCH(1);
  lsq_gemv_kernel<<<dim3(K, nrhs), 128, 0, s>>>(M, m, K, g, nrhs, coef);
  return cudaGetLastError();
}

cudaError_t lsq_extend(const double* E, int64_t ng, int K, const double* coef, int nrhs, int clamp, double* ug,
                       cudaStream_t s) {
  const size_t smem = (size_t)(K + 256) * sizeof(double);
  for (int r = 0; r < nrhs; ++r) {
    DPM_COUNT_LAUNCH(1);
    extend2_kernel<<<(unsigned)((ng + 31) / 32), 256, smem, s>>>(E, ng, K, coef, r, clamp, ug);
  }
  return cudaGetLastError();
}
