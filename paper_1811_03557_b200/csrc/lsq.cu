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
  const int c = blockIdx.y;   // column (no per-element 64-bit division)
  const double sc = scale[c];
  const size_t o = (size_t)c * m;
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < m; i += (long)gridDim.x * blockDim.x)
    A[o + i] = B[o + i] * sc;
}

// Blocked right-looking Cholesky G = R^T R (upper R, column-major K x K, upper triangle used),
// block size CB: (1) unblocked factor of the diagonal block in shared memory (one CTA),
// (2) row-panel solve R_kk^T X = G_k,j for the columns right of the block (one thread per column),
// (3) trailing update G_ij -= Σ_{k in block} R_ki R_kj for i <= j (2D grid).
constexpr int CB = 32;

// one warp: unblocked factor of the diagonal block with lane j holding column j in registers
// (row-k values by shuffle; a short last block is padded with the identity)
__global__ void chol_diag_kernel(double* G, int K, int k0, int* fail) {
  const int nb = min(CB, K - k0), j = threadIdx.x;
  double a[CB];   // a[i] = G(k0 + i, k0 + j), upper part used
#pragma unroll
  for (int i = 0; i < CB; ++i)
    a[i] = (i < nb && j < nb) ? G[(size_t)(k0 + j) * K + k0 + i] : (i == j ? 1.0 : 0.0);
  bool bad = false;
#pragma unroll
  for (int k = 0; k < CB; ++k) {
    const double d = __shfl_sync(0xffffffffu, a[k], k);   // a(k, k)
    bad |= !(d > 0.0);
    const double r = d > 0.0 ? sqrt(d) : 1.0, ir = 1.0 / r;
    if (j == k) a[k] = r;
    else if (j > k) a[k] *= ir;                            // row k right of the diagonal
    const double akj = a[k];
#pragma unroll
    for (int i = k + 1; i < CB; ++i) {                     // a(i, j) -= a(k, i) a(k, j), k < i <= j
      const double aki = __shfl_sync(0xffffffffu, a[k], i);
      if (i <= j && j > k) a[i] = fma(-aki, akj, a[i]);
    }
  }
  if (j == 0 && bad) *fail = 1;
  if (j < nb) {
#pragma unroll
    for (int i = 0; i < CB; ++i)
      if (i < nb) G[(size_t)(k0 + j) * K + k0 + i] = (i <= j) ? a[i] : 0.0;
  }
}

// row-panel solve R_kk^T X = G_k,j for the columns j right of the block: one warp per column, lane =
// row of the panel; R_kk (and 1/diag) staged in shared memory once per CTA
constexpr int CHOL_PW = 8;   // warps (columns) per CTA
__global__ void __launch_bounds__(32 * CHOL_PW) chol_panel_kernel(double* G, int K, int k0) {
  __shared__ double r[CB][CB + 1], rd[CB];
  const int nb = min(CB, K - k0), lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int e = threadIdx.x; e < nb * nb; e += blockDim.x) {
    const int i = e % nb, j = e / nb;
    r[i][j] = G[(size_t)(k0 + j) * K + k0 + i];
  }
  __syncthreads();
  if (threadIdx.x < nb) rd[threadIdx.x] = 1.0 / r[threadIdx.x][threadIdx.x];
  __syncthreads();
  const int j = k0 + nb + blockIdx.x * CHOL_PW + w;
  if (j >= K) return;
  double gv = lane < nb ? G[(size_t)j * K + k0 + lane] : 0.0;
  for (int q = 0; q < nb; ++q) {   // x_q = g_q / R_qq, then g_i -= R_qi x_q for i > q
    const double xq = __shfl_sync(0xffffffffu, gv, q) * rd[q];
    if (lane == q) gv = xq;
    else if (lane > q && lane < nb) gv = fma(-r[q][lane], xq, gv);
  }
  if (lane < nb) G[(size_t)j * K + k0 + lane] = gv;
}

__global__ void chol_update_kernel(double* G, int K, int k0) {
  const int nb = min(CB, K - k0);
  const int i = k0 + nb + blockIdx.y * 16 + threadIdx.y;
  const int j = k0 + nb + blockIdx.x * 16 + threadIdx.x;
  if (i >= K || j >= K || i > j) return;
  double s = 0.0;
  for (int q = 0; q < nb; ++q) s = fma(G[(size_t)i * K + k0 + q], G[(size_t)j * K + k0 + q], s);
  G[(size_t)j * K + i] -= s;
}

__global__ void zero_lower_kernel(double* G, int K) {
  const long t = blockIdx.x * (long)blockDim.x + threadIdx.x;
  if (t >= (long)K * K) return;
  const int i = (int)(t % K), j = (int)(t / K);
  if (i > j) G[t] = 0.0;
}

// Blocked inverse of an upper-triangular K x K R (col-major) by 32 x 32 tiles, nb = ceil(K/32):
//   X_bb = R_bb^{-1} (all diagonal tiles in parallel), then for each block diagonal d = 1..nb-1
//   X_{b,b+d} = -X_bb Σ_{k=b+1}^{b+d} R_{b,k} X_{k,b+d}   (independent tiles: one CTA each).
// Replaces a column-by-column back substitution whose K-step dependent chain of strided reads
// took ~1 ms at K = 578.  Entries beyond K are treated as the identity (never written).
constexpr int RT = 32;

__device__ __forceinline__ double rt_at(const double* R, int K, int i, int j) {   // padded R
  return (i < K && j < K) ? R[(size_t)j * K + i] : (i == j ? 1.0 : 0.0);
}

// one warp per diagonal tile: lane i computes row i of the inverse (x_i R = e_i, forward over j)
__global__ void rinv_diag_kernel(const double* __restrict__ R, int K, double* __restrict__ Ri) {
  __shared__ double a[RT][RT + 1], x[RT][RT + 1];
  const int b0 = blockIdx.x * RT, i = threadIdx.x;
  for (int e = 0; e < RT; ++e) a[i][e] = rt_at(R, K, b0 + i, b0 + e);   // a[row][col]
  __syncwarp();
  for (int j = 0; j < RT; ++j) {
    double v = (i == j) ? 1.0 : 0.0;
    if (j > i) {
      v = 0.0;
      for (int k = i; k < j; ++k) v = fma(x[i][k], a[k][j], v);
      v = -v;
    }
    x[i][j] = j < i ? 0.0 : v / a[j][j];
  }
  __syncwarp();
  for (int j = 0; j < RT; ++j)
    if (b0 + i < K && b0 + j < K) Ri[(size_t)(b0 + j) * K + b0 + i] = x[i][j];
}

// tile (b, b + d) of the inverse for the block diagonal d (grid: nb - d CTAs of 256 threads)
__global__ void __launch_bounds__(256) rinv_offdiag_kernel(const double* __restrict__ R, int K, int d,
                                                           double* __restrict__ Ri) {
  __shared__ double sa[RT][RT + 1], sb[RT][RT + 1];
  const int b = blockIdx.x, c = b + d;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;   // output (row ty + 8u, col tx)
  double acc[4] = {0, 0, 0, 0};
  // tile loads: lanes run over the (contiguous, col-major) row index
  for (int k = b + 1; k <= c; ++k) {   // T = Σ_k R_{b,k} X_{k,c}
    for (int q = ty; q < RT; q += 8) {
      sa[tx][q] = rt_at(R, K, b * RT + tx, k * RT + q);                     // R_{b,k}[tx][q]
      const int r = k * RT + tx, col = c * RT + q;
      sb[tx][q] = (r < K && col < K) ? Ri[(size_t)col * K + r] : (r == col ? 1.0 : 0.0);   // X_{k,c}[tx][q]
    }
    __syncthreads();
#pragma unroll 8
    for (int l = 0; l < RT; ++l) {
      const double bv = sb[l][tx];
#pragma unroll
      for (int u = 0; u < 4; ++u) acc[u] = fma(sa[ty + 8 * u][l], bv, acc[u]);
    }
    __syncthreads();
  }
  // X_{b,c} = -X_bb T
  for (int u = 0; u < 4; ++u) sb[ty + 8 * u][tx] = acc[u];
  for (int q = ty; q < RT; q += 8) {
    const int r = b * RT + tx, col = b * RT + q;
    sa[tx][q] = (r < K && col < K) ? Ri[(size_t)col * K + r] : (r == col ? 1.0 : 0.0);
  }
  __syncthreads();
  for (int u = 0; u < 4; ++u) {   // output (row tx, col ty + 8u): lanes store consecutive rows
    const int q = ty + 8 * u;
    double v = 0.0;
    for (int l = tx; l < RT; ++l) v = fma(sa[tx][l], sb[l][q], v);
    const int r = b * RT + tx, col = c * RT + q;
    if (r < K && col < K) Ri[(size_t)col * K + r] = -v;
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


// coef[r][c] = Σ_i M[c][i] g[r][i]: a 256-thread block per GEMV_ROWS rows of M, right-hand sides 2 at
// a time (each g element loaded once per GEMV_ROWS rows); 4 rows when that still gives >= 148 blocks
// (the DD / cfg4 operators), else 1 (small K: parallelism over rows matters more)
constexpr int GEMV_RC = 2;
template <int GEMV_ROWS, int GEMV_T>
__global__ void __launch_bounds__(GEMV_T) lsq_gemv_kernel(const double* __restrict__ M, int64_t m, int K,
                                                          const double* __restrict__ g, int nrhs,
                                                          double* __restrict__ coef) {
  pdl_prologue();
  const int c0 = blockIdx.x * GEMV_ROWS;
  __shared__ double red[GEMV_ROWS * GEMV_RC][GEMV_T / 32];
  const double* a[GEMV_ROWS];
#pragma unroll
  for (int q = 0; q < GEMV_ROWS; ++q) a[q] = M + (size_t)min(c0 + q, K - 1) * m;
  for (int r0 = 0; r0 < nrhs; r0 += GEMV_RC) {
    const int nr = min(GEMV_RC, nrhs - r0);
    const double* g0 = g + (size_t)r0 * m;
    const double* g1 = g + (size_t)(r0 + (nr > 1 ? 1 : 0)) * m;
    double acc[GEMV_ROWS][GEMV_RC];
#pragma unroll
    for (int q = 0; q < GEMV_ROWS; ++q) acc[q][0] = acc[q][1] = 0.0;
#pragma unroll 4
    for (int64_t i = threadIdx.x; i < m; i += GEMV_T) {
      const double x0 = __ldg(g0 + i), x1 = __ldg(g1 + i);
#pragma unroll
      for (int q = 0; q < GEMV_ROWS; ++q) {
        const double av = __ldg(a[q] + i);
        acc[q][0] = fma(av, x0, acc[q][0]);
        acc[q][1] = fma(av, x1, acc[q][1]);
      }
    }
#pragma unroll
    for (int q = 0; q < GEMV_ROWS; ++q)
#pragma unroll
      for (int r = 0; r < GEMV_RC; ++r) {
        double v = acc[q][r];
        for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if ((threadIdx.x & 31) == 0) red[q * GEMV_RC + r][threadIdx.x >> 5] = v;
      }
    __syncthreads();
    if (threadIdx.x < GEMV_ROWS * GEMV_RC) {
      const int q = threadIdx.x / GEMV_RC, r = threadIdx.x % GEMV_RC;
      double v = 0.0;
#pragma unroll
      for (int w = 0; w < GEMV_T / 32; ++w) v += red[threadIdx.x][w];
      if (c0 + q < K && r < nr) coef[(size_t)(r0 + r) * K + c0 + q] = v;
    }
    __syncthreads();
  }
}

void launch_gemv(const double* M, int64_t m, int K, const double* g, int nrhs, double* coef, cudaStream_t s) {
  DPM_COUNT_LAUNCH(1);
  if (K >= 4 * 148)
    launch_pdl(lsq_gemv_kernel<4, 512>, (K + 3) / 4, 512, 0, s, M, m, K, g, nrhs, coef);
  else if (K <= 2 * 148 && m >= 32768)   // few long rows (Test B: K = 150, |γ_in| ~ 6e4): 4x the loads in flight per row
    launch_pdl(lsq_gemv_kernel<1, 1024>, K, 1024, 0, s, M, m, K, g, nrhs, coef);
  else
    launch_pdl(lsq_gemv_kernel<1, 256>, K, 256, 0, s, M, m, K, g, nrhs, coef);
}

// u_γ[r][g] = Σ_c E[c][g] coef[r][c] (optionally clamped at 0, R17): 32 γ points x SL column slices
// per block (SL = 32: 1024 threads, ~K/32 independent coalesced loads per thread in flight — the E stream
// (|γ| x K, 19 MB at cfg3) is bandwidth-, not FMA-bound), up to 2 right-hand sides per pass (E read
// once), coefficients staged in shared memory.
template <int SL>
__global__ void __launch_bounds__(32 * SL) extend2_kernel(const double* __restrict__ E, int64_t ng, int K,
                                                         const double* __restrict__ coef, int r0, int nr, int clamp,
                                                         double* __restrict__ ug, double* __restrict__ clampmax) {
  pdl_prologue();
  extern __shared__ double sc[];   // nr * K coefficients + 2 x SL x 32 partial sums
  for (int i = threadIdx.x; i < nr * K; i += blockDim.x) sc[i] = coef[(size_t)r0 * K + i];
  double* part = sc + nr * K;
  __syncthreads();
  const int gl = threadIdx.x & 31, sl = threadIdx.x >> 5;
  const int64_t g = (int64_t)blockIdx.x * 32 + gl;
  double s0 = 0.0, s1 = 0.0;
  if (g < ng) {
#pragma unroll 4
    for (int c = sl; c < K; c += SL) {
      const double e = __ldg(E + (size_t)c * ng + g);
      s0 = fma(e, sc[c], s0);
      if (nr > 1) s1 = fma(e, sc[K + c], s1);
    }
  }
  part[sl * 32 + gl] = s0;
  part[SL * 32 + sl * 32 + gl] = s1;
  __syncthreads();
  double neg = 0.0;   // how far below 0 the reconstructed density went (the clamp magnitude, R17)
  if (sl < nr && g < ng) {
    double t = part[sl * SL * 32 + gl];
    for (int q = 1; q < SL; ++q) t += part[sl * SL * 32 + q * 32 + gl];
    ug[(size_t)(r0 + sl) * ng + g] = clamp ? fmax(t, 0.0) : t;
    neg = fmax(-t, 0.0);
  }
  if (clampmax && sl < 2) {   // warp max, one order-preserving atomicMax per warp (max is order-independent)
    for (int o = 16; o; o >>= 1) neg = fmax(neg, __shfl_xor_sync(0xffffffffu, neg, o));
    if (gl == 0) atomicMax((unsigned long long*)clampmax, (unsigned long long)__double_as_longlong(neg) | 0x8000000000000000ull);
  }
}

// The BEP least-squares residual of a step, max over the nrhs (<= 2) right-hand sides of
// ||B C - g||_2 / ||g||_2.  With the factorisation B D = Q R (column equilibration D, CholeskyQR2) the
// least-squares solution is C = D R^{-1} Q^T g, so ||B C - g||^2 = ||g||^2 - ||Q^T g||^2 with
// Q^T g = (R D^{-1}) C: a K x K GEMV with the operator formed once per factorisation (rdinv_kernel)
// instead of another pass over B.  The subtraction costs the digits of the residual's own smallness
// (~1e-8 relative noise floor).  The norms: one block, fixed reduction order (deterministic).
__global__ void rdinv_kernel(const double* __restrict__ R, const double* __restrict__ D, int K, double* RD) {
  const size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (size_t)K * K) return;
  const int i = (int)(e / K), j = (int)(e % K);   // row-major (i, j) = R(i, j) / D(j), upper
  RD[e] = j >= i ? R[(size_t)j * K + i] / D[j] : 0.0;
}

constexpr int RES_T = 1024;
__global__ void __launch_bounds__(RES_T) lsq_resid_kernel(const double* __restrict__ z, int K,
                                                          const double* __restrict__ g, int64_t m, int nrhs,
                                                          double* out) {
  // (||Q^T g||^2, ||g||^2) per right-hand side; four independent chains per sum (the g stream is ~|γ_in|
  // loads per right-hand side in one block: latency, not bandwidth)
  double acc[4][4];
#pragma unroll
  for (int q = 0; q < 4; ++q) acc[q][0] = acc[q][1] = acc[q][2] = acc[q][3] = 0.0;
  for (int q = 0; q < nrhs; ++q) {
    for (int i = threadIdx.x; i < K; i += RES_T) acc[2 * q][0] = fma(z[q * K + i], z[q * K + i], acc[2 * q][0]);
    const double* gq = g + (size_t)q * m;
    int64_t i = threadIdx.x;
    for (; i + 3 * RES_T < m; i += 4 * RES_T) {
      const double a = gq[i], b = gq[i + RES_T], c = gq[i + 2 * RES_T], d = gq[i + 3 * RES_T];
      acc[2 * q + 1][0] = fma(a, a, acc[2 * q + 1][0]);
      acc[2 * q + 1][1] = fma(b, b, acc[2 * q + 1][1]);
      acc[2 * q + 1][2] = fma(c, c, acc[2 * q + 1][2]);
      acc[2 * q + 1][3] = fma(d, d, acc[2 * q + 1][3]);
    }
    for (; i < m; i += RES_T) acc[2 * q + 1][0] = fma(gq[i], gq[i], acc[2 * q + 1][0]);
  }
  __shared__ double red[4][RES_T / 32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int q = 0; q < 4; ++q) {
    double v = (acc[q][0] + acc[q][1]) + (acc[q][2] + acc[q][3]);
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) red[q][w] = v;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double s[4] = {0.0, 0.0, 0.0, 0.0};
    for (int q = 0; q < 4; ++q)
      for (int k = 0; k < RES_T / 32; ++k) s[q] += red[q][k];
    double res = 0.0;
    for (int q = 0; q < nrhs; ++q)
      if (s[2 * q + 1] > 0) res = fmax(res, sqrt(fmax(s[2 * q + 1] - s[2 * q], 0.0) / s[2 * q + 1]));
    out[0] = res;
  }
}

}  // namespace
cudaError_t lsq_cholesky(double* G, int K, int* dfail, cudaStream_t s);
namespace {

// one CholeskyQR pass: R = chol(AᵀA) (upper; 64 x 64-tiled Gram), out = A R⁻¹ (R⁻¹ by warp-parallel
// back substitution, then a tiled upper-triangular GEMM; out != A).  Same building blocks as the
// octant DD's distributed CholeskyQR2.
dpm_status chol_qr_pass(dpm_ctx* ctx, const double* A, int64_t m, int K, double* Rout, double* Ri_ws, double* out,
                        int* dfail, cudaStream_t s) {
  DPM_CUDA_TRY(ctx, lsq_gram(A, m, K, Rout, s));
  DPM_CUDA_TRY(ctx, lsq_cholesky(Rout, K, dfail, s));
  DPM_CUDA_TRY(ctx, lsq_mul_rinv(A, m, K, Rout, Ri_ws, out, s));
  return DPM_OK;
}

}  // namespace

template <bool TRANS>
__global__ void __launch_bounds__(256) gemm_tri_kernel(const double* __restrict__ A, int64_t m, int K,
                                                        const double* __restrict__ T, const double* __restrict__ scale,
                                                        double* __restrict__ Cm);
template <bool TRANS>
cudaError_t launch_gemm_tri(const double* A, int64_t m, int K, const double* T, const double* scale, double* C,
                            cudaStream_t s);

// ---- block-diagonal factorisation (octant path, bep_sym.cu): columns of different reflection parities are
// exactly orthogonal over the symmetric γ_in, so AᵀA is block-diagonal by parity class and CholeskyQR2,
// R^{-1}, M = D R^{-1} Q^T and R D^{-1} factor class by class (the 8 blocks ~1/8 of the Gram flops, ~1/64 of
// the Cholesky / R^{-1} work).  The classes run as parallel branches of the captured factorisation graph; M,
// R D^{-1} and the column scales are scattered back to the original column order, so lsq_apply /
// lsq_residual / dpm_boundary_lsq are unchanged.
__global__ void permute_cols_kernel(const double* __restrict__ B, int64_t m, const int32_t* __restrict__ perm,
                                    double* __restrict__ Bp) {
  const int j = blockIdx.y;
  const double* src = B + (size_t)perm[j] * m;
  double* dst = Bp + (size_t)j * m;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = src[i];
}
__global__ void scatter_rows_kernel(const double* __restrict__ Mp, int64_t m, const int32_t* __restrict__ perm,
                                    double* __restrict__ M) {
  const int j = blockIdx.y;
  const double* src = Mp + (size_t)j * m;
  double* dst = M + (size_t)perm[j] * m;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = src[i];
}
__global__ void scatter_block_kernel(const double* __restrict__ RDp, const double* __restrict__ Rp,
                                     const double* __restrict__ cs, const int32_t* __restrict__ perm, int Kp, int K,
                                     double* RD, double* colscale, double* dg) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= Kp * Kp) return;
  const int a = e / Kp, b = e - a * Kp;
  RD[(size_t)perm[a] * K + perm[b]] = RDp[e];
  if (a == b) {
    colscale[perm[a]] = cs[a];
    dg[a] = fabs(Rp[(size_t)a * Kp + a]);
  }
}
__global__ void vec_ratio_kernel(const double* d, int K, double* out) {
  double mx = 0, mn = INFINITY;
  for (int i = 0; i < K; ++i) {
    mx = fmax(mx, d[i]);
    mn = fmin(mn, d[i]);
  }
  *out = mx / mn;
}

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
  double* Riw = R2 + (size_t)K * K;
  int* dfail = (int*)(Riw + (size_t)K * K);
  double* dcond = (double*)(dfail + 4);
  if (!ctx->Mlsq) DPM_CUDA_TRY(ctx, cudaMalloc(&ctx->Mlsq, (size_t)m * K * sizeof(double)));
  if (!ctx->RDinv) DPM_CUDA_TRY(ctx, cudaMalloc(&ctx->RDinv, (size_t)K * K * sizeof(double)));
  // The factorisation is ~80 small dependent kernels at K ~ 250 (blocked Cholesky, blocked R^{-1}): captured
  // once per (context, B) into a CUDA graph and replayed (Step 4b rebuilds the BEP at every new dt).
  // DPM_FACTOR_GRAPH=0 launches them directly.
  static const bool use_graph = [] {
    const char* v = getenv("DPM_FACTOR_GRAPH");
    return !(v && atoi(v) == 0);
  }();
  const bool blocks = bep_sym_blocks(ctx, B, s);
  if (blocks) {
    if (!ctx->sym_Bp) DPM_CUDA_TRY(ctx, cudaMalloc(&ctx->sym_Bp, (size_t)m * K * sizeof(double)));
    if (!ctx->sym_tmp) DPM_CUDA_TRY(ctx, cudaMalloc(&ctx->sym_tmp, (size_t)m * K * sizeof(double)));
    if (!ctx->sym_dg) DPM_CUDA_TRY(ctx, cudaMalloc(&ctx->sym_dg, (size_t)2 * K * sizeof(double)));
    for (int p = 0; p < 8; ++p)
      if (!ctx->sym_streams[p]) DPM_CUDA_TRY(ctx, cudaStreamCreateWithFlags(&ctx->sym_streams[p], cudaStreamNonBlocking));
    for (int p = 0; p < 9; ++p)
      if (!ctx->sym_ev[p]) DPM_CUDA_TRY(ctx, cudaEventCreateWithFlags(&ctx->sym_ev[p], cudaEventDisableTiming));
  }
  auto enqueue_blocks = [&](cudaStream_t q) -> dpm_status {
    double* cs = ctx->sym_dg;      // column scales, class order
    double* dg = ctx->sym_dg + K;  // |diag R|, class order
    DPM_CUDA_TRY(ctx, cudaMemsetAsync(dfail, 0, sizeof(int), q));
    DPM_CUDA_TRY(ctx, cudaMemsetAsync(ctx->RDinv, 0, (size_t)K * K * sizeof(double), q));
    const unsigned gm = (unsigned)std::max<int64_t>(1, std::min<int64_t>((m + TB - 1) / TB, 64));
    DPM_COUNT_LAUNCH(1);
    permute_cols_kernel<<<dim3(gm, K), TB, 0, q>>>(B, m, ctx->sym_perm, ctx->sym_Bp);
    DPM_CUDA_TRY(ctx, cudaEventRecord(ctx->sym_ev[8], q));
    size_t roff = 0;
    for (int p = 0; p < 8; ++p) {
      const int o = ctx->sym_off[p], Kp = ctx->sym_off[p + 1] - o;
      if (Kp == 0) continue;
      cudaStream_t st = ctx->sym_streams[p];
      DPM_CUDA_TRY(ctx, cudaStreamWaitEvent(st, ctx->sym_ev[8], 0));
      double* Bpp = ctx->sym_Bp + (size_t)o * m;
      double* Qp = ctx->Q + (size_t)o * m;
      double* Tp = ctx->sym_tmp + (size_t)o * m;
      double *R1p = R1 + roff, *R2p = R2 + roff, *Riwp = Riw + roff, *Rp = ctx->R + roff;
      roff += (size_t)Kp * Kp;
      DPM_COUNT_LAUNCH(2);
      colnorm_kernel<<<Kp, TB, 0, st>>>(Bpp, m, cs + o);
      scale_cols_kernel<<<dim3(gm, Kp), TB, 0, st>>>(Bpp, m, Kp, cs + o, Qp);
      dpm_status r;
      if ((r = chol_qr_pass(ctx, Qp, m, Kp, R1p, Riwp, Tp, dfail, st)) != DPM_OK) return r;
      if ((r = chol_qr_pass(ctx, Tp, m, Kp, R2p, Riwp, Qp, dfail, st)) != DPM_OK) return r;
      DPM_COUNT_LAUNCH(1);
      trmm_kernel<<<(Kp * Kp + 255) / 256, 256, 0, st>>>(R2p, R1p, Rp, Kp);
      DPM_CUDA_TRY(ctx, lsq_rinv(Rp, Kp, R1p, st));
      DPM_CUDA_TRY(ctx, launch_gemm_tri<true>(Qp, m, Kp, R1p, cs + o, Bpp, st));   // M_p rows into Bpp
      DPM_COUNT_LAUNCH(3);
      rdinv_kernel<<<(unsigned)(((size_t)Kp * Kp + 255) / 256), 256, 0, st>>>(Rp, cs + o, Kp, R2p);
      scatter_rows_kernel<<<dim3(gm, Kp), TB, 0, st>>>(Bpp, m, ctx->sym_perm + o, ctx->Mlsq);
      scatter_block_kernel<<<(Kp * Kp + 255) / 256, 256, 0, st>>>(R2p, Rp, cs + o, ctx->sym_perm + o, Kp, K,
                                                                  ctx->RDinv, ctx->colscale, dg + o);
      DPM_CUDA_TRY(ctx, cudaEventRecord(ctx->sym_ev[p], st));
      DPM_CUDA_TRY(ctx, cudaStreamWaitEvent(q, ctx->sym_ev[p], 0));
    }
    DPM_COUNT_LAUNCH(1);
    vec_ratio_kernel<<<1, 1, 0, q>>>(dg, K, dcond);
    DPM_CUDA_TRY(ctx, cudaGetLastError());
    return DPM_OK;
  };
  auto enqueue = [&](cudaStream_t q) -> dpm_status {
    if (blocks) return enqueue_blocks(q);
    DPM_CUDA_TRY(ctx, cudaMemsetAsync(dfail, 0, sizeof(int), q));
    DPM_COUNT_LAUNCH(1);
    colnorm_kernel<<<K, TB, 0, q>>>(B, m, ctx->colscale);
    DPM_COUNT_LAUNCH(1);
    scale_cols_kernel<<<dim3((unsigned)std::max<int64_t>(1, std::min<int64_t>((m + TB - 1) / TB, 64)), K), TB, 0, q>>>(
        B, m, K, ctx->colscale, ctx->Q);
    dpm_status st;
    // CholeskyQR2 ping-pong: Q -> Mlsq (scratch until the operator is formed) -> Q
    if ((st = chol_qr_pass(ctx, ctx->Q, m, K, R1, Riw, ctx->Mlsq, dfail, q)) != DPM_OK) return st;
    if ((st = chol_qr_pass(ctx, ctx->Mlsq, m, K, R2, Riw, ctx->Q, dfail, q)) != DPM_OK) return st;
    DPM_COUNT_LAUNCH(1);
    trmm_kernel<<<(K * K + 255) / 256, 256, 0, q>>>(R2, R1, ctx->R, K);
    DPM_COUNT_LAUNCH(1);
    diag_ratio_kernel<<<1, 1, 0, q>>>(ctx->R, K, dcond);
    // apply operator M = D R^{-1} Q^T (K x |γ_in|): each LSQ solve is then one GEMV
    double* Ri = R1;   // R1 is free after the trmm
    DPM_CUDA_TRY(ctx, lsq_rinv(ctx->R, K, Ri, q));
    DPM_CUDA_TRY(ctx, launch_gemm_tri<true>(ctx->Q, m, K, Ri, ctx->colscale, ctx->Mlsq, q));
    // the residual operator R D^{-1} (row-major K x K) of the per-step LSQ residual (lsq_residual)
    DPM_COUNT_LAUNCH(1);
    rdinv_kernel<<<(unsigned)(((size_t)K * K + 255) / 256), 256, 0, q>>>(ctx->R, ctx->colscale, K, ctx->RDinv);
    DPM_CUDA_TRY(ctx, cudaGetLastError());
    return DPM_OK;
  };
  if (!use_graph) {
    dpm_status st = enqueue(s);
    if (st != DPM_OK) return st;
  } else {
    if (!ctx->fac_exec || ctx->fac_B != B || ctx->fac_K != K || ctx->fac_m != m || ctx->fac_blocks != (int)blocks) {
      if (ctx->fac_exec) cudaGraphExecDestroy(ctx->fac_exec);
      ctx->fac_exec = nullptr;
      if (!ctx->fac_stream) DPM_CUDA_TRY(ctx, cudaStreamCreateWithFlags(&ctx->fac_stream, cudaStreamNonBlocking));
      const long long l0 = (long long)g_dpm_launches.load();
      DPM_CUDA_TRY(ctx, cudaStreamBeginCapture(ctx->fac_stream, cudaStreamCaptureModeThreadLocal));
      dpm_status st = enqueue(ctx->fac_stream);
      cudaGraph_t graph = nullptr;
      const cudaError_t ec = cudaStreamEndCapture(ctx->fac_stream, &graph);
      ctx->fac_launches = (long long)g_dpm_launches.load() - l0;
      g_dpm_launches.fetch_sub(ctx->fac_launches);   // counted on every replay
      if (st != DPM_OK) {
        if (graph) cudaGraphDestroy(graph);
        return st;
      }
      if (ec != cudaSuccess) { ctx->err = std::string("factor graph capture: ") + cudaGetErrorString(ec); return DPM_ERR_CUDA; }
      const cudaError_t ei = cudaGraphInstantiate(&ctx->fac_exec, graph, 0);
      cudaGraphDestroy(graph);
      if (ei != cudaSuccess) { ctx->err = std::string("factor graph instantiate: ") + cudaGetErrorString(ei); return DPM_ERR_CUDA; }
      ctx->fac_B = B;
      ctx->fac_K = K;
      ctx->fac_m = m;
      ctx->fac_blocks = (int)blocks;
    }
    DPM_CUDA_TRY(ctx, cudaGraphLaunch(ctx->fac_exec, s));
    g_dpm_launches.fetch_add(ctx->fac_launches);
  }
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
                      cudaStream_t s, double* clampmax) {
  const int K = ctx->K;
  const int64_t m = ctx->counts[DPM_SET_GAMMA_IN], ng = ctx->counts[DPM_SET_GAMMA];
  launch_gemv(ctx->Mlsq, m, K, g, nrhs, coef, s);
  if (u_gamma) return lsq_extend(ctx->E, ng, K, coef, nrhs, clamp, u_gamma, s, clampmax);
  return cudaGetLastError();
}

// C = A T' (m x K, column-major, ld m) for A m x K column-major and a triangular K x K factor from T
// (column-major): TRANS = false: T' = T upper (C = A T; replaces the row-by-row solve A <- A R^{-1} with
// T = R^{-1}); TRANS = true: T' = T^T lower (C = A T^T, so C^T = T A^T: the LSQ operator
// M = D R^{-1} Q^T stored as its transpose, with the column scale D).  64 x 64 output tiles, 16-deep
// k panels, 4 x 4 outputs per thread; k panels outside the triangle are skipped.
template <bool TRANS>
__global__ void __launch_bounds__(256) gemm_tri_kernel(const double* __restrict__ A, int64_t m, int K,
                                                        const double* __restrict__ T, const double* __restrict__ scale,
                                                        double* __restrict__ Cm) {
  const int64_t i0 = (int64_t)blockIdx.x * 64;
  const int j0 = blockIdx.y * 64;
  __shared__ double sA[16][65], sT[16][65];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  double acc[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b] = 0.0;
  const int kbeg = TRANS ? j0 - (j0 % 16) : 0, kend = TRANS ? K : min(K, j0 + 64);
  for (int k0 = kbeg; k0 < kend; k0 += 16) {
    for (int e = threadIdx.x; e < 16 * 64; e += 256) {
      const int r = e & 63, kk = e >> 6;
      const int64_t i = i0 + r;
      const int k = k0 + kk;
      sA[kk][r] = (i < m && k < K) ? A[(size_t)k * m + i] : 0.0;
      if (TRANS) {   // T'(k, j) = T(j, k) for k >= j: consecutive j are consecutive in memory
        const int c = e & 63, kk2 = e >> 6;
        const int k2 = k0 + kk2, j = j0 + c;
        sT[kk2][c] = (k2 < K && j < K && k2 >= j) ? T[(size_t)k2 * K + j] : 0.0;
      } else {
        const int kk2 = e & 15, c = e >> 4;
        const int k2 = k0 + kk2, j = j0 + c;
        sT[kk2][c] = (k2 < K && j < K && k2 <= j) ? T[(size_t)j * K + k2] : 0.0;
      }
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < 16; ++kk) {
      double av[4], tv[4];
#pragma unroll
      for (int a = 0; a < 4; ++a) av[a] = sA[kk][ty + 16 * a];
#pragma unroll
      for (int b = 0; b < 4; ++b) tv[b] = sT[kk][tx + 16 * b];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b] = fma(av[a], tv[b], acc[a][b]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int64_t i = i0 + ty + 16 * a;
      const int j = j0 + tx + 16 * b;
      if (i < m && j < K) Cm[(size_t)j * m + i] = scale ? scale[j] * acc[a][b] : acc[a][b];
    }
}

// G(i, j) += Σ_{r in this block's rows} A(r, i) A(r, j) for the upper 64 x 64 tiles (i <= j tiles);
// A m x K column-major; 16-row panels, 4 x 4 outputs per thread, atomics over the row splits.
__global__ void __launch_bounds__(256) gram64_kernel(const double* __restrict__ A, int64_t m, int K, double* G,
                                                      int64_t rows_per_split) {
  const int bi = blockIdx.x * 64, bj = blockIdx.y * 64;
  if (bj < bi) return;
  const int64_t r0 = (int64_t)blockIdx.z * rows_per_split, r1 = min(m, r0 + rows_per_split);
  __shared__ double sa[16][65], sb[16][65];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  double acc[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b] = 0.0;
  for (int64_t rr = r0; rr < r1; rr += 16) {
    for (int e = threadIdx.x; e < 16 * 64; e += 256) {
      const int r = e & 15, c = e >> 4;
      const int64_t row = rr + r;
      const bool ok = row < r1;
      sa[r][c] = (ok && bi + c < K) ? A[(size_t)(bi + c) * m + row] : 0.0;
      sb[r][c] = (ok && bj + c < K) ? A[(size_t)(bj + c) * m + row] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      double av[4], bv[4];
#pragma unroll
      for (int a = 0; a < 4; ++a) av[a] = sa[r][ty + 16 * a];
#pragma unroll
      for (int b = 0; b < 4; ++b) bv[b] = sb[r][tx + 16 * b];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b] = fma(av[a], bv[b], acc[a][b]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int i = bi + ty + 16 * a, j = bj + tx + 16 * b;
      if (i < K && j < K && i <= j) G[(size_t)blockIdx.z * K * K + (size_t)j * K + i] = acc[a][b];   // split slice
    }
}

// R^{-1} by recursive doubling (DPM_RINV_DOUBLING, default): with the diagonal 32 x 32 tiles inverted,
// level s (= 32, 64, 128, ...) joins each pair of inverted diagonal blocks [P_1 B; 0 P_2] of size s:
//   inv = [P_1^{-1}, -P_1^{-1} B P_2^{-1}; 0, P_2^{-1}],
// as two launches of 32 x 32-tile products over all pairs at once (T = B X_22, then X_12 = -X_11 T; the
// triangular factors' zero tiles skipped).  log2(K/32) levels instead of K/32 dependent block diagonals.
// mode 0: T[i][j] = Σ_{k in blk2, k <= j} R[i][k] Ri[k][j]      (i in blk1, j in blk2)
// mode 1: Ri[i][j] = -Σ_{k in blk1, k >= i} Ri[i][k] T[k][j]
__global__ void __launch_bounds__(256) rinv_pair_kernel(const double* __restrict__ R, int K, int s, int mode,
                                                        double* __restrict__ Ri, double* __restrict__ T) {
  __shared__ double sa[RT][RT + 1], sb[RT][RT + 1];
  const int nt = s / RT;                       // tiles per block side
  const int pair = blockIdx.x / (nt * nt), tt = blockIdx.x % (nt * nt);
  const int ti = tt / nt, tj = tt % nt;
  const int r1 = 2 * pair * s, r2 = r1 + s;    // block 1 rows/cols [r1, r2), block 2 [r2, min(r2 + s, K))
  if (r2 >= K) return;
  const int e2 = min(r2 + s, K);
  const int i0 = r1 + ti * RT, j0 = r2 + tj * RT;
  if (j0 >= e2) return;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  double acc[4] = {0, 0, 0, 0};
  const int kb = mode == 0 ? r2 : i0, ke = mode == 0 ? min(j0 + RT, e2) : r2;
  for (int k0 = kb; k0 < ke; k0 += RT) {
    for (int q = ty; q < RT; q += 8) {
      const int ra = i0 + tx, ca = k0 + q;     // left factor (row ra, col ca)
      const int rb = k0 + tx, cb = j0 + q;     // right factor (row rb, col cb)
      double av, bv;
      if (mode == 0) {
        av = (ra < K && ca < K) ? R[(size_t)ca * K + ra] : 0.0;
        bv = (rb < e2 && cb < e2 && rb <= cb) ? Ri[(size_t)cb * K + rb] : 0.0;
      } else {
        av = (ca < r2 && ra <= ca) ? Ri[(size_t)ca * K + ra] : 0.0;
        bv = (rb < r2 && cb < e2) ? T[(size_t)cb * K + rb] : 0.0;
      }
      sa[tx][q] = av;
      sb[tx][q] = bv;
    }
    __syncthreads();
#pragma unroll 8
    for (int l = 0; l < RT; ++l) {
      const double bv = sb[l][tx];
#pragma unroll
      for (int u = 0; u < 4; ++u) acc[u] = fma(sa[ty + 8 * u][l], bv, acc[u]);
    }
    __syncthreads();
  }
  // stage the tile (row ty + 8u, col tx) and store with lanes over consecutive rows
#pragma unroll
  for (int u = 0; u < 4; ++u) sb[ty + 8 * u][tx] = acc[u];
  __syncthreads();
  for (int q = ty; q < RT; q += 8) {
    const int r = i0 + tx, c = j0 + q;
    if (r < r2 && c < e2) {
      if (mode == 0) T[(size_t)c * K + r] = sb[tx][q];
      else Ri[(size_t)c * K + r] = -sb[tx][q];
    }
  }
}

// R^{-1} (upper triangular, col-major; lower triangle of Ri zeroed) by the blocked kernels above
cudaError_t lsq_rinv(const double* R, int K, double* Ri, cudaStream_t s) {
  cudaError_t e = cudaMemsetAsync(Ri, 0, (size_t)K * K * sizeof(double), s);
  if (e != cudaSuccess) return e;
  const int nb = (K + RT - 1) / RT;
  DPM_COUNT_LAUNCH(1);
  rinv_diag_kernel<<<nb, RT, 0, s>>>(R, K, Ri);
  static const bool doubling = [] {
    const char* v = getenv("DPM_RINV_DOUBLING");
    return !(v && atoi(v) == 0);
  }();
  if (doubling) {
    if (nb == 1) return cudaGetLastError();
    double* T = nullptr;
    if ((e = cudaMallocAsync(&T, (size_t)K * K * sizeof(double), s)) != cudaSuccess) return e;
    for (int sz = RT; sz < K; sz *= 2) {
      const int pairs = (K + 2 * sz - 1) / (2 * sz), nt = sz / RT;
      const unsigned grid = (unsigned)(pairs * nt * nt);
      DPM_COUNT_LAUNCH(2);
      rinv_pair_kernel<<<grid, 256, 0, s>>>(R, K, sz, 0, Ri, T);
      rinv_pair_kernel<<<grid, 256, 0, s>>>(R, K, sz, 1, Ri, T);
    }
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    return cudaFreeAsync(T, s);
  }
  for (int d = 1; d < nb; ++d) {
    DPM_COUNT_LAUNCH(1);
    rinv_offdiag_kernel<<<nb - d, 256, 0, s>>>(R, K, d, Ri);
  }
  return cudaGetLastError();
}

// ---- building blocks shared with the octant DD (dd.cu): distributed CholeskyQR2 ----
cudaError_t lsq_mul_rinv(const double* A, int64_t m, int K, const double* R, double* Ri_ws, double* out,
                         cudaStream_t s) {
  cudaError_t e = lsq_rinv(R, K, Ri_ws, s);
  if (e != cudaSuccess || m == 0) return e;
  return launch_gemm_tri<false>(A, m, K, Ri_ws, nullptr, out, s);
}

// out = A T with T = an already inverted upper-triangular factor (tiled GEMM; out != A)
cudaError_t lsq_mul_upper(const double* A, int64_t m, int K, const double* T, double* out, cudaStream_t s) {
  if (m == 0) return cudaSuccess;
  return launch_gemm_tri<false>(A, m, K, T, nullptr, out, s);
}

// M = diag(scale) Ri Q^T (stored K x m row-major) from an already inverted Ri = R^{-1}
cudaError_t lsq_operator_from_rinv(const double* Ri, const double* Q, int64_t m, int K, const double* scale, double* M,
                                   cudaStream_t s) {
  if (m == 0) return cudaSuccess;
  return launch_gemm_tri<true>(Q, m, K, Ri, scale, M, s);
}

// ---- fp64 tensor-pipe (DMMA.m8n8k4) versions of the Gram and the triangular GEMMs (DPM_LSQ_DMMA, default) ----
// 64 x 64 output tile per CTA, 8 warps each owning 2 x 4 fragment tiles of 8 x 8 (rows 16 (w/2)..,
// columns 32 (w%2)..), k staged 32 at a time by 8-byte cp.async (row counts may be odd) into shared
// memory laid out so every fragment load hits each 8-byte bank pair twice.
__device__ __forceinline__ void dmma_884(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}
__device__ __forceinline__ void cpasync8(double* dst, const double* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"((unsigned)__cvta_generic_to_shared(dst)), "l"(src));
}
constexpr int DG_RK = 32, DG_PG = 36;   // Gram: rows per stage, pitch of the [column][row] stage (36 = 4 mod 16)

// G(i, j) += Σ_r A(r, i) A(r, j) over this CTA's row split, upper 64 x 64 tiles (atomics over splits)
__global__ void __launch_bounds__(256) gram_dmma_kernel(const double* __restrict__ A, int64_t m, int K, double* G,
                                                        int64_t rows_per_split) {
  const int bi = blockIdx.x * 64, bj = blockIdx.y * 64;
  if (bj < bi) return;
  extern __shared__ __align__(16) double gsm[];   // sI[2][64 DG_PG] | sJ[2][64 DG_PG]
  double (*sI)[64 * DG_PG] = reinterpret_cast<double (*)[64 * DG_PG]>(gsm);
  double (*sJ)[64 * DG_PG] = reinterpret_cast<double (*)[64 * DG_PG]>(gsm + 2 * 64 * DG_PG);
  const int64_t r0 = (int64_t)blockIdx.z * rows_per_split, r1 = min(m, r0 + rows_per_split);
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  const int wi = 16 * (w >> 1), wj = 32 * (w & 1);
  const bool diag = bi == bj;
  auto stage = [&](int buf, int64_t rr) {   // rows rr .. rr+31 of columns bi.., bj.. -> [col][row]
    for (int e = t; e < 64 * DG_RK; e += 256) {
      const int c = e >> 5, r = e & 31;
      const int64_t row = rr + r;
      double* di = &sI[buf][c * DG_PG + r];
      if (row < r1 && bi + c < K) cpasync8(di, A + (size_t)(bi + c) * m + row); else *di = 0.0;
      if (!diag) {
        double* dj = &sJ[buf][c * DG_PG + r];
        if (row < r1 && bj + c < K) cpasync8(dj, A + (size_t)(bj + c) * m + row); else *dj = 0.0;
      }
    }
    asm volatile("cp.async.commit_group;\n" ::);
  };
  double acc[2][4][2];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
  int buf = 0;
  if (r0 < r1) stage(0, r0);
  for (int64_t rr = r0; rr < r1; rr += DG_RK, buf ^= 1) {
    if (rr + DG_RK < r1) {
      stage(buf ^ 1, rr + DG_RK);
      asm volatile("cp.async.wait_group 1;\n" ::);
    } else {
      asm volatile("cp.async.wait_group 0;\n" ::);
    }
    __syncthreads();
    const double* XI = sI[buf];
    const double* XJ = diag ? sI[buf] : sJ[buf];
#pragma unroll
    for (int ks = 0; ks < DG_RK / 4; ++ks) {
      const int kr = 4 * ks + (lane & 3);
      double af[2], bf[4];
#pragma unroll
      for (int a = 0; a < 2; ++a) af[a] = XI[(wi + 8 * a + (lane >> 2)) * DG_PG + kr];   // A_frag[i][k] = A(k, i)
#pragma unroll
      for (int b = 0; b < 4; ++b) bf[b] = XJ[(wj + 8 * b + (lane >> 2)) * DG_PG + kr];   // B_frag[k][j] = A(k, j)
#pragma unroll
      for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) dmma_884(acc[a][b], af[a], bf[b]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int i = bi + wi + 8 * a + (lane >> 2), j = bj + wj + 8 * b + 2 * (lane & 3) + h;
        if (i < K && j < K && i <= j) G[(size_t)blockIdx.z * K * K + (size_t)j * K + i] = acc[a][b][h];
      }
}

// G[j][i] (i <= j) = Σ_z P[z][j][i] in slice order; the lower triangle is zero
__global__ void gram_sum_kernel(const double* __restrict__ P, int nsplit, int K, double* __restrict__ G) {
  const size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x, KK = (size_t)K * K;
  if (e >= KK) return;
  const int j = (int)(e / K), i = (int)(e % K);
  double s = 0.0;
  if (i <= j)
    for (int z = 0; z < nsplit; ++z) s += P[z * KK + e];
  G[e] = s;
}

constexpr int DT_RK = 32, DT_P = 72;   // tri-GEMM: k per stage, pitch of the [k][64] stages (72 = 8 mod 16)

// C = A T' (m x K column-major) with T' = T upper (TRANS = false) or T^T lower with the column scale
// (TRANS = true: the LSQ operator), as gemm_tri_kernel but on the fp64 tensor pipe
template <bool TRANS>
__global__ void __launch_bounds__(256) gemm_tri_dmma_kernel(const double* __restrict__ A, int64_t m, int K,
                                                            const double* __restrict__ T,
                                                            const double* __restrict__ scale, double* __restrict__ Cm) {
  extern __shared__ __align__(16) double tsm[];   // sA[2][DT_RK][DT_P] | sT[2][DT_RK][DT_P]
  double* sA = tsm;
  double* sT = tsm + 2 * DT_RK * DT_P;
  const int64_t r0 = (int64_t)blockIdx.x * 64;
  const int j0 = blockIdx.y * 64;
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  const int wr = 16 * (w >> 1), wj = 32 * (w & 1);
  const int kbeg = TRANS ? j0 : 0, kend = TRANS ? K : min(K, j0 + 64);
  auto stage = [&](int buf, int k0) {
    double* a = sA + buf * DT_RK * DT_P;
    double* tt = sT + buf * DT_RK * DT_P;
    for (int e = t; e < DT_RK * 64; e += 256) {
      const int kk = e >> 6, c = e & 63;
      const int k = k0 + kk;
      const int64_t r = r0 + c;
      if (r < m && k < K) cpasync8(a + kk * DT_P + c, A + (size_t)k * m + r); else a[kk * DT_P + c] = 0.0;
      const int j = j0 + c;
      const bool nz = k < K && j < K && (TRANS ? k >= j : k <= j);
      if (nz) cpasync8(tt + kk * DT_P + c, TRANS ? T + (size_t)k * K + j : T + (size_t)j * K + k);
      else tt[kk * DT_P + c] = 0.0;
    }
    asm volatile("cp.async.commit_group;\n" ::);
  };
  double acc[2][4][2];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
  int buf = 0;
  if (kbeg < kend) stage(0, kbeg);
  for (int k0 = kbeg; k0 < kend; k0 += DT_RK, buf ^= 1) {
    if (k0 + DT_RK < kend) {
      stage(buf ^ 1, k0 + DT_RK);
      asm volatile("cp.async.wait_group 1;\n" ::);
    } else {
      asm volatile("cp.async.wait_group 0;\n" ::);
    }
    __syncthreads();
    const double* a = sA + buf * DT_RK * DT_P;
    const double* tt = sT + buf * DT_RK * DT_P;
#pragma unroll
    for (int ks = 0; ks < DT_RK / 4; ++ks) {
      const int kk = 4 * ks + (lane & 3);
      double af[2], bf[4];
#pragma unroll
      for (int x = 0; x < 2; ++x) af[x] = a[kk * DT_P + wr + 8 * x + (lane >> 2)];   // A_frag[r][k] = A(r, k)
#pragma unroll
      for (int y = 0; y < 4; ++y) bf[y] = tt[kk * DT_P + wj + 8 * y + (lane >> 2)];  // B_frag[k][j] = T'(k, j)
#pragma unroll
      for (int x = 0; x < 2; ++x)
#pragma unroll
        for (int y = 0; y < 4; ++y) dmma_884(acc[x][y], af[x], bf[y]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int x = 0; x < 2; ++x)
#pragma unroll
    for (int y = 0; y < 4; ++y)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int64_t r = r0 + wr + 8 * x + (lane >> 2);
        const int j = j0 + wj + 8 * y + 2 * (lane & 3) + h;
        if (r < m && j < K) Cm[(size_t)j * m + r] = scale ? scale[j] * acc[x][y][h] : acc[x][y][h];
      }
}

// The same product with 128 x 64 output tiles (DPM_TRI_BM = 128, default): 8 warps of 32 x 32 (4 x 4
// fragment tiles), so every fragment load feeds 4 DMMAs instead of 2-4 and the T tile is re-read for half
// as many row tiles.  Stage pitches 132 / 68 (≡ 4 mod 16: each 8-byte bank pair hit twice per load).
constexpr int DT2_PA = 132, DT2_PT = 68;
template <bool TRANS>
__global__ void __launch_bounds__(256) gemm_tri_dmma2_kernel(const double* __restrict__ A, int64_t m, int K,
                                                             const double* __restrict__ T,
                                                             const double* __restrict__ scale, double* __restrict__ Cm) {
  extern __shared__ __align__(16) double tsm[];   // sA[2][DT_RK][DT2_PA] | sT[2][DT_RK][DT2_PT]
  double* sA = tsm;
  double* sT = tsm + 2 * DT_RK * DT2_PA;
  const int64_t r0 = (int64_t)blockIdx.x * 128;
  const int j0 = blockIdx.y * 64;
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  const int wr = 32 * (w >> 1), wj = 32 * (w & 1);
  const int kbeg = TRANS ? j0 : 0, kend = TRANS ? K : min(K, j0 + 64);
  auto stage = [&](int buf, int k0) {
    double* a = sA + buf * DT_RK * DT2_PA;
    double* tt = sT + buf * DT_RK * DT2_PT;
    for (int e = t; e < DT_RK * 128; e += 256) {
      const int kk = e >> 7, c = e & 127;
      const int k = k0 + kk;
      const int64_t r = r0 + c;
      if (r < m && k < K) cpasync8(a + kk * DT2_PA + c, A + (size_t)k * m + r); else a[kk * DT2_PA + c] = 0.0;
    }
    for (int e = t; e < DT_RK * 64; e += 256) {
      const int kk = e >> 6, c = e & 63;
      const int k = k0 + kk, j = j0 + c;
      const bool nz = k < K && j < K && (TRANS ? k >= j : k <= j);
      if (nz) cpasync8(tt + kk * DT2_PT + c, TRANS ? T + (size_t)k * K + j : T + (size_t)j * K + k);
      else tt[kk * DT2_PT + c] = 0.0;
    }
    asm volatile("cp.async.commit_group;\n" ::);
  };
  double acc[4][4][2];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
  int buf = 0;
  if (kbeg < kend) stage(0, kbeg);
  for (int k0 = kbeg; k0 < kend; k0 += DT_RK, buf ^= 1) {
    if (k0 + DT_RK < kend) {
      stage(buf ^ 1, k0 + DT_RK);
      asm volatile("cp.async.wait_group 1;\n" ::);
    } else {
      asm volatile("cp.async.wait_group 0;\n" ::);
    }
    __syncthreads();
    const double* a = sA + buf * DT_RK * DT2_PA;
    const double* tt = sT + buf * DT_RK * DT2_PT;
#pragma unroll
    for (int ks = 0; ks < DT_RK / 4; ++ks) {
      const int kk = 4 * ks + (lane & 3);
      double af[4], bf[4];
#pragma unroll
      for (int x = 0; x < 4; ++x) af[x] = a[kk * DT2_PA + wr + 8 * x + (lane >> 2)];
#pragma unroll
      for (int y = 0; y < 4; ++y) bf[y] = tt[kk * DT2_PT + wj + 8 * y + (lane >> 2)];
#pragma unroll
      for (int x = 0; x < 4; ++x)
#pragma unroll
        for (int y = 0; y < 4; ++y) dmma_884(acc[x][y], af[x], bf[y]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int x = 0; x < 4; ++x)
#pragma unroll
    for (int y = 0; y < 4; ++y)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int64_t r = r0 + wr + 8 * x + (lane >> 2);
        const int j = j0 + wj + 8 * y + 2 * (lane & 3) + h;
        if (r < m && j < K) Cm[(size_t)j * m + r] = scale ? scale[j] * acc[x][y][h] : acc[x][y][h];
      }
}

static bool lsq_dmma() {
  static const bool on = [] {
    const char* v = getenv("DPM_LSQ_DMMA");
    return !(v && atoi(v) == 0);
  }();
  return on;
}

template <bool TRANS>
cudaError_t launch_gemm_tri(const double* A, int64_t m, int K, const double* T, const double* scale, double* C,
                            cudaStream_t s) {
  const dim3 grid((unsigned)((m + 63) / 64), (K + 63) / 64);
  DPM_COUNT_LAUNCH(1);
  static const int bm = [] {
    const char* v = getenv("DPM_TRI_BM");
    return v && atoi(v) == 64 ? 64 : 128;
  }();
  if (lsq_dmma() && bm == 128 && K >= 384) {   // (small K: the 64-row tiles give more CTAs)
    const size_t smem = 2 * DT_RK * (DT2_PA + DT2_PT) * sizeof(double);
    cudaError_t e = cudaFuncSetAttribute(gemm_tri_dmma2_kernel<TRANS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
    gemm_tri_dmma2_kernel<TRANS><<<dim3((unsigned)((m + 127) / 128), (K + 63) / 64), 256, smem, s>>>(A, m, K, T, scale, C);
    return cudaGetLastError();
  }
  if (lsq_dmma()) {
    const size_t smem = 4 * DT_RK * DT_P * sizeof(double);
    cudaError_t e = cudaFuncSetAttribute(gemm_tri_dmma_kernel<TRANS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
    gemm_tri_dmma_kernel<TRANS><<<grid, 256, smem, s>>>(A, m, K, T, scale, C);
  } else {
    gemm_tri_kernel<TRANS><<<grid, 256, 0, s>>>(A, m, K, T, scale, C);
  }
  return cudaGetLastError();
}

// G = A^T A (upper triangle).  The row range is split over nsplit slices whose partial Grams are written
// to a stream-ordered workspace and summed in slice order (deterministic: no atomics).
cudaError_t lsq_gram(const double* A, int64_t m, int K, double* G, cudaStream_t s) {
  const int tiles = (K + 63) / 64;
  const int64_t upper = (int64_t)tiles * (tiles + 1) / 2;
  const int64_t target_split = std::max<int64_t>(1, (148 * 4) / upper);
  const int64_t rps = std::max<int64_t>(64, ((m + target_split - 1) / target_split + 15) / 16 * 16);
  const int nsplit = (int)std::max<int64_t>(1, (m + rps - 1) / rps);
  double* P = G;
  cudaError_t e;
  if (nsplit > 1) {
    if ((e = cudaMallocAsync(&P, (size_t)nsplit * K * K * sizeof(double), s)) != cudaSuccess) return e;
  } else if ((e = cudaMemsetAsync(G, 0, (size_t)K * K * sizeof(double), s)) != cudaSuccess) {   // lower triangle
    return e;
  }
  DPM_COUNT_LAUNCH(1);
  if (lsq_dmma()) {
    const size_t smem = 4 * 64 * DG_PG * sizeof(double);
    if ((e = cudaFuncSetAttribute(gram_dmma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)) != cudaSuccess)
      return e;
    gram_dmma_kernel<<<dim3(tiles, tiles, nsplit), 256, smem, s>>>(A, m, K, P, (rps + DG_RK - 1) / DG_RK * DG_RK);
  } else
    gram64_kernel<<<dim3(tiles, tiles, nsplit), 256, 0, s>>>(A, m, K, P, rps);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  if (nsplit > 1) {
    DPM_COUNT_LAUNCH(1);
    gram_sum_kernel<<<(unsigned)(((size_t)K * K + 255) / 256), 256, 0, s>>>(P, nsplit, K, G);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    return cudaFreeAsync(P, s);
  }
  return cudaSuccess;
}

cudaError_t lsq_cholesky(double* G, int K, int* dfail, cudaStream_t s) {
  for (int k0 = 0; k0 < K; k0 += CB) {
    DPM_COUNT_LAUNCH(1);
    chol_diag_kernel<<<1, 32, 0, s>>>(G, K, k0, dfail);
    const int rest = K - k0 - std::min(CB, K - k0);
    if (rest > 0) {
      DPM_COUNT_LAUNCH(2);
      chol_panel_kernel<<<(rest + CHOL_PW - 1) / CHOL_PW, 32 * CHOL_PW, 0, s>>>(G, K, k0);
      chol_update_kernel<<<dim3((rest + 15) / 16, (rest + 15) / 16), dim3(16, 16), 0, s>>>(G, K, k0);
    }
  }
  DPM_COUNT_LAUNCH(1);
  zero_lower_kernel<<<(unsigned)(((long)K * K + 255) / 256), 256, 0, s>>>(G, K);
  return cudaGetLastError();
}

cudaError_t lsq_trmm(const double* A, const double* B, double* C, int K, cudaStream_t s) {
  DPM_COUNT_LAUNCH(1);
  trmm_kernel<<<(K * K + 255) / 256, 256, 0, s>>>(A, B, C, K);
  return cudaGetLastError();
}

cudaError_t lsq_scale_cols(const double* B, int64_t m, int K, const double* scale, double* A, cudaStream_t s) {
  DPM_COUNT_LAUNCH(1);
  scale_cols_kernel<<<dim3((unsigned)std::max<int64_t>(1, std::min<int64_t>((m + TB - 1) / TB, 64)), K), TB, 0, s>>>(
      B, m, K, scale, A);
  return cudaGetLastError();
}

// M = diag(scale) R^{-1} Q^T (K x m row-major); Ri_ws: K x K workspace
cudaError_t lsq_build_operator(const double* R, const double* Q, int64_t m, int K, const double* scale, double* M,
                               double* Ri_ws, cudaStream_t s) {
  cudaError_t e = lsq_rinv(R, K, Ri_ws, s);
  if (e != cudaSuccess || m == 0) return e;
  return launch_gemm_tri<true>(Q, m, K, Ri_ws, scale, M, s);
}

cudaError_t lsq_gemv(const double* M, int64_t m, int K, const double* g, int nrhs, double* coef, cudaStream_t s) {
  launch_gemv(M, m, K, g, nrhs, coef, s);
  return cudaGetLastError();
}

cudaError_t lsq_extend(const double* E, int64_t ng, int K, const double* coef, int nrhs, int clamp, double* ug,
                       cudaStream_t s, double* clampmax) {
  for (int r = 0; r < nrhs; r += 2) {
    const int nr = std::min(2, nrhs - r);
    DPM_COUNT_LAUNCH(1);
    if (K >= 64) {
      const size_t smem = (size_t)(nr * K + 2 * 32 * 32) * sizeof(double);
      if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(extend2_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
      }
      launch_pdl(extend2_kernel<32>, (unsigned)((ng + 31) / 32), 1024, smem, s, E, ng, K, coef, r, nr, clamp, ug,
                 clampmax);
    } else {
      const size_t smem = (size_t)(nr * K + 2 * 8 * 32) * sizeof(double);
      launch_pdl(extend2_kernel<8>, (unsigned)((ng + 31) / 32), 256, smem, s, E, ng, K, coef, r, nr, clamp, ug,
                 clampmax);
    }
  }
  return cudaGetLastError();
}

cudaError_t lsq_residual(dpm_ctx* ctx, const double* coef, const double* g, int nrhs, double* zws, double* out,
                         cudaStream_t s) {
  if (nrhs < 1 || nrhs > 2 || !ctx->RDinv) return cudaErrorInvalidValue;
  const int K = ctx->K;
  launch_gemv(ctx->RDinv, K, K, coef, nrhs, zws, s);                      // z = R D^{-1} C = Q^T g
  DPM_COUNT_LAUNCH(1);
  lsq_resid_kernel<<<1, RES_T, 0, s>>>(zws, K, g, ctx->counts[DPM_SET_GAMMA_IN], nrhs, out);
  return cudaGetLastError();
}
