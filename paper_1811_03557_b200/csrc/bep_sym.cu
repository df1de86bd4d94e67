// NEXT-1: BEP columns on one octant of the grid, by reflection symmetry.
//
// A BEP column is u_c = AP(q_c), q_c = χ_{M-}(I/dt - Δ_h)[E_c] on the band, then
// Tr_γ u_c and B[:, c] = E_in[:, c] - u_c[γ_in].  When the grid and the point sets are symmetric under the
// three reflections x_a -> -x_a of the box (n even, centred domain: cfg1-cfg4, the paper's sphere tests)
// and every column E_c is even or odd under each reflection (the real spherical-harmonic bases are:
// Y_lm has parity (-1)^m / (-1)^(m+1) in x, ±1 in y, (-1)^(l+m) in z), then q_c and u_c have the same
// parities (the 7-point operator commutes with the reflections), and u_c is fixed by its values on the
// octant [0, m)^3, m = n/2 (0-based interior indices; the mirror of i is n-1-i).  On the octant, with
// s_a = ±1 the parity along axis a, the AP is
//     (I/dt + T_x,sx + T_y,sy + T_z,sz) u = q,   T_s = tridiag(-1, 2, -1)/h^2 on i = 0..m-1,
//     u_{-1} = 0 (Dirichlet box wall), u_m = s u_{m-1} (the mirror),
// and T_s is diagonalised by S_s[j][b] = sin(π k_b (j+1)/(n+1)) with k_b = 2b+1 (s = +1) or 2b+2 (s = -1)
// (the DST-I modes of that parity; eigenvalues λ_k of R26, Σ_j S_s[j][b]^2 = (n+1)/4).  So:
//   (1) scatter the octant's band values of q_c into boxes zeroed once (m^3 per column);
//   (2) forward transform along y and z (per x-plane: Q = S_y^T P S_z, two DMMA GEMMs in shared memory);
//   (3) per (b, c) spectral pencil, the tridiagonal solve along x with the mirror row (Thomas, in
//       registers), times the inverse-transform scale (4/(n+1))^2;
//   (4) inverse transform along y and z (P = S_y U S_z^T);
//   (5) gather γ / γ_in through the octant map with the parity signs.
// Per column: m^3 = n^3/8 points, two 2-GEMM plane passes and one tridiagonal pass over 8 n^3/8 bytes each,
// instead of three full n^3 passes.
// Odd n (the paper's N = 127 Test B mesh): the octant is [0, m)^3 with m = (n+1)/2 and its last index the
// centre node, which is its own mirror.  Along an axis of even parity the unknowns are i = 0..m-1 with
// u_m = u_{m-2} (centre row d u_c - 2 u_{c-1}/h^2), the modes k = 2b+1, and the forward sum over the full line
// counts the centre once: weight 1/2 on the centre entry (a separate forward table, S[2..3]); along an axis of
// odd parity the centre value is 0, the unknowns i = 0..m-2 (plain Dirichlet), the modes k = 2b+2, b < m-1 (the
// centre row and the mode b = m-1 of that table are zero).
// Columns that are not parity-definite, asymmetric sets or (n+1)/2 > 64 take the full path (dpm_bep_columns).  DPM_BEP_SYM=0 disables, DPM_BEP_SYM=2 makes a
// context the octant path does not apply to fail (cudaErrorNotSupported) instead of falling back.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <vector>

#include "dpm_internal.h"

namespace {

constexpr int SYM_NW = 4, SYM_NT = SYM_NW * 32;
constexpr int SYM_MMAX = 64;

__device__ __forceinline__ void dmma884(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

template <int MP>
struct SymGeo {
  static constexpr int LD = MP + 4;                 // ≡ 4 mod 16 doubles: conflict-free B fragments
  static constexpr int RT = MP / 8, CF = MP / 8, KS = MP / 4;
  static constexpr int RF = (RT + SYM_NW - 1) / SYM_NW;
};

__device__ __forceinline__ void cp_async16(unsigned saddr, const double* g) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(saddr), "l"(g));
}
__device__ __forceinline__ void cp_async8(unsigned saddr, const double* g) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(saddr), "l"(g));
}

// A fragments of A[r][k] = S[k][r] (TRANS) or S[r][k] for this warp's row tiles, S the zero-padded
// MP x MP table
template <int MP>
__device__ __forceinline__ void sym_afrag(const double* __restrict__ S, bool trans,
                                          double (&A)[SymGeo<MP>::RF][SymGeo<MP>::KS]) {
  using G = SymGeo<MP>;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int f = 0; f < G::RF; ++f) {
    const int rt = warp * G::RF + f, row = rt * 8 + (lane >> 2);
#pragma unroll
    for (int ks = 0; ks < G::KS; ++ks) {
      const int kr = ks * 4 + (lane & 3);
      A[f][ks] = rt < G::RT ? __ldg(trans ? S + kr * MP + row : S + row * MP + kr) : 0.0;
    }
  }
}

// Y^T <- A X over MP x MP tiles in shared memory (X[k][col] at k*LD + col; the result D[row][col] is
// written to Y[col*LD + row]), A in registers (sym_afrag)
template <int MP>
__device__ __forceinline__ void sym_gemm(const double (&A)[SymGeo<MP>::RF][SymGeo<MP>::KS], const double* X, double* Y) {
  using G = SymGeo<MP>;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (warp * G::RF >= G::RT) return;
  double acc[G::RF][G::CF][2];
#pragma unroll
  for (int f = 0; f < G::RF; ++f)
#pragma unroll
    for (int c = 0; c < G::CF; ++c) acc[f][c][0] = acc[f][c][1] = 0.0;
#pragma unroll
  for (int ks = 0; ks < G::KS; ++ks) {
    const int kr = ks * 4 + (lane & 3);
    double b[G::CF];
#pragma unroll
    for (int c = 0; c < G::CF; ++c) b[c] = X[kr * G::LD + c * 8 + (lane >> 2)];
#pragma unroll
    for (int f = 0; f < G::RF; ++f)
#pragma unroll
      for (int c = 0; c < G::CF; ++c) dmma884(acc[f][c], A[f][ks], b[c]);
  }
#pragma unroll
  for (int f = 0; f < G::RF; ++f) {
    const int row = (warp * G::RF + f) * 8 + (lane >> 2);
#pragma unroll
    for (int c = 0; c < G::CF; ++c) {
      const int col = c * 8 + 2 * (lane & 3);
      Y[col * G::LD + row] = acc[f][c][0];
      Y[(col + 1) * G::LD + row] = acc[f][c][1];
    }
  }
}

// (2) / (4): per x-plane (column cc, plane i) of the m^3 octant boxes: forward Q = S_y^T P S_z, inverse
// P = S_y Q S_z^T (S_y, S_z the tables of the column's y / z parities, par bits 1 / 2).  Persistent CTAs over
// contiguous ranges of planes (a column's 64 planes share their tables: the A fragments stay in registers
// and are reloaded when the parity class changes); the next plane streams in by cp.async under the GEMMs.
template <int MP, bool FWD>
__global__ void __launch_bounds__(SYM_NT, 2) sym_yz_kernel(const double* in, double* out, int ncols, int m,
                                                           const uint8_t* __restrict__ par,
                                                           const double* __restrict__ S) {
  using G = SymGeo<MP>;
  extern __shared__ __align__(16) double sh[];
  double* Y = sh + 2 * MP * G::LD;
  if (m < MP) {   // rows / columns >= m stay zero (m = MP: every entry read is loaded or written first)
    for (int e = threadIdx.x; e < 3 * MP * G::LD; e += SYM_NT) sh[e] = 0.0;
    __syncthreads();
  }
  const long m2 = (long)m * m, nplanes = (long)ncols * m;
  const long per = (nplanes + gridDim.x - 1) / gridDim.x;
  const long p0 = blockIdx.x * per, p1 = min(nplanes, p0 + per);
  if (p0 >= p1) return;
  const unsigned sbase = (unsigned)__cvta_generic_to_shared(sh);
  const bool v2 = (m & 1) == 0;
  auto issue = [&](long p, int buf) {
    const double* src = in + p * m2;
    const unsigned sb = sbase + 8u * (unsigned)(buf * MP * G::LD);
    if (v2) {
      const int h = m / 2;
      for (int e = threadIdx.x; e < m * h; e += SYM_NT) {
        const int j = e / h, k = 2 * (e - j * h);
        cp_async16(sb + 8u * (unsigned)(j * G::LD + k), src + j * m + k);
      }
    } else {
      for (int e = threadIdx.x; e < m * m; e += SYM_NT) {
        const int j = e / m, k = e - j * m;
        cp_async8(sb + 8u * (unsigned)(j * G::LD + k), src + e);
      }
    }
    asm volatile("cp.async.commit_group;\n" ::);
  };
  issue(p0, 0);
  double A1[G::RF][G::KS], A2[G::RF][G::KS];
  int cls = -1;
  for (long p = p0; p < p1; ++p) {
    const int buf = (int)((p - p0) & 1);
    double* X = sh + buf * MP * G::LD;
    if (p + 1 < p1) issue(p + 1, buf ^ 1);
    else asm volatile("cp.async.commit_group;\n" ::);
    const int pr = par[p / m] & 6;
    if (pr != cls) {
      sym_afrag<MP>(S + ((FWD ? 2 : 0) + ((pr >> 1) & 1)) * MP * MP, FWD, A1);   // [0,1] inverse, [2,3] forward
      sym_afrag<MP>(S + ((FWD ? 2 : 0) + ((pr >> 2) & 1)) * MP * MP, FWD, A2);
      cls = pr;
    }
    asm volatile("cp.async.wait_group 1;\n" ::);
    __syncthreads();
    sym_gemm<MP>(A1, X, Y);
    __syncthreads();
    sym_gemm<MP>(A2, Y, X);
    __syncthreads();
    double* dst = out + p * m2;
    for (int e = threadIdx.x; e < m * MP; e += SYM_NT) {
      const int j = e / MP, k = e % MP;
      if (k < m) dst[j * m + k] = X[j * G::LD + k];
    }
    __syncthreads();
  }
}

// (3a): LU factors of the x tridiagonal of every spectral pencil (w = b*m + c) of every y/z parity class q:
// den_i = d - h2i e_{i-1}, r_i = 1/den_i, e_i = h2i r_i (i < m-1), and the last row's r for both x parities
// (u_m = +u_{m-1}: d - h2i; u_m = -u_{m-1}: d + h2i; odd n: the centre row d with -2 h2i below the diagonal
// for the even parity, and 0 for the odd parity, whose centre value is 0).  They depend on Δt and the geometry
// only, not on the column: built once per Δt, read by every column of the class.
__global__ void sym_lu_kernel(int m, int MP, int odd, const double* __restrict__ lamr, double inv_dt, double h2i,
                              double* R, double* Ef, double* Rl) {
  const long m2 = (long)m * m;
  const long id = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (id >= 4 * m2) return;
  const int q = (int)(id / m2), w = (int)(id - q * m2), b = w / m, c = w - b * m;
  const double d = ((inv_dt + lamr[(q & 1) * MP + b]) + lamr[((q >> 1) & 1) * MP + c]) + 2.0 * h2i;
  double e = 0.0;
  for (int i = 0; i < m - 1; ++i) {
    const double r = 1.0 / (d - h2i * e);
    e = h2i * r;
    R[((long)q * m + i) * m2 + w] = r;
    Ef[((long)q * m + i) * m2 + w] = e;
  }
  Rl[((long)q * 2 + 0) * m2 + w] = odd ? 1.0 / (d - 2.0 * h2i * e) : 1.0 / ((d - h2i) - h2i * e);
  Rl[((long)q * 2 + 1) * m2 + w] = odd ? 0.0 : 1.0 / ((d + h2i) - h2i * e);
}

// (3b): per spectral pencil (column cc, w = b*m + c): (1/dt + λ_b + λ_c + T_x,sx) v = q along x with the
// factors of (3a), then v *= scale.  The right-hand side in registers, the factors streamed (L2-resident).
template <int MP, bool EXACT>
__global__ void __launch_bounds__(SYM_NT) sym_x_kernel(double* u, int ncols, int m_rt, const uint8_t* __restrict__ par,
                                                       const double* __restrict__ R, const double* __restrict__ Ef,
                                                       const double* __restrict__ Rl, double h2i, double scale,
                                                       double lm_even) {
  const int m = EXACT ? MP : m_rt;
  const long m2 = (long)m * m, total = (long)ncols * m2;
  const long id = (long)blockIdx.x * SYM_NT + threadIdx.x;
  if (id >= total) return;
  const int cc = (int)(id / m2);
  const int w = (int)(id - (long)cc * m2);
  const int pr = par[cc], q = (pr >> 1) & 3;
  double* col = u + (long)cc * m2 * m + w;
  const double* Rq = R + (long)q * m * m2 + w;
  const double* Eq = Ef + (long)q * m * m2 + w;
  double g[MP];
#pragma unroll
  for (int i = 0; i < MP; ++i) g[i] = i < m ? col[(long)i * m2] : 0.0;
  const double rl = __ldg(Rl + ((long)q * 2 + (pr & 1)) * m2 + w);
  const double hl = (pr & 1) ? h2i : lm_even * h2i;   // last row's subdiagonal (odd n, even parity: 2/h^2)
  double gprev = 0.0, next = 0.0;
#pragma unroll
  for (int i = 0; i < MP; ++i) {
    if (i < m - 1) {
      gprev = (g[i] + h2i * gprev) * __ldg(Rq + (long)i * m2);
      g[i] = gprev;
    } else if (i == m - 1) {
      next = (g[i] + hl * gprev) * rl;
      col[(long)i * m2] = next * scale;
    }
  }
#pragma unroll
  for (int i = MP - 2; i >= 0; --i) {
    if (i < m - 1) {
      next = g[i] + __ldg(Eq + (long)i * m2) * next;
      col[(long)i * m2] = next * scale;
    }
  }
}

// (5): PgE = Tr_γ u, B = E_in - Tr_γin u through the octant map: gidx[r] = octant index | reflection bits << 24
__global__ void sym_gather_kernel(const double* __restrict__ U, long m3, const int32_t* __restrict__ gidx, long ng,
                                  long ngin, const int32_t* __restrict__ gin_pos, const double* __restrict__ E,
                                  int c0, int cout0, const uint8_t* __restrict__ par, double* PgE, double* B) {
  const int cc = blockIdx.y;
  const double* Uc = U + (long)cc * m3;
  const int pr = par[cc];
  const int col = c0 + cc - cout0;
  for (long r = blockIdx.x * (long)blockDim.x + threadIdx.x; r < ng + ngin; r += (long)gridDim.x * blockDim.x) {
    const int e = gidx[r];
    double v = Uc[e & 0xFFFFFF];
    if (__popc((e >> 24) & pr) & 1) v = -v;
    if (r < ng) {
      if (PgE) PgE[(long)col * ng + r] = v;
    } else if (B) {
      const long i = r - ng;
      B[(long)col * ngin + i] = E[(long)(c0 + cc) * ng + gin_pos[i]] - v;
    }
  }
}

// parity sums of every column of E: out[c] = {Σ E^2, Σ (E - E∘mirror_a)^2 (a = x, y, z), Σ (E + E∘mirror_a)^2}
__global__ void sym_parity_kernel(const double* __restrict__ E, long ng, const int32_t* __restrict__ mir, int K,
                                  double* out) {
  __shared__ double red[7][256];
  const int c = blockIdx.x;
  const double* Ec = E + (long)c * ng;
  double s[7] = {0, 0, 0, 0, 0, 0, 0};
  for (long r = threadIdx.x; r < ng; r += blockDim.x) {
    const double v = Ec[r];
    s[0] += v * v;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const double w = Ec[mir[a * ng + r]];
      s[1 + a] += (v - w) * (v - w);
      s[4 + a] += (v + w) * (v + w);
    }
  }
#pragma unroll
  for (int q = 0; q < 7; ++q) red[q][threadIdx.x] = s[q];
  __syncthreads();
  for (int st = 128; st > 0; st >>= 1) {
    if (threadIdx.x < st)
#pragma unroll
      for (int q = 0; q < 7; ++q) red[q][threadIdx.x] += red[q][threadIdx.x + st];
    __syncthreads();
  }
  if (threadIdx.x < 7) out[(long)c * 7 + threadIdx.x] = red[threadIdx.x][0];
}

// does every column of a BEP matrix B (|γ_in| x K, column-major) have the parity recorded for it?  flag = 1
// if some column is off by more than 1e-10 (relative, 2-norm) from it under some reflection
__global__ void sym_check_kernel(const double* __restrict__ B, long m, const int32_t* __restrict__ mir,
                                 const uint8_t* __restrict__ par, int* flag) {
  __shared__ double red[4][256];
  const int c = blockIdx.x, pr = par[c];
  const double* Bc = B + (long)c * m;
  double s[4] = {0, 0, 0, 0};
  for (long r = threadIdx.x; r < m; r += blockDim.x) {
    const double v = Bc[r];
    s[0] += v * v;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const double w = Bc[mir[a * m + r]], d = ((pr >> a) & 1) ? v + w : v - w;
      s[1 + a] += d * d;
    }
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) red[q][threadIdx.x] = s[q];
  __syncthreads();
  for (int st = 128; st > 0; st >>= 1) {
    if (threadIdx.x < st)
#pragma unroll
      for (int q = 0; q < 4; ++q) red[q][threadIdx.x] += red[q][threadIdx.x + st];
    __syncthreads();
  }
  if (threadIdx.x == 0)
    for (int a = 0; a < 3; ++a)
      if (!(red[1 + a][0] <= 1e-20 * red[0][0])) atomicExch(flag, 1);
}

template <typename T>
cudaError_t upload(T** dst, const std::vector<T>& v) {
  cudaError_t e = cudaMalloc(dst, std::max<size_t>(1, v.size()) * sizeof(T));
  if (e != cudaSuccess) return e;
  return v.empty() ? cudaSuccess : cudaMemcpy(*dst, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice);
}

int sym_mp(int m) { return m <= 8 ? 8 : m <= 16 ? 16 : m <= 32 ? 32 : 64; }

// octant sine tables S[0,1] (inverse) / S[2,3] (forward, half weight on the centre entry for odd n) of the
// even / odd parity, zero-padded to MP x MP, and their eigenvalues lam[2][MP]
void sym_tables(int n, double h, std::vector<double>& S, std::vector<double>& lam) {
  const int m = (n + 1) / 2, MP = sym_mp(m);
  const bool odd = n & 1;
  S.assign(4 * (size_t)MP * MP, 0.0);
  lam.assign(2 * MP, 0.0);
  const long per = 2L * (n + 1);
  for (int s = 0; s < 2; ++s)
    for (int b = 0; b < m; ++b) {
      const long k = 2L * b + 1 + s;
      for (int j = 0; j < m; ++j) {
        double v = std::sin(M_PI * (double)((k * (j + 1)) % per) / (n + 1));
        if (odd && s == 1 && (j == m - 1 || b == m - 1)) v = 0.0;   // sin(k π/2), k even / the mode k = n+1
        S[((size_t)s * MP + j) * MP + b] = v;
        S[((size_t)(2 + s) * MP + j) * MP + b] = odd && j == m - 1 ? 0.5 * v : v;
      }
      const double sk = std::sin((double)k * M_PI / (2.0 * (n + 1)));
      lam[s * MP + b] = (4.0 / (h * h)) * sk * sk;
    }
}

// Decide once per context whether the octant path applies and build its tables (host sync: first call only).
cudaError_t sym_prepare(dpm_ctx* ctx) {
  ctx->sym = -1;
  const char* env = getenv("DPM_BEP_SYM");
  if (env && atoi(env) == 0) return cudaSuccess;
  const int n = ctx->n;
  const int m = (n + 1) / 2;   // odd n: the last octant index is the centre node (its own mirror)
  const bool odd = n & 1;
  if (m > SYM_MMAX || m < 2 || !ctx->E || ctx->dd == 1 || ctx->K == 0) return cudaSuccess;
  const long nn = (long)n * n, n3 = nn * n;
  // the sets the potential RHS and the traces read: γ (gmap), the band, M+, γ_in
  const int sets[4] = {DPM_SET_GAMMA, DPM_SET_BAND, DPM_SET_MPLUS, DPM_SET_GAMMA_IN};
  std::vector<int64_t> L[4];
  cudaError_t e;
  for (int q = 0; q < 4; ++q) {
    L[q].resize(ctx->counts[sets[q]]);
    if (!L[q].empty() &&
        (e = cudaMemcpy(L[q].data(), ctx->lists[sets[q]], L[q].size() * 8, cudaMemcpyDeviceToHost)) != cudaSuccess)
      return e;
  }
  auto mirror = [&](int64_t p, int a) -> int64_t {
    const int i = (int)(p / nn), j = (int)((p / n) % n), k = (int)(p % n);
    if (a == 0) return ((int64_t)(n - 1 - i) * n + j) * n + k;
    if (a == 1) return ((int64_t)i * n + (n - 1 - j)) * n + k;
    return ((int64_t)i * n + j) * n + (n - 1 - k);
  };
  std::vector<uint8_t> in(n3);
  for (int q = 0; q < 4; ++q) {
    std::fill(in.begin(), in.end(), 0);
    for (int64_t p : L[q]) in[p] = 1;
    for (int64_t p : L[q])
      for (int a = 0; a < 3; ++a)
        if (!in[mirror(p, a)]) return cudaSuccess;   // not reflection-symmetric: full path
  }
  const std::vector<int64_t>& gam = L[0];
  const long ng = (long)gam.size(), ngin = (long)L[3].size();
  std::vector<int32_t> gpos(n3, -1);
  for (long r = 0; r < ng; ++r) gpos[gam[r]] = (int32_t)r;
  std::vector<int32_t> mir(3 * ng);
  for (int a = 0; a < 3; ++a)
    for (long r = 0; r < ng; ++r) mir[a * ng + r] = gpos[mirror(gam[r], a)];
  // parity of every column of E
  int32_t* dmir = nullptr;
  double* dsum = nullptr;
  const int K = ctx->K;
  if ((e = upload(&dmir, mir)) != cudaSuccess) return e;
  if ((e = cudaMalloc(&dsum, (size_t)K * 7 * sizeof(double))) != cudaSuccess) { cudaFree(dmir); return e; }
  DPM_COUNT_LAUNCH(1);
  sym_parity_kernel<<<K, 256>>>(ctx->E, ng, dmir, K, dsum);
  std::vector<double> sums((size_t)K * 7);
  e = cudaGetLastError();
  if (e == cudaSuccess) e = cudaMemcpy(sums.data(), dsum, sums.size() * 8, cudaMemcpyDeviceToHost);
  cudaFree(dmir);
  cudaFree(dsum);
  if (e != cudaSuccess) return e;
  std::vector<uint8_t> par(K);
  constexpr double tol = 1e-20;   // squared relative: a column within 1e-10 of even / odd
  for (int c = 0; c < K; ++c) {
    const double* s = &sums[(size_t)c * 7];
    uint8_t p = 0;
    for (int a = 0; a < 3; ++a) {
      if (s[1 + a] <= tol * s[0]) continue;          // even
      if (s[4 + a] <= tol * s[0]) { p |= 1 << a; continue; }   // odd
      return cudaSuccess;                             // not parity-definite: full path
    }
    par[c] = p;
  }
  // octant band list, γ / γ_in octant map, sine tables, reduced eigenvalues
  std::vector<int64_t> olist;
  std::vector<int32_t> odst;
  for (int64_t p : L[1]) {
    const int i = (int)(p / nn), j = (int)((p / n) % n), k = (int)(p % n);
    if (i < m && j < m && k < m) {
      olist.push_back(p);
      odst.push_back((int32_t)(((long)i * m + j) * m + k));
    }
  }
  auto octant = [&](int64_t p) -> int32_t {
    int i = (int)(p / nn), j = (int)((p / n) % n), k = (int)(p % n), bits = 0;
    if (i >= m) { i = n - 1 - i; bits |= 1; }
    if (j >= m) { j = n - 1 - j; bits |= 2; }
    if (k >= m) { k = n - 1 - k; bits |= 4; }
    return (int32_t)((((long)i * m + j) * m + k) | ((long)bits << 24));
  };
  std::vector<int32_t> gidx(ng + ngin);
  for (long r = 0; r < ng; ++r) gidx[r] = octant(gam[r]);
  for (long r = 0; r < ngin; ++r) gidx[ng + r] = octant(L[3][r]);
  const int MP = sym_mp(m);
  std::vector<double> S, lam;
  sym_tables(n, ctx->h, S, lam);
  if ((e = upload(&ctx->sym_list, olist)) != cudaSuccess) return e;
  if ((e = upload(&ctx->sym_dst, odst)) != cudaSuccess) return e;
  if ((e = upload(&ctx->sym_gidx, gidx)) != cudaSuccess) return e;
  if ((e = upload(&ctx->sym_par, par)) != cudaSuccess) return e;
  if ((e = upload(&ctx->sym_S, S)) != cudaSuccess) return e;
  if ((e = upload(&ctx->sym_lam, lam)) != cudaSuccess) return e;
  {   // LU factors of the x tridiagonals (sym_lu_kernel): R, E [4][m][m^2] and the last rows [4][2][m^2]
    const size_t m2 = (size_t)m * m;
    if ((e = cudaMalloc(&ctx->sym_R, (8 * m2 * m + 8 * m2) * sizeof(double))) != cudaSuccess) return e;
    ctx->sym_lu_dt = 0.0;
  }
  {   // columns grouped by parity class (stable): the block-diagonal BEP factorisation (lsq_factor)
    std::vector<int32_t> perm;
    for (int cl = 0; cl < 8; ++cl) {
      ctx->sym_off[cl] = (int)perm.size();
      for (int c = 0; c < K; ++c)
        if (par[c] == cl) perm.push_back(c);
    }
    ctx->sym_off[8] = K;
    std::vector<int32_t> ginpos(n3, -1), mirin(3 * ngin);
    for (long r = 0; r < ngin; ++r) ginpos[L[3][r]] = (int32_t)r;
    for (int a = 0; a < 3; ++a)
      for (long r = 0; r < ngin; ++r) mirin[a * ngin + r] = ginpos[mirror(L[3][r], a)];
    if ((e = upload(&ctx->sym_perm, perm)) != cudaSuccess) return e;
    if ((e = upload(&ctx->sym_mirin, mirin)) != cudaSuccess) return e;
  }
  ctx->sym_nlist = (int64_t)olist.size();
  ctx->sym_m = m;
  ctx->sym = 1;
  return cudaSuccess;
}

// the octant operator a solve runs on: tables, LU factor storage, and when to (re)build the factors
struct SymOp {
  int n, m;
  double h, dt;
  const double* S;
  const double* lam;
  double* R;
  bool build_lu;   // launch sym_lu_kernel before the solve
};

template <int MP>
cudaError_t sym_solve(const SymOp& op, const double* q, double* u, int nc, const uint8_t* par, cudaStream_t s) {
  const int m = op.m, n = op.n;
  const long m2 = (long)m * m;
  constexpr size_t smem_yz = 3 * (size_t)MP * SymGeo<MP>::LD * sizeof(double);
  cudaFuncSetAttribute(sym_yz_kernel<MP, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_yz);
  cudaFuncSetAttribute(sym_yz_kernel<MP, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_yz);
  const long planes = (long)nc * m;
  const int grid_yz = (int)std::min<long>(planes, 148L * 2);
  const long pencils = (long)nc * m2;
  const double h2i = 1.0 / (op.h * op.h), scale = (4.0 / (n + 1)) * (4.0 / (n + 1));
  const double lm = (n & 1) ? 2.0 : 1.0;
  if (op.build_lu) {   // (3a) once per Δt
    DPM_COUNT_LAUNCH(1);
    sym_lu_kernel<<<(unsigned)((4 * m2 + 127) / 128), 128, 0, s>>>(m, MP, n & 1, op.lam, 1.0 / op.dt, h2i, op.R,
                                                                   op.R + 4 * m2 * m, op.R + 8 * m2 * m);
  }
  const double* R = op.R;
  DPM_COUNT_LAUNCH(3);
  sym_yz_kernel<MP, true><<<grid_yz, SYM_NT, smem_yz, s>>>(q, u, nc, m, par, op.S);
  const unsigned gx = (unsigned)((pencils + SYM_NT - 1) / SYM_NT);
  if (m == MP)
    sym_x_kernel<MP, true><<<gx, SYM_NT, 0, s>>>(u, nc, m, par, R, R + 4 * m2 * m, R + 8 * m2 * m, h2i, scale, lm);
  else
    sym_x_kernel<MP, false><<<gx, SYM_NT, 0, s>>>(u, nc, m, par, R, R + 4 * m2 * m, R + 8 * m2 * m, h2i, scale, lm);
  sym_yz_kernel<MP, false><<<grid_yz, SYM_NT, smem_yz, s>>>(u, u, nc, m, par, op.S);
  return cudaGetLastError();
}

cudaError_t sym_solve_mp(const SymOp& op, const double* q, double* u, int nc, const uint8_t* par, cudaStream_t s) {
  switch (sym_mp(op.m)) {
    case 8: return sym_solve<8>(op, q, u, nc, par, s);
    case 16: return sym_solve<16>(op, q, u, nc, par, s);
    case 32: return sym_solve<32>(op, q, u, nc, par, s);
    default: return sym_solve<64>(op, q, u, nc, par, s);
  }
}

// ---- parity-split AP solve of dense boxes (octsplit_solve) ---------------------------------------------------
// fold: the 8 parity components of every field on the octant, Q[(f*8 + p)][i][j][k] =
// (1/8) Σ_σ (-1)^{popcount(p & σ)} q_f(σ(i, j, k)), σ the 8 reflections (bit a: axis a mirrored, i -> n-1-i; at
// the centre node of an odd n the mirror is the node itself and the odd components come out exactly 0)
__global__ void osp_fold_kernel(const double* __restrict__ q, double* __restrict__ Q, int nf, int n, int m) {
  const long m3 = (long)m * m * m, n2 = (long)n * n, n3 = n2 * n;
  const long id = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (id >= nf * m3) return;
  const int f = (int)(id / m3);
  const long o = id - (long)f * m3;
  const int i = (int)(o / ((long)m * m)), j = (int)((o / m) % m), k = (int)(o % m);
  const double* qf = q + (long)f * n3;
  double v[8];
#pragma unroll
  for (int sg = 0; sg < 8; ++sg) {
    const int ii = (sg & 1) ? n - 1 - i : i, jj = (sg & 2) ? n - 1 - j : j, kk = (sg & 4) ? n - 1 - k : k;
    v[sg] = qf[ii * n2 + (long)jj * n + kk];
  }
#pragma unroll
  for (int st = 1; st < 8; st <<= 1)   // 8-point Walsh-Hadamard transform
#pragma unroll
    for (int a = 0; a < 8; ++a)
      if (!(a & st)) {
        const double x = v[a], y = v[a | st];
        v[a] = x + y;
        v[a | st] = x - y;
      }
#pragma unroll
  for (int p = 0; p < 8; ++p) Q[((long)f * 8 + p) * m3 + o] = 0.125 * v[p];
}

// unfold: u_f(σ(i, j, k)) = Σ_p (-1)^{popcount(p & σ)} U[(f*8 + p)][i][j][k] for the 8 reflections σ of every octant
// point (the same Walsh-Hadamard transform; one thread per octant point reads its 8 components once and writes
// the 8 images; at the centre node of an odd n the images coincide and, the odd components being exactly 0
// there, so do the values written)
__global__ void osp_unfold_kernel(const double* __restrict__ U, double* __restrict__ u, int nf, int n, int m) {
  const long m3 = (long)m * m * m, n2 = (long)n * n, n3 = n2 * n;
  const long id = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (id >= nf * m3) return;
  const int f = (int)(id / m3);
  const long o = id - (long)f * m3;
  const int i = (int)(o / ((long)m * m)), j = (int)((o / m) % m), k = (int)(o % m);
  double v[8];
#pragma unroll
  for (int p = 0; p < 8; ++p) v[p] = U[((long)f * 8 + p) * m3 + o];
#pragma unroll
  for (int st = 1; st < 8; st <<= 1)
#pragma unroll
    for (int a = 0; a < 8; ++a)
      if (!(a & st)) {
        const double x = v[a], y = v[a | st];
        v[a] = x + y;
        v[a | st] = x - y;
      }
  double* uf = u + (long)f * n3;
#pragma unroll
  for (int sg = 0; sg < 8; ++sg) {
    const int ii = (sg & 1) ? n - 1 - i : i, jj = (sg & 2) ? n - 1 - j : j, kk = (sg & 4) ? n - 1 - k : k;
    uf[ii * n2 + (long)jj * n + kk] = v[sg];
  }
}

__global__ void osp_par_kernel(uint8_t* par, int ncols) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c < ncols) par[c] = (uint8_t)(c & 7);
}

}  // namespace

// Columns [c0, c1) by the octant path when it applies (*done = true), else *done = false and nothing runs.
cudaError_t bep_sym_columns(dpm_ctx* ctx, int c0, int c1, double* PgE, double* B, cudaStream_t s, bool* done) {
  *done = false;
  if (ctx->sym == 0) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(s, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) return cudaSuccess;
    cudaError_t e = cudaStreamSynchronize(s);   // E and the sets are ready
    if (e != cudaSuccess) return e;
    if ((e = sym_prepare(ctx)) != cudaSuccess) return e;
  }
  if (ctx->sym != 1) {   // DPM_BEP_SYM=2: the octant path is required (tests), its absence an error
    const char* env = getenv("DPM_BEP_SYM");
    return env && atoi(env) == 2 ? cudaErrorNotSupported : cudaSuccess;
  }
  const int m = ctx->sym_m;
  const long m3 = (long)m * m * m;
  const int64_t ng = ctx->counts[DPM_SET_GAMMA], ngin = ctx->counts[DPM_SET_GAMMA_IN];
  const int cap = (int)std::max<long>(1, std::min<long>(ctx->K, (1L << 31) / (m3 * 8)));
  const int want = std::min(cap, c1 - c0);
  cudaError_t e;
  if (ctx->sym_cols < want) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;   // no allocation inside a graph capture
    if (cudaStreamIsCapturing(s, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) return cudaSuccess;
    if (ctx->sym_zbox) cudaFree(ctx->sym_zbox);
    if (ctx->sym_work) cudaFree(ctx->sym_work);
    ctx->sym_zbox = ctx->sym_work = nullptr;
    ctx->sym_cols = 0;
    if ((e = cudaMalloc(&ctx->sym_zbox, (size_t)want * m3 * 8)) != cudaSuccess) return e;
    if ((e = cudaMalloc(&ctx->sym_work, (size_t)want * m3 * 8)) != cudaSuccess) return e;
    if ((e = cudaMemsetAsync(ctx->sym_zbox, 0, (size_t)want * m3 * 8, s)) != cudaSuccess) return e;
    ctx->sym_cols = want;
  }
  for (int a = c0; a < c1; a += cap) {
    const int nc = std::min(cap, c1 - a);
    const uint8_t* par = ctx->sym_par + a;
    // (1) the octant's band values of q_c into the zero boxes (the same positions for every chunk)
    if ((e = launch_potential_list(ctx, ctx->E + (size_t)a * ng, ng, ctx->sym_list, ctx->sym_dst, ctx->sym_nlist,
                                   ctx->sym_zbox, m3, nc, s)) != cudaSuccess)
      return e;
    // (2)-(4)
    {
      const SymOp op{ctx->n, m, ctx->h, ctx->dt, ctx->sym_S, ctx->sym_lam, ctx->sym_R, ctx->sym_lu_dt != ctx->dt};
      ctx->sym_lu_dt = ctx->dt;
      e = sym_solve_mp(op, ctx->sym_zbox, ctx->sym_work, nc, par, s);
    }
    if (e != cudaSuccess) return e;
    // (5)
    DPM_COUNT_LAUNCH(1);
    sym_gather_kernel<<<dim3((unsigned)std::max<int64_t>(1, std::min<int64_t>((ng + ngin + 255) / 256, 148L * 16)), nc),
                        256, 0, s>>>(ctx->sym_work, m3, ctx->sym_gidx, ng, ngin, ctx->gin_pos, ctx->E, a, c0, par, PgE,
                                     B);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
  }
  *done = true;
  return cudaSuccess;
}

// ---- parity-split AP solve: host side -------------------------------------------------------------------------
// 0 when s is not capturing, else the id of its capture sequence (never 0)
static unsigned long long osp_capture_id(cudaStream_t s) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  unsigned long long id = 0;
  if (cudaStreamGetCaptureInfo(s, &cs, &id) != cudaSuccess) return ~0ull;
  return cs == cudaStreamCaptureStatusNone ? 0ull : (id ? id : ~0ull);
}

cudaError_t octsplit_prepare(dpm_ctx* ctx, int64_t batch) {
  if (ctx->osp == 0) {
    const char* env = getenv("DPM_OCTSPLIT");
    const int n = ctx->n;
    // default: only where it measures faster than the generic passes, i.e. the exact 64^3 octant of n = 127 (the
    // paper's Test B mesh); other n pad the GEMMs or take 8-byte copies and lose (tools/octsplit_sweep.py), n <= 64
    // and n = 128 have their own fused plane passes.  DPM_OCTSPLIT=2: every 4 <= n < 128 (tests, A/B); 0: off.
    const int mode = env ? atoi(env) : 1;
    ctx->osp = mode == 2 ? (n >= 4 && n < 128 ? 1 : -1) : mode == 1 && n == 127 ? 1 : -1;
  }
  if (ctx->osp != 1 || batch <= 0) return cudaSuccess;
  const int n = ctx->n, m = (n + 1) / 2;
  const size_t m3 = (size_t)m * m * m, m2 = (size_t)m * m;
  cudaError_t e;
  if (!ctx->osp_S) {
    std::vector<double> S, lam;
    sym_tables(n, ctx->h, S, lam);
    if ((e = upload(&ctx->osp_S, S)) != cudaSuccess) return e;
    if ((e = upload(&ctx->osp_lam, lam)) != cudaSuccess) return e;
    for (int k = 0; k < 2; ++k)
      if ((e = cudaMalloc(&ctx->osp_R[k], (8 * m2 * m + 8 * m2) * sizeof(double))) != cudaSuccess) return e;
    ctx->osp_lu_dt = 0.0;
  }
  const int want = (int)std::min<int64_t>(batch, 32);
  if (ctx->osp_cap < want) {
    if (ctx->osp_Q) cudaFree(ctx->osp_Q);
    if (ctx->osp_U) cudaFree(ctx->osp_U);
    if (ctx->osp_par) cudaFree(ctx->osp_par);
    ctx->osp_Q = ctx->osp_U = nullptr;
    ctx->osp_par = nullptr;
    ctx->osp_cap = 0;
    if ((e = cudaMalloc(&ctx->osp_Q, (size_t)want * 8 * m3 * 8)) != cudaSuccess) return e;
    if ((e = cudaMalloc(&ctx->osp_U, (size_t)want * 8 * m3 * 8)) != cudaSuccess) return e;
    if ((e = cudaMalloc(&ctx->osp_par, (size_t)want * 8)) != cudaSuccess) return e;
    DPM_COUNT_LAUNCH(1);
    osp_par_kernel<<<(want * 8 + 255) / 256, 256>>>(ctx->osp_par, want * 8);
    if ((e = cudaDeviceSynchronize()) != cudaSuccess) return e;
    ctx->osp_cap = want;
  }
  return cudaSuccess;
}

cudaError_t octsplit_solve(dpm_ctx* ctx, const double* q, double* u, int64_t batch, cudaStream_t s, bool* done) {
  *done = false;
  if (ctx->osp == -1 || ctx->plan.solver != DPM_SOLVER_DST2_TRIDIAG || ctx->plan.prof || batch <= 0) return cudaSuccess;
  const unsigned long long cap_id = osp_capture_id(s);
  const bool cap = cap_id != 0;
  if (!cap) {
    cudaError_t e = octsplit_prepare(ctx, batch);
    if (e != cudaSuccess) return e;
  }
  if (ctx->osp != 1 || ctx->osp_cap == 0) return cudaSuccess;   // off, or a capture before any prepare: dst path
  const int n = ctx->n, m = (n + 1) / 2;
  const size_t m3 = (size_t)m * m * m, n3 = (size_t)n * n * n;
  const double dt = ctx->plan.dt;
  for (int64_t b0 = 0; b0 < batch; b0 += ctx->osp_cap) {
    const int nf = (int)std::min<int64_t>(ctx->osp_cap, batch - b0);
    bool build;
    int slot;
    if (cap) {   // inside a graph: slot 1, rebuilt by the first solve of every captured graph (one Δt per graph)
      slot = 1;
      build = ctx->osp_cap_id != cap_id || cap_id == ~0ull || ctx->osp_cap_dt != dt;
      ctx->osp_cap_id = cap_id;
      ctx->osp_cap_dt = dt;
    } else {
      slot = 0;
      build = ctx->osp_lu_dt != dt;
      ctx->osp_lu_dt = dt;
    }
    DPM_COUNT_LAUNCH(2);
    osp_fold_kernel<<<(unsigned)((nf * m3 + 255) / 256), 256, 0, s>>>(q + b0 * n3, ctx->osp_Q, nf, n, m);
    const SymOp op{n, m, ctx->h, dt, ctx->osp_S, ctx->osp_lam, ctx->osp_R[slot], build};
    cudaError_t e = sym_solve_mp(op, ctx->osp_Q, ctx->osp_U, nf * 8, ctx->osp_par, s);
    if (e != cudaSuccess) return e;
    osp_unfold_kernel<<<(unsigned)((nf * m3 + 255) / 256), 256, 0, s>>>(ctx->osp_U, u + b0 * n3, nf, n, m);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
  }
  *done = true;
  return cudaSuccess;
}

cudaError_t ctx_solve(dpm_ctx* ctx, const double* q, double* u, int64_t batch, cudaStream_t s) {
  bool done = false;
  cudaError_t e = octsplit_solve(ctx, q, u, batch, s, &done);
  if (e != cudaSuccess || done) return e;
  return dst_solve_batch(ctx->plan, q, u, batch, nullptr, 0, s);
}

void bep_sym_free(dpm_ctx* c) {
  for (void* p : {(void*)c->osp_S, (void*)c->osp_lam, (void*)c->osp_R[0], (void*)c->osp_R[1], (void*)c->osp_Q,
                  (void*)c->osp_U, (void*)c->osp_par})
    if (p) cudaFree(p);
  void* ptrs[] = {c->sym_list, c->sym_dst, c->sym_gidx, c->sym_par, c->sym_S, c->sym_lam, c->sym_zbox, c->sym_work, c->sym_R, c->sym_perm, c->sym_mirin, c->sym_Bp, c->sym_tmp, c->sym_dg, c->sym_flag};
  for (cudaStream_t st : c->sym_streams)
    if (st) cudaStreamDestroy(st);
  for (cudaEvent_t ev : c->sym_ev)
    if (ev) cudaEventDestroy(ev);
  for (void* p : ptrs)
    if (p) cudaFree(p);
}

// The block-diagonal factorisation of B applies: octant path on, and every column of B has its class parity
// (one check kernel and a host sync; DPM_BEP_SYM_FACTOR=0 disables).
bool bep_sym_blocks(dpm_ctx* ctx, const double* B, cudaStream_t s) {
  static const bool on = [] {
    const char* v = getenv("DPM_BEP_SYM_FACTOR");
    return !(v && atoi(v) == 0);
  }();
  if (!on || ctx->sym != 1 || !ctx->sym_perm) return false;
  if (!ctx->sym_flag && cudaMalloc(&ctx->sym_flag, sizeof(int)) != cudaSuccess) return false;
  const long m = ctx->counts[DPM_SET_GAMMA_IN];
  int h = 1;
  if (cudaMemsetAsync(ctx->sym_flag, 0, sizeof(int), s) != cudaSuccess) return false;
  DPM_COUNT_LAUNCH(1);
  sym_check_kernel<<<ctx->K, 256, 0, s>>>(B, m, ctx->sym_mirin, ctx->sym_par, ctx->sym_flag);
  if (cudaMemcpyAsync(&h, ctx->sym_flag, sizeof(int), cudaMemcpyDeviceToHost, s) != cudaSuccess) return false;
  if (cudaStreamSynchronize(s) != cudaSuccess) return false;
  return h == 0;
}
