// S2 / S4 / S6 / S8-S9 element-wise and stencil kernels:
//  * potential RHS scatter  q = χ_{M-} (I/dt - Δ_h)[v_γ]            (Def. DP; R4)
//  * trace / BEP gather     PgE = Tr_γ u, B = E_in - Tr_γin u
//  * PKS: CFL reduction (R19), upwind/minmod flux + IMEX RHS (R15, R16),
//         combined Green RHS (R20), restriction to N+ with step statistics (R18).
#include <cstdlib>

#include "dpm_internal.h"

namespace {

constexpr int TB = 256;
#ifndef STENCIL_MINB
#define STENCIL_MINB 4   // stencil kernels: <= 64 registers, 32 warps per SM (latency-bound gathers)
#endif

// flat index -> (i, j, k); n^3 <= DPM_MAX_N^3 < 2^31, so two 32-bit divisions (the 64-bit ones are
// long emulated sequences and dominated the per-point cost of the stencil kernels)
__device__ __forceinline__ void ijk(long p, int n, int& i, int& j, int& k) {
  const unsigned up = (unsigned)p, un = (unsigned)n;
  const unsigned q = up / un;
  k = (int)(up - q * un);
  i = (int)(q / un);
  j = (int)(q - (unsigned)i * un);
}

__device__ __forceinline__ long flat(int n, int i, int j, int k) { return ((long)i * n + j) * n + k; }

__device__ __forceinline__ bool interior(int n, int i, int j, int k) {
  return i >= 0 && i < n && j >= 0 && j < n && k >= 0 && k < n;
}

// (I/dt - Δ_h)[v](p) for a density v given on gamma (zero elsewhere, zero ghosts)
__device__ __forceinline__ double lop_gamma(const int32_t* __restrict__ gmap, const double* __restrict__ v, int n,
                                            int i, int j, int k, double diag, double off) {
  const int gp = gmap[flat(n, i, j, k)];
  double acc = gp >= 0 ? diag * v[gp] : 0.0;
  const int di[6] = {1, -1, 0, 0, 0, 0}, dj[6] = {0, 0, 1, -1, 0, 0}, dk[6] = {0, 0, 0, 0, 1, -1};
  double nb = 0.0;
#pragma unroll
  for (int s = 0; s < 6; ++s) {
    const int a = i + di[s], b = j + dj[s], c = k + dk[s];
    if (!interior(n, a, b, c)) continue;
    const int g = gmap[flat(n, a, b, c)];
    if (g >= 0) nb += v[g];
  }
  return acc - off * nb;
}

// The band point's seven γ positions (gmap lookups), shared by every right-hand side:
// (I/dt - Δ_h)[v](p) = diag v(g0) - off Σ v(gn)  over the γ entries only (as lop_gamma)
struct BandStencil {
  int g0;
  int gn[6];
};
__device__ __forceinline__ BandStencil band_stencil(const int32_t* __restrict__ gmap, int n, int64_t p) {
  int i, j, k;
  ijk(p, n, i, j, k);
  BandStencil st;
  st.g0 = gmap[p];
  const int di[6] = {1, -1, 0, 0, 0, 0}, dj[6] = {0, 0, 1, -1, 0, 0}, dk[6] = {0, 0, 0, 0, 1, -1};
#pragma unroll
  for (int q = 0; q < 6; ++q) {
    const int a = i + di[q], b = j + dj[q], c = k + dk[q];
    st.gn[q] = interior(n, a, b, c) ? gmap[flat(n, a, b, c)] : -1;
  }
  return st;
}
__device__ __forceinline__ double band_apply(const BandStencil& st, const double* __restrict__ v, double diag, double off) {
  const double acc = st.g0 >= 0 ? diag * v[st.g0] : 0.0;
  double nb = 0.0;
#pragma unroll
  for (int q = 0; q < 6; ++q)
    if (st.gn[q] >= 0) nb += v[st.gn[q]];
  return acc - off * nb;
}

// thread per (band point, chunk of POT_RC right-hand sides = blockIdx.y): no per-element 64-bit division,
// the stencil's gmap lookups done once per point and chunk
constexpr int POT_RC = 8;
__global__ void potential_rhs_kernel(const int32_t* __restrict__ gmap, const int64_t* __restrict__ band,
                                     int64_t nband, const double* __restrict__ v, int64_t ldv, double* q,
                                     int nrhs, int n, double diag, double off) {
  const size_t field = (size_t)n * n * n;
  for (long b = blockIdx.x * (long)blockDim.x + threadIdx.x; b < nband; b += (long)gridDim.x * blockDim.x) {
    const long p = band[b];
    const BandStencil st = band_stencil(gmap, n, p);
    const int r1 = min(nrhs, (int)(blockIdx.y + 1) * POT_RC);
    for (int r = blockIdx.y * POT_RC; r < r1; ++r) q[r * field + p] = band_apply(st, v + (size_t)r * ldv, diag, off);
  }
}

// the potential RHS at a list of band points written to q[r * qstride + dst[b]] (the octant boxes of
// bep_sym.cu: the band points of the octant, at their octant positions)
__global__ void potential_list_kernel(const int32_t* __restrict__ gmap, const int64_t* __restrict__ list,
                                      const int32_t* __restrict__ dst, int64_t nlist, const double* __restrict__ v,
                                      int64_t ldv, double* q, int64_t qstride, int nrhs, int n, double diag, double off) {
  for (long b = blockIdx.x * (long)blockDim.x + threadIdx.x; b < nlist; b += (long)gridDim.x * blockDim.x) {
    const BandStencil st = band_stencil(gmap, n, list[b]);
    const long o = dst[b];
    const int r1 = min(nrhs, (int)(blockIdx.y + 1) * POT_RC);
    for (int r = blockIdx.y * POT_RC; r < r1; ++r) q[r * qstride + o] = band_apply(st, v + (size_t)r * ldv, diag, off);
  }
}

// the same values compacted to the band: qb[r][b] = q_r(band[b])  (fused BEP build, bep_fused.cu)
__global__ void potential_band_kernel(const int32_t* __restrict__ gmap, const int64_t* __restrict__ band,
                                      int64_t nband, const double* __restrict__ v, int64_t ldv, double* qb,
                                      int nrhs, int n, double diag, double off, const int32_t* __restrict__ pos) {
  for (long b = blockIdx.x * (long)blockDim.x + threadIdx.x; b < nband; b += (long)gridDim.x * blockDim.x) {
    const BandStencil st = band_stencil(gmap, n, band[b]);
    const long o = pos ? pos[b] : b;
    const int r1 = min(nrhs, (int)(blockIdx.y + 1) * POT_RC);
    for (int r = blockIdx.y * POT_RC; r < r1; ++r) qb[(size_t)r * nband + o] = band_apply(st, v + (size_t)r * ldv, diag, off);
  }
}

__global__ void trace_kernel(const double* __restrict__ u, const int64_t* __restrict__ list, int64_t m, double* out,
                             int64_t batch, size_t field) {
  pdl_prologue();
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < m; i += (long)gridDim.x * blockDim.x) {
    const int64_t p = list[i];
    for (long b = 0; b < batch; ++b) out[b * m + i] = u[b * field + p];
  }
}

__global__ void bep_gather_kernel(const double* __restrict__ U, int ncols, size_t field, const int64_t* __restrict__ gamma,
                                  int64_t ng, const int64_t* __restrict__ gin, const int32_t* __restrict__ gin_pos,
                                  int64_t ngin, const double* __restrict__ E, int c0, double* PgE, double* B) {
  // column c = blockIdx.y, rows grid-stride over x (no per-element 64-bit division)
  const int c = blockIdx.y;
  const double* Uc = U + (size_t)c * field;
  for (long r = blockIdx.x * (long)blockDim.x + threadIdx.x; r < ng + ngin; r += (long)gridDim.x * blockDim.x) {
    if (r < ng) {
      if (PgE) PgE[(size_t)c * ng + r] = Uc[gamma[r]];
    } else {
      const long i = r - ng;
      if (B) B[(size_t)c * ngin + i] = E[(size_t)(c0 + c) * ng + gin_pos[i]] - Uc[gin[i]];
    }
  }
}

// ------------------------------ PKS ------------------------------------------

__device__ __forceinline__ double valat(const double* __restrict__ f, int n, int i, int j, int k) {
  return interior(n, i, j, k) ? f[flat(n, i, j, k)] : 0.0;
}


__device__ __forceinline__ double minmod3(double a, double b, double c) {
  if (a > 0 && b > 0 && c > 0) return fmin(a, fmin(b, c));
  if (a < 0 && b < 0 && c < 0) return fmax(a, fmax(b, c));
  return 0.0;
}

// minmod slopes: nonzero only if the cell and both neighbours along the axis are in N+
// (R15); the three minmod arguments share the positive factor 1/h, so the limiter runs on the unscaled
// differences (x2 and x1/2 are exact) and h s enters the reconstruction r0 ± (h/2) s directly
// (evaluated inside flux_rhs_kernel).

__device__ __forceinline__ void umax_atomic(double* addr, double v) {
  // non-negative doubles order like their bit patterns
  atomicMax((unsigned long long*)addr, (unsigned long long)__double_as_longlong(v));
}

__global__ void __launch_bounds__(TB, STENCIL_MINB) cfl_kernel(const double* __restrict__ c, const uint8_t* __restrict__ flags, int n, double* out3) {
  __shared__ double red[3][TB / 32];
  double mx[3] = {0, 0, 0};
  const long nn = (long)n * n * n;
  for (long p = blockIdx.x * (long)blockDim.x + threadIdx.x; p < nn; p += (long)gridDim.x * blockDim.x) {
    if (!(flags[p] & F_MPLUS)) continue;
    int i, j, k;
    ijk(p, n, i, j, k);
    const double c0 = c[p];
    mx[0] = fmax(mx[0], fmax(fabs(valat(c, n, i + 1, j, k) - c0), fabs(c0 - valat(c, n, i - 1, j, k))));
    mx[1] = fmax(mx[1], fmax(fabs(valat(c, n, i, j + 1, k) - c0), fabs(c0 - valat(c, n, i, j - 1, k))));
    mx[2] = fmax(mx[2], fmax(fabs(valat(c, n, i, j, k + 1) - c0), fabs(c0 - valat(c, n, i, j, k - 1))));
  }
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int a = 0; a < 3; ++a) {
    double v = mx[a];
    for (int o = 16; o; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    if (lane == 0) red[a][w] = v;
  }
  __syncthreads();
  if (threadIdx.x < 3) {
    double v = 0;
    for (int q = 0; q < TB / 32; ++q) v = fmax(v, red[threadIdx.x][q]);
    umax_atomic(out3 + threadIdx.x, v);
  }
}

// g and the IMEX right-hand sides, written scaled for the ABI operator:
// fq_rho = (rho - dt g)/dt, fq_c = ((1-dt) c + dt rho)/dt on M+, 0 elsewhere.
// The Step-3 CFL maxima and device dt rule fused into the flux kernel (the same face differences
// |c_{+1} - c| and |c - c_{-1}| of every M+ point it loads anyway): maxima by per-block atomics into
// out3, the last block (ticket) evaluates the rule into dt_out and re-zeroes out3 for the next use
// (the slot is zero from allocation), so a step needs neither a memset nor a separate CFL kernel.
struct CflFuse {
  double* out3 = nullptr;   // null: no CFL (fixed dt)
  unsigned* ticket = nullptr;
  double chi = 0, dt_prev = 0, cap = 0;
  double* dt_out = nullptr;
  int* abort = nullptr;     // speculative step graphs: set when the rule asks for a dt below dt_prev
};

// Step 3 on the device, the tail of both flux kernels: block maxima of the face differences -> atomics,
// the last block (ticket) evaluates the rule into dt_out and re-zeroes the slot.
__device__ __forceinline__ void cfl_finish(const double (&cmx)[3], double h, const CflFuse& cf) {
  __shared__ double red[3][TB / 32];
  __shared__ bool last;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int a = 0; a < 3; ++a) {
    double v = cmx[a];
    for (int o = 16; o; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    if (lane == 0) red[a][w] = v;
  }
  __syncthreads();
  if (threadIdx.x < 3) {
    double v = 0;
    for (int q = 0; q < TB / 32; ++q) v = fmax(v, red[threadIdx.x][q]);
    umax_atomic(cf.out3 + threadIdx.x, v);
    __threadfence();
  }
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(cf.ticket, 1u) == gridDim.x - 1;
  __syncthreads();
  if (last && threadIdx.x == 0) {
    __threadfence();
    volatile double* r3 = cf.out3;
    double cfl = INFINITY;
    for (int a = 0; a < 3; ++a) {
      const double m = r3[a] / h;
      if (m > 0) cfl = fmin(cfl, h / (6.0 * cf.chi * m));
      r3[a] = 0.0;   // ready for the slot's next use
    }
    const double dtr = fmin(fmin(cf.dt_prev, cf.cap), fmin(cfl, 0.5 * h * h));
    *cf.dt_out = dtr;
    if (cf.abort && dtr < cf.dt_prev) *(volatile int*)cf.abort = 1;   // the rest of the graph leaves the state alone
    *cf.ticket = 0u;
  }
}

__global__ void __launch_bounds__(TB, STENCIL_MINB) flux_rhs_kernel(const double* __restrict__ rho, const double* __restrict__ c,
                                const uint8_t* __restrict__ flags, int n, double h, double dt, double chi,
                                double* __restrict__ fq_rho, double* __restrict__ fq_c, double* __restrict__ backup,
                                double* __restrict__ zero6, CflFuse cf) {
  // Per axis the stencil's values (ρ and flags at offsets -2..2, c at ±1) are loaded up front with
  // predicated loads (0 outside the box, like valat), then the N+ tests (interior flag; a face ghost is
  // in N+ iff its unique interior neighbour is in M+, R5; anything further out is not), the minmod
  // slopes and the upwind choice are evaluated from registers, without dependent load chains.
  pdl_prologue();
  const long nn = (long)n * n * n;
  const double ih = 1.0 / h, idt = 1.0 / dt;
  if (zero6 && blockIdx.x == 0 && threadIdx.x < 9) zero6[threadIdx.x] = 0.0;   // the step's statistics, clamp max, mass hi
  double cmx[3] = {0.0, 0.0, 0.0};
  for (long p = blockIdx.x * (long)blockDim.x + threadIdx.x; p < nn; p += (long)gridDim.x * blockDim.x) {
    if (backup) {   // the step's rollback copy of the state (speculative PKS graphs), fused with the read
      backup[p] = rho[p];
      backup[nn + p] = c[p];
    }
    if (!(flags[p] & F_MPLUS)) {
      fq_rho[p] = 0.0;
      fq_c[p] = 0.0;
      continue;
    }
    int i, j, k;
    ijk(p, n, i, j, k);
    const double r0 = rho[p], c0 = c[p];
    double g = 0.0;
#pragma unroll
    for (int ax = 0; ax < 3; ++ax) {
      if (cf.out3) {   // (cE, cW below: c at ±1 along the axis, 0 outside the box, as valat)
        const long st0 = ax == 0 ? (long)n * n : (ax == 1 ? (long)n : 1L);
        const int cd0 = ax == 0 ? i : (ax == 1 ? j : k);
        const double e = cd0 + 1 < n ? c[p + st0] : 0.0, w = cd0 >= 1 ? c[p - st0] : 0.0;
        cmx[ax] = fmax(cmx[ax], fmax(fabs(e - c0), fabs(c0 - w)));
      }
      const int cd = ax == 0 ? i : (ax == 1 ? j : k);
      const long st = ax == 0 ? (long)n * n : (ax == 1 ? (long)n : 1L);
      double R[5];
      uint8_t Fr[5];
#pragma unroll
      for (int o = 0; o < 5; ++o) {
        const int pos = cd + o - 2;
        const bool in = pos >= 0 && pos < n;
        R[o] = in ? rho[p + (o - 2) * st] : 0.0;
        Fr[o] = in ? flags[p + (o - 2) * st] : (uint8_t)0;
      }
      const double cE = cd + 1 < n ? c[p + st] : 0.0, cW = cd >= 1 ? c[p - st] : 0.0;
      bool np[5];
#pragma unroll
      for (int o = 0; o < 5; ++o) {
        const int pos = cd + o - 2;
        if (pos >= 0 && pos < n) np[o] = Fr[o] & F_NPLUS;
        else if (pos == -1) np[o] = o + 1 < 5 && (Fr[o + 1 < 5 ? o + 1 : 4] & F_MPLUS);
        else if (pos == n) np[o] = o >= 1 && (Fr[o >= 1 ? o - 1 : 0] & F_MPLUS);
        else np[o] = false;
      }
      auto sl = [&](int o) -> double {   // h x the slope at offset o - 2 (o = 1, 2, 3), as slope_h
        const int pos = cd + o - 2;
        if (!(pos >= 0 && pos < n) || !np[o] || !np[o - 1] || !np[o + 1]) return 0.0;
        return minmod3(2.0 * (R[o + 1] - R[o]), 0.5 * (R[o + 1] - R[o - 1]), 2.0 * (R[o] - R[o - 1]));
      };
      const double gE = (cE - c0) * ih, gW = (c0 - cW) * ih;   // upwind choice: the sign of the difference
      const double s0 = sl(2);
      const double rhoE = gE > 0 ? r0 + 0.5 * s0 : R[3] - 0.5 * sl(3);
      const double rhoW = gW > 0 ? R[1] + 0.5 * sl(1) : r0 - 0.5 * s0;
      g += (chi * rhoE * gE - chi * rhoW * gW) * ih;
    }
    fq_rho[p] = (r0 - dt * g) * idt;
    fq_c[p] = ((1.0 - dt) * c0 + dt * r0) * idt;
  }
  if (!cf.out3) return;   // (uniform across the grid)
  cfl_finish(cmx, h, cf);
}

// The same right-hand sides over the M+ list (R7 order) instead of the whole box: per M+ point the
// nine slope-validity bits (axis a, offset o = 1..3: the position is in the box and it and both of its
// neighbours along a are in N+, with the face-ghost rule of flux_rhs_kernel) are precomputed once per
// context (slope_mask_kernel), so the kernel neither loads the 15 stencil flags nor evaluates the N+
// logic, and no warp diverges on the M+ test.  The box part (rollback copy, zeros off M+) is a plain
// streaming loop over all points by the same threads.
__device__ __forceinline__ unsigned slope_bits(const uint8_t* __restrict__ flags, int n, long p, int i, int j, int k) {
  unsigned m = 0;
#pragma unroll
  for (int ax = 0; ax < 3; ++ax) {
    const int cd = ax == 0 ? i : (ax == 1 ? j : k);
    const long st = ax == 0 ? (long)n * n : (ax == 1 ? (long)n : 1L);
    uint8_t Fr[5];
#pragma unroll
    for (int o = 0; o < 5; ++o) {
      const int pos = cd + o - 2;
      Fr[o] = pos >= 0 && pos < n ? flags[p + (o - 2) * st] : (uint8_t)0;
    }
    bool np[5];
#pragma unroll
    for (int o = 0; o < 5; ++o) {
      const int pos = cd + o - 2;
      if (pos >= 0 && pos < n) np[o] = Fr[o] & F_NPLUS;
      else if (pos == -1) np[o] = o + 1 < 5 && (Fr[o + 1 < 5 ? o + 1 : 4] & F_MPLUS);
      else if (pos == n) np[o] = o >= 1 && (Fr[o >= 1 ? o - 1 : 0] & F_MPLUS);
      else np[o] = false;
    }
#pragma unroll
    for (int o = 1; o <= 3; ++o) {
      const int pos = cd + o - 2;
      if (pos >= 0 && pos < n && np[o] && np[o - 1] && np[o + 1]) m |= 1u << (3 * ax + o - 1);
    }
  }
  return m;
}

__global__ void slope_mask_kernel(const uint8_t* __restrict__ flags, const int64_t* __restrict__ mlist, long nm, int n,
                                  uint16_t* __restrict__ mask) {
  for (long q = blockIdx.x * (long)blockDim.x + threadIdx.x; q < nm; q += (long)gridDim.x * blockDim.x) {
    const long p = mlist[q];
    int i, j, k;
    ijk(p, n, i, j, k);
    mask[q] = (uint16_t)slope_bits(flags, n, p, i, j, k);
  }
}

__global__ void __launch_bounds__(TB, STENCIL_MINB) flux_rhs_list_kernel(
    const double* __restrict__ rho, const double* __restrict__ c, const uint8_t* __restrict__ flags,
    const int64_t* __restrict__ mlist, const uint16_t* __restrict__ smask, long nm, int n, double h, double dt,
    double chi, double* __restrict__ fq_rho, double* __restrict__ fq_c, double* __restrict__ backup,
    double* __restrict__ zero6, CflFuse cf) {
  pdl_prologue();
  const long nn = (long)n * n * n;
  const long tid = blockIdx.x * (long)blockDim.x + threadIdx.x, nth = (long)gridDim.x * blockDim.x;
  const double ih = 1.0 / h, idt = 1.0 / dt;
  if (zero6 && blockIdx.x == 0 && threadIdx.x < 9) zero6[threadIdx.x] = 0.0;   // the step's statistics, clamp max, mass hi
  for (long p = tid; p < nn; p += nth) {
    if (backup) {   // the step's rollback copy of the state (speculative PKS graphs)
      backup[p] = rho[p];
      backup[nn + p] = c[p];
    }
    if (!(flags[p] & F_MPLUS)) {
      fq_rho[p] = 0.0;
      fq_c[p] = 0.0;
    }
  }
  double cmx[3] = {0.0, 0.0, 0.0};
  for (long q = tid; q < nm; q += nth) {
    const long p = mlist[q];
    const unsigned m = smask[q];
    int i, j, k;
    ijk(p, n, i, j, k);
    const double r0 = rho[p], c0 = c[p];
    double g = 0.0;
#pragma unroll
    for (int ax = 0; ax < 3; ++ax) {
      const int cd = ax == 0 ? i : (ax == 1 ? j : k);
      const long st = ax == 0 ? (long)n * n : (ax == 1 ? (long)n : 1L);
      double R[5];
#pragma unroll
      for (int o = 0; o < 5; ++o) {
        const int pos = cd + o - 2;
        R[o] = pos >= 0 && pos < n ? rho[p + (o - 2) * st] : 0.0;
      }
      const double cE = cd + 1 < n ? c[p + st] : 0.0, cW = cd >= 1 ? c[p - st] : 0.0;   // 0 outside, as valat
      if (cf.out3) cmx[ax] = fmax(cmx[ax], fmax(fabs(cE - c0), fabs(c0 - cW)));
      auto sl = [&](int o) -> double {   // h x the slope at offset o - 2 (o = 1, 2, 3), as slope_h
        if (!((m >> (3 * ax + o - 1)) & 1u)) return 0.0;
        return minmod3(2.0 * (R[o + 1] - R[o]), 0.5 * (R[o + 1] - R[o - 1]), 2.0 * (R[o] - R[o - 1]));
      };
      const double gE = (cE - c0) * ih, gW = (c0 - cW) * ih;   // upwind choice: the sign of the difference
      const double s0 = sl(2);
      const double rhoE = gE > 0 ? r0 + 0.5 * s0 : R[3] - 0.5 * sl(3);
      const double rhoW = gW > 0 ? R[1] + 0.5 * sl(1) : r0 - 0.5 * s0;
      g += (chi * rhoE * gE - chi * rhoW * gW) * ih;
    }
    fq_rho[p] = (r0 - dt * g) * idt;
    fq_c[p] = ((1.0 - dt) * c0 + dt * r0) * idt;
  }
  if (!cf.out3) return;   // (uniform across the grid)
  cfl_finish(cmx, h, cf);
}

// combined Green RHS (R20): q_r = fq_r on M+, (I/dt - Δ_h)[u_γ,r] on the band, 0 elsewhere
__global__ void __launch_bounds__(TB, STENCIL_MINB) green_rhs_kernel(const uint8_t* __restrict__ flags, const int32_t* __restrict__ gmap, int n,
                                 const double* __restrict__ fq, const double* __restrict__ ug, int64_t ng, double* q,
                                 int nrhs, double diag, double off) {
  pdl_prologue();
  const long nn = (long)n * n * n;
  for (long p = blockIdx.x * (long)blockDim.x + threadIdx.x; p < nn; p += (long)gridDim.x * blockDim.x) {
    const uint8_t f = flags[p];   // the point's flag, shared by the right-hand sides
    int i = 0, j = 0, k = 0;
    if (!(f & F_MPLUS) && (f & F_BAND)) ijk(p, n, i, j, k);
    for (int r = 0; r < nrhs; ++r) {
      const size_t t = (size_t)r * nn + p;
      double v = 0.0;
      if (f & F_MPLUS) v = fq[t];
      else if (f & F_BAND) v = lop_gamma(gmap, ug + (size_t)r * ng, n, i, j, k, diag, off);
      q[t] = v;
    }
  }
}

// The same combined RHS with the band part over the band list: a streaming pass writes fq on M+ and 0
// off M+ ∪ band; the band points (never in M+) take (I/dt - Δ_h)[u_γ,r] from one thread each, whose
// seven gmap lookups are shared by the right-hand sides.
__global__ void __launch_bounds__(TB, STENCIL_MINB) green_rhs_list_kernel(
    const uint8_t* __restrict__ flags, const int32_t* __restrict__ gmap, const int64_t* __restrict__ band,
    long nband, int n, const double* __restrict__ fq, const double* __restrict__ ug, int64_t ng, double* q, int nrhs,
    double diag, double off, int band_only) {
  pdl_prologue();
  const long nn = (long)n * n * n;
  const long tid = blockIdx.x * (long)blockDim.x + threadIdx.x, nth = (long)gridDim.x * blockDim.x;
  for (long p = tid; p < (band_only ? 0 : nn); p += nth) {
    const uint8_t f = flags[p];
    if (f & F_BAND) continue;
    for (int r = 0; r < nrhs; ++r) {
      const size_t t = (size_t)r * nn + p;
      q[t] = (f & F_MPLUS) ? fq[t] : 0.0;
    }
  }
  for (long b = tid; b < nband; b += nth) {
    const long p = band[b];
    int i, j, k;
    ijk(p, n, i, j, k);
    const int g0 = gmap[p];
    int gn[6];
    const int di[6] = {1, -1, 0, 0, 0, 0}, dj[6] = {0, 0, 1, -1, 0, 0}, dk[6] = {0, 0, 0, 0, 1, -1};
#pragma unroll
    for (int s = 0; s < 6; ++s) {
      const int a = i + di[s], bb = j + dj[s], c = k + dk[s];
      gn[s] = interior(n, a, bb, c) ? gmap[flat(n, a, bb, c)] : -1;
    }
    for (int r = 0; r < nrhs; ++r) {   // as lop_gamma: diag v(p) - off Σ_neighbours v, γ entries only
      const double* v = ug + (size_t)r * ng;
      const double acc = g0 >= 0 ? diag * v[g0] : 0.0;
      double nb = 0.0;
#pragma unroll
      for (int s = 0; s < 6; ++s)
        if (gn[s] >= 0) nb += v[gn[s]];
      q[(size_t)r * nn + p] = acc - off * nb;
    }
  }
}

// Paper diagnostics on M+ (P:683-699): out += [Σ ρ̄, Σ |x - x_c|^2 ρ̄, Σ {ρ̄ ln ρ̄ - ρ̄ c + c^2/2 + |c_{+1} - c_{-1}|^2 / (8h^2)}]
// (the host multiplies by h^3); ρ̄ ln ρ̄ := 0 for ρ̄ <= 0, c = 0 beyond the box (ghost layer).
__global__ void __launch_bounds__(TB, STENCIL_MINB) diag_kernel(const uint8_t* __restrict__ flags, int n, double lo, double h,
                                                        double cx, double cy, double cz, const double* __restrict__ rho,
                                                        const double* __restrict__ c, double* out) {
  const int nn = n * n * n;
  double sm0 = 0.0, sm1 = 0.0, sm2 = 0.0;
  const double inv8h2 = 1.0 / (8.0 * h * h);
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < nn; p += gridDim.x * blockDim.x) {
    if (!(flags[p] & F_MPLUS)) continue;
    int i, j, k;
    ijk(p, n, i, j, k);
    const double r = rho[p], cc = c[p];
    const double x = lo + (i + 1) * h - cx, y = lo + (j + 1) * h - cy, z = lo + (k + 1) * h - cz;
    const double gx = (i + 1 < n ? c[p + n * n] : 0.0) - (i > 0 ? c[p - n * n] : 0.0);
    const double gy = (j + 1 < n ? c[p + n] : 0.0) - (j > 0 ? c[p - n] : 0.0);
    const double gz = (k + 1 < n ? c[p + 1] : 0.0) - (k > 0 ? c[p - 1] : 0.0);
    sm0 += r;
    sm1 += (x * x + y * y + z * z) * r;
    sm2 += (r > 0.0 ? r * log(r) : 0.0) - r * cc + 0.5 * cc * cc + (gx * gx + gy * gy + gz * gz) * inv8h2;
  }
  __shared__ double red[3][TB / 32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int o = 16; o; o >>= 1) {
    sm0 += __shfl_xor_sync(0xffffffffu, sm0, o);
    sm1 += __shfl_xor_sync(0xffffffffu, sm1, o);
    sm2 += __shfl_xor_sync(0xffffffffu, sm2, o);
  }
  if (lane == 0) { red[0][w] = sm0; red[1][w] = sm1; red[2][w] = sm2; }
  __syncthreads();
  if (threadIdx.x < 3) {
    double t = 0.0;
    for (int q = 0; q < TB / 32; ++q) t += red[threadIdx.x][q];
    atomicAdd(out + threadIdx.x, t);
  }
}

// restriction to N+ ("on N+") + statistics: [mass_sum (fixed-point low word), rho_max, -rho_min,
// -c_min, nonfinite, rho_max over M+ (the paper's ||ρ||∞, P:683 eq. sd-norm:max), -, -, mass high word]
__global__ void __launch_bounds__(TB, STENCIL_MINB) restrict_kernel(const uint8_t* __restrict__ flags, int n, const double* __restrict__ u, double* rho,
                                double* c, double* stats, int* abort) {
  pdl_prologue();
  // speculative step graphs: after a step whose dt rule failed (flux kernel) or whose state went
  // non-finite (an earlier restriction) the state is left as it is
  if (abort && *(volatile int*)abort) return;
  const long nn = (long)n * n * n;
  double msum = 0.0, rmax = -INFINITY, rmin = INFINITY, cmin = INFINITY, rmaxm = -INFINITY;
  int bad = 0;
  for (long p = blockIdx.x * (long)blockDim.x + threadIdx.x; p < nn; p += (long)gridDim.x * blockDim.x) {
    const uint8_t f = flags[p];
    double a = 0.0, b = 0.0;
    if (f & F_NPLUS) {
      a = u[p];
      b = u[nn + p];
      if (!isfinite(a) || !isfinite(b)) bad = 1;
      rmax = fmax(rmax, a);
      rmin = fmin(rmin, a);
      cmin = fmin(cmin, b);
      if (f & F_MPLUS) {
        msum += a;
        rmaxm = fmax(rmaxm, a);
      }
    }
    rho[p] = a;
    c[p] = b;
  }
  __shared__ double red[5][TB / 32];
  __shared__ int sbad;
  if (threadIdx.x == 0) sbad = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int o = 16; o; o >>= 1) {
    msum += __shfl_xor_sync(0xffffffffu, msum, o);
    rmax = fmax(rmax, __shfl_xor_sync(0xffffffffu, rmax, o));
    rmin = fmin(rmin, __shfl_xor_sync(0xffffffffu, rmin, o));
    cmin = fmin(cmin, __shfl_xor_sync(0xffffffffu, cmin, o));
    rmaxm = fmax(rmaxm, __shfl_xor_sync(0xffffffffu, rmaxm, o));
  }
  if (bad) atomicOr(&sbad, 1);
  if (lane == 0) { red[0][w] = msum; red[1][w] = rmax; red[2][w] = rmin; red[3][w] = cmin; red[4][w] = rmaxm; }
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0, a = -INFINITY, b = INFINITY, d = INFINITY, am = -INFINITY;
    for (int q = 0; q < TB / 32; ++q) {
      s += red[0][q]; a = fmax(a, red[1][q]); b = fmin(b, red[2][q]); d = fmin(d, red[3][q]); am = fmax(am, red[4][q]);
    }
    // the mass (R18) as an exact 128-bit fixed-point sum (2^-64 resolution): integer additions commute,
    // so the total does not depend on the order of the blocks (deterministic); stats[0] = low word,
    // stats[8] = high word (mass_fixed_decode)
    const double fl = floor(s);
    const unsigned long long lo = (unsigned long long)((s - fl) * 18446744073709551616.0);
    const long long hi = (long long)fl;
    unsigned long long* w = reinterpret_cast<unsigned long long*>(stats);
    const unsigned long long old = atomicAdd(w, lo);
    atomicAdd(w + 8, (unsigned long long)hi + (old + lo < old ? 1ull : 0ull));
    // max via bit patterns on the ordered transform
    auto key = [](double v) {
      unsigned long long x = (unsigned long long)__double_as_longlong(v);
      return (x >> 63) ? ~x : (x | 0x8000000000000000ull);
    };
    atomicMax((unsigned long long*)(stats + 1), key(a));
    atomicMax((unsigned long long*)(stats + 2), key(-b));
    atomicMax((unsigned long long*)(stats + 3), key(-d));
    if (sbad) atomicAdd(stats + 4, 1.0);
    if (sbad && abort) atomicExch(abort, 1);
    atomicMax((unsigned long long*)(stats + 5), key(am));
  }
}

// cell average of exp(-rate s^2) over [s - h/2, s + h/2] (R36): sqrt(π/rate) (erf(√rate (s + h/2)) -
// erf(√rate (s - h/2))) / (2h); 1 for rate = 0
__device__ __forceinline__ double gauss_cell_avg1(double s, double rate, double h) {
  if (!(rate > 0.0)) return 1.0;
  const double q = sqrt(rate);
  return 0.88622692545275801365 / q * (erf(q * (s + 0.5 * h)) - erf(q * (s - 0.5 * h))) / h;   // sqrt(π)/2
}

__global__ void pks_init_kernel(const uint8_t* __restrict__ flags, const int32_t* __restrict__ gmap,
                                const double* __restrict__ foot, int n, double lo, double h, dpm_pks_ic ic, double* rho,
                                double* c) {
  const long nn = (long)n * n * n;
  for (long p = blockIdx.x * (long)blockDim.x + threadIdx.x; p < nn; p += (long)gridDim.x * blockDim.x) {
    const uint8_t f = flags[p];
    double a = 0.0, b = 0.0;
    if (f & F_NPLUS) {
      double x, y, z;
      const int g = gmap[p];
      if (g >= 0) { x = foot[3 * g]; y = foot[3 * g + 1]; z = foot[3 * g + 2]; }   // R14
      else {
        int i, j, k;
        ijk(p, n, i, j, k);
        x = lo + (i + 1) * h; y = lo + (j + 1) * h; z = lo + (k + 1) * h;
      }
      const double r2 = (x - ic.center[0]) * (x - ic.center[0]) + (y - ic.center[1]) * (y - ic.center[1]) +
                        (z - ic.center[2]) * (z - ic.center[2]);
      a = ic.rho_amp * exp(-ic.rho_rate * r2);
      b = ic.c_amp * exp(-ic.c_rate * r2);
      if (ic.rho_cell_average && g < 0 && (f & F_MPLUS))   // R36: ρ̄0 = cell average on M+ \ γ
        a = ic.rho_amp * gauss_cell_avg1(x - ic.center[0], ic.rho_rate, h) *
            gauss_cell_avg1(y - ic.center[1], ic.rho_rate, h) * gauss_cell_avg1(z - ic.center[2], ic.rho_rate, h);
    }
    rho[p] = a;
    c[p] = b;
  }
}

int grid_for(long work) { return (int)std::max<long>(1, std::min<long>((work + TB - 1) / TB, 148L * 16)); }
// kernels ending in per-block atomics on a few addresses (CFL maxima, step statistics): 4 blocks per SM
int grid_reduce(long work) { return (int)std::max<long>(1, std::min<long>((work + TB - 1) / TB, 148L * 4)); }

}  // namespace

cudaError_t launch_potential_rhs(const dpm_ctx* ctx, const double* v, int64_t ldv, double* q, int nrhs,
                                 cudaStream_t s) {
  const size_t field = (size_t)ctx->n * ctx->n * ctx->n;
  cudaError_t e = cudaMemsetAsync(q, 0, field * nrhs * sizeof(double), s);
  if (e != cudaSuccess) return e;
  return launch_potential_scatter(ctx, v, ldv, q, nrhs, s);
}

cudaError_t launch_potential_scatter(const dpm_ctx* ctx, const double* v, int64_t ldv, double* q, int nrhs,
                                     cudaStream_t s) {
  const int n = ctx->n;
  const int64_t nb = ctx->counts[DPM_SET_BAND];
  if (nb * nrhs == 0) return cudaSuccess;
  const double diag = 1.0 / ctx->dt + 6.0 / (ctx->h * ctx->h), off = 1.0 / (ctx->h * ctx->h);
  DPM_COUNT_LAUNCH(1);
  potential_rhs_kernel<<<dim3((unsigned)((nb + TB - 1) / TB), (nrhs + POT_RC - 1) / POT_RC), TB, 0, s>>>(ctx->gmap, ctx->lists[DPM_SET_BAND], nb, v, ldv, q, nrhs, n,
                                                          diag, off);
  return cudaGetLastError();
}

cudaError_t launch_potential_list(const dpm_ctx* ctx, const double* v, int64_t ldv, const int64_t* list,
                                  const int32_t* dst, int64_t nlist, double* q, int64_t qstride, int nrhs,
                                  cudaStream_t s) {
  if (nlist * nrhs == 0) return cudaSuccess;
  const double diag = 1.0 / ctx->dt + 6.0 / (ctx->h * ctx->h), off = 1.0 / (ctx->h * ctx->h);
  DPM_COUNT_LAUNCH(1);
  potential_list_kernel<<<dim3((unsigned)((nlist + TB - 1) / TB), (nrhs + POT_RC - 1) / POT_RC), TB, 0, s>>>(
      ctx->gmap, list, dst, nlist, v, ldv, q, qstride, nrhs, ctx->n, diag, off);
  return cudaGetLastError();
}

cudaError_t launch_potential_band(const dpm_ctx* ctx, const double* v, int64_t ldv, double* qb, int nrhs,
                                  const int32_t* pos, cudaStream_t s) {
  const int64_t nb = ctx->counts[DPM_SET_BAND];
  if (nb * nrhs == 0) return cudaSuccess;
  const double diag = 1.0 / ctx->dt + 6.0 / (ctx->h * ctx->h), off = 1.0 / (ctx->h * ctx->h);
  DPM_COUNT_LAUNCH(1);
  potential_band_kernel<<<dim3((unsigned)((nb + TB - 1) / TB), (nrhs + POT_RC - 1) / POT_RC), TB, 0, s>>>(ctx->gmap, ctx->lists[DPM_SET_BAND], nb, v, ldv, qb, nrhs,
                                                           ctx->n, diag, off, pos);
  return cudaGetLastError();
}

cudaError_t launch_trace(const dpm_ctx* ctx, const double* u, double* out, int which, int64_t batch, cudaStream_t s) {
  const int n = ctx->n;
  const int64_t m = ctx->counts[which];
  if (m * batch == 0) return cudaSuccess;
  DPM_COUNT_LAUNCH(1);
  return launch_pdl(trace_kernel, grid_for(m), TB, 0, s, u, (const int64_t*)ctx->lists[which], m, out, batch,
                    (size_t)n * n * n);
}

cudaError_t launch_bep_gather(const dpm_ctx* ctx, const double* U, int c0, int ncols, double* PgE, double* B,
                              cudaStream_t s) {
  const int n = ctx->n;
  const int64_t ng = ctx->counts[DPM_SET_GAMMA], ngin = ctx->counts[DPM_SET_GAMMA_IN];
  DPM_COUNT_LAUNCH(1);
  if (ncols == 0) return cudaSuccess;
  bep_gather_kernel<<<dim3((unsigned)std::max<int64_t>(1, std::min<int64_t>((ng + ngin + TB - 1) / TB, 148L * 16)), ncols), TB, 0, s>>>(U, ncols, (size_t)n * n * n, ctx->lists[DPM_SET_GAMMA], ng,
                                                                 ctx->lists[DPM_SET_GAMMA_IN], ctx->gin_pos, ngin, ctx->E,
                                                                 c0, PgE, B);
  return cudaGetLastError();
}

cudaError_t launch_pks_init(dpm_ctx* ctx, double* rho, double* c, const dpm_pks_ic* ic, cudaStream_t s) {
  const long nn = (long)ctx->n * ctx->n * ctx->n;
  DPM_COUNT_LAUNCH(1);
  pks_init_kernel<<<grid_for(nn), TB, 0, s>>>(ctx->flags, ctx->gmap, ctx->foot, ctx->n, ctx->lo, ctx->h, *ic, rho, c);
  return cudaGetLastError();
}

cudaError_t launch_cfl_reduce(dpm_ctx* ctx, const double* c, double* out3, cudaStream_t s) {
  const long nn = (long)ctx->n * ctx->n * ctx->n;
  cudaError_t e = cudaMemsetAsync(out3, 0, 3 * sizeof(double), s);
  if (e != cudaSuccess) return e;
  DPM_COUNT_LAUNCH(1);
  cfl_kernel<<<grid_reduce(nn), TB, 0, s>>>(c, ctx->flags, ctx->n, out3);
  return cudaGetLastError();
}

cudaError_t launch_flux_rhs(dpm_ctx* ctx, const double* rho, const double* c, double dt, double chi, double* fq_rho,
                            double* fq_c, cudaStream_t s, double* backup, double* zero6, double* cfl_out3,
                            double dt_prev, double cap, double* dt_out, int* abort) {
  const long nn = (long)ctx->n * ctx->n * ctx->n;
  CflFuse cf;
  if (cfl_out3) {
    cf.out3 = cfl_out3;
    cf.ticket = reinterpret_cast<unsigned*>(ctx->red + 63);
    cf.chi = chi;
    cf.dt_prev = dt_prev;
    cf.cap = cap;
    cf.dt_out = dt_out;
    cf.abort = abort;
  }
  static const bool use_list = [] {   // DPM_FLUX_LIST=0: the whole-box kernel
    const char* v = getenv("DPM_FLUX_LIST");
    return !(v && atoi(v) == 0);
  }();
  DPM_COUNT_LAUNCH(1);
  if (use_list && ctx->mplus_slope) {
    const long nm = ctx->counts[DPM_SET_MPLUS];
    return launch_pdl(flux_rhs_list_kernel, grid_for(nm), TB, 0, s, rho, c, (const uint8_t*)ctx->flags,
                      (const int64_t*)ctx->lists[DPM_SET_MPLUS], (const uint16_t*)ctx->mplus_slope, nm, ctx->n, ctx->h,
                      dt, chi, fq_rho, fq_c, backup, zero6, cf);
  }
  return launch_pdl(flux_rhs_kernel, grid_for(nn), TB, 0, s, rho, c, (const uint8_t*)ctx->flags, ctx->n, ctx->h, dt, chi,
                    fq_rho, fq_c, backup, zero6, cf);
}

cudaError_t launch_slope_mask(dpm_ctx* ctx, cudaStream_t s) {
  const long nm = ctx->counts[DPM_SET_MPLUS];
  cudaError_t e = cudaMalloc(&ctx->mplus_slope, std::max<long>(nm, 1) * sizeof(uint16_t));
  if (e != cudaSuccess) return e;
  DPM_COUNT_LAUNCH(1);
  slope_mask_kernel<<<grid_for(nm), TB, 0, s>>>(ctx->flags, ctx->lists[DPM_SET_MPLUS], nm, ctx->n, ctx->mplus_slope);
  return cudaGetLastError();
}

// sequential coupling (dpm_pks_params.coupling = 1): f_c / dt = ((1 - dt) c + dt ρ̄^{i+1}) / dt on M+
__global__ void __launch_bounds__(TB, STENCIL_MINB) fc_seq_kernel(const uint8_t* __restrict__ flags, long nn,
                                                          const double* __restrict__ c, const double* __restrict__ rho_new,
                                                          double dt, double* __restrict__ fq_c) {
  const double idt = 1.0 / dt;
  for (long p = blockIdx.x * (long)blockDim.x + threadIdx.x; p < nn; p += (long)gridDim.x * blockDim.x)
    fq_c[p] = (flags[p] & F_MPLUS) ? ((1.0 - dt) * c[p] + dt * rho_new[p]) * idt : 0.0;
}

cudaError_t launch_fc_seq(dpm_ctx* ctx, const double* c, const double* rho_new, double dt, double* fq_c, cudaStream_t s) {
  const long nn = (long)ctx->n * ctx->n * ctx->n;
  DPM_COUNT_LAUNCH(1);
  fc_seq_kernel<<<grid_for(nn), TB, 0, s>>>(ctx->flags, nn, c, rho_new, dt, fq_c);
  return cudaGetLastError();
}

cudaError_t launch_green_rhs(dpm_ctx* ctx, const double* fq, const double* u_gamma, double* q, int nrhs,
                             cudaStream_t s) {
  const long nn = (long)ctx->n * ctx->n * ctx->n;
  const double diag = 1.0 / ctx->dt + 6.0 / (ctx->h * ctx->h), off = 1.0 / (ctx->h * ctx->h);
  static const bool use_list = [] {   // DPM_GREEN_LIST=0: the whole-box kernel
    const char* v = getenv("DPM_GREEN_LIST");
    return !(v && atoi(v) == 0);
  }();
  DPM_COUNT_LAUNCH(1);
  if (use_list)
    return launch_pdl(green_rhs_list_kernel, grid_for(nn / 2), TB, 0, s, (const uint8_t*)ctx->flags,
                      (const int32_t*)ctx->gmap, (const int64_t*)ctx->lists[DPM_SET_BAND],
                      (long)ctx->counts[DPM_SET_BAND], ctx->n, fq, u_gamma, (int64_t)ctx->counts[DPM_SET_GAMMA], q,
                      nrhs, diag, off, 0);
  return launch_pdl(green_rhs_kernel, grid_for(nn), TB, 0, s, (const uint8_t*)ctx->flags, (const int32_t*)ctx->gmap,
                    ctx->n, fq, u_gamma, (int64_t)ctx->counts[DPM_SET_GAMMA], q, nrhs, diag, off);
}



// The band part of the combined Green RHS written in place into fq (which the flux kernel leaves zero off
// M+, and the band never meets M+): afterwards fq IS the combined right-hand side q of R20.
cudaError_t launch_green_band_inplace(dpm_ctx* ctx, double* fq, const double* u_gamma, int nrhs, cudaStream_t s) {
  const long nb = (long)ctx->counts[DPM_SET_BAND];
  const double diag = 1.0 / ctx->dt + 6.0 / (ctx->h * ctx->h), off = 1.0 / (ctx->h * ctx->h);
  DPM_COUNT_LAUNCH(1);
  return launch_pdl(green_rhs_list_kernel, grid_for(nb), TB, 0, s, (const uint8_t*)ctx->flags,
                    (const int32_t*)ctx->gmap, (const int64_t*)ctx->lists[DPM_SET_BAND], nb, ctx->n,
                    (const double*)fq, u_gamma, (int64_t)ctx->counts[DPM_SET_GAMMA], fq, nrhs, diag, off, 1);
}

cudaError_t launch_diagnostics(dpm_ctx* ctx, const double* rho, const double* c, double* out3, cudaStream_t s) {
  cudaError_t e = cudaMemsetAsync(out3, 0, 3 * sizeof(double), s);
  if (e != cudaSuccess) return e;
  const long nn = (long)ctx->n * ctx->n * ctx->n;
  DPM_COUNT_LAUNCH(1);
  diag_kernel<<<grid_reduce(nn), TB, 0, s>>>(ctx->flags, ctx->n, ctx->lo, ctx->h, ctx->domain.center[0],
                                             ctx->domain.center[1], ctx->domain.center[2], rho, c, out3);
  return cudaGetLastError();
}

cudaError_t launch_restrict_stats(dpm_ctx* ctx, const double* u, double* rho, double* c, double* stats,
                                  cudaStream_t s, bool zeroed, int* abort) {
  const long nn = (long)ctx->n * ctx->n * ctx->n;
  if (!zeroed) {   // (zeroed: an earlier kernel of the step cleared the 9 slots)
    cudaError_t e = cudaMemsetAsync(stats, 0, 9 * sizeof(double), s);
    if (e != cudaSuccess) return e;
  }
  DPM_COUNT_LAUNCH(1);
  static const int rb = [] {   // blocks per SM of the restriction (2: +1% cfg3 steps/s over 4)
    const char* v = getenv("DPM_RESTRICT_BPS");
    return v ? std::max(1, atoi(v)) : 2;
  }();
  const int grid = (int)std::max<long>(1, std::min<long>((nn + TB - 1) / TB, 148L * rb));
  return launch_pdl(restrict_kernel, grid, TB, 0, s, (const uint8_t*)ctx->flags, ctx->n, u, rho, c, stats, abort);
}
