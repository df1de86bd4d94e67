// Config 5: octant domain decomposition (the paper's DD with
// duplicated equations and averaged effective densities, Case 2 P:562-571).
//
// One dpm_ctx per octant subdomain, in its canonical frame p (box [-0.1, 1.1]^3, Ω = open octant ∩
// unit ball); physical coordinates x = σ ⊙ p.  Global unknowns (shared by all octants):
//   [cap: Y_ν | (d^2/2) Y_ν], ν < (Lc+1)^2          zero-Neumann cap, d = |x| - 1
//   [plane a: φ_jk | d φ_jk], j + k <= Li, a = x,y,z  2-term interface Cauchy data, d = x_a (R25)
// φ_jk(s, t) = P_j(s) P_k(t) (Legendre) of the two other physical coordinates in increasing axis
// order; (j, k) ordered by total degree g, then j = g..0.
// Piece assignment: p ∈ γ is on piece π iff its foot on π's carrier lies within ε = 2h of π and
// |distance to the carrier| < 2h.  Effective density A = mean of the assigned pieces' extension
// rows (used for the potentials); BEP rows: one per (p ∈ γ_in, π ∈ pieces(p)): E_π[p] - (P_γ A)[p].
// The global least squares over all octants is a distributed CholeskyQR2: Gram matrices and the
// per-step M_s g_s vectors are summed across octants by the caller (NCCL all-reduce).
#include <algorithm>
#include <cmath>
#include <vector>

#include "dpm_internal.h"
#include "sh_device.cuh"

namespace {

constexpr int TB = 256;

__device__ __forceinline__ void legendre_all(double x, int jmax, double* P) {
  P[0] = 1.0;
  if (jmax >= 1) P[1] = x;
  for (int j = 1; j < jmax; ++j) P[j + 1] = ((2 * j + 1) * x * P[j] - j * P[j - 1]) / (j + 1);
}

__device__ __forceinline__ double dist_quarter_disc(double s, double t) {
  const double ps = fmax(s, 0.0), pt = fmax(t, 0.0);
  const double r = hypot(ps, pt);
  const double sc = r > 1.0 ? 1.0 / r : 1.0;
  return hypot(s - ps * sc, t - pt * sc);
}

__device__ __forceinline__ double dist_octant_cap(const double f[3]) {
  double q[3], nq = 0.0;
  for (int a = 0; a < 3; ++a) {
    q[a] = fmax(f[a], 0.0);
    nq += q[a] * q[a];
  }
  nq = sqrt(nq);
  double d2 = 0.0;
  for (int a = 0; a < 3; ++a) {
    const double v = f[a] - (nq > 0 ? q[a] / nq : q[a]);
    d2 += v * v;
  }
  return sqrt(d2);
}

// Per γ point: piece bits, every piece's extension row (Eraw) and the averaged density row (A).
__global__ void dd_extension_kernel(const int64_t* gamma, int64_t ng, int n, double lo, double h, double radius,
                                    double sx, double sy, double sz, int Lc, int Li, int nphi, int K, double* Eraw,
                                    double* A, uint8_t* assign) {
  const long g = blockIdx.x * (long)blockDim.x + threadIdx.x;
  if (g >= ng) return;
  const int64_t pidx = gamma[g];
  const int i = (int)(pidx / ((long)n * n)), j = (int)((pidx / n) % n), k = (int)(pidx % n);
  const double P[3] = {lo + (i + 1) * h, lo + (j + 1) * h, lo + (k + 1) * h};   // canonical
  const double sg[3] = {sx, sy, sz};
  double X[3];
  for (int a = 0; a < 3; ++a) X[a] = sg[a] * P[a];                              // physical
  const double eps = 2.0 * h;
  const double r = sqrt(P[0] * P[0] + P[1] * P[1] + P[2] * P[2]);
  // assignment (frame-independent)
  int bits = 0;
  {
    const double f[3] = {P[0] / r, P[1] / r, P[2] / r};
    if (dist_octant_cap(f) <= eps && fabs(r - radius) < 2.0 * h) bits |= 1;
  }
  for (int a = 0; a < 3; ++a) {
    const int o0 = a == 0 ? 1 : 0, o1 = a == 2 ? 1 : 2;
    if (dist_quarter_disc(P[o0], P[o1]) <= eps && fabs(P[a]) < 2.0 * h) bits |= 2 << a;
  }
  assign[g] = (uint8_t)bits;
  const int cnt = __popc(bits);
  const double inv = cnt ? 1.0 / cnt : 0.0;
  // cap block: Y(x/|x|), (d^2/2) Y, d = |x| - radius
  const int nc = (Lc + 1) * (Lc + 1);
  const double dcap = r - radius;
  const double wc = 0.5 * dcap * dcap;
  const double ac = (bits & 1) ? inv : 0.0;
  real_sh_unit(X[0] / r, X[1] / r, X[2] / r, Lc, [&](int nu, double v) {
    Eraw[(size_t)nu * ng + g] = v;
    Eraw[(size_t)(nc + nu) * ng + g] = wc * v;
    A[(size_t)nu * ng + g] = ac * v;
    A[(size_t)(nc + nu) * ng + g] = ac * wc * v;
  });
  // plane blocks
  double Ps[32], Pt[32];
  for (int a = 0; a < 3; ++a) {
    const int o0 = a == 0 ? 1 : 0, o1 = a == 2 ? 1 : 2;
    legendre_all(X[o0], Li, Ps);
    legendre_all(X[o1], Li, Pt);
    const double d = X[a];
    const double ap = (bits & (2 << a)) ? inv : 0.0;
    const int c0 = 2 * nc + 2 * nphi * a;
    int m = 0;
    for (int gd = 0; gd <= Li; ++gd)
      for (int jj = gd; jj >= 0; --jj, ++m) {
        const double phi = Ps[jj] * Pt[gd - jj];
        Eraw[(size_t)(c0 + m) * ng + g] = phi;
        Eraw[(size_t)(c0 + nphi + m) * ng + g] = d * phi;
        A[(size_t)(c0 + m) * ng + g] = ap * phi;
        A[(size_t)(c0 + nphi + m) * ng + g] = ap * d * phi;
      }
  }
}

// u_γ[r][g] = Σ_c A[g][c] C[r][c] (r = 0, 1; optionally clamped at 0, R17) with the basis evaluated
// on the fly instead of streaming the n_gamma x K matrix A (~0.6 GB per octant at n = 128) every
// step: per γ point the piece weights (assignment bits), the real SH of the cap block and the
// Legendre products of the plane blocks, exactly as dd_extension_kernel builds A (the SH recursion
// coefficients come from shared-memory tables computed with the same expressions: identical values),
// contracted with the two coefficient vectors held in shared memory.  Pieces of weight 0 are skipped.
__global__ void __launch_bounds__(128) dd_extend_fly_kernel(const int64_t* __restrict__ gamma, int64_t ng, int n,
                                                            double lo, double h, double radius, double sx, double sy,
                                                            double sz, int Lc, int Li, int nphi, int K,
                                                            const uint8_t* __restrict__ assign,
                                                            const double* __restrict__ C, int clamp, double* ug) {
  extern __shared__ double fly_sm[];
  double2* cv = reinterpret_cast<double2*>(fly_sm);   // [K]: (C[0][c], C[1][c]) — one 16-byte load per basis value
  const int L1 = Lc + 1;
  double* ta = fly_sm + 2 * K;                 // [L1][L1]: a_lm
  double* tb = ta + L1 * L1;                   // [L1][L1]: b_lm
  double* tpm = tb + L1 * L1;                  // [L1]: sqrt((2m+1)/(2m))
  double* tz = tpm + L1;                       // [L1]: sqrt(2m+3)
  for (int i = threadIdx.x; i < K; i += blockDim.x) cv[i] = make_double2(C[i], C[K + i]);
  for (int e = threadIdx.x; e < L1 * L1; e += blockDim.x) {
    const int l = e / L1, m = e % L1;
    ta[e] = (l >= m + 2) ? sqrt((4.0 * l * l - 1.0) / ((double)l * l - (double)m * m)) : 0.0;
    tb[e] = (l >= m + 2) ? sqrt(((l - 1.0) * (l - 1.0) - (double)m * m) / (4.0 * (l - 1.0) * (l - 1.0) - 1.0)) : 0.0;
  }
  for (int m = threadIdx.x; m < L1; m += blockDim.x) {
    tpm[m] = m > 0 ? sqrt((2.0 * m + 1.0) / (2.0 * m)) : 1.0;
    tz[m] = sqrt(2.0 * m + 3.0);
  }
  __syncthreads();
  const int nc = L1 * L1;
  const double sg[3] = {sx, sy, sz};
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < ng; g += (int64_t)gridDim.x * blockDim.x) {
    const int64_t pidx = gamma[g];
    const unsigned up = (unsigned)pidx, un = (unsigned)n, q = up / un;   // n^3 < 2^31: 32-bit division
    const int k = (int)(up - q * un), i = (int)(q / un), j = (int)(q - (unsigned)i * un);
    const double P[3] = {lo + (i + 1) * h, lo + (j + 1) * h, lo + (k + 1) * h};
    double X[3];
    for (int a = 0; a < 3; ++a) X[a] = sg[a] * P[a];
    const double r = sqrt(P[0] * P[0] + P[1] * P[1] + P[2] * P[2]);
    const int bits = assign[g];
    const int cnt = __popc(bits);
    const double inv = cnt ? 1.0 / cnt : 0.0;
    double s0 = 0.0, s1 = 0.0;
    if (bits & 1) {   // cap: Y(x/|x|), (d^2/2) Y
      const double x = X[0] / r, y = X[1] / r, z = X[2] / r;
      const double dcap = r - radius, wc = 0.5 * dcap * dcap;
      double t0 = 0.0, t1 = 0.0;
      double pmm = 0.28209479177387814347, Cm = 1.0, Sm = 0.0;
      for (int m = 0; m <= Lc; ++m) {
        if (m > 0) {
          pmm *= tpm[m];
          const double Cn = x * Cm - y * Sm, Sn = x * Sm + y * Cm;
          Cm = Cn;
          Sm = Sn;
        }
        double p2 = 0.0, p1 = pmm;
        for (int l = m; l <= Lc; ++l) {
          double pl;
          if (l == m) pl = pmm;
          else if (l == m + 1) pl = z * tz[m] * pmm;
          else pl = ta[l * L1 + m] * (z * p1 - tb[l * L1 + m] * p2);
          if (l > m) { p2 = p1; p1 = pl; }
          if (m == 0) {
            const int nu = l * l + l;
            const double2 a = cv[nu], d = cv[nc + nu];
            t0 = fma(pl, fma(wc, d.x, a.x), t0);
            t1 = fma(pl, fma(wc, d.y, a.y), t1);
          } else {
            const double vc = 1.41421356237309504880 * pl * Cm, vs = 1.41421356237309504880 * pl * Sm;
            const int nup = l * l + l + m, nun = l * l + l - m;
            const double2 ap = cv[nup], dp = cv[nc + nup], an = cv[nun], dn = cv[nc + nun];
            t0 = fma(vc, fma(wc, dp.x, ap.x), t0);
            t1 = fma(vc, fma(wc, dp.y, ap.y), t1);
            t0 = fma(vs, fma(wc, dn.x, an.x), t0);
            t1 = fma(vs, fma(wc, dn.y, an.y), t1);
          }
        }
      }
      s0 = fma(inv, t0, s0);
      s1 = fma(inv, t1, s1);
    }
    for (int a = 0; a < 3; ++a) {   // planes: φ_jk = P_j P_k of the in-plane coordinates, {φ, d φ}
      if (!(bits & (2 << a))) continue;
      const int o0 = a == 0 ? 1 : 0, o1 = a == 2 ? 1 : 2;
      double Ps[32], Pt[32];
      legendre_all(X[o0], Li, Ps);
      legendre_all(X[o1], Li, Pt);
      const double d = X[a];
      const int cb = 2 * nc + 2 * nphi * a;
      double t0 = 0.0, t1 = 0.0;
      int m = 0;
      for (int gd = 0; gd <= Li; ++gd)
        for (int jj = gd; jj >= 0; --jj, ++m) {
          const double phi = Ps[jj] * Pt[gd - jj];
          const double2 a = cv[cb + m], e = cv[cb + nphi + m];
          t0 = fma(phi, fma(d, e.x, a.x), t0);
          t1 = fma(phi, fma(d, e.y, a.y), t1);
        }
      s0 = fma(inv, t0, s0);
      s1 = fma(inv, t1, s1);
    }
    ug[g] = clamp ? fmax(s0, 0.0) : s0;
    ug[ng + g] = clamp ? fmax(s1, 0.0) : s1;
  }
}

// u_γ for several octants of one canonical geometry at once (dpm_dd_green_rhs_shared).  Octant s
// evaluates the basis at X = σ_s ⊙ P, and every cap SH and plane Legendre function has a definite parity
// under each axis reflection, so b_ν(σ_s ⊙ P) = (-1)^{popcount(s & π(ν))} b_ν(P) with the parity class
// π(ν) = 4 p_x + 2 p_y + p_z (s = 4[σx<0] + 2[σy<0] + [σz<0]):
//   cap  m = 0: (0, 0, l);  Re (x+iy)^m part: (m, 0, l-m);  Im part: (m+1, 1, l-m)   (mod 2)
//   plane a, φ_jk = P_j(X_o0) P_k(X_o1): j on axis o0, k on axis o1; the d φ part adds axis a.
// The basis is evaluated once per γ point in the canonical frame, its terms summed per parity class
// (T_π, in the unrolled loop structure every class index is a compile-time constant), and
// u_s = Σ_π (-1)^{popcount(s&π)} T_π is an 8-point Walsh-Hadamard transform per field.
struct ExtOut {
  double* ug[8];
  int oct[8];
  int n;
};
__global__ void __launch_bounds__(128) dd_extend_shared_kernel(const int64_t* __restrict__ gamma, int64_t ng, int n,
                                                               double lo, double h, double radius, int Lc, int Li,
                                                               int nphi, int K, const uint8_t* __restrict__ assign,
                                                               const double* __restrict__ C, int clamp, ExtOut out) {
  extern __shared__ double fly_sm[];
  double2* cv = reinterpret_cast<double2*>(fly_sm);
  const int L1 = Lc + 1;
  double* ta = fly_sm + 2 * K;
  double* tb = ta + L1 * L1;
  double* tpm = tb + L1 * L1;
  double* tz = tpm + L1;
  for (int i = threadIdx.x; i < K; i += blockDim.x) cv[i] = make_double2(C[i], C[K + i]);
  for (int e = threadIdx.x; e < L1 * L1; e += blockDim.x) {
    const int l = e / L1, m = e % L1;
    ta[e] = (l >= m + 2) ? sqrt((4.0 * l * l - 1.0) / ((double)l * l - (double)m * m)) : 0.0;
    tb[e] = (l >= m + 2) ? sqrt(((l - 1.0) * (l - 1.0) - (double)m * m) / (4.0 * (l - 1.0) * (l - 1.0) - 1.0)) : 0.0;
  }
  for (int m = threadIdx.x; m < L1; m += blockDim.x) {
    tpm[m] = m > 0 ? sqrt((2.0 * m + 1.0) / (2.0 * m)) : 1.0;
    tz[m] = sqrt(2.0 * m + 3.0);
  }
  __syncthreads();
  const int nc = L1 * L1;
  constexpr double SQ2 = 1.41421356237309504880;
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < ng; g += (int64_t)gridDim.x * blockDim.x) {
    const int64_t pidx = gamma[g];
    const unsigned up = (unsigned)pidx, un = (unsigned)n, q = up / un;
    const int k = (int)(up - q * un), i = (int)(q / un), j = (int)(q - (unsigned)i * un);
    const double X[3] = {lo + (i + 1) * h, lo + (j + 1) * h, lo + (k + 1) * h};
    const double r = sqrt(X[0] * X[0] + X[1] * X[1] + X[2] * X[2]);
    const int bits = assign[g];
    const int cnt = __popc(bits);
    const double inv = cnt ? 1.0 / cnt : 0.0;
    double T[8][2];
#pragma unroll
    for (int c = 0; c < 8; ++c) T[c][0] = T[c][1] = 0.0;
    if (bits & 1) {   // cap
      const double x = X[0] / r, y = X[1] / r, z = X[2] / r;
      const double dcap = r - radius, wc = 0.5 * dcap * dcap;
      double pmm = 0.28209479177387814347, Cm = 1.0, Sm = 0.0;
      for (int m = 0; m <= Lc; ++m) {
        if (m > 0) {
          pmm *= tpm[m];
          const double Cn = x * Cm - y * Sm, Sn = x * Sm + y * Cm;
          Cm = Cn;
          Sm = Sn;
        }
        // (cos | sin part) x (l - m even | odd) x field
        double cE[2] = {0.0, 0.0}, cO[2] = {0.0, 0.0}, sE[2] = {0.0, 0.0}, sO[2] = {0.0, 0.0};
        auto term = [&](int l, double pl, double (&cs)[2], double (&sn)[2]) {
          if (m == 0) {
            const int nu = l * l + l;
            const double2 a = cv[nu], d = cv[nc + nu];
            cs[0] = fma(pl, fma(wc, d.x, a.x), cs[0]);
            cs[1] = fma(pl, fma(wc, d.y, a.y), cs[1]);
          } else {
            const double vc = SQ2 * pl * Cm, vs = SQ2 * pl * Sm;
            const int nup = l * l + l + m, nun = l * l + l - m;
            const double2 ap = cv[nup], dp = cv[nc + nup], an = cv[nun], dn = cv[nc + nun];
            cs[0] = fma(vc, fma(wc, dp.x, ap.x), cs[0]);
            cs[1] = fma(vc, fma(wc, dp.y, ap.y), cs[1]);
            sn[0] = fma(vs, fma(wc, dn.x, an.x), sn[0]);
            sn[1] = fma(vs, fma(wc, dn.y, an.y), sn[1]);
          }
        };
        term(m, pmm, cE, sE);
        double p2 = pmm, p1 = 0.0;
        if (m + 1 <= Lc) {
          p1 = z * tz[m] * pmm;
          term(m + 1, p1, cO, sO);
        }
        for (int l = m + 2; l <= Lc; l += 2) {
          double pl = ta[l * L1 + m] * (z * p1 - tb[l * L1 + m] * p2);
          p2 = p1;
          p1 = pl;
          term(l, pl, cE, sE);
          if (l + 1 <= Lc) {
            pl = ta[(l + 1) * L1 + m] * (z * p1 - tb[(l + 1) * L1 + m] * p2);
            p2 = p1;
            p1 = pl;
            term(l + 1, pl, cO, sO);
          }
        }
        // classes: cos (4(m&1), 0, even|odd) -> 4(m&1) + {0,1}; sin (4((m+1)&1) + 2 + {0,1})
#pragma unroll
        for (int f = 0; f < 2; ++f) {
          if (m & 1) {
            T[4][f] = fma(inv, cE[f], T[4][f]);
            T[5][f] = fma(inv, cO[f], T[5][f]);
            T[2][f] = fma(inv, sE[f], T[2][f]);
            T[3][f] = fma(inv, sO[f], T[3][f]);
          } else {
            T[0][f] = fma(inv, cE[f], T[0][f]);
            T[1][f] = fma(inv, cO[f], T[1][f]);
            T[6][f] = fma(inv, sE[f], T[6][f]);
            T[7][f] = fma(inv, sO[f], T[7][f]);
          }
        }
      }
    }
    auto plane = [&](auto ac) {
      constexpr int a = decltype(ac)::value;
      constexpr int o0 = a == 0 ? 1 : 0, o1 = a == 2 ? 1 : 2;
      constexpr int B0 = 4 >> o0, B1 = 4 >> o1, BA = 4 >> a;
      if (!(bits & (2 << a))) return;
      double Ps[32], Pt[32];
      legendre_all(X[o0], Li, Ps);
      legendre_all(X[o1], Li, Pt);
      const double d = X[a];
      const int cb = 2 * nc + 2 * nphi * a;
      int mi = 0;
      for (int gd = 0; gd <= Li; ++gd) {
        // jj ≡ gd (mod 2): parities (gd&1 on o0, 0 on o1); jj ≢ gd: (~gd&1 on o0, 1 on o1)
        double aS[2] = {0.0, 0.0}, eS[2] = {0.0, 0.0}, aD[2] = {0.0, 0.0}, eD[2] = {0.0, 0.0};
        for (int jj = gd; jj >= 0; jj -= 2) {
          {
            const double phi = Ps[jj] * Pt[gd - jj];
            const double2 av = cv[cb + mi], ev = cv[cb + nphi + mi];
            aS[0] = fma(phi, av.x, aS[0]);
            aS[1] = fma(phi, av.y, aS[1]);
            eS[0] = fma(phi, ev.x, eS[0]);
            eS[1] = fma(phi, ev.y, eS[1]);
            ++mi;
          }
          if (jj >= 1) {
            const double phi = Ps[jj - 1] * Pt[gd - jj + 1];
            const double2 av = cv[cb + mi], ev = cv[cb + nphi + mi];
            aD[0] = fma(phi, av.x, aD[0]);
            aD[1] = fma(phi, av.y, aD[1]);
            eD[0] = fma(phi, ev.x, eD[0]);
            eD[1] = fma(phi, ev.y, eD[1]);
            ++mi;
          }
        }
#pragma unroll
        for (int f = 0; f < 2; ++f) {
          if (gd & 1) {
            T[B0][f] = fma(inv, aS[f], T[B0][f]);
            T[B0 + BA][f] = fma(inv * d, eS[f], T[B0 + BA][f]);
            T[B1][f] = fma(inv, aD[f], T[B1][f]);
            T[B1 + BA][f] = fma(inv * d, eD[f], T[B1 + BA][f]);
          } else {
            T[0][f] = fma(inv, aS[f], T[0][f]);
            T[BA][f] = fma(inv * d, eS[f], T[BA][f]);
            T[B0 + B1][f] = fma(inv, aD[f], T[B0 + B1][f]);
            T[B0 + B1 + BA][f] = fma(inv * d, eD[f], T[B0 + B1 + BA][f]);
          }
        }
      }
    };
    plane(std::integral_constant<int, 0>{});
    plane(std::integral_constant<int, 1>{});
    plane(std::integral_constant<int, 2>{});
    // Walsh-Hadamard: T[s] <- Σ_π (-1)^{popcount(s & π)} T[π]
#pragma unroll
    for (int bit = 1; bit < 8; bit <<= 1)
#pragma unroll
      for (int c = 0; c < 8; ++c)
        if (!(c & bit))
#pragma unroll
          for (int f = 0; f < 2; ++f) {
            const double u = T[c][f], v = T[c | bit][f];
            T[c][f] = u + v;
            T[c | bit][f] = u - v;
          }
    for (int o = 0; o < out.n; ++o) {
      const int so = out.oct[o];
      double v0 = 0.0, v1 = 0.0;
#pragma unroll
      for (int c = 0; c < 8; ++c)
        if (c == so) {
          v0 = T[c][0];
          v1 = T[c][1];
        }
      out.ug[o][g] = clamp ? fmax(v0, 0.0) : v0;
      out.ug[o][ng + g] = clamp ? fmax(v1, 0.0) : v1;
    }
  }
}

// column block of each boundary piece: piece p owns columns [start[p], start[p+1])
struct PieceBlocks {
  int start[6];
  int npieces;
};

// B[i][c] = [c in block(piece_i)] Eraw[pos_i][c] - U_c[gamma[pos_i]]  (column-major n_rows x nc)
__global__ void dd_bep_gather_kernel(const double* __restrict__ U, int ncols, size_t field,
                                     const int64_t* __restrict__ gamma, int64_t ng, const int32_t* __restrict__ rows,
                                     int64_t nrows, const double* __restrict__ Eraw, int c0, PieceBlocks pb,
                                     double* B) {
  const int cl = blockIdx.y;   // column (no per-element 64-bit division)
  for (long ri = blockIdx.x * (long)blockDim.x + threadIdx.x; ri < nrows; ri += (long)gridDim.x * blockDim.x) {
    const int pos = rows[2 * ri], piece = rows[2 * ri + 1];
    const int c = c0 + cl;
    int blk = 0;
    for (int p = 1; p < pb.npieces; ++p) blk += c >= pb.start[p];
    double v = -U[(size_t)cl * field + gamma[pos]];
    if (blk == piece) v += Eraw[(size_t)c * ng + pos];
    B[(size_t)cl * nrows + ri] = v;
  }
}

// g[r][i] = u_r[gamma[pos_i]]  (BEP right-hand sides replicated over a point's pieces)
__global__ void dd_rows_trace_kernel(const double* __restrict__ U, size_t field, const int64_t* __restrict__ gamma,
                                     const int32_t* __restrict__ rows, int64_t nrows, int nrhs, double* g) {
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < nrows; i += (long)gridDim.x * blockDim.x) {
    const int64_t p = gamma[rows[2 * i]];
    for (int r = 0; r < nrhs; ++r) g[(size_t)r * nrows + i] = U[(size_t)r * field + p];
  }
}

__global__ void colsumsq_kernel(const double* __restrict__ B, int64_t m, double* out) {
  const int c = blockIdx.x;
  const double* col = B + (size_t)c * m;
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < m; i += blockDim.x) s = fma(col[i], col[i], s);
  __shared__ double red[TB / 32];
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0;
    for (int q = 0; q < TB / 32; ++q) t += red[q];
    out[c] = t;
  }
}

// R31 initial state: IC at the node on N+ (physical coordinates); on γ the average over the point's
// pieces of the piece's extension of the IC Cauchy data (cap: u0(foot); plane: u0 + d ∂_a u0).
__global__ void dd_ic_kernel(const uint8_t* __restrict__ flags, const int32_t* __restrict__ gmap,
                             const uint8_t* __restrict__ assign, int n, double lo, double h, double radius, double sx,
                             double sy, double sz, dpm_pks_ic ic, double* rho, double* c) {
  const long nn = (long)n * n * n;
  const double sg[3] = {sx, sy, sz};
  for (long p = blockIdx.x * (long)blockDim.x + threadIdx.x; p < nn; p += (long)gridDim.x * blockDim.x) {
    double a = 0.0, b = 0.0;
    if (flags[p] & F_NPLUS) {
      const int i = (int)(p / ((long)n * n)), j = (int)((p / n) % n), k = (int)(p % n);
      const double X[3] = {sg[0] * (lo + (i + 1) * h), sg[1] * (lo + (j + 1) * h), sg[2] * (lo + (k + 1) * h)};
      auto u0 = [&](const double F[3], double amp, double rate) {
        double r2 = 0.0;
        for (int q = 0; q < 3; ++q) r2 += (F[q] - ic.center[q]) * (F[q] - ic.center[q]);
        return amp * exp(-rate * r2);
      };
      const int gp = gmap[p];
      if (gp < 0) {
        a = u0(X, ic.rho_amp, ic.rho_rate);
        b = u0(X, ic.c_amp, ic.c_rate);
      } else {
        const int bits = assign[gp];
        const double r = sqrt(X[0] * X[0] + X[1] * X[1] + X[2] * X[2]);
        int cnt = 0;
        if (bits & 1) {
          const double F[3] = {radius * X[0] / r, radius * X[1] / r, radius * X[2] / r};
          a += u0(F, ic.rho_amp, ic.rho_rate);
          b += u0(F, ic.c_amp, ic.c_rate);
          ++cnt;
        }
        for (int ax = 0; ax < 3; ++ax) {
          if (!(bits & (2 << ax))) continue;
          double F[3] = {X[0], X[1], X[2]};
          F[ax] = 0.0;
          const double d = X[ax];
          const double ur = u0(F, ic.rho_amp, ic.rho_rate), uc = u0(F, ic.c_amp, ic.c_rate);
          a += ur + d * (-2.0 * ic.rho_rate * (F[ax] - ic.center[ax]) * ur);
          b += uc + d * (-2.0 * ic.c_rate * (F[ax] - ic.center[ax]) * uc);
          ++cnt;
        }
        a /= cnt;
        b /= cnt;
      }
    }
    rho[p] = a;
    c[p] = b;
  }
}

int grid_for(long work) { return (int)std::max<long>(1, std::min<long>((work + TB - 1) / TB, 148L * 16)); }

// ---- one operator pass for all octants of a device (dpm_dd_lsq_rhs_shared) ----------------------------
// S_s: the column signs of octant s's extension relative to octant 0's (E_s = E_0 diag(S_s): the cap SH and
// plane Legendre bases are even or odd under each reflection, and the recursions evaluate the reflected
// arguments to exactly ± the same values).  Per column: the γ point of octant 0's largest |E|, and the
// ratio there, required to be exactly ±1 (*bad set otherwise).
__global__ void dd_sign_kernel(const double* __restrict__ E0, const double* __restrict__ Es, int64_t ng,
                               double* sign, int* bad) {
  const int c = blockIdx.x;
  const double* a = E0 + (size_t)c * ng;
  double best = -1.0;
  int64_t arg = 0;
  for (int64_t g = threadIdx.x; g < ng; g += blockDim.x) {
    const double v = fabs(a[g]);
    if (v > best) { best = v; arg = g; }
  }
  __shared__ double sb[TB];
  __shared__ int64_t sa[TB];
  sb[threadIdx.x] = best;
  sa[threadIdx.x] = arg;
  __syncthreads();
  for (int o = TB / 2; o; o >>= 1) {
    if (threadIdx.x < o && (sb[threadIdx.x + o] > sb[threadIdx.x] ||
                            (sb[threadIdx.x + o] == sb[threadIdx.x] && sa[threadIdx.x + o] < sa[threadIdx.x]))) {
      sb[threadIdx.x] = sb[threadIdx.x + o];
      sa[threadIdx.x] = sa[threadIdx.x + o];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const double e0 = a[sa[0]], es = Es[(size_t)c * ng + sa[0]];
    const double r = e0 != 0.0 ? es / e0 : 1.0;
    if (r != 1.0 && r != -1.0) atomicOr(bad, 1);
    sign[c] = r < 0 ? -1.0 : 1.0;
  }
}

// Tall-skinny products of the shared apply on the fp64 tensor pipe (DMMA.m8n8k4):
//   part[split][r][c] = Σ_{i in split} A[c lda + i] X[r m + i]     c < M, r < NR <= 16, i < m
// (A given as M rows of length >= m: the columns of Q_0, or the columns of an upper-triangular K x K
// factor read as the rows of its transpose, TRI = 1 keeping i <= c).  A CTA = 8 warps on one 32-row tile
// (4 m-tiles x 2 n-tiles of 8 per warp) and one i-range of ICH; warp w takes its k-groups of 16 i
// (w, w + 8, ...), lane (g, t) holding i = i0 + 4t + j in k-step j (the same permutation of k for the A
// and B fragments, so each lane reads 4 consecutive doubles per row).  The 8 warps' partial tiles are
// summed in shared memory in warp order; the splits by dd_reduce_kernel in split order (deterministic).
constexpr int TS_ICH = 2048;
template <int TRI>
__global__ void __launch_bounds__(256) dd_gemm_ts_kernel(const double* __restrict__ A, int64_t lda, int M,
                                                         const double* __restrict__ X, int64_t m, int NR,
                                                         double* __restrict__ part) {
  __shared__ double red[8][32][17];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const int c0 = blockIdx.x * 32;
  const int64_t ib = (int64_t)blockIdx.y * TS_ICH, ie = m < ib + TS_ICH ? m : ib + TS_ICH;
  double acc[4][2][2];
  const double* ar[4];
  int cc[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    cc[q] = c0 + 8 * q + g;
    ar[q] = A + (size_t)min(cc[q], M - 1) * lda;
    acc[q][0][0] = acc[q][0][1] = acc[q][1][0] = acc[q][1][1] = 0.0;
  }
  const double* xr[2];
  bool xv[2];
#pragma unroll
  for (int nt = 0; nt < 2; ++nt) {
    xv[nt] = 8 * nt + g < NR;
    xr[nt] = X + (size_t)min(8 * nt + g, NR - 1) * m;
  }
  for (int64_t i0 = ib + 16 * warp; i0 < ie; i0 += 16 * 8) {
    double a[4][4], b[2][4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t i = i0 + 4 * t + j;
      const bool in = i < ie;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const bool ok = in && cc[q] < M && (TRI != 1 || i <= cc[q]);
        a[q][j] = ok ? __ldg(ar[q] + i) : 0.0;
      }
#pragma unroll
      for (int nt = 0; nt < 2; ++nt) b[nt][j] = (in && xv[nt]) ? __ldg(xr[nt] + i) : 0.0;
    }
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int q = 0; q < 4; ++q)
#pragma unroll
        for (int nt = 0; nt < 2; ++nt)
          asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                       : "+d"(acc[q][nt][0]), "+d"(acc[q][nt][1])
                       : "d"(a[q][j]), "d"(b[nt][j]));
  }
#pragma unroll
  for (int q = 0; q < 4; ++q)
#pragma unroll
    for (int nt = 0; nt < 2; ++nt) {
      red[warp][8 * q + g][8 * nt + 2 * t] = acc[q][nt][0];
      red[warp][8 * q + g][8 * nt + 2 * t + 1] = acc[q][nt][1];
    }
  __syncthreads();
  for (int e = threadIdx.x; e < 32 * 16; e += 256) {
    const int cl = e & 31, r = e >> 5;
    if (c0 + cl >= M || r >= NR) continue;
    double v = 0.0;
#pragma unroll
    for (int w = 0; w < 8; ++w) v += red[w][cl][r];
    part[((size_t)blockIdx.y * NR + r) * M + c0 + cl] = v;
  }
}

// out[o][c] = Σ_{v ≡ o mod nout} w[v / nout][c] Σ_split part[split][v][c]   (w nullable: 1), fixed order
__global__ void dd_reduce_kernel(const double* __restrict__ part, int nsplit, int NR, int M,
                                 const double* __restrict__ w, int nout, double* __restrict__ out,
                                 const double* __restrict__ dscale = nullptr) {
  const long tot = (long)nout * M;
  for (long e = blockIdx.x * (long)blockDim.x + threadIdx.x; e < tot; e += (long)gridDim.x * blockDim.x) {
    const int o = (int)(e / M), c = (int)(e - (long)o * M);
    double acc = 0.0;
    for (int v = o; v < NR; v += nout) {
      double sv = 0.0;
      for (int sp = 0; sp < nsplit; ++sp) sv += part[((size_t)sp * NR + v) * M + c];
      acc = w ? fma(w[(size_t)(v / nout) * M + c], sv, acc) : acc + sv;
    }
    out[e] = dscale ? dscale[c] * acc : acc;
  }
}

// part[chunk][r][c] = Σ_{i >= c, i in chunk} W[i K + c] V[r][i]  (W upper col-major; nr <= 2): 32 outputs x
// 8 i-slices per block (coalesced over c), blockIdx.y = i-chunk of UA_CH rows; slices summed in order,
// chunks by dd_reduce_kernel (which applies D)
constexpr int UA_CH = 64;
__global__ void __launch_bounds__(256) dd_upper_apply_kernel(const double* __restrict__ W, int K,
                                                             const double* __restrict__ V, int nr,
                                                             double* __restrict__ part) {
  __shared__ double red[8][2][32];
  const int cl = threadIdx.x & 31, sl = threadIdx.x >> 5, c = blockIdx.x * 32 + cl;
  const int ib = blockIdx.y * UA_CH, ie = min(K, ib + UA_CH);
  double a0 = 0.0, a1 = 0.0;
  if (c < K)
#pragma unroll 4
    for (int i = max(c, ib) + ((sl - max(c, ib) % 8 + 8) % 8); i < ie; i += 8) {
      const double wv = W[(size_t)i * K + c];
      a0 = fma(wv, V[i], a0);
      if (nr > 1) a1 = fma(wv, V[K + i], a1);
    }
  red[sl][0][cl] = a0;
  red[sl][1][cl] = a1;
  __syncthreads();
  if (sl < nr && c < K) {
    double v = 0.0;
#pragma unroll
    for (int q = 0; q < 8; ++q) v += red[q][sl][cl];
    part[((size_t)blockIdx.y * nr + sl) * K + c] = v;
  }
}

// the stacked column signs of the octants (one launch instead of a copy per octant)
struct SignPtrs {
  const double* p[8];
};
__global__ void dd_stack_signs_kernel(SignPtrs sp, int noct, int K, double* Sg) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < noct * K; e += gridDim.x * blockDim.x)
    Sg[e] = sp.p[e / K][e % K];
}

// ---- NEXT-3: the paper's two-subdomain DD, Case 1 (concentric, Z ∩ Γ = ∅) ----
// Pieces: Z (the interface |x| = r1, piece 0, bit 1) and Γ (|x| = r2, piece 1, bit 2).  Ω1 (sub 0):
// every point of ζ1 is on Z; Ω2 (sub 1): a point of γ ∪ ζ2 is on the nearer sphere (reading R38).
// Columns (zonal basis φ_l = P_l(cos θ), cos θ = x_z/|x|):
//   Z: [φ | d φ | (d²/2) φ], l <= mz, d = |x| - r1 (3-term, u, ∂_n u, ∂²_n u shared by Ω1 and Ω2:
//      the interface conditions P:477-480);   Γ: [φ | (d²/2) φ], l <= mg, d = |x| - r2 (zero Neumann).
__device__ __forceinline__ int dd1_piece(int sub, double r, double r1, double r2) {
  return (sub == 0 || fabs(r - r1) < fabs(r - r2)) ? 0 : 1;
}

__global__ void dd1_extension_kernel(const int64_t* gamma, int64_t ng, int n, double lo, double h, int sub,
                                     double r1, double r2, int mz, int mg, int K, double* Eraw, double* A,
                                     uint8_t* assign) {
  const long g = blockIdx.x * (long)blockDim.x + threadIdx.x;
  if (g >= ng) return;
  const int64_t pidx = gamma[g];
  const int i = (int)(pidx / ((long)n * n)), j = (int)((pidx / n) % n), k = (int)(pidx % n);
  const double P[3] = {lo + (i + 1) * h, lo + (j + 1) * h, lo + (k + 1) * h};
  const double r = sqrt(P[0] * P[0] + P[1] * P[1] + P[2] * P[2]);
  const int piece = dd1_piece(sub, r, r1, r2);
  assign[g] = (uint8_t)(1 << piece);
  for (int c = 0; c < K; ++c) {
    Eraw[(size_t)c * ng + g] = 0.0;
    A[(size_t)c * ng + g] = 0.0;
  }
  const double x = fmin(fmax(P[2] / r, -1.0), 1.0);
  const int M = piece == 0 ? mz : mg;
  const double d = r - (piece == 0 ? r1 : r2);
  const double w2 = 0.5 * (d * d);
  const int c0 = piece == 0 ? 0 : 3 * (mz + 1);
  double pm = 1.0, pl = x;
  for (int l = 0; l <= M; ++l) {   // Bonnet: (l+1) P_{l+1} = (2l+1) x P_l - l P_{l-1}
    const double v = l == 0 ? 1.0 : pl;
    double cols[3];
    int nc = 0;
    cols[nc++] = v;
    if (piece == 0) cols[nc++] = d * v;
    cols[nc++] = w2 * v;
    for (int q = 0; q < nc; ++q) {
      const size_t c = (size_t)(c0 + q * (M + 1) + l);
      Eraw[c * ng + g] = cols[q];
      A[c * ng + g] = cols[q];
    }
    if (l >= 1) {
      const double nx = ((2 * l + 1) * x * pl - l * pm) / (l + 1);
      pm = pl;
      pl = nx;
    }
  }
}

// Initial state (R38): the IC at the node on N+, except on Γ's γ points (the foot r2 x/|x|, R14); with
// ic.rho_cell_average, ρ̄ is the cell average (R36) on M+ and on the interface points ζ.
__global__ void dd1_ic_kernel(const uint8_t* __restrict__ flags, const int32_t* __restrict__ gmap,
                              const uint8_t* __restrict__ assign, int n, double lo, double h, double r2, dpm_pks_ic ic,
                              double* rho, double* c) {
  const long nn = (long)n * n * n;
  for (long p = blockIdx.x * (long)blockDim.x + threadIdx.x; p < nn; p += (long)gridDim.x * blockDim.x) {
    const uint8_t f = flags[p];
    double a = 0.0, b = 0.0;
    if (f & F_NPLUS) {
      const int i = (int)(p / ((long)n * n)), j = (int)((p / n) % n), k = (int)(p % n);
      double X[3] = {lo + (i + 1) * h, lo + (j + 1) * h, lo + (k + 1) * h};
      const int gp = gmap[p];
      const bool onG = gp >= 0 && (assign[gp] & 2);
      auto gauss = [&](const double F[3], double amp, double rate) {
        double q2 = 0.0;
        for (int q = 0; q < 3; ++q) q2 += (F[q] - ic.center[q]) * (F[q] - ic.center[q]);
        return amp * exp(-rate * q2);
      };
      a = gauss(X, ic.rho_amp, ic.rho_rate);
      b = gauss(X, ic.c_amp, ic.c_rate);
      if (ic.rho_cell_average && ((f & F_MPLUS) || (gp >= 0 && (assign[gp] & 1)))) {
        auto avg1 = [&](double s) {
          const double q = sqrt(ic.rho_rate);
          return 0.88622692545275801365 / q * (erf(q * (s + 0.5 * h)) - erf(q * (s - 0.5 * h))) / h;
        };
        a = ic.rho_amp * avg1(X[0] - ic.center[0]) * avg1(X[1] - ic.center[1]) * avg1(X[2] - ic.center[2]);
      }
      if (onG) {
        const double r = sqrt(X[0] * X[0] + X[1] * X[1] + X[2] * X[2]);
        const double F[3] = {r2 * (X[0] / r), r2 * (X[1] / r), r2 * (X[2] / r)};
        a = gauss(F, ic.rho_amp, ic.rho_rate);
        b = gauss(F, ic.c_amp, ic.c_rate);
      }
    }
    rho[p] = a;
    c[p] = b;
  }
}

}  // namespace

dpm_status dd_setup(dpm_ctx* ctx) {
  const int64_t ng = ctx->counts[DPM_SET_GAMMA], ngin = ctx->counts[DPM_SET_GAMMA_IN];
  cudaStream_t s = ctx->setup_stream;
  const int K = ctx->K;
  DPM_CUDA_TRY(ctx, cudaMalloc(&ctx->dd_Eraw, (size_t)ng * K * sizeof(double)));
  DPM_CUDA_TRY(ctx, cudaMalloc(&ctx->E, (size_t)ng * K * sizeof(double)));
  DPM_CUDA_TRY(ctx, cudaMalloc(&ctx->dd_assign, std::max<int64_t>(ng, 1)));
  DPM_CUDA_TRY(ctx, cudaMalloc(&ctx->foot, 8));   // unused for octants (IC computed from geometry)
  DPM_CUDA_TRY(ctx, cudaMalloc(&ctx->dist, 8));
  DPM_COUNT_LAUNCH(1);
  if (ctx->dd == 2)
    dd1_extension_kernel<<<(unsigned)((ng + 127) / 128), 128, 0, s>>>(
        ctx->lists[DPM_SET_GAMMA], ng, ctx->n, ctx->lo, ctx->h, ctx->dd1_sub, ctx->dd1_r1, ctx->dd1_r2, ctx->dd1_mz,
        ctx->dd1_mg, K, ctx->dd_Eraw, ctx->E, ctx->dd_assign);
  else
    dd_extension_kernel<<<(unsigned)((ng + 127) / 128), 128, 0, s>>>(
        ctx->lists[DPM_SET_GAMMA], ng, ctx->n, ctx->lo, ctx->h, ctx->radius, ctx->sigma[0], ctx->sigma[1],
        ctx->sigma[2], ctx->Lc, ctx->Li, ctx->nphi, K, ctx->dd_Eraw, ctx->E, ctx->dd_assign);
  DPM_CUDA_TRY(ctx, cudaGetLastError());
  // BEP rows: γ_in points (ascending) x their pieces (cap, x, y, z order)
  std::vector<uint8_t> bits(ng);
  std::vector<int32_t> ginpos(ngin);
  DPM_CUDA_TRY(ctx, cudaMemcpyAsync(bits.data(), ctx->dd_assign, ng, cudaMemcpyDeviceToHost, s));
  DPM_CUDA_TRY(ctx, cudaMemcpyAsync(ginpos.data(), ctx->gin_pos, ngin * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  DPM_CUDA_TRY(ctx, cudaStreamSynchronize(s));
  std::vector<int32_t> rows;
  for (int64_t i = 0; i < ng; ++i)
    if (bits[i] == 0) {
      ctx->err = "DD: a gamma point is on no boundary piece";
      return DPM_ERR_INVALID;
    }
  for (int64_t q = 0; q < ngin; ++q)
    for (int pc = 0; pc < 4; ++pc)
      if (bits[ginpos[q]] & (1 << pc)) {
        rows.push_back(ginpos[q]);
        rows.push_back(pc);
      }
  ctx->n_rows = (int64_t)rows.size() / 2;
  DPM_CUDA_TRY(ctx, cudaMalloc(&ctx->dd_rows, std::max<size_t>(rows.size(), 2) * sizeof(int32_t)));
  DPM_CUDA_TRY(ctx, cudaMemcpy(ctx->dd_rows, rows.data(), rows.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
  return DPM_OK;
}

namespace {
cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

dpm_status dd_check(dpm_ctx* ctx) {
  if (!ctx) return DPM_ERR_INVALID;
  if (!ctx->dd) { ctx->err = "not a DD subdomain context"; return DPM_ERR_INVALID; }
  cudaSetDevice(ctx->device);
  return DPM_OK;
}

dpm_status dd_alloc(dpm_ctx* ctx) {
  const size_t K = ctx->K, m = (size_t)std::max<int64_t>(ctx->n_rows, 1);
  if (!ctx->dd_B) DPM_CUDA_TRY(ctx, cudaMalloc(&ctx->dd_B, K * m * sizeof(double)));
  if (!ctx->dd_Q) DPM_CUDA_TRY(ctx, cudaMalloc(&ctx->dd_Q, K * m * sizeof(double)));
  if (!ctx->dd_M) DPM_CUDA_TRY(ctx, cudaMalloc(&ctx->dd_M, K * m * sizeof(double)));
  if (!ctx->dd_R) DPM_CUDA_TRY(ctx, cudaMalloc(&ctx->dd_R, 5 * K * K * sizeof(double) + 64));   // R1 R2 R W W2 fail
  if (!ctx->dd_D) DPM_CUDA_TRY(ctx, cudaMalloc(&ctx->dd_D, K * sizeof(double)));
  if (!ctx->dd_g) DPM_CUDA_TRY(ctx, cudaMalloc(&ctx->dd_g, 2 * m * sizeof(double)));
  return DPM_OK;
}
}  // namespace

namespace {
// u_γ = A C (R17), the basis evaluated on the fly (dd_extend_fly_kernel); ug: 2 x n_gamma
cudaError_t dd_extend_fly(dpm_ctx* ctx, const double* C, int clamp, double* ug, cudaStream_t s) {
  const int64_t ng = ctx->counts[DPM_SET_GAMMA];
  if (ctx->dd == 2) return lsq_extend(ctx->E, ng, ctx->K, C, 2, clamp, ug, s);   // A is small: |γ| x K
  const int L1 = ctx->Lc + 1;
  const size_t smem = (2 * (size_t)ctx->K + 2 * L1 * L1 + 2 * L1) * sizeof(double);
  cudaError_t e = cudaFuncSetAttribute(dd_extend_fly_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  DPM_COUNT_LAUNCH(1);
  dd_extend_fly_kernel<<<(unsigned)std::min<int64_t>((ng + 127) / 128, 148 * 8), 128, smem, s>>>(
      ctx->lists[DPM_SET_GAMMA], ng, ctx->n, ctx->lo, ctx->h, ctx->radius, ctx->sigma[0], ctx->sigma[1], ctx->sigma[2],
      ctx->Lc, ctx->Li, ctx->nphi, ctx->K, ctx->dd_assign, C, clamp, ug);
  return cudaGetLastError();
}
}  // namespace

extern "C" {

dpm_status dpm_create_octant(const dpm_grid* grid, int32_t octant, double radius, int32_t lmax_cap, int32_t deg_if,
                             double dt, int32_t device, dpm_ctx** out) {
  DPM_NVTX();
  if (out) *out = nullptr;
  if (!grid || !out || octant < 0 || octant > 7 || !(radius > 0) || lmax_cap < 0 || lmax_cap > 40 || deg_if < 0 ||
      deg_if > 30 || !(grid->lo < 0 && grid->hi > radius))
    return DPM_ERR_INVALID;
  dpm_domain D{};
  D.kind = DPM_OCTANT_CANON;
  D.semi[0] = D.semi[1] = D.semi[2] = radius;
  // dpm_create validates the grid and builds the point sets + AP plan; the extension data is ours
  dpm_status st = dpm_create_impl(grid, &D, 0, dt, DPM_BASIS_NEUMANN0, device, out);
  if (st != DPM_OK) return st;
  dpm_ctx* ctx = *out;
  ctx->dd = 1;
  ctx->octant = octant;
  for (int a = 0; a < 3; ++a) ctx->sigma[a] = ((octant >> (2 - a)) & 1) ? -1.0 : 1.0;
  ctx->radius = radius;
  ctx->Lc = lmax_cap;
  ctx->Li = deg_if;
  ctx->nphi = (deg_if + 1) * (deg_if + 2) / 2;
  ctx->K = 2 * (lmax_cap + 1) * (lmax_cap + 1) + 6 * ctx->nphi;
  ctx->lmax = lmax_cap;
  ctx->dd_npieces = 4;
  ctx->dd_blk[0] = 0;
  for (int p = 1; p <= 4; ++p) ctx->dd_blk[p] = 2 * (lmax_cap + 1) * (lmax_cap + 1) + 2 * ctx->nphi * (p - 1);
  if (ctx->E) { cudaFree(ctx->E); ctx->E = nullptr; }
  if (ctx->foot) { cudaFree(ctx->foot); ctx->foot = nullptr; }
  if (ctx->dist) { cudaFree(ctx->dist); ctx->dist = nullptr; }
  st = dd_setup(ctx);
  if (st != DPM_OK) {
    dpm_destroy(ctx);
    *out = nullptr;
  }
  return st;
}

dpm_status dpm_create_dd1(const dpm_grid* grid, int32_t sub, double r1, double r2, int32_t mz, int32_t mg, double dt,
                          int32_t device, dpm_ctx** out) {
  DPM_NVTX();
  if (out) *out = nullptr;
  if (!grid || !out || (sub != 0 && sub != 1) || !(r1 > 0) || !(r2 > r1) || mz < 0 || mg < 0 ||
      mz > DPM_MAX_ZONAL_L || mg > DPM_MAX_ZONAL_L)
    return DPM_ERR_INVALID;
  const double ro = sub == 0 ? r1 : r2;
  if (!(grid->lo < -ro && grid->hi > ro)) return DPM_ERR_INVALID;   // the subdomain strictly inside the box
  dpm_domain D{};
  if (sub == 0) {
    D.kind = DPM_SPHERE;
    D.semi[0] = D.semi[1] = D.semi[2] = r1;
  } else {
    D.kind = DPM_SHELL_CANON;
    D.semi[0] = r2;
    D.semi[1] = r1;
  }
  // dpm_create validates the grid and builds the point sets + AP plan; the extension data is ours
  dpm_status st = dpm_create_impl(grid, &D, 0, dt, DPM_BASIS_NEUMANN0_2TERM_ZONAL, device, out);
  if (st != DPM_OK) return st;
  dpm_ctx* ctx = *out;
  ctx->dd = 2;
  ctx->dd1_sub = sub;
  ctx->dd1_r1 = r1;
  ctx->dd1_r2 = r2;
  ctx->dd1_mz = mz;
  ctx->dd1_mg = mg;
  ctx->radius = ro;
  ctx->K = 3 * (mz + 1) + 2 * (mg + 1);
  ctx->lmax = mz;
  ctx->dd_npieces = 2;
  ctx->dd_blk[0] = 0;
  ctx->dd_blk[1] = 3 * (mz + 1);
  ctx->dd_blk[2] = ctx->K;
  if (ctx->E) { cudaFree(ctx->E); ctx->E = nullptr; }
  if (ctx->foot) { cudaFree(ctx->foot); ctx->foot = nullptr; }
  if (ctx->dist) { cudaFree(ctx->dist); ctx->dist = nullptr; }
  st = dd_setup(ctx);
  if (st != DPM_OK) {
    dpm_destroy(ctx);
    *out = nullptr;
  }
  return st;
}

dpm_status dpm_dd_info(const dpm_ctx* ctx, int64_t* n_rows, int32_t* K) {
  DPM_NVTX();
  if (!ctx || !ctx->dd || !n_rows || !K) return DPM_ERR_INVALID;
  *n_rows = ctx->n_rows;
  *K = ctx->K;
  return DPM_OK;
}

dpm_status dpm_dd_copy_assign(const dpm_ctx* ctx, uint8_t* host_bits) {
  DPM_NVTX();
  if (!ctx || !ctx->dd || !host_bits) return DPM_ERR_INVALID;
  cudaSetDevice(ctx->device);
  dpm_ctx* c = const_cast<dpm_ctx*>(ctx);
  DPM_CUDA_TRY(c, cudaMemcpy(host_bits, ctx->dd_assign, ctx->counts[DPM_SET_GAMMA], cudaMemcpyDeviceToHost));
  return DPM_OK;
}

dpm_status dpm_dd_bep_block(dpm_ctx* ctx, double* B_out, void* stream) {
  DPM_NVTX();
  dpm_status st = dd_check(ctx);
  if (st != DPM_OK) return st;
  if ((st = dd_alloc(ctx)) != DPM_OK) return st;
  cudaStream_t s = as_stream(stream);
  const size_t field = (size_t)ctx->n * ctx->n * ctx->n;
  const int K = ctx->K;
  const int64_t ng = ctx->counts[DPM_SET_GAMMA];
  const int ch = (int)std::max<size_t>(1, std::min<size_t>((size_t)K, ((size_t)2 << 30) / (field * 8)));
  if (ctx->work_boxes < (size_t)std::min(ch, K)) {
    if (ctx->work) cudaFree(ctx->work);
    ctx->work = nullptr;
    ctx->work_boxes = 0;
    DPM_CUDA_TRY(ctx, cudaMalloc(&ctx->work, (size_t)std::min(ch, K) * field * sizeof(double)));
    ctx->work_boxes = std::min(ch, K);
  }
  for (int a = 0; a < K; a += ch) {
    const int ncol = std::min(ch, K - a);
    if (bep_zbox_enabled() && ctx->K >= 128 && ctx->plan.solver == DPM_SOLVER_DST2_TRIDIAG) {   // (as dpm_bep_columns)
      double* zb = nullptr;
      DPM_CUDA_TRY(ctx, bep_zbox(ctx, ncol, &zb, s));
      DPM_CUDA_TRY(ctx, launch_potential_scatter(ctx, ctx->E + (size_t)a * ng, ng, zb, ncol, s));
      DPM_CUDA_TRY(ctx, dst_solve_batch(ctx->plan, zb, ctx->work, ncol, nullptr, 0, s));
    } else {
      DPM_CUDA_TRY(ctx, launch_potential_rhs(ctx, ctx->E + (size_t)a * ng, ng, ctx->work, ncol, s));
      DPM_CUDA_TRY(ctx, dst_solve_batch(ctx->plan, ctx->work, ctx->work, ncol, nullptr, 0, s));
    }
    DPM_COUNT_LAUNCH(1);
    PieceBlocks pb{};
    pb.npieces = ctx->dd_npieces;
    for (int p = 0; p <= ctx->dd_npieces && p < 6; ++p) pb.start[p] = ctx->dd_blk[p];
    dd_bep_gather_kernel<<<dim3((unsigned)std::max<int64_t>(1, std::min<int64_t>((ctx->n_rows + TB - 1) / TB, 148L * 16)), ncol), TB, 0, s>>>(
        ctx->work, ncol, field, ctx->lists[DPM_SET_GAMMA], ng, ctx->dd_rows, ctx->n_rows, ctx->dd_Eraw, a, pb,
        ctx->dd_B + (size_t)a * ctx->n_rows);
    DPM_CUDA_TRY(ctx, cudaGetLastError());
  }
  if (B_out)
    DPM_CUDA_TRY(ctx, cudaMemcpyAsync(B_out, ctx->dd_B, (size_t)K * ctx->n_rows * 8, cudaMemcpyDeviceToDevice, s));
  ctx->have_projection = 0;
  ctx->dt_bep = ctx->dt;
  return DPM_OK;
}

dpm_status dpm_dd_colnorm2(dpm_ctx* ctx, double* nrm2, void* stream) {
  DPM_NVTX();
  dpm_status st = dd_check(ctx);
  if (st != DPM_OK) return st;
  if (!nrm2 || !ctx->dd_B) return DPM_ERR_STATE;
  DPM_COUNT_LAUNCH(1);
  colsumsq_kernel<<<ctx->K, TB, 0, as_stream(stream)>>>(ctx->dd_B, ctx->n_rows, nrm2);
  DPM_CUDA_TRY(ctx, cudaGetLastError());
  return DPM_OK;
}

dpm_status dpm_dd_gram(dpm_ctx* ctx, int32_t pass, const double* nrm2_sum, double* G, void* stream) {
  DPM_NVTX();
  dpm_status st = dd_check(ctx);
  if (st != DPM_OK) return st;
  if (!G || !ctx->dd_B || (pass != 1 && pass != 2) || (pass == 1 && !nrm2_sum)) return DPM_ERR_INVALID;
  cudaStream_t s = as_stream(stream);
  const int K = ctx->K;
  if (pass == 1) {   // D = 1/||column|| of the stacked system; Q1 <- B D
    std::vector<double> h(K);
    DPM_CUDA_TRY(ctx, cudaMemcpyAsync(h.data(), nrm2_sum, K * 8, cudaMemcpyDeviceToHost, s));
    DPM_CUDA_TRY(ctx, cudaStreamSynchronize(s));
    for (int c = 0; c < K; ++c) h[c] = h[c] > 0 ? 1.0 / std::sqrt(h[c]) : 1.0;
    DPM_CUDA_TRY(ctx, cudaMemcpyAsync(ctx->dd_D, h.data(), K * 8, cudaMemcpyHostToDevice, s));
    DPM_CUDA_TRY(ctx, lsq_scale_cols(ctx->dd_B, ctx->n_rows, K, ctx->dd_D, ctx->dd_Q, s));
  }
  DPM_CUDA_TRY(ctx, lsq_gram(ctx->dd_Q, ctx->n_rows, K, G, s));
  return DPM_OK;
}

// dd_R layout: R1 | R2 | R = R2 R1 | W = Rp^{-1} of the last pass | W2 = R^{-1} | fail flag
dpm_status dpm_dd_chol(dpm_ctx* ctx, int32_t pass, const double* G_sum, void* stream) {
  DPM_NVTX();
  dpm_status st = dd_check(ctx);
  if (st != DPM_OK) return st;
  if (!G_sum || (pass != 1 && pass != 2)) return DPM_ERR_INVALID;
  cudaStream_t s = as_stream(stream);
  const size_t K = ctx->K;
  double* R1 = ctx->dd_R;
  double* R2 = R1 + K * K;
  double* R = R2 + K * K;
  double* W = R + K * K;
  double* W2 = W + K * K;
  int* dfail = reinterpret_cast<int*>(W2 + K * K);
  double* Rp = pass == 1 ? R1 : R2;
  DPM_CUDA_TRY(ctx, cudaMemcpyAsync(Rp, G_sum, K * K * 8, cudaMemcpyDeviceToDevice, s));
  DPM_CUDA_TRY(ctx, cudaMemsetAsync(dfail, 0, sizeof(int), s));
  DPM_CUDA_TRY(ctx, lsq_cholesky(Rp, (int)K, dfail, s));
  // Q <- Q Rp^{-1}: explicit triangular inverse W, then a tiled GEMM (into dd_M, then swap)
  DPM_CUDA_TRY(ctx, lsq_rinv(Rp, (int)K, W, s));
  DPM_CUDA_TRY(ctx, lsq_mul_upper(ctx->dd_Q, ctx->n_rows, (int)K, W, ctx->dd_M, s));
  std::swap(ctx->dd_Q, ctx->dd_M);
  if (pass == 2) {
    DPM_CUDA_TRY(ctx, lsq_trmm(R2, R1, R, (int)K, s));
    DPM_CUDA_TRY(ctx, lsq_rinv(R, (int)K, W2, s));
    DPM_CUDA_TRY(ctx, lsq_operator_from_rinv(W2, ctx->dd_Q, ctx->n_rows, (int)K, ctx->dd_D, ctx->dd_M, s));
  }
  int hfail = 0;
  DPM_CUDA_TRY(ctx, cudaMemcpyAsync(&hfail, dfail, sizeof(int), cudaMemcpyDeviceToHost, s));
  DPM_CUDA_TRY(ctx, cudaStreamSynchronize(s));
  if (hfail) { ctx->err = "octant DD: CholeskyQR2 breakdown (stacked BEP rank deficient)"; return DPM_ERR_RANK; }
  if (pass == 2) ctx->have_projection = 1;
  return DPM_OK;
}

// The same pass from an octant already factored with the same summed Gram on this device: the
// K x K factors and inverses are copied, only the octant's own GEMMs run.
dpm_status dpm_dd_chol_copy(dpm_ctx* ctx, int32_t pass, const dpm_ctx* src, void* stream) {
  DPM_NVTX();
  dpm_status st = dd_check(ctx);
  if (st != DPM_OK) return st;
  if (!src || !src->dd || !src->dd_R || src->K != ctx->K || src->device != ctx->device || (pass != 1 && pass != 2))
    return DPM_ERR_INVALID;
  if (pass == 2 && !src->have_projection) { ctx->err = "dd_chol_copy: source not factored"; return DPM_ERR_STATE; }
  cudaStream_t s = as_stream(stream);
  const size_t K = ctx->K, KK = K * K * 8;
  double* R1 = ctx->dd_R;
  double* R2 = R1 + K * K;
  double* R = R2 + K * K;
  double* W = R + K * K;
  double* W2 = W + K * K;
  const double* sR1 = src->dd_R;
  if (pass == 1) {
    DPM_CUDA_TRY(ctx, cudaMemcpyAsync(R1, sR1, KK, cudaMemcpyDeviceToDevice, s));
    DPM_CUDA_TRY(ctx, cudaMemcpyAsync(W, sR1 + 3 * K * K, KK, cudaMemcpyDeviceToDevice, s));
  } else {   // R2, R, W = R2^{-1}, W2 = R^{-1}
    DPM_CUDA_TRY(ctx, cudaMemcpyAsync(R2, sR1 + K * K, 4 * KK, cudaMemcpyDeviceToDevice, s));
  }
  DPM_CUDA_TRY(ctx, lsq_mul_upper(ctx->dd_Q, ctx->n_rows, (int)K, W, ctx->dd_M, s));
  std::swap(ctx->dd_Q, ctx->dd_M);
  if (pass == 2) {
    DPM_CUDA_TRY(ctx, lsq_operator_from_rinv(W2, ctx->dd_Q, ctx->n_rows, (int)K, ctx->dd_D, ctx->dd_M, s));
    ctx->have_projection = 1;
  }
  DPM_CUDA_TRY(ctx, cudaGetLastError());
  return DPM_OK;
}

dpm_status dpm_dd_pks_init(dpm_ctx* ctx, double* rho, double* c, const dpm_pks_ic* ic, void* stream) {
  DPM_NVTX();
  dpm_status st = dd_check(ctx);
  if (st != DPM_OK) return st;
  if (!rho || !c || !ic) return DPM_ERR_INVALID;
  const long nn = (long)ctx->n * ctx->n * ctx->n;
  DPM_COUNT_LAUNCH(1);
  if (ctx->dd == 2)
    dd1_ic_kernel<<<grid_for(nn), TB, 0, as_stream(stream)>>>(ctx->flags, ctx->gmap, ctx->dd_assign, ctx->n, ctx->lo,
                                                              ctx->h, ctx->dd1_r2, *ic, rho, c);
  else
    dd_ic_kernel<<<grid_for(nn), TB, 0, as_stream(stream)>>>(ctx->flags, ctx->gmap, ctx->dd_assign, ctx->n, ctx->lo,
                                                             ctx->h, ctx->radius, ctx->sigma[0], ctx->sigma[1],
                                                             ctx->sigma[2], *ic, rho, c);
  DPM_CUDA_TRY(ctx, cudaGetLastError());
  return DPM_OK;
}

dpm_status dpm_dd_cfl(dpm_ctx* ctx, const double* c, double chi, double* cfl_dt, void* stream) {
  DPM_NVTX();
  dpm_status st = dd_check(ctx);
  if (st != DPM_OK) return st;
  if (!c || !(chi > 0)) return DPM_ERR_INVALID;
  cudaStream_t s = as_stream(stream);
  DPM_CUDA_TRY(ctx, launch_cfl_reduce(ctx, c, ctx->red, s));
  DPM_CUDA_TRY(ctx, cudaMemcpyAsync(ctx->red_host, ctx->red, 3 * sizeof(double), cudaMemcpyDeviceToHost, s));
  if (!cfl_dt) return DPM_OK;   // asynchronous form: dpm_dd_cfl_result() later
  return dpm_dd_cfl_result(ctx, chi, cfl_dt, stream);
}

dpm_status dpm_dd_cfl_result(dpm_ctx* ctx, double chi, double* cfl_dt, void* stream) {
  DPM_NVTX();
  dpm_status st = dd_check(ctx);
  if (st != DPM_OK) return st;
  if (!cfl_dt || !(chi > 0)) return DPM_ERR_INVALID;
  DPM_CUDA_TRY(ctx, cudaStreamSynchronize(as_stream(stream)));
  const double h = ctx->h;
  double cfl = INFINITY;
  for (int a = 0; a < 3; ++a) {
    const double mx = ctx->red_host[a] / h;
    if (mx > 0) cfl = std::fmin(cfl, h / (6.0 * chi * mx));
  }
  *cfl_dt = cfl;
  return DPM_OK;
}


// Phase-level pieces of the DD step (caller-owned 2-field buffers), so that a rank can run each of
// the step's two AP solves for all its octants as one batched dpm_aux_solve_batch (the AP operator
// depends only on n, h and dt, shared by the octants).  local_begin = rhs + solve + lsq_rhs;
// local_finish = green_rhs + solve + restrict.
dpm_status dpm_dd_rhs(dpm_ctx* ctx, const double* rho, const double* c, double chi, double* fq, void* stream) {
  DPM_NVTX();
  dpm_status st = dd_check(ctx);
  if (st != DPM_OK) return st;
  if (!rho || !c || !fq) return DPM_ERR_INVALID;
  if (!ctx->have_projection || ctx->dt_bep != ctx->dt) { ctx->err = "octant DD: no factorisation at this dt"; return DPM_ERR_STATE; }
  const size_t field = (size_t)ctx->n * ctx->n * ctx->n;
  DPM_CUDA_TRY(ctx, launch_flux_rhs(ctx, rho, c, ctx->dt, chi, fq, fq + field, as_stream(stream)));   // Step 4a
  return DPM_OK;
}

dpm_status dpm_dd_lsq_rhs(dpm_ctx* ctx, const double* wk, double* y, void* stream) {
  DPM_NVTX();
  dpm_status st = dd_check(ctx);
  if (st != DPM_OK) return st;
  if (!wk || !y) return DPM_ERR_INVALID;
  cudaStream_t s = as_stream(stream);
  const size_t field = (size_t)ctx->n * ctx->n * ctx->n;
  if (!ctx->dd_g) return DPM_ERR_STATE;
  DPM_COUNT_LAUNCH(1);
  dd_rows_trace_kernel<<<grid_for(ctx->n_rows), TB, 0, s>>>(wk, field, ctx->lists[DPM_SET_GAMMA], ctx->dd_rows,
                                                                ctx->n_rows, 2, ctx->dd_g);
  DPM_CUDA_TRY(ctx, cudaGetLastError());
  DPM_CUDA_TRY(ctx, lsq_gemv(ctx->dd_M, ctx->n_rows, ctx->K, ctx->dd_g, 2, y, s));           // y_s = M_s g_s
  return DPM_OK;
}

// o->dd_sign: the column signs S of octant o's extension relative to o0's (E_o = E_0 diag(S)); computed once
// per pair (one host sync), DPM_ERR_INVALID (error on o0) if the extensions are not sign reflections
dpm_status dd_signs(dpm_ctx* o0, dpm_ctx* o, cudaStream_t s) {
  if (o->dd_sign && o->dd_sign_ref == o0) return DPM_OK;
  const int K = o0->K;
  const int64_t ng = o0->counts[DPM_SET_GAMMA];
  if (!o->dd_sign) DPM_CUDA_TRY(o0, cudaMalloc(&o->dd_sign, (size_t)K * sizeof(double) + 16));
  int* dbad = reinterpret_cast<int*>(o->dd_sign + K);
  DPM_CUDA_TRY(o0, cudaMemsetAsync(dbad, 0, sizeof(int), s));
  DPM_COUNT_LAUNCH(1);
  dd_sign_kernel<<<K, TB, 0, s>>>(o0->dd_Eraw, o->dd_Eraw, ng, o->dd_sign, dbad);
  int hbad = 0;
  DPM_CUDA_TRY(o0, cudaMemcpyAsync(&hbad, dbad, sizeof(int), cudaMemcpyDeviceToHost, s));
  DPM_CUDA_TRY(o0, cudaStreamSynchronize(s));
  if (hbad) { o0->err = "the octant extensions are not sign-reflections"; return DPM_ERR_INVALID; }
  o->dd_sign_ref = o0;
  return DPM_OK;
}

__global__ void dd_signed_copy_kernel(const double* __restrict__ B0, int64_t m, const double* __restrict__ sign,
                                      double* __restrict__ B) {
  const int c = blockIdx.y;
  const double sg = sign[c];
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
    B[(size_t)c * m + i] = sg * B0[(size_t)c * m + i];
}

dpm_status dpm_dd_bep_block_from(dpm_ctx* ctx, dpm_ctx* ref, double* B_out, void* stream) {
  DPM_NVTX();
  dpm_status st = dd_check(ctx);
  if (st != DPM_OK) return st;
  if (!ref || ref->dd != 1 || ctx->dd != 1 || ref->device != ctx->device || ref->n != ctx->n || ref->lo != ctx->lo ||
      ref->hi != ctx->hi || ref->K != ctx->K || ref->n_rows != ctx->n_rows || ref->radius != ctx->radius) {
    ctx->err = "dd_bep_block_from: the contexts are not octants of one canonical geometry on one device";
    return DPM_ERR_INVALID;
  }
  if (!ref->dd_B || ref->dt_bep != ctx->dt || ref->dt != ctx->dt) {
    ctx->err = "dd_bep_block_from: the reference block is not built at this dt";
    return DPM_ERR_STATE;
  }
  if ((st = dd_alloc(ctx)) != DPM_OK) return st;
  cudaStream_t s = as_stream(stream);
  if ((st = dd_signs(ref, ctx, s)) != DPM_OK) {
    ctx->err = ref->err;
    return st;
  }
  const int64_t m = ctx->n_rows;
  DPM_COUNT_LAUNCH(1);
  dd_signed_copy_kernel<<<dim3((unsigned)std::max<int64_t>(1, std::min<int64_t>((m + TB - 1) / TB, 64)), ctx->K), TB, 0,
                          s>>>(ref->dd_B, m, ctx->dd_sign, ctx->dd_B);
  DPM_CUDA_TRY(ctx, cudaGetLastError());
  if (B_out)
    DPM_CUDA_TRY(ctx, cudaMemcpyAsync(B_out, ctx->dd_B, (size_t)ctx->K * m * 8, cudaMemcpyDeviceToDevice, s));
  ctx->have_projection = 0;
  ctx->dt_bep = ctx->dt;
  return DPM_OK;
}

dpm_status dpm_dd_lsq_rhs_shared(dpm_ctx* const* octs, int32_t noct, const double* wk, double* y, void* stream) {
  DPM_NVTX();
  if (!octs || noct < 1 || !wk || !y) return DPM_ERR_INVALID;
  dpm_ctx* o0 = octs[0];
  dpm_status st = dd_check(o0);
  if (st != DPM_OK) return st;
  const int K = o0->K;
  for (int s = 0; s < noct; ++s) {
    dpm_ctx* o = octs[s];
    if (!o || o->dd != 1 || o->device != o0->device || o->n != o0->n || o->lo != o0->lo || o->hi != o0->hi ||
        o->K != K || o->n_rows != o0->n_rows || o->radius != o0->radius) {
      o0->err = "dd_lsq_rhs_shared: the contexts are not octants of one canonical geometry on one device";
      return DPM_ERR_INVALID;
    }
    if (!o->have_projection || o->dt_bep != o->dt) { o0->err = "dd_lsq_rhs_shared: no factorisation"; return DPM_ERR_STATE; }
  }
  cudaStream_t s = as_stream(stream);
  const size_t field = (size_t)o0->n * o0->n * o0->n;
  const int64_t ng = o0->counts[DPM_SET_GAMMA], m = o0->n_rows;
  const int nv = 2 * noct;
  // signs of every octant relative to octant 0 (geometry only: computed once per pair)
  for (int q = 0; q < noct; ++q)
    if ((st = dd_signs(o0, octs[q], s)) != DPM_OK) return st;
  const int nsplit = (int)((m + TS_ICH - 1) / TS_ICH), nsk = (K + TS_ICH - 1) / TS_ICH;
  const int nua = (K + UA_CH - 1) / UA_CH;   // i-chunks of the D R^{-1} apply (2 right-hand sides each)
  const int npart = std::max(std::max(1, std::max(nsplit, nsk)), (2 * nua + nv - 1) / nv);
  const size_t need = ((size_t)nv * m + (size_t)npart * nv * K + (size_t)nv * K + 4 * (size_t)K +
                       (size_t)noct * K) * sizeof(double);
  if (o0->dd_shared_bytes < need) {
    if (o0->dd_shared) cudaFree(o0->dd_shared);
    o0->dd_shared = nullptr;
    o0->dd_shared_bytes = 0;
    DPM_CUDA_TRY(o0, cudaMalloc(&o0->dd_shared, need));
    o0->dd_shared_bytes = need;
  }
  double* G = o0->dd_shared;              // [nv][m]: BEP right-hand sides of all octants
  double* Pt = G + (size_t)nv * m;        // split-K partials
  double* Z = Pt + (size_t)npart * nv * K;   // [nv][K]: Q_0^T g_v
  double* Tz = Z + (size_t)nv * K;        // [2][K]: Σ_s S_s R^T z_s
  double* Vz = Tz + 2 * (size_t)K;        // [2][K]: R^{-T} Tz
  double* Sg = Vz + 2 * (size_t)K;        // [noct][K]: the signs, stacked
  if (noct > 8) { o0->err = "dd_lsq_rhs_shared: at most 8 octants"; return DPM_ERR_INVALID; }
  SignPtrs sp{};
  for (int q = 0; q < noct; ++q) sp.p[q] = octs[q]->dd_sign;
  DPM_COUNT_LAUNCH(1);
  dd_stack_signs_kernel<<<(noct * K + TB - 1) / TB, TB, 0, s>>>(sp, noct, K, Sg);
  DPM_COUNT_LAUNCH(1);
  dd_rows_trace_kernel<<<grid_for(m), TB, 0, s>>>(wk, field, o0->lists[DPM_SET_GAMMA], o0->dd_rows, m, nv, G);
  const size_t KK = (size_t)K * K;
  const double* R = o0->dd_R + 2 * KK;    // R = R2 R1
  const double* W2 = o0->dd_R + 4 * KK;   // R^{-1}
  const unsigned ct = (unsigned)((K + 31) / 32);
  const int rb = (int)std::min<long>(148L * 8, ((long)K * nv + TB - 1) / TB);
  DPM_COUNT_LAUNCH(7);
  dd_gemm_ts_kernel<0><<<dim3(ct, nsplit), 256, 0, s>>>(o0->dd_Q, m, K, G, m, nv, Pt);       // one pass over Q_0
  dd_reduce_kernel<<<rb, TB, 0, s>>>(Pt, nsplit, nv, K, nullptr, nv, Z);
  dd_gemm_ts_kernel<1><<<dim3(ct, nsk), 256, 0, s>>>(R, K, K, Z, K, nv, Pt);                  // R^T z_v
  dd_reduce_kernel<<<rb, TB, 0, s>>>(Pt, nsk, nv, K, Sg, 2, Tz);                              // Σ_s S_s (.)
  dd_gemm_ts_kernel<1><<<dim3(ct, nsk), 256, 0, s>>>(W2, K, K, Tz, K, 2, Pt);                 // R^{-T}
  dd_reduce_kernel<<<rb, TB, 0, s>>>(Pt, nsk, 2, K, nullptr, 2, Vz);
  DPM_COUNT_LAUNCH(1);
  dd_upper_apply_kernel<<<dim3(ct, (unsigned)nua), 256, 0, s>>>(W2, K, Vz, 2, Pt);                         // R^{-1} V
  dd_reduce_kernel<<<rb, TB, 0, s>>>(Pt, nua, 2, K, nullptr, 2, y, o0->dd_D);              // D (.)
  DPM_CUDA_TRY(o0, cudaGetLastError());
  return DPM_OK;
}

dpm_status dpm_dd_green_rhs(dpm_ctx* ctx, const double* C, int32_t clamp, const double* fq, double* wk, void* stream) {
  DPM_NVTX();
  dpm_status st = dd_check(ctx);
  if (st != DPM_OK) return st;
  if (!C || !fq || !wk) return DPM_ERR_INVALID;
  cudaStream_t s = as_stream(stream);
  const int64_t ng = ctx->counts[DPM_SET_GAMMA];
  if (!ctx->dd_ug) DPM_CUDA_TRY(ctx, cudaMalloc(&ctx->dd_ug, (size_t)2 * ng * sizeof(double) + 64));
  DPM_CUDA_TRY(ctx, dd_extend_fly(ctx, C, clamp, ctx->dd_ug, s));
  DPM_CUDA_TRY(ctx, launch_green_rhs(ctx, fq, ctx->dd_ug, wk, 2, s));                        // R20
  return DPM_OK;
}

dpm_status dpm_dd_green_rhs_shared(dpm_ctx* const* octs, int32_t noct, const double* C, int32_t clamp, const double* fq,
                                   double* wk, void* stream) {
  DPM_NVTX();
  if (!octs || noct < 1 || noct > 8 || !C || !fq || !wk) return DPM_ERR_INVALID;
  dpm_ctx* o0 = octs[0];
  dpm_status st = dd_check(o0);
  if (st != DPM_OK) return st;
  ExtOut eo{};
  eo.n = noct;
  const int64_t ng = o0->counts[DPM_SET_GAMMA];
  for (int q = 0; q < noct; ++q) {
    dpm_ctx* o = octs[q];
    if (!o || o->dd != 1 || o->device != o0->device || o->n != o0->n || o->lo != o0->lo || o->hi != o0->hi ||
        o->K != o0->K || o->radius != o0->radius || o->Lc != o0->Lc || o->Li != o0->Li ||
        o->counts[DPM_SET_GAMMA] != ng) {
      o0->err = "dd_green_rhs_shared: the contexts are not octants of one canonical geometry on one device";
      return DPM_ERR_INVALID;
    }
    if (!o->dd_ug) DPM_CUDA_TRY(o0, cudaMalloc(&o->dd_ug, (size_t)2 * ng * sizeof(double) + 64));
    eo.ug[q] = o->dd_ug;
    eo.oct[q] = 4 * (o->sigma[0] < 0) + 2 * (o->sigma[1] < 0) + (o->sigma[2] < 0);
  }
  cudaStream_t s = as_stream(stream);
  const int L1 = o0->Lc + 1;
  const size_t smem = (2 * (size_t)o0->K + 2 * L1 * L1 + 2 * L1) * sizeof(double);
  DPM_CUDA_TRY(o0, cudaFuncSetAttribute(dd_extend_shared_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  DPM_COUNT_LAUNCH(1);
  dd_extend_shared_kernel<<<(unsigned)std::min<int64_t>((ng + 127) / 128, 148 * 8), 128, smem, s>>>(
      o0->lists[DPM_SET_GAMMA], ng, o0->n, o0->lo, o0->h, o0->radius, o0->Lc, o0->Li, o0->nphi, o0->K, o0->dd_assign,
      C, clamp, eo);
  DPM_CUDA_TRY(o0, cudaGetLastError());
  const size_t field = (size_t)o0->n * o0->n * o0->n;
  for (int q = 0; q < noct; ++q) {
    if (wk == fq)   // in place: the band values scattered into fq (zero there, as dpm_dd_rhs leaves it)
      DPM_CUDA_TRY(o0, launch_green_band_inplace(octs[q], wk + 2 * q * field, octs[q]->dd_ug, 2, s));
    else
      DPM_CUDA_TRY(o0, launch_green_rhs(octs[q], fq + 2 * q * field, octs[q]->dd_ug, wk + 2 * q * field, 2, s));   // R20
  }
  return DPM_OK;
}

dpm_status dpm_dd_restrict(dpm_ctx* ctx, const double* wk, double* rho, double* c, void* stream) {
  DPM_NVTX();
  dpm_status st = dd_check(ctx);
  if (st != DPM_OK) return st;
  if (!wk || !rho || !c) return DPM_ERR_INVALID;
  cudaStream_t s = as_stream(stream);
  DPM_CUDA_TRY(ctx, launch_restrict_stats(ctx, wk, rho, c, ctx->red + 32, s));
  DPM_CUDA_TRY(ctx, cudaMemcpyAsync(ctx->red_host + 32, ctx->red + 32, 9 * sizeof(double), cudaMemcpyDeviceToHost, s));
  return DPM_OK;   // dpm_dd_stats() reads the statistics
}

dpm_status dpm_dd_local_begin(dpm_ctx* ctx, const double* rho, const double* c, double chi, double* y, void* stream) {
  DPM_NVTX();
  dpm_status st = dd_check(ctx);
  if (st != DPM_OK) return st;
  if (!rho || !c || !y) return DPM_ERR_INVALID;
  if (!ctx->have_projection || ctx->dt_bep != ctx->dt) { ctx->err = "octant DD: no factorisation at this dt"; return DPM_ERR_STATE; }
  cudaStream_t s = as_stream(stream);
  const size_t field = (size_t)ctx->n * ctx->n * ctx->n;
  const size_t need = 4 * field * 8;
  if (!ctx->scratch || ctx->scratch_bytes < need) {
    if (ctx->scratch) cudaFree(ctx->scratch);
    ctx->scratch_bytes = need;
    DPM_CUDA_TRY(ctx, cudaMalloc(&ctx->scratch, need));
  }
  double* fq = ctx->scratch;
  double* wk = fq + 2 * field;
  DPM_CUDA_TRY(ctx, launch_flux_rhs(ctx, rho, c, ctx->dt, chi, fq, fq + field, s));          // Step 4a
  DPM_CUDA_TRY(ctx, dst_solve_batch(ctx->plan, fq, wk, 2, nullptr, 0, s));
  DPM_COUNT_LAUNCH(1);
  dd_rows_trace_kernel<<<grid_for(ctx->n_rows), TB, 0, s>>>(wk, field, ctx->lists[DPM_SET_GAMMA], ctx->dd_rows,
                                                                ctx->n_rows, 2, ctx->dd_g);
  DPM_CUDA_TRY(ctx, cudaGetLastError());
  DPM_CUDA_TRY(ctx, lsq_gemv(ctx->dd_M, ctx->n_rows, ctx->K, ctx->dd_g, 2, y, s));           // y_s = M_s g_s
  return DPM_OK;
}

dpm_status dpm_dd_local_finish(dpm_ctx* ctx, const double* C, int32_t clamp, double* rho, double* c, double* stats,
                               void* stream) {
  DPM_NVTX();
  dpm_status st = dd_check(ctx);
  if (st != DPM_OK) return st;
  if (!C || !rho || !c || !ctx->scratch) return DPM_ERR_INVALID;
  cudaStream_t s = as_stream(stream);
  const size_t field = (size_t)ctx->n * ctx->n * ctx->n;
  const int64_t ng = ctx->counts[DPM_SET_GAMMA];
  double* fq = ctx->scratch;
  double* wk = fq + 2 * field;
  if (!ctx->dd_ug) DPM_CUDA_TRY(ctx, cudaMalloc(&ctx->dd_ug, (size_t)2 * ng * sizeof(double) + 64));
  double* ug = ctx->dd_ug;
  DPM_CUDA_TRY(ctx, dd_extend_fly(ctx, C, clamp, ug, s));                                   // u_γ = A C (R17)
  DPM_CUDA_TRY(ctx, launch_green_rhs(ctx, fq, ug, wk, 2, s));                                // R20
  DPM_CUDA_TRY(ctx, dst_solve_batch(ctx->plan, wk, wk, 2, nullptr, 0, s));
  DPM_CUDA_TRY(ctx, launch_restrict_stats(ctx, wk, rho, c, ctx->red + 32, s));
  DPM_CUDA_TRY(ctx, cudaMemcpyAsync(ctx->red_host + 32, ctx->red + 32, 9 * sizeof(double), cudaMemcpyDeviceToHost, s));
  if (!stats) return DPM_OK;   // asynchronous form: dpm_dd_stats() later
  return dpm_dd_stats(ctx, stats, stream);
}

dpm_status dpm_dd_stats(dpm_ctx* ctx, double* stats, void* stream) {
  DPM_NVTX();
  dpm_status st = dd_check(ctx);
  if (st != DPM_OK) return st;
  if (!stats) return DPM_ERR_INVALID;
  DPM_CUDA_TRY(ctx, cudaStreamSynchronize(as_stream(stream)));
  const double* R = ctx->red_host + 32;   // [mass lo, rho_max, rho_min, c_min, nonfinite, rho_max M+, -, -, mass hi] (R18)
  stats[0] = mass_fixed_decode(R) * ctx->h * ctx->h * ctx->h;
  stats[1] = decode_key(R[1]);
  stats[2] = -decode_key(R[2]);
  stats[3] = -decode_key(R[3]);
  stats[4] = R[4];
  stats[5] = decode_key(R[5]);
  return DPM_OK;
}

}  // extern "C"
