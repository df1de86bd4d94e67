// S1 — setup on the device: point sets of Definition 1, gamma geometry for the
// extension operator (R10), real spherical harmonics (R8) and the
// extension matrix E = [Y | d Y] or [Y | d^2/2 Y] (R9).
#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>

#include "dpm_internal.h"
#include "sh_device.cuh"

namespace {

// fp64 membership value and a near-tie flag.  The decision is exact (R6) by construction: the fp64
// test decides every node whose value is farther than 1e-11 (relative) from the boundary, and the
// host re-decides the flagged rest in exact integer arithmetic (exact_inside below).  The fp64 error
// of Σ((x - c)/s)^2 is a few ulp, far below the flag band.
constexpr double TIE_BAND = 1e-11;
constexpr uint8_t F_TIE = 128;   // transient flag bit: resolved on the host before dilation

__device__ __forceinline__ uint8_t classify_node(const dpm_domain& D, double x, double y, double z, double scale) {
  if (D.kind == DPM_SHELL_CANON) {    // NEXT-3 Ω2: open shell semi[1] < |x| < semi[0]
    const double ro2 = D.semi[0] * D.semi[0], ri2 = D.semi[1] * D.semi[1];
    const double v = x * x + y * y + z * z;
    if (fabs(v - ro2) <= TIE_BAND * ro2 || fabs(v - ri2) <= TIE_BAND * ri2) return F_TIE;
    return (v > ri2 && v < ro2) ? F_MPLUS : 0;
  }
  if (D.kind == DPM_OCTANT_CANON) {   // cfg5 subdomain in its canonical frame (R24): open octant ∩ ball
    const double r2 = D.semi[0] * D.semi[0];
    const double v = x * x + y * y + z * z;
    const double tb = TIE_BAND * scale;
    if (fabs(x) <= tb || fabs(y) <= tb || fabs(z) <= tb || fabs(v - r2) <= TIE_BAND * r2) return F_TIE;
    return (x > 0.0 && y > 0.0 && z > 0.0 && v < r2) ? F_MPLUS : 0;
  }
  const double a = (x - D.center[0]) / D.semi[0];
  const double b = (y - D.center[1]) / D.semi[1];
  const double c = (z - D.center[2]) / D.semi[2];
  const double v = a * a + b * b + c * c;
  if (fabs(v - 1.0) <= TIE_BAND) return F_TIE;
  return v < 1.0 ? F_MPLUS : 0;   // open interior; ties -> M- (R6)
}

__global__ void classify_kernel(uint8_t* flags, int n, double lo, double h, double scale, dpm_domain D,
                                unsigned long long* nties) {
  const long nn = (long)n * n * n;
  for (long p = blockIdx.x * (long)blockDim.x + threadIdx.x; p < nn; p += (long)gridDim.x * blockDim.x) {
    const int i = (int)(p / ((long)n * n)), j = (int)((p / n) % n), k = (int)(p % n);
    const double x = lo + (i + 1) * h, y = lo + (j + 1) * h, z = lo + (k + 1) * h;
    const uint8_t f = classify_node(D, x, y, z, scale);
    flags[p] = f;
    if (f == F_TIE) atomicAdd(nties, 1ull);
  }
}

__global__ void tie_list_kernel(const uint8_t* flags, long nn, int64_t* list, unsigned long long* cnt) {
  for (long p = blockIdx.x * (long)blockDim.x + threadIdx.x; p < nn; p += (long)gridDim.x * blockDim.x)
    if (flags[p] == F_TIE) list[atomicAdd(cnt, 1ull)] = p;
}

__global__ void tie_set_kernel(uint8_t* flags, const int64_t* list, const uint8_t* val, long m) {
  const long i = blockIdx.x * (long)blockDim.x + threadIdx.x;
  if (i < m) flags[list[i]] = val[i];
}

// N± (within M0), gamma; counts ghost nodes of N+ (a face ghost has exactly one interior
// neighbour, so it lies in N+ iff that neighbour is in M+, and never in N- ∩ N+ — R5).
__global__ void dilate_kernel(uint8_t* flags, int n, unsigned long long* ghost_count) {
  const long nn = (long)n * n * n;
  for (long p = blockIdx.x * (long)blockDim.x + threadIdx.x; p < nn; p += (long)gridDim.x * blockDim.x) {
    const int i = (int)(p / ((long)n * n)), j = (int)((p / n) % n), k = (int)(p % n);
    const bool mp = flags[p] & F_MPLUS;
    bool anyp = mp, anym = !mp;
    int nghost = 0;
    const int di[6] = {1, -1, 0, 0, 0, 0}, dj[6] = {0, 0, 1, -1, 0, 0}, dk[6] = {0, 0, 0, 0, 1, -1};
    for (int s = 0; s < 6; ++s) {
      const int a = i + di[s], b = j + dj[s], c = k + dk[s];
      if (a < 0 || a >= n || b < 0 || b >= n || c < 0 || c >= n) { ++nghost; continue; }
      const bool q = flags[((long)a * n + b) * n + c] & F_MPLUS;
      anyp |= q;
      anym |= !q;
    }
    uint8_t f = mp ? F_MPLUS : 0;
    if (anyp) f |= F_NPLUS;
    if (anym) f |= F_NMINUS;
    if (anyp && anym) f |= F_GAMMA;
    flags[p] = f | (flags[p] & F_MPLUS);
    if (mp && nghost) atomicAdd(ghost_count, (unsigned long long)nghost);
  }
}

__global__ void band_kernel(uint8_t* flags, int n) {
  const long nn = (long)n * n * n;
  for (long p = blockIdx.x * (long)blockDim.x + threadIdx.x; p < nn; p += (long)gridDim.x * blockDim.x) {
    if (flags[p] & F_MPLUS) continue;
    const int i = (int)(p / ((long)n * n)), j = (int)((p / n) % n), k = (int)(p % n);
    bool g = flags[p] & F_GAMMA;
    const int di[6] = {1, -1, 0, 0, 0, 0}, dj[6] = {0, 0, 1, -1, 0, 0}, dk[6] = {0, 0, 0, 0, 1, -1};
    for (int s = 0; s < 6 && !g; ++s) {
      const int a = i + di[s], b = j + dj[s], c = k + dk[s];
      if (a < 0 || a >= n || b < 0 || b >= n || c < 0 || c >= n) continue;
      g = flags[((long)a * n + b) * n + c] & F_GAMMA;
    }
    if (g) flags[p] |= F_BAND;
  }
}

struct SetPred {
  const uint8_t* flags;
  int which;
  __device__ bool operator()(const int64_t& p) const {
    const uint8_t f = flags[p];
    switch (which) {
      case DPM_SET_MPLUS: return f & F_MPLUS;
      case DPM_SET_GAMMA: return f & F_GAMMA;
      case DPM_SET_GAMMA_IN: return (f & F_GAMMA) && (f & F_MPLUS);
      case DPM_SET_GAMMA_EX: return (f & F_GAMMA) && !(f & F_MPLUS);
      case DPM_SET_BAND: return f & F_BAND;
      default: return f & F_NPLUS;
    }
  }
};

__global__ void gmap_kernel(int32_t* gmap, const int64_t* gamma, int64_t ng) {
  const long i = blockIdx.x * (long)blockDim.x + threadIdx.x;
  if (i < ng) gmap[gamma[i]] = (int32_t)i;
}

__global__ void ginpos_kernel(int32_t* pos, const int32_t* gmap, const int64_t* gin, int64_t ngin) {
  const long i = blockIdx.x * (long)blockDim.x + threadIdx.x;
  if (i < ngin) pos[i] = gmap[gin[i]];
}

// Closest point of the ellipsoid: x_i = s_i^2 p_i / (s_i^2 + t) with
// F(t) = Σ (s_i p_i/(s_i^2 + t))^2 - 1 = 0, safeguarded Newton on a sign bracket.
__device__ void ellipsoid_foot(const double p[3], const double s[3], double x[3], double* d) {
  const double smin2 = fmin(s[0] * s[0], fmin(s[1] * s[1], s[2] * s[2]));
  auto F = [&](double t, double* dF) {
    double f = -1.0, df = 0.0;
    for (int a = 0; a < 3; ++a) {
      const double den = s[a] * s[a] + t;
      const double r = s[a] * p[a] / den;
      f += r * r;
      df += -2.0 * r * r / den;
    }
    *dF = df;
    return f;
  };
  double dF;
  const double f0 = F(0.0, &dF);
  double tl, tr;
  if (f0 > 0) {   // outside: root in (0, |p| s_max]
    tl = 0.0;
    const double pm = sqrt(p[0] * p[0] + p[1] * p[1] + p[2] * p[2]);
    tr = pm * fmax(s[0], fmax(s[1], s[2])) + 1e-300;
  } else {        // inside: root in (-smin2, 0]
    tl = -smin2;
    tr = 0.0;
  }
  double t = (f0 > 0) ? 0.0 : 0.0;
  for (int it = 0; it < 200; ++it) {
    const double f = F(t, &dF);
    if (f == 0.0) break;
    if (f > 0) tl = t; else tr = t;
    double tn = t - f / dF;
    if (!(tn > tl && tn < tr)) tn = 0.5 * (tl + tr);
    if (tn == t) break;
    t = tn;
    if (tr - tl <= 4e-16 * fmax(1.0, fabs(t))) break;
  }
  double dd = 0.0;
  for (int a = 0; a < 3; ++a) {
    x[a] = s[a] * s[a] * p[a] / (s[a] * s[a] + t);
    dd += (p[a] - x[a]) * (p[a] - x[a]);
  }
  *d = (t > 0 ? 1.0 : (t < 0 ? -1.0 : 0.0)) * sqrt(dd);
}

// Per gamma point: geometry, then all (L+1)^2 real SH (sh_device.cuh), written into E.
__global__ void geometry_sh_kernel(const int64_t* gamma, int64_t ng, int n, double lo, double h, dpm_domain D,
                                   int lmax, int basis, double* foot, double* dist, double* E) {
  const long g = blockIdx.x * (long)blockDim.x + threadIdx.x;
  if (g >= ng) return;
  const int64_t p = gamma[g];
  const int i = (int)(p / ((long)n * n)), j = (int)((p / n) % n), k = (int)(p % n);
  const double P[3] = {lo + (i + 1) * h - D.center[0], lo + (j + 1) * h - D.center[1], lo + (k + 1) * h - D.center[2]};
  double X[3], d, u[3];
  if (D.kind == DPM_SPHERE) {
    const double r = sqrt(P[0] * P[0] + P[1] * P[1] + P[2] * P[2]);
    for (int a = 0; a < 3; ++a) { u[a] = P[a] / r; X[a] = D.semi[0] * u[a]; }
    d = r - D.semi[0];
  } else {
    ellipsoid_foot(P, D.semi, X, &d);
    double nu = 0.0;
    for (int a = 0; a < 3; ++a) { u[a] = X[a] / D.semi[a]; nu += u[a] * u[a]; }
    nu = sqrt(nu);
    for (int a = 0; a < 3; ++a) u[a] /= nu;
  }
  for (int a = 0; a < 3; ++a) foot[g * 3 + a] = X[a] + D.center[a];
  dist[g] = d;
  const double w = (basis == DPM_BASIS_CAUCHY || basis == DPM_BASIS_CAUCHY_ZONAL) ? d : 0.5 * d * d;
  const bool two = basis_ncomp(basis) == 2;
  if (basis_zonal(basis)) {
    // phi_l = P_l^0(cos θ), cos θ = u_z; (l+1) P_{l+1} = (2l+1) x P_l - l P_{l-1}
    const double x = u[2];
    double pm = 1.0, pl = x;
    for (int l = 0; l <= lmax; ++l) {
      const double v = l == 0 ? 1.0 : pl;
      E[(size_t)l * ng + g] = v;
      if (two) E[(size_t)(lmax + 1 + l) * ng + g] = w * v;
      if (l >= 1) {
        const double nx = ((2 * l + 1) * x * pl - l * pm) / (l + 1);
        pm = pl;
        pl = nx;
      }
    }
    return;
  }
  const int nsh = (lmax + 1) * (lmax + 1);
  real_sh_unit(u[0], u[1], u[2], lmax, [&](int nu, double v) {
    E[(size_t)nu * ng + g] = v;
    if (two) E[(size_t)(nsh + nu) * ng + g] = w * v;
  });
}

// ---- exact classification of near-tie nodes (R6) -------------------------------------------------
// The configuration constants are read as decimals, the shortest decimal that round-trips the double
// (the oracle's Fraction(repr(x)), oracle/grid.py).  With every constant scaled to one power of ten,
// lo = L 10^e, hi = H 10^e, c_a = C_a 10^e, s_a = S_a 10^e, node i sits at x_i - c_a =
// X_a(i) 10^e / (n+1) with the integer X_a(i) = L (n+1) + (i+1)(H - L) - C_a (n+1), and
//   Σ_a ((x_a - c_a)/s_a)^2 < 1   <=>   Σ_a X_a^2 Π_{b≠a} S_b^2 < (n+1)^2 Π_b S_b^2,
//   octant (c = 0, radius R 10^e): X_a > 0 for all a and Σ_a X_a^2 < (n+1)^2 R^2.
// Small sign-magnitude big integers (base 2^32) evaluate it for the few flagged nodes.
struct BigInt {
  bool neg = false;
  std::vector<uint32_t> m;   // little-endian magnitude, no leading zero limbs
  static BigInt from_u64(unsigned long long v, bool neg = false) {
    BigInt r;
    while (v) { r.m.push_back((uint32_t)v); v >>= 32; }
    r.neg = neg && !r.m.empty();
    return r;
  }
  bool zero() const { return m.empty(); }
};

int cmp_mag(const std::vector<uint32_t>& a, const std::vector<uint32_t>& b) {
  if (a.size() != b.size()) return a.size() < b.size() ? -1 : 1;
  for (size_t i = a.size(); i-- > 0;)
    if (a[i] != b[i]) return a[i] < b[i] ? -1 : 1;
  return 0;
}

std::vector<uint32_t> add_mag(const std::vector<uint32_t>& a, const std::vector<uint32_t>& b) {
  std::vector<uint32_t> r(std::max(a.size(), b.size()) + 1, 0);
  unsigned long long carry = 0;
  for (size_t i = 0; i + 1 < r.size(); ++i) {
    const unsigned long long s = carry + (i < a.size() ? a[i] : 0) + (i < b.size() ? b[i] : 0);
    r[i] = (uint32_t)s;
    carry = s >> 32;
  }
  r.back() = (uint32_t)carry;
  while (!r.empty() && r.back() == 0) r.pop_back();
  return r;
}

std::vector<uint32_t> sub_mag(const std::vector<uint32_t>& a, const std::vector<uint32_t>& b) {   // |a| >= |b|
  std::vector<uint32_t> r(a.size(), 0);
  long long borrow = 0;
  for (size_t i = 0; i < a.size(); ++i) {
    long long d = (long long)a[i] - (i < b.size() ? b[i] : 0) - borrow;
    borrow = d < 0;
    if (d < 0) d += (1ll << 32);
    r[i] = (uint32_t)d;
  }
  while (!r.empty() && r.back() == 0) r.pop_back();
  return r;
}

BigInt add(const BigInt& a, const BigInt& b) {
  BigInt r;
  if (a.neg == b.neg) {
    r.m = add_mag(a.m, b.m);
    r.neg = a.neg;
  } else if (cmp_mag(a.m, b.m) >= 0) {
    r.m = sub_mag(a.m, b.m);
    r.neg = a.neg;
  } else {
    r.m = sub_mag(b.m, a.m);
    r.neg = b.neg;
  }
  if (r.m.empty()) r.neg = false;
  return r;
}

BigInt neg(BigInt a) {
  if (!a.zero()) a.neg = !a.neg;
  return a;
}

BigInt mul(const BigInt& a, const BigInt& b) {
  BigInt r;
  if (a.zero() || b.zero()) return r;
  std::vector<unsigned long long> acc(a.m.size() + b.m.size() + 1, 0);
  r.m.assign(a.m.size() + b.m.size(), 0);
  for (size_t i = 0; i < a.m.size(); ++i) {
    unsigned long long carry = 0;
    for (size_t j = 0; j < b.m.size(); ++j) {
      const unsigned long long t = (unsigned long long)a.m[i] * b.m[j] + r.m[i + j] + carry;
      r.m[i + j] = (uint32_t)t;
      carry = t >> 32;
    }
    size_t k = i + b.m.size();
    while (carry) {
      const unsigned long long t = (unsigned long long)r.m[k] + carry;
      r.m[k++] = (uint32_t)t;
      carry = t >> 32;
    }
  }
  while (!r.m.empty() && r.m.back() == 0) r.m.pop_back();
  r.neg = a.neg != b.neg && !r.m.empty();
  return r;
}

int cmp(const BigInt& a, const BigInt& b) {   // sign-aware
  if (a.neg != b.neg) return a.neg ? -1 : 1;
  const int c = cmp_mag(a.m, b.m);
  return a.neg ? -c : c;
}

// x = D 10^e with D an integer: the shortest decimal that round-trips the double (Python's repr).
struct Decimal {
  BigInt D;
  int e = 0;
};

Decimal to_decimal(double x) {
  char buf[64];
  for (int p = 1; p <= 17; ++p) {
    std::snprintf(buf, sizeof buf, "%.*e", p - 1, x);
    if (std::strtod(buf, nullptr) == x) break;
  }
  Decimal d;
  const char* c = buf;
  bool ng = false;
  if (*c == '-') { ng = true; ++c; }
  int frac_digits = 0;
  bool after_point = false;
  BigInt ten = BigInt::from_u64(10);
  for (; *c && *c != 'e'; ++c) {
    if (*c == '.') { after_point = true; continue; }
    d.D = add(mul(d.D, ten), BigInt::from_u64((unsigned long long)(*c - '0')));
    if (after_point) ++frac_digits;
  }
  const int ex = (*c == 'e') ? std::atoi(c + 1) : 0;
  d.e = ex - frac_digits;
  if (ng) d.D = neg(d.D);
  return d;
}

BigInt scaled(const Decimal& d, int e) {   // D 10^(d.e - e), d.e >= e
  BigInt r = d.D;
  const BigInt ten = BigInt::from_u64(10);
  for (int k = d.e; k > e; --k) r = mul(r, ten);
  return r;
}

// Exact M+ membership of node (i, j, k) (R6); octant: the canonical-frame subdomain (R24).
struct ExactClassifier {
  int n = 0;
  bool octant = false, shell = false;
  BigInt L, HL, C[3], W[3], rhs, rhs_in;   // X_a(i) = L (n+1) + (i+1) HL - C_a (n+1)
  ExactClassifier(int n_, double lo, double hi, const dpm_domain& Dm) : n(n_) {
    octant = Dm.kind == DPM_OCTANT_CANON;
    shell = Dm.kind == DPM_SHELL_CANON;   // semi[0] = outer, semi[1] = inner radius, centre 0
    std::vector<Decimal> ds = {to_decimal(lo), to_decimal(hi)};
    for (int a = 0; a < 3; ++a) ds.push_back(to_decimal(octant || shell ? 0.0 : Dm.center[a]));
    for (int a = 0; a < 3; ++a) ds.push_back(to_decimal(Dm.semi[a]));
    int e = 0;
    for (auto& d : ds) e = std::min(e, d.e);
    std::vector<BigInt> v;
    for (auto& d : ds) v.push_back(scaled(d, e));
    const BigInt np1 = BigInt::from_u64((unsigned long long)(n + 1));
    L = mul(v[0], np1);
    HL = add(v[1], neg(v[0]));
    for (int a = 0; a < 3; ++a) C[a] = mul(v[2 + a], np1);
    const BigInt np1sq = mul(np1, np1);
    if (octant || shell) {
      for (int a = 0; a < 3; ++a) W[a] = BigInt::from_u64(1);
      rhs = mul(np1sq, mul(v[5], v[5]));
      if (shell) rhs_in = mul(np1sq, mul(v[6], v[6]));
    } else {
      BigInt S2[3];
      for (int a = 0; a < 3; ++a) S2[a] = mul(v[5 + a], v[5 + a]);
      for (int a = 0; a < 3; ++a) W[a] = mul(S2[(a + 1) % 3], S2[(a + 2) % 3]);
      rhs = mul(np1sq, mul(S2[0], mul(S2[1], S2[2])));
    }
  }
  bool inside(int64_t p) const {
    const int idx[3] = {(int)(p / ((int64_t)n * n)), (int)((p / n) % n), (int)(p % n)};
    BigInt sum;
    for (int a = 0; a < 3; ++a) {
      const BigInt X = add(add(L, mul(BigInt::from_u64((unsigned long long)(idx[a] + 1)), HL)), neg(C[a]));
      if (octant && (X.neg || X.zero())) return false;   // on or behind a coordinate plane -> M-
      sum = add(sum, mul(mul(X, X), W[a]));
    }
    if (shell && cmp(sum, rhs_in) <= 0) return false;   // on or inside the inner sphere -> M-
    return cmp(sum, rhs) < 0;   // ties -> M- (R6)
  }
};

}  // namespace

dpm_status setup_point_sets(dpm_ctx* ctx) {
  const int n = ctx->n;
  const long nn = (long)n * n * n;
  cudaStream_t s = ctx->setup_stream;
  DPM_CUDA_TRY(ctx, cudaMalloc(&ctx->flags, nn));
  DPM_CUDA_TRY(ctx, cudaMalloc(&ctx->gmap, nn * sizeof(int32_t)));
  unsigned long long* dghost;
  DPM_CUDA_TRY(ctx, cudaMalloc(&dghost, 8));
  DPM_CUDA_TRY(ctx, cudaMemsetAsync(dghost, 0, 8, s));
  const int T = 256;
  const int G = (int)std::min<long>((nn + T - 1) / T, 148L * 32);
  unsigned long long* dties;
  DPM_CUDA_TRY(ctx, cudaMalloc(&dties, 16));
  DPM_CUDA_TRY(ctx, cudaMemsetAsync(dties, 0, 16, s));
  DPM_COUNT_LAUNCH(1);
  classify_kernel<<<G, T, 0, s>>>(ctx->flags, n, ctx->lo, ctx->h, std::max(std::fabs(ctx->lo), std::fabs(ctx->hi)),
                                   ctx->domain, dties);
  DPM_CUDA_TRY(ctx, cudaGetLastError());
  unsigned long long hties = 0;
  DPM_CUDA_TRY(ctx, cudaMemcpyAsync(&hties, dties, 8, cudaMemcpyDeviceToHost, s));
  DPM_CUDA_TRY(ctx, cudaStreamSynchronize(s));
  ctx->exact_ties = (int64_t)hties;
  if (hties) {   // R6: re-decide the near-tie nodes exactly on the host
    int64_t* dlist;
    uint8_t* dval;
    DPM_CUDA_TRY(ctx, cudaMalloc(&dlist, hties * sizeof(int64_t)));
    DPM_CUDA_TRY(ctx, cudaMalloc(&dval, hties));
    DPM_COUNT_LAUNCH(1);
    tie_list_kernel<<<G, T, 0, s>>>(ctx->flags, nn, dlist, dties + 1);
    std::vector<int64_t> list(hties);
    DPM_CUDA_TRY(ctx, cudaMemcpyAsync(list.data(), dlist, hties * sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    DPM_CUDA_TRY(ctx, cudaStreamSynchronize(s));
    const ExactClassifier ex(n, ctx->lo, ctx->hi, ctx->domain);
    std::vector<uint8_t> val(hties);
    int64_t in = 0;
    for (size_t i = 0; i < list.size(); ++i) {
      val[i] = ex.inside(list[i]) ? F_MPLUS : 0;
      in += val[i] != 0;
    }
    ctx->exact_ties_inside = in;
    DPM_CUDA_TRY(ctx, cudaMemcpyAsync(dval, val.data(), hties, cudaMemcpyHostToDevice, s));
    DPM_COUNT_LAUNCH(1);
    tie_set_kernel<<<(int)((hties + 255) / 256), 256, 0, s>>>(ctx->flags, dlist, dval, (long)hties);
    DPM_CUDA_TRY(ctx, cudaGetLastError());
    DPM_CUDA_TRY(ctx, cudaStreamSynchronize(s));
    cudaFree(dlist);
    cudaFree(dval);
  }
  cudaFree(dties);
  DPM_COUNT_LAUNCH(1);
  dilate_kernel<<<G, T, 0, s>>>(ctx->flags, n, dghost);
  DPM_COUNT_LAUNCH(1);
  band_kernel<<<G, T, 0, s>>>(ctx->flags, n);
  DPM_CUDA_TRY(ctx, cudaGetLastError());
  unsigned long long hg = 0;
  DPM_CUDA_TRY(ctx, cudaMemcpyAsync(&hg, dghost, 8, cudaMemcpyDeviceToHost, s));
  // compaction of every list (ascending flat index, R7)
  int64_t* dcount;
  DPM_CUDA_TRY(ctx, cudaMalloc(&dcount, 8));
  cub::CountingInputIterator<int64_t> it(0);
  size_t tmp_bytes = 0;
  cub::DeviceSelect::If(nullptr, tmp_bytes, it, (int64_t*)nullptr, dcount, nn, SetPred{ctx->flags, 0}, s);
  void* tmp;
  DPM_CUDA_TRY(ctx, cudaMalloc(&tmp, tmp_bytes));
  int64_t* buf;
  DPM_CUDA_TRY(ctx, cudaMalloc(&buf, nn * sizeof(int64_t)));
  for (int w = 0; w < 6; ++w) {
    size_t tb = tmp_bytes;
    DPM_CUDA_TRY(ctx, cub::DeviceSelect::If(tmp, tb, it, buf, dcount, nn, SetPred{ctx->flags, w}, s));
    int64_t cnt = 0;
    DPM_CUDA_TRY(ctx, cudaMemcpyAsync(&cnt, dcount, 8, cudaMemcpyDeviceToHost, s));
    DPM_CUDA_TRY(ctx, cudaStreamSynchronize(s));
    ctx->counts[w] = cnt;
    DPM_CUDA_TRY(ctx, cudaMalloc(&ctx->lists[w], std::max<int64_t>(cnt, 1) * sizeof(int64_t)));
    DPM_CUDA_TRY(ctx, cudaMemcpyAsync(ctx->lists[w], buf, cnt * sizeof(int64_t), cudaMemcpyDeviceToDevice, s));
  }
  DPM_CUDA_TRY(ctx, cudaStreamSynchronize(s));
  cudaFree(buf);
  cudaFree(tmp);
  cudaFree(dcount);
  cudaFree(dghost);
  ctx->ghosts_in_nplus = (int64_t)hg;
  const int64_t ng = ctx->counts[DPM_SET_GAMMA], ngin = ctx->counts[DPM_SET_GAMMA_IN];
  if (ctx->counts[DPM_SET_MPLUS] == 0 || ng == 0) {
    ctx->err = "domain contains no grid node (M+ or gamma empty)";
    return DPM_ERR_INVALID;
  }
  DPM_CUDA_TRY(ctx, cudaMemsetAsync(ctx->gmap, 0xff, nn * sizeof(int32_t), s));
  DPM_COUNT_LAUNCH(1);
  gmap_kernel<<<(ng + 255) / 256, 256, 0, s>>>(ctx->gmap, ctx->lists[DPM_SET_GAMMA], ng);
  DPM_CUDA_TRY(ctx, cudaMalloc(&ctx->gin_pos, std::max<int64_t>(ngin, 1) * sizeof(int32_t)));
  DPM_COUNT_LAUNCH(1);
  ginpos_kernel<<<(ngin + 255) / 256, 256, 0, s>>>(ctx->gin_pos, ctx->gmap, ctx->lists[DPM_SET_GAMMA_IN], ngin);
  DPM_CUDA_TRY(ctx, cudaGetLastError());
  DPM_CUDA_TRY(ctx, launch_slope_mask(ctx, s));
  DPM_CUDA_TRY(ctx, cudaStreamSynchronize(s));
  return DPM_OK;
}

dpm_status setup_geometry(dpm_ctx* ctx) {
  const int64_t ng = ctx->counts[DPM_SET_GAMMA];
  cudaStream_t s = ctx->setup_stream;
  DPM_CUDA_TRY(ctx, cudaMalloc(&ctx->foot, ng * 3 * sizeof(double)));
  DPM_CUDA_TRY(ctx, cudaMalloc(&ctx->dist, ng * sizeof(double)));
  DPM_CUDA_TRY(ctx, cudaMalloc(&ctx->E, (size_t)ng * ctx->K * sizeof(double)));
  DPM_COUNT_LAUNCH(1);
  geometry_sh_kernel<<<(ng + 127) / 128, 128, 0, s>>>(ctx->lists[DPM_SET_GAMMA], ng, ctx->n, ctx->lo, ctx->h,
                                                      ctx->domain, ctx->lmax, ctx->basis, ctx->foot, ctx->dist,
                                                      ctx->E);
  DPM_CUDA_TRY(ctx, cudaGetLastError());
  DPM_CUDA_TRY(ctx, cudaStreamSynchronize(s));
  return DPM_OK;
}
