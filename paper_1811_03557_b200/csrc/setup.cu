// S1 — setup on the device: point sets of Definition 1, gamma geometry for the
// extension operator (R10), real spherical harmonics (R8) and the
// extension matrix E = [Y | d Y] or [Y | d^2/2 Y] (R9).
#include <cub/cub.cuh>

#include "dpm_internal.h"
#include "sh_device.cuh"

namespace {

__device__ __forceinline__ bool inside_domain(const dpm_domain& D, double x, double y, double z) {
  if (D.kind == DPM_OCTANT_CANON)   // cfg5 subdomain in its canonical frame (R24): open octant ∩ ball
    return x > 0.0 && y > 0.0 && z > 0.0 && x * x + y * y + z * z < D.semi[0] * D.semi[0];
  const double a = (x - D.center[0]) / D.semi[0];
  const double b = (y - D.center[1]) / D.semi[1];
  const double c = (z - D.center[2]) / D.semi[2];
  return a * a + b * b + c * c < 1.0;   // open interior; ties -> M- (R6)
}

__global__ void classify_kernel(uint8_t* flags, int n, double lo, double h, dpm_domain D) {
  const long nn = (long)n * n * n;
  for (long p = blockIdx.x * (long)blockDim.x + threadIdx.x; p < nn; p += (long)gridDim.x * blockDim.x) {
    const int i = (int)(p / ((long)n * n)), j = (int)((p / n) % n), k = (int)(p % n);
    const double x = lo + (i + 1) * h, y = lo + (j + 1) * h, z = lo + (k + 1) * h;
    flags[p] = inside_domain(D, x, y, z) ? F_MPLUS : 0;
  }
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
  DPM_COUNT_LAUNCH(1);
  classify_kernel<<<G, T, 0, s>>>(ctx->flags, n, ctx->lo, ctx->h, ctx->domain);
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
