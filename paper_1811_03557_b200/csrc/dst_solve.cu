// S3 — batched Dirichlet modified-Helmholtz AP solve, (I/dt - Δ_h) u = q  (R4).
//
// Fast Poisson solver as 3D DST-I -> eigenvalue divide -> inverse 3D DST-I:
//   u = (2/(n+1))^3 S_x S_y S_z D^{-1} S_z S_y S_x q,  S_jk = sin(pi j k/(n+1)),
//   D_abc = (1/dt + λ_a) + λ_b + λ_c,  λ_m = (4/h^2) sin^2(m pi/(2(n+1)))   (R26).
//
// B200 design:
//  * sm_100a has no fp64 tcgen05 kind; the fp64 pipes are DFMA and DMMA.8x8x4, both
//    measured at ~37 TFLOP/s (tools/microbench_fp64.cu).  DMMA needs 8x fewer issue slots
//    and register operands per MAC, so the 1D transforms are DMMA contractions.
//  * Each 1D DST-I of length n is FOLDED by the even/odd symmetry
//    S_{n+1-j,k} = (-1)^{k+1} S_{jk}: s_j = x_j + x_{n+1-j}, d_j = x_j - x_{n+1-j};
//    odd outputs k = 2m+1 use s (plus the middle sample when n is odd), even outputs
//    k = 2m+2 use d.  Two ceil(n/2) x ceil(n/2) contractions: n^2/2 MACs per line
//    instead of n^2.
//  * Three tile kernels, each a persistent CTA loop over (field, 32-column) tiles that
//    hold ALL n samples of the transform axis in shared memory:
//      pass X: transform along x (stride n^2), columns = flat (y,z)
//      pass Y: transform along y (stride n),   columns = flat (x,z)
//      pass Z: transform along z (contiguous), divide by D (fused epilogue), inverse z
//    A solve is X, Y, Z, Y, X (DST-I is an involution up to the folded scale).
//  * Every warp keeps its sine-matrix fragments in REGISTERS for the whole kernel (computed
//    once with exact argument reduction), so the MMA loop only loads B fragments from
//    shared memory; row strides are padded (≡ 4 mod 16 doubles) for conflict-free
//    fragment loads.
//  * The batch is processed in chunks whose working set stays in the 126 MB L2, with the
//    intermediate living in the output buffer (u may alias q): HBM sees ~one read of q
//    and one write of u per solve.
#include <algorithm>

#include "dpm_internal.h"

namespace {

constexpr int NW = 8;         // warps per CTA
constexpr int NT = NW * 32;   // threads per CTA
constexpr int TC = 32;        // columns per tile
constexpr int LDX = TC + 4;   // smem row stride (doubles) for passes X/Y (≡ 4 mod 16)

__host__ __device__ inline int ldz_of(int n) { return ((n + 15) / 16) * 16 + 4; }

__device__ __forceinline__ void dmma884(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

// Folded sine-matrix entry. matrix 0: odd outputs k = 2m+1 against s rows j (0-based, j < Po,
// j == Pe is the middle sample when n is odd, weight sin(pi(2m+1)/2) = (-1)^m).
// matrix 1: even outputs k = 2m+2 against d rows j < Pe.
__device__ double fold_entry(int n, int Po, int Pe, int matrix, int m, int j) {
  if (matrix == 0) {
    if (m >= Po || j >= Po) return 0.0;
    if (j == Pe) return (m & 1) ? -1.0 : 1.0;
    const long arg = ((long)(j + 1) * (2 * m + 1)) % (2 * (n + 1));
    return sinpi((double)arg / (double)(n + 1));
  }
  if (m >= Pe || j >= Pe) return 0.0;
  const long arg = ((long)(j + 1) * (2 * m + 2)) % (2 * (n + 1));
  return sinpi((double)arg / (double)(n + 1));
}

struct WarpRole {
  int matrix;   // 0 odd / 1 even
  int nmt;      // m-tiles owned (0..2)
  int mt[2];    // local m-tile indices
  int nct;      // column tiles handled
  int ct0, ctstep;
};

__device__ WarpRole warp_role(int warp, int MTh) {
  WarpRole r;
  r.matrix = warp >> 2;
  const int wl = warp & 3;
  if (MTh >= 4) {
    r.mt[0] = wl;
    r.mt[1] = wl + 4;
    r.nmt = (wl + 4 < MTh) ? 2 : 1;
    r.ct0 = 0;
    r.ctstep = 1;
    r.nct = TC / 8;
  } else {
    const int G = 4 / MTh;
    const int cg = wl / MTh;
    r.mt[0] = wl % MTh;
    r.mt[1] = 0;
    r.nmt = (cg < G) ? 1 : 0;
    r.ct0 = cg;
    r.ctstep = G;
    r.nct = (cg < G) ? (TC / 8 - cg + G - 1) / G : 0;
  }
  return r;
}

// One folded DST-I of every column of the smem tile, in place.
// Element (row r, col c) lives at sm[r*rs + c*cs].  If DIVIDE, the epilogue multiplies
// output (row k, column c) by scale / (((inv_dt + lam[a]) + lam[b]) + lam[k]) with
// (a, b) = divmod(col0 + c, n) (pass Z after X and Y: spectral indices).
template <int KSMAX, bool DIVIDE>
__device__ __forceinline__ void fold_transform(double* sm, int rs, int cs, int n, int Po, int Pe, int KS,
                                               const WarpRole& role, const double (&afr)[2][KSMAX],
                                               const double* lam, double inv_dt, double scale, int col0,
                                               bool rows_fast) {
  const int tid = threadIdx.x, lane = tid & 31;
  // fold: s_j -> row j, d_j -> row n-1-j (middle row untouched)
  const int nf = Pe * TC;
  for (int idx = tid; idx < nf; idx += NT) {
    int j, c;
    if (rows_fast) { j = idx % Pe; c = idx / Pe; } else { j = idx / TC; c = idx % TC; }
    double* pa = sm + j * rs + c * cs;
    double* pb = sm + (n - 1 - j) * rs + c * cs;
    const double a = *pa, b = *pb;
    *pa = a + b;
    *pb = a - b;
  }
  __syncthreads();

  double acc[2][TC / 8][2];
#pragma unroll
  for (int t = 0; t < 2; ++t)
#pragma unroll
    for (int ct = 0; ct < TC / 8; ++ct) acc[t][ct][0] = acc[t][ct][1] = 0.0;

  if (role.nmt > 0) {
#pragma unroll
    for (int ks = 0; ks < KSMAX; ++ks) {
      if (ks < KS) {
        const int j = ks * 4 + (lane & 3);
        const int r = (role.matrix == 0) ? (j < Po ? j : 0) : (j < Pe ? n - 1 - j : 0);
        const double* rowp = sm + r * rs;
        double b[TC / 8];
#pragma unroll
        for (int ct = 0; ct < TC / 8; ++ct) {
          b[ct] = 0.0;
          if (ct < role.nct) b[ct] = rowp[((role.ct0 + ct * role.ctstep) * 8 + (lane >> 2)) * cs];
        }
#pragma unroll
        for (int t = 0; t < 2; ++t)
#pragma unroll
          for (int ct = 0; ct < TC / 8; ++ct)
            if (t < role.nmt && ct < role.nct) dmma884(acc[t][ct], afr[t][ks], b[ct]);
      }
    }
  }
  __syncthreads();
  // epilogue: odd m -> row 2m, even m -> row 2m+1
  if (role.nmt > 0) {
    const int P = role.matrix == 0 ? Po : Pe;
#pragma unroll
    for (int t = 0; t < 2; ++t) {
      if (t >= role.nmt) continue;
      const int m = role.mt[t] * 8 + (lane >> 2);
      if (m >= P) continue;
      const int row = role.matrix == 0 ? 2 * m : 2 * m + 1;
#pragma unroll
      for (int ct = 0; ct < TC / 8; ++ct) {
        if (ct >= role.nct) continue;
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          const int c = (role.ct0 + ct * role.ctstep) * 8 + 2 * (lane & 3) + i;
          double v = acc[t][ct][i];
          if (DIVIDE) {
            const int cg = col0 + c;
            if (cg < n * n) {
              const int a = cg / n, bb = cg - a * n;
              v *= scale / (((inv_dt + lam[a]) + lam[bb]) + lam[row]);
            }
          }
          sm[row * rs + c * cs] = v;
        }
      }
    }
  }
  __syncthreads();
}

// PASS 0: along x (row stride n^2, col = flat yz); PASS 1: along y (row stride n, col = flat xz);
// PASS 2: along z (contiguous rows, col = flat xy line) with divide and inverse.
template <int PASS>
__device__ __forceinline__ size_t goff(int n, int r, int cg) {
  if (PASS == 0) return (size_t)r * n * n + cg;
  if (PASS == 1) { const int x = cg / n; return (size_t)x * n * n + (size_t)r * n + (cg - x * n); }
  return (size_t)cg * n + r;
}

template <int KSMAX, int PASS>
__global__ void __launch_bounds__(NT, 2)
dst_pass_kernel(const double* __restrict__ in, double* __restrict__ out, int nfields, int n,
                const double* __restrict__ lam_g, double inv_dt, double scale) {
  extern __shared__ double sm[];
  const int Po = (n + 1) / 2, Pe = n / 2;
  const int MTh = (Po + 7) / 8;
  const int KS = (Po + 3) / 4;
  const int rs = PASS < 2 ? LDX : 1;
  const int cs = PASS < 2 ? 1 : ldz_of(n);
  const int tile_elems = PASS < 2 ? n * LDX : TC * ldz_of(n);
  double* lam = sm + tile_elems;
  if (PASS == 2)
    for (int i = threadIdx.x; i < n; i += NT) lam[i] = lam_g[i];

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const WarpRole role = warp_role(warp, MTh);
  double afr[2][KSMAX];
#pragma unroll
  for (int t = 0; t < 2; ++t)
#pragma unroll
    for (int ks = 0; ks < KSMAX; ++ks)
      afr[t][ks] = (t < role.nmt && ks < KS)
                       ? fold_entry(n, Po, Pe, role.matrix, role.mt[t] * 8 + (lane >> 2), ks * 4 + (lane & 3))
                       : 0.0;

  const int nn = n * n;
  const int tiles_per_field = (nn + TC - 1) / TC;
  const long ntiles = (long)nfields * tiles_per_field;
  const size_t field = (size_t)nn * n;
  for (long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int f = (int)(tile / tiles_per_field);
    const int col0 = (int)(tile - (long)f * tiles_per_field) * TC;
    const double* src = in + (size_t)f * field;
    double* dst = out + (size_t)f * field;
    // load (zero-fill ragged columns)
    const int ne = n * TC;
    for (int idx = threadIdx.x; idx < ne; idx += NT) {
      int r, c;
      if (PASS == 2) { r = idx % n; c = idx / n; } else { r = idx / TC; c = idx % TC; }
      const int cg = col0 + c;
      sm[r * rs + c * cs] = (cg < nn) ? __ldcg(src + goff<PASS>(n, r, cg)) : 0.0;
    }
    __syncthreads();
    fold_transform<KSMAX, PASS == 2>(sm, rs, cs, n, Po, Pe, KS, role, afr, lam, inv_dt, scale, col0,
                                     PASS == 2);
    if (PASS == 2)
      fold_transform<KSMAX, false>(sm, rs, cs, n, Po, Pe, KS, role, afr, lam, inv_dt, scale, col0, true);
    for (int idx = threadIdx.x; idx < ne; idx += NT) {
      int r, c;
      if (PASS == 2) { r = idx % n; c = idx / n; } else { r = idx / TC; c = idx % TC; }
      const int cg = col0 + c;
      if (cg < nn) __stcg(dst + goff<PASS>(n, r, cg), sm[r * rs + c * cs]);
    }
    __syncthreads();
  }
}

template <int KSMAX>
struct PassSet {
  static cudaError_t run(int pass, const double* in, double* out, int nfields, int n, const double* lam,
                         double inv_dt, double scale, cudaStream_t s) {
    const size_t smem = (size_t)(pass < 2 ? n * LDX : TC * ldz_of(n)) * 8 + (size_t)n * 8;
    void (*k)(const double*, double*, int, int, const double*, double, double) =
        pass == 0 ? dst_pass_kernel<KSMAX, 0> : pass == 1 ? dst_pass_kernel<KSMAX, 1> : dst_pass_kernel<KSMAX, 2>;
    static int occ[3] = {0, 0, 0};
    static int sms = 0;
    if (!sms) {
      int dev;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    }
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    if (!occ[pass]) {
      e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ[pass], k, NT, smem);
      if (e != cudaSuccess) return e;
      if (occ[pass] < 1) occ[pass] = 1;
    }
    const long ntiles = (long)nfields * ((n * n + TC - 1) / TC);
    const int grid = (int)std::min<long>(ntiles, (long)sms * occ[pass]);
    DPM_COUNT_LAUNCH(1);
    k<<<grid, NT, smem, s>>>(in, out, nfields, n, lam, inv_dt, scale);
    return cudaGetLastError();
  }
};

cudaError_t run_pass(int pass, const double* in, double* out, int nfields, int n, const double* lam, double inv_dt,
                     double scale, cudaStream_t s) {
  const int Po = (n + 1) / 2, KS = (Po + 3) / 4;
  if (KS <= 4) return PassSet<4>::run(pass, in, out, nfields, n, lam, inv_dt, scale, s);
  if (KS <= 8) return PassSet<8>::run(pass, in, out, nfields, n, lam, inv_dt, scale, s);
  return PassSet<16>::run(pass, in, out, nfields, n, lam, inv_dt, scale, s);
}

__global__ void eig_kernel(double* lam, int n, double h) {
  const int m = blockIdx.x * blockDim.x + threadIdx.x + 1;
  if (m <= n) {
    const double s = sinpi((double)m / (2.0 * (n + 1)));
    lam[m - 1] = (4.0 / (h * h)) * s * s;
  }
}

}  // namespace

cudaError_t dst_plan_init(DstPlan& p, int n, double h, double dt) {
  p.n = n;
  p.h = h;
  p.dt = dt;
  cudaError_t e = cudaMalloc(&p.lam, sizeof(double) * n);
  if (e != cudaSuccess) return e;
  DPM_COUNT_LAUNCH(1);
  eig_kernel<<<(n + 127) / 128, 128>>>(p.lam, n, h);
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  return cudaDeviceSynchronize();
}

void dst_plan_free(DstPlan& p) {
  if (p.lam) cudaFree(p.lam);
  p.lam = nullptr;
}

size_t dst_scratch_bytes(int, int) { return 0; }

cudaError_t dst_solve_batch(const DstPlan& p, const double* q, double* u, int64_t batch, double*, size_t,
                            cudaStream_t s) {
  const int n = p.n;
  const size_t field_bytes = (size_t)n * n * n * 8;
  // chunk so that the in-flight working set (~2 chunks) stays in L2
  const size_t budget = (size_t)40 << 20;
  int64_t chunk = std::max<int64_t>(1, (int64_t)(budget / field_bytes));
  const double inv_dt = 1.0 / p.dt;
  const double sc = 2.0 / (n + 1);
  const double scale = sc * sc * sc;
  const size_t fe = (size_t)n * n * n;
  for (int64_t b0 = 0; b0 < batch; b0 += chunk) {
    const int nf = (int)std::min<int64_t>(chunk, batch - b0);
    const double* qi = q + b0 * fe;
    double* ui = u + b0 * fe;
    cudaError_t e;
    if ((e = run_pass(0, qi, ui, nf, n, p.lam, inv_dt, scale, s)) != cudaSuccess) return e;
    if ((e = run_pass(1, ui, ui, nf, n, p.lam, inv_dt, scale, s)) != cudaSuccess) return e;
    if ((e = run_pass(2, ui, ui, nf, n, p.lam, inv_dt, scale, s)) != cudaSuccess) return e;
    if ((e = run_pass(1, ui, ui, nf, n, p.lam, inv_dt, scale, s)) != cudaSuccess) return e;
    if ((e = run_pass(0, ui, ui, nf, n, p.lam, inv_dt, scale, s)) != cudaSuccess) return e;
  }
  return cudaSuccess;
}
