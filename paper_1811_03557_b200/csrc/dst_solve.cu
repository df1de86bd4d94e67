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
//  * Three tile kernels, each a persistent CTA loop over (field, TC-column) tiles that
//    hold ALL n samples of the transform axis in shared memory:
//      pass X: transform along x (stride n^2), columns = flat (y,z)
//      pass Y: transform along y (stride n),   columns = flat (x,z)
//      pass Z: transform along z (contiguous), divide by D (fused epilogue), inverse z
//    A solve is X, Y, Z, Y, X (DST-I is an involution up to the folded scale).
//  * Tiles stream in with cp.async (16-B LDGSTS, zero-fill for ragged columns) into a
//    double buffer: the next tile's load overlaps the current tile's DMMA work.
//  * Every warp keeps its sine-matrix fragments in REGISTERS for the whole kernel (loaded
//    once from a table built at plan creation with exact argument reduction), so the MMA
//    loop only loads B fragments from shared memory; row strides are padded
//    (≡ 4 mod 16 doubles) for conflict-free fragment loads.
//  * n = 128 (the throughput config) has its own instantiation with every size a
//    compile-time constant: no predication in the MMA loop.
//  * The batch is processed in chunks whose working set stays in the 126 MB L2, with the
//    intermediate living in the output buffer (u may alias q): HBM sees ~one read of q
//    and one write of u per solve.
#include <algorithm>
#include <cstdlib>

#include "dpm_internal.h"

namespace {

constexpr int NW = 8;         // warps per CTA
constexpr int NT = NW * 32;   // threads per CTA
constexpr int KSMAX_ALL = 16; // k-steps of the largest register-fragment instance (n <= 128)
// n in (128, 320] (the paper's N = 132 / 255 / 260 meshes): up to 5 m-tiles per warp and 40 k-steps,
// i.e. up to 200 A values per lane - too many for registers, so those fragments are read from the
// (L1/L2-resident) table inside the MMA loop, each one reused over the warp's column tiles.
// n in (320, 520] (the paper's N = 516 reference mesh): 9 m-tiles and 65 k-steps per warp.
constexpr int MT_BIG = 5, KS_BIG = 40, MT_HUGE = 9, KS_HUGE = 65;
__host__ __device__ constexpr int mt_of(int n) { return n > 320 ? MT_HUGE : (n > 128 ? MT_BIG : 2); }
__host__ __device__ constexpr int ks_of(int n) { return n > 320 ? KS_HUGE : (n > 128 ? KS_BIG : KSMAX_ALL); }

__host__ __device__ constexpr int ldx_of(int tc) { return tc + 4; }            // ≡ 4 mod 16 for tc % 16 == 0
__host__ __device__ constexpr int ldz_of(int n) { return ((n + 15) / 16) * 16 + 4; }

__device__ __forceinline__ void dmma884(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

__device__ __forceinline__ void cp_async16(unsigned smem_addr, const double* gmem, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(smem_addr), "l"(gmem), "r"(valid ? 16 : 0));
}
__device__ __forceinline__ void cp_async8(unsigned smem_addr, const double* gmem, bool valid) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(smem_addr), "l"(gmem), "r"(valid ? 8 : 0));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_async_wait1() { asm volatile("cp.async.wait_group 1;\n" ::); }

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
  int nmt;      // m-tiles owned (0..MT_HUGE)
  int mt[MT_HUGE];  // local m-tile indices
  int nct;      // column tiles handled
  int ct0, ctstep;
};

__host__ __device__ inline WarpRole warp_role(int warp, int MTh, int NCT) {
  WarpRole r;
  r.matrix = warp >> 2;
  const int wl = warp & 3;
  if (MTh > 8) {   // n > 128: m-tiles wl, wl + 4, wl + 8, ...
    r.nmt = 0;
    for (int t = 0; t < MT_HUGE; ++t) {
      r.mt[t] = wl + 4 * t;
      if (wl + 4 * t < MTh) r.nmt = t + 1;
    }
    r.ct0 = 0;
    r.ctstep = 1;
    r.nct = NCT;
  } else if (MTh >= 4) {
    r.mt[0] = wl;
    r.mt[1] = wl + 4;
    for (int t = 2; t < MT_HUGE; ++t) r.mt[t] = 0;
    r.nmt = (wl + 4 < MTh) ? 2 : 1;
    r.ct0 = 0;
    r.ctstep = 1;
    r.nct = NCT;
  } else {
    const int G = 4 / MTh;
    const int cg = wl / MTh;
    r.mt[0] = wl % MTh;
    for (int t = 1; t < MT_HUGE; ++t) r.mt[t] = 0;
    r.nmt = (cg < G) ? 1 : 0;
    r.ct0 = cg;
    r.ctstep = G;
    r.nct = (cg < G) ? (NCT - cg + G - 1) / G : 0;
  }
  return r;
}

// A-fragment table: tab[((warp*mt_of(n) + t)*ks_of(n) + ks)*32 + lane], built once per plan.
__global__ void afrag_table_kernel(double* tab, int n, int NCT) {
  const int warp = blockIdx.x, t = blockIdx.y, ks = blockIdx.z, lane = threadIdx.x;
  const int MTM = mt_of(n), KSM = ks_of(n);
  const int Po = (n + 1) / 2, Pe = n / 2, MTh = (Po + 7) / 8, KS = (Po + 3) / 4;
  const WarpRole role = warp_role(warp, MTh, NCT);
  double v = 0.0;
  if (t < role.nmt && ks < KS)
    v = fold_entry(n, Po, Pe, role.matrix, role.mt[t] * 8 + (lane >> 2), ks * 4 + (lane & 3));
  tab[((warp * MTM + t) * KSM + ks) * 32 + lane] = v;
}

// Compile-time geometry when NFIX > 0 (n = NFIX); runtime otherwise.
template <int NFIX, int TC, int PASS>
struct Geo {
  int n, Po, Pe, MTh, KS, rs, cs, tile_elems;
  __device__ __forceinline__ explicit Geo(int n_rt) {
    n = NFIX ? NFIX : n_rt;
    Po = (n + 1) / 2;
    Pe = n / 2;
    MTh = (Po + 7) / 8;
    KS = (Po + 3) / 4;
    rs = PASS < 2 ? ldx_of(TC) : 1;
    cs = PASS < 2 ? 1 : ldz_of(n);
    tile_elems = PASS < 2 ? n * ldx_of(TC) : TC * ldz_of(n);
  }
};

extern __shared__ __align__(16) double sm[];

// One folded DST-I of every column of the smem tile at sm[base ...], in place.
// Element (row r, col c) lives at sm[base + r*rs + c*cs].  If DIVIDE, the epilogue multiplies
// output (row k, column c) by scale / (((inv_dt + lam[a]) + lam[b]) + lam[k]) with
// (a, b) = divmod(col0 + c, n) (pass Z after X and Y: spectral indices).
template <int NFIX, int KSMAX, int TC, int PASS, bool DIVIDE, int MT>
__device__ __forceinline__ void fold_transform(const Geo<NFIX, TC, PASS>& G, int base, const WarpRole& role,
                                               const double (&afr)[2][MT == 2 ? KSMAX : 1], const double* atw,
                                               const double* lam, double inv_dt, double scale, int col0) {
  constexpr int NCT = TC / 8;
  constexpr bool ROWS_FAST = PASS == 2;
  const int n = G.n, Po = G.Po, Pe = G.Pe, rs = G.rs, cs = G.cs;
  const int tid = threadIdx.x, lane = tid & 31;
  // fold: s_j -> row j, d_j -> row n-1-j (middle row untouched)
  const int nf = Pe * TC;
  for (int idx = tid; idx < nf; idx += NT) {
    int j, c;
    if (ROWS_FAST) { j = idx % Pe; c = idx / Pe; } else { j = idx / TC; c = idx % TC; }
    const int pa = base + j * rs + c * cs;
    const int pb = base + (n - 1 - j) * rs + c * cs;
    const double a = sm[pa], b = sm[pb];
    sm[pa] = a + b;
    sm[pb] = a - b;
  }
  __syncthreads();

  double acc[MT][NCT][2];
#pragma unroll
  for (int t = 0; t < MT; ++t)
#pragma unroll
    for (int ct = 0; ct < NCT; ++ct) acc[t][ct][0] = acc[t][ct][1] = 0.0;

  if (MT > 2 && role.nmt > 0) {   // table-read A fragments, prefetched one k-step ahead
    const int colb = base + ((role.ct0 * 8) + (lane >> 2)) * cs;
    double an[MT];
#pragma unroll
    for (int t = 0; t < MT; ++t) an[t] = t < role.nmt ? __ldg(atw + t * KSMAX * 32) : 0.0;
#pragma unroll 2
    for (int ks = 0; ks < G.KS; ++ks) {
      double a[MT];
#pragma unroll
      for (int t = 0; t < MT; ++t) {
        a[t] = an[t];
        an[t] = (t < role.nmt && ks + 1 < G.KS) ? __ldg(atw + (t * KSMAX + ks + 1) * 32) : 0.0;
      }
      const int j = ks * 4 + (lane & 3);
      const int r = (role.matrix == 0) ? (j < Po ? j : 0) : (j < Pe ? n - 1 - j : 0);
      const int rowb = colb + r * rs;
      double b[NCT];
#pragma unroll
      for (int ct = 0; ct < NCT; ++ct) b[ct] = sm[rowb + ct * 8 * cs];
#pragma unroll
      for (int t = 0; t < MT; ++t)
#pragma unroll
        for (int ct = 0; ct < NCT; ++ct)
          if (t < role.nmt) dmma884(acc[t][ct], a[t], b[ct]);
    }
  } else if (role.nmt > 0) {
    const int colb = base + ((role.ct0 * 8) + (lane >> 2)) * cs;
    const int cstep = role.ctstep * 8 * cs;
#pragma unroll
    for (int ks = 0; ks < KSMAX; ++ks) {
      if (ks < G.KS) {
        const int j = ks * 4 + (lane & 3);
        const int r = (role.matrix == 0) ? (j < Po ? j : 0) : (j < Pe ? n - 1 - j : 0);
        const int rowb = colb + r * rs;
        double b[NCT];
#pragma unroll
        for (int ct = 0; ct < NCT; ++ct) b[ct] = (ct < role.nct) ? sm[rowb + ct * cstep] : 0.0;
#pragma unroll
        for (int t = 0; t < MT; ++t) {
          double a;
          if constexpr (MT == 2) a = afr[t][ks];
          else a = t < role.nmt ? __ldg(atw + (t * KSMAX + ks) * 32) : 0.0;
#pragma unroll
          for (int ct = 0; ct < NCT; ++ct)
            if (t < role.nmt && ct < role.nct) dmma884(acc[t][ct], a, b[ct]);
        }
      }
    }
  }
  __syncthreads();
  // epilogue: odd m -> row 2m, even m -> row 2m+1
  if (role.nmt > 0) {
    const int P = role.matrix == 0 ? Po : Pe;
#pragma unroll
    for (int t = 0; t < MT; ++t) {
      if (t >= role.nmt) continue;
      const int m = role.mt[t] * 8 + (lane >> 2);
      if (m >= P) continue;
      const int row = role.matrix == 0 ? 2 * m : 2 * m + 1;
      const double lrow = DIVIDE ? lam[row] : 0.0;
#pragma unroll
      for (int ct = 0; ct < NCT; ++ct) {
        if (ct >= role.nct) continue;
        const int c = (role.ct0 + ct * role.ctstep) * 8 + 2 * (lane & 3);
        double v0 = acc[t][ct][0], v1 = acc[t][ct][1];
        if (DIVIDE) {
          const int cg = col0 + c;
          if (cg < n * n) {
            const int a = cg / n, bb = cg - a * n;
            v0 *= scale / (((inv_dt + lam[a]) + lam[bb]) + lrow);
          }
          if (cg + 1 < n * n) {
            const int a = (cg + 1) / n, bb = cg + 1 - a * n;
            v1 *= scale / (((inv_dt + lam[a]) + lam[bb]) + lrow);
          }
        }
        const int o = base + row * rs + c * cs;
        if (PASS < 2) {
          *reinterpret_cast<double2*>(&sm[o]) = make_double2(v0, v1);   // cs == 1, o even
        } else {
          sm[o] = v0;
          sm[o + cs] = v1;
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

// Issue the cp.async loads of one tile (VEC doubles per request; zero-fill ragged columns).
template <int NFIX, int TC, int PASS, int VEC>
__device__ __forceinline__ void load_tile(const Geo<NFIX, TC, PASS>& G, int base, const double* src, int col0) {
  const int n = G.n, nn = n * n;
  const unsigned sbase = (unsigned)__cvta_generic_to_shared(sm) + 8u * (unsigned)base;
  if (PASS < 2) {
    constexpr int per_row = TC / VEC;
    const int ne = n * per_row;
    for (int idx = threadIdx.x; idx < ne; idx += NT) {
      const int r = idx / per_row, c = (idx - r * per_row) * VEC;
      const int cg = col0 + c;
      const bool ok = cg < nn;
      const double* g = ok ? src + goff<PASS>(n, r, cg) : src;
      const unsigned sa = sbase + 8u * (unsigned)(r * G.rs + c * G.cs);
      if (VEC == 2) cp_async16(sa, g, ok);
      else cp_async8(sa, g, ok);
    }
  } else {
    const int per_col = n / VEC;
    const int ne = TC * per_col;
    for (int idx = threadIdx.x; idx < ne; idx += NT) {
      const int c = idx / per_col, r = (idx - c * per_col) * VEC;
      const int cg = col0 + c;
      const bool ok = cg < nn;
      const double* g = ok ? src + goff<PASS>(n, r, cg) : src;
      const unsigned sa = sbase + 8u * (unsigned)(r * G.rs + c * G.cs);
      if (VEC == 2) cp_async16(sa, g, ok);
      else cp_async8(sa, g, ok);
    }
  }
}

template <int NFIX, int TC, int PASS, int VEC>
__device__ __forceinline__ void store_tile(const Geo<NFIX, TC, PASS>& G, int base, double* dst, int col0) {
  const int n = G.n, nn = n * n;
  if (PASS < 2) {
    constexpr int per_row = TC / VEC;
    const int ne = n * per_row;
    for (int idx = threadIdx.x; idx < ne; idx += NT) {
      const int r = idx / per_row, c = (idx - r * per_row) * VEC;
      const int cg = col0 + c;
      if (cg >= nn) continue;
      const int o = base + r * G.rs + c * G.cs;
      if (VEC == 2) __stcg(reinterpret_cast<double2*>(dst + goff<PASS>(n, r, cg)), *reinterpret_cast<const double2*>(&sm[o]));
      else __stcg(dst + goff<PASS>(n, r, cg), sm[o]);
    }
  } else {
    const int per_col = n / VEC;
    const int ne = TC * per_col;
    for (int idx = threadIdx.x; idx < ne; idx += NT) {
      const int c = idx / per_col, r = (idx - c * per_col) * VEC;
      const int cg = col0 + c;
      if (cg >= nn) continue;
      const int o = base + r * G.rs + c * G.cs;
      if (VEC == 2) __stcg(reinterpret_cast<double2*>(dst + goff<PASS>(n, r, cg)), *reinterpret_cast<const double2*>(&sm[o]));
      else __stcg(dst + goff<PASS>(n, r, cg), sm[o]);
    }
  }
}

template <int KSMAX, int TC>
constexpr int min_blocks() { return (KSMAX >= 16 && TC >= 64) || (KSMAX > 16 && TC > 16) || KSMAX > KS_BIG ? 1 : 2; }

template <int NFIX, int KSMAX, int TC, int PASS, int VEC, int MT = 2>
__global__ void __launch_bounds__(NT, min_blocks<KSMAX, TC>())
dst_pass_kernel(const double* __restrict__ in, double* __restrict__ out, int nfields, int n_rt,
                const double* __restrict__ lam_g, const double* __restrict__ atab, double inv_dt, double scale) {
  pdl_prologue();
  const Geo<NFIX, TC, PASS> G(n_rt);
  const int n = G.n;
  double* lam = sm + 2 * G.tile_elems;
  if (PASS == 2)
    for (int i = threadIdx.x; i < n; i += NT) lam[i] = lam_g[i];

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const WarpRole role = warp_role(warp, G.MTh, TC / 8);
  double afr[2][MT == 2 ? KSMAX : 1];
  const double* atw = atab + (size_t)warp * MT * KSMAX * 32 + lane;   // MT_BIG: read in the MMA loop
  if constexpr (MT == 2) {
#pragma unroll
    for (int t = 0; t < 2; ++t)
#pragma unroll
      for (int ks = 0; ks < KSMAX; ++ks) afr[t][ks] = __ldg(atab + ((warp * 2 + t) * KSMAX_ALL + ks) * 32 + lane);
  }

  const int nn = n * n;
  const int tiles_per_field = (nn + TC - 1) / TC;
  const long ntiles = (long)nfields * tiles_per_field;
  const size_t field = (size_t)nn * n;
  long tile = blockIdx.x;
  if (tile < ntiles) {
    const int f = (int)(tile / tiles_per_field);
    load_tile<NFIX, TC, PASS, VEC>(G, 0, in + (size_t)f * field, (int)(tile - (long)f * tiles_per_field) * TC);
  }
  cp_async_commit();
  int cur = 0;
  for (; tile < ntiles; tile += gridDim.x, cur ^= 1) {
    const long nxt = tile + gridDim.x;
    if (nxt < ntiles) {
      const int f = (int)(nxt / tiles_per_field);
      load_tile<NFIX, TC, PASS, VEC>(G, (cur ^ 1) * G.tile_elems, in + (size_t)f * field,
                                     (int)(nxt - (long)f * tiles_per_field) * TC);
    }
    cp_async_commit();
    cp_async_wait1();
    __syncthreads();
    const int f = (int)(tile / tiles_per_field);
    const int col0 = (int)(tile - (long)f * tiles_per_field) * TC;
    const int base = cur * G.tile_elems;
    fold_transform<NFIX, KSMAX, TC, PASS, PASS == 2, MT>(G, base, role, afr, atw, lam, inv_dt, scale, col0);
    if (PASS == 2) fold_transform<NFIX, KSMAX, TC, PASS, false, MT>(G, base, role, afr, atw, lam, inv_dt, scale, col0);
    store_tile<NFIX, TC, PASS, VEC>(G, base, out + (size_t)f * field, col0);
    __syncthreads();
  }
}

template <int NFIX, int KSMAX, int TC, int VEC, int MT = 2>
cudaError_t run_pass_t(int pass, const double* in, double* out, int nfields, int n, const double* lam,
                       const double* atab, double inv_dt, double scale, cudaStream_t s) {
  const size_t tile = (size_t)(pass < 2 ? n * ldx_of(TC) : TC * ldz_of(n));
  const size_t smem = 2 * tile * 8 + (size_t)n * 8;
  void (*k)(const double*, double*, int, int, const double*, const double*, double, double) =
      pass == 0 ? dst_pass_kernel<NFIX, KSMAX, TC, 0, VEC, MT>
                : pass == 1 ? dst_pass_kernel<NFIX, KSMAX, TC, 1, VEC, MT> : dst_pass_kernel<NFIX, KSMAX, TC, 2, VEC, MT>;
  static int sms = 0;
  static int occ[3] = {0, 0, 0};
  static size_t occ_smem[3] = {0, 0, 0};
  if (!sms) {
    int dev;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  if (!occ[pass] || occ_smem[pass] != smem) {
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ[pass], k, NT, smem);
    if (e != cudaSuccess) return e;
    if (occ[pass] < 1) occ[pass] = 1;
    occ_smem[pass] = smem;
  }
  const long ntiles = (long)nfields * ((n * n + TC - 1) / TC);
  const int grid = (int)std::min<long>(ntiles, (long)sms * occ[pass]);
  DPM_COUNT_LAUNCH(1);
  return launch_pdl(k, grid, NT, smem, s, in, out, nfields, n, lam, atab, inv_dt, scale);
}

// Column-tile width of the n = 128 instance (DPM_TC128 = 32 | 64 selects; default below).
int tc128() {
  static int v = [] {
    const char* e = getenv("DPM_TC128");
    return (e && atoi(e) == 64) ? 64 : 32;   // 32: 2 CTAs/SM, 61% of DMMA peak vs 53% for 64 (profiles/)
  }();
  return v;
}

int tc_for(int n) { return n == 128 ? tc128() : (n > 128 ? 32 : (n > 64 ? 64 : 32)); }

cudaError_t run_pass(const DstPlan& p, int pass, const double* in, double* out, int nfields, double inv_dt,
                     double scale, cudaStream_t s) {
  const int n = p.n;
  const int Po = (n + 1) / 2, KS = (Po + 3) / 4;
  const bool even = (n % 2) == 0;
  if (n == 128 && pass < 2 && p.pfa) return dst128_pass(pass, in, out, nfields, p.atab128, s);
  if (n == 128) {
    if (tc128() == 32) return run_pass_t<128, 16, 32, 2>(pass, in, out, nfields, n, p.lam, p.atab, inv_dt, scale, s);
    return run_pass_t<128, 16, 64, 2>(pass, in, out, nfields, n, p.lam, p.atab, inv_dt, scale, s);
  }
  if (KS <= 4) {
    return even ? run_pass_t<0, 4, 32, 2>(pass, in, out, nfields, n, p.lam, p.atab, inv_dt, scale, s)
                : run_pass_t<0, 4, 32, 1>(pass, in, out, nfields, n, p.lam, p.atab, inv_dt, scale, s);
  }
  if (KS <= 8) {
    return even ? run_pass_t<0, 8, 32, 2>(pass, in, out, nfields, n, p.lam, p.atab, inv_dt, scale, s)
                : run_pass_t<0, 8, 32, 1>(pass, in, out, nfields, n, p.lam, p.atab, inv_dt, scale, s);
  }
  if (n > 320) {   // 320 < n <= 520: 9 m-tiles x 65 k-steps per warp, 16-column tiles (2 x 83 KB), 1 CTA/SM
    return even ? run_pass_t<0, KS_HUGE, 16, 2, MT_HUGE>(pass, in, out, nfields, n, p.lam, p.atab, inv_dt, scale, s)
                : run_pass_t<0, KS_HUGE, 16, 1, MT_HUGE>(pass, in, out, nfields, n, p.lam, p.atab, inv_dt, scale, s);
  }
  if (n > 128) {   // 128 < n <= 320: A fragments from the table (prefetched one k-step ahead);
    // TC = 16 (2 CTAs = 16 warps per SM) beats TC = 32 (1 CTA, twice the A reuse) by 5-8% at
    // n = 132 / 255 (tools/big_n_profile.py); DPM_TCBIG=32 selects the latter
    static const int tcb = [] {
      const char* e = getenv("DPM_TCBIG");
      return (e && atoi(e) == 32) ? 32 : 16;
    }();
    if (tcb == 16)
      return even ? run_pass_t<0, KS_BIG, 16, 2, MT_BIG>(pass, in, out, nfields, n, p.lam, p.atab, inv_dt, scale, s)
                  : run_pass_t<0, KS_BIG, 16, 1, MT_BIG>(pass, in, out, nfields, n, p.lam, p.atab, inv_dt, scale, s);
    return even ? run_pass_t<0, KS_BIG, 32, 2, MT_BIG>(pass, in, out, nfields, n, p.lam, p.atab, inv_dt, scale, s)
                : run_pass_t<0, KS_BIG, 32, 1, MT_BIG>(pass, in, out, nfields, n, p.lam, p.atab, inv_dt, scale, s);
  }
  return even ? run_pass_t<0, 16, 64, 2>(pass, in, out, nfields, n, p.lam, p.atab, inv_dt, scale, s)
              : run_pass_t<0, 16, 64, 1>(pass, in, out, nfields, n, p.lam, p.atab, inv_dt, scale, s);
}

// ---------------------------------------------------------------------------------------------
// Partial diagonalisation (DPM_SOLVER_DST2_TRIDIAG): after DST-I along x and y, every (a, b)
// line along z solves  (σ_ab - D_zz) v = r  with σ_ab = 1/dt + λ_a + λ_b and zero Dirichlet ends.
// h^2-scaled: T v = h^2 r, T = tridiag(-1, β, -1), β = 2 + h^2 σ_ab = μ + 1/μ, 0 < μ < 1.
// Exact identity: T = A + μ e1 e1^T with A = μ^{-1} (I - μL)(I - μU) (L/U = sub/super shift), so
//   A^{-1} r = μ z,  z = (I - μU)^{-1} (I - μL)^{-1} r   (two constant-coefficient recurrences)
//   T^{-1} r = μ z - s · μ (μ z_0) / (1 + μ s_0),   s_k = (μ^{k+1} - μ^{2n+1-k}) / (1 - μ^2)
// (Sherman-Morrison; s = A^{-1} e1 in closed form).  Two divisions per line, no pivot table.
//
// One warp per line (every n <= 128): lane l holds z = 4l..4l+3;
// each first-order recurrence is a local 4-step sweep plus a 5-step Kogge–Stone carry scan over the
// warp with multipliers μ^4, μ^8, ..., so no shared memory, no barriers and one 1 KB line per warp
// in flight; Sherman–Morrison powers μ^{k+1}, μ^{2n+1-k} by binary exponentiation per lane.
__device__ __forceinline__ double ipow(double b, int e) {   // b^e, e >= 0
  double r = 1.0;
  while (e > 0) {
    if (e & 1) r *= b;
    b *= b;
    e >>= 1;
  }
  return r;
}

template <int NFIX, int PER = 4>
__global__ void __launch_bounds__(256)
ztri_warp_kernel(double* __restrict__ u, int nlines, int n_rt, const double* __restrict__ lam_g, double inv_dt,
                 double h2, double rscale) {
  __shared__ double lam[DPM_MAX_N];
  const int n = NFIX ? NFIX : n_rt;
  for (int i = threadIdx.x; i < n; i += blockDim.x) lam[i] = lam_g[i];
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int w0 = (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5), nw = (int)((gridDim.x * blockDim.x) >> 5);
  const int nn = n * n, k0 = PER * lane;
  for (int line = w0; line < nlines; line += nw) {   // nlines < 2^31 (checked by the launcher)
    double* L = u + (size_t)line * n;
    double r[PER];
    if (NFIX == 32 * PER) {
#pragma unroll
      for (int i = 0; i < PER; i += 2) {
        const double2 a = __ldcg(reinterpret_cast<const double2*>(L + k0 + i));
        r[i] = a.x;
        r[i + 1] = a.y;
      }
    } else {
#pragma unroll
      for (int i = 0; i < PER; ++i) r[i] = k0 + i < n ? __ldcg(L + k0 + i) : 0.0;
    }
    const int lf = line % nn;
    const double hs = h2 * ((inv_dt + lam[lf / n]) + lam[lf % n]);
    const double disc = sqrt(hs * (hs + 4.0));
    const double mu = 2.0 / ((2.0 + hs) + disc);
    double mpow[PER + 1];   // μ^0 .. μ^PER
    mpow[0] = 1.0;
#pragma unroll
    for (int i = 1; i <= PER; ++i) mpow[i] = mpow[i - 1] * mu;
    double mp[5];   // μ^{PER·2^s}
    mp[0] = mpow[PER];
#pragma unroll
    for (int q = 1; q < 5; ++q) mp[q] = mp[q - 1] * mp[q - 1];
    // forward y_k = r_k + μ y_{k-1}
    double y[PER];
    y[0] = rscale * r[0];
#pragma unroll
    for (int i = 1; i < PER; ++i) y[i] = fma(mu, y[i - 1], rscale * r[i]);
    double C = y[PER - 1];
#pragma unroll
    for (int q = 0; q < 5; ++q) {
      const double t = __shfl_up_sync(0xffffffffu, C, 1 << q);
      C = fma(lane >= (1 << q) ? mp[q] : 0.0, t, C);
    }
    double cin = __shfl_up_sync(0xffffffffu, C, 1);
    cin = lane == 0 ? 0.0 : cin;
#pragma unroll
    for (int i = 0; i < PER; ++i) y[i] = fma(mpow[i + 1], cin, y[i]);
#pragma unroll
    for (int i = 0; i < PER; ++i)
      if (k0 + i >= n) y[i] = 0.0;   // padding beyond the line: ghost values
    // backward z_k = y_k + μ z_{k+1}
    double z[PER];
    z[PER - 1] = y[PER - 1];
#pragma unroll
    for (int i = PER - 2; i >= 0; --i) z[i] = fma(mu, z[i + 1], y[i]);
    double D = z[0];
#pragma unroll
    for (int q = 0; q < 5; ++q) {
      const double t = __shfl_down_sync(0xffffffffu, D, 1 << q);
      D = fma(lane + (1 << q) < 32 ? mp[q] : 0.0, t, D);
    }
    double din = __shfl_down_sync(0xffffffffu, D, 1);
    din = lane == 31 ? 0.0 : din;
#pragma unroll
    for (int i = 0; i < PER; ++i) z[i] = fma(mpow[PER - i], din, z[i]);
    // T^{-1} r = μ z - c2 (μ^{k+1} - μ^{2n+1-k}),  c2 = μ^2 z_0 / (1 - μ^{2n+2})
    // (Sherman–Morrison with s = A^{-1} e_1 in closed form; (1 + μ s_0)(1 - μ^2) = 1 - μ^{2n+2}).
    // Powers by binary exponentiation over the lane bits with the μ^{PER·2^s} table:
    //   μ^{k0+1} = μ · μ^{PER lane},  μ^{2n+2-PER-k0} = μ^{E} · μ^{PER(NL-1-lane)},
    //   E = 2n + 2 - PER·NL >= n + 3 - PER.
    const int NL = (n + PER - 1) / PER;   // lanes holding line data
    const int lr = max(0, NL - 1 - lane);
    double P1 = 1.0, P2 = 1.0;
#pragma unroll
    for (int q = 0; q < 5; ++q) {
      P1 *= (lane >> q) & 1 ? mp[q] : 1.0;
      P2 *= (lr >> q) & 1 ? mp[q] : 1.0;
    }
    const double muE = ipow(mu, 2 * n + 2 - PER * NL);                         // warp-uniform exponent
    const double muPL = __shfl_sync(0xffffffffu, P1, NL - 1) * mpow[PER];      // μ^{PER NL}
    const double mu2n2 = muE * muPL;                                           // μ^{2n+2}
    const double zf = __shfl_sync(0xffffffffu, z[0], 0);
    const double c2 = mpow[2] * zf / (1.0 - mu2n2);
    const double pa = mu * P1, pb = muE * P2;
    double o[PER];
#pragma unroll
    for (int i = 0; i < PER; ++i) o[i] = fma(mu, z[i], -c2 * (pa * mpow[i] - pb * mpow[PER - 1 - i]));
    if (NFIX == 32 * PER) {
#pragma unroll
      for (int i = 0; i < PER; i += 2) __stcg(reinterpret_cast<double2*>(L + k0 + i), make_double2(o[i], o[i + 1]));
    } else {
#pragma unroll
      for (int i = 0; i < PER; ++i)
        if (k0 + i < n) __stcg(L + k0 + i, o[i]);
    }
  }
}

// ---------------------------------------------------------------------------------------------
// Fused plane pass for n <= 64 (the PKS configs cfg2 / cfg3, whose AP batches hold only 2 fields):
// one CTA per x-mode plane a ([y][z], n x n, contiguous) with the plane and the sine matrix in
// shared memory: y DST-I (S^T P, 4 x 4 register tiles), the exact z tridiagonal of every y-mode row
// (warp per row, 2 entries per lane: the recurrences, Kogge–Stone carries and Sherman–Morrison of
// ztri_warp_kernel), inverse y DST-I.  One launch instead of three (y, z, y).
// PS_PP = 72 (≡ 8 mod 16): the DMMA B-fragment loads of the plane hit each 8-byte bank pair twice and its rows
// are 16-byte aligned (double2 row accesses in the tridiagonal); PS_SP = 66 (≡ 2 mod 8): the A-fragment loads
// of the sine matrix do the same (cfg3 12.75k -> 13.0k steps/s against 65 / 65)
#ifndef PS_PP
#define PS_PP 72
#endif
#ifndef PS_SP
#define PS_SP 66
#endif
#ifndef PS_TRI_VEC
#define PS_TRI_VEC 0   // double2 row pairs in the tridiagonal (needs an even PS_PP; measured slower: 12.8k vs 13.0k cfg3)
#endif
// largest n; shared-memory row pitches of the plane (PSP) and of the sine matrix (SSP)
constexpr int PSN = 64, PSP = PS_PP, SSP = PS_SP;

__global__ void sinmat_kernel(double* S, int n) {   // S[j][k] = sin(π (j+1)(k+1)/(n+1)), exact reduction
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n * n) return;
  const int j = e / n, k = e % n;
  S[e] = sinpi((double)(((j + 1) * (k + 1)) % (2 * (n + 1))) / (double)(n + 1));
}

// P <- S^T P in place (S symmetric); thread (rb, cb) = (t / 16, t % 16) owns rows 4rb..4rb+3 and
// columns cb + 16j; S and P are zero-padded to 64 x 64.  (512 threads with 2 x 4 tiles: slower.)
#ifndef PS_THREADS_CFG
#define PS_THREADS_CFG 256
#endif
constexpr int PS_THREADS = PS_THREADS_CFG;
__device__ __forceinline__ void ps_apply(const double* S, double* P, int n) {
  const int t = threadIdx.x, rb = t >> 4, cb = t & 15;
  double acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;
  if (4 * rb < n) {
    if ((n & 1) == 0) {
      // folded: sin(π(N-j)k/N) = (-1)^{k+1} sin(πjk/N), N = n + 1, so output row b (k = b + 1) needs
      // x_y + x_{n-1-y} (b even) or x_y - x_{n-1-y} (b odd) over y < n/2 only: half the products
#pragma unroll 2
      for (int y = 0; y < n / 2; ++y) {
        double sv[4], ap[4], am[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) sv[i] = S[y * SSP + 4 * rb + i];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const double p1 = P[y * PSP + cb + 16 * j], p2 = P[(n - 1 - y) * PSP + cb + 16 * j];
          ap[j] = p1 + p2;
          am[j] = p1 - p2;
        }
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[i][j] = fma(sv[i], (i & 1) ? am[j] : ap[j], acc[i][j]);
      }
    } else {
#pragma unroll 4
      for (int y = 0; y < n; ++y) {
        double sv[4], pv[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) sv[i] = S[y * SSP + 4 * rb + i];
#pragma unroll
        for (int j = 0; j < 4; ++j) pv[j] = P[y * PSP + cb + 16 * j];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[i][j] = fma(sv[i], pv[j], acc[i][j]);
      }
    }
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j)
      if (4 * rb + i < n && cb + 16 * j < n) P[(4 * rb + i) * PSP + cb + 16 * j] = acc[i][j];
  __syncthreads();
}

// The same y DST-I (P <- S P, even n) on the fp64 tensor pipe (DMMA.8x8x4): the folded products
// out[b] = Σ_{y < n/2} S[b][y] (P[y] ± P[n-1-y]) (+ for even b, - for odd b) are an (even rows | odd rows) x
// (y < n/2) x (z) product, m-tiles of 8 even or 8 odd output rows, n-tiles of 8 z, k-steps of 4 y.  Warp w
// owns n-tile w % NT and every (8 / NT)-th m-tile: its B± fragments are formed once per k-step (one DADD)
// and reused by all its m-tiles, whose accumulators are independent DMMA chains.  About 5x fewer issued
// instructions than the DFMA tiles of ps_apply for the same flops (the small-n plane pass is issue- and
// latency-bound, not fp64-throughput-bound).  Rows / columns >= n are zero in S and P; the A fragments
// of y >= n/2 are masked to 0.
__device__ __forceinline__ void ps_apply_dmma(const double* S, double* P, int n) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int half = n >> 1;
  const int NT = (n + 7) >> 3;                 // n-tiles of 8 z
  const int MH = (half + 7) >> 3;              // m-tiles per parity (8 output rows of one parity)
  const int wpn = max(1, (PS_THREADS / 32) / NT);
  const int nt = w % NT, mg = w / NT;
  const bool active = w < NT * wpn;
  const int KS = (half + 3) >> 2;              // k-steps of 4 y
  double acc[2][4][2];                          // [parity][m-tile slot][2]
#pragma unroll
  for (int s = 0; s < 2; ++s)
#pragma unroll
    for (int q = 0; q < 4; ++q) acc[s][q][0] = acc[s][q][1] = 0.0;
  const int zb = 8 * nt + (lane >> 2), rl = lane >> 2, kl = lane & 3;
  if (active) {
    for (int kk = 0; kk < KS; ++kk) {
      const int y = 4 * kk + kl;
      const bool yin = y < half;
      const double p1 = yin ? P[y * PSP + zb] : 0.0, p2 = yin ? P[(n - 1 - y) * PSP + zb] : 0.0;
      const double bp = p1 + p2, bm = p1 - p2;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int i = mg + q * wpn;            // m-tile index of this slot
        if (i >= MH) break;
        const int be = 2 * (8 * i + rl);       // this lane's A row (even set); the odd set is be + 1
        const double ae = yin ? S[be * SSP + y] : 0.0, ao = yin ? S[(be + 1) * SSP + y] : 0.0;
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(acc[0][q][0]), "+d"(acc[0][q][1]) : "d"(ae), "d"(bp));
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(acc[1][q][0]), "+d"(acc[1][q][1]) : "d"(ao), "d"(bm));
      }
    }
  }
  __syncthreads();                              // every read of P done
  if (active) {
    const int zc = 8 * nt + 2 * (lane & 3);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int i = mg + q * wpn;
      if (i >= MH) break;
#pragma unroll
      for (int s = 0; s < 2; ++s) {
        const int b = 2 * (8 * i + rl) + s;
        P[b * PSP + zc] = acc[s][q][0];
        P[b * PSP + zc + 1] = acc[s][q][1];
      }
    }
  }
  __syncthreads();
}

// exact solve of (hs + 2) v_k - v_{k-1} - v_{k+1} = rscale r_k (k < n <= 64, zero ends) in place, one
// warp; mu = μ(hs) and inv_den = 1/(1 - μ^{2n+2}) come precomputed (lane-parallel over the warp's rows)
__device__ __forceinline__ void ps_tri_row(double* row, int n, double mu, double inv_den, double rscale) {
  const int lane = threadIdx.x & 31, k0 = 2 * lane;
  const double mu2 = mu * mu;
  double mp[7];   // μ^{2·2^q}
  mp[0] = mu2;
#pragma unroll
  for (int q = 1; q < 7; ++q) mp[q] = mp[q - 1] * mp[q - 1];
  const double r0 = k0 < n ? row[k0] : 0.0, r1 = k0 + 1 < n ? row[k0 + 1] : 0.0;
  // forward y_k = r_k + μ y_{k-1}
  double y0 = rscale * r0, y1 = fma(mu, y0, rscale * r1);
  double C = y1;
#pragma unroll
  for (int q = 0; q < 5; ++q) {
    const double tq = __shfl_up_sync(0xffffffffu, C, 1 << q);
    if (lane >= (1 << q)) C = fma(mp[q], tq, C);
  }
  double cin = __shfl_up_sync(0xffffffffu, C, 1);
  cin = lane == 0 ? 0.0 : cin;
  y0 = fma(mu, cin, y0);
  y1 = fma(mu2, cin, y1);
  if (k0 >= n) y0 = 0.0;
  if (k0 + 1 >= n) y1 = 0.0;
  // backward z_k = y_k + μ z_{k+1}
  double z1 = y1, z0 = fma(mu, y1, y0);
  double D = z0;
#pragma unroll
  for (int q = 0; q < 5; ++q) {
    const double tq = __shfl_down_sync(0xffffffffu, D, 1 << q);
    if (lane + (1 << q) < 32) D = fma(mp[q], tq, D);
  }
  double din = __shfl_down_sync(0xffffffffu, D, 1);
  din = lane == 31 ? 0.0 : din;
  z1 = fma(mu, din, z1);
  z0 = fma(mu2, din, z0);
  // T^{-1} r = μ z - c2 (μ^{k+1} - μ^{2n+1-k}),  c2 = μ^2 z_0 / (1 - μ^{2n+2});  direct powers
  // μ^{2 lane} and μ^{2(n - lane)} from the bits of lane and n - lane
  const double zf = __shfl_sync(0xffffffffu, z0, 0);
  const double c2 = mu2 * zf * inv_den;
  const int rl = max(0, n - lane);
  double pl = 1.0, pr = 1.0;
#pragma unroll
  for (int q = 0; q < 7; ++q) {
    if ((lane >> q) & 1) pl *= mp[q];
    if ((rl >> q) & 1) pr *= mp[q];
  }
  const double pa0 = mu * pl;   // μ^{k0+1}
  const double pb1 = pr;        // μ^{2n-k0} = μ^{2n+1-(k0+1)}
  if (k0 < n) row[k0] = fma(mu, z0, -c2 * (pa0 - pb1 * mu));
  if (k0 + 1 < n) row[k0 + 1] = fma(mu, z1, -c2 * (pa0 * mu - pb1));
}

// ps_tri_row on R rows at once (their recurrences and shuffle scans interleaved: R independent chains per
// warp instead of one); rows with valid[r] == false are skipped (their lanes compute on zeros)
template <int R>
__device__ __forceinline__ void ps_tri_rows(double* const (&row)[R], const bool (&valid)[R], int n,
                                            const double (&mu)[R], const double (&inv_den)[R], double rscale) {
  const int lane = threadIdx.x & 31, k0 = 2 * lane;
  double mu2[R], mp[R][7], y0[R], y1[R], C[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    mu2[r] = mu[r] * mu[r];
    mp[r][0] = mu2[r];
#pragma unroll
    for (int q = 1; q < 7; ++q) mp[r][q] = mp[r][q - 1] * mp[r][q - 1];
    double r0 = 0.0, r1 = 0.0;
    if (valid[r] && k0 + 1 < n && (PSP % 2) == 0 && PS_TRI_VEC) {   // 16-byte aligned pair
      const double2 v = *reinterpret_cast<const double2*>(row[r] + k0);
      r0 = v.x;
      r1 = v.y;
    } else {
      r0 = (valid[r] && k0 < n) ? row[r][k0] : 0.0;
      r1 = (valid[r] && k0 + 1 < n) ? row[r][k0 + 1] : 0.0;
    }
    y0[r] = rscale * r0;
    y1[r] = fma(mu[r], y0[r], rscale * r1);
    C[r] = y1[r];
  }
#pragma unroll
  for (int q = 0; q < 5; ++q)
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const double tq = __shfl_up_sync(0xffffffffu, C[r], 1 << q);
      if (lane >= (1 << q)) C[r] = fma(mp[r][q], tq, C[r]);
    }
  double z0[R], z1[R], D[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    double cin = __shfl_up_sync(0xffffffffu, C[r], 1);
    cin = lane == 0 ? 0.0 : cin;
    y0[r] = fma(mu[r], cin, y0[r]);
    y1[r] = fma(mu2[r], cin, y1[r]);
    if (k0 >= n) y0[r] = 0.0;
    if (k0 + 1 >= n) y1[r] = 0.0;
    z1[r] = y1[r];
    z0[r] = fma(mu[r], y1[r], y0[r]);
    D[r] = z0[r];
  }
#pragma unroll
  for (int q = 0; q < 5; ++q)
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const double tq = __shfl_down_sync(0xffffffffu, D[r], 1 << q);
      if (lane + (1 << q) < 32) D[r] = fma(mp[r][q], tq, D[r]);
    }
  const int rl = max(0, n - lane);
#pragma unroll
  for (int r = 0; r < R; ++r) {
    double din = __shfl_down_sync(0xffffffffu, D[r], 1);
    din = lane == 31 ? 0.0 : din;
    z1[r] = fma(mu[r], din, z1[r]);
    z0[r] = fma(mu2[r], din, z0[r]);
    const double zf = __shfl_sync(0xffffffffu, z0[r], 0);
    const double c2 = mu2[r] * zf * inv_den[r];
    double pl = 1.0, pr = 1.0;
#pragma unroll
    for (int q = 0; q < 7; ++q) {
      if ((lane >> q) & 1) pl *= mp[r][q];
      if ((rl >> q) & 1) pr *= mp[r][q];
    }
    const double pa0 = mu[r] * pl, pb1 = pr;
    const double o0 = fma(mu[r], z0[r], -c2 * (pa0 - pb1 * mu[r]));
    const double o1 = fma(mu[r], z1[r], -c2 * (pa0 * mu[r] - pb1));
    if (valid[r] && k0 + 1 < n && (PSP % 2) == 0 && PS_TRI_VEC) {
      *reinterpret_cast<double2*>(row[r] + k0) = make_double2(o0, o1);
    } else {
      if (valid[r] && k0 < n) row[r][k0] = o0;
      if (valid[r] && k0 + 1 < n) row[r][k0 + 1] = o1;
    }
  }
}

#ifndef PS_ROWS
#define PS_ROWS 2
#endif
__device__ int g_ps_dmma = 1;   // DPM_PLANE_SMALL_DMMA=0 -> 0 (set by dst_plan_init)
__device__ __forceinline__ bool ps_dmma() { return g_ps_dmma != 0; }

// y DST-I, z tridiagonal of every y-mode row, inverse y DST-I of one plane held in shared memory
// (S: the sine matrix, P: the plane, both zero-padded to PSN x PSN at pitch PSP; a: the x mode)
__device__ __forceinline__ void plane_small_body(const double* S, double* P, const double* lam, int n, int a,
                                                 double inv_dt, double h2, double rscale) {
  const int t = threadIdx.x;
  const bool tc = ps_dmma() && (n & 1) == 0;
  if (tc) ps_apply_dmma(S, P, n); else ps_apply(S, P, n);
  {
    // warp w solves rows b = w + 8 i (i < 8); lane i first computes μ and 1/(1 - μ^{2n+2}) of row i
    const int w = t >> 5, lane = t & 31, nw = blockDim.x >> 5;
    double mu_l = 0.5, id_l = 1.0;
    const int bl = w + nw * lane;
    if (lane < 8 && bl < n) {
      const double hs = h2 * ((inv_dt + lam[a]) + lam[bl]);
      mu_l = 2.0 / ((2.0 + hs) + sqrt(hs * (hs + 4.0)));
      id_l = 1.0 / (1.0 - ipow(mu_l, 2 * n + 2));
    }
    for (int i = 0; i < 8; i += PS_ROWS) {   // PS_ROWS rows at a time: interleaved recurrence chains
      double* rows[PS_ROWS];
      bool valid[PS_ROWS];
      double mu[PS_ROWS], id[PS_ROWS];
#pragma unroll
      for (int r = 0; r < PS_ROWS; ++r) {
        rows[r] = P + (w + nw * (i + r)) * PSP;
        valid[r] = w + nw * (i + r) < n;
        mu[r] = __shfl_sync(0xffffffffu, mu_l, i + r);
        id[r] = __shfl_sync(0xffffffffu, id_l, i + r);
      }
      if (valid[0]) ps_tri_rows<PS_ROWS>(rows, valid, n, mu, id, rscale);
    }
  }
  __syncthreads();
  if (tc) ps_apply_dmma(S, P, n); else ps_apply(S, P, n);
}

__global__ void __launch_bounds__(PS_THREADS) plane_small_kernel(double* __restrict__ u, int n, const double* __restrict__ S_g,
                                                          const double* __restrict__ lam_g, double inv_dt, double h2,
                                                          double rscale) {
  pdl_prologue();
  extern __shared__ double psm_small[];
  double* S = psm_small;           // [64][SSP]
  double* P = S + PSN * SSP;       // [64][PSP]
  double* lam = P + PSN * PSP;     // [64]
  const long plane = blockIdx.x;   // field * n + a
  const int a = (int)(plane % n), t = threadIdx.x;
  double* g = u + (size_t)plane * n * n;
  {   // every load in flight at once (cp.async, zero-filled outside the n x n corner)
    const unsigned sS = (unsigned)__cvta_generic_to_shared(S), sP = (unsigned)__cvta_generic_to_shared(P);
#pragma unroll 4
    for (int e = t; e < PSN * PSN; e += PS_THREADS) {
      const int r = e / PSN, c = e % PSN;
      const bool in = r < n && c < n;
      cp_async8(sS + 8u * (unsigned)(r * SSP + c), in ? S_g + r * n + c : S_g, in);
      cp_async8(sP + 8u * (unsigned)(r * PSP + c), in ? g + (size_t)r * n + c : g, in);
    }
    cp_async_commit();
  }
  for (int i = t; i < n; i += blockDim.x) lam[i] = lam_g[i];
  asm volatile("cp.async.wait_group 0;\n" ::);
  __syncthreads();
  plane_small_body(S, P, lam, n, a, inv_dt, h2, rscale);
  for (int r = t >> 5; r < n; r += PS_THREADS / 32)   // (no per-element division)
    for (int c = t & 31; c < n; c += 32) g[r * n + c] = P[r * PSP + c];
}

// Batched small-n plane pass (Step-4b rebuilds: K fields at once): persistent CTAs that load the sine
// matrix once and stream planes through two buffers (the next plane's cp.async in flight under the
// current plane's transforms); the same per-plane arithmetic as plane_small_kernel.
__global__ void __launch_bounds__(PS_THREADS) plane_small_batch_kernel(double* __restrict__ u, int n,
                                                                       const double* __restrict__ S_g,
                                                                       const double* __restrict__ lam_g, double inv_dt,
                                                                       double h2, double rscale, long nplanes) {
  pdl_prologue();
  extern __shared__ double psm_small[];
  double* S = psm_small;              // [64][SSP]
  double* PB = S + PSN * SSP;         // 2 x [64][PSP]
  double* lam = PB + 2 * PSN * PSP;   // [64]
  const int t = threadIdx.x;
  auto load_plane = [&](double* P, long plane) {
    const double* g = u + (size_t)plane * n * n;
    const unsigned sP = (unsigned)__cvta_generic_to_shared(P);
#pragma unroll 4
    for (int e = t; e < PSN * PSN; e += PS_THREADS) {
      const int r = e / PSN, c = e % PSN;
      const bool in = r < n && c < n;
      cp_async8(sP + 8u * (unsigned)(r * PSP + c), in ? g + (size_t)r * n + c : g, in);
    }
  };
  {
    const unsigned sS = (unsigned)__cvta_generic_to_shared(S);
#pragma unroll 4
    for (int e = t; e < PSN * PSN; e += PS_THREADS) {
      const int r = e / PSN, c = e % PSN;
      const bool in = r < n && c < n;
      cp_async8(sS + 8u * (unsigned)(r * SSP + c), in ? S_g + r * n + c : S_g, in);
    }
  }
  for (int i = t; i < n; i += blockDim.x) lam[i] = lam_g[i];
  if ((long)blockIdx.x < nplanes) load_plane(PB, blockIdx.x);
  cp_async_commit();
  int b = 0;
  for (long plane = blockIdx.x; plane < nplanes; plane += gridDim.x, b ^= 1) {
    const long nxt = plane + gridDim.x;
    if (nxt < nplanes) load_plane(PB + (b ^ 1) * PSN * PSP, nxt);
    cp_async_commit();
    asm volatile("cp.async.wait_group 1;\n" ::);
    __syncthreads();
    double* P = PB + b * PSN * PSP;
    plane_small_body(S, P, lam, n, (int)(plane % n), inv_dt, h2, rscale);
    double* g = u + (size_t)plane * n * n;
    for (int r = t >> 5; r < n; r += PS_THREADS / 32)
      for (int c = t & 31; c < n; c += 32) g[r * n + c] = P[r * PSP + c];
    __syncthreads();   // the buffer is refilled by the prefetch of the next iteration but one
  }
  asm volatile("cp.async.wait_group 0;\n" ::);
}

cudaError_t run_plane_small(const DstPlan& p, double* u, int nfields, cudaStream_t s) {
  const int n = p.n;
  const size_t smem = ((size_t)PSN * (SSP + PSP) + PSN) * sizeof(double);
  cudaError_t e = cudaFuncSetAttribute(plane_small_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const double sc = 2.0 / (n + 1);
  const long planes = (long)nfields * n;
  static const bool batch_on = [] {   // DPM_PLANE_SMALL_BATCH=0: one CTA per plane at every batch size
    const char* v = getenv("DPM_PLANE_SMALL_BATCH");
    return !(v && atoi(v) == 0);
  }();
  if (batch_on && planes > 4L * 148) {
    const size_t bsmem = ((size_t)PSN * (SSP + 2 * PSP) + PSN) * sizeof(double);
    e = cudaFuncSetAttribute(plane_small_batch_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bsmem);
    if (e != cudaSuccess) return e;
    int occ = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, plane_small_batch_kernel, PS_THREADS, bsmem);
    DPM_COUNT_LAUNCH(1);
    return launch_pdl(plane_small_batch_kernel, (unsigned)std::min<long>(planes, 148L * std::max(1, occ)), PS_THREADS,
                      bsmem, s, u, n, (const double*)p.sinmat, (const double*)p.lam, 1.0 / p.dt, p.h * p.h,
                      sc * sc * p.h * p.h, planes);
  }
  DPM_COUNT_LAUNCH(1);
  return launch_pdl(plane_small_kernel, (unsigned)((long)nfields * n), PS_THREADS, smem, s, u, n,
                    (const double*)p.sinmat, (const double*)p.lam, 1.0 / p.dt, p.h * p.h, sc * sc * p.h * p.h);
}

cudaError_t run_ztri(const DstPlan& p, double* u, int nfields, cudaStream_t s) {
  const int n = p.n;
  const long nlines = (long)nfields * n * n;
  if (nlines >= (1L << 31)) return cudaErrorInvalidValue;
  static int sms = 0;
  if (!sms) {
    int dev;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  void (*k)(double*, int, int, const double*, double, double, double) =
      n == 128 ? ztri_warp_kernel<128, 4>
               : (n > 320 ? ztri_warp_kernel<0, 17>
                  : (n > 256 ? ztri_warp_kernel<0, 10> : (n > 128 ? ztri_warp_kernel<0, 8> : ztri_warp_kernel<0, 4>)));
  int occ = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, 256, 0);
  const long blocks = (nlines + 7) / 8;
  const int grid = (int)std::min<long>(blocks, (long)sms * std::max(1, occ));
  const double sc = 2.0 / (n + 1);
  DPM_COUNT_LAUNCH(1);
  k<<<grid, 256, 0, s>>>(u, (int)nlines, n, p.lam, 1.0 / p.dt, p.h * p.h, sc * sc * p.h * p.h);
  return cudaGetLastError();
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
  e = cudaMalloc(&p.atab, sizeof(double) * NW * mt_of(n) * ks_of(n) * 32);
  if (e != cudaSuccess) return e;
  DPM_COUNT_LAUNCH(2);
  eig_kernel<<<(n + 127) / 128, 128>>>(p.lam, n, h);
  afrag_table_kernel<<<dim3(NW, mt_of(n), ks_of(n)), 32>>>(p.atab, n, tc_for(n) / 8);
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  if (n <= PSN) {   // fused small-n plane pass (DPM_PLANE_SMALL=0 disables)
    const char* envs = getenv("DPM_PLANE_SMALL");
    if (!(envs && atoi(envs) == 0)) {
      if ((e = cudaMalloc(&p.sinmat, sizeof(double) * n * n)) != cudaSuccess) return e;
      const char* envd = getenv("DPM_PLANE_SMALL_DMMA");
      const int dm = (envd && atoi(envd) == 0) ? 0 : 1;
      if ((e = cudaMemcpyToSymbol(g_ps_dmma, &dm, sizeof(int))) != cudaSuccess) return e;
      DPM_COUNT_LAUNCH(1);
      sinmat_kernel<<<(n * n + 255) / 256, 256>>>(p.sinmat, n);
      if ((e = cudaGetLastError()) != cudaSuccess) return e;
    }
  }
  if (n == 128) {
    const char* env = getenv("DPM_PFA");
    p.pfa = !(env && atoi(env) == 0);
    const char* envp = getenv("DPM_PLANE");
    p.plane = !(envp && atoi(envp) == 0);
    if (p.pfa && (e = dst128_init()) != cudaSuccess) return e;
    if (p.pfa && (e = dst128_atab(&p.atab128)) != cudaSuccess) return e;
  }
  return cudaDeviceSynchronize();
}

void dst_plan_free(DstPlan& p) {
  if (p.side) cudaStreamDestroy(p.side);
  if (p.ev_fork) cudaEventDestroy(p.ev_fork);
  if (p.ev_join) cudaEventDestroy(p.ev_join);
  p.side = nullptr;
  if (p.lam) cudaFree(p.lam);
  if (p.atab) cudaFree(p.atab);
  if (p.atab128) cudaFree(p.atab128);
  if (p.sinmat) cudaFree(p.sinmat);
  p.atab128 = nullptr;
  p.sinmat = nullptr;
  p.lam = nullptr;
  p.atab = nullptr;
}

size_t dst_scratch_bytes(int, int) { return 0; }

cudaEvent_t PassProf::next() {
  if (used == pool.size()) {
    cudaEvent_t e = nullptr;
    if (cudaEventCreate(&e) != cudaSuccess) return nullptr;
    pool.push_back(e);
  }
  return pool[used++];
}

namespace {
// run `launch` between two events recorded on `s` when pass timing is enabled
template <typename F>
cudaError_t timed(const DstPlan& p, int kind, long long points, cudaStream_t s, F&& launch) {
  if (!p.prof) return launch();
  cudaEvent_t a = p.prof->next(), b = p.prof->next();
  if (!a || !b) return cudaErrorMemoryAllocation;
  cudaError_t e = cudaEventRecord(a, s);
  if (e != cudaSuccess) return e;
  if ((e = launch()) != cudaSuccess) return e;
  p.prof->kind.push_back(kind);
  p.prof->points.push_back(points);
  return cudaEventRecord(b, s);
}
}  // namespace

namespace {
// The passes between the two x transforms of the partial-diagonalisation solver, in place on nf
// x-transformed fields: the fused plane pass at n = 128, else y DST, z tridiagonal,
// y DST.
cudaError_t middle_passes(const DstPlan& p, double* ui, int nf, double inv_dt, double scale, cudaStream_t s) {
  const int n = p.n;
  const long long pts = (long long)nf * n * n * n;
  if (n == 128 && p.pfa && p.plane) {
    const double sc2 = 2.0 / (n + 1);
    return timed(p, 1, pts, s, [&] { return plane128_pass(ui, nf, p.lam, inv_dt, p.h * p.h, sc2 * sc2 * p.h * p.h, s); });
  }
  if (n <= PSN && p.sinmat) return timed(p, 1, pts, s, [&] { return run_plane_small(p, ui, nf, s); });
  auto pass = [&](int k) { return timed(p, k, pts, s, [&] { return run_pass(p, k, ui, ui, nf, inv_dt, scale, s); }); };
  cudaError_t e;
  if ((e = pass(1)) != cudaSuccess) return e;
  if ((e = timed(p, 2, pts, s, [&] { return run_ztri(p, ui, nf, s); })) != cudaSuccess) return e;
  return pass(1);
}
}  // namespace

cudaError_t dst_solve_middle(const DstPlan& p, double* u, int64_t batch, cudaStream_t s) {
  if (p.solver != DPM_SOLVER_DST2_TRIDIAG) return cudaErrorInvalidValue;
  const int n = p.n;
  const size_t fe = (size_t)n * n * n;
  const int64_t chunk = std::max<int64_t>(1, (int64_t)(((size_t)1024 << 20) / (fe * 8)));
  const double sc = 2.0 / (n + 1);
  for (int64_t b0 = 0; b0 < batch; b0 += chunk) {
    const int nf = (int)std::min<int64_t>(chunk, batch - b0);
    cudaError_t e = middle_passes(p, u + b0 * fe, nf, 1.0 / p.dt, sc * sc * sc, s);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

cudaError_t dst_solve_batch(const DstPlan& p, const double* q, double* u, int64_t batch, double*, size_t,
                            cudaStream_t s) {
  const int n = p.n;
  const size_t field_bytes = (size_t)n * n * n * 8;
  // Chunk of fields per pass launch.  Measured (profiles/r01/chunk_sweep.txt): each pass streams at
  // ~5.3 TB/s whether or not the chunk fits the 126 MB L2, while small chunks pay a fixed ~8 us of
  // launch ramp / tail per pass, so chunks are large (1 GiB; DPM_CHUNK_MB overrides).
  static const size_t budget = [] {
    const char* v = getenv("DPM_CHUNK_MB");
    return (size_t)(v ? atoi(v) : 1024) << 20;
  }();
  int64_t chunk = std::max<int64_t>(1, (int64_t)(budget / field_bytes));
  // equal chunks (no small tail launch): ceil(batch / ceil(batch / chunk)) fields each
  static const bool balanced = [] {
    const char* v = getenv("DPM_CHUNK_BALANCED");
    return !(v && atoi(v) == 0);
  }();
  if (balanced && batch > chunk) {
    const int64_t nch = (batch + chunk - 1) / chunk;
    chunk = (batch + nch - 1) / nch;
  }
  const double inv_dt = 1.0 / p.dt;
  const double sc = 2.0 / (n + 1);
  const double scale = sc * sc * sc;
  const size_t fe = (size_t)n * n * n;
  // Optional: alternate chunks over two streams (DPM_STREAMS=2) so one chunk's launch ramp and
  // tail overlap the next chunk's passes.
  static const int nstreams = [] {
    const char* v = getenv("DPM_STREAMS");
    return v && atoi(v) == 2 ? 2 : 1;
  }();
  const cudaStream_t s0 = s;
  const bool two = nstreams == 2 && batch > chunk && !p.prof;
  if (two) {
    if (!p.side) {
      cudaStreamCreateWithFlags(&const_cast<DstPlan&>(p).side, cudaStreamNonBlocking);
      cudaEventCreateWithFlags(&const_cast<DstPlan&>(p).ev_fork, cudaEventDisableTiming);
      cudaEventCreateWithFlags(&const_cast<DstPlan&>(p).ev_join, cudaEventDisableTiming);
    }
    cudaEventRecord(p.ev_fork, s0);
    cudaStreamWaitEvent(p.side, p.ev_fork, 0);
  }
  int64_t ci = 0;
  for (int64_t b0 = 0; b0 < batch; b0 += chunk, ++ci) {
    const int nf = (int)std::min<int64_t>(chunk, batch - b0);
    const double* qi = q + b0 * fe;
    double* ui = u + b0 * fe;
    if (two) s = (ci & 1) ? p.side : s0;
    cudaError_t e;
    const long long pts = (long long)nf * (long long)fe;
    auto pass = [&](int k, const double* in) { return timed(p, k, pts, s, [&] { return run_pass(p, k, in, ui, nf, inv_dt, scale, s); }); };
    // DPM_SKIP_XPASS / DPM_SKIP_PLANE = 1: timing experiments only (tools/pks_skip.py), results wrong;
    // compiled in only with -DDPM_TIMING_SKIPS=1
#if DPM_TIMING_SKIPS
    static const bool skip_x = getenv("DPM_SKIP_XPASS") && atoi(getenv("DPM_SKIP_XPASS")) == 1;
    static const bool skip_m = getenv("DPM_SKIP_PLANE") && atoi(getenv("DPM_SKIP_PLANE")) == 1;
#else
    constexpr bool skip_x = false, skip_m = false;
#endif
    if (!skip_x && (e = pass(0, qi)) != cudaSuccess) return e;
    if (p.solver == DPM_SOLVER_DST2_TRIDIAG) {
      if (!skip_m && (e = middle_passes(p, ui, nf, inv_dt, scale, s)) != cudaSuccess) return e;
    } else {
      if ((e = pass(1, ui)) != cudaSuccess) return e;
      if ((e = pass(2, ui)) != cudaSuccess) return e;
      if ((e = pass(1, ui)) != cudaSuccess) return e;
    }
    if (!skip_x && (e = pass(0, ui)) != cudaSuccess) return e;
  }
  if (two) {
    cudaEventRecord(p.ev_join, p.side);
    cudaStreamWaitEvent(s0, p.ev_join, 0);
  }
  return cudaSuccess;
}
