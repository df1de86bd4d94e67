// NEXT-1: sparse-in BEP column build for dpm_bep_columns at n = 128.
//
// A BEP column is u_c = AP(q_c) with q_c = χ_{M-}(I/dt - Δ_h)[E_c], then
// Tr_γ u_c and B[:, c] = E_in[:, c] - u_c[γ_in].  q_c is non-zero only on the band (R4).  With the
// partial-diagonalisation solver the first pass of the AP solve is a DST-I along x,
// so at n = 128:
//   * the band values of q_c are computed compactly (n_band per column, x-line-major), instead of
//     zero-filling an n³ box and scattering into it,
//   * the forward x pass (prime-factor kernel, MODE 1) gathers its tiles from them through a
//     32-byte entry per x-line (128-bit mask of the band x positions + start of its values),
//   * the fused plane pass, the inverse x pass and the γ gather run as in the dense path.
// HBM bytes per column: 5·8n³ instead of 7·8n³ (no zero fill, no dense read of the box).  Same
// arithmetic and rounding as the dense path (the identical kernels with a different tile load).
// Other n use the dense path.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <vector>

#include "dpm_internal.h"

namespace {


// x-line table of a point list (line L = p mod n², x = p / n²): tab[L] = {128-bit x mask, start},
// pos[i] = line-major position of point i (lines in order, x ascending within a line)
void line_table(const std::vector<int64_t>& pts, int n, std::vector<uint32_t>& tab, std::vector<int32_t>& pos) {
  const int64_t nn = (int64_t)n * n;
  tab.assign(nn * 8, 0u);
  std::vector<int32_t> cnt(nn, 0);
  for (int64_t p : pts) {
    const int64_t L = p % nn;
    const int x = (int)(p / nn);
    tab[L * 8 + (x >> 5)] |= 1u << (x & 31);
    ++cnt[L];
  }
  int32_t acc = 0;
  for (int64_t L = 0; L < nn; ++L) {
    tab[L * 8 + 4] = (uint32_t)acc;
    acc += cnt[L];
  }
  pos.resize(pts.size());
  for (size_t i = 0; i < pts.size(); ++i) {
    const int64_t L = pts[i] % nn;
    const int x = (int)(pts[i] / nn), w = x >> 5;
    int pre = 0;
    for (int q = 0; q < w; ++q) pre += __builtin_popcount(tab[L * 8 + q]);
    pos[i] = (int32_t)tab[L * 8 + 4] + pre + __builtin_popcount(tab[L * 8 + w] & ((1u << (x & 31)) - 1u));
  }
}

template <typename T>
cudaError_t upload(T** dst, const std::vector<T>& v) {
  cudaError_t e = cudaMalloc(dst, std::max<size_t>(1, v.size()) * sizeof(T));
  if (e != cudaSuccess) return e;
  return v.empty() ? cudaSuccess : cudaMemcpy(*dst, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice);
}

// x-line CSR of the γ points (line L = p mod n², x = p / n²; entries ordered by line then x) and the
// γ -> γ_in map, for the γ-out inverse pass
cudaError_t bepf_gamma_lines(dpm_ctx* ctx) {
  const int n = ctx->n;
  const int64_t nn = (int64_t)n * n, ng = ctx->counts[DPM_SET_GAMMA], ngin = ctx->counts[DPM_SET_GAMMA_IN];
  if (ng >= (1 << 20)) return cudaErrorInvalidValue;   // the packed entry holds 20 bits of γ position
  std::vector<int64_t> gam(ng);
  std::vector<int32_t> ginpos(ngin);
  cudaError_t e;
  if (ng && (e = cudaMemcpy(gam.data(), ctx->lists[DPM_SET_GAMMA], ng * 8, cudaMemcpyDeviceToHost)) != cudaSuccess)
    return e;
  if (ngin && (e = cudaMemcpy(ginpos.data(), ctx->gin_pos, ngin * 4, cudaMemcpyDeviceToHost)) != cudaSuccess) return e;
  std::vector<int32_t> start(nn + 1, 0), ent(ng), ginof(ng, -1);
  for (int64_t g = 0; g < ng; ++g) ++start[gam[g] % nn + 1];
  for (int64_t L = 0; L < nn; ++L) start[L + 1] += start[L];
  std::vector<int32_t> fill(start.begin(), start.end() - 1);
  for (int64_t g = 0; g < ng; ++g) {   // γ ascending by flat index = x-major: x ascends within each line
    const int64_t L = gam[g] % nn;
    const int x = (int)(gam[g] / nn);
    ent[fill[L]++] = (int32_t)((g << 11) | ((L & 15) << 7) | x);
  }
  for (int64_t i = 0; i < ngin; ++i) ginof[ginpos[i]] = (int32_t)i;
  std::vector<double> sn(258);
  for (int t = 0; t < 258; ++t) sn[t] = (double)sinl(3.141592653589793238462643383279502884L * (long double)t / 129.0L);
  if ((e = upload(&ctx->bepf_gstart, start)) != cudaSuccess) return e;
  if ((e = upload(&ctx->bepf_gent, ent)) != cudaSuccess) return e;
  if ((e = upload(&ctx->bepf_ginof, ginof)) != cudaSuccess) return e;
  return upload(&ctx->bepf_sin, sn);
}

cudaError_t bepf_prepare(dpm_ctx* ctx) {
  if (ctx->bepf_btab) return cudaSuccess;
  cudaError_t eg = bepf_gamma_lines(ctx);
  if (eg != cudaSuccess) return eg;
  const int64_t nb = ctx->counts[DPM_SET_BAND];
  std::vector<int64_t> band(nb);
  cudaError_t e;
  if (nb && (e = cudaMemcpy(band.data(), ctx->lists[DPM_SET_BAND], nb * 8, cudaMemcpyDeviceToHost)) != cudaSuccess) return e;
  std::vector<uint32_t> bt;
  std::vector<int32_t> bp;
  line_table(band, ctx->n, bt, bp);
  if ((e = upload(&ctx->bepf_btab, bt)) != cudaSuccess) return e;
  return upload(&ctx->bepf_bpos, bp);
}


// ---- sparse-in forward x pass and γ-out inverse x pass (round 2) ----------------------------------
// Both work on tiles of consecutive x-lines (a warp per tile) and use the exact DST-I sine table
// T[t] = sin(π t/129), t = (j k) mod 258, in shared memory.
constexpr int NX = 128, NXX = NX * NX, TPL = 8, SP_WARPS = 12, OUTP = NX + 1;   // staging [line][k], odd pitch
constexpr int TPLI = 8, INV_WARPS = 24;                                        // inverse: 8-line tiles

// X_k = Σ_{j in band(line)} x_j sin(π j k/129) for every line of an 8-line tile: only the band values of
// the line (compact, x-line-major, tab[L] = {128-bit x mask, start}) are read and multiplied, lane = outputs
// k = lane + 1 + 32 q (q < 4), the angle index (j k) mod 258 from per-lane shared tables (no integer
// division); a tile with no band point is written as zeros without arithmetic.  The outputs are staged in
// shared memory and stored as coalesced 128-byte row segments (same layout and scale as the dense x pass).
__global__ void __launch_bounds__(32 * SP_WARPS) bep_xfwd_sparse_kernel(double* __restrict__ out, int nfields,
                                                                       const uint32_t* __restrict__ tab,
                                                                       const double* __restrict__ vals, int64_t ldv,
                                                                       const double* __restrict__ sintab) {
  __shared__ double T[258];
  __shared__ uint16_t JK[NX + 1][32];   // (j (lane + 1)) mod 258
  __shared__ uint16_t ST[NX + 1];       // (32 j) mod 258
  extern __shared__ double spo[];       // [warp][16 lines][OUTP]
  for (int i = threadIdx.x; i < 258; i += blockDim.x) T[i] = sintab[i];
  for (int i = threadIdx.x; i < (NX + 1) * 32; i += blockDim.x) JK[i >> 5][i & 31] = (uint16_t)(((i >> 5) * ((i & 31) + 1)) % 258);
  for (int i = threadIdx.x; i <= NX; i += blockDim.x) ST[i] = (uint16_t)((32 * i) % 258);
  __syncthreads();
  const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
  double* O = spo + (size_t)wl * TPL * OUTP;
  const size_t field = (size_t)NXX * NX;
  constexpr int TPF = NXX / TPL;
  const int ntiles = nfields * TPF;
  const int gw = (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5), nw = (int)((gridDim.x * blockDim.x) >> 5);
  for (int t = gw; t < ntiles; t += nw) {
    const int f = t / TPF, c0 = (t - f * TPF) * TPL;
    double* fo = out + (size_t)f * field + c0;
    uint32_t mw[4] = {0, 0, 0, 0};
    int start = 0, m = 0;
    if (lane < TPL) {
      const uint4 a = __ldg(reinterpret_cast<const uint4*>(tab) + 2 * (size_t)(c0 + lane));
      mw[0] = a.x; mw[1] = a.y; mw[2] = a.z; mw[3] = a.w;
      start = (int)__ldg(tab + 8 * (size_t)(c0 + lane) + 4);
      m = __popc(mw[0]) + __popc(mw[1]) + __popc(mw[2]) + __popc(mw[3]);
    }
    const unsigned busy = __ballot_sync(0xffffffffu, m > 0);
    if (!busy) {   // no band point on the tile's lines: the transform is zero
      for (int r = lane >> 3; r < NX; r += 4) __stcg(fo + (size_t)r * NXX + (lane & 7), 0.0);
      continue;
    }
    const double* fv = vals + (size_t)f * ldv;
    for (int l = 0; l < TPL; ++l) {
      double acc[4] = {0.0, 0.0, 0.0, 0.0};
      if ((busy >> l) & 1u) {
        const int ml = __shfl_sync(0xffffffffu, m, l), sl = __shfl_sync(0xffffffffu, start, l);
        uint32_t w[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) w[q] = __shfl_sync(0xffffffffu, mw[q], l);
        for (int b0 = 0; b0 < ml; b0 += 32) {
          // lane i of the chunk: the (b0 + i)-th band point of the line: its value and x index (1-based)
          const int i = b0 + lane;
          int jl = 0;
          double vl = 0.0;
          if (i < ml) {
            int r = i, q = 0;
            while (r >= __popc(w[q])) r -= __popc(w[q++]);
            jl = 32 * q + (int)__fns(w[q], 0, r + 1) + 1;
            vl = __ldg(fv + sl + i);
          }
          const int cnt = min(32, ml - b0);
          for (int s = 0; s < cnt; ++s) {
            const int jj = __shfl_sync(0xffffffffu, jl, s);
            const double vv = __shfl_sync(0xffffffffu, vl, s);
            const int st = ST[jj];
            int tt = JK[jj][lane];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              acc[q] = fma(vv, T[tt], acc[q]);
              tt += st;
              tt -= tt >= 258 ? 258 : 0;
            }
          }
        }
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) O[l * OUTP + lane + 32 * q] = acc[q];
    }
    __syncwarp();
    for (int r = lane >> 3; r < NX; r += 4) __stcg(fo + (size_t)r * NXX + (lane & 7), O[(lane & 7) * OUTP + r]);
    __syncwarp();
  }
}

// γ-out inverse x pass: for the γ points of a tile's 8 lines only, u(x_k) = Σ_j v_j sin(π j k/129)
// (k = x + 1) over the line's 128 transformed values staged in shared memory; four lanes per γ point
// (32 terms each, combined by shuffles); PgE = u and B = E_in - u are written directly (replaces the
// dense inverse pass and the γ gather).  Tiles with no γ point are not read.  24 warps per SM hide the
// tile loads.
__global__ void __launch_bounds__(32 * INV_WARPS) bep_xinv_gamma_kernel(const double* __restrict__ in, int nfields,
                                                                       const int32_t* __restrict__ gstart,
                                                                       const int32_t* __restrict__ gent,
                                                                       const int32_t* __restrict__ ginof,
                                                                       const double* __restrict__ sintab,
                                                                       const double* __restrict__ E, int64_t ng,
                                                                       int64_t ngin, int c0col, double* PgE,
                                                                       double* B) {
  __shared__ double T[258];
  extern __shared__ double spi[];   // [warp][128][8]
  for (int i = threadIdx.x; i < 258; i += blockDim.x) T[i] = sintab[i];
  __syncthreads();
  const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5, sub = lane & 3;
  double* R = spi + (size_t)wl * NX * TPLI;
  const unsigned sb = (unsigned)__cvta_generic_to_shared(R);
  const size_t field = (size_t)NXX * NX;
  constexpr int TPF = NXX / TPLI;
  const int ntiles = nfields * TPF;
  const int gw = (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5), nw = (int)((gridDim.x * blockDim.x) >> 5);
  for (int t = gw; t < ntiles; t += nw) {
    const int f = t / TPF, c0 = (t - f * TPF) * TPLI;
    const int e0 = __ldg(gstart + c0), e1 = __ldg(gstart + c0 + TPLI);
    if (e0 == e1) continue;
    const double* fi = in + (size_t)f * field + c0;
    const int cc = 2 * (lane & 3);
#pragma unroll 4
    for (int r = lane >> 2; r < NX; r += 8)
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sb + 8u * (unsigned)(r * TPLI + cc)),
                   "l"(fi + (size_t)r * NXX + cc));
    asm volatile("cp.async.commit_group;\n" ::);
    asm volatile("cp.async.wait_group 0;\n" ::);
    __syncwarp();
    const int c = c0col + f;
    for (int eb = e0; eb < e1; eb += 8) {   // 8 γ points per pass, 4 lanes each
      const int e = eb + (lane >> 2);
      const bool ok = e < e1;
      int ent = ok ? __ldg(gent + e) : 0;
      const int kk = (ent & 127) + 1, l = (ent >> 7) & 7;
      // this lane's terms j = 32 sub .. 32 sub + 31 (1-based j + 1), angle index (j k) mod 258
      unsigned a = (unsigned)((32 * sub + 1) * kk);
      int tt = (int)(a - 258u * __umulhi(a, 16646912u));   // a mod 258 (a < 2^14)
      const double* Rl = R + 32 * sub * TPLI + l;
      double a0 = 0.0, a1 = 0.0;
#pragma unroll 8
      for (int j = 0; j < 32; j += 2) {
        a0 = fma(Rl[j * TPLI], T[tt], a0);
        tt += kk;
        tt -= tt >= 258 ? 258 : 0;
        a1 = fma(Rl[(j + 1) * TPLI], T[tt], a1);
        tt += kk;
        tt -= tt >= 258 ? 258 : 0;
      }
      double u = a0 + a1;
      u += __shfl_xor_sync(0xffffffffu, u, 1);
      u += __shfl_xor_sync(0xffffffffu, u, 2);
      if (ok && sub == 0) {
        const int g = ent >> 11;
        if (PgE) PgE[(size_t)f * ng + g] = u;
        const int gi = __ldg(ginof + g);
        if (B && gi >= 0) B[(size_t)f * ngin + gi] = __ldg(E + (size_t)c * ng + g) - u;
      }
    }
    __syncwarp();
  }
}

int sms_count() {
  static int sms = 0;
  if (!sms) {
    int dev;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  return sms;
}

}  // namespace

bool bep_fused_enabled(const dpm_ctx* ctx) {
  static const bool on = [] {
    const char* v = getenv("DPM_BEP_FUSED");
    return !(v && atoi(v) == 0);
  }();
  const DstPlan& p = ctx->plan;
  return on && p.solver == DPM_SOLVER_DST2_TRIDIAG && p.n == 128 && p.pfa && p.plane;
}

// columns [c0, c0 + nc) of the BEP (nc <= the work boxes of ctx): PgE (|γ| x nc, may be null) and
// B (|γ_in| x nc, may be null), both column-major.
cudaError_t bep_columns_fused(dpm_ctx* ctx, int c0, int nc, double* PgE, double* B, cudaStream_t s) {
  cudaError_t e = bepf_prepare(ctx);
  if (e != cudaSuccess) return e;
  const int64_t nb = ctx->counts[DPM_SET_BAND], ng = ctx->counts[DPM_SET_GAMMA];
  if (ctx->bepf_cols < nc) {
    if (ctx->bepf_qb) cudaFree(ctx->bepf_qb);
    ctx->bepf_qb = nullptr;
    ctx->bepf_cols = 0;
    if ((e = cudaMalloc(&ctx->bepf_qb, std::max<int64_t>(1, nb) * nc * sizeof(double))) != cudaSuccess) return e;
    ctx->bepf_cols = nc;
  }
  // (1) band values of q_c = χ_{M-}(I/dt - Δ_h)[E_c], x-line-major
  if ((e = launch_potential_band(ctx, ctx->E + (size_t)c0 * ng, ng, ctx->bepf_qb, nc, ctx->bepf_bpos, s)) != cudaSuccess)
    return e;
  static const bool sparse2 = [] {   // DPM_BEP_SPARSE2=0: the PFA x passes + dense inverse + γ gather
    const char* v = getenv("DPM_BEP_SPARSE2");
    return !(v && atoi(v) == 0);
  }();
  if (!sparse2) {
    // (2) forward x DST-I gathered from the band values into the work boxes
    if ((e = dst128_xpass_sparse(ctx->work, nc, ctx->bepf_btab, ctx->bepf_qb, nb, s)) != cudaSuccess) return e;
    // (3) fused plane pass, (4) inverse x DST-I, (5) γ gather and B = E_in - Tr_γin u
    if ((e = dst_solve_middle(ctx->plan, ctx->work, nc, s)) != cudaSuccess) return e;
    if ((e = dst128_pass(0, ctx->work, ctx->work, nc, ctx->plan.atab128, s)) != cudaSuccess) return e;
    return launch_bep_gather(ctx, ctx->work, c0, nc, PgE, B, s);
  }
  // (2) forward x DST-I of the band values only (sparse sine sums; empty tiles written as zeros)
  const size_t smem_f = (size_t)SP_WARPS * TPL * OUTP * sizeof(double);
  if ((e = cudaFuncSetAttribute(bep_xfwd_sparse_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_f)) !=
      cudaSuccess)
    return e;
  const int grid = sms_count() * 2;
  DPM_COUNT_LAUNCH(1);
  bep_xfwd_sparse_kernel<<<grid, 32 * SP_WARPS, smem_f, s>>>(ctx->work, nc, ctx->bepf_btab, ctx->bepf_qb, nb,
                                                               ctx->bepf_sin);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  // (3) fused plane pass
  if ((e = dst_solve_middle(ctx->plan, ctx->work, nc, s)) != cudaSuccess) return e;
  // (4) inverse x DST-I at the γ points only, writing PgE and B = E_in - Tr_γin u directly
  const size_t smem_i = (size_t)INV_WARPS * NX * TPLI * sizeof(double);
  if ((e = cudaFuncSetAttribute(bep_xinv_gamma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_i)) !=
      cudaSuccess)
    return e;
  DPM_COUNT_LAUNCH(1);
  bep_xinv_gamma_kernel<<<sms_count(), 32 * INV_WARPS, smem_i, s>>>(ctx->work, nc, ctx->bepf_gstart, ctx->bepf_gent,
                                                              ctx->bepf_ginof, ctx->bepf_sin, ctx->E, ng,
                                                              ctx->counts[DPM_SET_GAMMA_IN], c0, PgE, B);
  return cudaGetLastError();
}

void bep_fused_free(dpm_ctx* c) {
  void* ptrs[] = {c->bepf_btab, c->bepf_bpos, c->bepf_qb, c->bepf_gstart, c->bepf_gent, c->bepf_ginof, c->bepf_sin};
  for (void* p : ptrs)
    if (p) cudaFree(p);
}
