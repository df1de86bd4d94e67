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

cudaError_t bepf_prepare(dpm_ctx* ctx) {
  if (ctx->bepf_btab) return cudaSuccess;
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

}  // namespace

bool bep_zbox_enabled() {
  static const bool on = [] {
    const char* v = getenv("DPM_BEP_ZBOX");
    return !(v && atoi(v) == 0);
  }();
  return on;
}

// nc boxes that are zero off the band (allocated and zeroed once per context; grown when needed)
cudaError_t bep_zbox(dpm_ctx* ctx, int nc, double** out, cudaStream_t s) {
  if (ctx->bepf_zcols < nc) {
    if (ctx->bepf_zbox) cudaFree(ctx->bepf_zbox);
    ctx->bepf_zbox = nullptr;
    ctx->bepf_zcols = 0;
    const size_t bytes = (size_t)nc * ctx->n * ctx->n * ctx->n * sizeof(double);
    cudaError_t e = cudaMalloc(&ctx->bepf_zbox, bytes);
    if (e != cudaSuccess) return e;
    if ((e = cudaMemsetAsync(ctx->bepf_zbox, 0, bytes, s)) != cudaSuccess) return e;
    ctx->bepf_zcols = nc;
  }
  *out = ctx->bepf_zbox;
  return cudaSuccess;
}

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
  // (small-K builds, e.g. the zonal Case-1 subdomains, keep the sparse-in pass: their few columns do not
  // amortise the boxes' allocation and zeroing in a fresh context)
  if (bep_zbox_enabled() && ctx->K >= 128) {
    // (1') q_c scattered into boxes that stay zero off the band: every chunk writes the same band
    // positions, so the boxes are zeroed once, when allocated; (2') dense forward x pass box -> work
    double* zb = nullptr;
    if ((e = bep_zbox(ctx, nc, &zb, s)) != cudaSuccess) return e;
    if ((e = launch_potential_scatter(ctx, ctx->E + (size_t)c0 * ng, ng, zb, nc, s)) != cudaSuccess)
      return e;
    if ((e = dst128_pass(0, zb, ctx->work, nc, ctx->plan.atab128, s)) != cudaSuccess) return e;
  } else {
  // (1) band values of q_c = χ_{M-}(I/dt - Δ_h)[E_c], x-line-major
  if ((e = launch_potential_band(ctx, ctx->E + (size_t)c0 * ng, ng, ctx->bepf_qb, nc, ctx->bepf_bpos, s)) != cudaSuccess)
    return e;
  // (2) forward x DST-I gathered from the band values into the work boxes
  if ((e = dst128_xpass_sparse(ctx->work, nc, ctx->bepf_btab, ctx->bepf_qb, nb, s)) != cudaSuccess) return e;
  }
  // (3) fused plane pass, (4) inverse x DST-I, (5) γ gather and B = E_in - Tr_γin u
  if ((e = dst_solve_middle(ctx->plan, ctx->work, nc, s)) != cudaSuccess) return e;
  if ((e = dst128_pass(0, ctx->work, ctx->work, nc, ctx->plan.atab128, s)) != cudaSuccess) return e;
  return launch_bep_gather(ctx, ctx->work, c0, nc, PgE, B, s);
}

void bep_fused_free(dpm_ctx* c) {
  bep_sym_free(c);
  void* ptrs[] = {c->bepf_btab, c->bepf_bpos, c->bepf_qb, c->bepf_zbox};
  for (void* p : ptrs)
    if (p) cudaFree(p);
}
