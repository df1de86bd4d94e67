// extern "C" entry points of libdpm.so (declared and documented in include/dpm.h).
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <new>

#include "dpm_internal.h"

std::atomic<long long> g_dpm_launches{0};

thread_local int g_pdl_scope = 0;

bool pdl_enabled() {
  static const int mode = [] {
    const char* v = getenv("DPM_PDL");
    return v ? atoi(v) : 1;
  }();
  return mode == 2 || (mode == 1 && g_pdl_scope > 0);
}

namespace {

thread_local std::string g_create_err;

void free_ctx(dpm_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  void* ptrs[] = {c->flags, c->gmap, c->gin_pos, c->mplus_slope, c->foot, c->dist, c->E, c->B, c->Q, c->R, c->colscale, c->Mlsq, c->RDinv,
                  c->dd_Eraw, c->dd_assign, c->dd_rows, c->dd_B, c->dd_Q, c->dd_R, c->dd_M, c->dd_D, c->dd_g, c->dd_ug,
                  c->dd_sign, c->dd_shared,
                  c->lsq_ws, c->work, c->scratch, c->red};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  for (auto* l : c->lists)
    if (l) cudaFree(l);
  if (c->red_host) cudaFreeHost(c->red_host);
  bep_fused_free(c);
  dst_plan_free(c->plan);
  if (c->setup_stream) cudaStreamDestroy(c->setup_stream);
  if (c->h2d_stream) cudaStreamDestroy(c->h2d_stream);
  if (c->d2h_stream) cudaStreamDestroy(c->d2h_stream);
  for (cudaEvent_t e : c->pipe_ev)
    if (e) cudaEventDestroy(e);
  for (cudaEvent_t e : c->prof.pool) cudaEventDestroy(e);
  for (auto& g : c->pks_graphs)
    if (g.exec) cudaGraphExecDestroy(g.exec);
  if (c->graph_stream) cudaStreamDestroy(c->graph_stream);
  if (c->fac_exec) cudaGraphExecDestroy(c->fac_exec);
  if (c->fac_stream) cudaStreamDestroy(c->fac_stream);
  if (c->pks_log) cudaFree(c->pks_log);
  if (c->pks_log_host) cudaFreeHost(c->pks_log_host);
  if (c->pks_backup) cudaFree(c->pks_backup);
  if (c->side_stream) cudaStreamDestroy(c->side_stream);
  for (cudaEvent_t e : c->ev_side)
    if (e) cudaEventDestroy(e);
  delete c;
}

dpm_status ensure_work(dpm_ctx* ctx, size_t boxes) {
  if (ctx->work_boxes >= boxes) return DPM_OK;
  if (ctx->work) cudaFree(ctx->work);
  ctx->work = nullptr;
  ctx->work_boxes = 0;
  const size_t field = (size_t)ctx->n * ctx->n * ctx->n;
  if (cudaMalloc(&ctx->work, boxes * field * sizeof(double)) != cudaSuccess) {
    cudaGetLastError();
    ctx->err = "out of device memory for work boxes";
    return DPM_ERR_OOM;
  }
  ctx->work_boxes = boxes;
  return DPM_OK;
}

// columns processed per BEP chunk (bounded device memory: <= ~2 GB of boxes)
int bep_chunk(const dpm_ctx* ctx) {
  const size_t field = (size_t)ctx->n * ctx->n * ctx->n * sizeof(double);
  return (int)std::max<size_t>(1, std::min<size_t>((size_t)ctx->K, ((size_t)2 << 30) / field));
}

cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

}  // namespace

dpm_status dpm_create_impl(const dpm_grid* grid, const dpm_domain* domain, int32_t lmax, double dt, int32_t basis,
                           int32_t device, dpm_ctx** out) {
  DPM_NVTX();
  if (out) *out = nullptr;
  g_create_err.clear();
  if (!grid || !domain || !out) { g_create_err = "null argument"; return DPM_ERR_INVALID; }
  if (grid->n < 4 || grid->n > DPM_MAX_N) { g_create_err = "n out of range [4, DPM_MAX_N]"; return DPM_ERR_INVALID; }
  if (!(grid->lo < grid->hi)) { g_create_err = "lo >= hi"; return DPM_ERR_INVALID; }
  if (!(dt > 0) || !std::isfinite(dt)) { g_create_err = "dt must be > 0"; return DPM_ERR_INVALID; }
  if (basis < DPM_BASIS_CAUCHY || basis > DPM_BASIS_NEUMANN0_2TERM_ZONAL) { g_create_err = "bad basis"; return DPM_ERR_INVALID; }
  const bool zonal = basis_zonal(basis);
  if (lmax < 0 || lmax > (zonal ? DPM_MAX_ZONAL_L : 40)) { g_create_err = "lmax out of range"; return DPM_ERR_INVALID; }
  if (cudaSetDevice(device) != cudaSuccess) { g_create_err = "cudaSetDevice failed"; return DPM_ERR_CUDA; }
  {   // the stream-ordered workspaces (lsq_gram's split-K slices) keep their memory in the device's
      // default pool between calls instead of returning it to the driver at every synchronisation
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
      uint64_t thr = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
  }
  dpm_ctx* ctx = new (std::nothrow) dpm_ctx();
  if (!ctx) return DPM_ERR_OOM;
  ctx->device = device;
  ctx->n = grid->n;
  ctx->lo = grid->lo;
  ctx->hi = grid->hi;
  ctx->h = (grid->hi - grid->lo) / (grid->n + 1);
  ctx->dt = dt;
  ctx->domain = *domain;
  if (domain->kind == DPM_SPHERE) ctx->domain.semi[1] = ctx->domain.semi[2] = domain->semi[0];
  ctx->lmax = lmax;
  ctx->basis = basis;
  ctx->K = basis_ncomp(basis) * (zonal ? lmax + 1 : (lmax + 1) * (lmax + 1));
  dpm_status st = DPM_OK;
  if (cudaStreamCreateWithFlags(&ctx->setup_stream, cudaStreamNonBlocking) != cudaSuccess) st = DPM_ERR_CUDA;
  if (st == DPM_OK) st = setup_point_sets(ctx);
  if (st == DPM_OK && domain->kind < DPM_OCTANT_CANON) st = setup_geometry(ctx);   // DD subdomains: their own
  if (st == DPM_OK && dst_plan_init(ctx->plan, ctx->n, ctx->h, dt) != cudaSuccess) { st = DPM_ERR_CUDA; ctx->err = "plan init"; }
  if (st == DPM_OK && cudaMalloc(&ctx->red, 64 * sizeof(double)) != cudaSuccess) st = DPM_ERR_OOM;
  if (st == DPM_OK && cudaMemset(ctx->red, 0, 64 * sizeof(double)) != cudaSuccess) st = DPM_ERR_CUDA;   // [63]: ticket
  if (st == DPM_OK && cudaMallocHost(&ctx->red_host, 64 * sizeof(double)) != cudaSuccess) st = DPM_ERR_OOM;
  if (st != DPM_OK) {
    g_create_err = ctx->err.empty() ? "dpm_create failed" : ctx->err;
    free_ctx(ctx);
    return st;
  }
  *out = ctx;
  return DPM_OK;
}

extern "C" {

const char* dpm_last_error(const dpm_ctx* ctx) { return ctx ? ctx->err.c_str() : g_create_err.c_str(); }

dpm_status dpm_create(const dpm_grid* grid, const dpm_domain* domain, int32_t lmax, double dt, int32_t basis,
                      int32_t device, dpm_ctx** out) {
  DPM_NVTX();
  if (out) *out = nullptr;
  g_create_err.clear();
  if (!grid || !domain || !out) { g_create_err = "null argument"; return DPM_ERR_INVALID; }
  if (domain->kind != DPM_SPHERE && domain->kind != DPM_ELLIPSOID) { g_create_err = "bad domain kind"; return DPM_ERR_INVALID; }
  for (int a = 0; a < 3; ++a) {
    const double s = domain->kind == DPM_SPHERE ? domain->semi[0] : domain->semi[a];
    if (!(s > 0)) { g_create_err = "semi-axes must be > 0"; return DPM_ERR_INVALID; }
    if (!(domain->center[a] - s > grid->lo && domain->center[a] + s < grid->hi)) {
      g_create_err = "domain not strictly inside the box";
      return DPM_ERR_INVALID;
    }
  }
  return dpm_create_impl(grid, domain, lmax, dt, basis, device, out);
}

void dpm_destroy(dpm_ctx* ctx) {
  DPM_NVTX(); free_ctx(ctx); }

dpm_status dpm_query(const dpm_ctx* ctx, dpm_info* out) {
  DPM_NVTX();
  if (!ctx || !out) return DPM_ERR_INVALID;
  std::memset(out, 0, sizeof(*out));
  out->n = ctx->n;
  out->K = ctx->K;
  out->lmax = ctx->lmax;
  out->basis = ctx->basis;
  out->h = ctx->h;
  out->dt = ctx->dt;
  out->n_mplus = ctx->counts[DPM_SET_MPLUS];
  out->n_gamma = ctx->counts[DPM_SET_GAMMA];
  out->n_gamma_in = ctx->counts[DPM_SET_GAMMA_IN];
  out->n_gamma_ex = ctx->counts[DPM_SET_GAMMA_EX];
  out->n_band = ctx->counts[DPM_SET_BAND];
  out->n_nplus = ctx->counts[DPM_SET_NPLUS];
  out->ghosts_in_nplus = ctx->ghosts_in_nplus;
  out->have_projection = ctx->have_projection;
  out->bep_cond_est = ctx->bep_cond;
  out->solver = ctx->plan.solver;
  out->n_exact_ties = ctx->exact_ties;
  out->n_exact_ties_inside = ctx->exact_ties_inside;
  return DPM_OK;
}

dpm_status dpm_set_solver(dpm_ctx* ctx, int32_t solver) {
  DPM_NVTX();
  if (!ctx || (solver != DPM_SOLVER_DST3 && solver != DPM_SOLVER_DST2_TRIDIAG)) return DPM_ERR_INVALID;
  ctx->plan.solver = solver;
  return DPM_OK;
}

dpm_status dpm_copy_set(const dpm_ctx* ctx, int32_t which, int64_t* host_idx, int64_t cap) {
  DPM_NVTX();
  if (!ctx || !host_idx || which < 0 || which > 5) return DPM_ERR_INVALID;
  dpm_ctx* c = const_cast<dpm_ctx*>(ctx);
  if (cap < ctx->counts[which]) { c->err = "capacity too small"; return DPM_ERR_INVALID; }
  cudaSetDevice(ctx->device);
  DPM_CUDA_TRY(c, cudaMemcpy(host_idx, ctx->lists[which], ctx->counts[which] * sizeof(int64_t), cudaMemcpyDeviceToHost));
  return DPM_OK;
}

dpm_status dpm_copy_extension(const dpm_ctx* ctx, double* host_E, double* host_d) {
  DPM_NVTX();
  if (!ctx) return DPM_ERR_INVALID;
  dpm_ctx* c = const_cast<dpm_ctx*>(ctx);
  cudaSetDevice(ctx->device);
  const int64_t ng = ctx->counts[DPM_SET_GAMMA];
  if (host_E) DPM_CUDA_TRY(c, cudaMemcpy(host_E, ctx->E, (size_t)ng * ctx->K * sizeof(double), cudaMemcpyDeviceToHost));
  if (host_d) DPM_CUDA_TRY(c, cudaMemcpy(host_d, ctx->dist, (size_t)ng * sizeof(double), cudaMemcpyDeviceToHost));
  return DPM_OK;
}

dpm_status dpm_set_dt(dpm_ctx* ctx, double dt) {
  DPM_NVTX();
  if (!ctx || !(dt > 0) || !std::isfinite(dt)) return DPM_ERR_INVALID;
  if (dt != ctx->dt) {
    ctx->dt = dt;
    ctx->plan.dt = dt;
    ctx->have_projection = 0;
  }
  return DPM_OK;
}

dpm_status dpm_aux_solve_batch(dpm_ctx* ctx, const double* q, double* u, int64_t batch, void* stream) {
  DPM_NVTX();
  if (!ctx || batch < 0 || (batch > 0 && (!q || !u))) return DPM_ERR_INVALID;
  if (batch == 0) return DPM_OK;
  cudaSetDevice(ctx->device);
  DPM_CUDA_TRY(ctx, ctx_solve(ctx, q, u, batch, as_stream(stream)));
  return DPM_OK;
}

dpm_status dpm_aux_solve_batch_host(dpm_ctx* ctx, const double* host_q, double* host_u, int64_t batch, void* stream) {
  DPM_NVTX();
  if (!ctx || batch < 0 || (batch > 0 && (!host_q || !host_u))) return DPM_ERR_INVALID;
  if (batch == 0) return DPM_OK;
  cudaSetDevice(ctx->device);
  cudaStream_t s = as_stream(stream);
  const size_t field = (size_t)ctx->n * ctx->n * ctx->n;
  // Three-stage pipeline over chunks of <= 128 MB: H2D (copy-in stream) -> solve (caller's stream)
  // -> D2H (copy-out stream) over a ring of NBUF device buffers, so that chunk i+1 uploads and chunk
  // i-1 downloads while chunk i is solved (PCIe is full duplex; pinned host buffers give async
  // copies).  Three buffers: with two, the upload of chunk i+1 waited for the download of chunk i-1
  // (same buffer) and the two directions serialized at every buffer switch.
  constexpr int NBUF = 3;
  const int64_t chunk = std::max<int64_t>(1, std::min<int64_t>(batch, (int64_t)(((size_t)128 << 20) / (field * 8))));
  dpm_status st = ensure_work(ctx, NBUF * chunk);
  if (st != DPM_OK) return st;
  if (!ctx->h2d_stream) {
    DPM_CUDA_TRY(ctx, cudaStreamCreateWithFlags(&ctx->h2d_stream, cudaStreamNonBlocking));
    DPM_CUDA_TRY(ctx, cudaStreamCreateWithFlags(&ctx->d2h_stream, cudaStreamNonBlocking));
    for (int i = 0; i < 3 * NBUF; ++i) DPM_CUDA_TRY(ctx, cudaEventCreateWithFlags(&ctx->pipe_ev[i], cudaEventDisableTiming));
  }
  cudaEvent_t* up = ctx->pipe_ev;              // up[b]: upload into buffer b done
  cudaEvent_t* solved = ctx->pipe_ev + NBUF;
  cudaEvent_t* down = ctx->pipe_ev + 2 * NBUF; // down[b]: download from buffer b done (buffer free)
  for (int b = 0; b < NBUF; ++b) DPM_CUDA_TRY(ctx, cudaEventRecord(down[b], s));
  for (int64_t b0 = 0, it = 0; b0 < batch; b0 += chunk, ++it) {
    const int64_t nb = std::min<int64_t>(chunk, batch - b0);
    const int bi = (int)(it % NBUF);
    double* buf = ctx->work + (size_t)bi * chunk * field;
    DPM_CUDA_TRY(ctx, cudaStreamWaitEvent(ctx->h2d_stream, down[bi], 0));
    DPM_CUDA_TRY(ctx, cudaMemcpyAsync(buf, host_q + b0 * field, nb * field * 8, cudaMemcpyHostToDevice, ctx->h2d_stream));
    DPM_CUDA_TRY(ctx, cudaEventRecord(up[bi], ctx->h2d_stream));
    DPM_CUDA_TRY(ctx, cudaStreamWaitEvent(s, up[bi], 0));
    DPM_CUDA_TRY(ctx, ctx_solve(ctx, buf, buf, nb, s));
    DPM_CUDA_TRY(ctx, cudaEventRecord(solved[bi], s));
    DPM_CUDA_TRY(ctx, cudaStreamWaitEvent(ctx->d2h_stream, solved[bi], 0));
    DPM_CUDA_TRY(ctx, cudaMemcpyAsync(host_u + b0 * field, buf, nb * field * 8, cudaMemcpyDeviceToHost, ctx->d2h_stream));
    DPM_CUDA_TRY(ctx, cudaEventRecord(down[bi], ctx->d2h_stream));
  }
  DPM_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->d2h_stream));
  DPM_CUDA_TRY(ctx, cudaStreamSynchronize(s));
  return DPM_OK;
}

dpm_status dpm_potential_rhs(dpm_ctx* ctx, const double* v_gamma, double* q, int32_t nrhs, void* stream) {
  DPM_NVTX();
  if (!ctx || nrhs < 0 || (nrhs > 0 && (!v_gamma || !q))) return DPM_ERR_INVALID;
  if (nrhs == 0) return DPM_OK;
  cudaSetDevice(ctx->device);
  DPM_CUDA_TRY(ctx, launch_potential_rhs(ctx, v_gamma, ctx->counts[DPM_SET_GAMMA], q, nrhs, as_stream(stream)));
  return DPM_OK;
}

dpm_status dpm_trace(dpm_ctx* ctx, const double* u, double* out, int32_t which, int64_t batch, void* stream) {
  DPM_NVTX();
  if (!ctx || (which != DPM_SET_GAMMA && which != DPM_SET_GAMMA_IN) || batch < 0) return DPM_ERR_INVALID;
  if (batch == 0) return DPM_OK;
  if (!u || !out) return DPM_ERR_INVALID;
  cudaSetDevice(ctx->device);
  DPM_CUDA_TRY(ctx, launch_trace(ctx, u, out, which, batch, as_stream(stream)));
  return DPM_OK;
}

dpm_status dpm_bep_columns(dpm_ctx* ctx, int32_t c0, int32_t c1, double* PgE, double* B, void* stream) {
  DPM_NVTX();
  if (!ctx || c0 < 0 || c1 > ctx->K || c0 > c1) return DPM_ERR_INVALID;
  if (c0 == c1) return DPM_OK;
  cudaSetDevice(ctx->device);
  cudaStream_t s = as_stream(stream);
  const int ch = bep_chunk(ctx);
  dpm_status st = ensure_work(ctx, std::min(ch, c1 - c0));
  if (st != DPM_OK) return st;
  const int64_t ng = ctx->counts[DPM_SET_GAMMA], ngin = ctx->counts[DPM_SET_GAMMA_IN];
  {   // reflection-symmetric geometry with parity-definite columns: solved on the octant (bep_sym.cu)
    bool done = false;
    DPM_CUDA_TRY(ctx, bep_sym_columns(ctx, c0, c1, PgE, B, s, &done));
    if (done) return DPM_OK;
  }
  const bool fused = bep_fused_enabled(ctx);
  for (int a = c0; a < c1; a += ch) {
    const int nc = std::min(ch, c1 - a);
    if (fused) {   // sparse-in / γ-out (bep_fused.cu)
      DPM_CUDA_TRY(ctx, bep_columns_fused(ctx, a, nc, PgE ? PgE + (size_t)(a - c0) * ng : nullptr,
                                          B ? B + (size_t)(a - c0) * ngin : nullptr, s));
      continue;
    }
    // zero boxes (as in the fused n = 128 path): every chunk writes the same band positions, so boxes
    // zeroed once take the potential RHS by a band scatter and the solve reads them out of place
    // (DPM_BEP_ZBOX=0: zero-fill + scatter into the work boxes, solved in place)
    if (bep_zbox_enabled() && ctx->K >= 128 && ctx->plan.solver == DPM_SOLVER_DST2_TRIDIAG) {
      double* zb = nullptr;
      DPM_CUDA_TRY(ctx, bep_zbox(ctx, nc, &zb, s));
      DPM_CUDA_TRY(ctx, launch_potential_scatter(ctx, ctx->E + (size_t)a * ng, ng, zb, nc, s));
      DPM_CUDA_TRY(ctx, ctx_solve(ctx, zb, ctx->work, nc, s));
    } else {
      DPM_CUDA_TRY(ctx, launch_potential_rhs(ctx, ctx->E + (size_t)a * ng, ng, ctx->work, nc, s));
      DPM_CUDA_TRY(ctx, ctx_solve(ctx, ctx->work, ctx->work, nc, s));
    }
    DPM_CUDA_TRY(ctx, launch_bep_gather(ctx, ctx->work, a, nc, PgE ? PgE + (size_t)(a - c0) * ng : nullptr,
                                        B ? B + (size_t)(a - c0) * ngin : nullptr, s));
  }
  return DPM_OK;
}

dpm_status dpm_bep_factor(dpm_ctx* ctx, const double* B, void* stream) {
  DPM_NVTX();
  if (!ctx || !B) return DPM_ERR_INVALID;
  cudaSetDevice(ctx->device);
  dpm_status st = lsq_factor(ctx, B, as_stream(stream));
  if (st == DPM_OK) {
    ctx->have_projection = 1;
    ctx->dt_bep = ctx->dt;
  }
  return st;
}

dpm_status dpm_build_projection(dpm_ctx* ctx, double* PgE, double* B, void* stream) {
  DPM_NVTX();
  if (!ctx) return DPM_ERR_INVALID;
  cudaSetDevice(ctx->device);
  const int64_t ngin = ctx->counts[DPM_SET_GAMMA_IN];
  if (ctx->K >= ngin) { ctx->err = "K >= |gamma_in|"; return DPM_ERR_RANK; }
  if (!ctx->B) DPM_CUDA_TRY(ctx, cudaMalloc(&ctx->B, (size_t)ngin * ctx->K * sizeof(double)));
  dpm_status st = dpm_bep_columns(ctx, 0, ctx->K, PgE, ctx->B, stream);
  if (st != DPM_OK) return st;
  if (B) DPM_CUDA_TRY(ctx, cudaMemcpyAsync(B, ctx->B, (size_t)ngin * ctx->K * sizeof(double), cudaMemcpyDeviceToDevice,
                                           as_stream(stream)));
  return dpm_bep_factor(ctx, ctx->B, stream);
}

dpm_status dpm_boundary_lsq(dpm_ctx* ctx, const double* g, double* coef, double* u_gamma, int32_t nrhs, void* stream) {
  DPM_NVTX();
  if (!ctx || nrhs < 1 || nrhs > 2048 || !g || !coef) return DPM_ERR_INVALID;
  if (!ctx->have_projection || ctx->dt_bep != ctx->dt) { ctx->err = "no projection at the current dt"; return DPM_ERR_STATE; }
  cudaSetDevice(ctx->device);
  DPM_CUDA_TRY(ctx, lsq_apply(ctx, g, coef, u_gamma, nrhs, 0, as_stream(stream)));
  return DPM_OK;
}

dpm_status dpm_pks_init(dpm_ctx* ctx, double* rho, double* c, const dpm_pks_ic* ic, void* stream) {
  DPM_NVTX();
  if (!ctx || !rho || !c || !ic) return DPM_ERR_INVALID;
  cudaSetDevice(ctx->device);
  DPM_CUDA_TRY(ctx, launch_pks_init(ctx, rho, c, ic, as_stream(stream)));
  ctx->t = 0.0;
  ctx->dt_prev = INFINITY;
  ctx->pks_initialized = 1;
  return DPM_OK;
}

dpm_status dpm_pks_diagnostics(dpm_ctx* ctx, const double* rho, const double* c, double* out, void* stream) {
  DPM_NVTX();
  if (!ctx || !rho || !c || !out) return DPM_ERR_INVALID;
  if (ctx->dd) { ctx->err = "diagnostics: single-domain contexts only"; return DPM_ERR_INVALID; }
  cudaSetDevice(ctx->device);
  cudaStream_t s = as_stream(stream);
  DPM_CUDA_TRY(ctx, launch_diagnostics(ctx, rho, c, ctx->red + 16, s));
  DPM_CUDA_TRY(ctx, cudaMemcpyAsync(ctx->red_host + 16, ctx->red + 16, 3 * sizeof(double), cudaMemcpyDeviceToHost, s));
  DPM_CUDA_TRY(ctx, cudaStreamSynchronize(s));
  const double h3 = ctx->h * ctx->h * ctx->h;
  for (int i = 0; i < 3; ++i) out[i] = ctx->red_host[16 + i] * h3;
  return DPM_OK;
}

}  // extern "C"

double mass_fixed_decode(const double* stats) {
  unsigned long long lo, hi;
  std::memcpy(&lo, stats, 8);
  std::memcpy(&hi, stats + 8, 8);
  return (double)(long long)hi + (double)lo * 5.42101086242752217004e-20;   // 2^-64
}

double decode_key(double slot) {
  unsigned long long k;
  std::memcpy(&k, &slot, 8);
  unsigned long long x = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
  double v;
  std::memcpy(&v, &x, 8);
  return v;
}

extern "C" {


// Speculative step graphs without rollback copies (DPM_PKS_ABORT, default): the flux kernel's dt rule sets a
// device flag when a step asks for a smaller dt, a restriction that sees a non-finite value sets it too,
// and every later restriction of the graph then leaves (rho, c) alone — so the state after the graph is
// already the state at the start of the first rejected step (or right after the failing one), and no
// per-step copy of the state is written.  DPM_PKS_ABORT=0: the per-step rollback copies.
static bool pks_abort_on() {
  static const bool on = [] {
    const char* v = getenv("DPM_PKS_ABORT");
    return !(v && atoi(v) == 0);
  }();
  return on;
}
static int* pks_abort_flag(dpm_ctx* ctx) { return reinterpret_cast<int*>(ctx->red + 61); }

// Enqueue one PKS step (Steps 4a-7) at a fixed dt on stream s; `slot` receives red(3), dt_true
// (device dt rule from the state at the start of the step) and the step statistics.
static dpm_status enqueue_pks_step(dpm_ctx* ctx, double* rho, double* c, const dpm_pks_params* prm, double dt,
                                   double* slot, double* backup, cudaStream_t s, int* abort) {
  const size_t field = (size_t)ctx->n * ctx->n * ctx->n;
  const int64_t ng = ctx->counts[DPM_SET_GAMMA], ngin = ctx->counts[DPM_SET_GAMMA_IN];
  double* fq = ctx->scratch;              // 2 boxes: f/dt on M+
  double* wk = fq + 2 * field;            // 2 boxes: solves
  double* gvec = wk + 2 * field;          // |gamma_in| x 2
  double* ug = gvec + 2 * ngin;           // |gamma| x 2
  double* coef = ug + 2 * ng;             // K x 2
  // Step 3 on the device (did the speculative dt stay valid? slot[3] <- the rule's dt, from the CFL
  // maxima accumulated in slot[0..2]) and Step 4a (flux + IMEX right-hand sides) in one kernel; it also
  // writes the step's rollback copy of rho, c into `backup` when non-null and zeroes the statistics slot
  DPM_CUDA_TRY(ctx, launch_flux_rhs(ctx, rho, c, dt, prm->chi, fq, fq + field, s, backup, slot + 4,
                                    prm->dt_rule == 0 ? slot : nullptr, dt, prm->dt_cap, slot + 3, abort));
  if (prm->coupling == 1) {   // sequential: the whole ρ step, then the c step from ρ̄^{i+1}
    const int K = ctx->K;
    for (int r = 0; r < 2; ++r) {
      double* fr = fq + r * field;
      double* wr = wk + r * field;
      if (r == 1) DPM_CUDA_TRY(ctx, launch_fc_seq(ctx, c, wk, dt, fr, s));
      DPM_CUDA_TRY(ctx, ctx_solve(ctx, fr, wr, 1, s));
      DPM_CUDA_TRY(ctx, launch_trace(ctx, wr, gvec + r * ngin, DPM_SET_GAMMA_IN, 1, s));
      DPM_CUDA_TRY(ctx, lsq_apply(ctx, gvec + r * ngin, coef + (size_t)r * K, ug + r * ng, 1, prm->clamp, s));
      DPM_CUDA_TRY(ctx, launch_green_rhs(ctx, fr, ug + r * ng, wr, 1, s));
      DPM_CUDA_TRY(ctx, ctx_solve(ctx, wr, wr, 1, s));
    }
    DPM_CUDA_TRY(ctx, launch_restrict_stats(ctx, wk, rho, c, slot + 4, s, true, abort));
    return DPM_OK;
  }
  // DPM_STEP_SKIP (timing experiments only, tools/pks_skip.py, results wrong; compiled in only with
  // -DDPM_TIMING_SKIPS=1): bit 0 the particular solve, 1 the Green solve, 2 trace + least squares +
  // extension, 3 the Green RHS, 4 the restriction
#if DPM_TIMING_SKIPS
  static const int skip = [] {
    const char* v = getenv("DPM_STEP_SKIP");
    return v ? atoi(v) : 0;
  }();
#else
  constexpr int skip = 0;
#endif
  if (!(skip & 1)) DPM_CUDA_TRY(ctx, ctx_solve(ctx, fq, wk, 2, s));
  // Step 5: BEP right-hand side on gamma_in, least squares, extension, clamp (its magnitude -> slot[10])
  if (!(skip & 4)) {
  DPM_CUDA_TRY(ctx, launch_trace(ctx, wk, gvec, DPM_SET_GAMMA_IN, 2, s));
  DPM_CUDA_TRY(ctx, lsq_apply(ctx, gvec, coef, ug, 2, prm->clamp, s, slot + 10));
  }
  // the step's BEP least-squares residual ||B C - g|| / ||g|| -> slot[11], on a forked branch
  // of the graph (off the critical path), joined before the step ends (gvec / coef are reused)
  static const bool resid_on = [] {   // DPM_STEP_RESID=0: no residual (lsq_resid logged as NaN)
    const char* v = getenv("DPM_STEP_RESID");
    return !(v && atoi(v) == 0);
  }();
  const bool fork = resid_on && ctx->side_stream != nullptr;
  if (!fork) {
    const double nan = NAN;
    DPM_CUDA_TRY(ctx, cudaMemcpyAsync(slot + 11, &nan, sizeof(double), cudaMemcpyHostToDevice, s));
  }
  if (fork) {
    DPM_CUDA_TRY(ctx, cudaEventRecord(ctx->ev_side[0], s));
    DPM_CUDA_TRY(ctx, cudaStreamWaitEvent(ctx->side_stream, ctx->ev_side[0], 0));
    DPM_CUDA_TRY(ctx, lsq_residual(ctx, coef, gvec, 2, coef + 2 * ctx->K, slot + 11, ctx->side_stream));
    DPM_CUDA_TRY(ctx, cudaEventRecord(ctx->ev_side[1], ctx->side_stream));
  }
  // Steps 6-7: Green's formula as one solve of the combined RHS (R20), restricted to N+
  // (default: the band values written in place into fq, which is zero there, and the solve reads fq;
  // DPM_GREEN_INPLACE=0: a separate q box written by a streaming pass)
  static const bool inplace = [] {
    const char* v = getenv("DPM_GREEN_INPLACE");
    return !(v && atoi(v) == 0);
  }();
  if (inplace) {
    if (!(skip & 8)) DPM_CUDA_TRY(ctx, launch_green_band_inplace(ctx, fq, ug, 2, s));
    if (!(skip & 2)) DPM_CUDA_TRY(ctx, ctx_solve(ctx, fq, wk, 2, s));
  } else {
    if (!(skip & 8)) DPM_CUDA_TRY(ctx, launch_green_rhs(ctx, fq, ug, wk, 2, s));
    if (!(skip & 2)) DPM_CUDA_TRY(ctx, ctx_solve(ctx, wk, wk, 2, s));
  }
  if (!(skip & 16)) DPM_CUDA_TRY(ctx, launch_restrict_stats(ctx, wk, rho, c, slot + 4, s, true, abort));
  if (fork) DPM_CUDA_TRY(ctx, cudaStreamWaitEvent(s, ctx->ev_side[1], 0));
  return DPM_OK;
}

// Graph of K consecutive speculative steps at dt (captured once per (dt, K, params, fields), replayed).
static dpm_status pks_graph(dpm_ctx* ctx, double* rho, double* c, const dpm_pks_params* prm, double dt, int K,
                            dpm_ctx::PksGraph** out) {
  for (auto& g : ctx->pks_graphs)
    if (g.dt == dt && g.k == K && g.chi == prm->chi && g.cap == prm->dt_cap && g.rule == prm->dt_rule &&
        g.clamp == prm->clamp && g.coupling == prm->coupling && g.rho == rho && g.c == c &&
        g.solver == ctx->plan.solver) {
      *out = &g;
      return DPM_OK;
    }
  const size_t field = (size_t)ctx->n * ctx->n * ctx->n;
  cudaStream_t cs = ctx->graph_stream;
  PassProf* prof = ctx->plan.prof;
  ctx->plan.prof = nullptr;   // no timing events inside graphs
  const long long l0 = (long long)g_dpm_launches.load();
  DPM_CUDA_TRY(ctx, octsplit_prepare(ctx, 2));   // the parity-split solver's tables and boxes (no allocation in a capture)
  DPM_CUDA_TRY(ctx, cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
  dpm_status st = DPM_OK;
  static const int pdl_nmax = [] {   // programmatic dependent launch within the step graph (dpm_internal.h)
    const char* v = getenv("DPM_PDL_NMAX");
    return v ? atoi(v) : 64;
  }();
  const int pdl = ctx->n <= pdl_nmax;
  g_pdl_scope += pdl;
  int* abort = pks_abort_on() ? pks_abort_flag(ctx) : nullptr;
  if (abort) {
    const cudaError_t em = cudaMemsetAsync(abort, 0, sizeof(int), cs);
    if (em != cudaSuccess) { ctx->err = "capture memset"; st = DPM_ERR_CUDA; }
  }
  for (int i = 0; i < K && st == DPM_OK; ++i)
    st = enqueue_pks_step(ctx, rho, c, prm, dt, ctx->pks_log + 16 * i,
                          abort ? nullptr : ctx->pks_backup + (size_t)i * 2 * field, cs, abort);
  g_pdl_scope -= pdl;
  if (st == DPM_OK) {
    cudaError_t e = cudaMemcpyAsync(ctx->pks_log_host, ctx->pks_log, (size_t)K * 16 * 8, cudaMemcpyDeviceToHost, cs);
    if (e != cudaSuccess) { ctx->err = "capture memcpy"; st = DPM_ERR_CUDA; }
  }
  cudaGraph_t graph = nullptr;
  const cudaError_t ec = cudaStreamEndCapture(cs, &graph);
  ctx->plan.prof = prof;
  const long long nk = (long long)g_dpm_launches.load() - l0;
  g_dpm_launches.fetch_sub(nk);   // counted again on every replay
  if (st != DPM_OK) {
    if (graph) cudaGraphDestroy(graph);
    return st;
  }
  if (ec != cudaSuccess) { ctx->err = std::string("graph capture: ") + cudaGetErrorString(ec); return DPM_ERR_CUDA; }
  dpm_ctx::PksGraph g;
  g.dt = dt; g.k = K; g.chi = prm->chi; g.cap = prm->dt_cap; g.rule = prm->dt_rule; g.clamp = prm->clamp;
  g.coupling = prm->coupling;
  g.solver = ctx->plan.solver;   // dst_solve_batch reads it at capture time
  g.rho = rho; g.c = c; g.launches = nk;
  // A cached graph of the same shape that differs only in dt / dt_cap (every step of the Step-4b-every-step
  // regime runs at a new dt): update its kernel parameters in place instead of instantiating a new graph
  // (~0.4 ms per instantiation at cfg3).  DPM_GRAPH_UPDATE=0 always instantiates.
  static const bool upd = [] {
    const char* v = getenv("DPM_GRAPH_UPDATE");
    return !(v && atoi(v) == 0);
  }();
  if (upd)
    for (auto& e : ctx->pks_graphs)
      if (e.k == K && e.chi == prm->chi && e.rule == prm->dt_rule && e.clamp == prm->clamp &&
          e.coupling == prm->coupling && e.rho == rho && e.c == c && e.solver == ctx->plan.solver) {
        cudaGraphExecUpdateResultInfo info;
        if (cudaGraphExecUpdate(e.exec, graph, &info) == cudaSuccess) {
          e.dt = dt;
          e.cap = prm->dt_cap;
          e.launches = nk;
          cudaGraphDestroy(graph);
          *out = &e;
          return DPM_OK;
        }
        cudaGetLastError();   // topology differs: instantiate below
      }
  const cudaError_t ei = cudaGraphInstantiate(&g.exec, graph, 0);
  cudaGraphDestroy(graph);
  if (ei != cudaSuccess) { ctx->err = std::string("graph instantiate: ") + cudaGetErrorString(ei); return DPM_ERR_CUDA; }
  if (ctx->pks_graphs.size() >= 8) {   // bounded cache
    cudaGraphExecDestroy(ctx->pks_graphs.front().exec);
    ctx->pks_graphs.erase(ctx->pks_graphs.begin());
  }
  ctx->pks_graphs.push_back(g);
  *out = &ctx->pks_graphs.back();
  return DPM_OK;
}

dpm_status dpm_pks_step(dpm_ctx* ctx, double* rho, double* c, int32_t nsteps, const dpm_pks_params* prm,
                        dpm_step_log* log, void* stream) {
  DPM_NVTX();
  if (!ctx || !rho || !c || !prm || nsteps < 0) return DPM_ERR_INVALID;
  if (!(prm->dt_cap > 0) || !(prm->chi > 0)) { ctx->err = "dt_cap and chi must be > 0"; return DPM_ERR_INVALID; }
  if (prm->coupling != 0 && prm->coupling != 1) { ctx->err = "coupling must be 0 or 1"; return DPM_ERR_INVALID; }
  if (!ctx->pks_initialized) { ctx->t = 0.0; ctx->dt_prev = INFINITY; ctx->pks_initialized = 1; }
  if (nsteps == 0) return DPM_OK;
  cudaSetDevice(ctx->device);
  cudaStream_t s = as_stream(stream);
  const size_t field = (size_t)ctx->n * ctx->n * ctx->n;
  const int64_t ng = ctx->counts[DPM_SET_GAMMA], ngin = ctx->counts[DPM_SET_GAMMA_IN];
  if (!ctx->scratch || ctx->scratch_bytes < (size_t)(4 * field + 2 * ngin + 2 * ng + 4 * ctx->K) * 8) {
    if (ctx->scratch) cudaFree(ctx->scratch);
    ctx->scratch_bytes = (size_t)(4 * field + 2 * ngin + 2 * ng + 4 * ctx->K) * 8;   // + residual z (K x 2)
    DPM_CUDA_TRY(ctx, cudaMalloc(&ctx->scratch, ctx->scratch_bytes));
    for (auto& g : ctx->pks_graphs) cudaGraphExecDestroy(g.exec);   // captured with the old scratch
    ctx->pks_graphs.clear();
  }
  constexpr int KMAX = dpm_ctx::PKS_K;
  if (!ctx->graph_stream) {
    DPM_CUDA_TRY(ctx, cudaStreamCreateWithFlags(&ctx->graph_stream, cudaStreamNonBlocking));
    DPM_CUDA_TRY(ctx, cudaMalloc(&ctx->pks_log, KMAX * 16 * sizeof(double)));
    DPM_CUDA_TRY(ctx, cudaMemset(ctx->pks_log, 0, KMAX * 16 * sizeof(double)));   // CFL maxima start at 0
    DPM_CUDA_TRY(ctx, cudaMallocHost(&ctx->pks_log_host, KMAX * 16 * sizeof(double)));
    if (!pks_abort_on()) DPM_CUDA_TRY(ctx, cudaMalloc(&ctx->pks_backup, (size_t)KMAX * 2 * field * sizeof(double)));
    DPM_CUDA_TRY(ctx, cudaStreamCreateWithFlags(&ctx->side_stream, cudaStreamNonBlocking));
    for (auto& e : ctx->ev_side) DPM_CUDA_TRY(ctx, cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  cudaStream_t gs = ctx->graph_stream;
  // the caller's prior work on `s` (e.g. dpm_pks_init) precedes the steps
  DPM_CUDA_TRY(ctx, cudaStreamSynchronize(s));
  const double h = ctx->h;
  int done = 0;
  double dt_next = NAN;   // dt already decided by a rejected speculation (device rule, exact)
  while (done < nsteps) {
    // Step 3: dt for the next batch.  Speculate dt_i = dt_{i-1}; the device evaluates the rule for
    // every step of the batch and the batch is cut at the first step whose dt would decrease.
    double dt = prm->dt_cap;
    if (prm->dt_rule == 0) {
      if (!std::isnan(dt_next)) {
        dt = dt_next;
      } else if (std::isinf(ctx->dt_prev)) {   // first step: the rule on the host
        DPM_CUDA_TRY(ctx, launch_cfl_reduce(ctx, c, ctx->red, gs));
        DPM_CUDA_TRY(ctx, cudaMemcpyAsync(ctx->red_host, ctx->red, 3 * sizeof(double), cudaMemcpyDeviceToHost, gs));
        DPM_CUDA_TRY(ctx, cudaStreamSynchronize(gs));
        double cfl = INFINITY;
        for (int a = 0; a < 3; ++a) {
          const double mx = ctx->red_host[a] / h;
          if (mx > 0) cfl = std::fmin(cfl, h / (6.0 * prm->chi * mx));
        }
        dt = std::fmin(std::fmin(ctx->dt_prev, prm->dt_cap), std::fmin(cfl, 0.5 * h * h));
      } else {
        dt = ctx->dt_prev;
      }
    }
    dt_next = NAN;
    // Step 2 / 4b: (re)build the BEP when dt differs from the one it was built at
    int rebuilt = 0;
    if (!ctx->have_projection || dt != ctx->dt_bep) {
      dpm_status r = dpm_set_dt(ctx, dt);
      if (r != DPM_OK) return r;
      ctx->have_projection = 0;
      r = dpm_build_projection(ctx, nullptr, nullptr, gs);
      if (r != DPM_OK) return r;
      rebuilt = 1;
    }
    const int K = std::min(KMAX, nsteps - done);
    dpm_ctx::PksGraph* g = nullptr;
    dpm_status st = pks_graph(ctx, rho, c, prm, dt, K, &g);
    if (st != DPM_OK) return st;
    DPM_CUDA_TRY(ctx, cudaGraphLaunch(g->exec, gs));
    g_dpm_launches.fetch_add(g->launches);
    DPM_CUDA_TRY(ctx, cudaStreamSynchronize(gs));
    int accepted = K;
    for (int i = 0; i < K; ++i) {
      const double* L = ctx->pks_log_host + 16 * i;
      if (prm->dt_rule == 0 && L[3] < dt) {   // this step needs a smaller dt: roll back to its start
        if (ctx->pks_backup) {   // (abort mode: the graph already left the state at the step's start)
          DPM_CUDA_TRY(ctx, cudaMemcpyAsync(rho, ctx->pks_backup + (size_t)i * 2 * field, field * 8,
                                            cudaMemcpyDeviceToDevice, gs));
          DPM_CUDA_TRY(ctx, cudaMemcpyAsync(c, ctx->pks_backup + (size_t)i * 2 * field + field, field * 8,
                                            cudaMemcpyDeviceToDevice, gs));
          DPM_CUDA_TRY(ctx, cudaStreamSynchronize(gs));
        }
        dt_next = L[3];
        accepted = i;
        break;
      }
      ctx->dt_prev = dt;
      ctx->t += dt;
      if (L[8] != 0.0) {
        if (i + 1 < K && ctx->pks_backup) {   // leave the state right after the failing step
          DPM_CUDA_TRY(ctx, cudaMemcpyAsync(rho, ctx->pks_backup + (size_t)(i + 1) * 2 * field, field * 8,
                                            cudaMemcpyDeviceToDevice, gs));
          DPM_CUDA_TRY(ctx, cudaMemcpyAsync(c, ctx->pks_backup + (size_t)(i + 1) * 2 * field + field, field * 8,
                                            cudaMemcpyDeviceToDevice, gs));
          DPM_CUDA_TRY(ctx, cudaStreamSynchronize(gs));
        }
        ctx->err = "non-finite value in the PKS step";
        return DPM_ERR_NONFINITE;
      }
      if (log) {
        dpm_step_log& Lg = log[done + i];
        Lg.t = ctx->t;
        Lg.dt = dt;
        Lg.mass = mass_fixed_decode(L + 4) * h * h * h;
        Lg.rho_max = decode_key(L[5]);
        Lg.rho_min = -decode_key(L[6]);
        Lg.c_min = -decode_key(L[7]);
        Lg.rebuilt = (i == 0) ? rebuilt : 0;
        Lg.step = done + i;
        Lg.rho_max_mplus = decode_key(L[9]);
        Lg.clamp_max = prm->coupling == 0 ? decode_key(L[10]) : NAN;
        Lg.lsq_resid = prm->coupling == 0 ? L[11] : NAN;
      }
    }
    done += accepted;
  }
  return DPM_OK;
}

int64_t dpm_launch_count(void) {
  DPM_NVTX(); return (int64_t)g_dpm_launches.load(); }

dpm_status dpm_set_pass_timing(dpm_ctx* ctx, int32_t enable) {
  DPM_NVTX();
  if (!ctx) return DPM_ERR_INVALID;
  ctx->plan.prof = enable ? &ctx->prof : nullptr;
  ctx->prof.used = 0;
  ctx->prof.kind.clear();
  ctx->prof.points.clear();
  return DPM_OK;
}

dpm_status dpm_pass_times(dpm_ctx* ctx, double* ms, int64_t* launches, int64_t* points) {
  DPM_NVTX();
  if (!ctx || !ms || !launches || !points) return DPM_ERR_INVALID;
  cudaSetDevice(ctx->device);
  for (int k = 0; k < 3; ++k) {
    ms[k] = 0.0;
    launches[k] = 0;
    points[k] = 0;
  }
  PassProf& P = ctx->prof;
  for (size_t i = 0; i < P.kind.size(); ++i) {
    DPM_CUDA_TRY(ctx, cudaEventSynchronize(P.pool[2 * i + 1]));
    float t = 0.f;
    DPM_CUDA_TRY(ctx, cudaEventElapsedTime(&t, P.pool[2 * i], P.pool[2 * i + 1]));
    ms[P.kind[i]] += t;
    launches[P.kind[i]] += 1;
    points[P.kind[i]] += P.points[i];
  }
  P.used = 0;
  P.kind.clear();
  P.points.clear();
  return DPM_OK;
}

}  // extern "C"
