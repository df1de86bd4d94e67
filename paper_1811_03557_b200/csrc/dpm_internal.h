// Internal declarations shared by the CUDA translation units of libdpm.so.
// Not part of the ABI (include/dpm.h is).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <string>
#include <vector>

#include "../../include/dpm.h"

// internal domain kind of an octant subdomain (dpm_create_octant), canonical frame (+,+,+)
constexpr int DPM_OCTANT_CANON = 100;
// internal domain kind of the Case-1 DD outer subdomain (dpm_create_dd1, NEXT-3): the open shell
// semi[1] < |x| < semi[0] centred at the origin
constexpr int DPM_SHELL_CANON = 101;

// point-flag bits for the uint8 mask over the n^3 interior
enum : uint8_t {
  F_MPLUS = 1,   // M+
  F_NPLUS = 2,   // N+ ∩ M0
  F_GAMMA = 4,   // gamma
  F_BAND = 8,    // M- ∩ dil7(gamma)
  F_NMINUS = 16  // N- ∩ M0
};

// Optional per-pass timing (dpm_set_pass_timing): CUDA events recorded on the launching stream
// around every pass of dpm_aux_solve_batch, summed per pass kind by dpm_pass_times.
struct PassProf {
  std::vector<cudaEvent_t> pool;           // reused events (2 per recorded pass)
  std::vector<int> kind;                   // pass kind of record i (0 x, 1 y, 2 z / tridiagonal)
  std::vector<long long> points;           // grid points processed by record i
  size_t used = 0;                         // events handed out since the last readout
  cudaEvent_t next();
};

struct DstPlan {
  int n = 0;
  double h = 0, dt = 0;
  double* lam = nullptr;  // device, n eigenvalues λ_m (R26)
  double* atab = nullptr; // device, per-warp folded sine-matrix DMMA A fragments
  int solver = DPM_SOLVER_DST2_TRIDIAG;
  double* atab128 = nullptr;  // n = 128: A fragments of the prime-factor DST-I
  int pfa = 1;            // n = 128: prime-factor DST-I for the x / y passes (DPM_PFA=0 disables)
  int plane = 1;          // n = 128: fused y / z / y plane pass (DPM_PLANE=0 disables)
  double* sinmat = nullptr;   // n <= 64: device n x n sine matrix of the fused small-n plane pass
  PassProf* prof = nullptr;   // non-null while pass timing is enabled
  cudaStream_t side = nullptr;                    // second chunk stream (DPM_STREAMS=2)
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
};

struct dpm_ctx {
  int device = 0;
  int n = 0;
  double lo = 0, hi = 0, h = 0, dt = 0;
  dpm_domain domain{};
  int lmax = 0, basis = 0, K = 0;
  cudaStream_t setup_stream = nullptr;
  std::string err;

  // point sets (device)
  uint8_t* flags = nullptr;      // [n^3]
  int32_t* gmap = nullptr;       // [n^3] gamma position or -1
  int64_t* lists[6] = {nullptr}; // dpm_set order
  int64_t counts[6] = {0};
  int64_t ghosts_in_nplus = 0;
  int64_t exact_ties = 0;         // nodes within the fp64 tie band, decided exactly on the host (R6)
  int64_t exact_ties_inside = 0;  // of those, the ones in M+
  int32_t* gin_pos = nullptr;    // [n_gamma_in] position of gamma_in points inside gamma
  uint16_t* mplus_slope = nullptr;  // [n_M+] minmod-slope validity bits per M+ point (flux_rhs_list_kernel)

  // gamma geometry + extension matrix (device)
  double* foot = nullptr;        // [n_gamma][3]
  double* dist = nullptr;        // [n_gamma]
  double* E = nullptr;           // [K][n_gamma] (column-major |gamma| x K)

  DstPlan plan;

  // BEP / LSQ (device)
  int have_projection = 0;
  double dt_bep = 0;
  double* B = nullptr;           // [K][n_gin]
  double* Q = nullptr;           // [K][n_gin]  equilibrated Q
  double* R = nullptr;           // [K][K] col-major upper triangular
  double* colscale = nullptr;    // [K]
  double* Mlsq = nullptr;        // [K][n_gin] row-major: D R^{-1} Q^T (the LSQ apply operator)
  double* RDinv = nullptr;       // [K][K] row-major: R D^{-1} (the per-step LSQ residual, lsq_residual)
  double bep_cond = 0;
  double* lsq_ws = nullptr;      // scratch

  // workspaces
  double* work = nullptr;        // boxes for the solver / PKS
  size_t work_boxes = 0;
  double* scratch = nullptr;
  size_t scratch_bytes = 0;

  // PKS state
  double t = 0, dt_prev = 0;
  int pks_initialized = 0;
  PassProf prof;
  // PKS step graphs (dpm_pks_step): K speculative steps at a fixed dt captured once and replayed
#ifndef DPM_PKS_K
#define DPM_PKS_K 10
#endif
  static constexpr int PKS_K = DPM_PKS_K;
  struct PksGraph {
    double dt = 0, chi = 0, cap = 0;
    int k = 0, rule = 0, clamp = 0, coupling = 0, solver = 0;
    double* rho = nullptr;
    double* c = nullptr;
    cudaGraphExec_t exec = nullptr;
    long long launches = 0;
  };
  std::vector<PksGraph> pks_graphs;
  cudaStream_t graph_stream = nullptr;
  double* pks_log = nullptr;        // device [PKS_K][16]: red(3), dt_true, stats(6), clamp max (key), lsq residual
  double* pks_log_host = nullptr;   // pinned mirror
  double* pks_backup = nullptr;     // device [PKS_K][2][n^3]: state at the start of each step
  cudaStream_t side_stream = nullptr;   // PKS graphs: the residual runs on a forked branch
  cudaEvent_t ev_side[2] = {nullptr, nullptr};

  // octant DD subdomain (dpm_create_octant)
  int dd = 0;                       // 1 for an octant subdomain
  int octant = 0;                   // s = 4[σx<0] + 2[σy<0] + [σz<0]
  double sigma[3] = {1, 1, 1};
  double radius = 1.0;
  int Lc = 0, Li = 0, nphi = 0;
  double* dd_Eraw = nullptr;        // [K][n_gamma]: each piece's extension (block-sparse by column)
  uint8_t* dd_assign = nullptr;     // [n_gamma]: piece bits (1 cap, 2 x, 4 y, 8 z)
  int32_t* dd_rows = nullptr;       // [n_rows][2]: (gamma position, piece) of the BEP rows
  int64_t n_rows = 0;
  double* dd_B = nullptr;           // [K][n_rows] BEP block
  double* dd_Q = nullptr;           // [K][n_rows] equilibrated Q1 / Q
  double* dd_R = nullptr;           // [3][K][K]: R1, R2, R
  double* dd_M = nullptr;           // [K][n_rows] row-major: D R^{-1} Q^T
  double* dd_D = nullptr;           // [K] global column scaling
  double* dd_g = nullptr;           // [2][n_rows] per-step BEP right-hand sides
  double* dd_ug = nullptr;          // [2][n_gamma] u_γ = A C
  int dd_blk[6] = {0};              // first column of each piece's block (dd_blk[npieces] = K)
  double* dd_sign = nullptr;        // [K] (+ flag) column signs relative to octant dd_sign_ref (shared apply)
  const dpm_ctx* dd_sign_ref = nullptr;
  double* dd_shared = nullptr;      // workspace of dpm_dd_lsq_rhs_shared (on the first octant)
  size_t dd_shared_bytes = 0;
  int dd_npieces = 0;
  // Case-1 two-subdomain DD (dd == 2, dpm_create_dd1, NEXT-3): Ω1 = ball r1 (sub 0) or Ω2 = shell (sub 1)
  int dd1_sub = 0, dd1_mz = 0, dd1_mg = 0;
  double dd1_r1 = 0, dd1_r2 = 0;
  // fused BEP column build at n = 128 (bep_fused.cu)
  uint32_t* bepf_btab = nullptr;     // [n^2][8] band x-line table (mask, start); built on first use
  int32_t* bepf_bpos = nullptr;      // [n_band] line-major position of band point b
  double* bepf_qb = nullptr;         // [cols][n_band] band values of the potential RHS (line-major)
  int bepf_cols = 0;
  cudaGraphExec_t fac_exec = nullptr; // the captured factorisation (lsq_factor) for (fac_B, fac_K, fac_m)
  cudaStream_t fac_stream = nullptr;
  const double* fac_B = nullptr;
  int fac_K = 0;
  int64_t fac_m = 0;
  int fac_blocks = 0;                 // the captured factorisation is the block-diagonal one (bep_sym.cu)
  long long fac_launches = 0;
  double* bepf_zbox = nullptr;       // [zcols][n^3] boxes that are zero off the band (zero-box mode)
  int bepf_zcols = 0;
  // BEP columns on the octant by reflection symmetry (bep_sym.cu): 0 undecided, 1 on, -1 full path
  int sym = 0, sym_m = 0, sym_cols = 0;
  int64_t sym_nlist = 0;
  int64_t* sym_list = nullptr;       // [sym_nlist] band points inside the octant (flat n^3 index)
  int32_t* sym_dst = nullptr;        // [sym_nlist] their octant (m^3) index
  int32_t* sym_gidx = nullptr;       // [n_gamma + n_gamma_in] octant index | reflection bits << 24
  uint8_t* sym_par = nullptr;        // [K] column parities (bit a: odd under x_a -> -x_a)
  double* sym_S = nullptr;           // [2][MP][MP] octant sine matrices (even / odd parity)
  double* sym_lam = nullptr;         // [2][MP] their eigenvalues
  double* sym_zbox = nullptr;        // [sym_cols][m^3] octant boxes, zero off the band
  double* sym_work = nullptr;        // [sym_cols][m^3]
  double* sym_R = nullptr;           // x-tridiagonal LU factors (sym_lu_kernel), built at Δt = sym_lu_dt
  double sym_lu_dt = 0.0;
  int sym_off[9] = {0};              // parity-class column ranges in the class order sym_perm
  int32_t* sym_perm = nullptr;       // [K] class-ordered position -> column
  int32_t* sym_mirin = nullptr;      // [3][n_gamma_in] γ_in position of the mirror point
  double* sym_Bp = nullptr;          // [K][n_gamma_in] class-ordered B, then the operator blocks
  double* sym_tmp = nullptr;         // [K][n_gamma_in] CholeskyQR2 ping-pong
  double* sym_dg = nullptr;          // [K] |diag R| (class order)
  int* sym_flag = nullptr;
  // parity-split AP solve (bep_sym.cu, octsplit_solve; n = 127 by default): operator tables of its own (the BEP
  // octant path needs symmetric sets, the solver does not), LU factors in two slots (0: eager calls, cached
  // by Δt; 1: inside graph captures, rebuilt at the start of every captured graph), fold / solve boxes
  int osp = 0;                       // 0: undecided, 1: on, -1: off
  double* osp_S = nullptr;           // [4][MP][MP]
  double* osp_lam = nullptr;         // [2][MP]
  double* osp_R[2] = {nullptr, nullptr};
  double osp_lu_dt = 0.0;
  unsigned long long osp_cap_id = 0; // capture sequence whose graph already rebuilds slot 1 ...
  double osp_cap_dt = 0.0;           // ... at this Δt
  double* osp_Q = nullptr;           // [osp_cap * 8][m^3] class components of the right-hand sides
  double* osp_U = nullptr;           // [osp_cap * 8][m^3] their solutions
  uint8_t* osp_par = nullptr;        // [osp_cap * 8] class bits (column c: c & 7)
  int osp_cap = 0;                   // fields per chunk
  cudaStream_t sym_streams[8] = {};  // one capture branch per parity class
  cudaEvent_t sym_ev[9] = {};
  // host-buffer solve pipeline (dpm_aux_solve_batch_host)
  cudaStream_t h2d_stream = nullptr, d2h_stream = nullptr;
  cudaEvent_t pipe_ev[9] = {};   // host pipeline: up / solved / down per ring buffer (3)
  double* red = nullptr;         // device reduction slots
  double* red_host = nullptr;    // pinned
};

// process-wide launch counter (dpm_launch_count)
#include <atomic>
extern std::atomic<long long> g_dpm_launches;
#define DPM_COUNT_LAUNCH(k) (g_dpm_launches.fetch_add((k), std::memory_order_relaxed))

// Programmatic dependent launch (PDL) for the chain of small kernels of a PKS step (and every other use
// of these kernels): they are launched with cudaLaunchAttributeProgrammaticStreamSerialization and begin
// with pdl_prologue(): griddepcontrol.wait (before any global memory access; a no-op when launched
// without the attribute).  No explicit griddepcontrol.launch_dependents: the next kernel is triggered
// as this one's blocks exit, so its launch is prepared during this kernel's tail instead of after the
// kernel boundary, and no dependent CTA waits on an SM while this grid still needs it.  Used inside the
// PKS step graphs of n <= 64 (pdl_scope, set by dpm_pks_step; DPM_PDL_NMAX overrides the bound).
// Measured (tools/pdl_ab.sh): cfg2 +6-7% and cfg3 +1.7% steps/s over no PDL; triggering at kernel start
// (-DDPM_PDL_TRIGGER=1) instead costs 9% at cfg3, where the early dependents' waiting CTAs compete with
// the running grid.  DPM_PDL=0 disables, DPM_PDL=2 forces it for every launch of these kernels.
#ifndef DPM_PDL_TRIGGER
#define DPM_PDL_TRIGGER 0
#endif
__device__ __forceinline__ void pdl_prologue() {
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
#if DPM_PDL_TRIGGER
  asm volatile("griddepcontrol.launch_dependents;\n" :::);
#endif
}
bool pdl_enabled();
extern thread_local int g_pdl_scope;   // > 0 while enqueueing a small-grid PKS step
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, k, static_cast<KArgs>(args)...);
}

// NVTX range per C-ABI call (SURVEY §5 tracing): every extern "C" dpm_* entry point opens one named
// after itself, so nsys / ncu timelines show the ABI phases (header-only NVTX3, no extra library).
#include <nvtx3/nvToolsExt.h>
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};
#define DPM_NVTX() NvtxRange dpm_nvtx_range_(__func__)

// helpers
#define DPM_CUDA_TRY(ctx, call)                                                       \
  do {                                                                                \
    cudaError_t _e = (call);                                                          \
    if (_e != cudaSuccess) {                                                          \
      (ctx)->err = std::string(#call) + ": " + cudaGetErrorString(_e);                \
      return DPM_ERR_CUDA;                                                            \
    }                                                                                 \
  } while (0)

// dst_solve.cu
cudaError_t dst_plan_init(DstPlan& p, int n, double h, double dt);
void dst_plan_free(DstPlan& p);
cudaError_t dst_solve_batch(const DstPlan& p, const double* q, double* u, int64_t batch, double* scratch,
                            size_t scratch_bytes, cudaStream_t s);
size_t dst_scratch_bytes(int n, int chunk);
// the passes between the two x transforms (partial diagonalisation only), in place on x-transformed fields
cudaError_t dst_solve_middle(const DstPlan& p, double* u, int64_t batch, cudaStream_t s);

// dst128.cu (n = 128 prime-factor DST-I passes)
cudaError_t dst128_init();
cudaError_t dst128_atab(double** tab);
cudaError_t dst128_pass(int pass, const double* in, double* out, int nfields, const double* atab, cudaStream_t s);
cudaError_t plane128_pass(double* u, int nfields, const double* lam, double inv_dt, double h2, double rscale,
                          cudaStream_t s);
// forward x pass of the fused BEP build (bep_fused.cu) from x-line-major band values vals[f*ldv + .]
// through the band line table tab ([n^2][8] u32: 128-bit x mask, start)
cudaError_t dst128_xpass_sparse(double* out, int nfields, const uint32_t* tab, const double* vals, int64_t ldv,
                                cudaStream_t s);

// setup.cu
dpm_status setup_point_sets(dpm_ctx* ctx);
dpm_status setup_geometry(dpm_ctx* ctx);

// ops.cu
// scatter of the band values only (q must already be zero off the band)
cudaError_t launch_potential_scatter(const dpm_ctx* ctx, const double* v, int64_t ldv, double* q, int nrhs,
                                     cudaStream_t s);
cudaError_t launch_potential_rhs(const dpm_ctx* ctx, const double* v, int64_t ldv, double* q, int nrhs,
                                 cudaStream_t s);
cudaError_t launch_potential_band(const dpm_ctx* ctx, const double* v, int64_t ldv, double* qb, int nrhs,
                                  const int32_t* pos, cudaStream_t s);
cudaError_t launch_trace(const dpm_ctx* ctx, const double* u, double* out, int which, int64_t batch,
                         cudaStream_t s);
cudaError_t launch_bep_gather(const dpm_ctx* ctx, const double* U, int c0, int ncols, double* PgE,
                              double* B, cudaStream_t s);

// lsq.cu
dpm_status lsq_factor(dpm_ctx* ctx, const double* B, cudaStream_t s);
cudaError_t lsq_apply(dpm_ctx* ctx, const double* g, double* coef, double* u_gamma, int nrhs, int clamp,
                      cudaStream_t s, double* clampmax = nullptr);
// ||B C - g|| / ||g|| (max over nrhs <= 2) -> out[0], from the ctx's factorisation (lsq.cu)
// zws: K x nrhs scratch
cudaError_t lsq_residual(dpm_ctx* ctx, const double* coef, const double* g, int nrhs, double* zws, double* out,
                         cudaStream_t s);

// lsq.cu building blocks (octant DD)
cudaError_t lsq_gram(const double* A, int64_t m, int K, double* G, cudaStream_t s);
cudaError_t lsq_cholesky(double* G, int K, int* dfail, cudaStream_t s);
cudaError_t lsq_mul_upper(const double* A, int64_t m, int K, const double* T, double* out, cudaStream_t s);
cudaError_t lsq_operator_from_rinv(const double* Ri, const double* Q, int64_t m, int K, const double* scale, double* M,
                                   cudaStream_t s);
// R^{-1} of an upper-triangular K x K R (col-major), blocked by 32 x 32 tiles
cudaError_t lsq_rinv(const double* R, int K, double* Ri, cudaStream_t s);
cudaError_t lsq_trmm(const double* A, const double* B, double* C, int K, cudaStream_t s);
cudaError_t lsq_mul_rinv(const double* A, int64_t m, int K, const double* R, double* Ri_ws, double* out,
                         cudaStream_t s);   // out = A R^{-1} (R upper K x K)
cudaError_t lsq_scale_cols(const double* B, int64_t m, int K, const double* scale, double* A, cudaStream_t s);
cudaError_t lsq_build_operator(const double* R, const double* Q, int64_t m, int K, const double* scale, double* M,
                               double* Ri_ws, cudaStream_t s);
cudaError_t lsq_gemv(const double* M, int64_t m, int K, const double* g, int nrhs, double* coef, cudaStream_t s);
cudaError_t lsq_extend(const double* E, int64_t ng, int K, const double* coef, int nrhs, int clamp, double* ug,
                       cudaStream_t s, double* clampmax = nullptr);

// dd.cu (octant DD setup)
dpm_status dd_setup(dpm_ctx* ctx);
// dpm_abi.cu
// extension column sets (dpm.h dpm_basis): zonal modes only / number of components (1 or 2)
__host__ __device__ inline bool basis_zonal(int b) {
  return b == DPM_BASIS_CAUCHY_ZONAL || b == DPM_BASIS_NEUMANN0_ZONAL || b == DPM_BASIS_NEUMANN0_2TERM_ZONAL;
}
__host__ __device__ inline int basis_ncomp(int b) { return b == DPM_BASIS_NEUMANN0_2TERM || b == DPM_BASIS_NEUMANN0_2TERM_ZONAL ? 1 : 2; }

dpm_status dpm_create_impl(const dpm_grid* grid, const dpm_domain* domain, int32_t lmax, double dt, int32_t basis,
                           int32_t device, dpm_ctx** out);
double decode_key(double slot);   // order-preserving key of the reduction slots -> value
double mass_fixed_decode(const double* stats);   // 128-bit fixed-point mass (stats[0] low, stats[8] high) -> value

// pks.cu
cudaError_t launch_pks_init(dpm_ctx* ctx, double* rho, double* c, const dpm_pks_ic* ic, cudaStream_t s);
cudaError_t launch_cfl_reduce(dpm_ctx* ctx, const double* c, double* out3, cudaStream_t s);
cudaError_t launch_slope_mask(dpm_ctx* ctx, cudaStream_t s);   // ctx->mplus_slope from the flags (setup)
cudaError_t launch_flux_rhs(dpm_ctx* ctx, const double* rho, const double* c, double dt, double chi,
                            double* fq_rho, double* fq_c, cudaStream_t s,
                            double* backup = nullptr, double* zero6 = nullptr, double* cfl_out3 = nullptr,
                            double dt_prev = 0, double cap = 0, double* dt_out = nullptr, int* abort = nullptr);
cudaError_t launch_fc_seq(dpm_ctx* ctx, const double* c, const double* rho_new, double dt, double* fq_c, cudaStream_t s);
cudaError_t launch_green_band_inplace(dpm_ctx* ctx, double* fq, const double* u_gamma, int nrhs, cudaStream_t s);
cudaError_t launch_green_rhs(dpm_ctx* ctx, const double* fq, const double* u_gamma, double* q, int nrhs,
                             cudaStream_t s);
cudaError_t launch_diagnostics(dpm_ctx* ctx, const double* rho, const double* c, double* out3, cudaStream_t s);
cudaError_t launch_restrict_stats(dpm_ctx* ctx, const double* u, double* rho, double* c, double* stats,
                                  cudaStream_t s,
                                  bool zeroed = false, int* abort = nullptr);
// bep_fused.cu (sparse-in / gamma-out BEP columns)
bool bep_zbox_enabled();
cudaError_t bep_zbox(dpm_ctx* ctx, int nc, double** out, cudaStream_t s);
bool bep_fused_enabled(const dpm_ctx* ctx);
cudaError_t bep_columns_fused(dpm_ctx* ctx, int c0, int nc, double* PgE, double* B, cudaStream_t s);
void bep_fused_free(dpm_ctx* c);
cudaError_t launch_potential_list(const dpm_ctx* ctx, const double* v, int64_t ldv, const int64_t* list,
                                  const int32_t* dst, int64_t nlist, double* q, int64_t qstride, int nrhs,
                                  cudaStream_t s);
cudaError_t bep_sym_columns(dpm_ctx* ctx, int c0, int c1, double* PgE, double* B, cudaStream_t s, bool* done);
// AP solve of `batch` dense boxes by the 8 reflection-parity components on the octant (n = 127 by default,
// every 4 <= n < 128 with DPM_OCTSPLIT=2; default solver only); *done = false and nothing runs when it does not apply.  ctx_solve: that, else dst_solve_batch.
cudaError_t octsplit_prepare(dpm_ctx* ctx, int64_t batch);   // tables and boxes (allocates: not inside a capture)
cudaError_t octsplit_solve(dpm_ctx* ctx, const double* q, double* u, int64_t batch, cudaStream_t s, bool* done);
cudaError_t ctx_solve(dpm_ctx* ctx, const double* q, double* u, int64_t batch, cudaStream_t s);
void bep_sym_free(dpm_ctx* c);
bool bep_sym_blocks(dpm_ctx* ctx, const double* B, cudaStream_t s);
