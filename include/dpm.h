/*
 * dpm.h — C ABI of the B200-native Difference Potentials Method (DPM) hot path.
 *
 * Paper: arXiv 1811.03557, "Efficient Numerical Algorithms Based on Difference
 * Potentials for Chemotaxis Systems in 3D" (/root/reference/PAPER.md, cited P:<line>).
 * Scope: SURVEY.md §8 (hot-path scope table) — batched Dirichlet modified-Helmholtz
 * auxiliary-problem (AP) solves on the Cartesian box, restriction to the discrete grid
 * boundary γ, the boundary projection P_γ / reduced BEP, the least-squares solve for
 * spherical-harmonic Cauchy-data coefficients, and the PKS time step driving them.
 *
 * Conventions (all functions):
 *  - fp64 everywhere; no torch or C++ types cross this boundary; nothing throws.
 *  - Every entry point returns a dpm_status; on failure dpm_last_error(ctx) holds a
 *    human-readable message (thread-unsafe; one ctx per host thread / stream).
 *  - "device" pointers are CUDA device pointers on the ctx's device (e.g. torch
 *    tensor data_ptr()); the CALLER owns every field buffer; the ctx owns its
 *    workspaces, point-set lists and the BEP factorization.
 *  - `stream` is a cudaStream_t (NULL = legacy default stream).  Work is enqueued on
 *    it; functions that must make a host decision synchronize it and say so.
 *  - Grid: the cube [lo,hi]^3 has its faces on the Dirichlet ghost layer
 *    N0\M0; n unknowns per axis; h = (hi-lo)/(n+1); node i (0-based) sits at
 *    lo + (i+1) h.  Boxes are C-order [x][y][z] (z fastest), n^3 doubles, and a batch
 *    is [batch][n][n][n].  "Flat index" = (i*n + j)*n + k.
 *  - Point lists are ascending flat indices (int64) (R7).
 */
#ifndef DPM_H_
#define DPM_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  DPM_OK = 0,
  DPM_ERR_INVALID = 1,   /* bad argument: n<4 or n>DPM_MAX_N, lo>=hi, dt<=0, lmax<0, null ptr,
                            domain not strictly inside the box or containing no node      */
  DPM_ERR_OOM = 2,       /* device allocation failed                                       */
  DPM_ERR_CUDA = 3,      /* a CUDA runtime call or kernel launch failed                    */
  DPM_ERR_STATE = 4,     /* projection missing / built at another dt                       */
  DPM_ERR_RANK = 5,      /* K >= |gamma_in| (under-determined BEP) or R singular     */
  DPM_ERR_NONFINITE = 6  /* a PKS step produced a non-finite value                         */
} dpm_status;

#define DPM_MAX_N 520    /* largest n the AP-solve kernels are instantiated for            */

typedef struct { int32_t n; double lo, hi; } dpm_grid;

typedef enum { DPM_SPHERE = 0, DPM_ELLIPSOID = 1 } dpm_domain_kind;
/* Ω = { x : Σ_a ((x_a - center_a)/semi_a)^2 < 1 }  (sphere: semi = (r,r,r), P:596;
   ellipsoid: SURVEY R10).  Must lie strictly inside the box. */
typedef struct { int32_t kind; double center[3]; double semi[3]; } dpm_domain;

/* Extension-operator column sets; K = 2 (lmax+1)^2 columns,
   column c = comp*(lmax+1)^2 + nu, nu = l^2 + l + m (real SH without Condon-Shortley
   phase, R8).  comp 0: Y_nu(foot);  comp 1: d*Y_nu (CAUCHY) or (d^2/2)*Y_nu (NEUMANN0).
   The *_ZONAL sets are the paper's own basis (only the zonal modes
   phi_nu = P_nu^0(cos θ), the unnormalised Legendre polynomial of the foot point's polar
   angle about +z): K = 2 (lmax+1) columns, c = comp*(lmax+1) + l, same comp rule;
   lmax <= DPM_MAX_ZONAL_L (the paper's Test B uses up to 500 harmonics).
   NEUMANN0 is the 3-term extension (beta = 1 in P:263-267) with du/dn = 0;
   the *_2TERM sets are the 2-term extension with du/dn = 0 (beta = 0: pi = u|Γ, the d-term
   vanishes), one component: K = (lmax+1)^2 or (lmax+1) (zonal), c = nu or l.  The
   paper uses it for Test B. */
typedef enum {
  DPM_BASIS_CAUCHY = 0, DPM_BASIS_NEUMANN0 = 1, DPM_BASIS_CAUCHY_ZONAL = 2, DPM_BASIS_NEUMANN0_ZONAL = 3,
  DPM_BASIS_NEUMANN0_2TERM = 4, DPM_BASIS_NEUMANN0_2TERM_ZONAL = 5
} dpm_basis;
#define DPM_MAX_ZONAL_L 1000

/* Point sets of Definition 1. BAND = M- ∩ dil7(gamma) = support of every
   difference-potential right-hand side (R21). NPLUS = N+ restricted to M0. */
typedef enum {
  DPM_SET_MPLUS = 0, DPM_SET_GAMMA = 1, DPM_SET_GAMMA_IN = 2, DPM_SET_GAMMA_EX = 3,
  DPM_SET_BAND = 4, DPM_SET_NPLUS = 5
} dpm_set;

typedef struct {
  int32_t n, K, lmax, basis;
  double h, dt;
  int64_t n_mplus, n_gamma, n_gamma_in, n_gamma_ex, n_band, n_nplus;
  int64_t ghosts_in_nplus;   /* ghost nodes belonging to N+ (R5; 72 at cfg1)              */
  int32_t have_projection;   /* 1 once dpm_build_projection succeeded at the current dt    */
  double bep_cond_est;       /* κ(R) of the column-equilibrated BEP (diag ratio estimate)  */
  int32_t solver;            /* dpm_solver in use                                          */
  int64_t n_exact_ties;      /* nodes within 1e-11 of the boundary in fp64, decided in exact integer
                                arithmetic on the host (R6: the constants read as their shortest
                                round-trip decimals; ties -> M-)                                  */
  int64_t n_exact_ties_inside; /* of those, the nodes placed in M+                                */
} dpm_info;

typedef struct dpm_ctx dpm_ctx;

/* ---------------------------------------------------------------------------------
 * Setup (P:40-60 auxiliary cube + Def. 1; P:263-299 extension data).
 * Builds the point sets on the device (exact classification, ties -> M-, R6: an fp64 test decides
 * every node farther than 1e-11 from the boundary, the rest are decided exactly on the host), the
 * gamma geometry (foot point, signed distance d, SH angles; R10) and E (|gamma| x K).
 * 4 <= n <= DPM_MAX_N; basis one of dpm_basis; 0 <= lmax <= 40 for the full-SH sets,
 * <= DPM_MAX_ZONAL_L for the zonal ones (DPM_ERR_INVALID otherwise).  The paper's mesh
 * (N cells on [-r-2h, r+2h]^3, h = 2r/(N-4)) is n = N, lo = -r-5h/2, hi = r+5h/2.
 * Synchronous (uses an internal stream and waits). *out is NULL on failure.
 * ------------------------------------------------------------------------------- */
dpm_status dpm_create(const dpm_grid* grid, const dpm_domain* domain, int32_t lmax, double dt,
                      int32_t basis, int32_t device, dpm_ctx** out);
void       dpm_destroy(dpm_ctx* ctx);
dpm_status dpm_query(const dpm_ctx* ctx, dpm_info* out);
const char* dpm_last_error(const dpm_ctx* ctx);

/* Copy a point list (ascending flat indices) to HOST memory; cap = capacity in entries;
   DPM_ERR_INVALID if cap is too small. Synchronous. */
dpm_status dpm_copy_set(const dpm_ctx* ctx, int32_t which, int64_t* host_idx, int64_t cap);

/* Copy E (|gamma| x K, column-major) and the signed distances d (|gamma|) to HOST
   memory (either pointer may be NULL). Synchronous. */
dpm_status dpm_copy_extension(const dpm_ctx* ctx, double* host_E, double* host_d);

/* Change dt (the operator is I/dt - Δ_h, R4). Invalidates the projection iff dt changes. */
dpm_status dpm_set_dt(dpm_ctx* ctx, double dt);

/* ---------------------------------------------------------------------------------
 * S3 — the batched AP solve (fast Poisson solver P:166-168):
 *   u_b = (I/dt - Δ_h)^{-1} q_b  on the n^3 interior, zero Dirichlet ghosts,
 * by 3D DST-I, eigenvalue divide (λ_m = (4/h^2) sin^2(m pi/(2(n+1))), R26), inverse
 * 3D DST-I.  q, u: DEVICE [batch][n][n][n]; u may equal q (in place).  batch >= 0.
 * Asynchronous on `stream`.  The same solution by any of the library's exact factorisations of that
 * transform: DST-I along x and y with a tridiagonal solve along z (default), the literal 3D DST-I
 * (dpm_set_solver), and at n = 127 the 8 reflection-parity components solved on the octant
 * (DESIGN.md §6).  The first call at a new n may allocate work space on the device (it synchronises).
 * ------------------------------------------------------------------------------- */
dpm_status dpm_aux_solve_batch(dpm_ctx* ctx, const double* q, double* u, int64_t batch, void* stream);

/* AP solver variant (both give the same u up to rounding):
 *  DPM_SOLVER_DST3          DST-I along x, y and z, eigenvalue divide, inverse along z, y, x.
 *  DPM_SOLVER_DST2_TRIDIAG  DST-I along x and y; each (a,b) line along z solves the tridiagonal
 *                           (1/dt + λ_a + λ_b - D_zz) v = r exactly (constant-coefficient
 *                           factorisation + Sherman-Morrison boundary term); inverse y, x.
 *                           Two fewer transforms per solve.  Default. */
typedef enum { DPM_SOLVER_DST3 = 0, DPM_SOLVER_DST2_TRIDIAG = 1 } dpm_solver;
dpm_status dpm_set_solver(dpm_ctx* ctx, int32_t solver);

/* Same operation through HOST buffers (pinned for overlap; pageable works but serialises): chunks of
   <= 128 MB are uploaded on a ctx-owned copy stream, solved on `stream` and downloaded on a second
   copy stream, double-buffered so upload, solve and download of consecutive chunks overlap.
   Synchronous: returns after host_u is complete. */
dpm_status dpm_aux_solve_batch_host(dpm_ctx* ctx, const double* host_q, double* host_u, int64_t batch,
                                    void* stream);

/* ---------------------------------------------------------------------------------
 * S2 / S4 building blocks (exposed for parity tests and multi-GPU column sharding).
 * dpm_potential_rhs: q_c = χ_{M-} (I/dt - Δ_h)[v_c] for densities v (DEVICE,
 *   |gamma| x nrhs column-major, zero-extended off gamma; Def. DP P:196-207 with R4
 *   scaling) -> q DEVICE [nrhs][n][n][n] (fully written).
 * dpm_trace: out[b][i] = u_b[list[i]] for which = GAMMA or GAMMA_IN.
 * ------------------------------------------------------------------------------- */
dpm_status dpm_potential_rhs(dpm_ctx* ctx, const double* v_gamma, double* q, int32_t nrhs, void* stream);
dpm_status dpm_trace(dpm_ctx* ctx, const double* u, double* out, int32_t which, int64_t batch,
                     void* stream);

/* ---------------------------------------------------------------------------------
 * S2-S5 — boundary projection and reduced BEP (Step 2/4b P:425-431).
 * dpm_bep_columns: for columns c in [c0, c1): u_c = AP(potential_rhs(E_c));
 *   PgE[:, c-c0] = Tr_gamma u_c  (|gamma| x (c1-c0), col-major, DEVICE, nullable);
 *   B[:, c-c0]  = E[gamma_in, c] - Tr_gamma_in u_c  (|gamma_in| x (c1-c0), DEVICE, nullable).
 * dpm_bep_factor: factor B (|gamma_in| x K, DEVICE, col-major; not modified) for least
 *   squares: column equilibration + CholeskyQR2 (Q explicit, R upper). Stored in ctx.
 *   DPM_ERR_RANK if K >= |gamma_in| or the Cholesky breaks down.
 * dpm_build_projection = dpm_bep_columns(0, K) + dpm_bep_factor, B kept in ctx.
 * All asynchronous except dpm_bep_factor / dpm_build_projection (synchronize stream).
 * ------------------------------------------------------------------------------- */
dpm_status dpm_bep_columns(dpm_ctx* ctx, int32_t c0, int32_t c1, double* PgE, double* B, void* stream);
dpm_status dpm_bep_factor(dpm_ctx* ctx, const double* B, void* stream);
dpm_status dpm_build_projection(dpm_ctx* ctx, double* PgE, double* B, void* stream);

/* S8 — least squares for the spectral coefficients (Step 5 P:433):
 * coef = argmin || B coef - g ||_2 for each of nrhs right-hand sides.
 * g: DEVICE |gamma_in| x nrhs col-major; coef: DEVICE K x nrhs; u_gamma (nullable):
 * DEVICE |gamma| x nrhs = E coef (extension operator), not clamped.
 * DPM_ERR_STATE if no projection at the current dt. Asynchronous. */
dpm_status dpm_boundary_lsq(dpm_ctx* ctx, const double* g, double* coef, double* u_gamma, int32_t nrhs,
                            void* stream);

/* ---------------------------------------------------------------------------------
 * PKS time stepping (P:88-141 scheme; Steps 1-8 P:420-437; readings R13-R20).
 * Fields rho (cell averages) and c: DEVICE [n][n][n], meaningful on N+ ∩ M0 and 0
 * elsewhere (ghost nodes of N+ hold 0, R5).
 * ------------------------------------------------------------------------------- */
typedef struct {
  double center[3];        /* Gaussian centre                                    */
  double rho_amp, rho_rate;/* rho0 = rho_amp * exp(-rho_rate |x - center|^2)      */
  double c_amp, c_rate;    /* c0   = c_amp   * exp(-c_rate   |x - center|^2)      */
  int32_t rho_cell_average;/* 1: rho-bar on M+ \ gamma is the cell average of rho0 over
                              [x - h/2, x + h/2]^3 (the paper evolves cell averages, P:86;
                              R36), in closed form via erf; 0: node values (R14)         */
} dpm_pks_ic;

typedef struct {
  double chi;              /* chemotactic sensitivity (R27: 1)                   */
  double dt_cap;           /* configured dt                                      */
  int32_t dt_rule;         /* 0: dt_i = min(dt_{i-1}, dt_cap, CFL, h^2/2) (R13); 1: fixed dt_cap */
  int32_t clamp;           /* 1: u_gamma = max(u_gamma, 0) (R17)                  */
  int32_t coupling;        /* 0: the printed IMEX step (the c equation uses rho-bar^i);
                              1: sequential, the c equation uses rho-bar^{i+1} (an alternative
                              reading probed against Table 4)           */
} dpm_pks_params;

typedef struct {
  double t, dt, mass, rho_max, rho_min, c_min;  /* mass = h^3 Σ_{M+} rho (R18)   */
  int32_t rebuilt;                              /* 1 if Step 4b rebuilt the BEP  */
  int32_t step;
  double rho_max_mplus;   /* max of rho over M+: the paper's ||rho||_inf (eq. sd-norm:max);
                             rho_max above is over N+ (includes gamma_ex) */
  double clamp_max;       /* max over gamma and both fields of max(-u_gamma, 0) before the clamp of R17
                             (how far the reconstructed density went negative; NaN with coupling = 1) */
  double lsq_resid;       /* BEP least-squares residual of the step, max over rho and c of
                             ||B C - g||_2 / ||g||_2 (NaN with coupling = 1) */
} dpm_step_log;

/* Initial state (R14): IC at the node on M+\gamma (or, for rho with ic->rho_cell_average, its
   cell average there, R36), at the foot point on gamma, 0 elsewhere.
   Resets t and the dt history. Asynchronous. */
dpm_status dpm_pks_init(dpm_ctx* ctx, double* rho, double* c, const dpm_pks_ic* ic, void* stream);

/* The paper's per-step diagnostics of a state, HOST out[3] = {mass h^3 Σ_{M+} rho (R18),
   second moment M_h = h^3 Σ_{M+} |x - center|^2 rho (eq. sd-norm:second-moment), free energy
   E_h = h^3 Σ_{M+} {rho ln rho - rho c + c^2/2 + [(c_{j+1}-c_{j-1})^2 + (c_{k+1}-c_{k-1})^2 +
   (c_{l+1}-c_{l-1})^2]/(8h^2)} (eq. sd-norm:free-energy)}; rho ln rho := 0 for rho <= 0, c = 0 on the
   ghost layer, |x - center| from the domain centre (R35).  rho, c: device [n][n][n].  Synchronizes
   `stream`.  Single-domain contexts (DPM_ERR_INVALID for octants). */
dpm_status dpm_pks_diagnostics(dpm_ctx* ctx, const double* rho, const double* c, double* out, void* stream);

/* Advance nsteps steps in place (Steps 3-7).  Each step: flux + IMEX RHS ->
   2 particular AP solves -> Tr_gamma_in -> LSQ -> u_gamma = E C, clamp (R17) -> combined Green's-formula
   RHS (R20) -> 2 AP solves -> restriction to N+.
   Step 3 (R13) runs speculatively: up to 10 consecutive steps at dt_i = dt_{i-1} are replayed as one
   CUDA graph on a ctx-owned stream; every step also evaluates the dt rule on the device from its own
   input state.  From the first step whose rule asks for a smaller dt (or whose state went non-finite)
   on, the graph leaves (rho, c) unchanged (a device flag), so the state is that step's input; the host
   reads the batch's log once, rebuilds the BEP at the new dt (Step 4b) and stepping resumes.  The accepted dt sequence equals the host rule's.  The
   first step of a run evaluates the rule on the host.  The caller's `stream` is synchronized on entry
   and the call returns after the last step (synchronous).  log (HOST, nullable) receives nsteps
   entries.  DPM_ERR_NONFINITE on NaN/Inf (the state is left right after the failing step). */
dpm_status dpm_pks_step(dpm_ctx* ctx, double* rho, double* c, int32_t nsteps, const dpm_pks_params* params,
                        dpm_step_log* log, void* stream);

/* ---------------------------------------------------------------------------------
 * Config 5: octant domain decomposition (the paper's DD: coupled BEPs sharing
 * the interface Cauchy data P:477-480; duplicated equations + averaged effective density at
 * points near several pieces, Case 2 P:562-571; octant pieces, bases and rules: SURVEY R24,
 * R25, R31, listed in DESIGN.md §3).  One context per octant subdomain s (0..7, sign bits
 * s = 4[σx<0] + 2[σy<0] + [σz<0]) in its canonical frame: grid = the box [lo, hi]^3 (cfg5:
 * [-0.1, 1.1]^3), Ω_s = open octant ∩ ball(radius); physical coordinates x = σ ⊙ p.
 * K = 2 (lmax_cap+1)^2 + 6 nφ global unknowns, nφ = (deg_if+1)(deg_if+2)/2:
 *   [cap Y_ν | cap (d^2/2) Y_ν | plane x: φ, x φ | plane y: φ, y φ | plane z: φ, z φ],
 *   φ_jk = P_j(s) P_k(t) (Legendre, j + k <= deg_if, by total degree then j descending),
 *   (s, t) = the other two physical coordinates in axis order.
 * The global least squares (all octants' BEP rows stacked, columns equilibrated) is a
 * distributed CholeskyQR2; the caller sums, over all octants (NCCL all-reduce across ranks):
 *   colnorm2 -> gram(pass 1) -> chol(1) -> gram(2) -> chol(2)    (once per dt)
 *   per step: local_begin gives y_s (K x 2); C = Σ_s y_s; local_finish(C).
 * All pointers are DEVICE unless stated; all calls are on `stream`; "synchronous" ones say so.
 * ------------------------------------------------------------------------------- */
dpm_status dpm_create_octant(const dpm_grid* grid, int32_t octant, double radius, int32_t lmax_cap,
                             int32_t deg_if, double dt, int32_t device, dpm_ctx** out);
/* NEXT-3 — the paper's own two-subdomain DD, Case 1 (Z ∩ Γ = ∅, numerical setup P:594-641):
 * Ω = ball of radius r2 at the origin split by the interface Z = {|x| = r1} into Ω1 = ball r1 (sub = 0)
 * and Ω2 = shell r1 < |x| < r2 (sub = 1), each on its own grid (the paper's "N1/N2" meshes, P:627:
 * n = N_l, h_l = 2 r_l/(N_l - 4), lo = -r_l - 5h_l/2).  Pieces: Z (piece 0, assignment bit 1) and Γ
 * (piece 1, bit 2); Ω1's discrete boundary ζ1 is all Z, a point of Ω2's γ ∪ ζ2 is on the nearer sphere
 * (R38).  Global unknowns, K = 3 (mz+1) + 2 (mg+1), zonal basis φ_l = P_l(cos θ):
 *   [Z: φ | d φ | (d²/2) φ, d = |x| - r1 — the interface Cauchy data u, ∂_n u, ∂²_n u shared by both
 *    subdomains (interface conditions P:477-480) | Γ: φ | (d²/2) φ, d = |x| - r2 (zero Neumann)].
 * The returned context is a DD subdomain: every dpm_dd_* call below applies (BEP rows on ζ1,in or
 * γ_in ∪ ζ2,in: the reduced BEPs eqn:reduced_DD1_BEP1/2; the stacked least squares over both
 * subdomains by the same distributed CholeskyQR2, summed over the two contexts).  dpm_dd_pks_init (R38):
 * the IC at the node on N+, at the foot r2 x/|x| on Γ's points (R14); with rho_cell_average the cell
 * average (R36) of ρ on M+ and on the interface points.  DPM_ERR_INVALID on bad arguments or a box that
 * does not strictly contain the subdomain. */
dpm_status dpm_create_dd1(const dpm_grid* grid, int32_t sub, double r1, double r2, int32_t mz, int32_t mg, double dt,
                          int32_t device, dpm_ctx** out);
/* n_rows = BEP rows of this subdomain (γ_in points x their pieces), K = global unknowns (HOST). */
dpm_status dpm_dd_info(const dpm_ctx* ctx, int64_t* n_rows, int32_t* K);
/* HOST [n_gamma] piece bits of every γ point (1 cap, 2 x-plane, 4 y-plane, 8 z-plane). */
dpm_status dpm_dd_copy_assign(const dpm_ctx* ctx, uint8_t* host_bits);
/* K AP solves of the potentials of the effective density columns at the ctx's dt, then the
   BEP block B_s (n_rows x K column-major, kept in ctx; copied to B_out if non-NULL). */
dpm_status dpm_dd_bep_block(dpm_ctx* ctx, double* B_out, void* stream);
/* Config 5 (R24): the BEP block of octant ctx from the already built block of another octant `ref` of the
   same canonical geometry on the same device, B_s = B_ref diag(S) with S the column signs of ctx's extension
   relative to ref's (E_s = E_ref diag(S): every cap SH and plane Legendre function is even or odd under each
   reflection, and the K AP solves of P:241-253 are linear in their right-hand sides), instead of K AP solves.
   ref must hold its block at ctx's dt (dpm_dd_bep_block).  DPM_ERR_INVALID if the contexts are not octants of
   one geometry on one device or the extensions are not sign reflections; DPM_ERR_STATE if ref has no block at
   this dt.  Asynchronous on stream (the first call per pair synchronizes it once to check the signs). */
dpm_status dpm_dd_bep_block_from(dpm_ctx* ctx, dpm_ctx* ref, double* B_out, void* stream);
/* nrm2[c] = Σ_rows B_s[:, c]^2 (K). */
dpm_status dpm_dd_colnorm2(dpm_ctx* ctx, double* nrm2, void* stream);
/* pass 1: D = 1/sqrt(nrm2_sum) (synchronizes), Q1 = B_s D, G = Q1^T Q1;  pass 2: G = Q1^T Q1
   with the pass-1 Q1.  G: K x K (upper triangle valid). */
dpm_status dpm_dd_gram(dpm_ctx* ctx, int32_t pass, const double* nrm2_sum, double* G, void* stream);
/* Cholesky of the summed Gram (pass 1: R1, Q1 <- Q1 R1^{-1}; pass 2: R2, Q <- Q1 R2^{-1},
   R = R2 R1, M_s = D R^{-1} Q^T).  Synchronous; DPM_ERR_RANK on breakdown. */
dpm_status dpm_dd_chol(dpm_ctx* ctx, int32_t pass, const double* G_sum, void* stream);
/* The same pass for another octant of the SAME device and K whose dpm_dd_chol(pass) with the same
   G_sum has completed (src): copies the K x K factors and their inverses from src instead of
   refactoring, then forms this octant's Q (and, pass 2, M_s).  Asynchronous on stream.
   DPM_ERR_INVALID for a src on another device / with another K; DPM_ERR_STATE (pass 2) if src has
   no projection. */
dpm_status dpm_dd_chol_copy(dpm_ctx* ctx, int32_t pass, const dpm_ctx* src, void* stream);
/* R31 initial state (rho, c on N+, [n][n][n]). */
dpm_status dpm_dd_pks_init(dpm_ctx* ctx, double* rho, double* c, const dpm_pks_ic* ic, void* stream);
/* Local CFL bound h / (6 χ max|Δc|/h) (R19) -> *cfl_dt (HOST).  Synchronous; with
   cfl_dt == NULL it only enqueues the reduction and dpm_dd_cfl_result() (synchronous) returns it. */
dpm_status dpm_dd_cfl(dpm_ctx* ctx, const double* c, double chi, double* cfl_dt, void* stream);
dpm_status dpm_dd_cfl_result(dpm_ctx* ctx, double chi, double* cfl_dt, void* stream);
/* Step 4a-5 at the ctx's dt (the factorisation must be at this dt): flux + IMEX RHS, particular
   solves, BEP right-hand sides on the rows, y = M_s g (K x 2, field-major). */
dpm_status dpm_dd_local_begin(dpm_ctx* ctx, const double* rho, const double* c, double chi, double* y,
                              void* stream);
/* Steps 5-7 with the global C (K x 2): u_γ = A C (clamped at 0 if clamp, R17), Green's formula
   (R20), restriction to N+.  stats (HOST, 6): [h^3 Σ_{M+} ρ, max ρ over N+, min ρ, min c, nonfinite,
   max ρ over M+ (the paper's ||ρ||_inf, eq. dd-norm:max)]; synchronous when stats != NULL, otherwise
   asynchronous and dpm_dd_stats() (synchronous, the same 6 values) reads them. */
dpm_status dpm_dd_local_finish(dpm_ctx* ctx, const double* C, int32_t clamp, double* rho, double* c,
                               double* stats, void* stream);
dpm_status dpm_dd_stats(dpm_ctx* ctx, double* stats, void* stream);
/* The same step in phases over CALLER-OWNED 2-field buffers ([2][n][n][n] fp64, DEVICE), so that a
   rank runs each of the step's two AP solves for all its octants as one dpm_aux_solve_batch (the AP
   operator depends only on n, h, dt, which the octants share):
     dpm_dd_local_begin  = dpm_dd_rhs -> dpm_aux_solve_batch(fq -> wk) -> dpm_dd_lsq_rhs
     dpm_dd_local_finish = dpm_dd_green_rhs -> dpm_aux_solve_batch(wk, in place) -> dpm_dd_restrict
   dpm_dd_rhs: fq = the scaled IMEX RHS of Step 4a (R15, R16); DPM_ERR_STATE without a
   factorisation at the ctx's dt.  dpm_dd_lsq_rhs: BEP rows of the AP solutions wk, y = M_s g_s (K x 2).
   dpm_dd_green_rhs: u_γ = A C (clamped if clamp, R17), Green RHS from fq and u_γ into wk (R20).
   dpm_dd_restrict: restriction of the Green solutions wk to N+ into rho, c with the step statistics
   (read by dpm_dd_stats).  All asynchronous on stream. */
dpm_status dpm_dd_rhs(dpm_ctx* ctx, const double* rho, const double* c, double chi, double* fq, void* stream);
dpm_status dpm_dd_lsq_rhs(dpm_ctx* ctx, const double* wk, double* y, void* stream);
dpm_status dpm_dd_green_rhs(dpm_ctx* ctx, const double* C, int32_t clamp, const double* fq, double* wk,
                            void* stream);
/* dpm_dd_lsq_rhs over `noct` config-5 octant contexts of ONE device at once, summed: y = Σ_s M_s g_s (K x 2,
   DEVICE), the local contribution to C (the caller all-reduces it across ranks as the per-octant y_s).
   The octants share one canonical geometry, so B_s = B_0 diag(S_s) (their extensions differ only by
   column signs S_s, read off the extension matrices and required to be exactly ±1), hence
   Q_s = Q_0 R S_s R^{-1} and  y = D R^{-1} R^{-T} Σ_s S_s R^T (Q_0^T g_s):  one pass over octs[0]'s Q for all
   2 noct right-hand sides instead of one operator M_s per octant, then K x K products (same result up
   to rounding, ~κ(R) ε).  wk: DEVICE [noct][2][n^3], the particular solutions in the order of `octs`.
   DPM_ERR_INVALID if the contexts are not octants of one geometry on one device (same n, box, radius, K,
   rows) or their extensions are not sign reflections; DPM_ERR_STATE without a factorisation.
   Asynchronous on stream (the first call per octant pair synchronizes it once to check the signs). */
dpm_status dpm_dd_lsq_rhs_shared(dpm_ctx* const* octs, int32_t noct, const double* wk, double* y, void* stream);
/* dpm_dd_green_rhs for `noct` (<= 8) config-5 octant contexts of ONE device at once: the extension
   u_γ,s = A_s C (R17, clamped when clamp) of every octant from ONE evaluation of the basis per γ point,
   then each octant's combined Green RHS (R20).  The octants share one canonical geometry and A_s evaluates
   the basis at x = σ_s ⊙ p, where every cap SH and plane Legendre function is even or odd in each axis,
   so A_s = A_0 diag(S_s) with S_s(ν) = (-1)^{popcount(s & π(ν))} (π(ν) the 3-bit parity class, s the
   octant index): the basis terms are summed per parity class and an 8-point Walsh-Hadamard transform
   gives every octant (same values as dpm_dd_green_rhs up to the summation order).  C: DEVICE [2][K]
   (the global coefficients); fq, wk: DEVICE [noct][2][n^3] in the order of `octs`; wk == fq forms the
   right-hand sides in place (fq is zero off M+ after dpm_dd_rhs and the band never meets M+, so only the
   band values are written).  DPM_ERR_INVALID if
   the contexts are not octants of one geometry on one device.  Asynchronous on stream. */
dpm_status dpm_dd_green_rhs_shared(dpm_ctx* const* octs, int32_t noct, const double* C, int32_t clamp,
                                   const double* fq, double* wk, void* stream);
dpm_status dpm_dd_restrict(dpm_ctx* ctx, const double* wk, double* rho, double* c, void* stream);

/* Cumulative number of CUDA kernels this library has launched in the process (all
   contexts).  Lets a harness count the library's launches inside a timed region. */
int64_t dpm_launch_count(void);

/* Measurement hooks (bench.py's per-kernel roofline).  While enabled, every pass of
 * dpm_aux_solve_batch is bracketed by two CUDA events recorded on the caller's stream.
 * dpm_pass_times synchronizes those events and returns, per pass kind k (0: transform along x,
 * 1: transform along y, or the fused y / z / y plane pass at n = 128, 2: tridiagonal / transform
 * along z), the summed duration ms[k] (HOST,
 * milliseconds), the number of launches[k] and the grid points processed points[k] since the
 * last call (or since enabling), then resets.  Synchronous; DPM_ERR_INVALID on null pointers. */
dpm_status dpm_set_pass_timing(dpm_ctx* ctx, int32_t enable);
dpm_status dpm_pass_times(dpm_ctx* ctx, double* ms, int64_t* launches, int64_t* points);

#ifdef __cplusplus
}
#endif
#endif /* DPM_H_ */
