/*
 * lrbms.h -- C ABI of the B200-native LRBMS online step (arXiv 1405.2810).
 *
 * One time step of the Localized Reduced Basis Multiscale two-phase scheme,
 * alg:fullTwoPhaseScheme, with the fine mobility lambda(s^n)
 * itself as the parameter (direct online projection; reading R3):
 *
 *   a1  lambda_i, f_i from s_i          eq:brooksCorey P:183-186, eq:frationalFlow P:201-206
 *   a2  B_EE' = Phi_E^T A_EE'(lambda) Phi_E', r_E = Phi_E^T b(lambda)
 *                                        def:coarseScalePressure P:621-631 (k = 0 SWIP, R1/R2)
 *   a3  solve B c = r                    eq:reducedSystem P:818-821 (exact-solve reading A17)
 *   a4  p = sum_E Phi_E c_E
 *   a5  face fluxes + CFL time step      eq:velocityDG P:366-377 (k = 0), reading R4
 *   a6  explicit upwind transport        eq:saturationDG P:389-399, eq:upwind P:400-417
 *
 * Beside the online step: the paper's affine online variant (theta fit + sum_q theta_q b_q:
 * lrbms_set_profiles / lrbms_set_online), the fine-scale reference scheme (lrbms_run_fine), the offline
 * basis recipe on the GPU (lrbms_offline_basis), the K6 diagnostics (lrbms_diagnostics) and the online
 * step on the k = 1 SWIP-DG fine space with the P1 transport and the limiter (lrbms_k1_*).
 *
 * Everything is fp64 on one GPU (sm_100a).  The fine grid is a structured
 * Cartesian grid of nx*ny*nz cells, x fastest (cell c = i + nx*(j + ny*k),
 * P:245-262); the coarse partition is matching: subdomains of
 * sx*sy*sz cells, E = I + Sx*(J + Sy*L), local cell l = lx + sx*(ly + sy*lz).
 *
 * Conventions
 *  - Memory: the library never allocates device memory.  The caller (PyTorch in
 *    the Python binding) owns one workspace of lrbms_workspace_bytes() bytes and
 *    passes it to lrbms_bind().  All device work is enqueued on the bound stream.
 *  - (dev) marks device pointers, (host) host pointers.  set_* calls copy their
 *    inputs stream-ordered into the workspace; callers may free the inputs once
 *    the stream has synchronised.
 *  - Errors: no C++ exception crosses the ABI.  Every call returns a status and
 *    lrbms_last_error() explains it.  CONFIG = invalid sizes/inputs; NUMERICAL =
 *    non-positive pivot / breakdown, non-converged reduced solve, no flow, NaN
 *    (device-detected, reported at the end of lrbms_run); CUDA = a CUDA runtime
 *    error (the context is poisoned: every later call returns LRBMS_E_CUDA);
 *    STATE = a call out of order (e.g. run before bind / set_*).
 *  - A context is not thread-safe; separate contexts are independent.
 */
#ifndef LRBMS_H
#define LRBMS_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct lrbms_ctx lrbms_ctx;

typedef enum {
  LRBMS_OK = 0,
  LRBMS_E_CONFIG = 2,
  LRBMS_E_NUMERICAL = 3,
  LRBMS_E_IO = 4,
  LRBMS_E_CUDA = 5,
  LRBMS_E_STATE = 6
} lrbms_status;

/* Fine grid + coarse partition + local basis size.
 * dim = 2 requires nz = sz = 1.  sx | nx, sy | ny, sz | nz.  1 <= N <= 32; the k = 0 basis
 * (lrbms_set_basis) needs N <= sx*sy*sz, the k = 1 basis (lrbms_k1_set_basis) N <= (dim + 1) sx*sy*sz.
 * hx, hy, hz > 0 are the cell widths (|F|/d_F and the cell volume follow from them). */
typedef struct {
  int32_t dim, nx, ny, nz;
  double hx, hy, hz;
  int32_t sx, sy, sz;
  int32_t N;
} lrbms_grid;

/* Fluids (eq:brooksCorey P:183-189; reading R5): k_rw = S_e^nw, k_ro = (1 - S_e)^no,
 * S_e = clamp((s - swr)/(1 - swr - sor), 0, 1); lambda_w = k_rw/mu_w, lambda_o = k_ro/mu_o.
 * nw = no = 1 is the paper's linear law; BASELINE.json's configs use 2. */
typedef struct {
  double mu_w, mu_o, swr, sor, nw, no;
} lrbms_fluid;

/* Boundary data as links (reading R6/A13): a Dirichlet boundary face or a
 * well cell.  Link L couples fine cell cell[L] to the fixed pressure p[L] through the
 * face normal to axis[L] (0,1,2) at distance h/2: g_L = 2 |F|/h_axis * K_cell * lambda_cell.
 * s_ext[L] is the saturation entering through the link on inflow (eq:upwind P:405-406).
 * All arrays (host), n_links entries, copied at create.  Faces without a link are no-flow.
 * At least one link is required (otherwise A(lambda) is singular). */
typedef struct {
  int32_t n_links;
  const int32_t *cell;
  const int32_t *axis;
  const double *p;
  const double *s_ext;
} lrbms_links;

/* Reduced-solve options (a3).  The solve is preconditioned CG on the block-Jacobi-scaled system
 * L^-1 B L^-T y = L^-1 r (B_EE = L_E L_E^T) with a coarse level on the subdomain-indicator
 * coefficients (Galerkin coarse operator E = Z^T B Z), started from the B-optimal combination of the
 * last `history` solutions (Galerkin projection onto their span), iterated until the preconditioned
 * residual sqrt(rh.M^-1 rh) of the scaled system is <= rtol ||L^-1 r||_2 (rh = L^-1 (r - B c); an
 * energy-norm error proxy).  Coarse level: use_coarse = 2 (default) deflation (A-DEF2, P^T + Q, with
 * the DEF starting vector), whose coarse inverse is refreshed every coarse_refresh steps and kept
 * current in between by one Newton-Schulz correction per step; 1 = additive (I + Q; the inverse is
 * only refreshed every coarse_refresh steps); 0 = block Jacobi only. */
typedef struct {
  double rtol;            /* default 5e-13, on sqrt(r.M^-1 r) relative to ||L^-1 b|| */
  int32_t max_iters;      /* default 5000 */
  int32_t coarse_refresh; /* full coarse inverse every k steps (default 200; 1 = every step) */
  int32_t use_coarse;     /* 2 (default) = deflation, 1 = additive two-level, 0 = block Jacobi only */
  int32_t history;        /* previous solutions in the initial-guess projection, 0..8 (default 8) */
  int32_t onchip;         /* 1 (default): keep the scaled reduced operator on chip for the whole solve
                             (couplings in tensor memory / shared memory, one warp per subdomain) when
                             n_s <= 14 x SMs; 0: stream the couplings from L2 every iteration */
} lrbms_solver_opts;

typedef struct {
  int64_t steps;          /* steps taken since set_saturation */
  double t;               /* simulated time sum(dt) */
  double last_dt;
  int32_t last_iters;     /* PCG iterations of the last step */
  int64_t total_iters;    /* PCG iterations since set_saturation */
  int32_t coarse_rebuilds;
  double fprime_max;      /* max f_w'(s) used by the CFL step */
  int64_t ns_guard_trips; /* calls in which a Newton-Schulz update of the coarse inverse was dropped
                             because max|I - E X| reached 1; the inverse is then rebuilt on the device in
                             the same step (fp32 Gauss-Jordan), or, where that kernel cannot hold the
                             matrix, the call continues as block-Jacobi PCG and rebuilds at the next call */
  double ns_resid_max;    /* max_ij |(I - E X)_ij| of the last Newton-Schulz update (0 if none ran) */
} lrbms_stats;

/* Create a context (host only; no device work).  Validates the configuration. */
lrbms_status lrbms_create(const lrbms_grid *grid, const lrbms_fluid *fluid,
                          const lrbms_links *links, lrbms_ctx **out);
/* Bytes of device workspace the context needs (256-byte aligned). */
size_t lrbms_workspace_bytes(const lrbms_ctx *ctx);
/* Bind the caller-owned device workspace (>= lrbms_workspace_bytes) and a CUDA stream
 * (cudaStream_t passed as void*; NULL = legacy default stream). */
lrbms_status lrbms_bind(lrbms_ctx *ctx, void *workspace, size_t bytes, void *stream);
/* Permeability K (dev, n, natural cell order, > 0) and porosity phi (dev, n, > 0) or NULL (= 1). */
lrbms_status lrbms_set_medium(lrbms_ctx *ctx, const double *K, const double *phi);
/* Local reduced bases Phi (dev, [n_s][N][n_loc]: basis function k of subdomain E at local
 * cell l).  Each Phi_E must have full column rank (B must be SPD). */
lrbms_status lrbms_set_basis(lrbms_ctx *ctx, const double *Phi);
/* Saturation s^0 (dev, n, natural order); resets time, step count and the warm start. */
lrbms_status lrbms_set_saturation(lrbms_ctx *ctx, const double *s);
lrbms_status lrbms_set_solver(lrbms_ctx *ctx, const lrbms_solver_opts *opts);

/* NEXT-1, the paper's affine online variant of step a2 (eq:parameterizedMob P:570-589,
 * eq:leastSquaresFit P:581-586, sec:offlineOnlineDecomposition P:784-813, eq:reducedSystem
 * P:818-821): the reduced system of a step is sum_q theta_q b_q, sum_q theta_q d_q with theta the
 * least-squares fit of lambda_t(s^n) by M mobility profiles (normal equations; a profile that depends
 * on the previous ones is dropped), and b_q, d_q the projections of the operator and right-hand side
 * of profile q (c = e = 0 under reading R2).  The fluxes keep the true lambda(s^n).
 *
 * lrbms_profiles_bytes: size of the caller-owned profile workspace for M profiles (0 if M is not in
 * [1, 16]).  lrbms_set_profiles: s_profiles (dev, [M][n], natural order) are the SATURATION fields of
 * the profiles (the library evaluates lambda_t of them itself); ws (dev, 256-byte aligned, >= the
 * size above) stays owned by the caller and must outlive the context's use of the affine variant.
 * Computes lambda_q, b_q, d_q (M projections) and the Gram matrix once; synchronises the stream.
 * Needs set_medium and set_basis.  Errors: CONFIG (M, NULL, small or misaligned workspace), STATE.
 * lrbms_set_online: 1 = affine variant (needs set_profiles), 0 = direct projection (default).
 * lrbms_stage_theta: theta of the current saturation (dev, M doubles); a test hook. */
size_t       lrbms_profiles_bytes(const lrbms_ctx *ctx, int32_t M);
lrbms_status lrbms_set_profiles(lrbms_ctx *ctx, const double *s_profiles, int32_t M, void *ws,
                                size_t bytes);
lrbms_status lrbms_set_online(lrbms_ctx *ctx, int32_t affine);
lrbms_status lrbms_stage_theta(lrbms_ctx *ctx, double *theta);

/* NEXT-2: the fine-scale reference scheme on the GPU -- alg:highDimTwoPhaseFlow
 * at k = 0, i.e. the online step with Phi_E = I: per step the fine pressure
 * system of def:pressureDG, A(lambda) p = b(lambda) with A = sum_F w_F (e_a - e_b)
 * (e_a - e_b)^T + sum_L g_L e_a e_a^T and b = sum_L g_L p_L e_a (reading R2 weights), solved by a
 * CG (cooperative kernel, deterministic reductions) preconditioned by Jacobi plus an additive coarse
 * correction on the subdomain indicators (E = Z^T A Z inverted each step by the reduced solver's
 * Gauss-Jordan kernel, when that kernel fits the configuration), warm-started from the current
 * pressure and stopped when r.M^-1 r <= rtol^2 b.D^-1 b; then the same fluxes, CFL step
 * and upwind transport as lrbms_run.  The paper's comparison run (speed-up).
 *
 * lrbms_fine_bytes: size of the caller-owned fine workspace (10 n doubles + 2 n bytes + the coarse
 * stencil and its fp32 inverse, n_pad^2 floats + scratch).
 * lrbms_run_fine: n_steps, cfl, dt_fixed, dt_log as lrbms_run; ws (dev, 256-byte aligned, >= the
 * size above, owned by the caller, used only during the call); rtol > 0, max_iters > 0 per solve;
 * iters_total (host, NULL = skip) receives the CG iterations summed over the steps.  Needs
 * set_medium and set_saturation (not set_basis); the pressure of the last step is what
 * lrbms_get_state returns afterwards.  The reduced solver's history is not updated.  Errors: CONFIG
 * (arguments, workspace), STATE, NUMERICAL (non-convergence within max_iters, breakdown, NaN,
 * no flow), CUDA.  Synchronises the stream once at the end. */
size_t       lrbms_fine_bytes(const lrbms_ctx *ctx);
lrbms_status lrbms_run_fine(lrbms_ctx *ctx, int32_t n_steps, double cfl, double dt_fixed,
                            double *dt_log, void *ws, size_t bytes, double rtol, int32_t max_iters,
                            int64_t *iters_total);

/* NEXT-3: the offline basis recipe on the GPU -- the initialisation of
 * alg:lrbmsBasisConstruction, the training set, the fine snapshots
 * and the per-subdomain data compression (PCA) with the coarse unit functions
 * (P:1110-1111).  Its host reference is offline/recipe.py (readings A31/A32):
 *   1. the fine pressure at the current saturation s0 (the NEXT-2 solver, rtol) and the CFL step dt0 of
 *      its fluxes (reading R4, f'_max of the context's fluid);
 *   2. the time of flight of eq:timeOfFlight at k = 0 (upwind DG0; solved by relaxation
 *      sweeps to the exact fixed point of the flow-ordered triangular system);
 *   3. M mobility profiles: q = 1 the mobility of s0, q = M that of the injected saturation
 *      (the largest link s_ext), q = 2..M-1 the injected one where tau <= (q-1) T/(M-2), T = horizon_steps dt0;
 *   4. n_train fine snapshots p(lambda^(j)), lambda^(j) = sum_q mu_q lambda_{t,q};
 *   5. per subdomain E: Y = (I - v0 v0^T) P|_E (v0 = 1/sqrt(n_loc)), its thin SVD (one-sided Jacobi),
 *      Phi_E = [v0, the left singular vectors with sigma > eps_pca sigma_max (sigma_max over all E), at
 *      most N - 1 of them, then graded monomials of the local coordinates orthogonalised against the
 *      columns before them], each column signed so that its largest-magnitude entry is positive.
 * mu (host, [n_train][M], row-major): the training parameters (the caller's seeded sampler).
 * ws (dev, 256-byte aligned, >= lrbms_offline_bytes(ctx, n_train)): caller-owned scratch, used only
 * during the call (C5 with n_train = 64: ~0.7 GB).  Outputs: Phi (dev, [n_s][N][n_loc], the layout of
 * lrbms_set_basis; not installed -- call lrbms_set_basis with it), tau (dev, n, natural order, or
 * NULL), snapshots (dev, [n_train][n], natural order, or NULL), kept (host, n_s: POD modes kept, or
 * NULL), info (host, or NULL).  The pressure buffer is overwritten; the reduced solver rebuilds its
 * coarse inverse at its next step.  Errors: CONFIG (arguments, workspace, M not in [3, 16], n_train
 * not in [1, 64], a subdomain that cannot be completed to N), STATE (no medium or saturation),
 * NUMERICAL (no flow, a fine solve that does not converge, a flow cycle in the time of flight). */
typedef struct {
  double dt0;             /* CFL step of the s0 flow */
  double horizon;         /* T = horizon_steps * dt0 */
  int32_t tof_sweeps;     /* relaxation sweeps of the time of flight */
  int64_t fine_cg_iters;  /* CG iterations of the 1 + n_train fine solves */
} lrbms_offline_info;
size_t       lrbms_offline_bytes(const lrbms_ctx *ctx, int32_t n_train);
lrbms_status lrbms_offline_basis(lrbms_ctx *ctx, int32_t M, int32_t n_train, const double *mu,
                                 int32_t horizon_steps, double cfl, double eps_pca, double rtol, void *ws,
                                 size_t bytes, double *Phi, double *tau, double *snapshots, int32_t *kept,
                                 lrbms_offline_info *info);

/* NEXT-4: the online step on the k = 1 SWIP-DG fine space -- the paper's (inferred) fine
 * discretisation: pressure eq:swipBilP P:295-303 with the penalty eq:penaltyParam P:305-310 made
 * lambda-free by the Remark P:312-320 (sigma_F = c_F / max(mu_w, mu_n) * 2 K_1 K_2 / (K_1 + K_2), h_F =
 * diam(F)); velocity: the normal fluxes of eq:velocityDG P:366-377; saturation: eq:saturationDG
 * P:389-399 with eq:upwind P:400-417 (explicit Euler, two-point Gauss per direction); the limiter of
 * P:419-469 (shock detector, flagging, gradient scales, eq:limiterMain); the reduced pressure
 * def:coarseScalePressure P:621-631 on the P1 dofs with the mobility of the cell means.  Readings A4, A5,
 * A25-A30.
 * Dofs of a cell: the coefficients of 1 and of (x_a - centre_a) / h_a, a = 1..dim; P1 fields are
 * [dim + 1][n] (dof-major, natural cell order).  Phi1 (dev): [n_s][N][(dim + 1) n_loc], entry
 * a n_loc + l = dof a of local cell l; full row rank per subdomain is the caller's duty (a
 * rank-deficient Phi1_E makes the block Cholesky fail: NUMERICAL).
 * ws (dev, 256-byte aligned, >= lrbms_k1_bytes(ctx)): caller-owned, in use until the context is
 * destroyed or lrbms_k1_set_basis is called again; Phi1 is copied into it.  Every link must lie on a
 * domain-boundary face of its axis (they are the Dirichlet faces, A29): CONFIG otherwise.  Needs
 * set_medium; replaces the indicator coefficients of the k = 0 basis (call lrbms_set_basis again
 * before k = 0 steps) and resets the reduced solver's history.  Conversely lrbms_set_medium and
 * lrbms_set_basis invalidate the k = 1 setup (STATE until lrbms_k1_set_basis is called again).
 * lrbms_k1_set_saturation: s1 (dev, [dim + 1][n]).  lrbms_k1_run: as lrbms_run; limiter = 0 skips the
 * limiter.  lrbms_k1_get_state: s1, p1 (dev, [dim + 1][n]), c (dev, n_s N), n_flagged (host: cells the
 * limiter flagged in the last step); NULL = skip.  lrbms_k1_stage_project: the blocks and the
 * right-hand side of the current saturation, in the layout of lrbms_stage_project. */
size_t       lrbms_k1_bytes(const lrbms_ctx *ctx);
lrbms_status lrbms_k1_set_basis(lrbms_ctx *ctx, const double *Phi1, double c_pen, void *ws, size_t bytes);
lrbms_status lrbms_k1_set_saturation(lrbms_ctx *ctx, const double *s1);
lrbms_status lrbms_k1_run(lrbms_ctx *ctx, int32_t n_steps, double cfl, double dt_fixed, int32_t limiter,
                          double *dt_log);
lrbms_status lrbms_k1_get_state(lrbms_ctx *ctx, double *s1, double *p1, double *c, int32_t *n_flagged);
lrbms_status lrbms_k1_stage_project(lrbms_ctx *ctx, double *blocks, double *r);

/* Advance n_steps online steps a1..a6 on the bound stream, no host round trip per step.
 * dt_fixed > 0 overrides the CFL step (the paper's fixed N_T); otherwise
 * dt^n = cfl * min_i phi_i V_i / (f'_max Q_i) (reading R4).  dt_log (dev, n_steps) or NULL.
 * Synchronises the stream once at the end to report device-detected errors. */
lrbms_status lrbms_run(lrbms_ctx *ctx, int32_t n_steps, double cfl, double dt_fixed,
                       double *dt_log);
/* Same, end to end from HOST buffers: copies s_in (host, n, natural order; NULL = keep
 * the current state) to the device, runs, and copies s_out / p_out (host, n; NULL = skip)
 * back.  The call a user without device memory makes. */
lrbms_status lrbms_run_host(lrbms_ctx *ctx, int32_t n_steps, double cfl, double dt_fixed,
                            const double *s_in, double *s_out, double *p_out);
/* Current state (dev pointers, natural cell order; NULL = skip): s (n), p (n, pressure of
 * the last step), c (n_s*N, reduced coefficients of the last step). */
lrbms_status lrbms_get_state(lrbms_ctx *ctx, double *s, double *p, double *c);

/* Per-stage hooks (the same kernels lrbms_run uses), for parity tests.
 * project: a1+a2 at the current s; blocks (dev, [n_s][1+dim][N][N]: the diagonal block,
 *   then the coupling block to E+e_d for d < dim, zero where E has no such neighbour),
 *   r (dev, [n_s][N]); either may be NULL.
 * solve: a3 on the last projected system (warm start = current c); c (dev, [n_s][N]) or NULL.
 * reconstruct: a4 from the current c; p (dev, n, natural order) or NULL.
 * transport: a5+a6 from the current p and s; advances s; face_flux (dev, interior faces in
 *   global order: x-faces, then y, then z, each x fastest), link_flux (dev, n_links),
 *   dt (dev, 1); any may be NULL. */
lrbms_status lrbms_stage_project(lrbms_ctx *ctx, double *blocks, double *r);
lrbms_status lrbms_stage_solve(lrbms_ctx *ctx, double *c);
lrbms_status lrbms_stage_reconstruct(lrbms_ctx *ctx, double *p);
lrbms_status lrbms_stage_transport(lrbms_ctx *ctx, double cfl, double dt_fixed,
                                   double *face_flux, double *link_flux, double *dt);

lrbms_status lrbms_get_stats(lrbms_ctx *ctx, lrbms_stats *out);

/* K6 diagnostics of the last step (off the timed path; one kernel per subdomain + a
 * fixed-order sum, deterministic; synchronises the stream).  Needs a step since set_saturation
 * (STATE otherwise).  zeta is the paper's relative mass loss of the step's velocity,
 * zeta(T) = |int_dT u.n dS| / max_{x in dT} |u(x)|, with u.n on a face or link its
 * flux density F/|F| (A33); 0 for the fine scheme, > 0 for reduced bases.
 * coarse_defect = max_E |sum_{i in E} int_dT_i u.n| (0 when 1_E is in span Phi_E).
 * mass_balance = |mass - mass_prev + dt water_out| / max(mass, mass_prev) (pin P3: round-off). */
typedef struct {
  double mass_prev, mass;      /* sum_i phi_i V_i s_i before / after the last step */
  double s_min, s_max;         /* range of s after the last step */
  double zeta_max, zeta_mean;  /* relative mass loss over the cells */
  double coarse_defect;
  double water_out;            /* sum over links of F_L f(s_up) (water leaving per unit time) */
  double q_in, q_out;          /* total link inflow / outflow rates */
  double dt;                   /* dt of the last step */
  double mass_balance;
} lrbms_diag;
lrbms_status lrbms_diagnostics(lrbms_ctx *ctx, lrbms_diag *out);

/* Per-stage device timing with CUDA events on the bound stream (off by default).
 * Stages: 0 project (a1+a2), 1 coarse-level rebuild, 2 block Cholesky + scaling of the couplings,
 * 3 initial guess from the solution history, 4 PCG (a3), 5 reconstruction (a4), 6 flux + CFL (a5),
 * 7 transport (a6).  Enabling resets the sums. */
#define LRBMS_N_STAGES 8
lrbms_status lrbms_set_profiling(lrbms_ctx *ctx, int32_t enable);
/* ms[i] = accumulated device milliseconds, launches[i] = kernel launches of stage i, i < n. */
lrbms_status lrbms_get_stage_times(lrbms_ctx *ctx, double *ms, int64_t *launches, int32_t n);
/* Number of kernel launches the library enqueued since create (for launch accounting). */
int64_t lrbms_launch_count(const lrbms_ctx *ctx);
const char *lrbms_last_error(const lrbms_ctx *ctx);
const char *lrbms_version(void);
void lrbms_destroy(lrbms_ctx *ctx);

#ifdef __cplusplus
}
#endif
#endif /* LRBMS_H */
