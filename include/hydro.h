/*
 * hydro.h -- C ABI of the B200 corner-force library (libhydro.so).
 *
 * The one data-parallel hot path of arXiv 2104.11404 (Copeland, Cheung, Huynh,
 * Choi, "Reduced order models for Lagrangian hydrodynamics"): the high-order
 * finite-element force F(v, e, x) of the semi-discrete Euler system
 *     M_V dv/dt = -F.1,   M_E de/dt = F^T.v,   dx/dt = v
 * (PAPER.md Eq. fom; F.1 and F^T.v are Eq. forceOneforceTv),
 * the adaptive time-step estimate (Eq. adaptive-timestep), and the
 * hyper-reduced ROM online pieces: lifting (Eq. discretesolrepresentation,
 * P:864-871), sampled force evaluation ("the lifting is computed only for the
 * sampled degrees of freedom") and the least-squares projection
 * (Eq. sol-ls-hyper).  The entries of F are not written in the paper
 * (it defers to Dobrev et al. 2012); R1-R26 give the
 * reading implemented here, and DESIGN.md "Evaluation contract" fixes the
 * operation order that makes dt bit-reproducible.  Around the hot path:
 * the full-order RK2-average step and time loop, the ROM online step, loop
 * and time windows with the orthogonal and M-oblique transitions (P:847-906,
 * P:1175-1264), the offline POD / DEIM / Q-DEIM / oversampled sampling, the
 * Theorem-2 a-posteriori integrands and the index primitive of the
 * slab-sharded force's halo sum.  DESIGN.md R1-R29 list the readings.
 *
 * Conventions (all entry points):
 *   - FP64 everywhere; indices int32 (element->node table) / int64 (sizes).
 *   - Pointers are DEVICE pointers owned by the caller unless marked "host".
 *   - Calls are asynchronous on `stream`; outputs are overwritten, never
 *     accumulated.  Argument/shape errors return synchronously before any
 *     launch.  Device-side conditions (detJ <= 0 at a quadrature point, NaN
 *     time-step) are recorded in a sticky device status word and reported by
 *     hydro_status_sync(); output contents are unspecified in that case.
 *   - Layouts: H1 (kinematic) vectors SoA by component [dim][n_nodes]; L2
 *     (thermodynamic) vectors element-major [n_elem][k^dim] with local
 *     lexicographic Gauss-Legendre node order (j1 fastest); element->node table
 *     [n_elem][(k+1)^dim] with local lexicographic Gauss-Lobatto order (a1
 *     fastest).  Batched ROM arrays are [rows][B] (instance fastest).
 *   - F.1 is returned exactly as P:437 defines it (the momentum RHS is -F.1);
 *     no boundary condition is applied (v.n = g, is the solver's).
 *   - Results are bitwise reproducible run to run (no floating-point atomics).
 *   - One context/sample plan may be used by one stream at a time.
 */
#ifndef HYDRO_H_
#define HYDRO_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st *hydro_stream_t; /* == cudaStream_t; NULL = legacy default stream */

typedef struct hydro_ctx hydro_ctx;       /* opaque mesh context                         */
typedef struct hydro_sample hydro_sample; /* opaque sample-mesh plan (ROM mode)          */

typedef enum {
  HYDRO_OK = 0,
  HYDRO_ERR_ARG = 1,         /* bad pointer / size / unsupported combination             */
  HYDRO_ERR_UNSUPPORTED = 2, /* (dim, k, q) not compiled in                               */
  HYDRO_ERR_CUDA = 3,        /* a CUDA runtime call or launch failed                      */
  HYDRO_ERR_TANGLED = 4,     /* detJ <= 0 at some quadrature point (DESIGN R16)            */
  HYDRO_ERR_NONFINITE = 5,   /* some dt_q is NaN (DESIGN R15)                              */
  HYDRO_ERR_WORKSPACE = 6,   /* workspace too small or misaligned                          */
  HYDRO_ERR_NOT_CONVERGED = 7 /* an iterative solve (CG of M_V) stopped at its iteration cap
                                 with a finite residual above its tolerance                 */
} hydro_status;

/* Mesh description (kinematic H1 Q_k, thermodynamic L2 Q_{k-1}). */
typedef struct {
  int dim;                   /* 2 or 3                                                    */
  int order_h1;              /* k in {2, 3}; L2 order is k-1 (the only supported pair)    */
  int nq1d;                  /* Gauss-Legendre points per dim: 4 (k=2) or 6 (k=3)          */
  int64_t n_elem, n_nodes;   /* elements, H1 lattice nodes                                */
  const int32_t *elem_nodes; /* device [n_elem][(k+1)^dim]                                */
  const double *x0;          /* device [dim][n_nodes], initial (Lagrangian) positions     */
  const double *rho0;        /* device [n_elem], initial density, piecewise constant      */
} hydro_mesh_desc;

/* Artificial viscosity (DESIGN R3, BASELINE.json C0):
 *   mu = rho h (q1 cs + q2 h |min(lambda_min(eps(v)), 0)|),  sigma_a = mu eps(v).
 * enabled == 0 => mu = 0 (Gresho).                                     */
typedef struct { double q1, q2; int enabled; } hydro_visc;
/* CFL constants alpha, alpha_mu of Eq. adaptive-timestep (defaults 0.5, 2.5).  */
typedef struct { double alpha, alpha_mu; } hydro_cfl;

/* ------------------------------------------------------------------ context (setup, S0) */
/* Bytes of caller-provided device workspace hydro_ctx_create needs (0 on bad desc).       */
size_t hydro_ctx_workspace_bytes(const hydro_mesh_desc *desc /* host */);
/* Builds the per-quadrature-point mass m_q = rho0_K detJ0(xi_q) (density elimination,
 * P:389-391), the node->slot assembly map and the dt status block inside `workspace`
 * (device, >= hydro_ctx_workspace_bytes, 256-byte aligned).  Synchronises `stream`.
 * Copies desc (the pointers must stay valid for the context's lifetime).                  */
hydro_status hydro_ctx_create(const hydro_mesh_desc *desc /* host */, void *workspace,
                              size_t ws_bytes, hydro_stream_t stream, hydro_ctx **out /* host */);
hydro_status hydro_ctx_destroy(hydro_ctx *ctx);

/* ------------------------------------------------------------------ full-order force */
/* F1  = F.1  (assembled over shared H1 nodes, [dim][n_nodes]);
 * FTw = F^T.w (element-local, [n_elem][k^dim]); w == NULL means w = v.  The RK2-average
 * scheme needs w != v: F(U^n)^T v^{n+1/2}.
 * dt  = min over all quadrature points of alpha / (cs/h + alpha_mu mu / (rho h^2))
 *       (device scalar; NULL to skip), bit-identical to the oracle under the contract.
 * x, v, w: [dim][n_nodes]; e: [n_elem][k^dim]; gamma: [n_elem].                          */
hydro_status hydro_force_full(hydro_ctx *ctx, const double *x, const double *v, const double *e,
                              const double *w, const double *gamma, hydro_visc visc,
                              hydro_cfl cfl, double *F1, double *FTw, double *dt,
                              hydro_stream_t stream);
/* dt only (forward contractions + pointwise stage; no backward, no assembly).            */
hydro_status hydro_dt_estimate(hydro_ctx *ctx, const double *x, const double *v, const double *e,
                               const double *gamma, hydro_visc visc, hydro_cfl cfl, double *dt,
                               hydro_stream_t stream);
/* Two-pass form of F^T w for time integrators whose w depends on F.1 (RK2-average: w =
 * v^{n+1/2} = v^n - dt/2 M_V^-1 F.1).  hydro_force_full_store is hydro_force_full
 * with w = v that also stores the point stresses S_q = w_q detJ sigma J^-T in S (device,
 * hydro_force_stress_bytes(ctx) bytes, [n_elem][dim*dim][q^dim]); hydro_force_transpose then
 * evaluates FTw = F^T w = sum_q psi_j (S_q : gradhat w_q) for any w from the stored S without
 * repeating the pointwise stage (FTw within the element-local tolerance of hydro_force_full
 * with the same w).                                                                          */
size_t hydro_force_stress_bytes(const hydro_ctx *ctx);
hydro_status hydro_force_full_store(hydro_ctx *ctx, const double *x, const double *v, const double *e,
                                    const double *gamma, hydro_visc visc, hydro_cfl cfl, double *F1,
                                    double *FTw, double *dt, double *S, hydro_stream_t stream);
hydro_status hydro_force_transpose(hydro_ctx *ctx, const double *S, const double *w, double *FTw,
                                   hydro_stream_t stream);
/* Synchronises `stream`, returns the sticky device condition (TANGLED before NONFINITE)
 * and clears it.  *first_bad_elem (host, may be NULL) = lowest tangled element or -1.    */
hydro_status hydro_status_sync(hydro_ctx *ctx, hydro_stream_t stream, int64_t *first_bad_elem);

/* ------------------------------------------------------------------ ROM mode (C4) */
/* Sample plan for S0 = sample_elems (host, sorted, unique).  Closure = S0 plus every
 * element sharing an H1 node with S0 (DESIGN R20).  Row conventions:
 *   closure H1 rows   : c*n_cl_nodes + i, i over the ascending closure node ids;
 *   closure L2 rows   : l*k^dim + j, l over the ascending closure element ids;
 *   sampled F1 rows   : c*n_s0_nodes + i, i over the ascending node ids of S0 elements
 *                       (= the H1 dofs of S0 in ascending global SoA index);
 *   sampled FTw rows  : s*k^dim + j, s over S0 (ascending).
 * B = batch of independent instances evaluated per call (instance fastest).
 * Allocates its device tables with cudaMalloc (setup; never on the hot path).            */
hydro_status hydro_sample_create(hydro_ctx *ctx, const int32_t *sample_elems /* host */,
                                 int64_t n_sample, int B, hydro_sample **out /* host */);
hydro_status hydro_sample_destroy(hydro_sample *s);
/* Counts (host outputs, any may be NULL).                                                 */
hydro_status hydro_sample_info(const hydro_sample *s, int64_t *n_closure_elem,
                               int64_t *n_closure_nodes, int64_t *n_s0_nodes,
                               int64_t *s_v /* dim*n_s0_nodes */, int64_t *s_e /* |S0|*k^dim */);
/* Host copies of the ascending closure element ids / closure node ids / S0 node ids.     */
hydro_status hydro_sample_lists(const hydro_sample *s, int32_t *closure_elems /* host or NULL */,
                                int64_t *closure_nodes /* host or NULL */,
                                int64_t *s0_nodes /* host or NULL */);

/* Lift (restricted to sample-mesh rows):
 *   out[r][b] = os[r] (os_batched == 0) or os[r][b] (os_batched != 0)
 *               + sum_k Phi[r][k] Y[k][b],    r < rows, k < n, b < B.
 * Phi [rows][n] row-major, Y [n][B], out [rows][B].  Also serves the reduced position
 * RHS r_x = Phi_x^T v_os + (Phi_x^T Phi_v) Yhat_v with Phi = C_xv.  n <= 64,
 * B even and 16-byte aligned out (and batched os): the FP64 tensor pipe (mma.sync m8n8k4
 * f64); otherwise an FP64 FMA kernel (n <= 224: its shared-memory staging; larger n gives
 * HYDRO_ERR_ARG).  rows = 0 is a no-op (the row pointers may
 * be NULL).  Asynchronous; HYDRO_ERR_ARG on bad sizes.                                      */
hydro_status hydro_rom_lift(int64_t rows, int n, int B, const double *Phi, const double *os,
                            int os_batched, const double *Y, double *out, hydro_stream_t stream);

/* Sampled force: S1-S6 over (closure element, instance) pairs; F1_rows [s_v][B] at the
 * S0 nodes (complete: every element touching them is in the closure), FTw_rows [s_e][B]
 * of the S0 elements, dt [B] (min over the CLOSURE elements' quadrature points; NULL to
 * skip).  x_S, v_S, w_S: closure H1 rows [dim*n_cl_nodes][B]; e_S: closure L2 rows
 * [n_cl_elem*k^dim][B]; gamma: global [n_elem].  w_S == NULL means w = v.               */
hydro_status hydro_force_sampled(hydro_sample *s, const double *x_S, const double *v_S,
                                 const double *e_S, const double *w_S, const double *gamma,
                                 hydro_visc visc, hydro_cfl cfl, double *F1_rows,
                                 double *FTw_rows, double *dt, hydro_stream_t stream);
/* The sampled two-pass form (see hydro_force_full_store).  F^T w is needed only at the L2
 * rows of the S0 elements, so only their point stresses are kept: S [s_e/k^dim rows * B]
 * [dim*dim][q^dim] (S0 row r, instance b at r*B + b) of hydro_sample_stress_bytes(plan)
 * bytes, and the transposed pass runs over those S0 units only.  w_S: closure H1 rows
 * [dim*n_cl_nodes][B].                                                                         */
size_t hydro_sample_stress_bytes(const hydro_sample *s);
hydro_status hydro_force_sampled_store(hydro_sample *s, const double *x_S, const double *v_S,
                                       const double *e_S, const double *gamma, hydro_visc visc,
                                       hydro_cfl cfl, double *F1_rows, double *FTw_rows, double *dt,
                                       double *S, hydro_stream_t stream);
hydro_status hydro_sample_force_transpose(hydro_sample *s, const double *S, const double *w_S,
                                          double *FTw_rows, hydro_stream_t stream);
/* Sticky status of the sample plan (same semantics as hydro_status_sync; the element
 * index is global).                                                                        */
hydro_status hydro_sample_status_sync(hydro_sample *s, hydro_stream_t stream,
                                      int64_t *first_bad_elem);

/* Projection (Eq. sol-ls-hyper, P:778-799 with the precomputed (Z^T Phi)^dagger):
 *   r[i][b] = sum_s P[i][s] f[s][b],  P [n][s_rows] row-major, f [s_rows][B], r [n][B],
 * n <= 64, B <= 64.  Deterministic split-K: fixed contiguous row ranges per CTA, partials
 * summed in a fixed order.  n <= 40: the FP64 tensor pipe (cp.async-staged operands for even
 * B, register-tiled otherwise); n > 40: FP64 FMA.  `workspace` (device) >=
 * hydro_rom_project_workspace_bytes, else HYDRO_ERR_WORKSPACE.  s_rows = 0 (an empty
 * sample) sets r = 0 (P, f and the workspace may be NULL).  Asynchronous.                   */
size_t hydro_rom_project_workspace_bytes(int n, int64_t s_rows, int B);
hydro_status hydro_rom_project(int n, int64_t s_rows, int B, const double *P, const double *f,
                               double *r, void *workspace, size_t ws_bytes,
                               hydro_stream_t stream);

/* ------------------------------------------------------------------ FOM time step (NEXT-1) */
/* The full-order RK2-average step of PAPER Eq. RK2-avg around the force:
 *   v^{n+1/2} = v^n - dt/2 M_V^-1 F(U^n).1,   e^{n+1/2} = e^n + dt/2 M_E^-1 F(U^n)^T v^{n+1/2},
 *   x^{n+1/2} = x^n + dt/2 v^{n+1/2},
 *   v^{n+1}   = v^n - dt M_V^-1 F(U^{n+1/2}).1, e^{n+1} = e^n + dt M_E^-1 F(U^{n+1/2})^T vbar,
 *   x^{n+1}   = x^n + dt vbar,   vbar = (v^n + v^{n+1})/2.
 * M_V (kinematic mass, constant in time: P:389-391) is applied matrix-free and
 * inverted by Jacobi-preconditioned CG on the free dofs; M_E is block diagonal and inverted
 * exactly per element.  The boundary condition v.n = g with g = 0 is given as
 * the list of constrained velocity dofs (flat index c*n_nodes + node, host array); those
 * components of v are held at 0.  The scheme conserves 1/2 v^T M_V v + 1^T M_E e
 * up to the CG tolerance.  All reductions are fixed-order (deterministic).
 * hydro_fom_create allocates device memory (setup, never on the hot path) and
 * synchronises `stream`; it keeps `ctx` (which must outlive it).                          */
typedef struct hydro_fom hydro_fom;
hydro_status hydro_fom_create(hydro_ctx *ctx, const int64_t *bc_dofs /* host */, int64_t n_bc,
                              hydro_stream_t stream, hydro_fom **out /* host */);
hydro_status hydro_fom_destroy(hydro_fom *fom);
/* out = M_V in   (in, out: device [dim][n_nodes]; no boundary condition applied).         */
hydro_status hydro_mass_v_apply(hydro_fom *fom, const double *in, double *out,
                                hydro_stream_t stream);
/* sol = M_V^-1 rhs on the free dofs (0 on the constrained ones), PCG to the relative
 * preconditioned residual rel_tol or max_iter iterations; *iters, *relres (host, may be
 * NULL) report what was reached.  Synchronises `stream` (host-checked convergence).      */
hydro_status hydro_mass_v_solve(hydro_fom *fom, const double *rhs, double *sol, double rel_tol,
                                int max_iter, int *iters, double *relres, hydro_stream_t stream);
/* sol = M_E^-1 rhs  (device [n_elem][k^dim]).                                               */
hydro_status hydro_mass_e_solve(hydro_fom *fom, const double *rhs, double *sol,
                                hydro_stream_t stream);
/* out = M_E in (block-diagonal energy mass matrix; in/out device [n_elem][ne]).   */
hydro_status hydro_mass_e_apply(hydro_fom *fom, const double *in, double *out, hydro_stream_t stream);
/* Kinetic 1/2 v^T M_V v and internal 1^T M_E e energies (host outputs).  Synchronises.     */
hydro_status hydro_fom_energy(hydro_fom *fom, const double *v, const double *e,
                              double *kinetic, double *internal, hydro_stream_t stream);
/* The time-step controller of PAPER P:549-566 (defaults beta1 = 0.85, beta2 = 1.02,
 * gamma = 0.8).                                                                             */
typedef struct { double beta1, beta2, gamma; } hydro_dt_ctrl;
/* One RK2-average step of size dt, in place on the device state (x, v, e); per stage one
 * force evaluation storing S_q and one transposed F^T w pass, and a CG solve of M_V started
 * from the previous solve's solution (stopping test relative to the right-hand side).  *dt_est (host) = the min of
 * the two stages' time-step estimates for the caller's controller;
 * *cg_iters (host) = CG iterations used.  Device conditions (tangled, NaN) are reported by
 * hydro_status_sync on the context; a NaN CG residual (an invalid state) makes *dt_est NaN.
 * HYDRO_ERR_NOT_CONVERGED if a CG solve reaches cg_max_iter with a finite residual above
 * cg_tol (the state is then updated with that solve).  Synchronises `stream`.               */
hydro_status hydro_rk2avg_step(hydro_fom *fom, double *x, double *v, double *e,
                               const double *gamma, hydro_visc visc, hydro_cfl cfl, double dt,
                               double cg_tol, int cg_max_iter, double *dt_est /* host */,
                               int *cg_iters /* host */, hydro_stream_t stream);
/* Advance (x, v, e) in place from t0 to t_final with hydro_rk2avg_step under the controller
 * of P:549-566: a step with dt >= its estimate is undone (state restored from an internal
 * copy) and retried with beta1*dt; after an accepted step dt <- beta2*dt when
 * dt <= gamma*estimate; the step reaching t_final is shortened to land on it.  *dt (host,
 * in/out): the first trial step, returned as the controller's next step.  At most max_steps
 * accepted steps; *t_out (host) = the time reached, *steps / *rejected (host) = accepted and
 * rejected steps.  A trial step that tangles an element or whose estimate is NaN is rejected
 * like dt >= estimate (DESIGN R26) and retried with beta1*dt; after 10 000 rejections in a row
 * the loop stops with HYDRO_ERR_NONFINITE.  Errors of hydro_rk2avg_step (incl.
 * HYDRO_ERR_NOT_CONVERGED) end the loop and are returned.  Synchronises `stream`.            */
hydro_status hydro_fom_advance(hydro_fom *fom, double *x, double *v, double *e,
                               const double *gamma, hydro_visc visc, hydro_cfl cfl,
                               hydro_dt_ctrl ctrl, double t0, double t_final, double *dt,
                               int max_steps, double cg_tol, int cg_max_iter, double *t_out,
                               int *steps, int *rejected, hydro_stream_t stream);

/* ------------------------------------------------------------------ ROM online step (NEXT-2) */
/* The hyper-reduced RK2-average step of PAPER Eq. RK2-avg-rom-hr for the B
 * instances of a sample plan, on device, in place on the reduced coordinates
 * Yx [nx][B], Yv [nv][B], Ye [ne][B]:
 *   vhat^{n+1/2} = vhat^n - dt/2 R_v f1(U~^n)_S,   ehat^{n+1/2} = ehat^n + dt/2 R_e ftv(U~^n; v~^{n+1/2})_S,
 *   xhat^{n+1/2} = xhat^n + dt/2 (c_x + C_xv vhat^{n+1/2}),  and the second stage at U~^{n+1/2}
 *   with vbarhat = (vhat^n + vhat^{n+1})/2,
 * where U~ is lifted on the sample-mesh closure only through
 * Phi_{x,v,e}_S (closure rows, [rows][n] row-major) and the offsets (os_batched_flags bit 0/1/2:
 * x/v/e offset is [rows][B] instead of [rows]).  The offline operators are given:
 * R_v = Mhat_V^-1 Phi_v^T Phi_F1 (Z^T Phi_F1)^+ [nv][s_v], R_e likewise [ne][s_e] (Eq.
 * sol-ls-hyper), C_xv = Phi_x^T Phi_v [nx][nv], c_x = Phi_x^T v_os [nx] (
 * os_batched_flags bit 3: c_x is [nx][B], for per-instance velocity offsets).
 * dt: device [B] per-instance step; dt_est (device [B] or NULL) = min over both stages'
 * estimates.  Two sampled force evaluations per step (storing the S0 elements'
 * point stresses) and two transposed F^T w passes.  All device pointers are kept by the
 * object and must outlive it; buffers are allocated at create (setup).                   */
typedef struct hydro_rom hydro_rom;
hydro_status hydro_rom_create(hydro_sample *plan, int nx, int nv, int ne, const double *Phi_x_S,
                              const double *Phi_v_S, const double *Phi_e_S, const double *x_os_S,
                              const double *v_os_S, const double *e_os_S, int os_batched_flags,
                              const double *R_v, const double *R_e, const double *C_xv,
                              const double *c_x, hydro_rom **out /* host */);
hydro_status hydro_rom_destroy(hydro_rom *rom);
hydro_status hydro_rom_rk2avg_step(hydro_rom *rom, double *Yx, double *Yv, double *Ye,
                                   const double *gamma, hydro_visc visc, hydro_cfl cfl,
                                   const double *dt, double *dt_est, hydro_stream_t stream);
/* The online time loop t0 -> t_final for every instance under the controller of P:549-566
 * (as hydro_fom_advance, per instance: each instance is an independent simulation with its
 * own step).  dt (host [B], in/out): first trial steps, returned as the next steps.  The
 * instances step together; rejected and finished instances are restored from an internal
 * copy after each batched step.  At most max_iters batched steps; t_out, steps, rejected
 * (host [B] or NULL) per instance, *iters (host or NULL) = batched steps run.
 * HYDRO_ERR_NONFINITE on a NaN estimate.  Synchronises `stream`.                          */
hydro_status hydro_rom_advance(hydro_rom *rom, double *Yx, double *Yv, double *Ye,
                               const double *gamma, hydro_visc visc, hydro_cfl cfl,
                               hydro_dt_ctrl ctrl, double t0, double t_final, double *dt,
                               int max_iters, double *t_out, int *steps, int *rejected,
                               int *iters, hydro_stream_t stream);

/* ------------------------------------------------------------------ offline phase (NEXT-3) */
/* The half-stage state (x, v, e)^{n+1/2} of the last hydro_rk2avg_step (device copies; any
 * pointer may be NULL): the intermediate Runge-Kutta stages belong to the POD snapshot set
 * (P:921-943).                                                                              */
hydro_status hydro_fom_stage_state(hydro_fom *fom, double *x_half, double *v_half,
                                   double *e_half, hydro_stream_t stream);
/* POD of the snapshot matrix S (device, [ns][N] row-major: ONE SNAPSHOT PER ROW,
 * offsets already subtracted) by the method of snapshots: the Gram matrix S S^T on the GPU
 * (fixed-order split-K), its symmetric eigen-decomposition on the host (cyclic Jacobi,
 * ns x ns), sigma_i = sqrt(lambda_i), the energy criterion sum_{i<=k} sigma_i / sum sigma_i
 * >= eps (paper default 0.9999) with k <= max_k <= 128, and the basis
 * Phi = S^T V_k Sigma_k^-1 on the GPU followed by one CholQR pass (Phi <- Phi R^-1,
 * R^T R = Phi^T Phi: the Gram route alone is orthonormal only to ~eps (sigma_1/sigma_k)^2)
 * (device out [N][max_k] row-major, first k columns written; column c has the sign that
 * makes the largest-magnitude entry of the c-th Gram eigenvector positive).  sigma (host [ns] or NULL), *k_out (host).  Allocates its own
 * scratch (offline routine).  Synchronises `stream`.                                       */
hydro_status hydro_pod(const double *S, int ns, int64_t N, double eps, int max_k, double *Phi,
                       double *sigma, int *k_out, hydro_stream_t stream);
/* Greedy DEIM interpolation indices (Algorithm 1 of Chaturantabut-Sorensen) of
 * the basis U (device, [N][m] row-major): p_1 = argmax |u_1|; p_j = argmax |u_j - U_{<j} c|
 * with (P^T U_{<j}) c = P^T u_j (LU with partial pivoting, host).  Ties: the lowest row.
 * idx: host [m].  HYDRO_ERR_NONFINITE if some P^T U_{<j} is singular.  Synchronises.        */
hydro_status hydro_deim(const double *U, int64_t N, int m, int64_t *idx, hydro_stream_t stream);
/* Q-DEIM indices (Drmac-Gugercin): the first m pivots of a QR factorisation with
 * column pivoting of U^T, computed as pivoted Gram-Schmidt on the rows of U (device,
 * [N][m] row-major): pivot = the row with the largest residual norm (ties: the lowest row),
 * then every residual row loses its component along the pivot's normalised residual.
 * idx: host [m].  Allocates its own scratch (an [m][N] transposed copy of U).  Synchronises
 * `stream`.  HYDRO_ERR_NONFINITE if a residual vanishes before m pivots (U rank-deficient).  */
hydro_status hydro_qdeim(const double *U, int64_t N, int m, int64_t *idx, hydro_stream_t stream);
/* Oversampled greedy DEIM (gappy POD, the greedy of Carlberg et al. that allows
 * n_s >= m sample rows; R28 for the reading): basis column j (j = 0..m-1) adds
 * floor(n_s/m) (+1 while j < n_s mod m) rows: those outside the current set I with the largest
 * |u_j - U_{<j} c|, c the least-squares fit of U[I, <j] c ~ U[I, j] (host Householder QR),
 * taken one at a time in decreasing order (ties: the lowest row).  n_s = m is DEIM exactly.
 * U: device [N][m] row-major; idx: host [n_s] in selection order.  m <= n_s <= N.
 * Allocates its own scratch; synchronises `stream`.  HYDRO_ERR_NONFINITE on a rank-deficient fit. */
hydro_status hydro_deim_oversampled(const double *U, int64_t N, int m, int n_s, int64_t *idx,
                                    hydro_stream_t stream);
/* Time-window transition operators, so that yhat_w = T yhat_{w-1} + c:
 *   orthogonal, Eq. ic-tw (fom NULL or field 0 -- and always for the position field):
 *     T = Phi_w^T Phi_{w-1},  c = Phi_w^T (os_{w-1} - os_w);
 *   M-oblique, Eq. ic2-tw (fom given, field 1 = velocity with M_V, field 2 = energy with M_E):
 *     T = Mhat^-1 Phi_w^T M Phi_{w-1},  c = Mhat^-1 Phi_w^T M (os_{w-1} - os_w),
 *     Mhat = Phi_w^T M Phi_w  (n_w x n_w, LU-solved on the host).
 * Phi_new device [N][n_new], Phi_old device [N][n_old], os_new / os_old device [N][B] (B = 1 for
 * shared offsets), all row-major over the full FOM rows (N must match the field's size when
 * oblique).  T: device [n_new][n_old], c: device [n_new][B].  The products over N rows are
 * fixed-order split-K reductions (deterministic).  Allocates its own scratch; synchronises. */
hydro_status hydro_window_ops(hydro_fom *fom, int field, int64_t N, int n_new, int n_old, int B,
                              const double *Phi_new, const double *Phi_old, const double *os_new,
                              const double *os_old, double *T, double *c, hydro_stream_t stream);
/* Least-squares (gappy) pseudo-inverse of sampled basis rows, the offline factor of the
 * hyper-reduction (P:778-799 Eq. sol-ls-hyper; P:985-1000 SNS with M = I, DESIGN R21):
 *   P = (U[rows, :])^+ = (Z^T U)^+   [m][s]  (device out, row-major),
 * with U device [N][m] row-major and rows host [s] (0 <= rows[i] < N, m <= 128).  s >= m:
 * CholQR2 of the gathered rows (Q R = U[rows], two Cholesky-QR passes on the GPU with the
 * m x m Cholesky factorisations on the host) followed by P = R^-1 Q^T on the GPU; s < m (a
 * wide sample): the minimum-norm pseudo-inverse Q R^-T of U[rows]^T = Q R on the host.
 * HYDRO_ERR_NONFINITE if U[rows] is numerically rank-deficient.  Allocates its own scratch
 * (offline routine); synchronises `stream`.                                                */
hydro_status hydro_gappy_pinv(const double *U, int64_t N, int m, const int64_t *rows, int64_t s_rows,
                              double *P, hydro_stream_t stream);
/* The previous-window offset of a time-window transition, PAPER Eq. previous_os:
 *   os_w = os_{w-1} + Phi_{w-1} yhat_{w-1}(t_{w-1})      (os_new: device [rows][B], out)
 * -- the lift of the previous window's final state over the basis rows (the FOM rows, or the
 * sample-mesh closure rows of a hyper-reduced plan), per instance; os_prev is [rows] or
 * [rows][B] (os_prev_batched).  With this offset the new window starts from
 * yhat_w(t_{w-1}) = Phi_w^T (os_{w-1} + Phi_{w-1} yhat_{w-1} - os_w) = 0: Y_new (device
 * [n_new][B], or NULL with n_new = 0) is zeroed.  The offset-dependent operator of the new
 * window, c_x = Phi_x,w^T v_os,w, follows from hydro_basis_tproduct.  Asynchronous.         */
hydro_status hydro_rom_window_offset(int64_t rows, int n_prev, int B, const double *Phi_prev,
                                     const double *os_prev, int os_prev_batched, const double *Y_prev,
                                     double *os_new, int n_new, double *Y_new, hydro_stream_t stream);
/* out = Phi^T X  ([n][B], device): Phi device [N][n], X device [N][B], both row-major, by a
 * fixed-order split-K reduction over the N rows (deterministic).  E.g. c_x = Phi_x^T v_os
 * for per-instance offsets.  Allocates its own scratch; synchronises `stream`.   */
hydro_status hydro_basis_tproduct(int64_t N, int n, int B, const double *Phi, const double *X, double *out,
                                  hydro_stream_t stream);
/* The integrands of the a-posteriori bound, Theorem 2 Eq. aposteriori-semi, at
 * one (lifted) state (x, v, e) of a ROM trajectory (DESIGN R29):
 *   eta[0] = | (I - M_V Phi_v Mhat_V^-1 Phi_v^T P_F1) F.1(x, v, e) |_2,
 *   eta[1] = | (I - M_E Phi_e Mhat_E^-1 Phi_e^T P_Ftv) F^T.v(x, v, e) |_2,
 * Mhat = Phi^T M Phi, P f = U (U[Z,:])^+ f[Z] the (gappy, least-squares when s > m) DEIM
 * projector of the force basis U with sample rows Z.  The full-order force evaluation (w = v)
 * runs on all elements; M_V without boundary masking.  Device: x, v, e, gamma (the fom's
 * layouts), Phi_v [N_V][nv], Phi_e [N_E][ne], U1 [N_V][m1], U2 [N_E][m2]; host: Z1 [s1],
 * Z2 [s2] (s >= m), eta [2].  HYDRO_ERR_TANGLED / _NONFINITE if the state is invalid or a
 * small solve is singular.  Allocates its own scratch; synchronises `stream`.               */
hydro_status hydro_rom_indicator(hydro_fom *fom, const double *x, const double *v, const double *e,
                                 const double *gamma, hydro_visc visc, hydro_cfl cfl, int nv,
                                 const double *Phi_v, int ne, const double *Phi_e, int m1, const double *U1,
                                 int s1, const int64_t *Z1, int m2, const double *U2, int s2,
                                 const int64_t *Z2, double *eta, hydro_stream_t stream);
/* dst[c * ld_dst + dst_idx[i]] = (add ? that + : ) src[c * ld_src + src_idx[i]], i < n, c < dim
 * (NULL index = identity): the gather, fixed-order accumulate and scatter steps of the
 * slab-sharded force's halo sum (paper_2104_11404_b200/shard.py).  Device
 * pointers; the dst indices of one call must be distinct.  Asynchronous on `stream`.        */
hydro_status hydro_index_copy_add(int64_t n, int dim, const double *src, int64_t ld_src,
                                  const int64_t *src_idx, double *dst, int64_t ld_dst,
                                  const int64_t *dst_idx, int add, hydro_stream_t stream);


/* ------------------------------------------------------------------ profiling (host) */
/* When enabled, every hydro_force_full / hydro_dt_estimate / hydro_force_sampled call
 * records a pair of CUDA events around its force kernel on the call's stream (the
 * dominant kernel; bench.py's live roofline).  hydro_profile_read synchronises the
 * recorded events and returns the summed kernel time (ms) and launch count since the
 * last read, then clears them.  Profiling is global to the library (not per context). */
hydro_status hydro_profile_enable(int on);
hydro_status hydro_profile_read(double *total_ms /* host */, int64_t *count /* host */);
/* A call made while its stream is being captured into a CUDA graph records the pair as
 * external event-record nodes (cudaEventRecordExternal), so every replay of the graph
 * re-times the kernel.  hydro_profile_read_captured synchronises those events and returns
 * the summed kernel time of the most recent replay (they are kept, not cleared);
 * hydro_profile_release_captured returns them to the library once the graph is gone. */
hydro_status hydro_profile_read_captured(double *total_ms /* host */, int64_t *count /* host */);
hydro_status hydro_profile_release_captured(void);

/* ------------------------------------------------------------------ introspection (host) */
/* The library's own correctly rounded 1D tables for (k, q) (DESIGN R5, R6): xi[q], w[q],
 * B[q][k+1], G[q][k+1], Bl[q][k] (host outputs).  Pure host computation, no GPU needed. */
hydro_status hydro_basis_tables(int k, int q, double *xi, double *w, double *B, double *G,
                                double *Bl);
/* Kernel choice for 2D Q2/Q1 force evaluations (process-wide, all devices): 0 = by size
 * (default: one thread per element with >= 18 944 units, else one lane per point -- the
 * generic point-per-thread kernel when w != v),
 * 1 = always one thread per element (force2d_kernel), 2 = always one thread per point
 * (force_kernel), 3 = one lane per point with the Gauss column q1 per warp (force2d_pl_kernel;
 * w == v only, other calls keep the size-based choice).  Every kernel evaluates the same
 * contract: dt is bitwise identical; 1 and 2 share the backward FMA order (bitwise identical
 * F.1 / F^T.w), 3 sums the backward over q2 first (same values within the tolerances).
 * A test and A/B knob.  HYDRO_ERR_ARG otherwise.                                           */
hydro_status hydro_set_2d_kernel(int choice);
/* Number of kernel launches issued by this library since load (host counter).            */
int64_t hydro_launch_count(void);
/* Library version string.                                                                  */
const char *hydro_version(void);

#ifdef HYDRO_COUNT_ROT
/* Diagnostic builds only (-DHYDRO_COUNT_ROT, tools/rot_count.py): device counters of the
 * Jacobi fallback of the 3x3 eigen-solve -- out (host [12]): [0] lane-slots of executed
 * rotations, [1] rotations a lane needed, [2..9] per-sweep live lanes / executed lane-slots,
 * [10] points re-run with IEEE operators, [11] warps affected.  reset != 0 zeroes them.   */
hydro_status hydro_debug_rot_counts(unsigned long long *out, int reset);
#endif

/* ------------------------------------------------------------------ self-test (device) */
/* Checks the branch-free FP64 division / reciprocal / square-root fast paths the force
 * kernel's pointwise stage uses (csrc/ieee_fast.cuh; DESIGN "Kernels") against the IEEE
 * round-to-nearest operators on n seeded operands generated on the device (SplitMix64
 * counter stream of `seed`).  op: 0 = a/b, 1 = 1/b, 2 = sqrt.  dist: 0 = exponents in
 * [-64, 64], 1 = raw 64-bit patterns (NaN, inf, subnormals, extremes).  Atomically ADDS
 * to counts (device, 3 x uint64, caller zeroes them): [0] fast-path-valid results whose
 * bits differ from IEEE (the contract requires 0), [1] operands outside the fast range
 * (re-evaluated exactly by the caller), [2] operands tested.  Asynchronous on `stream`. */
hydro_status hydro_selftest_ieee_fast(uint64_t seed, int64_t n, int op, int dist,
                                      unsigned long long *counts, hydro_stream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* HYDRO_H_ */
