/*
 * etq.h — C ABI of libetq, the B200 (sm_100a) hot path for the enriched Taylor–Hood
 * Q2–Q1* saddle-point systems of arXiv 2303.10233.
 *
 * Citation keys: P:n = PAPER.md line n (the paper's LaTeX); readings R#/O# are listed in
 * DESIGN.md §3.  All entry points are `extern "C"`, take plain pointers and sizes and no
 * torch types.  Unless stated otherwise:
 *   - vector arguments are DEVICE pointers to fp64 arrays in the system layout
 *       [u_x (nq) | u_y (nq) | p_1 (n_k) | p_0 (n_0)],   nq = (2n+1)^2, n_k = (n+1)^2, n_0 = n^2,
 *     each block lexicographic with x fastest (Q2 node (i,j) -> i + (2n+1) j, Q1 vertex
 *     (a,c) -> a + (n+1) c, element (e,f) -> e + n f);
 *   - the caller owns every vector and every report buffer; the library owns the problem,
 *     its matrices and all workspaces (allocated in etq_assemble / etq_precond_setup, so
 *     apply/solve calls allocate nothing);
 *   - every call is enqueued on the problem's CUDA stream and is asynchronous w.r.t. the
 *     host, except the *_solve calls, which synchronise once at exit, and the *_host calls;
 *   - a problem is not thread-safe (one host thread per problem);
 *   - errors are returned as etq_status (< 0), never by abort; etq_status_string() names them.
 */
#ifndef ETQ_H
#define ETQ_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct etq_problem etq_problem;   /* opaque; created by etq_assemble, freed by etq_destroy */
typedef int32_t etq_status;

enum {
    ETQ_OK = 0,
    ETQ_NOT_CONVERGED = 1,    /* maxit reached; report.converged = 0 (a warning, not a failure) */
    ETQ_EINVAL = -1,          /* bad argument: n < 2, n/coarse_n not a power of two, nu <= 0, NULL */
    ETQ_ENOMEM = -2,          /* device allocation failed */
    ETQ_ECUDA = -3,           /* a CUDA runtime call failed */
    ETQ_EINDEFINITE = -4,     /* <z, v> < 0 in MINRES (Algorithm 1 lines 3/10) */
    ETQ_EBREAKDOWN = -5,      /* alpha_1 = 0 in MINRES or a non-happy Arnoldi breakdown */
    ETQ_ENOTSETUP = -6,       /* preconditioner kind not set up on this problem */
    ETQ_ENAN = -7             /* NaN/Inf in a scalar recurrence */
};

/* Grid: n x n squares on [-1,1]^2, h = 2/n.
 * bc = 0: regularised lid u = (1 - x^4, 0) on y = 1, no-slip elsewhere (reading R1);
 * bc = 1: homogeneous Dirichlet velocity on the whole boundary.
 * storage (velocity operators; results are bitwise identical in all modes):
 *   0 = compressed: interior SELL slices keep neither column indices (col = row + per-class
 *       offset) nor values when these equal the per-class stencil bitwise;
 *   1 = implicit column indices only;  2 = explicit SELL (indices and values stored).
 * enriched = 1: the paper's Q2-Q1* (pressure space Q1 + P0); enriched = 0: plain
 *   Taylor-Hood Q2-Q1 on the same mesh (Stokes only; for the local-conservation contrast of
 *   P:198-202).  The vector layout is the same; in plain mode the p_0 block is inert: the saddle
 *   apply is the reduced [A B1^T; B1 0] (p_0 rows 0), the right-hand side's p_0 block is 0, and
 *   ETQ_PC_P2_GMG becomes diag(one V-cycle, m_p-step Chebyshev-Jacobi on the Q1 mass Q_k)
 *   (the standard Taylor-Hood Stokes preconditioner; m_p = mass_cheb_steps). */
typedef struct { int32_t n; int32_t bc; int32_t storage; int32_t enriched; } etq_grid;

/* Convection field of the Oseen problem.
 * kind = 0: none (Stokes, viscosity ignored);
 * kind = 1: frozen cavity wind w = (2y(1-x^2), -2x(1-y^2)) (BASELINE.json configs[3]);
 * kind = 2: a nodal Q2 wind given later by etq_set_wind (zero until then), e.g. the previous
 *           Picard iterate.  Velocity operators are stored
 *           explicitly (grid.storage is taken as 2). */
typedef struct { int32_t kind; } etq_wind;

typedef enum {
    ETQ_PC_P1_EXACT = 0,   /* P1 = diag(A, M_Q): exact A^{-1}, exact augmented M_Q solve; n <= 32 */
    ETQ_PC_P2_GMG = 1,     /* P2 = diag(one Q2-GMG V-cycle, Pi C Pi) with C = m-step Chebyshev-SGS */
    ETQ_PC_OSEEN_M1 = 2,   /* M1 = [[V-cycle(F), B^T], [0, -(1/nu) M_Q~]] block upper triangular */
    ETQ_PC_OSEEN_PCD1 = 3, /* Step-I PCD: [[V-cycle(F), B1^T], [0, -Ap^{-1} F1 Mp^{-1}]] */
    ETQ_PC_P1_ITER = 4,    /* P1 at any n: A^{-1} by V-cycle-preconditioned CG and the
                              exact augmented M_Q solve through S_k (reading R21), both to inner_rtol */
    ETQ_PC_P3 = 5,         /* diag(one Q2-GMG V-cycle, exact M_Q solve through S_k): P2's velocity block with
                              P1's pressure block (NEXT-2; mesh-independent MINRES counts) */
    ETQ_PC_OSEEN_M2 = 6,   /* M2 = [[V-cycle(F), B^T], [0, -M_S]], two-field PCD M_S = diag(Q1,Q0) diag(F1,F0)^-1
                              B M^-1 B^T (NEXT-4; stagnates) */
    ETQ_PC_OSEEN_LSC = 7   /* M3 = [[V-cycle(F), B^T], [0, -M_S]], least-squares commutator M_S with H = M
                              (NEXT-4, reading R26) */
} etq_pc_kind;

/* Preconditioner parameters (defaults in brackets; readings R7, R9, R13). */
typedef struct {
    int32_t cheb_sgs_steps;   /* m, Chebyshev-SGS steps on M_Q [20] */
    double  cheb_sgs_lo;      /* a, lower end of the SGS-preconditioned spectrum; <= 0 -> auto:
                                 max(Lanczos estimate, 2/m^2) (reading R7) */
    int32_t lanczos_steps;    /* steps of the Lanczos estimate used when cheb_sgs_lo <= 0 [60] */
    int32_t smooth_degree;    /* Chebyshev smoother degree in D^{-1}A [3] (reading R9) */
    double  smooth_hi;        /* upper end of the smoother interval [1.6] */
    double  smooth_lo;        /* lower end [smooth_hi / 10] */
    int32_t coarse_n;         /* coarsest V-cycle grid [2 Stokes, 32 Oseen] */
    int32_t mass_cheb_steps;  /* m_p, Chebyshev-Jacobi steps for Mp^{-1} in PCD [10] (reading R13) */
    int32_t use_graphs;       /* capture solver iterations in CUDA graphs [1] */
    double  inner_rtol;       /* relative residual of the inner CG solves of P1_ITER / P3 [1e-10] */
    int32_t inner_maxit;      /* iteration cap of each inner CG solve [100] */
    int32_t inner_coarse_n;   /* coarsest grid of the Q1 S_k hierarchy [16] (reading R21) */
} etq_pc_params;

/* Solve report; history/lanczos buffers are caller-owned HOST arrays and may be NULL. */
typedef struct {
    int32_t iterations, converged, restarts, status;
    double rel_res;           /* MINRES: |eta|/gamma_1; GMRES: ||r||/||b|| */
    double abs_res;           /* MINRES: |eta|; GMRES: true ||b - K x||_2 */
    double ms_total;          /* device time of the solve (CUDA events) */
    double* history; int32_t history_cap;           /* |eta_j| (MINRES) or residual estimates (GMRES) */
    double* lanczos_delta; double* lanczos_gamma; int32_t lanczos_cap;   /* delta_j, gamma_j of Algorithm 1 */
} etq_report;

/* Assemble the Stokes (wind NULL or kind 0) or Oseen system on the device: the scalar
 * velocity operator L (a(u,v)) or F_s = nu L + N(w), shared by both
 * velocity components; B = [B1; B0] and its transpose (b(u,p) = -int p div u, P:122,
 * P:882); Dirichlet identity rows with lifting into f and g (reading R2); the MG
 * hierarchy is built later by etq_precond_setup.  `cuda_stream` may be NULL (legacy
 * stream) or a cudaStream_t.  *out receives the new problem. */
etq_status etq_assemble(const etq_grid* grid, double viscosity, const etq_wind* wind,
                        void* cuda_stream, etq_problem** out);

/* Dof counts: n_u = 2 (2n+1)^2, n_k = (n+1)^2, n_0 = n^2. Host outputs. */
etq_status etq_sizes(const etq_problem* p, int64_t* n_u, int64_t* n_k, int64_t* n_0);

/* Right-hand side b = [f; g] (device, length N): lifting of the boundary data (reading R2)
 * plus the Galerkin load f += M_v f_nodal (reading R10) when f_nodal (device, 2 nq,
 * component-major Q2 nodal values) is not NULL; boundary rows carry the Dirichlet values. */
etq_status etq_build_rhs(const etq_problem* p, const double* f_nodal, double* b);

/* y = K x with K = [A B^T; B 0] or the Oseen [F B^T; B 0];
 * reduced = 1 applies [F B1^T; B1 0] on [u; p_1] and leaves y's p_0 block 0.
 * x and y must not alias. */
etq_status etq_apply_saddle(const etq_problem* p, int32_t reduced, const double* x, double* y);

/* Build the preconditioner `kind` (MG hierarchy, dense factors, Chebyshev interval).
 * params may be NULL (defaults).  Re-calling replaces the previous setup of that kind. */
etq_status etq_precond_setup(etq_problem* p, etq_pc_kind kind, const etq_pc_params* params);

/* z = P^{-1} r for the set-up preconditioner (device vectors, length N; r and z must not alias). */
etq_status etq_apply_precond(const etq_problem* p, etq_pc_kind kind, const double* r, double* z);

/* Component applies used by the parity tests (device vectors):
 *   etq_apply_vcycle:   z_u = one V-cycle of the P2/M1 setup on each velocity component (length n_u)
 *   etq_apply_mass_pc:  z_p = Pi C Pi r_p (length n_p) of the P2 setup (reading R6)
 *   etq_apply_mass:     y_p = M_Q x_p (Prop 2.1)
 *   etq_sgs_sweep:      z_p = S(y_p): one forward+backward 5-colour Gauss-Seidel sweep on
 *                       M_Q z = r_p from y_p (reading R7); y may equal z (in place). */
etq_status etq_apply_vcycle(const etq_problem* p, etq_pc_kind kind, const double* r_u, double* z_u);
etq_status etq_apply_mass_pc(const etq_problem* p, const double* r_p, double* z_p);

/* Exact augmented M_Q solve at any n through the Schur complement S_k = Q_k - R^T Q_0^{-1} R
 * (reading R21): z_p with M_Q z_p + lambda k = r_p and k^T z_p = 0, to the inner CG tolerance of the
 * P3 / P1_ITER setup (either kind).  r_p, z_p: device, length n_p, must not alias.  Synchronises; if
 * cg_iterations is non-NULL it receives the CG iterations this call took (host). */
etq_status etq_apply_mass_exact(const etq_problem* p, const double* r_p, double* z_p, int32_t* cg_iterations);

/* Counters of the inner CG solves since setup: which = 0 exact M_Q solve, 1 velocity CG (P1_ITER).
 * Host outputs: total CG iterations and number of solves. */
etq_status etq_inner_stats(const etq_problem* p, int32_t which, double* iterations, double* solves);
etq_status etq_apply_mass(const etq_problem* p, const double* x_p, double* y_p);
etq_status etq_sgs_sweep(const etq_problem* p, const double* r_p, const double* y_p, double* z_p);

/* Lanczos estimate of lambda_min(C_sgs^{-1} M_Q) on the complement of k (reading R7) from the
 * device start vector v0 (length n_p).  Host output *lam. */
etq_status etq_estimate_sgs_lo(etq_problem* p, const double* v0, int32_t steps, double* lam);

/* Chebyshev interval actually used by the P2/M1 setup (host output). */
etq_status etq_get_cheb_sgs_lo(const etq_problem* p, double* a);

/* Preconditioned MINRES, Algorithm 1 with stopping test |eta|/gamma_1 < rtol
 * (P:511-514); kind = P1_EXACT, P2_GMG, P3 or P1_ITER (Stokes).  x is the initial guess on input and the solution on output (device).
 * Returns ETQ_OK, ETQ_NOT_CONVERGED or an error.  report may be NULL. */
etq_status etq_minres_solve(etq_problem* p, etq_pc_kind kind, const double* b, double* x,
                            double rtol, int32_t maxit, etq_report* report);

/* Same with HOST b and x (pageable or pinned): copies in, solves, copies out. */
etq_status etq_minres_solve_host(etq_problem* p, etq_pc_kind kind, const double* b_host,
                                 double* x_host, double rtol, int32_t maxit, etq_report* report);

/* Export an assembled operator to caller-owned HOST CSR buffers (tests).  which:
 *   0 = scalar velocity operator with Dirichlet rows (L or F_s) of MG level `level`,
 *   1 = B (n_p x n_u), 2 = B^T (n_u x n_p), 3 = Ap of Q1 level `level` (PCD set up),
 *   4 = F1 (PCD set up), 5 = S_k / 4^level of Q1 level `level` (P3 or P1_ITER set up, reading R21),
 *   6 = the two-field Laplacian B Mdiag^-1 B^T on [Q1; P0] of level `level` (M2 or LSC set up).
 * Call with rowptr == NULL to query *nrows and *nnz. */
etq_status etq_export_operator(const etq_problem* p, int32_t which, int32_t level,
                               int64_t* nrows, int64_t* nnz,
                               int64_t* rowptr, int32_t* col, double* val);

/* Largest GMRES restart length m accepted by etq_gmres_solve / etq_two_stage_solve /
 * etq_picard_solve (the Krylov basis holds m + 1 vectors; larger m returns ETQ_EINVAL). */
#define ETQ_MAX_RESTART 63

/* Right-preconditioned restarted GMRES(m) with classical Gram-Schmidt applied twice (
 * readings R14, R18) on the Oseen system [F B^T; B 0] (reduced = 0, kind = ETQ_PC_OSEEN_M1) or the
 * reduced Taylor-Hood system [F B1^T; B1 0] (reduced = 1, kind = ETQ_PC_OSEEN_PCD1; the p_0 block of
 * b is ignored and x's p_0 block is left unchanged); kinds ETQ_PC_OSEEN_M2 / ETQ_PC_OSEEN_LSC precondition the
 * full system (reduced = 0) with the NEXT-4 Schur approximations.  Stops when the residual estimate
 * |g_{j+1}| <= rtol * ||b||_2 (Euclidean residual); report.abs_res is the true
 * ||b - K x||_2 after the last restart, report.history the estimates (entry 0 = ||r_0||).
 * x is the initial guess on input (device).  Returns ETQ_OK, ETQ_NOT_CONVERGED or an error. */
etq_status etq_gmres_solve(etq_problem* p, int32_t reduced, etq_pc_kind kind, const double* b, double* x,
                           double rtol, int32_t restart, int32_t maxit, etq_report* report);

/* Two-stage PCD strategy: Step I = GMRES on the reduced system with the PCD
 * preconditioner from x = 0, stopped at ||r|| <= c eta ||b_red||; Step II = GMRES on the full
 * system with M1 from [u1*; q1*; 0], stopped at ||r|| <= eta ||b||.  Both kinds must be set up.
 * bound_out[0] = ||z*|| (full-system residual at the transition), bound_out[1] = the Prop 3.3 bound
 * sqrt(c^2 eta^2 ||b_red||^2 + ||g0 - B0 u1*||^2) (reading R16).  x: device output. */
etq_status etq_two_stage_solve(etq_problem* p, const double* b, double* x, double eta, double c,
                               int32_t restart, int32_t maxit, etq_report* st1, etq_report* st2,
                               double bound_out[2]);

/* Nodal wind (wind kind 2): w = [w_x | w_y] on the Q2 nodes (device, length n_u).  Rebuilds F = nu L +
 * N(w) on every MG level (4 x 4 Gauss points per square, exact for a Q2 wind; coarse winds by
 * injection), the smoother ellipses (reading R9'), the coarse inverse and, if PCD is set up, F1;
 * the next etq_build_rhs lifts with the new F.  Synchronises.  ETQ_EINVAL for other wind kinds. */
etq_status etq_set_wind(etq_problem* p, const double* w);

/* Picard loop of the steady Navier-Stokes problem: x^0 = solution of the
 * wind-0 system (its velocity is the Stokes velocity), then `steps` Oseen solves, solve k with the
 * wind u^{k-1}; each solve is etq_two_stage_solve(eta, c, restart, maxit) on the RHS of that
 * system.  Wind kind 2, M1 and PCD1 set up.  x: device, length N, receives x^steps (its wind
 * state is u^{steps-1}).  its (host, 2 (steps+1), may be NULL): Step I / II GMRES iterations per
 * solve; res (host, steps+1, may be NULL): true ||b_k - K_k x^k|| / ||b_k||; ms_total: device ms. */
etq_status etq_picard_solve(etq_problem* p, int32_t steps, double eta, double c, int32_t restart,
                            int32_t maxit, double* x, int32_t* its, double* res, double* ms_total);

/* z_p1 = M_S1^{-1} r_p1 = Ap^{-1} F1 Mp^{-1} r_p1 on the Q1 pressure block (length n_k; PCD set up;
 * paper order of Eq. (discrete-commutator1x), reading R11).  Test hook of the Step-I Schur apply. */
etq_status etq_apply_pcd_schur(const etq_problem* p, const double* r_p1, double* z_p1);

/* fp32-value variants for the kernel sweep (BASELINE.json configs[4]): y = K x with fp32 matrix
 * values, fp32 vectors and fp32 accumulation (device float arrays, same layout), and one Stokes
 * V-cycle (P2 set up) in fp32.  The solvers always run in fp64. */
etq_status etq_apply_saddle_f32(etq_problem* p, int32_t reduced, const float* x, float* y);
etq_status etq_apply_vcycle_f32(etq_problem* p, const float* r_u, float* z_u);

/* EST-MINRES estimate of the discrete inf-sup constant gamma^2 (NEXT-1 of SURVEY
 * §8(f)) from the Lanczos scalars of a MINRES solve: the tridiagonal T_k with diagonal
 * delta[0..k) and off-diagonal gamma[0..k-1) (report.lanczos_delta / report.lanczos_gamma, i.e.
 * delta_1..delta_k and gamma_2..gamma_k of Algorithm 1).  With lam (lam - 1) = sigma for the
 * eigenvalues sigma of M_S^{-1} B A^{-1} B^T, the negative Ritz value mu closest to 0 gives
 * *gamma2 = mu (mu - 1).  Host arrays; *gamma2 = NaN when T_k has no negative Ritz value. */
etq_status etq_est_minres(const double* delta, const double* gamma, int32_t k, double* gamma2);

/* Number of libetq kernel launches issued so far in this process: direct launches plus the
 * kernel nodes of every graph launch (launches recorded during graph capture are excluded).
 * Host output; never fails. */
etq_status etq_launch_count(int64_t* count);

/* Time `reps` back-to-back launches of one hot kernel with CUDA events on the problem's stream
 * (bench.py's roofline measurement) and report its algorithmic bytes per launch.
 * which: 0 = fused saddle SpMV [A B^T; B 0] x (matrix-free Stokes apply: bytes = x in + y out);
 *        1 = finest-level fused Chebyshev step of the V-cycle (SpMV + update, both components);
 *        2 = one V-cycle on both velocity components (P2 set up);
 *        3 = one Pi C Pi pressure apply (P2 set up; L2-resident, bytes reported as 0);
 *        4 = one P2 preconditioner apply (velocity and pressure branches concurrently);
 *        5 = fp32 fused saddle SpMV; 6 = fp32 V-cycle (P2 set up);
 *        7 = one exact M_Q solve through S_k (P3/P1_ITER set up; replays of one captured graph);
 *        8 = one Q1-GMG V-cycle on S_k; 9 = one P3 preconditioner apply (graph replays);
 *        10 = one Chebyshev-SGS step on the pressure vectors (the SGS tile kernel, P2 set up);
 *        11 / 12 = the finest level's temporally blocked pre- / post-smoothing pass (P2 set up).
 * Host outputs: *ms = average device time per launch, *bytes = algorithmic bytes per launch. */
etq_status etq_time_kernel(etq_problem* p, int32_t which, int32_t reps, double* ms, double* bytes);

/* Implementation A/B switches are not part of this ABI: see include/etq_debug.h (test and
 * measurement builds only). */

const char* etq_status_string(etq_status s);
void etq_destroy(etq_problem* p);

#ifdef __cplusplus
}
#endif
#endif /* ETQ_H */
