/*
 * phasefrac_b200.h -- C ABI of the B200 (sm_100a) phase-field fracture load-step library.
 *
 * The reference (arXiv:1511.08463 package `phasefrac`, pure Python) has no FFI; its
 * drop-in seams are Python callables.  Each entry point below
 * replaces one of them; the Python host package `paper_1511_08463_b200` binds them
 * with ctypes (INTEGRATION.md shows the binding a maintainer would add to the
 * reference).  Reference paths are relative to /root/reference/pkg/src/phasefrac.
 *
 * Conventions
 *  - fp64 everywhere; all field / vector pointers are DEVICE pointers into
 *    caller-owned (PyTorch) memory unless stated "host".
 *  - Layout contract (mesh.py:3-10): u interleaved per vertex (d comps), vertex
 *    (i,j) = i*(ny+1)+j; crossed centre vertices follow the corners (index
 *    (nx+1)(ny+1) + I*ny + J); 3D vertex (i,j,k) = (i*(ny+1)+j)*(nz+1)+k.
 *  - Every call takes a cudaStream_t (passed as void*); work is enqueued on it.
 *    Calls that return host scalars synchronise that stream.
 *  - Return value: PF_OK or an error code (pf_last_error gives the message).
 *    Codes map to the reference exceptions: PF_EBREAKDOWN -> BreakdownError
 *    (linalg.py:25), PF_ESTALL -> LinearSolverError "elastic CG stalled"
 *    (solver.py:139-141), PF_EINNER -> InnerSolverError (linalg.py:37),
 *    PF_EINVAL -> ValueError, PF_ECUDA -> RuntimeError.
 *    Non-convergence of a VI / Newton solve is a report flag, not an error
 *    (vi.py:262-264).
 *  - One context per stream; not thread-safe (SPEC threading model).
 */
#ifndef PHASEFRAC_B200_H
#define PHASEFRAC_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PF_OK 0
#define PF_EINVAL 1
#define PF_ECUDA 2
#define PF_EBREAKDOWN 3
#define PF_ESTALL 4
#define PF_EINNER 5
#define PF_ENOWS 6

enum { PF_UNION_JACK = 0, PF_RIGHT = 1, PF_CROSSED = 2, PF_KUHN6 = 3 };
enum { PF_PLANE_STRESS = 0, PF_PLANE_STRAIN = 1, PF_3D = 2 };
enum { PF_AT1 = 0, PF_AT2 = 1 };
enum { PF_BC_NONE = 0, PF_BC_ELIMINATE = 1 };          /* operator row/col treatment   */
enum { PF_ROWS_RAW = 0, PF_ROWS_ZERO = 1, PF_ROWS_VALUE = 2 }; /* residual Dirichlet rows */
enum { PF_PREC_JACOBI = 0, PF_PREC_GMG = 1 };

/* Mesh + material descriptor (replaces Mesh/Material/Discretization construction,
 * mesh.py:112-142, model.py:23-61, fem.py:101-145).  Geometry is implicit. */
typedef struct pf_desc {
    int32_t dim;       /* 2 or 3 */
    int32_t pattern;   /* PF_UNION_JACK | PF_RIGHT | PF_CROSSED | PF_KUHN6 */
    int32_t regime;    /* PF_PLANE_STRESS | PF_PLANE_STRAIN | PF_3D */
    int32_t model;     /* PF_AT1 | PF_AT2 */
    int64_t nx, ny, nz;            /* cells per direction (nz ignored in 2D) */
    double lx, ly, lz;             /* extents */
    double E, nu, Gc, ell, k_ell;  /* scalar material (per-cell fields override E/Gc) */
    int32_t skip;                  /* PF_SKIP_* bits: workspaces NOT to plan (0 = everything) */
    int32_t reserved;
} pf_desc;

/* pf_desc.skip: an operator-only context (e.g. the operator sweep at 8192^2) plans neither
 * the multigrid hierarchy nor the stacked Newton vectors; the entry points that need them
 * (pf_elastic_solve with PF_PREC_GMG, pf_newton) then fail with PF_EINVAL. */
#define PF_SKIP_GMG 1
#define PF_SKIP_NEWTON 2

typedef struct pf_ctx pf_ctx;

/* Linear solve options / report (cg_solve linalg.py:106-152 semantics:
 * stop when ||r|| <= max(rtol*||b||, atol); maxit <= 0 -> 10*n). */
typedef struct pf_lin_opts {
    int32_t precond;      /* PF_PREC_JACOBI | PF_PREC_GMG */
    int32_t warm_start;   /* 1: start from the u0 argument; 0: x0 = 0 as the reference */
    int64_t maxit;
    double rtol, atol;
    int32_t check_every;  /* host convergence poll interval (iterations) */
    int32_t gmg_levels;   /* 0 = automatic */
    int32_t cheb_degree;  /* GMG smoother degree */
    int32_t gmg_reuse;    /* 1: keep the GMG hierarchy of an earlier solve (same context) while
                           * it stays effective -- rebuilt after a Dirichlet-mask / cell-field
                           * change, when the iteration count grows past 1.5x that of the first
                           * solve on it, or (with a retry) when PCG breaks down on it.
                           * 0: rebuild for every solve (the hierarchy of the current alpha). */
} pf_lin_opts;

typedef struct pf_lin_report {
    int64_t iterations;
    double final_residual_norm;
    double b_norm;
    int32_t converged;
    int32_t status;
} pf_lin_report;

/* Reduced-space active-set VI options / report (VIConfig vi.py:68-75, ActiveSetReport
 * vi.py:78-86). */
typedef struct pf_vi_opts {
    double abs_tol;
    int32_t max_iterations;
    int32_t precond;        /* inner PCG preconditioner */
    double ls_backtrack, ls_min_step, armijo;
    double inner_rtol;      /* relative tolerance of the inactive-block PCG (damage solve);
                             * pf_newton: of the field-split block solves, <= 0 -> fieldsplit_rtol */
    int64_t inner_maxit;
    double zero_tol;        /* <= 0 -> 1e-10 (1 + |x0|_inf) as the reference */
    double fieldsplit_rtol; /* Newton only: MINRES rtol (solver.py:64) */
    int32_t inner_cycles;   /* Newton only: > 0 -> each field-split block solve is a fixed budget of
                             * this many PCG iterations at rtol 1e-12 (fieldsplit_inner = "cg",
                             * inner_cg linalg.py:446-456); 0 -> solved to inner_rtol.
                             * inner_mode 1: the Chebyshev degree of the C block (<= 0 -> 12) */
    int32_t inner_mode;     /* Newton: 0 -> block solves as above; 1 -> fixed linear SPD block
                             * preconditioners: A^-1 ~ one multigrid V-cycle, C^-1 ~ Chebyshev-Jacobi
                             * on [lmax/30, 1.5 lmax] (lmax by 30 power iterations, the reference
                             * ChebyshevPreconditioner recipe linalg.py:331-378), symmetric
                             * multiplicative split; 2 -> the same blocks, block-diagonal split.
                             * Damage solve: 1 -> inexact rsls Newton, inner rtol = min(1e-2, |Phi|).
                             * pf_newton: | 4 -> inexact Newton, MINRES rtol per iteration
                             * max(fieldsplit_rtol, min(1e-2, |Phi|)). */
} pf_vi_opts;

typedef struct pf_vi_report {
    int32_t iterations;
    int32_t converged;
    double final_residual_norm;
    int64_t total_krylov_iterations;
    int32_t steepest_descent_steps;
    int32_t linear_failures;
    int32_t status;
    int32_t n_history;
    double history[64];     /* sqrt(merit) per accepted iterate (first 64) */
} pf_vi_report;

/* ---- lifecycle (fem.py:93-105) ---------------------------------------------- */
int pf_ctx_create(const pf_desc* desc, pf_ctx** out);
void pf_ctx_destroy(pf_ctx* ctx);
const char* pf_last_error(const pf_ctx* ctx);       /* ctx may be NULL (creation errors) */
/* out: [n_vertices, n_udofs, n_elements, n_cells, n_corner_vertices, dim, elems_per_cell, 0] */
int pf_query(const pf_ctx* ctx, int64_t out[8]);
int64_t pf_workspace_bytes(const pf_ctx* ctx);
int pf_bind_workspace(pf_ctx* ctx, void* dev_ptr, int64_t bytes);

/* ---- per-step data ------------------------------------------------------------ */
/* Per-cell E / Gc (device, n_cells, cell index I-major); NULL -> scalar. */
int pf_set_cell_fields(pf_ctx* ctx, const double* E_cell, const double* Gc_cell);
/* Dirichlet data (DirichletBC fem.py:58-90): HOST sorted unique dofs + values; every dof
 * must belong to a boundary vertex.  n = 0 clears.  Enqueued on `stream`. */
int pf_set_dirichlet(pf_ctx* ctx, const int64_t* dofs, const double* vals, int64_t n,
                     void* stream);
/* Isotropic inelastic strain eps0 = e*(1,1,0) per element, given as a HOST table
 * e[type*ny + J] for element type `type` in cell row J (2D; profile in y only, as the
 * thermal-shock setups need, cases.py:66-80).  NULL clears. */
/* Graded (banded) meshes, banded_rect_mesh mesh.py:163-190: heights of the ny cell rows
 * (HOST array, bottom to top; their sum is the y extent).  NULL restores uniform rows ly/ny.
 * Columns stay uniform.  Invalidates the multigrid hierarchy. */
int pf_set_row_heights(pf_ctx* ctx, const double* row_heights, void* stream);
int pf_set_eps0_rows(pf_ctx* ctx, const double* table, void* stream);

/* ---- operators (fem.py:162-276) -------------------------------------------- */
/* y = Kuu(alpha) x; bc_mode PF_BC_ELIMINATE applies eliminate_dirichlet (fem.py:282-294). */
int pf_apply_Kuu(pf_ctx* ctx, const double* alpha, const double* x, double* y, int32_t bc_mode,
                 void* stream);
/* y = Kaa(u, alpha) x  (fem.py:266-276; AT2 adds the w'' reaction). */
int pf_apply_Kaa(pf_ctx* ctx, const double* u, const double* alpha, const double* x, double* y,
                 void* stream);
/* Damage-block coefficients at fixed u (alpha-independent for AT1/AT2): per-element reaction
 * kappa_e (n_elements, slot-major) and the affine remainder c = r_alpha - Kaa alpha (n_vertices;
 * may be NULL).  pf_apply_Kaa_coef then applies Kaa from those coefficients alone. */
int pf_kaa_coefficients(pf_ctx* ctx, const double* u, double* kappa, double* c, void* stream);
int pf_apply_Kaa_coef(pf_ctx* ctx, const double* kappa, const double* x, double* y, void* stream);
/* yu = Kua xa (fem.py:246-263), ya = Kua^T xu; bc_mode PF_BC_ELIMINATE zeroes Dirichlet rows. */
int pf_apply_Kua(pf_ctx* ctx, const double* u, const double* alpha, const double* xa, double* yu,
                 int32_t bc_mode, void* stream);
int pf_apply_Kau(pf_ctx* ctx, const double* u, const double* alpha, const double* xu, double* ya,
                 int32_t bc_mode, void* stream);
/* Fused physics pass: energies (assemble_energy fem.py:162-174), r_u (fem.py:177-189; rows
 * per `rows`), r_alpha (fem.py:202-218), the FB optimality residual Phi (solver.py:104-118,
 * vi.py:89-115).  Any of r_u / r_a / phi may be NULL.  out (HOST, may be NULL):
 * [E_el, E_d, E_tot, ||r_u||^2, ||Phi_alpha||^2, ||(r_u,Phi)||, 0, 0]. */
int pf_physics(pf_ctx* ctx, const double* u, const double* alpha, const double* alpha_lb,
               double* r_u, double* r_a, double* phi, int32_t rows, double* out, void* stream);
/* f = inelastic-strain load (assemble_load_u fem.py:192-199). */
int pf_load_u(pf_ctx* ctx, const double* alpha, double* f, void* stream);

/* ---- solvers (solver.py:129-241) ----------------------------------------------- */
/* elastic_step: u_out = argmin_u E(u, alpha) with Dirichlet data; u0 = initial guess
 * (NULL or warm_start = 0 -> zero).  u_out may alias u0. */
int pf_elastic_solve(pf_ctx* ctx, const double* alpha, const double* u0, double* u_out,
                     const pf_lin_opts* opts, pf_lin_report* rep, void* stream);
/* The multigrid V-cycle of Kuu(alpha) as a stand-alone fixed SPD preconditioner (replaces the
 * reference's SuperLU factor object, linalg.py:250-262, where a caller runs its own Krylov loop):
 * prepare builds the hierarchy for alpha and the context's Dirichlet mask, apply computes z = M r
 * (identity on eliminated rows).  Used by the element-list path on jittered structured meshes. */
int pf_gmg_prepare(pf_ctx* ctx, const double* alpha, void* stream);
int pf_gmg_apply(pf_ctx* ctx, const double* r, double* z, void* stream);
/* damage_step: alpha_out = rsls solution of the box QP at fixed u (vi.py:187-264). */
int pf_damage_solve(pf_ctx* ctx, const double* u, const double* alpha_lb, const double* alpha_in,
                    double* alpha_out, const pf_vi_opts* opts, pf_vi_report* rep, void* stream);
/* u_out = u_prev + omega (u_star - u_prev), then Dirichlet snap (solver.py:193-197). */
int pf_relax_u(pf_ctx* ctx, const double* u_prev, const double* u_star, double omega,
               double* u_out, void* stream);
/* Over-relaxed projected damage update with midpoint backtracking and d_alpha
 * (solver.py:202-216).  out (HOST): [omega_bar, d_alpha, halvings]. */
int pf_relax_alpha(pf_ctx* ctx, const double* a_prev, const double* a_star,
                   const double* alpha_lb, double omega, double* alpha_out, double* out,
                   void* stream);
/* The AM iteration tail in one sweep (north_star part 4): pf_relax_alpha fused with the physics
 * pass of the relaxed state (solver.py:202-219).  phys_out (HOST, 8) as pf_physics with
 * PF_ROWS_ZERO: [E_el, E_d, E_tot, |r_u|^2, |Phi_a|^2, |Phi|, 0, 0]; relax_out (HOST, 3) as
 * pf_relax_alpha.  2D: one relaxation-bits launch + one fused strip pass; 3D: two passes. */
int pf_relax_alpha_physics(pf_ctx* ctx, const double* u, const double* a_prev, const double* a_star,
                           const double* alpha_lb, double omega, double* alpha_out,
                           double* phys_out, double* relax_out, void* stream);
/* u[bc] = ubar (solver.py:121-123). */
int pf_snap_bc(pf_ctx* ctx, double* u, void* stream);
/* coupled_newton_solve (solver.py:303-330): reduced-space active-set Newton on (u, alpha)
 * with field-split preconditioned MINRES; writes the last merit-nonincreasing iterate. */
int pf_newton(pf_ctx* ctx, const double* u_in, const double* alpha_in, const double* alpha_lb,
              double* u_out, double* alpha_out, const pf_vi_opts* opts, pf_vi_report* rep,
              void* stream);

/* Counters for the bench: kernel launches issued by this context since creation. */
int64_t pf_launch_count(const pf_ctx* ctx);
/* Bounds-check aid (no reference counterpart).  A context created with PF_WS_GUARD=1 in the
 * environment puts a 16 KB guard zone after every workspace buffer (and every multigrid-level
 * buffer), filled with 0xA5 at pf_bind_workspace; *bad_bytes = how many guard bytes differ now,
 * i.e. out-of-bounds writes past any buffer since binding (0 without guards).  Synchronises. */
int pf_check_guards(pf_ctx* ctx, int64_t* bad_bytes, void* stream);
/* Per-kernel-class timing: when enabled, every launch is bracketed by CUDA events on its
 * stream.  pf_profile_read syncs and returns out[3k..3k+2] = (launches, total ms,
 * algorithmic bytes) for kernel class k = 0..nkinds-1 (order: Kuu, Kuu-CG, Kuu-diag, kappa,
 * Kaa, Kaa-CG, Kaa-diag, Kaa-trial, physics, rhs, Kua, Kau, Jacobian, CG-vector, vector,
 * GMG cycle, GMG setup) and resets the counters. */
int pf_profile(pf_ctx* ctx, int32_t enable);
int pf_profile_read(pf_ctx* ctx, double* out, int32_t nkinds);

/* ---- Element-list (unstructured / jittered) P1 meshes -------------------
 * The reference builds its thermal-shock mesh by jittering the interior vertices of a
 * structured triangulation (mesh.py:112-142, cases.py:195-234); geometry is then no longer
 * implicit.  pf_umesh holds an arbitrary positively oriented triangle (dim 2) or tetrahedron
 * (dim 3) mesh as element lists and applies the same centroid-quadrature operators as the
 * structured context (fem.py:221-276 assemble_* matvecs).  Vertex numbering is the caller's; u
 * is interleaved per vertex.  Mesh arrays in the descriptor are HOST arrays, read only during
 * pf_umesh_create (which validates orientation: PF_EINVAL "mesh contains non-CCW or degenerate
 * triangles", as Discretization construction raises, fem.py:107-123). */
typedef struct pf_umesh_desc {
    int32_t dim;               /* 2 or 3 */
    int32_t regime;            /* PF_PLANE_STRESS | PF_PLANE_STRAIN (dim 2) | PF_3D (dim 3) */
    int32_t model;             /* PF_AT1 | PF_AT2 */
    int32_t reserved;
    int64_t n_vertices, n_elements;
    const double* vertices;    /* host (n_vertices, dim) */
    const int64_t* elements;   /* host (n_elements, dim+1) */
    const double* E_elem;      /* host (n_elements) or NULL -> E */
    const double* Gc_elem;     /* host (n_elements) or NULL -> Gc */
    double E, nu, Gc, ell, k_ell;
} pf_umesh_desc;

typedef struct pf_umesh pf_umesh;

int pf_umesh_create(const pf_umesh_desc* desc, pf_umesh** out);
void pf_umesh_destroy(pf_umesh* m);
const char* pf_umesh_last_error(const pf_umesh* m);  /* m may be NULL (creation errors) */
int64_t pf_umesh_workspace_bytes(const pf_umesh* m);
/* Uploads the element records and vertex->element lists into the (256 B aligned, caller-owned)
 * device workspace; synchronises the stream. */
int pf_umesh_bind_workspace(pf_umesh* m, void* dev_ptr, int64_t bytes, void* stream);
/* Dirichlet dofs (host, interleaved dof indices) for PF_BC_ELIMINATE applies (fem.py:297-310). */
int pf_umesh_set_dirichlet(pf_umesh* m, const int64_t* dofs, int64_t n, void* stream);
/* y = Kuu(alpha) x (assemble_Kuu(...).matvec, fem.py:233-244); PF_BC_ELIMINATE: Dirichlet
 * rows/cols replaced by the identity. */
/* Inelastic strain per element (assemble_load_u / thermal_strain, fem.py:192-199, cases.py:66-80):
 * eps0 = DEVICE pointer to T x 3 (2D Voigt e11, e22, g12) or T x 6 (3D) doubles, caller-owned and
 * kept alive by the caller; NULL clears.  Every strain of u (energies, residuals, the damage
 * Hessian's elastic coupling) becomes B u - eps0; the Kuu apply is unchanged. */
int pf_umesh_set_eps0(pf_umesh* m, const double* eps0, void* stream);
int pf_umesh_apply_Kuu(pf_umesh* m, const double* alpha, const double* x, double* y, int32_t bc_mode,
                       void* stream);
/* y = Kaa(u, alpha) x (assemble_Kaa(...).matvec, fem.py:266-282). */
int pf_umesh_apply_Kaa(pf_umesh* m, const double* u, const double* alpha, const double* x, double* y,
                       void* stream);
/* Solve Kuu(alpha) x = b with Dirichlet rows/cols eliminated (pf_umesh_set_dirichlet) by Jacobi
 * PCG from x0 = 0 (cg_solve linalg.py:106-152: stop when ||r|| <= max(rtol ||b||, atol), polled
 * every check_every iterations; maxit <= 0 -> 10 n).  opts->precond must be PF_PREC_JACOBI.
 * Non-convergence is rep->converged = 0; p^T A p <= 0 is PF_EBREAKDOWN.  Fixed-order reductions:
 * bitwise-reproducible iterates. */
int pf_umesh_elastic_solve(pf_umesh* m, const double* alpha, const double* b, double* x,
                           const pf_lin_opts* opts, pf_lin_report* rep, void* stream);
/* Energy parts and gradients at (u, alpha) (assemble_energy / assemble_residual_u(apply_bc=False) /
 * assemble_residual_alpha, fem.py:162-218): r_u (device, d*V, raw rows) and r_alpha (device, V)
 * may be NULL; energy (HOST, 3: elastic, surface, total) may be NULL, else the stream is
 * synchronised.  No inelastic strain on this path. */
int pf_umesh_physics(pf_umesh* m, const double* u, const double* alpha, double* r_u, double* r_alpha,
                     double* energy, void* stream);
/* Damage half-step on the element-list mesh (damage_half_step, am.py / solver.py:160-191): alpha_out =
 * the rsls solution (vi.py:187-264) of the box QP min 1/2 a^T Kaa(u) a + c^T a, alpha_lb <= a <= 1, at
 * fixed u, started from clip(alpha_in) (alpha_out may alias alpha_in).  Reduced-space active set:
 * each iteration solves K_II d_I = -g_I by Jacobi PCG (opts->inner_rtol / inner_maxit), then a
 * projected Armijo backtracking step on 1/2 |Phi_FB|^2.  rep->status = PF_ESTALL when max_iterations
 * end unconverged (the call still returns PF_OK). */
int pf_umesh_damage_solve(pf_umesh* m, const double* u, const double* alpha_lb, const double* alpha_in,
                          double* alpha_out, const pf_vi_opts* opts, pf_vi_report* rep, void* stream);
int64_t pf_umesh_launch_count(const pf_umesh* m);

#ifdef __cplusplus
}
#endif
#endif
