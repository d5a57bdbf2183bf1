/*
 * TEST INFRASTRUCTURE ONLY -- the CPU restatement used as the parity checker.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load it; the product (paper_2107_05337_b200) never links or calls it.
 *
 * Plain-C restatement of the reference's hot path (arXiv 2107.05337 code,
 * /root/reference/proj/include/miga):  CSR kernels (sparse.hpp), ILUT
 * factor/apply (ilut.hpp), Gauss-Seidel and dense LU (solvers.hpp), the
 * h-multigrid W-cycle and p-multigrid V-cycle / solve (pmultigrid.hpp), the
 * theta-step propagator Phi (theta.hpp) and MGRIT (mgrit.hpp).  Arithmetic is
 * written in the reference's evaluation order and compiled with
 * -ffp-contract=off, so on identical operators it reproduces the reference
 * bit for bit (pinned against oracle/_ref, see tests/test_oracle_pin.py).
 *
 * Setup-time assembly (spline/quadrature/Galerkin assembly) is NOT restated:
 * spatial operators enter as CSR arrays (from oracle/_ref, the golden
 * fixtures, or the engine's own device assembly under test).
 */
#ifndef PHI_ORACLE_H
#define PHI_ORACLE_H

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
    int n_rows, n_cols;
    const int* row_offsets;
    const int* col_indices;
    const double* values;
} oc_csr;

typedef struct oc_disc oc_disc;
typedef struct oc_hier oc_hier;
typedef struct oc_stepper oc_stepper;
typedef struct oc_mgrit oc_mgrit;

const char* oc_last_error(void);

/* ---- sparse.hpp ---------------------------------------------------------- */
int oc_spmv(const oc_csr* a, const double* x, double* y);              /* sparse.hpp:114-124 */
int oc_spmv_transpose(const oc_csr* a, const double* x, double* y);    /* sparse.hpp:133-143 */
double oc_norm2(const double* x, int n);                               /* sparse.hpp:188-194 */

/* ---- solvers.hpp --------------------------------------------------------- */
int oc_gs_sweep(const oc_csr* a, const double* b, double* x, int backward); /* solvers.hpp:80-99 */

/* ---- the spatial discretization bundle (pmultigrid.hpp:71-159), borrowed -- */
oc_disc* oc_disc_create(const oc_csr* mass_p, const oc_csr* stiff_p, const oc_csr* transfer,
                        const double* inv_lumped_p, const double* inv_lumped_1, int n_h,
                        const oc_csr* h_mass, const oc_csr* h_stiff, const oc_csr* h_embed);
void oc_disc_free(oc_disc*);

/* ---- PMultigridHierarchy (pmultigrid.hpp:215-324) ------------------------ */
oc_hier* oc_hier_create(const oc_disc* d, double c, int nu_pre, int nu_post, int gs_pre,
                        int gs_post, double ilut_tau, int ilut_fill);
void oc_hier_free(oc_hier*);
/* which: 0 A_p, 1 L, 2 U, 100+l a_h[l]; two-pass export (null arrays -> sizes) */
int oc_hier_csr(const oc_hier* h, int which, int* n_rows, int* n_cols, int* nnz, int* ro, int* ci,
                double* v);
int oc_hier_n_levels(const oc_hier* h);
int oc_ilut_apply(const oc_hier* h, const double* r, double* z);
int oc_restrict(const oc_hier* h, const double* r, double* r1);
int oc_prolong(const oc_hier* h, const double* e1, double* ep);
int oc_hmg_wcycle(const oc_hier* h, const double* b1, double* x1);
int oc_coarse_solve(const oc_hier* h, const double* b, double* x);
int oc_vcycle(const oc_hier* h, const double* b, double* x);
int oc_solve(const oc_hier* h, const double* b, double* x, double rel_tol, int max_iter,
             int fixed_cycles, int x0_empty, int* iters, int* converged, double* final_rel,
             double* history, int history_cap);

/* ---- ThetaStepper (theta.hpp:92-146) ------------------------------------- */
oc_stepper* oc_stepper_create(const oc_disc* d, double kappa, double dt, double theta,
                              double rel_tol, int max_iter, int fixed_cycles);
/* the same with SpatialSolverKind (theta.hpp:64): 0 pmg, 1 cg (Jacobi-preconditioned,
 * solvers.hpp:21-75) */
oc_stepper* oc_stepper_create_kind(const oc_disc* d, double kappa, double dt, double theta,
                                   int kind, double rel_tol, int max_iter, int fixed_cycles);
void oc_stepper_free(oc_stepper*);
/* u_next = Phi(u_prev) + load (load may be NULL); guess may be NULL (empty) */
int oc_stepper_step(const oc_stepper* s, const double* u_prev, const double* load,
                    const double* guess, double* out, int* iters);

/* ---- sequential_integrate (theta.hpp:216-237) ----------------------------- */
/* loads: NULL (no source), steady vector (load_steady=1), or steps x n terms */
int oc_sequential_integrate(const oc_disc* d, double kappa, double t_final, int nt, double theta,
                            const double* u0, const double* loads, int load_steady,
                            double rel_tol, int max_iter, double* traj, long long* solves,
                            long long* iterations);

/* ---- MgritSolver (mgrit.hpp:50-331) -------------------------------------- */
oc_mgrit* oc_mgrit_create(const oc_disc* d, double kappa, double t_final, int nt, double theta,
                          const double* u0, const double* loads, int load_steady, int cycle,
                          int relax, int m, double halt_tol, int max_iter, int coarse_floor,
                          double rel_tol, int sp_max_iter);
oc_mgrit* oc_mgrit_create_kind(const oc_disc* d, double kappa, double t_final, int nt,
                               double theta, const double* u0, const double* loads,
                               int load_steady, int cycle, int relax, int m, double halt_tol,
                               int max_iter, int coarse_floor, int spatial_kind, double rel_tol,
                               int sp_max_iter);
void oc_mgrit_free(oc_mgrit*);
int oc_mgrit_levels(const oc_mgrit* g, int* steps, double* dts);
int oc_mgrit_solve(oc_mgrit* g, int* iterations, int* converged, double* g_norm, double* final_rel,
                   long long* solves, double* mean_iters, double* history, int history_cap);
int oc_mgrit_trajectory(const oc_mgrit* g, double* out);

#ifdef __cplusplus
}
#endif
#endif
