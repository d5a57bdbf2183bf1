/*
 * phi_engine.h -- C ABI of the B200 engine for the time-stepping operator Phi
 * of MGRIT + p-multigrid (arXiv 2107.05337 reference code `miga`,
 * /root/reference/proj/include/miga).
 *
 * Plain C: opaque handles, int32 indices, fp64 values, no torch types.  Every
 * entry point cites the reference interface it replaces.  All compute runs on
 * the GPU (sm_100a); there is no CPU fallback -- a missing device returns
 * PHI_ERR_CUDA.
 *
 * Status codes: 0 ok, 1 invalid argument (std::invalid_argument in the
 * reference), 2 non-convergence (std::runtime_error "spatial solve did not
 * converge ..."), 3 CUDA failure, 4 other runtime error (zero pivot, singular
 * coarse matrix ...).  phi_last_error() returns the thread-local message,
 * worded as the reference's exception text.
 */
#ifndef PHI_ENGINE_H
#define PHI_ENGINE_H

#ifdef __cplusplus
extern "C" {
#endif

#define PHI_OK 0
#define PHI_ERR_INVALID 1
#define PHI_ERR_NOT_CONVERGED 2
#define PHI_ERR_CUDA 3
#define PHI_ERR_RUNTIME 4

/* source / initial-condition kinds (the reference takes std::function values,
 * theta.hpp:17-48; the engine evaluates these named kinds on device) */
#define PHI_SOURCE_CONSTANT 0  /* SourceTerm::constant(param); 0 -> zero source */
#define PHI_SOURCE_SIN_EXP 1   /* transient param * exp(-t) * sin(pi x) sin(pi y) */
#define PHI_SOURCE_SIN 2       /* steady    param * sin(pi x) sin(pi y)           */
#define PHI_INIT_ZERO 0        /* ProblemSpec::initial empty                       */
#define PHI_INIT_SIN 1         /* sin(pi x) sin(pi y), L2-projected                */
#define PHI_INIT_COEFFS 2      /* spline sum_i c_i phi_i (free dofs), L2-projected */
#define PHI_INIT_VECTOR 3      /* init_coeffs IS the projected free-dof state u0 (a
                                * caller that ran project_initial itself, theta.hpp:150-160) */

typedef struct phi_disc phi_disc;
typedef struct phi_hier phi_hier;
typedef struct phi_stepper phi_stepper;
typedef struct phi_mgrit phi_mgrit;

/* PMultigridOptions, pmultigrid.hpp:161-168 */
typedef struct {
    double ilut_tau; /* 1e-13 */
    int ilut_fill;   /* 0 = average row fill */
    int nu_pre, nu_post, gs_pre, gs_post;
    /* summation order of every reduction on the solve path (row sums of the
     * operators and triangular factors, Gauss-Seidel rows, dot products):
     * 1 = the reference's sequential order -- results bit-identical to the
     *     reference on identical inputs;
     * 0 = reassociated parallel sums (default) -- results within the
     *     north-star tolerance (p-MG / MGRIT iteration counts +-1, final
     *     space-time solution <= 1e-8 relative L2), several times faster. */
    int exact;
} phi_pmg_options;

/* SpatialSolverKind, theta.hpp:64 */
enum { PHI_SOLVER_PMG = 0, PHI_SOLVER_CG = 1 };

/* SpatialSolverConfig, theta.hpp:66-75.  kind PHI_SOLVER_CG: Jacobi-
 * preconditioned CG on the left-hand operator (solvers.hpp:21-75,
 * theta.hpp:121-125); pmg and fixed_cycles are then unused. */
typedef struct {
    double rel_tol; /* 1e-12 */
    int max_iter;   /* 400 */
    int fixed_cycles;
    phi_pmg_options pmg;
    int kind; /* PHI_SOLVER_PMG (default) or PHI_SOLVER_CG */
} phi_solver_config;

/* MgritConfig, mgrit.hpp:17-31 (workers replaced by the device batch) */
typedef struct {
    int cycle; /* 0 V, 1 F, 2 two-level */
    int relax; /* 0 F, 1 FCF */
    int m;
    double halt_tol;
    int max_iter;
    int coarse_floor;
} phi_mgrit_config;

/* ProblemSpec, theta.hpp:42-62 (unit square; degree / mesh come from the disc) */
typedef struct {
    double kappa, t_final, theta;
    int n_time_steps;
    int source_kind;
    double source_param;
    int init_kind;
    const double* init_coeffs; /* n_free, PHI_INIT_COEFFS only */
    const double* load_terms;  /* optional caller load schedule: steps x n_free, or n_free if steady */
    int load_terms_steady;
} phi_problem;

/* MgritResult, mgrit.hpp:33-42 (trajectory via phi_mgrit_trajectory) */
typedef struct {
    int iterations;
    int converged;
    double g_norm;
    double final_relative_residual;
    long long total_spatial_solves;
    double mean_spatial_iterations;
} phi_mgrit_result;

const char* phi_last_error(void);
void phi_default_solver_config(phi_solver_config* cfg);
void phi_default_mgrit_config(phi_mgrit_config* cfg);
void phi_default_problem(phi_problem* ps);
int phi_device_count(void);
int phi_set_device(int device);
int phi_synchronize(void);

/* ---- SpatialDiscretization::build (pmultigrid.hpp:94-158), unit square ---- */
int phi_disc_build(int degree, int mesh_exponent, phi_disc** out);
void phi_disc_free(phi_disc* d);
/* info: [n_free_p, n_free_1, n_h_levels, n_elements, degree] */
int phi_disc_info(const phi_disc* d, int* info);
/* selectors as the reference fields: 0 mass_p, 1 stiff_p, 2 transfer_p1,
 * 100+l h_chain[l].mass, 200+l h_chain[l].stiff, 300+l h_chain[l].embed.
 * Two-pass: call with null arrays for the sizes. */
int phi_disc_export(const phi_disc* d, int which, int* n_rows, int* n_cols, int* nnz, int* row_offsets,
                    int* col_indices, double* values);
/* 0 inv_lumped_p, 1 inv_lumped_1 */
int phi_disc_vector(const phi_disc* d, int which, double* out);

/* ---- PMultigridHierarchy(disc, c, opt) (pmultigrid.hpp:217-224) ---------- */
int phi_hier_create(const phi_disc* d, double c, const phi_pmg_options* opt, phi_hier** out);
void phi_hier_free(phi_hier* h);
/* 0 op() = A_p, 1 smoother().lower, 2 smoother().upper, 100+l a_h[l] */
int phi_hier_export(const phi_hier* h, int which, int* n_rows, int* n_cols, int* nnz, int* row_offsets,
                    int* col_indices, double* values);
/* vcycle(b, x) (pmultigrid.hpp:256) on nrhs vectors with stride ld.
 * device_ptrs = 0: host arrays (copied in/out); 1: device arrays. */
int phi_hier_vcycle(phi_hier* h, const double* b, double* x, int nrhs, long long ld, int device_ptrs);
/* solve(b, x0, rel_tol, max_iter, fixed_cycles) (pmultigrid.hpp:271-307) per rhs;
 * x holds x0 on entry (ignored if x0_empty) and the solution on exit.
 * iters / converged / final_rel: nrhs entries each (host, nullable). */
int phi_hier_solve(phi_hier* h, const double* b, double* x, int nrhs, long long ld, double rel_tol,
                   int max_iter, int fixed_cycles, int x0_empty, int* iters, int* converged,
                   double* final_rel, int device_ptrs);
/* Y = A_p X for nrhs in {1, 16, 32, 64} vectors at once (spmv, sparse.hpp:114-124,
 * batched): X, Y are [n][nrhs] (right-hand sides contiguous); the SpMV / SpMM
 * kernels (reassociated sums). device_ptrs as above. */
int phi_hier_spmm(phi_hier* h, const double* x, double* y, int nrhs, int device_ptrs);
/* Kernel microbenchmark (BASELINE config 5): average device time (CUDA events)
 * of `reps` launches on seeded N(0,1) inputs -- which 0: the SpMM above,
 * which 1: one V(nu_pre, nu_post) cycle (pmultigrid.hpp:256-267) from x0 = 0
 * on nrhs right-hand sides (one CTA each).  flush_l2 = 1: read a 256 MB buffer
 * between reps (L2 left with clean lines), events around every single launch;
 * flush_l2 = 2 (which 0 only): 4 * reps back-to-back launches cycling through
 * four copies of the tiled operator (> L2 in total), events around the lot. */
int phi_hier_time(phi_hier* h, int which, int nrhs, int reps, int flush_l2, double* ms_out);
/* Algorithmic bytes of one V(nu_pre, nu_post) cycle on nrhs right-hand sides
 * (SURVEY.md 8(d) model: 8 B per stored operator nonzero per application and
 * batch + 8 B per vector entry read or written per right-hand side) */
int phi_hier_vcycle_bytes(const phi_hier* h, int nrhs, double* bytes);
/* Building blocks for parity tests (single vector, host arrays):
 * op 0 y = A_p x; 1 z = ilut_apply(r); 2 r1 = restrict_to_linear(r);
 * 3 x += prolong_from_linear(e1) (x in/out); 4 x1 = hmg_wcycle(b1, x1);
 * 5 x = gauss_seidel_sweep(a_h[arg], b, x, arg2 ? backward : forward) */
int phi_hier_unit(phi_hier* h, int op, int arg, int arg2, const double* in, int n_in, double* out,
                  int n_out);

/* ---- ThetaStepper (theta.hpp:92-146) ----------------------------------- */
int phi_stepper_create(const phi_disc* d, double kappa, double dt, double theta,
                       const phi_solver_config* cfg, phi_stepper** out);
void phi_stepper_free(phi_stepper* s);
/* step(u_prev, load, guess) for nrhs states (theta.hpp:132-137): x holds the
 * guess on entry (ignored if guess_empty) and Phi(u_prev) + ... on exit;
 * load may be null. Non-convergence of any rhs returns PHI_ERR_NOT_CONVERGED. */
int phi_stepper_step(phi_stepper* s, const double* u_prev, const double* load, double* x, int nrhs,
                     long long ld, int guess_empty, int* iters, int device_ptrs);
/* sequential_integrate (theta.hpp:216-237) with a given projected u0 and an
 * optional load schedule (steps x n, or n if steady). traj: (nt+1) x n host. */
int phi_sequential_integrate(phi_stepper* s, int nt, const double* u0, const double* loads, int load_steady,
                             double* traj, long long* solves, long long* iterations);

/* ---- MgritSolver (mgrit.hpp:50-331) ------------------------------------ */
int phi_mgrit_create(const phi_disc* d, const phi_problem* ps, const phi_mgrit_config* cfg,
                     const phi_solver_config* scfg, phi_mgrit** out);
void phi_mgrit_free(phi_mgrit* g);
int phi_mgrit_levels(const phi_mgrit* g, int* steps, double* dts);
/* solve() (mgrit.hpp:93-118); history: residual_history (nullable, cap entries) */
int phi_mgrit_solve(phi_mgrit* g, phi_mgrit_result* res, double* history, int history_cap);
/* level-0 free-dof trajectory after solve(): (steps+1) x n_free, host */
int phi_mgrit_trajectory(const phi_mgrit* g, double* out);
/* projected initial condition of the last initialize() (n_free) */
int phi_mgrit_initial(const phi_mgrit* g, double* out);
/* Phase-level entry points (for the time-sharded multi-GPU driver and tests) */
int phi_mgrit_initialize(phi_mgrit* g, double* g_norm);
int phi_mgrit_cycle(phi_mgrit* g, int level);
int phi_mgrit_residual_norm(phi_mgrit* g, int level, double* out);
/* ---- time-sharded multi-GPU support (paper_2107_05337_b200/timeshard.py,
 * DESIGN.md section 6): one rank per GPU owns the coarse intervals
 * [j_lo, j_hi) of level 0; coarser levels are replicated.  Per-point
 * reduction terms come back with zeros for points other ranks own, so an
 * elementwise sum over ranks plus the ordered host sum reproduces the
 * single-GPU reduction exactly. */
int phi_mgrit_set_range(phi_mgrit* g, int j_lo, int j_hi); /* j_hi = -1: all */
int phi_mgrit_initialize_state(phi_mgrit* g);               /* initialize() minus the g-norm */
/* steps_0 + 1 terms: [0] = |g_0|^2, [k] = squared norms of the load solves (mgrit.hpp:292-310) */
int phi_mgrit_gnorm_terms(phi_mgrit* g, double* terms);
/* steps_level + 1 per-point squared residuals (mgrit.hpp:200-214) */
int phi_mgrit_residual_terms(phi_mgrit* g, int level, double* terms);
/* per-solve p-MG cycle counts of the residual wave of `level` at the current
 * state (the Phi solves residual_norm performs, mgrit.hpp:197-214); iters:
 * steps_level + 1 host ints, [0] = 0.  The state is not modified. */
int phi_mgrit_residual_iters(phi_mgrit* g, int level, int* iters);
/* op 0 F-relaxation, 1 F+C relaxation, 2 restrict residual to level+1,
 * 3 inject the coarse correction into the C-points, 4 full cycle from level
 * (cycle_impl(level, cycle == F)), 5 the same without the F-schedule
 * (cycle_impl(level, false), the coarse call of the F-schedule's second pass,
 * mgrit.hpp:278-288) */
int phi_mgrit_phase(phi_mgrit* g, int level, int op);
/* copy `count` consecutive point vectors k0.. of level's u (which 0) or g (1)
 * to (set 0) or from (set 1) ptr, a host or device pointer */
int phi_mgrit_points(phi_mgrit* g, int level, int which, int k0, int count, double* ptr, int device_ptr,
                     int set);
/* [level-0 solves, level-0 p-MG cycles, coarser solves, coarser cycles] */
int phi_mgrit_stats(const phi_mgrit* g, long long* out4);
/* kernel launches issued by the last solve() (bench evidence) */
long long phi_mgrit_launches(const phi_mgrit* g);
/* replace the spline coefficients of a PHI_INIT_COEFFS problem (host array,
 * n_free); takes effect at the next solve() / initialize() */
int phi_mgrit_set_init_coeffs(phi_mgrit* g, const double* coeffs);
/* per-launch profiling of the Phi waves: when enabled, solve() records CUDA
 * events around every wave; phi_mgrit_wave_report returns the wave count and
 * the summed kernel time (ms) and algorithmic bytes (DESIGN.md byte model) */
int phi_mgrit_profile(phi_mgrit* g, int enable);
int phi_mgrit_wave_report(phi_mgrit* g, double* ms, double* bytes);
/* per MGRIT level (cap entries) of the last profiled solve: summed wave time
 * (ms), Phi solves, p-MG cycles, and the dependent steps of one single-RHS
 * V-cycle of that level's hierarchy (the latency model); call before
 * phi_mgrit_wave_report, which releases the records */
int phi_mgrit_wave_levels(phi_mgrit* g, double* ms, long long* points, long long* cycles, long long* chain_steps,
                          int cap);

/* ---- time sharding over GPUs (csrc/timeshard.cpp) -------
 * One rank per GPU owns a contiguous block of the level-0 coarse intervals;
 * operators and coarser levels are replicated.  With a communicator attached,
 * phi_mgrit_solve runs the sharded schedule in the engine: a halo shift of one
 * n-vector before every relaxation sweep, an allgather of the owned coarse
 * right-hand sides after the restriction, the coarse cycle replicated, and
 * point-ordered reductions (allgather of the owned per-point terms) -- the
 * same floating-point operations as one process, so the results are
 * identical for any rank count.  phi_mgrit_trajectory then gathers the
 * trajectory (collective: every rank calls it). */
typedef struct phi_comm phi_comm;
/* host-callback transport: host buffers; return 0 on success.
 * shift: send `count` values to rank + 1 (send null on the last rank) and
 * receive `count` from rank - 1 (recv null on rank 0);
 * allgather: recv[r * count ..] = rank r's send, in rank order. */
typedef struct {
    void* ctx;
    int (*shift)(void* ctx, const double* send, double* recv, long long count);
    int (*allgather)(void* ctx, const double* send, double* recv, long long count);
} phi_comm_ops;
/* NCCL transport (ncclSend/ncclRecv, ncclAllGather on the engine stream):
 * rank 0 creates the 128-byte id, the caller distributes it to every rank */
int phi_comm_nccl_unique_id(unsigned char* id128);
int phi_comm_create_nccl(const unsigned char* id128, int nranks, int rank, phi_comm** out);
int phi_comm_create_ops(const phi_comm_ops* ops, int nranks, int rank, phi_comm** out);
void phi_comm_free(phi_comm* c);
/* attach (null: detach -- single process); the comm must outlive its use */
int phi_mgrit_set_comm(phi_mgrit* g, phi_comm* c);

/* ---- host-side setup routines (no device needed) --------------------------
 * The inputs of the device assembly and of the coarse direct solve, exposed so
 * they can be pinned against the reference on a CPU-only box.
 *
 * phi_setup_tables_1d: the per-direction quadrature / basis tables of an open
 * uniform knot vector on [0,1] -- gauss_legendre_01 (quadrature.hpp:17-44),
 * open_uniform_knots (spline.hpp:48-63), eval_values_and_derivs
 * (spline.hpp:104-130), laid out as detail::DirTables (assembly.hpp:124-151):
 * nodes/weights [e*nq + q], vals/ders [(e*nq + q)*(degree+1) + a], first [e].
 * phi_setup_dense_lu: DenseLU's factors and permutation (solvers.hpp:136-167)
 * of a dense row-major n x n matrix; lu: n*n, piv: n.
 * phi_setup_level_steps: the time-grid hierarchy rule of
 * MgritSolver::build_levels (mgrit.hpp:217-233); cycle as phi_mgrit_config.
 * Writes at most cap step counts, *n_levels = the number of levels. */
int phi_setup_tables_1d(int degree, int n_elements, int nq, double* nodes, double* weights, double* vals,
                        double* ders, int* first);
int phi_setup_dense_lu(int n, const double* a, double* lu, int* piv);
int phi_setup_level_steps(int nt, int m, int cycle, int coarse_floor, int* steps, int cap, int* n_levels);

/* Developer knob (not part of the reference API): warps used by the sync-free
 * triangular solves / Gauss-Seidel sweeps and the readiness-poll back-off. */
int phi_dev_tuning(int tri_warps, int gs_warps, int sleep_ns);
/* Developer timing trace (enabled by phi_dev_tuning(.., .., -1)): copies up to
 * n clock64 stamps into out, returns the count. */
int phi_dev_trace(long long* out, int n);

#ifdef __cplusplus
}
#endif
#endif
