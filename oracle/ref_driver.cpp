// TEST INFRASTRUCTURE ONLY -- never linked into the product.
//
// Thin extern "C" driver over the UNMODIFIED reference library (header-only
// C++20 `miga`, /root/reference/proj/include).  It is compiled from the
// reference headers where they lie (see oracle/Makefile) into
// oracle/_ref/libmiga_ref.so and is used (a) to pin the C restatement in
// oracle/phi_oracle.c, (b) to generate the golden fixtures under tests/golden,
// and (c) as the CPU arm of bench.py (`--impl reference`, cpu_baseline kind
// "reference").  No reference source is copied: this file only calls the
// reference's public API:
//   SpatialDiscretization::build      pmultigrid.hpp:94-158
//   PMultigridHierarchy               pmultigrid.hpp:215-324
//   ThetaStepper                      theta.hpp:92-146
//   sequential_integrate              theta.hpp:216-237
//   MgritSolver / mgrit_solve         mgrit.hpp:50-331
//   detail::DirTables, DenseLU        assembly.hpp:124-151, solvers.hpp:102-172
#include <chrono>
#include <cmath>
#include <cstring>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "miga/mgrit.hpp"

using namespace miga;

namespace {

thread_local std::string g_err;

int fail(const std::exception& e) {
    g_err = e.what();
    return 1;
}

// CSR export helper: two-pass (call with null arrays to get sizes).
int export_csr(const SparseMatrix& a, int* n_rows, int* n_cols, int* nnz, int* ro, int* ci,
               double* v) {
    if (n_rows) *n_rows = a.n_rows;
    if (n_cols) *n_cols = a.n_cols;
    if (nnz) *nnz = a.nnz();
    if (ro) std::memcpy(ro, a.row_offsets.data(), sizeof(int) * (a.n_rows + 1));
    if (ci) std::memcpy(ci, a.col_indices.data(), sizeof(int) * a.nnz());
    if (v) std::memcpy(v, a.values.data(), sizeof(double) * a.nnz());
    return 0;
}

struct RefDisc {
    std::shared_ptr<SpatialDiscretization> d;
};

struct RefHier {
    std::shared_ptr<SpatialDiscretization> d;
    std::unique_ptr<PMultigridHierarchy> h;
};

// Source / initial-condition kinds shared with the engine's C-ABI
// (include/phi_engine.h: PHI_SOURCE_*, PHI_INIT_*).
SourceTerm make_source(int kind, double param) {
    switch (kind) {
        case 0:
            return SourceTerm::constant(param);
        case 1: {
            const double amp = param;
            return SourceTerm::transient([amp](double x, double y, double t) {
                return amp * std::exp(-t) * std::sin(M_PI * x) * std::sin(M_PI * y);
            });
        }
        case 2: {
            const double amp = param;
            return SourceTerm::steady(
                [amp](double x, double y) { return amp * std::sin(M_PI * x) * std::sin(M_PI * y); });
        }
        default:
            throw std::invalid_argument("unknown source kind");
    }
}

// Spline initial condition u0 = sum_i c_i phi_i over the free dofs, evaluated
// through the reference's own tensor basis evaluation (spline.hpp:165-186).
std::function<double(double, double)> make_initial(int kind, const SpatialDiscretization* d,
                                                   const double* coeffs) {
    if (kind == 0) return {};
    if (kind == 1) return [](double x, double y) { return std::sin(M_PI * x) * std::sin(M_PI * y); };
    if (kind == 2) {
        auto c = std::make_shared<std::vector<double>>(coeffs, coeffs + d->dofmap_p.n_free);
        const TensorBasis2D basis = d->basis_p;
        const DofMap dm = d->dofmap_p;
        return [c, basis, dm](double x, double y) {
            const auto s = eval_tensor(basis, x, y, TensorDeriv::value);
            double v = 0.0;
            for (std::size_t i = 0; i < s.indices.size(); ++i) {
                const int f = dm.free_of_global[s.indices[i]];
                if (f >= 0) v += (*c)[f] * s.values[i];
            }
            return v;
        };
    }
    throw std::invalid_argument("unknown initial kind");
}

struct RefMgrit {
    std::shared_ptr<SpatialDiscretization> d;
    ProblemSpec ps;
    MgritConfig cfg;
    SpatialSolverConfig scfg;
    std::unique_ptr<MgritSolver> solver;
    MgritResult res;
    double wall = 0.0;
};

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

void* ref_disc_build(int degree, int mesh_exponent, int workers) {
    try {
        ThreadPool pool(workers > 0 ? workers : 1);
        auto* r = new RefDisc;
        r->d = std::make_shared<SpatialDiscretization>(
            SpatialDiscretization::build(GeometryMap::unit_square(), degree, mesh_exponent, &pool));
        return r;
    } catch (const std::exception& e) {
        fail(e);
        return nullptr;
    }
}

void ref_disc_free(void* p) { delete static_cast<RefDisc*>(p); }

// info: [n_free_p, n_h_levels, n_elements, degree]
int ref_disc_info(void* p, int* info) {
    auto& d = *static_cast<RefDisc*>(p)->d;
    info[0] = d.dofmap_p.n_free;
    info[1] = static_cast<int>(d.h_chain.size());
    info[2] = d.n_elements;
    info[3] = d.degree;
    return 0;
}

// which: 0 mass_p, 1 stiff_p, 2 transfer_p1, 100+l h mass, 200+l h stiff, 300+l embed
int ref_disc_csr(void* p, int which, int* n_rows, int* n_cols, int* nnz, int* ro, int* ci, double* v) {
    auto& d = *static_cast<RefDisc*>(p)->d;
    const SparseMatrix* a = nullptr;
    if (which == 0) a = &d.mass_p;
    else if (which == 1) a = &d.stiff_p;
    else if (which == 2) a = &d.transfer_p1;
    else if (which >= 100 && which < 200) a = &d.h_chain.at(which - 100).mass;
    else if (which >= 200 && which < 300) a = &d.h_chain.at(which - 200).stiff;
    else if (which >= 300 && which < 400) a = &d.h_chain.at(which - 300).embed;
    if (!a) return 1;
    return export_csr(*a, n_rows, n_cols, nnz, ro, ci, v);
}

// which: 0 inv_lumped_p, 1 inv_lumped_1
int ref_disc_vec(void* p, int which, double* out) {
    auto& d = *static_cast<RefDisc*>(p)->d;
    const Vector& v = which == 0 ? d.inv_lumped_p : d.inv_lumped_1;
    std::memcpy(out, v.data(), sizeof(double) * v.size());
    return static_cast<int>(v.size());
}

void* ref_hier_build(void* disc, double c, int nu_pre, int nu_post, int gs_pre, int gs_post,
                     double tau, int fill) {
    try {
        auto* h = new RefHier;
        h->d = static_cast<RefDisc*>(disc)->d;
        PMultigridOptions opt;
        opt.nu_pre = nu_pre;
        opt.nu_post = nu_post;
        opt.gs_pre = gs_pre;
        opt.gs_post = gs_post;
        opt.ilut_tau = tau;
        opt.ilut_fill = fill;
        h->h = std::make_unique<PMultigridHierarchy>(*h->d, c, opt);
        return h;
    } catch (const std::exception& e) {
        fail(e);
        return nullptr;
    }
}

void ref_hier_free(void* p) { delete static_cast<RefHier*>(p); }

// which: 0 A_p, 1 L, 2 U, 100+l a_h[l]
int ref_hier_csr(void* p, int which, int* n_rows, int* n_cols, int* nnz, int* ro, int* ci, double* v) {
    auto& h = *static_cast<RefHier*>(p)->h;
    const SparseMatrix* a = nullptr;
    if (which == 0) a = &h.op();
    else if (which == 1) a = &h.smoother().lower;
    else if (which == 2) a = &h.smoother().upper;
    else if (which >= 100) {
        const auto lv = h.hmg_levels();
        a = lv.a.at(which - 100);
    }
    if (!a) return 1;
    return export_csr(*a, n_rows, n_cols, nnz, ro, ci, v);
}

int ref_hier_vcycle(void* p, const double* b, double* x, int n, int nrhs) {
    try {
        auto& h = *static_cast<RefHier*>(p)->h;
        for (int r = 0; r < nrhs; ++r) {
            Vector bb(b + (size_t)r * n, b + (size_t)(r + 1) * n);
            Vector xx(x + (size_t)r * n, x + (size_t)(r + 1) * n);
            h.vcycle(bb, xx);
            std::memcpy(x + (size_t)r * n, xx.data(), sizeof(double) * n);
        }
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// Parallel batched V-cycle with the reference's own thread pool, for the CPU
// baseline of the config-5 microbench (one shared, immutable hierarchy;
// pmultigrid.hpp:212-214).
double ref_hier_vcycle_timed(void* p, const double* b, double* x, int n, int nrhs, int workers) {
    auto& h = *static_cast<RefHier*>(p)->h;
    ThreadPool pool(workers > 0 ? workers : 1);
    const auto t0 = std::chrono::steady_clock::now();
    pool.parallel_for(nrhs, [&](std::size_t r) {
        Vector bb(b + r * n, b + (r + 1) * n);
        Vector xx(x + r * n, x + (r + 1) * n);
        h.vcycle(bb, xx);
        std::memcpy(x + r * n, xx.data(), sizeof(double) * n);
    });
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

int ref_hier_solve(void* p, const double* b, double* x, int n, double rel_tol, int max_iter,
                   int fixed_cycles, int x0_empty, int* iters, int* converged, double* final_rel,
                   double* history, int history_cap) {
    try {
        auto& h = *static_cast<RefHier*>(p)->h;
        Vector bb(b, b + n);
        Vector x0;
        if (!x0_empty) x0.assign(x, x + n);
        auto res = h.solve(bb, x0, rel_tol, max_iter, fixed_cycles);
        std::memcpy(x, res.x.data(), sizeof(double) * n);
        *iters = res.iterations;
        *converged = res.converged ? 1 : 0;
        *final_rel = res.final_relative_residual;
        for (int i = 0; i < (int)res.residual_history.size() && i < history_cap; ++i)
            history[i] = res.residual_history[i];
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// Exported building blocks for unit-level pinning.
int ref_ilut_apply(void* p, const double* r, double* z, int n) {
    auto& h = *static_cast<RefHier*>(p)->h;
    Vector rr(r, r + n), zz;
    ilut_apply(h.smoother(), rr, zz);
    std::memcpy(z, zz.data(), sizeof(double) * n);
    return 0;
}

int ref_restrict(void* p, const double* r, double* r1, int n) {
    auto& h = *static_cast<RefHier*>(p)->h;
    Vector rr(r, r + n);
    Vector out = h.restrict_to_linear(rr);
    std::memcpy(r1, out.data(), sizeof(double) * out.size());
    return 0;
}

int ref_prolong(void* p, const double* e1, int n1, double* ep) {
    auto& h = *static_cast<RefHier*>(p)->h;
    Vector ee(e1, e1 + n1);
    Vector out = h.prolong_from_linear(ee);
    std::memcpy(ep, out.data(), sizeof(double) * out.size());
    return 0;
}

int ref_hmg_wcycle(void* p, const double* b1, double* x1, int n1) {
    auto& h = *static_cast<RefHier*>(p)->h;
    Vector bb(b1, b1 + n1), xx(x1, x1 + n1);
    hmg_wcycle(h.hmg_levels(), 0, bb, xx);
    std::memcpy(x1, xx.data(), sizeof(double) * n1);
    return 0;
}

int ref_gs_sweep(void* p, int level, const double* b, double* x, int n, int backward) {
    auto& h = *static_cast<RefHier*>(p)->h;
    const auto lv = h.hmg_levels();
    Vector bb(b, b + n), xx(x, x + n);
    gauss_seidel_sweep(*lv.a.at(level), bb, xx,
                       backward ? SweepDirection::backward : SweepDirection::forward);
    std::memcpy(x, xx.data(), sizeof(double) * n);
    return 0;
}

int ref_coarse_solve(void* p, const double* b, double* x, int n) {
    auto& h = *static_cast<RefHier*>(p)->h;
    const auto lv = h.hmg_levels();
    Vector out = lv.coarse_lu->solve(Vector(b, b + n));
    std::memcpy(x, out.data(), sizeof(double) * n);
    return 0;
}

// ---- theta stepper / integration / MGRIT ---------------------------------

// Spline evaluation of free coefficients at (x, y) -> used to build golden
// initial conditions consistently with the reference's basis.
// spatial_kind: SpatialSolverKind (theta.hpp:64), 0 pmg, 1 cg
void* ref_mgrit_create_kind(int degree, int mesh_exponent, double kappa, double t_final, int nt,
                            double theta, int source_kind, double source_param, int init_kind,
                            const double* init_coeffs, int cycle, int relax, int m,
                            double halt_tol, int max_iter, int coarse_floor, int workers,
                            int spatial_kind, double rel_tol, int sp_max_iter) {
    try {
        auto* g = new RefMgrit;
        ThreadPool pool(workers > 0 ? workers : 1);
        g->d = std::make_shared<SpatialDiscretization>(
            SpatialDiscretization::build(GeometryMap::unit_square(), degree, mesh_exponent, &pool));
        g->ps.kappa = kappa;
        g->ps.t_final = t_final;
        g->ps.n_time_steps = nt;
        g->ps.theta = theta;
        g->ps.degree = degree;
        g->ps.mesh_exponent = mesh_exponent;
        g->ps.source = make_source(source_kind, source_param);
        g->ps.initial = make_initial(init_kind, g->d.get(), init_coeffs);
        g->cfg.cycle = cycle == 0 ? CycleType::v : (cycle == 1 ? CycleType::f : CycleType::two_level);
        g->cfg.relaxation = relax == 0 ? RelaxType::f : RelaxType::fcf;
        g->cfg.m = m;
        g->cfg.halt_tol = halt_tol;
        g->cfg.max_iter = max_iter;
        g->cfg.coarse_floor = coarse_floor;
        g->cfg.workers = workers > 0 ? workers : 1;
        g->scfg.kind = spatial_kind == 1 ? SpatialSolverKind::cg : SpatialSolverKind::pmg;
        g->scfg.rel_tol = rel_tol;
        g->scfg.max_iter = sp_max_iter;
        g->solver = std::make_unique<MgritSolver>(g->d, g->ps, g->cfg, g->scfg);
        return g;
    } catch (const std::exception& e) {
        fail(e);
        return nullptr;
    }
}

void* ref_mgrit_create(int degree, int mesh_exponent, double kappa, double t_final, int nt,
                       double theta, int source_kind, double source_param, int init_kind,
                       const double* init_coeffs, int cycle, int relax, int m, double halt_tol,
                       int max_iter, int coarse_floor, int workers, double rel_tol,
                       int sp_max_iter) {
    return ref_mgrit_create_kind(degree, mesh_exponent, kappa, t_final, nt, theta, source_kind,
                                 source_param, init_kind, init_coeffs, cycle, relax, m, halt_tol,
                                 max_iter, coarse_floor, workers, 0, rel_tol, sp_max_iter);
}

void ref_mgrit_free(void* p) { delete static_cast<RefMgrit*>(p); }

// info: [n_levels, steps_0, steps_1, ..., ]
int ref_mgrit_levels(void* p, int* steps, double* dts) {
    auto& g = *static_cast<RefMgrit*>(p);
    const int L = g.solver->n_levels();
    for (int l = 0; l < L; ++l) {
        steps[l] = g.solver->level(l).steps;
        dts[l] = g.solver->level(l).dt;
    }
    return L;
}

// Times MgritSolver::solve() only (the bench.hpp:146-149 window).
int ref_mgrit_solve(void* p, int* iterations, int* converged, double* g_norm, double* final_rel,
                    long long* solves, double* mean_iters, double* history, int history_cap,
                    double* wall) {
    try {
        auto& g = *static_cast<RefMgrit*>(p);
        const auto t0 = std::chrono::steady_clock::now();
        g.res = g.solver->solve();
        g.wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        *iterations = g.res.iterations;
        *converged = g.res.converged ? 1 : 0;
        *g_norm = g.res.g_norm;
        *final_rel = g.res.final_relative_residual;
        *solves = g.res.total_spatial_solves;
        *mean_iters = g.res.mean_spatial_iterations;
        for (int i = 0; i < (int)g.res.residual_history.size() && i < history_cap; ++i)
            history[i] = g.res.residual_history[i];
        *wall = g.wall;
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// Level-0 free-dof trajectory after solve(): (steps+1) x n_free.
int ref_mgrit_trajectory(void* p, double* out) {
    auto& g = *static_cast<RefMgrit*>(p);
    const auto& lev = g.solver->level(0);
    const int n = g.d->dofmap_p.n_free;
    for (int k = 0; k <= lev.steps; ++k) std::memcpy(out + (size_t)k * n, lev.u[k].data(), sizeof(double) * n);
    return 0;
}

// Time initialize() plus `cycles` MGRIT cycles with their residual norms
// (for extrapolating runs too long to finish on the CPU).
int ref_mgrit_partial(void* p, int cycles, double* t_init, double* t_cycles, double* history) {
    try {
        auto& g = *static_cast<RefMgrit*>(p);
        auto t0 = std::chrono::steady_clock::now();
        g.solver->initialize();
        *t_init = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        const double denom = g.solver->g_norm() > 0 ? g.solver->g_norm() : 1.0;
        t0 = std::chrono::steady_clock::now();
        for (int it = 0; it < cycles; ++it) {
            g.solver->mgrit_cycle(0);
            history[it] = g.solver->residual_norm(0) / denom;
        }
        *t_cycles = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// Projected initial condition and load schedule as the reference builds them
// (theta.hpp:150-160, 165-210), for handing identical inputs to other arms.
int ref_mgrit_initial(void* p, double* u0) {
    auto& g = *static_cast<RefMgrit*>(p);
    Vector v = project_initial(*g.d, g.ps.initial);
    std::memcpy(u0, v.data(), sizeof(double) * v.size());
    return static_cast<int>(v.size());
}

int ref_load_terms(void* p, double* out) {
    auto& g = *static_cast<RefMgrit*>(p);
    const double dt = g.ps.dt();
    LoadSchedule ls = LoadSchedule::build(*g.d, g.ps.source, dt, g.ps.theta, g.ps.n_time_steps);
    const int n = g.d->dofmap_p.n_free;
    if (ls.empty()) return 0;
    for (int k = 1; k <= g.ps.n_time_steps; ++k)
        std::memcpy(out + (size_t)(k - 1) * n, ls.term(k).data(), sizeof(double) * n);
    return 1;
}

int ref_sequential_integrate(void* p, double* out, long long* solves, long long* iters) {
    try {
        auto& g = *static_cast<RefMgrit*>(p);
        SolveStats st;
        auto traj = sequential_integrate(*g.d, g.ps, g.scfg, &st);
        const int n = g.d->dofmap_p.n_free;
        for (std::size_t k = 0; k < traj.size(); ++k)
            std::memcpy(out + k * n, traj[k].data(), sizeof(double) * n);
        *solves = st.solves.load();
        *iters = st.iterations.load();
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// initialize() / mgrit_cycle(l) / residual_norm(l) one at a time (mgrit.hpp:76-91,
// 185, 197-214), so a test can stop at any iteration and compare state.
int ref_mgrit_initialize(void* p, double* g_norm) {
    try {
        auto& g = *static_cast<RefMgrit*>(p);
        g.solver->initialize();
        *g_norm = g.solver->g_norm();
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

int ref_mgrit_cycle(void* p, int level) {
    try {
        static_cast<RefMgrit*>(p)->solver->mgrit_cycle(level);
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

int ref_mgrit_residual_norm(void* p, int level, double* out) {
    try {
        *out = static_cast<RefMgrit*>(p)->solver->residual_norm(level);
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// Copy `count` point vectors k0.. of level l's u (which 0) or g (1).
int ref_mgrit_points(void* p, int level, int which, int k0, int count, double* out) {
    auto& g = *static_cast<RefMgrit*>(p);
    const auto& lev = g.solver->level(level);
    const int n = g.d->dofmap_p.n_free;
    const auto& arr = which == 0 ? lev.u : lev.g;
    for (int k = 0; k < count; ++k) std::memcpy(out + (size_t)k * n, arr.at(k0 + k).data(), sizeof(double) * n);
    return 0;
}

// Per-solve p-multigrid iteration counts of the residual wave of level l at
// the solver's current state: for every point k = 1..steps the Phi solve that
// residual_norm(l) performs (mgrit.hpp:197-214 -> step_value 261-269:
// stepper->step(u[k-1], load(k), guess u[k])), each with its own SolveStats
// (theta.hpp:77-85), on `workers` threads.  iters: steps + 1 entries, [0] = 0.
// The state is not modified.
int ref_mgrit_residual_iters(void* p, int level, int workers, int* iters) {
    try {
        auto& g = *static_cast<RefMgrit*>(p);
        const auto& lev = g.solver->level(level);
        const int steps = lev.steps;
        iters[0] = 0;
        std::vector<std::string> errs(workers > 0 ? workers : 1);
        auto run = [&](int w, int nw) {
            try {
                for (int k = 1 + w; k <= steps; k += nw) {
                    SolveStats st;
                    static const Vector kEmpty;
                    const Vector& load = level == 0 ? lev.loads.term(k) : kEmpty;
                    (void)lev.stepper->step(lev.u[k - 1], load, lev.u[k], &st);
                    iters[k] = static_cast<int>(st.iterations.load());
                }
            } catch (const std::exception& e) {
                errs[w] = e.what();
            }
        };
        const int nw = workers > 0 ? workers : 1;
        std::vector<std::thread> th;
        for (int w = 0; w < nw; ++w) th.emplace_back(run, w, nw);
        for (auto& t : th) t.join();
        for (const auto& e : errs)
            if (!e.empty()) throw std::runtime_error(e);
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// The reference's per-direction quadrature / basis tables of an open uniform
// knot vector on [0, 1] (detail::DirTables::build over gauss_legendre_01 and
// eval_values_and_derivs).  Arrays sized by the caller: nodes/weights nel*nq,
// vals/ders nel*nq*(degree+1), first nel.
int ref_tables_1d(int degree, int n_elements, int nq, double* nodes, double* weights, double* vals,
                  double* ders, int* first) {
    try {
        const KnotVector kv = open_uniform_knots(degree, n_elements, 0.0, 1.0);
        const auto t = detail::DirTables::build(kv, nq);
        std::memcpy(nodes, t.quad.nodes.data(), sizeof(double) * t.quad.nodes.size());
        std::memcpy(weights, t.quad.weights.data(), sizeof(double) * t.quad.weights.size());
        std::memcpy(vals, t.vals.data(), sizeof(double) * t.vals.size());
        std::memcpy(ders, t.ders.data(), sizeof(double) * t.ders.size());
        std::memcpy(first, t.first.data(), sizeof(int) * t.first.size());
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// DenseLU(a).solve(b) for a dense row-major n x n matrix (zeros are not stored).
int ref_dense_solve(int n, const double* a, const double* b, double* x) {
    try {
        SparseMatrix m;
        m.n_rows = m.n_cols = n;
        m.row_offsets.assign(1, 0);
        for (int i = 0; i < n; ++i) {
            for (int j = 0; j < n; ++j)
                if (a[static_cast<std::size_t>(i) * n + j] != 0.0) {
                    m.col_indices.push_back(j);
                    m.values.push_back(a[static_cast<std::size_t>(i) * n + j]);
                }
            m.row_offsets.push_back(m.nnz());
        }
        const Vector out = DenseLU(m).solve(Vector(b, b + n));
        std::memcpy(x, out.data(), sizeof(double) * n);
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

}  // extern "C"
