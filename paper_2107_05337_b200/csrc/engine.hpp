// Host-side engine objects mirroring the reference's operator API
// (proj/include/miga): SpatialDiscretization, PMultigridHierarchy,
// ThetaStepper and MgritSolver.  They own device-resident operators and
// launch the kernels in phi_kernels.cu / assembly.cu.  All compute runs on the
// GPU; the host only builds the ILUT factors / coarse LU / solve schedules and
// drives the MGRIT control flow.
#pragma once

#include <memory>
#include <string>
#include <vector>

#include "common.hpp"
#include "device_types.cuh"
#include "phi_kernels.cuh"
#include "setup_host.hpp"
#include "timeshard.hpp"

namespace phi {

struct StencilBuf {
    int ru = 0, rv = 0, cu = 0, cv = 0, lo = 0, hi = 0;
    DevBuf<double> vals;
    DevStencil view() const { return DevStencil{ru, rv, cu, cv, lo, hi, vals.get()}; }
    size_t n_rows() const { return (size_t)ru * rv; }
    size_t width() const { return (size_t)(hi - lo + 1); }
    size_t size() const { return n_rows() * width() * width(); }
};

struct Tables1DDev {
    Tables1D host;
    DevBuf<double> w, vals, ders;
    DevTables1D view() const { return DevTables1D{host.p, host.nq, host.nel, w.get(), vals.get(), ders.get()}; }
};

/// SpatialDiscretization::build (pmultigrid.hpp:94-158), unit square, on device.
class Disc {
public:
    static std::shared_ptr<Disc> build(int degree, int mesh_exponent, cudaStream_t s = nullptr);

    int degree = 0, mesh_exponent = 0, n_elements = 0;
    int nf_p = 0, n_p = 0;  // free dofs per direction / total, order p
    int nf_1 = 0, n_1 = 0;  // order 1 on the fine mesh
    StencilBuf M, K;        // order p, free rows, offsets [-p, p]
    StencilBuf T, Tt;       // transfer p->1 and its transpose
    DevBuf<double> inv_lp, inv_l1;

    struct HLevel {
        int n_elements = 0, nf = 0, n = 0;
        StencilBuf M, K;
        HostCsr E, Et;  // embedding from the next coarser level (empty on the coarsest)
        DevBuf<int> e_ro, e_ci, et_ro, et_ci;
        DevBuf<double> e_v, et_v;
    };
    std::vector<HLevel> h;

    Tables1DDev tab_p;               // order-p tables (nq = p + 1) for load assembly
    DevBuf<double> sin_tab;          // sin(pi * node) per (element, q), host libm
    std::vector<double> sin_host;

    /// Free-dof CSR of a stencil matrix (download), reference layout.
    HostCsr to_csr(const StencilBuf& a) const;
    /// Load vector (free dofs) on device: see launch_assemble_load kinds.
    void assemble_load(int kind, double c0, double c1, const double* coeffs_dev, double* out,
                       cudaStream_t s) const;
};

struct HierOptions {  // PMultigridOptions (pmultigrid.hpp:161-168)
    double ilut_tau = 1e-13;
    int ilut_fill = 0;
    int nu_pre = 1, nu_post = 1, gs_pre = 2, gs_post = 2;
    int exact = 0;  // 1: the reference's summation order (bit-identical), 0: reassociated sums
    int dense_coarse_max = 256;    // reassociated mode: dense W-cycle operator from the first h-level this small
    int dense_cluster_max = 1024;  // ... in cluster mode (the product is split over the cluster's SMs)
};

struct SolverConfig {  // SpatialSolverConfig (theta.hpp:66-75)
    int kind = 0;  // SpatialSolverKind (theta.hpp:64): 0 pmg, 1 cg (Jacobi-preconditioned)
    double rel_tol = 1e-12;
    int max_iter = 400;
    int fixed_cycles = 0;
    HierOptions pmg;
};

/// Batch workspace (one slot per resident CTA) shared by objects on one stream.
struct Workspace {
    DevBuf<double> buf;
    long long stride = 0;
    int slots = 0;
    void ensure(const DevHier& H);
};

/// PMultigridHierarchy(disc, c, opt) (pmultigrid.hpp:215-324) on device.
class Hier {
public:
    /// cg_only: the CG kind's left-hand operator alone (A = M + c K; no ILUT,
    /// no h-levels -- the reference builds no hierarchy then, theta.hpp:99-102)
    Hier(std::shared_ptr<const Disc> disc, double c, const HierOptions& opt, cudaStream_t s = nullptr,
         bool cg_only = false);
    std::shared_ptr<const Disc> disc;
    double c = 0.0;
    bool cg_only = false;
    HierOptions opt;
    StencilBuf A;                       // M + c K
    std::vector<StencilBuf> a_h;        // per h-level
    HostCsr L_host, U_host;             // ILUT factors (host copy)
    TriPlan Lp, Up;
    struct TriDev {
        DevBuf<unsigned char> stream;
        DevBuf<int> block_info;
        int n_units = 0, n_blocks = 0, max_unit_bytes = 0;
        int prime[2 * (kTriSlots - 1)] = {};
    } Ld, Ud;
    std::vector<TriPlan> gs_plans;  // per h-level (but the coarsest): forward, backward
    std::vector<TriDev> gs_dev;
    struct BlkDev {
        DevBuf<unsigned char> stream;
        DevBuf<int> table;
        int n = 0, n_blocks = 0, parts = 1, mf0 = 0, lookahead = 0, max_unit_bytes = 0, win = 0, desc = 0;
        DevBlk view() const;
    } Lbd, Ubd;
    std::vector<BlkDev> gsb_dev;  // per h-level (but the coarsest): forward, backward
    std::vector<DevBuf<double>> gsl_dev;  // per h-level: line Gauss-Seidel coefficients (reassociated mode)
    DenseLUHost coarse;
    DevBuf<double> coarse_lu;
    int dense_level = -1;      // reassociated mode: W-cycle subtree collapsed to a dense operator
    DevBuf<double> a_tile[2];  // tiled copies of A for the streaming SpMV (0) / SpMM (1), built on first use
    const double* a_tiled(cudaStream_t s, int kind) {
        if (!a_tile[kind].get()) {
            a_tile[kind].alloc(tile_doubles(A.view(), kind));
            launch_tile(A.view(), a_tile[kind].get(), kind, s);
        }
        return a_tile[kind].get();
    }
    DevBuf<double> dense_op;
    int dense_level_cl = -1;   // the same for cluster mode (single-right-hand-side waves)
    DevBuf<double> dense_op_cl;
    DevBuf<int> coarse_piv;

    DevHier view(const SolverConfig& cfg) const;
    HostCsr a_h_csr(int l) const;
    /// Dependent steps on the critical path of one single-right-hand-side
    /// V-cycle (reassociated mode, cluster W-cycle): ILUT blocks of the
    /// smoothings, Gauss-Seidel lines / blocks of the W-cycle sweeps, one
    /// step per dense coarse application -- the latency model of bench.py.
    long long chain_steps() const;
    /// Byte model of one V-cycle: operator entries read per
    /// batch, vector entries read or written per right-hand side.
    double vcycle_matrix_entries() const;
    double vcycle_vector_entries() const;
};

/// Message of a failed spatial solve (theta.hpp:116-118, 123-124; a negative
/// residual marks a CG breakdown, solvers.hpp:59).
std::string spatial_failure(int kind, double rel);

/// ThetaStepper (theta.hpp:92-146): Phi(u) = (M + k dt th K)^-1 ((M - k dt (1-th) K) u + load).
class Stepper {
public:
    Stepper(std::shared_ptr<const Disc> disc, double kappa, double dt, double theta,
            const SolverConfig& cfg, cudaStream_t s = nullptr);
    std::shared_ptr<const Disc> disc;
    double kappa, dt, theta;
    SolverConfig cfg;
    std::unique_ptr<Hier> hier;
    StencilBuf Aminus;
    DevHier H;
};

/// Fewest coarse intervals of a level for which the coarse march is overlapped
/// with that level's interpolation (Mgrit::coarse_overlapped).
constexpr int kOverlapMinIntervals = 32;

struct MgritOptions {  // MgritConfig (mgrit.hpp:17-31)
    int cycle = 0;  // 0 V, 1 F, 2 two-level
    int relax = 1;  // 0 F, 1 FCF
    int m = 2;
    double halt_tol = 1e-10;
    int max_iter = 50;
    int coarse_floor = 8;
};

struct ProblemOptions {  // ProblemSpec (theta.hpp:42-62) + source / initial kinds
    double kappa = 1.0, t_final = 0.1, theta = 1.0;
    int n_time_steps = 64;
    int source_kind = 0;  // 0 constant, 1 amp e^-t sin sin (transient), 2 amp sin sin (steady)
    double source_param = 1.0;
    int init_kind = 0;  // 0 zero, 1 sin sin, 2 spline coefficients
    std::vector<double> init_coeffs;
    // optional caller-provided level-0 load terms (steps x n) -- drop-in path
    std::vector<double> load_terms;
    int load_terms_steady = 0;
};

struct MgritResultHost {
    int iterations = 0;
    bool converged = false;
    double g_norm = 0.0, final_relative_residual = 0.0;
    std::vector<double> residual_history;
    long long total_spatial_solves = 0;
    double mean_spatial_iterations = 0.0;
};

/// MgritSolver (mgrit.hpp:50-320) with the space-time state resident on device.
/// Step counts of the MGRIT time levels, finest first (the hierarchy rule of
/// MgritSolver::build_levels, mgrit.hpp:217-233).  cycle: 0 V, 1 F, 2 two-level.
std::vector<int> mgrit_level_steps(int nt, int m, int cycle, int coarse_floor);

class Mgrit {
public:
    Mgrit(std::shared_ptr<const Disc> disc, const ProblemOptions& ps, const MgritOptions& cfg,
          const SolverConfig& scfg, cudaStream_t s = nullptr);
    MgritResultHost solve();
    void initialize();
    void mgrit_cycle(int l);
    double residual_norm(int l);

    // ---- time-sharded driver support (one rank per GPU, see timeshard.py):
    // level 0 works on coarse intervals [j_lo, j_hi) only; coarser levels are
    // replicated.  Per-point reduction terms are returned with zeros for the
    // points other ranks own, so an elementwise sum over ranks followed by the
    // ordered host sum reproduces the single-GPU reduction exactly.
    int j_lo = 0, j_hi = -1;  // -1: all intervals
    void set_range(int lo, int hi);
    void initialize_state();                     // initialize() without the g-norm
    void gnorm_terms(double* host);              // steps_0 + 1 terms: [0] = |g_0|^2
    void residual_terms(int l, double* host);    // steps_l + 1 terms
    /// per-solve p-MG cycle counts of the residual wave (steps_l + 1 entries, [0] = 0)
    void residual_iters(int l, int* host);
    void phase(int l, int op);                   // see phi_mgrit_phase
    void points(int l, int which, int k0, int count, double* ptr, bool device, bool set);
    void stats(long long* out4) const;           // level-0 solves, iters; coarser solves, iters
    int n_levels() const { return (int)levels.size(); }

    // ---- time sharding in the C++ host (timeshard.cpp): with a communicator
    // attached, solve() runs the sharded schedule itself (halo shifts,
    // allgathered coarse right-hand sides, point-ordered reductions)
    Comm* comm = nullptr;
    bool traj_gathered = false;
    void set_comm(Comm* c);
    MgritResultHost solve_sharded();
    /// level-0 trajectory of every rank's points on every rank (collective)
    void gather_trajectory();

    struct Level {
        int steps = 0;
        double dt = 0.0;
        std::unique_ptr<Stepper> stepper;
        DevBuf<double> u, g;
        DevBuf<int> kF, kR, kAll;
    };
    std::vector<Level> levels;
    std::shared_ptr<const Disc> disc;
    ProblemOptions ps;
    MgritOptions cfg;
    SolverConfig scfg;
    cudaStream_t stream = nullptr;
    Workspace ws;
    DevBuf<double> loads;  // level-0 terms: steady (n) or transient (steps x n)
    bool has_loads = false, loads_steady = false;
    DevBuf<double> sq;
    DevBuf<unsigned long long> stat;    // level-0 Phi solves, p-MG cycles
    DevBuf<unsigned long long> stat_c;  // coarser levels
    DevBuf<int> err;
    DevBuf<double> err_rel;
    DevBuf<double> u0;
    double g_norm = 0.0;
    long long launches = 0;  // kernels launched by the solve (bench evidence)
    int* iters_dev = nullptr;  // per-task iteration counts of the next waves (nullable)
    // overlap of the coarse march with interpolation / residual (coarse_overlapped)
    bool overlap = true;        // PHI_OVERLAP=0 disables
    static constexpr int kSides = 4;  // side streams (chunks round-robin, each with its own workspace)
    cudaStream_t side[kSides] = {};
    cudaEvent_t ev_pre = nullptr, ev_join[kSides] = {}, ev_inj[kSides] = {};
    unsigned* prog_host = nullptr;  // host-mapped progress counter of the coarse march
    unsigned* prog_dev = nullptr;
    Workspace ws_side[kSides];
    bool sq_ready = false;      // level-0 residual terms of the current state are in `sq`
    bool top_cycle = false;     // inside mgrit_cycle(0)
    ~Mgrit();

    // Optional per-launch profile of the Phi waves (CUDA events on the engine
    // stream + device counters of p-MG cycles), for the bench's roofline.
    bool profile = false;
    struct WaveRec {
        cudaEvent_t start, stop;
        int level;
    };
    std::vector<WaveRec> recs;
    DevBuf<int> wstats;  // 3 ints per recorded wave: max cycles, sum cycles, points
    /// Sum of wave kernel times (ms) and of their algorithmic bytes (DESIGN.md
    /// section 5 byte model) over the last solve(); returns the wave count.
    int wave_report(double* ms, double* bytes);
    /// Per MGRIT level of the last profiled solve: summed wave time (ms),
    /// Phi solves and p-MG cycles.  Must be called before wave_report (which
    /// releases the records).
    void wave_levels(double* ms, long long* points, long long* cycles, int cap);
    void set_init_coeffs(const double* host);

private:
    void build_levels();
    void build_loads();
    void project_initial();
    double compute_g_norm();
    /// where a wave runs: stream, workspace, one CTA per task, progress counter
    struct Route {
        cudaStream_t s;
        Workspace* w;
        bool no_cluster;
        volatile unsigned* progress;
    };
    void wave(int l, int mode, int epi, int n_tasks, const int* k0, int len, double* CG = nullptr,
              double* CU = nullptr, const Route* route = nullptr);
    /// coarsest_solve(lc) + interpolate_and_correct(lc - 1) (+ the level-0
    /// residual terms when `residual`), with the fine-level work of every
    /// interval issued on a side stream as soon as the coarse march has
    /// published both of its C-points: the same operations per point as the
    /// serial phases (bit-identical results), overlapped with the march.
    void coarse_overlapped(int lc, bool residual);
    void check_errors();
    int range_lo(int l) const { return l == 0 ? j_lo : 0; }
    int range_hi(int l) const;
    void f_relax(int l, bool with_c);
    void c_relax(int l);
    void restrict_residual(int l);
    void interpolate_and_correct(int l);
    void coarsest_solve(int l);
    void cycle_impl(int l, bool f_schedule);
    void halo();
    void combine_coarse_rhs();
    void cycle0_sharded(bool f_schedule);
    std::vector<std::pair<int, int>> owned_points(int l) const;
};

/// Sequential Phi-march on device (sequential_integrate, theta.hpp:216-237):
/// traj[0] = u0, traj[k] = Phi(traj[k-1]) with guess traj[k-1].
struct SequentialResult {
    long long solves = 0, iterations = 0;
};

}  // namespace phi
