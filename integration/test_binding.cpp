// Compiles the binding (integration/miga_phi.hpp) against the reference's own
// headers and checks it against the reference classes on identical inputs:
// MgritSolver::solve() vs DeviceMgritSolver::solve(), ThetaStepper::step vs
// DeviceThetaStepper::step -- bit for bit (the engine's exact mode).  Inputs
// are the reference's own ProblemSpec std::functions (the binding runs them
// through the reference's LoadSchedule and project_initial).  Exit code 0
// when every case matches.  Run by tests/test_gpu_binding.py.
#include <cmath>
#include <cstdio>
#include <memory>
#include <random>

#include "miga_phi.hpp"

using namespace miga;

namespace {

int failures = 0;

void expect(bool ok, const char* what) {
    std::printf("  %-48s %s\n", what, ok ? "ok" : "MISMATCH");
    if (!ok) ++failures;
}

bool same(const std::vector<Vector>& a, const std::vector<Vector>& b) {
    if (a.size() != b.size()) return false;
    for (size_t k = 0; k < a.size(); ++k)
        if (a[k] != b[k]) return false;
    return true;
}

void mgrit_case(const char* name, int p, int k, ProblemSpec ps, MgritConfig cfg) {
    std::printf("%s (p=%d, h=2^-%d, Nt=%d, m=%d)\n", name, p, k, ps.n_time_steps, cfg.m);
    ps.degree = p;
    ps.mesh_exponent = k;
    auto disc = std::make_shared<SpatialDiscretization>(SpatialDiscretization::build(GeometryMap::unit_square(), p, k));
    SpatialSolverConfig scfg;
    MgritSolver ref(disc, ps, cfg, scfg);
    const MgritResult r = ref.solve();
    phi_b200::DeviceMgritSolver dev(disc, ps, cfg, scfg, /*exact=*/true);
    const MgritResult d = dev.solve();
    expect(d.iterations == r.iterations && d.converged == r.converged, "iterations, converged");
    expect(d.g_norm == r.g_norm, "g_norm");
    expect(d.residual_history == r.residual_history, "residual history");
    expect(d.total_spatial_solves == r.total_spatial_solves &&
               d.mean_spatial_iterations == r.mean_spatial_iterations,
           "spatial solves, mean p-MG cycles");
    expect(same(d.trajectory, r.trajectory), "trajectory (full dofs)");
}

void stepper_case(int p, int k) {
    std::printf("ThetaStepper::step (p=%d, h=2^-%d)\n", p, k);
    const SpatialDiscretization disc = SpatialDiscretization::build(GeometryMap::unit_square(), p, k);
    SpatialSolverConfig cfg;
    const double dt = 1e-3;
    ThetaStepper ref(disc, 1.0, dt, 1.0, cfg);
    phi_b200::DeviceThetaStepper dev(disc, 1.0, dt, 1.0, cfg, true);
    std::mt19937 g(7);
    std::uniform_real_distribution<double> u(-1.0, 1.0);
    const int n = disc.dofmap_p.n_free;
    Vector up(n), load(n), guess(n);
    for (int i = 0; i < n; ++i) {
        up[i] = u(g);
        load[i] = 1e-3 * u(g);
        guess[i] = u(g);
    }
    SolveStats sr, sd;
    expect(dev.step(up, load, guess, &sd) == ref.step(up, load, guess, &sr), "step(u, load, guess)");
    expect(dev.step(up, {}, {}, &sd) == ref.step(up, {}, {}, &sr), "step(u) from a zero guess");
    expect(sd.solves.load() == sr.solves.load() && sd.iterations.load() == sr.iterations.load(), "SolveStats");
}

}  // namespace

int main() {
    if (phi_device_count() < 1) {
        std::printf("no CUDA device\n");
        return 2;
    }
    {  // BASELINE config 1
        ProblemSpec ps;
        ps.t_final = 0.1;
        ps.n_time_steps = 100;
        ps.source = SourceTerm::constant(0.0);
        ps.initial = [](double x, double y) { return std::sin(M_PI * x) * std::sin(M_PI * y); };
        MgritConfig cfg;
        cfg.cycle = CycleType::two_level;
        cfg.m = 4;
        mgrit_case("config 1", 2, 4, ps, cfg);
    }
    {  // the config-2 shape at a small size: transient source, a non-polynomial u0
        ProblemSpec ps;
        ps.n_time_steps = 32;
        ps.source = SourceTerm::transient([](double x, double y, double t) {
            return 2.0 * M_PI * M_PI * std::exp(-t) * std::sin(M_PI * x) * std::sin(M_PI * y);
        });
        ps.initial = [](double x, double y) { return x * (1.0 - x) * y * (1.0 - y) * std::exp(x - y); };
        MgritConfig cfg;
        cfg.cycle = CycleType::two_level;
        cfg.m = 8;
        mgrit_case("transient source", 3, 4, ps, cfg);
    }
    {  // F-cycle over four levels, steady source, Crank-Nicolson
        ProblemSpec ps;
        ps.n_time_steps = 64;
        ps.theta = 0.5;
        ps.source = SourceTerm::steady([](double x, double y) { return 1.0 + x * y; });
        MgritConfig cfg;
        cfg.cycle = CycleType::f;
        cfg.m = 2;
        mgrit_case("F-cycle, theta 0.5", 2, 3, ps, cfg);
    }
    stepper_case(3, 5);
    std::printf(failures ? "FAILED (%d)\n" : "all cases bit-identical\n", failures);
    return failures ? 1 : 0;
}
