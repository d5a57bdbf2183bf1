// miga_phi.hpp -- the binding a `miga` maintainer adds next to theta.hpp to run
// the time-stepping operator Phi (and whole MGRIT solves) on the B200 engine.
// It uses only the reference's public types (proj/include/miga) and the
// engine's C ABI (include/phi_engine.h); compiled and run by
// integration/test_binding.cpp (built by integration/Makefile, checked by
// tests/test_gpu_binding.py).
//
//   DeviceThetaStepper  -- ThetaStepper(const SpatialDiscretization&, kappa, dt,
//                          theta, cfg) (theta.hpp:92-146) with step() on the GPU;
//   DeviceMgritSolver   -- MgritSolver(disc, ps, cfg, scfg) (mgrit.hpp:50-118)
//                          with solve() on the GPU.  The std::function parts of
//                          ProblemSpec stay on the host in the reference's own
//                          code: LoadSchedule::build (theta.hpp:165-210) at
//                          construction, project_initial (theta.hpp:150-160)
//                          inside solve() as MgritSolver::initialize does; the
//                          engine takes the load terms and the projected u0.
// exact = true selects the engine's reference summation order: results are
// bit-identical to the reference's own classes on the same inputs.
#pragma once

#include <cmath>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "miga/mgrit.hpp"
#include "phi_engine.h"

namespace miga::phi_b200 {

inline void check(int rc) {
    if (rc == PHI_OK) return;
    const std::string msg = phi_last_error();
    if (rc == PHI_ERR_INVALID) throw std::invalid_argument(msg);
    throw std::runtime_error(msg);  // the reference's exception texts
}

// The engine's discretization of the same (degree, mesh) on the unit square.
inline phi_disc* engine_disc(const SpatialDiscretization& disc) {
    if (disc.geom.kind != GeometryMap::Kind::unit_square)
        throw std::invalid_argument("phi_b200: the engine discretizes the unit square only");
    phi_disc* d = nullptr;
    check(phi_disc_build(disc.degree, disc.mesh_exponent, &d));
    int info[5];
    check(phi_disc_info(d, info));
    if (info[0] != disc.dofmap_p.n_free) {
        phi_disc_free(d);
        throw std::invalid_argument("phi_b200: discretization mismatch");
    }
    return d;
}

inline phi_solver_config engine_solver_config(const SpatialSolverConfig& cfg, bool exact) {
    phi_solver_config c;
    phi_default_solver_config(&c);
    c.rel_tol = cfg.rel_tol;
    c.max_iter = cfg.max_iter;
    c.fixed_cycles = cfg.pmg_fixed_cycles;
    c.kind = cfg.kind == SpatialSolverKind::cg ? PHI_SOLVER_CG : PHI_SOLVER_PMG;
    c.pmg.ilut_tau = cfg.pmg.ilut_tau;
    c.pmg.ilut_fill = cfg.pmg.ilut_fill;
    c.pmg.nu_pre = cfg.pmg.nu_pre;
    c.pmg.nu_post = cfg.pmg.nu_post;
    c.pmg.gs_pre = cfg.pmg.gs_pre;
    c.pmg.gs_post = cfg.pmg.gs_post;
    c.pmg.exact = exact ? 1 : 0;
    return c;
}

/// ThetaStepper (theta.hpp:92-146) with the spatial solve on the device.
class DeviceThetaStepper {
public:
    DeviceThetaStepper(const SpatialDiscretization& disc, double kappa, double dt, double theta,
                       const SpatialSolverConfig& cfg, bool exact = true)
        : n_(disc.dofmap_p.n_free) {
        disc_ = engine_disc(disc);
        const phi_solver_config c = engine_solver_config(cfg, exact);
        check(phi_stepper_create(disc_, kappa, dt, theta, &c, &s_));
    }
    DeviceThetaStepper(const DeviceThetaStepper&) = delete;
    DeviceThetaStepper& operator=(const DeviceThetaStepper&) = delete;
    ~DeviceThetaStepper() {
        phi_stepper_free(s_);
        phi_disc_free(disc_);
    }

    /// step(u_prev, load, guess, stats) (theta.hpp:132-137)
    Vector step(const Vector& u_prev, const Vector& load, Vector guess, SolveStats* stats = nullptr) const {
        if ((int)u_prev.size() != n_) throw std::invalid_argument("ThetaStepper::step: size mismatch");
        const bool empty = guess.empty();
        if (empty) guess.assign(n_, 0.0);
        int iters = 0;
        check(phi_stepper_step(s_, u_prev.data(), load.empty() ? nullptr : load.data(), guess.data(), 1, n_,
                               empty ? 1 : 0, &iters, 0));
        if (stats) stats->record(iters);
        return guess;
    }

private:
    int n_;
    phi_disc* disc_ = nullptr;
    phi_stepper* s_ = nullptr;
};

/// MgritSolver (mgrit.hpp:50-118) with the space-time state on the device.
class DeviceMgritSolver {
public:
    DeviceMgritSolver(std::shared_ptr<const SpatialDiscretization> disc, ProblemSpec ps, MgritConfig cfg,
                      SpatialSolverConfig scfg, bool exact = true)
        : disc_(std::move(disc)), ps_(std::move(ps)), cfg_(cfg) {
        ps_.validate();
        cfg_.validate();
        const int n = disc_->dofmap_p.n_free;
        d_ = engine_disc(*disc_);
        // the level-0 load schedule, built by the reference's own code (theta.hpp:165-210)
        const LoadSchedule ls = LoadSchedule::build(*disc_, ps_.source, ps_.dt(), ps_.theta, ps_.n_time_steps);
        phi_problem p;
        phi_default_problem(&p);
        p.kappa = ps_.kappa;
        p.t_final = ps_.t_final;
        p.theta = ps_.theta;
        p.n_time_steps = ps_.n_time_steps;
        p.source_kind = PHI_SOURCE_CONSTANT;
        p.source_param = 0.0;  // the loads below replace the built-in source kinds
        if (!ls.empty()) {
            if (!ps_.source.time_dependent) {
                loads_ = ls.term(1);
                p.load_terms_steady = 1;
            } else {
                loads_.reserve((size_t)n * ps_.n_time_steps);
                for (int k = 1; k <= ps_.n_time_steps; ++k) loads_.insert(loads_.end(), ls.term(k).begin(), ls.term(k).end());
            }
            p.load_terms = loads_.data();
        }
        zero_.assign(n, 0.0);
        p.init_kind = PHI_INIT_VECTOR;  // the projected u0 is set by solve()
        p.init_coeffs = zero_.data();
        phi_mgrit_config mc;
        phi_default_mgrit_config(&mc);
        mc.cycle = cfg_.cycle == CycleType::v ? 0 : (cfg_.cycle == CycleType::f ? 1 : 2);
        mc.relax = cfg_.relaxation == RelaxType::f ? 0 : 1;
        mc.m = cfg_.m;
        mc.halt_tol = cfg_.halt_tol;
        mc.max_iter = cfg_.max_iter;
        mc.coarse_floor = cfg_.coarse_floor;
        const phi_solver_config sc = engine_solver_config(scfg, exact);
        check(phi_mgrit_create(d_, &p, &mc, &sc, &g_));
    }
    DeviceMgritSolver(const DeviceMgritSolver&) = delete;
    DeviceMgritSolver& operator=(const DeviceMgritSolver&) = delete;
    ~DeviceMgritSolver() {
        phi_mgrit_free(g_);
        phi_disc_free(d_);
    }

    /// solve() (mgrit.hpp:93-118): the IC projection on the host in the
    /// reference's code (as initialize() does), everything else on the device.
    MgritResult solve() {
        const Vector u0 = project_initial(*disc_, ps_.initial);
        check(phi_mgrit_set_init_coeffs(g_, u0.data()));
        phi_mgrit_result r;
        std::vector<double> hist(cfg_.max_iter);
        check(phi_mgrit_solve(g_, &r, hist.data(), (int)hist.size()));
        MgritResult out;
        out.iterations = r.iterations;
        out.converged = r.converged != 0;
        out.g_norm = r.g_norm;
        out.final_relative_residual = r.final_relative_residual;
        out.residual_history.assign(hist.begin(), hist.begin() + r.iterations);
        out.total_spatial_solves = r.total_spatial_solves;
        out.mean_spatial_iterations = r.mean_spatial_iterations;
        const int n = disc_->dofmap_p.n_free;
        std::vector<double> flat((size_t)(ps_.n_time_steps + 1) * n);
        check(phi_mgrit_trajectory(g_, flat.data()));
        out.trajectory.reserve(ps_.n_time_steps + 1);
        for (int k = 0; k <= ps_.n_time_steps; ++k)
            out.trajectory.push_back(
                extend_vector(disc_->dofmap_p, Vector(flat.begin() + (size_t)k * n, flat.begin() + (size_t)(k + 1) * n)));
        return out;
    }

private:
    std::shared_ptr<const SpatialDiscretization> disc_;
    ProblemSpec ps_;
    MgritConfig cfg_;
    std::vector<double> loads_, zero_;
    phi_disc* d_ = nullptr;
    phi_mgrit* g_ = nullptr;
};

}  // namespace miga::phi_b200
