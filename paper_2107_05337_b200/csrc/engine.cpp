// Host orchestration of the device engine (see engine.hpp).
#include "engine.hpp"

#include <algorithm>
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <string>
#include <thread>
#include <chrono>

namespace phi {

namespace {

Tables1DDev upload_tables(const Tables1D& t, cudaStream_t s) {
    Tables1DDev d;
    d.host = t;
    d.w.upload(t.weights, s);
    d.vals.upload(t.vals, s);
    d.ders.upload(t.ders, s);
    return d;
}

void set_square(StencilBuf& a, int nr, int nc, int lo, int hi) {
    a.ru = a.rv = nr;
    a.cu = a.cv = nc;
    a.lo = lo;
    a.hi = hi;
    a.vals.alloc(a.size());
}

HostCsr stencil_to_csr(const StencilBuf& a) {
    const std::vector<double> v = a.vals.download();
    HostCsr c;
    c.n_rows = a.ru * a.rv;
    c.n_cols = a.cu * a.cv;
    const int w = a.hi - a.lo + 1;
    const size_t n = a.n_rows();
    for (int iv = 0; iv < a.rv; ++iv)
        for (int iu = 0; iu < a.ru; ++iu) {
            const int i = iu + a.ru * iv;
            for (int dv = a.lo; dv <= a.hi; ++dv) {
                if (iv + dv < 0 || iv + dv >= a.cv) continue;
                for (int du = a.lo; du <= a.hi; ++du) {
                    if (iu + du < 0 || iu + du >= a.cu) continue;
                    c.col_indices.push_back((iu + du) + a.cu * (iv + dv));
                    c.values.push_back(v[(size_t)((dv - a.lo) * w + (du - a.lo)) * n + i]);
                }
            }
            c.row_offsets.push_back(c.nnz());
        }
    return c;
}

template <typename T>
DevBuf<T> dev(const std::vector<T>& h, cudaStream_t s) {
    DevBuf<T> d;
    d.upload(h, s);
    return d;
}

}  // namespace

// ---------------------------------------------------------------------------
// Disc
// ---------------------------------------------------------------------------
std::shared_ptr<Disc> Disc::build(int degree, int k, cudaStream_t s) {
    TraceRange trace_range("phi.disc.assemble");
    if (degree < 1 || degree > 8) throw InvalidArgument("SpatialDiscretization: degree must be in [1, 8]");
    if (k < 1) throw InvalidArgument("SpatialDiscretization: mesh exponent must be >= 1");
    auto d = std::make_shared<Disc>();
    d->degree = degree;
    d->mesh_exponent = k;
    d->n_elements = 1 << k;
    const int nel = d->n_elements;
    const int p = degree;

    const Knots kvp = open_uniform_knots(p, nel);
    d->tab_p = upload_tables(build_tables(kvp, p + 1), s);
    d->nf_p = nel + p - 2;
    d->n_p = d->nf_p * d->nf_p;
    set_square(d->M, d->nf_p, d->nf_p, -p, p);
    set_square(d->K, d->nf_p, d->nf_p, -p, p);
    launch_assemble_mk(d->tab_p.view(), d->tab_p.view(), d->M.vals.get(), d->K.vals.get(), s);

    // order-1 chain: halve while the mesh stays even and >= 8 (pmultigrid.hpp:119-133)
    std::vector<Tables1DDev> tabs1;
    int nl = nel;
    for (;;) {
        HLevel hl;
        hl.n_elements = nl;
        hl.nf = nl - 1;
        hl.n = hl.nf * hl.nf;
        tabs1.push_back(upload_tables(build_tables(open_uniform_knots(1, nl), 2), s));
        set_square(hl.M, hl.nf, hl.nf, -1, 1);
        set_square(hl.K, hl.nf, hl.nf, -1, 1);
        launch_assemble_mk(tabs1.back().view(), tabs1.back().view(), hl.M.vals.get(), hl.K.vals.get(), s);
        d->h.push_back(std::move(hl));
        if (nl >= 8 && nl % 2 == 0)
            nl /= 2;
        else
            break;
    }
    for (size_t l = 0; l + 1 < d->h.size(); ++l) {
        HLevel& hl = d->h[l];
        hl.E = p1_embedding_free(hl.n_elements);
        hl.Et = transpose(hl.E);
        hl.e_ro = dev(hl.E.row_offsets, s);
        hl.e_ci = dev(hl.E.col_indices, s);
        hl.e_v = dev(hl.E.values, s);
        hl.et_ro = dev(hl.Et.row_offsets, s);
        hl.et_ci = dev(hl.Et.col_indices, s);
        hl.et_v = dev(hl.Et.values, s);
    }
    d->nf_1 = d->h[0].nf;
    d->n_1 = d->h[0].n;

    d->inv_lp.alloc(d->n_p);
    d->inv_l1.alloc(d->n_1);
    if (p == 1) {
        // degenerate hierarchy: identity transfer, unit lumped masses (pmultigrid.hpp:139-143)
        set_square(d->T, d->nf_p, d->nf_p, 0, 0);
        set_square(d->Tt, d->nf_p, d->nf_p, 0, 0);
        std::vector<double> ones(d->n_p, 1.0);
        d->T.vals.upload(ones, s);
        d->Tt.vals.upload(ones, s);
        d->inv_lp.upload(ones, s);
        d->inv_l1.upload(ones, s);
    } else {
        const LowTables lt = build_low_tables(open_uniform_knots(1, nel), d->tab_p.host);
        DevBuf<double> low = dev(lt.vals, s);
        set_square(d->T, d->nf_p, d->nf_1, -p, 1);
        d->T.ru = d->T.rv = d->nf_p;
        d->T.cu = d->T.cv = d->nf_1;
        launch_assemble_transfer(d->tab_p.view(), d->tab_p.view(), low.get(), low.get(), d->T.vals.get(), s);
        set_square(d->Tt, d->nf_1, d->nf_p, -1, p);
        launch_stencil_transpose(d->T.view(), d->Tt.vals.get(), s);
        DevBuf<int> bad(1);
        bad.zero(s);
        launch_lump_inv(d->M.vals.get(), p, nel, d->inv_lp.get(), bad.get(), s);
        launch_lump_inv(d->h[0].M.vals.get(), 1, nel, d->inv_l1.get(), bad.get(), s);
        if (bad.download(s)[0]) throw std::runtime_error("lump_mass: non-positive row sum");
        PHI_CUDA(cudaStreamSynchronize(s));  // `low` goes out of scope
    }

    // sin(pi * node) at the order-p quadrature nodes, host libm (load assembly)
    d->sin_host.resize(d->tab_p.host.nodes.size());
    for (size_t i = 0; i < d->sin_host.size(); ++i) d->sin_host[i] = std::sin(M_PI * d->tab_p.host.nodes[i]);
    d->sin_tab = dev(d->sin_host, s);
    PHI_CUDA(cudaStreamSynchronize(s));
    return d;
}

HostCsr Disc::to_csr(const StencilBuf& a) const { return stencil_to_csr(a); }

void Disc::assemble_load(int kind, double c0, double c1, const double* coeffs_dev, double* out,
                         cudaStream_t s) const {
    launch_assemble_load(tab_p.view(), tab_p.view(), kind, c0, c1, sin_tab.get(), sin_tab.get(),
                         coeffs_dev, out, s);
}

namespace {
// nnz of a stencil operator's valid (in-grid) entries = reference CSR nnz
long long stencil_nnz(const DevStencil& A) {
    long long s = 0;
    for (int iv = 0; iv < A.rv; ++iv) {
        const int dv = std::min(A.hi, A.cv - 1 - iv) - std::max(A.lo, -iv) + 1;
        for (int iu = 0; iu < A.ru; ++iu) s += (long long)dv * (std::min(A.hi, A.cu - 1 - iu) - std::max(A.lo, -iu) + 1);
    }
    return s;
}
}  // namespace

// ---------------------------------------------------------------------------
// Hier
// ---------------------------------------------------------------------------
namespace {
void upload_tri(const TriPlan& p, bool fast, Hier::TriDev& d, cudaStream_t s) {
    const TriStream ts = make_tri_stream(p, fast);
    d.stream = dev(ts.stream, s);  // cudaMalloc: 256-byte aligned
    d.block_info = dev(ts.block_info, s);
    d.n_blocks = ts.n_blocks;
    d.n_units = ts.n_units;
    d.max_unit_bytes = ts.max_unit_bytes;
    for (int k = 0; k < 2 * (kTriSlots - 1); ++k) d.prime[k] = ts.prime[k];
}
DevTri tri_view(const TriPlan& p, const Hier::TriDev& d) {
    DevTri t{};
    t.n = p.n;
    t.n_levels = p.n_levels;
    t.n_units = d.n_units;
    t.n_blocks = d.n_blocks;
    t.max_unit_bytes = d.max_unit_bytes;
    t.blocks = reinterpret_cast<const int4*>(d.block_info.get());
    for (int k = 0; k < 2 * (kTriSlots - 1); ++k) t.prime[k] = d.prime[k];
    t.stream = d.stream.get();
    return t;
}
void upload_blk(const BlkStream& b, Hier::BlkDev& d, cudaStream_t s) {
    d.stream = dev(b.stream, s);
    d.table = dev(b.table, s);
    d.n = b.n;
    d.n_blocks = b.n_blocks;
    d.parts = b.parts;
    d.mf0 = b.mf0;
    d.lookahead = b.lookahead;
    d.max_unit_bytes = b.max_unit_bytes;
    d.win = b.win;
    d.desc = b.desc;
}

// Block-recurrence streams of the two ILUT substitutions.  When the vector z
// does not fit in shared memory next to a ring of kBlkMinSlots units, the
// streams use the rolling-window layout (setup_host.hpp), which keeps only a
// band-wide window of z on chip.
void build_ilut_streams(const HostCsr& L, const HostCsr& U, int n, BlkStream& lb, BlkStream& ub) {
    lb = blk_lower(L);
    ub = blk_upper(U);
    auto slot = [](const BlkStream& a, const BlkStream& b) {
        return (size_t)(std::max(a.max_unit_bytes, b.max_unit_bytes) + 127) / 128 * 128;
    };
    const size_t zb = ((size_t)n + 2) * 8;
    if (zb < kPhiSmemBudgetBytes && (kPhiSmemBudgetBytes - zb) / slot(lb, ub) >= (size_t)kBlkMinSlots) return;
    const int wz = blk_window_for(ilut_span(L, U));
    if (!wz) return;
    BlkStream lw = blk_lower(L, wz), uw = blk_upper(U, wz);
    const size_t wb = ((size_t)wz + 2) * 8;
    if ((kPhiSmemBudgetBytes - wb) / slot(lw, uw) < (size_t)kBlkMinSlots) return;
    lb = std::move(lw);
    ub = std::move(uw);
}
}  // namespace

DevBlk Hier::BlkDev::view() const {
    DevBlk b{};
    b.n = n;
    b.n_blocks = n_blocks;
    b.parts = parts;
    b.mf0 = mf0;
    b.lookahead = lookahead;
    b.max_unit_bytes = max_unit_bytes;
    b.win = win;
    b.desc = desc;
    b.stream = stream.get();
    b.table = reinterpret_cast<const int4*>(table.get());
    return b;
}

Hier::Hier(std::shared_ptr<const Disc> disc_, double c_, const HierOptions& opt_, cudaStream_t s, bool cg_only_)
    : disc(std::move(disc_)), c(c_), opt(opt_), cg_only(cg_only_) {
    TraceRange trace_range("phi.hier.setup");
    const Disc& d = *disc;
    A.ru = A.rv = A.cu = A.cv = d.nf_p;
    A.lo = d.M.lo;
    A.hi = d.M.hi;
    A.vals.alloc(A.size());
    launch_axpby(d.M.vals.get(), c, d.K.vals.get(), A.vals.get(), A.size(), s);
    if (cg_only) return;
    device_ilut(A.view(), opt.ilut_tau, opt.ilut_fill, L_host, U_host, s);
    // exact mode: level-scheduled streams (the reference's summation order);
    // reassociated mode: block recurrences
    if (opt.exact) {
        Lp = plan_lower(L_host);
        Up = plan_upper(U_host);
        upload_tri(Lp, false, Ld, s);
        upload_tri(Up, false, Ud, s);
    } else {
        BlkStream lb, ub;
        build_ilut_streams(L_host, U_host, d.n_p, lb, ub);
        upload_blk(lb, Lbd, s);
        upload_blk(ub, Ubd, s);
    }
    for (const auto& hl : d.h) {
        StencilBuf a;
        a.ru = a.rv = a.cu = a.cv = hl.nf;
        a.lo = -1;
        a.hi = 1;
        a.vals.alloc(a.size());
        launch_axpby(hl.M.vals.get(), c, hl.K.vals.get(), a.vals.get(), a.size(), s);
        a_h.push_back(std::move(a));
    }
    // Gauss-Seidel sweeps of the h-levels as level-scheduled streams
    // (wavefronts), in the hierarchy's summation mode
    for (size_t l = 0; l + 1 < a_h.size(); ++l) {
        const HostCsr al = stencil_to_csr(a_h[l]);
        for (int dir = 0; dir < 2; ++dir) {
            if (opt.exact) {
                gs_plans.push_back(plan_gauss_seidel(al, dir == 1));
                gs_dev.emplace_back();
                upload_tri(gs_plans.back(), false, gs_dev.back(), s);
            } else {
                gsb_dev.emplace_back();
                upload_blk(blk_gauss_seidel(al, dir == 1), gsb_dev.back(), s);
            }
        }
        gsl_dev.emplace_back();
        if (!opt.exact && d.h[l].nf <= kLineMax && d.h[l].nf >= kLineMin) {
            gsl_dev.back().alloc((size_t)9 * d.h[l].n);
            launch_gs_line_coeffs(a_h[l].vals.get(), d.h[l].nf, gsl_dev.back().get(), s);
        }
    }
    coarse = dense_lu_factor(stencil_to_csr(a_h.back()));
    coarse_lu = dev(coarse.lu, s);
    coarse_piv = dev(coarse.piv, s);
    // Reassociated mode: below the first h-level with at most kDenseCoarseMax
    // rows the W-cycle (zero initial guess, hence linear) is applied as one
    // dense operator -- the latency-bound small sweeps and the serial LU
    // become one data-parallel matvec.  Same cycle, different rounding.
    if (!opt.exact && (opt.dense_coarse_max > 0 || opt.dense_cluster_max > 0)) {
        const int nh = (int)a_h.size();
        std::vector<HostCsr> ah, eh;
        for (int k = 0; k < nh; ++k) {
            ah.push_back(stencil_to_csr(a_h[k]));
            eh.push_back(d.h[k].E);
        }
        auto first = [&](int cap) {
            for (int l = 0; l + 1 < nh; ++l)
                if (d.h[l].n <= cap) return l;
            return -1;
        };
        dense_level = opt.dense_coarse_max > 0 ? first(opt.dense_coarse_max) : -1;
        dense_level_cl = opt.dense_cluster_max > 0 ? first(opt.dense_cluster_max) : -1;
        if (dense_level >= 0) dense_op = dev(wcycle_operator(ah, eh, coarse, dense_level, opt.gs_pre, opt.gs_post), s);
        if (dense_level_cl >= 0 && dense_level_cl != dense_level)
            dense_op_cl = dev(wcycle_operator(ah, eh, coarse, dense_level_cl, opt.gs_pre, opt.gs_post), s);
    }
    PHI_CUDA(cudaStreamSynchronize(s));
}

HostCsr Hier::a_h_csr(int l) const { return stencil_to_csr(a_h.at(l)); }

// Byte model of one V(nu_pre, nu_post) cycle, in
// fp64 entries: every stored nonzero of the operators the cycle applies,
// once per application and batch (A for the two smoothing residuals and the
// residual before the restriction, L and U twice, T and T^T, the h-chain
// with 2^l visits of level l: 4 sweeps + residual of A_l, E and E^T, the
// dense coarse LU); and per right-hand side every vector entry read or
// written.
double Hier::vcycle_matrix_entries() const {
    const Disc& d = *disc;
    double vmat = 3.0 * stencil_nnz(A.view()) + 2.0 * (L_host.nnz() + U_host.nnz()) + 2.0 * stencil_nnz(d.T.view());
    const int nh = (int)d.h.size();
    for (int l = 0; l + 1 < nh; ++l)
        vmat += std::ldexp(1.0, l) * (5.0 * stencil_nnz(a_h[l].view()) + 2.0 * d.h[l].E.nnz());
    vmat += std::ldexp(1.0, nh - 1) * (double)coarse.n * coarse.n;
    return vmat;
}

double Hier::vcycle_vector_entries() const {
    const Disc& d = *disc;
    const double n = d.n_p, n1 = d.n_1;
    double vvec = 18 * n + 3 * n + (n + n1) + (n1 + 2 * n);
    const int nh = (int)d.h.size();
    for (int l = 0; l + 1 < nh; ++l) {
        const double nl = d.h[l].n, nc = d.h[l + 1].n;
        vvec += std::ldexp(1.0, l) * (4 * 3 * nl + 3 * nl + (nl + nc) + nc + (nc + 2 * nl));
    }
    return vvec;
}

long long Hier::chain_steps() const {
    if (cg_only || opt.exact) return 0;
    const Disc& d = *disc;
    long long s = (long long)(opt.nu_pre + opt.nu_post) * (Lbd.n_blocks + Ubd.n_blocks);
    const int nh = (int)d.h.size();
    const int dl = dense_level_cl >= 0 ? dense_level_cl : (dense_level >= 0 ? dense_level : nh - 1);
    for (int l = 0; l < dl && l + 1 < nh; ++l) {
        const long long visits = 1LL << l;
        const bool line = d.h[l].nf <= kLineMax && d.h[l].nf >= kLineMin;
        const long long per_sweep = line ? d.h[l].nf : gsb_dev[2 * l].n_blocks;
        s += visits * (opt.gs_pre + opt.gs_post) * per_sweep;
    }
    s += 1LL << dl;  // dense (or LU) applications of the coarse subtree
    return s;
}

DevHier Hier::view(const SolverConfig& cfg) const {
    const Disc& d = *disc;
    if ((int)d.h.size() > kMaxH) throw InvalidArgument("too many h-levels");
    DevHier H{};
    if (cg_only) {  // CG kind: the operator and its diagonal (the centre plane)
        H.n_p = d.n_p;
        H.A = A.view();
        const int w = A.hi - A.lo + 1;
        H.diag = A.vals.get() + (size_t)((w * w - 1) / 2) * d.n_p;
        H.kind = 1;
        H.rel_tol = cfg.rel_tol;
        H.max_iter = cfg.max_iter;
        H.exact = opt.exact;
        return H;
    }
    H.n_p = d.n_p;
    H.n_1 = d.n_1;
    H.n_h = (int)d.h.size();
    H.A = A.view();
    H.T = d.T.view();
    H.Tt = d.Tt.view();
    H.inv_lp = d.inv_lp.get();
    H.inv_l1 = d.inv_l1.get();
    if (opt.exact) {
        H.L = tri_view(Lp, Ld);
        H.U = tri_view(Up, Ud);
    } else {
        H.Lb = Lbd.view();
        H.Ub = Ubd.view();
    }
    for (int l = 0; l < H.n_h; ++l) {
        const auto& hl = d.h[l];
        H.h[l].a = a_h[l].view();
        if (l + 1 < H.n_h && opt.exact) {
            H.h[l].gs_fwd = tri_view(gs_plans[2 * l], gs_dev[2 * l]);
            H.h[l].gs_bwd = tri_view(gs_plans[2 * l + 1], gs_dev[2 * l + 1]);
        } else if (l + 1 < H.n_h) {
            H.h[l].gsb_fwd = gsb_dev[2 * l].view();
            H.h[l].gsb_bwd = gsb_dev[2 * l + 1].view();
            H.h[l].gsl = gsl_dev[l].get();
        }
        H.h[l].nf = hl.nf;
        H.h[l].n = hl.n;
        if (l + 1 < H.n_h) {
            H.h[l].embed = DevCsr{hl.E.n_rows, hl.E.n_cols, hl.e_ro.get(), hl.e_ci.get(), hl.e_v.get()};
            H.h[l].embed_t = DevCsr{hl.Et.n_rows, hl.Et.n_cols, hl.et_ro.get(), hl.et_ci.get(), hl.et_v.get()};
        }
    }
    H.coarse_lu = coarse_lu.get();
    H.coarse_piv = coarse_piv.get();
    H.coarse_n = coarse.n;
    H.dense_level = dense_level;
    H.dense_op = dense_op.get();
    H.dense_level_cl = dense_level_cl;
    H.dense_op_cl = dense_level_cl == dense_level ? dense_op.get() : dense_op_cl.get();
    H.nu_pre = opt.nu_pre;
    H.nu_post = opt.nu_post;
    H.gs_pre = opt.gs_pre;
    H.gs_post = opt.gs_post;
    H.rel_tol = cfg.rel_tol;
    H.max_iter = cfg.max_iter;
    H.fixed_cycles = cfg.fixed_cycles;
    H.exact = opt.exact;
    return H;
}

void Workspace::ensure(const DevHier& H) {
    const long long need = (long long)phi_ws_doubles(H);
    const int want_slots = phi_max_slots(H);
    if (need > stride || want_slots > slots) {
        stride = std::max(stride, need);
        slots = std::max(slots, want_slots);
        buf.alloc((size_t)stride * slots);
    }
}

// ---------------------------------------------------------------------------
// Stepper
// ---------------------------------------------------------------------------
std::string spatial_failure(int kind, double rel) {
    if (kind == 1)
        return rel < 0.0 ? "cg_solve: breakdown, matrix not SPD" : "spatial solve did not converge (cg)";
    return "spatial solve did not converge (p-multigrid), residual " + std::to_string(rel);
}

Stepper::Stepper(std::shared_ptr<const Disc> disc_, double kappa_, double dt_, double theta_,
                 const SolverConfig& cfg_, cudaStream_t s)
    : disc(std::move(disc_)), kappa(kappa_), dt(dt_), theta(theta_), cfg(cfg_) {
    if (cfg.kind != 0 && cfg.kind != 1) throw InvalidArgument("unknown spatial solver kind");
    hier = std::make_unique<Hier>(disc, kappa * dt * theta, cfg.pmg, s, cfg.kind == 1);
    const Disc& d = *disc;
    Aminus.ru = Aminus.rv = Aminus.cu = Aminus.cv = d.nf_p;
    Aminus.lo = d.M.lo;
    Aminus.hi = d.M.hi;
    Aminus.vals.alloc(Aminus.size());
    launch_axpby(d.M.vals.get(), -kappa * dt * (1.0 - theta), d.K.vals.get(), Aminus.vals.get(),
                 Aminus.size(), s);
    H = hier->view(cfg);
    PHI_CUDA(cudaStreamSynchronize(s));
}

// ---------------------------------------------------------------------------
// Mgrit
// ---------------------------------------------------------------------------
Mgrit::Mgrit(std::shared_ptr<const Disc> disc_, const ProblemOptions& ps_, const MgritOptions& cfg_,
             const SolverConfig& scfg_, cudaStream_t s)
    : disc(std::move(disc_)), ps(ps_), cfg(cfg_), scfg(scfg_), stream(s) {
    if (!(ps.kappa > 0.0)) throw InvalidArgument("ProblemSpec: kappa must be > 0");
    if (!(ps.t_final > 0.0)) throw InvalidArgument("ProblemSpec: t_final must be > 0");
    if (ps.n_time_steps < 1) throw InvalidArgument("ProblemSpec: nt must be >= 1");
    if (!(ps.theta >= 0.0 && ps.theta <= 1.0)) throw InvalidArgument("ProblemSpec: theta must be in [0, 1]");
    if (cfg.m < 2) throw InvalidArgument("MgritConfig: m must be >= 2");
    if (cfg.max_iter < 1) throw InvalidArgument("MgritConfig: max_iter must be >= 1");
    if (!(cfg.halt_tol > 0.0)) throw InvalidArgument("MgritConfig: tol must be > 0");
    build_levels();
    build_loads();
    sq.alloc(levels[0].steps + 1);
    stat.alloc(2);
    stat_c.alloc(2);
    err.alloc(3);
    err_rel.alloc(1);
    u0.alloc(disc->n_p);
    for (auto& lv : levels) ws.ensure(lv.stepper->H);
    if (const char* e = std::getenv("PHI_OVERLAP")) overlap = std::atoi(e) != 0;
    PHI_CUDA(cudaStreamSynchronize(stream));
}

// Time-step counts of the MGRIT levels (the rules of mgrit.hpp:217-233): a level
// is coarsened while its step count is a positive multiple of m; past the first
// coarse level only if the next one keeps more than coarse_floor time points;
// the two-level cycle stops after one coarsening.
std::vector<int> mgrit_level_steps(int nt, int m, int cycle, int coarse_floor) {
    if (m < 2) throw InvalidArgument("MgritConfig: m must be >= 2");
    if (nt >= m && nt % m != 0)
        throw InvalidArgument("MGRIT: nt (" + std::to_string(nt) + ") not divisible by coarsening factor m (" +
                              std::to_string(m) + ")");
    std::vector<int> counts{nt};
    const size_t cap = cycle == 2 ? 2 : static_cast<size_t>(-1);
    while (counts.size() < cap) {
        const int fine = counts.back();
        if (fine < m || fine % m != 0) break;
        const int coarse = fine / m;
        const bool deep_enough = counts.size() == 1 || coarse + 1 > coarse_floor;
        if (!deep_enough) break;
        counts.push_back(coarse);
    }
    return counts;
}

void Mgrit::build_levels() {
    const int m = cfg.m, nt = ps.n_time_steps;
    const std::vector<int> steps = mgrit_level_steps(nt, m, cfg.cycle, cfg.coarse_floor);
    const double dt0 = ps.t_final / nt;
    const int n = disc->n_p;
    levels.resize(steps.size());
    for (size_t l = 0; l < steps.size(); ++l) {
        Level& lv = levels[l];
        lv.steps = steps[l];
        lv.dt = dt0 * (nt / steps[l]);
        lv.stepper = std::make_unique<Stepper>(disc, ps.kappa, lv.dt, ps.theta, scfg, stream);
        lv.u.alloc((size_t)(lv.steps + 1) * n);
        lv.g.alloc((size_t)(lv.steps + 1) * n);
        const int J = lv.steps / m;
        std::vector<int> kF(std::max(J, 1)), kR(std::max(J, 1)), kAll(std::max(lv.steps, 1));
        for (int j = 0; j < J; ++j) {
            kF[j] = j * m + 1;
            kR[j] = (j + 1) * m;
        }
        for (int k = 1; k <= lv.steps; ++k) kAll[k - 1] = k;
        lv.kF = dev(kF, stream);
        lv.kR = dev(kR, stream);
        lv.kAll = dev(kAll, stream);
    }
}

void Mgrit::build_loads() {
    const int n = disc->n_p, steps = ps.n_time_steps;
    const double dt = ps.t_final / steps;
    has_loads = false;
    loads_steady = false;
    if (!ps.load_terms.empty()) {
        has_loads = true;
        loads_steady = ps.load_terms_steady != 0;
        const size_t want = loads_steady ? (size_t)n : (size_t)n * steps;
        if (ps.load_terms.size() != want) throw InvalidArgument("load_terms: dimension mismatch");
        loads.upload(ps.load_terms, stream);
        return;
    }
    // LoadSchedule::build (theta.hpp:167-193)
    if (ps.source_kind == 0) {
        if (ps.source_param == 0.0) return;  // SourceTerm::zero
        has_loads = loads_steady = true;
        loads.alloc(n);
        disc->assemble_load(0, ps.source_param, 0.0, nullptr, loads.get(), stream);
        launch_scale(loads.get(), dt, n, stream);
    } else if (ps.source_kind == 2) {
        has_loads = loads_steady = true;
        loads.alloc(n);
        disc->assemble_load(2, ps.source_param, 0.0, nullptr, loads.get(), stream);
        launch_scale(loads.get(), dt, n, stream);
    } else if (ps.source_kind == 1) {
        has_loads = true;
        loads.alloc((size_t)n * steps);
        // F_k = dt (theta f(t_k) + (1 - theta) f(t_{k-1})) from raw assemblies
        DevBuf<double> prev(n), cur(n);
        disc->assemble_load(1, ps.source_param, std::exp(-(0 * dt)), nullptr, prev.get(), stream);
        for (int k = 1; k <= steps; ++k) {
            double* fk = loads.get() + (size_t)(k - 1) * n;
            disc->assemble_load(1, ps.source_param, std::exp(-(k * dt)), nullptr, cur.get(), stream);
            launch_copy(fk, cur.get(), n, stream);
            launch_theta_combine(fk, prev.get(), dt * ps.theta, dt * (1.0 - ps.theta), n, stream);
            std::swap(prev, cur);
        }
        PHI_CUDA(cudaStreamSynchronize(stream));
    } else {
        throw InvalidArgument("unknown source kind");
    }
}

void Mgrit::project_initial() {
    TraceRange trace_range("phi.mgrit.project_initial");
    const int n = disc->n_p;
    if (ps.init_kind == 0) {
        u0.zero(stream);
        return;
    }
    if (ps.init_kind == 3) {  // the caller's projected initial state, as is
        if ((int)ps.init_coeffs.size() != n) throw InvalidArgument("initial state: dimension mismatch");
        u0.upload(ps.init_coeffs, stream);
        PHI_CUDA(cudaStreamSynchronize(stream));
        return;
    }
    DevBuf<double> b(n), work(4 * (size_t)n), coeffs;
    DevBuf<int> res(2);
    if (ps.init_kind == 1) {
        disc->assemble_load(3, 0.0, 0.0, nullptr, b.get(), stream);
    } else if (ps.init_kind == 2) {
        if ((int)ps.init_coeffs.size() != n) throw InvalidArgument("init_coeffs: dimension mismatch");
        coeffs.upload(ps.init_coeffs, stream);
        disc->assemble_load(4, 0.0, 0.0, coeffs.get(), b.get(), stream);
    } else {
        throw InvalidArgument("unknown initial kind");
    }
    const DevStencil M = disc->M.view();
    const int p = disc->degree, w = 2 * p + 1;
    const double* diag = disc->M.vals.get() + (size_t)(p * w + p) * n;  // center entries
    launch_cg(M, diag, b.get(), u0.get(), work.get(), 1e-13, 2000, res.get(), scfg.pmg.exact, stream);
    launches += 2;
    const auto r = res.download(stream);
    if (r[0] < 0) throw std::runtime_error("cg_solve: breakdown, matrix not SPD");
    if (r[0] != 1) throw std::runtime_error("project_initial: mass solve did not converge");
}

void Mgrit::wave(int l, int mode, int epi, int n_tasks, const int* k0, int len, double* CG, double* CU,
                 const Route* route) {
    Level& lv = levels[l];
    const cudaStream_t st = route ? route->s : stream;
    Workspace& wsp = route && route->w ? *route->w : ws;
    WaveArgs a{};
    a.mode = mode;
    a.epi = epi;
    a.n_tasks = n_tasks;
    a.task_len = len;
    a.task_k0 = k0;
    a.n = disc->n_p;
    a.U = lv.u.get();
    a.G = lv.g.get();
    a.LOAD = (l == 0 && has_loads) ? loads.get() : nullptr;
    a.load_steady = loads_steady ? 1 : 0;
    a.CG = CG;
    a.CU = CU;
    a.m = cfg.m;
    a.SQ = sq.get();
    a.stat = l == 0 ? stat.get() : stat_c.get();
    a.err = err.get();
    a.err_rel = err_rel.get();
    a.level = l;
    a.x0_empty = mode == kModeSolve ? 1 : 0;  // g-norm solves start from zero (mgrit.hpp:301)
    a.iters_out = iters_dev;
    a.progress = route ? route->progress : nullptr;
    a.no_cluster = route && route->no_cluster ? 1 : 0;
    const bool rec = profile && recs.size() * 3 < wstats.size();
    if (rec) {
        WaveRec r{};
        r.level = l;
        PHI_CUDA(cudaEventCreate(&r.start));
        PHI_CUDA(cudaEventCreate(&r.stop));
        a.wave_max = wstats.get() + 3 * recs.size();
        PHI_CUDA(cudaEventRecord(r.start, st));
        recs.push_back(r);
    }
    launch_phi_wave(lv.stepper->H, lv.stepper->Aminus.view(), a, wsp.buf.get(), wsp.stride, wsp.slots, st);
    if (rec) PHI_CUDA(cudaEventRecord(recs.back().stop, st));
    ++launches;
}

Mgrit::~Mgrit() {
    for (int i = 0; i < kSides; ++i) {
        if (side[i]) {
            cudaStreamSynchronize(side[i]);
            cudaStreamDestroy(side[i]);
        }
        if (ev_join[i]) cudaEventDestroy(ev_join[i]);
        if (ev_inj[i]) cudaEventDestroy(ev_inj[i]);
    }
    if (ev_pre) cudaEventDestroy(ev_pre);
    if (prog_host) cudaFreeHost(prog_host);
}

void Mgrit::coarse_overlapped(int lc, bool residual) {
    TraceRange trace_range("phi.mgrit.coarse_march+interpolate");
    const int lf = lc - 1;
    Level& c = levels[lc];
    Level& f = levels[lf];
    const int n = disc->n_p, m = cfg.m, J = f.steps / m;
    if (!side[0]) {
        int lo = 0, hi = 0;
        PHI_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
        for (int i = 0; i < kSides; ++i) {
            PHI_CUDA(cudaStreamCreateWithPriority(&side[i], cudaStreamNonBlocking, lo));
            PHI_CUDA(cudaEventCreateWithFlags(&ev_join[i], cudaEventDisableTiming));
            PHI_CUDA(cudaEventCreateWithFlags(&ev_inj[i], cudaEventDisableTiming));
            for (auto& lv : levels) ws_side[i].ensure(lv.stepper->H);
        }
        PHI_CUDA(cudaEventCreateWithFlags(&ev_pre, cudaEventDisableTiming));
        PHI_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&prog_host), sizeof(unsigned), cudaHostAllocMapped));
        PHI_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&prog_dev), prog_host, 0));
        preload_overlap_kernels(f.stepper->H);
    }
    volatile unsigned* prog = prog_host;
    *prog = 0u;
    // the coarse march (coarsest_solve, mgrit.hpp:188-194), publishing its progress
    launch_copy(c.u.get(), c.g.get(), n, stream);
    ++launches;
    PHI_CUDA(cudaEventRecord(ev_pre, stream));  // everything the fine-level work depends on
    const Route coarse{stream, nullptr, false, prog_dev};
    wave(lc, kModeStep, kEpiStore, 1, c.kAll.get(), c.steps, nullptr, nullptr, &coarse);
    // the fine-level work, interval by interval as the coarse points land:
    // injection (mgrit.hpp:172-180), F-relaxation, and (residual) the terms
    // of residual_norm(0) (mgrit.hpp:197-214), on the side stream
    for (int i = 0; i < kSides; ++i) PHI_CUDA(cudaStreamWaitEvent(side[i], ev_pre, 0));
    if (residual) PHI_CUDA(cudaMemsetAsync(sq.get(), 0, sizeof(double) * (f.steps + 1), side[0]));
    int rr = 0;  // chunks go round-robin over the side streams (each chunk is m - 1 steps deep)
    // chunks of J/16 intervals (shrinking chunks towards the end of the march
    // measured no better: more launches)
    const int chunk = std::max(1, J / 16);
    int injected = 0, done = 0;  // C-points injected, intervals relaxed
    const bool dbg = std::getenv("PHI_OVERLAP_DEBUG") != nullptr;
    const auto t0 = std::chrono::steady_clock::now();
    auto since = [&]() { return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count(); };
    long long polls = 0;
    while (done < J) {
        ++polls;
        // coarse points 0..p are final (coarse point 0 is g[0], copied before the march)
        const unsigned pv = *prog;
        const int p = (int)std::min<unsigned>(pv, (unsigned)J);
        const int ready = p;  // interval j needs coarse points j and j + 1
        if (ready - done >= chunk || (p >= J && ready > done)) {
            if (dbg) std::fprintf(stderr, "overlap: %.2f ms progress %u -> intervals [%d, %d) (%lld polls)\n", since(), pv, done, ready, polls);
            const int cur = rr, prev = (rr + kSides - 1) % kSides;
            const cudaStream_t ss = side[cur];
            const Route sr{ss, &ws_side[cur], true, nullptr};
            rr = (rr + 1) % kSides;
            // the chunk's C-points [injected, p] -- disjoint from the other chunks'
            launch_inject_range(c.u.get(), f.u.get(), n, injected, p + 1, m, ss);
            ++launches;
            if (residual && injected == 0) {  // point 0 after its injection (stream 0: after the memset)
                launch_resid0(f.g.get(), f.u.get(), sq.get(), n, ss);
                ++launches;
            }
            injected = p + 1;
            // interval `done` starts from C-point done m, injected by the
            // previous chunk (another stream): wait for that injection only
            if (done > 0) PHI_CUDA(cudaStreamWaitEvent(ss, ev_inj[prev], 0));
            PHI_CUDA(cudaEventRecord(ev_inj[cur], ss));
            wave(lf, kModeStep, kEpiStore, ready - done, f.kF.get() + done, m - 1, nullptr, nullptr, &sr);
            if (residual)
                wave(lf, kModeStep, kEpiResid, (ready - done) * m, f.kAll.get() + done * m, 1, nullptr, nullptr, &sr);
            done = ready;
            continue;
        }
        // poll: the march publishes after every coarse step
        if (cudaStreamQuery(stream) == cudaErrorNotReady) {
            std::this_thread::sleep_for(std::chrono::microseconds(20));
        } else {
            PHI_CUDA(cudaGetLastError());
            if (dbg) std::fprintf(stderr, "overlap: %.2f ms march stream idle, progress %u\n", since(), *prog);
            if (*prog < (unsigned)J) {  // the march ended without finishing (an error): drain
                PHI_CUDA(cudaStreamSynchronize(stream));
                *prog = (unsigned)J;
            }
        }
    }
    for (int i = 0; i < kSides; ++i) {
        PHI_CUDA(cudaEventRecord(ev_join[i], side[i]));
        PHI_CUDA(cudaStreamWaitEvent(stream, ev_join[i], 0));
    }
    sq_ready = residual;
}

void Mgrit::check_errors() {
    const auto e = err.download(stream);
    if (e[0]) {
        const double rel = err_rel.download(stream)[0];
        throw NotConverged("MGRIT level " + std::to_string(e[2]) + ", time step " + std::to_string(e[1]) + ": " +
                           spatial_failure(scfg.kind, rel));
    }
}

// mgrit.hpp:122-141; with FCF the first F sweep also covers the C-point of its
// interval (same operations in the same order per point).
int Mgrit::range_hi(int l) const {
    const int J = levels[l].steps / cfg.m;
    return (l == 0 && j_hi >= 0) ? std::min(j_hi, J) : J;
}

// F-relaxation of every interval (mgrit.hpp:122-132); with_c adds the
// C-relaxation (135-141) as a second wave.  The two must not be fused per
// interval: interval j + 1 has to start from the C-point u[(j+1) m] as it was
// BEFORE interval j's C-relaxation updates it, which a fused task only sees
// while all intervals happen to be resident at once.
void Mgrit::f_relax(int l, bool with_c) {
    TraceRange trace_range("phi.mgrit.f_relax");
    Level& lv = levels[l];
    const int lo = range_lo(l), hi = range_hi(l);
    wave(l, kModeStep, kEpiStore, hi - lo, lv.kF.get() + lo, cfg.m - 1);
    if (with_c) c_relax(l);
}

void Mgrit::c_relax(int l) {
    TraceRange trace_range("phi.mgrit.c_relax");
    Level& lv = levels[l];
    const int lo = range_lo(l), hi = range_hi(l);
    wave(l, kModeStep, kEpiStore, hi - lo, lv.kR.get() + lo, 1);
}

void Mgrit::restrict_residual(int l) {
    TraceRange trace_range("phi.mgrit.restrict");
    Level& f = levels[l];
    Level& c = levels[l + 1];
    const int n = disc->n_p;
    const int lo = range_lo(l), hi = range_hi(l);
    launch_restrict_first(f.g.get(), f.u.get(), c.g.get(), c.u.get(), n, stream);
    ++launches;
    wave(l, kModeStep, kEpiRestrict, hi - lo, f.kR.get() + lo, 1, c.g.get(), c.u.get());
}

void Mgrit::interpolate_and_correct(int l) {
    TraceRange trace_range("phi.mgrit.interpolate");
    Level& f = levels[l];
    Level& c = levels[l + 1];
    launch_inject(c.u.get(), f.u.get(), disc->n_p, f.steps / cfg.m, cfg.m, stream);
    ++launches;
    f_relax(l, false);
}

void Mgrit::coarsest_solve(int l) {
    TraceRange trace_range("phi.mgrit.coarsest_solve");
    Level& lv = levels[l];
    launch_copy(lv.u.get(), lv.g.get(), disc->n_p, stream);
    ++launches;
    wave(l, kModeStep, kEpiStore, 1, lv.kAll.get(), lv.steps);
}

void Mgrit::cycle_impl(int l, bool f_schedule) {
    if (l + 1 == n_levels()) {
        coarsest_solve(l);
        return;
    }
    if (cfg.relax == 1) {
        f_relax(l, true);   // F + C
        f_relax(l, false);  // F
    } else {
        f_relax(l, false);
    }
    restrict_residual(l);
    const bool second_pass = f_schedule && l + 2 < n_levels();
    // (only where the interpolation wave has enough intervals to run one CTA
    // per interval anyway -- the overlapped waves always do, so the results
    // stay bit-identical to the serial phases)
    if (l + 2 == n_levels() && overlap && !comm && !scfg.pmg.exact && j_hi < 0 &&
        levels[l].steps / cfg.m >= kOverlapMinIntervals) {
        // the coarse march overlapped with this level's interpolation (and,
        // at the top of a cycle, with the residual terms residual_norm reads)
        coarse_overlapped(l + 1, l == 0 && top_cycle && !second_pass);
    } else {
        cycle_impl(l + 1, f_schedule);
        interpolate_and_correct(l);
    }
    if (second_pass) cycle_impl(l, false);
}

void Mgrit::mgrit_cycle(int l) {
    sq_ready = false;
    top_cycle = l == 0;
    cycle_impl(l, cfg.cycle == 1);
    top_cycle = false;
}

double Mgrit::residual_norm(int l) {
    std::vector<double> h(levels[l].steps + 1);
    residual_terms(l, h.data());
    double total = 0.0;
    for (double s : h) total += s;  // fixed order (mgrit.hpp:211-212)
    return std::sqrt(total);
}

void Mgrit::residual_terms(int l, double* host) {
    TraceRange trace_range("phi.mgrit.residual");
    Level& lv = levels[l];
    const int n = disc->n_p;
    const int lo = range_lo(l), hi = range_hi(l);
    if (l == 0 && sq_ready && !iters_dev) {  // computed alongside the coarse march (coarse_overlapped)
        sq_ready = false;
        PHI_CUDA(cudaMemcpyAsync(host, sq.get(), sizeof(double) * (lv.steps + 1), cudaMemcpyDeviceToHost, stream));
        PHI_CUDA(cudaStreamSynchronize(stream));
        check_errors();
        return;
    }
    sq_ready = false;
    PHI_CUDA(cudaMemsetAsync(sq.get(), 0, sizeof(double) * (lv.steps + 1), stream));
    if (lo == 0) {  // point 0 belongs to the first rank
        launch_resid0(lv.g.get(), lv.u.get(), sq.get(), n, stream);
        ++launches;
    }
    const int k_begin = lo * cfg.m + 1;
    const int k_end = (hi == lv.steps / cfg.m) ? lv.steps : hi * cfg.m;  // the last rank takes any tail
    if (k_end >= k_begin) wave(l, kModeStep, kEpiResid, k_end - k_begin + 1, lv.kAll.get() + (k_begin - 1), 1);
    PHI_CUDA(cudaMemcpyAsync(host, sq.get(), sizeof(double) * (lv.steps + 1), cudaMemcpyDeviceToHost, stream));
    PHI_CUDA(cudaStreamSynchronize(stream));
    check_errors();
}

void Mgrit::residual_iters(int l, int* host) {
    Level& lv = levels[l];
    const int lo = range_lo(l);
    DevBuf<int> it((size_t)lv.steps + 1);
    it.zero(stream);
    iters_dev = it.get() + lo * cfg.m + 1;  // task 0 of the residual wave is point lo m + 1
    std::vector<double> scratch(lv.steps + 1);
    try {
        residual_terms(l, scratch.data());
    } catch (...) {
        iters_dev = nullptr;
        throw;
    }
    iters_dev = nullptr;
    const std::vector<int> h = it.download(stream);
    std::copy(h.begin(), h.end(), host);
}

double Mgrit::compute_g_norm() {
    TraceRange trace_range("phi.mgrit.g_norm");
    std::vector<double> h(levels[0].steps + 1);
    gnorm_terms(h.data());
    double total = 0.0;
    for (double s : h) total += s;  // [0] = |g_0|^2 summed in index order, then the points
    return std::sqrt(total);
}

// g-norm terms (mgrit.hpp:292-310): [0] = |g_0|^2 (index-ordered), [k] =
// |Phi-solve of load_k|^2 for the transient loads of the owned points (a
// steady load contributes steps copies of one term, folded into [1]).
void Mgrit::gnorm_terms(double* host) {
    Level& lv0 = levels[0];
    const int n = disc->n_p;
    const int lo = range_lo(0), hi = range_hi(0);
    std::vector<double> h(lv0.steps + 1, 0.0);
    if (lo == 0) {
        std::vector<double> g0(n);
        PHI_CUDA(cudaMemcpyAsync(g0.data(), lv0.g.get(), sizeof(double) * n, cudaMemcpyDeviceToHost, stream));
        PHI_CUDA(cudaStreamSynchronize(stream));
        double t = 0.0;
        for (int i = 0; i < n; ++i) t += g0[i] * g0[i];
        h[0] = t;
    }
    if (has_loads) {
        PHI_CUDA(cudaMemsetAsync(sq.get(), 0, sizeof(double) * (lv0.steps + 1), stream));
        if (loads_steady) {
            if (lo == 0) {
                wave(0, kModeSolve, kEpiNorm, 1, lv0.kAll.get(), 1);
                double v = 0.0;
                PHI_CUDA(cudaMemcpyAsync(&v, sq.get() + 1, sizeof(double), cudaMemcpyDeviceToHost, stream));
                PHI_CUDA(cudaStreamSynchronize(stream));
                check_errors();
                h[1] = lv0.steps * v;
            }
        } else {
            const int k_begin = lo * cfg.m + 1;
            const int k_end = (hi == lv0.steps / cfg.m) ? lv0.steps : hi * cfg.m;
            if (k_end >= k_begin)
                wave(0, kModeSolve, kEpiNorm, k_end - k_begin + 1, lv0.kAll.get() + (k_begin - 1), 1);
            std::vector<double> s(lv0.steps + 1);
            PHI_CUDA(cudaMemcpyAsync(s.data(), sq.get(), sizeof(double) * s.size(), cudaMemcpyDeviceToHost, stream));
            PHI_CUDA(cudaStreamSynchronize(stream));
            check_errors();
            for (int k = 1; k <= lv0.steps; ++k) h[k] = s[k];
        }
    }
    std::copy(h.begin(), h.end(), host);
}

void Mgrit::initialize() {
    initialize_state();
    g_norm = compute_g_norm();
}

void Mgrit::initialize_state() {
    const int n = disc->n_p;
    for (auto& lv : levels) {
        lv.u.zero(stream);
        lv.g.zero(stream);
    }
    project_initial();
    launch_copy(levels[0].g.get(), u0.get(), n, stream);
    launch_copy(levels[0].u.get(), u0.get(), n, stream);
    launches += 2;
    stat.zero(stream);
    stat_c.zero(stream);
    const std::vector<int> e0{0, INT_MAX, -1};
    err.upload(e0, stream);
}

void Mgrit::set_range(int lo, int hi) {
    const int J = levels[0].steps / cfg.m;
    if (lo < 0 || (hi >= 0 && (hi < lo || hi > J))) throw InvalidArgument("MGRIT interval range out of bounds");
    j_lo = lo;
    j_hi = hi;
}

void Mgrit::phase(int l, int op) {
    if (l < 0 || l >= n_levels()) throw InvalidArgument("MGRIT level out of range");
    switch (op) {
        case 0: f_relax(l, false); break;
        case 1: f_relax(l, true); break;
        case 2:
            if (l + 1 >= n_levels()) throw InvalidArgument("restriction from the coarsest level");
            restrict_residual(l);
            break;
        case 3: {  // fine.u[j m] += coarse.u[j] for every C-point (mgrit.hpp:172-180)
            if (l + 1 >= n_levels()) throw InvalidArgument("interpolation to the coarsest level");
            Level& f = levels[l];
            Level& c = levels[l + 1];
            launch_inject(c.u.get(), f.u.get(), disc->n_p, f.steps / cfg.m, cfg.m, stream);
            ++launches;
            break;
        }
        case 4: cycle_impl(l, cfg.cycle == 1); break;
        case 5: cycle_impl(l, false); break;  // the F-schedule's second pass below level l - 1
        default: throw InvalidArgument("unknown MGRIT phase");
    }
    PHI_CUDA(cudaStreamSynchronize(stream));
    check_errors();
}

void Mgrit::points(int l, int which, int k0, int count, double* ptr, bool device, bool set) {
    if (l < 0 || l >= n_levels()) throw InvalidArgument("MGRIT level out of range");
    Level& lv = levels[l];
    if (k0 < 0 || count < 0 || k0 + count > lv.steps + 1) throw InvalidArgument("MGRIT point range out of bounds");
    const size_t n = disc->n_p;
    double* arr = (which == 0 ? lv.u.get() : lv.g.get()) + (size_t)k0 * n;
    const size_t bytes = sizeof(double) * n * count;
    if (set)
        PHI_CUDA(cudaMemcpyAsync(arr, ptr, bytes, device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, stream));
    else
        PHI_CUDA(cudaMemcpyAsync(ptr, arr, bytes, device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, stream));
    PHI_CUDA(cudaStreamSynchronize(stream));
}

void Mgrit::stats(long long* out4) const {
    const auto s0 = stat.download(stream);
    const auto sc = stat_c.download(stream);
    out4[0] = (long long)s0[0];
    out4[1] = (long long)s0[1];
    out4[2] = (long long)sc[0];
    out4[3] = (long long)sc[1];
}

void Mgrit::set_init_coeffs(const double* host) {
    if (ps.init_kind != 2 && ps.init_kind != 3)
        throw InvalidArgument("set_init_coeffs: problem has no coefficient initial condition");
    std::copy(host, host + disc->n_p, ps.init_coeffs.begin());
}



void Mgrit::wave_levels(double* ms, long long* points, long long* cycles, int cap) {
    for (int l = 0; l < cap; ++l) {
        ms[l] = 0.0;
        points[l] = cycles[l] = 0;
    }
    if (recs.empty()) return;
    std::vector<int> st(3 * recs.size());
    PHI_CUDA(cudaMemcpy(st.data(), wstats.get(), sizeof(int) * st.size(), cudaMemcpyDeviceToHost));
    for (size_t k = 0; k < recs.size(); ++k) {
        const int l = recs[k].level;
        if (l >= cap) continue;
        float t = 0.f;
        PHI_CUDA(cudaEventElapsedTime(&t, recs[k].start, recs[k].stop));
        ms[l] += t;
        cycles[l] += st[3 * k + 1];
        points[l] += st[3 * k + 2];
    }
}

// Algorithmic bytes: 8 B per stored nonzero of the reference
// operators read once per wave-phase (the batch shares them) plus 8 B per
// vector entry read or written once per right-hand side.
int Mgrit::wave_report(double* ms, double* bytes) {
    *ms = 0.0;
    *bytes = 0.0;
    if (recs.empty()) return 0;
    std::vector<int> st(3 * recs.size());
    PHI_CUDA(cudaMemcpy(st.data(), wstats.get(), sizeof(int) * st.size(), cudaMemcpyDeviceToHost));
    const Disc& d = *disc;
    const double n = d.n_p, n1 = d.n_1;
    for (size_t k = 0; k < recs.size(); ++k) {
        float t = 0.f;
        PHI_CUDA(cudaEventElapsedTime(&t, recs[k].start, recs[k].stop));
        *ms += t;
        const Stepper& S = *levels[recs[k].level].stepper;
        const Hier& H = *S.hier;
        const double nnzA = (double)stencil_nnz(H.A.view());
        const double cmax = st[3 * k], csum = st[3 * k + 1], pts = st[3 * k + 2];
        if (H.cg_only) {  // CG kind: A once per iteration (shared by the batch), 18 n per iteration and RHS
            const double mat = nnzA /* A- */ + (1 + cmax) * nnzA;
            const double vec = pts * (5 * n + 3 * n) + pts * 5 * n + csum * 18 * n;
            *bytes += 8.0 * (mat + vec);
            continue;
        }
        const double vmat = H.vcycle_matrix_entries(), vvec = H.vcycle_vector_entries();
        (void)n1;
        const double mat = nnzA /* A- */ + (1 + cmax) * nnzA + cmax * vmat;
        const double vec = pts * (5 * n + 3 * n) + (pts + csum) * 4 * n + csum * vvec;
        *bytes += 8.0 * (mat + vec);
        if (std::getenv("PHI_WAVE_DEBUG")) {
            float t0 = 0.f;  // start relative to the first recorded wave
            PHI_CUDA(cudaEventElapsedTime(&t0, recs[0].start, recs[k].start));
            std::fprintf(stderr, "wave %zu level %d: %.3f ms at +%.3f ms, points %d, cycles sum %d max %d, algorithmic %.4e B\n",
                         k, recs[k].level, t, t0, (int)pts, (int)csum, (int)cmax, 8.0 * (mat + vec));
        }
    }
    for (auto& r : recs) {
        cudaEventDestroy(r.start);
        cudaEventDestroy(r.stop);
    }
    const int nw = (int)recs.size();
    recs.clear();
    return nw;
}

MgritResultHost Mgrit::solve() {
    TraceRange trace_range("phi.mgrit.solve");
    if (comm) return solve_sharded();
    launches = 0;
    for (auto& r : recs) {
        cudaEventDestroy(r.start);
        cudaEventDestroy(r.stop);
    }
    recs.clear();
    if (profile) {
        if (wstats.size() == 0) wstats.alloc(3 * 8192);
        wstats.zero(stream);
    }
    initialize();
    MgritResultHost res;
    res.g_norm = g_norm;
    const double denom = g_norm > 0.0 ? g_norm : 1.0;
    for (int it = 1; it <= cfg.max_iter; ++it) {
        mgrit_cycle(0);
        const double rel = residual_norm(0) / denom;
        res.residual_history.push_back(rel);
        res.iterations = it;
        if (rel <= cfg.halt_tol) {
            res.converged = true;
            break;
        }
    }
    res.final_relative_residual = res.residual_history.back();
    long long st[4];
    stats(st);
    const long long solves = st[0] + st[2], iters = st[1] + st[3];
    res.total_spatial_solves = solves;
    res.mean_spatial_iterations = solves > 0 ? (double)iters / (double)solves : 0.0;
    return res;
}

}  // namespace phi
