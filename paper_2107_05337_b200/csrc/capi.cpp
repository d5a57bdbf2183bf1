// extern "C" boundary of the engine (include/phi_engine.h).  Maps the
// reference's exception types onto status codes and keeps the message
// thread-local, worded as the reference's exception text.
#include <climits>
#include <cmath>
#include <cstring>
#include <memory>
#include <string>

#include "../../include/phi_engine.h"
#include "engine.hpp"

using namespace phi;

namespace {

thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
    try {
        f();
        return PHI_OK;
    } catch (const InvalidArgument& e) {
        g_err = e.what();
        return PHI_ERR_INVALID;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return PHI_ERR_INVALID;
    } catch (const NotConverged& e) {
        g_err = e.what();
        return PHI_ERR_NOT_CONVERGED;
    } catch (const CudaError& e) {
        g_err = e.what();
        return PHI_ERR_CUDA;
    } catch (const std::exception& e) {
        g_err = e.what();
        return PHI_ERR_RUNTIME;
    }
}

int export_csr(const HostCsr& a, int* n_rows, int* n_cols, int* nnz, int* ro, int* ci, double* v) {
    if (n_rows) *n_rows = a.n_rows;
    if (n_cols) *n_cols = a.n_cols;
    if (nnz) *nnz = a.nnz();
    if (ro) std::memcpy(ro, a.row_offsets.data(), sizeof(int) * (a.n_rows + 1));
    if (ci) std::memcpy(ci, a.col_indices.data(), sizeof(int) * a.nnz());
    if (v) std::memcpy(v, a.values.data(), sizeof(double) * a.nnz());
    return PHI_OK;
}

HierOptions to_opts(const phi_pmg_options* o) {
    HierOptions h;
    if (o) {
        h.ilut_tau = o->ilut_tau;
        h.ilut_fill = o->ilut_fill;
        h.nu_pre = o->nu_pre;
        h.nu_post = o->nu_post;
        h.gs_pre = o->gs_pre;
        h.gs_post = o->gs_post;
        h.exact = o->exact;
    }
    return h;
}

SolverConfig to_cfg(const phi_solver_config* c) {
    SolverConfig s;
    if (c) {
        s.kind = c->kind;
        s.rel_tol = c->rel_tol;
        s.max_iter = c->max_iter;
        s.fixed_cycles = c->fixed_cycles;
        s.pmg = to_opts(&c->pmg);
    }
    return s;
}

void require_device() {
    int n = 0;
    const cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess || n == 0)
        throw CudaError(std::string("no CUDA device available (the engine has no CPU path): ") +
                        cudaGetErrorString(e));
}

/// Staging of host or device batch arrays (nrhs vectors, stride ld).
struct Batch {
    DevBuf<double> buf;
    double* ptr = nullptr;
    long long ld = 0;
    void in(const double* src, int nrhs, long long ld_, int n, int device_ptrs, cudaStream_t s) {
        if (!src) {
            ptr = nullptr;
            return;
        }
        if (device_ptrs) {
            ptr = const_cast<double*>(src);
            ld = ld_;
            return;
        }
        buf.alloc((size_t)nrhs * n);
        for (int r = 0; r < nrhs; ++r)
            PHI_CUDA(cudaMemcpyAsync(buf.get() + (size_t)r * n, src + (size_t)r * ld_, sizeof(double) * n,
                                     cudaMemcpyHostToDevice, s));
        ptr = buf.get();
        ld = n;
    }
    void out(double* dst, int nrhs, long long ld_, int n, int device_ptrs, cudaStream_t s) {
        if (device_ptrs) return;
        for (int r = 0; r < nrhs; ++r)
            PHI_CUDA(cudaMemcpyAsync(dst + (size_t)r * ld_, buf.get() + (size_t)r * n, sizeof(double) * n,
                                     cudaMemcpyDeviceToHost, s));
    }
};

}  // namespace

struct phi_disc {
    std::shared_ptr<Disc> d;
    HostCsr csr_cache(int which) const {
        if (which == 0) return d->to_csr(d->M);
        if (which == 1) return d->to_csr(d->K);
        if (which == 2) return d->to_csr(d->T);
        if (which >= 100 && which < 200) return d->to_csr(d->h.at(which - 100).M);
        if (which >= 200 && which < 300) return d->to_csr(d->h.at(which - 200).K);
        if (which >= 300 && which < 400) {
            const auto& hl = d->h.at(which - 300);
            if (which - 300 + 1 >= (int)d->h.size()) throw InvalidArgument("embed: coarsest level has none");
            return hl.E;
        }
        throw InvalidArgument("phi_disc_export: bad selector");
    }
};

struct phi_hier {
    std::unique_ptr<Hier> h;
    Workspace ws;
    cudaStream_t s = nullptr;
};

struct phi_stepper {
    std::unique_ptr<Stepper> st;
    Workspace ws;
    DevBuf<int> iters, conv;
    DevBuf<unsigned long long> stat;
    DevBuf<int> err;
    DevBuf<double> err_rel;
    cudaStream_t s = nullptr;
};

struct phi_mgrit {
    std::unique_ptr<Mgrit> g;
};

extern "C" {

const char* phi_last_error(void) { return g_err.c_str(); }

void phi_default_solver_config(phi_solver_config* c) {
    c->kind = PHI_SOLVER_PMG;
    c->rel_tol = 1e-12;
    c->max_iter = 400;
    c->fixed_cycles = 0;
    c->pmg.ilut_tau = 1e-13;
    c->pmg.ilut_fill = 0;
    c->pmg.nu_pre = c->pmg.nu_post = 1;
    c->pmg.gs_pre = c->pmg.gs_post = 2;
    c->pmg.exact = 0;
}

void phi_default_mgrit_config(phi_mgrit_config* c) {
    c->cycle = 0;
    c->relax = 1;
    c->m = 2;
    c->halt_tol = 1e-10;
    c->max_iter = 50;
    c->coarse_floor = 8;
}

void phi_default_problem(phi_problem* p) {
    std::memset(p, 0, sizeof *p);
    p->kappa = 1.0;
    p->t_final = 0.1;
    p->theta = 1.0;
    p->n_time_steps = 64;
    p->source_kind = PHI_SOURCE_CONSTANT;
    p->source_param = 1.0;
    p->init_kind = PHI_INIT_ZERO;
}

int phi_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) return 0;
    return n;
}

int phi_set_device(int device) {
    return guarded([&] { PHI_CUDA(cudaSetDevice(device)); });
}

int phi_synchronize(void) {
    return guarded([&] { PHI_CUDA(cudaDeviceSynchronize()); });
}

// ---- disc -----------------------------------------------------------------
int phi_disc_build(int degree, int mesh_exponent, phi_disc** out) {
    return guarded([&] {
        // argument errors come first, as the reference throws before any work
        if (degree < 1 || degree > 8) throw InvalidArgument("SpatialDiscretization: degree must be in [1, 8]");
        if (mesh_exponent < 1) throw InvalidArgument("SpatialDiscretization: mesh exponent must be >= 1");
        require_device();
        auto* d = new phi_disc;
        try {
            d->d = Disc::build(degree, mesh_exponent);
        } catch (...) {
            delete d;
            throw;
        }
        *out = d;
    });
}

void phi_disc_free(phi_disc* d) { delete d; }

int phi_disc_info(const phi_disc* d, int* info) {
    return guarded([&] {
        info[0] = d->d->n_p;
        info[1] = d->d->n_1;
        info[2] = (int)d->d->h.size();
        info[3] = d->d->n_elements;
        info[4] = d->d->degree;
    });
}

int phi_disc_export(const phi_disc* d, int which, int* n_rows, int* n_cols, int* nnz, int* ro, int* ci,
                    double* v) {
    return guarded([&] { export_csr(d->csr_cache(which), n_rows, n_cols, nnz, ro, ci, v); });
}

int phi_disc_vector(const phi_disc* d, int which, double* out) {
    return guarded([&] {
        const auto& b = which == 0 ? d->d->inv_lp : d->d->inv_l1;
        const auto h = b.download();
        std::memcpy(out, h.data(), sizeof(double) * h.size());
    });
}

// ---- hier -----------------------------------------------------------------
int phi_hier_create(const phi_disc* d, double c, const phi_pmg_options* opt, phi_hier** out) {
    return guarded([&] {
        auto h = std::make_unique<phi_hier>();
        h->h = std::make_unique<Hier>(d->d, c, to_opts(opt));
        *out = h.release();
    });
}

void phi_hier_free(phi_hier* h) { delete h; }

int phi_hier_export(const phi_hier* h, int which, int* n_rows, int* n_cols, int* nnz, int* ro, int* ci,
                    double* v) {
    return guarded([&] {
        if (which == 0)
            export_csr(h->h->disc->to_csr(h->h->A), n_rows, n_cols, nnz, ro, ci, v);
        else if (which == 1)
            export_csr(h->h->L_host, n_rows, n_cols, nnz, ro, ci, v);
        else if (which == 2)
            export_csr(h->h->U_host, n_rows, n_cols, nnz, ro, ci, v);
        else if (which >= 100 && which - 100 < (int)h->h->a_h.size())
            export_csr(h->h->a_h_csr(which - 100), n_rows, n_cols, nnz, ro, ci, v);
        else
            throw InvalidArgument("phi_hier_export: bad selector");
    });
}

int phi_hier_vcycle(phi_hier* h, const double* b, double* x, int nrhs, long long ld, int device_ptrs) {
    return guarded([&] {
        const int n = h->h->disc->n_p;
        if (ld < n) throw InvalidArgument("vcycle: dimension mismatch");
        SolverConfig cfg;
        const DevHier H = h->h->view(cfg);
        h->ws.ensure(H);
        Batch bb, xb;
        bb.in(b, nrhs, ld, n, device_ptrs, h->s);
        xb.in(x, nrhs, ld, n, device_ptrs, h->s);
        launch_vcycle(H, bb.ptr, bb.ld, xb.ptr, xb.ld, nrhs, h->ws.buf.get(), h->ws.stride, h->ws.slots, h->s);
        xb.out(x, nrhs, ld, n, device_ptrs, h->s);
        PHI_CUDA(cudaStreamSynchronize(h->s));
    });
}

int phi_hier_solve(phi_hier* h, const double* b, double* x, int nrhs, long long ld, double rel_tol,
                   int max_iter, int fixed_cycles, int x0_empty, int* iters, int* converged, double* final_rel,
                   int device_ptrs) {
    return guarded([&] {
        const int n = h->h->disc->n_p;
        if (ld < n) throw InvalidArgument("solve: dimension mismatch");
        SolverConfig cfg;
        cfg.rel_tol = rel_tol;
        cfg.max_iter = max_iter;
        cfg.fixed_cycles = fixed_cycles;
        const DevHier H = h->h->view(cfg);
        h->ws.ensure(H);
        Batch bb, xb;
        bb.in(b, nrhs, ld, n, device_ptrs, h->s);
        xb.in(x, nrhs, ld, n, device_ptrs, h->s);
        DevBuf<int> it(nrhs), cv(nrhs);
        DevBuf<double> fr(nrhs);
        WaveArgs a{};
        a.mode = kModeSolve;
        a.epi = kEpiSolve;
        a.n_tasks = nrhs;
        a.task_len = 1;
        a.n = n;
        a.B = bb.ptr;
        a.ldb = bb.ld;
        a.X = xb.ptr;
        a.ldx = xb.ld;
        a.x0_empty = x0_empty;
        a.iters_out = it.get();
        a.conv_out = cv.get();
        a.rel_out = fr.get();
        launch_phi_wave(H, h->h->A.view(), a, h->ws.buf.get(), h->ws.stride, h->ws.slots, h->s);
        xb.out(x, nrhs, ld, n, device_ptrs, h->s);
        const auto hi = it.download(h->s);
        const auto hc = cv.download(h->s);
        const auto hf = fr.download(h->s);
        for (int r = 0; r < nrhs; ++r) {
            if (iters) iters[r] = hi[r];
            if (converged) converged[r] = hc[r];
            if (final_rel) final_rel[r] = hf[r];
        }
    });
}

int phi_hier_spmm(phi_hier* h, const double* x, double* y, int nrhs, int device_ptrs) {
    return guarded([&] {
        const StencilBuf& A = h->h->A;
        const size_t n = (size_t)A.ru * A.rv, len = n * (size_t)nrhs;
        const double* At = h->h->a_tiled(h->s, tile_kind(nrhs));
        if (device_ptrs) {
            launch_spmm(A.view(), At, x, y, nrhs, h->s);
        } else {
            DevBuf<double> dx(len), dy(len);
            PHI_CUDA(cudaMemcpyAsync(dx.get(), x, sizeof(double) * len, cudaMemcpyHostToDevice, h->s));
            launch_spmm(A.view(), At, dx.get(), dy.get(), nrhs, h->s);
            PHI_CUDA(cudaMemcpyAsync(y, dy.get(), sizeof(double) * len, cudaMemcpyDeviceToHost, h->s));
        }
        PHI_CUDA(cudaStreamSynchronize(h->s));
    });
}

int phi_hier_vcycle_bytes(const phi_hier* h, int nrhs, double* bytes) {
    return guarded([&] {
        if (nrhs < 1) throw InvalidArgument("phi_hier_vcycle_bytes: nrhs must be positive");
        *bytes = 8.0 * (h->h->vcycle_matrix_entries() + nrhs * h->h->vcycle_vector_entries());
    });
}

int phi_hier_time(phi_hier* h, int which, int nrhs, int reps, int flush_l2, double* ms_out) {
    return guarded([&] {
        if (reps < 1 || nrhs < 1) throw InvalidArgument("phi_hier_time: reps and nrhs must be positive");
        const StencilBuf& A = h->h->A;
        const size_t n = (size_t)A.ru * A.rv, len = n * (size_t)nrhs;
        // seeded N(0,1) right-hand sides (mt19937_64 + Box-Muller, portable)
        std::vector<double> hb(len);
        unsigned long long st = 0x9E3779B97F4A7C15ULL;
        auto next = [&]() {
            st ^= st >> 12;
            st ^= st << 25;
            st ^= st >> 27;
            return (double)((st * 2685821657736338717ULL) >> 11) * (1.0 / 9007199254740992.0);
        };
        for (size_t i = 0; i < len; i += 2) {
            const double u1 = std::max(next(), 1e-300), u2 = next();
            const double r = std::sqrt(-2.0 * std::log(u1));
            hb[i] = r * std::cos(2.0 * M_PI * u2);
            if (i + 1 < len) hb[i + 1] = r * std::sin(2.0 * M_PI * u2);
        }
        DevBuf<double> b(len), x(len), flush;
        PHI_CUDA(cudaMemcpyAsync(b.get(), hb.data(), sizeof(double) * len, cudaMemcpyHostToDevice, h->s));
        if (flush_l2) {  // 256 MB > L2, zeroed once; each repetition reads it (clean lines, no write-backs)
            flush.alloc((size_t)32 << 20);
            PHI_CUDA(cudaMemsetAsync(flush.get(), 0, sizeof(double) * ((size_t)32 << 20), h->s));
        }
        SolverConfig cfg;
        const DevHier H = h->h->view(cfg);
        if (which == 1) h->ws.ensure(H);
        cudaEvent_t e0, e1;
        PHI_CUDA(cudaEventCreate(&e0));
        PHI_CUDA(cudaEventCreate(&e1));
        double total = 0.0;
        if (which == 0 && flush_l2 == 2) {
            // back-to-back launches over four copies of the operator (> L2 in
            // total at the config-5 sizes): the kernel's average launch duration
            // without the event pair's and the idle start's share of a ~10 us run
            const int kind = tile_kind(nrhs), copies = 4;
            const size_t td = tile_doubles(A.view(), kind);
            const double* at0 = h->h->a_tiled(h->s, kind);
            std::vector<DevBuf<double>> at(copies);
            for (auto& c : at) {
                c.alloc(td);
                PHI_CUDA(cudaMemcpyAsync(c.get(), at0, sizeof(double) * td, cudaMemcpyDeviceToDevice, h->s));
            }
            for (int c = 0; c < copies; ++c) launch_spmm(A.view(), at[c].get(), b.get(), x.get(), nrhs, h->s);
            PHI_CUDA(cudaEventRecord(e0, h->s));
            for (int r = 0; r < reps * copies; ++r)
                launch_spmm(A.view(), at[r % copies].get(), b.get(), x.get(), nrhs, h->s);
            PHI_CUDA(cudaEventRecord(e1, h->s));
            PHI_CUDA(cudaEventSynchronize(e1));
            float ms = 0.f;
            PHI_CUDA(cudaEventElapsedTime(&ms, e0, e1));
            total = (double)ms / copies;
        } else
        for (int r = -1; r < reps; ++r) {  // r = -1: warm-up
            if (flush_l2) launch_l2_flush_read(flush.get(), (size_t)32 << 20, x.get(), h->s);
            if (which == 1) PHI_CUDA(cudaMemsetAsync(x.get(), 0, sizeof(double) * len, h->s));  // x0 = 0
            PHI_CUDA(cudaEventRecord(e0, h->s));
            if (which == 0)
                launch_spmm(A.view(), h->h->a_tiled(h->s, tile_kind(nrhs)), b.get(), x.get(), nrhs, h->s);  // X, Y: [n][nrhs]
            else
                launch_vcycle(H, b.get(), (long long)n, x.get(), (long long)n, nrhs, h->ws.buf.get(), h->ws.stride,
                              h->ws.slots, h->s);
            PHI_CUDA(cudaEventRecord(e1, h->s));
            PHI_CUDA(cudaEventSynchronize(e1));
            float ms = 0.f;
            PHI_CUDA(cudaEventElapsedTime(&ms, e0, e1));
            if (r >= 0) total += ms;
        }
        PHI_CUDA(cudaEventDestroy(e0));
        PHI_CUDA(cudaEventDestroy(e1));
        *ms_out = total / reps;
    });
}

int phi_hier_unit(phi_hier* h, int op, int arg, int arg2, const double* in, int n_in, double* out, int n_out) {
    return guarded([&] {
        SolverConfig cfg;
        const DevHier H = h->h->view(cfg);
        h->ws.ensure(H);
        DevBuf<double> din(n_in), dout(n_out);
        PHI_CUDA(cudaMemcpyAsync(din.get(), in, sizeof(double) * n_in, cudaMemcpyHostToDevice, h->s));
        PHI_CUDA(cudaMemcpyAsync(dout.get(), out, sizeof(double) * n_out, cudaMemcpyHostToDevice, h->s));
        launch_unit(H, op, arg, arg2, din.get(), dout.get(), h->ws.buf.get(), h->ws.stride, h->s);
        PHI_CUDA(cudaMemcpyAsync(out, dout.get(), sizeof(double) * n_out, cudaMemcpyDeviceToHost, h->s));
        PHI_CUDA(cudaStreamSynchronize(h->s));
    });
}

// ---- stepper --------------------------------------------------------------
int phi_stepper_create(const phi_disc* d, double kappa, double dt, double theta, const phi_solver_config* cfg,
                       phi_stepper** out) {
    return guarded([&] {
        auto s = std::make_unique<phi_stepper>();
        s->st = std::make_unique<Stepper>(d->d, kappa, dt, theta, to_cfg(cfg));
        s->stat.alloc(2);
        s->err.alloc(3);
        s->err_rel.alloc(1);
        *out = s.release();
    });
}

void phi_stepper_free(phi_stepper* s) { delete s; }

static void stepper_reset_err(phi_stepper* s) {
    const std::vector<int> e0{0, INT_MAX, -1};
    s->err.upload(e0, s->s);
    s->stat.zero(s->s);
}

static void stepper_check(phi_stepper* s, const std::string& prefix) {
    const auto e = s->err.download(s->s);
    if (e[0]) {
        const double rel = s->err_rel.download(s->s)[0];
        throw NotConverged(prefix + spatial_failure(s->st->cfg.kind, rel));
    }
}

int phi_stepper_step(phi_stepper* s, const double* u_prev, const double* load, double* x, int nrhs, long long ld,
                     int guess_empty, int* iters, int device_ptrs) {
    return guarded([&] {
        const int n = s->st->disc->n_p;
        if (ld < n) throw InvalidArgument("step: dimension mismatch");
        s->ws.ensure(s->st->H);
        stepper_reset_err(s);
        Batch ub, lb, xb;
        ub.in(u_prev, nrhs, ld, n, device_ptrs, s->s);
        lb.in(load, nrhs, ld, n, device_ptrs, s->s);
        xb.in(x, nrhs, ld, n, device_ptrs, s->s);
        DevBuf<int> it(nrhs);
        WaveArgs a{};
        a.mode = kModeStep;
        a.epi = kEpiSolve;
        a.n_tasks = nrhs;
        a.task_len = 1;
        a.n = n;
        a.UPREV = ub.ptr;
        a.ldu = ub.ld;
        a.LOADV = lb.ptr;
        a.ldl = lb.ld;
        a.X = xb.ptr;
        a.ldx = xb.ld;
        a.x0_empty = guess_empty;
        a.iters_out = it.get();
        a.stat = s->stat.get();
        a.err = s->err.get();
        a.err_rel = s->err_rel.get();
        launch_phi_wave(s->st->H, s->st->Aminus.view(), a, s->ws.buf.get(), s->ws.stride, s->ws.slots, s->s);
        xb.out(x, nrhs, ld, n, device_ptrs, s->s);
        const auto hi = it.download(s->s);
        if (iters)
            for (int r = 0; r < nrhs; ++r) iters[r] = hi[r];
        stepper_check(s, "");
    });
}

int phi_sequential_integrate(phi_stepper* s, int nt, const double* u0, const double* loads, int load_steady,
                             double* traj, long long* solves, long long* iterations) {
    return guarded([&] {
        const int n = s->st->disc->n_p;
        if (nt < 1) throw InvalidArgument("ProblemSpec: nt must be >= 1");
        s->ws.ensure(s->st->H);
        stepper_reset_err(s);
        DevBuf<double> U((size_t)(nt + 1) * n), L;
        U.zero(s->s);
        if (u0) PHI_CUDA(cudaMemcpyAsync(U.get(), u0, sizeof(double) * n, cudaMemcpyHostToDevice, s->s));
        if (loads) {
            const size_t cnt = load_steady ? (size_t)n : (size_t)n * nt;
            L.alloc(cnt);
            PHI_CUDA(cudaMemcpyAsync(L.get(), loads, sizeof(double) * cnt, cudaMemcpyHostToDevice, s->s));
        }
        const std::vector<int> k0{1};
        DevBuf<int> dk0 = to_device(k0, s->s);
        WaveArgs a{};
        a.mode = kModeStep;
        a.epi = kEpiStore;
        a.n_tasks = 1;
        a.task_len = nt;
        a.task_k0 = dk0.get();
        a.n = n;
        a.U = U.get();
        a.LOAD = loads ? L.get() : nullptr;
        a.load_steady = load_steady;
        a.guess_prev = 1;
        a.stat = s->stat.get();
        a.err = s->err.get();
        a.err_rel = s->err_rel.get();
        launch_phi_wave(s->st->H, s->st->Aminus.view(), a, s->ws.buf.get(), s->ws.stride, s->ws.slots, s->s);
        PHI_CUDA(cudaMemcpyAsync(traj, U.get(), sizeof(double) * (size_t)(nt + 1) * n, cudaMemcpyDeviceToHost, s->s));
        PHI_CUDA(cudaStreamSynchronize(s->s));
        const auto st = s->stat.download(s->s);
        if (solves) *solves = (long long)st[0];
        if (iterations) *iterations = (long long)st[1];
        const auto e = s->err.download(s->s);
        if (e[0]) {
            const double rel = s->err_rel.download(s->s)[0];
            throw NotConverged("sequential_integrate: step " + std::to_string(e[1]) + ": " +
                               spatial_failure(s->st->cfg.kind, rel));
        }
    });
}

// ---- mgrit ----------------------------------------------------------------
int phi_mgrit_create(const phi_disc* d, const phi_problem* ps, const phi_mgrit_config* cfg,
                     const phi_solver_config* scfg, phi_mgrit** out) {
    return guarded([&] {
        ProblemOptions po;
        po.kappa = ps->kappa;
        po.t_final = ps->t_final;
        po.theta = ps->theta;
        po.n_time_steps = ps->n_time_steps;
        po.source_kind = ps->source_kind;
        po.source_param = ps->source_param;
        po.init_kind = ps->init_kind;
        const int n = d->d->n_p;
        if (ps->init_kind == PHI_INIT_COEFFS || ps->init_kind == PHI_INIT_VECTOR) {
            if (!ps->init_coeffs) throw InvalidArgument("init_coeffs missing");
            po.init_coeffs.assign(ps->init_coeffs, ps->init_coeffs + n);
        }
        if (ps->load_terms) {
            const size_t cnt = ps->load_terms_steady ? (size_t)n : (size_t)n * ps->n_time_steps;
            po.load_terms.assign(ps->load_terms, ps->load_terms + cnt);
            po.load_terms_steady = ps->load_terms_steady;
        }
        MgritOptions mo;
        if (cfg) {
            mo.cycle = cfg->cycle;
            mo.relax = cfg->relax;
            mo.m = cfg->m;
            mo.halt_tol = cfg->halt_tol;
            mo.max_iter = cfg->max_iter;
            mo.coarse_floor = cfg->coarse_floor;
        }
        auto g = std::make_unique<phi_mgrit>();
        g->g = std::make_unique<Mgrit>(d->d, po, mo, to_cfg(scfg));
        *out = g.release();
    });
}

void phi_mgrit_free(phi_mgrit* g) { delete g; }

int phi_mgrit_levels(const phi_mgrit* g, int* steps, double* dts) {
    const int L = g->g->n_levels();
    for (int l = 0; l < L; ++l) {
        if (steps) steps[l] = g->g->levels[l].steps;
        if (dts) dts[l] = g->g->levels[l].dt;
    }
    return L;
}

int phi_mgrit_solve(phi_mgrit* g, phi_mgrit_result* res, double* history, int history_cap) {
    return guarded([&] {
        const MgritResultHost r = g->g->solve();
        res->iterations = r.iterations;
        res->converged = r.converged ? 1 : 0;
        res->g_norm = r.g_norm;
        res->final_relative_residual = r.final_relative_residual;
        res->total_spatial_solves = r.total_spatial_solves;
        res->mean_spatial_iterations = r.mean_spatial_iterations;
        if (history)
            for (int i = 0; i < (int)r.residual_history.size() && i < history_cap; ++i)
                history[i] = r.residual_history[i];
    });
}

int phi_mgrit_trajectory(const phi_mgrit* g, double* out) {
    return guarded([&] {
        const_cast<phi_mgrit*>(g)->g->gather_trajectory();  // sharded: collective gather
        const auto& lv = g->g->levels[0];
        PHI_CUDA(cudaMemcpyAsync(out, lv.u.get(), sizeof(double) * lv.u.size(), cudaMemcpyDeviceToHost,
                                 g->g->stream));
        PHI_CUDA(cudaStreamSynchronize(g->g->stream));
    });
}

int phi_mgrit_initial(const phi_mgrit* g, double* out) {
    return guarded([&] {
        const auto h = g->g->u0.download(g->g->stream);
        std::memcpy(out, h.data(), sizeof(double) * h.size());
    });
}

int phi_mgrit_initialize(phi_mgrit* g, double* g_norm) {
    return guarded([&] {
        g->g->initialize();
        if (g_norm) *g_norm = g->g->g_norm;
    });
}

int phi_mgrit_cycle(phi_mgrit* g, int level) {
    return guarded([&] { g->g->mgrit_cycle(level); });
}

int phi_mgrit_residual_norm(phi_mgrit* g, int level, double* out) {
    return guarded([&] { *out = g->g->residual_norm(level); });
}

long long phi_mgrit_launches(const phi_mgrit* g) { return g->g->launches; }

int phi_mgrit_set_range(phi_mgrit* g, int j_lo, int j_hi) {
    return guarded([&] { g->g->set_range(j_lo, j_hi); });
}

int phi_mgrit_initialize_state(phi_mgrit* g) {
    return guarded([&] { g->g->initialize_state(); });
}

int phi_mgrit_gnorm_terms(phi_mgrit* g, double* terms) {
    return guarded([&] { g->g->gnorm_terms(terms); });
}

int phi_mgrit_residual_terms(phi_mgrit* g, int level, double* terms) {
    return guarded([&] { g->g->residual_terms(level, terms); });
}

int phi_mgrit_residual_iters(phi_mgrit* g, int level, int* iters) {
    return guarded([&] {
        if (level < 0 || level >= g->g->n_levels()) throw InvalidArgument("MGRIT level out of range");
        g->g->residual_iters(level, iters);
    });
}

int phi_mgrit_phase(phi_mgrit* g, int level, int op) {
    return guarded([&] { g->g->phase(level, op); });
}

int phi_mgrit_points(phi_mgrit* g, int level, int which, int k0, int count, double* ptr, int device_ptr, int set) {
    return guarded([&] { g->g->points(level, which, k0, count, ptr, device_ptr != 0, set != 0); });
}

int phi_mgrit_stats(const phi_mgrit* g, long long* out4) {
    return guarded([&] { g->g->stats(out4); });
}

int phi_mgrit_set_init_coeffs(phi_mgrit* g, const double* coeffs) {
    return guarded([&] { g->g->set_init_coeffs(coeffs); });
}

int phi_mgrit_profile(phi_mgrit* g, int enable) {
    return guarded([&] {
        g->g->profile = enable != 0;
        if (g->g->profile && g->g->wstats.size() == 0) {
            g->g->wstats.alloc(3 * 8192);
            g->g->wstats.zero(g->g->stream);
        }
    });
}

int phi_mgrit_wave_levels(phi_mgrit* g, double* ms, long long* points, long long* cycles, long long* chain_steps,
                          int cap) {
    return guarded([&] {
        g->g->wave_levels(ms, points, cycles, cap);
        for (int l = 0; l < cap; ++l)
            chain_steps[l] = l < g->g->n_levels() ? g->g->levels[l].stepper->hier->chain_steps() : 0;
    });
}

int phi_mgrit_wave_report(phi_mgrit* g, double* ms, double* bytes) {
    int n = 0;
    const int rc = guarded([&] { n = g->g->wave_report(ms, bytes); });
    return rc == PHI_OK ? n : -rc;
}

int phi_dev_tuning(int tri_warps, int gs_warps, int sleep_ns) {
    return guarded([&] { phi_set_tuning(tri_warps, gs_warps, sleep_ns); });
}

int phi_dev_trace(long long* out, int n) { return phi_read_trace(out, n); }

struct phi_comm {
    std::unique_ptr<Comm> c;
};

int phi_comm_nccl_unique_id(unsigned char* id128) {
    return guarded([&] {
        const NcclUniqueId id = nccl_unique_id();
        std::memcpy(id128, id.internal, sizeof id.internal);
    });
}

int phi_comm_create_nccl(const unsigned char* id128, int nranks, int rank, phi_comm** out) {
    return guarded([&] {
        NcclUniqueId id;
        std::memcpy(id.internal, id128, sizeof id.internal);
        auto* c = new phi_comm;
        c->c = make_nccl_comm(id, nranks, rank);
        *out = c;
    });
}

int phi_comm_create_ops(const phi_comm_ops* ops, int nranks, int rank, phi_comm** out) {
    return guarded([&] {
        if (!ops) throw InvalidArgument("phi_comm_ops: null");
        auto* c = new phi_comm;
        c->c = make_ops_comm(CommOps{ops->ctx, ops->shift, ops->allgather}, nranks, rank);
        *out = c;
    });
}

void phi_comm_free(phi_comm* c) { delete c; }

int phi_mgrit_set_comm(phi_mgrit* g, phi_comm* c) {
    return guarded([&] { g->g->set_comm(c ? c->c.get() : nullptr); });
}

int phi_setup_tables_1d(int degree, int n_elements, int nq, double* nodes, double* weights, double* vals,
                        double* ders, int* first) {
    return guarded([&] {
        if (degree > 30) throw InvalidArgument("phi_setup_tables_1d: degree must be <= 30");
        const Tables1D tb = build_tables(open_uniform_knots(degree, n_elements), nq);
        std::copy(tb.nodes.begin(), tb.nodes.end(), nodes);
        std::copy(tb.weights.begin(), tb.weights.end(), weights);
        std::copy(tb.vals.begin(), tb.vals.end(), vals);
        std::copy(tb.ders.begin(), tb.ders.end(), ders);
        std::copy(tb.first.begin(), tb.first.end(), first);
    });
}

int phi_setup_dense_lu(int n, const double* a, double* lu, int* piv) {
    return guarded([&] {
        if (n < 0) throw InvalidArgument("phi_setup_dense_lu: n must be >= 0");
        HostCsr m;
        m.n_rows = m.n_cols = n;
        m.row_offsets.assign(1, 0);
        for (int i = 0; i < n; ++i) {
            for (int j = 0; j < n; ++j) {
                const double v = a[static_cast<size_t>(i) * n + j];
                if (v == 0.0) continue;
                m.col_indices.push_back(j);
                m.values.push_back(v);
            }
            m.row_offsets.push_back(m.nnz());
        }
        const DenseLUHost f = dense_lu_factor(m);
        std::copy(f.lu.begin(), f.lu.end(), lu);
        std::copy(f.piv.begin(), f.piv.end(), piv);
    });
}

int phi_setup_level_steps(int nt, int m, int cycle, int coarse_floor, int* steps, int cap, int* n_levels) {
    return guarded([&] {
        const std::vector<int> s = mgrit_level_steps(nt, m, cycle, coarse_floor);
        for (int l = 0; l < static_cast<int>(s.size()) && l < cap; ++l) steps[l] = s[l];
        *n_levels = static_cast<int>(s.size());
    });
}


}  // extern "C"
