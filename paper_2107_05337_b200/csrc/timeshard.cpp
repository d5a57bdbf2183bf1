// Time-sharded MGRIT in the C++ host: one rank per
// GPU owns a contiguous block of the level-0 coarse intervals; operators and
// the coarser levels are replicated.  Per MGRIT iteration (mgrit.hpp:93-118,
// 278-288):
//   F / FC relaxation  local; the first owned interval starts from the C-point
//                      u[j0 m] that rank r-1 owns: a halo shift (one n-vector,
//                      r-1 -> r) precedes every relaxation sweep;
//   restriction        local; every rank then gathers all coarse right-hand
//                      sides (an allgather of the owned points only, padded to
//                      the largest share, in rank = point order);
//   coarse cycle       replicated; the F-schedule's second pass runs its
//                      coarse cycle without the schedule (cycle_impl(l, false));
//   correction         injection (replicated), then local F-relaxation;
//   residual / g-norm  per-point squared terms of the owned points, gathered
//                      in point order and summed sequentially on every rank:
//                      the single-process sum (mgrit.hpp:209-212, 306).
// With identical inputs the sharded solve performs the same floating-point
// operations as the single-process solve: identical results for any rank count.
//
// Transports (Comm): NCCL (send/recv + allgather on the engine stream, the
// library resolved at run time so the process shares whatever libnccl.so.2 is
// loaded already), or host callbacks (phi_comm_ops: tests, other fabrics).
#include <dlfcn.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "engine.hpp"
#include "timeshard.hpp"

namespace phi {

// ---------------------------------------------------------------------------
// NCCL, resolved at run time
// ---------------------------------------------------------------------------
namespace {

using nccl_result = int;
struct NcclApi {
    void* so = nullptr;
    nccl_result (*get_unique_id)(void*) = nullptr;
    nccl_result (*comm_init_rank)(void**, int, NcclUniqueId, int) = nullptr;
    nccl_result (*comm_destroy)(void*) = nullptr;
    nccl_result (*send)(const void*, size_t, int, int, void*, cudaStream_t) = nullptr;
    nccl_result (*recv)(void*, size_t, int, int, void*, cudaStream_t) = nullptr;
    nccl_result (*all_gather)(const void*, void*, size_t, int, void*, cudaStream_t) = nullptr;
    nccl_result (*group_start)() = nullptr;
    nccl_result (*group_end)() = nullptr;
    const char* (*error_string)(nccl_result) = nullptr;
};
constexpr int kNcclFloat64 = 8;  // ncclDouble (nccl.h)

const NcclApi& nccl() {
    static NcclApi api;
    static bool tried = false;
    if (!tried) {
        tried = true;
        api.so = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (api.so) {
            auto sym = [&](const char* n) { return dlsym(api.so, n); };
            api.get_unique_id = reinterpret_cast<decltype(api.get_unique_id)>(sym("ncclGetUniqueId"));
            api.comm_init_rank = reinterpret_cast<decltype(api.comm_init_rank)>(sym("ncclCommInitRank"));
            api.comm_destroy = reinterpret_cast<decltype(api.comm_destroy)>(sym("ncclCommDestroy"));
            api.send = reinterpret_cast<decltype(api.send)>(sym("ncclSend"));
            api.recv = reinterpret_cast<decltype(api.recv)>(sym("ncclRecv"));
            api.all_gather = reinterpret_cast<decltype(api.all_gather)>(sym("ncclAllGather"));
            api.group_start = reinterpret_cast<decltype(api.group_start)>(sym("ncclGroupStart"));
            api.group_end = reinterpret_cast<decltype(api.group_end)>(sym("ncclGroupEnd"));
            api.error_string = reinterpret_cast<decltype(api.error_string)>(sym("ncclGetErrorString"));
        }
    }
    if (!api.so || !api.comm_init_rank || !api.all_gather || !api.send)
        throw CudaError("NCCL unavailable: libnccl.so.2 could not be loaded");
    return api;
}

void nccl_check(nccl_result r, const char* what) {
    if (r != 0) {
        const char* msg = nccl().error_string ? nccl().error_string(r) : "?";
        throw CudaError(std::string("NCCL error in ") + what + ": " + msg);
    }
}

class NcclComm : public Comm {
public:
    NcclComm(const NcclUniqueId& id, int nranks, int r) {
        rank = r;
        size = nranks;
        nccl_check(nccl().comm_init_rank(&comm_, nranks, id, r), "ncclCommInitRank");
    }
    ~NcclComm() override {
        if (comm_) nccl().comm_destroy(comm_);
    }
    void shift(const double* send, double* recv, size_t count, cudaStream_t s) override {
        const NcclApi& a = nccl();
        nccl_check(a.group_start(), "ncclGroupStart");
        if (send && rank + 1 < size) nccl_check(a.send(send, count, kNcclFloat64, rank + 1, comm_, s), "ncclSend");
        if (recv && rank > 0) nccl_check(a.recv(recv, count, kNcclFloat64, rank - 1, comm_, s), "ncclRecv");
        nccl_check(a.group_end(), "ncclGroupEnd");
    }
    void allgather(const double* send, double* recv, size_t count, cudaStream_t s) override {
        nccl_check(nccl().all_gather(send, recv, count, kNcclFloat64, comm_, s), "ncclAllGather");
    }

private:
    void* comm_ = nullptr;
};

// Host-callback transport: device data staged through host buffers.
class OpsComm : public Comm {
public:
    OpsComm(const CommOps& ops, int nranks, int r) : ops_(ops) {
        rank = r;
        size = nranks;
    }
    void shift(const double* send, double* recv, size_t count, cudaStream_t s) override {
        std::vector<double> hs(send && rank + 1 < size ? count : 0), hr(recv && rank > 0 ? count : 0);
        if (!hs.empty()) PHI_CUDA(cudaMemcpyAsync(hs.data(), send, 8 * count, cudaMemcpyDeviceToHost, s));
        PHI_CUDA(cudaStreamSynchronize(s));
        if (ops_.shift(ops_.ctx, hs.empty() ? nullptr : hs.data(), hr.empty() ? nullptr : hr.data(),
                       (long long)count))
            throw CudaError("phi_comm_ops.shift failed");
        if (!hr.empty()) {
            PHI_CUDA(cudaMemcpyAsync(recv, hr.data(), 8 * count, cudaMemcpyHostToDevice, s));
            PHI_CUDA(cudaStreamSynchronize(s));
        }
    }
    void allgather(const double* send, double* recv, size_t count, cudaStream_t s) override {
        std::vector<double> hs(count), hr(count * size);
        PHI_CUDA(cudaMemcpyAsync(hs.data(), send, 8 * count, cudaMemcpyDeviceToHost, s));
        PHI_CUDA(cudaStreamSynchronize(s));
        if (ops_.allgather(ops_.ctx, hs.data(), hr.data(), (long long)count))
            throw CudaError("phi_comm_ops.allgather failed");
        PHI_CUDA(cudaMemcpyAsync(recv, hr.data(), 8 * count * size, cudaMemcpyHostToDevice, s));
        PHI_CUDA(cudaStreamSynchronize(s));
    }

private:
    CommOps ops_;
};

}  // namespace

NcclUniqueId nccl_unique_id() {
    NcclUniqueId id{};
    nccl_check(nccl().get_unique_id(&id), "ncclGetUniqueId");
    return id;
}

std::unique_ptr<Comm> make_nccl_comm(const NcclUniqueId& id, int nranks, int rank) {
    if (nranks < 1 || rank < 0 || rank >= nranks) throw InvalidArgument("phi_comm: rank out of range");
    return std::make_unique<NcclComm>(id, nranks, rank);
}

std::unique_ptr<Comm> make_ops_comm(const CommOps& ops, int nranks, int rank) {
    if (nranks < 1 || rank < 0 || rank >= nranks) throw InvalidArgument("phi_comm: rank out of range");
    if (!ops.shift || !ops.allgather) throw InvalidArgument("phi_comm_ops: missing callback");
    return std::make_unique<OpsComm>(ops, nranks, rank);
}

// ---------------------------------------------------------------------------
// the sharded solve
// ---------------------------------------------------------------------------
std::pair<int, int> shard_of(int n_intervals, int n_ranks, int rank) {
    const int base = n_intervals / n_ranks, extra = n_intervals % n_ranks;
    const int j0 = rank * base + std::min(rank, extra);
    return {j0, j0 + base + (rank < extra ? 1 : 0)};
}

namespace {

// Sum of per-point terms over the ranks, in point order: each rank owns the
// terms [k_lo(r), k_hi(r)) of one contiguous range; allgather of the padded
// owned segments, then the sequential sum on every rank.
double ordered_sum(Comm& c, const std::vector<double>& terms, const std::vector<std::pair<int, int>>& owned,
                   cudaStream_t s) {
    size_t width = 0;
    for (auto [a, b] : owned) width = std::max(width, (size_t)(b - a));
    width = std::max<size_t>(width, 1);
    const auto [lo, hi] = owned[c.rank];
    std::vector<double> mine(width, 0.0);
    std::copy(terms.begin() + lo, terms.begin() + hi, mine.begin());
    DevBuf<double> d_mine(width), d_all(width * c.size);
    d_mine.upload(mine, s);
    c.allgather(d_mine.get(), d_all.get(), width, s);
    const std::vector<double> all = d_all.download(s);
    double total = 0.0;
    for (int r = 0; r < c.size; ++r)
        for (int k = 0; k < owned[r].second - owned[r].first; ++k) total += all[r * width + k];
    return total;
}

}  // namespace

void Mgrit::set_comm(Comm* c) {
    comm = c;
    if (!c) {
        set_range(0, -1);
        return;
    }
    if (levels.size() < 2) throw InvalidArgument("time sharding needs at least two MGRIT levels");
    const int J = levels[0].steps / cfg.m;
    if (c->size > J) throw InvalidArgument("time sharding: more ranks than coarse intervals");
    const auto [a, b] = shard_of(J, c->size, c->rank);
    set_range(a, b);
}

void Mgrit::halo() {
    const int n = disc->n_p, m = cfg.m;
    Level& lv = levels[0];
    double* send = comm->rank + 1 < comm->size ? lv.u.get() + (size_t)j_hi * m * n : nullptr;
    double* recv = comm->rank > 0 ? lv.u.get() + (size_t)j_lo * m * n : nullptr;
    comm->shift(send, recv, n, stream);
}

void Mgrit::combine_coarse_rhs() {
    const int n = disc->n_p, J = levels[0].steps / cfg.m, R = comm->size;
    std::vector<std::pair<int, int>> shares(R);
    int width = 1;
    for (int r = 0; r < R; ++r) {
        shares[r] = shard_of(J, R, r);
        width = std::max(width, shares[r].second - shares[r].first);
    }
    Level& c = levels[1];
    DevBuf<double> mine((size_t)width * n), all((size_t)width * n * R);
    mine.zero(stream);
    const int own = j_hi - j_lo;
    if (own) launch_copy(mine.get(), c.g.get() + (size_t)(j_lo + 1) * n, (size_t)own * n, stream);
    comm->allgather(mine.get(), all.get(), (size_t)width * n, stream);
    for (int r = 0; r < R; ++r) {
        const int cnt = shares[r].second - shares[r].first;
        if (cnt)
            launch_copy(c.g.get() + (size_t)(shares[r].first + 1) * n, all.get() + (size_t)r * width * n,
                        (size_t)cnt * n, stream);
    }
    launches += 1 + R;
    // the restriction zeroes the coarse iterate at every restricted point
    PHI_CUDA(cudaMemsetAsync(c.u.get() + n, 0, sizeof(double) * (size_t)J * n, stream));
    PHI_CUDA(cudaStreamSynchronize(stream));  // `mine` / `all` go out of scope
}

std::vector<std::pair<int, int>> Mgrit::owned_points(int l) const {
    // point ranges of the residual / g-norm terms per rank (residual_terms)
    const int R = comm->size, J = levels[l].steps / cfg.m;
    std::vector<std::pair<int, int>> out(R);
    for (int r = 0; r < R; ++r) {
        const auto [a, b] = shard_of(J, R, r);
        const int k0 = a == 0 ? 0 : a * cfg.m + 1;
        const int k1 = b == J ? levels[l].steps : b * cfg.m;
        out[r] = {k0, k1 + 1};
    }
    return out;
}

void Mgrit::cycle0_sharded(bool f_schedule) {
    halo();
    if (cfg.relax == 1) {
        f_relax(0, true);
        halo();
    }
    f_relax(0, false);
    restrict_residual(0);
    combine_coarse_rhs();
    cycle_impl(1, f_schedule);  // replicated coarse cycle
    Level& f = levels[0];
    launch_inject(levels[1].u.get(), f.u.get(), disc->n_p, f.steps / cfg.m, cfg.m, stream);
    ++launches;
    halo();
    f_relax(0, false);
    if (f_schedule && n_levels() > 2) cycle0_sharded(false);
}

MgritResultHost Mgrit::solve_sharded() {
    launches = 0;
    traj_gathered = false;
    initialize_state();
    const auto own0 = owned_points(0);
    std::vector<double> t(levels[0].steps + 1);
    gnorm_terms(t.data());
    g_norm = std::sqrt(ordered_sum(*comm, t, own0, stream));
    MgritResultHost res;
    res.g_norm = g_norm;
    const double denom = g_norm > 0.0 ? g_norm : 1.0;
    for (int it = 1; it <= cfg.max_iter; ++it) {
        cycle0_sharded(cfg.cycle == 1);
        halo();
        residual_terms(0, t.data());
        const double rel = std::sqrt(ordered_sum(*comm, t, own0, stream)) / denom;
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
    // level-0 work is split over the ranks, the coarse work replicated
    std::vector<double> mine{(double)st[0], (double)st[1]};
    DevBuf<double> d_mine(2), d_all(2 * (size_t)comm->size);
    d_mine.upload(mine, stream);
    comm->allgather(d_mine.get(), d_all.get(), 2, stream);
    const std::vector<double> all = d_all.download(stream);
    long long s0 = 0, i0 = 0;
    for (int r = 0; r < comm->size; ++r) {
        s0 += (long long)all[2 * r];
        i0 += (long long)all[2 * r + 1];
    }
    res.total_spatial_solves = s0 + st[2];
    res.mean_spatial_iterations = res.total_spatial_solves > 0
                                      ? (double)(i0 + st[3]) / (double)res.total_spatial_solves
                                      : 0.0;
    return res;
}

void Mgrit::gather_trajectory() {
    if (!comm || traj_gathered) return;
    const int n = disc->n_p, m = cfg.m, R = comm->size;
    Level& lv = levels[0];
    const auto own = owned_points(0);  // [k0, k1] of every rank, as for the terms
    int width = 1;
    for (auto [a, b] : own) width = std::max(width, b - a);
    DevBuf<double> mine((size_t)width * n), all((size_t)width * n * R);
    mine.zero(stream);
    const auto [a, b] = own[comm->rank];
    launch_copy(mine.get(), lv.u.get() + (size_t)a * n, (size_t)(b - a) * n, stream);
    comm->allgather(mine.get(), all.get(), (size_t)width * n, stream);
    for (int r = 0; r < R; ++r)
        launch_copy(lv.u.get() + (size_t)own[r].first * n, all.get() + (size_t)r * width * n,
                    (size_t)(own[r].second - own[r].first) * n, stream);
    PHI_CUDA(cudaStreamSynchronize(stream));
    (void)m;
    traj_gathered = true;
}

}  // namespace phi
