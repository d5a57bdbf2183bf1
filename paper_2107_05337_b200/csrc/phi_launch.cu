// Host launchers of the Phi kernels: shared-memory plan, per-degree dispatch
// to the DegLaunch instantiations (phi_deg.cu) and the small elementwise
// MGRIT helpers.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "device_types.cuh"
#include "phi_kernels.cuh"

namespace phi {

namespace {

constexpr int kDotChunk = 2048;  // doubles of shared scratch for ordered dots

// ---- small elementwise MGRIT helpers --------------------------------------
// coarse.g[0] = fine.g[0] - fine.u[0]; coarse.u[0] = coarse.g[0]  (mgrit.hpp:155-166)
__global__ void restrict_first_kernel(const double* fg, const double* fu, double* cg, double* cu, int n) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const double v = fg[i] - fu[i];
        cg[i] = v;
        cu[i] = v;
    }
}

// fine.u[j*m] += coarse.u[j], j = j0..j1-1  (mgrit.hpp:172-180)
__global__ void inject_kernel(const double* cu, double* fu, int n, int j0, int j1, int m) {
    const size_t total = (size_t)(j1 - j0) * n;
    for (size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x; t < total; t += (size_t)gridDim.x * blockDim.x) {
        const size_t j = j0 + t / n, i = t % n;
        double* dst = fu + j * m * (size_t)n + i;
        *dst = *dst + cu[j * n + i];
    }
}

// sq[0] = |g[0] - u[0]|^2, index-ordered  (mgrit.hpp:202-203)
__global__ void resid0_kernel(const double* g, const double* u, double* sq, int n) {
    __shared__ double sh[4];
    __shared__ double scratch[kDotChunk];
    double s = 0.0;
    for (int c0 = 0; c0 < n; c0 += kDotChunk) {
        const int cnt = min(kDotChunk, n - c0);
        __syncthreads();
        for (int i = threadIdx.x; i < cnt; i += blockDim.x) {
            const double r = g[c0 + i] - u[c0 + i];
            scratch[i] = r * r;
        }
        __syncthreads();
        if (threadIdx.x == 0)
            for (int i = 0; i < cnt; ++i) s = s + scratch[i];
    }
    if (threadIdx.x == 0) sq[0] = s;
    (void)sh;
}

// Reads a buffer larger than L2 (an L2 flush that leaves only clean lines,
// so the timed kernel does not pay for write-backs); the sum is stored only
// under a condition that never holds for finite data.
__global__ void l2_flush_read_kernel(const double2* __restrict__ buf, size_t n2, double* sink) {
    double s = 0.0;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n2; i += (size_t)gridDim.x * blockDim.x) {
        const double2 v = __ldg(buf + i);
        s += v.x + v.y;
    }
    if (s != s) sink[0] = s;  // NaN only
}

__global__ void copy_kernel(double* dst, const double* src, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        dst[i] = src[i];
}

}  // namespace

// ---------------------------------------------------------------------------
// host launchers
// ---------------------------------------------------------------------------
size_t phi_ws_doubles(const DevHier& H) {
    size_t s = 6 * ((size_t)H.n_p + 2);
    for (int l = 0; l < H.n_h; ++l) s += 3 * (size_t)H.h[l].n + 1;
    return (s + 31) & ~size_t(31);
}

SmemPlan phi_smem_plan(const DevHier& H) {
    // Shared memory of one Phi CTA, by V-cycle phase:
    //   [0, tri)        TMA ring of the sweeps (ILUT factors and Gauss-Seidel)
    //                   + the exact mode's product scratch; the ordered-dot
    //                   scratch overlays it (norm phases)
    //   [tri, total)    the ILUT dependency vector z (smoothing) overlaid by
    //                   the order-1 h-level vectors b, x, r (W-cycle)
    // Block sweeps (reassociated mode) size the ring per phase: the smoothing
    // ring holds ILUT blocks in front of z, the W-cycle ring the (smaller)
    // Gauss-Seidel blocks in front of the h-level vectors.
    SmemPlan P{};
    const size_t budget = kPhiSmemBudgetBytes / 8;  // doubles
    P.ring_off = 0;
    P.dot_off = 0;
    P.win_off = -1;
    for (int l = 0; l < kMaxH; ++l) P.lvl_off[l] = -1;
    if (H.kind == 1) {  // CG kind: the ordered-dot scratch only (vectors in global memory)
        P.prod_off = P.z_off = P.cl_scr_off = -1;
        P.total = kDotChunk;
        return P;
    }
    size_t tri, gs_tri;
    if (H.exact) {
        int slot = std::max(H.L.max_unit_bytes, H.U.max_unit_bytes);
        for (int l = 0; l + 1 < H.n_h; ++l)
            slot = std::max(slot, std::max(H.h[l].gs_fwd.max_unit_bytes, H.h[l].gs_bwd.max_unit_bytes));
        P.slot_bytes = P.gs_slot_bytes = (slot + 127) / 128 * 128;
        P.n_slots = P.gs_n_slots = kTriSlots;
        tri = (size_t)kTriSlots * P.slot_bytes / 8;
        P.prod_off = (int)tri;
        tri += kTriMaxItems;
        gs_tri = tri;
        if (tri * 8 > kPhiSmemBudgetBytes) throw InvalidArgument("triangular-factor blocks exceed shared memory");
    } else {
        P.prod_off = -1;
        const int slot = std::max(H.Lb.max_unit_bytes, H.Ub.max_unit_bytes);
        int gslot = 16;
        for (int l = 0; l + 1 < H.n_h; ++l)
            gslot = std::max(gslot, std::max(H.h[l].gsb_fwd.max_unit_bytes, H.h[l].gsb_bwd.max_unit_bytes));
        P.slot_bytes = (slot + 127) / 128 * 128;
        P.gs_slot_bytes = (gslot + 127) / 128 * 128;
        const int min_slots = kBlkMinSlots;
        // the ILUT ring leaves room for z (or, rolling-window streams, for the window) when it can
        const int win = std::max(H.Lb.win, H.Ub.win);
        const size_t zb = win ? ((size_t)win + 2) * 8 : ((size_t)H.n_p + 2) * 8;
        int ns = (int)std::min<size_t>(kBlkMaxSlots, (kPhiSmemBudgetBytes - std::min(zb, kPhiSmemBudgetBytes)) / P.slot_bytes);
        if (win && ns < min_slots) throw InvalidArgument("rolling-window ILUT streams exceed shared memory");
        if (ns < min_slots) ns = (int)std::min<size_t>(kBlkMaxSlots, kPhiSmemBudgetBytes / P.slot_bytes);
        if (ns < min_slots) throw InvalidArgument("triangular-factor blocks exceed shared memory");
        P.n_slots = ns;
        tri = (size_t)ns * P.slot_bytes / 8;
        P.gs_n_slots = std::min(kBlkMaxSlots, 6);
        gs_tri = (size_t)P.gs_n_slots * P.gs_slot_bytes / 8;
    }
    size_t top = std::max(tri, gs_tri);
    if (!H.exact && std::max(H.Lb.win, H.Ub.win) > 0) {  // z global, its window after the ring
        P.z_off = -1;
        P.win_off = (int)tri;
        top = std::max(top, tri + std::max(H.Lb.win, H.Ub.win) + 2);
    } else if (tri + (size_t)H.n_p + 2 <= budget) {
        P.z_off = (int)tri;
        top = std::max(top, tri + H.n_p + 2);
    } else {
        P.z_off = -1;
    }
    // coarsest levels first: they are visited most often by the W-cycle
    size_t lv = gs_tri;
    for (int l = H.n_h - 1; l >= 0; --l) {
        const size_t need = 3 * (size_t)H.h[l].n + 1;
        if (lv + need <= budget) {
            P.lvl_off[l] = (int)lv;
            lv += need;
        }
    }
    top = std::max(top, lv);
    // scratch of the cluster dense coarse product (W-cycle phase): the sweep
    // ring below the level vectors if it is large enough, else above them
    if (gs_tri >= (size_t)kClScratch)
        P.cl_scr_off = 0;
    else if (lv + kClScratch <= budget)
        P.cl_scr_off = (int)lv, top = std::max(top, lv + kClScratch);
    else
        P.cl_scr_off = -1;
    P.total = (int)std::max(top, (size_t)kDotChunk);
    if (std::getenv("PHI_PLAN_DEBUG"))
        std::fprintf(stderr, "smem plan: slot %d B x %d, gs slot %d B x %d, prod @%d, z @%d, window @%d, levels @%d.., total %d doubles\n",
                     P.slot_bytes, P.n_slots, P.gs_slot_bytes, P.gs_n_slots, P.prod_off, P.z_off, P.win_off, P.lvl_off[0], P.total);
    return P;
}

size_t phi_smem_bytes(const DevHier& H) { return (size_t)phi_smem_plan(H).total * 8; }

// Kernels are instantiated per spline degree (compile-time stencil widths).
#define PHI_DEG_DISPATCH(deg, ...)                                                   \
    switch (deg) {                                                                    \
        case 1: { constexpr int DEG = 1; __VA_ARGS__; } break;                               \
        case 2: { constexpr int DEG = 2; __VA_ARGS__; } break;                               \
        case 3: { constexpr int DEG = 3; __VA_ARGS__; } break;                               \
        case 4: { constexpr int DEG = 4; __VA_ARGS__; } break;                               \
        case 5: { constexpr int DEG = 5; __VA_ARGS__; } break;                               \
        case 6: { constexpr int DEG = 6; __VA_ARGS__; } break;                               \
        case 7: { constexpr int DEG = 7; __VA_ARGS__; } break;                               \
        case 8: { constexpr int DEG = 8; __VA_ARGS__; } break;                               \
        default: throw InvalidArgument("unsupported spline degree");                  \
    }

static int degree_of(const DevStencil& A) { return (A.hi - A.lo) / 2; }

int phi_max_slots(const DevHier& H) {
    int r = 1;
    PHI_DEG_DISPATCH(degree_of(H.A), r = DegLaunch<DEG>::max_slots(H));
    return r;
}

void launch_phi_wave(const DevHier& H, const DevStencil& Am, const WaveArgs& a, double* ws, long long ws_stride,
                     int max_slots, cudaStream_t s) {
    if (a.n_tasks <= 0) return;
    const int grid = std::min(a.n_tasks, max_slots);
    PHI_DEG_DISPATCH(degree_of(H.A), DegLaunch<DEG>::wave(H, Am, a, ws, ws_stride, grid, s));
}

void launch_vcycle(const DevHier& H, const double* B, long long ldb, double* X, long long ldx, int nrhs, double* ws,
                   long long ws_stride, int max_slots, cudaStream_t s) {
    if (nrhs <= 0) return;
    const int grid = std::min(nrhs, max_slots);
    PHI_DEG_DISPATCH(degree_of(H.A), DegLaunch<DEG>::vcycle(H, B, ldb, X, ldx, nrhs, ws, ws_stride, grid, s));
}

void launch_unit(const DevHier& H, int op, int arg, int arg2, const double* in, double* out, double* ws,
                 long long ws_stride, cudaStream_t s) {
    PHI_DEG_DISPATCH(degree_of(H.A), DegLaunch<DEG>::unit(H, op, arg, arg2, in, out, ws, ws_stride, s));
}

void launch_cg(const DevStencil& A, const double* diag, const double* b, double* x, double* work, double rel_tol,
               int max_iter, int* result, int exact, cudaStream_t s) {
    PHI_DEG_DISPATCH(degree_of(A), DegLaunch<DEG>::cg(A, diag, b, x, work, rel_tol, max_iter, result, exact, s));
}

static DevBuf<long long> g_trace;

void phi_set_tuning(int tri_warps, int gs_warps, int sleep_ns) {

    (void)gs_warps;
    long long* trace = nullptr;
    if (sleep_ns < 0) {  // negative: enable the developer timing trace
        g_trace.alloc(kTraceLongs);
        g_trace.zero();
        trace = g_trace.get();
    }
    for (int d = 1; d <= 8; ++d) PHI_DEG_DISPATCH(d, DegLaunch<DEG>::set_trace(trace, tri_warps < 0 ? -tri_warps : 0));
}

int phi_read_trace(long long* out, int n) {
    if (!g_trace.get()) return 0;
    const auto h = g_trace.download();
    const int m = std::min<int>(n, (int)h.size());
    std::copy(h.begin(), h.begin() + m, out);
    return m;
}

void preload_overlap_kernels(const DevHier& H) {
    cudaFuncAttributes fa;
    PHI_CUDA(cudaFuncGetAttributes(&fa, inject_kernel));
    PHI_CUDA(cudaFuncGetAttributes(&fa, resid0_kernel));
    PHI_CUDA(cudaFuncGetAttributes(&fa, copy_kernel));
    PHI_DEG_DISPATCH(degree_of(H.A), DegLaunch<DEG>::preload_side(H));
}

void launch_restrict_first(const double* fg, const double* fu, double* cg, double* cu, int n, cudaStream_t s) {
    restrict_first_kernel<<<(n + 255) / 256, 256, 0, s>>>(fg, fu, cg, cu, n);
    PHI_CUDA(cudaGetLastError());
}

void launch_inject(const double* cu, double* fu, int n, int J, int m, cudaStream_t s) {
    launch_inject_range(cu, fu, n, 0, J + 1, m, s);
}

void launch_inject_range(const double* cu, double* fu, int n, int j0, int j1, int m, cudaStream_t s) {
    if (j1 <= j0) return;
    const size_t total = (size_t)(j1 - j0) * n;
    const int grid = (int)std::min<size_t>((total + 255) / 256, 4096);
    inject_kernel<<<grid, 256, 0, s>>>(cu, fu, n, j0, j1, m);
    PHI_CUDA(cudaGetLastError());
}

void launch_resid0(const double* g, const double* u, double* sq, int n, cudaStream_t s) {
    resid0_kernel<<<1, 256, 0, s>>>(g, u, sq, n);
    PHI_CUDA(cudaGetLastError());
}

void launch_l2_flush_read(const double* buf, size_t n, double* sink, cudaStream_t s) {
    l2_flush_read_kernel<<<148 * 8, 256, 0, s>>>(reinterpret_cast<const double2*>(buf), n / 2, sink);
    PHI_CUDA(cudaGetLastError());
}

void launch_copy(double* dst, const double* src, size_t n, cudaStream_t s) {
    if (!n) return;
    const int grid = (int)std::min<size_t>((n + 255) / 256, 4096);
    copy_kernel<<<grid, 256, 0, s>>>(dst, src, n);
    PHI_CUDA(cudaGetLastError());
}

}  // namespace phi
