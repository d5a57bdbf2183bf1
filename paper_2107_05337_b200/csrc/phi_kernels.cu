// The batched time-stepping operator Phi on B200 (sm_100a).
//
// Design: one CTA owns one right-hand side at a time and
// runs the WHOLE p-multigrid solve of theta.hpp:132-137 / pmultigrid.hpp:271-307
// for it -- right-hand-side product, residual checks, V(1,1) cycles with the
// ILUT smoother, the p->1 transfers and the order-1 h-multigrid W-cycle --
// without leaving the kernel.  Different right-hand sides (the concurrent MGRIT
// intervals, mgrit.hpp:122-141) are independent CTAs, so a wave needs no grid
// synchronisation and no host round trip.  Every reduction that the reference
// performs in index order (spmv, the triangular solves, Gauss-Seidel, dot /
// norm2) is performed here in the same order by one thread, without fused
// multiply-adds (-fmad=false), so on identical operators the result is
// bit-identical to the reference.
//
// Sync-free triangular solves: rows are processed level by level (levels from
// the host schedule, setup_host.cpp), warp w owning levels w, w+8, ...; a row
// waits only for the entries it actually reads.  Solved values are published
// with a single 64-bit store into a "sentinel" array (a signalling-NaN bit
// pattern marks "not yet solved"), so the readiness flag and the value are the
// same word: one shared-memory load per dependency, no fences.
#include <cuda_runtime.h>

#include <algorithm>

#include "device_types.cuh"
#include "phi_kernels.cuh"

namespace phi {

namespace {

constexpr int NT = kPhiThreads;
constexpr int NW = NT / 32;
constexpr unsigned long long kSentinel = 0x7FF4DEADBEEF0001ULL;

// ---------------------------------------------------------------------------
// dependency stores for the sync-free triangular solves
// ---------------------------------------------------------------------------
struct ZSmem {
    double* z;
    __device__ __forceinline__ double wait(int j) const {
        unsigned long long b;
        do {
            b = *reinterpret_cast<volatile unsigned long long*>(z + j);
        } while (b == kSentinel);
        return __longlong_as_double(static_cast<long long>(b));
    }
    __device__ __forceinline__ void put(int i, double v) const {
        *reinterpret_cast<volatile double*>(z + i) = v;
    }
    __device__ __forceinline__ void reset(int n) const {
        for (int i = threadIdx.x; i < n; i += NT)
            reinterpret_cast<unsigned long long*>(z)[i] = kSentinel;
    }
};

struct ZGlobal {
    double* z;
    __device__ __forceinline__ double wait(int j) const {
        unsigned long long b;
        do {
            asm volatile("ld.relaxed.cta.global.u64 %0, [%1];" : "=l"(b) : "l"(z + j) : "memory");
        } while (b == kSentinel);
        return __longlong_as_double(static_cast<long long>(b));
    }
    __device__ __forceinline__ void put(int i, double v) const {
        asm volatile("st.relaxed.cta.global.f64 [%0], %1;" ::"l"(z + i), "d"(v) : "memory");
    }
    __device__ __forceinline__ void reset(int n) const {
        for (int i = threadIdx.x; i < n; i += NT)
            reinterpret_cast<unsigned long long*>(z)[i] = kSentinel;
    }
};

// ---------------------------------------------------------------------------
// per-CTA workspace
// ---------------------------------------------------------------------------
struct Ws {
    double *b, *x, *r, *zg;
    double* hb[kMaxH];
    double* hx[kMaxH];
    double* hr[kMaxH];
};

__device__ Ws carve(double* base, const DevHier& H) {
    Ws w;
    const int n = H.n_p;
    w.b = base;
    w.x = base + n;
    w.r = base + 2 * (size_t)n;
    w.zg = base + 3 * (size_t)n;
    double* p = base + 4 * (size_t)n;
    for (int l = 0; l < H.n_h; ++l) {
        const int nl = H.h[l].n;
        w.hb[l] = p;
        w.hx[l] = p + nl;
        w.hr[l] = p + 2 * (size_t)nl;
        p += 3 * (size_t)nl;
    }
    return w;
}

// ---------------------------------------------------------------------------
// CTA-cooperative primitives.  Callers place __syncthreads() between phases.
// ---------------------------------------------------------------------------

// y[i] (op)= sum_e vals[e][i] * x[col(i, e)], entries in reference CSR order.
enum StencilOut : int { kOutSet = 0, kOutResid = 1, kOutScale = 2, kOutAddScaled = 3, kOutAddVec = 4 };

template <int OUT>
__device__ __forceinline__ void stencil_apply(const DevStencil& A, const double* __restrict__ x,
                                              double* __restrict__ y, const double* __restrict__ aux) {
    const int n = A.ru * A.rv;
    const int w = A.hi - A.lo + 1;
    for (int i = threadIdx.x; i < n; i += NT) {
        const int iv = i / A.ru;
        const int iu = i - iv * A.ru;
        const int dulo = max(A.lo, -iu), duhi = min(A.hi, A.cu - 1 - iu);
        const int dvlo = max(A.lo, -iv), dvhi = min(A.hi, A.cv - 1 - iv);
        double s = 0.0;
        for (int dv = dvlo; dv <= dvhi; ++dv) {
            const double* vr = A.vals + (size_t)((dv - A.lo) * w - A.lo) * n + i;
            const double* xr = x + (size_t)(iv + dv) * A.cu + iu;
            for (int du = dulo; du <= duhi; ++du) s = s + vr[(size_t)du * n] * xr[du];
        }
        if (OUT == kOutSet) y[i] = s;
        if (OUT == kOutResid) y[i] = aux[i] - s;         // r = b - A x
        if (OUT == kOutScale) y[i] = s * aux[i];         // (P^T r) .* 1/M^L
        if (OUT == kOutAddScaled) y[i] = y[i] + s * aux[i];  // x += (P e) .* 1/M^L
        if (OUT == kOutAddVec) y[i] = s + aux[i];        // rhs = A- u + load
    }
}

// y = A x (CSR, row order) or y += A x.
template <bool ADD>
__device__ __forceinline__ void csr_apply(const DevCsr& A, const double* __restrict__ x,
                                          double* __restrict__ y) {
    for (int i = threadIdx.x; i < A.n_rows; i += NT) {
        double s = 0.0;
        for (int e = A.ro[i]; e < A.ro[i + 1]; ++e) s = s + A.v[e] * x[A.ci[e]];
        if (ADD)
            y[i] = y[i] + s;
        else
            y[i] = s;
    }
}

// One lexicographic Gauss-Seidel sweep (solvers.hpp:80-99) executed by
// anti-diagonal wavefronts u + 2v = t: for the 9-point order-1 stencil every
// row of wavefront t reads updated values only from wavefronts < t and old
// values only from wavefronts > t, so the result equals the sequential sweep.
__device__ void gs_sweep(const DevStencil& A, const double* __restrict__ b, double* x, bool backward) {
    const int nu = A.ru, nv = A.rv, n = nu * nv;
    const int w = A.hi - A.lo + 1;
    const int T = (nu - 1) + 2 * (nv - 1);
    for (int t = 0; t <= T; ++t) {
        const int vlo = max(0, (t - (nu - 1) + 1) / 2);
        const int vhi = min(nv - 1, t / 2);
        for (int q = vlo + threadIdx.x; q <= vhi; q += NT) {
            const int u = t - 2 * q;
            const int iu = backward ? nu - 1 - u : u;
            const int iv = backward ? nv - 1 - q : q;
            const int i = iu + nu * iv;
            const int dulo = max(A.lo, -iu), duhi = min(A.hi, A.cu - 1 - iu);
            const int dvlo = max(A.lo, -iv), dvhi = min(A.hi, A.cv - 1 - iv);
            double diag = 0.0, s = b[i];
            for (int dv = dvlo; dv <= dvhi; ++dv) {
                const double* vr = A.vals + (size_t)((dv - A.lo) * w - A.lo) * n + i;
                const double* xr = x + (size_t)(iv + dv) * A.cu + iu;
                for (int du = dulo; du <= duhi; ++du) {
                    const double v = vr[(size_t)du * n];
                    if (du == 0 && dv == 0)
                        diag = v;
                    else
                        s = s - v * xr[du];
                }
            }
            x[i] = s / diag;
        }
        __syncthreads();
    }
}

// Forward substitution with the unit lower ILUT factor (ilut.hpp:150-156).
template <class Z>
__device__ void tri_lower(const DevTri& L, const double* __restrict__ r, const Z& z, double* zcopy) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int lv = warp; lv < L.n_levels; lv += NW) {
        const int c1 = L.level_chunk[lv + 1];
        for (int c = L.level_chunk[lv]; c < c1; ++c) {
            const int nr = L.chunk_nrows[c];
            if (lane < nr) {
                const int pos = L.chunk_row0[c] + lane;
                const int i = L.rows[pos];
                const int len = L.lens[pos];
                const int* cp = L.cols + L.chunk_base[c] + lane;
                const double* vp = L.vals + L.chunk_base[c] + lane;
                double s = r[i];
                for (int e = 0; e < len; ++e) {
                    const int j = __ldg(cp + e * nr);
                    const double v = __ldg(vp + e * nr);
                    s = s - v * z.wait(j);
                }
                if (zcopy) zcopy[i] = s;
                z.put(i, s);
            }
        }
    }
}

// Backward substitution with U (diagonal first, ilut.hpp:157-162), fused with
// the smoother update x += z (pmultigrid.hpp:315).
template <class Z>
__device__ void tri_upper(const DevTri& U, const double* __restrict__ zin, const Z& z, double* x) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int lv = warp; lv < U.n_levels; lv += NW) {
        const int c1 = U.level_chunk[lv + 1];
        for (int c = U.level_chunk[lv]; c < c1; ++c) {
            const int nr = U.chunk_nrows[c];
            if (lane < nr) {
                const int pos = U.chunk_row0[c] + lane;
                const int i = U.rows[pos];
                const int len = U.lens[pos];
                const int* cp = U.cols + U.chunk_base[c] + lane;
                const double* vp = U.vals + U.chunk_base[c] + lane;
                double s = zin[i];
                for (int e = 0; e < len; ++e) {
                    const int j = __ldg(cp + e * nr);
                    const double v = __ldg(vp + e * nr);
                    s = s - v * z.wait(j);
                }
                const double zi = s / U.diag[i];
                z.put(i, zi);
                x[i] = x[i] + zi;
            }
        }
    }
}

// Index-ordered dot product by a single thread (sparse.hpp:188-192); the value
// is broadcast through shared memory.  Keeps every norm bit-identical.
__device__ double cta_ordered_dot(const double* __restrict__ a, const double* __restrict__ b, int n,
                                  double* sh) {
    __syncthreads();
    if (threadIdx.x == 0) {
        double s = 0.0;
        int i = 0;
        for (; i + 8 <= n; i += 8) {
            double pa[8], pb[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                pa[k] = a[i + k];
                pb[k] = b[i + k];
            }
#pragma unroll
            for (int k = 0; k < 8; ++k) s = s + pa[k] * pb[k];
        }
        for (; i < n; ++i) s = s + a[i] * b[i];
        sh[0] = s;
    }
    __syncthreads();
    const double v = sh[0];
    __syncthreads();
    return v;
}

__device__ void cta_fill(double* y, double v, int n) {
    for (int i = threadIdx.x; i < n; i += NT) y[i] = v;
}
__device__ void cta_copy(double* y, const double* x, int n) {
    for (int i = threadIdx.x; i < n; i += NT) y[i] = x[i];
}

// Dense LU solve of the coarsest h-level (solvers.hpp:118-133), thread 0.
__device__ void coarse_solve(const DevHier& H, const double* b, double* x) {
    if (threadIdx.x == 0) {
        const int n = H.coarse_n;
        const double* lu = H.coarse_lu;
        for (int i = 0; i < n; ++i) x[i] = b[H.coarse_piv[i]];
        for (int i = 0; i < n; ++i) {
            double s = x[i];
            for (int j = 0; j < i; ++j) s = s - lu[i * n + j] * x[j];
            x[i] = s;
        }
        for (int i = n - 1; i >= 0; --i) {
            double s = x[i];
            for (int j = i + 1; j < n; ++j) s = s - lu[i * n + j] * x[j];
            x[i] = s / lu[i * n + i];
        }
    }
    __syncthreads();
}

// h-multigrid W-cycle (pmultigrid.hpp:184-200), recursion unrolled into an
// explicit per-level phase machine (no device stack):
//   phase 0: pre-smooth, restrict, first coarse visit
//   phase 1: second coarse visit (starting from the first visit's result)
//   phase 2: prolongate, post-smooth, return
__device__ void wcycle(const DevHier& H, const Ws& w, int l0) {
    int phase[kMaxH];
    int l = l0;
    phase[l] = 0;
    for (;;) {
        if (l + 1 == H.n_h) {
            coarse_solve(H, w.hb[l], w.hx[l]);
            if (l == l0) return;
            --l;
            continue;
        }
        const DevHLevel& lv = H.h[l];
        double* b = w.hb[l];
        double* x = w.hx[l];
        if (phase[l] == 0) {
            for (int s = 0; s < H.gs_pre; ++s) gs_sweep(lv.a, b, x, false);
            stencil_apply<kOutResid>(lv.a, x, w.hr[l], b);
            __syncthreads();
            csr_apply<false>(lv.embed_t, w.hr[l], w.hb[l + 1]);  // rc = E^T r
            cta_fill(w.hx[l + 1], 0.0, H.h[l + 1].n);              // ec = 0
            __syncthreads();
            phase[l] = 1;
            phase[++l] = 0;
        } else if (phase[l] == 1) {
            phase[l] = 2;
            phase[++l] = 0;
        } else {
            csr_apply<true>(lv.embed, w.hx[l + 1], x);  // x += E ec
            __syncthreads();
            for (int s = 0; s < H.gs_post; ++s) gs_sweep(lv.a, b, x, true);
            if (l == l0) return;
            --l;
        }
    }
}

// x += S (b - A x), S = ILUT application (pmultigrid.hpp:311-316).
template <class Z>
__device__ void smooth(const DevHier& H, const Ws& w, const Z& zs, bool smem_z) {
    stencil_apply<kOutResid>(H.A, w.x, w.r, w.b);
    zs.reset(H.n_p);
    __syncthreads();
    tri_lower(H.L, w.r, zs, smem_z ? w.zg : nullptr);
    __syncthreads();
    if (smem_z) {
        zs.reset(H.n_p);
        __syncthreads();
        tri_upper(H.U, w.zg, zs, w.x);
    } else {
        const Z zu{w.r};
        zu.reset(H.n_p);
        __syncthreads();
        tri_upper(H.U, w.zg, zu, w.x);
    }
    __syncthreads();
}

// One V(nu_pre, nu_post) cycle (pmultigrid.hpp:256-267).
template <class Z>
__device__ void vcycle(const DevHier& H, const Ws& w, const Z& zs, bool smem_z) {
    for (int s = 0; s < H.nu_pre; ++s) smooth(H, w, zs, smem_z);
    stencil_apply<kOutResid>(H.A, w.x, w.r, w.b);
    __syncthreads();
    stencil_apply<kOutScale>(H.Tt, w.r, w.hb[0], H.inv_l1);  // restrict_to_linear
    cta_fill(w.hx[0], 0.0, H.n_1);
    __syncthreads();
    wcycle(H, w, 0);
    stencil_apply<kOutAddScaled>(H.T, w.hx[0], w.x, H.inv_lp);  // x += prolong_from_linear
    __syncthreads();
    for (int s = 0; s < H.nu_post; ++s) smooth(H, w, zs, smem_z);
}

__device__ double rel_residual(const DevHier& H, const Ws& w, double bnorm, double* sh) {
    stencil_apply<kOutResid>(H.A, w.x, w.r, w.b);
    const double d = cta_ordered_dot(w.r, w.r, H.n_p, sh);
    return sqrt(d) / bnorm;
}

// One Phi application: build b, solve (pmultigrid.hpp:271-307), epilogue.
template <class Z>
__device__ void phi_point(const DevHier& H, const DevStencil& Am, const WaveArgs& a, const Ws& w,
                          const Z& zs, bool smem_z, int task, int k, double* sh) {
    const int n = H.n_p;
    // ---- right-hand side and initial guess
    if (a.mode == kModeStep) {
        const double* uprev = a.U ? a.U + (size_t)(k - 1) * n : a.UPREV + (size_t)task * a.ldu;
        const double* load = nullptr;
        if (a.LOAD) load = a.load_steady ? a.LOAD : a.LOAD + (size_t)(k - 1) * n;
        else if (a.LOADV) load = a.LOADV + (size_t)task * a.ldl;
        if (load)
            stencil_apply<kOutAddVec>(Am, uprev, w.b, load);  // rhs = A- u + load
        else
            stencil_apply<kOutSet>(Am, uprev, w.b, nullptr);
        const double* guess = a.U ? a.U + (size_t)(a.guess_prev ? k - 1 : k) * n : (a.x0_empty ? nullptr : a.X + (size_t)task * a.ldx);
        if (guess)
            cta_copy(w.x, guess, n);
        else
            cta_fill(w.x, 0.0, n);
    } else {
        const double* bsrc;
        if (a.B) bsrc = a.B + (size_t)task * a.ldb;
        else bsrc = a.load_steady ? a.LOAD : a.LOAD + (size_t)(k - 1) * n;
        cta_copy(w.b, bsrc, n);
        if (a.x0_empty)
            cta_fill(w.x, 0.0, n);
        else
            cta_copy(w.x, a.X + (size_t)task * a.ldx, n);
    }
    __syncthreads();

    // ---- p-multigrid solve
    int iters = 0, conv = 0;
    double rel = 0.0;
    const double bnorm = sqrt(cta_ordered_dot(w.b, w.b, n, sh));
    if (bnorm == 0.0) {
        cta_fill(w.x, 0.0, n);  // zero rhs -> zero solution, not the guess
        conv = 1;
        __syncthreads();
    } else if (H.fixed_cycles > 0) {
        for (int c = 0; c < H.fixed_cycles; ++c) vcycle(H, w, zs, smem_z);
        iters = H.fixed_cycles;
        rel = rel_residual(H, w, bnorm, sh);
        conv = 1;
    } else {
        rel = rel_residual(H, w, bnorm, sh);
        if (rel <= H.rel_tol) {
            conv = 1;
        } else {
            for (int it = 1; it <= H.max_iter; ++it) {
                vcycle(H, w, zs, smem_z);
                rel = rel_residual(H, w, bnorm, sh);
                iters = it;
                if (rel <= H.rel_tol) {
                    conv = 1;
                    break;
                }
            }
        }
    }

    // ---- bookkeeping (SolveStats::record, theta.hpp:81-84)
    if (threadIdx.x == 0) {
        if (a.stat) {
            atomicAdd(a.stat, 1ULL);
            atomicAdd(a.stat + 1, (unsigned long long)iters);
        }
        if (a.iters_out) a.iters_out[task] = iters;
        if (a.conv_out) a.conv_out[task] = conv;
        if (a.rel_out) a.rel_out[task] = rel;
        if (!conv && a.err) {
            // first failing time index wins deterministically
            if (atomicMin(a.err + 1, k) > k) {
                a.err_rel[0] = rel;
                a.err[2] = a.level;
            }
            atomicExch(a.err, 1);
        }
    }

    // ---- epilogue
    const double* g = a.G ? a.G + (size_t)k * n : nullptr;
    if (a.epi == kEpiStore) {
        double* out = a.U + (size_t)k * n;
        for (int i = threadIdx.x; i < n; i += NT) out[i] = g ? w.x[i] + g[i] : w.x[i];
    } else if (a.epi == kEpiRestrict) {
        const int j = k / a.m;
        const double* u = a.U + (size_t)k * n;
        double* cg = a.CG + (size_t)j * n;
        double* cu = a.CU + (size_t)j * n;
        for (int i = threadIdx.x; i < n; i += NT) {
            const double wv = g ? w.x[i] + g[i] : w.x[i];
            cg[i] = wv - u[i];
            cu[i] = 0.0;
        }
    } else if (a.epi == kEpiResid) {
        const double* u = a.U + (size_t)k * n;
        for (int i = threadIdx.x; i < n; i += NT) {
            const double wv = g ? w.x[i] + g[i] : w.x[i];
            w.r[i] = wv - u[i];
        }
        const double d = cta_ordered_dot(w.r, w.r, n, sh);
        if (threadIdx.x == 0) a.SQ[k] = d;
    } else if (a.epi == kEpiNorm) {
        const double d = cta_ordered_dot(w.x, w.x, n, sh);
        if (threadIdx.x == 0) a.SQ[k] = d;
    } else {
        double* out = a.X + (size_t)task * a.ldx;
        for (int i = threadIdx.x; i < n; i += NT) out[i] = w.x[i];
    }
    __syncthreads();
}

template <class Z, bool SMEM>
__global__ void __launch_bounds__(NT) phi_wave_kernel(const __grid_constant__ DevHier H, const __grid_constant__ DevStencil Am, const __grid_constant__ WaveArgs a,
                                                      double* ws_base, long long ws_stride) {
    extern __shared__ __align__(16) double smem_z[];
    __shared__ double sh[4];
    const Ws w = carve(ws_base + (size_t)blockIdx.x * ws_stride, H);
    const Z zs{SMEM ? smem_z : w.zg};
    for (int task = blockIdx.x; task < a.n_tasks; task += gridDim.x) {
        for (int s = 0; s < a.task_len; ++s) {
            const int k = a.task_k0 ? a.task_k0[task] + s : task;
            phi_point(H, Am, a, w, zs, SMEM, task, k, sh);
        }
    }
}

// ---- standalone V-cycle on a batch (PMultigridHierarchy::vcycle) ----------
template <class Z, bool SMEM>
__global__ void __launch_bounds__(NT) vcycle_kernel(const __grid_constant__ DevHier H, const double* B, long long ldb, double* X,
                                                    long long ldx, int nrhs, double* ws_base,
                                                    long long ws_stride) {
    extern __shared__ __align__(16) double smem_z[];
    const Ws w = carve(ws_base + (size_t)blockIdx.x * ws_stride, H);
    const Z zs{SMEM ? smem_z : w.zg};
    const int n = H.n_p;
    for (int t = blockIdx.x; t < nrhs; t += gridDim.x) {
        cta_copy(w.b, B + (size_t)t * ldb, n);
        cta_copy(w.x, X + (size_t)t * ldx, n);
        __syncthreads();
        vcycle(H, w, zs, SMEM);
        double* out = X + (size_t)t * ldx;
        for (int i = threadIdx.x; i < n; i += NT) out[i] = w.x[i];
        __syncthreads();
    }
}

// ---- unit-level kernels used by the parity tests -------------------------
// op: 0 y = A x, 1 z = ILUT(r), 2 r1 = restrict(r), 3 x += prolong(e1) (x given),
//     4 x1 = W-cycle(b1, x1), 5 x = GS(b, x) on level `arg` (arg2 = backward)
template <class Z, bool SMEM>
__global__ void __launch_bounds__(NT) unit_kernel(const __grid_constant__ DevHier H, int op, int arg, int arg2, const double* in,
                                                  double* out, double* ws_base, long long ws_stride) {
    extern __shared__ __align__(16) double smem_z[];
    const Ws w = carve(ws_base + (size_t)blockIdx.x * ws_stride, H);
    const Z zs{SMEM ? smem_z : w.zg};
    const int n = H.n_p;
    if (op == 0) {
        stencil_apply<kOutSet>(H.A, in, out, nullptr);
    } else if (op == 1) {
        cta_copy(w.r, in, n);
        zs.reset(n);
        __syncthreads();
        tri_lower(H.L, w.r, zs, SMEM ? w.zg : nullptr);
        __syncthreads();
        cta_fill(w.x, 0.0, n);
        if (SMEM) {
            zs.reset(n);
            __syncthreads();
            tri_upper(H.U, w.zg, zs, w.x);
        } else {
            const Z zu{w.r};
            zu.reset(n);
            __syncthreads();
            tri_upper(H.U, w.zg, zu, w.x);
        }
        __syncthreads();
        cta_copy(out, w.x, n);
    } else if (op == 2) {
        stencil_apply<kOutScale>(H.Tt, in, out, H.inv_l1);
    } else if (op == 3) {
        stencil_apply<kOutAddScaled>(H.T, in, out, H.inv_lp);
    } else if (op == 4) {
        cta_copy(w.hb[0], in, H.n_1);
        cta_copy(w.hx[0], out, H.n_1);
        __syncthreads();
        wcycle(H, w, 0);
        cta_copy(out, w.hx[0], H.n_1);
    } else if (op == 5) {
        gs_sweep(H.h[arg].a, in, out, arg2 != 0);
    }
}

// ---- IC projection: Jacobi-preconditioned CG on M (solvers.hpp:21-75) ------
// Single CTA; all dot products index-ordered.  work: 4 vectors of n.
__global__ void __launch_bounds__(NT) cg_kernel(const __grid_constant__ DevStencil A, const double* __restrict__ diag,
                                                const double* __restrict__ b, double* x, double* work,
                                                double rel_tol, int max_iter, int* result) {
    __shared__ double sh[4];
    const int n = A.ru * A.rv;
    double* r = work;
    double* z = work + n;
    double* p = work + 2 * (size_t)n;
    double* q = work + 3 * (size_t)n;
    const double bnorm = sqrt(cta_ordered_dot(b, b, n, sh));
    if (bnorm == 0.0) {
        cta_fill(x, 0.0, n);
        if (threadIdx.x == 0) {
            result[0] = 1;
            result[1] = 0;
        }
        return;
    }
    cta_fill(x, 0.0, n);
    __syncthreads();
    stencil_apply<kOutResid>(A, x, r, b);
    double rnorm = sqrt(cta_ordered_dot(r, r, n, sh));
    if (rnorm <= rel_tol * bnorm) {
        if (threadIdx.x == 0) {
            result[0] = 1;
            result[1] = 0;
        }
        return;
    }
    for (int i = threadIdx.x; i < n; i += NT) {
        z[i] = r[i] / diag[i];
        p[i] = z[i];
    }
    double rz = cta_ordered_dot(r, z, n, sh);
    int conv = 0, it = 1;
    for (; it <= max_iter; ++it) {
        stencil_apply<kOutSet>(A, p, q, nullptr);
        const double pq = cta_ordered_dot(p, q, n, sh);
        if (pq <= 0.0) {
            conv = -1;
            break;
        }
        const double alpha = rz / pq;
        for (int i = threadIdx.x; i < n; i += NT) {
            x[i] += alpha * p[i];
            r[i] += -alpha * q[i];
        }
        rnorm = sqrt(cta_ordered_dot(r, r, n, sh));
        if (rnorm <= rel_tol * bnorm) {
            conv = 1;
            break;
        }
        for (int i = threadIdx.x; i < n; i += NT) z[i] = r[i] / diag[i];
        const double rz_new = cta_ordered_dot(r, z, n, sh);
        const double beta = rz_new / rz;
        rz = rz_new;
        for (int i = threadIdx.x; i < n; i += NT) p[i] = z[i] + beta * p[i];
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        result[0] = conv;
        result[1] = it;
    }
}

// ---- small elementwise MGRIT helpers --------------------------------------
// coarse.g[0] = fine.g[0] - fine.u[0]; coarse.u[0] = coarse.g[0]  (mgrit.hpp:155-166)
__global__ void restrict_first_kernel(const double* fg, const double* fu, double* cg, double* cu, int n) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const double v = fg[i] - fu[i];
        cg[i] = v;
        cu[i] = v;
    }
}

// fine.u[j*m] += coarse.u[j], j = 0..J  (mgrit.hpp:172-180)
__global__ void inject_kernel(const double* cu, double* fu, int n, int J, int m) {
    const size_t total = (size_t)(J + 1) * n;
    for (size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x; t < total;
         t += (size_t)gridDim.x * blockDim.x) {
        const size_t j = t / n, i = t - j * n;
        double* dst = fu + j * m * (size_t)n + i;
        *dst = *dst + cu[t];
    }
}

// sq[0] = |g[0] - u[0]|^2, index-ordered (single block)  (mgrit.hpp:202-203)
__global__ void resid0_kernel(const double* g, const double* u, double* sq, int n) {
    __shared__ double sh[4];
    if (threadIdx.x == 0) {
        double s = 0.0;
        for (int i = 0; i < n; ++i) {
            const double r = g[i] - u[i];
            s = s + r * r;
        }
        sq[0] = s;
    }
    (void)sh;
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
    size_t s = 4 * (size_t)H.n_p;
    for (int l = 0; l < H.n_h; ++l) s += 3 * (size_t)H.h[l].n;
    return (s + 31) & ~size_t(31);
}

bool phi_smem_z(const DevHier& H) { return (size_t)H.n_p * 8 <= kPhiSmemZMaxBytes; }

size_t phi_smem_bytes(const DevHier& H) { return phi_smem_z(H) ? (size_t)H.n_p * 8 : 0; }

template <class K>
static int occupancy_grid(K kernel, size_t smem, int want) {
    static int n_sm = 0;
    if (!n_sm) {
        int dev = 0;
        PHI_CUDA(cudaGetDevice(&dev));
        PHI_CUDA(cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev));
    }
    if (smem > 48 * 1024)
        PHI_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int per_sm = 0;
    PHI_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, NT, smem));
    if (per_sm < 1) per_sm = 1;
    return max(1, min(want, per_sm * n_sm));
}

int phi_max_slots(const DevHier& H) {
    const size_t smem = phi_smem_bytes(H);
    if (phi_smem_z(H)) return occupancy_grid(phi_wave_kernel<ZSmem, true>, smem, 1 << 30);
    return occupancy_grid(phi_wave_kernel<ZGlobal, false>, smem, 1 << 30);
}

void launch_phi_wave(const DevHier& H, const DevStencil& Am, const WaveArgs& a, double* ws,
                     long long ws_stride, int max_slots, cudaStream_t s) {
    if (a.n_tasks <= 0) return;
    const size_t smem = phi_smem_bytes(H);
    const int grid = min(a.n_tasks, max_slots);
    if (phi_smem_z(H)) {
        auto k = phi_wave_kernel<ZSmem, true>;
        occupancy_grid(k, smem, grid);
        k<<<grid, NT, smem, s>>>(H, Am, a, ws, ws_stride);
    } else {
        auto k = phi_wave_kernel<ZGlobal, false>;
        occupancy_grid(k, smem, grid);
        k<<<grid, NT, smem, s>>>(H, Am, a, ws, ws_stride);
    }
    PHI_CUDA(cudaGetLastError());
}

void launch_vcycle(const DevHier& H, const double* B, long long ldb, double* X, long long ldx, int nrhs,
                   double* ws, long long ws_stride, int max_slots, cudaStream_t s) {
    if (nrhs <= 0) return;
    const size_t smem = phi_smem_bytes(H);
    const int grid = min(nrhs, max_slots);
    if (phi_smem_z(H)) {
        auto k = vcycle_kernel<ZSmem, true>;
        occupancy_grid(k, smem, grid);
        k<<<grid, NT, smem, s>>>(H, B, ldb, X, ldx, nrhs, ws, ws_stride);
    } else {
        auto k = vcycle_kernel<ZGlobal, false>;
        occupancy_grid(k, smem, grid);
        k<<<grid, NT, smem, s>>>(H, B, ldb, X, ldx, nrhs, ws, ws_stride);
    }
    PHI_CUDA(cudaGetLastError());
}

void launch_unit(const DevHier& H, int op, int arg, int arg2, const double* in, double* out, double* ws,
                 long long ws_stride, cudaStream_t s) {
    const size_t smem = phi_smem_bytes(H);
    if (phi_smem_z(H)) {
        auto k = unit_kernel<ZSmem, true>;
        occupancy_grid(k, smem, 1);
        k<<<1, NT, smem, s>>>(H, op, arg, arg2, in, out, ws, ws_stride);
    } else {
        auto k = unit_kernel<ZGlobal, false>;
        occupancy_grid(k, smem, 1);
        k<<<1, NT, smem, s>>>(H, op, arg, arg2, in, out, ws, ws_stride);
    }
    PHI_CUDA(cudaGetLastError());
}

void launch_cg(const DevStencil& A, const double* diag, const double* b, double* x, double* work,
               double rel_tol, int max_iter, int* result, cudaStream_t s) {
    cg_kernel<<<1, NT, 0, s>>>(A, diag, b, x, work, rel_tol, max_iter, result);
    PHI_CUDA(cudaGetLastError());
}

void launch_restrict_first(const double* fg, const double* fu, double* cg, double* cu, int n, cudaStream_t s) {
    restrict_first_kernel<<<(n + 255) / 256, 256, 0, s>>>(fg, fu, cg, cu, n);
    PHI_CUDA(cudaGetLastError());
}

void launch_inject(const double* cu, double* fu, int n, int J, int m, cudaStream_t s) {
    const size_t total = (size_t)(J + 1) * n;
    const int grid = (int)std::min<size_t>((total + 255) / 256, 4096);
    inject_kernel<<<grid, 256, 0, s>>>(cu, fu, n, J, m);
    PHI_CUDA(cudaGetLastError());
}

void launch_resid0(const double* g, const double* u, double* sq, int n, cudaStream_t s) {
    resid0_kernel<<<1, 32, 0, s>>>(g, u, sq, n);
    PHI_CUDA(cudaGetLastError());
}

void launch_copy(double* dst, const double* src, size_t n, cudaStream_t s) {
    if (!n) return;
    const int grid = (int)std::min<size_t>((n + 255) / 256, 4096);
    copy_kernel<<<grid, 256, 0, s>>>(dst, src, n);
    PHI_CUDA(cudaGetLastError());
}

}  // namespace phi
