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
// The solve is a chain of dependent steps (ILUT level sets, Gauss-Seidel
// wavefronts), so the kernel is organised for latency:
//  * sync-free triangular solves and Gauss-Seidel sweeps: a row waits only for
//    the values it reads.  Solved values are published with one 64-bit store
//    into a "sentinel" array (a signalling-NaN bit pattern means "not solved
//    yet"), so readiness flag and value are the same word -- one load per
//    dependency, no fences, no barriers inside a sweep;
//  * factor entries are streamed through a per-lane register ring (D deep), so
//    global-memory latency overlaps the dependent arithmetic;
//  * the dependency arrays and the order-1 h-levels live in shared memory when
//    they fit (SmemPlan), so the critical path runs at shared-memory latency;
//  * index-ordered dot products stage the products in shared memory and one
//    thread sums them in order.
#include <cuda_pipeline.h>
#include <cuda_runtime.h>

#include <algorithm>

#include "device_types.cuh"
#include "phi_kernels.cuh"
#include "setup_host.hpp"

namespace phi {

namespace {

constexpr int NT = kPhiThreads;
constexpr int NW = NT / 32;
constexpr int kDotChunk = 2048;  // doubles of shared scratch for ordered dots
constexpr int kRing = kTriRing;  // factor-entry prefetch depth per lane (setup_host.hpp)
constexpr unsigned long long kSentinel = 0x7FF4DEADBEEF0001ULL;

// Dynamic shared memory of every Phi kernel (laid out by SmemPlan).
extern __shared__ __align__(16) double g_smem[];

// Runtime tuning of the sync-free sweeps (developer knob, phi_dev_tuning).
struct Tuning {
    int tri_warps;  // warps taking part in a triangular solve (<= NW)
    int gs_warps;   // warps taking part in a Gauss-Seidel sweep (<= NW)
    int sleep_ns;   // back-off between failed readiness polls (0 = spin)
    int pad;
    long long* trace;  // developer timing trace of triangular-solve blocks (null = off)
};
__constant__ Tuning c_tune = {NW, NW, 0, 0, nullptr};

// CTA-scope relaxed accesses through generic pointers: shared memory, or
// global memory served by the SM's L1 (42 cycles, vs 289 for a volatile =
// system-scope global load; measured with tools/lat_probe.cu on B200).
__device__ __forceinline__ unsigned long long ld_rlx(const double* p) {
    unsigned long long v;
    asm volatile("ld.relaxed.cta.u64 %0, [%1];" : "=l"(v) : "l"(p));
    return v;
}
__device__ __forceinline__ double wait_val(const double* p) {
    unsigned long long b = ld_rlx(p);
    while (b == kSentinel) {
        if (c_tune.sleep_ns) __nanosleep(c_tune.sleep_ns);
        b = ld_rlx(p);
    }
    return __longlong_as_double(static_cast<long long>(b));
}
__device__ __forceinline__ void put_val(double* p, double v) {
    asm volatile("st.relaxed.cta.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}
// Explicit 32-bit shared-window accesses.  Deriving shared pointers inside hot
// loops makes the compiler re-read the window base (S2R SR_SWINHI /
// SR_CgaCtaId) per access; these take the address once, up front.
__device__ __forceinline__ unsigned sh_addr(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ unsigned long long lds_vol_u64(unsigned a) {
    unsigned long long v;
    asm volatile("ld.volatile.shared.u64 %0, [%1];" : "=l"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ double lds_f64(unsigned a) {
    double v;
    asm("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ int lds_s32(unsigned a) {
    int v;
    asm("ld.shared.s32 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ void sts_vol_f64(unsigned a, double v) {
    asm volatile("st.volatile.shared.f64 [%0], %1;" ::"r"(a), "d"(v) : "memory");
}
__device__ __forceinline__ void reset_sentinel(double* z, int n) {
    for (int i = threadIdx.x; i < n; i += NT) reinterpret_cast<unsigned long long*>(z)[i] = kSentinel;
}
// Triangular-solve dependency array: n sentinels plus the always-ready dummy
// slot z[n] = +0.0 that padded factor entries point at (see TriPlan).
__device__ __forceinline__ void reset_dep(double* z, int n) {
    reset_sentinel(z, n);
    if (threadIdx.x == 0) z[n] = 0.0;
}

// ---------------------------------------------------------------------------
// per-CTA workspace (generic pointers: shared memory or global per SmemPlan)
// ---------------------------------------------------------------------------
struct Ws {
    double *b, *x, *r, *zg;  // global
    double* z;               // in-place triangular-solve vector (n_p + 1 slots)
    double* dot;             // shared scratch for ordered dots
    int z_off, ring_off, prod_off, slot_bytes;  // g_smem offsets (-1: global)
    double* hb[kMaxH];
    double* hx[kMaxH];
    double* hx2[kMaxH];
    double* hr[kMaxH];
};

__device__ Ws carve(double* base, const DevHier& H, const SmemPlan& P, double* smem) {
    Ws w;
    const size_t np = (size_t)H.n_p + 2;  // room for the dummy slot z[n]
    w.b = base;
    w.x = base + np;
    w.r = base + 2 * np;
    w.zg = base + 3 * np;
    w.z = P.z_off >= 0 ? smem + P.z_off : base + 4 * np;
    w.dot = smem + P.dot_off;
    w.z_off = P.z_off;
    w.ring_off = P.ring_off;
    w.prod_off = P.prod_off;
    w.slot_bytes = P.slot_bytes;
    double* g = base + 6 * np;
    for (int l = 0; l < H.n_h; ++l) {
        const int nl = H.h[l].n;
        double* s = P.lvl_off[l] >= 0 ? smem + P.lvl_off[l] : g;
        w.hb[l] = s;
        w.hx[l] = s + nl;
        w.hx2[l] = s + 2 * (size_t)nl;
        w.hr[l] = s + 3 * (size_t)nl;
        g += 4 * (size_t)nl;
    }
    return w;
}

// ---------------------------------------------------------------------------
// CTA-cooperative primitives.  Callers place __syncthreads() between phases.
// ---------------------------------------------------------------------------
enum StencilOut : int { kOutSet = 0, kOutResid = 1, kOutScale = 2, kOutAddScaled = 3, kOutAddVec = 4 };

// y[i] (op)= sum_e vals[e][i] * x[col(i, e)], entries in reference CSR order
// (dv, du ascending), one sequential sum per row; the W loads of a stencil
// row are issued together.
template <int OUT, int W>
__device__ __forceinline__ void stencil_apply(const DevStencil& A, const double* __restrict__ x,
                                                double* __restrict__ y, const double* __restrict__ aux) {
    const int n = A.ru * A.rv;
    for (int i = threadIdx.x; i < n; i += NT) {
        const int iv = i / A.ru;
        const int iu = i - iv * A.ru;
        const int dulo = max(A.lo, -iu), duhi = min(A.hi, A.cu - 1 - iu);
        const int dvlo = max(A.lo, -iv), dvhi = min(A.hi, A.cv - 1 - iv);
        double s = 0.0;
        for (int dv = dvlo; dv <= dvhi; ++dv) {
            const double* vr = A.vals + (size_t)((dv - A.lo) * W) * n + i;
            const double* xr = x + (size_t)(iv + dv) * A.cu + iu;
            double pv[W], px[W];
#pragma unroll
            for (int q = 0; q < W; ++q) {
                const int du = A.lo + q;
                if (du >= dulo && du <= duhi) {
                    pv[q] = __ldg(vr + (size_t)q * n);
                    px[q] = xr[du];
                }
            }
#pragma unroll
            for (int q = 0; q < W; ++q) {
                const int du = A.lo + q;
                if (du >= dulo && du <= duhi) s = s + pv[q] * px[q];
            }
        }
        if (OUT == kOutSet) y[i] = s;
        if (OUT == kOutResid) y[i] = aux[i] - s;             // r = b - A x
        if (OUT == kOutScale) y[i] = s * aux[i];             // (P^T r) .* 1/M^L
        if (OUT == kOutAddScaled) y[i] = y[i] + s * aux[i];  // x += (P e) .* 1/M^L
        if (OUT == kOutAddVec) y[i] = s + aux[i];            // rhs = A- u + load
    }
}

// Compile-time stencil widths of a degree-P hierarchy: A = M + cK (2P+1),
// transfer P->1 (P+2; identity for P = 1), order-1 h-levels (3).
template <int P>
struct Widths {
    static constexpr int A = 2 * P + 1;
    static constexpr int T = P == 1 ? 1 : P + 2;
    static constexpr int H = 3;
};

// y = A x (CSR, row order) or y += A x.
template <bool ADD>
__device__ __forceinline__ void csr_apply(const DevCsr& A, const double* __restrict__ x, double* __restrict__ y) {
    for (int i = threadIdx.x; i < A.n_rows; i += NT) {
        const int e0 = A.ro[i], e1 = A.ro[i + 1];
        double pv[4], px[4];
#pragma unroll
        for (int q = 0; q < 4; ++q)
            if (e0 + q < e1) {
                pv[q] = __ldg(A.v + e0 + q);
                px[q] = x[__ldg(A.ci + e0 + q)];
            }
        double s = 0.0;
#pragma unroll
        for (int q = 0; q < 4; ++q)
            if (e0 + q < e1) s = s + pv[q] * px[q];
        for (int e = e0 + 4; e < e1; ++e) s = s + A.v[e] * x[A.ci[e]];
        if (ADD)
            y[i] = y[i] + s;
        else
            y[i] = s;
    }
}

// One lexicographic Gauss-Seidel sweep (solvers.hpp:80-99) for the 9-point
// order-1 operator, in place, by anti-diagonal wavefronts u + 2v = t
// (forward; mirrored for backward): a row of wavefront t reads updated values
// only from wavefronts < t and old values only from wavefronts > t, so
// updating a whole wavefront between two barriers gives exactly the
// sequential sweep.  Thread q owns row q of each wavefront; its nine matrix
// entries for the next wavefront are prefetched while the current one is
// solved.  Entries outside the grid carry a = +0.0 and x = +0.0, and
// s - (+0 * +0) == s, so the branch-free row sum is bit-identical.
template <bool SM>
__device__ __noinline__ void gs_sweep_impl(const DevStencil& A, const double* __restrict__ b, double* x,
                                           bool backward) {
    const unsigned b_s = SM ? sh_addr(b) : 0u, x_s = SM ? sh_addr(x) : 0u;
    const int nu = A.ru, nv = A.rv, n = nu * nv;
    const double* __restrict__ av = A.vals;  // cached: A lives in the param space
    const int T = (nu - 1) + 2 * (nv - 1);
    const int tid = threadIdx.x;
    auto row_of = [&](int t, int q, int& iu, int& iv) {
        const int vlo = max(0, (t - (nu - 1) + 1) / 2);
        const int vhi = min(nv - 1, t / 2);
        const int v = vlo + q;
        if (v > vhi) return -1;
        const int u = t - 2 * v;
        iu = backward ? nu - 1 - u : u;
        iv = backward ? nv - 1 - v : v;
        return iu + nu * iv;
    };
    // Unconditional loads: the stencil-major array stores +0.0 for entries
    // outside the grid, so no select (which would wait on the fresh load) is
    // needed, and +0 * +0 leaves the row sum bit-identical.
    auto fetch = [&](int t, double* a) {
        int iu = 0, iv = 0;
        int i = t <= T ? row_of(t, tid, iu, iv) : -1;
        if (i < 0) i = 0;
#pragma unroll
        for (int e = 0; e < 9; ++e) a[e] = __ldg(av + (size_t)e * n + i);
    };
    // two register buffers, alternated by a 2x-unrolled wavefront loop, so a
    // prefetched row is never copied (a copy would wait on the fresh load)
    double abuf0[9], abuf1[9];
    auto process = [&](int t, double (&a)[9]) {
        long long* tr = (c_tune.trace && tid == 0 && t < 1024) ? c_tune.trace + (size_t)NW * 1024 * 2 + (size_t)t * 4
                                                               : nullptr;
        if (tr) tr[0] = clock64();
        int iu = 0, iv = 0;
        for (int q = tid;; q += NT) {
            const int i = row_of(t, q, iu, iv);
            if (i < 0) break;
            if (q != tid) {  // rows beyond the first NT of a wavefront: no prefetch
#pragma unroll
                for (int e = 0; e < 9; ++e) a[e] = __ldg(av + (size_t)e * n + i);
            }
            double xv[9];
#pragma unroll
            for (int e = 0; e < 9; ++e) {
                const int dv = e / 3 - 1, du = e % 3 - 1;
                const bool ok = e != 4 && iu + du >= 0 && iu + du < nu && iv + dv >= 0 && iv + dv < nv;
                const int j = i + du + nu * dv;
                xv[e] = ok ? (SM ? lds_f64(x_s + 8u * j) : x[j]) : 0.0;
            }
            double s = SM ? lds_f64(b_s + 8u * i) : b[i];
            double p[9];
#pragma unroll
            for (int e = 0; e < 9; ++e) p[e] = a[e] * xv[e];
#pragma unroll
            for (int e = 0; e < 9; ++e)
                if (e != 4) s = s - p[e];
            if (tr && q == tid) tr[1] = clock64() + (long long)(s == 12345.678);  // s is ready
            const double xi = s / a[4];
            if (SM)
                asm volatile("st.shared.f64 [%0], %1;" ::"r"(x_s + 8u * i), "d"(xi) : "memory");
            else
                x[i] = xi;
            if (tr && q == tid) tr[2] = clock64() + (long long)(xi == 12345.678);
        }
        __syncthreads();
        if (tr) tr[3] = clock64();
    };
    // two register buffers alternated by a 2x-unrolled wavefront loop: a
    // prefetched row is consumed in place, never copied (a copy would wait on
    // the load that was just issued)
    fetch(0, abuf0);
    for (int t = 0; t <= T; t += 2) {
        fetch(t + 1, abuf1);
        process(t, abuf0);
        if (t + 1 > T) break;
        fetch(t + 2, abuf0);
        process(t + 1, abuf1);
    }
}

__device__ __forceinline__ void gs_sweep(const DevStencil& A, const double* b, double* x, bool backward) {
    if (__isShared(x))
        gs_sweep_impl<true>(A, b, x, backward);
    else
        gs_sweep_impl<false>(A, b, x, backward);
}

// ---- triangular solves: level-synchronous, TMA-fed ------------------------
// The factor is one level-ordered stream of blocks (TriStream), each holding a
// chunk of <= kTriRows rows of one level with all their entries.  A ring of
// kTriSlots shared-memory slots is filled by TMA bulk copies
// (cp.async.bulk + mbarrier complete_tx), kTriSlots-1 blocks ahead; the next
// block's address travels in the header of the block being consumed.
__device__ __forceinline__ void mbar_init(unsigned bar) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void bulk_fetch(unsigned dst, const void* src, int bytes, unsigned bar) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                 "l"(src), "r"(bytes), "r"(bar)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned bar, unsigned parity) {
    unsigned done;
    do {
        asm volatile(
            "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
            : "=r"(done)
            : "r"(bar), "r"(parity)
            : "memory");
    } while (!done);
}

// In-place substitution with an ILUT factor (ilut.hpp:146-163) on z, which
// holds the right-hand side on entry.  Lower: z_i -= sum_j L_ij z_j (unit
// diagonal).  Upper: z_i = (z_i - sum_j U_ij z_j) / U_ii, fused with the
// smoother update x += z (pmultigrid.hpp:315).  Per block: every thread forms
// products L_ij * z_j (all j belong to earlier levels), one barrier, then the
// row's thread subtracts them in CSR order -- the reference's exact sequence
// of roundings -- and publishes z_i; a second barrier closes the level.
// Padded entries (column n, value +0.0; z[n] = +0.0) are exactly neutral.
template <bool UPPER, bool ZSM>
__device__ __noinline__ void tri_solve_impl(const DevTri& T, double* zg, int z_off, double* xadd, int ring_off,
                                            int slot_bytes, int prod_off) {
    __shared__ unsigned long long bars[kTriSlots];
    const int tid = threadIdx.x;
    const unsigned ring = sh_addr(g_smem + ring_off);
    const unsigned prod = sh_addr(g_smem + prod_off);
    const unsigned zs = ZSM ? sh_addr(g_smem + z_off) : 0u;
    const unsigned bar = sh_addr(bars);
    if (tid == 0) {
        for (int k = 0; k < kTriSlots; ++k) mbar_init(bar + 8u * k);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        for (int k = 0; k < kTriSlots - 1 && k < T.n_blocks; ++k)
            bulk_fetch(ring + k * slot_bytes, T.stream + (size_t)T.prime[2 * k] * 16, T.prime[2 * k + 1],
                       bar + 8u * k);
    }
    // cached: T lives in the kernel parameter space (generic loads otherwise)
    const int n_blocks = T.n_blocks;
    const unsigned char* __restrict__ stream = T.stream;
    __syncthreads();
    for (int b = 0; b < n_blocks; ++b) {
        const int slot = b % kTriSlots;
        mbar_wait(bar + 8u * slot, (unsigned)(b / kTriSlots) & 1u);
        const unsigned blk = ring + slot * slot_bytes;
        int nr, span, row0, next_off;
        asm volatile("ld.shared.v4.s32 {%0, %1, %2, %3}, [%4];"
                     : "=r"(nr), "=r"(span), "=r"(row0), "=r"(next_off)
                     : "r"(blk));
        if (tid == 0) {
            const int next_bytes = lds_s32(blk + 16);
            // block b + kTriSlots - 1 refills the slot released by the last barrier
            if (next_bytes > 0)
                bulk_fetch(ring + ((b + kTriSlots - 1) % kTriSlots) * slot_bytes, stream + (size_t)next_off * 16,
                           next_bytes, bar + 8u * ((b + kTriSlots - 1) % kTriSlots));
        }
        const int items = nr * span;
        const unsigned cols = blk + kTriBlockPrefix;
        const unsigned vals = cols + 4u * items;
        for (int t = tid; t < items; t += NT) {
            const int j = lds_s32(cols + 4u * t);
            const double z = ZSM ? lds_f64(zs + 8u * j) : zg[j];
            asm volatile("st.shared.f64 [%0], %1;" ::"r"(prod + 8u * t), "d"(lds_f64(vals + 8u * t) * z));
        }
        __syncthreads();
        if (tid < nr) {
            const int i = lds_s32(blk + 32u + 4u * tid);
            double s = ZSM ? lds_f64(zs + 8u * i) : zg[i];
            const unsigned pp = prod + 8u * tid;
            int e = 0;
            for (; e + 8 <= span; e += 8) {
                double p[8];
#pragma unroll
                for (int q = 0; q < 8; ++q) p[q] = lds_f64(pp + 8u * (e + q) * nr);
#pragma unroll
                for (int q = 0; q < 8; ++q) s = s - p[q];
            }
            for (; e < span; ++e) s = s - lds_f64(pp + 8u * e * nr);
            if (UPPER) {
                s = s / lds_f64(blk + 64u + 8u * tid);
                xadd[i] = xadd[i] + s;
            }
            if (ZSM)
                asm volatile("st.shared.f64 [%0], %1;" ::"r"(zs + 8u * i), "d"(s) : "memory");
            else
                zg[i] = s;
        }
        __syncthreads();
    }
}

template <bool UPPER>
__device__ __forceinline__ void tri_solve(const DevTri& T, double* zg, int z_off, double* xadd, int ring_off,
                                          int slot_bytes, int prod_off) {
    if (z_off >= 0)
        tri_solve_impl<UPPER, true>(T, zg, z_off, xadd, ring_off, slot_bytes, prod_off);
    else
        tri_solve_impl<UPPER, false>(T, zg, z_off, xadd, ring_off, slot_bytes, prod_off);
}

// Index-ordered dot product (sparse.hpp:188-192): products in parallel into
// shared scratch, one thread sums them in index order.  Broadcast result.
__device__ double cta_ordered_dot(const double* a, const double* b, int n, double* scratch, double* sh) {
    double s = 0.0;
    for (int c0 = 0; c0 < n; c0 += kDotChunk) {
        const int cnt = min(kDotChunk, n - c0);
        __syncthreads();
        for (int i = threadIdx.x; i < cnt; i += NT) scratch[i] = a[c0 + i] * b[c0 + i];
        __syncthreads();
        if (threadIdx.x == 0) {
            int i = 0;
            for (; i + 8 <= cnt; i += 8) {
                double p[8];
#pragma unroll
                for (int q = 0; q < 8; ++q) p[q] = scratch[i + q];
#pragma unroll
                for (int q = 0; q < 8; ++q) s = s + p[q];
            }
            for (; i < cnt; ++i) s = s + scratch[i];
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) sh[0] = s;
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

// h-multigrid W-cycle (pmultigrid.hpp:184-200) as an explicit per-level
// phase machine (no device recursion):
//   phase 0: pre-smooth, restrict, first coarse visit
//   phase 1: second coarse visit (starting from the first visit's result)
//   phase 2: prolongate, post-smooth, return
// Solution of level l lives in w.hx[l]; the result of level 0 is w.hx[0].
template <int DEG>
__device__ __noinline__ void wcycle(const DevHier& H, const Ws& w) {
    int phase[kMaxH];
    int l = 0;
    phase[0] = 0;
    for (;;) {
        if (l + 1 == H.n_h) {
            coarse_solve(H, w.hb[l], w.hx[l]);
            if (l == 0) break;
            --l;
            continue;
        }
        const DevHLevel& lv = H.h[l];
        double* b = w.hb[l];
        double* x = w.hx[l];
        if (phase[l] == 0) {
            for (int s = 0; s < H.gs_pre; ++s) gs_sweep(lv.a, b, x, false);
            stencil_apply<kOutResid, Widths<DEG>::H>(lv.a, x, w.hr[l], b);
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
            if (l == 0) break;
            --l;
        }
    }
}

// x += S (b - A x), S = ILUT application (pmultigrid.hpp:311-316).
template <int DEG>
__device__ __noinline__ void smooth(const DevHier& H, const Ws& w) {
    stencil_apply<kOutResid, Widths<DEG>::A>(H.A, w.x, w.z, w.b);  // z = r = b - A x
    if (threadIdx.x == 0) w.z[H.n_p] = 0.0;                          // neutral padding slot
    __syncthreads();
    tri_solve<false>(H.L, w.z, w.z_off, nullptr, w.ring_off, w.slot_bytes, w.prod_off);
    tri_solve<true>(H.U, w.z, w.z_off, w.x, w.ring_off, w.slot_bytes, w.prod_off);
}

// One V(nu_pre, nu_post) cycle (pmultigrid.hpp:256-267).
template <int DEG>
__device__ __noinline__ void vcycle(const DevHier& H, const Ws& w) {
    for (int s = 0; s < H.nu_pre; ++s) smooth<DEG>(H, w);
    stencil_apply<kOutResid, Widths<DEG>::A>(H.A, w.x, w.r, w.b);
    __syncthreads();
    stencil_apply<kOutScale, Widths<DEG>::T>(H.Tt, w.r, w.hb[0], H.inv_l1);  // restrict_to_linear
    cta_fill(w.hx[0], 0.0, H.n_1);
    __syncthreads();
    wcycle<DEG>(H, w);
    stencil_apply<kOutAddScaled, Widths<DEG>::T>(H.T, w.hx[0], w.x, H.inv_lp);  // x += prolong_from_linear
    __syncthreads();
    for (int s = 0; s < H.nu_post; ++s) smooth<DEG>(H, w);
}

template <int DEG>
__device__ double rel_residual(const DevHier& H, const Ws& w, double bnorm, double* sh) {
    stencil_apply<kOutResid, Widths<DEG>::A>(H.A, w.x, w.r, w.b);
    const double d = cta_ordered_dot(w.r, w.r, H.n_p, w.dot, sh);
    return sqrt(d) / bnorm;
}

// One Phi application: build b, solve (pmultigrid.hpp:271-307), epilogue.
template <int DEG>
__device__ void phi_point(const DevHier& H, const DevStencil& Am, const WaveArgs& a, const Ws& w, int task,
                          int k, double* sh) {
    const int n = H.n_p;
    // ---- right-hand side and initial guess
    if (a.mode == kModeStep) {
        const double* uprev = a.U ? a.U + (size_t)(k - 1) * n : a.UPREV + (size_t)task * a.ldu;
        const double* load = nullptr;
        if (a.LOAD)
            load = a.load_steady ? a.LOAD : a.LOAD + (size_t)(k - 1) * n;
        else if (a.LOADV)
            load = a.LOADV + (size_t)task * a.ldl;
        if (load)
            stencil_apply<kOutAddVec, Widths<DEG>::A>(Am, uprev, w.b, load);  // rhs = A- u + load
        else
            stencil_apply<kOutSet, Widths<DEG>::A>(Am, uprev, w.b, nullptr);
        const double* guess =
            a.U ? a.U + (size_t)(a.guess_prev ? k - 1 : k) * n : (a.x0_empty ? nullptr : a.X + (size_t)task * a.ldx);
        if (guess)
            cta_copy(w.x, guess, n);
        else
            cta_fill(w.x, 0.0, n);
    } else {
        const double* bsrc;
        if (a.B)
            bsrc = a.B + (size_t)task * a.ldb;
        else
            bsrc = a.load_steady ? a.LOAD : a.LOAD + (size_t)(k - 1) * n;
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
    const double bnorm = sqrt(cta_ordered_dot(w.b, w.b, n, w.dot, sh));
    if (bnorm == 0.0) {
        cta_fill(w.x, 0.0, n);  // zero rhs -> zero solution, not the guess
        conv = 1;
        __syncthreads();
    } else if (H.fixed_cycles > 0) {
        for (int c = 0; c < H.fixed_cycles; ++c) vcycle<DEG>(H, w);
        iters = H.fixed_cycles;
        rel = rel_residual<DEG>(H, w, bnorm, sh);
        conv = 1;
    } else {
        rel = rel_residual<DEG>(H, w, bnorm, sh);
        if (rel <= H.rel_tol) {
            conv = 1;
        } else {
            for (int it = 1; it <= H.max_iter; ++it) {
                vcycle<DEG>(H, w);
                rel = rel_residual<DEG>(H, w, bnorm, sh);
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
        if (a.wave_max) {
            atomicMax(a.wave_max, iters);
            atomicAdd(a.wave_max + 1, iters);
            atomicAdd(a.wave_max + 2, 1);
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
        const double d = cta_ordered_dot(w.r, w.r, n, w.dot, sh);
        if (threadIdx.x == 0) a.SQ[k] = d;
    } else if (a.epi == kEpiNorm) {
        const double d = cta_ordered_dot(w.x, w.x, n, w.dot, sh);
        if (threadIdx.x == 0) a.SQ[k] = d;
    } else {
        double* out = a.X + (size_t)task * a.ldx;
        for (int i = threadIdx.x; i < n; i += NT) out[i] = w.x[i];
    }
    __syncthreads();
}

template <int DEG>
__global__ void __launch_bounds__(NT, 1)
    phi_wave_kernel(const __grid_constant__ DevHier H, const __grid_constant__ DevStencil Am,
                    const __grid_constant__ WaveArgs a, const __grid_constant__ SmemPlan P, double* ws_base,
                    long long ws_stride) {
    double* smem = g_smem;
    __shared__ double sh[4];
    const Ws w = carve(ws_base + (size_t)blockIdx.x * ws_stride, H, P, smem);
    for (int task = blockIdx.x; task < a.n_tasks; task += gridDim.x) {
        for (int s = 0; s < a.task_len; ++s) {
            const int k = a.task_k0 ? a.task_k0[task] + s : task;
            phi_point<DEG>(H, Am, a, w, task, k, sh);
        }
    }
}

// ---- standalone V-cycle on a batch (PMultigridHierarchy::vcycle) ----------
template <int DEG>
__global__ void __launch_bounds__(NT, 1)
    vcycle_kernel(const __grid_constant__ DevHier H, const double* B, long long ldb, double* X, long long ldx,
                  int nrhs, const __grid_constant__ SmemPlan P, double* ws_base, long long ws_stride) {
    double* smem = g_smem;
    const Ws w = carve(ws_base + (size_t)blockIdx.x * ws_stride, H, P, smem);
    const int n = H.n_p;
    for (int t = blockIdx.x; t < nrhs; t += gridDim.x) {
        cta_copy(w.b, B + (size_t)t * ldb, n);
        cta_copy(w.x, X + (size_t)t * ldx, n);
        __syncthreads();
        vcycle<DEG>(H, w);
        double* out = X + (size_t)t * ldx;
        for (int i = threadIdx.x; i < n; i += NT) out[i] = w.x[i];
        __syncthreads();
    }
}

// ---- unit-level kernel used by the parity tests ---------------------------
// op: 0 y = A x, 1 z = ILUT(r), 2 r1 = restrict(r), 3 x += prolong(e1) (x given),
//     4 x1 = W-cycle(b1, x1), 5 x = GS(b, x) on level `arg` (arg2 = backward)
template <int DEG>
__global__ void __launch_bounds__(NT, 1)
    unit_kernel(const __grid_constant__ DevHier H, int op, int arg, int arg2, const double* in, double* out,
                const __grid_constant__ SmemPlan P, double* ws_base, long long ws_stride) {
    double* smem = g_smem;
    const Ws w = carve(ws_base + (size_t)blockIdx.x * ws_stride, H, P, smem);
    const int n = H.n_p;
    if (op == 0) {
        stencil_apply<kOutSet, Widths<DEG>::A>(H.A, in, out, nullptr);
    } else if (op == 1) {
        cta_copy(w.z, in, n);
        cta_fill(w.x, 0.0, n);
        if (threadIdx.x == 0) w.z[n] = 0.0;
        __syncthreads();
        tri_solve<false>(H.L, w.z, w.z_off, nullptr, w.ring_off, w.slot_bytes, w.prod_off);
        tri_solve<true>(H.U, w.z, w.z_off, w.x, w.ring_off, w.slot_bytes, w.prod_off);
        cta_copy(out, w.z, n);
    } else if (op == 2) {
        stencil_apply<kOutScale, Widths<DEG>::T>(H.Tt, in, out, H.inv_l1);
    } else if (op == 3) {
        stencil_apply<kOutAddScaled, Widths<DEG>::T>(H.T, in, out, H.inv_lp);
    } else if (op == 4) {
        cta_copy(w.hb[0], in, H.n_1);
        cta_copy(w.hx[0], out, H.n_1);
        __syncthreads();
        wcycle<DEG>(H, w);
        cta_copy(out, w.hx[0], H.n_1);
    } else if (op == 5) {
        const DevHLevel& lv = H.h[arg];
        cta_copy(w.hb[arg], in, lv.n);
        cta_copy(w.hx[arg], out, lv.n);
        __syncthreads();
        gs_sweep(lv.a, w.hb[arg], w.hx[arg], arg2 != 0);
        cta_copy(out, w.hx[arg], lv.n);
    }
}

// ---- IC projection: Jacobi-preconditioned CG on M (solvers.hpp:21-75) ------
// Single CTA; all dot products index-ordered.  work: 4 vectors of n.
template <int DEG>
__global__ void __launch_bounds__(NT, 1)
    cg_kernel(const __grid_constant__ DevStencil A, const double* __restrict__ diag, const double* __restrict__ b,
              double* x, double* work, double rel_tol, int max_iter, int* result) {
    __shared__ double sh[4];
    __shared__ double scratch[kDotChunk];
    const int n = A.ru * A.rv;
    double* r = work;
    double* z = work + n;
    double* p = work + 2 * (size_t)n;
    double* q = work + 3 * (size_t)n;
    const double bnorm = sqrt(cta_ordered_dot(b, b, n, scratch, sh));
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
    stencil_apply<kOutResid, Widths<DEG>::A>(A, x, r, b);
    double rnorm = sqrt(cta_ordered_dot(r, r, n, scratch, sh));
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
    double rz = cta_ordered_dot(r, z, n, scratch, sh);
    int conv = 0, it = 1;
    for (; it <= max_iter; ++it) {
        stencil_apply<kOutSet, Widths<DEG>::A>(A, p, q, nullptr);
        const double pq = cta_ordered_dot(p, q, n, scratch, sh);
        if (pq <= 0.0) {
            conv = -1;
            break;
        }
        const double alpha = rz / pq;
        for (int i = threadIdx.x; i < n; i += NT) {
            x[i] += alpha * p[i];
            r[i] += -alpha * q[i];
        }
        rnorm = sqrt(cta_ordered_dot(r, r, n, scratch, sh));
        if (rnorm <= rel_tol * bnorm) {
            conv = 1;
            break;
        }
        for (int i = threadIdx.x; i < n; i += NT) z[i] = r[i] / diag[i];
        const double rz_new = cta_ordered_dot(r, z, n, scratch, sh);
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
    for (size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x; t < total; t += (size_t)gridDim.x * blockDim.x) {
        const size_t j = t / n, i = t - j * n;
        double* dst = fu + j * m * (size_t)n + i;
        *dst = *dst + cu[t];
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
    for (int l = 0; l < H.n_h; ++l) s += 4 * (size_t)H.h[l].n;
    return (s + 31) & ~size_t(31);
}

SmemPlan phi_smem_plan(const DevHier& H) {
    // The three users of shared memory are live in disjoint phases of a
    // V-cycle, so they overlay one another from offset 0:
    //   smoothing  : triangular-factor rings + dependency array z
    //   W-cycle    : the order-1 h-level vectors (restrict .. prolong)
    //   norms      : the ordered-dot scratch
    SmemPlan P{};
    const size_t budget = kPhiSmemBudgetBytes / 8;  // doubles
    P.ring_off = 0;
    P.dot_off = 0;
    P.slot_bytes = (std::max(H.L.max_block_bytes, H.U.max_block_bytes) + 127) / 128 * 128;
    size_t tri = (size_t)kTriSlots * P.slot_bytes / 8;
    P.prod_off = (int)tri;
    tri += ((size_t)std::max(H.L.max_items, H.U.max_items) + 1) / 2 * 2;
    if (tri * 8 > kPhiSmemBudgetBytes) throw InvalidArgument("triangular-factor blocks exceed shared memory");
    if (tri + (size_t)H.n_p + 2 <= budget) {
        P.z_off = (int)tri;
        tri += H.n_p + 2;
    } else {
        P.z_off = -1;
    }
    for (int l = 0; l < kMaxH; ++l) P.lvl_off[l] = -1;
    // coarsest levels first: they are visited most often by the W-cycle
    size_t lv = 0;
    for (int l = H.n_h - 1; l >= 0; --l) {
        const size_t need = 4 * (size_t)H.h[l].n;
        if (lv + need <= budget) {
            P.lvl_off[l] = (int)lv;
            lv += need;
        }
    }
    P.total = (int)std::max(std::max(tri, lv), (size_t)kDotChunk);
    return P;
}

size_t phi_smem_bytes(const DevHier& H) { return (size_t)phi_smem_plan(H).total * 8; }

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
    return std::max(1, std::min(want, per_sm * n_sm));
}

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
    PHI_DEG_DISPATCH(degree_of(H.A), r = occupancy_grid(phi_wave_kernel<DEG>, phi_smem_bytes(H), 1 << 30));
    return r;
}

void launch_phi_wave(const DevHier& H, const DevStencil& Am, const WaveArgs& a, double* ws, long long ws_stride,
                     int max_slots, cudaStream_t s) {
    if (a.n_tasks <= 0) return;
    const SmemPlan P = phi_smem_plan(H);
    const size_t smem = (size_t)P.total * 8;
    const int grid = std::min(a.n_tasks, max_slots);
    PHI_DEG_DISPATCH(degree_of(H.A), {
        occupancy_grid(phi_wave_kernel<DEG>, smem, grid);
        phi_wave_kernel<DEG><<<grid, NT, smem, s>>>(H, Am, a, P, ws, ws_stride);
    });
    PHI_CUDA(cudaGetLastError());
}

void launch_vcycle(const DevHier& H, const double* B, long long ldb, double* X, long long ldx, int nrhs, double* ws,
                   long long ws_stride, int max_slots, cudaStream_t s) {
    if (nrhs <= 0) return;
    const SmemPlan P = phi_smem_plan(H);
    const size_t smem = (size_t)P.total * 8;
    const int grid = std::min(nrhs, max_slots);
    PHI_DEG_DISPATCH(degree_of(H.A), {
        occupancy_grid(vcycle_kernel<DEG>, smem, grid);
        vcycle_kernel<DEG><<<grid, NT, smem, s>>>(H, B, ldb, X, ldx, nrhs, P, ws, ws_stride);
    });
    PHI_CUDA(cudaGetLastError());
}

void launch_unit(const DevHier& H, int op, int arg, int arg2, const double* in, double* out, double* ws,
                 long long ws_stride, cudaStream_t s) {
    const SmemPlan P = phi_smem_plan(H);
    const size_t smem = (size_t)P.total * 8;
    PHI_DEG_DISPATCH(degree_of(H.A), {
        occupancy_grid(unit_kernel<DEG>, smem, 1);
        unit_kernel<DEG><<<1, NT, smem, s>>>(H, op, arg, arg2, in, out, P, ws, ws_stride);
    });
    PHI_CUDA(cudaGetLastError());
}

void launch_cg(const DevStencil& A, const double* diag, const double* b, double* x, double* work, double rel_tol,
               int max_iter, int* result, cudaStream_t s) {
    PHI_DEG_DISPATCH(degree_of(A), (cg_kernel<DEG><<<1, NT, 0, s>>>(A, diag, b, x, work, rel_tol, max_iter, result)));
    PHI_CUDA(cudaGetLastError());
}

static DevBuf<long long> g_trace;

void phi_set_tuning(int tri_warps, int gs_warps, int sleep_ns) {
    Tuning t{std::max(1, std::min(tri_warps, NW)), std::max(1, std::min(gs_warps, NW)), std::max(0, sleep_ns), 0,
             nullptr};
    if (sleep_ns < 0) {  // negative: enable the block-timing trace
        g_trace.alloc((size_t)NW * 1024 * 6);
        g_trace.zero();
        t.trace = g_trace.get();
        t.sleep_ns = 0;
    }
    PHI_CUDA(cudaMemcpyToSymbol(c_tune, &t, sizeof t));
}

int phi_read_trace(long long* out, int n) {
    if (!g_trace.get()) return 0;
    const auto h = g_trace.download();
    const int m = std::min<int>(n, (int)h.size());
    std::copy(h.begin(), h.begin() + m, out);
    return m;
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
    resid0_kernel<<<1, 256, 0, s>>>(g, u, sq, n);
    PHI_CUDA(cudaGetLastError());
}

void launch_copy(double* dst, const double* src, size_t n, cudaStream_t s) {
    if (!n) return;
    const int grid = (int)std::min<size_t>((n + 255) / 256, 4096);
    copy_kernel<<<grid, 256, 0, s>>>(dst, src, n);
    PHI_CUDA(cudaGetLastError());
}

}  // namespace phi
