#pragma once
// Device code of the batched time-stepping operator Phi on B200 (sm_100a).
// Included by phi_deg.cu, which is compiled once per spline degree
// (-DPHI_DEG=1..8) so the degree-templated kernels build in parallel.
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
//  * data-parallel steps (stencil products, transfers, residuals) use all
//    warps of the CTA; the sequential sweeps (triangular solves, Gauss-Seidel)
//    run on ONE warp, one row per lane, so consecutive levels / wavefronts are
//    separated by __syncwarp() instead of CTA barriers;
//  * triangular-factor levels stream through shared memory by TMA bulk copies
//    (cp.async.bulk + mbarrier), several levels ahead of the solving warp;
//  * divisions on the critical path use a stored round-to-nearest reciprocal
//    and two Markstein corrections (fma), which return the correctly rounded
//    quotient -- the same bits as the reference's `/`;
//  * the dependency arrays and the order-1 h-levels live in shared memory when
//    they fit (SmemPlan), so the critical path runs at shared-memory latency;
//  * index-ordered dot products stage the products in shared memory and one
//    thread sums them in order.
#include <cuda_pipeline.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <vector>

#include "device_types.cuh"
#include "phi_kernels.cuh"
#include "setup_host.hpp"

namespace phi {

namespace {

constexpr int NT = kPhiThreads;
constexpr int NW = NT / 32;
constexpr int kDotChunk = 2048;  // doubles of shared scratch for ordered dots
constexpr int kDotThreads = 256;  // threads that form a reassociated dot product's partial sums
static_assert(NT >= kDotThreads && NT % 32 == 0, "a Phi CTA has at least the dot product's threads");

// Dynamic shared memory of every Phi kernel (laid out by SmemPlan).
extern __shared__ __align__(16) double g_smem[];

// Runtime tuning of the sync-free sweeps (developer knob, phi_dev_tuning).
struct Tuning {
    int xmask;      // developer timing experiments (phi_dev_tuning 1st arg; 0 = normal)
    int gs_warps;   // warps taking part in a Gauss-Seidel sweep (<= NW)
    int sleep_ns;   // back-off between failed readiness polls (0 = spin)
    int pad;
    long long* trace;  // developer timing trace of triangular-solve blocks (null = off)
};
__constant__ Tuning c_tune = {0, NW, 0, 0, nullptr};

// Explicit 32-bit shared-window accesses.  Deriving shared pointers inside hot
// loops makes the compiler re-read the window base (S2R SR_SWINHI /
// SR_CgaCtaId) per access; these take the address once, up front.
__device__ __forceinline__ unsigned sh_addr(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ double lds_f64(unsigned a) {
    double v;
    asm("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
    return v;
}
// Volatile variants: kept in program order relative to each other, so a load
// placed ahead of its use stays ahead (the scheduler may otherwise sink loads
// next to their uses under register pressure and serialise a chain).
__device__ __forceinline__ double vlds_f64(unsigned a) {
    double v;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ int vlds_s32(unsigned a) {
    int v;
    asm volatile("ld.shared.s32 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ int vlds_u16(unsigned a) {
    unsigned short v;
    asm volatile("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(a));
    return (int)v;
}
__device__ __forceinline__ int lds_s32(unsigned a) {
    int v;
    asm("ld.shared.s32 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
}
// Developer phase stamps (trace enabled, CTA 0, thread 0): (id, clock64) pairs
// after a counter at trace[kStampBase].
#ifndef PHI_TRACE_ON
#define PHI_TRACE_ON 0  // developer timing stamps (build with PHI_TRACE=1)
#endif
constexpr bool kTrace = PHI_TRACE_ON != 0;
constexpr int kStampBase = 40000, kStampMax = 4000;
constexpr int kTriTraceBase = 24000;  // 4 x 2048 stamps (< kStampBase)
constexpr int kAccBase = 33000;       // developer phase accumulators (wcycle)
__device__ __forceinline__ void pstamp(int id) {
    if (kTrace && c_tune.trace && blockIdx.x == 0 && threadIdx.x == 0) {
        const unsigned long long k = atomicAdd(reinterpret_cast<unsigned long long*>(c_tune.trace + kStampBase), 1ULL);
        if (k < kStampMax) {
            c_tune.trace[kStampBase + 1 + 2 * k] = id;
            c_tune.trace[kStampBase + 2 + 2 * k] = clock64();
        }
    }
}

// Butterfly sum of an fp64 value over aligned groups of 2^lg lanes (lg in
// 1..5, uniform across the warp): raw shfl.sync.bfly on the two halves, with
// no divergence checks; the group count is dispatched once.
__device__ __forceinline__ double shfl_bfly(double v, int o) {
    unsigned lo, hi;
    asm("mov.b64 {%0, %1}, %2;" : "=r"(lo), "=r"(hi) : "d"(v));
    asm volatile("shfl.sync.bfly.b32 %0, %0, %1, 0x1f, 0xffffffff;" : "+r"(lo) : "r"(o));
    asm volatile("shfl.sync.bfly.b32 %0, %0, %1, 0x1f, 0xffffffff;" : "+r"(hi) : "r"(o));
    double r;
    asm("mov.b64 %0, {%1, %2};" : "=d"(r) : "r"(lo), "r"(hi));
    return r;
}
__device__ __forceinline__ double bfly_sum(double t, int lg) {
    switch (lg) {
        case 5: t = t + shfl_bfly(t, 16); [[fallthrough]];
        case 4: t = t + shfl_bfly(t, 8); [[fallthrough]];
        case 3: t = t + shfl_bfly(t, 4); [[fallthrough]];
        case 2: t = t + shfl_bfly(t, 2); [[fallthrough]];
        default: t = t + shfl_bfly(t, 1);
    }
    return t;
}

// Correctly rounded s / d from r = RN(1 / d): q0 = RN(s r) is within two ulps,
// the first Markstein step brings it within one ulp and the second one then
// yields RN(s / d) exactly (residual s - d q exact by fma; valid without
// overflow / underflow, which the solver's operands never approach).  A zero
// numerator keeps the sign rules of IEEE division via q0 itself.
__device__ __forceinline__ double div_rn(double s, double d, double r) {
    const double q0 = s * r;
    const double e0 = __fma_rn(-q0, d, s);
    const double q1 = __fma_rn(e0, r, q0);
    const double e1 = __fma_rn(-q1, d, s);
    const double q2 = __fma_rn(e1, r, q1);
    return s == 0.0 ? q0 : q2;
}

// ---------------------------------------------------------------------------
// Thread-block clusters (single-right-hand-side waves, reassociated mode):
// the CTAs of a cluster run the same Phi application in lock step.  The
// data-parallel phases (operator products, copies, epilogues) are split over
// the CTAs by row (part = cluster rank); the sweeps and the W-cycle run on the
// main CTA (rank 0) while the others wait at the next cluster barrier.  Dot
// products are computed by every CTA over the whole vector (same code, same
// data: identical control decisions).  Without clusters rank = 0, size = 1.
// ---------------------------------------------------------------------------
__shared__ int g_cl[2];  // cluster rank, cluster size
__device__ __forceinline__ void cl_init() {
    if (threadIdx.x == 0) {
        unsigned r, n;
        asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
        asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(n));
        g_cl[0] = (int)r;
        g_cl[1] = (int)n;
    }
}
__device__ __forceinline__ int cl_rank() { return g_cl[0]; }
__device__ __forceinline__ int cl_size() { return g_cl[1]; }
// barrier of every thread of the cluster (memory ordered at cluster scope)
__device__ __forceinline__ void cl_sync() {
    if (g_cl[1] > 1) {
        asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
        asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
    } else {
        __syncthreads();
    }
}
// generic pointer to the main CTA's copy of a shared-memory address
__device__ __forceinline__ double* cl_main(double* p) {
    if (g_cl[1] <= 1 || !__isShared(p)) return p;
    unsigned long long out;
    asm volatile("mapa.u64 %0, %1, 0;" : "=l"(out) : "l"(reinterpret_cast<unsigned long long>(p)));
    return reinterpret_cast<double*>(out);
}

// ---------------------------------------------------------------------------
// per-CTA workspace (generic pointers: shared memory or global per SmemPlan)
// ---------------------------------------------------------------------------
struct Ws {
    // cluster-visible views of the vectors that live in the main CTA's shared
    // memory (z and the first h-level's b, x); equal to z / hb[0] / hx[0] when
    // the kernel runs without clusters
    double *zc, *hb0c, *hx0c;
    double* hbc[kMaxH];
    double* hxc[kMaxH];
    double* hrc[kMaxH];
    double *b, *x, *r, *zg;  // global
    double *cgp, *cgq;       // global: the CG kind's search direction and its product
    double* z;               // in-place triangular-solve vector (n_p + 1 slots)
    double* dot;             // shared scratch for ordered dots
    int z_off, ring_off, slot_bytes, prod_off;  // g_smem offsets (-1: global)
    int n_slots, gs_slot_bytes, gs_n_slots;     // block-sweep rings (SmemPlan)
    int cl_scr_off;                             // cluster dense-apply scratch (SmemPlan), -1: none
    int win_off;                                // rolling window of the ILUT substitutions (SmemPlan), -1: none
    int lvl_off[kMaxH];  // g_smem offset of level l's vectors (b, x, r), -1: global
    double* hb[kMaxH];
    double* hx[kMaxH];
    double* hr[kMaxH];
};

__device__ Ws carve(double* base, const DevHier& H, const SmemPlan& P, double* smem) {
    Ws w;
    const size_t np = (size_t)H.n_p + 2;  // room for the dummy slot z[n]
    w.b = base;
    w.x = base + np;
    w.r = base + 2 * np;
    w.zg = base + 3 * np;
    w.cgp = base + 4 * np;  // the CG kind's plan keeps z in shared memory or unused
    w.cgq = base + 5 * np;
    w.z = P.z_off >= 0 ? smem + P.z_off : base + 4 * np;
    w.dot = smem + P.dot_off;
    w.z_off = P.z_off;
    w.ring_off = P.ring_off;
    w.slot_bytes = P.slot_bytes;
    w.prod_off = P.prod_off;
    w.n_slots = P.n_slots;
    w.gs_slot_bytes = P.gs_slot_bytes;
    w.gs_n_slots = P.gs_n_slots;
    w.cl_scr_off = P.cl_scr_off;
    w.win_off = P.win_off;
    double* g = base + 6 * np;
    for (int l = 0; l < H.n_h; ++l) {
        const int nl = H.h[l].n;
        w.lvl_off[l] = P.lvl_off[l];
        double* s = P.lvl_off[l] >= 0 ? smem + P.lvl_off[l] : g;
        w.hb[l] = s;
        w.hx[l] = s + nl;
        w.hr[l] = s + 2 * (size_t)nl + 1;  // x has a zero slot x[n] (padded sweep entries)
        g += 3 * (size_t)nl + 1;
    }
    w.zc = cl_main(w.z);
    if (H.n_h == 0) return w;  // CG kind: no hierarchy
    w.hb0c = cl_main(w.hb[0]);
    w.hx0c = cl_main(w.hx[0]);
    for (int l = 0; l < H.n_h; ++l) {
        w.hbc[l] = cl_main(w.hb[l]);
        w.hxc[l] = cl_main(w.hx[l]);
        w.hrc[l] = cl_main(w.hr[l]);
    }
    return w;
}

// The hierarchy descriptor (and the wave description) are read from shared
// memory: as kernel parameters their fields are loop-invariant, and the
// compiler hoists them into registers for the whole solve -- about 150
// registers that the sweep loops then lack.  Shared-memory copies are
// re-read after each barrier instead.
__device__ __forceinline__ const DevHier& hier_shared(const DevHier& H) {
    __shared__ DevHier h_sh;
    if (threadIdx.x == 0) h_sh = H;
    __syncthreads();
    return h_sh;
}

// The workspace descriptor lives in shared memory: held in registers it would
// stay live across every call of the solve (about a hundred registers) and
// starve the register allocation of the sweep loops.
__device__ __forceinline__ const Ws& carve_shared(double* base, const DevHier& H, const SmemPlan& P, double* smem) {
    __shared__ Ws ws_sh;
    if (threadIdx.x == 0) ws_sh = carve(base, H, P, smem);
    __syncthreads();
    return ws_sh;
}

// ---------------------------------------------------------------------------
// CTA-cooperative primitives.  Callers place __syncthreads() between phases.
// ---------------------------------------------------------------------------
enum StencilOut : int { kOutSet = 0, kOutResid = 1, kOutScale = 2, kOutAddScaled = 3, kOutAddVec = 4 };

// y[i] (op)= sum_e vals[e][i] * x[col(i, e)], entries in reference CSR order
// (dv, du ascending), one sequential sum per row; the W loads of a stencil
// row are issued together.
// Pairwise sum of N compile-time-indexed values (reassociated mode).
template <int N>
struct Tree {
    static __device__ __forceinline__ double sum(const double* p) {
        return Tree<N / 2>::sum(p) + Tree<N - N / 2>::sum(p + N / 2);
    }
};
template <>
struct Tree<1> {
    static __device__ __forceinline__ double sum(const double* p) { return p[0]; }
};

// Reassociated mode: every row issues all of its loads at clamped (in-range)
// addresses, without branches (entries outside the column grid are selected
// to zero), in chunks of DVC stencil rows -- enough loads in flight per thread
// to cover the L2 latency -- and sums them by a tree per stencil row.
template <int OUT, int W>
__device__ __noinline__ void stencil_apply_fast(const DevStencil& A, const double* __restrict__ x,
                                                double* __restrict__ y, const double* __restrict__ aux, int part,
                                                int parts) {
    constexpr int DVC = W * W <= 25 ? W : (24 / W > 0 ? 24 / W : 1);
    const int n = A.ru * A.rv;
    for (int i = threadIdx.x + part * NT; i < n; i += NT * parts) {
        const int iv = i / A.ru;
        const int iu = i - iv * A.ru;
        int cu_[W];
        bool okq[W];
#pragma unroll
        for (int q = 0; q < W; ++q) {
            const int c = iu + A.lo + q;
            okq[q] = c >= 0 && c < A.cu;
            cu_[q] = min(max(c, 0), A.cu - 1);
        }
        double s = 0.0;
#pragma unroll
        for (int d0 = 0; d0 < W; d0 += DVC) {
            double pv[DVC][W], px[DVC][W];
#pragma unroll
            for (int a = 0; a < DVC; ++a) {
                if (d0 + a < W) {
                    const int r = iv + A.lo + d0 + a;
                    const bool okr = r >= 0 && r < A.cv;
                    const int rv = min(max(r, 0), A.cv - 1);
                    const double* vr = A.vals + (size_t)((d0 + a) * W) * n + i;
                    const double* xr = x + (size_t)rv * A.cu;
#pragma unroll
                    for (int q = 0; q < W; ++q) {
                        const double v = __ldg(vr + (size_t)q * n);
                        pv[a][q] = okr && okq[q] ? v : 0.0;  // entries outside the column grid
                        px[a][q] = xr[cu_[q]];
                    }
                }
            }
#pragma unroll
            for (int a = 0; a < DVC; ++a) {
                if (d0 + a < W) {
                    double pr[W];
#pragma unroll
                    for (int q = 0; q < W; ++q) pr[q] = pv[a][q] * px[a][q];
                    s = s + Tree<W>::sum(pr);
                }
            }
        }
        if (OUT == kOutSet) y[i] = s;
        if (OUT == kOutResid) y[i] = aux[i] - s;             // r = b - A x
        if (OUT == kOutScale) y[i] = s * aux[i];             // (P^T r) .* 1/M^L
        if (OUT == kOutAddScaled) y[i] = y[i] + s * aux[i];  // x += (P e) .* 1/M^L
        if (OUT == kOutAddVec) y[i] = s + aux[i];            // rhs = A- u + load
    }
}

// part / parts: rows interleaved over the CTAs of a cluster (fast mode only)
template <int OUT, int W>
__device__ __noinline__ void stencil_apply(const DevStencil& A, const double* __restrict__ x,
                                           double* __restrict__ y, const double* __restrict__ aux, bool exact = true,
                                           int part = 0, int parts = 1) {
    if (!exact) {
        stencil_apply_fast<OUT, W>(A, x, y, aux, part, parts);
        return;
    }
    const int n = A.ru * A.rv;
    for (int i = threadIdx.x; i < n; i += NT) {
        const int iv = i / A.ru;
        const int iu = i - iv * A.ru;
        const int dulo = max(A.lo, -iu), duhi = min(A.hi, A.cu - 1 - iu);
        const int dvlo = max(A.lo, -iv), dvhi = min(A.hi, A.cv - 1 - iv);
        double s = 0.0, s2 = 0.0;
        for (int dv = dvlo; dv <= dvhi; ++dv) {
            const double* vr = A.vals + (size_t)((dv - A.lo) * W) * n + i;
            const double* xr = x + (size_t)(iv + dv) * A.cu + iu;
            double pv[W], px[W];
#pragma unroll
            for (int q = 0; q < W; ++q) {
                const int du = A.lo + q;
                const bool ok = du >= dulo && du <= duhi;
                pv[q] = ok ? __ldg(vr + (size_t)q * n) : 0.0;
                px[q] = ok ? xr[du] : 0.0;
            }
            if (exact) {  // the reference's order: (dv, du) ascending, valid entries only
#pragma unroll
                for (int q = 0; q < W; ++q) {
                    const int du = A.lo + q;
                    if (du >= dulo && du <= duhi) s = s + pv[q] * px[q];
                }
            } else {  // reassociated: a tree per stencil row, two row accumulators
                double pr[W];
#pragma unroll
                for (int q = 0; q < W; ++q) pr[q] = pv[q] * px[q];
                const double g = Tree<W>::sum(pr);
                if ((dv - dvlo) & 1)
                    s2 = s2 + g;
                else
                    s = s + g;
            }
        }
        if (!exact) s = s + s2;
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
__device__ __forceinline__ void csr_apply(const DevCsr& A, const double* __restrict__ x, double* __restrict__ y,
                                          int part = 0, int parts = 1) {
    for (int i = threadIdx.x + part * NT; i < A.n_rows; i += NT * parts) {
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

// ---- triangular solves: one warp, TMA-fed ------------------------
// The factor is one level-ordered stream of blocks (TriStream), packed into
// fetch units.  A ring of kTriSlots shared-memory slots is filled by TMA bulk
// copies (cp.async.bulk + mbarrier complete_tx), kTriSlots-1 units ahead; the
// next unit's address travels in the header of the unit being consumed.
__device__ __forceinline__ void mbar_init(unsigned bar) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void bulk_fetch(unsigned dst, const void* src, int bytes, unsigned bar) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                 "l"(src), "r"(bytes), "r"(bar)
                 : "memory");
}
#ifndef PHI_SPIN_GUARD
#define PHI_SPIN_GUARD 1  // bounded spins: report and trap instead of hanging
#endif
__device__ __noinline__ void spin_fail(int what, int have, int want);
__device__ __forceinline__ void mbar_wait(unsigned bar, unsigned parity) {
    unsigned done;
    const long long t0 = PHI_SPIN_GUARD ? clock64() : 0;
    do {
        if (PHI_SPIN_GUARD && clock64() - t0 > 4000000000LL) spin_fail(3, (int)(bar & 0xffff), (int)parity);
        asm volatile(
            "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
            : "=r"(done)
            : "r"(bar), "r"(parity)
            : "memory");
    } while (!done);
}

// In-place substitution with an ILUT factor (ilut.hpp:146-163) on z, which
// holds the right-hand side on entry.  Lower: z_i -= sum_j L_ij z_j (unit
// diagonal).  Upper: z_i = (z_i - sum_j U_ij z_j) / U_ii.  Executed by ONE
// warp, block by block (a block holds the rows of one level, or a slice of a
// wide level; every z_j it reads belongs to an earlier block):
//  exact: 1. all 32 lanes form the block's products into shared scratch;
//         2. lane l subtracts row l's products in CSR order -- the
//            reference's exact sequence of roundings -- and publishes z_i;
//  fast:  G = 2^lg lanes per row (chosen per block on the host); each lane
//         sums its contiguous slice of the row with two accumulators, a
//         butterfly over the G lanes completes the sum, and the row's first
//         lane publishes z_i (division by the stored reciprocal).
// __syncwarp() (a memory barrier among the lanes) closes each block.  Padded
// entries (column n, value +0.0; z[n] = +0.0) are exactly neutral.
template <bool UPPER, bool ZSM, bool EXACT>
__device__ __noinline__ void tri_solve_warp_t(const DevTri& T, double* zg, int z_off, const double* rg, int r_off,
                                              int ring_off, int slot_bytes, int prod_off, unsigned bar) {
    const int lane = threadIdx.x & 31;
    const int xm = c_tune.xmask;  // developer experiments, 0 in production
    const unsigned ring = sh_addr(g_smem + ring_off);
    const unsigned prod = sh_addr(g_smem + prod_off);
    const unsigned zs = ZSM ? sh_addr(g_smem + z_off) : 0u;
    // right-hand side of row i: z_i itself (in-place ILUT substitution) or a
    // separate vector (Gauss-Seidel: b_i), shared (ZSM) or global
    const unsigned rs = ZSM ? sh_addr(g_smem + r_off) : 0u;
    // cached: T lives in the kernel parameter space (generic loads otherwise)
    const int n_units = T.n_units;
    const unsigned char* __restrict__ stream = T.stream;
    if (lane == 0)
        for (int k = 0; k < kTriSlots - 1 && k < n_units; ++k)
            bulk_fetch(ring + k * slot_bytes, stream + (size_t)T.prime[2 * k] * 16, T.prime[2 * k + 1],
                       bar + 8u * k);
    // developer trace (CTA 0, lane 0, first 1024 blocks): block start, data
    // ready, row sums done, block done, -, products / accumulation done --
    // at trace[kTriTraceBase + 8 b]
    long long* tr = (kTrace && c_tune.trace && blockIdx.x == 0 && lane == 0) ? c_tune.trace + kTriTraceBase : nullptr;
    int b = 0;
    for (int u = 0; u < n_units; ++u) {
        const int slot = u % kTriSlots;
        if (tr && b < 1024) tr[8 * b] = clock64();
        mbar_wait(bar + 8u * slot, (unsigned)(u / kTriSlots) & 1u);
        const unsigned unit = ring + slot * slot_bytes;
        int nblk, next_off, next_bytes, upad;
        asm volatile("ld.shared.v4.s32 {%0, %1, %2, %3}, [%4];"
                     : "=r"(nblk), "=r"(next_off), "=r"(next_bytes), "=r"(upad)
                     : "r"(unit));
        (void)upad;
        // unit u + kTriSlots - 1 refills the slot the warp left after unit u - 1
        if (lane == 0 && next_bytes > 0) {
            const int ns = (u + kTriSlots - 1) % kTriSlots;
            bulk_fetch(ring + ns * slot_bytes, stream + (size_t)next_off * 16, next_bytes, bar + 8u * ns);
        }
        unsigned blk = unit + 16u + ((2u * nblk + 15u) & ~15u);  // after the block-offset table
        for (int kb = 0; kb < nblk; ++kb, ++b) {
            if (tr && b < 1024) {
                if (kb) tr[8 * b] = clock64();
                tr[8 * b + 1] = clock64();
            }
            int nr, per, lg, bytes, cols_off, vals_off, diag_off, bpad;
            asm volatile("ld.shared.v4.s32 {%0, %1, %2, %3}, [%4];"
                         : "=r"(nr), "=r"(per), "=r"(lg), "=r"(bytes)
                         : "r"(blk));
            asm volatile("ld.shared.v4.s32 {%0, %1, %2, %3}, [%4];"
                         : "=r"(cols_off), "=r"(vals_off), "=r"(diag_off), "=r"(bpad)
                         : "r"(blk + 16));
            (void)bpad;
            const unsigned cols = blk + cols_off, vals = blk + vals_off;
            double s = 0.0;
            if constexpr (EXACT) {
                const int span = per;
                int i = 0;
                double dg = 1.0, rd = 1.0;
                if (lane < nr) {  // row data first: its latency overlaps phase 1
                    i = lds_s32(blk + 32u + 4u * lane);
                    s = ZSM ? lds_f64(rs + 8u * i) : rg[i];
                    if (UPPER) {
                        const unsigned dp = blk + diag_off + 8u * lane;
                        dg = lds_f64(dp);
                        rd = lds_f64(dp + 8u * nr);
                    }
                }
                // phase 1: all lanes form the block's products into shared scratch
                const int items = nr * span;
                for (int t0 = 0; t0 < items; t0 += 128) {
                    int j[4];
                    double v[4], zj[4];
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const int t = min(t0 + q * 32 + lane, items - 1);
                        j[q] = lds_s32(cols + 4u * t);
                        v[q] = lds_f64(vals + 8u * t);
                    }
#pragma unroll
                    for (int q = 0; q < 4; ++q) zj[q] = ZSM ? lds_f64(zs + 8u * j[q]) : zg[j[q]];
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const int t = t0 + q * 32 + lane;
                        if (t < items)
                            asm volatile("st.shared.f64 [%0], %1;" ::"r"(prod + 8u * t), "d"(v[q] * zj[q]) : "memory");
                    }
                }
                __syncwarp();
                if (tr && b < 1024) tr[8 * b + 5] = clock64();
                // phase 2: lane l subtracts row l's products in CSR order
                if (lane < nr) {
                    const unsigned pp = prod + 8u * lane, st = 8u * nr;
                    int e = 0;
                    for (; e + 8 <= span; e += 8) {
                        double pq[8];
#pragma unroll
                        for (int q = 0; q < 8; ++q) pq[q] = lds_f64(pp + (e + q) * st);
#pragma unroll
                        for (int q = 0; q < 8; ++q) s = s - pq[q];
                    }
                    for (; e < span; e += 2) {  // span is even
                        const double p0 = lds_f64(pp + e * st), p1 = lds_f64(pp + (e + 1) * st);
                        s = s - p0;
                        s = s - p1;
                    }
                    if (UPPER) s = div_rn(s, dg, rd);
                    if (ZSM)
                        asm volatile("st.shared.f64 [%0], %1;" ::"r"(zs + 8u * i), "d"(s) : "memory");
                    else
                        zg[i] = s;
                }
                if (tr && b < 1024) tr[8 * b + 2] = clock64();
            } else {
                const int m = per;
                // per-lane tables: the row index on a row's first lane (-1
                // elsewhere) and its reciprocal diagonal
                const int i = lds_s32(blk + 32u + 4u * lane);
                const bool head = i >= 0;
                double rd = 1.0, z0 = 0.0;
                if (head) {
                    z0 = ZSM ? lds_f64(rs + 8u * i) : rg[i];
                    if (UPPER) rd = lds_f64(blk + diag_off + 8u * lane);
                }
                // slice sums: slot q of every lane is one conflict-free load
                // (entry-major layout), in batches of 8 slots
                double t = 0.0;
                {
                    const unsigned cp = cols + 4u * lane, vp = vals + 8u * lane;
                    double a0 = 0.0, a1 = 0.0;
                    for (int q0 = 0; q0 < m; q0 += 8) {  // m: whole batches of 8 (host-padded)
                        int j[8];
                        double v[8], zj[8];
#pragma unroll
                        for (int q = 0; q < 8; ++q) {
                            j[q] = lds_s32(cp + 128u * (q0 + q));
                            v[q] = lds_f64(vp + 256u * (q0 + q));
                        }
#pragma unroll
                        for (int q = 0; q < 8; ++q)
                            zj[q] = (xm & 2) ? 1.0 : (ZSM ? lds_f64(zs + 8u * j[q]) : zg[j[q]]);
                        double pr[8];
#pragma unroll
                        for (int q = 0; q < 8; ++q) pr[q] = v[q] * zj[q];
                        a0 = a0 + ((pr[0] + pr[1]) + (pr[2] + pr[3]));
                        a1 = a1 + ((pr[4] + pr[5]) + (pr[6] + pr[7]));
                    }
                    t = a0 + a1;  // idle lanes hold zero slots
                }
                if (tr && b < 1024) tr[8 * b + 5] = clock64() + (long long)(t == 12345.678);
                if (!(xm & 1) && lg > 0) t = bfly_sum(t, lg);
                if (tr && b < 1024) tr[8 * b + 2] = clock64();
                if (head) {
                    s = z0 - t;
                    if (UPPER) s = s * rd;  // reassociated mode: within one ulp of the quotient
                    if (ZSM)
                        asm volatile("st.shared.f64 [%0], %1;" ::"r"(zs + 8u * i), "d"(s) : "memory");
                    else
                        zg[i] = s;
                }
            }
            __syncwarp();
            if (tr && b < 1024) tr[8 * b + 3] = clock64() + (long long)(s == 12345.678);
            blk += bytes;
        }
    }
}

// Warps that meet at the closing barrier of an exact-mode sweep.
constexpr int kSW = kSweepWarps;
constexpr int kSweepBar = kSW + 1;  // named barrier of all sweep warps
__device__ __forceinline__ void sweep_sync() { asm volatile("bar.sync %0, %1;" ::"r"(kSweepBar), "r"(32 * kSW) : "memory"); }

template <bool UPPER, bool ZSM>
__device__ __forceinline__ void tri_solve_warp(const DevTri& T, double* zg, int z_off, const double* rg, int r_off,
                                               int ring_off, int slot_bytes, int prod_off, unsigned bar, bool exact) {
    // exact mode only (the reassociated mode runs block sweeps): warp 0 solves
    (void)exact;
    if (threadIdx.x < 32)
        tri_solve_warp_t<UPPER, ZSM, true>(T, zg, z_off, rg, r_off, ring_off, slot_bytes, prod_off, bar);
    sweep_sync();  // all sweep warps done (the next sweep reuses the ring and mbarriers)
}

// ---- block-recurrence sweeps (reassociated mode) ---------------------------
// `count` consecutive sweeps (ILUT substitution or Gauss-Seidel) over one
// BlkStream (setup_host.hpp): blocks of 32 consecutive rows in solve order,
// block k solved as x_{R_k} = B_k^{-1} (rhs - old) - G_k x_{R_{k-1}} with the
// folded coupling G_k = B_k^{-1} N_k to block k-1.  The blocks of the `count`
// sweeps form one sequence g = s * nb + k.
//  * the solver warps take the blocks in rotation.  Per block a solver waits
//    until the workers' old sums are in and -- none of it depending on block
//    g-1 -- broadcasts rhs - old through shared memory, multiplies by the
//    dense inverse and loads G_k into registers; only then does it wait for
//    block g-1, whose last 8 mf values (in solve order, sy.xb) it multiplies
//    by G_k: the block-to-block critical path is the hand-off, 4 mf 16-byte
//    loads and 8 mf fused multiply-adds in four chains (fold_block);
//  * the other warps (the workers) each sum one interleaved part of the
//    block's old entries as soon as block g-2 is done (and, for a later
//    sweep, the previous sweep's rows they read), one block ahead of the
//    solver.
// The blocks stream through a shared-memory ring of n_slots units filled by
// TMA bulk copies: the workers wait for a unit's mbarrier, the solver
// refills the slot of block g (with block g + n_slots) once block g is done.
// Hand-offs are shared-memory flags with release / acquire semantics at CTA
// scope: `prog` (last block done, st.release after the block's values) and
// cnt[g % kBlkHand] (parts of block g summed, red.release.add); waiters spin
// with ld.acquire.  __syncwarp() orders the lanes' data stores before the
// releasing lane's flag update; a global-memory vector is fenced
// (__threadfence_block) before its flag.
__device__ __forceinline__ void st_volatile_s32(unsigned a, int v) {
    asm volatile("st.volatile.shared.b32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
__device__ __forceinline__ int ld_volatile_s32(unsigned a) {
    int v;
    asm volatile("ld.volatile.shared.b32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_s32(unsigned a, int v) {
    asm volatile("st.release.cta.shared.b32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
__device__ __forceinline__ int ld_acquire_s32(unsigned a) {
    int v;
    asm volatile("ld.acquire.cta.shared.b32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
    return v;
}
__device__ __forceinline__ void red_release_add(unsigned a, int v) {
    asm volatile("red.release.cta.shared.add.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
__device__ __noinline__ void spin_fail(int what, int have, int want) {
    printf("phi spin guard: block %d thread %d wait %d have %d want %d\n", blockIdx.x, threadIdx.x, what, have, want);
    __trap();
}
// spin until *a >= v; returns the value seen
__device__ __forceinline__ int wait_ge(unsigned a, int v) {
    int h = ld_acquire_s32(a);
    if (h >= v) return h;
    const long long t0 = PHI_SPIN_GUARD ? clock64() : 0;
    while ((h = ld_acquire_s32(a)) < v)
        if (PHI_SPIN_GUARD && clock64() - t0 > 4000000000LL) spin_fail(1, h, v);
    return h;
}
// x[j]: shared (XSM: byte address base + 8 j) or global
template <bool XSM>
__device__ __forceinline__ double xld(const double* xg, unsigned xs, int j) {
    if constexpr (XSM)
        return vlds_f64(xs + 8u * j);
    else
        return *reinterpret_cast<const volatile double*>(xg + j);
}
template <bool XSM>
__device__ __forceinline__ void xst(double* xg, unsigned xs, int j, double v) {
    if constexpr (XSM)
        asm volatile("st.shared.f64 [%0], %1;" ::"r"(xs + 8u * j), "d"(v) : "memory");
    else
        xg[j] = v;
}
__device__ __forceinline__ void lds_v2f64(unsigned a, double& x, double& y) {
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(x), "=d"(y) : "r"(a));
}
// predicated pair load: {x, y} = on ? [a] : {0, 0} (the load is not issued for the other lanes)
__device__ __forceinline__ void lds_v2f64_if(unsigned a, bool on, double& x, double& y) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.s32 p, %3, 0;\n\tmov.f64 %0, 0d0000000000000000;\n\t"
        "mov.f64 %1, 0d0000000000000000;\n\t@p ld.shared.v2.f64 {%0, %1}, [%2];\n\t}"
        : "=&d"(x), "=&d"(y)
        : "r"(a), "r"((int)on));
}
__device__ __forceinline__ void lds_slot(unsigned a, int& c, double& v) {  // {int32 col, pad, double val}
    int pad;
    asm volatile("ld.shared.v4.s32 {%0, %1, %2, %3}, [%4];" : "=r"(c), "=r"(pad), "=r"(reinterpret_cast<int*>(&v)[0]),
                 "=r"(reinterpret_cast<int*>(&v)[1]) : "r"(a));
    (void)pad;
}

struct __align__(16) BlkSync {
    double cbuf[kBlkHand][kBlkMaxParts][32];  // workers' partial old sums
    double tb[kBlkSolvers][32];               // per-solver broadcast of rhs - old (16-byte aligned)
    double xb[2][32];                         // block g's values in solve order at xb[g & 1] (the chain's input)
    unsigned long long bar[kBlkMaxSlots];
    int phase[kBlkMaxSlots];  // phases completed per slot since the kernel started
    int cnt[kBlkHand];
    int prog;
};
// One per CTA.  The ring's mbarriers are initialised once per kernel
// (blk_init) and never re-initialised: every sweep continues their phase
// sequence from `phase`.
__shared__ BlkSync g_blk;

__device__ __forceinline__ void blk_init() {
    if (threadIdx.x == 0) {
        const unsigned bar = sh_addr(g_blk.bar);
        for (int k = 0; k < kBlkMaxSlots; ++k) {
            mbar_init(bar + 8u * k);
            g_blk.phase[k] = 0;
        }
        for (int k = 0; k < kBlkHand; ++k) g_blk.cnt[k] = 0;
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    // the callers' next __syncthreads() publishes the initialisation
}

// named barriers of the solver hand-off: block g done -> solver (g + 1) % kBlkSolvers
__device__ __forceinline__ void hand_wait(int id) { asm volatile("bar.sync %0, 64;" ::"r"(id) : "memory"); }
__device__ __forceinline__ void hand_signal(int id) { asm volatile("bar.arrive %0, 64;" ::"r"(id) : "memory"); }
constexpr int kHandBar = 1;  // ids 1 .. kBlkSolvers

// One block of a folded block sweep for NG groups of four column pairs of
// G_k, from the point where the block's unit has landed and its inverse is
// in registers: G_k into registers (before any wait), the workers' old sums,
// y = B^{-1} (rhs - old) through a shared-memory broadcast, y pinned before
// the hand-off wait (nothing but the chain's own loads and fused
// multiply-adds after it), then y - G_k x_{g-1} in four chains.
// Once every part is in, the workers are done with the block's unit, and so
// is this warp (inverse and G_k are in registers): lane 0 refills the ring slot
// right there (refill_bytes > 0) -- a whole inverse product, chain and store
// earlier than after the block, which the TMA stream needs (issuing it ~500
// cycles later cost 20 % of the sweep).
struct BlkRefill {
    unsigned dst, bar;
    const unsigned char* src;
    int bytes;
};
template <int NG>
__device__ __forceinline__ double fold_block(unsigned gp, unsigned xp, const double (&iv)[32], double rhs, unsigned tb,
                                             unsigned cnt_a, int P, unsigned cbuf_a, int lane, int hand_id,
                                             const BlkRefill& rf, long long* tr) {
    double gq[NG > 0 ? 8 * NG : 1];
#pragma unroll
    for (int p2 = 0; p2 < 4 * NG; ++p2) lds_v2f64(gp + 512u * p2, gq[2 * p2], gq[2 * p2 + 1]);
    if (tr) tr[7] = clock64();
    // ---- all parts in: the partial old sums
    const int all = wait_ge(cnt_a, P);
    double part[kBlkMaxParts];
#pragma unroll
    for (int q = 0; q < kBlkMaxParts; ++q)
        part[q] = q < P ? vlds_f64(cbuf_a + 8u * (q * 32 + lane) + (unsigned)(all - P)) : 0.0;
    // the unit is consumed: its slot takes the unit n_slots blocks ahead.  (Every shared load of
    // the unit by this warp has returned -- the acquire load above was issued after them -- and the
    // workers' loads precede their release of the parts.)
    if (lane == 0 && rf.bytes > 0) bulk_fetch(rf.dst, rf.src, rf.bytes, rf.bar);
    double old = 0.0;
#pragma unroll
    for (int q = 0; q < kBlkMaxParts; ++q) old = old + part[q];
    const double c = rhs - old;
    asm volatile("st.shared.f64 [%0], %1;" ::"r"(tb + 8u * lane), "d"(c) : "memory");
    __syncwarp();
    double acc[8];
#pragma unroll
    for (int p2 = 0; p2 < 16; ++p2) {
        double t0, t1;
        lds_v2f64(tb + 16u * p2, t0, t1);
        if (p2 < 4) {
            acc[2 * p2] = iv[2 * p2] * t0;
            acc[2 * p2 + 1] = iv[2 * p2 + 1] * t1;
        } else {
            acc[(2 * p2) & 7] = __fma_rn(iv[2 * p2], t0, acc[(2 * p2) & 7]);
            acc[(2 * p2 + 1) & 7] = __fma_rn(iv[2 * p2 + 1], t1, acc[(2 * p2 + 1) & 7]);
        }
    }
    double y = ((acc[0] + acc[1]) + (acc[2] + acc[3])) + ((acc[4] + acc[5]) + (acc[6] + acc[7]));
    // y is complete before the wait (volatile asm statements keep their order)
    asm volatile("" : "+d"(y));
    if (tr) tr[4] = clock64();
    if (hand_id >= 0) hand_wait(hand_id);
    if (tr) tr[2] = clock64();
    if (NG == 0) return y;
    double f[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
    for (int p2 = 0; p2 < 4 * NG; ++p2) {
        double x0, x1;
        lds_v2f64(xp + 16u * (15 - p2), x0, x1);
        f[(2 * p2) & 3] = __fma_rn(gq[2 * p2], x0, f[(2 * p2) & 3]);
        f[(2 * p2 + 1) & 3] = __fma_rn(gq[2 * p2 + 1], x1, f[(2 * p2 + 1) & 3]);
    }
    return y - ((f[0] + f[1]) + (f[2] + f[3]));
}

// WIN (rolling-window streams, BlkStream::win): x_off is the window, the
// stream's columns are window slots (16-bit for the old entries), solved
// values go to the window slot row & (win - 1) and through to global xg.
template <bool XSM, bool RSM, bool WIN>
__device__ __noinline__ void blk_sweep_t(const DevBlk& T, int count, double* xg, int x_off, const double* rg,
                                         int r_off, int ring_off, int slot_bytes, int n_slots) {
    static_assert(!WIN || (XSM && !RSM), "the window is the shared x; the right-hand side is global");
    BlkSync& sy = g_blk;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int nb = T.n_blocks, P = T.parts, total = count * nb;
    const unsigned ring = sh_addr(g_smem + ring_off);
    const unsigned bar = sh_addr(sy.bar);
    const unsigned xs = XSM ? sh_addr(g_smem + x_off) : 0u;
    const unsigned rs = RSM ? sh_addr(g_smem + r_off) : 0u;
    const unsigned prog = sh_addr(&sy.prog), cnt = sh_addr(sy.cnt), cbuf = sh_addr(sy.cbuf);
    const unsigned char* __restrict__ stream = T.stream;
    const int4* __restrict__ table = T.table;
    constexpr int NS = kBlkSolvers, F = kBlkFresh;
    if (w < NS) {
        // ---- solver warps 0 .. NS-1 take blocks g = w, w + NS, ...  The parts'
        // count implies the block's unit has landed (each worker waited).
        const unsigned tb = sh_addr(sy.tb[w]);
        const unsigned xbs = sh_addr(sy.xb);
        int slot = w % n_slots, k = w % nb;
        int4 info = w < total ? __ldg(table + k) : make_int4(0, 0, 0, 0);  // (off16, bytes, mf, 0)
        int4 refill_next = make_int4(0, 0, 0, 0);
        if (lane == 0 && w + n_slots < total) refill_next = __ldg(table + (k + n_slots) % nb);
        // rows are taken in solve order: lane l of block k solves position 32 k + l
        auto row_of = [&](int kb) {
            const int pos = kb * kBlkRows + lane;
            return pos < T.n ? (T.desc ? T.n - 1 - pos : pos) : -1;
        };
        // a global right-hand side is prefetched one turn ahead (its rows are
        // not written before their own block), off the chain
        double rhs_next = 0.0;
        if constexpr (!RSM) {
            const int r0 = row_of(k);
            if (w < total && r0 >= 0) rhs_next = *reinterpret_cast<const volatile double*>(rg + r0);
        }
        for (int g = w; g < total; g += NS) {
            const int mf = info.z;
            int kn2 = k + NS;  // this solver's next block
            while (kn2 >= nb) kn2 -= nb;
            if (g + NS < total) info = __ldg(table + kn2);
            double rhs_pref = 0.0;
            if constexpr (!RSM) {
                rhs_pref = rhs_next;
                const int rn = row_of(kn2);
                if (g + NS < total && rn >= 0) rhs_next = *reinterpret_cast<const volatile double*>(rg + rn);
            }
            // the unit that refills this block's slot after the block: its
            // table entry was loaded one turn earlier (no L2 latency here)
            const int4 refill = refill_next;
            if (lane == 0 && g + NS + n_slots < total) {
                int kn = kn2 + n_slots;
                while (kn >= nb) kn -= nb;
                refill_next = __ldg(table + kn);
            }
            long long* tr = (kTrace && c_tune.trace && blockIdx.x == 0 && lane == 0 && g < 512)
                                ? c_tune.trace + kTriTraceBase + 16 * g
                                : nullptr;
            if (tr) tr[0] = clock64();
            // one part in: the unit has landed (each worker waited for it)
            const int seen = wait_ge(cnt + 4u * (g & (kBlkHand - 1)), 1);
            if (tr) tr[1] = clock64();
            // data dependence on the wait: none of these loads moves above it
            const unsigned u = ring + slot * slot_bytes + (unsigned)(seen > 0 ? 0 : 1);
            // ---- independent of block g-1: row, rhs, inverse, old sums, y = B^{-1} (rhs - old)
            const int row = RSM ? vlds_s32(u + 16u + 4u * lane) : row_of(k);
            double rhs = rhs_pref;
            if (RSM && row >= 0) rhs = vlds_f64(rs + 8u * row);
            double iv[32];
#pragma unroll
            for (int p2 = 0; p2 < 16; ++p2) {
                if constexpr (kBlkTri)  // lower triangle only: lanes above the diagonal keep exact zeros
                    lds_v2f64_if(u + kBlkInvOff + 16u * (p2 * (31 - p2) + lane), lane >= 2 * p2, iv[2 * p2],
                                 iv[2 * p2 + 1]);
                else
                    lds_v2f64(u + kBlkInvOff + 16u * (p2 * 32 + lane), iv[2 * p2], iv[2 * p2 + 1]);
            }
            // ---- G_k, the old sums, y = B^{-1} (rhs - old), the wait for block
            // g-1 (the previous solver), then the chain x_g = y - G_k x_{g-1}
            // over the last 8 mf values of block g-1 (mf: groups of four column pairs)
            const unsigned gp = u + kBlkFreshOff + 16u * lane;
            const unsigned xp = xbs + 256u * ((g + 1) & 1);
            const int hand_id = g > 0 ? kHandBar + (w == 0 ? NS - 1 : w - 1) : -1;
            const unsigned cnt_a = cnt + 4u * (g & (kBlkHand - 1));
            const unsigned cbuf_a = cbuf + 8u * ((g & (kBlkHand - 1)) * kBlkMaxParts * 32);
            BlkRefill rf{ring + slot * slot_bytes, bar + 8u * slot, stream + (size_t)refill.x * 16,
                         g + n_slots < total ? refill.y : 0};
            double z;
            switch (mf) {
                case 0: z = fold_block<0>(gp, xp, iv, rhs, tb, cnt_a, P, cbuf_a, lane, hand_id, rf, tr); break;
                case 1: z = fold_block<1>(gp, xp, iv, rhs, tb, cnt_a, P, cbuf_a, lane, hand_id, rf, tr); break;
                case 2: z = fold_block<2>(gp, xp, iv, rhs, tb, cnt_a, P, cbuf_a, lane, hand_id, rf, tr); break;
                case 3: z = fold_block<3>(gp, xp, iv, rhs, tb, cnt_a, P, cbuf_a, lane, hand_id, rf, tr); break;
                default: z = fold_block<4>(gp, xp, iv, rhs, tb, cnt_a, P, cbuf_a, lane, hand_id, rf, tr); break;
            }
            if (tr) tr[3] = clock64() + (long long)(z == 1.2345);
            // the values in solve order, for block g+1's chain
            asm volatile("st.shared.f64 [%0], %1;" ::"r"(xbs + 256u * (g & 1) + 8u * lane), "d"(z) : "memory");
            if constexpr (WIN) {
                if (row >= 0) {
                    xst<true>(xg, xs, row & (T.win - 1), z);
                    xg[row] = z;  // write-through: read by the next phases after the sweep
                }
            } else if (row >= 0) {
                xst<XSM>(xg, xs, row, z);
            }
            if constexpr (!XSM) __threadfence_block();  // global x: order the stores before the hand-off
            __syncwarp();
            if (g + 1 < total) hand_signal(kHandBar + w);  // the chain: block g+1 may start
            if (lane == 0) st_release_s32(prog, g);  // monotone; read by the workers (off the chain)
            if (tr) tr[5] = clock64();
            // ---- off the chain: bookkeeping for this solver's next block
            if (lane == 0) st_volatile_s32(cnt + 4u * (g & (kBlkHand - 1)), 0);  // reused by block g + kBlkHand
            if (tr) tr[6] = clock64();
            slot += NS;
            while (slot >= n_slots) slot -= n_slots;
            k = kn2;
        }
    } else if (w - NS < P) {
        // ---- worker q = w - NS: part q of every block's old sums
        const int q = w - NS;
        int k = 0, s = 0, slot = 0, ph = 0;
        for (int g = 0; g < total; ++g) {
            long long* tr = (kTrace && c_tune.trace && blockIdx.x == 0 && lane == 0 && q == 0 && g < 512)
                                ? c_tune.trace + kTriTraceBase + 16 * g
                                : nullptr;
            // columns solved by blocks <= g-F-1 of this sweep; for a later
            // sweep also the previous sweep's rows up to block k + lookahead
            int need = g - F - 1;
            if (s > 0) need = max(need, (s - 1) * nb + min(k + T.lookahead, nb - 1));
            // unit g was issued when block g - n_slots was done: with
            // n_slots >= F + 2 it is in flight already (this worker saw
            // prog >= g - F - 2 for its previous block); a shallower ring
            // waits for `need` first
            if (n_slots < F + 2) wait_ge(prog, need);
            mbar_wait(bar + 8u * slot, (unsigned)(sy.phase[slot] + ph) & 1u);
            if (tr) tr[8] = clock64();
            const unsigned u = ring + slot * slot_bytes;
            const int mo = vlds_s32(u), mf = vlds_s32(u + 12u);
            // part q: columns int32[mo][32] (window: uint16), then values double[mo][32]
            constexpr unsigned CB = WIN ? 2u : 4u;
            const unsigned pb = u + kBlkFreshOff + 2048u * mf + (32u * CB + 256u) * mo * q;
            const unsigned oc = pb + CB * lane;
            const unsigned ov = pb + 32u * CB * mo + 8u * lane;
            const int xpad = WIN ? T.win : T.n;
            auto ldc = [&](int e) { return WIN ? vlds_u16(oc + 32u * CB * e) : vlds_s32(oc + 32u * CB * e); };
            double a0 = 0.0, a1 = 0.0;
            if (mo <= 8) {  // the common case: every load issued before the wait
                int c[8];
                double v[8];
#pragma unroll
                for (int e = 0; e < 8; ++e) {
                    c[e] = e < mo ? ldc(e) : xpad;
                    v[e] = e < mo ? vlds_f64(ov + 256u * e) : 0.0;
                }
                if (tr) tr[9] = clock64();
                wait_ge(prog, need);
                if (tr) tr[10] = clock64();
                double xv[8];
#pragma unroll
                for (int e = 0; e < 8; ++e) xv[e] = e < mo ? xld<XSM>(xg, xs, c[e]) : 0.0;
                a0 = __fma_rn(v[0], xv[0], v[1] * xv[1]) + __fma_rn(v[4], xv[4], v[5] * xv[5]);
                a1 = __fma_rn(v[2], xv[2], v[3] * xv[3]) + __fma_rn(v[6], xv[6], v[7] * xv[7]);
            } else if (mo <= 16) {  // the same with sixteen slots in registers (degree 4 and 5 factors)
                int c[16];
                double v[16];
#pragma unroll
                for (int e = 0; e < 16; ++e) {
                    c[e] = e < mo ? ldc(e) : xpad;
                    v[e] = e < mo ? vlds_f64(ov + 256u * e) : 0.0;
                }
                if (tr) tr[9] = clock64();
                wait_ge(prog, need);
                if (tr) tr[10] = clock64();
                double xv[16];
#pragma unroll
                for (int e = 0; e < 16; ++e) xv[e] = e < mo ? xld<XSM>(xg, xs, c[e]) : 0.0;
                a0 = (__fma_rn(v[0], xv[0], v[1] * xv[1]) + __fma_rn(v[4], xv[4], v[5] * xv[5])) +
                     (__fma_rn(v[8], xv[8], v[9] * xv[9]) + __fma_rn(v[12], xv[12], v[13] * xv[13]));
                a1 = (__fma_rn(v[2], xv[2], v[3] * xv[3]) + __fma_rn(v[6], xv[6], v[7] * xv[7])) +
                     (__fma_rn(v[10], xv[10], v[11] * xv[11]) + __fma_rn(v[14], xv[14], v[15] * xv[15]));
            } else {
                if (tr) tr[9] = clock64();
                wait_ge(prog, need);
                if (tr) tr[10] = clock64();
                for (int e = 0; e < mo; e += 2) {
                    const int c0 = ldc(e), c1 = e + 1 < mo ? ldc(e + 1) : xpad;
                    const double v0 = vlds_f64(ov + 256u * e), v1 = e + 1 < mo ? vlds_f64(ov + 256u * (e + 1)) : 0.0;
                    a0 = __fma_rn(v0, xld<XSM>(xg, xs, c0), a0);
                    a1 = __fma_rn(v1, xld<XSM>(xg, xs, c1), a1);
                }
            }
            asm volatile("st.shared.f64 [%0], %1;" ::"r"(cbuf + 8u * (((g & (kBlkHand - 1)) * kBlkMaxParts + q) * 32 + lane)),
                         "d"(a0 + a1)
                         : "memory");
            __syncwarp();
            if (lane == 0) red_release_add(cnt + 4u * (g & (kBlkHand - 1)), 1);
            if (tr) tr[11] = clock64();
            if (++slot == n_slots) {
                slot = 0;
                ++ph;
            }
            if (++k == nb) {
                k = 0;
                ++s;
            }
        }
    }
}

// `count` sweeps over T: prime, the solver / worker split, closing barrier,
// phase bookkeeping.  Called by the whole CTA (blk_init ran at kernel start).
__device__ __forceinline__ void blk_sweep(const DevBlk& T, int count, double* xg, int x_off, const double* rg,
                                          int r_off, int ring_off, int slot_bytes, int n_slots, int win_off = -1) {
    BlkSync& sy = g_blk;
    const int nb = T.n_blocks, total = count * nb;
    if (total == 0) return;
    // the ring overlays buffers written through the generic proxy in other
    // phases: order those writes before the TMA (async-proxy) writes
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    const bool win = T.win > 0 && win_off >= 0;
    if (threadIdx.x == 0) {
        const unsigned bar = sh_addr(sy.bar);
        sy.prog = -1;
        if (win) g_smem[win_off + T.win] = 0.0;  // the window's zero slot (padding)
        const unsigned ring = sh_addr(g_smem + ring_off);
        for (int g = 0; g < n_slots && g < total; ++g) {
            const int4 e = __ldg(T.table + g % nb);
            bulk_fetch(ring + g * slot_bytes, T.stream + (size_t)e.x * 16, e.y, bar + 8u * g);
        }
    }
    __syncthreads();
    if (win)
        blk_sweep_t<true, false, true>(T, count, xg, win_off, rg, -1, ring_off, slot_bytes, n_slots);
    else if (x_off >= 0 && r_off >= 0)
        blk_sweep_t<true, true, false>(T, count, xg, x_off, rg, r_off, ring_off, slot_bytes, n_slots);
    else if (x_off >= 0)
        blk_sweep_t<true, false, false>(T, count, xg, x_off, rg, r_off, ring_off, slot_bytes, n_slots);
    else
        blk_sweep_t<false, false, false>(T, count, xg, x_off, rg, r_off, ring_off, slot_bytes, n_slots);
    __syncthreads();
    if (threadIdx.x == 0)  // units delivered per slot
        for (int g = 0; g < n_slots; ++g) sy.phase[g] += g < total ? (total - 1 - g) / n_slots + 1 : 0;
    // published by the next sweep's (or phase's) __syncthreads()
}

// Both substitutions of one ILUT application; warp 0 solves, the CTA joins at
// the closing barrier.  The ring's mbarriers are (re)initialised per call so
// their phase parity starts at 0.
__device__ __forceinline__ void ilut_solve(const DevTri& L, const DevTri& U, double* zg, int z_off, double* xadd,
                                           int ring_off, int slot_bytes, int prod_off, bool exact) {
    __shared__ unsigned long long bars[2 * kTriSlots];
    if (!exact) __trap();  // the reassociated mode runs ilut_solve_blk
    // the ring overlays buffers written through the generic proxy in other
    // phases: order those writes before the TMA (async-proxy) writes
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (threadIdx.x < 32 * kSW) {
        const unsigned bar = sh_addr(bars);
        if (threadIdx.x == 0) {
            for (int k = 0; k < 2 * kTriSlots; ++k) mbar_init(bar + 8u * k);
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        sweep_sync();
        if (z_off >= 0) {
            tri_solve_warp<false, true>(L, zg, z_off, zg, z_off, ring_off, slot_bytes, prod_off, bar, exact);
            tri_solve_warp<true, true>(U, zg, z_off, zg, z_off, ring_off, slot_bytes, prod_off, bar + 8u * kTriSlots,
                                       exact);
        } else {
            tri_solve_warp<false, false>(L, zg, z_off, zg, z_off, ring_off, slot_bytes, prod_off, bar, exact);
            tri_solve_warp<true, false>(U, zg, z_off, zg, z_off, ring_off, slot_bytes, prod_off, bar + 8u * kTriSlots,
                                        exact);
        }
    }
    __syncthreads();
    // the smoother update x += z (axpy(1, z, x), pmultigrid.hpp:315), off the
    // substitution's critical path
    if (xadd) {
        const double* z = z_off >= 0 ? g_smem + z_off : zg;
        for (int i = threadIdx.x; i < L.n; i += NT) xadd[i] = xadd[i] + z[i];
        __syncthreads();
    }
}

// Reassociated mode: both substitutions as block recurrences, then x += z.
__device__ __forceinline__ void ilut_solve_blk(const DevBlk& L, const DevBlk& U, double* zg, int z_off, double* xadd,
                                               const Ws& w) {
    blk_sweep(L, 1, zg, z_off, zg, z_off, w.ring_off, w.slot_bytes, w.n_slots, w.win_off);
    blk_sweep(U, 1, zg, z_off, zg, z_off, w.ring_off, w.slot_bytes, w.n_slots, w.win_off);
    if (xadd) {
        const double* z = z_off >= 0 ? g_smem + z_off : zg;
        for (int i = threadIdx.x; i < L.n; i += NT) xadd[i] = xadd[i] + z[i];
        __syncthreads();
    }
}

// Lexicographic Gauss-Seidel sweeps (solvers.hpp:80-99) of an order-1
// h-level, in place on x: the sweep is a level-scheduled "triangular" solve
// (TriStream built by plan_gauss_seidel): the levels are the anti-diagonal
// wavefronts u + 2v = t (mirrored backward), every row sums its eight
// off-diagonal entries against the current x -- updated values from earlier
// wavefronts, old ones from later wavefronts, exactly as the sequential sweep
// sees them -- and divides by its diagonal.  Warp 0 runs `count` sweeps; the
// CTA joins at the closing barrier.
__device__ __forceinline__ void gs_sweeps(const DevHLevel& lv, const double* b, double* x, bool backward, int count,
                                          bool exact, int x_off, int b_off, int ring_off, int slot_bytes,
                                          int prod_off) {
    __shared__ unsigned long long gbar[kTriSlots];
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (threadIdx.x < 32 * kSW) {
        const unsigned bar = sh_addr(gbar);
        const DevTri& T = backward ? lv.gs_bwd : lv.gs_fwd;
        for (int c = 0; c < count; ++c) {
            if (threadIdx.x == 0) {
                for (int k = 0; k < kTriSlots; ++k) mbar_init(bar + 8u * k);
                asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
            }
            sweep_sync();
            if (x_off >= 0 && b_off >= 0)
                tri_solve_warp<true, true>(T, x, x_off, b, b_off, ring_off, slot_bytes, prod_off, bar, exact);
            else
                tri_solve_warp<true, false>(T, x, -1, b, -1, ring_off, slot_bytes, prod_off, bar, exact);
        }
    }
    __syncthreads();
}

// Index-ordered dot product (sparse.hpp:188-192): products in parallel into
// shared scratch, one thread sums them in index order.  Broadcast result.
__device__ __noinline__ double cta_ordered_dot(const double* a, const double* b, int n, double* scratch, double* sh,
                                               bool exact = true) {
    double s = 0.0;
    if (!exact) {  // reassociated: strided partial sums, warp butterflies, warp totals in order
        // the partial sums are defined on kDotThreads threads whatever the CTA
        // size, so the rounding does not depend on the number of sweep warps
        constexpr int DT = kDotThreads;
        double t = 0.0;
        if (threadIdx.x < DT) {
            double a0 = 0.0, a1 = 0.0;
            for (int i = threadIdx.x; i < n; i += 2 * DT) {
                a0 = a0 + a[i] * b[i];
                if (i + DT < n) a1 = a1 + a[i + DT] * b[i + DT];
            }
            t = a0 + a1;
            for (int o = 16; o > 0; o >>= 1) t = t + __shfl_xor_sync(0xffffffffu, t, o);
        }
        __syncthreads();
        if (threadIdx.x < DT && (threadIdx.x & 31) == 0) scratch[threadIdx.x >> 5] = t;
        __syncthreads();
        if (threadIdx.x == 0) {
            double u = 0.0;
            for (int k = 0; k < DT / 32; ++k) u = u + scratch[k];
            sh[0] = u;
        }
        __syncthreads();
        const double v = sh[0];
        __syncthreads();
        return v;
    }
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

__device__ void cta_fill(double* y, double v, int n, int part = 0, int parts = 1) {
    for (int i = threadIdx.x + part * NT; i < n; i += NT * parts) y[i] = v;
}
__device__ void cta_copy(double* y, const double* x, int n, int part = 0, int parts = 1) {
    for (int i = threadIdx.x + part * NT; i < n; i += NT * parts) y[i] = x[i];
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

// Lexicographic Gauss-Seidel sweeps of a 9-point order-1 level along grid
// lines (reassociated mode; solvers.hpp:80-99 restated per line).  For a
// forward sweep the row (iu, v) reads new values of its west neighbour and of
// line v-1, old values of its east neighbour and of line v+1:
//   1. prologue, all threads: o_i = (b_i - sum_old a_ij x_j) / d_i;
//   2. warp 0, line by line: beta_i = o_i - sum_{prev line} (a_ij / d_i) x_j,
//      then the in-line recurrence x_i = beta_i + alpha_i x_{i-1} (alpha =
//      -a_W / d) as a warp scan of affine maps (R = ceil(nf / 32) rows per
//      lane, composed locally first).  The next line's o and coefficients are
//      loaded while the current line is solved.
// A backward sweep mirrors both orders (lines v descending, iu descending).
template <bool SM, int RM>
__device__ __noinline__ void gs_line_sweeps_t(const DevHLevel& lv, const double* b, double* x, double* o,
                                              const double* bc, const double* xc, double* oc, bool backward,
                                              int count) {
    // cluster mode: the prologue is split over the cluster (bc, xc, oc: the
    // main CTA's vectors as the cluster sees them), the chain runs on the
    // main CTA; without clusters part = 0, parts = 1 and bc = b, ...
    const int part = cl_rank(), parts = cl_size();
    // SM: x and o in shared memory (explicit shared accesses on the chain)
    const unsigned xs = SM ? sh_addr(x) : 0u, os = SM ? sh_addr(o) : 0u;
    auto ldx = [&](int j) -> double { return SM ? vlds_f64(xs + 8u * j) : x[j]; };
    // RM: rows per lane (compile time), R = RM
    const int nf = lv.nf, n = nf * nf;
    constexpr int R = RM;
    const double* __restrict__ a = lv.a.vals;
    const double4* __restrict__ cf = reinterpret_cast<const double4*>(lv.gsl) + (backward ? n : 0);
    const double* __restrict__ rd = lv.gsl + 8 * (size_t)n;
    const int sv = backward ? 1 : -1;  // the previous line in sweep order is v + sv
    for (int c = 0; c < count; ++c) {
        // ---- 1. old part, scaled by 1/d
        constexpr int U = 4;  // rows per thread and pass: independent loads in flight
        for (int i0 = threadIdx.x + part * U * NT; i0 < n; i0 += U * NT * parts) {
            double acc[U], sc[U];
#pragma unroll
            for (int uu = 0; uu < U; ++uu) {
                const int i = min(i0 + uu * NT, n - 1);
                const int iv = i / nf, iu = i - iv * nf;
                double t = bc[i];
                // forward: E, NW, N, NE (old); backward: W, SW, S, SE
                const int du_in = backward ? -1 : 1, dv = -sv;
                const int u1 = iu + du_in;
                if (u1 >= 0 && u1 < nf) t -= a[(size_t)(4 + du_in) * n + i] * xc[i + du_in];
                const int v1 = iv + dv;
                if (v1 >= 0 && v1 < nf) {
#pragma unroll
                    for (int du = -1; du <= 1; ++du) {
                        const int u = iu + du;
                        if (u >= 0 && u < nf) t -= a[(size_t)((dv + 1) * 3 + du + 1) * n + i] * xc[i + dv * nf + du];
                    }
                }
                acc[uu] = t;
                sc[uu] = rd[i];
            }
#pragma unroll
            for (int uu = 0; uu < U; ++uu)
                if (i0 + uu * NT < n) oc[i0 + uu * NT] = acc[uu] * sc[uu];
        }
        cl_sync();
        // ---- 2. the line chain
        if (threadIdx.x < 32 && part == 0) {
            const int lane = threadIdx.x;
            double on[RM];
            double4 cn[RM];
            auto load_line = [&](int q) {
                const int v = backward ? nf - 1 - q : q;
#pragma unroll
                for (int r = 0; r < RM; ++r) {
                    const int p = lane * R + r;
                    if (p < nf) {
                        const int i = v * nf + (backward ? nf - 1 - p : p);
                        on[r] = SM ? vlds_f64(os + 8u * i) : o[i];
                        const double2* c2 = reinterpret_cast<const double2*>(cf + i);
                        const double2 lo = __ldg(c2), hi = __ldg(c2 + 1);
                        cn[r] = make_double4(lo.x, lo.y, hi.x, hi.y);
                    } else {
                        on[r] = 0.0;
                        cn[r] = make_double4(0.0, 0.0, 0.0, 0.0);
                    }
                }
            };
            load_line(0);
            double xp[RM];  // the previous line's new values (sweep order); none before line 0
#pragma unroll
            for (int r = 0; r < RM; ++r) xp[r] = 0.0;
            for (int q = 0; q < nf; ++q) {
                long long* tr = (kTrace && c_tune.trace && blockIdx.x == 0 && lane == 0 && q < 1024)
                                    ? c_tune.trace + kTriTraceBase + 8 * q
                                    : nullptr;
                if (tr) tr[0] = clock64();
                const int v = backward ? nf - 1 - q : q, vp = v + sv;
                double oc[RM];
                double4 cc[RM];
#pragma unroll
                for (int r = 0; r < RM; ++r) {
                    oc[r] = on[r];
                    cc[r] = cn[r];
                }
                if (q + 1 < nf) load_line(q + 1);
                // beta: fresh entries of the previous line, whose values this
                // warp holds in registers (xp, sweep order); the neighbours
                // across a lane boundary come by shuffle; positions outside
                // the line hold zero (and carry zero coefficients)
                const double lft = __shfl_up_sync(0xffffffffu, xp[RM - 1], 1);
                const double rgt = __shfl_down_sync(0xffffffffu, xp[0], 1);
                double bl[RM], al[RM];
#pragma unroll
                for (int r = 0; r < RM; ++r) {
                    const double xl = r > 0 ? xp[r - 1] : (lane > 0 ? lft : 0.0);
                    const double xr = r + 1 < RM ? xp[r + 1] : (lane < 31 ? rgt : 0.0);
                    // coefficients in natural order: iu-1, iu, iu+1
                    const double xm = backward ? xr : xl, xq = backward ? xl : xr;
                    bl[r] = oc[r] - ((cc[r].y * xm + cc[r].z * xp[r]) + cc[r].w * xq);
                    al[r] = cc[r].x;
                }
                if (tr) tr[1] = clock64() + (long long)(bl[0] == 1.2345) + (long long)(al[0] == 1.5);
                // in-line recurrence: compose the lane's rows, scan the lanes
                double B = bl[0], A = al[0];
#pragma unroll
                for (int r = 1; r < RM; ++r) {
                    B = __fma_rn(al[r], B, bl[r]);
                    A = al[r] * A;
                    bl[r] = B;
                    al[r] = A;
                }
                double Bs = B, As = A;
#pragma unroll
                for (int sft = 1; sft < 32; sft <<= 1) {
                    const double Bp = __shfl_up_sync(0xffffffffu, Bs, sft), Ap = __shfl_up_sync(0xffffffffu, As, sft);
                    if (lane >= sft) {
                        Bs = __fma_rn(As, Bp, Bs);
                        As = As * Ap;
                    }
                }
                double prev = __shfl_up_sync(0xffffffffu, Bs, 1);
                if (lane == 0) prev = 0.0;
                if (tr) tr[2] = clock64() + (long long)(prev == 1.2345);
#pragma unroll
                for (int r = 0; r < RM; ++r) {
                    const int p = lane * R + r;
                    const double xval = r + 1 == R ? Bs : __fma_rn(al[r], prev, bl[r]);
                    xp[r] = p < nf ? xval : 0.0;
                    if (p < nf) {
                        const int j = v * nf + (backward ? nf - 1 - p : p);
                        if (SM)
                            asm volatile("st.shared.f64 [%0], %1;" ::"r"(xs + 8u * j), "d"(xval) : "memory");
                        else
                            x[j] = xval;
                    }
                }
                __syncwarp();
                if (tr) tr[3] = clock64();
            }
        }
        cl_sync();
    }
}

template <int RM>
__device__ __forceinline__ void gs_line_sweeps_r(const DevHLevel& lv, const double* b, double* x, double* o,
                                                 const double* bc, const double* xc, double* oc, bool backward,
                                                 int count) {
    if (__isShared(x) && __isShared(o))
        gs_line_sweeps_t<true, RM>(lv, b, x, o, bc, xc, oc, backward, count);
    else
        gs_line_sweeps_t<false, RM>(lv, b, x, o, bc, xc, oc, backward, count);
}
// Called by every CTA of the cluster (by the CTA alone without clusters).
__device__ __forceinline__ void gs_line_sweeps(const DevHLevel& lv, const double* b, double* x, double* o,
                                               const double* bc, const double* xc, double* oc, bool backward,
                                               int count) {
    const int r = (lv.nf + 31) / 32;
    if (r <= 1)
        gs_line_sweeps_r<1>(lv, b, x, o, bc, xc, oc, backward, count);
    else if (r <= 2)
        gs_line_sweeps_r<2>(lv, b, x, o, bc, xc, oc, backward, count);
    else if (r <= 4)
        gs_line_sweeps_r<4>(lv, b, x, o, bc, xc, oc, backward, count);
    else
        gs_line_sweeps_r<8>(lv, b, x, o, bc, xc, oc, backward, count);
}

// x += C r for a dense column-major n x n operator (the collapsed coarse
// W-cycle subtree).  Thread i owns row i; r is broadcast from shared or
// global memory.
__device__ __noinline__ void dense_apply(const double* __restrict__ c, int n, const double* b, double* x,
                                         int part = 0, int parts = 1) {
    for (int i = threadIdx.x + part * NT; i < n; i += NT * parts) {
        double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
        int j = 0;
        for (; j + 4 <= n; j += 4) {
            a0 = __fma_rn(__ldg(c + (size_t)j * n + i), b[j], a0);
            a1 = __fma_rn(__ldg(c + (size_t)(j + 1) * n + i), b[j + 1], a1);
            a2 = __fma_rn(__ldg(c + (size_t)(j + 2) * n + i), b[j + 2], a2);
            a3 = __fma_rn(__ldg(c + (size_t)(j + 3) * n + i), b[j + 3], a3);
        }
        for (; j < n; ++j) a0 = __fma_rn(__ldg(c + (size_t)j * n + i), b[j], a0);
        x[i] = x[i] + ((a0 + a1) + (a2 + a3));
    }
}

// Cluster version of dense_apply (scr: SmemPlan::cl_scr_off, free during the
// W-cycle; without it the main CTA sits out): the rows are cut into `parts`
// contiguous ranges; in each CTA four warps cover up to 128 rows and the other
// four the second half of the columns; r (in the main CTA) is first copied
// into this CTA's shared memory so that the column loop broadcasts it.
// Caller: cl_sync after.
__device__ __noinline__ void dense_apply_cl(const double* __restrict__ c, int n, const double* r_main,
                                            double* x_main, int part, int parts, double* scr) {
    double* rl = scr;           // n doubles
    double* pp = scr + n + 1;   // 8 x 32 partial sums (kClScratch leaves room for them)
    for (int j = threadIdx.x; j < n; j += NT) rl[j] = r_main[j];
    __syncthreads();
    const int chunk = (n + parts - 1) / parts;
    const int r0 = part * chunk, r1 = min(n, r0 + chunk);
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // rw warps cover 32 rows each, the other warps split the columns: with 61
    // rows per CTA (n = 961 on 16 CTAs) two row warps and four column quarters
    // (the first eight warps; a CTA with more sweep warps leaves the others out)
    const int rw = chunk > 64 ? 4 : (chunk > 32 ? 2 : 1), cs = 8 / rw;
    const bool act = w < 8;
    const int wr = w % rw, wc = act ? w / rw : 0;
    const int j0 = (int)((long long)n * wc / cs), j1 = (int)((long long)n * (wc + 1) / cs);
    for (int base = r0; base < r1; base += 32 * rw) {
        const int i = base + wr * 32 + lane;  // this thread's row
        double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
        if (act && i < r1) {
            // sixteen operator loads in flight per thread: the product is bound by
            // the latency of the loads from L2 (each CTA streams n^2 / parts entries)
            int j = j0;
            for (; j + 16 <= j1; j += 16) {
                double v[16];
#pragma unroll
                for (int u = 0; u < 16; ++u) v[u] = __ldg(c + (size_t)(j + u) * n + i);
#pragma unroll
                for (int u = 0; u < 16; u += 4) {
                    a0 = __fma_rn(v[u], rl[j + u], a0);
                    a1 = __fma_rn(v[u + 1], rl[j + u + 1], a1);
                    a2 = __fma_rn(v[u + 2], rl[j + u + 2], a2);
                    a3 = __fma_rn(v[u + 3], rl[j + u + 3], a3);
                }
            }
            for (; j < j1; ++j) a0 = __fma_rn(__ldg(c + (size_t)j * n + i), rl[j], a0);
        }
        if (act) pp[w * 32 + lane] = (a0 + a1) + (a2 + a3);
        __syncthreads();
        if (act && wc == 0 && i < r1) {
            double s = pp[wr * 32 + lane];
            for (int q = 1; q < cs; ++q) s = s + pp[(q * rw + wr) * 32 + lane];  // column parts in order
            x_main[i] = x_main[i] + s;
        }
        __syncthreads();
    }
}

// h-multigrid W-cycle (pmultigrid.hpp:184-200) as an explicit per-level
// phase machine (no device recursion):
//   phase 0: pre-smooth, restrict, first coarse visit
//   phase 1: second coarse visit (starting from the first visit's result)
//   phase 2: prolongate, post-smooth, return
// Solution of level l lives in w.hx[l]; the result of level 0 is w.hx[0].
template <int DEG>
__device__ __noinline__ void wcycle(const DevHier& H, const Ws& w) {
    // developer phase accounting (trace builds, CTA 0 thread 0): cycles per
    // category at trace[kAccBase + c]: sweeps of level l (c = l), residual +
    // restriction (20), prolongation (21), coarsest solve (22)
    long long* acc = (kTrace && c_tune.trace && blockIdx.x == 0 && threadIdx.x == 0) ? c_tune.trace + kAccBase : nullptr;
    long long ta = acc ? clock64() : 0;
    auto mark = [&](int c) {
        if (acc) {
            const long long t = clock64();
            acc[c] += t - ta;
            ta = t;
        }
    };
    // Cluster mode (cl_size() > 1): the sweeps and the coarsest LU run on the
    // main CTA, every other phase is split by row over the cluster (the level
    // vectors live in the main CTA's shared memory: hbc / hxc / hrc are their
    // cluster-visible views), with cluster barriers in between; the dense
    // coarse operator then starts at the cluster's own (larger) level.
    const int part = cl_rank(), parts = cl_size();
    const bool main = part == 0;
    const int dl = parts > 1 ? H.dense_level_cl : H.dense_level;
    const double* dop = parts > 1 ? H.dense_op_cl : H.dense_op;
    int phase[kMaxH];
    int l = 0;
    phase[0] = 0;
    // neutral slots x[n] of the padded sweep entries (the vectors overlay the
    // smoother's shared memory)
    if (threadIdx.x == 0 && main)
        for (int k = 0; k < H.n_h; ++k) w.hx[k][H.h[k].n] = 0.0;
    cl_sync();
    for (;;) {
        if (l + 1 == H.n_h) {
            mark(23);
            if (main) coarse_solve(H, w.hb[l], w.hx[l]);
            cl_sync();
            mark(22);
            if (l == 0) break;
            --l;
            continue;
        }
        if (l == dl && phase[l] == 0) {
            // the subtree from level l, a linear iteration: x += C (b - A x)
            // (C: the cycle from a zero guess; x is zero on the first visit)
            mark(23);
            stencil_apply<kOutResid, Widths<DEG>::H>(H.h[l].a, w.hxc[l], w.hrc[l], w.hbc[l], false, part, parts);
            cl_sync();
            if (parts > 1) {
                double* scr = g_smem + (w.cl_scr_off >= 0 ? w.cl_scr_off : 0);
                if (w.cl_scr_off >= 0)
                    dense_apply_cl(dop, H.h[l].n, w.hrc[l], w.hxc[l], part, parts, scr);
                else if (part > 0)  // the helpers' shared memory is free: they never sweep
                    dense_apply_cl(dop, H.h[l].n, w.hrc[l], w.hxc[l], part - 1, parts - 1, scr);
            } else
                dense_apply(dop, H.h[l].n, w.hrc[l], w.hxc[l]);
            cl_sync();
            mark(22);
            if (l == 0) break;
            --l;
            continue;
        }
        const DevHLevel& lv = H.h[l];
        double* b = w.hb[l];
        double* x = w.hx[l];
        const int bo = w.lvl_off[l], xo = bo >= 0 ? bo + lv.n : -1;
        if (phase[l] == 0) {
            mark(23);
            if (!H.exact && lv.gsl) {  // every CTA: the prologues are split over the cluster
                gs_line_sweeps(lv, b, x, w.hr[l], w.hbc[l], w.hxc[l], w.hrc[l], false, H.gs_pre);
            } else {
                if (main) {
                    if (H.exact)
                        gs_sweeps(lv, b, x, false, H.gs_pre, true, xo, bo, w.ring_off, w.slot_bytes, w.prod_off);
                    else
                        blk_sweep(lv.gsb_fwd, H.gs_pre, x, xo, b, bo, w.ring_off, w.gs_slot_bytes, w.gs_n_slots);
                }
                cl_sync();
            }
            mark(l);
            stencil_apply<kOutResid, Widths<DEG>::H>(lv.a, w.hxc[l], w.hrc[l], w.hbc[l], H.exact != 0, part, parts);
            cl_sync();
            csr_apply<false>(lv.embed_t, w.hrc[l], w.hbc[l + 1], part, parts);  // rc = E^T r
            cta_fill(w.hxc[l + 1], 0.0, H.h[l + 1].n, part, parts);             // ec = 0
            cl_sync();
            mark(20);
            phase[l] = 1;
            phase[++l] = 0;
        } else if (phase[l] == 1) {
            phase[l] = 2;
            phase[++l] = 0;
        } else {
            mark(23);
            csr_apply<true>(lv.embed, w.hxc[l + 1], w.hxc[l], part, parts);  // x += E ec
            cl_sync();
            mark(21);
            if (!H.exact && lv.gsl) {
                gs_line_sweeps(lv, b, x, w.hr[l], w.hbc[l], w.hxc[l], w.hrc[l], true, H.gs_post);
            } else {
                if (main) {
                    if (H.exact)
                        gs_sweeps(lv, b, x, true, H.gs_post, true, xo, bo, w.ring_off, w.slot_bytes, w.prod_off);
                    else
                        blk_sweep(lv.gsb_bwd, H.gs_post, x, xo, b, bo, w.ring_off, w.gs_slot_bytes, w.gs_n_slots);
                }
                cl_sync();
            }
            mark(l);
            if (l == 0) break;
            --l;
        }
    }
}

// x += S (b - A x), S = ILUT application (pmultigrid.hpp:311-316).
// r_valid: w.r already holds b - A x for the current x (the solve loop's
// residual check), so z = r is a copy -- the same values the product would
// give, in both summation modes.
template <int DEG>
__device__ __noinline__ void smooth(const DevHier& H, const Ws& w, bool r_valid = false) {
    pstamp(10);
    const int part = cl_rank(), parts = cl_size();
    if (r_valid)
        cta_copy(w.zc, w.r, H.n_p, part, parts);
    else
        stencil_apply<kOutResid, Widths<DEG>::A>(H.A, w.x, w.zc, w.b, H.exact != 0, part, parts);  // z = r = b - A x
    if (threadIdx.x == 0 && part == 0) w.z[H.n_p] = 0.0;  // neutral padding slot
    cl_sync();
    pstamp(11);
    if (part == 0) {  // the sweeps: main CTA
        if (H.exact)
            ilut_solve(H.L, H.U, w.z, w.z_off, w.x, w.ring_off, w.slot_bytes, w.prod_off, true);
        else
            ilut_solve_blk(H.Lb, H.Ub, w.z, w.z_off, w.x, w);
    }
    cl_sync();
    pstamp(12);
}

// One V(nu_pre, nu_post) cycle (pmultigrid.hpp:256-267).
template <int DEG>
__device__ __noinline__ void vcycle(const DevHier& H, const Ws& w, bool r_valid = false) {
    const int part = cl_rank(), parts = cl_size();
    for (int s = 0; s < H.nu_pre; ++s) smooth<DEG>(H, w, r_valid && s == 0);
    stencil_apply<kOutResid, Widths<DEG>::A>(H.A, w.x, w.r, w.b, H.exact != 0, part, parts);
    cl_sync();
    stencil_apply<kOutScale, Widths<DEG>::T>(H.Tt, w.r, w.hb0c, H.inv_l1, H.exact != 0, part,
                                             parts);  // restrict_to_linear
    cta_fill(w.hx0c, 0.0, H.n_1, part, parts);
    cl_sync();
    pstamp(20);
    wcycle<DEG>(H, w);  // cluster-aware: sweeps on the main CTA
    pstamp(21);
    stencil_apply<kOutAddScaled, Widths<DEG>::T>(H.T, w.hx0c, w.x, H.inv_lp, H.exact != 0, part,
                                                 parts);  // x += prolong_from_linear
    cl_sync();
    pstamp(22);
    for (int s = 0; s < H.nu_post; ++s) smooth<DEG>(H, w);
}

template <int DEG>
__device__ double rel_residual(const DevHier& H, const Ws& w, double bnorm, double* sh) {
    pstamp(30);
    stencil_apply<kOutResid, Widths<DEG>::A>(H.A, w.x, w.r, w.b, H.exact != 0, cl_rank(), cl_size());
    cl_sync();  // every CTA reads the whole residual
    const double d = cta_ordered_dot(w.r, w.r, H.n_p, w.dot, sh, H.exact != 0);
    pstamp(31);
    return sqrt(d) / bnorm;
}

// The CG kind's solve of one Phi (theta.hpp:121-125): Jacobi-preconditioned CG
// on A from the guess in w.x (solvers.hpp:21-75), b = w.b, |b| = bnorm > 0.
// The vectors live in the global workspace; with a cluster every phase is
// split by row over its CTAs (each CTA forms the dot products over the whole
// vectors in the same order, so all agree).  exact: the reference's operator
// rows and index-ordered dots.  rel < 0 on breakdown (p^T A p <= 0).
template <int DEG>
__device__ __noinline__ void cg_point(const DevHier& H, const Ws& w, double bnorm, double* sh, int& iters, int& conv,
                                      double& rel) {
    const int n = H.n_p;
    const int part = cl_rank(), parts = cl_size();
    const bool ex = H.exact != 0;
    const double* __restrict__ diag = H.diag;
    double *x = w.x, *r = w.r, *z = w.zg, *p = w.cgp, *q = w.cgq;
    stencil_apply<kOutResid, Widths<DEG>::A>(H.A, x, r, w.b, ex, part, parts);  // r = b - A x
    cl_sync();
    double rnorm = sqrt(cta_ordered_dot(r, r, n, w.dot, sh, ex));
    rel = rnorm / bnorm;
    if (rnorm <= H.rel_tol * bnorm) {
        conv = 1;
        return;
    }
    for (int i = threadIdx.x + part * NT; i < n; i += NT * parts) {
        const double zi = r[i] / diag[i];
        z[i] = zi;
        p[i] = zi;
    }
    cl_sync();
    double rz = cta_ordered_dot(r, z, n, w.dot, sh, ex);
    for (int it = 1; it <= H.max_iter; ++it) {
        stencil_apply<kOutSet, Widths<DEG>::A>(H.A, p, q, nullptr, ex, part, parts);
        cl_sync();
        const double pq = cta_ordered_dot(p, q, n, w.dot, sh, ex);
        if (pq <= 0.0) {  // breakdown: not SPD
            rel = -1.0;
            return;
        }
        const double alpha = rz / pq;
        for (int i = threadIdx.x + part * NT; i < n; i += NT * parts) {
            x[i] += alpha * p[i];
            r[i] += -alpha * q[i];
        }
        cl_sync();
        rnorm = sqrt(cta_ordered_dot(r, r, n, w.dot, sh, ex));
        iters = it;
        rel = rnorm / bnorm;
        if (rnorm <= H.rel_tol * bnorm) {
            conv = 1;
            return;
        }
        for (int i = threadIdx.x + part * NT; i < n; i += NT * parts) z[i] = r[i] / diag[i];
        cl_sync();
        const double rz_new = cta_ordered_dot(r, z, n, w.dot, sh, ex);
        const double beta = rz_new / rz;
        rz = rz_new;
        for (int i = threadIdx.x + part * NT; i < n; i += NT * parts) p[i] = z[i] + beta * p[i];
        cl_sync();
    }
}

// One Phi application: build b, solve (pmultigrid.hpp:271-307), epilogue.
template <int DEG>
__device__ __noinline__ void phi_point(const DevHier& H, const DevStencil& Am, const WaveArgs& a, const Ws& w, int task,
                          int k, double* sh) {
    const int n = H.n_p;
    const int part = cl_rank(), parts = cl_size();
    pstamp(50);
    // ---- right-hand side and initial guess
    if (a.mode == kModeStep) {
        const double* uprev = a.U ? a.U + (size_t)(k - 1) * n : a.UPREV + (size_t)task * a.ldu;
        const double* load = nullptr;
        if (a.LOAD)
            load = a.load_steady ? a.LOAD : a.LOAD + (size_t)(k - 1) * n;
        else if (a.LOADV)
            load = a.LOADV + (size_t)task * a.ldl;
        if (load)
            stencil_apply<kOutAddVec, Widths<DEG>::A>(Am, uprev, w.b, load, H.exact != 0, part,
                                                      parts);  // rhs = A- u + load
        else
            stencil_apply<kOutSet, Widths<DEG>::A>(Am, uprev, w.b, nullptr, H.exact != 0, part, parts);
        const double* guess =
            a.U ? a.U + (size_t)(a.guess_prev ? k - 1 : k) * n : (a.x0_empty ? nullptr : a.X + (size_t)task * a.ldx);
        if (guess)
            cta_copy(w.x, guess, n, part, parts);
        else
            cta_fill(w.x, 0.0, n, part, parts);
    } else {
        const double* bsrc;
        if (a.B)
            bsrc = a.B + (size_t)task * a.ldb;
        else
            bsrc = a.load_steady ? a.LOAD : a.LOAD + (size_t)(k - 1) * n;
        cta_copy(w.b, bsrc, n, part, parts);
        if (a.x0_empty)
            cta_fill(w.x, 0.0, n, part, parts);
        else
            cta_copy(w.x, a.X + (size_t)task * a.ldx, n, part, parts);
    }
    cl_sync();
    pstamp(51);

    // ---- p-multigrid solve
    int iters = 0, conv = 0;
    double rel = 0.0;
    const double bnorm = sqrt(cta_ordered_dot(w.b, w.b, n, w.dot, sh, H.exact != 0));
    pstamp(52);
    if (bnorm == 0.0) {
        cta_fill(w.x, 0.0, n, part, parts);  // zero rhs -> zero solution, not the guess
        conv = 1;
        cl_sync();
    } else if (H.kind == 1) {
        cg_point<DEG>(H, w, bnorm, sh, iters, conv, rel);
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
                vcycle<DEG>(H, w, true);  // w.r = b - A x from the residual check
                rel = rel_residual<DEG>(H, w, bnorm, sh);
                iters = it;
                if (rel <= H.rel_tol) {
                    conv = 1;
                    break;
                }
            }
        }
    }

    pstamp(53);
    // ---- bookkeeping (SolveStats::record, theta.hpp:81-84)
    if (threadIdx.x == 0 && part == 0) {
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
        for (int i = threadIdx.x + part * NT; i < n; i += NT * parts) out[i] = g ? w.x[i] + g[i] : w.x[i];
    } else if (a.epi == kEpiRestrict) {
        const int j = k / a.m;
        const double* u = a.U + (size_t)k * n;
        double* cg = a.CG + (size_t)j * n;
        double* cu = a.CU + (size_t)j * n;
        for (int i = threadIdx.x + part * NT; i < n; i += NT * parts) {
            const double wv = g ? w.x[i] + g[i] : w.x[i];
            cg[i] = wv - u[i];
            cu[i] = 0.0;
        }
    } else if (a.epi == kEpiResid) {
        const double* u = a.U + (size_t)k * n;
        for (int i = threadIdx.x + part * NT; i < n; i += NT * parts) {
            const double wv = g ? w.x[i] + g[i] : w.x[i];
            w.r[i] = wv - u[i];
        }
        cl_sync();
        const double d = cta_ordered_dot(w.r, w.r, n, w.dot, sh, H.exact != 0);
        if (threadIdx.x == 0 && part == 0) a.SQ[k] = d;
    } else if (a.epi == kEpiNorm) {
        const double d = cta_ordered_dot(w.x, w.x, n, w.dot, sh, H.exact != 0);
        if (threadIdx.x == 0 && part == 0) a.SQ[k] = d;
    } else {
        double* out = a.X + (size_t)task * a.ldx;
        for (int i = threadIdx.x + part * NT; i < n; i += NT * parts) out[i] = w.x[i];
    }
    cl_sync();
    pstamp(54);
}

// SIDE: a second instantiation for the side-stream waves that run while the
// coarse march (a cluster launch of the SIDE = 0 instance) is in flight
template <int DEG, int SIDE = 0>
__global__ void __launch_bounds__(NT, 1)
    phi_wave_kernel(const __grid_constant__ DevHier H_param, const __grid_constant__ DevStencil Am,
                    const __grid_constant__ WaveArgs a_param, const __grid_constant__ SmemPlan P, double* ws_base,
                    long long ws_stride) {
    double* smem = g_smem;
    __shared__ double sh[4];
    __shared__ WaveArgs a_sh;
    if (threadIdx.x == 0) a_sh = a_param;
    const WaveArgs& a = a_sh;
    cl_init();
    blk_init();
    const DevHier& H = hier_shared(H_param);
    // one workspace per cluster (the main CTA's); cluster c takes tasks c, c + nclusters, ...
    const int cid = blockIdx.x / cl_size(), ncl = gridDim.x / cl_size();
    const Ws& w = carve_shared(ws_base + (size_t)cid * ws_stride, H, P, smem);
    for (int task = cid; task < a.n_tasks; task += ncl) {
        for (int s = 0; s < a.task_len; ++s) {
            const int k = a.task_k0 ? a.task_k0[task] + s : task;
            phi_point<DEG>(H, Am, a, w, task, k, sh);
            // phi_point ends with a cluster barrier: every CTA's stores of
            // point k are done; publish k to the host system-wide
            if (a.progress && threadIdx.x == 0 && cl_rank() == 0) {
                __threadfence_system();
                *a.progress = (unsigned)k;
            }
        }
    }
}

// ---- standalone V-cycle on a batch (PMultigridHierarchy::vcycle) ----------
template <int DEG>
__global__ void __launch_bounds__(NT, 1)
    vcycle_kernel(const __grid_constant__ DevHier H_param, const double* B, long long ldb, double* X, long long ldx,
                  int nrhs, const __grid_constant__ SmemPlan P, double* ws_base, long long ws_stride) {
    double* smem = g_smem;
    cl_init();
    blk_init();
    const DevHier& H = hier_shared(H_param);
    // one workspace per cluster (a cluster of one CTA without clusters); cluster c takes c, c + nclusters, ...
    const int cid = blockIdx.x / cl_size(), ncl = gridDim.x / cl_size();
    const int part = cl_rank(), parts = cl_size();
    const Ws& w = carve_shared(ws_base + (size_t)cid * ws_stride, H, P, smem);
    const int n = H.n_p;
    for (int t = cid; t < nrhs; t += ncl) {
        cta_copy(w.b, B + (size_t)t * ldb, n, part, parts);
        cta_copy(w.x, X + (size_t)t * ldx, n, part, parts);
        cl_sync();
        vcycle<DEG>(H, w);
        double* out = X + (size_t)t * ldx;
        for (int i = threadIdx.x + part * NT; i < n; i += NT * parts) out[i] = w.x[i];
        cl_sync();
    }
}

// ---- unit-level kernel used by the parity tests ---------------------------
// op: 0 y = A x, 1 z = ILUT(r), 2 r1 = restrict(r), 3 x += prolong(e1) (x given),
//     4 x1 = W-cycle(b1, x1), 5 x = GS(b, x) on level `arg` (arg2 = backward)
template <int DEG>
__global__ void __launch_bounds__(NT, 1)
    unit_kernel(const __grid_constant__ DevHier H_param, int op, int arg, int arg2, const double* in, double* out,
                const __grid_constant__ SmemPlan P, double* ws_base, long long ws_stride) {
    double* smem = g_smem;
    cl_init();
    blk_init();
    const DevHier& H = hier_shared(H_param);
    const Ws& w = carve_shared(ws_base + (size_t)blockIdx.x * ws_stride, H, P, smem);
    const int n = H.n_p;
    if (op == 0) {
        stencil_apply<kOutSet, Widths<DEG>::A>(H.A, in, out, nullptr, H.exact != 0);
    } else if (op == 1) {
        cta_copy(w.z, in, n);
        cta_fill(w.x, 0.0, n);
        if (threadIdx.x == 0) w.z[n] = 0.0;
        __syncthreads();
        if (H.exact)
            ilut_solve(H.L, H.U, w.z, w.z_off, w.x, w.ring_off, w.slot_bytes, w.prod_off, true);
        else
            ilut_solve_blk(H.Lb, H.Ub, w.z, w.z_off, w.x, w);
        cta_copy(out, w.z, n);
    } else if (op == 2) {
        stencil_apply<kOutScale, Widths<DEG>::T>(H.Tt, in, out, H.inv_l1, H.exact != 0);
    } else if (op == 3) {
        stencil_apply<kOutAddScaled, Widths<DEG>::T>(H.T, in, out, H.inv_lp, H.exact != 0);
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
        if (threadIdx.x == 0) w.hx[arg][lv.n] = 0.0;  // neutral slot of padded sweep entries
        __syncthreads();
        const int bo = w.lvl_off[arg], xo = bo >= 0 ? bo + lv.n : -1;
        if (H.exact)
            gs_sweeps(lv, w.hb[arg], w.hx[arg], arg2 != 0, 1, true, xo, bo, w.ring_off, w.slot_bytes, w.prod_off);
        else if (lv.gsl)
            gs_line_sweeps(lv, w.hb[arg], w.hx[arg], w.hr[arg], w.hb[arg], w.hx[arg], w.hr[arg], arg2 != 0, 1);
        else
            blk_sweep(arg2 ? lv.gsb_bwd : lv.gsb_fwd, 1, w.hx[arg], xo, w.hb[arg], bo, w.ring_off, w.gs_slot_bytes,
                      w.gs_n_slots);
        cta_copy(out, w.hx[arg], lv.n);
    }
}

// ---- IC projection: Jacobi-preconditioned CG on M (solvers.hpp:21-75) ------
// One CTA, or one cluster of CTAs: the operator rows and the vector updates are
// split by row over the cluster, every CTA forms the dot products over the
// whole vectors in the same order (as cg_point), so all CTAs take the same
// decisions and the result does not depend on the cluster size -- bitwise, in
// both summation modes.  exact: index-ordered dot products and operator rows
// (the reference's rounding), else reassociated sums.  work: 4 vectors of n.
template <int DEG>
__global__ void __launch_bounds__(NT, 1)
    cg_kernel(const __grid_constant__ DevStencil A, const double* __restrict__ diag, const double* __restrict__ b,
              double* x, double* work, double rel_tol, int max_iter, int* result, int exact) {
    __shared__ double sh[4];
    __shared__ double scratch[kDotChunk];
    cl_init();
    __syncthreads();
    const int part = cl_rank(), parts = cl_size();
    const bool ex = exact != 0;
    const int n = A.ru * A.rv;
    double* r = work;
    double* z = work + n;
    double* p = work + 2 * (size_t)n;
    double* q = work + 3 * (size_t)n;
    auto finish = [&](int conv, int it) {
        if (threadIdx.x == 0 && part == 0) {
            result[0] = conv;
            result[1] = it;
        }
    };
    const double bnorm = sqrt(cta_ordered_dot(b, b, n, scratch, sh, ex));
    cta_fill(x, 0.0, n, part, parts);
    if (bnorm == 0.0) return finish(1, 0);
    cl_sync();
    stencil_apply<kOutResid, Widths<DEG>::A>(A, x, r, b, ex, part, parts);
    cl_sync();
    double rnorm = sqrt(cta_ordered_dot(r, r, n, scratch, sh, ex));
    if (rnorm <= rel_tol * bnorm) return finish(1, 0);
    for (int i = threadIdx.x + part * NT; i < n; i += NT * parts) {
        const double zi = r[i] / diag[i];
        z[i] = zi;
        p[i] = zi;
    }
    cl_sync();
    double rz = cta_ordered_dot(r, z, n, scratch, sh, ex);
    int conv = 0, it = 1;
    for (; it <= max_iter; ++it) {
        stencil_apply<kOutSet, Widths<DEG>::A>(A, p, q, nullptr, ex, part, parts);
        cl_sync();
        const double pq = cta_ordered_dot(p, q, n, scratch, sh, ex);
        if (pq <= 0.0) {
            conv = -1;
            break;
        }
        const double alpha = rz / pq;
        for (int i = threadIdx.x + part * NT; i < n; i += NT * parts) {
            x[i] += alpha * p[i];
            r[i] += -alpha * q[i];
        }
        cl_sync();
        rnorm = sqrt(cta_ordered_dot(r, r, n, scratch, sh, ex));
        if (rnorm <= rel_tol * bnorm) {
            conv = 1;
            break;
        }
        for (int i = threadIdx.x + part * NT; i < n; i += NT * parts) z[i] = r[i] / diag[i];
        cl_sync();
        const double rz_new = cta_ordered_dot(r, z, n, scratch, sh, ex);
        const double beta = rz_new / rz;
        rz = rz_new;
        for (int i = threadIdx.x + part * NT; i < n; i += NT * parts) p[i] = z[i] + beta * p[i];
        cl_sync();
    }
    finish(conv, it);
}

}  // namespace

template <class K>
static inline int occupancy_grid(K kernel, size_t smem, int want) {
    static int n_sm = 0;
    if (!n_sm) {
        int dev = 0;
        PHI_CUDA(cudaGetDevice(&dev));
        PHI_CUDA(cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev));
    }
    // the dynamic shared-memory limit is raised ONCE per kernel to the plan's
    // budget: changing a function attribute while an instance of the same
    // kernel runs serialises the next launch behind it (it defeated the
    // overlap of the coarse march with the side-stream waves)
    static std::vector<const void*> raised;
    const void* key = reinterpret_cast<const void*>(kernel);
    if (std::find(raised.begin(), raised.end(), key) == raised.end()) {
        PHI_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)std::max<size_t>(smem, kPhiSmemBudgetBytes)));
        raised.push_back(key);
    }
    int per_sm = 0;
    PHI_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, NT, smem));
    if (per_sm < 1) per_sm = 1;
    return std::max(1, std::min(want, per_sm * n_sm));
}


// The largest cluster size (a power of two <= cl_max) at which the device can
// keep n_tasks clusters of `kernel` resident at once (every task its own
// cluster, one round), 1 if none: cudaOccupancyMaxActiveClusters, cached.
template <class K>
static int pick_cluster(K kernel, size_t smem, int n_tasks, int cl_max) {
    static int cached_active[6] = {-1, -1, -1, -1, -1, -1};  // by log2(cl)
    static size_t cached_smem = 0;
    if (cached_smem != smem) {
        for (int& c : cached_active) c = -1;
        cached_smem = smem;
    }
    for (int cl = cl_max, lg = 0; cl > 1; cl /= 2) {
        if (cl & (cl - 1)) return 1;  // powers of two only
        for (lg = 0; (1 << lg) < cl; ++lg) {
        }
        if (lg > 5) continue;
        if (cached_active[lg] < 0) {
            if (cl > 8) PHI_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
            cudaLaunchConfig_t q{};
            q.gridDim = dim3((unsigned)cl);
            q.blockDim = dim3(NT);
            q.dynamicSmemBytes = smem;
            cudaLaunchAttribute qa[1];
            qa[0].id = cudaLaunchAttributeClusterDimension;
            qa[0].val.clusterDim.x = (unsigned)cl;
            qa[0].val.clusterDim.y = 1;
            qa[0].val.clusterDim.z = 1;
            q.attrs = qa;
            q.numAttrs = 1;
            int ncl = 0;
            if (cudaOccupancyMaxActiveClusters(&ncl, kernel, &q) != cudaSuccess) {
                (void)cudaGetLastError();
                ncl = 0;
            }
            cached_active[lg] = ncl;
        }
        if (cached_active[lg] >= n_tasks) return cl;
    }
    return 1;
}

template <int DEG>
int DegLaunch<DEG>::max_slots(const DevHier& H) {
    return occupancy_grid(phi_wave_kernel<DEG>, phi_smem_bytes(H), 1 << 30);
}

template <int DEG>
void DegLaunch<DEG>::wave(const DevHier& H, const DevStencil& Am, const WaveArgs& a, double* ws, long long ws_stride,
                          int grid, cudaStream_t s) {
    const SmemPlan P = phi_smem_plan(H);
    const size_t smem = (size_t)P.total * 8;
    occupancy_grid(phi_wave_kernel<DEG>, smem, grid);
    // a wave of few right-hand sides (the coarse march: one) runs each task on
    // a cluster of CTAs (reassociated mode): the data-parallel phases spread
    // over the cluster's SMs (developer override: PHI_CLUSTER=<size>, 0/1 off)
    static int cl = -1;
    if (cl < 0) {
        cl = kPhiCluster;
        if (const char* e = std::getenv("PHI_CLUSTER")) {
            cl = std::atoi(e);
        } else {
            // kPhiClusterWide CTAs (a non-portable size) when the device can
            // co-schedule such a cluster at the largest shared-memory plan
            PHI_CUDA(cudaFuncSetAttribute(phi_wave_kernel<DEG>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
            PHI_CUDA(cudaFuncSetAttribute(phi_wave_kernel<DEG>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)kPhiSmemBudgetBytes));
            cudaLaunchConfig_t q{};
            q.gridDim = dim3((unsigned)kPhiClusterWide);
            q.blockDim = dim3(NT);
            q.dynamicSmemBytes = kPhiSmemBudgetBytes;
            cudaLaunchAttribute qa[1];
            qa[0].id = cudaLaunchAttributeClusterDimension;
            qa[0].val.clusterDim.x = (unsigned)kPhiClusterWide;
            qa[0].val.clusterDim.y = 1;
            qa[0].val.clusterDim.z = 1;
            q.attrs = qa;
            q.numAttrs = 1;
            int ncl = 0;
            if (cudaOccupancyMaxActiveClusters(&ncl, phi_wave_kernel<DEG>, &q) == cudaSuccess && ncl >= 1)
                cl = kPhiClusterWide;
            else
                (void)cudaGetLastError();
        }
    }
    int n_sm = 0, dev = 0;
    PHI_CUDA(cudaGetDevice(&dev));
    PHI_CUDA(cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev));
    // the largest cluster (a power of two up to the device's limit) that still
    // gives every task its own cluster: 16 CTAs up to 9 tasks, 8 up to 18, ...
    int use = cl;
    if (a.n_tasks * cl > n_sm) {  // more than a few tasks: the largest size at which all their clusters are resident
        use = (!H.exact && !a.no_cluster && cl > 1 && H.n_p >= 4096)  // (small systems: the barriers outweigh the split)
                  ? pick_cluster(phi_wave_kernel<DEG>, smem, a.n_tasks, cl / 2)
                  : 1;
    }
    if (!H.exact && !a.no_cluster && use > 1) {
        const int cl = use;
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3((unsigned)(a.n_tasks * cl));
        cfg.blockDim = dim3(NT);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = s;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = (unsigned)cl;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        static bool nonportable = false;
        if (cl > 8 && !nonportable) {
            PHI_CUDA(cudaFuncSetAttribute(phi_wave_kernel<DEG>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
            nonportable = true;
        }
        PHI_CUDA(cudaLaunchKernelEx(&cfg, phi_wave_kernel<DEG>, H, Am, a, P, ws, ws_stride));
    } else {
        if (a.no_cluster) {
            occupancy_grid(phi_wave_kernel<DEG, 1>, smem, grid);
            phi_wave_kernel<DEG, 1><<<grid, NT, smem, s>>>(H, Am, a, P, ws, ws_stride);
        } else {
            phi_wave_kernel<DEG><<<grid, NT, smem, s>>>(H, Am, a, P, ws, ws_stride);
        }
    }
    PHI_CUDA(cudaGetLastError());
}

template <int DEG>
void DegLaunch<DEG>::vcycle(const DevHier& H, const double* B, long long ldb, double* X, long long ldx, int nrhs,
                            double* ws, long long ws_stride, int grid, cudaStream_t s) {
    const SmemPlan P = phi_smem_plan(H);
    const size_t smem = (size_t)P.total * 8;
    occupancy_grid(vcycle_kernel<DEG>, smem, grid);
    // few right-hand sides (reassociated mode): each on a cluster of CTAs, as
    // the single-right-hand-side waves (developer override: PHI_CLUSTER)
    int n_sm = 0, dev = 0;
    PHI_CUDA(cudaGetDevice(&dev));
    PHI_CUDA(cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev));
    int cl = kPhiClusterWide;
    if (const char* e = std::getenv("PHI_CLUSTER")) cl = std::atoi(e);
    // every right-hand side its own resident cluster (small systems: the barriers outweigh the split)
    cl = (!H.exact && cl > 1 && H.n_p >= 4096) ? pick_cluster(vcycle_kernel<DEG>, smem, nrhs, cl) : 1;
    if (cl > 1) {
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3((unsigned)(nrhs * cl));
        cfg.blockDim = dim3(NT);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = s;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = (unsigned)cl;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        PHI_CUDA(cudaLaunchKernelEx(&cfg, vcycle_kernel<DEG>, H, B, ldb, X, ldx, nrhs, P, ws, ws_stride));
    } else {
        vcycle_kernel<DEG><<<grid, NT, smem, s>>>(H, B, ldb, X, ldx, nrhs, P, ws, ws_stride);
    }
    PHI_CUDA(cudaGetLastError());
}

template <int DEG>
void DegLaunch<DEG>::unit(const DevHier& H, int op, int arg, int arg2, const double* in, double* out, double* ws,
                          long long ws_stride, cudaStream_t s) {
    const SmemPlan P = phi_smem_plan(H);
    const size_t smem = (size_t)P.total * 8;
    occupancy_grid(unit_kernel<DEG>, smem, 1);
    unit_kernel<DEG><<<1, NT, smem, s>>>(H, op, arg, arg2, in, out, P, ws, ws_stride);
    PHI_CUDA(cudaGetLastError());
}

template <int DEG>
void DegLaunch<DEG>::cg(const DevStencil& A, const double* diag, const double* b, double* x, double* work,
                        double rel_tol, int max_iter, int* result, int exact, cudaStream_t s) {
    // a cluster for systems large enough that the row split outweighs its
    // barriers (the threshold of the wave kernel); same result for any size
    static int cl = -1;
    if (cl < 0) {
        cl = 1;
        if (const char* e = std::getenv("PHI_CLUSTER")) {
            cl = std::max(1, std::atoi(e));
        } else {
            for (int c = kPhiClusterWide; c > 1 && cl == 1; c /= 2) {
                if (c > 8 && cudaFuncSetAttribute(cg_kernel<DEG>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) !=
                                 cudaSuccess) {
                    (void)cudaGetLastError();
                    continue;
                }
                cudaLaunchConfig_t q{};
                q.gridDim = dim3((unsigned)c);
                q.blockDim = dim3(NT);
                cudaLaunchAttribute qa[1];
                qa[0].id = cudaLaunchAttributeClusterDimension;
                qa[0].val.clusterDim.x = (unsigned)c;
                qa[0].val.clusterDim.y = 1;
                qa[0].val.clusterDim.z = 1;
                q.attrs = qa;
                q.numAttrs = 1;
                int ncl = 0;
                if (cudaOccupancyMaxActiveClusters(&ncl, cg_kernel<DEG>, &q) == cudaSuccess && ncl >= 1)
                    cl = c;
                else
                    (void)cudaGetLastError();
            }
        }
    }
    const int use = A.ru * A.rv >= 4096 ? cl : 1;
    if (use > 1) {
        if (use > 8) PHI_CUDA(cudaFuncSetAttribute(cg_kernel<DEG>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3((unsigned)use);
        cfg.blockDim = dim3(NT);
        cfg.stream = s;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = (unsigned)use;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        PHI_CUDA(cudaLaunchKernelEx(&cfg, cg_kernel<DEG>, A, diag, b, x, work, rel_tol, max_iter, result, exact));
    } else {
        cg_kernel<DEG><<<1, NT, 0, s>>>(A, diag, b, x, work, rel_tol, max_iter, result, exact);
    }
    PHI_CUDA(cudaGetLastError());
}

template <int DEG>
void DegLaunch<DEG>::preload_side(const DevHier& H) {
    cudaFuncAttributes fa;
    PHI_CUDA(cudaFuncGetAttributes(&fa, phi_wave_kernel<DEG, 1>));
    occupancy_grid(phi_wave_kernel<DEG, 1>, phi_smem_bytes(H), 1);
}

template <int DEG>
void DegLaunch<DEG>::set_trace(long long* trace, int xmask) {
    Tuning t{xmask, NW, 0, 0, trace};
    PHI_CUDA(cudaMemcpyToSymbol(c_tune, &t, sizeof t));
}

}  // namespace phi
