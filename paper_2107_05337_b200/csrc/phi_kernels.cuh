// Host-callable launchers for the Phi kernels (phi_kernels.cu) and the device
// assembly kernels (assembly.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstddef>

#include "common.hpp"
#include "device_types.cuh"

namespace phi {

// Threads per Phi CTA: 2 block-sweep solver warps + 6 worker warps by default
// (PHI_THREADS / PHI_BLK_SOLVERS: developer A/B builds with more solver warps).
constexpr int kPhiThreads = PHI_THREADS;
// Dynamic shared memory one Phi CTA may use for its latency-critical vectors
// (one CTA per SM; 227 KB is the sm_100 per-block maximum).
#ifndef PHI_SMEM_BUDGET_KB
#define PHI_SMEM_BUDGET_KB 212
#endif
constexpr size_t kPhiSmemBudgetBytes = PHI_SMEM_BUDGET_KB * 1024;
/// CTAs per cluster for waves of few right-hand sides (reassociated mode).
constexpr int kPhiCluster = 8;       // CTAs per single-RHS cluster (portable size)
constexpr int kPhiClusterWide = 16;  // ... when the device can co-schedule this many (non-portable)

size_t phi_ws_doubles(const DevHier& H);
SmemPlan phi_smem_plan(const DevHier& H);
size_t phi_smem_bytes(const DevHier& H);
int phi_max_slots(const DevHier& H);
void phi_set_tuning(int tri_warps, int gs_warps, int sleep_ns);
int phi_read_trace(long long* out, int n);

/// Degree-templated launchers, explicitly instantiated in phi_deg.cu.
template <int DEG>
struct DegLaunch {
    static int max_slots(const DevHier& H);
    static void wave(const DevHier& H, const DevStencil& Am, const WaveArgs& a, double* ws, long long ws_stride,
                     int grid, cudaStream_t s);
    static void vcycle(const DevHier& H, const double* B, long long ldb, double* X, long long ldx, int nrhs,
                       double* ws, long long ws_stride, int grid, cudaStream_t s);
    static void unit(const DevHier& H, int op, int arg, int arg2, const double* in, double* out, double* ws,
                     long long ws_stride, cudaStream_t s);
    static void cg(const DevStencil& A, const double* diag, const double* b, double* x, double* work,
                   double rel_tol, int max_iter, int* result, int exact, cudaStream_t s);
    static void set_trace(long long* trace, int xmask);
    /// load the side-stream wave kernel now (lazy module loading of a kernel
    /// while the coarse march runs serialises its launch behind the march)
    static void preload_side(const DevHier& H);
};
extern template struct DegLaunch<1>;
extern template struct DegLaunch<2>;
extern template struct DegLaunch<3>;
extern template struct DegLaunch<4>;
extern template struct DegLaunch<5>;
extern template struct DegLaunch<6>;
extern template struct DegLaunch<7>;
extern template struct DegLaunch<8>;
/// Longs in the developer trace buffer (phi_set_tuning(.., .., -1)).
constexpr size_t kTraceLongs = 49152;

void launch_phi_wave(const DevHier& H, const DevStencil& Am, const WaveArgs& a, double* ws,
                     long long ws_stride, int max_slots, cudaStream_t s);
void launch_vcycle(const DevHier& H, const double* B, long long ldb, double* X, long long ldx, int nrhs,
                   double* ws, long long ws_stride, int max_slots, cudaStream_t s);
void launch_unit(const DevHier& H, int op, int arg, int arg2, const double* in, double* out, double* ws,
                 long long ws_stride, cudaStream_t s);
void launch_cg(const DevStencil& A, const double* diag, const double* b, double* x, double* work,
               double rel_tol, int max_iter, int* result, int exact, cudaStream_t s);
void launch_restrict_first(const double* fg, const double* fu, double* cg, double* cu, int n,
                           cudaStream_t s);
void launch_inject(const double* cu, double* fu, int n, int J, int m, cudaStream_t s);
/// the same for the C-points j0 <= j < j1
void launch_inject_range(const double* cu, double* fu, int n, int j0, int j1, int m, cudaStream_t s);
void launch_resid0(const double* g, const double* u, double* sq, int n, cudaStream_t s);
/// Reads n doubles (a multiple of 4, > L2): flushes L2 leaving clean lines.
void launch_l2_flush_read(const double* buf, size_t n, double* sink, cudaStream_t s);
/// force-load every kernel the overlapped coarse phase launches on its side
/// stream (inject, resid0, the side wave kernel of H's degree)
void preload_overlap_kernels(const DevHier& H);
void launch_copy(double* dst, const double* src, size_t n, cudaStream_t s);

// ---- device ILUT (ilut.cu) ------------------------------------------------
/// Dual-threshold ILUT of a square stencil operator on the device, bit-identical
/// to ilut_factor (ilut.hpp:29-143); factors returned as host CSR (L strictly
/// lower, U with its diagonal first).  Throws on a zero pivot.
void device_ilut(const DevStencil& A, double tau, int fill_limit, HostCsr& lower, HostCsr& upper, cudaStream_t s);

// ---- device assembly (assembly.cu) ---------------------------------------
/// 1D tables on the device for one direction (see Tables1D).
struct DevTables1D {
    int p, nq, nel;
    const double* w;      // [e*nq + q]
    const double* vals;   // [(e*nq + q)*(p+1) + a]
    const double* ders;
};

/// Galerkin mass / stiffness of the degree-p tensor basis, free rows,
/// stencil-major with offsets [-p, p]^2 and FULL-grid column validity
/// (boundary columns kept for lumping).  Either output may be null.
void launch_assemble_mk(const DevTables1D& tu, const DevTables1D& tv, double* mass, double* stiff,
                        cudaStream_t s);
/// Row-sum lumped mass (assembly.hpp:437-446) of the full matrix restricted to
/// free rows, inverted: inv[i] = 1 / sum_j M(i, j).  Returns status via flag.
void launch_lump_inv(const double* mass, int p, int nel, double* inv, int* bad, cudaStream_t s);
/// Mixed order-p / order-1 transfer (assembly.hpp:376-433), free rows/cols,
/// offsets [-p, 1]^2.
void launch_assemble_transfer(const DevTables1D& tu, const DevTables1D& tv, const double* low_u,
                              const double* low_v, double* t, cudaStream_t s);
/// Transpose a stencil operator (rows on grid R with offsets [lo, hi]) into one
/// with rows on the column grid and offsets [-hi, -lo].
void launch_stencil_transpose(const DevStencil& a, double* out, cudaStream_t s);
/// out = a + c * b elementwise (sparse_add on a shared pattern, sparse.hpp:148-178).
void launch_axpby(const double* a, double c, const double* b, double* out, size_t n, cudaStream_t s);
/// Y = A X for nrhs in {1, 16, 32, 64}; X, Y [n][nrhs]; At: the tiled copy of A
/// of kind tile_kind(nrhs) (launch_tile, tile_doubles doubles) (spmm.cu).
int tile_kind(int nrhs);
void launch_tile(const DevStencil& A, double* At, int kind, cudaStream_t s);
size_t tile_doubles(const DevStencil& A, int kind);
void launch_spmm(const DevStencil& A, const double* At, const double* X, double* Y, int nrhs, cudaStream_t s);
/// Line Gauss-Seidel coefficients of a 9-point order-1 level (9 n doubles).
void launch_gs_line_coeffs(const double* a, int nf, double* out, cudaStream_t s);
/// Load vector (assembly.hpp:365-371 + restrict_vector) for free dofs.
/// kind: 0 constant(c0); 1 ((c0 * c1) * sx) * sy  [amp * exp(-t) * sin * sin];
/// 2 (c0 * sx) * sy [amp * sin * sin]; 3 sx * sy; 4 spline with free coeffs.
void launch_assemble_load(const DevTables1D& tu, const DevTables1D& tv, int kind, double c0, double c1,
                          const double* sx, const double* sy, const double* coeffs, double* out,
                          cudaStream_t s);
/// f_k = f_k * (dt*theta) + (dt*(1-theta)) * f_{k-1}   (theta.hpp:186-191)
void launch_theta_combine(double* fk, const double* fkm1, double a, double b, int n, cudaStream_t s);
void launch_scale(double* v, double a, size_t n, cudaStream_t s);
void launch_recip(const double* v, double* out, int n, cudaStream_t s);

}  // namespace phi
