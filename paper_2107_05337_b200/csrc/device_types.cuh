// Plain-old-data views of the device-resident operators, passed by value to the
// kernels (they live in the kernel parameter bank: uniform, cached loads).
#pragma once

#include <cstdint>

namespace phi {

/// Tensor-product stencil operator ("blocked CSR" of a clamped-rectangle
/// B-spline pattern, assembly.hpp:157-193 after Dirichlet elimination).
/// Rows live on an ru x rv grid, columns on a cu x cv grid; row (iu, iv) holds
/// columns (iu + du, iv + dv), du, dv in [lo, hi], clamped to the column grid.
/// Column indices are implicit.  Values are stencil-major:
///   vals[e * (ru*rv) + row],  e = (dv - lo) * (hi - lo + 1) + (du - lo)
/// so a warp over consecutive rows reads one coalesced 256 B line per entry.
/// The (dv, du)-ascending entry order is the reference CSR column order, so a
/// sequential sum over e reproduces spmv (sparse.hpp:114-124) bit for bit.
struct DevStencil {
    int ru, rv, cu, cv, lo, hi;
    const double* vals;
};

/// Generic CSR (sparse.hpp:17-22) -- used for the h-chain embeddings.
struct DevCsr {
    int n_rows, n_cols;
    const int* ro;
    const int* ci;
    const double* v;
};

/// Depth of the shared-memory ring that stages triangular-factor blocks.
constexpr int kTriSlots = 8;
/// Block sweeps: maximum ring depth and the depth of the worker -> solver
/// hand-off ring.
constexpr int kBlkMaxSlots = 8;
constexpr int kBlkHand = 4;
constexpr int kBlkMinSlots = 3;  // workers wait for unit g once block g - 3 is done
/// Warps that take turns on the blocks of a fast (reassociated) sweep.
constexpr int kSweepWarps = 6;
/// Bytes per triangular-factor block (TriPlan chunking) and the product
/// scratch that bound implies (12 bytes per entry: int32 column + fp64 value).
constexpr int kTriBlockCap = 5 * 1024;
constexpr int kTriMaxItems = kTriBlockCap / 12;

/// Level-scheduled triangular factor as a TMA block stream (TriStream).
struct DevTri {
    int n, n_levels, n_units, n_blocks;
    int max_unit_bytes;
    int prime[2 * (kTriSlots - 1)];  // (off16, bytes) of the first kTriSlots - 1 units
    const unsigned char* stream;  // 16-byte aligned
    const int4* blocks;           // per block: unit, byte offset in the unit, first-in-unit flag, 0
};

/// Block-recurrence sweep (BlkStream, setup_host.hpp): one fetch unit per
/// block of 32 rows in solve order; `table` holds (offset / 16, bytes).
struct DevBlk {
    int n, n_blocks, parts, mf0, lookahead, max_unit_bytes;
    int win;   // rolling-window layout (BlkStream::win), 0: absolute columns
    int desc;  // rows in descending order (upper factor, backward sweep)
    const unsigned char* stream;  // 16-byte aligned
    const int4* table;  // per block: offset / 16, bytes, fresh slots, 0
};

struct DevHLevel {
    DevStencil a;    // M_l + c K_l, 9-point
    DevTri gs_fwd, gs_bwd;  // Gauss-Seidel sweeps as level-scheduled streams (exact mode; empty on the coarsest)
    DevBlk gsb_fwd, gsb_bwd;  // the same sweeps as block recurrences (reassociated mode)
    // reassociated mode, nf <= kLineMax: line sweeps (gs_line_coeffs_kernel
    // layout: double4 forward[n], double4 backward[n], double rd[n]); null: none
    const double* gsl;
    int nf;
    DevCsr embed;    // level l+1 -> level l (empty on the coarsest)
    DevCsr embed_t;  // its transpose (restriction rows, ascending fine index)
    int n;
};

constexpr int kMaxH = 12;
/// Scratch of the cluster dense coarse product: r copy (<= 1024) + 256 partials.
constexpr int kClScratch = 1024 + 288;
/// Longest grid line of a line Gauss-Seidel sweep (32 lanes x 8 rows).
constexpr int kLineMax = 256;
/// Shortest grid line swept by lines (shorter levels: block sweeps).
constexpr int kLineMin = 24;

/// One p-multigrid hierarchy (PMultigridHierarchy, pmultigrid.hpp:215-324)
/// plus the spatial solver settings of its ThetaStepper (theta.hpp:66-75).
struct DevHier {
    int n_p, n_1, n_h;
    DevStencil A;   // A_p = M_p + c K_p
    DevStencil T;   // transfer_p1 (rows order p, cols order 1)
    DevStencil Tt;  // its transpose
    const double* inv_lp;
    const double* inv_l1;
    DevTri L, U;    // level-scheduled ILUT factors (exact mode)
    DevBlk Lb, Ub;  // block-recurrence ILUT factors (reassociated mode)
    DevHLevel h[kMaxH];
    const double* coarse_lu;
    const int* coarse_piv;
    int coarse_n;
    // reassociated mode: the W-cycle from h-level dense_level down (zero
    // initial guess) as a dense n x n operator, column-major (-1: none)
    int dense_level;
    const double* dense_op;
    int dense_level_cl;  // the same for cluster mode (larger: split over the cluster)
    const double* dense_op_cl;
    int nu_pre, nu_post, gs_pre, gs_post;
    double rel_tol;
    int max_iter;
    int fixed_cycles;
    int exact;  // 1: the reference's sequential summation order; 0: reassociated sums
    // SpatialSolverKind (theta.hpp:64): 0 p-multigrid, 1 Jacobi-preconditioned CG
    // (solvers.hpp:21-75; then only n_p, A and diag are set, n_h = 0)
    int kind;
    const double* diag;  // cg kind: diagonal_of(A) (sparse.hpp:180-184), the centre plane of A
};

/// Shared-memory placement of the latency-critical vectors of one CTA (offsets
/// in doubles into dynamic shared memory; -1 = global workspace).
struct SmemPlan {
    int ring_off;          // triangular-factor block ring (TMA staging)
    int slot_bytes;        // bytes per ring slot
    int n_slots;           // ring depth (block sweeps; level streams use kTriSlots)
    int gs_slot_bytes;     // ring slot / depth of the W-cycle phase (block sweeps)
    int gs_n_slots;
    int prod_off;          // triangular-solve product scratch (kTriMaxItems)
    int dot_off;           // ordered-dot scratch
    int z_off;             // in-place triangular-solve vector (n_p + 1)
    int lvl_off[kMaxH];    // per h-level: b, x, r (3 n_l)
    int cl_scr_off;        // cluster dense-apply scratch (kClScratch doubles) free during the W-cycle, -1: none
    int win_off;           // rolling window of the ILUT substitutions (win + 2 doubles), -1: none
    int total;             // doubles
};

/// Work description of one batched wave of Phi applications (one CTA per
/// right-hand side; see phi_kernels.cu).
enum PhiMode : int { kModeStep = 0, kModeSolve = 1 };
enum PhiEpi : int {
    kEpiStore = 0,     // U[k] = x + g[k]                (step_into, mgrit.hpp:253-258)
    kEpiRestrict = 1,  // CG[j] = x + g[k] - U[k]; CU[j] = 0   (mgrit.hpp:151-167)
    kEpiResid = 2,     // SQ[k] = |x + g[k] - U[k]|^2          (mgrit.hpp:197-214)
    kEpiNorm = 3,      // SQ[k] = |x|^2                        (mgrit.hpp:292-310)
    kEpiSolve = 4      // X[task] = x                          (solve / step API)
};

struct WaveArgs {
    int mode, epi;
    int n_tasks, task_len;
    const int* task_k0;  // per task: first time index k (step mode) or unused
    int n;               // n_p
    // level state, [k][n] row-major
    double* U;
    const double* G;
    const double* LOAD;
    int load_steady;
    const double* AMINUS_X;  // unused placeholder
    // restrict outputs
    double* CG;
    double* CU;
    int m;
    double* SQ;
    // plain batched solve / step API (strided vectors)
    const double* B;
    long long ldb;
    double* X;
    long long ldx;
    const double* UPREV;  // step API: u_prev rows
    long long ldu;
    const double* LOADV;  // step API: per-rhs load rows (nullable)
    long long ldl;
    int x0_empty;
    int guess_prev;  // step mode on U: guess = U[k-1] (sequential_integrate) instead of U[k]
    // per-task results (nullable)
    int* iters_out;
    int* conv_out;
    double* rel_out;
    // device counters
    int* wave_max;             // per-launch stats (nullable): [0] max cycles, [1] sum, [2] points
    unsigned long long* stat;  // [0] solves, [1] iterations
    int* err;                  // [0] flag, [1] first k, [2] level
    double* err_rel;
    int level;
    // overlap of the coarse march with the next phases (Mgrit::coarse_overlapped):
    // after every completed task step the main CTA publishes the time index k
    // just finished to this host-mapped counter (null: none)
    volatile unsigned* progress;
    int no_cluster;  // 1: one CTA per task even for few tasks (the side-stream waves)
};

}  // namespace phi
