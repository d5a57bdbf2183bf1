// Host-side setup for the engine: 1D quadrature / B-spline tables that feed the
// device assembly, the ILUT factorization, the dense coarse LU and the
// triangular-solve schedules.  All of it runs once per hierarchy (setup time,
// outside the solve() window, as in the reference).
#pragma once

#include <vector>

#include "common.hpp"
#include "device_types.cuh"

namespace phi {

/// n-point Gauss-Legendre rule on [0, 1] (same values as quadrature.hpp:17-44).
struct GaussRule {
    std::vector<double> nodes, weights;
};
GaussRule gauss_legendre_01(int n);

/// Open uniform knot vector on [0, 1] (same knots as spline.hpp:48-63).
struct Knots {
    std::vector<double> t;
    int degree = 0;
    int n_basis = 0;
    int find_span(double xi) const;  // spline.hpp:28-32
};
Knots open_uniform_knots(int degree, int n_elements);

/// Per-element 1D quadrature + basis tables for one parametric direction
/// (restates assembly.hpp:83-151, DirTables / SpanQuadrature).  Layouts:
/// nodes/weights [e*nq + q], vals/ders [(e*nq + q)*(p+1) + a].
struct Tables1D {
    int p = 0, nq = 0, nel = 0;
    std::vector<double> nodes, weights, vals, ders;
    std::vector<int> first;
};
Tables1D build_tables(const Knots& kv, int nq);

/// Order-1 basis values on the knot spans of `low` evaluated at the nodes of
/// `high` (eval_nonzero, spline.hpp:133-139): [(e*nq + q)*2 + a], first index
/// per (e, q).
struct LowTables {
    std::vector<double> vals;
    std::vector<int> first;
};
LowTables build_low_tables(const Knots& low, const Tables1D& high);

/// Canonical order-1 embedding coarse -> fine on free dofs and its transpose
/// (restates p1_embedding_full + take_submatrix, pmultigrid.hpp:15-64).
HostCsr p1_embedding_free(int n_elements_fine);
HostCsr transpose(const HostCsr& a);

/// Dense LU with partial pivoting (same factors and permutation as solvers.hpp:136-167).
struct DenseLUHost {
    int n = 0;
    std::vector<double> lu;
    std::vector<int> piv;
};
DenseLUHost dense_lu_factor(const HostCsr& a);

/// Operator of the order-1 h-multigrid W-cycle (pmultigrid.hpp:184-200) from
/// level `lc` down, applied to a zero initial guess: the cycle is then linear
/// in its right-hand side, x = C b.  Returned column-major (C[j * n + i] =
/// (C e_j)_i), n = a[lc].n_rows.  a: the level matrices, e: the embeddings
/// (e[l]: level l+1 -> level l), coarse: the dense LU of the coarsest level.
/// Host restatement of the same cycle the device runs (setup only).
std::vector<double> wcycle_operator(const std::vector<HostCsr>& a, const std::vector<HostCsr>& e,
                                    const DenseLUHost& coarse, int lc, int gs_pre, int gs_post);

/// Level schedule of a triangular factor.  Rows of one level depend only on
/// rows of earlier levels.  A level is split into chunks of <= kTriRows rows
/// (one lane of the solving warp each) and <= kTriBlockCap bytes.  Entry e of
/// row l of chunk c lives at base[c] + e * nrows[c] + l.
///
/// Every row of a chunk is padded to the chunk's `span` (the longest row,
/// rounded up to even) with neutral dummies (column n, value +0.0): the device
/// keeps z[n] = +0.0 and s - (+0.0 * +0.0) == s exactly, so the padded sum is
/// bit-identical.
constexpr int kTriRows = 32;
struct TriPlan {
    int n = 0, n_levels = 0, n_chunks = 0, max_row_len = 0;
    std::vector<int> level_chunk;  // n_levels + 1
    std::vector<int> chunk_meta;   // 4 per chunk: row0, nrows, base, span
    std::vector<int> rows;         // permuted original row indices
    std::vector<int> lens;         // true length per permuted row
    std::vector<int> cols;         // interleaved
    std::vector<double> vals;
    std::vector<double> diag;      // upper only, by original row
};
TriPlan plan_lower(const HostCsr& lower);
TriPlan plan_upper(const HostCsr& upper);
/// Level schedule of a lexicographic Gauss-Seidel sweep (rows: off-diagonal
/// entries in CSR order, diag = the diagonal; levels = wavefronts).
TriPlan plan_gauss_seidel(const HostCsr& a, bool backward);

/// Level-ordered stream for the TMA-fed warp solve.  The factor is a sequence
/// of blocks (one per plan chunk: rows of one level), packed into fetch units
/// of <= kTriUnitCap bytes; one cp.async.bulk moves one unit into a slot of the
/// shared-memory ring.
///   unit header (16 B): n_blocks, next_off16, next_bytes (unit
///                       u + kTriSlots - 1, 0 if none), pad; then uint16
///                       byte offsets of the unit's blocks (padded to 16 B)
///   block header (32 B): nr, span | m, lg, block_bytes, cols_off, vals_off,
///                        diag_off, pad
///   rows  int32[nr]   at 32 (padded to 8 bytes)
///   diag  double[nr]  at diag_off (upper only), rdiag = RN(1 / diag) after it
/// Exact layout (the reference's summation order): cols int32[span][nr],
/// vals double[span][nr], entry e of row l at e * nr + l, rows padded to
/// `span` (even) with neutral dummies.
/// Fast layout (reassociated sums): G = 2^lg lanes per row; lane L = r G + k
/// owns entries [k m, (k + 1) m) of row r, stored entry-major over a full
/// warp: cols int32[m][32], vals double[m][32] (slot q of lane L at
/// q * 32 + L), padded with dummies.
/// Dummies are column n with value +0.0 (the device keeps z[n] = +0.0), so
/// they are exactly neutral.  Offsets in headers are bytes from the block /
/// unit start; `next_off16` and `prime` are 16-byte units of `stream`;
/// `prime` holds (off16, bytes) of the first kTriSlots - 1 units.
constexpr int kTriUnitCap = 10 * 1024;
struct TriStream {
    std::vector<unsigned char> stream;
    std::vector<int> prime;  // 2 * (kTriSlots - 1)
    int n_blocks = 0;        // blocks (levels / level slices)
    int n_units = 0;
    int max_unit_bytes = 0;
    std::vector<int> block_info;  // 4 per block: unit, byte offset in the unit, first in unit, 0
};
TriStream make_tri_stream(const TriPlan& p, bool fast);

/// Block-recurrence schedule of a sweep (reassociated mode only).  The rows
/// are taken in solve order in blocks of kBlkRows = 32 consecutive rows, one
/// per lane.  For block k with rows R_k the sweep
///     x_i = (rhs_i - sum_{j before i} a_ij x_j(new) - sum_{j after i} a_ij x_j(old)) / d_i
/// (d_i = 1 for the unit lower ILUT factor) is
///     x_{R_k} = B_k^{-1} (rhs - old) - G_k x_{R_{k-1}},   B_k = D + (in-block lower part),
/// with the dense inverse B_k^{-1} and the folded coupling G_k = B_k^{-1} N_k
/// (N_k: the entries whose columns block k-1 solves) precomputed here in
/// extended precision.  Only G_k x_{R_{k-1}} -- a dense product over the last
/// 8 mf rows of block k-1 -- is on the block-to-block critical path; the
/// inverse product no longer is.  Entries of a row are
///   in-block lower  -> folded into B_k;
///   fresh           -> columns solved by block k-1 (F = 1): folded into G_k;
///   old             -> columns solved by blocks <= k-F-1 (final once block
///                      k-F-1 is done) or solved later (Gauss-Seidel's old values,
///                      in-block ones included); summed ahead of time by the
///                      worker warps, split into `parts` interleaved parts.
/// One block = one fetch unit (one cp.async.bulk):
///   header int32[4]: mo (old slots per part), 0, bytes, mf (groups of four column pairs of G_k)
///   rows   int32[32]                 at 16 (-1 on padding lanes)
///   inv    lower triangle of B_k^{-1} at 144, 4352 bytes: entries (L, 2p),
///                                    (L, 2p+1) for L >= 2p at (p (31 - p) + L) * 16
///                                    bytes (PHI_BLK_TRI = 0: the full double[16][32][2])
///   G      double[4 mf][32][2]       at kBlkFreshOff: pair q of lane L holds
///                                    G_k(L, 30 - 2q), G_k(L, 31 - 2q)
///   old    per part q: cols int32[mo][32], vals double[mo][32] at
///          kBlkFreshOff + 2048 mf + q * 384 mo  (slot s of lane L at s*32+L)
/// Padding slots are (column n, +0.0) against the zero slot x[n].  `table`
/// holds (offset / 16, bytes, mf, 0) per block.
constexpr int kBlkRows = 32;
constexpr int kBlkInvOff = 144;
/// PHI_BLK_TRI: the inverse (lower triangular in solve order) is stored as its
/// lower triangle -- column pair p keeps rows 2p .. 31 only, the pair of lane L
/// at slot p (31 - p) + L (16 bytes each; 272 slots = 4352 bytes instead of
/// 8192); lanes above the diagonal load nothing and use exact zeros.
#ifndef PHI_BLK_TRI
#define PHI_BLK_TRI 1
#endif
constexpr int kBlkTri = PHI_BLK_TRI;
constexpr int kBlkInvBytes = kBlkTri ? 16 * 272 : 8 * kBlkRows * kBlkRows;
constexpr int kBlkFreshOff = kBlkInvOff + kBlkInvBytes;
#ifndef PHI_BLK_SOLVERS
#define PHI_BLK_SOLVERS 2
#endif
constexpr int kBlkSolvers = PHI_BLK_SOLVERS;                  // solver warps in rotation
constexpr int kBlkMaxParts = PHI_THREADS / 32 - kBlkSolvers;  // worker warps
constexpr int kBlkFresh = 1;     // fresh distance F: columns of block k-1 (folded into G_k)
struct BlkStream {
    std::vector<unsigned char> stream;
    std::vector<int> table;  // 4 per block: offset / 16, bytes, G pair groups, 0
    int n = 0, n_blocks = 0, parts = 1, mf0 = 0, lookahead = 0, max_unit_bytes = 0;
    int win = 0;   // rolling-window layout (below), 0: absolute columns
    int desc = 0;  // solve order descending: block k, lane l solves row n - 1 - (32 k + l)
};
/// Rolling-window layout (win = WZ, a power of two; ILUT substitutions whose
/// vector does not fit in shared memory).  The factors are banded: every
/// column a row reads was solved at most `span` rows earlier in solve order
/// (ilut_span).  With WZ > span + 32 the device keeps only the last WZ solved
/// values in a shared-memory ring (slot j & (WZ - 1)) and writes the solution
/// through to global memory.  Columns in the stream are then window slots
/// (col & (WZ - 1); padding: the zero slot WZ) and the old entries are packed
/// with 16-bit columns: per part q, cols uint16[mo][32], vals double[mo][32]
/// at kBlkFreshOff + 2048 mf + q * 320 mo.
constexpr int kBlkMaxWin = 4096;
/// Largest distance in solve order between a row and a column it reads, over
/// both factors (the band of the IgA ILUT factors).
int ilut_span(const HostCsr& lower, const HostCsr& upper);
/// Window size for a span: the power of two >= span + 64 (0 if above kBlkMaxWin).
int blk_window_for(int span);
/// Unit lower ILUT factor (strictly lower entries stored), ascending.
BlkStream blk_lower(const HostCsr& lower, int win = 0);
/// Upper ILUT factor (diagonal first in each row), descending.
BlkStream blk_upper(const HostCsr& upper, int win = 0);
/// Lexicographic Gauss-Seidel sweep on A (solvers.hpp:80-99).
BlkStream blk_gauss_seidel(const HostCsr& a, bool backward);

}  // namespace phi
