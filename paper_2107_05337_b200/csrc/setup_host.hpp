// Host-side setup for the engine: 1D quadrature / B-spline tables that feed the
// device assembly, the ILUT factorization, the dense coarse LU and the
// triangular-solve schedules.  All of it runs once per hierarchy (setup time,
// outside the solve() window, as in the reference).
#pragma once

#include <vector>

#include "common.hpp"

namespace phi {

/// n-point Gauss-Legendre rule on [0, 1] (restates quadrature.hpp:17-44).
struct GaussRule {
    std::vector<double> nodes, weights;
};
GaussRule gauss_legendre_01(int n);

/// Open uniform knot vector on [0, 1] (restates spline.hpp:17-63).
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

/// Dual-threshold ILUT (restates ilut.hpp:29-143).  Throws on a zero pivot.
void ilut_factor(const HostCsr& a, double tau, int fill_limit, HostCsr& lower, HostCsr& upper);

/// Dense LU with partial pivoting (restates solvers.hpp:102-172).
struct DenseLUHost {
    int n = 0;
    std::vector<double> lu;
    std::vector<int> piv;
};
DenseLUHost dense_lu_factor(const HostCsr& a);

/// Level-ordered, lane-interleaved layout of a triangular factor for the
/// sync-free device solve.  Rows of one level are independent; a level is
/// split into chunks of <= 32 rows (one lane per row).  Entry e of lane l of
/// chunk c lives at base[c] + e * nrows[c] + l (coalesced per warp).
///
/// Every row of a chunk is padded to the chunk's `span` entries (a multiple of
/// kTriRing, plus one extra ring block so prefetches never leave the chunk)
/// with neutral dummies (column n, value +0.0): the device keeps z[n] = +0.0,
/// and s - (+0.0 * +0.0) == s exactly, so the padded sum is bit-identical.
constexpr int kTriRing = 8;
constexpr int kTriRows = 8;  // rows per chunk (one lane each)
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

/// Level-ordered block stream for the TMA-fed, level-synchronous device solve.
/// One block = one chunk (<= kTriRows rows of a single level) with every
/// entry of its rows, stored so that a single cp.async.bulk fetches it:
///   header (32 B): nr, span (entries per row, even), row0,
///                  next_off16, next_bytes (block b + kTriSlots - 1, 0 if none),
///                  3 x pad
///   rows: 8 x int32 (original row index per lane), diag: 8 x double (U only)
///   cols: span x nr int32   (entry e of row l at e * nr + l)
///   vals: span x nr double
/// Offsets are in 16-byte units of `stream`; `prime` holds (off16, bytes) of
/// the first kTriSlots - 1 blocks.
constexpr int kTriSlots = 4;
constexpr int kTriBlockPrefix = 128;  // header + rows + diag
struct TriStream {
    std::vector<unsigned char> stream;
    std::vector<int> prime;  // 2 * (kTriSlots - 1)
    int n_blocks = 0;
    int max_block_bytes = 0;
    int max_items = 0;       // max nr * span over blocks (product scratch)
};
TriStream make_tri_stream(const TriPlan& p);

}  // namespace phi
