// Host setup for the engine.  The numerical routines here (Gauss-Legendre rule,
// B-spline values / derivatives, dense LU) are written in the engine's own
// formulation but perform, per output value, the same sequence of IEEE
// operations as the reference routine each one cites (compiled with
// -ffp-contract=off), so the device operators built from these tables are
// bit-identical to the reference's.  tests/test_setup_host_cpu.py pins them
// against fixtures made by the compiled reference (phi_setup_* in the C ABI).
#include "setup_host.hpp"

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <functional>
#include <queue>
#include <string>

namespace phi {

namespace {

// P_n(x) and P_{n-1}(x) from k P_k = (2k-1) x P_{k-1} - (k-1) P_{k-2}.
struct LegendrePair {
    double pn, pnm1;
};
LegendrePair legendre_pair(int n, double x) {
    double below = 1.0, top = x;  // P_0, P_1
    for (int k = 2; k <= n; ++k) {
        const double up = (double(2 * k - 1) * x * top - double(k - 1) * below) / double(k);
        below = top;
        top = up;
    }
    return {top, below};
}

}  // namespace

// Roots of P_n by Newton from the Chebyshev-like guesses cos(pi (i + 3/4) / (n + 1/2)),
// the slope from (x^2 - 1) P_n' = n (x P_n - P_{n-1}); the rule on [-1, 1] has
// weights 2 / ((1 - x^2) P_n'^2), halved for [0, 1].  Same arithmetic per root as
// quadrature.hpp:17-44 (the tables feed a bit-exact assembly).
GaussRule gauss_legendre_01(int n) {
    if (n < 1) throw InvalidArgument("gauss_legendre_01: n must be >= 1");
    constexpr double kPi = 3.14159265358979323846;
    constexpr int kNewtonCap = 100;
    constexpr double kNewtonStep = 1e-15;
    GaussRule rule{std::vector<double>(n), std::vector<double>(n)};
    for (int i = 0; i < n; ++i) {
        double root = std::cos(kPi * (i + 0.75) / (n + 0.5));  // descending in i
        double slope = 0.0;
        for (int sweep = 0; sweep < kNewtonCap; ++sweep) {
            const LegendrePair P = legendre_pair(n, root);
            slope = n * (root * P.pn - P.pnm1) / (root * root - 1.0);
            const double step = P.pn / slope;
            root -= step;
            if (std::abs(step) < kNewtonStep) break;
        }
        rule.nodes[i] = 0.5 * (1.0 - root);  // ascending on [0, 1]
        rule.weights[i] = 1.0 / ((1.0 - root * root) * slope * slope);
    }
    return rule;
}

// The last knot s in [degree, n_basis) with t[s] <= xi (the right end maps to the
// last span): a uniform-spacing guess, corrected against the knots themselves, so
// the answer is the one a search over the knots gives (spline.hpp:28-32).
int Knots::find_span(double xi) const {
    const int lo = degree, hi = n_basis;  // spans lo .. hi-1
    if (xi >= t[hi]) return hi - 1;
    if (!(xi >= t[lo])) return lo - 1;
    const double rel = (xi - t[lo]) / (t[hi] - t[lo]);
    int s = lo + std::min(hi - lo - 1, std::max(0, static_cast<int>(rel * (hi - lo))));
    while (s > lo && t[s] > xi) --s;
    while (t[s + 1] <= xi) ++s;  // t[hi] > xi stops it
    return s;
}

// degree+1 copies of 0, the interior multiples of 1/n_elements, degree+1 copies of 1.
Knots open_uniform_knots(int degree, int n_elements) {
    if (degree < 1) throw InvalidArgument("open_uniform_knots: degree must be >= 1");
    if (n_elements < 1) throw InvalidArgument("open_uniform_knots: n_elements must be >= 1");
    Knots kv;
    kv.degree = degree;
    kv.n_basis = n_elements + degree;
    const double h = 1.0 / n_elements;
    kv.t.reserve(kv.n_basis + degree + 1);
    kv.t.assign(degree + 1, 0.0);
    for (int e = 1; e < n_elements; ++e) kv.t.push_back(e * h);
    kv.t.insert(kv.t.end(), degree + 1, 1.0);
    return kv;
}

namespace {

// One degree-raising step of the Cox-de Boor recurrence on the span [t[s], t[s+1]):
// with a_r = t[s+r+1] - xi, b_r = xi - t[s+1-d+r] and q_r = N_r^{d-1} / (a_r + b_r),
// N_r^d = b_{r-1} q_{r-1} + a_r q_r.  In place: N[0..d-1] holds degree d-1 on
// entry, N[0..d] degree d on exit.
inline void raise_degree(const std::vector<double>& t, int s, double xi, int d, double* N) {
    double carry = 0.0;
    for (int r = 0; r < d; ++r) {
        const double a = t[s + r + 1] - xi;
        const double b = xi - t[s + 1 - d + r];
        const double q = N[r] / (a + b);
        N[r] = carry + a * q;
        carry = b * q;
    }
    N[d] = carry;
}

// Values and first derivatives of the degree+1 functions alive at xi, in one
// pass up the degrees: the degree p-1 row is kept when it goes by, and
// N_i' = p (g_i - g_{i+1}), g_i = N_i^{p-1} / (t[i+p] - t[i])  (spline.hpp:104-130).
// Returns the index of the first of them.
int values_and_derivs(const Knots& kv, double xi, double* vals, double* ders) {
    const int p = kv.degree;
    const int s = kv.find_span(xi);
    const int first = s - p;
    double g[34];
    vals[0] = 1.0;
    for (int d = 1; d < p; ++d) raise_degree(kv.t, s, xi, d, vals);
    // vals[0..p-1]: degree p-1 functions first+1 .. first+p; g[r] belongs to function first+r
    g[0] = g[p + 1] = 0.0;
    for (int r = 1; r <= p; ++r) {
        const double width = kv.t[first + r + p] - kv.t[first + r];
        g[r] = width > 0.0 ? vals[r - 1] / width : 0.0;
    }
    raise_degree(kv.t, s, xi, p, vals);
    for (int r = 0; r <= p; ++r) ders[r] = p * (g[r] - g[r + 1]);
    return first;
}

}  // namespace

// One row per (element, quadrature point): the point's parametric coordinate,
// its weight scaled by the element length, and the p+1 values / derivatives
// alive there.  Elements are the knot spans of positive length, in order.
Tables1D build_tables(const Knots& kv, int nq) {
    const int p = kv.degree;
    const GaussRule unit = gauss_legendre_01(nq);
    Tables1D tb;
    tb.p = p;
    tb.nq = nq;
    for (int s = p; s < kv.n_basis; ++s) {
        const double x0 = kv.t[s], len = kv.t[s + 1] - kv.t[s];
        if (!(kv.t[s + 1] > x0)) continue;
        ++tb.nel;
        for (int q = 0; q < nq; ++q) {
            tb.nodes.push_back(x0 + unit.nodes[q] * len);
            tb.weights.push_back(unit.weights[q] * len);
        }
    }
    const size_t width = static_cast<size_t>(p) + 1, points = tb.nodes.size();
    tb.vals.resize(points * width);
    tb.ders.resize(points * width);
    tb.first.resize(tb.nel);
    for (size_t pt = 0; pt < points; ++pt)
        tb.first[pt / nq] = values_and_derivs(kv, tb.nodes[pt], &tb.vals[pt * width], &tb.ders[pt * width]);
    return tb;
}

LowTables build_low_tables(const Knots& low, const Tables1D& high) {
    LowTables lt;
    const int n = high.nel * high.nq;
    lt.vals.resize(static_cast<size_t>(n) * 2);
    lt.first.resize(n);
    for (int i = 0; i < n; ++i) {
        double v[2], d[2];
        lt.first[i] = values_and_derivs(low, high.nodes[i], v, d);
        lt.vals[2 * i] = v[0];
        lt.vals[2 * i + 1] = v[1];
    }
    return lt;
}

HostCsr p1_embedding_free(int nel_f) {
    if (nel_f % 2 != 0) throw InvalidArgument("p1_embedding_full: fine element count must be even");
    const int nf = nel_f + 1, nc = nel_f / 2 + 1;
    const int nff = nf - 2, ncf = nc - 2;  // free nodes per direction
    auto entries = [](int i, int* idx, double* w) {
        if (i % 2 == 0) {
            idx[0] = i / 2;
            w[0] = 1.0;
            return 1;
        }
        idx[0] = (i - 1) / 2;
        w[0] = 0.5;
        idx[1] = (i + 1) / 2;
        w[1] = 0.5;
        return 2;
    };
    HostCsr e;
    e.n_rows = nff * nff;
    e.n_cols = ncf * ncf;
    for (int iv = 1; iv <= nff; ++iv) {
        int jvs[2], jus[2];
        double wvs[2], wus[2];
        const int nv = entries(iv, jvs, wvs);
        for (int iu = 1; iu <= nff; ++iu) {
            const int nu = entries(iu, jus, wus);
            // (jv, ju) ascending == ascending global / free column index
            for (int a = 0; a < nv; ++a) {
                if (jvs[a] < 1 || jvs[a] > ncf) continue;
                for (int b = 0; b < nu; ++b) {
                    if (jus[b] < 1 || jus[b] > ncf) continue;
                    e.col_indices.push_back((jus[b] - 1) + ncf * (jvs[a] - 1));
                    e.values.push_back(wus[b] * wvs[a]);
                }
            }
            e.row_offsets.push_back(e.nnz());
        }
    }
    return e;
}

HostCsr transpose(const HostCsr& a) {
    HostCsr t;
    t.n_rows = a.n_cols;
    t.n_cols = a.n_rows;
    t.row_offsets.assign(a.n_cols + 1, 0);
    for (int c : a.col_indices) ++t.row_offsets[c + 1];
    for (int i = 0; i < a.n_cols; ++i) t.row_offsets[i + 1] += t.row_offsets[i];
    t.col_indices.resize(a.col_indices.size());
    t.values.resize(a.values.size());
    std::vector<int> next(t.row_offsets.begin(), t.row_offsets.end() - 1);
    for (int i = 0; i < a.n_rows; ++i)
        for (int e = a.row_offsets[i]; e < a.row_offsets[i + 1]; ++e) {
            const int pos = next[a.col_indices[e]]++;
            t.col_indices[pos] = i;
            t.values[pos] = a.values[e];
        }
    return t;
}

// LU with partial pivoting on a row-indirected dense copy: rows never move,
// `order` names the row at each position and becomes the permutation.  The pivot
// is the first largest |entry| below the diagonal, multipliers and updates are
// those of solvers.hpp:136-167 (zero multipliers skip their row), so the packed
// factors equal the reference's bit for bit.
DenseLUHost dense_lu_factor(const HostCsr& a) {
    if (a.n_rows != a.n_cols) throw InvalidArgument("DenseLU: matrix not square");
    const int n = a.n_rows;
    std::vector<double> work(static_cast<size_t>(n) * n, 0.0);
    for (int i = 0; i < n; ++i)
        for (int e = a.row_offsets[i]; e < a.row_offsets[i + 1]; ++e)
            work[static_cast<size_t>(i) * n + a.col_indices[e]] = a.values[e];
    std::vector<int> order(n);
    for (int i = 0; i < n; ++i) order[i] = i;
    auto row = [&](int pos) { return work.data() + static_cast<size_t>(order[pos]) * n; };
    for (int k = 0; k < n; ++k) {
        int where = k;
        double big = std::abs(row(k)[k]);
        for (int pos = k + 1; pos < n; ++pos) {
            const double mag = std::abs(row(pos)[k]);
            if (mag > big) big = mag, where = pos;
        }
        if (big == 0.0) throw std::runtime_error("DenseLU: singular matrix");
        std::swap(order[k], order[where]);
        const double* top = row(k);
        for (int pos = k + 1; pos < n; ++pos) {
            double* r = row(pos);
            const double mult = r[k] / top[k];
            r[k] = mult;
            if (mult == 0.0) continue;
            for (int j = k + 1; j < n; ++j) r[j] -= mult * top[j];
        }
    }
    DenseLUHost f;
    f.n = n;
    f.lu.resize(work.size());
    for (int pos = 0; pos < n; ++pos) std::copy(row(pos), row(pos) + n, f.lu.begin() + static_cast<size_t>(pos) * n);
    f.piv = std::move(order);
    return f;
}

namespace {
void host_spmv(const HostCsr& a, const double* x, double* y) {
    for (int i = 0; i < a.n_rows; ++i) {
        double acc = 0.0;
        for (int k = a.row_offsets[i]; k < a.row_offsets[i + 1]; ++k) acc += a.values[k] * x[a.col_indices[k]];
        y[i] = acc;
    }
}
void host_gs(const HostCsr& a, const double* b, double* x, bool backward) {  // solvers.hpp:80-99
    const int n = a.n_rows;
    for (int s = 0; s < n; ++s) {
        const int i = backward ? n - 1 - s : s;
        double acc = b[i], d = 0.0;
        for (int k = a.row_offsets[i]; k < a.row_offsets[i + 1]; ++k) {
            if (a.col_indices[k] == i)
                d = a.values[k];
            else
                acc -= a.values[k] * x[a.col_indices[k]];
        }
        x[i] = acc / d;
    }
}
void host_lu_solve(const DenseLUHost& f, const double* b, double* x) {  // solvers.hpp:118-133
    const int n = f.n;
    for (int i = 0; i < n; ++i) x[i] = b[f.piv[i]];
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < i; ++j) x[i] -= f.lu[static_cast<size_t>(i) * n + j] * x[j];
    for (int i = n - 1; i >= 0; --i) {
        for (int j = i + 1; j < n; ++j) x[i] -= f.lu[static_cast<size_t>(i) * n + j] * x[j];
        x[i] /= f.lu[static_cast<size_t>(i) * n + i];
    }
}
void host_wcycle(const std::vector<HostCsr>& a, const std::vector<HostCsr>& e, const DenseLUHost& coarse, int l,
                 int gs_pre, int gs_post, const double* b, double* x) {
    if (l + 1 == static_cast<int>(a.size())) {
        host_lu_solve(coarse, b, x);
        return;
    }
    const int n = a[l].n_rows, nc = e[l].n_cols;
    for (int s = 0; s < gs_pre; ++s) host_gs(a[l], b, x, false);
    std::vector<double> r(n), rc(nc, 0.0), ec(nc, 0.0);
    host_spmv(a[l], x, r.data());
    for (int i = 0; i < n; ++i) r[i] = b[i] - r[i];
    for (int i = 0; i < n; ++i)  // rc = E^T r
        for (int k = e[l].row_offsets[i]; k < e[l].row_offsets[i + 1]; ++k) rc[e[l].col_indices[k]] += e[l].values[k] * r[i];
    host_wcycle(a, e, coarse, l + 1, gs_pre, gs_post, rc.data(), ec.data());
    host_wcycle(a, e, coarse, l + 1, gs_pre, gs_post, rc.data(), ec.data());
    host_spmv(e[l], ec.data(), r.data());
    for (int i = 0; i < n; ++i) x[i] += r[i];
    for (int s = 0; s < gs_post; ++s) host_gs(a[l], b, x, true);
}
}  // namespace

std::vector<double> wcycle_operator(const std::vector<HostCsr>& a, const std::vector<HostCsr>& e,
                                    const DenseLUHost& coarse, int lc, int gs_pre, int gs_post) {
    const int n = a.at(lc).n_rows;
    std::vector<double> c(static_cast<size_t>(n) * n), b(n), x(n);
    for (int j = 0; j < n; ++j) {
        std::fill(b.begin(), b.end(), 0.0);
        std::fill(x.begin(), x.end(), 0.0);
        b[j] = 1.0;
        host_wcycle(a, e, coarse, lc, gs_pre, gs_post, b.data(), x.data());
        std::copy(x.begin(), x.end(), c.begin() + static_cast<size_t>(j) * n);
    }
    return c;
}

namespace {

// Row view of a level-scheduled sweep: row i's dependency columns, its
// summed entries (columns ascending = the reference's order) and, for a
// dividing sweep, its diagonal.
struct SweepRows {
    std::function<void(int, std::vector<int>&)> deps;
    std::function<void(int, std::vector<int>&, std::vector<double>&)> entries;
    std::function<double(int)> diag;  // empty: unit diagonal
};

TriPlan make_plan(int n, bool descending, const SweepRows& rv) {
    TriPlan p;
    p.n = n;
    std::vector<int> level(n, 0), dep;
    int max_level = -1;
    auto row_level = [&](int i) {
        int lv = 0;
        rv.deps(i, dep);
        for (int j : dep) lv = std::max(lv, level[j] + 1);
        level[i] = lv;
        max_level = std::max(max_level, lv);
    };
    if (descending)
        for (int i = n - 1; i >= 0; --i) row_level(i);
    else
        for (int i = 0; i < n; ++i) row_level(i);
    p.n_levels = max_level + 1;
    // bucket rows by level; within a level keep solve order
    std::vector<std::vector<int>> by_level(p.n_levels);
    if (descending)
        for (int i = n - 1; i >= 0; --i) by_level[level[i]].push_back(i);
    else
        for (int i = 0; i < n; ++i) by_level[level[i]].push_back(i);
    std::vector<std::vector<int>> rc(n);
    std::vector<std::vector<double>> rvv(n);
    for (int i = 0; i < n; ++i) rv.entries(i, rc[i], rvv[i]);
    p.level_chunk.push_back(0);
    for (int lv = 0; lv < p.n_levels; ++lv) {
        const auto& rs = by_level[lv];
        for (size_t c0 = 0; c0 < rs.size();) {
            // widest chunk within kTriRows rows and kTriBlockCap bytes
            int nr = 0, maxlen = 0;
            while (c0 + nr < rs.size() && nr < kTriRows) {
                const int ml = std::max(maxlen, static_cast<int>(rc[rs[c0 + nr]].size()));
                const int sp = std::max(2, (ml + 1) / 2 * 2);
                if (nr > 0 && 12 * (nr + 1) * sp + 20 * (nr + 1) + 64 > kTriBlockCap) break;
                maxlen = ml;
                ++nr;
            }
            const int span = std::max(2, (maxlen + 1) / 2 * 2);  // even: keeps vals 8-byte aligned
            const size_t base = p.cols.size();
            p.chunk_meta.push_back(static_cast<int>(p.rows.size()));
            p.chunk_meta.push_back(nr);
            p.chunk_meta.push_back(static_cast<int>(base));
            p.chunk_meta.push_back(span);
            p.cols.resize(base + static_cast<size_t>(span) * nr, n);  // dummy column n
            p.vals.resize(base + static_cast<size_t>(span) * nr, 0.0);
            for (int l = 0; l < nr; ++l) {
                const int i = rs[c0 + l];
                const int len = static_cast<int>(rc[i].size());
                p.rows.push_back(i);
                p.lens.push_back(len);
                p.max_row_len = std::max(p.max_row_len, len);
                for (int e = 0; e < len; ++e) {
                    p.cols[base + static_cast<size_t>(e) * nr + l] = rc[i][e];
                    p.vals[base + static_cast<size_t>(e) * nr + l] = rvv[i][e];
                }
            }
            c0 += nr;
        }
        p.level_chunk.push_back(static_cast<int>(p.chunk_meta.size() / 4));
    }
    p.n_chunks = static_cast<int>(p.chunk_meta.size() / 4);
    if (rv.diag) {
        p.diag.resize(n);
        for (int i = 0; i < n; ++i) p.diag[i] = rv.diag(i);
    }
    return p;
}

// triangular factor rows: every stored entry is summed and is a dependency;
// the upper factor's diagonal (first entry of each row) divides
SweepRows factor_rows(const HostCsr& m, bool upper) {
    SweepRows rv;
    const int skip = upper ? 1 : 0;
    rv.deps = [&m, skip](int i, std::vector<int>& d) {
        d.assign(m.col_indices.begin() + m.row_offsets[i] + skip, m.col_indices.begin() + m.row_offsets[i + 1]);
    };
    rv.entries = [&m, skip](int i, std::vector<int>& c, std::vector<double>& v) {
        c.assign(m.col_indices.begin() + m.row_offsets[i] + skip, m.col_indices.begin() + m.row_offsets[i + 1]);
        v.assign(m.values.begin() + m.row_offsets[i] + skip, m.values.begin() + m.row_offsets[i + 1]);
    };
    if (upper) rv.diag = [&m](int i) { return m.values[m.row_offsets[i]]; };
    return rv;
}

}  // namespace

TriPlan plan_lower(const HostCsr& lower) { return make_plan(lower.n_rows, false, factor_rows(lower, false)); }
TriPlan plan_upper(const HostCsr& upper) { return make_plan(upper.n_rows, true, factor_rows(upper, true)); }

TriPlan plan_gauss_seidel(const HostCsr& a, bool backward) {
    // gauss_seidel_sweep (solvers.hpp:80-99): row i sums every off-diagonal
    // entry in CSR order and divides by its diagonal; it must follow the rows
    // it reads updated (j < i forward, j > i backward).  For a symmetric
    // pattern these levels are the anti-diagonal wavefronts, and every row
    // that row i reads in its old state lies on a later level.
    SweepRows rv;
    rv.deps = [&a, backward](int i, std::vector<int>& d) {
        d.clear();
        for (int e = a.row_offsets[i]; e < a.row_offsets[i + 1]; ++e) {
            const int j = a.col_indices[e];
            if (backward ? j > i : j < i) d.push_back(j);
        }
    };
    rv.entries = [&a](int i, std::vector<int>& c, std::vector<double>& v) {
        c.clear();
        v.clear();
        for (int e = a.row_offsets[i]; e < a.row_offsets[i + 1]; ++e)
            if (a.col_indices[e] != i) {
                c.push_back(a.col_indices[e]);
                v.push_back(a.values[e]);
            }
    };
    rv.diag = [&a](int i) {
        for (int e = a.row_offsets[i]; e < a.row_offsets[i + 1]; ++e)
            if (a.col_indices[e] == i) return a.values[e];
        throw std::runtime_error("gauss_seidel_sweep: zero diagonal entry");
    };
    return make_plan(a.n_rows, backward, rv);
}

TriStream make_tri_stream(const TriPlan& p, bool fast) {
    const bool upper = !p.diag.empty();
    std::vector<int> block_of(p.n, -1);  // plan chunk (stream block) of every row
    for (int c = 0; c < p.n_chunks; ++c)
        for (int l = 0; l < p.chunk_meta[4 * c + 1]; ++l) block_of[p.rows[p.chunk_meta[4 * c] + l]] = c;
    // ---- block images
    std::vector<std::vector<unsigned char>> blocks;
    for (int c = 0; c < p.n_chunks; ++c) {
        if (fast) throw InvalidArgument("make_tri_stream: the reassociated mode uses block recurrences (BlkStream)");
        const int row0 = p.chunk_meta[4 * c], nr = p.chunk_meta[4 * c + 1], base = p.chunk_meta[4 * c + 2];
        const int span = p.chunk_meta[4 * c + 3];
        int lg = 0, m = span;
        // fast: entry-major over a full warp (slot q of lane L at q * 32 + L),
        // so that one load instruction reads one slot of every lane
        // conflict-free; exact: entry e of row l at e * nr + l
        const int lanes = fast ? 32 : nr;
        const int per = fast ? m : span;  // entries per lane (fast) / per row (exact)
        // exact: rows int32[nr] at 32, diag + rdiag double[nr] each at diag_off;
        // fast: per-lane tables at 32: row index of the row's first lane
        // (-1 elsewhere) int32[32], and at diag_off its reciprocal diagonal
        // double[32]
        const int rows_n = fast ? 32 : nr;
        const int diag_off = 32 + (4 * rows_n + 7) / 8 * 8;
        const int cols_off = diag_off + (upper ? (fast ? 8 * 32 : 16 * nr) : 0);
        const int vals_off = (cols_off + 4 * lanes * per + 15) / 16 * 16;
        const int bytes = (vals_off + 8 * lanes * per + 15) / 16 * 16;
        if (bytes + 16 > kTriUnitCap || (!fast && nr * span > kTriMaxItems))
            throw InvalidArgument("ILUT factor level slice exceeds the triangular-solve block capacity");
        std::vector<unsigned char> img(bytes, 0);
        const int hdr[8] = {nr, per, lg, bytes, cols_off, vals_off, diag_off, 0};
        std::memcpy(img.data(), hdr, sizeof hdr);
        int* rws = reinterpret_cast<int*>(img.data() + 32);
        double* dg = reinterpret_cast<double*>(img.data() + diag_off);
        if (fast) {
            for (int L = 0; L < 32; ++L) rws[L] = -1;
            for (int l = 0; l < nr; ++l) {
                const int i = p.rows[row0 + l];
                rws[l << lg] = i;
                if (upper) dg[l << lg] = 1.0 / p.diag[i];  // IEEE round-to-nearest reciprocal
            }
        } else {
            for (int l = 0; l < nr; ++l) rws[l] = p.rows[row0 + l];
            if (upper)
                for (int l = 0; l < nr; ++l) {
                    const double d = p.diag[p.rows[row0 + l]];
                    dg[l] = d;
                    dg[nr + l] = 1.0 / d;  // IEEE round-to-nearest reciprocal
                }
        }
        int* cols = reinterpret_cast<int*>(img.data() + cols_off);
        double* vals = reinterpret_cast<double*>(img.data() + vals_off);
        for (int l = 0; l < nr; ++l) {
            for (int e = 0; e < span; ++e) {  // plan entry e of row l (dummies past its length)
                const size_t src = static_cast<size_t>(base) + static_cast<size_t>(e) * nr + l;
                size_t dst;
                if (fast) {
                    const int k = e / m, q = e % m;
                    if (k >= (1 << lg)) continue;  // beyond the lanes: only dummies live there
                    dst = static_cast<size_t>(q) * 32 + (l << lg) + k;
                } else {
                    dst = static_cast<size_t>(e) * nr + l;
                }
                cols[dst] = p.cols[src];
                vals[dst] = p.vals[src];
            }
            if (fast)  // slots past the row's padded span
                for (int e = span; e < (m << lg); ++e) {
                    const size_t dst = static_cast<size_t>(e % m) * 32 + (l << lg) + e / m;
                    cols[dst] = p.n;
                    vals[dst] = 0.0;
                }
        }
        blocks.push_back(std::move(img));
    }
    // ---- units: header (16 B: n_blocks, next_off16, next_bytes, pad) + a
    // table of uint16 block offsets from the unit start (padded to 16 B),
    // then the blocks
    auto hdr_bytes = [](size_t nb) { return 16 + (2 * nb + 15) / 16 * 16; };
    TriStream ts;
    ts.n_blocks = static_cast<int>(blocks.size());
    std::vector<std::pair<size_t, size_t>> units;  // [first block, end block)
    {
        size_t b = 0;
        while (b < blocks.size()) {
            size_t e = b, bytes = 0;
            while (e < blocks.size() &&
                   (e == b || hdr_bytes(e + 1 - b) + bytes + blocks[e].size() <= static_cast<size_t>(kTriUnitCap)))
                bytes += blocks[e++].size();  // a block larger than the cap forms a unit of its own
            units.emplace_back(b, e);
            b = e;
        }
    }
    ts.n_units = static_cast<int>(units.size());
    std::vector<size_t> uoff, ubytes;
    size_t total = 0;
    for (const auto& u : units) {
        size_t bytes = hdr_bytes(u.second - u.first);
        for (size_t k = u.first; k < u.second; ++k) bytes += blocks[k].size();
        uoff.push_back(total);
        ubytes.push_back(bytes);
        total += bytes;
        ts.max_unit_bytes = std::max(ts.max_unit_bytes, static_cast<int>(bytes));
    }
    ts.stream.assign(total + 16, 0);
    ts.prime.assign(2 * (kTriSlots - 1), 0);
    for (int k = 0; k < kTriSlots - 1 && k < ts.n_units; ++k) {
        ts.prime[2 * k] = static_cast<int>(uoff[k] / 16);
        ts.prime[2 * k + 1] = static_cast<int>(ubytes[k]);
    }
    for (size_t u = 0; u < units.size(); ++u) {
        unsigned char* dst = ts.stream.data() + uoff[u];
        const size_t nb = units[u].second - units[u].first;
        int hdr[4] = {static_cast<int>(nb), 0, 0, 0};
        const size_t nxt = u + kTriSlots - 1;
        if (nxt < units.size()) {
            hdr[1] = static_cast<int>(uoff[nxt] / 16);
            hdr[2] = static_cast<int>(ubytes[nxt]);
        }
        std::memcpy(dst, hdr, sizeof hdr);
        auto* tab = reinterpret_cast<unsigned short*>(dst + 16);
        size_t o = hdr_bytes(nb);
        for (size_t k = units[u].first; k < units[u].second; ++k) {
            tab[k - units[u].first] = static_cast<unsigned short>(o);
            std::memcpy(dst + o, blocks[k].data(), blocks[k].size());
            ts.block_info.insert(ts.block_info.end(),
                                 {static_cast<int>(u), static_cast<int>(o), k == units[u].first ? 1 : 0, 0});
            o += blocks[k].size();
        }
    }
    return ts;
}


// ---------------------------------------------------------------------------
// Block-recurrence sweeps (setup_host.hpp BlkStream)
// ---------------------------------------------------------------------------
namespace {

struct BlkRowsView {
    int n = 0;
    bool descending = false;
    // off-diagonal entries of row i and its diagonal (1 for a unit factor)
    std::function<void(int, std::vector<int>&, std::vector<double>&)> entries;
    std::function<double(int)> diag;
};

BlkStream make_blk_stream(const BlkRowsView& rv, int win) {
    const int n = rv.n;
    BlkStream bs;
    bs.n = n;
    bs.win = win;
    bs.desc = rv.descending ? 1 : 0;
    // column as stored: absolute, or its window slot (padding: n, or the zero slot)
    auto stored = [&](int c) { return win ? (c & (win - 1)) : c; };
    const int pad = win ? win : n;
    bs.n_blocks = (n + kBlkRows - 1) / kBlkRows;
    auto pos_of = [&](int i) { return rv.descending ? n - 1 - i : i; };
    auto row_at = [&](int pos) { return rv.descending ? n - 1 - pos : pos; };
    std::vector<int> cols;
    std::vector<double> vals;
    struct Blk {
        long double B[kBlkRows][kBlkRows];
        std::vector<std::pair<int, double>> olde[kBlkRows], frsh[kBlkRows];
        int rows[kBlkRows];
        size_t maxold = 0, mf = 0;
    };
    std::vector<Blk> blks(bs.n_blocks);
    size_t maxold_all = 0;
    for (int k = 0; k < bs.n_blocks; ++k) {
        Blk& b = blks[k];
        for (auto& r : b.B)
            for (auto& v : r) v = 0.0L;
        for (int l = 0; l < kBlkRows; ++l) {
            const int pos = k * kBlkRows + l;
            if (pos >= n) {
                b.rows[l] = -1;
                b.B[l][l] = 1.0L;
                continue;
            }
            const int i = row_at(pos);
            b.rows[l] = i;
            b.B[l][l] = rv.diag(i);
            rv.entries(i, cols, vals);
            for (size_t e = 0; e < cols.size(); ++e) {
                const int pj = pos_of(cols[e]), kj = pj / kBlkRows;
                if (pj < pos && kj == k) {
                    b.B[l][pj - k * kBlkRows] += vals[e];
                } else if (pj < pos && kj >= k - kBlkFresh) {
                    b.frsh[l].emplace_back(cols[e], vals[e]);
                } else {
                    b.olde[l].emplace_back(cols[e], vals[e]);
                    if (pj > pos) bs.lookahead = std::max(bs.lookahead, kj - k);
                }
            }
            b.maxold = std::max(b.maxold, b.olde[l].size());
            // fresh columns lie in block k-1 (kBlkFresh = 1): the folded
            // coupling reaches back to local column 32 - nf of that block
            for (const auto& fe : b.frsh[l]) {
                const int jl = pos_of(fe.first) - (k - 1) * kBlkRows;
                if (jl < 0 || jl >= kBlkRows) throw std::logic_error("make_blk_stream: fresh column outside block k-1");
                b.mf = std::max<size_t>(b.mf, static_cast<size_t>(kBlkRows - jl));
            }
        }
        b.mf = (b.mf + 7) / 8;  // groups of four column pairs of the folded coupling G_k
        maxold_all = std::max(maxold_all, b.maxold);
    }
    // worker parts: about four old slots per part and lane
    bs.parts = static_cast<int>(std::min<size_t>(kBlkMaxParts, std::max<size_t>(1, (maxold_all + 3) / 4)));
    const int P = bs.parts;
    bs.mf0 = bs.n_blocks ? static_cast<int>(blks[0].mf) : 0;
    std::vector<std::vector<unsigned char>> units(bs.n_blocks);
    for (int k = 0; k < bs.n_blocks; ++k) {
        Blk& b = blks[k];
        const size_t mo = (b.maxold + P - 1) / P;
        const size_t mf = b.mf;
        // dense inverse of the lower-triangular block, column by column
        static long double inv[kBlkRows][kBlkRows];
        for (auto& r : inv)
            for (auto& v : r) v = 0.0L;
        for (int j = 0; j < kBlkRows; ++j)
            for (int l = j; l < kBlkRows; ++l) {
                long double acc = l == j ? 1.0L : 0.0L;
                for (int m = j; m < l; ++m) acc -= b.B[l][m] * inv[m][j];
                inv[l][j] = acc / b.B[l][l];
            }
        const size_t part_bytes = (win ? 320 : 384) * mo;
        const size_t bytes = kBlkFreshOff + 2048 * mf + static_cast<size_t>(P) * part_bytes;
        std::vector<unsigned char> img(bytes, 0);
        const int hdr[4] = {static_cast<int>(mo), 0, static_cast<int>(bytes), static_cast<int>(mf)};
        std::memcpy(img.data(), hdr, sizeof hdr);
        std::memcpy(img.data() + 16, b.rows, sizeof b.rows);
        double* iv = reinterpret_cast<double*>(img.data() + kBlkInvOff);
        for (int pj = 0; pj < kBlkRows / 2; ++pj)
            for (int l = kBlkTri ? 2 * pj : 0; l < kBlkRows; ++l) {
                const int slot = kBlkTri ? pj * (31 - pj) + l : pj * kBlkRows + l;
                iv[slot * 2] = static_cast<double>(inv[l][2 * pj]);
                iv[slot * 2 + 1] = static_cast<double>(inv[l][2 * pj + 1]);
            }
        // folded coupling to block k-1: G = B^{-1} N, N(l, j) = the fresh
        // entry of row l at local column j of block k-1; pair q holds the
        // columns (30 - 2q, 31 - 2q), so the chain walks back from the last
        // solved value and stops after mf pairs
        if (mf) {
            static long double nn[kBlkRows][kBlkRows], gg[kBlkRows][kBlkRows];
            for (auto& r : nn)
                for (auto& v : r) v = 0.0L;
            for (int l = 0; l < kBlkRows; ++l)
                for (const auto& fe : b.frsh[l]) nn[l][pos_of(fe.first) - (k - 1) * kBlkRows] += fe.second;
            for (int l = 0; l < kBlkRows; ++l)
                for (int j = 0; j < kBlkRows; ++j) {
                    long double acc = 0.0L;
                    for (int m = 0; m <= l; ++m) acc += inv[l][m] * nn[m][j];
                    gg[l][j] = acc;
                }
            double* gv = reinterpret_cast<double*>(img.data() + kBlkFreshOff);
            for (size_t q = 0; q < 4 * mf; ++q)
                for (int l = 0; l < kBlkRows; ++l) {
                    gv[(q * kBlkRows + l) * 2] = static_cast<double>(gg[l][30 - 2 * q]);
                    gv[(q * kBlkRows + l) * 2 + 1] = static_cast<double>(gg[l][31 - 2 * q]);
                }
        }
        for (int p = 0; p < P; ++p) {
            unsigned char* pb = img.data() + kBlkFreshOff + 2048 * mf + static_cast<size_t>(p) * part_bytes;
            const size_t cb = (win ? 2 : 4) * kBlkRows * mo;  // column bytes of the part
            double* ov = reinterpret_cast<double*>(pb + cb);
            auto put_col = [&](size_t slot, int c) {
                if (win) {
                    const unsigned short c16 = static_cast<unsigned short>(c);
                    std::memcpy(pb + 2 * slot, &c16, 2);
                } else {
                    std::memcpy(pb + 4 * slot, &c, 4);
                }
            };
            for (size_t s2 = 0; s2 < kBlkRows * mo; ++s2) put_col(s2, pad);  // neutral padding (zero slot)
            for (int l = 0; l < kBlkRows; ++l)
                for (size_t e = p, q = 0; e < b.olde[l].size(); e += P, ++q) {
                    put_col(q * kBlkRows + l, stored(b.olde[l][e].first));
                    ov[q * kBlkRows + l] = b.olde[l][e].second;
                }
        }
        units[k] = std::move(img);
    }
    size_t total = 0;
    for (int k = 0; k < bs.n_blocks; ++k) {
        const auto& u = units[k];
        bs.table.push_back(static_cast<int>(total / 16));
        bs.table.push_back(static_cast<int>(u.size()));
        bs.table.push_back(static_cast<int>(blks[k].mf));
        bs.table.push_back(0);
        bs.max_unit_bytes = std::max(bs.max_unit_bytes, static_cast<int>(u.size()));
        total += u.size();
    }
    bs.stream.reserve(total);
    for (const auto& u : units) bs.stream.insert(bs.stream.end(), u.begin(), u.end());
    return bs;
}

}  // namespace

int ilut_span(const HostCsr& lower, const HostCsr& upper) {
    int span = 0;
    for (const HostCsr* f : {&lower, &upper})
        for (int i = 0; i < f->n_rows; ++i)
            for (int e = f->row_offsets[i]; e < f->row_offsets[i + 1]; ++e)
                span = std::max(span, std::abs(i - f->col_indices[e]));
    return span;
}

int blk_window_for(int span) {
    int w = 64;
    while (w < span + 64) w *= 2;
    return w <= kBlkMaxWin ? w : 0;
}

BlkStream blk_lower(const HostCsr& m, int win) {
    BlkRowsView rv;
    rv.n = m.n_rows;
    rv.entries = [&m](int i, std::vector<int>& c, std::vector<double>& v) {
        c.assign(m.col_indices.begin() + m.row_offsets[i], m.col_indices.begin() + m.row_offsets[i + 1]);
        v.assign(m.values.begin() + m.row_offsets[i], m.values.begin() + m.row_offsets[i + 1]);
    };
    rv.diag = [](int) { return 1.0; };
    return make_blk_stream(rv, win);
}

BlkStream blk_upper(const HostCsr& m, int win) {
    BlkRowsView rv;
    rv.n = m.n_rows;
    rv.descending = true;
    rv.entries = [&m](int i, std::vector<int>& c, std::vector<double>& v) {
        c.assign(m.col_indices.begin() + m.row_offsets[i] + 1, m.col_indices.begin() + m.row_offsets[i + 1]);
        v.assign(m.values.begin() + m.row_offsets[i] + 1, m.values.begin() + m.row_offsets[i + 1]);
    };
    rv.diag = [&m](int i) { return m.values[m.row_offsets[i]]; };
    return make_blk_stream(rv, win);
}

BlkStream blk_gauss_seidel(const HostCsr& a, bool backward) {
    BlkRowsView rv;
    rv.n = a.n_rows;
    rv.descending = backward;
    rv.entries = [&a](int i, std::vector<int>& c, std::vector<double>& v) {
        c.clear();
        v.clear();
        for (int e = a.row_offsets[i]; e < a.row_offsets[i + 1]; ++e)
            if (a.col_indices[e] != i) {
                c.push_back(a.col_indices[e]);
                v.push_back(a.values[e]);
            }
    };
    rv.diag = [&a](int i) {
        for (int e = a.row_offsets[i]; e < a.row_offsets[i + 1]; ++e)
            if (a.col_indices[e] == i) return a.values[e];
        throw std::runtime_error("gauss_seidel_sweep: zero diagonal entry");
    };
    return make_blk_stream(rv, 0);
}

}  // namespace phi
