// Host-side check of the block-recurrence sweep schedules (setup_host.hpp
// BlkStream): the stream images are decoded and executed block by block on the
// CPU, in the order the device runs them (old sums, dense block
// inverse), and compared with the plain sequential sweeps of the reference
// (ilut.hpp:146-163 substitutions, solvers.hpp:80-99 Gauss-Seidel).
// Test infrastructure only (tests/test_blk_schedule.py builds and runs it).
#include <cmath>
#include <cstdio>
#include <cstring>
#include <algorithm>
#include <random>
#include <vector>

#include "setup_host.hpp"

using namespace phi;

// 2D tensor stencil of half-width w on an m x m grid (the IgA pattern),
// diagonally weighted so ILUT and Gauss-Seidel are well defined.
static HostCsr stencil_matrix(int m, int w, unsigned seed) {
    std::mt19937 g(seed);
    std::uniform_real_distribution<double> u(-1.0, 1.0);
    HostCsr a;
    a.n_rows = a.n_cols = m * m;  // row_offsets starts as {0}
    for (int iv = 0; iv < m; ++iv)
        for (int iu = 0; iu < m; ++iu) {
            for (int dv = -w; dv <= w; ++dv)
                for (int du = -w; du <= w; ++du) {
                    const int jv = iv + dv, ju = iu + du;
                    if (jv < 0 || jv >= m || ju < 0 || ju >= m) continue;
                    a.col_indices.push_back(jv * m + ju);
                    a.values.push_back(dv == 0 && du == 0 ? 4.0 * (2 * w + 1) * (2 * w + 1) : u(g));
                }
            a.row_offsets.push_back(static_cast<int>(a.col_indices.size()));
        }
    return a;
}

// Execute a BlkStream sweep on x (rhs: separate vector, or x itself), block
// by block in the device's order: old sums (per worker part), dense block
// inverse, folded coupling to the previous block.
// Rolling-window streams (bs.win > 0) read every column from a window of
// win slots (initialised to NaN, so a read of a slot not yet solved in this
// sweep poisons the result) plus the zero slot, with 16-bit old columns.
static void run_blk(const BlkStream& bs, std::vector<double>& x, const std::vector<double>& rhs) {
    const int n = bs.n, P = bs.parts, W = bs.win;
    x.resize(n + 1);
    x[n] = 0.0;
    std::vector<double> wv(W ? W + 1 : 0, std::nan(""));
    if (W) wv[W] = 0.0;
    double* xr = W ? wv.data() : x.data();  // what the column indices address
    const size_t cbytes = W ? 2 : 4;
    double zprev[32] = {0.0};  // the previous block's values in solve order
    for (int k = 0; k < bs.n_blocks; ++k) {
        const unsigned char* u = bs.stream.data() + static_cast<size_t>(bs.table[4 * k]) * 16;
        int hdr[4];
        std::memcpy(hdr, u, sizeof hdr);
        const int mo = hdr[0], mf = hdr[3];
        if (hdr[2] != bs.table[4 * k + 1] || hdr[3] != bs.table[4 * k + 2]) throw std::runtime_error("unit size mismatch");
        const int* rows = reinterpret_cast<const int*>(u + 16);
        const double* iv = reinterpret_cast<const double*>(u + kBlkInvOff);
        const unsigned char* fr = u + kBlkFreshOff;
        double t[32], z[32];
        for (int l = 0; l < 32; ++l) {
            double s = 0.0;
            for (int p = 0; p < P; ++p) {  // worker parts
                const unsigned char* pb = u + kBlkFreshOff + 2048 * mf + p * (32 * cbytes + 256) * mo;
                const double* ov = reinterpret_cast<const double*>(pb + 32 * cbytes * mo);
                for (int q = 0; q < mo; ++q) {
                    int c = 0;
                    if (W) {
                        unsigned short c16;
                        std::memcpy(&c16, pb + 2 * (q * 32 + l), 2);
                        c = c16;
                    } else {
                        std::memcpy(&c, pb + 4 * (q * 32 + l), 4);
                    }
                    s += ov[q * 32 + l] * xr[c];
                }
            }
            t[l] = (rows[l] >= 0 ? rhs[rows[l]] : 0.0) - s;
        }
        const double* gv = reinterpret_cast<const double*>(fr);
        for (int l = 0; l < 32; ++l) {
            z[l] = 0.0;
            // the inverse: full double[16][32][2], or (kBlkTri) its lower triangle -- column pair
            // p keeps the lanes l >= 2 p at slot p (31 - p) + l, the rest are exact zeros
            for (int j = 0; j < 32; ++j) {
                const int pj = j / 2;
                double v = 0.0;
                if (!kBlkTri)
                    v = iv[(pj * 32 + l) * 2 + (j & 1)];
                else if (l >= 2 * pj)
                    v = iv[(pj * (31 - pj) + l) * 2 + (j & 1)];
                z[l] += v * t[j];
            }
            // folded coupling: minus G_k times the last 8 mf values of block k-1
            for (int q = 0; q < 4 * mf; ++q)
                z[l] -= gv[(q * 32 + l) * 2] * zprev[30 - 2 * q] + gv[(q * 32 + l) * 2 + 1] * zprev[31 - 2 * q];
        }
        for (int l = 0; l < 32; ++l) {
            zprev[l] = z[l];
            if (rows[l] >= 0) {
                x[rows[l]] = z[l];
                if (W) wv[rows[l] & (W - 1)] = z[l];
            }
        }
    }
    x.resize(n);
}

// Exact banded LU without pivoting (the matrices are diagonally dominant):
// unit lower L (strict part stored) and U with its diagonal first, the layout
// of the reference's ILUT factors (ilut.hpp:17-22).  The block schedules only
// need triangular factors of the IgA band shape, not ILUT's particular fill.
static void band_lu(const HostCsr& a, int m, int w, HostCsr& L, HostCsr& U) {
    const int n = a.n_rows, b = w * (m + 1);
    const int wd = 2 * b + 1;
    std::vector<double> band((size_t)n * wd, 0.0);  // (i, j) at i * wd + (j - i + b)
    for (int i = 0; i < n; ++i)
        for (int e = a.row_offsets[i]; e < a.row_offsets[i + 1]; ++e)
            band[(size_t)i * wd + (a.col_indices[e] - i + b)] = a.values[e];
    auto at = [&](int i, int j) -> double& { return band[(size_t)i * wd + (j - i + b)]; };
    for (int k = 0; k < n; ++k)
        for (int i = k + 1; i <= std::min(n - 1, k + b); ++i) {
            const double l = at(i, k) / at(k, k);
            at(i, k) = l;
            for (int j = k + 1; j <= std::min(n - 1, k + b); ++j) at(i, j) -= l * at(k, j);
        }
    L = HostCsr{};
    U = HostCsr{};
    L.n_rows = L.n_cols = U.n_rows = U.n_cols = n;
    for (int i = 0; i < n; ++i) {
        for (int j = std::max(0, i - b); j < i; ++j)
            if (at(i, j) != 0.0) {
                L.col_indices.push_back(j);
                L.values.push_back(at(i, j));
            }
        L.row_offsets.push_back(L.nnz());
        U.col_indices.push_back(i);
        U.values.push_back(at(i, i));
        for (int j = i + 1; j <= std::min(n - 1, i + b); ++j)
            if (at(i, j) != 0.0) {
                U.col_indices.push_back(j);
                U.values.push_back(at(i, j));
            }
        U.row_offsets.push_back(U.nnz());
    }
}

static double rel(const std::vector<double>& a, const std::vector<double>& b) {
    double num = 0.0, den = 0.0;
    for (size_t i = 0; i < a.size(); ++i) {
        num += (a[i] - b[i]) * (a[i] - b[i]);
        den += b[i] * b[i];
    }
    return std::sqrt(num / den);
}

int main(int argc, char** argv) {
    const int m = argc > 1 ? std::atoi(argv[1]) : 40, w = argc > 2 ? std::atoi(argv[2]) : 3;
        const HostCsr a = stencil_matrix(m, w, 7);
    const int n = a.n_rows;
    HostCsr L, U;
    band_lu(a, m, w, L, U);
    std::mt19937 g(3);
    std::normal_distribution<double> nd;
    std::vector<double> r(n);
    for (auto& v : r) v = nd(g);
    // reference: forward then backward substitution (ilut.hpp:150-162)
    std::vector<double> z = r;
    for (int i = 0; i < n; ++i)
        for (int e = L.row_offsets[i]; e < L.row_offsets[i + 1]; ++e) z[i] -= L.values[e] * z[L.col_indices[e]];
    for (int i = n - 1; i >= 0; --i) {
        double s = z[i];
        for (int e = U.row_offsets[i] + 1; e < U.row_offsets[i + 1]; ++e) s -= U.values[e] * z[U.col_indices[e]];
        z[i] = s / U.values[U.row_offsets[i]];
    }
    std::vector<double> y = r;
    run_blk(blk_lower(L), y, r);
    const std::vector<double> y1 = y;
    run_blk(blk_upper(U), y, y1);
    const double e_ilut = rel(y, z);
    // the same substitutions from rolling-window streams
    const int wz = blk_window_for(ilut_span(L, U));
    double e_win = 0.0;
    if (wz) {
        std::vector<double> yw = r;
        run_blk(blk_lower(L, wz), yw, r);
        const std::vector<double> yw1 = yw;
        run_blk(blk_upper(U, wz), yw, yw1);
        e_win = rel(yw, z);
    }
    // Gauss-Seidel forward and backward (solvers.hpp:80-99)
    double e_gs[2];
    for (int dir = 0; dir < 2; ++dir) {
        std::vector<double> x0(n), xr, xb;
        for (auto& v : x0) v = nd(g);
        xr = x0;
        for (int s = 0; s < n; ++s) {
            const int i = dir ? n - 1 - s : s;
            double acc = r[i], d = 0.0;
            for (int e = a.row_offsets[i]; e < a.row_offsets[i + 1]; ++e) {
                if (a.col_indices[e] == i)
                    d = a.values[e];
                else
                    acc -= a.values[e] * xr[a.col_indices[e]];
            }
            xr[i] = acc / d;
        }
        xb = x0;
        run_blk(blk_gauss_seidel(a, dir == 1), xb, r);
        e_gs[dir] = rel(xb, xr);
    }
    std::printf("n %d ilut %.3e window %d: %.3e gs_fwd %.3e gs_bwd %.3e\n", n, e_ilut, wz, e_win, e_gs[0], e_gs[1]);
    return (e_ilut < 1e-12 && e_win < 1e-12 && e_gs[0] < 1e-12 && e_gs[1] < 1e-12) ? 0 : 1;
}
