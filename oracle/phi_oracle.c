/*
 * TEST INFRASTRUCTURE ONLY -- CPU restatement of the reference hot path, used
 * by tests/ and bench.py's cpu_baseline leg as the parity checker; never part
 * of the product.  See phi_oracle.h for scope.  Every function cites the
 * reference file:line (relative to /root/reference/proj/include/miga) whose
 * algorithm it restates.  Compile with -ffp-contract=off.
 */
#include "phi_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static char g_err[512];
const char* oc_last_error(void) { return g_err; }
static int set_err(const char* msg) {
    snprintf(g_err, sizeof g_err, "%s", msg);
    return 1;
}

/* ------------------------------------------------------------------------ */
/* owned CSR                                                                 */
/* ------------------------------------------------------------------------ */
typedef struct {
    int n_rows, n_cols, nnz, cap;
    int* ro;
    int* ci;
    double* v;
} mat;

static void mat_init(mat* a, int n_rows, int n_cols, int cap) {
    a->n_rows = n_rows;
    a->n_cols = n_cols;
    a->nnz = 0;
    a->cap = cap > 0 ? cap : 1;
    a->ro = (int*)calloc((size_t)n_rows + 1, sizeof(int));
    a->ci = (int*)malloc(sizeof(int) * (size_t)a->cap);
    a->v = (double*)malloc(sizeof(double) * (size_t)a->cap);
}
static void mat_push(mat* a, int j, double v) {
    if (a->nnz == a->cap) {
        a->cap *= 2;
        a->ci = (int*)realloc(a->ci, sizeof(int) * (size_t)a->cap);
        a->v = (double*)realloc(a->v, sizeof(double) * (size_t)a->cap);
    }
    a->ci[a->nnz] = j;
    a->v[a->nnz] = v;
    a->nnz++;
}
static void mat_free(mat* a) {
    free(a->ro);
    free(a->ci);
    free(a->v);
    memset(a, 0, sizeof *a);
}
static oc_csr view(const mat* a) {
    oc_csr c = {a->n_rows, a->n_cols, a->ro, a->ci, a->v};
    return c;
}
static int export_mat(const mat* a, int* n_rows, int* n_cols, int* nnz, int* ro, int* ci, double* v) {
    if (n_rows) *n_rows = a->n_rows;
    if (n_cols) *n_cols = a->n_cols;
    if (nnz) *nnz = a->nnz;
    if (ro) memcpy(ro, a->ro, sizeof(int) * ((size_t)a->n_rows + 1));
    if (ci) memcpy(ci, a->ci, sizeof(int) * (size_t)a->nnz);
    if (v) memcpy(v, a->v, sizeof(double) * (size_t)a->nnz);
    return 0;
}

/* ------------------------------------------------------------------------ */
/* sparse.hpp kernels                                                        */
/* ------------------------------------------------------------------------ */

/* sparse.hpp:114-124 -- fixed per-row summation order */
int oc_spmv(const oc_csr* a, const double* x, double* y) {
    for (int i = 0; i < a->n_rows; ++i) {
        double s = 0.0;
        for (int e = a->row_offsets[i]; e < a->row_offsets[i + 1]; ++e)
            s += a->values[e] * x[a->col_indices[e]];
        y[i] = s;
    }
    return 0;
}

/* sparse.hpp:133-143 -- scatter in row order, zero x skipped */
int oc_spmv_transpose(const oc_csr* a, const double* x, double* y) {
    for (int j = 0; j < a->n_cols; ++j) y[j] = 0.0;
    for (int i = 0; i < a->n_rows; ++i) {
        const double xi = x[i];
        if (xi == 0.0) continue;
        for (int e = a->row_offsets[i]; e < a->row_offsets[i + 1]; ++e)
            y[a->col_indices[e]] += a->values[e] * xi;
    }
    return 0;
}

/* sparse.hpp:188-194 -- index-ordered dot / norm */
static double dot(const double* x, const double* y, int n) {
    double s = 0.0;
    for (int i = 0; i < n; ++i) s += x[i] * y[i];
    return s;
}
double oc_norm2(const double* x, int n) { return sqrt(dot(x, x, n)); }

/* sparse.hpp:196-198 with alpha = 1 (the only use on the path) */
static void axpy1(const double* x, double* y, int n) {
    for (int i = 0; i < n; ++i) y[i] += 1.0 * x[i];
}

/* sparse.hpp:148-178 -- C = alpha A + beta B, union pattern */
static void sparse_add(double alpha, const oc_csr* a, double beta, const oc_csr* b, mat* c) {
    mat_init(c, a->n_rows, a->n_cols, a->row_offsets[a->n_rows] + 16);
    for (int i = 0; i < a->n_rows; ++i) {
        int pa = a->row_offsets[i], ea = a->row_offsets[i + 1];
        int pb = b->row_offsets[i], eb = b->row_offsets[i + 1];
        while (pa < ea || pb < eb) {
            const int ja = pa < ea ? a->col_indices[pa] : c->n_cols;
            const int jb = pb < eb ? b->col_indices[pb] : c->n_cols;
            if (ja == jb) {
                mat_push(c, ja, alpha * a->values[pa++] + beta * b->values[pb++]);
            } else if (ja < jb) {
                mat_push(c, ja, alpha * a->values[pa++]);
            } else {
                mat_push(c, jb, beta * b->values[pb++]);
            }
        }
        c->ro[i + 1] = c->nnz;
    }
}

/* ------------------------------------------------------------------------ */
/* solvers.hpp                                                               */
/* ------------------------------------------------------------------------ */

/* solvers.hpp:80-99 */
int oc_gs_sweep(const oc_csr* a, const double* b, double* x, int backward) {
    const int n = a->n_rows;
    const int begin = backward ? n - 1 : 0;
    const int step = backward ? -1 : 1;
    for (int i = begin; i >= 0 && i < n; i += step) {
        double diag = 0.0, s = b[i];
        for (int e = a->row_offsets[i]; e < a->row_offsets[i + 1]; ++e) {
            const int j = a->col_indices[e];
            if (j == i)
                diag = a->values[e];
            else
                s -= a->values[e] * x[j];
        }
        if (diag == 0.0) return set_err("gauss_seidel_sweep: zero diagonal entry");
        x[i] = s / diag;
    }
    return 0;
}

/* solvers.hpp:102-172 -- dense LU with partial pivoting */
typedef struct {
    int n;
    double* lu;
    int* piv;
} dense_lu;

static int dense_lu_factor(dense_lu* f, const oc_csr* a) {
    const int n = a->n_rows;
    f->n = n;
    f->lu = (double*)calloc((size_t)n * n, sizeof(double));
    f->piv = (int*)malloc(sizeof(int) * (size_t)n);
    double* lu = f->lu;
    for (int i = 0; i < n; ++i)
        for (int e = a->row_offsets[i]; e < a->row_offsets[i + 1]; ++e)
            lu[(size_t)i * n + a->col_indices[e]] = a->values[e];
    for (int i = 0; i < n; ++i) f->piv[i] = i;
    for (int k = 0; k < n; ++k) {
        int pivot = k;
        double best = fabs(lu[(size_t)k * n + k]);
        for (int i = k + 1; i < n; ++i) {
            const double v = fabs(lu[(size_t)i * n + k]);
            if (v > best) {
                best = v;
                pivot = i;
            }
        }
        if (best == 0.0) return set_err("DenseLU: singular matrix");
        if (pivot != k) {
            for (int j = 0; j < n; ++j) {
                const double t = lu[(size_t)k * n + j];
                lu[(size_t)k * n + j] = lu[(size_t)pivot * n + j];
                lu[(size_t)pivot * n + j] = t;
            }
            const int t = f->piv[k];
            f->piv[k] = f->piv[pivot];
            f->piv[pivot] = t;
        }
        const double d = lu[(size_t)k * n + k];
        for (int i = k + 1; i < n; ++i) {
            const double m = lu[(size_t)i * n + k] / d;
            lu[(size_t)i * n + k] = m;
            if (m == 0.0) continue;
            for (int j = k + 1; j < n; ++j) lu[(size_t)i * n + j] -= m * lu[(size_t)k * n + j];
        }
    }
    return 0;
}

/* solvers.hpp:118-133 */
static void dense_lu_solve(const dense_lu* f, const double* b, double* x) {
    const int n = f->n;
    const double* lu = f->lu;
    for (int i = 0; i < n; ++i) x[i] = b[f->piv[i]];
    for (int i = 0; i < n; ++i) {
        double s = x[i];
        for (int j = 0; j < i; ++j) s -= lu[(size_t)i * n + j] * x[j];
        x[i] = s;
    }
    for (int i = n - 1; i >= 0; --i) {
        double s = x[i];
        for (int j = i + 1; j < n; ++j) s -= lu[(size_t)i * n + j] * x[j];
        x[i] = s / lu[(size_t)i * n + i];
    }
}

/* ------------------------------------------------------------------------ */
/* ilut.hpp                                                                  */
/* ------------------------------------------------------------------------ */
typedef struct {
    int col;
    double val;
} entry;

static int cmp_keep(const void* pa, const void* pb) {
    /* ilut.hpp:124-129: larger |value| first, ties by smaller column */
    const entry* x = (const entry*)pa;
    const entry* y = (const entry*)pb;
    const double ax = fabs(x->val), ay = fabs(y->val);
    if (ax != ay) return ax > ay ? -1 : 1;
    return x->col < y->col ? -1 : (x->col > y->col);
}
static int cmp_col(const void* pa, const void* pb) {
    const entry* x = (const entry*)pa;
    const entry* y = (const entry*)pb;
    return x->col < y->col ? -1 : (x->col > y->col);
}
/* ilut.hpp:112-124 keep_largest: the fill_limit largest under a strict total
 * order (so the kept set is unique), then column order. */
static void keep_largest(entry* part, int* count, int fill_limit) {
    if (*count > fill_limit) {
        qsort(part, (size_t)*count, sizeof(entry), cmp_keep);
        *count = fill_limit;
    }
    qsort(part, (size_t)*count, sizeof(entry), cmp_col);
}

/* binary min-heap of column indices (the std::priority_queue of ilut.hpp:48) */
typedef struct {
    int* a;
    int n, cap;
} heap;
static void heap_push(heap* h, int v) {
    if (h->n == h->cap) {
        h->cap = h->cap ? 2 * h->cap : 64;
        h->a = (int*)realloc(h->a, sizeof(int) * (size_t)h->cap);
    }
    int i = h->n++;
    h->a[i] = v;
    while (i > 0) {
        const int p = (i - 1) / 2;
        if (h->a[p] <= h->a[i]) break;
        const int t = h->a[p];
        h->a[p] = h->a[i];
        h->a[i] = t;
        i = p;
    }
}
static int heap_pop(heap* h) {
    const int top = h->a[0];
    h->a[0] = h->a[--h->n];
    int i = 0;
    for (;;) {
        const int l = 2 * i + 1, r = l + 1;
        int m = i;
        if (l < h->n && h->a[l] < h->a[m]) m = l;
        if (r < h->n && h->a[r] < h->a[m]) m = r;
        if (m == i) break;
        const int t = h->a[m];
        h->a[m] = h->a[i];
        h->a[i] = t;
        i = m;
    }
    return top;
}

/* ilut.hpp:29-143 -- Saad dual-threshold ILU, natural order, no pivoting */
static int ilut_factor(const oc_csr* a, double tau, int fill_limit, mat* lower, mat* upper) {
    const int n = a->n_rows;
    const int nnz = a->row_offsets[n];
    if (fill_limit <= 0) fill_limit = (nnz + n - 1) / (n > 1 ? n : 1);
    mat_init(lower, n, n, nnz + 16);
    mat_init(upper, n, n, nnz + n + 16);
    double* w = (double*)calloc((size_t)n, sizeof(double));
    char* active = (char*)calloc((size_t)n, 1);
    int* touched = (int*)malloc(sizeof(int) * (size_t)n);
    int n_touched = 0;
    heap pending = {0, 0, 0};
    entry* lpart = (entry*)malloc(sizeof(entry) * (size_t)n);
    entry* upart = (entry*)malloc(sizeof(entry) * (size_t)n);
    int rc = 0;
    for (int i = 0; i < n && rc == 0; ++i) {
        double row_norm_sq = 0.0;
        for (int e = a->row_offsets[i]; e < a->row_offsets[i + 1]; ++e) {
            const int j = a->col_indices[e];
            const double v = a->values[e];
            row_norm_sq += v * v;
            w[j] = v;
            if (!active[j]) {
                active[j] = 1;
                touched[n_touched++] = j;
                if (j < i) heap_push(&pending, j);
            }
        }
        const double drop = tau * sqrt(row_norm_sq);
        while (pending.n > 0) {
            const int k = heap_pop(&pending);
            const int urow = upper->ro[k];
            const double beta = w[k] / upper->v[urow];
            if (fabs(beta) < drop) {
                w[k] = 0.0;
                continue;
            }
            w[k] = beta;
            for (int e = urow + 1; e < upper->ro[k + 1]; ++e) {
                const int j = upper->ci[e];
                if (!active[j]) {
                    active[j] = 1;
                    touched[n_touched++] = j;
                    w[j] = 0.0;
                    if (j < i) heap_push(&pending, j);
                }
                w[j] -= beta * upper->v[e];
            }
        }
        int nl = 0, nu = 0;
        double diag = 0.0;
        int diag_present = 0;
        for (int t = 0; t < n_touched; ++t) {
            const int j = touched[t];
            const double v = w[j];
            w[j] = 0.0;
            active[j] = 0;
            if (j == i) {
                diag = v;
                diag_present = 1;
            } else if (v != 0.0 && fabs(v) >= drop) {
                if (j < i) {
                    lpart[nl].col = j;
                    lpart[nl++].val = v;
                } else {
                    upart[nu].col = j;
                    upart[nu++].val = v;
                }
            }
        }
        n_touched = 0;
        if (!diag_present || diag == 0.0) {
            snprintf(g_err, sizeof g_err, "ilut_factor: zero pivot in row %d", i);
            rc = 1;
            break;
        }
        keep_largest(lpart, &nl, fill_limit);
        keep_largest(upart, &nu, fill_limit);
        for (int t = 0; t < nl; ++t) mat_push(lower, lpart[t].col, lpart[t].val);
        lower->ro[i + 1] = lower->nnz;
        mat_push(upper, i, diag);
        for (int t = 0; t < nu; ++t) mat_push(upper, upart[t].col, upart[t].val);
        upper->ro[i + 1] = upper->nnz;
    }
    free(w);
    free(active);
    free(touched);
    free(pending.a);
    free(lpart);
    free(upart);
    return rc;
}

/* ilut.hpp:146-163 -- forward (unit L) then backward (U, diagonal first) */
static void ilut_apply(const mat* lo, const mat* up, const double* r, double* z) {
    const int n = lo->n_rows;
    memcpy(z, r, sizeof(double) * (size_t)n);
    for (int i = 0; i < n; ++i) {
        double s = z[i];
        for (int e = lo->ro[i]; e < lo->ro[i + 1]; ++e) s -= lo->v[e] * z[lo->ci[e]];
        z[i] = s;
    }
    for (int i = n - 1; i >= 0; --i) {
        double s = z[i];
        const int begin = up->ro[i];
        for (int e = begin + 1; e < up->ro[i + 1]; ++e) s -= up->v[e] * z[up->ci[e]];
        z[i] = s / up->v[begin];
    }
}

/* ------------------------------------------------------------------------ */
/* pmultigrid.hpp                                                            */
/* ------------------------------------------------------------------------ */
struct oc_disc {
    oc_csr mass_p, stiff_p, transfer;
    const double* inv_lumped_p;
    const double* inv_lumped_1;
    int n_h;
    oc_csr* h_mass;
    oc_csr* h_stiff;
    oc_csr* h_embed; /* n_h - 1 */
    int n_p, n_1;
};

oc_disc* oc_disc_create(const oc_csr* mass_p, const oc_csr* stiff_p, const oc_csr* transfer,
                        const double* inv_lumped_p, const double* inv_lumped_1, int n_h,
                        const oc_csr* h_mass, const oc_csr* h_stiff, const oc_csr* h_embed) {
    oc_disc* d = (oc_disc*)calloc(1, sizeof(oc_disc));
    d->mass_p = *mass_p;
    d->stiff_p = *stiff_p;
    d->transfer = *transfer;
    d->inv_lumped_p = inv_lumped_p;
    d->inv_lumped_1 = inv_lumped_1;
    d->n_h = n_h;
    d->h_mass = (oc_csr*)malloc(sizeof(oc_csr) * (size_t)n_h);
    d->h_stiff = (oc_csr*)malloc(sizeof(oc_csr) * (size_t)n_h);
    d->h_embed = (oc_csr*)malloc(sizeof(oc_csr) * (size_t)(n_h > 1 ? n_h - 1 : 1));
    for (int l = 0; l < n_h; ++l) {
        d->h_mass[l] = h_mass[l];
        d->h_stiff[l] = h_stiff[l];
        if (l + 1 < n_h) d->h_embed[l] = h_embed[l];
    }
    d->n_p = mass_p->n_rows;
    d->n_1 = transfer->n_cols;
    return d;
}

void oc_disc_free(oc_disc* d) {
    if (!d) return;
    free(d->h_mass);
    free(d->h_stiff);
    free(d->h_embed);
    free(d);
}

struct oc_hier {
    const oc_disc* d;
    int nu_pre, nu_post, gs_pre, gs_post;
    mat a_p, lower, upper;
    mat* a_h;
    dense_lu coarse;
};

/* pmultigrid.hpp:217-224 */
oc_hier* oc_hier_create(const oc_disc* d, double c, int nu_pre, int nu_post, int gs_pre,
                        int gs_post, double ilut_tau, int ilut_fill) {
    oc_hier* h = (oc_hier*)calloc(1, sizeof(oc_hier));
    h->d = d;
    h->nu_pre = nu_pre;
    h->nu_post = nu_post;
    h->gs_pre = gs_pre;
    h->gs_post = gs_post;
    sparse_add(1.0, &d->mass_p, c, &d->stiff_p, &h->a_p);
    oc_csr ap = view(&h->a_p);
    if (ilut_factor(&ap, ilut_tau, ilut_fill, &h->lower, &h->upper)) {
        oc_hier_free(h);
        return NULL;
    }
    h->a_h = (mat*)calloc((size_t)d->n_h, sizeof(mat));
    for (int l = 0; l < d->n_h; ++l) sparse_add(1.0, &d->h_mass[l], c, &d->h_stiff[l], &h->a_h[l]);
    oc_csr last = view(&h->a_h[d->n_h - 1]);
    if (dense_lu_factor(&h->coarse, &last)) {
        oc_hier_free(h);
        return NULL;
    }
    return h;
}

void oc_hier_free(oc_hier* h) {
    if (!h) return;
    mat_free(&h->a_p);
    mat_free(&h->lower);
    mat_free(&h->upper);
    if (h->a_h)
        for (int l = 0; l < h->d->n_h; ++l) mat_free(&h->a_h[l]);
    free(h->a_h);
    free(h->coarse.lu);
    free(h->coarse.piv);
    free(h);
}

int oc_hier_n_levels(const oc_hier* h) { return h->d->n_h; }

int oc_hier_csr(const oc_hier* h, int which, int* n_rows, int* n_cols, int* nnz, int* ro, int* ci,
                double* v) {
    const mat* a = NULL;
    if (which == 0) a = &h->a_p;
    else if (which == 1) a = &h->lower;
    else if (which == 2) a = &h->upper;
    else if (which >= 100 && which - 100 < h->d->n_h) a = &h->a_h[which - 100];
    if (!a) return set_err("oc_hier_csr: bad selector");
    return export_mat(a, n_rows, n_cols, nnz, ro, ci, v);
}

int oc_ilut_apply(const oc_hier* h, const double* r, double* z) {
    ilut_apply(&h->lower, &h->upper, r, z);
    return 0;
}

/* pmultigrid.hpp:242-247 */
int oc_restrict(const oc_hier* h, const double* r, double* r1) {
    oc_spmv_transpose(&h->d->transfer, r, r1);
    for (int i = 0; i < h->d->n_1; ++i) r1[i] *= h->d->inv_lumped_1[i];
    return 0;
}

/* pmultigrid.hpp:250-254 */
int oc_prolong(const oc_hier* h, const double* e1, double* ep) {
    oc_spmv(&h->d->transfer, e1, ep);
    for (int i = 0; i < h->d->n_p; ++i) ep[i] *= h->d->inv_lumped_p[i];
    return 0;
}

int oc_coarse_solve(const oc_hier* h, const double* b, double* x) {
    dense_lu_solve(&h->coarse, b, x);
    return 0;
}

/* pmultigrid.hpp:184-200 */
static int wcycle(const oc_hier* h, int level, const double* b, double* x) {
    const oc_disc* d = h->d;
    if (level + 1 == d->n_h) {
        dense_lu_solve(&h->coarse, b, x);
        return 0;
    }
    oc_csr a = view(&h->a_h[level]);
    const int n = a.n_rows;
    const oc_csr* e = &d->h_embed[level];
    const int nc = e->n_cols;
    int rc = 0;
    for (int s = 0; s < h->gs_pre && !rc; ++s) rc = oc_gs_sweep(&a, b, x, 0);
    if (rc) return rc;
    double* r = (double*)malloc(sizeof(double) * (size_t)n);
    oc_spmv(&a, x, r);
    for (int i = 0; i < n; ++i) r[i] = b[i] - r[i];
    double* rc_ = (double*)malloc(sizeof(double) * (size_t)nc);
    double* ec = (double*)calloc((size_t)nc, sizeof(double));
    oc_spmv_transpose(e, r, rc_);
    rc = wcycle(h, level + 1, rc_, ec);
    if (!rc) rc = wcycle(h, level + 1, rc_, ec);
    if (!rc) {
        oc_spmv(e, ec, r); /* r reused as "up" */
        axpy1(r, x, n);
        for (int s = 0; s < h->gs_post && !rc; ++s) rc = oc_gs_sweep(&a, b, x, 1);
    }
    free(r);
    free(rc_);
    free(ec);
    return rc;
}

int oc_hmg_wcycle(const oc_hier* h, const double* b1, double* x1) { return wcycle(h, 0, b1, x1); }

/* pmultigrid.hpp:311-316 -- x += S (b - A x) */
static void smooth(const oc_hier* h, const double* b, double* x, double* r, double* z) {
    oc_csr a = view(&h->a_p);
    const int n = a.n_rows;
    oc_spmv(&a, x, r);
    for (int i = 0; i < n; ++i) r[i] = b[i] - r[i];
    ilut_apply(&h->lower, &h->upper, r, z);
    axpy1(z, x, n);
}

/* pmultigrid.hpp:256-267 */
int oc_vcycle(const oc_hier* h, const double* b, double* x) {
    const oc_disc* d = h->d;
    const int n = d->n_p, n1 = d->n_1;
    double* r = (double*)malloc(sizeof(double) * (size_t)n);
    double* z = (double*)malloc(sizeof(double) * (size_t)n);
    double* r1 = (double*)malloc(sizeof(double) * (size_t)n1);
    double* e1 = (double*)calloc((size_t)n1, sizeof(double));
    for (int s = 0; s < h->nu_pre; ++s) smooth(h, b, x, r, z);
    oc_csr a = view(&h->a_p);
    oc_spmv(&a, x, r);
    for (int i = 0; i < n; ++i) r[i] = b[i] - r[i];
    oc_restrict(h, r, r1);
    int rc = wcycle(h, 0, r1, e1);
    if (!rc) {
        oc_prolong(h, e1, z);
        axpy1(z, x, n);
        for (int s = 0; s < h->nu_post; ++s) smooth(h, b, x, r, z);
    }
    free(r);
    free(z);
    free(r1);
    free(e1);
    return rc;
}

static double residual_rel(const oc_hier* h, const double* b, const double* x, double bnorm,
                           double* r) {
    oc_csr a = view(&h->a_p);
    oc_spmv(&a, x, r);
    for (int i = 0; i < a.n_rows; ++i) r[i] = b[i] - r[i];
    return oc_norm2(r, a.n_rows) / bnorm;
}

/* pmultigrid.hpp:271-307 */
int oc_solve(const oc_hier* h, const double* b, double* x, double rel_tol, int max_iter,
             int fixed_cycles, int x0_empty, int* iters, int* converged, double* final_rel,
             double* history, int history_cap) {
    const int n = h->d->n_p;
    *iters = 0;
    *converged = 0;
    *final_rel = 0.0;
    const double bnorm = oc_norm2(b, n);
    if (bnorm == 0.0) {
        memset(x, 0, sizeof(double) * (size_t)n);
        *converged = 1;
        return 0;
    }
    if (x0_empty) memset(x, 0, sizeof(double) * (size_t)n);
    double* r = (double*)malloc(sizeof(double) * (size_t)n);
    int rc = 0;
    if (fixed_cycles > 0) {
        for (int it = 0; it < fixed_cycles && !rc; ++it) rc = oc_vcycle(h, b, x);
        *iters = fixed_cycles;
        *final_rel = residual_rel(h, b, x, bnorm, r);
        *converged = 1;
        free(r);
        return rc;
    }
    double rel = residual_rel(h, b, x, bnorm, r);
    if (rel <= rel_tol) {
        *converged = 1;
        *final_rel = rel;
        free(r);
        return 0;
    }
    for (int it = 1; it <= max_iter; ++it) {
        rc = oc_vcycle(h, b, x);
        if (rc) break;
        rel = residual_rel(h, b, x, bnorm, r);
        *iters = it;
        if (history && it - 1 < history_cap) history[it - 1] = rel;
        if (rel <= rel_tol) {
            *converged = 1;
            break;
        }
    }
    *final_rel = rel;
    free(r);
    return rc;
}

/* ------------------------------------------------------------------------ */
/* theta.hpp                                                                 */
/* ------------------------------------------------------------------------ */
struct oc_stepper {
    const oc_disc* d;
    mat a_plus, a_minus;
    int kind;      /* SpatialSolverKind (theta.hpp:64): 0 pmg, 1 cg */
    oc_hier* pmg;  /* pmg kind */
    double* diag;  /* cg kind: diagonal_of(a_plus) (sparse.hpp:180-184) */
    double rel_tol;
    int max_iter, fixed_cycles;
};

/* theta.hpp:94-103 */
oc_stepper* oc_stepper_create_kind(const oc_disc* d, double kappa, double dt, double theta,
                                   int kind, double rel_tol, int max_iter, int fixed_cycles) {
    if (kind != 0 && kind != 1) {
        set_err("unknown spatial solver kind");
        return NULL;
    }
    oc_stepper* s = (oc_stepper*)calloc(1, sizeof(oc_stepper));
    s->d = d;
    s->kind = kind;
    sparse_add(1.0, &d->mass_p, kappa * dt * theta, &d->stiff_p, &s->a_plus);
    sparse_add(1.0, &d->mass_p, -kappa * dt * (1.0 - theta), &d->stiff_p, &s->a_minus);
    if (kind == 0) {
        s->pmg = oc_hier_create(d, kappa * dt * theta, 1, 1, 2, 2, 1e-13, 0);
        if (!s->pmg) {
            oc_stepper_free(s);
            return NULL;
        }
    } else {
        const int n = s->a_plus.n_rows;
        s->diag = (double*)calloc((size_t)n, sizeof(double));
        for (int i = 0; i < n; ++i)
            for (int e = s->a_plus.ro[i]; e < s->a_plus.ro[i + 1]; ++e)
                if (s->a_plus.ci[e] == i) s->diag[i] = s->a_plus.v[e];
    }
    s->rel_tol = rel_tol;
    s->max_iter = max_iter;
    s->fixed_cycles = fixed_cycles;
    return s;
}

oc_stepper* oc_stepper_create(const oc_disc* d, double kappa, double dt, double theta,
                              double rel_tol, int max_iter, int fixed_cycles) {
    return oc_stepper_create_kind(d, kappa, dt, theta, 0, rel_tol, max_iter, fixed_cycles);
}

void oc_stepper_free(oc_stepper* s) {
    if (!s) return;
    mat_free(&s->a_plus);
    mat_free(&s->a_minus);
    oc_hier_free(s->pmg);
    free(s->diag);
    free(s);
}

/* solvers.hpp:21-75 -- Jacobi-preconditioned CG; x holds x0 (zeros when the
 * reference's x0 is empty).  Returns 0, or 3 on breakdown (p^T A p <= 0). */
static int cg_solve(const mat* am, const double* b, double* x, double rel_tol, int max_iter,
                    const double* diag, int* iters, int* converged) {
    const int n = am->n_rows;
    const oc_csr a = view(am);
    *iters = 0;
    *converged = 0;
    const double bnorm = sqrt(dot(b, b, n));
    if (bnorm == 0.0) {
        for (int i = 0; i < n; ++i) x[i] = 0.0;
        *converged = 1;
        return 0;
    }
    double* r = (double*)malloc(sizeof(double) * (size_t)n * 4);
    double *z = r + n, *p = r + 2 * (size_t)n, *q = r + 3 * (size_t)n;
    oc_spmv(&a, x, q);
    for (int i = 0; i < n; ++i) r[i] = b[i] - q[i];  /* subtract(b, spmv(a, x)) */
    double rnorm = sqrt(dot(r, r, n));
    int rc = 0;
    if (rnorm <= rel_tol * bnorm) {
        *converged = 1;
        goto done;
    }
    for (int i = 0; i < n; ++i) z[i] = r[i] / diag[i];
    for (int i = 0; i < n; ++i) p[i] = z[i];
    double rz = dot(r, z, n);
    for (int it = 1; it <= max_iter; ++it) {
        oc_spmv(&a, p, q);
        const double pq = dot(p, q, n);
        if (pq <= 0.0) {
            set_err("cg_solve: breakdown, matrix not SPD");
            rc = 3;
            goto done;
        }
        const double alpha = rz / pq;
        for (int i = 0; i < n; ++i) x[i] += alpha * p[i];
        for (int i = 0; i < n; ++i) r[i] += -alpha * q[i];
        rnorm = sqrt(dot(r, r, n));
        *iters = it;
        if (rnorm <= rel_tol * bnorm) {
            *converged = 1;
            goto done;
        }
        for (int i = 0; i < n; ++i) z[i] = r[i] / diag[i];
        const double rz_new = dot(r, z, n);
        const double beta = rz_new / rz;
        rz = rz_new;
        for (int i = 0; i < n; ++i) p[i] = z[i] + beta * p[i];
    }
done:
    free(r);
    return rc;
}

/* theta.hpp:111-126 -- solve_lhs */
static int solve_lhs(const oc_stepper* s, const double* rhs, const double* guess, double* out,
                     int* iters) {
    const int n = s->d->n_p;
    int conv = 0;
    double fr = 0.0;
    if (s->kind == 1) {
        if (guess)
            memcpy(out, guess, sizeof(double) * (size_t)n);
        else
            memset(out, 0, sizeof(double) * (size_t)n);
        const int rc = cg_solve(&s->a_plus, rhs, out, s->rel_tol, s->max_iter, s->diag, iters, &conv);
        if (rc) return rc;
        if (!conv) {
            set_err("spatial solve did not converge (cg)");
            return 2;
        }
        return 0;
    }
    if (guess) memcpy(out, guess, sizeof(double) * (size_t)n);
    int rc = oc_solve(s->pmg, rhs, out, s->rel_tol, s->max_iter, s->fixed_cycles, guess == NULL,
                      iters, &conv, &fr, NULL, 0);
    if (rc) return rc;
    if (!conv) {
        snprintf(g_err, sizeof g_err, "spatial solve did not converge (p-multigrid), residual %f", fr);
        return 2;
    }
    return 0;
}

/* theta.hpp:132-137 */
int oc_stepper_step(const oc_stepper* s, const double* u_prev, const double* load,
                    const double* guess, double* out, int* iters) {
    const int n = s->d->n_p;
    double* rhs = (double*)malloc(sizeof(double) * (size_t)n);
    oc_csr am = view(&s->a_minus);
    oc_spmv(&am, u_prev, rhs);
    if (load) axpy1(load, rhs, n);
    int it = 0;
    const int rc = solve_lhs(s, rhs, guess, out, &it);
    if (iters) *iters = it;
    free(rhs);
    return rc;
}

/* theta.hpp:216-237 -- u0 given (already projected), loads as described */
int oc_sequential_integrate(const oc_disc* d, double kappa, double t_final, int nt, double theta,
                            const double* u0, const double* loads, int load_steady,
                            double rel_tol, int max_iter, double* traj, long long* solves,
                            long long* iterations) {
    const int n = d->n_p;
    const double dt = t_final / nt;
    oc_stepper* s = oc_stepper_create(d, kappa, dt, theta, rel_tol, max_iter, 0);
    if (!s) return 1;
    if (u0)
        memcpy(traj, u0, sizeof(double) * (size_t)n);
    else
        memset(traj, 0, sizeof(double) * (size_t)n);
    *solves = 0;
    *iterations = 0;
    int rc = 0;
    for (int k = 1; k <= nt && !rc; ++k) {
        const double* load = NULL;
        if (loads) load = load_steady ? loads : loads + (size_t)(k - 1) * n;
        int it = 0;
        const double* prev = traj + (size_t)(k - 1) * n;
        rc = oc_stepper_step(s, prev, load, prev, traj + (size_t)k * n, &it);
        *solves += 1;
        *iterations += it;
        if (rc) {
            char buf[512];
            snprintf(buf, sizeof buf, "sequential_integrate: step %d: %s", k, g_err);
            set_err(buf);
        }
    }
    oc_stepper_free(s);
    return rc;
}

/* ------------------------------------------------------------------------ */
/* mgrit.hpp                                                                 */
/* ------------------------------------------------------------------------ */
typedef struct {
    int steps;
    double dt;
    oc_stepper* stepper;
    double* u; /* (steps+1) x n */
    double* g;
} level_t;

struct oc_mgrit {
    const oc_disc* d;
    int n, nt, n_levels, m, max_iter, cycle, relax;
    double halt_tol, g_norm, kappa, theta;
    const double* u0;
    const double* loads;
    int load_steady;
    level_t lev[32];
    long long solves, iters;
};

/* mgrit.hpp:217-244 build_levels */
oc_mgrit* oc_mgrit_create(const oc_disc* d, double kappa, double t_final, int nt, double theta,
                          const double* u0, const double* loads, int load_steady, int cycle,
                          int relax, int m, double halt_tol, int max_iter, int coarse_floor,
                          double rel_tol, int sp_max_iter) {
    return oc_mgrit_create_kind(d, kappa, t_final, nt, theta, u0, loads, load_steady, cycle, relax,
                                m, halt_tol, max_iter, coarse_floor, 0, rel_tol, sp_max_iter);
}

oc_mgrit* oc_mgrit_create_kind(const oc_disc* d, double kappa, double t_final, int nt,
                               double theta, const double* u0, const double* loads,
                               int load_steady, int cycle, int relax, int m, double halt_tol,
                               int max_iter, int coarse_floor, int spatial_kind, double rel_tol,
                               int sp_max_iter) {
    if (m < 2) {
        set_err("MgritConfig: m must be >= 2");
        return NULL;
    }
    if (nt >= m && nt % m != 0) {
        snprintf(g_err, sizeof g_err,
                 "MGRIT: nt (%d) not divisible by coarsening factor m (%d)", nt, m);
        return NULL;
    }
    oc_mgrit* g = (oc_mgrit*)calloc(1, sizeof(oc_mgrit));
    g->d = d;
    g->n = d->n_p;
    g->nt = nt;
    g->m = m;
    g->cycle = cycle;
    g->relax = relax;
    g->halt_tol = halt_tol;
    g->max_iter = max_iter;
    g->kappa = kappa;
    g->theta = theta;
    g->u0 = u0;
    g->loads = loads;
    g->load_steady = load_steady;
    int steps[32];
    int L = 0;
    steps[L++] = nt;
    for (;;) {
        const int cur = steps[L - 1];
        if (cur % m != 0 || cur < m) break;
        const int next = cur / m;
        const int first_coarse = (L == 1);
        if (!first_coarse && next + 1 <= coarse_floor) break;
        steps[L++] = next;
        if (cycle == 2) break; /* two_level */
        if (L == 32) break;
    }
    g->n_levels = L;
    const double dt0 = t_final / nt;
    for (int l = 0; l < L; ++l) {
        level_t* lv = &g->lev[l];
        lv->steps = steps[l];
        lv->dt = dt0 * (nt / steps[l]);
        lv->stepper = oc_stepper_create_kind(d, kappa, lv->dt, theta, spatial_kind, rel_tol, sp_max_iter, 0);
        if (!lv->stepper) {
            oc_mgrit_free(g);
            return NULL;
        }
        lv->u = (double*)calloc((size_t)(lv->steps + 1) * g->n, sizeof(double));
        lv->g = (double*)calloc((size_t)(lv->steps + 1) * g->n, sizeof(double));
    }
    return g;
}

void oc_mgrit_free(oc_mgrit* g) {
    if (!g) return;
    for (int l = 0; l < g->n_levels; ++l) {
        oc_stepper_free(g->lev[l].stepper);
        free(g->lev[l].u);
        free(g->lev[l].g);
    }
    free(g);
}

int oc_mgrit_levels(const oc_mgrit* g, int* steps, double* dts) {
    for (int l = 0; l < g->n_levels; ++l) {
        steps[l] = g->lev[l].steps;
        dts[l] = g->lev[l].dt;
    }
    return g->n_levels;
}

static const double* load_term(const oc_mgrit* g, int l, int k) {
    if (l != 0 || !g->loads) return NULL;
    return g->load_steady ? g->loads : g->loads + (size_t)(k - 1) * g->n;
}

/* mgrit.hpp:261-269 step_value: Phi(u[k-1]) + load, guess u[k] */
static int step_value(oc_mgrit* g, int l, int k, double* out) {
    level_t* lv = &g->lev[l];
    const int n = g->n;
    int it = 0;
    const int rc = oc_stepper_step(lv->stepper, lv->u + (size_t)(k - 1) * n, load_term(g, l, k),
                                   lv->u + (size_t)k * n, out, &it);
    g->solves += 1;
    g->iters += it;
    if (rc) {
        char buf[512];
        snprintf(buf, sizeof buf, "MGRIT level %d, time step %d: %s", l, k, g_err);
        set_err(buf);
    }
    return rc;
}

/* mgrit.hpp:253-258 step_into: u[k] <- step_value + g[k] */
static int step_into(oc_mgrit* g, int l, int k, double* w) {
    level_t* lv = &g->lev[l];
    const int n = g->n;
    const int rc = step_value(g, l, k, w);
    if (rc) return rc;
    axpy1(lv->g + (size_t)k * n, w, n);
    memcpy(lv->u + (size_t)k * n, w, sizeof(double) * (size_t)n);
    return 0;
}

/* mgrit.hpp:122-132 (intervals independent; run in index order here) */
static int f_relax(oc_mgrit* g, int l, double* w) {
    const int J = g->lev[l].steps / g->m;
    for (int j = 0; j < J; ++j)
        for (int t = 1; t < g->m; ++t) {
            const int rc = step_into(g, l, j * g->m + t, w);
            if (rc) return rc;
        }
    return 0;
}

/* mgrit.hpp:135-141 */
static int c_relax(oc_mgrit* g, int l, double* w) {
    const int J = g->lev[l].steps / g->m;
    for (int j = 0; j < J; ++j) {
        const int rc = step_into(g, l, (j + 1) * g->m, w);
        if (rc) return rc;
    }
    return 0;
}

/* mgrit.hpp:151-167 */
static int restrict_residual(oc_mgrit* g, int l, double* w) {
    level_t* f = &g->lev[l];
    level_t* c = &g->lev[l + 1];
    const int n = g->n;
    const int J = f->steps / g->m;
    for (int j = 0; j <= J; ++j) {
        const int k = j * g->m;
        double* cg = c->g + (size_t)j * n;
        if (j == 0) {
            for (int i = 0; i < n; ++i) cg[i] = f->g[i] - f->u[i];
        } else {
            const int rc = step_value(g, l, k, w);
            if (rc) return rc;
            axpy1(f->g + (size_t)k * n, w, n);
            for (int i = 0; i < n; ++i) cg[i] = w[i] - f->u[(size_t)k * n + i];
        }
        memset(c->u + (size_t)j * n, 0, sizeof(double) * (size_t)n);
    }
    memcpy(c->u, c->g, sizeof(double) * (size_t)n);
    return 0;
}

/* mgrit.hpp:172-180 */
static int interpolate_and_correct(oc_mgrit* g, int l, double* w) {
    level_t* f = &g->lev[l];
    level_t* c = &g->lev[l + 1];
    const int n = g->n;
    const int J = f->steps / g->m;
    for (int j = 0; j <= J; ++j) axpy1(c->u + (size_t)j * n, f->u + (size_t)j * g->m * n, n);
    return f_relax(g, l, w);
}

/* mgrit.hpp:188-194 */
static int coarsest_solve(oc_mgrit* g, int l, double* w) {
    level_t* lv = &g->lev[l];
    memcpy(lv->u, lv->g, sizeof(double) * (size_t)g->n);
    for (int k = 1; k <= lv->steps; ++k) {
        const int rc = step_into(g, l, k, w);
        if (rc) return rc;
    }
    return 0;
}

/* mgrit.hpp:197-214 */
static int residual_norm(oc_mgrit* g, int l, double* w, double* out) {
    level_t* lv = &g->lev[l];
    const int n = g->n;
    double* sq = (double*)calloc((size_t)lv->steps + 1, sizeof(double));
    for (int i = 0; i < n; ++i) w[i] = lv->g[i] - lv->u[i];
    sq[0] = dot(w, w, n);
    for (int k = 1; k <= lv->steps; ++k) {
        const int rc = step_value(g, l, k, w);
        if (rc) {
            free(sq);
            return rc;
        }
        axpy1(lv->g + (size_t)k * n, w, n);
        for (int i = 0; i < n; ++i) w[i] = w[i] - lv->u[(size_t)k * n + i];
        sq[k] = dot(w, w, n);
    }
    double total = 0.0;
    for (int k = 0; k <= lv->steps; ++k) total += sq[k];
    free(sq);
    *out = sqrt(total);
    return 0;
}

static int relax(oc_mgrit* g, int l, double* w) {
    int rc = f_relax(g, l, w);
    if (rc || g->relax == 0) return rc;
    rc = c_relax(g, l, w);
    if (rc) return rc;
    return f_relax(g, l, w);
}

/* mgrit.hpp:278-288 */
static int cycle_impl(oc_mgrit* g, int l, int f_schedule, double* w) {
    if (l + 1 == g->n_levels) return coarsest_solve(g, l, w);
    int rc = relax(g, l, w);
    if (!rc) rc = restrict_residual(g, l, w);
    if (!rc) rc = cycle_impl(g, l + 1, f_schedule, w);
    if (!rc) rc = interpolate_and_correct(g, l, w);
    if (!rc && f_schedule && l + 2 < g->n_levels) rc = cycle_impl(g, l, 0, w);
    return rc;
}

/* mgrit.hpp:292-310 compute_g_norm */
static int compute_g_norm(oc_mgrit* g, double* w, double* out) {
    level_t* lv = &g->lev[0];
    const int n = g->n;
    double total = dot(lv->g, lv->g, n);
    if (g->loads) {
        int it = 0;
        if (g->load_steady) {
            const int rc = solve_lhs(lv->stepper, g->loads, NULL, w, &it);
            g->solves += 1;
            g->iters += it;
            if (rc) return rc;
            total += lv->steps * dot(w, w, n);
        } else {
            double* sq = (double*)calloc((size_t)lv->steps + 1, sizeof(double));
            for (int k = 1; k <= lv->steps; ++k) {
                const int rc = solve_lhs(lv->stepper, g->loads + (size_t)(k - 1) * n, NULL, w, &it);
                g->solves += 1;
                g->iters += it;
                if (rc) {
                    free(sq);
                    return rc;
                }
                sq[k] = dot(w, w, n);
            }
            for (int k = 0; k <= lv->steps; ++k) total += sq[k];
            free(sq);
        }
    }
    *out = sqrt(total);
    return 0;
}

/* mgrit.hpp:78-91 initialize + 93-118 solve */
int oc_mgrit_solve(oc_mgrit* g, int* iterations, int* converged, double* g_norm, double* final_rel,
                   long long* solves, double* mean_iters, double* history, int history_cap) {
    const int n = g->n;
    for (int l = 0; l < g->n_levels; ++l) {
        memset(g->lev[l].u, 0, sizeof(double) * (size_t)(g->lev[l].steps + 1) * n);
        memset(g->lev[l].g, 0, sizeof(double) * (size_t)(g->lev[l].steps + 1) * n);
    }
    if (g->u0) {
        memcpy(g->lev[0].g, g->u0, sizeof(double) * (size_t)n);
        memcpy(g->lev[0].u, g->u0, sizeof(double) * (size_t)n);
    }
    g->solves = 0;
    g->iters = 0;
    double* w = (double*)malloc(sizeof(double) * (size_t)n);
    int rc = compute_g_norm(g, w, &g->g_norm);
    *iterations = 0;
    *converged = 0;
    double rel = 0.0;
    if (!rc) {
        const double denom = g->g_norm > 0.0 ? g->g_norm : 1.0;
        for (int it = 1; it <= g->max_iter; ++it) {
            rc = cycle_impl(g, 0, g->cycle == 1, w);
            if (rc) break;
            double rn = 0.0;
            rc = residual_norm(g, 0, w, &rn);
            if (rc) break;
            rel = rn / denom;
            if (history && it - 1 < history_cap) history[it - 1] = rel;
            *iterations = it;
            if (rel <= g->halt_tol) {
                *converged = 1;
                break;
            }
        }
    }
    free(w);
    *g_norm = g->g_norm;
    *final_rel = rel;
    *solves = g->solves;
    *mean_iters = g->solves > 0 ? (double)g->iters / (double)g->solves : 0.0;
    return rc;
}

int oc_mgrit_trajectory(const oc_mgrit* g, double* out) {
    memcpy(out, g->lev[0].u, sizeof(double) * (size_t)(g->lev[0].steps + 1) * g->n);
    return 0;
}
