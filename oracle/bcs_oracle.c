/* TEST INFRASTRUCTURE ONLY — CPU checker; see bcs_oracle.h for the contract.
 *
 * Restates the reference algorithms in plain C, in the reference's operation
 * order, so that (compiled with -ffp-contract=off, like the reference's own
 * -O3 build without -march) every result is bit-identical to
 * /root/reference/proj/core.  tests/test_oracle.py proves that against the
 * compiled reference (oracle/_ref) and the committed golden vectors.
 */
#include "bcs_oracle.h"

#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static char g_err[512];
const char* or_last_error(void) { return g_err; }

enum { OR_OK = 0, OR_INVALID = 1, OR_RUNTIME = 2 };
static int fail(int code, const char* msg) {
    snprintf(g_err, sizeof g_err, "%s", msg);
    return code;
}

static void* xcalloc(size_t n, size_t s) {
    void* p = calloc(n ? n : 1, s);
    if (!p) {
        fprintf(stderr, "bcs_oracle: out of memory\n");
        abort();
    }
    return p;
}

/* ------------------------------------------------------------------ BSR */
typedef struct {
    int rows, n, nnz;
    int* ro;
    int* ci;
    double* v;
} Bsr;

static void bsr_free(Bsr* a) {
    free(a->ro);
    free(a->ci);
    free(a->v);
    memset(a, 0, sizeof *a);
}

/* BlockCsrMatrix::find (block_csr.cpp:11-18): lower_bound in the row */
static int bsr_find(const Bsr* a, int row, int col) {
    int lo = a->ro[row], hi = a->ro[row + 1];
    while (lo < hi) {
        int mid = lo + (hi - lo) / 2;
        if (a->ci[mid] < col) lo = mid + 1;
        else hi = mid;
    }
    return (lo < a->ro[row + 1] && a->ci[lo] == col) ? lo : -1;
}

/* buildPlan (block_csr.cpp:56-80): per row diag + upper faces (owner==row) +
 * lower faces (neighbour==row) in face order, then sorted by column. */
int or_csr_plan(int nc, int nf, const int* owner, const int* neigh, int* row_off, int* cols, int* src) {
    int* fill = (int*)xcalloc((size_t)nc, sizeof(int));
    for (int r = 0; r <= nc; ++r) row_off[r] = 0;
    for (int c = 0; c < nc; ++c) row_off[c + 1] += 1;
    for (int f = 0; f < nf; ++f) {
        row_off[owner[f] + 1] += 1;
        row_off[neigh[f] + 1] += 1;
    }
    for (int r = 0; r < nc; ++r) row_off[r + 1] += row_off[r];
    for (int c = 0; c < nc; ++c) {
        int k = row_off[c] + fill[c]++;
        cols[k] = c;
        src[k] = c;
    }
    for (int f = 0; f < nf; ++f) {
        int k = row_off[owner[f]] + fill[owner[f]]++;
        cols[k] = neigh[f];
        src[k] = nc + f;
        k = row_off[neigh[f]] + fill[neigh[f]]++;
        cols[k] = owner[f];
        src[k] = nc + nf + f;
    }
    for (int r = 0; r < nc; ++r) /* insertion sort by column (columns distinct) */
        for (int k = row_off[r] + 1; k < row_off[r + 1]; ++k) {
            int c = cols[k], s = src[k], q = k - 1;
            while (q >= row_off[r] && cols[q] > c) {
                cols[q + 1] = cols[q];
                src[q + 1] = src[q];
                --q;
            }
            cols[q + 1] = c;
            src[q + 1] = s;
        }
    free(fill);
    return row_off[nc];
}

/* lduToBlockCsr / replaceValues value copy (block_csr.cpp:97-109, 120-127) */
void or_csr_values(int nc, int nf, int n, const int* src, const double* diag, const double* upper,
                   const double* lower, double* vals) {
    const size_t nn = (size_t)n * n;
    const int nnz = nc + 2 * nf;
    for (int k = 0; k < nnz; ++k) {
        const int s = src[k];
        const double* from = s < nc ? diag + (size_t)s * nn
                             : s < nc + nf ? upper + (size_t)(s - nc) * nn
                                           : lower + (size_t)(s - nc - nf) * nn;
        memcpy(vals + (size_t)k * nn, from, nn * sizeof(double));
    }
}

static void bsr_from_ldu(int nc, int nf, int n, const int* owner, const int* neigh, const double* diag,
                         const double* upper, const double* lower, Bsr* a) {
    a->rows = nc;
    a->n = n;
    a->nnz = nc + 2 * nf;
    a->ro = (int*)xcalloc((size_t)nc + 1, sizeof(int));
    a->ci = (int*)xcalloc((size_t)a->nnz, sizeof(int));
    a->v = (double*)xcalloc((size_t)a->nnz * n * n, sizeof(double));
    int* src = (int*)xcalloc((size_t)a->nnz, sizeof(int));
    or_csr_plan(nc, nf, owner, neigh, a->ro, a->ci, src);
    or_csr_values(nc, nf, n, src, diag, upper, lower, a->v);
    free(src);
}

/* topologySignature (block_csr.cpp:140-160) */
static uint64_t hash_combine(uint64_t h, uint64_t v) {
    h ^= v + 0x9e3779b97f4a7c15ull + (h << 6) + (h >> 2);
    return h;
}
static int face_cmp(const void* a, const void* b) {
    const int* x = (const int*)a;
    const int* y = (const int*)b;
    if (x[0] != y[0]) return x[0] < y[0] ? -1 : 1;
    if (x[1] != y[1]) return x[1] < y[1] ? -1 : 1;
    return 0;
}
unsigned long long or_signature(int nc, int nf, const int* owner, const int* neigh) {
    uint64_t h = hash_combine(0, (uint64_t)(int64_t)nc);
    int* fa = (int*)xcalloc((size_t)nf * 2, sizeof(int));
    for (int f = 0; f < nf; ++f) {
        fa[2 * f] = owner[f];
        fa[2 * f + 1] = neigh[f];
    }
    qsort(fa, (size_t)nf, 2 * sizeof(int), face_cmp);
    for (int f = 0; f < nf; ++f) {
        h = hash_combine(h, (uint64_t)(int64_t)fa[2 * f]);
        h = hash_combine(h, (uint64_t)(int64_t)fa[2 * f + 1]);
    }
    free(fa);
    return h;
}

/* ------------------------------------------------------ dense n x n blocks */
/* smallmat::matvecAdd (smallmat.hpp:17-24) */
static void mv_add(const double* A, const double* x, double* y, int n) {
    for (int i = 0; i < n; ++i) {
        double s = 0.0;
        for (int j = 0; j < n; ++j) s += A[i * n + j] * x[j];
        y[i] += s;
    }
}
/* smallmat::matvecSub (smallmat.hpp:27-34) */
static void mv_sub(const double* A, const double* x, double* y, int n) {
    for (int i = 0; i < n; ++i) {
        double s = 0.0;
        for (int j = 0; j < n; ++j) s += A[i * n + j] * x[j];
        y[i] -= s;
    }
}
/* smallmat::matmulSub (smallmat.hpp:48-56), skipping a == 0 */
static void mm_sub(const double* A, const double* B, double* C, int n) {
    for (int i = 0; i < n; ++i)
        for (int k = 0; k < n; ++k) {
            const double a = A[i * n + k];
            if (a == 0.0) continue;
            for (int j = 0; j < n; ++j) C[i * n + j] -= a * B[k * n + j];
        }
}
/* smallmat::luFactor (smallmat.hpp:67-94) in place; 0 ok, -1 singular.
 * Also serves denseFactor (smallmat.hpp:134-161), which is the same loop. */
static int lu_factor(double* lu, int* piv, int n) {
    for (int k = 0; k < n; ++k) {
        int p = k;
        double best = fabs(lu[(size_t)k * n + k]);
        for (int i = k + 1; i < n; ++i) {
            const double v = fabs(lu[(size_t)i * n + k]);
            if (v > best) {
                best = v;
                p = i;
            }
        }
        if (best < 1e-300) return -1;
        piv[k] = p;
        if (p != k)
            for (int j = 0; j < n; ++j) {
                double t = lu[(size_t)k * n + j];
                lu[(size_t)k * n + j] = lu[(size_t)p * n + j];
                lu[(size_t)p * n + j] = t;
            }
        const double d = lu[(size_t)k * n + k];
        for (int i = k + 1; i < n; ++i) {
            double m = lu[(size_t)i * n + k];
            m /= d;
            lu[(size_t)i * n + k] = m;
            for (int j = k + 1; j < n; ++j) lu[(size_t)i * n + j] -= m * lu[(size_t)k * n + j];
        }
    }
    return 0;
}
/* smallmat::luSolve / denseSolve (smallmat.hpp:97-108, 163-174) */
static void lu_solve(const double* lu, const int* piv, int n, double* x) {
    for (int k = 0; k < n; ++k)
        if (piv[k] != k) {
            double t = x[k];
            x[k] = x[piv[k]];
            x[piv[k]] = t;
        }
    for (int i = 1; i < n; ++i)
        for (int j = 0; j < i; ++j) x[i] -= lu[(size_t)i * n + j] * x[j];
    for (int i = n - 1; i >= 0; --i) {
        for (int j = i + 1; j < n; ++j) x[i] -= lu[(size_t)i * n + j] * x[j];
        x[i] /= lu[(size_t)i * n + i];
    }
}
/* smallmat::luSolveMat (smallmat.hpp:111-119), m = n columns */
static void lu_solve_mat(const double* lu, const int* piv, int n, double* B) {
    double col[64];
    for (int c = 0; c < n; ++c) {
        for (int i = 0; i < n; ++i) col[i] = B[i * n + c];
        lu_solve(lu, piv, n, col);
        for (int i = 0; i < n; ++i) B[i * n + c] = col[i];
    }
}
/* smallmat::frobNorm (smallmat.hpp:121-125) */
static double frob(const double* A, int n) {
    double s = 0.0;
    for (int i = 0; i < n * n; ++i) s += A[i] * A[i];
    return sqrt(s);
}

/* csrMatvec (block_csr.cpp:129-137) */
void or_csr_matvec(int rows, int n, const int* ro, const int* ci, const double* v, const double* x, double* y) {
    const size_t nn = (size_t)n * n;
    for (int r = 0; r < rows; ++r) {
        double* yr = y + (size_t)r * n;
        for (int i = 0; i < n; ++i) yr[i] = 0.0;
        for (int k = ro[r]; k < ro[r + 1]; ++k) mv_add(v + (size_t)k * nn, x + (size_t)ci[k] * n, yr, n);
    }
}
static void bsr_matvec(const Bsr* a, const double* x, double* y) { or_csr_matvec(a->rows, a->n, a->ro, a->ci, a->v, x, y); }

/* blockMatvec (block_matrix.cpp:104-119) */
void or_ldu_matvec(int nc, int nf, int n, const int* owner, const int* neigh, const double* diag,
                   const double* upper, const double* lower, const double* x, double* y) {
    const size_t nn = (size_t)n * n;
    for (size_t k = 0; k < (size_t)nc * n; ++k) y[k] = 0.0;
    for (int c = 0; c < nc; ++c) mv_add(diag + c * nn, x + (size_t)c * n, y + (size_t)c * n, n);
    for (int f = 0; f < nf; ++f) {
        mv_add(upper + f * nn, x + (size_t)neigh[f] * n, y + (size_t)owner[f] * n, n);
        mv_add(lower + f * nn, x + (size_t)owner[f] * n, y + (size_t)neigh[f] * n, n);
    }
}

/* ------------------------------------------------------- preconditioners */
typedef struct {
    int kind; /* 0 none, 1 LUSGS, 2 DILU, 3 AMG */
    const Bsr* A;
    double* lu; /* rows * n*n */
    int* piv;   /* rows * n */
    void* amg;
} Precond;

/* factorCsrDiagonals (preconditioner.cpp:9-22) */
static int lusgs_setup(Precond* p, const Bsr* A) {
    const int n = A->n;
    const size_t nn = (size_t)n * n;
    p->A = A;
    p->lu = (double*)xcalloc((size_t)A->rows * nn, sizeof(double));
    p->piv = (int*)xcalloc((size_t)A->rows * n, sizeof(int));
    for (int r = 0; r < A->rows; ++r) {
        const int d = bsr_find(A, r, r);
        char msg[128];
        if (d < 0) {
            snprintf(msg, sizeof msg, "preconditioner setup: missing diagonal in row %d", r);
            return fail(OR_RUNTIME, msg);
        }
        memcpy(p->lu + r * nn, A->v + (size_t)d * nn, nn * sizeof(double));
        if (lu_factor(p->lu + r * nn, p->piv + (size_t)r * n, n)) {
            snprintf(msg, sizeof msg, "preconditioner setup: singular diagonal block in cell %d", r);
            return fail(OR_RUNTIME, msg);
        }
    }
    return OR_OK;
}

/* CsrDiluPrecond ctor (preconditioner.cpp:101-126) */
static int dilu_setup(Precond* p, const Bsr* A) {
    const int n = A->n;
    const size_t nn = (size_t)n * n;
    p->A = A;
    p->lu = (double*)xcalloc((size_t)A->rows * nn, sizeof(double));
    p->piv = (int*)xcalloc((size_t)A->rows * n, sizeof(int));
    double t[64];
    for (int i = 0; i < A->rows; ++i) {
        const int d = bsr_find(A, i, i);
        char msg[128];
        if (d < 0) {
            snprintf(msg, sizeof msg, "DILU setup: missing diagonal in row %d", i);
            return fail(OR_RUNTIME, msg);
        }
        double* dt = p->lu + i * nn;
        memcpy(dt, A->v + (size_t)d * nn, nn * sizeof(double));
        for (int k = A->ro[i]; k < A->ro[i + 1]; ++k) {
            const int j = A->ci[k];
            if (j >= i) break;
            const int kji = bsr_find(A, j, i);
            if (kji < 0) continue;
            memcpy(t, A->v + (size_t)kji * nn, nn * sizeof(double));
            lu_solve_mat(p->lu + j * nn, p->piv + (size_t)j * n, n, t);
            mm_sub(A->v + (size_t)k * nn, t, dt, n);
        }
        if (lu_factor(dt, p->piv + (size_t)i * n, n)) {
            snprintf(msg, sizeof msg, "DILU setup: singular modified diagonal in cell %d", i);
            return fail(OR_RUNTIME, msg);
        }
    }
    return OR_OK;
}

/* CsrLusgsPrecond::apply (preconditioner.cpp:29-57) and CsrDiluPrecond::apply
 * (preconditioner.cpp:128-156) share the sweep structure; only the factored
 * diagonal differs (D vs D~). */
static void sweep_apply(const Precond* p, const double* r, double* z) {
    const Bsr* A = p->A;
    const int n = A->n;
    const size_t nn = (size_t)n * n;
    double tmp[64];
    for (int i = 0; i < A->rows; ++i) {
        double* zi = z + (size_t)i * n;
        for (int q = 0; q < n; ++q) zi[q] = r[(size_t)i * n + q];
        for (int k = A->ro[i]; k < A->ro[i + 1]; ++k) {
            const int j = A->ci[k];
            if (j >= i) break;
            mv_sub(A->v + (size_t)k * nn, z + (size_t)j * n, zi, n);
        }
        lu_solve(p->lu + i * nn, p->piv + (size_t)i * n, n, zi);
    }
    for (int i = A->rows - 1; i >= 0; --i) {
        for (int q = 0; q < n; ++q) tmp[q] = 0.0;
        for (int k = A->ro[i + 1] - 1; k >= A->ro[i]; --k) {
            const int j = A->ci[k];
            if (j <= i) break;
            mv_add(A->v + (size_t)k * nn, z + (size_t)j * n, tmp, n);
        }
        lu_solve(p->lu + i * nn, p->piv + (size_t)i * n, n, tmp);
        double* zi = z + (size_t)i * n;
        for (int q = 0; q < n; ++q) zi[q] -= tmp[q];
    }
}

/* -------------------------------------------------------------------- AMG */
/* pairwiseAggregate (amg.cpp:10-37) */
int or_aggregate(int rows, int n, const int* ro, const int* ci, const double* v, int* agg) {
    const size_t nn = (size_t)n * n;
    double* dn = (double*)xcalloc((size_t)rows, sizeof(double));
    Bsr a = {rows, n, ro[rows], (int*)ro, (int*)ci, (double*)v};
    for (int r = 0; r < rows; ++r) {
        const int d = bsr_find(&a, r, r);
        dn[r] = d >= 0 ? frob(v + (size_t)d * nn, n) : 0.0;
    }
    for (int r = 0; r < rows; ++r) agg[r] = -1;
    int next = 0;
    for (int r = 0; r < rows; ++r) {
        if (agg[r] >= 0) continue;
        int best = -1;
        double bs = -1.0;
        for (int k = ro[r]; k < ro[r + 1]; ++k) {
            const int j = ci[k];
            if (j == r || agg[j] >= 0) continue;
            double prod = dn[r] * dn[j];
            const double denom = sqrt(prod < 1e-300 ? 1e-300 : prod); /* std::max(prod, 1e-300) */
            const double s = frob(v + (size_t)k * nn, n) / denom;
            if (s > bs) {
                bs = s;
                best = j;
            }
        }
        agg[r] = next;
        if (best >= 0) agg[best] = next;
        ++next;
    }
    free(dn);
    return next;
}

/* galerkinCoarse (amg.cpp:39-71): sorted unique coarse columns per coarse row
 * plus the diagonal; values summed for fine rows ascending, k ascending. */
static int int_cmp(const void* a, const void* b) {
    const int x = *(const int*)a, y = *(const int*)b;
    return x < y ? -1 : (x > y ? 1 : 0);
}
static void galerkin(const Bsr* A, const int* agg, int nCoarse, Bsr* C) {
    const int n = A->n;
    const size_t nn = (size_t)n * n;
    /* gather fine rows per coarse row, ascending (rows scanned in order) */
    int* cnt = (int*)xcalloc((size_t)nCoarse + 1, sizeof(int));
    for (int r = 0; r < A->rows; ++r) cnt[agg[r] + 1] += A->ro[r + 1] - A->ro[r] + 0;
    int* cap = (int*)xcalloc((size_t)nCoarse + 1, sizeof(int));
    for (int c = 0; c < nCoarse; ++c) cap[c + 1] = cap[c] + cnt[c + 1] + 1;
    int* buf = (int*)xcalloc((size_t)cap[nCoarse] + 1, sizeof(int));
    int* fillc = (int*)xcalloc((size_t)nCoarse, sizeof(int));
    for (int r = 0; r < A->rows; ++r)
        for (int k = A->ro[r]; k < A->ro[r + 1]; ++k) buf[cap[agg[r]] + fillc[agg[r]]++] = agg[A->ci[k]];
    C->rows = nCoarse;
    C->n = n;
    C->ro = (int*)xcalloc((size_t)nCoarse + 1, sizeof(int));
    for (int c = 0; c < nCoarse; ++c) {
        int* b = buf + cap[c];
        int m = fillc[c];
        b[m++] = c; /* always keep the diagonal */
        qsort(b, (size_t)m, sizeof(int), int_cmp);
        int u = 0;
        for (int q = 0; q < m; ++q)
            if (q == 0 || b[q] != b[q - 1]) b[u++] = b[q];
        fillc[c] = u;
        C->ro[c + 1] = C->ro[c] + u;
    }
    C->nnz = C->ro[nCoarse];
    C->ci = (int*)xcalloc((size_t)C->nnz, sizeof(int));
    C->v = (double*)xcalloc((size_t)C->nnz * nn, sizeof(double));
    for (int c = 0; c < nCoarse; ++c) memcpy(C->ci + C->ro[c], buf + cap[c], (size_t)fillc[c] * sizeof(int));
    for (int r = 0; r < A->rows; ++r) {
        const int cr = agg[r];
        for (int k = A->ro[r]; k < A->ro[r + 1]; ++k) {
            const int cc = agg[A->ci[k]];
            int lo = C->ro[cr], hi = C->ro[cr + 1];
            while (lo < hi) {
                int mid = lo + (hi - lo) / 2;
                if (C->ci[mid] < cc) lo = mid + 1;
                else hi = mid;
            }
            double* dst = C->v + (size_t)lo * nn;
            const double* s = A->v + (size_t)k * nn;
            for (size_t q = 0; q < nn; ++q) dst[q] += s[q];
        }
    }
    free(cnt);
    free(cap);
    free(buf);
    free(fillc);
}

typedef struct {
    int depth;
    int cap;
    Bsr* A;
    int** agg;
    int* ncoarse;
    Precond* smoother;
    double* dense; /* coarsest LU, m x m */
    int* dpiv;
    int m;
    int pre, post;
} Amg;

static void amg_free(Amg* h) {
    if (!h) return;
    for (int l = 0; l < h->depth; ++l) {
        bsr_free(&h->A[l]);
        free(h->agg[l]);
        free(h->smoother[l].lu);
        free(h->smoother[l].piv);
    }
    free(h->A);
    free(h->agg);
    free(h->ncoarse);
    free(h->smoother);
    free(h->dense);
    free(h->dpiv);
    free(h);
}

/* AmgHierarchy ctor (amg.cpp:73-105) */
static int amg_build(const Bsr* fine, int maxLevels, int minCoarse, int pre, int post, Amg** out) {
    Amg* h = (Amg*)xcalloc(1, sizeof(Amg));
    h->cap = maxLevels + 1;
    h->A = (Bsr*)xcalloc((size_t)h->cap, sizeof(Bsr));
    h->agg = (int**)xcalloc((size_t)h->cap, sizeof(int*));
    h->ncoarse = (int*)xcalloc((size_t)h->cap, sizeof(int));
    h->smoother = (Precond*)xcalloc((size_t)h->cap, sizeof(Precond));
    h->pre = pre;
    h->post = post;
    const size_t nn = (size_t)fine->n * fine->n;
    Bsr* A0 = &h->A[0];
    A0->rows = fine->rows;
    A0->n = fine->n;
    A0->nnz = fine->nnz;
    A0->ro = (int*)xcalloc((size_t)fine->rows + 1, sizeof(int));
    A0->ci = (int*)xcalloc((size_t)fine->nnz, sizeof(int));
    A0->v = (double*)xcalloc((size_t)fine->nnz * nn, sizeof(double));
    memcpy(A0->ro, fine->ro, sizeof(int) * ((size_t)fine->rows + 1));
    memcpy(A0->ci, fine->ci, sizeof(int) * (size_t)fine->nnz);
    memcpy(A0->v, fine->v, sizeof(double) * (size_t)fine->nnz * nn);
    h->depth = 1;
    while (h->depth < maxLevels && h->A[h->depth - 1].rows > minCoarse) {
        const int l = h->depth - 1;
        int* agg = (int*)xcalloc((size_t)h->A[l].rows, sizeof(int));
        const int nC = or_aggregate(h->A[l].rows, h->A[l].n, h->A[l].ro, h->A[l].ci, h->A[l].v, agg);
        if (nC == h->A[l].rows) {
            free(agg);
            break;
        }
        h->agg[l] = agg;
        h->ncoarse[l] = nC;
        galerkin(&h->A[l], agg, nC, &h->A[l + 1]);
        h->depth++;
    }
    for (int l = 0; l + 1 < h->depth; ++l) {
        h->smoother[l].kind = 2;
        const int rc = dilu_setup(&h->smoother[l], &h->A[l]);
        if (rc) {
            amg_free(h);
            return rc;
        }
    }
    const Bsr* Ac = &h->A[h->depth - 1];
    const int n = Ac->n;
    h->m = Ac->rows * n;
    h->dense = (double*)xcalloc((size_t)h->m * h->m, sizeof(double));
    h->dpiv = (int*)xcalloc((size_t)h->m, sizeof(int));
    for (int r = 0; r < Ac->rows; ++r)
        for (int k = Ac->ro[r]; k < Ac->ro[r + 1]; ++k) {
            const int c = Ac->ci[k];
            const double* b = Ac->v + (size_t)k * nn;
            for (int i = 0; i < n; ++i)
                for (int j = 0; j < n; ++j) h->dense[(size_t)(r * n + i) * h->m + (c * n + j)] = b[i * n + j];
        }
    if (lu_factor(h->dense, h->dpiv, h->m)) {
        amg_free(h);
        return fail(OR_RUNTIME, "singular coarse-level matrix");
    }
    *out = h;
    return OR_OK;
}

/* AmgHierarchy::vcycle (amg.cpp:111-158) */
static void vcycle(const Amg* h, int l, const double* r, double* z) {
    const Bsr* A = &h->A[l];
    const int n = A->n;
    const size_t N = (size_t)A->rows * n;
    if (l == h->depth - 1) {
        memcpy(z, r, N * sizeof(double));
        lu_solve(h->dense, h->dpiv, h->m, z);
        return;
    }
    for (size_t i = 0; i < N; ++i) z[i] = 0.0;
    double* res = (double*)xcalloc(N, sizeof(double));
    double* corr = (double*)xcalloc(N, sizeof(double));
    for (int s = 0; s < h->pre; ++s) {
        bsr_matvec(A, z, res);
        for (size_t i = 0; i < N; ++i) res[i] = r[i] - res[i];
        sweep_apply(&h->smoother[l], res, corr);
        for (size_t i = 0; i < N; ++i) z[i] += corr[i];
    }
    bsr_matvec(A, z, res);
    for (size_t i = 0; i < N; ++i) res[i] = r[i] - res[i];
    const size_t Nc = (size_t)h->ncoarse[l] * n;
    double* rc = (double*)xcalloc(Nc, sizeof(double));
    double* zc = (double*)xcalloc(Nc, sizeof(double));
    for (int row = 0; row < A->rows; ++row) {
        const int c = h->agg[l][row];
        for (int q = 0; q < n; ++q) rc[(size_t)c * n + q] += res[(size_t)row * n + q];
    }
    vcycle(h, l + 1, rc, zc);
    for (int row = 0; row < A->rows; ++row) {
        const int c = h->agg[l][row];
        for (int q = 0; q < n; ++q) z[(size_t)row * n + q] += zc[(size_t)c * n + q];
    }
    for (int s = 0; s < h->post; ++s) {
        bsr_matvec(A, z, res);
        for (size_t i = 0; i < N; ++i) res[i] = r[i] - res[i];
        sweep_apply(&h->smoother[l], res, corr);
        for (size_t i = 0; i < N; ++i) z[i] += corr[i];
    }
    free(res);
    free(corr);
    free(rc);
    free(zc);
}

/* makeCsrPreconditioner (engine.cpp:21-29) */
static int precond_make(Precond* p, const Bsr* A, const or_cfg* cfg) {
    memset(p, 0, sizeof *p);
    p->kind = cfg->precond;
    p->A = A;
    switch (cfg->precond) {
        case 0: return OR_OK;
        case 1: return lusgs_setup(p, A);
        case 2: return dilu_setup(p, A);
        case 3: {
            Amg* h = NULL;
            const int rc = amg_build(A, cfg->amg_max_levels, cfg->amg_min_coarse_rows, cfg->amg_pre_sweeps,
                                     cfg->amg_post_sweeps, &h);
            p->amg = h;
            return rc;
        }
    }
    return fail(OR_INVALID, "unknown preconditioner kind");
}
static void precond_apply(const Precond* p, const double* r, double* z, size_t N) {
    if (p->kind == 0) memcpy(z, r, N * sizeof(double));
    else if (p->kind == 3) vcycle((const Amg*)p->amg, 0, r, z);
    else sweep_apply(p, r, z);
}
static void precond_free(Precond* p) {
    free(p->lu);
    free(p->piv);
    amg_free((Amg*)p->amg);
    memset(p, 0, sizeof *p);
}

/* ----------------------------------------------------------------- Krylov */
/* defaultDot (krylov.cpp:38-42).  Mode 1 (or_set_dot_mode) re-associates the
 * same sum pairwise over 256-element chunks: a reference-equivalent variant
 * used only to measure how strongly a Krylov history amplifies last-bit
 * differences of the reductions (tests/test_gpu_parity.py). */
static int g_dot_mode = 0;
void or_set_dot_mode(int mode) { g_dot_mode = mode; }
static double dot_pairwise(const double* a, const double* b, size_t n) {
    if (n <= 256) {
        double s = 0.0;
        for (size_t i = 0; i < n; ++i) s += a[i] * b[i];
        return s;
    }
    const size_t h = (n / 2 + 255) / 256 * 256;
    return dot_pairwise(a, b, h) + dot_pairwise(a + h, b + h, n - h);
}
static double dotp(const double* a, const double* b, size_t n) {
    if (g_dot_mode == 1) return dot_pairwise(a, b, n);
    double s = 0.0;
    for (size_t i = 0; i < n; ++i) s += a[i] * b[i];
    return s;
}

/* SolverConfig::validate (krylov.cpp:10-18) */
static int cfg_validate(const or_cfg* c) {
    if (!(c->rel_tol > 0.0) || !(c->abs_tol > 0.0)) return fail(OR_INVALID, "SolverConfig: tolerances must be positive");
    if (c->max_iters < 1) return fail(OR_INVALID, "SolverConfig: maxIters must be >= 1");
    if (c->gmres_restart < 1) return fail(OR_INVALID, "SolverConfig: gmresRestart must be >= 1");
    if (c->amg_max_levels < 1) return fail(OR_INVALID, "SolverConfig: amg.maxLevels must be >= 1");
    if (c->amg_pre_sweeps < 0 || c->amg_post_sweeps < 0) return fail(OR_INVALID, "SolverConfig: amg sweeps must be >= 0");
    return OR_OK;
}

typedef struct {
    double* h;
    int cap, n;
} Hist;
static void hist_push(Hist* hs, double v) {
    if (hs->h && hs->n < hs->cap) hs->h[hs->n] = v;
    hs->n++;
}
static void hist_set_last(Hist* hs, double v) {
    if (hs->n > 0 && hs->h && hs->n - 1 < hs->cap) hs->h[hs->n - 1] = v;
}

/* gmresSolve (krylov.cpp:59-150) */
static void gmres(const Bsr* A, const Precond* M, const double* b, double* x, const or_cfg* cfg, or_report* rep,
                  Hist* hs) {
    const size_t N = (size_t)A->rows * A->n;
    const int m = cfg->gmres_restart;
    double* r = (double*)xcalloc(N, sizeof(double));
    double* w = (double*)xcalloc(N, sizeof(double));
    double* z = (double*)xcalloc(N, sizeof(double));
    bsr_matvec(A, x, r);
    for (size_t i = 0; i < N; ++i) r[i] = b[i] - r[i];
    double beta = sqrt(dotp(r, r, N));
    const double beta0 = beta;
    rep->initial_residual = beta;
    const double tol = cfg->rel_tol * beta > cfg->abs_tol ? cfg->rel_tol * beta : cfg->abs_tol;
    if (beta <= tol) {
        rep->final_residual = beta;
        rep->converged = 1;
        free(r);
        free(w);
        free(z);
        return;
    }
    double* V = (double*)xcalloc((size_t)(m + 1) * N, sizeof(double));
    double* H = (double*)xcalloc((size_t)(m + 1) * m, sizeof(double));
    double* cs = (double*)xcalloc((size_t)m, sizeof(double));
    double* sn = (double*)xcalloc((size_t)m, sizeof(double));
    double* g = (double*)xcalloc((size_t)m + 1, sizeof(double));
    double* y = (double*)xcalloc((size_t)m, sizeof(double));
#define HH(i, j) H[(size_t)(i) * m + (j)]
    int total = 0;
    while (total < cfg->max_iters) {
        for (size_t i = 0; i < N; ++i) V[i] = r[i] / beta;
        for (int i = 0; i <= m; ++i) g[i] = 0.0;
        for (size_t i = 0; i < (size_t)(m + 1) * m; ++i) H[i] = 0.0;
        g[0] = beta;
        int j = 0, happy = 0;
        for (; j < m && total < cfg->max_iters; ++j, ++total) {
            double* vj = V + (size_t)j * N;
            precond_apply(M, vj, z, N);
            bsr_matvec(A, z, w);
            for (int i = 0; i <= j; ++i) {
                const double* vi = V + (size_t)i * N;
                HH(i, j) = dotp(w, vi, N);
                for (size_t q = 0; q < N; ++q) w[q] -= HH(i, j) * vi[q];
            }
            HH(j + 1, j) = sqrt(dotp(w, w, N));
            if (HH(j + 1, j) > 1e-290) {
                double* vn = V + (size_t)(j + 1) * N;
                for (size_t q = 0; q < N; ++q) vn[q] = w[q] / HH(j + 1, j);
            } else {
                happy = 1;
            }
            for (int i = 0; i < j; ++i) {
                const double t = cs[i] * HH(i, j) + sn[i] * HH(i + 1, j);
                HH(i + 1, j) = -sn[i] * HH(i, j) + cs[i] * HH(i + 1, j);
                HH(i, j) = t;
            }
            const double den = hypot(HH(j, j), HH(j + 1, j));
            cs[j] = den > 0.0 ? HH(j, j) / den : 1.0;
            sn[j] = den > 0.0 ? HH(j + 1, j) / den : 0.0;
            HH(j, j) = den;
            HH(j + 1, j) = 0.0;
            g[j + 1] = -sn[j] * g[j];
            g[j] = cs[j] * g[j];
            hist_push(hs, fabs(g[j + 1]) / beta0);
            if (fabs(g[j + 1]) <= tol || happy) {
                ++j;
                ++total;
                break;
            }
        }
        for (int i = j - 1; i >= 0; --i) {
            double s = g[i];
            for (int q = i + 1; q < j; ++q) s -= HH(i, q) * y[q];
            y[i] = s / HH(i, i);
        }
        for (size_t q = 0; q < N; ++q) w[q] = 0.0;
        for (int i = 0; i < j; ++i) {
            const double* vi = V + (size_t)i * N;
            for (size_t q = 0; q < N; ++q) w[q] += y[i] * vi[q];
        }
        precond_apply(M, w, z, N);
        for (size_t q = 0; q < N; ++q) x[q] += z[q];
        bsr_matvec(A, x, r);
        for (size_t i = 0; i < N; ++i) r[i] = b[i] - r[i];
        beta = sqrt(dotp(r, r, N));
        hist_set_last(hs, beta / beta0);
        rep->iterations = total;
        rep->final_residual = beta;
        if (beta <= tol) {
            rep->converged = 1;
            goto done;
        }
        if (happy && beta <= tol * 1.0000001) {
            rep->converged = 1;
            goto done;
        }
    }
    rep->iterations = total;
    rep->converged = rep->final_residual <= tol;
done:
#undef HH
    free(r);
    free(w);
    free(z);
    free(V);
    free(H);
    free(cs);
    free(sn);
    free(g);
    free(y);
}

/* bicgstabSolve (krylov.cpp:152-214); returns OR_RUNTIME on breakdown */
static int bicgstab(const Bsr* A, const Precond* M, const double* b, double* x, const or_cfg* cfg, or_report* rep,
                    Hist* hs) {
    const size_t N = (size_t)A->rows * A->n;
    double* r = (double*)xcalloc(N, sizeof(double));
    double* rh = (double*)xcalloc(N, sizeof(double));
    double* p = (double*)xcalloc(N, sizeof(double));
    double* v = (double*)xcalloc(N, sizeof(double));
    double* s = (double*)xcalloc(N, sizeof(double));
    double* t = (double*)xcalloc(N, sizeof(double));
    double* ph = (double*)xcalloc(N, sizeof(double));
    double* sh = (double*)xcalloc(N, sizeof(double));
    int rc = OR_OK;
    bsr_matvec(A, x, r);
    for (size_t i = 0; i < N; ++i) r[i] = b[i] - r[i];
    const double beta0 = sqrt(dotp(r, r, N));
    rep->initial_residual = beta0;
    const double tol = cfg->rel_tol * beta0 > cfg->abs_tol ? cfg->rel_tol * beta0 : cfg->abs_tol;
    if (beta0 <= tol) {
        rep->final_residual = beta0;
        rep->converged = 1;
        goto out;
    }
    memcpy(rh, r, N * sizeof(double));
    double rhoPrev = 1.0, alpha = 1.0, omega = 1.0;
    for (int it = 0; it < cfg->max_iters; ++it) {
        const double rho = dotp(rh, r, N);
        if (fabs(rho) < 1e-30) {
            rep->breakdown = 1;
            break;
        }
        if (it == 0) {
            memcpy(p, r, N * sizeof(double));
        } else {
            const double bf = (rho / rhoPrev) * (alpha / omega);
            for (size_t i = 0; i < N; ++i) p[i] = r[i] + bf * (p[i] - omega * v[i]);
        }
        precond_apply(M, p, ph, N);
        bsr_matvec(A, ph, v);
        const double rv = dotp(rh, v, N);
        if (fabs(rv) < 1e-300) {
            rep->breakdown = 1;
            break;
        }
        alpha = rho / rv;
        for (size_t i = 0; i < N; ++i) s[i] = r[i] - alpha * v[i];
        const double ns = sqrt(dotp(s, s, N));
        if (ns <= tol) {
            for (size_t i = 0; i < N; ++i) x[i] += alpha * ph[i];
            rep->iterations = it + 1;
            hist_push(hs, ns / beta0);
            break;
        }
        precond_apply(M, s, sh, N);
        bsr_matvec(A, sh, t);
        const double tt = dotp(t, t, N);
        omega = tt > 0.0 ? dotp(t, s, N) / tt : 0.0;
        for (size_t i = 0; i < N; ++i) x[i] += alpha * ph[i] + omega * sh[i];
        for (size_t i = 0; i < N; ++i) r[i] = s[i] - omega * t[i];
        rep->iterations = it + 1;
        if (fabs(omega) < 1e-30) {
            rep->breakdown = 1;
            break;
        }
        rhoPrev = rho;
        const double nr = sqrt(dotp(r, r, N));
        hist_push(hs, nr / beta0);
        if (nr <= tol) break;
    }
    bsr_matvec(A, x, r);
    for (size_t i = 0; i < N; ++i) r[i] = b[i] - r[i];
    rep->final_residual = sqrt(dotp(r, r, N));
    rep->converged = rep->final_residual <= tol;
    if (rep->converged) rep->breakdown = 0;
    if (rep->breakdown) {
        char msg[160];
        snprintf(msg, sizeof msg, "BiCGStab breakdown at iteration %d, residual %f", rep->iterations,
                 rep->final_residual);
        rc = fail(OR_RUNTIME, msg);
    }
out:
    free(r);
    free(rh);
    free(p);
    free(v);
    free(s);
    free(t);
    free(ph);
    free(sh);
    return rc;
}

int or_precond_apply(int nc, int nf, int n, const int* owner, const int* neigh, const double* diag,
                     const double* upper, const double* lower, const or_cfg* cfg, const double* r, double* z) {
    Bsr A;
    bsr_from_ldu(nc, nf, n, owner, neigh, diag, upper, lower, &A);
    Precond M;
    int rc = precond_make(&M, &A, cfg);
    if (rc == OR_OK) precond_apply(&M, r, z, (size_t)nc * n);
    precond_free(&M);
    bsr_free(&A);
    return rc;
}

int or_solve(int nc, int nf, int n, const int* owner, const int* neigh, const double* diag, const double* upper,
             const double* lower, const double* b, const double* x0, const or_cfg* cfg, double* x, or_report* rep,
             double* hist, int hist_cap, int* hist_n) {
    memset(rep, 0, sizeof *rep);
    Hist hs = {hist, hist_cap, 0};
    Bsr A;
    bsr_from_ldu(nc, nf, n, owner, neigh, diag, upper, lower, &A);
    Precond M;
    int rc = precond_make(&M, &A, cfg);
    if (rc == OR_OK) rc = cfg_validate(cfg);
    if (rc == OR_OK) {
        if (M.kind == 3) rep->amg_levels = ((Amg*)M.amg)->depth;
        memcpy(x, x0, sizeof(double) * (size_t)nc * n);
        if (cfg->method == 0) gmres(&A, &M, b, x, cfg, rep, &hs);
        else rc = bicgstab(&A, &M, b, x, cfg, rep, &hs);
    }
    if (hist_n) *hist_n = hs.n;
    precond_free(&M);
    bsr_free(&A);
    return rc;
}

void* or_amg_build(int nc, int nf, int n, const int* owner, const int* neigh, const double* diag,
                   const double* upper, const double* lower, int max_levels, int min_coarse_rows) {
    Bsr A;
    bsr_from_ldu(nc, nf, n, owner, neigh, diag, upper, lower, &A);
    Amg* h = NULL;
    const int rc = amg_build(&A, max_levels, min_coarse_rows, 1, 1, &h);
    bsr_free(&A);
    return rc == OR_OK ? h : NULL;
}
int or_amg_depth(void* h) { return ((Amg*)h)->depth; }
void or_amg_level_sizes(void* hv, int l, int* rows, int* nnz, int* agg_len) {
    Amg* h = (Amg*)hv;
    *rows = h->A[l].rows;
    *nnz = h->A[l].nnz;
    *agg_len = h->agg[l] ? h->A[l].rows : 0;
}
void or_amg_level_get(void* hv, int l, int* ro, int* ci, double* v, int* agg) {
    Amg* h = (Amg*)hv;
    const Bsr* A = &h->A[l];
    memcpy(ro, A->ro, sizeof(int) * ((size_t)A->rows + 1));
    memcpy(ci, A->ci, sizeof(int) * (size_t)A->nnz);
    memcpy(v, A->v, sizeof(double) * (size_t)A->nnz * A->n * A->n);
    if (agg && h->agg[l]) memcpy(agg, h->agg[l], sizeof(int) * (size_t)A->rows);
}
void or_amg_free(void* h) { amg_free((Amg*)h); }

/* ------------------------------------------------------------- partition */
/* rcbRecurse (partition.cpp:21-53) */
static const double* g_cen;
static int g_axis;
static int rcb_cmp(const void* a, const void* b) {
    const int x = *(const int*)a, y = *(const int*)b;
    const double cx = g_cen[3 * x + g_axis], cy = g_cen[3 * y + g_axis];
    if (cx != cy) return cx < cy ? -1 : 1;
    return x < y ? -1 : (x > y ? 1 : 0);
}
static void rcb(int* cells, int count, int r0, int r1, const double* cen, int* c2r) {
    const int nR = r1 - r0;
    if (nR == 1) {
        for (int i = 0; i < count; ++i) c2r[cells[i]] = r0;
        return;
    }
    double lo[3] = {1e300, 1e300, 1e300}, hi[3] = {-1e300, -1e300, -1e300};
    for (int i = 0; i < count; ++i)
        for (int a = 0; a < 3; ++a) {
            const double v = cen[3 * cells[i] + a];
            if (v < lo[a]) lo[a] = v;
            if (v > hi[a]) hi[a] = v;
        }
    int axis = 0;
    for (int a = 1; a < 3; ++a)
        if (hi[a] - lo[a] > hi[axis] - lo[axis] + 1e-14) axis = a;
    g_cen = cen;
    g_axis = axis;
    qsort(cells, (size_t)count, sizeof(int), rcb_cmp);
    const int nLeft = nR / 2;
    long long cl = ((long long)count * nLeft + nR / 2) / nR;
    if (cl < nLeft) cl = nLeft;
    if (cl > count - (nR - nLeft)) cl = count - (nR - nLeft);
    rcb(cells, (int)cl, r0, r0 + nLeft, cen, c2r);
    rcb(cells + cl, count - (int)cl, r0 + nLeft, r1, cen, c2r);
}

/* decompose (partition.cpp:57-85) */
int or_decompose(int nc, const double* cen, int nRanks, int* c2r, int* rro, int* o2n) {
    if (nRanks < 1 || nRanks > nc) return fail(OR_INVALID, "decompose: need 1 <= nRanks <= nCells");
    int* all = (int*)xcalloc((size_t)nc, sizeof(int));
    for (int c = 0; c < nc; ++c) all[c] = c;
    rcb(all, nc, 0, nRanks, cen, c2r);
    for (int r = 0; r <= nRanks; ++r) rro[r] = 0;
    for (int c = 0; c < nc; ++c) rro[c2r[c] + 1]++;
    for (int r = 0; r < nRanks; ++r) rro[r + 1] += rro[r];
    int* next = (int*)xcalloc((size_t)nRanks, sizeof(int));
    for (int r = 0; r < nRanks; ++r) next[r] = rro[r];
    for (int c = 0; c < nc; ++c) o2n[c] = next[c2r[c]]++;
    free(all);
    free(next);
    return OR_OK;
}
