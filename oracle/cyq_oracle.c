/* TEST INFRASTRUCTURE ONLY — the CPU checker for the KKT factor+solve path.
 *
 * Plain-C restatement of the reference algorithm (arXiv 2512.09058,
 * "Cyqlone"), one instance at a time, scalar (the reference's vlen = 1),
 * row-major dense blocks. Each function cites the reference file:line it
 * restates (paths relative to /root/reference/proj). The loop orders follow
 * the reference's lane loops with the lane dimension removed, so for vlen = 1
 * the arithmetic sequence is the reference's own.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's CPU legs use this
 * library; the product (paper_2512_09058_b200/) never links it.
 * Pinned against oracle/_ref/libcyqref.so (the reference built from its own
 * sources) and against tests/golden/ fixtures generated from it.
 */
#define _POSIX_C_SOURCE 200809L
#include "oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

typedef int64_t ix;

/* ---- FMA counter: batla::flops (kernels.cpp:8-15) ---------------------- */
static _Thread_local uint64_t g_fma;

/* ---- small dense kernels, row-major with leading dimension -------------- */
#define AT(a, ld, r, c) ((a)[(r) * (ld) + (c)])

static const double pivot_floor_rel = 1e-14; /* kernels.cpp:18 */

/* potrf (kernels.cpp:32-58): in-place lower Cholesky. Returns the failing
 * pivot index, or -1. */
static ix potrf(double *a, ix n, ix lda) {
    double dmax = 0; /* diag_max, kernels.cpp:21-29 */
    for (ix d = 0; d < n; ++d)
        if (fabs(AT(a, lda, d, d)) > dmax)
            dmax = fabs(AT(a, lda, d, d));
    for (ix k = 0; k < n; ++k) {
        double p = AT(a, lda, k, k);
        if (!(p > pivot_floor_rel * dmax) || !isfinite(p))
            return k;
        AT(a, lda, k, k) = sqrt(p);
        for (ix i = k + 1; i < n; ++i)
            AT(a, lda, i, k) /= AT(a, lda, k, k);
        for (ix j = k + 1; j < n; ++j)
            for (ix i = j; i < n; ++i)
                AT(a, lda, i, j) -= AT(a, lda, i, k) * AT(a, lda, j, k);
    }
    g_fma += (uint64_t)(n * (n + 1) * (n + 2) / 6);
    return -1;
}

enum { RLT, LL, LLT }; /* TrsmMode (kernels.hpp:57-61) */

/* trsm (kernels.cpp:95-156); b is rows x cols. */
static void trsm(double *b, ix rows, ix cols, ix ldb, const double *l,
                 ix ldl, int mode) {
    ix n = (mode == RLT) ? cols : rows;
    if (mode == RLT) {
        for (ix c = 0; c < n; ++c) {
            for (ix k = 0; k < c; ++k)
                for (ix r = 0; r < rows; ++r)
                    AT(b, ldb, r, c) -= AT(b, ldb, r, k) * AT(l, ldl, c, k);
            for (ix r = 0; r < rows; ++r)
                AT(b, ldb, r, c) /= AT(l, ldl, c, c);
        }
    } else if (mode == LL) {
        for (ix r = 0; r < n; ++r) {
            for (ix k = 0; k < r; ++k)
                for (ix c = 0; c < cols; ++c)
                    AT(b, ldb, r, c) -= AT(l, ldl, r, k) * AT(b, ldb, k, c);
            for (ix c = 0; c < cols; ++c)
                AT(b, ldb, r, c) /= AT(l, ldl, r, r);
        }
    } else {
        for (ix r = n; r-- > 0;) {
            for (ix k = r + 1; k < n; ++k)
                for (ix c = 0; c < cols; ++c)
                    AT(b, ldb, r, c) -= AT(l, ldl, k, r) * AT(b, ldb, k, c);
            for (ix c = 0; c < cols; ++c)
                AT(b, ldb, r, c) /= AT(l, ldl, r, r);
        }
    }
    ix other = (mode == RLT) ? rows : cols;
    g_fma += (uint64_t)(other * n * (n + 1) / 2);
}

/* syrk (kernels.cpp:158-168): C += alpha A A^T, lower; A is n x k. */
static void syrk(double *c, ix n, ix ldc, const double *a, ix k, ix lda,
                 double al) {
    for (ix kk = 0; kk < k; ++kk)
        for (ix j = 0; j < n; ++j)
            for (ix i = j; i < n; ++i)
                AT(c, ldc, i, j) += al * AT(a, lda, i, kk) * AT(a, lda, j, kk);
    g_fma += (uint64_t)(k * n * (n + 1) / 2);
}

/* gemm (kernels.cpp:170-188): C(m x n) += alpha op(A) op(B). */
static void gemm(double *c, ix m, ix n, ix ldc, const double *a, ix lda,
                 int ta, const double *b, ix ldb, int tb, ix ka, double al) {
    for (ix k = 0; k < ka; ++k)
        for (ix j = 0; j < n; ++j)
            for (ix i = 0; i < m; ++i) {
                double av = ta ? AT(a, lda, k, i) : AT(a, lda, i, k);
                double bv = tb ? AT(b, ldb, j, k) : AT(b, ldb, k, j);
                AT(c, ldc, i, j) += al * av * bv;
            }
    g_fma += (uint64_t)(m * n * ka);
}

enum { TR_RL, TR_LU, TR_LUT, TR_LL, TR_LLT }; /* TrmmMode kernels.hpp:73-79 */

/* trmm (kernels.cpp:190-244): X = alpha * (triangular product), out of
 * place. a is ar x ac (general), t is n x n. */
static void trmm(double *x, ix ldx, const double *a, ix ar, ix ac, ix lda,
                 const double *t, ix n, ix ldt, int mode, double al) {
    ix xr = (mode == TR_RL) ? ar : n, xc = (mode == TR_RL) ? n : ac;
    for (ix i = 0; i < xr; ++i)
        for (ix j = 0; j < xc; ++j)
            AT(x, ldx, i, j) = 0;
    uint64_t cnt = 0;
    switch (mode) {
    case TR_RL:
        for (ix j = 0; j < n; ++j)
            for (ix k = j; k < n; ++k)
                for (ix i = 0; i < ar; ++i)
                    AT(x, ldx, i, j) += al * AT(a, lda, i, k) * AT(t, ldt, k, j);
        cnt = (uint64_t)(ar * n * (n + 1) / 2);
        break;
    case TR_LU:
        for (ix i = 0; i < n; ++i)
            for (ix k = i; k < n; ++k)
                for (ix j = 0; j < ac; ++j)
                    AT(x, ldx, i, j) += al * AT(t, ldt, i, k) * AT(a, lda, k, j);
        cnt = (uint64_t)(ac * n * (n + 1) / 2);
        break;
    case TR_LUT:
        for (ix i = 0; i < n; ++i)
            for (ix k = 0; k <= i; ++k)
                for (ix j = 0; j < ac; ++j)
                    AT(x, ldx, i, j) += al * AT(t, ldt, k, i) * AT(a, lda, k, j);
        cnt = (uint64_t)(ac * n * (n + 1) / 2);
        break;
    case TR_LL:
        for (ix i = 0; i < n; ++i)
            for (ix k = 0; k <= i; ++k)
                for (ix j = 0; j < ac; ++j)
                    AT(x, ldx, i, j) += al * AT(t, ldt, i, k) * AT(a, lda, k, j);
        cnt = (uint64_t)(ac * n * (n + 1) / 2);
        break;
    case TR_LLT:
        for (ix i = 0; i < n; ++i)
            for (ix k = i; k < n; ++k)
                for (ix j = 0; j < ac; ++j)
                    AT(x, ldx, i, j) += al * AT(t, ldt, k, i) * AT(a, lda, k, j);
        cnt = (uint64_t)(ac * n * (n + 1) / 2);
        break;
    }
    g_fma += cnt;
}

/* trtri (kernels.cpp:246-271): in-place inverse of a lower triangle. */
static void trtri(double *l, ix n, ix ld) {
    for (ix j = 0; j < n; ++j) {
        AT(l, ld, j, j) = 1.0 / AT(l, ld, j, j);
        for (ix i = j + 1; i < n; ++i) {
            double s = 0;
            for (ix k = j; k < i; ++k)
                s += AT(l, ld, i, k) * AT(l, ld, k, j);
            AT(l, ld, i, j) = -s / AT(l, ld, i, i);
        }
    }
    g_fma += (uint64_t)(n * (n + 1) * (n + 2) / 6);
}

/* trsyrk (kernels.cpp:273-289): lower of T T^T, T upper. */
static void trsyrk(double *c, const double *t, ix n) {
    uint64_t cnt = 0;
    for (ix j = 0; j < n; ++j)
        for (ix i = j; i < n; ++i) {
            AT(c, n, i, j) = 0;
            for (ix k = i; k < n; ++k)
                AT(c, n, i, j) += AT(t, n, i, k) * AT(t, n, j, k);
            cnt += (uint64_t)(n - i);
        }
    g_fma += cnt;
}

static void add_scaled(double *dst, const double *src, ix cnt, double al) {
    for (ix i = 0; i < cnt; ++i)
        dst[i] += al * src[i];
    g_fma += (uint64_t)cnt;
}

/* mv (block_tridiag.cpp:18-27): y += alpha op(A) x, A is n x n here. */
static void mv(const double *a, ix n, int trans, const double *x, double *y,
               double al) {
    for (ix i = 0; i < n; ++i) {
        double s = 0;
        for (ix k = 0; k < n; ++k)
            s += (trans ? AT(a, n, k, i) : AT(a, n, i, k)) * x[k];
        y[i] += al * s;
    }
}

/* ---- problem access with pad_problem semantics (kkt_factor.cpp:27-47) -- */
typedef struct {
    ix N, Np, nx, nu, nux, P, n;
    const oc_ocp *p;
    ix b; /* instance */
} prob;

static const double *stage_mat(const prob *q, const double *base, ix j,
                               ix rows, ix cols, ix count) {
    return base + (q->b * count + j) * rows * cols;
}
/* entry of A_j, B_j, R_j, S_j, Q_j; padding stages: R = Q = I, A = B = S = 0 */
static double gA(const prob *q, ix j, ix r, ix c) {
    return j < q->N ? stage_mat(q, q->p->A, j, q->nx, q->nx, q->N)[r * q->nx + c] : 0;
}
static double gB(const prob *q, ix j, ix r, ix c) {
    return j < q->N ? stage_mat(q, q->p->B, j, q->nx, q->nu, q->N)[r * q->nu + c] : 0;
}
static double gR(const prob *q, ix j, ix r, ix c) {
    return j < q->N ? stage_mat(q, q->p->R, j, q->nu, q->nu, q->N)[r * q->nu + c]
                    : (r == c);
}
static double gS(const prob *q, ix j, ix r, ix c) {
    return j < q->N ? stage_mat(q, q->p->S, j, q->nu, q->nx, q->N)[r * q->nx + c] : 0;
}
static double gQ(const prob *q, ix j, ix r, ix c) {
    return j <= q->N ? stage_mat(q, q->p->Q, j, q->nx, q->nx, q->N + 1)[r * q->nx + c]
                     : (r == c);
}

/* Partition (kkt_solver.hpp:31-43) */
static ix stage_of(const prob *q, ix c, ix s) {
    ix j = q->n * c - s;
    return ((j % q->Np) + q->Np) % q->Np;
}
static ix x_index_of(const prob *q, ix c, ix s) {
    ix j = stage_of(q, c, s);
    return j == 0 ? q->Np : j;
}

/* ---- factor ------------------------------------------------------------ */
typedef struct {
    prob q;
    double *H, *BA, *BAt;             /* [s][c] nux^2, nx*nux, nux*nx */
    double *LH, *LB, *Acl;            /* [s][c] */
    double *LA, *T, *Mfwd, *Mbwd, *W; /* [c] nx^2 */
    double *Md, *Ks;                  /* Schur diag / subdiag [c] nx^2 */
    ix levels;                        /* log2 P */
    double *crL[32], *crU[32], *crY[32], *Mlvl[33], *Klvl[33];
    double *Lbase;
} ofac;

static void *zalloc(size_t n) { return calloc(n ? n : 1, sizeof(double)); }

static void ofac_free(ofac *f) {
    free(f->H); free(f->BA); free(f->BAt); free(f->LH); free(f->LB);
    free(f->Acl); free(f->LA); free(f->T); free(f->Mfwd); free(f->Mbwd);
    free(f->W); free(f->Md); free(f->Ks); free(f->Lbase);
    for (int l = 0; l < 32; ++l) {
        free(f->crL[l]); free(f->crU[l]); free(f->crY[l]);
    }
    for (int l = 0; l < 33; ++l) {
        free(f->Mlvl[l]); free(f->Klvl[l]);
    }
    memset(f, 0, sizeof(*f));
}

#define BLK(arr, s, c, sz) ((arr) + ((s) * q->P + (c)) * (sz))

/* pack_columns (kkt_factor.cpp:54-107) */
static void pack_columns(ofac *f) {
    const prob *q = &f->q;
    ix nx = q->nx, nu = q->nu, nux = q->nux;
    for (ix s = 0; s < q->n; ++s)
        for (ix c = 0; c < q->P; ++c) {
            ix j = stage_of(q, c, s), xi = x_index_of(q, c, s);
            double *H = BLK(f->H, s, c, nux * nux);
            double *BA = BLK(f->BA, s, c, nx * nux);
            double *BAt = BLK(f->BAt, s, c, nux * nx);
            for (ix a = 0; a < nu; ++a)
                for (ix b = 0; b <= a; ++b)
                    H[a * nux + b] = gR(q, j, a, b);
            for (ix a = 0; a < nx; ++a)
                for (ix b = 0; b <= a; ++b)
                    H[(nu + a) * nux + nu + b] = gQ(q, xi, a, b);
            if (j != 0)
                for (ix a = 0; a < nx; ++a)
                    for (ix b = 0; b < nu; ++b)
                        H[(nu + a) * nux + b] = gS(q, j, b, a);
            for (ix a = 0; a < nx; ++a)
                for (ix b = 0; b < nu; ++b) {
                    BA[a * nux + b] = gB(q, j, a, b);
                    BAt[b * nx + a] = gB(q, j, a, b);
                }
            if (j != 0)
                for (ix a = 0; a < nx; ++a)
                    for (ix b = 0; b < nx; ++b) {
                        BA[a * nux + nu + b] = gA(q, j, a, b);
                        BAt[(nu + b) * nx + a] = gA(q, j, a, b);
                    }
        }
}

/* factor_lanes for one column (kkt_factor.cpp:109-188). Returns the failing
 * (stage, pivot) through *fs / *fp, or 0 on success. */
static int factor_column(ofac *f, ix c, ix *fs, ix *fp) {
    const prob *q = &f->q;
    ix nx = q->nx, nu = q->nu, nux = q->nux, n = q->n;
    double *hat = zalloc((size_t)(nx * nux)), *hat2 = zalloc((size_t)(nx * nux));
    double *V = zalloc((size_t)(nux * nx));
    memcpy(hat, BLK(f->BA, 0, c, nx * nux), sizeof(double) * (size_t)(nx * nux));
    int rc = 0;
    for (ix s = 0; s < n; ++s) {
        double *lh = BLK(f->LH, s, c, nux * nux);
        memcpy(lh, BLK(f->H, s, c, nux * nux), sizeof(double) * (size_t)(nux * nux));
        if (s > 0)
            syrk(lh, nux, nux, V, nx, nx, +1);
        ix k = potrf(lh, nux, nux);
        if (k >= 0) {
            *fs = s;
            *fp = k;
            rc = 2;
            break;
        }
        for (ix r = 0; r < nux; ++r) /* LH is lower_triangular */
            for (ix cc = r + 1; cc < nux; ++cc)
                lh[r * nux + cc] = 0;
        const double *l_r = lh, *l_s = lh + nu * nux, *l_q = lh + nu * nux + nu;
        double *lb = BLK(f->LB, s, c, nx * nu);
        for (ix a = 0; a < nx; ++a)
            for (ix b = 0; b < nu; ++b)
                lb[a * nu + b] = hat[a * nux + b];
        trsm(lb, nx, nu, nu, l_r, nux, RLT);
        double *acl = BLK(f->Acl, s, c, nx * nx);
        for (ix a = 0; a < nx; ++a)
            for (ix b = 0; b < nx; ++b)
                acl[a * nx + b] = hat[a * nux + nu + b];
        gemm(acl, nx, nx, nx, lb, nu, 0, l_s, nux, 1, nu, -1);
        if (s + 1 < n) {
            memset(hat2, 0, sizeof(double) * (size_t)(nx * nux));
            gemm(hat2, nx, nux, nux, acl, nx, 0, BLK(f->BA, s + 1, c, nx * nux),
                 nux, 0, nx, +1);
            double *tmp = hat; hat = hat2; hat2 = tmp;
            trmm(V, nx, BLK(f->BAt, s + 1, c, nux * nx), nux, nx, nx, l_q, nx,
                 nux, TR_RL, 1);
        } else {
            double *la = f->LA + c * nx * nx;
            memcpy(la, acl, sizeof(double) * (size_t)(nx * nx));
            trsm(la, nx, nx, nx, l_q, nux, RLT);
        }
    }
    if (rc == 0) {
        /* Schur contributions (kkt_factor.cpp:163-185) */
        double *li = zalloc((size_t)(nx * nx)), *lat = zalloc((size_t)(nx * nx));
        const double *lq = BLK(f->LH, n - 1, c, nux * nux) + nu * nux + nu;
        for (ix a = 0; a < nx; ++a)
            for (ix b = 0; b <= a; ++b)
                li[a * nx + b] = lq[a * nux + b];
        trtri(li, nx, nx);
        double *t = f->T + c * nx * nx;
        for (ix a = 0; a < nx; ++a)
            for (ix b = 0; b < nx; ++b)
                t[a * nx + b] = li[b * nx + a];
        trsyrk(f->Mbwd + c * nx * nx, t, nx);
        const double *la = f->LA + c * nx * nx;
        for (ix a = 0; a < nx; ++a)
            for (ix b = 0; b < nx; ++b)
                lat[a * nx + b] = la[b * nx + a];
        trmm(f->W + c * nx * nx, nx, lat, nx, nx, nx, t, nx, nx, TR_LU, 1);
        double *mf = f->Mfwd + c * nx * nx;
        memset(mf, 0, sizeof(double) * (size_t)(nx * nx));
        for (ix s = 0; s < n; ++s)
            syrk(mf, nx, nx, BLK(f->LB, s, c, nx * nu), nu, nu, +1);
        syrk(mf, nx, nx, la, nx, nx, +1);
        free(li);
        free(lat);
    }
    free(hat);
    free(hat2);
    free(V);
    return rc;
}

/* assemble_schur (kkt_factor.cpp:194-212) */
static void assemble_schur(ofac *f) {
    const prob *q = &f->q;
    ix P = q->P, nx = q->nx, nn = nx * nx;
    for (ix c = 0; c < P; ++c) {
        ix prev = (c - 1 + P) % P;
        add_scaled(f->Md + c * nn, f->Mfwd + c * nn, nn, 1);
        add_scaled(f->Md + prev * nn, f->Mbwd + c * nn, nn, 1);
        if (c > 0)
            for (ix a = 0; a < nx; ++a)
                for (ix b = 0; b < nx; ++b)
                    f->Ks[prev * nn + a * nx + b] = -f->W[c * nn + b * nx + a];
    }
}

/* cr_factor / cr_level / cr_factor_base, non-circular
 * (block_tridiag.cpp:126-238). Returns 0, or 2 with lvl, idx, piv set. */
static int cr_factor(ofac *f, ix *lvl, ix *idx, ix *piv) {
    const prob *q = &f->q;
    ix P = q->P, n = q->nx, nn = n * n;
    ix lg = 0;
    while (((ix)1 << lg) < P)
        ++lg;
    f->levels = lg;
    f->Mlvl[0] = zalloc((size_t)(P * nn));
    f->Klvl[0] = zalloc((size_t)(P * nn));
    memcpy(f->Mlvl[0], f->Md, sizeof(double) * (size_t)(P * nn));
    memcpy(f->Klvl[0], f->Ks, sizeof(double) * (size_t)(P * nn));
    ix s = P;
    for (ix l = 0; l < lg; ++l, s /= 2) {
        ix half = s / 2;
        double *Ml = f->Mlvl[l], *Kl = f->Klvl[l];
        double *L = f->crL[l] = zalloc((size_t)(half * nn));
        double *U = f->crU[l] = zalloc((size_t)(half * nn));
        double *Y = f->crY[l] = zalloc((size_t)(half * nn));
        double *M2 = f->Mlvl[l + 1] = zalloc((size_t)(half * nn));
        double *K2 = f->Klvl[l + 1] = zalloc((size_t)(half * nn));
        for (ix mm = 0; mm < half; ++mm) {
            ix k = 2 * mm + 1;
            double *Lm = L + mm * nn;
            for (ix a = 0; a < n; ++a) /* copy of a symmetric_lower block */
                for (ix b = 0; b <= a; ++b)
                    Lm[a * n + b] = Ml[k * nn + a * n + b];
            ix pk = potrf(Lm, n, n);
            if (pk >= 0) {
                *lvl = l; *idx = k; *piv = pk;
                return 2;
            }
            double *Um = U + mm * nn;
            for (ix a = 0; a < n; ++a)
                for (ix b = 0; b < n; ++b)
                    Um[a * n + b] = Kl[(k - 1) * nn + b * n + a];
            trsm(Um, n, n, n, Lm, n, RLT);
            if (k < s - 1) {
                double *Ym = Y + mm * nn;
                memcpy(Ym, Kl + k * nn, sizeof(double) * (size_t)nn);
                trsm(Ym, n, n, n, Lm, n, RLT);
            }
        }
        for (ix mm = 0; mm < half; ++mm) {
            double *Md = M2 + mm * nn;
            for (ix a = 0; a < n; ++a)
                for (ix b = 0; b <= a; ++b)
                    Md[a * n + b] = Ml[2 * mm * nn + a * n + b];
            syrk(Md, n, n, U + mm * nn, n, n, -1);
            if (mm > 0)
                syrk(Md, n, n, Y + (mm - 1) * nn, n, n, -1);
            if (mm < half - 1)
                gemm(K2 + mm * nn, n, n, n, Y + mm * nn, n, 0, U + mm * nn, n,
                     1, n, -1);
        }
    }
    f->Lbase = zalloc((size_t)nn);
    for (ix a = 0; a < n; ++a)
        for (ix b = 0; b <= a; ++b)
            f->Lbase[a * n + b] = f->Mlvl[lg][a * n + b];
    ix pk = potrf(f->Lbase, n, n);
    if (pk >= 0) {
        *lvl = lg; *idx = 0; *piv = pk;
        return 2;
    }
    return 0;
}

static void set_st(oc_status *st, int code, int kind, ix inst, ix col,
                   ix stage, ix piv) {
    if (!st)
        return;
    st->code = code; st->kind = kind; st->instance = inst;
    st->column_or_level = col; st->stage = stage; st->pivot = piv;
}

/* factor (kkt_factor.cpp:251-313) for instance b of the batch. */
static int do_factor(const oc_dims *d, const oc_ocp *p, ix b, ofac *f,
                     oc_status *st) {
    memset(f, 0, sizeof(*f));
    ix P = d->P;
    if (P <= 0 || (P & (P - 1)) != 0) {
        set_st(st, 1, 0, b, 0, 0, 0);
        return 1;
    }
    prob *q = &f->q;
    q->N = d->N; q->nx = d->nx; q->nu = d->nu; q->nux = d->nx + d->nu;
    q->P = P; q->Np = P * ((d->N + P - 1) / P); q->n = q->Np / P;
    q->p = p; q->b = b;
    ix nx = q->nx, nux = q->nux, n = q->n, nn = nx * nx;
    f->H = zalloc((size_t)(n * P * nux * nux));
    f->BA = zalloc((size_t)(n * P * nx * nux));
    f->BAt = zalloc((size_t)(n * P * nux * nx));
    f->LH = zalloc((size_t)(n * P * nux * nux));
    f->LB = zalloc((size_t)(n * P * nx * q->nu));
    f->Acl = zalloc((size_t)(n * P * nn));
    f->LA = zalloc((size_t)(P * nn)); f->T = zalloc((size_t)(P * nn));
    f->Mfwd = zalloc((size_t)(P * nn)); f->Mbwd = zalloc((size_t)(P * nn));
    f->W = zalloc((size_t)(P * nn)); f->Md = zalloc((size_t)(P * nn));
    f->Ks = zalloc((size_t)(P * nn));
    pack_columns(f);
    for (ix c = 0; c < P; ++c) {
        ix fs = 0, fp = 0;
        if (factor_column(f, c, &fs, &fp)) {
            set_st(st, 2, 0, b, c, fs, fp);
            return 2;
        }
    }
    assemble_schur(f);
    ix lvl = 0, idx = 0, piv = 0;
    if (cr_factor(f, &lvl, &idx, &piv)) {
        set_st(st, 2, 1, b, lvl, idx, piv);
        return 2;
    }
    set_st(st, 0, 0, b, 0, 0, 0);
    return 0;
}

/* CRFactor::forward / backward (block_tridiag.cpp:252-333), non-circular. */
static void cr_forward(const ofac *f, double *x) {
    ix P = f->q.P, n = f->q.nx, nn = n * n, s = P;
    for (ix l = 0; l < f->levels; ++l, s /= 2) {
        ix half = s / 2, stride = P / s;
        for (ix mm = 0; mm < half; ++mm) {
            ix o = (2 * mm + 1) * stride;
            trsm(x + o * n, n, 1, 1, f->crL[l] + mm * nn, n, LL);
        }
        for (ix mm = 0; mm < half; ++mm) {
            double *ye = x + 2 * mm * stride * n;
            mv(f->crU[l] + mm * nn, n, 0, x + (2 * mm + 1) * stride * n, ye, -1);
            if (mm > 0)
                mv(f->crY[l] + (mm - 1) * nn, n, 0,
                   x + ((2 * (mm - 1) + 1) * stride % P) * n, ye, -1);
        }
    }
    trsm(x, n, 1, 1, f->Lbase, n, LL);
}

static void cr_backward(const ofac *f, double *x) {
    ix P = f->q.P, n = f->q.nx, nn = n * n;
    trsm(x, n, 1, 1, f->Lbase, n, LLT);
    ix s = P >> f->levels;
    for (ix l = f->levels; l-- > 0; s *= 2) {
        ix sl = 2 * s, half = sl / 2, stride = P / sl;
        for (ix mm = 0; mm < half; ++mm) {
            ix o = (2 * mm + 1) * stride;
            double *xo = x + o * n;
            mv(f->crU[l] + mm * nn, n, 1, x + 2 * mm * stride * n, xo, -1);
            ix onext = ((2 * mm + 2) * stride) % P;
            if (2 * mm + 2 < sl)
                mv(f->crY[l] + mm * nn, n, 1, x + onext * n, xo, -1);
            trsm(xo, n, 1, 1, f->crL[l] + mm * nn, n, LLT);
        }
    }
}

/* solve (kkt_solve.cpp:23-309) for instance b; rhs arrays of that batch. */
static void do_solve(const ofac *f, const oc_dims *d, const oc_ocp *p,
                     const oc_rhs *rhs, ix b, oc_sol *out) {
    const prob *q = &f->q;
    ix nx = q->nx, nu = q->nu, nux = q->nux, P = q->P, n = q->n, N = q->N;
    (void)d;
    double *wu = zalloc((size_t)(n * P * nu)), *wx = zalloc((size_t)(n * P * nx));
    double *wl = zalloc((size_t)(n * P * nx));
    double *fwd = zalloc((size_t)(P * nx)), *bwd = zalloc((size_t)(P * nx));
    double *t1 = zalloc((size_t)nx), *t2 = zalloc((size_t)nx);
    double *lam = zalloc((size_t)(P * nx));
    const double *ru = rhs->ru + b * N * nu, *qx = rhs->qx + b * (N + 1) * nx;
    const double *fd = rhs->fd + b * N * nx;
#define WU(s, c) (wu + ((s) * P + (c)) * nu)
#define WX(s, c) (wx + ((s) * P + (c)) * nx)
#define WL(s, c) (wl + ((s) * P + (c)) * nx)
    /* scatter (kkt_solve.cpp:41-63) */
    for (ix c = 0; c < P; ++c)
        for (ix s = 0; s < n; ++s) {
            ix j = stage_of(q, c, s), xi = x_index_of(q, c, s);
            if (j < N)
                memcpy(WU(s, c), ru + j * nu, sizeof(double) * (size_t)nu);
            if (xi <= N)
                memcpy(WX(s, c), qx + xi * nx, sizeof(double) * (size_t)nx);
            if (s + 1 < n) {
                ix j2 = stage_of(q, c, s + 1);
                if (j2 < N)
                    memcpy(WL(s, c), fd + j2 * nx, sizeof(double) * (size_t)nx);
            }
        }
    /* forward substitution (kkt_solve.cpp:72-134) */
    for (ix c = 0; c < P; ++c) {
        for (ix s = 0; s < n; ++s) {
            const double *lh = BLK(f->LH, s, c, nux * nux);
            const double *lr = lh, *ls = lh + nu * nux, *lq = lh + nu * nux + nu;
            double *u = WU(s, c), *x = WX(s, c);
            trsm(u, nu, 1, 1, lr, nux, LL);
            gemm(x, nx, 1, 1, ls, nux, 0, u, 1, 0, nu, -1);
            trsm(x, nx, 1, 1, lq, nux, LL);
            if (s + 1 < n) {
                double *w = WL(s, c);
                trmm(t1, 1, w, nx, 1, 1, lq, nx, nux, TR_LLT, -1);
                memcpy(w, t1, sizeof(double) * (size_t)nx);
                add_scaled(w, x, nx, -1);
                trmm(t2, 1, w, nx, 1, 1, lq, nx, nux, TR_LL, 1);
                const double *bat = BLK(f->BAt, s + 1, c, nux * nx);
                gemm(WU(s + 1, c), nu, 1, 1, bat, nx, 0, t2, 1, 0, nx, -1);
                gemm(WX(s + 1, c), nx, 1, 1, bat + nu * nx, nx, 0, t2, 1, 0, nx, -1);
            }
        }
        double *fv = fwd + c * nx;
        for (ix s = 0; s < n; ++s) {
            gemm(fv, nx, 1, 1, BLK(f->LB, s, c, nx * nu), nu, 0, WU(s, c), 1, 0,
                 nu, +1);
            const double *lq = BLK(f->LH, s, c, nux * nux) + nu * nux + nu;
            if (s + 1 < n) {
                memcpy(t1, WX(s, c), sizeof(double) * (size_t)nx);
                add_scaled(t1, WL(s, c), nx, +1);
                trsm(t1, nx, 1, 1, lq, nux, LLT);
                gemm(fv, nx, 1, 1, BLK(f->Acl, s, c, nx * nx), nx, 0, t1, 1, 0,
                     nx, +1);
            } else {
                gemm(fv, nx, 1, 1, f->LA + c * nx * nx, nx, 0, WX(s, c), 1, 0,
                     nx, +1);
                trmm(bwd + c * nx, 1, WX(s, c), nx, 1, 1, f->T + c * nx * nx,
                     nx, nx, TR_LU, 1);
            }
        }
    }
    /* Schur system (kkt_solve.cpp:137-182) */
    for (ix i = 0; i < P; ++i) {
        ix j = q->n * i;
        for (ix a = 0; a < nx; ++a) {
            double val = j < N ? fd[j * nx + a] : 0;
            val -= fwd[i * nx + a];
            val += bwd[((i + 1) % P) * nx + a];
            lam[i * nx + a] = val;
        }
    }
    cr_forward(f, lam);
    cr_backward(f, lam);
    for (ix i = 0; i < P * nx; ++i)
        lam[i] = -lam[i];
    /* back substitution (kkt_solve.cpp:185-266) */
    for (ix c = 0; c < P; ++c) {
        const double *lf = lam + c * nx, *lb = lam + ((c - 1 + P) % P) * nx;
        for (ix s = 0; s < n; ++s) {
            double *u = WU(s, c), *x = WX(s, c);
            gemm(u, nu, 1, 1, BLK(f->LB, s, c, nx * nu), nu, 1, lf, 1, 0, nx, -1);
            const double *lq = BLK(f->LH, s, c, nux * nux) + nu * nux + nu;
            if (s + 1 < n) {
                memset(t1, 0, sizeof(double) * (size_t)nx);
                gemm(t1, nx, 1, 1, BLK(f->Acl, s, c, nx * nx), nx, 1, lf, 1, 0,
                     nx, +1);
                trsm(t1, nx, 1, 1, lq, nux, LL);
                add_scaled(x, t1, nx, -1);
                double *w = WL(s, c);
                for (ix a = 0; a < nx; ++a)
                    w[a] = -w[a] - t1[a];
            } else {
                gemm(x, nx, 1, 1, f->LA + c * nx * nx, nx, 1, lf, 1, 0, nx, -1);
                trmm(t1, 1, lb, nx, 1, 1, f->T + c * nx * nx, nx, nx, TR_LUT, 1);
                add_scaled(x, t1, nx, +1);
            }
        }
        for (ix s = n; s-- > 0;) {
            const double *lh = BLK(f->LH, s, c, nux * nux);
            const double *lr = lh, *ls = lh + nu * nux, *lq = lh + nu * nux + nu;
            double *u = WU(s, c), *x = WX(s, c);
            if (s + 1 < n) {
                double *w = WL(s, c);
                const double *bat = BLK(f->BAt, s + 1, c, nux * nx);
                memset(t2, 0, sizeof(double) * (size_t)nx);
                gemm(t2, nx, 1, 1, bat, nx, 1, WU(s + 1, c), 1, 0, nu, +1);
                gemm(t2, nx, 1, 1, bat + nu * nx, nx, 1, WX(s + 1, c), 1, 0, nx,
                     +1);
                trmm(t1, 1, t2, nx, 1, 1, lq, nx, nux, TR_LLT, 1);
                add_scaled(w, t1, nx, -1);
                trmm(t1, 1, w, nx, 1, 1, lq, nx, nux, TR_LL, 1);
                for (ix a = 0; a < nx; ++a)
                    w[a] = -t1[a];
                memcpy(t1, w, sizeof(double) * (size_t)nx);
                trsm(t1, nx, 1, 1, lq, nux, LL);
                add_scaled(x, t1, nx, +1);
            }
            trsm(x, nx, 1, 1, lq, nux, LLT);
            gemm(u, nu, 1, 1, ls, nux, 1, x, 1, 0, nx, -1);
            trsm(u, nu, 1, 1, lr, nux, LLT);
        }
    }
    /* gather (kkt_solve.cpp:268-307) */
    double *ou = out->u + b * N * nu, *ox = out->x + b * (N + 1) * nx;
    double *ol = out->lam + b * N * nx;
    memcpy(ox, p->x_init + b * nx, sizeof(double) * (size_t)nx);
    for (ix c = 0; c < P; ++c)
        for (ix s = 0; s < n; ++s) {
            ix j = stage_of(q, c, s), xi = x_index_of(q, c, s);
            if (j < N)
                memcpy(ou + j * nu, WU(s, c), sizeof(double) * (size_t)nu);
            if (xi <= N)
                memcpy(ox + xi * nx, WX(s, c), sizeof(double) * (size_t)nx);
            if (s + 1 < n) {
                ix j2 = stage_of(q, c, s + 1);
                if (j2 < N)
                    memcpy(ol + j2 * nx, WL(s, c), sizeof(double) * (size_t)nx);
            }
        }
    for (ix i = 0; i < P; ++i) {
        ix j = q->n * i;
        if (j < N)
            memcpy(ol + j * nx, lam + i * nx, sizeof(double) * (size_t)nx);
    }
#undef WU
#undef WX
#undef WL
    free(wu); free(wx); free(wl); free(fwd); free(bwd); free(t1); free(t2);
    free(lam);
}

/* EqRhs::of_problem (ocp.cpp:154-174) */
void oc_rhs_of_problem(const oc_dims *d, const oc_ocp *p, double *ru,
                       double *qx, double *fd) {
    ix N = d->N, nx = d->nx, nu = d->nu;
    for (ix b = 0; b < d->batch; ++b) {
        double *rub = ru + b * N * nu, *qxb = qx + b * (N + 1) * nx;
        double *fdb = fd + b * N * nx;
        for (ix j = 0; j < N; ++j) {
            for (ix i = 0; i < nu; ++i)
                rub[j * nu + i] = -p->r[(b * N + j) * nu + i];
            for (ix i = 0; i < nx; ++i)
                fdb[j * nx + i] = -p->f[(b * N + j) * nx + i];
        }
        for (ix i = 0; i < nx; ++i)
            qxb[i] = 0;
        for (ix j = 1; j <= N; ++j)
            for (ix i = 0; i < nx; ++i)
                qxb[j * nx + i] = -p->q[(b * (N + 1) + j) * nx + i];
        const double *x0 = p->x_init + b * nx;
        const double *S0 = p->S + b * N * nu * nx, *A0 = p->A + b * N * nx * nx;
        for (ix i = 0; i < nu; ++i) { /* axpy(ru[0], S0, x_init, -1) */
            double s = 0;
            for (ix k = 0; k < nx; ++k)
                s += S0[i * nx + k] * x0[k];
            rub[i] += -1 * s;
        }
        for (ix i = 0; i < nx; ++i) {
            double s = 0;
            for (ix k = 0; k < nx; ++k)
                s += A0[i * nx + k] * x0[k];
            fdb[i] += -1 * s;
        }
    }
}

int oc_solve(const oc_dims *d, const oc_ocp *p, const oc_rhs *rhs,
             oc_sol *out, oc_status *st) {
    int worst = 0;
    for (ix b = 0; b < d->batch; ++b) {
        ofac f;
        int rc = do_factor(d, p, b, &f, st ? st + b : NULL);
        if (rc == 0)
            do_solve(&f, d, p, rhs, b, out);
        ofac_free(&f);
        if (rc > worst)
            worst = rc;
    }
    return worst;
}

int oc_solve_problem(const oc_dims *d, const oc_ocp *p, oc_sol *out,
                     oc_status *st) {
    ix N = d->N, nx = d->nx, nu = d->nu, B = d->batch;
    double *ru = zalloc((size_t)(B * N * nu)), *qx = zalloc((size_t)(B * (N + 1) * nx));
    double *fd = zalloc((size_t)(B * N * nx));
    oc_rhs_of_problem(d, p, ru, qx, fd);
    oc_rhs r = {ru, qx, fd};
    int rc = oc_solve(d, p, &r, out, st);
    free(ru); free(qx); free(fd);
    return rc;
}

int oc_factor_export(const oc_dims *d, const oc_ocp *p, oc_factor_blocks *o,
                     oc_status *st) {
    ofac f;
    int rc = do_factor(d, p, 0, &f, st);
    if (rc == 1) {
        ofac_free(&f);
        return rc;
    }
    const prob *q = &f.q;
    ix nx = q->nx, nu = q->nu, nux = q->nux, n = q->n, P = q->P, nn = nx * nx;
    memcpy(o->LH, f.LH, sizeof(double) * (size_t)(n * P * nux * nux));
    memcpy(o->LB, f.LB, sizeof(double) * (size_t)(n * P * nx * nu));
    memcpy(o->Acl, f.Acl, sizeof(double) * (size_t)(n * P * nn));
    memcpy(o->LA, f.LA, sizeof(double) * (size_t)(P * nn));
    memcpy(o->T, f.T, sizeof(double) * (size_t)(P * nn));
    memcpy(o->W, f.W, sizeof(double) * (size_t)(P * nn));
    memcpy(o->schur_sub, f.Ks, sizeof(double) * (size_t)(P * nn));
    for (ix c = 0; c < P; ++c)
        for (ix a = 0; a < nx; ++a)
            for (ix b = 0; b < nx; ++b) {
                ix lo = a >= b ? a * nx + b : b * nx + a;
                o->Mfwd[c * nn + a * nx + b] = f.Mfwd[c * nn + lo];
                o->Mbwd[c * nn + a * nx + b] = f.Mbwd[c * nn + lo];
                o->schur_diag[c * nn + a * nx + b] = f.Md[c * nn + lo];
            }
    ofac_free(&f);
    return rc;
}

/* kkt_residual_eq (ocp.cpp:180-230) */
void oc_kkt_residual(const oc_dims *d, const oc_ocp *p, const oc_rhs *rhs,
                     const oc_sol *s, double *out) {
    ix N = d->N, nx = d->nx, nu = d->nu;
    double *g = zalloc((size_t)(nx + nu));
    for (ix b = 0; b < d->batch; ++b) {
        const double *u = s->u + b * N * nu, *x = s->x + b * (N + 1) * nx;
        const double *lam = s->lam + b * N * nx;
        double su = 0, sx = 0, dy = 0, te = 0;
        for (ix j = 0; j < N; ++j) {
            const double *R = p->R + (b * N + j) * nu * nu;
            const double *S = p->S + (b * N + j) * nu * nx;
            const double *B = p->B + (b * N + j) * nx * nu;
            const double *A = p->A + (b * N + j) * nx * nx;
            for (ix i = 0; i < nu; ++i) {
                double v = -rhs->ru[(b * N + j) * nu + i], t = 0;
                for (ix k = 0; k < nu; ++k) t += R[i * nu + k] * u[j * nu + k];
                v += t;
                if (j > 0) {
                    t = 0;
                    for (ix k = 0; k < nx; ++k) t += S[i * nx + k] * x[j * nx + k];
                    v += t;
                }
                t = 0;
                for (ix k = 0; k < nx; ++k) t += B[k * nu + i] * lam[j * nx + k];
                v += t;
                if (fabs(v) > su) su = fabs(v);
            }
            for (ix i = 0; i < nx; ++i) {
                double v = -rhs->fd[(b * N + j) * nx + i], t = 0;
                for (ix k = 0; k < nu; ++k) t += B[i * nu + k] * u[j * nu + k];
                v += t;
                if (j > 0) {
                    t = 0;
                    for (ix k = 0; k < nx; ++k) t += A[i * nx + k] * x[j * nx + k];
                    v += t;
                }
                v -= x[(j + 1) * nx + i];
                if (fabs(v) > dy) dy = fabs(v);
            }
        }
        for (ix j = 1; j < N; ++j) {
            const double *S = p->S + (b * N + j) * nu * nx;
            const double *Q = p->Q + (b * (N + 1) + j) * nx * nx;
            const double *A = p->A + (b * N + j) * nx * nx;
            for (ix i = 0; i < nx; ++i) {
                double v = -rhs->qx[(b * (N + 1) + j) * nx + i], t = 0;
                for (ix k = 0; k < nu; ++k) t += S[k * nx + i] * u[j * nu + k];
                v += t;
                t = 0;
                for (ix k = 0; k < nx; ++k) t += Q[i * nx + k] * x[j * nx + k];
                v += t;
                t = 0;
                for (ix k = 0; k < nx; ++k) t += A[k * nx + i] * lam[j * nx + k];
                v += t;
                v -= lam[(j - 1) * nx + i];
                if (fabs(v) > sx) sx = fabs(v);
            }
        }
        {
            const double *Q = p->Q + (b * (N + 1) + N) * nx * nx;
            for (ix i = 0; i < nx; ++i) {
                double v = -rhs->qx[(b * (N + 1) + N) * nx + i], t = 0;
                for (ix k = 0; k < nx; ++k) t += Q[i * nx + k] * x[N * nx + k];
                v += t;
                v -= lam[(N - 1) * nx + i];
                if (fabs(v) > te) te = fabs(v);
            }
        }
        out[b * 4 + 0] = su; out[b * 4 + 1] = sx;
        out[b * 4 + 2] = dy; out[b * 4 + 3] = te;
    }
    free(g);
}

/* Counts from the reference's own counter semantics on a dummy
 * well-conditioned instance (counts depend only on the shape). */
void oc_fma_counts(const oc_dims *d, uint64_t *out) {
    ix N = d->N, nx = d->nx, nu = d->nu;
    oc_dims d1 = *d;
    d1.batch = 1;
    double *A = zalloc((size_t)(N * nx * nx)), *B = zalloc((size_t)(N * nx * nu));
    double *R = zalloc((size_t)(N * nu * nu)), *S = zalloc((size_t)(N * nu * nx));
    double *Q = zalloc((size_t)((N + 1) * nx * nx)), *f = zalloc((size_t)(N * nx));
    double *r = zalloc((size_t)(N * nu)), *q = zalloc((size_t)((N + 1) * nx));
    double *x0 = zalloc((size_t)nx);
    for (ix j = 0; j < N; ++j)
        for (ix i = 0; i < nu; ++i)
            R[j * nu * nu + i * nu + i] = 1;
    for (ix j = 0; j <= N; ++j)
        for (ix i = 0; i < nx; ++i)
            Q[j * nx * nx + i * nx + i] = 1;
    oc_ocp p = {A, B, R, S, Q, f, r, q, x0};
    ofac fc;
    g_fma = 0;
    do_factor(&d1, &p, 0, &fc, NULL);
    out[0] = g_fma;
    double *ru = zalloc((size_t)(N * nu)), *qx = zalloc((size_t)((N + 1) * nx));
    double *fd = zalloc((size_t)(N * nx));
    double *u = zalloc((size_t)(N * nu)), *x = zalloc((size_t)((N + 1) * nx));
    double *l = zalloc((size_t)(N * nx));
    oc_rhs rh = {ru, qx, fd};
    oc_sol so = {u, x, l};
    g_fma = 0;
    do_solve(&fc, &d1, &p, &rh, 0, &so);
    out[1] = g_fma;
    ofac_free(&fc);
    free(A); free(B); free(R); free(S); free(Q); free(f); free(r); free(q);
    free(x0); free(ru); free(qx); free(fd); free(u); free(x); free(l);
}

/* ---- instance-parallel CPU timing (the "port" baseline) ---------------- */
typedef struct {
    const oc_dims *d;
    const oc_ocp *p;
    const oc_rhs *rhs;
    oc_sol *out;
    int64_t n_solves;
    int64_t *next;
    pthread_mutex_t *mu;
    int failed;
} bench_arg;

static void *bench_worker(void *v) {
    bench_arg *a = (bench_arg *)v;
    for (;;) {
        pthread_mutex_lock(a->mu);
        int64_t i = (*a->next)++;
        pthread_mutex_unlock(a->mu);
        if (i >= a->n_solves)
            break;
        ix b = i % a->d->batch;
        ofac f;
        if (do_factor(a->d, a->p, b, &f, NULL) == 0)
            do_solve(&f, a->d, a->p, a->rhs, b, a->out);
        else
            a->failed = 1;
        ofac_free(&f);
    }
    return NULL;
}

double oc_bench_solve_problem(const oc_dims *d, const oc_ocp *p,
                              int64_t n_solves, int threads, oc_sol *out) {
    ix N = d->N, nx = d->nx, nu = d->nu, B = d->batch;
    double *ru = zalloc((size_t)(B * N * nu)), *qx = zalloc((size_t)(B * (N + 1) * nx));
    double *fd = zalloc((size_t)(B * N * nx));
    oc_rhs_of_problem(d, p, ru, qx, fd);
    oc_rhs r = {ru, qx, fd};
    if (threads < 1)
        threads = 1;
    int64_t next = 0;
    pthread_mutex_t mu = PTHREAD_MUTEX_INITIALIZER;
    bench_arg *args = calloc((size_t)threads, sizeof(bench_arg));
    pthread_t *th = calloc((size_t)threads, sizeof(pthread_t));
    struct timespec t0, t1;
    clock_gettime(CLOCK_MONOTONIC, &t0);
    for (int w = 0; w < threads; ++w) {
        args[w] = (bench_arg){d, p, &r, out, n_solves, &next, &mu, 0};
        pthread_create(&th[w], NULL, bench_worker, &args[w]);
    }
    int failed = 0;
    for (int w = 0; w < threads; ++w) {
        pthread_join(th[w], NULL);
        failed |= args[w].failed;
    }
    clock_gettime(CLOCK_MONOTONIC, &t1);
    free(args); free(th); free(ru); free(qx); free(fd);
    if (failed)
        return -1.0;
    return (double)(t1.tv_sec - t0.tv_sec) + 1e-9 * (double)(t1.tv_nsec - t0.tv_nsec);
}


/* ---- exact line search (qpalm::line_search_exact) ---------------------- */

typedef struct {
    double t, w;
} oc_bp;

static int oc_bp_cmp(const void *a, const void *b) {
    const double x = ((const oc_bp *)a)->t, y = ((const oc_bp *)b)->t;
    return (x > y) - (x < y);
}

/* LineSearchData::add_term (line_search.cpp:9-27) for every term, the
 * 0+ fold of the w < 0 breakpoints (line_search.cpp:116-124), the descent
 * check (:125-130), then the root on the sorted breakpoints: the
 * reference's final sort + scan (:154-171) applied to the whole set (its
 * pivot partitions only narrow the set the scan starts from). */
int oc_line_search(int64_t m, const double *alpha, const double *delta,
                   double eta, double beta, double *tau) {
    oc_bp *pts = (oc_bp *)malloc(sizeof(oc_bp) * (size_t)(m > 0 ? m : 1));
    int64_t np = 0;
    for (int64_t i = 0; i < m; ++i) {
        const double d = delta[i];
        if (d == 0)
            continue;
        const double t = alpha[i] / d;
        if (!isfinite(t))
            continue;
        const double w = d * fabs(d);
        if (t <= 0) {
            if (w > 0) {
                eta += w;
                beta -= t * w;
            }
            continue;
        }
        pts[np].t = t;
        pts[np].w = w;
        ++np;
    }
    double eta_c = eta, beta_c = beta;
    for (int64_t i = 0; i < np; ++i)
        if (pts[i].w < 0) {
            eta_c -= pts[i].w;
            beta_c += pts[i].t * pts[i].w;
        }
    if (beta_c >= 0) {
        free(pts);
        *tau = 0;
        return beta_c == 0 ? 0 : 1;
    }
    qsort(pts, (size_t)np, sizeof(oc_bp), oc_bp_cmp);
    for (int64_t i = 0; i < np; ++i) {
        if (eta_c * pts[i].t + beta_c >= 0)
            break;
        eta_c += pts[i].w;
        beta_c -= pts[i].t * pts[i].w;
    }
    *tau = -beta_c / eta_c;
    free(pts);
    return 0;
}

typedef struct {
    int64_t b0, b1, m;
    const double *alpha, *delta, *eta, *beta;
    double *tau;
} oc_ls_job;

static void *oc_ls_worker(void *arg) {
    oc_ls_job *j = (oc_ls_job *)arg;
    for (int64_t b = j->b0; b < j->b1; ++b)
        oc_line_search(j->m, j->alpha + b * j->m, j->delta + b * j->m, j->eta[b], j->beta[b],
                       j->tau + b);
    return NULL;
}

double oc_bench_line_search(int64_t batch, int64_t m, const double *alpha, const double *delta,
                            const double *eta, const double *beta, double *tau, int threads) {
    if (threads < 1)
        threads = 1;
    pthread_t th[256];
    oc_ls_job jobs[256];
    if (threads > 256)
        threads = 256;
    struct timespec t0, t1;
    clock_gettime(CLOCK_MONOTONIC, &t0);
    for (int k = 0; k < threads; ++k) {
        jobs[k] = (oc_ls_job){batch * k / threads, batch * (k + 1) / threads, m, alpha, delta, eta,
                              beta, tau};
        pthread_create(&th[k], NULL, oc_ls_worker, &jobs[k]);
    }
    for (int k = 0; k < threads; ++k)
        pthread_join(th[k], NULL);
    clock_gettime(CLOCK_MONOTONIC, &t1);
    return (double)(t1.tv_sec - t0.tv_sec) + 1e-9 * (double)(t1.tv_nsec - t0.tv_nsec);
}
