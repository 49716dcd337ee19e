/*
 * finom_oracle.c -- CPU restatement of the FINOM reference hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the
 * B200 CUDA path and the CPU baseline timed by bench.py ("kind": "port").
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load it.  The product path
 * (paper_2605_26659_b200) never links or calls it.
 *
 * It restates, sequentially and in the same operation order, the
 * reference package at /root/reference/pkg/src/finom (numba/numpy):
 *
 *   orc_dividing_index      kernel1d.py:55-62      searchsorted(side="right")
 *   rep_build               kernel1d.py:121-159    _build_rep_arrays
 *   op1_assemble            kernel1d.py:241-255    _assemble (4 reps)
 *   dp_apply / dp_blocks    _kernels.py:53-125     segmented fwd/bwd scans
 *   dp_apply_dyn/_blocks_dyn _kernels.py:128-203   on-the-fly exponents
 *   iter_1d                 _kernels.py:260-350    fused 1D iteration
 *   iter_2d_baked           _kernels.py:353-428    2D iteration, plain kernel
 *   iter_2d_dyn             _kernels.py:431-521    2D iteration, shift grids
 *   shift                   solver.py:135-153      _shift with np.interp fill
 *   run loop                solver.py:156-199      run_driver
 *   orc_sinkhorn_1d         solver.py:202-230      sinkhorn_1d
 *   cost_1d                 solver.py:252-271      transport_cost_fast
 *   orc_sinkhorn_2d         kernel2d.py:363-391    sinkhorn_2d
 *   cost_2d                 kernel2d.py:394-465    transport_cost_fast_2d
 *
 * Build with -ffp-contract=off (no FMA contraction), as numba's
 * fastmath=False lowering does (_backend.py:62).  exp/log are the libm
 * ones numba lowers np.exp/np.log to.  Table construction in the
 * reference uses numpy's vectorised np.exp, which may differ from libm
 * in the last ulp on rare arguments; the golden fixtures in
 * tests/golden pin the agreement that results (see tests/test_oracle.py).
 */
#define _POSIX_C_SOURCE 199309L
#include <math.h>
#include <stdint.h>
#include <time.h>
#include <stdlib.h>
#include <string.h>

typedef int64_t i64;

enum { ST_OK = 0, ST_ZERO_DENOM = 1, ST_NONFINITE = 2, ST_BADARG = 100 };

/* ------------------------------------------------------------------ */
/* kernel1d.py:55-62  zeta[i] = #{j : y_j <= x_i}                      */
void orc_dividing_index(const double *x, i64 n, const double *y, i64 m, i64 *z) {
    i64 j = 0;
    for (i64 i = 0; i < n; ++i) {
        while (j < m && y[j] <= x[i]) ++j;
        z[i] = j;
    }
}

/* One QuasiCollinearRep (kernel1d.py:65-111) as flat arrays. */
typedef struct {
    int lower;
    i64 n, m, ne;
    i64 *z;          /* borrowed */
    double *ratios;  /* n-1 */
    double *edges;   /* ne */
    i64 *owner;      /* ne */
    double *dist;    /* ne */
    double *gaps;    /* n-1 */
} rep_t;

static void rep_free(rep_t *r) {
    free(r->ratios); free(r->edges); free(r->owner); free(r->dist); free(r->gaps);
    memset(r, 0, sizeof(*r));
}

/* kernel1d.py:121-159 _build_rep_arrays */
static int rep_build(rep_t *r, const double *row, i64 n, const double *col, i64 m,
                     i64 *z, double eps, int lower, const double *ra, const double *ca) {
    memset(r, 0, sizeof(*r));
    r->lower = lower; r->n = n; r->m = m; r->z = z;
    i64 ng = n > 1 ? n - 1 : 0;
    r->gaps = (double *)malloc(sizeof(double) * (ng ? ng : 1));
    r->ratios = (double *)malloc(sizeof(double) * (ng ? ng : 1));
    for (i64 i = 0; i < ng; ++i) r->gaps[i] = row[i + 1] - row[i];
    i64 c0 = lower ? 0 : z[0];
    i64 c1 = lower ? z[n - 1] : m;
    r->ne = c1 - c0;
    i64 ne1 = r->ne ? r->ne : 1;
    r->edges = (double *)malloc(sizeof(double) * ne1);
    r->owner = (i64 *)malloc(sizeof(i64) * ne1);
    r->dist = (double *)malloc(sizeof(double) * ne1);
    if (!r->gaps || !r->ratios || !r->edges || !r->owner || !r->dist) return ST_BADARG;
    /* row_owner = np.repeat(arange(n), counts) */
    i64 k = 0;
    for (i64 i = 0; i < n; ++i) {
        i64 cnt;
        if (lower) cnt = z[i] - (i ? z[i - 1] : 0);
        else cnt = (i + 1 < n ? z[i + 1] : m) - z[i];
        for (i64 t = 0; t < cnt; ++t) r->owner[k++] = i;
    }
    for (i64 q = 0; q < r->ne; ++q) {
        i64 o = r->owner[q], c = c0 + q;
        r->dist[q] = lower ? row[o] - col[c] : col[c] - row[o];
    }
    for (i64 i = 0; i < ng; ++i) {
        double d = ra[i + 1] - ra[i];                 /* np.diff(row_abs) */
        double e = lower ? (-r->gaps[i] + d) : (-r->gaps[i] - d);
        r->ratios[i] = exp(e / eps);
        int conventional = lower ? (z[i] == 0) : (z[i + 1] == m);
        if (conventional) r->ratios[i] = 1.0;
    }
    for (i64 q = 0; q < r->ne; ++q) {
        i64 o = r->owner[q], c = c0 + q;
        r->edges[q] = exp(((-r->dist[q] + ra[o]) + ca[c]) / eps);
    }
    return ST_OK;
}

/* KernelOperator1D (kernel1d.py:194-255): 4 reps. */
typedef struct {
    i64 n, m;
    double eps;
    i64 *zf, *zt;
    rep_t lo, up, tlo, tup;
} op1_t;

static void op1_free(op1_t *op) {
    rep_free(&op->lo); rep_free(&op->up); rep_free(&op->tlo); rep_free(&op->tup);
    free(op->zf); free(op->zt);
    memset(op, 0, sizeof(*op));
}

/* kernel1d.py:241-255 _assemble */
static int op1_assemble(op1_t *op, const double *x, i64 n, const double *y, i64 m, double eps,
                        const double *a, const double *b) {
    memset(op, 0, sizeof(*op));
    op->n = n; op->m = m; op->eps = eps;
    op->zf = (i64 *)malloc(sizeof(i64) * n);
    op->zt = (i64 *)malloc(sizeof(i64) * m);
    if (!op->zf || !op->zt) return ST_BADARG;
    orc_dividing_index(x, n, y, m, op->zf);
    orc_dividing_index(y, m, x, n, op->zt);
    int s = 0;
    s |= rep_build(&op->lo, x, n, y, m, op->zf, eps, 1, a, b);
    s |= rep_build(&op->up, x, n, y, m, op->zf, eps, 0, a, b);
    s |= rep_build(&op->tlo, y, m, x, n, op->zt, eps, 1, b, a);
    s |= rep_build(&op->tup, y, m, x, n, op->zt, eps, 0, b, a);
    return s;
}

/* ------------------------------------------------------------------ */
/* _kernels.py:53-88 _dp_apply, :91-125 _dp_blocks (out==NULL -> blocks) */
static void dp_scan(const i64 *z, i64 n, const double *r_lo, const double *r_hi,
                    const double *lo, const double *hi, const double *psi, i64 m,
                    double *out, double *p, double *q) {
    i64 zprev = 0;
    double pv = 0.0;
    for (i64 i = 0; i < n; ++i) {
        i64 zi = z[i];
        double acc = 0.0;
        for (i64 t = zprev; t < zi; ++t) acc += lo[t] * psi[t];
        if (zprev > 0) {
            pv = r_lo[i - 1] * pv;
            if (zi > zprev) pv += acc;
        } else {
            pv = acc;
        }
        if (out) out[i] = pv; else p[i] = pv;
        zprev = zi;
    }
    i64 z0 = z[0], znext = m;
    double qv = 0.0;
    for (i64 i = n - 1; i >= 0; --i) {
        i64 zi = z[i];
        double acc = 0.0;
        for (i64 t = zi; t < znext; ++t) acc += hi[t - z0] * psi[t];
        if (znext < m) {
            qv = r_hi[i] * qv;
            if (znext > zi) qv += acc;
        } else {
            qv = acc;
        }
        if (out) out[i] += qv; else q[i] = qv;
        znext = zi;
    }
}

/* _kernels.py:128-165 _dp_apply_dyn, :168-203 _dp_blocks_dyn */
static void dp_scan_dyn(const i64 *z, i64 n, const double *dx, const double *lo_d,
                        const double *hi_d, const double *a, const double *b, double inv_eps,
                        const double *psi, i64 m, double *out, double *p, double *q) {
    i64 zprev = 0;
    double pv = 0.0;
    for (i64 i = 0; i < n; ++i) {
        i64 zi = z[i];
        double ai = a[i];
        double acc = 0.0;
        for (i64 t = zprev; t < zi; ++t) acc += exp((ai + b[t] - lo_d[t]) * inv_eps) * psi[t];
        if (zprev > 0) {
            pv = exp((ai - a[i - 1] - dx[i - 1]) * inv_eps) * pv;
            if (zi > zprev) pv += acc;
        } else {
            pv = acc;
        }
        if (out) out[i] = pv; else p[i] = pv;
        zprev = zi;
    }
    i64 z0 = z[0], znext = m;
    double qv = 0.0;
    for (i64 i = n - 1; i >= 0; --i) {
        i64 zi = z[i];
        double ai = a[i];
        double acc = 0.0;
        for (i64 t = zi; t < znext; ++t) acc += exp((ai + b[t] - hi_d[t - z0]) * inv_eps) * psi[t];
        if (znext < m) {
            qv = exp((ai - a[i + 1] - dx[i]) * inv_eps) * qv;
            if (znext > zi) qv += acc;
        } else {
            qv = acc;
        }
        if (out) out[i] += qv; else q[i] = qv;
        znext = zi;
    }
}


/* numpy's pairwise summation (np.sum of a contiguous float64 array). */
static double pairwise_sum(const double *a, i64 n) {
    if (n < 8) {
        double res = 0.0;
        for (i64 i = 0; i < n; ++i) res += a[i];
        return res;
    } else if (n <= 128) {
        double r[8];
        for (int j = 0; j < 8; ++j) r[j] = a[j];
        i64 i;
        for (i = 8; i < n - (n % 8); i += 8)
            for (int j = 0; j < 8; ++j) r[j] += a[i + j];
        double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
        for (; i < n; ++i) res += a[i];
        return res;
    } else {
        i64 n2 = n / 2;
        n2 -= n2 % 8;
        return pairwise_sum(a, n2) + pairwise_sum(a + n2, n - n2);
    }
}

/* ------------------------------------------------------------------ */
typedef struct { double err; int status; double psmax, psmin, phmax, phmin; } itres_t;

/* _kernels.py:260-350 _iter_1d_body (flat scatter + recurrence form) */
static itres_t iter_1d(const op1_t *op, const double *u, const double *v, double *phi, double *psi,
                       double *t, double *qm, double *s, double *qn) {
    itres_t R = {0.0, ST_OK, 0.0, 0.0, 0.0, 0.0};
    i64 n = op->n, m = op->m;
    const rep_t *lot = &op->tlo, *hit = &op->tup, *lof = &op->lo, *hif = &op->up;
    for (i64 j = 0; j < m; ++j) { t[j] = 0.0; qm[j] = 0.0; }
    for (i64 k = 0; k < lot->ne; ++k) t[lot->owner[k]] += lot->edges[k] * phi[k];
    for (i64 j = 1; j < m; ++j) t[j] += lot->ratios[j - 1] * t[j - 1];
    i64 z0t = op->zt[0];
    for (i64 k = 0; k < hit->ne; ++k) qm[hit->owner[k]] += hit->edges[k] * phi[k + z0t];
    double err = 0.0, psmax = 0.0, psmin = INFINITY, qv = 0.0;
    for (i64 j = m - 1; j >= 0; --j) {
        if (j == m - 1) qv = qm[j];
        else qv = qm[j] + hit->ratios[j] * qv;
        double tj = t[j] + qv, vj = v[j];
        err += fabs(psi[j] * tj - vj);
        if (tj == 0.0) {
            if (vj > 0.0) { R.err = err; R.status = ST_ZERO_DENOM; return R; }
            psi[j] = 0.0;
        } else {
            double w = vj / tj;
            if (!isfinite(w)) { R.err = err; R.status = ST_NONFINITE; return R; }
            psi[j] = w;
            if (vj > 0.0) {
                if (w > psmax) psmax = w;
                if (w < psmin) psmin = w;
            }
        }
    }
    for (i64 i = 0; i < n; ++i) { s[i] = 0.0; qn[i] = 0.0; }
    for (i64 k = 0; k < lof->ne; ++k) s[lof->owner[k]] += lof->edges[k] * psi[k];
    for (i64 i = 1; i < n; ++i) s[i] += lof->ratios[i - 1] * s[i - 1];
    i64 z0f = op->zf[0];
    for (i64 k = 0; k < hif->ne; ++k) qn[hif->owner[k]] += hif->edges[k] * psi[k + z0f];
    double phmax = 0.0, phmin = INFINITY;
    qv = 0.0;
    for (i64 i = n - 1; i >= 0; --i) {
        if (i == n - 1) qv = qn[i];
        else qv = qn[i] + hif->ratios[i] * qv;
        double si = s[i] + qv, ui = u[i];
        if (si == 0.0) {
            if (ui > 0.0) { R.err = err; R.status = ST_ZERO_DENOM; return R; }
            phi[i] = 0.0;
        } else {
            double w = ui / si;
            if (!isfinite(w)) { R.err = err; R.status = ST_NONFINITE; return R; }
            phi[i] = w;
            if (ui > 0.0) {
                if (w > phmax) phmax = w;
                if (w < phmin) phmin = w;
            }
        }
    }
    R.err = err; R.psmax = psmax; R.psmin = psmin; R.phmax = phmax; R.phmin = phmin;
    return R;
}

/* ------------------------------------------------------------------ */
/* solver.py:135-153 _shift: eps*log(scaling) on positive mass, np.interp
 * (by index, constant extrapolation) on zero mass.  The interp follows
 * numpy's arr_interp arithmetic: slope*(x - xp[j]) + fp[j]. */
static void shift(const double *w, const double *sc, i64 n, double eps, double *out) {
    i64 npos = 0;
    for (i64 i = 0; i < n; ++i) if (w[i] > 0) ++npos;
    for (i64 i = 0; i < n; ++i) if (w[i] > 0) out[i] = eps * log(sc[i]);
    if (npos == n || npos == 0) return;
    i64 prev = -1;
    for (i64 i = 0; i < n; ++i) {
        if (w[i] > 0) { prev = i; continue; }
        i64 next = i + 1;
        while (next < n && !(w[next] > 0)) ++next;
        if (prev < 0) { out[i] = out[next]; continue; }        /* left: fp[0]  */
        if (next >= n) { out[i] = out[prev]; continue; }       /* right: fp[-1] */
        double xj = (double)prev, xj1 = (double)next, yj = out[prev], yj1 = out[next];
        double slope = (yj1 - yj) / (xj1 - xj);
        double xv = (double)i;
        double r = slope * (xv - xj) + yj;
        if (isnan(r)) {
            r = slope * (xv - xj1) + yj1;
            if (isnan(r) && yj == yj1) r = yj;
        }
        out[i] = r;
    }
}

/* solver.py:252-271 transport_cost_fast */
static double cost_1d(const op1_t *op, const double *x, const double *y, const double *phi,
                      const double *psi) {
    i64 n = op->n, m = op->m;
    double *p = malloc(sizeof(double) * n), *q = malloc(sizeof(double) * n);
    double *pt = malloc(sizeof(double) * n), *qt = malloc(sizeof(double) * n);
    double *yp = malloc(sizeof(double) * m);
    for (i64 j = 0; j < m; ++j) yp[j] = y[j] * psi[j];
    dp_scan(op->zf, n, op->lo.ratios, op->up.ratios, op->lo.edges, op->up.edges, psi, m, NULL, p, q);
    dp_scan(op->zf, n, op->lo.ratios, op->up.ratios, op->lo.edges, op->up.edges, yp, m, NULL, pt, qt);
    /* np.sum: pairwise summation of phi * (x*(p-q) - pt + qt) */
    double *term = malloc(sizeof(double) * n);
    for (i64 i = 0; i < n; ++i) term[i] = phi[i] * (x[i] * (p[i] - q[i]) - pt[i] + qt[i]);
    double s = pairwise_sum(term, n);
    free(p); free(q); free(pt); free(qt); free(yp); free(term);
    return s;
}

/* ------------------------------------------------------------------ */
/* Driver (solver.py:156-199 run_driver) shared by 1D and 2D.         */
typedef itres_t (*iterate_fn)(void *ad, const double *u, const double *v, double *phi, double *psi);
typedef int (*absorb_fn)(void *ad, const double *da, const double *db);

typedef struct {
    double eps; i64 itr_max; double tol; int stabilize; double thr; i64 check_every;
} cfg_t;

/* info[0]=iterations_run info[1]=converged info[2]=status info[3]=n_absorb
 * info[4]=iteration of failure (0 if none)
 * hist[it-1] = err of iteration it (every iteration; cadence filtered by caller) */
static int run_driver(void *ad, iterate_fn it_fn, absorb_fn ab_fn, const double *u, i64 n,
                      const double *v, i64 m, const cfg_t *c, double *phi, double *psi,
                      double *hist, i64 *info, i64 *absorb_its) {
    for (i64 i = 0; i < n; ++i) phi[i] = 1.0 / (double)n;
    for (i64 j = 0; j < m; ++j) psi[j] = 1.0 / (double)n;
    double hi_cut = exp(c->thr), lo_cut = exp(-c->thr);
    double *da = malloc(sizeof(double) * n), *db = malloc(sizeof(double) * m);
    i64 it = 0, nab = 0;
    int converged = 0, status = ST_OK;
    while (it < c->itr_max) {
        itres_t r = it_fn(ad, u, v, phi, psi);
        it += 1;
        hist[it - 1] = r.err;
        if (r.status != ST_OK) { status = r.status; break; }
        if (c->tol > 0 && r.err <= c->tol) { converged = 1; break; }
        if (c->stabilize && (r.phmax > hi_cut || r.psmax > hi_cut || r.phmin < lo_cut ||
                             r.psmin < lo_cut)) {
            shift(u, phi, n, c->eps, da);
            shift(v, psi, m, c->eps, db);
            int s = ab_fn(ad, da, db);
            if (s) { status = s; break; }
            if (absorb_its) absorb_its[nab] = it;
            nab++;
            for (i64 i = 0; i < n; ++i) phi[i] = 1.0;
            for (i64 j = 0; j < m; ++j) psi[j] = 1.0;
        }
    }
    info[0] = it; info[1] = converged; info[2] = status; info[3] = nab;
    info[4] = status != ST_OK ? it : 0;
    free(da); free(db);
    return status;
}

/* ---------------------------- 1D solver ----------------------------- */
typedef struct {
    const double *x, *y; i64 n, m; double eps;
    double *a, *b;
    op1_t op;
    double *t, *qm, *s, *qn;
} ad1_t;

static itres_t ad1_iterate(void *p, const double *u, const double *v, double *phi, double *psi) {
    ad1_t *ad = (ad1_t *)p;
    return iter_1d(&ad->op, u, v, phi, psi, ad->t, ad->qm, ad->s, ad->qn);
}

/* kernel1d.py:313-325 absorb: rebuild every table from a+da, b+db */
static int ad1_absorb(void *p, const double *da, const double *db) {
    ad1_t *ad = (ad1_t *)p;
    for (i64 i = 0; i < ad->n; ++i) ad->a[i] = ad->a[i] + da[i];
    for (i64 j = 0; j < ad->m; ++j) ad->b[j] = ad->b[j] + db[j];
    op1_free(&ad->op);
    return op1_assemble(&ad->op, ad->x, ad->n, ad->y, ad->m, ad->eps, ad->a, ad->b);
}

static double now_s(void) {
    struct timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return ts.tv_sec + 1e-9 * ts.tv_nsec;
}

/* solver.py:202-230 sinkhorn_1d.  out_a/out_b receive the absorbed
 * shifts, hist[itr_max] the per-iteration errors, cost the W1 estimate.
 * timing (nullable): setup s, loop s (the reference's wall_time -
 * setup_time window, solver.py:172/:199), cost s. */
int orc_sinkhorn_1d_timed(i64 n, const double *x, i64 m, const double *y, const double *u,
                          const double *v, double eps, i64 itr_max, double tol, int stabilize,
                          double thr, i64 check_every, double *phi, double *psi, double *out_a,
                          double *out_b, double *hist, i64 *info, i64 *absorb_its, double *cost,
                          double *timing);
int orc_sinkhorn_1d(i64 n, const double *x, i64 m, const double *y, const double *u,
                    const double *v, double eps, i64 itr_max, double tol, int stabilize,
                    double thr, i64 check_every, double *phi, double *psi, double *out_a,
                    double *out_b, double *hist, i64 *info, i64 *absorb_its, double *cost) {
    return orc_sinkhorn_1d_timed(n, x, m, y, u, v, eps, itr_max, tol, stabilize, thr,
                                 check_every, phi, psi, out_a, out_b, hist, info, absorb_its,
                                 cost, NULL);
}

int orc_sinkhorn_1d_timed(i64 n, const double *x, i64 m, const double *y, const double *u,
                          const double *v, double eps, i64 itr_max, double tol, int stabilize,
                          double thr, i64 check_every, double *phi, double *psi, double *out_a,
                          double *out_b, double *hist, i64 *info, i64 *absorb_its, double *cost,
                          double *timing) {
    double t0 = now_s();
    if (n < 1 || m < 1 || !(eps > 0) || !isfinite(eps) || itr_max < 1) return ST_BADARG;
    ad1_t ad;
    memset(&ad, 0, sizeof(ad));
    ad.x = x; ad.y = y; ad.n = n; ad.m = m; ad.eps = eps; ad.a = out_a; ad.b = out_b;
    for (i64 i = 0; i < n; ++i) out_a[i] = 0.0;
    for (i64 j = 0; j < m; ++j) out_b[j] = 0.0;
    if (op1_assemble(&ad.op, x, n, y, m, eps, out_a, out_b)) return ST_BADARG;
    ad.t = malloc(sizeof(double) * m); ad.qm = malloc(sizeof(double) * m);
    ad.s = malloc(sizeof(double) * n); ad.qn = malloc(sizeof(double) * n);
    cfg_t c = {eps, itr_max, tol, stabilize, thr, check_every};
    double t1 = now_s();
    int st = run_driver(&ad, ad1_iterate, ad1_absorb, u, n, v, m, &c, phi, psi, hist, info,
                        absorb_its);
    double t2 = now_s();
    *cost = st == ST_OK ? cost_1d(&ad.op, x, y, phi, psi) : NAN;
    double t3 = now_s();
    if (timing) { timing[0] = t1 - t0; timing[1] = t2 - t1; timing[2] = t3 - t2; }
    op1_free(&ad.op);
    free(ad.t); free(ad.qm); free(ad.s); free(ad.qn);
    return st;
}

/* kernel1d.apply / apply_transpose / apply_blocks with shifts a, b
 * (kernel1d.py:284-310).  mode 0: out = K' vin (len n), 1: out = K'^T vin
 * (len m), 2: (out, out2) = (K'_L vin, K'_U vin) (len n). */
int orc_apply_1d(i64 n, const double *x, i64 m, const double *y, double eps, const double *a,
                 const double *b, const double *vin, int mode, double *out, double *out2) {
    op1_t op;
    double *za = NULL, *zb = NULL;
    if (!a) { za = calloc(n, sizeof(double)); a = za; }
    if (!b) { zb = calloc(m, sizeof(double)); b = zb; }
    if (op1_assemble(&op, x, n, y, m, eps, a, b)) return ST_BADARG;
    if (mode == 0)
        dp_scan(op.zf, n, op.lo.ratios, op.up.ratios, op.lo.edges, op.up.edges, vin, m, out, 0, 0);
    else if (mode == 1)
        dp_scan(op.zt, m, op.tlo.ratios, op.tup.ratios, op.tlo.edges, op.tup.edges, vin, n, out, 0,
                0);
    else
        dp_scan(op.zf, n, op.lo.ratios, op.up.ratios, op.lo.edges, op.up.edges, vin, m, NULL, out,
                out2);
    op1_free(&op);
    free(za); free(zb);
    return ST_OK;
}

/* transport_cost_fast for a given state (solver.py:252-271). */
int orc_cost_1d(i64 n, const double *x, i64 m, const double *y, double eps, const double *a,
                const double *b, const double *phi, const double *psi, double *cost) {
    op1_t op;
    if (op1_assemble(&op, x, n, y, m, eps, a, b)) return ST_BADARG;
    *cost = cost_1d(&op, x, y, phi, psi);
    op1_free(&op);
    return ST_OK;
}

/* Batch of independent 1D problems (no reference equivalent; per-problem
 * semantics = sinkhorn_1d).  Problem p uses x[xoff[p]..xoff[p+1]) etc. */
int orc_sinkhorn_1d_batch(i64 P, const i64 *xoff, const double *x, const i64 *yoff,
                          const double *y, const double *u, const double *v, const double *eps,
                          i64 itr_max, double tol, int stabilize, double thr, i64 check_every,
                          double *phi, double *psi, double *a, double *b, double *hist, i64 *info,
                          double *cost) {
    int worst = ST_OK;
    for (i64 p = 0; p < P; ++p) {
        i64 x0 = xoff[p], n = xoff[p + 1] - x0, y0 = yoff[p], m = yoff[p + 1] - y0;
        int s = orc_sinkhorn_1d(n, x + x0, m, y + y0, u + x0, v + y0, eps[p], itr_max, tol,
                                stabilize, thr, check_every, phi + x0, psi + y0, a + x0, b + y0,
                                hist + p * itr_max, info + p * 5, NULL, cost + p);
        if (s > worst) worst = s;
    }
    return worst;
}

/* ---------------------------- 2D solver ----------------------------- */
/* Arrays are Fortran ordered: A[k + j*rows]. */
typedef struct {
    i64 n1, m1, n2, m2;
    double eps, inv_eps;
    op1_t kx, ky;       /* shift-free factors (kernel2d.py:99-109) */
    double *A, *B;      /* shift grids; NULL until first absorb */
    double *S1, *T2, *S2, *T1, *rin, *rout;
} ad2_t;

#define AT(M, k, j, rows) ((M)[(k) + (i64)(j) * (rows)])

static itres_t epi_2d(const double *W, double *SC, const double *T, i64 rows, i64 cols,
                      double *err_acc, int with_err, double *mx, double *mn) {
    itres_t R = {0.0, ST_OK, 0, 0, 0, 0};
    double err = err_acc ? *err_acc : 0.0, vmax = 0.0, vmin = INFINITY;
    for (i64 j = 0; j < cols; ++j) {
        for (i64 k = 0; k < rows; ++k) {
            double w = AT(W, k, j, rows), t = AT(T, k, j, rows);
            if (with_err) err += fabs(AT(SC, k, j, rows) * t - w);
            if (t == 0.0) {
                if (w > 0.0) { R.status = ST_ZERO_DENOM; goto out; }
                AT(SC, k, j, rows) = 0.0;
            } else {
                double q = w / t;
                if (!isfinite(q)) { R.status = ST_NONFINITE; goto out; }
                AT(SC, k, j, rows) = q;
                if (w > 0.0) {
                    if (q > vmax) vmax = q;
                    if (q < vmin) vmin = q;
                }
            }
        }
    }
out:
    if (err_acc) *err_acc = err;
    *mx = vmax; *mn = vmin;
    return R;
}

/* _kernels.py:353-428 (baked) and :431-521 (dyn) */
static itres_t ad2_iterate(void *p, const double *u, const double *v, double *phi, double *psi) {
    ad2_t *ad = (ad2_t *)p;
    i64 n1 = ad->n1, m1 = ad->m1, n2 = ad->n2, m2 = ad->m2;
    itres_t R = {0.0, ST_OK, 0, 0, 0, 0};
    const op1_t *kx = &ad->kx, *ky = &ad->ky;
    double inv = ad->inv_eps;
    int dyn = ad->A != NULL;
    double *zero = calloc((size_t)(n1 > n2 ? n1 : n2) + (size_t)(m1 > m2 ? m1 : m2) + 1, sizeof(double));
    /* half A: S1[:,j] = Kx^T PHI[:,j]; T2[k,:] = Ky^T S1[k,:] */
    for (i64 j = 0; j < m1; ++j) {
        if (!dyn)
            dp_scan(kx->zt, n2, kx->tlo.ratios, kx->tup.ratios, kx->tlo.edges, kx->tup.edges,
                    &AT(phi, 0, j, n1), n1, &AT(ad->S1, 0, j, n2), 0, 0);
        else
            dp_scan_dyn(kx->zt, n2, kx->tlo.gaps, kx->tlo.dist, kx->tup.dist, zero,
                        &AT(ad->A, 0, j, n1), inv, &AT(phi, 0, j, n1), n1, &AT(ad->S1, 0, j, n2),
                        0, 0);
    }
    double *babs = malloc(sizeof(double) * (m1 > m2 ? m1 : m2));
    for (i64 k = 0; k < n2; ++k) {
        for (i64 j = 0; j < m1; ++j) ad->rin[j] = AT(ad->S1, k, j, n2);
        if (!dyn)
            dp_scan(ky->zt, m2, ky->tlo.ratios, ky->tup.ratios, ky->tlo.edges, ky->tup.edges,
                    ad->rin, m1, ad->rout, 0, 0);
        else {
            for (i64 j = 0; j < m2; ++j) babs[j] = AT(ad->B, k, j, n2);
            dp_scan_dyn(ky->zt, m2, ky->tlo.gaps, ky->tlo.dist, ky->tup.dist, babs, zero, inv,
                        ad->rin, m1, ad->rout, 0, 0);
        }
        for (i64 j = 0; j < m2; ++j) AT(ad->T2, k, j, n2) = ad->rout[j];
    }
    double err = 0.0;
    itres_t e = epi_2d(v, psi, ad->T2, n2, m2, &err, 1, &R.psmax, &R.psmin);
    R.err = err;
    if (e.status) { R.status = e.status; R.psmax = R.psmin = 0; goto done; }
    /* half B: S2[:,j] = Kx PSI[:,j]; T1[k,:] = Ky S2[k,:] */
    for (i64 j = 0; j < m2; ++j) {
        if (!dyn)
            dp_scan(kx->zf, n1, kx->lo.ratios, kx->up.ratios, kx->lo.edges, kx->up.edges,
                    &AT(psi, 0, j, n2), n2, &AT(ad->S2, 0, j, n1), 0, 0);
        else
            dp_scan_dyn(kx->zf, n1, kx->lo.gaps, kx->lo.dist, kx->up.dist, zero,
                        &AT(ad->B, 0, j, n2), inv, &AT(psi, 0, j, n2), n2, &AT(ad->S2, 0, j, n1),
                        0, 0);
    }
    for (i64 k = 0; k < n1; ++k) {
        for (i64 j = 0; j < m2; ++j) ad->rin[j] = AT(ad->S2, k, j, n1);
        if (!dyn)
            dp_scan(ky->zf, m1, ky->lo.ratios, ky->up.ratios, ky->lo.edges, ky->up.edges, ad->rin,
                    m2, ad->rout, 0, 0);
        else {
            for (i64 j = 0; j < m1; ++j) babs[j] = AT(ad->A, k, j, n1);
            dp_scan_dyn(ky->zf, m1, ky->lo.gaps, ky->lo.dist, ky->up.dist, babs, zero, inv,
                        ad->rin, m2, ad->rout, 0, 0);
        }
        for (i64 j = 0; j < m1; ++j) AT(ad->T1, k, j, n1) = ad->rout[j];
    }
    e = epi_2d(u, phi, ad->T1, n1, m1, NULL, 0, &R.phmax, &R.phmin);
    if (e.status) { R.status = e.status; R.psmax = R.psmin = R.phmax = R.phmin = 0; }
done:
    free(babs);
    free(zero);
    return R;
}

/* kernel2d.py:261-275 absorb_2d + :355-360 */
static int ad2_absorb(void *p, const double *da, const double *db) {
    ad2_t *ad = (ad2_t *)p;
    i64 N1 = ad->n1 * ad->m1, N2 = ad->n2 * ad->m2;
    if (!ad->A) { ad->A = calloc(N1, sizeof(double)); ad->B = calloc(N2, sizeof(double)); }
    for (i64 i = 0; i < N1; ++i) ad->A[i] = ad->A[i] + da[i];
    for (i64 i = 0; i < N2; ++i) ad->B[i] = ad->B[i] + db[i];
    return ST_OK;
}

/* kernel2d.py:394-465 transport_cost_fast_2d */
static double cost_2d(ad2_t *ad, const double *x1, const double *x2, const double *y1,
                      const double *y2, const double *phi, const double *psi) {
    i64 n1 = ad->n1, m1 = ad->m1, n2 = ad->n2, m2 = ad->m2;
    double inv = ad->inv_eps;
    const op1_t *kx = &ad->kx, *ky = &ad->ky;
    double *A = ad->A ? ad->A : calloc(n1 * m1, sizeof(double));
    double *B = ad->B ? ad->B : calloc(n2 * m2, sizeof(double));
    i64 big = n1 + n2 + m1 + m2 + 1;
    double *zero = calloc(big, sizeof(double));
    double *S = malloc(sizeof(double) * n1 * m2), *Rt = malloc(sizeof(double) * m1 * n2);
    double *row = malloc(sizeof(double) * big), *brow = malloc(sizeof(double) * big);
    for (i64 j = 0; j < m2; ++j)
        dp_scan_dyn(kx->zf, n1, kx->lo.gaps, kx->lo.dist, kx->up.dist, zero, &AT(B, 0, j, n2), inv,
                    &AT(psi, 0, j, n2), n2, &AT(S, 0, j, n1), 0, 0);
    for (i64 l = 0; l < n2; ++l) {
        for (i64 j = 0; j < m2; ++j) { row[j] = AT(psi, l, j, n2); brow[j] = AT(B, l, j, n2); }
        dp_scan_dyn(ky->zf, m1, ky->lo.gaps, ky->lo.dist, ky->up.dist, zero, brow, inv, row, m2,
                    &AT(Rt, 0, l, m1), 0, 0);
    }
    double *p = malloc(sizeof(double) * big), *q = malloc(sizeof(double) * big);
    double *pt = malloc(sizeof(double) * big), *qt = malloc(sizeof(double) * big);
    double *w = malloc(sizeof(double) * big), *w2 = malloc(sizeof(double) * big);
    double *ak = malloc(sizeof(double) * big);
    double xc = 0.0;
    for (i64 i = 0; i < m1; ++i) {
        for (i64 l = 0; l < n2; ++l) { w[l] = AT(Rt, i, l, m1); w2[l] = x2[l] * w[l]; }
        dp_scan_dyn(kx->zf, n1, kx->lo.gaps, kx->lo.dist, kx->up.dist, &AT(A, 0, i, n1), zero, inv,
                    w, n2, NULL, p, q);
        dp_scan_dyn(kx->zf, n1, kx->lo.gaps, kx->lo.dist, kx->up.dist, &AT(A, 0, i, n1), zero, inv,
                    w2, n2, NULL, pt, qt);
        for (i64 k = 0; k < n1; ++k)
            w[k] = AT(phi, k, i, n1) * (x1[k] * (p[k] - q[k]) - pt[k] + qt[k]);
        xc += pairwise_sum(w, n1);
    }
    double yc = 0.0;
    for (i64 k = 0; k < n1; ++k) {
        for (i64 j = 0; j < m2; ++j) { w[j] = AT(S, k, j, n1); w2[j] = y2[j] * w[j]; }
        for (i64 j = 0; j < m1; ++j) ak[j] = AT(A, k, j, n1);
        dp_scan_dyn(ky->zf, m1, ky->lo.gaps, ky->lo.dist, ky->up.dist, ak, zero, inv, w, m2, NULL,
                    p, q);
        dp_scan_dyn(ky->zf, m1, ky->lo.gaps, ky->lo.dist, ky->up.dist, ak, zero, inv, w2, m2, NULL,
                    pt, qt);
        for (i64 j = 0; j < m1; ++j)
            w[j] = AT(phi, k, j, n1) * (y1[j] * (p[j] - q[j]) - pt[j] + qt[j]);
        yc += pairwise_sum(w, m1);
    }
    if (!ad->A) free(A);
    if (!ad->B) free(B);
    free(zero); free(S); free(Rt); free(row); free(brow);
    free(p); free(q); free(pt); free(qt); free(w); free(w2); free(ak);
    return xc + yc;
}

/* kernel2d.py:363-391 sinkhorn_2d.  Grids: source (x1[n1], y1[m1]),
 * target (x2[n2], y2[m2]); U (n1 x m1), V (n2 x m2) Fortran ordered.
 * out_A/out_B receive the flattened (column-major) shift grids. */
int orc_sinkhorn_2d(i64 n1, const double *x1, i64 m1, const double *y1, i64 n2,
                    const double *x2, i64 m2, const double *y2, const double *U, const double *V,
                    double eps, i64 itr_max, double tol, int stabilize, double thr,
                    i64 check_every, double *phi, double *psi, double *out_A, double *out_B,
                    double *hist, i64 *info, i64 *absorb_its, double *cost) {
    ad2_t ad;
    memset(&ad, 0, sizeof(ad));
    ad.n1 = n1; ad.m1 = m1; ad.n2 = n2; ad.m2 = m2; ad.eps = eps; ad.inv_eps = 1.0 / eps;
    double *z1 = calloc(n1 + m1 + n2 + m2, sizeof(double));
    if (op1_assemble(&ad.kx, x1, n1, x2, n2, eps, z1, z1)) return ST_BADARG;
    if (op1_assemble(&ad.ky, y1, m1, y2, m2, eps, z1, z1)) return ST_BADARG;
    ad.S1 = malloc(sizeof(double) * n2 * m1); ad.T2 = malloc(sizeof(double) * n2 * m2);
    ad.S2 = malloc(sizeof(double) * n1 * m2); ad.T1 = malloc(sizeof(double) * n1 * m1);
    i64 big = (m1 > m2 ? m1 : m2) + 1;
    ad.rin = malloc(sizeof(double) * big); ad.rout = malloc(sizeof(double) * big);
    cfg_t c = {eps, itr_max, tol, stabilize, thr, check_every};
    int st = run_driver(&ad, ad2_iterate, ad2_absorb, U, n1 * m1, V, n2 * m2, &c, phi, psi, hist,
                        info, absorb_its);
    for (i64 i = 0; i < n1 * m1; ++i) out_A[i] = ad.A ? ad.A[i] : 0.0;
    for (i64 i = 0; i < n2 * m2; ++i) out_B[i] = ad.B ? ad.B[i] : 0.0;
    *cost = st == ST_OK ? cost_2d(&ad, x1, x2, y1, y2, phi, psi) : NAN;
    op1_free(&ad.kx); op1_free(&ad.ky);
    free(ad.A); free(ad.B); free(ad.S1); free(ad.T2); free(ad.S2); free(ad.T1);
    free(ad.rin); free(ad.rout); free(z1);
    return st;
}

/* transport_cost_fast_2d for a given state (kernel2d.py:394-465). */
int orc_cost_2d(i64 n1, const double *x1, i64 m1, const double *y1, i64 n2, const double *x2,
                i64 m2, const double *y2, double eps, const double *A, const double *B,
                const double *phi, const double *psi, double *cost) {
    ad2_t ad;
    memset(&ad, 0, sizeof(ad));
    ad.n1 = n1; ad.m1 = m1; ad.n2 = n2; ad.m2 = m2; ad.eps = eps; ad.inv_eps = 1.0 / eps;
    double *z1 = calloc(n1 + m1 + n2 + m2, sizeof(double));
    op1_assemble(&ad.kx, x1, n1, x2, n2, eps, z1, z1);
    op1_assemble(&ad.ky, y1, m1, y2, m2, eps, z1, z1);
    ad.A = (double *)A; ad.B = (double *)B;
    *cost = cost_2d(&ad, x1, x2, y1, y2, phi, psi);
    op1_free(&ad.kx); op1_free(&ad.ky); free(z1);
    return ST_OK;
}
