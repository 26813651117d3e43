/*
 * oracle.c -- C restatement of the reference solver path (CPU, OpenMP).
 *
 * TEST INFRASTRUCTURE / CPU BASELINE ONLY.  The product (libpmg.so) never
 * links or calls this.  It restates, per cell and in the reference's
 * operation order, the numpy code of panelmg:
 *   apply / residual      stencil.py:127-165   (diag3 stencil.py:105-109)
 *   half sweep            smoother.py:122-182  (pivots smoother.py:89-99)
 *   halo exchange         partition.py:158-191 (P = 1, periodic or mirror)
 *   restrict / prolong    multigrid.py:209-246
 *   V-cycle / mg_solve    multigrid.py:271-330
 *   pcg_solve             krylov.py:88-167 with ssor_apply smoother.py:224-244
 * and keeps the reference's N-sized caches (diag3, vband, invd).  Built
 * with -ffp-contract=off so every product and sum rounds like numpy.
 * Parity is pinned against oracle/port.py and the reference goldens in
 * tests/test_oracle_c.py.
 *
 * Field layout = reference Field (field.py:3-10): (nx+2) x (ny+2) x nz,
 * k fastest, one-cell halo ring.
 */
#include <math.h>
#include <omp.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

typedef struct {
    int nx, ny, nz;
    double omega2, vcoef;
    const double *wx, *wy, *av, *vh, *sumw; /* (nx+1,ny) (nx,ny+1) (nx,ny) C-order */
    const double *dr, *vprof, *volprof;
} or_level_desc;

typedef struct {
    int nx, ny, nz;
    double omega2, vcoef;
    double *wx, *wy, *av, *sumw, *vh;
    double *dr, *vprof, *volprof, *drw;
    double *diag3, *vband, *invd; /* (nx, ny, nz), (nx, ny, nz-1), (nx, ny, nz);
                                     NULL in lean mode (recomputed per column) */
    double *u, *f, *r;            /* scratch fields with halo */
} level_t;

typedef struct {
    int nlev, px, py;
    level_t *lv;
} hier_t;

#define OR_MAXT 512
static int or_nthreads(void) {
    const int n = omp_get_max_threads();
    return n < OR_MAXT ? n : OR_MAXT;
}

#define IDX(L, i, j, k) ((((size_t)(i)) * ((L)->ny + 2) + (size_t)(j)) * (L)->nz + (size_t)(k))

static size_t fsize(const level_t *L) { return (size_t)(L->nx + 2) * (L->ny + 2) * L->nz; }

static double *dup(const double *a, size_t n) {
    double *b = (double *)malloc(n * sizeof(double));
    memcpy(b, a, n * sizeof(double));
    return b;
}

/* diag3 / vband / invd of column q (stencil.py:105-109, stencil.py:79-81,
 * smoother.py:93-99), in the reference's expression order */
static void column_coefs(const level_t *L, size_t q, double *dg, double *vb, double *iv) {
    const int nz = L->nz;
    const double vh = L->vh[q], osw = L->omega2 * L->sumw[q], cv = L->vcoef * L->av[q];
    for (int k = 0; k < nz; ++k) {
        const double t1 = vh * L->volprof[k];
        const double t2 = osw * L->dr[k];
        const double t3 = cv * (L->vprof[k] + L->vprof[k + 1]);
        dg[k] = (t1 + t2) + t3;
    }
    for (int k = 1; k < nz; ++k) vb[k - 1] = cv * L->vprof[k];
    iv[0] = 1.0 / dg[0];
    for (int k = 1; k < nz; ++k) {
        const double sk = L->vprof[k] * cv;
        const double m = (sk * sk) * iv[k - 1];
        iv[k] = 1.0 / (dg[k] - m);
    }
}

static void level_init(level_t *L, const or_level_desc *d, int lean) {
    const int nx = d->nx, ny = d->ny, nz = d->nz;
    L->nx = nx; L->ny = ny; L->nz = nz;
    L->omega2 = d->omega2; L->vcoef = d->vcoef;
    L->wx = dup(d->wx, (size_t)(nx + 1) * ny);
    L->wy = dup(d->wy, (size_t)nx * (ny + 1));
    L->av = dup(d->av, (size_t)nx * ny);
    L->sumw = dup(d->sumw, (size_t)nx * ny);
    L->dr = dup(d->dr, nz);
    L->vprof = dup(d->vprof, nz + 1);
    L->vh = dup(d->vh, (size_t)nx * ny);
    L->volprof = dup(d->volprof, nz);
    L->drw = (double *)malloc(nz * sizeof(double));
    for (int k = 0; k < nz; ++k) L->drw[k] = d->omega2 * d->dr[k];
    const size_t N = (size_t)nx * ny * nz;
    L->diag3 = L->vband = L->invd = NULL;
    if (!lean) {
        /* the reference's N-sized caches (stencil.py:90-114, smoother.py:56-99) */
        L->diag3 = (double *)malloc(N * sizeof(double));
        L->vband = (double *)malloc((size_t)nx * ny * (nz > 1 ? nz - 1 : 1) * sizeof(double));
        L->invd = (double *)malloc(N * sizeof(double));
#pragma omp parallel for schedule(static)
        for (int i = 0; i < nx; ++i)
            for (int j = 0; j < ny; ++j) {
                const size_t q = (size_t)i * ny + j;
                column_coefs(L, q, L->diag3 + q * nz, L->vband + q * (nz > 1 ? nz - 1 : 1),
                             L->invd + q * nz);
            }
    }
    L->u = (double *)calloc(fsize(L), sizeof(double));
    L->f = (double *)calloc(fsize(L), sizeof(double));
    L->r = (double *)calloc(fsize(L), sizeof(double));
}

static void level_free(level_t *L) {
    free(L->wx); free(L->wy); free(L->av); free(L->sumw); free(L->dr); free(L->vprof);
    free(L->vh); free(L->volprof);
    free(L->drw); free(L->diag3); free(L->vband); free(L->invd);
    free(L->u); free(L->f); free(L->r);
}

/* partition.py:158-191 with one worker (periodic = Appendix B wrap) */
static void halo(const level_t *L, double *d, int px, int py) {
    const int m = L->nx, n = L->ny, nz = L->nz;
#pragma omp parallel for schedule(static)
    for (int j = 1; j <= n; ++j) {
        memcpy(d + IDX(L, 0, j, 0), d + IDX(L, px ? m : 1, j, 0), nz * sizeof(double));
        memcpy(d + IDX(L, m + 1, j, 0), d + IDX(L, px ? 1 : m, j, 0), nz * sizeof(double));
    }
#pragma omp parallel for schedule(static)
    for (int i = 0; i <= m + 1; ++i) {
        memcpy(d + IDX(L, i, 0, 0), d + IDX(L, i, py ? n : 1, 0), nz * sizeof(double));
        memcpy(d + IDX(L, i, n + 1, 0), d + IDX(L, i, py ? 1 : n, 0), nz * sizeof(double));
    }
}

/* stencil.py:140-156 (+ 162-164 when f != NULL); returns sum r^2 if norm */
static double apply_op(const level_t *L, const double *u, const double *f, double *out,
                       int norm) {
    const int nx = L->nx, ny = L->ny, nz = L->nz;
    double part[OR_MAXT];
    int nt = 1;
#pragma omp parallel num_threads(or_nthreads())
    {
    const int t = omp_get_thread_num();
    if (t == 0) nt = omp_get_num_threads();
    double s2 = 0.0;
    double *cb = L->diag3 ? NULL : (double *)malloc(3 * (size_t)nz * sizeof(double));
#pragma omp for schedule(static)
    for (int i = 0; i < nx; ++i)
        for (int j = 0; j < ny; ++j) {
            const size_t q = (size_t)i * ny + j;
            const double wxm = L->wx[(size_t)i * ny + j], wxp = L->wx[(size_t)(i + 1) * ny + j];
            const double wym = L->wy[(size_t)i * (ny + 1) + j], wyp = L->wy[(size_t)i * (ny + 1) + j + 1];
            const double *uc = u + IDX(L, i + 1, j + 1, 0);
            const double *uw = u + IDX(L, i, j + 1, 0), *ue = u + IDX(L, i + 2, j + 1, 0);
            const double *us = u + IDX(L, i + 1, j, 0), *un = u + IDX(L, i + 1, j + 2, 0);
            const double *dg, *vb;
            if (cb) {
                column_coefs(L, q, cb, cb + nz, cb + 2 * nz);
                dg = cb;
                vb = cb + nz;
            } else {
                dg = L->diag3 + q * nz;
                vb = L->vband + q * (nz - 1);
            }
            double *o = out ? out + IDX(L, i + 1, j + 1, 0) : NULL;
            const double *fc = f ? f + IDX(L, i + 1, j + 1, 0) : NULL;
            for (int k = 0; k < nz; ++k) {
                double acc = wxm * uw[k];
                acc = acc + wxp * ue[k];
                acc = acc + wym * us[k];
                acc = acc + wyp * un[k];
                acc = acc * L->drw[k];
                double res = dg[k] * uc[k] - acc;
                if (k >= 1) res = res - vb[k - 1] * uc[k - 1];
                if (k + 1 < nz) res = res - vb[k] * uc[k + 1];
                if (fc) res = fc[k] - res;
                if (o) o[k] = res;
                if (norm) s2 += res * res;
            }
        }
    free(cb);
    part[t] = s2;
    }
    double s2 = 0.0;
    for (int t = 0; t < nt; ++t) s2 += part[t];
    return s2;
}

/* smoother.py:122-170 for every column of one colour */
static void half_sweep(const level_t *L, double *u, const double *f, int color, double rho,
                       int zero_start, int nbr_zero, double post_scale) {
    const int nx = L->nx, ny = L->ny, nz = L->nz;
    const double *vp = L->vprof;
#pragma omp parallel
    {
        double *g = (double *)malloc(nz * sizeof(double));
        double *cb = L->invd ? NULL : (double *)malloc(3 * (size_t)nz * sizeof(double));
#pragma omp for schedule(static)
        for (int i = 0; i < nx; ++i)
            for (int j = 0; j < ny; ++j) {
                if (((i + j) & 1) != color) continue;
                const size_t q = (size_t)i * ny + j;
                const double cv = L->vcoef * L->av[q];
                const double *iv;
                if (cb) {
                    column_coefs(L, q, cb, cb + nz, cb + 2 * nz);
                    iv = cb + 2 * nz;
                } else {
                    iv = L->invd + q * nz;
                }
                const double *fc = f + IDX(L, i + 1, j + 1, 0);
                double *uc = u + IDX(L, i + 1, j + 1, 0);
                if (nbr_zero) {
                    for (int k = 0; k < nz; ++k) g[k] = fc[k];
                } else {
                    const double wxm = L->wx[(size_t)i * ny + j], wxp = L->wx[(size_t)(i + 1) * ny + j];
                    const double wym = L->wy[(size_t)i * (ny + 1) + j];
                    const double wyp = L->wy[(size_t)i * (ny + 1) + j + 1];
                    const double *uw = u + IDX(L, i, j + 1, 0), *ue = u + IDX(L, i + 2, j + 1, 0);
                    const double *us = u + IDX(L, i + 1, j, 0), *un = u + IDX(L, i + 1, j + 2, 0);
                    for (int k = 0; k < nz; ++k) {
                        double t = wxm * uw[k];
                        t = t + wxp * ue[k];
                        t = t + wym * us[k];
                        t = t + wyp * un[k];
                        t = t * L->drw[k];
                        g[k] = t + fc[k];
                    }
                }
                g[0] = g[0] * iv[0];
                for (int k = 1; k < nz; ++k) {
                    double t = g[k - 1] * cv;
                    t = t * vp[k];
                    g[k] = g[k] + t;
                    g[k] = g[k] * iv[k];
                }
                for (int k = nz - 2; k >= 0; --k) {
                    double t = g[k + 1] * cv;
                    t = t * vp[k + 1];
                    t = t * iv[k];
                    g[k] = g[k] + t;
                }
                if (zero_start) {
                    const double sc = rho * post_scale;
                    if (sc != 1.0)
                        for (int k = 0; k < nz; ++k) g[k] = g[k] * sc;
                } else if (rho != 1.0) {
                    const double omr = 1.0 - rho;
                    for (int k = 0; k < nz; ++k) g[k] = g[k] * rho + omr * uc[k];
                }
                memcpy(uc, g, nz * sizeof(double));
            }
        free(g);
        free(cb);
    }
}

static void sweep(const level_t *L, double *u, const double *f, int n, double rho, int px,
                  int py) {
    for (int s = 0; s < n; ++s) {
        half_sweep(L, u, f, 0, rho, 0, 0, 1.0);
        halo(L, u, px, py);
        half_sweep(L, u, f, 1, rho, 0, 0, 1.0);
        halo(L, u, px, py);
    }
}

/* multigrid.py:209-214, weight 1 */
static void restrict_sum(const level_t *F, const double *r, const level_t *Cl, double *cf) {
    const int nz = F->nz;
#pragma omp parallel for schedule(static)
    for (int I = 0; I < Cl->nx; ++I)
        for (int J = 0; J < Cl->ny; ++J) {
            const double *a = r + IDX(F, 2 * I + 1, 2 * J + 1, 0), *b = r + IDX(F, 2 * I + 2, 2 * J + 1, 0);
            const double *c = r + IDX(F, 2 * I + 1, 2 * J + 2, 0), *d = r + IDX(F, 2 * I + 2, 2 * J + 2, 0);
            double *o = cf + IDX(Cl, I + 1, J + 1, 0);
            for (int k = 0; k < nz; ++k) {
                double s = a[k] + b[k];
                s = s + c[k];
                s = s + d[k];
                o[k] = s;
            }
        }
}

/* multigrid.py:233-246 + 287-290: u += P e */
static void prolong_add(const level_t *F, double *u, const level_t *Cl, const double *c) {
    const int nz = F->nz;
#pragma omp parallel for schedule(static)
    for (int i = 0; i < F->nx; ++i)
        for (int j = 0; j < F->ny; ++j) {
            const int I = i >> 1, J = j >> 1;
            const int dI = (i & 1) ? 1 : -1, dJ = (j & 1) ? 1 : -1;
            const double *cc = c + IDX(Cl, I + 1, J + 1, 0);
            const double *cx = c + IDX(Cl, I + 1 + dI, J + 1, 0);
            const double *cy = c + IDX(Cl, I + 1, J + 1 + dJ, 0);
            const double *cd = c + IDX(Cl, I + 1 + dI, J + 1 + dJ, 0);
            double *o = u + IDX(F, i + 1, j + 1, 0);
            for (int k = 0; k < nz; ++k) {
                double e = 9.0 * cc[k];
                e = e + 3.0 * cx[k];
                e = e + 3.0 * cy[k];
                e = e + cd[k];
                e = e * 0.0625;
                o[k] = o[k] + e;
            }
        }
}

static void v_cycle(hier_t *H, int c, int nu_pre, int nu_post, int ncs, double rho) {
    level_t *L = &H->lv[c];
    if (c + 1 < H->nlev) {
        level_t *Cl = &H->lv[c + 1];
        sweep(L, L->u, L->f, nu_pre, rho, H->px, H->py);
        apply_op(L, L->u, L->f, L->r, 0);
        restrict_sum(L, L->r, Cl, Cl->f);
        memset(Cl->u, 0, fsize(Cl) * sizeof(double));
        v_cycle(H, c + 1, nu_pre, nu_post, ncs, rho);
        prolong_add(L, L->u, Cl, Cl->u);
        halo(L, L->u, H->px, H->py);
        sweep(L, L->u, L->f, nu_post, rho, H->px, H->py);
    } else {
        sweep(L, L->u, L->f, ncs, rho, H->px, H->py);
    }
}

/* owned-cell dot product: per-thread partials over static row blocks,
 * added in thread order, so the sum does not depend on the OpenMP runtime's
 * reduction order (bit-reproducible from run to run) */
static double dot_owned(const level_t *L, const double *a, const double *b) {
    double part[OR_MAXT];
    int nt = 1;
#pragma omp parallel num_threads(or_nthreads())
    {
        const int t = omp_get_thread_num();
        if (t == 0) nt = omp_get_num_threads();
        double s = 0.0;
#pragma omp for schedule(static)
        for (int i = 0; i < L->nx; ++i)
            for (int j = 0; j < L->ny; ++j) {
                const size_t o = IDX(L, i + 1, j + 1, 0);
                for (int k = 0; k < L->nz; ++k) s += a[o + k] * b[o + k];
            }
        part[t] = s;
    }
    double s = 0.0;
    for (int t = 0; t < nt; ++t) s += part[t];
    return s;
}

static double norm2_owned(const level_t *L, const double *a) { return dot_owned(L, a, a); }

static double now(void) {
    struct timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return ts.tv_sec + 1e-9 * ts.tv_nsec;
}

static void load_owned(const level_t *L, double *d, const double *src) {
#pragma omp parallel for schedule(static)
    for (int i = 0; i < L->nx; ++i)
        for (int j = 0; j < L->ny; ++j)
            memcpy(d + IDX(L, i + 1, j + 1, 0), src + ((size_t)i * L->ny + j) * L->nz,
                   L->nz * sizeof(double));
}

static void store_owned(const level_t *L, const double *d, double *dst) {
#pragma omp parallel for schedule(static)
    for (int i = 0; i < L->nx; ++i)
        for (int j = 0; j < L->ny; ++j)
            memcpy(dst + ((size_t)i * L->ny + j) * L->nz, d + IDX(L, i + 1, j + 1, 0),
                   L->nz * sizeof(double));
}

int or_threads(void) { return omp_get_max_threads(); }

/* lean != 0: no N-sized coefficient caches; diag3 / vband / invd are
 * recomputed per column with the same expressions (identical values, about
 * half the memory: the configs[4] parity check at 4096^2 x 128) */
void *or_hier_create_lean(int nlev, const or_level_desc *d, int px, int py, int lean) {
    hier_t *H = (hier_t *)calloc(1, sizeof(hier_t));
    H->nlev = nlev;
    H->px = px;
    H->py = py;
    H->lv = (level_t *)calloc(nlev, sizeof(level_t));
    for (int c = 0; c < nlev; ++c) level_init(&H->lv[c], &d[c], lean);
    return H;
}

void *or_hier_create(int nlev, const or_level_desc *d, int px, int py) {
    return or_hier_create_lean(nlev, d, px, py, 0);
}

void or_hier_destroy(void *h) {
    hier_t *H = (hier_t *)h;
    if (!H) return;
    for (int c = 0; c < H->nlev; ++c) level_free(&H->lv[c]);
    free(H->lv);
    free(H);
}

/* multigrid.py:297-330.  f, u_out: (nx, ny, nz) k fastest.  hist has room
 * for maxiter+1 entries.  max_cycles > 0 truncates (baseline sampling). */
int or_mg_solve(void *h, const double *f, double *u_out, double eps, int maxiter,
                int nu_pre, int nu_post, int ncs, double rho, int max_cycles, double *hist,
                int *iters, int *converged, double *wall) {
    hier_t *H = (hier_t *)h;
    level_t *L = &H->lv[0];
    for (int c = 0; c < H->nlev; ++c) memset(H->lv[c].u, 0, fsize(&H->lv[c]) * sizeof(double));
    memset(L->f, 0, fsize(L) * sizeof(double));
    load_owned(L, L->f, f);
    const double r0 = sqrt(norm2_owned(L, L->f));
    hist[0] = r0;
    *iters = 0;
    *converged = 1;
    *wall = 0.0;
    if (r0 == 0.0) return 0;
    *converged = 0;
    const int n = (max_cycles > 0 && max_cycles < maxiter) ? max_cycles : maxiter;
    const double t0 = now();
    for (int it = 0; it < n; ++it) {
        v_cycle(H, 0, nu_pre, nu_post, ncs, rho);
        const double rn = sqrt(apply_op(L, L->u, L->f, NULL, 1));
        hist[it + 1] = rn;
        *iters = it + 1;
        if (rn / r0 < eps) {
            *converged = 1;
            break;
        }
    }
    *wall = now() - t0;
    if (u_out) store_owned(L, L->u, u_out);
    return 0;
}

/* krylov.py:88-167 with SSORPreconditioner (smoother.py:224-244) on level 0 */
int or_pcg_solve(void *h, const double *f, double *u_out, double eps, int maxiter,
                 double rho, int max_iters, double *hist, int *iters, int *converged,
                 double *wall) {
    hier_t *H = (hier_t *)h;
    level_t *L = &H->lv[0];
    const size_t n = fsize(L);
    double *u = (double *)calloc(n, sizeof(double)), *r = (double *)calloc(n, sizeof(double));
    double *z = (double *)calloc(n, sizeof(double)), *p = (double *)calloc(n, sizeof(double));
    double *q = (double *)calloc(n, sizeof(double));
    load_owned(L, r, f);
    const double r0 = sqrt(norm2_owned(L, r));
    hist[0] = r0;
    *iters = 0;
    *converged = 1;
    *wall = 0.0;
    int rc = 0;
    if (r0 == 0.0) goto done;
    *converged = 0;
    {
        const double t0 = now();
#define SSOR(zz, rr)                                                           \
    do {                                                                       \
        memset(zz, 0, n * sizeof(double));                                     \
        half_sweep(L, zz, rr, 0, rho, 1, 1, 1.0);                              \
        halo(L, zz, H->px, H->py);                                             \
        half_sweep(L, zz, rr, 1, rho, 1, 0, 2.0 - rho);                        \
        halo(L, zz, H->px, H->py);                                             \
        half_sweep(L, zz, rr, 0, rho, 0, 0, 1.0);                              \
        halo(L, zz, H->px, H->py);                                             \
    } while (0)
        SSOR(z, r);
        memcpy(p, z, n * sizeof(double));
        double kappa = 0.0;
        {
            double s = 0.0;
            s = dot_owned(L, r, z);
            kappa = s;
        }
        if (kappa <= 0.0) { rc = -3; goto done; }
        const int nmax = (max_iters > 0 && max_iters < maxiter) ? max_iters : maxiter;
        for (int it = 1; it <= nmax; ++it) {
            apply_op(L, p, NULL, q, 0);
            double pq = 0.0;
            pq = dot_owned(L, p, q);
            if (pq <= 0.0) { rc = -3; goto done; }
            const double alpha = kappa / pq, malpha = -alpha;
#pragma omp parallel for schedule(static)
            for (size_t e = 0; e < n; ++e) {
                u[e] = u[e] + alpha * p[e];
                r[e] = r[e] + malpha * q[e];
            }
            const double rn = sqrt(norm2_owned(L, r));
            hist[it] = rn;
            *iters = it;
            if (rn / r0 < eps) { *converged = 1; break; }
            SSOR(z, r);
            double kn = 0.0;
            kn = dot_owned(L, r, z);
            if (kn <= 0.0) { rc = -3; goto done; }
            const double beta = kn / kappa;
#pragma omp parallel for schedule(static)
            for (size_t e = 0; e < n; ++e) p[e] = beta * p[e] + z[e];
            kappa = kn;
        }
#undef SSOR
        *wall = now() - t0;
    }
done:
    if (u_out) store_owned(L, u, u_out);
    free(u); free(r); free(z); free(p); free(q);
    return rc;
}

/* ---- per-operation entry points (tests/test_oracle_c.py pins each one
 * against the reference's own outputs, tests/golden/ops_*.npz).  Arrays are
 * owned (nx, ny, nz) k fastest; level c's scratch fields carry the halo. */

/* stencil.py:127-165: out = A u (f == NULL) or f - A u */
int or_apply(void *h, int c, const double *u, const double *f, double *out) {
    hier_t *H = (hier_t *)h;
    level_t *L = &H->lv[c];
    memset(L->u, 0, fsize(L) * sizeof(double));
    load_owned(L, L->u, u);
    halo(L, L->u, H->px, H->py);
    if (f) {
        memset(L->f, 0, fsize(L) * sizeof(double));
        load_owned(L, L->f, f);
    }
    memset(L->r, 0, fsize(L) * sizeof(double));
    apply_op(L, L->u, f ? L->f : NULL, L->r, 0);
    store_owned(L, L->r, out);
    return 0;
}

/* smoother.py:122-182: one colour of line relaxation of u (in / out) */
int or_half_sweep(void *h, int c, double *u, const double *f, int color, double rho,
                  int zero_start, int nbr_zero, double post_scale) {
    hier_t *H = (hier_t *)h;
    level_t *L = &H->lv[c];
    memset(L->u, 0, fsize(L) * sizeof(double));
    memset(L->f, 0, fsize(L) * sizeof(double));
    load_owned(L, L->u, u);
    load_owned(L, L->f, f);
    halo(L, L->u, H->px, H->py);
    half_sweep(L, L->u, L->f, color, rho, zero_start, nbr_zero, post_scale);
    store_owned(L, L->u, u);
    return 0;
}

/* smoother.py:184-191: nsweeps red-black sweeps of u (in / out) */
int or_sweep(void *h, int c, double *u, const double *f, int nsweeps, double rho) {
    hier_t *H = (hier_t *)h;
    level_t *L = &H->lv[c];
    memset(L->u, 0, fsize(L) * sizeof(double));
    memset(L->f, 0, fsize(L) * sizeof(double));
    load_owned(L, L->u, u);
    load_owned(L, L->f, f);
    halo(L, L->u, H->px, H->py);
    sweep(L, L->u, L->f, nsweeps, rho, H->px, H->py);
    store_owned(L, L->u, u);
    return 0;
}

/* smoother.py:224-244: z = M^-1 r (symmetric line SOR from zero) */
int or_ssor(void *h, int c, const double *r, double *z, double rho) {
    hier_t *H = (hier_t *)h;
    level_t *L = &H->lv[c];
    memset(L->f, 0, fsize(L) * sizeof(double));
    load_owned(L, L->f, r);
    memset(L->u, 0, fsize(L) * sizeof(double));
    half_sweep(L, L->u, L->f, 0, rho, 1, 1, 1.0);
    halo(L, L->u, H->px, H->py);
    half_sweep(L, L->u, L->f, 1, rho, 1, 0, 2.0 - rho);
    halo(L, L->u, H->px, H->py);
    half_sweep(L, L->u, L->f, 0, rho, 0, 0, 1.0);
    store_owned(L, L->u, z);
    return 0;
}

/* multigrid.py:209-230: coarse = weight x children sum of level c's fine */
int or_restrict(void *h, int c, const double *fine, double *coarse, double weight) {
    hier_t *H = (hier_t *)h;
    level_t *L = &H->lv[c], *Cl = &H->lv[c + 1];
    memset(L->r, 0, fsize(L) * sizeof(double));
    load_owned(L, L->r, fine);
    memset(Cl->f, 0, fsize(Cl) * sizeof(double));
    restrict_sum(L, L->r, Cl, Cl->f);
    if (weight != 1.0) {
        const size_t n = fsize(Cl);
        for (size_t e = 0; e < n; ++e) Cl->f[e] = Cl->f[e] * weight;
    }
    store_owned(Cl, Cl->f, coarse);
    return 0;
}

/* multigrid.py:233-246: fine (level c) = P coarse (level c + 1) */
int or_prolong(void *h, int c, const double *coarse, double *fine) {
    hier_t *H = (hier_t *)h;
    level_t *L = &H->lv[c], *Cl = &H->lv[c + 1];
    memset(Cl->u, 0, fsize(Cl) * sizeof(double));
    load_owned(Cl, Cl->u, coarse);
    halo(Cl, Cl->u, H->px, H->py);
    memset(L->r, 0, fsize(L) * sizeof(double));
    prolong_add(L, L->r, Cl, Cl->u);
    store_owned(L, L->r, fine);
    return 0;
}
