/*
 * c_solve.c -- a C host program driving libpmg.so through include/pmg.h
 * only (no Python): what a C / Fortran model would do to replace the
 * reference's Python solver (multigrid.mg_solve / krylov.pcg_solve).
 *
 *   c_solve in.bin out.bin
 *
 * in.bin (native endianness):
 *   int32  nx, ny, nz, nlev, periodic, maxiter, solver (0 MG, 1 CG+SSOR;
 *          2 MG, 3 CG+SSOR over a 2 x 2 decomposition whose four parts
 *          this process holds: the multi-part drivers, pmg_phier_*)
 *   double eps, omega2, vcoef
 *   per level l (nx_l = nx >> l, ny_l = ny >> l):
 *     double dr[nz], vprof[nz+1], volprof[nz],
 *            wx[ny_l][nx_l+1], wy[ny_l+1][nx_l], av[ny_l][nx_l],
 *            vh[ny_l][nx_l], sumw[ny_l][nx_l]
 *   double f[nx][ny][nz]                       (reference layout, k fastest)
 * out.bin:
 *   int32 iterations, converged; double hist[iterations + 1];
 *   double u[nx][ny][nz]
 */
#include <stdio.h>
#include <stdlib.h>

#include <cuda_runtime.h>

#include "pmg.h"

#define CHECK(x)                                                              \
    do {                                                                      \
        int rc_ = (x);                                                        \
        if (rc_) {                                                            \
            fprintf(stderr, "%s failed (%d): %s\n", #x, rc_, pmg_last_error()); \
            return 1;                                                         \
        }                                                                     \
    } while (0)
#define CUDA(x)                                                               \
    do {                                                                      \
        cudaError_t e_ = (x);                                                 \
        if (e_ != cudaSuccess) {                                              \
            fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e_));          \
            return 1;                                                         \
        }                                                                     \
    } while (0)

static double *read_doubles(FILE *fp, size_t n) {
    double *a = (double *)malloc(n * sizeof(double));
    if (a && fread(a, sizeof(double), n, fp) != n) {
        free(a);
        return NULL;
    }
    return a;
}

/* out.bin: iterations, converged, the history and u (reference layout) */
static int write_result(const char *path, int iters, int conv, const double *hist,
                        const double *u_host, size_t n, int solver) {
    FILE *out = fopen(path, "wb");
    if (!out) return 2;
    int res[2] = {iters, conv};
    fwrite(res, sizeof(int), 2, out);
    fwrite(hist, sizeof(double), iters + 1, out);
    fwrite(u_host, sizeof(double), n, out);
    fclose(out);
    printf("%s: %d iterations, converged %d, |r|/|r0| = %.3e\n", (solver & 1) ? "cg" : "mg",
           iters, conv, hist[iters] / hist[0]);
    return 0;
}

/* the (rows x cols) window at (r0, c0) of a row-major array with `cols_all` columns */
static double *window(const double *a, int cols_all, int r0, int c0, int rows, int cols) {
    double *w = (double *)malloc((size_t)rows * cols * sizeof(double));
    for (int r = 0; r < rows; ++r)
        for (int c = 0; c < cols; ++c) w[(size_t)r * cols + c] = a[(size_t)(r0 + r) * cols_all + c0 + c];
    return w;
}

/* solver 2 / 3: a px x py = 2 x 2 decomposition held by this process.  Part
 * (wi, wj) -- worker wi * py + wj, as the Python LevelLayout numbers them --
 * owns columns i in [wi mx, (wi + 1) mx), j in [wj my, (wj + 1) my) of
 * every level; its neighbours wrap around (periodic) or are -1 (mirror). */
static int solve_parts(FILE *in, const int *hdr, const double *par, const char *out_path) {
    const int nx = hdr[0], ny = hdr[1], nz = hdr[2], nlev = hdr[3], periodic = hdr[4];
    const int maxiter = hdr[5], solver = hdr[6];
    enum { PX = 2, PY = 2, NP = PX * PY };
    pmg_level *lv[NP * 32];
    for (int l = 0; l < nlev; ++l) {
        const int gx = nx >> l, gy = ny >> l, mx = gx / PX, my = gy / PY;
        double *dr = read_doubles(in, nz), *vp = read_doubles(in, nz + 1);
        double *vol = read_doubles(in, nz);
        double *wx = read_doubles(in, (size_t)gy * (gx + 1));
        double *wy = read_doubles(in, (size_t)(gy + 1) * gx);
        double *av = read_doubles(in, (size_t)gy * gx), *vh = read_doubles(in, (size_t)gy * gx);
        double *sw = read_doubles(in, (size_t)gy * gx);
        if (!dr || !vp || !vol || !wx || !wy || !av || !vh || !sw) return 2;
        for (int w = 0; w < NP; ++w) {
            const int i0 = (w / PY) * mx, j0 = (w % PY) * my;
            double *pwx = window(wx, gx + 1, j0, i0, my, mx + 1);
            double *pwy = window(wy, gx, j0, i0, my + 1, mx);
            double *pav = window(av, gx, j0, i0, my, mx), *pvh = window(vh, gx, j0, i0, my, mx);
            double *psw = window(sw, gx, j0, i0, my, mx);
            pmg_level_desc d = {mx, my, nz, i0, j0, par[1], par[2], dr, vp, vol,
                                pwx, pwy, pav, pvh, psw};
            CHECK(pmg_level_create(&d, &lv[w * nlev + l]));
            free(pwx); free(pwy); free(pav); free(pvh); free(psw);
        }
        free(dr); free(vp); free(vol); free(wx); free(wy); free(av); free(vh); free(sw);
    }
    const size_t n = (size_t)nx * ny * nz;
    double *f_host = read_doubles(in, n);
    fclose(in);
    if (!f_host) return 2;
    const int mx = nx / PX, my = ny / PY;
    const size_t np_cells = (size_t)mx * my * nz;
    const long long nd = pmg_level_field_doubles(lv[0]);
    double *f[NP], *u[NP], *staging, *blk = (double *)malloc(np_cells * sizeof(double));
    CUDA(cudaMalloc((void **)&staging, np_cells * sizeof(double)));
    pmg_part_desc parts[NP];
    for (int w = 0; w < NP; ++w) {
        const int wi = w / PY, wj = w % PY;
        CUDA(cudaMalloc((void **)&f[w], nd * sizeof(double)));
        CUDA(cudaMalloc((void **)&u[w], nd * sizeof(double)));
        for (int i = 0; i < mx; ++i)          /* the part's block, reference layout */
            for (int j = 0; j < my; ++j)
                for (int k = 0; k < nz; ++k)
                    blk[((size_t)i * my + j) * nz + k] =
                        f_host[(((size_t)(wi * mx + i)) * ny + wj * my + j) * nz + k];
        CHECK(pmg_fill(lv[w * nlev], f[w], 0.0, NULL));
        CHECK(pmg_field_upload(lv[w * nlev], blk, f[w], staging, NULL));
        const int dx[4] = {-1, 1, 0, 0}, dy[4] = {0, 0, -1, 1};
        parts[w].worker = w;
        for (int a = 0; a < 4; ++a) {
            int ni = wi + dx[a], nj = wj + dy[a];
            if (periodic) {
                ni = (ni + PX) % PX;
                nj = (nj + PY) % PY;
            }
            parts[w].nbr[a] = (ni < 0 || ni >= PX || nj < 0 || nj >= PY) ? -1 : ni * PY + nj;
        }
        for (int a = 0; a < 4; ++a) {         /* SW, SE, NW, NE */
            int ni = wi + (a & 1 ? 1 : -1), nj = wj + (a & 2 ? 1 : -1);
            if (periodic) {
                ni = (ni + PX) % PX;
                nj = (nj + PY) % PY;
            }
            parts[w].diag[a] = (ni < 0 || ni >= PX || nj < 0 || nj >= PY) ? -1 : ni * PY + nj;
        }
    }
    pmg_mg_desc md = {1, 1, 1, 1.0, periodic, periodic, 1, 1};
    pmg_phier *h;
    if (solver == 2) {           /* levels[part * nlev + level] */
        CHECK(pmg_phier_create((const pmg_level *const *)lv, nlev, NP, parts, &md, NULL, 1024,
                               &h));
    } else {                     /* CG needs the finest level of each part only */
        const pmg_level *fine[NP];
        for (int w = 0; w < NP; ++w) fine[w] = lv[w * nlev];
        CHECK(pmg_phier_create(fine, 1, NP, parts, &md, NULL, 1024, &h));
    }
    double *hist = (double *)calloc(maxiter + 1, sizeof(double));
    int iters = 0, conv = 0;
    if (solver == 2)
        CHECK(pmg_phier_mg_solve(h, (const double *const *)f, u, par[0], maxiter, hist, &iters,
                                 &conv, NULL));
    else
        CHECK(pmg_phier_pcg_solve(h, (const double *const *)f, u, par[0], maxiter, 1e-300, 1, 1.0,
                                  hist, &iters, &conv, NULL));
    double *u_host = (double *)malloc(n * sizeof(double));
    for (int w = 0; w < NP; ++w) {
        const int wi = w / PY, wj = w % PY;
        CHECK(pmg_field_download(lv[w * nlev], u[w], blk, staging, NULL));
        CUDA(cudaDeviceSynchronize());
        for (int i = 0; i < mx; ++i)
            for (int j = 0; j < my; ++j)
                for (int k = 0; k < nz; ++k)
                    u_host[(((size_t)(wi * mx + i)) * ny + wj * my + j) * nz + k] =
                        blk[((size_t)i * my + j) * nz + k];
    }
    CHECK(pmg_phier_destroy(h));
    const int rc = write_result(out_path, iters, conv, hist, u_host, n, solver);
    for (int w = 0; w < NP; ++w) {
        cudaFree(f[w]);
        cudaFree(u[w]);
    }
    for (int q = 0; q < NP * nlev; ++q) pmg_level_destroy(lv[q]);
    cudaFree(staging);
    free(f_host); free(u_host); free(hist); free(blk);
    return rc;
}

int main(int argc, char **argv) {
    if (argc != 3) {
        fprintf(stderr, "usage: %s in.bin out.bin\n", argv[0]);
        return 2;
    }
    FILE *in = fopen(argv[1], "rb");
    if (!in) return 2;
    int hdr[7];
    double par[3];
    if (fread(hdr, sizeof(int), 7, in) != 7 || fread(par, sizeof(double), 3, in) != 3) return 2;
    const int nx = hdr[0], ny = hdr[1], nz = hdr[2], nlev = hdr[3], periodic = hdr[4];
    const int maxiter = hdr[5], solver = hdr[6];
    const double eps = par[0];

    if (solver >= 2) return solve_parts(in, hdr, par, argv[2]);

    pmg_level *lv[32];
    for (int l = 0; l < nlev; ++l) {
        const int mx = nx >> l, my = ny >> l;
        double *dr = read_doubles(in, nz), *vp = read_doubles(in, nz + 1);
        double *vol = read_doubles(in, nz);
        double *wx = read_doubles(in, (size_t)my * (mx + 1));
        double *wy = read_doubles(in, (size_t)(my + 1) * mx);
        double *av = read_doubles(in, (size_t)my * mx), *vh = read_doubles(in, (size_t)my * mx);
        double *sw = read_doubles(in, (size_t)my * mx);
        if (!dr || !vp || !vol || !wx || !wy || !av || !vh || !sw) return 2;
        pmg_level_desc d = {mx, my, nz, 0, 0, par[1], par[2], dr, vp, vol, wx, wy, av, vh, sw};
        CHECK(pmg_level_create(&d, &lv[l]));     /* copies the arrays */
        free(dr); free(vp); free(vol); free(wx); free(wy); free(av); free(vh); free(sw);
    }
    const size_t n = (size_t)nx * ny * nz;
    double *f_host = read_doubles(in, n);
    fclose(in);
    if (!f_host) return 2;

    /* device fields in the library's layout, staged through one buffer */
    const long long nd = pmg_level_field_doubles(lv[0]);
    double *f, *u, *staging;
    CUDA(cudaMalloc((void **)&f, nd * sizeof(double)));
    CUDA(cudaMalloc((void **)&u, nd * sizeof(double)));
    CUDA(cudaMalloc((void **)&staging, n * sizeof(double)));
    CHECK(pmg_fill(lv[0], f, 0.0, NULL));
    CHECK(pmg_field_upload(lv[0], f_host, f, staging, NULL));

    double *hist = (double *)calloc(maxiter + 1, sizeof(double));
    int iters = 0, conv = 0;
    if (solver == 0) {
        pmg_mg_desc md = {1, 1, 1, 1.0, periodic, periodic, 1, 1};   /* V(1,1), rho = 1, lagged norm, red restriction */
        pmg_hier *h;
        CHECK(pmg_hier_create((const pmg_level *const *)lv, nlev, &md, &h));
        CHECK(pmg_mg_solve(h, f, u, eps, maxiter, hist, &iters, &conv, NULL));
        CHECK(pmg_hier_destroy(h));
    } else {
        double *work;
        CUDA(cudaMalloc((void **)&work, pmg_pcg_work_doubles(lv[0]) * sizeof(double)));
        CHECK(pmg_pcg_solve(lv[0], f, u, eps, maxiter, 1e-300, 1, 1.0, periodic, periodic, work,
                            hist, &iters, &conv, NULL));
        CUDA(cudaFree(work));
    }
    double *u_host = (double *)malloc(n * sizeof(double));
    CHECK(pmg_field_download(lv[0], u, u_host, staging, NULL));
    CUDA(cudaDeviceSynchronize());

    if (write_result(argv[2], iters, conv, hist, u_host, n, solver)) return 2;

    for (int l = 0; l < nlev; ++l) pmg_level_destroy(lv[l]);
    cudaFree(f); cudaFree(u); cudaFree(staging);
    free(f_host); free(u_host); free(hist);
    return 0;
}
