/*
 * c_solve.c -- a C host program driving libpmg.so through include/pmg.h
 * only (no Python): what a C / Fortran model would do to replace the
 * reference's Python solver (multigrid.mg_solve / krylov.pcg_solve).
 *
 *   c_solve in.bin out.bin
 *
 * in.bin (native endianness):
 *   int32  nx, ny, nz, nlev, periodic, maxiter, solver (0 MG, 1 CG+SSOR)
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

    FILE *out = fopen(argv[2], "wb");
    if (!out) return 2;
    int res[2] = {iters, conv};
    fwrite(res, sizeof(int), 2, out);
    fwrite(hist, sizeof(double), iters + 1, out);
    fwrite(u_host, sizeof(double), n, out);
    fclose(out);
    printf("%s: %d iterations, converged %d, |r|/|r0| = %.3e\n", solver ? "cg" : "mg", iters,
           conv, hist[iters] / hist[0]);

    for (int l = 0; l < nlev; ++l) pmg_level_destroy(lv[l]);
    cudaFree(f); cudaFree(u); cudaFree(staging);
    free(f_host); free(u_host); free(hist);
    return 0;
}
