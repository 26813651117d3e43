// libpmg C ABI (include/pmg.h): level set-up and the extern "C" entry points.
//
// Host-side coefficient tables are computed here in the reference's
// expression order (stencil.py:105-109, smoother.py:93-99); the host code is
// compiled with -ffp-contract=off so no FMA contraction changes a rounding.
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <algorithm>
#include <string>
#include <vector>

#include "pmg_common.cuh"
#include "pmg_trace.h"

namespace pmg {
extern std::atomic<long long> g_launches;
extern int g_smoother_exact;
extern int g_mode_gen;
cudaError_t launch_apply(const Lvl &, const double *, const double *, double *, int, double *,
                         int *, cudaStream_t);
cudaError_t launch_finalize(const double *, int, double *, cudaStream_t);
cudaError_t launch_residual_restrict(const Lvl &, const Lvl &, const double *, const double *,
                                     double *, cudaStream_t);
cudaError_t launch_half_sweep(const Lvl &, double *, const double *, int, double, int, int,
                              double, cudaStream_t);
cudaError_t launch_invd(const Lvl &, double *, cudaStream_t);
cudaError_t launch_restrict(const Lvl &, const Lvl &, const double *, double *, double,
                            cudaStream_t);
bool half_sweep_dot_ok(const Lvl &L);
bool half_sweep_res_ok(const Lvl &L);
bool half_sweep_bandv_ok(const Lvl &L);
bool residual_restrict_red_ok(const Lvl &F);
cudaError_t launch_half_sweep_fsq(const Lvl &L, double *u, const double *f, int color,
                                  int nbr_zero, double *partials, int *np, cudaStream_t st);
cudaError_t launch_residual_restrict_red(const Lvl &F, const Lvl &C, const double *u,
                                         const double *f, double *cf, cudaStream_t st,
                                         double *partials = nullptr, int *np = nullptr);
cudaError_t launch_half_sweep_res(const Lvl &L, const double *u, double *uw, const double *f,
                                  double *partials, int *np, cudaStream_t st);
cudaError_t launch_half_sweep_dot(const Lvl &L, double *u, const double *f, int color, double rho,
                                  int zero_start, int nbr_zero, double post_scale,
                                  double *partials, int *np, cudaStream_t st);
void setup_kernel_attributes();
cudaError_t launch_prolong(const Lvl &, const Lvl &, const double *, double *, int, int,
                           cudaStream_t);
cudaError_t launch_halo_self(const Lvl &, double *, int, int, cudaStream_t);
int face_len(const Lvl &, int);
cudaError_t launch_pack(const Lvl &, const double *, int, double *, cudaStream_t);
cudaError_t launch_unpack(const Lvl &, double *, int, const double *, int, cudaStream_t);
cudaError_t launch_dot(const Lvl &, const double *, const double *, double *, int *, cudaStream_t);
cudaError_t launch_axpy(long long, double, const double *, double *, cudaStream_t);
cudaError_t launch_fill(long long, double, double *, cudaStream_t);
cudaError_t launch_copy_block(const Lvl &, const double *, const Lvl &, double *, int, int, int, int,
                              int, int, cudaStream_t);
cudaError_t launch_xpby(long long, const double *, double, double *, cudaStream_t);
cudaError_t launch_cg_direction(long long, const double *, const double *, const double *,
                                double *, cudaStream_t);
cudaError_t launch_cg_update(const Lvl &, const double *, const double *, const double *,
                             const double *, double *, double *, double *, int *, cudaStream_t);
cudaError_t launch_from_ref(const Lvl &, const double *, double *, int, int, cudaStream_t);
cudaError_t launch_cg_up(long long, const double *, const double *, const double *, const double *,
                         const double *, double *, double *, cudaStream_t);
cudaError_t launch_to_ref(const Lvl &, const double *, double *, int, int, cudaStream_t);
}  // namespace pmg

using namespace pmg;

struct pmg_level {
    Lvl L;
    int i0, j0;
    std::vector<double> h_diag, h_band, h_invd;   // uniform tables (host copy)
    std::vector<double> h_seg;                    // fast solver tables
    std::vector<void *> owned;                    // device allocations to free
    double *invd_field = nullptr;                 // variable: per-cell pivots
    bool prepared = false;
};

static thread_local std::string g_err;

static int fail(int code, const std::string &msg) {
    g_err = msg;
    return code;
}

namespace pmg {
// error reporting for the other translation units of the library
int set_error(int code, const char *msg) { return fail(code, msg); }
// driver-internal view of a level whose black array lies `cstride` doubles
// from the red one (a red array in another allocation); shares the level's
// device tables, owns nothing
pmg_level *level_view(const pmg_level *lv, long long cstride, int hflags_or) {
    pmg_level *v = new pmg_level(*lv);
    v->owned.clear();
    v->L.cstride = cstride;
    v->L.hflags |= hflags_or;
    return v;
}
int level_hflags(const pmg_level *lv) { return lv->L.hflags; }
// the kernel-side view of a level (multi-part exchange kernels, pmg_parts.cu)
const Lvl &level_lvl(const pmg_level *lv) { return lv->L; }
void level_view_free(pmg_level *v) { delete v; }
}

static int cuda_fail(cudaError_t e, const char *where) {
    return fail(PMG_ERR_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

#define PMG_CHECK_LVL(l)                                                     \
    do {                                                                     \
        if (!(l)) return fail(PMG_ERR_VALUE, "null level handle");           \
    } while (0)

#define PMG_CUDA(call, where)                                                \
    do {                                                                     \
        cudaError_t e_ = (call);                                             \
        if (e_ != cudaSuccess) return cuda_fail(e_, where);                  \
    } while (0)

namespace pmg {
// rho = 1 half-sweep of a pmg_half_sweep_res_ok level that also sums f^2
// over the relaxed colour: per-CTA partials into partials[0 .. *np)
int half_sweep_fsq(const pmg_level *lv, double *u, const double *f, int color, int nbr_zero,
                   double *partials, int *np, void *st) {
    if (!lv->L.uniform && !lv->prepared) {
        int rc = pmg_level_prepare(const_cast<pmg_level *>(lv), st);
        if (rc) return rc;
    }
    PMG_CUDA(launch_half_sweep_fsq(lv->L, u, f, color, nbr_zero, partials, np, (cudaStream_t)st),
             "half_sweep_fsq");
    return PMG_OK;
}
int finalize(const double *partials, int n, double *out, void *st) {
    PMG_CUDA(launch_finalize(partials, n, out, (cudaStream_t)st), "finalize");
    return PMG_OK;
}
}  // namespace pmg

static cudaError_t upload(pmg_level *lv, const double *h, size_t n, const double **dst) {
    void *d = nullptr;
    cudaError_t e = cudaMalloc(&d, n * sizeof(double) + 8);
    if (e != cudaSuccess) return e;
    lv->owned.push_back(d);
    e = cudaMemcpy(d, h, n * sizeof(double), cudaMemcpyHostToDevice);
    *dst = (const double *)d;
    return e;
}

static bool all_equal(const double *a, size_t n) {
    for (size_t t = 1; t < n; ++t)
        if (a[t] != a[0]) return false;
    return true;
}

extern "C" {

int pmg_version(void) { return 1; }

int pmg_set_smoother_mode(int mode) {
    if (mode < 0 || mode > 1) return fail(PMG_ERR_VALUE, "smoother mode must be 0 (fast) or 1 (exact)");
    if (pmg::g_smoother_exact != mode) ++pmg::g_mode_gen;   // cached graphs / views go stale
    pmg::g_smoother_exact = mode;
    return PMG_OK;
}

int pmg_get_smoother_mode(void) { return pmg::g_smoother_exact; }

long long pmg_launch_count(void) { return g_launches.load(); }

int pmg_set_tracing(int on) {
    if (on < 0 || on > 1) return fail(PMG_ERR_VALUE, "tracing must be 0 (off) or 1 (on)");
    pmg::g_trace.store(on);
    return PMG_OK;
}

int pmg_get_tracing(void) { return pmg::g_trace.load(); }

const char *pmg_last_error(void) { return g_err.c_str(); }

int pmg_device_sm_count(int device, int *out) {
    PMG_CUDA(cudaDeviceGetAttribute(out, cudaDevAttrMultiProcessorCount, device), "sm count");
    return PMG_OK;
}

int pmg_level_create(const pmg_level_desc *d, pmg_level **out) {
    if (!d || !out) return fail(PMG_ERR_VALUE, "null argument");
    if (d->nx < 1 || d->ny < 1 || d->nz < 1)
        return fail(PMG_ERR_VALUE, "level needs nx, ny, nz >= 1");
    if (!d->dr || !d->vprof || !d->volprof || !d->wx || !d->wy || !d->av || !d->vh || !d->sumw)
        return fail(PMG_ERR_VALUE, "missing factor array");
    setup_kernel_attributes();
    const int nx = d->nx, ny = d->ny, nz = d->nz;
    auto *lv = new pmg_level();
    Lvl &L = lv->L;
    std::memset(&L, 0, sizeof(L));
    L.nx = nx;
    L.ny = ny;
    L.nz = nz;
    // row: h in [-1, nx>>1] at OFF-1 .. OFF+(nx>>1); pitch multiple of 8 doubles
    const int need = OFF + (nx >> 1) + 1;
    L.pitch = (need + 7) / 8 * 8;
    // row-major over j: a row's whole column data is one contiguous
    // nz * pitch block, so column-oriented kernels touch few 2 MB pages
    L.plane = L.pitch;
    L.jstride = (long long)nz * L.pitch;
    L.cstride = (long long)(ny + 2) * L.jstride;
    L.fcs = L.cstride;
    L.par = (d->i0 + d->j0) & 1;
    L.rx0 = 0, L.rxs = 1, L.rxn = ((nx + 1) / 2 + 31) / 32;   // whole part
    L.ry0 = 0, L.rys = 1, L.ryn = ny;
    L.omega2 = d->omega2;
    L.vcoef = d->vcoef;
    lv->i0 = d->i0;
    lv->j0 = d->j0;

    const size_t n2 = (size_t)nx * ny;
    const bool uni = all_equal(d->wx, (size_t)ny * (nx + 1)) &&
                     all_equal(d->wy, (size_t)(ny + 1) * nx) && all_equal(d->av, n2) &&
                     all_equal(d->vh, n2) && all_equal(d->sumw, n2);
    L.uniform = uni ? 1 : 0;
    std::vector<double> drw(nz);
    for (int k = 0; k < nz; ++k) drw[k] = d->omega2 * d->dr[k];   // stencil.py:103
    cudaError_t e;
    if ((e = upload(lv, drw.data(), nz, &L.drw)) != cudaSuccess ||
        (e = upload(lv, d->vprof, nz + 1, &L.vprof)) != cudaSuccess ||
        (e = upload(lv, d->volprof, nz, &L.volprof)) != cudaSuccess ||
        (e = upload(lv, d->dr, nz, &L.dr)) != cudaSuccess) {
        pmg_level_destroy(lv);
        return cuda_fail(e, "level upload");
    }
    if (uni) {
        const double wx0 = d->wx[0], wy0 = d->wy[0], av0 = d->av[0], vh0 = d->vh[0],
                     sw0 = d->sumw[0];
        L.wx0 = wx0;
        L.wy0 = wy0;
        L.csub0 = d->vcoef * av0;                                   // smoother.py:88
        lv->h_diag.resize(nz);
        lv->h_band.assign(nz + 1, 0.0);
        lv->h_invd.resize(nz);
        const double osw = d->omega2 * sw0;
        const double cv = d->vcoef * av0;
        for (int k = 0; k < nz; ++k) {                              // stencil.py:105-109
            const double t1 = vh0 * d->volprof[k];
            const double t2 = osw * d->dr[k];
            const double t3 = cv * (d->vprof[k] + d->vprof[k + 1]);
            lv->h_diag[k] = (t1 + t2) + t3;
        }
        for (int k = 0; k <= nz; ++k) lv->h_band[k] = cv * d->vprof[k];   // stencil.py:79-81
        lv->h_invd[0] = 1.0 / lv->h_diag[0];                        // smoother.py:93-99
        for (int k = 1; k < nz; ++k) {
            const double sk = d->vprof[k] * L.csub0;
            const double ss = sk * sk;
            const double m = ss * lv->h_invd[k - 1];
            lv->h_invd[k] = 1.0 / (lv->h_diag[k] - m);
        }
        for (int k = 0; k < nz; ++k)
            if (!std::isfinite(lv->h_invd[k]) || std::fabs(lv->h_diag[k]) < 1e-300) {
                pmg_level_destroy(lv);
                return fail(PMG_ERR_PIVOT, "zero pivot in the column factorisation");
            }
        // k-segmented solver tables: g_k = iota_k r_k + alpha_k g_{k-1},
        // x_k = g_k + mu_k x_{k+1}; pf / q = products of alpha / mu over the
        // segment from its start / to its end (segments of L.seg levels)
        int seg = 4;
        while (seg < 32 && (nz + seg - 1) / seg > 8) seg <<= 1;
        L.seg = ((nz + seg - 1) / seg <= 16) ? seg : 0;
        lv->h_seg.assign(5 * (size_t)nz, 0.0);
        double *al = lv->h_seg.data(), *mu = al + nz, *pf = mu + nz, *qq = pf + nz;
        double *ag = qq + nz;
        for (int k = 0; k < nz; ++k) {
            al[k] = (k == 0) ? 0.0 : (L.csub0 * d->vprof[k]) * lv->h_invd[k];
            mu[k] = (k + 1 < nz) ? (L.csub0 * d->vprof[k + 1]) * lv->h_invd[k] : 0.0;
        }
        if (L.seg) {
            for (int a = 0; a < nz; a += seg) {
                const int b = std::min(nz, a + seg) - 1;
                double p = 1.0;
                for (int k = a; k <= b; ++k) { p *= al[k]; pf[k] = p; }
                double q = 1.0;
                for (int k = b; k >= a; --k) { q *= mu[k]; qq[k] = q; }
                // ag[k] = d y_k / d G for the zero-boundary backward sweep
                double gg = 0.0;
                for (int k = b; k >= a; --k) { gg = pf[k] + mu[k] * gg; ag[k] = gg; }
            }
        }
        if ((e = upload(lv, lv->h_seg.data(), 5 * (size_t)nz, &L.segtab)) != cudaSuccess ||
            (e = upload(lv, lv->h_diag.data(), nz, &L.diag1)) != cudaSuccess ||
            (e = upload(lv, lv->h_band.data(), nz + 1, &L.band1)) != cudaSuccess ||
            (e = upload(lv, lv->h_invd.data(), nz, &L.invd1)) != cudaSuccess) {
            pmg_level_destroy(lv);
            return cuda_fail(e, "level tables");
        }
    } else {
        if ((e = upload(lv, d->wx, (size_t)ny * (nx + 1), &L.wx)) != cudaSuccess ||
            (e = upload(lv, d->wy, (size_t)(ny + 1) * nx, &L.wy)) != cudaSuccess ||
            (e = upload(lv, d->av, n2, &L.av)) != cudaSuccess ||
            (e = upload(lv, d->vh, n2, &L.vh)) != cudaSuccess ||
            (e = upload(lv, d->sumw, n2, &L.sumw)) != cudaSuccess) {
            pmg_level_destroy(lv);
            return cuda_fail(e, "level factors");
        }
        void *p = nullptr;
        if ((e = cudaMalloc(&p, 2 * L.cstride * sizeof(double))) != cudaSuccess) {
            pmg_level_destroy(lv);
            return cuda_fail(e, "pivot table");
        }
        lv->owned.push_back(p);
        lv->invd_field = (double *)p;
        L.invd = lv->invd_field;
    }
    *out = lv;
    return PMG_OK;
}

int pmg_level_destroy(pmg_level *lv) {
    if (!lv) return PMG_OK;
    for (void *p : lv->owned) cudaFree(p);
    delete lv;
    return PMG_OK;
}

long long pmg_level_field_doubles(const pmg_level *lv) {
    if (!lv) return -1;
    return 2 * lv->L.cstride;
}

int pmg_level_layout(const pmg_level *lv, int *pitch, long long *plane, long long *cstride,
                     int *parity, int *uniform) {
    PMG_CHECK_LVL(lv);
    if (pitch) *pitch = lv->L.pitch;
    if (plane) *plane = lv->L.plane;
    if (cstride) *cstride = lv->L.cstride;
    if (parity) *parity = lv->L.par;
    if (uniform) *uniform = lv->L.uniform;
    return PMG_OK;
}

int pmg_level_dims(const pmg_level *lv, int *nx, int *ny, int *nz) {
    PMG_CHECK_LVL(lv);
    if (nx) *nx = lv->L.nx;
    if (ny) *ny = lv->L.ny;
    if (nz) *nz = lv->L.nz;
    return PMG_OK;
}

int pmg_level_tables(const pmg_level *lv, double *diag, double *band, double *invd) {
    PMG_CHECK_LVL(lv);
    if (!lv->L.uniform) return fail(PMG_ERR_VALUE, "level has variable coefficients");
    const int nz = lv->L.nz;
    if (diag) std::memcpy(diag, lv->h_diag.data(), nz * sizeof(double));
    if (band) std::memcpy(band, lv->h_band.data(), (nz + 1) * sizeof(double));
    if (invd) std::memcpy(invd, lv->h_invd.data(), nz * sizeof(double));
    return PMG_OK;
}

int pmg_level_prepare(pmg_level *lv, void *stream) {
    PMG_CHECK_LVL(lv);
    if (lv->L.uniform || lv->prepared) return PMG_OK;
    PMG_CUDA(launch_invd(lv->L, lv->invd_field, (cudaStream_t)stream), "invd");
    lv->prepared = true;
    return PMG_OK;
}

int pmg_from_ref_layout(const pmg_level *lv, const double *src, double *field, void *st) {
    PMG_CHECK_LVL(lv);
    PMG_CUDA(launch_from_ref(lv->L, src, field, 0, lv->L.nx, (cudaStream_t)st),
             "from_ref_layout");
    return PMG_OK;
}

int pmg_to_ref_layout(const pmg_level *lv, const double *field, double *dst, void *st) {
    PMG_CHECK_LVL(lv);
    PMG_CUDA(launch_to_ref(lv->L, field, dst, 0, lv->L.nx, (cudaStream_t)st), "to_ref_layout");
    return PMG_OK;
}

int pmg_from_ref_layout_slab(const pmg_level *lv, const double *src, double *field, int i0,
                             int i1, void *st) {
    PMG_CHECK_LVL(lv);
    if (i0 < 0 || i1 > lv->L.nx || i0 > i1) return fail(PMG_ERR_VALUE, "slab out of range");
    PMG_CUDA(launch_from_ref(lv->L, src, field, i0, i1, (cudaStream_t)st), "from_ref_layout");
    return PMG_OK;
}

int pmg_to_ref_layout_slab(const pmg_level *lv, const double *field, double *dst, int i0, int i1,
                           void *st) {
    PMG_CHECK_LVL(lv);
    if (i0 < 0 || i1 > lv->L.nx || i0 > i1) return fail(PMG_ERR_VALUE, "slab out of range");
    PMG_CUDA(launch_to_ref(lv->L, field, dst, i0, i1, (cudaStream_t)st), "to_ref_layout");
    return PMG_OK;
}

int pmg_apply(const pmg_level *lv, const double *u, double *out, void *st) {
    PMG_CHECK_LVL(lv);
    int np = 0;
    PMG_CUDA(launch_apply(lv->L, u, nullptr, out, 0, nullptr, &np, (cudaStream_t)st), "apply");
    return PMG_OK;
}

int pmg_residual(const pmg_level *lv, const double *f, const double *u, double *r,
                 double *scratch, double *norm2, void *st) {
    PMG_CHECK_LVL(lv);
    if (norm2 && !scratch) return fail(PMG_ERR_VALUE, "norm needs a scratch buffer");
    int np = 0;
    PMG_CUDA(launch_apply(lv->L, u, f, r, 1, norm2 ? scratch : nullptr, &np, (cudaStream_t)st),
             "residual");
    if (norm2) PMG_CUDA(launch_finalize(scratch, np, norm2, (cudaStream_t)st), "residual norm");
    return PMG_OK;
}

int pmg_apply_dot(const pmg_level *lv, const double *p, double *q, double *scratch, double *dot,
                  void *st) {
    PMG_CHECK_LVL(lv);
    if (!scratch || !dot) return fail(PMG_ERR_VALUE, "apply_dot needs scratch and output");
    int np = 0;
    PMG_CUDA(launch_apply(lv->L, p, nullptr, q, 2, scratch, &np, (cudaStream_t)st), "apply_dot");
    PMG_CUDA(launch_finalize(scratch, np, dot, (cudaStream_t)st), "apply_dot reduce");
    return PMG_OK;
}

static int check_pair(const pmg_level *f, const pmg_level *c) {
    if (!f || !c) return fail(PMG_ERR_VALUE, "null level handle");
    if (c->L.nx * 2 != f->L.nx || c->L.ny * 2 != f->L.ny || c->L.nz != f->L.nz)
        return fail(PMG_ERR_VALUE, "coarse level must halve nx and ny at equal nz");
    return PMG_OK;
}

int pmg_residual_restrict(const pmg_level *fine, const pmg_level *coarse, const double *f,
                          const double *u, double *cf, void *st) {
    int rc = check_pair(fine, coarse);
    if (rc) return rc;
    PMG_CUDA(launch_residual_restrict(fine->L, coarse->L, u, f, cf, (cudaStream_t)st),
             "residual_restrict");
    return PMG_OK;
}

int pmg_residual_restrict_red_ok(const pmg_level *lv) {
    return lv && residual_restrict_red_ok(lv->L) ? 1 : 0;
}

int pmg_residual_restrict_red(const pmg_level *fine, const pmg_level *coarse, const double *f,
                              const double *u, double *cf, void *st) {
    int rc = check_pair(fine, coarse);
    if (rc) return rc;
    if (!residual_restrict_red_ok(fine->L))
        return fail(PMG_ERR_VALUE, "red-only restriction needs fast mode, uniform coefficients "
                                   "and nx a multiple of 4");
    PMG_CUDA(launch_residual_restrict_red(fine->L, coarse->L, u, f, cf, (cudaStream_t)st),
             "residual_restrict_red");
    return PMG_OK;
}

int pmg_red_residual_norm(const pmg_level *lv, const double *f, const double *u,
                          double *scratch, double *norm2, void *st) {
    PMG_CHECK_LVL(lv);
    if (!scratch || !norm2) return fail(PMG_ERR_VALUE, "norm needs scratch and output");
    if (!residual_restrict_red_ok(lv->L) || lv->L.nx < 4)
        return fail(PMG_ERR_VALUE, "red residual norm needs fast mode and nx a multiple of 4");
    // the column-quad grid of the red restriction: nx / 2 x ny / 2
    Lvl Cq = lv->L;
    Cq.nx = lv->L.nx / 2;
    Cq.ny = lv->L.ny / 2;
    int np = 0;
    PMG_CUDA(launch_residual_restrict_red(lv->L, Cq, u, f, nullptr, (cudaStream_t)st, scratch,
                                          &np),
             "red_residual_norm");
    PMG_CUDA(launch_finalize(scratch, np, norm2, (cudaStream_t)st), "red residual norm");
    return PMG_OK;
}

int pmg_half_sweep(const pmg_level *lv, double *u, const double *f, int color, double rho,
                   int zero_start, int neighbors_zero, double post_scale, void *st) {
    PMG_CHECK_LVL(lv);
    if (color != 0 && color != 1) return fail(PMG_ERR_VALUE, "colour must be 0 (red) or 1 (black)");
    if (!lv->L.uniform && !lv->prepared) {
        int rc = pmg_level_prepare(const_cast<pmg_level *>(lv), st);
        if (rc) return rc;
    }
    PMG_CUDA(launch_half_sweep(lv->L, u, f, color, rho, zero_start, neighbors_zero, post_scale,
                               (cudaStream_t)st),
             "half_sweep");
    return PMG_OK;
}

int pmg_half_sweep_region_ok(const pmg_level *lv) {
    if (!lv) return 0;
    const Lvl &L = lv->L;
    // the fast uniform column solvers (k_half_sweep_band / k_half_sweep_seg)
    // and the variable-coefficient band kernel walk tile regions; the exact
    // solver and the variable register kernel do not
    if (L.uniform)
        return (!g_smoother_exact && L.seg && (L.nz + L.seg - 1) / L.seg <= 8) ? 1 : 0;
    return half_sweep_bandv_ok(L) ? 1 : 0;
}

int pmg_half_sweep_region(const pmg_level *lv, double *u, const double *f, int color, double rho,
                          int zero_start, int neighbors_zero, double post_scale, int rx0, int rxs,
                          int rxn, int ry0, int rys, int ryn, void *st) {
    PMG_CHECK_LVL(lv);
    if (color != 0 && color != 1) return fail(PMG_ERR_VALUE, "colour must be 0 (red) or 1 (black)");
    if (!pmg_half_sweep_region_ok(lv))
        return fail(PMG_ERR_VALUE, "tile regions need the fast smoother on a uniform level "
                                   "or a band-kernel variable level");
    if (!lv->L.uniform && neighbors_zero && !(rho == 1.0 && !zero_start))
        return fail(PMG_ERR_VALUE, "variable-level regions with zero neighbours need rho = 1 "
                                   "and no zero start");
    if (!lv->L.uniform && !lv->prepared) {
        int rc = pmg_level_prepare(const_cast<pmg_level *>(lv), st);
        if (rc) return rc;
    }
    const Lvl &L0 = lv->L;
    const int hx = ((L0.nx + 1) / 2 + 31) / 32;
    if (rxn < 0 || ryn < 0 || rxs < 1 || rys < 1 || rx0 < 0 || ry0 < 0 ||
        (rxn > 0 && rx0 + (long long)(rxn - 1) * rxs >= hx) ||
        (ryn > 0 && ry0 + (long long)(ryn - 1) * rys >= L0.ny))
        return fail(PMG_ERR_VALUE, "tile region outside the part");
    if (rxn == 0 || ryn == 0) return PMG_OK;
    if (ryn == 1) rys = 1;
    if (rxn == 1) rxs = 1;
    if (!L0.uniform && rys != 1)
        return fail(PMG_ERR_VALUE, "variable-level regions take consecutive rows (rys = 1)");
    Lvl L = L0;
    L.rx0 = rx0, L.rxs = rxs, L.rxn = rxn;
    L.ry0 = ry0, L.rys = rys, L.ryn = ryn;
    PMG_CUDA(launch_half_sweep(L, u, f, color, rho, zero_start, neighbors_zero, post_scale,
                               (cudaStream_t)st),
             "half_sweep_region");
    return PMG_OK;
}

int pmg_half_sweep_res_ok(const pmg_level *lv) { return lv && half_sweep_res_ok(lv->L) ? 1 : 0; }

int pmg_half_sweep_res(const pmg_level *lv, const double *u, double *u_new, const double *f,
                       double *scratch, double *norm2, void *st) {
    PMG_CHECK_LVL(lv);
    if (!u || !u_new || !f || !scratch || !norm2) return fail(PMG_ERR_VALUE, "null argument");
    if (u == u_new) return fail(PMG_ERR_VALUE, "u_new must be a different buffer from u");
    if (!half_sweep_res_ok(lv->L))
        return fail(PMG_ERR_VALUE, "fused sweep + residual needs fast mode and nz a multiple "
                                   "of 16 (uniform: <= 128, variable: <= 256)");
    if (!lv->L.uniform && !lv->prepared) {
        int rc = pmg_level_prepare(const_cast<pmg_level *>(lv), st);
        if (rc) return rc;
    }
    int np = 0;
    PMG_CUDA(launch_half_sweep_res(lv->L, u, u_new, f, scratch, &np, (cudaStream_t)st),
             "half_sweep_res");
    PMG_CUDA(launch_finalize(scratch, np, norm2, (cudaStream_t)st), "half_sweep_res norm");
    return PMG_OK;
}

int pmg_restrict(const pmg_level *fine, const pmg_level *coarse, const double *ff, double *cf,
                 double weight, void *st) {
    int rc = check_pair(fine, coarse);
    if (rc) return rc;
    PMG_CUDA(launch_restrict(fine->L, coarse->L, ff, cf, weight, (cudaStream_t)st), "restrict");
    return PMG_OK;
}

int pmg_prolong(const pmg_level *fine, const pmg_level *coarse, const double *cu, double *fu,
                int add, void *st) {
    int rc = check_pair(fine, coarse);
    if (rc) return rc;
    PMG_CUDA(launch_prolong(fine->L, coarse->L, cu, fu, add, 3, (cudaStream_t)st), "prolong");
    return PMG_OK;
}

int pmg_prolong_add(const pmg_level *fine, const pmg_level *coarse, const double *cu, double *fu,
                    void *st) {
    return pmg_prolong(fine, coarse, cu, fu, 1, st);
}

int pmg_prolong_colors(const pmg_level *fine, const pmg_level *coarse, const double *cu, double *fu,
                       int add, int color_mask, void *st) {
    int rc = check_pair(fine, coarse);
    if (rc) return rc;
    if (color_mask < 1 || color_mask > 3) return fail(PMG_ERR_VALUE, "color_mask must be 1, 2 or 3");
    PMG_CUDA(launch_prolong(fine->L, coarse->L, cu, fu, add, color_mask, (cudaStream_t)st),
             "prolong_colors");
    return PMG_OK;
}

int pmg_halo_self(const pmg_level *lv, double *field, int px, int py, void *st) {
    PMG_CHECK_LVL(lv);
    PMG_CUDA(launch_halo_self(lv->L, field, px, py, (cudaStream_t)st), "halo_self");
    return PMG_OK;
}

long long pmg_face_doubles(const pmg_level *lv, int face) {
    if (!lv || face < 0 || face > 3) return -1;
    return (long long)face_len(lv->L, face) * lv->L.nz;
}

int pmg_pack_face(const pmg_level *lv, const double *field, int face, double *buf, void *st) {
    PMG_CHECK_LVL(lv);
    if (face < 0 || face > 3) return fail(PMG_ERR_VALUE, "face must be 0..3");
    PMG_CUDA(launch_pack(lv->L, field, face, buf, (cudaStream_t)st), "pack_face");
    return PMG_OK;
}

int pmg_unpack_face(const pmg_level *lv, double *field, int face, const double *buf, int mirror,
                    void *st) {
    PMG_CHECK_LVL(lv);
    if (face < 0 || face > 3) return fail(PMG_ERR_VALUE, "face must be 0..3");
    PMG_CUDA(launch_unpack(lv->L, field, face, buf, mirror, (cudaStream_t)st), "unpack_face");
    return PMG_OK;
}

long long pmg_partials_size(void) { return PARTIALS; }

int pmg_dot(const pmg_level *lv, const double *a, const double *b, double *scratch, double *out,
            void *st) {
    PMG_CHECK_LVL(lv);
    int np = 0;
    PMG_CUDA(launch_dot(lv->L, a, b, scratch, &np, (cudaStream_t)st), "dot");
    PMG_CUDA(launch_finalize(scratch, np, out, (cudaStream_t)st), "dot reduce");
    return PMG_OK;
}

int pmg_norm2(const pmg_level *lv, const double *a, double *scratch, double *out, void *st) {
    return pmg_dot(lv, a, a, scratch, out, st);
}

int pmg_field_alloc(const pmg_level *lv, double **out) {
    PMG_CHECK_LVL(lv);
    if (!out) return fail(PMG_ERR_VALUE, "out must not be NULL");
    *out = nullptr;
    const size_t bytes = sizeof(double) * (size_t)pmg_level_field_doubles(lv);
    void *d = nullptr;
    PMG_CUDA(cudaMalloc(&d, bytes), "field_alloc");
    cudaError_t e = cudaMemset(d, 0, bytes);
    if (e != cudaSuccess) {
        cudaFree(d);
        PMG_CUDA(e, "field_alloc");
    }
    *out = (double *)d;
    return PMG_OK;
}

int pmg_field_free(double *field) {
    if (field) PMG_CUDA(cudaFree(field), "field_free");
    return PMG_OK;
}

int pmg_fill(const pmg_level *lv, double *field, double value, void *st) {
    PMG_CHECK_LVL(lv);
    const long long n = lv->L.cstride * 2;
    if (value == 0.0 && !std::signbit(value)) {
        PMG_CUDA(cudaMemsetAsync(field, 0, sizeof(double) * n, (cudaStream_t)st), "fill");
    } else {
        PMG_CUDA(launch_fill(n, value, field, (cudaStream_t)st), "fill");
    }
    return PMG_OK;
}

int pmg_copy_block(const pmg_level *src_lvl, const double *src, const pmg_level *dst_lvl,
                   double *dst, int si, int sj, int di, int dj, int w, int h, void *st) {
    if (!src_lvl || !dst_lvl) return fail(PMG_ERR_VALUE, "null level handle");
    const Lvl &S = src_lvl->L, &D = dst_lvl->L;
    if (S.nz != D.nz) return fail(PMG_ERR_VALUE, "levels differ in nz");
    if (w < 0 || h < 0 || si < -1 || sj < -1 || di < -1 || dj < -1 || si + w > S.nx + 1 ||
        sj + h > S.ny + 1 || di + w > D.nx + 1 || dj + h > D.ny + 1)
        return fail(PMG_ERR_VALUE, "block outside the parts (halo ring included)");
    PMG_CUDA(launch_copy_block(S, src, D, dst, si, sj, di, dj, w, h, (cudaStream_t)st),
             "copy_block");
    return PMG_OK;
}

int pmg_copy(const pmg_level *lv, double *dst, const double *src, void *st) {
    PMG_CHECK_LVL(lv);
    PMG_CUDA(cudaMemcpyAsync(dst, src, sizeof(double) * lv->L.cstride * 2,
                             cudaMemcpyDeviceToDevice, (cudaStream_t)st), "copy");
    return PMG_OK;
}

int pmg_field_upload(const pmg_level *lv, const double *host, double *field, double *staging,
                     void *st) {
    PMG_CHECK_LVL(lv);
    if (!host || !field || !staging) return fail(PMG_ERR_VALUE, "null buffer");
    const size_t n = (size_t)lv->L.nx * lv->L.ny * lv->L.nz;
    PMG_CUDA(cudaMemcpyAsync(staging, host, n * sizeof(double), cudaMemcpyHostToDevice,
                             (cudaStream_t)st), "field upload");
    PMG_CUDA(launch_from_ref(lv->L, staging, field, 0, lv->L.nx, (cudaStream_t)st),
             "field upload layout");
    return PMG_OK;
}

int pmg_field_download(const pmg_level *lv, const double *field, double *host, double *staging,
                       void *st) {
    PMG_CHECK_LVL(lv);
    if (!host || !field || !staging) return fail(PMG_ERR_VALUE, "null buffer");
    const size_t n = (size_t)lv->L.nx * lv->L.ny * lv->L.nz;
    PMG_CUDA(launch_to_ref(lv->L, field, staging, 0, lv->L.nx, (cudaStream_t)st),
             "field download layout");
    PMG_CUDA(cudaMemcpyAsync(host, staging, n * sizeof(double), cudaMemcpyDeviceToHost,
                             (cudaStream_t)st), "field download");
    return PMG_OK;
}

int pmg_ssor_apply(const pmg_level *lv, const double *r, double *z, double rho, int periodic_x,
                   int periodic_y, double *scratch, double *rz_dev, void *st) {
    PMG_CHECK_LVL(lv);
    if (!(rho > 0.0 && rho < 2.0)) return fail(PMG_ERR_VALUE, "overrelaxation weight must lie in (0, 2)");
    if (rz_dev && !scratch) return fail(PMG_ERR_VALUE, "the <r, z> product needs a scratch buffer");
    int rc;
    // the reference zero-fills z first (smoother.py:235-238).  That fill is
    // dead work -- the first red half-sweep ignores z, the black one reads
    // only the fresh red values -- unless a periodic level is one column
    // wide: every cell is then its own neighbour through the wrap and the
    // black half-sweep does read (copies of) black values
    if ((periodic_x && lv->L.nx == 1) || (periodic_y && lv->L.ny == 1))
        if ((rc = pmg_fill(lv, z, 0.0, st))) return rc;
    if (rz_dev && half_sweep_dot_ok(lv->L)) {
        // <r, z> fused into the two half-sweeps that produce final values:
        // black (final after the black sweep) and the last red sweep
        cudaStream_t cs = (cudaStream_t)st;
        int n1 = 0, n2 = 0;
        if ((rc = pmg_half_sweep(lv, z, r, 0, rho, 1, 1, 1.0, st))) return rc;
        if ((rc = pmg_halo_self(lv, z, periodic_x, periodic_y, st))) return rc;
        PMG_CUDA(launch_half_sweep_dot(lv->L, z, r, 1, rho, 1, 0, 2.0 - rho, scratch, &n1, cs),
                 "ssor black");
        if ((rc = pmg_halo_self(lv, z, periodic_x, periodic_y, st))) return rc;
        PMG_CUDA(launch_half_sweep_dot(lv->L, z, r, 0, rho, 0, 0, 1.0, scratch + n1, &n2, cs),
                 "ssor red");
        if ((rc = pmg_halo_self(lv, z, periodic_x, periodic_y, st))) return rc;
        PMG_CUDA(launch_finalize(scratch, n1 + n2, rz_dev, cs), "ssor <r, z>");
        return PMG_OK;
    }
    // smoother.py:224-244: red from zero without neighbours, black from zero
    // scaled by (2 - rho), red; a halo refresh after each
    if ((rc = pmg_half_sweep(lv, z, r, 0, rho, 1, 1, 1.0, st))) return rc;
    if ((rc = pmg_halo_self(lv, z, periodic_x, periodic_y, st))) return rc;
    if ((rc = pmg_half_sweep(lv, z, r, 1, rho, 1, 0, 2.0 - rho, st))) return rc;
    if ((rc = pmg_halo_self(lv, z, periodic_x, periodic_y, st))) return rc;
    if ((rc = pmg_half_sweep(lv, z, r, 0, rho, 0, 0, 1.0, st))) return rc;
    if ((rc = pmg_halo_self(lv, z, periodic_x, periodic_y, st))) return rc;
    if (rz_dev) return pmg_dot(lv, r, z, scratch, rz_dev, st);
    return PMG_OK;
}

int pmg_axpy(long long n, double a, const double *x, double *y, void *st) {
    PMG_CUDA(launch_axpy(n, a, x, y, (cudaStream_t)st), "axpy");
    return PMG_OK;
}

int pmg_xpby(long long n, const double *x, double b, double *y, void *st) {
    PMG_CUDA(launch_xpby(n, x, b, y, (cudaStream_t)st), "xpby");
    return PMG_OK;
}

int pmg_cg_update(const pmg_level *lv, const double *num, const double *den, const double *p,
                  const double *q, double *u, double *r, double *scratch, double *rr, void *st) {
    PMG_CHECK_LVL(lv);
    int np = 0;
    PMG_CUDA(launch_cg_update(lv->L, num, den, p, q, u, r, scratch, &np, (cudaStream_t)st),
             "cg_update");
    PMG_CUDA(launch_finalize(scratch, np, rr, (cudaStream_t)st), "cg_update reduce");
    return PMG_OK;
}

int pmg_cg_step(long long n, const double *alpha_num, const double *alpha_den,
                const double *beta_num, const double *beta_den, const double *z, double *p,
                double *u, void *st) {
    PMG_CUDA(launch_cg_up(n, alpha_num, alpha_den, beta_num, beta_den, z, p, u, (cudaStream_t)st),
             "cg_step");
    return PMG_OK;
}

int pmg_cg_direction(long long n, const double *num, const double *den, const double *z,
                     double *p, void *st) {
    PMG_CUDA(launch_cg_direction(n, num, den, z, p, (cudaStream_t)st), "cg_direction");
    return PMG_OK;
}

}  // extern "C"
