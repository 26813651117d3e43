// Native solve drivers of libpmg (include/pmg.h, "drivers" section):
// the V-cycle / mg_solve of multigrid.py:271-330 and the preconditioned CG of
// krylov.py:88-167 for one part that is its own neighbour (one GPU per
// process, periodic or mirror halos), written over the level entry points
// of pmg_api.cu.  The V-cycle + convergence norm is captured once per
// (f, u, first-cycle, stream) into a CUDA graph and replayed; the host reads
// one scalar per cycle (CG: three per iteration) from host-mapped memory.
//
// Operation sequence = the Python drivers' fused path (multigrid.v_cycle
// with cfg.fused, krylov.pcg_solve), so both give bit-identical results.
#include <cmath>
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "../../include/pmg.h"
#include "pmg_trace.h"

namespace pmg {
extern int g_mode_gen;
int set_error(int code, const char *msg);
pmg_level *level_view(const pmg_level *lv, long long cstride, int hflags_or = 0);
void level_view_free(pmg_level *v);
int level_hflags(const pmg_level *lv);
constexpr int HF_WRAP = 8;   // pmg_common.cuh
int half_sweep_fsq(const pmg_level *lv, double *u, const double *f, int color, int nbr_zero,
                   double *partials, int *np, void *st);
int finalize(const double *partials, int n, double *out, void *st);
}

namespace {

int err(int code, const std::string &m) { return pmg::set_error(code, m.c_str()); }

int cuda_err(cudaError_t e, const char *where) {
    return err(PMG_ERR_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

#define TRY(x)                         \
    do {                               \
        int rc_ = (x);                 \
        if (rc_) return rc_;           \
    } while (0)
#define TRYC(x, where)                            \
    do {                                          \
        cudaError_t e_ = (x);                     \
        if (e_ != cudaSuccess) return cuda_err(e_, where); \
    } while (0)

struct Graph {
    const double *f;
    double *u;
    int first;   // 0/1: cycle + norm (first = zero start); >= 2: lagged-norm kinds
    cudaStream_t st;
    cudaGraphExec_t exec;
    long long launches;   // library kernels recorded in the graph
};

}  // namespace

struct pmg_hier {
    std::vector<const pmg_level *> lv;
    std::vector<long long> nd;       // field doubles per level
    pmg_mg_desc d;
    std::vector<double *> u, f;      // coarse-level iterates / right-hand sides (index >= 1)
    double *scratch = nullptr;       // reduction partials
    double *res_h = nullptr;         // host-mapped scalars [8]
    double *res_d = nullptr;
    std::vector<Graph> graphs;
    long long replayed = 0;          // kernels issued by graph replays
    // lagged norm: the second fine red array and the iteration count of the
    // previous solve (chooses which red array the first cycle writes)
    double *red1 = nullptr;
    int last_iters = 4;
    // wrap views of the levels (periodic neighbour reads, no halo ring
    // upkeep) for the lagged driver; empty when not eligible
    std::vector<pmg_level *> wv;
    long long wv_cs = 0;
    // the legacy default stream cannot be captured: solves issued on it run
    // on this stream, ordered after / before the caller's work by events
    cudaStream_t own = nullptr;
    cudaEvent_t ev_in = nullptr, ev_out = nullptr;
    int mode_gen = 0;                // pmg::g_mode_gen the graphs / views were made under
    pmg::CycleClock clock;           // per-cycle device times of the last traced solve
};

namespace {

void free_hier(pmg_hier *h) {
    for (auto &g : h->graphs) cudaGraphExecDestroy(g.exec);
    for (size_t c = 1; c < h->u.size(); ++c) {
        cudaFree(h->u[c]);
        cudaFree(h->f[c]);
    }
    if (h->scratch) cudaFree(h->scratch);
    if (h->red1) cudaFree(h->red1);
    for (auto *v : h->wv)
        if (v) pmg::level_view_free(v);
    if (h->res_h) cudaFreeHost(h->res_h);
    if (h->own) cudaStreamDestroy(h->own);
    if (h->ev_in) cudaEventDestroy(h->ev_in);
    if (h->ev_out) cudaEventDestroy(h->ev_out);
    delete h;
}

// graphs and wrap views record the kernel variants of the smoother mode
// they were made under: drop them when the mode has changed since
void sync_mode(pmg_hier *h) {
    if (h->mode_gen == pmg::g_mode_gen) return;
    for (auto &g : h->graphs) cudaGraphExecDestroy(g.exec);
    h->graphs.clear();
    for (auto *v : h->wv)
        if (v) pmg::level_view_free(v);
    h->wv.clear();
    h->mode_gen = pmg::g_mode_gen;
}

// the fine level seen through `view` (lagged norm: red array elsewhere)
// or the level itself
struct Fine {
    const pmg_level *view = nullptr;
    bool red_done = false;   // the cycle's first red half-sweep already ran
    // first cycle: ||f||^2 summed by its first red and black half-sweeps
    // (partials at fsq_part, the total into fsq_out)
    double *fsq_part = nullptr, *fsq_out = nullptr;
};

const pmg_level *lvl(const pmg_hier *h, int c, const Fine &fv) {
    if (c == 0 && fv.view) return fv.view;
    if (fv.view && c < (int)h->wv.size() && h->wv[c]) return h->wv[c];
    return h->lv[c];
}

// halo ring refresh, skipped on wrap views (their readers wrap around)
int halo(const pmg_hier *h, const pmg_level *l, double *x, cudaStream_t st) {
    pmg::Trace tr("halo exchange");
    if (pmg::level_hflags(l) & pmg::HF_WRAP) return PMG_OK;
    return pmg_halo_self(l, x, h->d.periodic_x, h->d.periodic_y, st);
}

int half_sweep(const pmg_hier *h, const pmg_level *l, double *u, const double *f, int color,
               int nbr_zero, cudaStream_t st) {
    TRY(pmg_half_sweep(l, u, f, color, h->d.rho, 0, nbr_zero, 1.0, st));
    return halo(h, l, u, st);
}

// red-black sweeps with a halo refresh after each half (smoother.py:184-191);
// from_zero: the iterate is zero on entry but unfilled, the first red
// half-sweep ignores it (neighbours zero; rhs = f exactly); red_done: the
// first red half-sweep was run by pmg_half_sweep_res
int sweeps(const pmg_hier *h, const pmg_level *l, double *u, const double *f, int n,
           bool from_zero, bool red_done, cudaStream_t st, const Fine *fsq = nullptr) {
    if (fsq && fsq->fsq_part && n >= 1 && !red_done) {
        // first sweep with ||f||^2 folded in
        int n1 = 0, n2 = 0;
        TRY(pmg::half_sweep_fsq(l, u, f, 0, from_zero ? 1 : 0, fsq->fsq_part, &n1, st));
        TRY(halo(h, l, u, st));
        TRY(pmg::half_sweep_fsq(l, u, f, 1, 0, fsq->fsq_part + n1, &n2, st));
        TRY(halo(h, l, u, st));
        TRY(pmg::finalize(fsq->fsq_part, n1 + n2, fsq->fsq_out, st));
        from_zero = false;
        n -= 1;
    }
    for (int s = 0; s < n; ++s) {
        if (red_done && s == 0)
            TRY(halo(h, l, u, st));
        else
            TRY(half_sweep(h, l, u, f, 0, (from_zero && s == 0) ? 1 : 0, st));
        TRY(half_sweep(h, l, u, f, 1, 0, st));
    }
    return PMG_OK;
}

// Alg. 1 (multigrid.py:271-294); level 0 works on the caller's u0 / f0
int vcycle(pmg_hier *h, int c, double *u0, const double *f0, bool first, cudaStream_t st,
           const Fine &fv = Fine()) {
    pmg::Trace tr("level %d", c);
    const int L = (int)h->lv.size();
    double *u = c ? h->u[c] : u0;
    const double *f = c ? h->f[c] : f0;
    const pmg_level *lc = lvl(h, c, fv);
    const bool red_done = c == 0 && fv.red_done;
    const bool lean = h->d.rho == 1.0;
    if (c + 1 < L) {
        TRY(sweeps(h, lc, u, f, h->d.nu_pre, lean && (c > 0 || first), red_done, st,
                   c == 0 ? &fv : nullptr));
        const pmg_level *lcc = lvl(h, c + 1, fv);
        if (h->d.red_restrict && lean && h->d.nu_pre >= 1 && pmg_residual_restrict_red_ok(lc))
            TRY(pmg_residual_restrict_red(lc, lcc, f, u, h->f[c + 1], st));
        else
            TRY(pmg_residual_restrict(lc, lcc, f, u, h->f[c + 1], st));
        // the coarse iterate starts from zero: skip the fill when its first
        // red half-sweep ignores it anyway
        const int first_sweeps = (c + 2 == L) ? h->d.coarse_sweeps : h->d.nu_pre;
        if (!(lean && first_sweeps >= 1))
            TRYC(cudaMemsetAsync(h->u[c + 1], 0, sizeof(double) * h->nd[c + 1], st), "coarse fill");
        TRY(vcycle(h, c + 1, u0, f0, false, st, fv));
        // u += P e (black cells only when the red half-sweep overwrites red)
        const int pmask = (lean && h->d.nu_post >= 1) ? 2 : 3;
        TRY(pmg_prolong_colors(lc, lcc, h->u[c + 1], u, 1, pmask, st));
        TRY(halo(h, lc, u, st));
        TRY(sweeps(h, lc, u, f, h->d.nu_post, false, false, st));
    } else {
        TRY(sweeps(h, lc, u, f, h->d.coarse_sweeps, lean && c > 0, false, st));
    }
    return PMG_OK;
}

int cycle_and_norm(pmg_hier *h, double *u, const double *f, bool first, cudaStream_t st) {
    TRY(vcycle(h, 0, u, f, first, st));
    return pmg_residual(h->lv[0], f, u, nullptr, h->scratch, h->res_d, st);
}

// lagged-norm cycle bodies.  Red array A = the caller's u (view: level 0),
// B = h->red1 (view: black array at the caller's u + cstride).  kind 2 + X:
// first cycle from zero relaxing into red array X; kind 4 + X: a cycle on
// X whose first red half-sweep already ran.  Both end with the next
// cycle's first red half-sweep from X into the other array, which also
// sums ||f - A u||^2 of this cycle's result into res_d[0].
struct Lag {
    const pmg_level *view[2];
    double *base[2];
};

// kinds 6 + X (predicted last cycle): as 4 + X but ending with the
// check-only red residual norm of the result (pmg_red_residual_norm: reads
// f_r, u_r, u_b; writes nothing).  Kinds 8 + X: a full cycle on X from an
// ordinary red half-sweep (after a check that did not converge), ending
// with the fused next red half-sweep.
int lagged_body(pmg_hier *h, const double *f, int kind, const Lag &g, cudaStream_t st) {
    const int x = kind & 1;
    const bool first = kind < 4;
    Fine fv;
    fv.view = g.view[x];
    fv.red_done = (kind >= 4 && kind < 8);
    if (first) {   // first cycle: ||f||^2 into res_d[1]
        fv.fsq_part = h->scratch + pmg_partials_size() / 2;
        fv.fsq_out = h->res_d + 1;
    }
    TRY(vcycle(h, 0, g.base[x], f, first, st, fv));
    if (kind == 6 || kind == 7)
        return pmg_red_residual_norm(g.view[x], f, g.base[x], h->scratch, h->res_d, st);
    return pmg_half_sweep_res(g.view[x], g.base[x], g.base[x ^ 1], f, h->scratch, h->res_d, st);
}

// the next cycle ends with the check-only norm when the last contraction
// predicts convergence with a factor-2 margin
bool predict_last(double rn, double prev, double r0, double eps) {
    if (!(prev > 0.0)) return false;
    return rn * (rn / prev) < 0.5 * eps * r0;
}

template <class Body>
int replay_kind(pmg_hier *h, double *u, const double *f, int kind, cudaStream_t st, Body body) {
    for (auto &g : h->graphs)
        if (g.f == f && g.u == u && g.first == kind && g.st == st) {
            TRYC(cudaGraphLaunch(g.exec, st), "graph launch");
            h->replayed += g.launches;
            return PMG_OK;
        }
    if (h->graphs.size() >= 32) {   // 4 cycle kinds x a few (f, u) pairs
        cudaGraphExecDestroy(h->graphs.front().exec);
        h->graphs.erase(h->graphs.begin());
    }
    pmg::Trace tr("capture cycle graph");
    cudaGraph_t graph;
    const long long l0 = pmg_launch_count();
    TRYC(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal), "capture");
    int rc = body();
    cudaError_t e = cudaStreamEndCapture(st, &graph);
    if (rc) {
        // a launch that failed inside the capture invalidates it: drop the
        // graph and clear the error state, so the caller's next call starts
        // clean (the failure itself is reported through rc)
        if (e == cudaSuccess) cudaGraphDestroy(graph);
        cudaGetLastError();
        return rc;
    }
    TRYC(e, "capture end");
    Graph g{f, u, kind, st, nullptr, pmg_launch_count() - l0};
    e = cudaGraphInstantiate(&g.exec, graph, 0);
    cudaGraphDestroy(graph);
    TRYC(e, "graph instantiate");
    h->graphs.push_back(g);
    TRYC(cudaGraphLaunch(g.exec, st), "graph launch");
    h->replayed += g.launches;
    return PMG_OK;
}

int replay(pmg_hier *h, double *u, const double *f, bool first, cudaStream_t st) {
    if (!st) return cycle_and_norm(h, u, f, first, st);   // legacy stream: no capture
    return replay_kind(h, u, f, first ? 1 : 0, st,
                       [&] { return cycle_and_norm(h, u, f, first, st); });
}

// every level can be read through a wrap view: periodic in x and y, fast
// mode (k_half_sweep_seg / k_half_sweep_segv), nx % 4 == 0 with a coarse
// level of >= 2 columns (column-quad restriction / prolongation)
bool wrap_ok(const pmg_hier *h) {
    if (!h->d.periodic_x || !h->d.periodic_y || pmg_get_smoother_mode() != 0) return false;
    for (size_t c = 0; c < h->lv.size(); ++c) {
        int nx, ny, nz, pitch, par, uni;
        long long plane, cs;
        if (pmg_level_dims(h->lv[c], &nx, &ny, &nz) ||
            pmg_level_layout(h->lv[c], &pitch, &plane, &cs, &par, &uni))
            return false;
        if (nz > 256 || nx % 2 || ny % 2) return false;
        if (c + 1 < h->lv.size() && (nx % 4 || nx < 4)) return false;
        if (!uni) {
            // variable levels: k_half_sweep_segv (16 warps) and, below the
            // coarsest, the red-only restriction (the full one reads halos)
            const int seg = nz / 16;
            if (nz % 16 || !(seg == 1 || seg == 2 || seg == 4 || seg == 8 || seg == 16))
                return false;
            if (c + 1 < h->lv.size() && !h->d.red_restrict) return false;
        }
    }
    return true;
}

bool lagged_ok(const pmg_hier *h) {
    int nx, ny, nz;
    if (pmg_level_dims(h->lv[0], &nx, &ny, &nz)) return false;
    // nx % 4: the fine residual-restriction is the column-quad kernel, the
    // one that reads f through Lvl::fcs
    // a variable fine level restricts with the red-only kernel (the general
    // variable restriction does not read Lvl::fcs)
    long long plane, cs;
    int pitch, par, uni;
    if (pmg_level_layout(h->lv[0], &pitch, &plane, &cs, &par, &uni)) return false;
    if (!uni && !(h->d.red_restrict && pmg_residual_restrict_red_ok(h->lv[0]))) return false;
    return h->d.lagged_norm && h->d.rho == 1.0 && h->d.nu_pre >= 1 && h->d.nu_post >= 1 &&
           h->lv.size() > 1 && nx % 4 == 0 &&
           pmg_half_sweep_res_ok(h->lv[0]);
}

}  // namespace

extern "C" {

int pmg_hier_create(const pmg_level *const *levels, int nlev, const pmg_mg_desc *desc,
                    pmg_hier **out) {
    if (!levels || !desc || !out || nlev < 1) return err(PMG_ERR_VALUE, "bad hierarchy arguments");
    if (desc->nu_pre < 0 || desc->nu_post < 0 || desc->coarse_sweeps < 0)
        return err(PMG_ERR_VALUE, "sweep counts must be non-negative");
    if (!(desc->rho > 0.0 && desc->rho < 2.0))
        return err(PMG_ERR_VALUE, "overrelaxation weight must lie in (0, 2)");
    int nx0 = 0, ny0 = 0, nz0 = 0;
    for (int c = 0; c < nlev; ++c) {
        int nx, ny, nz;
        TRY(pmg_level_dims(levels[c], &nx, &ny, &nz));
        if (c == 0) {
            nx0 = nx, ny0 = ny, nz0 = nz;
        } else if (nx != (nx0 >> c) || ny != (ny0 >> c) || nz != nz0 || (nx << c) != nx0 ||
                   (ny << c) != ny0) {
            return err(PMG_ERR_VALUE, "each level must halve nx and ny at equal nz");
        }
        // a periodic level one column wide is its own neighbour: the fused
        // cycle's identities (the black half-sweep reads no black value, the
        // black residual after it is zero) fail there
        if ((desc->periodic_x && nx == 1) || (desc->periodic_y && ny == 1))
            return err(PMG_ERR_VALUE,
                       "a periodic level one column wide is its own neighbour: use fewer "
                       "levels (the Python driver runs the plain cycle on such hierarchies)");
    }
    pmg_hier *h = new pmg_hier();
    h->d = *desc;
    h->lv.assign(levels, levels + nlev);
    h->u.assign(nlev, nullptr);
    h->f.assign(nlev, nullptr);
    for (int c = 0; c < nlev; ++c) h->nd.push_back(pmg_level_field_doubles(levels[c]));
    cudaError_t e = cudaSuccess;
    for (int c = 1; c < nlev && e == cudaSuccess; ++c) {
        e = cudaMalloc(&h->u[c], sizeof(double) * h->nd[c]);
        if (e == cudaSuccess) e = cudaMalloc(&h->f[c], sizeof(double) * h->nd[c]);
        // halos of a fresh coarse iterate must be finite
        if (e == cudaSuccess) e = cudaMemset(h->u[c], 0, sizeof(double) * h->nd[c]);
    }
    if (e == cudaSuccess) e = cudaMalloc(&h->scratch, sizeof(double) * pmg_partials_size());
    if (e == cudaSuccess) e = cudaHostAlloc(&h->res_h, 8 * sizeof(double), cudaHostAllocMapped);
    if (e == cudaSuccess) e = cudaHostGetDevicePointer((void **)&h->res_d, h->res_h, 0);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&h->own, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&h->ev_in, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&h->ev_out, cudaEventDisableTiming);
    if (e != cudaSuccess) {
        free_hier(h);
        return cuda_err(e, "hierarchy allocation");
    }
    *out = h;
    return PMG_OK;
}

int pmg_hier_destroy(pmg_hier *h) {
    if (h) free_hier(h);
    return PMG_OK;
}

long long pmg_hier_replayed_launches(const pmg_hier *h) { return h ? h->replayed : -1; }

int pmg_hier_cycle_times(const pmg_hier *h, double *ms, int cap) {
    if (!h || (cap > 0 && !ms)) return -1;
    return h->clock.copy_out(ms, cap);
}

long long pmg_hier_graph_launches(const pmg_hier *h, const double *f, const double *u,
                                  int first) {
    if (!h) return -1;
    for (auto &g : h->graphs)
        if (g.f == f && g.u == u && g.first == first) return g.launches;
    return -1;
}

int pmg_vcycle(pmg_hier *h, double *u, const double *f, int first, void *stream) {
    if (!h || !u || !f) return err(PMG_ERR_VALUE, "null argument");
    sync_mode(h);
    if (first && !(h->d.rho == 1.0 && h->lv.size() > 1 && h->d.nu_pre >= 1))
        return err(PMG_ERR_VALUE, "first = 1 needs rho = 1, nu_pre >= 1 and two levels");
    return vcycle(h, 0, u, f, first != 0, (cudaStream_t)stream);
}

// mg_solve with the lagged norm (pmg_mg_desc.lagged_norm): cycle k's
// residual norm is summed by the first red half-sweep of cycle k + 1, which
// writes its red values into the other red array, so u_k stays intact
// until the norm decides.  The first cycle relaxes into the red array that
// makes the expected last iterate (the previous solve's count) land in the
// caller's u; otherwise one red-array copy at the end.
static int mg_solve_lagged(pmg_hier *h, const double *f, double *u, double eps, int maxiter,
                           double *hist, int *iters, int *converged, cudaStream_t st) {
    const pmg_level *l0 = h->lv[0];
    long long plane, cs;
    int pitch, parity, uniform;
    TRY(pmg_level_layout(l0, &pitch, &plane, &cs, &parity, &uniform));
    if (!h->red1) TRYC(cudaMalloc(&h->red1, sizeof(double) * cs), "red array");
    // variable levels compute their pivot field before any view of them is
    // taken (a view shares the field; preparing through a view would index
    // it with the view's colour stride) and outside any graph capture
    for (auto *l : h->lv) TRY(pmg_level_prepare(const_cast<pmg_level *>(l), st));
    if (h->wv.empty()) {
        // wrap views of every level when all of them qualify
        const int wrap = wrap_ok(h) ? pmg::HF_WRAP : 0;
        h->wv.assign(h->lv.size(), nullptr);
        if (wrap) {
            for (size_t c = 0; c < h->lv.size(); ++c) {
                long long pc2, cs2;
                int p2, par2, uni2;
                TRY(pmg_level_layout(h->lv[c], &p2, &pc2, &cs2, &par2, &uni2));
                h->wv[c] = pmg::level_view(h->lv[c], cs2, wrap);
            }
        }
    }
    const int wrap = h->wv[0] ? pmg::HF_WRAP : 0;
    // black array of the caller's u, seen from red1
    const long long csb =
        (long long)(((intptr_t)(u + cs) - (intptr_t)h->red1) / (intptr_t)sizeof(double));
    pmg_level *vb = pmg::level_view(l0, csb, wrap);
    struct Free {
        pmg_level *v;
        ~Free() { pmg::level_view_free(v); }
    } guard{vb};
    Lag g{{wrap ? h->wv[0] : l0, vb}, {u, h->red1}};
    // iterate k lives in red array (x0 + k - 1) & 1; want the last one in A
    int x = (h->last_iters & 1) ? 0 : 1;
    int kind = 2 + x;
    *iters = 0;
    *converged = 0;
    double r0 = 0.0, prev = 0.0;
    bool predict = pmg_residual_restrict_red_ok(l0) != 0;
    for (int it = 0; it < maxiter; ++it) {
        pmg::Trace tr("cycle %d", it + 1);
        TRYC(h->clock.start(st), "cycle clock");
        TRY(replay_kind(h, u, f, kind, st, [&] { return lagged_body(h, f, kind, g, st); }));
        TRYC(h->clock.stop(st), "cycle clock");
        TRYC(cudaStreamSynchronize(st), "sync");
        if (it == 0) {
            // r0 = ||f|| (multigrid.py:307-309), summed by the first cycle
            r0 = std::sqrt(h->res_h[1]);
            hist[0] = r0;
            if (r0 == 0.0) {   // multigrid.py:317-318: u = 0, no iterations
                TRY(pmg_fill(l0, u, 0.0, st));
                *converged = 1;
                return PMG_OK;
            }
        }
        const double rn = std::sqrt(h->res_h[0]);
        hist[it + 1] = rn;
        *iters = it + 1;
        if (rn / r0 < eps) {
            *converged = 1;
            break;
        }
        if (it + 1 == maxiter) break;   // u_maxiter stays in red array x
        if (kind == 6 || kind == 7) {
            // predicted convergence missed: the next cycle starts with an
            // ordinary red half-sweep on the same red array; no more guesses
            kind = 8 + x;
            predict = false;
        } else {
            x ^= 1;   // the fused sweep relaxed red into the other array
            kind = (predict && predict_last(rn, prev, r0, eps)) ? 6 + x : 4 + x;
        }
        prev = rn;
    }
    h->last_iters = *iters;
    if (x == 1)   // the result's red array is red1: copy it into u
        TRYC(cudaMemcpyAsync(u, h->red1, sizeof(double) * cs, cudaMemcpyDeviceToDevice, st),
             "red array copy");
    // wrap views left the halo ring stale: refresh it for the caller
    if (wrap) TRY(pmg_halo_self(l0, u, h->d.periodic_x, h->d.periodic_y, st));
    return PMG_OK;
}

static int mg_solve_on(pmg_hier *h, const double *f, double *u, double eps, int maxiter,
                       double *hist, int *iters, int *converged, cudaStream_t st) {
    if (maxiter >= 1 && lagged_ok(h))
        return mg_solve_lagged(h, f, u, eps, maxiter, hist, iters, converged, st);
    const pmg_level *l0 = h->lv[0];
    // variable levels compute their pivot field here, outside the graph
    // capture (a lazy prepare inside the capture would be replayed per cycle)
    for (auto *l : h->lv) TRY(pmg_level_prepare(const_cast<pmg_level *>(l), st));
    // r0 = ||f|| (multigrid.py:307-309)
    TRY(pmg_dot(l0, f, f, h->scratch, h->res_d, st));
    TRYC(cudaStreamSynchronize(st), "sync");
    const double r0 = std::sqrt(h->res_h[0]);
    hist[0] = r0;
    *iters = 0;
    *converged = 0;
    if (r0 == 0.0) {
        TRY(pmg_fill(l0, u, 0.0, st));
        *converged = 1;
        return PMG_OK;
    }

    // rho = 1: the first cycle starts from zero without filling u
    const bool lean_first = h->d.rho == 1.0 && h->d.nu_pre >= 1 && h->lv.size() > 1;
    if (!lean_first) TRY(pmg_fill(l0, u, 0.0, st));
    for (int it = 0; it < maxiter; ++it) {
        pmg::Trace tr("cycle %d", it + 1);
        TRYC(h->clock.start(st), "cycle clock");
        TRY(replay(h, u, f, lean_first && it == 0, st));
        TRYC(h->clock.stop(st), "cycle clock");
        TRYC(cudaStreamSynchronize(st), "sync");
        const double rn = std::sqrt(h->res_h[0]);
        hist[it + 1] = rn;
        *iters = it + 1;
        if (rn / r0 < eps) {
            *converged = 1;
            break;
        }
    }
    return PMG_OK;
}

int pmg_mg_solve(pmg_hier *h, const double *f, double *u, double eps, int maxiter, double *hist,
                 int *iters, int *converged, void *stream) {
    if (!h || !f || !u || !hist || !iters || !converged) return err(PMG_ERR_VALUE, "null argument");
    if (maxiter < 0 || !(eps > 0.0)) return err(PMG_ERR_VALUE, "need eps > 0 and maxiter >= 0");
    cudaStream_t st = (cudaStream_t)stream;
    sync_mode(h);
    pmg::Trace tr("pmg_mg_solve");
    h->clock.reset();
    if (st) return mg_solve_on(h, f, u, eps, maxiter, hist, iters, converged, st);
    // legacy stream: run on the hierarchy's stream, ordered by events
    TRYC(cudaEventRecord(h->ev_in, 0), "event");
    TRYC(cudaStreamWaitEvent(h->own, h->ev_in, 0), "event wait");
    const int rc = mg_solve_on(h, f, u, eps, maxiter, hist, iters, converged, h->own);
    TRYC(cudaEventRecord(h->ev_out, h->own), "event");
    TRYC(cudaStreamWaitEvent(0, h->ev_out, 0), "event wait");
    return rc;
}

// Alg. 2 (krylov.py:88-167, the Python pcg_solve's sequence without a
// callback): SSOR (precond = 1) or identity (precond = 0) preconditioner;
// alpha and beta stay on the device and the host reads <p,q>, ||r||^2 and
// the <r,z> of the step once per iteration.  The iterate update of
// iteration k is deferred into the direction update of iteration k+1
// (pmg_cg_step) and flushed at exit.  PMG_ERR_BREAKDOWN on <p,q> <= 0 or
// <r,z> <= 0.  work: pmg_pcg_work_doubles() device doubles.
int pmg_pcg_solve(const pmg_level *lv, const double *f, double *u, double eps, int maxiter,
                  double tau, int precond, double rho, int periodic_x, int periodic_y,
                  double *work, double *hist, int *iters, int *converged, void *stream) {
    if (!lv || !f || !u || !work || !hist || !iters || !converged)
        return err(PMG_ERR_VALUE, "null argument");
    if (!(eps > 0.0 && eps < 1.0)) return err(PMG_ERR_VALUE, "relative tolerance must lie in (0, 1)");
    if (precond && !(rho > 0.0 && rho < 2.0))
        return err(PMG_ERR_VALUE, "overrelaxation weight must lie in (0, 2)");
    pmg::Trace tr("pmg_pcg_solve");
    cudaStream_t st = (cudaStream_t)stream;
    const long long n = pmg_level_field_doubles(lv);
    double *r = work, *z = work + n, *p = work + 2 * n, *q = work + 3 * n;
    double *scratch = work + 4 * n;
    double *kap = scratch + pmg_partials_size();   // device scalars: kappa, pq, rr, kappa_new
    double *pq = kap + 1, *rr = kap + 2, *kapn = kap + 3;
    double *res_h = nullptr, *res_d = nullptr;
    TRYC(cudaHostAlloc(&res_h, 4 * sizeof(double), cudaHostAllocMapped), "pinned scalars");
    struct Free {
        double *p;
        ~Free() { cudaFreeHost(p); }
    } guard{res_h};
    TRYC(cudaHostGetDevicePointer((void **)&res_d, res_h, 0), "pinned scalars");
    // z = M r and rz_dev[0] = <r, z> (fused into the SSOR half-sweeps)
    auto precondition = [&](double *rz_dev) -> int {
        if (precond)
            return pmg_ssor_apply(lv, r, z, rho, periodic_x, periodic_y, scratch, rz_dev, stream);
        TRY(pmg_copy(lv, z, r, stream));
        TRY(pmg_halo_self(lv, z, periodic_x, periodic_y, stream));
        return pmg_dot(lv, r, z, scratch, rz_dev, stream);
    };
    auto read = [&](const double *dev, int k) -> int {
        TRYC(cudaMemcpyAsync(res_d, dev, k * sizeof(double), cudaMemcpyDeviceToDevice, st),
             "scalar read");
        TRYC(cudaStreamSynchronize(st), "sync");
        return PMG_OK;
    };
    // u = 0, r = f (full allocation), r0 = ||r||
    TRY(pmg_fill(lv, u, 0.0, stream));
    TRY(pmg_copy(lv, r, f, stream));
    TRY(pmg_dot(lv, r, r, scratch, res_d, stream));
    TRYC(cudaStreamSynchronize(st), "sync");
    const double r0 = std::sqrt(res_h[0]);
    hist[0] = r0;
    *iters = 0;
    *converged = 0;
    if (r0 == 0.0 || r0 < tau) {
        *converged = 1;
        return PMG_OK;
    }
    TRY(precondition(kap));
    TRY(pmg_copy(lv, p, z, stream));
    TRY(read(kap, 1));
    if (!(res_h[0] > 0.0)) return err(PMG_ERR_BREAKDOWN, "<r, z> <= 0: preconditioner is not positive definite");
    bool pending = false;
    for (int it = 1; it <= maxiter; ++it) {
        pmg::Trace ti("iteration %d", it);
        TRY(pmg_apply_dot(lv, p, q, scratch, pq, stream));
        TRY(pmg_cg_update(lv, kap, pq, p, q, nullptr, r, scratch, rr, stream));
        pending = true;
        TRY(read(kap, 3));                        // kappa, pq, rr
        if (!(res_h[0] > 0.0)) return err(PMG_ERR_BREAKDOWN, "<r, z> <= 0: preconditioner is not positive definite");
        if (!(res_h[1] > 0.0)) return err(PMG_ERR_BREAKDOWN, "<p, A p> <= 0: operator is not positive definite");
        const double rn = std::sqrt(res_h[2]);
        hist[it] = rn;
        *iters = it;
        if (rn / r0 < eps || rn < tau) {
            *converged = 1;
            break;
        }
        TRY(precondition(kapn));
        // u += (kappa / pq) p ; p = z + (kappa_new / kappa) p
        TRY(pmg_cg_step(n, kap, pq, kapn, kap, z, p, u, stream));
        pending = false;
        TRYC(cudaMemcpyAsync(kap, kapn, sizeof(double), cudaMemcpyDeviceToDevice, st), "kappa");
    }
    if (pending) TRY(pmg_cg_step(n, kap, pq, kap, kap, nullptr, p, u, stream));
    TRY(read(kap, 1));
    if (!*converged && !(res_h[0] > 0.0))
        return err(PMG_ERR_BREAKDOWN, "<r, z> <= 0: preconditioner is not positive definite");
    return PMG_OK;
}

long long pmg_pcg_work_doubles(const pmg_level *lv) {
    if (!lv) return -1;
    return 4 * pmg_level_field_doubles(lv) + pmg_partials_size() + 8;
}

}  // extern "C"
