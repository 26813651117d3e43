// Native multi-part solve driver of libpmg (include/pmg.h, "multi-part
// drivers"): the V-cycle / mg_solve of multigrid.py:271-330 over a px x py
// horizontal decomposition, with the halo exchange of
// partition.py:158-191 and the reductions of partition.py:267-286 issued by
// the library, inside the captured CUDA graph of each cycle.
//
// A hierarchy holds the parts this process owns: all of them (in-process
// decomposition on one device: the exchange is a device copy between
// parts), or one part per rank with a library-owned NCCL communicator
// (pmg_comm_create; the exchange is ncclSend / ncclRecv over NVLink, the
// reductions an ncclAllGather of the per-part sums added in worker order).
// Either way one cycle is one graph replay and one 8-byte host read.
//
// Boundary-first relaxation: on levels wide enough, a
// half-sweep first relaxes the frame -- the rows and 32-cell strips that
// hold the part's boundary columns (pmg_half_sweep_region) -- then forks
// the halo exchange of those values onto a second stream while the
// interior relaxes; the two join before anything reads the halo.  The
// interior reads no halo cell and the exchange touches only frame and
// halo cells, so the result is the unsplit sweep's, bit for bit.
//
// NCCL is resolved at run time (dlopen of libnccl.so.2, normally the copy
// torch already loaded): the library links no NCCL and runs without one.
#include <dlfcn.h>

#include <array>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include <cuda_runtime.h>
#include <nccl.h>   // types and prototypes only; symbols come from dlsym

#include "pmg_common.cuh"
#include "pmg_trace.h"

namespace pmg {
extern std::atomic<long long> g_launches;
extern int g_mode_gen;
int set_error(int code, const char *msg);
const Lvl &level_lvl(const pmg_level *lv);
pmg_level *level_view(const pmg_level *lv, long long cstride, int hflags_or = 0);
void level_view_free(pmg_level *v);
int half_sweep_fsq(const pmg_level *lv, double *u, const double *f, int color, int nbr_zero,
                   double *partials, int *np, void *st);
int finalize(const double *partials, int n, double *out, void *st);
}

namespace {

int err(int code, const std::string &m) { return pmg::set_error(code, m.c_str()); }

#define TRY(x)                         \
    do {                               \
        int rc_ = (x);                 \
        if (rc_) return rc_;           \
    } while (0)
#define TRYC(x, where)                                                                  \
    do {                                                                                \
        cudaError_t e_ = (x);                                                           \
        if (e_ != cudaSuccess)                                                          \
            return err(PMG_ERR_CUDA, std::string(where) + ": " + cudaGetErrorString(e_)); \
    } while (0)

// ---- NCCL, resolved at run time ------------------------------------------
struct Nccl {
    decltype(&ncclGetUniqueId) get_unique_id = nullptr;
    decltype(&ncclCommInitRank) comm_init_rank = nullptr;
    decltype(&ncclCommDestroy) comm_destroy = nullptr;
    decltype(&ncclSend) send = nullptr;
    decltype(&ncclRecv) recv = nullptr;
    decltype(&ncclGroupStart) group_start = nullptr;
    decltype(&ncclGroupEnd) group_end = nullptr;
    decltype(&ncclAllGather) all_gather = nullptr;
    decltype(&ncclGetErrorString) error_string = nullptr;
};

const Nccl *nccl() {
    static Nccl n;
    static int state = 0;   // 0 untried, 1 ok, -1 unavailable
    if (state == 0) {
        void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        state = -1;
        if (h) {
            n.get_unique_id = (decltype(n.get_unique_id))dlsym(h, "ncclGetUniqueId");
            n.comm_init_rank = (decltype(n.comm_init_rank))dlsym(h, "ncclCommInitRank");
            n.comm_destroy = (decltype(n.comm_destroy))dlsym(h, "ncclCommDestroy");
            n.send = (decltype(n.send))dlsym(h, "ncclSend");
            n.recv = (decltype(n.recv))dlsym(h, "ncclRecv");
            n.group_start = (decltype(n.group_start))dlsym(h, "ncclGroupStart");
            n.group_end = (decltype(n.group_end))dlsym(h, "ncclGroupEnd");
            n.all_gather = (decltype(n.all_gather))dlsym(h, "ncclAllGather");
            n.error_string = (decltype(n.error_string))dlsym(h, "ncclGetErrorString");
            if (n.get_unique_id && n.comm_init_rank && n.comm_destroy && n.send && n.recv &&
                n.group_start && n.group_end && n.all_gather && n.error_string)
                state = 1;
        }
    }
    return state == 1 ? &n : nullptr;
}

int nccl_err(ncclResult_t r, const char *where) {
    const Nccl *n = nccl();
    return err(PMG_ERR_CUDA, std::string(where) + ": " + (n ? n->error_string(r) : "nccl"));
}

#define TRYN(x, where)                                    \
    do {                                                  \
        ncclResult_t r_ = (x);                            \
        if (r_ != ncclSuccess) return nccl_err(r_, where); \
    } while (0)

// worker-order sum of n per-part scalars (the in-process order of
// partition.reduce_parts: ((v0 + v1) + v2) + ...), one thread
__global__ void k_sum_ordered(const double *__restrict__ v, int n, double *__restrict__ out) {
    double s = 0.0;
    for (int i = 0; i < n; ++i) s += v[i];
    *out = s;
}

constexpr int OPP[4] = {1, 0, 3, 2};
// directions of the single-phase exchange: W, E, S, N, SW, SE, NW, NE; a
// strip sent towards d lands in the receiver's halo on side OPP8[d]
constexpr int OPP8[8] = {1, 0, 3, 2, 7, 6, 5, 4};

// ---- exchange kernels: ONE launch fills the whole halo ring of every part
// (x faces, y faces and the four corner columns).  The two-phase exchange of
// partition.py:158-191 -- x faces, then y faces over the extended range --
// gives corner (a, b) the value found by resolving x first (the a-side
// neighbour's column, or the mirrored own column at a physical boundary) and
// then y on the part reached; both kernels below read that cell directly, so
// the ring holds the two-phase exchange's values bit for bit.
constexpr int MAXP = 16;   // in-process parts per hierarchy

// in-process: halo cell of part p <- the owned cell it images; blockIdx.z =
// 4 p + face (faces 2, 3 cover the extended range -1 .. nx: the corners).
// Reads only owned cells, writes only halo cells: race-free within the launch.
struct LocalX {
    int np;
    pmg::Lvl L[MAXP];
    double *u[MAXP];
    int nbr[MAXP][4];   // local part index, -1 mirror
};

__global__ void k_halo_local(const __grid_constant__ LocalX x) {
    const int p = blockIdx.z >> 2, face = blockIdx.z & 3;
    const pmg::Lvl &L = x.L[p];
    const int len = face < 2 ? L.ny : L.nx + 2;
    const int t = blockIdx.x * blockDim.x + threadIdx.x, k = blockIdx.y;
    if (t >= len) return;
    int i, j;
    pmg::face_pos(L, face, t, true, i, j);
    int sp = p, si = i, sj = j;
    if (i < 0) {
        const int q = x.nbr[sp][0];
        si = q >= 0 ? L.nx - 1 : 0;
        if (q >= 0) sp = q;
    } else if (i >= L.nx) {
        const int q = x.nbr[sp][1];
        si = q >= 0 ? 0 : L.nx - 1;
        if (q >= 0) sp = q;
    }
    if (j < 0) {
        const int q = x.nbr[sp][2];
        sj = q >= 0 ? L.ny - 1 : 0;
        if (q >= 0) sp = q;
    } else if (j >= L.ny) {
        const int q = x.nbr[sp][3];
        sj = q >= 0 ? 0 : L.ny - 1;
        if (q >= 0) sp = q;
    }
    x.u[p][pmg::cell(L, i, j, k)] = x.u[sp][pmg::cell(x.L[sp], si, sj, k)];
}

// one part's boundary strips into / out of its eight message buffers:
// faces W, E (ny x nz, buf[k * ny + j]), S, N ((nx + 2) x nz over the
// extended range, buf[k * (nx + 2) + i + 1]) and corners SW, SE, NW, NE (nz).
// blockIdx.z = face.  An extended position of a y strip carries the sender's
// mirrored boundary column where its x side is a physical boundary (what
// the two-phase exchange's y strips carry there); next to an x neighbour it
// is unused -- that corner travels as its own message from the diagonal part.
struct FaceX {
    pmg::Lvl L;
    double *u;
    double *buf[8];
    int nbr[8];     // peer worker per direction, -1 none
};

__global__ void k_pack_all(const __grid_constant__ FaceX x) {
    const int face = blockIdx.z;
    if (x.nbr[face] < 0) return;
    const pmg::Lvl &L = x.L;
    const int len = face < 2 ? L.ny : L.nx + 2;
    const int t = blockIdx.x * blockDim.x + threadIdx.x, k = blockIdx.y;
    if (t >= len) return;
    int i, j;
    pmg::face_pos(L, face, t, false, i, j);
    if (face >= 2 && (i < 0 || i >= L.nx)) {
        const int a = i < 0 ? 0 : 1;
        if (x.nbr[a] >= 0) return;             // the diagonal part's message
        i = i < 0 ? 0 : L.nx - 1;              // mirrored own column
    }
    const double v = x.u[pmg::cell(L, i, j, k)];
    x.buf[face][(long long)k * len + t] = v;
    if (face >= 2 && (i == 0 || i == L.nx - 1) && t >= 1 && t <= L.nx) {
        // the owned corner column also travels to the diagonal neighbour
        if (i == 0) {
            const int d = 4 + 2 * (face - 2);
            if (x.nbr[d] >= 0) x.buf[d][k] = v;
        }
        if (i == L.nx - 1) {
            const int d = 5 + 2 * (face - 2);
            if (x.nbr[d] >= 0) x.buf[d][k] = v;
        }
    }
}

__global__ void k_unpack_all(const __grid_constant__ FaceX x) {
    const int face = blockIdx.z;
    const pmg::Lvl &L = x.L;
    const int len = face < 2 ? L.ny : L.nx + 2;
    const int t = blockIdx.x * blockDim.x + threadIdx.x, k = blockIdx.y;
    if (t >= len) return;
    int i, j;
    pmg::face_pos(L, face, t, true, i, j);
    double v;
    if (face < 2) {
        v = x.nbr[face] >= 0 ? x.buf[face][(long long)k * L.ny + j]
                             : x.u[pmg::cell(L, face == 0 ? 0 : L.nx - 1, j, k)];
    } else if (i >= 0 && i < L.nx) {
        v = x.nbr[face] >= 0 ? x.buf[face][(long long)k * (L.nx + 2) + t]
                             : x.u[pmg::cell(L, i, face == 2 ? 0 : L.ny - 1, k)];
    } else {
        // corner (a, face): x first, then y on the part reached
        const int a = i < 0 ? 0 : 1, d = 4 + 2 * (face - 2) + a;
        const int jb = face == 2 ? 0 : L.ny - 1;
        if (x.nbr[a] >= 0 && x.nbr[face] >= 0) v = x.buf[d][k];
        else if (x.nbr[face] >= 0) v = x.buf[face][(long long)k * (L.nx + 2) + t];
        else if (x.nbr[a] >= 0) v = x.buf[a][(long long)k * L.ny + jb];
        else v = x.u[pmg::cell(L, a == 0 ? 0 : L.nx - 1, jb, k)];
    }
    x.u[pmg::cell(L, i, j, k)] = v;
}

dim3 face_grid(const pmg::Lvl &L, int nz, int z) {
    const int len = (L.nx + 2 > L.ny) ? L.nx + 2 : L.ny;
    return dim3((unsigned)((len + 127) / 128), (unsigned)nz, (unsigned)z);
}

}  // namespace

struct pmg_comm {
    ncclComm_t c = nullptr;
    int nranks = 0, rank = 0;
};

namespace {

// one part at one level
struct PL {
    const pmg_level *lv = nullptr;
    double *u = nullptr, *f = nullptr;   // level >= 1: owned; level 0: the caller's
    // NCCL message buffers per direction (W, E, S, N, SW, SE, NW, NE): the
    // packed own strips, the received halo strips, and their doubles
    double *sb[8] = {}, *rb[8] = {};
    long long fd[8] = {};
    int nx = 0, ny = 0, nz = 0;
};

struct PGraph {
    std::vector<const double *> f;
    std::vector<double *> u;
    int kind;
    cudaStream_t st;
    cudaGraphExec_t exec;
    long long launches;
};

}  // namespace

struct pmg_phier {
    int np = 0, nlev = 0;
    std::vector<int> worker;                  // per local part, ascending
    std::vector<std::array<int, 4>> nbr;      // per local part: W, E, S, N worker or -1
    std::vector<std::array<int, 4>> diag;     // per local part: SW, SE, NW, NE worker or -1
    std::vector<int> local;                   // worker -> local part index or -1
    std::vector<std::vector<PL>> P;           // [part][level]
    pmg_mg_desc d{};
    pmg_comm *comm = nullptr;
    int overlap_nx = 0;                       // boundary-first on levels with nx >= this
    double *scr[2] = {nullptr, nullptr};      // reduction partials (solve / side stream)
    double *slots = nullptr;                  // device [np + nranks + 8]
    double *res_h = nullptr, *res_d = nullptr;   // host-mapped [8]
    cudaStream_t side = nullptr, own = nullptr;
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr, ev_in = nullptr, ev_out = nullptr;
    std::vector<PGraph> graphs;
    long long replayed = 0;
    long long exchanges = 0;                  // halo exchanges issued (per level, counted once)
    int mode_gen = 0;
    // lagged norm (pmg_driver.cu's identities per part): each part's second
    // red array, the level-0 view the cycle being issued works through (its
    // red array elsewhere), and the previous solve's cycle count
    std::vector<double *> red1;
    std::vector<const pmg_level *> fine_view;
    int last_iters = 4;
    // CG work fields per part (r, z, p, q), allocated on first use
    std::vector<double *> cgw;
    pmg::CycleClock clock;                    // per-cycle device times of the last traced solve
};

namespace {

void free_phier(pmg_phier *h) {
    for (auto &g : h->graphs) cudaGraphExecDestroy(g.exec);
    for (auto &pp : h->P)
        for (size_t c = 0; c < pp.size(); ++c) {
            PL &q = pp[c];
            if (c > 0) {
                cudaFree(q.u);
                cudaFree(q.f);
            }
            for (int a = 0; a < 8; ++a) {
                cudaFree(q.sb[a]);
                cudaFree(q.rb[a]);
            }
        }
    for (auto *s : h->scr) cudaFree(s);
    for (auto *r : h->red1) cudaFree(r);
    for (auto *w : h->cgw) cudaFree(w);
    cudaFree(h->slots);
    if (h->res_h) cudaFreeHost(h->res_h);
    if (h->side) cudaStreamDestroy(h->side);
    if (h->own) cudaStreamDestroy(h->own);
    for (auto e : {h->ev_fork, h->ev_join, h->ev_in, h->ev_out})
        if (e) cudaEventDestroy(e);
    delete h;
}

void sync_mode(pmg_phier *h) {
    if (h->mode_gen == pmg::g_mode_gen) return;
    for (auto &g : h->graphs) cudaGraphExecDestroy(g.exec);
    h->graphs.clear();
    h->mode_gen = pmg::g_mode_gen;
}

// level c of part p as the cycle being issued sees it: the lagged norm's
// level-0 view (red array in the other allocation) while one is set
const pmg_level *LV(const pmg_phier *h, int p, int c) {
    if (c == 0 && !h->fine_view.empty() && h->fine_view[p]) return h->fine_view[p];
    return h->P[p][c].lv;
}

// halo exchange of level c's fields x[p] (partition.py:158-191: x faces,
// then y faces over the extended range, periodic neighbours or mirrored
// physical boundaries) as ONE phase on stream s: in-process, one launch
// fills every part's halo ring; with a communicator, one pack launch, one
// NCCL group carrying the four faces and the four corner columns (the plan
// of pmg_exchange_plan8), one unpack launch.
int exchange(pmg_phier *h, int c, double *const *x, cudaStream_t s) {
    pmg::Trace tr("halo exchange level %d", c);
    ++h->exchanges;
    const PL &q = h->P[0][c];
    if (!h->comm) {
        LocalX lx;
        lx.np = h->np;
        for (int p = 0; p < h->np; ++p) {
            lx.L[p] = pmg::level_lvl(LV(h, p, c));
            lx.u[p] = x[p];
            for (int a = 0; a < 4; ++a) {
                const int nb = h->nbr[p][a];
                lx.nbr[p][a] = nb < 0 ? -1 : h->local[nb];
            }
        }
        k_halo_local<<<face_grid(lx.L[0], q.nz, 4 * h->np), 128, 0, s>>>(lx);
        pmg::g_launches.fetch_add(1, std::memory_order_relaxed);
        TRYC(cudaGetLastError(), "halo exchange");
        return PMG_OK;
    }
    // one part (this rank's)
    FaceX fx;
    fx.L = pmg::level_lvl(LV(h, 0, c));
    fx.u = x[0];
    int nbr8[8];
    for (int a = 0; a < 4; ++a) {
        nbr8[a] = h->nbr[0][a];
        nbr8[4 + a] = h->diag[0][a];
    }
    for (int a = 0; a < 8; ++a) {
        fx.buf[a] = q.sb[a];
        fx.nbr[a] = nbr8[a];
    }
    k_pack_all<<<face_grid(fx.L, q.nz, 4), 128, 0, s>>>(fx);
    pmg::g_launches.fetch_add(1, std::memory_order_relaxed);
    TRYC(cudaGetLastError(), "pack");
    const Nccl *n = nccl();
    int ops[48], nops = 0;
    TRY(pmg_exchange_plan8(nbr8, ops, &nops));
    if (nops) {
        TRYN(n->group_start(), "ncclGroupStart");
        for (int o = 0; o < nops; ++o) {
            const int kind = ops[3 * o], dir = ops[3 * o + 1], peer = ops[3 * o + 2];
            ncclResult_t r = kind == 0
                ? n->send(q.sb[dir], (size_t)q.fd[dir], ncclDouble, peer, h->comm->c, s)
                : n->recv(q.rb[dir], (size_t)q.fd[dir], ncclDouble, peer, h->comm->c, s);
            if (r != ncclSuccess) {
                n->group_end();
                return nccl_err(r, kind == 0 ? "ncclSend" : "ncclRecv");
            }
        }
        TRYN(n->group_end(), "ncclGroupEnd");
    }
    for (int a = 0; a < 8; ++a) fx.buf[a] = q.rb[a];
    k_unpack_all<<<face_grid(fx.L, q.nz, 4), 128, 0, s>>>(fx);
    pmg::g_launches.fetch_add(1, std::memory_order_relaxed);
    TRYC(cudaGetLastError(), "unpack");
    return PMG_OK;
}

std::vector<double *> level_u(pmg_phier *h, int c, double *const *u0) {
    std::vector<double *> v(h->np);
    for (int p = 0; p < h->np; ++p) v[p] = c ? h->P[p][c].u : u0[p];
    return v;
}
std::vector<const double *> level_f(pmg_phier *h, int c, const double *const *f0) {
    std::vector<const double *> v(h->np);
    for (int p = 0; p < h->np; ++p) v[p] = c ? h->P[p][c].f : f0[p];
    return v;
}

// sum of the per-part scalars slots[0 .. np) over every part of every rank,
// in worker order, into out (device or host-mapped)
int global_sum(pmg_phier *h, double *out, cudaStream_t s, const double *vals = nullptr) {
    if (!vals) vals = h->slots;
    if (h->comm) {
        // one part per rank: gather the rank sums, add them in rank order
        double *gath = h->slots + 2 * h->np;
        TRYN(nccl()->all_gather(vals, gath, 1, ncclDouble, h->comm->c, s), "ncclAllGather");
        k_sum_ordered<<<1, 1, 0, s>>>(gath, h->comm->nranks, out);
    } else {
        k_sum_ordered<<<1, 1, 0, s>>>(vals, h->np, out);
    }
    pmg::g_launches.fetch_add(1, std::memory_order_relaxed);
    TRYC(cudaGetLastError(), "ordered sum");
    return PMG_OK;
}

// whether level c relaxes boundary-first: every part region-capable, wide
// and tall enough that the frame is a small share of the sweep
bool overlapped(const pmg_phier *h, int c) {
    if (!h->overlap_nx) return false;
    for (int p = 0; p < h->np; ++p) {
        const PL &q = h->P[p][c];
        if (q.nx < h->overlap_nx || q.nx < 256 || q.ny < 16 ||
            !pmg_half_sweep_region_ok(LV(h, p, c)))
            return false;
    }
    return true;
}

// one half-sweep of colour `color` on every part of level c, then the halo
// exchange (boundary-first when the level qualifies)
int half_sweep_x(pmg_phier *h, int c, double *const *u, const double *const *f, int color,
                 int nbr_zero, cudaStream_t s) {
    const double rho = h->d.rho;
    // variable-level regions run the band kernel, which relaxes against zero
    // neighbours only as a plain rho = 1 sweep
    const bool var_nz = nbr_zero && rho != 1.0 && !pmg::level_lvl(LV(h, 0, c)).uniform;
    if (var_nz || !overlapped(h, c)) {
        for (int p = 0; p < h->np; ++p)
            TRY(pmg_half_sweep(LV(h, p, c), u[p], f[p], color, rho, 0, nbr_zero, 1.0, s));
        return exchange(h, c, u, s);
    }
    // frame: rows 0 and ny - 1 (all strips), the first and last strip of
    // rows 1 .. ny - 2; then the interior strips 1 .. n - 2 of those rows.
    // Every region is a run of whole rows, so each runs on the kernel the
    // whole-part sweep would use (the same column solves, bit for bit)
    for (int p = 0; p < h->np; ++p) {
        const PL &q = h->P[p][c];
        const int ns = ((q.nx + 1) / 2 + 31) / 32;
        TRY(pmg_half_sweep_region(LV(h, p, c), u[p], f[p], color, rho, 0, nbr_zero, 1.0, 0, 1, ns, 0, 1,
                                  1, s));
        TRY(pmg_half_sweep_region(LV(h, p, c), u[p], f[p], color, rho, 0, nbr_zero, 1.0, 0, 1, ns,
                                  q.ny - 1, 1, 1, s));
        TRY(pmg_half_sweep_region(LV(h, p, c), u[p], f[p], color, rho, 0, nbr_zero, 1.0, 0, ns - 1, 2,
                                  1, 1, q.ny - 2, s));
    }
    TRYC(cudaEventRecord(h->ev_fork, s), "fork");
    TRYC(cudaStreamWaitEvent(h->side, h->ev_fork, 0), "fork wait");
    TRY(exchange(h, c, u, h->side));
    for (int p = 0; p < h->np; ++p) {
        const PL &q = h->P[p][c];
        const int ns = ((q.nx + 1) / 2 + 31) / 32;
        TRY(pmg_half_sweep_region(LV(h, p, c), u[p], f[p], color, rho, 0, nbr_zero, 1.0, 1, 1, ns - 2,
                                  1, 1, q.ny - 2, s));
    }
    TRYC(cudaEventRecord(h->ev_join, h->side), "join");
    TRYC(cudaStreamWaitEvent(s, h->ev_join, 0), "join wait");
    return PMG_OK;
}

// fine-level state of a lagged-norm cycle (pmg_driver.cu's Fine): the first
// red half-sweep already ran (the previous cycle's fused-residual sweep), or
// the first two half-sweeps sum f^2 (the first cycle's ||f||)
struct Fine {
    bool red_done = false;
    bool fsq = false;
};

// first cycle: red and black half-sweeps with per-part f^2 partials (part
// p's at scr[0] + p * 1024), ||f||^2 over all parts into res_d[1]
int fsq_sweeps(pmg_phier *h, double *const *u, const double *const *f, bool from_zero,
               cudaStream_t s) {
    double *fs = h->slots + h->np;
    int n1[MAXP];
    for (int p = 0; p < h->np; ++p)
        TRY(pmg::half_sweep_fsq(LV(h, p, 0), u[p], f[p], 0, from_zero ? 1 : 0,
                                h->scr[0] + p * 1024, &n1[p], s));
    TRY(exchange(h, 0, u, s));
    for (int p = 0; p < h->np; ++p) {
        int n2 = 0;
        TRY(pmg::half_sweep_fsq(LV(h, p, 0), u[p], f[p], 1, 0, h->scr[0] + p * 1024 + n1[p], &n2,
                                s));
        TRY(pmg::finalize(h->scr[0] + p * 1024, n1[p] + n2, fs + p, s));
    }
    TRY(exchange(h, 0, u, s));
    return global_sum(h, h->res_d + 1, s, fs);
}

// a level-0 half-sweep with the SSOR flags (smoother.py:224-244) on every
// part, then the halo exchange
int half_sweep_y(pmg_phier *h, double *const *u, const double *const *f, int color, double rho,
                 int zero_start, int nbr_zero, double post_scale, cudaStream_t s) {
    for (int p = 0; p < h->np; ++p)
        TRY(pmg_half_sweep(h->P[p][0].lv, u[p], f[p], color, rho, zero_start, nbr_zero,
                           post_scale, s));
    return exchange(h, 0, u, s);
}

int sweeps(pmg_phier *h, int c, double *const *u, const double *const *f, int n, bool from_zero,
           cudaStream_t s, const Fine *fv = nullptr) {
    const bool red_done = fv && fv->red_done;
    if (fv && fv->fsq && n >= 1 && !red_done) {
        TRY(fsq_sweeps(h, u, f, from_zero, s));
        from_zero = false;
        n -= 1;
    }
    for (int k = 0; k < n; ++k) {
        if (red_done && k == 0)
            TRY(exchange(h, c, u, s));   // the red values the fused sweep wrote
        else
            TRY(half_sweep_x(h, c, u, f, 0, (from_zero && k == 0) ? 1 : 0, s));
        TRY(half_sweep_x(h, c, u, f, 1, 0, s));
    }
    return PMG_OK;
}

// Alg. 1 (multigrid.py:271-294): the operation sequence of the Python
// v_cycle's fused path for every part, level by level (level 0 through
// LV's view under the lagged norm)
int vcycle(pmg_phier *h, int c, double *const *u0, const double *const *f0, bool first,
           cudaStream_t s, const Fine *fv = nullptr) {
    pmg::Trace tr("level %d", c);
    const int L = h->nlev;
    const auto u = level_u(h, c, u0);
    const auto f = level_f(h, c, f0);
    const bool lean = h->d.rho == 1.0;
    if (c + 1 < L) {
        TRY(sweeps(h, c, u.data(), f.data(), h->d.nu_pre, lean && (c > 0 || first), s,
                   c == 0 ? fv : nullptr));
        for (int p = 0; p < h->np; ++p) {
            const pmg_level *lf = LV(h, p, c), *lc = h->P[p][c + 1].lv;
            if (h->d.red_restrict && lean && h->d.nu_pre >= 1 && pmg_residual_restrict_red_ok(lf))
                TRY(pmg_residual_restrict_red(lf, lc, f[p], u[p], h->P[p][c + 1].f, s));
            else
                TRY(pmg_residual_restrict(lf, lc, f[p], u[p], h->P[p][c + 1].f, s));
        }
        const int first_sweeps = (c + 2 == L) ? h->d.coarse_sweeps : h->d.nu_pre;
        if (!(lean && first_sweeps >= 1))
            for (int p = 0; p < h->np; ++p)
                TRY(pmg_fill(h->P[p][c + 1].lv, h->P[p][c + 1].u, 0.0, s));
        TRY(vcycle(h, c + 1, u0, f0, false, s));
        const int pmask = (lean && h->d.nu_post >= 1) ? 2 : 3;
        for (int p = 0; p < h->np; ++p)
            TRY(pmg_prolong_colors(LV(h, p, c), h->P[p][c + 1].lv, h->P[p][c + 1].u, u[p], 1,
                                   pmask, s));
        TRY(exchange(h, c, u.data(), s));
        TRY(sweeps(h, c, u.data(), f.data(), h->d.nu_post, false, s));
    } else {
        TRY(sweeps(h, c, u.data(), f.data(), h->d.coarse_sweeps, lean && c > 0, s));
    }
    return PMG_OK;
}

// ||f - A u||^2 over every part (the convergence check, multigrid.py:324)
int norm2(pmg_phier *h, double *const *u, const double *const *f, double *out, cudaStream_t s) {
    for (int p = 0; p < h->np; ++p)
        TRY(pmg_residual(h->P[p][0].lv, f[p], u[p], nullptr, h->scr[0], h->slots + p, s));
    return global_sum(h, out, s);
}

template <class Body>
int replay(pmg_phier *h, double *const *u, const double *const *f, int kind, cudaStream_t s,
           Body body) {
    for (auto &g : h->graphs) {
        bool same = g.kind == kind && g.st == s;
        for (int p = 0; same && p < h->np; ++p) same = g.f[p] == f[p] && g.u[p] == u[p];
        if (same) {
            TRYC(cudaGraphLaunch(g.exec, s), "graph launch");
            h->replayed += g.launches;
            return PMG_OK;
        }
    }
    if (h->graphs.size() >= 16) {
        cudaGraphExecDestroy(h->graphs.front().exec);
        h->graphs.erase(h->graphs.begin());
    }
    pmg::Trace tr("capture cycle graph");
    cudaGraph_t graph;
    const long long l0 = pmg_launch_count();
    TRYC(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal), "capture");
    int rc = body();
    cudaError_t e = cudaStreamEndCapture(s, &graph);
    if (rc) {
        // a launch that failed inside the capture invalidates it: drop the
        // graph and clear the error state, so the caller's next call starts
        // clean (the failure itself is reported through rc)
        if (e == cudaSuccess) cudaGraphDestroy(graph);
        cudaGetLastError();
        return rc;
    }
    TRYC(e, "capture end");
    PGraph g{std::vector<const double *>(f, f + h->np), std::vector<double *>(u, u + h->np), kind,
             s, nullptr, pmg_launch_count() - l0};
    e = cudaGraphInstantiate(&g.exec, graph, 0);
    cudaGraphDestroy(graph);
    TRYC(e, "graph instantiate");
    h->graphs.push_back(g);
    TRYC(cudaGraphLaunch(g.exec, s), "graph launch");
    h->replayed += g.launches;
    return PMG_OK;
}

// the single-part driver's lagged-norm conditions (pmg_driver.cu lagged_ok)
// for every part
bool lagged_ok(const pmg_phier *h) {
    if (!h->d.lagged_norm || h->d.rho != 1.0 || h->d.nu_pre < 1 || h->d.nu_post < 1 ||
        h->nlev < 2)
        return false;
    for (int p = 0; p < h->np; ++p) {
        const pmg_level *l0 = h->P[p][0].lv;
        int pitch, par, uni;
        long long plane, cs;
        if (pmg_level_layout(l0, &pitch, &plane, &cs, &par, &uni)) return false;
        if (!uni && !(h->d.red_restrict && pmg_residual_restrict_red_ok(l0))) return false;
        if (h->P[p][0].nx % 4 || !pmg_half_sweep_res_ok(l0)) return false;
    }
    return true;
}

// mg_solve with the lagged norm (pmg_driver.cu mg_solve_lagged, per part):
// cycle k's ||f - A u|| is summed by the first red half-sweep of cycle k + 1
// (pmg_half_sweep_res), which writes the relaxed red values into the other
// red array of each part; the first cycle's red and black half-sweeps sum
// ||f||^2.  Kinds: 2 + X first cycle relaxing into red array X, 4 + X a
// later cycle on X; each ends with the next cycle's fused sweep from X.
int mg_solve_lagged(pmg_phier *h, const double *const *f, double *const *u, double eps,
                    int maxiter, double *hist, int *iters, int *converged, cudaStream_t s) {
    const int np = h->np;
    long long cs = 0;
    {
        int pitch, par, uni;
        long long plane;
        TRY(pmg_level_layout(h->P[0][0].lv, &pitch, &plane, &cs, &par, &uni));
    }
    if (h->red1.empty()) {
        h->red1.assign(np, nullptr);
        for (int p = 0; p < np; ++p)
            TRYC(cudaMalloc(&h->red1[p], sizeof(double) * cs), "red array");
    }
    // per part: view 1 = the level seen from red1 (black array at u + cs)
    std::vector<pmg_level *> vb(np, nullptr);
    struct Free {
        std::vector<pmg_level *> &v;
        pmg_phier *h;
        ~Free() {
            for (auto *x : v)
                if (x) pmg::level_view_free(x);
            h->fine_view.clear();
        }
    } guard{vb, h};
    for (int p = 0; p < np; ++p) {
        const long long csb =
            (long long)(((intptr_t)(u[p] + cs) - (intptr_t)h->red1[p]) / (intptr_t)sizeof(double));
        vb[p] = pmg::level_view(h->P[p][0].lv, csb, 0);
    }
    std::vector<double *> base[2] = {std::vector<double *>(u, u + np), h->red1};
    auto body = [&](int kind) -> int {
        const int x = kind & 1;
        h->fine_view.assign(np, nullptr);
        if (x)
            for (int p = 0; p < np; ++p) h->fine_view[p] = vb[p];
        Fine fv;
        fv.red_done = kind >= 4 && kind < 8;
        fv.fsq = kind < 4;
        int rc = vcycle(h, 0, base[x].data(), f, kind < 4, s, &fv);
        for (int p = 0; !rc && p < np; ++p) {
            if (kind == 6 || kind == 7)   // predicted last cycle: the check-only norm
                rc = pmg_red_residual_norm(LV(h, p, 0), f[p], base[x][p], h->scr[0] + p * 1024,
                                           h->slots + p, s);
            else   // the next cycle's first red half-sweep into the other array
                rc = pmg_half_sweep_res(LV(h, p, 0), base[x][p], base[x ^ 1][p], f[p],
                                        h->scr[0] + p * 1024, h->slots + p, s);
        }
        if (!rc) rc = global_sum(h, h->res_d, s);
        h->fine_view.clear();
        return rc;
    };
    int x = (h->last_iters & 1) ? 0 : 1;   // want the last iterate in the caller's array
    int kind = 2 + x;
    *iters = 0;
    *converged = 0;
    double r0 = 0.0, prev = 0.0;
    // kinds 6 + X (predicted last cycle, pmg_driver.cu): when the last
    // contraction predicts convergence with a factor-2 margin the cycle ends
    // with the check-only red residual norm; a miss continues with kind
    // 8 + X (an ordinary first red half-sweep on the same array)
    bool predict = true;
    for (int p = 0; p < np; ++p) predict = predict && pmg_residual_restrict_red_ok(h->P[p][0].lv);
    for (int it = 0; it < maxiter; ++it) {
        // graphs are keyed on the caller's arrays (the views depend on them)
        pmg::Trace tr("cycle %d", it + 1);
        TRYC(h->clock.start(s), "cycle clock");
        TRY(replay(h, u, f, kind, s, [&] { return body(kind); }));
        TRYC(h->clock.stop(s), "cycle clock");
        TRYC(cudaStreamSynchronize(s), "sync");
        if (it == 0) {
            r0 = std::sqrt(h->res_h[1]);
            hist[0] = r0;
            if (r0 == 0.0) {   // multigrid.py:317-318
                for (int p = 0; p < np; ++p) TRY(pmg_fill(h->P[p][0].lv, u[p], 0.0, s));
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
            kind = 8 + x;                // the guess missed: same array, no more guesses
            predict = false;
        } else {
            x ^= 1;                      // the fused sweep relaxed red into the other array
            kind = (predict && prev > 0.0 && rn * (rn / prev) < 0.5 * eps * r0) ? 6 + x : 4 + x;
        }
        prev = rn;
    }
    h->last_iters = *iters;
    if (x == 1)   // the result's red array is red1: copy it (halo included) into u
        for (int p = 0; p < np; ++p)
            TRYC(cudaMemcpyAsync(u[p], h->red1[p], sizeof(double) * cs, cudaMemcpyDeviceToDevice,
                                 s),
                 "red array copy");
    return PMG_OK;
}

int mg_solve_on(pmg_phier *h, const double *const *f, double *const *u, double eps, int maxiter,
                double *hist, int *iters, int *converged, cudaStream_t s) {
    for (int p = 0; p < h->np; ++p)
        for (int c = 0; c < h->nlev; ++c)
            TRY(pmg_level_prepare(const_cast<pmg_level *>(h->P[p][c].lv), s));
    if (maxiter >= 1 && lagged_ok(h))
        return mg_solve_lagged(h, f, u, eps, maxiter, hist, iters, converged, s);
    // r0 = ||f|| (multigrid.py:307-309)
    for (int p = 0; p < h->np; ++p)
        TRY(pmg_dot(h->P[p][0].lv, f[p], f[p], h->scr[0], h->slots + p, s));
    TRY(global_sum(h, h->res_d, s));
    TRYC(cudaStreamSynchronize(s), "sync");
    const double r0 = std::sqrt(h->res_h[0]);
    hist[0] = r0;
    *iters = 0;
    *converged = 0;
    if (r0 == 0.0) {   // multigrid.py:317-318
        for (int p = 0; p < h->np; ++p) TRY(pmg_fill(h->P[p][0].lv, u[p], 0.0, s));
        *converged = 1;
        return PMG_OK;
    }
    const bool lean_first = h->d.rho == 1.0 && h->d.nu_pre >= 1 && h->nlev > 1;
    if (!lean_first)
        for (int p = 0; p < h->np; ++p) TRY(pmg_fill(h->P[p][0].lv, u[p], 0.0, s));
    for (int it = 0; it < maxiter; ++it) {
        const int kind = (lean_first && it == 0) ? 1 : 0;
        pmg::Trace tr("cycle %d", it + 1);
        TRYC(h->clock.start(s), "cycle clock");
        TRY(replay(h, u, f, kind, s, [&] {
            TRY(vcycle(h, 0, u, f, kind == 1, s));
            return norm2(h, u, f, h->res_d, s);
        }));
        TRYC(h->clock.stop(s), "cycle clock");
        TRYC(cudaStreamSynchronize(s), "sync");
        const double rn = std::sqrt(h->res_h[0]);
        hist[it + 1] = rn;
        *iters = it + 1;
        if (rn / r0 < eps) {   // strict, multigrid.py:326
            *converged = 1;
            break;
        }
    }
    return PMG_OK;
}

// Preconditioned CG over every part (krylov.py:88-167; the Python driver's
// sequence -- pcg_solve without a callback -- issued by the library): per
// iteration q = A p with <p, q>, the fused update r -= alpha q with
// ||r||^2, one host read of (kappa, <p,q>, ||r||^2) for the breakdown checks
// and the stopping test, z = M r by the line SSOR (red, black, red
// half-sweeps, each followed by the halo exchange; smoother.py:224-244) or
// the identity (copy + exchange), <r, z>, and p = z + beta p with the
// deferred u += alpha p.  Dots are per-part sums added in worker order
// across parts and ranks (global_sum).
int pcg_solve_on(pmg_phier *h, const double *const *f, double *const *u, double eps,
                 int maxiter, double tau, int precond, double rho, double *hist, int *iters,
                 int *converged, cudaStream_t s) {
    const int np = h->np;
    std::vector<long long> nd(np);
    for (int p = 0; p < np; ++p) nd[p] = pmg_level_field_doubles(h->P[p][0].lv);
    if (h->cgw.empty()) {
        h->cgw.assign(4 * np, nullptr);
        for (int p = 0; p < np; ++p)
            for (int v = 0; v < 4; ++v)
                TRYC(cudaMalloc(&h->cgw[4 * p + v], sizeof(double) * nd[p]), "CG work");
    }
    std::vector<double *> r(np), z(np), pp(np), q(np);
    for (int p = 0; p < np; ++p) {
        r[p] = h->cgw[4 * p];
        z[p] = h->cgw[4 * p + 1];
        pp[p] = h->cgw[4 * p + 2];
        q[p] = h->cgw[4 * p + 3];
    }
    // device scalars kappa, <p,q>, ||r||^2, kappa_new (every thread of the
    // update kernels reads them: device memory, after the per-part and the
    // gathered rank sums in slots); copied to the host-mapped res for reads
    double *kap = h->slots + 2 * np + (h->comm ? h->comm->nranks : 0);
    double *pq = kap + 1, *rr = kap + 2, *kapn = kap + 3;
    const double *kap_h = h->res_h + 2, *pq_h = h->res_h + 3, *rr_h = h->res_h + 4;
    auto read3 = [&]() -> int {   // (kappa, <p,q>, ||r||^2) to the host
        TRYC(cudaMemcpyAsync(h->res_d + 2, kap, 3 * sizeof(double), cudaMemcpyDeviceToDevice, s),
             "scalar read");
        TRYC(cudaStreamSynchronize(s), "sync");
        return PMG_OK;
    };
    auto dots = [&](const std::vector<double *> &a, const std::vector<double *> &b,
                    double *out) -> int {
        for (int p = 0; p < np; ++p)
            TRY(pmg_dot(h->P[p][0].lv, a[p], b[p], h->scr[0], h->slots + p, s));
        return global_sum(h, out, s);
    };
    auto precondition = [&](double *rz) -> int {
        if (precond) {
            TRY(half_sweep_y(h, z.data(), r.data(), 0, rho, 1, 1, 1.0, s));
            TRY(half_sweep_y(h, z.data(), r.data(), 1, rho, 1, 0, 2.0 - rho, s));
            TRY(half_sweep_y(h, z.data(), r.data(), 0, rho, 0, 0, 1.0, s));
        } else {
            for (int p = 0; p < np; ++p) TRY(pmg_copy(h->P[p][0].lv, z[p], r[p], s));
            TRY(exchange(h, 0, z.data(), s));
        }
        return dots(r, z, rz);
    };
    for (int p = 0; p < np; ++p) {
        TRY(pmg_fill(h->P[p][0].lv, u[p], 0.0, s));
        TRY(pmg_copy(h->P[p][0].lv, r[p], f[p], s));
    }
    TRY(dots(r, r, h->res_d));
    TRYC(cudaStreamSynchronize(s), "sync");
    const double r0 = std::sqrt(h->res_h[0]);
    hist[0] = r0;
    *iters = 0;
    *converged = 0;
    if (r0 == 0.0 || r0 < tau) {
        *converged = 1;
        return PMG_OK;
    }
    TRY(precondition(kap));
    for (int p = 0; p < np; ++p) TRY(pmg_copy(h->P[p][0].lv, pp[p], z[p], s));
    TRY(read3());
    if (!(*kap_h > 0.0))
        return err(PMG_ERR_BREAKDOWN, "<r, z> <= 0: preconditioner is not positive definite");
    bool pending = false;
    for (int it = 1; it <= maxiter; ++it) {
        pmg::Trace ti("iteration %d", it);
        for (int p = 0; p < np; ++p)
            TRY(pmg_apply_dot(h->P[p][0].lv, pp[p], q[p], h->scr[0], h->slots + p, s));
        TRY(global_sum(h, pq, s));
        for (int p = 0; p < np; ++p)
            TRY(pmg_cg_update(h->P[p][0].lv, kap, pq, pp[p], q[p], nullptr, r[p], h->scr[0],
                              h->slots + p, s));
        TRY(global_sum(h, rr, s));
        pending = true;
        TRY(read3());   // kappa, <p,q>, ||r||^2
        if (!(*kap_h > 0.0))
            return err(PMG_ERR_BREAKDOWN, "<r, z> <= 0: preconditioner is not positive definite");
        if (!(*pq_h > 0.0))
            return err(PMG_ERR_BREAKDOWN, "<p, A p> <= 0: operator is not positive definite");
        const double rn = std::sqrt(*rr_h);
        hist[it] = rn;
        *iters = it;
        if (rn / r0 < eps || rn < tau) {
            *converged = 1;
            break;
        }
        TRY(precondition(kapn));
        // u += (kappa / pq) p ; p = z + (kappa_new / kappa) p
        for (int p = 0; p < np; ++p)
            TRY(pmg_cg_step(nd[p], kap, pq, kapn, kap, z[p], pp[p], u[p], s));
        pending = false;
        TRYC(cudaMemcpyAsync(kap, kapn, sizeof(double), cudaMemcpyDeviceToDevice, s), "kappa");
    }
    if (pending)
        for (int p = 0; p < np; ++p)
            TRY(pmg_cg_step(nd[p], kap, pq, kap, kap, nullptr, pp[p], u[p], s));
    TRY(read3());
    if (!*converged && !(*kap_h > 0.0))
        return err(PMG_ERR_BREAKDOWN, "<r, z> <= 0: preconditioner is not positive definite");
    return PMG_OK;
}

template <class Fn>
int on_stream(pmg_phier *h, void *stream, Fn fn) {
    cudaStream_t st = (cudaStream_t)stream;
    if (st) return fn(st);
    // the legacy default stream cannot be captured: run on the hierarchy's
    // own stream, ordered after / before the caller's work by events
    TRYC(cudaEventRecord(h->ev_in, 0), "event");
    TRYC(cudaStreamWaitEvent(h->own, h->ev_in, 0), "event wait");
    const int rc = fn(h->own);
    TRYC(cudaEventRecord(h->ev_out, h->own), "event");
    TRYC(cudaStreamWaitEvent(0, h->ev_out, 0), "event wait");
    return rc;
}

}  // namespace

extern "C" {

int pmg_exchange_plan(const int *nbr, int phase, int *ops, int *nops) {
    if (!nbr || !ops || !nops || phase < 0 || phase > 1)
        return err(PMG_ERR_VALUE, "exchange_plan: bad arguments");
    // [send a, recv b, send b, recv a]: two strips exchanged with the same
    // peer (2 parts along a periodic axis, or a part that is its own
    // neighbour) pair up under NCCL's in-order matching per peer
    const int a = 2 * phase, b = a + 1;
    int n = 0;
    for (int pass = 0; pass < 2; ++pass) {
        const int sf = pass ? b : a, rf = pass ? a : b;
        if (nbr[sf] >= 0) {
            ops[3 * n] = 0, ops[3 * n + 1] = sf, ops[3 * n + 2] = nbr[sf];
            ++n;
        }
        if (nbr[rf] >= 0) {
            ops[3 * n] = 1, ops[3 * n + 1] = rf, ops[3 * n + 2] = nbr[rf];
            ++n;
        }
    }
    *nops = n;
    return PMG_OK;
}

int pmg_exchange_plan8(const int *nbr8, int *ops, int *nops) {
    if (!nbr8 || !ops || !nops) return err(PMG_ERR_VALUE, "exchange_plan8: bad arguments");
    // per direction d (W, E, S, N, SW, SE, NW, NE): send the strip of side d
    // to the part there, receive the halo of the opposite side from the part
    // there.  Part A's sends to B, in this order, are the directions d with
    // A + d = B; B's receives from A are the sides OPP8[d] of the same d's in
    // the same order -- they pair up under NCCL's in-order matching per peer
    // whatever the grid (2 parts along a periodic axis, a part that is its
    // own neighbour, diagonal neighbours that coincide with face neighbours)
    int n = 0;
    for (int d = 0; d < 8; ++d) {
        if (nbr8[d] >= 0) {
            ops[3 * n] = 0, ops[3 * n + 1] = d, ops[3 * n + 2] = nbr8[d];
            ++n;
        }
        const int r = OPP8[d];
        if (nbr8[r] >= 0) {
            ops[3 * n] = 1, ops[3 * n + 1] = r, ops[3 * n + 2] = nbr8[r];
            ++n;
        }
    }
    *nops = n;
    return PMG_OK;
}

int pmg_comm_available(void) { return nccl() ? 1 : 0; }

int pmg_comm_unique_id(void *id) {
    if (!id) return err(PMG_ERR_VALUE, "null argument");
    const Nccl *n = nccl();
    if (!n) return err(PMG_ERR_VALUE, "libnccl.so.2 is not available");
    ncclUniqueId u;
    TRYN(n->get_unique_id(&u), "ncclGetUniqueId");
    std::memcpy(id, &u, sizeof(u));
    return PMG_OK;
}

int pmg_comm_create(const void *id, int nranks, int rank, pmg_comm **out) {
    if (!id || !out || nranks < 1 || rank < 0 || rank >= nranks)
        return err(PMG_ERR_VALUE, "comm_create: bad arguments");
    const Nccl *n = nccl();
    if (!n) return err(PMG_ERR_VALUE, "libnccl.so.2 is not available");
    ncclUniqueId u;
    std::memcpy(&u, id, sizeof(u));
    auto *c = new pmg_comm();
    ncclResult_t r = n->comm_init_rank(&c->c, nranks, u, rank);
    if (r != ncclSuccess) {
        delete c;
        return nccl_err(r, "ncclCommInitRank");
    }
    c->nranks = nranks;
    c->rank = rank;
    *out = c;
    return PMG_OK;
}

int pmg_comm_destroy(pmg_comm *c) {
    if (!c) return PMG_OK;
    if (c->c && nccl()) nccl()->comm_destroy(c->c);
    delete c;
    return PMG_OK;
}

int pmg_phier_create(const pmg_level *const *levels, int nlev, int nparts,
                     const pmg_part_desc *parts, const pmg_mg_desc *desc, pmg_comm *comm,
                     int overlap_nx, pmg_phier **out) {
    if (!levels || !parts || !desc || !out || nlev < 1 || nparts < 1)
        return err(PMG_ERR_VALUE, "bad multi-part hierarchy arguments");
    if (desc->nu_pre < 0 || desc->nu_post < 0 || desc->coarse_sweeps < 0)
        return err(PMG_ERR_VALUE, "sweep counts must be non-negative");
    if (!(desc->rho > 0.0 && desc->rho < 2.0))
        return err(PMG_ERR_VALUE, "overrelaxation weight must lie in (0, 2)");
    if (comm && (nparts != 1 || parts[0].worker != comm->rank))
        return err(PMG_ERR_VALUE, "with a communicator each rank holds one part: its rank");
    if (nparts > MAXP)
        return err(PMG_ERR_VALUE, "at most 16 in-process parts per hierarchy");
    int maxw = -1;
    for (int p = 0; p < nparts; ++p) {
        if (parts[p].worker < 0 || (p && parts[p].worker <= parts[p - 1].worker))
            return err(PMG_ERR_VALUE, "parts must be listed in ascending worker order");
        maxw = std::max(maxw, parts[p].worker);
        for (int a = 0; a < 4; ++a) maxw = std::max(maxw, parts[p].nbr[a]);
        for (int a = 0; a < 4; ++a) {
            // diagonal a = SW, SE, NW, NE lies across x side (a & 1) and y side 2 + (a >> 1)
            maxw = std::max(maxw, parts[p].diag[a]);
            const bool both = parts[p].nbr[a & 1] >= 0 && parts[p].nbr[2 + (a >> 1)] >= 0;
            if (both != (parts[p].diag[a] >= 0))
                return err(PMG_ERR_VALUE, "a part has a diagonal neighbour exactly where it has "
                                          "both face neighbours (pmg_part_desc.diag)");
        }
    }
    if (comm && maxw >= comm->nranks)
        return err(PMG_ERR_VALUE, "a neighbour worker is not a rank of the communicator");
    pmg_phier *h = new pmg_phier();
    h->np = nparts;
    h->nlev = nlev;
    h->d = *desc;
    h->comm = comm;
    h->overlap_nx = overlap_nx;
    h->mode_gen = pmg::g_mode_gen;
    h->local.assign(maxw + 1, -1);
    for (int p = 0; p < nparts; ++p) {
        h->worker.push_back(parts[p].worker);
        h->nbr.push_back({parts[p].nbr[0], parts[p].nbr[1], parts[p].nbr[2], parts[p].nbr[3]});
        h->diag.push_back({parts[p].diag[0], parts[p].diag[1], parts[p].diag[2], parts[p].diag[3]});
        h->local[parts[p].worker] = p;
    }
    if (!comm)
        for (int p = 0; p < nparts; ++p)
            for (int a = 0; a < 4; ++a) {
                const int nb = h->nbr[p][a];
                if (nb >= 0 && h->local[nb] < 0) {
                    free_phier(h);
                    return err(PMG_ERR_VALUE, "without a communicator every neighbour must be "
                                              "a part of this hierarchy");
                }
                if (nb >= 0 && h->nbr[h->local[nb]][OPP[a]] != parts[p].worker) {
                    free_phier(h);
                    return err(PMG_ERR_VALUE, "neighbour relation is not symmetric");
                }
            }
    if (!comm)   // the in-process exchange walks x then y: the diagonals must agree
        for (int p = 0; p < nparts; ++p)
            for (int a = 0; a < 4; ++a) {
                const int nx_ = h->nbr[p][a & 1];
                if (h->diag[p][a] >= 0 &&
                    h->nbr[h->local[nx_]][2 + (a >> 1)] != h->diag[p][a]) {
                    free_phier(h);
                    return err(PMG_ERR_VALUE, "diagonal neighbour is not the y neighbour of the "
                                              "x neighbour");
                }
            }
    h->P.assign(nparts, std::vector<PL>(nlev));
    cudaError_t e = cudaSuccess;
    int rc = PMG_OK;
    for (int p = 0; p < nparts && !rc && e == cudaSuccess; ++p) {
        for (int c = 0; c < nlev && !rc && e == cudaSuccess; ++c) {
            PL &q = h->P[p][c];
            q.lv = levels[p * nlev + c];
            if (!q.lv) {
                rc = err(PMG_ERR_VALUE, "null level handle");
                break;
            }
            rc = pmg_level_dims(q.lv, &q.nx, &q.ny, &q.nz);
            if (rc) break;
            const PL &q0 = h->P[p][0];
            const PL &r0 = h->P[0][c];
            if (c && (q.nx != (q0.nx >> c) || q.ny != (q0.ny >> c) || q.nz != q0.nz ||
                      (q.nx << c) != q0.nx || (q.ny << c) != q0.ny)) {
                rc = err(PMG_ERR_VALUE, "each level must halve nx and ny at equal nz");
                break;
            }
            if (p && (q.nx != r0.nx || q.ny != r0.ny || q.nz != r0.nz)) {
                rc = err(PMG_ERR_VALUE, "all parts of a level must have the same shape");
                break;
            }
            // a part that is its own neighbour across a side one column
            // wide couples every cell to itself (see pmg_hier_create)
            if ((q.nx == 1 && (h->nbr[p][0] == h->worker[p] || h->nbr[p][1] == h->worker[p])) ||
                (q.ny == 1 && (h->nbr[p][2] == h->worker[p] || h->nbr[p][3] == h->worker[p]))) {
                rc = err(PMG_ERR_VALUE, "a periodic level one column wide is its own neighbour: "
                                        "use fewer levels");
                break;
            }
            const long long nd = pmg_level_field_doubles(q.lv);
            if (c) {
                e = cudaMalloc(&q.u, sizeof(double) * nd);
                if (e == cudaSuccess) e = cudaMalloc(&q.f, sizeof(double) * nd);
                if (e == cudaSuccess) e = cudaMemset(q.u, 0, sizeof(double) * nd);
            }
            for (int a = 0; a < 8 && e == cudaSuccess; ++a) {
                q.fd[a] = a < 4 ? pmg_face_doubles(q.lv, a) : q.nz;
                if ((a < 4 ? h->nbr[p][a] : h->diag[p][a - 4]) < 0 || !comm) continue;
                e = cudaMalloc(&q.sb[a], sizeof(double) * q.fd[a]);
                if (e == cudaSuccess) e = cudaMalloc(&q.rb[a], sizeof(double) * q.fd[a]);
            }
        }
    }
    const long long ps = pmg_partials_size();
    if (!rc && e == cudaSuccess) e = cudaMalloc(&h->scr[0], sizeof(double) * ps);
    if (!rc && e == cudaSuccess) e = cudaMalloc(&h->scr[1], sizeof(double) * 1024);
    if (!rc && e == cudaSuccess)
        e = cudaMalloc(&h->slots, sizeof(double) * (2 * nparts + (comm ? comm->nranks : 0) + 8));
    if (!rc && e == cudaSuccess) e = cudaHostAlloc(&h->res_h, 8 * sizeof(double), cudaHostAllocMapped);
    if (!rc && e == cudaSuccess) e = cudaHostGetDevicePointer((void **)&h->res_d, h->res_h, 0);
    if (!rc && e == cudaSuccess) e = cudaStreamCreateWithFlags(&h->side, cudaStreamNonBlocking);
    if (!rc && e == cudaSuccess) e = cudaStreamCreateWithFlags(&h->own, cudaStreamNonBlocking);
    for (cudaEvent_t *ev : {&h->ev_fork, &h->ev_join, &h->ev_in, &h->ev_out})
        if (!rc && e == cudaSuccess) e = cudaEventCreateWithFlags(ev, cudaEventDisableTiming);
    if (rc || e != cudaSuccess) {
        free_phier(h);
        if (rc) return rc;
        TRYC(e, "multi-part hierarchy allocation");
    }
    if (comm) {
        // one exchange of the coarsest level (its iterate is zero: the ring
        // stays zero) and one all-gather OUTSIDE any stream capture: NCCL
        // sets up its connection to every neighbour rank on first use, and
        // the first use would otherwise be inside the first cycle's capture
        rc = PMG_OK;
        if (nlev > 1) {
            double *x[1] = {h->P[0][nlev - 1].u};
            rc = exchange(h, nlev - 1, x, h->own);
        }
        if (!rc) rc = global_sum(h, h->slots + 1, h->own);
        if (!rc && cudaStreamSynchronize(h->own) != cudaSuccess)
            rc = err(PMG_ERR_CUDA, "communicator warm-up");
        h->exchanges = 0;
        if (rc) {
            free_phier(h);
            return rc;
        }
    }
    *out = h;
    return PMG_OK;
}

int pmg_phier_destroy(pmg_phier *h) {
    if (h) free_phier(h);
    return PMG_OK;
}

int pmg_phier_mg_solve(pmg_phier *h, const double *const *f, double *const *u, double eps,
                       int maxiter, double *hist, int *iters, int *converged, void *stream) {
    if (!h || !f || !u || !hist || !iters || !converged) return err(PMG_ERR_VALUE, "null argument");
    if (maxiter < 0 || !(eps > 0.0)) return err(PMG_ERR_VALUE, "need eps > 0 and maxiter >= 0");
    for (int p = 0; p < h->np; ++p)
        if (!f[p] || !u[p]) return err(PMG_ERR_VALUE, "null field");
    sync_mode(h);
    pmg::Trace tr("pmg_phier_mg_solve");
    h->clock.reset();
    return on_stream(h, stream, [&](cudaStream_t s) {
        return mg_solve_on(h, f, u, eps, maxiter, hist, iters, converged, s);
    });
}

int pmg_phier_pcg_solve(pmg_phier *h, const double *const *f, double *const *u, double eps,
                        int maxiter, double tau, int precond, double rho, double *hist, int *iters,
                        int *converged, void *stream) {
    if (!h || !f || !u || !hist || !iters || !converged) return err(PMG_ERR_VALUE, "null argument");
    if (!(eps > 0.0 && eps < 1.0)) return err(PMG_ERR_VALUE, "relative tolerance must lie in (0, 1)");
    if (precond && !(rho > 0.0 && rho < 2.0))
        return err(PMG_ERR_VALUE, "overrelaxation weight must lie in (0, 2)");
    sync_mode(h);
    pmg::Trace tr("pmg_phier_pcg_solve");
    return on_stream(h, stream, [&](cudaStream_t s) {
        return pcg_solve_on(h, f, u, eps, maxiter, tau, precond, rho, hist, iters, converged, s);
    });
}

int pmg_phier_vcycle(pmg_phier *h, double *const *u, const double *const *f, int first,
                     void *stream) {
    if (!h || !u || !f) return err(PMG_ERR_VALUE, "null argument");
    sync_mode(h);
    if (first && !(h->d.rho == 1.0 && h->nlev > 1 && h->d.nu_pre >= 1))
        return err(PMG_ERR_VALUE, "first = 1 needs rho = 1, nu_pre >= 1 and two levels");
    return on_stream(h, stream, [&](cudaStream_t s) { return vcycle(h, 0, u, f, first != 0, s); });
}

int pmg_phier_halo_exchange(pmg_phier *h, int level, double *const *fields, void *stream) {
    if (!h || !fields || level < 0 || level >= h->nlev) return err(PMG_ERR_VALUE, "bad arguments");
    return on_stream(h, stream, [&](cudaStream_t s) { return exchange(h, level, fields, s); });
}

int pmg_phier_dot(pmg_phier *h, int level, const double *const *a, const double *const *b,
                  double *out, void *stream) {
    if (!h || !a || !b || !out || level < 0 || level >= h->nlev)
        return err(PMG_ERR_VALUE, "bad arguments");
    return on_stream(h, stream, [&](cudaStream_t s) {
        for (int p = 0; p < h->np; ++p)
            TRY(pmg_dot(h->P[p][level].lv, a[p], b[p], h->scr[0], h->slots + p, s));
        return global_sum(h, out, s);
    });
}

long long pmg_phier_replayed_launches(const pmg_phier *h) { return h ? h->replayed : -1; }

int pmg_phier_cycle_times(const pmg_phier *h, double *ms, int cap) {
    if (!h || (cap > 0 && !ms)) return -1;
    return h->clock.copy_out(ms, cap);
}
long long pmg_phier_exchanges(const pmg_phier *h) { return h ? h->exchanges : -1; }

}  // extern "C"
