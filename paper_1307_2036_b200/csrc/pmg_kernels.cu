// libpmg device kernels for B200 (sm_100a).
//
// Every kernel is HBM-bound fp64 stencil / tridiagonal / BLAS-1 work
// (SURVEY.md section 8d): no tensor cores.  Arithmetic follows the
// reference's numpy expression trees term by term and the library is
// compiled with --fmad=false, so operator, smoother and transfers are
// bit-identical to the reference (see tests/test_gpu_parity.py).
//
// Layout: red/black split, horizontal index fastest (include/pmg.h).
#include <atomic>
#include <cstdlib>

#include <cudaTypedefs.h>

#include "pmg_common.cuh"

namespace pmg {

// kernel launches issued by this library (host-side count, incl. launches
// recorded into CUDA graphs)
std::atomic<long long> g_launches{0};
// tracing mode (pmg_set_tracing, pmg_trace.h)
std::atomic<int> g_trace{0};
int g_smoother_exact = 0;
// bumped whenever the smoother mode changes: kernel variants are chosen when a
// driver graph is captured, so graphs and views cached under another mode are
// discarded (pmg_driver.cu sync_mode)
int g_mode_gen = 0;

// ---------------------------------------------------------------------------
// block reduction helpers (deterministic: fixed shuffle tree + fixed
// block-partial order)
// ---------------------------------------------------------------------------
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    return v;
}

// Sum over the block; result valid in thread 0.  blockDim multiple of 32.
__device__ double block_sum(double v) {
    __shared__ double red[32];
    const int tid = threadIdx.x + blockDim.x * (threadIdx.y + blockDim.y * threadIdx.z);
    const int nthr = blockDim.x * blockDim.y * blockDim.z;
    v = warp_sum(v);
    __syncthreads();
    if ((tid & 31) == 0) red[tid >> 5] = v;
    __syncthreads();
    double s = 0.0;
    if (tid < 32) {
        s = (tid < (nthr >> 5)) ? red[tid] : 0.0;
        s = warp_sum(s);
    }
    return s;
}

__global__ void k_finalize(const double *__restrict__ part, int n, double *__restrict__ out) {
    double s = 0.0;
    for (int t = threadIdx.x; t < n; t += blockDim.x) s += part[t];
    s = block_sum(s);
    if (threadIdx.x == 0) out[0] = s;
}

// ---------------------------------------------------------------------------
// operator apply / residual (stencil.py:127-165, Appendix A of SURVEY)
//
// Block: 32 lanes along h  x  (2*TY) warps = TY rows x 2 colours, so both
// colours of a row strip are streamed by the same CTA (the other-colour
// neighbours are then L1/L2 hits).  Each thread walks its column in k with
// a register window u[k-1], u[k], u[k+1].
// MODE 0: out = A u.  MODE 1: out = f - A u (out may be null).  MODE 2:
// out = A u and partial p.(A p).
// ---------------------------------------------------------------------------
constexpr int AP_TY = 4;

template <bool UNI, int MODE, bool NORM>
__global__ void __launch_bounds__(32 * 2 * AP_TY)
k_apply(Lvl L, const double *__restrict__ u, const double *__restrict__ f,
        double *__restrict__ out, double *__restrict__ partials, int kc) {
    const int lane = threadIdx.x;
    const int c = threadIdx.y & 1;
    const int j = blockIdx.y * AP_TY + (threadIdx.y >> 1);
    const int h = blockIdx.x * 32 + lane;
    const int i = 2 * h + ((j + L.par + c) & 1);
    const int k0 = blockIdx.z * kc;
    const int k1 = min(L.nz, k0 + kc);
    double acc2 = 0.0;
    if (j < L.ny && i < L.nx) {
        const int o = c ^ 1;
        const long long pc = at(L, c, 0, j, h);
        const long long pW = at(L, o, 0, j, (i - 1) >> 1);
        const long long pE = at(L, o, 0, j, (i + 1) >> 1);
        const long long pS = at(L, o, 0, j - 1, h);
        const long long pN = at(L, o, 0, j + 1, h);
        double wxm, wxp, wym, wyp, cv, vhc = 0.0, osw = 0.0;
        if (UNI) {
            wxm = wxp = L.wx0;
            wym = wyp = L.wy0;
            cv = L.csub0;
        } else {
            wxm = L.wx[(long long)j * (L.nx + 1) + i];
            wxp = L.wx[(long long)j * (L.nx + 1) + i + 1];
            wym = L.wy[(long long)j * L.nx + i];
            wyp = L.wy[(long long)(j + 1) * L.nx + i];
            cv = L.vcoef * L.av[(long long)j * L.nx + i];
            vhc = L.vh[(long long)j * L.nx + i];
            osw = L.omega2 * L.sumw[(long long)j * L.nx + i];
        }
        const int nz = L.nz;
        const long long pl = L.plane;
        double um = (k0 > 0) ? u[pc + (long long)(k0 - 1) * pl] : 0.0;
        double u0 = u[pc + (long long)k0 * pl], up = 0.0;
#pragma unroll 4
        for (int k = k0; k < k1; ++k) {
            const long long ko = (long long)k * pl;
            up = (k + 1 < nz) ? u[pc + ko + pl] : 0.0;
            double acc = wxm * u[pW + ko];
            acc = acc + wxp * u[pE + ko];
            acc = acc + wym * u[pS + ko];
            acc = acc + wyp * u[pN + ko];
            acc = acc * L.drw[k];
            double d;
            if (UNI) {
                d = L.diag1[k];
            } else {
                d = vhc * L.volprof[k];
                d = d + osw * L.dr[k];
                d = d + cv * (L.vprof[k] + L.vprof[k + 1]);
            }
            double res = d * u0 - acc;
            if (k >= 1) res = res - (UNI ? L.band1[k] : cv * L.vprof[k]) * um;
            if (k + 1 < nz) res = res - (UNI ? L.band1[k + 1] : cv * L.vprof[k + 1]) * up;
            if (MODE == 1) res = f[pc + ko] - res;
            if (out) out[pc + ko] = res;
            if (NORM) acc2 += (MODE == 2) ? u0 * res : res * res;
            um = u0;
            u0 = up;
        }
    }
    if (NORM) {
        const double s = block_sum(acc2);
        if (threadIdx.x == 0 && threadIdx.y == 0)
            partials[(blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x] = s;
    }
}


// ---------------------------------------------------------------------------
// Vectorised column-pair stencil (uniform coefficients): a thread owns the
// adjacent same-colour columns h = 2m, 2m+1 of one row; every row segment it
// needs is one 16-byte load (own u, f, S, N rows) and the W/E neighbours of
// both columns come from the other colour's pair o[2m..2m+1] plus ONE scalar
// (o[2m+2] if the row's shift s = 1, else o[2m-1]).  Same arithmetic and
// order per cell as stencil.py:140-164.
// ---------------------------------------------------------------------------
struct D2 { double x, y; };

__device__ __forceinline__ D2 ld2(const double *p) {
    const double2 v = *reinterpret_cast<const double2 *>(p);
    return D2{v.x, v.y};
}

// per-column coefficients of a column pair (variable levels; uniform levels
// use the level scalars)
struct Col2 {
    double wxm, wxp, wym, wyp, cv, vh, osw;
};

template <bool UNI>
__device__ __forceinline__ Col2 col2_coeffs(const Lvl &L, int i, int j) {
    Col2 C;
    if (UNI) {
        C.wxm = C.wxp = L.wx0;
        C.wym = C.wyp = L.wy0;
        C.cv = L.csub0;
        C.vh = C.osw = 0.0;
    } else {
        C.wxm = L.wx[(long long)j * (L.nx + 1) + i];
        C.wxp = L.wx[(long long)j * (L.nx + 1) + i + 1];
        C.wym = L.wy[(long long)j * L.nx + i];
        C.wyp = L.wy[(long long)(j + 1) * L.nx + i];
        C.cv = L.vcoef * L.av[(long long)j * L.nx + i];
        C.vh = L.vh[(long long)j * L.nx + i];
        C.osw = L.omega2 * L.sumw[(long long)j * L.nx + i];
    }
    return C;
}

// shared 1-D tables of a level: uniform -> drw, diag, band; variable ->
// drw, volprof, dr, vprof
struct Tabs {
    double *drw, *diag, *band, *vol, *dr, *vp;
};

__device__ __forceinline__ void load_tabs(const Lvl &L, const Tabs &T) {
    const int nthr = blockDim.x * blockDim.y;
    for (int t = threadIdx.x + blockDim.x * threadIdx.y; t <= L.nz; t += nthr) {
        if (t < L.nz) T.drw[t] = L.drw[t];
        if (L.uniform) {
            if (t < L.nz) T.diag[t] = L.diag1[t];
            T.band[t] = L.band1[t];
        } else {
            if (t < L.nz) {
                T.vol[t] = L.volprof[t];
                T.dr[t] = L.dr[t];
            }
            T.vp[t] = L.vprof[t];
        }
    }
}

template <int MODE, int KB, bool UNI>
__device__ __forceinline__ double cell_res(const Lvl &L, const Tabs &T, const Col2 &C, int k,
                                           double w, double e, double sn, double nn, double um,
                                           double u0, double up, double fv) {
    const int nz = L.nz;
    const int kk = min(k, nz - 1);
    double acc = C.wxm * w;
    acc = acc + C.wxp * e;
    acc = acc + C.wym * sn;
    acc = acc + C.wyp * nn;
    acc = acc * T.drw[kk];
    double d;
    if (UNI) {
        d = T.diag[kk];
    } else {
        d = C.vh * T.vol[kk];
        d = d + C.osw * T.dr[kk];
        d = d + C.cv * (T.vp[kk] + T.vp[kk + 1]);
    }
    double r = d * u0 - acc;
    if (k >= 1) r = r - (UNI ? T.band[min(k, nz)] : C.cv * T.vp[min(k, nz)]) * um;
    if (k + 1 < nz) r = r - (UNI ? T.band[k + 1] : C.cv * T.vp[k + 1]) * up;
    if (MODE == 1) r = fv - r;
    return r;
}

template <int MODE, int KB, bool UNI = true>
__device__ __forceinline__ void stencil_batch2(
    const Lvl &L, const double *__restrict__ u, const double *__restrict__ f, int k0, int s,
    long long pc, long long po, long long pS, long long pN, long long px, const Tabs &T,
    const Col2 &A, const Col2 &B, double (&r0)[KB], double (&r1)[KB], double (&u0)[KB],
    double (&u1)[KB]) {
    const int nz = L.nz;
    const long long pl = L.plane;
    D2 uc[KB + 2], vo[KB], vs[KB], vn[KB], vf[KB];
    double vx[KB];
    uc[0] = ld2(u + pc - ((k0 > 0) ? pl : 0));
#pragma unroll
    for (int t = 0; t < KB; ++t) {
        const long long ko = (long long)min(t, nz - 1 - k0) * pl;
        uc[t + 1] = ld2(u + pc + ko);
        vo[t] = ld2(u + po + ko);
        vx[t] = u[px + ko];
        vs[t] = ld2(u + pS + ko);
        vn[t] = ld2(u + pN + ko);
        if (MODE == 1) vf[t] = ld2(f + pc + ko);
    }
    uc[KB + 1] = ld2(u + pc + (long long)min(KB, nz - 1 - k0) * pl);
#pragma unroll
    for (int t = 0; t < KB; ++t) {
        const int k = k0 + t;
        // W/E of column 2m (a) and 2m+1 (b)
        const double wa = s ? vo[t].x : vx[t];
        const double ea = s ? vo[t].y : vo[t].x;
        const double wb = ea;
        const double eb = s ? vx[t] : vo[t].y;
        u0[t] = uc[t + 1].x;
        u1[t] = uc[t + 1].y;
        r0[t] = cell_res<MODE, KB, UNI>(L, T, A, k, wa, ea, vs[t].x, vn[t].x, uc[t].x,
                                        uc[t + 1].x, uc[t + 2].x, MODE == 1 ? vf[t].x : 0.0);
        r1[t] = cell_res<MODE, KB, UNI>(L, T, B, k, wb, eb, vs[t].y, vn[t].y, uc[t].y,
                                        uc[t + 1].y, uc[t + 2].y, MODE == 1 ? vf[t].y : 0.0);
    }
}

// tile = 64 columns x AP_TY rows x 2 colours, column-pair threads walk k
template <int MODE, bool NORM, int KB, bool UNI = true>
__global__ void __launch_bounds__(32 * 2 * AP_TY, 2)
k_apply_v(Lvl L, const double *__restrict__ u, const double *__restrict__ f,
          double *__restrict__ out, double *__restrict__ partials, int hx, int jy, int ntiles,
          int kcs) {
    __shared__ double s_drw[256], s_a[257], s_b[257], s_c[257];
    const Tabs T{s_drw, s_a, s_b, s_a, s_b, s_c};
    load_tabs(L, T);
    __syncthreads();
    const int lane = threadIdx.x;
    const int c = threadIdx.y & 1;
    const int nz = L.nz;
    const int o = c ^ 1;
    const long long pl = L.plane;
    const int nkc = (nz + kcs - 1) / kcs;
    double acc2 = 0.0;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int kcI = tile % nkc;
        const int t2 = tile / nkc;
        const int jb = t2 / hx;
        const int hb = t2 - jb * hx;
        const int j = jb * AP_TY + (threadIdx.y >> 1);
        if (j >= L.ny) continue;
        const int s = (j + L.par + c) & 1;
        const int ncol = ((L.nx - s) + 1) / 2;          // columns of this colour in row j
        const int m = hb * 32 + lane;
        const bool act = 2 * m < ncol;
        const int mm = act ? m : (ncol - 1) / 2;
        const int h = 2 * mm;
        const bool two = act && (h + 1 < ncol);
        const int kbeg = kcI * kcs, kend = min(nz, kbeg + kcs);
        const Col2 A = col2_coeffs<UNI>(L, 2 * h + s, j);
        const Col2 B = col2_coeffs<UNI>(L, min(2 * h + 2 + s, L.nx - 1), j);
        long long pc = at(L, c, kbeg, j, h);
        long long po = at(L, o, kbeg, j, h);
        long long pS = at(L, o, kbeg, j - 1, h);
        long long pN = at(L, o, kbeg, j + 1, h);
        long long px = at(L, o, kbeg, j, s ? h + 2 : h - 1);
        for (int k0 = kbeg; k0 < kend; k0 += KB) {
            double r0[KB], r1[KB], u0[KB], u1[KB];
            stencil_batch2<MODE, KB, UNI>(L, u, f, k0, s, pc, po, pS, pN, px, T, A, B, r0, r1,
                                          u0, u1);
            if (act) {
#pragma unroll
                for (int t = 0; t < KB; ++t) {
                    if (k0 + t < kend) {
                        const long long q = pc + (long long)t * pl;
                        if (out) {
                            if (two) {
                                *reinterpret_cast<double2 *>(out + q) = make_double2(r0[t], r1[t]);
                            } else {
                                out[q] = r0[t];
                            }
                        }
                        if (NORM) {
                            acc2 += (MODE == 2) ? u0[t] * r0[t] : r0[t] * r0[t];
                            if (two) acc2 += (MODE == 2) ? u1[t] * r1[t] : r1[t] * r1[t];
                        }
                    }
                }
            }
            const long long step = (long long)KB * pl;
            pc += step; po += step; pS += step; pN += step; px += step;
        }
    }
    if (NORM) {
        const double s2 = block_sum(acc2);
        if (threadIdx.x == 0 && threadIdx.y == 0) partials[blockIdx.x] = s2;
    }
}

// Convergence norm ||f - A u||^2 (uniform coefficients, nz a multiple of
// KB): k_apply_v's column-pair tiles with a lean inner loop -- the k-plane
// stride a compile-time constant (PLC, 0 = runtime), per-level tables read
// once for both cells, the vertical couplings as zero-padded tables
// (bm[k] = band[k] for k >= 1 else 0, bp[k] = band[k+1] for k < nz-1 else 0)
// so no per-cell predicates.  Same operation order as cell_res (the padded
// terms subtract an exact zero).  Partial sums per CTA in a fixed order.
// MODE 1: ||f - A u||^2 only; MODE 2: out = A u and u . (A u) (CG's
// q = A p with <p, q>, krylov.py:139-140).
template <int KB, int PLC, int MINB, int MODE = 1>
__global__ void __launch_bounds__(32 * 2 * AP_TY, MINB)
k_norm_v(Lvl L, const double *__restrict__ u, const double *__restrict__ f,
         double *__restrict__ partials, int hx, int jy, int ntiles, int kcs,
         double *__restrict__ out) {
    __shared__ double s_drw[256], s_dg[256], s_bm[256], s_bp[256];
    const int nz = L.nz;
    for (int t = threadIdx.x + blockDim.x * threadIdx.y; t < nz; t += blockDim.x * blockDim.y) {
        s_drw[t] = L.drw[t];
        s_dg[t] = L.diag1[t];
        s_bm[t] = (t >= 1) ? L.band1[t] : 0.0;
        s_bp[t] = (t + 1 < nz) ? L.band1[t + 1] : 0.0;
    }
    __syncthreads();
    const int lane = threadIdx.x;
    const int c = threadIdx.y & 1;
    const int o = c ^ 1;
    const long long pl = PLC ? (long long)PLC : L.plane;
    const int nkc = nz / kcs;
    const double wx = L.wx0, wy = L.wy0;
    double acc2 = 0.0;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int kcI = tile % nkc;
        const int t2 = tile / nkc;
        const int jb = t2 / hx;
        const int hb = t2 - jb * hx;
        const int j = jb * AP_TY + (threadIdx.y >> 1);
        if (j >= L.ny) continue;
        const int s = (j + L.par + c) & 1;
        const int ncol = ((L.nx - s) + 1) / 2;
        const int m = hb * 32 + lane;
        const bool act = 2 * m < ncol;
        const int mm = act ? m : (ncol - 1) / 2;
        const int h = 2 * mm;
        const bool two = act && (h + 1 < ncol);
        const int kbeg = kcI * kcs, kend = kbeg + kcs;
        const double *pc = u + at(L, c, kbeg, j, h);
        const double *pf = f + at(L, c, kbeg, j, h);
        const double *po = u + at(L, o, kbeg, j, h);
        const double *pS = u + at(L, o, kbeg, j - 1, h);
        const double *pN = u + at(L, o, kbeg, j + 1, h);
        const double *px = u + at(L, o, kbeg, j, s ? h + 2 : h - 1);
        D2 um = ld2(pc - ((kbeg > 0) ? pl : 0));
        for (int k0 = kbeg; k0 < kend; k0 += KB) {
            D2 uc[KB + 1], vo[KB], vs[KB], vn[KB], vf[KB];
            double vx[KB];
#pragma unroll
            for (int t = 0; t < KB; ++t) {
                uc[t] = ld2(pc + t * pl);
                vo[t] = ld2(po + t * pl);
                vx[t] = px[t * pl];
                vs[t] = ld2(pS + t * pl);
                vn[t] = ld2(pN + t * pl);
                if (MODE == 1) vf[t] = ld2(pf + t * pl);
            }
            uc[KB] = ld2(pc + ((k0 + KB < nz) ? KB * pl : (KB - 1) * pl));
#pragma unroll
            for (int t = 0; t < KB; ++t) {
                const int k = k0 + t;
                const double drw = s_drw[k], dg = s_dg[k], bm = s_bm[k], bp = s_bp[k];
                const D2 ul = t ? uc[t - 1] : um;
                const double wa = s ? vo[t].x : vx[t];
                const double ea = s ? vo[t].y : vo[t].x;
                const double eb = s ? vx[t] : vo[t].y;
                double a0 = wx * wa;
                a0 = a0 + wx * ea;
                a0 = a0 + wy * vs[t].x;
                a0 = a0 + wy * vn[t].x;
                a0 = a0 * drw;
                double r0 = dg * uc[t].x - a0;
                r0 = r0 - bm * ul.x;
                r0 = r0 - bp * uc[t + 1].x;
                if (MODE == 1) r0 = vf[t].x - r0;
                double a1 = wx * ea;
                a1 = a1 + wx * eb;
                a1 = a1 + wy * vs[t].y;
                a1 = a1 + wy * vn[t].y;
                a1 = a1 * drw;
                double r1 = dg * uc[t].y - a1;
                r1 = r1 - bm * ul.y;
                r1 = r1 - bp * uc[t + 1].y;
                if (MODE == 1) r1 = vf[t].y - r1;
                if (act) {
                    if (MODE == 1) {
                        acc2 += r0 * r0;
                        if (two) acc2 += r1 * r1;
                    } else {
                        const long long q = (pc - u) + t * pl;
                        if (two) *reinterpret_cast<double2 *>(out + q) = make_double2(r0, r1);
                        else out[q] = r0;
                        acc2 += uc[t].x * r0;
                        if (two) acc2 += uc[t].y * r1;
                    }
                }
            }
            um = uc[KB - 1];
            pc += KB * pl; pf += KB * pl; po += KB * pl; pS += KB * pl; pN += KB * pl;
            px += KB * pl;
        }
    }
    const double s2 = block_sum(acc2);
    if (threadIdx.x == 0 && threadIdx.y == 0) partials[blockIdx.x] = s2;
}

// Vectorised residual + children-sum restriction (uniform): tile = 64
// coarse columns I (= fine h) of coarse row J; warp (row rr, colour c)
// computes the residual of fine columns h = 2m, 2m+1 in fine row 2J + rr;
// children are combined in shared memory in the reference order and each
// thread writes coarse I = 2m and 2m+1 (one per colour array, coalesced).
template <int KB, bool UNI = true>
__global__ void __launch_bounds__(128, 4)
k_residual_restrict_v(Lvl F, Lvl C, const double *__restrict__ u, const double *__restrict__ f,
                      double *__restrict__ cf, int hx, int ntiles, int kcs) {
    __shared__ double s_drw[256], s_a[257], s_b[257], s_c[257];
    __shared__ double rs[4][KB][65];
    const Tabs T{s_drw, s_a, s_b, s_a, s_b, s_c};
    load_tabs(F, T);
    __syncthreads();
    const int lane = threadIdx.x;
    const int ty = threadIdx.y;              // 2 * rr + c
    const int c = ty & 1, rr = ty >> 1;
    const int nz = F.nz;
    const int o = c ^ 1;
    const long long pl = F.plane;
    const int nkc = (nz + kcs - 1) / kcs;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int kcI = tile % nkc;
        const int t2 = tile / nkc;
        const int J = t2 / hx;
        const int hb = t2 - J * hx;
        const int j = 2 * J + rr;
        const int kbeg = kcI * kcs, kend = min(nz, kbeg + kcs);
        const int s = (j + F.par + c) & 1;
        const int m = hb * 32 + lane;                  // coarse I = 2m, 2m+1
        const bool act = 2 * m < C.nx;
        const int h = act ? 2 * m : 2 * ((C.nx - 1) / 2);
        long long pc = at(F, c, kbeg, j, h);
        long long po = at(F, o, kbeg, j, h);
        long long pS = at(F, o, kbeg, j - 1, h);
        long long pN = at(F, o, kbeg, j + 1, h);
        long long px = at(F, o, kbeg, j, s ? h + 2 : h - 1);
        const int slot = 2 * rr + s;
        const Col2 A = col2_coeffs<UNI>(F, 2 * h + s, j);
        const Col2 B = col2_coeffs<UNI>(F, min(2 * h + 2 + s, F.nx - 1), j);
        const int cc0 = (2 * m + J + C.par) & 1;       // colour of coarse I = 2m
        const long long q0 = act ? at(C, cc0, kbeg, J, m) : 0;
        const long long q1 = act ? at(C, cc0 ^ 1, kbeg, J, m) : 0;
        const bool two = act && (2 * m + 1 < C.nx);
        for (int k0 = kbeg; k0 < kend; k0 += KB) {
            double r0[KB], r1[KB], u0[KB], u1[KB];
            stencil_batch2<1, KB, UNI>(F, u, f, k0, s, pc, po, pS, pN, px, T, A, B, r0, r1,
                                       u0, u1);
#pragma unroll
            for (int t = 0; t < KB; ++t) {
                rs[slot][t][2 * lane] = r0[t];
                rs[slot][t][2 * lane + 1] = r1[t];
            }
            __syncthreads();
            for (int t = ty; t < KB; t += 4) {
                const int k = k0 + t;
                if (act && k < kend) {
                    const long long ko = (long long)(k - kbeg) * C.plane;
                    double a = rs[0][t][2 * lane] + rs[1][t][2 * lane];
                    a = a + rs[2][t][2 * lane];
                    a = a + rs[3][t][2 * lane];
                    cf[q0 + ko] = a;
                    if (two) {
                        double b = rs[0][t][2 * lane + 1] + rs[1][t][2 * lane + 1];
                        b = b + rs[2][t][2 * lane + 1];
                        b = b + rs[3][t][2 * lane + 1];
                        cf[q1 + ko] = b;
                    }
                }
            }
            __syncthreads();
            const long long step = (long long)KB * pl;
            pc += step; po += step; pS += step; pN += step; px += step;
        }
    }
}

// Residual + children-sum restriction, one thread per coarse column pair
// (uniform coefficients, fine nx a multiple of 4).  Thread (J, m) owns the
// fine window i = 4m .. 4m+3 of rows 2J, 2J+1: per level it loads both
// colours of the two centre rows as double2 (each colour's pair is the
// other colour's W/E neighbours) plus the two outer W/E scalars, both
// colours of rows 2J-1 and 2J+2 (S/N) and f: 12 double2 + 4 scalars for 8
// residuals, no shared-memory reduction, no barriers.  Vertical
// neighbours slide through registers.  Same cell arithmetic (cell_res,
// stencil.py:140-164) and children order (multigrid.py:210-212) as
// k_residual_restrict_v: bit-identical results.
template <int MINB = 2, bool NORM = false>
__global__ void __launch_bounds__(128, MINB)
k_residual_restrict_q(Lvl F, Lvl C, const double *__restrict__ u, const double *__restrict__ f,
                      double *__restrict__ cf, int mb32, int ntiles, int kcs,
                      double *__restrict__ partials) {
    // NORM: the convergence residual ||f - A u||^2 instead of the
    // restriction (C describes the row-pair / column-quad grid only)
    double acc2 = 0.0;
    __shared__ double s_drw[256], s_a[257], s_b[257], s_c[257];
    const Tabs T{s_drw, s_a, s_b, s_a, s_b, s_c};
    load_tabs(F, T);
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int nwarp = gridDim.x * (blockDim.x >> 5);
    const int nz = F.nz;
    const long long pl = F.plane;
    const int nkc = (nz + kcs - 1) / kcs;
    const int npair = C.nx >> 1;
    const Col2 W = col2_coeffs<true>(F, 0, 0);
    for (int wt = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); wt < ntiles; wt += nwarp) {
        const int kcI = wt % nkc;
        const int t2 = wt / nkc;
        const int J = t2 / mb32;
        const int m0 = (t2 - J * mb32) * 32;
        const bool act = m0 + lane < npair;
        const int m = act ? m0 + lane : npair - 1;
        const int kbeg = kcI * kcs, kend = min(nz, kbeg + kcs);
        const int ja = 2 * J, jb = ja + 1;
        const int cAa = (ja + F.par) & 1, cAb = cAa ^ 1;     // colour at even i, rows ja / jb
        // row bases at level 0 (colour at even i first, then odd i)
        const long long a_e = at(F, cAa, 0, ja, 2 * m), a_o = at(F, cAa ^ 1, 0, ja, 2 * m);
        const long long b_e = at(F, cAb, 0, jb, 2 * m), b_o = at(F, cAb ^ 1, 0, jb, 2 * m);
        // outer W / E neighbours: fine i = 4m - 1 / 4m + 4 (wrapped when the level wraps)
        const int iw = wrapx(F, 4 * m - 1) >> 1, ie = wrapx(F, 4 * m + 4) >> 1;
        const long long al = at(F, cAa ^ 1, 0, ja, iw), ar = at(F, cAa, 0, ja, ie);
        const long long bl = at(F, cAb ^ 1, 0, jb, iw), br = at(F, cAb, 0, jb, ie);
        // row ja-1: even-i colour = cAb (parity flips with j); row jb+1: cAa
        const int js = wrapy(F, ja - 1), jn = wrapy(F, jb + 1);
        const long long s_e = at(F, cAb, 0, js, 2 * m), s_o = at(F, cAa, 0, js, 2 * m);
        const long long n_e = at(F, cAa, 0, jn, 2 * m), n_o = at(F, cAb, 0, jn, 2 * m);
        // f's colour arrays may lie fcs apart instead of cstride (Lvl::fcs)
        const long long fd = F.fcs - F.cstride;
        const double *fa_e = f + a_e + cAa * fd, *fa_o = f + a_o + (cAa ^ 1) * fd;
        const double *fb_e = f + b_e + cAb * fd, *fb_o = f + b_o + (cAb ^ 1) * fd;
        const int cc0 = (2 * m + J + C.par) & 1;
        const long long q0 = at(C, cc0, 0, J, m), q1 = at(C, cc0 ^ 1, 0, J, m);
        // vertical window of the centre values: [0] k-1, [1] k, [2] k+1
        D2 ce[3], co[3], de[3], dd[3];   // row ja even / odd i, row jb even / odd i
        {
            const long long km = (long long)max(kbeg - 1, 0) * pl, k0 = (long long)kbeg * pl;
            ce[0] = ld2(u + a_e + km); co[0] = ld2(u + a_o + km);
            de[0] = ld2(u + b_e + km); dd[0] = ld2(u + b_o + km);
            ce[1] = ld2(u + a_e + k0); co[1] = ld2(u + a_o + k0);
            de[1] = ld2(u + b_e + k0); dd[1] = ld2(u + b_o + k0);
        }
        for (int k = kbeg; k < kend; ++k) {
            const long long ko = (long long)k * pl;
            const long long kp = (long long)min(k + 1, nz - 1) * pl;
            ce[2] = ld2(u + a_e + kp); co[2] = ld2(u + a_o + kp);
            de[2] = ld2(u + b_e + kp); dd[2] = ld2(u + b_o + kp);
            const double xal = u[al + ko], xar = u[ar + ko], xbl = u[bl + ko], xbr = u[br + ko];
            const D2 se = ld2(u + s_e + ko), so = ld2(u + s_o + ko);
            const D2 ne = ld2(u + n_e + ko), no = ld2(u + n_o + ko);
            const D2 fae = ld2(fa_e + ko), fao = ld2(fa_o + ko);
            const D2 fbe = ld2(fb_e + ko), fbo = ld2(fb_o + ko);
            // row ja: cells 4m (ce.x), 4m+1 (co.x), 4m+2 (ce.y), 4m+3 (co.y)
            const double ra0 = cell_res<1, 1, true>(F, T, W, k, xal, co[1].x, se.x, de[1].x,
                                                    ce[0].x, ce[1].x, ce[2].x, fae.x);
            const double ra1 = cell_res<1, 1, true>(F, T, W, k, ce[1].x, ce[1].y, so.x, dd[1].x,
                                                    co[0].x, co[1].x, co[2].x, fao.x);
            const double ra2 = cell_res<1, 1, true>(F, T, W, k, co[1].x, co[1].y, se.y, de[1].y,
                                                    ce[0].y, ce[1].y, ce[2].y, fae.y);
            const double ra3 = cell_res<1, 1, true>(F, T, W, k, ce[1].y, xar, so.y, dd[1].y,
                                                    co[0].y, co[1].y, co[2].y, fao.y);
            // row jb: S neighbours are row ja, N neighbours row jb+1
            const double rb0 = cell_res<1, 1, true>(F, T, W, k, xbl, dd[1].x, ce[1].x, ne.x,
                                                    de[0].x, de[1].x, de[2].x, fbe.x);
            const double rb1 = cell_res<1, 1, true>(F, T, W, k, de[1].x, de[1].y, co[1].x, no.x,
                                                    dd[0].x, dd[1].x, dd[2].x, fbo.x);
            const double rb2 = cell_res<1, 1, true>(F, T, W, k, dd[1].x, dd[1].y, ce[1].y, ne.y,
                                                    de[0].y, de[1].y, de[2].y, fbe.y);
            const double rb3 = cell_res<1, 1, true>(F, T, W, k, de[1].y, xbr, co[1].y, no.y,
                                                    dd[0].y, dd[1].y, dd[2].y, fbo.y);
            if (NORM) {
                if (act) {
                    acc2 += ra0 * ra0; acc2 += ra1 * ra1; acc2 += ra2 * ra2; acc2 += ra3 * ra3;
                    acc2 += rb0 * rb0; acc2 += rb1 * rb1; acc2 += rb2 * rb2; acc2 += rb3 * rb3;
                }
            } else if (act) {
                const long long cko = (long long)k * C.plane;
                double a = ra0 + ra1;
                a = a + rb0;
                a = a + rb1;
                double b = ra2 + ra3;
                b = b + rb2;
                b = b + rb3;
                cf[q0 + cko] = a;
                cf[q1 + cko] = b;
            }
            ce[0] = ce[1]; co[0] = co[1]; de[0] = de[1]; dd[0] = dd[1];
            ce[1] = ce[2]; co[1] = co[2]; de[1] = de[2]; dd[1] = dd[2];
        }
    }
    if (NORM) {
        const double s2 = block_sum(acc2);
        if (threadIdx.x == 0) partials[blockIdx.x] = s2;
    }
}


// Red-only residual + restriction (fast mode, rho = 1): right after a
// black half-sweep with exact line solves the black residual is zero, so
// R r sums only the two red children of each coarse cell (adding the
// black children's exact zeros changes nothing; their computed values are
// rounding noise).  Same thread mapping as k_residual_restrict_q; per
// level it loads the red centre values (vertical windows), the black
// centre / outer / S / N neighbours and f at red cells only: 14 N
// algorithmic bytes instead of 18 N.  PAR = the level's parity (red at
// even i in the even fine rows when 0).
// NORM: instead of the restriction, partials[blockIdx.x] = this CTA's sum
// of (f - A u)^2 over the red cells (the lagged driver's check-only
// convergence norm; C then only describes the column-quad grid).
template <int PAR, int MINB = 2, bool UNI = true, bool NORM = false>
__global__ void __launch_bounds__(128, MINB)
k_residual_restrict_red(Lvl F, Lvl C, const double *__restrict__ u, const double *__restrict__ f,
                        double *__restrict__ cf, int mb32, int ntiles, int kcs,
                        double *__restrict__ partials) {
    double acc2 = 0.0;
    __shared__ double s_drw[256], s_a[257], s_b[257], s_c[257];
    const Tabs T{s_drw, s_a, s_b, s_a, s_b, s_c};
    load_tabs(F, T);
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int nwarp = gridDim.x * (blockDim.x >> 5);
    const int nz = F.nz;
    const long long pl = F.plane;
    const int nkc = (nz + kcs - 1) / kcs;
    const int npair = C.nx >> 1;
    const Col2 W = col2_coeffs<true>(F, 0, 0);
    for (int wt = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); wt < ntiles; wt += nwarp) {
        const int kcI = wt % nkc;
        const int t2 = wt / nkc;
        const int J = t2 / mb32;
        const int m0 = (t2 - J * mb32) * 32;
        const bool act = m0 + lane < npair;
        const int m = act ? m0 + lane : npair - 1;
        const int kbeg = kcI * kcs, kend = min(nz, kbeg + kcs);
        const int ja = 2 * J, jb = ja + 1;
        // colour 0 (red) / 1 (black); row ja holds red at even i when PAR = 0
        // red pairs: row ja at i = 4m + PAR, +2; row jb at i = 4m + 1 - PAR, +2
        const long long ra = at(F, 0, 0, ja, 2 * m), rb = at(F, 0, 0, jb, 2 * m);
        const long long ba = at(F, 1, 0, ja, 2 * m), bb = at(F, 1, 0, jb, 2 * m);
        // outer black scalars: row ja W of its first red cell (PAR = 0: i = 4m-1)
        // or E of its last (PAR = 1: i = 4m+4); row jb the other way round
        // (fine i = 4m - 1 / 4m + 4, wrapped when the level wraps)
        const int iw = wrapx(F, 4 * m - 1) >> 1, ie = wrapx(F, 4 * m + 4) >> 1;
        const long long xa = PAR ? at(F, 1, 0, ja, ie) : at(F, 1, 0, ja, iw);
        const long long xb = PAR ? at(F, 1, 0, jb, iw) : at(F, 1, 0, jb, ie);
        // S of row ja = row ja-1 (black at row ja's red positions), N of
        // row jb = row jb+1 (black at row jb's red positions)
        const long long sa = at(F, 1, 0, wrapy(F, ja - 1), 2 * m);
        const long long nb = at(F, 1, 0, wrapy(F, jb + 1), 2 * m);
        const double *fa = f + ra, *fb = f + rb;   // colour 0: no fcs offset
        const int cc0 = (2 * m + J + C.par) & 1;
        const long long q0 = at(C, cc0, 0, J, m), q1 = at(C, cc0 ^ 1, 0, J, m);
        // per-column coefficients of the four red cells (variable levels)
        const int ia = 4 * m + PAR, ib = 4 * m + 1 - PAR;
        const Col2 Wa0 = UNI ? W : col2_coeffs<UNI>(F, ia, ja);
        const Col2 Wa2 = UNI ? W : col2_coeffs<UNI>(F, ia + 2, ja);
        const Col2 Wb0 = UNI ? W : col2_coeffs<UNI>(F, ib, jb);
        const Col2 Wb2 = UNI ? W : col2_coeffs<UNI>(F, ib + 2, jb);
        D2 ca[3], cb[3];   // red pairs of rows ja / jb: [0] k-1, [1] k, [2] k+1
        {
            const long long km = (long long)max(kbeg - 1, 0) * pl, k0 = (long long)kbeg * pl;
            ca[0] = ld2(u + ra + km); cb[0] = ld2(u + rb + km);
            ca[1] = ld2(u + ra + k0); cb[1] = ld2(u + rb + k0);
        }
        for (int k = kbeg; k < kend; ++k) {
            const long long ko = (long long)k * pl;
            const long long kp = (long long)min(k + 1, nz - 1) * pl;
            ca[2] = ld2(u + ra + kp); cb[2] = ld2(u + rb + kp);
            const D2 va = ld2(u + ba + ko), vb = ld2(u + bb + ko);   // black pairs
            const D2 vs = ld2(u + sa + ko), vn = ld2(u + nb + ko);
            const double xao = u[xa + ko], xbo = u[xb + ko];
            const D2 ffa = ld2(fa + ko), ffb = ld2(fb + ko);
            double a, b;
            if (PAR == 0) {
                // row ja red at 4m (ca.x), 4m+2 (ca.y); black at 4m+1 (va.x), 4m+3 (va.y)
                // row jb red at 4m+1 (cb.x), 4m+3 (cb.y); black at 4m (vb.x), 4m+2 (vb.y)
                const double r0 = cell_res<1, 1, UNI>(F, T, Wa0, k, xao, va.x, vs.x, vb.x,
                                                      ca[0].x, ca[1].x, ca[2].x, ffa.x);
                const double r2 = cell_res<1, 1, UNI>(F, T, Wa2, k, va.x, va.y, vs.y, vb.y,
                                                      ca[0].y, ca[1].y, ca[2].y, ffa.y);
                const double r1 = cell_res<1, 1, UNI>(F, T, Wb0, k, vb.x, vb.y, va.x, vn.x,
                                                      cb[0].x, cb[1].x, cb[2].x, ffb.x);
                const double r3 = cell_res<1, 1, UNI>(F, T, Wb2, k, vb.y, xbo, va.y, vn.y,
                                                      cb[0].y, cb[1].y, cb[2].y, ffb.y);
                a = r0 + r1;        // ((r(4m,ja) + 0) + 0) + r(4m+1,jb)
                b = r2 + r3;
                if (NORM && act) {
                    acc2 += r0 * r0; acc2 += r1 * r1; acc2 += r2 * r2; acc2 += r3 * r3;
                }
            } else {
                // row ja red at 4m+1 (ca.x), 4m+3 (ca.y); black at 4m (va.x), 4m+2 (va.y)
                // row jb red at 4m (cb.x), 4m+2 (cb.y); black at 4m+1 (vb.x), 4m+3 (vb.y)
                const double r1 = cell_res<1, 1, UNI>(F, T, Wa0, k, va.x, va.y, vs.x, vb.x,
                                                      ca[0].x, ca[1].x, ca[2].x, ffa.x);
                const double r3 = cell_res<1, 1, UNI>(F, T, Wa2, k, va.y, xao, vs.y, vb.y,
                                                      ca[0].y, ca[1].y, ca[2].y, ffa.y);
                const double r0 = cell_res<1, 1, UNI>(F, T, Wb0, k, xbo, vb.x, va.x, vn.x,
                                                      cb[0].x, cb[1].x, cb[2].x, ffb.x);
                const double r2 = cell_res<1, 1, UNI>(F, T, Wb2, k, vb.x, vb.y, va.y, vn.y,
                                                      cb[0].y, cb[1].y, cb[2].y, ffb.y);
                a = r1 + r0;        // ((0 + r(4m+1,ja)) + r(4m,jb)) + 0
                b = r3 + r2;
                if (NORM && act) {
                    acc2 += r1 * r1; acc2 += r0 * r0; acc2 += r3 * r3; acc2 += r2 * r2;
                }
            }
            if (!NORM && act) {
                const long long cko = (long long)k * C.plane;
                cf[q0 + cko] = a;
                cf[q1 + cko] = b;
            }
            ca[0] = ca[1]; cb[0] = cb[1];
            ca[1] = ca[2]; cb[1] = cb[2];
        }
    }
    if (NORM) {
        const double s2 = block_sum(acc2);
        if (threadIdx.x == 0) partials[blockIdx.x] = s2;
    }
}

// ---------------------------------------------------------------------------
// residual fused with children-sum restriction (multigrid.py:278-282):
// each thread owns one coarse column (I, J) and computes the residual of
// its 4 fine children in registers; the fine residual is never stored.
// The children sum keeps the reference order
// ((r(2I,2J) + r(2I+1,2J)) + r(2I,2J+1)) + r(2I+1,2J+1).
// ---------------------------------------------------------------------------
template <bool UNI>
__device__ __forceinline__ double resid_cell(const Lvl &L, const double *__restrict__ u,
                                             const double *__restrict__ f, int i, int j,
                                             int k, double um, double u0, double up) {
    const int c = colour(L, i, j), o = c ^ 1;
    const int h = i >> 1;
    double wxm, wxp, wym, wyp, cv;
    if (UNI) {
        wxm = wxp = L.wx0;
        wym = wyp = L.wy0;
        cv = L.csub0;
    } else {
        wxm = L.wx[(long long)j * (L.nx + 1) + i];
        wxp = L.wx[(long long)j * (L.nx + 1) + i + 1];
        wym = L.wy[(long long)j * L.nx + i];
        wyp = L.wy[(long long)(j + 1) * L.nx + i];
        cv = L.vcoef * L.av[(long long)j * L.nx + i];
    }
    double acc = wxm * u[at(L, o, k, j, (i - 1) >> 1)];
    acc = acc + wxp * u[at(L, o, k, j, (i + 1) >> 1)];
    acc = acc + wym * u[at(L, o, k, j - 1, h)];
    acc = acc + wyp * u[at(L, o, k, j + 1, h)];
    acc = acc * L.drw[k];
    double d;
    if (UNI) {
        d = L.diag1[k];
    } else {
        const long long q = (long long)j * L.nx + i;
        d = L.vh[q] * L.volprof[k];
        d = d + (L.omega2 * L.sumw[q]) * L.dr[k];
        d = d + cv * (L.vprof[k] + L.vprof[k + 1]);
    }
    double res = d * u0 - acc;
    if (k >= 1) res = res - (UNI ? L.band1[k] : cv * L.vprof[k]) * um;
    if (k + 1 < L.nz) res = res - (UNI ? L.band1[k + 1] : cv * L.vprof[k + 1]) * up;
    return f[at(L, c, k, j, h)] - res;
}

template <bool UNI>
__global__ void __launch_bounds__(256)
k_residual_restrict(Lvl F, Lvl C, const double *__restrict__ u, const double *__restrict__ f,
                    double *__restrict__ cf, int kc) {
    const int I = blockIdx.x * blockDim.x + threadIdx.x;
    const int J = blockIdx.z * blockDim.y + threadIdx.y;
    if (I >= C.nx || J >= C.ny) return;
    const int k0 = blockIdx.y * kc;
    const int k1 = min(F.nz, k0 + kc);
    const int i0 = 2 * I, j0 = 2 * J;
    const long long q00 = cell(F, i0, j0, 0), q10 = cell(F, i0 + 1, j0, 0);
    const long long q01 = cell(F, i0, j0 + 1, 0), q11 = cell(F, i0 + 1, j0 + 1, 0);
    const long long pl = F.plane;
    const long long kb = (long long)k0 * pl;
    double m00 = 0, m10 = 0, m01 = 0, m11 = 0;
    if (k0 > 0) {
        m00 = u[q00 + kb - pl]; m10 = u[q10 + kb - pl];
        m01 = u[q01 + kb - pl]; m11 = u[q11 + kb - pl];
    }
    double c00 = u[q00 + kb], c10 = u[q10 + kb], c01 = u[q01 + kb], c11 = u[q11 + kb];
    const long long qc = cell(C, I, J, 0);
    for (int k = k0; k < k1; ++k) {
        const long long ko = (long long)k * pl;
        const bool nx_ = k + 1 < F.nz;
        const double p00 = nx_ ? u[q00 + ko + pl] : 0.0, p10 = nx_ ? u[q10 + ko + pl] : 0.0;
        const double p01 = nx_ ? u[q01 + ko + pl] : 0.0, p11 = nx_ ? u[q11 + ko + pl] : 0.0;
        double s = resid_cell<UNI>(F, u, f, i0, j0, k, m00, c00, p00);
        s = s + resid_cell<UNI>(F, u, f, i0 + 1, j0, k, m10, c10, p10);
        s = s + resid_cell<UNI>(F, u, f, i0, j0 + 1, k, m01, c01, p01);
        s = s + resid_cell<UNI>(F, u, f, i0 + 1, j0 + 1, k, m11, c11, p11);
        cf[qc + (long long)k * C.plane] = s;
        m00 = c00; m10 = c10; m01 = c01; m11 = c11;
        c00 = p00; c10 = p10; c01 = p01; c11 = p11;
    }
}

// ---------------------------------------------------------------------------
// Line smoother half-sweep (smoother.py:122-182).
//
// CTA = 32 columns of one colour in one row (lane = column) x NW warps.
// Phase 1 (all warps, k interleaved across warps): assemble the RHS
//   g = wxm uW; g += wxp uE; g += wym uS; g += wyp uN; g *= drw[k]; g += f
// into shared memory s[k][lane] (coalesced 256-byte row loads per k).
// Phase 2 (warp 0): the exact Thomas recurrence of smoother.py:151-161 per
// lane, forward in shared memory, backward straight to HBM with the relax
// step (smoother.py:163-170).  Several CTAs per SM overlap phase 1 loads of
// some CTAs with the serial phase of others.
// ---------------------------------------------------------------------------
constexpr int HS_THREADS = 128;

template <bool UNI>
__global__ void __launch_bounds__(HS_THREADS, 6)
k_half_sweep(Lvl L, double *__restrict__ u, const double *__restrict__ f, int c, double rho,
             int zero_start, int nbr_zero, double post_scale, int stage) {
    // stage: bit 0 -- the old values (rho != 1) are staged in shared memory,
    // bit 1 -- the pivots of a variable level are; tall columns that do not
    // fit read them from HBM in the serial phase instead (half_sweep_stage)
    extern __shared__ double smem[];
    const int nz = L.nz;
    const bool need_old = !zero_start && rho != 1.0;
    const bool st_old = need_old && (stage & 1), st_inv = !UNI && (stage & 2);
    double *s = smem;                                    // [nz][32]  rhs -> g
    double *so = s + nz * 32;                            // [nz][32]  u_old (rho != 1)
    double *sinv = so + (st_old ? nz * 32 : 0);          // [nz][32]  pivots (variable)
    double *tvp = sinv + (st_inv ? nz * 32 : 0);         // [nz+1]    vprof
    double *tinv = tvp + nz + 1;                         // [nz]      pivots (uniform)
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int j = blockIdx.y;
    const int h = blockIdx.x * 32 + lane;
    const int i = 2 * h + ((j + L.par + c) & 1);
    const bool act = i < L.nx;
    const int o = c ^ 1;
    const long long pc = at(L, c, 0, j, h);
    const long long pl = L.plane;

    for (int t = threadIdx.x; t <= nz; t += blockDim.x) {
        tvp[t] = L.vprof[t];
        if (UNI && t < nz) tinv[t] = L.invd1[t];
    }
    if (act) {
        double wxm = L.wx0, wxp = L.wx0, wym = L.wy0, wyp = L.wy0;
        if (!UNI) {
            wxm = L.wx[(long long)j * (L.nx + 1) + i];
            wxp = L.wx[(long long)j * (L.nx + 1) + i + 1];
            wym = L.wy[(long long)j * L.nx + i];
            wyp = L.wy[(long long)(j + 1) * L.nx + i];
        }
        const long long pW = at(L, o, 0, j, (i - 1) >> 1);
        const long long pE = at(L, o, 0, j, (i + 1) >> 1);
        const long long pS = at(L, o, 0, j - 1, h);
        const long long pN = at(L, o, 0, j + 1, h);
#pragma unroll 4
        for (int k = w; k < nz; k += nw) {
            const long long ko = (long long)k * pl;
            double g;
            if (nbr_zero) {
                g = f[pc + ko];
            } else {
                g = wxm * u[pW + ko];
                g = g + wxp * u[pE + ko];
                g = g + wym * u[pS + ko];
                g = g + wyp * u[pN + ko];
                g = g * L.drw[k];
                g = g + f[pc + ko];
            }
            s[k * 32 + lane] = g;
            if (st_old) so[k * 32 + lane] = u[pc + ko];
            if (st_inv) sinv[k * 32 + lane] = L.invd[pc + ko];
        }
    }
    __syncthreads();
    if (w != 0 || !act) return;
    double cv = L.csub0;
    if (!UNI) cv = L.vcoef * L.av[(long long)j * L.nx + i];
    // forward elimination (smoother.py:151-156)
    auto piv = [&](int k) {
        return UNI ? tinv[k] : (st_inv ? sinv[k * 32 + lane] : L.invd[pc + (long long)k * pl]);
    };
    double g = s[lane] * piv(0);
    s[lane] = g;
#pragma unroll 8
    for (int k = 1; k < nz; ++k) {
        double t = g * cv;
        t = t * tvp[k];
        g = s[k * 32 + lane] + t;
        g = g * piv(k);
        s[k * 32 + lane] = g;
    }
    // back substitution (smoother.py:157-161) + relaxation (163-170)
    const double scale = rho * post_scale;
    const double omr = 1.0 - rho;
    double x = g;
#pragma unroll 8
    for (int k = nz - 1; k >= 0; --k) {
        if (k < nz - 1) {
            double t = x * cv;
            t = t * tvp[k + 1];
            t = t * piv(k);
            x = s[k * 32 + lane] + t;
        }
        double y = x;
        if (zero_start) {
            if (scale != 1.0) y = y * scale;
        } else if (rho != 1.0) {
            y = y * rho;
            y = y + omr * (st_old ? so[k * 32 + lane] : u[pc + (long long)k * pl]);
        }
        u[pc + (long long)k * pl] = y;
    }
}


// shared-memory address and mbarrier helpers (TMA-fed kernels)
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, int count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
                 : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n .reg .pred p;\n"
        "WAIT_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}


// ---------------------------------------------------------------------------
// Line smoother half-sweep, EXACT arithmetic, fed by tensor-map TMA
// (uniform coefficients).
//
// Every warp of the persistent CTA is an independent pipeline over its own
// tiles (32 columns of one row x nz levels, lane = column): lane 0 streams
// chunks of KC levels of the tile's four rows -- f, the other colour's W/E
// row (36 wide), S and N -- into a ring of R shared-memory slots with one
// 3-D cp.async.bulk.tensor box per row and chunk (mbarrier complete_tx),
// R chunks ahead, across tile boundaries; the lanes run the reference's
// sequential Thomas recurrence (smoother.py:137-170, same operation order as
// k_half_sweep: bit-identical) and keep g in a per-warp [nz][32] buffer for
// the back substitution, which streams x to HBM while the ring already
// fills with the next tile.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void tma_box3(void *dst, const CUtensorMap *map, int x, int y, int z,
                                         uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar))
        : "memory");
}


// ---------------------------------------------------------------------------
// Line smoother half-sweep, FAST mode (default, uniform coefficients):
// k-segmented column solve.
//
// CTA = 32 columns x NW warps; warp w owns levels [w*SEG, (w+1)*SEG) of
// every column in registers.  The Thomas recurrences are linear:
//   forward  g_k = iota_k r_k + alpha_k g_{k-1}
//   backward x_k = g_k + mu_k x_{k+1}
// so each warp solves its segment with zero incoming value (h, y), the
// segment ends are joined by a scan of NW terms in shared memory and
// g = h + pf G, x = y + q X fix the segments up (pf, q: products of alpha,
// mu over the segment, per-level tables).  Every warp issues its loads in
// batches of 8 levels x 4 rows (E neighbours by warp shuffle) with the
// full L1 available -- no serial chain, no large shared buffers.  Same
// operator and RHS as smoother.py:137-170; reassociated elimination
// (agrees with the sequential solve to ~1e-15 relative; the exact mode is
// k_half_sweep).
// ---------------------------------------------------------------------------
// Column solve of one tile of the k-segmented smoother, given r[e] =
// iota_k * rhs_k for this warp's levels: local forward, segment scan,
// local backward, segment scan, fix-up, relaxation and store (+ halo
// copies) of k_half_sweep_seg.
template <int SEG, bool DOT = false, bool LEAN = false>
__device__ __forceinline__ void seg_solve_store(
    const Lvl &L, double *__restrict__ u, double (&r)[SEG], const double2 *ti,
    const double2 *tb, const double *tq, double *hend, double *ybeg, int c, int j, int h0,
    int s0, int i, int nact, int kn, long long pc, long long pl, int zero_start, double rho,
    double scale, double omr, const double *__restrict__ f = nullptr, double *dacc = nullptr) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int nz = L.nz;
    const int k0 = w * SEG;
        // ---- local forward: h_k = iota_k r_k + alpha_k h_{k-1} ----
    double hp = 0.0;
#pragma unroll
    for (int e = 0; e < SEG; ++e) {
        if (e < kn) {
            hp = __fma_rn(ti[k0 + e].y, hp, r[e]);
            r[e] = hp;
        }
    }
    if (kn > 0) hend[w * 32 + lane] = hp;
    __syncthreads();
    // incoming G = g_{k0-1}: scan over the segments below
    double G = 0.0;
    for (int sgm = 0; sgm < w; ++sgm)
        G = __fma_rn(tb[min(nz, (sgm + 1) * SEG) - 1].x, G, hend[sgm * 32 + lane]);
    // ---- fix-up + local backward: y_k = g_k + mu_k y_{k+1} ----
    double yp = 0.0;
#pragma unroll
    for (int e = SEG - 1; e >= 0; --e) {
        if (e < kn) {
            const double2 pm = tb[k0 + e];
            const double g = __fma_rn(pm.x, G, r[e]);
            yp = __fma_rn(pm.y, yp, g);
            r[e] = yp;
        }
    }
    if (kn > 0) ybeg[w * 32 + lane] = yp;
    __syncthreads();
    double X = 0.0;
    for (int sgm = nw - 1; sgm > w; --sgm) {
        const int a = sgm * SEG;
        if (a < nz) X = __fma_rn(tq[a], X, ybeg[sgm * 32 + lane]);
    }
    // ---- fix-up, relaxation, store ----
    if (lane < nact) {
#pragma unroll
        for (int e = 0; e < SEG; ++e) {
            if (e < kn) {
                const int k = k0 + e;
                double y = __fma_rn(tq[k], X, r[e]);
                const long long q = pc + (long long)e * pl;
                // LEAN: rho = 1 without zero start at compile time
                if (!LEAN && zero_start) {
                    if (scale != 1.0) y = y * scale;
                } else if (!LEAN && rho != 1.0) {
                    y = y * rho;
                    y = y + omr * u[q];
                }
                u[q] = y;
                if (DOT) *dacc += f[q] * y;       // <rhs, new value> (CG's <r, z>)
            }
        }
    }
}

template <int SEG, int PMG_SEG_B, int MINB, int NBZ = -1, bool FULL = false, int PLC = 0,
          bool DOT = false, int RES = 0, bool LEAN = false>
__global__ void __launch_bounds__(256, MINB)
k_half_sweep_seg(Lvl L, double *__restrict__ u, const double *__restrict__ f, int c, double rho,
                 int zero_start, int nbr_zero_rt, double post_scale, int ntiles, int htiles,
                 double *__restrict__ dotp, double *__restrict__ uw) {
    // DOT: also dotp[blockIdx.x] = sum over this CTA's cells of f * (new u),
    // fixed order (CG's <r, z> fused into the SSOR half-sweeps)
    // RES = 1 (rho = 1, FULL, NBZ = 0): u is only read; the relaxed
    // colour-c values go to uw (same offsets, another buffer), and
    // dotp[blockIdx.x] receives this CTA's sum of (f - A u)^2 over its
    // colour-c cells of the INCOMING iterate: the lagged convergence norm
    // of the previous V-cycle.  The line's right-hand side
    // f + drw (wx (u_W + u_E) + wy (u_S + u_N)) is the sweep's own
    // (g = iota rhs, so rhs = g / iota), and r = rhs - (d u_k - bm u_{k-1}
    // - bp u_{k+1}): 5 fp64 operations per cell on top of the sweep.
    // RES = 3: an ordinary in-place half-sweep that also sums f^2 over its
    // colour-c cells into dotp[blockIdx.x] (||f||^2 of mg_solve's first
    // cycle, multigrid.py:307-309, without a separate pass over f)
    // NBZ = 0/1: neighbours-zero mode fixed at compile time; FULL: every warp
    // owns exactly SEG levels (nz % SEG == 0) -- no per-level predicates;
    // PLC: the k-plane stride as a compile-time constant (0: runtime), so
    // every level's load is base + immediate -- no address arithmetic
    const int nbr_zero = (NBZ >= 0) ? NBZ : nbr_zero_rt;
    extern __shared__ double ssm[];
    const int nz = L.nz;
    // tables, paired for 16-byte shared loads:
    //   tw[k] = (iota drw wx0, iota drw wy0), ti[k] = (iota, alpha),
    //   tb[k] = (pf, mu), tq[k] = q
    double2 *tw = reinterpret_cast<double2 *>(ssm);   // [nz]
    double2 *ti = tw + nz;                              // [nz]
    double2 *tb = ti + nz;                              // [nz]
    double *tq = reinterpret_cast<double *>(tb + nz);   // [nz]
    // segment-end values, double-buffered by tile parity so a warp can
    // start the next tile while others still read the previous scan
    double *hend0 = tq + nz;            // [2][16][32]
    double *ybeg0 = hend0 + 2 * 16 * 32;  // [2][16][32]
    // RES: (1 / iota, diag) and zero-padded vertical couplings (bm, bp) as in k_norm_v
    double2 *tr1 = reinterpret_cast<double2 *>(ybeg0 + 2 * 16 * 32);   // [nz]
    double2 *tr2 = tr1 + nz;                                          // [nz]
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int t = threadIdx.x; t < nz; t += blockDim.x) {
        const double io = L.invd1[t], dd = io * L.drw[t];
        tw[t] = make_double2(dd * L.wx0, dd * L.wy0);
        ti[t] = make_double2(io, L.segtab[t]);
        tb[t] = make_double2(L.segtab[2 * nz + t], L.segtab[nz + t]);
        tq[t] = L.segtab[3 * nz + t];
        if (RES == 1) {
            tr1[t] = make_double2(1.0 / io, L.diag1[t]);
            tr2[t] = make_double2((t >= 1) ? L.band1[t] : 0.0, (t + 1 < nz) ? L.band1[t + 1] : 0.0);
        }
    }
    __syncthreads();
    const int o = c ^ 1;
    const long long pl = PLC ? (long long)PLC : L.plane;
    const int k0 = w * SEG;
    const int kn = FULL ? SEG : min(SEG, nz - k0);   // levels of this warp (may be <= 0)
    const double scale = rho * post_scale;
    const double omr = 1.0 - rho;
    double dacc = 0.0;
    int par = 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x, par ^= 1) {
        double *hend = hend0 + par * 16 * 32;
        double *ybeg = ybeg0 + par * 16 * 32;
        // tile t of the region: row ry0 + (t / htiles) rys, strip
        // rx0 + (t % htiles) rxs (the whole part by default)
        const int tj = t / htiles;
        const int j = L.ry0 + tj * L.rys;
        const int h0 = (L.rx0 + (t - tj * htiles) * L.rxs) * 32;
        const int s0 = (j + L.par + c) & 1;
        const int nact = min(32, ((L.nx - s0) + 1) / 2 - h0);
        const int ln = min(lane, nact - 1);
        const bool lastlane = (ln == nact - 1);
        const int h = h0 + ln;
        const int i = 2 * h + s0;
        const long long pc = at(L, c, k0, j, h);
        const long long pW = at(L, o, k0, j, wrapx(L, i - 1) >> 1);
        const long long pE = at(L, o, k0, j, wrapx(L, i + 1) >> 1);
        const long long pS = at(L, o, k0, wrapy(L, j - 1), h);
        const long long pN = at(L, o, k0, wrapy(L, j + 1), h);
        double r[SEG];
        // RES: incoming colour-c values below / above this warp's levels
        // (bm[0] = 0 and bp[nz-1] = 0 make the clamped loads inert)
        double um = 0.0, un = 0.0, rpend = 0.0, bpend = 0.0;
        if (RES == 1) {
            um = u[pc - ((k0 > 0) ? pl : 0)];
            un = u[pc + ((k0 + SEG < nz) ? SEG : SEG - 1) * pl];
        }
        // ---- RHS assembly, batches of 8 levels ----
#pragma unroll
        for (int b8 = 0; b8 < SEG; b8 += (SEG < PMG_SEG_B ? SEG : PMG_SEG_B)) {
            constexpr int B = SEG < PMG_SEG_B ? SEG : PMG_SEG_B;
            double vf[B], vw[B], vs[B], vn[B], vx[B], vo[B];
#pragma unroll
            for (int e = 0; e < B; ++e) {
                const int kk = b8 + e;
                if (kk < kn) {
                    const long long ko = (long long)kk * pl;
                    vf[e] = f[pc + ko];
                    if (RES == 1) vo[e] = u[pc + ko];
                    if (!nbr_zero) {
                        vw[e] = u[pW + ko];
                        vs[e] = u[pS + ko];
                        vn[e] = u[pN + ko];
                        vx[e] = lastlane ? u[pE + ko] : 0.0;
                    }
                }
            }
#pragma unroll
            for (int e = 0; e < B; ++e) {
                const int kk = b8 + e;
                double ve = __shfl_down_sync(0xffffffffu, nbr_zero ? 0.0 : vw[e], 1);
                if (lastlane) ve = vx[e];
                if (kk < kn) {
                    // iota_k * rhs_k (the forward step's first term)
                    const double2 ia = ti[k0 + kk];
                    double g = ia.x * vf[e];
                    if (!nbr_zero) {
                        const double2 cw = tw[k0 + kk];
                        g = __fma_rn(cw.y, vs[e] + vn[e], g);
                        g = __fma_rn(cw.x, vw[e] + ve, g);
                    }
                    r[b8 + e] = g;
                    if (RES == 3 && lane < nact) dacc = __fma_rn(vf[e], vf[e], dacc);
                }
                if (RES == 1) {
                    // residual of level k - 1 completes with u_k; level k's
                    // waits for u_{k+1}
                    const double2 t1 = tr1[k0 + kk], t2 = tr2[k0 + kk];
                    if (kk > 0) {
                        const double q = __fma_rn(bpend, vo[e], rpend);
                        if (lane < nact) dacc = __fma_rn(q, q, dacc);
                    }
                    const double tu = __fma_rn(-t2.x, um, t1.y * vo[e]);   // d u_k - bm u_{k-1}
                    rpend = __fma_rn(r[b8 + e], t1.x, -tu);                // rhs_k - that
                    bpend = t2.y;
                    um = vo[e];
                }
            }
        }
        if (RES == 1) {
            const double q = __fma_rn(bpend, un, rpend);
            if (lane < nact) dacc = __fma_rn(q, q, dacc);
        }
        seg_solve_store<SEG, DOT, RES == 1 || LEAN>(L, (RES == 1) ? uw : u, r, ti, tb, tq, hend, ybeg, c, j,
                                        h0, s0, i, nact, kn, pc, pl, zero_start, rho, scale, omr,
                                        f, &dacc);
    }
    if (DOT || RES) {
        const double s2 = block_sum(dacc);
        if (threadIdx.x == 0) dotp[blockIdx.x] = s2;
    }
}

// ---------------------------------------------------------------------------
// Row-marching TMA half-sweep (fast mode, uniform, nz = 128: 8 warps x 16
// levels, the column solve of k_half_sweep_seg).  One persistent CTA per SM
// walks units of (strip of 32 columns, band of rows).  Per row j it needs f
// at row j and the other colour's rows j-1, j, j+1 (the W/E neighbours and
// the S/N rows): each row of the other colour is streamed into shared
// memory ONCE by a 3-D tensor-map box (34 columns x nz levels) and reused by
// the three rows that read it -- the register kernel loads it three times
// (L2 hits) and waits on every load batch.  Rings: 4 rows of the other
// colour, 2 rows of f; the boxes for rows j+3 / j+2 are issued as soon as
// step j's right-hand sides are assembled (after the first barrier of its
// column solve), so the copies overlap the solves.  On a wrap view the
// strip-edge neighbours (i = -1, nx) come from a 2-column box of the
// periodic image.  Same arithmetic as k_half_sweep_seg: bit-identical.
// ---------------------------------------------------------------------------
constexpr int BAND_NZ = 128, BAND_W = 32;
static size_t band_smem();
static size_t bandv_smem();

__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
template <int NW>
__device__ __forceinline__ void bar_compute() {   // the NW compute warps only
    asm volatile("bar.sync 1, %0;" ::"n"(32 * NW) : "memory");
}

// RES (rho = 1): the lagged norm's fused red sweep (k_half_sweep_seg's
// RES = 1 mode): u is only read -- the relaxed values go to uw -- and
// partials[blockIdx.x] receives this CTA's sum of (f - A u)^2 over its
// cells of the incoming iterate, formed from the sweep's own line
// right-hand side; each lane loads its column's incoming values (its
// levels and one on either side) at the start of the row step.
// DOT: also partials[blockIdx.x] = this CTA's sum of f * (new value) over
// its cells (CG's <r, z> fused into the SSOR half-sweeps, as
// k_half_sweep_seg's DOT mode); the f row is then released after the store.
// FSQ: partials[blockIdx.x] = this CTA's sum of f^2 (mg_solve's ||f|| in the
// first cycle, k_half_sweep_seg's RES = 3 mode).
// NW: compute warps (8: 16 levels each, the level's own segment tables;
// 16: 8 levels each, 8-level segment products formed in the prologue)
template <int PLC, bool DOT = false, bool FSQ = false, bool LEAN = false, int NW = 8,
          bool RES = false>
__global__ void __launch_bounds__(32 * (NW + 1), 1)
k_half_sweep_band(Lvl L, double *__restrict__ u, int c, double rho, int zero_start,
                  double post_scale, int nstrip, int nband, int band_rows,
                  const __grid_constant__ CUtensorMap mF, const __grid_constant__ CUtensorMap mB,
                  const __grid_constant__ CUtensorMap mE, double *__restrict__ partials,
                  double *__restrict__ uw) {
    constexpr int NZ = BAND_NZ, SEG = NZ / NW, B = 4;
    extern __shared__ __align__(128) double bsm_raw[];
    double *bsm = bsm_raw + (((128u - (smem_u32(bsm_raw) & 127u)) & 127u) >> 3);
    // (TMA box starts must be 16-byte aligned: the other colour's row is
    // two boxes, columns h0 .. h0 + 31 and the 2-column edge the row's
    // colour parity needs -- h0 - 2, h0 - 1 (W of lane 0) or h0 + 32,
    // h0 + 33 (E of lane 31), the periodic image's on a wrap view)
    double *ring = bsm;                              // [4][NZ][32] other colour rows
    double *fring = ring + 4 * NZ * BAND_W;          // [2][NZ][32] f rows
    double *edge = fring + 2 * NZ * 32;              // [4][NZ][2]  edge columns
    double2 *ti = reinterpret_cast<double2 *>(edge + 4 * NZ * 2);
    double2 *tb = ti + NZ;
    double2 *tw = tb + NZ;                           // (iota drw wx0, iota drw wy0)
    double2 *tr1 = tw + NZ;                          // RES: (1 / iota, diag)
    double2 *tr2 = tr1 + NZ;                         // RES: (bm, bp), zero-padded
    double *tq = reinterpret_cast<double *>(tr2 + NZ);
    double *hend = tq + NZ;                           // [NW][32]
    double *ybeg = hend + NW * 32;                    // [NW][32]
    uint64_t *fullB = reinterpret_cast<uint64_t *>(ybeg + NW * 32);  // [4]
    uint64_t *fullF = fullB + 4;                                     // [2]
    uint64_t *emptyB = fullF + 2;                                    // [4]
    uint64_t *emptyF = emptyB + 4;                                   // [2]
    double *wsum = reinterpret_cast<double *>(emptyF + 2);           // DOT: [NW]
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int t = threadIdx.x; t < NZ; t += blockDim.x) {
        const double io = L.invd1[t], dd = io * L.drw[t];
        tw[t] = make_double2(dd * L.wx0, dd * L.wy0);
        if (RES) {
            tr1[t] = make_double2(1.0 / io, L.diag1[t]);
            tr2[t] = make_double2((t >= 1) ? L.band1[t] : 0.0, (t + 1 < NZ) ? L.band1[t + 1] : 0.0);
        }
        ti[t] = make_double2(L.invd1[t], L.segtab[t]);
        double pf = L.segtab[2 * NZ + t], qq = L.segtab[3 * NZ + t];
        if (SEG != 16) {
            // products of alpha from the segment start to t and of mu from
            // the segment end down to t (the host's order, pmg_level_create)
            const int a = t / SEG * SEG, b = a + SEG - 1;
            pf = 1.0;
            for (int k = a; k <= t; ++k) pf *= L.segtab[k];
            qq = 1.0;
            for (int k = b; k >= t; --k) qq *= L.segtab[NZ + k];
        }
        tb[t] = make_double2(pf, L.segtab[NZ + t]);
        tq[t] = qq;
    }
    if (threadIdx.x == 0) {
        for (int q = 0; q < 4; ++q) {
            mbar_init(fullB + q, 1);
            mbar_init(emptyB + q, NW);
        }
        for (int q = 0; q < 2; ++q) {
            mbar_init(fullF + q, 1);
            mbar_init(emptyF + q, NW);
        }
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncthreads();
    const bool wrap = (L.hflags & HF_WRAP) != 0;
    const int hrow = L.nx / 2;                       // cells of one colour per row
    const int nunits = nstrip * nband;
    if (w == NW) {
        // ---- producer warp: streams every row of this CTA's units in the
        // consumers' order; a slot is refilled once all 8 compute warps have
        // released its previous row (empty barriers) ----
        if (lane != 0) return;
        unsigned nb = 0, nf = 0;
        for (int unit = blockIdx.x; unit < nunits; unit += gridDim.x) {
            // units tile the region: strips rx0 + s rxs, rows ry0 .. ry0 + ryn
            const int strip = L.rx0 + (unit % nstrip) * L.rxs, band = unit / nstrip;
            const int h0 = strip * 32;
            const int j0 = L.ry0 + band * band_rows, j1 = min(L.ry0 + L.ryn, j0 + band_rows);
            if (j0 >= j1) continue;
            const bool eleft = wrap && h0 == 0, eright = wrap && h0 + 32 == hrow;
            const uint32_t bytesb = NZ * BAND_W * 8 + NZ * 2 * 8;
            const int xw = eleft ? OFF + hrow - 2 : OFF + h0 - 2;
            const int xe = eright ? OFF : OFF + h0 + 32;
            // black rows j0 - 1 .. j1 and f rows j0 .. j1 - 1, interleaved as
            // the consumers need them: black j0-1, j0, j0+1, f j0, then per
            // step j: black j+2, f j+1
            auto put_b = [&](int r) {
                const int slot = nb & 3;
                if (nb >= 4) mbar_wait(emptyB + slot, ((nb >> 2) + 1) & 1);
                const int rr = wrap ? (r < 0 ? r + L.ny : (r >= L.ny ? r - L.ny : r)) : r;
                fence_proxy_async();
                mbar_expect_tx(fullB + slot, bytesb);
                tma_box3(ring + slot * NZ * BAND_W, &mB, OFF + h0, 0, rr + 1, fullB + slot);
                // as the centre row r, the W neighbour of lane 0 (colour
                // parity 0) or the E neighbour of lane 31 (parity 1)
                tma_box3(edge + slot * NZ * 2, &mE, ((r + L.par + c) & 1) ? xe : xw, 0, rr + 1,
                         fullB + slot);
                ++nb;
            };
            auto put_f = [&](int r) {
                const int slot = nf & 1;
                if (nf >= 2) mbar_wait(emptyF + slot, ((nf >> 1) + 1) & 1);
                fence_proxy_async();
                mbar_expect_tx(fullF + slot, NZ * 32 * 8);
                tma_box3(fring + slot * NZ * 32, &mF, OFF + h0, 0, r + 1, fullF + slot);
                ++nf;
            };
            put_b(j0 - 1);
            put_b(j0);
            for (int j = j0; j < j1; ++j) {
                put_b(j + 1);
                put_f(j);
            }
        }
        return;
    }
    // ---- NW compute warps ----
    const int o = c ^ 1;
    (void)o;
    constexpr long long pl = PLC;                    // plane stride (compile time)
    const int k0 = w * SEG;
    const double scale = rho * post_scale;
    const double omr = 1.0 - rho;
    double dacc = 0.0;
    unsigned seqb = 0, seqf = 0;                     // sequence of the unit's first rows
    for (int unit = blockIdx.x; unit < nunits; unit += gridDim.x) {
        const int strip = L.rx0 + (unit % nstrip) * L.rxs, band = unit / nstrip;
        const int h0 = strip * 32;
        const int j0 = L.ry0 + band * band_rows, j1 = min(L.ry0 + L.ryn, j0 + band_rows);
        if (j0 >= j1) continue;
        // RES: the incoming values of this lane's column (levels k0 - 1 ..
        // k0 + SEG; the clamped out-of-column loads meet zero couplings),
        // loaded one row step ahead so the loads overlap a column solve
        double vo[RES ? SEG : 1], um = 0.0, un = 0.0;
        auto load_old = [&](int jj) {
            const long long p0 = at(L, c, k0, jj, h0 + lane);
#pragma unroll
            for (int e = 0; e < SEG; ++e) vo[e] = u[p0 + (long long)e * pl];
            um = u[p0 - ((k0 > 0) ? pl : 0)];
            un = u[p0 + (long long)((k0 + SEG < NZ) ? SEG : SEG - 1) * pl];
        };
        if (RES) load_old(j0);
        for (int j = j0; j < j1; ++j) {
            const long long pc = at(L, c, k0, j, h0 + lane);
            // black row r of this unit = sequence seqb + r - (j0 - 1)
            for (int r = (j == j0 ? j - 1 : j + 1); r <= j + 1; ++r) {
                const unsigned q = seqb + (unsigned)(r - (j0 - 1));
                mbar_wait(fullB + (q & 3), (q >> 2) & 1);
            }
            const unsigned qf = seqf + (unsigned)(j - j0);
            mbar_wait(fullF + (qf & 1), (qf >> 1) & 1);
            const unsigned qs = seqb + (unsigned)(j - 1 - (j0 - 1));
            const double *Srow = ring + (qs & 3) * NZ * BAND_W;
            const double *Crow = ring + ((qs + 1) & 3) * NZ * BAND_W;
            const double *Nrow = ring + ((qs + 2) & 3) * NZ * BAND_W;
            const double *Ce = edge + ((qs + 1) & 3) * NZ * 2;
            const double *Frow = fring + (qf & 1) * NZ * 32;
            const int s0 = (j + L.par + c) & 1;
            // W / E columns of this lane: h0 + lane - 1 + s0 and h0 + lane + s0
            // (box column 0 = h0); lane 0's W (s0 = 0) and lane 31's E
            // (s0 = 1) come from the edge boxes
            const int iw = max(lane - 1 + s0, 0), ie = min(lane + s0, 31);
            const bool wfix = s0 == 0 && lane == 0, efix = s0 == 1 && lane == 31;
            double r[SEG];
            double rpend = 0.0, bpend = 0.0;
#pragma unroll
            for (int b8 = 0; b8 < SEG; b8 += B) {
#pragma unroll
                for (int e = 0; e < B; ++e) {
                    const int k = k0 + b8 + e;
                    const double *cr = Crow + k * BAND_W;
                    double vw = cr[iw], ve = cr[ie];
                    if (wfix) vw = Ce[k * 2 + 1];
                    if (efix) ve = Ce[k * 2 + 0];
                    const double vs = Srow[k * BAND_W + lane];
                    const double vn = Nrow[k * BAND_W + lane];
                    const double fv = Frow[k * 32 + lane];
                    if (FSQ) dacc = __fma_rn(fv, fv, dacc);
                    double g = ti[k].x * fv;
                    const double2 cw = tw[k];
                    g = __fma_rn(cw.y, vs + vn, g);
                    g = __fma_rn(cw.x, vw + ve, g);
                    r[b8 + e] = g;
                    if (RES) {
                        // residual of level k - 1 completes with u_k; level
                        // k's waits for u_{k+1} (k_half_sweep_seg's order)
                        const double2 t1 = tr1[k], t2 = tr2[k];
                        const double vk = vo[b8 + e];
                        if (b8 + e > 0) {
                            const double q = __fma_rn(bpend, vk, rpend);
                            dacc = __fma_rn(q, q, dacc);
                        }
                        const double tu = __fma_rn(-t2.x, um, t1.y * vk);   // d u_k - bm u_{k-1}
                        rpend = __fma_rn(g, t1.x, -tu);                   // rhs_k - that
                        bpend = t2.y;
                        um = vk;
                    }
                }
            }
            if (RES) {
                const double q = __fma_rn(bpend, un, rpend);
                dacc = __fma_rn(q, q, dacc);
                if (j + 1 < j1) load_old(j + 1);
            }
            // this warp is done with the S row and f row j (and, at the
            // unit's last row, with rows j and j + 1)
            __syncwarp();
            if (lane == 0) {
                mbar_arrive(emptyB + (qs & 3));
                if (!DOT) mbar_arrive(emptyF + (qf & 1));
                if (j == j1 - 1) {
                    mbar_arrive(emptyB + ((qs + 1) & 3));
                    mbar_arrive(emptyB + ((qs + 2) & 3));
                }
            }
            // ---- column solve (seg_solve_store's sequence) ----
            double hp = 0.0;
#pragma unroll
            for (int e = 0; e < SEG; ++e) {
                hp = __fma_rn(ti[k0 + e].y, hp, r[e]);
                r[e] = hp;
            }
            hend[w * 32 + lane] = hp;
            bar_compute<NW>();
            double G = 0.0;
            for (int sgm = 0; sgm < w; ++sgm)
                G = __fma_rn(tb[(sgm + 1) * SEG - 1].x, G, hend[sgm * 32 + lane]);
            double yp = 0.0;
#pragma unroll
            for (int e = SEG - 1; e >= 0; --e) {
                const double2 pm = tb[k0 + e];
                const double g = __fma_rn(pm.x, G, r[e]);
                yp = __fma_rn(pm.y, yp, g);
                r[e] = yp;
            }
            ybeg[w * 32 + lane] = yp;
            bar_compute<NW>();
            double X = 0.0;
            for (int sgm = NW - 1; sgm > w; --sgm)
                X = __fma_rn(tq[sgm * SEG], X, ybeg[sgm * 32 + lane]);
#pragma unroll
            for (int e = 0; e < SEG; ++e) {
                double y = __fma_rn(tq[k0 + e], X, r[e]);
                const long long q = pc + (long long)e * pl;
                // LEAN (and RES): rho = 1 without zero start at compile time
                if (!LEAN && !RES && zero_start) {
                    if (scale != 1.0) y = y * scale;
                } else if (!LEAN && !RES && rho != 1.0) {
                    y = y * rho;
                    y = y + omr * u[q];
                }
                if (RES) uw[q] = y;
                else u[q] = y;
                if (DOT) dacc += Frow[(k0 + e) * 32 + lane] * y;
            }
            if (DOT) {   // the f row is free only now
                __syncwarp();
                if (lane == 0) mbar_arrive(emptyF + (qf & 1));
            }
        }
        seqb += (unsigned)(j1 - j0 + 2);
        seqf += (unsigned)(j1 - j0);
    }
    if (DOT || FSQ || RES) {   // fixed-order reduction over the compute warps
        const double ws = warp_sum(dacc);
        if (lane == 0) wsum[w] = ws;
        bar_compute<NW>();
        if (threadIdx.x == 0) {
            double t = 0.0;
            for (int q = 0; q < NW; ++q) t += wsum[q];
            partials[blockIdx.x] = t;
        }
    }
}


// ---------------------------------------------------------------------------
// FAST half-sweep for VARIABLE coefficients (configs[4]): the k-segmented
// solve of k_half_sweep_seg with per-column weights / vertical coupling and
// the per-cell pivots of the level (L.invd, smoother.py:93-99) loaded with
// the RHS batch; the segment products (pf, q) are formed on the fly and
// published with the boundary values.  nz must be a multiple of SEG.
// ---------------------------------------------------------------------------
// RES = 1: as k_half_sweep_seg's RES mode (u read only, relaxed values into
// uw, dotp[blockIdx.x] = sum over the colour's cells of (f - A u)^2 of the
// incoming iterate); the line RHS g here is the reference's own
// (smoother.py:137-145), so r_k = g_k - (d_k u_k - bm_k u_{k-1} - bp_k
// u_{k+1}) with d_k of stencil.py:105-109 from the column's coefficients.
// RES = 3: in-place sweep that also sums f^2 over the colour (first cycle).
template <int SEG, int NBZ, int RES = 0, bool LEAN = false>
__global__ void __launch_bounds__(512, 1)
k_half_sweep_segv(Lvl L, double *__restrict__ u, const double *__restrict__ f, int c, double rho,
                  int zero_start, int post_scale_unused, double post_scale, int ntiles,
                  int htiles, double *__restrict__ dotp, double *__restrict__ uw) {
    extern __shared__ double vsm[];
    const int nz = L.nz;
    double *tdrw = vsm;                  // [nz]
    double *tvp = tdrw + nz;             // [nz+1]
    double *xh = tvp + ((nz + 2) & ~1);  // [16][32] segment end h
    double *xp = xh + 16 * 32;           // [16][32] segment product of alpha
    double *xy = xp + 16 * 32;           // [16][32] segment start y
    double *xq = xy + 16 * 32;           // [16][32] segment product of mu
    double *tvol = xq + 16 * 32;         // RES: [nz] volprof
    double *tdr = tvol + nz;             // RES: [nz] dr
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int t = threadIdx.x; t <= nz; t += blockDim.x) {
        if (t < nz) tdrw[t] = L.drw[t];
        tvp[t] = L.vprof[t];
        if (RES == 1 && t < nz) {
            tvol[t] = L.volprof[t];
            tdr[t] = L.dr[t];
        }
    }
    __syncthreads();
    double dacc = 0.0;
    // the pivot field keeps the level's own colour stride (a lagged-norm
    // view moves only the iterate's red array: Lvl::fcs)
    const double *invdc = L.invd + (long long)c * (L.fcs - L.cstride);
    const int o = c ^ 1;
    const long long pl = L.plane;
    const int k0 = w * SEG;
    const double scale = rho * post_scale;
    const double omr = 1.0 - rho;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const int j = t / htiles;
        const int h0 = (t - j * htiles) * 32;
        const int s0 = (j + L.par + c) & 1;
        const int nact = min(32, ((L.nx - s0) + 1) / 2 - h0);
        const int ln = min(lane, nact - 1);
        const bool lastlane = (ln == nact - 1);
        const int h = h0 + ln;
        const int i = 2 * h + s0;
        const long long pc = at(L, c, k0, j, h);
        const long long pW = at(L, o, k0, j, wrapx(L, i - 1) >> 1);
        const long long pE = at(L, o, k0, j, wrapx(L, i + 1) >> 1);
        const long long pS = at(L, o, k0, wrapy(L, j - 1), h);
        const long long pN = at(L, o, k0, wrapy(L, j + 1), h);
        const long long q2 = (long long)j * L.nx + i;
        const double wxm = L.wx[(long long)j * (L.nx + 1) + i];
        const double wxp = L.wx[(long long)j * (L.nx + 1) + i + 1];
        const double wym = L.wy[q2];
        const double wyp = L.wy[(long long)(j + 1) * L.nx + i];
        const double cv = L.vcoef * L.av[q2];
        // RES: the column's diagonal coefficients (stencil.py:105-109) and
        // the incoming values next to this warp's levels
        double vh = 0.0, osw = 0.0, um = 0.0, un = 0.0, rpend = 0.0, bpend = 0.0;
        if (RES == 1) {
            vh = L.vh[q2];
            osw = L.omega2 * L.sumw[q2];
            um = u[pc - ((k0 > 0) ? pl : 0)];
            un = u[pc + ((k0 + SEG < nz) ? SEG : SEG - 1) * pl];
        }
        double r[SEG], vi[SEG], pq[SEG];
        constexpr int B = SEG < 4 ? SEG : (RES == 1 ? 2 : 4);
#pragma unroll
        for (int b8 = 0; b8 < SEG; b8 += B) {
            double vf[B], vw[B], vs[B], vn[B], vx[B], vv[B], vo[B];
#pragma unroll
            for (int e = 0; e < B; ++e) {
                const long long ko = (long long)(b8 + e) * pl;
                vf[e] = f[pc + ko];
                vv[e] = invdc[pc + ko];
                if (RES == 1) vo[e] = u[pc + ko];
                if (!NBZ) {
                    vw[e] = u[pW + ko];
                    vs[e] = u[pS + ko];
                    vn[e] = u[pN + ko];
                    vx[e] = lastlane ? u[pE + ko] : 0.0;
                }
            }
#pragma unroll
            for (int e = 0; e < B; ++e) {
                double g;
                if (NBZ) {
                    g = vf[e];
                } else {
                    double ve = __shfl_down_sync(0xffffffffu, vw[e], 1);
                    if (lastlane) ve = vx[e];
                    g = wxm * vw[e];
                    g = g + wxp * ve;
                    g = g + wym * vs[e];
                    g = g + wyp * vn[e];
                    g = g * tdrw[k0 + b8 + e];
                    g = g + vf[e];
                }
                r[b8 + e] = g;
                vi[b8 + e] = vv[e];
                if (RES == 3 && lane < nact) dacc = __fma_rn(vf[e], vf[e], dacc);
                if (RES == 1) {
                    const int k = k0 + b8 + e;
                    const double bm = (k >= 1) ? cv * tvp[k] : 0.0;
                    const double bp = (k + 1 < nz) ? cv * tvp[k + 1] : 0.0;
                    if (b8 + e > 0) {
                        const double q = __fma_rn(bpend, vo[e], rpend);
                        if (lane < nact) dacc = __fma_rn(q, q, dacc);
                    }
                    double d = vh * tvol[k];
                    d = d + osw * tdr[k];
                    d = d + cv * (tvp[k] + tvp[k + 1]);
                    const double tu = __fma_rn(-bm, um, d * vo[e]);   // d u_k - bm u_{k-1}
                    rpend = g - tu;
                    bpend = bp;
                    um = vo[e];
                }
            }
        }
        if (RES == 1) {
            const double q = __fma_rn(bpend, un, rpend);
            if (lane < nact) dacc = __fma_rn(q, q, dacc);
        }
        // local forward h_k = iota_k r_k + alpha_k h_{k-1}, alpha_k = (cv vp_k) iota_k
        double hp = 0.0, pf = 1.0;
#pragma unroll
        for (int e = 0; e < SEG; ++e) {
            const int k = k0 + e;
            const double al = (k == 0) ? 0.0 : (cv * tvp[k]) * vi[e];
            pf *= al;
            pq[e] = pf;
            hp = __fma_rn(al, hp, vi[e] * r[e]);
            r[e] = hp;
        }
        xh[w * 32 + lane] = hp;
        xp[w * 32 + lane] = pf;
        __syncthreads();
        double G = 0.0;
        for (int sg = 0; sg < w; ++sg) G = __fma_rn(xp[sg * 32 + lane], G, xh[sg * 32 + lane]);
        // fix-up g = h + pf G, local backward y_k = g_k + mu_k y_{k+1}
        double yp = 0.0, qq = 1.0;
#pragma unroll
        for (int e = SEG - 1; e >= 0; --e) {
            const int k = k0 + e;
            const double mu = (k + 1 < nz) ? (cv * tvp[k + 1]) * vi[e] : 0.0;
            const double g = __fma_rn(pq[e], G, r[e]);
            qq *= mu;
            pq[e] = qq;
            yp = __fma_rn(mu, yp, g);
            r[e] = yp;
        }
        xy[w * 32 + lane] = yp;
        xq[w * 32 + lane] = qq;
        __syncthreads();
        double X = 0.0;
        for (int sg = nw - 1; sg > w; --sg) X = __fma_rn(xq[sg * 32 + lane], X, xy[sg * 32 + lane]);
        if (lane < nact) {
#pragma unroll
            for (int e = 0; e < SEG; ++e) {
                double y = __fma_rn(pq[e], X, r[e]);
                const long long q = pc + (long long)e * pl;
                // LEAN (and RES = 1): rho = 1 without zero start at compile time
                if (!LEAN && RES != 1 && zero_start) {
                    if (scale != 1.0) y = y * scale;
                } else if (!LEAN && RES != 1 && rho != 1.0) {
                    y = y * rho;
                    y = y + omr * u[q];
                }
                if (RES == 1) uw[q] = y;
                else u[q] = y;
            }
        }
        __syncthreads();
    }
    if (RES) {
        const double s2 = block_sum(dacc);
        if (threadIdx.x == 0) dotp[blockIdx.x] = s2;
    }
}

// ---------------------------------------------------------------------------
// Row-marching TMA half-sweep for VARIABLE coefficients (configs[4]): the
// producer / ring structure of k_half_sweep_band (f row j and the other
// colour's row j+1 as tensor-map boxes, each other-colour row serving as N,
// centre and S row) with k_half_sweep_segv's arithmetic: 16 compute warps of
// 8 levels, the column's face weights and vertical coupling from the 2-D
// factors (smoother.py:137-145 order), the per-cell pivots of the level
// (L.invd), segment products formed on the fly -- bit-identical to
// k_half_sweep_segv<8>.  Per lane, the next row's column coefficients are
// loaded right after this row's RHS assembly and its pivots right after
// this row's backward pass, so both loads overlap a column solve.
// RES = 1 / 3: k_half_sweep_segv's fused-residual / f^2 modes.
// ---------------------------------------------------------------------------
// NBZ: neighbours zero (the first red half-sweep from a zero iterate): no
// other-colour rows are streamed, the line right-hand side is f itself
template <int PLC, int RES = 0, bool LEAN = false, bool NBZ = false>
__global__ void __launch_bounds__(32 * 16, 1)
k_half_sweep_bandv(Lvl L, double *__restrict__ u, int c, double rho, int zero_start,
                   double post_scale, int nstrip, int nband, int band_rows,
                   const __grid_constant__ CUtensorMap mF, const __grid_constant__ CUtensorMap mB,
                   const __grid_constant__ CUtensorMap mE, double *__restrict__ partials,
                   double *__restrict__ uw) {
    constexpr int NW = 16, NZ = BAND_NZ, SEG = NZ / NW, B = 4;
    extern __shared__ __align__(128) double bsm_raw[];
    double *bsm = bsm_raw + (((128u - (smem_u32(bsm_raw) & 127u)) & 127u) >> 3);
    double *ring = bsm;                              // [4][NZ][32] other colour rows
    double *fring = ring + 4 * NZ * BAND_W;          // [2][NZ][32] f rows
    double *edge = fring + 2 * NZ * 32;              // [4][NZ][2]  edge columns
    double *tdrw = edge + 4 * NZ * 2;                // [NZ]   omega2 dr
    double *tvp = tdrw + NZ;                         // [NZ+2] vprof (padded)
    double *tvol = tvp + NZ + 2;                     // RES: [NZ] volprof
    double *tdr = tvol + NZ;                         // RES: [NZ] dr
    double *xh = tdr + NZ;                           // [NW][32] segment end h
    double *xp = xh + NW * 32;                       // [NW][32] segment product of alpha
    double *xy = xp + NW * 32;                       // [NW][32] segment start y
    double *xq = xy + NW * 32;                       // [NW][32] segment product of mu
    uint64_t *fullB = reinterpret_cast<uint64_t *>(xq + NW * 32);   // [4]
    uint64_t *fullF = fullB + 4;                                     // [2]
    double *wsum = reinterpret_cast<double *>(fullF + 2);            // [NW]
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int t = threadIdx.x; t <= NZ; t += blockDim.x) {
        if (t < NZ) {
            tdrw[t] = L.drw[t];
            if (RES == 1) {
                tvol[t] = L.volprof[t];
                tdr[t] = L.dr[t];
            }
        }
        tvp[t] = L.vprof[t];
    }
    if (threadIdx.x == 0) {
        for (int q = 0; q < 4; ++q) mbar_init(fullB + q, 1);
        for (int q = 0; q < 2; ++q) mbar_init(fullF + q, 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncthreads();
    const bool wrap = (L.hflags & HF_WRAP) != 0;
    const int hrow = L.nx / 2;
    const int nunits = nstrip * nband;
    // ---- 16 compute warps; thread 0 also issues the rows' tensor-map
    // boxes.  No warp of its own and no empty barriers: a ring slot is
    // refilled only after the CTA barrier that follows the last right-hand
    // side assembly reading it (the column solve reads registers and the
    // segment arrays, never the rings), so slots are free by construction.
    // At step j (after that barrier) it issues other-colour row j + 3 and f
    // row j + 2; a unit's first step issues its first four rows and two f rows.
    // 512 threads: 128 registers per thread ----
    constexpr long long pl = PLC;
    const int k0 = w * SEG;
    const double scale = rho * post_scale;
    const double omr = 1.0 - rho;
    // the pivot field keeps the level's own colour stride (a lagged-norm
    // view moves only the iterate's red array: Lvl::fcs)
    const double *invdc = L.invd + (long long)c * (L.fcs - L.cstride);
    double dacc = 0.0;
    unsigned seqb = 0, seqf = 0;
    for (int unit = blockIdx.x; unit < nunits; unit += gridDim.x) {
        const int strip = L.rx0 + (unit % nstrip) * L.rxs, band = unit / nstrip;
        const int h0 = strip * 32;
        const int j0 = L.ry0 + band * band_rows, j1 = min(L.ry0 + L.ryn, j0 + band_rows);
        if (j0 >= j1) continue;
        const bool eleft = wrap && h0 == 0, eright = wrap && h0 + 32 == hrow;
        const int xw = eleft ? OFF + hrow - 2 : OFF + h0 - 2;
        const int xe = eright ? OFF : OFF + h0 + 32;
        // tensor-map boxes of other-colour row r (sequence number sq) and f row r
        auto put_b = [&](int r, unsigned sq) {
            const int slot = sq & 3;
            const int rr = wrap ? (r < 0 ? r + L.ny : (r >= L.ny ? r - L.ny : r)) : r;
            fence_proxy_async();
            mbar_expect_tx(fullB + slot, NZ * BAND_W * 8 + NZ * 2 * 8);
            tma_box3(ring + slot * NZ * BAND_W, &mB, OFF + h0, 0, rr + 1, fullB + slot);
            tma_box3(edge + slot * NZ * 2, &mE, ((r + L.par + c) & 1) ? xe : xw, 0, rr + 1,
                     fullB + slot);
        };
        auto put_f = [&](int r, unsigned sq) {
            const int slot = sq & 1;
            fence_proxy_async();
            mbar_expect_tx(fullF + slot, NZ * 32 * 8);
            tma_box3(fring + slot * NZ * 32, &mF, OFF + h0, 0, r + 1, fullF + slot);
        };
        if (threadIdx.x == 0) {
            if (!NBZ) {
                put_b(j0 - 1, seqb);
                put_b(j0, seqb + 1);
                put_b(j0 + 1, seqb + 2);
                if (j0 + 2 <= j1) put_b(j0 + 2, seqb + 3);
            }
            put_f(j0, seqf);
            if (j0 + 1 < j1) put_f(j0 + 1, seqf + 1);
        }
        // the column coefficients and pivots of row jj (loaded a row ahead)
        double wxm, wxp, wym, wyp, cvn, vhn = 0.0, oswn = 0.0;
        double vi[SEG];
        auto load_coef = [&](int jj) {
            const int i = 2 * (h0 + lane) + ((jj + L.par + c) & 1);
            const long long q2 = (long long)jj * L.nx + i;
            wxm = L.wx[(long long)jj * (L.nx + 1) + i];
            wxp = L.wx[(long long)jj * (L.nx + 1) + i + 1];
            wym = L.wy[q2];
            wyp = L.wy[(long long)(jj + 1) * L.nx + i];
            cvn = L.vcoef * L.av[q2];
            if (RES == 1) {
                vhn = L.vh[q2];
                oswn = L.omega2 * L.sumw[q2];
            }
        };
        auto load_piv = [&](int jj) {
            const long long p0 = at(L, c, k0, jj, h0 + lane);
#pragma unroll
            for (int e = 0; e < SEG; ++e) vi[e] = invdc[p0 + (long long)e * pl];
        };
        // RES: the incoming values of this lane's column (as the band kernel)
        double vo[RES == 1 ? SEG : 1], um = 0.0, un = 0.0;
        auto load_old = [&](int jj) {
            const long long p0 = at(L, c, k0, jj, h0 + lane);
#pragma unroll
            for (int e = 0; e < SEG; ++e) vo[e] = u[p0 + (long long)e * pl];
            um = u[p0 - ((k0 > 0) ? pl : 0)];
            un = u[p0 + (long long)((k0 + SEG < NZ) ? SEG : SEG - 1) * pl];
        };
        load_coef(j0);
        load_piv(j0);
        if (RES == 1) load_old(j0);
        for (int j = j0; j < j1; ++j) {
            const long long pc = at(L, c, k0, j, h0 + lane);
            for (int r = (j == j0 ? j - 1 : j + 1); !NBZ && r <= j + 1; ++r) {
                const unsigned q = seqb + (unsigned)(r - (j0 - 1));
                mbar_wait(fullB + (q & 3), (q >> 2) & 1);
            }
            const unsigned qf = seqf + (unsigned)(j - j0);
            mbar_wait(fullF + (qf & 1), (qf >> 1) & 1);
            const unsigned qs = seqb + (unsigned)(j - 1 - (j0 - 1));
            const double *Srow = ring + (qs & 3) * NZ * BAND_W;
            const double *Crow = ring + ((qs + 1) & 3) * NZ * BAND_W;
            const double *Nrow = ring + ((qs + 2) & 3) * NZ * BAND_W;
            const double *Ce = edge + ((qs + 1) & 3) * NZ * 2;
            const double *Frow = fring + (qf & 1) * NZ * 32;
            const int s0 = (j + L.par + c) & 1;
            const int iw = max(lane - 1 + s0, 0), ie = min(lane + s0, 31);
            const bool wfix = s0 == 0 && lane == 0, efix = s0 == 1 && lane == 31;
            const double cv = cvn, vh = vhn, osw = oswn;
            double r[SEG], pq[SEG];
            double rpend = 0.0, bpend = 0.0;
#pragma unroll
            for (int b8 = 0; b8 < SEG; b8 += B) {
#pragma unroll
                for (int e = 0; e < B; ++e) {
                    const int k = k0 + b8 + e;
                    const double *cr = Crow + k * BAND_W;
                    double vw = cr[iw], ve = cr[ie];
                    if (wfix) vw = Ce[k * 2 + 1];
                    if (efix) ve = Ce[k * 2 + 0];
                    const double vs = Srow[k * BAND_W + lane];
                    const double vn = Nrow[k * BAND_W + lane];
                    const double fv = Frow[k * 32 + lane];
                    if (RES == 3) dacc = __fma_rn(fv, fv, dacc);
                    double g;
                    if (NBZ) {
                        g = fv;   // smoother.py:137-145 with neighbours_zero
                    } else {
                        g = wxm * vw;
                        g = g + wxp * ve;
                        g = g + wym * vs;
                        g = g + wyp * vn;
                        g = g * tdrw[k];
                        g = g + fv;
                    }
                    r[b8 + e] = g;
                    if (RES == 1) {
                        const double vk = vo[b8 + e];
                        const double bm = (k >= 1) ? cv * tvp[k] : 0.0;
                        const double bp = (k + 1 < NZ) ? cv * tvp[k + 1] : 0.0;
                        if (b8 + e > 0) {
                            const double q = __fma_rn(bpend, vk, rpend);
                            dacc = __fma_rn(q, q, dacc);
                        }
                        double d = vh * tvol[k];
                        d = d + osw * tdr[k];
                        d = d + cv * (tvp[k] + tvp[k + 1]);
                        const double tu = __fma_rn(-bm, um, d * vk);   // d u_k - bm u_{k-1}
                        rpend = g - tu;
                        bpend = bp;
                        um = vk;
                    }
                }
            }
            if (RES == 1) {
                const double q = __fma_rn(bpend, un, rpend);
                dacc = __fma_rn(q, q, dacc);
                if (j + 1 < j1) load_old(j + 1);
            }
            if (j + 1 < j1) load_coef(j + 1);
            // local forward h_k = iota_k r_k + alpha_k h_{k-1}, alpha_k = (cv vp_k) iota_k
            double hp = 0.0, pf = 1.0;
#pragma unroll
            for (int e = 0; e < SEG; ++e) {
                const int k = k0 + e;
                const double al = (k == 0) ? 0.0 : (cv * tvp[k]) * vi[e];
                pf *= al;
                pq[e] = pf;
                hp = __fma_rn(al, hp, vi[e] * r[e]);
                r[e] = hp;
            }
            xh[w * 32 + lane] = hp;
            xp[w * 32 + lane] = pf;
            bar_compute<NW>();
            // every warp has assembled step j: the slots of other-colour row
            // j - 1 and f row j are free -- for rows j + 3 and j + 2 (two
            // rows of look-ahead in both rings)
            if (threadIdx.x == 0) {
                if (!NBZ && j + 3 <= j1) put_b(j + 3, seqb + (unsigned)(j + 3 - (j0 - 1)));
                if (j + 2 < j1) put_f(j + 2, seqf + (unsigned)(j + 2 - j0));
            }
            double G = 0.0;
            for (int sg = 0; sg < w; ++sg) G = __fma_rn(xp[sg * 32 + lane], G, xh[sg * 32 + lane]);
            double yp = 0.0, qq = 1.0;
#pragma unroll
            for (int e = SEG - 1; e >= 0; --e) {
                const int k = k0 + e;
                const double mu = (k + 1 < NZ) ? (cv * tvp[k + 1]) * vi[e] : 0.0;
                const double g = __fma_rn(pq[e], G, r[e]);
                qq *= mu;
                pq[e] = qq;
                yp = __fma_rn(mu, yp, g);
                r[e] = yp;
            }
            if (j + 1 < j1) load_piv(j + 1);
            xy[w * 32 + lane] = yp;
            xq[w * 32 + lane] = qq;
            bar_compute<NW>();
            double X = 0.0;
            for (int sg = NW - 1; sg > w; --sg)
                X = __fma_rn(xq[sg * 32 + lane], X, xy[sg * 32 + lane]);
#pragma unroll
            for (int e = 0; e < SEG; ++e) {
                double y = __fma_rn(pq[e], X, r[e]);
                const long long q = pc + (long long)e * pl;
                if (!LEAN && RES != 1 && zero_start) {
                    if (scale != 1.0) y = y * scale;
                } else if (!LEAN && RES != 1 && rho != 1.0) {
                    y = y * rho;
                    y = y + omr * u[q];
                }
                if (RES == 1) uw[q] = y;
                else u[q] = y;
            }
        }
        seqb += (unsigned)(j1 - j0 + 2);
        seqf += (unsigned)(j1 - j0);
    }
    if (RES) {   // fixed-order reduction over the compute warps
        const double ws = warp_sum(dacc);
        if (lane == 0) wsum[w] = ws;
        bar_compute<NW>();
        if (threadIdx.x == 0) {
            double t = 0.0;
            for (int q = 0; q < NW; ++q) t += wsum[q];
            partials[blockIdx.x] = t;
        }
    }
}

// per-column pivots of a variable-coefficient level (smoother.py:93-99)
__global__ void k_invd(Lvl L, double *__restrict__ invd) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const int j = blockIdx.y;
    if (i >= L.nx) return;
    const long long q = (long long)j * L.nx + i;
    const double cv = L.vcoef * L.av[q];
    const double vhc = L.vh[q], osw = L.omega2 * L.sumw[q];
    const long long p0 = cell(L, i, j, 0);
    double prev = 0.0;
    for (int k = 0; k < L.nz; ++k) {
        double d = vhc * L.volprof[k];
        d = d + osw * L.dr[k];
        d = d + cv * (L.vprof[k] + L.vprof[k + 1]);
        double v;
        if (k == 0) {
            v = 1.0 / d;
        } else {
            const double sk = L.vprof[k] * cv;
            v = 1.0 / (d - (sk * sk) * prev);
        }
        invd[p0 + (long long)k * L.plane] = v;
        prev = v;
    }
}

// ---------------------------------------------------------------------------
// transfers (multigrid.py:209-246)
// ---------------------------------------------------------------------------
__global__ void k_restrict(Lvl F, Lvl C, const double *__restrict__ fu, double *__restrict__ cu,
                           double weight) {
    const int I = blockIdx.x * blockDim.x + threadIdx.x;
    const int k = blockIdx.y;
    const int J = blockIdx.z;
    if (I >= C.nx) return;
    const int i0 = 2 * I, j0 = 2 * J;
    double a = fu[cell(F, i0, j0, k)] + fu[cell(F, i0 + 1, j0, k)];
    a = a + fu[cell(F, i0, j0 + 1, k)];
    a = a + fu[cell(F, i0 + 1, j0 + 1, k)];
    if (weight != 1.0) a = a * weight;
    cu[cell(C, I, J, k)] = a;
}

// The column-pair prolongation with JB coarse rows per thread: the coarse rows J0-1 ..
// J0+JB form a sliding window (JB + 2 row loads instead of 3 JB), and all
// loads of the thread's rows are issued before any arithmetic.  Same
// arithmetic and order: bit-identical to k_prolong.
template <int JB, int CM = 0>
__global__ void __launch_bounds__(128)
k_prolong_w(Lvl F, Lvl C, const double *__restrict__ cu, double *__restrict__ fu, int add,
            int cmask_rt) {
    // CM: the colour mask at compile time (2 = black only, the V-cycle's
    // case), 0 = runtime
    const int cmask = CM ? CM : cmask_rt;
    const int lane = threadIdx.x & 31;
    const int npair = C.nx >> 1;
    const int m0 = blockIdx.x * 128 + (threadIdx.x & ~31);
    if (m0 >= npair) return;
    const int k = blockIdx.y, J0 = blockIdx.z * JB;
    const int nact = min(32, npair - m0);
    const bool act = lane < nact;
    const int m = m0 + (act ? lane : nact - 1);
    const bool first = lane == 0, last = lane == nact - 1;
    const int ix0 = wrapx(C, 2 * m - 1), ix3 = wrapx(C, 2 * m + 2);
    double e0[JB + 2], e1[JB + 2], xl[JB + 2], xr[JB + 2];
#pragma unroll
    for (int d = 0; d < JB + 2; ++d) {
        const int Y = wrapy(C, min(J0 - 1 + d, C.ny));   // rows past the part: halo / wrap
        e0[d] = cu[cell(C, 2 * m, Y, k)];
        e1[d] = cu[cell(C, 2 * m + 1, Y, k)];
        xl[d] = first ? cu[cell(C, ix0, Y, k)] : 0.0;
        xr[d] = last ? cu[cell(C, ix3, Y, k)] : 0.0;
    }
    const int nj = min(JB, C.ny - J0);
    D2 old[JB][2][2];
    if (add) {
#pragma unroll
        for (int jj = 0; jj < JB; ++jj)
#pragma unroll
            for (int r = 0; r < 2; ++r)
#pragma unroll
                for (int c = 0; c < 2; ++c)
                    if ((cmask >> c & 1) && jj < nj && act)
                        old[jj][r][c] = ld2(fu + at(F, c, k, 2 * (J0 + jj) + r, 2 * m));
    }
#pragma unroll
    for (int jj = 0; jj < JB; ++jj) {
        if (jj >= nj) break;
        double el[3], er[3], a0[3], a1[3];
#pragma unroll
        for (int d = 0; d < 3; ++d) {
            a0[d] = e0[jj + d];
            a1[d] = e1[jj + d];
            el[d] = __shfl_up_sync(0xffffffffu, a1[d], 1);
            er[d] = __shfl_down_sync(0xffffffffu, a0[d], 1);
            if (first) el[d] = xl[jj + d];
            if (last) er[d] = xr[jj + d];
        }
        const int J = J0 + jj;
#pragma unroll
        for (int r = 0; r < 2; ++r) {
            const int j = 2 * J + r;
            const int yn = r ? 2 : 0;
#pragma unroll
            for (int c = 0; c < 2; ++c) {
                if (!(cmask >> c & 1)) continue;
                const int sc = (j + F.par + c) & 1;
                double v[2];
#pragma unroll
                for (int q = 0; q < 2; ++q) {
                    const double cc1 = q ? a1[1] : a0[1], ccn = q ? a1[yn] : a0[yn];
                    const double xc1 = sc ? (q ? er[1] : a1[1]) : (q ? a0[1] : el[1]);
                    const double xcn = sc ? (q ? er[yn] : a1[yn]) : (q ? a0[yn] : el[yn]);
                    double e = 9.0 * cc1;
                    e = e + 3.0 * xc1;
                    e = e + 3.0 * ccn;
                    e = e + xcn;
                    v[q] = e * 0.0625;
                }
                if (act) {
                    const long long qf = at(F, c, k, j, 2 * m);
                    if (add) {
                        v[0] = old[jj][r][c].x + v[0];
                        v[1] = old[jj][r][c].y + v[1];
                    }
                    *reinterpret_cast<double2 *>(fu + qf) = make_double2(v[0], v[1]);
                }
            }
        }
    }
}


__global__ void k_prolong(Lvl F, Lvl C, const double *__restrict__ cu, double *__restrict__ fu,
                          int add, int cmask) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    const int k = blockIdx.y;
    const int j = blockIdx.z;
    // cmask 3: both colours interleaved in a warp; 1 / 2: red / black only
    const int c = (cmask == 3) ? (t & 1) : (cmask >> 1);
    const int h = (cmask == 3) ? (t >> 1) : t;
    const int i = 2 * h + ((j + F.par + c) & 1);
    if (i >= F.nx) return;
    const int I = i >> 1, J = j >> 1;
    const int dI = (i & 1) ? 1 : -1, dJ = (j & 1) ? 1 : -1;
    const double cc = cu[cell(C, I, J, k)];
    const double cx = cu[cell(C, I + dI, J, k)];
    const double cy = cu[cell(C, I, J + dJ, k)];
    const double cd = cu[cell(C, I + dI, J + dJ, k)];
    double e = 9.0 * cc;
    e = e + 3.0 * cx;
    e = e + 3.0 * cy;
    e = e + cd;
    e = e * 0.0625;
    const long long q = at(F, c, k, j, h);
    const double v = add ? fu[q] + e : e;
    fu[q] = v;
}


// ---------------------------------------------------------------------------
// halos (partition.py:158-191)
// ---------------------------------------------------------------------------
__device__ __forceinline__ int hmap(int i, int n, int periodic) {
    if (i < 0) return periodic ? n - 1 : 0;
    if (i >= n) return periodic ? 0 : n - 1;
    return i;
}

// whole ring of a part that is its own neighbour in both directions.
// Work items: first the two y strips (j = -1, ny; i in [-1, nx]) with i
// fastest, then the two x strips (i = -1, nx; j in [0, ny)) with k fastest,
// so consecutive threads touch contiguous memory.  Sources are always owned
// cells (hmap), so both parts run concurrently.
__global__ void k_halo_self(Lvl L, double *__restrict__ d, int px, int py) {
    const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    const int w = 2 * (L.nx + 2);
    const long long ny_items = (long long)w * L.nz;
    const long long nx_items = 2LL * L.ny * L.nz;
    int i, j, k;
    if (t < ny_items) {
        const int q = (int)(t % w);
        k = (int)(t / w);
        i = (q % (L.nx + 2)) - 1;
        j = (q < L.nx + 2) ? -1 : L.ny;
    } else if (t < ny_items + nx_items) {
        const long long u2 = t - ny_items;
        k = (int)(u2 % L.nz);
        const int r = (int)(u2 / L.nz);
        j = r % L.ny;
        i = (r < L.ny) ? -1 : L.nx;
    } else {
        return;
    }
    d[cell(L, i, j, k)] = d[cell(L, hmap(i, L.nx, px), hmap(j, L.ny, py), k)];
}


__global__ void k_pack_face(Lvl L, const double *__restrict__ d, int face, double *__restrict__ buf,
                            int len) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    const int k = blockIdx.y;
    if (t >= len) return;
    int i, j;
    face_pos(L, face, t, false, i, j);
    buf[(long long)k * len + t] = d[cell(L, i, j, k)];
}

__global__ void k_unpack_face(Lvl L, double *__restrict__ d, int face, const double *__restrict__ buf,
                              int len, int mirror) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    const int k = blockIdx.y;
    if (t >= len) return;
    int i, j;
    face_pos(L, face, t, true, i, j);
    double v;
    if (mirror) {
        int si, sj;
        face_pos(L, face, t, false, si, sj);
        v = d[cell(L, si, sj, k)];
    } else {
        v = buf[(long long)k * len + t];
    }
    d[cell(L, i, j, k)] = v;
}


// Vectorised owned-cell dot / norm: owned rows (c, j, k) are contiguous
// [OFF, OFF + nh) segments; a thread covers one double2 of RPB rows at once
// (all loads in flight before the accumulation), grid-stride over row
// blocks in a fixed order (deterministic).  SAME: a == b, loaded once.
template <int RPB, bool SAME>
__global__ void __launch_bounds__(256)
k_dot2(Lvl L, const double *__restrict__ a, const double *__restrict__ b,
       double *__restrict__ partials, int nch) {
    // items = (owned row (c, j, k), chunk of 2 * blockDim elements)
    const int nrows = 2 * L.nz * L.ny;
    const int nitems = nrows * nch;
    const int span = 2 * blockDim.x;
    double s = 0.0;
    for (int i0 = blockIdx.x * RPB; i0 < nitems; i0 += gridDim.x * RPB) {
        double2 va[RPB], vb[RPB];
        int lim[RPB];
#pragma unroll
        for (int q = 0; q < RPB; ++q) {
            const int it = min(i0 + q, nitems - 1);
            const int r = it / nch, ch = it - r * nch;
            const int k = r % L.nz;
            const int cj = r / L.nz;
            const int j = cj % L.ny, c = cj / L.ny;
            const int s0 = (j + L.par + c) & 1;
            const int nh = ((L.nx - s0) + 1) / 2;
            const int e0 = ch * span + 2 * threadIdx.x;
            lim[q] = (i0 + q < nitems) ? nh - e0 : 0;        // valid elements from e0
            const int e = min(e0, max(nh - 2, 0));
            const long long base = at(L, c, k, j, 0);
            va[q] = *reinterpret_cast<const double2 *>(a + base + e);
            vb[q] = SAME ? va[q] : *reinterpret_cast<const double2 *>(b + base + e);
        }
#pragma unroll
        for (int q = 0; q < RPB; ++q) {
            if (lim[q] > 0) s += va[q].x * vb[q].x;
            if (lim[q] > 1) s += va[q].y * vb[q].y;
        }
    }
    s = block_sum(s);
    if (threadIdx.x == 0) partials[blockIdx.x] = s;
}

// block copy between two parts' layouts (coarse-level folding,
// partition.py:194-240): dst cell (di + i, dj + j, k) = src cell
// (si + i, sj + j, k) for i < w, j < h, all k; halo indices allowed
__global__ void k_copy_block(Lvl S, const double *__restrict__ src, Lvl D, double *__restrict__ dst,
                             int si, int sj, int di, int dj, int w, int h) {
    const long long n = (long long)w * h * S.nz;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < n;
         t += (long long)gridDim.x * blockDim.x) {
        const int i = (int)(t % w);
        const int j = (int)((t / w) % h);
        const int k = (int)(t / ((long long)w * h));
        dst[cell(D, di + i, dj + j, k)] = src[cell(S, si + i, sj + j, k)];
    }
}

__global__ void k_fill(long long n, double v, double *__restrict__ y) {
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n;
         e += (long long)gridDim.x * blockDim.x)
        y[e] = v;
}

__global__ void k_axpy(long long n, double a, const double *__restrict__ x, double *__restrict__ y) {
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n;
         e += (long long)gridDim.x * blockDim.x)
        y[e] = y[e] + a * x[e];
}

__global__ void k_xpby(long long n, const double *__restrict__ x, double b, double *__restrict__ y) {
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n;
         e += (long long)gridDim.x * blockDim.x)
        y[e] = b * y[e] + x[e];
}

// p = z + (num/den) p   (krylov.py:157, partition.py:150-155)
__global__ void k_cg_direction(long long n, const double *__restrict__ num,
                               const double *__restrict__ den, const double *__restrict__ z,
                               double *__restrict__ p) {
    const double b = num[0] / den[0];
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n;
         e += (long long)gridDim.x * blockDim.x)
        p[e] = b * p[e] + z[e];
}

// u += (an/ad) p ; p = z + (bn/bd) p over the full allocation: the CG
// iterate update of iteration k (krylov.py:143) deferred into the direction
// update of iteration k+1 (krylov.py:157), which reads p_k anyway.
__global__ void k_cg_up(long long n, const double *__restrict__ an, const double *__restrict__ ad,
                        const double *__restrict__ bn, const double *__restrict__ bd,
                        const double *__restrict__ z, double *__restrict__ p,
                        double *__restrict__ u) {
    const double a = an[0] / ad[0];
    if (z == nullptr) {   // final iterate update only
        for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n;
             e += (long long)gridDim.x * blockDim.x)
            u[e] = u[e] + a * p[e];
        return;
    }
    const double b = bn[0] / bd[0];
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n;
         e += (long long)gridDim.x * blockDim.x) {
        const double pv = p[e];
        u[e] = u[e] + a * pv;
        p[e] = b * pv + z[e];
    }
}

// u += alpha p ; r -= alpha q over the full allocation (halo included, as
// DistField.add_scaled, partition.py:145-148); partial ||r||^2 over owned.
// Rows of the allocation are (c, jj, k) with jj in [0, ny+2), pitch wide.
__global__ void __launch_bounds__(256)
k_cg_update(Lvl L, const double *__restrict__ num, const double *__restrict__ den,
            const double *__restrict__ p, const double *__restrict__ q, double *__restrict__ u,
            double *__restrict__ r, double *__restrict__ partials) {
    const double alpha = num[0] / den[0];
    const double malpha = -alpha;
    const int nrows = 2 * (L.ny + 2) * L.nz;
    double s = 0.0;
    for (int row = blockIdx.x; row < nrows; row += gridDim.x) {
        const int jj = (row / L.nz) % (L.ny + 2);
        const int c = row / ((L.ny + 2) * L.nz);
        const int j = jj - 1;
        const int s0 = (j + L.par + c) & 1;
        const long long base = (long long)row * L.pitch;
        const bool owned_row = (j >= 0 && j < L.ny);
        for (int t = threadIdx.x; t < L.pitch; t += blockDim.x) {
            const long long e = base + t;
            if (u != nullptr) u[e] = u[e] + alpha * p[e];
            const double rv = r[e] + malpha * q[e];
            r[e] = rv;
            const int h = t - OFF;
            if (owned_row && h >= 0 && 2 * h + s0 < L.nx) s += rv * rv;
        }
    }
    s = block_sum(s);
    if (threadIdx.x == 0) partials[blockIdx.x] = s;
}

// Vectorised CG updates (double2, four independent iterations per thread in
// flight): the element arithmetic of k_cg_up / k_cg_update unchanged.
__global__ void __launch_bounds__(256)
k_cg_up_v(long long n2, const double *__restrict__ an, const double *__restrict__ ad,
          const double *__restrict__ bn, const double *__restrict__ bd,
          const double2 *__restrict__ z, double2 *__restrict__ p, double2 *__restrict__ u) {
    const double a = an[0] / ad[0];
    const double b = z ? bn[0] / bd[0] : 0.0;
    const long long stride = (long long)gridDim.x * blockDim.x;
    long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    for (; e + 3 * stride < n2; e += 4 * stride) {
        double2 pv[4], uv[4], zv[4];
#pragma unroll
        for (int t = 0; t < 4; ++t) {
            pv[t] = p[e + t * stride];
            uv[t] = u[e + t * stride];
            if (z) zv[t] = z[e + t * stride];
        }
#pragma unroll
        for (int t = 0; t < 4; ++t) {
            double2 nu;
            nu.x = uv[t].x + a * pv[t].x;
            nu.y = uv[t].y + a * pv[t].y;
            u[e + t * stride] = nu;
            if (z) {
                double2 np;
                np.x = b * pv[t].x + zv[t].x;
                np.y = b * pv[t].y + zv[t].y;
                p[e + t * stride] = np;
            }
        }
    }
    for (; e < n2; e += stride) {
        const double2 pv = p[e], uv = u[e];
        u[e] = make_double2(uv.x + a * pv.x, uv.y + a * pv.y);
        if (z) {
            const double2 zv = z[e];
            p[e] = make_double2(b * pv.x + zv.x, b * pv.y + zv.y);
        }
    }
}

// one warp per allocation row (c, jj, k): u += alpha p (if u), r -= alpha q
// over the whole row, ||r||^2 over its owned cells; double2 accesses
__global__ void __launch_bounds__(256)
k_cg_update_v(Lvl L, const double *__restrict__ num, const double *__restrict__ den,
              const double *__restrict__ p, const double *__restrict__ q,
              double *__restrict__ u, double *__restrict__ r, double *__restrict__ partials) {
    const double alpha = num[0] / den[0];
    const double malpha = -alpha;
    const int nrows = 2 * (L.ny + 2) * L.nz;
    const int lane = threadIdx.x & 31;
    const int np2 = L.pitch >> 1;
    double s = 0.0;
    for (int row = blockIdx.x * 8 + (threadIdx.x >> 5); row < nrows; row += gridDim.x * 8) {
        const int jj = (row / L.nz) % (L.ny + 2);
        const int c = row / ((L.ny + 2) * L.nz);
        const int j = jj - 1;
        const int s0 = (j + L.par + c) & 1;
        const long long base = (long long)row * L.pitch;
        const bool owned_row = (j >= 0 && j < L.ny);
        const double2 *q2 = reinterpret_cast<const double2 *>(q + base);
        double2 *r2 = reinterpret_cast<double2 *>(r + base);
#pragma unroll 4
        for (int t2 = lane; t2 < np2; t2 += 32) {
            if (u != nullptr) {
                const double2 pv = reinterpret_cast<const double2 *>(p + base)[t2];
                double2 *u2 = reinterpret_cast<double2 *>(u + base);
                const double2 uv = u2[t2];
                u2[t2] = make_double2(uv.x + alpha * pv.x, uv.y + alpha * pv.y);
            }
            const double2 qv = q2[t2], rv0 = r2[t2];
            const double2 rv = make_double2(rv0.x + malpha * qv.x, rv0.y + malpha * qv.y);
            r2[t2] = rv;
            const int h = 2 * t2 - OFF;
            if (owned_row && h >= 0 && 2 * h + s0 < L.nx) s += rv.x * rv.x;
            if (owned_row && h + 1 >= 0 && 2 * (h + 1) + s0 < L.nx) s += rv.y * rv.y;
        }
    }
    s = block_sum(s);
    if (threadIdx.x == 0) partials[blockIdx.x] = s;
}

// ---------------------------------------------------------------------------
// layout conversion: reference (nx, ny, nz) k-fastest <-> split layout.
// 32x32 (i, k) tiles through shared memory so both sides are coalesced.
// ---------------------------------------------------------------------------
// Columns ib <= i < ie only (a contiguous slab of the reference block: i is
// its slowest index), so a host transfer can be converted slab by slab.
__global__ void k_from_ref(Lvl L, const double *__restrict__ src, double *__restrict__ d, int ib,
                           int ie) {
    __shared__ double tile[32][33];
    const int i0 = ib + blockIdx.x * 32, k0 = blockIdx.y * 32, j = blockIdx.z;
    const int tx = threadIdx.x, ty = threadIdx.y;   // 32 x 8
    for (int r = ty; r < 32; r += 8) {
        const int i = i0 + r, k = k0 + tx;
        if (i < ie && k < L.nz) tile[r][tx] = src[((long long)i * L.ny + j) * L.nz + k];
    }
    __syncthreads();
    for (int r = ty; r < 32; r += 8) {
        const int i = i0 + tx, k = k0 + r;
        if (i < ie && k < L.nz) d[cell(L, i, j, k)] = tile[tx][r];
    }
}

__global__ void k_to_ref(Lvl L, const double *__restrict__ d, double *__restrict__ dst, int ib,
                         int ie) {
    __shared__ double tile[32][33];
    const int i0 = ib + blockIdx.x * 32, k0 = blockIdx.y * 32, j = blockIdx.z;
    const int tx = threadIdx.x, ty = threadIdx.y;
    for (int r = ty; r < 32; r += 8) {
        const int i = i0 + tx, k = k0 + r;
        if (i < ie && k < L.nz) tile[tx][r] = d[cell(L, i, j, k)];
    }
    __syncthreads();
    for (int r = ty; r < 32; r += 8) {
        const int i = i0 + r, k = k0 + tx;
        if (i < ie && k < L.nz) dst[((long long)i * L.ny + j) * L.nz + k] = tile[r][tx];
    }
}

// ===========================================================================
// host launchers
// ===========================================================================
static int g_sms = 0;
static int sm_count() {
    if (!g_sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, dev);
        if (g_sms <= 0) g_sms = 148;
    }
    return g_sms;
}

static inline dim3 apply_grid(const Lvl &L) {
    const int hx = ((L.nx + 1) / 2 + 31) / 32;
    return dim3(hx, (L.ny + AP_TY - 1) / AP_TY);
}

static inline int k_chunk(const Lvl &L, long long columns, int want_blocks_per_sm_x148) {
    // split k so that small levels still fill the machine
    int kc = L.nz;
    while (kc > 8 && columns * (L.nz / kc) < want_blocks_per_sm_x148) kc >>= 1;
    return kc;
}


cudaError_t launch_apply(const Lvl &L, const double *u, const double *f, double *out, int mode,
                         double *partials, int *nparts, cudaStream_t st) {
    g_launches.fetch_add(1, std::memory_order_relaxed);
    if (((mode == 1 && !out) || mode == 2) && partials && L.uniform && L.nz % 4 == 0 &&
        L.nz <= 256) {
        constexpr int KB = 4;
        const int hx = ((L.nx + 1) / 2 + 63) / 64, jy = (L.ny + AP_TY - 1) / AP_TY;
        auto go = [&](auto kern) {
            int occ = 1;
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 32 * 2 * AP_TY, 0);
            const int cap = sm_count() * (occ > 0 ? occ : 1);
            int kcs = L.nz;
            while (kcs > 2 * KB && kcs % (2 * KB) == 0 &&
                   (long long)hx * jy * (L.nz / kcs) < 2LL * cap)
                kcs >>= 1;
            const int ntiles = hx * jy * (L.nz / kcs);
            const int grid = ntiles < cap ? ntiles : cap;
            *nparts = grid;
            kern<<<grid, dim3(32, 2 * AP_TY), 0, st>>>(L, u, f, partials, hx, jy, ntiles, kcs,
                                                       out);
        };
        if (mode == 2) {
            if (L.plane == 520) go(k_norm_v<KB, 520, 2, 2>);
            else go(k_norm_v<KB, 0, 2, 2>);
        } else if (L.plane == 520) {
            go(k_norm_v<KB, 520, 2>);
        } else {
            go(k_norm_v<KB, 0, 2>);
        }
        return cudaGetLastError();
    }
    const dim3 g0 = apply_grid(L), b(32, 2 * AP_TY);
    const bool norm = partials != nullptr;
    if (L.nz <= 256) {
        // vectorised column pairs
        constexpr int KB = 4;
        const int hx = ((L.nx + 1) / 2 + 63) / 64, jy = (L.ny + AP_TY - 1) / AP_TY;
        const bool norm = partials != nullptr;
        auto go = [&](auto kern) {
            int occ = 1;
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 32 * 2 * AP_TY, 0);
            const int cap = sm_count() * (occ > 0 ? occ : 1);
            int kcs = L.nz;
            while (kcs > 2 * KB && (long long)hx * jy * ((L.nz + kcs - 1) / kcs) < 2LL * cap) kcs >>= 1;
            kcs = (kcs + KB - 1) / KB * KB;
            const int ntiles = hx * jy * ((L.nz + kcs - 1) / kcs);
            const int grid = ntiles < cap ? ntiles : cap;
            *nparts = grid;
            kern<<<grid, dim3(32, 2 * AP_TY), 0, st>>>(L, u, f, out, partials, hx, jy, ntiles, kcs);
        };
        if (L.uniform) {
            if (mode == 0) go(k_apply_v<0, false, KB, true>);
            else if (mode == 1) { if (norm) go(k_apply_v<1, true, KB, true>); else go(k_apply_v<1, false, KB, true>); }
            else go(k_apply_v<2, true, KB, true>);
        } else {
            if (mode == 0) go(k_apply_v<0, false, KB, false>);
            else if (mode == 1) { if (norm) go(k_apply_v<1, true, KB, false>); else go(k_apply_v<1, false, KB, false>); }
            else go(k_apply_v<2, true, KB, false>);
        }
        return cudaGetLastError();
    }
    const int kc = k_chunk(L, (long long)L.nx * L.ny, 148 * 2048 * 2);
    const dim3 g(g0.x, g0.y, (L.nz + kc - 1) / kc);
    *nparts = g.x * g.y * g.z;
    if ((long long)g.x * g.y * g.z > PARTIALS) return cudaErrorInvalidValue;
#define PMG_AP(U, M, N) k_apply<U, M, N><<<g, b, 0, st>>>(L, u, f, out, partials, kc)
    if (L.uniform) {
        if (mode == 0) PMG_AP(true, 0, false);
        else if (mode == 1) { if (norm) PMG_AP(true, 1, true); else PMG_AP(true, 1, false); }
        else PMG_AP(true, 2, true);
    } else {
        if (mode == 0) PMG_AP(false, 0, false);
        else if (mode == 1) { if (norm) PMG_AP(false, 1, true); else PMG_AP(false, 1, false); }
        else PMG_AP(false, 2, true);
    }
#undef PMG_AP
    return cudaGetLastError();
}

cudaError_t launch_finalize(const double *partials, int n, double *out, cudaStream_t st) {
    g_launches.fetch_add(1, std::memory_order_relaxed);
    k_finalize<<<1, 1024, 0, st>>>(partials, n, out);
    return cudaGetLastError();
}

cudaError_t launch_residual_restrict(const Lvl &F, const Lvl &C, const double *u, const double *f,
                                     double *cf, cudaStream_t st) {
    g_launches.fetch_add(1, std::memory_order_relaxed);
    if (F.uniform && F.nz <= 256 && F.nx % 4 == 0 && C.nx >= 2) {
        const int mb32 = ((C.nx >> 1) + 31) / 32;
        auto runq = [&](auto kern) {
            int occ = 1;
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 128, 0);
            const int capw = sm_count() * (occ > 0 ? occ : 1) * 4;
            int kcs = F.nz;
            while (kcs > 8 && (long long)mb32 * C.ny * ((F.nz + kcs - 1) / kcs) < 2LL * capw)
                kcs >>= 1;
            const int ntiles = mb32 * C.ny * ((F.nz + kcs - 1) / kcs);
            int grid = (ntiles + 3) / 4;
            if (grid > capw / 4) grid = capw / 4;
            kern<<<grid, 128, 0, st>>>(F, C, u, f, cf, mb32, ntiles, kcs, nullptr);
        };
        runq(k_residual_restrict_q<2>);
        return cudaGetLastError();
    }
    if (F.fcs != F.cstride) return cudaErrorInvalidValue;   // only the column-quad kernel reads fcs
    if (F.nz <= 256) {
        constexpr int KB = 4;
        const int hx = (C.nx + 63) / 64;
        int occ = 1;
        if (F.uniform)
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_residual_restrict_v<KB, true>, 128, 0);
        else
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_residual_restrict_v<KB, false>, 128, 0);
        const int cap = sm_count() * (occ > 0 ? occ : 1);
        int kcs = F.nz;
        while (kcs > 2 * KB && (long long)hx * C.ny * ((F.nz + kcs - 1) / kcs) < 2LL * cap) kcs >>= 1;
        kcs = (kcs + KB - 1) / KB * KB;
        const int ntiles = hx * C.ny * ((F.nz + kcs - 1) / kcs);
        const int grid = ntiles < cap ? ntiles : cap;
        if (F.uniform)
            k_residual_restrict_v<KB, true><<<grid, dim3(32, 4), 0, st>>>(F, C, u, f, cf, hx, ntiles, kcs);
        else
            k_residual_restrict_v<KB, false><<<grid, dim3(32, 4), 0, st>>>(F, C, u, f, cf, hx, ntiles, kcs);
        return cudaGetLastError();
    }
    const int kc = k_chunk(F, (long long)C.nx * C.ny, 148 * 2048 * 2);
    const dim3 b(32, 8), g((C.nx + 31) / 32, (F.nz + kc - 1) / kc, (C.ny + 7) / 8);
    if (F.uniform) k_residual_restrict<true><<<g, b, 0, st>>>(F, C, u, f, cf, kc);
    else k_residual_restrict<false><<<g, b, 0, st>>>(F, C, u, f, cf, kc);
    return cudaGetLastError();
}

// red-only residual + restriction (k_residual_restrict_red): fast mode,
// uniform coefficients, fine nx a multiple of 4
bool residual_restrict_red_ok(const Lvl &F) {
    return !g_smoother_exact && F.nz <= 256 && F.nx % 4 == 0;
}

cudaError_t launch_residual_restrict_red(const Lvl &F, const Lvl &C, const double *u,
                                         const double *f, double *cf, cudaStream_t st,
                                         double *partials, int *np) {
    g_launches.fetch_add(1, std::memory_order_relaxed);
    const int mb32 = ((C.nx >> 1) + 31) / 32;
    auto runq = [&](auto kern) {
        int occ = 1;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 128, 0);
        const int capw = sm_count() * (occ > 0 ? occ : 1) * 4;
        // k-chunks of at most 32 levels: more, shorter warp tasks balance the
        // persistent warps (configs[1] fine level: 331 us at 64, 314 at 32,
        // 317 at 16)
        int kcs = F.nz < 32 ? F.nz : 32;
        while (kcs > 8 && (long long)mb32 * C.ny * ((F.nz + kcs - 1) / kcs) < 2LL * capw)
            kcs >>= 1;
        const int ntiles = mb32 * C.ny * ((F.nz + kcs - 1) / kcs);
        int grid = (ntiles + 3) / 4;
        if (grid > capw / 4) grid = capw / 4;
        if (np) *np = grid;
        kern<<<grid, 128, 0, st>>>(F, C, u, f, cf, mb32, ntiles, kcs, partials);
    };
    const bool norm = partials != nullptr;
    if (F.uniform) {
        if (norm) {
            if (F.par & 1) runq(k_residual_restrict_red<1, 2, true, true>);
            else runq(k_residual_restrict_red<0, 2, true, true>);
        } else {
            if (F.par & 1) runq(k_residual_restrict_red<1>);
            else runq(k_residual_restrict_red<0>);
        }
    } else {
        // variable coefficients: 3 CTAs / SM (166 registers; the per-column
        // coefficients of four cells): 1024^2 491.7 -> 433.4 us against 2
        // CTAs / SM, 530.2 us at 4 (spills)
        if (norm) {
            if (F.par & 1) runq(k_residual_restrict_red<1, 3, false, true>);
            else runq(k_residual_restrict_red<0, 3, false, true>);
        } else {
            if (F.par & 1) runq(k_residual_restrict_red<1, 3, false>);
            else runq(k_residual_restrict_red<0, 3, false>);
        }
    }
    return cudaGetLastError();
}

constexpr size_t HS_SMEM_MAX = 200 * 1024;
size_t half_sweep_smem(const Lvl &L, bool need_old, int stage = 3) {
    size_t n = (size_t)L.nz * 32;
    return sizeof(double) * (n + ((need_old && (stage & 1)) ? n : 0) +
                             ((!L.uniform && (stage & 2)) ? n : 0) + 2 * L.nz + 1);
}
// what the exact half-sweep stages in shared memory beside the right-hand
// sides: everything when it fits (bits 0, 1), else the pivots stay in HBM,
// then the old values too (columns of up to ~790 levels)
int half_sweep_stage(const Lvl &L, bool need_old) {
    for (int stage : {3, 1, 0})
        if (half_sweep_smem(L, need_old, stage) <= HS_SMEM_MAX) return stage;
    return 0;
}



static cudaError_t launch_half_sweep_k(const Lvl &L, double *u, const double *f, int color,
                                       double rho, int zero_start, int nbr_zero,
                                       double post_scale, cudaStream_t st);

cudaError_t launch_halo_self(const Lvl &L, double *d, int px, int py, cudaStream_t st);

cudaError_t launch_half_sweep(const Lvl &L0, double *u, const double *f, int color, double rho,
                              int zero_start, int nbr_zero, double post_scale, cudaStream_t st) {
    g_launches.fetch_add(1, std::memory_order_relaxed);
    // every half-sweep kernel reads f at the relaxed colour only: a view
    // whose f colour stride differs shifts the f base instead
    f += (long long)color * (L0.fcs - L0.cstride);
    return launch_half_sweep_k(L0, u, f, color, rho, zero_start, nbr_zero, post_scale, st);
}

// fast half-sweep with the fused <f, new u> partial sums (CG's <r, z>):
// available for uniform levels whose 16-level segments tile nz;
// partials[0 .. *np) receive per-CTA sums in a fixed order.
bool half_sweep_dot_ok(const Lvl &L) {
    return !g_smoother_exact && L.uniform && L.seg == 16 && L.nz % 16 == 0 && L.nz / 16 <= 8;
}

static bool launch_half_sweep_band(const Lvl &L, double *u, const double *f, int color,
                                   double rho, int zero_start, int nbr_zero, double post_scale,
                                   cudaStream_t st, double *partials, int *np, bool fsq,
                                   double *res_uw = nullptr);

// variable-coefficient levels the TMA band kernel (k_half_sweep_bandv) runs:
// nz = 128, a planned plane pitch, whole 32-column strips of at least two
// per colour row, eight rows or more.  Its units walk tile regions (rows in
// consecutive runs), so these levels also relax boundary-first.
bool half_sweep_bandv_ok(const Lvl &L) {
    const int hrow = L.nx / 2;
    return !g_smoother_exact && !L.uniform && L.nz == BAND_NZ &&
           (L.plane == 2056 || L.plane == 1032 || L.plane == 520 || L.plane == 264 ||
            L.plane == 136) &&
           L.nx % 2 == 0 && hrow % 32 == 0 && hrow >= 64 && L.ny >= 8;
}
static bool launch_half_sweep_bandv(const Lvl &L, double *u, const double *f, int color,
                                    double rho, int zero_start, int nbr_zero, double post_scale,
                                    cudaStream_t st, int mode, double *partials, int *np,
                                    double *res_uw);

cudaError_t launch_half_sweep_dot(const Lvl &L, double *u, const double *f, int color, double rho,
                                  int zero_start, int nbr_zero, double post_scale,
                                  double *partials, int *np, cudaStream_t st) {
    g_launches.fetch_add(1, std::memory_order_relaxed);
    if (launch_half_sweep_band(L, u, f, color, rho, zero_start, nbr_zero, post_scale, st,
                               partials, np, false))
        return cudaGetLastError();
    const int hx = ((L.nx + 1) / 2 + 31) / 32;
    const int nw = L.nz / 16;
    const size_t sm = sizeof(double) * (7 * (size_t)L.nz + 4 * 16 * 32);
    const int ntiles = hx * L.ny;
    auto run = [&](auto kern) {
        int occ = 1;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 32 * nw, sm);
        const int cap = sm_count() * (occ > 0 ? occ : 1);
        const int grid = ntiles < cap ? ntiles : cap;
        *np = grid;
        kern<<<grid, 32 * nw, sm, st>>>(L, u, f, color, rho, zero_start, nbr_zero, post_scale,
                                        ntiles, hx, partials, nullptr);
    };
    if (nbr_zero) {
        if (L.plane == 520) run(k_half_sweep_seg<16, 4, 2, 1, true, 520, true>);
        else run(k_half_sweep_seg<16, 4, 2, 1, true, 0, true>);
    } else {
        if (L.plane == 520) run(k_half_sweep_seg<16, 4, 2, 0, true, 520, true>);
        else run(k_half_sweep_seg<16, 4, 2, 0, true, 0, true>);
    }
    return cudaGetLastError();
}

// variable-coefficient levels the fast smoother handles with
// k_half_sweep_segv (16 warps, SEG = nz / 16)
static int segv_seg(const Lvl &L) {
    if (g_smoother_exact || L.uniform || L.nz > 256 || L.nz % 16)
        return 0;
    const int seg = L.nz / 16;
    return (seg == 1 || seg == 2 || seg == 4 || seg == 8 || seg == 16) ? seg : 0;
}

// k_half_sweep_segv in mode RES (1: fused residual into uw, 3: f^2) with
// per-CTA partial sums; grid as launch_half_sweep_k's variable branch
template <int RES>
static void launch_segv_mode(const Lvl &L, double *u, double *uw, const double *f, int color,
                             int nbr_zero, double *partials, int *np, cudaStream_t st) {
    const int hx = ((L.nx + 1) / 2 + 31) / 32;
    const int seg = segv_seg(L);
    const int nw = L.nz / seg;
    const size_t sm =
        sizeof(double) * (L.nz + ((L.nz + 2) & ~1) + 4 * 16 * 32 + (RES == 1 ? 2 * L.nz : 0));
    const int ntiles = hx * L.ny;
    auto runv = [&](auto kern) {
        int occ = 1;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 32 * nw, sm);
        const int cap = sm_count() * (occ > 0 ? occ : 1);
        const int grid = ntiles < cap ? ntiles : cap;
        *np = grid;
        kern<<<grid, 32 * nw, sm, st>>>(L, u, f, color, 1.0, 0, 0, 1.0, ntiles, hx, partials,
                                        uw);
    };
#define PMG_SEGVM(S)                                                               \
    do {                                                                           \
        if (RES != 1 && nbr_zero) runv(k_half_sweep_segv<S, 1, RES, true>);        \
        else runv(k_half_sweep_segv<S, 0, RES, true>);                             \
    } while (0)
    switch (seg) {
    case 1: PMG_SEGVM(1); break;
    case 2: PMG_SEGVM(2); break;
    case 4: PMG_SEGVM(4); break;
    case 8: PMG_SEGVM(8); break;
    default: PMG_SEGVM(16); break;
    }
#undef PMG_SEGVM
}

// red half-sweep (rho = 1) with the lagged convergence residual: reads the
// iterate u, writes the relaxed red values into uw's red array and the
// per-CTA sums of (f - A u)^2 over u's red cells into partials[0 .. *np).
// Fast mode, no fused halo: uniform levels whose 16-level segments tile nz
// (k_half_sweep_seg) or variable levels of k_half_sweep_segv.
bool half_sweep_res_ok(const Lvl &L) {
    return half_sweep_dot_ok(L) || segv_seg(L);
}

cudaError_t launch_half_sweep_res(const Lvl &L, const double *u, double *uw, const double *f,
                                  double *partials, int *np, cudaStream_t st) {
    g_launches.fetch_add(1, std::memory_order_relaxed);
    if (!L.uniform) {
        if (!launch_half_sweep_bandv(L, const_cast<double *>(u), f, 0, 1.0, 0, 0, 1.0, st, 1,
                                     partials, np, uw))
            launch_segv_mode<1>(L, const_cast<double *>(u), uw, f, 0, 0, partials, np, st);
        return cudaGetLastError();
    }
    // the TMA band kernel (16 compute warps) where the level's half-sweeps
    // run on it: same column solves as those sweeps
    if (launch_half_sweep_band(L, const_cast<double *>(u), f, 0, 1.0, 0, 0, 1.0, st, partials, np,
                               false, uw))
        return cudaGetLastError();
    const int hx = ((L.nx + 1) / 2 + 31) / 32;
    const int nw = L.nz / 16;
    const size_t sm = sizeof(double) * (11 * (size_t)L.nz + 4 * 16 * 32);
    const int ntiles = hx * L.ny;
    auto run = [&](auto kern) {
        int occ = 1;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 32 * nw, sm);
        const int cap = sm_count() * (occ > 0 ? occ : 1);
        const int grid = ntiles < cap ? ntiles : cap;
        *np = grid;
        kern<<<grid, 32 * nw, sm, st>>>(L, const_cast<double *>(u), f, 0, 1.0, 0, 0, 1.0, ntiles,
                                        hx, partials, uw);
    };
    // register loads at 2 CTAs / SM (128 registers, no spills): 413 us at
    // configs[1]'s fine level; at 3 CTAs / SM (80 registers, spills) 517 us,
    // with the incoming values staged in shared memory by cp.async 413 /
    // 538 us at 2 / 3 CTAs
    if (L.plane == 520) run(k_half_sweep_seg<16, 4, 2, 0, true, 520, false, 1>);
    else if (L.plane == 264) run(k_half_sweep_seg<16, 4, 2, 0, true, 264, false, 1>);
    else run(k_half_sweep_seg<16, 4, 2, 0, true, 0, false, 1>);
    return cudaGetLastError();
}

// half-sweep that also sums f^2 over the relaxed colour (mg_solve's ||f||
// folded into the first cycle's two half-sweeps); half_sweep_res_ok levels
cudaError_t launch_half_sweep_fsq(const Lvl &L, double *u, const double *f, int color,
                                  int nbr_zero, double *partials, int *np, cudaStream_t st) {
    g_launches.fetch_add(1, std::memory_order_relaxed);
    f += (long long)color * (L.fcs - L.cstride);   // see launch_half_sweep
    if (!L.uniform) {
        if (!launch_half_sweep_bandv(L, u, f, color, 1.0, 0, nbr_zero, 1.0, st, 3, partials, np,
                                     nullptr))
            launch_segv_mode<3>(L, u, nullptr, f, color, nbr_zero, partials, np, st);
        return cudaGetLastError();
    }
    if (launch_half_sweep_band(L, u, f, color, 1.0, 0, nbr_zero, 1.0, st, partials, np, true))
        return cudaGetLastError();
    const int hx = ((L.nx + 1) / 2 + 31) / 32;
    const int nw = L.nz / 16;
    const size_t sm = sizeof(double) * (11 * (size_t)L.nz + 4 * 16 * 32);
    const int ntiles = hx * L.ny;
    auto run = [&](auto kern) {
        int occ = 1;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 32 * nw, sm);
        const int cap = sm_count() * (occ > 0 ? occ : 1);
        const int grid = ntiles < cap ? ntiles : cap;
        *np = grid;
        kern<<<grid, 32 * nw, sm, st>>>(L, u, f, color, 1.0, 0, nbr_zero, 1.0, ntiles, hx,
                                        partials, nullptr);
    };
#define PMG_FSQ(P)                                                                   \
    do {                                                                             \
        if (nbr_zero) run(k_half_sweep_seg<16, 4, 3, 1, true, P, false, 3>); \
        else run(k_half_sweep_seg<16, 4, 3, 0, true, P, false, 3>);         \
    } while (0)
    if (L.plane == 520) PMG_FSQ(520);
    else if (L.plane == 264) PMG_FSQ(264);
    else PMG_FSQ(0);
#undef PMG_FSQ
    return cudaGetLastError();
}


template <int P, int NW>
static void band_attrs_nw() {
    const int sm = (int)band_smem();
    cudaFuncSetAttribute(k_half_sweep_band<P, false, false, false, NW>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    cudaFuncSetAttribute(k_half_sweep_band<P, false, false, true, NW>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    cudaFuncSetAttribute(k_half_sweep_band<P, true, false, false, NW>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    cudaFuncSetAttribute(k_half_sweep_band<P, false, true, false, NW>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
}
template <int P>
static void bandv_attrs() {
    const int sm = (int)bandv_smem();
    cudaFuncSetAttribute(k_half_sweep_bandv<P, 0, false>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    cudaFuncSetAttribute(k_half_sweep_bandv<P, 0, true>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    cudaFuncSetAttribute(k_half_sweep_bandv<P, 1, true>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    cudaFuncSetAttribute(k_half_sweep_bandv<P, 3, true>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    cudaFuncSetAttribute(k_half_sweep_bandv<P, 0, true, true>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    cudaFuncSetAttribute(k_half_sweep_bandv<P, 3, true, true>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
}
template <int P>
static void band_attrs() {
    bandv_attrs<P>();
    band_attrs_nw<P, 8>();
    band_attrs_nw<P, 16>();
    cudaFuncSetAttribute(k_half_sweep_band<P, false, false, true, 16, true>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)band_smem());
}

// one-time kernel attributes (outside any stream capture: called from
// pmg_level_create)
void setup_kernel_attributes() {
    static bool done = false;
    if (done) return;
    done = true;
    // the exact half-sweep's opt-in shared memory (tall columns); set here so
    // that its first launch may sit inside a stream capture
    cudaFuncSetAttribute(k_half_sweep<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)HS_SMEM_MAX);
    cudaFuncSetAttribute(k_half_sweep<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)HS_SMEM_MAX);
    bandv_attrs<2056>();
    band_attrs<1032>();
    band_attrs<520>();
    band_attrs<264>();
    band_attrs<136>();
    cudaGetLastError();
}


// tensor maps of the band kernel: 3-D views (pitch, nz, ny + 2) of one
// colour array with a box of boxw columns x kc levels x 1 row
static PFN_cuTensorMapEncodeTiled_v12000 tmap_encoder() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static bool tried = false;
    if (!tried) {
        tried = true;
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
                cudaSuccess && q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }
    return fn;
}

static bool make_tmap(CUtensorMap *m, const double *base, const Lvl &L, int boxw, int kc) {
    auto enc = tmap_encoder();
    if (!enc) return false;
    const cuuint64_t dims[3] = {(cuuint64_t)L.plane, (cuuint64_t)L.nz, (cuuint64_t)L.ny + 2};
    const cuuint64_t strides[2] = {(cuuint64_t)L.plane * 8, (cuuint64_t)L.jstride * 8};
    const cuuint32_t box[3] = {(cuuint32_t)boxw, (cuuint32_t)kc, 1};
    const cuuint32_t es[3] = {1, 1, 1};
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double *>(base), dims, strides,
               box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}


// k_half_sweep_band: configs[1]'s fine level shape (nz = 128, plane 520),
// neighbours read, no fused halo
// k_half_sweep_bandv: the same rings, tables tdrw tvp(+2) tvol tdr, the four
// [16][32] segment arrays, barriers and warp sums
static size_t bandv_smem() {
    return sizeof(double) * (4 * BAND_NZ * BAND_W + 2 * BAND_NZ * 32 + 4 * BAND_NZ * 2 +
                             4 * BAND_NZ + 2 + 4 * 16 * 32 + 16) + 12 * 8 + 128;
}

static size_t band_smem() {   // sized for up to 16 compute warps
    // rings (4 other-colour rows, 2 f rows, 4 edge pairs), tables ti tb tw
    // tr1 tr2 (double2) and tq, hend / ybeg, barriers, warp sums
    return sizeof(double) * (4 * BAND_NZ * BAND_W + 2 * BAND_NZ * 32 + 4 * BAND_NZ * 2 +
                             11 * BAND_NZ + 2 * 16 * 32 + 16) + 12 * 8 + 128;
}


// compute warps of k_half_sweep_band: 16 (8 levels each) on rows of >= 512
// cells per colour -- 2048^2: 1214 -> 1008 us, 1024^2: 284 -> 260 us per
// half-sweep -- and 8 (16 levels each) below, where 16 warps measured slower
// (512^2: 71.4 -> 75.5 us, 256^2: 20.9 -> 23.5 us)
static int band_nw(const Lvl &L) { return (L.nx / 2 >= 512) ? 16 : 8; }


static bool launch_half_sweep_band(const Lvl &L, double *u, const double *f, int color,
                                   double rho, int zero_start, int nbr_zero, double post_scale,
                                   cudaStream_t st, double *partials, int *np,
                                   bool fsq, double *res_uw) {
    const int hrow = L.nx / 2;
    if (g_smoother_exact || !L.uniform || L.nz != BAND_NZ ||
        !(L.plane == 1032 || L.plane == 520 || L.plane == 264 || L.plane == 136) ||
        L.seg != 16 || nbr_zero || L.nx % 2 || hrow % 32 || hrow < 64 ||
        L.ny < 8 || L.rys != 1 || L.rxn < 1 || L.ryn < 1)
        return false;
    // the fused-residual mode fits the registers of the 16-warp kernel only
    // (the 8-warp levels keep k_half_sweep_seg's, bit-identical to theirs)
    if (res_uw && band_nw(L) != 16) return false;
    const int o = color ^ 1;
    CUtensorMap mF, mB, mE;
    if (!make_tmap(&mF, f + (long long)color * L.cstride, L, 32, BAND_NZ) ||
        !make_tmap(&mB, u + (long long)o * L.cstride, L, BAND_W, BAND_NZ) ||
        !make_tmap(&mE, u + (long long)o * L.cstride, L, 2, BAND_NZ))
        return false;
    // the tile region: L.rxn strips (stride L.rxs) x L.ryn consecutive rows
    const int nstrip = L.rxn, nrows = L.ryn;
    // units per SM: a multiple of the SM count keeps the CTAs balanced;
    // measured best 4 at 16 strips (nx = 1024: 269 us; 2 -> 373, 8 -> 278),
    // 2 at 8 strips (nx = 512: 76.3 us; 4 -> 80.3), 1 below
    // (the smallest count that makes strips x bands a multiple of the SMs:
    // nstrip / gcd(nstrip, SMs) -- 8 at 32 strips on 148 SMs)
    int gcd = nstrip, bsm = sm_count();
    while (bsm) {
        const int t = gcd % bsm;
        gcd = bsm;
        bsm = t;
    }
    const int ups = nstrip / gcd;
    int nband = (ups * sm_count() + nstrip - 1) / nstrip;
    if (nband > nrows) nband = nrows;
    const int band_rows = (nrows + nband - 1) / nband;
    nband = (nrows + band_rows - 1) / band_rows;
    const int nunits = nstrip * nband;
    const int grid = nunits < sm_count() ? nunits : sm_count();
    if (np) *np = grid;
    const bool lean = rho == 1.0 && !zero_start;
#define PMG_BANDK(P, NW)                                                                    \
    do {                                                                                    \
        const int nt = 32 * (NW + 1);                                                       \
        if (res_uw)                                                                         \
            k_half_sweep_band<P, false, false, true, 16, true><<<grid, nt, band_smem(), st>>>( \
                L, u, color, rho, zero_start, post_scale, nstrip, nband, band_rows, mF, mB, \
                mE, partials, res_uw);                                                  \
        else if (lean && !partials)                                                              \
            k_half_sweep_band<P, false, false, true, NW><<<grid, nt, band_smem(), st>>>(    \
                L, u, color, rho, zero_start, post_scale, nstrip, nband, band_rows, mF, mB, \
                mE, nullptr, nullptr);                                                           \
        else if (partials && fsq)                                                           \
            k_half_sweep_band<P, false, true, false, NW><<<grid, nt, band_smem(), st>>>(    \
                L, u, color, rho, zero_start, post_scale, nstrip, nband, band_rows, mF, mB, \
                mE, partials, nullptr);                                                          \
        else if (partials)                                                                  \
            k_half_sweep_band<P, true, false, false, NW><<<grid, nt, band_smem(), st>>>(    \
                L, u, color, rho, zero_start, post_scale, nstrip, nband, band_rows, mF, mB, \
                mE, partials, nullptr);                                                          \
        else                                                                                \
            k_half_sweep_band<P, false, false, false, NW><<<grid, nt, band_smem(), st>>>(   \
                L, u, color, rho, zero_start, post_scale, nstrip, nband, band_rows, mF, mB, \
                mE, nullptr, nullptr);                                                           \
    } while (0)
#define PMG_BANDL(P)                                                                        \
    do {                                                                                    \
        if (band_nw(L) == 16) PMG_BANDK(P, 16);                                             \
        else PMG_BANDK(P, 8);                                                               \
    } while (0)
    if (L.plane == 520) PMG_BANDL(520);
    else if (L.plane == 264) PMG_BANDL(264);
    else if (L.plane == 1032) PMG_BANDL(1032);
    else PMG_BANDL(136);
#undef PMG_BANDL
#undef PMG_BANDK
    return true;
}

// k_half_sweep_bandv (variable coefficients, nz = 128): mode 0 plain, 1 the
// fused residual into uw, 3 with the f^2 partial sums; false if the level
// does not fit it (then k_half_sweep_segv runs)
static bool launch_half_sweep_bandv(const Lvl &L, double *u, const double *f, int color,
                                    double rho, int zero_start, int nbr_zero, double post_scale,
                                    cudaStream_t st, int mode, double *partials, int *np,
                                    double *res_uw) {
    if (!L.invd || !half_sweep_bandv_ok(L) ||
        (nbr_zero && !(rho == 1.0 && !zero_start && mode != 1)) || L.rys != 1 || L.rxn < 1 ||
        L.ryn < 1)
        return false;
    const int o = color ^ 1;
    CUtensorMap mF, mB, mE;
    if (!make_tmap(&mF, f + (long long)color * L.cstride, L, 32, BAND_NZ) ||
        !make_tmap(&mB, u + (long long)o * L.cstride, L, BAND_W, BAND_NZ) ||
        !make_tmap(&mE, u + (long long)o * L.cstride, L, 2, BAND_NZ))
        return false;
    const int nstrip = L.rxn, nrows = L.ryn;
    int gcd = nstrip, bsm = sm_count();
    while (bsm) {
        const int t = gcd % bsm;
        gcd = bsm;
        bsm = t;
    }
    const int ups = nstrip / gcd;
    int nband = (ups * sm_count() + nstrip - 1) / nstrip;
    if (nband > nrows) nband = nrows;
    const int band_rows = (nrows + nband - 1) / nband;
    nband = (nrows + band_rows - 1) / band_rows;
    const int nunits = nstrip * nband;
    const int grid = nunits < sm_count() ? nunits : sm_count();
    if (np) *np = grid;
    const bool lean = rho == 1.0 && !zero_start;
#define PMG_BANDV(P)                                                                         \
    do {                                                                                     \
        if (nbr_zero && mode == 3)                                                           \
            k_half_sweep_bandv<P, 3, true, true><<<grid, 512, bandv_smem(), st>>>(           \
                L, u, color, rho, zero_start, post_scale, nstrip, nband, band_rows, mF, mB,  \
                mE, partials, nullptr);                                                      \
        else if (nbr_zero)                                                                   \
            k_half_sweep_bandv<P, 0, true, true><<<grid, 512, bandv_smem(), st>>>(           \
                L, u, color, rho, zero_start, post_scale, nstrip, nband, band_rows, mF, mB,  \
                mE, nullptr, nullptr);                                                       \
        else if (mode == 1)                                                                       \
            k_half_sweep_bandv<P, 1, true><<<grid, 512, bandv_smem(), st>>>(                  \
                L, u, color, rho, zero_start, post_scale, nstrip, nband, band_rows, mF, mB,  \
                mE, partials, res_uw);                                                       \
        else if (mode == 3)                                                                  \
            k_half_sweep_bandv<P, 3, true><<<grid, 512, bandv_smem(), st>>>(                  \
                L, u, color, rho, zero_start, post_scale, nstrip, nband, band_rows, mF, mB,  \
                mE, partials, nullptr);                                                      \
        else if (lean)                                                                       \
            k_half_sweep_bandv<P, 0, true><<<grid, 512, bandv_smem(), st>>>(                  \
                L, u, color, rho, zero_start, post_scale, nstrip, nband, band_rows, mF, mB,  \
                mE, nullptr, nullptr);                                                       \
        else                                                                                 \
            k_half_sweep_bandv<P, 0, false><<<grid, 512, bandv_smem(), st>>>(                 \
                L, u, color, rho, zero_start, post_scale, nstrip, nband, band_rows, mF, mB,  \
                mE, nullptr, nullptr);                                                       \
    } while (0)
    if (L.plane == 2056) PMG_BANDV(2056);   // configs[4]'s 4096^2 fine level
    else if (L.plane == 1032) PMG_BANDV(1032);
    else if (L.plane == 520) PMG_BANDV(520);
    else if (L.plane == 264) PMG_BANDV(264);
    else PMG_BANDV(136);
#undef PMG_BANDV
    return true;
}

static cudaError_t launch_half_sweep_k(const Lvl &L, double *u, const double *f, int color,
                                       double rho, int zero_start, int nbr_zero,
                                       double post_scale, cudaStream_t st) {
    if (launch_half_sweep_band(L, u, f, color, rho, zero_start, nbr_zero, post_scale, st, nullptr,
                               nullptr, false)) {
        return cudaGetLastError();
    }
    const int hx = ((L.nx + 1) / 2 + 31) / 32;
    const dim3 g(hx, L.ny);
    if (launch_half_sweep_bandv(L, u, f, color, rho, zero_start, nbr_zero, post_scale, st, 0,
                                nullptr, nullptr, nullptr))
        return cudaGetLastError();
    if (!g_smoother_exact && !L.uniform && L.nz <= 256) {
        // variable coefficients: 16 warps, SEG = nz / 16 (must divide)
        int seg = 0;
        if (L.nz % 16 == 0 && L.nz / 16 <= 16) seg = L.nz / 16;
        if (seg == 1 || seg == 2 || seg == 4 || seg == 8 || seg == 16) {
            const int nw = L.nz / seg;
            const size_t sm = sizeof(double) * (L.nz + ((L.nz + 2) & ~1) + 4 * 16 * 32);
            const int ntiles = hx * L.ny;
            auto runv = [&](auto kern) {
                int occ = 1;
                cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 32 * nw, sm);
                const int cap = sm_count() * (occ > 0 ? occ : 1);
                const int grid = ntiles < cap ? ntiles : cap;
                kern<<<grid, 32 * nw, sm, st>>>(L, u, f, color, rho, zero_start, 0, post_scale,
                                                ntiles, hx, nullptr, nullptr);
            };
#define PMG_SEGV(S)                                                                   \
    do {                                                                              \
        const bool lean_ = rho == 1.0 && !zero_start;                                 \
        if (lean_ && nbr_zero) runv(k_half_sweep_segv<S, 1, 0, true>);                \
        else if (lean_) runv(k_half_sweep_segv<S, 0, 0, true>);                       \
        else if (nbr_zero) runv(k_half_sweep_segv<S, 1>);                             \
        else runv(k_half_sweep_segv<S, 0>);                                           \
    } while (0)
            switch (seg) {
            case 1: PMG_SEGV(1); break;
            case 2: PMG_SEGV(2); break;
            case 4: PMG_SEGV(4); break;
            case 8: PMG_SEGV(8); break;
            default: PMG_SEGV(16); break;
            }
#undef PMG_SEGV
            return cudaGetLastError();
        }
    }
    if (!g_smoother_exact && L.uniform && L.seg && (L.nz + L.seg - 1) / L.seg <= 8) {
        const int nw = (L.nz + L.seg - 1) / L.seg;
        const size_t sm = sizeof(double) * (7 * (size_t)L.nz + 4 * 16 * 32);
        // the level's tile region (the whole part unless a boundary-first
        // sweep restricts it): L.rxn strips x L.ryn rows
        const int ntiles = L.rxn * L.ryn;
        if (ntiles <= 0) return cudaSuccess;
        auto run = [&](auto kern) {
            int occ = 1;
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 32 * nw, sm);
            const int cap = sm_count() * (occ > 0 ? occ : 1);
            const int grid = ntiles < cap ? ntiles : cap;
            kern<<<grid, 32 * nw, sm, st>>>(L, u, f, color, rho, zero_start, nbr_zero, post_scale,
                                            ntiles, L.rxn, nullptr, nullptr);
        };
        {
            // compile-time neighbour mode, predicate-free when the segments
            // tile nz exactly (all BASELINE configs)
            const bool full = (L.nz % L.seg) == 0;
            const bool lean = rho == 1.0 && !zero_start;   // compile-time store path
            // compile-time plane stride for the large levels of nz = 128
            // (pitch of nx = 1024, 512, 256)
            const int plc = (L.seg == 16 && full) ? (int)L.plane : 0;
#define PMG_SEGP(S, P)                                                                \
    do {                                                                              \
        if (lean && nbr_zero) run(k_half_sweep_seg<S, 4, 3, 1, true, P, false, 0, true>); \
        else if (lean) run(k_half_sweep_seg<S, 4, 3, 0, true, P, false, 0, true>); \
        else if (nbr_zero) run(k_half_sweep_seg<S, 4, 3, 1, true, P>);        \
        else run(k_half_sweep_seg<S, 4, 3, 0, true, P>);                      \
    } while (0)
#define PMG_SEGF(S)                                                                   \
    do {                                                                              \
        if (full) {                                                                   \
            if (nbr_zero) run(k_half_sweep_seg<S, 4, 3, 1, true>);                    \
            else run(k_half_sweep_seg<S, 4, 3, 0, true>);                             \
        } else {                                                                      \
            run(k_half_sweep_seg<S, 4, 2>);                                           \
        }                                                                             \
    } while (0)
            // levels of <= 64 tiles (nx <= 64 at nz = 128): 5.5 -> 4.5 us per
            // sweep; 256 tiles (nx = 128) is slower this way (6.6 -> 7.9)
            if (L.seg == 16 && full && ntiles <= 64) {
                // launch-latency-bound small level: all 16 levels' loads of a
                // tile in one batch (one memory round trip per tile)
                if (lean && nbr_zero) run(k_half_sweep_seg<16, 16, 1, 1, true, 0, false, 0, true>);
                else if (lean) run(k_half_sweep_seg<16, 16, 1, 0, true, 0, false, 0, true>);
                else if (nbr_zero) run(k_half_sweep_seg<16, 16, 1, 1, true, 0>);
                else run(k_half_sweep_seg<16, 16, 1, 0, true, 0>);
            } else if (plc == 520) PMG_SEGP(16, 520);
            else if (plc == 264) PMG_SEGP(16, 264);
            else if (plc == 136) PMG_SEGP(16, 136);
            else switch (L.seg) {
            case 4: PMG_SEGF(4); break;
            case 8: PMG_SEGF(8); break;
            case 16: PMG_SEGF(16); break;
            default: run(k_half_sweep_seg<32, 4, 1>); break;
            }
#undef PMG_SEGF
#undef PMG_SEGP
            return cudaGetLastError();
        }
    }
    const bool need_old = !zero_start && rho != 1.0;
    const int stage = half_sweep_stage(L, need_old);
    const size_t sm = half_sweep_smem(L, need_old, stage);
    const dim3 b(HS_THREADS);
    static bool attr_set[2] = {false, false};
    if (L.uniform) {
        if (!attr_set[0]) {
            cudaFuncSetAttribute(k_half_sweep<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)HS_SMEM_MAX);
            cudaFuncSetAttribute(k_half_sweep<true>,
                                 cudaFuncAttributePreferredSharedMemoryCarveout, 100);
            attr_set[0] = true;
        }
        k_half_sweep<true><<<g, b, sm, st>>>(L, u, f, color, rho, zero_start, nbr_zero, post_scale,
                                             stage);
    } else {
        if (!attr_set[1]) {
            cudaFuncSetAttribute(k_half_sweep<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)HS_SMEM_MAX);
            cudaFuncSetAttribute(k_half_sweep<false>,
                                 cudaFuncAttributePreferredSharedMemoryCarveout, 100);
            attr_set[1] = true;
        }
        k_half_sweep<false><<<g, b, sm, st>>>(L, u, f, color, rho, zero_start, nbr_zero,
                                              post_scale, stage);
    }
    return cudaGetLastError();
}

cudaError_t launch_invd(const Lvl &L, double *invd, cudaStream_t st) {
    g_launches.fetch_add(1, std::memory_order_relaxed);
    k_invd<<<dim3((L.nx + 127) / 128, L.ny), 128, 0, st>>>(L, invd);
    return cudaGetLastError();
}

cudaError_t launch_restrict(const Lvl &F, const Lvl &C, const double *fu, double *cu, double w,
                            cudaStream_t st) {
    g_launches.fetch_add(1, std::memory_order_relaxed);
    k_restrict<<<dim3((C.nx + 127) / 128, C.nz, C.ny), 128, 0, st>>>(F, C, fu, cu, w);
    return cudaGetLastError();
}

cudaError_t launch_prolong(const Lvl &F, const Lvl &C, const double *cu, double *fu, int add,
                           int cmask, cudaStream_t st) {
    g_launches.fetch_add(1, std::memory_order_relaxed);
    if (F.nx % 4 == 0 && C.nx >= 2) {
        const int npair = C.nx >> 1;
        // two coarse rows per thread (measured on B200 at configs[1]'s fine
        // level, black only: 1 row -> 310 us, 2 -> 252, 4 -> 274, 8 -> 341)
        const int gx = (npair + 127) / 128;
        if (cmask == 2)
            k_prolong_w<2, 2><<<dim3(gx, F.nz, (C.ny + 1) / 2), 128, 0, st>>>(F, C, cu, fu, add, cmask);
        else
            k_prolong_w<2><<<dim3(gx, F.nz, (C.ny + 1) / 2), 128, 0, st>>>(F, C, cu, fu, add, cmask);
        return cudaGetLastError();
    }
    const int n2 = (cmask == 3 ? 2 : 1) * ((F.nx + 1) / 2);
    k_prolong<<<dim3((n2 + 127) / 128, F.nz, F.ny), 128, 0, st>>>(F, C, cu, fu, add, cmask);
    return cudaGetLastError();
}

cudaError_t launch_halo_self(const Lvl &L, double *d, int px, int py, cudaStream_t st) {
    g_launches.fetch_add(1, std::memory_order_relaxed);
    const long long n = 2LL * (L.nx + 2) * L.nz + 2LL * L.ny * L.nz;
    k_halo_self<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(L, d, px, py);
    return cudaGetLastError();
}

int face_len(const Lvl &L, int face) { return face < 2 ? L.ny : L.nx + 2; }

cudaError_t launch_pack(const Lvl &L, const double *d, int face, double *buf, cudaStream_t st) {
    g_launches.fetch_add(1, std::memory_order_relaxed);
    const int len = face_len(L, face);
    k_pack_face<<<dim3((len + 127) / 128, L.nz), 128, 0, st>>>(L, d, face, buf, len);
    return cudaGetLastError();
}

cudaError_t launch_unpack(const Lvl &L, double *d, int face, const double *buf, int mirror,
                          cudaStream_t st) {
    g_launches.fetch_add(1, std::memory_order_relaxed);
    const int len = face_len(L, face);
    k_unpack_face<<<dim3((len + 127) / 128, L.nz), 128, 0, st>>>(L, d, face, buf, len, mirror);
    return cudaGetLastError();
}

static inline int stream_blocks(long long n) {
    long long b = (n + 255) / 256;
    long long cap = 4LL * sm_count();
    return (int)(b < cap ? (b > 0 ? b : 1) : cap);
}

cudaError_t launch_dot(const Lvl &L, const double *a, const double *b, double *partials, int *np,
                       cudaStream_t st) {
    g_launches.fetch_add(1, std::memory_order_relaxed);
    constexpr int RPB = 4;
    const int nh = (L.nx + 1) / 2;
    int bs = (nh / 2 + 31) / 32 * 32;
    bs = bs < 32 ? 32 : (bs > 256 ? 256 : bs);
    const int nch = (nh + 2 * bs - 1) / (2 * bs);
    const int nitems = 2 * L.nz * L.ny * nch;
    int g = (nitems + RPB - 1) / RPB;
    const int cap = 8 * sm_count();
    if (g > cap) g = cap;
    *np = g;
    if (a == b)
        k_dot2<RPB, true><<<g, bs, 0, st>>>(L, a, b, partials, nch);
    else
        k_dot2<RPB, false><<<g, bs, 0, st>>>(L, a, b, partials, nch);
    return cudaGetLastError();
}

cudaError_t launch_copy_block(const Lvl &S, const double *src, const Lvl &D, double *dst, int si,
                              int sj, int di, int dj, int w, int h, cudaStream_t st) {
    g_launches.fetch_add(1, std::memory_order_relaxed);
    const long long n = (long long)w * h * S.nz;
    if (n <= 0) return cudaSuccess;
    k_copy_block<<<stream_blocks(n), 256, 0, st>>>(S, src, D, dst, si, sj, di, dj, w, h);
    return cudaGetLastError();
}

cudaError_t launch_fill(long long n, double v, double *y, cudaStream_t st) {
    g_launches.fetch_add(1, std::memory_order_relaxed);
    k_fill<<<stream_blocks(n), 256, 0, st>>>(n, v, y);
    return cudaGetLastError();
}

cudaError_t launch_axpy(long long n, double a, const double *x, double *y, cudaStream_t st) {
    g_launches.fetch_add(1, std::memory_order_relaxed);
    k_axpy<<<stream_blocks(n), 256, 0, st>>>(n, a, x, y);
    return cudaGetLastError();
}

cudaError_t launch_xpby(long long n, const double *x, double b, double *y, cudaStream_t st) {
    g_launches.fetch_add(1, std::memory_order_relaxed);
    k_xpby<<<stream_blocks(n), 256, 0, st>>>(n, x, b, y);
    return cudaGetLastError();
}

cudaError_t launch_cg_direction(long long n, const double *num, const double *den, const double *z,
                                double *p, cudaStream_t st) {
    g_launches.fetch_add(1, std::memory_order_relaxed);
    k_cg_direction<<<stream_blocks(n), 256, 0, st>>>(n, num, den, z, p);
    return cudaGetLastError();
}

cudaError_t launch_cg_up(long long n, const double *an, const double *ad, const double *bn,
                         const double *bd, const double *z, double *p, double *u, cudaStream_t st) {
    g_launches.fetch_add(1, std::memory_order_relaxed);
    if (n % 2 == 0) {
        // whole allocations: even length, 16-byte aligned
        const long long n2 = n / 2;
        long long b = (n2 + 255) / 256;
        if (b > 8LL * sm_count()) b = 8LL * sm_count();
        k_cg_up_v<<<(int)b, 256, 0, st>>>(n2, an, ad, bn, bd,
                                          reinterpret_cast<const double2 *>(z),
                                          reinterpret_cast<double2 *>(p),
                                          reinterpret_cast<double2 *>(u));
        return cudaGetLastError();
    }
    k_cg_up<<<stream_blocks(n), 256, 0, st>>>(n, an, ad, bn, bd, z, p, u);
    return cudaGetLastError();
}

cudaError_t launch_cg_update(const Lvl &L, const double *num, const double *den,
                             const double *p, const double *q, double *u, double *r,
                             double *partials, int *np, cudaStream_t st) {
    g_launches.fetch_add(1, std::memory_order_relaxed);
    const long long n = 2LL * L.cstride;
    if (L.pitch % 2 == 0) {
        const int rows = 2 * L.nz * (L.ny + 2);
        int g = 8 * sm_count();
        if (g > (rows + 7) / 8) g = (rows + 7) / 8;
        *np = g;
        k_cg_update_v<<<g, 256, 0, st>>>(L, num, den, p, q, u, r, partials);
        return cudaGetLastError();
    }
    int g = stream_blocks(n);
    if (g > 2 * L.nz * (L.ny + 2)) g = 2 * L.nz * (L.ny + 2);
    *np = g;
    k_cg_update<<<g, 256, 0, st>>>(L, num, den, p, q, u, r, partials);
    return cudaGetLastError();
}

cudaError_t launch_from_ref(const Lvl &L, const double *src, double *d, int ib, int ie,
                            cudaStream_t st) {
    if (ie <= ib) return cudaSuccess;
    g_launches.fetch_add(1, std::memory_order_relaxed);
    k_from_ref<<<dim3((ie - ib + 31) / 32, (L.nz + 31) / 32, L.ny), dim3(32, 8), 0, st>>>(
        L, src, d, ib, ie);
    return cudaGetLastError();
}

cudaError_t launch_to_ref(const Lvl &L, const double *d, double *dst, int ib, int ie,
                          cudaStream_t st) {
    if (ie <= ib) return cudaSuccess;
    g_launches.fetch_add(1, std::memory_order_relaxed);
    k_to_ref<<<dim3((ie - ib + 31) / 32, (L.nz + 31) / 32, L.ny), dim3(32, 8), 0, st>>>(
        L, d, dst, ib, ie);
    return cudaGetLastError();
}

}  // namespace pmg
