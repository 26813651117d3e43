// libpmg device kernels for B200 (sm_100a).
//
// Every kernel is HBM-bound fp64 stencil / tridiagonal / BLAS-1 work
// (SURVEY.md section 8d): no tensor cores.  Arithmetic follows the
// reference's numpy expression trees term by term and the library is
// compiled with --fmad=false, so operator, smoother and transfers are
// bit-identical to the reference (see tests/test_gpu_parity.py).
//
// Layout: red/black split, horizontal index fastest (include/pmg.h).
#include "pmg_common.cuh"

namespace pmg {

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
        double *__restrict__ out, double *__restrict__ partials) {
    const int lane = threadIdx.x;
    const int c = threadIdx.y & 1;
    const int j = blockIdx.y * AP_TY + (threadIdx.y >> 1);
    const int h = blockIdx.x * 32 + lane;
    const int i = 2 * h + ((j + L.par + c) & 1);
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
        double um = 0.0, u0 = u[pc], up = 0.0;
#pragma unroll 4
        for (int k = 0; k < nz; ++k) {
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
            partials[blockIdx.y * gridDim.x + blockIdx.x] = s;
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
                    double *__restrict__ cf) {
    const int I = blockIdx.x * blockDim.x + threadIdx.x;
    const int J = blockIdx.y * blockDim.y + threadIdx.y;
    if (I >= C.nx || J >= C.ny) return;
    const int i0 = 2 * I, j0 = 2 * J;
    const long long q00 = cell(F, i0, j0, 0), q10 = cell(F, i0 + 1, j0, 0);
    const long long q01 = cell(F, i0, j0 + 1, 0), q11 = cell(F, i0 + 1, j0 + 1, 0);
    const long long pl = F.plane;
    double m00 = 0, m10 = 0, m01 = 0, m11 = 0;
    double c00 = u[q00], c10 = u[q10], c01 = u[q01], c11 = u[q11];
    const long long qc = cell(C, I, J, 0);
    for (int k = 0; k < F.nz; ++k) {
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
template <bool UNI>
__global__ void __launch_bounds__(256, 3)
k_half_sweep(Lvl L, double *__restrict__ u, const double *__restrict__ f, int c, double rho,
             int zero_start, int nbr_zero, double post_scale) {
    extern __shared__ double smem[];
    const int nz = L.nz;
    double *s = smem;                                // [nz][32]  rhs -> g
    double *so = smem + nz * 32;                     // [nz][32]  u_old (rho != 1)
    double *sinv = so + ((!zero_start && rho != 1.0) ? nz * 32 : 0);   // [nz][32] (var)
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int j = blockIdx.y;
    const int h = blockIdx.x * 32 + lane;
    const int i = 2 * h + ((j + L.par + c) & 1);
    const bool act = i < L.nx;
    const bool need_old = !zero_start && rho != 1.0;
    const int o = c ^ 1;
    const long long pc = at(L, c, 0, j, h);
    const long long pl = L.plane;

    double cv = L.csub0;
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
            if (need_old) so[k * 32 + lane] = u[pc + ko];
            if (!UNI) sinv[k * 32 + lane] = L.invd[pc + ko];
        }
    }
    __syncthreads();
    if (w != 0 || !act) return;
    if (!UNI) cv = L.vcoef * L.av[(long long)j * L.nx + i];
    const double *vp = L.vprof;
    // forward elimination (smoother.py:151-156)
    double g = s[lane] * (UNI ? L.invd1[0] : sinv[lane]);
    s[lane] = g;
#pragma unroll 4
    for (int k = 1; k < nz; ++k) {
        double t = g * cv;
        t = t * vp[k];
        g = s[k * 32 + lane] + t;
        g = g * (UNI ? L.invd1[k] : sinv[k * 32 + lane]);
        s[k * 32 + lane] = g;
    }
    // back substitution (smoother.py:157-161) + relaxation (163-170)
    const double scale = rho * post_scale;
    const double omr = 1.0 - rho;
    double x = g;
    for (int k = nz - 1; k >= 0; --k) {
        if (k < nz - 1) {
            double t = x * cv;
            t = t * vp[k + 1];
            t = t * (UNI ? L.invd1[k] : sinv[k * 32 + lane]);
            x = s[k * 32 + lane] + t;
        }
        double y = x;
        if (zero_start) {
            if (scale != 1.0) y = y * scale;
        } else if (rho != 1.0) {
            y = y * rho;
            y = y + omr * so[k * 32 + lane];
        }
        u[pc + (long long)k * pl] = y;
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
    const int J = blockIdx.y;
    const int k = blockIdx.z;
    if (I >= C.nx) return;
    const int i0 = 2 * I, j0 = 2 * J;
    double a = fu[cell(F, i0, j0, k)] + fu[cell(F, i0 + 1, j0, k)];
    a = a + fu[cell(F, i0, j0 + 1, k)];
    a = a + fu[cell(F, i0 + 1, j0 + 1, k)];
    if (weight != 1.0) a = a * weight;
    cu[cell(C, I, J, k)] = a;
}

__global__ void k_prolong(Lvl F, Lvl C, const double *__restrict__ cu, double *__restrict__ fu,
                          int add) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    const int j = blockIdx.y;
    const int k = blockIdx.z;
    const int c = t & 1;                 // interleave colours inside a warp
    const int h = t >> 1;
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
    fu[q] = add ? fu[q] + e : e;
}

// ---------------------------------------------------------------------------
// halos (partition.py:158-191)
// ---------------------------------------------------------------------------
__device__ __forceinline__ int hmap(int i, int n, int periodic) {
    if (i < 0) return periodic ? n - 1 : 0;
    if (i >= n) return periodic ? 0 : n - 1;
    return i;
}

// whole ring of a part that is its own neighbour in both directions
__global__ void k_halo_self(Lvl L, double *__restrict__ d, int px, int py) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    const int k = blockIdx.y;
    const int nring = 2 * (L.nx + 2) + 2 * L.ny;
    if (t >= nring) return;
    int i, j;
    if (t < L.nx + 2) {
        i = t - 1; j = -1;
    } else if (t < 2 * (L.nx + 2)) {
        i = t - (L.nx + 2) - 1; j = L.ny;
    } else if (t < 2 * (L.nx + 2) + L.ny) {
        i = -1; j = t - 2 * (L.nx + 2);
    } else {
        i = L.nx; j = t - 2 * (L.nx + 2) - L.ny;
    }
    d[cell(L, i, j, k)] = d[cell(L, hmap(i, L.nx, px), hmap(j, L.ny, py), k)];
}

__device__ __forceinline__ void face_pos(const Lvl &L, int face, int t, bool halo, int &i, int &j) {
    if (face < 2) {
        j = t;
        i = (face == 0) ? (halo ? -1 : 0) : (halo ? L.nx : L.nx - 1);
    } else {
        i = t - 1;
        j = (face == 2) ? (halo ? -1 : 0) : (halo ? L.ny : L.ny - 1);
    }
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

// ---------------------------------------------------------------------------
// reductions and BLAS-1 (partition.py:138-155, 267-286)
// ---------------------------------------------------------------------------
// Owned cells enumerated as rows (c, k, j) x h; block b takes rows b,
// b+grid, ...; fixed grid => fixed summation order (deterministic).
__global__ void __launch_bounds__(256)
k_dot(Lvl L, const double *__restrict__ a, const double *__restrict__ b,
      double *__restrict__ partials) {
    const int rowlen = (L.nx + 1) >> 1;
    const int nrows = 2 * L.nz * L.ny;
    double s = 0.0;
    for (int r = blockIdx.x; r < nrows; r += gridDim.x) {
        const int j = r % L.ny;
        const int ck = r / L.ny;
        const int k = ck % L.nz, c = ck / L.nz;
        const int s0 = (j + L.par + c) & 1;
        const long long base = at(L, c, k, j, 0);
        for (int h = threadIdx.x; h < rowlen; h += blockDim.x) {
            if (2 * h + s0 < L.nx) s += a[base + h] * b[base + h];
        }
    }
    s = block_sum(s);
    if (threadIdx.x == 0) partials[blockIdx.x] = s;
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

// u += alpha p ; r -= alpha q over the full allocation (halo included, as
// DistField.add_scaled, partition.py:145-148); partial ||r||^2 over owned.
// Rows of the allocation are (c, k, jj) with jj in [0, ny+2), pitch wide.
__global__ void __launch_bounds__(256)
k_cg_update(Lvl L, const double *__restrict__ num, const double *__restrict__ den,
            const double *__restrict__ p, const double *__restrict__ q, double *__restrict__ u,
            double *__restrict__ r, double *__restrict__ partials) {
    const double alpha = num[0] / den[0];
    const double malpha = -alpha;
    const int rows_per_plane = L.ny + 2;
    const int nrows = 2 * L.nz * rows_per_plane;
    double s = 0.0;
    for (int row = blockIdx.x; row < nrows; row += gridDim.x) {
        const int jj = row % rows_per_plane;
        const int c = row / (rows_per_plane * L.nz);
        const int j = jj - 1;
        const int s0 = (j + L.par + c) & 1;
        const long long base = (long long)row * L.pitch;
        const bool owned_row = (j >= 0 && j < L.ny);
        for (int t = threadIdx.x; t < L.pitch; t += blockDim.x) {
            const long long e = base + t;
            u[e] = u[e] + alpha * p[e];
            const double rv = r[e] + malpha * q[e];
            r[e] = rv;
            const int h = t - OFF;
            if (owned_row && h >= 0 && 2 * h + s0 < L.nx) s += rv * rv;
        }
    }
    s = block_sum(s);
    if (threadIdx.x == 0) partials[blockIdx.x] = s;
}

// ---------------------------------------------------------------------------
// layout conversion: reference (nx, ny, nz) k-fastest <-> split layout.
// 32x32 (i, k) tiles through shared memory so both sides are coalesced.
// ---------------------------------------------------------------------------
__global__ void k_from_ref(Lvl L, const double *__restrict__ src, double *__restrict__ d) {
    __shared__ double tile[32][33];
    const int i0 = blockIdx.x * 32, k0 = blockIdx.z * 32, j = blockIdx.y;
    const int tx = threadIdx.x, ty = threadIdx.y;   // 32 x 8
    for (int r = ty; r < 32; r += 8) {
        const int i = i0 + r, k = k0 + tx;
        if (i < L.nx && k < L.nz) tile[r][tx] = src[((long long)i * L.ny + j) * L.nz + k];
    }
    __syncthreads();
    for (int r = ty; r < 32; r += 8) {
        const int i = i0 + tx, k = k0 + r;
        if (i < L.nx && k < L.nz) d[cell(L, i, j, k)] = tile[tx][r];
    }
}

__global__ void k_to_ref(Lvl L, const double *__restrict__ d, double *__restrict__ dst) {
    __shared__ double tile[32][33];
    const int i0 = blockIdx.x * 32, k0 = blockIdx.z * 32, j = blockIdx.y;
    const int tx = threadIdx.x, ty = threadIdx.y;
    for (int r = ty; r < 32; r += 8) {
        const int i = i0 + tx, k = k0 + r;
        if (i < L.nx && k < L.nz) tile[tx][r] = d[cell(L, i, j, k)];
    }
    __syncthreads();
    for (int r = ty; r < 32; r += 8) {
        const int i = i0 + r, k = k0 + tx;
        if (i < L.nx && k < L.nz) dst[((long long)i * L.ny + j) * L.nz + k] = tile[r][tx];
    }
}

// ===========================================================================
// host launchers
// ===========================================================================
static inline dim3 apply_grid(const Lvl &L) {
    const int hx = ((L.nx + 1) / 2 + 31) / 32;
    return dim3(hx, (L.ny + AP_TY - 1) / AP_TY);
}

cudaError_t launch_apply(const Lvl &L, const double *u, const double *f, double *out, int mode,
                         double *partials, int *nparts, cudaStream_t st) {
    const dim3 g = apply_grid(L), b(32, 2 * AP_TY);
    *nparts = g.x * g.y;
    if ((long long)g.x * g.y > PARTIALS) return cudaErrorInvalidValue;
    const bool norm = partials != nullptr;
#define PMG_AP(U, M, N) k_apply<U, M, N><<<g, b, 0, st>>>(L, u, f, out, partials)
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
    k_finalize<<<1, 1024, 0, st>>>(partials, n, out);
    return cudaGetLastError();
}

cudaError_t launch_residual_restrict(const Lvl &F, const Lvl &C, const double *u, const double *f,
                                     double *cf, cudaStream_t st) {
    const dim3 b(32, 8), g((C.nx + 31) / 32, (C.ny + 7) / 8);
    if (F.uniform) k_residual_restrict<true><<<g, b, 0, st>>>(F, C, u, f, cf);
    else k_residual_restrict<false><<<g, b, 0, st>>>(F, C, u, f, cf);
    return cudaGetLastError();
}

size_t half_sweep_smem(const Lvl &L, bool need_old) {
    size_t n = (size_t)L.nz * 32;
    return sizeof(double) * (n + (need_old ? n : 0) + (L.uniform ? 0 : n));
}

cudaError_t launch_half_sweep(const Lvl &L, double *u, const double *f, int color, double rho,
                              int zero_start, int nbr_zero, double post_scale, cudaStream_t st) {
    const bool need_old = !zero_start && rho != 1.0;
    const size_t sm = half_sweep_smem(L, need_old);
    const int hx = ((L.nx + 1) / 2 + 31) / 32;
    const dim3 g(hx, L.ny);
    const int nw = L.nz >= 8 ? 8 : (L.nz >= 4 ? 4 : (L.nz >= 2 ? 2 : 1));
    const dim3 b(32 * nw);
    static bool attr_set[2] = {false, false};
    if (L.uniform) {
        if (!attr_set[0]) {
            cudaFuncSetAttribute(k_half_sweep<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 200 * 1024);
            attr_set[0] = true;
        }
        k_half_sweep<true><<<g, b, sm, st>>>(L, u, f, color, rho, zero_start, nbr_zero, post_scale);
    } else {
        if (!attr_set[1]) {
            cudaFuncSetAttribute(k_half_sweep<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 200 * 1024);
            attr_set[1] = true;
        }
        k_half_sweep<false><<<g, b, sm, st>>>(L, u, f, color, rho, zero_start, nbr_zero, post_scale);
    }
    return cudaGetLastError();
}

cudaError_t launch_invd(const Lvl &L, double *invd, cudaStream_t st) {
    k_invd<<<dim3((L.nx + 127) / 128, L.ny), 128, 0, st>>>(L, invd);
    return cudaGetLastError();
}

cudaError_t launch_restrict(const Lvl &F, const Lvl &C, const double *fu, double *cu, double w,
                            cudaStream_t st) {
    k_restrict<<<dim3((C.nx + 127) / 128, C.ny, C.nz), 128, 0, st>>>(F, C, fu, cu, w);
    return cudaGetLastError();
}

cudaError_t launch_prolong(const Lvl &F, const Lvl &C, const double *cu, double *fu, int add,
                           cudaStream_t st) {
    const int n2 = 2 * ((F.nx + 1) / 2);
    k_prolong<<<dim3((n2 + 127) / 128, F.ny, F.nz), 128, 0, st>>>(F, C, cu, fu, add);
    return cudaGetLastError();
}

cudaError_t launch_halo_self(const Lvl &L, double *d, int px, int py, cudaStream_t st) {
    const int nring = 2 * (L.nx + 2) + 2 * L.ny;
    k_halo_self<<<dim3((nring + 127) / 128, L.nz), 128, 0, st>>>(L, d, px, py);
    return cudaGetLastError();
}

int face_len(const Lvl &L, int face) { return face < 2 ? L.ny : L.nx + 2; }

cudaError_t launch_pack(const Lvl &L, const double *d, int face, double *buf, cudaStream_t st) {
    const int len = face_len(L, face);
    k_pack_face<<<dim3((len + 127) / 128, L.nz), 128, 0, st>>>(L, d, face, buf, len);
    return cudaGetLastError();
}

cudaError_t launch_unpack(const Lvl &L, double *d, int face, const double *buf, int mirror,
                          cudaStream_t st) {
    const int len = face_len(L, face);
    k_unpack_face<<<dim3((len + 127) / 128, L.nz), 128, 0, st>>>(L, d, face, buf, len, mirror);
    return cudaGetLastError();
}

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

static inline int stream_blocks(long long n) {
    long long b = (n + 255) / 256;
    long long cap = 4LL * sm_count();
    return (int)(b < cap ? (b > 0 ? b : 1) : cap);
}

cudaError_t launch_dot(const Lvl &L, const double *a, const double *b, double *partials, int *np,
                       cudaStream_t st) {
    const long long n = 2LL * L.nz * L.ny * ((L.nx + 1) >> 1);
    int g = stream_blocks(n);
    if (g > 2 * L.nz * L.ny) g = 2 * L.nz * L.ny;
    *np = g;
    k_dot<<<g, 256, 0, st>>>(L, a, b, partials);
    return cudaGetLastError();
}

cudaError_t launch_axpy(long long n, double a, const double *x, double *y, cudaStream_t st) {
    k_axpy<<<stream_blocks(n), 256, 0, st>>>(n, a, x, y);
    return cudaGetLastError();
}

cudaError_t launch_xpby(long long n, const double *x, double b, double *y, cudaStream_t st) {
    k_xpby<<<stream_blocks(n), 256, 0, st>>>(n, x, b, y);
    return cudaGetLastError();
}

cudaError_t launch_cg_direction(long long n, const double *num, const double *den, const double *z,
                                double *p, cudaStream_t st) {
    k_cg_direction<<<stream_blocks(n), 256, 0, st>>>(n, num, den, z, p);
    return cudaGetLastError();
}

cudaError_t launch_cg_update(const Lvl &L, const double *num, const double *den,
                             const double *p, const double *q, double *u, double *r,
                             double *partials, int *np, cudaStream_t st) {
    const long long n = 2LL * L.cstride;
    int g = stream_blocks(n);
    if (g > 2 * L.nz * (L.ny + 2)) g = 2 * L.nz * (L.ny + 2);
    *np = g;
    k_cg_update<<<g, 256, 0, st>>>(L, num, den, p, q, u, r, partials);
    return cudaGetLastError();
}

cudaError_t launch_from_ref(const Lvl &L, const double *src, double *d, cudaStream_t st) {
    k_from_ref<<<dim3((L.nx + 31) / 32, L.ny, (L.nz + 31) / 32), dim3(32, 8), 0, st>>>(L, src, d);
    return cudaGetLastError();
}

cudaError_t launch_to_ref(const Lvl &L, const double *d, double *dst, cudaStream_t st) {
    k_to_ref<<<dim3((L.nx + 31) / 32, L.ny, (L.nz + 31) / 32), dim3(32, 8), 0, st>>>(L, d, dst);
    return cudaGetLastError();
}

}  // namespace pmg
