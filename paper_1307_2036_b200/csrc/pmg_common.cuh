// Shared definitions of libpmg (sm_100a).  See include/pmg.h for the layout.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include "../../include/pmg.h"

namespace pmg {

constexpr int OFF = PMG_OFF;
constexpr long long PARTIALS = 1LL << 22;   // doubles in a reduction scratch (32 MB)

// Kernel-side view of one level of one part.  Passed by value.
struct Lvl {
    int nx, ny, nz, pitch, par, uniform;
    long long plane;     // stride between vertical levels k (= pitch)
    long long jstride;   // stride between rows j (= nz * pitch)
    long long cstride;   // stride between the two colour arrays
    long long fcs;       // the same for right-hand sides f (= cstride, except in
                         // the lagged-norm driver's view of a red array held
                         // in another allocation: pmg_driver.cu)
    double omega2, vcoef;
    // uniform coefficients (2-D factors constant)
    double wx0, wy0, csub0;
    // 1-D device tables
    const double *drw;      // omega2 * dr[k]                       (stencil.py:103)
    const double *vprof;    // nz+1
    const double *volprof;  // nz
    const double *dr;       // nz
    const double *diag1;    // uniform diag3[k]                     (stencil.py:105-109)
    const double *band1;    // uniform (vcoef*av)*vprof[k], k=0..nz  (stencil.py:79-81)
    const double *invd1;    // uniform pivots                       (smoother.py:93-99)
    // k-segmented fast line solver (uniform): seg levels per warp and the
    // tables alpha[nz] mu[nz] pf[nz] q[nz] (see k_half_sweep_seg)
    int seg;
    const double *segtab;
    // bit3 (HF_WRAP): the part is periodic in x and y and the neighbour
    // reads of the half-sweep, residual-restriction and prolongation
    // kernels wrap around instead of reading the halo ring (which is then
    // not maintained: pmg_driver.cu's wrap views)
    int hflags;
    // tile region of the fast uniform half-sweeps (k_half_sweep_seg,
    // k_half_sweep_band): the 32-cell strips rx0 + s * rxs (s < rxn) of the
    // colour arrays, and the rows ry0 + t * rys (t < ryn).  The level's own
    // region is the whole part (0, 1, strips, 0, 1, ny); a boundary-first
    // multi-part sweep relaxes the frame and the interior as separate
    // regions (pmg_half_sweep_region, pmg_parts.cu)
    int rx0, rxs, rxn, ry0, rys, ryn;
    // 2-D device factors (variable coefficients)
    const double *wx, *wy, *av, *vh, *sumw;
    const double *invd;     // variable: per-cell pivots, field layout
};

constexpr int HF_WRAP = 8;

// neighbour coordinates: the periodic image when the level wraps, else the
// coordinate itself (-1 and n address the halo ring)
__host__ __device__ __forceinline__ int wrapx(const Lvl &L, int i) {
    return (L.hflags & HF_WRAP) ? (i < 0 ? i + L.nx : (i >= L.nx ? i - L.nx : i)) : i;
}
__host__ __device__ __forceinline__ int wrapy(const Lvl &L, int j) {
    return (L.hflags & HF_WRAP) ? (j < 0 ? j + L.ny : (j >= L.ny ? j - L.ny : j)) : j;
}

__host__ __device__ __forceinline__ long long at(const Lvl &L, int c, int k, int j, int h) {
    return (long long)c * L.cstride + (long long)(j + 1) * L.jstride + (long long)k * L.plane + OFF + h;
}
// natural (i, j) -> colour
__host__ __device__ __forceinline__ int colour(const Lvl &L, int i, int j) {
    return (i + j + L.par) & 1;
}
__host__ __device__ __forceinline__ long long cell(const Lvl &L, int i, int j, int k) {
    return at(L, colour(L, i, j), k, j, i >> 1);
}


// cell (i, j) of position t along face `face` (0 W, 1 E: t = j; 2 S, 3 N:
// t = i + 1 over the extended range -1 .. nx), on the halo ring or the
// adjacent owned row / column (partition.py:158-191)
__host__ __device__ __forceinline__ void face_pos(const Lvl &L, int face, int t, bool halo, int &i, int &j) {
    if (face < 2) {
        j = t;
        i = (face == 0) ? (halo ? -1 : 0) : (halo ? L.nx : L.nx - 1);
    } else {
        i = t - 1;
        j = (face == 2) ? (halo ? -1 : 0) : (halo ? L.ny : L.ny - 1);
    }
}

}  // namespace pmg
