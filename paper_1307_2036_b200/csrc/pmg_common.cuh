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
    // 2-D device factors (variable coefficients)
    const double *wx, *wy, *av, *vh, *sumw;
    const double *invd;     // variable: per-cell pivots, field layout
};

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

}  // namespace pmg
