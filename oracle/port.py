"""CPU oracle: a numpy restatement of the reference solver path.

TEST INFRASTRUCTURE ONLY.  Nothing in ``paper_1307_2036_b200`` imports
this module; only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may use it,
and only as the checker or as the timed CPU baseline.

It restates, operation by operation, the arithmetic of the reference
package ``panelmg`` (``/root/reference/pkg/src/panelmg``) for one worker
holding the whole grid, so results match the reference to the last bit
wherever numpy evaluates the same expression tree.  Parity of this port
is pinned against outputs of the real reference (run with the SURVEY
Appendix B injection) stored under ``tests/golden/`` by
``tests/golden/make_golden.py``; see ``tests/test_oracle_golden.py``.

Field layout is the reference's (``field.py:3-10``): a global array of
shape ``(nx+2, ny+2, nz)`` with a one-cell horizontal halo ring, vertical
index fastest.  Unlike the reference this port allows ``nx != ny``
(needed for the rectangular multi-GPU grids); square grids reproduce the
reference exactly.

Halo semantics per horizontal axis: ``periodic`` wraps (the Appendix B
neighbour override), otherwise the halo mirrors the adjacent owned value
(``partition.py:172-190``).
"""

from __future__ import annotations

import math
import time
from dataclasses import dataclass, field

import numpy as np

# ---------------------------------------------------------------------------
# coefficients (geometry.py:141-240 GridFactors / build_factors)
# ---------------------------------------------------------------------------


@dataclass(frozen=True)
class Factors:
    """Tensor-product stencil factors (reference ``GridFactors``,
    ``geometry.py:141-174``), rectangular: wx (nx+1, ny), wy (nx, ny+1),
    av/vh/sumw (nx, ny), dr/volprof (nz,), vprof (nz+1,)."""

    wx: np.ndarray
    wy: np.ndarray
    av: np.ndarray
    vh: np.ndarray
    sumw: np.ndarray
    dr: np.ndarray
    vprof: np.ndarray
    volprof: np.ndarray

    @property
    def nx(self):
        return self.av.shape[0]

    @property
    def ny(self):
        return self.av.shape[1]

    @property
    def nz(self):
        return self.dr.shape[0]


def uniform_levels(nz: int, depth: float) -> np.ndarray:
    """Level radii ``1 + H k/nz`` (uniform dz)."""
    return 1.0 + depth * np.arange(nz + 1, dtype=float) / nz


def graded_levels(nz: int, depth: float, stretch: float) -> np.ndarray:
    """Geometrically graded levels, dz_k = dz_0 * stretch**k, summing to
    ``depth``; last entry forced to exactly ``1 + depth`` as
    ``PanelGrid.__post_init__`` requires (``geometry.py:112-113``)."""
    dz = stretch ** np.arange(nz, dtype=float)
    dz *= depth / dz.sum()
    lv = np.empty(nz + 1)
    lv[0] = 1.0
    lv[1:] = 1.0 + np.cumsum(dz)
    lv[-1] = 1.0 + depth
    return lv


def reference_graded_levels(nz: int, depth: float) -> np.ndarray:
    """Reference default grading ``r_k = 1 + H (k/nz)^2`` (geometry.py:72-77)."""
    k = np.arange(nz + 1, dtype=float)
    return 1.0 + depth * (k / nz) ** 2


def omega_profile_config4(x, y):
    """configs[4] horizontal coefficient shape: 1 + 0.5 sin2πx sin2πy."""
    return 1.0 + 0.5 * np.sin(2.0 * math.pi * x) * np.sin(2.0 * math.pi * y)


def config_factors(nx: int, ny: int, levels: np.ndarray, omega_shape=None) -> Factors:
    """Factors of the BASELINE configs: flat
    doubly periodic unit square with dx = 1/nx (square cells, so ny must
    give the same spacing: the global domain is ny/nx long in y), face
    Dirichlet u=0 on top and bottom (vprof[0] = 2/dr[0], vprof[nz] =
    2/dr[-1]).  ``omega_shape(x, y)`` optionally scales the horizontal
    face weights at face midpoints and ``av`` at cell centres (configs[4]).
    """
    lv = np.asarray(levels, dtype=float)
    nz = lv.shape[0] - 1
    dxi = 1.0 / nx
    wx = np.ones((nx + 1, ny))
    wy = np.ones((nx, ny + 1))
    av = np.full((nx, ny), dxi * dxi)
    vh = np.full((nx, ny), dxi * dxi)
    if omega_shape is not None:
        xe = dxi * np.arange(nx + 1)
        xc = dxi * (np.arange(nx) + 0.5)
        ye = dxi * np.arange(ny + 1)
        yc = dxi * (np.arange(ny) + 0.5)
        wx = wx * omega_shape(xe[:, None], yc[None, :])
        wy = wy * omega_shape(xc[:, None], ye[None, :])
        av = av * omega_shape(xc[:, None], yc[None, :])
    sumw = wx[:-1, :] + wx[1:, :] + wy[:, :-1] + wy[:, 1:]
    dr = np.diff(lv)
    vprof = np.zeros(nz + 1)
    if nz > 1:
        vprof[1:nz] = 2.0 / (lv[2:] - lv[:-2])
    vprof[0] = 2.0 / dr[0]
    vprof[nz] = 2.0 / dr[-1]
    volprof = dr.copy()
    return Factors(wx, wy, av, vh, sumw, dr, vprof, volprof)


def flat_neumann_factors(nx: int, levels: np.ndarray) -> Factors:
    """The reference's own flat-mode factors (``geometry.py:190-206``):
    box [-1,1]^2, zero-flux lateral and vertical boundaries."""
    lv = np.asarray(levels, dtype=float)
    nz = lv.shape[0] - 1
    dr = np.diff(lv)
    vprof = np.zeros(nz + 1)
    if nz > 1:
        vprof[1:nz] = 2.0 / (lv[2:] - lv[:-2])
    volprof = dr.copy()
    dxi = 2.0 / nx
    wx = np.ones((nx + 1, nx))
    wx[0, :] = wx[nx, :] = 0.0
    wy = np.ones((nx, nx + 1))
    wy[:, 0] = wy[:, nx] = 0.0
    av = np.full((nx, nx), dxi * dxi)
    vh = np.full((nx, nx), dxi * dxi)
    sumw = wx[:-1, :] + wx[1:, :] + wy[:, :-1] + wy[:, 1:]
    return Factors(wx, wy, av, vh, sumw, dr, vprof, volprof)


# ---------------------------------------------------------------------------
# level operator (stencil.py:87-165)
# ---------------------------------------------------------------------------


class Level:
    """One grid level: factors + cached diagonal, vertical band, pivots.

    ``diag3`` follows ``stencil.py:105-109``; ``vband`` ``stencil.py:79-81``;
    the per-column pivots ``invd`` follow ``smoother.py:89-99``.
    """

    def __init__(self, fac: Factors, omega2: float, lambda2: float,
                 periodic=(True, True)):
        self.fac = fac
        self.nx, self.ny, self.nz = fac.nx, fac.ny, fac.nz
        self.omega2 = omega2
        self.vcoef = omega2 * lambda2
        self.periodic = tuple(periodic)
        f = fac
        self.diag3 = (
            f.vh[:, :, None] * f.volprof[None, None, :]
            + self.omega2 * f.sumw[:, :, None] * f.dr[None, None, :]
            + self.vcoef * f.av[:, :, None] * (f.vprof[:-1] + f.vprof[1:])[None, None, :]
        )
        self.drw = self.omega2 * f.dr[None, None, :]
        nz = self.nz
        self.vband = (self.vcoef * f.av[:, :, None] * f.vprof[None, None, 1:nz]
                      if nz > 1 else None)
        self.csub = self.vcoef * f.av                     # smoother.py:88
        invd = np.empty_like(self.diag3)                  # smoother.py:93-99
        invd[:, :, 0] = 1.0 / self.diag3[:, :, 0]
        for k in range(1, nz):
            sk = f.vprof[k] * self.csub
            invd[:, :, k] = 1.0 / (self.diag3[:, :, k] - sk * sk * invd[:, :, k - 1])
        self.invd = invd
        self.wxm = f.wx[:-1, :][:, :, None]
        self.wxp = f.wx[1:, :][:, :, None]
        self.wym = f.wy[:, :-1][:, :, None]
        self.wyp = f.wy[:, 1:][:, :, None]

    def zeros(self):
        return np.zeros((self.nx + 2, self.ny + 2, self.nz))

    def field(self, owned):
        d = self.zeros()
        d[1:-1, 1:-1, :] = owned
        halo_exchange(d, self.periodic)
        return d


def halo_exchange(d: np.ndarray, periodic=(True, True)) -> None:
    """Two-phase halo refresh of one whole-grid field (partition.py:158-191
    with P=1; periodic = the App. B wrapping neighbour map)."""
    m, n = d.shape[0] - 2, d.shape[1] - 2
    if periodic[0]:
        d[0, 1:-1, :] = d[m, 1:-1, :]
        d[m + 1, 1:-1, :] = d[1, 1:-1, :]
    else:
        d[0, 1:-1, :] = d[1, 1:-1, :]
        d[m + 1, 1:-1, :] = d[m, 1:-1, :]
    if periodic[1]:
        d[:, 0, :] = d[:, n, :]
        d[:, n + 1, :] = d[:, 1, :]
    else:
        d[:, 0, :] = d[:, 1, :]
        d[:, n + 1, :] = d[:, n, :]


def apply(lev: Level, d: np.ndarray, out=None) -> np.ndarray:
    """v = A u over owned cells, operation order of stencil.py:140-156."""
    if out is None:
        out = lev.zeros()
    uo = d[1:-1, 1:-1, :]
    res = out[1:-1, 1:-1, :]
    acc = lev.wxm * d[0:-2, 1:-1, :]
    tmp = lev.wxp * d[2:, 1:-1, :]
    acc += tmp
    np.multiply(lev.wym, d[1:-1, 0:-2, :], out=tmp)
    acc += tmp
    np.multiply(lev.wyp, d[1:-1, 2:, :], out=tmp)
    acc += tmp
    acc *= lev.drw
    np.multiply(lev.diag3, uo, out=res)
    res -= acc
    nz = lev.nz
    if nz > 1:
        t = tmp[:, :, :nz - 1]
        np.multiply(lev.vband, uo[:, :, :-1], out=t)
        res[:, :, 1:] -= t
        np.multiply(lev.vband, uo[:, :, 1:], out=t)
        res[:, :, :-1] -= t
    return out


def residual(lev: Level, f: np.ndarray, u: np.ndarray, out=None) -> np.ndarray:
    """r = f - A u (stencil.py:159-165)."""
    out = apply(lev, u, out)
    np.subtract(f[1:-1, 1:-1, :], out[1:-1, 1:-1, :], out=out[1:-1, 1:-1, :])
    return out


def norm(d: np.ndarray) -> float:
    """Owned-cell L2 norm (partition.py:267-286, one worker)."""
    o = d[1:-1, 1:-1, :]
    return math.sqrt(float(np.einsum("ijk,ijk->", o, o)))


def dot(a: np.ndarray, b: np.ndarray) -> float:
    return float(np.einsum("ijk,ijk->", a[1:-1, 1:-1, :], b[1:-1, 1:-1, :]))


# ---------------------------------------------------------------------------
# scalar Thomas algorithm (tridiag.py:59-100, paper Alg. 3)
# ---------------------------------------------------------------------------


def thomas_scalar(a, b, c, f) -> np.ndarray:
    """One tridiagonal system by forward elimination and back substitution,
    in the reference's operation order (tridiag.py:79-100): row 0 divides by
    its pivot, later rows multiply by the reciprocal.  Raises
    ``ArithmeticError`` at a pivot below 1e-300 in magnitude."""
    n = len(a)
    wp = np.empty(n)
    yp = np.empty(n)
    piv = a[0]
    if abs(piv) < 1e-300:
        raise ArithmeticError("zero pivot at row 0")
    if n == 1:
        return np.array([f[0] / piv])
    wp[0] = b[0] / piv
    yp[0] = f[0] / piv
    for i in range(1, n):
        piv = a[i] - wp[i - 1] * c[i - 1]
        if abs(piv) < 1e-300:
            raise ArithmeticError(f"zero pivot at row {i}")
        inv = 1.0 / piv
        if i + 1 < n:
            wp[i] = b[i] * inv
        yp[i] = (f[i] - yp[i - 1] * c[i - 1]) * inv
    x = np.empty(n)
    x[n - 1] = yp[n - 1]
    for i in range(n - 2, -1, -1):
        x[i] = yp[i] - wp[i] * x[i + 1]
    return x


# ---------------------------------------------------------------------------
# line smoother (smoother.py:102-244)
# ---------------------------------------------------------------------------

RED, BLACK = 0, 1


def half_sweep(lev: Level, u: np.ndarray, f: np.ndarray, color: int,
               rho: float = 1.0, zero_start: bool = False,
               neighbors_zero: bool = False, post_scale: float = 1.0) -> None:
    """Update every column of one colour (smoother.py:122-182).

    Red = (i + j) even in global indices (smoother.py:66).  The
    reference splits a colour into strided sub-lattices only for
    vectorisation; per column the arithmetic is identical, so this port
    treats all columns of one colour at once via a boolean mask.
    """
    nz = lev.nz
    vp = lev.fac.vprof
    ii, jj = np.meshgrid(np.arange(lev.nx), np.arange(lev.ny), indexing="ij")
    mask = ((ii + jj) % 2) == color
    ci, cj = ii[mask], jj[mask]
    fo = f[1 + ci, 1 + cj, :]
    if neighbors_zero:
        g = fo.copy()
    else:
        g = lev.wxm[ci, cj] * u[ci, 1 + cj, :]
        tmp = lev.wxp[ci, cj] * u[2 + ci, 1 + cj, :]
        g += tmp
        np.multiply(lev.wym[ci, cj], u[1 + ci, cj, :], out=tmp)
        g += tmp
        np.multiply(lev.wyp[ci, cj], u[1 + ci, 2 + cj, :], out=tmp)
        g += tmp
        g *= lev.drw[0]
        g += fo
    invd = lev.invd[ci, cj, :]
    csub = lev.csub[ci, cj]
    g[:, 0] *= invd[:, 0]
    for k in range(1, nz):
        tmp = g[:, k - 1] * csub
        tmp *= vp[k]
        g[:, k] += tmp
        g[:, k] *= invd[:, k]
    for k in range(nz - 2, -1, -1):
        tmp = g[:, k + 1] * csub
        tmp *= vp[k + 1]
        tmp *= invd[:, k]
        g[:, k] += tmp
    if zero_start:
        scale = rho * post_scale
        if scale != 1.0:
            g *= scale
    elif rho != 1.0:
        g *= rho
        g += (1.0 - rho) * u[1 + ci, 1 + cj, :]
    u[1 + ci, 1 + cj, :] = g


def sweep(lev: Level, u, f, nsweeps: int = 1, rho: float = 1.0) -> None:
    """Red-black sweep with an exchange after each half (smoother.py:184-191)."""
    for _ in range(nsweeps):
        half_sweep(lev, u, f, RED, rho)
        halo_exchange(u, lev.periodic)
        half_sweep(lev, u, f, BLACK, rho)
        halo_exchange(u, lev.periodic)


def symmetric_sweep(lev: Level, u, f, nsweeps: int = 1, rho: float = 1.0) -> None:
    """smoother.py:193-208."""
    for _ in range(nsweeps):
        half_sweep(lev, u, f, RED, rho)
        halo_exchange(u, lev.periodic)
        half_sweep(lev, u, f, BLACK, rho)
        if rho != 1.0:
            half_sweep(lev, u, f, BLACK, rho)
        halo_exchange(u, lev.periodic)
        half_sweep(lev, u, f, RED, rho)
        halo_exchange(u, lev.periodic)


def jacobi_sweep(lev: Level, u, f, nsweeps: int = 1, rho: float = 1.0) -> None:
    """Block-Jacobi line relaxation (smoother.py:210-222): every column
    from the pre-sweep state."""
    for _ in range(nsweeps):
        old = u.copy()
        for color in (RED, BLACK):
            tmp = old.copy()
            half_sweep(lev, tmp, f, color, rho)
            ii, jj = np.meshgrid(np.arange(lev.nx), np.arange(lev.ny), indexing="ij")
            mask = ((ii + jj) % 2) == color
            u[1:-1, 1:-1, :][mask] = tmp[1:-1, 1:-1, :][mask]
        halo_exchange(u, lev.periodic)


def ssor_apply(lev: Level, r: np.ndarray, rho: float = 1.0, out=None) -> np.ndarray:
    """z = M^{-1} r (smoother.py:224-244)."""
    z = lev.zeros() if out is None else out
    z.fill(0.0)
    half_sweep(lev, z, r, RED, rho, zero_start=True, neighbors_zero=True)
    halo_exchange(z, lev.periodic)
    half_sweep(lev, z, r, BLACK, rho, zero_start=True, post_scale=2.0 - rho)
    halo_exchange(z, lev.periodic)
    half_sweep(lev, z, r, RED, rho)
    halo_exchange(z, lev.periodic)
    return z


# ---------------------------------------------------------------------------
# transfers (multigrid.py:209-268)
# ---------------------------------------------------------------------------


def restrict_into(fine: np.ndarray, coarse: np.ndarray, weight: float) -> None:
    """Children sum (weight 1, V-cycle) or mean (0.25), multigrid.py:209-214."""
    fo = fine[1:-1, 1:-1, :]
    co = coarse[1:-1, 1:-1, :]
    co[...] = fo[0::2, 0::2, :] + fo[1::2, 0::2, :]
    co += fo[0::2, 1::2, :]
    co += fo[1::2, 1::2, :]
    if weight != 1.0:
        co *= weight


def prolong_into(cdata: np.ndarray, out: np.ndarray) -> None:
    """9-3-3-1 bilinear cell-centre interpolation, multigrid.py:233-246.
    ``cdata`` needs a current halo including corners; writes owned cells."""
    cc = cdata[1:-1, 1:-1, :]
    cw = cdata[0:-2, 1:-1, :]
    ce = cdata[2:, 1:-1, :]
    cs = cdata[1:-1, 0:-2, :]
    cn = cdata[1:-1, 2:, :]
    csw = cdata[0:-2, 0:-2, :]
    cse = cdata[2:, 0:-2, :]
    cnw = cdata[0:-2, 2:, :]
    cne = cdata[2:, 2:, :]
    o = out[1:-1, 1:-1, :]
    o[0::2, 0::2, :] = (9.0 * cc + 3.0 * cw + 3.0 * cs + csw) * 0.0625
    o[1::2, 0::2, :] = (9.0 * cc + 3.0 * ce + 3.0 * cs + cse) * 0.0625
    o[0::2, 1::2, :] = (9.0 * cc + 3.0 * cw + 3.0 * cn + cnw) * 0.0625
    o[1::2, 1::2, :] = (9.0 * cc + 3.0 * ce + 3.0 * cn + cne) * 0.0625


# ---------------------------------------------------------------------------
# solvers (multigrid.py:271-330, krylov.py:88-167)
# ---------------------------------------------------------------------------


@dataclass
class Report:
    """Mirror of ``SolveReport`` (krylov.py:33-58)."""

    iterations: int
    residual_history: list
    converged: bool
    wall_time: float
    residual_drift: float = 0.0


class Hierarchy:
    """Levels finest first (multigrid.py:116-206, explicit level count).

    ``factor_fn(nx, ny)`` returns the factors of a level (the App. B
    factory is looked up per level the same way, ``multigrid.py:195``).
    """

    def __init__(self, nx, ny, nlevels, factor_fn, omega2, lambda2,
                 periodic=(True, True)):
        self.levels = []
        for c in range(nlevels):
            if nx < 1 or ny < 1:
                raise ValueError("too many levels for the grid")
            self.levels.append(Level(factor_fn(nx, ny), omega2, lambda2, periodic))
            nx //= 2
            ny //= 2
        self.scratch = [(lv.zeros(), lv.zeros(), lv.zeros()) for lv in self.levels]


def v_cycle(h: Hierarchy, nu_pre=1, nu_post=1, coarse_sweeps=1, rho=1.0, c=0) -> None:
    """Alg. 1, multigrid.py:271-294."""
    lev = h.levels[c]
    u, f, r = h.scratch[c]
    if c + 1 < len(h.levels):
        sweep(lev, u, f, nu_pre, rho)
        residual(lev, f, u, out=r)
        cu, cf, _ = h.scratch[c + 1]
        restrict_into(r, cf, 1.0)
        cu.fill(0.0)
        v_cycle(h, nu_pre, nu_post, coarse_sweeps, rho, c + 1)
        prolong_into(cu, r)
        u[1:-1, 1:-1, :] += r[1:-1, 1:-1, :]
        halo_exchange(u, lev.periodic)
        sweep(lev, u, f, nu_post, rho)
    else:
        sweep(lev, u, f, coarse_sweeps, rho)


def mg_solve(h: Hierarchy, f_owned: np.ndarray, eps=1e-5, maxiter=100,
             nu_pre=1, nu_post=1, coarse_sweeps=1, rho=1.0, max_cycles=None):
    """multigrid.py:297-330.  ``max_cycles`` truncates the loop (CPU
    baseline sampling only; the report then says not converged)."""
    u, f, r = h.scratch[0]
    for lv_u, lv_f, lv_r in h.scratch:
        lv_u.fill(0.0)
    f.fill(0.0)
    f[1:-1, 1:-1, :] = f_owned
    lev = h.levels[0]
    r0 = norm(f)
    hist = [r0]
    if r0 == 0.0:
        return u, Report(0, hist, True, 0.0)
    conv = False
    t0 = time.perf_counter()
    n = maxiter if max_cycles is None else min(maxiter, max_cycles)
    for _ in range(n):
        v_cycle(h, nu_pre, nu_post, coarse_sweeps, rho)
        rn = norm(residual(lev, f, u, out=r))
        hist.append(rn)
        if rn / r0 < eps:
            conv = True
            break
    return u, Report(len(hist) - 1, hist, conv, time.perf_counter() - t0)


class BreakdownError(ArithmeticError):
    pass


def pcg_solve(lev: Level, f_owned: np.ndarray, eps=1e-5, maxiter=500,
              tau=1e-300, rho=1.0, precond="ssor", max_iters=None):
    """krylov.py:88-167 with the SSOR line preconditioner (krylov.py:70-85)
    or the identity (krylov.py:61-67)."""
    f = lev.zeros()
    f[1:-1, 1:-1, :] = f_owned
    u = lev.zeros()
    r = f.copy()
    r0 = norm(r)
    hist = [r0]
    if r0 == 0.0 or r0 < tau:
        return u, Report(0, hist, True, 0.0)

    zbuf = lev.zeros()

    def prec(rr):
        if precond == "ssor":
            return ssor_apply(lev, rr, rho, out=zbuf)
        z = rr.copy()
        halo_exchange(z, lev.periodic)
        return z

    t0 = time.perf_counter()
    z = prec(r)
    p = z.copy()
    kappa = dot(r, z)
    if kappa <= 0.0:
        raise BreakdownError("<r, z> <= 0")
    q = lev.zeros()
    conv = False
    it = 0
    rn = r0
    n = maxiter if max_iters is None else min(maxiter, max_iters)
    for it in range(1, n + 1):
        apply(lev, p, out=q)
        pq = dot(p, q)
        if pq <= 0.0:
            raise BreakdownError("<p, A p> <= 0")
        alpha = kappa / pq
        u += alpha * p
        r -= alpha * q
        rn = norm(r)
        hist.append(rn)
        if rn / r0 < eps or rn < tau:
            conv = True
            break
        z = prec(r)
        kn = dot(r, z)
        if kn <= 0.0:
            raise BreakdownError("<r, z> <= 0")
        p *= kn / kappa
        p += z
        kappa = kn
    wall = time.perf_counter() - t0
    true = norm(residual(lev, f, u))
    return u, Report(it, hist, conv, wall, residual_drift=abs(true - rn))


# ---------------------------------------------------------------------------
# BASELINE configs and the seeded right-hand side (bench.py:170-174)
# ---------------------------------------------------------------------------


def rhs(nx: int, ny: int, nz: int, seed: int = 0) -> np.ndarray:
    """``default_rng(seed).uniform(-1, 1, (nx, ny, nz))`` (bench.py:173-174)."""
    return np.random.default_rng(seed).uniform(-1.0, 1.0, size=(nx, ny, nz))


def rhs_block(nx_glob, ny_glob, nz, i0, j0, mx, my, seed=0) -> np.ndarray:
    """Rows [i0, i0+mx) x [j0, j0+my) of ``rhs`` without materialising the
    global array: PCG64 streams advanced per row."""
    out = np.empty((mx, my, nz))
    for ii in range(mx):
        bg = np.random.PCG64(seed)
        bg.advance(((i0 + ii) * ny_glob + j0) * nz)
        out[ii] = np.random.Generator(bg).uniform(-1.0, 1.0, (my, nz))
    return out


@dataclass
class Config:
    nx: int
    ny: int
    nz: int
    depth: float
    omega2: float
    lambda2: float
    levels: int
    stretch: float | None = None
    variable_omega: bool = False

    def level_radii(self):
        if self.stretch is None:
            return uniform_levels(self.nz, self.depth)
        return graded_levels(self.nz, self.depth, self.stretch)

    def factor_fn(self):
        lv = self.level_radii()
        shape = omega_profile_config4 if self.variable_omega else None
        return lambda nx, ny: config_factors(nx, ny, lv, shape)

    def hierarchy(self):
        return Hierarchy(self.nx, self.ny, self.levels, self.factor_fn(),
                         self.omega2, self.lambda2)

    def level(self):
        return Level(self.factor_fn()(self.nx, self.ny), self.omega2, self.lambda2)


CONFIGS = {
    0: Config(64, 64, 32, 0.01, 1e-3, 1.0, 4),
    1: Config(1024, 1024, 128, 0.01, 1e-3, 1.0, 7),
    2: Config(1024, 1024, 128, 0.01, 1e-3, 1.0, 7),
    3: Config(2048, 2048, 128, 0.01, 1e-3, 1.0, 8),
    4: Config(4096, 4096, 128, 0.01, 1e-3, 1.0, 9, stretch=1.05, variable_omega=True),
}
