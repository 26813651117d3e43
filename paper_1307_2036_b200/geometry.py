"""Grids and tensor-product stencil factors (reference ``geometry.py``).

The solver consumes ``GridFactors`` exactly as the reference does
(``geometry.py:141-174``): horizontal transmissibility ``wx[i,j]*dr[k]``,
vertical ``av[i,j]*vprof[k]``, volume ``vh[i,j]*volprof[k]``.  Three
problem families are built here:

* ``flat_mode=True`` -- the reference's flat box ``[-1,1]^2`` with
  zero-flux boundaries (``geometry.py:190-206``);
* default -- the reference's gnomonic cubed-sphere panel
  (``geometry.py:207-236``), re-derived here from the same geometric
  definitions (chord cross products, parallelepiped volumes);
* ``periodic=True`` -- the BASELINE configs: the doubly periodic unit
  square with face-Dirichlet top/bottom (``dirichlet_z``) and an optional
  ``omega_shape(x, y)`` scaling of the horizontal coefficient
  (SURVEY Appendix B).  ``ny`` may differ from ``nx`` (rectangular
  global grids of the multi-GPU configs).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Callable, Optional

import numpy as np

from .params import is_power_of_two


def vertical_levels(nz: int, depth: float) -> np.ndarray:
    """Reference grading ``r_k = 1 + depth (k/nz)^2`` (geometry.py:72-77)."""
    if nz < 1:
        raise ValueError("nz must be at least 1")
    k = np.arange(nz + 1, dtype=float)
    return 1.0 + depth * (k / nz) ** 2


def uniform_levels(nz: int, depth: float) -> np.ndarray:
    """Uniform spacing ``1 + depth k / nz`` (configs[0-3])."""
    return 1.0 + depth * np.arange(nz + 1, dtype=float) / nz


def graded_levels(nz: int, depth: float, stretch: float) -> np.ndarray:
    """Geometric grading dz_k = dz_0 stretch^k from the bottom (configs[4]);
    the top is pinned to exactly ``1 + depth``."""
    dz = stretch ** np.arange(nz, dtype=float)
    dz *= depth / dz.sum()
    lv = np.empty(nz + 1)
    lv[0] = 1.0
    lv[1:] = 1.0 + np.cumsum(dz)
    lv[-1] = 1.0 + depth
    return lv


def map_to_sphere(xi1, xi2, r, depth: float | None = None):
    """Gnomonic panel map (geometry.py:47-69): r (xi1, xi2, 1)/|(xi1, xi2, 1)|."""
    xi1 = np.asarray(xi1, dtype=float)
    xi2 = np.asarray(xi2, dtype=float)
    r = np.asarray(r, dtype=float)
    if np.any(np.abs(xi1) > 1.0) or np.any(np.abs(xi2) > 1.0):
        raise ValueError("panel coordinates must lie in [-1, 1]")
    if np.any(r < 1.0):
        raise ValueError("radius must be >= 1 (shell inner boundary)")
    if depth is not None and np.any(r > 1.0 + depth):
        raise ValueError("radius exceeds the shell outer boundary")
    s = 1.0 / np.sqrt(1.0 + xi1 * xi1 + xi2 * xi2)
    return r * xi1 * s, r * xi2 * s, r * s


@dataclass(frozen=True)
class PanelGrid:
    """nx x ny columns of nz cells (reference ``PanelGrid``,
    geometry.py:87-130, extended with the BASELINE boundary options)."""

    nx: int
    nz: int
    depth: float
    levels: np.ndarray = field(repr=False)
    flat_mode: bool = False
    ny: Optional[int] = None
    periodic: bool = False
    dirichlet_z: bool = False
    omega_shape: Optional[Callable] = field(default=None, repr=False)

    def __post_init__(self):
        if self.ny is None:
            object.__setattr__(self, "ny", self.nx)
        if not (is_power_of_two(self.nx) and is_power_of_two(self.ny)):
            raise ValueError("nx must be a power of two >= 1")
        if self.nz < 1:
            raise ValueError("nz must be at least 1")
        lv = np.asarray(self.levels, dtype=float)
        if lv.shape != (self.nz + 1,):
            raise ValueError("levels must have length nz + 1")
        if np.any(np.diff(lv) <= 0.0):
            raise ValueError("levels must be strictly increasing")
        if lv[0] != 1.0 or lv[-1] != 1.0 + self.depth:
            raise ValueError("levels must run from 1 to 1 + depth exactly")
        if self.ny != self.nx and not self.periodic:
            raise ValueError("rectangular grids are only supported for periodic boxes")
        object.__setattr__(self, "levels", lv)

    @property
    def dxi(self) -> float:
        return 1.0 / self.nx if self.periodic else 2.0 / self.nx

    def xi_edges(self) -> np.ndarray:
        lo = 0.0 if self.periodic else -1.0
        return lo + self.dxi * np.arange(self.nx + 1)

    def xi_centers(self) -> np.ndarray:
        lo = 0.0 if self.periodic else -1.0
        return lo + self.dxi * (np.arange(self.nx) + 0.5)

    def coarsen(self) -> "PanelGrid":
        if self.nx < 2 or self.ny < 2:
            raise ValueError("cannot coarsen a single-column grid")
        return PanelGrid(self.nx // 2, self.nz, self.depth, self.levels, self.flat_mode,
                         self.ny // 2, self.periodic, self.dirichlet_z, self.omega_shape)

    @property
    def dof(self) -> int:
        return self.nx * self.ny * self.nz


def panel_grid(nx: int, nz: int, depth: float = 0.01, flat_mode: bool = False,
               levels: np.ndarray | None = None, **extra) -> PanelGrid:
    """Reference constructor (geometry.py:133-138); ``extra`` takes the
    BASELINE options ``ny``, ``periodic``, ``dirichlet_z``, ``omega_shape``."""
    if levels is None:
        levels = vertical_levels(nz, depth)
    return PanelGrid(nx, nz, depth, np.asarray(levels, dtype=float), flat_mode, **extra)


def periodic_box(nx: int, nz: int, depth: float = 0.01, levels=None, ny=None,
                 omega_shape=None) -> PanelGrid:
    """The BASELINE problem family: doubly periodic unit-spacing box,
    face-Dirichlet top and bottom."""
    if levels is None:
        levels = uniform_levels(nz, depth)
    return PanelGrid(nx, nz, depth, np.asarray(levels, dtype=float), True, ny, True, True,
                     omega_shape)


@dataclass(frozen=True)
class GridFactors:
    """Tensor-product factors (geometry.py:141-174); wx (nx+1, ny), wy
    (nx, ny+1), av/vh/sumw (nx, ny), dr/volprof (nz,), vprof (nz+1,)."""

    wx: np.ndarray
    wy: np.ndarray
    av: np.ndarray
    vh: np.ndarray
    sumw: np.ndarray
    dr: np.ndarray
    vprof: np.ndarray
    volprof: np.ndarray

    @property
    def nx(self) -> int:
        return self.av.shape[0]

    @property
    def ny(self) -> int:
        return self.av.shape[1]

    @property
    def nz(self) -> int:
        return self.dr.shape[0]

    def volumes(self) -> np.ndarray:
        return self.vh[:, :, None] * self.volprof[None, None, :]


def _directions(a, b):
    a, b = np.broadcast_arrays(np.asarray(a, float), np.asarray(b, float))
    s = 1.0 / np.sqrt(1.0 + a * a + b * b)
    return np.stack((a * s, b * s, s), axis=-1)


def _cross_len(p, q):
    c = np.cross(p, q)
    return np.sqrt(np.einsum("...i,...i->...", c, c))


def build_factors(grid: PanelGrid) -> GridFactors:
    nx, ny, nz = grid.nx, grid.ny, grid.nz
    lv = grid.levels
    dr = np.diff(lv)
    vprof = np.zeros(nz + 1)
    if grid.flat_mode or grid.periodic:
        if nz > 1:
            vprof[1:nz] = 2.0 / (lv[2:] - lv[:-2])
        volprof = dr.copy()
    else:
        rc = 0.5 * (lv[:-1] + lv[1:])
        if nz > 1:
            vprof[1:nz] = 2.0 * lv[1:nz] ** 2 / (lv[2:] - lv[:-2])
        volprof = rc ** 2 * dr
    if grid.dirichlet_z:
        # face-Dirichlet u = 0: ghost -u, half-cell distance
        vprof[0] = 2.0 / dr[0]
        vprof[nz] = 2.0 / dr[-1]

    if grid.periodic:
        dxi = grid.dxi
        wx = np.ones((nx + 1, ny))
        wy = np.ones((nx, ny + 1))
        av = np.full((nx, ny), dxi * dxi)
        vh = np.full((nx, ny), dxi * dxi)
        if grid.omega_shape is not None:
            xe = dxi * np.arange(nx + 1)
            xc = dxi * (np.arange(nx) + 0.5)
            ye = dxi * np.arange(ny + 1)
            yc = dxi * (np.arange(ny) + 0.5)
            wx = wx * grid.omega_shape(xe[:, None], yc[None, :])
            wy = wy * grid.omega_shape(xc[:, None], ye[None, :])
            av = av * grid.omega_shape(xc[:, None], yc[None, :])
    elif grid.flat_mode:
        dxi = grid.dxi
        wx = np.ones((nx + 1, nx))
        wx[0, :] = wx[nx, :] = 0.0
        wy = np.ones((nx, nx + 1))
        wy[:, 0] = wy[:, nx] = 0.0
        av = np.full((nx, nx), dxi * dxi)
        vh = np.full((nx, nx), dxi * dxi)
    else:
        xe = grid.xi_edges()
        xc = grid.xi_centers()
        corner = _directions(xe[:, None], xe[None, :])
        centre = _directions(xc[:, None], xc[None, :])
        ex = _directions(xe[:, None], xc[None, :])
        ey = _directions(xc[:, None], xe[None, :])
        wx = np.zeros((nx + 1, nx))
        wx[1:-1, :] = (_cross_len(corner[1:-1, :-1], corner[1:-1, 1:])
                       / np.linalg.norm(centre[1:] - centre[:-1], axis=-1))
        wy = np.zeros((nx, nx + 1))
        wy[:, 1:-1] = (_cross_len(corner[:-1, 1:-1], corner[1:, 1:-1])
                       / np.linalg.norm(centre[:, 1:] - centre[:, :-1], axis=-1))
        av = 0.5 * _cross_len(corner[1:, 1:] - corner[:-1, :-1],
                              corner[:-1, 1:] - corner[1:, :-1])
        vh = np.abs(np.einsum("ijk,ijk->ij",
                              np.cross(ex[1:] - ex[:-1], ey[:, 1:] - ey[:, :-1]), centre))
    sumw = wx[:-1, :] + wx[1:, :] + wy[:, :-1] + wy[:, 1:]
    return GridFactors(wx=wx, wy=wy, av=av, vh=vh, sumw=sumw, dr=dr, vprof=vprof,
                       volprof=volprof)


def omega_shape_config4(x, y):
    """configs[4]: omega^2(x, y) / omega_0^2 = 1 + 0.5 sin(2 pi x) sin(2 pi y)."""
    return 1.0 + 0.5 * np.sin(2.0 * math.pi * x) * np.sin(2.0 * math.pi * y)
