"""Matrix-free 7-point operator on the device (reference ``stencil.py``).

``PanelOperator`` keeps the reference's constructor, attributes and
``apply`` / ``residual`` semantics (``stencil.py:87-165``).  The
coefficients are not cached as N-sized arrays: each part gets one
``pmg_level`` holding the 1-D diagonal / band / pivot tables when the
2-D factors are constant (BASELINE configs[0-3]) or the 2-D factor
arrays otherwise (``PAPER.md:509``: recalculated whenever used).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from ._lib import call
from .geometry import GridFactors, PanelGrid, build_factors
from .params import ModelParameters
from .partition import (Decomposition, DistField, LevelHandle, LevelLayout, _ptr,
                        _Scratch, _stream, reduce_parts)


@dataclass(frozen=True)
class VerticalBlock:
    """Tridiagonal restriction of the operator to one column (stencil.py:47-58)."""

    sub: np.ndarray
    diag: np.ndarray
    sup: np.ndarray


def _part_factors(f: GridFactors, i0, j0, mx, my):
    """Owned-window slices of the global factors, transposed to [j][i]."""
    wx = f.wx[i0:i0 + mx + 1, j0:j0 + my].T
    wy = f.wy[i0:i0 + mx, j0:j0 + my + 1].T
    av = f.av[i0:i0 + mx, j0:j0 + my].T
    vh = f.vh[i0:i0 + mx, j0:j0 + my].T
    sw = f.sumw[i0:i0 + mx, j0:j0 + my].T
    return wx, wy, av, vh, sw


class PanelOperator:
    """The model operator bound to one grid level and one layout."""

    def __init__(self, grid: PanelGrid, params: ModelParameters,
                 layout: LevelLayout | None = None, factors: GridFactors | None = None):
        if layout is None:
            layout = Decomposition(grid.nx, 1, ny=grid.ny,
                                   periodic=grid.periodic).layout(grid.nx)
        if layout.nx != grid.nx or layout.ny != grid.ny:
            raise ValueError("layout does not match the grid size")
        layout.decomp.bind_periodic(grid.periodic)
        self.grid = grid
        self.params = params
        self.layout = layout
        self.factors = factors if factors is not None else build_factors(grid)
        self.omega2 = params.omega2
        self.vcoef = params.omega2 * params.lambda2
        f = self.factors
        self.handles = {}
        for w in layout.local_workers:
            i0, j0 = layout.origin(w)
            wx, wy, av, vh, sw = _part_factors(f, i0, j0, layout.mx, layout.my)
            self.handles[w] = LevelHandle(layout.mx, layout.my, grid.nz, i0, j0, self.omega2,
                                          self.vcoef, f.dr, f.vprof, f.volprof, wx, wy, av, vh,
                                          sw)

    @property
    def nz(self) -> int:
        return self.grid.nz

    @property
    def self_coupled(self) -> bool:
        """A periodic grid one column wide: every cell is its own neighbour
        through the wrap, so the red-black identities the fused paths rest
        on (a half-sweep never reads its own colour) do not hold."""
        return bool(self.grid.periodic) and (self.grid.nx == 1 or self.grid.ny == 1)

    @property
    def uniform(self) -> bool:
        return all(h.uniform for h in self.handles.values())

    def _check(self, u: DistField) -> None:
        if u.layout is not self.layout and (u.layout.nx != self.layout.nx
                                            or u.layout.ny != self.layout.ny
                                            or u.layout.px != self.layout.px
                                            or u.layout.py != self.layout.py):
            raise ValueError("field layout does not match the operator layout")
        if u.nz != self.grid.nz:
            raise ValueError("field vertical size does not match the grid")

    def apply(self, u: DistField, out: DistField | None = None) -> DistField:
        """v = A u over owned cells (u halos must be current)."""
        self._check(u)
        if out is None:
            out = DistField.zeros(self.layout, self.nz)
        st = _stream()
        for w, uf in u.parts.items():
            call("pmg_apply", self.handles[w].h, uf.ptr, out.parts[w].ptr, st)
        return out

    def residual(self, f: DistField, u: DistField, out: DistField | None = None) -> DistField:
        """r = f - A u over owned cells."""
        self._check(u)
        if out is None:
            out = DistField.zeros(self.layout, self.nz)
        st = _stream()
        for w, uf in u.parts.items():
            call("pmg_residual", self.handles[w].h, f.parts[w].ptr, uf.ptr, out.parts[w].ptr,
                 None, None, st)
        return out

    def residual_norm2_dev(self, f: DistField, u: DistField, out: DistField | None,
                           res: torch.Tensor) -> None:
        """||f - A u||^2 per part into res[part index] (device), optionally
        storing r; no host synchronisation."""
        scratch, _ = _Scratch.get()
        st = _stream()
        for n, (w, uf) in enumerate(u.parts.items()):
            call("pmg_residual", self.handles[w].h, f.parts[w].ptr, uf.ptr,
                 None if out is None else out.parts[w].ptr, _ptr(scratch),
                 C.c_void_p(res.data_ptr() + 8 * n), st)

    def residual_norm(self, f: DistField, u: DistField, out: DistField | None = None) -> float:
        from .partition import scalar_buffer
        res = scalar_buffer(len(u.parts))
        self.residual_norm2_dev(f, u, out, res)
        return float(np.sqrt(reduce_parts(res)))

    def apply_dot_dev(self, p: DistField, q: DistField, res: torch.Tensor) -> None:
        """q = A p and p.q per part into res (device)."""
        scratch, _ = _Scratch.get()
        st = _stream()
        for n, (w, pf) in enumerate(p.parts.items()):
            call("pmg_apply_dot", self.handles[w].h, pf.ptr, q.parts[w].ptr, _ptr(scratch),
                 C.c_void_p(res.data_ptr() + 8 * n), st)

    def assemble(self):
        """Explicit sparse host matrix equal to the matrix-free operator
        (stencil.py:182-232): a testing oracle for small grids only, refused
        above ``ORACLE_CELL_CAP`` cells."""
        n = self.grid.nx * self.grid.ny * self.grid.nz
        if n > ORACLE_CELL_CAP:
            raise ValueError(f"assembled-matrix oracle capped at {ORACLE_CELL_CAP} cells, "
                             f"got {n}")
        return _assemble_rows(self)

    def column_block(self, i: int, j: int) -> VerticalBlock:
        """Tridiagonal block of column (i, j) in global indices (stencil.py:167-180)."""
        nx, ny, nz = self.grid.nx, self.grid.ny, self.grid.nz
        if not (0 <= i < nx and 0 <= j < ny):
            raise ValueError("column index out of range")
        f = self.factors
        diag = (f.vh[i, j] * f.volprof + self.omega2 * f.sumw[i, j] * f.dr
                + self.vcoef * f.av[i, j] * (f.vprof[:-1] + f.vprof[1:]))
        sub = np.zeros(nz)
        sup = np.zeros(nz)
        if nz > 1:
            coup = -self.vcoef * f.av[i, j] * f.vprof[1:nz]
            sub[1:] = coup
            sup[:-1] = coup
        return VerticalBlock(sub=sub, diag=diag, sup=sup)


def _assemble_rows(op: "PanelOperator"):
    """Host CSR matrix with the rows of the matrix-free operator: every
    cell's diagonal and its (up to) six couplings taken from the cell's own
    face weights, exactly the terms ``apply`` subtracts -- W/E faces
    wx[i], wx[i+1], S/N faces wy[j], wy[j+1] (wrapping on a periodic grid,
    zero-weight boundary faces dropped) and the vertical faces vprof[k],
    vprof[k+1].  Unknowns are numbered nz * (ny * i + j) + k."""
    import scipy.sparse as sp

    g, f = op.grid, op.factors
    nx, ny, nz = g.nx, g.ny, g.nz
    n = nx * ny * nz
    I, J, K = np.meshgrid(np.arange(nx), np.arange(ny), np.arange(nz), indexing="ij")
    row = (nz * (ny * I + J) + K).ravel()
    diag = (f.vh[:, :, None] * f.volprof[None, None, :]
            + op.omega2 * f.sumw[:, :, None] * f.dr[None, None, :]
            + op.vcoef * f.av[:, :, None] * (f.vprof[:-1] + f.vprof[1:])[None, None, :])
    rows, cols, vals = [row], [row], [diag.ravel()]

    def couple(weight, di, dj, dk):
        """One neighbour direction: column ids of the neighbour cells and
        -weight, for the cells that have that neighbour."""
        ii, jj, kk = I + di, J + dj, K + dk
        if g.periodic:
            ii, jj = ii % nx, jj % ny
        ok = ((ii >= 0) & (ii < nx) & (jj >= 0) & (jj < ny) & (kk >= 0) & (kk < nz)
              & (weight != 0.0)).ravel()
        rows.append(row[ok])
        cols.append((nz * (ny * ii + jj) + kk).ravel()[ok])
        vals.append(-weight.ravel()[ok])

    drw = op.omega2 * f.dr[None, None, :]
    one = np.ones((nx, ny, nz))
    couple(f.wx[:-1, :, None] * drw, -1, 0, 0)
    couple(f.wx[1:, :, None] * drw, +1, 0, 0)
    couple(f.wy[:, :-1, None] * drw, 0, -1, 0)
    couple(f.wy[:, 1:, None] * drw, 0, +1, 0)
    vert = op.vcoef * f.av[:, :, None] * one
    couple(vert * f.vprof[None, None, :-1], 0, 0, -1)
    couple(vert * f.vprof[None, None, 1:], 0, 0, +1)
    a = sp.coo_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                      shape=(n, n))
    return a.tocsr()


#: largest grid (cells) ``assemble`` accepts (stencil.py:43)
ORACLE_CELL_CAP = 100_000


def assemble_matrix(grid: PanelGrid, params: ModelParameters):
    """Sparse host matrix of the operator on a small grid (stencil.py:260-262):
    the reference's testing oracle, kept for the same purpose -- no solver
    path uses it."""
    return PanelOperator(grid, params).assemble()


def apply_operator(u, grid: PanelGrid, params: ModelParameters):
    """Single-part convenience wrapper (stencil.py:243-248): u is a global
    (nx, ny, nz) array; returns A u as a host array."""
    from .partition import gather_owned, halo_exchange, scatter_owned
    op = PanelOperator(grid, params)
    du = scatter_owned(np.asarray(u, dtype=float), op.layout)
    halo_exchange(du)
    return gather_owned(op.apply(du))


def compute_residual(f, u, grid: PanelGrid, params: ModelParameters):
    from .partition import gather_owned, halo_exchange, scatter_owned
    op = PanelOperator(grid, params)
    du = scatter_owned(np.asarray(u, dtype=float), op.layout)
    halo_exchange(du)
    df = scatter_owned(np.asarray(f, dtype=float), op.layout)
    return gather_owned(op.residual(df, du))


def vertical_blocks(grid: PanelGrid, params: ModelParameters):
    return PanelOperator(grid, params).column_block
