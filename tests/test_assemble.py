"""Host-side assembled-matrix oracle (``stencil._assemble_rows``, the
reference's ``PanelOperator.assemble``, stencil.py:182-232) against a
cell-by-cell loop restatement of the 7-point finite-volume stencil; no GPU."""

import types

import numpy as np
import pytest

import paper_1307_2036_b200 as pmg
from paper_1307_2036_b200.stencil import _assemble_rows


def fake_op(grid, omega2, lambda2):
    """What _assemble_rows reads of a PanelOperator (no device handle)."""
    return types.SimpleNamespace(grid=grid, factors=pmg.build_factors(grid), omega2=omega2,
                                 vcoef=omega2 * lambda2)


def loop_matrix(op):
    g, f = op.grid, op.factors
    nx, ny, nz = g.nx, g.ny, g.nz
    a = np.zeros((nx * ny * nz,) * 2)

    def cid(i, j, k):
        return nz * (ny * i + j) + k

    for i in range(nx):
        for j in range(ny):
            for k in range(nz):
                r = cid(i, j, k)
                a[r, r] = (f.vh[i, j] * f.volprof[k] + op.omega2 * f.sumw[i, j] * f.dr[k]
                           + op.vcoef * f.av[i, j] * (f.vprof[k] + f.vprof[k + 1]))
                for w, ii, jj in ((f.wx[i, j], i - 1, j), (f.wx[i + 1, j], i + 1, j),
                                  (f.wy[i, j], i, j - 1), (f.wy[i, j + 1], i, j + 1)):
                    if g.periodic:
                        ii, jj = ii % nx, jj % ny
                    if 0 <= ii < nx and 0 <= jj < ny and w != 0.0:
                        a[r, cid(ii, jj, k)] += -w * (op.omega2 * f.dr[k])
                if k > 0:
                    a[r, cid(i, j, k - 1)] = -op.vcoef * f.av[i, j] * f.vprof[k]
                if k + 1 < nz:
                    a[r, cid(i, j, k + 1)] = -op.vcoef * f.av[i, j] * f.vprof[k + 1]
    return a


GRIDS = {
    "flat": lambda: pmg.panel_grid(4, 3, depth=1.0, flat_mode=True),
    "curved": lambda: pmg.panel_grid(4, 3, depth=0.01),
    "periodic": lambda: pmg.periodic_box(4, 3, 0.01),
    "periodic_rect": lambda: pmg.periodic_box(4, 3, 0.01, ny=8),
    "variable": lambda: pmg.periodic_box(4, 3, 0.01, pmg.graded_levels(3, 0.01, 1.05),
                                         omega_shape=pmg.geometry.omega_shape_config4),
}


@pytest.mark.parametrize("kind", sorted(GRIDS))
def test_rows_equal_loop_stencil(kind):
    op = fake_op(GRIDS[kind](), 0.7, 1.3)
    a = _assemble_rows(op)
    ref = loop_matrix(op)
    assert a.shape == ref.shape
    assert np.array_equal(a.toarray(), ref)
    assert np.diff(a.indptr).max() <= 7
    if kind != "variable":
        assert abs(a - a.T).max() == 0.0
    w = np.linalg.eigvalsh(0.5 * (ref + ref.T))
    assert w.min() > 0.0


def test_row_sums_and_wrap():
    # closed (no-flux) boundaries: rows sum to the cell volume (mass term)
    op = fake_op(GRIDS["curved"](), 0.7, 1.3)
    a = _assemble_rows(op)
    assert np.allclose(np.asarray(a.sum(axis=1)).ravel(), op.factors.volumes().ravel(),
                       rtol=1e-12)
    # periodic: cell (0, j) couples to (nx - 1, j)
    op = fake_op(GRIDS["periodic"](), 0.7, 1.3)
    a = _assemble_rows(op).toarray()
    nz, ny, nx = 3, 4, 4
    assert a[nz * (ny * 0 + 1) + 2, nz * (ny * (nx - 1) + 1) + 2] < 0.0
    # Dirichlet faces add to the diagonal only
    assert np.all(np.asarray(a.sum(axis=1)).ravel() > 0.0)


def test_size_cap_constant():
    assert pmg.ORACLE_CELL_CAP == 100_000
