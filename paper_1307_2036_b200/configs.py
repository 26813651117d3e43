"""The BASELINE.json problem configurations.

configs[0]  64 x 64 x 32,    MG L=4, omega2=1e-3, lambda2=1   (CPU-runnable)
configs[1]  1024^2 x 128,    MG L=7                           (bench workload)
configs[2]  1024^2 x 128,    CG + line SSOR, omega2 sweep
configs[3]  2048^2 x 128 per GPU, weak scaling (px x py parts)
configs[4]  4096^2 x 128,    graded 1.05, omega2(x, y) = 1e-3 (1 + 0.5 sin sin)

All: doubly periodic unit-spacing box (dx = 1/nx), depth H = 0.01,
face-Dirichlet u = 0 top/bottom, f ~ U[-1, 1] from default_rng(0) in
(i, j, k) C-order, u0 = 0, V(1,1), rho = 1, coarse_sweeps = 1, eps = 1e-5.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .geometry import graded_levels, omega_shape_config4, periodic_box, uniform_levels
from .multigrid import MGConfig
from .params import toy_parameters


@dataclass(frozen=True)
class Problem:
    nx: int
    ny: int
    nz: int
    omega2: float = 1e-3
    lambda2: float = 1.0
    levels: int = 7
    depth: float = 0.01
    stretch: float | None = None
    variable_omega: bool = False

    @property
    def dof(self) -> int:
        return self.nx * self.ny * self.nz

    def grid(self):
        lv = (uniform_levels(self.nz, self.depth) if self.stretch is None
              else graded_levels(self.nz, self.depth, self.stretch))
        return periodic_box(self.nx, self.nz, self.depth, lv, ny=self.ny,
                            omega_shape=omega_shape_config4 if self.variable_omega else None)

    def params(self):
        return toy_parameters(self.nx, self.nz, self.omega2, self.lambda2)

    def mg_config(self, **kw):
        return MGConfig(policy="explicit", explicit_levels=self.levels, eps=1e-5, **kw)


def config(i: int, gpus: int = 1, omega2: float | None = None) -> Problem:
    """BASELINE configs[i]; configs[3] scales the global grid with ``gpus``."""
    w = 1e-3 if omega2 is None else omega2
    if i == 0:
        return Problem(64, 64, 32, w, 1.0, 4)
    if i in (1, 2):
        return Problem(1024, 1024, 128, w, 1.0, 7)
    if i == 3:
        px = {1: 1, 2: 2, 4: 2, 8: 4}[gpus]
        py = gpus // px
        return Problem(2048 * px, 2048 * py, 128, w, 1.0, 8)
    if i == 4:
        return Problem(4096, 4096, 128, w, 1.0, 9, stretch=1.05, variable_omega=True)
    raise ValueError(f"no config {i}")


def rhs(nx: int, ny: int, nz: int, seed: int = 0) -> np.ndarray:
    """f ~ U[-1, 1] from default_rng(seed), (nx, ny, nz) C-order
    (reference bench.py:173-174)."""
    return np.random.default_rng(seed).uniform(-1.0, 1.0, size=(nx, ny, nz))


def rhs_block(nx, ny, nz, i0, j0, mx, my, seed=0) -> np.ndarray:
    """Rows [i0, i0+mx) x [j0, j0+my) of ``rhs`` without the global array
    (PCG64 advanced per row; bit-identical to slicing ``rhs``)."""
    out = np.empty((mx, my, nz))
    for ii in range(mx):
        bg = np.random.PCG64(seed)
        bg.advance(((i0 + ii) * ny + j0) * nz)
        out[ii] = np.random.Generator(bg).uniform(-1.0, 1.0, (my, nz))
    return out
