"""Run the REAL reference package (panelmg) on a BASELINE config.

TEST INFRASTRUCTURE / CPU BASELINE ONLY -- the product never imports this.

The reference cannot express the BASELINE configs natively (periodic
lateral boundaries, hand-set coefficients), so SURVEY Appendix B's
injection is applied at import time without editing any reference file
(the same recipe as tests/golden/make_golden.py):

1. ``panelmg.stencil.build_factors`` -> the config factors (looked up at
   call time, reference ``stencil.py:100``);
2. ``panelmg.partition.LevelLayout.neighbor`` wraps periodically, so
   ``halo_exchange`` (``partition.py:158-191``) is periodic.

Where the reference comes from: ``baseline/_ref`` (the offline
``pip install --target baseline/_ref`` of the reference package; it travels
to the GPU box with the repo snapshot), else ``$PANELMG_SRC``.  bench.py's
``cpu_baseline`` leg times ``mg_solve`` through it (SolveReport.wall_time:
the iteration loop only, reference ``multigrid.py:321-329``).
"""

from __future__ import annotations

import os
import sys

import numpy as np

from . import port

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _import_panelmg():
    for cand in (os.path.join(ROOT, "baseline", "_ref"), os.environ.get("PANELMG_SRC")):
        if cand and os.path.isdir(os.path.join(cand, "panelmg")):
            if cand not in sys.path:
                sys.path.insert(0, cand)
            break
    import panelmg  # noqa: F401  (ImportError when no copy is available)
    return panelmg


def available() -> bool:
    try:
        _import_panelmg()
        return True
    except ImportError:
        return False


def _inject(variable_omega: bool):
    _import_panelmg()
    import panelmg.partition as pt
    import panelmg.stencil as st
    from panelmg.geometry import GridFactors

    def make_factors(grid):
        shape = port.omega_profile_config4 if variable_omega else None
        fac = port.config_factors(grid.nx, grid.nx, grid.levels, shape)
        return GridFactors(wx=fac.wx, wy=fac.wy, av=fac.av, vh=fac.vh, sumw=fac.sumw,
                           dr=fac.dr, vprof=fac.vprof, volprof=fac.volprof)

    def periodic_neighbor(self, worker, di, dj):
        ai, aj = self.coords(worker)
        return self.worker_at((ai + di) % self.pside, (aj + dj) % self.pside)

    st.build_factors = make_factors
    pt.LevelLayout.neighbor = periodic_neighbor


def mg_solve(cfg: "port.Config", f: np.ndarray | None = None, seed: int = 0):
    """Reference ``mg_solve`` (multigrid.py:297-330) on ``cfg`` (square grids)
    with f = U[-1, 1] from default_rng(seed); returns (u_owned, SolveReport)."""
    if cfg.nx != cfg.ny:
        raise ValueError("the reference's panel grids are square")
    _inject(cfg.variable_omega)
    from panelmg import MGConfig, ModelParameters, build_hierarchy, panel_grid
    from panelmg import mg_solve as ref_mg_solve
    from panelmg.partition import Decomposition, gather_owned, scatter_owned

    levels = cfg.level_radii()
    grid = panel_grid(cfg.nx, cfg.nz, depth=cfg.depth, flat_mode=True, levels=levels)
    prm = ModelParameters(nx=cfg.nx, nz=cfg.nz, dx=1.0 / cfg.nx, dt=1.0, omega2=cfg.omega2,
                          lambda2=cfg.lambda2, courant=1.0)
    mcfg = MGConfig(policy="explicit", explicit_levels=cfg.levels, eps=1e-5)
    hier = build_hierarchy(grid, prm, mcfg, Decomposition(cfg.nx, 1))
    if f is None:
        f = port.rhs(cfg.nx, cfg.ny, cfg.nz, seed)
    fd = scatter_owned(f, hier.levels[0].layout)
    u, rep = ref_mg_solve(fd, hier, mcfg)
    return gather_owned(u), rep
