"""Generate golden fixtures by running the REAL reference package.

Run in the build container (where ``/root/reference`` exists):

    python tests/golden/make_golden.py small      # seconds; per-op + configs[0]
    python tests/golden/make_golden.py big        # ~40 min; configs[1], configs[2]

The reference ``panelmg`` cannot express the BASELINE configs natively
(periodic lateral boundaries, face-Dirichlet top/bottom, hand-set
coefficients), so this script applies the SURVEY Appendix B injection
without editing any reference file:

1. ``panelmg.stencil.build_factors`` is replaced by a factory returning
   the config factors (looked up at call time, ``stencil.py:100``);
2. ``panelmg.partition.LevelLayout.neighbor`` wraps periodically, so
   ``halo_exchange`` (``partition.py:158-191``) becomes periodic.

The "neumann" fixtures run the reference UNMODIFIED (its own flat-mode
factors and mirror halos) to pin the non-periodic path.

Outputs are small ``.npz`` files next to this script.  Inputs are not
stored: they are regenerated from the seeds recorded in each file.
"""

from __future__ import annotations

import math
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF = os.environ.get("PANELMG_SRC", "/root/reference/pkg/src")
sys.path.insert(0, REF)
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import panelmg  # noqa: E402
import panelmg.partition as pt  # noqa: E402
import panelmg.stencil as st  # noqa: E402
from panelmg.geometry import GridFactors  # noqa: E402
from panelmg import (MGConfig, ModelParameters, SSORPreconditioner,  # noqa: E402
                     build_hierarchy, mg_solve, panel_grid, pcg_solve)
from panelmg.multigrid import prolong, restrict, v_cycle  # noqa: E402
from panelmg.partition import (Decomposition, DistField, gather_owned,  # noqa: E402
                               halo_exchange, scatter_owned)
from panelmg.smoother import BLACK, RED, LineSmoother  # noqa: E402

from oracle import port  # noqa: E402  (only for the factor formulas)

_ORIG_BUILD = st.build_factors
_ORIG_NEIGHBOR = pt.LevelLayout.neighbor


def _periodic_neighbor(self, worker, di, dj):
    ai, aj = self.coords(worker)
    return self.worker_at((ai + di) % self.pside, (aj + dj) % self.pside)


def inject(variable_omega=False):
    """Appendix B: config factors + periodic neighbour map."""

    def make_factors(grid):
        shape = port.omega_profile_config4 if variable_omega else None
        fac = port.config_factors(grid.nx, grid.nx, grid.levels, shape)
        return GridFactors(wx=fac.wx, wy=fac.wy, av=fac.av, vh=fac.vh, sumw=fac.sumw,
                           dr=fac.dr, vprof=fac.vprof, volprof=fac.volprof)

    st.build_factors = make_factors
    pt.LevelLayout.neighbor = _periodic_neighbor


def uninject():
    st.build_factors = _ORIG_BUILD
    pt.LevelLayout.neighbor = _ORIG_NEIGHBOR


def params(nx, nz, omega2, lambda2):
    return ModelParameters(nx=nx, nz=nz, dx=1.0 / nx, dt=1.0, omega2=omega2,
                           lambda2=lambda2, courant=1.0)


def uni(shape, seed):
    return np.random.default_rng(seed).uniform(-1.0, 1.0, size=shape)


def ops_fixture(name, nx, nz, omega2, lambda2, levels, periodic, variable=False,
                nlev=3):
    """Per-op goldens on one grid: apply, residual, half sweeps, SSOR,
    transfers, one V-cycle and a full MG solve + CG solve."""
    if periodic:
        inject(variable)
    else:
        uninject()
    try:
        depth = levels[-1] - 1.0
        grid = panel_grid(nx, nz, depth=depth, flat_mode=True, levels=levels)
        prm = params(nx, nz, omega2, lambda2)
        cfg = MGConfig(policy="explicit", explicit_levels=nlev, eps=1e-5)
        hier = build_hierarchy(grid, prm, cfg, Decomposition(nx, 1))
        fine, coarse = hier.levels[0], hier.levels[1]
        op = fine.op
        lay = fine.layout
        ug, fg = uni((nx, nx, nz), 1), uni((nx, nx, nz), 2)

        def field(a):
            d = scatter_owned(a, lay)
            halo_exchange(d)
            return d

        out = {"nx": nx, "nz": nz, "omega2": omega2, "lambda2": lambda2,
               "levels": np.asarray(levels), "periodic": periodic,
               "variable": variable, "nlev": nlev, "seed_u": 1, "seed_f": 2,
               "seed_c": 3}
        u, f = field(ug), field(fg)
        out["apply"] = gather_owned(op.apply(u))
        out["residual"] = gather_owned(op.residual(f, u))
        sm = LineSmoother(op)
        for rho in (1.0, 1.4):
            uu = field(ug)
            sm.half_sweep(uu, f, RED, rho)
            out[f"half_red_rho{rho}"] = gather_owned(uu).copy()
            halo_exchange(uu)
            sm.half_sweep(uu, f, BLACK, rho)
            out[f"half_black_rho{rho}"] = gather_owned(uu).copy()
        uu = field(ug)
        sm.sweep(uu, f, nsweeps=2, rho=1.0)
        out["sweep2"] = gather_owned(uu)
        for rho in (1.0, 1.3):
            out[f"ssor_rho{rho}"] = gather_owned(sm.ssor_apply(f, rho))
        out["restrict_mean"] = gather_owned(restrict(u, fine, coarse))
        cg = uni((nx // 2, nx // 2, nz), 3)
        cd = scatter_owned(cg, coarse.layout)
        halo_exchange(cd)
        out["prolong"] = gather_owned(prolong(cd, coarse, fine))
        # one V-cycle from zero on f
        scratch = hier.make_scratch()
        for w, part in scratch[0].f.parts.items():
            part.data[...] = f.parts[w].data
        v_cycle(hier, cfg, scratch)
        out["vcycle1"] = gather_owned(scratch[0].u)
        # full MG solve
        ud, rep = mg_solve(scatter_owned(fg, lay), hier, cfg)
        out["mg_history"] = np.array(rep.residual_history)
        out["mg_u"] = gather_owned(ud)
        # CG with the line SSOR preconditioner
        pre = SSORPreconditioner(LineSmoother(op))
        uc, rc = pcg_solve(scatter_owned(fg, lay), op, pre, eps=1e-8, maxiter=200)
        out["cg_history"] = np.array(rc.residual_history)
        out["cg_u"] = gather_owned(uc)
        np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)
        print(name, "mg", rep.iterations, "cg", rc.iterations)
    finally:
        uninject()


def config_solve(name, nx, nz, omega2, lambda2, nlev, solver, variable=False,
                 stretch=None, keep_u=False, seed=0):
    """A BASELINE config solve through the injected reference."""
    inject(variable)
    try:
        lv = (port.uniform_levels(nz, 0.01) if stretch is None
              else port.graded_levels(nz, 0.01, stretch))
        grid = panel_grid(nx, nz, depth=0.01, flat_mode=True, levels=lv)
        prm = params(nx, nz, omega2, lambda2)
        fg = np.random.default_rng(seed).uniform(-1.0, 1.0, size=(nx, nx, nz))
        t0 = time.time()
        if solver == "mg":
            cfg = MGConfig(policy="explicit", explicit_levels=nlev, eps=1e-5)
            hier = build_hierarchy(grid, prm, cfg, Decomposition(nx, 1))
            ud, rep = mg_solve(scatter_owned(fg, hier.fine.layout), hier, cfg)
        else:
            op = st.PanelOperator(grid, prm, Decomposition(nx, 1).layout(nx))
            pre = SSORPreconditioner(LineSmoother(op))
            ud, rep = pcg_solve(scatter_owned(fg, op.layout), op, pre, eps=1e-5,
                                maxiter=2000)
        wall = time.time() - t0
        ug = gather_owned(ud)
        rng = np.random.default_rng(12345)
        idx = np.stack([rng.integers(0, nx, 256), rng.integers(0, nx, 256),
                        rng.integers(0, nz, 256)], axis=1)
        out = {"nx": nx, "nz": nz, "omega2": omega2, "lambda2": lambda2,
               "nlev": nlev, "solver": solver, "variable": variable,
               "stretch": -1.0 if stretch is None else stretch, "seed": seed,
               "history": np.array(rep.residual_history),
               "iterations": rep.iterations, "wall_time": rep.wall_time,
               "u_sum": float(ug.sum()), "u_sumsq": float((ug * ug).sum()),
               "u_absmax": float(np.abs(ug).max()),
               "sample_idx": idx, "sample_u": ug[idx[:, 0], idx[:, 1], idx[:, 2]]}
        if keep_u:
            out["u"] = ug
        np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)
        print(name, solver, rep.iterations, rep.residual_history, f"{wall:.1f}s",
              flush=True)
    finally:
        uninject()


def native_fixture(name, nx, nz, dt, flat, policy="standard"):
    """The reference's OWN problem family, unmodified: cubed-sphere panel (or
    its flat box), zero-flux boundaries, graded levels, derived parameters
    (tests/test_partition.py:122-136 setup)."""
    uninject()
    from panelmg import derive_parameters
    grid = panel_grid(nx, nz, flat_mode=flat)
    prm = derive_parameters(nx, nz, dt)
    fg = np.random.default_rng(3).uniform(-1, 1, (nx, nx, nz))
    cfg = MGConfig(policy=policy)
    hier = build_hierarchy(grid, prm, cfg, Decomposition(nx, 1))
    ud, rep = mg_solve(scatter_owned(fg, hier.fine.layout), hier, cfg)
    op = hier.fine.op
    pre = SSORPreconditioner(LineSmoother(op))
    uc, rc = pcg_solve(scatter_owned(fg, op.layout), op, pre, eps=1e-5, maxiter=500)
    u = scatter_owned(np.random.default_rng(4).uniform(-1, 1, (nx, nx, nz)), op.layout)
    halo_exchange(u)
    out = {"nx": nx, "nz": nz, "dt": dt, "flat": flat, "policy": policy,
           "omega2": prm.omega2, "lambda2": prm.lambda2,
           "apply": gather_owned(op.apply(u)),
           "mg_history": np.array(rep.residual_history), "mg_u": gather_owned(ud),
           "cg_history": np.array(rc.residual_history), "cg_u": gather_owned(uc),
           "levels": hier.level_sizes()}
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)
    print(name, "mg", rep.iterations, "cg", rc.iterations)


def thomas_fixture(name):
    """The reference's scalar Thomas solve (tridiag.py:59-100) on seeded
    diagonally dominant systems of the sizes its own test uses
    (tests/test_tridiag.py:33-47), plus a 1e-12-dominant near-singular case."""
    from panelmg import TridiagonalSystem, thomas_solve
    rng = np.random.default_rng(21)
    out = {}
    for n in (1, 2, 3, 64, 128, 257):
        ns = 16
        a = rng.uniform(2.5, 4.0, (ns, n))
        b = rng.uniform(-1.0, 1.0, (ns, n - 1))
        c = rng.uniform(-1.0, 1.0, (ns, n - 1))
        f = rng.uniform(-1.0, 1.0, (ns, n))
        x = np.stack([thomas_solve(TridiagonalSystem(a[s], b[s], c[s], f[s]))
                      for s in range(ns)])
        out.update({f"a{n}": a, f"b{n}": b, f"c{n}": c, f"f{n}": f, f"x{n}": x})
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)
    print(name)


def orderings_fixture(name, nx, nz, omega2, lambda2, levels, periodic):
    """The reference's alternative smoother orderings (smoother.py:193-222)
    and its ``smooth`` dispatcher (smoother.py:247-256) on one grid."""
    from panelmg.smoother import SmootherConfig, smooth
    if periodic:
        inject(False)
    else:
        uninject()
    try:
        grid = panel_grid(nx, nz, depth=levels[-1] - 1.0, flat_mode=True, levels=levels)
        op = st.PanelOperator(grid, params(nx, nz, omega2, lambda2),
                              Decomposition(nx, 1).layout(nx))
        sm = LineSmoother(op)
        ug, fg = uni((nx, nx, nz), 1), uni((nx, nx, nz), 2)

        def field(a):
            d = scatter_owned(a, op.layout)
            halo_exchange(d)
            return d

        f = field(fg)
        out = {"nx": nx, "nz": nz, "omega2": omega2, "lambda2": lambda2,
               "levels": np.asarray(levels), "periodic": periodic, "variable": False,
               "nlev": 1, "seed_u": 1, "seed_f": 2}
        for rho in (1.0, 1.3):
            u = field(ug)
            sm.symmetric_sweep(u, f, nsweeps=2, rho=rho)
            out[f"symmetric_rho{rho}"] = gather_owned(u)
            u = field(ug)
            sm.jacobi_sweep(u, f, nsweeps=2, rho=rho)
            out[f"jacobi_rho{rho}"] = gather_owned(u)
            for ordering in ("redblack", "symmetric", "jacobi"):
                u = field(ug)
                smooth(u, f, sm, SmootherConfig(ordering=ordering, sweeps=3, rho=rho))
                out[f"smooth_{ordering}_rho{rho}"] = gather_owned(u)
        np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)
        print(name)
    finally:
        uninject()


def main(which):
    if which in ("orderings", "small", "all"):
        orderings_fixture("orderings_periodic", 16, 8, 0.7, 1.3,
                          port.uniform_levels(8, 1.0), periodic=True)
        orderings_fixture("orderings_neumann", 16, 8, 0.7, 1.3,
                          port.uniform_levels(8, 1.0), periodic=False)
    if which in ("thomas", "small", "all"):
        thomas_fixture("thomas")
    if which in ("small", "all"):
        # per-op fixtures: periodic config factors, the reference's own
        # Neumann flat factors, and configs[4]-style variable coefficients
        ops_fixture("ops_periodic", 16, 8, 0.7, 1.3,
                    port.uniform_levels(8, 1.0), periodic=True)
        ops_fixture("ops_neumann", 16, 8, 0.7, 1.3,
                    port.uniform_levels(8, 1.0), periodic=False)
        ops_fixture("ops_variable", 16, 16, 1e-3, 1.0,
                    port.graded_levels(16, 0.01, 1.05), periodic=True,
                    variable=True, nlev=3)
        ops_fixture("ops_config", 16, 16, 1e-3, 1.0,
                    port.uniform_levels(16, 0.01), periodic=True, nlev=3)
        config_solve("config0_mg", 64, 32, 1e-3, 1.0, 4, "mg", keep_u=True)
        config_solve("config0_cg", 64, 32, 1e-3, 1.0, 4, "cg", keep_u=True)
        for w in (1e-4, 1e-3, 1e-2, 1e-1):
            config_solve(f"sweep128_cg_w{w:g}", 128, 64, w, 1.0, 4, "cg")
            config_solve(f"sweep128_mg_w{w:g}", 128, 64, w, 1.0, 4, "mg")
        config_solve("config4_like_mg", 64, 128, 1e-3, 1.0, 4, "mg",
                     variable=True, stretch=1.05)
        config_solve("config4_like256_mg", 256, 128, 1e-3, 1.0, 5, "mg",
                     variable=True, stretch=1.05)
    if which in ("native", "small", "all"):
        native_fixture("native_panel32", 32, 8, 4800.0, flat=False)
        native_fixture("native_flat32", 32, 8, 4800.0, flat=True)
        native_fixture("native_panel64_shallow", 64, 16, 2400.0, flat=False, policy="very_shallow")
    if which in ("big", "all"):
        config_solve("config1_mg", 1024, 128, 1e-3, 1.0, 7, "mg")
        for w in (1e-4, 1e-3, 1e-2, 1e-1):
            config_solve(f"config2_cg_w{w:g}", 1024, 128, w, 1.0, 7, "cg")
        for w in (1e-4, 1e-2, 1e-1):
            config_solve(f"config2_mg_w{w:g}", 1024, 128, w, 1.0, 7, "mg")


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "small")
