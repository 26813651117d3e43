"""Pin the C oracle (oracle/oracle.c via oracle/coracle.py) against the real
reference's outputs.

oracle.c is the CPU baseline that bench.py times (``cpu_baseline`` and the
``--impl reference`` arm) and the checker of the whole-field full-size GPU
parity tests (tests/test_full_parity.py), so it is pinned here against the
fixtures that running the reference package itself produced
(tests/golden/make_golden.py, SURVEY Appendix B injection):

* per operation (apply, residual, half-sweeps with rho = 1 / 1.4, sweeps,
  SSOR, mean restriction, prolongation, one V-cycle): <= 1e-15 relative;
* solves (configs[0], the 128^2 omega^2 sweep, the configs[4]-like graded /
  variable-omega^2 problem, configs[1] at full size): equal iteration counts,
  histories <= 1e-12 relative, solutions <= 1e-12 (whole field where the
  fixture holds it, else the reference's 256 samples and moments).
"""

import os

import numpy as np
import pytest

from oracle import coracle, port

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def load(name):
    return np.load(os.path.join(GOLD, name + ".npz"))


def uni(shape, seed):
    return np.random.default_rng(seed).uniform(-1.0, 1.0, size=shape)


def rel(a, b):
    return np.max(np.abs(a - b)) / max(1.0, np.max(np.abs(b)))


def hist_rel(h, ref):
    h, ref = np.asarray(h), np.asarray(ref)
    assert h.shape == ref.shape, (h.shape, ref.shape)
    return np.max(np.abs(h - ref) / ref)


def fixture_hier(g):
    nx = int(g["nx"])
    lv = g["levels"]
    periodic = bool(g["periodic"])
    if periodic:
        shape = port.omega_profile_config4 if bool(g["variable"]) else None
        fn = lambda a, b: port.config_factors(a, b, lv, shape)  # noqa: E731
    else:
        fn = lambda a, b: port.flat_neumann_factors(a, lv)  # noqa: E731
    return coracle.Hierarchy(nx, nx, int(g["nlev"]), fn, float(g["omega2"]),
                             float(g["lambda2"]), (periodic, periodic))


#: CG's scalars are global dot products whose summation order is the BLAS
#: ddot's in the reference and an OpenMP reduction here (the
#: reduction order is not pinned by the reference); later residuals are
#: small differences of O(1) terms, so CG histories carry ~1e-12 relative
#: noise.  The reference's own CG tolerance (ops fixtures) is 1e-10.
CG_TOL = 1e-10

OPS = ["ops_periodic", "ops_neumann", "ops_variable", "ops_config"]


@pytest.mark.parametrize("name", OPS)
def test_c_oracle_ops_match_reference(name):
    g = load(name)
    nx, nz = int(g["nx"]), int(g["nz"])
    h = fixture_hier(g)
    ug, fg = uni((nx, nx, nz), 1), uni((nx, nx, nz), 2)
    assert rel(h.apply(ug), g["apply"]) <= 1e-15
    assert rel(h.residual(fg, ug), g["residual"]) <= 1e-15
    for rho in (1.0, 1.4):
        u = ug.copy()
        h.half_sweep(u, fg, port.RED, rho)
        assert rel(u, g[f"half_red_rho{rho}"]) <= 1e-15
        h.half_sweep(u, fg, port.BLACK, rho)
        assert rel(u, g[f"half_black_rho{rho}"]) <= 1e-15
    u = ug.copy()
    h.sweep(u, fg, 2, 1.0)
    assert rel(u, g["sweep2"]) <= 1e-15
    for rho in (1.0, 1.3):
        assert rel(h.ssor(fg, rho), g[f"ssor_rho{rho}"]) <= 1e-15
    assert rel(h.restrict(ug, 0.25), g["restrict_mean"]) <= 1e-15
    assert rel(h.prolong(uni((nx // 2, nx // 2, nz), 3)), g["prolong"]) <= 1e-15
    # one V-cycle from zero (multigrid.py:271-294)
    u1, rep = h.mg_solve(fg, eps=1e-300, max_cycles=1)
    assert rep.iterations == 1
    assert rel(u1, g["vcycle1"]) <= 1e-14


@pytest.mark.parametrize("name", OPS)
def test_c_oracle_solvers_match_reference(name):
    g = load(name)
    nx, nz = int(g["nx"]), int(g["nz"])
    fg = uni((nx, nx, nz), 2)
    h = fixture_hier(g)
    u, rep = h.mg_solve(fg)
    assert hist_rel(rep.residual_history, g["mg_history"]) <= 1e-12
    assert rel(u, g["mg_u"]) <= 1e-12
    u, rep = h.pcg_solve(fg, eps=1e-8, maxiter=200)
    assert hist_rel(rep.residual_history, g["cg_history"]) <= 1e-10
    assert rel(u, g["cg_u"]) <= 1e-10


@pytest.mark.parametrize("solver", ["mg", "cg"])
def test_c_oracle_config0(solver):
    g = load(f"config0_{solver}")
    cfg = port.CONFIGS[0]
    fg = port.rhs(cfg.nx, cfg.ny, cfg.nz, 0)
    h = coracle.config_hierarchy(cfg)
    if solver == "mg":
        u, rep = h.mg_solve(fg)
    else:
        u, rep = h.pcg_solve(fg, eps=1e-5, maxiter=2000)
    assert rep.iterations == int(g["iterations"])
    tol = 1e-12 if solver == "mg" else CG_TOL
    assert hist_rel(rep.residual_history, g["history"]) <= tol
    assert rel(u, g["u"]) <= tol


@pytest.mark.parametrize("w", ["0.0001", "0.001", "0.01", "0.1"])
@pytest.mark.parametrize("solver", ["mg", "cg"])
def test_c_oracle_omega_sweep128(w, solver):
    g = load(f"sweep128_{solver}_w{w}")
    cfg = port.Config(128, 128, 64, 0.01, float(w), 1.0, 4)
    fg = port.rhs(128, 128, 64, 0)
    h = coracle.config_hierarchy(cfg)
    if solver == "mg":
        u, rep = h.mg_solve(fg)
    else:
        u, rep = h.pcg_solve(fg, eps=1e-5, maxiter=2000)
    assert rep.iterations == int(g["iterations"])
    tol = 1e-12 if solver == "mg" else CG_TOL
    assert hist_rel(rep.residual_history, g["history"]) <= tol
    check_samples(u, g, tol)


def check_samples(u, g, tol=1e-12):
    """The reference's 256 sampled values and whole-field moments."""
    idx = g["sample_idx"]
    got = u[idx[:, 0], idx[:, 1], idx[:, 2]]
    amax = float(g["u_absmax"])
    assert np.max(np.abs(got - g["sample_u"])) <= tol * amax
    assert abs(float(np.abs(u).max()) - amax) <= tol * amax
    assert abs(float(u.sum()) - float(g["u_sum"])) <= 1e-9 * amax * u.size ** 0.5
    assert abs(float((u * u).sum()) / float(g["u_sumsq"]) - 1.0) <= 1e-11


@pytest.mark.parametrize("name,nx", [("config4_like_mg", 64), ("config4_like256_mg", 256)])
def test_c_oracle_config4_like(name, nx):
    g = load(name)
    cfg = port.Config(nx, nx, 128, 0.01, 1e-3, 1.0, int(g["nlev"]), stretch=1.05,
                      variable_omega=True)
    h = coracle.config_hierarchy(cfg)
    u, rep = h.mg_solve(port.rhs(nx, nx, 128, 0))
    assert rep.iterations == int(g["iterations"])
    assert hist_rel(rep.residual_history, g["history"]) <= 1e-12
    check_samples(u, g)


def test_c_oracle_config1_full_size():
    """configs[1] at full size (134M unknowns): the reference's 4-cycle history."""
    g = load("config1_mg")
    cfg = port.CONFIGS[1]
    h = coracle.config_hierarchy(cfg)
    u, rep = h.mg_solve(port.rhs(cfg.nx, cfg.ny, cfg.nz, 0))
    assert rep.iterations == int(g["iterations"]) == 4
    assert hist_rel(rep.residual_history, g["history"]) <= 1e-12
    check_samples(u, g)


def test_c_oracle_matches_port_on_rectangular_grid():
    """2:1 periodic grid (the 2 x 1 decomposition's global shape): oracle.c
    against the numpy port, history and whole field."""
    cfg = port.Config(64, 32, 16, 0.01, 1e-3, 1.0, 3)
    f = port.rhs(64, 32, 16, 0)
    uc, rc = coracle.config_hierarchy(cfg).mg_solve(f)
    up, rp = port.mg_solve(cfg.hierarchy(), f)
    assert rc.iterations == rp.iterations
    assert hist_rel(rc.residual_history, rp.residual_history) <= 1e-12
    assert rel(uc, up[1:-1, 1:-1, :]) <= 1e-12


@pytest.mark.parametrize("solver,w", [("cg", "0.001"), ("mg", "0.1")])
def test_c_oracle_config2_full_size(w, solver):
    """configs[2] at full size (1024^2 x 128): one CG and one MG point of the
    omega^2 sweep (the whole sweep is pinned at 128^2 above and compared with
    the GPU at full size in tests/test_full_parity.py)."""
    name = "config1_mg" if (solver, w) == ("mg", "0.001") else f"config2_{solver}_w{w}"
    g = load(name)
    cfg = port.Config(1024, 1024, 128, 0.01, float(w), 1.0, 7)
    h = coracle.config_hierarchy(cfg)
    f = port.rhs(1024, 1024, 128, 0)
    if solver == "mg":
        u, rep = h.mg_solve(f)
    else:
        u, rep = h.pcg_solve(f, eps=1e-5, maxiter=2000)
    assert rep.iterations == int(g["iterations"])
    tol = 1e-12 if solver == "mg" else CG_TOL
    assert hist_rel(rep.residual_history, g["history"]) <= tol
    check_samples(u, g, tol)


def test_c_oracle_matches_live_reference():
    """oracle.c against the reference package itself, run live on a
    256^2 x 128 configs[1]-like problem (5 levels) through
    oracle/refharness.py (baseline/_ref or $PANELMG_SRC; skipped when no
    copy of the reference is present): same cycles, history <= 1e-12 and
    the same solution to the last bit (measured: 0.0 difference)."""
    from oracle import refharness
    if not refharness.available():
        pytest.skip("reference package not installed (baseline/_ref)")
    cfg = port.Config(256, 256, 128, 0.01, 1e-3, 1.0, 5)
    f = port.rhs(256, 256, 128, 0)
    ur, rr = refharness.mg_solve(cfg, f)
    uc, rc = coracle.config_hierarchy(cfg).mg_solve(f)
    assert rc.iterations == rr.iterations
    assert hist_rel(rc.residual_history, rr.residual_history) <= 1e-12
    assert rel(uc, ur) <= 1e-15


@pytest.mark.parametrize("variable", [False, True])
def test_c_oracle_lean_mode_identical(variable):
    """The lean hierarchy (coefficients recomputed per column instead of the
    reference's N-sized caches; used for the 4096^2 configs[4] parity check)
    gives the same bits as the cached one, MG and CG."""
    cfg = port.Config(64, 64, 32, 0.01, 1e-3, 1.0, 4, stretch=1.05 if variable else None,
                      variable_omega=variable)
    f = port.rhs(64, 64, 32, 0)
    for solve in ("mg_solve", "pcg_solve"):
        ua, ra = getattr(coracle.config_hierarchy(cfg), solve)(f)
        ub, rb = getattr(coracle.config_hierarchy(cfg, lean=True), solve)(f)
        assert ra.residual_history == rb.residual_history
        assert np.array_equal(ua, ub)
