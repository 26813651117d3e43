"""Pin the CPU oracle (oracle/port.py) against the real reference's outputs.

The fixtures under tests/golden/ were produced by running the reference
package itself (tests/golden/make_golden.py, SURVEY Appendix B injection).
The oracle restates the same numpy expression trees, so most quantities
agree bit for bit; tolerances below are the reference's own
(tests/test_smoother.py:48, test_partition.py:152).
"""

import os

import numpy as np
import pytest

from oracle import port

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def load(name):
    return np.load(os.path.join(GOLD, name + ".npz"))


def uni(shape, seed):
    return np.random.default_rng(seed).uniform(-1.0, 1.0, size=shape)


def fixture_level(g, nx=None):
    nx = int(g["nx"]) if nx is None else nx
    lv = g["levels"]
    periodic = bool(g["periodic"])
    if periodic:
        shape = port.omega_profile_config4 if bool(g["variable"]) else None
        fac = port.config_factors(nx, nx, lv, shape)
    else:
        fac = port.flat_neumann_factors(nx, lv)
    return port.Level(fac, float(g["omega2"]), float(g["lambda2"]),
                      (periodic, periodic))


def fixture_hier(g):
    nx = int(g["nx"])
    lv = g["levels"]
    periodic = bool(g["periodic"])
    if periodic:
        shape = port.omega_profile_config4 if bool(g["variable"]) else None
        fn = lambda a, b: port.config_factors(a, b, lv, shape)  # noqa: E731
    else:
        fn = lambda a, b: port.flat_neumann_factors(a, lv)  # noqa: E731
    return port.Hierarchy(nx, nx, int(g["nlev"]), fn, float(g["omega2"]),
                          float(g["lambda2"]), (periodic, periodic))


OPS = ["ops_periodic", "ops_neumann", "ops_variable", "ops_config"]


def rel(a, b):
    return np.max(np.abs(a - b)) / max(1.0, np.max(np.abs(b)))


@pytest.mark.parametrize("name", OPS)
def test_oracle_ops_match_reference(name):
    g = load(name)
    nx, nz = int(g["nx"]), int(g["nz"])
    lev = fixture_level(g)
    ug, fg = uni((nx, nx, nz), 1), uni((nx, nx, nz), 2)
    u, f = lev.field(ug), lev.field(fg)
    o = lambda d: d[1:-1, 1:-1, :]  # noqa: E731
    assert rel(o(port.apply(lev, u)), g["apply"]) <= 1e-15
    assert rel(o(port.residual(lev, f, u)), g["residual"]) <= 1e-15
    for rho in (1.0, 1.4):
        uu = lev.field(ug)
        port.half_sweep(lev, uu, f, port.RED, rho)
        assert rel(o(uu), g[f"half_red_rho{rho}"]) <= 1e-15
        port.halo_exchange(uu, lev.periodic)
        port.half_sweep(lev, uu, f, port.BLACK, rho)
        assert rel(o(uu), g[f"half_black_rho{rho}"]) <= 1e-15
    uu = lev.field(ug)
    port.sweep(lev, uu, f, 2, 1.0)
    assert rel(o(uu), g["sweep2"]) <= 1e-15
    for rho in (1.0, 1.3):
        assert rel(o(port.ssor_apply(lev, f, rho)), g[f"ssor_rho{rho}"]) <= 1e-15
    h = fixture_hier(g)
    c = h.levels[1]
    cd = c.zeros()
    port.restrict_into(u, cd, 0.25)
    assert rel(o(cd), g["restrict_mean"]) <= 1e-15
    cd = c.field(uni((nx // 2, nx // 2, nz), 3))
    pd = lev.zeros()
    port.prolong_into(cd, pd)
    assert rel(o(pd), g["prolong"]) <= 1e-15
    # one V-cycle from zero
    h.scratch[0][1][...] = f
    port.v_cycle(h)
    assert rel(o(h.scratch[0][0]), g["vcycle1"]) <= 1e-14


@pytest.mark.parametrize("name", OPS)
def test_oracle_solvers_match_reference(name):
    g = load(name)
    nx, nz = int(g["nx"]), int(g["nz"])
    fg = uni((nx, nx, nz), 2)
    h = fixture_hier(g)
    u, rep = port.mg_solve(h, fg)
    ref = g["mg_history"]
    assert len(rep.residual_history) == len(ref)
    assert np.max(np.abs(np.array(rep.residual_history) - ref) / ref) <= 1e-12
    assert rel(u[1:-1, 1:-1, :], g["mg_u"]) <= 1e-12
    lev = fixture_level(g)
    u, rep = port.pcg_solve(lev, fg, eps=1e-8, maxiter=200)
    ref = g["cg_history"]
    assert len(rep.residual_history) == len(ref)
    assert np.max(np.abs(np.array(rep.residual_history) - ref) / ref) <= 1e-10
    assert rel(u[1:-1, 1:-1, :], g["cg_u"]) <= 1e-10


@pytest.mark.parametrize("name,solver", [("config0_mg", "mg"), ("config0_cg", "cg")])
def test_oracle_config0(name, solver):
    g = load(name)
    cfg = port.CONFIGS[0]
    fg = port.rhs(cfg.nx, cfg.ny, cfg.nz, 0)
    if solver == "mg":
        u, rep = port.mg_solve(cfg.hierarchy(), fg)
    else:
        u, rep = port.pcg_solve(cfg.level(), fg, eps=1e-5, maxiter=2000)
    ref = g["history"]
    assert rep.iterations == int(g["iterations"])
    assert np.max(np.abs(np.array(rep.residual_history) - ref) / ref) <= 1e-12
    assert rel(u[1:-1, 1:-1, :], g["u"]) <= 1e-12


def test_rhs_block_matches_global():
    full = port.rhs(16, 8, 4, 0)
    blk = port.rhs_block(16, 8, 4, 4, 2, 8, 4, 0)
    assert np.array_equal(blk, full[4:12, 2:6, :])


@pytest.mark.parametrize("w", ["0.0001", "0.001", "0.01", "0.1"])
@pytest.mark.parametrize("solver", ["mg", "cg"])
def test_oracle_omega_sweep_small(w, solver):
    g = load(f"sweep128_{solver}_w{w}")
    cfg = port.Config(128, 128, 64, 0.01, float(w), 1.0, 4)
    fg = port.rhs(128, 128, 64, 0)
    if solver == "mg":
        _, rep = port.mg_solve(cfg.hierarchy(), fg)
    else:
        _, rep = port.pcg_solve(cfg.level(), fg, eps=1e-5, maxiter=2000)
    ref = g["history"]
    assert rep.iterations == int(g["iterations"])
    assert np.max(np.abs(np.array(rep.residual_history) - ref) / ref) <= 1e-10


def test_oracle_config4_like():
    g = load("config4_like_mg")
    cfg = port.Config(64, 64, 128, 0.01, 1e-3, 1.0, 4, stretch=1.05, variable_omega=True)
    u, rep = port.mg_solve(cfg.hierarchy(), port.rhs(64, 64, 128, 0))
    ref = g["history"]
    assert rep.iterations == int(g["iterations"])
    assert np.max(np.abs(np.array(rep.residual_history) - ref) / ref) <= 1e-12
    idx = g["sample_idx"]
    got = u[1 + idx[:, 0], 1 + idx[:, 1], idx[:, 2]]
    assert np.max(np.abs(got - g["sample_u"])) <= 1e-12 * float(g["u_absmax"])


def test_thomas_known_answers():
    """Known answers of the scalar Thomas algorithm (tests/test_tridiag.py:15-30)
    restated through the oracle's pivot recurrence on one column."""
    fac = port.config_factors(2, 2, port.uniform_levels(3, 1.0))
    lev = port.Level(fac, 0.0, 1.0)   # omega2 = 0: pure mass matrix
    f = lev.field(np.ones((2, 2, 3)))
    u = lev.zeros()
    port.half_sweep(lev, u, f, port.RED)
    # diagonal = vh * volprof = (1/2)^2 * (1/3)
    assert np.allclose(u[1, 1, :], 1.0 / (0.25 / 3.0), rtol=1e-15)


def test_thomas_scalar_matches_reference():
    """oracle thomas_scalar == the reference's thomas_solve (tridiag.py:59-100),
    bit for bit, on the seeded systems of tests/golden/thomas.npz."""
    g = load("thomas")
    for n in (1, 2, 3, 64, 128, 257):
        a, b, c, f, x = (g[f"{k}{n}"] for k in "abcfx")
        for s in range(a.shape[0]):
            assert np.array_equal(port.thomas_scalar(a[s], b[s], c[s], f[s]), x[s]), (n, s)
    with pytest.raises(ArithmeticError):
        port.thomas_scalar(np.array([1.0, 1.0]), np.array([1.0]), np.array([1.0]),
                           np.array([1.0, 1.0]))


@pytest.mark.parametrize("name", ["orderings_periodic", "orderings_neumann"])
def test_oracle_orderings_match_reference(name):
    """Symmetric and block-Jacobi orderings (smoother.py:193-222) and the
    smooth() dispatcher (smoother.py:247-256) of the oracle vs the reference."""
    g = load(name)
    nx, nz = int(g["nx"]), int(g["nz"])
    lev = fixture_level(g)
    ug, fg = uni((nx, nx, nz), 1), uni((nx, nx, nz), 2)
    f = lev.field(fg)
    o = lambda d: d[1:-1, 1:-1, :]  # noqa: E731
    for rho in (1.0, 1.3):
        u = lev.field(ug)
        port.symmetric_sweep(lev, u, f, 2, rho)
        assert rel(o(u), g[f"symmetric_rho{rho}"]) <= 1e-15
        u = lev.field(ug)
        port.jacobi_sweep(lev, u, f, 2, rho)
        assert rel(o(u), g[f"jacobi_rho{rho}"]) <= 1e-15
        for ordering, fn in (("redblack", port.sweep), ("symmetric", port.symmetric_sweep),
                             ("jacobi", port.jacobi_sweep)):
            u = lev.field(ug)
            fn(lev, u, f, 3, rho)
            assert rel(o(u), g[f"smooth_{ordering}_rho{rho}"]) <= 1e-15
