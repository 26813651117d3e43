"""Device line solves and the remaining reference behaviours (needs a B200):

* ``thomas_solve`` / ``thomas_solve_batch`` (pmg_thomas_batch) against the
  reference's scalar Thomas solves (tests/golden/thomas.npz, bit for bit),
  its known answers (tests/test_tridiag.py:15-30), 1000 random dominant
  systems against dense elimination (tests/test_tridiag.py:33-47, 1e-12),
  and its zero-pivot detection (tests/test_tridiag.py:68-77);
* the symmetric and block-Jacobi orderings and ``smooth`` against the
  reference (tests/golden/orderings_*.npz): bit-identical in exact smoother
  mode, the reference's 1e-12 half-sweep tolerance in fast mode;
* ``BreakdownError`` raised by device solves on an indefinite operator:
  the reference's ``_Negated`` double (tests/test_krylov.py:60-82) through
  the Python driver, and a negative-mass level through the native
  ``pmg_pcg_solve`` (krylov.py:131-156).
"""

import ctypes as C
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def pmg():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1307_2036_b200 as m
    return m


def load(name):
    return np.load(os.path.join(GOLD, name + ".npz"))


def test_thomas_known_answers(pmg):
    S = pmg.TridiagonalSystem
    x = pmg.thomas_solve(S(np.ones(3), np.zeros(2), np.zeros(2), np.array([3.0, 1.0, 4.0])))
    assert np.array_equal(x, [3.0, 1.0, 4.0])
    x = pmg.thomas_solve(S(np.array([2.0, 2.0]), np.array([1.0]), np.array([1.0]),
                           np.array([3.0, 3.0])))
    assert np.allclose(x, [1.0, 1.0], rtol=0, atol=1e-15)
    x = pmg.thomas_solve(S(np.array([4.0]), np.zeros(0), np.zeros(0), np.array([2.0])))
    assert x[0] == 0.5


def test_thomas_bitwise_vs_reference(pmg):
    """One batch per size: every system's solution equals the reference's
    scalar solve bit for bit (same operation order, no FMA contraction)."""
    g = load("thomas")
    for n in (1, 2, 3, 64, 128, 257):
        a, b, c, f, x = (g[f"{k}{n}"] for k in "abcfx")
        got = pmg.thomas_solve_batch(a, b, c, f)
        assert np.array_equal(got, x), n
        # the one-system API agrees with the batch
        s = pmg.TridiagonalSystem(a[0], b[0], c[0], f[0])
        assert np.array_equal(pmg.thomas_solve(s), x[0])


def test_thomas_dense_and_linearity(pmg):
    rng = np.random.default_rng(11)
    for n in (1, 2, 3, 64, 128, 257):
        ns = 167
        a = rng.uniform(2.5, 4.0, (ns, n))
        b = rng.uniform(-1.0, 1.0, (ns, n - 1))
        c = rng.uniform(-1.0, 1.0, (ns, n - 1))
        f = rng.uniform(-1.0, 1.0, (ns, n))
        g2 = rng.uniform(-1.0, 1.0, (ns, n))
        x = pmg.thomas_solve_batch(a, b, c, f)
        y = pmg.thomas_solve_batch(a, b, c, 1.7 * f - 0.3 * g2)
        xg = pmg.thomas_solve_batch(a, b, c, g2)
        for s in range(0, ns, 7):
            dense = np.diag(a[s])
            if n > 1:
                dense += np.diag(b[s], 1) + np.diag(c[s], -1)
            ref = np.linalg.solve(dense, f[s])
            assert np.max(np.abs(x[s] - ref)) <= 1e-12 * max(1.0, np.max(np.abs(ref)))
        assert np.max(np.abs(y - (1.7 * x - 0.3 * xg))) <= 1e-12 * np.max(np.abs(y))


def test_thomas_zero_pivot(pmg):
    S = pmg.TridiagonalSystem
    with pytest.raises(pmg.ZeroPivotError, match="row 0"):
        pmg.thomas_solve(S(np.array([0.0]), np.zeros(0), np.zeros(0), np.array([1.0])))
    with pytest.raises(pmg.ZeroPivotError, match="row 1"):
        pmg.thomas_solve(S(np.array([1.0, 1.0]), np.array([1.0]), np.array([1.0]),
                           np.array([1.0, 1.0])))
    # in a batch the first failing row over all systems is reported
    # system 1: pivots 1, 2 - 1 * 1 = 1, then 2 - 1 * 2 = 0 at row 2
    a = np.array([[2.0, 2.0, 2.0], [1.0, 2.0, 2.0]])
    b = np.array([[1.0, 1.0], [1.0, 1.0]])
    c = np.array([[1.0, 1.0], [1.0, 2.0]])
    with pytest.raises(pmg.ZeroPivotError, match="row 2"):
        pmg.thomas_solve_batch(a, b, c, np.ones((2, 3)))


@pytest.mark.parametrize("exact", [True, False])
@pytest.mark.parametrize("name", ["orderings_periodic", "orderings_neumann"])
def test_orderings_vs_reference(pmg, name, exact):
    g = load(name)
    nx, nz = int(g["nx"]), int(g["nz"])
    lv = g["levels"]
    if bool(g["periodic"]):
        grid = pmg.periodic_box(nx, nz, float(lv[-1] - 1.0), lv)
    else:
        grid = pmg.panel_grid(nx, nz, depth=float(lv[-1] - 1.0), flat_mode=True, levels=lv)
    params = pmg.toy_parameters(nx, nz, float(g["omega2"]), float(g["lambda2"]))
    tol = 0.0 if exact else 1e-12
    rng1 = np.random.default_rng(1).uniform(-1, 1, (nx, nx, nz))
    rng2 = np.random.default_rng(2).uniform(-1, 1, (nx, nx, nz))
    for workers in (1, 4):
        op = pmg.PanelOperator(grid, params, pmg.Decomposition(nx, workers).layout(nx))
        sm = pmg.LineSmoother(op)

        def field(a):
            d = pmg.scatter_owned(a, op.layout)
            pmg.halo_exchange(d)
            return d

        def close(u, key):
            got, ref = pmg.gather_owned(u), g[key]
            if tol == 0.0:
                return np.array_equal(got, ref)
            return np.max(np.abs(got - ref)) <= tol * max(1.0, np.max(np.abs(ref)))

        f = field(rng2)
        with pmg.exact_smoother(exact):
            for rho in (1.0, 1.3):
                u = field(rng1)
                sm.symmetric_sweep(u, f, nsweeps=2, rho=rho)
                assert close(u, f"symmetric_rho{rho}"), (workers, rho)
                u = field(rng1)
                sm.jacobi_sweep(u, f, nsweeps=2, rho=rho)
                assert close(u, f"jacobi_rho{rho}"), (workers, rho)
                for ordering in ("redblack", "symmetric", "jacobi"):
                    u = field(rng1)
                    cfg = pmg.SmootherConfig(ordering=ordering, sweeps=3, rho=rho)
                    pmg.smooth(u, f, sm, cfg)
                    assert close(u, f"smooth_{ordering}_rho{rho}"), (workers, ordering, rho)


class _Negated:
    """Sign-flipped operator (the reference's test double,
    tests/test_krylov.py:60-75): layout, nz, apply, residual."""

    def __init__(self, op):
        self._op = op
        self.layout = op.layout
        self.nz = op.nz

    def apply(self, u, out=None):
        out = self._op.apply(u, out)
        for part in out.parts.values():
            part.data.neg_()
        return out

    def residual(self, f, u, out=None):
        raise NotImplementedError


@pytest.mark.parametrize("workers", [1, 4])
def test_breakdown_negated_operator(pmg, workers):
    grid = pmg.periodic_box(16, 8, 0.01)
    params = pmg.toy_parameters(16, 8, 1e-3, 1.0)
    op = pmg.PanelOperator(grid, params, pmg.Decomposition(16, workers).layout(16))
    f = pmg.scatter_owned(np.random.default_rng(3).uniform(-1, 1, (16, 16, 8)), op.layout)
    with pytest.raises(pmg.BreakdownError, match="A p"):
        pmg.pcg_solve(f, _Negated(op), None, eps=1e-6, maxiter=10)
    # with the (positive definite) line SSOR of the true operator the
    # first <p, A p> is still negative
    pre = pmg.SSORPreconditioner(pmg.LineSmoother(op))
    with pytest.raises(pmg.BreakdownError):
        pmg.pcg_solve(f, _Negated(op), pre, eps=1e-6, maxiter=10)


@pytest.mark.parametrize("precond", [0, 1])
def test_breakdown_native_negative_mass(pmg, precond):
    """A level whose mass term vh * volprof is negative and dominant makes A
    (and the line SSOR built from it) negative definite: the native CG
    driver returns PMG_ERR_BREAKDOWN before updating the iterate
    (krylov.py:131-132, 141-142), which the wrapper maps to BreakdownError."""
    from paper_1307_2036_b200 import _lib
    from paper_1307_2036_b200.partition import DevField, LevelHandle
    lib = _lib.load()
    n, nz = 16, 8
    dz = np.full(nz, 0.01 / nz)
    vprof = np.empty(nz + 1)
    vprof[1:nz] = 1.0 / dz[:-1]
    vprof[0], vprof[nz] = 2.0 / dz[0], 2.0 / dz[-1]
    one = np.ones(1)
    h = LevelHandle(n, n, nz, 0, 0, 1e-3, 1e-3, dz, vprof, -1e5 * dz,
                    np.broadcast_to(one, (n, n + 1)), np.broadcast_to(one, (n + 1, n)),
                    np.broadcast_to(one / n**2, (n, n)), np.broadcast_to(one / n**2, (n, n)),
                    np.broadcast_to(4 * one, (n, n)))
    f = DevField(h)
    src = torch.from_numpy(np.random.default_rng(5).uniform(-1, 1, (n, n, nz))).cuda()
    st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    _lib.call("pmg_from_ref_layout", h.h, C.c_void_p(src.data_ptr()), f.ptr, st)
    u = DevField(h)
    work = torch.empty(int(lib.pmg_pcg_work_doubles(h.h)), dtype=torch.float64, device="cuda")
    hist = np.zeros(11)
    iters, conv = C.c_int(), C.c_int()
    rc = lib.pmg_pcg_solve(h.h, f.ptr, u.ptr, 1e-6, 10, 1e-300, precond, 1.0, 1, 1,
                           C.c_void_p(work.data_ptr()), hist.ctypes.data_as(C.c_void_p),
                           C.byref(iters), C.byref(conv), st)
    assert rc == _lib.PMG_ERR_BREAKDOWN
    with pytest.raises(pmg.BreakdownError):
        _lib.check(rc, "pmg_pcg_solve")
    # detected before any iterate update: no iteration is reported
    assert iters.value == 0 and conv.value == 0
