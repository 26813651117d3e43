"""Device path against first principles (needs a B200).

The golden / oracle parity tests pin the CUDA path to the reference's
outputs; this file pins it to the mathematics instead, the way the
reference's own unit tests do (tests/test_stencil.py, test_smoother.py,
test_krylov.py, test_multigrid.py): the operator is assembled as an
explicit sparse matrix on the host (``PanelOperator.assemble``, the
reference's testing oracle, stencil.py:182-232) and every device kernel is
compared with what linear algebra says it must compute --

* apply / residual == A u, f - A u (flat, curved, periodic, variable omega^2);
* A symmetric positive definite, at most seven entries per row, column
  blocks equal to the matrix's tridiagonal column restrictions;
* a half sweep == one block Gauss-Seidel update of that colour's columns
  on the assembled matrix, any rho; the exact solution is a fixed point;
  the energy norm of the error never grows;
* SSOR == rho (2 - rho) (D + rho U)^-1 D (D + rho L)^-1 in the red-first
  block ordering, a symmetric positive definite preconditioner;
* restriction = mean of children, prolongation reproduces constants,
  coarse operator = rediscretisation;
* CG and multigrid converge to the sparse direct solution; CG's error
  decreases monotonically in the energy norm; the V-cycle's error
  propagation contracts.

Nothing here imports oracle/ or the golden fixtures.
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
sla = pytest.importorskip("scipy.linalg")
spl = pytest.importorskip("scipy.sparse.linalg")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pmg():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1307_2036_b200 as m
    return m


class Case:
    """One small problem: grid, operator, its assembled matrix."""

    def __init__(self, pmg, kind, nx, nz, omega2, lambda2, workers=1):
        self.pmg = pmg
        if kind == "flat":
            grid = pmg.panel_grid(nx, nz, depth=1.0, flat_mode=True)
        elif kind == "curved":
            grid = pmg.panel_grid(nx, nz, depth=0.01)
        elif kind == "periodic":
            grid = pmg.periodic_box(nx, nz, 0.01)
        elif kind == "variable":
            grid = pmg.periodic_box(nx, nz, 0.01, pmg.graded_levels(nz, 0.01, 1.05),
                                    omega_shape=pmg.geometry.omega_shape_config4)
        else:
            raise AssertionError(kind)
        self.grid = grid
        self.params = pmg.toy_parameters(nx, nz, omega2, lambda2)
        self.decomp = pmg.Decomposition(nx, workers, periodic=grid.periodic)
        self.layout = self.decomp.layout(nx)
        self.op = pmg.PanelOperator(grid, self.params, self.layout)
        self.a = self.op.assemble()
        self.shape = (grid.nx, grid.ny, grid.nz)

    def field(self, arr):
        d = self.pmg.scatter_owned(np.ascontiguousarray(arr, dtype=float), self.layout)
        self.pmg.halo_exchange(d)
        return d

    def get(self, d):
        return self.pmg.gather_owned(d)

    def mat(self, v):
        return (self.a @ np.asarray(v).ravel()).reshape(self.shape)

    def direct(self, f):
        u = spl.spsolve(self.a.tocsc(), f.ravel())
        u = u + spl.spsolve(self.a.tocsc(), f.ravel() - self.a @ u)   # one refinement
        return u.reshape(self.shape)

    def energy(self, e):
        v = np.asarray(e).ravel()
        return float(v @ (self.a @ v))

    def colour_mask(self, c):
        i, j = np.meshgrid(np.arange(self.shape[0]), np.arange(self.shape[1]), indexing="ij")
        return ((i + j) % 2 == c)[:, :, None] & np.ones(self.shape, dtype=bool)


KINDS = [("flat", 8, 4, 0.7, 1.3), ("curved", 8, 4, 0.7, 1.3), ("periodic", 8, 4, 0.7, 1.3),
         ("variable", 16, 8, 6.7e-4, 3.3e-2), ("periodic", 16, 32, 1e-3, 1.0),
         ("curved", 16, 128, 6.7e-4, 3.3e-2)]


@pytest.mark.parametrize("kind,nx,nz,o2,l2", KINDS)
@pytest.mark.parametrize("workers", [1, 4])
def test_apply_and_residual_equal_matrix(pmg, kind, nx, nz, o2, l2, workers):
    if nx * nx * nz > pmg.ORACLE_CELL_CAP:
        pytest.skip("above the oracle cap")
    s = Case(pmg, kind, nx, nz, o2, l2, workers)
    rng = np.random.default_rng(4)
    ug, fg = rng.standard_normal(s.shape), rng.standard_normal(s.shape)
    u, f = s.field(ug), s.field(fg)
    ref = s.mat(ug)
    scale = np.max(np.abs(ref))
    assert np.max(np.abs(s.get(s.op.apply(u)) - ref)) <= 1e-13 * scale
    assert np.max(np.abs(s.get(s.op.residual(f, u)) - (fg - ref))) <= 1e-13 * scale
    # f - A 0 is f itself, bit for bit
    assert np.array_equal(s.get(s.op.residual(f, s.field(np.zeros(s.shape)))), fg)
    # the fused norm agrees with the residual field
    rn = s.op.residual_norm(f, u)
    assert abs(rn - np.linalg.norm(fg - ref)) <= 1e-12 * np.linalg.norm(fg - ref)


@pytest.mark.parametrize("kind,nx,nz,o2,l2", KINDS[:4])
def test_matrix_structure(pmg, kind, nx, nz, o2, l2):
    s = Case(pmg, kind, nx, nz, o2, l2)
    a = s.a
    asym = abs(a - a.T).max()
    # wrap faces of a variable coefficient are evaluated at x = 0 and x = 1:
    # equal to rounding, not bit for bit
    assert asym <= (1e-15 * abs(a).max() if kind == "variable" else 0.0)
    assert np.diff(a.tocsr().indptr).max() <= 7
    w = sla.eigvalsh(0.5 * (a + a.T).toarray()) if a.shape[0] <= 2048 else \
        spl.eigsh(a, k=1, which="SA", return_eigenvectors=False)
    assert np.min(w) > 0.0
    # constants see only the mass term (the stencil's rows sum to the cell
    # volume) except through Dirichlet faces
    one = np.ones(s.shape)
    vols = s.op.factors.volumes()
    if not s.grid.dirichlet_z:
        assert np.allclose(s.mat(one), vols, rtol=1e-12)
        assert np.allclose(s.get(s.op.apply(s.field(one))), vols, rtol=1e-12)
    # device symmetry: <A u, v> = <u, A v>
    rng = np.random.default_rng(10)
    for _ in range(5):
        u, v = s.field(rng.standard_normal(s.shape)), s.field(rng.standard_normal(s.shape))
        au_v, u_av = pmg.dist_dot(s.op.apply(u), v), pmg.dist_dot(u, s.op.apply(v))
        assert abs(au_v - u_av) <= 1e-12 * max(abs(au_v), abs(u_av))
        assert pmg.dist_dot(u, s.op.apply(u)) > 0.0


def test_column_blocks_and_cap(pmg):
    s = Case(pmg, "curved", 8, 4, 0.7, 1.3)
    a = s.a.toarray()
    nz = 4
    for i, j in ((0, 0), (3, 5), (7, 7), (4, 0)):
        b = s.op.column_block(i, j)
        base = nz * (8 * i + j)
        blk = a[base:base + nz, base:base + nz]
        assert np.allclose(np.diag(blk), b.diag, rtol=1e-15)
        assert np.allclose(np.diag(blk, -1), b.sub[1:], rtol=1e-15)
        assert np.allclose(np.diag(blk, 1), b.sup[:-1], rtol=1e-15)
        assert b.sub[0] == 0.0 and b.sup[-1] == 0.0
        # strictly dominant: the line solves need no pivoting
        assert np.all(b.diag > np.abs(b.sub) + np.abs(b.sup))
    assert pmg.vertical_blocks(s.grid, s.params)(3, 5).diag.shape == (nz,)
    with pytest.raises(ValueError):
        s.op.column_block(8, 0)
    big = pmg.panel_grid(64, 32, depth=0.01)
    assert 64 * 64 * 32 > pmg.ORACLE_CELL_CAP
    with pytest.raises(ValueError):
        pmg.PanelOperator(big, pmg.toy_parameters(64, 32, 1e-3, 1.0)).assemble()
    a2 = pmg.assemble_matrix(s.grid, s.params)
    assert abs(a2 - s.a).max() == 0.0


def block_gs(s, ug, fg, c, rho):
    """One colour's block Gauss-Seidel update on the assembled matrix: every
    column of colour c solved exactly against the current other colour
    (columns of one colour do not couple), relaxed by rho."""
    a = s.a.tocsr()
    m = s.colour_mask(c).ravel()
    idx, oth = np.flatnonzero(m), np.flatnonzero(~m)
    acc = a[idx][:, idx].tocsc()
    rhs = fg.ravel()[idx] - a[idx][:, oth] @ ug.ravel()[oth]
    new = spl.spsolve(acc, rhs)
    out = ug.ravel().copy()
    out[idx] = (1.0 - rho) * out[idx] + rho * new
    return out.reshape(s.shape)


@pytest.mark.parametrize("exact", [True, False])
@pytest.mark.parametrize("rho", [0.7, 1.0, 1.3])
@pytest.mark.parametrize("kind,nx,nz,o2,l2", KINDS[:5])
def test_half_sweep_is_block_gauss_seidel(pmg, kind, nx, nz, o2, l2, rho, exact):
    s = Case(pmg, kind, nx, nz, o2, l2)
    rng = np.random.default_rng(5)
    ug, fg = rng.standard_normal(s.shape), rng.standard_normal(s.shape)
    sm = pmg.LineSmoother(s.op)
    with pmg.exact_smoother(exact):
        for c in (0, 1):
            u, f = s.field(ug), s.field(fg)
            sm.half_sweep(u, f, c, rho)
            ref = block_gs(s, ug, fg, c, rho)
            got = s.get(u)
            assert np.max(np.abs(got - ref)) <= 1e-12 * np.max(np.abs(ref)), (c, rho)
            # the other colour is untouched
            m = s.colour_mask(1 - c)
            assert np.array_equal(got[m], ug[m])


@pytest.mark.parametrize("rho", [0.7, 1.0, 1.3])
def test_sweep_fixed_point_and_energy(pmg, rho):
    s = Case(pmg, "curved", 8, 4, 6.7e-4, 3.3e-2)
    rng = np.random.default_rng(6)
    fg = rng.standard_normal(s.shape)
    ustar = s.direct(fg)
    sm = pmg.LineSmoother(s.op)
    u, f = s.field(ustar), s.field(fg)
    sm.sweep(u, f, 1, rho)
    assert np.max(np.abs(s.get(u) - ustar)) <= 1e-12 * np.max(np.abs(ustar))
    # the A-norm of the error never grows under the relaxation (0 < rho < 2)
    u = s.field(rng.standard_normal(s.shape))
    last = s.energy(s.get(u) - ustar)
    for _ in range(6):
        sm.sweep(u, f, 1, rho)
        pmg.halo_exchange(u)
        e = s.energy(s.get(u) - ustar)
        assert e <= last * (1.0 + 1e-12)
        last = e


def test_single_column_solved_exactly(pmg):
    """nx = 1: the line solve is the whole solve (coarsest level of the
    standard policy)."""
    grid = pmg.panel_grid(1, 16, depth=0.01)
    params = pmg.toy_parameters(1, 16, 6.7e-4, 3.3e-2)
    op = pmg.PanelOperator(grid, params)
    fg = np.random.default_rng(7).standard_normal((1, 1, 16))
    u = pmg.scatter_owned(np.zeros((1, 1, 16)), op.layout)
    f = pmg.scatter_owned(fg, op.layout)
    pmg.LineSmoother(op).half_sweep(u, f, 0, 1.0)
    ref = np.linalg.solve(op.assemble().toarray(), fg.ravel())
    assert np.max(np.abs(pmg.gather_owned(u).ravel() - ref)) <= 1e-13 * np.max(np.abs(ref))


@pytest.mark.parametrize("rho", [0.7, 1.0, 1.3])
def test_ssor_closed_form(pmg, rho):
    """z = rho (2 - rho) (D + rho U)^-1 D (D + rho L)^-1 r with D the column
    blocks and the red columns ordered first."""
    nx, nz = 4, 3
    s = Case(pmg, "flat", nx, nz, 6.7e-4, 3.3e-2)
    a = s.a.toarray()
    n = a.shape[0]
    red = np.flatnonzero(s.colour_mask(0).ravel())
    blk = np.flatnonzero(s.colour_mask(1).ravel())
    perm = np.concatenate((red, blk))
    ap = a[np.ix_(perm, perm)]
    col_of = perm // nz                      # column id of each permuted unknown
    same = col_of[:, None] == col_of[None, :]
    d = np.where(same, ap, 0.0)
    low = np.where(~same & (np.arange(n)[:, None] > np.arange(n)[None, :]), ap, 0.0)
    m_inv = rho * (2.0 - rho) * np.linalg.inv(d + rho * low.T) @ d @ np.linalg.inv(d + rho * low)
    sm = pmg.LineSmoother(s.op)
    rng = np.random.default_rng(8)
    rg = rng.standard_normal(s.shape)
    z = s.get(sm.ssor_apply(s.field(rg), rho))
    ref = np.empty(n)
    ref[perm] = m_inv @ rg.ravel()[perm]
    assert np.max(np.abs(z.ravel() - ref)) <= 1e-12 * np.max(np.abs(ref))
    # symmetric, positive definite and linear as an operator on the device
    pre = pmg.SSORPreconditioner(sm, rho)
    x, y = rng.standard_normal(s.shape), rng.standard_normal(s.shape)
    mx, my = s.get(pre.apply(s.field(x))), s.get(pre.apply(s.field(y)))
    assert abs(np.vdot(mx, y) - np.vdot(x, my)) <= 1e-12 * abs(np.vdot(mx, y))
    assert np.vdot(mx, x) > 0.0
    mz = s.get(pre.apply(s.field(2.0 * x - 0.5 * y)))
    assert np.max(np.abs(mz - (2.0 * mx - 0.5 * my))) <= 1e-12 * np.max(np.abs(mz))


def test_transfers(pmg):
    s = Case(pmg, "curved", 16, 4, 6.7e-4, 3.3e-2)
    cfg = pmg.MGConfig(policy="explicit", explicit_levels=3)
    hier = pmg.build_hierarchy(s.grid, s.params, cfg, s.decomp)
    fine, coarse = hier.levels[0], hier.levels[1]
    rng = np.random.default_rng(9)
    fg = rng.standard_normal(s.shape)
    rc = pmg.gather_owned(pmg.restrict(s.field(fg), fine, coarse))
    mean = 0.25 * (fg[0::2, 0::2] + fg[1::2, 0::2] + fg[0::2, 1::2] + fg[1::2, 1::2])
    assert np.max(np.abs(rc - mean)) <= 1e-15
    # a constant is reproduced by both transfers; a checkerboard restricts to 0
    one = np.full(s.shape, 3.25)
    assert np.array_equal(pmg.gather_owned(pmg.restrict(s.field(one), fine, coarse)),
                          np.full(rc.shape, 3.25))
    i, j = np.meshgrid(np.arange(16), np.arange(16), indexing="ij")
    cb = (((i + j) % 2) * 2.0 - 1.0)[:, :, None] * np.ones(s.shape)
    assert np.max(np.abs(pmg.gather_owned(pmg.restrict(s.field(cb), fine, coarse)))) == 0.0
    cc = pmg.scatter_owned(np.full(rc.shape, 3.25), coarse.layout)
    pmg.halo_exchange(cc)
    pg = pmg.gather_owned(pmg.prolong(cc, coarse, fine))
    assert np.max(np.abs(pg - 3.25)) <= 1e-15
    # the coarse operator is the rediscretisation on the coarse grid
    cgrid = pmg.panel_grid(8, 4, depth=0.01)
    ac = pmg.PanelOperator(cgrid, s.params).assemble()
    assert abs(coarse.op.assemble() - ac).max() <= 1e-15 * abs(ac).max()


@pytest.mark.filterwarnings("ignore:recursive residual drifted")
@pytest.mark.parametrize("kind,nx,nz,o2,l2", [("curved", 8, 4, 0.7, 1.3),
                                               ("periodic", 16, 32, 1e-3, 1.0),
                                               ("variable", 16, 8, 6.7e-4, 3.3e-2)])
def test_cg_matches_direct_solve(pmg, kind, nx, nz, o2, l2):
    s = Case(pmg, kind, nx, nz, o2, l2)
    fg = np.random.default_rng(11).standard_normal(s.shape)
    ustar = s.direct(fg)
    pre = pmg.SSORPreconditioner(pmg.LineSmoother(s.op))
    u, rep = pmg.pcg_solve(s.field(fg), s.op, pre, eps=1e-12, maxiter=300)
    assert rep.converged
    assert np.max(np.abs(s.get(u) - ustar)) <= 1e-9 * np.max(np.abs(ustar))
    # the energy norm of the error decreases monotonically with the
    # iteration cap (CG's defining property), down to the rounding floor
    e_init = last = s.energy(ustar)
    for k in range(1, 8):
        uk, _ = pmg.pcg_solve(s.field(fg), s.op, pre, eps=1e-30, maxiter=k)
        e = s.energy(s.get(uk) - ustar)
        assert e <= last * (1.0 + 1e-10) + 1e-20 * e_init, k
        last = e
    # without a preconditioner the same tolerance needs many more iterations
    _, plain = pmg.pcg_solve(s.field(fg), s.op, pmg.IdentityPreconditioner(), eps=1e-8,
                             maxiter=5000)
    _, ssor = pmg.pcg_solve(s.field(fg), s.op, pre, eps=1e-8, maxiter=5000)
    assert plain.iterations > ssor.iterations


@pytest.mark.parametrize("kind,nx,nz,o2,l2,nlev", [("curved", 8, 4, 6.7e-4, 3.3e-2, 4),
                                                    ("flat", 16, 8, 6.7e-4, 3.3e-2, 5),
                                                    ("periodic", 16, 32, 1e-3, 1.0, 4),
                                                    ("variable", 16, 8, 6.7e-4, 3.3e-2, 3)])
def test_multigrid_matches_direct_solve(pmg, kind, nx, nz, o2, l2, nlev):
    s = Case(pmg, kind, nx, nz, o2, l2)
    cfg = pmg.MGConfig(policy="explicit", explicit_levels=nlev, eps=1e-12, maxiter=60)
    hier = pmg.build_hierarchy(s.grid, s.params, cfg, s.decomp)
    fg = np.random.default_rng(12).standard_normal(s.shape)
    ustar = s.direct(fg)
    u, rep = pmg.mg_solve(s.field(fg), hier, cfg)
    assert rep.converged and rep.iterations < 40
    assert np.max(np.abs(s.get(u) - ustar)) <= 1e-9 * np.max(np.abs(ustar))
    # the reported history is the true residual norm of the iterates
    assert abs(rep.residual_history[0] - np.linalg.norm(fg)) <= 1e-12 * np.linalg.norm(fg)
    true = np.linalg.norm(fg - s.mat(s.get(u)))
    assert abs(rep.residual_history[-1] - true) <= 1e-6 * rep.residual_history[0]
    # zero right-hand side: immediate return
    u0, rep0 = pmg.mg_solve(s.field(np.zeros(s.shape)), hier, cfg)
    assert rep0.iterations == 0 and rep0.converged and not np.any(s.get(u0))
    # an impossible tolerance is reported, not raised
    cfg1 = pmg.MGConfig(policy="explicit", explicit_levels=nlev, eps=1e-30, maxiter=2)
    _, rep1 = pmg.mg_solve(s.field(fg), hier, cfg1)
    assert rep1.iterations == 2 and not rep1.converged


def test_v_cycle_fixed_point_and_contraction(pmg):
    s = Case(pmg, "curved", 8, 4, 6.7e-4, 3.3e-2)
    cfg = pmg.MGConfig()
    hier = pmg.build_hierarchy(s.grid, s.params, cfg, s.decomp)
    fg = np.random.default_rng(1).standard_normal(s.shape)
    ustar = s.direct(fg)
    scratch = hier.make_scratch()
    w = s.layout.workers[0]

    def cycle_from(u0):
        scratch[0].f.parts[w].load_owned(fg)
        scratch[0].u.parts[w].load_owned(np.ascontiguousarray(u0))
        pmg.halo_exchange(scratch[0].u)
        pmg.v_cycle(hier, cfg, scratch)
        return s.get(scratch[0].u)

    # the exact solution stays put (to the noise of evaluating its residual)
    u1 = cycle_from(ustar)
    assert np.max(np.abs(u1 - ustar)) <= 1e-12 * np.max(np.abs(ustar))
    # the error propagation operator contracts in the energy norm
    rng = np.random.default_rng(2)
    for _ in range(3):
        e0 = rng.standard_normal(s.shape)
        e1 = cycle_from(ustar + e0) - ustar
        assert s.energy(e1) <= 0.25 * s.energy(e0)
