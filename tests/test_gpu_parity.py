"""CUDA path vs the oracle / reference goldens (needs a B200).

Operator, smoother and transfers are compiled without FMA contraction and
in the reference's expression order, so they must match the reference
BIT FOR BIT (tolerance 0).  Solver histories involve reductions whose
order differs (block trees vs numpy pairwise): 1e-8 relative per
north_star, with equal iteration counts; in practice ~1e-14.
"""

import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def load(name):
    return np.load(os.path.join(GOLD, name + ".npz"))


def uni(shape, seed):
    return np.random.default_rng(seed).uniform(-1.0, 1.0, size=shape)


def hist_err(h, ref):
    """Max relative history deviation; entries near the rounding floor of
    the residual evaluation (~1e-13 ||r0||) are compared absolutely."""
    h, ref = np.asarray(h, dtype=float), np.asarray(ref, dtype=float)
    return float(np.max(np.abs(h - ref) / (ref + 1e-13 * ref[0])))


@pytest.fixture(scope="module")
def pmg():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1307_2036_b200 as m
    return m


def grid_of(pmg, g, nx=None):
    nx = int(g["nx"]) if nx is None else nx
    nz = int(g["nz"])
    lv = g["levels"]
    depth = float(lv[-1] - 1.0)
    if bool(g["periodic"]):
        shape = pmg.geometry.omega_shape_config4 if bool(g["variable"]) else None
        return pmg.periodic_box(nx, nz, depth, lv, omega_shape=shape)
    return pmg.panel_grid(nx, nz, depth=depth, flat_mode=True, levels=lv)


def setup(pmg, name, workers=1):
    g = load(name)
    grid = grid_of(pmg, g)
    params = pmg.toy_parameters(grid.nx, grid.nz, float(g["omega2"]), float(g["lambda2"]))
    cfg = pmg.MGConfig(policy="explicit", explicit_levels=int(g["nlev"]), eps=1e-5)
    dec = pmg.Decomposition(grid.nx, workers)
    hier = pmg.build_hierarchy(grid, params, cfg, dec)
    return g, grid, params, cfg, hier


def field(pmg, arr, layout):
    d = pmg.scatter_owned(arr, layout)
    pmg.halo_exchange(d)
    return d


OPS = ["ops_periodic", "ops_neumann", "ops_variable", "ops_config"]


@pytest.mark.parametrize("workers", [1, 4])
@pytest.mark.parametrize("name", OPS)
def test_ops_bitwise(pmg, name, workers):
    """Exact smoother mode: every operator / smoother / transfer output is
    bit-identical to the reference."""
    with pmg.exact_smoother():
        _ops_check(pmg, name, workers, 0.0)


@pytest.mark.parametrize("workers", [1, 4])
@pytest.mark.parametrize("name", OPS)
def test_ops_fast_smoother(pmg, name, workers):
    """Default (fast, k-segmented) smoother: the reference's own half-sweep
    tolerance (tests/test_smoother.py:48 uses 1e-12 against a column-wise
    Thomas solve); operator and transfers stay bit-identical."""
    with pmg.exact_smoother(False):
        _ops_check(pmg, name, workers, 1e-12)


def _close(got, ref, tol):
    if tol == 0.0:
        return np.array_equal(got, ref)
    return np.max(np.abs(got - ref)) <= tol * max(1.0, np.max(np.abs(ref)))


def _ops_check(pmg, name, workers, tol):
    g, grid, params, cfg, hier = setup(pmg, name, workers)
    nx, nz = grid.nx, grid.nz
    fine, coarse = hier.levels[0], hier.levels[1]
    op, lay = fine.op, fine.layout
    ug, fg = uni((nx, nx, nz), 1), uni((nx, nx, nz), 2)
    u, f = field(pmg, ug, lay), field(pmg, fg, lay)
    G = pmg.gather_owned
    assert np.array_equal(G(op.apply(u)), g["apply"])
    assert np.array_equal(G(op.residual(f, u)), g["residual"])
    sm = fine.smoother
    for rho in (1.0, 1.4):
        uu = field(pmg, ug, lay)
        sm.half_sweep(uu, f, 0, rho)
        assert _close(G(uu), g[f"half_red_rho{rho}"], tol)
        pmg.halo_exchange(uu)
        sm.half_sweep(uu, f, 1, rho)
        assert _close(G(uu), g[f"half_black_rho{rho}"], tol)
    uu = field(pmg, ug, lay)
    sm.sweep(uu, f, nsweeps=2, rho=1.0)
    assert _close(G(uu), g["sweep2"], tol)
    for rho in (1.0, 1.3):
        assert _close(G(sm.ssor_apply(f, rho)), g[f"ssor_rho{rho}"], tol)
    assert np.array_equal(G(pmg.restrict(u, fine, coarse)), g["restrict_mean"])
    cd = field(pmg, uni((nx // 2, nx // 2, nz), 3), coarse.layout)
    assert np.array_equal(G(pmg.prolong(cd, coarse, fine)), g["prolong"])
    # one V-cycle from zero, unfused and fused (same arithmetic)
    for fused in (False, True):
        c2 = pmg.MGConfig(policy="explicit", explicit_levels=int(g["nlev"]), fused=fused)
        scratch = hier.make_scratch()
        scratch[0].f.copy_from(f)
        pmg.v_cycle(hier, c2, scratch)
        assert _close(G(scratch[0].u), g["vcycle1"], tol)


@pytest.mark.parametrize("name", OPS)
def test_solvers_exact_mode_vs_reference(pmg, name):
    """Exact smoother: MG histories agree to reduction-order rounding."""
    g, grid, params, cfg, hier = setup(pmg, name)
    nx, nz = grid.nx, grid.nz
    with pmg.exact_smoother():
        u, rep = pmg.mg_solve(pmg.scatter_owned(uni((nx, nx, nz), 2), hier.fine.layout),
                              hier, cfg)
    ref = g["mg_history"]
    assert rep.iterations == len(ref) - 1
    assert np.max(np.abs(np.array(rep.residual_history) - ref) / ref) <= 1e-12
    got = pmg.gather_owned(u)
    assert np.max(np.abs(got - g["mg_u"])) <= 1e-12 * np.max(np.abs(g["mg_u"]))


@pytest.mark.parametrize("graph", [False, True])
@pytest.mark.parametrize("name", OPS)
def test_solvers_vs_reference(pmg, name, graph):
    g, grid, params, cfg, hier = setup(pmg, name)
    nx, nz = grid.nx, grid.nz
    fg = uni((nx, nx, nz), 2)
    cfg = pmg.MGConfig(policy="explicit", explicit_levels=int(g["nlev"]), eps=1e-5,
                       graph=graph)
    f = pmg.scatter_owned(fg, hier.fine.layout)
    u, rep = pmg.mg_solve(f, hier, cfg)
    # fast (k-segmented) smoother: reassociated elimination -> ~1e-12;
    # north_star bar is 1e-8
    ref = g["mg_history"]
    assert rep.iterations == len(ref) - 1
    assert np.max(np.abs(np.array(rep.residual_history) - ref) / ref) <= 1e-10
    got = pmg.gather_owned(u)
    assert np.max(np.abs(got - g["mg_u"])) <= 1e-10 * np.max(np.abs(g["mg_u"]))
    op = hier.fine.op
    pre = pmg.SSORPreconditioner(pmg.LineSmoother(op))
    uc, rc = pmg.pcg_solve(f, op, pre, eps=1e-8, maxiter=200)
    ref = g["cg_history"]
    assert rc.iterations == len(ref) - 1
    assert np.max(np.abs(np.array(rc.residual_history) - ref) / ref) <= 1e-10
    got = pmg.gather_owned(uc)
    assert np.max(np.abs(got - g["cg_u"])) <= 1e-10 * np.max(np.abs(g["cg_u"]))


@pytest.mark.parametrize("solver", ["mg", "cg"])
def test_config0_vs_reference(pmg, solver):
    from paper_1307_2036_b200 import configs
    g = load(f"config0_{solver}")
    prob = configs.config(0)
    fg = configs.rhs(prob.nx, prob.ny, prob.nz, 0)
    grid, params = prob.grid(), prob.params()
    if solver == "mg":
        cfg = prob.mg_config()
        hier = pmg.build_hierarchy(grid, params, cfg)
        u, rep = pmg.mg_solve(pmg.scatter_owned(fg, hier.fine.layout), hier, cfg)
    else:
        op = pmg.PanelOperator(grid, params)
        pre = pmg.SSORPreconditioner(pmg.LineSmoother(op))
        u, rep = pmg.pcg_solve(pmg.scatter_owned(fg, op.layout), op, pre, eps=1e-5,
                               maxiter=2000)
    ref = g["history"]
    assert rep.iterations == int(g["iterations"])
    assert np.max(np.abs(np.array(rep.residual_history) - ref) / ref) <= 1e-8
    got = pmg.gather_owned(u)
    assert np.max(np.abs(got - g["u"])) <= 1e-8 * np.max(np.abs(g["u"]))


@pytest.mark.parametrize("w", ["0.0001", "0.001", "0.01", "0.1"])
@pytest.mark.parametrize("solver", ["mg", "cg"])
def test_omega_sweep_small(pmg, w, solver):
    from paper_1307_2036_b200 import configs
    g = load(f"sweep128_{solver}_w{w}")
    prob = configs.Problem(128, 128, 64, float(w), 1.0, 4)
    fg = configs.rhs(128, 128, 64, 0)
    grid, params = prob.grid(), prob.params()
    if solver == "mg":
        cfg = prob.mg_config()
        hier = pmg.build_hierarchy(grid, params, cfg)
        _, rep = pmg.mg_solve(pmg.scatter_owned(fg, hier.fine.layout), hier, cfg)
    else:
        op = pmg.PanelOperator(grid, params)
        pre = pmg.SSORPreconditioner(pmg.LineSmoother(op))
        _, rep = pmg.pcg_solve(pmg.scatter_owned(fg, op.layout), op, pre, eps=1e-5,
                               maxiter=2000)
    ref = g["history"]
    assert rep.iterations == int(g["iterations"])
    assert np.max(np.abs(np.array(rep.residual_history) - ref) / ref) <= 1e-8


@pytest.mark.parametrize("name,nx,nlev", [("config4_like_mg", 64, 4),
                                          ("config4_like256_mg", 256, 5)])
def test_config4_like(pmg, name, nx, nlev):
    from paper_1307_2036_b200 import configs
    g = load(name)
    prob = configs.Problem(nx, nx, 128, 1e-3, 1.0, nlev, stretch=1.05, variable_omega=True)
    fg = configs.rhs(nx, nx, 128, 0)
    cfg = prob.mg_config()
    hier = pmg.build_hierarchy(prob.grid(), prob.params(), cfg)
    assert not hier.fine.op.uniform
    u, rep = pmg.mg_solve(pmg.scatter_owned(fg, hier.fine.layout), hier, cfg)
    ref = g["history"]
    assert rep.iterations == int(g["iterations"])
    assert np.max(np.abs(np.array(rep.residual_history) - ref) / ref) <= 1e-8
    ug = pmg.gather_owned(u)
    idx = g["sample_idx"]
    got = ug[idx[:, 0], idx[:, 1], idx[:, 2]]
    assert np.max(np.abs(got - g["sample_u"])) <= 1e-8 * float(g["u_absmax"])


@pytest.mark.parametrize("workers", [2, 4, 8, 16])
@pytest.mark.parametrize("periodic", [True, False])
def test_partition_invariance(pmg, workers, periodic):
    """tests/test_partition.py:122-154 on the device: parts emulated on one
    GPU exchange halos through the pack/unpack kernels."""
    nx, nz = 32, 8
    if periodic:
        grid = pmg.periodic_box(nx, nz, 0.01)
    else:
        grid = pmg.panel_grid(nx, nz, flat_mode=True)
    params = pmg.toy_parameters(nx, nz, 6.7e-4 if not periodic else 1e-3, 3.3e-2)
    fg = uni((nx, nx, nz), 3)
    hist = {}
    cg = {}
    for p in (1, workers):
        cfg = pmg.MGConfig(policy="explicit", explicit_levels=3, graph=False)
        hier = pmg.build_hierarchy(grid, params, cfg, pmg.Decomposition(nx, p))
        f = pmg.scatter_owned(fg, hier.fine.layout)
        _, rep = pmg.mg_solve(f, hier, cfg)
        hist[p] = np.array(rep.residual_history)
        op = hier.fine.op
        pre = pmg.SSORPreconditioner(pmg.LineSmoother(op))
        _, rc = pmg.pcg_solve(f, op, pre, eps=1e-5, maxiter=100)
        cg[p] = np.array(rc.residual_history)
    for h in (hist, cg):
        assert len(h[1]) == len(h[workers])
        assert np.max(np.abs(h[workers] - h[1]) / h[1]) <= 1e-10


def test_exchange_counts(pmg):
    """1 + 2(nu_pre + nu_post) exchanges per level per cycle, 2 per coarse
    sweep (tests/test_multigrid.py:165-177)."""
    grid = pmg.periodic_box(32, 4, 0.01)
    params = pmg.toy_parameters(32, 4, 1e-3, 1.0)
    cfg = pmg.MGConfig(policy="explicit", explicit_levels=3, graph=False, maxiter=1, eps=0.5)
    hier = pmg.build_hierarchy(grid, params, cfg, pmg.Decomposition(32, 4))
    f = pmg.scatter_owned(uni((32, 32, 4), 0), hier.fine.layout)
    scratch = hier.make_scratch()
    scratch[0].f.copy_from(f)
    hier.reset_counters()
    pmg.v_cycle(hier, cfg, scratch)
    counts = [lev.layout.halo_count for lev in hier.levels]
    assert counts[:-1] == [5] * 2 and counts[-1] == 2


def test_layout_round_trip(pmg):
    for nx, ny, nz, p in ((16, 16, 4, 1), (32, 16, 3, 2), (8, 8, 5, 4)):
        grid = pmg.periodic_box(nx, nz, 0.01, ny=ny)
        dec = pmg.Decomposition(nx, p, ny=ny, periodic=True)
        lay = dec.layout(nx)
        a = uni((nx, ny, nz), 7)
        assert np.array_equal(pmg.gather_owned(pmg.scatter_owned(a, lay)), a)


def test_rectangular_periodic_vs_oracle(pmg):
    """nx != ny periodic grids (the 2- and 8-GPU global grids of configs[3]),
    split into 1, 2 and 8 parts, against the oracle on the same grid."""
    from oracle import port
    nx, ny, nz = 32, 16, 8
    lv = port.uniform_levels(nz, 1.0)
    fg = uni((nx, ny, nz), 5)
    h = port.Hierarchy(nx, ny, 3, lambda a, b: port.config_factors(a, b, lv), 0.7, 1.3)
    ou, orep = port.mg_solve(h, fg)
    grid = pmg.periodic_box(nx, nz, 1.0, lv, ny=ny)
    params = pmg.toy_parameters(nx, nz, 0.7, 1.3)
    for exact, tol in ((True, 1e-10), (False, 1e-8)):
        for p in (1, 2, 8):
            cfg = pmg.MGConfig(policy="explicit", explicit_levels=3)
            dec = pmg.Decomposition(nx, p, ny=ny)
            hier = pmg.build_hierarchy(grid, params, cfg, dec)
            with pmg.exact_smoother(exact):
                u, rep = pmg.mg_solve(pmg.scatter_owned(fg, hier.fine.layout), hier, cfg)
            assert rep.iterations == orep.iterations > 3
            assert hist_err(rep.residual_history, orep.residual_history) <= tol
            ug = pmg.gather_owned(u)
            assert np.max(np.abs(ug - ou[1:-1, 1:-1, :])) <= tol * np.max(np.abs(ug))


def test_zero_rhs_and_breakdown(pmg):
    grid = pmg.periodic_box(16, 4, 0.01)
    params = pmg.toy_parameters(16, 4, 1e-3, 1.0)
    cfg = pmg.MGConfig(policy="explicit", explicit_levels=2)
    hier = pmg.build_hierarchy(grid, params, cfg)
    f = pmg.scatter_owned(np.zeros((16, 16, 4)), hier.fine.layout)
    u, rep = pmg.mg_solve(f, hier, cfg)
    assert rep.iterations == 0 and rep.converged and rep.residual_history == [0.0]
    u, rep = pmg.pcg_solve(f, hier.fine.op)
    assert rep.iterations == 0 and rep.converged


@pytest.mark.slow
def test_config1_full_size(pmg):
    """BASELINE configs[1] at full size (1024^2 x 128, 7 levels) against the
    reference's own history (tests/golden/config1_mg.npz)."""
    path = os.path.join(GOLD, "config1_mg.npz")
    if not os.path.exists(path):
        pytest.skip("config1 golden not generated")
    from paper_1307_2036_b200 import configs
    g = load("config1_mg")
    prob = configs.config(1)
    fg = configs.rhs(prob.nx, prob.ny, prob.nz, 0)
    cfg = prob.mg_config()
    hier = pmg.build_hierarchy(prob.grid(), prob.params(), cfg)
    u, rep = pmg.mg_solve(pmg.scatter_owned(fg, hier.fine.layout), hier, cfg)
    ref = g["history"]
    assert rep.iterations == int(g["iterations"])
    assert np.max(np.abs(np.array(rep.residual_history) - ref) / ref) <= 1e-8
    ug = pmg.gather_owned(u)
    idx = g["sample_idx"]
    got = ug[idx[:, 0], idx[:, 1], idx[:, 2]]
    assert np.max(np.abs(got - g["sample_u"])) <= 1e-8 * float(g["u_absmax"])
    assert abs(ug.sum() - float(g["u_sum"])) <= 1e-8 * float(g["u_absmax"]) * ug.size ** 0.5


@pytest.mark.slow
@pytest.mark.parametrize("w", ["0.0001", "0.001", "0.01", "0.1"])
def test_config2_cg_full_size(pmg, w):
    """BASELINE configs[2]: CG + line SSOR at 1024^2 x 128 for the omega^2
    sweep, against the reference's own full histories (make_golden.py big)."""
    path = os.path.join(GOLD, f"config2_cg_w{w}.npz")
    if not os.path.exists(path):
        pytest.skip("config2 golden not generated")
    from paper_1307_2036_b200 import configs
    g = load(f"config2_cg_w{w}")
    prob = configs.config(2, omega2=float(w))
    op = pmg.PanelOperator(prob.grid(), prob.params())
    pre = pmg.SSORPreconditioner(pmg.LineSmoother(op))
    f = pmg.scatter_owned(configs.rhs(prob.nx, prob.ny, prob.nz, 0), op.layout)
    u, rep = pmg.pcg_solve(f, op, pre, eps=1e-5, maxiter=2000)
    assert rep.iterations == int(g["iterations"])
    assert hist_err(rep.residual_history, g["history"]) <= 1e-8
    ug = pmg.gather_owned(u)
    idx = g["sample_idx"]
    got = ug[idx[:, 0], idx[:, 1], idx[:, 2]]
    assert np.max(np.abs(got - g["sample_u"])) <= 1e-8 * float(g["u_absmax"])


@pytest.mark.slow
@pytest.mark.parametrize("w", ["0.0001", "0.01", "0.1"])
def test_config2_mg_full_size(pmg, w):
    """configs[2] companion: MG iteration counts stay flat across omega^2."""
    path = os.path.join(GOLD, f"config2_mg_w{w}.npz")
    if not os.path.exists(path):
        pytest.skip("config2 MG golden not generated")
    from paper_1307_2036_b200 import configs
    g = load(f"config2_mg_w{w}")
    prob = configs.config(2, omega2=float(w))
    cfg = prob.mg_config()
    hier = pmg.build_hierarchy(prob.grid(), prob.params(), cfg)
    f = pmg.scatter_owned(configs.rhs(prob.nx, prob.ny, prob.nz, 0), hier.fine.layout)
    u, rep = pmg.mg_solve(f, hier, cfg)
    assert rep.iterations == int(g["iterations"])
    assert hist_err(rep.residual_history, g["history"]) <= 1e-8


@pytest.mark.parametrize("name", ["native_panel32", "native_flat32", "native_panel64_shallow"])
def test_reference_native_problem(pmg, name):
    """The reference's own problem family run UNMODIFIED by the reference:
    gnomonic cubed-sphere panel (or flat box), zero-flux boundaries, graded
    levels, derived Table-1 parameters, standard / very-shallow policies
    (down to a single column).  Our geometry factors, mirror halos and
    solvers reproduce its operator, MG and CG."""
    g = load(name)
    nx, nz = int(g["nx"]), int(g["nz"])
    grid = pmg.panel_grid(nx, nz, flat_mode=bool(g["flat"]))
    params = pmg.derive_parameters(nx, nz, float(g["dt"]))
    assert params.omega2 == float(g["omega2"]) and params.lambda2 == float(g["lambda2"])
    cfg = pmg.MGConfig(policy=str(g["policy"]))
    hier = pmg.build_hierarchy(grid, params, cfg)
    assert hier.level_sizes() == list(g["levels"])
    op = hier.fine.op
    u = pmg.scatter_owned(np.random.default_rng(4).uniform(-1, 1, (nx, nx, nz)), op.layout)
    pmg.halo_exchange(u)
    ref = g["apply"]
    assert np.max(np.abs(pmg.gather_owned(op.apply(u)) - ref)) <= 1e-13 * np.max(np.abs(ref))
    fg = np.random.default_rng(3).uniform(-1, 1, (nx, nx, nz))
    ud, rep = pmg.mg_solve(pmg.scatter_owned(fg, hier.fine.layout), hier, cfg)
    assert rep.iterations == len(g["mg_history"]) - 1
    assert hist_err(rep.residual_history, g["mg_history"]) <= 1e-8
    mu = g["mg_u"]
    assert np.max(np.abs(pmg.gather_owned(ud) - mu)) <= 1e-8 * np.max(np.abs(mu))
    pre = pmg.SSORPreconditioner(pmg.LineSmoother(op))
    uc, rc = pmg.pcg_solve(pmg.scatter_owned(fg, op.layout), op, pre, eps=1e-5, maxiter=500)
    assert rc.iterations == len(g["cg_history"]) - 1
    assert hist_err(rc.residual_history, g["cg_history"]) <= 1e-8


class _FakeDist:
    """In-process stand-in for torch.distributed P2P: every 'rank' is a
    thread; messages go through a mailbox as device-to-device copies.  Lets
    the multi-rank halo path (pack -> message plan -> unpack) run with the
    real kernels on one GPU without ranks waiting on each other's kernels."""

    def __init__(self):
        import threading
        self.box = {}
        self.cv = threading.Condition()
        self.local = threading.local()
        self.isend, self.irecv = "send", "recv"

    def get_backend(self):          # device buffers move directly, as with NCCL
        return "nccl"

    class P2POp:
        def __init__(self, op, tensor, peer, tag=0):
            self.op, self.tensor, self.peer, self.tag = op, tensor, peer, tag

    def batch_isend_irecv(self, ops):
        me = self.local.rank
        with self.cv:
            for op in ops:
                if op.op == "send":
                    self.box.setdefault((me, op.peer, op.tag), []).append(op.tensor.clone())
            self.cv.notify_all()
        for op in ops:
            if op.op == "recv":
                key = (op.peer, me, op.tag)
                with self.cv:
                    self.cv.wait_for(lambda: self.box.get(key))
                    op.tensor.copy_(self.box[key].pop(0))

        class _Done:
            def wait(self):
                pass
        return [_Done()]


@pytest.mark.parametrize("px,py,periodic", [(2, 1, True), (2, 2, True), (4, 2, True),
                                            (2, 2, False)])
def test_rank_halo_path_on_device(pmg, px, py, periodic):
    import threading
    from paper_1307_2036_b200 import partition as pt
    nx, ny, nz = 16 * px, 8 * py, 6
    dec = pmg.Decomposition(nx, px * py, ny=ny, px=px, py=py, periodic=periodic)
    lay = dec.layout(nx)
    a = uni((nx, ny, nz), 11)
    ref = pmg.scatter_owned(a, lay)
    pmg.halo_exchange(ref)                      # in-process exchange (reference path)
    ranks = {}
    for w in lay.workers:
        part = pt.DevField(lay.geometry(w, nz))
        i0, j0 = lay.origin(w)
        part.load_owned(a[i0:i0 + lay.mx, j0:j0 + lay.my, :])
        ranks[w] = pt.DistField(lay, {w: part})
    fake = _FakeDist()
    torch.cuda.synchronize()
    errors = []

    def run(w):
        try:
            fake.local.rank = w
            for faces in ((0, 1), (2, 3)):
                pt._phase_dist(ranks[w], faces, pt._stream(), fake)
            torch.cuda.synchronize()
        except Exception as err:  # pragma: no cover
            errors.append(err)
    th = [threading.Thread(target=run, args=(w,)) for w in lay.workers]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=60)
    assert not errors, errors
    for w in lay.workers:
        assert torch.equal(ranks[w].parts[w].data, ref.parts[w].data), w


@pytest.mark.parametrize("periodic", [True, False])
def test_native_drivers_match_python(pmg, periodic):
    """pmg_mg_solve / pmg_pcg_solve (C++ drivers, CUDA-graph replay) against
    the Python drivers over the same kernels: bit-identical histories and
    iterates, on the legacy stream and on a side stream."""
    from paper_1307_2036_b200 import krylov as kr
    from paper_1307_2036_b200 import multigrid as mgm
    nx, nz = 32, 8
    grid = pmg.periodic_box(nx, nz, 0.01) if periodic else pmg.panel_grid(nx, nz, flat_mode=True)
    params = pmg.toy_parameters(nx, nz, 1e-3, 3.3e-2)
    cfg = pmg.MGConfig(policy="explicit", explicit_levels=3, eps=1e-9, lagged_norm=False)
    hier = pmg.build_hierarchy(grid, params, cfg)
    f = pmg.scatter_owned(uni((nx, nx, nz), 5), hier.fine.layout)
    res = {}
    for native in (False, True):
        mgm.USE_NATIVE = kr.USE_NATIVE = native
        try:
            u, rep = pmg.mg_solve(f, hier, cfg)
            side = torch.cuda.Stream()
            side.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(side):
                u2, rep2 = pmg.mg_solve(f, hier, cfg)
            torch.cuda.current_stream().wait_stream(side)
            op = hier.fine.op
            cg = {}
            for name, pre in (("ssor", pmg.SSORPreconditioner(pmg.LineSmoother(op))),
                              ("ssor13", pmg.SSORPreconditioner(pmg.LineSmoother(op), 1.3)),
                              ("id", pmg.IdentityPreconditioner())):
                uc, rc = pmg.pcg_solve(f, op, pre, eps=1e-8, maxiter=200)
                cg[name] = (rc.residual_history, pmg.gather_owned(uc), rc.converged)
            res[native] = (rep.residual_history, pmg.gather_owned(u), rep2.residual_history,
                           pmg.gather_owned(u2), cg)
        finally:
            mgm.USE_NATIVE = kr.USE_NATIVE = True
    a, b = res[False], res[True]
    assert a[0] == b[0] and np.array_equal(a[1], b[1])
    assert b[2] == b[0] and np.array_equal(b[3], b[1])
    for name in a[4]:
        assert a[4][name][0] == b[4][name][0], name
        assert np.array_equal(a[4][name][1], b[4][name][1]), name
        assert a[4][name][2] and b[4][name][2]


def test_native_hierarchy_errors(pmg):
    from paper_1307_2036_b200 import _lib
    lib = _lib.load()
    grid = pmg.periodic_box(16, 4, 0.01)
    params = pmg.toy_parameters(16, 4, 1e-3, 1.0)
    cfg = pmg.MGConfig(policy="explicit", explicit_levels=2)
    hier = pmg.build_hierarchy(grid, params, cfg)
    w = hier.fine.layout.local_workers[0]
    hs = [hier.levels[1].op.handles[w].h.value, hier.levels[0].op.handles[w].h.value]
    import ctypes as C
    arr = (C.c_void_p * 2)(*hs)
    d = _lib.MGDesc(1, 1, 1, 1.0, 1, 1)
    out = C.c_void_p()
    assert lib.pmg_hier_create(arr, 2, C.byref(d), C.byref(out)) == _lib.PMG_ERR_VALUE
    d = _lib.MGDesc(1, 1, 1, 2.5, 1, 1)
    arr = (C.c_void_p * 2)(*hs[::-1])
    assert lib.pmg_hier_create(arr, 2, C.byref(d), C.byref(out)) == _lib.PMG_ERR_VALUE
    # breakdown maps to BreakdownError: an indefinite "preconditioner" is not
    # reachable through the API, so check the status mapping directly
    with pytest.raises(pmg.BreakdownError):
        _lib.check(_lib.PMG_ERR_BREAKDOWN, "pmg_pcg_solve")


@pytest.mark.parametrize("solver", ["mg", "cg", "mg_parts", "cg_parts"])
def test_c_host_program(pmg, tmp_path, solver):
    """examples/c_solve.c: a plain C program builds the levels, uploads f,
    solves and downloads u through include/pmg.h alone; its history and
    solution equal the Python drop-in's bit for bit (same kernels).  The
    *_parts solvers cut the grid into a 2 x 2 decomposition in C and run
    the multi-part drivers (pmg_phier_mg_solve / pmg_phier_pcg_solve)
    against the Python drop-in on the same decomposition."""
    import shutil
    import subprocess
    from paper_1307_2036_b200 import _lib, configs
    from paper_1307_2036_b200.geometry import build_factors
    from paper_1307_2036_b200.stencil import _part_factors
    if shutil.which("gcc") is None:
        pytest.skip("no C compiler")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    exe = tmp_path / "c_solve"
    cuda = "/usr/local/cuda"
    libdir = os.path.dirname(_lib.LIB_PATH)
    subprocess.run(["gcc", "-O2", "-o", str(exe), os.path.join(root, "examples", "c_solve.c"),
                    "-I", os.path.join(root, "include"), "-I", f"{cuda}/include",
                    "-L", libdir, "-lpmg", "-L", f"{cuda}/lib64", "-lcudart",
                    f"-Wl,-rpath,{libdir}:{cuda}/lib64"], check=True)
    prob = configs.config(0)
    cfg = prob.mg_config()
    hier = pmg.build_hierarchy(prob.grid(), prob.params(), cfg)
    fg = configs.rhs(prob.nx, prob.ny, prob.nz, 0)
    maxiter = 50
    code = {"mg": 0, "cg": 1, "mg_parts": 2, "cg_parts": 3}[solver]
    with open(tmp_path / "in.bin", "wb") as fp:
        np.array([prob.nx, prob.ny, prob.nz, len(hier.levels), 1, maxiter, code],
                 dtype=np.int32).tofile(fp)
        op0 = hier.fine.op
        np.array([1e-5, op0.omega2, op0.vcoef]).tofile(fp)
        for lev in hier.levels:
            fac = build_factors(lev.grid)
            for a in (fac.dr, fac.vprof, fac.volprof,
                      *_part_factors(fac, 0, 0, lev.grid.nx, lev.grid.ny)):
                np.ascontiguousarray(a, dtype=np.float64).tofile(fp)
        fg.tofile(fp)
    run = subprocess.run([str(exe), str(tmp_path / "in.bin"), str(tmp_path / "out.bin")],
                         capture_output=True, text=True)
    assert run.returncode == 0, run.stderr
    raw = open(tmp_path / "out.bin", "rb").read()
    iters, conv = np.frombuffer(raw[:8], dtype=np.int32)
    hist = np.frombuffer(raw[8:8 + 8 * (iters + 1)])
    u_c = np.frombuffer(raw[8 + 8 * (iters + 1):]).reshape(prob.nx, prob.ny, prob.nz)
    if solver.endswith("_parts"):
        hier = pmg.build_hierarchy(prob.grid(), prob.params(), cfg,
                                   pmg.Decomposition(prob.nx, 4, px=2, py=2))
    f = pmg.scatter_owned(fg, hier.fine.layout)
    if solver.startswith("mg"):
        u, rep = pmg.mg_solve(f, hier, cfg)
    else:
        op = hier.fine.op
        u, rep = pmg.pcg_solve(f, op, pmg.SSORPreconditioner(pmg.LineSmoother(op)), eps=1e-5,
                               maxiter=maxiter)
    assert conv == 1 and iters == rep.iterations
    assert list(hist) == rep.residual_history
    assert np.array_equal(u_c, pmg.gather_owned(u))
    if solver.startswith("mg"):          # and the reference's own history
        g = load("config0_mg")
        ref = np.asarray(g["history"])
        assert len(ref) == len(hist)
        assert np.max(np.abs(hist - ref) / ref[0]) <= 1e-10


@pytest.mark.parametrize("workers", [4, 16])
@pytest.mark.parametrize("l_split", [None, 3])
def test_folding_partition_invariance(pmg, workers, l_split):
    """Standard policy (down to one global column) on P parts: the coarse
    levels fold onto fewer workers through collect / distribute
    (partition.py:194-240); histories equal P = 1 to 1e-10
    (tests/test_partition.py:122-154), fold counters as the reference."""
    nx, nz = 32, 8
    grid = pmg.panel_grid(nx, nz, flat_mode=True)
    params = pmg.toy_parameters(nx, nz, 6.7e-4, 3.3e-2)
    fg = uni((nx, nx, nz), 9)
    hist = {}
    for p in (1, workers):
        cfg = pmg.MGConfig(policy="standard", l_split=l_split, graph=False)
        hier = pmg.build_hierarchy(grid, params, cfg, pmg.Decomposition(nx, p))
        if p > 1:
            assert hier.first_fold_level() is not None
        f = pmg.scatter_owned(fg, hier.fine.layout)
        hier.reset_counters()
        _, rep = pmg.mg_solve(f, hier, cfg)
        hist[p] = np.array(rep.residual_history)
        if p > 1:
            folds = sum(lev.fold_layout is not None for lev in hier.levels)
            assert hier.decomp.collect_calls == folds * rep.iterations
            assert hier.decomp.distribute_calls == folds * rep.iterations
    assert len(hist[1]) == len(hist[workers])
    assert np.max(np.abs(hist[workers] - hist[1]) / hist[1][0]) <= 1e-10


def test_collect_distribute_round_trip(pmg):
    nx, nz = 16, 3
    dec = pmg.Decomposition(nx, 16)
    lay = dec.layout(nx)
    fold = dec.layout(nx, active=(2, 2))
    a = uni((nx, nx, nz), 4)
    df = pmg.scatter_owned(a, lay)
    pmg.halo_exchange(df)
    from paper_1307_2036_b200.partition import collect, distribute
    big = collect(df, fold)
    assert np.array_equal(pmg.gather_owned(big), a)
    back = distribute(big, lay)
    assert np.array_equal(pmg.gather_owned(back), a)


@pytest.mark.parametrize("nx,nz,workers", [(32, 32, 1), (64, 64, 1), (64, 128, 1),
                                           (128, 128, 4), (256, 32, 1)])
def test_staged_smoother_vs_exact(pmg, nx, nz, workers):
    """The fast half-sweep at nz multiples of 16 and parts of >= 32 columns
    (k_half_sweep_seg with compile-time plane strides) against the exact
    sequential solver, every mode of
    LineSmoother.half_sweep (rho, zero start, no neighbours, post scale) and
    ssor_apply: 1e-12 (tests/test_smoother.py:48)."""
    grid = pmg.periodic_box(nx, nz, 0.01)
    params = pmg.toy_parameters(nx, nz, 1e-3, 1.0)
    op = pmg.PanelOperator(grid, params, pmg.Decomposition(nx, workers).layout(nx))
    sm = pmg.LineSmoother(op)
    ug, fg = uni((nx, nx, nz), 21), uni((nx, nx, nz), 22)
    f = pmg.scatter_owned(fg, op.layout)
    G = pmg.gather_owned
    runs = {}
    for exact in (True, False):
        with pmg.exact_smoother(exact):
            out = []
            for color, rho, zs, nb, ps in ((0, 1.0, False, False, 1.0), (1, 1.0, False, False, 1.0),
                                           (0, 1.4, False, False, 1.0), (0, 1.0, True, True, 1.0),
                                           (1, 1.3, True, False, 0.7)):
                u = pmg.scatter_owned(ug, op.layout)
                pmg.halo_exchange(u)
                sm.half_sweep(u, f, color, rho, zs, nb, ps)
                out.append(G(u))
            out.append(G(sm.ssor_apply(f, 1.0)))
            runs[exact] = out
    for a, b in zip(runs[True], runs[False]):
        assert _close(b, a, 1e-12)


@pytest.mark.parametrize("nx,nz", [(4, 1), (8, 2), (8, 3), (16, 5), (32, 17), (16, 33),
                                   (32, 100), (8, 255), (8, 256), (8, 257), (8, 300)])
def test_shapes_vs_oracle(pmg, nx, nz):
    """Ragged and extreme vertical sizes (single level, odd nz, non-multiples
    of the segment length, the 256-level limits of the batched kernels and
    beyond): MG and SSOR-CG against the oracle, both smoother modes."""
    from oracle import port
    lv = port.uniform_levels(nz, 0.01)
    nlev = min(3, int(np.log2(nx)) + 1)
    fg = uni((nx, nx, nz), nz)
    h = port.Hierarchy(nx, nx, nlev, lambda a, b: port.config_factors(a, b, lv), 1e-3, 1.0)
    ou, orep = port.mg_solve(h, fg, eps=1e-6)
    oc, crep = port.pcg_solve(h.levels[0], fg, eps=1e-6, maxiter=300)
    grid = pmg.periodic_box(nx, nz, 0.01, lv)
    params = pmg.toy_parameters(nx, nz, 1e-3, 1.0)
    for exact, tol in ((True, 1e-10), (False, 1e-8)):
        cfg = pmg.MGConfig(policy="explicit", explicit_levels=nlev, eps=1e-6)
        hier = pmg.build_hierarchy(grid, params, cfg)
        f = pmg.scatter_owned(fg, hier.fine.layout)
        with pmg.exact_smoother(exact):
            u, rep = pmg.mg_solve(f, hier, cfg)
            op = hier.fine.op
            uc, rc = pmg.pcg_solve(f, op, pmg.SSORPreconditioner(pmg.LineSmoother(op)),
                                   eps=1e-6, maxiter=300)
        assert rep.iterations == orep.iterations, exact
        # relative agreement down to the residual evaluation's rounding floor
        # (~1e-15 ||r0|| for the reassociated fast solver)
        h, ref = np.array(rep.residual_history), np.array(orep.residual_history)
        assert np.all(np.abs(h - ref) <= tol * ref + 1e-13 * ref[0]), (exact, h, ref)
        ug = pmg.gather_owned(u)
        assert np.max(np.abs(ug - ou[1:-1, 1:-1, :])) <= tol * max(1.0, np.max(np.abs(ug)))
        assert abs(rc.iterations - crep.iterations) <= (0 if exact else 1)
        assert rc.converged


def _red_mask(nx, ny, nz):
    i, j = np.meshgrid(np.arange(nx), np.arange(ny), indexing="ij")
    return np.broadcast_to((((i + j) % 2) == 0)[:, :, None], (nx, ny, nz))


@pytest.mark.parametrize("nx,nz,variable", [(32, 128, False), (128, 80, False), (64, 96, False),
                                            (64, 128, True), (32, 64, True)])
def test_half_sweep_res(pmg, nx, nz, variable):
    """pmg_half_sweep_res: the relaxed red values equal pmg_half_sweep's bit
    for bit (written into the other buffer, the input untouched), and the
    fused sum equals ||f - A u||^2 over the red cells of the input."""
    import ctypes as C
    from paper_1307_2036_b200 import _lib
    lib = _lib.load()
    from paper_1307_2036_b200 import configs
    ny = nx
    if variable:      # configs[4]'s graded levels and omega^2(x, y)
        prob = configs.Problem(nx, nx, nz, 1e-3, 1.0, 1, stretch=1.05, variable_omega=True)
        grid, params = prob.grid(), prob.params()
    else:
        grid = pmg.periodic_box(nx, nz, 0.01)
        params = pmg.toy_parameters(nx, nz, 1e-3, 1.0)
    cfg = pmg.MGConfig(policy="explicit", explicit_levels=1)
    hier = pmg.build_hierarchy(grid, params, cfg)
    assert hier.fine.op.uniform == (not variable)
    lay = hier.fine.layout
    w = lay.local_workers[0]
    h = hier.fine.op.handles[w].h
    assert lib.pmg_half_sweep_res_ok(h) == 1
    ua, fa = uni((nx, ny, nz), 1), uni((nx, ny, nz), 2)
    u, f = field(pmg, ua, lay), field(pmg, fa, lay)
    u_before = u.parts[w].data.clone()
    un = pmg.DistField.zeros(lay, nz)
    scratch = torch.empty(int(lib.pmg_partials_size()), dtype=torch.float64, device="cuda")
    nrm = torch.zeros(1, dtype=torch.float64, device="cuda")
    _lib.call("pmg_half_sweep_res", h, u.parts[w].ptr, un.parts[w].ptr, f.parts[w].ptr,
              C.c_void_p(scratch.data_ptr()), C.c_void_p(nrm.data_ptr()),
              C.c_void_p(torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    assert torch.equal(u.parts[w].data, u_before)          # input untouched
    r = pmg.gather_owned(hier.fine.op.residual(f, u))
    red = _red_mask(nx, ny, nz)
    want = float(np.sum(r[red] ** 2))
    assert abs(nrm.item() - want) <= 1e-12 * want
    ref = u.copy()
    hier.fine.smoother.half_sweep(ref, f, 0)
    got = pmg.gather_owned(un)
    assert np.array_equal(got[red], pmg.gather_owned(ref)[red])
    assert not np.any(got[~red])                             # black array untouched
    # ineligible levels are refused: uniform with nz = 32 (4-level
    # segments), variable with nz = 8 (not a multiple of 16)
    for g2 in (pmg.periodic_box(16, 32, 0.01), pmg.panel_grid(16, 8, flat_mode=True)):
        h2 = pmg.build_hierarchy(g2, pmg.toy_parameters(16, g2.nz, 1e-3, 1.0),
                                 pmg.MGConfig(policy="explicit", explicit_levels=1))
        w2 = h2.fine.layout.local_workers[0]
        assert lib.pmg_half_sweep_res_ok(h2.fine.op.handles[w2].h) == 0
        z = pmg.DistField.zeros(h2.fine.layout, g2.nz)
        z2 = pmg.DistField.zeros(h2.fine.layout, g2.nz)
        with pytest.raises(ValueError):
            _lib.call("pmg_half_sweep_res", h2.fine.op.handles[w2].h, z.parts[w2].ptr,
                      z2.parts[w2].ptr, z.parts[w2].ptr, C.c_void_p(scratch.data_ptr()),
                      C.c_void_p(nrm.data_ptr()), None)


@pytest.mark.parametrize("case", ["box256", "box96", "box80", "box128", "var128", "var256",
                                  "box2048"])
def test_lagged_norm_solve(pmg, case):
    """Native mg_solve with the lagged convergence norm against the plain
    one: equal iteration counts and iterates BIT FOR BIT (same kernels, the
    relaxed red values only land in the other red array), histories within
    1e-10 (the black cells' residual after an exact black line solve is
    rounding noise).  Odd and even cycle counts, repeated solves (the
    red-array parity follows the previous count) and maxiter cut-offs."""
    from paper_1307_2036_b200 import _lib, configs
    nx, nz, nlev = {"box256": (256, 128, 5), "box96": (64, 96, 3), "box80": (32, 80, 2),
                    "box128": (128, 128, 3), "var128": (128, 128, 3),
                    "var256": (256, 128, 5), "box2048": (2048, 128, 4)}[case]
    if case.startswith("var"):    # configs[4]-like: graded levels, omega^2(x, y)
        prob = configs.Problem(nx, nx, nz, 1e-3, 1.0, nlev, stretch=1.05, variable_omega=True)
        grid, params = prob.grid(), prob.params()
    else:
        grid = pmg.periodic_box(nx, nz, 0.01)
        params = pmg.toy_parameters(nx, nz, 1e-3, 1.0)
    fa = uni((nx, nx, nz), 9)
    # (the 2048^2 case -- a 4 GB fine level -- checks one tolerance only)
    for eps in ((1e-5,) if nx >= 2048 else (1e-5, 1e-7, 1e-9)):
        runs = {}
        for lag in (False, True):
            cfg = pmg.MGConfig(policy="explicit", explicit_levels=nlev, eps=eps, lagged_norm=lag)
            hier = pmg.build_hierarchy(grid, params, cfg)
            lay = hier.fine.layout
            assert _lib.load().pmg_half_sweep_res_ok(
                hier.fine.op.handles[lay.local_workers[0]].h) == 1
            f = pmg.scatter_owned(fa, lay)
            out = []
            for _ in range(3):      # the parity guess changes after the first solve
                u, rep = pmg.mg_solve(f, hier, cfg)
                out.append((rep.iterations, rep.converged, np.array(rep.residual_history),
                            pmg.gather_owned(u)))
                # the returned iterate's halo ring is current (the lagged
                # driver reads neighbours by wrap-around and refreshes the
                # ring once at the end)
                v = u.copy()
                pmg.halo_exchange(v)
                for w in u.parts:
                    assert torch.equal(u.parts[w].data, v.parts[w].data)
            for maxiter in (1, 2, 3):
                c2 = pmg.MGConfig(policy="explicit", explicit_levels=nlev, eps=1e-14,
                                  maxiter=maxiter, lagged_norm=lag)
                u, rep = pmg.mg_solve(f, hier, c2)
                out.append((rep.iterations, rep.converged, np.array(rep.residual_history),
                            pmg.gather_owned(u)))
            runs[lag] = out
        for a, b in zip(runs[False], runs[True]):
            assert a[0] == b[0] and a[1] == b[1]
            # ||f|| summed inside the first cycle's half-sweeps (other order)
            assert abs(a[2][0] - b[2][0]) <= 1e-14 * a[2][0]
            # the dropped black residual is ~1e-14 ||r0|| (rounding of the
            # exact black line solve): relative 1e-10 plus that floor
            assert np.all(np.abs(b[2] - a[2]) <= 1e-10 * a[2] + 1e-14 * a[2][0])
            assert np.array_equal(a[3], b[3])
    # f = 0: no cycles, u = 0, history [0] (multigrid.py:317-318), after a
    # solve that left a non-zero iterate behind
    cfg = pmg.MGConfig(policy="explicit", explicit_levels=nlev, eps=1e-5)
    hier = pmg.build_hierarchy(grid, params, cfg)
    f = pmg.scatter_owned(fa, hier.fine.layout)
    pmg.mg_solve(f, hier, cfg)
    u, rep = pmg.mg_solve(pmg.scatter_owned(np.zeros_like(fa), hier.fine.layout), hier, cfg)
    assert rep.iterations == 0 and rep.converged and rep.residual_history == [0.0]
    assert not np.any(pmg.gather_owned(u))


def test_red_residual_norm(pmg):
    """pmg_red_residual_norm = the sum of squares of pmg_residual's (bit-exact)
    residual over the red cells (the lagged driver's check-only norm)."""
    import ctypes as C
    from paper_1307_2036_b200 import _lib
    lib = _lib.load()
    nx, nz = 64, 128
    grid = pmg.periodic_box(nx, nz, 0.01)
    hier = pmg.build_hierarchy(grid, pmg.toy_parameters(nx, nz, 1e-3, 1.0),
                               pmg.MGConfig(policy="explicit", explicit_levels=1))
    lay = hier.fine.layout
    w = lay.local_workers[0]
    u, f = field(pmg, uni((nx, nx, nz), 4), lay), field(pmg, uni((nx, nx, nz), 5), lay)
    scratch = torch.empty(int(lib.pmg_partials_size()), dtype=torch.float64, device="cuda")
    nrm = torch.zeros(1, dtype=torch.float64, device="cuda")
    _lib.call("pmg_red_residual_norm", hier.fine.op.handles[w].h, f.parts[w].ptr,
              u.parts[w].ptr, C.c_void_p(scratch.data_ptr()), C.c_void_p(nrm.data_ptr()),
              C.c_void_p(torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    r = pmg.gather_owned(hier.fine.op.residual(f, u))
    want = float(np.sum(r[_red_mask(nx, nx, nz)] ** 2))
    assert abs(nrm.item() - want) <= 1e-13 * want


def test_predicted_check_matches(pmg, tmp_path):
    """The lagged driver's predicted check-only last norm (default) against
    PMG_NO_PREDICT=1, in a subprocess: same iterates bit for bit, same
    cycle counts, histories within rounding."""
    import subprocess
    import sys
    code = (
        "import sys, json, numpy as np; sys.path.insert(0, %r)\n"
        "import paper_1307_2036_b200 as pmg\n"
        "out = []\n"
        "for nx, nz, nl in ((256, 128, 5), (128, 128, 3)):\n"
        "    g = pmg.periodic_box(nx, nz, 0.01); p = pmg.toy_parameters(nx, nz, 1e-3, 1.0)\n"
        "    fa = np.random.default_rng(7).uniform(-1, 1, (nx, nx, nz))\n"
        "    for eps in (1e-5, 1e-8):\n"
        "        cfg = pmg.MGConfig(policy='explicit', explicit_levels=nl, eps=eps)\n"
        "        h = pmg.build_hierarchy(g, p, cfg)\n"
        "        f = pmg.scatter_owned(fa, h.fine.layout)\n"
        "        for _ in range(2):\n"
        "            u, rep = pmg.mg_solve(f, h, cfg)\n"
        "        np.save(%r + f'/u_{nx}_{eps}.npy', pmg.gather_owned(u))\n"
        "        out.append(rep.residual_history)\n"
        "print(json.dumps(out))\n") % (os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                        str(tmp_path))
    res = {}
    for tag, env in (("pred", {}), ("nopred", {"PMG_NO_PREDICT": "1"})):
        d = tmp_path / tag
        d.mkdir()
        r = subprocess.run([sys.executable, "-c", code.replace(str(tmp_path), str(d))],
                           capture_output=True, text=True, env={**os.environ, **env})
        assert r.returncode == 0, r.stderr[-2000:]
        import json
        res[tag] = (json.loads(r.stdout.strip().splitlines()[-1]), d)
    (ha, da), (hb, db) = res["pred"], res["nopred"]
    for a, b in zip(ha, hb):
        a, b = np.array(a), np.array(b)
        assert len(a) == len(b)
        assert np.all(np.abs(a - b) <= 1e-10 * b + 1e-14 * b[0])
    for fn in sorted(os.listdir(da)):
        assert np.array_equal(np.load(da / fn), np.load(db / fn)), fn


@pytest.mark.parametrize("par", [0, 1])
@pytest.mark.parametrize("mx,my,nz", [(32, 16, 16), (64, 8, 128), (4, 4, 8)])
def test_residual_restrict_red(pmg, par, mx, my, nz):
    """pmg_residual_restrict_red on a part of either parity (i0 = par): the
    coarse values equal the reference children sums of pmg_residual's
    (bit-exact) residual with the black children replaced by zero -- bit
    for bit."""
    import ctypes as C
    from paper_1307_2036_b200 import _lib
    from paper_1307_2036_b200.partition import DevField, LevelHandle, _stream
    rng = np.random.default_rng(3 + par)
    dr = rng.uniform(0.5, 1.5, nz)
    vprof = rng.uniform(0.5, 1.5, nz + 1)
    vol = dr.copy()

    def level(m, n, i0):
        one = np.ones(1)
        return LevelHandle(m, n, nz, i0, 0, 1e-3, 3.3e-2, dr, vprof, vol,
                           np.broadcast_to(one, (n, m + 1)), np.broadcast_to(one, (n + 1, m)),
                           np.broadcast_to(0.7 * one, (n, m)), np.broadcast_to(1.3 * one, (n, m)),
                           np.broadcast_to(4 * one, (n, m)))
    fine, coarse = level(mx, my, par), level(mx // 2, my // 2, 0)
    assert fine.parity == par
    u, f, r, cf = DevField(fine), DevField(fine), DevField(fine), DevField(coarse)
    u.load_owned(rng.uniform(-1, 1, (mx, my, nz)))
    f.load_owned(rng.uniform(-1, 1, (mx, my, nz)))
    st = _stream()
    _lib.call("pmg_halo_self", fine.h, u.ptr, 1, 1, st)
    _lib.call("pmg_residual", fine.h, f.ptr, u.ptr, r.ptr, None, None, st)
    assert _lib.load().pmg_residual_restrict_red_ok(fine.h) == 1
    _lib.call("pmg_residual_restrict_red", fine.h, coarse.h, f.ptr, u.ptr, cf.ptr, st)
    torch.cuda.synchronize()
    res = r.owned_array()
    i, j = np.meshgrid(np.arange(mx), np.arange(my), indexing="ij")
    red = (((i + par + j) % 2) == 0)[:, :, None]
    rr = np.where(red, res, 0.0)
    want = ((rr[0::2, 0::2] + rr[1::2, 0::2]) + rr[0::2, 1::2]) + rr[1::2, 1::2]
    assert np.array_equal(cf.owned_array(), want)
    # and the full restriction differs only by the black residual
    cfull = DevField(coarse)
    _lib.call("pmg_residual_restrict", fine.h, coarse.h, f.ptr, u.ptr, cfull.ptr, st)
    full = ((res[0::2, 0::2] + res[1::2, 0::2]) + res[0::2, 1::2]) + res[1::2, 1::2]
    assert np.array_equal(cfull.owned_array(), full)


def test_red_restrict_solve(pmg):
    """V-cycles with the red-only restriction against the full one on
    configs[1]'s shape at 256^2 x 128: equal cycle counts, histories and
    iterates within rounding (the dropped black residual is ~1e-16 of the
    red one), native and Python drivers bit-identical to each other."""
    from paper_1307_2036_b200 import multigrid as mgm
    nx, nz = 256, 128
    grid = pmg.periodic_box(nx, nz, 0.01)
    params = pmg.toy_parameters(nx, nz, 1e-3, 1.0)
    fa = uni((nx, nx, nz), 4)
    out = {}
    for red in (False, True):
        for native in (False, True):
            cfg = pmg.MGConfig(policy="explicit", explicit_levels=5, eps=1e-8,
                               red_restrict=red, lagged_norm=False)
            hier = pmg.build_hierarchy(grid, params, cfg)
            f = pmg.scatter_owned(fa, hier.fine.layout)
            mgm.USE_NATIVE = native
            try:
                u, rep = pmg.mg_solve(f, hier, cfg)
            finally:
                mgm.USE_NATIVE = True
            out[red, native] = (np.array(rep.residual_history), pmg.gather_owned(u))
    for red in (False, True):
        assert np.array_equal(out[red, False][0], out[red, True][0])
        assert np.array_equal(out[red, False][1], out[red, True][1])
    (h0, u0), (h1, u1) = out[False, True], out[True, True]
    assert len(h0) == len(h1)
    # the black children's residual is rounding noise (~1e-16 ||r0||): the
    # histories agree to 1e-10 relative above a 1e-14 ||r0|| floor
    assert np.all(np.abs(h1 - h0) <= 1e-10 * h0 + 1e-14 * h0[0])
    assert np.max(np.abs(u1 - u0)) <= 1e-10 * np.max(np.abs(u0))


@pytest.mark.parametrize("nx", [256, 512, 1024, 2048])
def test_band_half_sweep_matches_exact(pmg, nx):
    """The TMA band half-sweep (nx = 256 ... 2048 at nz = 128, halo-ring
    mode) against the exact sequential-Thomas smoother (bit-identical to
    the reference): within the fast mode's 1e-12 (tests/test_smoother.py:48)."""
    from paper_1307_2036_b200 import configs
    prob = configs.Problem(nx, nx, 128, 1e-3, 1.0, 1)
    hier = pmg.build_hierarchy(prob.grid(), prob.params(),
                               pmg.MGConfig(policy="explicit", explicit_levels=1))
    lay = hier.fine.layout
    f = pmg.scatter_owned(configs.rhs(prob.nx, prob.ny, prob.nz, 0), lay)
    u0 = pmg.scatter_owned(uni((prob.nx, prob.ny, prob.nz), 11), lay)
    pmg.halo_exchange(u0)
    out = []
    for exact in (False, True):
        u = u0.copy()
        if exact:
            with pmg.exact_smoother():
                hier.fine.smoother.half_sweep(u, f, 1)
                hier.fine.smoother.half_sweep(u, f, 0)
        else:
            hier.fine.smoother.half_sweep(u, f, 1)
            hier.fine.smoother.half_sweep(u, f, 0)
        out.append(pmg.gather_owned(u))
    fast, ex = out
    assert np.max(np.abs(fast - ex)) <= 1e-12 * np.max(np.abs(ex))


def test_field_alloc_and_prolong_add(pmg):
    """pmg_field_alloc: a zeroed field of pmg_level_field_doubles doubles,
    released by pmg_field_free; pmg_prolong_add = pmg_prolong(add = 1)
    bit for bit (SURVEY 8b's names)."""
    import ctypes as C
    from paper_1307_2036_b200 import _lib
    lib = _lib.load()
    nx, nz = 64, 16
    grid = pmg.periodic_box(nx, nz, 0.01)
    hier = pmg.build_hierarchy(grid, pmg.toy_parameters(nx, nz, 1e-3, 1.0),
                               pmg.MGConfig(policy="explicit", explicit_levels=2))
    lay, cl = hier.fine.layout, hier.levels[1].layout
    w = lay.local_workers[0]
    fh, ch = hier.fine.op.handles[w].h, hier.levels[1].op.handles[w].h
    n = int(lib.pmg_level_field_doubles(fh))
    p = C.c_void_p()
    _lib.call("pmg_field_alloc", fh, C.byref(p))
    assert p.value
    got = torch.empty(n, dtype=torch.float64, device="cuda")
    st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    _lib.call("pmg_copy", fh, C.c_void_p(got.data_ptr()), p, st)
    torch.cuda.synchronize()
    assert got.abs().max().item() == 0.0
    _lib.call("pmg_field_free", p)
    _lib.call("pmg_field_free", C.c_void_p(None))
    cu = field(pmg, uni((nx // 2, nx // 2, nz), 8), cl)
    pmg.halo_exchange(cu)
    a, b = field(pmg, uni((nx, nx, nz), 9), lay), field(pmg, uni((nx, nx, nz), 9), lay)
    _lib.call("pmg_prolong", fh, ch, cu.parts[w].ptr, a.parts[w].ptr, 1, st)
    _lib.call("pmg_prolong_add", fh, ch, cu.parts[w].ptr, b.parts[w].ptr, st)
    torch.cuda.synchronize()
    assert np.array_equal(pmg.gather_owned(a), pmg.gather_owned(b))


@pytest.mark.parametrize("name", ["ops_config", "ops_variable"])
def test_mode_switch_recaptures_graphs(pmg, name):
    """A fast-mode solve followed by an exact-mode solve on the SAME hierarchy
    and buffers must run the exact kernels (graphs captured under the fast
    mode are not replayed): bit-identical to an exact solve on a fresh
    hierarchy, and the exact single V-cycle equals the reference's."""
    g, grid, params, cfg, hier = setup(pmg, name)
    nx, nz = grid.nx, grid.nz
    fg = uni((nx, nx, nz), 2)
    f = pmg.scatter_owned(fg, hier.fine.layout)
    u = pmg.DistField.zeros(hier.fine.layout, nz)
    for _ in range(2):
        pmg.mg_solve(f, hier, cfg, out=u)          # fast mode, graphs cached
    with pmg.exact_smoother():
        u, rep = pmg.mg_solve(f, hier, cfg, out=u)
        got = pmg.gather_owned(u)
        _, _, _, _, hier2 = setup(pmg, name)
        f2 = pmg.scatter_owned(fg, hier2.fine.layout)
        u2, rep2 = pmg.mg_solve(f2, hier2, cfg)
        want = pmg.gather_owned(u2)
    assert rep.residual_history == rep2.residual_history
    assert np.array_equal(got, want)
    # and back: the fast mode is restored on the same buffers
    u3, rep3 = pmg.mg_solve(f, hier, cfg, out=u)
    assert rep3.iterations == rep.iterations


@pytest.mark.parametrize("nx,ny,nz,slabs", [(64, 64, 32, 1), (128, 64, 32, 4), (256, 256, 128, 8)])
def test_solve_pipeline_matches_direct(pmg, nx, ny, nz, slabs):
    """SolvePipeline.run (pinned host blocks in, host solutions out, the
    block converted slab by slab while the next slab is on the bus) returns
    exactly what scatter_owned -> mg_solve -> gather_owned returns, for one
    step per call and for a stream of steps; the slab entry points equal the
    whole-block layout conversion."""
    import ctypes as C
    from paper_1307_2036_b200 import _lib
    from paper_1307_2036_b200.pipeline import SolvePipeline
    grid = pmg.periodic_box(nx, nz, 0.01, ny=ny)
    params = pmg.toy_parameters(nx, nz, 1e-3, 1.0)
    cfg = pmg.MGConfig(policy="explicit", explicit_levels=4, eps=1e-5)
    hier = pmg.build_hierarchy(grid, params, cfg, pmg.Decomposition(nx, 1, ny=ny))
    fs = [uni((nx, ny, nz), 40 + s) for s in range(3)]
    direct = []
    for fg in fs:
        u, rep = pmg.mg_solve(field(pmg, fg, hier.fine.layout), hier, cfg)
        direct.append((pmg.gather_owned(u), rep))
    pipe = SolvePipeline(hier, cfg, nz, slabs=slabs, min_slab_bytes=1)
    assert len(pipe.slabs) == slabs and pipe.slabs[0][0] == 0 and pipe.slabs[-1][1] == nx
    fh = [torch.from_numpy(f).pin_memory() for f in fs]
    uh = [torch.empty((nx, ny, nz), dtype=torch.float64).pin_memory() for _ in fs]
    reps = pipe.run(fh, uh)                       # a stream of steps
    for (ud, rd), u, r in zip(direct, uh, reps):
        assert r.iterations == rd.iterations and r.residual_history == rd.residual_history
        assert np.array_equal(u.numpy(), ud)
    for k in range(3):                            # one step per call
        uh[k].zero_()
        (r,) = pipe.run([fh[k]], [uh[k]])
        assert r.residual_history == direct[k][1].residual_history
        assert np.array_equal(uh[k].numpy(), direct[k][0])
    # slab entry points against the whole-block conversion
    lay = hier.fine.layout
    (w,) = lay.local_workers
    a, b = pmg.DistField.zeros(lay, nz), pmg.DistField.zeros(lay, nz)
    src = torch.from_numpy(fs[0]).cuda()
    st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    h = a.parts[w].geom.h
    _lib.call("pmg_from_ref_layout", h, C.c_void_p(src.data_ptr()), a.parts[w].ptr, st)
    for i0, i1 in ((0, 32), (32, 40), (40, nx)):
        _lib.call("pmg_from_ref_layout_slab", h, C.c_void_p(src.data_ptr()), b.parts[w].ptr,
                  i0, i1, st)
    assert torch.equal(a.parts[w].data, b.parts[w].data)
    back = torch.zeros_like(src)
    for i0, i1 in ((0, 7), (7, 64), (64, nx)):
        _lib.call("pmg_to_ref_layout_slab", h, a.parts[w].ptr, C.c_void_p(back.data_ptr()),
                  i0, i1, st)
    assert torch.equal(back, src)
    with pytest.raises(ValueError):
        _lib.call("pmg_to_ref_layout_slab", h, a.parts[w].ptr, C.c_void_p(back.data_ptr()),
                  0, nx + 1, st)
