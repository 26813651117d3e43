"""Native multi-part driver (pmg_phier, pmg_parts.cu) on the device.

* In-process decompositions (2x1, 1x2, 2x2, 4x2; periodic and mirror): the
  native driver -- every part's V-cycle, the halo exchanges and the
  worker-order reductions captured in one graph per cycle -- gives the
  Python multi-part driver's iterates and histories bit for bit, with and
  without boundary-first overlap (frame regions relaxed first, their halo
  exchange on a second stream while the interior relaxes); and it agrees
  with the single-part solve of the same global grid to the reference's
  partition-invariance tolerance (tests/test_partition.py:122-154).
* The NCCL transport: a one-rank library communicator whose part is its
  own periodic neighbour sends every halo strip to itself through
  ncclSend / ncclRecv (captured in the cycle graph) and reduces through
  ncclAllGather; iterates equal the in-process driver's bit for bit.  (Only
  one GPU is available; ranks on separate GPUs run the same code with other
  peers -- the per-pair message order is checked on CPU in test_parts.py.)
"""

import ctypes as C

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pmg():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1307_2036_b200 as m
    return m


def uni(shape, seed):
    return np.random.default_rng(seed).uniform(-1.0, 1.0, size=shape)


def solve(pmg, grid, params, fg, px, py, native, overlap=True, levels=4, exact=False,
          lagged=True):
    from paper_1307_2036_b200 import multigrid as mg
    cfg = pmg.MGConfig(policy="explicit", explicit_levels=levels, overlap=overlap,
                       lagged_norm=lagged)
    dec = pmg.Decomposition(grid.nx, px * py, ny=grid.ny, px=px, py=py)
    hier = pmg.build_hierarchy(grid, params, cfg, dec)
    f = pmg.scatter_owned(fg, hier.fine.layout)
    prev = mg.USE_NATIVE_PARTS
    mg.USE_NATIVE_PARTS = native
    try:
        with pmg.exact_smoother(exact):
            u, rep = pmg.mg_solve(f, hier, cfg)
            # a second solve replays the captured graphs
            u2, rep2 = pmg.mg_solve(f, hier, cfg)
    finally:
        mg.USE_NATIVE_PARTS = prev
    assert rep2.residual_history == rep.residual_history
    g = pmg.gather_owned(u)
    assert np.array_equal(g, pmg.gather_owned(u2))
    return g, rep, hier


CASES = [  # (nx, ny, nz, px, py, periodic)
    (512, 256, 32, 2, 1, True),
    (256, 512, 32, 1, 2, True),
    (512, 512, 32, 2, 2, True),
    (1024, 512, 32, 4, 2, True),
    (512, 512, 32, 2, 2, False),
    (64, 32, 16, 2, 2, True),
]


@pytest.mark.parametrize("nx,ny,nz,px,py,periodic", CASES)
def test_native_parts_match_python(pmg, nx, ny, nz, px, py, periodic):
    if periodic:
        grid = pmg.periodic_box(nx, nz, 0.01, ny=ny)
    else:
        grid = pmg.panel_grid(nx, nz, flat_mode=True)
    params = pmg.toy_parameters(nx, nz, 1e-3, 1.0)
    fg = uni((nx, ny, nz), 3)
    levels = 4 if min(nx, ny) >= 64 else 3
    ref, rep_ref, _ = solve(pmg, grid, params, fg, px, py, native=False, levels=levels)
    for overlap, lagged in ((True, False), (False, False), (True, True), (False, True)):
        got, rep, hier = solve(pmg, grid, params, fg, px, py, native=True, overlap=overlap,
                               levels=levels, lagged=lagged)
        assert rep.iterations == rep_ref.iterations
        # iterates bit for bit (the lagged norm only moves where the residual
        # norm is summed and where the red values land)
        assert np.array_equal(got, ref), (overlap, lagged)
        if not lagged:
            assert rep.residual_history == rep_ref.residual_history, overlap
        else:
            # ||f|| summed inside the first cycle's sweeps; the black cells'
            # rounding-level residual dropped (test_lagged_norm_solve's bar)
            a, b = np.array(rep_ref.residual_history), np.array(rep.residual_history)
            assert abs(a[0] - b[0]) <= 1e-14 * a[0]
            assert np.all(np.abs(b - a) <= 1e-10 * a + 1e-14 * a[0])
        # the native driver really ran: its graphs replayed library kernels
        nh = hier.native_parts(pmg.MGConfig(policy="explicit", explicit_levels=levels,
                                            overlap=overlap, lagged_norm=lagged))
        assert nh.replayed_launches() > 0 and nh.exchanges() > 0
    # partition invariance against the single-part solve (<= 1e-10)
    one, rep1, _ = solve(pmg, grid, params, fg, 1, 1, native=True, levels=levels)
    assert rep1.iterations == rep.iterations
    h, h1 = np.array(rep.residual_history), np.array(rep1.residual_history)
    assert np.max(np.abs(h - h1) / (h1 + 1e-13 * h1[0])) <= 1e-10
    assert np.max(np.abs(got - one)) <= 1e-10 * np.max(np.abs(one))


def test_native_parts_exact_mode(pmg):
    """Exact smoother: no tile regions (overlap off by construction), the
    same native sequence, bit-identical to the Python driver."""
    grid = pmg.periodic_box(128, 16, 0.01)
    params = pmg.toy_parameters(128, 16, 1e-3, 1.0)
    fg = uni((128, 128, 16), 4)
    ref, r0, _ = solve(pmg, grid, params, fg, 2, 2, native=False, exact=True)
    got, r1, _ = solve(pmg, grid, params, fg, 2, 2, native=True, exact=True)
    assert r0.residual_history == r1.residual_history
    assert np.array_equal(got, ref)


def _nccl_self_hier(pmg, hier, cfg, lagged=0, nbr=(0, 0, 0, 0)):
    from paper_1307_2036_b200 import _lib
    lib = _lib.load()
    if not lib.pmg_comm_available():
        pytest.skip("libnccl.so.2 not loadable")
    uid = (C.c_ubyte * 128)()
    _lib.call("pmg_comm_unique_id", uid)
    comm = C.c_void_p()
    _lib.call("pmg_comm_create", uid, 1, 0, C.byref(comm))
    lay = hier.fine.layout
    (w,) = lay.local_workers
    levels = [lev.op.handles[w].h.value for lev in hier.levels]
    arr = (C.c_void_p * len(levels))(*levels)
    parts = (_lib.PartDesc * 1)()
    parts[0].worker = 0
    for a in range(4):
        parts[0].nbr[a] = nbr[a]     # 0: its own periodic neighbour, through NCCL; -1: mirror
        parts[0].diag[a] = 0 if nbr[a & 1] >= 0 and nbr[2 + (a >> 1)] >= 0 else -1
    d = _lib.MGDesc(cfg.nu_pre, cfg.nu_post, cfg.resolved_coarse_sweeps(), 1.0, 1, 1, lagged, 1)
    h = C.c_void_p()
    _lib.call("pmg_phier_create", arr, len(levels), 1, parts, C.byref(d), comm, 256,
              C.byref(h))
    return lib, comm, h, w


@pytest.mark.parametrize("lagged", [0, 1])
@pytest.mark.parametrize("nx,nz", [(512, 32), (64, 16)])
def test_nccl_self_exchange_matches(pmg, nx, nz, lagged):
    from paper_1307_2036_b200 import _lib, multigrid as mg
    grid = pmg.periodic_box(nx, nz, 0.01)
    params = pmg.toy_parameters(nx, nz, 1e-3, 1.0)
    cfg = pmg.MGConfig(policy="explicit", explicit_levels=4 if nx >= 64 else 3)
    hier = pmg.build_hierarchy(grid, params, cfg)
    fg = uni((nx, nx, nz), 5)
    f = pmg.scatter_owned(fg, hier.fine.layout)
    # reference: the Python single-part driver (pmg_halo_self exchanges)
    prev = mg.USE_NATIVE
    mg.USE_NATIVE = False
    try:
        uref, rref = pmg.mg_solve(f, hier, cfg)
    finally:
        mg.USE_NATIVE = prev
    lib, comm, h, w = _nccl_self_hier(pmg, hier, cfg, lagged)
    try:
        u = pmg.DistField.zeros(hier.fine.layout, nz)
        hist = np.zeros(cfg.maxiter + 1)
        iters, conv = C.c_int(), C.c_int()
        fp = (C.c_void_p * 1)(f.parts[w].data.data_ptr())
        up = (C.c_void_p * 1)(u.parts[w].data.data_ptr())
        st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
        for _ in range(3):   # capture, then replay (the lagged driver alternates red arrays)
            _lib.call("pmg_phier_mg_solve", h, fp, up, float(cfg.eps), int(cfg.maxiter),
                      hist.ctypes.data_as(C.c_void_p), C.byref(iters), C.byref(conv), st)
            assert iters.value == rref.iterations and conv.value == 1
            got = hist[:iters.value + 1]
            a = np.array(rref.residual_history)
            if lagged:
                assert np.all(np.abs(got - a) <= 1e-10 * a + 1e-14 * a[0])
            else:
                assert got.tolist() == rref.residual_history
            assert np.array_equal(pmg.gather_owned(u), pmg.gather_owned(uref))
        assert lib.pmg_phier_exchanges(h) > 0
        # the standalone exchange and dot entry points over NCCL
        v = pmg.scatter_owned(uni((nx, nx, nz), 6), hier.fine.layout)
        ref = v.copy()
        pmg.halo_exchange(ref)
        vp = (C.c_void_p * 1)(v.parts[w].data.data_ptr())
        _lib.call("pmg_phier_halo_exchange", h, 0, vp, st)
        assert torch.equal(v.parts[w].data, ref.parts[w].data)
        out = torch.zeros(1, dtype=torch.float64, device="cuda")
        _lib.call("pmg_phier_dot", h, 0, vp, vp, C.c_void_p(out.data_ptr()), st)
        assert float(out.item()) == pytest.approx(pmg.dist_dot(v, v), rel=1e-14)
    finally:
        lib.pmg_phier_destroy(h)
        lib.pmg_comm_destroy(comm)


@pytest.mark.parametrize("px,py", [(2, 2), (2, 1)])
def test_native_parts_variable_coefficients(pmg, px, py, monkeypatch):
    """configs[4]'s problem family (graded levels, omega^2(x, y)) on the
    native multi-part driver, with boundary-first overlap on the fine
    level (threshold lowered to the 256-column parts: the variable band
    kernel walks the frame and interior regions): iterates bit-identical
    to the Python multi-part driver, histories within the lagged-norm
    bar, and the single-part solve within the partition-invariance bar."""
    from paper_1307_2036_b200 import configs, multigrid as mg
    monkeypatch.setattr(mg, "OVERLAP_NX", 256)
    prob = configs.Problem(512, 512, 128, 1e-3, 1.0, 5, stretch=1.05, variable_omega=True)
    grid, params = prob.grid(), prob.params()
    fg = configs.rhs(512, 512, 128, 0)
    ref, rep_ref, _ = solve(pmg, grid, params, fg, px, py, native=False, levels=5)
    got, rep, _ = solve(pmg, grid, params, fg, px, py, native=True, levels=5)
    assert rep.iterations == rep_ref.iterations
    assert np.array_equal(got, ref)
    a, b = np.array(rep_ref.residual_history), np.array(rep.residual_history)
    assert np.all(np.abs(b - a) <= 1e-10 * a + 1e-14 * a[0])
    one, rep1, _ = solve(pmg, grid, params, fg, 1, 1, native=True, levels=5)
    assert rep1.iterations == rep.iterations
    assert np.max(np.abs(got - one)) <= 1e-10 * np.max(np.abs(one))


def _cg(pmg, f, op, pre, native):
    from paper_1307_2036_b200 import krylov
    prev = krylov.USE_NATIVE_PARTS
    krylov.USE_NATIVE_PARTS = native
    try:
        return pmg.pcg_solve(f, op, pre, eps=1e-8, maxiter=2000)
    finally:
        krylov.USE_NATIVE_PARTS = prev


@pytest.mark.parametrize("precond", ["ssor", "identity"])
@pytest.mark.parametrize("nx,ny,px,py,periodic", [(128, 128, 2, 2, True), (256, 128, 4, 2, True),
                                                  (128, 128, 2, 2, False)])
def test_native_parts_pcg(pmg, nx, ny, px, py, periodic, precond):
    """The multi-part CG driver (pmg_phier_pcg_solve): iterates and
    histories bit-identical to the Python multi-part pcg_solve, and the
    single-part solve's within the partition-invariance bar."""
    nz = 16
    grid = (pmg.periodic_box(nx, nz, 0.01, ny=ny) if periodic
            else pmg.panel_grid(nx, nz, flat_mode=True))
    ny = grid.ny
    params = pmg.toy_parameters(nx, nz, 1e-3, 1.0)
    fg = uni((nx, ny, nz), 8)
    out = {}
    for parts in ((px, py), (1, 1)):
        dec = pmg.Decomposition(nx, parts[0] * parts[1], ny=ny, px=parts[0], py=parts[1])
        op = pmg.PanelOperator(grid, params, dec.layout(nx))
        pre = (pmg.SSORPreconditioner(pmg.LineSmoother(op)) if precond == "ssor"
               else pmg.IdentityPreconditioner())
        f = pmg.scatter_owned(fg, op.layout)
        for native in ((True, False) if parts != (1, 1) else (False,)):
            u, rep = _cg(pmg, f, op, pre, native)
            out[(parts, native)] = (rep, pmg.gather_owned(u))
    (rn, un), (rp, up) = out[((px, py), True)], out[((px, py), False)]
    assert rn.iterations == rp.iterations and rn.converged
    assert rn.residual_history == rp.residual_history
    assert np.array_equal(un, up)
    r1, u1 = out[((1, 1), False)]
    assert r1.iterations == rn.iterations
    h, h1 = np.array(rn.residual_history), np.array(r1.residual_history)
    assert np.max(np.abs(h - h1) / (h1 + 1e-13 * h1[0])) <= 1e-10
    assert np.max(np.abs(un - u1)) <= 1e-10 * np.max(np.abs(u1))


def _random_ring(pmg, lay, nz, seed):
    """A field whose every double -- owned cells, halo ring, padding -- is random."""
    v = pmg.DistField.zeros(lay, nz)
    g = torch.Generator(device="cuda").manual_seed(seed)
    for part in v.parts.values():
        part.data.copy_(torch.rand(part.data.shape, dtype=torch.float64, device="cuda",
                                   generator=g))
    return v


@pytest.mark.parametrize("nx,ny,nz,px,py,periodic", [
    (64, 64, 8, 2, 2, True), (64, 64, 8, 2, 2, False), (64, 32, 8, 2, 1, True),
    (64, 64, 8, 2, 1, False), (64, 64, 8, 1, 2, False), (128, 64, 8, 4, 2, True),
    (128, 128, 8, 4, 2, False)])
def test_single_phase_exchange_in_process(pmg, nx, ny, nz, px, py, periodic):
    """The native driver's one-launch exchange (faces and corner columns
    resolved x first, then y) leaves the whole halo ring as the two-phase
    exchange of partition.py:158-191 (pack / unpack entry points, x faces
    then y faces over the extended range) does, bit for bit."""
    from paper_1307_2036_b200 import _lib
    grid = (pmg.periodic_box(nx, nz, 0.01, ny=ny) if periodic
            else pmg.panel_grid(nx, nz, flat_mode=True))
    params = pmg.toy_parameters(nx, nz, 1e-3, 1.0)
    cfg = pmg.MGConfig(policy="explicit", explicit_levels=2)
    dec = pmg.Decomposition(nx, px * py, ny=ny, px=px, py=py)
    hier = pmg.build_hierarchy(grid, params, cfg, dec)
    nh = hier.native_parts(cfg)
    st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    for level in (0, 1):
        lay = hier.levels[level].layout
        v = _random_ring(pmg, lay, nz, 11 + level)
        ref = v.copy()
        pmg.halo_exchange(ref)
        _lib.call("pmg_phier_halo_exchange", nh.h, level, nh.ptrs(v), st)
        for w in lay.local_workers:
            assert torch.equal(v.parts[w].data, ref.parts[w].data), (level, w)


@pytest.mark.parametrize("nbr", [(0, 0, 0, 0), (-1, -1, 0, 0), (0, 0, -1, -1), (-1, -1, -1, -1)])
def test_single_phase_exchange_nccl_self(pmg, nbr):
    """The NCCL form of the exchange (one pack, one group of up to 8 sends
    and 8 receives, one unpack) with a one-rank communicator: the part is
    its own neighbour across the sides marked 0 and mirrored across the
    others -- every corner rule (diagonal message, the y strip's extended
    position, the x strip's end, own cell) against the two-phase exchange
    built from the pack / unpack entry points."""
    from paper_1307_2036_b200 import _lib
    nx, nz = 64, 8
    grid = pmg.periodic_box(nx, nz, 0.01)
    params = pmg.toy_parameters(nx, nz, 1e-3, 1.0)
    cfg = pmg.MGConfig(policy="explicit", explicit_levels=2)
    hier = pmg.build_hierarchy(grid, params, cfg)
    lib, comm, h, w = _nccl_self_hier(pmg, hier, cfg, 0, nbr)
    opp = (1, 0, 3, 2)
    try:
        st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
        for level in (0, 1):
            lay = hier.levels[level].layout
            v = _random_ring(pmg, lay, nz, 21 + level)
            ref = v.copy()
            part = ref.parts[w]
            for faces in ((0, 1), (2, 3)):
                for face in faces:
                    if nbr[face] < 0:
                        _lib.call("pmg_unpack_face", part.geom.h, part.ptr, face, None, 1, st)
                        continue
                    n = int(lib.pmg_face_doubles(part.geom.h, face))
                    buf = torch.empty(n, dtype=torch.float64, device="cuda")
                    _lib.call("pmg_pack_face", part.geom.h, part.ptr, opp[face],
                              C.c_void_p(buf.data_ptr()), st)
                    _lib.call("pmg_unpack_face", part.geom.h, part.ptr, face,
                              C.c_void_p(buf.data_ptr()), 0, st)
            vp = (C.c_void_p * 1)(v.parts[w].data.data_ptr())
            _lib.call("pmg_phier_halo_exchange", h, level, vp, st)
            assert torch.equal(v.parts[w].data, part.data), (level, nbr)
    finally:
        lib.pmg_phier_destroy(h)
        lib.pmg_comm_destroy(comm)
