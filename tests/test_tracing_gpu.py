"""Tracing mode on the device (tracing.py, pmg_set_tracing): every driver
-- the C++ single-part and multi-part drivers and the Python graph driver
-- reports one device time per V-cycle, inside the solve's wall time, and
tracing changes no result bit (the NVTX ranges and the event pair around
each replay are host-side)."""

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


@pytest.mark.parametrize("driver", ["native", "parts", "python"])
def test_cycle_times(pmg, driver, monkeypatch):
    from paper_1307_2036_b200 import multigrid as mg
    nx, nz = 256, 32
    grid = pmg.periodic_box(nx, nz, 0.01)
    params = pmg.toy_parameters(nx, nz, 1e-3, 1.0)
    cfg = pmg.MGConfig(policy="explicit", explicit_levels=5)
    parts = 4 if driver == "parts" else 1
    dec = pmg.Decomposition(nx, parts, ny=nx, px=2 if parts == 4 else 1,
                            py=2 if parts == 4 else 1)
    hier = pmg.build_hierarchy(grid, params, cfg, dec)
    if driver == "python":
        monkeypatch.setattr(mg, "USE_NATIVE", False)
    fg = np.random.default_rng(2).uniform(-1, 1, (nx, nx, nz))
    f = pmg.scatter_owned(fg, hier.fine.layout)
    u0, r0 = pmg.mg_solve(f, hier, cfg)
    assert r0.cycle_times_ms == []
    with pmg.tracing():
        u1, r1 = pmg.mg_solve(f, hier, cfg)
    assert r1.residual_history == r0.residual_history
    assert np.array_equal(pmg.gather_owned(u1), pmg.gather_owned(u0))
    t = np.array(r1.cycle_times_ms)
    assert len(t) == r1.iterations and np.all(t > 0.0)
    assert t.sum() <= 1e3 * r1.wall_time * 1.05 + 0.1
    # untraced again: no times
    _, r2 = pmg.mg_solve(f, hier, cfg)
    assert r2.cycle_times_ms == []
