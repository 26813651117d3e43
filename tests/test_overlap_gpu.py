"""Boundary-first relaxation (needs a B200): a half-sweep split into the
tile regions a multi-part sweep relaxes separately -- the rows and strips
holding the part's boundary columns (the "frame"), then the interior --
gives the same values, bit for bit, as one whole-part call.  This is the
property the overlapped halo exchange rests on: the frame's
values are final before the interior starts, and neither region reads a
value the other writes (a half-sweep reads only the other colour)."""

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


def frame_and_interior(nstrip, ny):
    """(rx0, rxs, rxn, ry0, rys, ryn) regions as the multi-part driver
    issues them: row 0 and row ny-1 (all strips), the first and last strip
    of rows 1 .. ny-2, then the interior."""
    return [(0, 1, nstrip, 0, 1, 1), (0, 1, nstrip, ny - 1, 1, 1),
            (0, max(nstrip - 1, 1), 2 if nstrip > 1 else 1, 1, 1, ny - 2),
            (1, 1, nstrip - 2, 1, 1, ny - 2)]


def test_strided_rows_match_whole(pmg):
    """Row strides (a region of non-adjacent rows) run on the register
    kernel: same values as that kernel's whole-part sweep (a level below
    the TMA band kernel's sizes)."""
    from paper_1307_2036_b200 import _lib
    nx, nz = 128, 32
    grid = pmg.periodic_box(nx, nz, 0.01)
    op = pmg.PanelOperator(grid, pmg.toy_parameters(nx, nz, 1e-3, 1.0),
                           pmg.Decomposition(nx, 1).layout(nx))
    (w, h), = op.handles.items()
    rng = np.random.default_rng(8)
    u0 = pmg.scatter_owned(rng.uniform(-1, 1, (nx, nx, nz)), op.layout)
    pmg.halo_exchange(u0)
    f = pmg.scatter_owned(rng.uniform(-1, 1, (nx, nx, nz)), op.layout)
    st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    a, b = u0.copy(), u0.copy()
    _lib.call("pmg_half_sweep", h.h, a.parts[w].ptr, f.parts[w].ptr, 0, 1.0, 0, 0, 1.0, st)
    for reg in ((0, 1, 2, 0, 2, nx // 2), (0, 1, 2, 1, 2, nx // 2)):   # even rows, odd rows
        _lib.call("pmg_half_sweep_region", h.h, b.parts[w].ptr, f.parts[w].ptr, 0, 1.0, 0, 0,
                  1.0, *reg, st)
    assert torch.equal(a.parts[w].data, b.parts[w].data)


@pytest.mark.parametrize("nx,ny,nz", [(256, 64, 128), (512, 512, 128), (1024, 256, 128),
                                      (128, 64, 32), (2048, 16, 128)])
def test_region_sweep_matches_whole(pmg, nx, ny, nz):
    from paper_1307_2036_b200 import _lib
    lib = _lib.load()
    grid = pmg.periodic_box(nx, nz, 0.01, ny=ny) if ny != nx else pmg.periodic_box(nx, nz, 0.01)
    params = pmg.toy_parameters(nx, nz, 1e-3, 1.0)
    op = pmg.PanelOperator(grid, params, pmg.Decomposition(nx, 1, ny=ny).layout(nx))
    (w, h), = op.handles.items()
    assert lib.pmg_half_sweep_region_ok(h.h) == 1
    rng = np.random.default_rng(7)
    u0 = pmg.scatter_owned(rng.uniform(-1, 1, (nx, ny, nz)), op.layout)
    pmg.halo_exchange(u0)
    f = pmg.scatter_owned(rng.uniform(-1, 1, (nx, ny, nz)), op.layout)
    nstrip = ((nx + 1) // 2 + 31) // 32
    st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    for color in (0, 1):
        for rho, zs, nbz in ((1.0, 0, 0), (1.3, 0, 0), (1.0, 1, 1), (1.2, 1, 0)):
            a, b = u0.copy(), u0.copy()
            _lib.call("pmg_half_sweep", h.h, a.parts[w].ptr, f.parts[w].ptr, color, rho, zs,
                      nbz, 1.0, st)
            for reg in frame_and_interior(nstrip, ny):
                _lib.call("pmg_half_sweep_region", h.h, b.parts[w].ptr, f.parts[w].ptr, color,
                          rho, zs, nbz, 1.0, *reg, st)
            assert torch.equal(a.parts[w].data, b.parts[w].data), (color, rho, zs, nbz)
    # a region outside the part is refused
    with pytest.raises(ValueError):
        _lib.call("pmg_half_sweep_region", h.h, u0.parts[w].ptr, f.parts[w].ptr, 0, 1.0, 0, 0,
                  1.0, 0, 1, nstrip + 1, 0, 1, ny, st)


@pytest.mark.parametrize("nx,ny", [(256, 64), (512, 512), (1024, 256), (2048, 16)])
def test_variable_region_sweep_matches_whole(pmg, nx, ny):
    """configs[4]'s level family (graded dz, omega^2(x, y)): the variable
    band kernel walks the same regions, bit for bit the whole-part sweep;
    strided rows and zero neighbours with rho != 1 are refused (the band
    kernel does not run them)."""
    from paper_1307_2036_b200 import _lib, configs
    lib = _lib.load()
    nz = 128
    prob = configs.Problem(nx, ny, nz, 1e-3, 1.0, 4, stretch=1.05, variable_omega=True)
    op = pmg.PanelOperator(prob.grid(), prob.params(),
                           pmg.Decomposition(nx, 1, ny=ny).layout(nx))
    (w, h), = op.handles.items()
    assert lib.pmg_half_sweep_region_ok(h.h) == 1
    rng = np.random.default_rng(11)
    u0 = pmg.scatter_owned(rng.uniform(-1, 1, (nx, ny, nz)), op.layout)
    pmg.halo_exchange(u0)
    f = pmg.scatter_owned(rng.uniform(-1, 1, (nx, ny, nz)), op.layout)
    nstrip = ((nx + 1) // 2 + 31) // 32
    st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    for color in (0, 1):
        for rho, zs, nbz in ((1.0, 0, 0), (1.3, 0, 0), (1.0, 0, 1), (1.2, 1, 0)):
            a, b = u0.copy(), u0.copy()
            _lib.call("pmg_half_sweep", h.h, a.parts[w].ptr, f.parts[w].ptr, color, rho, zs,
                      nbz, 1.0, st)
            for reg in frame_and_interior(nstrip, ny):
                _lib.call("pmg_half_sweep_region", h.h, b.parts[w].ptr, f.parts[w].ptr, color,
                          rho, zs, nbz, 1.0, *reg, st)
            assert torch.equal(a.parts[w].data, b.parts[w].data), (color, rho, zs, nbz)
    with pytest.raises(ValueError):
        _lib.call("pmg_half_sweep_region", h.h, u0.parts[w].ptr, f.parts[w].ptr, 0, 1.0, 0, 0,
                  1.0, 0, 1, nstrip, 0, 2, ny // 2, st)
    with pytest.raises(ValueError):
        _lib.call("pmg_half_sweep_region", h.h, u0.parts[w].ptr, f.parts[w].ptr, 0, 1.3, 0, 1,
                  1.0, 0, 1, nstrip, 0, 1, ny, st)


def test_variable_region_refused_below_band(pmg):
    """Variable levels below the band kernel's sizes have no regions."""
    from paper_1307_2036_b200 import _lib, configs
    prob = configs.Problem(64, 64, 128, 1e-3, 1.0, 3, stretch=1.05, variable_omega=True)
    op = pmg.PanelOperator(prob.grid(), prob.params(), pmg.Decomposition(64, 1).layout(64))
    (w, h), = op.handles.items()
    assert _lib.load().pmg_half_sweep_region_ok(h.h) == 0
