"""Small workloads of the hand-rolled synchronisation kernels for
compute-sanitizer (tests/test_sanitizers.py): the TMA band half-sweep (8 and
16 compute warps: mbarrier rings, named barriers), its fused-residual and
<f, u> modes, tile regions, the variable-coefficient band kernel, and a
configs[0] MG + CG solve.

    python tools/sanitize_case.py band|solve
"""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1307_2036_b200 as pmg  # noqa: E402
from paper_1307_2036_b200 import _lib, configs  # noqa: E402


def band():
    lib = _lib.load()
    st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    # nx = 256: 8 compute warps; nx = 1024 (few rows): 16 compute warps
    for nx, ny in ((256, 16), (1024, 8)):
        grid = pmg.periodic_box(nx, 128, 0.01, ny=ny)
        op = pmg.PanelOperator(grid, pmg.toy_parameters(nx, 128, 1e-3, 1.0),
                               pmg.Decomposition(nx, 1, ny=ny).layout(nx))
        (w, h), = op.handles.items()
        rng = np.random.default_rng(1)
        u = pmg.scatter_owned(rng.uniform(-1, 1, (nx, ny, 128)), op.layout)
        pmg.halo_exchange(u)
        f = pmg.scatter_owned(rng.uniform(-1, 1, (nx, ny, 128)), op.layout)
        un = u.copy()
        for color in (0, 1):
            _lib.call("pmg_half_sweep", h.h, u.parts[w].ptr, f.parts[w].ptr, color, 1.0, 0, 0, 1.0, st)
        ns = nx // 64
        _lib.call("pmg_half_sweep_region", h.h, u.parts[w].ptr, f.parts[w].ptr, 0, 1.0, 0, 0, 1.0,
                  1, 1, ns - 2, 1, 1, ny - 2, st)
        scr = torch.empty(int(lib.pmg_partials_size()), dtype=torch.float64, device="cuda")
        res = torch.zeros(1, dtype=torch.float64, device="cuda")
        if lib.pmg_half_sweep_res_ok(h.h):
            _lib.call("pmg_half_sweep_res", h.h, u.parts[w].ptr, un.parts[w].ptr, f.parts[w].ptr,
                      C.c_void_p(scr.data_ptr()), C.c_void_p(res.data_ptr()), st)
        z = pmg.DistField.zeros(op.layout, 128)
        _lib.call("pmg_ssor_apply", h.h, f.parts[w].ptr, z.parts[w].ptr, 1.0, 1, 1,
                  C.c_void_p(scr.data_ptr()), C.c_void_p(res.data_ptr()), st)
    # the variable-coefficient band kernel (thread-0 TMA issue after the CTA
    # barrier): plain, zero-neighbour, fused-residual modes and a region
    prob = configs.Problem(256, 16, 128, 1e-3, 1.0, 3, stretch=1.05, variable_omega=True)
    op = pmg.PanelOperator(prob.grid(), prob.params(), pmg.Decomposition(256, 1, ny=16).layout(256))
    (w, h), = op.handles.items()
    rng = np.random.default_rng(2)
    u = pmg.scatter_owned(rng.uniform(-1, 1, (256, 16, 128)), op.layout)
    pmg.halo_exchange(u)
    f = pmg.scatter_owned(rng.uniform(-1, 1, (256, 16, 128)), op.layout)
    un = u.copy()
    for color in (0, 1):
        _lib.call("pmg_half_sweep", h.h, u.parts[w].ptr, f.parts[w].ptr, color, 1.0, 0, 0, 1.0, st)
    _lib.call("pmg_half_sweep", h.h, u.parts[w].ptr, f.parts[w].ptr, 0, 1.0, 0, 1, 1.0, st)
    _lib.call("pmg_half_sweep_region", h.h, u.parts[w].ptr, f.parts[w].ptr, 1, 1.0, 0, 0, 1.0,
              1, 1, 2, 1, 1, 14, st)
    if lib.pmg_half_sweep_res_ok(h.h):
        _lib.call("pmg_half_sweep_res", h.h, u.parts[w].ptr, un.parts[w].ptr, f.parts[w].ptr,
                  C.c_void_p(scr.data_ptr()), C.c_void_p(res.data_ptr()), st)
    torch.cuda.synchronize()
    print("band ok")


def solve():
    prob = configs.config(0)
    fg = configs.rhs(prob.nx, prob.ny, prob.nz, 0)
    cfg = prob.mg_config()
    hier = pmg.build_hierarchy(prob.grid(), prob.params(), cfg)
    f = pmg.scatter_owned(fg, hier.fine.layout)
    u, rep = pmg.mg_solve(f, hier, cfg)
    op = hier.fine.op
    uc, rc = pmg.pcg_solve(f, op, pmg.SSORPreconditioner(pmg.LineSmoother(op)), eps=1e-5)
    # a four-part in-process decomposition through the native multi-part driver
    hier4 = pmg.build_hierarchy(prob.grid(), prob.params(), cfg,
                                pmg.Decomposition(prob.nx, 4))
    u4, rep4 = pmg.mg_solve(pmg.scatter_owned(fg, hier4.fine.layout), hier4, cfg)
    torch.cuda.synchronize()
    assert rep.iterations == rep4.iterations == 2 and rc.converged
    print("solve ok", rep.iterations, rc.iterations)


if __name__ == "__main__":
    {"band": band, "solve": solve}[sys.argv[1]]()
