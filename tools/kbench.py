"""Dev micro-benchmark: fine-level kernel times at configs[1] size (or
--nx/--nz), CUDA events, L2-cold (fields >> L2)."""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1307_2036_b200 as pmg  # noqa: E402
from paper_1307_2036_b200 import configs, multigrid as mg  # noqa: E402


def timeit(fn, reps=20):
    fn()
    torch.cuda.synchronize()
    if os.environ.get("KB_GRAPH"):
        # replay a captured sequence: no host launch overhead in the timing
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            with torch.cuda.graph(g, stream=s):
                for _ in range(reps):
                    fn()
        torch.cuda.current_stream().wait_stream(s)
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


ap = argparse.ArgumentParser()
ap.add_argument("--nx", type=int, default=1024)
ap.add_argument("--nz", type=int, default=128)
ap.add_argument("--ny", type=int, default=0)
ap.add_argument("--levels", type=int, default=7)
ap.add_argument("--variable", action="store_true")
ap.add_argument("--no-solve", action="store_true")
a = ap.parse_args()
a.ny = a.ny or a.nx
prob = configs.Problem(a.nx, a.ny, a.nz, 1e-3, 1.0, a.levels, stretch=1.05 if a.variable else None,
                       variable_omega=a.variable)
cfg = prob.mg_config()
hier = pmg.build_hierarchy(prob.grid(), prob.params(), cfg)
sc = hier.persistent_scratch()
f = pmg.scatter_owned(configs.rhs(a.nx, a.ny, a.nz, 0), hier.fine.layout)
sc[0].f.copy_from(f)
out = {}
res = torch.zeros(1, dtype=torch.float64, device="cuda")
for c, lev in enumerate(hier.levels):
    s = sc[c]
    n = lev.layout.nx * lev.layout.ny * a.nz
    row = {}
    flip = [0]

    def hs():
        lev.smoother.half_sweep(s.u, s.f, flip[0] & 1, 1.0)
        flip[0] += 1
    t = timeit(hs)
    row["half_sweep"] = (round(t * 1e3, 1), round(12 * n / t / 1e6))
    lib = pmg._lib.load()
    w = lev.layout.local_workers[0]
    hh = lev.op.handles[w].h
    if lib.pmg_half_sweep_res_ok(hh):
        import ctypes as C
        scr = torch.empty(int(lib.pmg_partials_size()), dtype=torch.float64, device="cuda")
        st = C.c_void_p(torch.cuda.current_stream().cuda_stream)

        def hsr():
            lib.pmg_half_sweep_res(hh, s.u.parts[w].ptr, s.r.parts[w].ptr, s.f.parts[w].ptr,
                                   C.c_void_p(scr.data_ptr()), C.c_void_p(res.data_ptr()),
                                   C.c_void_p(torch.cuda.current_stream().cuda_stream))
        t = timeit(hsr)
        row["half_sweep_res"] = (round(t * 1e3, 1), round(16 * n / t / 1e6))
    t = timeit(lambda: lev.op.residual_norm2_dev(s.f, s.u, None, res))
    row["resid_norm"] = (round(t * 1e3, 1), round(16 * n / t / 1e6))
    if c + 1 < len(hier.levels):
        co = hier.levels[c + 1]
        t = timeit(lambda: mg._residual_restrict(lev, co, s.f, s.u, sc[c + 1].f))
        row["resid_restrict"] = (round(t * 1e3, 1), round(18 * n / t / 1e6))
        if lib.pmg_residual_restrict_red_ok(hh):
            t = timeit(lambda: mg._residual_restrict(lev, co, s.f, s.u, sc[c + 1].f, True))
            row["resid_restrict_red"] = (round(t * 1e3, 1), round(14 * n / t / 1e6))
        t = timeit(lambda: mg._prolong_add(sc[c + 1].u, co, lev, s.u))
        row["prolong_add"] = (round(t * 1e3, 1), round(18 * n / t / 1e6))
        t = timeit(lambda: mg._prolong_add(sc[c + 1].u, co, lev, s.u, black_only=True))
        row["prolong_black"] = (round(t * 1e3, 1), round(10 * n / t / 1e6))
    t = timeit(lambda: pmg.halo_exchange(s.u))
    row["halo"] = round(t * 1e3, 1)
    print(f"L{c} nx={lev.layout.nx}: " + json.dumps(row), flush=True)
# full solve (lagged convergence norm on / off)
import dataclasses  # noqa: E402
for lag, red in () if a.no_solve else ((True, True), (True, False), (False, False)):
    cfg = dataclasses.replace(cfg, lagged_norm=lag, red_restrict=red)
    for _ in range(2):
        u, rep = pmg.mg_solve(f, hier, cfg)
    t = timeit(lambda: pmg.mg_solve(f, hier, cfg, out=u), 5)
    print(json.dumps({"lagged_norm": lag, "red_restrict": red, "solve_ms": round(t, 3), "iters": rep.iterations,
                      "hist": rep.residual_history}))
