"""Dev benchmark: configs[2] (CG + line SSOR) and configs[4] (variable
coefficients, graded) solves on one GPU; prints iterations, histories, time."""
import argparse
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1307_2036_b200 as pmg  # noqa: E402
from paper_1307_2036_b200 import configs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--which", default="cg")
ap.add_argument("--omega2", type=float, default=1e-3)
ap.add_argument("--nx", type=int, default=1024)
ap.add_argument("--levels", type=int, default=7)
a = ap.parse_args()
if a.which == "cg":
    prob = configs.Problem(a.nx, a.nx, 128, a.omega2, 1.0, a.levels)
    f_h = configs.rhs(prob.nx, prob.ny, prob.nz, 0)
    op = pmg.PanelOperator(prob.grid(), prob.params())
    pre = pmg.SSORPreconditioner(pmg.LineSmoother(op))
    f = pmg.scatter_owned(f_h, op.layout)
    for _ in range(2):
        u, rep = pmg.pcg_solve(f, op, pre, eps=1e-5, maxiter=2000)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    u, rep = pmg.pcg_solve(f, op, pre, eps=1e-5, maxiter=2000)
    torch.cuda.synchronize()
    t = time.perf_counter() - t0
    print(json.dumps({"which": "cg", "omega2": a.omega2, "iters": rep.iterations,
                      "solve_ms": t * 1e3, "ms_per_iter": t * 1e3 / rep.iterations,
                      "hist": rep.residual_history, "drift": rep.residual_drift}))
else:
    prob = configs.Problem(a.nx, a.nx, 128, 1e-3, 1.0, a.levels, stretch=1.05,
                           variable_omega=True)
    cfg = prob.mg_config()
    t0 = time.perf_counter()
    hier = pmg.build_hierarchy(prob.grid(), prob.params(), cfg)
    tb = time.perf_counter() - t0
    f_h = configs.rhs(prob.nx, prob.ny, prob.nz, 0)
    f = pmg.scatter_owned(f_h, hier.fine.layout)
    del f_h
    for _ in range(2):
        u, rep = pmg.mg_solve(f, hier, cfg)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    u, rep = pmg.mg_solve(f, hier, cfg, out=u)
    torch.cuda.synchronize()
    t = time.perf_counter() - t0
    print(json.dumps({"which": "config4", "nx": a.nx, "iters": rep.iterations,
                      "solve_ms": t * 1e3, "build_s": tb, "hist": rep.residual_history,
                      "mem_GB": torch.cuda.max_memory_allocated() / 1e9}))
