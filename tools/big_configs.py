"""Full-size single-GPU solves of the larger BASELINE workloads: configs[3]'s
per-GPU block (2048^2 x 128, periodic, 8 levels) and configs[4]
(4096^2 x 128, graded levels, variable omega^2, 9 levels) on one B200."""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1307_2036_b200 as pmg  # noqa: E402
from paper_1307_2036_b200 import configs  # noqa: E402

for name, prob in (("configs[3] per-GPU block", configs.config(3, 1)),
                   ("configs[4]", configs.config(4))):
    t0 = time.perf_counter()
    cfg = prob.mg_config()
    hier = pmg.build_hierarchy(prob.grid(), prob.params(), cfg)
    lay = hier.fine.layout
    f = pmg.DistField.zeros(lay, prob.nz)
    (w, part), = f.parts.items()
    part.load_owned(configs.rhs_block(prob.nx, prob.ny, prob.nz, 0, 0, prob.nx, prob.ny, 0))
    setup = time.perf_counter() - t0
    u = pmg.DistField.zeros(lay, prob.nz)
    u, rep = pmg.mg_solve(f, hier, cfg, out=u)          # graph capture
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    n = 3
    for _ in range(n):
        u, rep = pmg.mg_solve(f, hier, cfg, out=u)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / n
    print(json.dumps({"workload": name, "grid": [prob.nx, prob.ny, prob.nz],
                      "levels": len(hier.levels), "cycles": rep.iterations,
                      "solve_ms": round(ms, 2), "dof_per_s": prob.dof / (ms * 1e-3),
                      "history": rep.residual_history, "setup_s": round(setup, 1),
                      "gpu_mem_gb": round(torch.cuda.max_memory_allocated() / 1e9, 1)}),
          flush=True)
    del hier, f, u
    torch.cuda.empty_cache()
    torch.cuda.reset_peak_memory_stats()
