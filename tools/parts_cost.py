"""Device time of one configs[3]-block-sized solve (2048^2 x 128, 8 levels)
split into px x py in-process parts on one GPU through the native multi-part
driver (pmg_phier), against the single-part driver: the per-GPU cost of the
multi-part cycle (exchanges as device copies, no NCCL) and of the overlap."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1307_2036_b200 as pmg  # noqa: E402
from paper_1307_2036_b200 import configs  # noqa: E402
from paper_1307_2036_b200.partition import scatter_block  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
prob = configs.Problem(n, n, 128, 1e-3, 1.0, 8)
fg = configs.rhs(n, n, 128, 0)
for px, py, overlap in ((1, 1, True), (2, 1, True), (2, 2, True), (2, 2, False), (4, 2, True)):
    cfg = pmg.MGConfig(policy="explicit", explicit_levels=8 - (px > 1) - (px > 2), eps=1e-5,
                       overlap=overlap)
    dec = pmg.Decomposition(n, px * py, px=px, py=py)
    hier = pmg.build_hierarchy(prob.grid(), prob.params(), cfg, dec)
    f = pmg.scatter_owned(fg, hier.fine.layout)
    u = pmg.DistField.zeros(hier.fine.layout, 128)
    for _ in range(2):
        u, rep = pmg.mg_solve(f, hier, cfg, out=u)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        u, rep = pmg.mg_solve(f, hier, cfg, out=u)
    e1.record()
    torch.cuda.synchronize()
    print(json.dumps({"parts": f"{px}x{py}", "overlap": overlap, "levels": len(hier.levels),
                      "solve_ms": round(e0.elapsed_time(e1) / 3, 2), "cycles": rep.iterations,
                      "history": rep.residual_history}), flush=True)
    del hier, f, u
    torch.cuda.empty_cache()
