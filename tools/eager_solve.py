"""Host-overhead probe: configs[1] MG solve through the Python V-cycle
without CUDA graphs (the multi-rank code path's launch pattern) vs the
graph-replayed native driver, one GPU, one part."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1307_2036_b200 as pmg  # noqa: E402
from paper_1307_2036_b200 import configs, multigrid as mg  # noqa: E402

prob = configs.config(1)
for graph, native in ((True, True), (False, False)):
    mg.USE_NATIVE = native
    cfg = prob.mg_config(graph=graph)
    hier = pmg.build_hierarchy(prob.grid(), prob.params(), cfg)
    f = pmg.scatter_owned(configs.rhs(prob.nx, prob.ny, prob.nz, 0), hier.fine.layout)
    u = pmg.DistField.zeros(hier.fine.layout, prob.nz)
    for _ in range(3):
        u, rep = pmg.mg_solve(f, hier, cfg, out=u)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    n = 10
    for _ in range(n):
        u, rep = pmg.mg_solve(f, hier, cfg, out=u)
    torch.cuda.synchronize()
    print(f"graph={graph} native={native}: {(time.perf_counter() - t0) / n * 1e3:.2f} ms/solve, "
          f"{rep.iterations} cycles")
