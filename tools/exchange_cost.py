"""GPU-side cost of the multi-part halo exchanges: configs[1]-sized parts,
P in-process parts on one GPU (graph-replayed Python V-cycle: pack, copy,
unpack per face, the same kernels the multi-rank path launches around its
NCCL calls) vs one part.  time(P) / P - time(1) = exchange overhead per
part-solve."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1307_2036_b200 as pmg  # noqa: E402
from paper_1307_2036_b200 import configs, multigrid as mg  # noqa: E402

for px, py in ((1, 1), (2, 1), (2, 2)):
    prob = configs.Problem(1024 * px, 1024 * py, 128, 1e-3, 1.0, 7)
    cfg = prob.mg_config()
    dec = pmg.Decomposition(prob.nx, px * py, ny=prob.ny, px=px, py=py, periodic=True)
    hier = pmg.build_hierarchy(prob.grid(), prob.params(), cfg, dec)
    f = pmg.scatter_owned(configs.rhs(prob.nx, prob.ny, prob.nz, 0), hier.fine.layout)
    u = pmg.DistField.zeros(hier.fine.layout, prob.nz)
    for _ in range(2):
        u, rep = pmg.mg_solve(f, hier, cfg, out=u)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    n = 5
    for _ in range(n):
        u, rep = pmg.mg_solve(f, hier, cfg, out=u)
    torch.cuda.synchronize()
    t = (time.perf_counter() - t0) / n * 1e3
    print(f"{px}x{py} parts: {t:.2f} ms/solve ({t / (px * py):.2f} per part), "
          f"{rep.iterations} cycles", flush=True)
    del hier, f, u
    torch.cuda.empty_cache()
