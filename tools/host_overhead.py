"""Host-side cost of one mg_solve call: wall time per solve of configs[0]
(64 x 64 x 32, 4 levels -- the device work is ~0.3 ms) through the Python
API, against the sum of its cycles' device times."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1307_2036_b200 as pmg
from paper_1307_2036_b200 import configs
import cProfile, pstats

for idx in (0, 1):
    prob = configs.config(idx)
    cfg = prob.mg_config()
    hier = pmg.build_hierarchy(prob.grid(), prob.params(), cfg)
    f = pmg.scatter_owned(configs.rhs(prob.nx, prob.ny, prob.nz, 0), hier.fine.layout)
    u = pmg.DistField.zeros(hier.fine.layout, prob.nz)
    for _ in range(5):
        u, rep = pmg.mg_solve(f, hier, cfg, out=u)
    torch.cuda.synchronize()
    n = 200 if idx == 0 else 30
    t0 = time.perf_counter()
    for _ in range(n):
        u, rep = pmg.mg_solve(f, hier, cfg, out=u)
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) / n * 1e3
    with pmg.tracing():
        u, trep = pmg.mg_solve(f, hier, cfg, out=u)
    print(f"configs[{idx}]: {wall:.3f} ms per solve wall, cycles {rep.iterations}, "
          f"device cycle sum {sum(trep.cycle_times_ms):.3f} ms, report wall {rep.wall_time*1e3:.3f} ms")
    if idx == 0:
        pr = cProfile.Profile()
        pr.enable()
        for _ in range(200):
            u, rep = pmg.mg_solve(f, hier, cfg, out=u)
        pr.disable()
        pstats.Stats(pr).sort_stats("cumulative").print_stats(14)
