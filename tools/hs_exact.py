"""Exact-mode half-sweep timing at configs[1]'s fine level (graph replay),
for comparing the exact solver with the fast
default."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1307_2036_b200 as pmg  # noqa: E402
from paper_1307_2036_b200 import configs  # noqa: E402

prob = configs.config(1)
cfg = prob.mg_config()
hier = pmg.build_hierarchy(prob.grid(), prob.params(), cfg)
lev = hier.fine
sc = hier.persistent_scratch()
f = pmg.scatter_owned(configs.rhs(prob.nx, prob.ny, prob.nz, 0), lev.layout)
sc[0].f.copy_from(f)
u = sc[0].u
for exact in (False, True):
    pmg.set_exact_smoother(exact)
    flip = [0]

    def hs():
        lev.smoother.half_sweep(u, sc[0].f, flip[0] & 1, 1.0)
        flip[0] += 1
    hs()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            for _ in range(20):
                hs()
    torch.cuda.current_stream().wait_stream(s)
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / 20 * 1e3
    n = prob.dof
    print(f"exact={exact} "
          f"{t:.1f} us, {12 * n / t / 1e3:.0f} GB/s",
          flush=True)
