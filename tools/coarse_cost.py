"""Cost of the coarse part of the configs[1] V-cycle: one V-cycle (native
pmg_vcycle, graph-replayed) of the sub-hierarchies that start at level 2
(256^2), 3 (128^2) and 4 (64^2), nz = 128."""
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1307_2036_b200 as pmg  # noqa: E402
from paper_1307_2036_b200 import configs  # noqa: E402
from paper_1307_2036_b200._lib import call  # noqa: E402

for nx, nlev in ((256, 5), (128, 4), (64, 3), (32, 2)):
    prob = configs.Problem(nx, nx, 128, 1e-3, 1.0, nlev)
    cfg = prob.mg_config()
    hier = pmg.build_hierarchy(prob.grid(), prob.params(), cfg)
    f = pmg.scatter_owned(configs.rhs(nx, nx, 128, 0), hier.fine.layout)
    u = pmg.DistField.zeros(hier.fine.layout, 128)
    nh = hier.native(cfg)
    (w, uf), = u.parts.items()

    def cyc():
        call("pmg_vcycle", nh.h, uf.ptr, f.parts[w].ptr, 0,
             C.c_void_p(torch.cuda.current_stream().cuda_stream))
    cyc()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            for _ in range(10):
                cyc()
    torch.cuda.current_stream().wait_stream(s)
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    print(f"V-cycle from {nx}^2 x 128 ({nlev} levels): {e0.elapsed_time(e1) / 10 * 1e3:.1f} us",
          flush=True)
