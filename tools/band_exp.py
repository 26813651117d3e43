"""Band-interleaved black half-sweep + residual-restrict (pmg_debug_band):
does the RR get cheaper when it reads rows the sweep just touched (L2)?"""
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1307_2036_b200 as pmg  # noqa: E402
from paper_1307_2036_b200 import configs  # noqa: E402
from paper_1307_2036_b200._lib import load  # noqa: E402

lib = load()
# needs the (removed) pmg_debug_band experiment entry point; kept for the record
lib.pmg_debug_band.argtypes = [C.c_void_p] * 5 + [C.c_int, C.c_void_p]
prob = configs.config(1)
cfg = prob.mg_config()
hier = pmg.build_hierarchy(prob.grid(), prob.params(), cfg)
sc = hier.persistent_scratch()
f = pmg.scatter_owned(configs.rhs(prob.nx, prob.ny, prob.nz, 0), hier.fine.layout)
sc[0].f.copy_from(f)
w = hier.fine.layout.local_workers[0]
hf, hc = hier.levels[0].op.handles[w].h, hier.levels[1].op.handles[w].h
u, ff, cf = sc[0].u.parts[w].ptr, sc[0].f.parts[w].ptr, sc[1].f.parts[w].ptr
ref = None
for R in (0, 8, 16, 32, 64, 128, 256):
    def run():
        lib.pmg_debug_band(hf, hc, u, ff, cf, R, C.c_void_p(torch.cuda.current_stream().cuda_stream))
    run()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            for _ in range(10):
                run()
    torch.cuda.current_stream().wait_stream(s)
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    out = pmg.gather_owned(sc[1].f)
    if ref is None:
        ref = out
    print(f"R={R}: {e0.elapsed_time(e1) / 10 * 1e3:.1f} us per sweep+RR, "
          f"same result {bool((out == ref).all())}", flush=True)
