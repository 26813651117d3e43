"""RR (and sweep) on a band of rows: L2-hot (the band was just read) vs
cold (256 MB written in between)."""
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1307_2036_b200 as pmg  # noqa: E402
from paper_1307_2036_b200 import configs  # noqa: E402
from paper_1307_2036_b200._lib import load  # noqa: E402

lib = load()
lib.pmg_debug_rr_band.argtypes = [C.c_void_p] * 5 + [C.c_int, C.c_int, C.c_int, C.c_void_p]
prob = configs.config(1)
cfg = prob.mg_config()
hier = pmg.build_hierarchy(prob.grid(), prob.params(), cfg)
sc = hier.persistent_scratch()
f = pmg.scatter_owned(configs.rhs(prob.nx, prob.ny, prob.nz, 0), hier.fine.layout)
sc[0].f.copy_from(f)
w = hier.fine.layout.local_workers[0]
hf, hc = hier.levels[0].op.handles[w].h, hier.levels[1].op.handles[w].h
u, ff, cf = sc[0].u.parts[w].ptr, sc[0].f.parts[w].ptr, sc[1].f.parts[w].ptr
flush = torch.empty(256 * 2 ** 20 // 8, dtype=torch.float64, device="cuda")


def timed(seq, reps=10):
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        seq()
        with torch.cuda.graph(g, stream=s):
            for _ in range(reps):
                seq()
    torch.cuda.current_stream().wait_stream(s)
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


def st():
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


for n in (8, 16, 32):
    for sw in (0, 1):
        op = lambda: lib.pmg_debug_rr_band(hf, hc, u, ff, cf, 100, n, sw, st())
        hot = timed(op)
        fl = timed(lambda: flush.fill_(1.0))
        cold = timed(lambda: (flush.fill_(1.0), op())) - fl
        print(f"{'sweep' if sw else 'RR'} band of {n} coarse rows ({2 * n} fine): hot {hot:.1f} us, "
              f"cold {cold:.1f} us (full-level rate would be "
              f"{(328.0 if sw else 495.0) * 2 * n / 1024:.1f} us)", flush=True)
