"""Does a kernel slow down under sustained load?  The fine-level band
half-sweep of the 2048^2 x 128 block, graph-replayed back to back for 20 /
100 / 400 launches (CUDA events), with NVML SM clock and power samples."""
import json
import os
import sys
import threading
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1307_2036_b200 as pmg  # noqa: E402
from paper_1307_2036_b200 import configs  # noqa: E402

import pynvml  # noqa: E402
pynvml.nvmlInit()
hdl = pynvml.nvmlDeviceGetHandleByIndex(0)

prob = configs.Problem(2048, 2048, 128, 1e-3, 1.0, 2)
cfg = prob.mg_config()
hier = pmg.build_hierarchy(prob.grid(), prob.params(), cfg)
sc = hier.persistent_scratch()
sc[0].f.copy_from(pmg.scatter_owned(configs.rhs(2048, 2048, 128, 0), hier.fine.layout))
lev = hier.fine
flip = [0]


def hs():
    lev.smoother.half_sweep(sc[0].u, sc[0].f, flip[0] & 1, 1.0)
    flip[0] += 1


for reps in (20, 100, 400, 20):
    hs()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            for _ in range(reps):
                hs()
    torch.cuda.current_stream().wait_stream(s)
    g.replay()
    torch.cuda.synchronize()
    samples, stop = [], threading.Event()

    def run():
        while not stop.is_set():
            samples.append((pynvml.nvmlDeviceGetClockInfo(hdl, pynvml.NVML_CLOCK_SM),
                            pynvml.nvmlDeviceGetClockInfo(hdl, pynvml.NVML_CLOCK_MEM),
                            pynvml.nvmlDeviceGetPowerUsage(hdl) / 1000.0))
            time.sleep(0.005)
    th = threading.Thread(target=run)
    th.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    stop.set()
    th.join()
    ms = e0.elapsed_time(e1) / reps
    sm = sorted(x[0] for x in samples)
    pw = sorted(x[2] for x in samples)
    print(json.dumps({"reps": reps, "us_per_sweep": round(ms * 1e3, 1),
                      "sm_mhz_median": sm[len(sm) // 2] if sm else None,
                      "mem_mhz": samples[0][1] if samples else None,
                      "power_w_median": pw[len(pw) // 2] if pw else None,
                      "samples": len(samples)}), flush=True)
    del g
