"""A/B helper: one configs[1] MG solve (or --nx/--levels), prints the
history, a hash of the iterate and the graph-replayed solve time; run it
under different configurations and compare (bit-identical paths must print
the same hash)."""
import argparse
import hashlib
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1307_2036_b200 as pmg  # noqa: E402
from paper_1307_2036_b200 import configs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--nx", type=int, default=1024)
ap.add_argument("--levels", type=int, default=7)
a = ap.parse_args()
prob = configs.Problem(a.nx, a.nx, 128, 1e-3, 1.0, a.levels)
cfg = prob.mg_config()
hier = pmg.build_hierarchy(prob.grid(), prob.params(), cfg)
f = pmg.scatter_owned(configs.rhs(a.nx, a.nx, 128, 0), hier.fine.layout)
u = pmg.DistField.zeros(hier.fine.layout, 128)
for _ in range(3):
    u, rep = pmg.mg_solve(f, hier, cfg, out=u)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
n = 10
for _ in range(n):
    u, rep = pmg.mg_solve(f, hier, cfg, out=u)
e1.record()
torch.cuda.synchronize()
h = hashlib.sha256(pmg.gather_owned(u).tobytes()).hexdigest()[:16]
print(json.dumps({"solve_ms": round(e0.elapsed_time(e1) / n, 3), "iters": rep.iterations,
                  "hash": h, "hist": rep.residual_history}))
