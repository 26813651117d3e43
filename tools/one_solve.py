"""One warm-up and one timed MG solve of a BASELINE workload (for ncu launch
lists: `ncu --metrics gpu__time_duration.sum -c N python tools/one_solve.py
config4`).  Workloads: config1, config3 (2048^2 block), config4."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1307_2036_b200 as pmg  # noqa: E402
from paper_1307_2036_b200 import configs  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "config4"
prob = {"config1": lambda: configs.config(1), "config3": lambda: configs.config(3, 1),
        "config4": lambda: configs.config(4)}[name]()
cfg = prob.mg_config()
hier = pmg.build_hierarchy(prob.grid(), prob.params(), cfg)
lay = hier.fine.layout
f = pmg.DistField.zeros(lay, prob.nz)
(w, part), = f.parts.items()
part.load_owned(configs.rhs_block(prob.nx, prob.ny, prob.nz, 0, 0, prob.nx, prob.ny, 0))
u = pmg.DistField.zeros(lay, prob.nz)
for _ in range(int(os.environ.get("SOLVES", "2"))):
    u, rep = pmg.mg_solve(f, hier, cfg, out=u)
torch.cuda.synchronize()
print(name, rep.iterations, rep.residual_history)
