"""Fine-level red half-sweep with the fused convergence residual
(pmg_half_sweep_res) at configs[1] size, a few launches, for ncu capture:
`ncu -k regex:k_half_sweep_seg -c 1 python tools/hs_res.py`."""
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1307_2036_b200 as pmg  # noqa: E402
from paper_1307_2036_b200 import _lib, configs  # noqa: E402

NX = int(os.environ.get("NX", "1024"))
prob = configs.Problem(NX, NX, 128, 1e-3, 1.0, 1)
cfg = prob.mg_config()
hier = pmg.build_hierarchy(prob.grid(), prob.params(), pmg.MGConfig(policy="explicit",
                                                                    explicit_levels=1))
lay = hier.fine.layout
w = lay.local_workers[0]
f = pmg.scatter_owned(configs.rhs(prob.nx, prob.ny, prob.nz, 0), lay)
u, un = f.copy(), pmg.DistField.zeros(lay, prob.nz)
pmg.halo_exchange(u)
lib = _lib.load()
scr = torch.empty(int(lib.pmg_partials_size()), dtype=torch.float64, device="cuda")
res = torch.zeros(1, dtype=torch.float64, device="cuda")
h = hier.fine.op.handles[w].h
for _ in range(int(os.environ.get("N", "3"))):
    _lib.call("pmg_half_sweep_res", h, u.parts[w].ptr, un.parts[w].ptr, f.parts[w].ptr,
              C.c_void_p(scr.data_ptr()), C.c_void_p(res.data_ptr()),
              C.c_void_p(torch.cuda.current_stream().cuda_stream))
torch.cuda.synchronize()
print("norm2", res.item())
if os.environ.get("TIME"):          # CUDA-event mean over back-to-back launches
    st = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = int(os.environ["TIME"])
    e0.record(st)
    for _ in range(n):
        _lib.call("pmg_half_sweep_res", h, u.parts[w].ptr, un.parts[w].ptr, f.parts[w].ptr,
                  C.c_void_p(scr.data_ptr()), C.c_void_p(res.data_ptr()),
                  C.c_void_p(st.cuda_stream))
    e1.record(st)
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / n * 1e3
    print(f"half_sweep_res nx={NX}: {us:.1f} us, {16 * NX * NX * 128 / us / 1e3:.0f} GB/s, "
          f"checksum {float(un.parts[w].data.sum().item())!r}")
