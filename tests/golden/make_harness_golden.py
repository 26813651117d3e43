"""Golden rows of the reference's experiment harness (bench.py), generated
by importing the reference package in the build container:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_harness_golden.py

Writes tests/golden/harness.json: the param_space table (nx 256 .. 16384)
and the rows of small MG / CG solves and of the weak_scaling / levels /
robustness tables (wall-time columns dropped)."""
import json
import os
import sys

sys.path.insert(0, os.environ.get("PANELMG_SRC", "/root/reference/pkg/src"))
from panelmg import ExperimentSpec, run_experiment, run_table  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "harness.json")
SKIP = ("wall_time_s", "time_per_iter_s")


def clean(rows):
    return [{k: str(v) for k, v in r.items() if k not in SKIP} for r in rows]


res = {"param_space": clean(run_table("param_space", None, nx=256, nx_max=16384, nz=128,
                                      dt=600.0))}
res["runs"] = {}
for name, kw in {
    "mg16": dict(nx=16, nz=4, dt=600.0, solver="mg"),
    "cg16": dict(nx=16, nz=8, dt=600.0, solver="cg"),
    "mg32_shallow_w4": dict(nx=32, nz=8, dt=600.0, solver="mg", policy="shallow", workers=4),
    "mg16_seed7_det": dict(nx=16, nz=4, dt=600.0, solver="mg", seed=7, deterministic=True),
    "mg32_manufactured": dict(nx=32, nz=8, dt=1200.0, solver="mg", rhs="manufactured",
                              eps=1e-10),
    "mg16_flat": dict(nx=16, nz=4, dt=600.0, solver="mg", flat=True),
}.items():
    res["runs"][name] = {"spec": kw, "row": clean([run_experiment(ExperimentSpec(**kw))[1]])[0]}
res["weak_scaling"] = clean(run_table("weak_scaling", None, nx=8, nx_max=16, nz=4, dt=600.0))
res["levels"] = clean(run_table("levels", None, nx=8, nz=4, dt=600.0))
res["robustness"] = clean(run_table("robustness", None, nx=8, nz=4, dt=600.0))
json.dump(res, open(OUT, "w"), indent=1)
print("wrote", OUT)
