"""Turn gpurun_out/ (bench.json, launches.csv, prof_fine.ncu-rep) into the
committed evidence under profiles/: per-kernel share of the solve, DRAM
traffic per launch of the fine-level kernels (ncu_traffic.json, read by
bench.py), and a text summary."""
import collections
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GO = os.path.join(ROOT, "gpurun_out")
PR = os.path.join(ROOT, "profiles")
tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
os.makedirs(PR, exist_ok=True)
lines = []

# ---- launch list: per-kernel totals ----
p = os.path.join(GO, "launches.csv")
if os.path.exists(p):
    rows = list(csv.reader(open(p)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, mi, vi, ui = (h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"),
                      h.index("Metric Unit"))
    gi = h.index("Grid Size") if "Grid Size" in h else None
    idi = h.index("ID")
    per = collections.defaultdict(dict)
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(",", ""))
        unit = r[ui]
        scale = {"nsecond": 1.0, "usecond": 1e3, "msecond": 1e6, "byte": 1.0, "Kbyte": 1e3,
                 "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1.0)
        per[r[idi]][r[mi]] = v * scale
        per[r[idi]]["name"] = r[ki].split("(")[0].replace("void ", "")
        per[r[idi]]["grid"] = r[gi] if gi is not None else ""
    tot = collections.defaultdict(lambda: [0.0, 0, 0.0])
    for d in per.values():
        key = d["name"]
        tot[key][0] += d.get("gpu__time_duration.sum", 0.0)
        tot[key][1] += 1
        tot[key][2] += d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
    T = sum(v[0] for v in tot.values())
    lines.append(f"# ncu launch list ({len(per)} launches, cold-cache serialised)")
    lines.append(f"{'kernel':45s} {'share':>6s} {'ms':>9s} {'n':>5s} {'GB':>8s}")
    for k, (t, n, b) in sorted(tot.items(), key=lambda x: -x[1][0]):
        lines.append(f"{k[:45]:45s} {100 * t / T:5.1f}% {t / 1e6:9.3f} {n:5d} {b / 1e9:8.3f}")
    lines.append("")

# ---- full capture of fine-level kernels ----
traffic = {}
import glob
CURRENT = ["k_half_sweep_band", "hs_res", "k_residual_restrict_red", "k_prolong_w"]
for p in [os.path.join(GO, f"prof_{k}.ncu-rep") for k in CURRENT]:
    if not os.path.exists(p):
        continue
    raw = subprocess.run(["ncu", "-i", p, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units = rows[0], rows[1]
    want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
            "sm__throughput.avg.pct_of_peak_sustained_elapsed",
            "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
            "launch__grid_size", "launch__block_size"]
    lines.append(f"# ncu --set full, fine level (1024^2 x 128): {os.path.basename(p)}")
    for r in rows[2:]:
        name = r[h.index("Kernel Name")].split("(")[0].replace("void ", "")
        vals = {}
        for m in want:
            if m in h:
                vals[m] = (r[h.index(m)], units[h.index(m)])
        lines.append(f"## {name}")
        for m, (v, u) in vals.items():
            lines.append(f"   {m:60s} {v} {u}")

        def num(m):
            v, u = vals[m]
            s = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
            return float(v.replace(",", "")) * s
        base = name.split("<")[0]
        if base not in traffic:
            traffic[base] = num("dram__bytes_read.sum") + num("dram__bytes_write.sum")
    # merge: bench.py reads the "<kernel>@<nx>" entries of earlier captures
    tp = os.path.join(PR, "ncu_traffic.json")
    merged = json.load(open(tp)) if os.path.exists(tp) else {}
    merged.update(traffic)
    json.dump(merged, open(tp, "w"), indent=1)

p = os.path.join(GO, "bench.json")
if os.path.exists(p):
    txt = open(p).read().strip().splitlines()
    if txt:
        b = json.loads(txt[-1])
        json.dump(b, open(os.path.join(PR, f"bench_{tag}.json"), "w"), indent=1)
        lines.insert(0, f"# bench {tag}: {b['value']:.4g} DOF/s, {b['ms_per_step']:.2f} ms/solve, "
                        f"half-sweep {b['roofline']['achieved']:.0f} GB/s "
                        f"({100 * b['roofline']['frac']:.1f}% of {b['roofline']['peak']})\n")
open(os.path.join(PR, f"summary_{tag}.txt"), "w").write("\n".join(lines) + "\n")
print("\n".join(lines))
