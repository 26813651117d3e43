"""Top stalled SASS instructions of an ncu report (needs --import-source/-lineinfo)."""
import csv
import io
import subprocess
import sys

path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
raw = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h = rows[1]
si, wi = h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
data = []
for r in rows[2:]:
    if len(r) < len(h) or r[0] == "Kernel Name":
        break
    data.append(r)
tot = sum(int(r[wi]) for r in data)
cols = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
print("instructions", len(data), "samples", tot)
idx = sorted(range(len(data)), key=lambda i: -int(data[i][wi]))[:top]
for i in sorted(idx):
    r = data[i]
    st = {c[6:]: int(r[h.index(c)]) for c in cols if r[h.index(c)] not in ("0", "")}
    print(f"{i:5d} {int(r[wi]):6d} {r[si].strip()[:58]:58s} {st}")
