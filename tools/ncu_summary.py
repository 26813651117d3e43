"""Summarise ncu --set full reports: time, DRAM bytes, throughput, occupancy, top stalls."""
import csv
import io
import subprocess
import sys

WANT = [
    ("gpu__time_duration.sum", "time"),
    ("dram__bytes_read.sum", "dram_rd"),
    ("dram__bytes_write.sum", "dram_wr"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram%"),
    ("lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum", "l2_rd_hit_sec"),
    ("lts__t_sectors_srcunit_tex_op_read.sum", "l2_rd_sec"),
    ("l1tex__t_sector_hit_rate.pct", "l1_hit%"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occ%"),
    ("launch__registers_per_thread", "regs"),
    ("launch__occupancy_limit_registers", "lim_regs"),
    ("launch__occupancy_limit_shared_mem", "lim_smem"),
    ("launch__occupancy_limit_warps", "lim_warps"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm%"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "l2%"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "l1%"),
]


def summarize(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units = rows[0], rows[1]
    for r in rows[2:]:
        name = r[h.index("Kernel Name")][:60]
        print(f"== {path}: {name}")
        for m, short in WANT:
            if m in h:
                i = h.index(m)
                print(f"   {short:14s} {r[i]} {units[i]}")
        stalls = [(c, r[i]) for i, c in enumerate(h)
                  if c.startswith("smsp__average_warp_latency_issue_stalled") or
                  (c.startswith("smsp__pcsamp_warps_issue_stalled_") and not c.endswith("not_issued"))]
        vals = []
        for c, v in stalls:
            try:
                vals.append((float(v.replace(",", "")), c))
            except ValueError:
                pass
        for v, c in sorted(vals, reverse=True)[:6]:
            print(f"   stall {c.split('stalled_')[-1]:30s} {v}")


if __name__ == "__main__":
    for p in sys.argv[1:]:
        summarize(p)
