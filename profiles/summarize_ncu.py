"""Summarise ncu outputs brought back from gpurun into small committed text files.

    python profiles/summarize_ncu.py launches <launches.csv> [regex]   # per-kernel share of device time
    python profiles/summarize_ncu.py report <prof.ncu-rep>               # key metrics of each profiled launch
"""

import csv
import re
import subprocess
import sys
from collections import defaultdict

KEYS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_sector_hit_rate.pct",
    "l1tex__throughput.avg.pct_of_peak_sustained_active",
    "l1tex__t_sector_hit_rate.pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread",
    "launch__grid_size",
    "launch__block_size",
    "launch__occupancy_limit_shared_mem",
    "smsp__inst_executed.sum",
]


def launches(path, pattern=None):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    h = rows[hdr]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows[hdr + 1 :]:
        if len(r) <= vi:
            continue
        name = r[ki]
        if pattern and not re.search(pattern, name):
            continue
        agg[name[:90]][0] += 1
        agg[name[:90]][1] += float(r[vi].replace(",", ""))
    tot = sum(v[1] for v in agg.values())
    print(f"{'launches':>8} {'total_ms':>10} {'share':>6}  kernel")
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{v[0]:8d} {v[1] / 1e6:10.3f} {100 * v[1] / tot:5.1f}%  {k}")


def report(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, units = rows[0], rows[1]
    for r in rows[2:]:
        print(f"== {r[h.index('Kernel Name')][:100]}")
        for k in KEYS:
            if k in h:
                j = h.index(k)
                print(f"  {k:70s} {r[j]} {units[j]}")


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else None)
    else:
        report(sys.argv[2])
