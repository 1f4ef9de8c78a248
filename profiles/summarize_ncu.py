"""Summarise ncu outputs brought back from gpurun into small committed text files.

    python profiles/summarize_ncu.py launches <launches.csv> [regex]   # per-kernel share of device time
    python profiles/summarize_ncu.py report <prof.ncu-rep>               # key metrics of each profiled launch
    python profiles/summarize_ncu.py traffic <config> <rep> <kernel> [<rep> <kernel> ...]  # ncu_traffic.json
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


def traffic(paths, config, kernels):
    """Record the DRAM bytes and tensor-pipe activity of the tile stage's kernels (one launch each,
    captured with --set full) for `config` in profiles/ncu_traffic.json, stamped with the native
    source hash the captures were built from (bench.py uses an entry only when the hash matches its
    own build). Several (rep, kernel) pairs are summed: the Gram kernel and, where the split items
    matter (C3), the feature-product kernel that runs them."""
    import json
    import os

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from paper_2511_03126_b200.build import source_hash

    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1.0, "usecond": 1e3,
             "msecond": 1e6, "second": 1e9, "ns": 1.0, "us": 1e3, "ms": 1e6, "s": 1e9, "%": 1.0, "": 1.0}
    rd = wr = dur = tp = 0.0
    for path, kernel in zip(paths, kernels):
        out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True,
                             check=True).stdout
        rows = list(csv.reader(out.splitlines()))
        h, units = rows[0], rows[1]
        r = next(r for r in rows[2:] if re.search(kernel, r[h.index("Kernel Name")]))

        def val(k):  # bytes / nanoseconds / percent
            j = h.index(k)
            return float(r[j].replace(",", "")) * scale.get(units[j], 1.0)

        d = val("gpu__time_duration.sum")
        rd += val("dram__bytes_read.sum")
        wr += val("dram__bytes_write.sum")
        tp += d * val("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active") / 100.0
        dur += d
    fn = os.path.join(os.path.dirname(os.path.abspath(__file__)), "ncu_traffic.json")
    db = json.load(open(fn)) if os.path.exists(fn) else {}
    db[config] = {"kernel": "+".join(kernels), "dram_bytes_per_launch": int(rd + wr), "read": int(rd), "write": int(wr),
                  "duration_ms": dur / 1e6, "tensor_pipe_active": tp / dur if dur else None,
                  "source_hash": source_hash(),
                  "source": "ncu --set full --clock-control none, " + ", ".join(os.path.basename(q) for q in paths)}
    json.dump(db, open(fn, "w"), indent=1)
    print(json.dumps(db[config]))


if __name__ == "__main__":
    if sys.argv[1] == "traffic":  # traffic <config> <rep> <kernel regex> [<rep> <kernel regex> ...]
        traffic(sys.argv[3::2], sys.argv[2], sys.argv[4::2])
    elif sys.argv[1] == "launches":
        launches(sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else None)
    else:
        report(sys.argv[2])
