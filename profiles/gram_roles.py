"""Instruction and stall-sample shares of k_tile_gram by warp role (source-line ranges of
csrc/pf_gram.cu), from an ncu report captured with --import-source on.

    python profiles/gram_roles.py <report.ncu-rep> [top]
"""
import collections
import csv
import subprocess
import sys
from pathlib import Path

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", "regex:k_tile_gram", "--print-source",
                      "cuda,sass"], capture_output=True, text=True).stdout
cur = hdr = None
out = []
for r in csv.reader(txt.splitlines()):
    if r and r[0] in ("File Path", "File Name"):
        cur = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr and r and r[0].isdigit():
        d = dict(zip(hdr, r))
        try:
            out.append((int(d.get("Instructions Executed") or 0), int(d.get("Warp Stall Sampling (All Samples)") or 0),
                        cur, int(r[0]), r[1].strip()[:90]))
        except ValueError:
            pass
tot = sum(o[0] for o in out) or 1
ts = sum(o[1] for o in out) or 1
src = (Path(__file__).resolve().parent.parent / "paper_2511_03126_b200/csrc/pf_gram.cu").read_text().split("\n")


def find(pat):
    return next(i + 1 for i, line in enumerate(src) if pat in line)


marks = [("setup", "// ---- setup"), ("loader", "// ================= loaders"), ("mma", "// ================= MMA issuer"),
         ("builder", "// ================= builders"), ("acc", "// ================= accumulators"),
         ("tail", "if (PROF && P.dbg && lane == 0)")]
bounds = [(name, find(pat)) for name, pat in marks] + [("end", len(src) + 1)]
ws = [o for o in out if o[2] == "pf_gram.cu"]
print(f"warp-instructions {tot}, stall samples {ts}")
for (name, a), (_, b) in zip(bounds, bounds[1:]):
    ins = sum(o[0] for o in ws if a <= o[3] < b)
    st = sum(o[1] for o in ws if a <= o[3] < b)
    print(f"  {name:8s} inst {ins / tot:6.1%}  stall samples {st / ts:6.1%}")
other = collections.Counter()
for o in out:
    if o[2] != "pf_gram.cu":
        other[o[2]] += o[0]
print("  inlined helpers:", {k: f"{v / tot:.1%}" for k, v in other.most_common()})
for o in sorted(out, key=lambda x: -x[0])[:top]:
    print(f"{o[0] / tot:6.1%}i {o[1] / ts:6.1%}s {o[2]}:{o[3]} {o[4]}")
