"""Top source lines of one kernel in an ncu report by warp-stall samples / instructions.

    python profiles/hot_lines.py <report.ncu-rep> <kernel-regex> [N]
"""
import csv
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", kern, "--print-source",
                      "cuda,sass"], capture_output=True, text=True).stdout
cur, hdr, out = None, None, []
for r in csv.reader(txt.splitlines()):
    if r and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr and r and r[0].isdigit():
        d = dict(zip(hdr, r))
        try:
            out.append((int(d.get("Warp Stall Sampling (All Samples)") or 0),
                        int(d.get("Instructions Executed") or 0), cur, r[0], r[1].strip()[:80],
                        {k[6:]: d[k] for k in hdr if k.startswith("stall_") and "Not Issued" not in k
                         and d.get(k, "0") not in ("0", "")}))
        except ValueError:
            pass
ts = sum(o[0] for o in out) or 1
ti = sum(o[1] for o in out) or 1
print(f"samples {ts}  warp-instructions {ti}")
for o in sorted(out, key=lambda x: -x[0])[:top]:
    st = sorted(o[5].items(), key=lambda kv: -int(kv[1]))[:3]
    print(f"{100*o[0]/ts:5.1f}%s {100*o[1]/ti:5.1f}%i {o[2]}:{o[3]:<4} {o[4]:<80} {st}")
