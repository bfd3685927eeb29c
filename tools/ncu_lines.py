"""Per-source-line instruction / stall attribution from an ncu report
(--page source --print-source cuda,sass).  usage: ncu_lines.py REP [topN]"""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 50
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
fname = ""
agg = {}
hdr = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        ie = hdr.index("Instructions Executed")
        ss = hdr.index("Warp Stall Sampling (All Samples)")
        continue
    if hdr is None or r[0] == "" or r[0] == "Function Name":
        continue
    try:
        n = float(r[ie]); st = float(r[ss])
    except (ValueError, IndexError):
        continue
    k = (fname, int(r[0]))
    a = agg.setdefault(k, [0.0, 0.0, r[1][:100]])
    a[0] += n; a[1] += st
tot = sum(a[0] for a in agg.values()); tst = sum(a[1] for a in agg.values())
print(f"total warp instructions {tot:.4g}, stall samples {tst:.4g}")
for (f, l), (n, st, src) in sorted(agg.items(), key=lambda x: -x[1][0])[:top]:
    print(f"{100 * n / tot:5.1f}% inst {100 * st / tst:5.1f}% stall  {f}:{l}: {src}")
