"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list:
per kernel, launches and the last launch's time, plus its share of one step."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
i = [k for k, r in enumerate(rows) if r and r[0] == "ID"][0]
hdr, data = rows[i], rows[i + 1:]
ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
agg = defaultdict(list)
for r in data:
    agg[r[ki].split("(")[0].replace("void ", "")].append(float(r[vi]))
ours = {k: v for k, v in agg.items() if k.startswith("gs::")}
step = sum(v[-1] for k, v in ours.items() if "block_bounds" not in k)
print(f"{'kernel':58s} {'n':>4s} {'last_us':>10s} {'share':>6s}")
for k, v in sorted(ours.items(), key=lambda x: -x[1][-1]):
    print(f"{k[:58]:58s} {len(v):4d} {v[-1] / 1e3:10.1f} {100 * v[-1] / step:5.1f}%")
print(f"{'step (sum of last launches, cold-cache serialised)':58s} {'':4s} {step / 1e3:10.1f}")
