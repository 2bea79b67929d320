"""Summarise an ncu --metrics gpu__time_duration.sum launch list (CSV)."""
import csv
import sys
from collections import defaultdict

lines = [ln for ln in open(sys.argv[1]) if not ln.startswith("==")]
rows = list(csv.DictReader(lines))
d = defaultdict(list)
for r in rows:
    if r["Metric Name"] == "gpu__time_duration.sum":
        name = r["Kernel Name"]
        short = name.split("(")[0].replace("void ", "")[:80]
        d[short].append(float(r["Metric Value"]))
tot = sum(sum(v) for v in d.values())
print(f"{'launches':>8} {'total us':>10} {'share':>6}  kernel")
for k, v in sorted(d.items(), key=lambda x: -sum(x[1])):
    print(f"{len(v):8d} {sum(v) / 1e3:10.1f} {100 * sum(v) / tot:5.1f}%  {k}  (mean {sum(v) / len(v) / 1e3:.1f} us)")
