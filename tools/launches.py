"""Summarise an ncu --metrics gpu__time_duration.sum launch list (CSV)."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
hdr = rows[start]
kn, mv = hdr.index("Kernel Name"), hdr.index("Metric Value")
agg = defaultdict(list)
for r in rows[start + 1:]:
    name = r[kn].split("(")[0].replace("lkk::<unnamed>::", "")
    agg[name].append(float(r[mv].replace(",", "")) / 1000.0)
tot = sum(sum(v) for v in agg.values())
print(f"{'kernel':45s} {'n':>4s} {'avg_us':>10s} {'total_us':>10s} {'share':>6s}")
for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    print(f"{k[:45]:45s} {len(v):4d} {sum(v)/len(v):10.1f} {sum(v):10.1f} {100*sum(v)/tot:6.1f}")
