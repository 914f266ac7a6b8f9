"""Per-kernel averages of an `ncu --metrics ... --csv` log, as JSON (for
profiles/ncu_kernels.json, which bench.py reads for the rooflines of the
extras legs). usage: ncu_metrics_json.py log.csv [log2.csv ...] > out.json"""
import csv
import json
import re
import sys
from collections import defaultdict

acc = defaultdict(lambda: defaultdict(list))
for path in sys.argv[1:]:
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    h = rows[start]
    kn, mn, mv = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    for r in rows[start + 1:]:
        m = re.search(r"\b(k_\w+)", r[kn])
        if not m:
            continue
        try:
            acc[m.group(1)][r[mn]].append(float(r[mv].replace(",", "")))
        except ValueError:
            pass
out = {k: {name: sum(v) / len(v) for name, v in d.items()} | {"launches": max(len(v) for v in d.values())}
       for k, d in acc.items()}
print(json.dumps(out, indent=1, sort_keys=True))
