"""Top SASS lines by warp-stall samples from `ncu -i REP --page source --csv
--print-source=sass -k KERNEL` output (profiling helper)."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
hdr = next(r for r in rows if r and r[0] == "Address")
i_s, i_e = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
data = []
for r in rows:
    if len(r) > i_e and r[0] != "Address" and r[i_s].replace(".", "").isdigit():
        data.append((r[0], r[1], int(float(r[i_s])), int(float(r[i_e] or 0))))
tot = sum(d[2] for d in data) or 1
print(f"samples {tot}  instructions {sum(d[3] for d in data)}")
for a, s, w, e in sorted(data, key=lambda x: -x[2])[:n]:
    print(f"{a:>6s} {100 * w / tot:5.1f}% {e:>9d}  {s}")
