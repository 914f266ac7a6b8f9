"""Attribute an ncu source-page SASS export (ncu -i X.ncu-rep --page source
--csv --print-source sass) to CUDA source lines via nvdisasm -g line info of
the cubin: L2 theoretical sectors, warp-stall samples and instructions per
line. usage: sass_lines.py sass.csv file.cubin kernel_substring [N]"""
import collections
import csv
import re
import subprocess
import sys

csv_path, cubin, kern = sys.argv[1:4]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 25
dis = subprocess.run(["nvdisasm", "-g", cubin], capture_output=True, text=True).stdout.splitlines()
cur, line, amap = None, None, {}
for l in dis:
    s = l.strip()
    if s.startswith(".text.") and s.endswith(":"):
        cur = s[6:-1]
        continue
    if cur is None or kern not in cur:
        continue
    m = re.search(r'File "([^"]+)", line (\d+)', l)
    if s.startswith("//##") and m:
        line = (m.group(1), int(m.group(2)))
        continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", l)
    if m:
        amap[int(m.group(1), 16)] = line
rows = list(csv.reader(open(csv_path)))
h, data = rows[1], rows[2:]
ia, isrc = h.index("Address"), h.index("Source")
cols = {"sec": h.index("L2 Theoretical Sectors Global"), "stall": h.index("Warp Stall Sampling (All Samples)"),
        "inst": h.index("Instructions Executed")}
base = min(int(r[ia], 16) for r in data if r[ia].startswith("0x"))
agg = collections.defaultdict(lambda: collections.Counter())
tot = collections.Counter()
for r in data:
    if not r[ia].startswith("0x"):
        continue
    ln = amap.get(int(r[ia], 16) - base)
    for k, c in cols.items():
        v = float(r[c] or 0)
        agg[ln][k] += v
        tot[k] += v
srcs = {}


def text_of(ln):
    if not ln:
        return ""
    f, n = ln
    if f not in srcs:
        try:
            srcs[f] = open(f).read().splitlines()
        except OSError:
            srcs[f] = []
    lines = srcs[f]
    return (f.split("/")[-1] + ":" + str(n) + "  " + (lines[n - 1].strip() if n <= len(lines) else ""))[:110]


print(f"totals: L2 sectors {tot['sec']:.4g}, stall samples {tot['stall']:.4g}, warp instructions {tot['inst']:.4g}")
for key in ("sec", "stall"):
    print(f"--- top lines by {key}")
    for ln, v in sorted(agg.items(), key=lambda kv: -kv[1][key])[:top]:
        text = text_of(ln)
        print(f"  sec {100 * v['sec'] / max(tot['sec'], 1):5.1f}%  stall {100 * v['stall'] / max(tot['stall'], 1):5.1f}%"
              f"  inst {100 * v['inst'] / max(tot['inst'], 1):5.1f}%  {text}")

# optional: LINE_RANGES="lk_ring.cuh:14-50,lk_ring.cuh:200-360" sums the
# metrics of each source-line range
for spec in filter(None, __import__("os").environ.get("LINE_RANGES", "").split(",")):
    fname, rng = spec.split(":")
    a, b = (int(x) for x in rng.split("-"))
    s = collections.Counter()
    for ln, v in agg.items():
        if ln and ln[0].endswith(fname) and a <= ln[1] <= b:
            s.update(v)
    print(f"range {spec:28s} sec {100 * s['sec'] / max(tot['sec'], 1):5.1f}%  stall "
          f"{100 * s['stall'] / max(tot['stall'], 1):5.1f}%  inst {100 * s['inst'] / max(tot['inst'], 1):5.1f}%")
