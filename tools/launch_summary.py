"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list:
per kernel launches, mean and total microseconds."""
import collections
import csv
import sys


def main(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    d = collections.OrderedDict()
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr) and r[hdr.index("Metric Name")] == "gpu__time_duration.sum":
            name = r[hdr.index("Kernel Name")].split("(")[0].replace("lkk::<unnamed>::", "")
            unit = r[hdr.index("Metric Unit")]
            v = float(r[hdr.index("Metric Value")].replace(",", ""))
            v = v / 1000.0 if unit in ("ns", "nsecond") else (v * 1000.0 if unit in ("ms", "msecond") else v)
            d.setdefault(name, []).append(v)
    print(f"{'kernel':40s} {'n':>4s} {'mean_us':>10s} {'total_us':>10s}")
    for k, v in d.items():
        print(f"{k[:40]:40s} {len(v):4d} {sum(v) / len(v):10.1f} {sum(v):10.1f}")


if __name__ == "__main__":
    main(sys.argv[1])
