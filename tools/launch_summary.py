"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list:
per kernel name: launches, mean duration, share of the listed time."""
import csv
import sys
from collections import defaultdict


def main(path):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[start]
    ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    d = defaultdict(list)
    for r in rows[start + 1:]:
        if len(r) > vi and r[mi] == "gpu__time_duration.sum":
            d[r[ki].split("(")[0][:70]].append(float(r[vi].replace(",", "")))
    tot = sum(sum(v) for v in d.values())
    print("%-70s %6s %12s %7s" % ("kernel", "n", "mean_ns", "share"))
    for k, v in sorted(d.items(), key=lambda x: -sum(x[1])):
        print("%-70s %6d %12.1f %7.3f" % (k, len(v), sum(v) / len(v), sum(v) / tot))


if __name__ == "__main__":
    main(sys.argv[1])
