"""Sum ncu source-page (SASS) executed instructions and stall samples over
runs of consecutive instructions with equal execution counts (~basic blocks).
usage: python tools/ncu_regions.py PREFIX.source.csv [top]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
k = 1 if rows[0] and rows[0][0] == "Kernel Name" else 0
hdr, data = rows[k], rows[k + 1:]
ex = hdr.index("Instructions Executed")
si = hdr.index("Warp Stall Sampling (All Samples)")
L = []
for i, r in enumerate(data):
    try:
        e = int(r[ex])
    except (ValueError, IndexError):
        continue
    L.append((i, r[1], e, int(r[si]) if r[si].isdigit() else 0))
reg, cur = [], None
for i, s, e, smp in L:
    if cur and cur["e"] == e:
        cur["end"] = i; cur["sum"] += e; cur["smp"] += smp; cur["n"] += 1
    else:
        if cur:
            reg.append(cur)
        cur = {"beg": i, "end": i, "e": e, "sum": e, "smp": smp, "n": 1, "first": s}
reg.append(cur)
tot = sum(r["sum"] for r in reg)
ts = sum(r["smp"] for r in reg)
print("executed", tot, "samples", ts)
for r in sorted(reg, key=lambda r: -r["sum"])[:int(sys.argv[2]) if len(sys.argv) > 2 else 30]:
    print("rows %4d-%4d n=%3d each=%9d  exec %5.1f%%  samples %5.1f%%  %s" % (
        r["beg"], r["end"], r["n"], r["e"], 100 * r["sum"] / tot, 100 * r["smp"] / max(ts, 1), r["first"][:48]))
