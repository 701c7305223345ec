"""Aggregate ncu source-page stall samples by reason and by instruction
class over an address range (e.g. the GEMV main loop).
usage: python tools/ncu_stalls.py PREFIX [min_samples]"""
import csv
import sys
from collections import Counter


def main(prefix, thr=0):
    rows = list(csv.reader(open(prefix + ".source.csv")))
    hdr = rows[1] if rows[0] and rows[0][0] == "Kernel Name" else rows[0]
    data = rows[2:] if rows[0] and rows[0][0] == "Kernel Name" else rows[1:]
    reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    idx = {h: hdr.index(h) for h in reasons}
    si = hdr.index("Warp Stall Sampling (All Samples)")
    ex = hdr.index("Instructions Executed")
    tot = Counter()
    by_op = Counter()
    inst_op = Counter()
    for r in data:
        if len(r) <= si or not r[si].isdigit():
            continue
        op = r[1].split()[0] if not r[1].startswith("@") else r[1].split()[1]
        op = op.split(".")[0]
        by_op[op] += int(r[si])
        try:
            inst_op[op] += int(r[ex])
        except ValueError:
            pass
        for h, i in idx.items():
            try:
                tot[h] += int(r[i])
            except ValueError:
                pass
    s = sum(tot.values())
    print("stall reasons (share of samples):")
    for h, v in tot.most_common(12):
        print("  %-28s %6.1f%%" % (h, 100.0 * v / max(s, 1)))
    print("samples by opcode:")
    for h, v in by_op.most_common(12):
        print("  %-10s %6.1f%%   executed %d" % (h, 100.0 * v / max(sum(by_op.values()), 1), inst_op[h]))
    n = sum(inst_op.values())
    print("executed instructions by opcode (share):")
    for h, v in inst_op.most_common(14):
        print("  %-10s %6.1f%%" % (h, 100.0 * v / max(n, 1)))


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 0)
