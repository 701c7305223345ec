"""Writes profiles/<round>/ncu_traffic.json: dram bytes (read + write) per launch
of each kernel in an `ncu --page raw --csv` export (bench.py's roofline.traffic)."""
import csv
import json
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, data = rows[0], rows[2:]
ki = hdr.index("Kernel Name")
rd, wr = hdr.index("dram__bytes_read.sum"), hdr.index("dram__bytes_write.sum")
unit_r, unit_w = rows[1][rd], rows[1][wr]
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
out = {}
for r in data:
    name = "k_chain" if "k_chain" in r[ki] else "k_lm_head" if "k_lm_head" in r[ki] else r[ki][:40]
    v = float(r[rd].replace(",", "")) * scale.get(unit_r, 1) + float(r[wr].replace(",", "")) * scale.get(unit_w, 1)
    out.setdefault(name, []).append(v)
res = {k: sum(v) / len(v) for k, v in out.items()}
json.dump(res, open(sys.argv[2], "w"), indent=1)
print(res)
