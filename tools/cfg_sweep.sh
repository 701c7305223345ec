#!/bin/bash
# GEMV tiling sweep on the Llama shapes (B=1, d=2, C=256), graph-timed.
for c in "2,16,3" "1,16,3" "4,8,3" "2,8,3" "4,16,2" "1,8,3"; do
FASQ_GEMV_CFG=$c python - <<PY
import sys, json; sys.path.insert(0, ".")
from tools.gemv_sweep import run
for (o, i) in [(4096, 4096), (1024, 4096), (14336, 4096), (4096, 14336)]:
    try:
        r = run(o, i, 2, 256, 1, flags=1); r["cfg"] = "$c"; print(json.dumps(r), flush=True)
    except Exception as e:
        print(json.dumps({"cfg": "$c", "shape": [o, i], "error": str(e)[:200]}), flush=True)
PY
done
