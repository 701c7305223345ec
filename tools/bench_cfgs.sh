#!/bin/bash
# decode-step tok/s for several GEMV tilings (bench.py workload, no side runs)
for c in ${CFGS:-"4,8,3" "8,4,3" "4,4,4" "2,8,4" "8,8,2" "2,16,3"}; do
  echo "cfg $c"; FASQ_GEMV_CFG=$c timeout 300 python bench.py --steps 100 --warmup 3 --no-side 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'cfg':'$c','tok_s':d['value'],'frac':d['roofline']['frac'],'e2e':d['e2e']['value']}))"
done
