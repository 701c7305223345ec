"""bench.prefill_model alone (development tool): whole PQ-stack prefill pass at M = 128 / 512 / 2048."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench

pk, _ = bench._peaks()
print(json.dumps(bench.prefill_model(pk.get("bf16_tflops", 1590.0))))
