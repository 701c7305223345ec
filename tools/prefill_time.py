"""Whole-model prefill timing (development tool): the bench model (32 Llama-3-8B
blocks, d = 2 / C = 256), one 128-token prompt through fasq_llama_prefill;
eager calls vs the same call captured in a CUDA graph (launch gaps), CUDA
events.  Under `ncu --metrics gpu__time_duration.sum` with --ncu it runs ONE
call after warm-up so the launch list is one prefill."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench

M = int(os.environ.get("PF_M", "128"))
model, _ = bench.build_llama(0, 1)
toks = torch.arange(1000, 1000 + M, dtype=torch.int32, device="cuda")
model.prefill(toks, 0)
torch.cuda.synchronize()
if "--ncu" in sys.argv:
    torch.cuda.cudart().cudaProfilerStart()
    model.prefill(toks, 0)
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStop()
    sys.exit(0)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    model.prefill(toks, 0)
e1.record()
torch.cuda.synchronize()
eager = e0.elapsed_time(e1) / 5
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
g = torch.cuda.CUDAGraph()
with torch.cuda.stream(s):
    model.prefill(toks, 0)
    torch.cuda.synchronize()
    with torch.cuda.graph(g, stream=s):
        model.prefill(toks, 0)
torch.cuda.synchronize()
g.replay()
torch.cuda.synchronize()
e0.record()
for _ in range(5):
    g.replay()
e1.record()
torch.cuda.synchronize()
print(json.dumps({"M": M, "eager_ms": round(eager, 3), "graph_ms": round(e0.elapsed_time(e1) / 5, 3)}))
