"""ncu driver: whole-model decode (bench.build_llama, 32 Llama-3-8B blocks,
(2,256), B=1): 6 eager steps (k_chain MODEL + k_lm_head per step)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench

model, by = bench.build_llama(0, 1)
model.reset([128000], bench.PROMPT)
for _ in range(int(os.environ.get("NSTEPS", "6"))):
    model.step()
torch.cuda.synchronize()
print("done", by)
