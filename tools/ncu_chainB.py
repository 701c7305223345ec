"""ncu driver: the 32-block PQ chain (bench pq_chain / decode_batch) at batch B:
3 runs of one k_chain launch.  usage: python tools/ncu_chainB.py B"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2605_04084_b200 as F
import synth

B = int(sys.argv[1]) if len(sys.argv) > 1 else 8
NAMES = [("q_proj", "k_proj", "v_proj"), ("o_proj",), ("gate_proj", "up_proj"), ("down_proj",)]
blocks = []
for b in range(32):
    Ls = {}
    for li, (name, fo, fi) in enumerate(synth.LLAMA3_8B_LAYERS):
        cb, idx = synth.torch_random_layer(fo, fi, 2, 256, seed=b * 7 + li)
        Ls[name] = F.import_layer(cb, idx, fi)
    blocks.append(Ls)
steps = []
for b in range(32):
    for i in range(4):
        steps.append(([blocks[b][n] for n in NAMES[i]], None if not steps else (len(steps) - 1, 0)))
ch = F.Chain(steps, B=B)
x = synth.torch_activation(B, 4096)
for _ in range(3):
    ch.run(x)
torch.cuda.synchronize()
print("done")
