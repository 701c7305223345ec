"""ncu driver: GPU k-means pack of one 4096x4096 layer (d=2, C=256, 25 rounds)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2605_04084_b200 as F
import synth

W = synth.torch_activation(4096, 4096, seed=5, std=0.02)
for _ in range(2):
    F.pack(W, d=2, C=256, group=1, seed=0, iters=25).free()
torch.cuda.synchronize()
print("done")
