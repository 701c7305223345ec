"""Small driver for ncu captures of the GEMV kernel (development tool)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2605_04084_b200 as F
import synth

shapes = [(int(a), int(b)) for a, b in (s.split("x") for s in (sys.argv[1:] or ["4096x4096", "14336x4096"]))]
for (o, i) in shapes:
    cb, idx = synth.torch_random_layer(o, i, 2, 256, seed=1)
    L = F.import_layer(cb, idx, i)
    x = synth.torch_activation(1, i)
    for _ in range(3):
        y = F.gemv(L, x)
torch.cuda.synchronize()
print("done")
