"""ncu driver: a few chained GEMVs of each Llama shape (launch-list capture)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2605_04084_b200 as F
import synth
Ls = []
for (o, i) in [(4096, 4096), (1024, 4096), (14336, 4096), (4096, 14336)]:
    cb, idx = synth.torch_random_layer(o, i, 2, 256, seed=1)
    Ls.append((F.import_layer(cb, idx, i), i))
for rep in range(3):
    for L, i in Ls:
        x = synth.torch_activation(1, i)
        F.gemv(L, x)
torch.cuda.synchronize()
print("done")
