"""ncu driver: repeated GEMVs on one layer shape (argv: F_out F_in [B])."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2605_04084_b200 as F
import synth
o, i = int(sys.argv[1]), int(sys.argv[2])
B = int(sys.argv[3]) if len(sys.argv) > 3 else 1
cb, idx = synth.torch_random_layer(o, i, 2, 256, seed=1)
L = F.import_layer(cb, idx, i)
x = synth.torch_activation(B, i)
for _ in range(5):
    F.gemv(L, x)
torch.cuda.synchronize()
print("done")
