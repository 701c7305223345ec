"""ncu driver for the round-2 per-launch kernels: python tools/ncu_newk.py {tc|packed|dim0}
(tc: tcgen05 batched decode B = 16 on 4096x14336; packed: 10-bit (2,1024) GEMV on
14336x4096, B = 1; dim0: dim = 0 GEMV on 4096x4096, B = 8).  Three launches each."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2605_04084_b200 as F
import synth

what = sys.argv[1]
if what == "tc":
    cb, idx = synth.torch_random_layer(4096, 14336, 2, 256, seed=1)
    L, B, fi = F.import_layer(cb, idx, 14336), 16, 14336
elif what == "packed":
    cb, idx = synth.torch_random_layer(14336, 4096, 2, 1024, seed=1)
    L, B, fi = F.import_layer(cb, idx, 4096, packed=True), 1, 4096
else:
    g = torch.Generator(device="cuda"); g.manual_seed(1)
    cb = (torch.randn((2048, 256, 2), generator=g, device="cuda") / 64).half()
    idx = torch.randint(0, 256, (2048, 4096), generator=g, device="cuda", dtype=torch.int32).to(torch.uint8)
    L, B, fi = F.import_layer(cb, idx, 4096, dim0=True), 8, 4096
x = synth.torch_activation(B, fi)
for _ in range(3):
    F.gemv(L, x)
torch.cuda.synchronize()
print("done")
