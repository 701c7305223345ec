"""One EXPAND launch at M = 128 on 4096 x 4096 (split-K 8) for ncu (development tool)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("FASQ_GEMM_TC_DECODE_MAX", "0")
import torch

import paper_2605_04084_b200 as F
import synth

o, i, M = (int(v) for v in (sys.argv[1:4] if len(sys.argv) > 3 else (4096, 4096, 128)))
cb, idx = synth.torch_random_layer(o, i, 2, 256, seed=1)
L = F.import_layer(cb, idx, i)
X = synth.torch_activation(M, i)
Y = torch.empty((M, o), dtype=torch.float16, device="cuda")
for _ in range(3):
    F.gemm(L, X, out=Y)
torch.cuda.synchronize()
