"""ncu driver: prefill GEMM (EXPAND tcgen05 or LUT) on one layer shape.
usage: python tools/ncu_gemm.py F_out F_in M [expand|lut]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2605_04084_b200 as F
import synth

o, i, M = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
algo = F.GEMM_LUT if len(sys.argv) > 4 and sys.argv[4] == "lut" else F.GEMM_EXPAND_TC
cb, idx = synth.torch_random_layer(o, i, 2, 256, seed=1)
L = F.import_layer(cb, idx, i)
X = synth.torch_activation(M, i)
Y = torch.empty((M, o), dtype=torch.float16, device="cuda")
for _ in range(3):
    F.gemm(L, X, out=Y, algo=algo)
torch.cuda.synchronize()
print("done")
