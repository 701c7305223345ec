"""Times one decode token of the persistent chain (32 Llama-3-8B blocks, B=1)
with CUDA events; prints ms/token and algorithmic TB/s.  Environment knobs of
the library (FASQ_CHAIN_CFG, FASQ_CHAIN_DBG, ...) apply.
usage: python tools/chain_time.py [d] [C] [B]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2605_04084_b200 as F
import synth

NAMES = [("q_proj", "k_proj", "v_proj"), ("o_proj",), ("gate_proj", "up_proj"), ("down_proj",)]
d = int(sys.argv[1]) if len(sys.argv) > 1 else 2
C = int(sys.argv[2]) if len(sys.argv) > 2 else 256
B = int(sys.argv[3]) if len(sys.argv) > 3 else 1
nb = 32
blocks, nbytes = [], 0
for b in range(nb):
    Ls = {}
    for li, (name, fo, fi) in enumerate(synth.LLAMA3_8B_LAYERS):
        cb, idx = synth.torch_random_layer(fo, fi, d, C, seed=int(os.environ.get("SEEDBASE", "0")) + b * 7 + li)
        Ls[name] = F.import_layer(cb, idx, fi)
        nbytes += fo * fi // d + (fi // d) * C * d * 2 + 2 * B * fi + 4 * B * fo
    blocks.append(Ls)
steps = []
for b in range(nb):
    for i in range(4):
        steps.append(([blocks[b][n] for n in NAMES[i]], None if not steps else (len(steps) - 1, 0)))
ch = F.Chain(steps, B=B)
x = synth.torch_activation(B, 4096)
if os.environ.get("XZERO"):
    x.zero_()
for _ in range(int(os.environ.get("WARM", "5"))):
    ch.run(x)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
n = int(os.environ.get("NRUN", "50"))
e0.record()
for _ in range(n):
    ch.run(x)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / n
print("d=%d C=%d B=%d env=%s  %.4f ms/token  %.1f tok/s  %.3f TB/s algorithmic" % (
    d, C, B, {k: v for k, v in os.environ.items() if k.startswith("FASQ_")}, ms, 1e3 / ms, nbytes / ms / 1e9))
