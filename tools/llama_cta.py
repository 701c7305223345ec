"""Per-CTA compute time (t2 -> t3) of one step kind of the whole-model chain,
median over blocks: which CTAs are the slow tail?  usage: llama_cta.py [kind]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
sys.argv += [] 
import tools.llama_trace as lt

kind = sys.argv[1] if len(sys.argv) > 1 else "down"
KI = {"qkv": 0, "attn": 1, "o": 2, "gateup": 3, "down": 4}[kind]
model = lt.build(32, 2, 256, 1)
for _ in range(5):
    model.step()
torch.cuda.synchronize()
T = 161
buf = torch.zeros((T, model.chain.ctas, 4), dtype=torch.int64, device="cuda")
model.chain.trace(buf)
model.step()
torch.cuda.synchronize()
t = buf.cpu().numpy().astype(np.int64)
comp = np.stack([t[1 + 5 * l + KI, :, 3] - t[1 + 5 * l + KI, :, 2] for l in range(32)])   # [blocks][ctas]
wait = np.stack([t[1 + 5 * l + KI, :, 1] - t[1 + 5 * l + KI, :, 0] for l in range(32)])
med = np.median(comp, axis=0) / 1e3
wmed = np.median(wait, axis=0) / 1e3
order = np.argsort(-med)
print("slowest CTAs (cta, comp_us, stage_wait_us):", [(int(c), round(float(med[c]), 2), round(float(wmed[c]), 2)) for c in order[:12]])
print("fastest:", [(int(c), round(float(med[c]), 2)) for c in order[-6:]])
print("median comp %.2f, mean %.2f" % (np.median(med), med.mean()))
