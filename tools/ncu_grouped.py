"""ncu driver: grouped GEMVs of one Llama block (qkv, o, gate+up, down)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2605_04084_b200 as F
import synth
Ls = {}
for li, (name, fo, fi) in enumerate(synth.LLAMA3_8B_LAYERS):
    cb, idx = synth.torch_random_layer(fo, fi, 2, 256, seed=li)
    Ls[name] = F.import_layer(cb, idx, fi)
h = synth.torch_activation(1, 4096)
for _ in range(3):
    q, k, v = F.gemv_grouped([Ls["q_proj"], Ls["k_proj"], Ls["v_proj"]], h, out_dtype=torch.float16)
    o = F.gemv(Ls["o_proj"], q, out_dtype=torch.float16)
    g, u = F.gemv_grouped([Ls["gate_proj"], Ls["up_proj"]], o, out_dtype=torch.float16)
    d = F.gemv(Ls["down_proj"], g, out_dtype=torch.float16)
torch.cuda.synchronize()
print("done")
