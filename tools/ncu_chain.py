"""ncu driver: one Llama block as a decode chain in FASQ_ACC_I64 mode (as bench.py N=1)."""
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
z = lambda n: torch.zeros((1, n), dtype=torch.int64, device="cuda")
for _ in range(3):
    q, k, v = F.gemv_grouped([Ls["q_proj"], Ls["k_proj"], Ls["v_proj"]], h, outs=[z(4096), z(1024), z(1024)],
                             next_layers=[Ls["o_proj"]])
    o, = F.gemv_grouped([Ls["o_proj"]], q, outs=[z(4096)], next_layers=[Ls["gate_proj"], Ls["up_proj"]])
    g, u = F.gemv_grouped([Ls["gate_proj"], Ls["up_proj"]], o, outs=[z(14336), z(14336)], next_layers=[Ls["down_proj"]])
    d, = F.gemv_grouped([Ls["down_proj"]], g, outs=[z(4096)])
torch.cuda.synchronize()
print("done")
