"""Times fasq_gemm on one layer shape: python tools/gemm_time.py F_out F_in M [expand|lut] [iters]
(FASQ_GEMM_KSPLIT applies)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2605_04084_b200 as F
import synth

o, i, M = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
algo = F.GEMM_LUT if len(sys.argv) > 4 and sys.argv[4] == "lut" else F.GEMM_EXPAND_TC
it = int(sys.argv[5]) if len(sys.argv) > 5 else 20
cb, idx = synth.torch_random_layer(o, i, 2, 256, seed=1)
L = F.import_layer(cb, idx, i)
X = synth.torch_activation(M, i)
Y = torch.empty((M, o), dtype=torch.float16, device="cuda")
for _ in range(3):
    F.gemm(L, X, out=Y, algo=algo)
torch.cuda.synchronize()
# device time: the launches replayed from a CUDA graph (host overhead excluded)
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
g = torch.cuda.CUDAGraph()
with torch.cuda.stream(s):
    with torch.cuda.graph(g, stream=s):
        for _ in range(it):
            F.gemm(L, X, out=Y, algo=algo)
torch.cuda.synchronize()
g.replay()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
g.replay()
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / it
print("%dx%d M=%d ks=%s  %.4f ms  %.1f TFLOP/s" % (o, i, M, os.environ.get("FASQ_GEMM_KSPLIT", "auto"), ms,
                                                   2.0 * M * o * i / ms / 1e9))
