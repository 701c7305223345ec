"""GEMM-LUT short-L split-K A/B (FASQ_LUT_KSPLIT=1 disables): ms per launch."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2605_04084_b200 as F
import synth
for (fo, fi) in [(4096, 4096), (4096, 14336)]:
    cb, idx = synth.torch_random_layer(fo, fi, 2, 256, seed=1)
    L = F.import_layer(cb, idx, fi)
    for M in (8, 32, 128):
        X = synth.torch_activation(M, fi)
        Y = torch.empty((M, fo), dtype=torch.float16, device="cuda")
        for _ in range(3):
            F.gemm(L, X, out=Y, algo=F.GEMM_LUT)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            F.gemm(L, X, out=Y, algo=F.GEMM_LUT)
        e1.record()
        torch.cuda.synchronize()
        print("%dx%d M=%d ks=%s %.4f ms" % (fo, fi, M, os.environ.get("FASQ_LUT_KSPLIT", "auto"), e0.elapsed_time(e1) / 10))
