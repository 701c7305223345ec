"""Short-L / large-batch dispatch sweep (NEXT-3): per Llama
shape and M, device time of the decode GEMV (M <= 8), GEMM-LUT (split-K for
short L) and GEMM-EXPAND (tcgen05), each from a CUDA graph of 20 launches over
8 layer replicas (> L2 for the big shapes).  Prints one JSON line per (shape, M)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2605_04084_b200 as F
import synth


def timeit(fn, n=20):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn(0)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for i in range(n):
            fn(i)
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


for (fo, fi) in [(4096, 4096), (14336, 4096), (4096, 14336)]:
    Ls = []
    for r in range(8):
        cb, idx = synth.torch_random_layer(fo, fi, 2, 256, seed=r)
        Ls.append(F.import_layer(cb, idx, fi))
    for M in (1, 4, 8, 16, 32, 64, 128, 256):
        X = synth.torch_activation(M, fi)
        Y = torch.empty((M, fo), dtype=torch.float16, device="cuda")
        out = {"shape": "%dx%d" % (fo, fi), "M": M}
        if M <= 8:
            out["gemv_ms"] = round(timeit(lambda i: F.gemv(Ls[i % 8], X, out=Y)), 4)
        for name, algo in (("lut", F.GEMM_LUT), ("expand", F.GEMM_EXPAND_TC)):
            try:
                out[name + "_ms"] = round(timeit(lambda i: F.gemm(Ls[i % 8], X, out=Y, algo=algo)), 4)
            except Exception as e:
                out[name + "_ms"] = str(e)[:60]
        print(json.dumps(out), flush=True)
    for L in Ls:
        L.free()
