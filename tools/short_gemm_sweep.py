"""Short-L prefill (fasq_gemm AUTO, M = 8..256): the tcgen05 decode kernel
(FASQ_GEMM_TC_DECODE_MAX >= M) vs the EXPAND / LUT path (=0), Llama shapes;
CUDA graph of 20 launches, CUDA events."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2605_04084_b200 as F
import synth


def run(o, i, M, short, it=20):
    os.environ["FASQ_GEMM_TC_DECODE_MAX"] = "256" if short else "0"
    cb, idx = synth.torch_random_layer(o, i, 2, 256, seed=1)
    L = F.import_layer(cb, idx, i)
    X = synth.torch_activation(M, i)
    Y = torch.empty((M, o), dtype=torch.float16, device="cuda")
    for _ in range(3):
        F.gemm(L, X, out=Y)
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            for _ in range(it):
                F.gemm(L, X, out=Y)
    torch.cuda.synchronize()
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / it
    return {"F_out": o, "F_in": i, "M": M, "path": "tcgen05-decode" if short else "expand/lut", "us": round(us, 2),
            "tflops": round(2.0 * M * o * i / us / 1e6, 1)}


if __name__ == "__main__":
    for (o, i) in ((4096, 4096), (14336, 4096), (4096, 14336), (1024, 4096)):
        for M in (16, 32, 64, 96, 128, 192, 256):
            for short in (False, True):
                print(json.dumps(run(o, i, M, short)), flush=True)
