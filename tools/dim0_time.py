"""NEXT-4 per-launch GEMV timing: Eq. 3's input-axis layout vs the paper's
dim = 0 (output-axis) layout on the Llama-3-8B shapes, d = 2, C = 256 (B = 1, 8;
CUDA graph of launches over > L2 of replicas; development tool -- bench.py
reports the same under side.dim0_gemv)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2605_04084_b200 as F
import synth


def run(F_out, F_in, dim0, B=1, C=256, iters=200, min_bytes=600e6, flags=1):
    lb = (F_in // 2) * F_out + (F_in // 2) * C * 4 + 2 * B * F_in + 4 * B * F_out
    nrep = max(2, int(min_bytes // lb) + 1)
    layers = []
    for r in range(nrep):
        if dim0:
            g = torch.Generator(device="cuda")
            g.manual_seed(r)
            cb = (torch.randn((F_out // 2, C, 2), generator=g, device="cuda") / F_in ** 0.5).half()
            idx = torch.randint(0, C, (F_out // 2, F_in), generator=g, device="cuda", dtype=torch.int32).to(torch.uint8)
        else:
            cb, idx = synth.torch_random_layer(F_out, F_in, 2, C, seed=r)
        layers.append(F.import_layer(cb, idx, F_in, dim0=dim0))
        del cb, idx
    x = synth.torch_activation(B, F_in)
    ys = [torch.empty((B, F_out), dtype=torch.float32, device="cuda") for _ in range(nrep)]
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for i in range(2 * nrep):
            F.gemv(layers[i % nrep], x, out=ys[i % nrep], flags=flags)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            for i in range(iters):
                F.gemv(layers[i % nrep], x, out=ys[i % nrep], flags=flags)
    torch.cuda.synchronize()
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.replay(); g.replay()
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / (2 * iters)
    del layers
    torch.cuda.empty_cache()
    return {"F_out": F_out, "F_in": F_in, "dim0": dim0, "B": B, "us": round(us, 3), "bytes": lb,
            "GBps": round(lb / us / 1e3, 1)}


if __name__ == "__main__":
    for (o, i) in ((4096, 4096), (14336, 4096), (4096, 14336), (1024, 4096)):
        for B in (1, 8):
            for dim0 in (False, True):
                print(json.dumps(run(o, i, dim0, B=B)), flush=True)
