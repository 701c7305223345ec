"""Per-layer GEMV timing sweep (development tool; bench.py is the contract).

Cycles through enough layer replicas to exceed L2 so every launch streams
from HBM; CUDA events on the launching stream; algorithmic bytes =
indices + codebooks + x + y.
"""
import argparse
import json
import sys
import os

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2605_04084_b200 as F
import synth
from oracle import sizemodel as sm


def run(F_out, F_in, d, C, B, iters=200, flags=0, min_bytes=600e6):
    lb = sm.gemv_algorithmic_bytes(F_out, F_in, d, C, 1, B, 4)
    nrep = max(2, int(min_bytes // lb) + 1)
    layers = []
    for r in range(nrep):
        cb, idx = synth.torch_random_layer(F_out, F_in, d, C, seed=r)
        layers.append(F.import_layer(cb, idx, F_in))
        del cb, idx
    x = synth.torch_activation(B, F_in)
    ys = [torch.empty((B, F_out), dtype=torch.float32, device="cuda") for _ in range(nrep)]
    # warm-up on the capture stream (sizes that stream's split-K workspace
    # outside capture, as a user of a captured decode loop would)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for i in range(2 * nrep):
            F.gemv(layers[i % nrep], x, out=ys[i % nrep], flags=flags)
    torch.cuda.synchronize()
    # capture `iters` launches in a CUDA graph so host overhead is excluded
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
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / iters
    return {"F_out": F_out, "F_in": F_in, "d": d, "C": C, "B": B, "us": round(us, 3),
            "GBps": round(lb / us / 1e3, 1), "reps": nrep, "flags": flags}


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--quick", action="store_true")
    a = ap.parse_args()
    shapes = [(4096, 4096), (1024, 4096), (14336, 4096), (4096, 14336)]
    for (o, i) in shapes:
        for C in (256, 128):
            for flags in (0, 1):
                print(json.dumps(run(o, i, 2, C, 1, flags=flags)), flush=True)
    for B in (2, 4, 8):
        print(json.dumps(run(4096, 4096, 2, 256, B)), flush=True)
        print(json.dumps(run(14336, 4096, 2, 256, B)), flush=True)
    for d, C in ((1, 256), (4, 256), (8, 256), (2, 16), (2, 64)):
        print(json.dumps(run(4096, 4096, d, C, 1)), flush=True)
