"""NEXT-2 per-launch GEMV timing: byte indices vs ceil(log2 C)-bit packed
indices on the Llama-3-8B shapes (development tool; bench.py reports the same
numbers under side.packed_gemv).  Replicas over > L2, CUDA graph of launches,
CUDA events; algorithmic bytes = Eq. 4 index bits + codebooks + x + y."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2605_04084_b200 as F
import synth


def layer_bytes(F_out, F_in, C, bits, B=1):
    N_ss = F_in // 2
    return (N_ss * F_out * bits + 7) // 8 + N_ss * C * 2 * 2 + 2 * B * F_in + 4 * B * F_out


def run(F_out, F_in, C, packed, B=1, iters=200, min_bytes=600e6, flags=1):
    bits = max(1, (C - 1).bit_length()) if packed else 8
    lb = layer_bytes(F_out, F_in, C, bits, B)
    nrep = max(2, int(min_bytes // lb) + 1)
    layers = []
    for r in range(nrep):
        cb, idx = synth.torch_random_layer(F_out, F_in, 2, C, seed=r)
        layers.append(F.import_layer(cb, idx, F_in, packed=packed))
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
    return {"F_out": F_out, "F_in": F_in, "C": C, "bits": bits, "B": B, "us": round(us, 3),
            "bytes": lb, "GBps": round(lb / us / 1e3, 1)}


if __name__ == "__main__":
    shapes = [(4096, 4096), (14336, 4096), (4096, 14336)]
    for (o, i) in shapes:
        for C, packed in ((256, False), (128, False), (128, True), (512, True), (1024, True)):
            print(json.dumps(run(o, i, C, packed)), flush=True)
    for B in (2, 8):
        for C, packed in ((256, False), (512, True)):
            print(json.dumps(run(4096, 4096, C, packed, B=B)), flush=True)
