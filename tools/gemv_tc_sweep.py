"""Per-launch decode GEMV at batch B: the CUDA-core kernels (B <= 8) / prefill
GEMM (B > 8) vs the tcgen05 decode kernel (gemv_tc.cu), Llama-3-8B shapes,
d = 2, C = 256; CUDA graph of launches over > L2 of layer replicas, CUDA events.
Prints one JSON line per (shape, B, path)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2605_04084_b200 as F
import synth


def run(F_out, F_in, B, tc, iters=100, min_bytes=400e6):
    os.environ["FASQ_GEMV_TC_MIN_B"] = "1" if tc else "0"
    lb = (F_in // 2) * F_out + (F_in // 2) * 256 * 4 + 2 * B * F_in + 4 * B * F_out
    nrep = max(2, int(min_bytes // lb) + 1)
    layers = []
    for r in range(nrep):
        cb, idx = synth.torch_random_layer(F_out, F_in, 2, 256, seed=r)
        layers.append(F.import_layer(cb, idx, F_in))
        del cb, idx
    x = synth.torch_activation(B, F_in)
    ys = [torch.empty((B, F_out), dtype=torch.float32, device="cuda") for _ in range(nrep)]
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for i in range(2 * nrep):
            F.gemv(layers[i % nrep], x, out=ys[i % nrep])
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            for i in range(iters):
                F.gemv(layers[i % nrep], x, out=ys[i % nrep])
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
    return {"F_out": F_out, "F_in": F_in, "B": B, "path": "tcgen05" if tc else "default", "us": round(us, 3),
            "GBps": round(lb / us / 1e3, 1)}


if __name__ == "__main__":
    for (o, i) in ((4096, 4096), (14336, 4096), (4096, 14336), (1024, 4096)):
        for B in (1, 2, 4, 8, 16, 32, 64):
            for tc in (False, True):
                print(json.dumps(run(o, i, B, tc)), flush=True)
