"""Decode GEMV throughput vs batch (B = 1..8): per-launch grouped GEMV over the
Llama-3-8B gate/up pair and the persistent chain over 8 blocks; HBM bytes =
indices + codebooks per launch (x, y negligible).  Graph-timed."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import json

import torch

import paper_2605_04084_b200 as F
import synth

NAMES = [("q_proj", "k_proj", "v_proj"), ("o_proj",), ("gate_proj", "up_proj"), ("down_proj",)]


def graph_time(fn, reps=50):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn()
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        fn()
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    nb = 8
    blocks = []
    for b in range(nb):
        Ls = {}
        for li, (name, fo, fi) in enumerate(synth.LLAMA3_8B_LAYERS):
            cb, idx = synth.torch_random_layer(fo, fi, 2, 256, seed=b * 7 + li)
            Ls[name] = F.import_layer(cb, idx, fi)
        blocks.append(Ls)
    byt_block = sum(fi // 2 * fo + fi // 2 * 256 * 4 for (_, fo, fi) in synth.LLAMA3_8B_LAYERS)
    gu = [blocks[0]["gate_proj"], blocks[0]["up_proj"]]
    byt_gu = 2 * (2048 * 14336 + 2048 * 256 * 4)
    for B in (1, 2, 4, 8):
        x = synth.torch_activation(B, 4096)
        outs = [torch.empty((B, 14336), dtype=torch.float16, device="cuda") for _ in range(2)]
        ms = graph_time(lambda: F.gemv_grouped(gu, x, outs=outs))
        steps = []
        for b in range(nb):
            for i in range(4):
                steps.append(([blocks[b][n] for n in NAMES[i]], None if not steps else (len(steps) - 1, 0)))
        ch = F.Chain(steps, B=B)
        msc = graph_time(lambda: ch.run(x))
        ch.free()
        print(json.dumps({"B": B, "gateup_launch_us": ms * 1e3, "gateup_TBps": byt_gu / (ms * 1e-3) / 1e12,
                          "chain_8blocks_us": msc * 1e3, "chain_TBps": nb * byt_block / (msc * 1e-3) / 1e12,
                          "chain_tokens_per_s": B * 32 / nb * 0 + B * 1000.0 / (msc * 32 / nb)}))


if __name__ == "__main__":
    main()
