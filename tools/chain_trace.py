"""Per-(step, CTA) timeline of the persistent decode-chain kernel
(fasq_chain_trace): where does a decode token's time go?

    python tools/chain_trace.py [--blocks 32] [--json out.json]

Stamps per (step, CTA): t0 step entry, t1 inputs final + staged (dataflow
wait), t2 CTA synchronised, t3 outputs stored.  Reported per step kind (qkv,
o, gateup, down), medians over blocks: step span (last t3 of the previous
step -> last t3 of this step), "barrier" = input wait (last t3 of prev ->
median t1), "xstage" = t2 - t1, compute (t2 -> t3) min / median / max over
CTAs, and the idle tail (max t3 - median t3).
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

import paper_2605_04084_b200 as F
import synth

KINDS = ["qkv", "o", "gateup", "down"]
NAMES = [("q_proj", "k_proj", "v_proj"), ("o_proj",), ("gate_proj", "up_proj"), ("down_proj",)]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--blocks", type=int, default=32)
    ap.add_argument("--d", type=int, default=2)
    ap.add_argument("--C", type=int, default=256)
    ap.add_argument("--json", default=None)
    a = ap.parse_args()
    blocks = []
    for b in range(a.blocks):
        Ls = {}
        for li, (name, fo, fi) in enumerate(synth.LLAMA3_8B_LAYERS):
            cb, idx = synth.torch_random_layer(fo, fi, a.d, a.C, seed=b * 7 + li)
            Ls[name] = F.import_layer(cb, idx, fi)
        blocks.append(Ls)
    steps = []
    for b in range(a.blocks):
        for i in range(4):
            steps.append(([blocks[b][n] for n in NAMES[i]], None if not steps else (len(steps) - 1, 0)))
    ch = F.Chain(steps, B=1)
    x = synth.torch_activation(1, 4096)
    T = len(steps)
    buf = torch.zeros((T, ch.ctas, 4), dtype=torch.int64, device="cuda")
    for _ in range(3):
        ch.run(x)
    torch.cuda.synchronize()
    # untraced timing for reference
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        ch.run(x)
    e1.record()
    torch.cuda.synchronize()
    plain_us = e0.elapsed_time(e1) * 100.0
    ch.trace(buf)
    ch.run(x)
    torch.cuda.synchronize()
    t = buf.cpu().numpy().astype(np.int64)
    ch.trace(None)
    t0 = t[:, :, 0].min()
    t = np.where(t > 0, t - t0, 0)
    prev_end = 0
    rows = {k: [] for k in KINDS}
    for s in range(T):
        st = t[s]
        end = st[:, 3].max()
        have = st[:, 2] > 0   # CTAs with work in this step
        rec = {
            "span": end - prev_end,
            "notice_min": st[have, 1].min() - prev_end if s else 0,
            "notice_max": st[have, 1].max() - prev_end if s else 0,
            "barrier": np.median(st[:, 1]) - prev_end if s else 0,
            "xstage": np.median(st[have, 2] - st[have, 1]),
            "comp_min": (st[have, 3] - st[have, 2]).min(),
            "comp_med": np.median(st[have, 3] - st[have, 2]),
            "comp_max": (st[have, 3] - st[have, 2]).max(),
            "active": int(have.sum()) * 1000,
            "tail": end - np.median(st[:, 3]),
            # staging latency of CTAs whose inputs were already final when they
            # started polling (t0 after the previous step's end): ~ one poll round trip
            "stage_min": (st[have, 1] - st[have, 0]).min(),
            "stage_med": np.median(st[have, 1] - st[have, 0]),
        }
        rows[KINDS[s % 4]].append(rec)
        prev_end = end
    total = t[:, :, 3].max()
    out = {"plain_us": plain_us, "traced_us": float(total) / 1e3, "kinds": {}}
    print(f"token: {plain_us:.1f} us untraced, {total / 1e3:.1f} us traced; {T} steps, {ch.ctas} CTAs")
    print(f"{'kind':8s} " + " ".join(f"{k:>9s}" for k in rows[KINDS[0]][0]))
    for k in KINDS:
        med = {f: float(np.median([r[f] for r in rows[k]])) / 1e3 for f in rows[k][0]}
        out["kinds"][k] = med
        print(f"{k:8s} " + " ".join(f"{v:9.2f}" for v in med.values()))
    if a.json:
        with open(a.json, "w") as f:
            json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
