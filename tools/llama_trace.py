"""Per-step timeline of whole-model decode (fasq_llama_*; chain trace stamps):
where does a Llama-3-8B-shaped decode token's time go?

    python tools/llama_trace.py [--layers 32] [--B 1] [--C 256] [--json out.json]

Per step kind (embed, qkv, attn, o, gateup, down), medians over blocks: span
(last t3 of the previous step -> last t3 of this step), input wait, compute
min/median/max over CTAs with work, idle tail.  The lm_head kernel is timed
as the step time minus the traced chain span (upper bound: includes the
launch gap)."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2605_04084_b200 as F
import synth

KINDS = ["qkv", "attn", "o", "gateup", "down"]


def build(nl, d, C, B, max_T=256):
    hid, H, KV, hd, ffn, vocab = 4096, 32, 8, 128, 14336, 128256
    shapes = {"q": (H * hd, hid), "k": (KV * hd, hid), "v": (KV * hd, hid), "o": (hid, H * hd),
              "gate": (ffn, hid), "up": (ffn, hid), "down": (hid, ffn)}
    g = torch.Generator(device="cuda")
    g.manual_seed(0)
    layers = []
    for l in range(nl):
        L = {}
        for i, (n, (fo, fi)) in enumerate(shapes.items()):
            cb, idx = synth.torch_random_layer(fo, fi, d, C, seed=l * 7 + i)
            L[n] = F.import_layer(cb, idx, fi)
        L["attn_norm"] = (1 + 0.1 * torch.randn(hid, generator=g, device="cuda")).half()
        L["mlp_norm"] = (1 + 0.1 * torch.randn(hid, generator=g, device="cuda")).half()
        layers.append(L)
    fn = (1 + 0.1 * torch.randn(hid, generator=g, device="cuda")).half()
    emb = torch.randn((vocab, hid), generator=g, device="cuda").half()
    lm = (torch.randn((vocab, hid), generator=g, device="cuda") / hid ** 0.5).half()
    model = F.Llama(layers, fn, emb, lm, H, KV, hd, vocab, max_T=max_T, pos_wrap=128, B=B)
    for l in range(nl):
        K, V = model.kv_cache(l)
        K.normal_(generator=g)
        V.normal_(generator=g)
    model.reset([128000 + b for b in range(B)], 128)
    return model


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", type=int, default=32)
    ap.add_argument("--B", type=int, default=1)
    ap.add_argument("--d", type=int, default=2)
    ap.add_argument("--C", type=int, default=256)
    ap.add_argument("--json", default=None)
    a = ap.parse_args()
    model = build(a.layers, a.d, a.C, a.B)
    for _ in range(5):
        model.step()
    torch.cuda.synchronize()
    e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    n = 20
    e[0].record()
    for _ in range(n):
        model.step()
    e[1].record()
    torch.cuda.synchronize()
    step_us = e[0].elapsed_time(e[1]) * 1e3 / n
    T = 1 + 5 * a.layers
    ctas = model.chain.ctas
    buf = torch.zeros((T, ctas, 4), dtype=torch.int64, device="cuda")
    model.chain.trace(buf)
    model.step()
    torch.cuda.synchronize()
    t = buf.cpu().numpy().astype(np.int64)
    model.chain.trace(None)
    t0 = t[:, :, 0][t[:, :, 0] > 0].min()
    t = np.where(t > 0, t - t0, 0)
    rows = {k: [] for k in KINDS}
    prev_end = 0
    emb = None
    for s in range(T):
        st = t[s]
        have = st[:, 3] > 0
        end = st[have, 3].max()
        rec = {
            "span": end - prev_end,
            "wait_med": np.median(st[have, 1]) - prev_end if s else 0,
            "wait_max": st[have, 1].max() - prev_end if s else 0,
            "comp_min": (st[have, 3] - st[have, 2]).min(),
            "comp_med": np.median(st[have, 3] - st[have, 2]),
            "comp_max": (st[have, 3] - st[have, 2]).max(),
            "ctas": int(have.sum()) * 1000,
            "tail": end - np.median(st[have, 3]),
        }
        if s == 0:
            emb = rec
        else:
            rows[KINDS[(s - 1) % 5]].append(rec)
        prev_end = end
    total = t[:, :, 3].max()
    out = {"step_us": step_us, "traced_chain_us": float(total) / 1e3, "embed": {k: float(v) / 1e3 for k, v in emb.items()},
           "kinds": {}}
    print(f"step (chain + lm_head): {step_us:.1f} us; traced chain {total / 1e3:.1f} us; {T} steps, {ctas} CTAs")
    print(f"{'kind':8s} " + " ".join(f"{k:>9s}" for k in rows[KINDS[0]][0]) + "   (us, medians over blocks; sum of spans)")
    for k in KINDS:
        med = {f: float(np.median([r[f] for r in rows[k]])) / 1e3 for f in rows[k][0]}
        out["kinds"][k] = med
        tot = sum(r["span"] for r in rows[k]) / 1e3
        out["kinds"][k]["span_sum"] = tot
        print(f"{k:8s} " + " ".join(f"{v:9.2f}" for v in med.values()) + f"   {tot:8.1f}")
    print("embed span %.2f us" % (emb["span"] / 1e3))
    if a.json:
        with open(a.json, "w") as f:
            json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
