"""Times whole-model Llama-3-8B-shaped greedy decode (fasq_llama_*: the
persistent chain with embedding, RMSNorm, RoPE + KV cache + attention, SwiGLU,
residuals, then the fp16 lm_head + argmax) with CUDA events on a CUDA graph of
one decode step.  KV positions cycle over [128, 256) (prompt 128 / gen 128,
P:438).  Prints ms/token, tok/s and the per-token algorithmic bytes.
usage: python tools/llama_time.py [d] [C] [B] [n_layers]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2605_04084_b200 as F
import synth

d = int(sys.argv[1]) if len(sys.argv) > 1 else 2
C = int(sys.argv[2]) if len(sys.argv) > 2 else 256
B = int(sys.argv[3]) if len(sys.argv) > 3 else 1
nl = int(sys.argv[4]) if len(sys.argv) > 4 else 32
hid, H, KV, hd, ffn, vocab = 4096, 32, 8, 128, 14336, 128256
shapes = {"q": (H * hd, hid), "k": (KV * hd, hid), "v": (KV * hd, hid), "o": (hid, H * hd),
          "gate": (ffn, hid), "up": (ffn, hid), "down": (hid, ffn)}
g = torch.Generator(device="cuda")
g.manual_seed(0)
layers, nbytes = [], 0
for l in range(nl):
    L = {}
    for i, (n, (fo, fi)) in enumerate(shapes.items()):
        cb, idx = synth.torch_random_layer(fo, fi, d, C, seed=l * 7 + i)
        L[n] = F.import_layer(cb, idx, fi)
        nbytes += fo * fi // d + (fi // d) * C * d * 2
    L["attn_norm"] = (1 + 0.1 * torch.randn(hid, generator=g, device="cuda")).half()
    L["mlp_norm"] = (1 + 0.1 * torch.randn(hid, generator=g, device="cuda")).half()
    layers.append(L)
fn = (1 + 0.1 * torch.randn(hid, generator=g, device="cuda")).half()
emb = torch.randn((vocab, hid), generator=g, device="cuda").half()
lm = (torch.randn((vocab, hid), generator=g, device="cuda") / hid ** 0.5).half()
nbytes += vocab * hid * 2
max_T = 256
model = F.Llama(layers, fn, emb, lm, H, KV, hd, vocab, max_T=max_T, pos_wrap=128, B=B)
for l in range(nl):
    K, V = model.kv_cache(l)
    K.normal_(generator=g)
    V.normal_(generator=g)
model.reset([128000 + b for b in range(B)], 128)
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    model.step(stream=s)
s.synchronize()
gr = torch.cuda.CUDAGraph()
with torch.cuda.graph(gr, stream=s):
    model.step(stream=s)
for _ in range(int(os.environ.get("WARM", "10"))):
    gr.replay()
torch.cuda.synchronize()
n = int(os.environ.get("NRUN", "128"))
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(n):
    gr.replay()
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / n
print("llama d=%d C=%d B=%d layers=%d: %.4f ms/token-step  %.1f tok/s  %.3f GB/token  %.3f TB/s algorithmic" % (
    d, C, B, nl, ms, B * 1e3 / ms, nbytes / 1e9, nbytes / ms / 1e9))
print("tokens", model.tokens().cpu().tolist())
