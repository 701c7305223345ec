"""FASQ B200 benchmark (driver contract: one JSON line on rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl fasq|reference]

Workload (BASELINE.json configs[4] / north_star "whole-model Llama-3-8B-shaped
decode"; metric "Llama-3-8B PQ decode tok/s"): greedy decode of a random-init
Llama-3-8B-shaped model whose 224 linear layers (32 blocks x q, k, v, o, gate,
up, down) are FASQ layers at the paper's effective 4-bit setting (d=2, C=256,
uint8 indices, fp16 codebooks), batch 1, with the fp16 embedding, RMSNorms,
RoPE + KV-cache attention, SwiGLU, residuals, fp16 lm_head and argmax -- the
paper's E2E setting (prompt 128, 128 generated tokens; the KV cache of
the 128 prompt positions is seeded, decode cycles over positions 128..255).
One step = one token: 5.2 GB of weights, far larger than the 126 MB L2.

At N > 1 GPUs the model is Megatron-sharded (q/k/v, gate/up: heads / ffn rows;
o, down: K slices; lm_head: vocab rows); the all-reduces / gathers are fused
into the chain kernel's counted stores over NVLink peer memory (no NCCL on the
data path), the argmax is reduced across ranks by red.max.

value  = decode tokens/s (1 token per step at B = 1), device time via CUDA
         events around K graph replays, max over ranks.
e2e    = the same through the public C-ABI calls with HOST buffers (token
         H2D + step + chosen-token D2H per step), wall clock.
roofline: dominant kernel = k_chain (the persistent whole-model chain, one
         launch per token), timed live with CUDA events around eager launches
         on the launch stream; algorithmic bytes = PQ indices + codebooks +
         fp16 activations of the 224 layers + embedding row + the KV rows
         attention reads; traffic = ncu dram bytes of one launch from the
         committed capture (profiles/r02/ncu_traffic.json) or null.
cpu_baseline: the C oracle (fp64 reconstruct-then-multiply) timed on a
         bounded row sample of each layer shape on the host cores.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

METRIC = "Llama-3-8B PQ decode tok/s + GEMV HBM GB/s vs 8 TB/s; prefill GEMM TFLOP/s"
D, C = 2, 256


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled (every 50 ms) during the
    timed region (B200_PROFILING.md clocks line)."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.samples = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), "--query-gpu=" + self.Q,
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            time.sleep(0.3)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc is None:
            return
        time.sleep(0.1)
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except Exception:
            self.proc.kill()
            out = ""
        for line in (out or "").splitlines():
            v = [x.strip() for x in line.split(",")]
            if len(v) >= 7:
                self.samples.append(v)

    def summary(self):
        def num(x):
            try:
                return float(x)
            except ValueError:
                return None
        sm = [num(s[0]) for s in self.samples if num(s[0]) is not None]
        mx = [num(s[1]) for s in self.samples if num(s[1]) is not None]
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if s[3 + i].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(sm)}


# ----------------------------------------------------------------------------
# whole model (the headline): Llama-3-8B-shaped greedy decode, fasq_llama_*
# ----------------------------------------------------------------------------
LLAMA = dict(n_layers=32, hidden=4096, n_heads=32, n_kv=8, head_dim=128, ffn=14336, vocab=128256)
PROMPT, MAX_T = 128, 256   # the paper's E2E protocol: prompt 128, 128 generated tokens


def build_llama(rank: int, world: int, d: int = D, c: int = C, B: int = 1, seed: int = 0, n_layers=None):
    """Random-init Llama-3-8B-shaped model whose 224 linear layers are FASQ
    layers (uniform random uint8 indices, N(0, 1/F_in) fp16 codebooks -- the
    synth recipe), fp16 embedding / lm_head / norm weights, and this rank's
    Megatron shards (q/k/v and gate/up: heads / ffn rows; o and down: K
    slices; lm_head: vocab rows).  Every rank draws the same full layers from
    the same seeds and keeps its shard, so the model does not depend on the
    world size.  The KV cache of the first PROMPT positions is seeded N(0, 1)
    (the state after a 128-token prompt); decoding cycles over positions
    [PROMPT, MAX_T) (pos_wrap).  Returns (model, bytes dict)."""
    import torch

    import paper_2605_04084_b200 as F
    import synth
    m = LLAMA
    nl = m["n_layers"] if n_layers is None else n_layers
    hid, H, KV, hd, ffn, V = m["hidden"], m["n_heads"], m["n_kv"], m["head_dim"], m["ffn"], m["vocab"]
    Hl, KVl, Fl, Vl = H // world, KV // world, ffn // world, V // world
    shapes = {"q": (H * hd, hid), "k": (KV * hd, hid), "v": (KV * hd, hid), "o": (hid, H * hd),
              "gate": (ffn, hid), "up": (ffn, hid), "down": (hid, ffn)}
    rows = {"q": Hl * hd, "k": KVl * hd, "v": KVl * hd, "gate": Fl, "up": Fl}
    kcols = {"o": Hl * hd, "down": Fl}
    g = torch.Generator(device="cuda")
    g.manual_seed(seed * 7919 + 17)
    layers, pq_bytes = [], 0
    for l in range(nl):
        L = {}
        for i, (n, (fo, fi)) in enumerate(shapes.items()):
            cb, idx = synth.torch_random_layer(fo, fi, d, c, seed=seed * 1000 + l * 7 + i)
            if world > 1 and n in rows:
                r = rows[n]
                idx = idx[:, rank * r:(rank + 1) * r].contiguous()
                fi_l = fi
            elif world > 1:
                s0, s1 = rank * kcols[n] // d, (rank + 1) * kcols[n] // d
                cb, idx = cb[s0:s1].contiguous(), idx[s0:s1].contiguous()
                fi_l = kcols[n]
            else:
                fi_l = fi
            L[n] = F.import_layer(cb, idx, fi_l)
            pq_bytes += idx.numel() + cb.numel() * 2
            del cb, idx
        L["attn_norm"] = (1 + 0.1 * torch.randn(hid, generator=g, device="cuda")).half()
        L["mlp_norm"] = (1 + 0.1 * torch.randn(hid, generator=g, device="cuda")).half()
        layers.append(L)
    fn = (1 + 0.1 * torch.randn(hid, generator=g, device="cuda")).half()
    emb = torch.randn((V, hid), generator=g, device="cuda").half()
    lm = (torch.randn((V, hid), generator=g, device="cuda") / hid ** 0.5).half()
    lm = lm[rank * Vl:(rank + 1) * Vl].contiguous()
    torch.cuda.synchronize()
    model = F.Llama(layers, fn, emb, lm, H, KV, hd, V, max_T=MAX_T, pos_wrap=PROMPT, B=B, world=world, rank=rank)
    gk = torch.Generator(device="cuda")
    gk.manual_seed(seed * 31 + 5)
    for l in range(nl):
        K_, V_ = model.kv_cache(l)
        K_.normal_(generator=gk)
        V_.normal_(generator=gk)
    torch.cuda.synchronize()
    model._bench_keep = (layers, fn, emb, lm)
    # algorithmic bytes per step (this rank): PQ weights (indices + codebooks),
    # fp16 activations in/out of every PQ layer, the embedding row, the KV rows
    # attention reads (T = positions incl. the new one, averaged over the
    # decode cycle [PROMPT, MAX_T)), and the lm_head (separate kernel)
    act = 0
    for n, (fo, fi) in shapes.items():
        fo_l = rows.get(n, fo) if world > 1 else fo
        fi_l = kcols.get(n, fi) if world > 1 else fi
        act += 2 * B * (fo_l + fi_l)
    t_avg = (PROMPT + 1 + MAX_T) / 2.0
    kv = 2 * KVl * t_avg * hd * 2 * B
    chain = pq_bytes + nl * (act + kv) + 2 * hid * B
    lm_b = Vl * hid * 2 + 2 * hid * B
    return model, {"pq": pq_bytes, "chain": chain, "lm_head": lm_b, "step": chain + lm_b, "kv_t_avg": t_avg}


def llama_timed(model, steps, warmup, rank, world):
    """ms per decode step (device time: CUDA graph of one step, K replays
    between CUDA events, max over ranks)."""
    model.reset([128000 + b for b in range(model.B)], PROMPT)
    g = capture(lambda: model.step(), world)
    return timed(g, steps, warmup, rank, world), g


def llama_sustained(g, seconds=2.5):
    """Sustained decode (burst vs sustained): the one-step CUDA graph
    replayed back to back for >= `seconds` (long enough for the 1 kW board power
    cap to act), CUDA events around chunks of 200 replays; tok/s over the whole
    window and over its last half, with the clocks sampled during it."""
    import torch
    chunks = []
    t_end = time.time() + seconds
    with ClockSampler(torch.cuda.current_device()) as clk:
        while time.time() < t_end:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(200):
                g.replay()
            e1.record()
            e1.synchronize()
            chunks.append(e0.elapsed_time(e1))
    tot_ms = sum(chunks)
    half = chunks[len(chunks) // 2:]
    return {"seconds": round(tot_ms / 1e3, 2), "tok_s": round(200 * len(chunks) * 1e3 / tot_ms, 1),
            "tok_s_last_half": round(200 * len(half) * 1e3 / sum(half), 1),
            "ms_per_token_last_half": round(sum(half) / (200 * len(half)), 4), "clocks": clk.summary()}


def llama_prefill_side(model, M=PROMPT, reps=5):
    """The paper's E2E protocol on the bench model: a 128-token prompt
    through fasq_llama_prefill (whole model: RMSNorm, PQ q/k/v/o/gate/up/down on
    the tcgen05 decode kernel at M = 128, RoPE, KV-cache write, causal attention,
    SwiGLU, residuals, lm_head + argmax of the last position), then 128 greedy
    decode steps (one CUDA graph per step); CUDA events."""
    import torch
    toks = torch.arange(1000, 1000 + M, dtype=torch.int32, device="cuda")
    model.prefill(toks, 0)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        model.prefill(toks, 0)
    e1.record()
    torch.cuda.synchronize()
    pf_ms = e0.elapsed_time(e1) / reps
    g = capture(lambda: model.step(), 1)
    model.prefill(toks, 0)
    e2, e3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e2.record()
    model.prefill(toks, 0)
    for _ in range(MAX_T - PROMPT):
        g.replay()
    e3.record()
    torch.cuda.synchronize()
    tot = e2.elapsed_time(e3)
    return {"prompt": M, "prefill_ms": round(pf_ms, 3), "prefill_tok_s": round(M * 1e3 / pf_ms, 1),
            "e2e_prompt128_gen128_ms": round(tot, 2),
            "e2e_gen_tok_s": round((MAX_T - PROMPT) * 1e3 / (tot - pf_ms), 1)}


def llama_kernel_ms(model, reps, world):
    """Per-kernel device time of the two launches of a step (chain, lm_head):
    eager steps with CUDA events before / between (fasq_llama_step_ex
    parts 1 and 2) / after, on the launch stream, averaged."""
    import torch
    import torch.distributed as dist
    if world > 1:
        torch.cuda.synchronize()
        dist.barrier()
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(reps)]
    for e in evs:
        e[0].record()
        model.step_part(1)
        e[1].record()
        model.step_part(2)
        e[2].record()
    torch.cuda.synchronize()
    ch = sum(e[0].elapsed_time(e[1]) for e in evs) / reps
    lm = sum(e[1].elapsed_time(e[2]) for e in evs) / reps
    return ch, lm


def llama_split(model, ms_step, n_layers=32):
    """Per-component time split of one decode token: one traced chain run
    (%globaltimer stamps per step and CTA, fasq_chain_trace); a step's span is
    last output of the previous step -> last output of this step.  Sums over
    the 32 blocks per step kind; lm_head = step time - traced chain span."""
    import numpy as np
    import torch
    T = 1 + 5 * n_layers
    buf = torch.zeros((T, model.chain.ctas, 4), dtype=torch.int64, device="cuda")
    model.chain.trace(buf)
    model.step()
    torch.cuda.synchronize()
    model.chain.trace(None)
    t = buf.cpu().numpy().astype(np.int64)
    t0 = t[:, :, 0][t[:, :, 0] > 0].min()
    ends = np.array([t[s][t[s, :, 3] > 0, 3].max() for s in range(T)]) - t0
    spans = np.diff(np.concatenate([[0], ends])) / 1e3
    kinds = ["qkv (RMSNorm + PQ q/k/v)", "attention (RoPE + KV + softmax)", "o_proj (PQ, attention merge)",
             "gate/up (RMSNorm + PQ)", "down (SwiGLU + PQ + residual)"]
    out = {"embedding": round(float(spans[0]), 2)}
    for k, name in enumerate(kinds):
        out[name] = round(float(spans[1 + k::5].sum()), 1)
    out["lm_head + argmax (+ launch gap)"] = round(ms_step * 1e3 - float(ends[-1]) / 1e3, 1)
    out["unit"] = "us per token"
    return out


def llama_e2e(model, steps, warmup, rank, world):
    """End to end through the public C-ABI call with HOST buffers: every step
    (fasq_llama_step_io) copies the B tokens to decode to the device (through
    the model's pinned staging), runs the chain + lm_head and copies the chosen
    tokens back; wall clock around K synchronous steps, max over ranks."""
    import torch
    import torch.distributed as dist
    toks = [128000 + b for b in range(model.B)]
    model.reset(toks, PROMPT)
    for _ in range(warmup):
        toks = model.step_io(toks, -1)
    if world > 1:
        torch.cuda.synchronize()
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(steps):
        toks = model.step_io(toks, -1)   # H2D of the tokens, chain + lm_head, D2H of the choice: one sync
    dt = (time.perf_counter() - t0) * 1e3 / steps
    if world > 1:
        t = torch.tensor([dt], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dt = float(t.item())
    return dt


# ----------------------------------------------------------------------------
# PQ linear stack only (the round-1 headline; side measurement now)
# ----------------------------------------------------------------------------
def build_model(rank: int, world: int, seed: int = 0):
    """Row-sharded PQ layers of every block (random-init, paper shapes)."""
    import torch

    import paper_2605_04084_b200 as F
    import synth

    blocks = []
    for b in range(synth.LLAMA3_8B_BLOCKS):
        layers = {}
        for li, (name, fo, fi) in enumerate(synth.LLAMA3_8B_LAYERS):
            rows = fo // world
            # draw the full layer deterministically, keep this rank's rows
            cb, idx = synth.torch_random_layer(fo, fi, D, C, seed=seed * 1000 + b * 7 + li)
            if world > 1:
                idx = idx[:, rank * rows:(rank + 1) * rows].contiguous()
            layers[name] = F.import_layer(cb, idx, fi)
            del cb, idx
        blocks.append(layers)
    torch.cuda.synchronize()
    return blocks


def layer_bytes(world: int):
    """Algorithmic bytes a decode step must move per rank:
    uint8 indices N_ss*F_out + fp16 codebooks N_ss*C*d*2 + x (2*F_in) +
    y (2*F_out), summed over the 224 layers."""
    import synth
    tot = 0
    for (_, fo, fi) in synth.LLAMA3_8B_LAYERS:
        n_ss = fi // D
        tot += n_ss * (fo // world) + n_ss * C * D * 2 + 2 * fi + 2 * (fo // world)
    return tot * synth.LLAMA3_8B_BLOCKS


class DecodeStep:
    """One decode step = the 224 chained PQ GEMVs of the 32 blocks, launched as
    4 grouped launches per block: {q,k,v} (same input), o, {gate,up} (same
    input), down -- every layer packed separately.

    N = 1 (default): the 128 grouped launches run as ONE persistent kernel
    (fasq_chain_*); FASQ_BENCH_CHAIN=0 uses one launch per step instead, where
    every launch writes FASQ_ACC_I64 accumulators (exact int64 fixed
    point, deterministic, no split-K merge phase); the consumer rounds them to
    fp16 x on load; each launch zeroes the accumulators of the launch two
    steps back (no longer read) and warms L2 with the next launch's first
    stages.  N > 1: rows are sharded; by default the token still runs as ONE
    chain kernel per GPU (fasq_chain_create_tp) whose GEMV epilogues red.add
    every rank's rows into every rank's arena over NVLink peer memory (the
    row-shard all-gather fused into the GEMV; arena IPC handles exchanged once
    through torch.distributed).  FASQ_BENCH_TP=nccl selects the baseline:
    per-launch GEMVs with each chain output (q, o, gate, down) materialised as
    fp16 and all-gathered with NCCL."""

    NAMES = [("q_proj", "k_proj", "v_proj"), ("o_proj",), ("gate_proj", "up_proj"), ("down_proj",)]
    FEEDS = {1: "q_proj", 2: "o_proj", 3: "gate_proj"}   # launch i reads this output of launch i-1

    def __init__(self, blocks, rank, world, pg=None):
        import torch
        import synth
        self.blocks, self.rank, self.world, self.pg = blocks, rank, world, pg
        dev = torch.device("cuda", torch.cuda.current_device())
        f16 = torch.float16
        self.h = torch.zeros((1, 4096), dtype=f16, device=dev)
        self.shapes = {n: (fo, fi) for (n, fo, fi) in synth.LLAMA3_8B_LAYERS}
        self.seq = [(b, i) for b in range(len(blocks)) for i in range(4)]
        self.acc_mode = world == 1
        self.chain = None
        use_chain = os.environ.get("FASQ_BENCH_CHAIN", "1") == "1"
        if world > 1:
            use_chain = use_chain and os.environ.get("FASQ_BENCH_TP", "fused") != "nccl"
        self.tp_mode = "single-gpu" if world == 1 else "fused-p2p"
        if use_chain:
            # the whole token as ONE persistent kernel per GPU (fasq_chain_*)
            import paper_2605_04084_b200 as F
            steps = []
            for (b, i) in self.seq:
                pos = len(steps)
                src = None if pos == 0 else (pos - 1, 0)
                steps.append(([blocks[b][k] for k in self.NAMES[i]], src))
            self.chain = F.Chain(steps, B=1, world=world, rank=rank)
            if world > 1:
                import torch.distributed as dist
                handles = [None] * world
                dist.all_gather_object(handles, self.chain.ipc_handle(), group=pg)
                self.chain.set_peers(handles)
            self.out_f16 = torch.empty((1, 4096), dtype=f16, device=dev)
            self.acc_mode = True
        elif self.acc_mode:
            # one int64 accumulator slab per launch position of the token
            self.acc = []
            for (b, i) in self.seq:
                tot = sum(self.shapes[n][0] for n in self.NAMES[i])
                slab = torch.zeros((tot,), dtype=torch.int64, device=dev)
                outs, off = {}, 0
                for n in self.NAMES[i]:
                    fo = self.shapes[n][0]
                    outs[n] = slab[off:off + fo].view(1, fo)
                    off += fo
                self.acc.append((slab, outs))
            self.out_f16 = torch.empty((1, 4096), dtype=f16, device=dev)
        else:
            self.tp_mode = "nccl-allgather"
            self.bufs = {}
            for (name, fo, fi) in synth.LLAMA3_8B_LAYERS:
                self.bufs[name] = torch.empty((1, fo // world), dtype=f16, device=dev)
                self.bufs[name + "_full"] = torch.empty((1, fo), dtype=f16, device=dev)
        self.launches = 0

    def _gather(self, name):
        """Row-shard all-gather over NCCL (paper_2605_04084_b200.shard)."""
        from paper_2605_04084_b200 import shard
        return shard.gather_rows(self.bufs[name], self.bufs[name + "_full"], group=self.pg)

    def run(self, flags=0, prefetch=None):
        import paper_2605_04084_b200 as F
        if prefetch is None:
            prefetch = os.environ.get("FASQ_BENCH_PREFETCH", "1") == "1"
        n = 0
        T = len(self.seq)
        if self.chain is not None:
            self.chain.run(self.h)
            n += F.last_launch_count()
            self.chain.output(T - 1, 0, out=self.out_f16)
            n += 1
            self.out = self.out_f16
            self.launches = n
            return self.out
        for pos, (b, i) in enumerate(self.seq):
            layers = [self.blocks[b][k] for k in self.NAMES[i]]
            nxt = None
            if prefetch and pos + 1 < T:
                b2, i2 = self.seq[pos + 1]
                nxt = [self.blocks[b2][k] for k in self.NAMES[i2]]
            if self.acc_mode:
                if pos == 0:
                    x = self.h
                else:
                    x = self.acc[pos - 1][1][self.FEEDS[i] if i else "down_proj"]
                F.gemv_grouped(layers, x, outs=[self.acc[pos][1][k] for k in self.NAMES[i]], flags=flags,
                               next_layers=nxt, zero=self.acc[(pos - 2) % T][0])
                n += F.last_launch_count()
            else:
                if pos == 0:
                    x = self.h
                elif i == 0:
                    x = self._gather("down_proj")
                else:
                    x = self._gather(self.FEEDS[i])
                F.gemv_grouped(layers, x, outs=[self.bufs[k] for k in self.NAMES[i]], flags=flags,
                               next_layers=nxt)
                n += F.last_launch_count()
        if self.acc_mode:
            F.acc_convert(self.acc[T - 1][1]["down_proj"], out=self.out_f16)
            n += F.last_launch_count()
            self.out = self.out_f16
        else:
            self.out = self._gather("down_proj")
        self.launches = n
        return self.out


def capture(fn, world=1):
    import torch
    if world > 1:   # TP chain kernels spin-wait on their peers: start together
        import torch.distributed as dist
        torch.cuda.synchronize()
        dist.barrier()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn()           # warm allocator / plans outside capture
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        fn()
    torch.cuda.synchronize()
    return g


def timed(graph, steps, warmup, rank, world, pg=None):
    import torch
    import torch.distributed as dist
    if world > 1:
        torch.cuda.synchronize()
        dist.barrier()
    for _ in range(warmup):
        graph.replay()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        graph.replay()
    e1.record()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms = e0.elapsed_time(e1)
    if world > 1:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    return ms / steps


# ----------------------------------------------------------------------------
# CPU oracle baseline (bounded sample)
# ----------------------------------------------------------------------------
class OracleSampler:
    """CPU oracle baseline on a bounded sample: the fp64 reconstruct-then-
    multiply GEMV (oracle/) on the first `rows` rows of one seeded layer of
    each Llama-3-8B shape, extrapolated per row to the 224-layer decode step."""

    def __init__(self):
        import oracle
        import synth
        self.oracle = oracle
        self.shapes = sorted({(fo, fi) for (_, fo, fi) in synth.LLAMA3_8B_LAYERS})
        self.layers = {}
        for (fo, fi) in self.shapes:
            cb, idx = synth.random_layer(min(fo, 4096), fi, D, C, seed=7)   # rows beyond the sample unused
            self.layers[(fo, fi)] = (cb, idx, synth.activation(1, fi, seed=1))
        self.threads = oracle.num_threads()

    def step(self, rows: int):
        """One sampled step; returns (estimated full-step seconds, seconds spent)."""
        import synth
        t_all = time.perf_counter()
        per_row = {}
        for key, (cb, idx, x) in self.layers.items():
            r = min(rows, idx.shape[1])
            t0 = time.perf_counter()
            self.oracle.gemv(cb, idx, x, rows=(0, r))
            per_row[key] = (time.perf_counter() - t0) / r
        est = synth.LLAMA3_8B_BLOCKS * sum(per_row[(fo, fi)] * fo for (_, fo, fi) in synth.LLAMA3_8B_LAYERS)
        return est, time.perf_counter() - t_all

    def calibrate(self, budget_s: float):
        """Rows per step so one sampled step costs about budget_s."""
        _, dt = self.step(64)
        return max(16, min(4096, int(64 * budget_s / max(dt, 1e-3))))

    def describe(self, rows):
        return ("oracle fp64 GEMV (reconstruct-then-multiply) on the first %d rows of one seeded layer "
                "of each Llama-3-8B shape (d=2, C=256, B=1), time per row extrapolated to the 224 "
                "layers of one decode step" % rows)


def oracle_decode_rate(budget_s: float = 15.0):
    s = OracleSampler()
    rows = s.calibrate(budget_s)
    est, spent = s.step(rows)
    return 1.0 / est, s.threads, s.describe(rows), spent


# ----------------------------------------------------------------------------
# side measurements (not part of the timed region)
# ----------------------------------------------------------------------------
def prefill_tflops(M=2048, iters=10):
    """configs[3]: prefill PQ GEMM on the Llama-3-8B shapes, EXPAND (tcgen05)
    vs LUT; EXPAND's fraction is against the measured dense bf16 peak (fp16
    tensor-core rate = bf16 rate, MEASURED_PEAKS.json)."""
    import torch
    pk, _ = _peaks()
    dense_peak = float(pk.get("bf16_tflops", 1692.0))

    import paper_2605_04084_b200 as F
    import synth
    out = {}
    for (fo, fi) in [(4096, 4096), (14336, 4096), (4096, 14336)]:
        cb, idx = synth.torch_random_layer(fo, fi, D, C, seed=3)
        L = F.import_layer(cb, idx, fi)
        X = synth.torch_activation(M, fi)
        Y = torch.empty((M, fo), dtype=torch.float16, device="cuda")
        res = {}
        for name, algo in (("expand_tc", F.GEMM_EXPAND_TC), ("lut", F.GEMM_LUT)):
            try:
                n_it = iters if algo == F.GEMM_EXPAND_TC else 2
                # device time: n_it launches replayed from a CUDA graph (the
                # ~40 us of Python/ctypes/tensor-map host work per call would
                # otherwise starve the GPU at these sizes)
                gs = torch.cuda.Stream()
                gs.wait_stream(torch.cuda.current_stream())
                with torch.cuda.stream(gs):
                    F.gemm(L, X, out=Y, algo=algo)   # sizes the capture stream's workspace outside capture
                torch.cuda.synchronize()
                gr = torch.cuda.CUDAGraph()
                with torch.cuda.stream(gs):
                    with torch.cuda.graph(gr, stream=gs):
                        for _ in range(n_it):
                            F.gemm(L, X, out=Y, algo=algo)
                torch.cuda.synchronize()
                gr.replay()
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                gr.replay()
                e1.record()
                torch.cuda.synchronize()
                ms = e0.elapsed_time(e1) / n_it
                tf = 2.0 * M * fo * fi / ms / 1e9
                res[name] = {"ms": round(ms, 4), "tflops": round(tf, 2)}
                if algo == F.GEMM_EXPAND_TC:
                    res[name]["frac_of_dense_peak"] = round(tf / dense_peak, 3)
            except Exception as e:  # report, never hide
                res[name] = {"error": str(e)[:200]}
        out["%dx%d" % (fo, fi)] = res
        L.free()
    return out


KINDS = (("qkv", ("q_proj", "k_proj", "v_proj")), ("o", ("o_proj",)), ("gate_up", ("gate_proj", "up_proj")),
         ("down", ("down_proj",)))


def prefill_model(dense_peak, Ms=(128, 512, 2048), reps=3):
    """configs[4] at N = 1: the prefill pass of the whole PQ linear stack --
    M tokens through the 224 Llama-3-8B-shaped PQ layers (AUTO at M = 128 --
    the paper's prompt length, P:438 -- EXPAND on tcgen05 above), fp16
    activations chained block to block like the decode chain; q/k/v and
    gate/up read the same input and run as fasq_gemm_grouped (one EXPAND launch
    each); attention / norms excluded.  Replayed from a CUDA graph; tok/s = M /
    pass time."""
    import torch

    import paper_2605_04084_b200 as F
    import synth

    nb = synth.LLAMA3_8B_BLOCKS
    shapes = {n: (fo, fi) for (n, fo, fi) in synth.LLAMA3_8B_LAYERS}
    blocks = []
    for b in range(nb):
        Ls = {}
        for li, (name, fo, fi) in enumerate(synth.LLAMA3_8B_LAYERS):
            cb, idx = synth.torch_random_layer(fo, fi, D, C, seed=11000 + b * 7 + li)
            Ls[name] = F.import_layer(cb, idx, fi)
            del cb, idx
        blocks.append(Ls)
    flops = 2.0 * nb * sum(fo * fi for (fo, fi) in shapes.values())
    out = {}
    for M in Ms:
        algo = F.GEMM_AUTO if M <= 128 else F.GEMM_EXPAND_TC
        x0 = synth.torch_activation(M, 4096)
        bufs = {n: torch.empty((M, fo), dtype=torch.float16, device="cuda") for n, (fo, fi) in shapes.items()}

        def one_pass():
            h = x0
            for Ls in blocks:
                qkv = ("q_proj", "k_proj", "v_proj")
                F.gemm_grouped([Ls[n] for n in qkv], h, outs=[bufs[n] for n in qkv], algo=algo)
                F.gemm(Ls["o_proj"], bufs["q_proj"], out=bufs["o_proj"], algo=algo)
                gu = ("gate_proj", "up_proj")
                F.gemm_grouped([Ls[n] for n in gu], bufs["o_proj"], outs=[bufs[n] for n in gu], algo=algo)
                F.gemm(Ls["down_proj"], bufs["gate_proj"], out=bufs["down_proj"], algo=algo)
                h = bufs["down_proj"]
        gs = torch.cuda.Stream()
        gs.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(gs):
            one_pass()                  # sizes the capture stream's split-K workspace outside capture
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(gs):
            with torch.cuda.graph(g, stream=gs):
                one_pass()
        torch.cuda.synchronize()
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            g.replay()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        tf = flops * M / (ms * 1e-3) / 1e12
        out["M%d" % M] = {"ms_per_pass": round(ms, 3), "tok_s": round(M * 1e3 / ms, 1), "tflops": round(tf, 1),
                          "frac_of_dense_peak": round(tf / dense_peak, 3)}
        del g, bufs
    for Ls in blocks:
        for L in Ls.values():
            L.free()
    torch.cuda.synchronize()
    return out


def prefill_token_sharded(world, rank, dense_peak, M=2048):
    """NEXT-1 (iii) token-sharded prefill: every rank holds the whole PQ model
    (4.1 GB of weights: replicas fit 180 GB HBM easily) and runs M / world of
    the M prompt tokens through the 224 PQ GEMMs (EXPAND) -- no collective on
    the data path.  tok/s = M / (max over ranks of the pass time)."""
    import torch
    import torch.distributed as dist
    m_local = M // world
    r = prefill_model(dense_peak, Ms=(m_local,))["M%d" % m_local]
    ms = r["ms_per_pass"]
    if world > 1:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    return {"global_tokens": M, "tokens_per_rank": m_local, "ranks": world, "ms_per_pass": round(ms, 3),
            "tok_s": round(M * 1e3 / ms, 1), "collective": "none (weights replicated per rank)"}


def decode_batch(peak, batches=(2, 4, 8), runs=20):
    """decode batch B in {2, 4, 8} at (2,256) through the
    chain kernel (one step = B tokens through the 224 layers).  Bytes per step
    = indices + codebooks + B x (x + y accumulator words)."""
    import torch

    import paper_2605_04084_b200 as F
    import synth

    nb = synth.LLAMA3_8B_BLOCKS
    blocks = []
    for b in range(nb):
        Ls = {}
        for li, (name, fo, fi) in enumerate(synth.LLAMA3_8B_LAYERS):
            cb, idx = synth.torch_random_layer(fo, fi, D, C, seed=9000 + b * 7 + li)
            Ls[name] = F.import_layer(cb, idx, fi)
            del cb, idx
        blocks.append(Ls)
    out = {}
    for B in batches:
        steps = []
        for b in range(nb):
            for (_, names) in KINDS:
                steps.append(([blocks[b][n] for n in names], None if not steps else (len(steps) - 1, 0)))
        ch = F.Chain(steps, B=B)
        x = synth.torch_activation(B, 4096)
        for _ in range(3):
            ch.run(x)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(runs):
            ch.run(x)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / runs
        bts = nb * sum(fo * fi // D + (fi // D) * C * D * 2 + B * (2 * fi + 8 * fo)
                       for (_, fo, fi) in synth.LLAMA3_8B_LAYERS)
        out["B%d" % B] = {"ms_per_step": round(ms, 4), "tok_s": round(B * 1e3 / ms, 1),
                          "GBps": round(bts / (ms * 1e-3) / 1e9, 1), "frac": round(bts / (ms * 1e-3) / 1e9 / peak, 3)}
        del ch
    for Ls in blocks:
        for L in Ls.values():
            L.free()
    torch.cuda.synchronize()
    return out


def decode_sweep(peak, settings=((2, 256), (2, 128), (4, 256), (1, 256), (2, 64), (8, 256)), runs=30):
    """configs[1]/[2]: the whole-model decode token through the chain kernel at
    each (d, C) of the sweep (effective 4-bit (2,256), 3-bit (2,128), ...),
    plus per-LAYER-SHAPE GEMV throughput measured inside the token: the
    %globaltimer trace of one run gives every step's span (last output of the
    previous step -> last output of this step, median over the 32 blocks), and
    that step's algorithmic bytes / span is its GB/s.  Bytes per layer =
    indices F_out*F_in/d + codebooks (F_in/d)*C*d*2 + x + y (counted
    accumulator words, 8 B).  Model size fraction = (PQ bytes of the 224
    layers + fp16 embedding, lm_head and norms) / fp16 model bytes."""
    import numpy as np
    import torch

    import paper_2605_04084_b200 as F
    import synth

    shapes = {n: (fo, fi) for (n, fo, fi) in synth.LLAMA3_8B_LAYERS}
    nb = synth.LLAMA3_8B_BLOCKS
    dense_other = 2 * (2 * 128256 * 4096 + (2 * nb + 1) * 4096)   # embed + lm_head + norms, fp16 bytes
    dense_lin = 2 * nb * sum(fo * fi for (fo, fi) in shapes.values())
    out = {}
    for (d, c) in settings:
        blocks = []
        for b in range(nb):
            Ls = {}
            for li, (name, fo, fi) in enumerate(synth.LLAMA3_8B_LAYERS):
                cb, idx = synth.torch_random_layer(fo, fi, d, c, seed=7000 + b * 7 + li)
                Ls[name] = F.import_layer(cb, idx, fi)
                del cb, idx
            blocks.append(Ls)

        def lbytes(n):
            fo, fi = shapes[n]
            return fo * fi // d + (fi // d) * c * d * 2 + 2 * fi + 8 * fo
        steps = []
        for b in range(nb):
            for (_, names) in KINDS:
                steps.append(([blocks[b][n] for n in names], None if not steps else (len(steps) - 1, 0)))
        ch = F.Chain(steps, B=1)
        x = synth.torch_activation(1, 4096)
        for _ in range(3):
            ch.run(x)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(runs):
            ch.run(x)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / runs
        tok_bytes = nb * sum(lbytes(n) for n in shapes)
        T = len(steps)
        buf = torch.zeros((T, ch.ctas, 4), dtype=torch.int64, device="cuda")
        ch.trace(buf)
        ch.run(x)
        torch.cuda.synchronize()
        ch.trace(None)
        t = buf.cpu().numpy().astype(np.int64)
        ends = t[:, :, 3].max(axis=1)
        spans = np.diff(np.concatenate([[t[0, :, 0][t[0, :, 0] > 0].min()], ends]))
        per = {}
        for k, (kind, names) in enumerate(KINDS):
            us = float(np.median(spans[k::len(KINDS)])) / 1e3
            bts = sum(lbytes(n) for n in names)
            gbs = bts / (us * 1e-6) / 1e9
            per[kind] = {"shapes": ["%dx%d" % shapes[n] for n in names], "us": round(us, 3),
                         "GBps": round(gbs, 1), "frac": round(gbs / peak, 3)}
        info = blocks[0]["q_proj"].info
        pq = nb * sum(blocks[0][n].info["index_bytes"] + blocks[0][n].info["codebook_bytes"] for n in shapes)
        out["d%d_C%d" % (d, c)] = {
            "ms_per_token": round(ms, 4), "tok_s": round(1e3 / ms, 1),
            "GBps": round(tok_bytes / (ms * 1e-3) / 1e9, 1), "frac": round(tok_bytes / (ms * 1e-3) / 1e9 / peak, 3),
            "bits_per_weight_4096x4096": round(info["bits_per_weight"], 4),
            "model_size_frac_of_fp16": round((pq + dense_other) / (dense_lin + dense_other), 4),
            "per_layer_shape": per}
        del ch
        for Ls in blocks:
            for L in Ls.values():
                L.free()
        del blocks
        torch.cuda.synchronize()
    return out


def packed_gemv_side(peak):
    """NEXT-2 (Eq. 4): per-launch decode GEMV (B = 1, CUDA graph of
    launches over > L2 of replicas) with byte indices vs ceil(log2 C)-bit
    packed indices on the Llama-3-8B shapes; bytes = Eq. 4 index bits +
    codebooks + x + y."""
    from tools.packed_time import run
    out = {}
    for tag, C, packed in (("d2_C256_u8", 256, False), ("d2_C128_u8", 128, False), ("d2_C128_p7", 128, True),
                           ("d2_C512_p9", 512, True), ("d2_C1024_p10", 1024, True)):
        per = {}
        for (o, i) in ((4096, 4096), (14336, 4096), (4096, 14336)):
            r = run(o, i, C, packed, iters=100)
            per["%dx%d" % (o, i)] = {"us": r["us"], "bytes": r["bytes"], "GBps": r["GBps"],
                                     "frac": round(r["GBps"] / peak, 3)}
        out[tag] = per
    return out


def dim0_gemv_side(peak):
    """NEXT-4: per-launch decode GEMV on the paper's dim = 0 layout (output-axis
    subspaces) next to Eq. 3's input-axis layout, d = 2, C = 256, B = 1 / 8."""
    from tools.dim0_time import run
    out = {}
    for B in (1, 8):
        for dim0 in (False, True):
            per = {}
            for (o, i) in ((4096, 4096), (14336, 4096), (4096, 14336), (1024, 4096)):
                r = run(o, i, dim0, B=B, iters=100)
                per["%dx%d" % (o, i)] = {"us": r["us"], "GBps": r["GBps"], "frac": round(r["GBps"] / peak, 3)}
            out["%s_B%d" % ("dim0" if dim0 else "dim1", B)] = per
    return out


def batch_gemv_side(peak):
    """NEXT-3 / G5: per-launch decode GEMV at B = 8 / 16 / 64 on the tcgen05 decode
    kernel (gemv_tc.cu; the default dispatch for B >= 5) next to the CUDA-core
    GEMV (B = 8) / prefill EXPAND (B > 8) it replaces, Llama-3-8B shapes."""
    from tools.gemv_tc_sweep import run
    out = {}
    for B in (8, 16, 64):
        per = {}
        for (o, i) in ((4096, 4096), (14336, 4096), (4096, 14336)):
            tc = run(o, i, B, True, iters=50)
            base = run(o, i, B, False, iters=50)
            per["%dx%d" % (o, i)] = {"tcgen05_us": tc["us"], "tcgen05_GBps": tc["GBps"],
                                     "tcgen05_frac": round(tc["GBps"] / peak, 3), "previous_path_us": base["us"]}
        out["B%d" % B] = per
    os.environ.pop("FASQ_GEMV_TC_MIN_B", None)
    return out


def pack_time():
    """GPU k-means pack (Alg. 1, 25 Lloyd rounds, d=2, C=256) of one seeded
    layer of each Llama-3-8B shape, and the whole-model estimate (x 32 blocks);
    the paper quotes ~10 minutes for all layers on one GPU."""
    import torch

    import paper_2605_04084_b200 as F
    import synth
    per, first = {}, {}
    block_s = 0.0
    for (name, fo, fi) in synth.LLAMA3_8B_LAYERS:
        key = "%dx%d" % (fo, fi)
        if key not in per:
            W = synth.torch_activation(fo, fi, seed=5, std=0.02)
            # the first pack of a shape grows the allocator pools / CUB temp
            # storage and is reported separately; the estimate uses the fastest
            # of three warm packs of the same layer (host wall clock: the pack
            # loop synchronises with the host, which adds run-to-run noise)
            for rep in range(4):
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                L = F.pack(W, d=D, C=C, group=1, seed=0, iters=25)
                torch.cuda.synchronize()
                dt = round(time.perf_counter() - t0, 4)
                if rep == 0:
                    first[key] = dt
                else:
                    per[key] = min(per.get(key, dt), dt)
                L.free()
            del W
        block_s += per[key]
    # NEXT-4 packing variants on one 4096 x 4096 layer (k-means++ init, reseeding)
    W = synth.torch_activation(4096, 4096, seed=5, std=0.02)
    var = {}
    for name, kw in (("kmeanspp", {"init": 1}), ("reseed", {"empty": 1}), ("kmeanspp+reseed", {"init": 1, "empty": 1})):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        L = F.pack(W, d=D, C=C, group=1, seed=0, iters=25, **kw)
        torch.cuda.synchronize()
        var[name] = round(time.perf_counter() - t0, 4)
        L.free()
    return {"d": D, "C": C, "iters": 25, "seconds_per_layer_shape": per, "first_pack_seconds": first,
            "whole_model_seconds_est": round(block_s * synth.LLAMA3_8B_BLOCKS, 2),
            "variants_4096x4096_seconds": var}


# ----------------------------------------------------------------------------
def run_reference(args, rank, world):
    """--impl reference: the CPU oracle on the host cores, each step a bounded
    sample of the same workload (whole run ~2 minutes for any K)."""
    if rank != 0:
        return
    sampler = OracleSampler()
    per_step = max(0.05, min(2.0, 120.0 / max(1, args.steps + args.warmup)))
    rows = sampler.calibrate(per_step)
    for _ in range(args.warmup):
        sampler.step(rows)
    ests = [sampler.step(rows)[0] for _ in range(args.steps)]
    v = 1.0 / statistics.median(ests)
    line = {"metric": METRIC, "value": v, "unit": "tok/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1000.0 / v, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "impl": "reference",
            "config": {"workload": "llama3-8b-pq-greedy-decode-d2-C256-b1 (CPU oracle: sampled rows of the PQ "
                                   "products, which are > 99% of its per-token time)",
                       "global_batch": 1, "seq_len": 1, "parallelism": "host-cores"},
            "cpu_baseline": {"value": v, "unit": "tok/s", "cores": sampler.threads, "kind": "oracle",
                             "sample": sampler.describe(rows)},
            "e2e": {"value": v, "unit": "tok/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def pq_chain_side(peak, steps=50):
    """The PQ linear stack alone (the round-1 headline): 224 chained PQ GEMVs
    of a token in the persistent chain kernel, N = 1."""
    import torch
    blocks = build_model(0, 1, seed=3)
    step = DecodeStep(blocks, 0, 1, None)
    step.h.copy_(__import__("synth").torch_activation(1, 4096, seed=11))
    for _ in range(3):
        step.chain.run(step.h)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        step.chain.run(step.h)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    gb = layer_bytes(1)
    out = {"ms_per_token": round(ms, 4), "tok_s": round(1e3 / ms, 1), "GBps": round(gb / ms / 1e6, 1),
           "frac": round(gb / ms / 1e6 / peak, 3), "algorithmic_bytes": gb}
    step.chain.free()
    for Ls in blocks:
        for L in Ls.values():
            L.free()
    torch.cuda.synchronize()
    return out


def llama_side(peak, settings=((2, 128, 1), (2, 256, 8)), steps=30):
    """Whole-model decode at effective 3-bit (2,128) and at batch 8, N = 1."""
    import torch
    out = {}
    for (d, c, B) in settings:
        model, by = build_llama(0, 1, d=d, c=c, B=B, seed=1)
        ms, g = llama_timed(model, steps, 3, 0, 1)
        ch, lm = llama_kernel_ms(model, 10, 1)
        out["d%d_C%d_B%d" % (d, c, B)] = {
            "ms_per_step": round(ms, 4), "tok_s": round(B * 1e3 / ms, 1),
            "chain_ms": round(ch, 4), "chain_frac": round(by["chain"] / ch / 1e6 / peak, 3),
            "lm_head_ms": round(lm, 4), "step_GBps": round(by["step"] / ms / 1e6, 1),
            "step_frac": round(by["step"] / ms / 1e6 / peak, 3)}
        del g
        model.free()
        torch.cuda.synchronize()
    return out


def _ncu_traffic(kernel: str):
    """dram__bytes_read.sum + dram__bytes_write.sum of one launch of `kernel`
    from the committed `ncu --set full` capture summary (profiles/), or None."""
    for path in (os.path.join(ROOT, "profiles", "r02", "ncu_traffic.json"),):
        try:
            with open(path) as f:
                v = json.load(f).get(kernel)
            if v:
                return v
        except Exception:
            pass
    return None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="fasq", choices=["fasq", "reference"])
    ap.add_argument("--no-side", action="store_true", help="skip prefill/pack/cpu side measurements")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    args.warmup = max(args.warmup, 3)

    import torch
    import torch.distributed as dist
    torch.cuda.set_device(local)
    pg = None
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        pg = dist.group.WORLD

    import paper_2605_04084_b200 as F

    B = 1
    model, by = build_llama(rank, world, B=B)
    if world > 1:
        handles = [None] * world
        dist.all_gather_object(handles, model.ipc_handle(), group=pg)
        model.set_peers(handles)
    peaks, peak_src = _peaks()
    peak = float(peaks.get("hbm_gbs", 6650.0))

    # ---- device-resident timed region: CUDA graph of one decode step ----
    with ClockSampler(local) as clk:
        ms, g = llama_timed(model, args.steps, args.warmup, rank, world)
    clocks = clk.summary()
    # ---- the two kernels of a step, timed separately on the launch stream ----
    ch_ms, lm_ms = llama_kernel_ms(model, max(10, min(50, args.steps)), world)
    # ---- e2e through the public API with host buffers ----
    ms_e2e = llama_e2e(model, args.steps, args.warmup, rank, world)

    if world > 1:   # every rank runs the traced step (the chains wait on each other)
        torch.cuda.synchronize()
        dist.barrier()
    split = llama_split(model, ms)
    tok_s = B * 1000.0 / ms
    achieved = by["chain"] / (ch_ms * 1e-3) / 1e9
    lm_gbs = by["lm_head"] / (lm_ms * 1e-3) / 1e9

    side = {}
    if world > 1 and not args.no_side:
        try:   # every rank takes part (NEXT-1 iii; at N = 1 it is side.prefill_model M2048); reported by rank 0
            side["prefill_token_sharded"] = prefill_token_sharded(world, rank, float(peaks.get("bf16_tflops", 1692.0)))
        except Exception as e:
            side["prefill_token_sharded"] = {"error": str(e)[:300]}
    if rank == 0 and world == 1 and not args.no_side:
        try:
            side["sustained_decode"] = llama_sustained(g)
        except Exception as e:
            side["sustained_decode"] = {"error": str(e)[:300]}
        try:
            side["prefill_e2e"] = llama_prefill_side(model)
        except Exception as e:
            side["prefill_e2e"] = {"error": str(e)[:300]}
    if rank == 0 and not args.no_side:
        del g
        for name, fn in (("pq_chain", lambda: pq_chain_side(peak)),
                         ("llama_variants", lambda: llama_side(peak)),
                         ("prefill_gemm_M512", lambda: prefill_tflops(M=512)),
                         ("prefill_gemm_M2048", lambda: prefill_tflops(M=2048)),
                         ("decode_sweep", lambda: decode_sweep(peak)),
                         ("decode_batch", lambda: decode_batch(peak)),
                         ("prefill_model", lambda: prefill_model(float(peaks.get("bf16_tflops", 1692.0)))),
                         ("gpu_pack", pack_time),
                         ("packed_gemv", lambda: packed_gemv_side(peak)),
                         ("dim0_gemv", lambda: dim0_gemv_side(peak)),
                         ("batch_gemv", lambda: batch_gemv_side(peak))):
            try:
                side[name] = fn()
            except Exception as e:  # report, never hide
                side[name] = {"error": str(e)[:300]}

    cpu = None
    if rank == 0 and world == 1 and not args.no_side:
        r, thr, sample, _ = oracle_decode_rate(budget_s=15.0)
        cpu = {"value": r, "unit": "tok/s", "cores": thr, "kind": "oracle", "sample": sample,
               "cpu": _cpu_model()}
        try:   # the same on one thread, and the oracle's pack of configs[0]
            import oracle
            import synth
            oracle.set_threads(1)
            r1, _, sample1, _ = oracle_decode_rate(budget_s=3.0)
            oracle.set_threads(thr)
            W0 = synth.weight(256, 512, seed=0)
            t0 = time.perf_counter()
            oracle.pack(W0, d=4, C=256, group=128, seed=0, iters=25)
            cpu["one_thread"] = {"value": r1, "sample": sample1}
            cpu["pack_config0_seconds"] = round(time.perf_counter() - t0, 3)
        except Exception as e:
            cpu["one_thread"] = {"error": str(e)[:200]}

    if rank == 0:
        line = {
            "metric": METRIC, "value": tok_s, "unit": "tok/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f16", "data": "synthetic",
            "config": {"workload": "llama3-8b-pq-greedy-decode-d2-C256-b1: whole Llama-3-8B-shaped model "
                                   "(embedding, 32 x {RMSNorm, PQ q/k/v, RoPE + KV cache + attention, PQ o + "
                                   "residual, RMSNorm, PQ gate/up, SwiGLU, PQ down + residual}, final RMSNorm, "
                                   "fp16 lm_head, greedy argmax), KV positions %d..%d (prompt %d, gen %d, P:438)"
                                   % (PROMPT, MAX_T - 1, PROMPT, MAX_T - PROMPT),
                       "executor": "fasq_llama: persistent chain kernel (all 161 steps) + lm_head/argmax kernel",
                       "global_batch": B, "seq_len": 1,
                       "parallelism": ("megatron-tp%d (fused NVLink all-reduce/gather in the counted stores)"
                                       % world) if world > 1 else "single-gpu",
                       "d": D, "C": C, "pq_bytes_per_step": by["pq"], "bytes_per_step": by["step"],
                       "l2": "inputs larger than L2 (%.2f GB per step vs 126 MB L2)" % (by["step"] / 1e9),
                       "timing": "CUDA graph of one step (2 launches), K replays between CUDA events, max over ranks"},
            "e2e": {"value": B * 1000.0 / ms_e2e, "unit": "tok/s", "h2d_bytes_per_step": 4 * B,
                    "d2h_bytes_per_step": 4 * B,
                    "how": "per step fasq_llama_step_io: H2D of the B tokens (pinned staging), chain + lm_head, "
                           "D2H of the chosen tokens, one synchronisation; wall clock"},
            "gpu_launches": 2 * args.steps,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": _ncu_traffic("k_chain"),
                         "kernel": "k_chain (whole-model decode chain; %.1f%% of the step)"
                                   % (100.0 * ch_ms / (ch_ms + lm_ms)),
                         "kernel_ms": ch_ms, "algorithmic_bytes": by["chain"],
                         "peak_source": "%s hbm_gbs" % peak_src,
                         "lm_head": {"kernel": "k_lm_head", "ms": lm_ms, "algorithmic_bytes": by["lm_head"],
                                     "GBps": lm_gbs, "frac": lm_gbs / peak,
                                     "traffic": _ncu_traffic("k_lm_head")},
                         "step_frac": by["step"] / (ms * 1e-3) / 1e9 / peak},
            "component_split": split,
            "clocks": clocks,
            "cpu_baseline": cpu,
            "side": side,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def _cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


if __name__ == "__main__":
    main()
