"""Parity at the configurations bench.py times (VERDICT r1 "weak 1"): the
full-size runs are checked against the oracle on SAMPLED outputs the oracle
computes one by one, with the GPU's own inputs of each step ("teacher
forcing": a step's input is the GPU's previous output, rounded exactly as the
kernel rounds it), so a wrong result anywhere in the 32 blocks fails here.

* the PQ-only decode chain (bench side "pq_chain" / decode_sweep / decode_batch):
  32 Llama-3-8B blocks x {qkv, o, gate/up, down}, 148 CTAs, at (2,256) B=1,
  (2,128) B=1 and (2,256) B=8;
* the whole-model decode (bench headline, bench.build_llama): every block's
  q/k/v, attention, h', gate/up and h'' plus the lm_head logits and the greedy
  token, at the first (pos 128) and last (pos 255) position of the timed cycle;
* the prefill GEMM-EXPAND at M = 2048 on every Llama shape (full-K waves and
  the split-K tail launch) and GEMM-LUT on a full Llama shape.

Tolerances: north_star's rel-L2 <= 1e-3 and max-abs <= 5e-3 ||x||_inf sqrt(K)
(fasq_testutil.parity_ok) for every PQ product; 1e-3 rel-L2 for attention
outputs, residual sums and logits.
"""
import numpy as np
import pytest
import torch

import synth
from fasq_testutil import parity_ok
from oracle import llama as ol

pytestmark = pytest.mark.gpu

NAMES = [("q_proj", "k_proj", "v_proj"), ("o_proj",), ("gate_proj", "up_proj"), ("down_proj",)]


@pytest.fixture(scope="module")
def F():
    import paper_2605_04084_b200 as F
    return F


def _rel(y, ref):
    y, ref = np.asarray(y, np.float64), np.asarray(ref, np.float64)
    return float(np.linalg.norm(y - ref) / max(np.linalg.norm(ref), 1e-300))


def _windows(F_out, rng, n=48):
    """First, a random and the last row window of a layer (rows [j0, j1))."""
    j = int(rng.integers(n, F_out - 2 * n))
    return ((0, n), (j, j + n), (F_out - n, F_out))


def _check_rows(oracle_lib, layer, xin, y_all, rng, tag):
    """y_all [B][F_out] (GPU, fp32) vs the oracle on sampled row windows of
    the layer, input xin [B][F_in] (fp16, the GPU's own)."""
    cb, idx = layer.export()
    cbn = cb.cpu().numpy()
    for (j0, j1) in _windows(layer.F_out, rng):
        idxn = idx[:, j0:j1].contiguous().cpu().numpy()
        ref = oracle_lib.gemv(cbn, idxn, xin)
        ok, info = parity_ok(y_all[:, j0:j1], ref, xin, xin.shape[1])
        assert ok, (tag, j0, info)


@pytest.mark.parametrize("d,C,B", [(2, 256, 1), (2, 128, 1), (2, 256, 8)])
def test_pq_chain_full_bench_config(F, oracle_lib, d, C, B):
    """The 128-step PQ chain of 32 Llama-3-8B blocks (one launch per token, the
    planner's uneven K ranges on every SM) at the benched settings."""
    blocks = []
    for b in range(32):
        Ls = {}
        for li, (name, fo, fi) in enumerate(synth.LLAMA3_8B_LAYERS):
            cb, idx = synth.torch_random_layer(fo, fi, d, C, seed=4000 + b * 7 + li)
            Ls[name] = F.import_layer(cb, idx, fi)
            del cb, idx
        blocks.append(Ls)
    steps = []
    for b in range(32):
        for i in range(4):
            steps.append(([blocks[b][n] for n in NAMES[i]], None if not steps else (len(steps) - 1, 0)))
    ch = F.Chain(steps, B=B)
    x = synth.torch_activation(B, 4096, seed=21)
    for _ in range(2):   # both arena parities
        ch.run(x)
    torch.cuda.synchronize()
    ch.check()
    rng = np.random.default_rng(d * 1000 + C + B)
    for s in range(len(steps)):
        b, i = divmod(s, 4)
        xin = x.cpu().numpy() if s == 0 else ch.output(s - 1, 0, out_dtype=torch.float16).cpu().numpy()
        for l, n in enumerate(NAMES[i]):
            y = ch.output(s, l, out_dtype=torch.float32).cpu().numpy()
            _check_rows(oracle_lib, blocks[b][n], xin, y, rng, (d, C, B, b, n))
    ch.free()
    for Ls in blocks:
        for L in Ls.values():
            L.free()


def _llama_check_step(F, oracle_lib, model, keep, pos, B, rng, logits_gpu, tokens_gpu, lm_host):
    """Teacher-forced check of one decode step of every block (see module doc)."""
    layers, fn, emb, _ = keep
    hd, H, KV = 128, 32, 8
    acc = lambda s, l=0: model.output(s, l, out_dtype=torch.int64).cpu().numpy().astype(np.float64) * 2.0 ** -32
    h = acc(0)   # the embedding rows (exact)
    hist = model.token_history().cpu().numpy()
    for b in range(B):
        tok = int(hist[b, pos])
        assert np.array_equal(h[b], emb[tok].float().cpu().numpy().astype(np.float64)), ("embed", b)
    for l, L in enumerate(layers):
        base = 1 + 5 * l
        an = L["attn_norm"].cpu().numpy()
        mn = L["mlp_norm"].cpu().numpy()
        # q/k/v: products of fp16(RMSNorm(h) * gamma), sampled rows
        x = np.stack([ol.fp16(ol.rmsnorm(h[b], an, 1e-5)) for b in range(B)])
        qkv = []
        for li, n in enumerate(("q", "k", "v")):
            y = acc(base, li)
            qkv.append(y)
            _check_rows(oracle_lib, L[n], x.astype(np.float16), y, rng, ("llama", pos, l, n))
        # attention: the GPU's q/k/v, the GPU's cache rows < pos, fp64
        Kc, Vc = model.kv_cache(l)
        att = acc(base + 1)
        for b in range(B):
            kc = Kc[b, :, :pos].float().cpu().numpy().astype(np.float64)
            vc = Vc[b, :, :pos].float().cpu().numpy().astype(np.float64)
            o_ref, k_new, v_new = ol.attention_decode(qkv[0][b], qkv[1][b], qkv[2][b], kc, vc, pos, H, KV, 500000.0)
            assert _rel(att[b], o_ref) <= 1e-3, ("attn", pos, l, b, _rel(att[b], o_ref))
            kn = Kc[b, :, pos].float().cpu().numpy()
            assert _rel(kn, k_new) <= 2e-3, ("k_new", pos, l, b)
        # o + residual (lazy sum), sampled rows of o through the GPU's attention output
        h_mid = acc(base + 2)
        xo = att.astype(np.float16)
        cb, idx = L["o"].export()
        cbn = cb.cpu().numpy()
        for (j0, j1) in _windows(4096, rng):
            ref = oracle_lib.gemv(cbn, idx[:, j0:j1].contiguous().cpu().numpy(), xo) + h[:, j0:j1]
            assert _rel(h_mid[:, j0:j1], ref) <= 1e-3, ("h_mid", pos, l, j0)
        # gate/up from RMSNorm(h'), then down(silu(g) * u) + h'
        xm = np.stack([ol.fp16(ol.rmsnorm(h_mid[b], mn, 1e-5)) for b in range(B)])
        g = acc(base + 3, 0)
        u = acc(base + 3, 1)
        _check_rows(oracle_lib, L["gate"], xm.astype(np.float16), g, rng, ("llama", pos, l, "gate"))
        _check_rows(oracle_lib, L["up"], xm.astype(np.float16), u, rng, ("llama", pos, l, "up"))
        h_out = acc(base + 4)
        act = ol.fp16(ol.silu_mul(g, u)).astype(np.float16)
        cb, idx = L["down"].export()
        cbn = cb.cpu().numpy()
        for (j0, j1) in _windows(4096, rng):
            ref = oracle_lib.gemv(cbn, idx[:, j0:j1].contiguous().cpu().numpy(), act) + h_mid[:, j0:j1]
            assert _rel(h_out[:, j0:j1], ref) <= 1e-3, ("h_out", pos, l, j0)
        h = h_out
    # lm_head over the GPU's final h: full logits (fp64), greedy token
    fnn = fn.cpu().numpy()
    for b in range(B):
        lg_ref = ol.lm_head_logits(h[b], fnn, lm_host, 1e-5)
        assert _rel(logits_gpu[b], lg_ref) <= 1e-3, ("logits", pos, b)
        top = np.sort(lg_ref)[-2:]
        t = int(tokens_gpu[b])
        if top[1] - top[0] > 1e-2 * max(1.0, abs(top[1])):
            assert t == ol.greedy(lg_ref), ("token", pos, b)
        else:   # a near tie: the GPU's choice must be one of the maxima within tolerance
            assert lg_ref[t] >= top[1] - 2e-2 * max(1.0, abs(top[1])), ("token (near tie)", pos, b)


@pytest.mark.parametrize("d,C,B,n_layers", [(2, 256, 1, 32), (2, 128, 1, 32), (2, 256, 8, 4)])
def test_llama_full_bench_config(F, oracle_lib, d, C, B, n_layers):
    """bench.py's headline model (bench.build_llama: 32 Llama-3-8B blocks,
    fp16 embedding / lm_head, 148 CTAs, 4 cache parts, KV positions
    128..255), checked block by block at the first and the last position of
    the decode cycle (B = 8: 4 blocks, same kernels and plan per step)."""
    import bench
    model, _ = bench.build_llama(0, 1, d=d, c=C, B=B, seed=3, n_layers=n_layers)
    keep = model._bench_keep
    lm_host = keep[3].cpu().numpy()
    logits = model.enable_logits(True)
    model.reset([128000 + 17 * b for b in range(B)], bench.PROMPT)
    rng = np.random.default_rng(d + C + B)
    for it in range(bench.MAX_T - bench.PROMPT):
        model.step()
        pos = bench.PROMPT + it
        if it in (0, bench.MAX_T - bench.PROMPT - 1):
            torch.cuda.synchronize()
            _llama_check_step(F, oracle_lib, model, keep, pos, B, rng, logits.cpu().numpy(),
                              model.tokens().cpu().numpy(), lm_host)
    model.free()


@pytest.mark.parametrize("F_out,F_in", [(4096, 4096), (1024, 4096), (14336, 4096), (4096, 14336)])
def test_gemm_expand_M2048_all_shapes(F, oracle_lib, F_out, F_in):
    """Prefill EXPAND at M = 2048 (bench configs[3]): 4096-row layers run the
    full-K single launch (128 tiles), 14336-row layers three full waves plus
    the split-K tail launch -- sampled tokens over the whole M range (every
    token tile, including the last), sampled row windows."""
    cb, idx = synth.torch_random_layer(F_out, F_in, 2, 256, seed=F_out * 3 + F_in)
    L = F.import_layer(cb, idx, F_in)
    X = synth.torch_activation(2048, F_in, seed=9)
    Y = F.gemm(L, X, out_dtype=torch.float32, algo=F.GEMM_EXPAND_TC)
    torch.cuda.synchronize()
    toks = np.concatenate([np.arange(0, 2048, 128) + (np.arange(16) * 7) % 128, [2047]])
    Xs = X[torch.from_numpy(toks).cuda()].cpu().numpy()
    Ys = Y[torch.from_numpy(toks).cuda()].cpu().numpy()
    cbn = cb.cpu().numpy()
    rng = np.random.default_rng(F_out)
    for (j0, j1) in _windows(F_out, rng, n=64):
        ref = oracle_lib.gemm(cbn, idx[:, j0:j1].contiguous().cpu().numpy(), Xs)
        ok, info = parity_ok(Ys[:, j0:j1], ref, Xs, F_in)
        assert ok, (F_out, F_in, j0, info)
    L.free()


def test_gemm_lut_full_llama_shape(F, oracle_lib):
    """GEMM-LUT on a full Llama-3-8B shape (4096 x 14336), M = 64 (LUT is
    the short-L path), sampled rows."""
    F_out, F_in, M = 4096, 14336, 64
    cb, idx = synth.torch_random_layer(F_out, F_in, 2, 256, seed=55)
    L = F.import_layer(cb, idx, F_in)
    X = synth.torch_activation(M, F_in, seed=56)
    Y = F.gemm(L, X, out_dtype=torch.float32, algo=F.GEMM_LUT).cpu().numpy()
    Xn = X.cpu().numpy()
    cbn = cb.cpu().numpy()
    rng = np.random.default_rng(5)
    for (j0, j1) in _windows(F_out, rng, n=64):
        ref = oracle_lib.gemm(cbn, idx[:, j0:j1].contiguous().cpu().numpy(), Xn)
        ok, info = parity_ok(Y[:, j0:j1], ref, Xn, F_in)
        assert ok, (j0, info)
    L.free()
