"""Whole-model decode oracle -- TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Plain numpy fp64 reference of one greedy decode step of a Llama-shaped decoder
whose linear layers are FASQ layers: the paper's end-to-end setting (Meta-
Llama-3-8B, every linear layer of the decoder blocks product-quantized, P:219;
embeddings / norms / lm_head uncompressed; greedy decode with a prompt
of 128 and 128 generated tokens).  The paper does not restate the
Llama architecture; the block below is the public HF Llama definition
(reading R14): pre-norm RMSNorm, RoPE
rotate-half with theta, grouped-query attention, SwiGLU MLP, residuals.

The PQ products are the C oracle's fp64 reconstruct-then-multiply (Eq. 3,
P:200-203).  Everything else is fp64, with fp16 rounding exactly where the
fp16 model holds fp16 tensors (reading R15): the inputs of every
PQ product (Eq. 3 takes fp16 x; "FP16 activations") and the KV cache.
No blocking, fusion or reordering: each function is its textbook formula.
"""
from __future__ import annotations

import numpy as np

from . import gemv as pq_gemv


def fp16(x) -> np.ndarray:
    """Round to fp16 (IEEE RN, numpy) and return as fp64."""
    return np.asarray(x, np.float64).astype(np.float16).astype(np.float64)


def rmsnorm(h, gamma, eps: float) -> np.ndarray:
    """RMSNorm(h) = h / sqrt(mean(h^2) + eps) * gamma, over the last axis."""
    h = np.asarray(h, np.float64)
    ms = np.mean(h * h, axis=-1, keepdims=True)
    return h / np.sqrt(ms + eps) * np.asarray(gamma, np.float64)


def rope(x, pos: int, theta: float) -> np.ndarray:
    """Rotate-half RoPE of one head vector (or [..., hd]) at position pos:
    x'[i] = x[i] cos(a_i) - x[i+hd/2] sin(a_i), x'[i+hd/2] = x[i+hd/2] cos(a_i)
    + x[i] sin(a_i), a_i = pos * theta^(-2i/hd)."""
    x = np.asarray(x, np.float64)
    hd = x.shape[-1]
    half = hd // 2
    i = np.arange(half, dtype=np.float64)
    a = pos * theta ** (-2.0 * i / hd)
    c, s = np.cos(a), np.sin(a)
    x0, x1 = x[..., :half], x[..., half:]
    return np.concatenate([x0 * c - x1 * s, x1 * c + x0 * s], axis=-1)


def silu_mul(g, u) -> np.ndarray:
    """SwiGLU: silu(g) * u with silu(g) = g / (1 + exp(-g))."""
    g = np.asarray(g, np.float64)
    return g / (1.0 + np.exp(-g)) * np.asarray(u, np.float64)


def attention_decode(q, k, v, k_cache, v_cache, pos: int, n_heads: int, n_kv: int, theta: float):
    """One token's attention at position pos for ONE sequence.
    q [n_heads*hd], k/v [n_kv*hd] (pre-RoPE projections); k_cache/v_cache
    [n_kv][>=pos][hd] hold positions < pos (fp16 values).  The new k (after
    RoPE) and v enter the cache as fp16.  Returns (o [n_heads*hd], k_new fp16
    [n_kv][hd], v_new fp16 [n_kv][hd])."""
    q = np.asarray(q, np.float64)
    hd = q.size // n_heads
    k = np.asarray(k, np.float64).reshape(n_kv, hd)
    v = np.asarray(v, np.float64).reshape(n_kv, hd)
    k_new = fp16(np.stack([rope(k[j], pos, theta) for j in range(n_kv)]))
    v_new = fp16(v)
    grp = n_heads // n_kv
    o = np.zeros((n_heads, hd))
    for h in range(n_heads):
        j = h // grp
        K = np.concatenate([np.asarray(k_cache[j][:pos], np.float64), k_new[j][None]], 0)
        V = np.concatenate([np.asarray(v_cache[j][:pos], np.float64), v_new[j][None]], 0)
        s = K @ rope(q[h * hd:(h + 1) * hd], pos, theta) / np.sqrt(hd)
        p = np.exp(s - s.max())
        p /= p.sum()
        o[h] = p @ V
    return o.reshape(-1), k_new, v_new


def block_decode(h, layer, pos: int, k_cache, v_cache, n_heads: int, n_kv: int, eps: float, theta: float):
    """One decoder block for ONE sequence at position pos.
    h fp64 [hidden]; layer: dict of PQ layers (codebooks, indices) for q, k, v,
    o, gate, up, down and fp16 norm weights attn_norm, mlp_norm.  Returns the
    intermediates: x (fp16 normed input), q, k, v, attn, h_mid, xm, gate, up,
    act (fp16), h_out, k_new, v_new."""
    r = {}
    h = np.asarray(h, np.float64)
    r["x"] = fp16(rmsnorm(h, layer["attn_norm"], eps))
    for n in ("q", "k", "v"):
        cb, idx = layer[n]
        r[n] = pq_gemv(cb, idx, r["x"].astype(np.float16))[0]
    r["attn"], r["k_new"], r["v_new"] = attention_decode(r["q"], r["k"], r["v"], k_cache, v_cache, pos, n_heads,
                                                         n_kv, theta)
    cb, idx = layer["o"]
    r["o"] = pq_gemv(cb, idx, fp16(r["attn"]).astype(np.float16))[0]
    r["h_mid"] = h + r["o"]
    r["xm"] = fp16(rmsnorm(r["h_mid"], layer["mlp_norm"], eps))
    for n in ("gate", "up"):
        cb, idx = layer[n]
        r[n] = pq_gemv(cb, idx, r["xm"].astype(np.float16))[0]
    r["act"] = fp16(silu_mul(r["gate"], r["up"]))
    cb, idx = layer["down"]
    r["down"] = pq_gemv(cb, idx, r["act"].astype(np.float16))[0]
    r["h_out"] = r["h_mid"] + r["down"]
    return r


def lm_head_logits(h, final_norm, W_lm, eps: float) -> np.ndarray:
    """logits = W_lm . fp16(RMSNorm(h) * gamma), fp64 (W_lm fp16 [V][hidden])."""
    x = fp16(rmsnorm(h, final_norm, eps))
    W_lm = np.asarray(W_lm)
    out = np.empty(W_lm.shape[0])
    for r0 in range(0, W_lm.shape[0], 8192):   # rows in slices only to bound host memory
        out[r0:r0 + 8192] = W_lm[r0:r0 + 8192].astype(np.float64) @ x
    return out


def greedy(logits) -> int:
    """argmax with ties to the lowest token id (numpy's first maximum)."""
    return int(np.argmax(np.asarray(logits)))


def prefill(tokens, layers, embed, k_cache, v_cache, pos0: int, n_heads: int, n_kv: int, eps: float, theta: float):
    """Causal prefill of ONE sequence: the prompt tokens at positions pos0, pos0+1, ...
    By definition of causal attention this is the decode step applied to each
    prompt token in order with the KV cache growing (no blocking, no batching).
    k_cache / v_cache: per layer, per KV head, python lists of fp16-valued rows for
    positions < pos0 (extended in place).  Returns the last position's h_out and
    the per-layer new K/V rows [M][n_kv][hd]."""
    new_k = [[] for _ in layers]
    new_v = [[] for _ in layers]
    h = None
    for i, t in enumerate(tokens):
        pos = pos0 + i
        h = np.asarray(embed[t], np.float64)
        for l, L in enumerate(layers):
            hd = L["q"][1].shape[1] // n_heads          # q rows (T_index [N_ss][F_out]) / heads
            K = [np.asarray(k_cache[l][j], np.float64).reshape(len(k_cache[l][j]), hd) for j in range(n_kv)]
            V = [np.asarray(v_cache[l][j], np.float64).reshape(len(v_cache[l][j]), hd) for j in range(n_kv)]
            r = block_decode(h, L, pos, K, V, n_heads, n_kv, eps, theta)
            for j in range(n_kv):
                k_cache[l][j].append(r["k_new"][j])
                v_cache[l][j].append(r["v_new"][j])
            new_k[l].append(r["k_new"])
            new_v[l].append(r["v_new"])
            h = r["h_out"]
    return h, [np.array(x) for x in new_k], [np.array(x) for x in new_v]
