"""Pins of the whole-model decode oracle (oracle/llama.py) -- not GPU.

Each function is pinned by something other than its own formula:
  * RMSNorm: the closed form of the output's mean square, scale invariance,
    a constant vector;
  * RoPE: position 0 is the identity, each (i, i+hd/2) pair is a complex
    multiplication by exp(i*pos*theta_i) (numpy complex arithmetic), norms are
    preserved and <rope(q,m), rope(k,n)> depends only on m - n;
  * SwiGLU: silu(0) = 0, silu(x) -> x (x >> 0) and -> 0 (x << 0), scalar math;
  * attention: a single position returns v; equal keys return the mean of
    the values; a dominant key returns its value; GQA head -> KV-head mapping;
  * the block: all-zero PQ weights make it the identity (the residuals);
  * greedy: ties go to the lowest token id.
"""
import cmath
import math

import numpy as np

from oracle import llama as ol


def test_fp16_rounding():
    assert ol.fp16(1.0 + 2 ** -12) == 1.0            # below half an ulp of 1.0 (2^-10)
    assert ol.fp16(1.0 + 3 * 2 ** -12) == 1.0 + 2 ** -10
    assert ol.fp16(65520.0) == np.inf                # rounds past the largest finite fp16


def test_rmsnorm_closed_form_and_invariance():
    rng = np.random.default_rng(0)
    h = rng.normal(size=(3, 64))
    eps = 1e-5
    y = ol.rmsnorm(h, np.ones(64), eps)
    ms = np.mean(h * h, axis=1)
    assert np.allclose(np.mean(y * y, axis=1), ms / (ms + eps), rtol=1e-12)
    assert np.allclose(ol.rmsnorm(7.5 * h, np.ones(64), 0.0), ol.rmsnorm(h, np.ones(64), 0.0), rtol=1e-12)
    c = ol.rmsnorm(np.full(8, -3.0), np.arange(8.0), 0.0)
    assert np.allclose(c, -np.arange(8.0))
    g = rng.normal(size=64)
    assert np.allclose(ol.rmsnorm(h, g, eps), y * g)


def test_rope_is_complex_rotation():
    rng = np.random.default_rng(1)
    hd, theta = 16, 500000.0
    x = rng.normal(size=hd)
    assert np.array_equal(ol.rope(x, 0, theta), x)
    for pos in (1, 7, 300):
        y = ol.rope(x, pos, theta)
        for i in range(hd // 2):
            z = complex(x[i], x[i + hd // 2]) * cmath.exp(1j * pos * theta ** (-2.0 * i / hd))
            assert abs(y[i] - z.real) < 1e-12 and abs(y[i + hd // 2] - z.imag) < 1e-12
        assert abs(np.linalg.norm(y) - np.linalg.norm(x)) < 1e-12


def test_rope_relative_position():
    rng = np.random.default_rng(2)
    q, k = rng.normal(size=32), rng.normal(size=32)
    a = ol.rope(q, 10, 10000.0) @ ol.rope(k, 4, 10000.0)
    b = ol.rope(q, 106, 10000.0) @ ol.rope(k, 100, 10000.0)
    assert abs(a - b) < 1e-9


def test_silu_mul():
    assert ol.silu_mul(0.0, 5.0) == 0.0
    assert abs(ol.silu_mul(40.0, 1.0) - 40.0) < 1e-12
    assert abs(ol.silu_mul(-40.0, 1.0)) < 1e-15
    for g in (-2.5, -0.3, 0.7, 3.0):
        assert abs(ol.silu_mul(g, 2.0) - 2.0 * g / (1.0 + math.exp(-g))) < 1e-15


def _cache(n_kv, T, hd, seed):
    rng = np.random.default_rng(seed)
    return ol.fp16(rng.normal(size=(n_kv, T, hd))), ol.fp16(rng.normal(size=(n_kv, T, hd)))


def test_attention_single_position_returns_v():
    rng = np.random.default_rng(3)
    n_heads, n_kv, hd = 4, 2, 8
    q, k, v = rng.normal(size=n_heads * hd), rng.normal(size=n_kv * hd), rng.normal(size=n_kv * hd)
    kc, vc = _cache(n_kv, 4, hd, 4)
    o, _, v_new = ol.attention_decode(q, k, v, kc, vc, 0, n_heads, n_kv, 10000.0)
    for h in range(n_heads):                              # GQA: heads 0,1 -> kv 0; 2,3 -> kv 1
        assert np.allclose(o[h * hd:(h + 1) * hd], ol.fp16(v[(h // 2) * hd:(h // 2 + 1) * hd]))
    assert np.array_equal(v_new, ol.fp16(v.reshape(n_kv, hd)))


def test_attention_equal_keys_is_mean_of_values():
    rng = np.random.default_rng(5)
    n_heads, n_kv, hd, pos = 2, 1, 8, 5
    k = np.zeros(hd)                                       # rope(0) = 0: every key (cached too) is 0
    kc = np.zeros((n_kv, pos, hd))
    vc = ol.fp16(rng.normal(size=(n_kv, pos, hd)))
    v = rng.normal(size=hd)
    q = rng.normal(size=n_heads * hd)
    o, _, v_new = ol.attention_decode(q, k, v, kc, vc, pos, n_heads, n_kv, 10000.0)
    mean = (vc[0].sum(0) + v_new[0]) / (pos + 1)
    assert np.allclose(o[:hd], mean) and np.allclose(o[hd:], mean)


def test_attention_dominant_key():
    n_heads, n_kv, hd, pos = 1, 1, 4, 3
    kc = np.zeros((1, pos, hd))
    kc[0, 1] = [60.0, 0, 0, 0]
    vc = np.zeros((1, pos, hd))
    vc[0, 1] = [1.0, 2.0, 3.0, 4.0]
    q = ol.rope(np.array([60.0, 0, 0, 0]), -pos, 10000.0)   # rotated to (60, 0, 0, 0) at pos (rope(-pos) inverts)
    o, _, _ = ol.attention_decode(q, np.zeros(hd), np.zeros(hd), kc, vc, pos, n_heads, n_kv, 10000.0)
    assert np.allclose(o, [1.0, 2.0, 3.0, 4.0], atol=1e-12)


def test_block_with_zero_weights_is_identity():
    rng = np.random.default_rng(6)
    hidden, n_heads, n_kv, ffn, d, C = 64, 4, 2, 96, 2, 4

    def zero(fo, fi):
        return np.zeros((fi // d, C, d), np.float16), rng.integers(0, C, size=(fi // d, fo)).astype(np.uint8)
    hd = hidden // n_heads
    layer = {"q": zero(hidden, hidden), "k": zero(n_kv * hd, hidden), "v": zero(n_kv * hd, hidden),
             "o": zero(hidden, hidden), "gate": zero(ffn, hidden), "up": zero(ffn, hidden),
             "down": zero(hidden, ffn), "attn_norm": np.ones(hidden, np.float16),
             "mlp_norm": np.ones(hidden, np.float16)}
    h = rng.normal(size=hidden)
    kc, vc = _cache(n_kv, 3, hd, 7)
    r = ol.block_decode(h, layer, 3, kc, vc, n_heads, n_kv, 1e-5, 500000.0)
    assert np.array_equal(r["h_mid"], h) and np.array_equal(r["h_out"], h)
    assert np.all(r["o"] == 0.0) and np.all(r["down"] == 0.0)


def test_greedy_ties_lowest_id():
    assert ol.greedy([1.0, 3.0, 3.0, 2.0]) == 1
    assert ol.greedy([-1.0, -1.0]) == 0


def test_lm_head_is_dense_product():
    rng = np.random.default_rng(8)
    W = rng.normal(size=(10, 16)).astype(np.float16)
    h = rng.normal(size=16)
    g = np.ones(16, np.float16)
    x = ol.fp16(h / np.sqrt(np.mean(h * h) + 1e-5))
    assert np.allclose(ol.lm_head_logits(h, g, W, 1e-5), [float(np.dot(W[i].astype(np.float64), x)) for i in range(10)])
