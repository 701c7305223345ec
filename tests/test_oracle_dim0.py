"""Pins of the oracle's dim = 0 partition (NEXT-4): subspaces along the OUTPUT
axis (Eq. 2 first case; the layout of the paper's experiments,
P:444) -- not GPU.

  * saturation: with <= C distinct column slices per codebook the pack is
    exact (reconstruction == W bitwise) and the product equals numpy's
    fp64 W . x of the original W (a library routine);
  * the product against exact rational brute force written from the
    definition y[ss*d+e] = sum_j x[j] * T_cluster[ss/group][T_index[ss][j]][e];
  * C = 1 closed form: y[ss*d+e] = c[ss/group][0][e] * sum_j x[j];
  * every stored index is a nearest centroid of the stored codebook (fp64);
  * the output-axis geometry: reconstruct_dim0 puts codebook entry e of
    subspace ss on output row ss*d+e (a transposed-operand slip fails it).
"""
from fractions import Fraction

import numpy as np
import pytest

import synth


def _structured_dim0(F_out, F_in, d, n, group, seed):
    # column slices of d consecutive rows drawn from <= n distinct vectors per
    # codebook: the dim = 1 structure of the transposed matrix
    return np.ascontiguousarray(synth.structured_weight(F_in, F_out, d, n, group=group, seed=seed).T)


@pytest.mark.parametrize("d,C,group,n", [(2, 16, 1, 9), (2, 256, 4, 200), (4, 32, 2, 32), (1, 8, 1, 8),
                                         (8, 4, 1, 3)])
def test_saturation_exact_dim0(oracle_lib, d, C, group, n):
    F_out, F_in = 32 * d, 96
    W = _structured_dim0(F_out, F_in, d, n, group, seed=d + C)
    cb, idx, _ = oracle_lib.pack_dim0(W, d=d, C=C, group=group, seed=2)
    assert idx.shape == (F_out // d, F_in)
    What = oracle_lib.reconstruct_dim0(cb, idx, F_out, group=group)
    Wc = W.view(np.uint16).copy()
    Wc[Wc == 0x8000] = 0
    assert np.array_equal(What.view(np.uint16), Wc)
    x = synth.activation(2, F_in, seed=3)
    y = oracle_lib.gemm_dim0(cb, idx, x, group=group)
    assert np.allclose(y, x.astype(np.float64) @ W.astype(np.float64).T, rtol=1e-12, atol=1e-12)


def test_product_brute_force_dim0(oracle_lib):
    d, C, group, F_out, F_in = 2, 5, 2, 8, 6
    N_ss = F_out // d
    g = synth.rng(4)
    cb = g.normal(size=(N_ss // group, C, d)).astype(np.float16)
    idx = g.integers(0, C, size=(N_ss, F_in), dtype=np.uint8)
    x = synth.activation(2, F_in, seed=5)
    y = oracle_lib.gemm_dim0(cb, idx, x, group=group)
    for b in range(2):
        for ss in range(N_ss):
            for e in range(d):
                terms = [Fraction(float(x[b, j])) * Fraction(float(cb[ss // group, int(idx[ss, j]), e]))
                         for j in range(F_in)]
                exact = sum(terms, Fraction(0))
                bound = F_in * 2.0 ** -53 * float(sum(abs(t) for t in terms))
                assert abs(y[b, ss * d + e] - float(exact)) <= bound + 1e-300


def test_C1_closed_form_dim0(oracle_lib):
    d, group, F_out, F_in = 4, 2, 16, 40
    g = synth.rng(7)
    cb = g.normal(size=(F_out // d // group, 1, d)).astype(np.float16)
    idx = np.zeros((F_out // d, F_in), np.uint8)
    x = synth.activation(1, F_in, seed=8)
    y = oracle_lib.gemm_dim0(cb, idx, x, group=group)
    sx = sum(Fraction(float(v)) for v in x[0])
    for o in range(F_out):
        ss, e = divmod(o, d)
        want = Fraction(float(cb[ss // group, 0, e])) * sx
        assert abs(y[0, o] - float(want)) <= 1e-12 * max(1.0, abs(float(want)))


def test_indices_nearest_dim0(oracle_lib):
    d, C, group, F_out, F_in = 2, 16, 2, 64, 80
    W = synth.weight(F_out, F_in, seed=6)
    cb, idx, _ = oracle_lib.pack_dim0(W, d=d, C=C, group=group, seed=1, iters=10)
    for ss in range(F_out // d):
        c = cb[ss // group].astype(np.float64)
        p = W[ss * d:(ss + 1) * d, :].T.astype(np.float64)          # F_in points of dimension d
        D = ((p[:, None, :] - c[None]) ** 2).sum(-1)
        chosen = D[np.arange(F_in), idx[ss]]
        assert np.all(chosen <= D.min(1) * (1 + 1e-6) + 1e-30)


def test_geometry_dim0(oracle_lib):
    d, C, F_out, F_in = 2, 3, 6, 4
    cb = np.arange(3 * C * d, dtype=np.float16).reshape(3, C, d)
    idx = np.array([[0, 1, 2, 0], [2, 2, 1, 0], [1, 0, 0, 2]], np.uint8)
    What = oracle_lib.reconstruct_dim0(cb, idx, F_out).astype(np.float64)
    for o in range(F_out):
        for j in range(F_in):
            assert What[o, j] == float(cb[o // d, idx[o // d, j], o % d])
