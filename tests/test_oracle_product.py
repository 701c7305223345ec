"""Pins of the oracle's product y = W_hat . x (Eq. 3) -- not GPU.

  * brute force: exact rational arithmetic (fractions) over the fp16 values,
    compared with the oracle's fp64 result within fp64 summation rounding;
  * saturation: y == W . x for the ORIGINAL W (numpy fp64 matmul, a library
    routine) when the codebook is saturated;
  * C = 1: every output equals sum_ss dot(x_ss, c_ss);
  * basis vectors x = e_i give column i of W_hat; x = 0 gives 0;
  * linearity in x (north_star); GEMM row l == GEMV(x_l);
  * sampled rows equal the full product's rows.
"""
from fractions import Fraction

import numpy as np
import pytest

import synth


@pytest.mark.parametrize("d,C,group", [(1, 3, 1), (2, 4, 1), (2, 5, 3), (4, 2, 2), (8, 3, 1)])
def test_brute_force_exact(oracle_lib, d, C, group):
    F_out, F_in = 5, 8 * 3 if d < 8 else 24
    if (F_in // d) % group:
        F_in = d * group * 2
    cb, idx = synth.random_layer(F_out, F_in, d, C, group=group, seed=d + C, std=1.0)
    x = synth.activation(2, F_in, seed=9)
    y = oracle_lib.gemv(cb, idx, x, group=group)
    N_ss = F_in // d
    for b in range(2):
        for j in range(F_out):
            exact = Fraction(0)
            for ss in range(N_ss):
                k = int(idx[ss, j])
                for e in range(d):
                    exact += Fraction(float(cb[ss // group, k, e])) * Fraction(float(x[b, ss * d + e]))
            # fp64 left-to-right sum of F_in exact terms: |err| <= F_in * eps * sum|terms|
            bound = F_in * 2.0 ** -53 * float(sum(abs(Fraction(float(cb[ss // group, int(idx[ss, j]), e]))
                                                       * Fraction(float(x[b, ss * d + e])))
                                                   for ss in range(N_ss) for e in range(d)))
            assert abs(y[b, j] - float(exact)) <= bound + 1e-300


def test_saturation_equals_dense(oracle_lib):
    W = synth.structured_weight(96, 64, 2, 7, group=1, seed=3)
    cb, idx, _ = oracle_lib.pack(W, d=2, C=8, group=1, seed=0)
    x = synth.activation(3, 64, seed=4)
    y = oracle_lib.gemv(cb, idx, x)
    ref = x.astype(np.float64) @ W.astype(np.float64).T
    assert np.allclose(y, ref, rtol=1e-13, atol=1e-13)


def test_C1_constant_rows(oracle_lib):
    cb, idx = synth.random_layer(40, 32, 2, 1, seed=2)
    idx[:] = 0
    x = synth.activation(1, 32, seed=1)
    y = oracle_lib.gemv(cb, idx, x)
    want = sum(float(np.dot(cb[ss, 0].astype(np.float64), x[0, 2 * ss:2 * ss + 2].astype(np.float64)))
               for ss in range(16))
    assert np.allclose(y, want, rtol=1e-14)


def test_basis_vectors_give_columns(oracle_lib):
    cb, idx = synth.random_layer(33, 24, 4, 16, group=2, seed=6)
    What = oracle_lib.reconstruct(cb, idx, 24, group=2).astype(np.float64)
    X = np.eye(24, dtype=np.float16)
    Y = oracle_lib.gemm(cb, idx, X, group=2)
    assert np.array_equal(Y, What.T)
    assert np.all(oracle_lib.gemv(cb, idx, np.zeros((1, 24), np.float16), group=2) == 0)


def test_linearity(oracle_lib):
    cb, idx = synth.random_layer(64, 128, 2, 32, seed=1)
    x1 = synth.activation(1, 128, seed=1)
    x2 = synth.activation(1, 128, seed=2)
    # integer-valued fp16 combos keep 2*x1 and x1+x2 exact in fp16
    a = oracle_lib.gemv(cb, idx, (x1.astype(np.float32) * 2).astype(np.float16))
    assert np.allclose(a, 2 * oracle_lib.gemv(cb, idx, x1), rtol=1e-14, atol=1e-14)
    s = (x1.astype(np.float64) + x2.astype(np.float64))
    if np.array_equal(s.astype(np.float16).astype(np.float64), s):
        b = oracle_lib.gemv(cb, idx, s.astype(np.float16))
        assert np.allclose(b, oracle_lib.gemv(cb, idx, x1) + oracle_lib.gemv(cb, idx, x2), rtol=1e-12, atol=1e-12)
    # general check via reconstruct: y(x1+x2) - y(x1) - y(x2) within rounding of the fp16 sum
    What = oracle_lib.reconstruct(cb, idx, 128).astype(np.float64)
    assert np.allclose(oracle_lib.gemv(cb, idx, x1)[0], What @ x1[0].astype(np.float64), rtol=1e-12, atol=1e-12)


def test_gemm_rows_equal_gemv(oracle_lib):
    cb, idx = synth.random_layer(48, 64, 2, 16, seed=3)
    X = synth.activation(5, 64, seed=7)
    Y = oracle_lib.gemm(cb, idx, X)
    for l in range(5):
        assert np.array_equal(Y[l], oracle_lib.gemv(cb, idx, X[l:l + 1])[0])


def test_row_sampling(oracle_lib):
    cb, idx = synth.random_layer(100, 64, 2, 16, seed=4)
    X = synth.activation(2, 64, seed=7)
    Y = oracle_lib.gemm(cb, idx, X)
    assert np.array_equal(oracle_lib.gemm(cb, idx, X, rows=(17, 63)), Y[:, 17:63])
