"""Pins of the oracle's wide-index entry points (NEXT-2) -- not GPU.

Eq. 4 stores one ceil(log2 K_s)-bit index per datapoint and
subspace; Table 2 uses K_s up to 1024 (2-512 at #W 4.5, 2-1024 at
#W 5.0).  The oracle keeps its arithmetic and widens only the stored index
(uint16 for C <= 1024).  Pinned here against things other than itself:

  * ceil(log2 C) against the paper's printed #W (tests/golden) and against
    integer arithmetic for every C in 1..1024;
  * saturation at C = 512 / 1024 with more than 256 distinct sub-vectors per
    codebook: reconstruction == W bitwise, and indices above 255 occur (a
    uint8 truncation anywhere would break exactness);
  * the lowest-k tie rule with duplicated init slots above 256;
  * the product with uint16 indices against exact rational brute force;
  * Lloyd's fixed-point conditions at C = 300 (exact cluster means, nearest
    centroid in fp64);
  * validation: C = 1025 rejected, C = 257 rejected by the uint8 entry point.
"""
from fractions import Fraction

import numpy as np
import pytest

import synth


def test_index_bits_matches_eq4_and_table2(oracle_lib, pins):
    for C in range(1, 1025):
        b = oracle_lib.index_bits(C)
        assert (1 << b) >= C and (b == 0 or (1 << (b - 1)) < C), C
    for name, w in pins["eff_bits_W"].items():
        if name.startswith("_"):
            continue
        d, C = (int(v) for v in name.split("-"))
        assert oracle_lib.index_bits(C) / d == w, name


@pytest.mark.parametrize("C,n_distinct,group", [(512, 400, 1), (1024, 900, 2), (1024, 1024, 4)])
def test_saturation_exact_wide(oracle_lib, C, n_distinct, group):
    d = 2
    F_out, F_in = 1100, 4 * d * group
    W = synth.structured_weight(F_out, F_in, d, n_distinct, group=group, seed=C + n_distinct)
    cb, idx, _ = oracle_lib.pack(W, d=d, C=C, group=group, seed=5, iters=3)
    assert idx.dtype == np.uint16
    assert int(idx.max()) > 255                     # wide indices really occur
    What = oracle_lib.reconstruct(cb, idx, F_in, group=group)
    Wc = W.view(np.uint16).copy()
    Wc[Wc == 0x8000] = 0                            # reading R2
    assert np.array_equal(What.view(np.uint16), Wc)


def test_tie_rule_lowest_k_wide(oracle_lib):
    """Reading R5 with C > 256: slots >= m copy slot 0 (R3), so points equal to
    codebook[0] tie with slots m..C-1; the lowest k (0) must win and no index
    may reach a duplicate slot."""
    d, C, n_distinct = 2, 700, 300
    W = synth.structured_weight(2000, 4 * d, d, n_distinct, group=1, seed=12)
    cb, idx, _ = oracle_lib.pack(W, d=d, C=C, group=1, seed=1, iters=0)
    for g in range(cb.shape[0]):
        pts = W[:, g * d:(g + 1) * d].view(np.uint16).copy()
        pts[pts == 0x8000] = 0
        m = len({tuple(p) for p in pts})
        assert 256 < m < C
        c = cb[g].view(np.uint16)
        assert all(np.array_equal(c[k], c[0]) for k in range(m, C))
        assert int(idx[g].max()) < m
        at0 = np.all(pts == c[0], axis=1)
        assert at0.any() and np.all(idx[g][at0] == 0)


def test_product_brute_force_wide(oracle_lib):
    d, C, group, F_out, F_in = 2, 777, 2, 4, 16
    cb, idx = synth.random_layer(F_out, F_in, d, C, group=group, seed=3, std=1.0)
    assert idx.dtype == np.uint16 and int(idx.max()) > 255
    x = synth.activation(2, F_in, seed=4)
    y = oracle_lib.gemv(cb, idx, x, group=group)
    N_ss = F_in // d
    for b in range(2):
        for j in range(F_out):
            terms = [Fraction(float(cb[ss // group, int(idx[ss, j]), e])) * Fraction(float(x[b, ss * d + e]))
                     for ss in range(N_ss) for e in range(d)]
            exact = sum(terms, Fraction(0))
            bound = F_in * 2.0 ** -53 * float(sum(abs(t) for t in terms))
            assert abs(y[b, j] - float(exact)) <= bound + 1e-300


def test_fixed_point_conditions_wide(oracle_lib):
    W = synth.weight(600, 4, seed=21)
    d, C, group = 2, 300, 2
    cent, asg, ran = oracle_lib.lloyd_fp32(W, d, C, group, seed=2, iters=400, g=0)
    assert ran < 400, "expected convergence"
    pts = np.concatenate([W[:, s * d:(s + 1) * d] for s in range(group)]).astype(np.float64)
    assert asg.max() > 255
    for k in range(C):
        members = pts[asg == k]
        if len(members) == 0:
            continue
        for e in range(d):
            exact = sum(Fraction(float(v)) for v in members[:, e]) / len(members)
            assert abs(float(exact) - float(cent[k, e])) <= 2.0 ** -23 * max(abs(float(exact)), 2.0 ** -126) * 2
    D = ((pts[:, None, :] - cent[None].astype(np.float64)) ** 2).sum(-1)
    chosen = D[np.arange(len(pts)), asg]
    assert np.all(chosen <= D.min(1) * (1 + 1e-6) + 1e-30)


def test_wide_validation(oracle_lib):
    lib = oracle_lib.lib()
    assert lib.fasq_ref_validate16(4096, 8, 2, 1024, 1) == 0
    assert lib.fasq_ref_validate16(4096, 8, 2, 1025, 1) == -6
    assert lib.fasq_ref_validate(4096, 8, 2, 257, 1) == -6
    W = synth.weight(64, 4, seed=0)
    with pytest.raises(oracle_lib.OracleError) as e:
        oracle_lib.pack(W, d=2, C=1025)
    assert e.value.code == -6
