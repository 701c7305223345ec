"""Pins of the oracle's packing variants (NEXT-4; not GPU): exact-integer
k-means++ initialisation (reading R17) and empty-cluster
reseeding from the farthest point (reading R18).

* k-means++ keeps the saturation exactness (C >= distinct sub-vectors ->
  W_hat == W bitwise): D^2 sampling never picks a point at distance 0.
* The first centre is point splitmix64(seed ^ (g+1) * golden) % n (the
  generator is pinned against its published outputs elsewhere).
* D^2 sampling: over many seeds, the frequency of every (first, second)
  centre pair of a 3-point set matches the exact k-means++ probability
  (1/n) * D^2(i, j) / sum_k D^2(i, k) (a binomial 4-sigma band).
* Reseeding: whenever the fp16 codebook entries are distinct and the
  codebook has >= C distinct points, every entry ends up used by some index
  (a reseeded centre is a data point, nearest to itself), while with the
  plain rule a seed search finds an unused entry.
"""
import numpy as np
import pytest

import oracle
import synth


def test_kmeanspp_keeps_saturation_exactness():
    for (d, C, nd, seed) in [(2, 16, 16, 0), (2, 64, 40, 1), (4, 32, 9, 2), (1, 8, 8, 3)]:
        W = synth.structured_weight(96, 64, d, nd, seed=seed)
        cb, idx, _ = oracle.pack(W, d=d, C=C, group=1, seed=seed, iters=25, init=1)
        What = oracle.reconstruct(cb, idx, 64)
        assert np.array_equal(What.view(np.uint16), W.view(np.uint16)), (d, C, nd)


def test_kmeanspp_first_centre_is_seeded_uniform_point():
    W = synth.weight(50, 8, seed=7)          # d = 2: 4 codebooks of 50 points
    golden = 0x9E3779B97F4A7C15
    for seed in (0, 1, 12345):
        cb, _, _ = oracle.pack(W, d=2, C=1, group=1, seed=seed, iters=0, init=1)
        for g in range(4):
            st = (seed ^ ((g + 1) * golden)) & (2**64 - 1)
            t0 = int(oracle.splitmix64(st, 1)[0]) % 50
            assert np.array_equal(cb[g, 0].view(np.uint16), W[t0, 2 * g:2 * g + 2].view(np.uint16)), (seed, g)


def test_kmeanspp_d2_sampling_distribution():
    pts = np.array([0.0, 1.0, 3.0], np.float16)
    W = pts.reshape(3, 1)                    # d = 1: one codebook of 3 points
    N = 3000
    counts = {}
    for seed in range(N):
        cb, _, _ = oracle.pack(W, d=1, C=2, group=1, seed=seed, iters=0, init=1)
        pair = (float(cb[0, 0, 0]), float(cb[0, 1, 0]))
        counts[pair] = counts.get(pair, 0) + 1
    vals = [0.0, 1.0, 3.0]
    for i in vals:
        tot = sum((i - k) ** 2 for k in vals)
        for j in vals:
            if j == i:
                assert (i, j) not in counts          # never a point at distance 0
                continue
            p = (1.0 / 3.0) * (i - j) ** 2 / tot
            got = counts.get((i, j), 0)
            sd = np.sqrt(N * p * (1 - p))
            assert abs(got - N * p) <= 4 * sd + 1, ((i, j), got, N * p)


def _used_all(cb, idx, C):
    """True if every codebook with distinct fp16 entries uses all C of them;
    None if no codebook has distinct entries (the claim needs them)."""
    ok, any_distinct = True, False
    for g in range(cb.shape[0]):
        ent = cb[g].view(np.uint16).reshape(C, -1)
        if len({tuple(r) for r in ent}) < C:
            continue
        any_distinct = True
        ok &= len(set(idx[g].tolist())) == C
    return ok if any_distinct else None


def _case(trial):
    """Seeded 2-D point sets (d = 2, one codebook of n points, two outliers)
    -- the seed search that found empty clusters under the plain rule."""
    rng = np.random.default_rng(1)
    for t in range(trial + 1):
        n = int(rng.integers(10, 30))
        C = int(rng.integers(4, 10))
        pts = rng.normal(0, 1, size=(n, 2))
        pts[rng.integers(0, n, size=2)] *= 8
    return pts.astype(np.float16).reshape(n, 2), C


def test_reseed_leaves_no_unused_entry():
    plain_unused = 0
    for trial in range(0, 300, 1):
        W, C = _case(trial) if trial in (124, 263) or trial % 10 == 0 else (None, None)
        if W is None:
            continue
        for init in (0, 1):
            cb1, idx1, _ = oracle.pack(W, d=2, C=C, group=1, seed=trial, iters=25, init=init, empty=1)
            assert _used_all(cb1, idx1, C) is not False, (trial, init)
            cb0, idx0, _ = oracle.pack(W, d=2, C=C, group=1, seed=trial, iters=25, init=init, empty=0)
            plain_unused += _used_all(cb0, idx0, C) is False
    assert plain_unused >= 2, "no empty cluster under the plain rule: the pin would be vacuous"


def test_variant_argument_errors():
    W = synth.weight(8, 8, seed=0)
    with pytest.raises(oracle.OracleError):
        oracle.pack(W, d=2, C=4, init=2)
    with pytest.raises(oracle.OracleError):
        oracle.pack(W, d=2, C=4, empty=5)
