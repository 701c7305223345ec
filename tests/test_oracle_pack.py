"""Pins of the oracle's pack (Alg. 1) -- not GPU.

The paper prints no codebooks or indices, so the pack is pinned by what the
mathematics of k-means and the paper's own claims fix:
  * SPEC S:76 worked example ({0,1,10,11}, k=2 -> {0.5,10.5});
  * exactness at saturation (north_star): C >= #distinct
    sub-vectors per codebook  =>  W_hat == W bitwise;
  * C = 1: the centroid is the mean, checked against the EXACT rational mean
    (fractions) to within one fp16 rounding;
  * Lloyd fixed point at convergence: every centroid equals the exact mean of
    its cluster (to fp32 rounding) and every point sits at its nearest
    centroid (fp64 distances);
  * optimality bounds: WCSS >= the exhaustive optimum on tiny inputs and >=
    the textbook O(k n^2) 1-D dynamic-programming optimum for d = 1;
  * WCSS non-increasing over Lloyd iterations; thread-count determinism;
  * the stored indices are nearest in the stored fp16 codebook.
"""
import itertools
from fractions import Fraction

import numpy as np
import pytest

import synth


def _wcss(points, cent, asg):
    p = np.asarray(points, np.float64)
    c = np.asarray(cent, np.float64)
    return float(((p - c[asg]) ** 2).sum())


def _points_of(W, d, group, g):
    """Reading R1: point t = (ss - g*group)*F_out + j is W[j, ss*d:(ss+1)*d]."""
    F_out = W.shape[0]
    rows = []
    for s in range(group):
        ss = g * group + s
        rows.append(W[:, ss * d:(ss + 1) * d])
    return np.concatenate(rows, 0).astype(np.float64)


def test_worked_example(oracle_lib, pins):
    ex = pins["kmeans_worked_example"]
    W = np.array(ex["points"], np.float16)[:, None]      # F_out=4 points, F_in=1, d=1
    for seed in range(16):
        cb, idx, its = oracle_lib.pack(W, d=1, C=ex["k"], group=1, seed=seed)
        cents = sorted(float(v) for v in cb[0, :, 0])
        assert cents == ex["centroids"]
        part = sorted(sorted(np.nonzero(idx[0] == k)[0].tolist()) for k in range(2))
        assert part == ex["partition"]


@pytest.mark.parametrize("d,C,group,n_distinct", [(1, 8, 1, 8), (2, 16, 1, 9), (4, 32, 2, 32),
                                                   (8, 4, 1, 3), (2, 256, 4, 200), (4, 256, 128, 256)])
def test_saturation_exact(oracle_lib, d, C, group, n_distinct):
    F_out, F_in = 64, 32 * d * (1 if group <= 4 else 4)
    if (F_in // d) % group:
        F_in = group * d
    W = synth.structured_weight(F_out, F_in, d, n_distinct, group=group, seed=d * 100 + C)
    cb, idx, _ = oracle_lib.pack(W, d=d, C=C, group=group, seed=3)
    What = oracle_lib.reconstruct(cb, idx, F_in, group=group)
    assert np.array_equal(What.view(np.uint16), W.view(np.uint16))


def test_saturation_group1_config1(oracle_lib):
    """configs[0] shape with group=1: 256 points per subspace = C -> exact."""
    W = synth.weight(256, 512, seed=0)
    cb, idx, _ = oracle_lib.pack(W, d=4, C=256, group=1, seed=0)
    What = oracle_lib.reconstruct(cb, idx, 512, group=1)
    Wc = W.view(np.uint16).copy()
    Wc[Wc == 0x8000] = 0                               # reading R2 (-0 -> +0)
    assert np.array_equal(What.view(np.uint16), Wc)


def test_C1_is_exact_mean(oracle_lib):
    W = synth.weight(300, 24, seed=5)
    d, group = 2, 3
    cb, idx, _ = oracle_lib.pack(W, d=d, C=1, group=group, seed=0, iters=5)
    assert np.all(idx == 0)
    for g in range(cb.shape[0]):
        pts = _points_of(W, d, group, g)
        for e in range(d):
            exact = sum(Fraction(float(v)) for v in pts[:, e]) / len(pts)
            got = Fraction(float(cb[g, 0, e]))
            # fp16 spacing near the mean bounds one rounding
            ulp = Fraction(float(np.spacing(np.float16(float(exact)))))
            assert abs(got - exact) <= ulp, (g, e, float(got), float(exact))


def test_fixed_point_conditions(oracle_lib):
    """At convergence Lloyd is a fixed point: centroid = exact cluster mean
    (to fp32 rounding), point -> nearest centroid (fp64, tie slack)."""
    W = synth.weight(200, 8, seed=11)
    d, C, group = 2, 6, 4
    for g in range(1):
        cent, asg, ran = oracle_lib.lloyd_fp32(W, d, C, group, seed=1, iters=200, g=g)
        assert ran < 200, "expected convergence"
        pts = _points_of(W, d, group, g)
        for k in range(C):
            members = pts[asg == k]
            if len(members) == 0:
                continue
            for e in range(d):
                exact = sum(Fraction(float(v)) for v in members[:, e]) / len(members)
                rel = abs(float(exact) - float(cent[k, e]))
                assert rel <= 2.0 ** -23 * max(abs(float(exact)), 2.0 ** -126) * 2
        D = ((pts[:, None, :] - cent[None].astype(np.float64)) ** 2).sum(-1)
        best = D.min(1)
        chosen = D[np.arange(len(pts)), asg]
        assert np.all(chosen <= best * (1 + 1e-6) + 1e-30)


def _brute_wcss(pts, k):
    best = np.inf
    n = len(pts)
    for lab in itertools.product(range(k), repeat=n):
        lab = np.array(lab)
        tot = 0.0
        for c in range(k):
            m = pts[lab == c]
            if len(m):
                tot += ((m - m.mean(0)) ** 2).sum()
        best = min(best, tot)
    return best


@pytest.mark.parametrize("seed", range(6))
def test_brute_force_lower_bound(oracle_lib, seed):
    g = np.random.Generator(np.random.PCG64(seed))
    n, d, k = 8, 2, 3
    W = g.normal(0, 1, size=(n, d)).astype(np.float16)
    cent, asg, _ = oracle_lib.lloyd_fp32(W, d, k, 1, seed=seed, iters=50, g=0)
    pts = W.astype(np.float64)
    ours = _wcss(pts, cent, asg)
    opt = _brute_wcss(pts, k)
    assert ours >= opt * (1 - 1e-6)


def _dp_1d_opt(x, k):
    """Textbook optimal 1-D k-means (Ckmeans.1d.dp style O(k n^2) DP)."""
    x = np.sort(np.asarray(x, np.float64))
    n = len(x)
    ps = np.concatenate([[0.0], np.cumsum(x)])
    ps2 = np.concatenate([[0.0], np.cumsum(x * x)])

    def sse(i, j):  # x[i..j] inclusive
        m = j - i + 1
        s = ps[j + 1] - ps[i]
        return (ps2[j + 1] - ps2[i]) - s * s / m

    INF = np.inf
    D = np.full((k + 1, n + 1), INF)
    D[0, 0] = 0.0
    for q in range(1, k + 1):
        for j in range(1, n + 1):
            D[q, j] = min((D[q - 1, i] + sse(i, j - 1) for i in range(q - 1, j)), default=INF)
    return D[k, n]


@pytest.mark.parametrize("seed", range(4))
def test_1d_dp_lower_bound_and_separated_equality(oracle_lib, seed):
    g = np.random.Generator(np.random.PCG64(100 + seed))
    x = g.normal(0, 1, size=40).astype(np.float16)
    W = x[:, None]
    for k in (2, 3, 5):
        cent, asg, _ = oracle_lib.lloyd_fp32(W, 1, k, 1, seed=seed, iters=100, g=0)
        ours = _wcss(W.astype(np.float64), cent, asg)
        assert ours >= _dp_1d_opt(x, k) * (1 - 1e-6)
    # well separated clusters whose count equals C: distinct-sample init can
    # still pick two seeds in one cluster, so equality is required only when
    # the init covered every cluster (then Lloyd must reach the optimum)
    centers = np.array([-40.0, -10.0, 15.0, 60.0])
    x = (centers[g.integers(0, 4, 60)] + g.normal(0, 0.5, 60)).astype(np.float16)
    cent, asg, _ = oracle_lib.lloyd_fp32(x[:, None], 1, 4, 1, seed=seed, iters=100, g=0)
    hit = {int(np.argmin(abs(centers - c))) for c in cent[:, 0]}
    if len(hit) == 4:
        ours = _wcss(x[:, None].astype(np.float64), cent, asg)
        assert ours == pytest.approx(_dp_1d_opt(x, 4), rel=1e-6)


def test_wcss_non_increasing(oracle_lib):
    W = synth.weight(512, 16, seed=3)
    d, C, group = 2, 16, 8
    pts = _points_of(W, d, group, 0)
    prev = np.inf
    for T in range(1, 15):
        cent, asg, _ = oracle_lib.lloyd_fp32(W, d, C, group, seed=9, iters=T, g=0)
        w = _wcss(pts, cent, asg)
        assert w <= prev * (1 + 1e-6)
        prev = w


def test_indices_nearest_in_stored_codebook(oracle_lib):
    W = synth.weight(128, 64, seed=4)
    d, C, group = 2, 16, 2
    cb, idx, _ = oracle_lib.pack(W, d=d, C=C, group=group, seed=2, iters=10)
    N_ss = 64 // d
    for ss in range(N_ss):
        c = cb[ss // group].astype(np.float64)
        p = W[:, ss * d:(ss + 1) * d].astype(np.float64)
        D = ((p[:, None, :] - c[None]) ** 2).sum(-1)
        chosen = D[np.arange(len(p)), idx[ss]]
        assert np.all(chosen <= D.min(1) * (1 + 1e-6) + 1e-30)


def test_init_is_seeded_distinct_sample(oracle_lib):
    """iters=0: codebook = init.  Rows < m are distinct members of the point
    set, rows >= m copy row 0 (reading R3), and the draw follows the partial
    Fisher-Yates over the sorted unique keys with the pinned splitmix64."""
    W = synth.structured_weight(64, 8, 2, 5, group=1, seed=1)   # 5 distinct per subspace
    C = 8
    cb, idx, its = oracle_lib.pack(W, d=2, C=C, group=1, seed=42, iters=0)
    assert np.all(its == 0)
    for ss in range(4):
        keys = W.view(np.uint16)[:, 2 * ss:2 * ss + 2]
        U = np.unique(keys, axis=0)                      # sorted, element 0 most significant
        m = min(C, len(U))
        st_seed = 42 ^ (((ss + 1) * 0x9E3779B97F4A7C15) & (2**64 - 1))
        draws = oracle_lib.splitmix64(st_seed, m)
        order = list(range(len(U)))
        for i in range(m):
            j = i + draws[i] % (len(U) - i)
            order[i], order[j] = order[j], order[i]
        want = np.array([U[order[k if k < m else 0]] for k in range(C)], np.uint16)
        assert np.array_equal(cb[ss].view(np.uint16), want)


def test_thread_count_determinism(oracle_lib):
    W = synth.weight(300, 64, seed=8)
    outs = []
    for t in (1, 2, 8):
        oracle_lib.set_threads(t)
        outs.append(oracle_lib.pack(W, d=2, C=32, group=1, seed=5, iters=8))
    oracle_lib.set_threads(0)
    for o in outs[1:]:
        assert np.array_equal(o[0].view(np.uint16), outs[0][0].view(np.uint16))
        assert np.array_equal(o[1], outs[0][1])
        assert np.array_equal(o[2], outs[0][2])


def test_cb_range_matches_full(oracle_lib):
    W = synth.weight(96, 32, seed=2)
    full = oracle_lib.pack(W, d=2, C=8, group=2, seed=1)
    part = oracle_lib.pack(W, d=2, C=8, group=2, seed=1, cb_range=(3, 6))
    assert np.array_equal(part[0][3:6].view(np.uint16), full[0][3:6].view(np.uint16))
    assert np.array_equal(part[1][6:12], full[1][6:12])


def test_negative_zero_canonicalised(oracle_lib):
    W = np.zeros((16, 4), np.float16)
    W[::2] = -0.0
    cb, idx, _ = oracle_lib.pack(W, d=2, C=1, group=1)
    assert np.all(cb.view(np.uint16) == 0)


@pytest.mark.parametrize("shape,d,C,group,code", [
    ((8, 6), 4, 2, 1, -2),       # F_in % d
    ((8, 8), 2, 2, 3, -2),       # N_ss % group
    ((4, 8), 2, 5, 1, -3),       # C > group*F_out (ClusterOverflow)
    ((300, 8), 2, 257, 1, -6),   # C > 256 (uint8 indices)
    ((8, 9), 3, 2, 1, -6),       # d not in {1,2,4,8}
])
def test_validation_errors(oracle_lib, shape, d, C, group, code):
    assert oracle_lib.validate(shape[0], shape[1], d, C, group) == code


def test_nonfinite_rejected(oracle_lib):
    W = np.zeros((8, 4), np.float16)
    W[3, 1] = np.inf
    with pytest.raises(oracle_lib.OracleError) as e:
        oracle_lib.pack(W, d=2, C=2)
    assert e.value.code == -4


def test_tie_rule_lowest_k_duplicated_centroids(oracle_lib):
    """Reading R5 / SPEC S:145: an exact distance tie goes to the LOWEST k.
    With fewer distinct sub-vectors than C, init slots >= m copy slot 0
    (reading R3), so every point equal to codebook[0] is at distance 0 from
    slots 0 and m..C-1 at once: the lowest-k rule must pick 0 and no index
    may ever point at a duplicate slot (a '<=' slip would pick C-1)."""
    d, C, n_distinct = 2, 16, 5
    W = synth.structured_weight(64, 8 * d, d, n_distinct, group=1, seed=77)
    cb, idx, _ = oracle_lib.pack(W, d=d, C=C, group=1, seed=3, iters=0)
    for g in range(cb.shape[0]):
        pts = _points_of(W, d, 1, g)
        m = len({tuple(p) for p in pts})
        assert m < C
        c = cb[g].astype(np.float64)
        assert all(np.array_equal(c[k], c[0]) for k in range(m, C))   # slots >= m duplicate slot 0
        assert idx[g].max() < m
        at0 = np.all(pts == c[0], axis=1)
        assert at0.any() and np.all(idx[g][at0] == 0)


@pytest.mark.parametrize("seed", range(6))
def test_tie_rule_lowest_k_equidistant_point(oracle_lib, seed):
    """Exact equidistance between two DISTINCT centroids: 1-D points
    {0, 1, 2} (x64 rows), C = 2, no Lloyd round (iters = 0, the codebook is
    the seeded init).  Whenever the init picked {0, 2}, point 1 lies at
    distance exactly 1 from both and must take the lower of their two slots."""
    W = np.repeat(np.array([0.0, 1.0, 2.0], np.float16), 64)[:, None]
    cb, idx, _ = oracle_lib.pack(W, d=1, C=2, group=1, seed=seed, iters=0)
    cents = [float(v) for v in cb[0, :, 0]]
    one = idx[0][W[:, 0] == 1.0]
    if sorted(cents) == [0.0, 2.0]:
        assert np.all(one == 0)
    else:   # 1 is itself a centroid: exact match wins
        assert np.all(one == cents.index(1.0))


def test_tie_rule_case_occurs():
    """Guard for the parametrised test above: some seed in range(6) must hit
    the {0, 2} init (otherwise the tie branch is untested)."""
    import oracle
    W = np.repeat(np.array([0.0, 1.0, 2.0], np.float16), 64)[:, None]
    hits = [s for s in range(6)
            if sorted(float(v) for v in oracle.pack(W, d=1, C=2, group=1, seed=s, iters=0)[0][0, :, 0]) == [0.0, 2.0]]
    assert hits, "no seed produced the equidistant init"
