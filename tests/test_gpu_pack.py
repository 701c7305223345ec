"""GPU pack (fasq_pack) vs the CPU oracle: identical codebook and index BYTES
for the same (d, C, group, seed, iters) -- BASELINE.json north_star."""
import numpy as np
import pytest
import torch

import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def F():
    import paper_2605_04084_b200 as F
    return F


def _gpu_pack(F, W, d, C, group, seed, iters):
    L = F.pack(torch.from_numpy(W).cuda(), d=d, C=C, group=group, seed=seed, iters=iters)
    cb, idx = L.export()
    torch.cuda.synchronize()
    return cb.cpu().numpy(), idx.cpu().numpy(), L


def _assert_same(a_cb, a_idx, b_cb, b_idx):
    assert np.array_equal(a_cb.view(np.uint16), b_cb.view(np.uint16)), "codebooks differ"
    assert np.array_equal(a_idx, b_idx), "indices differ"


CASES = [
    # F_out, F_in, d, C, group, seed, iters
    (64, 32, 2, 16, 1, 0, 25),
    (100, 48, 1, 8, 1, 1, 25),
    (96, 64, 4, 32, 2, 2, 25),
    (80, 64, 8, 16, 1, 3, 10),
    (300, 128, 2, 256, 1, 4, 25),       # C > distinct? (300 points, 256 clusters)
    (256, 64, 2, 1, 1, 5, 5),           # C = 1
    (200, 32, 2, 7, 16, 6, 25),         # one shared codebook
    (513, 96, 2, 64, 3, 7, 0),          # iters = 0 (init -> finalize)
    (128, 64, 2, 255, 8, 8, 3),
]


@pytest.mark.parametrize("F_out,F_in,d,C,group,seed,iters", CASES)
def test_pack_bit_exact_small(F, oracle_lib, F_out, F_in, d, C, group, seed, iters):
    W = synth.weight(F_out, F_in, seed=seed)
    ref_cb, ref_idx, _ = oracle_lib.pack(W, d=d, C=C, group=group, seed=seed, iters=iters)
    cb, idx, _ = _gpu_pack(F, W, d, C, group, seed, iters)
    _assert_same(cb, idx, ref_cb, ref_idx)


def test_pack_config1(F, oracle_lib):
    """configs[0]: 256x512, d=4, C=256, one codebook (group=128), T=25."""
    W = synth.weight(256, 512, seed=0)
    ref_cb, ref_idx, _ = oracle_lib.pack(W, d=4, C=256, group=128, seed=0, iters=25)
    cb, idx, _ = _gpu_pack(F, W, 4, 256, 128, 0, 25)
    _assert_same(cb, idx, ref_cb, ref_idx)


def test_pack_saturated_and_negzero(F, oracle_lib):
    W = synth.structured_weight(512, 64, 2, 11, group=1, seed=3)
    W[::7, ::3] = np.float16(-0.0)
    ref_cb, ref_idx, _ = oracle_lib.pack(W, d=2, C=16, group=1, seed=9)
    cb, idx, _ = _gpu_pack(F, W, 2, 16, 1, 9, 25)
    _assert_same(cb, idx, ref_cb, ref_idx)
    assert not np.any(cb.view(np.uint16) == 0x8000)


@pytest.mark.parametrize("F_out,F_in,C", [(4096, 4096, 256), (14336, 4096, 128)])
def test_pack_llama_sampled_codebooks(F, oracle_lib, F_out, F_in, C):
    """Full Llama layer packed on the GPU; the oracle packs a sample of
    codebooks (each is an independent k-means problem, Alg. 1)."""
    W = synth.weight(F_out, F_in, seed=F_out)
    cb, idx, _ = _gpu_pack(F, W, 2, C, 1, 17, 25)
    N_cb = F_in // 2
    for g0 in (0, N_cb // 2 + 3, N_cb - 2):
        ref_cb, ref_idx, _ = oracle_lib.pack(W, d=2, C=C, group=1, seed=17, iters=25, cb_range=(g0, g0 + 2))
        _assert_same(cb[g0:g0 + 2], idx[g0:g0 + 2], ref_cb[g0:g0 + 2], ref_idx[g0:g0 + 2])


def test_pack_then_gemv(F, oracle_lib):
    from fasq_testutil import parity_ok
    W = synth.weight(1024, 1024, seed=4)
    cb, idx, L = _gpu_pack(F, W, 2, 64, 1, 0, 8)
    x = synth.activation(1, 1024, seed=5)
    y = F.gemv(L, torch.from_numpy(x).cuda()).cpu().numpy()
    ok, info = parity_ok(y, oracle_lib.gemv(cb, idx, x), x, 1024)
    assert ok, info


def test_pack_errors(F):
    W = synth.weight(64, 32, seed=0)
    W[5, 5] = np.inf
    with pytest.raises(F.FasqError) as e:
        F.pack(torch.from_numpy(W).cuda(), d=2, C=4)
    assert e.value.code == -4
    with pytest.raises(F.FasqError) as e:
        F.pack(torch.from_numpy(synth.weight(4, 8)).cuda(), d=2, C=5)
    assert e.value.code == -3


VARIANT_CASES = [
    # F_out, F_in, d, C, group, seed, iters
    (64, 32, 2, 16, 1, 0, 25),
    (100, 48, 1, 8, 1, 1, 25),
    (96, 64, 4, 32, 2, 2, 25),
    (80, 64, 8, 16, 1, 3, 10),
    (300, 128, 2, 256, 1, 4, 25),
    (200, 32, 2, 7, 16, 6, 25),
    (513, 96, 2, 64, 3, 7, 0),
    (1024, 256, 2, 256, 1, 9, 25),
]


@pytest.mark.parametrize("init,empty", [(1, 0), (0, 1), (1, 1)])
@pytest.mark.parametrize("F_out,F_in,d,C,group,seed,iters", VARIANT_CASES)
def test_pack_variants_bit_exact(F, oracle_lib, F_out, F_in, d, C, group, seed, iters, init, empty):
    """NEXT-4 packing variants (SPEC S:138 k-means++, S:140 reseed; readings
    R17/R18): the GPU's bytes equal the oracle's."""
    W = synth.weight(F_out, F_in, seed=seed)
    ref_cb, ref_idx, _ = oracle_lib.pack(W, d=d, C=C, group=group, seed=seed, iters=iters, init=init, empty=empty)
    L = F.pack(torch.from_numpy(W).cuda(), d=d, C=C, group=group, seed=seed, iters=iters, init=init, empty=empty)
    cb, idx = L.export()
    torch.cuda.synchronize()
    _assert_same(cb.cpu().numpy(), idx.cpu().numpy(), ref_cb, ref_idx)
    L.free()


def test_pack_variant_arguments(F):
    W = torch.from_numpy(synth.weight(64, 32, seed=0)).cuda()
    for kw in ({"init": 2}, {"empty": -1}):
        with pytest.raises(F.FasqError):
            F.pack(W, d=2, C=8, **kw)


def test_dedup_distinct_centroids_and_lowest_copy(F, oracle_lib):
    """P:241 dedup: the layer reports the distinct fp16 centroids per codebook
    (counted independently here with numpy), and indices only ever reference
    the FIRST copy of a repeated centroid (ties -> lowest k), so dropping the
    later copies needs no index rewrite."""
    W = synth.structured_weight(128, 64, 2, 5, seed=3)     # <= 5 distinct sub-vectors per codebook, C = 16
    cb, idx, L = _gpu_pack(F, W, 2, 16, 1, 0, 25)
    bits = cb.view(np.uint16)
    want = sum(len({tuple(r) for r in bits[g]}) for g in range(bits.shape[0]))
    assert L.distinct_centroids() == want
    for g in range(bits.shape[0]):
        first = {}
        for k in range(16):
            first.setdefault(tuple(bits[g, k]), k)
        for k in set(idx[g].tolist()):
            assert first[tuple(bits[g, k])] == k, (g, k)
    L.free()
