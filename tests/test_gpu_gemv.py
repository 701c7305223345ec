"""GPU parity of the decode GEMV (C-ABI fasq_gemv) against the fp64 oracle.

Tolerance (BASELINE.json north_star): rel-L2 <= 1e-3 and
max-abs <= 5e-3 * ||x||_inf * sqrt(F_in).
"""
import numpy as np
import pytest
import torch

import synth
from fasq_testutil import parity_ok

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def F():
    import paper_2605_04084_b200 as F
    return F


def _import(F, cb, idx, F_in, group):
    return F.import_layer(torch.from_numpy(cb).cuda(), torch.from_numpy(idx).cuda(), F_in, group)


def _gemv(F, L, x, out_dtype=torch.float32, flags=0):
    y = F.gemv(L, torch.from_numpy(x).cuda(), out_dtype=out_dtype, flags=flags)
    torch.cuda.synchronize()
    return y.float().cpu().numpy().astype(np.float64)


SMALL = [
    # F_out, F_in, d, C, group, B
    (1000, 640, 2, 256, 1, 1),     # ragged rows (pad to 1024), 10 groups
    (3000, 1000, 2, 128, 1, 1),    # 3 row tiles, ragged last group (N_ss=500)
    (2048, 2048, 2, 256, 1, 1),
    (777, 96, 1, 16, 1, 1),        # d=1 (entries padded to 4 B)
    (1500, 1024, 4, 256, 2, 1),    # d=4, shared codebooks
    (600, 1024, 8, 64, 1, 1),      # d=8
    (1024, 512, 2, 1, 1, 1),       # C=1
    (1024, 512, 2, 2, 4, 1),       # C=2, group=4
    (4096, 512, 2, 7, 1, 1),       # odd C
    (1000, 640, 2, 256, 1, 2),
    (1000, 640, 2, 256, 1, 3),
    (1000, 640, 2, 256, 1, 4),
    (1000, 640, 2, 256, 1, 5),
    (1000, 640, 2, 256, 1, 8),
    (1500, 1024, 4, 256, 2, 8),
    (600, 1024, 8, 64, 1, 6),
    (777, 96, 1, 16, 1, 7),
    (33, 64, 2, 4, 1, 1),          # tiny
]


@pytest.mark.parametrize("F_out,F_in,d,C,group,B", SMALL)
def test_gemv_small(F, oracle_lib, F_out, F_in, d, C, group, B):
    cb, idx = synth.random_layer(F_out, F_in, d, C, group=group, seed=F_out + F_in + d + C + B)
    x = synth.activation(B, F_in, seed=B + 3)
    L = _import(F, cb, idx, F_in, group)
    y = _gemv(F, L, x)
    y_ref = oracle_lib.gemv(cb, idx, x, group=group)
    ok, info = parity_ok(y, y_ref, x, F_in)
    assert ok, info


def test_gemv_fp16_out(F, oracle_lib):
    cb, idx = synth.random_layer(2048, 1024, 2, 256, seed=5)
    x = synth.activation(2, 1024, seed=6)
    L = _import(F, cb, idx, 1024, 1)
    y = _gemv(F, L, x, out_dtype=torch.float16)
    ok, info = parity_ok(y, oracle_lib.gemv(cb, idx, x), x, 1024)
    assert ok, info


def test_gemv_config1_oracle_packed(F, oracle_lib):
    """configs[0]: 256x512 fp16 W, d=4, C=256, one codebook (group=128)."""
    W = synth.weight(256, 512, seed=0)
    cb, idx, _ = oracle_lib.pack(W, d=4, C=256, group=128, seed=0)
    x = synth.activation(1, 512, seed=1)
    L = _import(F, cb, idx, 512, 128)
    y = _gemv(F, L, x)
    ok, info = parity_ok(y, oracle_lib.gemv(cb, idx, x, group=128), x, 512)
    assert ok, info


def test_gemv_special_inputs(F, oracle_lib):
    cb, idx = synth.random_layer(1100, 768, 2, 64, seed=9)
    L = _import(F, cb, idx, 768, 1)
    z = _gemv(F, L, np.zeros((1, 768), np.float16))
    assert np.all(z == 0)
    What = oracle_lib.reconstruct(cb, idx, 768).astype(np.float64)
    for i in (0, 1, 333, 767):
        e = np.zeros((1, 768), np.float16)
        e[0, i] = 1
        y = _gemv(F, L, e)
        assert np.array_equal(y[0], What[:, i]), i       # single exact term


def test_gemv_deterministic(F):
    cb, idx = synth.random_layer(4096, 4096, 2, 256, seed=2)
    x = synth.activation(1, 4096, seed=3)
    L = _import(F, cb, idx, 4096, 1)
    a = _gemv(F, L, x)
    b = _gemv(F, L, x)
    assert np.array_equal(a, b)


def test_import_export_roundtrip(F):
    for (F_out, F_in, d, C, group) in [(1000, 640, 2, 256, 1), (600, 1024, 8, 64, 1), (777, 96, 1, 16, 3)]:
        cb, idx = synth.random_layer(F_out, F_in, d, C, group=group, seed=1)
        L = _import(F, cb, idx, F_in, group)
        cb2, idx2 = L.export()
        torch.cuda.synchronize()
        assert np.array_equal(cb2.cpu().numpy().view(np.uint16), cb.view(np.uint16))
        assert np.array_equal(idx2.cpu().numpy(), idx)


LLAMA = [(4096, 4096), (1024, 4096), (14336, 4096), (4096, 14336)]


@pytest.mark.parametrize("F_out,F_in", LLAMA)
@pytest.mark.parametrize("C", [256, 128])
def test_gemv_llama_shapes_sampled(F, oracle_lib, F_out, F_in, C):
    """Full-size layers in the bench launch configuration, checked on three
    contiguous windows of rows that the oracle computes one by one."""
    cb, idx = synth.random_layer(F_out, F_in, 2, C, seed=F_out * 7 + F_in + C)
    x = synth.activation(1, F_in, seed=11)
    L = _import(F, cb, idx, F_in, 1)
    y = _gemv(F, L, x, flags=F.FLAG_PDL)
    for j0 in (0, F_out // 2 - 37, F_out - 96):
        ref = oracle_lib.gemv(cb, idx, x, rows=(j0, j0 + 96))
        ok, info = parity_ok(y[:, j0:j0 + 96], ref, x, F_in)
        assert ok, (j0, info)


def test_gemv_batch8_llama(F, oracle_lib):
    cb, idx = synth.random_layer(4096, 4096, 2, 256, seed=4)
    x = synth.activation(8, 4096, seed=12)
    L = _import(F, cb, idx, 4096, 1)
    y = _gemv(F, L, x)
    ref = oracle_lib.gemv(cb, idx, x, rows=(1000, 1200))
    ok, info = parity_ok(y[:, 1000:1200], ref, x, 4096)
    assert ok, info


def test_shard_rows(F, oracle_lib):
    cb, idx = synth.random_layer(2048, 1024, 2, 256, seed=8)
    x = synth.activation(1, 1024, seed=2)
    L = _import(F, cb, idx, 1024, 1)
    ref = oracle_lib.gemv(cb, idx, x)
    for world in (2, 4, 8):
        parts = []
        for r in range(world):
            S = L.shard_rows(r, world)
            assert S.info["row_offset"] == r * 2048 // world
            c2, i2 = S.export()
            torch.cuda.synchronize()
            assert np.array_equal(i2.cpu().numpy(), idx[:, r * 2048 // world:(r + 1) * 2048 // world])
            parts.append(_gemv(F, S, x))
        y = np.concatenate(parts, axis=1)
        ok, info = parity_ok(y, ref, x, 1024)
        assert ok, (world, info)


def test_gemv_host_e2e(F, oracle_lib):
    cb, idx = synth.random_layer(4096, 4096, 2, 256, seed=21)
    x = synth.activation(1, 4096, seed=22)
    L = _import(F, cb, idx, 4096, 1)
    xh = torch.from_numpy(x).pin_memory()
    yh = torch.empty((1, 4096), dtype=torch.float32).pin_memory()
    F.gemv_host(L, xh, yh)
    ref = oracle_lib.gemv(cb, idx, x, rows=(0, 512))
    ok, info = parity_ok(yh.numpy()[:, :512], ref, x, 4096)
    assert ok, info


def test_errors(F):
    cb, idx = synth.random_layer(64, 64, 2, 16, seed=1)
    L = _import(F, cb, idx, 64, 1)
    with pytest.raises(F.FasqError):   # B > 128 runs fasq_gemm: flags are not supported there
        F.gemv(L, torch.zeros((129, 64), dtype=torch.float16, device="cuda"), flags=F.FLAG_PDL)
    with pytest.raises(F.FasqError):
        F.gemv(L, torch.zeros((1, 32), dtype=torch.float16, device="cuda"))   # shape
    with pytest.raises(F.FasqError) as e:
        F.import_layer(torch.from_numpy(cb).cuda(), torch.from_numpy(idx).cuda(), 63, 1)
    assert e.value.code == -2


def test_gemv_grouped_matches_separate(F, oracle_lib):
    shapes = [(4096, 1024), (1024, 1024), (1024, 1024)]
    x = synth.activation(1, 1024, seed=31)
    layers, refs = [], []
    for i, (fo, fi) in enumerate(shapes):
        cb, idx = synth.random_layer(fo, fi, 2, 256, seed=40 + i)
        layers.append(_import(F, cb, idx, fi, 1))
        refs.append(oracle_lib.gemv(cb, idx, x))
    ys = F.gemv_grouped(layers, torch.from_numpy(x).cuda(), flags=F.FLAG_PDL)
    torch.cuda.synchronize()
    for y, ref in zip(ys, refs):
        ok, info = parity_ok(y.cpu().numpy(), ref, x, 1024)
        assert ok, info
    with pytest.raises(F.FasqError):
        cb, idx = synth.random_layer(64, 512, 2, 16, seed=1)
        F.gemv_grouped([layers[0], _import(F, cb, idx, 512, 1)], torch.from_numpy(x).cuda())


def test_gemv_grouped_prefetch_hint_no_effect_on_results(F, oracle_lib):
    cb, idx = synth.random_layer(4096, 1024, 2, 256, seed=51)
    cb2, idx2 = synth.random_layer(1024, 4096, 2, 256, seed=52)
    L1 = _import(F, cb, idx, 1024, 1)
    L2 = _import(F, cb2, idx2, 4096, 1)
    x = synth.activation(1, 1024, seed=53)
    a = F.gemv_grouped([L1], torch.from_numpy(x).cuda(), next_layers=[L2], flags=F.FLAG_PDL)[0]
    b = F.gemv_grouped([L1], torch.from_numpy(x).cuda())[0]
    torch.cuda.synchronize()
    assert torch.equal(a, b)
    ok, info = parity_ok(a.cpu().numpy(), oracle_lib.gemv(cb, idx, x), x, 1024)
    assert ok, info


def test_gemv_acc_mode_and_chain(F, oracle_lib):
    """FASQ_ACC_I64 outputs (int64 fixed point, red.add) are deterministic and
    match the oracle; an ACC output fed as the next layer's x matches the
    oracle chain; the zero side job clears its range."""
    cb1, idx1 = synth.random_layer(2048, 1024, 2, 256, seed=61)
    cb2, idx2 = synth.random_layer(1024, 2048, 2, 256, seed=62)
    L1 = _import(F, cb1, idx1, 1024, 1)
    L2 = _import(F, cb2, idx2, 2048, 1)
    x = synth.activation(1, 1024, seed=63)
    xt = torch.from_numpy(x).cuda()
    junk = torch.full((1000,), 7, dtype=torch.int64, device="cuda")
    a1 = F.gemv_grouped([L1], xt, out_dtype=torch.int64, zero=junk)[0]
    a1b = F.gemv_grouped([L1], xt, out_dtype=torch.int64)[0]
    torch.cuda.synchronize()
    assert torch.equal(a1, a1b)
    assert int(junk.abs().sum()) == 0
    y1 = F.acc_convert(a1, out_dtype=torch.float32).cpu().numpy()
    ref1 = oracle_lib.gemv(cb1, idx1, x)
    ok, info = parity_ok(y1, ref1, x, 1024)
    assert ok, info
    a2 = F.gemv_grouped([L2], a1, out_dtype=torch.int64)[0]      # x = ACC input
    y2 = F.acc_convert(a2, out_dtype=torch.float32).cpu().numpy()
    x2 = F.acc_convert(a1, out_dtype=torch.float16).cpu().numpy()  # the fp16 x the kernel used
    ref2 = oracle_lib.gemv(cb2, idx2, x2)
    ok, info = parity_ok(y2, ref2, x2, 2048)
    assert ok, info


@pytest.mark.parametrize("F_out,F_in,B", [(1000, 640, 5), (1000, 640, 7), (4096, 1024, 16), (3000, 2048, 33),
                                          (14336, 4096, 8), (700, 4096, 64)])
def test_gemv_tc_batched_decode(F, oracle_lib, F_out, F_in, B):
    """The tcgen05 batched-decode kernel (gemv_tc.cu, B >= 5): ragged row tiles
    (384 rows per CTA), token tiles NT = 16 / 32 / 64 with zero-filled rows past
    B, split-K slices; fp32 and fp16 outputs, PDL, run-to-run bit identity."""
    cb, idx = synth.random_layer(F_out, F_in, 2, 256, seed=F_out + B)
    x = synth.activation(B, F_in, seed=B)
    L = _import(F, cb, idx, F_in, 1)
    rows = (0, F_out) if F_out <= 4096 else (F_out - 512, F_out)
    y = _gemv(F, L, x)
    ok, m = parity_ok(y[:, rows[0]:rows[1]], oracle_lib.gemv(cb, idx, x, rows=rows), x, F_in)
    assert ok, m
    assert np.array_equal(_gemv(F, L, x, flags=F.FLAG_PDL), y)
    yh = _gemv(F, L, x, out_dtype=torch.float16)
    ok, m = parity_ok(yh[:, rows[0]:rows[1]], oracle_lib.gemv(cb, idx, x, rows=rows), x, F_in)
    assert ok, m
