"""GPU parity of NEXT-4's dim = 0 partition (subspaces along the OUTPUT axis:
Eq. 2 first case; the layout of the paper's experiments)
through the C ABI, against the fp64 oracle (oracle.gemm_dim0):

  * import -> export is the identity on the logical [F_out/d][F_in] table;
  * the dim = 0 decode GEMV within north_star's tolerance for d = 1/2/4/8,
    B = 1..8, ragged subspace groups and column ranges, and on sampled rows of
    the full Llama-3-8B shapes;
  * the GPU dim = 0 pack is bit-identical to oracle.pack_dim0;
  * fasq_gemm (8-token GEMV slices), output dtypes, determinism, errors.
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


def _layer(F_out, F_in, d, C, group, seed):
    """dim = 0 logical layer: codebooks [N_cb][C][d], indices [F_out/d][F_in]."""
    g = synth.rng(seed)
    N_ss = F_out // d
    cb = g.normal(0.0, 1.0 / np.sqrt(F_in), size=(N_ss // group, C, d)).astype(np.float16)
    idx = g.integers(0, C, size=(N_ss, F_in), dtype=np.uint8)
    return cb, idx


def _import(F, cb, idx, F_in, group=1):
    return F.import_layer(torch.from_numpy(cb).cuda(), torch.from_numpy(idx).cuda(), F_in, group, dim0=True)


def _gemv(F, L, x, out_dtype=torch.float32):
    y = F.gemv(L, torch.from_numpy(x).cuda(), out_dtype=out_dtype)
    torch.cuda.synchronize()
    return y.float().cpu().numpy().astype(np.float64)


def test_import_export_roundtrip(F):
    cb, idx = _layer(1000, 650, 2, 256, 1, seed=1)      # N_ss = 500 (ragged group), F_in ragged to 64
    L = _import(F, cb, idx, 650)
    assert L.dim0 and L.F_out == 1000 and L.N_ss == 500
    cb2, idx2 = L.export()
    torch.cuda.synchronize()
    assert np.array_equal(cb2.cpu().numpy().view(np.uint16), cb.view(np.uint16))
    assert np.array_equal(idx2.cpu().numpy(), idx)


SMALL = [
    # F_out, F_in, d, C, group, B
    (1000, 640, 2, 256, 1, 1),
    (3000, 1000, 2, 128, 1, 1),     # ragged columns (K_pad 1024)
    (2048, 2048, 2, 256, 2, 1),
    (777, 96, 1, 16, 1, 1),
    (1500, 1024, 4, 256, 3, 1),     # N_ss = 375, group 3
    (600, 1024, 8, 64, 1, 1),
    (64, 90, 2, 16, 1, 1),          # F_in % 8 != 0: scalar x loads
    (1000, 640, 2, 256, 1, 2),
    (1000, 640, 2, 256, 1, 3),
    (1000, 640, 2, 256, 1, 4),
    (1000, 640, 2, 256, 1, 5),
    (1000, 640, 2, 256, 1, 8),
    (1500, 1024, 4, 256, 3, 8),
    (600, 1024, 8, 64, 1, 6),
    (777, 96, 1, 16, 1, 7),
]


@pytest.mark.parametrize("F_out,F_in,d,C,group,B", SMALL)
def test_dim0_gemv_small(F, oracle_lib, F_out, F_in, d, C, group, B):
    cb, idx = _layer(F_out, F_in, d, C, group, seed=F_out + F_in + d + C + B)
    x = synth.activation(B, F_in, seed=B + 11)
    L = _import(F, cb, idx, F_in, group)
    y = _gemv(F, L, x)
    y_ref = oracle_lib.gemm_dim0(cb, idx, x, group=group)
    ok, m = parity_ok(y, y_ref, x, F_in)
    assert ok, m


@pytest.mark.parametrize("F_out,F_in", [(4096, 4096), (14336, 4096), (4096, 14336), (1024, 4096)])
@pytest.mark.parametrize("B", [1, 8])
def test_dim0_llama_shapes_sampled(F, oracle_lib, F_out, F_in, B):
    cb, idx = _layer(F_out, F_in, 2, 256, 1, seed=F_out // 3 + F_in + B)
    x = synth.activation(B, F_in, seed=6)
    L = _import(F, cb, idx, F_in)
    y = _gemv(F, L, x)
    for j0 in (0, F_out // 2 + 38, F_out - 64):
        y_ref = oracle_lib.gemm_dim0(cb, idx, x, rows=(j0, j0 + 64))
        ok, m = parity_ok(y[:, j0:j0 + 64], y_ref, x, F_in)
        assert ok, (j0, m)


@pytest.mark.parametrize("out_dtype", [torch.float16, torch.int64])
def test_dim0_output_dtypes(F, oracle_lib, out_dtype):
    F_out, F_in, B = 1024, 2048, 3
    cb, idx = _layer(F_out, F_in, 2, 256, 1, seed=21)
    x = synth.activation(B, F_in, seed=22)
    L = _import(F, cb, idx, F_in)
    xd = torch.from_numpy(x).cuda()
    if out_dtype == torch.int64:
        y = torch.zeros((B, F_out), dtype=torch.int64, device="cuda")
        F.gemv_grouped([L], xd, outs=[y], out_dtype=torch.int64)
        yv = y.cpu().numpy().astype(np.float64) * 2.0 ** -32
    else:
        yv = F.gemv(L, xd, out_dtype=out_dtype).float().cpu().numpy().astype(np.float64)
    ok, m = parity_ok(yv, oracle_lib.gemm_dim0(cb, idx, x), x, F_in)
    assert ok, m


def test_dim0_deterministic(F):
    cb, idx = _layer(4096, 4096, 2, 256, 1, seed=4)
    x = synth.activation(1, 4096, seed=5)
    L = _import(F, cb, idx, 4096)
    a = _gemv(F, L, x)
    for _ in range(3):
        assert np.array_equal(_gemv(F, L, x), a)


@pytest.mark.parametrize("F_out,F_in,d,C,group", [(256, 96, 2, 16, 1), (128, 300, 2, 64, 2), (96, 200, 4, 32, 1),
                                                  (64, 512, 2, 256, 4)])
def test_gpu_pack_dim0_bit_exact(F, oracle_lib, F_out, F_in, d, C, group):
    W = synth.weight(F_out, F_in, seed=F_out + F_in)
    cb_ref, idx_ref, _ = oracle_lib.pack_dim0(W, d=d, C=C, group=group, seed=3, iters=7)
    L = F.pack(torch.from_numpy(W).cuda(), d=d, C=C, group=group, seed=3, iters=7, dim0=True)
    cb, idx = L.export()
    torch.cuda.synchronize()
    assert np.array_equal(cb.cpu().numpy().view(np.uint16), cb_ref.view(np.uint16))
    assert np.array_equal(idx.cpu().numpy(), idx_ref)
    x = synth.activation(2, F_in, seed=1)
    ok, m = parity_ok(_gemv(F, L, x), oracle_lib.gemm_dim0(cb_ref, idx_ref, x, group=group), x, F_in)
    assert ok, m


def test_dim0_gemm_slices(F, oracle_lib):
    F_out, F_in, M = 512, 768, 19
    cb, idx = _layer(F_out, F_in, 2, 128, 1, seed=9)
    X = synth.activation(M, F_in, seed=10)
    L = _import(F, cb, idx, F_in)
    Y = F.gemm(L, torch.from_numpy(X).cuda()).float().cpu().numpy()
    ok, m = parity_ok(Y, oracle_lib.gemm_dim0(cb, idx, X), X, F_in)
    assert ok, m


def test_dim0_errors(F):
    cb, idx = _layer(128, 64, 2, 16, 1, seed=1)
    L = _import(F, cb, idx, 64)
    with pytest.raises(F.FasqError) as e:
        F.Chain([([L], None)])
    assert e.value.code == -6
    with pytest.raises(F.FasqError) as e:
        L.shard_rows(0, 2)
    assert e.value.code == -6
    cb3 = np.zeros((42, 16, 3), np.float16)             # F_out % d != 0 -> -2 / d = 3 -> -6
    with pytest.raises(F.FasqError):
        F.import_layer(torch.from_numpy(cb3).cuda(), torch.zeros((42, 64), dtype=torch.uint8).cuda(), 64,
                       dim0=True)


def test_dim0_host_and_large_batch(F, oracle_lib):
    """dim = 0 layers through fasq_gemv_host (host buffers) and fasq_gemv with
    B > 8 (fasq_gemm's GEMV slices)."""
    F_out, F_in = 512, 1024
    cb, idx = _layer(F_out, F_in, 2, 256, 1, seed=41)
    L = _import(F, cb, idx, F_in)
    x = synth.activation(2, F_in, seed=42)
    y_host = torch.empty((2, F_out), dtype=torch.float32)
    F.gemv_host(L, torch.from_numpy(x), y_host)
    ok, m = parity_ok(y_host.numpy(), oracle_lib.gemm_dim0(cb, idx, x), x, F_in)
    assert ok, m
    X = synth.activation(11, F_in, seed=43)
    Y = F.gemv(L, torch.from_numpy(X).cuda()).float().cpu().numpy()
    ok, m = parity_ok(Y, oracle_lib.gemm_dim0(cb, idx, X), X, F_in)
    assert ok, m
