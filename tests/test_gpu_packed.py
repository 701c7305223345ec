"""GPU parity of NEXT-2: ceil(log2 C)-bit packed indices (Eq. 4, P:224-231;
Table 2's 2-128 / 2-512 / 2-1024 points) through the C ABI.

  * import -> export is the identity on the logical table (bit-exact), for
    every index width 1..10 bits;
  * the packed decode GEMV matches the fp64 oracle (uint16 reconstruct-then-
    multiply) within north_star's tolerance, B = 1..8, ragged rows / groups,
    and on sampled rows of the full Llama-3-8B shapes at C = 128 / 512 / 1024;
  * the GPU packer at C = 512 / 1024 (and packed storage at C = 128) is
    bit-identical to the oracle's pack;
  * the Eq. 4 index bits are what the layer reports and stores;
  * fasq_gemm on a packed layer (8-token GEMV slices), determinism, errors.
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


def _dev_idx(idx):
    a = np.ascontiguousarray(idx)
    return torch.from_numpy(a.view(np.int16) if a.dtype == np.uint16 else a).cuda()


def _import(F, cb, idx, F_in, group=1, packed=True):
    return F.import_layer(torch.from_numpy(cb).cuda(), _dev_idx(idx), F_in, group, packed=packed)


def _gemv(F, L, x, out_dtype=torch.float32):
    y = F.gemv(L, torch.from_numpy(x).cuda(), out_dtype=out_dtype)
    torch.cuda.synchronize()
    return y.float().cpu().numpy().astype(np.float64)


def _export_np(L):
    cb, idx = L.export()
    torch.cuda.synchronize()
    idx = idx.cpu().numpy()
    return cb.cpu().numpy(), (idx.view(np.uint16) if idx.dtype == np.int16 else idx)


@pytest.mark.parametrize("C", [2, 3, 8, 16, 33, 64, 100, 128, 256, 300, 512, 1000, 1024])
def test_import_export_roundtrip(F, C):
    F_out, F_in = 200, 2 * 70       # ragged rows (pad to 256) and groups (N_ss = 70)
    cb, idx = synth.random_layer(F_out, F_in, 2, C, seed=C)
    L = _import(F, cb, idx, F_in)
    bits = int(np.ceil(np.log2(C)))
    assert L.index_bits == bits
    assert L.info["index_bytes"] == (70 * F_out * bits + 7) // 8    # Eq. 4 index table
    cb2, idx2 = _export_np(L)
    assert np.array_equal(cb2.view(np.uint16), cb.view(np.uint16))
    assert idx2.dtype == idx.dtype and np.array_equal(idx2, idx)


SMALL = [
    # F_out, F_in, C, group, B
    (1000, 640, 128, 1, 1),      # 7-bit, ragged rows, 10 groups
    (3000, 1000, 512, 1, 1),     # 9-bit, 3 row tiles, ragged last group (N_ss = 500)
    (1000, 640, 1024, 1, 1),     # 10-bit, one codebook slot
    (777, 96, 48, 1, 1),         # 6-bit, tiny K
    (1024, 512, 2, 4, 1),        # 1-bit, shared codebooks
    (2048, 2048, 1024, 2, 1),    # group = 2
    (1000, 640, 128, 1, 2),
    (1000, 640, 512, 1, 3),
    (1000, 640, 1024, 1, 4),
    (1000, 640, 128, 1, 5),
    (1000, 640, 1024, 1, 8),
    (600, 1024, 300, 1, 6),
    (33, 64, 4, 1, 1),           # tiny
]


@pytest.mark.parametrize("F_out,F_in,C,group,B", SMALL)
def test_packed_gemv_small(F, oracle_lib, F_out, F_in, C, group, B):
    cb, idx = synth.random_layer(F_out, F_in, 2, C, group=group, seed=F_out + F_in + C + B)
    x = synth.activation(B, F_in, seed=B + 7)
    L = _import(F, cb, idx, F_in, group)
    y = _gemv(F, L, x)
    y_ref = oracle_lib.gemv(cb, idx, x, group=group)
    ok, m = parity_ok(y, y_ref, x, F_in)
    assert ok, m


@pytest.mark.parametrize("B", [1, 8])
@pytest.mark.parametrize("out_dtype", [torch.float16, torch.int64])
def test_packed_output_dtypes(F, oracle_lib, B, out_dtype):
    F_out, F_in, C = 1500, 1024, 512
    cb, idx = synth.random_layer(F_out, F_in, 2, C, seed=11)
    x = synth.activation(B, F_in, seed=12)
    L = _import(F, cb, idx, F_in)
    xd = torch.from_numpy(x).cuda()
    if out_dtype == torch.int64:   # FASQ_ACC_I64: added into a caller-zeroed buffer
        y = torch.zeros((B, F_out), dtype=torch.int64, device="cuda")
        F.gemv_grouped([L], xd, outs=[y], out_dtype=torch.int64)
        yv = y.cpu().numpy().astype(np.float64) * 2.0 ** -32
    else:
        yv = F.gemv(L, xd, out_dtype=out_dtype).float().cpu().numpy().astype(np.float64)
    y_ref = oracle_lib.gemv(cb, idx, x)
    ok, m = parity_ok(yv, y_ref, x, F_in)
    assert ok, m


@pytest.mark.parametrize("F_out,F_in", [(4096, 4096), (14336, 4096), (4096, 14336), (1024, 4096)])
@pytest.mark.parametrize("C", [128, 512, 1024])
def test_packed_llama_shapes_sampled(F, oracle_lib, F_out, F_in, C):
    cb, idx = synth.random_layer(F_out, F_in, 2, C, seed=F_out // 7 + F_in + C)
    x = synth.activation(1, F_in, seed=5)
    L = _import(F, cb, idx, F_in)
    y = _gemv(F, L, x)
    for j0 in (0, F_out // 2 + 37, F_out - 64):
        y_ref = oracle_lib.gemv(cb, idx, x, rows=(j0, j0 + 64))
        ok, m = parity_ok(y[:, j0:j0 + 64], y_ref, x, F_in)
        assert ok, (j0, m)


def test_packed_deterministic(F):
    cb, idx = synth.random_layer(4096, 4096, 2, 1024, seed=3)
    x = synth.activation(1, 4096, seed=4)
    L = _import(F, cb, idx, 4096)
    a = _gemv(F, L, x)
    for _ in range(3):
        assert np.array_equal(_gemv(F, L, x), a)


@pytest.mark.parametrize("C,group,F_out,F_in", [(512, 2, 400, 64), (1024, 1, 1100, 32), (300, 4, 200, 48)])
def test_gpu_pack_wide_bit_exact(F, oracle_lib, C, group, F_out, F_in):
    W = synth.weight(F_out, F_in, seed=C + group)
    cb_ref, idx_ref, _ = oracle_lib.pack(W, d=2, C=C, group=group, seed=9, iters=6)
    L = F.pack(torch.from_numpy(W).cuda(), d=2, C=C, group=group, seed=9, iters=6)
    assert L.index_bits == int(np.ceil(np.log2(C)))
    cb, idx = _export_np(L)
    assert np.array_equal(cb.view(np.uint16), cb_ref.view(np.uint16))
    assert idx.dtype == np.uint16 and np.array_equal(idx, idx_ref)


def test_gpu_pack_packed_C128_bit_exact(F, oracle_lib):
    W = synth.weight(512, 128, seed=2)
    cb_ref, idx_ref, _ = oracle_lib.pack(W, d=2, C=128, group=1, seed=4, iters=8)
    L = F.pack(torch.from_numpy(W).cuda(), d=2, C=128, group=1, seed=4, iters=8, packed=True)
    assert L.index_bits == 7
    cb, idx = _export_np(L)
    assert np.array_equal(cb.view(np.uint16), cb_ref.view(np.uint16))
    assert np.array_equal(idx, idx_ref)
    x = synth.activation(2, 128, seed=1)
    ok, m = parity_ok(_gemv(F, L, x), oracle_lib.gemv(cb_ref, idx_ref, x), x, 128)
    assert ok, m


def test_packed_gemm_slices(F, oracle_lib):
    F_out, F_in, C, M = 700, 512, 1024, 21
    cb, idx = synth.random_layer(F_out, F_in, 2, C, seed=8)
    X = synth.activation(M, F_in, seed=9)
    L = _import(F, cb, idx, F_in)
    Y = F.gemm(L, torch.from_numpy(X).cuda()).float().cpu().numpy()
    ok, m = parity_ok(Y, oracle_lib.gemm(cb, idx, X), X, F_in)
    assert ok, m


def test_packed_errors(F):
    cb, idx = synth.random_layer(128, 64, 2, 300, seed=1)
    idx[5, 7] = 300                                      # >= C
    with pytest.raises(F.FasqError) as e:
        _import(F, cb, idx, 64)
    assert e.value.code == -1
    cb4, idx4 = synth.random_layer(128, 64, 4, 64, seed=1)   # packed needs d = 2
    with pytest.raises(F.FasqError) as e:
        _import(F, cb4, idx4, 64, packed=True)
    assert e.value.code == -6
    cb, idx = synth.random_layer(128, 64, 2, 128, seed=1)
    L = _import(F, cb, idx, 64)
    with pytest.raises(F.FasqError) as e:               # the decode chain reads byte indices only
        F.Chain([([L], None)])
    assert e.value.code == -6


def test_packed_shard_host_and_large_batch(F, oracle_lib):
    """Packed layers through the other entry points: fasq_shard_rows (row shards
    keep the packed layout and export the same rows), fasq_gemv_host (host
    buffers) and fasq_gemv with B > 8 (dispatched to fasq_gemm's GEMV slices)."""
    F_out, F_in, C = 1024, 512, 512
    cb, idx = synth.random_layer(F_out, F_in, 2, C, seed=31)
    L = _import(F, cb, idx, F_in)
    for r in range(2):
        S = L.shard_rows(r, 2)
        assert S.index_bits == 9 and S.F_out == F_out // 2
        _, sidx = _export_np(S)
        assert np.array_equal(sidx, idx[:, r * 512:(r + 1) * 512])
    x = synth.activation(3, F_in, seed=32)
    y_host = torch.empty((3, F_out), dtype=torch.float32)
    F.gemv_host(L, torch.from_numpy(x), y_host)
    ok, m = parity_ok(y_host.numpy(), oracle_lib.gemv(cb, idx, x), x, F_in)
    assert ok, m
    X = synth.activation(12, F_in, seed=33)
    Y = F.gemv(L, torch.from_numpy(X).cuda()).float().cpu().numpy()
    ok, m = parity_ok(Y, oracle_lib.gemm(cb, idx, X), X, F_in)
    assert ok, m
