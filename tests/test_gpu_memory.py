"""Device memory and layer immutability (VERDICT r1 "boundary"; SURVEY 8(b)
fasq_set_allocator): per-call split-K workspaces, so one layer may run on
several streams at once and inside CUDA-graph capture without a warm-up call;
the library's buffers can come from torch's caching allocator."""
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


def _layer(F, F_out, F_in, seed):
    cb, idx = synth.random_layer(F_out, F_in, 2, 256, seed=seed)
    return F.import_layer(torch.from_numpy(cb).cuda(), torch.from_numpy(idx).cuda(), F_in), cb, idx


def test_gemv_two_streams_one_layer(F, oracle_lib):
    """fasq_gemv with dense fp32 outputs uses split-K (partials + tickets) on
    this shape; 16 launches alternating on two streams with different inputs,
    all in flight together, each result checked against the oracle."""
    L, cb, idx = _layer(F, 4096, 4096, 31)
    xs = [synth.activation(1, 4096, seed=100 + i) for i in range(16)]
    xd = [torch.from_numpy(x).cuda() for x in xs]
    ys = [torch.empty((1, 4096), dtype=torch.float32, device="cuda") for _ in xs]
    s = [torch.cuda.Stream(), torch.cuda.Stream()]
    torch.cuda.synchronize()
    for i in range(16):
        F.gemv(L, xd[i], out=ys[i], stream=s[i % 2])
    torch.cuda.synchronize()
    for i in range(16):
        ref = oracle_lib.gemv(cb, idx, xs[i])
        ok, info = parity_ok(ys[i].cpu().numpy(), ref, xs[i], 4096)
        assert ok, (i, info)
    L.free()


def test_gemm_split_k_two_streams_one_layer(F, oracle_lib):
    """fasq_gemm EXPAND at M = 512 on 4096 x 4096 runs split-K over a
    workspace; two streams, different X, concurrently."""
    L, cb, idx = _layer(F, 4096, 4096, 32)
    Xs = [synth.activation(512, 4096, seed=200 + i) for i in range(4)]
    Xd = [torch.from_numpy(X).cuda() for X in Xs]
    Ys = [torch.empty((512, 4096), dtype=torch.float32, device="cuda") for _ in Xs]
    s = [torch.cuda.Stream(), torch.cuda.Stream()]
    torch.cuda.synchronize()
    for i in range(4):
        F.gemm(L, Xd[i], out=Ys[i], algo=F.GEMM_EXPAND_TC, stream=s[i % 2])
    torch.cuda.synchronize()
    for i in range(4):
        sub = slice(0, 512, 61)
        ref = oracle_lib.gemm(cb, idx[:, :256], Xs[i][sub])
        ok, info = parity_ok(Ys[i][sub, :256].cpu().numpy(), ref, Xs[i][sub], 4096)
        assert ok, (i, info)
    L.free()


def test_split_k_inside_graph_capture_first_call(F, oracle_lib):
    """The first ever split-K call of a layer may be inside stream capture (the
    workspace is a stream-ordered allocation node, not a grown per-layer buffer)."""
    L, cb, idx = _layer(F, 14336, 4096, 33)
    x = synth.activation(2, 4096, seed=7)
    xd = torch.from_numpy(x).cuda()
    y = torch.empty((2, 14336), dtype=torch.float32, device="cuda")
    st = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        F.gemv(L, xd, out=y)
    g.replay()
    g.replay()
    torch.cuda.synchronize()
    ref = oracle_lib.gemv(cb, idx[:, :512], x)
    ok, info = parity_ok(y[:, :512].cpu().numpy(), ref, x, 4096)
    assert ok, info
    L.free()


def test_torch_allocator_hook(F, oracle_lib):
    """With use_torch_allocator() the layer storage, workspaces and chain
    buffers come from torch's caching allocator (its allocated bytes grow by
    at least the layer's storage); results are unchanged; switching back
    releases through torch again (each pointer remembers its allocator)."""
    torch.cuda.synchronize()
    before = torch.cuda.memory_allocated()
    F.use_torch_allocator(True)
    try:
        L, cb, idx = _layer(F, 4096, 4096, 34)
        torch.cuda.synchronize()
        grown = torch.cuda.memory_allocated() - before
        assert grown >= L.info["index_bytes"], (grown, L.info)
        x = synth.activation(1, 4096, seed=8)
        y = F.gemv(L, torch.from_numpy(x).cuda(), out_dtype=torch.float32)
        chain = F.Chain([([L], None), ([L], (0, 0))], B=1)
        chain.run(torch.from_numpy(x).cuda())
        y2 = chain.output(0, 0, out_dtype=torch.float32)
        torch.cuda.synchronize()
        ref = oracle_lib.gemv(cb, idx, x)
        for yy in (y, y2):
            ok, info = parity_ok(yy.cpu().numpy(), ref, x, 4096)
            assert ok, info
    finally:
        F.use_torch_allocator(False)
    chain.free()
    L.free()   # allocated by torch: released through torch although the hook is off now
    torch.cuda.synchronize()
    assert torch.cuda.memory_allocated() - before < 1 << 20
