"""Persistent decode-chain executor (fasq_chain_*) vs the fp64 oracle, step by
step, on a small transformer-block-shaped chain (q/k/v -> o -> gate/up ->
down -> next block)."""
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


def _layer(F, fo, fi, seed, C=256):
    cb, idx = synth.random_layer(fo, fi, 2, C, seed=seed)
    return F.import_layer(torch.from_numpy(cb).cuda(), torch.from_numpy(idx).cuda(), fi, 1), cb, idx


@pytest.mark.parametrize("B", [1, 3])
def test_chain_matches_oracle(F, oracle_lib, B):
    h, ffn, kv = 1024, 2048, 256
    blocks = []
    seed = 100
    for b in range(2):
        blk = {}
        for name, fo, fi in [("q", h, h), ("k", kv, h), ("v", kv, h), ("o", h, h), ("g", ffn, h), ("u", ffn, h),
                             ("d", h, ffn)]:
            blk[name] = _layer(F, fo, fi, seed, C=256 if name != "k" else 128)
            seed += 1
        blocks.append(blk)
    steps = []
    for b, blk in enumerate(blocks):
        s0 = len(steps)
        steps.append(([blk["q"][0], blk["k"][0], blk["v"][0]], None if b == 0 else (s0 - 1, 0)))
        steps.append(([blk["o"][0]], (s0, 0)))
        steps.append(([blk["g"][0], blk["u"][0]], (s0 + 1, 0)))
        steps.append(([blk["d"][0]], (s0 + 2, 0)))
    chain = F.Chain(steps, B=B)
    x = synth.activation(B, h, seed=7)
    chain.run(torch.from_numpy(x).cuda())
    torch.cuda.synchronize()
    flat = [(blocks[b], names) for b in range(2) for names in (("q", "k", "v"), ("o",), ("g", "u"), ("d",))]
    for s, (blk, names) in enumerate(flat):
        src = steps[s][1]
        xin = x if src is None else chain.output(src[0], src[1], out_dtype=torch.float16).cpu().numpy()
        for l, name in enumerate(names):
            _, cb, idx = blk[name]
            y = chain.output(s, l, out_dtype=torch.float32).cpu().numpy()
            ref = oracle_lib.gemv(cb, idx, xin)
            ok, info = parity_ok(y, ref, xin, idx.shape[0] * 2)
            assert ok, (s, name, info)
    # deterministic across runs
    a = chain.output(len(steps) - 1, 0, out_dtype=torch.int64).clone()
    chain.run(torch.from_numpy(x).cuda())
    b_ = chain.output(len(steps) - 1, 0, out_dtype=torch.int64)
    torch.cuda.synchronize()
    assert torch.equal(a, b_)
    chain.free()


def test_chain_errors(F):
    L1, _, _ = _layer(F, 256, 512, 1)
    L2, _, _ = _layer(F, 256, 1024, 2)
    with pytest.raises(F.FasqError):
        F.Chain([([L1], None), ([L2], (0, 0))])     # F_out 256 != F_in 1024
    with pytest.raises(F.FasqError):
        F.Chain([([L1], (1, 0))])                  # forward reference
