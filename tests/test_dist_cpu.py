"""Multi-process (world size 2, gloo, CPU) test of the row-shard + all-gather
plumbing.  Each rank computes its row slice of a PQ layer with
the ORACLE (no GPU here), the slices are all-gathered, and the result must be
bit-identical to the unsharded oracle product (rows are independent sums)."""
import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, B, q):
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        import synth
        from paper_2605_04084_b200 import shard  # noqa: F401  (pure torch.distributed plumbing)
        F_out, F_in = 512, 256
        cb, idx = synth.random_layer(F_out, F_in, 2, 64, seed=3)
        x = synth.activation(B, F_in, seed=4)
        local_idx = shard.shard_indices(torch.from_numpy(idx), rank, world).numpy()
        y_local = torch.from_numpy(oracle.gemv(cb, local_idx, x))
        y = shard.gather_rows(y_local)
        full = oracle.gemv(cb, idx, x)
        ok = bool(np.array_equal(y.numpy(), full))
        # chained second layer: the gathered activation feeds the next sharded layer
        cb2, idx2 = synth.random_layer(256, F_out, 2, 16, seed=5)
        x2 = y.numpy().astype(np.float16)
        y2 = shard.gather_rows(torch.from_numpy(oracle.gemv(cb2, shard.shard_indices(torch.from_numpy(idx2), rank, world).numpy(), x2)))
        ok2 = bool(np.array_equal(y2.numpy(), oracle.gemv(cb2, idx2, x2)))
        q.put((rank, ok, ok2))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("B", [1, 3])
def test_row_shard_allgather_gloo(B):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, B, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    res = sorted(q.get(timeout=10) for _ in range(world))
    assert all(r[1] and r[2] for r in res), res


def test_row_range_arithmetic():
    from paper_2605_04084_b200 import shard
    for F_out in (1024, 4096, 14336):
        for world in (1, 2, 4, 8):
            spans = [shard.row_range(F_out, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == F_out
            assert all(spans[i][1] == spans[i + 1][0] for i in range(world - 1))
    with pytest.raises(ValueError):
        shard.row_range(1000, 0, 3)
