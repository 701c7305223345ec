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


@pytest.mark.parametrize("B", [1, 3, 8])
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


def _chain_vs_oracle(F, oracle_lib, specs, B, d, C, seed0=300, max_ctas=0, runs=1):
    """specs: list of (layers [(F_out, F_in)], src) -> builds, runs, checks every layer."""
    rng_seed = seed0
    built = []
    steps = []
    for shapes, src in specs:
        ls = []
        for (fo, fi) in shapes:
            cb, idx = synth.random_layer(fo, fi, d, C, seed=rng_seed)
            rng_seed += 1
            L = F.import_layer(torch.from_numpy(cb).cuda(), torch.from_numpy(idx).cuda(), fi, 1)
            ls.append((L, cb, idx))
        built.append(ls)
        steps.append(([t[0] for t in ls], src))
    chain = F.Chain(steps, B=B, max_ctas=max_ctas)
    x = synth.activation(B, specs[0][0][0][1], seed=seed0)
    for _ in range(runs):
        chain.run(torch.from_numpy(x).cuda())
    torch.cuda.synchronize()
    for s, ls in enumerate(built):
        src = steps[s][1]
        xin = x if src is None else chain.output(src[0], src[1], out_dtype=torch.float16).cpu().numpy()
        for l, (_, cb, idx) in enumerate(ls):
            y = chain.output(s, l, out_dtype=torch.float32).cpu().numpy()
            ref = oracle_lib.gemv(cb, idx, xin)
            ok, info = parity_ok(y, ref, xin, xin.shape[1])
            assert ok, (s, l, info)
    chain.free()


@pytest.mark.parametrize("d,C,B", [(1, 64, 1), (4, 256, 2), (8, 128, 1), (2, 256, 8), (2, 200, 4)])
def test_chain_entry_sizes_and_batches(F, oracle_lib, d, C, B):
    # ragged shapes: F_out not a multiple of 64, N_ss not a multiple of 32
    specs = [([(1000, 1016), (88, 1016)], None), ([(1016, 1000)], (0, 0)), ([(472, 1016)], (1, 0))]
    _chain_vs_oracle(F, oracle_lib, specs, B, d, C)


@pytest.mark.parametrize("d,C,ctas", [(2, 256, 3), (2, 128, 5), (1, 256, 2)])
def test_chain_long_k_ranges_codebook_pairs(F, oracle_lib, d, C, ctas):
    """Few CTAs -> every item spans many groups (odd and even counts, items
    starting at odd groups, a last group whose pair partner lies past the
    layer): the codebook PAIR ring (d <= 2) wraps many times; three runs in a
    row also cycle the double-buffered arenas."""
    specs = [([(640, 4096), (192, 4096)], None), ([(4096, 640)], (0, 0)), ([(704, 4096)], (1, 0))]
    _chain_vs_oracle(F, oracle_lib, specs, 1, d, C, seed0=900, max_ctas=ctas, runs=3)


def test_chain_input_from_other_layer_and_step(F, oracle_lib):
    # a step may read any earlier step's output, including layer 1 of a grouped step
    specs = [([(512, 768), (768, 768)], None), ([(768, 768)], (0, 1)), ([(640, 512)], (0, 0)),
             ([(768, 640)], (2, 0))]
    _chain_vs_oracle(F, oracle_lib, specs, 1, 2, 256)


@pytest.mark.parametrize("B", [1, 8])
def test_chain_llama_block_sampled(F, oracle_lib, B):
    """One Llama-3-8B-shaped block at full size (the bench's k_chain launch
    configuration; B = 8 uses 128-row tiles -> several items per CTA), checked
    on sampled rows of every layer."""
    sh = [("q", 4096, 4096), ("k", 1024, 4096), ("v", 1024, 4096), ("o", 4096, 4096), ("g", 14336, 4096),
          ("u", 14336, 4096), ("d", 4096, 14336)]
    Ls = {}
    for i, (n, fo, fi) in enumerate(sh):
        cb, idx = synth.torch_random_layer(fo, fi, 2, 256, seed=900 + i)
        Ls[n] = (F.import_layer(cb, idx, fi), cb, idx)
    steps = [([Ls["q"][0], Ls["k"][0], Ls["v"][0]], None), ([Ls["o"][0]], (0, 0)),
             ([Ls["g"][0], Ls["u"][0]], (1, 0)), ([Ls["d"][0]], (2, 0))]
    chain = F.Chain(steps, B=B)
    x = synth.torch_activation(B, 4096, seed=5)
    chain.run(x)
    torch.cuda.synchronize()
    names = [("q", "k", "v"), ("o",), ("g", "u"), ("d",)]
    rng = np.random.default_rng(0)
    for s, ns in enumerate(names):
        src = steps[s][1]
        xin = x.cpu().numpy() if src is None else chain.output(src[0], src[1], out_dtype=torch.float16).cpu().numpy()
        for l, n in enumerate(ns):
            _, cb, idx = Ls[n]
            F_out = idx.shape[1]
            yall = chain.output(s, l, out_dtype=torch.float32).cpu().numpy()
            cbn, idxn = cb.cpu().numpy(), idx.cpu().numpy()
            j = int(rng.integers(64, F_out - 128))
            for (j0, j1) in ((0, 32), (j, j + 64), (F_out - 32, F_out)):   # first, random, last rows
                ref = oracle_lib.gemv(cbn, idxn, xin, rows=(j0, j1))
                ok, info = parity_ok(yall[:, j0:j1], ref, xin, xin.shape[1])
                assert ok, (s, n, j0, info)
    chain.free()


@pytest.mark.parametrize("world", [2, 4])
def test_chain_tensor_parallel_fused_gather(F, oracle_lib, world):
    """fasq_chain_create_tp: `world` row-sharded ranks emulated as chains of
    ONE process on one GPU (max_ctas = SMs / world each, concurrent streams),
    peers wired with fasq_chain_set_peer_chains.  Every rank's outputs are the
    full vectors (the fused all-gather) and match the oracle of the unsharded
    layers; repeated runs are deterministic (arena parity flips)."""
    h, ffn, kv = 1024, 2048, 256
    names = [("q", h, h), ("k", kv, h), ("v", kv, h), ("o", h, h), ("g", ffn, h), ("u", ffn, h), ("d", h, ffn)]
    full = {}
    for i, (n, fo, fi) in enumerate(names):
        full[n] = synth.random_layer(fo, fi, 2, 256, seed=700 + i)
    nsm = torch.cuda.get_device_properties(0).multi_processor_count
    chains, keep = [], []
    for r in range(world):
        L = {}
        for (n, fo, fi) in names:
            cb, idx = full[n]
            rows = fo // world
            L[n] = F.import_layer(torch.from_numpy(cb).cuda(),
                                  torch.from_numpy(np.ascontiguousarray(idx[:, r * rows:(r + 1) * rows])).cuda(), fi)
        keep.append(L)
        steps = [([L["q"], L["k"], L["v"]], None), ([L["o"]], (0, 0)), ([L["g"], L["u"]], (1, 0)),
                 ([L["d"]], (2, 0))]
        chains.append(F.Chain(steps, B=1, world=world, rank=r, max_ctas=nsm // world))
    for c in chains:
        c.set_peer_chains(chains)
    x = synth.activation(1, h, seed=3)
    xd = torch.from_numpy(x).cuda()
    streams = [torch.cuda.Stream() for _ in range(world)]
    outs = []
    for rep in range(2):
        torch.cuda.synchronize()
        for c, s in zip(chains, streams):
            c.run(xd, stream=s)
        torch.cuda.synchronize()
        outs.append([c.output(3, 0, out_dtype=torch.int64).clone() for c in chains])
    torch.cuda.synchronize()
    for r in range(1, world):
        assert torch.equal(outs[0][0], outs[0][r])          # every rank holds the same gathered vector
    assert torch.equal(outs[0][0], outs[1][0])              # deterministic across runs
    flat = [("q", "k", "v"), ("o",), ("g", "u"), ("d",)]
    srcs = [None, (0, 0), (1, 0), (2, 0)]
    c0 = chains[world - 1]
    for s, ns in enumerate(flat):
        xin = x if srcs[s] is None else c0.output(srcs[s][0], srcs[s][1], out_dtype=torch.float16).cpu().numpy()
        for l, n in enumerate(ns):
            cb, idx = full[n]
            y = c0.output(s, l, out_dtype=torch.float32).cpu().numpy()
            ok, info = parity_ok(y, oracle_lib.gemv(cb, idx, xin), xin, xin.shape[1])
            assert ok, (world, s, n, info)
    for c in chains:
        c.free()


@pytest.mark.parametrize("world", [2, 4])
def test_chain_tp_bit_identical_to_single_gpu(F, world):
    """in the deterministic (default) TP plan the K ranges are the
    unsharded chain's, so every rank's gathered outputs equal the world-1
    chain's outputs byte for byte (shard F_out multiples of 64)."""
    h, ffn, kv = 1024, 2048, 256
    names = [("q", h, h), ("k", kv, h), ("v", kv, h), ("o", h, h), ("g", ffn, h), ("u", ffn, h), ("d", h, ffn)]
    full = {n: synth.random_layer(fo, fi, 2, 256, seed=800 + i) for i, (n, fo, fi) in enumerate(names)}
    x = torch.from_numpy(synth.activation(1, h, seed=4)).cuda()

    def steps_of(L):
        return [([L["q"], L["k"], L["v"]], None), ([L["o"]], (0, 0)), ([L["g"], L["u"]], (1, 0)), ([L["d"]], (2, 0)),
                ([L["q"], L["k"]], (3, 0))]
    L1 = {n: F.import_layer(torch.from_numpy(cb).cuda(), torch.from_numpy(idx).cuda(), idx.shape[0] * 2)
          for n, (cb, idx) in full.items()}
    single = F.Chain(steps_of(L1), B=1)
    single.run(x)
    torch.cuda.synchronize()
    ref = [[single.output(s, l, out_dtype=torch.int64).clone() for l in range(len(st[0]))]
           for s, st in enumerate(steps_of(L1))]
    nsm = torch.cuda.get_device_properties(0).multi_processor_count
    chains, keep = [], []
    for r in range(world):
        L = {}
        for (n, fo, fi) in names:
            cb, idx = full[n]
            rows = fo // world
            L[n] = F.import_layer(torch.from_numpy(cb).cuda(),
                                  torch.from_numpy(np.ascontiguousarray(idx[:, r * rows:(r + 1) * rows])).cuda(), fi)
        keep.append(L)
        chains.append(F.Chain(steps_of(L), B=1, world=world, rank=r, max_ctas=nsm // world))
    for c in chains:
        c.set_peer_chains(chains)
    streams = [torch.cuda.Stream() for _ in range(world)]
    for rep in range(3):   # arena parity cycles; the DONE protocol orders the runs
        for c, s in zip(chains, streams):
            c.run(x, stream=s)
    torch.cuda.synchronize()
    for c in chains:
        for s, outs in enumerate(ref):
            for l, want in enumerate(outs):
                got = c.output(s, l, out_dtype=torch.int64)
                assert torch.equal(got, want), (world, s, l)
    for c in chains:
        c.free()
    single.free()


def test_chain_out_of_range_partial_is_flagged(F):
    """A K-split partial beyond |v| < 2^18 (value units) is not silently
    clamped: the run's float outputs are NaN and check() raises FASQ_E_RANGE;
    the flag clears and the next in-range run is clean."""
    fo, fi = 256, 512
    cb = np.full((fi // 2, 16, 2), 60000.0, np.float16)
    idx = np.zeros((fi // 2, fo), np.uint8)
    L = F.import_layer(torch.from_numpy(cb).cuda(), torch.from_numpy(idx).cuda(), fi)
    ch = F.Chain([([L], None)], B=1)
    x = torch.full((1, fi), 8.0, dtype=torch.float16, device="cuda")   # 512 * 60000 * 8 >> 2^18
    ch.run(x)
    y = ch.output(0, 0, out_dtype=torch.float32)
    torch.cuda.synchronize()
    assert torch.isnan(y).all()
    with pytest.raises(F.FasqError) as e:
        ch.check()
    assert e.value.code == -9
    ch.run(torch.full((1, fi), 1e-4, dtype=torch.float16, device="cuda"))
    y = ch.output(0, 0, out_dtype=torch.float32)
    ch.check()
    assert torch.isfinite(y).all()
    ch.free()


def test_chain_run_host_end_to_end(F, oracle_lib):
    """fasq_chain_run_host: host x in, host y out (H2D, chain, D2H)."""
    cb, idx = synth.random_layer(768, 1024, 2, 256, seed=61)
    L = F.import_layer(torch.from_numpy(cb).cuda(), torch.from_numpy(idx).cuda(), 1024)
    ch = F.Chain([([L], None)], B=2)
    x = synth.activation(2, 1024, seed=62)
    y = torch.empty((2, 768), dtype=torch.float32).pin_memory()
    ch.run_host(torch.from_numpy(x).pin_memory(), y, 0, 0)
    ok, info = parity_ok(y.numpy(), oracle_lib.gemv(cb, idx, x), x, 1024)
    assert ok, info
    with pytest.raises(F.FasqError):
        ch.run(torch.zeros((2, 1000), dtype=torch.float16, device="cuda"))   # shape checked in the binding
    ch.free()


def _ipc_worker(rank, world, port, q):
    import os
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist
    import paper_2605_04084_b200 as F
    try:
        torch.cuda.set_device(0)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        cb, idx = synth.random_layer(512, 512, 2, 64, seed=rank)
        L = F.import_layer(torch.from_numpy(cb).cuda(), torch.from_numpy(idx).cuda(), 512)
        ch = F.Chain([([L], None)], B=1, world=world, rank=rank, max_ctas=8)
        handles = [None] * world
        dist.all_gather_object(handles, ch.ipc_handle())
        ch.set_peers(handles)          # opens the peer arenas (cudaIpcOpenMemHandle)
        dist.barrier()
        ch.free()
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except Exception as e:            # reported to the parent
        q.put((rank, repr(e)))


def test_chain_ipc_handles_between_processes():
    """The multi-process plumbing of the TP chain: two ranks (processes) on one
    GPU export their arena IPC handles, exchange them through
    torch.distributed and open each other's arena.  (Running the TP kernels
    needs one GPU per rank: two processes time-slice one GPU; the kernel path
    is covered in-process by test_chain_tensor_parallel_fused_gather.)"""
    import multiprocessing as mp
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_ipc_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=240) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    assert res == {0: "ok", 1: "ok"}, res
