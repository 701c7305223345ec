"""GPU parity of the prefill GEMM (C-ABI fasq_gemm, LUT and EXPAND_TC
variants) against the fp64 oracle (reconstruct-then-multiply)."""
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


def _run(F, cb, idx, X, F_in, group, algo, out_dtype=torch.float32):
    L = F.import_layer(torch.from_numpy(cb).cuda(), torch.from_numpy(idx).cuda(), F_in, group)
    Y = F.gemm(L, torch.from_numpy(X).cuda(), out_dtype=out_dtype, algo=algo)
    torch.cuda.synchronize()
    return Y.float().cpu().numpy().astype(np.float64)


CASES = [
    # F_out, F_in, C, M
    (256, 64, 256, 128),      # one tile
    (512, 256, 256, 300),     # ragged M (3 token tiles)
    (1000, 640, 128, 200),    # ragged rows (F_out_pad 1024 -> partial last tile)
    (300, 128, 7, 33),        # odd C, rows not a multiple of 32
    (2048, 1024, 256, 512),
]


@pytest.mark.parametrize("algo", ["tc", "lut"])
@pytest.mark.parametrize("F_out,F_in,C,M", CASES)
def test_gemm_small(F, oracle_lib, algo, F_out, F_in, C, M):
    cb, idx = synth.random_layer(F_out, F_in, 2, C, seed=F_out + M)
    X = synth.activation(M, F_in, seed=M)
    a = F.GEMM_EXPAND_TC if algo == "tc" else F.GEMM_LUT
    Y = _run(F, cb, idx, X, F_in, 1, a)
    ref = oracle_lib.gemm(cb, idx, X)
    ok, info = parity_ok(Y, ref, X, F_in)
    assert ok, info


def test_gemm_rows_match_gemv(F):
    cb, idx = synth.random_layer(1024, 512, 2, 256, seed=1)
    X = synth.activation(130, 512, seed=2)
    L = F.import_layer(torch.from_numpy(cb).cuda(), torch.from_numpy(idx).cuda(), 512, 1)
    Y = F.gemm(L, torch.from_numpy(X).cuda(), algo=F.GEMM_EXPAND_TC)
    y = F.gemv(L, torch.from_numpy(X[129:130]).cuda())
    torch.cuda.synchronize()
    assert np.allclose(Y[129].cpu().numpy(), y[0].cpu().numpy(), rtol=1e-5, atol=1e-5)


def test_gemm_fp16_out(F, oracle_lib):
    cb, idx = synth.random_layer(512, 256, 2, 256, seed=3)
    X = synth.activation(256, 256, seed=4)
    for algo in (F.GEMM_EXPAND_TC, F.GEMM_LUT):
        Y = _run(F, cb, idx, X, 256, 1, algo, out_dtype=torch.float16)
        ok, info = parity_ok(Y, oracle_lib.gemm(cb, idx, X), X, 256)
        assert ok, (algo, info)


def test_gemm_saturated_exact_w(F, oracle_lib):
    """Saturated codebook: W_hat == W, so Y == X . W^T (numpy fp64 matmul)."""
    W = synth.structured_weight(512, 256, 2, 9, group=1, seed=5)
    cb, idx, _ = oracle_lib.pack(W, d=2, C=16, group=1, seed=0)
    X = synth.activation(128, 256, seed=6)
    Y = _run(F, cb, idx, X, 256, 1, F.GEMM_EXPAND_TC)
    ref = X.astype(np.float64) @ W.astype(np.float64).T
    ok, info = parity_ok(Y, ref, X, 256)
    assert ok, info


@pytest.mark.parametrize("F_out,F_in", [(4096, 4096), (14336, 4096), (4096, 14336), (1024, 4096)])
def test_gemm_llama_sampled(F, oracle_lib, F_out, F_in):
    """Full Llama shapes at M=512 (bench configuration), sampled rows/tokens."""
    cb, idx = synth.random_layer(F_out, F_in, 2, 256, seed=F_out + F_in)
    X = synth.activation(512, F_in, seed=3)
    Y = _run(F, cb, idx, X, F_in, 1, F.GEMM_EXPAND_TC)
    for j0 in (0, F_out - 64):
        ref = oracle_lib.gemm(cb, idx, X[::37], rows=(j0, j0 + 64))
        ok, info = parity_ok(Y[::37, j0:j0 + 64], ref, X[::37], F_in)
        assert ok, (j0, info)


@pytest.mark.parametrize("F_out,F_in,M,ks", [(512, 2048, 100, 0), (1000, 2496, 300, 4), (256, 4096, 17, 0),
                                             (1000, 2496, 300, 3), (512, 4096, 77, 5), (768, 4096, 260, 6),
                                             (256, 4096, 129, 7)])
def test_gemm_tc_split_k(F, oracle_lib, monkeypatch, F_out, F_in, M, ks):
    """Small M -> fewer tiles than SMs -> split-K over gridDim.z with an fp32
    workspace merged by the last CTA of each tile in fixed order (ks = 0: the
    library's choice; 4: forced, uneven chunk counts (39 chunks); 3 / 5 / 6 / 7: the merge deals
    the 8 column chunks of a tile unevenly over the K slices).  Two calls in a row also
    check the per-tile ticket reset, and the result must be bit-identical."""
    if ks:
        monkeypatch.setenv("FASQ_GEMM_KSPLIT", str(ks))
    cb, idx = synth.random_layer(F_out, F_in, 2, 256, seed=F_out + M + 7)
    X = synth.activation(M, F_in, seed=M + 1)
    L = F.import_layer(torch.from_numpy(cb).cuda(), torch.from_numpy(idx).cuda(), F_in, 1)
    Xd = torch.from_numpy(X).cuda()
    Y1 = F.gemm(L, Xd, out_dtype=torch.float32, algo=F.GEMM_EXPAND_TC)
    Y2 = F.gemm(L, Xd, out_dtype=torch.float32, algo=F.GEMM_EXPAND_TC)
    torch.cuda.synchronize()
    assert torch.equal(Y1, Y2)
    ref = oracle_lib.gemm(cb, idx, X)
    ok, info = parity_ok(Y1.cpu().numpy().astype(np.float64), ref, X, F_in)
    assert ok, info


def test_gemm_tc_tail_wave_split_k(F, oracle_lib, monkeypatch):
    """More tiles than SMs with a small last wave (5 row tiles x 30 token tiles =
    150 tiles on 148 SMs): the full waves run as one launch, the 2 tail tiles as a
    split-K launch.  The tail tiles (last 256 tokens) are checked against the
    oracle, the whole output against the single-launch path."""
    F_out, F_in, M = 1280, 1024, 7680
    cb, idx = synth.random_layer(F_out, F_in, 2, 256, seed=77)
    X = synth.activation(M, F_in, seed=78)
    L = F.import_layer(torch.from_numpy(cb).cuda(), torch.from_numpy(idx).cuda(), F_in, 1)
    Xd = torch.from_numpy(X).cuda()
    Y = F.gemm(L, Xd, out_dtype=torch.float32, algo=F.GEMM_EXPAND_TC)
    monkeypatch.setenv("FASQ_GEMM_KSPLIT", "1")
    Y1 = F.gemm(L, Xd, out_dtype=torch.float32, algo=F.GEMM_EXPAND_TC)
    torch.cuda.synchronize()
    tail = slice(M - 256, M)
    ref = oracle_lib.gemm(cb, idx, X[tail])
    ok, info = parity_ok(Y[tail].cpu().numpy().astype(np.float64), ref, X[tail], F_in)
    assert ok, info
    d = (Y - Y1).abs().max().item()
    assert d <= 1e-3 * max(1.0, Y1.abs().max().item()), d


@pytest.mark.parametrize("d,C,F_out,F_in,M", [(4, 256, 512, 1024, 100), (8, 128, 300, 512, 37), (1, 64, 256, 256, 50),
                                              (4, 16, 1000, 2048, 7)])
def test_gemm_lut_all_subvector_sizes(F, oracle_lib, d, C, F_out, F_in, M):
    """GEMM-LUT (and AUTO, which routes d != 2 to it) for every sub-vector size:
    the LUT entry is dot(x_ss, c_k) over d elements, gathered by index."""
    cb, idx = synth.random_layer(F_out, F_in, d, C, seed=F_out + d + M)
    X = synth.activation(M, F_in, seed=M + d)
    ref = oracle_lib.gemm(cb, idx, X)
    for algo in (F.GEMM_LUT, F.GEMM_AUTO):
        Y = _run(F, cb, idx, X, F_in, 1, algo)
        ok, info = parity_ok(Y, ref, X, F_in)
        assert ok, (algo, info)


@pytest.mark.parametrize("F_out,F_in,M,ks", [(4096, 4096, 8, 0), (1000, 2496, 5, 0), (512, 1024, 13, 7),
                                             (4096, 14336, 32, 0)])
def test_gemm_lut_split_k_short_L(F, oracle_lib, monkeypatch, F_out, F_in, M, ks):
    """NEXT-3 (Alg. 3's split-K for short L): with fewer (row, token)
    tiles than 2 waves the groups are split over gridDim.z (fp32 partials in a
    per-call workspace, merged in fixed order).  ks = 0: the library's choice;
    7: forced, uneven group ranges.  Oracle parity on sampled rows; two calls
    are bit-identical (deterministic merge)."""
    if ks:
        monkeypatch.setenv("FASQ_LUT_KSPLIT", str(ks))
    cb, idx = synth.random_layer(F_out, F_in, 2, 256, seed=F_out + M)
    X = synth.activation(M, F_in, seed=M + 5)
    L = F.import_layer(torch.from_numpy(cb).cuda(), torch.from_numpy(idx).cuda(), F_in, 1)
    Xd = torch.from_numpy(X).cuda()
    Y1 = F.gemm(L, Xd, out_dtype=torch.float32, algo=F.GEMM_LUT)
    Y2 = F.gemm(L, Xd, out_dtype=torch.float32, algo=F.GEMM_LUT)
    torch.cuda.synchronize()
    assert torch.equal(Y1, Y2)
    for j0 in (0, F_out - 64):
        ref = oracle_lib.gemm(cb, idx[:, j0:j0 + 64], X)
        ok, info = parity_ok(Y1[:, j0:j0 + 64].cpu().numpy().astype(np.float64), ref, X, F_in)
        assert ok, (j0, info)
    L.free()


@pytest.mark.parametrize("B", [9, 16, 33, 64, 80, 128, 140])
def test_gemv_large_batch_dispatches_to_gemm(F, oracle_lib, B):
    """NEXT-3: fasq_gemv with B > 8 runs the tcgen05 decode kernel up to
    B = 128 (gemv_tc.cu, PDL allowed) and the prefill GEMM above (AUTO -> EXPAND,
    no flags); same product, oracle parity."""
    cb, idx = synth.random_layer(2048, 4096, 2, 256, seed=B)
    x = synth.activation(B, 4096, seed=B + 1)
    L = F.import_layer(torch.from_numpy(cb).cuda(), torch.from_numpy(idx).cuda(), 4096, 1)
    y = F.gemv(L, torch.from_numpy(x).cuda(), out_dtype=torch.float32)
    torch.cuda.synchronize()
    ref = oracle_lib.gemm(cb, idx[:, :256], x)
    ok, info = parity_ok(y[:, :256].cpu().numpy().astype(np.float64), ref, x, 4096)
    assert ok, info
    if B <= 128:
        y2 = F.gemv(L, torch.from_numpy(x).cuda(), out_dtype=torch.float32, flags=F.FLAG_PDL)
        assert torch.equal(y2, y)
    else:
        with pytest.raises(F.FasqError):
            F.gemv(L, torch.from_numpy(x).cuda(), out_dtype=torch.float32, flags=F.FLAG_PDL)
    L.free()


@pytest.mark.parametrize("F_out,F_in,M", [(4096, 4096, 2048), (14336, 4096, 2048), (4096, 14336, 1536),
                                          (1000, 512, 1300)])
def test_gemm_tc_pair_cta_group2(F, oracle_lib, monkeypatch, F_out, F_in, M):
    """The opt-in 2-CTA EXPAND (FASQ_GEMM_PAIR=1: cta_group::2, each CTA of a
    cluster expands half of the 256-row B tile, the leader issues M = 256 MMAs):
    sampled rows against the fp64 oracle, and equal to the 1-CTA kernel's Y
    (same K order per output)."""
    monkeypatch.setenv("FASQ_GEMM_PAIR", "1")
    cb, idx = synth.random_layer(F_out, F_in, 2, 256, seed=F_out + M)
    X = synth.activation(M, F_in, seed=3)
    L = F.import_layer(torch.from_numpy(cb).cuda(), torch.from_numpy(idx).cuda(), F_in)
    Xd = torch.from_numpy(X).cuda()
    Y = F.gemm(L, Xd, algo=F.GEMM_EXPAND_TC).float().cpu().numpy()
    rows = (F_out // 2 - 32, F_out // 2 + 32)
    Y_ref = oracle_lib.gemm(cb, idx, X[::97], rows=rows)
    ok, m = parity_ok(Y[::97, rows[0]:rows[1]], Y_ref, X[::97], F_in)
    assert ok, m
    monkeypatch.setenv("FASQ_GEMM_PAIR", "0")
    Y1 = F.gemm(L, Xd, algo=F.GEMM_EXPAND_TC).float().cpu().numpy()
    rel = np.linalg.norm(Y - Y1) / np.linalg.norm(Y1)
    assert rel <= 1e-6, rel


@pytest.mark.parametrize("F_out,F_in,M", [(4096, 4096, 32), (14336, 4096, 13), (4096, 14336, 64), (1000, 2048, 61),
                                          (4096, 4096, 128), (1024, 4096, 100), (14336, 4096, 29)])
def test_gemm_auto_short_L_runs_tcgen05_decode(F, oracle_lib, F_out, F_in, M):
    """Short-L prefill (NEXT-3): fasq_gemm AUTO at M up to the measured
    crossover (16 / 32 / 64 by shape) runs the tcgen05 decode kernel (weights as
    UMMA M), above it EXPAND with split-K (M = 128 / 100 / 29: one real
    accumulator per tile); sampled rows against the oracle and against the
    EXPAND kernel's Y."""
    cb, idx = synth.random_layer(F_out, F_in, 2, 256, seed=M)
    X = synth.activation(M, F_in, seed=M + 1)
    L = F.import_layer(torch.from_numpy(cb).cuda(), torch.from_numpy(idx).cuda(), F_in)
    Xd = torch.from_numpy(X).cuda()
    Y = F.gemm(L, Xd).float().cpu().numpy()
    rows = (F_out // 2 - 64, F_out // 2 + 64)
    ok, m = parity_ok(Y[:, rows[0]:rows[1]], oracle_lib.gemm(cb, idx, X, rows=rows), X, F_in)
    assert ok, m
    Ye = F.gemm(L, Xd, algo=F.GEMM_EXPAND_TC).float().cpu().numpy()
    assert np.linalg.norm(Y - Ye) / np.linalg.norm(Ye) <= 1e-5


@pytest.mark.parametrize("M", [1, 77, 128, 129, 255, 256, 257, 384, 640])
def test_gemm_tc_token_tile_edges(F, oracle_lib, M):
    """EXPAND's token tiling at every edge of its 256-token CTA tile: an odd
    token-tile count (row-major tiles, no phantom tile), tiles with <= 128 real
    tokens (one accumulator drained by both warp halves, no phantom workspace
    rows), split-K chosen automatically (few row tiles -> ks up to 8) and the
    column-major partial-tile merge; sampled rows at both ends and the middle
    against the oracle, and bit-identical repeats (fixed merge order)."""
    F_out, F_in = 768, 4096
    cb, idx = synth.random_layer(F_out, F_in, 2, 256, seed=M + 5)
    X = synth.activation(M, F_in, seed=M + 6)
    L = F.import_layer(torch.from_numpy(cb).cuda(), torch.from_numpy(idx).cuda(), F_in)
    Xd = torch.from_numpy(X).cuda()
    Y = F.gemm(L, Xd, out_dtype=torch.float32, algo=F.GEMM_EXPAND_TC)
    Y2 = F.gemm(L, Xd, out_dtype=torch.float32, algo=F.GEMM_EXPAND_TC)
    torch.cuda.synchronize()
    Yn = Y.cpu().numpy().astype(np.float64)
    assert np.array_equal(Yn, Y2.cpu().numpy().astype(np.float64))
    for r0 in (0, 352, F_out - 32):
        ok, m = parity_ok(Yn[:, r0:r0 + 32], oracle_lib.gemm(cb, idx, X, rows=(r0, r0 + 32)), X, F_in)
        assert ok, (r0, m)


@pytest.mark.parametrize("M,algo", [(128, "auto"), (300, "tc"), (2048, "tc"), (16, "auto")])
def test_gemm_grouped_qkv_gate_up(F, oracle_lib, M, algo):
    """fasq_gemm_grouped: q / k / v (4096 / 1024 / 1024 rows) and gate / up of
    one input.  Above the short-L crossover ONE EXPAND launch covers all row
    tiles (launch count 1 or 2 with a tail wave); at M = 16 AUTO runs one
    fasq_gemm per layer.  Each Y against the oracle on sampled rows, against
    the single-layer fasq_gemm (within the fp32 split-K rounding), and
    bit-identical on repeat."""
    a = F.GEMM_AUTO if algo == "auto" else F.GEMM_EXPAND_TC
    X = synth.activation(M, 4096, seed=M + 70)
    Xd = torch.from_numpy(X).cuda()
    for shapes in (((4096, 4096), (1024, 4096), (1024, 4096)), ((14336, 4096), (14336, 4096))):
        host, Ls = [], []
        for i, (fo, fi) in enumerate(shapes):
            cb, idx = synth.random_layer(fo, fi, 2, 256, seed=M + 10 * i + fo)
            host.append((cb, idx))
            Ls.append(F.import_layer(torch.from_numpy(cb).cuda(), torch.from_numpy(idx).cuda(), fi))
        Ys = F.gemm_grouped(Ls, Xd, algo=a)
        n_launch = F.last_launch_count()
        Ys2 = F.gemm_grouped(Ls, Xd, algo=a)
        torch.cuda.synchronize()
        if M >= 128:
            assert n_launch <= 2, n_launch
        for (cb, idx), L, Y, Y2 in zip(host, Ls, Ys, Ys2):
            Yn = Y.cpu().numpy().astype(np.float64)
            assert np.array_equal(Yn, Y2.cpu().numpy().astype(np.float64))
            fo = L.F_out
            for r0 in (0, fo // 2 + 64, fo - 64):
                ok, m = parity_ok(Yn[:, r0:r0 + 64], oracle_lib.gemm(cb, idx, X, rows=(r0, r0 + 64)), X, 4096)
                assert ok, (fo, r0, m)
            Ys1 = F.gemm(L, Xd, algo=a).cpu().numpy().astype(np.float64)
            assert np.linalg.norm(Yn - Ys1) / np.linalg.norm(Ys1) <= 1e-5


def test_gemm_grouped_errors(F):
    cb, idx = synth.random_layer(256, 512, 2, 16, seed=1)
    cb2, idx2 = synth.random_layer(256, 1024, 2, 16, seed=2)
    L1 = F.import_layer(torch.from_numpy(cb).cuda(), torch.from_numpy(idx).cuda(), 512)
    L2 = F.import_layer(torch.from_numpy(cb2).cuda(), torch.from_numpy(idx2).cuda(), 1024)
    X = torch.zeros((4, 512), dtype=torch.float16, device="cuda")
    with pytest.raises(F.FasqError) as e:
        F.gemm_grouped([L1, L2], X)
    assert e.value.code == -5


def test_split_k_workspace_shared_across_shapes(F):
    """The per-stream split-K workspace is shared by every layer and call: EXPAND
    (and the tcgen05 decode kernel) keep their arrive / depart tickets in a
    FIXED header, so a call after one with another tile count / K split can
    never find its counters on the earlier call's partial tiles.  Interleaved
    calls of different shapes, repeated: bit-identical every time (a misplaced
    ticket made the first call after a shape change race)."""
    cases = [(1024, 4096, 300), (4096, 4096, 300), (768, 4096, 129), (14336, 4096, 100), (4096, 14336, 200),
             (1024, 4096, 16), (4096, 4096, 24), (14336, 4096, 12)]
    layers, xs = [], []
    for i, (fo, fi, M) in enumerate(cases):
        cb, idx = synth.random_layer(fo, fi, 2, 256, seed=900 + i)
        layers.append(F.import_layer(torch.from_numpy(cb).cuda(), torch.from_numpy(idx).cuda(), fi))
        xs.append(torch.from_numpy(synth.activation(M, fi, seed=950 + i)).cuda())
    first = None
    for rep in range(3):
        order = list(range(len(cases)))
        if rep == 1:
            order.reverse()
        ys = {}
        for i in order:
            ys[i] = F.gemm(layers[i], xs[i], out_dtype=torch.float32).cpu()
        if first is None:
            first = ys
        else:
            for i in range(len(cases)):
                assert torch.equal(ys[i], first[i]), (rep, cases[i])


def test_gemm_grouped_fp16_and_lut_fallback(F, oracle_lib):
    """fasq_gemm_grouped with fp16 outputs (one EXPAND launch) and with the LUT
    algorithm (no grouped kernel: one fasq_gemm per layer, in order): each Y
    within tolerance of the oracle, and the fp16 grouped result equal to the
    per-layer fp16 EXPAND result to fp16 rounding."""
    M = 200
    X = synth.activation(M, 1024, seed=501)
    Xd = torch.from_numpy(X).cuda()
    host, Ls = [], []
    for i, fo in enumerate((768, 256, 256)):
        cb, idx = synth.random_layer(fo, 1024, 2, 64, seed=510 + i)
        host.append((cb, idx))
        Ls.append(F.import_layer(torch.from_numpy(cb).cuda(), torch.from_numpy(idx).cuda(), 1024))
    Yh = F.gemm_grouped(Ls, Xd, out_dtype=torch.float16, algo=F.GEMM_EXPAND_TC)
    Yl = F.gemm_grouped(Ls, Xd, algo=F.GEMM_LUT)
    torch.cuda.synchronize()
    for (cb, idx), L, yh, yl in zip(host, Ls, Yh, Yl):
        ref = oracle_lib.gemm(cb, idx, X)
        ok, m = parity_ok(yl.cpu().numpy().astype(np.float64), ref, X, 1024)
        assert ok, m
        y1 = F.gemm(L, Xd, out_dtype=torch.float16, algo=F.GEMM_EXPAND_TC).float().cpu().numpy()
        yg = yh.float().cpu().numpy()
        assert np.max(np.abs(yg - y1)) <= 2.0 ** -10 * (np.max(np.abs(y1)) + 1e-3)
