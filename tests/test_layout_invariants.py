"""Host-side checks of the decode kernels' SMEM mapping invariants
(gemv_core.cuh, DESIGN.md "Row-set mapping" and "Codebook pair stages").

The formulas are restated here from DESIGN.md (no device code is imported):

* index stage, per (64-row block, subspace s): 64 bytes at s*64, the 16-row chunk
  c stored at 16-B position (c + s//2) & 3 (fasq_internal.cuh idx_offset);
* row-set mapping with G lanes per set: lane l = G*a + u owns rows
  {G*a + t, 32 + G*a + t : t < G} of its warp's 64 and, in phase p, subspace
  sigma = G*((a + p) % (32//G)) + u;
* codebook pair stage: the gather address of (k, half h, subspace s) is
  (k << 8) | (h*128 + 4*s), i.e. bank s whatever k is.
"""
import itertools

import pytest


def idx_byte_offset(row, s):
    """Byte of (row in a 64-row block, subspace s) inside the block's 2 KiB."""
    c, r = row >> 4, row & 15
    return s * 64 + 16 * ((c + (s >> 1)) & 3) + r


def set_rows(G, lane):
    a, u = lane // G, lane % G
    return [G * a + t for t in range(G)] + [32 + G * a + t for t in range(G)]


def set_sigma(G, lane, p):
    a, u = lane // G, lane % G
    return G * ((a + p) % (32 // G)) + u


@pytest.mark.parametrize("G", [2, 4, 8])
def test_row_set_phases_are_permutations_and_cover_every_pair_once(G):
    K = 32 // G
    seen = set()
    for p in range(K):
        sig = [set_sigma(G, lane, p) for lane in range(32)]
        assert sorted(sig) == list(range(32))      # 32 distinct subspaces -> 32 distinct banks per gather
        for lane in range(32):
            for row in set_rows(G, lane):
                pair = (row, sig[lane])
                assert pair not in seen
                seen.add(pair)
    assert len(seen) == 64 * 32                    # every (row, subspace) of the warp exactly once


@pytest.mark.parametrize("G", [2, 4, 8])
def test_row_set_reduction_leaves_lane_rows_l_and_32_plus_l(G):
    # register (2*(t % G) + t // G) accumulates set row t; a transposed butterfly over
    # the G lanes of the set (masks G/2 .. 1) keeps, for lane u, registers
    # i + (2u) .. i.e. set rows u and G + u -> warp rows lane and 32 + lane
    for lane in range(32):
        a, u = lane // G, lane % G
        regs = {2 * (t % G) + t // G: set_rows(G, lane)[t] for t in range(2 * G)}
        kept = [regs[2 * u + h] for h in range(2)]
        assert kept == [lane, 32 + lane]


@pytest.mark.parametrize("G,wavefront_lanes,width", [(8, 16, 8), (4, 32, 4), (2, 32, 2)])
def test_row_set_index_loads_at_most_two_way_conflicts(G, wavefront_lanes, width):
    """Index bytes of (sigma_p, G rows): G = 8 -> LDS.64 (16 lanes per wavefront),
    G = 4 -> LDS.32, G = 2 -> LDS.U16.  Conflict-free for G = 8, <= 2-way otherwise."""
    worst = 0
    for p, part in itertools.product(range(32 // G), range(2)):
        for w0 in range(0, 32, wavefront_lanes):
            banks = {}
            for lane in range(w0, w0 + wavefront_lanes):
                sg = set_sigma(G, lane, p)
                row0 = set_rows(G, lane)[G * part]
                addr = idx_byte_offset(row0, sg)
                assert all(idx_byte_offset(row0 + t, sg) == addr + t for t in range(G))   # contiguous bytes
                for wd in range(addr // 4, (addr + width - 1) // 4 + 1):
                    banks.setdefault(wd % 32, set()).add(wd // 32)
            worst = max(worst, max(len(v) for v in banks.values()))
    assert worst == (1 if G == 8 else 2)


def test_lane_subspace_index_chunks_conflict_free():
    # the lane = subspace loop's LDS.128 (16 rows of subspace s): every quarter-warp
    # hits 8 distinct 16-B bank groups
    for c in range(4):
        for q0 in range(0, 32, 8):
            groups = {(idx_byte_offset(16 * c, s) // 16) % 8 for s in range(q0, q0 + 8)}
            assert len(groups) == 8


def test_pair_stage_gather_hits_bank_s_for_any_k():
    for k, h in itertools.product((0, 1, 77, 128, 255), (0, 1)):
        banks = [(((k << 8) | (h * 128 + 4 * s)) // 4) % 32 for s in range(32)]
        assert banks == list(range(32))


# ---- host-only chain planner (K-split counts must fit the 6-bit
# counted-word field for the full Llama shapes at every world size) ----------
def test_chain_planner_llama_shapes_all_world_sizes():
    import paper_2605_04084_b200 as F
    blocks = {"qkv": [(4096, 4096), (1024, 4096), (1024, 4096)], "o": [(4096, 4096)],
              "gateup": [(14336, 4096), (14336, 4096)], "down": [(4096, 14336)]}
    for world in (1, 2, 4, 8):
        for nctas in (148, 148 // world):
            for B in (1, 2, 4, 8):
                for name, shapes in blocks.items():
                    # row shards (q/k/v, gate/up) and Megatron K shards (o, down)
                    if name in ("o", "down"):
                        sh = [(fo, fi // world) for fo, fi in shapes]
                    else:
                        sh = [(fo // world, fi) for fo, fi in shapes]
                    ks = F.plan_ks(sh, nctas=nctas, d=2, B=B)
                    assert all(1 <= k <= 63 for k in ks), (world, nctas, B, name, ks)
                    full = F.plan_ks(shapes, nctas=nctas, d=2, B=B)
                    assert all(1 <= k <= 63 for k in full), (world, nctas, B, name, full)
