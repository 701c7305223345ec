"""Size / bit-rate invariants (Eq. 4-5, #W) -- not GPU."""
import math

import numpy as np
import pytest

import synth
from oracle import sizemodel as sm


def test_eff_bits_table2(pins):
    for key, want in pins["eff_bits_W"].items():
        if key.startswith("_"):
            continue
        d, C = map(int, key.split("-"))
        assert sm.eff_bits(d, C) == want


def test_paper_size_percent_reproduced(pins):
    archs = {"Llama-3-8B": sm.LLAMA3_8B, "Qwen3-8B": sm.QWEN3_8B,
             "LLaMA-2-7B": sm.LLAMA2_7B, "LLaMA-2-13B": sm.LLAMA2_13B}
    n = 0
    for name, table in pins["size_percent"].items():
        if name.startswith("_"):
            continue
        for key, printed in table.items():
            d, C = map(int, key.split("-"))
            got = sm.model_size_percent_paper_fit(archs[name], d, C)
            assert abs(got - printed) <= 0.15, (name, key, got, printed)
            n += 1
    assert n == 17


def test_fp16_model_bytes(pins):
    mib = sm.LLAMA3_8B.fp16_bytes() / 2**20
    assert round(mib) == pins["fp16_llama3_8b_MB"]["value"]


def test_our_storage_inside_paper_range(pins):
    lo, hi = pins["size_range_percent"]["lo"], pins["size_range_percent"]["hi"]
    for d, C in [(2, 256), (2, 128)]:          # the paper's eff. 4-bit / 3-bit
        p = sm.model_size_percent_ours(sm.LLAMA3_8B, d, C)
        assert lo <= p <= hi, (d, C, p)


@pytest.mark.parametrize("F_out,F_in,d,C,group", [(4096, 4096, 2, 256, 1), (1024, 4096, 2, 256, 1),
                                                  (256, 512, 4, 256, 128), (4096, 14336, 2, 128, 1)])
def test_bits_per_weight_closed_form(F_out, F_in, d, C, group):
    sb = sm.stored_bytes(F_out, F_in, d, C, group)
    bpw = 8 * sb["total_bytes"] / (F_out * F_in)
    assert bpw == pytest.approx(sm.bits_per_weight(F_out, F_in, d, C, group), rel=1e-15)


def test_stored_bytes_match_packed_arrays(oracle_lib):
    W = synth.weight(64, 32, seed=1)
    cb, idx, _ = oracle_lib.pack(W, d=2, C=16, group=2, seed=0, iters=3)
    sb = sm.stored_bytes(64, 32, 2, 16, 2)
    assert cb.nbytes == sb["codebook_bytes"] and idx.nbytes == sb["index_bytes"]


def test_paper_traffic_arithmetic(pins):
    p = pins["index_bytes_4096"]
    assert sm.stored_bytes(4096, 4096, 2, 256)["index_bytes"] == p["sz2_MiB"] * 2**20
    assert sm.stored_bytes(4096, 4096, 1, 256)["index_bytes"] == p["sz1_MiB"] * 2**20
    assert 4096 * 4096 * 2 == p["fp16_MiB"] * 2**20
    assert 256 * 2 * 2 == pins["codebook_per_subspace_bytes_2_256"]["value"]
    assert round(100 * 255 / 256, 1) == pins["lut_waste_percent_256"]["value"]
    # Eq. 4 at 4096^2 (2,256): 16*256*4096 + 8*2048*4096 bits
    assert sm.eq4_layer_bits(256, 4096, 2048, 4096) == 16 * 256 * 4096 + 8 * 2048 * 4096


def test_paper_split_planner(pins):
    s = pins["split_k"]
    assert sm.paper_split_k(s["n_sm"], s["blocks_per_sm"], s["batch"], s["f_out"]) == s["value"]
    assert sm.paper_split_k(82, 8, 1, 4096, n_ss=8) == 8          # SPEC S:182 clamp
    assert sm.paper_split_k(1, 1, 1, 128, n_ss=2048) == 1
