"""Pins of the oracle's binary16 conversions and PRNG (not GPU).

fp32 -> fp16 roundTiesToEven is pinned against numpy's float32->float16 cast
(a library routine implementing IEEE roundTiesToEven) on a structured cover of
every exponent/rounding case plus 16M random patterns.  fp16 -> fp32 is pinned exhaustively (2^16)
against numpy too.  splitmix64 is pinned by its published reference outputs.
"""
import numpy as np
import pytest


def test_f16_to_f32_exhaustive(oracle_lib):
    h = np.arange(1 << 16, dtype=np.uint32).astype(np.uint16)
    ours = oracle_lib.f16_bits_to_f32(h)
    ref = h.view(np.float16).astype(np.float32)
    nan = np.isnan(ref)
    assert np.array_equal(np.isnan(ours), nan)
    assert np.array_equal(ours[~nan].view(np.uint32), ref[~nan].view(np.uint32))


def _f32_cases():
    """Structured cover of fp32 -> fp16 rounding: every (sign, exponent, top-10
    mantissa bits) with the low-13-bit patterns that decide rounding (exact,
    just below/at/above the tie, max), every exponent whose result is a
    binary16 subnormal with all of its top-16 mantissa bits, and 16M uniformly
    random bit patterns.  (A full 2^32 sweep costs ~8 min with numpy's cast.)"""
    se = np.arange(512, dtype=np.uint32) << 23
    top = np.arange(1024, dtype=np.uint32) << 13
    low = np.array([0, 1, 0x7FF, 0xFFF, 0x1000, 0x1001, 0x17FF, 0x1FFF], np.uint32)
    a = (se[:, None, None] | top[None, :, None] | low[None, None, :]).ravel()
    sub_e = np.arange(100, 114, dtype=np.uint32) << 23
    m16 = np.arange(1 << 16, dtype=np.uint32) << 7
    b = (sub_e[:, None] | m16[None, :]).ravel()
    b = np.concatenate([b, b | 0x40, b | 0x3F, b | (1 << 31)])
    c = np.random.Generator(np.random.PCG64(7)).integers(0, 1 << 32, size=1 << 24, dtype=np.uint64).astype(np.uint32)
    return np.concatenate([a, b, c])


def test_f32_to_f16_vs_numpy(oracle_lib):
    bits = _f32_cases()
    f = bits.view(np.float32)
    ours = oracle_lib.f32_to_f16_bits(f)
    with np.errstate(over="ignore", invalid="ignore"):
        ref = f.astype(np.float16).view(np.uint16)
    nan = np.isnan(f)
    # NaN payloads are unspecified; both must still be NaN
    assert np.all((ours[nan] & 0x7C00) == 0x7C00) and np.all((ours[nan] & 0x3FF) != 0)
    bad = np.nonzero(ours[~nan] != ref[~nan])[0]
    assert bad.size == 0, [hex(int(x)) for x in bits[~nan][bad[:5]]]


def test_f32_to_f16_ties_and_boundaries(oracle_lib):
    # hand-picked cases from the binary16 definition
    cases = [
        (0.0, 0x0000), (-0.0, 0x8000), (1.0, 0x3C00), (65504.0, 0x7BFF),
        (65519.99, 0x7BFF), (65520.0, 0x7C00),             # overflow threshold
        (2.0 ** -24, 0x0001), (2.0 ** -25, 0x0000),        # tie to even (0)
        (1.5 * 2.0 ** -24, 0x0002),                        # tie 1.5 ulp -> 2 (even)
        (2.0 ** -14, 0x0400),                              # min normal
        (1.0 + 2.0 ** -11, 0x3C00),                        # tie -> even (1.0)
        (1.0 + 3 * 2.0 ** -11, 0x3C02),                    # tie -> even (1+2^-9)
    ]
    for v, h in cases:
        assert int(oracle_lib.lib().fasq_ref_f32_to_f16(v)) == h, (v, hex(h))


def test_splitmix64_reference_vectors(oracle_lib, pins):
    want = [int(v, 16) for v in pins["splitmix64_seed0"]["values"]]
    assert oracle_lib.splitmix64(0, 3) == want
