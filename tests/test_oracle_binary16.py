"""Pins for oracle.binary16 (the fp16 wire codec, reading R7).

Pinned against: the binary16 format definition (hand-decoded patterns), NumPy's
independent float16 conversion (a library routine the oracle does not call), the
format's rounding-error bound, and monotonicity.
"""
import os

import numpy as np
import pytest

from oracle import binary16 as b16


@pytest.mark.parametrize("x,bits", [
    (1.0, 0x3C00),                      # SPEC S:55 / format definition
    (0.0, 0x0000),
    (-0.0, 0x8000),
    (1.0 + 2.0 ** -10, 0x3C01),          # one ulp above 1
    (1.0 + 2.0 ** -11, 0x3C00),          # exact tie -> even (RNE)
    (1.0 + 3 * 2.0 ** -11, 0x3C02),      # tie between 0x3C01 and 0x3C02 -> even
    (2.0 ** -24, 0x0001),                # smallest subnormal
    (2.0 ** -25, 0x0000),                # tie with zero -> even (0)
    (3 * 2.0 ** -25, 0x0002),            # tie between 1 and 2 quanta -> even
    (2.0 ** -14, 0x0400),                # smallest normal
    (2.0 ** -14 - 2.0 ** -25, 0x0400),   # tie between largest subnormal and smallest normal
    (65504.0, 0x7BFF),                   # largest finite
    (65519.99, 0x7BFF),
    (-2.0, 0xC000),
    (0.1, 0x2E66),                       # 0.1 = 1.6 * 2^-4 -> fraction round(0.6*1024)=614=0x266
])
def test_known_patterns(x, bits):
    assert int(b16.to_binary16(x)) == bits


def test_saturation_counted():
    out, n = b16.to_binary16(np.array([65504.0, 65505.0, 65520.0, -1e9, 3.0]), return_saturation=True)
    assert list(out) == [0x7BFF, 0x7BFF, 0x7BFF, 0xFBFF, 0x4200]
    assert n == 3   # |x| > 65504


def test_nonfinite_raises_first_index():
    with pytest.raises(b16.NonFiniteError) as e:
        b16.to_binary16(np.array([1.0, 2.0, np.inf, np.nan]))
    assert e.value.index == 2


def test_from_binary16_exhaustive_vs_numpy():
    bits = np.arange(65536, dtype=np.uint32).astype(np.uint16)
    ref = bits.view(np.float16).astype(np.float64)
    ok = ~np.isnan(ref)
    got = b16.from_binary16(bits[ok])
    assert np.array_equal(got, ref[ok])
    assert np.array_equal(np.signbit(got), np.signbit(ref[ok]))
    with pytest.raises(b16.NonFiniteError):
        b16.from_binary16(np.array([0x7E00], dtype=np.uint16))


def test_known_decodes():
    assert b16.from_binary16(np.uint16(0x0001)) == 2.0 ** -24
    assert b16.from_binary16(np.uint16(0x3C00)) == 1.0
    assert b16.from_binary16(np.uint16(0x7BFF)) == 65504.0


def _numpy_ref(x32):
    """NumPy's float32->float16 (RNE) plus the saturation reading."""
    with np.errstate(over="ignore"):
        h = x32.astype(np.float16)
    h = np.where(np.isinf(h), np.copysign(np.float16(65504.0), x32), h).astype(np.float16)
    return h.view(np.uint16)


def _check_patterns(pat):
    x = pat.view(np.float32)
    x = x[np.isfinite(x)]
    got = b16.to_binary16(x.astype(np.float64))
    ref = _numpy_ref(x)
    bad = np.nonzero(got != ref)[0]
    assert bad.size == 0, (x[bad[:5]], got[bad[:5]], ref[bad[:5]])


def test_vs_numpy_random_fp32_patterns():
    r = np.random.default_rng(5)
    _check_patterns(r.integers(0, 2 ** 32, 2 ** 21, dtype=np.uint64).astype(np.uint32))


def test_vs_numpy_all_fp32_in_fp16_range_strided():
    # every fp32 pattern whose exponent lies in the range fp16 resolves
    # (2^-26 .. 2^16), low mantissa bits strided: covers every rounding boundary
    # class (below/at/above tie) in every binade.
    exps = np.arange(127 - 26, 127 + 17, dtype=np.uint32)
    mant = np.concatenate([np.arange(0, 1 << 23, 4093, dtype=np.uint32),
                           # around every binary16 tie: fraction bits 12..0 = 0x1000 +- 2
                           ((np.arange(1 << 10, dtype=np.uint32) << 13)[:, None]
                            + np.array([0xFFE, 0xFFF, 0x1000, 0x1001, 0x1002], dtype=np.uint32)).ravel()])
    pat = (exps[:, None] << 23 | mant[None, :]).ravel()
    _check_patterns(pat)
    _check_patterns(pat | np.uint32(0x80000000))


@pytest.mark.slow
@pytest.mark.skipif(os.environ.get("LMSGD_EXHAUSTIVE") != "1", reason="set LMSGD_EXHAUSTIVE=1")
def test_vs_numpy_all_fp32_patterns():
    for hi in range(0, 1 << 32, 1 << 24):
        _check_patterns(np.arange(hi, hi + (1 << 24), dtype=np.uint64).astype(np.uint32))


def test_roundtrip_bound():
    # |from(to(x)) - x| <= max(2^-11 |x|, 2^-24) for |x| <= 65504
    r = np.random.default_rng(6)
    x = np.concatenate([r.standard_normal(10 ** 6) * 10.0 ** r.uniform(-9, 4.5, 10 ** 6),
                        r.uniform(-65504, 65504, 10 ** 5)])
    x = x[np.abs(x) <= 65504]
    y = b16.from_binary16(b16.to_binary16(x))
    assert np.all(np.abs(y - x) <= np.maximum(2.0 ** -11 * np.abs(x), 2.0 ** -24))


def test_monotone():
    x = np.sort(np.random.default_rng(7).uniform(0, 70000, 10 ** 5))
    bits = b16.to_binary16(x).astype(np.int64)
    assert np.all(np.diff(bits) >= 0)
