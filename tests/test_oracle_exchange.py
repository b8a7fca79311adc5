"""Pins for oracle.exchange (readings R7-R11).

Pinned against: exact rational arithmetic (fractions.Fraction brute force on small
inputs), NumPy's float16 conversion for the k = 1 round trip, algebraic special
cases (identical payloads, integer payloads, permutations), and the rigorous
rounding-error bound of the two fp16 roundings.
"""
import itertools
from fractions import Fraction

import numpy as np
import pytest

from oracle import binary16 as b16
from oracle import exchange as ex


def _rand_fp16_bits(r, shape, lo=-24, hi=15):
    x = r.standard_normal(shape) * 2.0 ** r.integers(lo, hi, shape)
    return b16.to_binary16(np.clip(x, -65504, 65504))


def test_reduce_is_exact_rational_sum():
    r = np.random.default_rng(1)
    for k in (1, 2, 3, 5, 8):
        h = [_rand_fp16_bits(r, 400) for _ in range(k)]
        S = ex.reduce_sum(h)
        for j in range(400):
            exact = sum(Fraction(float(b16.from_binary16(hi[j]))) for hi in h)
            assert Fraction(float(S[j])) == exact


def test_reduce_exact_adversarial():
    # largest magnitude with smallest subnormal: needs all 40 bits
    big, tiny = b16.to_binary16(65504.0), b16.to_binary16(2.0 ** -24)
    h = [np.array([big, tiny, big], dtype=np.uint16), np.array([tiny, big, b16.to_binary16(-65504.0)],
                                                              dtype=np.uint16)]
    S = ex.reduce_sum(h)
    assert S[0] == 65504.0 + 2.0 ** -24 and S[1] == 65504.0 + 2.0 ** -24 and S[2] == 0.0


def test_k1_roundtrip_matches_numpy_float16():
    r = np.random.default_rng(2)
    g = (r.standard_normal(10 ** 5) * 10.0 ** r.uniform(-6, -1, 10 ** 5)).astype(np.float32)
    for s in (1.0, 1024.0):
        res = ex.exchange([g], s)
        ref = ((np.float32(s) * g).astype(np.float16).astype(np.float32)) * np.float32(1.0 / s)
        assert np.array_equal(res.ghat, ref)


def test_identical_payloads_average_to_themselves():
    r = np.random.default_rng(3)
    h = b16.from_binary16(_rand_fp16_bits(r, 1000, -20, 10)).astype(np.float32)   # fp16-exact values
    for k in (2, 4, 8):
        res = ex.exchange([h] * k, 1.0)
        assert np.array_equal(res.ghat, h)


def test_integer_payloads_exact():
    r = np.random.default_rng(4)
    g = [r.integers(-200, 200, 500).astype(np.float32) for _ in range(5)]
    res = ex.exchange(g, 1.0)
    exact = np.sum(g, axis=0).astype(np.float64)
    assert np.array_equal(res.S, exact)
    assert np.array_equal(res.R, b16.to_binary16(exact))


def test_permutation_invariance_bitwise():
    r = np.random.default_rng(5)
    g = [(r.standard_normal(2000) * 1e-3).astype(np.float32) for _ in range(4)]
    base = ex.exchange(g, 1024.0)
    for perm in itertools.permutations(range(4)):
        res = ex.exchange([g[i] for i in perm], 1024.0)
        assert np.array_equal(res.ghat, base.ghat) and np.array_equal(res.R, base.R)


@pytest.mark.parametrize("k,s", [(1, 1.0), (2, 1.0), (4, 1024.0), (8, 1024.0), (8, 1.0), (3, 16.0)])
def test_wire_error_bound(k, s):
    """|ghat - ideal| <= (2^-11 sum|s g_i| + k 2^-25 + 2^-11 |S| + 2^-25) / (k s) + fp32 unpack
    rounding (2^-24 |ghat|): each fp16 rounding errs by at most half an ulp."""
    r = np.random.default_rng(6)
    g = [(r.standard_normal(20000) * 10.0 ** r.uniform(-6, -1, 20000)).astype(np.float32)
         for _ in range(k)]
    res = ex.exchange(g, s)
    ideal = ex.ideal(g)
    bound = (2.0 ** -11 * np.sum(np.abs(np.array(g, dtype=np.float64)) * s, axis=0)
             + k * 2.0 ** -25 + 2.0 ** -11 * np.abs(res.S) + 2.0 ** -25) / (k * s) \
        + 2.0 ** -24 * np.abs(res.ghat.astype(np.float64))
    assert np.all(np.abs(res.ghat - ideal) <= bound)


def test_saturation_counts():
    g = [np.array([70000.0, 40000.0, 1.0], dtype=np.float32),
         np.array([-1.0, 40000.0, 1.0], dtype=np.float32)]
    res = ex.exchange(g, 1.0)
    assert res.pack_saturations == 1          # 70000 > 65504 at pack
    assert res.sum_saturations == 1           # 40000 + 40000 > 65504 at wire-2
    assert b16.from_binary16(res.R[1]) == 65504.0
    assert res.ghat[2] == 1.0


def test_nonfinite_raises_first_index():
    g = np.ones(10, dtype=np.float32)
    g[7] = np.nan
    g[9] = np.inf
    with pytest.raises(b16.NonFiniteError) as e:
        ex.exchange([np.ones(10, dtype=np.float32), g])
    assert e.value.index == 7


def test_loss_scale_must_be_power_of_two():
    with pytest.raises(ValueError):
        ex.exchange([np.ones(4, dtype=np.float32)], 3.0)
    with pytest.raises(ValueError):
        ex.exchange([np.ones(4, dtype=np.float32)], 0.0)


def test_loss_scale_reduces_subnormal_loss():
    # R11: s = 2^10 keeps small gradients out of the fp16 subnormal range
    g = np.full(4, 3e-6, dtype=np.float32)
    e1 = abs(float(ex.exchange([g], 1.0).ghat[0]) - 3e-6) / 3e-6
    e2 = abs(float(ex.exchange([g], 1024.0).ghat[0]) - 3e-6) / 3e-6
    assert e2 < 2.0 ** -11 < e1


def test_nonfinite_index_is_minimum_over_workers():
    # R7: the smallest flat index at which ANY worker is non-finite
    a = np.ones(100, dtype=np.float32)
    b = np.ones(100, dtype=np.float32)
    a[60] = np.nan
    b[25] = np.inf
    with pytest.raises(b16.NonFiniteError) as e:
        ex.exchange([a, b])
    assert e.value.index == 25


# ------------------------------------------------------------------ pins of exchange.ideal
# ideal(g) = sum_i g_i / k in float64 (the no-wire reference the fp16 deviation is
# reported against).  Pinned to exact rational arithmetic, a fixed point and the
# cases where the fp16 wire is exact.

def test_ideal_matches_exact_rational_mean():
    from fractions import Fraction
    r = np.random.default_rng(21)
    for k in (1, 2, 3, 5, 8):
        g = [(r.standard_normal(64) * 10.0 ** r.uniform(-6, 2, 64)).astype(np.float32) for _ in range(k)]
        got = ex.ideal(g)
        for j in range(64):
            exact = sum(Fraction(float(gi[j])) for gi in g) / k
            absum = sum(abs(Fraction(float(gi[j]))) for gi in g) / k
            # k - 1 float64 additions and one division, each within half an ulp
            assert abs(Fraction(float(got[j])) - exact) <= Fraction(k + 1, 2 ** 53) * absum, (k, j)


def test_ideal_of_identical_workers_is_the_gradient():
    g = (np.random.default_rng(22).standard_normal(1000) * 1e-3).astype(np.float32)
    for k in (1, 2, 3, 4, 8):
        assert np.array_equal(ex.ideal([g] * k), g.astype(np.float64))


def test_ideal_equals_ghat_where_the_wire_is_exact():
    # small integer gradients at s = 1: every pack, sum and 1/k (k a power of two) is exact
    r = np.random.default_rng(23)
    for k in (1, 2, 4, 8):
        g = [r.integers(-100, 101, 500).astype(np.float32) for _ in range(k)]
        assert np.array_equal(ex.exchange(g, 1.0).ghat.astype(np.float64), ex.ideal(g))


def test_ideal_is_permutation_invariant_and_linear():
    r = np.random.default_rng(24)
    g = [(r.standard_normal(300) * 1e-2).astype(np.float32) for _ in range(4)]
    base = ex.ideal(g)
    for perm in itertools.permutations(range(4)):
        assert np.allclose(ex.ideal([g[i] for i in perm]), base, rtol=4 * 2.0 ** -52, atol=0)
    assert np.array_equal(ex.ideal([x * np.float32(2.0) for x in g]), 2.0 * base)   # power-of-two scaling
