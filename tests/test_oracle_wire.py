"""Pins for the oracle's fp16 factor wire (NEXT-4(ii); "half precision floating point numbers
for both computation ...", reading R-23): oracle.wire_fp16 against IEEE 754 binary16 facts worked by
hand (11-bit significand, ties to even, largest finite 65504, smallest subnormal 2^-24, overflow to
inf), and oracle.reduce_scatter(wire=...) against the definition of a mean of wire values."""
import math

import numpy as np
import pytest

from synth import shapes


# (x, expected binary16 value): each worked from the format, not from a conversion routine
HAND = [
    (1.0, 1.0),
    (1 + 2 ** -10, 1 + 2 ** -10),          # ulp(1) = 2^-10: representable
    (1 + 2 ** -11, 1.0),                   # halfway 1 | 1+2^-10, tie -> even significand (1)
    (1 + 3 * 2 ** -11, 1 + 2 ** -9),       # halfway 1+2^-10 (odd) | 1+2^-9 (even) -> 1+2^-9
    (1 + 2 ** -11 + 2 ** -20, 1 + 2 ** -10),  # just above the tie -> up
    (-(1 + 2 ** -11), -1.0),               # sign-symmetric
    (2049.0, 2048.0),                      # ulp(2048) = 2: 2049 is a tie -> even (2048)
    (2051.0, 2052.0),                      # tie between 2050 (odd significand) and 2052 -> 2052
    (65504.0, 65504.0),                    # largest finite
    (65519.99, 65504.0),                   # below the overflow threshold 65520
    (65520.0, math.inf),                   # halfway to 2^16 -> rounds to inf
    (2.0 ** -14, 2.0 ** -14),              # smallest normal
    (2.0 ** -24, 2.0 ** -24),              # smallest subnormal
    (2.0 ** -25, 0.0),                     # halfway 0 | 2^-24 -> even (0)
    (3 * 2.0 ** -26, 2.0 ** -24),          # 0.75 ulp -> up
    (5 * 2.0 ** -24 + 2.0 ** -25, 6 * 2.0 ** -24),  # subnormal tie 5 | 6 -> even (6)
    (0.1, 1638.0 / 16384.0),               # 0.1 = 1.6 * 2^-4, significand 1638.4/1024 -> 1638 * 2^-14
]


@pytest.mark.parametrize("x,want", HAND)
def test_wire_fp16_hand_values(orc, x, want):
    assert orc.wire_fp16(np.array([x]))[0] == want


def test_wire_fp16_scale_is_exact(orc):
    # a power-of-two scale moves the value into the normal range and back without extra error
    x = np.array([3 * 2.0 ** -30, 1 + 2 ** -11, 7.0 * 2 ** 20])
    got = orc.wire_fp16(x, 2.0 ** 10)
    assert got[0] == 3 * 2.0 ** -30                       # 3*2^-20 is a subnormal half: exact
    assert got[1] == 1.0                                  # 1024 + 0.5 tie -> 1024
    assert math.isinf(got[2])                             # 7 * 2^30 overflows
    assert orc.wire_fp16(np.array([3 * 2.0 ** -30]))[0] == 0.0  # unscaled: below 2^-25 -> 0
    with pytest.raises(ValueError):
        orc.wire_fp16(x, 3.0)


def test_wire_fp16_error_bound_and_idempotence(orc):
    # normal range: |wire(x) - x| <= 2^-11 |x| (half an ulp of an 11-bit significand); wire(wire(x)) = wire(x)
    rng = np.random.default_rng(23)
    x = rng.standard_normal(100000) * np.exp2(rng.integers(-12, 14, 100000))
    x = x[(np.abs(x) >= 2.0 ** -14) & (np.abs(x) < 65504)]  # the normal range
    w = orc.wire_fp16(x)
    assert np.all(np.abs(w - x) <= 2.0 ** -11 * np.abs(x))
    assert np.array_equal(orc.wire_fp16(w), w)
    # every result has at most 11 significant bits
    m, _ = np.frexp(w[w != 0])
    assert np.all(m * 2 ** 11 == np.round(m * 2 ** 11))


def _layers():
    return [shapes.conv("a", 4, 8, 3, 1, 1, 5, bias=1), shapes.linear("fc", 12, 6), shapes.conv("b", 8, 8, 1, 1, 0, 5)]


@pytest.mark.parametrize("P", [1, 2, 3])
def test_reduce_scatter_wire(orc, P):
    layers = _layers()
    pl = orc.plan(layers, P, orc.POLICY_RR)
    rng = np.random.default_rng(P)
    sends = [rng.standard_normal(P * pl["rs_chunk"]) for _ in range(P)]
    sc = (2.0 ** 3, 2.0 ** -2)
    exact = orc.reduce_scatter(sends, pl)
    got = orc.reduce_scatter(sends, pl, wire=sc, layers=layers)
    for r in range(P):
        for l, (o_w, o_a, o_g) in pl["local"][r].items():
            a, g = orc.dims(layers[l])
            # dW: fp32 wire, the exact mean
            assert np.array_equal(got[r][o_w:o_w + g * a], exact[r][o_w:o_w + g * a])
            for o, n, s in ((o_a, a, sc[0]), (o_g, g, sc[1])):
                seg = slice(o, o + n * (n + 1) // 2)
                # within one wire rounding per contribution of the exact mean (|wire(x) - x| <= 2^-11 |x|)
                bound = 2.0 ** -11 * sum(np.abs(sends[q][r * pl["rs_chunk"]:][seg]) for q in range(P)) / P
                assert np.all(np.abs(got[r][seg] - exact[r][seg]) <= bound)
                # every contribution is on the fp16 grid: P * mean * scale is a sum of P binary16 values,
                # an integer multiple of 2^-24 (the smallest subnormal) -- and not the unrounded sum
                tot = got[r][seg] * P * s
                assert np.all(np.abs(tot * 2.0 ** 24 - np.round(tot * 2.0 ** 24)) <= 1e-6 * np.abs(tot * 2.0 ** 24))
                assert not np.array_equal(got[r][seg], exact[r][seg])
    if P == 1:  # one rank: the wire is one rounding of the factor
        for l, (o_w, o_a, o_g) in pl["local"][0].items():
            a, g = orc.dims(layers[l])
            assert np.array_equal(got[0][o_a:o_a + a * (a + 1) // 2],
                                  orc.wire_fp16(sends[0][o_a:o_a + a * (a + 1) // 2], sc[0]))
