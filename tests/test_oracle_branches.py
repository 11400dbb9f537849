"""Pins for oracle a3: hue, the three branches and the AND merge.

Hue is pinned against the textbook hexagonal formula in exact rationals
(tests/brute.py) -- a different formulation from the oracle's integer sector
numerator -- plus the +120 degree cyclic-shift law and band rotation
invariance.
"""
from fractions import Fraction

import numpy as np

import oracle
from tests import brute


def _hue(r, g, b):
    hn, C = oracle.hue_num(r, g, b)
    return None if C == 0 else Fraction(hn, C)


def test_hue_spec_examples():
    assert _hue(255, 0, 0) == 0
    assert _hue(0, 255, 0) == 120
    assert _hue(77, 77, 77) is None
    assert _hue(10, 200, 30) == Fraction(24000, 190)


def test_hue_computed_values():                                # survey c3
    assert _hue(200, 120, 90) == Fraction(60 * 30, 110)
    assert _hue(200, 50, 60) == 356
    assert _hue(120, 95, 100) == 348
    assert _hue(255, 255, 0) == 60
    assert _hue(255, 0, 255) == 300
    assert _hue(0, 255, 255) == 180


def test_hue_matches_textbook_exact():
    rng = np.random.default_rng(3)
    trip = rng.integers(0, 256, (20000, 3))
    # plus every triple with small channel values (ties and sign cases)
    small = np.array(np.meshgrid(*[np.arange(0, 256, 51)] * 3)).reshape(3, -1).T
    for r, g, b in np.concatenate([trip, small]):
        h = _hue(int(r), int(g), int(b))
        t = brute.hue_textbook(int(r), int(g), int(b))
        assert h == t, (r, g, b, h, t)
        if h is not None:
            assert 0 <= h < 360


def test_hue_cyclic_shift_plus_120():
    rng = np.random.default_rng(4)
    for r, g, b in rng.integers(0, 256, (5000, 3)):
        h = _hue(int(r), int(g), int(b))
        h2 = _hue(int(b), int(r), int(g))
        if h is None:
            assert h2 is None
        else:
            assert h2 == (h + 120) % 360


def test_band_membership_exact_and_rotation():
    rng = np.random.default_rng(5)
    for _ in range(20000):
        r, g, b = (int(v) for v in rng.integers(0, 256, 3))
        a1, a2 = (int(v) for v in rng.integers(0, 360, 2))
        hn, C = oracle.hue_num(r, g, b)
        if C == 0:
            continue
        got = oracle.in_band(hn, C, a1, a2)
        h = Fraction(hn, C)
        assert got == int(brute.in_band_exact(h, a1, a2))


def test_band_rotation_invariance_integer_hues():
    # rotate hue and band together by d: membership is unchanged
    rng = np.random.default_rng(6)
    for _ in range(20000):
        hdeg, a1, a2, d = (int(v) for v in rng.integers(0, 360, 4))
        C = 1
        base = brute.in_band_exact(Fraction(hdeg), a1, a2)
        assert oracle.in_band(hdeg, C, a1, a2) == int(base)
        assert oracle.in_band((hdeg + d) % 360, C, (a1 + d) % 360, (a2 + d) % 360) == int(base)


def test_spec_band_examples():
    assert oracle.in_band(10, 1, 340, 25) == 1
    assert oracle.in_band(180, 1, 340, 25) == 0


def _frame_from_pixels(pix):
    pix = np.asarray(pix, np.uint8).reshape(1, -1, 3)
    return pix


def _stages(pix, lo, hi, **kw):
    f = _frame_from_pixels(pix)
    p = oracle.make_params(f.shape[1], 1, **kw)
    lo = np.broadcast_to(np.asarray(lo, np.uint8), f.shape).copy()
    hi = np.broadcast_to(np.asarray(hi, np.uint8), f.shape).copy()
    rec, st = oracle.segment(p, f, lo, hi)
    return rec, st


def test_branch_background_examples():
    rec, st = _stages([(140, 100, 100), (100, 100, 100), (90, 110, 95)], 90, 110)
    assert st["r1"].ravel().tolist() == [1, 0, 0]
    # identical frame, margin 0 -> all zero
    rng = np.random.default_rng(7)
    f = rng.integers(0, 256, (1, 40, 3), dtype=np.uint8)
    p = oracle.make_params(40, 1)
    rec, st = oracle.segment(p, f, f, f)
    assert not st["r1"].any()


def test_branch_gray_examples_reading_L5():
    pix = [(100, 100, 100), (200, 50, 50), (120, 95, 100)]
    _, st = _stages(pix, 0, 0, gray_tol_S=30)
    assert st["r2"].ravel().tolist()[:2] == [0, 1]
    _, st = _stages(pix, 0, 0, gray_tol_S=25)
    assert st["r2"].ravel().tolist()[2] == 1                   # paper: keep iff C >= S
    _, st = _stages(pix, 0, 0, gray_tol_S=26)
    assert st["r2"].ravel().tolist()[2] == 0                   # SPEC's strict rule = S+1


def test_merge_is_and_and_monotone():
    rng = np.random.default_rng(8)
    f = rng.integers(0, 256, (1, 3000, 3), dtype=np.uint8)
    lo = rng.integers(0, 128, (1, 3000, 3), dtype=np.uint8)
    hi = (lo.astype(int) + rng.integers(0, 128, (1, 3000, 3))).astype(np.uint8)
    p = oracle.make_params(3000, 1, se_radius=1)
    rec, st = oracle.segment(p, f, lo, hi)
    assert np.array_equal(st["merged"], st["r1"] & st["r2"] & st["r3"])
    assert rec.fg_merged == int(st["merged"].sum())
    prev = None
    for S in (0, 10, 30, 60, 120):
        _, s2 = oracle.segment(oracle.make_params(3000, 1, gray_tol_S=S), f, lo, hi)
        if prev is not None:
            assert (s2["r2"] <= prev).all()
        prev = s2["r2"]
    _, narrow = oracle.segment(oracle.make_params(3000, 1, hue_lo_deg=350, hue_hi_deg=15), f, lo, hi)
    _, wide = oracle.segment(oracle.make_params(3000, 1, hue_lo_deg=300, hue_hi_deg=40), f, lo, hi)
    assert (narrow["r3"] <= wide["r3"]).all()


def test_achromatic_never_skin_reading_L9():
    pix = [(v, v, v) for v in range(0, 256, 5)]
    _, st = _stages(pix, 0, 0, gray_tol_S=0, hue_lo_deg=0, hue_hi_deg=359)
    assert not st["r3"].any()
