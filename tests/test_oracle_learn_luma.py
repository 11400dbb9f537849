"""Pins for oracle a1 (background learning) and a2 (brightness correction).

a1: S:135-143 examples, S:452, S:164-165 invariants.
a2: closed forms of the integer mean (Rec.601 weights sum to 1000), S:200-202,
    readings L19-L22, and the LUT pinned by exact rational bracketing for
    rational gammas (no pow) -- tests/brute.py.
"""
import math
from fractions import Fraction

import numpy as np
import pytest

import oracle
from tests import brute


# ------------------------------------------------------------------ a1 learn
def test_learn_identical_frames_margin0():
    rng = np.random.default_rng(1)
    f = rng.integers(0, 256, (6, 5, 3), dtype=np.uint8)
    lo, hi = oracle.learn(np.stack([f] * 10), 0)
    assert np.array_equal(lo, f) and np.array_equal(hi, f)


def test_learn_alternating_margin5():
    frames = np.zeros((8, 4, 4, 3), np.uint8)
    frames[0::2] = 100
    frames[1::2] = 110
    lo, hi = oracle.learn(frames, 5)
    assert (lo == 95).all() and (hi == 115).all()


def test_learn_saturates():
    frames = np.zeros((3, 2, 2, 3), np.uint8)
    frames[:, 0, 0] = 3
    frames[:, 1, 1] = 250
    lo, hi = oracle.learn(frames, 10)
    assert lo[0, 0].tolist() == [0, 0, 0] and hi[0, 0].tolist() == [13, 13, 13]
    assert lo[1, 1].tolist() == [240] * 3 and hi[1, 1].tolist() == [255] * 3


def test_learn_constant_width20():
    v = np.arange(256, dtype=np.uint8).reshape(16, 16)
    frames = np.stack([np.stack([v] * 3, axis=-1)] * 30)
    lo, hi = oracle.learn(frames, 10)
    width = hi.astype(int) - lo.astype(int)
    inner = (v >= 10) & (v <= 245)
    assert (width[inner] == 20).all()
    assert (width[~inner] < 20).all()


def test_learn_invariants():
    rng = np.random.default_rng(2)
    frames = rng.integers(0, 256, (7, 9, 11, 3), dtype=np.uint8)
    for m in (0, 4, 10):
        lo, hi = oracle.learn(frames, m)
        assert ((frames >= lo) & (frames <= hi)).all()
        lo2, hi2 = oracle.learn(frames[:4], m)                 # subset -> narrower
        assert (lo2 >= lo).all() and (hi2 <= hi).all()


def test_learn_empty_is_error():
    with pytest.raises(ValueError):
        oracle.learn(np.zeros((0, 2, 2, 3), np.uint8), 10)


# ---------------------------------------------------------------- a2 luminosity
def test_mean_uniform_gray_is_value():
    # weights 299 + 587 + 114 = 1000: a uniform gray v has exact mean v
    for v in range(256):
        f = np.full((3, 5, 3), v, np.uint8)
        assert oracle.mean_luma(f)[0] == v


def test_mean_rounds_half_up():
    # half 0 / half 255 -> exact mean 127.5 -> 128 (reading L19)
    f = np.zeros((2, 8, 3), np.uint8)
    f[1] = 255
    assert oracle.mean_luma(f)[0] == 128
    # exact mean 0.5 -> 1; 0.499 -> 0
    f = np.zeros((1, 2, 3), np.uint8)
    f[0, 0] = (1, 1, 1)
    assert oracle.mean_luma(f)[0] == 1   # (1000)/(2*1000)=0.5 -> 1


def test_mean_rgb_cube_is_128():
    # every (r,g,b) once: each channel averages 127.5 -> mean 127.5 -> 128
    r, g, b = np.meshgrid(np.arange(256), np.arange(256), np.arange(256), indexing="ij")
    cube = np.stack([r, g, b], -1).astype(np.uint8).reshape(4096, 4096, 3)
    m, s = oracle.mean_luma(cube)
    assert s == 1000 * 4096 * 4096 * 255 // 2
    assert m == 128


def test_gamma_passthrough_and_limits():
    p = oracle.make_params(4, 4)
    for m in range(60, 191):
        assert oracle.gamma(p, m) == (1.0, 0)
    assert oracle.gamma(p, 0) == (0.4, 1)
    assert oracle.gamma(p, 255) == (2.5, 1)
    assert oracle.lut(0.4)[0] == 0                           # all-black stays black


def test_gamma_maps_mean_to_target_or_clamps():
    # the unclamped gamma solves 255 (m/255)^g = target; clamping keeps the
    # corrected mean on the same side of the target
    p = oracle.make_params(4, 4)
    n_unclamped = 0
    for m in list(range(1, 60)) + list(range(191, 255)):
        g, c = oracle.gamma(p, m)
        assert c == 1 and 0.4 <= g <= 2.5
        v = 255.0 * (m / 255.0) ** g
        if g == 0.4:
            assert v < 128
        elif g == 2.5:
            assert v > 128
        else:
            n_unclamped += 1
            assert abs(v - 128) < 1e-9
    # computed regimes: 46..59 and 191..193 are unclamped
    assert n_unclamped == 14 + 3


@pytest.mark.parametrize("p,q", [(2, 5), (5, 2), (2, 1), (1, 2), (1, 1)])
def test_lut_exact_rational_gamma(p, q):
    assert np.array_equal(oracle.lut(p / q), brute.lut_rational_gamma(p, q))


def test_lut_spec_220_reading_L22():
    # S:202 vs clamp: uniform gray 220 -> gamma clamps to 2.5 -> 176
    pr = oracle.make_params(4, 4)
    g, c = oracle.gamma(pr, 220)
    assert g == 2.5 and oracle.lut(g)[220] == 176


def test_lut_monotone_all_means():
    pr = oracle.make_params(4, 4)
    for m in range(256):
        g, _ = oracle.gamma(pr, m)
        L = oracle.lut(g).astype(int)
        assert L[0] == 0 and L[255] == 255 and (np.diff(L) >= 0).all()


def test_lut_tie_margin():
    # no LUT entry in any regime lies within 1e-6 of a rounding tie, so 1-2 ulp
    # differences in log/pow cannot change an entry (reading L21)
    pr = oracle.make_params(4, 4)
    worst = 1.0
    for m in range(256):
        g, c = oracle.gamma(pr, m)
        if not c:
            continue
        for x in range(256):
            v = 255.0 * math.pow(x / 255.0, g) + 0.5
            worst = min(worst, abs(v - round(v)) if x not in (0, 255) else 1.0)
    assert worst > 1e-6
