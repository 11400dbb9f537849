"""Pins for oracle a4 (morphology), a5-a7 (labelling, blob filter, largest blob).

Morphology is pinned against scipy.ndimage binary_erosion / binary_dilation
with border_value=0 (S:68, S:76 zero padding) on random and exhaustive masks,
plus closed forms (digital discs lose exactly their 4 tips).  Labelling is
pinned against scipy.ndimage.label (8-connectivity) relabelled by min raster
index (reading L15) on 1000 random 32x32 masks.
"""
import numpy as np
import pytest

import oracle
from tests import brute
from tests.helpers import all_masks, mask_frames


@pytest.mark.parametrize("r", [1, 2])
def test_erode_dilate_vs_scipy_random(r):
    rng = np.random.default_rng(10 + r)
    for _ in range(500):
        m = (rng.random((8, 8)) < rng.random()).astype(np.uint8)
        assert np.array_equal(oracle.erode(m, r), brute.erode(m, r))
        assert np.array_equal(oracle.dilate(m, r), brute.dilate(m, r))
        assert np.array_equal(oracle.open_close(m, r), brute.open_close(m, r))


def test_morph_exhaustive_4x4():
    for m in all_masks(4, 4):
        assert np.array_equal(oracle.open_close(m, 1), brute.open_close(m, 1))


def test_morph_spec_examples():
    ones = np.ones((5, 5), np.uint8)
    e = oracle.erode(ones)
    assert e.sum() == 9 and e[1:4, 1:4].all()
    dot = np.zeros((5, 5), np.uint8)
    dot[2, 2] = 1
    assert oracle.erode(dot).sum() == 0
    d = oracle.dilate(dot)
    assert d.sum() == 9 and d[1:4, 1:4].all()
    assert oracle.dilate(np.zeros((5, 5), np.uint8)).sum() == 0


def test_morph_duality_and_extensivity():
    rng = np.random.default_rng(12)
    for _ in range(200):
        m = (rng.random((9, 7)) < 0.5).astype(np.uint8)
        d, e = oracle.dilate(m), oracle.erode(m)
        assert (d >= m).all() and (e <= m).all()
        # duality with swapped padding: erode(m) = not dilate(not m) when the
        # outside is treated as 0 for erosion <=> as 1 for the complement
        pad = np.pad(m, 1, constant_values=0)
        dual = 1 - oracle.dilate(1 - pad)[1:-1, 1:-1]
        assert np.array_equal(e, dual)


def _disc(h, w, cx, cy, R):
    y, x = np.mgrid[:h, :w]
    return (((x - cx) ** 2 + (y - cy) ** 2) <= R * R).astype(np.uint8)


@pytest.mark.parametrize("R", [5, 10, 20, 30])
def test_open_close_disc_loses_four_tips(R):
    # integer-centred digital disc: open->close removes exactly the 4 axis tips
    h = w = 2 * R + 9
    c = R + 4
    m = _disc(h, w, c, c, R)
    o = oracle.open_close(m)
    tips = np.zeros_like(m)
    for (x, y) in ((c - R, c), (c + R, c), (c, c - R), (c, c + R)):
        tips[y, x] = 1
    assert np.array_equal(o, m & (1 - tips))
    gauss = sum(1 for x in range(-R, R + 1) for y in range(-R, R + 1) if x * x + y * y <= R * R)
    assert o.sum() == gauss - 4


def test_open_close_rectangles_and_bars():
    m = np.zeros((20, 30), np.uint8)
    m[3:10, 4:15] = 1                     # 7x11 rectangle: unchanged
    assert np.array_equal(oracle.open_close(m), m)
    ones = np.ones((240, 320), np.uint8)
    assert oracle.open_close(ones).sum() == 238 * 318
    bars = np.zeros((20, 40), np.uint8)
    bars[5:7, 2:38] = 1                   # 2-px thick: removed
    bars[12:15, 2:38] = 1                 # 3-px thick: kept
    o = oracle.open_close(bars)
    assert not o[:9].any() and np.array_equal(o[9:], bars[9:])


def test_label_vs_scipy_1000_random():
    rng = np.random.default_rng(13)
    for _ in range(1000):
        m = (rng.random((32, 32)) < rng.uniform(0.05, 0.7)).astype(np.uint8)
        lab, n = oracle.label(m)
        ref = brute.canonical_label(m)
        assert np.array_equal(lab, ref)
        assert n == len(np.unique(ref)) - (1 if (ref == 0).any() else 0)


def test_label_diagonal_joins():
    m = np.zeros((4, 4), np.uint8)
    m[1, 1] = m[2, 2] = 1
    lab, n = oracle.label(m)
    assert n == 1 and lab[2, 2] == lab[1, 1] == 1 * 4 + 1 + 1


def _segment_mask(mask, **kw):
    fr, lo, hi = mask_frames(mask[None])
    h, w = mask.shape
    p = oracle.make_params(w, h, **kw)
    return oracle.segment(p, fr[0], lo, hi)


def test_block_area_centroid():
    m = np.zeros((40, 30), np.uint8)
    m[20:23, 10:13] = 1
    rec, st = _segment_mask(m, min_blob_ppm=0)
    assert rec.blob_area == 9 and (rec.cx, rec.cy) == (11.0, 21.0)
    assert list(rec.bbox) == [10, 20, 12, 22] and rec.blob_label == 20 * 30 + 10 + 1


def test_area_threshold_exact():
    # N = 320*240 = 76800, ppm 5000 -> threshold exactly 384 px
    h, w = 240, 320
    m = np.zeros((h, w), np.uint8)
    m[10:34, 10:26] = 1                   # 24x16 = 384 -> kept
    m[100:123, 100:116] = 1               # 23x16 = 368 -> dropped
    rec, st = _segment_mask(m)
    assert rec.n_comp_total == 2 and rec.n_comp_kept == 1
    assert rec.blob_area == 384 and rec.fg_final == 384
    assert st["final_mask"][100:123, 100:116].sum() == 0


def test_largest_tie_smaller_label():
    m = np.zeros((30, 40), np.uint8)
    m[20:25, 2:8] = 1                     # later in raster order
    m[3:8, 30:36] = 1                     # earlier in raster order
    rec, _ = _segment_mask(m, min_blob_ppm=0)
    assert rec.blob_label == 3 * 40 + 30 + 1 and rec.blob_area == 30
    assert (rec.cx, rec.cy) == (32.5, 5.0)


def test_brute_force_16x16_frames():
    # north star: brute force on tiny 16x16 frames, whole pipeline
    rng = np.random.default_rng(14)
    for it in range(60):
        f = rng.integers(0, 256, (16, 16, 3), dtype=np.uint8)
        if it % 2:
            # blobs of skin-like colour on a random background
            m = brute.dilate((rng.random((16, 16)) < 0.08).astype(np.uint8), 1).astype(bool)
            k = int(m.sum())
            f[m] = np.stack([rng.integers(190, 240, k), rng.integers(100, 130, k),
                             rng.integers(90, 110, k)], -1)
        lo = rng.integers(0, 120, (16, 16, 3)).astype(np.uint8)
        hi = (lo + rng.integers(0, 136, (16, 16, 3))).astype(np.uint8)
        S = int(rng.integers(0, 60))
        a1, a2 = (int(v) for v in rng.integers(0, 360, 2))
        ppm = int(rng.choice([0, 5000, 20000]))
        p = oracle.make_params(16, 16, gray_tol_S=S, hue_lo_deg=a1, hue_hi_deg=a2,
                               min_blob_ppm=ppm)
        rec, st = oracle.segment(p, f, lo, hi)
        lut = oracle.lut(rec.gamma) if rec.corrected else None
        ref, stats = brute.segment(f, lo, hi, S, a1, a2, 1, ppm, lut=lut)
        for k_or, k_br in (("r1", "r1"), ("r2", "r2"), ("r3", "r3"), ("merged", "merged"),
                           ("oc", "oc"), ("labels", "labels"), ("final_mask", "final")):
            assert np.array_equal(st[k_or], ref[k_br]), (it, k_or)
        for k in ("n_comp_total", "n_comp_kept", "blob_label", "blob_area", "fg_merged",
                  "fg_final"):
            assert getattr(rec, k) == stats[k], (it, k)
        if stats["blob_label"]:
            assert rec.sum_x == stats["sum_x"] and rec.sum_y == stats["sum_y"]
            assert list(rec.bbox) == stats["bbox"]
