"""Independent brute-force re-statement of the pipeline for tiny frames.

Used only to pin the C oracle (tests/test_oracle_*.py).  It deliberately uses
different formulations from oracle/fizi_oracle.c:
  * hue: the textbook hexagonal formula 60*((g-b)/C mod 6) etc. in exact
    rationals (fractions.Fraction), not the oracle's sector numerator;
  * gamma LUT: exact rational bracketing of 255*(x/255)**gamma for rational
    gamma = p/q (no pow);
  * morphology: scipy.ndimage.binary_erosion / binary_dilation with
    border_value=0;
  * labelling: scipy.ndimage.label with a 3x3 structure, relabelled by min
    raster index.
"""
from __future__ import annotations

from fractions import Fraction

import numpy as np
from scipy import ndimage


def hue_textbook(r: int, g: int, b: int):
    """Exact hue in degrees as a Fraction, or None when achromatic."""
    M, m = max(r, g, b), min(r, g, b)
    C = M - m
    if C == 0:
        return None
    if M == r:
        h = 60 * ((Fraction(g - b, C)) % 6)
    elif M == g:
        h = 60 * (Fraction(b - r, C) + 2)
    else:
        h = 60 * (Fraction(r - g, C) + 4)
    return h % 360


def in_band_exact(h: Fraction, a1: int, a2: int) -> bool:
    if a1 <= a2:
        return a1 <= h <= a2
    return h >= a1 or h <= a2


def lut_rational_gamma(p: int, q: int) -> np.ndarray:
    """L[x] = floor(255 (x/255)^(p/q) + 0.5) by exact bracketing.

    v = 255 (x/255)^(p/q)  <=>  v^q = 255^q (x/255)^p = 255^(q-p) x^p.
    L[x] = k  <=>  (k - 1/2)^q <= 255^(q-p) x^p < (k + 1/2)^q  (v >= 0).
    """
    out = np.zeros(256, np.uint8)
    for x in range(256):
        target = Fraction(255) ** (q - p) * Fraction(x) ** p
        k = 0
        while Fraction(2 * k + 1, 2) ** q <= target:
            k += 1
        out[x] = k
    return out


def erode(mask: np.ndarray, r: int) -> np.ndarray:
    se = np.ones((2 * r + 1, 2 * r + 1), bool)
    return ndimage.binary_erosion(mask.astype(bool), structure=se, border_value=0).astype(np.uint8)


def dilate(mask: np.ndarray, r: int) -> np.ndarray:
    se = np.ones((2 * r + 1, 2 * r + 1), bool)
    return ndimage.binary_dilation(mask.astype(bool), structure=se, border_value=0).astype(np.uint8)


def open_close(mask: np.ndarray, r: int) -> np.ndarray:
    return erode(dilate(dilate(erode(mask, r), r), r), r)


def canonical_label(mask: np.ndarray) -> np.ndarray:
    lab, n = ndimage.label(mask.astype(bool), structure=np.ones((3, 3), int))
    out = np.zeros(mask.shape, np.uint32)
    flat = lab.ravel()
    for k in range(1, n + 1):
        idx = np.flatnonzero(flat == k)
        out.ravel()[idx] = idx.min() + 1
    return out


def segment(frame: np.ndarray, lo: np.ndarray, hi: np.ndarray, S: int, a1: int, a2: int,
            r: int, ppm: int, lut=None):
    """Return dict of stage masks + blob stats for one tiny frame."""
    h, w, _ = frame.shape
    f = frame.astype(np.int64)
    if lut is not None:
        f = lut[f].astype(np.int64)
    inside = np.all((f >= lo) & (f <= hi), axis=2)
    r1 = (~inside).astype(np.uint8)
    spread = f.max(axis=2) - f.min(axis=2)
    r2 = (spread >= S).astype(np.uint8)
    r3 = np.zeros((h, w), np.uint8)
    for y in range(h):
        for x in range(w):
            hh = hue_textbook(*[int(v) for v in f[y, x]])
            r3[y, x] = 0 if hh is None else int(in_band_exact(hh, a1, a2))
    merged = r1 & r2 & r3
    oc = open_close(merged, r)
    labels = canonical_label(oc)
    N = h * w
    final = np.zeros((h, w), np.uint8)
    comps = {}
    for L in np.unique(labels):
        if L == 0:
            continue
        sel = labels == L
        area = int(sel.sum())
        comps[int(L)] = area
        if area * 10**6 >= ppm * N:
            final[sel] = 1
    kept = {L: a for L, a in comps.items() if a * 10**6 >= ppm * N}
    best = None
    for L in sorted(kept):
        if best is None or kept[L] > kept[best]:
            best = L
    stats = dict(n_comp_total=len(comps), n_comp_kept=len(kept), blob_label=best or 0,
                 blob_area=kept[best] if best else 0, fg_merged=int(merged.sum()),
                 fg_final=int(final.sum()))
    if best:
        ys, xs = np.nonzero(labels == best)
        stats.update(sum_x=int(xs.sum()), sum_y=int(ys.sum()),
                     bbox=[int(xs.min()), int(ys.min()), int(xs.max()), int(ys.max())])
    return dict(r1=r1, r2=r2, r3=r3, merged=merged, oc=oc, labels=labels, final=final), stats
