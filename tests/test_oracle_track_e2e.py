"""Pins for oracle a8 (Mouse fold) and end-to-end closed forms on config 1.

Tracker: S:296-298, S:548 and the dyadic closed form (beta = 0.5 with integer
centroids is exact in binary64) checked in exact rationals.
End to end (C1, BASELINE.json configs[0]): learning frames re-segment to an
exactly empty mask; each processed frame's final mask is exactly the painted
disc minus its four tips, with the centroid at the disc centre.
"""
from fractions import Fraction

import numpy as np

import oracle
import synth


def _fold(recs, **kw):
    p = oracle.make_params(4, 4, **kw)
    tr = oracle.Tracker(p)
    return [tr.update(r) for r in recs]


def test_snap_on_acquisition():
    out = _fold([oracle.record_from_blob(0, 10, 100.0, 50.0)])
    assert out[0].visible == 1 and (out[0].px, out[0].py) == (100.0, 50.0)
    assert out[0].clicked == 0 and out[0].dwell_ms == 0


def test_dwell_click_once_at_frame_25():
    recs = [oracle.record_from_blob(33 * k, 50, 60.0, 70.0) for k in range(30)]
    out = _fold(recs)
    clicks = [k for k, r in enumerate(out) if r.clicked]
    assert clicks == [25] and out[25].dwell_ms == 825
    out14 = _fold([oracle.record_from_blob(33 * k, 50, 60.0, 70.0) for k in range(14)])
    assert not any(r.clicked for r in out14)


def test_lost_after_timeout():
    recs = [oracle.record_from_blob(0, 50, 10.0, 10.0)]
    recs += [oracle.record_from_blob(33 * k) for k in range(1, 20)]
    out = _fold(recs)
    vis = [r.visible for r in out]
    # t - last > 500 first at t = 528 (frame 16)
    assert vis[:16] == [1] * 16 and vis[16:] == [0] * 4
    assert not any(r.clicked for r in out)


def test_dyadic_closed_form():
    rng = np.random.default_rng(20)
    cs = rng.integers(0, 640, (40, 2))
    recs = [oracle.record_from_blob(33 * k, 100, float(x), float(y)) for k, (x, y) in enumerate(cs)]
    out = _fold(recs, dwell_radius_px=1e9, dwell_time_ms=10 ** 12)
    px, py = Fraction(int(cs[0, 0])), Fraction(int(cs[0, 1]))
    for k in range(1, 40):
        px = Fraction(int(cs[k, 0]), 2) + px / 2
        py = Fraction(int(cs[k, 1]), 2) + py / 2
        assert Fraction(out[k].px) == px and Fraction(out[k].py) == py


def test_convex_hull_and_click_invariants():
    rng = np.random.default_rng(21)
    for _ in range(20):
        n = 200
        t = np.cumsum(rng.integers(0, 60, n))
        pres = rng.random(n) < 0.8
        cs = rng.uniform(0, 500, (n, 2))
        recs = [oracle.record_from_blob(int(t[k]), 10 if pres[k] else 0, *cs[k]) for k in range(n)]
        out = _fold(recs, beta=float(rng.uniform(0.1, 1.0)))
        seen = cs[pres]
        for k, r in enumerate(out):
            if r.clicked:
                assert r.visible
            if pres[k]:
                upto = cs[: k + 1][pres[: k + 1]]
                assert upto[:, 0].min() - 1e-9 <= r.px <= upto[:, 0].max() + 1e-9
                assert upto[:, 1].min() - 1e-9 <= r.py <= upto[:, 1].max() + 1e-9
        assert len(seen) > 0


def test_c1_end_to_end_closed_form():
    cfg = synth.CONFIGS[1]
    L = synth.learning_frames_host(cfg)
    lo, hi = oracle.learn(L, synth.MARGIN)
    p = oracle.make_params(cfg.W, cfg.H)
    # precondition: the hand (red >= 206) is outside the envelope everywhere
    assert int(hi[..., 0].max()) < 206
    for f in L:                                                # empty re-segmentation
        rec, st = oracle.segment(p, f, lo, hi)
        assert 60 <= rec.mean_luma <= 190 and rec.fg_merged == 0 and rec.fg_final == 0
    pf = synth.frame_params(cfg, 0, range(cfg.n_proc))
    F = synth.frames_host(cfg, 0, range(cfg.n_proc))
    tr = oracle.Tracker(p)
    px = py = None
    y, x = np.mgrid[:cfg.H, :cfg.W]
    for k in range(cfg.n_proc):
        cx, cy, R = (int(v) for v in pf[k, 2:5])
        rec, st = oracle.segment(p, F[k], lo, hi, t_ms=synth.t_ms(k))
        disc = ((x - cx) ** 2 + (y - cy) ** 2 <= R * R).astype(np.uint8)
        for (tx, ty) in ((cx - R, cy), (cx + R, cy), (cx, cy - R), (cx, cy + R)):
            disc[ty, tx] = 0
        assert np.array_equal(st["final_mask"], disc)
        assert rec.blob_area == 2817 and (rec.cx, rec.cy) == (float(cx), float(cy))
        assert list(rec.bbox) == [cx - R + 1, cy - R + 1, cx + R - 1, cy + R - 1]
        assert rec.blob_label == int(np.flatnonzero(disc)[0]) + 1
        tr.update(rec)
        if px is None:
            px, py = Fraction(cx), Fraction(cy)
        else:
            px, py = Fraction(cx, 2) + px / 2, Fraction(cy, 2) + py / 2
        assert Fraction(rec.px) == px and Fraction(rec.py) == py
