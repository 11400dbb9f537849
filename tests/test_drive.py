"""NEXT-2 drive mapping.

CPU: the oracle (oracle/drive.py) against the SPEC's examples, closed forms on
the rim and the stated properties (odd symmetry, ranges, purity, decay).
GPU: fizi_drive through the C ABI against the oracle on random pointer tracks
(steering within 1e-9, has_steering and throttle exact)."""
import math

import numpy as np
import pytest

from oracle.drive import Drive, Wheel, steering_from_cursor

W = Wheel(cx=320.0, cy=260.0, radius=140.0, theta_max=90.0)


def _rim(theta_deg, w=W, frac=1.0):
    t = math.radians(theta_deg)                 # 12 o'clock = -y, clockwise = +x
    return w.cx + frac * w.radius * math.sin(t), w.cy - frac * w.radius * math.cos(t)


def test_spec_examples_steering():
    assert steering_from_cursor(True, *_rim(0.0), W) == 0.0           # 12 o'clock
    assert abs(steering_from_cursor(True, *_rim(90.0), W) - 1.0) < 1e-9   # 3 o'clock
    assert abs(steering_from_cursor(True, *_rim(-60.0), W) + 2.0 / 3.0) < 1e-9   # 10 o'clock
    assert steering_from_cursor(False, *_rim(45.0), W) is None         # invisible
    assert steering_from_cursor(True, W.cx, W.cy, W) is None          # centre: outside annulus
    assert steering_from_cursor(True, *_rim(45.0, frac=1.5), W) is None   # beyond outer
    assert steering_from_cursor(True, *_rim(45.0, frac=0.5), W) is None   # inside inner
    assert steering_from_cursor(True, *_rim(2.9), W) == 0.0            # dead zone (3 degrees)
    assert steering_from_cursor(True, *_rim(180.0), W) == 1.0          # 6 o'clock: theta = +180, clamped
    assert abs(steering_from_cursor(True, *_rim(45.0), W) - 0.5) < 1e-9
    assert steering_from_cursor(True, *_rim(-135.0), W) == -1.0


def test_steering_odd_symmetry_ranges_purity():
    # wheel centred on x = 0 so that the mirror image (-px) is exact
    w0 = Wheel(cx=0.0, cy=260.0, radius=140.0)
    rng = np.random.default_rng(11)
    for _ in range(10000):
        px, py = rng.uniform(-320, 320), rng.uniform(0, 480)
        a = steering_from_cursor(True, px, py, w0)
        b = steering_from_cursor(True, -px, py, w0)                     # mirror across x = cx
        assert (a is None) == (b is None)
        if a is not None:
            assert a == -b or (a == 1.0 and b == 1.0 and px == 0.0)     # 6 o'clock maps to +180
            assert -1.0 <= a <= 1.0
            assert steering_from_cursor(True, px, py, w0) == a


def test_spec_examples_make_command():
    d = Drive(Wheel(cx=0, cy=0, radius=10, hold_ms=100))
    c = d.update(False, 0, 0, 0)                                       # both absent, first frame
    assert (c.steering, c.throttle) == (0.0, 0.0)
    d = Drive(Wheel(cx=0, cy=0, radius=10, hold_ms=100))
    c = d.update(True, *_rim(45.0, Wheel(0, 0, 10)), 0, throttle_opt=0.8)
    assert abs(c.steering - 0.5) < 1e-12 and c.throttle == 0.8
    d = Drive(Wheel(cx=0, cy=0, radius=10, hold_ms=100))
    d.update(True, *_rim(90.0, Wheel(0, 0, 10)), 0)                    # steering 1.0
    assert d.update(False, 0, 0, 50).steering == 1.0                   # held within hold_ms
    assert d.update(False, 0, 0, 100).steering == 1.0                  # boundary: not > hold
    assert d.update(False, 0, 0, 133).steering == 0.8                  # decays by 0.8
    assert abs(d.update(False, 0, 0, 166).steering - 0.64) < 1e-15


@pytest.mark.gpu
def test_fizi_drive_matches_oracle():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_1907_04393_b200 import RESULT_DTYPE, Fizi, FiziError, commands_numpy
    rng = np.random.default_rng(5)
    n = 400
    rec = np.zeros(n, RESULT_DTYPE)
    t = np.cumsum(rng.integers(20, 60, n)).astype(np.int64)
    rec["t_ms"] = t
    vis = rng.random(n) < 0.8
    # a wandering pointer around the wheel, with exact rim / axis / dead-zone points mixed in
    ang = np.cumsum(rng.normal(0, 12, n))
    frac = rng.uniform(0.3, 1.7, n)
    px = W.cx + frac * W.radius * np.sin(np.radians(ang))
    py = W.cy - frac * W.radius * np.cos(np.radians(ang))
    for i, (a, f) in zip(range(0, n, 37), [(0, 1), (90, 1), (-60, 1), (180, 1), (3, 1), (-3, 1),
                                            (45, 0.6), (45, 1.4), (0, 0), (30, 1), (-179, 1)]):
        px[i], py[i] = _rim(a, frac=f)
        vis[i] = True
    rec["visible"] = vis
    rec["px"], rec["py"] = px, py
    fz = Fizi(640, 480, max_batch=16)
    with pytest.raises(FiziError):
        fz.drive(torch.zeros((1, 128), dtype=torch.uint8, device="cuda"))   # no wheel yet
    fz.set_wheel(W.cx, W.cy, W.radius, theta_max_deg=W.theta_max, hold_ms=W.hold_ms)
    dev = torch.from_numpy(rec.view(np.uint8).reshape(n, 128).copy()).cuda()
    out = np.concatenate([commands_numpy(fz.drive(dev[i:i + 64])) for i in range(0, n, 64)])
    d = Drive(W)
    for i in range(n):
        c = d.update(bool(vis[i]), float(px[i]), float(py[i]), int(t[i]))
        assert bool(out[i]["has_steering"]) == c.has_steering, i
        assert abs(out[i]["steering"] - c.steering) <= 1e-9, (i, out[i]["steering"], c.steering)
        assert out[i]["throttle"] == c.throttle and out[i]["t_ms"] == c.t_ms
    fz.close()


# ---- throttle from a NEXT-3 slider zone (reading L36)
def test_throttle_follows_slider_value_events():
    from oracle.interface import SLIDER, VALUE, HitTest, Zone
    slider = Zone(SLIDER, 500, 100, 40, 200)                 # value = 1 - (py - 100) / 200
    ht = HitTest([slider])
    d = Drive(W)
    seq = [(True, 520.0, 140.0), (True, 520.0, 140.0), (False, 0.0, 0.0), (True, 520.0, 300.0),
           (True, *_rim(90))]
    want = [0.8, 0.8, 0.8, 0.0, 0.0]                          # value, unchanged, held, bottom, off
    for k, ((vis, x, y), w) in enumerate(zip(seq, want)):
        (_, ev, v), = ht.update(vis, False, x, y)
        c = d.update(vis, x, y, 33 * k, v if ev & VALUE else None)
        assert c.throttle == w, (k, c.throttle)
    assert c.steering == 1.0 and c.has_steering                 # S:393 3 o'clock on the rim


@pytest.mark.gpu
def test_fizi_drive_throttle_matches_oracle():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from oracle.interface import BUTTON, SLIDER, VALUE, HitTest, Zone
    from paper_1907_04393_b200 import RESULT_DTYPE, Fizi, FiziError, commands_numpy
    from paper_1907_04393_b200.fizi import Zone as CZone
    layout = [Zone(BUTTON, 20, 20, 60, 60), Zone(SLIDER, 480, 60, 80, 360)]
    rng = np.random.default_rng(11)
    n = 300
    rec = np.zeros(n, RESULT_DTYPE)
    t = np.cumsum(rng.integers(20, 60, n)).astype(np.int64)
    vis = rng.random(n) < 0.85
    px = np.clip(np.cumsum(rng.normal(0, 30, n)) + 450, 0, 639)
    py = np.clip(np.cumsum(rng.normal(0, 30, n)) + 240, 0, 479)
    rec["t_ms"], rec["visible"], rec["px"], rec["py"] = t, vis, px, py
    fz = Fizi(640, 480, max_batch=16)
    cz = []
    for z in layout:
        c = CZone()
        c.kind, c.x, c.y, c.w, c.h = z.kind, z.x, z.y, z.w, z.h
        cz.append(c)
    fz.set_zones(cz)
    fz.set_wheel(W.cx, W.cy, W.radius, theta_max_deg=W.theta_max, hold_ms=W.hold_ms)
    dev = torch.from_numpy(rec.view(np.uint8).reshape(n, 128).copy()).cuda()
    ev0 = fz.hit_test(dev[:1])
    with pytest.raises(FiziError):
        fz.drive(dev[:1], events=ev0, slider_zone=0)          # zone 0 is a button
    fz.set_zones(cz)                                           # reset the hit state
    fz.set_wheel(W.cx, W.cy, W.radius, theta_max_deg=W.theta_max, hold_ms=W.hold_ms)
    out = []
    for i in range(0, n, 64):
        ev = fz.hit_test(dev[i:i + 64])
        out.append(commands_numpy(fz.drive(dev[i:i + 64], events=ev, slider_zone=1)))
    out = np.concatenate(out)
    ht, d = HitTest(layout), Drive(W)
    moved = 0
    for i in range(n):
        _, (_, ev, v) = ht.update(bool(vis[i]), False, float(px[i]), float(py[i]))
        c = d.update(bool(vis[i]), float(px[i]), float(py[i]), int(t[i]),
                     v if ev & VALUE else None)
        moved += bool(ev & VALUE)
        assert abs(out[i]["steering"] - c.steering) <= 1e-9, i
        assert abs(out[i]["throttle"] - c.throttle) <= 1e-9, (i, out[i]["throttle"], c.throttle)
        assert bool(out[i]["has_steering"]) == c.has_steering and out[i]["t_ms"] == c.t_ms
    assert moved > 5
    fz.close()
