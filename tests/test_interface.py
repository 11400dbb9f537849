"""NEXT-3 interface hit-test: oracle pins (the
SPEC's examples and properties) and fizi_hit_test through the C ABI against
the oracle on random pointer tracks over an overlapping layout."""
import math

import numpy as np
import pytest

from oracle.interface import BUTTON, CLICK, ENTER, LEAVE, SLIDER, VALUE, WHEEL, HitTest, Zone


def test_spec_examples():
    q = Zone(BUTTON, x=10, y=10, w=20, h=20)
    ht = HitTest([q])
    assert ht.update(True, False, 0, 0) == [(False, 0, 0.0)]
    assert ht.update(True, False, 15, 15) == [(True, ENTER, 0.0)]
    assert ht.update(True, True, 15, 15) == [(True, CLICK, 0.0)]
    assert ht.update(True, False, 30, 30) == [(True, 0, 0.0)]                 # inclusive edge
    assert ht.update(False, False, 15, 15) == [(False, LEAVE, 0.0)]           # pointer lost
    s = Zone(SLIDER, x=0, y=100, w=40, h=200)
    ht = HitTest([s])
    inside, ev, v = ht.update(True, False, 20, 200)[0]                        # vertical midpoint
    assert inside and ev == ENTER | VALUE and v == 0.5
    assert ht.update(True, False, 20, 201)[0] == (True, 0, 0.0)               # change < 0.01
    inside, ev, v = ht.update(True, False, 20, 204)[0]
    assert ev == VALUE and abs(v - 0.48) < 1e-12
    w = Zone(WHEEL, cx=320, cy=260, r=140, theta_max=90)
    ht = HitTest([w])
    inside, ev, v = ht.update(True, False, 320 + 140 * math.sin(math.radians(45)),
                              260 - 140 * math.cos(math.radians(45)))[0]
    assert inside and ev == ENTER | VALUE and abs(v - 0.5) < 1e-9


def test_properties_alternation_and_ranges():
    rng = np.random.default_rng(3)
    zones = [Zone(BUTTON, 50, 50, 100, 80), Zone(SLIDER, 120, 40, 60, 300),
             Zone(WHEEL, cx=320, cy=260, r=140)]
    ht = HitTest(zones)
    state = [False] * 3
    for _ in range(5000):
        res = ht.update(bool(rng.random() < 0.9), bool(rng.random() < 0.1),
                        float(rng.uniform(0, 640)), float(rng.uniform(0, 480)))
        for k, (inside, ev, v) in enumerate(res):
            if ev & ENTER:
                assert not state[k]
            if ev & LEAVE:
                assert state[k]
            state[k] = inside
            if zones[k].kind == SLIDER and ev & VALUE:
                assert 0.0 <= v <= 1.0


@pytest.mark.gpu
def test_fizi_hit_test_matches_oracle():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_1907_04393_b200 import RESULT_DTYPE, ZONE_EVENT_DTYPE, Fizi, FiziError
    from paper_1907_04393_b200.fizi import Zone as CZone
    layout = [Zone(BUTTON, 50, 50, 100, 80), Zone(SLIDER, 120, 40, 60, 300),
              Zone(WHEEL, cx=320, cy=260, r=140, theta_max=90), Zone(BUTTON, 100, 100, 40, 40)]
    rng = np.random.default_rng(9)
    n = 500
    rec = np.zeros(n, RESULT_DTYPE)
    vis = rng.random(n) < 0.85
    clk = rng.random(n) < 0.1
    px = np.clip(np.cumsum(rng.normal(0, 25, n)) + 300, 0, 639)
    py = np.clip(np.cumsum(rng.normal(0, 25, n)) + 240, 0, 479)
    px[::50], py[::50] = 50.0, 130.0                                   # exact rectangle corners
    rec["visible"], rec["clicked"], rec["px"], rec["py"] = vis, clk, px, py
    fz = Fizi(640, 480, max_batch=16)
    with pytest.raises(FiziError):
        fz.hit_test(torch.zeros((1, 128), dtype=torch.uint8, device="cuda"))
    cz = []
    for z in layout:
        c = CZone()
        c.kind, c.x, c.y, c.w, c.h = z.kind, z.x, z.y, z.w, z.h
        c.cx, c.cy, c.r, c.theta_max_deg = z.cx, z.cy, z.r, z.theta_max
        cz.append(c)
    fz.set_zones(cz)
    dev = torch.from_numpy(rec.view(np.uint8).reshape(n, 128).copy()).cuda()
    got = np.concatenate([fz.hit_test(dev[i:i + 100]).cpu().numpy() for i in range(0, n, 100)])
    got = got.reshape(n, len(layout), 16).view(ZONE_EVENT_DTYPE).reshape(n, len(layout))
    ht = HitTest(layout)
    for i in range(n):
        ref = ht.update(bool(vis[i]), bool(clk[i]), float(px[i]), float(py[i]))
        for k, (inside, ev, v) in enumerate(ref):
            assert bool(got[i, k]["inside"]) == inside, (i, k)
            assert int(got[i, k]["events"]) == ev, (i, k, int(got[i, k]["events"]), ev)
            assert abs(got[i, k]["value"] - v) <= 1e-9
    fz.close()
