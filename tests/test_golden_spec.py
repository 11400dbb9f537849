"""SPEC worked examples (tests/golden/spec_examples.json) against the oracle."""
import json
import os

import numpy as np

import oracle

G = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def _seg1(rgb, lo, hi, **kw):
    f = np.asarray(rgb, np.uint8).reshape(1, 1, 3)
    p = oracle.make_params(1, 1, **kw)
    _, st = oracle.segment(p, f, np.full((1, 1, 3), lo, np.uint8), np.full((1, 1, 3), hi, np.uint8))
    return st


def test_golden_hue():
    for e in G["hue"]:
        assert oracle.hue_num(*e["rgb"]) == (e["hue_num"], e["C"]), e["cite"]


def test_golden_gray():
    for e in G["gray"]:
        assert int(_seg1(e["rgb"], 0, 0, gray_tol_S=e["S"])["r2"][0, 0]) == e["r2"], e["cite"]


def test_golden_background():
    for e in G["background"]:
        assert int(_seg1(e["rgb"], e["lo"], e["hi"])["r1"][0, 0]) == e["r1"], e["cite"]


def test_golden_band():
    for e in G["band"]:
        assert oracle.in_band(e["hue"], 1, e["a1"], e["a2"]) == e["in"], e["cite"]


def test_golden_learn():
    for e in G["learn"]:
        fr = np.array([np.full((2, 2, 3), v, np.uint8) for v in e["values"] * 3])
        lo, hi = oracle.learn(fr, e["margin"])
        assert (lo == e["lo"]).all() and (hi == e["hi"]).all(), e["cite"]
