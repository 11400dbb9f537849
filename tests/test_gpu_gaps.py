"""GPU parity for cases the round-1 suite did not reach: the whole K0 table
(every mean luma, two parameter sets), inverted (lo > hi) envelopes, and the
full record of every exhaustive 4x4 mask."""
import numpy as np
import pytest

import oracle
from tests.gpu_common import compare_record
from tests.helpers import all_masks, mask_frames

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_1907_04393_b200 import Fizi, results_numpy  # noqa: E402

DEV = torch.device("cuda", 0)


def _t(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(DEV)


LUT_PARAMS = [
    dict(),                                                         # S:187 defaults
    dict(luma_target=100, luma_lo=70, luma_hi=160, gamma_min=0.5, gamma_max=2.0),
    dict(luma_target=200, luma_lo=199, luma_hi=201, gamma_min=0.25, gamma_max=4.0),
]


@pytest.mark.parametrize("params", LUT_PARAMS)
def test_k0_table_every_mean_matches_oracle(params):
    """a2 (§3.2; L19-L21): the device's 256 x 256 LUT table byte for
    byte against oracle.lut(oracle.gamma(m)) for every mean m, and gamma /
    corrected per row (this includes the unclamped rows on both sides)."""
    fz = Fizi(64, 8, **params)
    lut, gam, cor = fz.get_lut_table()
    torch.cuda.synchronize()
    lut, gam, cor = lut.cpu().numpy(), gam.cpu().numpy(), cor.cpu().numpy()
    p = oracle.make_params(64, 8, **params)
    unclamped = 0
    for m in range(256):
        g, c = oracle.gamma(p, m)
        assert int(cor[m]) == c, m
        assert abs(float(gam[m]) - g) <= 1e-12, (m, float(gam[m]), g)
        want = oracle.lut(g) if c else np.arange(256, dtype=np.uint8)
        assert np.array_equal(lut[m], want), (m, np.nonzero(lut[m] != want)[0][:8])
        unclamped += c and p.gamma_min < g < p.gamma_max
    assert unclamped >= 3
    fz.close()


def test_inverted_envelope_lo_gt_hi():
    """include/fizi.h allows lo > hi (fizi_set_background): such a byte is
    never inside [lo, hi] (reading L2), so R1 = 1 there.  Mixed
    ordered / inverted envelopes over several tiles, fast path and generic."""
    for W, H in ((64, 48), (50, 37)):
        rng = np.random.default_rng(W)
        n = 4
        frames = rng.integers(0, 256, (n, H, W, 3), dtype=np.uint8)
        frames[:, 10:30, 10:40] = (210, 120, 110)
        lo = rng.integers(0, 256, (H, W, 3)).astype(np.uint8)
        hi = rng.integers(0, 256, (H, W, 3)).astype(np.uint8)
        # half the rows: a wide ordered envelope, the rest random (many lo > hi)
        lo[: H // 2] = 0
        hi[: H // 2] = 255
        inv = lo > hi
        assert inv.any() and (~inv).any()
        fz = Fizi(W, H, max_batch=n, debug=1, min_blob_ppm=0)
        fz.set_background(_t(lo), _t(hi))
        masks, res = fz.segment_frames(_t(frames))
        res, masks = results_numpy(res), masks.cpu().numpy()
        p = oracle.make_params(W, H, min_blob_ppm=0)
        for k in range(n):
            rec, st = oracle.segment(p, frames[k], lo, hi)
            compare_record(res[k], rec, k)
            assert np.array_equal(masks[k], st["final_mask"]), k
            for sname, oname in (("r1", "r1"), ("merged", "merged")):
                got = fz.debug_stage(sname, k).cpu().numpy()
                assert np.array_equal(got, st[oname]), (W, k, sname)
            # the inverted bytes are outside: R1 = 1 wherever any channel is inverted
            assert (st["r1"][inv.any(-1)] == 1).all()
        fz.close()


def test_exhaustive_4x4_masks_full_records():
    """All 2^16 4x4 masks (generic path): every field of every record, not
    only the labelling fields."""
    masks = all_masks(4, 4)
    frames, lo, hi = mask_frames(masks)
    n = frames.shape[0]
    fz = Fizi(4, 4, n_streams=1, max_batch=65535, min_blob_ppm=0)
    fz.set_background(_t(lo), _t(hi))
    gm, gr = [], []
    for b in range(0, n, 65535):
        m, r = fz.segment_frames(_t(frames[b:b + 65535]))
        gm.append(m.cpu().numpy())
        gr.append(results_numpy(r))
    gm, gr = np.concatenate(gm), np.concatenate(gr)
    p = oracle.make_params(4, 4, min_blob_ppm=0)
    recs, om = oracle.segment_batch(p, frames, lo, hi, nthreads=8)
    assert np.array_equal(gm, om)
    # vectorised full-record comparison (every integer field, bbox, FP fields)
    want = {f: np.array([getattr(r, f) for r in recs]) for f in
            ("mean_luma", "corrected", "fg_merged", "fg_final", "n_comp_total", "n_comp_kept",
             "blob_area", "blob_label", "sum_x", "sum_y", "gamma", "cx", "cy")}
    for f in ("mean_luma", "corrected", "fg_merged", "fg_final", "n_comp_total", "n_comp_kept",
              "blob_area", "blob_label", "sum_x", "sum_y"):
        assert np.array_equal(gr[f].astype(np.int64), want[f].astype(np.int64)), f
    for f in ("gamma", "cx", "cy"):
        assert np.abs(gr[f] - want[f]).max() <= 1e-3, f
    has = want["blob_area"] > 0
    wb = np.array([list(r.bbox) for r in recs])
    assert np.array_equal(gr["bbox"][has], wb[has])
    fz.close()


def test_exhaustive_5x5_masks_morphology_and_labelling():
    """All 2^25 5x5 merged masks (morphology a4 and
    labelling a5-a7): the final mask and every labelling field of
    the record, GPU vs oracle, in chunks of 2^20 masks."""
    import os
    n_all, chunk, B = 1 << 25, 1 << 20, 65535
    p = oracle.make_params(5, 5, min_blob_ppm=0)
    fz = Fizi(5, 5, n_streams=1, max_batch=B, min_blob_ppm=0)
    lo = hi = None
    nthreads = os.cpu_count() or 8
    shifts = np.arange(25, dtype=np.int64)
    for c0 in range(0, n_all, chunk):
        idx = np.arange(c0, c0 + chunk, dtype=np.int64)
        masks = ((idx[:, None] >> shifts[None, :]) & 1).reshape(-1, 5, 5).astype(np.uint8)
        frames, lo_c, hi_c = mask_frames(masks)
        if lo is None:
            lo, hi = lo_c, hi_c
            fz.set_background(_t(lo), _t(hi))
        fr_d = _t(frames)
        gm = torch.empty((chunk, 5, 5), dtype=torch.uint8, device=DEV)
        gr = torch.empty((chunk, 128), dtype=torch.uint8, device=DEV)
        for b in range(0, chunk, B):
            e = min(chunk, b + B)
            fz.segment_frames(fr_d[b:e], masks=gm[b:e], results=gr[b:e])
        recs, om = oracle.segment_batch(p, frames, lo, hi, nthreads=nthreads, as_array=True)
        gm, gr = gm.cpu().numpy(), results_numpy(gr)
        bad = np.nonzero((gm != om).reshape(chunk, -1).any(1))[0]
        assert bad.size == 0, ("mask", int(c0 + bad[0]))
        for f in ("fg_merged", "fg_final", "n_comp_total", "n_comp_kept", "blob_area",
                  "blob_label", "sum_x", "sum_y"):
            bad = np.nonzero(gr[f].astype(np.int64) != recs[f].astype(np.int64))[0]
            assert bad.size == 0, (f, int(c0 + bad[0]))
        has = recs["blob_area"] > 0
        assert np.array_equal(gr["bbox"][has], recs["bbox"][has])
        assert np.abs(gr["cx"] - recs["cx"]).max() <= 1e-3
        assert np.abs(gr["cy"] - recs["cy"]).max() <= 1e-3
    fz.close()


def test_tall_frames_tree_ordered_block_merging():
    """Frames taller than 384 four-row blocks take the labelling's tree-ordered
    boundary merging (k_ccl.cu, kCclTreeBlocks): random masks, a tall snake
    component spanning the whole height, and vertical stripes, against the
    oracle's labels and records."""
    W, H = 64, 2048
    rng = np.random.default_rng(2048)
    masks = np.zeros((3, H, W), np.uint8)
    masks[0] = rng.random((H, W)) < 0.45
    masks[1][:, 30:34] = 1                                  # one tall component
    masks[1][::7, 5:60] = 1
    masks[2][:, ::3] = 1                                    # many tall thin stripes (removed by the opening)
    masks[2][:, 40:50] = 1
    frames, lo, hi = mask_frames(masks)
    fz = Fizi(W, H, max_batch=3, min_blob_ppm=0, debug=1)
    fz.set_background(_t(lo), _t(hi))
    gm, gr = fz.segment_frames(_t(frames))
    gm, gr = gm.cpu().numpy(), results_numpy(gr)
    p = oracle.make_params(W, H, min_blob_ppm=0)
    for k in range(3):
        rec, st = oracle.segment(p, frames[k], lo, hi)
        compare_record(gr[k], rec, k)
        assert np.array_equal(gm[k], st["final_mask"]), k
        lab = fz.debug_stage("labels", k).cpu().numpy().view(np.uint32)
        assert np.array_equal(lab, st["labels"]), k
    fz.close()
