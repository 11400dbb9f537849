"""Shared helpers for the -m gpu parity tests (comparison only, no method arithmetic)."""
import numpy as np

import oracle

INT_FIELDS = ("mean_luma", "corrected", "fg_merged", "fg_final", "n_comp_total", "n_comp_kept",
              "blob_area", "blob_label", "sum_x", "sum_y")
TRACK_INT = ("visible", "clicked", "dwell_ms")
FP_FIELDS = ("gamma", "cx", "cy")
TRACK_FP = ("px", "py")
TOL = 1e-3          # north star: floating-point outputs within 1e-3 (pixels / gain)


def compare_record(r, rec, k=None, track=False):
    """r: row of RESULT_DTYPE (GPU), rec: oracle.Record."""
    for f in INT_FIELDS + (TRACK_INT if track else ()):
        assert int(r[f]) == int(getattr(rec, f)), (k, f, int(r[f]), int(getattr(rec, f)))
    if rec.blob_area:
        assert [int(v) for v in r["bbox"]] == list(rec.bbox), (k, "bbox")
    for f in FP_FIELDS + (TRACK_FP if track else ()):
        assert abs(float(r[f]) - float(getattr(rec, f))) <= TOL, (k, f, float(r[f]), getattr(rec, f))
    assert int(r["t_ms"]) == int(rec.t_ms)


def oracle_run(params, frames, lo, hi, t_ms, stages=False, nthreads=8):
    """Oracle records (+ optional stage dicts) for a batch of one stream."""
    if stages:
        out = [oracle.segment(params, frames[k], lo, hi, t_ms=int(t_ms[k])) for k in range(len(frames))]
        return [o[0] for o in out], [o[1] for o in out]
    recs, masks = oracle.segment_batch(params, frames, lo, hi, t_ms=t_ms, nthreads=nthreads)
    return recs, masks
