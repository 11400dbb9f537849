"""Oracle of NEXT-1, the relearn trigger (TEST INFRASTRUCTURE ONLY; shares no
code with the CUDA path).

SPEC S:153-161 (paper §3.3, "re-initiate partly the machine learning
techniques" on a change of luminosity): relearn_trigger(prev, cur, threshold)
is true iff |cur - prev| > threshold (strict).  Folded over a stream's frames
in order with the a2 mean luma; the first frame (no previous mean) gives
false.
"""
from __future__ import annotations


def relearn_trigger(prev: int, cur: int, threshold: int) -> bool:
    return abs(int(cur) - int(prev)) > int(threshold)


def relearn_flags(means, threshold: int = 40):
    """Flags of a stream's frames in order (first frame: no previous mean)."""
    out, prev = [], None
    for m in means:
        out.append(prev is not None and relearn_trigger(prev, m, threshold))
        prev = int(m)
    return out


# --------------------------------------------------------------------------
# In-stream relearning (the composition the trigger drives).  Readings (DESIGN
# L37, §3.3 "re-initiate partly the machine learning techniques",
# SPEC S:170 "on trigger, runtime pauses tracking and relearns"
# "Relearning swaps the model atomically between frames"):
#   - every frame's a2 mean luma is compared with the previous frame's of the
#     stream; a trigger (|cur - prev| > threshold) on a frame segmented
#     normally (with the current model, tracker updated) starts relearning;
#   - the stream's next F frames are learning frames: not segmented (empty
#     mask, a3-a7 fields zero), tracking paused (visible = clicked = 0,
#     px = py = 0, dwell 0, tracker state untouched); their means still feed
#     the trigger comparison, but triggers are ignored while learning;
#   - after the F-th learning frame the model becomes learn(those F raw
#     frames, margin) (the start-up rule) and the tracker is reset
#     (as after the start-up learning); the next frame uses the new model.
# Flags per frame: 1 = learning frame, 2 = the model is swapped after this
# frame, 4 = trigger.
RELEARN_LEARN, RELEARN_SWAP, RELEARN_TRIGGER = 1, 2, 4


def run_stream_relearn(params, frames, t_ms, lo, hi, threshold: int, n_learn: int, margin: int):
    """One stream through a2..a8 with in-stream relearning (plain loop over
    the oracle's per-step functions).  Returns (records, final masks, flags,
    list of (frame index after which the model was swapped, lo, hi))."""
    import numpy as np

    import oracle
    assert n_learn >= 1
    tr = oracle.Tracker(params)
    prev = None
    remaining = 0
    acc = []
    recs, masks, flags, swaps = [], [], [], []
    for k, frame in enumerate(frames):
        m, _ = oracle.mean_luma(frame)
        trig = prev is not None and relearn_trigger(prev, m, threshold)
        prev = m
        f = 0
        if remaining > 0:                       # a learning frame
            f |= RELEARN_LEARN
            acc.append(frame)
            remaining -= 1
            g, corrected = oracle.gamma(params, m)
            rec = oracle.Record()
            rec.t_ms = int(t_ms[k])
            rec.mean_luma = m
            rec.corrected = corrected
            rec.gamma = g
            mask = np.zeros(frame.shape[:2], np.uint8)
            if remaining == 0:                  # the model swap after this frame
                f |= RELEARN_SWAP
                lo, hi = oracle.learn(np.stack(acc), margin)
                acc = []
                tr = oracle.Tracker(params)
                swaps.append((k, lo, hi))
        else:
            rec, st = oracle.segment(params, frame, lo, hi, t_ms=int(t_ms[k]))
            tr.update(rec)
            mask = st["final_mask"]
            if trig:
                f |= RELEARN_TRIGGER
                remaining = n_learn
        recs.append(rec)
        masks.append(mask)
        flags.append(f)
    return recs, masks, flags, swaps
