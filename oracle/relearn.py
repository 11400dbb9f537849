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
