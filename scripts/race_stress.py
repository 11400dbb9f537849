"""Race detection by repetition (compute-sanitizer is closed on this pool):
the pipelined launch configurations bench.py times (C3: calls of 64 frames,
C5: calls of the current frame of all 256 streams), REPS repetitions of
several calls in flight without a flush, each repetition's every mask and
record compared bit for bit with joined (non-overlapped) calls."""
import hashlib
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_1907_04393_b200 import RESULT_BYTES, Fizi  # noqa: E402

dev = torch.device("cuda", 0)
REPS = int(os.environ.get("REPS", "10"))


def run(cid, B, ncalls, pipelined, reps):
    cfg = synth.CONFIGS[cid]
    S = cfg.streams
    fz = Fizi(cfg.W, cfg.H, n_streams=S, max_batch=B)
    for s in range(S):
        fz.learn_background(synth.frames_dev(cfg, s, range(cfg.n_learn), learning=True), stream=s,
                            margin=synth.MARGIN)
    calls = []
    for j in range(ncalls):
        if S == 1:
            ks = list(range(90 + j * B, 90 + (j + 1) * B))
            fr = synth.frames_dev(cfg, 0, ks)
            calls.append((fr, None, np.array([synth.t_ms(k) for k in ks], np.int64)))
        else:
            fr = torch.empty((S, cfg.H, cfg.W, 3), dtype=torch.uint8, device=dev)
            for s in range(S):
                synth.frames_dev(cfg, s, [j], out=fr[s:s + 1])
            calls.append((fr, np.arange(S, dtype=np.uint32), np.full(S, synth.t_ms(j), np.int64)))
    fz.set_pipeline(pipelined)
    digests = []
    for r in range(reps):
        outs = [(torch.empty((B, cfg.H, cfg.W), dtype=torch.uint8, device=dev),
                 torch.empty((B, RESULT_BYTES), dtype=torch.uint8, device=dev)) for _ in calls]
        for s in range(S):                       # every repetition starts from a fresh tracker
            fz.reset_tracker(s)
        for j, (fr, sids, t) in enumerate(calls):
            fz.process_frames(fr, streams=sids, t_ms=t, masks=outs[j][0], results=outs[j][1])
        fz.flush()
        torch.cuda.synchronize()
        h = hashlib.sha256()
        for m, rs in outs:
            h.update(m.cpu().numpy().tobytes())
            h.update(rs.cpu().numpy().tobytes())
        digests.append(h.hexdigest())
    fz.close()
    return digests


for cid, B, ncalls in ((3, 64, 6), (5, 256, 4), (4, 64, 3)):
    ref = run(cid, B, ncalls, False, 1)[0]
    got = run(cid, B, ncalls, True, REPS)
    bad = sum(d != ref for d in got)
    print(f"C{cid}: {REPS} pipelined repetitions x {ncalls} calls of {B} frames in flight: "
          f"{REPS - bad} identical to joined calls, {bad} differ", flush=True)
    assert bad == 0
