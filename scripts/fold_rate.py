"""Diagnostics: a8 fold rate of fizi_track_runs (one thread folds in order):
records per microsecond for a window of 16 steps x 8 ranks x 64 frames."""
import os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1907_04393_b200 import RESULT_DTYPE, Fizi

dev = torch.device("cuda", 0)
fz = Fizi(1920, 1080, max_batch=64)
for n in (1024, 8192):
    rec = np.zeros(n, RESULT_DTYPE)
    rng = np.random.default_rng(1)
    rec["t_ms"] = np.arange(n) * 33
    rec["blob_area"] = np.where(rng.random(n) < 0.9, 5000, 0)
    rec["cx"] = 960 + np.cumsum(rng.normal(0, 3, n))
    rec["cy"] = 540 + np.cumsum(rng.normal(0, 3, n))
    res = torch.from_numpy(rec.view(np.uint8).reshape(n, 128)).to(dev)
    runs = [(o, 64) for o in range(0, n, 64)][:256]
    for _ in range(3):
        fz.reset_tracker()
        fz.track_runs(res, runs)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 10
    e0.record()
    for _ in range(reps):
        fz.track_runs(res, runs)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    m = sum(l for _, l in runs)
    print("records %d runs %d: %.1f us per launch, %.3f us per record" % (m, len(runs), ms * 1e3, ms * 1e3 / m))
