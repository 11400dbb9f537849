"""Diagnostics: per-CTA timeline of the morphology kernel (FIZI_MORPH_TRACE=1)."""
import ctypes, os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth
from paper_1907_04393_b200 import Fizi, lib
cfg = synth.CONFIGS[3]
dev = torch.device("cuda", 0)
fz = Fizi(cfg.W, cfg.H, max_batch=64)
fz.learn_background(synth.frames_dev(cfg, 0, range(30), learning=True))
fr = synth.frames_dev(cfg, 0, range(64))
masks = torch.empty((64, cfg.H, cfg.W), dtype=torch.uint8, device=dev)
for it in range(3):
    fz.process_frames(fr, t_ms=np.arange(64) * 33 + it * 10000, masks=masks)
torch.cuda.synchronize()
n = 68 * 64
buf = (ctypes.c_ulonglong * (5 * n))()
lib().fizi_diag_morph_trace(buf, n)
a = np.frombuffer(buf, dtype=np.uint64).reshape(n, 5).astype(np.int64)
t0 = a[:, 0].min()
s, e, nz = (a[:, 0] - t0) / 1e3, (a[:, 1] - t0) / 1e3, a[:, 2]
print("kernel span us", e.max())
for lab, m in (("zero", nz == 0), ("nonzero", nz == 1)):
    d = e[m] - s[m]
    print(lab, "count", m.sum(), "dur us: mean %.2f p50 %.2f max %.2f" % (d.mean(), np.median(d), d.max()),
          "start us: min %.2f max %.2f" % (s[m].min(), s[m].max()), "end max %.2f" % e[m].max())
m = nz == 1
st = (a[m, 3] - a[m, 0]) / 1e3; pp = (a[m, 4] - a[m, 3]) / 1e3; em = (a[m, 1] - a[m, 4]) / 1e3
print("nonzero phases us: staging %.2f pipeline %.2f emit_runs %.2f" % (st.mean(), pp.mean(), em.mean()))
