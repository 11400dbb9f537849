"""Diagnostics: per-CTA timeline of the labelling kernel (FIZI_CCL_TRACE=1)."""
import ctypes, os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth
from paper_1907_04393_b200 import Fizi, lib
cfg = synth.CONFIGS[int(os.environ.get("CT_CONFIG", "3"))]
dev = torch.device("cuda", 0)
fz = Fizi(cfg.W, cfg.H, max_batch=64)
fz.learn_background(synth.frames_dev(cfg, 0, range(30), learning=True))
fr = synth.frames_dev(cfg, 0, range(64))
masks = torch.empty((64, cfg.H, cfg.W), dtype=torch.uint8, device=dev)
mk = None if os.environ.get("CT_NOMASK") else masks
for it in range(3):
    fz.process_frames(fr, t_ms=np.arange(64) * 33 + it * 10000, masks=mk)
torch.cuda.synchronize()
n = 64
buf = (ctypes.c_ulonglong * (12 * n))()
lib().fizi_diag_ccl_trace(buf, n)
a = np.frombuffer(buf, dtype=np.uint64).reshape(n, 12).astype(np.int64)
t0 = a[:, 0].min()
s, e = (a[:, 0] - t0) / 1e3, (a[:, 1] - t0) / 1e3
d = e - s
rounds = a[:, 2] >> 32
a[:, 2] &= 0xFFFFFFFF
print("T", a[:, 2].min(), a[:, 2].max(), "phase 5a (mask bytes) us p50/max", np.median(rounds) / 1965.0, rounds.max() / 1965.0)
print("start us min %.2f max %.2f | dur us min %.2f p50 %.2f max %.2f | end max %.2f" % (s.min(), s.max(), d.min(), np.median(d), d.max(), e.max()))
f = a[:, 3]
if (f > 0).any():
    print("fold end us %.2f (fold %.2f us after the last CTA end)" % ((f.max() - t0) / 1e3, (f.max() - a[:, 1].max()) / 1e3))

# phase clocks (cycles since kernel entry, 1.965 GHz) -> per-phase us
names = ["entry->load", "load", "union", "flatten", "stats", "select", "blob", "mask/clear"]
ck = a[:, 4:12].astype(np.float64)
prev = np.zeros(n)
for k, nm in enumerate(names):
    dk = (ck[:, k] - prev) / 1965.0
    prev = ck[:, k]
    print("%-12s p50 %7.2f us  max %7.2f us" % (nm, np.median(dk), dk.max()))
print("T per frame p50", int(np.median(a[:, 2])))
