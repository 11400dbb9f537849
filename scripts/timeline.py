"""Diagnostics: device timeline of pipelined calls (FIZI_TIMELINE=1).

Per call: first-CTA start / last-CTA end of each kernel kind (globaltimer),
relative to the call's segmentation start, plus the per-call period."""
import ctypes, os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["FIZI_TIMELINE"] = "1"
import synth
from paper_1907_04393_b200 import Fizi, lib

cid = int(os.environ.get("TL_CONFIG", "3"))
B = int(os.environ.get("TL_BATCH", "64"))
pipelined = os.environ.get("TL_PIPELINE", "1") == "1"
cfg = synth.CONFIGS[cid]
dev = torch.device("cuda", 0)
multi = cfg.streams > 1 and os.environ.get("TL_MULTI") == "1"   # C5: one frame of each of B streams
fz = Fizi(cfg.W, cfg.H, n_streams=B if multi else 1, max_batch=B)
for sid in range(B if multi else 1):
    fz.learn_background(synth.frames_dev(cfg, sid, range(cfg.n_learn), learning=True), stream=sid,
                        margin=synth.MARGIN)
fz.set_pipeline(pipelined)
nb = 4
if multi:
    frames = []
    for b in range(nb):
        fr = torch.empty((B, cfg.H, cfg.W, 3), dtype=torch.uint8, device=dev)
        for sid in range(B):
            synth.frames_dev(cfg, sid, [b], out=fr[sid:sid + 1])
        frames.append(fr)
    sids = np.arange(B, dtype=np.uint32)
else:
    frames = [synth.frames_dev(cfg, 0, range(b * B, (b + 1) * B)) for b in range(nb)]
    sids = None
masks = [torch.empty((B, cfg.H, cfg.W), dtype=torch.uint8, device=dev) for _ in range(4)]
res = [torch.empty((B, 128), dtype=torch.uint8, device=dev) for _ in range(4)]
ncalls = int(os.environ.get("TL_NCALLS", "48"))
nwarm = int(os.environ.get("TL_WARM", "0"))
import time
L0 = lib()
L0.fizi_diag_host_ns.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
hc, hsync = ctypes.c_ulonglong(), ctypes.c_ulonglong()
for i in range(nwarm):          # untimed calls, then an idle pipeline (as bench.py's warm-up)
    fz.process_frames(frames[i % nb], t_ms=np.arange(B, dtype=np.int64) * 33 + (i - nwarm) * B * 33,
                      masks=masks[i % 4], results=res[i % 4])
fz.flush()
torch.cuda.synchronize()
L0.fizi_diag_host_ns(fz._h, ctypes.byref(hc), ctypes.byref(hsync))
c0, s0 = hc.value, hsync.value
tp0 = time.perf_counter()
for i in range(ncalls):
    t = (np.full(B, i * 33, np.int64) if multi else np.arange(B, dtype=np.int64) * 33 + i * B * 33)
    fz.process_frames(frames[i % nb], streams=sids, t_ms=t,
                      masks=None if os.environ.get("TL_NOMASK") else masks[i % 4], results=res[i % 4])
tp1 = time.perf_counter()
L0.fizi_diag_host_ns(fz._h, ctypes.byref(hc), ctypes.byref(hsync))
print("host per call: python+lib %.1f us, inside run_call %.1f us, of which slot wait %.1f us" % (
    (tp1 - tp0) / ncalls * 1e6, (hc.value - c0) / ncalls / 1e3, (hsync.value - s0) / ncalls / 1e3))
fz.flush()
torch.cuda.synchronize()
L = lib()
L.fizi_diag_timeline.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
buf = np.zeros(2 * 8 * 256, np.uint64)
rc = L.fizi_diag_timeline(fz._h, buf.ctypes.data)
assert rc == 0, rc
st = buf[:8 * 256].reshape(8, 256).astype(np.float64)
en = buf[8 * 256:].reshape(8, 256).astype(np.float64)
names = ["seg", "slow", "fix", "zero", "morph", "ccl", "fold"]
print("pipelined" if pipelined else "joined", "C%d B=%d" % (cid, B))
print("call " + " ".join("%15s" % n for n in names) + "   period")
rows = range(nwarm + ncalls) if nwarm else range(ncalls - 12, ncalls)
for k in rows:
    t0 = st[0, k]
    cells = []
    kinds = {"seg": 0, "fix": 1, "zero": 2, "morph": 3, "ccl": 4, "fold": 5, "slow": 6}
    for n in names:
        j = kinds[n]
        if st[j, k] > 1e19:
            cells.append("%15s" % "-")
        else:
            cells.append("%6.1f..%6.1f" % ((st[j, k] - t0) / 1e3, (en[j, k] - t0) / 1e3))
    per = (st[0, k] - st[0, k - 1]) / 1e3
    print("%4d " % k + " ".join(cells) + "   %6.1f" % per)
if nwarm:
    k0, k1 = nwarm, nwarm + ncalls - 1
    span = (max(en[j, k1] for j in range(7) if en[j, k1] < 1e19 and st[j, k1] < 1e19) - st[0, k0]) / 1e3
    print("timed calls %d..%d: first seg start -> last end %.1f us = %.1f us/call -> %.0f frames/s"
          % (k0, k1, span, span / ncalls, B * ncalls / span * 1e6))
per = (st[0, ncalls - 1] - st[0, 8]) / 1e3 / (ncalls - 9)
print("mean period %.1f us -> %.0f frames/s" % (per, B / per * 1e6))
