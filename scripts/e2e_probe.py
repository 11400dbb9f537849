"""fizi_process_frames_host on C3 (64 frames per call): time per call with and
without the mask read-back, and the pure H2D time of the same bytes."""
import os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth
from paper_1907_04393_b200 import Fizi, RESULT_DTYPE
cfg = synth.CONFIGS[3]
B = 64
fe = Fizi(cfg.W, cfg.H, max_batch=B)
fe.learn_background(synth.frames_dev(cfg, 0, range(cfg.n_learn), learning=True), margin=synth.MARGIN)
fr = synth.frames_dev(cfg, 0, range(B))
h = torch.empty((B, cfg.H, cfg.W, 3), dtype=torch.uint8).pin_memory()
h.copy_(fr)
hn = h.numpy()
mh = torch.empty((B, cfg.H, cfg.W), dtype=torch.uint8).pin_memory().numpy()
res = np.zeros(B, RESULT_DTYPE)
t = np.arange(B, dtype=np.int64) * 33
step = [0]
if os.environ.get("E2E_PIPE"):
    fe.set_pipeline(True)
for masks in (mh, None):
    for i in range(3):
        step[0] += 1
        fe.process_frames_host(hn, t_ms=t + step[0] * 100000, masks=masks, results=res)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    K = 10
    for i in range(K):
        step[0] += 1
        fe.process_frames_host(hn, t_ms=t + step[0] * 100000, masks=masks, results=res)
    dt = (time.perf_counter() - t0) / K
    print("masks" if masks is not None else "no masks", "per call %.2f ms -> %.0f frames/s, H2D %.1f GB/s"
          % (dt * 1e3, B / dt, hn.nbytes / dt / 1e9))
d = torch.empty_like(fr)
torch.cuda.synchronize(); t0 = time.perf_counter()
for i in range(10):
    d.copy_(h, non_blocking=True)
torch.cuda.synchronize(); dt = (time.perf_counter() - t0) / 10
print("pure H2D per call %.2f ms (%.1f GB/s)" % (dt * 1e3, hn.nbytes / dt / 1e9))
