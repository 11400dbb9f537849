"""Diagnostics: host time of the first calls after an idle, synchronised
pipeline (the driver's timed region starts that way)."""
import ctypes, gc, os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth
from paper_1907_04393_b200 import Fizi, lib

cfg = synth.CONFIGS[3]
B = 64
dev = torch.device("cuda", 0)
fz = Fizi(cfg.W, cfg.H, max_batch=B)
fz.learn_background(synth.frames_dev(cfg, 0, range(cfg.n_learn), learning=True), margin=synth.MARGIN)
fz.set_pipeline(True)
frames = [synth.frames_dev(cfg, 0, range(b * B, (b + 1) * B)) for b in range(4)]
masks = [torch.empty((B, cfg.H, cfg.W), dtype=torch.uint8, device=dev) for _ in range(4)]
res = [torch.empty((B, 128), dtype=torch.uint8, device=dev) for _ in range(4)]
L = lib()
L.fizi_diag_host_ns.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
hc, hs = ctypes.c_ulonglong(), ctypes.c_ulonglong()
k = [0]


def call():
    i = k[0]
    k[0] += 1
    L.fizi_diag_host_ns(fz._h, ctypes.byref(hc), ctypes.byref(hs))
    c0, s0 = hc.value, hs.value
    t0 = time.perf_counter()
    fz.process_frames(frames[i % 4], t_ms=np.arange(B, dtype=np.int64) * 33 + i * B * 33,
                      masks=masks[i % 4], results=res[i % 4])
    t1 = time.perf_counter()
    L.fizi_diag_host_ns(fz._h, ctypes.byref(hc), ctypes.byref(hs))
    return (t1 - t0) * 1e6, (hc.value - c0) / 1e3, (hs.value - s0) / 1e3


for variant in ["plain", "plain", "sleep1ms", "spin", "nogc"]:
    for _ in range(5):
        call()
    fz.flush()
    torch.cuda.synchronize()
    if variant == "sleep1ms":
        time.sleep(0.001)
    if variant == "spin":
        t = time.perf_counter()
        while time.perf_counter() - t < 0.002:
            pass
    if variant == "nogc":
        gc.collect(); gc.disable()
    out = [call() for _ in range(5)]
    gc.enable()
    print(variant, " ".join("%.0f/%.0f/%.0f" % o for o in out), flush=True)
fz.flush()
torch.cuda.synchronize()
