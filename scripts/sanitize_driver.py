"""Small workload for compute-sanitizer (memcheck / racecheck / synccheck /
initcheck): C1 end to end (joined, debug stages), C2 batches in pipelined
mode (every kernel of the pipelined tail, LUT re-test frames included), a
multi-stream call (seg_multi_kernel) and the fold / NEXT kernels; each result
is checked against the oracle so a sanitizer run also confirms parity."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
import synth  # noqa: E402
from paper_1907_04393_b200 import Fizi, results_numpy  # noqa: E402

dev = torch.device("cuda", 0)


def check(res, masks, frames, lo, hi, p, t):
    res = results_numpy(res)
    tr = oracle.Tracker(p)
    for k in range(len(frames)):
        rec, st = oracle.segment(p, frames[k], lo, hi, t_ms=int(t[k]))
        tr.update(rec)
        assert int(res[k]["fg_final"]) == rec.fg_final and int(res[k]["blob_area"]) == rec.blob_area, k
        assert np.array_equal(masks[k], st["final_mask"]), k


# C1 joined, debug stages
cfg = synth.CONFIGS[1]
learn = synth.learning_frames_host(cfg)
frames = synth.frames_host(cfg, 0, range(cfg.n_proc))
t = np.array([synth.t_ms(k) for k in range(cfg.n_proc)], np.int64)
fz = Fizi(cfg.W, cfg.H, max_batch=cfg.n_proc, debug=1)
fz.learn_background(torch.from_numpy(learn).to(dev), margin=synth.MARGIN)
m, r = fz.process_frames(torch.from_numpy(frames).to(dev), t_ms=t)
for s in ("r1", "r2", "r3", "merged", "openclose", "labels", "final", "contour"):
    fz.debug_stage(s, 3)
torch.cuda.synchronize()
lo, hi = oracle.learn(learn, synth.MARGIN)
check(r, m.cpu().numpy(), frames, lo, hi, oracle.make_params(cfg.W, cfg.H), t)
fz.close()
print("C1 ok", flush=True)

# C2 pipelined, 3 calls in flight (the over-exposure ramp: LUT re-test frames)
cfg = synth.CONFIGS[2]
learn = synth.learning_frames_host(cfg)
lo, hi = oracle.learn(learn, synth.MARGIN)
fz = Fizi(cfg.W, cfg.H, max_batch=16)
fz.learn_background(torch.from_numpy(learn).to(dev), margin=synth.MARGIN)
fz.set_pipeline(True)
outs = []
for b in range(3):
    ks = list(range(100 + 16 * b, 116 + 16 * b))
    fr = synth.frames_host(cfg, 0, ks)
    tt = np.array([synth.t_ms(k) for k in ks], np.int64)
    mk = torch.empty((16, cfg.H, cfg.W), dtype=torch.uint8, device=dev)
    rs = torch.empty((16, 128), dtype=torch.uint8, device=dev)
    fz.process_frames(torch.from_numpy(fr).to(dev), t_ms=tt, masks=mk, results=rs)
    outs.append((fr, tt, mk, rs))
fz.flush()
torch.cuda.synchronize()
p = oracle.make_params(cfg.W, cfg.H)
tr = oracle.Tracker(p)
for fr, tt, mk, rs in outs:
    rr = results_numpy(rs)
    for k in range(len(fr)):
        rec, st = oracle.segment(p, fr[k], lo, hi, t_ms=int(tt[k]))
        tr.update(rec)
        assert int(rr[k]["fg_final"]) == rec.fg_final and int(rr[k]["visible"]) == rec.visible
        assert np.array_equal(mk[k].cpu().numpy(), st["final_mask"])
fz.close()
print("C2 pipelined ok", flush=True)

# multi-stream call (seg_multi_kernel), 6 streams
cfg = synth.CONFIGS[5]
S = 6
fz = Fizi(cfg.W, cfg.H, n_streams=S, max_batch=S)
envs = []
for s in range(S):
    ln = synth.learning_frames_host(cfg, s)
    fz.learn_background(torch.from_numpy(ln).to(dev), stream=s, margin=synth.MARGIN)
    envs.append(oracle.learn(ln, synth.MARGIN))
fr = np.stack([synth.frames_host(cfg, s, [4])[0] for s in range(S)])
m, r = fz.process_frames(torch.from_numpy(fr).to(dev), streams=np.arange(S, dtype=np.uint32),
                         t_ms=np.full(S, 132, np.int64))
torch.cuda.synchronize()
rr, mm = results_numpy(r), m.cpu().numpy()
p = oracle.make_params(cfg.W, cfg.H)
for s in range(S):
    rec, st = oracle.segment(p, fr[s], *envs[s], t_ms=132)
    assert int(rr[s]["fg_final"]) == rec.fg_final and np.array_equal(mm[s], st["final_mask"]), s
flags = fz.relearn_flags(r[:1], stream=0)
torch.cuda.synchronize()
fz.close()
print("C5 multi-stream ok", flush=True)
