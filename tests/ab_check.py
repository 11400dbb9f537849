"""Parity check run in a subprocess by tests/test_gpu_ab_paths.py, so that an
experiment switch (environment variable read once per process by libfizi)
takes effect: C2 frames 30-93 (the over-exposure ramp: LUT re-test frames)
as two joined calls of 32 and two pipelined calls of 32, every mask and
record against the oracle; C3 16 frames joined; multi-stream calls (8 C5
streams).  Prints OK."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
import synth  # noqa: E402
from paper_1907_04393_b200 import RESULT_BYTES, Fizi, results_numpy  # noqa: E402
from tests.gpu_common import compare_record  # noqa: E402

DEV = torch.device("cuda", 0)


def run(cid, ks, B, pipelined):
    cfg = synth.CONFIGS[cid]
    learn = synth.frames_dev(cfg, 0, range(cfg.n_learn), learning=True, device=DEV)
    frames = synth.frames_dev(cfg, 0, ks, device=DEV)
    t = np.array([synth.t_ms(k) for k in ks], np.int64)
    fz = Fizi(cfg.W, cfg.H, max_batch=B)
    fz.learn_background(learn, margin=synth.MARGIN)
    fz.set_pipeline(pipelined)
    outs = []
    for j in range(0, len(ks), B):
        m = torch.empty((B, cfg.H, cfg.W), dtype=torch.uint8, device=DEV)
        r = torch.empty((B, RESULT_BYTES), dtype=torch.uint8, device=DEV)
        fz.process_frames(frames[j:j + B], t_ms=t[j:j + B], masks=m, results=r)
        outs.append((m, r))
    fz.flush()
    torch.cuda.synchronize()
    lo, hi = oracle.learn(learn.cpu().numpy(), synth.MARGIN)
    p = oracle.make_params(cfg.W, cfg.H)
    tr = oracle.Tracker(p)
    recs, om = oracle.segment_batch(p, frames.cpu().numpy(), lo, hi, t_ms=t, nthreads=8)
    corrected = 0
    for j, (m, r) in enumerate(outs):
        rp, mm = results_numpy(r), m.cpu().numpy()
        for i in range(B):
            k = j * B + i
            tr.update(recs[k])
            compare_record(rp[i], recs[k], ks[k], track=True)
            assert np.array_equal(mm[i], om[k]), ks[k]
            corrected += recs[k].corrected
    fz.close()
    return corrected


def run_multi(S=8, rounds=2):
    """C5-like multi-stream calls: the current frame of each of S streams."""
    cfg = synth.CONFIGS[5]
    fz = Fizi(cfg.W, cfg.H, n_streams=S, max_batch=S)
    p = oracle.make_params(cfg.W, cfg.H)
    envs, trs = [], []
    for sid in range(S):
        learn = synth.frames_dev(cfg, sid, range(cfg.n_learn), learning=True, device=DEV)
        fz.learn_background(learn, stream=sid, margin=synth.MARGIN)
        envs.append(oracle.learn(learn.cpu().numpy(), synth.MARGIN))
        trs.append(oracle.Tracker(p))
    ids = np.arange(S, dtype=np.uint32)
    for k in range(100, 100 + rounds):
        fr = torch.empty((S, cfg.H, cfg.W, 3), dtype=torch.uint8, device=DEV)
        for sid in range(S):
            synth.frames_dev(cfg, sid, [k], out=fr[sid:sid + 1], device=DEV)
        t = np.full(S, synth.t_ms(k), np.int64)
        masks, res = fz.process_frames(fr, streams=ids, t_ms=t)
        rp, mm, fh = results_numpy(res), masks.cpu().numpy(), fr.cpu().numpy()
        for sid in range(S):
            rec, st = oracle.segment(p, fh[sid], *envs[sid], t_ms=int(t[sid]))
            trs[sid].update(rec)
            compare_record(rp[sid], rec, (sid, k), track=True)
            assert np.array_equal(mm[sid], st["final_mask"]), (sid, k)
    fz.close()


if __name__ == "__main__":
    run_multi()
    c = run(2, list(range(30, 94)), 32, False)
    c += run(2, list(range(30, 94)), 32, True)
    assert c > 20, c
    run(3, list(range(96, 112)), 16, False)
    print("OK")
