"""GPU parity of pipelined calls in the launch configuration bench.py times:
several calls in flight with no flush between them (call k's tail overlaps
call k+1's segmentation), one flush at the end, then every output compared
with joined calls (bit-exact) and sampled frames with the oracle."""
import numpy as np
import pytest

import oracle
import synth
from tests.gpu_common import compare_record

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_1907_04393_b200 import RESULT_BYTES, Fizi, results_numpy  # noqa: E402

DEV = torch.device("cuda", 0)


def _t(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(DEV)


@pytest.mark.parametrize("B,ncalls", [(32, 6), (64, 4)])
def test_pipelined_c3_calls_in_flight(B, ncalls):
    """C3 (1920x1080), pipelined calls back to back (64 frames per call =
    bench.py's launch configuration), no flush until the end, each call with
    its own output buffers."""
    cfg = synth.CONFIGS[3]
    learn = synth.frames_dev(cfg, 0, range(cfg.n_learn), learning=True, device=DEV)
    ks = list(range(80, 80 + B * ncalls))          # includes a dwell pause (frames 100-139)
    frames = synth.frames_dev(cfg, 0, ks, device=DEV)
    t = np.array([synth.t_ms(k) for k in ks], np.int64)
    pip = Fizi(cfg.W, cfg.H, max_batch=B)
    ref = Fizi(cfg.W, cfg.H, max_batch=B)
    for fz in (pip, ref):
        fz.learn_background(learn, margin=synth.MARGIN)
    pip.set_pipeline(True)
    outs = [(torch.empty((B, cfg.H, cfg.W), dtype=torch.uint8, device=DEV),
             torch.empty((B, RESULT_BYTES), dtype=torch.uint8, device=DEV)) for _ in range(ncalls)]
    for j in range(ncalls):
        sl = slice(j * B, (j + 1) * B)
        pip.process_frames(frames[sl], t_ms=t[sl], masks=outs[j][0], results=outs[j][1])
    pip.flush()
    torch.cuda.synchronize()
    lo, hi = oracle.learn(learn.cpu().numpy(), synth.MARGIN)
    p = oracle.make_params(cfg.W, cfg.H)
    tr = oracle.Tracker(p)
    for j in range(ncalls):
        sl = slice(j * B, (j + 1) * B)
        mr, rr = ref.process_frames(frames[sl], t_ms=t[sl])
        assert torch.equal(mr, outs[j][0]), j
        assert torch.equal(rr, outs[j][1]), j
        rp = results_numpy(outs[j][1])
        fr_h = frames[sl].cpu().numpy()
        for i in range(B):
            sample = i in (0, B - 1) or (j * B + i) % 37 == 0
            rec, st = oracle.segment(p, fr_h[i], lo, hi, t_ms=int(t[j * B + i]), stages=sample)
            tr.update(rec)
            compare_record(rp[i], rec, ks[j * B + i], track=True)
            if sample:
                assert np.array_equal(outs[j][0][i].cpu().numpy(), st["final_mask"])
    pip.close()
    ref.close()


def test_pipelined_c4_two_calls_of_64_in_flight():
    """C4 (3840x2160) in bench.py's launch configuration: pipelined calls of
    64 frames, two in flight, one flush; every mask and record of all 128
    frames against the oracle (frame-parallel over the host cores) and the
    fold over them, in order."""
    import os
    cfg = synth.CONFIGS[4]
    B, ncalls = 64, 2
    learn = synth.frames_dev(cfg, 0, range(cfg.n_learn), learning=True, device=DEV)
    ks = list(range(64, 64 + B * ncalls))          # hand present, a dwell pause at 100-139
    frames = synth.frames_dev(cfg, 0, ks, device=DEV)
    t = np.array([synth.t_ms(k) for k in ks], np.int64)
    fz = Fizi(cfg.W, cfg.H, max_batch=B)
    fz.learn_background(learn, margin=synth.MARGIN)
    fz.set_pipeline(True)
    outs = [(torch.empty((B, cfg.H, cfg.W), dtype=torch.uint8, device=DEV),
             torch.empty((B, RESULT_BYTES), dtype=torch.uint8, device=DEV)) for _ in range(ncalls)]
    for j in range(ncalls):
        sl = slice(j * B, (j + 1) * B)
        fz.process_frames(frames[sl], t_ms=t[sl], masks=outs[j][0], results=outs[j][1])
    fz.flush()
    torch.cuda.synchronize()
    lo, hi = oracle.learn(learn.cpu().numpy(), synth.MARGIN)
    p = oracle.make_params(cfg.W, cfg.H)
    tr = oracle.Tracker(p)
    nthreads = max(1, min(32, os.cpu_count() or 1))
    for j in range(ncalls):
        sl = slice(j * B, (j + 1) * B)
        recs, om = oracle.segment_batch(p, frames[sl].cpu().numpy(), lo, hi, t_ms=t[sl],
                                        nthreads=nthreads)
        rp = results_numpy(outs[j][1])
        got = outs[j][0].cpu().numpy()
        for i in range(B):
            tr.update(recs[i])
            compare_record(rp[i], recs[i], ks[j * B + i], track=True)
            assert np.array_equal(got[i], om[i]), ks[j * B + i]
    fz.close()


def test_pipelined_c2_drift_four_calls_in_flight():
    """C2 (640x480, lighting drift) in bench.py's launch configuration: four
    pipelined calls of 64 frames in flight over frames 0-255, which hold the
    over-exposure ramp (LUT re-test frames, every gamma regime) and a dwell
    pause; every mask and record against the oracle, the fold in order."""
    cfg = synth.CONFIGS[2]
    B, ncalls = 64, 4
    learn = synth.frames_dev(cfg, 0, range(cfg.n_learn), learning=True, device=DEV)
    ks = list(range(B * ncalls))
    frames = synth.frames_dev(cfg, 0, ks, device=DEV)
    t = np.array([synth.t_ms(k) for k in ks], np.int64)
    fz = Fizi(cfg.W, cfg.H, max_batch=B)
    fz.learn_background(learn, margin=synth.MARGIN)
    fz.set_pipeline(True)
    outs = [(torch.empty((B, cfg.H, cfg.W), dtype=torch.uint8, device=DEV),
             torch.empty((B, RESULT_BYTES), dtype=torch.uint8, device=DEV)) for _ in range(ncalls)]
    for j in range(ncalls):
        sl = slice(j * B, (j + 1) * B)
        fz.process_frames(frames[sl], t_ms=t[sl], masks=outs[j][0], results=outs[j][1])
    fz.flush()
    torch.cuda.synchronize()
    lo, hi = oracle.learn(learn.cpu().numpy(), synth.MARGIN)
    p = oracle.make_params(cfg.W, cfg.H)
    tr = oracle.Tracker(p)
    corrected = 0
    for j in range(ncalls):
        sl = slice(j * B, (j + 1) * B)
        recs, om = oracle.segment_batch(p, frames[sl].cpu().numpy(), lo, hi, t_ms=t[sl], nthreads=8)
        rp = results_numpy(outs[j][1])
        got = outs[j][0].cpu().numpy()
        for i in range(B):
            tr.update(recs[i])
            compare_record(rp[i], recs[i], ks[j * B + i], track=True)
            assert np.array_equal(got[i], om[i]), ks[j * B + i]
            corrected += recs[i].corrected
    assert corrected > 50
    fz.close()


def test_pipelined_c5_all_streams_four_calls_in_flight():
    """C5: each call holds the current frame of all 256 streams (bench.py's
    launch configuration), 4 pipelined calls without a flush between them."""
    cfg = synth.CONFIGS[5]
    S, ncalls = cfg.streams, 4
    pip = Fizi(cfg.W, cfg.H, n_streams=S, max_batch=S)
    ref = Fizi(cfg.W, cfg.H, n_streams=S, max_batch=S)
    for s in range(S):
        learn = synth.frames_dev(cfg, s, range(cfg.n_learn), learning=True, device=DEV)
        pip.learn_background(learn, stream=s, margin=synth.MARGIN)
        ref.learn_background(learn, stream=s, margin=synth.MARGIN)
    pip.set_pipeline(True)
    sids = np.arange(S, dtype=np.uint32)
    calls = []
    for k in range(ncalls):
        fr = torch.empty((S, cfg.H, cfg.W, 3), dtype=torch.uint8, device=DEV)
        for s in range(S):
            synth.frames_dev(cfg, s, [k], out=fr[s:s + 1], device=DEV)
        calls.append((fr, np.full(S, synth.t_ms(k), np.int64)))
    outs = [(torch.empty((S, cfg.H, cfg.W), dtype=torch.uint8, device=DEV),
             torch.empty((S, RESULT_BYTES), dtype=torch.uint8, device=DEV)) for _ in range(ncalls)]
    for k, (fr, t) in enumerate(calls):
        pip.process_frames(fr, streams=sids, t_ms=t, masks=outs[k][0], results=outs[k][1])
    pip.flush()
    torch.cuda.synchronize()
    for k, (fr, t) in enumerate(calls):
        mr, rr = ref.process_frames(fr, streams=sids, t_ms=t)
        assert torch.equal(mr, outs[k][0]), k
        assert torch.equal(rr, outs[k][1]), k
    p = oracle.make_params(cfg.W, cfg.H)
    for s in (0, 77, 255):
        lo, hi = oracle.learn(synth.learning_frames_host(cfg, s), synth.MARGIN)
        tr = oracle.Tracker(p)
        for k, (fr, t) in enumerate(calls):
            rec, st = oracle.segment(p, fr[s].cpu().numpy(), lo, hi, t_ms=int(t[s]))
            tr.update(rec)
            compare_record(results_numpy(outs[k][1])[s], rec, (s, k), track=True)
            assert np.array_equal(outs[k][0][s].cpu().numpy(), st["final_mask"]), (s, k)
    pip.close()
    ref.close()


def test_reset_tracker_ordered_after_pipelined_fold():
    """fizi_reset_tracker between pipelined calls (no flush): the reset is
    ordered after the earlier call's fold, so the next call starts from the
    initial tracker state (timestamps may restart)."""
    cfg = synth.CONFIGS[1]
    learn = synth.learning_frames_host(cfg)
    frames = _t(synth.frames_host(cfg, 0, range(cfg.n_proc)))
    t = np.array([synth.t_ms(k) for k in range(cfg.n_proc)], np.int64)
    fz = Fizi(cfg.W, cfg.H, max_batch=cfg.n_proc)
    fz.learn_background(_t(learn), margin=synth.MARGIN)
    fz.set_pipeline(True)
    r1 = torch.empty((cfg.n_proc, RESULT_BYTES), dtype=torch.uint8, device=DEV)
    r2 = torch.empty_like(r1)
    fz.process_frames(frames, t_ms=t, results=r1)
    fz.reset_tracker()
    fz.process_frames(frames, t_ms=t, results=r2)       # same timestamps again
    fz.flush()
    torch.cuda.synchronize()
    a, b = results_numpy(r1), results_numpy(r2)
    assert a.tobytes() == b.tobytes()
    fz.close()


def test_track_runs_equals_track_of_concatenation():
    """fizi_track_runs (the sharded path's window fold: rows of several rank
    blocks, in frame order, one launch) equals fizi_track over the
    concatenated records, and the oracle fold."""
    cfg = synth.CONFIGS[3]
    ks = list(range(95, 95 + 24))                       # a dwell pause starts at frame 100
    learn = synth.frames_dev(cfg, 0, range(cfg.n_learn), learning=True, device=DEV)
    frames = synth.frames_dev(cfg, 0, ks, device=DEV)
    t = np.array([synth.t_ms(k) for k in ks], np.int64)
    seg = Fizi(cfg.W, cfg.H, max_batch=24)
    seg.learn_background(learn, margin=synth.MARGIN)
    _, rec = seg.segment_frames(frames, t_ms=t, masks=None)
    # a "gathered" buffer: 2 rank blocks of 2 steps x 6 rows, frames laid out
    # step-major, then rank (rank r's step j = frames (2j + r) * 6 ..)
    G, B, world = 2, 6, 2
    gathered = torch.empty((world * G * B, RESULT_BYTES), dtype=torch.uint8, device=DEV)
    runs = []
    for j in range(G):
        for r in range(world):
            src = (j * world + r) * B
            dst = r * G * B + j * B
            gathered[dst: dst + B] = rec[src: src + B]
            runs.append((dst, B))
    ref = rec[: world * G * B].clone()
    a = Fizi(cfg.W, cfg.H, max_batch=24)
    b = Fizi(cfg.W, cfg.H, max_batch=24)
    a.track(ref)
    b.track_runs(gathered, runs)
    torch.cuda.synchronize()
    got = torch.cat([gathered[o: o + n] for o, n in runs])
    assert torch.equal(got, ref)
    p = oracle.make_params(cfg.W, cfg.H)
    tr = oracle.Tracker(p)
    rows = results_numpy(ref)
    for i, row in enumerate(rows):
        o = oracle.record_from_blob(int(row["t_ms"]), int(row["blob_area"]), float(row["cx"]),
                                    float(row["cy"]))
        tr.update(o)
        assert (int(row["visible"]), int(row["clicked"]), int(row["dwell_ms"])) == (
            o.visible, o.clicked, o.dwell_ms), i
        assert abs(float(row["px"]) - o.px) <= 1e-3 and abs(float(row["py"]) - o.py) <= 1e-3
    for fz in (seg, a, b):
        fz.close()
