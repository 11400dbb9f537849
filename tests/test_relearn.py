"""NEXT-1 relearn trigger: oracle pins (the SPEC's
examples) and the device fold (fizi_relearn_flags) against the oracle over the
mean luma of C2's lighting-drift stream, across call boundaries."""
import numpy as np
import pytest

from oracle.relearn import relearn_flags, relearn_trigger


def test_spec_examples():
    assert relearn_trigger(100, 100, 40) is False
    assert relearn_trigger(100, 180, 40) is True
    assert relearn_trigger(100, 140, 40) is False           # S:161 (strict)
    assert relearn_trigger(140, 100, 40) is False
    assert relearn_trigger(180, 100, 40) is True            # |cur - prev|, either direction
    assert relearn_flags([100, 100, 180, 181, 100], 40) == [False, False, True, False, True]


@pytest.mark.gpu
def test_device_flags_match_oracle_on_drift_stream():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import synth
    from paper_1907_04393_b200 import Fizi, results_numpy
    cfg = synth.CONFIGS[2]
    fz = Fizi(cfg.W, cfg.H, max_batch=64)
    fz.learn_background(torch.from_numpy(synth.learning_frames_host(cfg)).cuda(), margin=synth.MARGIN)
    import oracle
    means, flags = [], []
    for k0 in range(0, 640, 64):                  # flags fold across calls
        ks = range(k0, k0 + 64)
        fh = synth.frames_host(cfg, 0, ks)
        fr = torch.from_numpy(fh).cuda()
        _, res = fz.process_frames(fr, t_ms=np.array([synth.t_ms(k) for k in ks], np.int64))
        # the oracle's own a2 mean of every frame (not the device's record field)
        means += [oracle.mean_luma(f)[0] for f in fh]
        flags += [bool(f) for f in fz.relearn_flags(res, threshold=20).cpu().numpy()]
    ref = relearn_flags(means, 20)
    assert flags == ref
    assert any(ref)                               # the drift stream has exposure steps
    fz.close()


# ---------------------------------------------- in-stream relearning (oracle)
def _step_scene(n_before, n_after, gain_after, hand=False, seed=7):
    """A static textured scene (C1 geometry), a lighting step of gain
    `gain_after` (Q10) from frame n_before on; optionally the C1 disc hand."""
    import synth
    cfg = synth.CONFIGS[1]
    n = n_before + n_after
    pf = synth.frame_params(cfg, 0, range(n))
    pf[:, 1] = [1024] * n_before + [gain_after] * n_after
    if not hand:
        pf[:, 4] = 0
    # skin-hued static clutter baked into the background (C4's kind): inside
    # the learned envelope until the lighting changes
    ell = np.array([[80, 60, 40, 30], [240, 170, 50, 35]], np.int32)
    frames = synth.gen_host(cfg.W, cfg.H, cfg.seed, 0, pf, ell)
    lpf = synth.frame_params(cfg, 0, range(cfg.n_learn), learning=True)
    learn = synth.gen_host(cfg.W, cfg.H, cfg.seed, 0, lpf, ell)
    return cfg, frames, learn


def test_relearn_never_triggered_equals_plain_path():
    import oracle
    import synth
    from oracle.relearn import run_stream_relearn
    cfg, frames, learn = _step_scene(4, 4, 1400, hand=True)
    lo, hi = oracle.learn(learn, synth.MARGIN)
    p = oracle.make_params(cfg.W, cfg.H)
    t = np.arange(len(frames)) * 33
    recs, masks, flags, swaps = run_stream_relearn(p, frames, t, lo, hi, 255, 3, synth.MARGIN)
    tr = oracle.Tracker(p)
    assert flags == [0] * len(frames) and swaps == []
    for k in range(len(frames)):
        rec, st = oracle.segment(p, frames[k], lo, hi, t_ms=int(t[k]))
        tr.update(rec)
        assert rec.as_dict() == recs[k].as_dict()
        assert np.array_equal(st["final_mask"], masks[k])


def test_relearn_after_lighting_step_relearns_the_new_background():
    """Static background, exposure x1.25 from frame 3: frame 3 triggers (it is
    segmented with the old model, which now sees the brighter background as
    foreground), frames 4..4+F-1 are learning frames, the model learned from
    them makes the later frames exactly empty again (noise a = 4 <= margin/2,
    the c3 'learn' pin), and the swap's model is learn(those F frames)."""
    import oracle
    import synth
    from oracle.relearn import RELEARN_LEARN, RELEARN_SWAP, RELEARN_TRIGGER, run_stream_relearn
    F = 5
    cfg, frames, learn = _step_scene(3, 12, 1280)
    lo, hi = oracle.learn(learn, synth.MARGIN)
    p = oracle.make_params(cfg.W, cfg.H, min_blob_ppm=0)
    t = np.arange(len(frames)) * 33
    recs, masks, flags, swaps = run_stream_relearn(p, frames, t, lo, hi, 20, F, synth.MARGIN)
    m = [oracle.mean_luma(f)[0] for f in frames]
    assert m[3] - m[2] > 20 and all(abs(m[k] - m[k - 1]) <= 20 for k in range(4, len(m)))
    assert flags == [0, 0, 0, RELEARN_TRIGGER] + [RELEARN_LEARN] * (F - 1) + \
        [RELEARN_LEARN | RELEARN_SWAP] + [0] * (len(frames) - 4 - F)
    assert [k for k, _, _ in swaps] == [3 + F]
    nlo, nhi = oracle.learn(frames[4:4 + F], synth.MARGIN)
    assert np.array_equal(swaps[0][1], nlo) and np.array_equal(swaps[0][2], nhi)
    assert recs[3].fg_merged > 1000                      # the old model fails on the step frame
    assert recs[3].blob_area > 0                         # (the brightened clutter is a "hand")
    for k in range(4, 4 + F):                            # learning: not segmented, not tracked
        assert masks[k].sum() == 0 and recs[k].fg_merged == 0 and recs[k].visible == 0
        assert recs[k].mean_luma == m[k]
    for k in range(4 + F, len(frames)):                  # the relearned model: exactly empty
        assert masks[k].sum() == 0 and recs[k].fg_merged == 0


def test_relearn_ignores_triggers_while_learning_and_resets_the_tracker():
    """Two steps 2 frames apart: the second falls inside the learning window
    and does not restart it; with the hand present the tracker is paused while
    learning and snaps to the centroid (reset) on the first frame after the swap."""
    import oracle
    import synth
    from oracle.relearn import RELEARN_LEARN, RELEARN_TRIGGER, run_stream_relearn
    import synth as sy
    cfg = sy.CONFIGS[1]
    n = 14
    pf = sy.frame_params(cfg, 0, range(n))
    pf[:, 1] = [1024] * 3 + [1300] * 2 + [900] * (n - 5)
    frames = sy.gen_host(cfg.W, cfg.H, cfg.seed, 0, pf, sy.clutter(cfg, 0))
    lo, hi = oracle.learn(sy.learning_frames_host(cfg), sy.MARGIN)
    p = oracle.make_params(cfg.W, cfg.H)
    t = np.arange(n) * 33
    F = 4
    recs, masks, flags, swaps = run_stream_relearn(p, frames, t, lo, hi, 20, F, sy.MARGIN)
    assert flags[3] == RELEARN_TRIGGER
    assert all(flags[k] & RELEARN_LEARN for k in range(4, 4 + F))   # frame 5's step ignored
    assert not any(flags[k] & RELEARN_TRIGGER for k in range(4, 4 + F))
    assert len(swaps) == 1 and swaps[0][0] == 3 + F
    k = 4 + F
    assert recs[k].blob_area > 0 and recs[k].visible == 1
    assert recs[k].px == recs[k].cx and recs[k].py == recs[k].cy    # snapped: tracker reset
    assert recs[k].dwell_ms == 0


# ------------------------------------------ in-stream relearning (GPU vs oracle)
def _gpu_relearn_case(W, H, frames, learn, t, threshold, F, batches, params=None):
    """Run the stream through the device in calls of the given sizes with
    relearning enabled; compare every record (flags, tracker) and mask with
    the oracle composition."""
    import torch
    import oracle
    import synth
    from oracle.relearn import run_stream_relearn
    from paper_1907_04393_b200 import Fizi, results_numpy
    from tests.gpu_common import compare_record
    params = params or {}
    p = oracle.make_params(W, H, **params)
    lo, hi = oracle.learn(learn, synth.MARGIN)
    recs, masks, flags, swaps = run_stream_relearn(p, frames, t, lo, hi, threshold, F, synth.MARGIN)
    fz = Fizi(W, H, max_batch=max(batches), **params)
    fz.learn_background(torch.from_numpy(learn).cuda(), margin=synth.MARGIN)
    fz.set_relearn(threshold=threshold, n_frames=F, margin=synth.MARGIN)
    k0 = 0
    for b in batches:
        if k0 >= len(frames):
            break
        sl = slice(k0, min(len(frames), k0 + b))
        m, r = fz.process_frames(torch.from_numpy(frames[sl]).cuda(), t_ms=t[sl])
        r, m = results_numpy(r), m.cpu().numpy()
        for i, k in enumerate(range(sl.start, sl.stop)):
            assert int(r[i]["relearn"]) == flags[k], (k, int(r[i]["relearn"]), flags[k])
            compare_record(r[i], recs[k], k, track=True)
            assert np.array_equal(m[i], masks[k]), k
        k0 = sl.stop
    # the stream's model after the run = the oracle's last swap model
    if swaps:
        glo, ghi = fz.get_background()
        assert np.array_equal(glo.cpu().numpy(), swaps[-1][1])
        assert np.array_equal(ghi.cpu().numpy(), swaps[-1][2])
    fz.close()
    return flags


@pytest.mark.gpu
@pytest.mark.parametrize("batches", [[15], [4] * 4, [1] * 15, [2, 7, 6]])
def test_gpu_relearn_lighting_step_any_batching(batches):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    cfg, frames, learn = _step_scene(3, 12, 1280)
    t = np.arange(len(frames), dtype=np.int64) * 33
    flags = _gpu_relearn_case(cfg.W, cfg.H, frames, learn, t, 20, 5, batches,
                              dict(min_blob_ppm=0))
    assert flags.count(0) < len(flags)


@pytest.mark.gpu
def test_gpu_relearn_generic_path_and_two_swaps_in_one_call():
    """W % 32 != 0 (generic path); two lighting steps far enough apart that two
    models are learned and swapped inside one call (F = 2)."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import synth
    cfg = synth.CONFIGS[1]
    W, H, n = 100, 60, 16
    pf = synth.frame_params(cfg, 0, range(n))
    pf[:, 2] = 50
    pf[:, 3] = 30
    pf[:, 4] = 12
    pf[:, 1] = [1024] * 3 + [1300] * 6 + [800] * 7
    ell = np.array([[20, 15, 10, 8], [80, 45, 12, 9]], np.int32)
    frames = synth.gen_host(W, H, cfg.seed, 0, pf, ell)
    lpf = synth.frame_params(cfg, 0, range(cfg.n_learn), learning=True)
    learn = synth.gen_host(W, H, cfg.seed, 0, lpf, ell)
    t = np.arange(n, dtype=np.int64) * 33
    flags = _gpu_relearn_case(W, H, frames, learn, t, 20, 2, [16], dict(min_blob_ppm=0))
    from oracle.relearn import RELEARN_SWAP
    assert sum(1 for f in flags if f & RELEARN_SWAP) == 2


@pytest.mark.gpu
def test_gpu_relearn_c2_drift_stream():
    """C2's lighting drift (exposure steps, over-exposure ramp) with relearning
    (threshold 20, F = 10) over 320 frames in calls of 64."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import synth
    cfg = synth.CONFIGS[2]
    ks = list(range(0, 320))
    frames = synth.frames_host(cfg, 0, ks)
    learn = synth.learning_frames_host(cfg)
    t = np.array([synth.t_ms(k) for k in ks], np.int64)
    flags = _gpu_relearn_case(cfg.W, cfg.H, frames, learn, t, 20, 10, [64] * 5)
    from oracle.relearn import RELEARN_SWAP
    assert any(f & RELEARN_SWAP for f in flags)


@pytest.mark.gpu
def test_gpu_relearn_multistream_pipelined_context():
    """Two streams in interleaved calls on a pipelined context: stream 1
    relearns (its calls run joined), stream 0 does not; each stream's records
    and masks equal its own oracle run (the oracle composition for stream 1,
    the plain path for stream 0)."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import oracle
    import synth
    from oracle.relearn import run_stream_relearn
    from paper_1907_04393_b200 import Fizi, results_numpy
    from tests.gpu_common import compare_record
    cfg, step_frames, step_learn = _step_scene(3, 9, 1280)       # stream 1: lighting step
    plain = synth.frames_host(cfg, 0, range(12))                  # stream 0: C1 orbit
    plain_learn = synth.learning_frames_host(cfg)
    p = oracle.make_params(cfg.W, cfg.H, min_blob_ppm=0)
    t = np.arange(12, dtype=np.int64) * 33
    lo0, hi0 = oracle.learn(plain_learn, synth.MARGIN)
    lo1, hi1 = oracle.learn(step_learn, synth.MARGIN)
    r1, m1, f1, _ = run_stream_relearn(p, step_frames, t, lo1, hi1, 20, 4, synth.MARGIN)
    fz = Fizi(cfg.W, cfg.H, n_streams=2, max_batch=8, min_blob_ppm=0)
    fz.learn_background(torch.from_numpy(plain_learn).cuda(), stream=0, margin=synth.MARGIN)
    fz.learn_background(torch.from_numpy(step_learn).cuda(), stream=1, margin=synth.MARGIN)
    fz.set_relearn(stream=1, threshold=20, n_frames=4, margin=synth.MARGIN)
    fz.set_pipeline(True)
    tr0 = oracle.Tracker(p)
    outs = []
    for k0 in range(0, 12, 3):                                    # calls of 3 + 3 frames, interleaved
        ks = list(range(k0, k0 + 3))
        fr = np.concatenate([plain[ks], step_frames[ks]])
        sof = np.array([0, 0, 0, 1, 1, 1], np.uint32)
        tt = np.concatenate([t[ks], t[ks]])
        mk = torch.empty((6, cfg.H, cfg.W), dtype=torch.uint8, device="cuda")
        rs = torch.empty((6, 128), dtype=torch.uint8, device="cuda")
        fz.process_frames(torch.from_numpy(fr).cuda(), streams=sof, t_ms=tt, masks=mk, results=rs)
        outs.append((ks, mk, rs))
    fz.flush()
    torch.cuda.synchronize()
    for ks, mk, rs in outs:
        rr, mm = results_numpy(rs), mk.cpu().numpy()
        for i, k in enumerate(ks):
            rec0, st0 = oracle.segment(p, plain[k], lo0, hi0, t_ms=int(t[k]))
            tr0.update(rec0)
            compare_record(rr[i], rec0, ("s0", k), track=True)
            assert int(rr[i]["relearn"]) == 0
            assert np.array_equal(mm[i], st0["final_mask"])
            compare_record(rr[3 + i], r1[k], ("s1", k), track=True)
            assert int(rr[3 + i]["relearn"]) == f1[k]
            assert np.array_equal(mm[3 + i], m1[k])
    assert any(f1)
    fz.close()
