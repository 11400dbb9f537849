"""GPU parity: the CUDA path through the C ABI vs the CPU oracle, element by
element on the same seeded inputs.  Masks, labels and integer fields must be
bit-exact; gamma / centroid / pointer within 1e-3 (north star)."""
import numpy as np
import pytest

import oracle
import synth
from tests.gpu_common import compare_record, oracle_run
from tests.helpers import all_masks, mask_frames

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_1907_04393_b200 import Fizi, FiziError, results_numpy  # noqa: E402

DEV = torch.device("cuda", 0)
STAGE_MAP = {"r1": "r1", "r2": "r2", "r3": "r3", "merged": "merged", "openclose": "oc",
             "labels": "labels", "final": "final_mask", "contour": "contour"}


def _t(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(DEV)


def _ctx(W, H, **kw):
    n_streams = kw.pop("n_streams", 1)
    max_batch = kw.pop("max_batch", 64)
    return Fizi(W, H, n_streams=n_streams, max_batch=max_batch, **kw)


def _run_stages_case(W, H, frames, lo, hi, params, t_ms=None):
    """Install (lo, hi) on the GPU, run the batch, compare every stage + record."""
    n = frames.shape[0]
    t_ms = np.arange(n, dtype=np.int64) * 33 if t_ms is None else t_ms
    fz = _ctx(W, H, debug=1, max_batch=max(n, 1), **params)
    fz.set_background(_t(lo), _t(hi))
    masks, res = fz.process_frames(_t(frames), t_ms=t_ms)
    res = results_numpy(res)
    masks = masks.cpu().numpy()
    p = oracle.make_params(W, H, **params)
    tr = oracle.Tracker(p)
    for k in range(n):
        rec, st = oracle.segment(p, frames[k], lo, hi, t_ms=int(t_ms[k]))
        tr.update(rec)
        compare_record(res[k], rec, k, track=True)
        assert np.array_equal(masks[k], st["final_mask"]), k
        for sname, oname in STAGE_MAP.items():
            got = fz.debug_stage(sname, k).cpu().numpy()
            want = st[oname]
            if sname == "labels":
                got = got.view(np.uint32)
            assert np.array_equal(got, want), (k, sname, int((got != want).sum()))
    fz.close()


# ------------------------------------------------------------------ config 1
def test_config1_end_to_end():
    cfg = synth.CONFIGS[1]
    learn = synth.learning_frames_host(cfg)
    frames = synth.frames_host(cfg, 0, range(cfg.n_proc))
    t = np.array([synth.t_ms(k) for k in range(cfg.n_proc)], np.int64)
    fz = _ctx(cfg.W, cfg.H, debug=1, max_batch=cfg.n_proc)
    fz.learn_background(_t(learn), margin=synth.MARGIN)
    lo, hi = oracle.learn(learn, synth.MARGIN)
    glo, ghi = fz.get_background()
    assert np.array_equal(glo.cpu().numpy(), lo) and np.array_equal(ghi.cpu().numpy(), hi)
    masks, res = fz.process_frames(_t(frames), t_ms=t)
    res = results_numpy(res)
    masks = masks.cpu().numpy()
    p = oracle.make_params(cfg.W, cfg.H)
    tr = oracle.Tracker(p)
    for k in range(cfg.n_proc):
        rec, st = oracle.segment(p, frames[k], lo, hi, t_ms=int(t[k]))
        tr.update(rec)
        compare_record(res[k], rec, k, track=True)
        assert np.array_equal(masks[k], st["final_mask"])
        for sname, oname in STAGE_MAP.items():
            got = fz.debug_stage(sname, k).cpu().numpy()
            if sname == "labels":
                got = got.view(np.uint32)
            assert np.array_equal(got, st[oname]), (k, sname)
    fz.close()


def test_learning_frames_segment_empty():
    cfg = synth.CONFIGS[1]
    learn = synth.learning_frames_host(cfg)
    fz = _ctx(cfg.W, cfg.H)
    fz.learn_background(_t(learn), margin=synth.MARGIN)
    masks, res = fz.segment_frames(_t(learn))
    res = results_numpy(res)
    assert int(masks.sum()) == 0 and (res["fg_merged"] == 0).all()
    fz.close()


# -------------------------------------------------------- random frames, stages
@pytest.mark.parametrize("W,H", [(64, 48), (96, 33), (50, 37), (7, 5), (1, 1)])
def test_random_frames_all_stages(W, H):
    rng = np.random.default_rng(W * 1000 + H)
    n = 6
    frames = rng.integers(0, 256, (n, H, W, 3), dtype=np.uint8)
    # paint skin-ish blobs so components exist
    for k in range(n):
        m = rng.random((H, W)) < 0.3
        kk = int(m.sum())
        frames[k][m] = np.stack([rng.integers(170, 256, kk), rng.integers(60, 140, kk),
                                 rng.integers(40, 120, kk)], -1)
    lo = rng.integers(0, 140, (H, W, 3)).astype(np.uint8)
    hi = np.minimum(255, lo.astype(int) + rng.integers(0, 120, (H, W, 3))).astype(np.uint8)
    for params in (dict(), dict(gray_tol_S=0, hue_lo_deg=10, hue_hi_deg=200, min_blob_ppm=0),
                   dict(se_radius=2, min_blob_ppm=20000, hue_lo_deg=300, hue_hi_deg=60)):
        _run_stages_case(W, H, frames, lo, hi, params)


@pytest.mark.parametrize("W,H,params", [(4160, 40, dict()),                 # P = 130 words > 128
                                         (96, 64, dict(se_radius=5)),       # r > 4
                                         (4128, 24, dict(se_radius=6, min_blob_ppm=0))])
def test_generic_morphology_path(W, H, params):
    """Rows wider than 4096 pixels or structuring elements with r > 4 take
    the shared-memory morphology kernel (morph_runs_kernel) beside the fused
    segmentation; masks and records against the oracle, with and without the
    debug stages."""
    rng = np.random.default_rng(W + H)
    n = 4
    frames = rng.integers(0, 256, (n, H, W, 3), dtype=np.uint8)
    for k in range(n):
        yy, xx = np.mgrid[0:H, 0:W]
        cx, cy, r = rng.integers(0, W), rng.integers(0, H), rng.integers(8, 30)
        m = ((xx - cx) ** 2 + (yy - cy) ** 2 < r * r) | (rng.random((H, W)) < 0.05)
        frames[k][m] = (210, 120, 110)
    lo = rng.integers(0, 140, (H, W, 3)).astype(np.uint8)
    hi = np.minimum(255, lo.astype(int) + rng.integers(0, 120, (H, W, 3))).astype(np.uint8)
    _run_stages_case(W, H, frames, lo, hi, params)
    t = np.arange(n, dtype=np.int64) * 33
    fz = _ctx(W, H, max_batch=n, **params)
    fz.set_background(_t(lo), _t(hi))
    masks, res = fz.process_frames(_t(frames), t_ms=t)
    res, masks = results_numpy(res), masks.cpu().numpy()
    p = oracle.make_params(W, H, **params)
    tr = oracle.Tracker(p)
    for k in range(n):
        rec, st = oracle.segment(p, frames[k], lo, hi, t_ms=int(t[k]))
        tr.update(rec)
        compare_record(res[k], rec, k, track=True)
        assert np.array_equal(masks[k], st["final_mask"]), k
    fz.close()


def test_brightness_regimes_all_means():
    # uniform-ish frames at every mean luma -> every LUT regime, fast path
    W, H = 64, 32
    rng = np.random.default_rng(7)
    frames = []
    for m in range(0, 256, 5):
        f = np.clip(m + rng.integers(-3, 4, (H, W, 3)), 0, 255).astype(np.uint8)
        f[8:20, 10:40] = np.clip(np.array([m + 60, m - 20, m - 30]), 0, 255)
        frames.append(f)
    frames = np.stack(frames)
    lo = np.full((H, W, 3), 90, np.uint8)
    hi = np.full((H, W, 3), 110, np.uint8)
    _run_stages_case(W, H, frames, lo, hi, dict(min_blob_ppm=0))


# ----------------------------------------------------------- exhaustive masks
def test_exhaustive_4x4_masks_generic_path():
    masks = all_masks(4, 4)
    frames, lo, hi = mask_frames(masks)
    n = frames.shape[0]
    fz = Fizi(4, 4, n_streams=1, max_batch=65535, min_blob_ppm=0)
    fz.set_background(_t(lo), _t(hi))
    out = []
    for b in range(0, n, 65535):
        m, r = fz.segment_frames(_t(frames[b:b + 65535]))
        out.append((m.cpu().numpy(), results_numpy(r)))
    gm = np.concatenate([o[0] for o in out])
    gr = np.concatenate([o[1] for o in out])
    p = oracle.make_params(4, 4, min_blob_ppm=0)
    recs, om = oracle.segment_batch(p, frames, lo, hi, nthreads=8)
    assert np.array_equal(gm, om)
    for k in range(0, n, 1):
        r, rec = gr[k], recs[k]
        if (int(r["n_comp_total"]), int(r["blob_label"]), int(r["blob_area"]), int(r["sum_x"]),
                int(r["sum_y"])) != (rec.n_comp_total, rec.blob_label, rec.blob_area, rec.sum_x,
                                     rec.sum_y):
            compare_record(r, rec, k)
    fz.close()


def test_random_32x32_masks_fast_path():
    rng = np.random.default_rng(11)
    masks = (rng.random((1000, 32, 32)) < rng.uniform(0.05, 0.8, (1000, 1, 1))).astype(np.uint8)
    frames, lo, hi = mask_frames(masks)
    fz = Fizi(32, 32, n_streams=1, max_batch=1000, min_blob_ppm=0, debug=1)
    fz.set_background(_t(lo), _t(hi))
    gm, gr = fz.segment_frames(_t(frames))
    gm, gr = gm.cpu().numpy(), results_numpy(gr)
    p = oracle.make_params(32, 32, min_blob_ppm=0)
    for k in range(0, 1000, 1):
        rec, st = oracle.segment(p, frames[k], lo, hi)
        assert np.array_equal(gm[k], st["final_mask"]), k
        compare_record(gr[k], rec, k)
        if k % 50 == 0:
            lab = fz.debug_stage("labels", k).cpu().numpy().view(np.uint32)
            assert np.array_equal(lab, st["labels"]), k
    fz.close()


# ---------------------------------------------------------------- RGB cube
@pytest.mark.parametrize("case", ["default", "nowrap", "S0", "dark", "bright"])
def test_rgb_cube_merged_bit_exact(case):
    r, g, b = np.meshgrid(np.arange(256), np.arange(256), np.arange(256), indexing="ij")
    cube = np.stack([r, g, b], -1).astype(np.uint8).reshape(4096, 4096, 3)
    params = dict(min_blob_ppm=0)
    if case == "nowrap":
        params.update(hue_lo_deg=5, hue_hi_deg=50)
    if case == "S0":
        params.update(gray_tol_S=0, hue_lo_deg=0, hue_hi_deg=359)
    if case == "dark":            # >= 7382 rows of 0 -> mean <= 45 -> gamma 0.4
        cube = np.concatenate([cube, np.zeros((7424, 4096, 3), np.uint8)])
    if case == "bright":          # >= 4396 rows of 255 -> mean >= 194 -> gamma 2.5
        cube = np.concatenate([cube, np.full((4416, 4096, 3), 255, np.uint8)])
    H, W = cube.shape[:2]
    rng = np.random.default_rng(3)
    lo = rng.integers(0, 100, (H, W, 3)).astype(np.uint8)
    hi = (lo.astype(int) + rng.integers(0, 150, (H, W, 3))).clip(0, 255).astype(np.uint8)
    fz = Fizi(W, H, n_streams=1, max_batch=1, debug=1, **params)
    fz.set_background(_t(lo), _t(hi))
    _, res = fz.segment_frames(_t(cube[None]))
    res = results_numpy(res)
    got = fz.debug_stage("merged", 0).cpu().numpy()
    p = oracle.make_params(W, H, **params)
    rec, st = oracle.segment(p, cube, lo, hi)
    assert int(res[0]["mean_luma"]) == rec.mean_luma
    if case == "dark":
        assert rec.gamma == 0.4
    if case == "bright":
        assert rec.gamma == 2.5
    assert np.array_equal(got, st["merged"]), int((got != st["merged"]).sum())
    compare_record(res[0], rec)
    fz.close()


# --------------------------------------------------------- configs 2 .. 5
def _config_parity(cid, ks, stream=0, full_stages=False):
    cfg = synth.CONFIGS[cid]
    learn = synth.learning_frames_host(cfg, stream)
    frames = synth.frames_host(cfg, stream, ks)
    t = np.array([synth.t_ms(k) for k in ks], np.int64)
    fz = _ctx(cfg.W, cfg.H, max_batch=len(ks))
    fz.learn_background(_t(learn), margin=synth.MARGIN)
    masks, res = fz.process_frames(_t(frames), t_ms=t)
    res = results_numpy(res)
    masks = masks.cpu().numpy()
    lo, hi = oracle.learn(learn, synth.MARGIN)
    p = oracle.make_params(cfg.W, cfg.H)
    recs, om = oracle_run(p, frames, lo, hi, t)
    tr = oracle.Tracker(p)
    for k in range(len(ks)):
        tr.update(recs[k])
        compare_record(res[k], recs[k], ks[k], track=True)
        assert np.array_equal(masks[k], om[k]), ks[k]
    fz.close()
    return res


def test_config2_lighting_drift_full_sequence():
    # 1000 frames in batches of 64 through one context: drift, exposure steps,
    # every gamma regime, pauses (clicks) and absences (visibility timeout)
    cfg = synth.CONFIGS[2]
    learn = synth.learning_frames_host(cfg)
    lo, hi = oracle.learn(learn, synth.MARGIN)
    p = oracle.make_params(cfg.W, cfg.H)
    tr = oracle.Tracker(p)
    fz = _ctx(cfg.W, cfg.H, max_batch=64)
    fz.learn_background(_t(learn), margin=synth.MARGIN)
    corrected = clicks = 0
    for b0 in range(0, cfg.n_proc, 64):
        ks = list(range(b0, min(cfg.n_proc, b0 + 64)))
        frames = synth.frames_host(cfg, 0, ks)
        t = np.array([synth.t_ms(k) for k in ks], np.int64)
        masks, res = fz.process_frames(_t(frames), t_ms=t)
        res, masks = results_numpy(res), masks.cpu().numpy()
        recs, om = oracle_run(p, frames, lo, hi, t)
        for i, k in enumerate(ks):
            tr.update(recs[i])
            compare_record(res[i], recs[i], k, track=True)
            assert np.array_equal(masks[i], om[i]), k
            corrected += recs[i].corrected
            clicks += recs[i].clicked
    assert corrected > 100 and clicks >= 2
    fz.close()


def test_config3_sampled_batch():
    _config_parity(3, list(range(96, 96 + 16)))


def test_config4_sampled_batch():
    _config_parity(4, [0, 1, 700, 2000])


def test_config5_multi_stream_batch():
    cfg = synth.CONFIGS[5]
    S = 8
    fz = _ctx(cfg.W, cfg.H, n_streams=S, max_batch=3 * S)
    envs = []
    for s in range(S):
        learn = synth.learning_frames_host(cfg, s)
        fz.learn_background(_t(learn), stream=s, margin=synth.MARGIN)
        envs.append(oracle.learn(learn, synth.MARGIN))
    # 3 steps x S streams, interleaved stream order within the batch
    ks = [0, 1, 2]
    frames, sof, t = [], [], []
    for k in ks:
        for s in range(S):
            frames.append(synth.frames_host(cfg, s, [k])[0])
            sof.append(s)
            t.append(synth.t_ms(k))
    frames = np.stack(frames)
    masks, res = fz.process_frames(_t(frames), streams=sof, t_ms=t)
    res, masks = results_numpy(res), masks.cpu().numpy()
    p = oracle.make_params(cfg.W, cfg.H)
    trs = [oracle.Tracker(p) for _ in range(S)]
    for i in range(len(frames)):
        s = sof[i]
        rec, st = oracle.segment(p, frames[i], envs[s][0], envs[s][1], t_ms=t[i])
        trs[s].update(rec)
        compare_record(res[i], rec, i, track=True)
        assert int(res[i]["stream"]) == s
        assert np.array_equal(masks[i], st["final_mask"])
    fz.close()


def test_config5_all_streams_one_call_sampled():
    """bench.py's C5 launch configuration: one call holds the current frame of
    all 256 streams (device-learned per-stream envelopes, device-generated
    frames); 12 sampled streams are checked against the oracle (envelope,
    record with the fold, final mask)."""
    cfg = synth.CONFIGS[5]
    S = cfg.streams
    fz = _ctx(cfg.W, cfg.H, n_streams=S, max_batch=S)
    for s in range(S):
        fz.learn_background(synth.frames_dev(cfg, s, range(cfg.n_learn), learning=True,
                                             device=DEV), stream=s, margin=synth.MARGIN)
    k = 7
    fr = torch.empty((S, cfg.H, cfg.W, 3), dtype=torch.uint8, device=DEV)
    for s in range(S):
        synth.frames_dev(cfg, s, [k], out=fr[s:s + 1], device=DEV)
    t = np.full(S, synth.t_ms(k), np.int64)
    masks, res = fz.process_frames(fr, streams=np.arange(S, dtype=np.uint32), t_ms=t)
    res = results_numpy(res)
    p = oracle.make_params(cfg.W, cfg.H)
    for s in [0, 1, 31, 32, 63, 64, 100, 127, 128, 200, 254, 255]:
        lo, hi = oracle.learn(synth.learning_frames_host(cfg, s), synth.MARGIN)
        glo, ghi = fz.get_background(s)
        assert np.array_equal(glo.cpu().numpy(), lo) and np.array_equal(ghi.cpu().numpy(), hi), s
        frame = synth.frames_host(cfg, s, [k])[0]
        assert np.array_equal(fr[s].cpu().numpy(), frame), s
        rec, st = oracle.segment(p, frame, lo, hi, t_ms=int(t[s]))
        oracle.Tracker(p).update(rec)
        compare_record(res[s], rec, s, track=True)
        assert int(res[s]["stream"]) == s
        assert np.array_equal(masks[s].cpu().numpy(), st["final_mask"]), s
    fz.close()


# ------------------------------------------------------------ invariances
def test_batch_size_invariance_and_sharded_track():
    cfg = synth.CONFIGS[3]
    ks = list(range(0, 32))
    learn = synth.learning_frames_host(cfg)
    frames = _t(synth.frames_host(cfg, 0, ks))
    t = np.array([synth.t_ms(k) for k in ks], np.int64)
    a = _ctx(cfg.W, cfg.H, max_batch=32)
    a.learn_background(_t(learn))
    _, ra = a.process_frames(frames, t_ms=t)
    b = _ctx(cfg.W, cfg.H, max_batch=32)
    b.learn_background(_t(learn))
    parts = []
    for i in range(0, 32, 5):              # ragged batches of 5, stateless + track
        _, r = b.segment_frames(frames[i:i + 5], t_ms=t[i:i + 5])
        parts.append(r)
    rb = torch.cat(parts)
    b.track(rb)
    na, nb = results_numpy(ra), results_numpy(rb)
    for name in na.dtype.names:
        if name != "frame_idx":                # index within its call, by definition
            assert np.array_equal(na[name], nb[name]), name
    a.close()
    b.close()


def test_pipelined_graph_calls_match_oracle():
    """Pipelined mode (tails overlap the next call, double-buffered slots)
    and CUDA-graph replay vs direct launches: the same outputs, call after
    call, with the fold running across calls; sampled frames vs the oracle."""
    import os
    cfg = synth.CONFIGS[3]
    learn = synth.learning_frames_host(cfg)
    ks = list(range(40, 40 + 30))
    frames = _t(synth.frames_host(cfg, 0, ks))
    t = np.array([synth.t_ms(k) for k in ks], np.int64)
    calls = [(0, 7), (7, 14), (14, 21), (21, 24), (24, 30)]   # ragged: several graph shapes
    os.environ["FIZI_NO_GRAPH"] = "1"
    try:
        ref = _ctx(cfg.W, cfg.H, max_batch=8)                 # direct launches, joined tails
    finally:
        del os.environ["FIZI_NO_GRAPH"]
    ref.learn_background(_t(learn), margin=synth.MARGIN)
    pip = _ctx(cfg.W, cfg.H, max_batch=8)
    pip.learn_background(_t(learn), margin=synth.MARGIN)
    pip.set_pipeline(True)
    bufs = [(torch.empty((8, cfg.H, cfg.W), dtype=torch.uint8, device=DEV),
             torch.empty((8, 128), dtype=torch.uint8, device=DEV)) for _ in range(2)]
    out_ref, out_pip = [], []
    for j, (a, b) in enumerate(calls):
        mr, rr = ref.process_frames(frames[a:b], t_ms=t[a:b])
        out_ref.append((mr.cpu().numpy(), results_numpy(rr)))
        mk, rs = bufs[j & 1]
        pip.process_frames(frames[a:b], t_ms=t[a:b], masks=mk[: b - a], results=rs[: b - a])
        if j & 1:                      # both slots in flight, then collect them
            pip.flush()
            torch.cuda.synchronize()
            for jj in (j - 1, j):
                aa, bb = calls[jj]
                m2, r2 = bufs[jj & 1]
                out_pip.append((m2[: bb - aa].cpu().numpy(), results_numpy(r2[: bb - aa])))
    pip.flush()
    torch.cuda.synchronize()
    j = len(calls) - 1
    m2, r2 = bufs[j & 1]
    out_pip.append((m2[: calls[j][1] - calls[j][0]].cpu().numpy(),
                    results_numpy(r2[: calls[j][1] - calls[j][0]])))
    for (ma, ra), (mb, rb) in zip(out_ref, out_pip):
        assert np.array_equal(ma, mb)
        assert ra.tobytes() == rb.tobytes()
    # sampled frames of the pipelined run against the oracle (fold included)
    p = oracle.make_params(cfg.W, cfg.H)
    lo, hi = oracle.learn(learn, synth.MARGIN)
    tr = oracle.Tracker(p)
    fr_h = frames.cpu().numpy()
    flat = [(m, r) for (mm, rr) in out_pip for m, r in zip(mm, rr)]
    for i in range(len(ks)):
        rec, st = oracle.segment(p, fr_h[i], lo, hi, t_ms=int(t[i]), stages=i in (3, 22))
        tr.update(rec)
        compare_record(flat[i][1], rec, ks[i], track=True)
        if i in (3, 22):
            assert np.array_equal(flat[i][0], st["final_mask"])
    ref.close()
    pip.close()


def test_pipelined_multistream_and_segment_only():
    """Pipelined calls of interleaved streams (per-stream fold on the fold
    stream) and stateless segment_frames + track equal joined calls."""
    cfg = synth.CONFIGS[5]
    S = 4
    ref = _ctx(cfg.W, cfg.H, n_streams=S, max_batch=2 * S)
    pip = _ctx(cfg.W, cfg.H, n_streams=S, max_batch=2 * S)
    seg = _ctx(cfg.W, cfg.H, n_streams=S, max_batch=2 * S)
    for s_ in range(S):
        learn = _t(synth.learning_frames_host(cfg, s_))
        for fz in (ref, pip, seg):
            fz.learn_background(learn, stream=s_, margin=synth.MARGIN)
    pip.set_pipeline(True)
    seg.set_pipeline(True)
    out_ref, out_pip, out_seg = [], [], []
    bufs = [(torch.empty((2 * S, cfg.H, cfg.W), dtype=torch.uint8, device=DEV),
             torch.empty((2 * S, 128), dtype=torch.uint8, device=DEV)) for _ in range(3)]
    sbufs = [torch.empty((2 * S, 128), dtype=torch.uint8, device=DEV) for _ in range(3)]
    for step in range(5):
        ks = [2 * step, 2 * step + 1]
        frames, sof, t = [], [], []
        for k in ks:
            for s_ in range(S):
                frames.append(synth.frames_host(cfg, s_, [k])[0])
                sof.append(s_)
                t.append(synth.t_ms(k))
        fr = _t(np.stack(frames))
        mr, rr = ref.process_frames(fr, streams=sof, t_ms=t)
        out_ref.append((mr.cpu().numpy(), results_numpy(rr)))
        mk, rs = bufs[step % 3]
        pip.process_frames(fr, streams=sof, t_ms=t, masks=mk, results=rs)
        seg.segment_frames(fr, streams=sof, t_ms=t, masks=None, results=sbufs[step % 3])
        pip.flush()
        seg.flush()
        torch.cuda.synchronize()
        out_pip.append((mk.cpu().numpy(), results_numpy(rs)))
        r2 = sbufs[step % 3].clone()
        for s_ in range(S):                      # fold each stream's records in order
            idx = [i for i in range(len(sof)) if sof[i] == s_]
            sub = r2[idx].contiguous()
            seg.track(sub, stream=s_)
            r2[idx] = sub
        torch.cuda.synchronize()
        out_seg.append(results_numpy(r2))
    for (ma, ra), (mb, rb), rc in zip(out_ref, out_pip, out_seg):
        assert np.array_equal(ma, mb)
        assert ra.tobytes() == rb.tobytes()
        for name in ra.dtype.names:
            assert np.array_equal(ra[name], rc[name]), name
    for fz in (ref, pip, seg):
        fz.close()


@pytest.mark.parametrize("cid,n", [(1, None), (3, 12)])
def test_host_entry_matches_device_entry(cid, n):
    """fizi_process_frames_host (chunked H2D / path / D2H overlap; C3 frames
    give several ~32 MB chunks) equals the device entry point."""
    cfg = synth.CONFIGS[cid]
    learn = synth.learning_frames_host(cfg)
    n = n or cfg.n_proc
    frames = synth.frames_host(cfg, 0, range(n))
    t = np.array([synth.t_ms(k) for k in range(n)], np.int64)
    a = _ctx(cfg.W, cfg.H, max_batch=20)
    a.learn_background(_t(learn))
    ma, ra = a.process_frames(_t(frames), t_ms=t)
    b = _ctx(cfg.W, cfg.H, max_batch=20)
    b.learn_background(_t(learn))
    mh = np.empty((n, cfg.H, cfg.W), np.uint8)
    _, rh = b.process_frames_host(frames, t_ms=t, masks=mh)
    assert np.array_equal(ma.cpu().numpy(), mh)
    assert results_numpy(ra).tobytes() == rh.tobytes()
    a.close()
    b.close()


def test_device_generator_matches_host():
    synth.build_dev()
    for cid, ks in ((1, [0, 5]), (2, [151, 400]), (4, [3])):
        cfg = synth.CONFIGS[cid]
        h = synth.frames_host(cfg, 0, ks)
        d = synth.frames_dev(cfg, 0, ks).cpu().numpy()
        assert np.array_equal(h, d), cid


# ------------------------------------------------------------------ errors
def test_error_codes():
    from paper_1907_04393_b200 import fizi as F
    cfg = synth.CONFIGS[1]
    fz = _ctx(cfg.W, cfg.H, n_streams=2, max_batch=4)
    frames = _t(synth.frames_host(cfg, 0, range(2)))
    with pytest.raises(FiziError) as e:
        fz.process_frames(frames, t_ms=[0, 33])
    assert e.value.status == F.E_NOMODEL
    with pytest.raises(FiziError) as e:
        fz.learn_background(frames[:0])
    assert e.value.status == F.E_EMPTY
    fz.learn_background(_t(synth.learning_frames_host(cfg)))
    with pytest.raises(FiziError) as e:
        fz.process_frames(frames, t_ms=[33, 0])
    assert e.value.status == F.E_TIME
    fz.process_frames(frames, t_ms=[0, 33])
    with pytest.raises(FiziError) as e:
        fz.process_frames(frames, t_ms=[10, 20])          # earlier than the last call
    assert e.value.status == F.E_TIME
    with pytest.raises(FiziError) as e:
        fz.process_frames(_t(np.zeros((5, cfg.H, cfg.W, 3), np.uint8)))
    assert e.value.status == F.E_CAPACITY
    with pytest.raises(FiziError) as e:
        fz.process_frames(frames, streams=[5, 5], t_ms=[100, 200])
    assert e.value.status == F.E_CAPACITY
    small = _t(np.zeros((1, 10, 10, 3), np.uint8))
    with pytest.raises(FiziError) as e:
        fz.segment_frames(small)
    assert e.value.status == F.E_DIMS
    with pytest.raises(FiziError) as e:
        Fizi(320, 240, se_radius=0)
    assert e.value.status == F.E_ARG
    fz.close()


def test_binding_validates_output_buffers():
    """The binding checks every caller-supplied buffer before the C call
    (ADVICE r01): too small, wrong dtype, non-contiguous or host buffers raise
    instead of reaching the library."""
    cfg = synth.CONFIGS[1]
    fz = _ctx(cfg.W, cfg.H, max_batch=4)
    fz.learn_background(_t(synth.learning_frames_host(cfg)))
    frames = _t(synth.frames_host(cfg, 0, range(2)))
    t = np.array([0, 33], np.int64)
    ok_res = torch.empty((2, 128), dtype=torch.uint8, device=DEV)
    with pytest.raises(ValueError):
        fz.process_frames(frames, t_ms=t, results=torch.empty((1, 128), dtype=torch.uint8, device=DEV))
    with pytest.raises(ValueError):
        fz.process_frames(frames, t_ms=t, results=ok_res,
                          masks=torch.empty((1, cfg.H, cfg.W), dtype=torch.uint8, device=DEV))
    with pytest.raises(TypeError):
        fz.process_frames(frames, t_ms=t, results=ok_res,
                          masks=torch.empty((2, cfg.H, cfg.W), dtype=torch.float32, device=DEV))
    with pytest.raises(TypeError):
        fz.process_frames(frames, t_ms=t, results=torch.empty((2, 128), dtype=torch.uint8))
    with pytest.raises(ValueError):
        fz.process_frames(frames, t_ms=t, results=torch.empty((128, 4), dtype=torch.uint8,
                                                              device=DEV).t())
    with pytest.raises(ValueError):
        fz.track(torch.empty((2, 64), dtype=torch.uint8, device=DEV))
    with pytest.raises(TypeError):
        fz.process_frames_host(synth.frames_host(cfg, 0, range(2)), t_ms=t,
                               results=np.zeros(2, np.float64))
    m, r = fz.process_frames(frames, t_ms=t, results=ok_res)
    assert r.data_ptr() == ok_res.data_ptr()
    fz.close()
