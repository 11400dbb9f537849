"""World-size-2 gloo test of the sharded path's host logic.

Each rank segments its batches of a config-1/2-shaped stream with the oracle
(the per-frame, stateless part), the ranks all_gather the 128-byte records per
round, and every rank folds the gathered records in frame order.  The result
must equal a single-process run over all frames, on every rank.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import synth
from paper_1907_04393_b200 import shard
from paper_1907_04393_b200.fizi import RESULT_BYTES, RESULT_DTYPE


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _to_result_bytes(recs, ks):
    out = np.zeros(len(recs), RESULT_DTYPE)
    for i, (r, k) in enumerate(zip(recs, ks)):
        out[i]["t_ms"] = r.t_ms
        out[i]["frame_idx"] = k
        out[i]["blob_area"] = r.blob_area
        out[i]["cx"] = r.cx
        out[i]["cy"] = r.cy
    return out.view(np.uint8).reshape(len(recs), RESULT_BYTES)


def _fold(params, rows):
    tr = oracle.Tracker(params)
    out = []
    for row in rows:
        rec = oracle.record_from_blob(int(row["t_ms"]), int(row["blob_area"]), float(row["cx"]),
                                      float(row["cy"]))
        tr.update(rec)
        out.append((int(row["frame_idx"]), rec.visible, rec.clicked, rec.px, rec.py, rec.dwell_ms))
    return out


def _stream(cid, n_frames):
    cfg = synth.CONFIGS[cid]
    learn = synth.learning_frames_host(cfg)
    lo, hi = oracle.learn(learn, synth.MARGIN)
    frames = synth.frames_host(cfg, 0, range(n_frames))
    return cfg, lo, hi, frames


def _worker(rank, world, port, cid, n_frames, batch, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg, lo, hi, frames = _stream(cid, n_frames)
    p = oracle.make_params(cfg.W, cfg.H)
    folded = []
    gathered = torch.zeros(world * batch, RESULT_BYTES, dtype=torch.uint8)
    tr = oracle.Tracker(p)
    for rnd in range(shard.n_rounds(n_frames, batch, world)):
        b = shard.round_batch(n_frames, batch, world, rank, rnd)
        mine = torch.zeros(batch, RESULT_BYTES, dtype=torch.uint8)
        if b is not None:
            ks = list(range(b.k0, b.k1))
            recs = [oracle.segment(p, frames[k], lo, hi, t_ms=synth.t_ms(k), stages=False)[0]
                    for k in ks]
            mine[: b.n] = torch.from_numpy(_to_result_bytes(recs, ks))
        parts = list(gathered.chunk(world))
        dist.all_gather(parts, mine)
        gathered = torch.cat(parts)
        rows = gathered.numpy().view(RESULT_DTYPE).reshape(-1)
        for off, n in shard.gathered_slices(n_frames, batch, world, rnd):
            for row in rows[off: off + n]:
                rec = oracle.record_from_blob(int(row["t_ms"]), int(row["blob_area"]),
                                              float(row["cx"]), float(row["cy"]))
                tr.update(rec)
                folded.append((int(row["frame_idx"]), rec.visible, rec.clicked, rec.px, rec.py,
                               rec.dwell_ms))
    q.put((rank, folded))
    dist.destroy_process_group()


def _worker_windowed(rank, world, port, cid, n_frames, batch, window, q):
    """bench.py's sharded path: records of `window` steps gathered at once
    (one all_gather of window x batch records per rank), folded in frame order."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg, lo, hi, frames = _stream(cid, n_frames)
    p = oracle.make_params(cfg.W, cfg.H)
    tr = oracle.Tracker(p)
    folded = []
    resw = torch.zeros(window, batch, RESULT_BYTES, dtype=torch.uint8)
    rounds = []

    def drain():
        parts = [torch.zeros(window * batch, RESULT_BYTES, dtype=torch.uint8) for _ in range(world)]
        dist.all_gather(parts, resw.reshape(window * batch, RESULT_BYTES))
        rows = torch.cat(parts).numpy().view(RESULT_DTYPE).reshape(-1)
        for off, n in shard.window_slices(n_frames, batch, world, rounds, window):
            for row in rows[off: off + n]:
                rec = oracle.record_from_blob(int(row["t_ms"]), int(row["blob_area"]),
                                              float(row["cx"]), float(row["cy"]))
                tr.update(rec)
                folded.append((int(row["frame_idx"]), rec.visible, rec.clicked, rec.px, rec.py,
                               rec.dwell_ms))
        rounds.clear()

    for rnd in range(shard.n_rounds(n_frames, batch, world)):
        b = shard.round_batch(n_frames, batch, world, rank, rnd)
        if b is not None:
            ks = list(range(b.k0, b.k1))
            recs = [oracle.segment(p, frames[k], lo, hi, t_ms=synth.t_ms(k), stages=False)[0]
                    for k in ks]
            resw[len(rounds), : b.n] = torch.from_numpy(_to_result_bytes(recs, ks))
        rounds.append(rnd)
        if len(rounds) == window:
            drain()
    if rounds:
        drain()
    q.put((rank, folded))
    dist.destroy_process_group()


@pytest.mark.parametrize("window", [3])   # 4 rounds: a full and a partial window
def test_two_ranks_windowed_gather_matches_single_process(window):
    world, cid, n_frames, batch = 2, 1, 20, 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_windowed,
                         args=(r, world, port, cid, n_frames, batch, window, q))
             for r in range(world)]
    for pr in procs:
        pr.start()
    results = dict(q.get(timeout=600) for _ in range(world))
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    cfg, lo, hi, frames = _stream(cid, n_frames)
    p = oracle.make_params(cfg.W, cfg.H)
    recs = [oracle.segment(p, frames[k], lo, hi, t_ms=synth.t_ms(k), stages=False)[0]
            for k in range(n_frames)]
    ref = _fold(p, _to_result_bytes(recs, range(n_frames)).view(RESULT_DTYPE).reshape(-1))
    for r in range(world):
        assert results[r] == ref


def test_shard_assignment_covers_every_frame_once():
    for n_frames, batch, world in [(10000, 64, 1), (10000, 64, 2), (10000, 64, 8), (30, 4, 3),
                                   (7, 8, 2)]:
        seen = []
        for rnd in range(shard.n_rounds(n_frames, batch, world)):
            for r in range(world):
                b = shard.round_batch(n_frames, batch, world, r, rnd)
                if b:
                    seen.extend(range(b.k0, b.k1))
        assert seen == list(range(n_frames))


@pytest.mark.parametrize("cid,n_frames,batch", [(1, 20, 3), (2, 12, 4)])
def test_two_ranks_match_single_process(cid, n_frames, batch):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, cid, n_frames, batch, q))
             for r in range(world)]
    for pr in procs:
        pr.start()
    results = dict(q.get(timeout=600) for _ in range(world))
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    # reference: one process, all frames in order
    cfg, lo, hi, frames = _stream(cid, n_frames)
    p = oracle.make_params(cfg.W, cfg.H)
    recs = [oracle.segment(p, frames[k], lo, hi, t_ms=synth.t_ms(k), stages=False)[0]
            for k in range(n_frames)]
    ref = _fold(p, _to_result_bytes(recs, range(n_frames)).view(RESULT_DTYPE).reshape(-1))
    for r in range(world):
        assert results[r] == ref


# ------------------------------------------------ camera-stream sharding (C5)
def test_stream_shard_partition():
    for S, world in [(256, 1), (256, 2), (256, 8), (6, 4), (5, 2), (3, 8)]:
        owned = [shard.stream_shard(S, world, r) for r in range(world)]
        flat = sorted(s for o in owned for s in o)
        assert flat == list(range(S))
        assert all(s % world == r for r, o in enumerate(owned) for s in o)
        ids = shard.gathered_stream_ids(S, world)
        assert len(ids) == world * shard.streams_per_rank(S, world)
        order = shard.stream_order(S, world)
        assert [ids[i] for i in order] == list(range(S))


def _stream_worker(rank, world, port, n_streams, n_steps, q):
    """bench.py's sharded C5 path with the oracle in place of the GPU: rank r
    owns streams s mod world == r (their envelopes and trackers), processes
    the current frame of each per step, and the step's records are
    all-gathered into a global view."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg = synth.CONFIGS[5]
    p = oracle.make_params(cfg.W, cfg.H)
    mine = shard.stream_shard(n_streams, world, rank)
    per = shard.streams_per_rank(n_streams, world)
    envs = {s: oracle.learn(synth.learning_frames_host(cfg, s), synth.MARGIN) for s in mine}
    trackers = {s: oracle.Tracker(p) for s in mine}
    order = shard.stream_order(n_streams, world)
    views = []
    for k in range(n_steps):
        buf = torch.zeros(per, RESULT_BYTES, dtype=torch.uint8)
        rows = np.zeros(per, RESULT_DTYPE)
        for j, s in enumerate(mine):
            rec, _ = oracle.segment(p, synth.frames_host(cfg, s, [k])[0], *envs[s],
                                    t_ms=synth.t_ms(k), stages=False)
            trackers[s].update(rec)
            rows[j]["t_ms"] = rec.t_ms
            rows[j]["stream"] = s
            rows[j]["blob_area"] = rec.blob_area
            rows[j]["cx"], rows[j]["cy"] = rec.cx, rec.cy
            rows[j]["visible"], rows[j]["px"], rows[j]["py"] = rec.visible, rec.px, rec.py
        buf[:] = torch.from_numpy(rows.view(np.uint8).reshape(per, RESULT_BYTES))
        parts = [torch.zeros(per, RESULT_BYTES, dtype=torch.uint8) for _ in range(world)]
        dist.all_gather(parts, buf)
        g = torch.cat(parts).numpy().view(RESULT_DTYPE).reshape(-1)[order]
        views.append([(int(r["stream"]), int(r["t_ms"]), int(r["blob_area"]), float(r["px"]),
                       float(r["py"]), int(r["visible"])) for r in g])
    q.put((rank, views))
    dist.destroy_process_group()


def test_two_ranks_stream_sharding_matches_single_process():
    world, n_streams, n_steps = 2, 5, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_stream_worker, args=(r, world, port, n_streams, n_steps, q))
             for r in range(world)]
    for pr in procs:
        pr.start()
    results = dict(q.get(timeout=600) for _ in range(world))
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    # reference: one process, every stream with its own envelope and tracker
    cfg = synth.CONFIGS[5]
    p = oracle.make_params(cfg.W, cfg.H)
    ref = []
    trackers = [oracle.Tracker(p) for _ in range(n_streams)]
    envs = [oracle.learn(synth.learning_frames_host(cfg, s), synth.MARGIN) for s in range(n_streams)]
    for k in range(n_steps):
        step = []
        for s in range(n_streams):
            rec, _ = oracle.segment(p, synth.frames_host(cfg, s, [k])[0], *envs[s],
                                    t_ms=synth.t_ms(k), stages=False)
            trackers[s].update(rec)
            step.append((s, rec.t_ms, rec.blob_area, rec.px, rec.py, rec.visible))
        ref.append(step)
    for r in range(world):
        assert results[r] == ref
