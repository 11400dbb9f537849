#!/usr/bin/env python3
"""Benchmark of the FIZI + Mouse per-frame pixel path (arXiv 1907.04393) on B200.

Default workload (N=1): BASELINE.json configs[2] -- one 1920x1080 camera stream,
10,000 synthetic frames resident in HBM, batches of 64 frames per launch (the
config the metric is quoted on at 1/2/4/8 GPUs).  A step = one batch through the
whole hot path.  N = 1: fizi_process_frames (a2..a8: luma + three branches,
open-close, labelling, blob filter, hand blob, u8 mask write, Mouse fold).
N > 1: fizi_segment_frames (a2..a7) on the rank's batch, an NCCL all_gather
of the tiny per-frame records, then fizi_track (a8) over the gathered
records in frame order.  Rank r takes batch b
when b % N == r (weak scaling: 64 frames per rank per step).

--config 5 (BASELINE.json configs[4], 256 camera streams): stream s lives on
rank s mod N with its own envelope and tracker; a step is the current frame of
every stream (each rank: fizi_process_frames over its 256/N streams, then one
NCCL all_gather of the step's records for a global view; strong scaling).

Prints ONE JSON line (rank 0).  `--impl reference` times the CPU oracle instead
(the reference arm for this tier).
"""
from __future__ import annotations

import argparse
import gc
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "frames/s and Mpixel/s per GPU and at 2/4/8 B200; % of HBM roofline"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=628)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="fizi", choices=["fizi", "reference"])
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--batch", type=int, default=0, help="frames per launch (default: config's)")
    ap.add_argument("--e2e-steps", type=int, default=0, help="0 = same as --steps (capped)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--gather-every", type=int, default=0,
                    help="sharded path: steps per record gather + fold window "
                         "(0: max(1, 16 // N), so that the last window's fold stays short)")
    ap.add_argument("--force-gather", action="store_true",
                    help="N=1: run the sharded path (segment + NCCL gather + fold) on a one-rank group")
    ap.add_argument("--no-pipeline", action="store_true",
                    help="N=1: join every call's tail into the stream (no cross-call overlap)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-spot-check", action="store_true")
    ap.add_argument("--cpu-sample-frames", type=int, default=0)
    ap.add_argument("--diag-no-masks", action="store_true",
                    help="diagnostic only: do not request the u8 masks (masks_dev = NULL)")
    ap.add_argument("--diag-no-hand", action="store_true",
                    help="diagnostic only: frames without the hand (pure background path)")
    return ap.parse_args()


def ncu_alone(traffic_src):
    """The fused kernel timed alone by ncu (same capture as the traffic)."""
    if not traffic_src:
        return None
    with open(os.path.join(ROOT, traffic_src)) as f:
        d = json.load(f)
    if "ncu_duration_us" not in d:
        return None
    g = d["algorithmic_bytes_per_launch"] / d["ncu_duration_us"] / 1e3
    return {"achieved": g, "frac": g / peaks()[0], "duration_us": d["ncu_duration_us"],
            "source": traffic_src,
            "note": "one launch alone under ncu --set full (serialised, cold cache)"}


def ncu_traffic(seg_bytes, kernel):
    """DRAM bytes per launch of the fused kernel from the latest committed ncu
    --set full capture of that kernel on the same per-launch workload
    (profiles/r*_*_traffic.json)."""
    import glob
    best = None
    for path in sorted(glob.glob(os.path.join(ROOT, "profiles", "r*_traffic.json"))):
        with open(path) as f:
            d = json.load(f)
        if d.get("kernel", "seg_fast_kernel") != kernel:
            continue
        if abs(d.get("algorithmic_bytes_per_launch", 0) - seg_bytes) > 1:
            continue
        best = (d["dram_bytes_per_launch"], os.path.relpath(path, ROOT))
    return best if best else (None, None)


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            d = json.load(f)
        return float(d.get("hbm_gbs", 6650.0)), "measured"
    return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """NVML SM clock + throttle reasons, sampled in a thread; only the samples
    taken while `active` is set (the timed region) are kept.  The thread is
    started before the warm-up, so its start-up and NVML initialisation do not
    compete with the timed calls for the GIL or the host caches."""

    def __init__(self, index: int):
        self.samples, self.reasons, self.ok = [], set(), False
        self.max_mhz = None
        self.active = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            nv = pynvml
            self.names = {
                "hw_slowdown": getattr(nv, "nvmlClocksEventReasonHwSlowdown", 0x8),
                "hw_thermal_slowdown": getattr(nv, "nvmlClocksEventReasonHwThermalSlowdown", 0x40),
                "sw_thermal_slowdown": getattr(nv, "nvmlClocksEventReasonSwThermalSlowdown", 0x20),
                "sw_power_cap": getattr(nv, "nvmlClocksEventReasonSwPowerCap", 0x4),
                "hw_power_brake": getattr(nv, "nvmlClocksEventReasonHwPowerBrakeSlowdown", 0x80),
            }
            self.ok = True
        except Exception:
            self.ok = False
        self._stop = threading.Event()

    def _run(self):
        while not self._stop.is_set():
            if self.active:
                self.sample_now()
            time.sleep(0.002)

    def sample_now(self):
        """One sample (also called by the main thread right after the timed
        region's end event is recorded, while the GPU still runs its queued
        work: a short timed region may see no thread sample)."""
        if not self.ok or not self.active:
            return
        nv = self.nv
        try:
            mhz = nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)
            try:
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            except AttributeError:
                r = nv.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)
            self.samples.append(mhz)
            for k, bit in self.names.items():
                if r & bit:
                    self.reasons.add(k)
        except Exception:
            pass

    def start(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def stop(self):
        self.active = False
        if self.ok:
            self._stop.set()
            self.t.join()
            self.in_region = len(self.samples)
            if not self.samples:          # a timed region shorter than one sample period
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))

    def summary(self):
        if not self.ok:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml unavailable"]}
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples),
                "samples_in_timed_region": getattr(self, "in_region", len(self.samples))}


def workload_config(cfg, args, world):
    """The `config` object of the JSON line; the reference arm prints the same
    one (its per-step oracle sample is described in its `cpu_baseline`)."""
    from paper_1907_04393_b200 import shard
    sharded = world > 1 or args.force_gather
    pipelined = not args.no_pipeline
    S = cfg.streams
    N = cfg.W * cfg.H
    if S > 1:
        S_r = len(shard.stream_shard(S, world, 0))
        B = min(args.batch or S_r, S_r) if not sharded else S_r
        need = min(-(-S_r // B) * cfg.n_proc, args.warmup + args.steps)
        workload = (f"C{cfg.cid}: {S} streams of {cfg.W}x{cfg.H}, {cfg.n_proc} frames "
                    f"each, per-stream envelopes, stream s on rank s mod {world}; "
                    f"each call takes the current frame of {B} of the rank's "
                    f"{S_r} streams (BASELINE.json configs[{cfg.cid - 1}])")
    else:
        B = args.batch or cfg.batch
        need = min(shard.n_rounds(cfg.n_proc, B, world), args.warmup + args.steps)
        workload = (f"C{cfg.cid}: {cfg.W}x{cfg.H} stream, {cfg.n_proc} frames, "
                    f"batches of {B} per launch (BASELINE.json configs[{cfg.cid - 1}])")
    return {"workload": workload,
            "frames_per_step_per_gpu": B, "pipelined_calls": pipelined,
            "sharded_path": sharded, "resident_batches_per_gpu": need,
            "l2": (f"inputs larger than L2: {B * 3 * N / 1e6:.0f} MB of frames per step"
                   if B * 3 * N > 126e6 else
                   f"inputs larger than L2: {B * 3 * N / 1e6:.0f} MB of frames per step, "
                   f"cycled over {need} resident batches ({need * B * 3 * N / 1e9:.1f} GB)"),
            "parallelism": (f"frames sharded by batch, dp{world}" if S == 1 else
                            f"camera streams sharded (s mod {world}), dp{world}")}


# ------------------------------------------------------------- reference arm
def run_reference(args, cfg, rank, world):
    """CPU oracle as it stands, frame-parallel over the host cores."""
    if rank != 0:
        return
    import oracle
    import synth
    cores = os.cpu_count() or 1
    per_step = max(1, min(cores, 16))
    learn = synth.learning_frames_host(cfg)
    lo, hi = oracle.learn(learn, synth.MARGIN)
    p = oracle.make_params(cfg.W, cfg.H)
    pool = synth.frames_host(cfg, 0, range(per_step * 2))
    t = np.array([synth.t_ms(k) for k in range(per_step * 2)], np.int64)
    for i in range(args.warmup):
        sl = slice((i % 2) * per_step, (i % 2 + 1) * per_step)
        oracle.segment_batch(p, pool[sl], lo, hi, t_ms=t[sl], nthreads=cores)
    t0 = time.perf_counter()
    for i in range(args.steps):
        sl = slice((i % 2) * per_step, (i % 2 + 1) * per_step)
        recs, _ = oracle.segment_batch(p, pool[sl], lo, hi, t_ms=t[sl], nthreads=cores)
        tr = oracle.Tracker(p)
        for r in recs:
            tr.update(r)
    dt = time.perf_counter() - t0
    frames = per_step * args.steps
    v = frames / dt
    out = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "frames/s",
        "mpix_per_s": v * cfg.npx / 1e6, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": dt * 1e3 / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u8", "data": "synthetic",
        "config": workload_config(cfg, args, world),
        "cpu_baseline": {"value": v, "unit": "frames/s", "cores": cores, "kind": "oracle",
                         "cpu_model": cpu_model(),
                         "sample": f"each step: {per_step} frames of C{cfg.cid} "
                                   f"({cfg.W}x{cfg.H}) through the oracle (masks + records "
                                   f"+ fold), frame-parallel over {cores} host threads; "
                                   f"{args.steps} steps"},
        "e2e": {"value": v, "unit": "frames/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(out), flush=True)


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or "unknown"


def _oracle_pass(cfg, p, frames, envs, sids, nthreads, tracker):
    """One pass of the oracle over the sample: frames of one stream in one
    frame-parallel batch (+ the sequential fold), or one frame per stream
    (C5: per-stream envelopes) over a thread pool."""
    import oracle
    if envs is None:
        lo, hi = tracker[1]
        recs, _ = oracle.segment_batch(p, frames, lo, hi, nthreads=nthreads, want_masks=True)
        for r in recs:
            tracker[0].update(r)
        return
    from concurrent.futures import ThreadPoolExecutor

    def one(j):
        lo, hi = envs[j]
        recs, _ = oracle.segment_batch(p, frames[j:j + 1], lo, hi, nthreads=1, want_masks=True)
        return recs[0]
    with ThreadPoolExecutor(max_workers=nthreads) as ex:
        recs = list(ex.map(one, range(len(frames))))
    for j, r in enumerate(recs):
        tracker[2][sids[j]].update(r)


def cpu_baseline(cfg, n_frames=0, target_s=8.0, single_s=4.0):
    """The oracle as it stands on the host cores: frame-parallel
    over all cores (the reported value) and single-core, each a bounded sample
    of passes over the first frames of the workload (C5: the first frame of
    the first streams, each with its own envelope)."""
    import oracle
    import synth
    cores = os.cpu_count() or 1
    n = n_frames or max(8, min(64, 2 * cores))
    p = oracle.make_params(cfg.W, cfg.H)
    if cfg.streams == 1:
        lo, hi = oracle.learn(synth.learning_frames_host(cfg), synth.MARGIN)
        frames = synth.frames_host(cfg, 0, range(n))
        envs, sids = None, None
        what = f"the first {n} frames of C{cfg.cid} ({cfg.W}x{cfg.H})"
    else:
        n = min(n, cfg.streams)
        sids = list(range(n))
        envs = [oracle.learn(synth.learning_frames_host(cfg, s), synth.MARGIN) for s in sids]
        frames = __import__("numpy").stack([synth.frames_host(cfg, s, [0])[0] for s in sids])
        lo = hi = None
        what = (f"frame 0 of streams 0..{n - 1} of C{cfg.cid} ({cfg.W}x{cfg.H}, per-stream "
                f"envelopes)")

    def timed(nthreads, budget):
        tracker = (oracle.Tracker(p), (lo, hi), [oracle.Tracker(p) for _ in range(n)])
        passes, done, t0 = 0, 0, time.perf_counter()
        while True:
            _oracle_pass(cfg, p, frames, envs, sids, nthreads, tracker)
            passes += 1
            done += n
            dt = time.perf_counter() - t0
            if dt >= budget or passes >= 200:
                return done / dt, passes, done, dt

    v, passes, done, dt = timed(cores, target_s)
    v1, passes1, done1, dt1 = timed(1, single_s)
    return {"value": v, "unit": "frames/s", "cores": cores, "kind": "oracle",
            "cpu_model": cpu_model(),
            "sample": f"{passes} passes over {what} = {done} frames, frame-parallel oracle "
                      f"(masks + records + fold) over {cores} host threads, {dt:.1f} s",
            "single_core": {"value": v1, "unit": "frames/s", "cores": 1,
                            "sample": f"{passes1} passes = {done1} frames on one thread, {dt1:.1f} s"}}


def host_gaps(hts):
    """Host time per step call inside the timed region (diagnostics: the
    calls are asynchronous, so a long gap is the host waiting for a call slot
    or being descheduled)."""
    d = np.diff(np.asarray(hts)) * 1e6
    if d.size == 0:
        return None
    return {"median_us": float(np.median(d)), "max_us": float(d.max()),
            "first_us": [round(float(x), 1) for x in d[:3]],
            "over_1ms": int((d > 1000).sum()), "sum_over_1ms_ms": float(d[d > 1000].sum() / 1e3)}


def spot_check(cfg, frames_dev, masks_dev, res_dev, sids, idx):
    """Bench-side parity spot check of frames `idx` of the last timed call:
    the final mask and the stateless record fields (a2-a7) against the oracle
    (the fold state depends on every earlier frame, so it is not checked here)."""
    import oracle
    import synth
    from paper_1907_04393_b200 import results_numpy
    p = oracle.make_params(cfg.W, cfg.H)
    res = results_numpy(res_dev)
    checked = []
    for i in idx:
        s = int(sids[i]) if sids is not None else 0
        lo, hi = oracle.learn(synth.learning_frames_host(cfg, s), synth.MARGIN)
        rec, st = oracle.segment(p, frames_dev[i].cpu().numpy(), lo, hi)
        ok = bool(masks_dev is None or (masks_dev[i].cpu().numpy() == st["final_mask"]).all())
        for f in ("mean_luma", "corrected", "fg_merged", "fg_final", "n_comp_total", "n_comp_kept",
                  "blob_area", "blob_label", "sum_x", "sum_y"):
            ok = ok and int(res[i][f]) == int(getattr(rec, f))
        ok = ok and abs(float(res[i]["cx"]) - rec.cx) <= 1e-3 and abs(float(res[i]["cy"]) - rec.cy) <= 1e-3
        checked.append({"frame_in_call": int(i), "stream": s, "match": ok})
    return {"frames": checked, "all_match": all(c["match"] for c in checked)}


# ------------------------------------------------------------------ GPU arm
def main():
    args = parse()
    import synth
    cfg = synth.CONFIGS[args.config]
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, cfg, rank, world)
        return

    import torch
    import torch.distributed as dist
    from paper_1907_04393_b200 import RESULT_BYTES, Fizi

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    # sharded path (segment + gather + fold): N > 1, or N = 1 with --force-gather
    # (a one-rank NCCL group, to exercise the multi-GPU code path on one GPU)
    sharded = world > 1 or args.force_gather
    if sharded:
        if world == 1:
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", str(29500 + os.getpid() % 1000))
            dist.init_process_group("nccl", device_id=dev, rank=0, world_size=1)
        else:
            dist.init_process_group("nccl", device_id=dev)

    S = cfg.streams
    from paper_1907_04393_b200 import shard
    frames_by_round = []
    if S > 1:
        # C5: camera streams are sharded, stream s on rank s mod N with its
        # own envelope and tracker (local id = index in the rank's shard);
        # each call takes the current frame of B of the rank's streams
        # (default: all of them; 32 per call is 1.9x slower at N = 1,
        # scripts/gpu_c5_batch.sh), round r = frame k = r // G5 of group
        # g = r % G5 of the rank's streams
        sids_r = shard.stream_shard(S, world, rank)
        S_r = len(sids_r)
        B = min(args.batch or S_r, S_r) if not sharded else S_r
        G5 = -(-S_r // B)
        need = min(G5 * cfg.n_proc, args.warmup + args.steps)
        for rnd in range(need):
            g, k = rnd % G5, rnd // G5
            loc = list(range(g * B, min(S_r, (g + 1) * B)))
            fr = torch.empty((len(loc), cfg.H, cfg.W, 3), dtype=torch.uint8, device=dev)
            for j, l in enumerate(loc):
                synth.frames_dev(cfg, sids_r[l], [k], out=fr[j:j + 1], device=dev)
            frames_by_round.append((loc, fr, np.full(len(loc), synth.t_ms(k), np.int64)))
    else:
        S_r = 1
        B = args.batch or cfg.batch
        # round r: rank takes batch r*world + rank (weak scaling, B frames per
        # rank per step); the resident rounds are cycled if warmup + steps
        # exceeds them
        need = min(shard.n_rounds(cfg.n_proc, B, world), args.warmup + args.steps)
        for rnd in range(need):
            b = shard.round_batch(cfg.n_proc, B, world, rank, rnd)
            if b is None:
                frames_by_round.append(None)
                continue
            ks = list(range(b.k0, b.k1))
            t_base = np.asarray([synth.t_ms(k) for k in ks], np.int64)
            if args.diag_no_hand:
                pf = synth.frame_params(cfg, 0, ks)
                pf[:, 4] = 0
                fr = synth.gen_dev(cfg.W, cfg.H, cfg.seed, 0, pf, synth.clutter(cfg, 0), device=dev)
            else:
                fr = synth.frames_dev(cfg, 0, ks, device=dev)
            frames_by_round.append((ks, fr, t_base))
    fz = Fizi(cfg.W, cfg.H, n_streams=S_r, max_batch=B, device=local)
    for loc in range(S_r):
        sid = sids_r[loc] if S > 1 else 0
        learn = synth.frames_dev(cfg, sid, range(cfg.n_learn), learning=True, device=dev)
        fz.learn_background(learn, stream=loc, margin=synth.MARGIN)
    # N = 1: pipelined calls (a call's tail overlaps the next calls'
    # segmentation), so outputs rotate over CALL_SLOTS buffers and the timed
    # region ends with fz.flush() (N > 1: segment_frames, windowed gather + fold)
    pipelined = not args.no_pipeline
    fz.set_pipeline(pipelined)
    # sharded path: the records of G steps are gathered and folded together on
    # a fold stream (one NCCL all_gather per window), while the next window's
    # calls run; the folds of every rank cover every frame, in frame order
    # one window's fold costs ~0.15 us per record in one thread (every rank
    # folds every rank's records): N x 64 x G records per window, so the
    # window shrinks with N to keep the fold of the last window (the only one
    # not hidden behind later calls) short
    G = (max(1, args.gather_every) if args.gather_every else max(1, 16 // world)) if sharded else 1
    Bg = shard.streams_per_rank(S, world) if S > 1 else B   # rows per rank and step in the gather
    # windows rotate over NWIN record buffers: a window's calls wait only for
    # the gather of the window NWIN back (not for the previous window's tails)
    NWIN = 4
    resw_ring = [torch.zeros((G, Bg, RESULT_BYTES), dtype=torch.uint8, device=dev)
                 for _ in range(NWIN)]
    ev_ring = [None] * NWIN
    win_no = [0]
    gathered_w = torch.empty((world * G * Bg, RESULT_BYTES), dtype=torch.uint8, device=dev)
    fold_stream = torch.cuda.Stream(device=dev)
    window = []
    NBUF = fz.call_slots                 # = the context's call slots (include/fizi.h)
    masks2 = [torch.empty((B, cfg.H, cfg.W), dtype=torch.uint8, device=dev) for _ in range(NBUF)]
    res2 = [torch.empty((B, RESULT_BYTES), dtype=torch.uint8, device=dev) for _ in range(NBUF)]
    del learn
    # per-round views, made once (the step itself only enqueues work)
    views = []
    for item in frames_by_round:
        if item is None:
            views.append(None)
            continue
        ks, fr, t_base = item
        n = len(ks)
        views.append((n, fr[:n], [None if args.diag_no_masks else m[:n] for m in masks2],
                      [r[:n] for r in res2], t_base, np.asarray(ks, np.uint32) if S > 1 else None))
    t_pass = synth.t_ms(cfg.n_proc)

    def step(i):
        rnd = i % need
        v = views[rnd]
        n = 0
        if v is not None:
            n, fr_n, mks, ress, t_base, sids = v
            mk, res_n = mks[i % NBUF], ress[i % NBUF]
            # timestamps keep increasing across passes over the resident rounds
            t = t_base + (i // need) * t_pass
            if not sharded:            # the whole path in one call (fold fused into labelling)
                fz.process_frames(fr_n, streams=sids, t_ms=t, masks=mk, results=res_n)
                return n
            if S > 1:                  # streams are rank-local: the whole path, folds included
                fz.process_frames(fr_n, streams=sids, t_ms=t, masks=mk, results=cur_resw()[len(window)][:n])
            else:                      # one stream across ranks: stateless part, fold after the gather
                fz.segment_frames(fr_n, t_ms=t, masks=mk, results=cur_resw()[len(window)][:n])
        window.append(rnd)
        if len(window) == G:
            drain()
        return n

    def cur_resw():
        w = win_no[0] % NWIN
        if not window and ev_ring[w] is not None:
            torch.cuda.current_stream(dev).wait_event(ev_ring[w])   # its previous gather is done
            ev_ring[w] = None
        return resw_ring[w]

    def drain():
        # a8 across ranks: gather the window's records (frame order = step
        # order, then rank order) and fold them on every rank
        if not window:
            return
        main = torch.cuda.current_stream(dev)
        fold_stream.wait_stream(main)
        with torch.cuda.stream(fold_stream):
            fz.flush()                      # the window's tails, joined into the fold stream
            dist.all_gather_into_tensor(gathered_w, resw_ring[win_no[0] % NWIN])
            gathered_ev = torch.cuda.Event()
            gathered_ev.record(fold_stream)
            ev_ring[win_no[0] % NWIN] = gathered_ev
            if S == 1:                      # (C5: records already folded per stream, on their rank)
                # the window's records in frame order: runs of rows of
                # the rank blocks (step-major, then rank)
                runs = []
                for o, cnt in shard.window_slices(cfg.n_proc, B, world, window, G):
                    if runs and runs[-1][0] + runs[-1][1] == o:
                        runs[-1][1] += cnt
                    else:
                        runs.append([o, cnt])
                for i in range(0, len(runs), 256):  # the window's folds in one launch
                    fz.track_runs(gathered_w, runs[i:i + 256])
        win_no[0] += 1
        window.clear()

    def finish():
        # the last (partial) window, its folds, and every outstanding tail
        drain()
        torch.cuda.current_stream(dev).wait_stream(fold_stream)
        fz.flush()

    # a round of another size (the last, partial batch) is run once before the
    # warm-up, with earlier timestamps, so that its call shape is captured
    # outside the timed region (the library captures a new shape for all slots)
    if not sharded:
        common = views[0][0] if views and views[0] else None
        for v in views:
            if v is not None and v[0] != common:
                n_v, fr_v, mks_v, ress_v, tb_v, sids_v = v
                fz.process_frames(fr_v, streams=sids_v, t_ms=tb_v - 10**12, masks=mks_v[0],
                                  results=ress_v[0])
                fz.flush()
                break
    # no cyclic-GC pause inside the timed region (a full collection over the
    # interpreter's objects takes milliseconds; the step loop allocates little).
    # The collection runs before the warm-up: right before the timed region it
    # leaves the host caches cold, and the first timed call then takes ~190 us
    # of host time instead of ~35 (scripts/first_call.py)
    clk = ClockSampler(torch.cuda.current_device()).start()
    gc.collect()
    gc.disable()
    for i in range(args.warmup):
        step(i)
    finish()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    # the timed region replays the captured launch sequence (no profiling events)
    fz.profile_enable(0)
    st = torch.cuda.current_stream(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches0 = fz.kernel_launches()
    frames_done = 0
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk.active = True
    e0.record(st)
    h0 = time.perf_counter()
    hts = [time.perf_counter()]
    for i in range(args.steps):
        frames_done += step(args.warmup + i)
        hts.append(time.perf_counter())
    finish()                         # every tail (and fold) of the timed calls is inside
    host_ms = (time.perf_counter() - h0) * 1e3
    e1.record(st)
    gpu_busy = not e1.query()            # the GPU is still inside the timed region
    if gpu_busy:
        clk.sample_now()
    torch.cuda.synchronize()
    clk.stop()
    gc.enable()
    if world > 1:
        dist.barrier()
    launches = fz.kernel_launches() - launches0
    ms = e0.elapsed_time(e1)
    spot = None
    if rank == 0 and not sharded and not args.no_spot_check:
        # the last timed call's outputs, checked against the oracle (untimed)
        i_last = args.warmup + args.steps - 1
        v = views[i_last % need]
        if v is not None:
            n_l, fr_l, mks_l, ress_l, _, sids_l = v
            mk_l = mks_l[i_last % NBUF]
            spot = spot_check(cfg, fr_l, mk_l, ress_l[i_last % NBUF],
                              sids_l if S > 1 else None, sorted({0, n_l - 1}))
    # the fused kernel's launch duration: a second pass of the same K steps
    # with CUDA events around that kernel on its launching stream (direct
    # launches: events cannot be accumulated across graph replays)
    fz.profile_enable(2)
    fz.profile_read(reset=True)
    for i in range(args.steps):
        step(args.warmup + args.steps + i)
    finish()
    torch.cuda.synchronize()
    prof = fz.profile_read(reset=True)
    # per-stage breakdown: a separate, untimed pass with events around every
    # stage, calls joined (not pipelined) so that each stage's events bracket
    # that stage's own kernels
    fz.set_pipeline(False)
    fz.profile_enable(1)
    nb = min(args.steps, 50)
    for i in range(nb):
        step(args.warmup + 2 * args.steps + i)
    finish()
    torch.cuda.synchronize()
    breakdown = fz.profile_read(reset=True)
    fz.profile_enable(False)
    fz.set_pipeline(pipelined)
    tmax = torch.tensor([ms], dtype=torch.float64, device=dev)
    tot = torch.tensor([frames_done], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
        dist.all_reduce(tot, op=dist.ReduceOp.SUM)
    ms_max = float(tmax.item())
    total_frames = float(tot.item())
    value = total_frames / (ms_max / 1e3)

    # ---------------------------------------------------------- roofline
    N = cfg.npx
    hbm, peak_kind = peaks()
    seg_ms, seg_n = prof["segment"]
    # algorithmic bytes the fused segmentation kernel moves per step: B frames
    # read (3N each), the stream's envelope once (6N), B bit masks written
    # (N/8 each); a step may issue several launches (sub-batches), so the
    # achieved rate is total algorithmic bytes / total kernel time
    seg_bytes = B * (3 * N + N / 8) + 6 * N * min(S, B)   # C5: one envelope per frame
    launches_per_step = seg_n / max(args.steps, 1)
    seg_gbs = seg_bytes * args.steps / (seg_ms / 1e3) / 1e9 if seg_n else None
    step_bytes = B * (3 * N + N) + 6 * N * min(S, B)   # whole-path algorithmic bytes per step
    step_ms = ms_max / args.steps
    kname = "seg_multi_kernel" if (S > 1 and B > 1) else "seg_fast_kernel"
    traffic, traffic_src = ncu_traffic(seg_bytes, kname) if launches_per_step == 1 else (None, None)
    roofline = {
        "bound": "hbm", "kernel": f"{kname} (fused luma + R1/R2/R3, a2+a3)",
        "achieved": seg_gbs, "peak": hbm, "unit": "GB/s",
        "frac": (seg_gbs / hbm) if seg_gbs else None, "traffic": traffic,
        "traffic_source": traffic_src,
        "alone": ncu_alone(traffic_src),
        "peak_kind": peak_kind,
        "algorithmic_bytes_per_step": seg_bytes,
        "launches_per_step": launches_per_step,
        "kernel_ms_per_step": seg_ms / max(args.steps, 1),
        "kernel_timing": "CUDA events around every fused-kernel launch on its stream, "
                         "second pass of the same K steps with direct launches",
        "graph_replay": {"timed_region": True, "kernel_timing_pass": False},
        "step": {"achieved": step_bytes / (step_ms / 1e3) / 1e9,
                 "frac": step_bytes / (step_ms / 1e3) / 1e9 / hbm,
                 "algorithmic_bytes_per_step": step_bytes},
        "stage_ms_per_step": {k: (v[0] / max(nb, 1)) for k, v in breakdown.items()},
        "stage_breakdown": "separate pass, calls joined (not pipelined), events around each stage",
        "stage_share": {k: v[0] / max(sum(x[0] for x in breakdown.values()), 1e-9)
                        for k, v in breakdown.items()},
    }

    out = {
        "metric": METRIC, "value": value, "unit": "frames/s",
        "mpix_per_s": value * N / 1e6, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_max / args.steps,
        "host_enqueue_ms_per_step": host_ms / args.steps, "higher_is_better": True,
        "scaling": "weak" if S == 1 else "strong", "vs_baseline": None, "dtype": "u8",
        "data": "synthetic",
        "config": workload_config(cfg, args, world),
        "gpu_launches": launches,
        "gather_window_steps": G if sharded else None,
        "host_step_gaps": host_gaps(hts),
        "spot_check": spot,
        "roofline": roofline,
        "clocks": clk.summary(),
    }

    # --------------------------------------------------------------- e2e
    if not args.no_e2e:
        # end to end through fizi_process_frames_host: the step's frames copied
        # in from pinned host memory, masks and records copied out, per call
        k2 = args.e2e_steps or min(args.steps, 40)
        fe = Fizi(cfg.W, cfg.H, n_streams=S_r, max_batch=B, device=local)
        for loc in range(S_r):
            sid = sids_r[loc] if S > 1 else 0
            learn = synth.frames_dev(cfg, sid, range(cfg.n_learn), learning=True, device=dev)
            fe.learn_background(learn, stream=loc, margin=synth.MARGIN)
        del learn
        hosts = []
        for item in [x for x in frames_by_round if x is not None][:2]:
            ks, fr, _ = item
            h = torch.empty((len(ks), cfg.H, cfg.W, 3), dtype=torch.uint8).pin_memory()
            h.copy_(fr[: len(ks)])
            hosts.append((ks, h.numpy()))
        mask_h = torch.empty((B, cfg.H, cfg.W), dtype=torch.uint8).pin_memory().numpy()
        from paper_1907_04393_b200 import RESULT_DTYPE
        res_h = np.zeros(B, RESULT_DTYPE)
        t_base = 0

        def estep(i):
            ks, h = hosts[i % len(hosts)]
            if S > 1:               # (ks = local stream ids; one frame of each, one time step)
                t = np.full(len(ks), synth.t_ms(i), np.int64)
                fe.process_frames_host(h, streams=np.asarray(ks, np.uint32), t_ms=t,
                                       masks=mask_h[: len(ks)], results=res_h[: len(ks)])
                return len(ks)
            t = np.asarray([synth.t_ms(k) for k in ks], np.int64) + i * synth.t_ms(cfg.n_proc)
            fe.process_frames_host(h, t_ms=t, masks=mask_h[: len(ks)], results=res_h[: len(ks)])
            return len(ks)

        for i in range(3):
            estep(i)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        nfr = 0
        for i in range(k2):
            nfr += estep(3 + i)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        tt = torch.tensor([dt], dtype=torch.float64, device=dev)
        nn = torch.tensor([nfr], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            dist.all_reduce(nn, op=dist.ReduceOp.SUM)
        out["e2e"] = {"value": float(nn.item()) / float(tt.item()), "unit": "frames/s",
                      "h2d_bytes_per_step": B * 3 * N, "d2h_bytes_per_step": B * (N + RESULT_BYTES),
                      "steps": k2, "api": "fizi_process_frames_host (pinned host buffers)"}
        fe.close()

    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline(cfg, args.cpu_sample_frames)
    if rank == 0:
        print(json.dumps(out), flush=True)
    fz.close()
    if sharded:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
