"""Seeded synthetic workloads for the FIZI + Mouse path (input generators only).

This module holds none of the method's arithmetic.  It defines the five
BASELINE.json configurations, computes per-frame geometry / exposure gains on
the host (double, round-half-up) and materialises frames either on the host
(``synth_host.c`` via ctypes) or directly in HBM (``synth_dev.cu``), the two
being byte-identical (tests/test_synth.py).  Both the oracle-side tests and
the CUDA-side tests / bench draw their inputs from here.
"""
from __future__ import annotations

import ctypes
import math
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_HOST_SRC = os.path.join(_HERE, "synth_host.c")
_HOST_LIB = os.path.join(_HERE, "libsynth_host.so")
_DEV_SRC = os.path.join(_HERE, "synth_dev.cu")
_DEV_LIB = os.path.join(_HERE, "libsynth_dev.so")

T_STEP_MS = 33          # S:548 frame spacing
NOISE_A = 4             # sensor noise amplitude (<= margin/2)
MARGIN = 10             # envelope margin
PF_STRIDE = 8


@dataclass(frozen=True)
class Config:
    cid: int
    W: int
    H: int
    n_learn: int
    n_proc: int
    R: int
    orbit_step: float
    streams: int = 1
    batch: int = 64
    drift: bool = False
    n_clutter: int = 0
    arm: bool = False
    events: bool = True          # dwell pauses + absent windows (tracker coverage)

    @property
    def seed(self) -> int:
        return 0x5EED0000 + self.cid

    @property
    def npx(self) -> int:
        return self.W * self.H


CONFIGS = {
    1: Config(1, 320, 240, 10, 20, 30, 2 * math.pi / 20, batch=20, events=False),
    2: Config(2, 640, 480, 30, 1000, 60, 2 * math.pi / 90, drift=True, batch=64),
    3: Config(3, 1920, 1080, 30, 10000, 135, 2 * math.pi / 90, batch=64),
    4: Config(4, 3840, 2160, 30, 4000, 648, 2 * math.pi / 90, batch=64, n_clutter=64, arm=True),
    5: Config(5, 640, 480, 30, 300, 60, 2 * math.pi / 90, streams=256, batch=32),
}


def round_half_up(v: float) -> int:
    return int(math.floor(v + 0.5))


def t_ms(k: int) -> int:
    """Timestamp of processed frame k (33 ms spacing)."""
    return T_STEP_MS * k


def _gain_q10(cfg: Config, k: int) -> int:
    if not cfg.drift:
        return 1024
    g = 1.0 + 0.6 * math.sin(2 * math.pi * k / 400.0)
    # three abrupt exposure steps ("brutal changes")
    if any(s <= k < s + 30 for s in (150, 500, 800)):
        g *= 0.6
    # an over-exposure ramp near the drift's peak ("over-exposed
    # environment"): x1.0 .. x1.5 over frames 40-139, so the mean luma climbs
    # through the unclamped gamma > 1 rows (191-193) into the clamped ones
    if 40 <= k < 140:
        g *= 1.0 + 0.5 * (k - 40) / 100.0
    return round_half_up(1024.0 * g)


def _hand_state(cfg: Config, k: int):
    """(present, motion counter) for processed frame k."""
    if not cfg.events:
        return True, k
    m = 0
    present = True
    # motion counter: angle holds during pauses (k % 300 in [100,140)) -> dwell click
    full, rem = divmod(k, 300)
    m = full * (300 - 40) + min(rem, 100) + max(0, rem - 140)
    if 200 <= rem < 225:
        present = False
    return present, m


def frame_params(cfg: Config, stream: int, ks, learning: bool = False) -> np.ndarray:
    """int32 (n, 8) per-frame blocks: id, gain_q10, cx, cy, R, arm_w, 0, 0."""
    ks = list(ks)
    out = np.zeros((len(ks), PF_STRIDE), np.int32)
    rho = 0.25 * cfg.H
    theta0 = 2 * math.pi * stream / max(cfg.streams, 1)
    for i, k in enumerate(ks):
        if learning:
            out[i, 0] = k
            out[i, 1] = 1024
            continue
        out[i, 0] = cfg.n_learn + k
        out[i, 1] = _gain_q10(cfg, k)
        present, m = _hand_state(cfg, k)
        th = theta0 + cfg.orbit_step * m
        out[i, 2] = round_half_up(cfg.W / 2 + rho * math.cos(th))
        out[i, 3] = round_half_up(cfg.H / 2 + rho * math.sin(th))
        out[i, 4] = cfg.R if present else 0
        out[i, 5] = round_half_up(0.6 * cfg.R) if (cfg.arm and present) else 0
    return out


def clutter(cfg: Config, stream: int) -> np.ndarray:
    """Static skin-hued ellipses baked into the background (C4)."""
    if cfg.n_clutter == 0:
        return np.zeros((0, 4), np.int32)
    rng = np.random.default_rng(cfg.seed * 1000 + stream)
    e = np.zeros((cfg.n_clutter, 4), np.int32)
    e[:, 0] = rng.integers(0, cfg.W, cfg.n_clutter)
    e[:, 1] = rng.integers(0, cfg.H, cfg.n_clutter)
    e[:, 2] = rng.integers(20, 121, cfg.n_clutter)
    e[:, 3] = rng.integers(20, 121, cfg.n_clutter)
    return e


# ------------------------------------------------------------- host generator
_host = None


def _host_lib():
    global _host
    if _host is None:
        if not os.path.exists(_HOST_LIB) or os.path.getmtime(_HOST_LIB) < os.path.getmtime(_HOST_SRC):
            subprocess.check_call(["gcc", "-std=c99", "-O2", "-fPIC", "-shared", "-o",
                                   _HOST_LIB, _HOST_SRC])
        _host = ctypes.CDLL(_HOST_LIB)
        _host.synth_frames.argtypes = [
            ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint32,
            ctypes.c_uint32, ctypes.c_void_p, ctypes.c_uint32, ctypes.c_void_p, ctypes.c_void_p]
    return _host


def gen_host(W: int, H: int, seed: int, stream: int, pf: np.ndarray, ell: np.ndarray,
             noise_a: int = NOISE_A) -> np.ndarray:
    pf = np.ascontiguousarray(pf, np.int32)
    ell = np.ascontiguousarray(ell, np.int32).reshape(-1, 4)
    n = pf.shape[0]
    out = np.empty((n, H, W, 3), np.uint8)
    _host_lib().synth_frames(W, H, seed, stream, noise_a, n, pf.ctypes.data, ell.shape[0],
                             ell.ctypes.data if ell.size else None, out.ctypes.data)
    return out


def learning_frames_host(cfg: Config, stream: int = 0) -> np.ndarray:
    pf = frame_params(cfg, stream, range(cfg.n_learn), learning=True)
    return gen_host(cfg.W, cfg.H, cfg.seed, stream, pf, clutter(cfg, stream))


def frames_host(cfg: Config, stream: int, ks) -> np.ndarray:
    pf = frame_params(cfg, stream, ks)
    return gen_host(cfg.W, cfg.H, cfg.seed, stream, pf, clutter(cfg, stream))


# ----------------------------------------------------------- device generator
def build_dev(nvcc: str = "nvcc", force: bool = False) -> str:
    if force or not os.path.exists(_DEV_LIB) or os.path.getmtime(_DEV_LIB) < os.path.getmtime(_DEV_SRC):
        subprocess.check_call([nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-O3",
                               "-lineinfo", "-Xcompiler", "-fPIC", "-shared", "-o", _DEV_LIB,
                               _DEV_SRC])
    return _DEV_LIB


_dev = None


def _dev_lib():
    global _dev
    if _dev is None:
        if not os.path.exists(_DEV_LIB):
            raise RuntimeError(f"{_DEV_LIB} missing: run __graft_entry__.build()")
        _dev = ctypes.CDLL(_DEV_LIB)
        _dev.synth_frames_dev.argtypes = [
            ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint32,
            ctypes.c_uint32, ctypes.c_void_p, ctypes.c_uint32, ctypes.c_void_p, ctypes.c_void_p,
            ctypes.c_void_p, ctypes.c_void_p]
        _dev.synth_frames_dev.restype = ctypes.c_int
    return _dev


def gen_dev(W: int, H: int, seed: int, stream: int, pf: np.ndarray, ell: np.ndarray,
            out=None, device="cuda", noise_a: int = NOISE_A):
    """Materialise frames in HBM; returns a torch uint8 tensor (n, H, W, 3)."""
    import torch
    pf_t = torch.as_tensor(np.ascontiguousarray(pf, np.int32), device=device)
    ell_t = torch.as_tensor(np.ascontiguousarray(ell, np.int32).reshape(-1, 4), device=device)
    n = pf_t.shape[0]
    if out is None:
        out = torch.empty((n, H, W, 3), dtype=torch.uint8, device=device)
    plate = torch.empty((H, W, 3), dtype=torch.uint8, device=device)
    st = torch.cuda.current_stream(out.device).cuda_stream
    rc = _dev_lib().synth_frames_dev(W, H, seed, stream, noise_a, n, pf_t.data_ptr(),
                                     ell_t.shape[0], ell_t.data_ptr() if ell_t.numel() else None,
                                     plate.data_ptr(), out.data_ptr(), st)
    if rc != 0:
        raise RuntimeError(f"synth_frames_dev failed: {rc}")
    torch.cuda.current_stream(out.device).synchronize()
    return out


def frames_dev(cfg: Config, stream: int, ks, learning: bool = False, out=None, device="cuda"):
    pf = frame_params(cfg, stream, ks, learning=learning)
    return gen_dev(cfg.W, cfg.H, cfg.seed, stream, pf, clutter(cfg, stream), out=out,
                   device=device)
