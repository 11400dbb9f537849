"""TEST INFRASTRUCTURE ONLY -- the CPU oracle for the FIZI + Mouse pixel path.

ctypes wrapper over ``oracle/liboracle.so`` (built from ``fizi_oracle.c`` with
plain gcc ``-O2 -ffp-contract=off``).  Only ``tests/``, ``__graft_entry__.smoke()``
and ``bench.py``'s cpu_baseline / ``--impl reference`` legs may import this
package.  The product package ``paper_1907_04393_b200`` never imports it and
shares no code with it.

Every function cites the PAPER.md / SPEC.md passage it follows in the C source;
the pins that check it against the paper and mathematics live in
``tests/test_oracle_*.py``.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "fizi_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

_u8p = ctypes.POINTER(ctypes.c_uint8)
_u32p = ctypes.POINTER(ctypes.c_uint32)


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (no SIMD intrinsics, no FMA contraction)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call([
            "gcc", "-std=c99", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fPIC",
            "-shared", "-o", _LIB, _SRC, "-lm", "-lpthread"])
    return _LIB


class Params(ctypes.Structure):
    """The oracle's own parameter struct (defaults: S:187)."""
    _fields_ = [
        ("width", ctypes.c_uint32), ("height", ctypes.c_uint32),
        ("gray_tol_S", ctypes.c_uint32),
        ("hue_lo_deg", ctypes.c_uint32), ("hue_hi_deg", ctypes.c_uint32),
        ("se_radius", ctypes.c_uint32), ("min_blob_ppm", ctypes.c_uint32),
        ("luma_target", ctypes.c_uint32), ("luma_lo", ctypes.c_uint32),
        ("luma_hi", ctypes.c_uint32),
        ("gamma_min", ctypes.c_double), ("gamma_max", ctypes.c_double),
        ("beta", ctypes.c_double), ("dwell_radius_px", ctypes.c_double),
        ("dwell_time_ms", ctypes.c_int64), ("lost_timeout_ms", ctypes.c_int64),
    ]


DEFAULTS = dict(gray_tol_S=30, hue_lo_deg=340, hue_hi_deg=25, se_radius=1,
                min_blob_ppm=5000, luma_target=128, luma_lo=60, luma_hi=190,
                gamma_min=0.4, gamma_max=2.5, beta=0.5, dwell_radius_px=15.0,
                dwell_time_ms=800, lost_timeout_ms=500)


def make_params(width: int, height: int, **kw) -> Params:
    d = dict(DEFAULTS)
    d.update(kw)
    return Params(width=width, height=height, **d)


class Record(ctypes.Structure):
    _fields_ = [
        ("t_ms", ctypes.c_int64), ("sum_luma", ctypes.c_uint64),
        ("mean_luma", ctypes.c_uint32), ("corrected", ctypes.c_uint32),
        ("gamma", ctypes.c_double),
        ("fg_merged", ctypes.c_uint32), ("fg_final", ctypes.c_uint32),
        ("n_comp_total", ctypes.c_uint32), ("n_comp_kept", ctypes.c_uint32),
        ("blob_area", ctypes.c_uint32), ("blob_label", ctypes.c_uint32),
        ("bbox", ctypes.c_uint32 * 4),
        ("sum_x", ctypes.c_uint64), ("sum_y", ctypes.c_uint64),
        ("cx", ctypes.c_double), ("cy", ctypes.c_double),
        ("visible", ctypes.c_uint32), ("clicked", ctypes.c_uint32),
        ("px", ctypes.c_double), ("py", ctypes.c_double),
        ("dwell_ms", ctypes.c_int64),
    ]

    def as_dict(self) -> dict:
        out = {}
        for name, _ in self._fields_:
            v = getattr(self, name)
            out[name] = list(v) if name == "bbox" else v
        return out


class TState(ctypes.Structure):
    _fields_ = [
        ("vis", ctypes.c_int), ("px", ctypes.c_double), ("py", ctypes.c_double),
        ("last_t", ctypes.c_int64), ("ax", ctypes.c_double), ("ay", ctypes.c_double),
        ("anchor_t", ctypes.c_int64), ("dwell", ctypes.c_int64), ("fired", ctypes.c_int),
    ]


class Stages(ctypes.Structure):
    _fields_ = [("r1", _u8p), ("r2", _u8p), ("r3", _u8p), ("merged", _u8p),
                ("oc", _u8p), ("labels", _u32p), ("final_mask", _u8p), ("contour", _u8p)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        L = _lib
        L.or_learn.argtypes = [_u8p, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32,
                               ctypes.c_uint32, _u8p, _u8p]
        L.or_mean_luma.argtypes = [_u8p, ctypes.c_uint32, ctypes.c_uint32,
                                   ctypes.POINTER(ctypes.c_uint64)]
        L.or_mean_luma.restype = ctypes.c_uint32
        L.or_gamma.argtypes = [ctypes.POINTER(Params), ctypes.c_uint32, _u32p]
        L.or_gamma.restype = ctypes.c_double
        L.or_lut.argtypes = [ctypes.c_double, _u8p]
        L.or_hue_num.argtypes = [_u8p, ctypes.POINTER(ctypes.c_int64)]
        L.or_hue_num.restype = ctypes.c_int
        L.or_in_band.argtypes = [ctypes.c_int64, ctypes.c_int, ctypes.c_uint32, ctypes.c_uint32]
        L.or_in_band.restype = ctypes.c_int
        for fn in (L.or_erode, L.or_dilate, L.or_open_close):
            fn.argtypes = [_u8p, _u8p, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32]
        L.or_label.argtypes = [_u8p, ctypes.c_uint32, ctypes.c_uint32, _u32p]
        L.or_label.restype = ctypes.c_uint32
        L.or_segment.argtypes = [ctypes.POINTER(Params), _u8p, _u8p, _u8p, ctypes.c_int64,
                                 ctypes.POINTER(Stages), ctypes.POINTER(Record)]
        L.or_track_init.argtypes = [ctypes.POINTER(TState)]
        L.or_track.argtypes = [ctypes.POINTER(Params), ctypes.POINTER(TState),
                               ctypes.POINTER(Record)]
        L.or_segment_batch.argtypes = [ctypes.POINTER(Params), _u8p, ctypes.c_uint32, _u8p, _u8p,
                                       ctypes.POINTER(ctypes.c_int64), ctypes.c_uint32,
                                       ctypes.POINTER(Record), _u8p]
        assert L.or_sizeof_record() == ctypes.sizeof(Record)
        assert L.or_sizeof_params() == ctypes.sizeof(Params)
        assert L.or_sizeof_tstate() == ctypes.sizeof(TState)
    return _lib


def _p(a: np.ndarray, t=_u8p):
    return a.ctypes.data_as(t)


def _c(a, dtype=np.uint8) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=dtype)


# ------------------------------------------------------------------ a1 learn
def learn(frames: np.ndarray, margin: int):
    """frames (n,h,w,3) u8 -> (lo, hi) (h,w,3) u8 envelope."""
    frames = _c(frames)
    n, h, w, _ = frames.shape
    lo = np.empty((h, w, 3), np.uint8)
    hi = np.empty((h, w, 3), np.uint8)
    rc = lib().or_learn(_p(frames), n, w, h, margin, _p(lo), _p(hi))
    if rc != 0:
        raise ValueError(f"or_learn failed: {rc}")
    return lo, hi


# --------------------------------------------------------------- a2 luminosity
def mean_luma(frame: np.ndarray):
    frame = _c(frame)
    h, w, _ = frame.shape
    s = ctypes.c_uint64()
    m = lib().or_mean_luma(_p(frame), w, h, ctypes.byref(s))
    return int(m), int(s.value)


def gamma(params: Params, mean: int):
    c = ctypes.c_uint32()
    g = lib().or_gamma(ctypes.byref(params), mean, ctypes.byref(c))
    return float(g), int(c.value)


def lut(g: float) -> np.ndarray:
    out = np.empty(256, np.uint8)
    lib().or_lut(g, _p(out))
    return out


# ------------------------------------------------------------ a3 branches
def hue_num(r: int, g: int, b: int):
    v = (ctypes.c_uint8 * 3)(r, g, b)
    hn = ctypes.c_int64()
    C = lib().or_hue_num(v, ctypes.byref(hn))
    return int(hn.value), int(C)


def in_band(hn: int, C: int, a1: int, a2: int) -> int:
    return int(lib().or_in_band(hn, C, a1, a2))


# ---------------------------------------------------------- a4 morphology
def _morph(fn, mask: np.ndarray, r: int) -> np.ndarray:
    mask = _c(mask)
    h, w = mask.shape
    out = np.empty_like(mask)
    fn(_p(mask), _p(out), w, h, r)
    return out


def erode(mask, r=1):
    return _morph(lib().or_erode, mask, r)


def dilate(mask, r=1):
    return _morph(lib().or_dilate, mask, r)


def open_close(mask, r=1):
    return _morph(lib().or_open_close, mask, r)


def label(mask: np.ndarray):
    mask = _c(mask)
    h, w = mask.shape
    lab = np.empty((h, w), np.uint32)
    n = lib().or_label(_p(mask), w, h, _p(lab, _u32p))
    return lab, int(n)


# ------------------------------------------------------- whole frame / fold
STAGE_NAMES = ("r1", "r2", "r3", "merged", "oc", "labels", "final_mask", "contour")


def segment(params: Params, frame: np.ndarray, lo: np.ndarray, hi: np.ndarray,
            t_ms: int = 0, stages: bool = True):
    """One frame through a2..a7.  Returns (record dict, dict of stage arrays)."""
    frame, lo, hi = _c(frame), _c(lo), _c(hi)
    h, w = params.height, params.width
    assert frame.shape == (h, w, 3) and lo.shape == (h, w, 3) and hi.shape == (h, w, 3)
    st = Stages()
    arrs = {}
    if stages:
        for name in STAGE_NAMES:
            if name == "labels":
                arrs[name] = np.zeros((h, w), np.uint32)
                setattr(st, name, _p(arrs[name], _u32p))
            else:
                arrs[name] = np.zeros((h, w), np.uint8)
                setattr(st, name, _p(arrs[name]))
    rec = Record()
    rc = lib().or_segment(ctypes.byref(params), _p(frame), _p(lo), _p(hi), int(t_ms),
                          ctypes.byref(st), ctypes.byref(rec))
    if rc != 0:
        raise ValueError(f"or_segment failed: {rc}")
    return rec, arrs


def segment_batch(params: Params, frames: np.ndarray, lo, hi, t_ms=None, nthreads: int = 1,
                  want_masks: bool = True, as_array: bool = False):
    """Frame-parallel batch (threads over frames; no tracking).  as_array:
    the records as one numpy structured array (fields of Record) instead of
    a list of Record."""
    frames, lo, hi = _c(frames), _c(lo), _c(hi)
    n = frames.shape[0]
    recs = (Record * max(n, 1))()
    masks = np.zeros((n, params.height, params.width), np.uint8) if want_masks else None
    if t_ms is None:
        t_ms = np.zeros(n, np.int64)
    t_ms = _c(t_ms, np.int64)
    lib().or_segment_batch(ctypes.byref(params), _p(frames), n, _p(lo), _p(hi),
                           t_ms.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), nthreads,
                           recs, _p(masks) if masks is not None else None)
    if as_array:
        return np.ctypeslib.as_array(recs)[:n].copy(), masks
    return [recs[i] for i in range(n)], masks


class Tracker:
    """Sequential Mouse fold for one stream (a8)."""

    def __init__(self, params: Params):
        self.params = params
        self.state = TState()
        lib().or_track_init(ctypes.byref(self.state))

    def update(self, rec: Record) -> Record:
        lib().or_track(ctypes.byref(self.params), ctypes.byref(self.state), ctypes.byref(rec))
        return rec


def record_from_blob(t_ms: int, area: int = 0, cx: float = 0.0, cy: float = 0.0) -> Record:
    """A record carrying only what the fold reads (blob_area, cx, cy, t_ms)."""
    r = Record()
    r.t_ms = t_ms
    r.blob_area = area
    r.cx = cx
    r.cy = cy
    return r
