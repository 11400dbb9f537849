"""Thin ctypes binding of libfizi.so (include/fizi.h).

Argument marshalling only: every step of the pixel path runs in the CUDA
kernels behind the C ABI.  PyTorch provides device memory and the current CUDA
stream.  There is no CPU fallback: if libfizi.so is missing or no CUDA device
is present, constructing a ``Fizi`` raises.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
# FIZI_LIB=checked selects the build with device-side invariant checks;
# FIZI_LIB=<file>.so an alternative in-tree build (A/B experiments)
_lib_env = os.environ.get("FIZI_LIB", "")
LIB_PATH = os.path.join(HERE, "libfizi_checked.so" if _lib_env == "checked"
                        else _lib_env if _lib_env.endswith(".so") else "libfizi.so")

# fizi_status
OK, E_ARG, E_EMPTY, E_DIMS, E_NOMODEL, E_TIME, E_CUDA, E_OOM, E_CAPACITY = 0, -1, -2, -3, -4, -5, -6, -7, -8

STAGES = {"r1": 0, "r2": 1, "r3": 2, "merged": 3, "openclose": 4, "labels": 5, "final": 6,
          "contour": 7}


class FiziError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{msg} (status {status})")
        self.status = status


class Params(ctypes.Structure):
    _fields_ = [
        ("width", ctypes.c_uint32), ("height", ctypes.c_uint32),
        ("gray_tol_S", ctypes.c_uint32), ("hue_lo_deg", ctypes.c_uint32),
        ("hue_hi_deg", ctypes.c_uint32), ("se_radius", ctypes.c_uint32),
        ("min_blob_ppm", ctypes.c_uint32), ("luma_target", ctypes.c_uint32),
        ("luma_lo", ctypes.c_uint32), ("luma_hi", ctypes.c_uint32),
        ("gamma_min", ctypes.c_double), ("gamma_max", ctypes.c_double),
        ("beta", ctypes.c_double), ("dwell_radius_px", ctypes.c_double),
        ("dwell_time_ms", ctypes.c_int64), ("lost_timeout_ms", ctypes.c_int64),
        ("debug", ctypes.c_uint32), ("_reserved", ctypes.c_uint32),
    ]


# fizi_result as a numpy structured dtype (128 bytes, offsets of include/fizi.h)
RESULT_DTYPE = np.dtype({
    "names": ["t_ms", "stream", "frame_idx", "mean_luma", "corrected", "visible", "clicked",
              "fg_merged", "fg_final", "n_comp_total", "n_comp_kept", "blob_area", "blob_label",
              "bbox", "relearn", "sum_x", "sum_y", "gamma", "cx", "cy", "px", "py", "dwell_ms"],
    "formats": ["<i8", "<u4", "<u4", "u1", "u1", "u1", "u1", "<u4", "<u4", "<u4", "<u4", "<u4",
                "<u4", ("<u4", (4,)), "<u4", "<u8", "<u8", "<f8", "<f8", "<f8", "<f8", "<f8",
                "<i8"],
    "offsets": [0, 8, 12, 16, 17, 18, 19, 20, 24, 28, 32, 36, 40, 44, 60, 64, 72, 80, 88, 96,
                104, 112, 120],
    "itemsize": 128,
})
RESULT_BYTES = 128
RELEARN_LEARN, RELEARN_SWAP, RELEARN_TRIGGER = 1, 2, 4   # fizi_result.relearn flags (NEXT-1)
CALL_SLOTS = 4          # FIZI_CALL_SLOTS default (include/fizi.h); Fizi.call_slots = the loaded build's


class Wheel(ctypes.Structure):
    """fizi_wheel (NEXT-2 drive mapping, include/fizi.h)."""
    _fields_ = [("cx", ctypes.c_double), ("cy", ctypes.c_double), ("radius", ctypes.c_double),
                ("theta_max_deg", ctypes.c_double), ("inner", ctypes.c_double),
                ("outer", ctypes.c_double), ("dead_zone_deg", ctypes.c_double),
                ("hold_ms", ctypes.c_int64)]


class Zone(ctypes.Structure):
    """fizi_zone (NEXT-3 interface hit-test, include/fizi.h)."""
    _fields_ = [("kind", ctypes.c_uint32), ("_pad", ctypes.c_uint32),
                ("x", ctypes.c_double), ("y", ctypes.c_double), ("w", ctypes.c_double),
                ("h", ctypes.c_double), ("cx", ctypes.c_double), ("cy", ctypes.c_double),
                ("r", ctypes.c_double), ("theta_max_deg", ctypes.c_double)]


ZONE_BUTTON, ZONE_SLIDER, ZONE_WHEEL = 0, 1, 2
EV_ENTER, EV_LEAVE, EV_CLICK, EV_VALUE = 1, 2, 4, 8
ZONE_EVENT_DTYPE = np.dtype({"names": ["inside", "events", "value"], "formats": ["u1", "u1", "<f8"],
                             "offsets": [0, 1, 8], "itemsize": 16})

# fizi_command (32 bytes)
COMMAND_DTYPE = np.dtype({"names": ["steering", "throttle", "t_ms", "has_steering"],
                          "formats": ["<f8", "<f8", "<i8", "<u4"],
                          "offsets": [0, 8, 16, 24], "itemsize": 32})
COMMAND_BYTES = 32
PROF_NAMES = ("segment", "fixup", "morph", "ccl", "expand", "track", "slow", "maskzero")
PROF_SLOTS = len(PROF_NAMES)

_lib = None


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is missing: run __graft_entry__.build() "
                               "(no CPU fallback exists)")
        L = ctypes.CDLL(LIB_PATH)
        vp, u32, u8, i32 = ctypes.c_void_p, ctypes.c_uint32, ctypes.c_uint8, ctypes.c_int
        L.fizi_params_default.argtypes = [ctypes.POINTER(Params), u32, u32]
        L.fizi_create.argtypes = [ctypes.POINTER(Params), i32, u32, u32, ctypes.POINTER(vp)]
        L.fizi_learn_background.argtypes = [vp, u32, vp, u32, u32, u32, u8, vp]
        for fn in (L.fizi_process_frames, L.fizi_segment_frames, L.fizi_process_frames_host):
            fn.argtypes = [vp, vp, vp, u32, u32, u32, vp, vp, vp, vp]
        L.fizi_track.argtypes = [vp, u32, vp, u32, vp]
        L.fizi_track_runs.argtypes = [vp, u32, vp, vp, vp, u32, vp]
        L.fizi_reset_tracker.argtypes = [vp, u32, vp]
        L.fizi_debug_stage.argtypes = [vp, i32, u32, vp, vp]
        L.fizi_get_background.argtypes = [vp, u32, vp, vp, vp]
        L.fizi_set_background.argtypes = [vp, u32, vp, vp, vp]
        L.fizi_profile_enable.argtypes = [vp, i32]
        L.fizi_profile_enable.restype = i32
        L.fizi_profile_read.argtypes = [vp, vp, vp, i32]
        L.fizi_profile_read.restype = i32
        L.fizi_kernel_launches.argtypes = [vp]
        L.fizi_kernel_launches.restype = ctypes.c_uint64
        L.fizi_call_slots.argtypes = []
        L.fizi_call_slots.restype = ctypes.c_uint32
        L.fizi_last_error.argtypes = [vp]
        L.fizi_last_error.restype = ctypes.c_char_p
        L.fizi_status_string.argtypes = [i32]
        L.fizi_status_string.restype = ctypes.c_char_p
        L.fizi_destroy.argtypes = [vp]
        L.fizi_set_pipeline.argtypes = [vp, i32]
        L.fizi_wheel_default.argtypes = [ctypes.POINTER(Wheel), ctypes.c_double, ctypes.c_double,
                                         ctypes.c_double]
        L.fizi_set_wheel.argtypes = [vp, u32, ctypes.POINTER(Wheel)]
        L.fizi_drive.argtypes = [vp, u32, vp, u32, vp, vp]
        L.fizi_drive_throttle.argtypes = [vp, u32, vp, u32, vp, u32, u32, vp, vp]
        L.fizi_relearn_flags.argtypes = [vp, u32, vp, u32, u32, vp, vp]
        L.fizi_set_relearn.argtypes = [vp, u32, u32, u32, u8]
        L.fizi_set_zones.argtypes = [vp, u32, vp, u32]
        L.fizi_hit_test.argtypes = [vp, u32, vp, u32, vp, vp]
        L.fizi_flush.argtypes = [vp, vp]
        L.fizi_get_lut_table.argtypes = [vp, vp, vp, vp, vp]
        for name in ("fizi_set_pipeline", "fizi_flush", "fizi_wheel_default", "fizi_set_wheel",
                     "fizi_drive", "fizi_drive_throttle", "fizi_relearn_flags", "fizi_set_relearn", "fizi_set_zones", "fizi_hit_test", "fizi_params_default", "fizi_create", "fizi_learn_background",
                     "fizi_process_frames", "fizi_segment_frames", "fizi_process_frames_host",
                     "fizi_track", "fizi_track_runs", "fizi_reset_tracker", "fizi_debug_stage",
                     "fizi_get_background", "fizi_set_background", "fizi_get_lut_table"):
            getattr(L, name).restype = i32
        _lib = L
    return _lib


def default_params(width: int, height: int, **kw) -> Params:
    p = Params()
    lib().fizi_params_default(ctypes.byref(p), width, height)
    for k, v in kw.items():
        if not hasattr(p, k):
            raise TypeError(f"unknown parameter {k}")
        setattr(p, k, v)
    return p


def _stream_handle(device) -> int:
    import torch
    raw = getattr(torch._C, "_cuda_getCurrentRawStream", None)
    if raw is not None:                         # the current stream's handle, without a Stream object
        return raw(device.index if hasattr(device, "index") else int(device))
    return torch.cuda.current_stream(device).cuda_stream


def _u32(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.uint32))


def _i64(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.int64))


class Fizi:
    """One libfizi context: n_streams camera streams of width x height frames."""

    def __init__(self, width: int, height: int, n_streams: int = 1, max_batch: int = 64,
                 device: int = 0, **params):
        import torch
        if not torch.cuda.is_available():
            raise RuntimeError("libfizi needs a CUDA device (no CPU fallback)")
        self.W, self.H = int(width), int(height)
        self.n_streams, self.max_batch = int(n_streams), int(max_batch)
        self._learned = {}                 # stream -> (frames learned, margin), for FIZIBG1
        self._nz = {}                      # stream -> zones of its layout (NEXT-3)
        self._zeros_u32 = np.zeros(self.max_batch, np.uint32)
        self._zeros_i64 = np.zeros(self.max_batch, np.int64)
        self.device = torch.device("cuda", device)
        self._dev_index = int(device)
        self.params = default_params(self.W, self.H, **params)
        self._h = ctypes.c_void_p()
        rc = lib().fizi_create(ctypes.byref(self.params), device, self.n_streams,
                               self.max_batch, ctypes.byref(self._h))
        if rc != OK:
            raise FiziError(rc, f"fizi_create failed: {lib().fizi_status_string(rc).decode()}")

    # ------------------------------------------------------------ helpers
    def _check(self, rc: int, what: str):
        if rc != OK:
            raise FiziError(rc, f"{what}: {lib().fizi_status_string(rc).decode()}: "
                                f"{lib().fizi_last_error(self._h).decode()}")

    def _frames(self, frames):
        import torch
        if not (isinstance(frames, torch.Tensor) and frames.is_cuda and frames.dtype == torch.uint8):
            raise TypeError("frames must be a CUDA uint8 tensor (n, H, W, 3)")
        if not frames.is_contiguous():
            raise ValueError("frames must be contiguous")
        if frames.dim() == 3:
            frames = frames.unsqueeze(0)
        if frames.dim() != 4 or frames.shape[3] != 3:
            raise ValueError("frames must have shape (n, H, W, 3)")
        if frames.get_device() != self._dev_index:
            raise ValueError(f"frames are on {frames.device}, the context on {self.device}")
        return frames

    def _dev_buf(self, t, nbytes: int, what: str):
        """A caller-supplied device output buffer: contiguous, on the context's
        device, and at least the nbytes the C side writes."""
        import torch
        if not (isinstance(t, torch.Tensor) and t.is_cuda):
            raise TypeError(f"{what} must be a CUDA tensor")
        if t.get_device() != self._dev_index:
            raise ValueError(f"{what} is on {t.device}, the context on {self.device}")
        if not t.is_contiguous():
            raise ValueError(f"{what} must be contiguous")
        if t.numel() * t.element_size() < nbytes:
            raise ValueError(f"{what} holds {t.numel() * t.element_size()} bytes, needs {nbytes}")
        return t

    @staticmethod
    def _host_buf(a, dtype, count: int, what: str):
        if not (isinstance(a, np.ndarray) and a.dtype == dtype and a.flags.c_contiguous):
            raise TypeError(f"{what} must be a C-contiguous numpy array of {dtype}")
        if a.size < count:
            raise ValueError(f"{what} holds {a.size} elements, needs {count}")
        return a

    def close(self):
        if self._h:
            lib().fizi_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -------------------------------------------------------------- API
    def learn_background(self, frames, stream: int = 0, margin: int = 10):
        frames = self._frames(frames)
        n = frames.shape[0]
        self._learned[stream] = (n, margin)
        self._check(lib().fizi_learn_background(self._h, stream, frames.data_ptr(), n,
                                                frames.shape[2], frames.shape[1], margin,
                                                _stream_handle(self.device)),
                    "fizi_learn_background")

    def _call(self, fn, name, frames, streams, t_ms, masks, results):
        import torch
        frames = self._frames(frames)
        n = frames.shape[0]
        if streams is None:
            streams = self._zeros_u32[:n] if n <= self.max_batch else np.zeros(n, np.uint32)
        elif not (isinstance(streams, np.ndarray) and streams.dtype == np.uint32
                  and streams.shape == (n,) and streams.flags.c_contiguous):
            streams = _u32(np.broadcast_to(np.asarray(streams, np.uint32), (n,)))
        if t_ms is None:
            t = self._zeros_i64[:n] if n <= self.max_batch else np.zeros(n, np.int64)
        elif not (isinstance(t_ms, np.ndarray) and t_ms.dtype == np.int64 and t_ms.flags.c_contiguous):
            t = _i64(t_ms)
        else:
            t = t_ms
        if t.shape != (n,):
            raise ValueError("t_ms must have one timestamp per frame")
        if masks is True:
            masks = torch.empty((n, self.H, self.W), dtype=torch.uint8, device=self.device)
        elif masks is not None:
            self._dev_buf(masks, n * self.H * self.W, "masks")
            if masks.dtype != torch.uint8:
                raise TypeError("masks must be uint8")
        if results is None:
            results = torch.empty((n, RESULT_BYTES), dtype=torch.uint8, device=self.device)
        else:
            self._dev_buf(results, n * RESULT_BYTES, "results")
        self._last_frames = frames          # R1/R2/R3 debug stages re-read the last frames
        self._check(fn(self._h, streams.ctypes.data, frames.data_ptr(), n, frames.shape[2],
                       frames.shape[1], t.ctypes.data, masks.data_ptr() if masks is not None else None,
                       results.data_ptr(), _stream_handle(self.device)), name)
        return masks, results

    def process_frames(self, frames, streams=None, t_ms=None, masks=True, results=None):
        """Full path a2..a8; returns (masks uint8 (n,H,W) or None, results (n,128) uint8)."""
        return self._call(lib().fizi_process_frames, "fizi_process_frames", frames, streams,
                          t_ms, masks, results)

    def segment_frames(self, frames, streams=None, t_ms=None, masks=True, results=None):
        """Stateless a2..a7 (tracker untouched)."""
        return self._call(lib().fizi_segment_frames, "fizi_segment_frames", frames, streams,
                          t_ms, masks, results)

    def track(self, results, stream: int = 0):
        """Fold records (device (n,128) uint8 tensor) through stream's tracker in place."""
        n = results.shape[0]
        self._dev_buf(results, n * RESULT_BYTES, "results")
        self._check(lib().fizi_track(self._h, stream, results.data_ptr(), n,
                                     _stream_handle(self.device)), "fizi_track")
        return results

    def track_runs(self, results, runs, stream: int = 0):
        """Fold the rows results[o:o+n] for (o, n) in runs, in that order, through
        stream's tracker (one launch; records gathered from several ranks)."""
        runs = list(runs)
        n_all = results.shape[0]
        self._dev_buf(results, n_all * RESULT_BYTES, "results")
        off = _u32([o for o, _ in runs])
        ln = _u32([n for _, n in runs])
        if any(o + n > n_all for o, n in runs):
            raise ValueError("a run exceeds the results buffer")
        self._check(lib().fizi_track_runs(self._h, stream, results.data_ptr(), off.ctypes.data,
                                          ln.ctypes.data, len(runs), _stream_handle(self.device)),
                    "fizi_track_runs")
        return results

    def process_frames_host(self, frames: np.ndarray, streams=None, t_ms=None,
                            masks: np.ndarray | None = None, results: np.ndarray | None = None):
        """End-to-end on host buffers (H2D + path + D2H inside the call)."""
        frames = np.ascontiguousarray(frames, np.uint8)
        if frames.ndim == 3:
            frames = frames[None]
        if frames.ndim != 4 or frames.shape[3] != 3:
            raise ValueError("frames must have shape (n, H, W, 3)")
        n = frames.shape[0]
        streams = _u32(np.broadcast_to(np.asarray(0 if streams is None else streams, np.uint32), (n,)))
        t = _i64(np.zeros(n) if t_ms is None else t_ms)
        if t.shape != (n,):
            raise ValueError("t_ms must have one timestamp per frame")
        if results is None:
            results = np.zeros(n, RESULT_DTYPE)
        self._host_buf(results, RESULT_DTYPE, n, "results")
        if masks is not None:
            self._host_buf(masks, np.uint8, n * self.H * self.W, "masks")
        self._check(lib().fizi_process_frames_host(
            self._h, streams.ctypes.data, frames.ctypes.data, n, frames.shape[2], frames.shape[1],
            t.ctypes.data,
            masks.ctypes.data if masks is not None else None, results.ctypes.data,
            _stream_handle(self.device)), "fizi_process_frames_host")
        return masks, results

    def reset_tracker(self, stream: int = 0):
        self._check(lib().fizi_reset_tracker(self._h, stream, _stream_handle(self.device)),
                    "fizi_reset_tracker")

    def debug_stage(self, stage, frame: int = 0):
        import torch
        sid = STAGES[stage] if isinstance(stage, str) else int(stage)
        dt = torch.int32 if sid == STAGES["labels"] else torch.uint8
        out = torch.empty((self.H, self.W), dtype=dt, device=self.device)
        self._check(lib().fizi_debug_stage(self._h, sid, frame, out.data_ptr(),
                                           _stream_handle(self.device)), "fizi_debug_stage")
        return out

    def get_lut_table(self):
        """K0 tables (device): LUT rows (256, 256) u8, gamma (256,) f64, corrected (256,) u8."""
        import torch
        lut = torch.empty((256, 256), dtype=torch.uint8, device=self.device)
        gam = torch.empty(256, dtype=torch.float64, device=self.device)
        cor = torch.empty(256, dtype=torch.uint8, device=self.device)
        self._check(lib().fizi_get_lut_table(self._h, lut.data_ptr(), gam.data_ptr(), cor.data_ptr(),
                                             _stream_handle(self.device)), "fizi_get_lut_table")
        return lut, gam, cor

    def get_background(self, stream: int = 0):
        import torch
        lo = torch.empty((self.H, self.W, 3), dtype=torch.uint8, device=self.device)
        hi = torch.empty_like(lo)
        self._check(lib().fizi_get_background(self._h, stream, lo.data_ptr(), hi.data_ptr(),
                                              _stream_handle(self.device)), "fizi_get_background")
        return lo, hi

    def set_background(self, lo, hi, stream: int = 0):
        for a, nm in ((lo, "lo"), (hi, "hi")):
            self._dev_buf(a, self.H * self.W * 3, nm)
        self._check(lib().fizi_set_background(self._h, stream, lo.data_ptr(), hi.data_ptr(),
                                              _stream_handle(self.device)), "fizi_set_background")

    def save_background(self, dst, stream: int = 0, frames_learned: int | None = None,
                        margin: int | None = None):
        """Write stream's envelope as a FIZIBG1 file (persist.py, NEXT-4)."""
        import torch
        from .persist import BackgroundModel, save_background
        lo, hi = self.get_background(stream)
        torch.cuda.current_stream(self.device).synchronize()
        n0, m0 = self._learned.get(stream, (0, 0))
        save_background(dst, BackgroundModel(lo.cpu().numpy(), hi.cpu().numpy(),
                                             n0 if frames_learned is None else frames_learned,
                                             m0 if margin is None else margin))

    def load_background(self, src, stream: int = 0):
        """Install a FIZIBG1 file as stream's envelope; returns the model."""
        import torch
        from .persist import load_background
        m = load_background(src)
        if (m.width, m.height) != (self.W, self.H):
            raise ValueError(f"model is {m.width}x{m.height}, context is {self.W}x{self.H}")
        lo = torch.from_numpy(m.lo).to(self.device)
        hi = torch.from_numpy(m.hi).to(self.device)
        self.set_background(lo, hi, stream)
        torch.cuda.current_stream(self.device).synchronize()
        self._learned[stream] = (m.frames_learned, m.margin)
        return m

    def dump_stages(self, directory, frame_no: int, frame: int = 0):
        """Write frame `frame` of the last batch's stage masks as
        <frame_no>_{r1,r2,r3,merged,final}.pgm (needs debug=1)."""
        import torch
        from .persist import DUMP_STAGES, dump_stages
        st = {s: self.debug_stage(s, frame) for s in DUMP_STAGES}
        torch.cuda.current_stream(self.device).synchronize()
        return dump_stages(directory, frame_no, {s: m.cpu().numpy() for s, m in st.items()})

    def relearn_flags(self, results, stream: int = 0, threshold: int = 40):
        """NEXT-1: u8 flag per record, 1 iff the mean luma jumped by more than
        `threshold` since the stream's previous frame (device (n,) tensor)."""
        import torch
        n = results.shape[0]
        self._dev_buf(results, n * RESULT_BYTES, "results")
        flags = torch.empty(n, dtype=torch.uint8, device=self.device)
        self._check(lib().fizi_relearn_flags(self._h, stream, results.data_ptr(), n, threshold,
                                             flags.data_ptr(), _stream_handle(self.device)),
                    "fizi_relearn_flags")
        return flags

    def set_relearn(self, stream: int = 0, threshold: int = 40, n_frames: int = 30,
                    margin: int = 10):
        """NEXT-1 in-stream relearning of `stream` (fizi_set_relearn); n_frames=0 disables.
        Records carry the RELEARN_* flags in their `relearn` field."""
        self._check(lib().fizi_set_relearn(self._h, stream, threshold, n_frames, margin),
                    "fizi_set_relearn")

    def set_zones(self, zones, stream: int = 0):
        """NEXT-3: install a layout (sequence of Zone) for `stream`."""
        arr = (Zone * max(len(zones), 1))(*zones)
        self._check(lib().fizi_set_zones(self._h, stream, ctypes.cast(arr, ctypes.c_void_p),
                                         len(zones)), "fizi_set_zones")
        self._nz[stream] = len(zones)

    def hit_test(self, results, stream: int = 0):
        """NEXT-3: per frame and zone membership + events (device (n, n_zones, 16) uint8)."""
        import torch
        n = results.shape[0]
        self._dev_buf(results, n * RESULT_BYTES, "results")
        nz = self._nz.get(stream, 0)
        out = torch.empty((n, max(nz, 1), 16), dtype=torch.uint8, device=self.device)
        self._check(lib().fizi_hit_test(self._h, stream, results.data_ptr(), n, out.data_ptr(),
                                        _stream_handle(self.device)), "fizi_hit_test")
        return out

    def set_wheel(self, cx: float, cy: float, radius: float, stream: int = 0, **kw):
        """NEXT-2: install the virtual steering wheel of `stream` (fizi_set_wheel);
        keyword overrides: theta_max_deg, inner, outer, dead_zone_deg, hold_ms."""
        w = Wheel()
        self._check(lib().fizi_wheel_default(ctypes.byref(w), cx, cy, radius), "fizi_wheel_default")
        for k, v in kw.items():
            setattr(w, k, v)
        self._check(lib().fizi_set_wheel(self._h, stream, ctypes.byref(w)), "fizi_set_wheel")
        return w

    def drive(self, results, stream: int = 0, commands=None, events=None, slider_zone=None):
        """NEXT-2: fold records (device (n,128) uint8) into drive commands
        (device (n,32) uint8 tensor of fizi_command).  With `events` (the
        hit_test output for the same records) and `slider_zone`, the throttle
        follows that slider (fizi_drive_throttle)."""
        import torch
        n = results.shape[0]
        self._dev_buf(results, n * RESULT_BYTES, "results")
        if commands is None:
            commands = torch.empty((n, COMMAND_BYTES), dtype=torch.uint8, device=self.device)
        else:
            self._dev_buf(commands, n * COMMAND_BYTES, "commands")
        if events is None:
            self._check(lib().fizi_drive(self._h, stream, results.data_ptr(), n,
                                         commands.data_ptr(), _stream_handle(self.device)),
                        "fizi_drive")
        else:
            nz = events.numel() // (16 * n) if n else 0
            self._dev_buf(events, n * nz * 16, "events")
            self._check(lib().fizi_drive_throttle(self._h, stream, results.data_ptr(), n,
                                                  events.data_ptr(), nz, int(slider_zone),
                                                  commands.data_ptr(), _stream_handle(self.device)),
                        "fizi_drive_throttle")
        return commands

    def set_pipeline(self, enable: bool = True):
        """Pipelined mode (include/fizi.h): a call's tail overlaps the next call;
        outputs are complete on the current stream after flush()."""
        self._check(lib().fizi_set_pipeline(self._h, int(bool(enable))), "fizi_set_pipeline")

    def flush(self):
        """Join every outstanding call tail into the current stream."""
        self._check(lib().fizi_flush(self._h, _stream_handle(self.device)), "fizi_flush")

    def profile_enable(self, mode=True):
        """mode True/1: every stage; 2: the fused segmentation kernel only; False/0: off."""
        self._check(lib().fizi_profile_enable(self._h, int(mode)), "fizi_profile_enable")

    def profile_read(self, reset: bool = True) -> dict:
        ms = np.zeros(PROF_SLOTS, np.float64)
        cnt = np.zeros(PROF_SLOTS, np.uint64)
        self._check(lib().fizi_profile_read(self._h, ms.ctypes.data, cnt.ctypes.data, int(reset)),
                    "fizi_profile_read")
        return {name: (float(ms[i]), int(cnt[i])) for i, name in enumerate(PROF_NAMES)}

    def kernel_launches(self) -> int:
        return int(lib().fizi_kernel_launches(self._h))

    @property
    def call_slots(self) -> int:
        """FIZI_CALL_SLOTS of the loaded library (output buffers a pipelined
        caller may rotate)."""
        return int(lib().fizi_call_slots())


def results_numpy(results) -> np.ndarray:
    """(n,128) uint8 tensor/array of fizi_result -> numpy structured array."""
    try:
        import torch
        if isinstance(results, torch.Tensor):
            results = results.cpu().numpy()
    except ImportError:
        pass
    a = np.ascontiguousarray(results)
    if a.dtype == RESULT_DTYPE:
        return a
    return a.view(np.uint8).reshape(-1, RESULT_BYTES).view(RESULT_DTYPE).reshape(-1)


def commands_numpy(commands) -> np.ndarray:
    """(n,32) uint8 tensor/array of fizi_command -> numpy structured array."""
    try:
        import torch
        if isinstance(commands, torch.Tensor):
            commands = commands.cpu().numpy()
    except ImportError:
        pass
    return np.ascontiguousarray(commands).view(COMMAND_DTYPE).reshape(-1)
