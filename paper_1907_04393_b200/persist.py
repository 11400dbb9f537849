"""Background-model persistence and raw frame streams.

Host-side file plumbing around the device envelope (fizi_get_background /
fizi_set_background); no pixel arithmetic happens here.

FIZIBG1: magic b"FIZIBG1\\0", little-endian u32
width, u32 height, u32 frames_learned, u8 margin, 3 padding bytes, then the
min plane (w*h*3 bytes, interleaved RGB) and the max plane (same size).
load(save(m)) == m bit-exactly; a wrong magic or a truncated file raises
FormatError naming the byte offset / expected vs actual length.

FIZIRAW1: 16-byte header b"FIZIRAW1" + u32 width + u32 height, then
frames of w*h*3 bytes back to back.
"""
from __future__ import annotations

import io
import os
import struct
from dataclasses import dataclass

import numpy as np

BG_MAGIC = b"FIZIBG1\0"
BG_HEADER = struct.Struct("<8sIIIB3x")            # 24 bytes
RAW_MAGIC = b"FIZIRAW1"
RAW_HEADER = struct.Struct("<8sII")               # 16 bytes


class FormatError(ValueError):
    """Malformed FIZIBG1 / FIZIRAW1 data; the message names the byte offset."""


@dataclass
class BackgroundModel:
    lo: np.ndarray                 # (H, W, 3) u8, I_bg_min after widening
    hi: np.ndarray                 # (H, W, 3) u8, I_bg_max after widening
    frames_learned: int
    margin: int

    @property
    def width(self) -> int:
        return int(self.lo.shape[1])

    @property
    def height(self) -> int:
        return int(self.lo.shape[0])


def _open(dst, mode):
    if isinstance(dst, (str, os.PathLike)):
        return open(dst, mode), True
    return dst, False


def save_background(dst, model: BackgroundModel) -> None:
    """Write `model` as FIZIBG1 to a path or a binary file object."""
    lo = np.ascontiguousarray(model.lo, np.uint8)
    hi = np.ascontiguousarray(model.hi, np.uint8)
    if lo.ndim != 3 or lo.shape[2] != 3 or hi.shape != lo.shape:
        raise ValueError("lo / hi must both be (H, W, 3) uint8")
    if not 0 <= model.margin <= 255 or model.frames_learned < 0:
        raise ValueError("margin must be in [0, 255], frames_learned >= 0")
    f, own = _open(dst, "wb")
    try:
        f.write(BG_HEADER.pack(BG_MAGIC, lo.shape[1], lo.shape[0], int(model.frames_learned),
                               int(model.margin)))
        f.write(lo.tobytes())
        f.write(hi.tobytes())
    finally:
        if own:
            f.close()


def load_background(src) -> BackgroundModel:
    """Read a FIZIBG1 model from a path, bytes or a binary file object."""
    if isinstance(src, (bytes, bytearray, memoryview)):
        data = bytes(src)
    else:
        f, own = _open(src, "rb")
        try:
            data = f.read()
        finally:
            if own:
                f.close()
    if len(data) < BG_HEADER.size:
        raise FormatError(f"truncated header: expected {BG_HEADER.size} bytes, got {len(data)} "
                          f"(at byte offset {len(data)})")
    magic, w, h, frames_learned, margin = BG_HEADER.unpack_from(data, 0)
    if magic != BG_MAGIC:
        raise FormatError(f"bad magic {magic!r} at byte offset 0 (expected {BG_MAGIC!r})")
    plane = w * h * 3
    need = BG_HEADER.size + 2 * plane
    if len(data) < need:
        which = "min" if len(data) < BG_HEADER.size + plane else "max"
        raise FormatError(f"truncated in the {which} plane: expected {need} bytes, got "
                          f"{len(data)} (at byte offset {len(data)})")
    off = BG_HEADER.size
    lo = np.frombuffer(data, np.uint8, plane, off).reshape(h, w, 3).copy()
    hi = np.frombuffer(data, np.uint8, plane, off + plane).reshape(h, w, 3).copy()
    return BackgroundModel(lo, hi, int(frames_learned), int(margin))


def write_rawstream(dst, frames: np.ndarray) -> None:
    """Write (n, H, W, 3) u8 frames as a FIZIRAW1 stream."""
    frames = np.ascontiguousarray(frames, np.uint8)
    if frames.ndim != 4 or frames.shape[3] != 3:
        raise ValueError("frames must be (n, H, W, 3) uint8")
    f, own = _open(dst, "wb")
    try:
        f.write(RAW_HEADER.pack(RAW_MAGIC, frames.shape[2], frames.shape[1]))
        f.write(frames.tobytes())
    finally:
        if own:
            f.close()


class RawStream:
    """Reader of a FIZIRAW1 file: batches of frames as (n, H, W, 3) u8 arrays
    (memory-mapped; copy into pinned memory before fizi_process_frames_host)."""

    def __init__(self, path):
        with open(path, "rb") as f:
            head = f.read(RAW_HEADER.size)
        if len(head) < RAW_HEADER.size:
            raise FormatError(f"truncated header: expected {RAW_HEADER.size} bytes, got {len(head)} "
                              f"(at byte offset {len(head)})")
        magic, w, h = RAW_HEADER.unpack(head)
        if magic != RAW_MAGIC:
            raise FormatError(f"bad magic {magic!r} at byte offset 0 (expected {RAW_MAGIC!r})")
        self.width, self.height = w, h
        size = os.path.getsize(path) - RAW_HEADER.size
        fb = w * h * 3
        if fb == 0 or size % fb:
            raise FormatError(f"stream body of {size} bytes is not a whole number of {fb}-byte "
                              f"frames (at byte offset {RAW_HEADER.size + size - size % fb if fb else 0})")
        self.n_frames = size // fb
        self._mm = np.memmap(path, np.uint8, "r", RAW_HEADER.size, (self.n_frames, h, w, 3))

    def __len__(self) -> int:
        return self.n_frames

    def batch(self, start: int, count: int) -> np.ndarray:
        return self._mm[start:start + count]

    def batches(self, size: int):
        for s in range(0, self.n_frames, size):
            yield s, self._mm[s:s + size]


def model_bytes(model: BackgroundModel) -> bytes:
    buf = io.BytesIO()
    save_background(buf, model)
    return buf.getvalue()


# ---- PGM / PPM debug dumps ("Mask debug dump: binary PGM (P5),
# 0 -> 0, 1 -> 255. Frame dump: binary PPM (P6)"; "Debug flag emits
# per-stage masks as PGM files named <frame#>_{r1,r2,r3,merged,final}.pgm").

DUMP_STAGES = ("r1", "r2", "r3", "merged", "final")


def write_pgm(dst, mask: np.ndarray) -> None:
    """Write an (H, W) {0,1} mask as binary PGM (P5, maxval 255): 0 -> 0, 1 -> 255."""
    m = np.asarray(mask)
    if m.ndim != 2:
        raise ValueError("mask must be (H, W)")
    if m.size and (m.min() < 0 or m.max() > 1):
        raise ValueError("mask values must be 0 or 1")
    body = (m.astype(np.uint8) * np.uint8(255)).tobytes()
    f, own = _open(dst, "wb")
    try:
        f.write(b"P5\n%d %d\n255\n" % (m.shape[1], m.shape[0]))
        f.write(body)
    finally:
        if own:
            f.close()


def write_ppm(dst, frame: np.ndarray) -> None:
    """Write an (H, W, 3) u8 interleaved-RGB frame as binary PPM (P6, maxval 255)."""
    fr = np.ascontiguousarray(frame, np.uint8)
    if fr.ndim != 3 or fr.shape[2] != 3:
        raise ValueError("frame must be (H, W, 3) uint8")
    f, own = _open(dst, "wb")
    try:
        f.write(b"P6\n%d %d\n255\n" % (fr.shape[1], fr.shape[0]))
        f.write(fr.tobytes())
    finally:
        if own:
            f.close()


def read_pnm(src) -> np.ndarray:
    """Read a binary P5 / P6 file (maxval 255) written by write_pgm / write_ppm:
    (H, W) u8 for P5, (H, W, 3) u8 for P6 (raw values, no 255 -> 1 mapping)."""
    f, own = _open(src, "rb")
    try:
        data = f.read()
    finally:
        if own:
            f.close()
    toks, pos = [], 0
    while len(toks) < 4:
        while pos < len(data) and data[pos:pos + 1].isspace():
            pos += 1
        if pos < len(data) and data[pos:pos + 1] == b"#":
            while pos < len(data) and data[pos:pos + 1] != b"\n":
                pos += 1
            continue
        start = pos
        while pos < len(data) and not data[pos:pos + 1].isspace():
            pos += 1
        if start == pos:
            raise FormatError(f"truncated PNM header (at byte offset {pos})")
        toks.append(data[start:pos])
    pos += 1                                      # the single whitespace before the raster
    magic = toks[0]
    if magic not in (b"P5", b"P6"):
        raise FormatError(f"bad magic {magic!r} at byte offset 0 (expected b'P5' or b'P6')")
    w, h, maxval = (int(t) for t in toks[1:])
    if maxval != 255:
        raise FormatError(f"maxval {maxval} unsupported (expected 255)")
    ch = 1 if magic == b"P5" else 3
    need = w * h * ch
    if len(data) - pos != need:
        raise FormatError(f"raster of {len(data) - pos} bytes at byte offset {pos}, expected {need}")
    a = np.frombuffer(data, np.uint8, need, pos)
    return a.reshape(h, w).copy() if ch == 1 else a.reshape(h, w, 3).copy()


def dump_stages(directory, frame_no: int, stages: dict) -> list:
    """Write `stages` ({name: (H, W) {0,1} array}, names from DUMP_STAGES) as
    <frame_no>_<name>.pgm under `directory`; returns the paths."""
    os.makedirs(directory, exist_ok=True)
    paths = []
    for name in DUMP_STAGES:
        if name in stages:
            p = os.path.join(directory, f"{frame_no}_{name}.pgm")
            write_pgm(p, np.asarray(stages[name]))
            paths.append(p)
    return paths
