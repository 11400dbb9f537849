"""Input helpers shared by tests (no method arithmetic)."""
import numpy as np

BG = (100, 100, 100)     # gray background: inside its own envelope, R2 = 0
SKIN = (210, 120, 110)   # skin: outside the gray envelope, C = 100 >= S, hue 6 deg


def mask_frames(masks: np.ndarray):
    """Frames whose merged mask A equals `masks` (n,h,w) under default params.

    Returns (frames (n,h,w,3), lo, hi) with a margin-10 envelope around the
    constant gray background; every frame's mean luma lies in [100, 146], so
    no brightness correction applies.
    """
    masks = np.asarray(masks, bool)
    n, h, w = masks.shape
    frames = np.empty((n, h, w, 3), np.uint8)
    frames[:] = BG
    frames[masks] = SKIN
    lo = np.full((h, w, 3), BG[0] - 10, np.uint8)
    hi = np.full((h, w, 3), BG[0] + 10, np.uint8)
    return frames, lo, hi


def all_masks(h: int, w: int) -> np.ndarray:
    """Every binary h x w mask, (2**(h*w), h, w) u8, bit i = raster pixel i."""
    n = h * w
    idx = np.arange(2 ** n, dtype=np.int64)
    bits = (idx[:, None] >> np.arange(n)[None, :]) & 1
    return bits.reshape(-1, h, w).astype(np.uint8)
