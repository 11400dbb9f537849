"""Oracle of NEXT-2, the drive mapping (TEST INFRASTRUCTURE ONLY: only tests/,
__graft_entry__.smoke() and bench.py's CPU baseline may import it; it shares
no code with the CUDA path).

Follows SPEC module `drive`, the paper's §4 driving application
("a rotation around an imaginary wheel"), step by step in scalar
Python floats (IEEE double), one call per frame:

  steering_from_cursor: none when the cursor is invisible or its
  radial distance d from the wheel centre is outside [inner·R, outer·R]
  (bounds inclusive, reading L32); else θ = signed angle of (cursor − centre)
  from the 12-o'clock direction, clockwise positive, in (−180, 180] degrees
  (image y grows downwards, so 12 o'clock is −y and 3 o'clock is +x);
  |θ| ≤ dead_zone ⇒ 0, else clamp(θ / theta_max, −1, 1).

  make_command: steering = the new value when present; else the
  previous steering, multiplied by 0.8 on every frame whose time since the
  last reading exceeds hold_ms (strict >, reading L33; no reading yet counts
  as exceeded); throttle = the slider value when present, else the previous
  throttle (no slider source without NEXT-3: always the previous, 0 at
  start); both clamped to their ranges.  The first frame with nothing
  present gives (0, 0).

Parity pins (tests/test_drive.py): the SPEC's examples (S:392-394,
S:401-403), the stated properties (odd symmetry, ranges, purity),
closed forms on the rim.
"""
from __future__ import annotations

import math
from dataclasses import dataclass


@dataclass
class Wheel:
    cx: float
    cy: float
    radius: float
    theta_max: float = 90.0       # degrees, (0, 180]
    inner: float = 0.6            # annulus, fractions of the radius
    outer: float = 1.4
    dead_zone: float = 3.0        # degrees
    hold_ms: int = 200


def steering_from_cursor(visible: bool, px: float, py: float, w: Wheel):
    """S:389-394; returns None or a steering value in [-1, 1]."""
    if not visible:
        return None
    dx = px - w.cx
    dy = py - w.cy
    d = math.sqrt(dx * dx + dy * dy)
    if d < w.inner * w.radius or d > w.outer * w.radius:
        return None
    theta = math.degrees(math.atan2(dx, -dy))       # 12 o'clock = 0, clockwise > 0
    if theta == -180.0:
        theta = 180.0                               # range (-180, 180]
    if abs(theta) <= w.dead_zone:
        return 0.0
    return max(-1.0, min(1.0, theta / w.theta_max))


@dataclass
class Command:
    steering: float = 0.0
    throttle: float = 0.0
    t_ms: int = 0
    has_steering: bool = False


class Drive:
    """make_command folded over the frames of one stream."""

    def __init__(self, wheel: Wheel):
        self.wheel = wheel
        self.prev = Command()
        self.last_reading = None                    # t_ms of the last steering reading

    def update(self, visible: bool, px: float, py: float, t_ms: int,
               throttle_opt: float | None = None) -> Command:
        s = steering_from_cursor(visible, px, py, self.wheel)
        if s is not None:
            steering = s
            self.last_reading = t_ms
        else:
            steering = self.prev.steering
            if self.last_reading is None or t_ms - self.last_reading > self.wheel.hold_ms:
                steering = steering * 0.8
        throttle = self.prev.throttle if throttle_opt is None else throttle_opt
        steering = max(-1.0, min(1.0, steering))
        throttle = max(0.0, min(1.0, throttle))
        self.prev = Command(steering, throttle, t_ms, s is not None)
        return self.prev
