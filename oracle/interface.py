"""Oracle of NEXT-3, the interface hit-test (TEST INFRASTRUCTURE ONLY; shares
no code with the CUDA path).

SPEC S:322-351 (paper §2, "determines the interface zone activated by
the pointer"), one call per frame and stream, zones independent (all
containing zones receive events, in document order):
  membership: the pointer must be visible (reading L34); rectangles
    (button, slider) inclusive of their edges: x <= px <= x + w and
    y <= py <= y + h; wheels by squared distance: dx^2 + dy^2 <= r^2;
  enter iff member now and not before; leave iff member before and not now;
  click iff member and the pointer clicked this frame;
  slider value = clamp(1 - (py - y) / h, 0, 1), wheel value = the drive
    module's steering for a wheel of this centre / radius / theta_max with
    the default annulus and dead zone (reading L35); emitted as
    value_changed when the zone is a member, the value exists, and it is
    the zone's first value or differs from the last emitted one by >= 0.01.
"""
from __future__ import annotations

from dataclasses import dataclass

from .drive import Wheel, steering_from_cursor

BUTTON, SLIDER, WHEEL = 0, 1, 2
ENTER, LEAVE, CLICK, VALUE = 1, 2, 4, 8


@dataclass
class Zone:
    kind: int
    x: float = 0.0
    y: float = 0.0
    w: float = 0.0
    h: float = 0.0
    cx: float = 0.0
    cy: float = 0.0
    r: float = 0.0
    theta_max: float = 90.0


class HitTest:
    def __init__(self, zones):
        self.zones = list(zones)
        self.inside = [False] * len(self.zones)
        self.last = [None] * len(self.zones)

    def update(self, visible: bool, clicked: bool, px: float, py: float):
        """Returns [(inside, events, value)] per zone for this frame."""
        out = []
        for k, z in enumerate(self.zones):
            if not visible:
                member = False
            elif z.kind == WHEEL:
                dx, dy = px - z.cx, py - z.cy
                member = dx * dx + dy * dy <= z.r * z.r
            else:
                member = z.x <= px <= z.x + z.w and z.y <= py <= z.y + z.h
            ev = 0
            if member and not self.inside[k]:
                ev |= ENTER
            if not member and self.inside[k]:
                ev |= LEAVE
            if member and clicked:
                ev |= CLICK
            value = 0.0
            if member:
                v = None
                if z.kind == SLIDER:
                    v = min(1.0, max(0.0, 1.0 - (py - z.y) / z.h))
                elif z.kind == WHEEL:
                    v = steering_from_cursor(True, px, py, Wheel(z.cx, z.cy, z.r, z.theta_max))
                if v is not None and (self.last[k] is None or abs(v - self.last[k]) >= 0.01):
                    ev |= VALUE
                    value = v
                    self.last[k] = v
            self.inside[k] = member
            out.append((member, ev, value))
        return out
