// track.cuh -- a8, the Mouse fold for one record (shared by the fold kernels
// and the fused labelling kernel).
//
// §2, "This hand zone is converted into a pointer by the
// Mouse module ... its movement, its state (click or not)"; readings L25-L27
// (S:290-298): EMA with beta, snap on acquisition, visibility timeout (strict
// >), dwell anchor / radius / time, one click per dwell episode.  Each product
// and sum is a separate correctly-rounded IEEE operation: no FMA contraction.
#pragma once

#include "fizi_internal.cuh"

namespace fizi {

__device__ __forceinline__ void track_reset(TrackState& s) {
  s.vis = 0; s.fired = 0;
  s.px = s.py = s.ax = s.ay = 0.0;
  s.last_t = s.anchor_t = s.dwell = 0;
}

// r.relearn (NEXT-1, reading L37): a learning frame is not tracked (the state
// is untouched, the pointer outputs are zero); after the last learning frame
// (the model swap) the state restarts from its initial value.
__device__ __forceinline__ void track_one(const fizi_params& p, TrackState& s, fizi_result& r) {
  if (r.relearn & FIZI_RELEARN_LEARN) {
    r.visible = 0; r.clicked = 0;
    r.px = 0.0; r.py = 0.0; r.dwell_ms = 0;
    if (r.relearn & FIZI_RELEARN_SWAP) track_reset(s);
    return;
  }
  const int64_t t = r.t_ms;
  if (r.blob_area > 0) {
    if (s.vis) {
      const double b = p.beta, ob = __dadd_rn(1.0, -p.beta);
      s.px = __dadd_rn(__dmul_rn(b, r.cx), __dmul_rn(ob, s.px));
      s.py = __dadd_rn(__dmul_rn(b, r.cy), __dmul_rn(ob, s.py));
      const double dx = __dadd_rn(s.px, -s.ax), dy = __dadd_rn(s.py, -s.ay);
      const double d2 = __dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy));
      const double R2 = __dmul_rn(p.dwell_radius_px, p.dwell_radius_px);
      if (d2 > R2) {
        s.ax = s.px; s.ay = s.py; s.anchor_t = t;
        s.dwell = 0; s.fired = 0;
      } else {
        s.dwell = t - s.anchor_t;
      }
    } else {
      s.px = r.cx; s.py = r.cy;
      s.ax = r.cx; s.ay = r.cy; s.anchor_t = t;
      s.dwell = 0; s.fired = 0;
    }
    s.vis = 1;
    s.last_t = t;
  } else {
    if (s.vis && t - s.last_t > p.lost_timeout_ms) {
      s.vis = 0; s.dwell = 0; s.fired = 0;
    } else if (s.vis) {
      s.dwell = t - s.anchor_t;
    }
  }
  const int clicked = s.vis && !s.fired && s.dwell >= p.dwell_time_ms;
  if (clicked) s.fired = 1;
  r.visible = (uint8_t)s.vis;
  r.clicked = (uint8_t)clicked;
  r.px = s.px;
  r.py = s.py;
  r.dwell_ms = s.dwell;
}


}  // namespace fizi
