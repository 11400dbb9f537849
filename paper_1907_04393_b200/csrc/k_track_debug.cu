// k_track_debug.cu -- K7 (the Mouse fold, a8) and the parity/debug stage
// kernels behind fizi_debug_stage.
//
// a8: §2, "This hand zone is converted into a pointer by the
// Mouse module ... its movement, its state (click or not)"; reading L25-L27
// (S:290-298): EMA with beta, snap on acquisition, visibility timeout (strict
// >), dwell anchor / radius / time, one click per dwell episode.  Sequential
// per stream (the only cross-frame dependency of the path); each product and
// sum is a separate correctly-rounded IEEE operation (__dmul_rn/__dadd_rn):
// no FMA contraction.
#include "fizi_internal.cuh"
#include "track.cuh"

namespace fizi {

// One stream: the inputs of up to kTrackChunk records are staged in shared
// memory by the whole block, one thread folds them, the block writes back.
constexpr int kTrackChunk = 512;

__global__ void __launch_bounds__(256) track_stream_kernel(fizi_params p, uint32_t n,
                                                           fizi_result* __restrict__ res,
                                                           TrackState* __restrict__ ts) {
  __shared__ int64_t t_s[kTrackChunk];
  __shared__ double cx_s[kTrackChunk], cy_s[kTrackChunk];
  __shared__ uint32_t ar_s[kTrackChunk];
  __shared__ uint32_t fl_s[kTrackChunk];
  __shared__ int64_t dw_o[kTrackChunk];
  __shared__ double px_o[kTrackChunk], py_o[kTrackChunk];
  __shared__ uint8_t vc_o[kTrackChunk];
  TrackState st;
  if (threadIdx.x == 0) st = *ts;
  for (uint32_t base = 0; base < n; base += kTrackChunk) {
    const uint32_t m = min((uint32_t)kTrackChunk, n - base);
    for (uint32_t i = threadIdx.x; i < m; i += blockDim.x) {
      const fizi_result& r = res[base + i];
      t_s[i] = r.t_ms; ar_s[i] = r.blob_area; cx_s[i] = r.cx; cy_s[i] = r.cy; fl_s[i] = r.relearn;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      // the next record's inputs are loaded before the current fold step
      // (separate output arrays: no aliasing between the two)
      int64_t t_n = t_s[0];
      uint32_t a_n = ar_s[0], l_n = fl_s[0];
      double x_n = cx_s[0], y_n = cy_s[0];
      for (uint32_t i = 0; i < m; i++) {
        fizi_result r;
        r.t_ms = t_n; r.blob_area = a_n; r.cx = x_n; r.cy = y_n; r.relearn = l_n;
        if (i + 1 < m) {
          t_n = t_s[i + 1]; a_n = ar_s[i + 1]; x_n = cx_s[i + 1]; y_n = cy_s[i + 1]; l_n = fl_s[i + 1];
        }
        track_one(p, st, r);
        dw_o[i] = r.dwell_ms; px_o[i] = r.px; py_o[i] = r.py;
        vc_o[i] = (uint8_t)(r.visible | (r.clicked << 1));
      }
    }
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < m; i += blockDim.x) {
      fizi_result& r = res[base + i];
      r.visible = vc_o[i] & 1u;
      r.clicked = vc_o[i] >> 1;
      r.px = px_o[i];
      r.py = py_o[i];
      r.dwell_ms = dw_o[i];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) *ts = st;
}

// ----------------------------------------------------- NEXT-1 relearn trigger
// relearn_trigger(prev, cur, threshold) = |cur - prev| > threshold
// over the stream's frames in order; one thread.
__global__ void relearn_kernel(int32_t* prev_mean, const fizi_result* __restrict__ res, uint32_t n,
                               int32_t threshold, uint8_t* __restrict__ flags) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  int32_t prev = *prev_mean;
  for (uint32_t i = 0; i < n; i++) {
    const int32_t cur = res[i].mean_luma;
    flags[i] = (prev >= 0 && abs(cur - prev) > threshold) ? 1u : 0u;
    prev = cur;
  }
  *prev_mean = prev;
}

__global__ void relearn_reset_kernel(int32_t* prev_mean, uint32_t count) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < count) prev_mean[i] = -1;
}

cudaError_t launch_relearn_flags(Ctx& c, uint32_t stream, const fizi_result* res, uint32_t n,
                                 uint32_t threshold, uint8_t* flags, cudaStream_t st) {
  relearn_kernel<<<1, 32, 0, st>>>(c.prev_mean + stream, res, n, (int32_t)threshold, flags);
  c.launches += 1;
  return cudaGetLastError();
}

cudaError_t launch_relearn_reset(Ctx& c, uint32_t first, uint32_t count, cudaStream_t st) {
  relearn_reset_kernel<<<(count + 255) / 256, 256, 0, st>>>(c.prev_mean + first, count);
  c.launches += 1;
  return cudaGetLastError();
}

// ---------------------------------------------------- NEXT-3 interface hit-test
// One thread per zone, frames in order (zones are independent; S:350 all
// containing zones receive events).  Membership needs a visible pointer;
// rectangles have inclusive edges, circles use squared distance <= r^2.
__device__ __forceinline__ bool wheel_steering(const fizi_zone& z, double px, double py,
                                               double& steering);

__global__ void hit_test_kernel(HitState* hs, const fizi_result* __restrict__ res, uint32_t n,
                                fizi_zone_event* __restrict__ out) {
  const uint32_t nz = hs->n_zones;
  const uint32_t k = threadIdx.x;
  if (k >= nz) return;
  const fizi_zone z = hs->zones[k];
  bool inside = hs->inside[k] != 0, has_value = hs->has_value[k] != 0;
  double last = hs->last_value[k];
  for (uint32_t i = 0; i < n; i++) {
    const fizi_result& r = res[i];
    const bool vis = r.visible != 0;
    const double px = r.px, py = r.py;
    bool in = false;
    if (vis) {
      if (z.kind == FIZI_ZONE_WHEEL) {
        const double dx = __dadd_rn(px, -z.cx), dy = __dadd_rn(py, -z.cy);
        in = __dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)) <= __dmul_rn(z.r, z.r);
      } else {
        in = px >= z.x && px <= __dadd_rn(z.x, z.w) && py >= z.y && py <= __dadd_rn(z.y, z.h);
      }
    }
    uint8_t ev = 0;
    if (in && !inside) ev |= FIZI_EV_ENTER;
    if (!in && inside) ev |= FIZI_EV_LEAVE;
    if (in && r.clicked) ev |= FIZI_EV_CLICK;
    double value = 0.0;
    if (in) {
      double v = 0.0;
      bool have = false;
      if (z.kind == FIZI_ZONE_SLIDER) {
        v = fmin(1.0, fmax(0.0, __dadd_rn(1.0, -__ddiv_rn(__dadd_rn(py, -z.y), z.h))));
        have = true;
      } else if (z.kind == FIZI_ZONE_WHEEL) {
        have = wheel_steering(z, px, py, v);
      }
      if (have && (!has_value || fabs(__dadd_rn(v, -last)) >= 0.01)) {
        ev |= FIZI_EV_VALUE;
        value = v;
        last = v;
        has_value = true;
      }
    }
    inside = in;
    fizi_zone_event e;
    e.inside = in ? 1u : 0u;
    e.events = ev;
    for (int j = 0; j < 6; j++) e._pad[j] = 0;
    e.value = value;
    out[(uint64_t)i * nz + k] = e;
  }
  hs->inside[k] = inside ? 1u : 0u;
  hs->has_value[k] = has_value ? 1u : 0u;
  hs->last_value[k] = last;
}

cudaError_t launch_hit_test(Ctx& c, uint32_t stream, const fizi_result* res, uint32_t n,
                            fizi_zone_event* out, cudaStream_t st) {
  hit_test_kernel<<<1, kMaxZones, 0, st>>>(reinterpret_cast<HitState*>(c.hstate) + stream, res, n,
                                           out);
  c.launches += 1;
  return cudaGetLastError();
}

// ------------------------------------------------------ NEXT-2 drive mapping
// steering_from_cursor and the make_command fold for
// one stream, in frame order, one thread.  Every product / sum is a separate
// correctly rounded operation (no FMA contraction); the angle is atan2 in
// double, converted to degrees with the factor 180/pi.
__device__ __forceinline__ bool steering_from_cursor(const fizi_wheel& w, bool visible, double px,
                                                     double py, double& steering) {
  if (!visible) return false;
  const double dx = __dadd_rn(px, -w.cx), dy = __dadd_rn(py, -w.cy);
  const double d = __dsqrt_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)));
  if (d < __dmul_rn(w.inner, w.radius) || d > __dmul_rn(w.outer, w.radius)) return false;
  double theta = __dmul_rn(atan2(dx, -dy), 57.29577951308232);   // 12 o'clock 0, clockwise > 0
  if (theta == -180.0) theta = 180.0;                              // (-180, 180]
  if (fabs(theta) <= w.dead_zone_deg) { steering = 0.0; return true; }
  steering = fmin(1.0, fmax(-1.0, __ddiv_rn(theta, w.theta_max_deg)));
  return true;
}

// a wheel zone steers like a wheel of the drive module with the default
// annulus and dead zone (reading L35)
__device__ __forceinline__ bool wheel_steering(const fizi_zone& z, double px, double py,
                                               double& steering) {
  fizi_wheel w;
  w.cx = z.cx; w.cy = z.cy; w.radius = z.r; w.theta_max_deg = z.theta_max_deg;
  w.inner = 0.6; w.outer = 1.4; w.dead_zone_deg = 3.0; w.hold_ms = 200;
  return steering_from_cursor(w, true, px, py, steering);
}

// ev == nullptr: no throttle source (make_command's slider_throttle_opt is
// always absent).  Else the slider value of frame i is ev[i * nz + zi].value
// when that event carries FIZI_EV_VALUE (fizi_hit_test's output, L36).
__global__ void drive_kernel(DriveState* ds, const fizi_result* __restrict__ res, uint32_t n,
                             const fizi_zone_event* __restrict__ ev, uint32_t nz, uint32_t zi,
                             fizi_command* __restrict__ out) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  DriveState s = *ds;
  for (uint32_t i = 0; i < n; i++) {
    const fizi_result& r = res[i];
    const int64_t t = r.t_ms;
    double st = 0.0;
    const bool on = steering_from_cursor(s.wheel, r.visible != 0, r.px, r.py, st);
    if (on) {
      s.last_reading = t;
      s.has_reading = 1;
    } else {
      st = s.steering;
      if (!s.has_reading || t - s.last_reading > s.wheel.hold_ms) st = __dmul_rn(st, 0.8);
    }
    s.steering = fmin(1.0, fmax(-1.0, st));
    if (ev != nullptr) {
      const fizi_zone_event& e = ev[(size_t)i * nz + zi];
      if (e.events & FIZI_EV_VALUE) s.throttle = e.value;
    }
    s.throttle = fmin(1.0, fmax(0.0, s.throttle));
    fizi_command c;
    c.steering = s.steering;
    c.throttle = s.throttle;
    c.t_ms = t;
    c.has_steering = on ? 1u : 0u;
    c._pad = 0;
    out[i] = c;
  }
  *ds = s;
}

__global__ void drive_set_kernel(DriveState* ds, fizi_wheel w) {
  DriveState s;
  s.steering = 0.0;
  s.throttle = 0.0;
  s.last_reading = 0;
  s.has_reading = 0;
  s.has_wheel = 1;
  s.wheel = w;
  *ds = s;
}

cudaError_t launch_drive_set(Ctx& c, uint32_t stream, const fizi_wheel& w, cudaStream_t st) {
  drive_set_kernel<<<1, 1, 0, st>>>(reinterpret_cast<DriveState*>(c.dstate) + stream, w);
  c.launches += 1;
  return cudaGetLastError();
}

cudaError_t launch_drive(Ctx& c, uint32_t stream, const fizi_result* res, uint32_t n,
                         const fizi_zone_event* ev, uint32_t nz, uint32_t zi, fizi_command* out,
                         cudaStream_t st) {
  drive_kernel<<<1, 32, 0, st>>>(reinterpret_cast<DriveState*>(c.dstate) + stream, res, n, ev, nz,
                                 zi, out);
  c.launches += 1;
  return cudaGetLastError();
}

__global__ void tstate_reset_kernel(TrackState* ts, uint32_t count) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < count) {
    TrackState z;
    z.vis = 0; z.fired = 0;
    z.px = z.py = z.ax = z.ay = 0.0;
    z.last_t = z.anchor_t = z.dwell = 0;
    ts[i] = z;
  }
}


cudaError_t launch_track_stream(Ctx& c, uint32_t stream, fizi_result* res, uint32_t n,
                                cudaStream_t st) {
  track_stream_kernel<<<1, 256, 0, st>>>(c.p, n, res, reinterpret_cast<TrackState*>(c.tstate) + stream);
  c.launches += 1;
  return cudaGetLastError();
}

// fizi_track_runs: the records of up to kMaxRuns runs of consecutive rows,
// folded run after run (rows of a window gathered from several ranks, in
// frame order).  Inputs are staged run by run through the same chunked
// shared-memory scheme as track_stream_kernel; the fold order is the
// concatenation of the runs.
struct TrackRuns {
  uint32_t n_runs;
  uint32_t off[kMaxTrackRuns], len[kMaxTrackRuns];
};

__global__ void __launch_bounds__(256) track_runs_kernel(fizi_params p, TrackRuns runs,
                                                         fizi_result* __restrict__ res,
                                                         TrackState* __restrict__ ts) {
  __shared__ int64_t t_s[kTrackChunk];
  __shared__ double cx_s[kTrackChunk], cy_s[kTrackChunk];
  __shared__ uint32_t ar_s[kTrackChunk];
  __shared__ uint32_t fl_s[kTrackChunk];
  __shared__ int64_t dw_o[kTrackChunk];
  __shared__ double px_o[kTrackChunk], py_o[kTrackChunk];
  __shared__ uint8_t vc_o[kTrackChunk];
  TrackState st;
  if (threadIdx.x == 0) st = *ts;
  for (uint32_t k = 0; k < runs.n_runs; k++) {
    fizi_result* rr = res + runs.off[k];
    const uint32_t n = runs.len[k];
    for (uint32_t base = 0; base < n; base += kTrackChunk) {
      const uint32_t m = min((uint32_t)kTrackChunk, n - base);
      for (uint32_t i = threadIdx.x; i < m; i += blockDim.x) {
        const fizi_result& r = rr[base + i];
        t_s[i] = r.t_ms; ar_s[i] = r.blob_area; cx_s[i] = r.cx; cy_s[i] = r.cy; fl_s[i] = r.relearn;
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        int64_t t_n = t_s[0];
        uint32_t a_n = ar_s[0], l_n = fl_s[0];
        double x_n = cx_s[0], y_n = cy_s[0];
        for (uint32_t i = 0; i < m; i++) {
          fizi_result r;
          r.t_ms = t_n; r.blob_area = a_n; r.cx = x_n; r.cy = y_n; r.relearn = l_n;
          if (i + 1 < m) {
          t_n = t_s[i + 1]; a_n = ar_s[i + 1]; x_n = cx_s[i + 1]; y_n = cy_s[i + 1]; l_n = fl_s[i + 1];
        }
          track_one(p, st, r);
          dw_o[i] = r.dwell_ms; px_o[i] = r.px; py_o[i] = r.py;
          vc_o[i] = (uint8_t)(r.visible | (r.clicked << 1));
        }
      }
      __syncthreads();
      for (uint32_t i = threadIdx.x; i < m; i += blockDim.x) {
        fizi_result& r = rr[base + i];
        r.visible = vc_o[i] & 1u;
        r.clicked = vc_o[i] >> 1;
        r.px = px_o[i];
        r.py = py_o[i];
        r.dwell_ms = dw_o[i];
      }
      __syncthreads();
    }
  }
  if (threadIdx.x == 0) *ts = st;
}

cudaError_t launch_track_runs(Ctx& c, uint32_t stream, fizi_result* res, const uint32_t* off,
                              const uint32_t* len, uint32_t n_runs, cudaStream_t st) {
  TrackRuns r;
  r.n_runs = n_runs;
  for (uint32_t k = 0; k < n_runs; k++) { r.off[k] = off[k]; r.len[k] = len[k]; }
  track_runs_kernel<<<1, 256, 0, st>>>(c.p, r, res, reinterpret_cast<TrackState*>(c.tstate) + stream);
  c.launches += 1;
  return cudaGetLastError();
}

cudaError_t launch_tstate_reset(Ctx& c, uint32_t first, uint32_t count, cudaStream_t st) {
  tstate_reset_kernel<<<(count + 255) / 256, 256, 0, st>>>(
      reinterpret_cast<TrackState*>(c.tstate) + first, count);
  c.launches += 1;
  return cudaGetLastError();
}

// ------------------------------------------------------------- debug stages
// R1/R2/R3 recomputed per pixel from the last call's frames with the frame's
// LUT; masks expanded from the bit planes; labels painted from the runs.
__global__ void debug_branch_kernel(const uint8_t* __restrict__ frame, uint64_t N,
                                    const uint8_t* __restrict__ env_lo,
                                    const uint8_t* __restrict__ env_hi, bool fast,
                                    const uint8_t* __restrict__ L, int stage, int S, int a1,
                                    int a2, uint8_t* __restrict__ out) {
  const uint64_t q = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (q >= N) return;
  const int v[3] = {L[frame[3 * q]], L[frame[3 * q + 1]], L[frame[3 * q + 2]]};
  uint8_t o = 0;
  if (stage == FIZI_STAGE_R1) {
    bool inside = true;
    for (int ch = 0; ch < 3; ch++) {
      const uint64_t e = env_perm_index(3 * q + ch, fast);
      inside = inside && v[ch] >= env_lo[e] && v[ch] <= env_hi[e];
    }
    o = !inside;
  } else {
    const int M = max(v[0], max(v[1], v[2])), m = min(v[0], min(v[1], v[2])), C = M - m;
    if (stage == FIZI_STAGE_R2) {
      o = C >= S;
    } else {
      int d, base;
      if (M == v[0]) { d = v[1] - v[2]; base = v[1] < v[2] ? 360 : 0; }
      else if (M == v[1]) { d = v[2] - v[0]; base = 120; }
      else { d = v[0] - v[1]; base = 240; }
      const int Hn = 60 * d + base * C, lo = a1 * C, hi = a2 * C;
      const bool band = (a1 <= a2) ? (Hn >= lo && Hn <= hi) : (Hn >= lo || Hn <= hi);
      o = (C > 0) && band;
    }
  }
  out[q] = o;
}

__global__ void debug_labels_kernel(const Run* __restrict__ runs, const uint32_t* __restrict__ parent,
                                    const uint32_t* __restrict__ frame_runs, uint32_t W,
                                    uint32_t* __restrict__ out) {
  const uint32_t T = *frame_runs;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < T; i += gridDim.x * blockDim.x) {
    const Run rg = runs[i];
    const Run rr = runs[parent[i]];
    const uint32_t label = 1u + (uint32_t)rr.y * W + rr.x0;
    for (uint32_t x = rg.x0; x <= rg.x1; x++) out[(uint64_t)rg.y * W + x] = label;
  }
}

__global__ void debug_contour_kernel(const uint32_t* __restrict__ F, uint32_t W, uint32_t H,
                                     uint32_t P, uint8_t* __restrict__ out) {
  const uint64_t q = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (q >= (uint64_t)W * H) return;
  const int x = (int)(q % W), y = (int)(q / W);
  auto bit = [&](int xx, int yy) -> uint32_t {
    if (xx < 0 || yy < 0 || xx >= (int)W || yy >= (int)H) return 0u;
    return (F[(uint64_t)yy * P + (xx >> 5)] >> (xx & 31)) & 1u;
  };
  const uint32_t c = bit(x, y);
  uint32_t all = 1;
  for (int dy = -1; dy <= 1; dy++)
    for (int dx = -1; dx <= 1; dx++) all &= bit(x + dx, y + dy);
  out[q] = (uint8_t)(c & (all ^ 1u));
}

cudaError_t launch_expand_from(Ctx& c, const uint32_t* bits, uint32_t n, uint8_t* masks,
                               cudaStream_t st);

cudaError_t launch_debug_stage(Ctx& c, int stage, uint32_t f, void* out, cudaStream_t st) {
  const uint64_t wpf = (uint64_t)c.H * c.P;
  const unsigned blocks = (unsigned)((c.N + 255) / 256);
  switch (stage) {
    case FIZI_STAGE_R1:
    case FIZI_STAGE_R2:
    case FIZI_STAGE_R3: {
      // the frame's LUT row: recompute the mean from the luma sum of the call
      unsigned long long sum = 0;
      cudaMemcpyAsync(&sum, c.luma + f, sizeof(sum), cudaMemcpyDeviceToHost, st);
      uint32_t s = 0;
      cudaMemcpyAsync(&s, c.frame_stream + f, sizeof(s), cudaMemcpyDeviceToHost, st);
      cudaStreamSynchronize(st);
      const uint64_t mean = (sum + 500ull * c.N) / (1000ull * c.N);
      const uint8_t* lo = c.env + (uint64_t)s * 2 * c.env_plane;
      debug_branch_kernel<<<blocks, 256, 0, st>>>(c.last_frames + (uint64_t)f * c.N * 3, c.N, lo,
                                                  lo + c.env_plane, c.fast, c.lut + mean * 256,
                                                  stage, (int)c.p.gray_tol_S, (int)c.p.hue_lo_deg,
                                                  (int)c.p.hue_hi_deg, (uint8_t*)out);
      c.launches += 1;
      return cudaGetLastError();
    }
    case FIZI_STAGE_MERGED:
      return launch_expand_from(c, c.bitA + f * wpf, 1, (uint8_t*)out, st);
    case FIZI_STAGE_OPENCLOSE:
      return launch_expand_from(c, c.bitOC + f * wpf, 1, (uint8_t*)out, st);
    case FIZI_STAGE_FINAL:
      return launch_expand_from(c, c.bitO + f * wpf, 1, (uint8_t*)out, st);
    case FIZI_STAGE_LABELS: {
      cudaMemsetAsync(out, 0, c.N * sizeof(uint32_t), st);
      debug_labels_kernel<<<256, 256, 0, st>>>(c.runs + (uint64_t)f * c.cap_runs,
                                               c.parent + (uint64_t)f * c.cap_runs,
                                               c.frame_runs + f, c.W, (uint32_t*)out);
      c.launches += 1;
      return cudaGetLastError();
    }
    case FIZI_STAGE_CONTOUR:
      debug_contour_kernel<<<blocks, 256, 0, st>>>(c.bitO + f * wpf, c.W, c.H, c.P, (uint8_t*)out);
      c.launches += 1;
      return cudaGetLastError();
    default:
      return cudaErrorInvalidValue;
  }
}

}  // namespace fizi
