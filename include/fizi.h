/*
 * include/fizi.h -- C ABI of libfizi.so, the B200 (sm_100a) implementation of
 * the per-frame FIZI + Mouse pixel path of arXiv 1907.04393.
 *
 * Citations: P:<n> = PAPER.md line n (/root/reference, read-only), S:<n> =
 * SPEC.md line n.  DESIGN.md lists every reading (L1..L31) of a passage that is
 * silent, garbled or contradictory.
 *
 * Conventions shared by every entry point
 *   - Return value: fizi_status (0 = FIZI_OK, < 0 = error).  No entry point
 *     throws, aborts or prints; fizi_last_error(ctx) describes the last error.
 *   - Device pointers ("_dev") are plain CUDA device addresses on the
 *     context's device (e.g. torch.Tensor.data_ptr()); host pointers ("_host")
 *     are ordinary (preferably pinned) host memory.  The caller owns every
 *     frame, mask and result buffer; the library owns envelopes, tracker
 *     states, the LUT table and all scratch, sized once at fizi_create.
 *   - Inputs are const and never modified.
 *   - Work is stream-ordered on the caller's CUDA stream (fizi_stream_t is a
 *     cudaStream_t; NULL = legacy default stream).  Outputs are valid once that
 *     stream is synchronised.  Calls on one context must be externally
 *     serialised (one logical consumer).
 *   - Frame layout (a0): row-major, top row first, interleaved
 *     (r,g,b) u8, tightly packed: frame i of a batch starts at byte
 *     i * width * height * 3.  Mask layout: u8 {0,1}, one byte per pixel,
 *     row-major, frame i at byte i * width * height.
 *   - A CUDA failure is sticky (FIZI_E_CUDA): the context must be destroyed.
 */
#ifndef FIZI_H
#define FIZI_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st *fizi_stream_t;   /* == cudaStream_t */
typedef struct fizi_ctx fizi_ctx;

typedef enum {
    FIZI_OK = 0,
    FIZI_E_ARG = -1,      /* parameter out of range or NULL pointer   */
    FIZI_E_EMPTY = -2,    /* learn with n_frames = 0: "empty sequence"          */
    FIZI_E_DIMS = -3,     /* width/height differ from the context       */
    FIZI_E_NOMODEL = -4,  /* process before fizi_learn_background for that stream       */
    FIZI_E_TIME = -5,     /* decreasing timestamps within a stream (pre of S:292)       */
    FIZI_E_CUDA = -6,     /* CUDA error (sticky)                                        */
    FIZI_E_OOM = -7,      /* device allocation failed at fizi_create                    */
    FIZI_E_CAPACITY = -8  /* batch larger than max_batch, or stream id >= n_streams     */
} fizi_status;

/* Immutable parameter snapshot.  Defaults (fizi_params_default):
 * S:187 segmentation, S:285 tracker, S:169 margin is passed to learn. */
typedef struct fizi_params {
    uint32_t width, height;        /* fixed per context; 1..65535                          */
    uint32_t gray_tol_S;           /* 30: keep iff max-min >= S (reading L5); <=255  */
    uint32_t hue_lo_deg;           /* 340: alpha_1 in degrees [0,360) (reading L7)  */
    uint32_t hue_hi_deg;           /* 25:  alpha_2; alpha_1 > alpha_2 = band through 0 deg */
    uint32_t se_radius;            /* 1: square SE side 2r+1; 1..8            */
    uint32_t min_blob_ppm;         /* 5000: drop components with area*1e6 < ppm*W*H (L13)  */
    uint32_t luma_target;          /* 128                                          */
    uint32_t luma_lo, luma_hi;     /* 60, 190: identity iff lo <= mean <= hi       */
    double   gamma_min, gamma_max; /* 0.4, 2.5; 0 < min <= max                    */
    double   beta;                 /* 0.5: EMA weight of the new centroid, [0,1]   */
    double   dwell_radius_px;      /* 15, >= 0                                     */
    int64_t  dwell_time_ms;        /* 800, >= 0                                    */
    int64_t  lost_timeout_ms;      /* 500, >= 0                                    */
    uint32_t debug;                /* 1 = keep per-stage state for fizi_debug_stage        */
    uint32_t _reserved;
} fizi_params;

/* One record per processed frame (128 bytes), written to device memory. */
typedef struct fizi_result {
    int64_t  t_ms;                 /* the caller's timestamp                               */
    uint32_t stream;               /* camera stream id                                     */
    uint32_t frame_idx;            /* index of the frame within its call                   */
    uint8_t  mean_luma;            /* a2: floor((sum Y + 500N)/(1000N)), Y = 299r+587g+114b */
    uint8_t  corrected;            /* 1 iff a non-identity gamma LUT was applied           */
    uint8_t  visible, clicked;     /* a8 (fizi_track / fizi_process_frames only)           */
    uint32_t fg_merged;            /* popcount of A = R1 & R2 & R3 (a3)                    */
    uint32_t fg_final;             /* popcount of the final mask (a6)                      */
    uint32_t n_comp_total;         /* 8-connected components of the open-close mask (a5)   */
    uint32_t n_comp_kept;          /* components passing the area filter (a6)              */
    uint32_t blob_area;            /* a7: largest kept component (0 if none)               */
    uint32_t blob_label;           /*     its label = 1 + min raster index y*W+x (L15)     */
    uint32_t bbox[4];              /*     x_min, y_min, x_max, y_max                       */
    uint32_t relearn;              /* NEXT-1 flags (fizi_set_relearn): 1 learning frame,    */
                                   /* 2 model swapped after it, 4 trigger; 0 otherwise      */
    uint64_t sum_x, sum_y;         /*     exact moments: sum of x (column), sum of y (row) */
    double   gamma;                /* a2: 1.0 when not corrected                           */
    double   cx, cy;               /* a7: centroid sum/area (L17); 0 if no blob            */
    double   px, py;               /* a8: smoothed pointer                                 */
    int64_t  dwell_ms;             /* a8: dwell time at the anchor                         */
} fizi_result;

enum { FIZI_RELEARN_LEARN = 1, FIZI_RELEARN_SWAP = 2, FIZI_RELEARN_TRIGGER = 4 };

/* Stages for fizi_debug_stage (SPEC S:265 stage dumps). */
typedef enum {
    FIZI_STAGE_R1 = 0,        /* I_R1 background branch, u8 {0,1}         */
    FIZI_STAGE_R2 = 1,        /* I_R2 gray branch         */
    FIZI_STAGE_R3 = 2,        /* I_R3 hue branch         */
    FIZI_STAGE_MERGED = 3,    /* A = R1 & R2 & R3         */
    FIZI_STAGE_OPENCLOSE = 4, /* O = E(D(D(E(A))))         */
    FIZI_STAGE_LABELS = 5,    /* u32 canonical labels of O, 0 = background (L15)        */
    FIZI_STAGE_FINAL = 6,     /* I_FIZI: O restricted to kept components        */
    FIZI_STAGE_CONTOUR = 7    /* inner boundary FINAL & !erode_1(FINAL) (L30)           */
} fizi_stage;

/* Fill *p with the defaults above for a width x height context. */
int fizi_params_default(fizi_params *p, uint32_t width, uint32_t height);

/* Create a context on CUDA device `cuda_device` for n_streams camera streams
 * (each with its own envelope and tracker state) and batches of at most
 * max_batch frames (<= 65535).  Validates params (FIZI_E_ARG), allocates all
 * device memory (FIZI_E_OOM) and builds the 256x256 gamma-LUT table on the
 * device.  *out is NULL on error. */
int fizi_create(const fizi_params *params, int cuda_device, uint32_t n_streams,
                uint32_t max_batch, fizi_ctx **out);

/* a1: learn stream `stream`'s envelope from n_frames
 * frames (device, frame layout above) -- per pixel and channel
 * lo = sat(min_k F_k - margin), hi = sat(max_k F_k + margin).  Replaces any
 * previous model and resets the stream's tracker.  n_frames = 0 ->
 * FIZI_E_EMPTY; width/height != context -> FIZI_E_DIMS. */
int fizi_learn_background(fizi_ctx *ctx, uint32_t stream, const uint8_t *frames_dev,
                          uint32_t n_frames, uint32_t width, uint32_t height,
                          uint8_t margin, fizi_stream_t cuda_stream);

/* The whole per-frame path (§3.1, §3.2) for a batch of n frames:
 * frame i belongs to stream stream_of_frame_host[i] and carries timestamp
 * t_ms_host[i] (both host arrays of n entries).  Frames of one stream are
 * processed in index order; timestamps must be non-decreasing per stream,
 * also across calls (FIZI_E_TIME).  Writes masks_dev (n*W*H u8 {0,1}, may be
 * NULL) and results_dev (n records).  = fizi_segment_frames + fizi_track. */
int fizi_process_frames(fizi_ctx *ctx, const uint32_t *stream_of_frame_host,
                        const uint8_t *frames_dev, uint32_t n, uint32_t width,
                        uint32_t height, const int64_t *t_ms_host, uint8_t *masks_dev,
                        fizi_result *results_dev, fizi_stream_t cuda_stream);

/* Stateless part a2..a7: like fizi_process_frames but leaves every stream's
 * tracker untouched and writes visible = clicked = 0, px = py = 0,
 * dwell_ms = 0 (for sharded multi-GPU runs, §8(e)); no timestamp check. */
int fizi_segment_frames(fizi_ctx *ctx, const uint32_t *stream_of_frame_host,
                        const uint8_t *frames_dev, uint32_t n, uint32_t width,
                        uint32_t height, const int64_t *t_ms_host, uint8_t *masks_dev,
                        fizi_result *results_dev, fizi_stream_t cuda_stream);

/* a8: fold n records of stream `stream`, in
 * order, through the stream's tracker state; reads t_ms, blob_area, cx, cy and
 * writes visible, clicked, px, py, dwell_ms in place.  Used after gathering
 * the records of a sharded stream. */
int fizi_track(fizi_ctx *ctx, uint32_t stream, fizi_result *results_dev, uint32_t n,
               fizi_stream_t cuda_stream);

/* a8 over records gathered from several ranks: folds, through stream
 * `stream`'s tracker state, the n_runs (<= 256) runs of consecutive records
 * results_dev[run_off[k] .. run_off[k] + run_len[k]) for k = 0 .. n_runs-1, in
 * that order (run_off / run_len: host arrays); = fizi_track on the
 * concatenation of the runs, in one launch.  FIZI_E_ARG if n_runs > 256. */
int fizi_track_runs(fizi_ctx *ctx, uint32_t stream, fizi_result *results_dev,
                    const uint32_t *run_off_host, const uint32_t *run_len_host, uint32_t n_runs,
                    fizi_stream_t cuda_stream);

/* End-to-end variant of fizi_process_frames on HOST buffers: copies frames
 * (n*W*H*3 bytes) host->device, runs the path, copies masks (may be NULL) and
 * results back device->host, all on cuda_stream; returns after the stream has
 * completed (results are valid on return). */
int fizi_process_frames_host(fizi_ctx *ctx, const uint32_t *stream_of_frame_host,
                             const uint8_t *frames_host, uint32_t n, uint32_t width,
                             uint32_t height, const int64_t *t_ms_host, uint8_t *masks_host,
                             fizi_result *results_host, fizi_stream_t cuda_stream);

/* Reset stream `stream`'s tracker to its initial state (invisible), in
 * cuda_stream order after every earlier call's fold (outstanding pipelined
 * tails are joined into cuda_stream first).  Timestamps of the stream may
 * restart from any value afterwards. */
int fizi_reset_tracker(fizi_ctx *ctx, uint32_t stream, fizi_stream_t cuda_stream);

/* ---- NEXT-1: relearn trigger ("re-initiate partly the machine
 * learning techniques" on a luminosity change).  Folds the
 * a2 mean luma of n records of stream `stream` (device), in order, through
 * the stream's trigger state and writes flags_dev[i] (device u8) = 1 iff
 * |mean_i - mean_prev| > threshold (strict; the first frame after a reset
 * has no previous mean and gives 0).  The caller re-learns the envelope from
 * later frames (fizi_learn_background swaps the model between calls, and
 * resets this state).  threshold <= 255. */
int fizi_relearn_flags(fizi_ctx *ctx, uint32_t stream, const fizi_result *results_dev, uint32_t n,
                       uint32_t threshold, uint8_t *flags_dev, fizi_stream_t cuda_stream);

/* ---- NEXT-1, in-stream relearning (§3.3; SPEC S:153-161, S:170
 * "on trigger, runtime pauses tracking and relearns", "Relearning swaps
 * the model atomically between frames"; reading L37).  With
 * n_frames > 0, every later call folds stream `stream`'s frames in order
 * through a relearn state: a frame whose a2 mean luma differs from the
 * previous frame's by more than `threshold` (strict) is processed normally
 * and flagged FIZI_RELEARN_TRIGGER; the stream's next n_frames frames are
 * learning frames (FIZI_RELEARN_LEARN: empty mask, a3-a7 fields 0, tracker
 * paused: visible = clicked = 0, px = py = 0, dwell 0); after the last one
 * (FIZI_RELEARN_SWAP) the stream's model becomes the a1 envelope of those raw
 * frames with `margin`, and the tracker restarts.  Triggers are ignored while
 * learning; learning may span calls.  Results do not depend on how frames are
 * batched.  Calls holding a relearning stream run joined even in pipelined
 * mode.  n_frames = 0 disables (and frees the model pool); threshold <= 255.
 * fizi_learn_background / fizi_set_background restart the relearn state. */
int fizi_set_relearn(fizi_ctx *ctx, uint32_t stream, uint32_t threshold, uint32_t n_frames,
                     uint8_t margin);

/* ---- NEXT-3: interface hit-test ("determines the interface zone
 * activated by the pointer").  Zones of a stream's layout
 * (parsed on the host) are tested against the a8 pointer of each frame, in
 * order; per frame and zone the membership and its events are written.
 * Readings L34/L35. */
enum { FIZI_ZONE_BUTTON = 0, FIZI_ZONE_SLIDER = 1, FIZI_ZONE_WHEEL = 2 };
enum { FIZI_EV_ENTER = 1, FIZI_EV_LEAVE = 2, FIZI_EV_CLICK = 4, FIZI_EV_VALUE = 8 };

typedef struct fizi_zone {         /* 72 bytes                                            */
    uint32_t kind;                 /* FIZI_ZONE_*                                          */
    uint32_t _pad;
    double   x, y, w, h;           /* button / slider rectangle, inclusive edges, w,h > 0  */
    double   cx, cy, r;            /* wheel circle (membership: squared distance <= r^2)   */
    double   theta_max_deg;        /* wheel: full lock angle, (0, 180]                     */
} fizi_zone;

typedef struct fizi_zone_event {   /* 16 bytes, one per frame and zone                     */
    uint8_t  inside;               /* membership after this frame                          */
    uint8_t  events;               /* FIZI_EV_* bits                                       */
    uint8_t  _pad[6];
    double   value;                /* slider [0,1] / wheel steering [-1,1] when FIZI_EV_VALUE, else 0 */
} fizi_zone_event;

/* Install the layout of stream `stream` (host array of n_zones <= 64 zones,
 * validated: FIZI_E_ARG) and reset its hit state (no zone entered). */
int fizi_set_zones(fizi_ctx *ctx, uint32_t stream, const fizi_zone *zones_host, uint32_t n_zones);

/* Hit-test n records of stream `stream` (device; visible, clicked, px, py),
 * in order; writes n * n_zones events (frame-major) to events_dev (device).
 * FIZI_E_NOMODEL if no layout was set. */
int fizi_hit_test(fizi_ctx *ctx, uint32_t stream, const fizi_result *results_dev, uint32_t n,
                  fizi_zone_event *events_dev, fizi_stream_t cuda_stream);

/* ---- NEXT-2: drive mapping ("a rotation around an imaginary
 * wheel"; SPEC module drive S:376-403).  The pointer of a8 is mapped to a
 * signed steering value on a virtual wheel and folded into one command per
 * frame.  Readings L32/L33. */
typedef struct fizi_wheel {
    double   cx, cy;               /* wheel centre, pixels                                  */
    double   radius;               /* > 0                                                   */
    double   theta_max_deg;        /* 90: |theta| at full lock, (0, 180]                    */
    double   inner, outer;         /* 0.6, 1.4: annulus in fractions of the radius, inner<1<outer */
    double   dead_zone_deg;        /* 3: |theta| <= dead zone steers 0, >= 0                */
    int64_t  hold_ms;              /* 200: steering held after the last reading, then x0.8/frame */
} fizi_wheel;

typedef struct fizi_command {      /* 32 bytes per frame                                    */
    double   steering;             /* [-1, 1], negative = left                              */
    double   throttle;             /* [0, 1]: last slider value (fizi_drive_throttle), 0 at start */
    int64_t  t_ms;                 /* the frame's timestamp                                 */
    uint32_t has_steering;         /* 1 iff the pointer was on the wheel in this frame      */
    uint32_t _pad;
} fizi_command;

/* Fill *w with the defaults above for a wheel at (cx, cy) of the given radius. */
int fizi_wheel_default(fizi_wheel *w, double cx, double cy, double radius);

/* Install (validated: FIZI_E_ARG) the wheel of stream `stream` and reset its
 * drive state to the neutral command (0, 0) with no reading. */
int fizi_set_wheel(fizi_ctx *ctx, uint32_t stream, const fizi_wheel *wheel);

/* Fold n records of stream `stream` (device; fields visible, px, py, t_ms as
 * written by a8), in order, through the stream's drive state; writes n
 * commands to commands_dev (device).  FIZI_E_NOMODEL if no wheel was set.
 * Joins outstanding pipelined tails into cuda_stream first. */
int fizi_drive(fizi_ctx *ctx, uint32_t stream, const fizi_result *results_dev, uint32_t n,
               fizi_command *commands_dev, fizi_stream_t cuda_stream);

/* As fizi_drive, with the throttle source of make_command (S:396-399:
 * "throttle: slider value when present, else previous throttle"): events_dev
 * (device) holds the n * n_zones events fizi_hit_test wrote for the same n
 * records of this stream (frame-major); the slider value of frame i is
 * events_dev[i * n_zones + slider_zone].value when that event carries
 * FIZI_EV_VALUE, else absent.  FIZI_E_NOMODEL without a wheel or a layout;
 * FIZI_E_ARG if n_zones is not the layout's zone count or slider_zone is not
 * a FIZI_ZONE_SLIDER of it.  Reading L36. */
int fizi_drive_throttle(fizi_ctx *ctx, uint32_t stream, const fizi_result *results_dev, uint32_t n,
                        const fizi_zone_event *events_dev, uint32_t n_zones, uint32_t slider_zone,
                        fizi_command *commands_dev, fizi_stream_t cuda_stream);

/* Parity/debug: write stage `stage` of frame `frame_in_last_batch` of the last
 * fizi_process_frames / fizi_segment_frames call to out_dev (u8 per pixel;
 * u32 per pixel for FIZI_STAGE_LABELS).  Needs params.debug = 1 and, for
 * R1/R2/R3, the last call's frames still resident. */
int fizi_debug_stage(fizi_ctx *ctx, int stage, uint32_t frame_in_last_batch, void *out_dev,
                     fizi_stream_t cuda_stream);

/* Parity/debug: copy the context's K0 brightness tables (a2, §3.2;
 * readings L19-L21) to device memory: lut_dev (256 x 256 u8, row m = the
 * per-channel LUT of integer mean luma m, identity rows for luma_lo <= m <=
 * luma_hi), gamma_dev (256 doubles, gamma(m)) and corrected_dev (256 u8, 1
 * iff row m is not the identity).  Any of the three may be NULL. */
int fizi_get_lut_table(fizi_ctx *ctx, uint8_t *lut_dev, double *gamma_dev, uint8_t *corrected_dev,
                       fizi_stream_t cuda_stream);

/* Copy stream `stream`'s envelope out as two interleaved-RGB planes
 * (W*H*3 u8 each, the S:174 plane layout) to device memory. */
int fizi_get_background(fizi_ctx *ctx, uint32_t stream, uint8_t *lo_dev, uint8_t *hi_dev,
                        fizi_stream_t cuda_stream);

/* Install an envelope (same layout as fizi_get_background; lo <= hi is not
 * required) for stream `stream`, e.g. one broadcast from another rank. */
int fizi_set_background(fizi_ctx *ctx, uint32_t stream, const uint8_t *lo_dev,
                        const uint8_t *hi_dev, fizi_stream_t cuda_stream);

/* Pipelined mode (enable = 1; default 0).  By default every output of a
 * fizi_process_frames / fizi_segment_frames call is complete in cuda_stream
 * order when the call returns.  In pipelined mode a call runs as four stages
 * on the context's internal streams (segmentation; per-pixel words + LUT
 * re-test; a4 + the u8 mask; a5-a7 + the a8 fold), each stage in call order,
 * and is NOT joined into cuda_stream, so that the stages of consecutive calls
 * overlap; per-call state is multi-buffered inside the context.  A call's
 * stages start after the caller's earlier work on cuda_stream.  The context
 * keeps FIZI_CALL_SLOTS call slots: every write of call k+FIZI_CALL_SLOTS is
 * ordered after the last stage of call k, so a caller may rotate
 * FIZI_CALL_SLOTS output buffers across calls without waiting.  Outputs of a
 * pipelined call are complete in a stream's order after fizi_flush on that
 * stream; until then the caller must not read them, nor overwrite the call's
 * frames.  Every other entry point that touches the stages' state (learn /
 * set_background / track / reset_tracker / relearn / drive / hit test / debug
 * / host entry) joins the outstanding stages into its stream itself.  Calls
 * holding a relearning stream (fizi_set_relearn) always run joined. */
#ifndef FIZI_CALL_SLOTS
#define FIZI_CALL_SLOTS 4
#endif
int fizi_set_pipeline(fizi_ctx *ctx, int enable);

/* FIZI_CALL_SLOTS as this library was built with (a build may override the
 * header default with -DFIZI_CALL_SLOTS=k; callers size their output rotation
 * from this value). */
uint32_t fizi_call_slots(void);

/* Make cuda_stream wait for the tails of all previous calls (no-op when
 * nothing is outstanding).  Enqueues only; does not block the host. */
int fizi_flush(fizi_ctx *ctx, fizi_stream_t cuda_stream);

/* Per-stage device timing.  mode 1: every subsequent call records CUDA
 * events on its streams around each stage; mode 2: around the fused
 * segmentation kernel only (two events per call); 0: off.
 * fizi_profile_read synchronises those events and returns the accumulated
 * milliseconds and the number of timed launches per slot (FIZI_PROF_*),
 * optionally resetting them. */
enum {
    FIZI_PROF_SEGMENT = 0,    /* fused luma + three branches (a2+a3)          */
    FIZI_PROF_FIXUP = 1,      /* mean -> gamma, LUT re-test of corrected frames */
    FIZI_PROF_MORPH = 2,      /* open-close (a4)                              */
    FIZI_PROF_CCL = 3,        /* labelling, filter, hand blob (a5-a7)         */
    FIZI_PROF_EXPAND = 4,     /* final u8 mask write (a6 output)              */
    FIZI_PROF_TRACK = 5,      /* Mouse fold (a8)                              */
    FIZI_PROF_SLOW = 6,       /* per-pixel R1/R2/R3 of the words queued by the fused kernel */
    FIZI_PROF_MASKZERO = 7,   /* u8 mask target cleared before the labelling writes it */
    FIZI_PROF_SLOTS = 8
};
int fizi_profile_enable(fizi_ctx *ctx, int mode);
int fizi_profile_read(fizi_ctx *ctx, double *ms_out, uint64_t *count_out, int reset);

/* Number of kernels this context has launched so far (evidence for the
 * bench's gpu_launches count). */
uint64_t fizi_kernel_launches(const fizi_ctx *ctx);

/* Human-readable description of the last error on ctx (never NULL). */
const char *fizi_last_error(const fizi_ctx *ctx);

/* Static name of a status code. */
const char *fizi_status_string(int status);

/* Free every device and host resource of ctx (NULL is a no-op). */
void fizi_destroy(fizi_ctx *ctx);

#ifdef __cplusplus
}
#endif

#endif /* FIZI_H */
