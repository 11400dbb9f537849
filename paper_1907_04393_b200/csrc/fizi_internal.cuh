// fizi_internal.cuh -- context layout and kernel launchers of libfizi.so.
//
// Device data layout:
//   envelope   per stream: two planes (lo, hi), each nchunks*1536 bytes, in the
//              chunk-permuted order the fused segmentation kernel reads with
//              coalesced 16-byte loads (see k_segment.cu: env_perm_index).
//   bit masks  per frame: H rows x P = ceil(W/32) u32 words, bit i of word k
//              = pixel x = 32k + i (LSB first); padding bits are always 0.
//   runs       per frame: up to cap_runs = H * ceil(W/2) compact runs; row y's
//              runs are row_cnt[y] entries from row_base[y] (sorted by x),
//              rows in arbitrary order; union-find parent + per-root stats.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cuda_runtime.h>

#include "fizi.h"

namespace fizi {

constexpr int kChunkPx = 512;            // pixels per warp-chunk in the fused kernel
constexpr int kChunkBytes = 3 * kChunkPx;
constexpr int kWarpsPerCta = 8;          // chunks per CTA tile
constexpr int kTileBytes = kChunkBytes * kWarpsPerCta;   // 12 KiB frame bytes per tile
constexpr int kFrameGroup = 32;          // frames sharing one envelope load (<= 32)
constexpr int kMaxRadius = 8;
constexpr size_t kMorphSmem = 200 * 1024;  // dynamic smem budget of the morphology CTA
constexpr uint32_t kCclSmemRuns = 4096;     // runs labelled in shared memory (else global)
constexpr uint32_t kMaxSub = 8;             // sub-batches per call (stream pipeline)
constexpr uint32_t kSlots = FIZI_CALL_SLOTS;  // per-call state slots (pipelined calls in flight)

struct Run {                             // one horizontal run of foreground pixels
  uint16_t x0, x1, y, pad;
};

// Per-call pointers, uploaded with the per-call table so that the kernels of
// one call shape are launch-invariant (a captured CUDA graph replays them).
struct CallPtrs {
  const uint8_t* frames;                 // n x 3N interleaved RGB (device)
  uint8_t* masks;                        // u8 mask target of the fused path, or nullptr
  fizi_result* res;                      // n records (device)
  uint64_t n;
  int64_t single_stream;                 // stream id when every frame is of one stream, else -1
  uint64_t call_id;                      // diagnostics: timeline slot (FIZI_TIMELINE)
  unsigned long long* tl;                // diagnostics: timeline buffer or nullptr
};

// Diagnostics timeline (env FIZI_TIMELINE=1): per kernel kind and call, the
// earliest CTA start and the latest CTA end (globaltimer ns).
constexpr int kTlKinds = 8, kTlCalls = 256;
enum { kTlSeg = 0, kTlFix = 1, kTlZero = 2, kTlMorph = 3, kTlCcl = 4, kTlFold = 5, kTlSlow = 6 };
#ifdef __CUDACC__
__device__ __forceinline__ void tl_mark(const CallPtrs* call, int kind, int end) {
  unsigned long long* tl = call->tl;
  if (!tl) return;
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  const uint64_t i = (uint64_t)kind * kTlCalls + call->call_id % kTlCalls;
  if (end) atomicMax(tl + kTlKinds * kTlCalls + i, t);
  else atomicMin(tl + i, t);
}
#endif

struct RootStats {                       // per component (indexed by its root run)
  uint32_t area;
  uint32_t xmin, xmax, ymin, ymax;
  uint32_t pad;
  unsigned long long sx, sy;
};

struct RelearnState {                    // NEXT-1 in-stream relearning, per stream (k_relearn.cu)
  int32_t prev_mean;                     // a2 mean of the stream's previous frame, -1 = none
  uint32_t remaining;                    // learning frames still to come (0: segmenting)
  uint32_t continuing;                   // the current learning began in an earlier call
  uint32_t enabled, threshold, frames, margin, pool_slots;
  uint64_t pool;                         // device: pool_slots models (2 planes each)
  uint64_t acc;                          // device: carried min / max (2 planes)
};

struct Ctx {
  fizi_params p{};
  int device = 0;
  uint32_t n_streams = 0, max_batch = 0;
  uint32_t W = 0, H = 0, P = 0;          // P = words per bit-mask row
  uint64_t N = 0;                        // pixels per frame
  uint32_t nchunks = 0;                  // ceil(N / 512)
  uint64_t env_plane = 0;                // bytes per envelope plane (nchunks*1536)
  uint64_t cap_runs = 0;                 // run capacity per frame
  bool fast = false;                     // W % 32 == 0: fused bulk-copy kernels
  int sms = 148;
  uint32_t seg_persist = 5;              // persistent fused kernel: half-CTAs per SM (0: off)
  uint32_t group_max = kFrameGroup;      // frames per same-stream group (fused-kernel item)
  bool use_dirty = false;                // clean chunks of A are not written (dirty bitmap)
  bool inline_words = false;             // per-pixel words evaluated inside the fused kernel (A/B)
  bool mask_by_morph = true;             // u8 mask rows written by the morphology (else zero + kept runs)
  uint32_t morph_tr = 0;                 // output rows per morphology CTA
  uint64_t launches = 0;
  unsigned long long* tl = nullptr;      // diagnostics timeline (FIZI_TIMELINE)
  uint64_t call_counter = 0;
  uint64_t host_call_ns = 0, host_sync_ns = 0;   // diagnostics
  std::string err;
  bool sticky = false;

  // device
  uint8_t* env = nullptr;                // n_streams * 2 * env_plane
  uint8_t* lut = nullptr;                // 256 means x 256 entries
  double* gamma_tab = nullptr;           // 256
  uint8_t* corr_tab = nullptr;           // 256
  uint32_t* skin_tab = nullptr;          // 2^24 bits: R2 & R3 of every corrected colour
  // Per-call state lives in two slots (calls alternate between them) so that
  // a call's tail can still run while the next call segments (pipelined
  // mode).  The pointers below are views of the current slot (select_slot).
  uint8_t* zero_blocks[kSlots] = {};          // per-call counters (cleared each call)
  uint32_t* bitAs[kSlots] = {};               // merged masks A
  // morphology outputs (O, runs) per slot: call k+1's morphology writes its
  // own while call k's labelling reads call k's
  uint32_t* bitOs[kSlots] = {};
  uint32_t* row_cnts[kSlots] = {};
  uint32_t* row_bases[kSlots] = {};
  Run* runss[kSlots] = {};
  CallPtrs* calls[kSlots] = {};               // per-call tables
  uint8_t* zero_block = nullptr;         // views of the current slot's block below
  uint64_t zero_bytes = 0;
  unsigned long long* luma = nullptr;    // max_batch
  uint32_t* fg = nullptr;                // max_batch (fg_merged)
  uint32_t* frame_done = nullptr;        // max_batch (CTAs finished per frame)
  uint32_t* dirty = nullptr;             // max_batch x dirty_words: chunks with non-zero A words
  uint32_t dirty_words = 0;              // ceil(nchunks / 32)
  uint32_t* sub_done = nullptr;          // kMaxSub (CCL CTAs finished per sub-batch)
  uint32_t* fold_sync = nullptr;         // kMaxSub x (2 + max_batch): fold lock / cursor / ready
  uint32_t* bitA = nullptr;              // max_batch * H * P
  uint32_t* bitO = nullptr;              // max_batch * H * P (view of the slot's)
  uint32_t* bitOC = nullptr;             // debug copy of O
  uint32_t* row_cnt = nullptr;           // max_batch * H   (runs per row)
  uint32_t* row_base = nullptr;          // max_batch * H   (first run of the row)
  uint32_t* frame_runs = nullptr;        // max_batch       (runs per frame)
  Run* runs = nullptr;                   // max_batch * cap_runs
  uint32_t* parent = nullptr;            // max_batch * cap_runs
  RootStats* stats = nullptr;            // max_batch * cap_runs
  uint32_t* frame_stream = nullptr;      // max_batch
  CallPtrs* call = nullptr;              // start of the per-call table (device)
  int64_t* frame_t = nullptr;            // max_batch
  uint32_t* group_frames = nullptr;      // max_batch (frame ids ordered by group)
  uint32_t* group_off = nullptr;         // max_batch + 1
  uint32_t* fix_count = nullptr;         // kMaxSub x (1 + max_batch): per sub-batch count + list
  uint32_t* item_counter = nullptr;      // kMaxSub: fused-kernel work items taken
  uint32_t* slow_count = nullptr;        // kMaxSub: words queued for the per-pixel kernel
  unsigned long long* slow_items = nullptr;   // view of the slot's queue below
  // max_batch x nchunks x 16 queue per slot: call k's tail reads its queue
  // while call k+1's head (another slot) fills its own
  unsigned long long* slow_itemss[kSlots] = {};
  uint8_t* tstate = nullptr;             // n_streams tracker states
  uint8_t* dstate = nullptr;             // n_streams drive states (NEXT-2)
  int32_t* prev_mean = nullptr;          // n_streams relearn-trigger states (NEXT-1), -1 = none
  // NEXT-1 in-stream relearning (fizi_set_relearn)
  uint8_t* rstate = nullptr;             // n_streams RelearnState
  bool rl_active = false;                // the current call has a relearning stream (joined)
  uint32_t* rl_role = nullptr;           // max_batch: 0 / 1 learning / 2 re-segmented with rl_env
  uint32_t* rl_pair = nullptr;           // max_batch: version a learning frame belongs to
  uint64_t* rl_env = nullptr;            // max_batch: model of a role-2 frame
  uint32_t* rl_list = nullptr;           // 1 + max_batch: count, frames with a non-zero role
  uint32_t* rl_pairs = nullptr;          // max_batch x 4: versions of the call
  uint32_t* rl_counts = nullptr;         // versions, commits, commits x (stream, slot)
  uint32_t rl_max_pairs = 1, rl_max_commits = 1;
  std::vector<uint8_t> rl_enabled;       // host copy of RelearnState::enabled
  std::vector<uint8_t*> rl_mem;          // per stream: pool + accumulator allocation
  std::vector<RelearnState> rl_state_host;   // per stream: the configured initial state
  uint8_t* hstate = nullptr;             // n_streams hit-test states (NEXT-3)
  cudaStream_t side = nullptr;           // tail: LUT re-test + morphology (joined: whole tail)
  cudaStream_t cclst = nullptr;          // pipelined tail: labelling + u8 mask + fold, call order
  cudaStream_t morphst = nullptr;        // pipelined tail: morphology, call order
  cudaStream_t side2 = nullptr;          // head branch: u8 mask zeroing
  cudaStream_t side3 = nullptr;          // tail branch: LUT re-test
  cudaStream_t head = nullptr;           // pipelined head: segmentation (call order)
  cudaStream_t prep = nullptr;           // pipelined: the slot's table upload + counter clear, ahead
  cudaEvent_t ev_prep[kSlots] = {};      // pipelined: slot's table uploaded and counters cleared
  cudaEvent_t ev_hfork = nullptr, ev_hjoin = nullptr;   // head: u8 mask clear branch
  cudaStream_t h2d = nullptr, d2h = nullptr;   // fizi_process_frames_host copy streams
  std::vector<cudaEvent_t> host_ev;            // fizi_process_frames_host chunk events
  fizi_result* pinned_results = nullptr;       // fizi_process_frames_host record staging
  cudaEvent_t ev_in[kSlots] = {};        // pipelined: caller's stream reached the call
  cudaEvent_t ev_zfork = nullptr, ev_zjoin = nullptr;   // tail: LUT re-test branch
  cudaEvent_t ev_seg[kMaxSub] = {};      // segment(k) done on the caller's stream
  cudaEvent_t ev_join = nullptr;         // tail of the call done on the side stream
  cudaEvent_t ev_start = nullptr;        // call start on the caller's stream
  cudaEvent_t ev_head[kSlots] = {};           // pipelined: slot's segmentation done
  cudaEvent_t ev_morph[kSlots] = {};          // pipelined: slot's morphology done
  cudaEvent_t ev_words[kSlots] = {};          // pipelined: slot's per-pixel words + LUT re-test done
  cudaEvent_t ev_tail[kSlots] = {};           // slot's last call fully done (slot reusable)
  bool pipeline = false;                 // fizi_set_pipeline: tails not joined per call
  bool tail_pending = false;             // some pipelined tail may be outstanding
  uint32_t last_slot = 0;
  uint32_t sub_frames = 65535;           // frames per sub-batch (default: whole call)
  uint8_t* stage_frames = nullptr;       // device staging for fizi_process_frames_host
  uint8_t* stage_masks = nullptr;
  fizi_result* stage_results = nullptr;

  // host
  std::vector<uint8_t> env_valid;
  std::vector<uint8_t> has_wheel;        // NEXT-2: fizi_set_wheel called per stream
  std::vector<uint32_t> n_zones;         // NEXT-3: zones per stream (0: no layout)
  std::vector<uint64_t> slider_zones;    // NEXT-3: bit k set iff zone k of the stream is a slider
  std::vector<int64_t> last_t;
  std::vector<int> fc_slot;               // fill_call scratch: stream -> bucket (-1: none)
  std::vector<uint32_t> fc_order, fc_start;
  std::vector<uint8_t> has_t;
  uint8_t* pinned[kSlots] = {};               // staging for the per-call upload (one per slot)
  size_t pinned_bytes = 0;
  cudaEvent_t pinned_ev[kSlots] = {};
  cudaEvent_t slot_upload[kSlots] = {};  // the event that marks the slot's last table upload done
  uint32_t pinned_next = 0;
  // captured launch sequences, one per call shape and pinned slot
  struct GraphEntry {
    std::vector<uint32_t> key;
    cudaGraphExec_t exec[kSlots] = {};
    uint64_t kernels = 0;                // kernel nodes per replay
    uint64_t used = 0;
  };
  std::vector<GraphEntry> graphs;
  uint64_t graph_clock = 0;
  bool use_graphs = true;                // FIZI_NO_GRAPH=1 disables (A/B timing)
  cudaStream_t cap = nullptr;            // capture origin stream
  // per-stage timing (fizi_profile_*)
  bool prof = false;
  int prof_mode = 0;                     // 1: all stages, 2: fused kernel only
  bool prof_skip = false;
  struct ProfRec { int slot; cudaEvent_t a, b; };
  std::vector<ProfRec> prof_pending;
  std::vector<cudaEvent_t> prof_free;
  double prof_ms[FIZI_PROF_SLOTS] = {0};
  uint64_t prof_n[FIZI_PROF_SLOTS] = {0};
  cudaEvent_t prof_open = nullptr;
  // last call (debug)
  const uint8_t* last_frames = nullptr;
  uint32_t last_n = 0;
};

struct DriveState {                      // NEXT-2 make_command fold state
  double steering, throttle;
  int64_t last_reading;                  // t_ms of the last steering reading
  int32_t has_reading, has_wheel;
  fizi_wheel wheel;
};

constexpr uint32_t kMaxZones = 64;
struct HitState {                        // NEXT-3 layout + per-zone state of one stream
  uint32_t n_zones, pad;
  fizi_zone zones[kMaxZones];
  uint8_t inside[kMaxZones];
  uint8_t has_value[kMaxZones];
  double last_value[kMaxZones];
};

struct TrackState {                      // Mouse fold state (c1 step 11)
  int32_t vis, fired;
  double px, py, ax, ay;
  int64_t last_t, anchor_t, dwell;
};

// ------------------------------------------------------------ envelope layout
// Fast path: linear frame byte b -> chunk c = b/1536, lane l = (b%1536)/48,
// piece k = (b%48)/16, byte j = b%16 -> c*1536 + 512k + 16l + j, so that warp
// lane l reads its 48 frame bytes' envelope with three coalesced 16-byte
// loads at 512k + 16l.  Generic path: identity.
__host__ __device__ __forceinline__ uint64_t env_perm_index(uint64_t b, bool fast) {
  if (!fast) return b;
  uint64_t c = b / kChunkBytes, o = b % kChunkBytes;
  uint32_t l = (uint32_t)(o / 48), q = (uint32_t)(o % 48);
  return c * kChunkBytes + 512u * (q / 16) + 16u * l + (q % 16);
}

// ----------------------------------------------------------------- launchers
// All return cudaGetLastError() of their launches; each increments
// ctx.launches by the number of kernels launched.
cudaError_t launch_lut_table(Ctx& c, cudaStream_t st);
cudaError_t launch_skin_table(Ctx& c, cudaStream_t st);
cudaError_t launch_learn(Ctx& c, uint32_t stream, const uint8_t* frames, uint32_t n,
                         uint32_t margin, cudaStream_t st);
cudaError_t launch_env_export(Ctx& c, uint32_t stream, uint8_t* lo, uint8_t* hi, bool import,
                              const uint8_t* ilo, const uint8_t* ihi, cudaStream_t st);
// frames / records / u8 masks of a call come from c.call (the uploaded CallPtrs)
cudaError_t launch_seg_main(Ctx& c, uint32_t f0, uint32_t n, uint32_t g0, uint32_t ng, uint32_t sub,
                            cudaStream_t st);
cudaError_t launch_seg_fix(Ctx& c, uint32_t f0, uint32_t n, uint32_t sub, cudaStream_t st);
// per-pixel R1 & R2 & R3 of the words the fused kernel queued (fast path)
cudaError_t launch_slow_words(Ctx& c, uint32_t f0, uint32_t n, uint32_t sub, cudaStream_t st);
// the segment launcher marks the SEGMENT -> FIXUP boundary through this hook
void prof_begin(Ctx& c, cudaStream_t st);
void prof_end(Ctx& c, int slot, cudaStream_t st);
// write_masks: the morphology writes the u8 rows of O into c.call->masks
// (the labelling then clears the dropped components' runs)
cudaError_t launch_morph(Ctx& c, uint32_t f0, uint32_t n, bool write_masks, cudaStream_t st);
// masks_zeroed: c.call->masks (if any) was zeroed by launch_zero_masks (the
// labelling writes the kept runs), else it holds O (the labelling clears the
// dropped runs)
// g0 / ng: the sub-batch's same-stream groups (the per-stream fold walks them)
cudaError_t launch_ccl(Ctx& c, uint32_t f0, uint32_t n, uint32_t sub, uint32_t g0, uint32_t ng,
                       bool masks_zeroed, int track_stream, cudaStream_t st);
cudaError_t launch_zero_masks(Ctx& c, uint32_t n, cudaStream_t st);
cudaError_t launch_expand(Ctx& c, uint32_t f0, uint32_t n, uint8_t* masks, cudaStream_t st);
cudaError_t launch_track_stream(Ctx& c, uint32_t stream, fizi_result* res, uint32_t n,
                                cudaStream_t st);
constexpr uint32_t kMaxTrackRuns = 256;
cudaError_t launch_track_runs(Ctx& c, uint32_t stream, fizi_result* res, const uint32_t* off,
                              const uint32_t* len, uint32_t n_runs, cudaStream_t st);
// NEXT-1: relearn-trigger flags of a stream's records / reset of the state
cudaError_t launch_relearn_flags(Ctx& c, uint32_t stream, const fizi_result* res, uint32_t n,
                                 uint32_t threshold, uint8_t* flags, cudaStream_t st);
cudaError_t launch_relearn_reset(Ctx& c, uint32_t first, uint32_t count, cudaStream_t st);
// NEXT-1 in-stream relearning: roles + models of the call (after the means),
// re-segmentation of role-2 frames / emptying of learning frames (fast path),
// model commit at the end of the call, per-stream state upload
cudaError_t launch_relearn_plan(Ctx& c, uint32_t n, cudaStream_t st);
cudaError_t launch_relearn_reseg(Ctx& c, uint32_t n, cudaStream_t st);
cudaError_t launch_relearn_commit(Ctx& c, cudaStream_t st);
cudaError_t launch_relearn_state(Ctx& c, uint32_t stream, const RelearnState& v, cudaStream_t st);
// NEXT-3: hit-test of a stream's records against its layout (state in c.hstate)
cudaError_t launch_hit_test(Ctx& c, uint32_t stream, const fizi_result* res, uint32_t n,
                            fizi_zone_event* out, cudaStream_t st);
// NEXT-2: install a wheel (resets the drive state) / fold records into commands
cudaError_t launch_drive_set(Ctx& c, uint32_t stream, const fizi_wheel& w, cudaStream_t st);
cudaError_t launch_drive(Ctx& c, uint32_t stream, const fizi_result* res, uint32_t n,
                         const fizi_zone_event* ev, uint32_t nz, uint32_t zi, fizi_command* out,
                         cudaStream_t st);
cudaError_t launch_tstate_reset(Ctx& c, uint32_t first, uint32_t count, cudaStream_t st);
cudaError_t launch_debug_stage(Ctx& c, int stage, uint32_t frame, void* out, cudaStream_t st);

// Experiment switch FIZI_CARVEOUT=<0..100>: the preferred shared-memory
// carveout of the per-call kernels (unset: the driver's choice per launch).
inline cudaError_t set_carveout(const void* fn) {
  static const int pct = getenv("FIZI_CARVEOUT") ? atoi(getenv("FIZI_CARVEOUT")) : -1;
  if (pct < 0) return cudaSuccess;
  return cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, pct);
}

// Diagnostics only: FIZI_DIAG_SKIP=<stage>[,<stage>] skips a pipeline stage
// (the outputs are then wrong) to measure what that stage costs; announced
// once on stderr so that it cannot pass unnoticed.
inline bool diag_skip(const char* stage) {
  const char* v = getenv("FIZI_DIAG_SKIP");
  if (!v || !strstr(v, stage)) return false;
  static bool warned = false;
  if (!warned) {
    fprintf(stderr, "libfizi: FIZI_DIAG_SKIP=%s is set: stages are skipped, outputs are NOT valid\n", v);
    warned = true;
  }
  return true;
}

}  // namespace fizi
