// fizi_api.cu -- the C ABI of libfizi.so (include/fizi.h): argument
// validation, context / memory management and the per-call launch sequence
//   segment (a2+a3) -> morphology (a4) -> labelling + filter + blob (a5-a7)
//   -> final u8 mask (a6 output) -> Mouse fold (a8)
// on the caller's CUDA stream.  No pixel is touched on the host.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include "fizi_internal.cuh"

namespace fizi {
uint32_t morph_tile_rows(const Ctx& c, size_t smem_budget);
cudaError_t init_morph(Ctx& c);
cudaError_t init_segment(Ctx& c);
cudaError_t init_ccl(Ctx& c);
}  // namespace fizi

struct fizi_ctx {
  fizi::Ctx c;
};

using fizi::Ctx;

namespace fizi {

static cudaEvent_t prof_event(Ctx& c) {
  if (!c.prof_free.empty()) {
    cudaEvent_t e = c.prof_free.back();
    c.prof_free.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  return e;
}

static void prof_resolve(Ctx& c) {
  for (auto& r : c.prof_pending) {
    cudaEventSynchronize(r.b);
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, r.a, r.b) == cudaSuccess) {
      c.prof_ms[r.slot] += ms;
      c.prof_n[r.slot] += 1;
    }
    c.prof_free.push_back(r.a);
    c.prof_free.push_back(r.b);
  }
  c.prof_pending.clear();
}

void prof_begin(Ctx& c, cudaStream_t st) {
  if (!c.prof) return;
  c.prof_skip = false;
  c.prof_open = prof_event(c);
  cudaEventRecord(c.prof_open, st);
}

void prof_end(Ctx& c, int slot, cudaStream_t st) {
  if (!c.prof || !c.prof_open) return;
  if (c.prof_mode == 2 && slot != FIZI_PROF_SEGMENT) {   // mode 2: fused kernel only
    c.prof_free.push_back(c.prof_open);
    c.prof_open = nullptr;
    return;
  }
  cudaEvent_t b = prof_event(c);
  cudaEventRecord(b, st);
  c.prof_pending.push_back({slot, c.prof_open, b});
  c.prof_open = nullptr;
  if (c.prof_pending.size() > 4096) prof_resolve(c);
}

}  // namespace fizi

using fizi::prof_begin;
using fizi::prof_end;

namespace {

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int d) {
    cudaGetDevice(&prev);
    if (prev != d) cudaSetDevice(d);
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

int fail(Ctx& c, int code, const std::string& msg) {
  c.err = msg;
  return code;
}

int cuda_fail(Ctx& c, cudaError_t e, const char* where) {
  c.sticky = true;
  c.err = std::string(where) + ": " + cudaGetErrorName(e) + " (" + cudaGetErrorString(e) + ")";
  return FIZI_E_CUDA;
}

int validate_params(const fizi_params* p, std::string& why) {
  auto bad = [&](const char* m) { why = m; return FIZI_E_ARG; };
  if (!p) return bad("params is NULL");
  if (p->width < 1 || p->width > 65535 || p->height < 1 || p->height > 65535)
    return bad("width/height must be in [1, 65535]");
  if (p->gray_tol_S > 255) return bad("gray_tol_S must be <= 255");
  if (p->hue_lo_deg >= 360 || p->hue_hi_deg >= 360) return bad("hue bounds must be in [0, 360)");
  if (p->se_radius < 1 || p->se_radius > (uint32_t)fizi::kMaxRadius)
    return bad("se_radius must be in [1, 8]");
  if (p->min_blob_ppm > 1000000) return bad("min_blob_ppm must be <= 1e6");
  if (p->luma_target > 255 || p->luma_hi > 255 || !(p->luma_lo < p->luma_target) ||
      !(p->luma_target < p->luma_hi))
    return bad("need luma_lo < luma_target < luma_hi <= 255 (S:189)");
  if (!(std::isfinite(p->gamma_min) && std::isfinite(p->gamma_max)) || !(p->gamma_min > 0.0) ||
      !(p->gamma_min <= p->gamma_max))
    return bad("need 0 < gamma_min <= gamma_max");
  if (!(p->beta >= 0.0 && p->beta <= 1.0)) return bad("beta must be in [0, 1]");
  if (!(p->dwell_radius_px >= 0.0) || !std::isfinite(p->dwell_radius_px))
    return bad("dwell_radius_px must be >= 0");
  if (p->dwell_time_ms < 0 || p->lost_timeout_ms < 0) return bad("times must be >= 0");
  return FIZI_OK;
}

template <typename T>
cudaError_t dalloc(T** p, size_t bytes) {
  return cudaMalloc(reinterpret_cast<void**>(p), bytes ? bytes : 16);
}

void destroy_graphs(Ctx& c);

void free_all(Ctx& c) {
  for (uint32_t i = 0; i < fizi::kSlots; i++) {
    if (c.zero_blocks[i]) cudaFree(c.zero_blocks[i]);
    if (c.bitAs[i]) cudaFree(c.bitAs[i]);
    if (c.slow_itemss[i]) cudaFree(c.slow_itemss[i]);
    for (void* q : {(void*)c.bitOs[i], (void*)c.row_cnts[i], (void*)c.row_bases[i], (void*)c.runss[i]})
      if (q) cudaFree(q);
    if (c.calls[i]) cudaFree(c.calls[i]);
  }
  for (uint8_t* q : c.rl_mem)
    if (q) cudaFree(q);
  c.rl_mem.clear();
  void* ptrs[] = {c.env, c.lut, c.gamma_tab, c.corr_tab, c.skin_tab, c.bitOC,
                  c.rstate, c.rl_role, c.rl_pair, c.rl_env, c.rl_list, c.rl_pairs, c.rl_counts,
                  c.parent, c.stats, c.tl, c.dstate,
                  c.prev_mean, c.hstate,
                  c.tstate, c.stage_frames, c.stage_masks, c.stage_results};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  destroy_graphs(c);
  for (uint32_t i = 0; i < fizi::kSlots; i++) {
    if (c.pinned[i]) cudaFreeHost(c.pinned[i]);
    if (c.pinned_ev[i]) cudaEventDestroy(c.pinned_ev[i]);
  }
  if (c.cap) cudaStreamDestroy(c.cap);
  for (auto ev : c.ev_seg)
    if (ev) cudaEventDestroy(ev);
  if (c.ev_join) cudaEventDestroy(c.ev_join);
  if (c.ev_start) cudaEventDestroy(c.ev_start);
  for (uint32_t i = 0; i < fizi::kSlots; i++) {
    if (c.ev_head[i]) cudaEventDestroy(c.ev_head[i]);
    if (c.ev_morph[i]) cudaEventDestroy(c.ev_morph[i]);
    if (c.ev_words[i]) cudaEventDestroy(c.ev_words[i]);
    if (c.ev_tail[i]) cudaEventDestroy(c.ev_tail[i]);
  }
  if (c.side) cudaStreamDestroy(c.side);
  if (c.side2) cudaStreamDestroy(c.side2);
  if (c.side3) cudaStreamDestroy(c.side3);
  if (c.head) cudaStreamDestroy(c.head);
  if (c.prep) cudaStreamDestroy(c.prep);
  for (auto ev : c.ev_prep)
    if (ev) cudaEventDestroy(ev);
  if (c.cclst) cudaStreamDestroy(c.cclst);
  if (c.morphst) cudaStreamDestroy(c.morphst);
  if (c.pinned_results) cudaFreeHost(c.pinned_results);
  if (c.h2d) cudaStreamDestroy(c.h2d);
  if (c.d2h) cudaStreamDestroy(c.d2h);
  for (auto ev : c.host_ev) cudaEventDestroy(ev);
  for (uint32_t i = 0; i < fizi::kSlots; i++)
    if (c.ev_in[i]) cudaEventDestroy(c.ev_in[i]);
  for (cudaEvent_t ev : {c.ev_zfork, c.ev_zjoin, c.ev_hfork, c.ev_hjoin})
    if (ev) cudaEventDestroy(ev);
  for (auto& r : c.prof_pending) { cudaEventDestroy(r.a); cudaEventDestroy(r.b); }
  for (auto e : c.prof_free) cudaEventDestroy(e);
  if (c.prof_open) cudaEventDestroy(c.prof_open);
}

// Point the context's per-call views at slot s.
void select_slot(Ctx& c, uint32_t s) {
  const uint64_t mb = c.max_batch;
  uint8_t* z = c.zero_blocks[s];
  c.zero_block = z;
  c.luma = reinterpret_cast<unsigned long long*>(z); z += mb * 8;
  c.fg = reinterpret_cast<uint32_t*>(z); z += mb * 4;
  c.frame_done = reinterpret_cast<uint32_t*>(z); z += mb * 4;
  c.frame_runs = reinterpret_cast<uint32_t*>(z); z += mb * 4;
  c.sub_done = reinterpret_cast<uint32_t*>(z); z += fizi::kMaxSub * 4;
  c.fold_sync = reinterpret_cast<uint32_t*>(z); z += fizi::kMaxSub * (mb + 2) * 4;
  c.fix_count = reinterpret_cast<uint32_t*>(z); z += fizi::kMaxSub * (mb + 1) * 4;
  c.item_counter = reinterpret_cast<uint32_t*>(z); z += fizi::kMaxSub * 4;
  c.slow_count = reinterpret_cast<uint32_t*>(z); z += fizi::kMaxSub * 4;
  c.dirty = reinterpret_cast<uint32_t*>(z);
  c.bitA = c.bitAs[s];
  c.bitO = c.bitOs[s];
  c.slow_items = c.slow_itemss[s];
  c.row_cnt = c.row_cnts[s];
  c.row_base = c.row_bases[s];
  c.runs = c.runss[s];
  c.call = c.calls[s];
  c.frame_t = reinterpret_cast<int64_t*>(c.call + 1);
  c.frame_stream = reinterpret_cast<uint32_t*>(c.frame_t + mb);
  c.group_frames = c.frame_stream + mb;
  c.group_off = c.group_frames + mb;
}

// Make st wait for every outstanding pipelined tail (side stream is in order).
cudaError_t join_tail(Ctx& c, cudaStream_t st) {
  if (!c.tail_pending) return cudaSuccess;
  return cudaStreamWaitEvent(st, c.ev_tail[c.last_slot], 0);
}

struct SubBatch {
  uint32_t f0, n, g0, ng;
};

// Host side of the per-call table: CallPtrs, timestamps, streams and the
// same-stream groups, written into pinned slot `slot`.  Frames are cut into
// sub-batches of c.sub_frames (at most kMaxSub); inside a sub-batch, groups
// are the frames of one stream in index order, split every kFrameGroup frames.
void fill_call(Ctx& c, uint32_t slot, const fizi::CallPtrs& cp, const uint32_t* sof,
               const int64_t* t, uint32_t n, std::vector<SubBatch>& subs) {
  const uint32_t mb = c.max_batch;
  *reinterpret_cast<fizi::CallPtrs*>(c.pinned[slot]) = cp;
  int64_t* ht = reinterpret_cast<int64_t*>(c.pinned[slot] + sizeof(fizi::CallPtrs));
  uint32_t* hs = reinterpret_cast<uint32_t*>(ht + mb);
  uint32_t* hg = hs + mb;
  uint32_t* ho = hg + mb;
  for (uint32_t i = 0; i < n; i++) {
    ht[i] = t ? t[i] : 0;
    hs[i] = sof[i];
  }
  uint32_t sb = c.sub_frames;
  if ((n + sb - 1) / sb > fizi::kMaxSub) sb = (n + fizi::kMaxSub - 1) / fizi::kMaxSub;
  subs.clear();
  // per sub-batch: the frames bucketed by stream (streams in order of first
  // appearance, frames in index order; a counting sort, O(frames + streams)),
  // each bucket cut into groups of at most group_max frames
  if (c.fc_slot.size() != c.n_streams) c.fc_slot.assign(c.n_streams, -1);
  std::vector<uint32_t>& order = c.fc_order;     // streams of the sub-batch, first appearance
  std::vector<uint32_t>& start = c.fc_start;     // bucket offsets
  uint32_t pos = 0, g = 0;
  for (uint32_t f0 = 0; f0 < n; f0 += sb) {
    const uint32_t f1 = std::min(n, f0 + sb);
    SubBatch b{f0, f1 - f0, g, 0};
    order.clear();
    start.clear();
    for (uint32_t i = f0; i < f1; i++) {
      int& k = c.fc_slot[sof[i]];
      if (k < 0) {
        k = (int)order.size();
        order.push_back(sof[i]);
        start.push_back(0);
      }
      start[k]++;
    }
    uint32_t acc = pos;
    for (uint32_t& v : start) {                  // counts -> bucket starts
      const uint32_t cnt = v;
      v = acc;
      acc += cnt;
    }
    for (size_t k = 0; k < order.size(); k++) {  // group starts, group_max frames each
      const uint32_t b0 = start[k], b1 = k + 1 < order.size() ? start[k + 1] : acc;
      for (uint32_t q = b0; q < b1; q += c.group_max) ho[g++] = q;
    }
    for (uint32_t i = f0; i < f1; i++) hg[start[c.fc_slot[sof[i]]]++] = i;
    for (uint32_t st : order) c.fc_slot[st] = -1;
    pos = acc;
    b.ng = g - b.g0;
    subs.push_back(b);
  }
  ho[g] = pos;
}

struct CallPlan {
  uint32_t n = 0, slot = 0;
  std::vector<SubBatch> subs;
  int fold = -2;               // -2 no fold, -1 per-stream end fold, >= 0 single-stream fold
  bool fused_mask = false;     // the labelling kernel writes the u8 mask (pre-zeroed)
  bool relearn = false;        // NEXT-1: a stream of the call relearns (joined, one sub-batch)
  bool premask = false;        // u8 mask: zeroed beside the segmentation, kept runs by labelling
  bool morphmask = false;      // u8 mask: rows of O by the morphology, dropped runs cleared
  uint8_t* masks = nullptr;    // caller's u8 masks (expand path only)
};

// Parts of a call's launch sequence.  kWhole: everything on the caller's
// stream st (sub-batch k's tail forked to the side stream, overlapping the
// segmentation of sub-batch k+1, joined back).  Pipelined mode splits the
// call into kHead (upload + counters + fused segmentation, on st) and kTail
// (u8 mask zeroing, LUT re-test, a4 morphology, a5-a7 labelling + u8 mask,
// a8 fold, on the side stream) so that call k's tail overlaps call k+1's head.
enum Part { kWhole = 0, kHead = 1, kTail = 2, kTailCcl = 3, kTailMorph = 4 };

int enqueue_head(Ctx& c, const CallPlan& pl, cudaStream_t st) {
  cudaError_t e = cudaMemcpyAsync(c.call, c.pinned[pl.slot], c.pinned_bytes, cudaMemcpyHostToDevice, st);
  if (e != cudaSuccess) return cuda_fail(c, e, "cudaMemcpyAsync(call table)");
  e = cudaMemsetAsync(c.zero_block, 0, c.zero_bytes, st);   // every per-call counter
  if (e != cudaSuccess) return cuda_fail(c, e, "memset");
  return FIZI_OK;
}

int enqueue_tail(Ctx& c, const CallPlan& pl, const SubBatch& b, uint32_t k, cudaStream_t sd,
                 cudaEvent_t before_ccl, bool with_fix) {
  cudaError_t e = cudaSuccess;
  if (with_fix) {
    e = fizi::launch_seg_fix(c, b.f0, b.n, k, sd);
    if (e == cudaSuccess && c.rl_active) e = fizi::launch_relearn_reseg(c, b.n, sd);
    if (e != cudaSuccess) return cuda_fail(c, e, "fixup");
  }
  prof_begin(c, sd);
  e = fizi::launch_morph(c, b.f0, b.n, pl.morphmask, sd);
  prof_end(c, FIZI_PROF_MORPH, sd);
  if (e != cudaSuccess) return cuda_fail(c, e, "morph");
  if (c.p.debug) {
    const size_t w = (size_t)c.H * c.P;
    e = cudaMemcpyAsync(c.bitOC + b.f0 * w, c.bitO + b.f0 * w, (size_t)b.n * w * 4,
                        cudaMemcpyDeviceToDevice, sd);
    if (e != cudaSuccess) return cuda_fail(c, e, "debug copy");
  }
  if (before_ccl) {
    e = cudaStreamWaitEvent(sd, before_ccl, 0);
    if (e != cudaSuccess) return cuda_fail(c, e, "join");
  }
  prof_begin(c, sd);
  e = fizi::launch_ccl(c, b.f0, b.n, k, b.g0, b.ng, pl.premask, pl.fold, sd);
  prof_end(c, FIZI_PROF_CCL, sd);
  if (e != cudaSuccess) return cuda_fail(c, e, "ccl");
  if (pl.masks && !pl.fused_mask) {
    prof_begin(c, sd);
    e = fizi::launch_expand(c, b.f0, b.n, pl.masks, sd);
    prof_end(c, FIZI_PROF_EXPAND, sd);
    if (e != cudaSuccess) return cuda_fail(c, e, "expand");
  }
  return FIZI_OK;
}

// The launch sequence of one part on stream st.  It is identical for every
// call of the same plan (all per-call pointers travel in the uploaded
// CallPtrs), so it is captured once into a CUDA graph and replayed.
int enqueue_part(Ctx& c, const CallPlan& pl, int part, cudaStream_t st) {
  cudaError_t e = cudaSuccess;
  int rc = FIZI_OK;
  if (part == kHead) {
    // the fused segmentation kernel beside the u8 mask clear (a branch on
    // side2, joined back); the table upload and counter clear ran ahead on
    // the prep stream
    if (pl.premask) {
      e = cudaEventRecord(c.ev_hfork, st);
      if (e == cudaSuccess) e = cudaStreamWaitEvent(c.side2, c.ev_hfork, 0);
      if (e == cudaSuccess) e = fizi::launch_zero_masks(c, pl.n, c.side2);
      if (e == cudaSuccess) e = cudaEventRecord(c.ev_hjoin, c.side2);
      if (e != cudaSuccess) return cuda_fail(c, e, "mask zero");
    }
    e = fizi::launch_seg_main(c, 0, pl.n, 0, pl.subs[0].ng, 0, st);
    if (e != cudaSuccess) return cuda_fail(c, e, "segment");
    if (pl.premask) {
      e = cudaStreamWaitEvent(st, c.ev_hjoin, 0);
      if (e != cudaSuccess) return cuda_fail(c, e, "join");
    }
    return FIZI_OK;
  }
  if (part == kTail) {
    // the queued per-pixel words and the LUT re-test of corrected frames
    // open the tail (the morphology needs them, the next call's
    // segmentation does not); the two touch disjoint frames, so the LUT
    // re-test runs on a branch (side3) and joins before the morphology.
    // The a8 fold runs inside the labelling kernel (the CTA holding the
    // fold lock folds the ready records in order).
    e = cudaEventRecord(c.ev_zfork, st);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(c.side3, c.ev_zfork, 0);
    if (e == cudaSuccess) e = fizi::launch_seg_fix(c, 0, pl.n, 0, c.side3);
    if (e == cudaSuccess) e = cudaEventRecord(c.ev_zjoin, c.side3);
    if (e != cudaSuccess) return cuda_fail(c, e, "fixup");
    if (c.fast) {
      e = fizi::launch_slow_words(c, 0, pl.n, 0, st);
      if (e != cudaSuccess) return cuda_fail(c, e, "slow words");
    }
    e = cudaStreamWaitEvent(st, c.ev_zjoin, 0);
    return e == cudaSuccess ? FIZI_OK : cuda_fail(c, e, "join");
  }
  if (part == kTailMorph) {
    prof_begin(c, st);
    e = fizi::launch_morph(c, 0, pl.n, pl.morphmask, st);
    prof_end(c, FIZI_PROF_MORPH, st);
    return e == cudaSuccess ? FIZI_OK : cuda_fail(c, e, "morph");
  }
  if (part == kTailCcl) {                  // a5-a7 + u8 mask + a8 fold (fused)
    prof_begin(c, st);
    e = fizi::launch_ccl(c, 0, pl.n, 0, pl.subs[0].g0, pl.subs[0].ng, pl.premask, pl.fold, st);
    prof_end(c, FIZI_PROF_CCL, st);
    if (e != cudaSuccess) return cuda_fail(c, e, "ccl");
    if (pl.masks && !pl.fused_mask) {
      prof_begin(c, st);
      e = fizi::launch_expand(c, 0, pl.n, pl.masks, st);
      prof_end(c, FIZI_PROF_EXPAND, st);
      if (e != cudaSuccess) return cuda_fail(c, e, "expand");
    }
    return FIZI_OK;
  }
  rc = enqueue_head(c, pl, st);
  if (rc) return rc;
  cudaStream_t sd = c.side;
  e = cudaEventRecord(c.ev_start, st);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(sd, c.ev_start, 0);
  if (e != cudaSuccess) return cuda_fail(c, e, "fork");
  // the u8 mask target is zeroed on the side stream while the fused
  // segmentation kernel runs; the labelling kernel then writes the bytes of
  // the kept components only
  if (pl.premask) {
    e = fizi::launch_zero_masks(c, pl.n, sd);
    if (e != cudaSuccess) return cuda_fail(c, e, "mask zero");
  }
  for (size_t k = 0; k < pl.subs.size(); k++) {
    const SubBatch& b = pl.subs[k];
    e = fizi::launch_seg_main(c, b.f0, b.n, b.g0, b.ng, (uint32_t)k, st);
    // NEXT-1: roles and models from the means before any per-pixel word
    if (e == cudaSuccess && c.rl_active && c.fast) e = fizi::launch_relearn_plan(c, b.n, st);
    if (e == cudaSuccess && c.fast) e = fizi::launch_slow_words(c, b.f0, b.n, (uint32_t)k, st);
    if (e != cudaSuccess) return cuda_fail(c, e, "segment");
    e = cudaEventRecord(c.ev_seg[k], st);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(sd, c.ev_seg[k], 0);
    if (e != cudaSuccess) return cuda_fail(c, e, "event");
    rc = enqueue_tail(c, pl, b, (uint32_t)k, sd, nullptr, true);
    if (rc) return rc;
  }
  if (c.rl_active) {                                    // NEXT-1: install the newest models
    e = fizi::launch_relearn_commit(c, sd);
    if (e != cudaSuccess) return cuda_fail(c, e, "relearn commit");
  }
  e = cudaEventRecord(c.ev_join, sd);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(st, c.ev_join, 0);
  if (e != cudaSuccess) return cuda_fail(c, e, "join");
  return FIZI_OK;
}

void destroy_graphs(Ctx& c) {
  for (auto& g : c.graphs)
    for (auto x : g.exec)
      if (x) cudaGraphExecDestroy(x);
  c.graphs.clear();
}

// Run one part: replay (capturing on first use) the graph of this plan's
// shape, or launch directly (profiling, or graphs disabled).
int run_part(Ctx& c, const CallPlan& pl, int part, cudaStream_t st) {
  const bool graph = c.use_graphs && !c.prof && !(pl.masks && !pl.fused_mask);
  if (!graph) return enqueue_part(c, pl, part, st);
  std::vector<uint32_t> key = {(uint32_t)part, pl.n, (uint32_t)(pl.fold + 2), (uint32_t)pl.premask,
                               (uint32_t)pl.fused_mask, (uint32_t)pl.morphmask, (uint32_t)pl.relearn};
  for (const SubBatch& b : pl.subs) {
    key.push_back(b.n);
    key.push_back(b.g0);
    key.push_back(b.ng);
  }
  Ctx::GraphEntry* ent = nullptr;
  for (auto& g : c.graphs)
    if (g.key == key) { ent = &g; break; }
  if (!ent) {
    constexpr size_t kMaxGraphs = 16;
    if (c.graphs.size() >= kMaxGraphs) {               // evict the least recently used
      size_t lru = 0;
      for (size_t i = 1; i < c.graphs.size(); i++)
        if (c.graphs[i].used < c.graphs[lru].used) lru = i;
      for (auto x : c.graphs[lru].exec)
        if (x) cudaGraphExecDestroy(x);
      c.graphs.erase(c.graphs.begin() + (long)lru);
    }
    c.graphs.emplace_back();
    ent = &c.graphs.back();
    ent->key = key;
  }
  ent->used = ++c.graph_clock;
  if (!ent->exec[pl.slot]) {
    // a new call shape: capture it for every slot now (the slots' pointers
    // differ), so that later calls of this shape never stall on a capture
    for (uint32_t s = 0; s < fizi::kSlots; s++) {
      if (ent->exec[s]) continue;
      select_slot(c, s);
      CallPlan ps = pl;
      ps.slot = s;
      const uint64_t l0 = c.launches;
      cudaError_t e = cudaStreamBeginCapture(c.cap, cudaStreamCaptureModeThreadLocal);
      if (e != cudaSuccess) { select_slot(c, pl.slot); return cuda_fail(c, e, "cudaStreamBeginCapture"); }
      const int rc = enqueue_part(c, ps, part, c.cap);
      cudaGraph_t g = nullptr;
      e = cudaStreamEndCapture(c.cap, &g);
      if (rc) {
        if (g) cudaGraphDestroy(g);
        select_slot(c, pl.slot);
        return rc;
      }
      if (e == cudaSuccess) e = cudaGraphInstantiate(&ent->exec[s], g, 0);
      if (g) cudaGraphDestroy(g);
      ent->kernels = c.launches - l0;
      c.launches = l0;
      if (e != cudaSuccess) { select_slot(c, pl.slot); return cuda_fail(c, e, "graph capture"); }
    }
    select_slot(c, pl.slot);
  }
  cudaError_t e = cudaGraphLaunch(ent->exec[pl.slot], st);
  if (e != cudaSuccess) return cuda_fail(c, e, "cudaGraphLaunch");
  c.launches += ent->kernels;
  return FIZI_OK;
}

int check_call(Ctx& c, const uint32_t* sof, const uint8_t* frames, uint32_t n, uint32_t w,
               uint32_t h, fizi_result* results) {
  if (c.sticky) return fail(c, FIZI_E_CUDA, "context has a sticky CUDA error: " + c.err);
  if (w != c.W || h != c.H) return fail(c, FIZI_E_DIMS, "frame dimensions differ from the context");
  if (n > c.max_batch) return fail(c, FIZI_E_CAPACITY, "n exceeds max_batch");
  if (n == 0) return FIZI_OK;
  if (!sof || !frames || !results) return fail(c, FIZI_E_ARG, "NULL pointer argument");
  if (c.fast && (reinterpret_cast<uintptr_t>(frames) & 15u))
    return fail(c, FIZI_E_ARG, "frames_dev must be 16-byte aligned");
  for (uint32_t i = 0; i < n; i++) {
    if (sof[i] >= c.n_streams) return fail(c, FIZI_E_CAPACITY, "stream id >= n_streams");
    if (!c.env_valid[sof[i]])
      return fail(c, FIZI_E_NOMODEL, "stream " + std::to_string(sof[i]) + " has no background model");
  }
  return FIZI_OK;
}

int run_call(Ctx& c, const uint32_t* sof, const uint8_t* frames, uint32_t n, const int64_t* t,
             uint8_t* masks, fizi_result* res, bool track, cudaStream_t st) {
  CallPlan pl;
  pl.n = n;
  bool single = true;
  for (uint32_t i = 1; i < n && single; i++) single = sof[i] == sof[0];
  pl.fold = !track ? -2 : (single ? (int)sof[0] : -1);
  // the u8 mask is written by the labelling kernel when the register-pipelined
  // morphology runs; otherwise it is expanded from the final bit mask
  pl.fused_mask = c.fast && c.P <= 128 && c.p.se_radius <= 4;
  pl.premask = masks && pl.fused_mask && !c.mask_by_morph;
  pl.morphmask = masks && pl.fused_mask && c.mask_by_morph;
  pl.masks = masks;
  // NEXT-1: a call with a relearning stream runs joined (the model swap
  // orders the next call's segmentation after this call's relearning)
  c.rl_active = false;
  if (!c.rl_enabled.empty())
    for (uint32_t i = 0; i < n && !c.rl_active; i++) c.rl_active = c.rl_enabled[sof[i]] != 0;
  pl.relearn = c.rl_active;
  const bool pipelined = c.pipeline && !c.p.debug && !pl.relearn;
  pl.slot = c.pinned_next;
  c.pinned_next = (c.pinned_next + 1) % fizi::kSlots;
  const auto h0 = std::chrono::steady_clock::now();
  cudaError_t e = cudaEventSynchronize(c.slot_upload[pl.slot] ? c.slot_upload[pl.slot]
                                                               : c.pinned_ev[pl.slot]);   // slot's last upload consumed
  const auto h1 = std::chrono::steady_clock::now();
  c.host_sync_ns += (uint64_t)std::chrono::duration_cast<std::chrono::nanoseconds>(h1 - h0).count();
  if (e != cudaSuccess) return cuda_fail(c, e, "cudaEventSynchronize");
  fizi::CallPtrs cp{frames, pl.fused_mask ? masks : nullptr, res, n,
                    single ? (int64_t)sof[0] : -1, c.call_counter++, c.tl};
  const uint32_t sub_frames = c.sub_frames;
  if (pipelined || pl.relearn) c.sub_frames = 65535;  // one sub-batch (the tail is the overlap / the relearn plan sees every frame)
  fill_call(c, pl.slot, cp, sof, t, n, pl.subs);
  c.sub_frames = sub_frames;
  select_slot(c, pl.slot);
  // the slot's previous call (kSlots calls back) must be complete
  e = cudaStreamWaitEvent(st, c.ev_tail[pl.slot], 0);
  if (e != cudaSuccess) return cuda_fail(c, e, "cudaStreamWaitEvent");
  int rc;
  if (!pipelined) {
    e = join_tail(c, st);                               // earlier pipelined tails (fold order)
    if (e != cudaSuccess) return cuda_fail(c, e, "join");
    rc = run_part(c, pl, kWhole, st);
    if (rc) return rc;
    e = cudaEventRecord(c.pinned_ev[pl.slot], st);
    if (e == cudaSuccess) e = cudaEventRecord(c.ev_tail[pl.slot], st);
    c.slot_upload[pl.slot] = c.pinned_ev[pl.slot];
    if (e != cudaSuccess) return cuda_fail(c, e, "cudaEventRecord");
  } else {
    // Four graph launches per call, each on a stream that runs its stage
    // in call order: the head (table upload, counter clear, fused
    // segmentation) on the head stream; the per-pixel words + LUT re-test on
    // the side stream; the morphology (+ u8 mask rows) on the morphology
    // stream; the labelling (+ the fused a8 fold) on the labelling stream.
    // So call k's labelling, call k+1's morphology, call k+2's per-pixel
    // words and call k+3's segmentation can run at once
    // (every buffer a stage writes is per slot; the labelling scratch and the
    // tracker state are only touched by the in-order labelling stage).  st
    // itself is not joined (fizi_flush does that); st already waits for the
    // slot's previous call (above), and every stage is ordered after st.
    // The slot's table upload and counter clear run ahead on the prep
    // stream, as soon as the slot's previous call is done, so the
    // segmentation starts the moment the previous one ends.
    cudaStream_t hs = c.head;
    e = cudaStreamWaitEvent(c.prep, c.ev_tail[pl.slot], 0);
    if (e != cudaSuccess) return cuda_fail(c, e, "prep");
    rc = enqueue_head(c, pl, c.prep);
    if (rc) return rc;
    e = cudaEventRecord(c.ev_prep[pl.slot], c.prep);   // (also: the pinned table consumed)
    if (e == cudaSuccess) e = cudaEventRecord(c.ev_in[pl.slot], st);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(hs, c.ev_in[pl.slot], 0);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(hs, c.ev_prep[pl.slot], 0);
    if (e != cudaSuccess) return cuda_fail(c, e, "fork");
    rc = run_part(c, pl, kHead, hs);
    if (rc) return rc;
    e = cudaEventRecord(c.ev_head[pl.slot], hs);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(c.side, c.ev_head[pl.slot], 0);
    if (e != cudaSuccess) return cuda_fail(c, e, "fork");
    rc = run_part(c, pl, kTail, c.side);
    if (rc) return rc;
    e = cudaEventRecord(c.ev_words[pl.slot], c.side);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(c.morphst, c.ev_words[pl.slot], 0);
    if (e != cudaSuccess) return cuda_fail(c, e, "fork");
    rc = run_part(c, pl, kTailMorph, c.morphst);
    if (rc) return rc;
    e = cudaEventRecord(c.ev_morph[pl.slot], c.morphst);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(c.cclst, c.ev_morph[pl.slot], 0);
    if (e != cudaSuccess) return cuda_fail(c, e, "fork");
    rc = run_part(c, pl, kTailCcl, c.cclst);
    if (rc) return rc;
    e = cudaEventRecord(c.ev_tail[pl.slot], c.cclst);
    if (e != cudaSuccess) return cuda_fail(c, e, "cudaEventRecord");
    c.slot_upload[pl.slot] = c.ev_prep[pl.slot];
  }
  c.tail_pending = true;
  c.host_call_ns += (uint64_t)std::chrono::duration_cast<std::chrono::nanoseconds>(
                        std::chrono::steady_clock::now() - h0).count();
  c.last_slot = pl.slot;
  c.last_frames = frames;
  c.last_n = n;
  return FIZI_OK;
}

int check_times(Ctx& c, const uint32_t* sof, const int64_t* t, uint32_t n) {
  if (!t) return fail(c, FIZI_E_ARG, "t_ms_host is NULL");
  std::vector<int64_t> last(c.last_t);
  std::vector<uint8_t> has(c.has_t);
  for (uint32_t i = 0; i < n; i++) {
    const uint32_t s = sof[i];
    if (has[s] && t[i] < last[s])
      return fail(c, FIZI_E_TIME, "decreasing timestamp in stream " + std::to_string(s));
    last[s] = t[i];
    has[s] = 1;
  }
  return FIZI_OK;
}

void commit_times(Ctx& c, const uint32_t* sof, const int64_t* t, uint32_t n) {
  for (uint32_t i = 0; i < n; i++) {
    c.last_t[sof[i]] = t[i];
    c.has_t[sof[i]] = 1;
  }
}

}  // namespace

extern "C" {

int fizi_params_default(fizi_params* p, uint32_t width, uint32_t height) {
  if (!p) return FIZI_E_ARG;
  std::memset(p, 0, sizeof(*p));
  p->width = width;
  p->height = height;
  p->gray_tol_S = 30;
  p->hue_lo_deg = 340;
  p->hue_hi_deg = 25;
  p->se_radius = 1;
  p->min_blob_ppm = 5000;
  p->luma_target = 128;
  p->luma_lo = 60;
  p->luma_hi = 190;
  p->gamma_min = 0.4;
  p->gamma_max = 2.5;
  p->beta = 0.5;
  p->dwell_radius_px = 15.0;
  p->dwell_time_ms = 800;
  p->lost_timeout_ms = 500;
  p->debug = 0;
  return FIZI_OK;
}

int fizi_create(const fizi_params* params, int cuda_device, uint32_t n_streams,
                uint32_t max_batch, fizi_ctx** out) {
  if (!out) return FIZI_E_ARG;
  *out = nullptr;
  std::string why;
  int rc = validate_params(params, why);
  if (rc) return rc;
  if (n_streams < 1 || max_batch < 1 || max_batch > 65535) return FIZI_E_ARG;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || cuda_device < 0 || cuda_device >= ndev) {
    cudaGetLastError();
    return FIZI_E_CUDA;
  }
  DeviceGuard guard(cuda_device);
  fizi_ctx* x = new (std::nothrow) fizi_ctx();
  if (!x) return FIZI_E_OOM;
  Ctx& c = x->c;
  c.p = *params;
  c.device = cuda_device;
  c.n_streams = n_streams;
  c.max_batch = max_batch;
  c.W = params->width;
  c.H = params->height;
  c.P = (c.W + 31) / 32;
  c.N = (uint64_t)c.W * c.H;
  c.fast = (c.W % 32) == 0;
  c.nchunks = (uint32_t)((c.N + fizi::kChunkPx - 1) / fizi::kChunkPx);
  c.env_plane = c.fast ? (uint64_t)c.nchunks * fizi::kChunkBytes : c.N * 3;
  c.cap_runs = (uint64_t)c.H * ((c.W + 1) / 2);
  cudaDeviceGetAttribute(&c.sms, cudaDevAttrMultiProcessorCount, cuda_device);
  c.morph_tr = fizi::morph_tile_rows(c, fizi::kMorphSmem);
  // clean chunks of the merged mask are left unwritten when the register-
  // pipelined morphology (which reads the dirty bitmap) runs and no debug
  // stage needs the full mask
  c.use_dirty = c.fast && c.P <= 128 && params->se_radius <= 4 && !params->debug;
  if (c.morph_tr == 0) {
    delete x;
    return FIZI_E_ARG;
  }
  const uint64_t mb = max_batch;
  const uint64_t wpf = (uint64_t)c.H * c.P;
  cudaError_t e = cudaSuccess;
  auto A = [&](cudaError_t r) { if (e == cudaSuccess) e = r; };
  A(dalloc(&c.env, (uint64_t)n_streams * 2 * c.env_plane));
  A(dalloc(&c.lut, 256 * 256));
  A(dalloc(&c.gamma_tab, 256 * sizeof(double)));
  A(dalloc(&c.corr_tab, 256));
  A(dalloc(&c.skin_tab, (1u << 19) * 4));
  // per-call counters and flags: one block, cleared by one memset per call
  c.dirty_words = (c.nchunks + 31) / 32;
  {
    const uint64_t zb = mb * 8 + mb * 4 * 3 + fizi::kMaxSub * 4 + fizi::kMaxSub * (mb + 2) * 4 +
                        fizi::kMaxSub * (mb + 1) * 4 + fizi::kMaxSub * 4 * 2 + mb * c.dirty_words * 4;
    c.zero_bytes = zb;
    for (uint32_t i = 0; i < fizi::kSlots; i++) A(dalloc(&c.zero_blocks[i], zb));
  }

  for (uint32_t i = 0; i < fizi::kSlots; i++) A(dalloc(&c.bitAs[i], mb * wpf * 4));
  for (uint32_t i = 0; i < fizi::kSlots; i++) {
    A(dalloc(&c.bitOs[i], mb * wpf * 4));
    A(dalloc(&c.row_cnts[i], mb * c.H * 4));
    A(dalloc(&c.row_bases[i], mb * c.H * 4));
    A(dalloc(&c.runss[i], mb * c.cap_runs * sizeof(fizi::Run)));
  }
  if (c.p.debug) A(dalloc(&c.bitOC, mb * wpf * 4));
  if (c.fast)
    for (uint32_t i = 0; i < fizi::kSlots; i++)
      A(dalloc(&c.slow_itemss[i], mb * c.nchunks * 16 * sizeof(unsigned long long)));
  A(dalloc(&c.parent, mb * c.cap_runs * 4));
  A(dalloc(&c.stats, mb * c.cap_runs * sizeof(fizi::RootStats)));
  const size_t table_bytes = sizeof(fizi::CallPtrs) + mb * 8 + mb * 4 * 2 + (mb + 1) * 4;
  for (uint32_t i = 0; i < fizi::kSlots; i++) A(dalloc(&c.calls[i], table_bytes));
  A(dalloc(&c.tstate, (uint64_t)n_streams * sizeof(fizi::TrackState)));
  A(dalloc(&c.dstate, (uint64_t)n_streams * sizeof(fizi::DriveState)));
  A(dalloc(&c.prev_mean, (uint64_t)n_streams * sizeof(int32_t)));
  A(dalloc(&c.rstate, (uint64_t)n_streams * sizeof(fizi::RelearnState)));
  A(dalloc(&c.rl_role, mb * 4));
  A(dalloc(&c.rl_pair, mb * 4));
  A(dalloc(&c.rl_env, mb * 8));
  A(dalloc(&c.rl_list, (mb + 1) * 4));
  A(dalloc(&c.rl_pairs, mb * 16));
  A(dalloc(&c.rl_counts, (2 + 2 * (uint64_t)n_streams) * 4));
  A(dalloc(&c.hstate, (uint64_t)n_streams * sizeof(fizi::HitState)));
  for (uint32_t i = 0; i < fizi::kSlots && e == cudaSuccess; i++) {
    e = cudaMallocHost(reinterpret_cast<void**>(&c.pinned[i]), table_bytes);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c.pinned_ev[i], cudaEventDisableTiming);
  }
  if (e == cudaSuccess) {
    // the tail runs at the highest priority: its CTAs take SM slots as the
    // next call's segmentation CTAs retire
    int lo_prio = 0, hi_prio = 0;
    cudaDeviceGetStreamPriorityRange(&lo_prio, &hi_prio);
    // stream priorities: head (segmentation) > tail (mask clear, per-pixel
    // words, morphology, labelling, fold) > the caller's streams.  Experiment
    // switches: FIZI_SIDE_PRIO=0/1/2 -> tail at lowest / highest / one below
    // highest (default 2); FIZI_HEAD_PRIO=0 -> head at lowest.
    const int mid_prio = hi_prio < lo_prio ? hi_prio + 1 : hi_prio;
    const char* spe = getenv("FIZI_SIDE_PRIO");
    const int side_prio = !spe ? mid_prio : atoi(spe) == 0 ? lo_prio : atoi(spe) == 1 ? hi_prio : mid_prio;
    e = cudaStreamCreateWithPriority(&c.side, cudaStreamNonBlocking,
                                     side_prio);
    if (e == cudaSuccess)
      e = cudaStreamCreateWithPriority(&c.side2, cudaStreamNonBlocking,
                                       side_prio);
    if (e == cudaSuccess)
      e = cudaStreamCreateWithPriority(&c.side3, cudaStreamNonBlocking,
                                       side_prio);
    for (uint32_t i = 0; i < fizi::kSlots && e == cudaSuccess; i++)
      e = cudaEventCreateWithFlags(&c.ev_in[i], cudaEventDisableTiming);
    const char* hp = getenv("FIZI_HEAD_PRIO");
    if (e == cudaSuccess)
      e = cudaStreamCreateWithPriority(&c.head, cudaStreamNonBlocking,
                                       (hp && atoi(hp) == 0) ? lo_prio : hi_prio);
    if (e == cudaSuccess) e = cudaStreamCreateWithPriority(&c.cclst, cudaStreamNonBlocking, side_prio);
    if (e == cudaSuccess) e = cudaStreamCreateWithPriority(&c.prep, cudaStreamNonBlocking, hi_prio);
    for (uint32_t i = 0; i < fizi::kSlots && e == cudaSuccess; i++)
      e = cudaEventCreateWithFlags(&c.ev_prep[i], cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaStreamCreateWithPriority(&c.morphst, cudaStreamNonBlocking, side_prio);
    for (cudaEvent_t* ev : {&c.ev_zfork, &c.ev_zjoin, &c.ev_hfork, &c.ev_hjoin})
      if (e == cudaSuccess) e = cudaEventCreateWithFlags(ev, cudaEventDisableTiming);
  }
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&c.cap, cudaStreamNonBlocking);
  for (uint32_t k = 0; k < fizi::kMaxSub && e == cudaSuccess; k++)
    e = cudaEventCreateWithFlags(&c.ev_seg[k], cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c.ev_join, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c.ev_start, cudaEventDisableTiming);
  for (uint32_t i = 0; i < fizi::kSlots && e == cudaSuccess; i++) {
    e = cudaEventCreateWithFlags(&c.ev_head[i], cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c.ev_morph[i], cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c.ev_words[i], cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c.ev_tail[i], cudaEventDisableTiming);
  }
  c.use_graphs = getenv("FIZI_NO_GRAPH") == nullptr;
  if (const char* mm = getenv("FIZI_MASK_MODE"))       // experiment switch: zero | morph
    c.mask_by_morph = std::strcmp(mm, "zero") != 0;
  if (const char* gm = getenv("FIZI_GROUP")) {          // experiment switch (1..32)
    const int g = atoi(gm);
    if (g >= 1 && g <= (int)fizi::kFrameGroup) c.group_max = (uint32_t)g;
  }
  if (getenv("FIZI_TIMELINE") && e == cudaSuccess) {
    const size_t tb = 2ull * fizi::kTlKinds * fizi::kTlCalls * 8;
    e = cudaMalloc(reinterpret_cast<void**>(&c.tl), tb);
    if (e == cudaSuccess) e = cudaMemset(c.tl, 0xFF, tb / 2);
    if (e == cudaSuccess) e = cudaMemset(c.tl + fizi::kTlKinds * fizi::kTlCalls, 0, tb / 2);
  }
  if (const char* sf = getenv("FIZI_SUB_FRAMES")) c.sub_frames = (uint32_t)atoi(sf) > 0 ? (uint32_t)atoi(sf) : 65535;
  if (e != cudaSuccess) {
    cudaGetLastError();
    free_all(c);
    delete x;
    return FIZI_E_OOM;
  }
  c.pinned_bytes = table_bytes;
  select_slot(c, 0);
  c.env_valid.assign(n_streams, 0);
  c.last_t.assign(n_streams, 0);
  c.has_t.assign(n_streams, 0);
  e = fizi::init_segment(c);
  if (e == cudaSuccess) e = fizi::init_morph(c);
  if (e == cudaSuccess) e = fizi::init_ccl(c);
  if (e == cudaSuccess) e = cudaMemset(c.env, 0, (uint64_t)n_streams * 2 * c.env_plane);
  if (e == cudaSuccess) e = cudaMemset(c.dstate, 0, (uint64_t)n_streams * sizeof(fizi::DriveState));
  if (e == cudaSuccess) e = cudaMemset(c.rstate, 0, (uint64_t)n_streams * sizeof(fizi::RelearnState));
  c.rl_enabled.assign(n_streams, 0);
  c.rl_mem.assign(n_streams, nullptr);
  if (e == cudaSuccess) e = fizi::launch_relearn_reset(c, 0, n_streams, 0);
  if (e == cudaSuccess) e = fizi::launch_lut_table(c, 0);
  if (e == cudaSuccess) e = fizi::launch_skin_table(c, 0);
  if (e == cudaSuccess) e = fizi::launch_tstate_reset(c, 0, n_streams, 0);
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    cudaGetLastError();
    free_all(c);
    delete x;
    return FIZI_E_CUDA;
  }
  *out = x;
  return FIZI_OK;
}

int fizi_learn_background(fizi_ctx* ctx, uint32_t stream, const uint8_t* frames_dev,
                          uint32_t n_frames, uint32_t width, uint32_t height, uint8_t margin,
                          fizi_stream_t cuda_stream) {
  if (!ctx) return FIZI_E_ARG;
  Ctx& c = ctx->c;
  if (c.sticky) return fail(c, FIZI_E_CUDA, "context has a sticky CUDA error: " + c.err);
  if (stream >= c.n_streams) return fail(c, FIZI_E_CAPACITY, "stream id >= n_streams");
  if (n_frames == 0) return fail(c, FIZI_E_EMPTY, "learning needs at least one frame (S:139)");
  if (width != c.W || height != c.H) return fail(c, FIZI_E_DIMS, "frame dimensions differ from the context");
  if (!frames_dev) return fail(c, FIZI_E_ARG, "frames_dev is NULL");
  if (c.fast && (reinterpret_cast<uintptr_t>(frames_dev) & 15u))
    return fail(c, FIZI_E_ARG, "frames_dev must be 16-byte aligned");
  DeviceGuard guard(c.device);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(cuda_stream);
  cudaError_t e = join_tail(c, st);                   // pipelined tails read the envelope
  if (e != cudaSuccess) return cuda_fail(c, e, "join");
  e = fizi::launch_learn(c, stream, frames_dev, n_frames, margin, st);
  if (e != cudaSuccess) return cuda_fail(c, e, "learn");
  e = fizi::launch_tstate_reset(c, stream, 1, st);
  if (e == cudaSuccess) e = fizi::launch_relearn_reset(c, stream, 1, st);
  if (e == cudaSuccess && c.rl_enabled[stream])          // a new model: relearning starts over
    e = fizi::launch_relearn_state(c, stream, c.rl_state_host[stream], st);
  if (e != cudaSuccess) return cuda_fail(c, e, "tracker reset");
  c.env_valid[stream] = 1;
  c.has_t[stream] = 0;
  return FIZI_OK;
}

int fizi_segment_frames(fizi_ctx* ctx, const uint32_t* sof, const uint8_t* frames_dev, uint32_t n,
                        uint32_t width, uint32_t height, const int64_t* t_ms, uint8_t* masks_dev,
                        fizi_result* results_dev, fizi_stream_t cuda_stream) {
  if (!ctx) return FIZI_E_ARG;
  Ctx& c = ctx->c;
  int rc = check_call(c, sof, frames_dev, n, width, height, results_dev);
  if (rc || n == 0) return rc;
  DeviceGuard guard(c.device);
  return run_call(c, sof, frames_dev, n, t_ms, masks_dev, results_dev, false,
                  reinterpret_cast<cudaStream_t>(cuda_stream));
}

int fizi_process_frames(fizi_ctx* ctx, const uint32_t* sof, const uint8_t* frames_dev, uint32_t n,
                        uint32_t width, uint32_t height, const int64_t* t_ms, uint8_t* masks_dev,
                        fizi_result* results_dev, fizi_stream_t cuda_stream) {
  if (!ctx) return FIZI_E_ARG;
  Ctx& c = ctx->c;
  int rc = check_call(c, sof, frames_dev, n, width, height, results_dev);
  if (rc || n == 0) return rc;
  rc = check_times(c, sof, t_ms, n);
  if (rc) return rc;
  DeviceGuard guard(c.device);
  rc = run_call(c, sof, frames_dev, n, t_ms, masks_dev, results_dev, true,
                reinterpret_cast<cudaStream_t>(cuda_stream));
  if (rc == FIZI_OK) commit_times(c, sof, t_ms, n);
  return rc;
}

int fizi_track(fizi_ctx* ctx, uint32_t stream, fizi_result* results_dev, uint32_t n,
               fizi_stream_t cuda_stream) {
  if (!ctx) return FIZI_E_ARG;
  Ctx& c = ctx->c;
  if (c.sticky) return fail(c, FIZI_E_CUDA, "context has a sticky CUDA error: " + c.err);
  if (stream >= c.n_streams) return fail(c, FIZI_E_CAPACITY, "stream id >= n_streams");
  if (n == 0) return FIZI_OK;
  if (!results_dev) return fail(c, FIZI_E_ARG, "results_dev is NULL");
  DeviceGuard guard(c.device);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(cuda_stream);
  cudaError_t e = join_tail(c, st);                   // fold order after pipelined tails
  if (e != cudaSuccess) return cuda_fail(c, e, "join");
  prof_begin(c, st);
  e = fizi::launch_track_stream(c, stream, results_dev, n, st);
  prof_end(c, FIZI_PROF_TRACK, st);
  if (e != cudaSuccess) return cuda_fail(c, e, "track");
  return FIZI_OK;
}

int fizi_track_runs(fizi_ctx* ctx, uint32_t stream, fizi_result* results_dev,
                    const uint32_t* run_off, const uint32_t* run_len, uint32_t n_runs,
                    fizi_stream_t cuda_stream) {
  if (!ctx) return FIZI_E_ARG;
  Ctx& c = ctx->c;
  if (c.sticky) return fail(c, FIZI_E_CUDA, "context has a sticky CUDA error: " + c.err);
  if (stream >= c.n_streams) return fail(c, FIZI_E_CAPACITY, "stream id >= n_streams");
  if (n_runs > fizi::kMaxTrackRuns) return fail(c, FIZI_E_ARG, "n_runs must be <= 256");
  if (n_runs == 0) return FIZI_OK;
  if (!results_dev || !run_off || !run_len) return fail(c, FIZI_E_ARG, "NULL pointer argument");
  DeviceGuard guard(c.device);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(cuda_stream);
  cudaError_t e = join_tail(c, st);                   // fold order after pipelined tails
  prof_begin(c, st);
  if (e == cudaSuccess) e = fizi::launch_track_runs(c, stream, results_dev, run_off, run_len, n_runs, st);
  prof_end(c, FIZI_PROF_TRACK, st);
  if (e != cudaSuccess) return cuda_fail(c, e, "track runs");
  return FIZI_OK;
}

int fizi_process_frames_host(fizi_ctx* ctx, const uint32_t* sof, const uint8_t* frames_host,
                             uint32_t n, uint32_t width, uint32_t height, const int64_t* t_ms,
                             uint8_t* masks_host, fizi_result* results_host,
                             fizi_stream_t cuda_stream) {
  if (!ctx) return FIZI_E_ARG;
  Ctx& c = ctx->c;
  if (c.sticky) return fail(c, FIZI_E_CUDA, "context has a sticky CUDA error: " + c.err);
  if (n == 0) return FIZI_OK;
  if (!frames_host || !results_host) return fail(c, FIZI_E_ARG, "NULL pointer argument");
  if (width != c.W || height != c.H) return fail(c, FIZI_E_DIMS, "frame dimensions differ from the context");
  if (n > c.max_batch) return fail(c, FIZI_E_CAPACITY, "n exceeds max_batch");
  DeviceGuard guard(c.device);
  cudaError_t e = cudaSuccess;
  if (!c.stage_frames) {
    e = dalloc(&c.stage_frames, (uint64_t)c.max_batch * c.N * 3);
    if (e == cudaSuccess) e = dalloc(&c.stage_masks, (uint64_t)c.max_batch * c.N);
    if (e == cudaSuccess) e = dalloc(&c.stage_results, (uint64_t)c.max_batch * sizeof(fizi_result));
    if (e == cudaSuccess)
      e = cudaMallocHost(reinterpret_cast<void**>(&c.pinned_results),
                         (uint64_t)c.max_batch * sizeof(fizi_result));
    if (e != cudaSuccess) {
      cudaGetLastError();
      return fail(c, FIZI_E_OOM, "staging allocation failed");
    }
  }
  cudaStream_t st = reinterpret_cast<cudaStream_t>(cuda_stream);
  // The batch moves in chunks of ~32 MB of frames: chunk j+1 is copied in
  // (copy stream h2d) while chunk j is processed (st) and chunk j-1's masks
  // and records are copied out (copy stream d2h), so the two PCIe directions
  // and the path overlap.  Chunks are processed in order on st, so the
  // tracker sees the frames in index order.
  const uint64_t fb = c.N * 3;
  static const uint64_t chunk_mb = getenv("FIZI_HOST_CHUNK_MB") ? (uint64_t)atoi(getenv("FIZI_HOST_CHUNK_MB")) : 32;
  const uint32_t m = std::max<uint32_t>(1u, std::min<uint64_t>(n, (chunk_mb << 20) / fb));
  const uint32_t nchunk = (n + m - 1) / m;
  if (!c.h2d) {
    e = cudaStreamCreateWithFlags(&c.h2d, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&c.d2h, cudaStreamNonBlocking);
    if (e != cudaSuccess) return cuda_fail(c, e, "copy streams");
  }
  while (c.host_ev.size() < 2ull * nchunk + 1) {
    cudaEvent_t ev = nullptr;
    e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
    if (e != cudaSuccess) return cuda_fail(c, e, "cudaEventCreate");
    c.host_ev.push_back(ev);
  }
  // a pageable mask buffer is filled by one copy at the end (a pageable
  // destination makes every copy synchronous)
  bool masks_pinned = false;
  if (masks_host) {
    cudaPointerAttributes pa{};
    masks_pinned = cudaPointerGetAttributes(&pa, masks_host) == cudaSuccess &&
                   pa.type == cudaMemoryTypeHost;
    cudaGetLastError();
  }
  // the copies start after the caller's earlier work on st
  e = cudaEventRecord(c.host_ev[2 * nchunk], st);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(c.h2d, c.host_ev[2 * nchunk], 0);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(c.d2h, c.host_ev[2 * nchunk], 0);
  if (e != cudaSuccess) return cuda_fail(c, e, "fork");
  // the chunks run as pipelined calls (each chunk's tail overlaps the next
  // chunk's segmentation; outputs are complete when this entry returns), and
  // each chunk's read-back waits for that chunk's last stage only
  const bool pipeline_saved = c.pipeline;
  c.pipeline = true;
  struct Restore {
    Ctx& c;
    bool v;
    ~Restore() { c.pipeline = v; }
  } restore{c, pipeline_saved};
  for (uint32_t j = 0; j < nchunk; j++) {
    const uint32_t j0 = j * m, mj = std::min(m, n - j0);
    cudaEvent_t ev_in = c.host_ev[2 * j];
    e = cudaMemcpyAsync(c.stage_frames + (uint64_t)j0 * fb, frames_host + (uint64_t)j0 * fb,
                        (size_t)mj * fb, cudaMemcpyHostToDevice, c.h2d);
    if (e == cudaSuccess) e = cudaEventRecord(ev_in, c.h2d);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(st, ev_in, 0);
    if (e != cudaSuccess) return cuda_fail(c, e, "H2D frames");
    int rc = fizi_process_frames(ctx, sof + j0, c.stage_frames + (uint64_t)j0 * fb, mj, width, height,
                                 t_ms ? t_ms + j0 : nullptr,
                                 masks_host ? c.stage_masks + (uint64_t)j0 * c.N : nullptr,
                                 c.stage_results + j0, cuda_stream);
    if (rc) return rc;
    e = cudaStreamWaitEvent(c.d2h, c.ev_tail[c.last_slot], 0);   // this chunk's outputs
    if (e != cudaSuccess) return cuda_fail(c, e, "join");
    if (masks_pinned) {
      e = cudaMemcpyAsync(masks_host + (uint64_t)j0 * c.N, c.stage_masks + (uint64_t)j0 * c.N,
                          (size_t)mj * c.N, cudaMemcpyDeviceToHost, c.d2h);
      if (e != cudaSuccess) return cuda_fail(c, e, "D2H masks");
    }
    // records go through a pinned staging buffer (a pageable destination
    // would make the copy synchronous and serialise the chunks)
    e = cudaMemcpyAsync(c.pinned_results + j0, c.stage_results + j0, (size_t)mj * sizeof(fizi_result),
                        cudaMemcpyDeviceToHost, c.d2h);
    if (e != cudaSuccess) return cuda_fail(c, e, "D2H results");
  }
  if (masks_host && !masks_pinned) {
    e = cudaMemcpyAsync(masks_host, c.stage_masks, (size_t)n * c.N, cudaMemcpyDeviceToHost, c.d2h);
    if (e != cudaSuccess) return cuda_fail(c, e, "D2H masks");
  }
  e = join_tail(c, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(c.d2h);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return cuda_fail(c, e, "cudaStreamSynchronize");
  memcpy(results_host, c.pinned_results, (size_t)n * sizeof(fizi_result));
  for (uint32_t i = 0; i < n; i++) results_host[i].frame_idx = i;   // index in this call
  return FIZI_OK;
}

int fizi_reset_tracker(fizi_ctx* ctx, uint32_t stream, fizi_stream_t cuda_stream) {
  if (!ctx) return FIZI_E_ARG;
  Ctx& c = ctx->c;
  if (c.sticky) return fail(c, FIZI_E_CUDA, "context has a sticky CUDA error: " + c.err);
  if (stream >= c.n_streams) return fail(c, FIZI_E_CAPACITY, "stream id >= n_streams");
  DeviceGuard guard(c.device);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(cuda_stream);
  // every earlier fold of this stream (pipelined tails on the fold stream,
  // joined calls on their caller's stream) is ordered before the reset
  cudaError_t e = join_tail(c, st);
  if (e == cudaSuccess) e = fizi::launch_tstate_reset(c, stream, 1, st);
  if (e != cudaSuccess) return cuda_fail(c, e, "tracker reset");
  c.has_t[stream] = 0;
  return FIZI_OK;
}

int fizi_debug_stage(fizi_ctx* ctx, int stage, uint32_t frame, void* out_dev,
                     fizi_stream_t cuda_stream) {
  if (!ctx) return FIZI_E_ARG;
  Ctx& c = ctx->c;
  if (!c.p.debug) return fail(c, FIZI_E_ARG, "context was created with debug = 0");
  if (!out_dev) return fail(c, FIZI_E_ARG, "out_dev is NULL");
  if (frame >= c.last_n) return fail(c, FIZI_E_ARG, "frame index beyond the last call");
  if (stage < FIZI_STAGE_R1 || stage > FIZI_STAGE_CONTOUR) return fail(c, FIZI_E_ARG, "bad stage");
  DeviceGuard guard(c.device);
  cudaError_t e = join_tail(c, reinterpret_cast<cudaStream_t>(cuda_stream));
  if (e == cudaSuccess)
    e = fizi::launch_debug_stage(c, stage, frame, out_dev, reinterpret_cast<cudaStream_t>(cuda_stream));
  if (e != cudaSuccess) return cuda_fail(c, e, "debug stage");
  return FIZI_OK;
}

int fizi_get_lut_table(fizi_ctx* ctx, uint8_t* lut_dev, double* gamma_dev, uint8_t* corrected_dev,
                       fizi_stream_t cuda_stream) {
  if (!ctx) return FIZI_E_ARG;
  Ctx& c = ctx->c;
  if (c.sticky) return fail(c, FIZI_E_CUDA, "context has a sticky CUDA error: " + c.err);
  DeviceGuard guard(c.device);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(cuda_stream);
  cudaError_t e = cudaSuccess;
  if (lut_dev) e = cudaMemcpyAsync(lut_dev, c.lut, 256 * 256, cudaMemcpyDeviceToDevice, st);
  if (e == cudaSuccess && gamma_dev)
    e = cudaMemcpyAsync(gamma_dev, c.gamma_tab, 256 * sizeof(double), cudaMemcpyDeviceToDevice, st);
  if (e == cudaSuccess && corrected_dev)
    e = cudaMemcpyAsync(corrected_dev, c.corr_tab, 256, cudaMemcpyDeviceToDevice, st);
  if (e != cudaSuccess) return cuda_fail(c, e, "get_lut_table");
  return FIZI_OK;
}

int fizi_get_background(fizi_ctx* ctx, uint32_t stream, uint8_t* lo_dev, uint8_t* hi_dev,
                        fizi_stream_t cuda_stream) {
  if (!ctx) return FIZI_E_ARG;
  Ctx& c = ctx->c;
  if (stream >= c.n_streams) return fail(c, FIZI_E_CAPACITY, "stream id >= n_streams");
  if (!c.env_valid[stream]) return fail(c, FIZI_E_NOMODEL, "stream has no background model");
  if (!lo_dev || !hi_dev) return fail(c, FIZI_E_ARG, "NULL pointer argument");
  DeviceGuard guard(c.device);
  cudaError_t e = fizi::launch_env_export(c, stream, lo_dev, hi_dev, false, nullptr, nullptr,
                                          reinterpret_cast<cudaStream_t>(cuda_stream));
  if (e != cudaSuccess) return cuda_fail(c, e, "get_background");
  return FIZI_OK;
}

int fizi_set_background(fizi_ctx* ctx, uint32_t stream, const uint8_t* lo_dev,
                        const uint8_t* hi_dev, fizi_stream_t cuda_stream) {
  if (!ctx) return FIZI_E_ARG;
  Ctx& c = ctx->c;
  if (stream >= c.n_streams) return fail(c, FIZI_E_CAPACITY, "stream id >= n_streams");
  if (!lo_dev || !hi_dev) return fail(c, FIZI_E_ARG, "NULL pointer argument");
  DeviceGuard guard(c.device);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(cuda_stream);
  cudaError_t e = join_tail(c, st);
  if (e == cudaSuccess) e = fizi::launch_env_export(c, stream, nullptr, nullptr, true, lo_dev, hi_dev, st);
  if (e == cudaSuccess) e = fizi::launch_tstate_reset(c, stream, 1, st);
  if (e == cudaSuccess && c.rl_enabled[stream])          // a new model: relearning starts over
    e = fizi::launch_relearn_state(c, stream, c.rl_state_host[stream], st);
  if (e != cudaSuccess) return cuda_fail(c, e, "set_background");
  c.env_valid[stream] = 1;
  c.has_t[stream] = 0;
  return FIZI_OK;
}

int fizi_set_zones(fizi_ctx* ctx, uint32_t stream, const fizi_zone* zones, uint32_t n_zones) {
  if (!ctx) return FIZI_E_ARG;
  Ctx& c = ctx->c;
  if (stream >= c.n_streams) return fail(c, FIZI_E_CAPACITY, "stream id >= n_streams");
  if (n_zones > fizi::kMaxZones) return fail(c, FIZI_E_CAPACITY, "more than 64 zones");
  if (n_zones && !zones) return fail(c, FIZI_E_ARG, "zones is NULL");
  fizi::HitState h;
  memset(&h, 0, sizeof(h));
  h.n_zones = n_zones;
  for (uint32_t k = 0; k < n_zones; k++) {
    const fizi_zone& z = zones[k];
    bool ok = false;
    if (z.kind == FIZI_ZONE_BUTTON || z.kind == FIZI_ZONE_SLIDER)
      ok = std::isfinite(z.x) && std::isfinite(z.y) && z.w > 0.0 && z.h > 0.0 &&
           std::isfinite(z.w) && std::isfinite(z.h);
    else if (z.kind == FIZI_ZONE_WHEEL)
      ok = std::isfinite(z.cx) && std::isfinite(z.cy) && z.r > 0.0 && std::isfinite(z.r) &&
           z.theta_max_deg > 0.0 && z.theta_max_deg <= 180.0;
    if (!ok) return fail(c, FIZI_E_ARG, "zone " + std::to_string(k) + ": bad kind or geometry");
    h.zones[k] = z;
  }
  DeviceGuard guard(c.device);
  cudaError_t e = cudaDeviceSynchronize();              // no hit test of this stream in flight
  if (e == cudaSuccess)
    e = cudaMemcpy(reinterpret_cast<fizi::HitState*>(c.hstate) + stream, &h, sizeof(h),
                   cudaMemcpyHostToDevice);
  if (e != cudaSuccess) return cuda_fail(c, e, "set_zones");
  if (c.n_zones.size() < c.n_streams) c.n_zones.assign(c.n_streams, 0);
  if (c.slider_zones.size() < c.n_streams) c.slider_zones.assign(c.n_streams, 0);
  c.n_zones[stream] = n_zones;
  c.slider_zones[stream] = 0;
  for (uint32_t k = 0; k < n_zones; k++)
    if (zones[k].kind == FIZI_ZONE_SLIDER) c.slider_zones[stream] |= 1ull << k;
  return FIZI_OK;
}

int fizi_hit_test(fizi_ctx* ctx, uint32_t stream, const fizi_result* results_dev, uint32_t n,
                  fizi_zone_event* events_dev, fizi_stream_t cuda_stream) {
  if (!ctx) return FIZI_E_ARG;
  Ctx& c = ctx->c;
  if (c.sticky) return fail(c, FIZI_E_CUDA, "context has a sticky CUDA error: " + c.err);
  if (stream >= c.n_streams) return fail(c, FIZI_E_CAPACITY, "stream id >= n_streams");
  if (c.n_zones.size() <= stream || c.n_zones[stream] == 0)
    return fail(c, FIZI_E_NOMODEL, "no layout set for this stream (fizi_set_zones)");
  if (n == 0) return FIZI_OK;
  if (!results_dev || !events_dev) return fail(c, FIZI_E_ARG, "NULL pointer argument");
  DeviceGuard guard(c.device);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(cuda_stream);
  cudaError_t e = join_tail(c, st);
  if (e == cudaSuccess) e = fizi::launch_hit_test(c, stream, results_dev, n, events_dev, st);
  if (e != cudaSuccess) return cuda_fail(c, e, "hit test");
  return FIZI_OK;
}

int fizi_relearn_flags(fizi_ctx* ctx, uint32_t stream, const fizi_result* results_dev, uint32_t n,
                       uint32_t threshold, uint8_t* flags_dev, fizi_stream_t cuda_stream) {
  if (!ctx) return FIZI_E_ARG;
  Ctx& c = ctx->c;
  if (c.sticky) return fail(c, FIZI_E_CUDA, "context has a sticky CUDA error: " + c.err);
  if (stream >= c.n_streams) return fail(c, FIZI_E_CAPACITY, "stream id >= n_streams");
  if (threshold > 255) return fail(c, FIZI_E_ARG, "threshold must be <= 255");
  if (n == 0) return FIZI_OK;
  if (!results_dev || !flags_dev) return fail(c, FIZI_E_ARG, "NULL pointer argument");
  DeviceGuard guard(c.device);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(cuda_stream);
  cudaError_t e = join_tail(c, st);
  if (e == cudaSuccess) e = fizi::launch_relearn_flags(c, stream, results_dev, n, threshold, flags_dev, st);
  if (e != cudaSuccess) return cuda_fail(c, e, "relearn flags");
  return FIZI_OK;
}

int fizi_set_relearn(fizi_ctx* ctx, uint32_t stream, uint32_t threshold, uint32_t n_frames,
                     uint8_t margin) {
  if (!ctx) return FIZI_E_ARG;
  Ctx& c = ctx->c;
  if (c.sticky) return fail(c, FIZI_E_CUDA, "context has a sticky CUDA error: " + c.err);
  if (stream >= c.n_streams) return fail(c, FIZI_E_CAPACITY, "stream id >= n_streams");
  if (threshold > 255) return fail(c, FIZI_E_ARG, "threshold must be <= 255");
  DeviceGuard guard(c.device);
  cudaError_t e = cudaDeviceSynchronize();              // no call of this stream in flight
  if (e != cudaSuccess) return cuda_fail(c, e, "set_relearn");
  if (c.rl_mem[stream]) {
    cudaFree(c.rl_mem[stream]);
    c.rl_mem[stream] = nullptr;
  }
  fizi::RelearnState v{};
  v.prev_mean = -1;
  if (n_frames > 0) {
    // models one call can complete: every one but a continued one needs a
    // trigger frame + n_frames learning frames of the call
    const uint32_t slots = (c.max_batch + n_frames) / (n_frames + 1) + 1;
    uint8_t* mem = nullptr;
    e = cudaMalloc(reinterpret_cast<void**>(&mem), (uint64_t)(slots + 1) * 2 * c.env_plane);
    if (e != cudaSuccess) {
      cudaGetLastError();
      return fail(c, FIZI_E_OOM, "relearn model pool allocation failed");
    }
    c.rl_mem[stream] = mem;
    v.enabled = 1;
    v.threshold = threshold;
    v.frames = n_frames;
    v.margin = margin;
    v.pool_slots = slots;
    v.pool = reinterpret_cast<uint64_t>(mem);
    v.acc = reinterpret_cast<uint64_t>(mem + (uint64_t)slots * 2 * c.env_plane);
  }
  e = fizi::launch_relearn_state(c, stream, v, 0);
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e != cudaSuccess) return cuda_fail(c, e, "set_relearn");
  c.rl_enabled[stream] = v.enabled ? 1 : 0;
  c.rl_state_host.resize(c.n_streams);
  c.rl_state_host[stream] = v;
  uint32_t pairs = 0, commits = 0;
  for (uint32_t s = 0; s < c.n_streams; s++)
    if (c.rl_enabled[s]) { pairs += c.rl_state_host[s].pool_slots; commits++; }
  c.rl_max_pairs = std::max(1u, std::min(pairs, c.max_batch));
  c.rl_max_commits = std::max(1u, commits);
  destroy_graphs(c);                                     // captured calls carry the launch grids
  return FIZI_OK;
}

int fizi_wheel_default(fizi_wheel* w, double cx, double cy, double radius) {
  if (!w) return FIZI_E_ARG;
  w->cx = cx;
  w->cy = cy;
  w->radius = radius;
  w->theta_max_deg = 90.0;
  w->inner = 0.6;
  w->outer = 1.4;
  w->dead_zone_deg = 3.0;
  w->hold_ms = 200;
  return FIZI_OK;
}

int fizi_set_wheel(fizi_ctx* ctx, uint32_t stream, const fizi_wheel* w) {
  if (!ctx) return FIZI_E_ARG;
  Ctx& c = ctx->c;
  if (stream >= c.n_streams) return fail(c, FIZI_E_CAPACITY, "stream id >= n_streams");
  if (!w) return fail(c, FIZI_E_ARG, "wheel is NULL");
  const bool ok = std::isfinite(w->cx) && std::isfinite(w->cy) && w->radius > 0.0 &&
                  std::isfinite(w->radius) && w->theta_max_deg > 0.0 && w->theta_max_deg <= 180.0 &&
                  w->inner >= 0.0 && w->inner < 1.0 && w->outer > 1.0 && std::isfinite(w->outer) &&
                  w->dead_zone_deg >= 0.0 && w->hold_ms >= 0;
  if (!ok) return fail(c, FIZI_E_ARG, "wheel: need radius > 0, 0 < theta_max <= 180, 0 <= inner < 1 < outer, dead zone >= 0, hold >= 0");
  DeviceGuard guard(c.device);
  // no drive fold of this stream may still be in flight on any stream
  cudaError_t e = cudaDeviceSynchronize();
  if (e == cudaSuccess) e = fizi::launch_drive_set(c, stream, *w, 0);
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e != cudaSuccess) return cuda_fail(c, e, "set_wheel");
  if (c.has_wheel.size() < c.n_streams) c.has_wheel.assign(c.n_streams, 0);
  c.has_wheel[stream] = 1;
  return FIZI_OK;
}

int fizi_drive(fizi_ctx* ctx, uint32_t stream, const fizi_result* results_dev, uint32_t n,
               fizi_command* commands_dev, fizi_stream_t cuda_stream) {
  if (!ctx) return FIZI_E_ARG;
  Ctx& c = ctx->c;
  if (c.sticky) return fail(c, FIZI_E_CUDA, "context has a sticky CUDA error: " + c.err);
  if (stream >= c.n_streams) return fail(c, FIZI_E_CAPACITY, "stream id >= n_streams");
  if (c.has_wheel.size() <= stream || !c.has_wheel[stream])
    return fail(c, FIZI_E_NOMODEL, "no wheel set for this stream (fizi_set_wheel)");
  if (n == 0) return FIZI_OK;
  if (!results_dev || !commands_dev) return fail(c, FIZI_E_ARG, "NULL pointer argument");
  DeviceGuard guard(c.device);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(cuda_stream);
  cudaError_t e = join_tail(c, st);
  if (e == cudaSuccess)
    e = fizi::launch_drive(c, stream, results_dev, n, nullptr, 0, 0, commands_dev, st);
  if (e != cudaSuccess) return cuda_fail(c, e, "drive");
  return FIZI_OK;
}

int fizi_drive_throttle(fizi_ctx* ctx, uint32_t stream, const fizi_result* results_dev, uint32_t n,
                        const fizi_zone_event* events_dev, uint32_t n_zones, uint32_t slider_zone,
                        fizi_command* commands_dev, fizi_stream_t cuda_stream) {
  if (!ctx) return FIZI_E_ARG;
  Ctx& c = ctx->c;
  if (c.sticky) return fail(c, FIZI_E_CUDA, "context has a sticky CUDA error: " + c.err);
  if (stream >= c.n_streams) return fail(c, FIZI_E_CAPACITY, "stream id >= n_streams");
  if (c.has_wheel.size() <= stream || !c.has_wheel[stream])
    return fail(c, FIZI_E_NOMODEL, "no wheel set for this stream (fizi_set_wheel)");
  if (c.n_zones.size() <= stream || c.n_zones[stream] == 0)
    return fail(c, FIZI_E_NOMODEL, "no layout set for this stream (fizi_set_zones)");
  if (n_zones != c.n_zones[stream])
    return fail(c, FIZI_E_ARG, "n_zones differs from the stream's layout");
  if (slider_zone >= n_zones || !((c.slider_zones[stream] >> slider_zone) & 1))
    return fail(c, FIZI_E_ARG, "slider_zone is not a slider zone of the stream's layout");
  if (n == 0) return FIZI_OK;
  if (!results_dev || !events_dev || !commands_dev) return fail(c, FIZI_E_ARG, "NULL pointer argument");
  DeviceGuard guard(c.device);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(cuda_stream);
  cudaError_t e = join_tail(c, st);
  if (e == cudaSuccess)
    e = fizi::launch_drive(c, stream, results_dev, n, events_dev, n_zones, slider_zone,
                           commands_dev, st);
  if (e != cudaSuccess) return cuda_fail(c, e, "drive_throttle");
  return FIZI_OK;
}

int fizi_set_pipeline(fizi_ctx* ctx, int enable) {
  if (!ctx || enable < 0 || enable > 1) return FIZI_E_ARG;
  ctx->c.pipeline = enable != 0;
  return FIZI_OK;
}

int fizi_flush(fizi_ctx* ctx, fizi_stream_t cuda_stream) {
  if (!ctx) return FIZI_E_ARG;
  Ctx& c = ctx->c;
  DeviceGuard guard(c.device);
  cudaError_t e = join_tail(c, reinterpret_cast<cudaStream_t>(cuda_stream));
  if (e != cudaSuccess) return cuda_fail(c, e, "join");
  return FIZI_OK;
}

int fizi_profile_enable(fizi_ctx* ctx, int mode) {
  if (!ctx || mode < 0 || mode > 2) return FIZI_E_ARG;
  ctx->c.prof = mode != 0;
  ctx->c.prof_mode = mode;
  return FIZI_OK;
}

int fizi_profile_read(fizi_ctx* ctx, double* ms_out, uint64_t* count_out, int reset) {
  if (!ctx) return FIZI_E_ARG;
  Ctx& c = ctx->c;
  DeviceGuard guard(c.device);
  fizi::prof_resolve(c);
  for (int i = 0; i < FIZI_PROF_SLOTS; i++) {
    if (ms_out) ms_out[i] = c.prof_ms[i];
    if (count_out) count_out[i] = c.prof_n[i];
    if (reset) { c.prof_ms[i] = 0; c.prof_n[i] = 0; }
  }
  return FIZI_OK;
}

uint64_t fizi_kernel_launches(const fizi_ctx* ctx) { return ctx ? ctx->c.launches : 0; }

uint32_t fizi_call_slots(void) { return fizi::kSlots; }

const char* fizi_last_error(const fizi_ctx* ctx) {
  if (!ctx) return "NULL context";
  return ctx->c.err.c_str();
}

const char* fizi_status_string(int s) {
  switch (s) {
    case FIZI_OK: return "FIZI_OK";
    case FIZI_E_ARG: return "FIZI_E_ARG";
    case FIZI_E_EMPTY: return "FIZI_E_EMPTY";
    case FIZI_E_DIMS: return "FIZI_E_DIMS";
    case FIZI_E_NOMODEL: return "FIZI_E_NOMODEL";
    case FIZI_E_TIME: return "FIZI_E_TIME";
    case FIZI_E_CUDA: return "FIZI_E_CUDA";
    case FIZI_E_OOM: return "FIZI_E_OOM";
    case FIZI_E_CAPACITY: return "FIZI_E_CAPACITY";
    default: return "FIZI_E_UNKNOWN";
  }
}

void fizi_destroy(fizi_ctx* ctx) {
  if (!ctx) return;
  DeviceGuard guard(ctx->c.device);
  cudaDeviceSynchronize();
  free_all(ctx->c);
  delete ctx;
}

}  // extern "C"

// diagnostics (not part of include/fizi.h): copy the timeline (start array,
// then end array, kTlKinds x kTlCalls each) to host memory
extern "C" int fizi_diag_timeline(fizi_ctx* ctx, unsigned long long* host) {
  if (!ctx || !ctx->c.tl) return FIZI_E_ARG;
  return (int)cudaMemcpy(host, ctx->c.tl, 2ull * fizi::kTlKinds * fizi::kTlCalls * 8,
                         cudaMemcpyDeviceToHost);
}

// diagnostics: host nanoseconds spent in run_call and in its slot wait
extern "C" int fizi_diag_host_ns(fizi_ctx* ctx, unsigned long long* call_ns, unsigned long long* sync_ns) {
  if (!ctx) return FIZI_E_ARG;
  *call_ns = ctx->c.host_call_ns;
  *sync_ns = ctx->c.host_sync_ns;
  return FIZI_OK;
}
