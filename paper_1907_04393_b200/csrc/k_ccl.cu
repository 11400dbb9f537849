// k_ccl.cu -- K5/K6: connected components of the open-close mask, the
// small-blob filter, the hand blob and the final mask (a5, a6, a7).
//
// P:72 "contour detection parameters" / P:75-76 the Mouse module "tracks the
// hand corresponding zone"; readings L13-L17, L30:
// 8-connected components, canonical label = 1 + min raster index, keep iff
// area * 1e6 >= ppm * W * H, hand = largest kept (ties -> smaller label),
// centroid = (sum x / area, sum y / area).
//
// Run-based labelling on the compact runs the morphology kernel extracted
// (row y's runs at row_base[y] .. + row_cnt[y], sorted by x; rows in any
// order).  One CTA (1024 threads) per frame.  The frame's runs and the
// union-find forest live in shared memory (up to kCclSmemRuns runs, else in
// global memory), so every find / link is a shared-memory access:
//   0. load runs, parent[i] = i, zero the per-root statistics
//   1. union runs of adjacent rows whose x ranges overlap within one pixel
//      (8-connectivity), one thread per row, two-pointer sweep over the two
//      sorted rows; lock-free linking by CAS, the root with the larger raster
//      key y*W+x0 goes under the smaller one, path halving in find
//   2. flatten: parent = root = the run holding the component's first pixel
//      in raster order, so label = 1 + key(root) = 1 + min raster index
//   3. per-root area, sum x, sum y, bbox: warp-aggregated global atomics
//   4. block reduction: #components, #kept, sum of kept areas, the largest
//      (max area, ties -> smaller label)
//   5. clear dropped components' runs from the mask words (final mask F)
#include <cstdio>
#include <cstdlib>

#include "dev_util.cuh"
#include "fizi_internal.cuh"
#include "track.cuh"

namespace fizi {

struct CclArgs {
  uint32_t f0;
  uint32_t* O;
  uint32_t W, H, P;
  uint64_t N;
  const uint32_t* row_cnt;
  const uint32_t* row_base;
  const uint32_t* frame_runs;
  const Run* runs;
  uint32_t* parent;
  RootStats* stats;
  uint64_t cap_runs;
  const CallPtrs* call;         // records + u8 mask target of the call (device)
  const uint32_t* fg;
  uint32_t ppm;
  // fused a6 output / a8 fold
  // call->masks, the u8 final mask: written by morphology (dropped blobs
  // cleared here) or, when pre-zeroed, written here from the kept runs
  bool masks_zeroed;
  uint32_t n;                   // frames in the launch (sub-batch)
  uint32_t* sub_done;           // CTAs finished in this launch
  uint32_t* fold_sync;          // [0] lock, [1] cursor, [2 + i] frame f0+i ready (zeroed per call)
  int track_stream;             // -2: no fold; -1: per-stream fold; >= 0: single stream
  int trace;                    // diagnostics: block 0 prints phase clocks
  uint32_t n_streams;
  const uint32_t* frame_stream;
  const uint32_t* group_frames;            // the sub-batch's same-stream groups (frames in order)
  const uint32_t* group_off;
  uint32_t n_groups;
  TrackState* tstate;
  fizi_params p;
};

// max over the warp of a 64-bit key: the high words first, then the low
// words of the lanes holding the maximal high word (two REDUX instructions)
__device__ __forceinline__ unsigned long long warp_max_u64(unsigned long long v) {
  const uint32_t hi = (uint32_t)(v >> 32), lo = (uint32_t)v;
  const uint32_t mh = __reduce_max_sync(0xFFFFFFFFu, hi);
  const uint32_t ml = __reduce_max_sync(0xFFFFFFFFu, hi == mh ? lo : 0u);
  return ((unsigned long long)mh << 32) | ml;
}

__device__ __forceinline__ bool kept_area(uint32_t area, uint32_t ppm, uint64_t N) {
  return (uint64_t)area * 1000000ull >= (uint64_t)ppm * N;
}

template <bool kShared>
__device__ __forceinline__ uint32_t ld_par(const uint32_t* p) {
  if (kShared) return *reinterpret_cast<const volatile uint32_t*>(p);
  return __ldcg(p);
}

template <bool kShared>
__device__ __forceinline__ uint32_t find_root(uint32_t* par, uint32_t x) {
  while (true) {
    const uint32_t p = ld_par<kShared>(par + x);
    if (p == x) return x;
    const uint32_t gp = ld_par<kShared>(par + p);
    if (gp != p) atomicCAS(par + x, p, gp);            // path halving
    x = gp;
  }
}

__device__ __forceinline__ uint32_t run_key(const Run* R, uint32_t i, uint32_t W) {
  const Run r = R[i];
  return (uint32_t)r.y * W + r.x0;
}

template <bool kShared>
__device__ __forceinline__ void unite(uint32_t* par, const Run* R, uint32_t W, uint32_t a,
                                      uint32_t b) {
  while (true) {
    a = find_root<kShared>(par, a);
    b = find_root<kShared>(par, b);
    if (a == b) return;
    if (run_key(R, a, W) < run_key(R, b, W)) { const uint32_t t = a; a = b; b = t; }
    const uint32_t old = atomicCAS(par + a, a, b);      // a: larger key, goes under b
    if (old == a) return;
    a = old;
  }
}

#define CCL_MARK(k) if (a.trace && threadIdx.x == 0) t_mark[k] = clock64();

// above this many 4-row blocks the block boundaries are merged in
// log2(blocks) tree rounds instead of one pass (C3: 270 blocks, one pass
// 2.2 us vs 9 rounds 7.8 us; C4: 540 blocks, one pass 21.5 us vs 12.2 us)
constexpr uint32_t kCclTreeBlocks = 384;

template <bool kShared>
__device__ void ccl_frame(const CclArgs& a, uint32_t f, Run* R, uint32_t* par, uint32_t* s_area,
                          uint32_t T, long long* t_mark) {
  __shared__ unsigned long long s_best[32];
  __shared__ uint32_t s_cnt[3][32];
  __shared__ unsigned long long s_key;
  __shared__ uint32_t s_drop;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, nthr = blockDim.x;
  const uint32_t W = a.W, H = a.H, P = a.P;
  const uint32_t* cnt = a.row_cnt + (uint64_t)f * H;
  const uint32_t* rb = a.row_base + (uint64_t)f * H;
  const Run* gruns = a.runs + (uint64_t)f * a.cap_runs;
  uint32_t* gpar = a.parent + (uint64_t)f * a.cap_runs;
  RootStats* stats = a.stats + (uint64_t)f * a.cap_runs;

  CCL_MARK(0)
  // loaded early (their loads would otherwise sit on the critical path of
  // phases 4 and 5): merged foreground count, record and mask pointers
  const uint32_t fg_merged = a.fg[f];
  fizi_result* const res = a.call->res;
  uint8_t* const masks = a.call->masks;
  // component area of root i: shared memory for frames labelled in shared memory
  auto area_of = [&](uint32_t i) -> uint32_t {
    return kShared ? s_area[i] : __ldcg(&stats[i].area);
  };
  // 0. load
  for (uint32_t i = tid; i < T; i += nthr) {
    if (kShared) { R[i] = gruns[i]; s_area[i] = 0u; }
    par[i] = i;
    RootStats z;
    z.area = 0; z.xmin = 0xFFFFFFFFu; z.xmax = 0; z.ymin = 0xFFFFFFFFu; z.ymax = 0;
    z.pad = 0; z.sx = 0; z.sy = 0;
    stats[i] = z;
  }
  __syncthreads();

  CCL_MARK(1)
  // 1. union of every run with the 8-connected runs of the previous row.
  //    Rows are taken in blocks of kRowBlock: one thread unites the row pairs
  //    inside a block in order (no contention, runs end up one link from the
  //    block's top component), then the block boundaries are united in
  //    parallel, so trees stay shallow even for tall components.
  constexpr uint32_t kRowBlock = 4;
  auto unite_rows = [&](uint32_t y) {                  // row pair (y - 1, y)
    const uint32_t n = cnt[y], np = cnt[y - 1];
    if (!n || !np) return;
    const uint32_t cb = rb[y], pb = rb[y - 1];
    uint32_t h = 0;
    for (uint32_t j = 0; j < n; j++) {
      const Run rc = R[cb + j];
      while (h < np && (uint32_t)R[pb + h].x1 + 1 < rc.x0) h++;
      for (uint32_t h2 = h; h2 < np && R[pb + h2].x0 <= (uint32_t)rc.x1 + 1; h2++)
        unite<kShared>(par, R, W, cb + j, pb + h2);
    }
  };
  for (uint32_t blk = tid; blk * kRowBlock < H; blk += nthr) {
    const uint32_t y1 = min(blk * kRowBlock + kRowBlock, H);
    for (uint32_t y = blk * kRowBlock + 1; y < y1; y++) unite_rows(y);
  }
  __syncthreads();
  const uint32_t nblk = (H + kRowBlock - 1) / kRowBlock;
  if (nblk <= kCclTreeBlocks) {
    // all block boundaries at once (a tall component links its block roots
    // into a chain, walked with path halving: cheap for a few hundred blocks)
    for (uint32_t blk = tid + 1; blk < nblk; blk += nthr) unite_rows(blk * kRowBlock);
    __syncthreads();
  } else {
    // tall frames: boundaries merged as a tree, in round s the boundary at
    // block (2k+1)s joins two merged groups of s blocks, so trees grow by at
    // most one level per round (C4: the union phase 21.5 -> 12.2 us per frame)
    for (uint32_t sd = 1; sd < nblk; sd <<= 1) {
      for (uint32_t k = tid; (2 * k + 1) * sd < nblk; k += nthr) unite_rows((2 * k + 1) * sd * kRowBlock);
      __syncthreads();
    }
  }

  CCL_MARK(2)
  // 2. flatten: every run walks to its root, halving the path as it goes
  //    (the forest no longer changes shape, so plain stores of an ancestor
  //    are safe while other threads walk); once every walk is over, each
  //    run points at its root
  constexpr uint32_t kMaxPer = 8;                        // runs per thread kept in registers
  uint32_t roots[kMaxPer];
  const bool in_regs = T <= kMaxPer * (uint32_t)nthr;
#pragma unroll
  for (uint32_t k = 0; k < kMaxPer; k++) {
    const uint32_t i = tid + k * nthr;
    uint32_t x = i;
    if (i < T) {
      while (true) {
        const uint32_t p = ld_par<kShared>(par + x);
        if (p == x) break;
        const uint32_t gp = ld_par<kShared>(par + p);
        if (gp == p) { x = p; break; }
        par[x] = gp;
        x = gp;
      }
    }
    roots[k] = x;
  }
  __syncthreads();
  if (in_regs) {
#pragma unroll
    for (uint32_t k = 0; k < kMaxPer; k++) {
      const uint32_t i = tid + k * nthr;
      if (i < T) par[i] = roots[k];
    }
  } else {                                  // large frames: lockstep pointer jumping
    while (true) {
      int changed = 0;
      for (uint32_t i = tid; i < T; i += nthr) {
        const uint32_t p = ld_par<kShared>(par + i);
        const uint32_t gp = ld_par<kShared>(par + p);
        if (gp != p) { par[i] = gp; changed = 1; }
      }
      if (!__syncthreads_or(changed)) break;
    }
  }
  __syncthreads();
  CCL_MARK(3)

  // 3. statistics, aggregated over lanes of a warp that share a root
  for (uint32_t i0 = 0; i0 < T; i0 += nthr) {
    const uint32_t i = i0 + tid;
    const bool act = i < T;
    uint32_t root = 0xFFFFFFFFu, len = 0, x0 = 0xFFFFFFFFu, x1 = 0, y = 0;
    unsigned long long sx = 0, sy = 0;
    if (act) {
      const Run r = R[i];
      root = ld_par<kShared>(par + i);
      len = (uint32_t)r.x1 - r.x0 + 1;
      x0 = r.x0; x1 = r.x1; y = r.y;
      sx = (unsigned long long)(r.x0 + r.x1) * len / 2;
      sy = (unsigned long long)r.y * len;
    }
    if (__all_sync(0xFFFFFFFFu, !act)) continue;
    const uint32_t m = __match_any_sync(0xFFFFFFFFu, root);
    uint32_t g_area = 0, g_x0 = 0xFFFFFFFFu, g_x1 = 0, g_y0 = 0xFFFFFFFFu, g_y1 = 0;
    unsigned long long g_sx = 0, g_sy = 0;
    if (__all_sync(0xFFFFFFFFu, m == 0xFFFFFFFFu)) {        // one root for the whole warp
      g_area = __reduce_add_sync(0xFFFFFFFFu, len);
      g_x0 = __reduce_min_sync(0xFFFFFFFFu, x0);
      g_x1 = __reduce_max_sync(0xFFFFFFFFu, x1);
      g_y0 = __reduce_min_sync(0xFFFFFFFFu, y);
      g_y1 = __reduce_max_sync(0xFFFFFFFFu, y);
      g_sx = sx;
      g_sy = sy;
#pragma unroll
      for (int d = 16; d > 0; d >>= 1) {
        g_sx += __shfl_xor_sync(0xFFFFFFFFu, g_sx, d);
        g_sy += __shfl_xor_sync(0xFFFFFFFFu, g_sy, d);
      }
    } else
#pragma unroll 4
    for (int l = 0; l < 32; l++) {
      const uint32_t o_len = __shfl_sync(0xFFFFFFFFu, len, l);
      const uint32_t o_x0 = __shfl_sync(0xFFFFFFFFu, x0, l);
      const uint32_t o_x1 = __shfl_sync(0xFFFFFFFFu, x1, l);
      const uint32_t o_y = __shfl_sync(0xFFFFFFFFu, y, l);
      const unsigned long long o_sx = __shfl_sync(0xFFFFFFFFu, sx, l);
      const unsigned long long o_sy = __shfl_sync(0xFFFFFFFFu, sy, l);
      if ((m >> l) & 1u) {
        g_area += o_len; g_sx += o_sx; g_sy += o_sy;
        g_x0 = min(g_x0, o_x0); g_x1 = max(g_x1, o_x1);
        g_y0 = min(g_y0, o_y); g_y1 = max(g_y1, o_y);
      }
    }
    if (act && (uint32_t)lane == (uint32_t)(__ffs(m) - 1)) {
      RootStats* st = stats + root;
      if (kShared) atomicAdd(&s_area[root], g_area);
      atomicAdd(&st->area, g_area);
      atomicAdd(&st->sx, g_sx);
      atomicAdd(&st->sy, g_sy);
      atomicMin(&st->xmin, g_x0);
      atomicMax(&st->xmax, g_x1);
      atomicMin(&st->ymin, g_y0);
      atomicMax(&st->ymax, g_y1);
    }
  }
  __syncthreads();

  CCL_MARK(4)
  // 4. counts and the hand blob: key = area << 32 | ~label
  uint32_t n_tot = 0, n_kept = 0, fg_final = 0;
  unsigned long long best = 0;
  for (uint32_t i = tid; i < T; i += nthr) {
    if (ld_par<kShared>(par + i) != i) continue;
    n_tot++;
    const uint32_t area = area_of(i);
    if (!kept_area(area, a.ppm, a.N)) continue;
    n_kept++;
    fg_final += area;
    const uint32_t label = 1u + run_key(R, i, W);
    const unsigned long long key = ((unsigned long long)area << 32) | (0xFFFFFFFFu - label);
    best = key > best ? key : best;
  }
  n_tot = __reduce_add_sync(0xFFFFFFFFu, n_tot);
  n_kept = __reduce_add_sync(0xFFFFFFFFu, n_kept);
  fg_final = __reduce_add_sync(0xFFFFFFFFu, fg_final);
  best = warp_max_u64(best);
  if (lane == 0) {
    s_cnt[0][warp] = n_tot;
    s_cnt[1][warp] = n_kept;
    s_cnt[2][warp] = fg_final;
    s_best[warp] = best;
  }
  __syncthreads();
  if (warp == 0) {
    const int nw = nthr >> 5;
    n_tot = __reduce_add_sync(0xFFFFFFFFu, lane < nw ? s_cnt[0][lane] : 0u);
    n_kept = __reduce_add_sync(0xFFFFFFFFu, lane < nw ? s_cnt[1][lane] : 0u);
    fg_final = __reduce_add_sync(0xFFFFFFFFu, lane < nw ? s_cnt[2][lane] : 0u);
    best = warp_max_u64(lane < nw ? s_best[lane] : 0ull);
    if (lane == 0) {
      fizi_result* r = res + f;
      r->fg_merged = fg_merged;
      r->fg_final = fg_final;
      r->n_comp_total = n_tot;
      r->n_comp_kept = n_kept;
      s_key = best;
      s_drop = n_tot - n_kept;
    }
  }
  __syncthreads();
  CCL_MARK(5)
  const unsigned long long bk = s_key;
  if (bk) {                                   // the best root's thread writes the blob
    const uint32_t blabel = 0xFFFFFFFFu - (uint32_t)(bk & 0xFFFFFFFFu);
    for (uint32_t i = tid; i < T; i += nthr) {
      if (ld_par<kShared>(par + i) != i || 1u + run_key(R, i, W) != blabel) continue;
      fizi_result* r = res + f;
      const RootStats* st = stats + i;
      const uint32_t area = __ldcg(&st->area);
      const unsigned long long sx = __ldcg(&st->sx), sy = __ldcg(&st->sy);
      r->blob_area = area;
      r->blob_label = blabel;
      r->bbox[0] = __ldcg(&st->xmin); r->bbox[1] = __ldcg(&st->ymin);
      r->bbox[2] = __ldcg(&st->xmax); r->bbox[3] = __ldcg(&st->ymax);
      r->sum_x = sx;
      r->sum_y = sy;
      r->cx = __ddiv_rn(__ull2double_rn(sx), __uint2double_rn(area));
      r->cy = __ddiv_rn(__ull2double_rn(sy), __uint2double_rn(area));
    }
  }
  if (kShared)                                 // forest for fizi_debug_stage(LABELS)
    for (uint32_t i = tid; i < T; i += nthr) gpar[i] = par[i];

  CCL_MARK(6)
  // 5a. pre-zeroed u8 mask: write the bytes of every run of a kept component,
  //     one thread per run: bytes up to 4-byte alignment, words up to 16-byte
  //     alignment, 16-byte stores, then words and bytes (runs are disjoint,
  //     so no two threads write the same byte)
  if (masks && a.masks_zeroed) {
    const uint32_t k1 = 0x01010101u;
    for (uint32_t i = tid; i < T; i += nthr) {
      if (!kept_area(area_of(ld_par<kShared>(par + i)), a.ppm, a.N)) continue;
      const Run rg = R[i];
      uint8_t* p = masks + ((uint64_t)f * H + rg.y) * W;
      uintptr_t x = reinterpret_cast<uintptr_t>(p) + rg.x0;
      const uintptr_t xe = reinterpret_cast<uintptr_t>(p) + (uint32_t)rg.x1 + 1;
      for (; x < xe && (x & 3u); x++) __stcg(reinterpret_cast<uint8_t*>(x), (uint8_t)1);
      for (; x + 4 <= xe && (x & 15u); x += 4) __stcg(reinterpret_cast<uint32_t*>(x), k1);
      for (; x + 16 <= xe; x += 16) __stcg(reinterpret_cast<uint4*>(x), make_uint4(k1, k1, k1, k1));
      for (; x + 4 <= xe; x += 4) __stcg(reinterpret_cast<uint32_t*>(x), k1);
      for (; x < xe; x++) __stcg(reinterpret_cast<uint8_t*>(x), (uint8_t)1);
    }
  }

  if (a.trace && tid == 0) t_mark[8] = clock64();
  // 5. clear the runs of dropped components from the bit mask (final mask F)
  if (s_drop == 0) return;
  uint32_t* Of = a.O + (uint64_t)f * H * P;
  for (uint32_t i = tid; i < T; i += nthr) {
    const uint32_t root = ld_par<kShared>(par + i);
    if (kept_area(area_of(root), a.ppm, a.N)) continue;
    const Run rg = R[i];
    uint32_t* row = Of + (uint64_t)rg.y * P;
    for (uint32_t k = rg.x0 >> 5; k <= (uint32_t)(rg.x1 >> 5); k++) {
      const uint32_t b0 = k == (uint32_t)(rg.x0 >> 5) ? (rg.x0 & 31u) : 0u;
      const uint32_t b1 = k == (uint32_t)(rg.x1 >> 5) ? (rg.x1 & 31u) : 31u;
      const uint32_t m = (b1 == 31u ? 0xFFFFFFFFu : ((1u << (b1 + 1)) - 1u)) & ~((1u << b0) - 1u);
      atomicAnd(row + k, ~m);
    }
    if (masks && !a.masks_zeroed) {
      uint8_t* mrow = masks + ((uint64_t)f * H + rg.y) * W;
      for (uint32_t x = rg.x0; x <= rg.x1; x++) mrow[x] = 0;
    }
  }
}

// a8 fold of the launch's records, run by the last CTA to finish: frames in
// index order, one thread per stream (records staged through shared memory
// for the single-stream case).
__device__ void fold_records(const CclArgs& a, uint8_t* smem) {
  const uint32_t f0 = a.f0, n = a.n;
  if (a.track_stream >= 0) {
    constexpr uint32_t kChunk = 512;
    int64_t* t_s = reinterpret_cast<int64_t*>(smem);              // in: t, out: dwell
    double* cx_s = reinterpret_cast<double*>(t_s + kChunk);       // in: cx, out: px
    double* cy_s = cx_s + kChunk;                                 // in: cy, out: py
    uint32_t* ar_s = reinterpret_cast<uint32_t*>(cy_s + kChunk);  // in: area, out: vis | clk<<1
    uint32_t* fl_s = ar_s + kChunk;                                // in: relearn flags
    TrackState st;
    if (threadIdx.x == 0) st = a.tstate[a.track_stream];
    for (uint32_t base = 0; base < n; base += kChunk) {
      const uint32_t m = min(kChunk, n - base);
      for (uint32_t i = threadIdx.x; i < m; i += blockDim.x) {
        const fizi_result& r = a.call->res[f0 + base + i];
        t_s[i] = __ldcg(&r.t_ms);
        ar_s[i] = __ldcg(&r.blob_area);
        fl_s[i] = __ldcg(&r.relearn);
        cx_s[i] = __ldcg(&r.cx);
        cy_s[i] = __ldcg(&r.cy);
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        for (uint32_t i = 0; i < m; i++) {
          fizi_result r;
          r.t_ms = t_s[i]; r.blob_area = ar_s[i]; r.cx = cx_s[i]; r.cy = cy_s[i]; r.relearn = fl_s[i];
          track_one(a.p, st, r);
          t_s[i] = r.dwell_ms; cx_s[i] = r.px; cy_s[i] = r.py;
          ar_s[i] = (uint32_t)r.visible | ((uint32_t)r.clicked << 1);
        }
      }
      __syncthreads();
      for (uint32_t i = threadIdx.x; i < m; i += blockDim.x) {
        fizi_result& o = a.call->res[f0 + base + i];
        o.visible = (uint8_t)(ar_s[i] & 1u); o.clicked = (uint8_t)(ar_s[i] >> 1);
        o.px = cx_s[i]; o.py = cy_s[i]; o.dwell_ms = t_s[i];
      }
      __syncthreads();
    }
    if (threadIdx.x == 0) a.tstate[a.track_stream] = st;
  } else {
    // one thread per stream: a stream's groups are consecutive in the group
    // list and hold its frames in index order (fill_call), so the thread that
    // owns a stream's first group folds the stream's frames in order
    for (uint32_t g = threadIdx.x; g < a.n_groups; g += blockDim.x) {
      const uint32_t s = a.frame_stream[a.group_frames[a.group_off[g]]];
      if (g > 0 && a.frame_stream[a.group_frames[a.group_off[g - 1]]] == s) continue;
      TrackState st = a.tstate[s];
      for (uint32_t gg = g; gg < a.n_groups; gg++) {
        const uint32_t q0 = a.group_off[gg], q1 = a.group_off[gg + 1];
        if (a.frame_stream[a.group_frames[q0]] != s) break;
        for (uint32_t q = q0; q < q1; q++) {
          const uint32_t f = a.group_frames[q];
          fizi_result r;
          r.t_ms = __ldcg(&a.call->res[f].t_ms); r.blob_area = __ldcg(&a.call->res[f].blob_area);
          r.cx = __ldcg(&a.call->res[f].cx); r.cy = __ldcg(&a.call->res[f].cy);
          r.relearn = __ldcg(&a.call->res[f].relearn);
          track_one(a.p, st, r);
          fizi_result& o = a.call->res[f];
          o.visible = r.visible; o.clicked = r.clicked;
          o.px = r.px; o.py = r.py; o.dwell_ms = r.dwell_ms;
        }
      }
      a.tstate[s] = st;
    }
  }
}

__device__ unsigned long long g_ccl_trace[4096][12];   // start, end, T, fold end, phase clocks          // diagnostics (FIZI_CCL_TRACE)
__device__ __forceinline__ unsigned long long gtimer_ccl() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

__global__ void __launch_bounds__(1024) ccl_kernel(CclArgs a) {
  const unsigned long long g_t0 = a.trace ? gtimer_ccl() : 0ull;
  if (threadIdx.x == 0) tl_mark(a.call, kTlCcl, 0);
  struct TlEnd {
    const CallPtrs* call;
    __device__ ~TlEnd() { if (threadIdx.x == 0) tl_mark(call, kTlCcl, 1); }
  } tl_end{a.call};
  extern __shared__ __align__(16) uint8_t smc[];
  const uint32_t f = a.f0 + blockIdx.x;
  const uint32_t T = a.frame_runs[f];
  FIZI_DCHECK(T <= a.cap_runs && f < a.call->n);
  __shared__ long long t_mark[10];
  if (a.trace && threadIdx.x == 0) t_mark[9] = clock64();
  if (T <= kCclSmemRuns) {
    Run* R = reinterpret_cast<Run*>(smc);
    uint32_t* par = reinterpret_cast<uint32_t*>(smc + sizeof(Run) * kCclSmemRuns);
    uint32_t* s_area = par + kCclSmemRuns;
    ccl_frame<true>(a, f, R, par, s_area, T, t_mark);
  } else {
    ccl_frame<false>(a, f, const_cast<Run*>(a.runs + (uint64_t)f * a.cap_runs),
                     a.parent + (uint64_t)f * a.cap_runs, nullptr, T, t_mark);
  }
  if (a.trace && threadIdx.x == 0 && blockIdx.x < 4096) {
    t_mark[7] = clock64();
    g_ccl_trace[blockIdx.x][0] = g_t0;
    g_ccl_trace[blockIdx.x][1] = gtimer_ccl();
    g_ccl_trace[blockIdx.x][2] = T | ((unsigned long long)(t_mark[8] - t_mark[6]) << 32);
    for (int k = 0; k < 8; k++) g_ccl_trace[blockIdx.x][4 + k] = (unsigned long long)(t_mark[k] - t_mark[9]);
  }
  if (a.track_stream == -2) return;
  if (a.track_stream >= 0) {
    // single stream: the fold advances while other frames are still being
    // labelled.  Frame f is marked ready; the CTA that holds the fold lock
    // loads the ready records from the cursor on (all threads, in parallel)
    // and thread 0 folds them from shared memory.  After releasing the lock
    // the holder re-checks the cursor, so a frame that became ready while
    // the lock was held is never left behind.  Nobody waits for another CTA.
    __shared__ uint32_t s_own, s_i0, s_cnt;
    __syncthreads();                          // this frame's record is complete
    if (threadIdx.x == 0) {
      __threadfence();
      atomicExch(a.fold_sync + 2 + (f - a.f0), 1u);
    }
    int64_t* t_s = reinterpret_cast<int64_t*>(smc);
    double* cx_s = reinterpret_cast<double*>(t_s + 1024);
    double* cy_s = cx_s + 1024;
    uint32_t* ar_s = reinterpret_cast<uint32_t*>(cy_s + 1024);
    uint32_t* fl_s = ar_s + 1024;
    int64_t* od_s = reinterpret_cast<int64_t*>(fl_s + 1024);     // out: dwell
    double* opx_s = reinterpret_cast<double*>(od_s + 1024);      // out: px
    double* opy_s = opx_s + 1024;                                 // out: py
    uint32_t* ov_s = reinterpret_cast<uint32_t*>(opy_s + 1024);  // out: vis | clk<<1
    while (true) {
      if (threadIdx.x == 0) {
        s_own = atomicCAS(a.fold_sync, 0u, 1u) == 0u;
        if (s_own) {
          __threadfence();
          s_i0 = *reinterpret_cast<volatile uint32_t*>(a.fold_sync + 1);
          s_cnt = 0xFFFFFFFFu;
        }
      }
      __syncthreads();
      if (!s_own) break;                                   // someone else folds
      const uint32_t i0 = s_i0;
      // length of the ready prefix from the cursor (at most blockDim frames)
      const uint32_t i = i0 + threadIdx.x;
      const bool rdy = i < a.n && atomicAdd(a.fold_sync + 2 + i, 0u) != 0u;
      if (!rdy && i <= a.n) atomicMin(&s_cnt, threadIdx.x);
      __syncthreads();
      const uint32_t cnt = min(s_cnt, blockDim.x);
      if (threadIdx.x < cnt) {
        __threadfence();
        const fizi_result& r = a.call->res[a.f0 + i];
        t_s[threadIdx.x] = __ldcg(&r.t_ms);
        ar_s[threadIdx.x] = __ldcg(&r.blob_area);
        fl_s[threadIdx.x] = __ldcg(&r.relearn);
        cx_s[threadIdx.x] = __ldcg(&r.cx);
        cy_s[threadIdx.x] = __ldcg(&r.cy);
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        // one thread folds in order; the next record's inputs are read from
        // shared memory before the current one is folded (outputs go to
        // separate arrays), so the loads overlap the FP64 chain
        TrackState st = a.tstate[a.track_stream];
        int64_t nt = cnt ? t_s[0] : 0;
        uint32_t na = cnt ? ar_s[0] : 0u, nfl = cnt ? fl_s[0] : 0u;
        double nx = cnt ? cx_s[0] : 0.0, ny = cnt ? cy_s[0] : 0.0;
        for (uint32_t k = 0; k < cnt; k++) {
          fizi_result q;
          q.t_ms = nt; q.blob_area = na; q.cx = nx; q.cy = ny; q.relearn = nfl;
          if (k + 1 < cnt) {
            nt = t_s[k + 1]; na = ar_s[k + 1]; nfl = fl_s[k + 1]; nx = cx_s[k + 1]; ny = cy_s[k + 1];
          }
          track_one(a.p, st, q);
          od_s[k] = q.dwell_ms; opx_s[k] = q.px; opy_s[k] = q.py;
          ov_s[k] = (uint32_t)q.visible | ((uint32_t)q.clicked << 1);
        }
        a.tstate[a.track_stream] = st;
      }
      __syncthreads();
      if (threadIdx.x < cnt) {
        fizi_result& o = a.call->res[a.f0 + i];
        o.visible = (uint8_t)(ov_s[threadIdx.x] & 1u); o.clicked = (uint8_t)(ov_s[threadIdx.x] >> 1);
        o.px = opx_s[threadIdx.x]; o.py = opy_s[threadIdx.x]; o.dwell_ms = od_s[threadIdx.x];
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        const uint32_t nxt = i0 + cnt;
        *reinterpret_cast<volatile uint32_t*>(a.fold_sync + 1) = nxt;
        __threadfence();
        atomicExch(a.fold_sync, 0u);                        // release
        __threadfence();
        // retry iff a frame at the cursor became ready meanwhile
        s_own = nxt < a.n && atomicAdd(a.fold_sync + 2 + nxt, 0u) != 0u;
      }
      __syncthreads();
      if (!s_own) break;
    }
    return;
  }
  __shared__ uint32_t s_last;
  __syncthreads();                            // this frame's record is complete
  if (threadIdx.x == 0) {
    __threadfence();
    s_last = atomicAdd(a.sub_done, 1u) == a.n - 1;
    __threadfence();
  }
  __syncthreads();
  if (s_last) {
    fold_records(a, smc);
    if (a.trace && threadIdx.x == 0 && blockIdx.x < 4096) g_ccl_trace[blockIdx.x][3] = gtimer_ccl();
  }
}

constexpr size_t kCclSmem = (sizeof(Run) + 2 * sizeof(uint32_t)) * kCclSmemRuns;
static_assert(kCclSmem >= 1024 * 60, "fold staging fits the labelling shared memory");

__global__ void __launch_bounds__(512) zero_masks_kernel(const CallPtrs* call, uint64_t N);

cudaError_t init_ccl(Ctx& c) {
  (void)c;
  cudaError_t e = cudaFuncSetAttribute(ccl_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)kCclSmem);
  if (e == cudaSuccess) e = set_carveout((const void*)ccl_kernel);
  if (e == cudaSuccess) e = set_carveout((const void*)zero_masks_kernel);
  return e;
}

cudaError_t launch_ccl(Ctx& c, uint32_t f0, uint32_t n, uint32_t sub, uint32_t g0, uint32_t ng,
                       bool masks_zeroed, int track_stream, cudaStream_t st) {
  CclArgs a;
  a.f0 = f0;
  a.call = c.call;
  a.masks_zeroed = masks_zeroed;
  a.n = n;
  a.sub_done = c.sub_done + sub;
  a.fold_sync = c.fold_sync + (uint64_t)sub * (c.max_batch + 2);
  a.track_stream = track_stream;
  a.n_streams = c.n_streams;
  a.frame_stream = c.frame_stream;
  a.group_frames = c.group_frames;
  a.group_off = c.group_off + g0;
  a.n_groups = ng;
  a.tstate = reinterpret_cast<TrackState*>(c.tstate);
  a.p = c.p;
  static const int trace = getenv("FIZI_CCL_TRACE") ? atoi(getenv("FIZI_CCL_TRACE")) : 0;
  a.trace = trace;
  a.O = c.bitO;
  a.W = c.W; a.H = c.H; a.P = c.P;
  a.N = c.N;
  a.row_cnt = c.row_cnt;
  a.row_base = c.row_base;
  a.frame_runs = c.frame_runs;
  a.runs = c.runs;
  a.parent = c.parent;
  a.stats = c.stats;
  a.cap_runs = c.cap_runs;
  a.fg = c.fg;
  a.ppm = c.p.min_blob_ppm;
  static const int threads = getenv("FIZI_CCL_THREADS") ? atoi(getenv("FIZI_CCL_THREADS")) : 512;
  ccl_kernel<<<n, threads, kCclSmem, st>>>(a);
  c.launches += 1;
  return cudaGetLastError();
}

// ------------------------------------------------- final u8 mask (a6 output)

__global__ void expand16_kernel(const uint32_t* __restrict__ F, uint8_t* __restrict__ out,
                                uint64_t total16, uint32_t blocks_per_row, uint32_t P, uint32_t W) {
  const uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (t >= total16) return;
  const uint64_t row = t / blocks_per_row;            // frame-major rows
  const uint32_t j = (uint32_t)(t % blocks_per_row);
  const uint32_t w = __ldg(F + row * P + (j >> 1));
  const uint32_t b = (w >> (16 * (j & 1))) & 0xFFFFu;
  uint4 o;
  o.x = expand4(b & 0xF);
  o.y = expand4((b >> 4) & 0xF);
  o.z = expand4((b >> 8) & 0xF);
  o.w = expand4(b >> 12);
  __stcs(reinterpret_cast<uint4*>(out + row * W + 16ull * j), o);
}

__global__ void expand1_kernel(const uint32_t* __restrict__ F, uint8_t* __restrict__ out,
                               uint64_t total, uint32_t W, uint32_t P) {
  const uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (t >= total) return;
  const uint64_t row = t / W;
  const uint32_t x = (uint32_t)(t % W);
  out[t] = (uint8_t)((F[row * P + (x >> 5)] >> (x & 31)) & 1u);
}

cudaError_t launch_expand_from(Ctx& c, const uint32_t* bits, uint32_t n, uint8_t* masks,
                               cudaStream_t st) {
  const uint64_t rows = (uint64_t)n * c.H;
  if (c.W % 16 == 0) {
    const uint32_t bpr = c.W / 16;
    const uint64_t total = rows * bpr;
    expand16_kernel<<<(unsigned)((total + 255) / 256), 256, 0, st>>>(bits, masks, total, bpr, c.P, c.W);
  } else {
    const uint64_t total = rows * c.W;
    expand1_kernel<<<(unsigned)((total + 255) / 256), 256, 0, st>>>(bits, masks, total, c.W, c.P);
  }
  c.launches += 1;
  return cudaGetLastError();
}

// zero the call's u8 mask target (call->masks, call->n frames); runs on the
// side stream while the fused segmentation kernel streams the frames
__global__ void __launch_bounds__(512) zero_masks_kernel(const CallPtrs* call, uint64_t N) {
  if (threadIdx.x == 0) tl_mark(call, kTlZero, 0);
  uint8_t* m = call->masks;
  if (!m) return;
  const uint64_t total = call->n * N;
  const uint64_t gt = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  const uint64_t head = min(total, (uint64_t)((16u - (reinterpret_cast<uintptr_t>(m) & 15u)) & 15u));
  if (gt < head) m[gt] = 0;
  uint4* body = reinterpret_cast<uint4*>(m + head);
  const uint64_t nb = (total - head) / 16;
  const uint4 z = make_uint4(0u, 0u, 0u, 0u);
  for (uint64_t i = gt; i < nb; i += stride) __stcs(body + i, z);   // streaming: evict first
  const uint64_t tail = head + nb * 16;
  if (gt < total - tail) m[tail + gt] = 0;
  if (threadIdx.x == 0) tl_mark(call, kTlZero, 1);
}

cudaError_t launch_zero_masks(Ctx& c, uint32_t n, cudaStream_t st) {
  (void)n;
  prof_begin(c, st);
  zero_masks_kernel<<<c.sms * 2, 512, 0, st>>>(c.call, c.N);
  prof_end(c, FIZI_PROF_MASKZERO, st);
  c.launches += 1;
  return cudaGetLastError();
}

cudaError_t launch_expand(Ctx& c, uint32_t f0, uint32_t n, uint8_t* masks, cudaStream_t st) {
  return launch_expand_from(c, c.bitO + (uint64_t)f0 * c.H * c.P, n, masks + (uint64_t)f0 * c.N, st);
}

}  // namespace fizi

extern "C" int fizi_diag_ccl_trace(unsigned long long* host, unsigned int n) {
  return (int)cudaMemcpyFromSymbol(host, fizi::g_ccl_trace, sizeof(unsigned long long) * 12 * n);
}
