// k_morph.cu -- K4: open-close morphology on the bit-packed mask (a4), fused
// with the run extraction that starts the labelling (a5, step 1).
//
// §3.1 P:138-139 "morphological operations, combining erosion and dilatation
// operators ... remove the small noisy objects and ... connect neighborhood
// zones"; reading L12: square SE of side 2r+1, O = E(D(D(E(A)))), positions
// outside the frame count as 0 for both operators.
//
// One CTA (32 x 8 threads) = a band of TR output rows of one frame.  The band
// plus a 4r-row halo is staged in shared memory once; the four passes run in
// shared memory (ping-pong), each shrinking the valid band by r rows.  A
// 32-pixel word is one thread's work: shifts across the neighbouring words
// give the horizontal op, rows y-r..y+r the vertical op (separable square SE).
// The band's final rows are then written out and scanned for horizontal runs
// of 1-bits; each non-empty row reserves a contiguous range of the frame's
// compact run array with one atomicAdd (row_base[y], row_cnt[y]), its runs
// sorted by x inside the range.  Rows land in arbitrary order: the labelling
// identifies components by the raster key y*W+x0 of their runs, not by index.
#include <cstring>
#include <cstdlib>

#include "dev_util.cuh"
#include "fizi_internal.cuh"

namespace fizi {


struct MorphArgs {
  const CallPtrs* call;         // diagnostics timeline only
  uint32_t f0;                  // first frame of the launch (sub-batch)
  bool write_masks;             // write the u8 mask rows of O into call->masks (fast path)
  bool masks_zeroed;            // (always false when write_masks)
  const uint32_t* dirty;        // per-frame chunk bitmap (fast path) or nullptr
  uint32_t dirty_words;
  bool write_zero_o;            // zero bands still write their O rows (debug / expand)
  int trace;
  const uint32_t* A;
  uint32_t* O;
  uint32_t W, H, P, TR;
  uint64_t cap_runs;
  uint32_t* row_cnt;
  uint32_t* row_base;
  uint32_t* frame_runs;
  Run* runs;
};

template <int R, bool kErode>
__device__ __forceinline__ uint32_t hop(const uint32_t* row, uint32_t k, uint32_t P) {
  const uint32_t w = row[k];
  const uint32_t L = k > 0 ? row[k - 1] : 0u;
  const uint32_t Rw = k + 1 < P ? row[k + 1] : 0u;
  uint32_t h = w;
#pragma unroll
  for (int d = 1; d <= R; d++) {
    const uint32_t left = (w << d) | (L >> (32 - d));      // pixel x-d
    const uint32_t right = (w >> d) | (Rw << (32 - d));    // pixel x+d
    h = kErode ? (h & left & right) : (h | left | right);
  }
  return h;
}

template <int R, bool kErode>
__device__ __forceinline__ void morph_pass(const uint32_t* src, uint32_t* dst, uint32_t rows,
                                           uint32_t P, int ybase, uint32_t H, uint32_t lastmask,
                                           uint32_t pass) {
  const uint32_t tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const uint32_t lo = (pass + 1) * R, hi = rows - (pass + 1) * R;
  for (uint32_t rr = lo + ty; rr < hi; rr += 8) {
    const int gy = ybase + (int)rr;
    const bool in = gy >= 0 && gy < (int)H;
    for (uint32_t k = tx; k < P; k += 32) {
      uint32_t out = 0;
      if (in) {
        uint32_t acc = hop<R, kErode>(src + (rr - R) * P, k, P);
#pragma unroll
        for (int dy = 1 - R; dy <= R; dy++) {
          const uint32_t h = hop<R, kErode>(src + (rr + dy) * P, k, P);
          acc = kErode ? (acc & h) : (acc | h);
        }
        out = (k == P - 1) ? (acc & lastmask) : acc;
      }
      dst[rr * P + k] = out;
    }
  }
}

template <int R>
__global__ void __launch_bounds__(256) morph_runs_kernel(MorphArgs a) {
  extern __shared__ uint32_t sm[];
  const uint32_t P = a.P, H = a.H, TR = a.TR;
  const uint32_t rows = TR + 8 * R;
  uint32_t* b0 = sm;
  uint32_t* b1 = sm + rows * P;
  const uint32_t f = a.f0 + blockIdx.y;
  const int y0 = (int)(blockIdx.x * TR);
  const int ybase = y0 - 4 * R;
  const uint32_t tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const uint32_t lastmask = (a.W & 31u) ? ((1u << (a.W & 31u)) - 1u) : 0xFFFFFFFFu;
  const uint32_t* Af = a.A + (uint64_t)f * H * P;

  for (uint32_t rr = ty; rr < rows; rr += 8) {
    const int gy = ybase + (int)rr;
    const bool in = gy >= 0 && gy < (int)H;
    for (uint32_t k = tx; k < P; k += 32) b0[rr * P + k] = in ? __ldg(Af + (uint64_t)gy * P + k) : 0u;
  }
  __syncthreads();
  morph_pass<R, true>(b0, b1, rows, P, ybase, H, lastmask, 0);
  __syncthreads();
  morph_pass<R, false>(b1, b0, rows, P, ybase, H, lastmask, 1);
  __syncthreads();
  morph_pass<R, false>(b0, b1, rows, P, ybase, H, lastmask, 2);
  __syncthreads();
  morph_pass<R, true>(b1, b0, rows, P, ybase, H, lastmask, 3);
  __syncthreads();

  // write O and extract the runs of each output row (one warp per row)
  uint32_t* Of = a.O + (uint64_t)f * H * P;
  Run* runs = a.runs + (uint64_t)f * a.cap_runs;
  for (uint32_t i = ty; i < TR; i += 8) {
    const uint32_t gy = (uint32_t)y0 + i;
    if (gy >= H) break;
    const uint32_t* row = b0 + (4 * R + i) * P;
    // pass 1: count the row's runs
    uint32_t cnt = 0;
    for (uint32_t k0 = 0; k0 < P; k0 += 32) {
      const uint32_t k = k0 + tx;
      const uint32_t w = k < P ? row[k] : 0u;
      if (k < P) Of[(uint64_t)gy * P + k] = w;
      const uint32_t prev = (k > 0 && k <= P) ? row[k - 1] : 0u;
      cnt += __popc(w & ~((w << 1) | (prev >> 31)));
    }
    cnt = warp_sum_u32(cnt);
    uint32_t base = 0;
    if (tx == 0) {
      if (cnt) base = atomicAdd(a.frame_runs + f, cnt);
      FIZI_DCHECK(base + cnt <= a.cap_runs);
      a.row_cnt[(uint64_t)f * H + gy] = cnt;
      a.row_base[(uint64_t)f * H + gy] = base;
    }
    if (!cnt) continue;
    base = __shfl_sync(0xFFFFFFFFu, base, 0);
    // pass 2: emit (x0, x1, y); the k-th start and the k-th end pair up
    uint32_t rank_s = 0, rank_e = 0;
    for (uint32_t k0 = 0; k0 < P; k0 += 32) {
      const uint32_t k = k0 + tx;
      const uint32_t w = k < P ? row[k] : 0u;
      const uint32_t prev = (k > 0 && k <= P) ? row[k - 1] : 0u;
      const uint32_t next = k + 1 < P ? row[k + 1] : 0u;
      uint32_t st = w & ~((w << 1) | (prev >> 31));
      uint32_t en = w & ~((w >> 1) | (next << 31));
      const uint32_t ns = __popc(st), ne = __popc(en);
      uint32_t ps = ns, pe = ne;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const uint32_t u = __shfl_up_sync(0xFFFFFFFFu, ps, d);
        const uint32_t v = __shfl_up_sync(0xFFFFFFFFu, pe, d);
        if ((int)tx >= d) { ps += u; pe += v; }
      }
      uint32_t is = base + rank_s + ps - ns, ie = base + rank_e + pe - ne;
      while (st) {
        const uint32_t bit = __ffs(st) - 1;
        st &= st - 1;
        runs[is].x0 = (uint16_t)(32 * k + bit);
        runs[is].y = (uint16_t)gy;
        is++;
      }
      while (en) {
        const uint32_t bit = __ffs(en) - 1;
        en &= en - 1;
        runs[ie].x1 = (uint16_t)(32 * k + bit);
        ie++;
      }
      rank_s += __shfl_sync(0xFFFFFFFFu, ps, 31);
      rank_e += __shfl_sync(0xFFFFFFFFu, pe, 31);
    }
  }
}

// ---------------------------------------------------------------------------
// Register-pipelined variant (P <= 128 words, i.e. W <= 4096): one warp owns
// a band of kBandRows output rows of one frame and the full row width (lane l
// holds words l*WPL .. l*WPL+WPL-1).  Input rows stream through the four
// passes as a software pipeline: each pass keeps the last 2R+1 horizontally
// processed rows of its input in registers and emits row y as soon as row
// y+R arrives, so pass 4 emits row y when input row y+4R is read.  Neighbour
// words across lanes come from warp shuffles; no shared memory, no barriers.
#ifndef FIZI_BAND_ROWS
#define FIZI_BAND_ROWS 16
#endif
constexpr int kBandRows = FIZI_BAND_ROWS;

template <int WPL>
struct RowW {
  uint32_t w[WPL];
};

// lmask / rmask: all-ones except 0 on lane 0 / lane 31 (no neighbour there)
template <int R, bool kErode, int WPL>
__device__ __forceinline__ RowW<WPL> hrow(const RowW<WPL>& in, uint32_t lmask, uint32_t rmask) {
  const uint32_t left_nb = __shfl_up_sync(0xFFFFFFFFu, in.w[WPL - 1], 1) & lmask;
  const uint32_t right_nb = __shfl_down_sync(0xFFFFFFFFu, in.w[0], 1) & rmask;
  RowW<WPL> o;
#pragma unroll
  for (int j = 0; j < WPL; j++) {
    const uint32_t w = in.w[j];
    const uint32_t L = j > 0 ? in.w[j - 1] : left_nb;
    const uint32_t Rw = j + 1 < WPL ? in.w[j + 1] : right_nb;
    uint32_t h = w;
#pragma unroll
    for (int d = 1; d <= R; d++) {
      const uint32_t lft = __funnelshift_l(L, w, d);      // pixel x-d
      const uint32_t rgt = __funnelshift_r(w, Rw, d);     // pixel x+d
      h = kErode ? (h & lft & rgt) : (h | lft | rgt);
    }
    o.w[j] = h;
  }
  return o;
}

// One pass of the pipeline: the last 2R+1 horizontally processed input rows
// are kept as a set (AND / OR are commutative), row yi in slot yi mod (2R+1),
// so with the row loop unrolled by 2R+1 every slot index is static.
template <int R, bool kErode, int WPL>
struct Pass {
  RowW<WPL> win[2 * R + 1];

  __device__ __forceinline__ void init() {
#pragma unroll
    for (int i = 0; i < 2 * R + 1; i++)
#pragma unroll
      for (int j = 0; j < WPL; j++) win[i].w[j] = 0u;
  }

  template <int SLOT>
  __device__ __forceinline__ RowW<WPL> push(const RowW<WPL>& in, uint32_t lm, uint32_t rm) {
    win[SLOT] = hrow<R, kErode, WPL>(in, lm, rm);
    RowW<WPL> out;
#pragma unroll
    for (int j = 0; j < WPL; j++) {
      uint32_t acc = win[0].w[j];
#pragma unroll
      for (int i = 1; i <= 2 * R; i++) acc = kErode ? (acc & win[i].w[j]) : (acc | win[i].w[j]);
      out.w[j] = acc;
    }
    return out;
  }
};

template <int R, int WPL>
struct MorphPipe {
  const MorphArgs& a;
  uint32_t f, H, P, lastmask;
  int y0, y_end, lane;
  uint32_t lmask, rmask, wmask[WPL];       // lane-edge masks, valid bits of each word
  const uint32_t* Af;
  const uint32_t* band;                    // shared-memory copy of input rows [first, last)
                                           // (output rows overwrite consumed input rows)
  int first;
  uint32_t* Of;
  uint8_t* Mf;                             // u8 mask of the frame (W % 32 == 0) or nullptr
  Run* runs;
  Pass<R, true, WPL> p1;
  Pass<R, false, WPL> p2, p3;
  Pass<R, true, WPL> p4;
  RowW<WPL> pre[2 * R + 1];                // prefetched input rows yi .. yi + 2R

  __device__ __forceinline__ MorphPipe(const MorphArgs& args, uint32_t frame, int band0)
      : a(args), f(frame), H(args.H), P(args.P), y0(band0) {
    lane = threadIdx.x & 31;
    y_end = min((int)H, y0 + kBandRows);
    lastmask = (a.W & 31u) ? ((1u << (a.W & 31u)) - 1u) : 0xFFFFFFFFu;
    lmask = lane == 0 ? 0u : 0xFFFFFFFFu;
    rmask = lane == 31 ? 0u : 0xFFFFFFFFu;
#pragma unroll
    for (int j = 0; j < WPL; j++) {
      const uint32_t k = (uint32_t)(lane * WPL + j);
      wmask[j] = k < P ? (k == P - 1 ? lastmask : 0xFFFFFFFFu) : 0u;
    }
    Af = a.A + (uint64_t)f * H * P;
    Of = a.O + (uint64_t)f * H * P;
    Mf = (a.write_masks && a.call->masks) ? a.call->masks + (uint64_t)f * H * a.W : nullptr;
    runs = a.runs + (uint64_t)f * a.cap_runs;
    p1.init(); p2.init(); p3.init(); p4.init();
  }

  // input row yy of the band from shared memory (rows outside the band and
  // the frame are zero there)
  __device__ __forceinline__ RowW<WPL> load_row(int yy) const {
    RowW<WPL> r;
    const int i = yy - first;
    const bool rin = i >= 0 && i < (int)(kBandRows + 8 * R);
    const uint32_t* row = band + (rin ? i : 0) * (int)P + lane * WPL;
#pragma unroll
    for (int j = 0; j < WPL; j++) r.w[j] = (rin && wmask[j]) ? row[j] : 0u;
    return r;
  }

  __device__ __forceinline__ void clean(RowW<WPL>& r, int y) const {   // zero padding
    const uint32_t rowm = (y >= 0 && y < (int)H) ? 0xFFFFFFFFu : 0u;
#pragma unroll
    for (int j = 0; j < WPL; j++) r.w[j] &= wmask[j] & rowm;
  }

  // input row yi (slot = yi - first mod 2R+1); emits output row yi - 4R
  template <int SLOT>
  __device__ __forceinline__ void step(int yi) {
    const RowW<WPL> in = pre[SLOT];
    pre[SLOT] = load_row(yi + 2 * R + 1);
    RowW<WPL> o = p1.template push<SLOT>(in, lmask, rmask);
    clean(o, yi - R);
    o = p2.template push<SLOT>(o, lmask, rmask);
    clean(o, yi - 2 * R);
    o = p3.template push<SLOT>(o, lmask, rmask);
    clean(o, yi - 3 * R);
    o = p4.template push<SLOT>(o, lmask, rmask);
    const int yo = yi - 4 * R;
    if (yo >= y0 && yo < y_end) {
      clean(o, yo);
      emit(o, yo);
    }
  }

  // band whose input rows are all zero: every output row is zero
  __device__ __forceinline__ void zero_band() const {
    for (int yo = y0; yo < y_end; yo++) {
      if (a.write_zero_o)
        for (uint32_t k = lane; k < P; k += 32) Of[(uint64_t)yo * P + k] = 0u;
      if (Mf && !a.masks_zeroed) {
        uint8_t* row = Mf + (uint64_t)yo * a.W;
        for (uint32_t b = 16u * lane; b < a.W; b += 512u)
          __stcs(reinterpret_cast<uint4*>(row + b), make_uint4(0u, 0u, 0u, 0u));
      }
      if (lane == 0) {
        a.row_cnt[(uint64_t)f * H + yo] = 0u;
        a.row_base[(uint64_t)f * H + yo] = 0u;
      }
    }
  }

  // output row yo: u8 mask + O row to global memory, words kept in the band
  // buffer (the slot of input row yo was consumed long before) and the row's
  // run count in lane (yo - y0); runs are emitted after the band is done
  uint32_t my_cnt = 0;

  __device__ __forceinline__ void emit(const RowW<WPL>& o4, int yo) {
    const uint32_t prev_last = __shfl_up_sync(0xFFFFFFFFu, o4.w[WPL - 1], 1) & lmask;
    uint32_t ns = 0;
    uint32_t* slot = const_cast<uint32_t*>(band) + (yo - first) * (int)P + lane * WPL;
#pragma unroll
    for (int j = 0; j < WPL; j++) {
      const uint32_t w = o4.w[j];
      if (lane * WPL + j < (int)P) slot[j] = w;
      const uint32_t pv = j > 0 ? o4.w[j - 1] : prev_last;
      ns += __popc(w & ~((w << 1) | (pv >> 31)));
    }
    const uint32_t cnt = warp_sum_u32(ns);
    if (lane == yo - y0) my_cnt = cnt;
  }

  // after the pipeline: the band's O rows (one bulk store) and u8 mask rows
  __device__ __forceinline__ void write_rows() {
    const uint32_t* out0 = band + (y0 - first) * (int)P;
    const uint32_t nrows = (uint32_t)(y_end - y0);
    __syncwarp();
    if ((P & 3u) == 0u) {
      if (lane == 0) bulk_s2g(Of + (uint64_t)y0 * P, out0, nrows * P * 4u);
    } else {
      for (uint32_t i = lane; i < nrows * P; i += 32) Of[(uint64_t)y0 * P + i] = out0[i];
    }
    if (Mf && !a.masks_zeroed) {                        // (else the labelling kernel writes them)
      const uint32_t groups = a.W / 16;                 // 16-pixel groups per row
      for (uint32_t r = 0; r < nrows; r++) {
        const uint32_t rc = __shfl_sync(0xFFFFFFFFu, my_cnt, r);
        if (a.masks_zeroed && rc == 0u) continue;       // zero row already zeroed
        const uint32_t* row = out0 + r * P;
        uint8_t* mrow = Mf + (uint64_t)(y0 + r) * a.W;
        for (uint32_t g = lane; g < groups; g += 32) {
          const uint32_t b = (row[g >> 1] >> (16 * (g & 1))) & 0xFFFFu;
          uint4 q;
          q.x = expand4(b & 0xF); q.y = expand4((b >> 4) & 0xF);
          q.z = expand4((b >> 8) & 0xF); q.w = expand4(b >> 12);
          __stcs(reinterpret_cast<uint4*>(mrow + 16ull * g), q);
        }
      }
    }
  }

  // one atomic reservation for the band's runs, then (x0, x1, y) per run
  __device__ __forceinline__ void emit_runs() {
    uint32_t incl = my_cnt;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t u = __shfl_up_sync(0xFFFFFFFFu, incl, d);
      if (lane >= d) incl += u;
    }
    const uint32_t total = __shfl_sync(0xFFFFFFFFu, incl, 31);
    uint32_t base = 0;
    if (lane == 0 && total) base = atomicAdd(a.frame_runs + f, total);
    base = __shfl_sync(0xFFFFFFFFu, base, 0);
    const uint32_t row_base = base + incl - my_cnt;
    FIZI_DCHECK(base + total <= a.cap_runs);
    if (lane < y_end - y0) {
      a.row_cnt[(uint64_t)f * H + y0 + lane] = my_cnt;
      a.row_base[(uint64_t)f * H + y0 + lane] = my_cnt ? row_base : 0u;
    }
    if (!total) return;
    __syncwarp();
    // one lane per output row: scan the row's words (shared memory) and write
    // its runs in order; the k-th start and the k-th end of a row pair up
    if (lane < y_end - y0 && my_cnt) {
      const int yo = y0 + lane;
      const uint32_t* row = band + (yo - first) * (int)P;
      uint32_t slot = row_base, prev = 0u, x0 = 0u;
      for (uint32_t k = 0; k < P; k++) {
        const uint32_t w = row[k];
        if (w == 0u && !(prev >> 31)) { prev = w; continue; }
        const uint32_t nx = k + 1 < P ? row[k + 1] : 0u;
        uint32_t st = w & ~((w << 1) | (prev >> 31));
        uint32_t en = w & ~((w >> 1) | (nx << 31));
        while (st | en) {
          const uint32_t bs = st ? __ffs(st) - 1 : 32u, be = en ? __ffs(en) - 1 : 32u;
          if (bs <= be) {                        // a run starts (it may also end here)
            x0 = 32 * k + bs;
            st &= st - 1;
          } else {
            Run r;
            r.x0 = (uint16_t)x0; r.x1 = (uint16_t)(32 * k + be); r.y = (uint16_t)yo; r.pad = 0;
            runs[slot++] = r;
            en &= en - 1;
          }
        }
        prev = w;
      }
    }
  }
};

template <int R, int WPL, int SLOT>
__device__ __forceinline__ void unrolled_steps(MorphPipe<R, WPL>& mp, int yi, int last) {
  if constexpr (SLOT < 2 * R + 1) {
    if (yi + SLOT < last) mp.template step<SLOT>(yi + SLOT);
    unrolled_steps<R, WPL, SLOT + 1>(mp, yi, last);
  }
}

// kWarps independent warps per CTA, one band each (a warp's band depends on
// blockIdx and its warp index only, so every branch is warp-uniform and the
// warps never synchronise with each other).
__device__ unsigned long long g_morph_trace[16384][5];      // diagnostics (FIZI_MORPH_TRACE)
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

template <int R, int WPL, int kWarps>
__global__ void __launch_bounds__(32 * kWarps) morph_rows_kernel(MorphArgs a) {
  extern __shared__ uint32_t band_all[];                      // kWarps x (kBandRows + 8R) x P words
  const int warp = (int)(threadIdx.x >> 5);
  const uint32_t band_id = blockIdx.x * kWarps + warp;
  uint32_t* band = band_all + (size_t)warp * (kBandRows + 8 * R) * a.P;
  const int y0 = (int)(band_id * kBandRows);
  if (y0 >= (int)a.H) return;
  const unsigned long long t_start = a.trace ? gtimer() : 0ull;
  if ((threadIdx.x & 31) == 0) tl_mark(a.call, kTlMorph, 0);
  struct TraceEnd {
    const MorphArgs& a; unsigned long long t0; uint32_t band_id; int nz = 0;
    unsigned long long t_staged = 0, t_piped = 0;
    __device__ ~TraceEnd() {
      if ((threadIdx.x & 31) == 0) tl_mark(a.call, kTlMorph, 1);
      if (a.trace && (threadIdx.x & 31) == 0) {
        const uint32_t id = blockIdx.y * ((a.H + kBandRows - 1) / kBandRows) + band_id;
        if (id < 16384) {
          g_morph_trace[id][0] = t0; g_morph_trace[id][1] = gtimer(); g_morph_trace[id][2] = nz;
          g_morph_trace[id][3] = t_staged; g_morph_trace[id][4] = t_piped;
        }
      }
    }
  } trace_end{a, t_start, band_id};
  MorphPipe<R, WPL> mp(a, a.f0 + blockIdx.y, y0);
  const int first = y0 - 4 * R, last = mp.y_end + 4 * R;     // input rows [first, last)
  mp.band = band;
  mp.first = first;
  const uint32_t* dmap = a.dirty ? a.dirty + (uint64_t)mp.f * a.dirty_words : nullptr;
  if (dmap) {                           // zero band from the dirty-chunk bitmap, no loads
    const int r0 = max(first, 0), r1 = min(last, (int)a.H);
    const uint32_t c0 = (uint32_t)((uint64_t)r0 * a.P / 16);
    const uint32_t c1 = (uint32_t)(((uint64_t)r1 * a.P - 1) / 16);
    bool any = false;
    for (uint32_t wi = (c0 >> 5) + (threadIdx.x & 31); wi <= (c1 >> 5); wi += 32) {
      uint32_t m = __ldg(dmap + wi);
      if (wi == (c0 >> 5)) m &= 0xFFFFFFFFu << (c0 & 31);
      if (wi == (c1 >> 5) && (c1 & 31) != 31) m &= (2u << (c1 & 31)) - 1u;
      any |= m != 0u;
    }
    if (!__any_sync(0xFFFFFFFFu, any)) {
      mp.zero_band();
      return;
    }
  }
  if (dmap && (a.P & 3u) == 0) {        // TMA: the band's rows are one contiguous range
    __shared__ __align__(8) uint64_t sbars[kWarps];
    uint64_t& sbar = sbars[warp];
    const uint32_t P = a.P;
    const int r0 = max(first, 0), r1 = min(first + kBandRows + 8 * R, (int)a.H);
    const uint32_t bytes = (uint32_t)(r1 - r0) * P * 4u;
    uint32_t* dst = band + (r0 - first) * (int)P;
    if (mp.lane == 0) {
      mbar_init(&sbar, 1);
      fence_mbar_init();
      mbar_arrive_expect_tx(&sbar, bytes);
      bulk_g2s(dst, mp.Af + (uint64_t)r0 * P, bytes, &sbar, policy_evict_first());
    }
    // rows of the band outside the frame are zero
    for (uint32_t i = mp.lane; i < (uint32_t)(r0 - first) * P; i += 32) band[i] = 0u;
    const uint32_t tail0 = (uint32_t)(r1 - first) * P, tend = (uint32_t)(kBandRows + 8 * R) * P;
    for (uint32_t i = tail0 + mp.lane; i < tend; i += 32) band[i] = 0u;
    __syncwarp();
    mbar_wait(&sbar, 0);
    // words of clean chunks were not written this call: zero them
    const uint64_t w0 = (uint64_t)r0 * P, w1 = (uint64_t)r1 * P;     // frame word range
    const uint32_t c0 = (uint32_t)(w0 >> 4), c1 = (uint32_t)((w1 - 1) >> 4);
    for (uint32_t cc = c0 + mp.lane; cc <= c1; cc += 32) {
      if ((__ldg(dmap + (cc >> 5)) >> (cc & 31)) & 1u) continue;
      const uint64_t a0 = max((uint64_t)cc * 16, w0), a1 = min((uint64_t)cc * 16 + 16, w1);
      for (uint64_t wi = a0; wi < a1; wi++) dst[wi - w0] = 0u;
    }
    __syncwarp();
  } else {                              // stage the band (all loads in flight), detect zero bands
    constexpr int kRows = kBandRows + 8 * R;
    uint32_t any = 0;
    const uint32_t P = a.P;
    const int lane = mp.lane;
    uint32_t* dst = band + lane * WPL;
#pragma unroll
    for (int rr = 0; rr < kRows; rr++) {
      const int yy = first + rr;
      const bool rin = yy >= 0 && yy < (int)a.H;
      const uint32_t* src = mp.Af + (uint64_t)(rin ? yy : 0) * P + lane * WPL;
      RowW<WPL> v;
#pragma unroll
      for (int j = 0; j < WPL; j++) {
        bool ld = rin && mp.wmask[j];
        if (dmap && ld) {                // words of clean chunks are zero and unwritten
          const uint32_t c = (uint32_t)(((uint64_t)yy * P + lane * WPL + j) >> 4);
          ld = (__ldg(dmap + (c >> 5)) >> (c & 31)) & 1u;
        }
        v.w[j] = ld ? __ldg(src + j) : 0u;
      }
#pragma unroll
      for (int j = 0; j < WPL; j++) {
        if (lane * WPL + j < (int)P) dst[rr * P + j] = v.w[j];
        any |= v.w[j];
      }
    }
    if (!__any_sync(0xFFFFFFFFu, any != 0u)) {
      mp.zero_band();
      return;
    }
    __syncwarp();
  }
  trace_end.nz = 1;
  if (a.trace) trace_end.t_staged = gtimer();
#pragma unroll
  for (int q = 0; q < 2 * R + 1; q++) mp.pre[q] = mp.load_row(first + q);
  for (int yi = first; yi < last; yi += 2 * R + 1) unrolled_steps<R, WPL, 0>(mp, yi, last);
  __syncwarp();
  if (a.trace) trace_end.t_piped = gtimer();
  mp.write_rows();
  mp.emit_runs();
  if (mp.lane == 0 && (a.P & 3u) == 0u) bulk_s2g_wait();
}

uint32_t morph_tile_rows(const Ctx& c, size_t smem_budget) {
  const size_t per_row = 2ull * c.P * sizeof(uint32_t);
  const size_t max_rows = smem_budget / per_row;
  if (max_rows <= 8ull * c.p.se_radius) return 0;
  uint32_t tr = (uint32_t)(max_rows - 8ull * c.p.se_radius);
  // ~48 KB per CTA keeps 4 CTAs per SM; never fewer than 8 output rows
  const size_t target = (48 * 1024) / per_row;
  if (target > 8ull * c.p.se_radius + 8 && tr > target - 8ull * c.p.se_radius)
    tr = (uint32_t)(target - 8ull * c.p.se_radius);
  if (tr > 64) tr = 64;
  if (tr > c.H) tr = c.H;
  return tr;
}

template <int R>
static void launch_r(const MorphArgs& a, uint32_t n, size_t smem, cudaStream_t st) {
  morph_runs_kernel<R><<<dim3((a.H + a.TR - 1) / a.TR, n), 256, smem, st>>>(a);
}

cudaError_t launch_morph(Ctx& c, uint32_t f0, uint32_t n, bool write_masks, cudaStream_t st) {
  // diagnostics only (wrong results): FIZI_DIAG_SKIP=morph, see launch_slow_words
  static const bool skip = diag_skip("morph");
  if (skip) return cudaSuccess;
  MorphArgs a;
  a.f0 = f0;
  a.call = c.call;
  a.write_masks = write_masks;
  a.masks_zeroed = false;
  a.dirty = c.fast ? c.dirty : nullptr;
  a.dirty_words = c.dirty_words;
  a.write_zero_o = c.p.debug != 0;
  static const int trace = getenv("FIZI_MORPH_TRACE") ? 1 : 0;
  a.trace = trace;
  a.A = c.bitA;
  a.O = c.bitO;
  a.W = c.W; a.H = c.H; a.P = c.P; a.TR = c.morph_tr;
  a.cap_runs = c.cap_runs;
  a.row_cnt = c.row_cnt;
  a.row_base = c.row_base;
  a.frame_runs = c.frame_runs;
  a.runs = c.runs;
  const uint32_t r = c.p.se_radius;
  if (c.P <= 128 && r <= 4) {
    constexpr int kw = 4;               // warps (bands) per CTA; 1/2/8 measured no better
    const uint32_t nbands = (c.H + kBandRows - 1) / kBandRows;
    const dim3 grid((nbands + kw - 1) / kw, n);
    const size_t band_smem = (size_t)kw * (kBandRows + 8 * r) * c.P * sizeof(uint32_t);
#define FIZI_MORPH_ROWS(RR, WW) morph_rows_kernel<RR, WW, kw><<<grid, 32 * kw, band_smem, st>>>(a)
#define FIZI_MORPH_WPL(RR)                                    \
    if (c.P <= 32) FIZI_MORPH_ROWS(RR, 1);                    \
    else if (c.P <= 64) FIZI_MORPH_ROWS(RR, 2);               \
    else FIZI_MORPH_ROWS(RR, 4);
    switch (r) {
      case 1: FIZI_MORPH_WPL(1) break;
      case 2: FIZI_MORPH_WPL(2) break;
      case 3: FIZI_MORPH_WPL(3) break;
      default: FIZI_MORPH_WPL(4) break;
    }
#undef FIZI_MORPH_WPL
#undef FIZI_MORPH_ROWS
    c.launches += 1;
    return cudaGetLastError();
  }
  const size_t smem = 2ull * (a.TR + 8 * r) * c.P * sizeof(uint32_t);
  switch (r) {
    case 1: launch_r<1>(a, n, smem, st); break;
    case 2: launch_r<2>(a, n, smem, st); break;
    case 3: launch_r<3>(a, n, smem, st); break;
    case 4: launch_r<4>(a, n, smem, st); break;
    case 5: launch_r<5>(a, n, smem, st); break;
    case 6: launch_r<6>(a, n, smem, st); break;
    case 7: launch_r<7>(a, n, smem, st); break;
    default: launch_r<8>(a, n, smem, st); break;
  }
  c.launches += 1;
  return cudaGetLastError();
}

cudaError_t init_morph(Ctx& c) {
  (void)c;
  cudaError_t e = cudaSuccess;
  auto set = [&](const void* fn) {
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kMorphSmem);
  };
  // register-pipelined kernel: 4 warps x (kBandRows + 32) rows x 128 words
#define FIZI_MORPH_SET_W(RR, WW) set((const void*)morph_rows_kernel<RR, WW, 4>);
#define FIZI_MORPH_SET(RR) FIZI_MORPH_SET_W(RR, 1) FIZI_MORPH_SET_W(RR, 2) FIZI_MORPH_SET_W(RR, 4)
  FIZI_MORPH_SET(1) FIZI_MORPH_SET(2) FIZI_MORPH_SET(3) FIZI_MORPH_SET(4)
#undef FIZI_MORPH_SET
#undef FIZI_MORPH_SET_W
  set((const void*)morph_runs_kernel<1>);
  set((const void*)morph_runs_kernel<2>);
  set((const void*)morph_runs_kernel<3>);
  set((const void*)morph_runs_kernel<4>);
  set((const void*)morph_runs_kernel<5>);
  set((const void*)morph_runs_kernel<6>);
  set((const void*)morph_runs_kernel<7>);
  set((const void*)morph_runs_kernel<8>);
  for (const void* fn : {(const void*)morph_rows_kernel<1, 1, 4>, (const void*)morph_rows_kernel<1, 2, 4>,
                         (const void*)morph_rows_kernel<1, 4, 4>})
    if (e == cudaSuccess) e = set_carveout(fn);
  return e;
}

}  // namespace fizi

// diagnostics only (not part of include/fizi.h)
extern "C" int fizi_diag_morph_trace(unsigned long long* host, unsigned int n) {
  return (int)cudaMemcpyFromSymbol(host, fizi::g_morph_trace, sizeof(unsigned long long) * 5 * n);
}
