// k_ccl.cu -- K5/K6: connected components of the open-close mask, the
// small-blob filter, the hand blob and the final mask (a5, a6, a7).
//
// P:72 "contour detection parameters" / P:75-76 the Mouse module "tracks the
// hand corresponding zone"; readings L13-L17, L30:
// 8-connected components, canonical label = 1 + min raster index, keep iff
// area * 1e6 >= ppm * W * H, hand = largest kept (ties -> smaller label),
// centroid = (sum x / area, sum y / area).
//
// Run-based labelling, one CTA (1024 threads) per frame, working only on the
// bit-packed mask (N/8 bytes) and on horizontal runs of 1-bits:
//   1. runs per row (popcount of run starts, warp per row)
//   2. exclusive block scan -> run index of each row's first run (raster order)
//   3. emit runs (x0, x1, y): the k-th start and k-th end of a row pair up
//   4. union-find over overlapping runs of adjacent rows (|dx| <= 1 overlap =
//      8-connectivity), lock-free with atomicMin on parent (parent[g] <= g)
//   5. path flattening: parent = root = the component's first run in raster
//      order, whose first pixel is the component's min raster index
//   6. per-root area, sum x, sum y, bbox (atomics)
//   7. block reduction: #components, #kept, sum of kept areas, the largest
//   8. dropped components' runs are cleared from the mask words in place
#include "dev_util.cuh"
#include "fizi_internal.cuh"

namespace fizi {

struct CclArgs {
  uint32_t* O;
  uint32_t W, H, P;
  uint64_t N;
  uint32_t* row_cnt;
  uint32_t* row_off;
  Run* runs;
  uint32_t* parent;
  RootStats* stats;
  uint64_t cap_runs;
  fizi_result* res;
  const uint32_t* fg;
  uint32_t ppm;
};

__device__ __forceinline__ uint32_t find_root(const uint32_t* parent, uint32_t g) {
  uint32_t p = __ldcg(parent + g);
  while (p != g) {
    g = p;
    p = __ldcg(parent + g);
  }
  return g;
}

__device__ __forceinline__ void unite(uint32_t* parent, uint32_t a, uint32_t b) {
  while (true) {
    a = find_root(parent, a);
    b = find_root(parent, b);
    if (a == b) return;
    if (a < b) { const uint32_t t = a; a = b; b = t; }   // link the larger root under the smaller
    const uint32_t old = atomicMin(parent + a, b);
    if (old == a) return;
    a = old;                                             // a was re-linked concurrently: retry
  }
}

__device__ __forceinline__ bool kept_area(uint32_t area, uint32_t ppm, uint64_t N) {
  return (uint64_t)area * 1000000ull >= (uint64_t)ppm * N;
}

__global__ void __launch_bounds__(1024) ccl_kernel(CclArgs a) {
  __shared__ uint32_t s_tot;
  __shared__ uint32_t s_wsum[32];
  __shared__ unsigned long long s_best[32];
  __shared__ uint32_t s_cnt[3][32];

  const uint32_t f = blockIdx.x;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t W = a.W, H = a.H, P = a.P;
  uint32_t* Of = a.O + (uint64_t)f * H * P;
  uint32_t* rc = a.row_cnt + (uint64_t)f * H;
  uint32_t* ro = a.row_off + (uint64_t)f * (H + 1);
  Run* runs = a.runs + (uint64_t)f * a.cap_runs;
  uint32_t* parent = a.parent + (uint64_t)f * a.cap_runs;
  RootStats* stats = a.stats + (uint64_t)f * a.cap_runs;

  // 1. runs per row
  for (uint32_t y = warp; y < H; y += 32) {
    const uint32_t* row = Of + (uint64_t)y * P;
    uint32_t cnt = 0, carry = 0;
    for (uint32_t k0 = 0; k0 < P; k0 += 32) {
      const uint32_t k = k0 + lane;
      const uint32_t w = k < P ? row[k] : 0u;
      uint32_t prev = __shfl_up_sync(0xFFFFFFFFu, w, 1);
      if (lane == 0) prev = carry;
      cnt += __popc(w & ~((w << 1) | (prev >> 31)));
      carry = __shfl_sync(0xFFFFFFFFu, w, 31);
    }
    cnt = warp_sum_u32(cnt);
    if (lane == 0) rc[y] = cnt;
  }
  __syncthreads();

  // 2. exclusive scan of H row counts (each thread a contiguous segment)
  {
    const uint32_t seg = (H + 1023) / 1024;
    const uint32_t b0 = tid * seg, b1 = min(H, b0 + seg);
    uint32_t local = 0;
    for (uint32_t y = b0; y < b1; y++) local += rc[y];
    uint32_t incl = local;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t v = __shfl_up_sync(0xFFFFFFFFu, incl, d);
      if (lane >= d) incl += v;
    }
    if (lane == 31) s_wsum[warp] = incl;
    __syncthreads();
    if (warp == 0) {
      uint32_t v = s_wsum[lane], inc = v;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const uint32_t u = __shfl_up_sync(0xFFFFFFFFu, inc, d);
        if (lane >= d) inc += u;
      }
      s_wsum[lane] = inc - v;                // exclusive warp offsets
      if (lane == 31) s_tot = inc;
    }
    __syncthreads();
    uint32_t run = s_wsum[warp] + incl - local;
    for (uint32_t y = b0; y < b1; y++) {
      ro[y] = run;
      run += rc[y];
    }
    if (tid == 0) ro[H] = s_tot;
  }
  __syncthreads();
  const uint32_t T = s_tot;

  // 3. emit runs in raster order
  for (uint32_t y = warp; y < H; y += 32) {
    const uint32_t* row = Of + (uint64_t)y * P;
    const uint32_t base = ro[y];
    uint32_t rank_s = 0, rank_e = 0, carry = 0;
    for (uint32_t k0 = 0; k0 < P; k0 += 32) {
      const uint32_t k = k0 + lane;
      const uint32_t w = k < P ? row[k] : 0u;
      uint32_t prev = __shfl_up_sync(0xFFFFFFFFu, w, 1);
      if (lane == 0) prev = carry;
      uint32_t next = __shfl_down_sync(0xFFFFFFFFu, w, 1);
      if (lane == 31) next = (k0 + 32 < P) ? row[k0 + 32] : 0u;
      carry = __shfl_sync(0xFFFFFFFFu, w, 31);
      uint32_t st = w & ~((w << 1) | (prev >> 31));
      uint32_t en = w & ~((w >> 1) | (next << 31));
      const uint32_t ns = __popc(st), ne = __popc(en);
      uint32_t ps = ns, pe = ne;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const uint32_t u = __shfl_up_sync(0xFFFFFFFFu, ps, d);
        const uint32_t v = __shfl_up_sync(0xFFFFFFFFu, pe, d);
        if (lane >= d) { ps += u; pe += v; }
      }
      uint32_t is = base + rank_s + ps - ns, ie = base + rank_e + pe - ne;
      while (st) {
        const uint32_t bit = __ffs(st) - 1;
        st &= st - 1;
        runs[is].x0 = (uint16_t)(32 * k + bit);
        runs[is].y = (uint16_t)y;
        parent[is] = is;
        RootStats z;
        z.area = 0; z.xmin = 0xFFFFFFFFu; z.xmax = 0; z.ymin = 0xFFFFFFFFu; z.ymax = 0;
        z.pad = 0; z.sx = 0; z.sy = 0;
        stats[is] = z;
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
  __syncthreads();

  // 4. union overlapping runs of row y-1 (8-connectivity: [x0-1, x1+1])
  for (uint32_t g = tid; g < T; g += 1024) {
    const Run rg = runs[g];
    if (rg.y == 0) continue;
    uint32_t lo = ro[rg.y - 1], hi = ro[rg.y];
    const int x0 = (int)rg.x0 - 1, x1 = (int)rg.x1 + 1;
    while (lo < hi) {                                  // first run with x1 >= x0-1
      const uint32_t mid = (lo + hi) >> 1;
      if ((int)runs[mid].x1 < x0) lo = mid + 1; else hi = mid;
    }
    for (uint32_t h = lo, e = ro[rg.y]; h < e && (int)runs[h].x0 <= x1; h++) unite(parent, g, h);
  }
  __syncthreads();

  // 5. flatten
  for (uint32_t g = tid; g < T; g += 1024) parent[g] = find_root(parent, g);
  __syncthreads();

  // 6. per-root statistics
  for (uint32_t g = tid; g < T; g += 1024) {
    const Run rg = runs[g];
    const uint32_t root = __ldcg(parent + g);
    const uint32_t len = (uint32_t)rg.x1 - rg.x0 + 1;
    RootStats* s = stats + root;
    atomicAdd(&s->area, len);
    atomicAdd(&s->sx, (unsigned long long)((uint64_t)(rg.x0 + rg.x1) * len / 2));
    atomicAdd(&s->sy, (unsigned long long)rg.y * len);
    atomicMin(&s->xmin, (uint32_t)rg.x0);
    atomicMax(&s->xmax, (uint32_t)rg.x1);
    atomicMin(&s->ymin, (uint32_t)rg.y);
    atomicMax(&s->ymax, (uint32_t)rg.y);
  }
  __syncthreads();

  // 7. counts and the hand blob: key = area << 32 | ~label (max area, then min label)
  uint32_t n_tot = 0, n_kept = 0, fg_final = 0;
  unsigned long long best = 0;
  for (uint32_t g = tid; g < T; g += 1024) {
    if (__ldcg(parent + g) != g) continue;
    n_tot++;
    const uint32_t area = __ldcg(&stats[g].area);
    if (!kept_area(area, a.ppm, a.N)) continue;
    n_kept++;
    fg_final += area;
    const Run rg = runs[g];
    const uint32_t label = 1u + (uint32_t)rg.y * W + rg.x0;
    const unsigned long long key = ((unsigned long long)area << 32) | (0xFFFFFFFFu - label);
    best = key > best ? key : best;
  }
  n_tot = warp_sum_u32(n_tot);
  n_kept = warp_sum_u32(n_kept);
  fg_final = warp_sum_u32(fg_final);
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) {
    const unsigned long long o = __shfl_xor_sync(0xFFFFFFFFu, best, d);
    best = o > best ? o : best;
  }
  if (lane == 0) {
    s_cnt[0][warp] = n_tot;
    s_cnt[1][warp] = n_kept;
    s_cnt[2][warp] = fg_final;
    s_best[warp] = best;
  }
  __syncthreads();
  if (warp == 0) {
    n_tot = warp_sum_u32(s_cnt[0][lane]);
    n_kept = warp_sum_u32(s_cnt[1][lane]);
    fg_final = warp_sum_u32(s_cnt[2][lane]);
    best = s_best[lane];
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) {
      const unsigned long long o = __shfl_xor_sync(0xFFFFFFFFu, best, d);
      best = o > best ? o : best;
    }
    if (lane == 0) {
      fizi_result* r = a.res + f;
      r->fg_merged = a.fg[f];
      r->fg_final = fg_final;
      r->n_comp_total = n_tot;
      r->n_comp_kept = n_kept;
      if (best) {
        const uint32_t label = 0xFFFFFFFFu - (uint32_t)(best & 0xFFFFFFFFu);
        const uint32_t ly = (label - 1) / W, lx = (label - 1) % W;
        // root run = the run of row ly starting at lx: binary search
        uint32_t lo = ro[ly], hi = ro[ly + 1];
        while (lo < hi) {
          const uint32_t mid = (lo + hi) >> 1;
          if (runs[mid].x0 < lx) lo = mid + 1; else hi = mid;
        }
        const RootStats* s = stats + lo;
        const uint32_t area = __ldcg(&s->area);
        const unsigned long long sx = __ldcg(&s->sx), sy = __ldcg(&s->sy);
        r->blob_area = area;
        r->blob_label = label;
        r->bbox[0] = __ldcg(&s->xmin); r->bbox[1] = __ldcg(&s->ymin);
        r->bbox[2] = __ldcg(&s->xmax); r->bbox[3] = __ldcg(&s->ymax);
        r->sum_x = sx;
        r->sum_y = sy;
        r->cx = __ddiv_rn(__ull2double_rn(sx), __uint2double_rn(area));
        r->cy = __ddiv_rn(__ull2double_rn(sy), __uint2double_rn(area));
      }
      s_cnt[0][0] = n_tot - n_kept;          // dropped components
    }
  }
  __syncthreads();

  // 8. clear the runs of dropped components from the mask (final mask F)
  if (s_cnt[0][0] == 0) return;
  for (uint32_t g = tid; g < T; g += 1024) {
    const uint32_t root = __ldcg(parent + g);
    if (kept_area(__ldcg(&stats[root].area), a.ppm, a.N)) continue;
    const Run rg = runs[g];
    uint32_t* row = Of + (uint64_t)rg.y * P;
    for (uint32_t k = rg.x0 >> 5; k <= (uint32_t)(rg.x1 >> 5); k++) {
      const uint32_t b0 = k == (uint32_t)(rg.x0 >> 5) ? (rg.x0 & 31u) : 0u;
      const uint32_t b1 = k == (uint32_t)(rg.x1 >> 5) ? (rg.x1 & 31u) : 31u;
      const uint32_t m = (b1 == 31u ? 0xFFFFFFFFu : ((1u << (b1 + 1)) - 1u)) & ~((1u << b0) - 1u);
      atomicAnd(row + k, ~m);
    }
  }
}

cudaError_t launch_ccl(Ctx& c, uint32_t n, fizi_result* res, cudaStream_t st) {
  CclArgs a;
  a.O = c.bitO;
  a.W = c.W; a.H = c.H; a.P = c.P;
  a.N = c.N;
  a.row_cnt = c.row_cnt;
  a.row_off = c.row_off;
  a.runs = c.runs;
  a.parent = c.parent;
  a.stats = c.stats;
  a.cap_runs = c.cap_runs;
  a.res = res;
  a.fg = c.fg;
  a.ppm = c.p.min_blob_ppm;
  ccl_kernel<<<n, 1024, 0, st>>>(a);
  c.launches += 1;
  return cudaGetLastError();
}

// ------------------------------------------------- final u8 mask (a6 output)
__device__ __forceinline__ uint32_t expand4(uint32_t v) { return (v * 0x00204081u) & 0x01010101u; }

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

cudaError_t launch_expand(Ctx& c, uint32_t n, uint8_t* masks, cudaStream_t st) {
  return launch_expand_from(c, c.bitO, n, masks, st);
}

}  // namespace fizi
