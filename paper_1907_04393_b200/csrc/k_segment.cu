// k_segment.cu -- K2+K3: brightness statistics and the three-branch test.
//
// a2 (§3.2): exact luma sum per frame -> integer mean -> gamma LUT.
// a3 (§3.1): R1 background envelope test, R2 gray-spread test,
//     R3 hue-band test, AND-merged into a bit-packed mask (bit = pixel).
//
// Fast path (W % 32 == 0): one CTA = 8 warps = 8 chunks of 512 pixels (a
// 12 KiB tile of interleaved RGB bytes) x a group of up to 32 frames of one
// stream.  The tile of every frame streams through a kStages-deep ring of
// shared-memory buffers filled by the TMA engine (cp.async.bulk, mbarrier
// completion), so every frame byte is read from HBM exactly once; warps
// release stages through a shared counter instead of a block barrier; the
// stream's envelope for the chunk is loaded once into registers and reused
// for all frames of the group.
// The luma sum is computed in the same pass (IDP.4A); the mask is computed
// speculatively with the identity LUT, which is exact for every frame whose
// mean lands in [luma_lo, luma_hi] (the common case).  The few frames outside
// are recomputed by fix_fast_kernel with their LUT after finalize_kernel has
// the means -- same arithmetic, same result as the two-pass definition.
//
// Per thread: 16 pixels = 48 bytes = 12 words.  The common case is a warp
// whose 512 pixels are all inside the envelope (background): R1 = 0, the
// AND is 0, and the warp only runs the SWAR envelope test (16-bit lanes,
// IADD3 + LOP3) and the luma dot products.  Warps with any pixel outside the
// envelope evaluate R1/R2/R3 per pixel in exact integer arithmetic (the hue is
// compared by cross-multiplication, reading L8).
#include <cstdlib>
#include <cstring>

#include "dev_util.cuh"
#include "fizi_internal.cuh"

namespace fizi {

#ifndef FIZI_MULTI_STAGES
#define FIZI_MULTI_STAGES 2
#endif
constexpr int kMultiStages = FIZI_MULTI_STAGES;   // ring depth of the multi-stream kernel

struct SegArgs {
  const CallPtrs* call;         // frames / records of the call (device)
  uint64_t frame_bytes;         // 3N
  uint64_t N;
  uint32_t nchunks, tiles, words_per_frame;
  const uint8_t* env;
  uint64_t env_plane;
  const uint32_t* frame_stream;
  const uint32_t* group_frames;
  const uint32_t* group_off;
  uint32_t* bitA;
  unsigned long long* luma;
  uint32_t* fg;
  const uint8_t* lut_table;
  const uint32_t* fix;          // [0] = count, [1..] = frame ids needing a LUT
  uint32_t S, a1, a2;
  const uint32_t* skin;         // 2^24-bit R2 & R3 colour table
  uint32_t* dirty;              // per frame: bit c = chunk c has a non-zero mask word
  uint32_t dirty_words;         // words per frame of the dirty bitmap
  bool write_zero;              // background chunks still write their zero words
  uint32_t f0, n;               // frame range of this launch (sub-batch)
  uint32_t n_groups;            // same-stream groups of this launch (items = tiles x groups)
  unsigned long long* slow_items;   // deferred words: f << 32 | (chunk * 16 + word)
  uint32_t* slow_count;             // deferred words queued by this launch
  bool persist;                 // persistent grid: CTAs take items from *item_counter
  uint32_t* item_counter;
  // in-kernel finalisation (fast path): the last CTA of a frame writes its record
  uint32_t* frame_done;         // per-frame count of finished CTAs
  const double* gtab;
  const uint8_t* ctab;
  const int64_t* frame_t;
  // NEXT-1 relearning (nullptr when no frame of the call is of a relearning
  // stream): per frame 0 = segmented with the stream's model, 1 = learning
  // frame (not segmented), 2 = segmented with a model learned in this call
  // (rl_env[f]); frames with a non-zero role are skipped by the per-pixel and
  // LUT re-test kernels and re-segmented by the reseg launch (reseg = true:
  // list = fix, envelope = rl_env[f])
  const uint32_t* rl_role;
  const uint64_t* rl_env;
  bool reseg;
};

__device__ __forceinline__ bool valid_chunk(const SegArgs& a, uint32_t c) { return c < a.nchunks; }

// a2 finalisation of frame f from its exact luma sum: integer mean, gamma,
// record header; corrected frames join the sub-batch's LUT re-test list.
__device__ __forceinline__ void finalize_frame(const SegArgs& a, uint32_t f,
                                               unsigned long long sum, uint32_t* fix,
                                               uint32_t* fg) {
  const uint32_t mean = (uint32_t)((sum + 500ull * a.N) / (1000ull * a.N));
  fizi_result r;
  memset(&r, 0, sizeof(r));
  r.t_ms = a.frame_t[f];
  r.stream = a.frame_stream[f];
  r.frame_idx = f;
  r.mean_luma = (uint8_t)mean;
  r.corrected = a.ctab[mean];
  r.gamma = a.gtab[mean];
  a.call->res[f] = r;
  if (r.corrected) {             // the LUT re-test rewrites every word of the frame
    const uint32_t pos = atomicAdd(&fix[0], 1u);
    FIZI_DCHECK(pos < a.n);
    fix[1 + pos] = f;
    fg[f] = 0;                   // the LUT re-test recounts the frame's merged pixels
  }
}

// Rec.601 weights split so every dp4a weight fits a byte:
// 299 r + 587 g + 114 b = 256 (r + 2 g) + (43 r + 75 g + 114 b).
// Word i of an interleaved run starting at a pixel boundary holds channels
// (i%3 = 0: r g b r), (1: g b r g), (2: b r g b).
__constant__ uint32_t kWlo[3] = {0x2B724B2Bu, 0x4B2B724Bu, 0x724B2B72u};
__constant__ uint32_t kWhi[3] = {0x01000201u, 0x02010002u, 0x00020100u};

struct SegArgs;
__device__ __forceinline__ bool valid_chunk(const SegArgs& a, uint32_t c);

__device__ __forceinline__ uint32_t byte_of(const uint32_t (&w)[12], int b) {
  return (w[b >> 2] >> (8 * (b & 3))) & 0xFFu;
}

// Exact R2 & R3 for one corrected pixel (readings L5, L7, L8, L9).
__device__ __forceinline__ uint32_t gray_and_skin(int r, int g, int b, int S, int a1, int a2) {
  const int M = max(r, max(g, b));
  const int m = min(r, min(g, b));
  const int C = M - m;
  int d, base;
  if (M == r) { d = g - b; base = g < b ? 360 : 0; }
  else if (M == g) { d = b - r; base = 120; }
  else { d = r - g; base = 240; }
  const int Hn = 60 * d + base * C;            // hue = Hn / C degrees
  const int lo = a1 * C, hi = a2 * C;
  const bool band = (a1 <= a2) ? (Hn >= lo && Hn <= hi) : (Hn >= lo || Hn <= hi);
  return (uint32_t)((C >= S) & (C > 0) & band);
}

// Envelope of the thread's 48 bytes, even / odd bytes in signed 16-bit
// lanes: NlX = -lo, NhX = -(hi + 1).  Per lane v + NlX >= 0 iff v >= lo and
// v + NhX < 0 iff v <= hi; the fused add + min / add + max DPX instruction
// (VIADDMNMX.S16x2) accumulates both tests over all 48 bytes.
// R2 & R3 as a function of the corrected colour only: bit (r<<16 | g<<8 | b)
// of a 2^24-bit table built once per context from the same exact integer
// test (gray_and_skin), so a per-pixel test is one load + a bit extract.
__global__ void skin_table_kernel(uint32_t* __restrict__ tab, int S, int a1, int a2) {
  const uint32_t wi = blockIdx.x * blockDim.x + threadIdx.x;    // word index, 2^19 words
  if (wi >= (1u << 19)) return;
  uint32_t w = 0;
  for (int j = 0; j < 32; j++) {
    const uint32_t c = wi * 32 + j;
    w |= gray_and_skin((int)(c >> 16), (int)((c >> 8) & 0xFF), (int)(c & 0xFF), S, a1, a2) << j;
  }
  tab[wi] = w;
}

cudaError_t launch_skin_table(Ctx& c, cudaStream_t st) {
  skin_table_kernel<<<(1u << 19) / 256, 256, 0, st>>>(c.skin_tab, (int)c.p.gray_tol_S,
                                                      (int)c.p.hue_lo_deg, (int)c.p.hue_hi_deg);
  c.launches += 1;
  return cudaGetLastError();
}

struct EnvRegs {
  uint32_t NlE[12], NlO[12], NhE[12], NhO[12];
};

__device__ __forceinline__ uint32_t even_bytes(uint32_t w) { return w & 0x00FF00FFu; }
__device__ __forceinline__ uint32_t odd_bytes(uint32_t w) { return __byte_perm(w, 0u, 0x4341); }

// per 16-bit lane: -x (x in [0, 255]), -(x + 1)
__device__ __forceinline__ uint32_t neg_lanes(uint32_t x) { return __vsub2(0u, x); }
__device__ __forceinline__ uint32_t neg1_lanes(uint32_t x) { return __vsub2(0xFFFFFFFFu, x); }

__device__ __forceinline__ void load_env(EnvRegs& e, const uint8_t* elo, const uint8_t* ehi) {
#pragma unroll
  for (int k = 0; k < 3; k++) {
    const uint4 l = __ldg(reinterpret_cast<const uint4*>(elo + 512 * k));
    const uint4 h = __ldg(reinterpret_cast<const uint4*>(ehi + 512 * k));
    const uint32_t lw[4] = {l.x, l.y, l.z, l.w}, hw[4] = {h.x, h.y, h.z, h.w};
#pragma unroll
    for (int j = 0; j < 4; j++) {
      e.NlE[4 * k + j] = neg_lanes(even_bytes(lw[j]));
      e.NlO[4 * k + j] = neg_lanes(odd_bytes(lw[j]));
      e.NhE[4 * k + j] = neg1_lanes(even_bytes(hw[j]));
      e.NhO[4 * k + j] = neg1_lanes(odd_bytes(hw[j]));
    }
  }
}

__device__ __forceinline__ void zero_env(EnvRegs& e) {
#pragma unroll
  for (int i = 0; i < 12; i++) {
    e.NlE[i] = e.NlO[i] = 0u;                 // lo = 0
    e.NhE[i] = e.NhO[i] = 0xFF00FF00u;        // hi = 255: -(256) per lane
  }
}

// per-byte inside flags of word i: bit 15 / bit 31 of the returned E / O words
__device__ __forceinline__ void r1_lanes(uint32_t w, const EnvRegs& e, int i, uint32_t& tE,
                                         uint32_t& tO) {
  const uint32_t vE = even_bytes(w), vO = odd_bytes(w);
  const uint32_t aE = __viaddmax_s16x2(vE, e.NlE[i], 0x80008000u);   // v - lo (no carry)
  const uint32_t bE = __viaddmax_s16x2(vE, e.NhE[i], 0x80008000u);   // v - hi - 1
  const uint32_t aO = __viaddmax_s16x2(vO, e.NlO[i], 0x80008000u);
  const uint32_t bO = __viaddmax_s16x2(vO, e.NhO[i], 0x80008000u);
  tE = ~aE & bE;                              // sign(v-lo) = 0 and sign(v-hi-1) = 1
  tO = ~aO & bO;
}

__device__ __forceinline__ void load48(const uint8_t* px48, bool valid, uint32_t (&fr)[12]) {
  const uint4* q = reinterpret_cast<const uint4*>(px48);
  uint4 q0 = make_uint4(0, 0, 0, 0), q1 = q0, q2 = q0;
  if (valid) { q0 = q[0]; q1 = q[1]; q2 = q[2]; }
  fr[0] = q0.x; fr[1] = q0.y; fr[2] = q0.z; fr[3] = q0.w;
  fr[4] = q1.x; fr[5] = q1.y; fr[6] = q1.z; fr[7] = q1.w;
  fr[8] = q2.x; fr[9] = q2.y; fr[10] = q2.z; fr[11] = q2.w;
}

__device__ __forceinline__ void apply_lut(uint32_t (&fr)[12], const uint8_t* lut_s) {
#pragma unroll
  for (int i = 0; i < 12; i++) {
    const uint32_t w = fr[i];
    fr[i] = (uint32_t)lut_s[w & 0xFF] | ((uint32_t)lut_s[(w >> 8) & 0xFF] << 8) |
            ((uint32_t)lut_s[(w >> 16) & 0xFF] << 16) | ((uint32_t)lut_s[w >> 24] << 24);
  }
}

// Exact sum of 299 r + 587 g + 114 b over the thread's 16 pixels.
__device__ __forceinline__ uint32_t luma16(const uint32_t (&fr)[12]) {
  uint32_t alo[4] = {0, 0, 0, 0}, ahi[4] = {0, 0, 0, 0};
#pragma unroll
  for (int i = 0; i < 12; i++) {
    alo[i & 3] = __dp4a(fr[i], kWlo[i % 3], alo[i & 3]);
    ahi[i & 3] = __dp4a(fr[i], kWhi[i % 3], ahi[i & 3]);
  }
  return (((ahi[0] + ahi[1]) + (ahi[2] + ahi[3])) << 8) + ((alo[0] + alo[1]) + (alo[2] + alo[3]));
}

// R1 on all 48 bytes: true iff every byte lies inside its envelope (then the
// 16 pixels are background and their merged bits are 0).  Running min of
// (v - lo) and max of (v - hi - 1) per 16-bit lane, four accumulator chains.
__device__ __forceinline__ bool all_inside16(const uint32_t (&fr)[12], const EnvRegs& e) {
  uint32_t amin[2] = {0x7FFF7FFFu, 0x7FFF7FFFu}, bmax[2] = {0x80008000u, 0x80008000u};
#pragma unroll
  for (int i = 0; i < 12; i++) {
    const uint32_t vE = even_bytes(fr[i]), vO = odd_bytes(fr[i]);
    amin[i & 1] = __viaddmin_s16x2(vE, e.NlE[i], amin[i & 1]);
    bmax[i & 1] = __viaddmax_s16x2(vE, e.NhE[i], bmax[i & 1]);
    amin[i & 1] = __viaddmin_s16x2(vO, e.NlO[i], amin[i & 1]);
    bmax[i & 1] = __viaddmax_s16x2(vO, e.NhO[i], bmax[i & 1]);
  }
  const uint32_t am = __vimin3_s16x2(amin[0], amin[1], amin[1]);
  const uint32_t bm = __vimax3_s16x2(bmax[0], bmax[1], bmax[1]);
  return ((am | ~bm) & 0x80008000u) == 0u;
}

// The same test from the raw envelope bytes with the byte-SIMD
// sum-of-absolute-differences instruction (VABSDIFF4.U8.ACC): for lo <= hi,
// |v - lo| + |v - hi| >= hi - lo with equality iff lo <= v <= hi, so the 48
// bytes are all inside iff sum(|v - lo| + |v - hi|) == sum(hi - lo) =: W.
// W and the lo <= hi check (sum|hi - lo| == sum hi - sum lo) are computed once
// per thread when the envelope is loaded.
struct EnvRaw {
  uint32_t lo[12], hi[12];
  uint32_t W;
  bool ordered;                               // lo <= hi for all 48 bytes
};

__device__ __forceinline__ uint32_t sad4(uint32_t a, uint32_t b, uint32_t acc) {
  uint32_t d;
  asm("vabsdiff4.u32.u32.u32.add %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(acc));
  return d;
}

__device__ __forceinline__ void load_env_raw(EnvRaw& e, const uint8_t* elo, const uint8_t* ehi) {
#pragma unroll
  for (int k = 0; k < 3; k++) {
    const uint4 l = __ldg(reinterpret_cast<const uint4*>(elo + 512 * k));
    const uint4 h = __ldg(reinterpret_cast<const uint4*>(ehi + 512 * k));
    e.lo[4 * k + 0] = l.x; e.lo[4 * k + 1] = l.y; e.lo[4 * k + 2] = l.z; e.lo[4 * k + 3] = l.w;
    e.hi[4 * k + 0] = h.x; e.hi[4 * k + 1] = h.y; e.hi[4 * k + 2] = h.z; e.hi[4 * k + 3] = h.w;
  }
  uint32_t w = 0, slo = 0, shi = 0;
#pragma unroll
  for (int i = 0; i < 12; i++) {
    w = sad4(e.lo[i], e.hi[i], w);
    slo = sad4(e.lo[i], 0u, slo);
    shi = sad4(e.hi[i], 0u, shi);
  }
  e.W = w;
  e.ordered = w == shi - slo;
}

__device__ __forceinline__ void full_env_raw(EnvRaw& e) {
#pragma unroll
  for (int i = 0; i < 12; i++) { e.lo[i] = 0u; e.hi[i] = 0xFFFFFFFFu; }
  e.W = 48u * 255u;
  e.ordered = true;
}

__device__ __forceinline__ bool all_inside_sad(const uint32_t (&fr)[12], const EnvRaw& e) {
  uint32_t acc[2] = {0u, 0u};
#pragma unroll
  for (int i = 0; i < 12; i++) {
    acc[i & 1] = sad4(fr[i], e.lo[i], acc[i & 1]);
    acc[i & 1] = sad4(fr[i], e.hi[i], acc[i & 1]);
  }
  return e.ordered && acc[0] + acc[1] == e.W;
}

// Per-pixel R1 & R2 & R3 of the thread's 16 pixels (bit p = pixel p) from the
// raw envelope bytes: per byte lo <= v <= hi (two byte-SIMD compares; lo > hi
// is never inside, L2), the three byte flags of each pixel gathered into R,
// G and B planes by byte permutes (a pixel is background iff all three are
// inside, L3), and one colour-table lookup (R2 & R3) per pixel outside.
__device__ __forceinline__ uint32_t slow_bits16_raw(const uint32_t (&fr)[12], const uint32_t (&lo)[12],
                                                    const uint32_t (&hi)[12],
                                                    const uint32_t* __restrict__ skin) {
  uint32_t m[12];
#pragma unroll
  for (int i = 0; i < 12; i++) m[i] = __vcmpgeu4(fr[i], lo[i]) & __vcmpleu4(fr[i], hi[i]);
  uint32_t outm = 0;                                   // bit p: pixel p has a byte outside
#pragma unroll
  for (int q = 0; q < 4; q++) {
    const uint32_t w0 = m[3 * q], w1 = m[3 * q + 1], w2 = m[3 * q + 2];
    const uint32_t R = __byte_perm(__byte_perm(w0, w1, 0x0630), w2, 0x5210);
    const uint32_t G = __byte_perm(__byte_perm(w0, w1, 0x0741), w2, 0x6210);
    const uint32_t B = __byte_perm(__byte_perm(w0, w1, 0x0052), w2, 0x7410);
    outm |= (((((~(R & G & B)) >> 7) & 0x01010101u) * 0x01020408u) >> 24) << (4 * q);
  }
  uint32_t bits = 0;
#pragma unroll
  for (int p = 0; p < 16; p++) {
    const int b0 = 3 * p;
    const uint32_t wl = fr[b0 >> 2], wh = fr[(b0 >> 2) + ((b0 & 3) > 1 ? 1 : 0)];
    const uint32_t o = b0 & 3;
    const uint32_t sel = ((o + 2) & 0x7) | (((o + 1) & 0x7) << 4) | ((o & 0x7) << 8) | 0x4000u;
    const uint32_t idx = __byte_perm(wl, wh, sel) & 0x00FFFFFFu;
    const uint32_t t = ((outm >> p) & 1u) ? (__ldg(skin + (idx >> 5)) >> (idx & 31)) & 1u : 0u;
    bits |= t << p;
  }
  return bits;
}

// Per-pixel R1 & R2 & R3 of the thread's 16 pixels (bit p = pixel p):
// R1 per byte from the envelope lanes, R2 & R3 from the colour table.
__device__ __forceinline__ uint32_t slow_bits16(const uint32_t (&fr)[12], const EnvRegs& e,
                                                const uint32_t* __restrict__ skin) {
  uint64_t inside = 0;
#pragma unroll
  for (int i = 0; i < 12; i++) {
    uint32_t tE, tO;
    r1_lanes(fr[i], e, i, tE, tO);
    const uint32_t f4 = ((tE >> 15) & 1u) | ((tO >> 14) & 2u) | ((tE >> 29) & 4u) | ((tO >> 28) & 8u);
    inside |= (uint64_t)f4 << (4 * i);
  }
  // colour index r<<16 | g<<8 | b of pixel p from the interleaved words
  uint32_t tw[16];
#pragma unroll
  for (int p = 0; p < 16; p++) {
    const int b0 = 3 * p;                              // byte of r
    const uint32_t lo = fr[b0 >> 2], hi = fr[(b0 >> 2) + ((b0 & 3) > 1 ? 1 : 0)];
    // bytes r, g, b sit at b0, b0+1, b0+2 of the pair (lo, hi); PRMT them into b | g<<8 | r<<16
    const uint32_t o = b0 & 3;
    const uint32_t sel = ((o + 2) & 0x7) | (((o + 1) & 0x7) << 4) | ((o & 0x7) << 8) | 0x4000u;
    const uint32_t idx = __byte_perm(lo, hi, sel) & 0x00FFFFFFu;
    tw[p] = ((inside >> b0) & 7u) == 7u ? 0u : (__ldg(skin + (idx >> 5)) >> (idx & 31)) & 1u;
  }
  uint32_t bits = 0;
#pragma unroll
  for (int p = 0; p < 16; p++) bits |= tw[p] << p;
  return bits;
}

// Process this thread's 16 pixels of one frame in one go (LUT re-test path).
template <bool kLut>
__device__ __forceinline__ uint32_t seg16(const uint8_t* px48, const EnvRegs& e, bool valid,
                                          const uint8_t* lut_s, const uint32_t* skin,
                                          uint32_t& luma_acc, bool& slow) {
  uint32_t fr[12];
  load48(px48, valid, fr);
  if (kLut) apply_lut(fr, lut_s);
  else luma_acc += luma16(fr);
  const bool all_inside = all_inside16(fr, e) || !valid;
  if (!__any_sync(0xFFFFFFFFu, !all_inside)) return 0u;   // whole warp is background
  slow = true;
  const uint32_t bits = slow_bits16(fr, e, skin);
  return valid ? bits : 0u;
}

// ---------------------------------------------------------------- fast path
// Fast path.  Work item = one 12 KiB tile (8 chunks of 512 pixels) of every
// frame of a same-stream group; CTA = 8 warps, one chunk each.  Tiles stream
// through a kStages-deep ring of shared-memory buffers filled by the TMA
// engine (cp.async.bulk, mbarrier completion).  Warps consume independently:
// each warp counts itself out of stage s when done (shared atomic); the last
// one re-issues the stage for frame i + kStages.  No block barrier inside the
// frame loop.
//
// The grid is persistent when a.persist is set: a fixed number of CTAs per
// SM take items from a per-call counter, so the kernel holds a fixed share
// of every SM for its whole duration and the pipelined tail kernels of the
// previous call run beside it in the rest.  The ring's stage / parity run on
// across items (g0 counts the frames this CTA has streamed so far).
template <int kMinBlocks, int kStages, bool kInline>
__global__ void __launch_bounds__(256, kMinBlocks) seg_fast_kernel(SegArgs a) {
  static_assert(kStages >= 2 && kStages <= kFrameGroup, "ring depth");
  extern __shared__ __align__(128) uint8_t sm[];          // kStages x 12 KiB tiles
  __shared__ __align__(8) uint64_t full[kStages];
  __shared__ uint32_t empty_cnt[kStages];
  // per-frame partial luma sums of the CTA: <= 8 warps * 512 px * 255000 < 2^32
  __shared__ uint32_t acc_y[kFrameGroup];
  __shared__ uint32_t acc_fg[kFrameGroup];                  // kInline: merged pixels per frame
  __shared__ uint32_t s_item;
  // words queued for the per-pixel kernel, staged per work item: (frame
  // index in the group, warp, word); moved to the global queue at the end of
  // the item with one reservation
  __shared__ uint16_t q_item[kFrameGroup * kWarpsPerCta * 16];
  __shared__ uint32_t q_tail, q_base;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) tl_mark(a.call, kTlSeg, 0);
  const uint8_t* frames = a.call->frames;
  const uint32_t n_items = a.tiles * a.n_groups;
  if (tid < kStages) empty_cnt[tid] = 0;
  if (tid == 0) {
#pragma unroll
    for (int s = 0; s < kStages; s++) mbar_init(&full[s], 1);
    fence_mbar_init();
  }
  uint32_t g0 = 0;                                           // frames streamed by this CTA
  for (uint32_t item = blockIdx.x;;) {
    if (a.persist) {
      if (tid == 0) s_item = atomicAdd(a.item_counter, 1u);
      __syncthreads();
      item = s_item;
    }
    if (item >= n_items) break;
    const uint32_t tile = item % a.tiles, grp = item / a.tiles;
    const uint32_t f_begin = a.group_off[grp];
    const uint32_t nf = a.group_off[grp + 1] - f_begin;
    // frame ids of the group, lane i holds frame i (nf <= kFrameGroup <= 32)
    const uint32_t fid_lane = (uint32_t)lane < nf ? a.group_frames[f_begin + lane] : 0u;
    const uint32_t stream = a.frame_stream[__shfl_sync(0xFFFFFFFFu, fid_lane, 0)];
    const uint64_t toff = (uint64_t)tile * kTileBytes;
    const uint64_t trem = a.frame_bytes - toff;
    const uint32_t tbytes = trem < (uint64_t)kTileBytes ? (uint32_t)trem : (uint32_t)kTileBytes;
    const uint32_t n_active = min((uint32_t)kWarpsPerCta, a.nchunks - tile * kWarpsPerCta);
    const uint8_t* src0 = frames + toff;
    if (tid < kFrameGroup) { acc_y[tid] = 0; acc_fg[tid] = 0; }
    if (tid == 0) q_tail = 0;
    __syncthreads();
    uint64_t pol = 0;
    if (warp == 0) {                                         // prologue: fill the ring
      pol = policy_evict_first();
#pragma unroll
      for (int k = 0; k < kStages; k++) {
        const uint32_t f = __shfl_sync(0xFFFFFFFFu, fid_lane, k);
        const uint32_t s = (g0 + k) % kStages;
        if (lane == 0 && (uint32_t)k < nf) {
          mbar_arrive_expect_tx(&full[s], tbytes);
          bulk_g2s(sm + s * kTileBytes, src0 + (uint64_t)f * a.frame_bytes, tbytes, &full[s], pol);
        }
      }
    }
    const uint32_t c = tile * kWarpsPerCta + warp;
    if (c < a.nchunks) {
      const uint64_t coff = (uint64_t)c * kChunkBytes;
      const bool valid = coff + 48u * lane < a.frame_bytes;
      EnvRaw e;
      if (valid) {
        const uint8_t* elo = a.env + (uint64_t)stream * 2 * a.env_plane + coff + 16 * lane;
        load_env_raw(e, elo, elo + a.env_plane);
      } else {
        full_env_raw(e);
      }
      if (warp != 0) pol = policy_evict_first();
      const uint8_t* my = sm + warp * kChunkBytes + 48 * lane;
      uint32_t luma_lane = 0;                                // lane i: this warp's luma of frame i
      uint32_t fg_lane = 0;                                  // kInline: lane i: merged pixels of frame i
      for (uint32_t i = 0; i < nf; i++) {
        const uint32_t gi = g0 + i;
        const uint32_t s = gi % kStages;
        const uint32_t f = __shfl_sync(0xFFFFFFFFu, fid_lane, i);
        mbar_wait(&full[s], (gi / kStages) & 1u);
        uint32_t fr[12];
        load48(my + s * kTileBytes, valid, fr);
        // the envelope test consumes all 12 words, so once every lane has it
        // the stage can be released (the luma is computed after the release)
        const bool inside = all_inside_sad(fr, e) || !valid;
        const uint32_t out_lanes = __ballot_sync(0xFFFFFFFFu, !inside);
        const uint32_t fnext = __shfl_sync(0xFFFFFFFFu, fid_lane, (i + kStages) & 31);
        if (lane == 0 && atomicAdd(&empty_cnt[s], 1u) == n_active - 1) {
          empty_cnt[s] = 0;                                  // last warp out: refill stage s
          if (i + kStages < nf) {
            mbar_arrive_expect_tx(&full[s], tbytes);
            bulk_g2s(sm + s * kTileBytes, src0 + (uint64_t)fnext * a.frame_bytes, tbytes,
                     &full[s], pol);
          }
        }
        const uint32_t y = warp_sum_u32(luma16(fr));
        if ((uint32_t)lane == i) luma_lane = y;
        // background chunks write nothing: their words are implied zero by
        // the frame's dirty bitmap (only chunks with non-zero words are
        // marked).  In a chunk touching the foreground, the words with a pixel
        // outside the envelope are queued for the per-pixel kernel (one item
        // each) and the others written as 0.
        if (kInline && out_lanes) {
          // per-pixel R1 & R2 & R3 right here, from the registers (A/B
          // variant: no queue, no re-read, but the CTA's ring advances at
          // the pace of its slowest warp)
          const uint32_t bits = inside ? 0u : slow_bits16_raw(fr, e.lo, e.hi, a.skin);
          const uint32_t word = bits | (__shfl_down_sync(0xFFFFFFFFu, bits, 1) << 16);
          const bool writer = !(lane & 1) && valid;
          const uint32_t pc = warp_sum_u32(writer ? __popc(word) : 0u);
          if ((uint32_t)lane == i) fg_lane += pc;
          if ((pc || a.write_zero) && writer)
            a.bitA[(uint64_t)f * a.words_per_frame + (uint64_t)c * 16 + (lane >> 1)] = word;
          if (pc && lane == 0)
            atomicOr(a.dirty + (uint64_t)f * a.dirty_words + (c >> 5), 1u << (c & 31));
        } else if (out_lanes) {
          const uint32_t slow_words = (out_lanes | (out_lanes >> 1)) & 0x55555555u;   // bit 2k
          uint32_t base = 0;
          if (lane == 0) base = atomicAdd(&q_tail, (uint32_t)__popc(slow_words));
          base = __shfl_sync(0xFFFFFFFFu, base, 0);
          if (!(lane & 1)) {
            const uint32_t qpos = base + __popc(slow_words & ((1u << lane) - 1u));
            if ((slow_words >> lane) & 1u) {
              FIZI_DCHECK(qpos < kFrameGroup * kWarpsPerCta * 16);
              q_item[qpos] = (uint16_t)((i << 7) | (warp << 4) | (lane >> 1));
            } else if (valid) {
              a.bitA[(uint64_t)f * a.words_per_frame + (uint64_t)c * 16 + (lane >> 1)] = 0u;
            }
          }
        } else if (a.write_zero && !(lane & 1) && valid) {
          a.bitA[(uint64_t)f * a.words_per_frame + (uint64_t)c * 16 + (lane >> 1)] = 0u;
        }
      }
      if ((uint32_t)lane < nf) {
        atomicAdd(&acc_y[lane], luma_lane);
        if (kInline && fg_lane) atomicAdd(&acc_fg[lane], fg_lane);
      }
    }
    g0 += nf;
    __syncthreads();                                         // flush the CTA's sums and queue
    const uint32_t nq = q_tail;
    if (nq) {
      if (tid == 0) q_base = atomicAdd(a.slow_count, nq);
      __syncthreads();
      const uint32_t qb = q_base;
      for (uint32_t q = tid; q < nq; q += blockDim.x) {
        const uint32_t it = q_item[q];
        const uint32_t i = it >> 7, w = (it >> 4) & 7u, k = it & 15u;
        const uint32_t f = a.group_frames[f_begin + i];
        FIZI_DCHECK(qb + q < a.n * a.nchunks * 16u && i < nf);
        a.slow_items[qb + q] = ((unsigned long long)f << 32) | ((tile * kWarpsPerCta + w) * 16u + k);
      }
    }
    if (tid < (int)nf) {
      const uint32_t f = a.group_frames[f_begin + tid];
      atomicAdd(&a.luma[f], (unsigned long long)acc_y[tid]);
      if (kInline && acc_fg[tid]) atomicAdd(&a.fg[f], acc_fg[tid]);
      __threadfence();
      if (atomicAdd(&a.frame_done[f], 1u) == a.tiles - 1) {   // last CTA of frame f
        __threadfence();
        const unsigned long long sum = atomicAdd(&a.luma[f], 0ull);
        finalize_frame(a, f, sum, const_cast<uint32_t*>(a.fix), a.fg);
      }
    }
    if (!a.persist) break;
  }
  if (tid == 0) tl_mark(a.call, kTlSeg, 1);
}

// Multi-stream calls (every same-stream group holds one frame, e.g. C5: the
// current frame of each of 256 camera streams): the envelope is read once per
// frame, so it streams exactly like the frame.  Work item = one 12 KiB tile
// of one frame; a kStages-deep ring of shared-memory stages each holds the
// frame tile and its two envelope tiles (lo, hi planes: 3 x 12 KiB), all
// three filled by TMA bulk copies on one mbarrier.  Each CTA owns a
// contiguous range of items (consecutive tiles of consecutive frames), so
// the ring is refilled without any claim: the last warp out of a stage
// issues the copies of the item kStages rounds ahead at once, then does the
// round's bookkeeping.  The luma of consecutive tiles of one frame is summed
// in shared memory and flushed to the frame's global sum (with the frame-done
// count, the last CTA of the frame finalises its record) when the frame
// changes, once per frame and CTA.  An item past the range arrives on its
// stage's barrier without data and ends the consumers.
template <int kStages, int kMinBlocks>
__global__ void __launch_bounds__(256, kMinBlocks) seg_multi_kernel(SegArgs a) {
  constexpr uint32_t kStageBytes = 3 * kTileBytes;
  extern __shared__ __align__(128) uint8_t sm[];          // kStages x (frame, lo, hi) tiles
  __shared__ __align__(8) uint64_t full[kStages];
  __shared__ uint32_t empty_cnt[kStages];
  __shared__ uint32_t acc_y[kStages];
  __shared__ uint32_t cur_f, cur_n;                        // frame being summed, its tiles so far
  __shared__ unsigned long long cur_sum;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) tl_mark(a.call, kTlSeg, 0);
  const uint8_t* frames = a.call->frames;
  const uint32_t n_items = a.tiles * a.n_groups;
  const uint32_t per = (n_items + gridDim.x - 1) / gridDim.x;
  const uint32_t it0 = min(n_items, blockIdx.x * per), it1 = min(n_items, it0 + per);
  if (tid < kStages) { empty_cnt[tid] = 0; acc_y[tid] = 0; }
  if (tid == 0) {
    cur_f = 0xFFFFFFFFu;
    cur_n = 0;
    cur_sum = 0;
#pragma unroll
    for (int s = 0; s < kStages; s++) mbar_init(&full[s], 1);
    fence_mbar_init();
  }
  __syncthreads();
  // start the copies of item `it` into stage s (or end the ring there)
  auto issue = [&](uint32_t s, uint32_t it) {
    if (it < it1) {
      const uint32_t tile = it % a.tiles, grp = it / a.tiles;
      const uint32_t f = a.group_frames[a.group_off[grp]];
      const uint32_t stream = a.frame_stream[f];
      const uint64_t toff = (uint64_t)tile * kTileBytes;
      const uint64_t trem = a.frame_bytes - toff;
      const uint32_t tbytes = trem < (uint64_t)kTileBytes ? (uint32_t)trem : (uint32_t)kTileBytes;
      const uint32_t ebytes = min((uint32_t)kWarpsPerCta, a.nchunks - tile * kWarpsPerCta) * kChunkBytes;
      const uint64_t pol = policy_evict_first();
      uint8_t* dst = sm + s * kStageBytes;
      const uint8_t* env = a.env + (uint64_t)stream * 2 * a.env_plane + toff;
      mbar_arrive_expect_tx(&full[s], tbytes + 2 * ebytes);
      bulk_g2s(dst, frames + (uint64_t)f * a.frame_bytes + toff, tbytes, &full[s], pol);
      bulk_g2s(dst + kTileBytes, env, ebytes, &full[s], pol);
      bulk_g2s(dst + 2 * kTileBytes, env + a.env_plane, ebytes, &full[s], pol);
    } else {
      mbar_arrive(&full[s]);                     // no data: the end of the range
    }
  };
  // a frame's summed tiles -> its global luma sum and done count
  auto flush = [&](uint32_t f, unsigned long long sum, uint32_t ntiles) {
    atomicAdd(&a.luma[f], sum);
    __threadfence();
    if (atomicAdd(&a.frame_done[f], ntiles) + ntiles == a.tiles) {   // frame f complete
      __threadfence();
      const unsigned long long tot = atomicAdd(&a.luma[f], 0ull);
      finalize_frame(a, f, tot, const_cast<uint32_t*>(a.fix), a.fg);
    }
  };
  if (tid == 0)
    for (int s = 0; s < kStages; s++) issue(s, it0 + s);
  for (uint32_t k = 0;; k++) {
    const uint32_t s = k % kStages;
    const uint32_t it = it0 + k;
    mbar_wait(&full[s], (k / kStages) & 1u);
    if (it >= it1) break;
    const uint32_t tile = it % a.tiles, grp = it / a.tiles;
    const uint32_t f = a.group_frames[a.group_off[grp]];
    const uint32_t c = tile * kWarpsPerCta + warp;
    if (c < a.nchunks) {
      const uint64_t coff = (uint64_t)c * kChunkBytes;
      const bool valid = coff + 48u * lane < a.frame_bytes;
      const uint8_t* st0 = sm + s * kStageBytes + warp * kChunkBytes;
      uint32_t fr[12];
      load48(st0 + 48 * lane, valid, fr);
      EnvRaw e;
      if (valid) {
#pragma unroll
        for (int q = 0; q < 3; q++) {
          const uint4 l = *reinterpret_cast<const uint4*>(st0 + kTileBytes + 512 * q + 16 * lane);
          const uint4 h = *reinterpret_cast<const uint4*>(st0 + 2 * kTileBytes + 512 * q + 16 * lane);
          e.lo[4 * q + 0] = l.x; e.lo[4 * q + 1] = l.y; e.lo[4 * q + 2] = l.z; e.lo[4 * q + 3] = l.w;
          e.hi[4 * q + 0] = h.x; e.hi[4 * q + 1] = h.y; e.hi[4 * q + 2] = h.z; e.hi[4 * q + 3] = h.w;
        }
        uint32_t w = 0, slo = 0, shi = 0;
#pragma unroll
        for (int i = 0; i < 12; i++) {
          w = sad4(e.lo[i], e.hi[i], w);
          slo = sad4(e.lo[i], 0u, slo);
          shi = sad4(e.hi[i], 0u, shi);
        }
        e.W = w;
        e.ordered = w == shi - slo;
      } else {
        full_env_raw(e);
      }
      const bool inside = all_inside_sad(fr, e) || !valid;
      const uint32_t out_lanes = __ballot_sync(0xFFFFFFFFu, !inside);
      const uint32_t y = warp_sum_u32(luma16(fr));
      if (out_lanes) {
        // words with an outside pixel go to the per-pixel kernel, the others
        // of the chunk are written as 0
        const uint32_t slow_words = (out_lanes | (out_lanes >> 1)) & 0x55555555u;   // bit 2k
        uint32_t base = 0;
        if (lane == 0) base = atomicAdd(a.slow_count, (uint32_t)__popc(slow_words));
        base = __shfl_sync(0xFFFFFFFFu, base, 0);
        if (!(lane & 1)) {
          if ((slow_words >> lane) & 1u) {
            FIZI_DCHECK(base + __popc(slow_words & ((1u << lane) - 1u)) < a.n * a.nchunks * 16u);
            a.slow_items[base + __popc(slow_words & ((1u << lane) - 1u))] =
                ((unsigned long long)f << 32) | (c * 16u + (lane >> 1));
          }
          else if (valid)
            a.bitA[(uint64_t)f * a.words_per_frame + (uint64_t)c * 16 + (lane >> 1)] = 0u;
        }
      } else if (a.write_zero && !(lane & 1) && valid) {
        a.bitA[(uint64_t)f * a.words_per_frame + (uint64_t)c * 16 + (lane >> 1)] = 0u;
      }
      if (lane == 0) atomicAdd(&acc_y[s], y);
    }
    __syncwarp();
    if (lane == 0) {
      __threadfence_block();
      if (atomicAdd(&empty_cnt[s], 1u) == kWarpsPerCta - 1) {   // last warp out of stage s
        empty_cnt[s] = 0;
        const uint32_t y = atomicExch(&acc_y[s], 0u);
        issue(s, it + kStages);                                  // refill first
        if (f != cur_f) {
          if (cur_n) flush(cur_f, cur_sum, cur_n);
          cur_f = f;
          cur_sum = 0;
          cur_n = 0;
        }
        cur_sum += y;
        cur_n += 1;
      }
    }
  }
  __syncthreads();
  if (tid == 0 && cur_n) flush(cur_f, cur_sum, cur_n);
  if (tid == 0) tl_mark(a.call, kTlSeg, 1);
}

// The words queued by the fused kernel (a pixel outside the envelope): a pair
// of lanes per word re-reads its 32 pixels and their envelope and applies R1
// per byte and R2 & R3 through the colour table.  Words of frames that get
// the LUT re-test are skipped (that kernel rewrites the whole frame).
// Grid-stride over the queue, foreground counts aggregated per frame.
// FIZI_SLOW_THREADS / FIZI_SLOW_MINB: CTA size and minimum resident CTAs per
// SM.  5 x 256 caps the kernel at 48 registers (no spill), so more of it
// co-resides with the persistent fused kernel: C4 116.8k -> 119.6k, C3 624k
// -> 636k frames/s; 128-thread CTAs at 48 / 56 registers were no better and a
// 40-register cap spills (profiles/r02_slow_words_occupancy.txt)
#ifndef FIZI_SLOW_THREADS
#define FIZI_SLOW_THREADS 256
#endif
#ifndef FIZI_SLOW_MINB
#define FIZI_SLOW_MINB 5
#endif
#define FIZI_SLOW_BOUNDS __launch_bounds__(FIZI_SLOW_THREADS, FIZI_SLOW_MINB)
__global__ void FIZI_SLOW_BOUNDS slow_words_kernel(SegArgs a) {
  const int lane = threadIdx.x & 31;
  if (threadIdx.x == 0) tl_mark(a.call, kTlSlow, 0);
  struct TlEnd {
    const CallPtrs* call;
    __device__ ~TlEnd() { if (threadIdx.x == 0) tl_mark(call, kTlSlow, 1); }
  } tl_end{a.call};
  const uint32_t count = *a.slow_count;
  const uint8_t* frames = a.call->frames;
  const int64_t single = a.call->single_stream;
  const bool any_fix = a.fix[0] != 0u;                        // frames getting the LUT re-test
  const uint32_t warps = gridDim.x * (blockDim.x >> 5);
  for (uint32_t q0 = (blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * 16u; q0 < count;
       q0 += warps * 16u) {
    const uint32_t qi = q0 + (lane >> 1);
    bool act = qi < count;
    const unsigned long long it = act ? a.slow_items[qi] : 0ull;
    const uint32_t f = (uint32_t)(it >> 32), wd = (uint32_t)it;
    const uint32_t cq = wd >> 4, k = wd & 15u;
    FIZI_DCHECK(!act || (f < a.call->n && cq < a.nchunks));
    if (act && any_fix) {
      const uint64_t mean = (a.luma[f] + 500ull * a.N) / (1000ull * a.N);
      act = a.ctab[mean] == 0;
    }
    if (act && a.rl_role) act = a.rl_role[f] == 0;       // relearn: learning / re-segmented
    const uint32_t L = 2 * k + (lane & 1);                   // lane of the chunk
    const uint64_t coff = (uint64_t)cq * kChunkBytes;
    const bool valid = act && coff + 48u * L < a.frame_bytes;
    const uint32_t stream = single >= 0 ? (uint32_t)single : (act ? a.frame_stream[f] : 0u);
    const uint8_t* elo = a.env + (uint64_t)stream * 2 * a.env_plane + coff + 16 * L;
    uint32_t lo[12], hi[12];
#pragma unroll
    for (int k = 0; k < 3; k++) {
      uint4 l = make_uint4(0, 0, 0, 0), h = make_uint4(~0u, ~0u, ~0u, ~0u);
      if (valid) {
        l = __ldg(reinterpret_cast<const uint4*>(elo + 512 * k));
        h = __ldg(reinterpret_cast<const uint4*>(elo + a.env_plane + 512 * k));
      }
      lo[4 * k] = l.x; lo[4 * k + 1] = l.y; lo[4 * k + 2] = l.z; lo[4 * k + 3] = l.w;
      hi[4 * k] = h.x; hi[4 * k + 1] = h.y; hi[4 * k + 2] = h.z; hi[4 * k + 3] = h.w;
    }
    uint32_t fr[12];
    load48(frames + (uint64_t)f * a.frame_bytes + coff + 48 * L, valid, fr);
    uint32_t bits = slow_bits16_raw(fr, lo, hi, a.skin);
    bits = valid ? bits : 0u;
    const uint32_t word = bits | (__shfl_down_sync(0xFFFFFFFFu, bits, 1) << 16);
    const bool writer = !(lane & 1) && valid;
    const uint32_t pc = writer ? __popc(word) : 0u;
    if (writer) a.bitA[(uint64_t)f * a.words_per_frame + (uint64_t)cq * 16 + k] = word;
    if (pc) atomicOr(a.dirty + (uint64_t)f * a.dirty_words + (cq >> 5), 1u << (cq & 31));
    // foreground pixels per frame: one atomic per distinct frame of the warp
    const uint32_t key = pc ? f : 0xFFFFFFFFu;
    const uint32_t grp = __match_any_sync(0xFFFFFFFFu, key);
    const uint32_t tot = __reduce_add_sync(grp, pc);
    if (pc && lane == __ffs(grp) - 1) atomicAdd(&a.fg[f], tot);
  }
}

cudaError_t launch_slow_words(Ctx& c, uint32_t f0, uint32_t n, uint32_t sub, cudaStream_t st);

// Frames whose mean luma is outside [luma_lo, luma_hi]: recompute their tiles
// with the frame's gamma LUT (persistent grid over fix-list x tiles).
__global__ void __launch_bounds__(256, 2) fix_fast_kernel(SegArgs a) {
  extern __shared__ __align__(128) uint8_t sm[];
  __shared__ __align__(8) uint64_t bar;
  __shared__ __align__(16) uint8_t lut_s[256];
  __shared__ uint32_t red_f[kWarpsPerCta];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) tl_mark(a.call, kTlFix, 0);
  const uint32_t count = a.fix[0];
  const uint64_t items = (uint64_t)count * a.tiles;
  if (blockIdx.x >= items) {
    if (tid == 0) tl_mark(a.call, kTlFix, 1);
    return;
  }
  uint64_t pol = 0;
  if (tid == 0) {
    pol = policy_evict_first();
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  __syncthreads();
  uint32_t phase = 0;
  const uint8_t* frames = a.call->frames;
  for (uint64_t it = blockIdx.x; it < items; it += gridDim.x) {
    const uint32_t f = a.fix[1 + it / a.tiles];
    FIZI_DCHECK(f < a.call->n);
    if (!a.reseg && a.rl_role && a.rl_role[f] != 0) continue;   // re-segmented by the reseg launch
    const uint32_t tile = (uint32_t)(it % a.tiles);
    const uint64_t tile_off = (uint64_t)tile * kTileBytes;
    const uint64_t rem = a.frame_bytes - tile_off;
    const uint32_t tile_bytes = rem < (uint64_t)kTileBytes ? (uint32_t)rem : (uint32_t)kTileBytes;
    if (tid == 0) {
      mbar_arrive_expect_tx(&bar, tile_bytes);
      bulk_g2s(sm, frames + (uint64_t)f * a.frame_bytes + tile_off, tile_bytes, &bar, pol);
    }
    const uint64_t mean = (a.luma[f] + 500ull * a.N) / (1000ull * a.N);
    if (tid < 64)
      reinterpret_cast<uint32_t*>(lut_s)[tid] =
          reinterpret_cast<const uint32_t*>(a.lut_table + mean * 256)[tid];
    const uint32_t c = tile * kWarpsPerCta + warp;
    const bool valid = (uint64_t)c * kChunkBytes + 48u * lane < a.frame_bytes;
    const uint32_t stream = a.frame_stream[f];
    EnvRegs e;
    if (valid) {
      const uint8_t* env = (a.reseg && a.rl_role[f] == 2) ? reinterpret_cast<const uint8_t*>(a.rl_env[f])
                                                          : a.env + (uint64_t)stream * 2 * a.env_plane;
      const uint8_t* elo = env + (uint64_t)c * kChunkBytes + 16 * lane;
      load_env(e, elo, elo + a.env_plane);
    } else {
      zero_env(e);
    }
    __syncthreads();                          // LUT in shared memory
    mbar_wait(&bar, phase);
    uint32_t y = 0;
    bool slow = false;
    const bool learning = a.reseg && a.rl_role[f] == 1;       // NEXT-1 learning frame: empty
    const uint32_t bits = learning ? 0u : seg16<true>(sm + warp * kChunkBytes + 48 * lane, e, valid,
                                                      lut_s, a.skin, y, slow);
    const uint32_t word = bits | (__shfl_down_sync(0xFFFFFFFFu, bits, 1) << 16);
    uint32_t pc = 0;
    if (!(lane & 1) && valid) {
      a.bitA[(uint64_t)f * a.words_per_frame + (uint64_t)c * 16 + (lane >> 1)] = word;
      pc = __popc(word);
    }
    pc = warp_sum_u32(pc);
    if (lane == 0) {
      red_f[warp] = pc;
      if (pc && valid_chunk(a, c)) atomicOr(a.dirty + (uint64_t)f * a.dirty_words + (c >> 5), 1u << (c & 31));
    }
    __syncthreads();
    if (tid == 0) {
      uint32_t sf = 0;
      for (int w = 0; w < kWarpsPerCta; w++) sf += red_f[w];
      if (sf) atomicAdd(&a.fg[f], sf);
    }
    __syncthreads();                          // smem tile + LUT reused next item
    phase ^= 1u;
  }
  if (tid == 0) tl_mark(a.call, kTlFix, 1);
}

// The LUT re-test of corrected frames (and NEXT-1's re-segmented / learning
// frames, reseg = true) as a streaming kernel: work item = one 12 KiB tile of
// a listed frame; a 2-deep ring of stages per CTA, two CTAs per SM, each
// stage holding the frame tile, its two envelope tiles and the frame's
// 256-byte LUT row, all four filled by TMA bulk copies on one mbarrier; each
// CTA owns a contiguous range of the (frames x tiles) items.  Every word of a
// listed frame is rewritten (the fused kernel's identity-LUT words are void
// for it); words whose 16-pixel lanes are all inside are written as 0
// without the per-pixel test.  Items of frames another launch handles arrive
// on their stage without data and are skipped.
constexpr int kFixStages = 2;
constexpr uint32_t kFixStageBytes = 3 * kTileBytes + 256;
__global__ void __launch_bounds__(256, 2) fix_ring_kernel(SegArgs a) {
  extern __shared__ __align__(128) uint8_t sm[];           // kFixStages x (tile, lo, hi, LUT)
  __shared__ __align__(8) uint64_t full[kFixStages];
  __shared__ uint32_t empty_cnt[kFixStages];
  __shared__ uint32_t st_skip[kFixStages];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) tl_mark(a.call, kTlFix, 0);
  const uint32_t count = a.fix[0];
  const uint32_t n_items = count * a.tiles;
  const uint32_t per = (n_items + gridDim.x - 1) / gridDim.x;
  const uint32_t it0 = min(n_items, blockIdx.x * per), it1 = min(n_items, it0 + per);
  if (it0 >= it1) {
    if (tid == 0) tl_mark(a.call, kTlFix, 1);
    return;
  }
  if (tid < kFixStages) { empty_cnt[tid] = 0; st_skip[tid] = 0; }
  if (tid == 0) {
#pragma unroll
    for (int s = 0; s < kFixStages; s++) mbar_init(&full[s], 1);
    fence_mbar_init();
  }
  __syncthreads();
  const uint8_t* frames = a.call->frames;
  auto frame_of = [&](uint32_t it) { return a.fix[1 + it / a.tiles]; };
  auto skip_of = [&](uint32_t f) {
    return a.reseg ? a.rl_role[f] == 1u : (a.rl_role != nullptr && a.rl_role[f] != 0u);
  };
  auto issue = [&](uint32_t s, uint32_t it) {
    if (it >= it1) { mbar_arrive(&full[s]); return; }
    const uint32_t f = frame_of(it);
    if (skip_of(f)) {                           // nothing to load (skipped or emptied below)
      st_skip[s] = 1;
      mbar_arrive(&full[s]);
      return;
    }
    st_skip[s] = 0;
    const uint32_t tile = it % a.tiles;
    const uint64_t toff = (uint64_t)tile * kTileBytes;
    const uint64_t trem = a.frame_bytes - toff;
    const uint32_t tbytes = trem < (uint64_t)kTileBytes ? (uint32_t)trem : (uint32_t)kTileBytes;
    const uint32_t ebytes = min((uint32_t)kWarpsPerCta, a.nchunks - tile * kWarpsPerCta) * kChunkBytes;
    const uint8_t* env = (a.reseg && a.rl_role[f] == 2u)
                             ? reinterpret_cast<const uint8_t*>(a.rl_env[f])
                             : a.env + (uint64_t)a.frame_stream[f] * 2 * a.env_plane;
    const uint64_t mean = (a.luma[f] + 500ull * a.N) / (1000ull * a.N);
    const uint64_t pol = policy_evict_first();
    uint8_t* dst = sm + s * kFixStageBytes;
    mbar_arrive_expect_tx(&full[s], tbytes + 2 * ebytes + 256);
    bulk_g2s(dst, frames + (uint64_t)f * a.frame_bytes + toff, tbytes, &full[s], pol);
    bulk_g2s(dst + kTileBytes, env + toff, ebytes, &full[s], pol);
    bulk_g2s(dst + 2 * kTileBytes, env + a.env_plane + toff, ebytes, &full[s], pol);
    bulk_g2s(dst + 3 * kTileBytes, a.lut_table + mean * 256, 256, &full[s], pol);
  };
  if (tid == 0)
    for (int s = 0; s < kFixStages; s++) issue(s, it0 + s);
  for (uint32_t k = 0;; k++) {
    const uint32_t s = k % kFixStages;
    const uint32_t it = it0 + k;
    mbar_wait(&full[s], (k / kFixStages) & 1u);
    if (it >= it1) break;
    const uint32_t f = frame_of(it);
    const uint32_t tile = it % a.tiles;
    const uint32_t c = tile * kWarpsPerCta + warp;
    const bool skipped = *reinterpret_cast<volatile uint32_t*>(&st_skip[s]) != 0u;
    if (c < a.nchunks && (!skipped || a.reseg)) {
      const uint64_t coff = (uint64_t)c * kChunkBytes;
      const bool valid = coff + 48u * lane < a.frame_bytes;
      uint32_t bits = 0;
      if (!skipped) {                           // (a skipped reseg item is a learning frame: empty)
        const uint8_t* st0 = sm + s * kFixStageBytes + warp * kChunkBytes;
        const uint8_t* lut_s = sm + s * kFixStageBytes + 3 * kTileBytes;
        uint32_t fr[12];
        load48(st0 + 48 * lane, valid, fr);
        apply_lut(fr, lut_s);
        EnvRaw e;
        if (valid) {
#pragma unroll
          for (int q = 0; q < 3; q++) {
            const uint4 l = *reinterpret_cast<const uint4*>(st0 + kTileBytes + 512 * q + 16 * lane);
            const uint4 h = *reinterpret_cast<const uint4*>(st0 + 2 * kTileBytes + 512 * q + 16 * lane);
            e.lo[4 * q + 0] = l.x; e.lo[4 * q + 1] = l.y; e.lo[4 * q + 2] = l.z; e.lo[4 * q + 3] = l.w;
            e.hi[4 * q + 0] = h.x; e.hi[4 * q + 1] = h.y; e.hi[4 * q + 2] = h.z; e.hi[4 * q + 3] = h.w;
          }
          uint32_t w = 0, slo = 0, shi = 0;
#pragma unroll
          for (int i = 0; i < 12; i++) {
            w = sad4(e.lo[i], e.hi[i], w);
            slo = sad4(e.lo[i], 0u, slo);
            shi = sad4(e.hi[i], 0u, shi);
          }
          e.W = w;
          e.ordered = w == shi - slo;
        } else {
          full_env_raw(e);
        }
        const bool inside = all_inside_sad(fr, e) || !valid;
        if (__any_sync(0xFFFFFFFFu, !inside))
          bits = inside ? 0u : slow_bits16_raw(fr, e.lo, e.hi, a.skin);
      }
      const uint32_t word = bits | (__shfl_down_sync(0xFFFFFFFFu, bits, 1) << 16);
      const bool writer = !(lane & 1) && valid;
      if (writer) a.bitA[(uint64_t)f * a.words_per_frame + (uint64_t)c * 16 + (lane >> 1)] = word;
      const uint32_t pc = warp_sum_u32(writer ? __popc(word) : 0u);
      if (pc && lane == 0) {
        atomicAdd(&a.fg[f], pc);
        atomicOr(a.dirty + (uint64_t)f * a.dirty_words + (c >> 5), 1u << (c & 31));
      }
    }
    __syncwarp();
    if (lane == 0) {
      __threadfence_block();
      if (atomicAdd(&empty_cnt[s], 1u) == kWarpsPerCta - 1) {   // last warp out of stage s
        empty_cnt[s] = 0;
        issue(s, it + kFixStages);
      }
    }
  }
  if (tid == 0) tl_mark(a.call, kTlFix, 1);
}

// ------------------------------------------------------------- generic path
// Any width: thread per pixel for the luma sum, warp per 32-pixel word of a
// bit-mask row for the branch tests (ballot), after the means are known.
__global__ void luma_generic_kernel(const CallPtrs* call, uint64_t N, uint32_t f0,
                                    unsigned long long* __restrict__ luma) {
  const uint8_t* frames = call->frames;
  const uint64_t q = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  const uint32_t f = f0 + blockIdx.y;
  uint32_t y = 0;
  if (q < N) {
    const uint8_t* p = frames + ((uint64_t)f * N + q) * 3;
    y = 299u * p[0] + 587u * p[1] + 114u * p[2];
  }
  y = warp_sum_u32(y);
  if ((threadIdx.x & 31) == 0 && y) atomicAdd(&luma[f], (unsigned long long)y);
}

__global__ void mask_generic_kernel(SegArgs a, uint32_t W, uint32_t H, uint32_t P, uint32_t n) {
  const uint64_t gw = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const uint64_t per_frame = (uint64_t)H * P;
  if (gw >= per_frame * n) return;
  const uint32_t f = a.f0 + (uint32_t)(gw / per_frame);
  const uint32_t rw = (uint32_t)(gw % per_frame);
  const uint32_t yrow = rw / P, k = rw % P;
  const uint32_t x = 32 * k + lane;
  const uint64_t mean = (a.luma[f] + 500ull * a.N) / (1000ull * a.N);
  const uint8_t* L = a.lut_table + mean * 256;      // identity row when not corrected
  uint32_t bit = 0;
  if (x < W) {
    const uint64_t q = (uint64_t)yrow * W + x;
    const uint8_t* p = a.call->frames + ((uint64_t)f * a.N + q) * 3;
    const uint32_t stream = a.frame_stream[f];
    const uint32_t role = a.rl_role ? a.rl_role[f] : 0u;
    const uint8_t* env = role == 2 ? reinterpret_cast<const uint8_t*>(a.rl_env[f])
                                   : a.env + (uint64_t)stream * 2 * a.env_plane;
    const uint8_t* lo = env + q * 3;
    const uint8_t* hi = lo + a.env_plane;
    const int r = L[p[0]], g = L[p[1]], b = L[p[2]];
    const bool inside = r >= lo[0] && r <= hi[0] && g >= lo[1] && g <= hi[1] && b >= lo[2] &&
                        b <= hi[2];
    bit = role == 1 ? 0u : (uint32_t)!inside & gray_and_skin(r, g, b, (int)a.S, (int)a.a1, (int)a.a2);
  }
  const uint32_t word = __ballot_sync(0xFFFFFFFFu, bit);
  if (lane == 0) {
    a.bitA[(uint64_t)f * per_frame + rw] = word;
    if (word) atomicAdd(&a.fg[f], (uint32_t)__popc(word));
  }
}

// ------------------------------------------------------------ finalize (a2)
__global__ void finalize_kernel(uint32_t f0, uint32_t n, uint64_t N,
                                const unsigned long long* __restrict__ luma,
                                uint32_t* __restrict__ fg, const double* __restrict__ gtab,
                                const uint8_t* __restrict__ ctab,
                                const uint32_t* __restrict__ frame_stream,
                                const int64_t* __restrict__ frame_t, const CallPtrs* call,
                                uint32_t* __restrict__ fix) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint32_t f = f0 + i;
  const uint32_t mean = (uint32_t)((luma[f] + 500ull * N) / (1000ull * N));
  fizi_result r;
  memset(&r, 0, sizeof(r));
  r.t_ms = frame_t[f];
  r.stream = frame_stream[f];
  r.frame_idx = f;
  r.mean_luma = (uint8_t)mean;
  r.corrected = ctab[mean];
  r.gamma = gtab[mean];
  call->res[f] = r;
  if (r.corrected) {
    const uint32_t pos = atomicAdd(&fix[0], 1u);
    FIZI_DCHECK(pos < n);
    fix[1 + pos] = f;
    fg[f] = 0;
  }
}

static SegArgs seg_args(Ctx& c, uint32_t f0, uint32_t n, uint32_t g0, uint32_t sub) {
  SegArgs a;
  a.call = c.call;
  a.frame_bytes = c.N * 3;
  a.N = c.N;
  a.nchunks = c.nchunks;
  a.tiles = (c.nchunks + kWarpsPerCta - 1) / kWarpsPerCta;
  a.words_per_frame = c.H * c.P;
  a.env = c.env;
  a.env_plane = c.env_plane;
  a.frame_stream = c.frame_stream;
  a.group_frames = c.group_frames;
  a.group_off = c.group_off + g0;
  a.bitA = c.bitA;
  a.luma = c.luma;
  a.fg = c.fg;
  a.lut_table = c.lut;
  a.fix = c.fix_count + (uint64_t)sub * (c.max_batch + 1);
  a.slow_items = c.slow_items + (uint64_t)f0 * c.nchunks * 16;
  a.slow_count = c.slow_count + sub;
  a.S = c.p.gray_tol_S;
  a.a1 = c.p.hue_lo_deg;
  a.a2 = c.p.hue_hi_deg;
  a.skin = c.skin_tab;
  a.dirty = c.dirty;
  a.dirty_words = c.dirty_words;
  a.write_zero = !c.use_dirty;
  a.f0 = f0;
  a.n = n;
  a.frame_done = c.frame_done;
  a.gtab = c.gamma_tab;
  a.ctab = c.corr_tab;
  a.frame_t = c.frame_t;
  a.rl_role = c.rl_active ? c.rl_role : nullptr;
  a.rl_env = c.rl_env;
  a.reseg = false;
  return a;
}

// a2 + a3 main pass over frames [f0, f0+n) (same-stream groups g0 .. g0+ng-1).
cudaError_t launch_seg_main(Ctx& c, uint32_t f0, uint32_t n, uint32_t g0, uint32_t ng,
                            uint32_t sub, cudaStream_t st) {
  SegArgs a = seg_args(c, f0, n, g0, sub);
  prof_begin(c, st);
  if (c.fast) {
    a.n_groups = ng;
    a.item_counter = c.item_counter + sub;
    const uint32_t items = a.tiles * ng;
    // persistent grid of c.seg_persist CTAs per SM (0: one CTA per item)
    const uint32_t per_sm = c.seg_persist;
    static const uint32_t grid_env = getenv("FIZI_SEG_GRID") ? (uint32_t)atoi(getenv("FIZI_SEG_GRID")) : 0u;
    // default: 2.5 CTAs per SM (half of the SMs keep room for the previous
    // call's tail kernels beside the fused kernel)
    const uint32_t pgrid = grid_env ? grid_env : (uint32_t)c.sms * per_sm / 2u;
    a.persist = pgrid > 0 && items > pgrid;
    const uint32_t grid = a.persist ? pgrid : items;
    if (ng == n && n > 1) {
      // one frame per same-stream group (multi-stream call): the envelope
      // streams with the frame through the TMA ring
      a.persist = true;
      // two CTAs per SM, each a 2-deep ring of 36 KiB stages (measured on
      // C5: 1.69M frames/s, vs 1.54M with one CTA per SM and a 4-deep ring,
      // 1.61M with 2 x 3-deep, 1.58M with 3 x 2-deep; FIZI_MULTI_CFG=1
      // selects the 1 x 4-deep variant)
      static const int cfg = getenv("FIZI_MULTI_CFG") ? atoi(getenv("FIZI_MULTI_CFG")) : 0;
      if (cfg == 1)
        seg_multi_kernel<4, 1><<<c.sms, 256, 4 * 3 * kTileBytes, st>>>(a);
      else
        seg_multi_kernel<kMultiStages, 2><<<2 * c.sms, 256, kMultiStages * 3 * kTileBytes, st>>>(a);
    } else {
      // 3 CTAs/SM x 4-deep ring; FIZI_INLINE=1: per-pixel words inside (A/B)
      // (ring depth 2 / 6 measured: C3 606k / 551k vs 623k frames/s)
      if (c.inline_words) seg_fast_kernel<3, 4, true><<<grid, 256, 4 * kTileBytes, st>>>(a);
      else seg_fast_kernel<3, 4, false><<<grid, 256, 4 * kTileBytes, st>>>(a);
    }
  } else {
    luma_generic_kernel<<<dim3((unsigned)((c.N + 255) / 256), n), 256, 0, st>>>(c.call, c.N, f0,
                                                                                c.luma);
  }
  prof_end(c, FIZI_PROF_SEGMENT, st);
  c.launches += 1;
  return cudaGetLastError();
}

cudaError_t launch_slow_words(Ctx& c, uint32_t f0, uint32_t n, uint32_t sub, cudaStream_t st) {
  // diagnostics only (wrong results): FIZI_DIAG_SKIP=slow measures the
  // pipeline without this stage, an upper bound for speeding it up
  static const bool skip = diag_skip("slow");
  if (skip) return cudaSuccess;
  SegArgs a = seg_args(c, f0, n, 0, sub);
  prof_begin(c, st);
  // colour-table test (an arithmetic R2 & R3 test kept the ALU pipe 83 %
  // busy on C4 and was slower: 290 vs 223 us per C4 call in round 1)
  // grid-stride over the queue with 16 CTAs per SM (5 resident alone; the
  // rest fill in beside the fused kernel): 8 / 16 / 32 per SM measured C4
  // 119.6k / 121.2k / 120.6k, C2 713k / 728k / 731k, C3 633k / 633k / 630k
  // (FIZI_SLOW_GRID, profiles/r02_slow_words_grid.txt)
  static const uint32_t per_sm = getenv("FIZI_SLOW_GRID") ? (uint32_t)atoi(getenv("FIZI_SLOW_GRID")) : 16u;
  slow_words_kernel<<<c.sms * per_sm * (256 / FIZI_SLOW_THREADS), FIZI_SLOW_THREADS, 0, st>>>(a);
  prof_end(c, FIZI_PROF_SLOW, st);
  c.launches += 1;
  return cudaGetLastError();
}

// a2 finalisation (mean -> gamma, record header) and the LUT re-test of the
// sub-batch's corrected frames (fast path) / the branch tests (generic path).
// NEXT-1: the frames segmented with a model learned in this call (role 2),
// recomputed with their LUT against that model (fast path; the generic path
// handles roles inside mask_generic_kernel)
cudaError_t launch_relearn_reseg(Ctx& c, uint32_t n, cudaStream_t st) {
  if (!c.fast) return cudaSuccess;
  SegArgs a = seg_args(c, 0, n, 0, 0);
  a.fix = c.rl_list;
  a.reseg = true;
  fix_ring_kernel<<<2 * c.sms, 256, kFixStages * kFixStageBytes, st>>>(a);
  c.launches += 1;
  return cudaGetLastError();
}

cudaError_t launch_seg_fix(Ctx& c, uint32_t f0, uint32_t n, uint32_t sub, cudaStream_t st) {
  SegArgs a = seg_args(c, f0, n, 0, sub);
  prof_begin(c, st);
  if (c.fast) {                      // finalisation already done by the fused kernel
    static const bool old_fix = getenv("FIZI_FIX_OLD") != nullptr;   // A/B: round-1 kernel
    if (old_fix) fix_fast_kernel<<<c.sms, 256, kTileBytes, st>>>(a);
    else fix_ring_kernel<<<2 * c.sms, 256, kFixStages * kFixStageBytes, st>>>(a);
    c.launches += 1;
  } else {
    const unsigned fin_blocks = (n + 255) / 256;
    finalize_kernel<<<fin_blocks, 256, 0, st>>>(f0, n, c.N, c.luma, c.fg, c.gamma_tab, c.corr_tab,
                                                 c.frame_stream, c.frame_t, c.call,
                                                 const_cast<uint32_t*>(a.fix));
    if (c.rl_active) {               // roles need the means (NEXT-1)
      cudaError_t e = launch_relearn_plan(c, n, st);
      if (e != cudaSuccess) return e;
    }
    const uint64_t warps = (uint64_t)c.H * c.P * n;
    mask_generic_kernel<<<(unsigned)((warps * 32 + 255) / 256), 256, 0, st>>>(a, c.W, c.H, c.P, n);
    c.launches += 2;
  }
  prof_end(c, FIZI_PROF_FIXUP, st);
  return cudaGetLastError();
}

cudaError_t init_segment(Ctx& c) {
  (void)c;
  cudaError_t e = cudaFuncSetAttribute(seg_fast_kernel<3, 4, false>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * kTileBytes);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(seg_fast_kernel<3, 4, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             4 * kTileBytes);

  c.inline_words = getenv("FIZI_INLINE") != nullptr && atoi(getenv("FIZI_INLINE")) == 1;
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(seg_multi_kernel<kMultiStages, 2>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, kMultiStages * 3 * kTileBytes);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(seg_multi_kernel<4, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             4 * 3 * kTileBytes);
  const char* ps = getenv("FIZI_SEG_PERSIST");          // experiment switch
  c.seg_persist = ps ? 2u * (uint32_t)atoi(ps) : 5u;      // in half CTAs per SM
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(fix_fast_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kTileBytes);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(fix_ring_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             kFixStages * kFixStageBytes);
  for (const void* fn : {(const void*)seg_fast_kernel<3, 4, false>, (const void*)seg_fast_kernel<3, 4, true>,
                         (const void*)seg_multi_kernel<kMultiStages, 2>, (const void*)seg_multi_kernel<4, 1>,
                         (const void*)fix_ring_kernel, (const void*)slow_words_kernel})
    if (e == cudaSuccess) e = set_carveout(fn);
  return e;
}

}  // namespace fizi
