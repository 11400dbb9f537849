// k_morph.cu -- K4: open-close morphology on the bit-packed mask (a4).
//
// §3.1 P:138-139 "morphological operations, combining erosion and dilatation
// operators ... remove the small noisy objects and ... connect neighborhood
// zones"; reading L12: square SE of side 2r+1, O = E(D(D(E(A)))), positions
// outside the frame count as 0 for both operators.
//
// One CTA = a band of TR output rows of one frame.  The band plus a 4r-row
// halo is staged in shared memory once; the four passes run in shared memory
// (ping-pong buffers), each shrinking the valid band by r rows.  A pixel word
// (32 pixels) is processed by one thread with shifts across the neighbouring
// words: horizontal op on rows y-r..y+r, then the vertical op, fused.
#include "fizi_internal.cuh"

namespace fizi {

__device__ __forceinline__ uint32_t hop(const uint32_t* row, uint32_t k, uint32_t P, uint32_t r,
                                        bool ero) {
  const uint32_t w = row[k];
  const uint32_t L = k > 0 ? row[k - 1] : 0u;
  const uint32_t R = k + 1 < P ? row[k + 1] : 0u;
  uint32_t h = w;
  for (uint32_t d = 1; d <= r; d++) {
    const uint32_t left = (w << d) | (L >> (32 - d));     // pixel x-d
    const uint32_t right = (w >> d) | (R << (32 - d));    // pixel x+d
    h = ero ? (h & left & right) : (h | left | right);
  }
  return h;
}

__global__ void __launch_bounds__(256) morph_kernel(const uint32_t* __restrict__ A,
                                                    uint32_t* __restrict__ O, uint32_t W,
                                                    uint32_t H, uint32_t P, uint32_t r,
                                                    uint32_t TR) {
  extern __shared__ uint32_t sm[];
  const uint32_t rows = TR + 8 * r;
  uint32_t* buf[2] = {sm, sm + rows * P};
  const uint32_t f = blockIdx.y;
  const int y0 = (int)(blockIdx.x * TR);
  const int ybase = y0 - 4 * (int)r;
  const uint32_t* Af = A + (uint64_t)f * H * P;
  const uint32_t lastmask = (W & 31u) ? ((1u << (W & 31u)) - 1u) : 0xFFFFFFFFu;

  for (uint32_t i = threadIdx.x; i < rows * P; i += blockDim.x) {
    const int gy = ybase + (int)(i / P);
    buf[0][i] = (gy >= 0 && gy < (int)H) ? Af[(uint64_t)gy * P + (i % P)] : 0u;
  }
  __syncthreads();
#pragma unroll 1
  for (uint32_t j = 0; j < 4; j++) {
    const bool ero = (j == 0 || j == 3);
    const uint32_t* src = buf[j & 1];
    uint32_t* dst = buf[(j + 1) & 1];
    const uint32_t lo = (j + 1) * r, hi = rows - (j + 1) * r;
    for (uint32_t i = threadIdx.x; i < (hi - lo) * P; i += blockDim.x) {
      const uint32_t rr = lo + i / P, k = i % P;
      const int gy = ybase + (int)rr;
      uint32_t out = 0;
      if (gy >= 0 && gy < (int)H) {
        uint32_t acc = ero ? 0xFFFFFFFFu : 0u;
        for (uint32_t dy = rr - r; dy <= rr + r; dy++) {
          const uint32_t h = hop(src + dy * P, k, P, r, ero);
          acc = ero ? (acc & h) : (acc | h);
        }
        out = (k == P - 1) ? (acc & lastmask) : acc;
      }
      dst[rr * P + k] = out;
    }
    __syncthreads();
  }
  uint32_t* Of = O + (uint64_t)f * H * P;
  const uint32_t* res = buf[0];                    // pass 4 wrote buf[0]
  for (uint32_t i = threadIdx.x; i < TR * P; i += blockDim.x) {
    const uint32_t rr = 4 * r + i / P;
    const int gy = ybase + (int)rr;
    if (gy < (int)H) Of[(uint64_t)gy * P + (i % P)] = res[rr * P + (i % P)];
  }
}

uint32_t morph_tile_rows(const Ctx& c, size_t smem_budget) {
  const size_t per_row = 2ull * c.P * sizeof(uint32_t);
  const size_t max_rows = smem_budget / per_row;
  if (max_rows <= 8ull * c.p.se_radius) return 0;
  uint32_t tr = (uint32_t)(max_rows - 8ull * c.p.se_radius);
  if (tr > 64) tr = 64;
  if (tr > c.H) tr = c.H;
  return tr;
}

cudaError_t launch_morph(Ctx& c, uint32_t n, cudaStream_t st) {
  const uint32_t r = c.p.se_radius;
  const uint32_t TR = c.morph_tr;
  const size_t smem = 2ull * (TR + 8 * r) * c.P * sizeof(uint32_t);
  morph_kernel<<<dim3((c.H + TR - 1) / TR, n), 256, smem, st>>>(c.bitA, c.bitO, c.W, c.H, c.P, r, TR);
  c.launches += 1;
  return cudaGetLastError();
}

cudaError_t init_morph(Ctx& c) {
  return cudaFuncSetAttribute(morph_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              kMorphSmem);
}

}  // namespace fizi
