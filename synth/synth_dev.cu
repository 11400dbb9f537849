// synth/synth_dev.cu -- the device twin of synth/synth_host.c (input generator).
//
// Same integer recipe, byte-identical output (tests/test_synth.py).  Used only
// to materialise large synthetic workloads directly in HBM before a timed
// region (bench.py, large-size parity tests); it holds none of the method's
// arithmetic.  The static background plate (texture + clutter, no noise) is
// built once per call, then frames add hand, noise and gain.
#include <cstdint>
#include <cuda_runtime.h>

namespace {

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

uint64_t mix64_host(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__global__ void plate_kernel(uint32_t W, uint32_t H, uint64_t bgseed, uint32_t n_ell,
                             const int32_t* __restrict__ ell, uint8_t* __restrict__ plate) {
  uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i >= (uint64_t)W * H) return;
  uint32_t x = (uint32_t)(i % W), y = (uint32_t)(i / W);
  int tex = (int)((x * 7u + y * 3u) & 15u) - 8;
  uint64_t hc = mix64(bgseed ^ (((uint64_t)(y >> 4) << 32) | (x >> 4)));
  uint32_t k = (uint32_t)(hc % 4u);
  uint32_t h1 = (uint32_t)(hc >> 8), h2 = (uint32_t)(hc >> 24), h3 = (uint32_t)(hc >> 40);
  int r, g, b;
  if (k == 0) { int v = 80 + (int)(h1 % 50u); r = g = b = v; }
  else if (k == 1) { r = 50 + (int)(h1 % 30u); g = 80 + (int)(h2 % 30u); b = 150 + (int)(h3 % 40u); }
  else if (k == 2) { r = 60 + (int)(h1 % 30u); g = 130 + (int)(h2 % 40u); b = 70 + (int)(h3 % 30u); }
  else { r = 90 + (int)(h1 % 20u); g = 110 + (int)(h2 % 20u); b = 120 + (int)(h3 % 20u); }
  r += tex; g += tex; b += tex;
  for (uint32_t e = 0; e < n_ell; e++) {
    int64_t ex = ell[4 * e], ey = ell[4 * e + 1], ea = ell[4 * e + 2], eb = ell[4 * e + 3];
    int64_t dx = (int64_t)x - ex, dy = (int64_t)y - ey;
    if (eb * eb * dx * dx + ea * ea * dy * dy <= ea * ea * eb * eb) {
      r = 150 + tex; g = 90 + tex; b = 80 + tex;
      break;
    }
  }
  plate[3 * i] = (uint8_t)r; plate[3 * i + 1] = (uint8_t)g; plate[3 * i + 2] = (uint8_t)b;
}

__global__ void frames_kernel(uint32_t W, uint32_t H, uint64_t nseed, uint32_t noise_a,
                              const int32_t* __restrict__ pf, const uint8_t* __restrict__ plate,
                              uint8_t* __restrict__ out) {
  uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  uint32_t f = blockIdx.y;
  if (i >= (uint64_t)W * H) return;
  const int32_t* P = pf + 8 * (size_t)f;
  uint32_t x = (uint32_t)(i % W), y = (uint32_t)(i / W);
  uint64_t fseed = mix64(nseed ^ (uint64_t)(uint32_t)P[0]);
  uint32_t gain = (uint32_t)P[1];
  int64_t cx = P[2], cy = P[3], R = P[4], armw = P[5];
  int rgb[3] = {plate[3 * i], plate[3 * i + 1], plate[3 * i + 2]};
  if (R > 0) {
    int64_t dx = (int64_t)x - cx, dy = (int64_t)y - cy;
    bool in_disc = dx * dx + dy * dy <= R * R;
    bool in_arm = armw > 0 && (int64_t)y >= cy && 2 * (dx < 0 ? -dx : dx) <= armw;
    if (in_disc || in_arm) { rgb[0] = 210; rgb[1] = 120; rgb[2] = 110; }
  }
  uint64_t h = mix64(fseed ^ (((uint64_t)y << 32) | x));
  uint32_t span = 2u * noise_a + 1u;
  uint8_t* o = out + ((size_t)f * W * H + i) * 3;
#pragma unroll
  for (int c = 0; c < 3; c++) {
    int nz = noise_a ? (int)((uint32_t)((h >> (16 * c)) & 0xFFFFu) % span) - (int)noise_a : 0;
    int v = rgb[c] + nz;
    v = v < 0 ? 0 : (v > 255 ? 255 : v);
    uint32_t g = ((uint32_t)v * gain + 512u) >> 10;
    o[c] = (uint8_t)(g > 255u ? 255u : g);
  }
}

}  // namespace

extern "C" int synth_frames_dev(uint32_t W, uint32_t H, uint64_t seed, uint32_t stream,
                                uint32_t noise_a, uint32_t n, const int32_t* pf_dev,
                                uint32_t n_ell, const int32_t* ell_dev, uint8_t* plate_dev,
                                uint8_t* out_dev, cudaStream_t st) {
  if (n == 0) return 0;
  uint64_t bgseed = mix64_host(seed ^ 0xB6B6B6B6ull ^ ((uint64_t)stream << 40));
  uint64_t nseed = mix64_host(seed ^ ((uint64_t)stream * 0x9E3779B97F4A7C15ull));
  uint64_t npx = (uint64_t)W * H;
  unsigned blocks = (unsigned)((npx + 255) / 256);
  plate_kernel<<<blocks, 256, 0, st>>>(W, H, bgseed, n_ell, ell_dev, plate_dev);
  for (uint32_t f0 = 0; f0 < n; f0 += 65535u) {
    uint32_t nf = n - f0 < 65535u ? n - f0 : 65535u;
    frames_kernel<<<dim3(blocks, nf), 256, 0, st>>>(W, H, nseed, noise_a, pf_dev + 8 * (size_t)f0,
                                                    plate_dev, out_dev + (size_t)f0 * npx * 3);
  }
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : -(int)e;
}
