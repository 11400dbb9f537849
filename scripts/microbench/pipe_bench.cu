// pipe_bench.cu -- issue rate of the instructions in the fused segmentation
// kernel's inner loop (warp instructions per SM per cycle).  Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pipe_bench pipe_bench.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kIters = 4096;
constexpr int kChains = 8;

#define BENCH(NAME, EXPR)                                                              \
  __global__ void NAME(uint32_t seed, uint32_t* out, long long* cyc) {                \
    uint32_t v[kChains];                                                               \
    _Pragma("unroll") for (int c = 0; c < kChains; c++) v[c] = seed * (c + 1) + threadIdx.x; \
    const uint32_t k1 = seed ^ 0x01020304u, k2 = seed + 0x7f7f7f7fu;                  \
    __syncthreads();                                                                   \
    long long t0 = clock64();                                                          \
    for (int i = 0; i < kIters; i++) {                                                 \
      _Pragma("unroll") for (int c = 0; c < kChains; c++) { uint32_t x = v[c]; v[c] = EXPR; } \
    }                                                                                  \
    __syncthreads();                                                                   \
    long long t1 = clock64();                                                          \
    uint32_t acc = 0;                                                                  \
    _Pragma("unroll") for (int c = 0; c < kChains; c++) acc ^= v[c];                   \
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;                                  \
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;                                   \
  }

BENCH(b_viaddmax, __viaddmax_s16x2(x, k1, k2))
BENCH(b_viaddmin, __viaddmin_s16x2(x, k1, x))
BENCH(b_vimax3, __vimax3_s16x2(x, k1, k2))
BENCH(b_dp4a, __dp4a(x, k1, x))
BENCH(b_prmt, __byte_perm(x, k1, 0x4341))
BENCH(b_lop3, (x & k1) ^ k2)
BENCH(b_iadd, x + k1)
BENCH(b_vsub2, __vsub2(x, k1))
BENCH(b_vmax2, __vmaxs2(x, k1))
BENCH(b_vabsdiff4, __vabsdiffu4(x, k1))
BENCH(b_vcmpgeu4, __vcmpgeu4(x, k1) ^ x)
BENCH(b_imad, x * k1 + k2)

__device__ __forceinline__ uint32_t sad4(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d;
  asm("vabsdiff4.u32.u32.u32.add %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}
BENCH(b_sad4, sad4(k1, x, x))
BENCH(b_vsadu4, __vsadu4(x, k1) + x)

template <typename K>
void run(const char* name, K k) {
  uint32_t* out;
  long long* cyc;
  cudaMalloc(&out, 148 * 1024 * 4);
  cudaMalloc(&cyc, 148 * 8);
  k<<<148, 1024>>>(1u, out, cyc);
  cudaDeviceSynchronize();
  k<<<148, 1024>>>(3u, out, cyc);
  long long h[148];
  cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
  double c = 0;
  for (int i = 0; i < 148; i++) c += h[i];
  c /= 148;
  const double warp_instr = 32.0 * kIters * kChains;   // per SM (32 warps)
  printf("%-12s %7.3f warp-instr/SM/clk (%.2f per SMSP)  [cycles %.0f]\n", name, warp_instr / c,
         warp_instr / c / 4, c);
  cudaFree(out);
  cudaFree(cyc);
}

int main() {
  run("viaddmax", b_viaddmax);
  run("viaddmin", b_viaddmin);
  run("vimax3", b_vimax3);
  run("dp4a", b_dp4a);
  run("prmt", b_prmt);
  run("lop3", b_lop3);
  run("iadd", b_iadd);
  run("vsub2", b_vsub2);
  run("vmaxs2", b_vmax2);
  run("vabsdiffu4", b_vabsdiff4);
  run("vcmpgeu4^", b_vcmpgeu4);
  run("imad", b_imad);
  run("sad4(ptx)", b_sad4);
  run("vsadu4+add", b_vsadu4);
  printf("status %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
