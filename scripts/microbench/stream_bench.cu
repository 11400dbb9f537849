// stream_bench.cu -- how fast can the fused kernel's access pattern stream?
// Reads 64 frames of 1920x1080x3 bytes (398 MB) with the fused kernel's
// tiling (12 KiB tiles x groups of frames) and no pixel work, to separate
// memory-pipeline limits from compute limits.  Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o stream_bench stream_bench.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile("{\n .reg .pred p;\nW_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W_%=;\n}\n"
               ::"r"(smem_u32(bar)), "r"(parity) : "memory");
}

constexpr uint64_t FB = 1920ull * 1080 * 3;
constexpr int NF = 64;

// A: CTA ring of STAGES x TILE bytes, released by a warp counter (as the fused kernel)
template <int STAGES, int TILE>
__global__ void __launch_bounds__(256) tma_ring(const uint8_t* frames, int group, uint32_t* sink) {
  extern __shared__ __align__(128) uint8_t sm[];
  __shared__ __align__(8) uint64_t full[STAGES];
  __shared__ uint32_t cnt[STAGES];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint64_t toff = (uint64_t)blockIdx.x * TILE;
  const uint32_t tb = (uint32_t)min((uint64_t)TILE, FB - toff);
  const int f0 = blockIdx.y * group;
  if (tid < STAGES) { cnt[tid] = 0; mbar_init(&full[tid], 1); }
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();
  if (tid == 0)
    for (int s = 0; s < STAGES && s < group; s++) {
      mbar_expect(&full[s], tb);
      bulk(sm + s * TILE, frames + (f0 + s) * FB + toff, tb, &full[s]);
    }
  uint32_t acc = 0;
  for (int i = 0; i < group; i++) {
    const int s = i % STAGES;
    mbar_wait(&full[s], (i / STAGES) & 1);
    acc += reinterpret_cast<const uint32_t*>(sm + s * TILE)[(tid * 4) % (TILE / 4)];
    __syncwarp();
    if (lane == 0 && atomicAdd(&cnt[s], 1u) == 7) {
      cnt[s] = 0;
      if (i + STAGES < group) {
        mbar_expect(&full[s], tb);
        bulk(sm + s * TILE, frames + (f0 + i + STAGES) * FB + toff, tb, &full[s]);
      }
    }
  }
  if (acc == 0x12345678u) sink[0] = acc;
}

// B: plain coalesced LDG.128 streaming, UNROLL loads in flight per thread
template <int UNROLL>
__global__ void __launch_bounds__(256) ldg_stream(const uint4* p, uint64_t n16, uint32_t* sink) {
  uint32_t acc = 0;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n16; i += stride * UNROLL) {
    uint4 v[UNROLL];
#pragma unroll
    for (int u = 0; u < UNROLL; u++) v[u] = (i + u * stride < n16) ? __ldcs(p + i + u * stride) : make_uint4(0, 0, 0, 0);
#pragma unroll
    for (int u = 0; u < UNROLL; u++) acc ^= v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
  }
  if (acc == 0x12345678u) sink[0] = acc;
}

template <typename F>
float timeit(F f, int reps = 10) {
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  f();
  cudaDeviceSynchronize();
  cudaEventRecord(a);
  for (int r = 0; r < reps; r++) f();
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return ms / reps;
}

template <int STAGES, int TILE>
void run_ring(const uint8_t* d, uint32_t* sink, int group, int minblocks_hint) {
  const int smem = STAGES * TILE;
  cudaFuncSetAttribute(tma_ring<STAGES, TILE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const unsigned tiles = (unsigned)((FB + TILE - 1) / TILE);
  dim3 grid(tiles, NF / group);
  float ms = timeit([&] { tma_ring<STAGES, TILE><<<grid, 256, smem>>>(d, group, sink); });
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, tma_ring<STAGES, TILE>, 256, smem);
  printf("tma_ring stages=%2d tile=%6d group=%2d grid=%6u occ=%d : %8.1f us  %7.0f GB/s\n", STAGES,
         TILE, group, tiles * (NF / group), occ, ms * 1e3, NF * FB / (ms * 1e-3) / 1e9);
  (void)minblocks_hint;
}

int main() {
  uint8_t* d;
  uint32_t* sink;
  cudaMalloc(&d, NF * FB + 4096);
  cudaMalloc(&sink, 64);
  cudaMemset(d, 1, NF * FB);
  // flush-sized buffer is not needed: 398 MB >> 126 MB L2
  const uint64_t n16 = NF * FB / 16;
  for (int blocks : {148 * 4, 148 * 8, 148 * 16}) {
    float ms = timeit([&] { ldg_stream<4><<<blocks, 256>>>((const uint4*)d, n16, sink); });
    printf("ldg_stream unroll=4 blocks=%5d : %8.1f us  %7.0f GB/s\n", blocks, ms * 1e3, NF * FB / (ms * 1e-3) / 1e9);
  }
  run_ring<8, 12288>(d, sink, 32, 2);
  run_ring<8, 12288>(d, sink, 16, 2);
  run_ring<4, 12288>(d, sink, 32, 4);
  run_ring<16, 6144>(d, sink, 32, 2);
  run_ring<4, 24576>(d, sink, 32, 2);
  run_ring<8, 6144>(d, sink, 32, 4);
  run_ring<2, 12288>(d, sink, 32, 8);
  cudaError_t e = cudaDeviceSynchronize();
  printf("status %s\n", cudaGetErrorString(e));
  return 0;
}
