// k_lut_learn.cu -- K0 (gamma-LUT table, a2) and K1 (background envelope, a1).
#include "fizi_internal.cuh"

namespace fizi {

// ---------------------------------------------------------------- K0 table
// a2 / §3.2, readings L19-L21: for every integer mean luma m the frame
// gets gamma(m) and the per-channel table L_m[x] = floor(255 (x/255)^g + 0.5),
// identity when luma_lo <= m <= luma_hi.  Built once per context (params are
// immutable), so the per-frame work is a table row selection.
__global__ void lut_table_kernel(fizi_params p, uint8_t* __restrict__ lut,
                                 double* __restrict__ gtab, uint8_t* __restrict__ ctab) {
  const uint32_t m = blockIdx.x, x = threadIdx.x;
  const bool ident = m >= p.luma_lo && m <= p.luma_hi;
  double g = 1.0;
  if (!ident) {
    if (m == 0) g = p.gamma_min;
    else if (m == 255) g = p.gamma_max;
    else {
      g = log((double)p.luma_target / 255.0) / log((double)m / 255.0);
      g = g < p.gamma_min ? p.gamma_min : g;
      g = g > p.gamma_max ? p.gamma_max : g;
    }
  }
  uint32_t v = x;
  if (!ident) {
    double t = floor(__dadd_rn(__dmul_rn(255.0, pow((double)x / 255.0, g)), 0.5));
    v = t < 0.0 ? 0u : (t > 255.0 ? 255u : (uint32_t)t);
  }
  lut[m * 256 + x] = (uint8_t)v;
  if (x == 0) {
    gtab[m] = g;
    ctab[m] = ident ? 0 : 1;
  }
}

cudaError_t launch_lut_table(Ctx& c, cudaStream_t st) {
  lut_table_kernel<<<256, 256, 0, st>>>(c.p, c.lut, c.gamma_tab, c.corr_tab);
  c.launches += 1;
  return cudaGetLastError();
}

// ------------------------------------------------------------------- K1 learn
// a1: lo = sat(min_k F_k - margin), hi = sat(max_k F_k + margin)
// per pixel and channel.  One thread per 16 linear frame bytes (fast path:
// 3N % 16 == 0) or per byte (generic).
__global__ void learn16_kernel(const uint8_t* __restrict__ frames, uint32_t n, uint64_t nbytes,
                               uint32_t margin, uint8_t* __restrict__ lo,
                               uint8_t* __restrict__ hi) {
  uint64_t seg = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (seg * 16 >= nbytes) return;
  uint4 mn = make_uint4(0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu);
  uint4 mx = make_uint4(0, 0, 0, 0);
  for (uint32_t k = 0; k < n; k++) {
    uint4 v = __ldg(reinterpret_cast<const uint4*>(frames + k * nbytes) + seg);
    mn.x = __vminu4(mn.x, v.x); mn.y = __vminu4(mn.y, v.y);
    mn.z = __vminu4(mn.z, v.z); mn.w = __vminu4(mn.w, v.w);
    mx.x = __vmaxu4(mx.x, v.x); mx.y = __vmaxu4(mx.y, v.y);
    mx.z = __vmaxu4(mx.z, v.z); mx.w = __vmaxu4(mx.w, v.w);
  }
  const uint32_t m4 = margin * 0x01010101u;
  mn.x = __vsubus4(mn.x, m4); mn.y = __vsubus4(mn.y, m4);
  mn.z = __vsubus4(mn.z, m4); mn.w = __vsubus4(mn.w, m4);
  mx.x = __vaddus4(mx.x, m4); mx.y = __vaddus4(mx.y, m4);
  mx.z = __vaddus4(mx.z, m4); mx.w = __vaddus4(mx.w, m4);
  uint64_t dst = env_perm_index(seg * 16, true);   // 16-byte piece stays contiguous
  *reinterpret_cast<uint4*>(lo + dst) = mn;
  *reinterpret_cast<uint4*>(hi + dst) = mx;
}

__global__ void learn1_kernel(const uint8_t* __restrict__ frames, uint32_t n, uint64_t nbytes,
                              uint32_t margin, uint8_t* __restrict__ lo, uint8_t* __restrict__ hi) {
  uint64_t b = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (b >= nbytes) return;
  int mn = 255, mx = 0;
  for (uint32_t k = 0; k < n; k++) {
    int v = frames[k * nbytes + b];
    mn = min(mn, v);
    mx = max(mx, v);
  }
  lo[b] = (uint8_t)max(mn - (int)margin, 0);
  hi[b] = (uint8_t)min(mx + (int)margin, 255);
}

cudaError_t launch_learn(Ctx& c, uint32_t stream, const uint8_t* frames, uint32_t n,
                         uint32_t margin, cudaStream_t st) {
  uint8_t* lo = c.env + (uint64_t)stream * 2 * c.env_plane;
  uint8_t* hi = lo + c.env_plane;
  uint64_t nbytes = c.N * 3;
  if (c.fast) {
    uint64_t segs = nbytes / 16;
    learn16_kernel<<<(unsigned)((segs + 255) / 256), 256, 0, st>>>(frames, n, nbytes, margin, lo, hi);
  } else {
    learn1_kernel<<<(unsigned)((nbytes + 255) / 256), 256, 0, st>>>(frames, n, nbytes, margin, lo, hi);
  }
  c.launches += 1;
  return cudaGetLastError();
}

// ---------------------------------------------- envelope export / import
__global__ void env_copy_kernel(uint8_t* __restrict__ plane_lo, uint8_t* __restrict__ plane_hi,
                                uint8_t* __restrict__ lin_lo, uint8_t* __restrict__ lin_hi,
                                const uint8_t* __restrict__ in_lo, const uint8_t* __restrict__ in_hi,
                                uint64_t nbytes, bool fast, bool import) {
  uint64_t b = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (b >= nbytes) return;
  uint64_t q = env_perm_index(b, fast);
  if (import) {
    plane_lo[q] = in_lo[b];
    plane_hi[q] = in_hi[b];
  } else {
    lin_lo[b] = plane_lo[q];
    lin_hi[b] = plane_hi[q];
  }
}

cudaError_t launch_env_export(Ctx& c, uint32_t stream, uint8_t* lo, uint8_t* hi, bool import,
                              const uint8_t* ilo, const uint8_t* ihi, cudaStream_t st) {
  uint8_t* plo = c.env + (uint64_t)stream * 2 * c.env_plane;
  uint8_t* phi = plo + c.env_plane;
  uint64_t nbytes = c.N * 3;
  env_copy_kernel<<<(unsigned)((nbytes + 255) / 256), 256, 0, st>>>(plo, phi, lo, hi, ilo, ihi,
                                                                   nbytes, c.fast, import);
  c.launches += 1;
  return cudaGetLastError();
}

}  // namespace fizi
