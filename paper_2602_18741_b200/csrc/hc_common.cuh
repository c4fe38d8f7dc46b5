// hadacodec-b200: shared device helpers and the kernel-parameter layouts.
//
// Small codec tables (E k×n, D n×k, the folded 3×k XYZ projection, the 3×3
// IEC sRGB matrix, CMF rows, light codes / spectra) are passed BY VALUE as
// kernel parameters.  Parameters live in the constant bank, so every
// warp-uniform coefficient becomes a `c[0x0][...]` FFMA operand: no load
// instruction, no register, broadcast to all lanes (sm_100a, CUDA >= 12.1
// allows up to 32 KB of kernel parameters).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace hcb {

constexpr int kWarp = 32;

// Codec coefficients for a fixed (n, k).
template <int N, int K>
struct CodecConst {
  float E[K * N];     // encoder, row-major k x n           (codec.hpp:52-58)
  float D[N * K];     // decoder, row-major n x k
  float Mxyz[3 * K];  // dlambda * CMF * D, 3 x k (folding precedent renderer.cpp:249-263)
  float Crgb[9];      // IEC 61966-2-1 XYZ -> linear sRGB (colorimetry.cpp:22-26)
  float cmf[3 * N];   // dlambda * CMF rows (colorimetry.cpp:75-87)
};

__device__ __forceinline__ void xyz_to_rgb(const float* __restrict__ C, const float xyz[3],
                                           float rgb[3]) {
#pragma unroll
  for (int r = 0; r < 3; ++r)
    rgb[r] = fmaf(C[3 * r + 2], xyz[2], fmaf(C[3 * r + 1], xyz[1], C[3 * r + 0] * xyz[0]));
}

// Streaming (evict-first) 128-bit global load / store: data touched once.
__device__ __forceinline__ float4 ldg_stream(const float4* p) {
  float4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
               : "l"(p));
  return r;
}
__device__ __forceinline__ uint32_t ldg_stream_u32(const uint32_t* p) {
  uint32_t r;
  asm volatile("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(r) : "l"(p));
  return r;
}
__device__ __forceinline__ void stg_stream(float4* p, float4 v) {
  asm volatile("st.global.L1::no_allocate.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(v.x), "f"(v.y),
               "f"(v.z), "f"(v.w)
               : "memory");
}

// Copy `count` floats global -> shared with 16-byte vectors (both 16-byte aligned,
// count a multiple of 4), all threads of the block participating.
__device__ __forceinline__ void block_copy_g2s(float* __restrict__ dst, const float* __restrict__ src,
                                               int count) {
  const float4* s4 = reinterpret_cast<const float4*>(src);
  float4* d4 = reinterpret_cast<float4*>(dst);
  for (int i = threadIdx.x; i < (count >> 2); i += blockDim.x) d4[i] = ldg_stream(s4 + i);
}
__device__ __forceinline__ void block_copy_s2g(float* __restrict__ dst, const float* __restrict__ src,
                                               int count) {
  const float4* s4 = reinterpret_cast<const float4*>(src);
  float4* d4 = reinterpret_cast<float4*>(dst);
  for (int i = threadIdx.x; i < (count >> 2); i += blockDim.x) stg_stream(d4 + i, s4[i]);
}
// Scalar variants for unaligned / ragged tails.
__device__ __forceinline__ void block_copy_g2s_scalar(float* __restrict__ dst,
                                                      const float* __restrict__ src, int count) {
  for (int i = threadIdx.x; i < count; i += blockDim.x) dst[i] = src[i];
}
__device__ __forceinline__ void block_copy_s2g_scalar(float* __restrict__ dst,
                                                      const float* __restrict__ src, int count) {
  for (int i = threadIdx.x; i < count; i += blockDim.x) dst[i] = src[i];
}

__device__ __forceinline__ bool aligned16(const void* p) {
  return (reinterpret_cast<uintptr_t>(p) & 15u) == 0;
}

// Table (palette / illuminant codes or spectra) global -> shared at kernel start, all
// threads of the block.  Every CTA of a launch reads the same few KB right after the PDL
// wait, so the latency is on the critical path of short launches: each thread issues R
// 16-byte loads before its R stores (one L2 round trip per 4R elements instead of one
// per element; the element-at-a-time loop cost ~1.1 us of a 23.5 us 1080p shading
// frame).  R stays small: the loop is inlined into kernels whose register budget it
// must not raise (R = 8 took a 96-register kernel to 212).
template <int R = 2>
__device__ __forceinline__ void block_load_table(float* __restrict__ dst, const float* __restrict__ src, int count) {
  const int nt = blockDim.x;
  if (aligned16(src) && aligned16(dst) && (count & 3) == 0) {
    const float4* s4 = reinterpret_cast<const float4*>(src);
    float4* d4 = reinterpret_cast<float4*>(dst);
    const int n4 = count >> 2;
    for (int base = threadIdx.x; base < n4; base += R * nt) {
      float4 v[R];
#pragma unroll
      for (int r = 0; r < R; ++r)
        if (base + r * nt < n4) v[r] = __ldg(s4 + base + r * nt);
#pragma unroll
      for (int r = 0; r < R; ++r)
        if (base + r * nt < n4) d4[base + r * nt] = v[r];
    }
  } else {  // unaligned tables (not the library's own buffers): plain loop
    for (int i = threadIdx.x; i < count; i += nt) dst[i] = __ldg(src + i);
  }
}

}  // namespace hcb
