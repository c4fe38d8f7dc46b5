// hadacodec-b200: multi-bounce accumulation (config 4).
//
// Per sample s of pixel p (following the renderer's NEE
// and throughput updates renderer.cpp:505-510, :530-533 and
// multibounce_eval's z (.)= E(R_b) chain evaluation.cpp:50-76):
//   thr = 1, rad = 0
//   for d < DEPTH:  rad += thr * albedo_d * le * t_d ;  thr *= albedo_d
//   acc += double(rad)                                (renderer.cpp:548-551)
// pixel = float(acc / spp)                             (renderer.cpp:588-592)
//
// Mapping: 8 lanes per pixel (4 pixels per warp), lane g owns samples
// g, g+8, ...: every sample stream (u8x4 palette indices, u8 illuminant index,
// float4 throughput factors) is read as 8 consecutive records per pixel, i.e.
// coalesced 32/8/128-byte segments.  Palette / illuminant tables sit in shared
// memory.  Per-lane fp64 sums are reduced over the 8 lanes with shuffles.
#pragma once

#include "hc_common.cuh"
#include "hc_ops.cuh"

namespace hcb {

constexpr int kChainLanes = 8;
constexpr int kMaxIllum = 256;

template <int K>
struct ChainLatentParams {
  float Mxyz[3 * K];
  float Crgb[9];
  const float* pal;  // n_pal x K
  const float* ill;  // n_ill x K
  int n_pal, n_ill;
  const uint32_t* pidx;  // [P][spp] packed u8 x 4 (depth 4)
  const uint8_t* iidx;   // [P][spp]
  const float4* tw;      // [P][spp] float x 4
  int64_t P;
  int spp;
  float* latent;  // P x K   (nullable)
  float* xyz;     // P x 3   (nullable)
  float* rgb;     // P x 3   (nullable)
  int* err;
};

template <int K>
__global__ void __launch_bounds__(256) chain_latent_kernel(const __grid_constant__ ChainLatentParams<K> p) {
  extern __shared__ __align__(16) float tab[];
  float* pal = tab;
  float* ill = tab + p.n_pal * K;
  block_load_table(pal, p.pal, p.n_pal * K);
  block_load_table(ill, p.ill, p.n_ill * K);
  __syncthreads();

  const int lane = threadIdx.x & 31;
  const int g = lane & (kChainLanes - 1);
  // Warp-uniform loop over pixel quads so the group shuffles never see exited lanes.
  constexpr int kPixPerWarp = 32 / kChainLanes;
  const int64_t warp_id = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  const uint32_t npal = static_cast<uint32_t>(p.n_pal), nill = static_cast<uint32_t>(p.n_ill);
  for (int64_t q = warp_id; q * kPixPerWarp < p.P; q += nwarps) {
    const int64_t pix = q * kPixPerWarp + lane / kChainLanes;
    const bool valid = pix < p.P;
    double acc[K];
#pragma unroll
    for (int j = 0; j < K; ++j) acc[j] = 0.0;
    const int64_t base = pix * p.spp;
    bool bad = false;
    for (int s = g; valid && s < p.spp; s += kChainLanes) {
      const uint32_t pk = __ldg(p.pidx + base + s);
      uint32_t li = __ldg(p.iidx + base + s);
      const float4 t4 = ldg_stream(p.tw + base + s);
      const float tw[4] = {t4.x, t4.y, t4.z, t4.w};
      if (li >= nill) { bad = true; li = 0; }
      const float* le = ill + li * K;
      float thr[K], rad[K];
#pragma unroll
      for (int j = 0; j < K; ++j) {
        thr[j] = 1.f;
        rad[j] = 0.f;
      }
#pragma unroll
      for (int d = 0; d < 4; ++d) {
        uint32_t ai = (pk >> (8 * d)) & 0xffu;
        if (ai >= npal) { bad = true; ai = 0; }
        const float* albedo = pal + ai * K;
#pragma unroll
        for (int j = 0; j < K; ++j) {
          const float a = albedo[j];
          rad[j] = fmaf(thr[j] * a * le[j], tw[d], rad[j]);
          thr[j] *= a;
        }
      }
#pragma unroll
      for (int j = 0; j < K; ++j) acc[j] += static_cast<double>(rad[j]);
    }
    if (bad) atomicOr(p.err, kErrIndexRange);
#pragma unroll
    for (int o = kChainLanes / 2; o > 0; o >>= 1)
#pragma unroll
      for (int j = 0; j < K; ++j) acc[j] += __shfl_xor_sync(0xffffffffu, acc[j], o);
    if (valid && g == 0) {
      const double inv = 1.0 / p.spp;
      float z[K];
#pragma unroll
      for (int j = 0; j < K; ++j) z[j] = static_cast<float>(acc[j] * inv);
      if (p.latent)
#pragma unroll
        for (int j = 0; j < K; ++j) p.latent[pix * K + j] = z[j];
      float xyz[3], rgb[3];
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        float a = p.Mxyz[c * K] * z[0];
#pragma unroll
        for (int j = 1; j < K; ++j) a = fmaf(p.Mxyz[c * K + j], z[j], a);
        xyz[c] = a;
      }
      xyz_to_rgb(p.Crgb, xyz, rgb);
      if (p.xyz)
#pragma unroll
        for (int c = 0; c < 3; ++c) p.xyz[pix * 3 + c] = xyz[c];
      if (p.rgb)
#pragma unroll
        for (int c = 0; c < 3; ++c) p.rgb[pix * 3 + c] = rgb[c];
    }
  }
}

// Replicated-table variant for small even-padded k (k = 3, 6): the code tables are
// stored as float2 rows replicated 16x across bank pairs, lane l of each
// half-warp reading replica l % 16, so every LDS.64 of the 5 random lookups per
// sample is bank-conflict free whatever the indices.  Per sample the chain is
// re-associated (SURVEY Appendix A #7 allows it):
//   thr_d = thr_{d-1} (.) a_d ;  s = sum_d t_d thr_d ;  rad = le (.) s
// and each lane sums its samples in fp32 before the fp64 cross-lane reduction.
//
// SHFL_ILL (n_ill <= 16, config 4): the illuminant codes live in registers instead — lane
// l holds illuminant l % 16 — and each sample's illuminant code is fetched with 2*KP
// shuffles, so only the 4 palette lookups per sample touch shared memory.  The L1 data
// pipe (shared-memory wavefronts plus the sample records' global loads) is this kernel's
// bottleneck (r01 ncu: 83 % busy); the shuffles do not use it.
template <int K, bool SHFL_ILL>
__global__ void __launch_bounds__(256) chain_latent_rep_kernel(const __grid_constant__ ChainLatentParams<K> p) {
  constexpr int KP = (K + 1) / 2;  // float2 per code
  extern __shared__ __align__(16) float2 rep[];
  const int n_ent = SHFL_ILL ? p.n_pal : p.n_pal + p.n_ill;
  constexpr int R = 8;  // loads in flight per thread before its stores (block_load_table)
  for (int base = threadIdx.x; base < n_ent * KP * 16; base += R * blockDim.x) {
    float2 v[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int i = base + r * blockDim.x;
      if (i < n_ent * KP * 16) {
        const int q = i >> 4;
        const int e = q / KP, c2 = q - e * KP;
        const float* src = e < p.n_pal ? p.pal + e * K : p.ill + (e - p.n_pal) * K;
        v[r] = make_float2(__ldg(src + 2 * c2), 2 * c2 + 1 < K ? __ldg(src + 2 * c2 + 1) : 0.f);
      }
    }
#pragma unroll
    for (int r = 0; r < R; ++r)
      if (base + r * blockDim.x < n_ent * KP * 16) rep[base + r * blockDim.x] = v[r];
  }
  __syncthreads();

  const int lane = threadIdx.x & 31;
  const int g = lane & (kChainLanes - 1);
  const float2* mine = rep + (lane & 15);
  float ill_reg[2 * KP];  // SHFL_ILL: illuminant lane % 16 (zero past n_ill)
#pragma unroll
  for (int j = 0; j < 2 * KP; ++j)
    ill_reg[j] = SHFL_ILL && (lane & 15) < p.n_ill && j < K ? __ldg(p.ill + (lane & 15) * K + j) : 0.f;
  constexpr int kPixPerWarp = 32 / kChainLanes;
  const int64_t warp_id = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  const uint32_t npal = static_cast<uint32_t>(p.n_pal), nill = static_cast<uint32_t>(p.n_ill);
  for (int64_t qd = warp_id; qd * kPixPerWarp < p.P; qd += nwarps) {
    const int64_t pix = qd * kPixPerWarp + lane / kChainLanes;
    const bool valid = pix < p.P;
    float part[2 * KP];
#pragma unroll
    for (int j = 0; j < 2 * KP; ++j) part[j] = 0.f;
    const int64_t base = pix * p.spp;
    bool bad = false;
    // SHFL_ILL: every lane runs the sample loop (warp-wide shuffles); a past-the-end pixel's
    // lanes load nothing and are never stored.
    const int per_lane = valid || SHFL_ILL ? p.spp / kChainLanes : 0;
    {
      // Warm L2 with the next quad's sample records (no registers held): the 8 lanes
      // of a pixel group each touch one 128-byte line of the next pixel's streams.
      const int64_t npix = (qd + nwarps) * kPixPerWarp + lane / kChainLanes;
      if (npix < p.P) {
        const int64_t nb = npix * p.spp;
        const char* twl = reinterpret_cast<const char*>(p.tw + nb);
        for (int off = g * 128; off < p.spp * 16; off += kChainLanes * 128)
          asm volatile("prefetch.global.L2 [%0];" ::"l"(twl + off));
        const char* pkl = reinterpret_cast<const char*>(p.pidx + nb);
        for (int off = g * 128; off < p.spp * 4; off += kChainLanes * 128)
          asm volatile("prefetch.global.L2 [%0];" ::"l"(pkl + off));
        if (g == 0) asm volatile("prefetch.global.L2 [%0];" ::"l"(p.iidx + nb));
      }
    }
    // Samples in groups of kGroup per lane with every load of the group issued
    // before any use: ~170 B in flight per lane keeps HBM busy (the kernel was
    // long-scoreboard bound issuing one sample's loads at a time).
    constexpr int kGroup = 8;
    for (int m0 = 0; m0 < per_lane; m0 += kGroup) {
      uint32_t pkg[kGroup], lig[kGroup];
      float4 t4g[kGroup];
#pragma unroll
      for (int m = 0; m < kGroup; ++m) {
        const int64_t s = base + g + static_cast<int64_t>(m0 + m) * kChainLanes;
        const bool in = m0 + m < per_lane && valid;
        pkg[m] = in ? __ldg(p.pidx + s) : 0u;
        lig[m] = in ? static_cast<uint32_t>(__ldg(p.iidx + s)) : 0u;
        t4g[m] = in ? ldg_stream(p.tw + s) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
    for (int m = 0; m < kGroup; ++m) {
      if (m0 + m >= per_lane) break;
      const uint32_t pk = pkg[m];
      uint32_t li = lig[m];
      const float4 t4 = t4g[m];
      const float tw[4] = {t4.x, t4.y, t4.z, t4.w};
      if (li >= nill) { bad = true; li = 0; }
      float thr[2 * KP], acc[2 * KP];
#pragma unroll
      for (int d = 0; d < 4; ++d) {
        uint32_t ai = (pk >> (8 * d)) & 0xffu;
        if (ai >= npal) { bad = true; ai = 0; }
        const float2* row = mine + ai * (KP * 16);
#pragma unroll
        for (int c2 = 0; c2 < KP; ++c2) {
          const float2 a = row[c2 * 16];
          if (d == 0) {
            thr[2 * c2] = a.x;
            thr[2 * c2 + 1] = a.y;
            acc[2 * c2] = tw[0] * a.x;
            acc[2 * c2 + 1] = tw[0] * a.y;
          } else {
            thr[2 * c2] *= a.x;
            thr[2 * c2 + 1] *= a.y;
            acc[2 * c2] = fmaf(tw[d], thr[2 * c2], acc[2 * c2]);
            acc[2 * c2 + 1] = fmaf(tw[d], thr[2 * c2 + 1], acc[2 * c2 + 1]);
          }
        }
      }
      if constexpr (SHFL_ILL) {
#pragma unroll
        for (int j = 0; j < 2 * KP; ++j)
          part[j] = fmaf(__shfl_sync(0xffffffffu, ill_reg[j], static_cast<int>(li)), acc[j], part[j]);
      } else {
        const float2* lrow = mine + (npal + li) * (KP * 16);
#pragma unroll
        for (int c2 = 0; c2 < KP; ++c2) {
          const float2 le = lrow[c2 * 16];
          part[2 * c2] = fmaf(le.x, acc[2 * c2], part[2 * c2]);
          part[2 * c2 + 1] = fmaf(le.y, acc[2 * c2 + 1], part[2 * c2 + 1]);
        }
      }
    }
    }
    if (bad) atomicOr(p.err, kErrIndexRange);
    double acc[K];
#pragma unroll
    for (int j = 0; j < K; ++j) acc[j] = static_cast<double>(part[j]);
#pragma unroll
    for (int o = kChainLanes / 2; o > 0; o >>= 1)
#pragma unroll
      for (int j = 0; j < K; ++j) acc[j] += __shfl_xor_sync(0xffffffffu, acc[j], o);
    if (valid && g == 0) {
      const double inv = 1.0 / p.spp;
      float z[K];
#pragma unroll
      for (int j = 0; j < K; ++j) z[j] = static_cast<float>(acc[j] * inv);
      if (p.latent)
#pragma unroll
        for (int j = 0; j < K; ++j) p.latent[pix * K + j] = z[j];
      float xyz[3], rgb[3];
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        float a = p.Mxyz[c * K] * z[0];
#pragma unroll
        for (int j = 1; j < K; ++j) a = fmaf(p.Mxyz[c * K + j], z[j], a);
        xyz[c] = a;
      }
      xyz_to_rgb(p.Crgb, xyz, rgb);
      if (p.xyz)
#pragma unroll
        for (int c = 0; c < 3; ++c) p.xyz[pix * 3 + c] = xyz[c];
      if (p.rgb)
#pragma unroll
        for (int c = 0; c < 3; ++c) p.rgb[pix * 3 + c] = rgb[c];
    }
  }
}

// Naive n-sample chain: the same recursion per wavelength.  Loop order is
// wavelength-outer so per-lane state stays in registers; the pixel spectrum
// value float(acc/spp) is projected to XYZ on the fly (colorimetry.cpp:75-87).
template <int N>
struct ChainSpectralParams {
  float cmf[3 * N];
  float Crgb[9];
  const float* pal;  // n_pal x N
  const float* ill;  // n_ill x N
  int n_pal, n_ill;
  const uint32_t* pidx;
  const uint8_t* iidx;
  const float4* tw;
  int64_t P;
  int spp;
  float* xyz;
  float* rgb;
  int* err;
};

template <int N, int SPL>  // SPL = samples per lane (spp / 8)
__global__ void __launch_bounds__(256) chain_spectral_kernel(const __grid_constant__ ChainSpectralParams<N> p) {
  extern __shared__ __align__(16) float tab[];
  float* pal = tab;
  float* ill = tab + p.n_pal * N;
  block_load_table(pal, p.pal, p.n_pal * N);
  block_load_table(ill, p.ill, p.n_ill * N);
  __syncthreads();

  const int lane = threadIdx.x & 31;
  const int g = lane & (kChainLanes - 1);
  // Warp-uniform loop over pixel quads so the group shuffles never see exited lanes.
  constexpr int kPixPerWarp = 32 / kChainLanes;
  const int64_t warp_id = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  const uint32_t npal = static_cast<uint32_t>(p.n_pal), nill = static_cast<uint32_t>(p.n_ill);
  for (int64_t q = warp_id; q * kPixPerWarp < p.P; q += nwarps) {
    const int64_t pix = q * kPixPerWarp + lane / kChainLanes;
    const bool valid = pix < p.P;
    const int64_t base = (valid ? pix : 0) * p.spp;
    uint32_t pk[SPL], li[SPL];
    float4 t4[SPL];
    bool bad = false;
#pragma unroll
    for (int m = 0; m < SPL; ++m) {
      const int s = g + m * kChainLanes;
      pk[m] = valid ? __ldg(p.pidx + base + s) : 0u;
      li[m] = valid ? __ldg(p.iidx + base + s) : 0u;
      t4[m] = valid ? ldg_stream(p.tw + base + s) : make_float4(0.f, 0.f, 0.f, 0.f);
      if (li[m] >= nill) { bad = true; li[m] = 0; }
#pragma unroll
      for (int d = 0; d < 4; ++d)
        if (((pk[m] >> (8 * d)) & 0xffu) >= npal) { bad = true; pk[m] &= ~(0xffu << (8 * d)); }
    }
    if (bad) atomicOr(p.err, kErrIndexRange);
    const double inv = 1.0 / p.spp;
    float xyz[3] = {0.f, 0.f, 0.f};
#pragma unroll 1
    for (int i = 0; i < N; ++i) {
      double acc = 0.0;
#pragma unroll
      for (int m = 0; m < SPL; ++m) {
        const float le = ill[li[m] * N + i];
        const float tw[4] = {t4[m].x, t4[m].y, t4[m].z, t4[m].w};
        float thr = 1.f, rad = 0.f;
#pragma unroll
        for (int d = 0; d < 4; ++d) {
          const float a = pal[((pk[m] >> (8 * d)) & 0xffu) * N + i];
          rad = fmaf(thr * a * le, tw[d], rad);
          thr *= a;
        }
        acc += static_cast<double>(rad);
      }
#pragma unroll
      for (int o = kChainLanes / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
      const float s = static_cast<float>(acc * inv);
      xyz[0] = fmaf(p.cmf[i], s, xyz[0]);
      xyz[1] = fmaf(p.cmf[N + i], s, xyz[1]);
      xyz[2] = fmaf(p.cmf[2 * N + i], s, xyz[2]);
    }
    if (valid && g == 0) {
      float rgb[3];
      xyz_to_rgb(p.Crgb, xyz, rgb);
      if (p.xyz)
#pragma unroll
        for (int c = 0; c < 3; ++c) p.xyz[pix * 3 + c] = xyz[c];
      if (p.rgb)
#pragma unroll
        for (int c = 0; c < 3; ++c) p.rgb[pix * 3 + c] = rgb[c];
    }
  }
}

}  // namespace hcb
