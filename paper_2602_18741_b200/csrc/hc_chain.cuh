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

// k = 6 chain, instruction-lean (config 4).  chain_latent_rep_kernel is bounded by the L1
// data pipe (the random code lookups: 5 x 24 B per sample) *and* by issue (~100
// instructions per sample: per-lookup bounds checks, IMAD row addressing, 48 scalar FP ops).
// This kernel keeps the lookup bytes (the codes are fp32) and cuts the instructions:
//  * rows are 256 B: [c0..c3] as a float4 replicated 8x (LDS.128, each quarter-warp phase
//    reads 8 distinct 16-byte slots = all 32 banks) then [c4 c5] as a float2 replicated 16x
//    (LDS.64, conflict-free per half-warp), so a row address is (index << 8) | lane offset,
//    built by ONE byte permute (PRMT) straight from the packed u8x4 palette word;
//  * the palette table always has 256 rows (zero past n_pal), so a u8 index can never read
//    out of bounds: out-of-range indices are detected once per pixel from a running byte-wise
//    max (__vmaxu4) instead of per lookup; illuminant indices are clamped (min) and tracked;
//  * the chain is evaluated in Horner form on packed pairs (fma.rn.f32x2 / mul.rn.f32x2):
//      S = a0 (.) (t0 + a1 (.) (t1 + a2 (.) (t2 + t3 a3))),  part += le (.) S
//    = sum_d t_d prod_{e<=d} a_e (.) le, the reference's rad (renderer.cpp:505-510, :530-533)
//    re-associated: 5 packed ops per code pair, 15 per sample.
// Shared memory: 64 KB palette + 256 B per illuminant + 6.2 KB of staging (config 4: 74 KB,
// 3 CTAs / SM).
#ifndef HC_CHAIN_IIDX128
#define HC_CHAIN_IIDX128 0
#endif
// Bulk-copied records (kTma), option: a pixel's 64 illuminant bytes read as 4 LDS.128 that the pixel's 8
// lanes share (one wavefront each for the warp's 4 pixels) instead of 8 byte loads per lane.
// Measured neutral to slightly slower (72.0 vs 72.2-72.8 % with the shuffle sums), so off.
#ifndef HC_CHAIN_TMA_IIDX128
#define HC_CHAIN_TMA_IIDX128 0
#endif
// Pixel sums: 1 = fp32 reduce-scatter over the 8 lanes by shuffles (11 SHFL per quad),
// 0 = fp32 partials staged through shared memory and added in fp64 (20 wavefronts per quad).
#ifndef HC_CHAIN_SUM_SHFL
#define HC_CHAIN_SUM_SHFL 1
#endif
constexpr int kChainV3Row = 256;
constexpr int kChainV3Stage = 6 * 33;  // floats of per-warp staging for the pixel sums
__host__ __device__ constexpr int chain_v3_stage_bytes(int warps) { return (warps * kChainV3Stage * 4 + 15) / 16 * 16; }

__device__ __forceinline__ uint64_t chain_fma2(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ uint64_t chain_mul2(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ uint64_t chain_dup(float x) {
  uint64_t d;
  asm("mov.b64 %0, {%1, %1};" : "=l"(d) : "f"(x));
  return d;
}

// One sample of the v3 chain: the 5 lookups and the packed Horner chain into part[3].
template <bool kCheckPal>
__device__ __forceinline__ void chain_v3_sample(const unsigned char* tab3, const unsigned char* ill_tab, uint32_t offs,
                                                uint32_t pk, uint32_t li_raw, float4 t4, uint32_t ill_last,
                                                uint32_t& pmax, uint32_t& imax, uint64_t part[3]) {
  if (kCheckPal) pmax = __vmaxu4(pmax, pk);
  imax = max(imax, li_raw);
  const uint32_t li = min(li_raw, ill_last);
  uint64_t a[4][3];
#pragma unroll
  for (int d = 0; d < 4; ++d) {
    const uint32_t o4 = __byte_perm(pk, offs, 0x6604u | (d << 4));  // (idx << 8) | off4
    const uint32_t o2 = __byte_perm(pk, offs, 0x6605u | (d << 4));  // (idx << 8) | off2
    const ulonglong2 v = *reinterpret_cast<const ulonglong2*>(tab3 + o4);
    a[d][0] = v.x;
    a[d][1] = v.y;
    a[d][2] = *reinterpret_cast<const unsigned long long*>(tab3 + o2);
  }
  const uint32_t lo4 = __byte_perm(li, offs, 0x6604u), lo2 = __byte_perm(li, offs, 0x6605u);
  const ulonglong2 lv = *reinterpret_cast<const ulonglong2*>(ill_tab + lo4);
  const uint64_t le[3] = {lv.x, lv.y, *reinterpret_cast<const unsigned long long*>(ill_tab + lo2)};
  const uint64_t T0 = chain_dup(t4.x), T1 = chain_dup(t4.y), T2 = chain_dup(t4.z), T3 = chain_dup(t4.w);
#pragma unroll
  for (int j = 0; j < 3; ++j) {
    uint64_t u = chain_fma2(a[3][j], T3, T2);
    u = chain_fma2(a[2][j], u, T1);
    u = chain_fma2(a[1][j], u, T0);
    part[j] = chain_fma2(le[j], chain_mul2(a[0][j], u), part[j]);
  }
}

// kTma (spp == 64, 16-byte aligned pidx / iidx): a pixel quad's palette-index words and
// illuminant bytes arrive by bulk copies (cp.async.bulk, one mbarrier per warp, double-buffered)
// into per-pixel slots padded so the lanes' reads are conflict-free (pixel strides 288 B and
// 80 B): 16 L1 wavefronts per quad for the two streams instead of ~48 through LDG (4 pixels =
// 4 lines per 32-bit load, 2 per byte load), and the L2 prefetches of those streams go away.
constexpr int kChainTmaPidx = 4 * 288;              // pidx slot: 4 pixels x (256 + 32 pad) B
constexpr int kChainTmaSlot = kChainTmaPidx + 4 * 80;  // + iidx: 4 pixels x (64 + 16 pad) B
constexpr int kChainTmaWarp = 16 + 2 * kChainTmaSlot;  // mbarrier + two slots
#ifndef HC_CHAIN_TMA_T
#define HC_CHAIN_TMA_T 384
#endif
constexpr int kChainTmaThreads = HC_CHAIN_TMA_T;

// kCheckPal: n_pal < 256, so palette indices are range-checked (byte-wise running max).
template <bool kCheckPal, bool kTma = false>
__global__ void __launch_bounds__(kTma ? kChainTmaThreads : 256, kTma ? 2 : 0)
    chain_latent_v3_kernel(const __grid_constant__ ChainLatentParams<6> p) {
  extern __shared__ __align__(16) unsigned char tab3[];
  // Table fill: row r (palette r < 256, illuminant 256 + i), 16-byte chunk c of 16.
  const int n_rows = 256 + p.n_ill;
  for (int i = threadIdx.x; i < n_rows * 16; i += blockDim.x) {
    const int r = i >> 4, c = i & 15;
    const float* src = r < 256 ? (r < p.n_pal ? p.pal + r * 6 : nullptr) : p.ill + (r - 256) * 6;
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    if (src) {
      if (c < 8) v = make_float4(__ldg(src), __ldg(src + 1), __ldg(src + 2), __ldg(src + 3));
      else v = make_float4(__ldg(src + 4), __ldg(src + 5), __ldg(src + 4), __ldg(src + 5));
    }
    *reinterpret_cast<float4*>(tab3 + r * kChainV3Row + c * 16) = v;
  }
  __syncthreads();

  const int lane = threadIdx.x & 31;
  const int g = lane & (kChainLanes - 1);
  // Byte 0: this lane's float4 replica offset, byte 1: its float2 replica offset.
  const uint32_t offs = static_cast<uint32_t>((lane & 7) * 16) | (static_cast<uint32_t>(128 + (lane & 15) * 8) << 8);
  const unsigned char* ill_tab = tab3 + 256 * kChainV3Row;
  float* stg = reinterpret_cast<float*>(tab3 + n_rows * kChainV3Row) + (threadIdx.x >> 5) * kChainV3Stage;
  constexpr int kPixPerWarp = 32 / kChainLanes;
  const int64_t warp_id = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  // kTma: this warp's mbarrier and two record slots
  unsigned char* tma_w = tab3 + n_rows * kChainV3Row + chain_v3_stage_bytes(blockDim.x >> 5) +
                         (threadIdx.x >> 5) * kChainTmaWarp;
  uint64_t* tbar = reinterpret_cast<uint64_t*>(tma_w);
  auto issue_quad = [&](int64_t q, int slot) {  // whole warp; elect.sync issues
    unsigned char* dst = tma_w + 16 + slot * kChainTmaSlot;
    const int64_t left = p.P - q * kPixPerWarp;
    const int npx = left < kPixPerWarp ? static_cast<int>(left) : kPixPerWarp;
    mbar_arrive_expect_tx_w(tbar, npx * (64 * 4 + 64));
    for (int pp = 0; pp < npx; ++pp) {
      const int64_t px = q * kPixPerWarp + pp;
      bulk_g2s_w(dst + pp * 288, p.pidx + px * 64, 64 * 4, tbar);
      bulk_g2s_w(dst + kChainTmaPidx + pp * 80, p.iidx + px * 64, 64, tbar);
    }
  };
  if constexpr (kTma) {
    if ((threadIdx.x & 31) == 0) {
      mbar_init(tbar, 1);
      fence_mbar_init();
    }
    __syncwarp();
    if (warp_id * kPixPerWarp < p.P) issue_quad(warp_id, 0);
  }
  int titer = 0;
  const uint32_t ill_last = static_cast<uint32_t>(p.n_ill - 1);
  uint32_t pmax = 0, imax = 0;  // running maxima of the palette / illuminant indices
  const int per_lane = p.spp / kChainLanes;
  for (int64_t qd = warp_id; qd * kPixPerWarp < p.P; qd += nwarps) {
    const int64_t pix = qd * kPixPerWarp + lane / kChainLanes;
    const bool valid = pix < p.P;
    uint64_t part[3] = {0ull, 0ull, 0ull};
    const int64_t base = pix * p.spp;
    {
      const int64_t npix = (qd + nwarps) * kPixPerWarp + lane / kChainLanes;
      if (npix < p.P) {
        const int64_t nb = npix * p.spp;
        const char* twl = reinterpret_cast<const char*>(p.tw + nb);
        for (int off = g * 128; off < p.spp * 16; off += kChainLanes * 128)
          asm volatile("prefetch.global.L2 [%0];" ::"l"(twl + off));
        if constexpr (!kTma) {
          const char* pkl = reinterpret_cast<const char*>(p.pidx + nb);
          for (int off = g * 128; off < p.spp * 4; off += kChainLanes * 128)
            asm volatile("prefetch.global.L2 [%0];" ::"l"(pkl + off));
          if (g == 0) asm volatile("prefetch.global.L2 [%0];" ::"l"(p.iidx + nb));
        }
      }
    }
    if constexpr (kTma) {  // spp == 64: one group of 8 samples per lane, records from the slot
      const int slot = titer & 1;
      mbar_wait(tbar, titer & 1);  // one quad in flight per warp: completions in quad order
      const unsigned char* src = tma_w + 16 + slot * kChainTmaSlot;
      const int pp = lane / kChainLanes;
      uint32_t pkg[8], lig[8];
      float4 t4g[8];
#pragma unroll
      for (int m = 0; m < 8; ++m) {
        const int smp = g + m * kChainLanes;
        pkg[m] = valid ? *reinterpret_cast<const uint32_t*>(src + pp * 288 + smp * 4) : 0u;
        if (!HC_CHAIN_TMA_IIDX128) lig[m] = valid ? static_cast<uint32_t>(src[kChainTmaPidx + pp * 80 + smp]) : 0u;
        t4g[m] = valid ? ldg_stream(p.tw + base + smp) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
      if (HC_CHAIN_TMA_IIDX128) {
        // 16-byte chunk c holds samples 16c .. 16c+15: lane g's samples g + 16c and g + 8 + 16c are
        // byte g % 4 of word g / 4 and of word 2 + g / 4.
        const uint4* irow = reinterpret_cast<const uint4*>(src + kChainTmaPidx + pp * 80);
        const uint32_t bsel = 0x4440u | static_cast<uint32_t>(g & 3);
        const bool hw = g >= 4;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const uint4 w = valid ? irow[c] : make_uint4(0u, 0u, 0u, 0u);
          lig[2 * c] = __byte_perm(hw ? w.y : w.x, 0u, bsel);
          lig[2 * c + 1] = __byte_perm(hw ? w.w : w.z, 0u, bsel);
        }
      }
      // the other slot was read one quad ago: refill it with the next quad's records
      if (qd + nwarps < (p.P + kPixPerWarp - 1) / kPixPerWarp) issue_quad(qd + nwarps, slot ^ 1);
      ++titer;
#pragma unroll
      for (int m = 0; m < 8; ++m)
        chain_v3_sample<kCheckPal>(tab3, ill_tab, offs, pkg[m], lig[m], t4g[m], ill_last, pmax, imax, part);
    } else {
    // Samples in groups of kGroup per lane, every load of a group issued before any use
    // (~170 B in flight per lane); a past-the-end pixel's lanes load zeros (index 0, weight 0).
    constexpr int kGroup = 8;
    const int full = per_lane - per_lane % kGroup;
    for (int m0 = 0; m0 < full; m0 += kGroup) {
      uint32_t pkg[kGroup], lig[kGroup];
      float4 t4g[kGroup];
#pragma unroll
      for (int m = 0; m < kGroup; ++m) {
        const int64_t s = base + g + static_cast<int64_t>(m0 + m) * kChainLanes;
        pkg[m] = valid ? __ldg(p.pidx + s) : 0u;
        if (!HC_CHAIN_IIDX128) lig[m] = valid ? static_cast<uint32_t>(__ldg(p.iidx + s)) : 0u;
        t4g[m] = valid ? ldg_stream(p.tw + s) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
      if (HC_CHAIN_IIDX128) {
        // The group's 64 illuminant bytes of this pixel in 4 LDG.128 (the pixel group's 8 lanes
        // load the same addresses: 2 L1 tag lookups per instruction instead of 8 byte loads at
        // 2 each); lane g keeps words 2m + g/4 and extracts byte g % 4.  Needs spp % 16 == 0 and
        // a 16-byte aligned iidx (checked by the launcher).
        const uint4* blk = reinterpret_cast<const uint4*>(p.iidx + base + static_cast<int64_t>(m0) * kChainLanes);
        const uint32_t hsel = static_cast<uint32_t>(g >> 2), bsel = 0x4440u | static_cast<uint32_t>(g & 3);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const uint4 w = valid ? __ldg(blk + q) : make_uint4(0u, 0u, 0u, 0u);
          lig[2 * q] = __byte_perm(hsel ? w.y : w.x, 0u, bsel);
          lig[2 * q + 1] = __byte_perm(hsel ? w.w : w.z, 0u, bsel);
        }
      }
#pragma unroll
      for (int m = 0; m < kGroup; ++m)
        chain_v3_sample<kCheckPal>(tab3, ill_tab, offs, pkg[m], lig[m], t4g[m], ill_last, pmax, imax, part);
    }
    for (int m = full; m < per_lane; ++m) {
      const int64_t s = base + g + static_cast<int64_t>(m) * kChainLanes;
      chain_v3_sample<kCheckPal>(tab3, ill_tab, offs, valid ? __ldg(p.pidx + s) : 0u,
                                 valid ? static_cast<uint32_t>(__ldg(p.iidx + s)) : 0u,
                                 valid ? ldg_stream(p.tw + s) : make_float4(0.f, 0.f, 0.f, 0.f), ill_last, pmax,
                                 imax, part);
    }
    }  // !kTma
    // Pixel sums: the 8 lanes' fp32 partials are transposed through a per-warp staging area
    // (6 rows of 33 words: conflict-free both ways), lane g < 6 of each pixel group adds the 8
    // partials of code g in fp64 (renderer.cpp:548-551) and the group's lane 0 gathers the 6
    // codes by shuffle for the XYZ / sRGB projection: 20 L1 wavefronts per pixel quad instead of
    // the 36 of an fp64 butterfly (the kernel is bound by the L1 data pipe).
    const int grp0 = lane & ~(kChainLanes - 1);
    float zz[6];
    if (HC_CHAIN_SUM_SHFL) {
      // Reduce-scatter in fp32 over the 8 lanes (xor 4, 2, 1): 3 + 2 + 1 shuffles leave code
      // 0, 1, 2, 2, 3, 4, 5, 5 in lanes g = 0..7, then the group's lane 0 gathers codes 1..5 (5
      // shuffles): 11 L1 wavefronts per pixel quad instead of 20 through the staging area.
      float pv[6];
#pragma unroll
      for (int j = 0; j < 3; ++j) {
        float2 f;
        memcpy(&f, &part[j], 8);
        pv[2 * j] = f.x;
        pv[2 * j + 1] = f.y;
      }
      const bool b2 = (g & 4) != 0, b1 = (g & 2) != 0, b0 = (g & 1) != 0;
      float q[3];
#pragma unroll
      for (int i = 0; i < 3; ++i) {
        const float r = __shfl_xor_sync(0xffffffffu, b2 ? pv[i] : pv[3 + i], 4);
        q[i] = (b2 ? pv[3 + i] : pv[i]) + r;
      }
      const float r0 = __shfl_xor_sync(0xffffffffu, b1 ? q[0] : q[2], 2);
      const float r1 = __shfl_xor_sync(0xffffffffu, q[1], 2);
      const float s0 = (b1 ? q[2] : q[0]) + r0, s1 = q[1] + r1;  // s1 is used by b1 == 0 lanes only
      const float r2 = __shfl_xor_sync(0xffffffffu, (!b1 && !b0) ? s1 : s0, 1);
      const float t = ((!b1 && b0) ? s1 : s0) + r2;
      const float z = static_cast<float>(static_cast<double>(t) * (1.0 / p.spp));
      const int code = (b2 ? 3 : 0) + (b1 ? 2 : (b0 ? 1 : 0));
      if (valid && p.latent && !(b1 && b0)) p.latent[pix * 6 + code] = z;
      zz[0] = z;
      zz[1] = __shfl_sync(0xffffffffu, z, grp0 + 1);
      zz[2] = __shfl_sync(0xffffffffu, z, grp0 + 2);
      zz[3] = __shfl_sync(0xffffffffu, z, grp0 + 4);
      zz[4] = __shfl_sync(0xffffffffu, z, grp0 + 5);
      zz[5] = __shfl_sync(0xffffffffu, z, grp0 + 6);
    } else {
    __syncwarp();  // the previous quad's staging reads are done
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      float2 f;
      memcpy(&f, &part[j], 8);
      stg[(2 * j) * 33 + lane] = f.x;
      stg[(2 * j + 1) * 33 + lane] = f.y;
    }
    __syncwarp();
    float z = 0.f;
    if (g < 6) {
      double acc = 0.0;
#pragma unroll
      for (int m = 0; m < kChainLanes; ++m) acc += static_cast<double>(stg[g * 33 + grp0 + m]);
      z = static_cast<float>(acc * (1.0 / p.spp));
      if (valid && p.latent) p.latent[pix * 6 + g] = z;
    }
#pragma unroll
    for (int j = 0; j < 6; ++j) zz[j] = __shfl_sync(0xffffffffu, z, grp0 + j);
    }
    if (valid && g == 0) {
      float xyz[3], rgb[3];
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        float a = p.Mxyz[c * 6] * zz[0];
#pragma unroll
        for (int j = 1; j < 6; ++j) a = fmaf(p.Mxyz[c * 6 + j], zz[j], a);
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
  const uint32_t pm = max(max(pmax & 0xffu, (pmax >> 8) & 0xffu), max((pmax >> 16) & 0xffu, pmax >> 24));
  if (pm >= static_cast<uint32_t>(p.n_pal) || imax > ill_last) atomicOr(p.err, kErrIndexRange);
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

// Naive n-sample chain with the lanes over wavelengths (config 4 ground truth, n <= 96): a warp
// takes one pixel, lane j owns lambda j, j + 32, j + 64.  Every random lookup of a sample is then
// one palette row read by the whole warp at consecutive addresses (conflict-free, 128 B per
// wavefront) instead of 32 random rows at stride n (bank conflicts: the thread-per-pixel kernel
// above spends ~3 wavefronts per lookup).  A sample's records (u8x4 palette indices, u8
// illuminant index, float4 throughput factors) are loaded by lane s % 32 (coalesced), staged per
// warp in shared memory and read back as broadcasts.  Per sample and wavelength the chain is the
// Horner form of chain_latent_v3_kernel (re-associated); each lane sums 8
// samples in fp32, then in fp64 (renderer.cpp:548-551); XYZ partials reduce across the warp.
constexpr int kChainLanesRow = 96;  // padded table row (floats)

template <int N>
__global__ void __launch_bounds__(256) chain_spectral_lanes_kernel(const __grid_constant__ ChainSpectralParams<N> p) {
  static_assert(N > 64 && N <= kChainLanesRow, "three wavelength slots per lane");
  extern __shared__ __align__(16) float ltab[];
  float* pal = ltab;
  float* ill = ltab + p.n_pal * kChainLanesRow;
  for (int i = threadIdx.x; i < (p.n_pal + p.n_ill) * kChainLanesRow; i += blockDim.x) {
    const int r = i / kChainLanesRow, l = i - r * kChainLanesRow;
    float v = 0.f;
    if (l < N) v = r < p.n_pal ? __ldg(p.pal + r * N + l) : __ldg(p.ill + (r - p.n_pal) * N + l);
    ltab[i] = v;
  }
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  // per-warp record staging: 32 samples x (u32 palette word, u32 illuminant index, float4 weights)
  uint32_t* rec = reinterpret_cast<uint32_t*>(ltab + (p.n_pal + p.n_ill) * kChainLanesRow) + wib * 32 * 6;
  __syncthreads();
  const int l0 = lane, l1 = lane + 32, l2 = lane + 64;
  const bool has2 = l2 < N;
  const int64_t warp_id = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  const uint32_t npal = static_cast<uint32_t>(p.n_pal), nill = static_cast<uint32_t>(p.n_ill);
  bool bad = false;
  for (int64_t pix = warp_id; pix < p.P; pix += nwarps) {
    const int64_t base = pix * p.spp;
    double acc0 = 0.0, acc1 = 0.0, acc2 = 0.0;
    for (int c0 = 0; c0 < p.spp; c0 += 32) {
      const int cnt = p.spp - c0 < 32 ? p.spp - c0 : 32;  // multiple of 8
      __syncwarp();
      if (lane < cnt) {
        uint32_t pk = __ldg(p.pidx + base + c0 + lane);
        uint32_t li = __ldg(p.iidx + base + c0 + lane);
        const float4 t = ldg_stream(p.tw + base + c0 + lane);
        if (li >= nill) { bad = true; li = 0; }
#pragma unroll
        for (int d = 0; d < 4; ++d)
          if (((pk >> (8 * d)) & 0xffu) >= npal) { bad = true; pk &= ~(0xffu << (8 * d)); }
        rec[lane * 6 + 0] = pk;
        rec[lane * 6 + 1] = li;
        *reinterpret_cast<float2*>(rec + lane * 6 + 2) = make_float2(t.x, t.y);
        *reinterpret_cast<float2*>(rec + lane * 6 + 4) = make_float2(t.z, t.w);
      }
      __syncwarp();
      for (int g0 = 0; g0 < cnt; g0 += 8) {
        float part0 = 0.f, part1 = 0.f, part2 = 0.f;
#pragma unroll 8
        for (int q = g0; q < g0 + 8; ++q) {
          const uint32_t pk = rec[q * 6 + 0], li = rec[q * 6 + 1];  // broadcasts
          const float2 t01 = *reinterpret_cast<const float2*>(rec + q * 6 + 2);
          const float2 t23 = *reinterpret_cast<const float2*>(rec + q * 6 + 4);
          const float4 t = make_float4(t01.x, t01.y, t23.x, t23.y);
          const float* r0 = pal + (pk & 0xffu) * kChainLanesRow;
          const float* r1 = pal + ((pk >> 8) & 0xffu) * kChainLanesRow;
          const float* r2 = pal + ((pk >> 16) & 0xffu) * kChainLanesRow;
          const float* r3 = pal + (pk >> 24) * kChainLanesRow;
          const float* le = ill + li * kChainLanesRow;
          {
            float u = fmaf(r3[l0], t.w, t.z);
            u = fmaf(r2[l0], u, t.y);
            u = fmaf(r1[l0], u, t.x);
            part0 = fmaf(le[l0], r0[l0] * u, part0);
          }
          {
            float u = fmaf(r3[l1], t.w, t.z);
            u = fmaf(r2[l1], u, t.y);
            u = fmaf(r1[l1], u, t.x);
            part1 = fmaf(le[l1], r0[l1] * u, part1);
          }
          if (has2) {
            float u = fmaf(r3[l2], t.w, t.z);
            u = fmaf(r2[l2], u, t.y);
            u = fmaf(r1[l2], u, t.x);
            part2 = fmaf(le[l2], r0[l2] * u, part2);
          }
        }
        acc0 += static_cast<double>(part0);
        acc1 += static_cast<double>(part1);
        acc2 += static_cast<double>(part2);
      }
    }
    const double inv = 1.0 / p.spp;
    const float s0 = static_cast<float>(acc0 * inv), s1 = static_cast<float>(acc1 * inv),
                s2 = has2 ? static_cast<float>(acc2 * inv) : 0.f;
    float xyz[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      float v = fmaf(p.cmf[c * N + l1], s1, p.cmf[c * N + l0] * s0);
      if (has2) v = fmaf(p.cmf[c * N + l2], s2, v);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      xyz[c] = v;
    }
    if (lane == 0) {
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
  if (bad) atomicOr(p.err, kErrIndexRange);
}

}  // namespace hcb
