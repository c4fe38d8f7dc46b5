// hadacodec-b200: the colour-metric tail — the reference's
// consumers of the shading path's output, on the device:
//   exposure_for        renderer.cpp:721-752   luminance nearest-rank percentile -> 1 / value
//   tonemap_srgb8       renderer.cpp:754-773   exposure, clamp, sRGB OETF, 8-bit
//   error_map           renderer.cpp:775-802   per-pixel linear-RGB MSE + mean
//   scene_color_report  evaluation.cpp:122-154 Delta E76 mean / p95 (Lab, D65) + MSE + exposure
//   Delta E94 report    evaluation.cpp:59-86   per-pixel form of multibounce_eval's metric
//
// Arithmetic is fp64 in the reference's operation order; this file is compiled with
// -fmad=false (build.py) so no multiply-add is contracted, which keeps luminance,
// image_to_linear_rgb and the per-pixel MSE bit-identical to the reference.  Only the
// libm calls (cbrt, hypot, pow) differ from glibc by <= 2 ulp.
//
// Percentiles are exact order statistics from a radix select over order-preserving
// 64-bit keys of the doubles, with no sort and no host round trip:
//   1. the kernel that produces the values also writes their keys and a histogram of
//      the top 15 key bits (sign, exponent, 3 mantissa bits; per-CTA 128 KB shared-
//      memory histogram with warp-aggregated increments, non-zero bins flushed);
//   2. one CTA scans the 32768 bins and fixes the bucket holding the wanted rank;
//   3. keys of that bucket are compacted (warp-aggregated appends) — typically a few
//      percent of the pixels;
//   4. four 12/13-bit digit passes over the candidates fix the remaining 49 bits.
// Traffic per select is one extra read of the keys.  Means are per-CTA fp64 partial
// sums reduced in a fixed order (deterministic run to run).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>

#include "hadacodec_b200.h"
#include "hc_internal.h"

namespace hcb {
namespace {

constexpr int kMaxN = 81;
constexpr int kThreads = 256;
constexpr int kProdThreads = 1024;                 // producer kernels: 1 CTA/SM (128 KB histogram)
constexpr int kTopShift = 49;                      // top digit = key bits [49, 64)
constexpr int kTopBins = 1 << (64 - kTopShift);    // 32768
constexpr int kTopSmem = kTopBins * 4;
constexpr int kFineBins = 8192;                    // <= 13-bit digits over the candidates
constexpr int kFineShift[4] = {37, 25, 13, 0};
constexpr int kFineBits[4] = {12, 12, 12, 13};

struct CmfRows {
  double row[3][kMaxN];  // xbar, ybar, zbar (unscaled, the grid's CmfTable rows)
  double dlambda;
  int n;
};

// IEC 61966-2-1 matrices (colorimetry.cpp:22-31).
__constant__ double kXyzToRgbD[9] = {3.2404542, -1.5371385, -0.4985314, -0.9692660, 1.8760108,
                                     0.0415560, 0.0556434,  -0.2040259, 1.0572252};
__constant__ double kRgbToXyzD[9] = {0.4124564, 0.3575761, 0.1804375, 0.2126729, 0.7151522,
                                     0.0721750, 0.0193339, 0.1191920, 0.9503041};

struct SelectState {
  unsigned long long prefix;  // key bits fixed so far
  unsigned long long rank;    // 0-based rank still to find inside the prefix
  unsigned int count;         // candidates (keys of the selected top bucket)
  unsigned int pad;
  unsigned int hist[kFineBins];
};

// Top-digit histogram in dynamic shared memory: zero, add (warp-aggregated: lanes
// with the same bucket add once), flush the non-zero bins to the global histogram.
__device__ __forceinline__ void top_hist_zero(unsigned int* h) {
  for (int i = threadIdx.x; i < kTopBins; i += blockDim.x) h[i] = 0;
  __syncthreads();
}
__device__ __forceinline__ void top_hist_add(unsigned int* h, unsigned long long key, bool valid) {
  const unsigned int active = __ballot_sync(0xffffffffu, valid);
  if (!valid) return;
  const unsigned int bin = static_cast<unsigned int>(key >> kTopShift);
  const unsigned int peers = __match_any_sync(active, bin);
  if ((threadIdx.x & 31) == __ffs(peers) - 1) atomicAdd(&h[bin], __popc(peers));
}
__device__ __forceinline__ void top_hist_flush(const unsigned int* h, unsigned int* g) {
  __syncthreads();
  for (int i = threadIdx.x; i < kTopBins; i += blockDim.x)
    if (h[i]) atomicAdd(&g[i], h[i]);
}

// Order-preserving map double -> uint64 (negatives reversed below positives).
__device__ __forceinline__ unsigned long long dkey(double v) {
  const unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(v));
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ double dval(unsigned long long k) {
  const unsigned long long b = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
  return __longlong_as_double(static_cast<long long>(b));
}

template <int NT>
__device__ __forceinline__ double block_sum(double v) {
  __shared__ double warp_sums[NT / 32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) warp_sums[threadIdx.x >> 5] = v;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.x == 0)
    for (int w = 0; w < NT / 32; ++w) t += warp_sums[w];
  return t;  // valid in thread 0
}

// xyz_to_lab (colorimetry.cpp:118-135).
__device__ __forceinline__ void xyz_to_lab(const double* xyz, const double* white, double* lab) {
  const double delta = 6.0 / 29.0;
  const double delta3 = delta * delta * delta;
  double f[3];
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    const double t = xyz[i] / white[i];
    f[i] = t > delta3 ? cbrt(t) : t / (3.0 * delta * delta) + 4.0 / 29.0;
  }
  lab[0] = 116.0 * f[1] - 16.0;
  lab[1] = 500.0 * (f[0] - f[1]);
  lab[2] = 200.0 * (f[1] - f[2]);
}

// ---------------------------------------------------------------- per-pixel kernels
// Producer kernels run 1024 threads per CTA, one CTA per SM (128 KB top histogram), and
// walk the pixels in warp-uniform strides so the warp-synchronous histogram update is legal.
#define HC_WARP_LOOP(P)                                                                            \
  for (int64_t base = int64_t(blockIdx.x) * kProdThreads + (threadIdx.x & ~31); base < (P);       \
       base += int64_t(gridDim.x) * kProdThreads)

// exposure_for's luminance (renderer.cpp:730-742) -> keys + top histogram.
__global__ void __launch_bounds__(kProdThreads) lum_keys_kernel(const float* __restrict__ img, int64_t P,
                                                                int channels, const __grid_constant__ CmfRows c,
                                                                unsigned long long* __restrict__ keys,
                                                                unsigned int* __restrict__ top_hist) {
  extern __shared__ unsigned int th[];
  top_hist_zero(th);
  HC_WARP_LOOP(P) {
    const int64_t p = base + (threadIdx.x & 31);
    const bool valid = p < P;
    unsigned long long key = 0;
    if (valid) {
      const float* px = img + p * channels;
      double v = 0.0;
      if (channels == 3) {
        v = 0.2126 * static_cast<double>(px[0]) + 0.7152 * static_cast<double>(px[1]) +
            0.0722 * static_cast<double>(px[2]);
      } else {
        for (int i = 0; i < channels; ++i) v += c.row[1][i] * static_cast<double>(px[i]);
        v *= c.dlambda;
      }
      key = dkey(v);
      keys[p] = key;
    }
    top_hist_add(th, key, valid);
  }
  top_hist_flush(th, top_hist);
}

// image_to_linear_rgb for spectral images (renderer.cpp:692-719, colorimetry.cpp:75-87, :103-105).
__global__ void __launch_bounds__(kThreads) spectra_to_rgb_d_kernel(const float* __restrict__ img, int64_t P,
                                                                    const __grid_constant__ CmfRows c,
                                                                    float* __restrict__ rgb) {
  for (int64_t p = blockIdx.x * int64_t(kThreads) + threadIdx.x; p < P; p += int64_t(gridDim.x) * kThreads) {
    const float* px = img + p * c.n;
    double x = 0.0, y = 0.0, z = 0.0;
    for (int i = 0; i < c.n; ++i) {
      const double s = static_cast<double>(px[i]);
      x += c.row[0][i] * s;
      y += c.row[1][i] * s;
      z += c.row[2][i] * s;
    }
    const double xyz[3] = {x * c.dlambda, y * c.dlambda, z * c.dlambda};
#pragma unroll
    for (int r = 0; r < 3; ++r)
      rgb[p * 3 + r] = static_cast<float>(kXyzToRgbD[3 * r] * xyz[0] + kXyzToRgbD[3 * r + 1] * xyz[1] +
                                          kXyzToRgbD[3 * r + 2] * xyz[2]);
  }
}

// error_map's per-pixel term (renderer.cpp:785-797): mean of squared channel differences.
__device__ __forceinline__ double pixel_mse(const float* a, const float* b) {
  double acc = 0.0;
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    const double d = static_cast<double>(a[c]) - static_cast<double>(b[c]);
    acc += d * d;
  }
  return acc / 3.0;
}

// tonemap_srgb8's per-channel byte (renderer.cpp:764-768, srgb_encode colorimetry.cpp:159-162).
__device__ __forceinline__ uint8_t srgb8(float x, double exposure) {
  double v = static_cast<double>(x) * exposure;
  v = v < 0.0 ? 0.0 : (v > 1.0 ? 1.0 : v);
  const double enc = v <= 0.0031308 ? 12.92 * v : 1.055 * pow(v, 1.0 / 2.4) - 0.055;
  return static_cast<uint8_t>(enc * 255.0 + 0.5);
}

// error_map per pixel (mse may be NULL) + per-CTA partial sums.
__global__ void __launch_bounds__(kThreads) mse_kernel(const float* __restrict__ a, const float* __restrict__ b,
                                                       int64_t P, float* __restrict__ mse, double* partials) {
  double acc_all = 0.0;
  for (int64_t p = blockIdx.x * int64_t(kThreads) + threadIdx.x; p < P; p += int64_t(gridDim.x) * kThreads) {
    const double m = pixel_mse(a + p * 3, b + p * 3);
    if (mse) mse[p] = static_cast<float>(m);
    acc_all += m;
  }
  const double t = block_sum<kThreads>(acc_all);
  if (threadIdx.x == 0) partials[blockIdx.x] = t;
}

// scene_color_report's pixel loop (evaluation.cpp:136-149): exposure-scaled linear RGB ->
// XYZ -> Lab (sRGB white) of both images, Delta E76 -> keys + top histogram + partial sum;
// in the same pass error_map's MSE term (:152) and, optionally, the preview bytes
// tonemap_srgb8(test, exposure) that run_report writes next to the report
// (tools/main.cpp:604-623).
__global__ void __launch_bounds__(kProdThreads) de76_kernel(const float* __restrict__ gt,
                                                            const float* __restrict__ test, int64_t P,
                                                            const double* __restrict__ exposure,
                                                            unsigned long long* __restrict__ keys,
                                                            unsigned int* __restrict__ top_hist,
                                                            double* partials, uint8_t* __restrict__ test_srgb8) {
  extern __shared__ unsigned int th[];
  top_hist_zero(th);
  const double e = *exposure;
  const double white[3] = {0.95047, 1.0, 1.08883};  // srgb_reference_white (colorimetry.cpp:111-116)
  double acc_de = 0.0, acc_mse = 0.0;
  HC_WARP_LOOP(P) {
    const int64_t p = base + (threadIdx.x & 31);
    const bool valid = p < P;
    unsigned long long key = 0;
    if (valid) {
      const float* g = gt + p * 3;
      const float* t = test + p * 3;
      double a[3], b[3], xa[3], xb[3], la[3], lb[3];
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        a[c] = static_cast<double>(g[c]) * e;
        b[c] = static_cast<double>(t[c]) * e;
      }
#pragma unroll
      for (int r = 0; r < 3; ++r) {
        xa[r] = kRgbToXyzD[3 * r] * a[0] + kRgbToXyzD[3 * r + 1] * a[1] + kRgbToXyzD[3 * r + 2] * a[2];
        xb[r] = kRgbToXyzD[3 * r] * b[0] + kRgbToXyzD[3 * r + 1] * b[1] + kRgbToXyzD[3 * r + 2] * b[2];
      }
      xyz_to_lab(xa, white, la);
      xyz_to_lab(xb, white, lb);
      const double dl = la[0] - lb[0], da = la[1] - lb[1], db = la[2] - lb[2];
      const double de = sqrt(dl * dl + da * da + db * db);  // delta_e76 (colorimetry.cpp:137-142)
      key = dkey(de);
      keys[p] = key;
      acc_de += de;
      acc_mse += pixel_mse(g, t);
      if (test_srgb8) {
#pragma unroll
        for (int c = 0; c < 3; ++c) test_srgb8[p * 3 + c] = srgb8(t[c], e);
      }
    }
    top_hist_add(th, key, valid);
  }
  top_hist_flush(th, top_hist);
  const double sd = block_sum<kProdThreads>(acc_de);
  __syncthreads();
  const double sm = block_sum<kProdThreads>(acc_mse);
  if (threadIdx.x == 0) {
    partials[blockIdx.x] = sd;
    partials[gridDim.x + blockIdx.x] = sm;
  }
}

// multibounce_eval's Delta E94 (evaluation.cpp:63-74) per pixel: the white is D65 scaled to
// the ground truth's luminance; delta_e94 with graphic-arts constants (colorimetry.cpp:145-157).
__global__ void __launch_bounds__(kProdThreads) de94_kernel(const float* __restrict__ xyz_gt,
                                                            const float* __restrict__ xyz_test, int64_t P,
                                                            double wx, double wy, double wz,
                                                            float* __restrict__ de_out,
                                                            unsigned long long* __restrict__ keys,
                                                            unsigned int* __restrict__ top_hist, double* partials) {
  extern __shared__ unsigned int th[];
  top_hist_zero(th);
  double acc = 0.0;
  HC_WARP_LOOP(P) {
    const int64_t p = base + (threadIdx.x & 31);
    const bool valid = p < P;
    unsigned long long key = 0;
    if (valid) {
      double g[3], t[3], w[3], lg[3], lt[3];
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        g[c] = static_cast<double>(xyz_gt[p * 3 + c]);
        t[c] = static_cast<double>(xyz_test[p * 3 + c]);
      }
      const double y_white = g[1] > 1e-6 ? g[1] : 1e-6;
      const double scale = y_white / wy;
      w[0] = wx * scale;
      w[1] = wy * scale;
      w[2] = wz * scale;
      xyz_to_lab(g, w, lg);
      xyz_to_lab(t, w, lt);
      const double dl = lg[0] - lt[0];
      const double c1 = hypot(lg[1], lg[2]);
      const double c2 = hypot(lt[1], lt[2]);
      const double dc = c1 - c2;
      const double da = lg[1] - lt[1];
      const double db = lg[2] - lt[2];
      double dh2 = da * da + db * db - dc * dc;
      dh2 = dh2 > 0.0 ? dh2 : 0.0;
      const double sc = 1.0 + 0.045 * c1;
      const double sh = 1.0 + 0.015 * c1;
      const double de = sqrt(dl * dl + (dc / sc) * (dc / sc) + dh2 / (sh * sh));
      if (de_out) de_out[p] = static_cast<float>(de);
      key = dkey(de);
      keys[p] = key;
      acc += de;
    }
    top_hist_add(th, key, valid);
  }
  top_hist_flush(th, top_hist);
  const double t = block_sum<kProdThreads>(acc);
  if (threadIdx.x == 0) partials[blockIdx.x] = t;
}

// tonemap_srgb8 (renderer.cpp:754-773) over 3P channel values; the exposure is `exposure`,
// or *exposure_dev when given (device-resident pipelines).
__global__ void __launch_bounds__(kThreads) tonemap_kernel(const float* __restrict__ rgb, int64_t count,
                                                            double exposure, const double* exposure_dev,
                                                            uint8_t* __restrict__ out) {
  const double e = exposure_dev ? *exposure_dev : exposure;
  for (int64_t i = blockIdx.x * int64_t(kThreads) + threadIdx.x; i < count; i += int64_t(gridDim.x) * kThreads)
    out[i] = srgb8(rgb[i], e);
}

// ---------------------------------------------------------------- radix select
// Top bucket: one CTA, 32 bins per thread.  Fixes prefix = bucket << 49 and the rank
// inside it, resets the candidate count and the fine histogram.
__global__ void __launch_bounds__(1024) top_scan_kernel(const unsigned int* __restrict__ top_hist, SelectState* st,
                                                        unsigned long long rank) {
  __shared__ unsigned long long s[1024];
  constexpr int kPer = kTopBins / 1024;
  const int t = threadIdx.x;
  unsigned long long local = 0;
  for (int j = 0; j < kPer; ++j) local += top_hist[t * kPer + j];
  s[t] = local;
  __syncthreads();
  for (int o = 1; o < 1024; o <<= 1) {  // Hillis-Steele inclusive scan
    const unsigned long long v = t >= o ? s[t - o] : 0ull;
    __syncthreads();
    s[t] += v;
    __syncthreads();
  }
  unsigned long long cum = s[t] - local;
  if (cum <= rank && rank < cum + local) {
    for (int j = 0; j < kPer; ++j) {
      const unsigned long long c = top_hist[t * kPer + j];
      if (rank < cum + c) {
        st->prefix = static_cast<unsigned long long>(t * kPer + j) << kTopShift;
        st->rank = rank - cum;
        break;
      }
      cum += c;
    }
  }
  if (t == 0) st->count = 0;
  for (int i = t; i < kFineBins; i += 1024) st->hist[i] = 0;
}

// Keys of the selected top bucket -> cand[] (warp-aggregated appends).
__global__ void __launch_bounds__(kThreads) compact_kernel(const unsigned long long* __restrict__ keys, int64_t P,
                                                           SelectState* st, unsigned long long* __restrict__ cand) {
  const unsigned long long want = st->prefix >> kTopShift;
  const int lane = threadIdx.x & 31;
  for (int64_t base = int64_t(blockIdx.x) * kThreads + (threadIdx.x & ~31); base < P;
       base += int64_t(gridDim.x) * kThreads) {
    const int64_t p = base + lane;
    const unsigned long long k = p < P ? keys[p] : 0ull;
    const bool match = p < P && (k >> kTopShift) == want;
    const unsigned int ball = __ballot_sync(0xffffffffu, match);
    if (!ball) continue;
    const int leader = __ffs(ball) - 1;
    unsigned int pos = 0;
    if (lane == leader) pos = atomicAdd(&st->count, static_cast<unsigned int>(__popc(ball)));
    pos = __shfl_sync(0xffffffffu, pos, leader);
    if (match) cand[pos + __popc(ball & ((1u << lane) - 1u))] = k;
  }
}

__global__ void __launch_bounds__(kThreads) fine_hist_kernel(const unsigned long long* __restrict__ cand,
                                                             SelectState* st, int shift, int bits,
                                                             unsigned long long hi_mask) {
  __shared__ unsigned int h[kFineBins];
  for (int i = threadIdx.x; i < kFineBins; i += kThreads) h[i] = 0;
  __syncthreads();
  const unsigned int count = st->count;
  const unsigned long long prefix = st->prefix;
  const unsigned int dmask = (1u << bits) - 1u;
  for (unsigned int i = blockIdx.x * kThreads + threadIdx.x; i < count; i += gridDim.x * kThreads) {
    const unsigned long long k = cand[i];
    if ((k & hi_mask) == prefix) atomicAdd(&h[(k >> shift) & dmask], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < kFineBins; i += kThreads)
    if (h[i]) atomicAdd(&st->hist[i], h[i]);
}

// One CTA, 8 bins per thread: fix the digit holding the rank, clear the histogram.
__global__ void __launch_bounds__(1024) fine_scan_kernel(SelectState* st, int shift, int bits) {
  __shared__ unsigned long long s[1024];
  constexpr int kPer = kFineBins / 1024;
  const int t = threadIdx.x;
  const int nb = 1 << bits;
  unsigned int c[kPer];
  unsigned long long local = 0;
#pragma unroll
  for (int j = 0; j < kPer; ++j) {
    c[j] = t * kPer + j < nb ? st->hist[t * kPer + j] : 0u;
    local += c[j];
  }
  s[t] = local;
  __syncthreads();
  for (int o = 1; o < 1024; o <<= 1) {
    const unsigned long long v = t >= o ? s[t - o] : 0ull;
    __syncthreads();
    s[t] += v;
    __syncthreads();
  }
  unsigned long long cum = s[t] - local;
  const unsigned long long rank = st->rank;
  __syncthreads();
  if (cum <= rank && rank < cum + local) {
#pragma unroll
    for (int j = 0; j < kPer; ++j) {
      if (rank < cum + c[j]) {
        st->prefix |= static_cast<unsigned long long>(t * kPer + j) << shift;
        st->rank = rank - cum;
        break;
      }
      cum += c[j];
    }
  }
#pragma unroll
  for (int j = 0; j < kPer; ++j) st->hist[t * kPer + j] = 0;
}

// result = the selected double (mode 0) or exposure_for's 1 / value (mode 1).
__global__ void select_value_kernel(const SelectState* st, int mode, double* out) {
  if (threadIdx.x == 0) {
    const double v = dval(st->prefix);
    *out = mode == 0 ? v : (v > 1e-12 ? 1.0 / v : 1.0);
  }
}

// Fixed-order reduction of per-CTA partial sums -> sum / divisor.
__global__ void __launch_bounds__(kThreads) mean_kernel(const double* partials, int count, double divisor, double* out) {
  double v = 0.0;
  for (int i = threadIdx.x; i < count; i += kThreads) v += partials[i];
  const double t = block_sum<kThreads>(v);
  if (threadIdx.x == 0) *out = t / divisor;
}

#undef HC_WARP_LOOP

// ---------------------------------------------------------------- host side
struct Scratch {
  unsigned long long* keys;  // P
  unsigned long long* cand;  // P (worst case)
  unsigned int* top_hist;    // kTopBins
  SelectState* st;
  double* partials;  // 2 x grid_max
  double* results;   // [8]
  float* rgb_a;      // P x 3 (spectral inputs only)
  float* rgb_b;
  int grid;       // 256-thread kernels
  int prod_grid;  // producer kernels (1 CTA / SM)
};

int value_grid(hc_ctx ctx, int64_t P) {
  const int64_t g = (P + kThreads - 1) / kThreads;
  return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(g, int64_t(ctx->sm_count) * 8)));
}

int configure_producers() {
  static int done = 0;
  if (done) return HC_OK;
  HC_CUDA_TRY(cudaFuncSetAttribute(lum_keys_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kTopSmem));
  HC_CUDA_TRY(cudaFuncSetAttribute(de76_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kTopSmem));
  HC_CUDA_TRY(cudaFuncSetAttribute(de94_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kTopSmem));
  done = 1;
  return HC_OK;
}

int get_scratch(hc_ctx ctx, int64_t P, bool rgb_a, bool rgb_b, Scratch* s) {
  int rc = configure_producers();
  if (rc != HC_OK) return rc;
  auto up = [](size_t b) { return (b + 255) & ~size_t(255); };
  s->grid = value_grid(ctx, P);
  s->prod_grid = static_cast<int>(std::max<int64_t>(
      1, std::min<int64_t>((P + kProdThreads - 1) / kProdThreads, int64_t(ctx->sm_count))));
  const int pmax = std::max(s->grid, s->prod_grid);
  const size_t kb = up(sizeof(unsigned long long) * P), hb = up(sizeof(unsigned int) * kTopBins),
               sb = up(sizeof(SelectState)), pb = up(sizeof(double) * 2 * pmax), rb = up(sizeof(double) * 8),
               cb = up(sizeof(float) * 3 * P);
  rc = ensure_scratch(ctx, 2 * kb + hb + sb + pb + rb + (rgb_a ? cb : 0) + (rgb_b ? cb : 0));
  if (rc != HC_OK) return rc;
  char* b = static_cast<char*>(ctx->scratch);
  s->keys = reinterpret_cast<unsigned long long*>(b);
  s->cand = reinterpret_cast<unsigned long long*>(b + kb);
  s->top_hist = reinterpret_cast<unsigned int*>(b + 2 * kb);
  s->st = reinterpret_cast<SelectState*>(b + 2 * kb + hb);
  s->partials = reinterpret_cast<double*>(b + 2 * kb + hb + sb);
  s->results = reinterpret_cast<double*>(b + 2 * kb + hb + sb + pb);
  char* rest = b + 2 * kb + hb + sb + pb + rb;
  s->rgb_a = rgb_a ? reinterpret_cast<float*>(rest) : nullptr;
  s->rgb_b = rgb_b ? reinterpret_cast<float*>(rest + (rgb_a ? cb : 0)) : nullptr;
  return HC_OK;
}

// Nearest-rank index of percentile p over `count` values (renderer.cpp:744-747,
// evaluation.cpp:17-20); negative percentiles clamp to the minimum.
int64_t nearest_rank_index(int64_t count, double p) {
  const double rank = p / 100.0 * static_cast<double>(count);
  const double c = std::ceil(rank);
  if (!(c > 0.0)) return 0;
  int64_t idx = c >= 9.2e18 ? count : static_cast<int64_t>(c);
  idx = idx == 0 ? 0 : idx - 1;
  return std::min<int64_t>(idx, count - 1);
}

int clear_top_hist(hc_ctx ctx, const Scratch& s) {
  HC_CUDA_TRY(cudaMemsetAsync(s.top_hist, 0, sizeof(unsigned int) * kTopBins, ctx->stream));
  return HC_OK;
}

// Exact order statistic `rank` of keys[0, P) whose top histogram is built -> out (mode 0
// value, 1 exposure).  The top histogram is left intact (several ranks of one key set).
int select_rank(hc_ctx ctx, const Scratch& s, int64_t P, int64_t rank, int mode, double* out) {
  top_scan_kernel<<<1, 1024, 0, ctx->stream>>>(s.top_hist, s.st, static_cast<unsigned long long>(rank));
  HC_CHECK_LAUNCH(ctx, "top_scan_kernel");
  compact_kernel<<<s.grid, kThreads, 0, ctx->stream>>>(s.keys, P, s.st, s.cand);
  HC_CHECK_LAUNCH(ctx, "compact_kernel");
  const int fg = std::min(s.grid, ctx->sm_count * 2);
  for (int pass = 0; pass < 4; ++pass) {
    const int shift = kFineShift[pass], bits = kFineBits[pass];
    fine_hist_kernel<<<fg, kThreads, 0, ctx->stream>>>(s.cand, s.st, shift, bits, ~0ull << (shift + bits));
    HC_CHECK_LAUNCH(ctx, "fine_hist_kernel");
    fine_scan_kernel<<<1, 1024, 0, ctx->stream>>>(s.st, shift, bits);
    HC_CHECK_LAUNCH(ctx, "fine_scan_kernel");
  }
  select_value_kernel<<<1, 32, 0, ctx->stream>>>(s.st, mode, out);
  HC_CHECK_LAUNCH(ctx, "select_value_kernel");
  return HC_OK;
}

CmfRows cmf_rows(hc_codec c) {
  CmfRows r;
  std::memset(&r, 0, sizeof(r));
  r.n = c->n;
  r.dlambda = c->dlambda;
  for (int row = 0; row < 3; ++row)
    for (int i = 0; i < c->n; ++i) r.row[row][i] = c->cmf[row * c->n + i];
  return r;
}

int check_image(hc_codec c, const float* img, int channels, const char* what) {
  if (!img) return set_error(HC_EINVAL, std::string(what) + ": null image");
  if (channels != 3 && channels != c->n)
    return set_error(HC_EINVAL, std::string(what) + ": expected 3 or n channels (decode latent images first)");
  return HC_OK;
}

// Linear RGB view of an image: itself (3 channels) or its fp64 image_to_linear_rgb in `tmp`.
int linear_rgb(hc_codec c, const float* img, int channels, int64_t P, float* tmp, const float** out) {
  if (channels == 3) {
    *out = img;
    return HC_OK;
  }
  hc_ctx ctx = c->ctx;
  spectra_to_rgb_d_kernel<<<value_grid(ctx, P), kThreads, 0, ctx->stream>>>(img, P, cmf_rows(c), tmp);
  HC_CHECK_LAUNCH(ctx, "spectra_to_rgb_d_kernel");
  *out = tmp;
  return HC_OK;
}

// exposure_for into *out_dev (device).
int exposure_launch(hc_codec c, const Scratch& s, const float* img, int channels, int64_t P, double percentile,
                    double* out_dev) {
  hc_ctx ctx = c->ctx;
  int rc = clear_top_hist(ctx, s);
  if (rc != HC_OK) return rc;
  lum_keys_kernel<<<s.prod_grid, kProdThreads, kTopSmem, ctx->stream>>>(img, P, channels, cmf_rows(c), s.keys,
                                                                         s.top_hist);
  HC_CHECK_LAUNCH(ctx, "lum_keys_kernel");
  return select_rank(ctx, s, P, nearest_rank_index(P, percentile), 1, out_dev);
}

// scene_color_report into out4_dev = {mean_de76, p95_de76, mse, exposure} (device).
int scene_report_launch(hc_codec c, const Scratch& s, const float* gt, int cgt, const float* test, int ctest,
                        int64_t P, double* out4_dev, uint8_t* test_srgb8) {
  hc_ctx ctx = c->ctx;
  int rc = exposure_launch(c, s, gt, cgt, P, 99.5, out4_dev + 3);
  if (rc != HC_OK) return rc;
  const float *ra, *rb;
  if ((rc = linear_rgb(c, gt, cgt, P, s.rgb_a, &ra)) != HC_OK) return rc;
  if ((rc = linear_rgb(c, test, ctest, P, s.rgb_b, &rb)) != HC_OK) return rc;
  if ((rc = clear_top_hist(ctx, s)) != HC_OK) return rc;
  de76_kernel<<<s.prod_grid, kProdThreads, kTopSmem, ctx->stream>>>(ra, rb, P, out4_dev + 3, s.keys, s.top_hist,
                                                                     s.partials, test_srgb8);
  HC_CHECK_LAUNCH(ctx, "de76_kernel");
  mean_kernel<<<1, kThreads, 0, ctx->stream>>>(s.partials, s.prod_grid, static_cast<double>(P), out4_dev);
  HC_CHECK_LAUNCH(ctx, "mean_kernel");
  mean_kernel<<<1, kThreads, 0, ctx->stream>>>(s.partials + s.prod_grid, s.prod_grid, static_cast<double>(P),
                                               out4_dev + 2);
  HC_CHECK_LAUNCH(ctx, "mean_kernel");
  return select_rank(ctx, s, P, nearest_rank_index(P, 95.0), 0, out4_dev + 1);
}

int fetch_results(hc_ctx ctx, const Scratch& s, double* host, int count) {
  HC_CUDA_TRY(cudaMemcpyAsync(host, s.results, sizeof(double) * count, cudaMemcpyDeviceToHost, ctx->stream));
  HC_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  return HC_OK;
}

}  // namespace
}  // namespace hcb

using namespace hcb;

extern "C" {

int hc_exposure_for(hc_codec c, const float* img, int64_t P, int channels, double percentile, double* exposure) {
  HC_REQUIRE(c && exposure, HC_EINVAL, "exposure_for: null argument");
  HC_REQUIRE(P > 0, HC_EINVAL, "exposure_for: empty image");
  int rc = check_image(c, img, channels, "exposure_for");
  if (rc != HC_OK) return rc;
  Scratch s;
  rc = get_scratch(c->ctx, P, false, false, &s);
  if (rc != HC_OK) return rc;
  rc = exposure_launch(c, s, img, channels, P, percentile, s.results);
  if (rc != HC_OK) return rc;
  return fetch_results(c->ctx, s, exposure, 1);
}

int hc_tonemap_srgb8(hc_ctx ctx, const float* rgb, int64_t P, double exposure, uint8_t* out) {
  HC_REQUIRE(ctx, HC_EINVAL, "tonemap_srgb8: null context");
  HC_REQUIRE(P >= 0, HC_EINVAL, "tonemap_srgb8: negative pixel count");
  if (P == 0) return HC_OK;
  HC_REQUIRE(rgb && out, HC_EINVAL, "tonemap_srgb8: null buffer");
  tonemap_kernel<<<value_grid(ctx, 3 * P), kThreads, 0, ctx->stream>>>(rgb, 3 * P, exposure, nullptr, out);
  HC_CHECK_LAUNCH(ctx, "tonemap_kernel");
  return HC_OK;
}

int hc_error_map(hc_codec c, const float* a, int channels_a, const float* b, int channels_b, int64_t P, float* mse,
                 double* mean_mse) {
  HC_REQUIRE(c && mean_mse, HC_EINVAL, "error_map: null argument");
  HC_REQUIRE(P > 0, HC_EINVAL, "error_map: empty image");
  int rc = check_image(c, a, channels_a, "error_map");
  if (rc == HC_OK) rc = check_image(c, b, channels_b, "error_map");
  if (rc != HC_OK) return rc;
  hc_ctx ctx = c->ctx;
  Scratch s;
  rc = get_scratch(ctx, P, channels_a != 3, channels_b != 3, &s);
  if (rc != HC_OK) return rc;
  const float *ra, *rb;
  if ((rc = linear_rgb(c, a, channels_a, P, s.rgb_a, &ra)) != HC_OK) return rc;
  if ((rc = linear_rgb(c, b, channels_b, P, s.rgb_b, &rb)) != HC_OK) return rc;
  mse_kernel<<<s.grid, kThreads, 0, ctx->stream>>>(ra, rb, P, mse, s.partials);
  HC_CHECK_LAUNCH(ctx, "mse_kernel");
  mean_kernel<<<1, kThreads, 0, ctx->stream>>>(s.partials, s.grid, static_cast<double>(P), s.results);
  HC_CHECK_LAUNCH(ctx, "mean_kernel");
  return fetch_results(ctx, s, mean_mse, 1);
}

int hc_scene_color_report_dev(hc_codec c, const float* gt, int channels_gt, const float* test, int channels_test,
                              int64_t P, double* out4_dev, uint8_t* test_srgb8) {
  HC_REQUIRE(c && out4_dev, HC_EINVAL, "scene_color_report: null argument");
  HC_REQUIRE(P > 0, HC_EINVAL, "scene_color_report: empty image");
  int rc = check_image(c, gt, channels_gt, "scene_color_report");
  if (rc == HC_OK) rc = check_image(c, test, channels_test, "scene_color_report");
  if (rc != HC_OK) return rc;
  Scratch s;
  rc = get_scratch(c->ctx, P, channels_gt != 3, channels_test != 3, &s);
  if (rc != HC_OK) return rc;
  return scene_report_launch(c, s, gt, channels_gt, test, channels_test, P, out4_dev, test_srgb8);
}

int hc_scene_color_report(hc_codec c, const float* gt, int channels_gt, const float* test, int channels_test,
                          int64_t P, double* out4) {
  HC_REQUIRE(c && out4, HC_EINVAL, "scene_color_report: null argument");
  HC_REQUIRE(P > 0, HC_EINVAL, "scene_color_report: empty image");
  int rc = check_image(c, gt, channels_gt, "scene_color_report");
  if (rc == HC_OK) rc = check_image(c, test, channels_test, "scene_color_report");
  if (rc != HC_OK) return rc;
  Scratch s;
  rc = get_scratch(c->ctx, P, channels_gt != 3, channels_test != 3, &s);
  if (rc != HC_OK) return rc;
  rc = scene_report_launch(c, s, gt, channels_gt, test, channels_test, P, s.results, nullptr);
  if (rc != HC_OK) return rc;
  return fetch_results(c->ctx, s, out4, 4);
}

int hc_delta_e94_report(hc_ctx ctx, const float* xyz_gt, const float* xyz_test, int64_t P, const double* white_xyz,
                        float* de, double* out3) {
  HC_REQUIRE(ctx && out3 && white_xyz, HC_EINVAL, "delta_e94_report: null argument");
  HC_REQUIRE(P > 0, HC_EINVAL, "delta_e94_report: empty image");
  HC_REQUIRE(xyz_gt && xyz_test, HC_EINVAL, "delta_e94_report: null image");
  for (int i = 0; i < 3; ++i)
    HC_REQUIRE(white_xyz[i] > 0.0, HC_EDOMAIN, "xyz_to_lab: white point must be positive");
  Scratch s;
  int rc = get_scratch(ctx, P, false, false, &s);
  if (rc != HC_OK) return rc;
  if ((rc = clear_top_hist(ctx, s)) != HC_OK) return rc;
  de94_kernel<<<s.prod_grid, kProdThreads, kTopSmem, ctx->stream>>>(xyz_gt, xyz_test, P, white_xyz[0], white_xyz[1],
                                                                     white_xyz[2], de, s.keys, s.top_hist, s.partials);
  HC_CHECK_LAUNCH(ctx, "de94_kernel");
  mean_kernel<<<1, kThreads, 0, ctx->stream>>>(s.partials, s.prod_grid, static_cast<double>(P), s.results);
  HC_CHECK_LAUNCH(ctx, "mean_kernel");
  if ((rc = select_rank(ctx, s, P, nearest_rank_index(P, 50.0), 0, s.results + 1)) != HC_OK) return rc;
  if ((rc = select_rank(ctx, s, P, nearest_rank_index(P, 95.0), 0, s.results + 2)) != HC_OK) return rc;
  return fetch_results(ctx, s, out3, 3);
}

}  // extern "C"
