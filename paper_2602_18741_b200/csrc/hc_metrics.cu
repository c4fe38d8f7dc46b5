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
//   1. the kernel that produces the values also writes their keys and histograms of
//      the top 15 and top 9 key bits (per-CTA 130 KB shared-memory histograms with
//      warp-aggregated increments, non-zero bins flushed);
//   2. the bucket holding the wanted rank is found from a 512-bin coarse histogram and
//      the 64 top bins under it;
//   3. keys of that bucket are compacted (per-CTA reserved ranges);
//   4. a 12-bit digit pass over the candidates, a second compaction, and three more
//      digit passes — on one CTA once few candidates remain — fix the other 49 bits.
// Steps 2-4 are one cooperative launch (grid syncs between the phases).
// Traffic per select is one extra read of the keys.  Means are per-CTA fp64 partial
// sums reduced in a fixed order (deterministic run to run).
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
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
constexpr int kCoarseShift = 55;                   // coarse digit = key bits [55, 64): 512 bins
constexpr int kCoarseBins = 1 << (64 - kCoarseShift);
constexpr int kSubBins = kTopBins / kCoarseBins;    // 64 top bins per coarse bin
constexpr int kTopSmem = (kTopBins + kCoarseBins) * 4;
constexpr unsigned int kSmallCand = 32768;         // finish on one CTA below this many keys
constexpr int kFineBins = 8192;                    // <= 13-bit digits over the candidates
// fine digit passes: shift 37, 25, 13, 0; widths 12, 12, 12, 13
__host__ __device__ constexpr int fine_shift(int pass) { return pass == 3 ? 0 : 37 - 12 * pass; }
__host__ __device__ constexpr int fine_bits(int pass) { return pass == 3 ? 13 : 12; }

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
};

// Top-digit histogram in dynamic shared memory (kTopBins fine + kCoarseBins coarse
// counters): zero, add (warp-aggregated: lanes with the same bucket add once), flush the
// non-zero bins to the global histogram (same layout).
__device__ __forceinline__ void top_hist_zero(unsigned int* h) {
  for (int i = threadIdx.x; i < kTopBins + kCoarseBins; i += blockDim.x) h[i] = 0;
  __syncthreads();
}
__device__ __forceinline__ void top_hist_add(unsigned int* h, unsigned long long key, bool valid) {
  const unsigned int active = __ballot_sync(0xffffffffu, valid);
  if (!valid) return;
  const unsigned int bin = static_cast<unsigned int>(key >> kTopShift);
  const unsigned int peers = __match_any_sync(active, bin);
  if ((threadIdx.x & 31) == __ffs(peers) - 1) atomicAdd(&h[bin], __popc(peers));
  const unsigned int cbin = bin / kSubBins;
  const unsigned int cpeers = __match_any_sync(active, cbin);
  if ((threadIdx.x & 31) == __ffs(cpeers) - 1) atomicAdd(&h[kTopBins + cbin], __popc(cpeers));
}
__device__ __forceinline__ void top_hist_flush(const unsigned int* h, unsigned int* g) {
  __syncthreads();
  for (int i = threadIdx.x; i < kTopBins + kCoarseBins; i += blockDim.x)
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

// xyz_to_lab (colorimetry.cpp:118-135), with the white point given as its reciprocal:
// xyz / white -> xyz * (1 / white) and the linear branch's / (3 delta^2) -> * constant,
// <= 1 ulp apart from the reference's quotients (the Delta E bars are 1e-12 relative).
__device__ __forceinline__ void xyz_to_lab(const double* xyz, const double* inv_white, double* lab) {
  const double delta = 6.0 / 29.0;
  const double delta3 = delta * delta * delta;
  const double inv_lin = 1.0 / (3.0 * delta * delta);
  double f[3];
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    const double t = xyz[i] * inv_white[i];
    f[i] = t > delta3 ? cbrt(t) : t * inv_lin + 4.0 / 29.0;
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

// exposure_for's luminance (renderer.cpp:730-742) -> keys + top histogram.  Four pixels
// per lane per iteration keep four independent loads in flight.
__global__ void __launch_bounds__(kProdThreads) lum_keys_kernel(const float* __restrict__ img, int64_t P,
                                                                int channels, const __grid_constant__ CmfRows c,
                                                                unsigned long long* __restrict__ keys,
                                                                unsigned int* __restrict__ top_hist) {
  extern __shared__ unsigned int th[];
  top_hist_zero(th);
  constexpr int U = 4;
  const int lane = threadIdx.x & 31;
  for (int64_t base = (int64_t(blockIdx.x) * kProdThreads + (threadIdx.x & ~31)) * U; base < P;
       base += int64_t(gridDim.x) * kProdThreads * U) {
    unsigned long long key[U];
    bool valid[U];
    if (channels == 3) {
      float r[U][3];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t p = base + u * 32 + lane;
        valid[u] = p < P;
        const float* px = img + (valid[u] ? p : 0) * 3;
        r[u][0] = __ldg(px);
        r[u][1] = __ldg(px + 1);
        r[u][2] = __ldg(px + 2);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const double v = 0.2126 * static_cast<double>(r[u][0]) + 0.7152 * static_cast<double>(r[u][1]) +
                         0.0722 * static_cast<double>(r[u][2]);
        key[u] = dkey(v);
      }
    } else {
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t p = base + u * 32 + lane;
        valid[u] = p < P;
        const float* px = img + (valid[u] ? p : 0) * channels;
        double v = 0.0;
        for (int i = 0; i < channels; ++i) v += c.row[1][i] * static_cast<double>(__ldg(px + i));
        v *= c.dlambda;
        key[u] = dkey(v);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (valid[u]) keys[base + u * 32 + lane] = key[u];
      top_hist_add(th, key[u], valid[u]);
    }
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

// Per-curve XYZ in fp64 (the by-value spectrum_to_xyz / xyz_of_reflectance of the drop-in,
// colorimetry.cpp:75-101): radiance convention (CMF rows, then x dlambda) or, with `w` set,
// the reflectance convention (D65-weighted rows, no scaling); sums in the reference's order.
struct XyzRows {
  double row[3][kMaxN];
  double scale;  // dlambda (radiance) or 1 (reflectance)
  int n;
};
__global__ void __launch_bounds__(kThreads) spectra_to_xyz_f64_kernel(const double* __restrict__ S, int64_t rows,
                                                                      const __grid_constant__ XyzRows c,
                                                                      double* __restrict__ xyz) {
  for (int64_t p = blockIdx.x * int64_t(kThreads) + threadIdx.x; p < rows; p += int64_t(gridDim.x) * kThreads) {
    const double* s = S + p * c.n;
    double x = 0.0, y = 0.0, z = 0.0;
    for (int i = 0; i < c.n; ++i) {
      x += c.row[0][i] * s[i];
      y += c.row[1][i] * s[i];
      z += c.row[2][i] * s[i];
    }
    if (c.scale != 1.0) {
      x *= c.scale;
      y *= c.scale;
      z *= c.scale;
    }
    xyz[p * 3] = x;
    xyz[p * 3 + 1] = y;
    xyz[p * 3 + 2] = z;
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
// The fp64 pow is only needed when the scaled value lands within 0.01 of a rounding
// boundary: a float pow (relative error ~1e-6, i.e. ~3e-4 of a code value) decides all
// other cases identically, so the bytes equal the fp64 reference's.
__device__ __forceinline__ uint8_t srgb8(float x, double exposure) {
  double v = static_cast<double>(x) * exposure;
  v = v < 0.0 ? 0.0 : (v > 1.0 ? 1.0 : v);
  if (v <= 0.0031308) return static_cast<uint8_t>(12.92 * v * 255.0 + 0.5);
  const float t = (1.055f * __powf(static_cast<float>(v), 1.0f / 2.4f) - 0.055f) * 255.0f + 0.5f;
  const float frac = t - floorf(t);
  if (frac > 0.01f && frac < 0.99f) return static_cast<uint8_t>(t);
  const double enc = 1.055 * pow(v, 1.0 / 2.4) - 0.055;
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
  // 1 / srgb_reference_white (colorimetry.cpp:111-116)
  const double white[3] = {1.0 / 0.95047, 1.0, 1.0 / 1.08883};
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
                                                            double wx, double wy, double wz,  // 1/wx, wy, 1/wz
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
      const double inv_scale = wy / y_white;  // 1 / (y_white / wy); wx, wz passed as reciprocals
      w[0] = inv_scale * wx;
      w[1] = 1.0 / y_white;
      w[2] = inv_scale * wz;
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
// Block-wide search of a shared-memory histogram hs[nbins]: the digit whose cumulative
// count passes `rank` and the count below it.  Each thread owns nbins / blockDim
// contiguous bins (read with a per-lane skew: conflict-free), the per-thread sums are
// scanned with warp shuffles.  Every thread returns the same (digit, below).
template <int NT, int NBINS>
__device__ __forceinline__ void find_digit(const unsigned int* hs, unsigned long long rank, int* digit,
                                           unsigned long long* below) {
  constexpr int kPer = NBINS / NT;
  static_assert(kPer >= 1 && (kPer & (kPer - 1)) == 0, "find_digit: power-of-two bins per thread");
  __shared__ unsigned long long warp_tot[NT / 32];
  __shared__ int s_digit;
  __shared__ unsigned long long s_below;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  unsigned long long local = 0;
#pragma unroll 8
  for (int j = 0; j < kPer; ++j) local += hs[t * kPer + ((j + lane) & (kPer - 1))];
  unsigned long long incl = local;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned long long v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  if (lane == 31) warp_tot[warp] = incl;
  __syncthreads();
  unsigned long long warp_base = 0;
  for (int w = 0; w < warp; ++w) warp_base += warp_tot[w];
  unsigned long long cum = warp_base + incl - local;
  if (cum <= rank && rank < cum + local) {
    for (int j = 0; j < kPer; ++j) {
      const unsigned long long cnt = hs[t * kPer + j];
      if (rank < cum + cnt) {
        s_digit = t * kPer + j;
        s_below = cum;
        break;
      }
      cum += cnt;
    }
  }
  __syncthreads();
  *digit = s_digit;
  *below = s_below;
  __syncthreads();
}

// Warp 0 finds, among nb <= 64 bins in shared memory, the one holding `rank`; result in
// (*digit, *below) for the whole block.
__device__ __forceinline__ void find_small(const unsigned int* bins, int nb, unsigned long long rank, int* digit,
                                           unsigned long long* below) {
  __shared__ int s_d;
  __shared__ unsigned long long s_b;
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    const unsigned long long c0 = 2 * lane < nb ? bins[2 * lane] : 0ull;
    const unsigned long long c1 = 2 * lane + 1 < nb ? bins[2 * lane + 1] : 0ull;
    unsigned long long incl = c0 + c1;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += v;
    }
    const unsigned long long cum = incl - c0 - c1;
    if (cum <= rank && rank < cum + c0) {
      s_d = 2 * lane;
      s_b = cum;
    } else if (cum + c0 <= rank && rank < cum + c0 + c1) {
      s_d = 2 * lane + 1;
      s_b = cum + c0;
    }
  }
  __syncthreads();
  *digit = s_d;
  *below = s_b;
  __syncthreads();
}

// Candidates matching `want` (the key bits above `shift`) -> out[] with warp-aggregated
// appends (one global atomic per warp with a match; the buckets are narrow, so matches
// are a few percent of the keys at most).
template <int U>
__device__ __forceinline__ void compact_range(const unsigned long long* __restrict__ src, int64_t n, int shift,
                                              unsigned long long want, unsigned int* counter,
                                              unsigned long long* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t step = int64_t(gridDim.x) * blockDim.x * U;
  for (int64_t base = (int64_t(blockIdx.x) * blockDim.x + (threadIdx.x & ~31)) * U; base < n; base += step) {
    unsigned long long k[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t p = base + u * 32 + lane;
      k[u] = p < n ? __ldcg(src + p) : ~0ull;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const bool match = base + u * 32 + lane < n && (k[u] >> shift) == want;
      const unsigned int ball = __ballot_sync(0xffffffffu, match);
      if (!ball) continue;
      const int leader = __ffs(ball) - 1;
      unsigned int pos = 0;
      if (lane == leader) pos = atomicAdd(counter, static_cast<unsigned int>(__popc(ball)));
      pos = __shfl_sync(0xffffffffu, pos, leader);
      if (match) out[pos + __popc(ball & ((1u << lane) - 1u))] = k[u];
    }
  }
}

// Block-synchronous compaction through a shared-memory staging buffer: per iteration the
// CTA's matches (at most kSelThreads * U) are appended with shared atomics, then one
// global atomic reserves their range and the block copies them out coalesced.  Used for
// the top-bucket pass, where thousands of matches would otherwise serialise on one
// global counter.
template <int U>
__device__ __forceinline__ void compact_staged(const unsigned long long* __restrict__ src, int64_t n, int shift,
                                               unsigned long long want, unsigned int* counter,
                                               unsigned long long* __restrict__ out, unsigned long long* stage) {
  __shared__ unsigned int s_fill, s_base;
  const int lane = threadIdx.x & 31;
  const int64_t step = int64_t(gridDim.x) * blockDim.x * U;
  const int64_t first = int64_t(blockIdx.x) * blockDim.x * U;
  if (threadIdx.x == 0) s_fill = 0;
  __syncthreads();
  for (int64_t chunk = first; chunk < n; chunk += step) {  // block-uniform
    const int64_t base = chunk + (threadIdx.x & ~31) * U;
    unsigned long long k[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t p = base + u * 32 + lane;
      k[u] = p < n ? __ldcs(src + p) : ~0ull;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const bool match = base + u * 32 + lane < n && (k[u] >> shift) == want;
      const unsigned int ball = __ballot_sync(0xffffffffu, match);
      if (!ball) continue;
      const int leader = __ffs(ball) - 1;
      unsigned int pos = 0;
      if (lane == leader) pos = atomicAdd(&s_fill, static_cast<unsigned int>(__popc(ball)));
      pos = __shfl_sync(0xffffffffu, pos, leader);
      if (match) stage[pos + __popc(ball & ((1u << lane) - 1u))] = k[u];
    }
    __syncthreads();
    const unsigned int fill = s_fill;
    if (fill) {
      if (threadIdx.x == 0) s_base = atomicAdd(counter, fill);
      __syncthreads();
      for (unsigned int i = threadIdx.x; i < fill; i += blockDim.x) out[s_base + i] = stage[i];
      __syncthreads();
      if (threadIdx.x == 0) s_fill = 0;
      __syncthreads();
    }
  }
}

// One digit pass over `count` candidates: shared histogram of the digit at `shift` for keys
// matching `prefix` above it.
__device__ __forceinline__ void digit_hist(unsigned int* hs, const unsigned long long* __restrict__ cand,
                                           unsigned int count, unsigned long long prefix, int shift, int bits,
                                           unsigned int first, unsigned int stride) {
  const unsigned long long hi_mask = ~0ull << (shift + bits);
  const unsigned int dmask = (1u << bits) - 1u;
  for (int i = threadIdx.x; i < (1 << bits); i += blockDim.x) hs[i] = 0;
  __syncthreads();
  for (unsigned int i = first; i < count; i += stride) {
    const unsigned long long k = __ldcg(cand + i);
    if ((k & hi_mask) == prefix) atomicAdd(&hs[(k >> shift) & dmask], 1u);
  }
  __syncthreads();
}

// The whole select in one cooperative launch (co-resident grid, one CTA per SM):
//   A. every CTA reads the 512-bin coarse histogram and the 64 top bins under the selected
//      coarse bin (L2-resident) and finds the top bucket holding `rank`;
//   B. the keys of that bucket are compacted into cand[];
//   C. digit pass 0 (bits 37-48) over the candidates on the whole grid (shared histograms
//      flushed to a global one, grid sync, every CTA scans it identically), then the
//      candidates matching the 27 fixed bits are compacted again into cand2[] — typically
//      a handful — and, below kSmallCand of them, CTA 0 alone runs passes 1-3.
// work = [count, count2, 2 x pad, 4 x kFineBins histograms] (16-byte aligned), zeroed
// before the launch.
constexpr int kSelThreads = 512;
__global__ void __launch_bounds__(kSelThreads) select_kernel(const unsigned long long* __restrict__ keys, int64_t P,
                                                             const unsigned int* __restrict__ top_hist,
                                                             unsigned long long rank, unsigned long long* cand,
                                                             unsigned long long* cand2, unsigned int* work, int mode,
                                                             double* out, long long* trace) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  extern __shared__ unsigned int hs[];  // kFineBins histogram (+ staging)
  const bool tr = trace && blockIdx.x == 0 && threadIdx.x == 0;
  if (tr) trace[0] = clock64();
  // ---- A
  for (int i = threadIdx.x; i < kCoarseBins; i += kSelThreads) hs[i] = __ldcg(top_hist + kTopBins + i);
  __syncthreads();
  int d;
  unsigned long long below;
  find_digit<kSelThreads, kCoarseBins>(hs, rank, &d, &below);
  rank -= below;
  const int coarse = d;
  for (int i = threadIdx.x; i < kSubBins; i += kSelThreads) hs[kCoarseBins + i] = __ldcg(top_hist + coarse * kSubBins + i);
  __syncthreads();
  find_small(hs + kCoarseBins, kSubBins, rank, &d, &below);
  rank -= below;
  const unsigned long long bucket = static_cast<unsigned long long>(coarse * kSubBins + d);
  unsigned long long prefix = bucket << kTopShift;
  if (tr) trace[1] = clock64();
  // ---- B
  static_assert(kSelThreads * 8 * 8 <= kFineBins * 4, "staging buffer fits the shared histogram");
  compact_staged<8>(keys, P, kTopShift, bucket, &work[0], cand, reinterpret_cast<unsigned long long*>(hs));
  if (tr) trace[2] = clock64();
  grid.sync();
  const unsigned int count = __ldcg(&work[0]);
  if (tr) trace[3] = clock64();
  // ---- C, pass 0 on the grid
  {
    const int shift = fine_shift(0), bits = fine_bits(0);
    digit_hist(hs, cand, count, prefix, shift, bits, blockIdx.x * kSelThreads + threadIdx.x, gridDim.x * kSelThreads);
    constexpr int kBins0 = 1 << 12;  // fine_bits(0)
    unsigned int* g = work + 4;
    for (int i = threadIdx.x; i < kBins0; i += kSelThreads)
      if (hs[i]) atomicAdd(&g[i], hs[i]);
    grid.sync();
    for (int i = threadIdx.x * 4; i < kBins0; i += kSelThreads * 4)
      *reinterpret_cast<uint4*>(hs + i) = __ldcg(reinterpret_cast<const uint4*>(g + i));
    __syncthreads();
    find_digit<kSelThreads, kBins0>(hs, rank, &d, &below);
    prefix |= static_cast<unsigned long long>(d) << shift;
    rank -= below;
  }
  if (tr) trace[4] = clock64();
  compact_range<2>(cand, count, fine_shift(0), prefix >> fine_shift(0), &work[1], cand2);
  grid.sync();
  const unsigned int count2 = __ldcg(&work[1]);
  if (tr) {
    trace[5] = clock64();
    trace[20] = count;
    trace[21] = count2;
  }
  const bool small = count2 <= kSmallCand;
  if (small && blockIdx.x != 0) return;
  // ---- C, passes 1-3 (CTA 0 alone when few candidates remain, else the grid)
  for (int pass = 1; pass < 4; ++pass) {
    const int shift = fine_shift(pass), bits = fine_bits(pass);
    for (int i = (1 << bits) + threadIdx.x; i < kFineBins; i += kSelThreads) hs[i] = 0;  // unused digits
    if (small) {
      digit_hist(hs, cand2, count2, prefix, shift, bits, threadIdx.x, kSelThreads);
    } else {
      digit_hist(hs, cand2, count2, prefix, shift, bits, blockIdx.x * kSelThreads + threadIdx.x,
                 gridDim.x * kSelThreads);
      unsigned int* g = work + 4 + pass * kFineBins;
      for (int i = threadIdx.x; i < kFineBins; i += kSelThreads)
        if (hs[i]) atomicAdd(&g[i], hs[i]);
      grid.sync();
      for (int i = threadIdx.x * 4; i < kFineBins; i += kSelThreads * 4)
        *reinterpret_cast<uint4*>(hs + i) = __ldcg(reinterpret_cast<const uint4*>(g + i));
      __syncthreads();
    }
    find_digit<kSelThreads, kFineBins>(hs, rank, &d, &below);
    prefix |= static_cast<unsigned long long>(d) << shift;
    rank -= below;
    if (tr) trace[5 + pass] = clock64();
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    const double v = dval(prefix);
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
  unsigned long long* cand2; // P (worst case)
  unsigned int* top_hist;    // kTopBins
  unsigned int* fine;        // select work area: count, 3 x pad, 4 x kFineBins histograms
  SelectState* st;
  double* partials;  // 2 x grid_max
  double* results;   // [8]
  float* rgb_a;      // P x 3 (spectral inputs only)
  float* rgb_b;
  int grid;       // 256-thread kernels
  int prod_grid;  // producer kernels (1 CTA / SM)
  int sel_grid;   // cooperative select (co-resident)
};

int value_grid(hc_ctx ctx, int64_t P) {
  const int64_t g = (P + kThreads - 1) / kThreads;
  return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(g, int64_t(ctx->sm_count) * 8)));
}

int configure_producers() {
  static std::atomic<uint64_t> done{0};  // per device (attributes are per device)
  if (configured_here(done)) return HC_OK;
  HC_CUDA_TRY(cudaFuncSetAttribute(lum_keys_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kTopSmem));
  HC_CUDA_TRY(cudaFuncSetAttribute(de76_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kTopSmem));
  HC_CUDA_TRY(cudaFuncSetAttribute(de94_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kTopSmem));
  mark_configured_here(done);
  return HC_OK;
}

// Co-resident grid of the cooperative select: one CTA per SM.
int sel_grid_size(hc_ctx ctx) {
  static int blocks_per_sm = -1;
  if (blocks_per_sm < 0 &&
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks_per_sm, select_kernel, kSelThreads, kFineBins * 4) !=
          cudaSuccess)
    blocks_per_sm = 0;
  return std::min(blocks_per_sm, 1) * ctx->sm_count;
}

int get_scratch(hc_ctx ctx, int64_t P, bool rgb_a, bool rgb_b, Scratch* s) {
  int rc = configure_producers();
  if (rc != HC_OK) return rc;
  auto up = [](size_t b) { return (b + 255) & ~size_t(255); };
  s->grid = value_grid(ctx, P);
  s->prod_grid = static_cast<int>(std::max<int64_t>(
      1, std::min<int64_t>((P + kProdThreads - 1) / kProdThreads, int64_t(ctx->sm_count))));
  const int pmax = std::max(s->grid, s->prod_grid);
  s->sel_grid = sel_grid_size(ctx);
  if (s->sel_grid < 1) return set_error(HC_EUNSUPPORTED, "select: cooperative grid does not fit");
  const size_t kb = up(sizeof(unsigned long long) * P), hb = up(sizeof(unsigned int) * (kTopBins + kCoarseBins)),
               fb = up(sizeof(unsigned int) * (4 + 4 * kFineBins)), sb = up(sizeof(SelectState)),
               pb = up(sizeof(double) * 2 * pmax), rb = up(sizeof(double) * 8), cb = up(sizeof(float) * 3 * P);
  rc = ensure_scratch(ctx, 3 * kb + hb + fb + sb + pb + rb + (rgb_a ? cb : 0) + (rgb_b ? cb : 0));
  if (rc != HC_OK) return rc;
  char* b0 = static_cast<char*>(ctx->scratch);
  s->cand2 = reinterpret_cast<unsigned long long*>(b0);
  char* b = b0 + kb;
  s->keys = reinterpret_cast<unsigned long long*>(b);
  s->cand = reinterpret_cast<unsigned long long*>(b + kb);
  s->top_hist = reinterpret_cast<unsigned int*>(b + 2 * kb);
  s->fine = reinterpret_cast<unsigned int*>(b + 2 * kb + hb);
  s->st = reinterpret_cast<SelectState*>(b + 2 * kb + hb + fb);
  s->partials = reinterpret_cast<double*>(b + 2 * kb + hb + fb + sb);
  s->results = reinterpret_cast<double*>(b + 2 * kb + hb + fb + sb + pb);
  char* rest = b + 2 * kb + hb + fb + sb + pb + rb;
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
  HC_CUDA_TRY(cudaMemsetAsync(s.top_hist, 0, sizeof(unsigned int) * (kTopBins + kCoarseBins), ctx->stream));
  return HC_OK;
}

// Exact order statistic `rank` of keys[0, P) whose top histogram is built -> out (mode 0
// value, 1 exposure).  The top histogram is left intact (several ranks of one key set).
int select_rank(hc_ctx ctx, const Scratch& s, int64_t P, int64_t rank, int mode, double* out) {
  static long long* sel_trace = nullptr;  // HC_SELECT_TRACE=1: per-phase clock64 of CTA 0 (debug)
  if (!sel_trace && std::getenv("HC_SELECT_TRACE")) cudaMalloc(&sel_trace, 24 * sizeof(long long));
  HC_CUDA_TRY(cudaMemsetAsync(s.fine, 0, sizeof(unsigned int) * (4 + 4 * kFineBins), ctx->stream));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(s.sel_grid);
  cfg.blockDim = dim3(kSelThreads);
  cfg.dynamicSmemBytes = kFineBins * 4;
  cfg.stream = ctx->stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  HC_CUDA_TRY(cudaLaunchKernelEx(&cfg, select_kernel, static_cast<const unsigned long long*>(s.keys), P,
                                 static_cast<const unsigned int*>(s.top_hist), static_cast<unsigned long long>(rank),
                                 s.cand, s.cand2, s.fine, mode, out, sel_trace));
  HC_CHECK_LAUNCH(ctx, "select_kernel");
  if (sel_trace) {
    long long h[24];
    cudaMemcpy(h, sel_trace, sizeof(h), cudaMemcpyDeviceToHost);
    std::fprintf(stderr, "[hc] select: P=%lld cand=%lld cand2=%lld A=%lld B=%lld sync=%lld pass0=%lld compact2=%lld "
                 "p1=%lld p2=%lld p3=%lld\n", static_cast<long long>(P), h[20], h[21], h[1] - h[0], h[2] - h[1],
                 h[3] - h[2], h[4] - h[3], h[5] - h[4], h[6] - h[5], h[7] - h[6], h[8] - h[7]);
  }
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

int hc_spectra_to_xyz_f64(hc_codec c, const double* S, int64_t rows, const double* weights, double* xyz) {
  HC_REQUIRE(c && xyz, HC_EINVAL, "spectra_to_xyz_f64: null argument");
  HC_REQUIRE(rows >= 0, HC_EINVAL, "spectra_to_xyz_f64: negative row count");
  if (rows == 0) return HC_OK;
  HC_REQUIRE(S, HC_EINVAL, "spectra_to_xyz_f64: null spectra");
  XyzRows r;
  std::memset(&r, 0, sizeof(r));
  r.n = c->n;
  for (int row = 0; row < 3; ++row)
    for (int i = 0; i < c->n; ++i) r.row[row][i] = weights ? weights[row * c->n + i] : c->cmf[row * c->n + i];
  r.scale = weights ? 1.0 : c->dlambda;
  hc_ctx ctx = c->ctx;
  spectra_to_xyz_f64_kernel<<<value_grid(ctx, rows), kThreads, 0, ctx->stream>>>(S, rows, r, xyz);
  HC_CHECK_LAUNCH(ctx, "spectra_to_xyz_f64_kernel");
  return HC_OK;
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
  de94_kernel<<<s.prod_grid, kProdThreads, kTopSmem, ctx->stream>>>(xyz_gt, xyz_test, P, 1.0 / white_xyz[0],
                                                                     white_xyz[1], 1.0 / white_xyz[2], de, s.keys,
                                                                     s.top_hist, s.partials);
  HC_CHECK_LAUNCH(ctx, "de94_kernel");
  mean_kernel<<<1, kThreads, 0, ctx->stream>>>(s.partials, s.prod_grid, static_cast<double>(P), s.results);
  HC_CHECK_LAUNCH(ctx, "mean_kernel");
  if ((rc = select_rank(ctx, s, P, nearest_rank_index(P, 50.0), 0, s.results + 1)) != HC_OK) return rc;
  if ((rc = select_rank(ctx, s, P, nearest_rank_index(P, 95.0), 0, s.results + 2)) != HC_OK) return rc;
  return fetch_results(ctx, s, out3, 3);
}

}  // extern "C"
