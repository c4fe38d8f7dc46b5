// hadacodec-b200: the reference's RGB -> code upsampler (upsampler.hpp:13-50,
// upsampler.cpp:42-72, :170-190) on the GPU, in the reference's own arithmetic: fp64, a
// 3 -> hidden -> hidden -> k network with SiLU after the first two layers and an identity
// head, negative outputs clamped to zero by `upsample` (with the clamped-entry telemetry).
//
// (The tensor-core MLP of hc_mlp.cu is the BASELINE.json variant — 3 -> 64 -> 64 -> 6, ReLU,
// softplus head, bf16 — used for the headline texture-conversion config; this file is the
// drop-in for callers of the reference's `upsample`.)
//
// One warp per texel; every dot product runs in the reference's order (the bias first,
// then the inputs in index order, separate multiply and add: -fmad=false), layer 2 with the
// lanes' outputs i = lane + 32 q as independent chains and the weights transposed so the
// lanes read them coalesced.  SiLU is x / (1 + exp(-x)) as in the reference, with CUDA's exp
// (<= 1 ulp from glibc's), so outputs agree with the reference to ~1e-15 relative rather
// than bit for bit.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <vector>

#include "hadacodec_b200.h"
#include "hc_internal.h"

struct hc_upsampler_s {
  hc_ctx ctx = nullptr;
  int k = 0, hidden = 0;
  double* w = nullptr;  // device: W1 (h x 3) | b1 | W2^T (h x h) | b2 | W3 (k x h) | b3
};

namespace hcb {
namespace {

constexpr int kMaxHidden = 512;
constexpr int kWarps = 4;  // warps per block

__device__ inline double silu(double x) {  // upsampler.cpp:16-19
  const double s = 1.0 / (1.0 + exp(-x));
  return x * s;
}

template <int Q>  // Q = ceil(hidden / 32) outputs per lane in layers 1-2
__global__ void __launch_bounds__(32 * kWarps) upsample_kernel(const double* __restrict__ W, int k, int h,
                                                               const double* __restrict__ rgb, int64_t P, int clamp,
                                                               double* __restrict__ codes,
                                                               unsigned long long* __restrict__ clamped) {
  __shared__ double hbuf[kWarps][2][kMaxHidden];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const double* W1 = W;
  const double* b1 = W1 + 3 * h;
  const double* W2T = b1 + h;
  const double* b2 = W2T + static_cast<size_t>(h) * h;
  const double* W3 = b2 + h;
  const double* b3 = W3 + static_cast<size_t>(k) * h;
  double* h1 = hbuf[warp][0];
  double* h2 = hbuf[warp][1];
  unsigned long long nclamp = 0;
  for (int64_t p = int64_t(blockIdx.x) * kWarps + warp; p < P; p += int64_t(gridDim.x) * kWarps) {
    const double r = rgb[p * 3 + 0], g = rgb[p * 3 + 1], b = rgb[p * 3 + 2];
    // layer 1 (upsampler.cpp:46-54)
    for (int i = lane; i < h; i += 32) {
      double acc = b1[i];
      acc += W1[i * 3 + 0] * r;
      acc += W1[i * 3 + 1] * g;
      acc += W1[i * 3 + 2] * b;
      h1[i] = silu(acc);
    }
    __syncwarp();
    // layer 2 (:55-62): Q independent chains per lane
    double acc[Q];
#pragma unroll
    for (int q = 0; q < Q; ++q) acc[q] = (lane + 32 * q < h) ? b2[lane + 32 * q] : 0.0;
    for (int j = 0; j < h; ++j) {
      const double x = h1[j];
      const double* col = W2T + static_cast<size_t>(j) * h;
#pragma unroll
      for (int q = 0; q < Q; ++q)
        if (lane + 32 * q < h) acc[q] += col[lane + 32 * q] * x;
    }
#pragma unroll
    for (int q = 0; q < Q; ++q)
      if (lane + 32 * q < h) h2[lane + 32 * q] = silu(acc[q]);
    __syncwarp();
    // layer 3 (:63-70) and the clamp of `upsample` (:179-190)
    for (int i = lane; i < k; i += 32) {
      double z = b3[i];
      const double* row = W3 + static_cast<size_t>(i) * h;
      for (int j = 0; j < h; ++j) z += row[j] * h2[j];
      if (clamp && z < 0.0) {
        z = 0.0;
        ++nclamp;
      }
      codes[p * k + i] = z;
    }
    __syncwarp();
  }
  for (int o = 16; o > 0; o >>= 1) nclamp += __shfl_xor_sync(0xffffffffu, nclamp, o);
  if (lane == 0 && nclamp) atomicAdd(clamped, nclamp);
}

}  // namespace
}  // namespace hcb

using namespace hcb;

extern "C" {

int hc_upsampler_create(hc_ctx ctx, int k, int hidden, const double* w1, const double* b1, const double* w2,
                        const double* b2, const double* w3, const double* b3, hc_upsampler* out) {
  HC_REQUIRE(ctx && out, HC_EINVAL, "upsampler: null argument");
  // validate (upsampler.cpp:130-144)
  HC_REQUIRE(k > 0, HC_EINVAL, "upsampler: k must be positive");
  HC_REQUIRE(hidden > 0, HC_EINVAL, "upsampler: hidden width must be positive");
  HC_REQUIRE(hidden <= kMaxHidden, HC_EUNSUPPORTED, "upsampler: hidden width above 512");
  HC_REQUIRE(w1 && b1 && w2 && b2 && w3 && b3, HC_EINVAL, "upsampler: null weight array");
  const size_t h = static_cast<size_t>(hidden), kk = static_cast<size_t>(k);
  auto finite = [](const double* v, size_t n) {
    for (size_t i = 0; i < n; ++i)
      if (!std::isfinite(v[i])) return false;
    return true;
  };
  HC_REQUIRE(finite(w1, h * 3) && finite(b1, h) && finite(w2, h * h) && finite(b2, h) && finite(w3, kk * h) &&
                 finite(b3, kk),
             HC_EINVAL, "upsampler: weights must be finite");
  std::vector<double> host;
  host.reserve(h * 3 + h + h * h + h + kk * h + kk);
  host.insert(host.end(), w1, w1 + h * 3);
  host.insert(host.end(), b1, b1 + h);
  for (size_t j = 0; j < h; ++j)
    for (size_t i = 0; i < h; ++i) host.push_back(w2[i * h + j]);  // W2^T
  host.insert(host.end(), b2, b2 + h);
  host.insert(host.end(), w3, w3 + kk * h);
  host.insert(host.end(), b3, b3 + kk);
  auto* u = new hc_upsampler_s();
  u->ctx = ctx;
  u->k = k;
  u->hidden = hidden;
  cudaError_t e = cudaMalloc(&u->w, sizeof(double) * host.size());
  if (e != cudaSuccess) {
    delete u;
    return cuda_error(e, "cudaMalloc(upsampler)");
  }
  e = cudaMemcpy(u->w, host.data(), sizeof(double) * host.size(), cudaMemcpyHostToDevice);
  if (e != cudaSuccess) {
    cudaFree(u->w);
    delete u;
    return cuda_error(e, "cudaMemcpy(upsampler)");
  }
  *out = u;
  return HC_OK;
}

int hc_upsampler_destroy(hc_upsampler u) {
  if (u) {
    cudaFree(u->w);
    delete u;
  }
  return HC_OK;
}

int hc_upsample_f64(hc_upsampler u, const double* rgb, int64_t P, int clamp, double* codes,
                    uint64_t* clamped_entries) {
  HC_REQUIRE(u, HC_EINVAL, "upsample: null upsampler");
  HC_REQUIRE(P >= 0, HC_EINVAL, "upsample: negative texel count");
  if (P == 0) return HC_OK;
  HC_REQUIRE(rgb && codes, HC_EINVAL, "upsample: null buffer");
  hc_ctx ctx = u->ctx;
  int rc = ensure_scratch(ctx, 64);
  if (rc != HC_OK) return rc;
  auto* counter = static_cast<unsigned long long*>(ctx->scratch);
  HC_CUDA_TRY(cudaMemsetAsync(counter, 0, sizeof(unsigned long long), ctx->stream));
  const int blocks = static_cast<int>(std::min<int64_t>((P + kWarps - 1) / kWarps, int64_t(ctx->sm_count) * 8));
  const int q = (u->hidden + 31) / 32;
  auto launch = [&](auto Qc) {
    upsample_kernel<decltype(Qc)::value><<<blocks, 32 * kWarps, 0, ctx->stream>>>(u->w, u->k, u->hidden, rgb, P, clamp,
                                                                                 codes, counter);
  };
  if (q <= 1) launch(std::integral_constant<int, 1>{});
  else if (q <= 2) launch(std::integral_constant<int, 2>{});
  else if (q <= 4) launch(std::integral_constant<int, 4>{});
  else if (q <= 8) launch(std::integral_constant<int, 8>{});
  else launch(std::integral_constant<int, 16>{});
  HC_CHECK_LAUNCH(ctx, "upsample_kernel");
  unsigned long long n = 0;
  HC_CUDA_TRY(cudaMemcpyAsync(&n, counter, sizeof(n), cudaMemcpyDeviceToHost, ctx->stream));
  HC_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  if (clamped_entries) *clamped_entries += static_cast<uint64_t>(n);
  return HC_OK;
}

}  // extern "C"
