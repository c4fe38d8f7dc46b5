// hadacodec-b200: the fp64 codec of the reference's encode / decode tools (SURVEY.md §8f
// row 3), bit-identical to the reference.
//
//   run_encode (tools/main.cpp:285-308): resample (spectrum.cpp:60-91) every CSV curve onto
//   the canonical grid, zero it outside the active band (:93-98), encode (codec.cpp:36-46);
//   run_decode (:310-328): decode (codec.cpp:52-71) with its non-negativity check.
//
// The reference computes these in fp64 with sequential sums and no FMA contraction; this
// file is compiled with -fmad=false (build.py FILE_FLAGS) and keeps the same operation
// order, so codes and spectra match bit for bit and the CSVs written from them byte for
// byte.  The resampling plan (which source interval each canonical wavelength falls in, and
// its interpolation weight) depends only on the two grids; it is computed once on the host
// exactly as the reference computes it per curve, and the kernels apply it to every row.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <string>
#include <vector>

#include "hadacodec_b200.h"
#include "hc_internal.h"

namespace hcb {
namespace {

constexpr double kActiveBandMin = 400.0;  // spectrum.hpp:18-19
constexpr double kActiveBandMax = 700.0;

enum : int8_t { kFront = 0, kBack = 1, kLerp = 2, kZero = 3, kIdent = 4 };

template <int K, int N>
__global__ void __launch_bounds__(128) resample_encode_kernel(const double* __restrict__ vals, int64_t rows, int m,
                                                              const int* __restrict__ lo_idx,
                                                              const double* __restrict__ tt,
                                                              const int8_t* __restrict__ mode,
                                                              const double* __restrict__ E,
                                                              double* __restrict__ codes) {
  __shared__ double sE[K * N];
  __shared__ double st[N];
  __shared__ int slo[N];
  __shared__ int8_t smode[N];
  for (int i = threadIdx.x; i < K * N; i += blockDim.x) sE[i] = E[i];
  for (int i = threadIdx.x; i < N; i += blockDim.x) {
    st[i] = tt[i];
    slo[i] = lo_idx[i];
    smode[i] = mode[i];
  }
  __syncthreads();
  for (int64_t r = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; r < rows; r += int64_t(gridDim.x) * blockDim.x) {
    const double* v = vals + r * m;
    double acc[K];
#pragma unroll
    for (int j = 0; j < K; ++j) acc[j] = 0.0;
    for (int i = 0; i < N; ++i) {
      double s;
      const int8_t md = smode[i];
      if (md == kLerp) {
        const double a = v[slo[i]], b = v[slo[i] + 1];
        s = a + st[i] * (b - a);  // spectrum.cpp:84-86
      } else if (md == kIdent) {
        s = v[i];  // plain encode of a curve already on the grid
      } else if (md == kFront) {
        s = v[0];
      } else if (md == kBack) {
        s = v[m - 1];
      } else {
        s = 0.0;  // zero_outside_active_band
      }
#pragma unroll
      for (int j = 0; j < K; ++j) acc[j] += sE[j * N + i] * s;  // codec.cpp:41-43
    }
#pragma unroll
    for (int j = 0; j < K; ++j) codes[r * K + j] = acc[j];
  }
}

template <int K, int N>
__global__ void __launch_bounds__(128) decode_f64_kernel(const double* __restrict__ codes, int64_t rows,
                                                         const double* __restrict__ D, double* __restrict__ out,
                                                         unsigned long long* __restrict__ first_bad) {
  __shared__ double sD[N * K];
  for (int i = threadIdx.x; i < N * K; i += blockDim.x) sD[i] = D[i];
  __syncthreads();
  for (int64_t r = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; r < rows; r += int64_t(gridDim.x) * blockDim.x) {
    double z[K];
    bool ok = true;
#pragma unroll
    for (int j = 0; j < K; ++j) {
      z[j] = codes[r * K + j];
      ok &= z[j] >= 0.0;  // codec.cpp:56-62 (NaN fails too)
    }
    if (!ok) atomicMin(first_bad, static_cast<unsigned long long>(r));
    for (int i = 0; i < N; ++i) {
      double acc = 0.0;
#pragma unroll
      for (int j = 0; j < K; ++j) acc += sD[i * K + j] * z[j];  // codec.cpp:64-68
      out[r * N + i] = acc;
    }
  }
}

int grid_rows(hc_ctx ctx, int64_t rows) {
  const int64_t g = (rows + 127) / 128;
  return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(g, int64_t(ctx->sm_count) * 8)));
}

template <class F>
int dispatch_kn(int k, int n, F&& f) {
  if (n == 47) {
    if (k == 3) return f(std::integral_constant<int, 3>{}, std::integral_constant<int, 47>{});
    if (k == 6) return f(std::integral_constant<int, 6>{}, std::integral_constant<int, 47>{});
    if (k == 9) return f(std::integral_constant<int, 9>{}, std::integral_constant<int, 47>{});
  } else if (n == 81) {
    if (k == 3) return f(std::integral_constant<int, 3>{}, std::integral_constant<int, 81>{});
    if (k == 6) return f(std::integral_constant<int, 6>{}, std::integral_constant<int, 81>{});
    if (k == 9) return f(std::integral_constant<int, 9>{}, std::integral_constant<int, 81>{});
  }
  return set_error(HC_EUNSUPPORTED, "codec64: compiled for n in {47, 81}, k in {3, 6, 9}");
}

int launch_encode(hc_codec codec, const double* values, int64_t rows, int m, const std::vector<int>& lo,
                  const std::vector<double>& t, const std::vector<int8_t>& mode, double* codes);

}  // namespace
}  // namespace hcb

using namespace hcb;

extern "C" {

int hc_encode_resampled_f64(hc_codec codec, const double* src_wavelengths, int m, const double* values, int64_t rows,
                            double lambda_min, double lambda_step, int zero_outside, double* codes) {
  HC_REQUIRE(codec, HC_EINVAL, "encode_resampled: null codec");
  HC_REQUIRE(rows >= 0, HC_EINVAL, "encode_resampled: negative row count");
  // resample's argument checks (spectrum.cpp:63-73)
  HC_REQUIRE(m > 0 && src_wavelengths, HC_EINVAL, "resample: empty source grid");
  for (int i = 1; i < m; ++i)
    HC_REQUIRE(src_wavelengths[i] > src_wavelengths[i - 1], HC_EINVAL,
               "resample: source grid must be strictly increasing");
  if (rows == 0) return HC_OK;
  HC_REQUIRE(values && codes, HC_EINVAL, "encode_resampled: null buffer");
  const int n = codec->n;
  // the plan, as resample computes it per curve (spectrum.cpp:74-90)
  std::vector<int> lo(n, 0);
  std::vector<double> t(n, 0.0);
  std::vector<int8_t> mode(n, kFront);
  for (int i = 0; i < n; ++i) {
    const double lambda = lambda_min + lambda_step * i;  // wavelength_at (spectrum.hpp:21)
    if (lambda <= src_wavelengths[0]) {
      mode[i] = kFront;
    } else if (lambda >= src_wavelengths[m - 1]) {
      mode[i] = kBack;
    } else {
      const int hi = static_cast<int>(std::upper_bound(src_wavelengths, src_wavelengths + m, lambda) - src_wavelengths);
      lo[i] = hi - 1;
      t[i] = (lambda - src_wavelengths[hi - 1]) / (src_wavelengths[hi] - src_wavelengths[hi - 1]);
      mode[i] = kLerp;
    }
    if (zero_outside && (lambda < kActiveBandMin || lambda > kActiveBandMax)) mode[i] = kZero;
  }
  return launch_encode(codec, values, rows, m, lo, t, mode, codes);
}

int hc_encode_f64(hc_codec codec, const double* spectra, int64_t rows, double* codes) {
  HC_REQUIRE(codec, HC_EINVAL, "encode_f64: null codec");
  HC_REQUIRE(rows >= 0, HC_EINVAL, "encode_f64: negative row count");
  if (rows == 0) return HC_OK;
  HC_REQUIRE(spectra && codes, HC_EINVAL, "encode_f64: null buffer");
  const int n = codec->n;
  std::vector<int> lo(n);
  for (int i = 0; i < n; ++i) lo[i] = i;
  return launch_encode(codec, spectra, rows, n, lo, std::vector<double>(n, 0.0), std::vector<int8_t>(n, kIdent),
                       codes);
}

}  // extern "C"

namespace hcb {
namespace {
int launch_encode(hc_codec codec, const double* values, int64_t rows, int m, const std::vector<int>& lo,
                  const std::vector<double>& t, const std::vector<int8_t>& mode, double* codes) {
  hc_ctx ctx = codec->ctx;
  const int n = codec->n, k = codec->k;
  // device copies: E (k x n), plan
  const size_t eb = sizeof(double) * k * n, pb = (sizeof(int) + sizeof(double) + 1) * n;
  int rc = ensure_scratch(ctx, eb + pb + 64);
  if (rc != HC_OK) return rc;
  char* base = static_cast<char*>(ctx->scratch);
  double* dE = reinterpret_cast<double*>(base);
  double* dt = reinterpret_cast<double*>(base + eb);
  int* dlo = reinterpret_cast<int*>(base + eb + sizeof(double) * n);
  int8_t* dmode = reinterpret_cast<int8_t*>(base + eb + (sizeof(double) + sizeof(int)) * n);
  HC_CUDA_TRY(cudaMemcpyAsync(dE, codec->Ed.data(), eb, cudaMemcpyHostToDevice, ctx->stream));
  HC_CUDA_TRY(cudaMemcpyAsync(dt, t.data(), sizeof(double) * n, cudaMemcpyHostToDevice, ctx->stream));
  HC_CUDA_TRY(cudaMemcpyAsync(dlo, lo.data(), sizeof(int) * n, cudaMemcpyHostToDevice, ctx->stream));
  HC_CUDA_TRY(cudaMemcpyAsync(dmode, mode.data(), n, cudaMemcpyHostToDevice, ctx->stream));
  rc = dispatch_kn(k, n, [&](auto K, auto N) {
    resample_encode_kernel<decltype(K)::value, decltype(N)::value>
        <<<grid_rows(ctx, rows), 128, 0, ctx->stream>>>(values, rows, m, dlo, dt, dmode, dE, codes);
    HC_CHECK_LAUNCH(ctx, "resample_encode_kernel");
    return HC_OK;
  });
  if (rc != HC_OK) return rc;
  HC_CUDA_TRY(cudaStreamSynchronize(ctx->stream));  // host plan buffers go out of scope
  return HC_OK;
}
}  // namespace
}  // namespace hcb

extern "C" {

int hc_decode_f64(hc_codec codec, const double* codes, int64_t rows, double* spectra, int64_t* first_negative_row) {
  HC_REQUIRE(codec, HC_EINVAL, "decode_f64: null codec");
  HC_REQUIRE(rows >= 0, HC_EINVAL, "decode_f64: negative row count");
  if (first_negative_row) *first_negative_row = -1;
  if (rows == 0) return HC_OK;
  HC_REQUIRE(codes && spectra, HC_EINVAL, "decode_f64: null buffer");
  hc_ctx ctx = codec->ctx;
  const int n = codec->n, k = codec->k;
  const size_t db = sizeof(double) * n * k;
  int rc = ensure_scratch(ctx, db + 64);
  if (rc != HC_OK) return rc;
  double* dD = static_cast<double*>(ctx->scratch);
  unsigned long long* bad = reinterpret_cast<unsigned long long*>(static_cast<char*>(ctx->scratch) + db);
  const unsigned long long none = ~0ull;
  HC_CUDA_TRY(cudaMemcpyAsync(dD, codec->Dd.data(), db, cudaMemcpyHostToDevice, ctx->stream));
  HC_CUDA_TRY(cudaMemcpyAsync(bad, &none, sizeof(none), cudaMemcpyHostToDevice, ctx->stream));
  rc = dispatch_kn(k, n, [&](auto K, auto N) {
    decode_f64_kernel<decltype(K)::value, decltype(N)::value>
        <<<grid_rows(ctx, rows), 128, 0, ctx->stream>>>(codes, rows, dD, spectra, bad);
    HC_CHECK_LAUNCH(ctx, "decode_f64_kernel");
    return HC_OK;
  });
  if (rc != HC_OK) return rc;
  unsigned long long first = none;
  HC_CUDA_TRY(cudaMemcpyAsync(&first, bad, sizeof(first), cudaMemcpyDeviceToHost, ctx->stream));
  HC_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  if (first != none) {
    if (first_negative_row) *first_negative_row = static_cast<int64_t>(first);
    return set_error(HC_EDOMAIN, "decode: latent codes are non-negative; refusing to decode a negative entry (row " +
                                     std::to_string(first) + ")");
  }
  return HC_OK;
}

}  // extern "C"
