// hadacodec-b200: C-ABI runtime — contexts, codecs, argument validation,
// small utility kernels (single-pass shading, reassembly, Hadamard product,
// seeded input generators, L2 flush) and the host-buffer entry points.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "hc_common.cuh"
#include "hc_internal.h"
#include "hc_ops.cuh"

namespace hcb {

static thread_local std::string g_last_error;

int set_error(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

int cuda_error(cudaError_t e, const char* where) {
  return set_error(HC_ECUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

void note_launch(hc_ctx ctx, int n) { ctx->launches.fetch_add(n, std::memory_order_relaxed); }

int ensure_scratch(hc_ctx ctx, size_t bytes, size_t keep) {
  if (ctx->scratch_bytes >= bytes) return HC_OK;
  void* fresh = nullptr;
  HC_CUDA_TRY(cudaMalloc(&fresh, bytes));
  if (ctx->scratch) {
    if (keep) HC_CUDA_TRY(cudaMemcpyAsync(fresh, ctx->scratch, std::min(keep, ctx->scratch_bytes),
                                          cudaMemcpyDeviceToDevice, ctx->stream));
    HC_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    cudaFree(ctx->scratch);
  }
  ctx->scratch = fresh;
  ctx->scratch_bytes = bytes;
  return HC_OK;
}

int encode_rows_tmap_swizzle128(CUtensorMap* map, const void* base, int64_t rows, int row_floats, int box_rows) {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  static std::mutex mu;
  {
    std::lock_guard<std::mutex> lk(mu);
    if (!encode) {
      void* fn = nullptr;
      cudaDriverEntryPointQueryResult q;
      HC_CUDA_TRY(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
      if (!fn || q != cudaDriverEntryPointSuccess)
        return set_error(HC_ECUDA, "cuTensorMapEncodeTiled not available from the driver");
      encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    }
  }
  const cuuint64_t dims[2] = {static_cast<cuuint64_t>(row_floats), static_cast<cuuint64_t>(rows)};
  const cuuint64_t strides[1] = {static_cast<cuuint64_t>(row_floats) * 4};
  const cuuint32_t box[2] = {static_cast<cuuint32_t>(row_floats), static_cast<cuuint32_t>(box_rows)};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(base), dims, strides, box,
                            estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return set_error(HC_ECUDA, "cuTensorMapEncodeTiled failed (" + std::to_string(int(r)) + ")");
  return HC_OK;
}

int ensure_aux_streams(hc_ctx ctx) {
  if (ctx->ev_fork) return HC_OK;
  for (auto& st : ctx->aux) HC_CUDA_TRY(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  HC_CUDA_TRY(cudaEventCreateWithFlags(&ctx->ev_fork, cudaEventDisableTiming));
  return HC_OK;
}

// ------------------------------------------------------------------ RNG (rng.cpp:7-96)
__host__ __device__ inline uint64_t splitmix_mix(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}
constexpr uint64_t kGamma = 0x9e3779b97f4a7c15ull;

// Value i of the counter stream with key `key` (splitmix64_next on state key + i*gamma).
__host__ __device__ inline uint64_t ctr_u64(uint64_t key, uint64_t i) { return splitmix_mix(key + (i + 1) * kGamma); }
__host__ __device__ inline float u24(uint64_t v) { return static_cast<float>(v >> 40) * (1.0f / 16777216.0f); }

struct Xoshiro {
  uint64_t s[4];
  __device__ explicit Xoshiro(uint64_t seed) {
    uint64_t st = seed;
    for (int i = 0; i < 4; ++i) {
      st += kGamma;
      s[i] = splitmix_mix(st);
    }
  }
  __device__ static uint64_t rotl(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }
  __device__ uint64_t next() {
    const uint64_t result = rotl(s[0] + s[3], 23) + s[0];
    const uint64_t t = s[1] << 17;
    s[2] ^= s[0];
    s[3] ^= s[1];
    s[1] ^= s[2];
    s[0] ^= s[3];
    s[2] ^= t;
    s[3] = rotl(s[3], 45);
    return result;
  }
  __device__ double uniform() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }
  __device__ double uniform(double a, double b) { return a + (b - a) * uniform(); }
  __device__ uint32_t index(uint32_t n) { return static_cast<uint32_t>(next() % n); }
};

__global__ void gm_spectra_kernel(uint64_t key, int64_t first, int64_t count, int n, double lmin,
                                  double step, float* out) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= count) return;
  Xoshiro r(ctr_u64(key, static_cast<uint64_t>(first + i)));
  const int m = 1 + static_cast<int>(r.index(4));
  double c[4], sg[4], a[4];
  for (int q = 0; q < m; ++q) {
    c[q] = r.uniform(380.0, 780.0);
    sg[q] = r.uniform(10.0, 100.0);
    a[q] = r.uniform(0.0, 1.0);
  }
  float* o = out + i * n;
  for (int l = 0; l < n; ++l) {
    const double lam = lmin + step * l;
    double acc = 0.0;
    for (int q = 0; q < m; ++q) {
      const double d = (lam - c[q]) / sg[q];
      acc = acc + a[q] * exp(-0.5 * d * d);
    }
    acc = acc < 0.0 ? 0.0 : (acc > 1.0 ? 1.0 : acc);
    o[l] = static_cast<float>(acc);
  }
}

__global__ void gbuffer_kernel(uint64_t kidx, uint64_t kcos, int64_t first, int64_t P, int L, int n_pal,
                               uint32_t* idx, float* cosv) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < P * L; i += stride) {
    cosv[i] = u24(ctr_u64(kcos, static_cast<uint64_t>(first * L + i)));
    if (i < P) idx[i] = static_cast<uint32_t>(ctr_u64(kidx, static_cast<uint64_t>(first + i)) % static_cast<uint64_t>(n_pal));
  }
}

__global__ void chain_synth_kernel(uint64_t kp, uint64_t ki, uint64_t kt, int64_t first, int64_t P, int spp,
                                   int n_pal, int n_ill, uint8_t* pidx, uint8_t* iidx, float* tw) {
  const int64_t nsamp = P * spp;
  const int64_t s0 = first * spp;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < nsamp * 4; i += stride) {
    const uint64_t g = static_cast<uint64_t>(s0 * 4 + i);
    pidx[i] = static_cast<uint8_t>(ctr_u64(kp, g) % static_cast<uint64_t>(n_pal));
    tw[i] = u24(ctr_u64(kt, g));
    if (i < nsamp) iidx[i] = static_cast<uint8_t>(ctr_u64(ki, static_cast<uint64_t>(s0 + i)) % static_cast<uint64_t>(n_ill));
  }
}

__global__ void uniform_kernel(uint64_t key, int64_t first, int64_t count, float* out) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < count; i += stride)
    out[i] = u24(ctr_u64(key, static_cast<uint64_t>(first + i)));
}

// One thread that returns after `cycles` SM clocks (measurement helper, see hc_spin).
__global__ void spin_kernel(long long cycles) {
  const long long t0 = clock64();
  while (clock64() - t0 < cycles) {
  }
}

__global__ void flush_kernel(uint4* buf, int64_t n16, uint32_t salt) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n16; i += stride)
    buf[i] = make_uint4(salt, static_cast<uint32_t>(i), salt ^ 0x5bd1e995u, 0u);
}

// ------------------------------------------------------------------ API-compat kernels
// blockwise_hadamard (codec.cpp:77-85) over rows x k values.
__global__ void hadamard_kernel(const float* a, const float* b, int64_t count, float* out) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < count; i += stride)
    out[i] = a[i] * b[i];
}

// One 3-channel pass (slice_pass renderer.cpp:274-283): channels 3b..3b+2.
__global__ void shade_pass_kernel(int k, int pass, const float* pal, int n_pal, const float* light, int L,
                                  const uint32_t* idx, const float* cosv, int64_t P, float* out,
                                  int* err) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t p = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; p < P; p += stride) {
    uint32_t id = idx[p];
    if (id >= static_cast<uint32_t>(n_pal)) {
      atomicOr(err, kErrIndexRange);
      id = 0;
    }
    for (int c = 0; c < 3; ++c) {
      const int ch = 3 * pass + c;
      float acc = 0.f;
      for (int l = 0; l < L; ++l) acc = fmaf(cosv[p * L + l], light[l * k + ch], acc);
      out[p * 3 + c] = pal[id * k + ch] * acc;
    }
  }
}

struct ReassembleArgs {
  const float* passes[8];
};
__global__ void reassemble_kernel(ReassembleArgs a, int blocks, int64_t P, float* latent) {
  const int k = blocks * 3;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < P * k; i += stride) {
    const int64_t p = i / k;
    const int ch = static_cast<int>(i - p * k);
    latent[i] = a.passes[ch / 3][p * 3 + (ch % 3)];
  }
}

static int grid_for(hc_ctx ctx, int64_t work, int threads = 256) {
  const int64_t g = (work + threads - 1) / threads;
  return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(g, static_cast<int64_t>(ctx->sm_count) * 16)));
}

// IEC 61966-2-1 XYZ -> linear sRGB (colorimetry.cpp:22-26).
static const double kXyzToRgb[9] = {3.2404542, -1.5371385, -0.4985314, -0.9692660, 1.8760108,
                                    0.0415560, 0.0556434,  -0.2040259, 1.0572252};

// softplus (codec.cpp:8-12)
static double softplus(double raw, double beta) {
  const double t = beta * raw;
  if (t > 30.0) return raw;
  return std::log1p(std::exp(t)) / beta;
}

static uint64_t fnv1a64(const char* s) {
  uint64_t h = 0xcbf29ce484222325ull;
  for (; *s; ++s) {
    h ^= static_cast<unsigned char>(*s);
    h *= 0x100000001b3ull;
  }
  return h;
}

}  // namespace hcb

using namespace hcb;

extern "C" {

const char* hc_last_error(void) { return g_last_error.c_str(); }
const char* hc_version(void) { return "hadacodec-b200 0.1 (sm_100a)"; }

int hc_ctx_create(int device, void* stream, hc_ctx* out) {
  HC_REQUIRE(out != nullptr, HC_EINVAL, "hc_ctx_create: out is NULL");
  int ndev = 0;
  HC_CUDA_TRY(cudaGetDeviceCount(&ndev));
  HC_REQUIRE(device >= 0 && device < ndev, HC_EINVAL, "hc_ctx_create: no such device");
  HC_CUDA_TRY(cudaSetDevice(device));
  cudaDeviceProp prop;
  HC_CUDA_TRY(cudaGetDeviceProperties(&prop, device));
  if (prop.major != 10)
    return set_error(HC_EUNSUPPORTED, std::string("hc_ctx_create: built for sm_100a, device is ") + prop.name);
  hc_ctx c = new hc_ctx_s();
  c->device = device;
  c->stream = static_cast<cudaStream_t>(stream);
  c->sm_count = prop.multiProcessorCount;
  c->max_smem_optin = prop.sharedMemPerBlockOptin;
  if (const char* pdl = std::getenv("HC_PDL")) c->pdl = pdl[0] != '0';
  cudaError_t e = cudaMalloc(&c->d_err, sizeof(int));
  if (e != cudaSuccess) {
    delete c;
    return cuda_error(e, "hc_ctx_create");
  }
  e = cudaMemset(c->d_err, 0, sizeof(int));
  if (e != cudaSuccess) {
    cudaFree(c->d_err);
    delete c;
    return cuda_error(e, "hc_ctx_create");
  }
  *out = c;
  return HC_OK;
}

int hc_ctx_destroy(hc_ctx ctx) {
  if (!ctx) return HC_OK;
  cudaSetDevice(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  if (ctx->scratch) cudaFree(ctx->scratch);
  for (auto st : ctx->aux)
    if (st) cudaStreamDestroy(st);
  if (ctx->ev_fork) cudaEventDestroy(ctx->ev_fork);

  if (ctx->d_partials) cudaFree(ctx->d_partials);
  if (ctx->d_err) cudaFree(ctx->d_err);
  delete ctx;
  return HC_OK;
}

int hc_ctx_set_stream(hc_ctx ctx, void* stream) {
  HC_REQUIRE(ctx, HC_EINVAL, "null context");
  ctx->stream = static_cast<cudaStream_t>(stream);
  return HC_OK;
}

int hc_ctx_synchronize(hc_ctx ctx) {
  HC_REQUIRE(ctx, HC_EINVAL, "null context");
  HC_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  int flags = 0;
  HC_CUDA_TRY(cudaMemcpy(&flags, ctx->d_err, sizeof(int), cudaMemcpyDeviceToHost));
  if (flags) {
    HC_CUDA_TRY(cudaMemset(ctx->d_err, 0, sizeof(int)));
    if (flags & kErrNegativeCode)
      return set_error(HC_EDOMAIN,
                       "decode: latent codes are non-negative; refusing to decode a negative entry");
    return set_error(HC_EINVAL, "shading: palette / illuminant index out of range");
  }
  return HC_OK;
}

int64_t hc_ctx_launch_count(hc_ctx ctx) { return ctx ? ctx->launches.load() : -1; }

// ------------------------------------------------------------------ codec
static int codec_finish(hc_ctx ctx, int k, int n, std::vector<double> Ed, std::vector<double> Dd,
                        const double* cmf, double dlambda, hc_codec* out) {
  hc_codec c = new hc_codec_s();
  c->ctx = ctx;
  c->k = k;
  c->n = n;
  c->dlambda = dlambda;
  c->E.assign(Ed.begin(), Ed.end());
  c->D.assign(Dd.begin(), Dd.end());
  c->Ed = std::move(Ed);
  c->Dd = std::move(Dd);
  c->cmf.assign(cmf, cmf + 3 * n);
  c->Mxyz.resize(3 * k);
  c->cmf_dl.resize(3 * n);
  for (int r = 0; r < 3; ++r) {
    for (int i = 0; i < n; ++i) c->cmf_dl[r * n + i] = static_cast<float>(cmf[r * n + i] * dlambda);
    for (int j = 0; j < k; ++j) {
      double acc = 0.0;
      for (int i = 0; i < n; ++i) acc += cmf[r * n + i] * static_cast<double>(c->D[i * k + j]);
      c->Mxyz[r * k + j] = static_cast<float>(acc * dlambda);
    }
  }
  for (int i = 0; i < 9; ++i) c->Crgb[i] = static_cast<float>(kXyzToRgb[i]);
  *out = c;
  return HC_OK;
}

static int validate_dims(hc_ctx ctx, int k, int n, const void* a, const void* b, const double* cmf,
                         double dlambda, hc_codec* out) {
  HC_REQUIRE(ctx && out, HC_EINVAL, "codec: null context / output");
  HC_REQUIRE(k > 0 && k % 3 == 0, HC_EINVAL, "codec weights: k must be a positive multiple of 3");
  HC_REQUIRE(n > 0, HC_EINVAL, "codec weights: n must be positive");
  HC_REQUIRE(a && b && cmf, HC_EINVAL, "codec: null weight / cmf pointer");
  HC_REQUIRE(std::isfinite(dlambda) && dlambda > 0.0, HC_EINVAL, "codec: dlambda must be positive");
  HC_REQUIRE((n == 47 || n == 81) && (k == 3 || k == 6 || k == 9), HC_EUNSUPPORTED,
             "codec: compiled for n in {47, 81}, k in {3, 6, 9}");
  return HC_OK;
}

int hc_codec_create(hc_ctx ctx, int k, int n, const float* E, const float* D, const double* cmf,
                    double dlambda, hc_codec* out) {
  int rc = validate_dims(ctx, k, n, E, D, cmf, dlambda, out);
  if (rc != HC_OK) return rc;
  std::vector<double> e(E, E + k * n), d(D, D + n * k);
  for (double v : e) HC_REQUIRE(std::isfinite(v), HC_EINVAL, "codec weights: non-finite encoder entry");
  for (double v : d) HC_REQUIRE(std::isfinite(v), HC_EINVAL, "codec weights: non-finite decoder entry");
  return codec_finish(ctx, k, n, std::move(e), std::move(d), cmf, dlambda, out);
}

int hc_codec_create_f64(hc_ctx ctx, int k, int n, const double* E, const double* D, const double* cmf,
                        double dlambda, hc_codec* out) {
  int rc = validate_dims(ctx, k, n, E, D, cmf, dlambda, out);
  if (rc != HC_OK) return rc;
  std::vector<double> e(E, E + k * n), d(D, D + n * k);
  for (double v : e) HC_REQUIRE(std::isfinite(v), HC_EINVAL, "codec weights: non-finite encoder entry");
  for (double v : d) HC_REQUIRE(std::isfinite(v), HC_EINVAL, "codec weights: non-finite decoder entry");
  return codec_finish(ctx, k, n, std::move(e), std::move(d), cmf, dlambda, out);
}

int hc_codec_create_raw(hc_ctx ctx, int k, int n, double beta, const double* raw_enc, const double* raw_dec,
                        const double* cmf, double dlambda, hc_codec* out) {
  int rc = validate_dims(ctx, k, n, raw_enc, raw_dec, cmf, dlambda, out);
  if (rc != HC_OK) return rc;
  HC_REQUIRE(beta > 0.0, HC_EINVAL, "codec weights: beta must be positive");
  std::vector<double> e(k * n), d(n * k);
  for (int i = 0; i < k * n; ++i) {
    HC_REQUIRE(std::isfinite(raw_enc[i]), HC_EINVAL, "codec weights: non-finite encoder entry");
    HC_REQUIRE(std::isfinite(raw_dec[i]), HC_EINVAL, "codec weights: non-finite decoder entry");
    e[i] = softplus(raw_enc[i], beta);  // effective_weights (codec.cpp:21-34), kept in fp64
    d[i] = softplus(raw_dec[i], beta);
  }
  return codec_finish(ctx, k, n, std::move(e), std::move(d), cmf, dlambda, out);
}

int hc_codec_destroy(hc_codec c) {
  delete c;
  return HC_OK;
}

int hc_codec_effective_f64(hc_codec c, double* E, double* D) {
  HC_REQUIRE(c, HC_EINVAL, "null codec");
  if (E) std::copy(c->Ed.begin(), c->Ed.end(), E);
  if (D) std::copy(c->Dd.begin(), c->Dd.end(), D);
  return HC_OK;
}

int hc_codec_dims(hc_codec c, int* k, int* n) {
  HC_REQUIRE(c, HC_EINVAL, "null codec");
  if (k) *k = c->k;
  if (n) *n = c->n;
  return HC_OK;
}

int hc_codec_xyz_projection(hc_codec c, float* out) {
  HC_REQUIRE(c && out, HC_EINVAL, "null codec / output");
  std::memcpy(out, c->Mxyz.data(), sizeof(float) * c->Mxyz.size());
  return HC_OK;
}

#define HC_REQUIRE_ROWS(rows) HC_REQUIRE((rows) >= 0, HC_EINVAL, "negative row count")

int hc_encode(hc_codec c, const float* S, int64_t rows, float* Z) {
  HC_REQUIRE(c, HC_EINVAL, "null codec");
  HC_REQUIRE_ROWS(rows);
  HC_REQUIRE(rows == 0 || (S && Z), HC_EINVAL, "encode: null buffer");
  return codec_launch(c, kEncode, S, rows, Z, nullptr, nullptr, nullptr, 0);
}

int hc_decode(hc_codec c, const float* Z, int64_t rows, float* S, float* xyz, float* rgb, int check_negative) {
  HC_REQUIRE(c, HC_EINVAL, "null codec");
  HC_REQUIRE_ROWS(rows);
  HC_REQUIRE(rows == 0 || Z, HC_EINVAL, "decode: null input");
  return codec_launch(c, kDecode, Z, rows, S, xyz, rgb, nullptr, check_negative);
}

int hc_roundtrip(hc_codec c, const float* S, int64_t rows, float* Z, float* S2, float* xyz, float* rgb) {
  HC_REQUIRE(c, HC_EINVAL, "null codec");
  HC_REQUIRE_ROWS(rows);
  HC_REQUIRE(rows == 0 || S, HC_EINVAL, "roundtrip: null input");
  return codec_launch(c, kRoundtrip, S, rows, Z, S2, xyz, rgb, 0);
}

int hc_spectra_to_xyz_rgb(hc_codec c, const float* S, int64_t rows, float* xyz, float* rgb) {
  HC_REQUIRE(c, HC_EINVAL, "null codec");
  HC_REQUIRE_ROWS(rows);
  HC_REQUIRE(rows == 0 || S, HC_EINVAL, "spectra_to_xyz_rgb: null input");
  return codec_launch(c, kProject, S, rows, xyz, rgb, nullptr, nullptr, 0);
}

int hc_blockwise_hadamard(hc_ctx ctx, const float* A, const float* B, int64_t rows, int k, float* out) {
  HC_REQUIRE(ctx, HC_EINVAL, "null context");
  HC_REQUIRE(k > 0, HC_EINVAL, "blockwise_hadamard: dimension mismatch");
  HC_REQUIRE_ROWS(rows);
  if (rows == 0) return HC_OK;
  HC_REQUIRE(A && B && out, HC_EINVAL, "blockwise_hadamard: null buffer");
  const int64_t count = rows * k;
  hadamard_kernel<<<grid_for(ctx, count), 256, 0, ctx->stream>>>(A, B, count, out);
  HC_CHECK_LAUNCH(ctx, "hadamard_kernel");
  return HC_OK;
}

static int check_shade_args(hc_codec c, const float* pal, int n_pal, const float* light, int L,
                            const uint32_t* idx, const float* cosv, int64_t P) {
  HC_REQUIRE(c, HC_EINVAL, "null codec");
  HC_REQUIRE_ROWS(P);
  HC_REQUIRE(n_pal >= 1 && n_pal <= kMaxPalette, HC_EINVAL, "shade: palette size must be in [1, 256]");
  HC_REQUIRE(L >= 1, HC_EINVAL, "shade: need at least one light");
  HC_REQUIRE(pal && light, HC_EINVAL, "shade: null palette / light table");
  HC_REQUIRE(P == 0 || (idx && cosv), HC_EINVAL, "shade: null G-buffer");
  return HC_OK;
}

int hc_shade_latent(hc_codec c, const float* pal_codes, int n_pal, const float* light_codes, int L,
                    const uint32_t* idx, const float* cosv, int64_t P, float* latent, float* spectra,
                    float* xyz, float* rgb) {
  int rc = check_shade_args(c, pal_codes, n_pal, light_codes, L, idx, cosv, P);
  if (rc != HC_OK) return rc;
  return shade_latent_launch(c, pal_codes, n_pal, light_codes, L, idx, cosv, P, latent, spectra, xyz, rgb);
}

int hc_shade_latent_pass(hc_codec c, int pass, const float* pal_codes, int n_pal, const float* light_codes,
                         int L, const uint32_t* idx, const float* cosv, int64_t P, float* pass_image) {
  int rc = check_shade_args(c, pal_codes, n_pal, light_codes, L, idx, cosv, P);
  if (rc != HC_OK) return rc;
  HC_REQUIRE(pass >= 0 && pass < c->k / 3, HC_EINVAL, "shade_latent_pass: pass out of range");
  if (P == 0) return HC_OK;
  HC_REQUIRE(pass_image, HC_EINVAL, "shade_latent_pass: null output");
  hc_ctx ctx = c->ctx;
  rc = ensure_scratch(ctx, sizeof(float) * L * c->k);
  if (rc != HC_OK) return rc;
  HC_CUDA_TRY(cudaMemcpyAsync(ctx->scratch, light_codes, sizeof(float) * L * c->k, cudaMemcpyHostToDevice, ctx->stream));
  shade_pass_kernel<<<grid_for(ctx, P), 256, 0, ctx->stream>>>(c->k, pass, pal_codes, n_pal,
                                                              static_cast<const float*>(ctx->scratch), L, idx,
                                                              cosv, P, pass_image, ctx->d_err);
  HC_CHECK_LAUNCH(ctx, "shade_pass_kernel");
  return HC_OK;
}

int hc_reassemble(hc_ctx ctx, const float* const* passes, int blocks, int64_t P, float* latent) {
  HC_REQUIRE(ctx && passes, HC_EINVAL, "reassemble: null argument");
  HC_REQUIRE(blocks >= 1 && blocks <= 8, HC_EINVAL, "reassemble: 1..8 passes");
  HC_REQUIRE_ROWS(P);
  if (P == 0) return HC_OK;
  HC_REQUIRE(latent, HC_EINVAL, "reassemble: null output");
  ReassembleArgs a;
  for (int b = 0; b < blocks; ++b) {
    HC_REQUIRE(passes[b], HC_EINVAL, "reassemble: null pass image");
    a.passes[b] = passes[b];
  }
  reassemble_kernel<<<grid_for(ctx, P * blocks * 3), 256, 0, ctx->stream>>>(a, blocks, P, latent);
  HC_CHECK_LAUNCH(ctx, "reassemble_kernel");
  return HC_OK;
}

int hc_shade_spectral(hc_codec c, const float* pal_spectra, int n_pal, const float* light_spectra, int L,
                      const uint32_t* idx, const float* cosv, int64_t P, float* spectra, float* xyz,
                      float* rgb) {
  int rc = check_shade_args(c, pal_spectra, n_pal, light_spectra, L, idx, cosv, P);
  if (rc != HC_OK) return rc;
  return shade_spectral_launch(c, pal_spectra, n_pal, light_spectra, L, idx, cosv, P, spectra, xyz, rgb);
}

int hc_multibounce_latent(hc_codec c, const float* pal_codes, int n_pal, const float* ill_codes, int n_ill,
                          const uint8_t* pidx, const uint8_t* iidx, const float* tw, int64_t P, int spp,
                          float* latent, float* xyz, float* rgb) {
  HC_REQUIRE(c && pal_codes && ill_codes, HC_EINVAL, "multibounce: null argument");
  HC_REQUIRE_ROWS(P);
  HC_REQUIRE(P == 0 || (pidx && iidx && tw), HC_EINVAL, "multibounce: null sample buffer");
  return chain_latent_launch(c, pal_codes, n_pal, ill_codes, n_ill, pidx, iidx, tw, P, spp, latent, xyz, rgb);
}

int hc_multibounce_spectral(hc_codec c, const float* pal_spectra, int n_pal, const float* ill_spectra,
                            int n_ill, const uint8_t* pidx, const uint8_t* iidx, const float* tw, int64_t P,
                            int spp, float* xyz, float* rgb) {
  HC_REQUIRE(c && pal_spectra && ill_spectra, HC_EINVAL, "multibounce: null argument");
  HC_REQUIRE_ROWS(P);
  HC_REQUIRE(P == 0 || (pidx && iidx && tw), HC_EINVAL, "multibounce: null sample buffer");
  return chain_spectral_launch(c, pal_spectra, n_pal, ill_spectra, n_ill, pidx, iidx, tw, P, spp, xyz, rgb);
}

int hc_hadamard_loss(hc_codec c, const float* A, const float* B, int64_t pairs, double* sum_dev) {
  HC_REQUIRE(c && sum_dev, HC_EINVAL, "hadamard_loss: null argument");
  HC_REQUIRE_ROWS(pairs);
  HC_REQUIRE(pairs == 0 || (A && B), HC_EINVAL, "hadamard_loss: null input");
  return loss_launch(c, A, B, pairs, sum_dev);
}

// ------------------------------------------------------------------ host-buffer entry points
// Pipelined host-buffer calls: every frame is cut into 256K-pixel chunks, and chunk i
// (counted across all frames of the call) runs H2D copies -> kernel -> D2H copies on
// aux stream i % kAux with device slot i % kAux, so chunk i's H2D, chunk i-1's kernel
// and chunk i-2's D2H overlap, and stream order alone orders each slot's reuse.
// Measured on the B200 host (tools/e2e_sweep.sh): 256K-pixel chunks
// balance the ~4 us per-copy cost against pipeline fill / drain; role streams (all H2D
// on one stream, all D2H on another), a ramped chunk schedule, letting the kernel
// write pinned outputs over PCIe (zero copy) and letting its bulk loads read the pinned
// inputs over PCIe (1.08-1.16 against 1.34 Gpix/s, any chunk size) all measured slower.  With several frames
// per call the pipeline does not drain between frames: frame f + 1's first uploads
// run under frame f's last downloads.
int hc_shade_latent_host_frames(hc_codec c, const float* pal_codes, int n_pal, const float* light_codes, int L,
                                int nframes, const uint32_t* const* idx, const float* const* cosv, int64_t P,
                                float* const* xyz, float* const* rgb) {
  HC_REQUIRE(c, HC_EINVAL, "null codec");
  HC_REQUIRE(nframes >= 0, HC_EINVAL, "shade_latent_host_frames: negative frame count");
  HC_REQUIRE(nframes == 0 || (idx && cosv && xyz && rgb), HC_EINVAL, "shade_latent_host_frames: null frame table");
  for (int f = 0; f < nframes; ++f) {
    int rc = check_shade_args(c, pal_codes, n_pal, light_codes, L, idx[f], cosv[f], P);
    if (rc != HC_OK) return rc;
  }
  if (P == 0 || nframes == 0) return HC_OK;
  hc_ctx ctx = c->ctx;
  static const int64_t kChunk = [] {  // pixels (multiple of every tile size); HC_HOST_CHUNK: tuning only
    const char* e = std::getenv("HC_HOST_CHUNK");
    const int64_t v = e ? std::atoll(e) : 0;
    return v >= 4096 && v % 4096 == 0 ? v : int64_t(262144);
  }();
  constexpr int kSlots = hc_ctx_s::kAux;
  const int64_t cp = P < kChunk ? P : kChunk;
  const size_t pal_b = sizeof(float) * n_pal * c->k;
  auto up = [](size_t b) { return (b + 255) & ~size_t(255); };
  const size_t idx_b = up(sizeof(uint32_t) * cp), cos_b = up(sizeof(float) * cp * L), out_b = up(sizeof(float) * cp * 3);
  const size_t slot_b = idx_b + cos_b + 2 * out_b;
  int rc = ensure_scratch(ctx, up(pal_b) + kSlots * slot_b);
  if (rc != HC_OK) return rc;
  rc = ensure_aux_streams(ctx);
  if (rc != HC_OK) return rc;
  char* base = static_cast<char*>(ctx->scratch);
  float* d_pal = reinterpret_cast<float*>(base);
  HC_CUDA_TRY(cudaMemcpyAsync(d_pal, pal_codes, pal_b, cudaMemcpyHostToDevice, ctx->stream));
  HC_CUDA_TRY(cudaEventRecord(ctx->ev_fork, ctx->stream));
  for (auto st : ctx->aux) HC_CUDA_TRY(cudaStreamWaitEvent(st, ctx->ev_fork, 0));
  cudaStream_t home = ctx->stream;
  // On any error the aux streams are drained before returning: copies in flight read and
  // write the caller's host buffers and the shared scratch.
  auto enqueue = [&]() -> int {
  int64_t ci = 0;
  for (int f = 0; f < nframes; ++f) {
    for (int64_t p0 = 0; p0 < P; p0 += kChunk, ++ci) {
      const int64_t n = P - p0 < kChunk ? P - p0 : kChunk;
      const int s = static_cast<int>(ci % kSlots);
      cudaStream_t st = ctx->aux[ci % hc_ctx_s::kAux];
      char* slot = base + up(pal_b) + s * slot_b;
      uint32_t* d_idx = reinterpret_cast<uint32_t*>(slot);
      float* d_cos = reinterpret_cast<float*>(slot + idx_b);
      float* d_xyz = reinterpret_cast<float*>(slot + idx_b + cos_b);
      float* d_rgb = reinterpret_cast<float*>(slot + idx_b + cos_b + out_b);
      HC_CUDA_TRY(cudaMemcpyAsync(d_idx, idx[f] + p0, sizeof(uint32_t) * n, cudaMemcpyHostToDevice, st));
      HC_CUDA_TRY(cudaMemcpyAsync(d_cos, cosv[f] + p0 * L, sizeof(float) * n * L, cudaMemcpyHostToDevice, st));
      ctx->stream = st;
      rc = shade_latent_launch(c, d_pal, n_pal, light_codes, L, d_idx, d_cos, n, nullptr, nullptr,
                               xyz[f] ? d_xyz : nullptr, rgb[f] ? d_rgb : nullptr);
      ctx->stream = home;
      if (rc != HC_OK) return rc;
      if (xyz[f]) HC_CUDA_TRY(cudaMemcpyAsync(xyz[f] + p0 * 3, d_xyz, sizeof(float) * n * 3, cudaMemcpyDeviceToHost, st));
      if (rgb[f]) HC_CUDA_TRY(cudaMemcpyAsync(rgb[f] + p0 * 3, d_rgb, sizeof(float) * n * 3, cudaMemcpyDeviceToHost, st));
    }
  }
  return HC_OK;
  };
  const int rq = enqueue();
  cudaError_t es = cudaSuccess;
  for (auto st : ctx->aux) {
    const cudaError_t e = cudaStreamSynchronize(st);
    if (es == cudaSuccess) es = e;
  }
  if (rq != HC_OK) return rq;
  if (es != cudaSuccess) return cuda_error(es, "shade_latent_host_frames");
  return hc_ctx_synchronize(ctx);
}

int hc_shade_latent_host(hc_codec c, const float* pal_codes, int n_pal, const float* light_codes, int L,
                         const uint32_t* idx, const float* cosv, int64_t P, float* xyz, float* rgb) {
  return hc_shade_latent_host_frames(c, pal_codes, n_pal, light_codes, L, 1, &idx, &cosv, P, &xyz, &rgb);
}

int hc_roundtrip_host(hc_codec c, const float* S, int64_t rows, float* Z, float* S2, float* xyz, float* rgb) {
  HC_REQUIRE(c, HC_EINVAL, "null codec");
  HC_REQUIRE_ROWS(rows);
  if (rows == 0) return HC_OK;
  HC_REQUIRE(S, HC_EINVAL, "roundtrip: null input");
  hc_ctx ctx = c->ctx;
  auto up = [](size_t b) { return (b + 255) & ~size_t(255); };
  const size_t sb = sizeof(float) * rows * c->n, zb = sizeof(float) * rows * c->k, ob = sizeof(float) * rows * 3;
  int rc = ensure_scratch(ctx, 2 * up(sb) + up(zb) + 2 * up(ob));
  if (rc != HC_OK) return rc;
  char* base = static_cast<char*>(ctx->scratch);
  float* d_s = reinterpret_cast<float*>(base);
  float* d_s2 = reinterpret_cast<float*>(base + up(sb));
  float* d_z = reinterpret_cast<float*>(base + 2 * up(sb));
  float* d_x = reinterpret_cast<float*>(base + 2 * up(sb) + up(zb));
  float* d_r = reinterpret_cast<float*>(base + 2 * up(sb) + up(zb) + up(ob));
  HC_CUDA_TRY(cudaMemcpyAsync(d_s, S, sb, cudaMemcpyHostToDevice, ctx->stream));
  rc = codec_launch(c, kRoundtrip, d_s, rows, Z ? d_z : nullptr, S2 ? d_s2 : nullptr, xyz ? d_x : nullptr,
                    rgb ? d_r : nullptr, 0);
  if (rc != HC_OK) return rc;
  if (Z) HC_CUDA_TRY(cudaMemcpyAsync(Z, d_z, zb, cudaMemcpyDeviceToHost, ctx->stream));
  if (S2) HC_CUDA_TRY(cudaMemcpyAsync(S2, d_s2, sb, cudaMemcpyDeviceToHost, ctx->stream));
  if (xyz) HC_CUDA_TRY(cudaMemcpyAsync(xyz, d_x, ob, cudaMemcpyDeviceToHost, ctx->stream));
  if (rgb) HC_CUDA_TRY(cudaMemcpyAsync(rgb, d_r, ob, cudaMemcpyDeviceToHost, ctx->stream));
  return hc_ctx_synchronize(ctx);
}

// ------------------------------------------------------------------ synthetic inputs
uint64_t hc_stream_key(uint64_t seed, const char* purpose) {
  // Rng::stream (rng.cpp:38-43): st = seed ^ fnv1a64(purpose); seed' = splitmix64_next(st).
  const uint64_t st = seed ^ fnv1a64(purpose ? purpose : "");
  return splitmix_mix(st + kGamma);
}

int hc_synth_gm_spectra(hc_ctx ctx, uint64_t key, int64_t first, int64_t count, int n, double lmin,
                        double step, float* out) {
  HC_REQUIRE(ctx && out && n > 0 && count >= 0, HC_EINVAL, "synth_gm_spectra: bad argument");
  if (count == 0) return HC_OK;
  const int64_t blocks = (count + 127) / 128;
  gm_spectra_kernel<<<static_cast<unsigned>(blocks), 128, 0, ctx->stream>>>(key, first, count, n, lmin, step, out);
  HC_CHECK_LAUNCH(ctx, "gm_spectra_kernel");
  return HC_OK;
}

int hc_synth_gbuffer(hc_ctx ctx, uint64_t key_idx, uint64_t key_cos, int64_t first, int64_t P, int L, int n_pal,
                     uint32_t* idx, float* cosv) {
  HC_REQUIRE(ctx && idx && cosv && L > 0 && n_pal > 0 && P >= 0, HC_EINVAL, "synth_gbuffer: bad argument");
  if (P == 0) return HC_OK;
  gbuffer_kernel<<<grid_for(ctx, P * L), 256, 0, ctx->stream>>>(key_idx, key_cos, first, P, L, n_pal, idx, cosv);
  HC_CHECK_LAUNCH(ctx, "gbuffer_kernel");
  return HC_OK;
}

int hc_synth_chain(hc_ctx ctx, uint64_t kp, uint64_t ki, uint64_t kt, int64_t first, int64_t P, int spp, int n_pal,
                   int n_ill, uint8_t* pidx, uint8_t* iidx, float* tw) {
  HC_REQUIRE(ctx && pidx && iidx && tw && spp > 0 && n_pal > 0 && n_pal <= 256 && n_ill > 0 && n_ill <= 256 && P >= 0,
             HC_EINVAL, "synth_chain: bad argument");
  if (P == 0) return HC_OK;
  chain_synth_kernel<<<grid_for(ctx, P * spp * 4), 256, 0, ctx->stream>>>(kp, ki, kt, first, P, spp, n_pal, n_ill,
                                                                         pidx, iidx, tw);
  HC_CHECK_LAUNCH(ctx, "chain_synth_kernel");
  return HC_OK;
}

int hc_synth_uniform(hc_ctx ctx, uint64_t key, int64_t first, int64_t count, float* out) {
  HC_REQUIRE(ctx && out && count >= 0, HC_EINVAL, "synth_uniform: bad argument");
  if (count == 0) return HC_OK;
  uniform_kernel<<<grid_for(ctx, count), 256, 0, ctx->stream>>>(key, first, count, out);
  HC_CHECK_LAUNCH(ctx, "uniform_kernel");
  return HC_OK;
}

int hc_spin(hc_ctx ctx, int64_t cycles) {
  HC_REQUIRE(ctx && cycles >= 0, HC_EINVAL, "spin: bad argument");
  spin_kernel<<<1, 1, 0, ctx->stream>>>(cycles);
  HC_CHECK_LAUNCH(ctx, "spin_kernel");
  return HC_OK;
}

int hc_flush_l2(hc_ctx ctx, void* buf, int64_t bytes) {
  HC_REQUIRE(ctx && buf && bytes >= 16, HC_EINVAL, "flush_l2: bad argument");
  static uint32_t salt = 1;
  flush_kernel<<<ctx->sm_count * 4, 512, 0, ctx->stream>>>(static_cast<uint4*>(buf), bytes / 16, salt++);
  HC_CHECK_LAUNCH(ctx, "flush_kernel");
  return HC_OK;
}

}  // extern "C"
