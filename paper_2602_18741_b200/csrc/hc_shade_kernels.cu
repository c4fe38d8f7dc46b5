// hadacodec-b200: G-buffer shading kernels — latent (fused k/3 passes +
// reassembly + decode/projection) and naive n-sample spectral.
// Reference: renderer.cpp:161-271 (compile_scene), :274-283 (slice_pass),
// :505-510 (NEE channel loop), :645-657 (reassembly), :661-719 (decode/project).
#include <algorithm>
#include <cstring>

#include "hc_launch.cuh"
#include "hc_ops.cuh"

#ifndef HC_C2_T
#define HC_C2_T 256
#endif
#ifndef HC_C2_THREADS
#define HC_C2_THREADS 256
#endif
#ifndef HC_SPEC_T  // spectra-writing variants (config 3)
#define HC_SPEC_T 64
#endif
#ifndef HC_SPEC_STAGES
#define HC_SPEC_STAGES 2
#endif
#ifndef HC_C2_STAGES
#define HC_C2_STAGES 4
#endif

namespace hcb {

// ---------------------------------------------------------------- any light count
// Runtime-L shading for light counts without a fused TMA instantiation (the
// reference accepts any number of emitters): thread per pixel, G-buffer read with
// plain loads, light codes / SPDs in the constant bank (L <= kMaxGenericLights).
constexpr int kMaxGenericLights = 64;

template <int N, int K>
struct GenericLatentParams {
  CodecConst<N, K> cc;
  float light[kMaxGenericLights * K];
  int L, n_pal;
  const uint32_t* idx;
  const float* cosv;
  const float* pal;
  int64_t P;
  float *latent, *spectra, *xyz, *rgb;
  int* err;
};

template <int N, int K>
__global__ void __launch_bounds__(256) shade_latent_generic_kernel(const __grid_constant__ GenericLatentParams<N, K> p) {
  __shared__ __align__(16) float pal[kMaxPalette * K];
  block_load_table(pal, p.pal, p.n_pal * K);
  __syncthreads();
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t px = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; px < p.P; px += stride) {
    uint32_t id = p.idx[px];
    if (id >= static_cast<uint32_t>(p.n_pal)) {
      atomicOr(p.err, kErrIndexRange);
      id = 0;
    }
    float acc[K];
#pragma unroll
    for (int j = 0; j < K; ++j) acc[j] = 0.f;
    const float* c = p.cosv + px * p.L;
    for (int l = 0; l < p.L; ++l) {
      const float w = c[l];
#pragma unroll
      for (int j = 0; j < K; ++j) acc[j] = fmaf(w, p.light[l * K + j], acc[j]);
    }
    float z[K];
#pragma unroll
    for (int j = 0; j < K; ++j) z[j] = pal[id * K + j] * acc[j];
    if (p.latent)
#pragma unroll
      for (int j = 0; j < K; ++j) p.latent[px * K + j] = z[j];
    if (p.spectra)
#pragma unroll
      for (int i = 0; i < N; ++i) {
        float a = p.cc.D[i * K] * z[0];
#pragma unroll
        for (int j = 1; j < K; ++j) a = fmaf(p.cc.D[i * K + j], z[j], a);
        p.spectra[px * N + i] = a;
      }
    float xyz[3], rgb[3];
#pragma unroll
    for (int cc = 0; cc < 3; ++cc) {
      float a = p.cc.Mxyz[cc * K] * z[0];
#pragma unroll
      for (int j = 1; j < K; ++j) a = fmaf(p.cc.Mxyz[cc * K + j], z[j], a);
      xyz[cc] = a;
    }
    xyz_to_rgb(p.cc.Crgb, xyz, rgb);
#pragma unroll
    for (int cc = 0; cc < 3; ++cc) {
      if (p.xyz) p.xyz[px * 3 + cc] = xyz[cc];
      if (p.rgb) p.rgb[px * 3 + cc] = rgb[cc];
    }
  }
}

template <int N>
struct GenericSpectralParams {
  float light[kMaxGenericLights * N];
  float cmf[3 * N];
  float Crgb[9];
  int L, n_pal;
  const uint32_t* idx;
  const float* cosv;
  const float* pal;  // n_pal x N (read through L1: random rows)
  int64_t P;
  float *spectra, *xyz, *rgb;
  int* err;
};

template <int N>
__global__ void __launch_bounds__(256) shade_spectral_generic_kernel(const __grid_constant__ GenericSpectralParams<N> p) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t px = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; px < p.P; px += stride) {
    uint32_t id = p.idx[px];
    if (id >= static_cast<uint32_t>(p.n_pal)) {
      atomicOr(p.err, kErrIndexRange);
      id = 0;
    }
    const float* c = p.cosv + px * p.L;
    const float* R = p.pal + static_cast<int64_t>(id) * N;
    float xyz[3] = {0.f, 0.f, 0.f};
    for (int i = 0; i < N; ++i) {
      float illum = 0.f;
      for (int l = 0; l < p.L; ++l) illum = fmaf(c[l], p.light[l * N + i], illum);
      const float s = __ldg(R + i) * illum;
      if (p.spectra) p.spectra[px * N + i] = s;
      xyz[0] = fmaf(p.cmf[i], s, xyz[0]);
      xyz[1] = fmaf(p.cmf[N + i], s, xyz[1]);
      xyz[2] = fmaf(p.cmf[2 * N + i], s, xyz[2]);
    }
    float rgb[3];
    xyz_to_rgb(p.Crgb, xyz, rgb);
#pragma unroll
    for (int cc = 0; cc < 3; ++cc) {
      if (p.xyz) p.xyz[px * 3 + cc] = xyz[cc];
      if (p.rgb) p.rgb[px * 3 + cc] = rgb[cc];
    }
  }
}

static int generic_grid(hc_ctx ctx, int64_t P) {
  const int64_t g = (P + 255) / 256;
  return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(g, static_cast<int64_t>(ctx->sm_count) * 8)));
}

template <int N, int K>
int shade_latent_generic(hc_codec c, const float* pal, int n_pal, const float* light, int L, const uint32_t* idx,
                         const float* cosv, int64_t P, float* latent, float* spectra, float* xyz, float* rgb) {
  if (L > kMaxGenericLights) return set_error(HC_EUNSUPPORTED, "shade_latent: at most 64 lights");
  if (P <= 0) return HC_OK;
  GenericLatentParams<N, K> p;
  fill_codec_const<N, K>(c, &p.cc);
  for (int i = 0; i < L * K; ++i) p.light[i] = light[i];
  p.L = L;
  p.n_pal = n_pal;
  p.idx = idx;
  p.cosv = cosv;
  p.pal = pal;
  p.P = P;
  p.latent = latent;
  p.spectra = spectra;
  p.xyz = xyz;
  p.rgb = rgb;
  p.err = c->ctx->d_err;
  shade_latent_generic_kernel<N, K><<<generic_grid(c->ctx, P), 256, 0, c->ctx->stream>>>(p);
  HC_CHECK_LAUNCH(c->ctx, "shade_latent_generic_kernel");
  return HC_OK;
}

template <int N>
int shade_spectral_generic(hc_codec c, const float* pal, int n_pal, const float* light, int L, const uint32_t* idx,
                           const float* cosv, int64_t P, float* spectra, float* xyz, float* rgb) {
  if (L > kMaxGenericLights) return set_error(HC_EUNSUPPORTED, "shade_spectral: at most 64 lights");
  if (P <= 0) return HC_OK;
  GenericSpectralParams<N> p;
  for (int i = 0; i < L * N; ++i) p.light[i] = light[i];
  for (int i = 0; i < 3 * N; ++i) p.cmf[i] = c->cmf_dl[i];
  for (int i = 0; i < 9; ++i) p.Crgb[i] = c->Crgb[i];
  p.L = L;
  p.n_pal = n_pal;
  p.idx = idx;
  p.cosv = cosv;
  p.pal = pal;
  p.P = P;
  p.spectra = spectra;
  p.xyz = xyz;
  p.rgb = rgb;
  p.err = c->ctx->d_err;
  shade_spectral_generic_kernel<N><<<generic_grid(c->ctx, P), 256, 0, c->ctx->stream>>>(p);
  HC_CHECK_LAUNCH(c->ctx, "shade_spectral_generic_kernel");
  return HC_OK;
}

template <int N, int K, int L, int OUTS>
int shade_latent_nkl(hc_codec c, const float* pal, int n_pal, const float* light, const uint32_t* idx,
                     const float* cosv, int64_t P, float* latent, float* spectra, float* xyz,
                     float* rgb) {
  constexpr bool SPEC = (OUTS & kOutSpectra) != 0;
  constexpr bool C2 = L == 8 && OUTS == (kOutXyz | kOutRgb);
  constexpr int T = SPEC ? HC_SPEC_T : (C2 ? HC_C2_T : 256);
  constexpr int THREADS = C2 ? HC_C2_THREADS : T;
  constexpr int STAGES = SPEC ? HC_SPEC_STAGES : (C2 ? HC_C2_STAGES : 3);
  using Op = ShadeLatentOp<N, K, L, OUTS, T, THREADS, STAGES>;
  typename Op::Params p;
  fill_codec_const<N, K>(c, &p.cc);
  for (int i = 0; i < L * K; ++i) p.light[i] = light[i];
  p.idx = idx;
  p.cosv = cosv;
  p.pal_codes = pal;
  p.n_pal = n_pal;
  p.xyz = xyz;
  p.rgb = rgb;
  p.latent = latent;
  p.spectra = spectra;
  p.err = c->ctx->d_err;
  std::memset(&p.cos_map, 0, sizeof(p.cos_map));
  if constexpr (Op::kTensorStream >= 0) {
    if (P >= T && al16(cosv)) {
      const int rc = encode_rows_tmap_swizzle128(&p.cos_map, cosv, P, L, T);
      if (rc != HC_OK) return rc;
    }
  }
  return launch_tile_op<Op>(c->ctx, p, P);
}

template <int N, int K>
int shade_latent_nk(hc_codec c, const float* pal, int n_pal, const float* light, int L,
                    const uint32_t* idx, const float* cosv, int64_t P, float* latent, float* spectra,
                    float* xyz, float* rgb) {
  // Compiled output sets: the BASELINE ones (config 2: XYZ + sRGB; config 3: spectra +
  // sRGB) and the general set (all four; disabled outputs are simply not stored).
  const int want = (xyz ? kOutXyz : 0) | (rgb ? kOutRgb : 0) | (latent ? kOutLatent : 0) | (spectra ? kOutSpectra : 0);
  constexpr int kC2 = kOutXyz | kOutRgb, kC3 = kOutRgb | kOutSpectra, kAll = 15;
#define HC_SHADE_L(LL)                                                                                  \
  if (L == LL) {                                                                                       \
    if (want == kC2) return shade_latent_nkl<N, K, LL, kC2>(c, pal, n_pal, light, idx, cosv, P, latent, spectra, xyz, rgb); \
    if (want == kC3) return shade_latent_nkl<N, K, LL, kC3>(c, pal, n_pal, light, idx, cosv, P, latent, spectra, xyz, rgb); \
    return shade_latent_nkl<N, K, LL, kAll>(c, pal, n_pal, light, idx, cosv, P, latent, spectra, xyz, rgb);                 \
  }
  HC_SHADE_L(8)
  HC_SHADE_L(32)
#undef HC_SHADE_L
  return shade_latent_generic<N, K>(c, pal, n_pal, light, L, idx, cosv, P, latent, spectra, xyz, rgb);
}

int shade_latent_launch(hc_codec c, const float* pal, int n_pal, const float* light, int L,
                        const uint32_t* idx, const float* cosv, int64_t P, float* latent,
                        float* spectra, float* xyz, float* rgb) {
  HC_DISPATCH_NK(c->n, c->k, shade_latent_nk, c, pal, n_pal, light, L, idx, cosv, P, latent, spectra,
                 xyz, rgb);
}

template <int N, int L, bool SPEC>
int shade_spectral_nl(hc_codec c, const float* pal, int n_pal, const float* light, const uint32_t* idx,
                      const float* cosv, int64_t P, float* spectra, float* xyz, float* rgb) {
#ifndef HC_NAIVE_T
#define HC_NAIVE_T 256  // measured: 128 -> 256 threads per CTA +9.5 % (tools/sweep_naive.sh)
#endif
  constexpr int T = SPEC ? 64 : HC_NAIVE_T;
#ifndef HC_NAIVE_F2
#define HC_NAIVE_F2 1
#endif
  if constexpr (!SPEC && HC_NAIVE_F2 && L <= 8) {  // packed-FFMA2 variant (ShadeSpectralF2Op)
#ifndef HC_NAIVE_F2_T
#define HC_NAIVE_F2_T 1024  // one 84 KB palette copy per 32 warps: 256 / 512 / 1024 -> 14.0 / 20.0 / 24.0 Gpix/s
#endif
    using Op2 = ShadeSpectralF2Op<N, L, HC_NAIVE_F2_T, HC_NAIVE_F2_T, 2>;
    typename Op2::Params q;
    constexpr int H = Op2::NP / 2;
    auto pair = [](float lo, float hi) {
      const float f[2] = {lo, hi};
      unsigned long long v;
      std::memcpy(&v, f, 8);
      return v;
    };
    for (int l = 0; l < L; ++l)
      for (int h = 0; h < H; ++h)
        q.light2[l * H + h] = pair(light[l * N + 2 * h], 2 * h + 1 < N ? light[l * N + 2 * h + 1] : 0.f);
    for (int cc = 0; cc < 3; ++cc)
      for (int h = 0; h < H; ++h)
        q.cmf2[cc * H + h] = pair(c->cmf_dl[cc * N + 2 * h], 2 * h + 1 < N ? c->cmf_dl[cc * N + 2 * h + 1] : 0.f);
    for (int i = 0; i < 9; ++i) q.Crgb[i] = c->Crgb[i];
    q.idx = idx;
    q.cosv = cosv;
    q.pal_spectra = pal;
    q.n_pal = n_pal;
    q.xyz = xyz;
    q.rgb = rgb;
    q.err = c->ctx->d_err;
    return launch_tile_op<Op2>(c->ctx, q, P);
  }
  using Op = ShadeSpectralOp<N, L, SPEC, T, T, 2>;
  typename Op::Params p;
  for (int i = 0; i < L * N; ++i) p.light[i] = light[i];
  for (int i = 0; i < 3 * N; ++i) p.cmf[i] = c->cmf_dl[i];
  for (int i = 0; i < 9; ++i) p.Crgb[i] = c->Crgb[i];
  p.idx = idx;
  p.cosv = cosv;
  p.pal_spectra = pal;
  p.n_pal = n_pal;
  p.xyz = xyz;
  p.rgb = rgb;
  p.spectra = spectra;
  p.err = c->ctx->d_err;
  return launch_tile_op<Op>(c->ctx, p, P);
}

template <int N>
int shade_spectral_n(hc_codec c, const float* pal, int n_pal, const float* light, int L,
                     const uint32_t* idx, const float* cosv, int64_t P, float* spectra, float* xyz,
                     float* rgb) {
  const bool spec = spectra != nullptr;
  if (L == 8)
    return spec ? shade_spectral_nl<N, 8, true>(c, pal, n_pal, light, idx, cosv, P, spectra, xyz, rgb)
                : shade_spectral_nl<N, 8, false>(c, pal, n_pal, light, idx, cosv, P, spectra, xyz, rgb);
  if (L == 32)
    return spec ? shade_spectral_nl<N, 32, true>(c, pal, n_pal, light, idx, cosv, P, spectra, xyz, rgb)
                : shade_spectral_nl<N, 32, false>(c, pal, n_pal, light, idx, cosv, P, spectra, xyz, rgb);
  return shade_spectral_generic<N>(c, pal, n_pal, light, L, idx, cosv, P, spectra, xyz, rgb);
}

int shade_spectral_launch(hc_codec c, const float* pal, int n_pal, const float* light, int L,
                          const uint32_t* idx, const float* cosv, int64_t P, float* spectra,
                          float* xyz, float* rgb) {
  if (c->n == 81) return shade_spectral_n<81>(c, pal, n_pal, light, L, idx, cosv, P, spectra, xyz, rgb);
  if (c->n == 47) return shade_spectral_n<47>(c, pal, n_pal, light, L, idx, cosv, P, spectra, xyz, rgb);
  return set_error(HC_EUNSUPPORTED, "shade_spectral: n must be 47 or 81");
}

}  // namespace hcb
