// hadacodec-b200: G-buffer shading kernels — latent (fused k/3 passes +
// reassembly + decode/projection) and naive n-sample spectral.
// Reference: renderer.cpp:161-271 (compile_scene), :274-283 (slice_pass),
// :505-510 (NEE channel loop), :645-657 (reassembly), :661-719 (decode/project).
#include <cstring>

#include "hc_launch.cuh"
#include "hc_ops.cuh"

namespace hcb {

template <int N, int K, int L, int OUTS>
int shade_latent_nkl(hc_codec c, const float* pal, int n_pal, const float* light, const uint32_t* idx,
                     const float* cosv, int64_t P, float* latent, float* spectra, float* xyz,
                     float* rgb) {
  constexpr bool SPEC = (OUTS & kOutSpectra) != 0;
  constexpr int T = SPEC ? 64 : 256;
  constexpr int THREADS = T;
  constexpr int STAGES = SPEC ? 2 : 3;
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
  return set_error(HC_EUNSUPPORTED, "shade_latent: light count must be 8 or 32");
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
  constexpr int T = SPEC ? 64 : 128;
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
  return set_error(HC_EUNSUPPORTED, "shade_spectral: light count must be 8 or 32");
}

int shade_spectral_launch(hc_codec c, const float* pal, int n_pal, const float* light, int L,
                          const uint32_t* idx, const float* cosv, int64_t P, float* spectra,
                          float* xyz, float* rgb) {
  if (c->n == 81) return shade_spectral_n<81>(c, pal, n_pal, light, L, idx, cosv, P, spectra, xyz, rgb);
  if (c->n == 47) return shade_spectral_n<47>(c, pal, n_pal, light, L, idx, cosv, P, spectra, xyz, rgb);
  return set_error(HC_EUNSUPPORTED, "shade_spectral: n must be 47 or 81");
}

}  // namespace hcb
