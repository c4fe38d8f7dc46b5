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

// ---------------------------------------------------------------- naive, lanes over wavelengths
// The thread-per-pixel naive shade (ShadeSpectralOp) needs, per wavelength, the L light SPD
// values as shared-memory broadcasts (L / 4 LDS.128 per L FMAs): at L = 32 it ran at 12 % of its
// fp32-issue bound.  Here a warp shades one pixel at a time with the lanes over wavelengths:
// lane j owns lambda j, j + 32, j + 64 and keeps those wavelengths of all L light SPDs in
// registers (packed pairs for lambda j, j + 32 -> FFMA2), so the only per-pixel broadcast is
// the pixel's L cosines (L / 4 LDS.128 from a per-warp staging of 32 pixels' G-buffer rows).
// Per pixel: S(lambda) = R_idx(lambda) * sum_l c_l L_l(lambda) (renderer.cpp:187-190 at C = n,
// :505-510), the spectra row written coalesced, XYZ = dlambda * CMF . S as per-lane partials
// reduced across the warp (colorimetry.cpp:75-87), sRGB.  The light sum runs in 4 partial
// chains (l mod 4): fp32, re-associated against the reference's order (within 1e-6).
constexpr int kLanesThreads = 384;  // 12 warps, one CTA per SM (~140 registers per thread)

template <int N, int L>
struct NaiveLanesParams {
  float light[L * N];
  float cmf[3 * N];
  float Crgb[9];
  const uint32_t* idx;
  const float* cosv;
  const float* pal;
  int n_pal;
  int64_t P;
  float* spectra;
  float* xyz;
  float* rgb;
  int* err;
};

__device__ __forceinline__ uint64_t nl_pack(float lo, float hi) {
  uint64_t d;
  asm("mov.b64 %0, {%1, %2};" : "=l"(d) : "f"(lo), "f"(hi));
  return d;
}
__device__ __forceinline__ uint64_t nl_fma2(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ float2 nl_unpack(uint64_t v) {
  float2 f;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(f.x), "=f"(f.y) : "l"(v));
  return f;
}

template <int N, int L>
__global__ void __launch_bounds__(kLanesThreads, 1) naive_lanes_kernel(const __grid_constant__ NaiveLanesParams<N, L> p) {
  static_assert(N > 64 && N <= 96 && L % 16 == 0, "three wavelength slots per lane, L a multiple of 16");
  // per warp: 32 pixels' cosine rows (32 x L floats), then the XYZ partials [3][32 px][32 lanes]
  extern __shared__ __align__(16) float stage_dyn[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int l0 = lane, l1 = lane + 32, l2 = lane + 64;
  const bool has2 = l2 < N;
  uint64_t L01[L];  // (L_l(lambda j), L_l(lambda j + 32))
  float L2[L];      // L_l(lambda j + 64)
#pragma unroll
  for (int l = 0; l < L; ++l) {
    L01[l] = nl_pack(p.light[l * N + l0], p.light[l * N + l1]);
    L2[l] = has2 ? p.light[l * N + l2] : 0.f;
  }
  float cm[3][3];
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    cm[c][0] = p.cmf[c * N + l0];
    cm[c][1] = p.cmf[c * N + l1];
    cm[c][2] = has2 ? p.cmf[c * N + l2] : 0.f;
  }
  float* st = stage_dyn + wib * (32 * L + 3 * 32 * 32);
  float* red = st + 32 * L;
  const int64_t warp_id = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  const uint32_t npal = static_cast<uint32_t>(p.n_pal);
  bool bad = false;
  for (int64_t r0 = warp_id * 32; r0 < p.P; r0 += nwarps * 32) {
    const int cnt = p.P - r0 < 32 ? static_cast<int>(p.P - r0) : 32;
    // stage the 32 pixels' cosine rows (32 x L floats, contiguous in the G-buffer)
    __syncwarp();
    const float4* src = reinterpret_cast<const float4*>(p.cosv + r0 * L);
#pragma unroll
    for (int i = 0; i < L / 4; ++i) {
      const int q = i * 32 + lane;  // float4 index within the round
      const float4 v = q < cnt * (L / 4) ? ldg_stream(src + q) : make_float4(0.f, 0.f, 0.f, 0.f);
      reinterpret_cast<float4*>(st)[q] = v;
    }
    uint32_t my_id = lane < cnt ? __ldg(p.idx + r0 + lane) : 0u;
    if (my_id >= npal) {
      bad = true;
      my_id = 0;
    }
    __syncwarp();
    float my_x = 0.f, my_y = 0.f, my_z = 0.f;
    for (int q = 0; q < cnt; ++q) {
      const uint32_t id = __shfl_sync(0xffffffffu, my_id, q);
      const float4* row = reinterpret_cast<const float4*>(st + q * L);
      uint64_t a01[4] = {0ull, 0ull, 0ull, 0ull};
      float a2[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int l4 = 0; l4 < L / 4; ++l4) {
        const float4 c4 = row[l4];  // same address in every lane: broadcast
        const float cs[4] = {c4.x, c4.y, c4.z, c4.w};
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int l = 4 * l4 + u;
          a01[u] = nl_fma2(L01[l], nl_pack(cs[u], cs[u]), a01[u]);
          a2[u] = fmaf(L2[l], cs[u], a2[u]);
        }
      }
      const float2 s01a = nl_unpack(a01[0]), s01b = nl_unpack(a01[1]), s01c = nl_unpack(a01[2]),
                   s01d = nl_unpack(a01[3]);
      const float il0 = (s01a.x + s01b.x) + (s01c.x + s01d.x);
      const float il1 = (s01a.y + s01b.y) + (s01c.y + s01d.y);
      const float il2 = (a2[0] + a2[1]) + (a2[2] + a2[3]);
      const float* R = p.pal + static_cast<int64_t>(id) * N;
      const float s0 = __ldg(R + l0) * il0, s1 = __ldg(R + l1) * il1, s2 = has2 ? __ldg(R + l2) * il2 : 0.f;
      if (p.spectra) {
        float* o = p.spectra + (r0 + q) * N;
        __stcs(o + l0, s0);
        __stcs(o + l1, s1);
        if (has2) __stcs(o + l2, s2);
      }
      // this lane's XYZ partial of pixel q, column (lane + q) mod 32 (conflict-free both ways)
      const int col = (lane + q) & 31;
      red[(0 * 32 + q) * 32 + col] = fmaf(cm[0][2], s2, fmaf(cm[0][1], s1, cm[0][0] * s0));
      red[(1 * 32 + q) * 32 + col] = fmaf(cm[1][2], s2, fmaf(cm[1][1], s1, cm[1][0] * s0));
      red[(2 * 32 + q) * 32 + col] = fmaf(cm[2][2], s2, fmaf(cm[2][1], s1, cm[2][0] * s0));
    }
    __syncwarp();
    if (lane < cnt) {  // lane q adds the 32 lanes' partials of its pixel
      float xs[4] = {0.f, 0.f, 0.f, 0.f}, ys[4] = {0.f, 0.f, 0.f, 0.f}, zs[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        const int col = (i + lane) & 31;
        xs[i & 3] += red[(0 * 32 + lane) * 32 + col];
        ys[i & 3] += red[(1 * 32 + lane) * 32 + col];
        zs[i & 3] += red[(2 * 32 + lane) * 32 + col];
      }
      my_x = (xs[0] + xs[1]) + (xs[2] + xs[3]);
      my_y = (ys[0] + ys[1]) + (ys[2] + ys[3]);
      my_z = (zs[0] + zs[1]) + (zs[2] + zs[3]);
    }
    if (lane < cnt) {
      const float xyz[3] = {my_x, my_y, my_z};
      float rgb[3];
      xyz_to_rgb(p.Crgb, xyz, rgb);
      const int64_t px = r0 + lane;
      if (p.xyz)
#pragma unroll
        for (int c = 0; c < 3; ++c) p.xyz[px * 3 + c] = xyz[c];
      if (p.rgb)
#pragma unroll
        for (int c = 0; c < 3; ++c) p.rgb[px * 3 + c] = rgb[c];
    }
  }
  if (bad) atomicOr(p.err, kErrIndexRange);
}

template <int N, int L>
int naive_lanes_launch(hc_codec c, const float* pal, int n_pal, const float* light, const uint32_t* idx,
                       const float* cosv, int64_t P, float* spectra, float* xyz, float* rgb) {
  NaiveLanesParams<N, L> p;
  for (int i = 0; i < L * N; ++i) p.light[i] = light[i];
  for (int i = 0; i < 3 * N; ++i) p.cmf[i] = c->cmf_dl[i];
  for (int i = 0; i < 9; ++i) p.Crgb[i] = c->Crgb[i];
  p.idx = idx;
  p.cosv = cosv;
  p.pal = pal;
  p.n_pal = n_pal;
  p.P = P;
  p.spectra = spectra;
  p.xyz = xyz;
  p.rgb = rgb;
  p.err = c->ctx->d_err;
  const int64_t rounds = (P + 31) / 32;
  const int warps = kLanesThreads / 32;
  const int grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>((rounds + warps - 1) / warps, c->ctx->sm_count)));
  const int smem = kLanesThreads / 32 * (32 * L + 3 * 32 * 32) * 4;
  static std::atomic<uint64_t> configured{0};  // per device; the attribute call is idempotent
  if (!configured_here(configured)) {
    HC_CUDA_TRY(cudaFuncSetAttribute(naive_lanes_kernel<N, L>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    mark_configured_here(configured);
  }
  naive_lanes_kernel<N, L><<<grid, kLanesThreads, smem, c->ctx->stream>>>(p);
  HC_CHECK_LAUNCH(c->ctx, "naive_lanes_kernel");
  return HC_OK;
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
#ifndef HC_NAIVE_LANES
#define HC_NAIVE_LANES 1
#endif
  // L = 32 (config 3): lanes over wavelengths; needs 16-byte aligned cosine rows
  if constexpr (L % 16 == 0 && N > 64 && N <= 96) {
    if (HC_NAIVE_LANES && (reinterpret_cast<uintptr_t>(cosv) & 15u) == 0)
      return naive_lanes_launch<N, L>(c, pal, n_pal, light, idx, cosv, P, spectra, xyz, rgb);
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
