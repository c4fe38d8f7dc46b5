// hadacodec-b200: per-item compute bodies plugged into the tile pipeline.
//
// Each Op is thread-per-item: the item's row sits in shared memory (odd row
// strides n = 47 / 81 make the column walk bank-conflict free), the codec
// coefficients are kernel parameters (constant-bank FFMA operands), and the
// results are written to shared staging that the pipeline bulk-stores.
//
// Reference lines restated (fp32 arithmetic; parity within 1e-5 relative of
// the fp64 reference):
//   encode            codec.cpp:36-46
//   decode / image    codec.cpp:52-71, renderer.cpp:661-690
//   XYZ / sRGB        colorimetry.cpp:75-87, :103-105, renderer.cpp:692-719
//   latent shading    renderer.cpp:462-471, :505-510 (NEE), slice_pass :274-283,
//                     reassembly :645-657
//   naive shading     the same loops at C = n (renderer.cpp:187-190, :203-205)
//   loss residual     trainer.cpp:49-71
#pragma once

#include <cuda.h>

#include "hc_common.cuh"
#include "hc_tma.cuh"


namespace hcb {

enum : int {
  kErrNegativeCode = 1,  // decode of a negative code (codec.cpp:56-62) -> HC_EDOMAIN
  kErrIndexRange = 2,    // palette index >= palette size (renderer.cpp:166-181) -> HC_EINVAL
};

// ---------------------------------------------------------------- codec
enum CodecMode : int { kRoundtrip = 0, kEncode = 1, kDecode = 2, kProject = 3 };

template <int N, int K, int MODE, int T_, int THREADS_, int STAGES_>
struct CodecOp {
  static constexpr int T = T_, THREADS = THREADS_, STAGES = STAGES_;
  static constexpr int NIN = 1;
  __host__ __device__ static constexpr int in_bytes(int) { return (MODE == kDecode ? K : N) * 4; }
  // out streams: 0 codes, 1 spectra, 2 XYZ, 3 sRGB
  static constexpr int NOUT = MODE == kEncode ? 1 : (MODE == kProject ? 2 : (MODE == kDecode ? 3 : 4));
  //   roundtrip: codes, spectra, XYZ, sRGB | encode: codes | decode: spectra, XYZ, sRGB
  //   project: XYZ, sRGB
  __host__ __device__ static constexpr int out_bytes(int i) {
    return MODE == kRoundtrip ? (i == 0 ? K * 4 : (i == 1 ? N * 4 : 12))
         : MODE == kEncode    ? K * 4
         : MODE == kDecode    ? (i == 0 ? N * 4 : 12)
                              : 12;
  }
  static constexpr int EXTRA_SMEM = 0;
  static constexpr int kTensorStream = -1;
  static constexpr bool kWarpSpecialized = false;
  static constexpr bool kEvictFirstLoads = false;

  struct Params {
    CodecConst<N, K> cc;
    const float* in;
    float* out[4];
    int* err;
    int check_negative;
  };
  __host__ __device__ static const void* tensor_map(const Params&) { return nullptr; }
  struct State {};
  __device__ static void init_state(State&) {}
  __host__ __device__ static const void* in_ptr(const Params& p, int) { return p.in; }
  __host__ __device__ static void* out_ptr(const Params& p, int i) { return p.out[i]; }
  __device__ static void setup(const Params&, unsigned char*) {}
  __device__ static void finish(const Params&, State&, unsigned char*) {}

  __device__ static void compute(const Params& p, State&, const unsigned char* const* ins,
                                 unsigned char* const* outs, unsigned char*, int item, int64_t) {
    if constexpr (MODE == kProject) {
      const float* s = reinterpret_cast<const float*>(ins[0]) + item * N;
      float xyz[3] = {0.f, 0.f, 0.f};
#pragma unroll
      for (int i = 0; i < N; ++i) {
        const float v = s[i];
        xyz[0] = fmaf(p.cc.cmf[i], v, xyz[0]);
        xyz[1] = fmaf(p.cc.cmf[N + i], v, xyz[1]);
        xyz[2] = fmaf(p.cc.cmf[2 * N + i], v, xyz[2]);
      }
      float rgb[3];
      xyz_to_rgb(p.cc.Crgb, xyz, rgb);
      float* ox = reinterpret_cast<float*>(outs[0]) + item * 3;
      float* orgb = reinterpret_cast<float*>(outs[1]) + item * 3;
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        ox[c] = xyz[c];
        orgb[c] = rgb[c];
      }
      return;
    }
    float z[K];
    if constexpr (MODE == kDecode) {
      const float* zi = reinterpret_cast<const float*>(ins[0]) + item * K;
      bool neg = false;
#pragma unroll
      for (int j = 0; j < K; ++j) {
        z[j] = zi[j];
        neg |= !(z[j] >= 0.f);
      }
      if (neg && p.check_negative) atomicOr(p.err, kErrNegativeCode);
    } else {
      const float* s = reinterpret_cast<const float*>(ins[0]) + item * N;
#pragma unroll
      for (int j = 0; j < K; ++j) z[j] = 0.f;
#pragma unroll
      for (int i = 0; i < N; ++i) {
        const float v = s[i];
#pragma unroll
        for (int j = 0; j < K; ++j) z[j] = fmaf(p.cc.E[j * N + i], v, z[j]);
      }
      float* oz = reinterpret_cast<float*>(outs[0]) + item * K;
#pragma unroll
      for (int j = 0; j < K; ++j) oz[j] = z[j];
      if constexpr (MODE == kEncode) return;
    }
    constexpr int kSpec = MODE == kRoundtrip ? 1 : 0;
    constexpr int kXyz = kSpec + 1, kRgb = kSpec + 2;
    if (p.out[MODE == kRoundtrip ? 1 : 0] != nullptr) {
      float* os = reinterpret_cast<float*>(outs[kSpec]) + item * N;
#pragma unroll
      for (int i = 0; i < N; ++i) {
        float acc = p.cc.D[i * K] * z[0];
#pragma unroll
        for (int j = 1; j < K; ++j) acc = fmaf(p.cc.D[i * K + j], z[j], acc);
        os[i] = acc;
      }
    }
    float xyz[3], rgb[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      float acc = p.cc.Mxyz[c * K] * z[0];
#pragma unroll
      for (int j = 1; j < K; ++j) acc = fmaf(p.cc.Mxyz[c * K + j], z[j], acc);
      xyz[c] = acc;
    }
    xyz_to_rgb(p.cc.Crgb, xyz, rgb);
    float* ox = reinterpret_cast<float*>(outs[kXyz]) + item * 3;
    float* orgb = reinterpret_cast<float*>(outs[kRgb]) + item * 3;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      ox[c] = xyz[c];
      orgb[c] = rgb[c];
    }
  }
};

// ---------------------------------------------------------------- latent shading
// G-buffer item: idx (u32, palette entry) + L fp32 Lambert weights c_{p,l}.
// z = zR[idx] (.) sum_l c_l zL_l  (renderer.cpp:505-510 with thr = 1,
// w = c_{p,l}), all k channels at once: the k/3 RGB passes of slice_pass are
// channel-disjoint, so writing channel 3b+c of the HWC latent image IS the
// reassembly of renderer.cpp:645-657.  Then XYZ = Mxyz z, sRGB, and optionally
// the full decoded spectrum D z.
constexpr int kMaxPalette = 256;

// Output streams of a latent shade, selected at compile time (unused outputs get
// no staging shared memory): bit 0 XYZ, bit 1 linear sRGB, bit 2 latent, bit 3 spectra.
enum : int { kOutXyz = 1, kOutRgb = 2, kOutLatent = 4, kOutSpectra = 8 };

__host__ __device__ constexpr int popcount4(int m) { return (m & 1) + ((m >> 1) & 1) + ((m >> 2) & 1) + ((m >> 3) & 1); }
// Kind of the i-th enabled output of mask m.
__host__ __device__ constexpr int out_kind(int m, int i) {
  for (int b = 0; b < 4; ++b)
    if (m & (1 << b)) {
      if (i == 0) return 1 << b;
      --i;
    }
  return 0;
}
// Stream slot of output `kind` in mask m.
__host__ __device__ constexpr int out_slot(int m, int kind) { return popcount4(m & (kind - 1)); }

template <int N, int K, int L, int OUTS, int T_, int THREADS_, int STAGES_>
struct ShadeLatentOp {
  static constexpr int T = T_, THREADS = THREADS_, STAGES = STAGES_;
  static constexpr int NIN = 2;
  __host__ __device__ static constexpr int in_bytes(int i) { return i == 0 ? 4 : L * 4; }
  static constexpr int NOUT = popcount4(OUTS);
  __host__ __device__ static constexpr int out_bytes(int i) {
    return out_kind(OUTS, i) == kOutLatent ? K * 4 : (out_kind(OUTS, i) == kOutSpectra ? N * 4 : 12);
  }
  static constexpr int EXTRA_SMEM = kMaxPalette * K * 4;
  static constexpr int kTensorStream = (L * 4 == 128) ? 1 : -1;  // 128-byte cos rows: swizzled 2-D TMA
  // Pipeline choice (measured, profiles/README.md): the spectra-writing variant runs the
  // warp-specialised pipeline (78 -> 85 % HBM); the small-output variant streams its
  // inputs with an L2 evict-first policy (80 -> 81 %).
#ifdef HC_C2_WS  // tuning only: force the warp-specialised pipeline for every output set
  static constexpr bool kWarpSpecialized = true;
#else
  static constexpr bool kWarpSpecialized = (OUTS & kOutSpectra) != 0;
#endif
  static constexpr bool kEvictFirstLoads = (OUTS & kOutSpectra) == 0;

  struct Params {
    CUtensorMap cos_map;  // 2-D map of cos [P][L] with the 128-byte swizzle (used when L == 32)
    CodecConst<N, K> cc;
    float light[L * K];
    const uint32_t* idx;
    const float* cosv;
    const float* pal_codes;
    int n_pal;
    float* xyz;
    float* rgb;
    float* latent;
    float* spectra;
    int* err;
  };
  __host__ __device__ static const void* tensor_map(const Params& p) { return &p.cos_map; }
  struct State {};
  __device__ static void init_state(State&) {}
  __host__ __device__ static const void* in_ptr(const Params& p, int i) {
    return i == 0 ? static_cast<const void*>(p.idx) : static_cast<const void*>(p.cosv);
  }
  __host__ __device__ static void* out_ptr(const Params& p, int i) {
    const int k = out_kind(OUTS, i);
    return k == kOutXyz ? p.xyz : (k == kOutRgb ? p.rgb : (k == kOutLatent ? p.latent : p.spectra));
  }
  __device__ static void setup(const Params& p, unsigned char* extra) {
#ifdef HC_PROBE_NO_PAL_COPY  // timing probe only: palette left uninitialised (wrong results)
    return;
#endif
    block_load_table(reinterpret_cast<float*>(extra), p.pal_codes, p.n_pal * K);
  }
  __device__ static void finish(const Params&, State&, unsigned char*) {}

  __device__ static void compute(const Params& p, State&, const unsigned char* const* ins,
                                 unsigned char* const* outs, unsigned char* extra, int item, int64_t) {
    uint32_t id = reinterpret_cast<const uint32_t*>(ins[0])[item];
    if (id >= static_cast<uint32_t>(p.n_pal)) {
      atomicOr(p.err, kErrIndexRange);
      id = 0;
    }
    const unsigned char* crow = ins[1] + item * (L * 4);
    float acc[K];
#pragma unroll
    for (int j = 0; j < K; ++j) acc[j] = 0.f;
#pragma unroll
    for (int l4 = 0; l4 < L; l4 += 4) {
      // swizzled rows (kTensorStream): 16-byte chunk q of row r sits at chunk q ^ (r & 7)
      const int q = kTensorStream >= 0 ? ((l4 >> 2) ^ (item & 7)) : (l4 >> 2);
      const float4 w4 = *reinterpret_cast<const float4*>(crow + q * 16);
      const float w[4] = {w4.x, w4.y, w4.z, w4.w};
#pragma unroll
      for (int e = 0; e < 4; ++e)
#pragma unroll
        for (int j = 0; j < K; ++j) acc[j] = fmaf(w[e], p.light[(l4 + e) * K + j], acc[j]);
    }
    const float* zr = reinterpret_cast<const float*>(extra) + id * K;
    float z[K];
#pragma unroll
    for (int j = 0; j < K; ++j) z[j] = zr[j] * acc[j];
    if constexpr ((OUTS & kOutLatent) != 0) {
      float* ol = reinterpret_cast<float*>(outs[out_slot(OUTS, kOutLatent)]) + item * K;
#pragma unroll
      for (int j = 0; j < K; ++j) ol[j] = z[j];
    }
    if constexpr ((OUTS & kOutSpectra) != 0) {
      float* os = reinterpret_cast<float*>(outs[out_slot(OUTS, kOutSpectra)]) + item * N;
#pragma unroll
      for (int i = 0; i < N; ++i) {
        float a = p.cc.D[i * K] * z[0];
#pragma unroll
        for (int j = 1; j < K; ++j) a = fmaf(p.cc.D[i * K + j], z[j], a);
        os[i] = a;
      }
    }
    if constexpr ((OUTS & (kOutXyz | kOutRgb)) != 0) {
      float xyz[3], rgb[3];
#pragma unroll
      for (int cc = 0; cc < 3; ++cc) {
        float a = p.cc.Mxyz[cc * K] * z[0];
#pragma unroll
        for (int j = 1; j < K; ++j) a = fmaf(p.cc.Mxyz[cc * K + j], z[j], a);
        xyz[cc] = a;
      }
      if constexpr ((OUTS & kOutXyz) != 0) {
        float* ox = reinterpret_cast<float*>(outs[out_slot(OUTS, kOutXyz)]) + item * 3;
#pragma unroll
        for (int cc = 0; cc < 3; ++cc) ox[cc] = xyz[cc];
      }
      if constexpr ((OUTS & kOutRgb) != 0) {
        xyz_to_rgb(p.cc.Crgb, xyz, rgb);
        float* orgb = reinterpret_cast<float*>(outs[out_slot(OUTS, kOutRgb)]) + item * 3;
#pragma unroll
        for (int cc = 0; cc < 3; ++cc) orgb[cc] = rgb[cc];
      }
    }
  }
};

// ---------------------------------------------------------------- naive spectral shading
// S(lambda) = R_idx(lambda) * sum_l c_l L_l(lambda) per wavelength (the same
// NEE loop at C = n, renderer.cpp:187-190 / :505-510), XYZ = dlambda * CMF . S
// (colorimetry.cpp:75-87), sRGB.  Palette spectra live in shared memory; light
// SPDs and CMF rows are constant-bank operands.
template <int N, int L, bool SPEC, int T_, int THREADS_, int STAGES_>
struct ShadeSpectralOp {
  static constexpr int T = T_, THREADS = THREADS_, STAGES = STAGES_;
  static constexpr int NIN = 2;
  __host__ __device__ static constexpr int in_bytes(int i) { return i == 0 ? 4 : L * 4; }
  static constexpr int NOUT = SPEC ? 3 : 2;  // XYZ, sRGB, [spectra]
  __host__ __device__ static constexpr int out_bytes(int i) { return i < 2 ? 12 : N * 4; }
#ifndef HC_NAIVE_PALG_SPEC
#define HC_NAIVE_PALG_SPEC 1
#endif
#ifndef HC_NAIVE_PALG
#define HC_NAIVE_PALG 0
#endif
  // kPalG: palette rows read through L1 (__ldg) instead of an 83 KB shared-memory copy per
  // CTA, and the light SPDs as shared-memory rows [lambda][light] read by broadcast LDS.128
  // instead of L x n constant-bank operands (10 KB at L = 32, beyond the constant cache).
  // The spectra-writing variant ran 1 CTA (2 warps) per SM with the smem palette.
  static constexpr bool kPalG = SPEC ? HC_NAIVE_PALG_SPEC : HC_NAIVE_PALG;
#ifndef HC_NAIVE_LSMEM
#define HC_NAIVE_LSMEM 0
#endif
  static constexpr bool kLightSmem = kPalG || HC_NAIVE_LSMEM;  // light rows in smem (else constant bank)
  static constexpr int kPalOff = kLightSmem ? N * L * 4 : 0;   // palette copy after the light rows
  static constexpr int EXTRA_SMEM = kPalOff + (kPalG ? 0 : kMaxPalette * N * 4);
  static constexpr int kTensorStream = -1;
  static constexpr bool kWarpSpecialized = kPalG && SPEC;
  static constexpr bool kEvictFirstLoads = false;

  struct Params {
    float light[L * N];
    float cmf[3 * N];
    float Crgb[9];
    const uint32_t* idx;
    const float* cosv;
    const float* pal_spectra;
    int n_pal;
    float* xyz;
    float* rgb;
    float* spectra;
    int* err;
  };
  __host__ __device__ static const void* tensor_map(const Params&) { return nullptr; }
  struct State {};
  __device__ static void init_state(State&) {}
  __host__ __device__ static const void* in_ptr(const Params& p, int i) {
    return i == 0 ? static_cast<const void*>(p.idx) : static_cast<const void*>(p.cosv);
  }
  __host__ __device__ static void* out_ptr(const Params& p, int i) {
    return i == 0 ? p.xyz : (i == 1 ? p.rgb : p.spectra);
  }
  __device__ static void setup(const Params& p, unsigned char* extra) {
    if constexpr (kLightSmem) {
      float* ls = reinterpret_cast<float*>(extra);  // [lambda][light]
      for (int x = threadIdx.x; x < N * L; x += blockDim.x) {
        const int i = x / L, l = x - i * L;
        ls[x] = p.light[l * N + i];
      }
    }
    if constexpr (!kPalG) block_load_table(reinterpret_cast<float*>(extra + kPalOff), p.pal_spectra, p.n_pal * N);
  }
  __device__ static void finish(const Params&, State&, unsigned char*) {}

  __device__ static void compute(const Params& p, State&, const unsigned char* const* ins,
                                 unsigned char* const* outs, unsigned char* extra, int item, int64_t) {
    uint32_t id = reinterpret_cast<const uint32_t*>(ins[0])[item];
    if (id >= static_cast<uint32_t>(p.n_pal)) {
      atomicOr(p.err, kErrIndexRange);
      id = 0;
    }
    const float* c = reinterpret_cast<const float*>(ins[1]) + item * L;
    float w[L];
#pragma unroll
    for (int l4 = 0; l4 < L; l4 += 4) {
      const float4 w4 = *reinterpret_cast<const float4*>(c + l4);
      w[l4] = w4.x;
      w[l4 + 1] = w4.y;
      w[l4 + 2] = w4.z;
      w[l4 + 3] = w4.w;
    }
    const float* R = kPalG ? p.pal_spectra + id * N : reinterpret_cast<const float*>(extra + kPalOff) + id * N;
    float* os = SPEC ? reinterpret_cast<float*>(outs[2]) + item * N : nullptr;
    float xyz[3] = {0.f, 0.f, 0.f};
#pragma unroll
    for (int i = 0; i < N; ++i) {
      float illum;
      if constexpr (kLightSmem) {
        const float4* lr = reinterpret_cast<const float4*>(extra) + i * (L / 4);  // broadcast row
        float lv[L];
#pragma unroll
        for (int c4 = 0; c4 < L / 4; ++c4) {
          const float4 v = lr[c4];
          lv[4 * c4] = v.x;
          lv[4 * c4 + 1] = v.y;
          lv[4 * c4 + 2] = v.z;
          lv[4 * c4 + 3] = v.w;
        }
        illum = w[0] * lv[0];
#pragma unroll
        for (int l = 1; l < L; ++l) illum = fmaf(w[l], lv[l], illum);
      } else {
        illum = w[0] * p.light[i];
#pragma unroll
        for (int l = 1; l < L; ++l) illum = fmaf(w[l], p.light[l * N + i], illum);
      }
      const float Ri = kPalG ? __ldg(R + i) : R[i];
      const float s = Ri * illum;
      if constexpr (SPEC) os[i] = s;
      xyz[0] = fmaf(p.cmf[i], s, xyz[0]);
      xyz[1] = fmaf(p.cmf[N + i], s, xyz[1]);
      xyz[2] = fmaf(p.cmf[2 * N + i], s, xyz[2]);
    }
    float rgb[3];
    xyz_to_rgb(p.Crgb, xyz, rgb);
    float* ox = reinterpret_cast<float*>(outs[0]) + item * 3;
    float* orgb = reinterpret_cast<float*>(outs[1]) + item * 3;
#pragma unroll
    for (int cc = 0; cc < 3; ++cc) {
      ox[cc] = xyz[cc];
      orgb[cc] = rgb[cc];
    }
  }
};

// ---------------------------------------------------------------- naive shading, packed
// The naive n-sample shade of configs 2 (no spectra written), restated for the fp32x2
// pipe: wavelengths are processed in pairs with packed FFMA2 (fma.rn.f32x2), so the
// light sum (L FMAs), the reflectance product and the 3 CMF accumulations of two
// wavelengths issue as L + 1 + 3 instructions instead of 2 (L + 4): the kernel was
// issue-bound (ShadeSpectralOp, ~13 instructions per wavelength).  The arithmetic per
// wavelength is unchanged (the same products and sums, fp32); XYZ sums the even- and
// odd-wavelength partials at the end.  Palette rows are padded to an even length in
// shared memory and read as float2; light SPD and CMF pairs are constant-bank operands.
__device__ __forceinline__ uint64_t f2pack(float lo, float hi) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ uint64_t f2fma(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ float2 f2unpack(uint64_t v) {
  float2 r;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(r.x), "=f"(r.y) : "l"(v));
  return r;
}

template <int N, int L, int T_, int THREADS_, int STAGES_>
struct ShadeSpectralF2Op {
  static constexpr int T = T_, THREADS = THREADS_, STAGES = STAGES_;
  static constexpr int NP = (N + 1) / 2 * 2;  // padded row length
  static constexpr int NIN = 2;
  __host__ __device__ static constexpr int in_bytes(int i) { return i == 0 ? 4 : L * 4; }
  static constexpr int NOUT = 2;  // XYZ, sRGB
  __host__ __device__ static constexpr int out_bytes(int) { return 12; }
  static constexpr int EXTRA_SMEM = kMaxPalette * NP * 4;
  static constexpr int kTensorStream = -1;
  static constexpr bool kWarpSpecialized = false;
  static constexpr bool kEvictFirstLoads = false;

  struct Params {
    unsigned long long light2[L * NP / 2];  // (L_l(2h), L_l(2h + 1)) pairs, [l][h]
    unsigned long long cmf2[3 * NP / 2];    // dlambda * CMF pairs, [c][h]
    float Crgb[9];
    const uint32_t* idx;
    const float* cosv;
    const float* pal_spectra;
    int n_pal;
    float* xyz;
    float* rgb;
    int* err;
  };
  __host__ __device__ static const void* tensor_map(const Params&) { return nullptr; }
  struct State {};
  __device__ static void init_state(State&) {}
  __host__ __device__ static const void* in_ptr(const Params& p, int i) {
    return i == 0 ? static_cast<const void*>(p.idx) : static_cast<const void*>(p.cosv);
  }
  __host__ __device__ static void* out_ptr(const Params& p, int i) { return i == 0 ? p.xyz : p.rgb; }
  __device__ static void setup(const Params& p, unsigned char* extra) {
    float* pal = reinterpret_cast<float*>(extra);
    for (int x = threadIdx.x; x < p.n_pal * NP; x += blockDim.x) {
      const int r = x / NP, i = x - r * NP;
      pal[x] = i < N ? __ldg(p.pal_spectra + r * N + i) : 0.f;
    }
  }
  __device__ static void finish(const Params&, State&, unsigned char*) {}

  __device__ static void compute(const Params& p, State&, const unsigned char* const* ins,
                                 unsigned char* const* outs, unsigned char* extra, int item, int64_t) {
    uint32_t id = reinterpret_cast<const uint32_t*>(ins[0])[item];
    if (id >= static_cast<uint32_t>(p.n_pal)) {
      atomicOr(p.err, kErrIndexRange);
      id = 0;
    }
    const float* c = reinterpret_cast<const float*>(ins[1]) + item * L;
    uint64_t w2[L];
#pragma unroll
    for (int l4 = 0; l4 < L; l4 += 4) {
      const float4 w4 = *reinterpret_cast<const float4*>(c + l4);
      w2[l4] = f2pack(w4.x, w4.x);
      w2[l4 + 1] = f2pack(w4.y, w4.y);
      w2[l4 + 2] = f2pack(w4.z, w4.z);
      w2[l4 + 3] = f2pack(w4.w, w4.w);
    }
    const float2* R = reinterpret_cast<const float2*>(extra) + id * (NP / 2);
    uint64_t acc[3] = {0ull, 0ull, 0ull};
#pragma unroll
    for (int h = 0; h < NP / 2; ++h) {
      uint64_t il = f2fma(w2[0], p.light2[h], 0ull);
#pragma unroll
      for (int l = 1; l < L; ++l) il = f2fma(w2[l], p.light2[l * (NP / 2) + h], il);
      const float2 r = R[h];
      const uint64_t s = f2fma(f2pack(r.x, r.y), il, 0ull);
#pragma unroll
      for (int cc = 0; cc < 3; ++cc) acc[cc] = f2fma(p.cmf2[cc * (NP / 2) + h], s, acc[cc]);
    }
    float xyz[3], rgb[3];
#pragma unroll
    for (int cc = 0; cc < 3; ++cc) {
      const float2 a = f2unpack(acc[cc]);
      xyz[cc] = a.x + a.y;
    }
    xyz_to_rgb(p.Crgb, xyz, rgb);
    float* ox = reinterpret_cast<float*>(outs[0]) + item * 3;
    float* orgb = reinterpret_cast<float*>(outs[1]) + item * 3;
#pragma unroll
    for (int cc = 0; cc < 3; ++cc) {
      ox[cc] = xyz[cc];
      orgb[cc] = rgb[cc];
    }
  }
};

// ---------------------------------------------------------------- loss
// sum over pairs and lambda of (D (E a (.) E b) - a (.) b)^2, computed the way the
// reference computes it (forward_pair + mse_n, trainer.cpp:49-71): the residual
// r_l = sum_j D_lj zp_j - a_l b_l is formed per wavelength and squared, in fp64 (the
// reference's precision).  The loss measures how close the codec is to
// multiplicative, so r_l is routinely 1e-8 of a_l b_l; an fp32 residual (or the
// expanded zp^T G zp - 2 zp.D^T(ab) + |ab|^2 form of round 1) is then rounding noise.
//
// ~1,650 fp64 operations per 648-byte pair put the fp64 pipe next to HBM, so the layout
// is about feeding it:
//  * G warp groups share each pair (kLanesPerItem = G; G = 3 for n = 81): group h
//    (threads [h*T, (h+1)*T)) takes wavelengths [h*R, (h+1)*R) of every pair of the tile,
//    which gives 3x the warps per SM at the same TMA ring;
//  * a warp is always at one wavelength, so E comes from the constant bank at a uniform
//    index and D from a shared-memory table as same-address double2 broadcasts (both in the
//    constant bank thrash its cache: 73 % hits), and a lane's a_l / b_l reads (row stride
//    81 words, odd) are bank-conflict free;
//  * both passes are software pipelined: the floats of the next batch of wavelengths are
//    loaded (LDS) and converted (F2F, variable latency) while the current batch's DFMAs
//    issue;
//  * pass 1 accumulates the group's partial codes, the groups exchange them through
//    shared memory (one barrier; every group adds the partials in group order, so all hold
//    the same zp), pass 2 decodes zp at the group's wavelengths starting from -a_l b_l (an
//    exact fp64 product of two floats) and accumulates r_l^2.
// Pairs accumulate in fp64 per thread, then per CTA into partials[].
#ifndef HC_LOSS_B1
#define HC_LOSS_B1 27  // pass-1 batch (wavelengths); must divide N / G, else 1
#endif
#ifndef HC_LOSS_B2
#define HC_LOSS_B2 27  // pass-2 batch
#endif
#ifndef HC_LOSS_VLOAD
#define HC_LOSS_VLOAD 0
#endif
#ifndef HC_LOSS_SPLIT  // pass 2: (D zp)_l as two interleaved 3-term chains
#define HC_LOSS_SPLIT 0
#endif
#ifndef HC_LOSS_ABREG  // a_l b_l formed in pass 1 and kept in registers (pass 2 reads no a / b)
#define HC_LOSS_ABREG 0
#endif
#ifndef HC_LOSS_WS  // warp-specialised pipeline; the code exchange syncs only the G warps of a 32-pair slice
#define HC_LOSS_WS 0
#endif
#ifndef HC_LOSS_CE2  // both passes per warp group with E / D from the constant bank, a_l b_l in registers
#define HC_LOSS_CE2 0
#endif
#ifndef HC_LOSS_CE  // pass 1 specialised per warp group: E as compile-time constant-bank operands
#define HC_LOSS_CE 0
#endif
// Pass 2 on the fp64 tensor-core path (mma.sync m8n8k4), see LossOp::pass2_dmma.  Measured option,
// off: 36.7-37.2 % of HBM against 53 % for the DFMA form (parity tests green either way) -- DMMA and
// DFMA share one pipe and a mix of the two runs at ~60 % of either alone (profiles/r02/dmma_probe.txt),
// and pass 1 stays DFMA (as MMAs its 6-of-8 code padding costs more than its 82 % DFMA rate).
#ifndef HC_LOSS_DMMA
#define HC_LOSS_DMMA 0
#endif

// C (8 x 8, fp64) += A (8 x 4, row) . B (4 x 8, col).  Fragments: A[i = lane / 4][k = lane % 4],
// B[k = lane % 4][j = lane / 4], C[i = lane / 4][j = 2 (lane % 4) + {0, 1}] (tools/f2f_dfma_probe.cu
// verifies the layout).  Each product-sum is an IEEE fp64 FMA chain over k.
__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

template <int N, int K, int T_, int THREADS_, int STAGES_>
struct LossOp {
  static constexpr int T = T_, THREADS = THREADS_, STAGES = STAGES_;
  static constexpr int G = N % 3 == 0 ? 3 : 1;  // warp groups per pair
  static constexpr int R = N / G;               // wavelengths per group
  static constexpr int B1 = R % HC_LOSS_B1 == 0 ? HC_LOSS_B1 : 1;
  static constexpr int B2 = R % HC_LOSS_B2 == 0 ? HC_LOSS_B2 : 1;
  static constexpr int kLanesPerItem = G;
  static_assert(THREADS == G * T && T % 32 == 0, "G whole warp groups per tile");
  static constexpr int NIN = 2;
  __host__ __device__ static constexpr int in_bytes(int) { return N * 4; }
  static constexpr int NOUT = 0;
  __host__ __device__ static constexpr int out_bytes(int) { return 0; }
  static constexpr int KP = (K + 1) / 2 * 2;
  // Pass 2 as fp64 MMAs (3 warp groups, whole warps of 32 pairs).
  static constexpr bool kDmma = HC_LOSS_DMMA && !HC_LOSS_WS && !HC_LOSS_CE2 && G == 3 && T % 32 == 0;
  // Row stride of the exchange buffer: + 4 doubles so the fragment reads (8 pairs x 4 codes per
  // warp) spread over all banks.
  static constexpr int TS = kDmma ? T + 4 : T;
  // [group][2K][TS] fp64 partial codes (item fastest: conflict-free 64-bit accesses)
  static constexpr int kXchg = G > 1 ? G * 2 * K * TS * 8 : 0;
  static constexpr int kTabD = N * KP * 8;  // D rows [l][KP], fp64
  static constexpr int EXTRA_SMEM = 32 * 8 + kXchg + kTabD;
  static constexpr int kTensorStream = -1;
  static constexpr bool kWarpSpecialized = HC_LOSS_WS;
  static constexpr bool kEvictFirstLoads = false;

  struct Params {
    double E[K * N];  // encoder, row-major k x n, fp64 (exact widening of the fp32 weights)
    double D[N * K];  // decoder, row-major n x k
    const float* a;
    const float* b;
    double* partials;  // one per CTA
    int partial_offset;
    int64_t pairs;  // pairs at or past this index (tile_generic's ragged tile) are discarded
  };
  __host__ __device__ static const void* tensor_map(const Params&) { return nullptr; }
  struct State {
    double acc;
  };
  __device__ static void init_state(State& s) { s.acc = 0.0; }
  __host__ __device__ static const void* in_ptr(const Params& p, int i) {
    return i == 0 ? static_cast<const void*>(p.a) : static_cast<const void*>(p.b);
  }
  __host__ __device__ static void* out_ptr(const Params&, int) { return nullptr; }
  __device__ static void setup(const Params& p, unsigned char* extra) {
    double* td = reinterpret_cast<double*>(extra + 32 * 8 + kXchg);
    for (int x = threadIdx.x; x < N * KP; x += blockDim.x) {
      const int l = x / KP, c = x % KP;
      td[x] = c < K ? p.D[l * K + c] : 0.0;
    }
  }

  // Pass 1 of warp group GRP with every E offset a compile-time constant, so each DFMA takes
  // its E value straight from the constant bank (c[0x0][imm] operand) instead of through a
  // uniform-register load (LDCU) on the dependency chain; all R floats of a and b are loaded
  // up front.
  template <int GRP>
  __device__ static void pass1_ce(const Params& p, const float* a, const float* b, double za[K], double zb[K]) {
    float fa[R], fb[R];
#pragma unroll
    for (int i = 0; i < R; ++i) {
      fa[i] = a[i];
      fb[i] = b[i];
    }
#pragma unroll
    for (int i = 0; i < R; ++i) {
      const double va = static_cast<double>(fa[i]), vb = static_cast<double>(fb[i]);
#pragma unroll
      for (int j = 0; j < K; ++j) {
        const double e = p.E[j * N + GRP * R + i];
        za[j] = fma(e, va, za[j]);
        zb[j] = fma(e, vb, zb[j]);
      }
    }
  }

  // HC_LOSS_CE2: pass 1 also forms a_l b_l (exact) into registers; pass 2 is then pure DFMA with
  // D at compile-time constant-bank offsets, j outer so the R residual chains run side by side.
  template <int GRP>
  __device__ static void pass1_ce2(const Params& p, const float* a, const float* b, double za[K], double zb[K],
                                   double ab[R]) {
    float fa[R], fb[R];
#pragma unroll
    for (int i = 0; i < R; ++i) {
      fa[i] = a[i];
      fb[i] = b[i];
    }
#pragma unroll
    for (int i = 0; i < R; ++i) {
      const double va = static_cast<double>(fa[i]), vb = static_cast<double>(fb[i]);
      ab[i] = va * vb;
#pragma unroll
      for (int j = 0; j < K; ++j) {
        const double e = p.E[j * N + GRP * R + i];
        za[j] = fma(e, va, za[j]);
        zb[j] = fma(e, vb, zb[j]);
      }
    }
  }
  template <int GRP>
  __device__ static double pass2_ce2(const Params& p, const double zp[K], const double ab[R]) {
    double r[R];
#pragma unroll
    for (int i = 0; i < R; ++i) r[i] = -ab[i];
#pragma unroll
    for (int j = 0; j < K; ++j)
#pragma unroll
      for (int i = 0; i < R; ++i) r[i] = fma(p.D[(GRP * R + i) * K + j], zp[j], r[i]);
    double acc = 0.0;
#pragma unroll
    for (int i = 0; i < R; ++i) acc = fma(r[i], r[i], acc);
    return acc;
  }

  // Pass 2 on the fp64 tensor-core path.  The DFMA form needs one D value from shared memory or
  // the constant bank per DFMA and ran at 34 % of the fp64 peak (profiles/r02/loss_mix_probe.txt);
  // as MMAs the D rows are register fragments and one instruction does 8 pairs x 8 wavelengths
  // x 4 codes.  The groups' partial codes go through the exchange buffer as before; each lane
  // then reads the summed codes of the pairs / code slots of its A fragments
  // (zp[pair 8m + lane / 4][code 4s + lane % 4]) and forms the products.  The wavelengths are
  // re-split over the warp groups in 8-wide column tiles (81 -> 4 + 4 + 3 tiles), column
  // 2c + e of a tile standing for wavelength c + 4e so a lane's two accumulator columns are 4
  // words apart in the a / b rows (2-way instead of 4-way bank conflicts); the accumulators start
  // at -a_l b_l (exact: two floats) and end as the residuals r_l = (D zp)_l - a_l b_l
  // (trainer.cpp:56-71), squared and summed in fp64 per pair.
  __device__ static void pass2_dmma(const Params& p, State& st, const unsigned char* const* ins,
                                    unsigned char* extra, int grp, int item, int64_t g, const double* za,
                                    const double* zb) {
    constexpr int KS = (K + 3) / 4;          // k steps (4 codes each)
    constexpr int NT = (N + 7) / 8;          // wavelength tiles
    constexpr int TPG = (NT + G - 1) / G;    // tiles per warp group
    double* xchg = reinterpret_cast<double*>(extra + 32 * 8);
    const double* td = reinterpret_cast<const double*>(extra + 32 * 8 + kXchg);
#pragma unroll
    for (int j = 0; j < K; ++j) {
      xchg[(grp * 2 * K + j) * TS + item] = za[j];
      xchg[(grp * 2 * K + K + j) * TS + item] = zb[j];
    }
    __syncthreads();
    const int lane = threadIdx.x & 31, fi = lane >> 2, fc = lane & 3;
    const int pbase = item & ~31;  // the warp's first pair of the tile
    double af[4][KS];
#pragma unroll
    for (int m = 0; m < 4; ++m)
#pragma unroll
      for (int s = 0; s < KS; ++s) {
        const int j = 4 * s + fc, pl = pbase + 8 * m + fi;
        double sa = 0.0, sb = 0.0;
        if (j < K) {
#pragma unroll
          for (int h = 0; h < G; ++h) {  // the order of the DFMA path: group 0 + 1 + 2
            sa += xchg[(h * 2 * K + j) * TS + pl];
            sb += xchg[(h * 2 * K + K + j) * TS + pl];
          }
        }
        af[m][s] = sa * sb;  // zp = za (.) zb (codec.cpp:77-85); 0 in the padding slots
      }
    const float* arow = reinterpret_cast<const float*>(ins[0]) + (pbase + fi) * N;
    const float* brow = reinterpret_cast<const float*>(ins[1]) + (pbase + fi) * N;
    double accm[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
    for (int t = 0; t < TPG; ++t) {
      const int tn = grp * TPG + t;  // warp-uniform
      if (tn < NT) {
        const int wb = 8 * tn + (fi >> 1) + 4 * (fi & 1);  // B fragment column fi <-> wavelength
        double bf[KS];
#pragma unroll
        for (int s = 0; s < KS; ++s)
          bf[s] = (wb < N && 4 * s + fc < K) ? td[wb * KP + 4 * s + fc] : 0.0;
        const int w0 = 8 * tn + fc, w1 = w0 + 4;  // accumulator columns 2 fc, 2 fc + 1
        double c0[4], c1[4];
#pragma unroll
        for (int m = 0; m < 4; ++m) {
          float a0 = 0.f, b0 = 0.f, a1 = 0.f, b1 = 0.f;
          if (w0 < N) {
            a0 = arow[8 * m * N + w0];
            b0 = brow[8 * m * N + w0];
          }
          if (w1 < N) {
            a1 = arow[8 * m * N + w1];
            b1 = brow[8 * m * N + w1];
          }
          c0[m] = -(static_cast<double>(a0) * static_cast<double>(b0));  // exact
          c1[m] = -(static_cast<double>(a1) * static_cast<double>(b1));
        }
        // k step outer: the four pair blocks' MMAs are independent, a block's next step is 4 MMAs on
#pragma unroll
        for (int s = 0; s < KS; ++s)
#pragma unroll
          for (int m = 0; m < 4; ++m) dmma884(c0[m], c1[m], af[m][s], bf[s]);
#pragma unroll
        for (int m = 0; m < 4; ++m) {
          accm[m] = fma(c0[m], c0[m], accm[m]);
          accm[m] = fma(c1[m], c1[m], accm[m]);
        }
      }
    }
    const int64_t g0 = g - item + pbase + fi;  // global index of the lane's first pair
#pragma unroll
    for (int m = 0; m < 4; ++m)
      if (g0 + 8 * m < p.pairs) st.acc += accm[m];
  }

  __device__ static void compute(const Params& p, State& st, const unsigned char* const* ins,
                                 unsigned char* const*, unsigned char* extra, int item, int64_t g) {
    // Every thread of the CTA gets here exactly once per tile (tile_generic runs all T
    // pairs of a ragged tile), so the barrier below is uniform.
    // warp-uniform group (the shuffle lets the compiler see it; G = 1 ragged tiles run partial warps)
    const int grp = G > 1 ? __shfl_sync(0xffffffffu, static_cast<int>(threadIdx.x) / T, 0) : 0;
    const int L0 = grp * R;
    const float* a = reinterpret_cast<const float*>(ins[0]) + item * N + L0;
    const float* b = reinterpret_cast<const float*>(ins[1]) + item * N + L0;
    double* xchg = reinterpret_cast<double*>(extra + 32 * 8);
    const double2* td = reinterpret_cast<const double2*>(extra + 32 * 8 + kXchg) + L0 * (KP / 2);
    const double* E = p.E + L0;

    // pass 1: partial za = E a, zb = E b over [L0, L0 + R) (codec.cpp:36-46, trainer.cpp:52-53)
    constexpr bool kAbReg = HC_LOSS_ABREG && B1 == R && B2 == R;
    double ab[kAbReg ? R : 1];  // kAbReg: a_l b_l (exact fp64 products of two floats)
    double za[K], zb[K];
#pragma unroll
    for (int j = 0; j < K; ++j) za[j] = zb[j] = 0.0;
    constexpr bool kCe2 = HC_LOSS_CE2 && (G == 1 || G == 3);
    double abv[kCe2 ? R : 1];
    if constexpr (kCe2) {
      if (G == 1 || grp == 0) pass1_ce2<0>(p, a, b, za, zb, abv);
      else if (grp == 1) pass1_ce2<G == 3 ? 1 : 0>(p, a, b, za, zb, abv);
      else pass1_ce2<G == 3 ? 2 : 0>(p, a, b, za, zb, abv);
    } else if constexpr (HC_LOSS_CE && !kAbReg) {
      if constexpr (G == 1) {
        pass1_ce<0>(p, a, b, za, zb);
      } else {
        static_assert(G == 1 || G == 3, "warp groups");
        if (grp == 0) pass1_ce<0>(p, a, b, za, zb);
        else if (grp == 1) pass1_ce<G == 3 ? 1 : 0>(p, a, b, za, zb);
        else pass1_ce<G == 3 ? 2 : 0>(p, a, b, za, zb);
      }
    } else {
      float fa[B1], fb[B1];
      double va[B1], vb[B1];
#pragma unroll
      for (int i = 0; i < B1; ++i) {
#if HC_LOSS_VLOAD  // pinned at the top: every LDS of the batch in flight before the first use
        asm volatile("ld.shared.f32 %0, [%1];" : "=f"(fa[i]) : "r"(smem_u32(a + i)));
        asm volatile("ld.shared.f32 %0, [%1];" : "=f"(fb[i]) : "r"(smem_u32(b + i)));
#else
        fa[i] = a[i];
        fb[i] = b[i];
#endif
      }
#pragma unroll
      for (int i = 0; i < B1; ++i) {
        va[i] = static_cast<double>(fa[i]);
        vb[i] = static_cast<double>(fb[i]);
      }
      if (B1 < R) {
#pragma unroll
        for (int i = 0; i < B1; ++i) {
          fa[i] = a[B1 + i];
          fb[i] = b[B1 + i];
        }
      }
#pragma unroll 1
      for (int l0 = 0; l0 < R; l0 += B1) {
#pragma unroll
        for (int i = 0; i < B1; ++i)
#pragma unroll
          for (int j = 0; j < K; ++j) {
            const double e = E[j * N + l0 + i];  // warp-uniform: constant bank
            za[j] = fma(e, va[i], za[j]);
            zb[j] = fma(e, vb[i], zb[j]);
          }
        if constexpr (kAbReg) {
#pragma unroll
          for (int i = 0; i < B1; ++i) ab[i] = va[i] * vb[i];
        }
        if (l0 + B1 < R) {  // next batch: convert the floats loaded one batch ago, load the one after
#pragma unroll
          for (int i = 0; i < B1; ++i) {
            va[i] = static_cast<double>(fa[i]);
            vb[i] = static_cast<double>(fb[i]);
          }
          if (l0 + 2 * B1 < R) {
#pragma unroll
            for (int i = 0; i < B1; ++i) {
              fa[i] = a[l0 + 2 * B1 + i];
              fb[i] = b[l0 + 2 * B1 + i];
            }
          }
        }
      }
    }
    if constexpr (kDmma) {
      pass2_dmma(p, st, ins, extra, grp, item, g, za, zb);
      return;
    }
    // exchange the groups' partial codes; zp = za (.) zb (codec.cpp:77-85)
    if constexpr (G > 1) {
#pragma unroll
      for (int j = 0; j < K; ++j) {
        xchg[(grp * 2 * K + j) * T + item] = za[j];
        xchg[(grp * 2 * K + K + j) * T + item] = zb[j];
      }
      // Warp-specialised: only the G warps holding this 32-pair slice exchange (named barrier
      // 1 + slice); the CTA-barrier pipelines use the CTA barrier.
      if constexpr (kWarpSpecialized)
        asm volatile("bar.sync %0, %1;" ::"r"(1 + item / 32), "r"(32 * G) : "memory");
      else
        __syncthreads();
#pragma unroll
      for (int j = 0; j < K; ++j) {
        za[j] = xchg[j * T + item];
        zb[j] = xchg[(K + j) * T + item];
#pragma unroll
        for (int h = 1; h < G; ++h) {
          za[j] += xchg[(h * 2 * K + j) * T + item];
          zb[j] += xchg[(h * 2 * K + K + j) * T + item];
        }
      }
      // ws: the slice's next tile overwrites these partials; no CTA barrier separates tiles there
      if constexpr (kWarpSpecialized) asm volatile("bar.sync %0, %1;" ::"r"(1 + item / 32), "r"(32 * G) : "memory");
    }
#pragma unroll
    for (int j = 0; j < K; ++j) za[j] *= zb[j];

    // pass 2: r_l = (D zp)_l - a_l b_l over [L0, L0 + R), sum of r_l^2 (trainer.cpp:56-71)
    double acc = 0.0;
    if constexpr (kCe2) {
      if (G == 1 || grp == 0) acc = pass2_ce2<0>(p, za, abv);
      else if (grp == 1) acc = pass2_ce2<G == 3 ? 1 : 0>(p, za, abv);
      else acc = pass2_ce2<G == 3 ? 2 : 0>(p, za, abv);
    } else {
      float fa[B2], fb[B2];
      double d[B2][KP];
      auto load = [&](int l0) {
#pragma unroll
        for (int i = 0; i < B2; ++i) {
          if constexpr (!kAbReg) {
            fa[i] = a[l0 + i];
            fb[i] = b[l0 + i];
          }
#pragma unroll
          for (int c = 0; c < KP / 2; ++c) {
            const double2 v = td[(l0 + i) * (KP / 2) + c];  // same address in every lane: broadcast
            d[i][2 * c] = v.x;
            d[i][2 * c + 1] = v.y;
          }
        }
      };
      load(0);
#pragma unroll 1
      for (int l0 = 0; l0 < R; l0 += B2) {
        double s[B2];
#pragma unroll
        for (int i = 0; i < B2; ++i)
          s[i] = kAbReg ? -ab[i] : -(static_cast<double>(fa[i]) * static_cast<double>(fb[i]));  // exact
        double dc[B2][KP];
#pragma unroll
        for (int i = 0; i < B2; ++i)
#pragma unroll
          for (int c = 0; c < KP; ++c) dc[i][c] = d[i][c];
        if (l0 + B2 < R) load(l0 + B2);
#pragma unroll
        for (int i = 0; i < B2; ++i) {
          if (HC_LOSS_SPLIT && K % 2 == 0) {
            double s2 = dc[i][K / 2] * za[K / 2];
#pragma unroll
            for (int j = 0; j < K / 2; ++j) s[i] = fma(dc[i][j], za[j], s[i]);
#pragma unroll
            for (int j = K / 2 + 1; j < K; ++j) s2 = fma(dc[i][j], za[j], s2);
            s[i] += s2;
          } else {
#pragma unroll
            for (int j = 0; j < K; ++j) s[i] = fma(dc[i][j], za[j], s[i]);
          }
          acc = fma(s[i], s[i], acc);
        }
      }
    }
    if (g < p.pairs) st.acc += acc;
  }
  __device__ static void finish(const Params& p, State& st, unsigned char* extra) {
    double v = st.acc;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    double* red = reinterpret_cast<double*>(extra);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    __syncthreads();
    if (lane == 0) red[warp] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = 0.0;
      for (int w = 0; w < (THREADS + 31) / 32; ++w) t += red[w];
      p.partials[p.partial_offset + blockIdx.x] = t;
    }
  }
};

}  // namespace hcb
