/* ORACLE / TEST INFRASTRUCTURE — NOT PART OF THE PRODUCT.  See hc_oracle.h.
 *
 * Every function cites the reference lines it restates.  Arithmetic order and
 * precision deliberately match the reference so that tests/test_oracle.py can
 * hold this file bit-exact against the compiled reference (oracle/_ref).
 */
#include "hc_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* IEC 61966-2-1 XYZ -> linear sRGB, Y normalised to 1 (colorimetry.cpp:22-26). */
static const double kXyzToRgb[9] = {
    3.2404542, -1.5371385, -0.4985314,
    -0.9692660, 1.8760108, 0.0415560,
    0.0556434, -0.2040259, 1.0572252,
};

/* codec.cpp:8-12 */
double orc_softplus(double raw, double beta) {
  const double t = beta * raw;
  if (t > 30.0) return raw;
  return log1p(exp(t)) / beta;
}

/* codec.cpp:36-46 (encode): one double accumulator per code entry, i ascending. */
void orc_encode(const float* E, int k, int n, const float* S, int64_t rows, double* zd, float* zf) {
  for (int64_t r = 0; r < rows; ++r) {
    const float* s = S + r * n;
    for (int j = 0; j < k; ++j) {
      const float* e = E + (int64_t)j * n;
      double acc = 0.0;
      for (int i = 0; i < n; ++i) acc += (double)e[i] * (double)s[i];
      if (zd) zd[r * k + j] = acc;
      if (zf) zf[r * k + j] = (float)acc;
    }
  }
}

/* renderer.cpp:661-690 (decode_image): double accumulation over j ascending of
 * row[j] * double(latent(x, y, j)), stored as float. */
void orc_decode(const float* D, int k, int n, const float* Z, int64_t rows, float* S) {
  for (int64_t r = 0; r < rows; ++r) {
    const float* z = Z + r * k;
    for (int i = 0; i < n; ++i) {
      const float* row = D + (int64_t)i * k;
      double acc = 0.0;
      for (int j = 0; j < k; ++j) acc += (double)row[j] * (double)z[j];
      S[r * n + i] = (float)acc;
    }
  }
}

/* spectrum_to_xyz (colorimetry.cpp:75-87): sums of cmf*s in double, times the
 * grid step; xyz_to_linear_rgb (colorimetry.cpp:103-105, apply3x3 :28-37). */
static void xyz_rgb_of(const double* cmf, double dlambda, int n, const float* s, double xyz[3],
                       double rgb[3]) {
  double x = 0, y = 0, z = 0;
  for (int i = 0; i < n; ++i) {
    const double v = (double)s[i];
    x += cmf[i] * v;
    y += cmf[n + i] * v;
    z += cmf[2 * n + i] * v;
  }
  xyz[0] = x * dlambda;
  xyz[1] = y * dlambda;
  xyz[2] = z * dlambda;
  for (int r = 0; r < 3; ++r)
    rgb[r] = kXyzToRgb[3 * r + 0] * xyz[0] + kXyzToRgb[3 * r + 1] * xyz[1] +
             kXyzToRgb[3 * r + 2] * xyz[2];
}

/* image_to_linear_rgb (renderer.cpp:692-719) plus spectrum_to_xyz per pixel. */
void orc_spectra_to_outputs(const double* cmf, double dlambda, int n, const float* S, int64_t rows,
                            float* xyz, float* rgb) {
  double X[3], R[3];
  for (int64_t r = 0; r < rows; ++r) {
    xyz_rgb_of(cmf, dlambda, n, S + r * n, X, R);
    for (int c = 0; c < 3; ++c) {
      if (xyz) xyz[r * 3 + c] = (float)X[c];
      if (rgb) rgb[r * 3 + c] = (float)R[c];
    }
  }
}

static float* scratch(int64_t count) {
  float* p = (float*)malloc((size_t)(count > 0 ? count : 1) * sizeof(float));
  if (!p) abort();
  return p;
}

void orc_codec_roundtrip(const float* E, const float* D, int k, int n, const double* cmf,
                         double dlambda, const float* S, int64_t rows, float* Z, float* S2,
                         float* xyz, float* rgb) {
  float* z = scratch((int64_t)k);
  float* s2 = scratch((int64_t)n);
  for (int64_t r = 0; r < rows; ++r) {
    orc_encode(E, k, n, S + r * n, 1, NULL, z);
    orc_decode(D, k, n, z, 1, s2);
    if (Z) memcpy(Z + r * k, z, sizeof(float) * (size_t)k);
    if (S2) memcpy(S2 + r * n, s2, sizeof(float) * (size_t)n);
    orc_spectra_to_outputs(cmf, dlambda, n, s2, 1, xyz ? xyz + r * 3 : NULL, rgb ? rgb + r * 3 : NULL);
  }
  free(z);
  free(s2);
}

/* code_to_floats (renderer.cpp:117-125) with gain 1. */
void orc_asset_codes(const float* E, int k, int n, const float* S, int64_t count, float* Z) {
  orc_encode(E, k, n, S, count, NULL, Z);
}

/* R1: NEE channel loop rad[c] += thr[c]*albedo[c]*le[c]*w (renderer.cpp:505-510)
 * with thr = 1 and w = c_{p,l}, evaluated left to right in float; the pixel
 * value is float(double(rad) * (1/spp)) with spp = 1 (renderer.cpp:548-551,
 * :588-592).  Channels are independent, so the k/3-pass execution
 * (renderer.cpp:274-283) and reassembly out(3b+c) = pass_b(c)
 * (renderer.cpp:645-657) give these values channel for channel. */
void orc_shade_latent(const float* D, int k, int n, const double* cmf, double dlambda,
                      const float* pal_codes, const float* light_codes, int L,
                      const uint32_t* idx, const float* cosv, int64_t P, float* latent,
                      float* S2, float* xyz, float* rgb) {
  float* z = scratch((int64_t)k);
  float* s2 = scratch((int64_t)n);
  for (int64_t p = 0; p < P; ++p) {
    const float* albedo = pal_codes + (int64_t)idx[p] * k;
    for (int b = 0; b < k / 3; ++b) {
      for (int c = 3 * b; c < 3 * b + 3; ++c) {
        float rad = 0.f;
        for (int l = 0; l < L; ++l) rad += 1.0f * albedo[c] * light_codes[l * k + c] * cosv[p * L + l];
        z[c] = (float)((double)rad * (1.0 / 1));
      }
    }
    if (latent) memcpy(latent + p * k, z, sizeof(float) * (size_t)k);
    orc_decode(D, k, n, z, 1, s2);
    if (S2) memcpy(S2 + p * n, s2, sizeof(float) * (size_t)n);
    orc_spectra_to_outputs(cmf, dlambda, n, s2, 1, xyz ? xyz + p * 3 : NULL, rgb ? rgb + p * 3 : NULL);
  }
  free(z);
  free(s2);
}

/* The same loop at C = n with curve_to_floats assets (renderer.cpp:187-190). */
void orc_shade_spectral(int n, const double* cmf, double dlambda, const float* pal_spectra,
                        const float* light_spectra, int L, const uint32_t* idx,
                        const float* cosv, int64_t P, float* S2, float* xyz, float* rgb) {
  float* s = scratch((int64_t)n);
  for (int64_t p = 0; p < P; ++p) {
    const float* albedo = pal_spectra + (int64_t)idx[p] * n;
    for (int c = 0; c < n; ++c) {
      float rad = 0.f;
      for (int l = 0; l < L; ++l) rad += 1.0f * albedo[c] * light_spectra[l * n + c] * cosv[p * L + l];
      s[c] = (float)(double)rad;
    }
    if (S2) memcpy(S2 + p * n, s, sizeof(float) * (size_t)n);
    orc_spectra_to_outputs(cmf, dlambda, n, s, 1, xyz ? xyz + p * 3 : NULL, rgb ? rgb + p * 3 : NULL);
  }
  free(s);
}

/* R2: per sample thr = 1, rad = 0; for d < depth:
 * rad += thr*albedo_d*le*t_d (renderer.cpp:505-510), thr *= albedo_d
 * (:530-533); acc += double(rad) over samples (:548-551); out = float(acc/spp)
 * (:588-592).  Layouts: pidx [P][spp][depth], iidx [P][spp], tw [P][spp][depth]. */
void orc_chain(int C, const float* pal, const float* ill, const uint8_t* pidx,
               const uint8_t* iidx, const float* tw, int64_t P, int spp, int depth, float* out) {
  double* acc = (double*)malloc(sizeof(double) * (size_t)C);
  float* thr = scratch(C);
  float* rad = scratch(C);
  if (!acc) abort();
  for (int64_t p = 0; p < P; ++p) {
    for (int c = 0; c < C; ++c) acc[c] = 0.0;
    for (int s = 0; s < spp; ++s) {
      const int64_t smp = p * spp + s;
      const float* le = ill + (int64_t)iidx[smp] * C;
      for (int c = 0; c < C; ++c) {
        thr[c] = 1.f;
        rad[c] = 0.f;
      }
      for (int d = 0; d < depth; ++d) {
        const float* albedo = pal + (int64_t)pidx[smp * depth + d] * C;
        const float w = tw[smp * depth + d];
        for (int c = 0; c < C; ++c) rad[c] += thr[c] * albedo[c] * le[c] * w;
        for (int c = 0; c < C; ++c) thr[c] *= albedo[c];
      }
      for (int c = 0; c < C; ++c) acc[c] += (double)rad[c];
    }
    const double inv_spp = 1.0 / spp;
    for (int c = 0; c < C; ++c) out[p * C + c] = (float)(acc[c] * inv_spp);
  }
  free(acc);
  free(thr);
  free(rad);
}

/* Round-to-nearest-even to bf16, returned as the float it represents. */
float orc_bf16_round(float x) {
  uint32_t u;
  memcpy(&u, &x, 4);
  if ((u & 0x7f800000u) == 0x7f800000u) return x;
  u += 0x7fffu + ((u >> 16) & 1u);
  u &= 0xffff0000u;
  float r;
  memcpy(&r, &u, 4);
  return r;
}

/* R3: forward (upsampler.cpp:42-72) — h1 = act(W1 x + b1), h2 = act(W2 h1 + b2),
 * z = head(W3 h2 + b3) — with BASELINE's ReLU hidden layers and softplus(beta=1)
 * head (codec.cpp:8-12).  Tensor-core operands are bf16: the input and the hidden
 * activations are rounded to bf16 before each layer (weights arrive as
 * bf16-representable floats); accumulation in double. */
void orc_mlp_forward(const float* rgb, int64_t P, int hidden, int k, const float* w1,
                     const float* b1, const float* w2, const float* b2, const float* w3,
                     const float* b3, float* out) {
  double* h1 = (double*)malloc(sizeof(double) * (size_t)hidden);
  double* h2 = (double*)malloc(sizeof(double) * (size_t)hidden);
  if (!h1 || !h2) abort();
  for (int64_t p = 0; p < P; ++p) {
    double x[3];
    for (int j = 0; j < 3; ++j) x[j] = orc_bf16_round(rgb[p * 3 + j]);
    for (int i = 0; i < hidden; ++i) {
      double acc = b1[i];
      for (int j = 0; j < 3; ++j) acc += (double)w1[i * 3 + j] * x[j];
      h1[i] = orc_bf16_round((float)(acc > 0.0 ? acc : 0.0));
    }
    for (int i = 0; i < hidden; ++i) {
      double acc = b2[i];
      for (int j = 0; j < hidden; ++j) acc += (double)w2[i * hidden + j] * h1[j];
      h2[i] = orc_bf16_round((float)(acc > 0.0 ? acc : 0.0));
    }
    for (int i = 0; i < k; ++i) {
      double acc = b3[i];
      for (int j = 0; j < hidden; ++j) acc += (double)w3[i * hidden + j] * h2[j];
      out[p * k + i] = (float)orc_softplus(acc, 1.0);
    }
  }
  free(h1);
  free(h2);
}

/* R4: forward_pair (trainer.cpp:49-62) — zp = E(a) o E(b), s_hat = D zp,
 * s = a o b — and sum over lambda of (s_hat - s)^2 (mse_n trainer.cpp:64-71
 * without the 1/n), summed over pairs in double. */
double orc_hadamard_loss(const float* E, const float* D, int k, int n, const float* A,
                         const float* B, int64_t pairs) {
  double* za = (double*)malloc(sizeof(double) * (size_t)k);
  double* zb = (double*)malloc(sizeof(double) * (size_t)k);
  if (!za || !zb) abort();
  double total = 0.0;
  for (int64_t r = 0; r < pairs; ++r) {
    const float* a = A + r * n;
    const float* b = B + r * n;
    orc_encode(E, k, n, a, 1, za, NULL);
    orc_encode(E, k, n, b, 1, zb, NULL);
    for (int j = 0; j < k; ++j) za[j] = za[j] * zb[j];
    for (int i = 0; i < n; ++i) {
      double acc = 0.0;
      for (int j = 0; j < k; ++j) acc += (double)D[(int64_t)i * k + j] * za[j];
      const double d = acc - (double)a[i] * (double)b[i];
      total += d * d;
    }
  }
  free(za);
  free(zb);
  return total;
}

/* spectrum_to_xyz (colorimetry.cpp:75-87) on a double-precision curve (KAT pinning). */
void orc_spectrum_to_xyz_d(const double* cmf, double dlambda, int n, const double* s, double* xyz) {
  double x = 0, y = 0, z = 0;
  for (int i = 0; i < n; ++i) {
    x += cmf[i] * s[i];
    y += cmf[n + i] * s[i];
    z += cmf[2 * n + i] * s[i];
  }
  xyz[0] = x * dlambda;
  xyz[1] = y * dlambda;
  xyz[2] = z * dlambda;
}

/* ===================================================================== colour-metric tail
 * the reference's consumers of the hot path's output —
 * exposure_for / tonemap_srgb8 / error_map (renderer.cpp:721-802),
 * scene_color_report (evaluation.cpp:122-154) and the per-chain Delta E94 of
 * multibounce_eval (evaluation.cpp:59-86) — over pixel arrays instead of
 * ChannelImage (P = width * height pixels, HWC). */

/* IEC 61966-2-1 linear sRGB -> XYZ (colorimetry.cpp:27-31). */
static const double kRgbToXyz[9] = {
    0.4124564, 0.3575761, 0.1804375,
    0.2126729, 0.7151522, 0.0721750,
    0.0193339, 0.1191920, 0.9503041,
};

static int cmp_double(const void* a, const void* b) {
  const double x = *(const double*)a, y = *(const double*)b;
  return (x > y) - (x < y);
}

/* percentile_nearest_rank (evaluation.cpp:14-21); the same index rule as exposure_for
 * (renderer.cpp:744-747).  Sorts a copy. */
double orc_percentile_nearest_rank(const double* v, int64_t count, double p) {
  if (count <= 0) return 0.0;
  double* s = (double*)malloc(sizeof(double) * (size_t)count);
  if (!s) abort();
  memcpy(s, v, sizeof(double) * (size_t)count);
  qsort(s, (size_t)count, sizeof(double), cmp_double);
  const double rank = p / 100.0 * (double)count;
  int64_t idx = (int64_t)ceil(rank);
  idx = idx == 0 ? 0 : idx - 1;
  if (idx > count - 1) idx = count - 1;
  const double r = s[idx];
  free(s);
  return r;
}

/* Per-pixel luminance of exposure_for (renderer.cpp:730-742): Rec.709 luma of linear RGB
 * (3 channels) or dlambda * sum_i ybar_i s_i (n channels). */
void orc_luminance(const float* img, int64_t P, int channels, const double* ybar, double dlambda,
                   double* lum) {
  for (int64_t p = 0; p < P; ++p) {
    const float* px = img + p * channels;
    double v = 0.0;
    if (channels == 3) {
      v = 0.2126 * (double)px[0] + 0.7152 * (double)px[1] + 0.0722 * (double)px[2];
    } else {
      for (int i = 0; i < channels; ++i) v += ybar[i] * (double)px[i];
      v *= dlambda;
    }
    lum[p] = v;
  }
}

/* exposure_for (renderer.cpp:721-752): 1 / nearest-rank percentile of the luminance. */
double orc_exposure_for(const float* img, int64_t P, int channels, const double* ybar, double dlambda,
                        double percentile) {
  double* lum = (double*)malloc(sizeof(double) * (size_t)(P > 0 ? P : 1));
  if (!lum) abort();
  orc_luminance(img, P, channels, ybar, dlambda, lum);
  const double ref = orc_percentile_nearest_rank(lum, P, percentile);
  free(lum);
  return ref > 1e-12 ? 1.0 / ref : 1.0;
}

/* srgb_encode (colorimetry.cpp:159-162). */
double orc_srgb_encode(double linear) {
  if (linear <= 0.0031308) return 12.92 * linear;
  return 1.055 * pow(linear, 1.0 / 2.4) - 0.055;
}

/* tonemap_srgb8 (renderer.cpp:754-773). */
void orc_tonemap_srgb8(const float* rgb, int64_t P, double exposure, uint8_t* out) {
  for (int64_t i = 0; i < P * 3; ++i) {
    double v = (double)rgb[i] * exposure;
    v = v < 0.0 ? 0.0 : (v > 1.0 ? 1.0 : v);
    out[i] = (uint8_t)(orc_srgb_encode(v) * 255.0 + 0.5);
  }
}

/* image_to_linear_rgb (renderer.cpp:692-719): identity for 3 channels, else
 * spectrum_to_xyz (colorimetry.cpp:75-87) + xyz_to_linear_rgb (:103-105) in double. */
void orc_image_to_linear_rgb(const float* img, int64_t P, int channels, const double* cmf, double dlambda,
                             float* rgb) {
  for (int64_t p = 0; p < P; ++p) {
    const float* px = img + p * channels;
    if (channels == 3) {
      rgb[p * 3] = px[0];
      rgb[p * 3 + 1] = px[1];
      rgb[p * 3 + 2] = px[2];
      continue;
    }
    double x = 0, y = 0, z = 0;
    for (int i = 0; i < channels; ++i) {
      x += cmf[i] * (double)px[i];
      y += cmf[channels + i] * (double)px[i];
      z += cmf[2 * channels + i] * (double)px[i];
    }
    const double xyz[3] = {x * dlambda, y * dlambda, z * dlambda};
    for (int r = 0; r < 3; ++r)
      rgb[p * 3 + r] = (float)(kXyzToRgb[3 * r] * xyz[0] + kXyzToRgb[3 * r + 1] * xyz[1] +
                               kXyzToRgb[3 * r + 2] * xyz[2]);
  }
}

/* error_map (renderer.cpp:775-802): per-pixel mean of squared linear-RGB differences
 * (float), returns the mean over pixels (double).  mse may be NULL. */
double orc_error_map(const float* a, int ca, const float* b, int cb, int64_t P, const double* cmf,
                     double dlambda, float* mse) {
  float* ra = (float*)malloc(sizeof(float) * (size_t)(P > 0 ? P : 1) * 3);
  float* rb = (float*)malloc(sizeof(float) * (size_t)(P > 0 ? P : 1) * 3);
  if (!ra || !rb) abort();
  orc_image_to_linear_rgb(a, P, ca, cmf, dlambda, ra);
  orc_image_to_linear_rgb(b, P, cb, cmf, dlambda, rb);
  double total = 0.0;
  for (int64_t p = 0; p < P; ++p) {
    double acc = 0.0;
    for (int c = 0; c < 3; ++c) {
      const double d = (double)ra[p * 3 + c] - (double)rb[p * 3 + c];
      acc += d * d;
    }
    acc /= 3.0;
    if (mse) mse[p] = (float)acc;
    total += acc;
  }
  free(ra);
  free(rb);
  return total / (double)P;
}

/* xyz_to_lab (colorimetry.cpp:118-135). */
void orc_xyz_to_lab(const double* xyz, const double* white, double* lab) {
  const double delta = 6.0 / 29.0;
  const double delta3 = delta * delta * delta;
  double f[3];
  for (int i = 0; i < 3; ++i) {
    const double t = xyz[i] / white[i];
    f[i] = t > delta3 ? cbrt(t) : t / (3.0 * delta * delta) + 4.0 / 29.0;
  }
  lab[0] = 116.0 * f[1] - 16.0;
  lab[1] = 500.0 * (f[0] - f[1]);
  lab[2] = 200.0 * (f[1] - f[2]);
}

/* delta_e76 / delta_e94 (colorimetry.cpp:137-157; graphic-arts constants). */
double orc_delta_e76(const double* a, const double* b) {
  const double dl = a[0] - b[0], da = a[1] - b[1], db = a[2] - b[2];
  return sqrt(dl * dl + da * da + db * db);
}
double orc_delta_e94(const double* ref, const double* sample) {
  const double dl = ref[0] - sample[0];
  const double c1 = hypot(ref[1], ref[2]);
  const double c2 = hypot(sample[1], sample[2]);
  const double dc = c1 - c2;
  const double da = ref[1] - sample[1];
  const double db = ref[2] - sample[2];
  double dh2 = da * da + db * db - dc * dc;
  dh2 = dh2 > 0.0 ? dh2 : 0.0;
  const double sc = 1.0 + 0.045 * c1;
  const double sh = 1.0 + 0.015 * c1;
  return sqrt(dl * dl + (dc / sc) * (dc / sc) + dh2 / (sh * sh));
}

/* scene_color_report (evaluation.cpp:122-154): out = {mean_de76, p95_de76, mse, exposure}.
 * ybar = cmf + n (row 1) when the ground truth is spectral. */
void orc_scene_color_report(const float* gt, int cgt, const float* test, int ctest, int64_t P,
                            const double* cmf, double dlambda, double* out) {
  const double exposure = orc_exposure_for(gt, P, cgt, cgt == 3 ? NULL : cmf + cgt, dlambda, 99.5);
  float* ga = (float*)malloc(sizeof(float) * (size_t)(P > 0 ? P : 1) * 3);
  float* ta = (float*)malloc(sizeof(float) * (size_t)(P > 0 ? P : 1) * 3);
  double* des = (double*)malloc(sizeof(double) * (size_t)(P > 0 ? P : 1));
  if (!ga || !ta || !des) abort();
  orc_image_to_linear_rgb(gt, P, cgt, cmf, dlambda, ga);
  orc_image_to_linear_rgb(test, P, ctest, cmf, dlambda, ta);
  const double white[3] = {0.95047, 1.0, 1.08883}; /* srgb_reference_white, colorimetry.cpp:111-116 */
  double sum = 0.0;
  for (int64_t p = 0; p < P; ++p) {
    double a[3], b[3], xa[3], xb[3], la[3], lb[3];
    for (int c = 0; c < 3; ++c) {
      a[c] = (double)ga[p * 3 + c] * exposure;
      b[c] = (double)ta[p * 3 + c] * exposure;
    }
    for (int r = 0; r < 3; ++r) {
      xa[r] = kRgbToXyz[3 * r] * a[0] + kRgbToXyz[3 * r + 1] * a[1] + kRgbToXyz[3 * r + 2] * a[2];
      xb[r] = kRgbToXyz[3 * r] * b[0] + kRgbToXyz[3 * r + 1] * b[1] + kRgbToXyz[3 * r + 2] * b[2];
    }
    orc_xyz_to_lab(xa, white, la);
    orc_xyz_to_lab(xb, white, lb);
    des[p] = orc_delta_e76(la, lb);
    sum += des[p];
  }
  out[0] = P > 0 ? sum / (double)P : 0.0; /* mean_of (evaluation.cpp:23-28) */
  out[1] = orc_percentile_nearest_rank(des, P, 95.0);
  out[2] = orc_error_map(gt, cgt, test, ctest, P, cmf, dlambda, NULL);
  out[3] = exposure;
  free(ga);
  free(ta);
  free(des);
}

/* R5: the Delta E94 of multibounce_eval (evaluation.cpp:59-86) per
 * pixel of a ground-truth and a test XYZ image: white = D65 white scaled to the ground
 * truth's luminance (max(Y_gt, 1e-6) / Y_white), Lab of both, delta_e94(gt, test).
 * out = {mean, median, p95}; de (may be NULL) per pixel. */
void orc_delta_e94_report(const float* xyz_gt, const float* xyz_test, int64_t P, const double* white_d65,
                          float* de, double* out) {
  double* v = (double*)malloc(sizeof(double) * (size_t)(P > 0 ? P : 1));
  if (!v) abort();
  double sum = 0.0;
  for (int64_t p = 0; p < P; ++p) {
    double g[3], t[3], w[3], lg[3], lt[3];
    for (int c = 0; c < 3; ++c) {
      g[c] = (double)xyz_gt[p * 3 + c];
      t[c] = (double)xyz_test[p * 3 + c];
    }
    const double y_white = g[1] > 1e-6 ? g[1] : 1e-6;
    const double scale = y_white / white_d65[1];
    for (int c = 0; c < 3; ++c) w[c] = white_d65[c] * scale;
    orc_xyz_to_lab(g, w, lg);
    orc_xyz_to_lab(t, w, lt);
    v[p] = orc_delta_e94(lg, lt);
    if (de) de[p] = (float)v[p];
    sum += v[p];
  }
  out[0] = P > 0 ? sum / (double)P : 0.0;
  out[1] = orc_percentile_nearest_rank(v, P, 50.0);
  out[2] = orc_percentile_nearest_rank(v, P, 95.0);
  free(v);
}
