// Drop-in API tests: the reference's own codec / colorimetry test cases
// (proj/tests/test_codec.cpp, test_colorimetry.cpp) re-run through
// include/hadacodec_b200.hpp on the GPU.  Exact checks stay exact; checks the
// reference makes at 1e-14 against fp64 arithmetic are made at fp32 tolerance.
#include <cmath>
#include <cstdio>
#include <limits>
#include <stdexcept>
#include <string>
#include <vector>

#include "hadacodec_b200.hpp"

using namespace hadacodec::b200;

static int g_fail = 0, g_checks = 0;
#define CHECK(cond)                                                        \
  do {                                                                     \
    ++g_checks;                                                            \
    if (!(cond)) {                                                         \
      ++g_fail;                                                            \
      std::fprintf(stderr, "FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond); \
    }                                                                      \
  } while (0)
#define CHECK_THROWS_AS(expr, ex)      \
  do {                                 \
    bool _t = false;                   \
    try {                              \
      (void)(expr);                    \
    } catch (const ex&) {              \
      _t = true;                       \
    } catch (...) {                    \
    }                                  \
    CHECK(_t && #ex);                  \
  } while (0)

static bool rel_close(double a, double b, double rel) { return std::fabs(a - b) <= rel * std::max(1.0, std::fabs(b)); }

// xoshiro-free deterministic values (the reference's tests use Rng streams; any
// seeded values exercise the same contracts).
static double lcg(uint64_t& s) {
  s = s * 6364136223846793005ull + 1442695040888963407ull;
  return static_cast<double>(s >> 11) * 0x1.0p-53;
}

static CodecWeights random_weights(int k, int n, uint64_t seed) {  // test_codec.cpp:16-27
  CodecWeights w;
  w.k = k;
  w.n = n;
  w.raw_enc.resize(static_cast<size_t>(k) * n);
  w.raw_dec.resize(static_cast<size_t>(n) * k);
  for (double& v : w.raw_enc) v = -0.3 + 0.6 * lcg(seed);
  for (double& v : w.raw_dec) v = -0.3 + 0.6 * lcg(seed);
  return w;
}

int main() {
  // softplus values and branches (test_codec.cpp:35-60): host arithmetic, exact contract
  CHECK(rel_close(softplus(0.0, 10.0), 0.069314718055994526, 1e-14));
  CHECK(rel_close(softplus(-1.0, 10.0), 4.5398899216864648e-06, 1e-12));
  CHECK(rel_close(softplus(0.2, 10.0), 0.21269280110429728, 1e-14));
  CHECK(softplus(3.1, 10.0) == 3.1);
  CHECK(softplus(1000.0, 10.0) == 1000.0);
  CHECK(softplus_derivative(3.1, 10.0) == 1.0);
  CHECK(rel_close(softplus_derivative(0.2, 10.0), 0.88079707797788231, 1e-14));

  Device dev(0);
  const Grid g47 = Grid::reference47();

  // effective weights strictly positive (test_codec.cpp:70-79)
  const CodecWeights w = random_weights(6, 47, 17);
  const EffectiveWeights e = effective_weights(w);
  for (double v : e.enc) CHECK(v > 0.0);
  for (double v : e.dec) CHECK(v > 0.0);

  // encode / decode = explicit mat-vec (test_codec.cpp:81-111): the by-value calls run the
  // fp64 kernels in the reference's order, so they equal the plain sequential loops exactly
  Codec codec(dev, e, g47);
  uint64_t s = 99;
  SpectralCurve sc(47);
  for (int i = 0; i < 47; ++i) sc[i] = lcg(s);
  const LatentCode z = encode(codec, sc);
  CHECK(z.k() == 6);
  for (int j = 0; j < 6; ++j) {
    double acc = 0.0;
    for (int i = 0; i < 47; ++i) acc += e.enc[j * 47 + i] * sc[i];
    CHECK(z[j] == acc);
    CHECK(z[j] >= 0.0);
  }
  const SpectralCurve d = decode(codec, z);
  for (int i = 0; i < 47; ++i) {
    double acc = 0.0;
    for (int j = 0; j < 6; ++j) acc += e.dec[i * 6 + j] * z[j];
    CHECK(d[i] == acc);
  }
  // CodecWeights overload agrees with the EffectiveWeights path (same softplus, bit for bit)
  Codec codec_raw(dev, w, g47);
  const LatentCode z2 = encode(codec_raw, sc);
  for (int j = 0; j < 6; ++j) CHECK(z2[j] == z[j]);
  // encode_resampled on the codec's own grid without zeroing = encode
  {
    std::vector<double> wl(47);
    for (int i = 0; i < 47; ++i) wl[static_cast<size_t>(i)] = g47.wavelength_at(i);
    const std::vector<LatentCode> zr = encode_resampled(codec, wl, {sc.v}, /*zero_outside=*/false);
    CHECK(zr.size() == 1u && zr[0].z == z.z);
    CHECK_THROWS_AS(encode_resampled(codec, {400.0, 400.0}, {{1.0, 2.0}}), std::invalid_argument);
  }

  // linearity (test_codec.cpp:113-137) at fp32 tolerance
  for (int it = 0; it < 20; ++it) {
    SpectralCurve a(47), b(47), ab(47), as(47);
    const double alpha = 5.0 * lcg(s);
    for (int i = 0; i < 47; ++i) {
      a[i] = 2.0 * lcg(s);
      b[i] = 2.0 * lcg(s);
      ab[i] = static_cast<double>(static_cast<float>(a[i]) + static_cast<float>(b[i]));
      as[i] = alpha * a[i];
    }
    const LatentCode za = encode(codec, a), zb = encode(codec, b), zs = encode(codec, ab), zc = encode(codec, as);
    for (int j = 0; j < 6; ++j) {
      CHECK(std::fabs(zs[j] - (za[j] + zb[j])) <= 2e-6 * std::max(1.0, std::fabs(za[j] + zb[j])));
      CHECK(std::fabs(zc[j] - alpha * za[j]) <= 2e-6 * std::max(1.0, std::fabs(alpha * za[j])));
    }
  }

  // decode rejects negative codes and wrong dimensions (test_codec.cpp:139-152)
  LatentCode zz;
  zz.z = {0.1, 0.2, 0.3, 0.4, 0.5, 0.6};
  (void)decode(codec, zz);
  zz[2] = -1e-9;
  CHECK_THROWS_AS(decode(codec, zz), std::domain_error);
  zz.z = {0.1, 0.2, 0.3};
  CHECK_THROWS_AS(decode(codec, zz), std::invalid_argument);

  // blockwise hadamard and block packing (test_codec.cpp:154-180): exact
  LatentCode ha, hb;
  ha.z = {1.0, 2.0, 3.0, 4.0, 5.0, 6.0};
  hb.z = {0.5, 0.5, 2.0, 0.0, 1.0, 3.0};
  const LatentCode h = blockwise_hadamard(ha, hb);
  const double expect[6] = {0.5, 1.0, 6.0, 0.0, 5.0, 18.0};
  for (int j = 0; j < 6; ++j) CHECK(h[j] == expect[j]);
  LatentCode shortc;
  shortc.z = {1.0, 2.0, 3.0};
  CHECK_THROWS_AS(blockwise_hadamard(ha, shortc), std::invalid_argument);
  const auto blocks = split_blocks(ha);
  CHECK(blocks.size() == 2u && blocks[1][2] == 6.0);
  const LatentCode joined = join_blocks(blocks);
  for (int j = 0; j < 6; ++j) CHECK(joined[j] == ha[j]);
  LatentCode bad;
  bad.z = {1.0, 2.0, 3.0, 4.0};
  CHECK_THROWS_AS(split_blocks(bad), std::invalid_argument);

  // weight validation (test_codec.cpp:182-216)
  CodecWeights v = w;
  v.k = 0;
  CHECK_THROWS_AS(validate(v, g47), std::invalid_argument);
  v = w;
  v.k = 5;
  v.raw_enc.resize(5u * 47u);
  v.raw_dec.resize(47u * 5u);
  CHECK_THROWS_AS(validate(v, g47), std::invalid_argument);
  v = w;
  v.n = 46;
  CHECK_THROWS_AS(validate(v, g47), std::invalid_argument);
  v = w;
  v.beta = 0.0;
  CHECK_THROWS_AS(validate(v, g47), std::invalid_argument);
  v = w;
  v.raw_dec[3] = std::numeric_limits<double>::quiet_NaN();
  CHECK_THROWS_AS(validate(v, g47), std::invalid_argument);

  // radiance-convention XYZ of ones (test_colorimetry.cpp:66-70) at fp32 tolerance
  const ColorTriple xyz = spectrum_to_xyz(codec, SpectralCurve(47, 1.0));
  CHECK(rel_close(xyz[0], 106.852687015155, 1e-6));
  CHECK(rel_close(xyz[1], 106.858452950433, 1e-6));
  CHECK(rel_close(xyz[2], 106.836643798253, 1e-6));
  // sRGB white (test_colorimetry.cpp:157-165)
  ColorTriple wh;
  wh.c = {0.95047, 1.0, 1.08883};
  const ColorTriple rgbw = xyz_to_linear_rgb(wh);
  for (int c = 0; c < 3; ++c) CHECK(std::fabs(rgbw[c] - 1.0) < 1e-6);

  // decode_image / image_to_linear_rgb on a 7 x 5 latent image (renderer.cpp:661-719)
  ChannelImage lat;
  lat.width = 7;
  lat.height = 5;
  lat.channels = 6;
  lat.data.resize(7 * 5 * 6);
  for (float& x : lat.data) x = static_cast<float>(lcg(s));
  const ChannelImage spec = decode_image(codec, lat);
  CHECK(spec.channels == 47 && spec.data.size() == 7u * 5u * 47u);
  for (int p = 0; p < 35; ++p)
    for (int i = 0; i < 47; ++i) {
      double acc = 0.0;
      for (int j = 0; j < 6; ++j)
        acc += static_cast<double>(static_cast<float>(e.dec[i * 6 + j])) * lat.data[p * 6 + j];
      CHECK(rel_close(spec.data[p * 47 + i], acc, 2e-6));
    }
  const ChannelImage rgb = image_to_linear_rgb(codec, spec);
  CHECK(rgb.channels == 3 && rgb.data.size() == 35u * 3u);
  lat.channels = 5;
  CHECK_THROWS_AS(decode_image(codec, lat), std::invalid_argument);

  // G-buffer shading through the drop-in API: multipass/fused latent vs naive, finite
  GBuffer gb;
  gb.width = 16;
  gb.height = 8;
  gb.lights = 8;
  for (int p = 0; p < 128; ++p) gb.palette_index.push_back(static_cast<uint32_t>(lcg(s) * 4));
  for (int i = 0; i < 128 * 8; ++i) gb.cos_terms.push_back(static_cast<float>(lcg(s)));
  std::vector<float> pal_spec(4 * 47), light_spec(8 * 47);
  for (float& x : pal_spec) x = static_cast<float>(lcg(s));
  for (float& x : light_spec) x = static_cast<float>(lcg(s));
  const std::vector<float> pal_codes = encode_batch(codec, pal_spec), light_codes = encode_batch(codec, light_spec);
  const ShadedFrame lf = shade_latent(codec, pal_codes, light_codes, gb);
  const ShadedFrame nf = shade_spectral(codec, pal_spec, light_spec, gb);
  for (int p = 0; p < 128; ++p) {
    // latent channel c = zR[idx] * sum_l cos_l zL_l (renderer.cpp:505-510)
    for (int c = 0; c < 6; ++c) {
      double acc = 0.0;
      for (int l = 0; l < 8; ++l) acc += gb.cos_terms[p * 8 + l] * light_codes[l * 6 + c];
      CHECK(rel_close(lf.latent.data[p * 6 + c], pal_codes[gb.palette_index[p] * 6 + c] * acc, 2e-6));
    }
    CHECK(std::isfinite(nf.xyz.data[p * 3 + 1]) && nf.xyz.data[p * 3 + 1] >= 0.f);
  }
  {  // frame stream through the host pipeline == frame by frame
    GBuffer gb2 = gb;
    for (float& x : gb2.cos_terms) x = 1.f - x;
    const std::vector<ShadedFrame> fs = shade_latent_frames(codec, pal_codes, light_codes, {gb, gb2, gb});
    const ShadedFrame lf2 = shade_latent(codec, pal_codes, light_codes, gb2);
    CHECK(fs.size() == 3u);
    CHECK(fs[0].xyz.data == lf.xyz.data && fs[0].linear_rgb.data == lf.linear_rgb.data);
    CHECK(fs[1].xyz.data == lf2.xyz.data && fs[1].linear_rgb.data == lf2.linear_rgb.data);
    CHECK(fs[2].linear_rgb.data == lf.linear_rgb.data);
    GBuffer small = gb;
    small.width = 8;
    small.palette_index.resize(64);
    small.cos_terms.resize(64 * 8);
    CHECK_THROWS_AS(shade_latent_frames(codec, pal_codes, light_codes, {gb, small}), std::invalid_argument);
  }
  gb.palette_index[3] = 77;  // out of range of the 4-entry palette
  CHECK_THROWS_AS(shade_latent(codec, pal_codes, light_codes, gb), std::invalid_argument);

  // colour-metric tail (renderer.cpp:721-802, evaluation.cpp:122-154, colorimetry.cpp:159-162)
  {
    ChannelImage grey;
    grey.width = 4;
    grey.height = 2;
    grey.channels = 3;
    grey.data.assign(24, 0.25f);
    const double e = exposure_for(codec, grey);
    const double lum = 0.2126 * 0.25 + 0.7152 * 0.25 + 0.0722 * 0.25;
    CHECK(e == 1.0 / lum);
    ChannelImage half = grey;
    half.data.assign(24, 0.5f);
    const std::vector<unsigned char> b = tonemap_srgb8(dev, half, 1.0);
    CHECK(b.size() == 24u && b[0] == 188 && b[23] == 188);  // srgb_encode(0.5) = 0.73535698 -> 188
    CHECK(tonemap_srgb8(dev, half, 10.0)[5] == 255);
    ChannelImage dark = grey;
    dark.data.assign(24, 0.0f);
    CHECK(exposure_for(codec, dark) == 1.0);
    const ErrorMap em = error_map(codec, grey, half);
    CHECK(em.mse.size() == 8u && rel_close(em.mse[0], 0.0625, 1e-7) && rel_close(em.mean_mse, 0.0625, 1e-12));
    const SceneColorReport same = scene_color_report(codec, half, half);
    CHECK(same.mean_de76 == 0.0 && same.p95_de76 == 0.0 && same.mse == 0.0);
    const SceneColorReport diff = scene_color_report(codec, half, grey);
    CHECK(diff.mean_de76 > 0.0 && diff.p95_de76 == diff.mean_de76 && rel_close(diff.mse, 0.0625, 1e-12));
    ChannelImage five = grey;
    five.channels = 5;
    five.data.assign(40, 0.1f);
    CHECK_THROWS_AS(exposure_for(codec, five), std::invalid_argument);
    CHECK_THROWS_AS(tonemap_srgb8(dev, five, 1.0), std::invalid_argument);
    ChannelImage wide = grey;
    wide.width = 8;
    wide.height = 1;
    CHECK_THROWS_AS(error_map(codec, grey, ChannelImage{3, 1, 3, std::vector<float>(9, 0.f)}), std::invalid_argument);
    (void)wide;
  }

  // path tracer (renderer.hpp:93-107): multipass == single latent render at fixed depth,
  // path hashes identical across modes, counters in native units, invalid jobs rejected.
  {
    const int n = codec.n();
    Scene sc;
    sc.materials.push_back(SpectralCurve(n, 0.7));
    SpectralCurve red(n, 0.0);
    for (int i = 0; i < n; ++i) red[i] = 0.1 + 0.5 * i / n;
    sc.materials.push_back(red);
    sc.wall_material = {1, 0, 0, 0, 0, -1};
    SceneObject sphere;
    sphere.center = {0.3, 0.4, -0.2};
    sphere.radius = 0.35;
    sc.objects.push_back(sphere);
    SceneLight light;
    light.corner = {-0.25, 1.999, -0.25};
    light.edge_u = {0.5, 0.0, 0.0};
    light.edge_v = {0.0, 0.0, 0.5};
    light.spd = SpectralCurve(n, 1.0);
    light.scale = 12.0;
    sc.lights.push_back(light);
    RenderJob job;
    job.width = 24;
    job.height = 16;
    job.spp = 4;
    job.collect_path_hashes = true;
    job.mode = RenderMode::latent;
    const ChannelImage lat = render(codec, sc, job);
    const ChannelImage mp = render_latent_multipass(codec, sc, job);
    CHECK(lat.channels == codec.k() && lat.data == mp.data && lat.path_hashes == mp.path_hashes);
    job.mode = RenderMode::spectral;
    const ChannelImage spec = render(codec, sc, job);
    job.mode = RenderMode::rgb;
    const ChannelImage rgb = render(codec, sc, job);
    CHECK(spec.channels == n && rgb.channels == 3);
    CHECK(spec.path_hashes == lat.path_hashes && rgb.path_hashes == lat.path_hashes);
    CHECK(spec.shading_evals == rgb.shading_evals * static_cast<uint64_t>(n) && lat.shading_evals == rgb.shading_evals * 2);
    job.spp = 0;
    CHECK_THROWS_AS(render(codec, sc, job), std::invalid_argument);
    job.spp = 2;
    sc.wall_material[4] = 9;
    CHECK_THROWS_AS(render(codec, sc, job), std::invalid_argument);
  }

  {  // the reference's upsampler (upsampler.cpp:42-72, :170-190) against plain fp64 loops here
    UpsamplerWeights uw;
    uw.k = 6;
    uw.hidden = 24;
    uint64_t us = 7;
    auto fill = [&](std::vector<double>& v, size_t n, double scale) {
      v.resize(n);
      for (double& x : v) x = scale * (2.0 * lcg(us) - 1.0);
    };
    fill(uw.w1, 24 * 3, 0.8);
    fill(uw.b1, 24, 0.1);
    fill(uw.w2, 24 * 24, 0.4);
    fill(uw.b2, 24, 0.1);
    fill(uw.w3, 6 * 24, 0.5);
    fill(uw.b3, 6, 0.1);
    Upsampler up(dev, uw);
    auto silu = [](double x) { return x * (1.0 / (1.0 + std::exp(-x))); };
    std::uint64_t clamped = 0, want_clamped = 0;
    for (int t = 0; t < 16; ++t) {
      const std::array<double, 3> rgb{lcg(us), lcg(us), lcg(us)};
      double h1[24], h2[24];
      for (int i = 0; i < 24; ++i) {
        double a = uw.b1[i];
        for (int j = 0; j < 3; ++j) a += uw.w1[i * 3 + j] * rgb[j];
        h1[i] = silu(a);
      }
      for (int i = 0; i < 24; ++i) {
        double a = uw.b2[i];
        for (int j = 0; j < 24; ++j) a += uw.w2[i * 24 + j] * h1[j];
        h2[i] = silu(a);
      }
      const LatentCode raw = upsample_raw(up, rgb);
      const LatentCode z = upsample(up, rgb, &clamped);
      for (int i = 0; i < 6; ++i) {
        double a = uw.b3[i];
        for (int j = 0; j < 24; ++j) a += uw.w3[i * 24 + j] * h2[j];
        CHECK(rel_close(raw[i], a, 1e-13));
        CHECK(z[i] == (raw[i] < 0.0 ? 0.0 : raw[i]));
        if (raw[i] < 0.0) ++want_clamped;
      }
    }
    CHECK(clamped == want_clamped && want_clamped > 0);
    uw.w2[5] = std::nan("");
    CHECK_THROWS_AS(Upsampler(dev, uw), std::invalid_argument);
  }

  {  // spectra CSV round trip with and without ids, malformed files (test_io.cpp:43-86)
    const std::string path = "/tmp/hc_b200_dropin_spectra.csv";
    std::vector<SpectralCurve> curves(2, SpectralCurve(47));
    for (int i = 0; i < 47; ++i) {
      const double l = g47.wavelength_at(i);
      curves[0][i] = 0.8 * std::exp(-0.5 * (l - 550.0) * (l - 550.0) / (40.0 * 40.0));
      curves[1][i] = 0.25;
    }
    write_spectra_csv(dev, path, {"a", "b"}, curves);
    const SpectraCsv back = read_spectra_csv(dev, path);
    CHECK(back.rows.size() == 2u && back.wavelengths.size() == 47u);
    CHECK(back.ids == std::vector<std::string>({"a", "b"}));
    CHECK(back.wavelengths[0] == 368.0);
    for (int i = 0; i < 47; ++i) CHECK(rel_close(back.rows[0][static_cast<size_t>(i)], curves[0][i], 1e-8));
    write_spectra_csv(dev, path, {}, curves);
    const SpectraCsv noid = read_spectra_csv(dev, path);
    CHECK(noid.ids.empty() && noid.rows.size() == 2u);
    auto put = [&](const char* t) {
      FILE* f = std::fopen(path.c_str(), "wb");
      std::fputs(t, f);
      std::fclose(f);
    };
    put("");
    CHECK_THROWS_AS(read_spectra_csv(dev, path), FormatError);
    put("400,500\n0.5\n");  // row shorter than header
    CHECK_THROWS_AS(read_spectra_csv(dev, path), FormatError);
    put("400,500\n0.5,abc\n");  // non-numeric value
    CHECK_THROWS_AS(read_spectra_csv(dev, path), FormatError);
    CHECK_THROWS_AS(read_spectra_csv(dev, "/nonexistent/dir/spectra.csv"), FormatError);
    std::remove(path.c_str());
  }

  {  // codes CSV round trip and validation (test_io.cpp:133-155)
    const std::string path = "/tmp/hc_b200_dropin_codes.csv";
    LatentCode a, b;
    a.z = {0.1, 0.25, 1.0 / 3.0, 0.0, 5e-17, 2.0};
    b.z = {1, 2, 3, 4, 5, 6};
    write_codes_csv(dev, path, {"x", "y"}, {a, b});
    const CodesCsv back = read_codes_csv(dev, path);
    CHECK(back.codes.size() == 2u);
    CHECK(back.ids.size() == 2u && back.ids[0] == "x" && back.ids[1] == "y");
    CHECK(back.codes[0].k() == 6);
    for (int i = 0; i < 6; ++i) {
      CHECK(back.codes[0][i] == a[i]);  // %.17g round-trips doubles bit-exactly
      CHECK(back.codes[1][i] == b[i]);
    }
    auto write_text = [&](const char* t) {
      FILE* f = std::fopen(path.c_str(), "wb");
      std::fputs(t, f);
      std::fclose(f);
    };
    write_text("id,c0,c9\nx,1,2\n");  // wrong column labels
    CHECK_THROWS_AS(read_codes_csv(dev, path), FormatError);
    write_text("id,c0,c1\nx,1\n");  // short row
    CHECK_THROWS_AS(read_codes_csv(dev, path), FormatError);
    LatentCode c;
    c.z = {1, 2};
    CHECK_THROWS_AS(write_codes_csv(dev, path, {"x", "y"}, {a, c}), FormatError);  // inconsistent dimensions
    CHECK_THROWS_AS(write_codes_csv(dev, path, {"x"}, {a, b}), FormatError);       // id count
    CHECK_THROWS_AS(read_codes_csv(dev, "/nonexistent/dir/codes.csv"), FormatError);
    std::remove(path.c_str());
  }

  std::printf("drop-in: %d checks, %d failures, %lld kernel launches\n", g_checks, g_fail,
              static_cast<long long>(dev.launches()));
  return g_fail ? 1 : 0;
}
