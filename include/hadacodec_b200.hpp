// hadacodec-b200 — C++ drop-in host API for the reference's per-pixel codec /
// latent-shading path, over the C ABI (include/hadacodec_b200.h).
//
// Mirrors the reference's public headers (/root/reference/proj/core/include/
// hadacodec/{codec,colorimetry,renderer}.hpp): same type and function names,
// argument meaning and exception types (std::invalid_argument, std::domain_error),
// in namespace hadacodec::b200 so both libraries can be linked side by side.
// Differences a caller should know:
//   * the grid is a runtime property (n = 47 reference grid, or 81 = BASELINE grid)
//     instead of the compile-time kSampleCount, so SpectralCurve is a vector;
//   * the batched / image calls compute in fp32 on the GPU (reference: fp64), agreeing to
//     ~1e-6 relative; the by-value encode / decode and the file tools' paths run fp64
//     kernels in the reference's operation order and are bit-identical;
//   * every call runs on a Device (one per GPU, one CUDA stream); the by-value
//     calls copy in and out and synchronise, the *_batch / shade_* calls take
//     whole images — the form the hot path should use.
#pragma once

#include <array>
#include <cstddef>
#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <string_view>
#include <vector>

#include "hadacodec_b200.h"

namespace hadacodec {
namespace b200 {

// spectrum.hpp:10-21 — the reference's canonical grid (source compatibility: the
// reference-signature overloads below default to it; the BASELINE grid is Grid::baseline81).
inline constexpr int kSampleCount = 47;
inline constexpr double kLambdaMin = 368.0;
inline constexpr double kLambdaMax = 830.0;
inline constexpr double kLambdaStep = (kLambdaMax - kLambdaMin) / (kSampleCount - 1);
inline constexpr double kActiveBandMin = 400.0;
inline constexpr double kActiveBandMax = 700.0;
constexpr double wavelength_at(int i) { return kLambdaMin + kLambdaStep * i; }

// spectrum.hpp:10-21 — runtime grid.
struct Grid {
  int n = 81;
  double lambda_min = 380.0;
  double lambda_step = 5.0;
  double wavelength_at(int i) const { return lambda_min + lambda_step * i; }
  static Grid reference47();  // 368..830 nm, 47 samples (the reference's kSampleCount)
  static Grid baseline81();   // 380..780 nm, 81 samples (BASELINE.json)
  static Grid for_samples(int n);
};

// spectrum.hpp:25-39.  Default-constructed curves have the reference's kSampleCount zero
// samples (as its std::array); SpectralCurve(81) is a curve on the BASELINE grid.
struct SpectralCurve {
  std::vector<double> v;
  SpectralCurve() : v(static_cast<size_t>(kSampleCount), 0.0) {}
  explicit SpectralCurve(int n, double value = 0.0) : v(static_cast<size_t>(n), value) {}
  int size() const { return static_cast<int>(v.size()); }
  double& operator[](int i) { return v[static_cast<size_t>(i)]; }
  const double& operator[](int i) const { return v[static_cast<size_t>(i)]; }
  static SpectralCurve flat(double value) { return SpectralCurve(kSampleCount, value); }
  static SpectralCurve zero() { return SpectralCurve(); }
  static SpectralCurve ones() { return flat(1.0); }
  double max_value() const {
    double m = v.empty() ? 0.0 : v[0];
    for (double x : v) m = x > m ? x : m;
    return m;
  }
  double sum() const {
    double t = 0.0;
    for (double x : v) t += x;
    return t;
  }
};

// codec.hpp:14-22
struct LatentCode {
  std::vector<double> z;
  int k() const { return static_cast<int>(z.size()); }
  double& operator[](int i) { return z[static_cast<size_t>(i)]; }
  const double& operator[](int i) const { return z[static_cast<size_t>(i)]; }
};

// codec.hpp:24-29
struct CodecTrainingMeta {
  std::uint64_t seed = 0;
  std::array<double, 5> lambda_weights{};  // e2e, rec, code, col, alg
  int epochs = 0;
};

// codec.hpp:34-43
struct CodecWeights {
  int k = 6;
  int n = kSampleCount;
  double beta = 10.0;
  std::vector<double> raw_enc;  // k x n
  std::vector<double> raw_dec;  // n x k
  CodecTrainingMeta meta;
  int blocks() const { return k / 3; }
};

// codec.hpp:52-58
struct EffectiveWeights {
  int k = 0;
  int n = 0;
  std::vector<double> enc;  // k x n
  std::vector<double> dec;  // n x k
};

// colorimetry.hpp:9-22
enum class ColorSpace { XYZ, LinearRGB, Lab };
struct ColorTriple {
  ColorSpace space = ColorSpace::XYZ;
  std::array<double, 3> c{};
  double& operator[](int i) { return c[static_cast<size_t>(i)]; }
  const double& operator[](int i) const { return c[static_cast<size_t>(i)]; }
};

// renderer.hpp:73-89 (row-major y, x, channel)
struct ChannelImage {
  int width = 0, height = 0, channels = 0;
  std::vector<float> data;
  std::uint64_t shading_evals = 0;          // render: shading units (renderer.hpp:78-81)
  std::vector<std::uint64_t> path_hashes;   // render with collect_path_hashes
  float& at(int x, int y, int c) { return data[(static_cast<size_t>(y) * width + x) * channels + c]; }
  float at(int x, int y, int c) const { return data[(static_cast<size_t>(y) * width + x) * channels + c]; }
};

// One GPU + one CUDA stream (hc_ctx).  Non-copyable; owns device scratch.
class Device {
 public:
  explicit Device(int device = 0, void* stream = nullptr);
  ~Device();
  Device(const Device&) = delete;
  Device& operator=(const Device&) = delete;
  hc_ctx handle() const { return ctx_; }
  void synchronize();  // throws the latched device-side violations
  int64_t launches() const;

 private:
  hc_ctx ctx_ = nullptr;
};

// A codec resident on a Device: E, D and the folded 3 x k XYZ projection.
class Codec {
 public:
  Codec(Device& dev, const EffectiveWeights& w, const Grid& grid);
  Codec(Device& dev, const CodecWeights& w, const Grid& grid);  // softplus on the host
  ~Codec();
  Codec(const Codec&) = delete;
  Codec& operator=(const Codec&) = delete;
  hc_codec handle() const { return codec_; }
  int k() const { return k_; }
  int n() const { return n_; }
  const Grid& grid() const { return grid_; }
  Device& device() const { return *dev_; }

 private:
  Device* dev_;
  hc_codec codec_ = nullptr;
  int k_ = 0, n_ = 0;
  Grid grid_;
};

// ---- codec.hpp:46-82
double softplus(double raw, double beta);
double softplus_derivative(double raw, double beta);
EffectiveWeights effective_weights(const CodecWeights& w);
void validate(const CodecWeights& w, const Grid& grid);
// By-value encode / decode run the fp64 kernels: bit-identical to the reference's.
LatentCode encode(const Codec& c, const SpectralCurve& s);
SpectralCurve decode(const Codec& c, const LatentCode& z);  // throws std::domain_error on negative codes
// resample (spectrum.cpp:60-98) of curves given on `wavelengths` onto the codec's grid, then
// encode — run_encode's per-curve step for a whole file at once, fp64, bit-identical.
std::vector<LatentCode> encode_resampled(const Codec& c, const std::vector<double>& wavelengths,
                                         const std::vector<std::vector<double>>& rows, bool zero_outside = true);
LatentCode blockwise_hadamard(const LatentCode& a, const LatentCode& b);
std::vector<std::array<double, 3>> split_blocks(const LatentCode& z);
LatentCode join_blocks(const std::vector<std::array<double, 3>>& blocks);

// ---- upsampler.hpp:13-50: the reference's fp64 RGB -> code network (3 -> hidden -> hidden
// -> k, SiLU, identity head) on the GPU; results within ~1e-15 relative of the reference
// (SiLU's exp is CUDA's).
struct UpsamplerWeights {
  int k = 6;
  int hidden = 128;
  std::vector<double> w1, b1;  // hidden x 3, hidden
  std::vector<double> w2, b2;  // hidden x hidden, hidden
  std::vector<double> w3, b3;  // k x hidden, k
  CodecTrainingMeta meta;
};
void validate(const UpsamplerWeights& w);  // std::invalid_argument, as upsampler.cpp:130-144
class Upsampler {
 public:
  Upsampler(Device& dev, const UpsamplerWeights& w);
  ~Upsampler();
  Upsampler(const Upsampler&) = delete;
  Upsampler& operator=(const Upsampler&) = delete;
  hc_upsampler handle() const { return up_; }
  int k() const { return k_; }
  Device& device() const { return *dev_; }

 private:
  Device* dev_;
  hc_upsampler up_ = nullptr;
  int k_ = 0;
};
LatentCode upsample_raw(const Upsampler& u, const std::array<double, 3>& linear_rgb);
LatentCode upsample(const Upsampler& u, const std::array<double, 3>& linear_rgb,
                    std::uint64_t* clamped_entries = nullptr);
// A whole texture at once (the form the tools should use): rows of (r, g, b) -> codes.
std::vector<LatentCode> upsample_batch(const Upsampler& u, const std::vector<std::array<double, 3>>& linear_rgb,
                                       std::uint64_t* clamped_entries = nullptr);

// ---- batched codec (row-major host buffers; rows x n spectra, rows x k codes)
std::vector<float> encode_batch(const Codec& c, const std::vector<float>& spectra);
struct RoundTrip {
  std::vector<float> codes, spectra, xyz, rgb;
};
RoundTrip roundtrip_batch(const Codec& c, const std::vector<float>& spectra);

// ---- colorimetry.hpp:45-56 (radiance convention, IEC sRGB), computed on the GPU
ColorTriple spectrum_to_xyz(const Codec& c, const SpectralCurve& s);
ColorTriple xyz_to_linear_rgb(const ColorTriple& xyz);

// ---- renderer.hpp:109-115
ChannelImage decode_image(const Codec& c, const ChannelImage& latent);   // k -> n channels
ChannelImage image_to_linear_rgb(const Codec& c, const ChannelImage& img);  // n -> 3 channels

// ---- path tracer (renderer.hpp:12-107), computed on the GPU
struct Vec3 {
  double x = 0, y = 0, z = 0;
};
struct Camera {
  Vec3 position{0, 1, 3.25};
  Vec3 look_at{0, 1, 0};
  Vec3 up{0, 1, 0};
  double vfov_degrees = 40.0;
};
struct SceneLight {
  Vec3 corner, edge_u, edge_v;
  SpectralCurve spd;
  double scale = 1.0;
};
struct SceneObject {
  enum class Kind { sphere, block };
  Kind kind = Kind::sphere;
  Vec3 center;
  double radius = 0;
  Vec3 box_min, box_max;
  int material = 0;
};
struct Scene {
  Camera camera;
  Vec3 box_min{-1, 0, -1}, box_max{1, 2, 1};
  std::array<int, 6> wall_material{-1, -1, -1, -1, -1, -1};
  std::vector<SpectralCurve> materials;
  std::vector<SceneObject> objects;
  std::vector<SceneLight> lights;
};
enum class RenderMode { spectral, latent, rgb };
struct RenderJob {
  RenderMode mode = RenderMode::spectral;
  int width = 128, height = 128, spp = 64, max_depth = 3;
  std::uint64_t seed = 0;
  bool collect_path_hashes = false;
};
// The codec supplies the grid (and, in latent mode, the codes).
ChannelImage render(const Codec& c, const Scene& scene, const RenderJob& job);
ChannelImage render_latent_multipass(const Codec& c, const Scene& scene, const RenderJob& job);

// ---- colour-metric tail (renderer.hpp:117-133, evaluation.hpp:48-59), computed on the GPU.
// Images are linear RGB (3 channels) or spectra (n channels), as in the reference.
double exposure_for(const Codec& c, const ChannelImage& img, double percentile = 99.5);
std::vector<unsigned char> tonemap_srgb8(Device& dev, const ChannelImage& linear_rgb, double exposure);
struct ErrorMap {  // renderer.hpp:127-131
  int width = 0, height = 0;
  std::vector<float> mse;
  double mean_mse = 0;
};
ErrorMap error_map(const Codec& c, const ChannelImage& a, const ChannelImage& b);
struct SceneColorReport {  // evaluation.hpp:50-55
  double mean_de76 = 0;
  double p95_de76 = 0;
  double mse = 0;
  double exposure = 0;
};
SceneColorReport scene_color_report(const Codec& c, const ChannelImage& ground_truth, const ChannelImage& test);

// ---- codes CSV (io.hpp:19-23, :48-56): %.17g formatting and strtod parsing on the GPU,
// byte-identical files / bit-identical values.  Malformed input raises FormatError with
// the path and the first bad line, as the reference does (the message text differs); a
// ragged code set is rejected before anything is written.
class FormatError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};
struct CodesCsv {
  std::vector<std::string> ids;
  std::vector<LatentCode> codes;
};
CodesCsv read_codes_csv(Device& dev, const std::string& path);
// Codec weight files (io.hpp:62-66, JSON): byte-identical to the reference's (same library,
// nlohmann::json dump(2)); FormatError for unreadable / malformed / invalid files.
CodecWeights load_codec_weights(const std::string& path);
void save_codec_weights(const std::string& path, const CodecWeights& w);
UpsamplerWeights load_upsampler_weights(const std::string& path);  // io.cpp:405-431
void save_upsampler_weights(const std::string& path, const UpsamplerWeights& w);  // io.cpp:433-445
// HCF1 raw channel images and binary PPM (io.hpp:71-84), same checks and FormatError causes.
ChannelImage read_raw_image(const std::string& path);
void write_raw_image(const std::string& path, const ChannelImage& img);
struct Ppm8 {
  int width = 0, height = 0;
  std::vector<unsigned char> rgb;
};
void write_ppm(const std::string& path, int width, int height, const std::vector<unsigned char>& rgb8);
Ppm8 read_ppm(const std::string& path);
// Spectra CSV (io.hpp:26-40): %.9g writer and exact reader on the GPU.  The writer's grid is
// the curves' (Grid::for_samples(curve size)); ids empty = no id column.
struct SpectraCsv {
  std::vector<double> wavelengths;
  std::vector<std::string> ids;  // empty when the file has no id column
  std::vector<std::vector<double>> rows;
};
SpectraCsv read_spectra_csv(Device& dev, const std::string& path);
void write_spectra_csv(Device& dev, const std::string& path, const std::vector<std::string>& ids,
                       const std::vector<SpectralCurve>& curves);
void write_codes_csv(Device& dev, const std::string& path, const std::vector<std::string>& ids,
                     const std::vector<LatentCode>& codes);

// ---- G-buffer latent shading (configs 2/3): one frame, host buffers.
struct GBuffer {
  int width = 0, height = 0, lights = 0;
  std::vector<uint32_t> palette_index;  // width * height
  std::vector<float> cos_terms;         // width * height * lights
};
struct ShadedFrame {
  ChannelImage latent;   // k channels (reassembled k/3 passes)
  ChannelImage xyz;      // 3 channels
  ChannelImage linear_rgb;
};
// palette_codes: n_pal x k, light_codes: L x k (e.g. from encode_batch on the assets,
// as compile_scene does, renderer.cpp:201-225).
ShadedFrame shade_latent(const Codec& c, const std::vector<float>& palette_codes,
                         const std::vector<float>& light_codes, const GBuffer& g);
// A stream of frames of one scene through the host-buffer pipeline
// (hc_shade_latent_host_frames): xyz and linear_rgb of every frame (latent left empty),
// identical to shade_latent frame by frame.
std::vector<ShadedFrame> shade_latent_frames(const Codec& c, const std::vector<float>& palette_codes,
                                             const std::vector<float>& light_codes,
                                             const std::vector<GBuffer>& frames);
// Naive n-sample path on the same G-buffer (palette_spectra n_pal x n, light_spectra L x n).
ShadedFrame shade_spectral(const Codec& c, const std::vector<float>& palette_spectra,
                           const std::vector<float>& light_spectra, const GBuffer& g);

// ===================================================================== reference signatures
// The reference's free functions with its exact signatures (codec.hpp:60-78,
// colorimetry.hpp:47-55, renderer.hpp:100-133, upsampler.hpp:32-40, spectrum.hpp:42-72,
// rng.hpp), so code written against `hadacodec` compiles against `hadacodec::b200` with only
// the namespace changed.  The GPU work runs on a per-thread default Device (CUDA device
// HADACODEC_B200_DEVICE, default 0) with codecs / upsamplers cached by the weights they were
// built from (a small per-thread LRU keyed by the weight arrays), so repeated calls with the
// same weights pay the upload once.  Grids come from the curves / weights (47 or 81 samples).
Device& default_device();

// ---- spectrum.hpp:42-72 (host value helpers)
bool curve_is_valid(const SpectralCurve& s, bool reflectance = false);
SpectralCurve scale(const SpectralCurve& s, double alpha);  // std::domain_error for alpha < 0 / non-finite
SpectralCurve add(const SpectralCurve& a, const SpectralCurve& b);
SpectralCurve hadamard(const SpectralCurve& a, const SpectralCurve& b);
SpectralCurve resample(const std::vector<double>& source_wavelengths, const std::vector<double>& source_values,
                       bool zero_outside_active_band);  // onto the kSampleCount grid
void zero_outside_active_band(SpectralCurve& s);
SpectralCurve gaussian_curve(double center_nm, double sigma_nm, double amplitude);

// ---- rng.hpp: the reference's deterministic streams (xoshiro256++ seeded by splitmix64)
std::uint64_t fnv1a64(const void* data, std::size_t size, std::uint64_t basis = 0xcbf29ce484222325ull);
std::uint64_t splitmix64_next(std::uint64_t& state);
class Rng {
 public:
  explicit Rng(std::uint64_t seed);
  static Rng stream(std::uint64_t seed, std::string_view purpose);
  static Rng pixel_stream(std::uint64_t seed, int x, int y, int sample, std::uint32_t lane);
  std::uint64_t next_u64();
  double uniform();
  double uniform(double a, double b);
  double log_uniform(double a, double b);
  std::uint32_t index(std::uint32_t n);
  double normal();

 private:
  std::uint64_t s_[4];
  double cached_normal_ = 0.0;
  bool has_cached_normal_ = false;
};

// ---- codec.hpp:60-78
void validate(const CodecWeights& w);  // n must be a supported grid (47 or 81)
LatentCode encode(const EffectiveWeights& w, const SpectralCurve& s);
LatentCode encode(const CodecWeights& w, const SpectralCurve& s);
SpectralCurve decode(const EffectiveWeights& w, const LatentCode& z);  // std::domain_error on negative codes
SpectralCurve decode(const CodecWeights& w, const LatentCode& z);

// ---- colorimetry.hpp:25-77.  spectrum_to_xyz / xyz_of_reflectance run the fp64 GPU kernel
// (hc_spectra_to_xyz_f64, the reference's summation order); CmfTable is the grid's tabulated
// CIE 1931 / D65 rows (package data, tools/make_cmf_tables.py); the scalar Lab / Delta E / sRGB
// helpers are the reference's formulas on one value (their per-pixel batched forms run on the
// GPU in hc_scene_color_report / hc_delta_e94_report).
class CmfTable {
 public:
  static const CmfTable& instance();       // the reference grid (kSampleCount = 47)
  static const CmfTable& for_grid(int n);  // 47 or 81
  const SpectralCurve& xbar() const { return xbar_; }
  const SpectralCurve& ybar() const { return ybar_; }
  const SpectralCurve& zbar() const { return zbar_; }
  const SpectralCurve& d65() const { return d65_; }
  const SpectralCurve& wx() const { return wx_; }  // D65-weighted rows, unit reflectance -> Y = 100
  const SpectralCurve& wy() const { return wy_; }
  const SpectralCurve& wz() const { return wz_; }
  ColorTriple white_xyz() const;

 private:
  explicit CmfTable(int n);
  SpectralCurve xbar_, ybar_, zbar_, d65_, wx_, wy_, wz_;
};
ColorTriple spectrum_to_xyz(const SpectralCurve& s);     // radiance convention, on the curve's grid
ColorTriple xyz_of_reflectance(const SpectralCurve& r);  // reflectance convention
ColorTriple linear_rgb_to_xyz(const ColorTriple& rgb);
ColorTriple srgb_reference_white();
ColorTriple xyz_to_lab(const ColorTriple& xyz, const ColorTriple& white);  // std::domain_error: white <= 0
double delta_e76(const ColorTriple& lab_a, const ColorTriple& lab_b);
double delta_e94(const ColorTriple& lab_reference, const ColorTriple& lab_sample);
double srgb_encode(double linear);
double srgb_decode(double encoded);

// ---- renderer.hpp:100-133
ChannelImage render(const Scene& scene, const RenderJob& job, const CodecWeights* codec = nullptr);
ChannelImage render_latent_multipass(const Scene& scene, const RenderJob& job, const CodecWeights& codec);
ChannelImage decode_image(const ChannelImage& latent, const CodecWeights& w);
ChannelImage image_to_linear_rgb(const ChannelImage& img);
double exposure_for(const ChannelImage& img, double percentile = 99.5);
std::vector<unsigned char> tonemap_srgb8(const ChannelImage& linear_rgb, double exposure);
ErrorMap error_map(const ChannelImage& a, const ChannelImage& b);

// ---- upsampler.hpp:32-40
LatentCode upsample_raw(const UpsamplerWeights& w, const std::array<double, 3>& linear_rgb);
LatentCode upsample(const UpsamplerWeights& w, const std::array<double, 3>& linear_rgb,
                    std::uint64_t* clamped_entries = nullptr);

}  // namespace b200
}  // namespace hadacodec
