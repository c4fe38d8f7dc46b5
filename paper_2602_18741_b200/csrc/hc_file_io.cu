// hadacodec-b200: the reference's small file formats for the C++ drop-in layer (SURVEY.md
// §8f row 3).  Host code only — none of them has per-element work:
//   * codec weight files (io.cpp:331-403): a few kilobytes of JSON per codec.  The reference
//     serialises with nlohmann::json (`dump(2)`, keys in the library's sorted order, its
//     shortest round-trip number format); the same library is used here, so a saved file is
//     byte-identical to the reference's and every reference file loads to the same doubles;
//   * HCF1 raw channel images and binary PPM (io.cpp:450-536): a header and a raw payload.
#include <algorithm>
#include <cerrno>
#include <cctype>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <iterator>
#include <stdexcept>
#include <string>
#include <vector>

#include "hadacodec_b200.hpp"

#if HC_HAVE_NLOHMANN_JSON
#include "nlohmann/json.hpp"
#endif

namespace hadacodec {
namespace b200 {

namespace {
constexpr const char* kToolVersion = "1.0.0";  // io.hpp:17
}  // namespace

#if HC_HAVE_NLOHMANN_JSON
using nlohmann::json;

CodecWeights load_codec_weights(const std::string& path) {  // io.cpp:370-393
  std::ifstream f(path);
  if (!f) throw FormatError(path + ": cannot open for reading");
  json j;
  try {
    j = json::parse(f);
  } catch (const json::exception& e) {
    throw FormatError(path + ": JSON parse error: " + e.what());
  }
  CodecWeights w;
  try {
    if (j.at("format").get<std::string>() != "codec-weights") throw FormatError(path + ": not a codec weights file");
    w.k = j.at("k").get<int>();
    w.n = j.at("n").get<int>();
    w.beta = j.at("beta").get<double>();
    w.raw_enc = j.at("raw_enc").get<std::vector<double>>();
    w.raw_dec = j.at("raw_dec").get<std::vector<double>>();
    if (j.contains("meta")) {
      const json& m = j.at("meta");
      w.meta.seed = m.at("seed").get<std::uint64_t>();
      const auto lw = m.at("lambda_weights").get<std::vector<double>>();
      if (lw.size() != w.meta.lambda_weights.size())
        throw FormatError("weights file: lambda_weights must have 5 entries");
      for (size_t i = 0; i < lw.size(); ++i) w.meta.lambda_weights[i] = lw[i];
      w.meta.epochs = m.at("epochs").get<int>();
    }
  } catch (const json::exception& e) {
    throw FormatError(path + ": bad codec weights: " + e.what());
  }
  try {
    validate(w, Grid::for_samples(w.n));
  } catch (const std::invalid_argument& e) {
    throw FormatError(path + ": " + e.what());
  }
  return w;
}

void save_codec_weights(const std::string& path, const CodecWeights& w) {  // io.cpp:395-403
  validate(w, Grid::for_samples(w.n));
  const json meta{{"seed", w.meta.seed}, {"lambda_weights", w.meta.lambda_weights}, {"epochs", w.meta.epochs}};
  const json j{{"format", "codec-weights"}, {"version", kToolVersion}, {"k", w.k}, {"n", w.n}, {"beta", w.beta},
               {"raw_enc", w.raw_enc}, {"raw_dec", w.raw_dec}, {"meta", meta}};
  std::ofstream f(path);
  if (!f) throw FormatError(path + ": cannot open for writing");
  f << j.dump(2) << '\n';
  f.flush();
  if (!f.good()) throw FormatError(path + ": write failed");
}

UpsamplerWeights load_upsampler_weights(const std::string& path) {  // io.cpp:405-431
  std::ifstream f(path);
  if (!f) throw FormatError(path + ": cannot open for reading");
  json j;
  try {
    j = json::parse(f);
  } catch (const json::exception& e) {
    throw FormatError(path + ": JSON parse error: " + e.what());
  }
  UpsamplerWeights w;
  try {
    if (j.at("format").get<std::string>() != "upsampler-weights")
      throw FormatError(path + ": not an upsampler weights file");
    w.k = j.at("k").get<int>();
    w.hidden = j.at("hidden").get<int>();
    w.w1 = j.at("w1").get<std::vector<double>>();
    w.b1 = j.at("b1").get<std::vector<double>>();
    w.w2 = j.at("w2").get<std::vector<double>>();
    w.b2 = j.at("b2").get<std::vector<double>>();
    w.w3 = j.at("w3").get<std::vector<double>>();
    w.b3 = j.at("b3").get<std::vector<double>>();
    if (j.contains("meta")) {
      const json& m = j.at("meta");
      w.meta.seed = m.at("seed").get<std::uint64_t>();
      const auto lw = m.at("lambda_weights").get<std::vector<double>>();
      if (lw.size() != w.meta.lambda_weights.size())
        throw FormatError("weights file: lambda_weights must have 5 entries");
      for (size_t i = 0; i < lw.size(); ++i) w.meta.lambda_weights[i] = lw[i];
      w.meta.epochs = m.at("epochs").get<int>();
    }
  } catch (const json::exception& e) {
    throw FormatError(path + ": bad upsampler weights: " + e.what());
  }
  try {
    validate(w);
  } catch (const std::invalid_argument& e) {
    throw FormatError(path + ": " + e.what());
  }
  return w;
}

void save_upsampler_weights(const std::string& path, const UpsamplerWeights& w) {  // io.cpp:433-445
  validate(w);
  const json meta{{"seed", w.meta.seed}, {"lambda_weights", w.meta.lambda_weights}, {"epochs", w.meta.epochs}};
  const json j{{"format", "upsampler-weights"}, {"version", kToolVersion}, {"k", w.k}, {"hidden", w.hidden},
               {"w1", w.w1}, {"b1", w.b1}, {"w2", w.w2}, {"b2", w.b2}, {"w3", w.w3}, {"b3", w.b3}, {"meta", meta}};
  std::ofstream f(path);
  if (!f) throw FormatError(path + ": cannot open for writing");
  f << j.dump(2) << '\n';
  f.flush();
  if (!f.good()) throw FormatError(path + ": write failed");
}

#else

UpsamplerWeights load_upsampler_weights(const std::string& path) {
  throw FormatError(path + ": built without nlohmann/json (weight files unavailable)");
}
void save_upsampler_weights(const std::string& path, const UpsamplerWeights&) {
  throw FormatError(path + ": built without nlohmann/json (weight files unavailable)");
}

CodecWeights load_codec_weights(const std::string& path) {
  throw FormatError(path + ": built without nlohmann/json (weight files unavailable)");
}
void save_codec_weights(const std::string& path, const CodecWeights&) {
  throw FormatError(path + ": built without nlohmann/json (weight files unavailable)");
}

#endif

// ------------------------------------------------------------------ HCF1 raw images (io.cpp:450-492)
ChannelImage read_raw_image(const std::string& path) {
  std::ifstream f(path, std::ios::in | std::ios::binary);
  if (!f) throw FormatError(path + ": cannot open for reading");
  char magic[4];
  if (!f.read(magic, 4) || std::memcmp(magic, "HCF1", 4) != 0) throw FormatError(path + ": bad magic (expected HCF1)");
  std::uint32_t dims[3];
  if (!f.read(reinterpret_cast<char*>(dims), sizeof dims)) throw FormatError(path + ": truncated header");
  ChannelImage img;
  img.width = static_cast<int>(dims[0]);
  img.height = static_cast<int>(dims[1]);
  img.channels = static_cast<int>(dims[2]);
  if (img.width <= 0 || img.height <= 0 || img.channels <= 0 || img.width > 1 << 16 || img.height > 1 << 16 ||
      img.channels > 1024)
    throw FormatError(path + ": implausible image dimensions");
  img.data.resize(static_cast<size_t>(img.width) * img.height * img.channels);
  if (!f.read(reinterpret_cast<char*>(img.data.data()), static_cast<std::streamsize>(img.data.size() * sizeof(float))))
    throw FormatError(path + ": truncated pixel data");
  return img;
}

void write_raw_image(const std::string& path, const ChannelImage& img) {
  if (img.width <= 0 || img.height <= 0 || img.channels <= 0 ||
      img.data.size() != static_cast<size_t>(img.width) * img.height * img.channels)
    throw FormatError(path + ": image dimensions do not match data size");
  std::ofstream f(path, std::ios::out | std::ios::binary);
  if (!f) throw FormatError(path + ": cannot open for writing");
  f.write("HCF1", 4);
  const std::uint32_t dims[3] = {static_cast<std::uint32_t>(img.width), static_cast<std::uint32_t>(img.height),
                                 static_cast<std::uint32_t>(img.channels)};
  f.write(reinterpret_cast<const char*>(dims), sizeof dims);
  f.write(reinterpret_cast<const char*>(img.data.data()), static_cast<std::streamsize>(img.data.size() * sizeof(float)));
  f.flush();
  if (!f.good()) throw FormatError(path + ": write failed");
}

// ------------------------------------------------------------------ binary PPM (io.cpp:494-536)
void write_ppm(const std::string& path, int width, int height, const std::vector<unsigned char>& rgb8) {
  if (rgb8.size() != static_cast<size_t>(width) * height * 3)
    throw FormatError(path + ": pixel buffer does not match dimensions");
  std::ofstream f(path, std::ios::out | std::ios::binary);
  if (!f) throw FormatError(path + ": cannot open for writing");
  f << "P6\n" << width << ' ' << height << "\n255\n";
  f.write(reinterpret_cast<const char*>(rgb8.data()), static_cast<std::streamsize>(rgb8.size()));
  f.flush();
  if (!f.good()) throw FormatError(path + ": write failed");
}

Ppm8 read_ppm(const std::string& path) {
  std::ifstream f(path, std::ios::in | std::ios::binary);
  if (!f) throw FormatError(path + ": cannot open for reading");
  const std::string b((std::istreambuf_iterator<char>(f)), std::istreambuf_iterator<char>());
  size_t p = 0;
  auto token = [&]() {  // operator>> on a std::string: skip whitespace, read to the next
    while (p < b.size() && std::isspace(static_cast<unsigned char>(b[p]))) ++p;
    const size_t s0 = p;
    while (p < b.size() && !std::isspace(static_cast<unsigned char>(b[p]))) ++p;
    return b.substr(s0, p - s0);
  };
  if (token() != "P6") throw FormatError(path + ": expected binary PPM (P6)");
  auto next_token = [&]() {
    for (;;) {
      std::string t = token();
      if (t.empty()) throw FormatError(path + ": truncated PPM header");
      if (t[0] != '#') return t;
      while (p < b.size() && b[p] != '\n') ++p;  // the comment's line (getline)
      if (p < b.size()) ++p;
    }
  };
  auto parse_int = [&](const std::string& t) -> long long {  // std::stoll, fully consumed (io.cpp:90-100)
    errno = 0;
    char* end = nullptr;
    const long long v = std::strtoll(t.c_str(), &end, 10);
    if (end == t.c_str() || errno == ERANGE) throw FormatError(path + ":0: expected an integer, got '" + t + "'");
    if (static_cast<size_t>(end - t.c_str()) != t.size())
      throw FormatError(path + ":0: trailing junk in number '" + t + "'");
    return v;
  };
  Ppm8 img;
  img.width = static_cast<int>(parse_int(next_token()));
  img.height = static_cast<int>(parse_int(next_token()));
  const int maxval = static_cast<int>(parse_int(next_token()));
  if (img.width <= 0 || img.height <= 0 || maxval != 255) throw FormatError(path + ": unsupported PPM header");
  if (p < b.size()) ++p;  // single whitespace after maxval
  const size_t need = static_cast<size_t>(img.width) * img.height * 3;
  if (b.size() - p < need) throw FormatError(path + ": truncated PPM pixel data");  // p <= b.size()
  img.rgb.assign(b.begin() + static_cast<std::ptrdiff_t>(p), b.begin() + static_cast<std::ptrdiff_t>(p + need));
  return img;
}

}  // namespace b200
}  // namespace hadacodec
