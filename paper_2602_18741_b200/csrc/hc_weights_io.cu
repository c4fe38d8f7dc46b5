// hadacodec-b200: codec weight files (io.cpp:331-393) for the C++
// drop-in layer.  Host code only: the files are a few kilobytes of JSON per codec.  The
// reference serialises with nlohmann::json (`dump(2)`, keys in the library's sorted order,
// its shortest round-trip number format); the same library is used here, so a saved file
// is byte-identical to the reference's and every reference file loads to the same doubles.
#include <fstream>
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

#else

CodecWeights load_codec_weights(const std::string& path) {
  throw FormatError(path + ": built without nlohmann/json (weight files unavailable)");
}
void save_codec_weights(const std::string& path, const CodecWeights&) {
  throw FormatError(path + ": built without nlohmann/json (weight files unavailable)");
}

#endif

}  // namespace b200
}  // namespace hadacodec
