// Weight-file round trip through the C++ drop-in (no GPU needed): load <in>, save <out>
// (codec weights; with a leading "upsampler" argument, upsampler weights).
// Exit 0 on success, 3 when load threw FormatError (message on stderr), 1 otherwise.
#include <cstdio>
#include <exception>
#include <string>

#include "hadacodec_b200.hpp"

int main(int argc, char** argv) {
  if (argc == 4 && std::string(argv[1]) == "upsampler") {
    try {
      const hadacodec::b200::UpsamplerWeights w = hadacodec::b200::load_upsampler_weights(argv[2]);
      hadacodec::b200::save_upsampler_weights(argv[3], w);
      std::printf("k=%d hidden=%d epochs=%d\n", w.k, w.hidden, w.meta.epochs);
      return 0;
    } catch (const hadacodec::b200::FormatError& e) {
      std::fprintf(stderr, "FormatError: %s\n", e.what());
      return 3;
    } catch (const std::exception& e) {
      std::fprintf(stderr, "error: %s\n", e.what());
      return 1;
    }
  }
  if (argc != 3) return 1;
  try {
    const hadacodec::b200::CodecWeights w = hadacodec::b200::load_codec_weights(argv[1]);
    hadacodec::b200::save_codec_weights(argv[2], w);
    std::printf("k=%d n=%d beta=%.17g epochs=%d\n", w.k, w.n, w.beta, w.meta.epochs);
    return 0;
  } catch (const hadacodec::b200::FormatError& e) {
    std::fprintf(stderr, "FormatError: %s\n", e.what());
    return 3;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 1;
  }
}
