// Weight-file round trip through the C++ drop-in (no GPU needed): load <in>, save <out>.
// Exit 0 on success, 3 when load threw FormatError (message on stderr), 1 otherwise.
#include <cstdio>
#include <exception>

#include "hadacodec_b200.hpp"

int main(int argc, char** argv) {
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
