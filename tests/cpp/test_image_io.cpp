// HCF1 / PPM through the C++ drop-in (no GPU needed): `raw <in> <out>` or `ppm <in> <out>`
// reads a file and writes it back.  Exit 0 on success, 3 on FormatError, 1 otherwise.
#include <cstdio>
#include <cstring>
#include <exception>

#include "hadacodec_b200.hpp"

using namespace hadacodec::b200;

int main(int argc, char** argv) {
  if (argc != 4) return 1;
  try {
    if (std::strcmp(argv[1], "raw") == 0) {
      const ChannelImage img = read_raw_image(argv[2]);
      write_raw_image(argv[3], img);
      std::printf("%d %d %d\n", img.width, img.height, img.channels);
    } else {
      const Ppm8 img = read_ppm(argv[2]);
      write_ppm(argv[3], img.width, img.height, img.rgb);
      std::printf("%d %d\n", img.width, img.height);
    }
    return 0;
  } catch (const FormatError& e) {
    std::fprintf(stderr, "FormatError: %s\n", e.what());
    return 3;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 1;
  }
}
