// hadacodec-b200: codec kernels — encode, decode(+XYZ/sRGB), fused round trip,
// spectral projection.  Reference: codec.cpp:36-71, renderer.cpp:661-719,
// colorimetry.cpp:75-105.  See hc_ops.cuh (CodecOp) and hc_pipeline.cuh.
#include "hc_launch.cuh"
#include "hc_ops.cuh"

namespace hcb {

// Tile shapes: thread-per-spectrum, TMA-staged.  (T, THREADS, STAGES)
template <int N, int K, int MODE>
struct CodecTile;
template <int N, int K>
struct CodecTile<N, K, kRoundtrip> {
#ifndef HC_RT_T
#define HC_RT_T 64
#endif
#ifndef HC_RT_STAGES
#define HC_RT_STAGES 2
#endif
  static constexpr int T = HC_RT_T, THREADS = HC_RT_T, STAGES = HC_RT_STAGES;
};
template <int N, int K>
struct CodecTile<N, K, kEncode> {
  static constexpr int T = 128, THREADS = 128, STAGES = 3;
};
template <int N, int K>
struct CodecTile<N, K, kDecode> {
  static constexpr int T = 128, THREADS = 128, STAGES = 2;
};
template <int N, int K>
struct CodecTile<N, K, kProject> {
  static constexpr int T = 128, THREADS = 128, STAGES = 3;
};

template <int N, int K, int MODE>
int codec_mode_launch(hc_codec c, const float* in, int64_t rows, float* o0, float* o1, float* o2,
                      float* o3, int check_negative) {
  using Tile = CodecTile<N, K, MODE>;
  using Op = CodecOp<N, K, MODE, Tile::T, Tile::THREADS, Tile::STAGES>;
  typename Op::Params p;
  fill_codec_const<N, K>(c, &p.cc);
  p.in = in;
  p.out[0] = o0;
  p.out[1] = o1;
  p.out[2] = o2;
  p.out[3] = o3;
  p.err = c->ctx->d_err;
  p.check_negative = check_negative;
  return launch_tile_op<Op>(c->ctx, p, rows);
}

template <int N, int K>
int codec_launch_nk(hc_codec c, int mode, const float* in, int64_t rows, float* o0, float* o1,
                    float* o2, float* o3, int check_negative) {
  switch (mode) {
    case kRoundtrip:
      return codec_mode_launch<N, K, kRoundtrip>(c, in, rows, o0, o1, o2, o3, check_negative);
    case kEncode:
      return codec_mode_launch<N, K, kEncode>(c, in, rows, o0, o1, o2, o3, check_negative);
    case kDecode:
      return codec_mode_launch<N, K, kDecode>(c, in, rows, o0, o1, o2, o3, check_negative);
    case kProject:
      return codec_mode_launch<N, K, kProject>(c, in, rows, o0, o1, o2, o3, check_negative);
  }
  return set_error(HC_EINVAL, "codec_launch: bad mode");
}

int codec_launch(hc_codec c, int mode, const float* in, int64_t rows, float* o0, float* o1, float* o2,
                 float* o3, int check_negative) {
  HC_DISPATCH_NK(c->n, c->k, codec_launch_nk, c, mode, in, rows, o0, o1, o2, o3, check_negative);
}

}  // namespace hcb
