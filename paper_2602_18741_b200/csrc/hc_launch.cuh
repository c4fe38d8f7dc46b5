// hadacodec-b200: host-side launch of the tile pipeline.
#pragma once

#include <cuda.h>

#include <algorithm>
#include <atomic>
#include <utility>

#include "hc_internal.h"
#include "hc_pipeline.cuh"

namespace hcb {

template <class Op>
struct TileLaunchCache {
  static std::atomic<uint64_t> configured;  // one bit per device (attributes are per device)
  static int occ_pipeline, occ_generic;  // occ_pipeline: of tile_pipeline_ws for warp-specialised ops
};
template <class Op>
std::atomic<uint64_t> TileLaunchCache<Op>::configured{0};
template <class Op>
int TileLaunchCache<Op>::occ_pipeline = 1;
template <class Op>
int TileLaunchCache<Op>::occ_generic = 1;


template <class Op>
int configure_tile_op() {
  using Cache = TileLaunchCache<Op>;
  if (configured_here(Cache::configured)) return HC_OK;
  const int smem = TileLayout<Op>::smem_bytes();
  HC_CUDA_TRY(cudaFuncSetAttribute(tile_pipeline<Op>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  HC_CUDA_TRY(cudaFuncSetAttribute(tile_generic<Op>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  HC_CUDA_TRY(cudaFuncSetAttribute(tile_pipeline<Op>, cudaFuncAttributePreferredSharedMemoryCarveout,
                                   cudaSharedmemCarveoutMaxShared));
  HC_CUDA_TRY(cudaFuncSetAttribute(tile_generic<Op>, cudaFuncAttributePreferredSharedMemoryCarveout,
                                   cudaSharedmemCarveoutMaxShared));
  int a = 0, b = 0, w = 1;
  if constexpr (Op::kWarpSpecialized) {
    const int smem_ws = WsLayout<Op>::smem_bytes();
    HC_CUDA_TRY(cudaFuncSetAttribute(tile_pipeline_ws<Op>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_ws));
    HC_CUDA_TRY(cudaFuncSetAttribute(tile_pipeline_ws<Op>, cudaFuncAttributePreferredSharedMemoryCarveout,
                                     cudaSharedmemCarveoutMaxShared));
    HC_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&w, tile_pipeline_ws<Op>,
                                                              Op::THREADS + kProducerWarp, smem_ws));
    a = w;
  } else {
    HC_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&a, tile_pipeline<Op>, Op::THREADS, smem));
  }
  HC_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, tile_generic<Op>, Op::THREADS, smem));
  if (a < 1 || b < 1 || w < 1) return set_error(HC_EUNSUPPORTED, "tile kernel does not fit on an SM");
  Cache::occ_pipeline = a;
  Cache::occ_generic = b;
  mark_configured_here(Cache::configured);
  return HC_OK;
}

// Launch with the programmatic-stream-serialization attribute (PDL) when the
// context allows it: the kernel may begin while the previous kernel on the
// stream drains; kernels using this must call pdl_wait_prior_grids() before
// their first global access (tile_pipeline / tile_generic do).
template <class... KArgs, class... Args>
cudaError_t launch_k(hc_ctx ctx, void (*kern)(KArgs...), int grid, int block, int smem, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = ctx->stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = ctx->pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

inline bool al16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

// 2-D tensor map over a [rows][row_floats] f32 array, box [box_rows][row_floats],
// 128-byte swizzle (row_floats * 4 must be 128).  cuTensorMapEncodeTiled is
// reached through the runtime's driver entry point (no libcuda link).
int encode_rows_tmap_swizzle128(CUtensorMap* map, const void* base, int64_t rows, int row_floats, int box_rows);

// Launch Op over `items` items.  Full tiles of 16-byte-aligned streams go
// through the TMA pipeline; the ragged tail (and everything, if any stream is
// misaligned) through tile_generic.  `grid_out` (optional) receives the grid
// sizes used: [pipeline, generic].
template <class Op>
int launch_tile_op(hc_ctx ctx, const typename Op::Params& p, int64_t items, int* grid_out = nullptr) {
  if (items <= 0) {
    if (grid_out) grid_out[0] = grid_out[1] = 0;
    return HC_OK;
  }
  int rc = configure_tile_op<Op>();
  if (rc != HC_OK) return rc;
  using Cache = TileLaunchCache<Op>;
  bool aligned = true;
  for (int i = 0; i < Op::NIN; ++i) aligned &= al16(Op::in_ptr(p, i));
  for (int i = 0; i < Op::NOUT; ++i) aligned &= al16(Op::out_ptr(p, i));
  const int smem = TileLayout<Op>::smem_bytes();
  const int64_t full = aligned ? items / Op::T : 0;
  int g0 = 0, g1 = 0;
  if (full > 0) {
    g0 = static_cast<int>(std::min<int64_t>(full, static_cast<int64_t>(Cache::occ_pipeline) * ctx->sm_count));
    if constexpr (Op::kWarpSpecialized) {
      HC_CUDA_TRY(launch_k(ctx, tile_pipeline_ws<Op>, g0, Op::THREADS + kProducerWarp,
                           WsLayout<Op>::smem_bytes(), p, full));
    } else {
      HC_CUDA_TRY(launch_k(ctx, tile_pipeline<Op>, g0, Op::THREADS, smem, p, full));
    }
    HC_CHECK_LAUNCH(ctx, "tile_pipeline");
  }
  const int64_t begin = full * Op::T;
  if (begin < items) {
    const int64_t tiles = (items - begin + Op::T - 1) / Op::T;
    g1 = static_cast<int>(std::min<int64_t>(tiles, static_cast<int64_t>(Cache::occ_generic) * ctx->sm_count));
    HC_CUDA_TRY(launch_k(ctx, tile_generic<Op>, g1, Op::THREADS, smem, p, begin, items));
    HC_CHECK_LAUNCH(ctx, "tile_generic");
  }
  if (grid_out) {
    grid_out[0] = g0;
    grid_out[1] = g1;
  }
  return HC_OK;
}

template <int N, int K>
void fill_codec_const(const hc_codec_s* c, CodecConst<N, K>* cc) {
  for (int i = 0; i < K * N; ++i) cc->E[i] = c->E[i];
  for (int i = 0; i < N * K; ++i) cc->D[i] = c->D[i];
  for (int i = 0; i < 3 * K; ++i) cc->Mxyz[i] = c->Mxyz[i];
  for (int i = 0; i < 9; ++i) cc->Crgb[i] = c->Crgb[i];
  for (int i = 0; i < 3 * N; ++i) cc->cmf[i] = c->cmf_dl[i];
}

}  // namespace hcb

// (n, k) dispatch over the compiled instantiations.
#define HC_DISPATCH_NK(n, k, FN, ...)                                                      \
  do {                                                                                     \
    if ((n) == 81 && (k) == 6) return FN<81, 6>(__VA_ARGS__);                              \
    if ((n) == 81 && (k) == 9) return FN<81, 9>(__VA_ARGS__);                              \
    if ((n) == 81 && (k) == 3) return FN<81, 3>(__VA_ARGS__);                              \
    if ((n) == 47 && (k) == 6) return FN<47, 6>(__VA_ARGS__);                              \
    if ((n) == 47 && (k) == 9) return FN<47, 9>(__VA_ARGS__);                              \
    if ((n) == 47 && (k) == 3) return FN<47, 3>(__VA_ARGS__);                              \
    return ::hcb::set_error(HC_EUNSUPPORTED, "unsupported (n, k); compiled: n in {47, 81}, k in {3, 6, 9}"); \
  } while (0)
