// hadacodec-b200: the persistent tile pipeline shared by the bandwidth-bound
// kernels (codec round trip, latent / spectral G-buffer shading, loss).
//
//   HBM --cp.async.bulk--> smem in[stage] --thread-per-item compute--> smem out[stage]
//       --cp.async.bulk--> HBM
//
// Every stream (G-buffer idx, cos rows, spectra, codes, XYZ, sRGB) is a dense
// row-major array, so a tile of T consecutive items is ONE contiguous byte run
// per stream: one bulk copy each, fully coalesced, no register staging.  The
// input ring has STAGES slots; loads for tile t+STAGES are issued as soon as
// tile t's slot is consumed, keeping STAGES tiles of bytes in flight per CTA.
// Output slots are recycled once the bulk store that read them has drained
// (cp.async.bulk.wait_group.read).
//
// An Op supplies (all static):
//   T, THREADS, STAGES, NIN, NOUT, in_bytes(i), out_bytes(i) (bytes/item),
//   EXTRA_SMEM (bytes for op tables, e.g. the palette), Params, State,
//   in_ptr(p, i), out_ptr(p, i) (nullptr = stream disabled),
//   setup(p, extra_smem), compute(p, st, in[], out[], extra, item, global_item),
//   finish(p, st, extra)
// Ragged tails and unaligned pointers go through tile_generic, which runs the
// same compute on word copies (no TMA).
#pragma once

#include "hc_common.cuh"
#include "hc_tma.cuh"

namespace hcb {

template <class Op>
struct TileLayout {
  static constexpr int in_item_bytes() {
    int s = 0;
    for (int i = 0; i < Op::NIN; ++i) s += Op::in_bytes(i);
    return s;
  }
  static constexpr int out_item_bytes() {
    int s = 0;
    for (int i = 0; i < Op::NOUT; ++i) s += Op::out_bytes(i);
    return s;
  }
  static constexpr int kInTile = Op::T * in_item_bytes();
  static constexpr int kOutTile = Op::T * out_item_bytes();
  static constexpr int kBarBytes = 128;
  static constexpr int smem_bytes() {
    return kBarBytes + Op::STAGES * (kInTile + kOutTile) + Op::EXTRA_SMEM;
  }
};

template <class Op>
__global__ void __launch_bounds__(Op::THREADS)
    tile_pipeline(const __grid_constant__ typename Op::Params p, int64_t ntiles) {
  using Lay = TileLayout<Op>;
  constexpr int S = Op::STAGES;
  constexpr int T = Op::T;
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem);
  unsigned char* in_base = smem + Lay::kBarBytes;
  unsigned char* out_base = in_base + S * Lay::kInTile;
  unsigned char* extra = out_base + S * Lay::kOutTile;
  const int tid = threadIdx.x;

  Op::setup(p, extra);
  if (tid == 0) {
    for (int s = 0; s < S; ++s) mbar_init(&bar[s], 1);
    fence_mbar_init();
  }
  __syncthreads();

  auto issue_loads = [&](int64_t tile, int s) {
    unsigned char* dst = in_base + s * Lay::kInTile;
    mbar_arrive_expect_tx(&bar[s], Lay::kInTile);
#pragma unroll
    for (int i = 0; i < Op::NIN; ++i) {
      const unsigned char* src = static_cast<const unsigned char*>(Op::in_ptr(p, i));
      bulk_g2s(dst, src + tile * T * Op::in_bytes(i), T * Op::in_bytes(i), &bar[s]);
      dst += T * Op::in_bytes(i);
    }
  };

  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      const int64_t tile = blockIdx.x + static_cast<int64_t>(s) * gridDim.x;
      if (tile < ntiles) issue_loads(tile, s);
    }
  }

  typename Op::State st;
  Op::init_state(st);
  int iter = 0;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++iter) {
    const int s = iter % S;
    const uint32_t phase = (iter / S) & 1;
    if (tid == 0) bulk_wait_read<S - 1>();  // out[s] no longer read by the store of tile - S
    mbar_wait(&bar[s], phase);
    __syncthreads();

    const unsigned char* ins[Op::NIN > 0 ? Op::NIN : 1];
    unsigned char* outs[Op::NOUT > 0 ? Op::NOUT : 1];
    {
      const unsigned char* q = in_base + s * Lay::kInTile;
#pragma unroll
      for (int i = 0; i < Op::NIN; ++i) {
        ins[i] = q;
        q += T * Op::in_bytes(i);
      }
      unsigned char* o = out_base + s * Lay::kOutTile;
#pragma unroll
      for (int i = 0; i < Op::NOUT; ++i) {
        outs[i] = o;
        o += T * Op::out_bytes(i);
      }
    }
    for (int item = tid; item < T; item += Op::THREADS)
      Op::compute(p, st, ins, outs, extra, item, tile * T + item);
    if (Op::NOUT > 0) fence_proxy_async_smem();
    __syncthreads();

    if (tid == 0) {
      if (Op::NOUT > 0) {
#pragma unroll
        for (int i = 0; i < Op::NOUT; ++i) {
          unsigned char* dst = static_cast<unsigned char*>(Op::out_ptr(p, i));
          if (dst) bulk_s2g(dst + tile * T * Op::out_bytes(i), outs[i], T * Op::out_bytes(i));
        }
        bulk_commit();
      }
      const int64_t next = tile + static_cast<int64_t>(S) * gridDim.x;
      if (next < ntiles) issue_loads(next, s);
    }
  }
  if (tid == 0) bulk_wait_all<0>();
  Op::finish(p, st, extra);
}

// Same computation without TMA: word-granular copies, any alignment, any item
// range [item_begin, item_end).  Used for ragged tails and unaligned buffers.
template <class Op>
__global__ void __launch_bounds__(Op::THREADS)
    tile_generic(const __grid_constant__ typename Op::Params p, int64_t item_begin, int64_t item_end) {
  using Lay = TileLayout<Op>;
  constexpr int T = Op::T;
  extern __shared__ __align__(128) unsigned char smem[];
  unsigned char* in_base = smem + Lay::kBarBytes;
  unsigned char* out_base = in_base + Op::STAGES * Lay::kInTile;
  unsigned char* extra = out_base + Op::STAGES * Lay::kOutTile;
  const int tid = threadIdx.x;
  Op::setup(p, extra);
  __syncthreads();
  typename Op::State st;
  Op::init_state(st);
  const int64_t nitems = item_end - item_begin;
  const int64_t ntiles = (nitems + T - 1) / T;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t first = item_begin + tile * T;
    const int cnt = static_cast<int>(nitems - tile * T < T ? nitems - tile * T : T);
    const unsigned char* ins[Op::NIN > 0 ? Op::NIN : 1];
    unsigned char* outs[Op::NOUT > 0 ? Op::NOUT : 1];
    {
      unsigned char* q = in_base;
#pragma unroll
      for (int i = 0; i < Op::NIN; ++i) {
        const uint32_t* src = reinterpret_cast<const uint32_t*>(
            static_cast<const unsigned char*>(Op::in_ptr(p, i)) + first * Op::in_bytes(i));
        uint32_t* dst = reinterpret_cast<uint32_t*>(q);
        const int words = cnt * Op::in_bytes(i) / 4;
        for (int w = tid; w < words; w += Op::THREADS) dst[w] = src[w];
        ins[i] = q;
        q += T * Op::in_bytes(i);
      }
      unsigned char* o = out_base;
#pragma unroll
      for (int i = 0; i < Op::NOUT; ++i) {
        outs[i] = o;
        o += T * Op::out_bytes(i);
      }
    }
    __syncthreads();
    for (int item = tid; item < cnt; item += Op::THREADS)
      Op::compute(p, st, ins, outs, extra, item, first + item);
    __syncthreads();
#pragma unroll
    for (int i = 0; i < Op::NOUT; ++i) {
      unsigned char* dstb = static_cast<unsigned char*>(Op::out_ptr(p, i));
      if (!dstb) continue;
      uint32_t* dst = reinterpret_cast<uint32_t*>(dstb + first * Op::out_bytes(i));
      const uint32_t* src = reinterpret_cast<const uint32_t*>(outs[i]);
      const int words = cnt * Op::out_bytes(i) / 4;
      for (int w = tid; w < words; w += Op::THREADS) dst[w] = src[w];
    }
    __syncthreads();
  }
  Op::finish(p, st, extra);
}

}  // namespace hcb
