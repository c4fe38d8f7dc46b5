// hadacodec-b200: the persistent tile pipeline shared by the bandwidth-bound
// kernels (codec round trip, latent / spectral G-buffer shading, loss).
//
//   HBM --TMA--> smem in[stage] --thread-per-item compute--> smem out[stage] --TMA--> HBM
//
// Every stream (G-buffer idx, cos rows, spectra, codes, XYZ, sRGB) is a dense
// row-major array, so a tile of T consecutive items is ONE contiguous byte run
// per stream: one bulk copy each (cp.async.bulk), fully coalesced, no register
// staging.  One stream per Op may instead arrive through a 2-D tensor map with
// the 128-byte swizzle (Op::kTensorStream): rows of exactly 128 bytes whose 16-byte
// chunk c of row r lands at chunk c ^ (r & 7), which makes a quarter-warp's
// LDS.128 of the same chunk index of 8 consecutive rows bank-conflict free.
// The input ring has STAGES slots; loads for tile t+STAGES are issued as soon as
// tile t's slot is consumed.  Output slots are recycled once the bulk store that
// read them has drained (cp.async.bulk.wait_group.read).
//
// An Op supplies (all static):
//   T, THREADS, STAGES, NIN, NOUT, in_bytes(i), out_bytes(i) (bytes/item),
//   kTensorStream (-1 = none) and tensor_map(p),
//   EXTRA_SMEM (bytes for op tables, e.g. the palette), Params, State,
//   in_ptr(p, i), out_ptr(p, i) (nullptr = stream disabled),
//   setup(p, extra_smem), compute(p, st, in[], out[], extra, item, global_item),
//   finish(p, st, extra),
//   kWarpSpecialized (run tile_pipeline_ws instead of tile_pipeline),
//   kEvictFirstLoads (stream the inputs through L2 with an evict-first policy),
//   optionally kLanesPerItem (default 1): that many threads call compute() for
//   the same item -- threads item, item + THREADS/LPI, ... (warp groups) -- and
//   the op splits the item's work by threadIdx.x / (THREADS/LPI)
// Ragged tails and unaligned pointers go through tile_generic, which runs the
// same compute on word copies (no TMA; the swizzle is applied in software).
#pragma once

#include <type_traits>

#include "hc_common.cuh"
#include "hc_tma.cuh"

namespace hcb {

template <class Op, class = void>
struct LanesPerItem {
  static constexpr int value = 1;
};
template <class Op>
struct LanesPerItem<Op, std::void_t<decltype(Op::kLanesPerItem)>> {
  static constexpr int value = Op::kLanesPerItem;
};

constexpr int kTileAlign = 1024;  // every stream tile starts 1024-byte aligned (swizzle requirement)

__host__ __device__ constexpr int align_up(int x, int a) { return (x + a - 1) / a * a; }

template <class Op>
struct TileLayout {
  // Offset of input stream i within one stage (i == NIN gives the stage size).  The
  // swizzled tensor stream starts 1024-byte aligned, every other stream 128-byte.
  static constexpr int in_align(int i) { return i == Op::kTensorStream ? kTileAlign : 128; }
  static constexpr int in_off(int i) {
    int s = 0;
    for (int j = 0; j < i; ++j) s = align_up(s, in_align(j)) + Op::T * Op::in_bytes(j);
    return i < Op::NIN ? align_up(s, in_align(i)) : align_up(s, kTileAlign);
  }
  static constexpr int out_off(int i) {
    int s = 0;
    for (int j = 0; j < i; ++j) s = align_up(s, 128) + Op::T * Op::out_bytes(j);
    return align_up(s, 128);
  }
  static constexpr int kInTile = in_off(Op::NIN);
  static constexpr int kOutTile = align_up(out_off(Op::NOUT), kTileAlign);
  static constexpr int kInBytes() {
    int s = 0;
    for (int j = 0; j < Op::NIN; ++j) s += Op::T * Op::in_bytes(j);
    return s;
  }
  static constexpr int kBarBytes = 1024;
  static constexpr int smem_bytes() {
    return kBarBytes + Op::STAGES * (kInTile + kOutTile) + Op::EXTRA_SMEM + 1024;  // + base alignment slack
  }
};

// Dynamic shared memory, rounded up to a 1024-byte boundary.
__device__ __forceinline__ unsigned char* aligned_smem_base(unsigned char* raw) {
  const uint32_t a = smem_u32(raw);
  return raw + ((kTileAlign - (a & (kTileAlign - 1))) & (kTileAlign - 1));
}

#ifndef HC_PIPE_WARP  // 1: TMA issue from a whole warp (elect.sync), 0: from thread 0
#define HC_PIPE_WARP 0
#endif
#if HC_PIPE_WARP
#define HC_PW(fn) fn##_w
#else
#define HC_PW(fn) fn
#endif

template <class Op>
__global__ void __launch_bounds__(Op::THREADS)
    tile_pipeline(const __grid_constant__ typename Op::Params p, int64_t ntiles) {
  using Lay = TileLayout<Op>;
  constexpr int S = Op::STAGES;
  constexpr int T = Op::T;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = aligned_smem_base(smem_raw);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem);
  unsigned char* in_base = smem + Lay::kBarBytes;
  unsigned char* out_base = in_base + S * Lay::kInTile;
  unsigned char* extra = out_base + S * Lay::kOutTile;
  const int tid = threadIdx.x;
  const bool issuer = HC_PIPE_WARP ? tid < 32 : tid == 0;  // warp 0 (elect.sync) or thread 0

  auto issue_loads = [&](int64_t tile, int s) {
    unsigned char* stage = in_base + s * Lay::kInTile;
    HC_PW(mbar_arrive_expect_tx)(&bar[s], Lay::kInBytes());
#pragma unroll
    for (int i = 0; i < Op::NIN; ++i) {
      unsigned char* dst = stage + Lay::in_off(i);
      if (i == Op::kTensorStream) {
        HC_PW(tma_load_2d)(dst, Op::tensor_map(p), 0, static_cast<int>(tile * T), &bar[s]);
      } else {
        const unsigned char* src = static_cast<const unsigned char*>(Op::in_ptr(p, i));
        if constexpr (Op::kEvictFirstLoads)
          HC_PW(bulk_g2s_evict_first)(dst, src + tile * T * Op::in_bytes(i), T * Op::in_bytes(i), &bar[s],
                                      policy_evict_first());
        else
          HC_PW(bulk_g2s)(dst, src + tile * T * Op::in_bytes(i), T * Op::in_bytes(i), &bar[s]);
      }
    }
  };

  // The grid is persistent (<= one wave), so the next kernel may be scheduled
  // right away: its CTAs take SM slots as ours exit and do their setup while
  // our tail drains.  Global memory is touched only after every prior grid is
  // complete (pdl_wait_prior_grids), so any aliasing between launches is safe.
  pdl_launch_dependents();
  if (tid == 0) {
    for (int s = 0; s < S; ++s) mbar_init(&bar[s], 1);
    fence_mbar_init();
  }
  pdl_wait_prior_grids();
  // The first STAGES tiles are requested before the op's table setup (e.g. the
  // palette copy) so the two latencies overlap at kernel start.
  if (issuer) {
    for (int s = 0; s < S; ++s) {
      const int64_t tile = blockIdx.x + static_cast<int64_t>(s) * gridDim.x;
      if (tile < ntiles) issue_loads(tile, s);
    }
  }
  Op::setup(p, extra);
  __syncthreads();

  typename Op::State st;
  Op::init_state(st);
  int iter = 0;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++iter) {
    const int s = iter % S;
    const uint32_t phase = (iter / S) & 1;
    if (issuer) bulk_wait_read<S - 1>();  // out[s] no longer read by the store of tile - S
    mbar_wait(&bar[s], phase);
    __syncthreads();

    const unsigned char* ins[Op::NIN > 0 ? Op::NIN : 1];
    unsigned char* outs[Op::NOUT > 0 ? Op::NOUT : 1];
#pragma unroll
    for (int i = 0; i < Op::NIN; ++i) ins[i] = in_base + s * Lay::kInTile + Lay::in_off(i);
#pragma unroll
    for (int i = 0; i < Op::NOUT; ++i) outs[i] = out_base + s * Lay::kOutTile + Lay::out_off(i);
    constexpr int LPI = LanesPerItem<Op>::value;
    for (int item = tid % (Op::THREADS / LPI); item < T; item += Op::THREADS / LPI)
      Op::compute(p, st, ins, outs, extra, item, tile * T + item);
    if (Op::NOUT > 0) fence_proxy_async_smem();
    __syncthreads();

    if (issuer) {
      if (Op::NOUT > 0) {
#pragma unroll
        for (int i = 0; i < Op::NOUT; ++i) {
          unsigned char* dst = static_cast<unsigned char*>(Op::out_ptr(p, i));
          if (dst) HC_PW(bulk_s2g)(dst + tile * T * Op::out_bytes(i), outs[i], T * Op::out_bytes(i));
        }
        HC_PW(bulk_commit)();
      }
      const int64_t next = tile + static_cast<int64_t>(S) * gridDim.x;
      if (next < ntiles) issue_loads(next, s);
    }
  }
  if (issuer) bulk_wait_all<0>();
  Op::finish(p, st, extra);
}

// Warp-specialised variant: THREADS consumer threads + one producer warp, no
// CTA-wide barrier inside the loop.  Per input slot s: full[s] (TMA bytes
// landed) and empty[s] (one arrival per consumer warp once it has read in[s]
// and written its outputs).  Outputs use their own ring of OUT_STAGES slots;
// ofree[o] is re-armed by the producer once the bulk store that read out[o] has
// drained, so a warp that finishes tile t early moves on to tile t+1 without
// waiting for the slowest warp.
constexpr int kOutStages = 2;
constexpr int kProducerWarp = 32;

template <class Op>
struct WsLayout {
  using Lay = TileLayout<Op>;
  static constexpr int kOutSlots = Op::NOUT > 0 ? kOutStages : 0;
  static constexpr int smem_bytes() {
    return Lay::kBarBytes + Op::STAGES * Lay::kInTile + kOutSlots * Lay::kOutTile + Op::EXTRA_SMEM + 1024;
  }
};

template <class Op>
__global__ void __launch_bounds__(Op::THREADS + kProducerWarp)
    tile_pipeline_ws(const __grid_constant__ typename Op::Params p, int64_t ntiles) {
  using Lay = TileLayout<Op>;
  constexpr int S = Op::STAGES;
  constexpr int SO = kOutStages;
  constexpr int T = Op::T;
  constexpr int NCW = Op::THREADS / 32;  // consumer warps
  static_assert(Op::THREADS % 32 == 0, "consumer threads must be whole warps");
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = aligned_smem_base(smem_raw);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);
  uint64_t* empty = full + S;
  uint64_t* ofree = empty + S;
  unsigned char* in_base = smem + Lay::kBarBytes;
  unsigned char* out_base = in_base + S * Lay::kInTile;
  unsigned char* extra = out_base + WsLayout<Op>::kOutSlots * Lay::kOutTile;
  const int tid = threadIdx.x;
  // the producer is the extra warp (elect.sync issue) or its first thread
  const bool producer = HC_PIPE_WARP ? tid >= Op::THREADS : tid == Op::THREADS;

  auto issue_loads = [&](int64_t tile, int s) {
    unsigned char* stage = in_base + s * Lay::kInTile;
    HC_PW(mbar_arrive_expect_tx)(&full[s], Lay::kInBytes());
#pragma unroll
    for (int i = 0; i < Op::NIN; ++i) {
      unsigned char* dst = stage + Lay::in_off(i);
      if (i == Op::kTensorStream) {
        HC_PW(tma_load_2d)(dst, Op::tensor_map(p), 0, static_cast<int>(tile * T), &full[s]);
      } else {
        const unsigned char* src = static_cast<const unsigned char*>(Op::in_ptr(p, i));
        if constexpr (Op::kEvictFirstLoads)
          HC_PW(bulk_g2s_evict_first)(dst, src + tile * T * Op::in_bytes(i), T * Op::in_bytes(i), &full[s],
                                      policy_evict_first());
        else
          HC_PW(bulk_g2s)(dst, src + tile * T * Op::in_bytes(i), T * Op::in_bytes(i), &full[s]);
      }
    }
  };

  pdl_launch_dependents();
  if (tid == Op::THREADS) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NCW);
    }
    for (int o = 0; o < SO; ++o) mbar_init(&ofree[o], 1);
    fence_mbar_init();
  }
  pdl_wait_prior_grids();
  if (producer) {
    for (int s = 0; s < S; ++s) {
      const int64_t tile = blockIdx.x + static_cast<int64_t>(s) * gridDim.x;
      if (tile < ntiles) issue_loads(tile, s);
    }
    for (int o = 0; o < SO; ++o) HC_PW(mbar_arrive)(&ofree[o]);  // every output slot starts free
  }
  Op::setup(p, extra);
  __syncthreads();

  typename Op::State st;
  Op::init_state(st);
  if (tid < Op::THREADS) {
    int iter = 0;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++iter) {
      const int s = iter % S;
      const int o = iter % SO;
      mbar_wait(&full[s], (iter / S) & 1);
      if (Op::NOUT > 0) mbar_wait(&ofree[o], (iter / SO) & 1);
      const unsigned char* ins[Op::NIN > 0 ? Op::NIN : 1];
      unsigned char* outs[Op::NOUT > 0 ? Op::NOUT : 1];
#pragma unroll
      for (int i = 0; i < Op::NIN; ++i) ins[i] = in_base + s * Lay::kInTile + Lay::in_off(i);
#pragma unroll
      for (int i = 0; i < Op::NOUT; ++i) outs[i] = out_base + o * Lay::kOutTile + Lay::out_off(i);
      constexpr int LPI = LanesPerItem<Op>::value;
      for (int item = tid % (Op::THREADS / LPI); item < T; item += Op::THREADS / LPI)
        Op::compute(p, st, ins, outs, extra, item, tile * T + item);
      if (Op::NOUT > 0) fence_proxy_async_smem();
      __syncwarp();
      if ((tid & 31) == 0) mbar_arrive(&empty[s]);
    }
  } else if (producer) {
    int iter = 0;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++iter) {
      const int s = iter % S;
      mbar_wait(&empty[s], (iter / S) & 1);
      if (Op::NOUT > 0) {
        unsigned char* ob = out_base + (iter % SO) * Lay::kOutTile;
#pragma unroll
        for (int i = 0; i < Op::NOUT; ++i) {
          unsigned char* dst = static_cast<unsigned char*>(Op::out_ptr(p, i));
          if (dst) HC_PW(bulk_s2g)(dst + tile * T * Op::out_bytes(i), ob + Lay::out_off(i), T * Op::out_bytes(i));
        }
        HC_PW(bulk_commit)();
      }
      const int64_t next = tile + static_cast<int64_t>(S) * gridDim.x;
      if (next < ntiles) issue_loads(next, s);
      if (Op::NOUT > 0 && iter + 1 >= SO) {
        bulk_wait_read<SO - 1>();  // the store of tile iter + 1 - SO has read its slot
        HC_PW(mbar_arrive)(&ofree[(iter + 1) % SO]);
      }
    }
    bulk_wait_all<0>();
  }
  Op::finish(p, st, extra);
}

// Same computation without TMA: word-granular copies, any alignment, any item
// range [item_begin, item_end).  Used for ragged tails and unaligned buffers.
template <class Op>
__global__ void __launch_bounds__(Op::THREADS)
    tile_generic(const __grid_constant__ typename Op::Params p, int64_t item_begin, int64_t item_end) {
  using Lay = TileLayout<Op>;
  constexpr int T = Op::T;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = aligned_smem_base(smem_raw);
  unsigned char* in_base = smem + Lay::kBarBytes;
  unsigned char* out_base = in_base + Op::STAGES * Lay::kInTile;
  unsigned char* extra = out_base + Op::STAGES * Lay::kOutTile;
  const int tid = threadIdx.x;
  pdl_wait_prior_grids();
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
#pragma unroll
    for (int i = 0; i < Op::NIN; ++i) {
      const uint32_t* src = reinterpret_cast<const uint32_t*>(
          static_cast<const unsigned char*>(Op::in_ptr(p, i)) + first * Op::in_bytes(i));
      uint32_t* dst = reinterpret_cast<uint32_t*>(in_base + Lay::in_off(i));
      const int words = cnt * Op::in_bytes(i) / 4;
      if (i == Op::kTensorStream) {
        // software 128-byte swizzle: word w of row r -> chunk ((w / 4) ^ (r & 7))
        for (int w = tid; w < words; w += Op::THREADS) {
          const int r = w >> 5, c = (w >> 2) & 7, e = w & 3;
          dst[r * 32 + ((c ^ (r & 7)) << 2) + e] = src[w];
        }
      } else {
        for (int w = tid; w < words; w += Op::THREADS) dst[w] = src[w];
      }
      ins[i] = in_base + Lay::in_off(i);
    }
#pragma unroll
    for (int i = 0; i < Op::NOUT; ++i) outs[i] = out_base + Lay::out_off(i);
    __syncthreads();
    // Ops with several lanes per item run every item of the tile (whole warps take
    // part in their shuffles); they discard items at or past item_end themselves.
    constexpr int LPI = LanesPerItem<Op>::value;
    for (int item = tid % (Op::THREADS / LPI); item < (LPI > 1 ? T : cnt); item += Op::THREADS / LPI)
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
