// hadacodec-b200: multi-bounce accumulation launchers (config 4).
// Reference: evaluation.cpp:50-76, renderer.cpp:457-551 (see hc_chain.cuh).
#include <algorithm>
#include <map>
#include <mutex>
#include <utility>

#include "hc_chain.cuh"
#include "hc_launch.cuh"

namespace hcb {

// Occupancy per (kernel, dynamic smem) is cached: the launchers also run inside
// CUDA-graph capture, where attribute / occupancy queries are best avoided.
template <class KernelFn>
int chain_grid(hc_ctx ctx, KernelFn fn, int smem, int64_t P, int* grid, int threads = 256) {
  static std::mutex mu;
  static std::map<std::pair<std::pair<const void*, int>, int>, int> cache;  // ((kernel, smem), device)
  int occ = 0;
  {
    std::lock_guard<std::mutex> lk(mu);
    int dev = 0;
    HC_CUDA_TRY(cudaGetDevice(&dev));  // attributes are per device
    auto key = std::make_pair(std::make_pair(reinterpret_cast<const void*>(fn), smem), dev);
    auto it = cache.find(key);
    if (it != cache.end()) {
      occ = it->second;
    } else {
      // The dynamic shared-memory limit is one attribute per kernel and device, while the table
      // sizes (and so `smem`) vary per call: only ever raise it.  (Setting it to each new size
      // lowered it under an earlier, cached, larger size, whose next launch then failed with
      // "invalid argument" -- found by tests/test_gpu_random_sweep.py.)
      static std::map<std::pair<const void*, int>, int> attr_max;  // (kernel, device) -> configured limit
      int& limit = attr_max[std::make_pair(reinterpret_cast<const void*>(fn), dev)];
      if (smem > limit) {
        HC_CUDA_TRY(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        limit = smem;
      }
      HC_CUDA_TRY(cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout,
                                       cudaSharedmemCarveoutMaxShared));
      HC_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, threads, smem));
      cache[key] = occ;
    }
  }
  if (occ < 1) return set_error(HC_EUNSUPPORTED, "chain kernel does not fit on an SM");
  const int64_t px_per_block = threads / 8;  // 8 lanes per pixel
  const int64_t blocks_needed = (P + px_per_block - 1) / px_per_block;
  *grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(blocks_needed, static_cast<int64_t>(occ) * ctx->sm_count)));
  return HC_OK;
}

template <int K>
int chain_latent_k(hc_codec c, const float* pal, int n_pal, const float* ill, int n_ill,
                   const uint8_t* pidx, const uint8_t* iidx, const float* tw, int64_t P, int spp,
                   float* latent, float* xyz, float* rgb) {
  ChainLatentParams<K> p;
  for (int i = 0; i < 3 * K; ++i) p.Mxyz[i] = c->Mxyz[i];
  for (int i = 0; i < 9; ++i) p.Crgb[i] = c->Crgb[i];
  p.pal = pal;
  p.ill = ill;
  p.n_pal = n_pal;
  p.n_ill = n_ill;
  p.pidx = reinterpret_cast<const uint32_t*>(pidx);
  p.iidx = iidx;
  p.tw = reinterpret_cast<const float4*>(tw);
  p.P = P;
  p.spp = spp;
  p.latent = latent;
  p.xyz = xyz;
  p.rgb = rgb;
  p.err = c->ctx->d_err;
  int grid = 0;
#ifndef HC_CHAIN_V3
#define HC_CHAIN_V3 1
#endif
  if constexpr (K == 6) {
    if (HC_CHAIN_V3 && (!HC_CHAIN_IIDX128 || (spp % 16 == 0 && (reinterpret_cast<uintptr_t>(iidx) & 15u) == 0))) {  // instruction-lean k = 6 kernel (256-row palette table, packed Horner chain)
#ifndef HC_CHAIN_TMA
#define HC_CHAIN_TMA 1
#endif
      // palette-index / illuminant records by bulk copy: spp == 64, 16-byte aligned streams
      const bool tma = HC_CHAIN_TMA && spp == 64 && (reinterpret_cast<uintptr_t>(pidx) & 15u) == 0 &&
                       (reinterpret_cast<uintptr_t>(iidx) & 15u) == 0;
      const int threads = tma ? kChainTmaThreads : 256;
      const int smem = (256 + n_ill) * kChainV3Row + chain_v3_stage_bytes(threads / 32) +
                       (tma ? (threads / 32) * kChainTmaWarp : 0);
      auto fn = n_pal < 256 ? (tma ? chain_latent_v3_kernel<true, true> : chain_latent_v3_kernel<true, false>)
                            : (tma ? chain_latent_v3_kernel<false, true> : chain_latent_v3_kernel<false, false>);
      int rc = chain_grid(c->ctx, fn, smem, P, &grid, threads);
      if (rc != HC_OK) return rc;
      fn<<<grid, threads, smem, c->ctx->stream>>>(p);
      HC_CHECK_LAUNCH(c->ctx, "chain_latent_v3_kernel");
      return HC_OK;
    }
  }
  if constexpr (K <= 6) {
#ifndef HC_CHAIN_SHFL_ILL
#define HC_CHAIN_SHFL_ILL 0
#endif
    if (HC_CHAIN_SHFL_ILL && n_ill <= 16) {  // illuminant codes by shuffle, palette in smem
      const int smem = n_pal * ((K + 1) / 2) * 16 * 8;
      int rc = chain_grid(c->ctx, chain_latent_rep_kernel<K, true>, smem, P, &grid);
      if (rc != HC_OK) return rc;
      chain_latent_rep_kernel<K, true><<<grid, 256, smem, c->ctx->stream>>>(p);
      HC_CHECK_LAUNCH(c->ctx, "chain_latent_rep_kernel");
      return HC_OK;
    }
    const int smem = (n_pal + n_ill) * ((K + 1) / 2) * 16 * 8;  // replicated float2 tables
    int rc = chain_grid(c->ctx, chain_latent_rep_kernel<K, false>, smem, P, &grid);
    if (rc != HC_OK) return rc;
    chain_latent_rep_kernel<K, false><<<grid, 256, smem, c->ctx->stream>>>(p);
    HC_CHECK_LAUNCH(c->ctx, "chain_latent_rep_kernel");
  } else {
    const int smem = (n_pal + n_ill) * K * 4;
    int rc = chain_grid(c->ctx, chain_latent_kernel<K>, smem, P, &grid);
    if (rc != HC_OK) return rc;
    chain_latent_kernel<K><<<grid, 256, smem, c->ctx->stream>>>(p);
    HC_CHECK_LAUNCH(c->ctx, "chain_latent_kernel");
  }
  return HC_OK;
}

static bool chain_args_ok(int n_pal, int n_ill, const uint8_t* pidx, const float* tw, int spp) {
  if (n_pal < 1 || n_pal > 256 || n_ill < 1 || n_ill > kMaxIllum) return false;
  if (spp < 8 || spp % 8 != 0) return false;
  if ((reinterpret_cast<uintptr_t>(pidx) & 3u) || (reinterpret_cast<uintptr_t>(tw) & 15u)) return false;
  return true;
}

int chain_latent_launch(hc_codec c, const float* pal, int n_pal, const float* ill, int n_ill,
                        const uint8_t* pidx, const uint8_t* iidx, const float* tw, int64_t P, int spp,
                        float* latent, float* xyz, float* rgb) {
  if (!chain_args_ok(n_pal, n_ill, pidx, tw, spp))
    return set_error(HC_EINVAL, "multibounce: need 1 <= n_pal, n_ill <= 256, spp % 8 == 0, pidx 4-aligned, tw 16-aligned");
  if (P <= 0) return HC_OK;
  switch (c->k) {
    case 3: return chain_latent_k<3>(c, pal, n_pal, ill, n_ill, pidx, iidx, tw, P, spp, latent, xyz, rgb);
    case 6: return chain_latent_k<6>(c, pal, n_pal, ill, n_ill, pidx, iidx, tw, P, spp, latent, xyz, rgb);
    case 9: return chain_latent_k<9>(c, pal, n_pal, ill, n_ill, pidx, iidx, tw, P, spp, latent, xyz, rgb);
  }
  return set_error(HC_EUNSUPPORTED, "multibounce_latent: k must be 3, 6 or 9");
}

template <int N, int SPL>
int chain_spectral_ns(hc_codec c, const float* pal, int n_pal, const float* ill, int n_ill,
                      const uint8_t* pidx, const uint8_t* iidx, const float* tw, int64_t P, int spp,
                      float* xyz, float* rgb) {
  ChainSpectralParams<N> p;
  for (int i = 0; i < 3 * N; ++i) p.cmf[i] = c->cmf_dl[i];
  for (int i = 0; i < 9; ++i) p.Crgb[i] = c->Crgb[i];
  p.pal = pal;
  p.ill = ill;
  p.n_pal = n_pal;
  p.n_ill = n_ill;
  p.pidx = reinterpret_cast<const uint32_t*>(pidx);
  p.iidx = iidx;
  p.tw = reinterpret_cast<const float4*>(tw);
  p.P = P;
  p.spp = spp;
  p.xyz = xyz;
  p.rgb = rgb;
  p.err = c->ctx->d_err;
  int grid = 0;
#ifndef HC_CHAIN_NAIVE_LANES
#define HC_CHAIN_NAIVE_LANES 1
#endif
  if constexpr (N > 64 && N <= kChainLanesRow) {
    if (HC_CHAIN_NAIVE_LANES) {  // lanes over wavelengths (one pixel per warp)
      const int smem = (n_pal + n_ill) * kChainLanesRow * 4 + 8 * 32 * 6 * 4;
      int rc = chain_grid(c->ctx, chain_spectral_lanes_kernel<N>, smem, P * 8, &grid);  // 8 lanes-worth per pixel
      if (rc != HC_OK) return rc;
      chain_spectral_lanes_kernel<N><<<grid, 256, smem, c->ctx->stream>>>(p);
      HC_CHECK_LAUNCH(c->ctx, "chain_spectral_lanes_kernel");
      return HC_OK;
    }
  }
  const int smem = (n_pal + n_ill) * N * 4;
  int rc = chain_grid(c->ctx, chain_spectral_kernel<N, SPL>, smem, P, &grid);
  if (rc != HC_OK) return rc;
  chain_spectral_kernel<N, SPL><<<grid, 256, smem, c->ctx->stream>>>(p);
  HC_CHECK_LAUNCH(c->ctx, "chain_spectral_kernel");
  return HC_OK;
}

int chain_spectral_launch(hc_codec c, const float* pal, int n_pal, const float* ill, int n_ill,
                          const uint8_t* pidx, const uint8_t* iidx, const float* tw, int64_t P,
                          int spp, float* xyz, float* rgb) {
  if (!chain_args_ok(n_pal, n_ill, pidx, tw, spp))
    return set_error(HC_EINVAL, "multibounce: need 1 <= n_pal, n_ill <= 256, spp % 8 == 0, pidx 4-aligned, tw 16-aligned");
  if (P <= 0) return HC_OK;
  const int spl = spp / 8;
  if (c->n == 81) {
    if (spl == 8) return chain_spectral_ns<81, 8>(c, pal, n_pal, ill, n_ill, pidx, iidx, tw, P, spp, xyz, rgb);
    if (spl == 1) return chain_spectral_ns<81, 1>(c, pal, n_pal, ill, n_ill, pidx, iidx, tw, P, spp, xyz, rgb);
    if (spl == 2) return chain_spectral_ns<81, 2>(c, pal, n_pal, ill, n_ill, pidx, iidx, tw, P, spp, xyz, rgb);
    if (spl == 4) return chain_spectral_ns<81, 4>(c, pal, n_pal, ill, n_ill, pidx, iidx, tw, P, spp, xyz, rgb);
  } else if (c->n == 47) {
    if (spl == 8) return chain_spectral_ns<47, 8>(c, pal, n_pal, ill, n_ill, pidx, iidx, tw, P, spp, xyz, rgb);
    if (spl == 1) return chain_spectral_ns<47, 1>(c, pal, n_pal, ill, n_ill, pidx, iidx, tw, P, spp, xyz, rgb);
  }
  return set_error(HC_EUNSUPPORTED, "multibounce_spectral: compiled for n=81 spp in {8,16,32,64}, n=47 spp in {8,64}");
}

}  // namespace hcb
