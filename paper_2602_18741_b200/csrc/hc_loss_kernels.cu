// hadacodec-b200: near-multiplicativity loss (config 5b).
// Reference: forward_pair + mse_n (trainer.cpp:49-71).  Per-CTA fp64 partials
// are summed by a single-block kernel in a fixed order (deterministic).
#include "hc_launch.cuh"
#include "hc_ops.cuh"

namespace hcb {

__global__ void sum_partials_kernel(const double* partials, int count, double* out) {
  __shared__ double red[32];
  double v = 0.0;
  for (int i = threadIdx.x; i < count; i += blockDim.x) v += partials[i];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (blockDim.x + 31) / 32; ++w) t += red[w];
    *out = t;
  }
}

#ifndef HC_LOSS_T
#define HC_LOSS_T 64
#endif
#ifndef HC_LOSS_STAGES
#define HC_LOSS_STAGES 2
#endif

template <int N, int K>
int loss_nk(hc_codec c, const float* A, const float* B, int64_t pairs, double* sum_dev) {
  // 64-pair tiles (two 64-thread halves) x 2 stages = 96 KB smem: 2 CTAs / SM (8 warps), one
  // tile computing + one loading each
  using Op = LossOp<N, K, HC_LOSS_T, (N % 3 == 0 ? 3 : 1) * HC_LOSS_T, HC_LOSS_STAGES>;
  hc_ctx ctx = c->ctx;
  int rc = configure_tile_op<Op>();
  if (rc != HC_OK) return rc;
  const int cap = (TileLaunchCache<Op>::occ_pipeline + TileLaunchCache<Op>::occ_generic) * ctx->sm_count;
  if (ctx->partial_capacity < cap) {
    if (ctx->d_partials) cudaFree(ctx->d_partials);
    ctx->d_partials = nullptr;
    HC_CUDA_TRY(cudaMalloc(&ctx->d_partials, sizeof(double) * cap));
    ctx->partial_capacity = cap;
  }
  typename Op::Params p;
  for (int i = 0; i < K * N; ++i) p.E[i] = static_cast<double>(c->E[i]);
  for (int i = 0; i < N * K; ++i) p.D[i] = static_cast<double>(c->D[i]);
  p.a = A;
  p.b = B;
  p.partials = ctx->d_partials;
  p.partial_offset = 0;
  p.pairs = pairs;
  // Main (TMA) pass over full tiles first, then the tail with offset partials.
  const bool aligned = al16(A) && al16(B);
  const int64_t full = aligned ? pairs / Op::T : 0;
  int used = 0;
  if (full > 0) {
    int g[2];
    rc = launch_tile_op<Op>(ctx, p, full * Op::T, g);
    if (rc != HC_OK) return rc;
    used = g[0];
  }
  if (full * Op::T < pairs) {
    p.partial_offset = used;
    const int smem = TileLayout<Op>::smem_bytes();
    const int64_t tiles = (pairs - full * Op::T + Op::T - 1) / Op::T;
    const int g1 = static_cast<int>(std::min<int64_t>(tiles, static_cast<int64_t>(TileLaunchCache<Op>::occ_generic) * ctx->sm_count));
    tile_generic<Op><<<g1, Op::THREADS, smem, ctx->stream>>>(p, full * Op::T, pairs);
    HC_CHECK_LAUNCH(ctx, "loss tile_generic");
    used += g1;
  }
  if (used == 0) {
    HC_CUDA_TRY(cudaMemsetAsync(sum_dev, 0, sizeof(double), ctx->stream));
    return HC_OK;
  }
  sum_partials_kernel<<<1, 256, 0, ctx->stream>>>(ctx->d_partials, used, sum_dev);
  HC_CHECK_LAUNCH(ctx, "sum_partials_kernel");
  return HC_OK;
}

int loss_launch(hc_codec c, const float* A, const float* B, int64_t pairs, double* sum_dev) {
  HC_DISPATCH_NK(c->n, c->k, loss_nk, c, A, B, pairs, sum_dev);
}

}  // namespace hcb
