// Microbenchmark: throughput of W concurrent chains of dependent tcgen05.mma (kind::f16, M = 128,
// K = 16 per instruction, A from TMEM, fp32 accumulators) on one SM.  Every issuer warp issues
// warp-wide (elect.sync inside the asm, as mlp_kernel does) `n` MMAs into its own accumulator, the
// first with accumulate = 0, then commits and waits on its mbarrier; R rounds.  `split` spreads a
// warp's n MMAs round-robin over that many accumulators (dependency distance = split).
//
// Question: is mlp_kernel (10 MMAs per 128-pixel tile in chains of 1 / 5 / 4, ~55-60 cycles per
// MMA at 3 or 4 tile streams) bound by tiles in flight (TMEM) or by the rate at which the tensor
// pipe retires short dependent chains?  If cycles per MMA stop falling as W grows, it is the latter.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/bin/mma_chains tools/mma_chains.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint64_t desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46);
}
__host__ __device__ constexpr uint32_t idesc(int M, int N) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void wait_bar(uint64_t* b, uint32_t ph) {
  asm volatile("{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W;\n}\n" ::"r"(
                   smem_u32(b)),
               "r"(ph));
}
__device__ __forceinline__ void commit_w(uint64_t* b) {
  asm volatile(
      "{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}\n" ::"r"(smem_u32(b))
      : "memory");
}
__device__ __forceinline__ void mma_ts_w(uint32_t tD, uint32_t tA, uint64_t bd, uint32_t id, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p, e;\nsetp.ne.b32 p, %4, 0;\nelect.sync _|e, 0xffffffff;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(tD),
      "r"(tA), "l"(bd), "r"(id), "r"(acc));
}

// Accumulator columns: warp w, accumulator q at (w * split + q) * N (wrapped into 384 columns: timing
// only, results are not read); A operand at columns 384.. (never written: zeros or garbage).
template <int N>
__global__ void probe(int W, int n, int split, int R, long long* out) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint64_t wbar[16];
  __shared__ uint32_t slot;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < 32 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0x3c003c00u;
  if (tid == 0) {
    for (int w = 0; w < 16; ++w) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&wbar[w])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = slot;
  const uint64_t bd = desc(smem_u32(sm), N * 16, 128);
  constexpr uint32_t id = idesc(128, N);
  __syncthreads();
  const long long t0 = clock64();
  if (warp < W) {
    for (int i = 0; i < R; ++i) {
      for (int j = 0; j < n; ++j) {
        // split < 0: every warp accumulates into ONE shared accumulator (K steps of one chain
        // issued by different warps)
        const uint32_t col = split < 0 ? 0u : ((warp * split + j % split) * N) % 384;
        mma_ts_w(tmem + col, tmem + 384 + ((warp + j) % 8) * 8, bd, id, split < 0 ? 1 : j >= split);
      }
      commit_w(&wbar[warp]);
      wait_bar(&wbar[warp], i & 1);
      asm volatile("tcgen05.fence::after_thread_sync;");
    }
  }
  __syncthreads();
  const long long t1 = clock64();
  if (tid == 0) out[0] = t1 - t0;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

template <int N>
void run(int W, int n, int split) {
  long long* d;
  cudaMalloc(&d, sizeof(long long));
  cudaFuncSetAttribute(probe<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, 32 * 1024);
  const int R1 = 16, R2 = 528;
  long long a, b;
  probe<N><<<1, 512, 32 * 1024>>>(W, n, split, R1, d);
  cudaMemcpy(&a, d, sizeof(a), cudaMemcpyDeviceToHost);
  probe<N><<<1, 512, 32 * 1024>>>(W, n, split, R2, d);
  cudaMemcpy(&b, d, sizeof(b), cudaMemcpyDeviceToHost);
  const double per_round = double(b - a) / (R2 - R1);
  printf("N=%3d  %2d warps x %d MMAs over %d accumulator(s): %7.1f cycles per round, %6.1f cycles per MMA  %s\n", N, W, n,
         split, per_round, per_round / (W * n), cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}

int main() {
  for (int n : {1, 5})
    for (int W : {1, 2, 3, 4, 6, 8, 12, 16}) run<64>(W, n, 1);
  for (int W : {1, 4, 8}) run<64>(W, 4, 2);   // two interleaved 2-step chains per warp
  for (int W : {1, 4, 8}) run<64>(W, 6, 2);   // two interleaved 3-step chains per warp
  for (int W : {1, 4, 8, 16}) run<16>(W, 4, 1);
  for (int W : {1, 4, 8}) run<16>(W, 4, 2);
  for (int W : {1, 4, 8}) run<128>(W, 5, 1);
  // one chain's K steps spread over several issuer warps (same accumulator)
  run<64>(5, 1, -1);
  run<64>(2, 3, -1);
  run<64>(3, 2, -1);
  run<64>(4, 1, -1);
  run<16>(4, 1, -1);
  run<16>(2, 2, -1);
  return 0;
}
