// Microbenchmark: cycles per tcgen05.mma.cta_group::2 (kind::f16, M = 256 over a CTA
// pair, bf16 -> f32), SS and TS, vs N.  Launch: clusters of 2 CTAs, one per SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/bin/mma_probe2 tools/mma_probe2.cu
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
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

template <bool TS, int N>
__global__ void __cluster_dims__(2, 1, 1) probe(int R, long long* out) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int tid = threadIdx.x;
  uint32_t rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  for (int i = tid; i < 48 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0x3f803f80u;
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (tid < 32) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  cluster_sync();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = slot;
  long long t0 = clock64();
  if (rank == 0 && tid == 0) {
    const uint32_t sA = smem_u32(sm), sB = smem_u32(sm + 16384);
    const uint64_t ad = desc(sA, 128 * 16, 128), bd = desc(sB, (N / 2) * 16, 128);
    const uint32_t id = idesc(256, N);
    const uint32_t tD = tmem + 256, tA = tmem;
    for (int i = 0; i < R; ++i) {
      if (TS)
        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(tD),
                     "r"(tA), "l"(bd), "r"(id), "r"(1));
      else
        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tD),
                     "l"(ad), "l"(bd), "r"(id), "r"(1));
    }
    asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                     smem_u32(&bar)),
                 "h"((unsigned short)3));
  }
  if (tid == 0) {
    asm volatile(
        "{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}\n" ::"r"(smem_u32(&bar)));
    long long t1 = clock64();
    out[blockIdx.x] = t1 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  cluster_sync();
  if (tid < 32) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

template <bool TS, int N>
void run(int sms) {
  long long* d;
  cudaMalloc(&d, sizeof(long long) * sms);
  auto k = probe<TS, N>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 48 * 1024);
  const int R1 = 64, R2 = 1088;
  static long long a[1024], b[1024];
  k<<<sms, 128, 48 * 1024>>>(R1, d);
  cudaMemcpy(a, d, sizeof(long long) * sms, cudaMemcpyDeviceToHost);
  k<<<sms, 128, 48 * 1024>>>(R2, d);
  cudaMemcpy(b, d, sizeof(long long) * sms, cudaMemcpyDeviceToHost);
  double s = 0;
  for (int i = 0; i < sms; i += 2) s += double(b[i] - a[i]) / (R2 - R1);
  const double cyc = s / (sms / 2);
  printf("2SM %s N=%-3d  %7.1f cycles/MMA per pair  (%6.0f MAC/clk/SM)  %s\n", TS ? "TS" : "SS", N, cyc,
         256.0 * N * 16 / cyc / 2, cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<false, 16>(sms);
  run<false, 32>(sms);
  run<false, 64>(sms);
  run<false, 128>(sms);
  run<false, 256>(sms);
  run<true, 32>(sms);
  run<true, 64>(sms);
  run<true, 128>(sms);
  run<true, 256>(sms);
  return 0;
}
