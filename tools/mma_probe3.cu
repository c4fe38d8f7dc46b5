// Microbenchmark: is the >= 45-cycle cost of a small tcgen05.mma (mma_probe.cu) a
// throughput limit or the latency of accumulating into the same TMEM columns?
// One elected thread issues R MMAs (kind::f16, bf16 -> f32, M = 128, cta_group::1)
// that rotate over C independent accumulators (D at column 256 + (i % C) * N), so
// consecutive MMAs only depend on each other every C instructions.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/bin/mma_probe3 tools/mma_probe3.cu
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

template <bool TS, int N, int C>
__global__ void probe(int R, long long* out) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int tid = threadIdx.x;
  for (int i = tid; i < 48 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0x3f803f80u;
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (tid < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = slot;
  if (tid == 0) {
    const uint32_t sA = smem_u32(sm), sB = smem_u32(sm + 16384);
    const uint64_t ad = desc(sA, 128 * 16, 128), bd = desc(sB, N * 16, 128);
    const uint32_t id = idesc(128, N);
    const uint32_t tA = tmem;  // A (TS) in columns [0, 8)
    long long t0 = clock64();
    for (int i = 0; i < R; i += C) {
#pragma unroll
      for (int c = 0; c < C; ++c) {
        const uint32_t tD = tmem + 256 + c * N;
        if (TS)
          asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(tD),
                       "r"(tA), "l"(bd), "r"(id), "r"(1));
        else
          asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tD),
                       "l"(ad), "l"(bd), "r"(id), "r"(1));
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
    asm volatile(
        "{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}\n" ::"r"(smem_u32(&bar)));
    long long t1 = clock64();
    out[blockIdx.x] = t1 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (tid < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

template <bool TS, int N, int C>
void run(int sms) {
  long long* d;
  cudaMalloc(&d, sizeof(long long) * sms);
  auto k = probe<TS, N, C>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 48 * 1024);
  const int R1 = 64, R2 = 1088;
  static long long a[1024], b[1024];
  k<<<sms, 128, 48 * 1024>>>(R1, d);
  cudaMemcpy(a, d, sizeof(long long) * sms, cudaMemcpyDeviceToHost);
  k<<<sms, 128, 48 * 1024>>>(R2, d);
  cudaMemcpy(b, d, sizeof(long long) * sms, cudaMemcpyDeviceToHost);
  double s = 0;
  for (int i = 0; i < sms; ++i) s += double(b[i] - a[i]) / (R2 - R1);
  const double cyc = s / sms;
  printf("%s N=%-3d chains=%d  %6.1f cycles/MMA  (%5.0f MAC/clk/SM)  %s\n", TS ? "TS" : "SS", N, C, cyc,
         128.0 * N * 16 / cyc, cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}


// W warps each issue R MMAs (own accumulator, own commit barrier): is the per-instruction
// cost a per-issuing-thread limit or a per-SM tensor-pipe limit?
template <int N, int W>
__global__ void probe_mw(int R, long long* out) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint64_t bar[8];
  __shared__ uint32_t slot;
  __shared__ long long tmax;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < 48 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0x3f803f80u;
  if (tid == 0) {
    for (int w = 0; w < 8; ++w) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[w])));
    asm volatile("fence.mbarrier_init.release.cluster;");
    tmax = 0;
  }
  if (tid < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = slot;
  long long t0 = clock64();
  if ((tid & 31) == 0 && warp < W) {
    const uint32_t sB = smem_u32(sm + 16384);
    const uint64_t bd = desc(sB, N * 16, 128);
    const uint32_t id = idesc(128, N);
    const uint32_t tD = tmem + 256 + warp * N, tA = tmem + warp * 8;
    for (int i = 0; i < R; ++i)
      asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(tD),
                   "r"(tA), "l"(bd), "r"(id), "r"(1));
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar[warp])));
    asm volatile(
        "{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}\n" ::"r"(smem_u32(&bar[warp])));
    long long t1 = clock64();
    atomicMax(reinterpret_cast<unsigned long long*>(&tmax), static_cast<unsigned long long>(t1 - t0));
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (tid == 0) out[blockIdx.x] = tmax;
  if (tid < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

template <int N, int W>
void run_mw(int sms) {
  long long* d;
  cudaMalloc(&d, sizeof(long long) * sms);
  auto k = probe_mw<N, W>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 48 * 1024);
  const int R1 = 64, R2 = 1088;
  static long long a[1024], b[1024];
  k<<<sms, 256, 48 * 1024>>>(R1, d);
  cudaMemcpy(a, d, sizeof(long long) * sms, cudaMemcpyDeviceToHost);
  k<<<sms, 256, 48 * 1024>>>(R2, d);
  cudaMemcpy(b, d, sizeof(long long) * sms, cudaMemcpyDeviceToHost);
  double s = 0;
  for (int i = 0; i < sms; ++i) s += double(b[i] - a[i]) / (R2 - R1);
  const double cyc = s / sms / W;
  printf("TS N=%-3d issuing warps=%d  %6.1f cycles/MMA per SM  (%5.0f MAC/clk/SM)  %s\n", N, W, cyc,
         128.0 * N * 16 / cyc, cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<false, 16, 1>(sms);
  run<false, 16, 4>(sms);
  run<false, 16, 8>(sms);
  run<false, 64, 1>(sms);
  run<false, 64, 2>(sms);
  run<false, 64, 4>(sms);
  run<true, 16, 1>(sms);
  run<true, 16, 4>(sms);
  run<true, 16, 8>(sms);
  run<true, 64, 1>(sms);
  run<true, 64, 2>(sms);
  run<true, 64, 4>(sms);
  run<true, 128, 2>(sms);
  run_mw<16, 1>(sms);
  run_mw<16, 2>(sms);
  run_mw<16, 4>(sms);
  run_mw<64, 2>(sms);
  run_mw<64, 4>(sms);
  return 0;
}
