// Microbenchmark: the ~45-cycle cost per tcgen05.mma of one issuing thread (mma_probe3.cu) —
// is it the compiler's per-thread "waterfall" (ELECT / R2UR.BROADCAST / BRA.U.ANY around
// every UTCHMMA when the MMA sits under `if (tid == 0)` with register operands), and does
// issuing from a warp-uniform context (elect.sync inside the asm, operands uniform) avoid it?
// One thread / warp issues R TS MMAs (bf16, M = 128, N = 64) over C = 4 accumulators.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/bin/mma_probe4 tools/mma_probe4.cu
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

template <int MODE, int N>  // 0: if (tid == 0) {mma}; 1: whole warp, elect.sync inside the asm
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
  const uint32_t sB = smem_u32(sm + 16384);
  const uint64_t bd = desc(sB, N * 16, 128);
  constexpr uint32_t id = idesc(128, N);
  long long t0 = 0, t1 = 0;
  if (MODE == 0) {
    if (tid == 0) {
      t0 = clock64();
      for (int i = 0; i < R; i += 4) {
#pragma unroll
        for (int c = 0; c < 4; ++c)
          asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(256u + c * N),
                       "r"(0u), "l"(bd), "r"(id), "r"(1));
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
    }
  } else {
    if (tid < 32) {
      t0 = clock64();
      for (int i = 0; i < R; i += 4) {
#pragma unroll
        for (int c = 0; c < 4; ++c)
          asm volatile("{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, 1;\n}\n" ::"r"(256u + c * N),
                       "r"(0u), "l"(bd), "r"(id));
      }
      asm volatile("{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}\n" ::"r"(smem_u32(&bar)));
    }
  }
  if (tid == 0) {
    asm volatile("{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}\n" ::"r"(smem_u32(&bar)));
    t1 = clock64();
    out[blockIdx.x] = t1 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (tid < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(slot));
}

template <int MODE, int N>
void run(int sms) {
  long long* d;
  cudaMalloc(&d, sizeof(long long) * sms);
  auto k = probe<MODE, N>;
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
  printf("%-34s N=%-3d %6.1f cycles/MMA  (%5.0f MAC/clk/SM)  %s\n",
         MODE == 0 ? "if (tid == 0) { mma }" : "warp: elect.sync + @p mma (asm)", N, cyc, 128.0 * N * 16 / cyc,
         cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<0, 16>(sms);
  run<1, 16>(sms);
  run<0, 64>(sms);
  run<1, 64>(sms);
  run<0, 128>(sms);
  run<1, 128>(sms);
  return 0;
}
