// Microbenchmark: legacy warp-level tensor-core MMA (mma.sync.m16n8k16 bf16 -> fp32, SASS HMMA) on
// B200, per SM, against the tcgen05 rate (4096 bf16 MAC/clk/SM measured by tools/mma_probe4.cu).
// Question for the config-5a MLP: could register-resident accumulators (no TMEM, no mbarrier round
// trips) carry the 3 -> 64 -> 64 -> 6 network faster than the latency-bound tcgen05 chain?
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bin/hmma_probe tools/hmma_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ void hmma(float (&d)[4], const uint32_t (&a)[4], const uint32_t (&b)[2]) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}

template <int CHAINS>
__global__ void probe(float* out, int iters) {
  uint32_t a[4], b[2];
  for (int i = 0; i < 4; ++i) a[i] = 0x3f803f80u + threadIdx.x + i;
  for (int i = 0; i < 2; ++i) b[i] = 0x3f803f80u + 7 * threadIdx.x + i;
  float d[CHAINS][4];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c)
#pragma unroll
    for (int i = 0; i < 4; ++i) d[c][i] = 0.f;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) hmma(d[c], a, b);
  }
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c)
#pragma unroll
    for (int i = 0; i < 4; ++i) s += d[c][i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int CHAINS>
void run(int warps) {
  float* out;
  cudaMalloc(&out, sizeof(float) * 148 * 1024);
  const int iters = 4000;
  probe<CHAINS><<<148, 32 * warps>>>(out, 10);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  probe<CHAINS><<<148, 32 * warps>>>(out, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  int clk;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const double macs = 148.0 * warps * iters * CHAINS * 16 * 8 * 16;
  const double per_sm_clk = macs / 148.0 / (ms * 1e-3 * clk * 1e3);
  std::printf("HMMA m16n8k16 bf16  chains/warp=%d warps/SM=%2d  %7.1f MAC/clk/SM (%4.1f%% of tcgen05 4096)  %s\n", CHAINS,
              warps, per_sm_clk, per_sm_clk / 4096 * 100, cudaGetErrorString(cudaGetLastError()));
  cudaFree(out);
}

int main() {
  for (int w : {4, 8, 16, 32}) {
    run<1>(w);
    run<4>(w);
    run<8>(w);
  }
  return 0;
}
