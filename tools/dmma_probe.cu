// Microbenchmark: does the fp64 tensor-core path (mma.sync m8n8k4 f64, DMMA) run beside the
// fp64 vector pipe (DFMA) on B200, or share it?  Per SM: DMMA-only, DFMA-only and a warp mix.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bin/dmma_probe tools/dmma_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

template <int MODE>  // 0 DMMA, 1 DFMA, 2 half the warps DMMA / half DFMA
__global__ void probe(double* out, int iters) {
  double acc[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) acc[i] = threadIdx.x * 1e-9 + i;
  const double a = 1.0 + threadIdx.x * 1e-12, b = 0.999999;
  const bool tensor = MODE == 0 || (MODE == 2 && (threadIdx.x / 32) % 2 == 0);
  for (int it = 0; it < iters; ++it) {
    if (tensor) {
#pragma unroll
      for (int i = 0; i < 8; ++i) dmma(acc[2 * i], acc[2 * i + 1], a, b);
    } else {
#pragma unroll
      for (int r = 0; r < 16; ++r)   // 256 FMAs per thread per iteration = 8 DMMA's worth per warp
#pragma unroll
        for (int i = 0; i < 16; ++i) acc[i] = fma(acc[i], b, a);
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int MODE>
void run(const char* name, int warps) {
  double* out;
  cudaMalloc(&out, sizeof(double) * 148 * 1024);
  const int iters = 2000;
  probe<MODE><<<148, 32 * warps>>>(out, 10);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  probe<MODE><<<148, 32 * warps>>>(out, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  int clk;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  // FMAs: DMMA 256 per warp-instruction; DFMA 1 per thread
  double fma_total;
  if (MODE == 0) fma_total = 148.0 * warps * iters * 8 * 256;
  else if (MODE == 1) fma_total = 148.0 * warps * 32 * iters * 256;
  else fma_total = 148.0 * (warps / 2) * iters * 8 * 256 + 148.0 * (warps / 2) * 32 * iters * 256;
  const double per_sm_clk = fma_total / 148.0 / (ms * 1e-3 * clk * 1e3);
  std::printf("%-28s warps/SM=%2d  %8.1f fp64 FMA/clk/SM  (%.3f ms)  %s\n", name, warps, per_sm_clk, ms,
              cudaGetErrorString(cudaGetLastError()));
  cudaFree(out);
}

int main() {
  for (int w : {4, 8, 16}) {
    run<0>("DMMA m8n8k4", w);
    run<1>("DFMA", w);
    run<2>("half DMMA + half DFMA", w);
  }
  return 0;
}
