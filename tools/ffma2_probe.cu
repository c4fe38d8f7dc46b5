// Microbenchmark: FFMA2 (fma.rn.f32x2) vs FFMA throughput and dependent latency on one SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bin/ffma2_probe tools/ffma2_probe.cu
#include <cstdio>
#include <cuda_runtime.h>
// Packed fp32 FMA (same helper shape as a kernel would use).
__device__ __forceinline__ float2 ffma2(float2 a, float s, float2 c) {
  unsigned long long ar, sr, cr, d;
  asm("mov.b64 %0, {%1, %2};" : "=l"(ar) : "f"(a.x), "f"(a.y));
  asm("mov.b64 %0, {%1, %1};" : "=l"(sr) : "f"(s));
  asm("mov.b64 %0, {%1, %2};" : "=l"(cr) : "f"(c.x), "f"(c.y));
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(ar), "l"(sr), "l"(cr));
  float2 r;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(r.x), "=f"(r.y) : "l"(d));
  return r;
}

template <bool PAIR, int CH>
__global__ void k(int R, float s, float* out, long long* cyc) {
  float2 a[CH];
  for (int c = 0; c < CH; ++c) a[c] = make_float2(threadIdx.x * 1e-3f + c, c * 0.5f);
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < R; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      if (PAIR) {
        a[c] = ffma2(a[c], s, make_float2(0.25f, 0.5f));
      } else {
        a[c].x = fmaf(a[c].x, s, 0.25f);
        a[c].y = fmaf(a[c].y, s, 0.5f);
      }
    }
  }
  __syncthreads();
  long long t1 = clock64();
  float t = 0.f;
  for (int c = 0; c < CH; ++c) t += a[c].x + a[c].y;
  out[blockIdx.x * blockDim.x + threadIdx.x] = t;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <bool PAIR, int CH>
void run(int threads) {
  float* o;
  long long* c;
  cudaMalloc(&o, 4 * 1024 * 148);
  cudaMalloc(&c, 8 * 148);
  const int R = 4096;
  k<PAIR, CH><<<148, threads>>>(R, 0.999f, o, c);
  k<PAIR, CH><<<148, threads>>>(R, 0.999f, o, c);
  long long h;
  cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  const double fmas = 2.0 * CH * R * threads;
  printf("%s chains=%d threads=%4d: %7.1f fp32 FMA/clk/SM, %6.2f cycles per dependent step  %s\n",
         PAIR ? "FFMA2" : "FFMA ", CH, threads, fmas / h, double(h) / R, cudaGetErrorString(cudaGetLastError()));
  cudaFree(o);
  cudaFree(c);
}

int main() {
  run<false, 1>(32);
  run<true, 1>(32);
  run<false, 4>(32);
  run<true, 4>(32);
  run<false, 8>(128);
  run<true, 8>(128);
  run<false, 8>(512);
  run<true, 8>(512);
  run<false, 8>(1024);
  run<true, 8>(1024);
  return 0;
}
