// Microbenchmark: latency of a dependent fp64 add chain (DADD) and of add + select, one
// warp, as in the ordered batch reductions of hc_train.cu.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false -o tools/bin/dadd_probe tools/dadd_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void chain_add(const double* x, int n, double* out, long long* cyc) {
  double acc = 0.0;
  const double a = x[threadIdx.x], b = x[threadIdx.x + 32];
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
    acc = acc + a;
    acc = acc + b;
  }
  long long t1 = clock64();
  out[threadIdx.x] = acc;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}

__global__ void chain_sel(const double* x, int n, double* out, long long* cyc) {
  double acc = 0.0;
  const double a = x[threadIdx.x], b = x[threadIdx.x + 32];
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
    const double s = acc + a;
    acc = (a != 0.0) ? s : acc;
    acc = acc + b;
  }
  long long t1 = clock64();
  out[threadIdx.x] = acc;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}

int main() {
  double *x, *out;
  long long* cyc;
  cudaMalloc(&x, 64 * 8);
  cudaMalloc(&out, 64 * 8);
  cudaMalloc(&cyc, 8);
  double hx[64];
  for (int i = 0; i < 64; ++i) hx[i] = 1e-3 * (i + 1);
  cudaMemcpy(x, hx, sizeof hx, cudaMemcpyHostToDevice);
  long long c1 = 0, c2 = 0;
  const int n = 100000;
  chain_add<<<1, 32>>>(x, n, out, cyc);
  chain_add<<<1, 32>>>(x, n, out, cyc);
  cudaMemcpy(&c1, cyc, 8, cudaMemcpyDeviceToHost);
  chain_sel<<<1, 32>>>(x, n, out, cyc);
  chain_sel<<<1, 32>>>(x, n, out, cyc);
  cudaMemcpy(&c2, cyc, 8, cudaMemcpyDeviceToHost);
  printf("dependent DADD: %.1f cycles/add; add+select+add: %.1f cycles/iteration (%s)\n", double(c1) / (2.0 * n),
         double(c2) / n, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
