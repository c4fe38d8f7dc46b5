// Read/write-mix copy ceiling: how fast can a plain streaming kernel move a config's bytes when
// reads and writes are in the config's proportion?  (MEASURED_PEAKS.json's hbm_gbs is a 50/50
// copy; config 3 reads 132 B and writes 336 B per pixel, config 1 reads 324 and writes 372.)
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bin/rw_ceiling tools/rw_ceiling.cu
//   tools/bin/rw_ceiling <read_bytes> <write_bytes> [reps]
//
// One launch reads `read_bytes` and writes `write_bytes` as two coalesced float4 streams
// (grid-stride, 148 x 8 CTAs of 256 threads, streaming cache hints); two buffer sets alternate
// so nothing stays in L2.  Prints GB/s of (read + write) bytes, CUDA events, best and median.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>

__global__ void rw_kernel(const float4* __restrict__ in, float4* __restrict__ out, long long nr, long long nw) {
  const long long n = nr > nw ? nr : nw;
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
    if (i < nr) {
      const float4 v = __ldcs(in + i);
      acc.x += v.x;
      acc.y += v.y;
      acc.z += v.z;
      acc.w += v.w;
    }
    if (i < nw) __stcs(out + i, acc);
  }
}

int main(int argc, char** argv) {
  if (argc < 3) {
    std::fprintf(stderr, "usage: rw_ceiling <read_bytes> <write_bytes> [reps]\n");
    return 2;
  }
  const long long rb = std::atoll(argv[1]), wb = std::atoll(argv[2]);
  const int reps = argc > 3 ? std::atoi(argv[3]) : 20;
  const long long nr = rb / 16, nw = wb / 16;
  float4 *in[2], *out[2];
  for (int s = 0; s < 2; ++s) {
    cudaMalloc(&in[s], nr * 16 + 16);
    cudaMalloc(&out[s], nw * 16 + 16);
    cudaMemset(in[s], 0, nr * 16 + 16);
  }
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int grid = sms * 8;
  for (int w = 0; w < 4; ++w) rw_kernel<<<grid, 256>>>(in[w & 1], out[w & 1], nr, nw);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  std::vector<float> ms;
  for (int r = 0; r < reps; ++r) {
    cudaEventRecord(e0);
    rw_kernel<<<grid, 256>>>(in[r & 1], out[r & 1], nr, nw);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float t = 0.f;
    cudaEventElapsedTime(&t, e0, e1);
    ms.push_back(t);
  }
  std::sort(ms.begin(), ms.end());
  const double bytes = static_cast<double>(nr * 16 + nw * 16);
  std::printf("{\"read_bytes\": %lld, \"write_bytes\": %lld, \"best_gbs\": %.1f, \"median_gbs\": %.1f, \"median_ms\": %.4f, \"err\": \"%s\"}\n",
              nr * 16, nw * 16, bytes / (ms.front() * 1e6), bytes / (ms[ms.size() / 2] * 1e6), ms[ms.size() / 2],
              cudaGetErrorString(cudaGetLastError()));
  return 0;
}
