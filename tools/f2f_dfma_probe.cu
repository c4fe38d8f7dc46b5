// Microbenchmark for the loss kernel's pass-1 instruction mix (config 5b): per "wavelength" two
// fp32 values widened to fp64 and 12 DFMAs with a warp-uniform E operand (6 codes x 2 inputs).
// Variants: conversion by F2F (cvt.f64.f32), by integer bit manipulation (ALU pipe), or none
// (operands already fp64); warps per SM 4..32.  Reports fp64 FMAs per clock per SM.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bin/f2f_dfma_probe tools/f2f_dfma_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__constant__ double cE[6 * 81];

// exact float -> double for finite floats by integer ops (normal and zero; denormals flushed to
// a signed zero): sign | (exp + 896) << 52 | mantissa << 29
__device__ __forceinline__ double f2d_int(float f) {
  const uint32_t u = __float_as_uint(f);
  const uint32_t mag = u & 0x7fffffffu;
  uint32_t hi = (mag >> 3) + 0x38000000u;
  hi = (mag < 0x00800000u) ? 0u : hi;  // zero / denormal -> 0
  hi |= u & 0x80000000u;
  const uint32_t lo = mag << 29;
  return __hiloint2double(static_cast<int>(hi), static_cast<int>(lo));
}

template <int MODE>  // 0 F2F, 1 integer widening, 2 no conversion (fp64 loads)
__global__ void probe(double* out, int iters) {
  __shared__ double buf[2 * 32 * 81];  // fp64 rows (MODE 2) or fp32 rows (the first half)
  float* sa = reinterpret_cast<float*>(buf);
  float* sb = sa + 32 * 81;
  double* da = buf;
  double* db = buf + 32 * 81;
  const int lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 32 * 81; i += blockDim.x) {
    if (MODE == 2) {
      da[i] = 0.5 + i * 1e-4;
      db[i] = 0.25 + i * 1e-4;
    } else {
      sa[i] = 0.5f + i * 1e-4f;
      sb[i] = 0.25f + i * 1e-4f;
    }
  }
  __syncthreads();
  double za[6] = {0, 0, 0, 0, 0, 0}, zb[6] = {0, 0, 0, 0, 0, 0};
  for (int it = 0; it < iters; ++it) {
    const int base = (it * 27) % 54;
#pragma unroll 27
    for (int l = 0; l < 27; ++l) {
      double va, vb;
      if (MODE == 2) {
        va = da[lane * 81 + base + l];
        vb = db[lane * 81 + base + l];
      } else {
        const float fa = sa[lane * 81 + base + l], fb = sb[lane * 81 + base + l];
        va = MODE == 0 ? static_cast<double>(fa) : f2d_int(fa);
        vb = MODE == 0 ? static_cast<double>(fb) : f2d_int(fb);
      }
#pragma unroll
      for (int j = 0; j < 6; ++j) {
        const double e = cE[j * 81 + base + l];
        za[j] = fma(e, va, za[j]);
        zb[j] = fma(e, vb, zb[j]);
      }
    }
  }
  double s = 0;
#pragma unroll
  for (int j = 0; j < 6; ++j) s += za[j] * zb[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// Pass-2 mix: per wavelength r = (D zp)_l - a_l b_l (6 DFMA chain from an exact DMUL), acc += r^2.
// MODE 10: D rows from shared memory (3 LDS.128 broadcasts, the kernel's table), one acc chain;
// 11: same with three partial sums; 12: D from the constant bank (uniform), one acc chain.
template <int MODE>
__global__ void probe2(double* out, int iters) {
  __shared__ float sa[32 * 81], sb[32 * 81];
  __shared__ double2 td[81 * 3];
  const int lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 32 * 81; i += blockDim.x) {
    sa[i] = 0.5f + i * 1e-4f;
    sb[i] = 0.25f + i * 1e-4f;
  }
  for (int i = threadIdx.x; i < 81 * 3; i += blockDim.x) td[i] = make_double2(0.01 * i, 0.02 * i);
  __syncthreads();
  double zp[6];
#pragma unroll
  for (int j = 0; j < 6; ++j) zp[j] = 0.1 * (j + 1) + threadIdx.x * 1e-9;
  double acc[3] = {0, 0, 0};
  for (int it = 0; it < iters; ++it) {
    const int base = (it * 27) % 54;
#pragma unroll 27
    for (int l = 0; l < 27; ++l) {
      double r;
      if (MODE == 13 || MODE == 14) {  // a_l b_l precomputed (fp64, from shared memory): no F2F, no DMUL
        r = -reinterpret_cast<const double*>(sa)[(lane * 81 + base + l) >> 1];
      } else {
        const float fa = sa[lane * 81 + base + l], fb = sb[lane * 81 + base + l];
        r = -(static_cast<double>(fa) * static_cast<double>(fb));
      }
      double d[6];
      if (MODE == 12 || MODE == 14) {
#pragma unroll
        for (int j = 0; j < 6; ++j) d[j] = cE[(base + l) * 6 + j];
      } else {
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          const double2 v = td[(base + l) * 3 + c];
          d[2 * c] = v.x;
          d[2 * c + 1] = v.y;
        }
      }
#pragma unroll
      for (int j = 0; j < 6; ++j) r = fma(d[j], zp[j], r);
      if (MODE == 11) acc[l % 3] = fma(r, r, acc[l % 3]);
      else acc[0] = fma(r, r, acc[0]);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc[0] + acc[1] + acc[2];
}

template <int MODE>
void run2(const char* name, int warps) {
  double* out;
  cudaMalloc(&out, sizeof(double) * 148 * 1024);
  const int iters = 400;
  probe2<MODE><<<148, 32 * warps>>>(out, 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  probe2<MODE><<<148, 32 * warps>>>(out, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  int clk;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const double fma_total = 148.0 * warps * 32 * iters * 27 * 8;  // DMUL + 6 DFMA + r^2
  const double per_sm_clk = fma_total / 148.0 / (ms * 1e-3 * clk * 1e3);
  std::printf("%-22s warps/SM=%2d  %6.1f fp64 op/clk/SM  (%.3f ms)  %s\n", name, warps, per_sm_clk, ms,
              cudaGetErrorString(cudaGetLastError()));
  cudaFree(out);
}

// Pass 2 on the fp64 tensor core (mma.sync m8n8k4 f64): a warp = 32 pairs x 32 wavelengths
// (27 real) x 8 codes (6 real); D^T fragments in registers, C initialised to -a b.
__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}
__global__ void probe_dmma(double* out, int iters) {
  __shared__ float sa[32 * 81], sb[32 * 81];
  const int lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 32 * 81; i += blockDim.x) {
    sa[i] = 0.5f + i * 1e-4f;
    sb[i] = 0.25f + i * 1e-4f;
  }
  __syncthreads();
  double bf[4][2];  // B fragments: D[wl = 8n + lane/4][code = 4k + lane%4]
#pragma unroll
  for (int n = 0; n < 4; ++n)
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const int wl = 8 * n + lane / 4, code = 4 * k + lane % 4;
      bf[n][k] = (wl < 27 && code < 6) ? cE[wl * 6 + code] : 0.0;
    }
  double zp[6];
#pragma unroll
  for (int j = 0; j < 6; ++j) zp[j] = 0.1 * (j + 1) + threadIdx.x * 1e-9;
  double acc = 0.0;
  for (int it = 0; it < iters; ++it) {
    const int base = (it * 27) % 54;
    // A fragments: zp of pair 8m + lane/4, code 4k + lane%4 (shuffles from the owning lane)
    double af[4][2];
#pragma unroll
    for (int m = 0; m < 4; ++m)
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        double v[4];
#pragma unroll
        for (int c = 0; c < 4; ++c) v[c] = (4 * k + c < 6) ? __shfl_sync(0xffffffffu, zp[(4 * k + c) % 6], 8 * m + lane / 4) : 0.0;
        const int c = lane % 4;
        af[m][k] = c == 0 ? v[0] : c == 1 ? v[1] : c == 2 ? v[2] : v[3];
      }
#pragma unroll
    for (int m = 0; m < 4; ++m)
#pragma unroll
      for (int n = 0; n < 4; ++n) {
        const int pr = 8 * m + lane / 4, wl = 8 * n + 2 * (lane % 4);
        double c0 = wl < 27 ? -(double(sa[pr * 81 + base + wl]) * double(sb[pr * 81 + base + wl])) : 0.0;
        double c1 = wl + 1 < 27 ? -(double(sa[pr * 81 + base + wl + 1]) * double(sb[pr * 81 + base + wl + 1])) : 0.0;
        dmma(c0, c1, af[m][0], bf[n][0]);
        dmma(c0, c1, af[m][1], bf[n][1]);
        acc = fma(c0, c0, acc);
        acc = fma(c1, c1, acc);
      }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

void run_dmma(int warps) {
  double* out;
  cudaMalloc(&out, sizeof(double) * 148 * 1024);
  const int iters = 400;
  probe_dmma<<<148, 32 * warps>>>(out, 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  probe_dmma<<<148, 32 * warps>>>(out, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  int clk;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  // useful work counted as in probe2: 27 wavelengths x 8 ops per pair
  const double fma_total = 148.0 * warps * 32 * iters * 27 * 8;
  const double per_sm_clk = fma_total / 148.0 / (ms * 1e-3 * clk * 1e3);
  std::printf("%-22s warps/SM=%2d  %6.1f fp64 op/clk/SM  (%.3f ms)  %s\n", "pass 2, DMMA", warps, per_sm_clk, ms,
              cudaGetErrorString(cudaGetLastError()));
  cudaFree(out);
}

// Layout check: C = A(8x4) B(4x8) with A[i][k] = i + 10k, B[k][j] = k + 100 j.
__global__ void dmma_layout(double* out) {
  const int lane = threadIdx.x;
  const double a = (lane >> 2) + 10.0 * (lane & 3);
  const double b = (lane & 3) + 100.0 * (lane >> 2);
  double c0 = 0, c1 = 0;
  dmma(c0, c1, a, b);
  out[lane * 2] = c0;
  out[lane * 2 + 1] = c1;
}

template <int MODE>
void run(const char* name, int warps) {
  double* out;
  cudaMalloc(&out, sizeof(double) * 148 * 1024);
  const int iters = 400;
  probe<MODE><<<148, 32 * warps>>>(out, 4);
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
  const double fma_total = 148.0 * warps * 32 * iters * 27 * 12;
  const double per_sm_clk = fma_total / 148.0 / (ms * 1e-3 * clk * 1e3);
  std::printf("%-22s warps/SM=%2d  %6.1f fp64 FMA/clk/SM  (%.3f ms)  %s\n", name, warps, per_sm_clk, ms,
              cudaGetErrorString(cudaGetLastError()));
  cudaFree(out);
}

int main() {
  double h[6 * 81];
  for (int i = 0; i < 6 * 81; ++i) h[i] = 0.01 * (i % 17) + 0.001;
  cudaMemcpyToSymbol(cE, h, sizeof(h));
  // one CTA per SM by grid (148 CTAs): warps per SM = CTA size
  for (int w : {4, 8, 12, 16, 24, 32}) {
    run<0>("F2F widening", w);
    run<1>("integer widening", w);
    run<2>("fp64 operands", w);
  }
  {
    double* d;
    cudaMalloc(&d, 64 * sizeof(double));
    dmma_layout<<<1, 32>>>(d);
    double h2[64];
    cudaMemcpy(h2, d, sizeof(h2), cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int lane = 0; lane < 32; ++lane)
      for (int i = 0; i < 2; ++i) {
        const int r = lane >> 2, c = (lane & 3) * 2 + i;
        double want = 0;
        for (int k = 0; k < 4; ++k) want += (r + 10.0 * k) * (k + 100.0 * c);
        bad += h2[lane * 2 + i] != want;
      }
    std::printf("DMMA m8n8k4 layout (A row: i = lane/4, k = lane%%4; B col: k = lane%%4, j = lane/4; "
                "C: i = lane/4, j = 2 (lane%%4) + {0,1}): %s\n", bad ? "MISMATCH" : "ok");
  }
  for (int w : {4, 8, 12, 16, 24}) run_dmma(w);
  for (int w : {4, 8, 12, 16, 24, 32}) {
    run2<10>("pass 2, D smem", w);
    run2<11>("pass 2, D smem, acc x3", w);
    run2<12>("pass 2, D const", w);
    run2<13>("pass 2, D smem, ab f64", w);
    run2<14>("pass 2, D const, ab f64", w);
  }
  return 0;
}
