// Microbenchmark: round-trip latencies of the MLP's building blocks on one idle SM
// (one CTA, one issuing thread), to tell an intrinsic latency chain from contention.
//   (a) n MMAs (kind::f16, M = 128, N, K = 16 each, SS or TS) + commit -> mbarrier wait, serial
//   (b) 4 warps: tcgen05.ld 64 columns + wait::ld
//   (c) 4 warps: tcgen05.st 32 columns + wait::st
//   (d) ping-pong: issuer MMA + commit -> 4 epilogue warps wait, ld 64 cols, st 32 cols,
//       fence, arrive -> issuer waits (one hidden layer of mlp_kernel, serially)
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/bin/mma_latency tools/mma_latency.cu
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
__device__ __forceinline__ void commit(uint64_t* b) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(b)));
}
__device__ __forceinline__ void mma(bool ts, uint32_t tD, uint32_t tA, uint64_t ad, uint64_t bd, uint32_t id, int acc) {
  if (ts)
    asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(tD),
                 "r"(tA), "l"(bd), "r"(id), "r"(acc));
  else
    asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tD),
                 "l"(ad), "l"(bd), "r"(id), "r"(acc));
}

// mode 0: (a); mode 1: (b); mode 2: (c); mode 3: (d)
__global__ void probe(int mode, int ts, int N, int nmma, int R, long long* out) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint64_t bar[2];
  __shared__ uint64_t wbar[8];
  __shared__ uint32_t slot;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < 48 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0x3c003c00u;
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[0])));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 4;" ::"r"(smem_u32(&bar[1])));
    for (int w = 0; w < 8; ++w) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&wbar[w])));
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
  const uint32_t lane_off = static_cast<uint32_t>((warp & 3) * 32) << 16;
  const uint64_t ad = desc(smem_u32(sm), 128 * 16, 128), bd = desc(smem_u32(sm + 16384), N * 16, 128);
  const uint32_t id = idesc(128, N);
  long long t0 = clock64();
  if (mode == 0) {
    if (tid == 0) {
      for (int i = 0; i < R; ++i) {
        for (int j = 0; j < nmma; ++j) mma(ts, tmem + 256, tmem + j * 8, ad, bd, id, j > 0);
        commit(&bar[0]);
        wait_bar(&bar[0], i & 1);
        asm volatile("tcgen05.fence::after_thread_sync;");
      }
    }
  } else if (mode == 4) {  // W = nmma >> 8 warps, each (nmma & 255) MMAs + commit + wait, R times
    const int W = nmma >> 8, n = nmma & 255;
    if (warp < W && (tid & 31) == 0) {
      for (int i = 0; i < R; ++i) {
        for (int j = 0; j < n; ++j) mma(ts, tmem + 128 + warp * 64, tmem + j * 8, ad, bd, id, j > 0);
        commit(&wbar[warp]);
        wait_bar(&wbar[warp], i & 1);
        asm volatile("tcgen05.fence::after_thread_sync;");
      }
    }
    __syncthreads();
  } else if (mode == 1 || mode == 2) {
    if (warp < 4) {
      uint32_t v[16];
      for (int i = 0; i < R; ++i) {
        if (mode == 1) {
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            asm volatile(
                "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                  "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
                : "r"(tmem + 256 + q * 16 + lane_off));
          }
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
          if (v[0] == 12345u && v[15] == 7u) out[1] = 1;
        } else {
#pragma unroll
          for (int q = 0; q < 16; ++q) v[q] = i + q;
#pragma unroll
          for (int q = 0; q < 2; ++q)
            asm volatile(
                "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
                    tmem + q * 16 + lane_off),
                "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]),
                "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
                : "memory");
          asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        }
      }
    }
  } else {
    if (warp == 4) {
      for (int i = 0; i < R; ++i) {
        if (tid == 128) {
          for (int j = 0; j < nmma; ++j) mma(ts, tmem + 256, tmem + j * 8, ad, bd, id, j > 0);
          commit(&bar[0]);
        }
        __syncwarp();
        wait_bar(&bar[1], i & 1);
        asm volatile("tcgen05.fence::after_thread_sync;");
      }
    } else if (warp < 4) {
      uint32_t v[4][16];
      for (int i = 0; i < R; ++i) {
        wait_bar(&bar[0], i & 1);
        asm volatile("tcgen05.fence::after_thread_sync;");
#pragma unroll
        for (int q = 0; q < 4; ++q)
          asm volatile(
              "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
              : "=r"(v[q][0]), "=r"(v[q][1]), "=r"(v[q][2]), "=r"(v[q][3]), "=r"(v[q][4]), "=r"(v[q][5]),
                "=r"(v[q][6]), "=r"(v[q][7]), "=r"(v[q][8]), "=r"(v[q][9]), "=r"(v[q][10]), "=r"(v[q][11]),
                "=r"(v[q][12]), "=r"(v[q][13]), "=r"(v[q][14]), "=r"(v[q][15])
              : "r"(tmem + 256 + q * 16 + lane_off));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int q = 0; q < 2; ++q)
          asm volatile(
              "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
                  tmem + 128 + q * 16 + lane_off),
              "r"(v[q][0] & 0x7f7f7f7fu), "r"(v[q][1]), "r"(v[q][2]), "r"(v[q][3]), "r"(v[q][4]), "r"(v[q][5]),
              "r"(v[q][6]), "r"(v[q][7]), "r"(v[q + 2][8]), "r"(v[q + 2][9]), "r"(v[q + 2][10]), "r"(v[q + 2][11]),
              "r"(v[q + 2][12]), "r"(v[q + 2][13]), "r"(v[q + 2][14]), "r"(v[q + 2][15])
              : "memory");
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        asm volatile("tcgen05.fence::before_thread_sync;");
        __syncwarp();
        if ((tid & 31) == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&bar[1])));
      }
    }
  }
  long long t1 = clock64();
  if (tid == 0 || tid == 128) out[blockIdx.x * 2 + (tid == 128)] = t1 - t0;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

void run(const char* name, int mode, int ts, int N, int nmma) {
  long long* d;
  cudaMalloc(&d, sizeof(long long) * 4);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 48 * 1024);
  const int R1 = 16, R2 = 528;
  long long a[2], b[2];
  probe<<<1, 160, 48 * 1024>>>(mode, ts, N, nmma, R1, d);
  cudaMemcpy(a, d, sizeof(a), cudaMemcpyDeviceToHost);
  probe<<<1, 160, 48 * 1024>>>(mode, ts, N, nmma, R2, d);
  cudaMemcpy(b, d, sizeof(b), cudaMemcpyDeviceToHost);
  printf("%-44s %7.1f cycles per round trip  %s\n", name, double(b[0] - a[0]) / (R2 - R1),
         cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}

int main() {
  run("SS N=64 x1 + commit + wait", 0, 0, 64, 1);
  run("TS N=64 x1 + commit + wait", 0, 1, 64, 1);
  run("TS N=64 x4 + commit + wait", 0, 1, 64, 4);
  run("TS N=64 x5 + commit + wait", 0, 1, 64, 5);
  run("TS N=16 x4 + commit + wait", 0, 1, 16, 4);
  run("TS N=128 x4 + commit + wait", 0, 1, 128, 4);
  run("4 warps: ld 64 cols + wait::ld", 1, 0, 64, 0);
  run("4 warps: st 32 cols + wait::st", 2, 0, 64, 0);
  run("ping-pong SS N=64 x1 -> ld64/st32 -> arrive", 3, 0, 64, 1);
  run("ping-pong TS N=64 x5 -> ld64/st32 -> arrive", 3, 1, 64, 5);
  run("ping-pong TS N=16 x4 -> ld64/st32 -> arrive", 3, 1, 16, 4);
  // mode 4: is a commit round trip a per-warp latency or a per-SM serialising cost?
  const int ns[3] = {1, 2, 5};
  for (int w = 1; w <= 4; w *= 2)
    for (int q = 0; q < 3; ++q) {
      char name[64];
      snprintf(name, sizeof name, "%d warps x (TS N=64 x%d + commit + wait)", w, ns[q]);
      run(name, 4, 1, 64, (w << 8) | ns[q]);
    }
  return 0;
}
