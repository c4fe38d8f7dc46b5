// hadacodec-b200: RGB -> code upsampler MLP (config 5a) on 5th-gen tensor cores.
//
// Reference: forward (upsampler.cpp:42-72) and upsample's non-negative output
// (upsampler.cpp:179-190); BASELINE config 5 fixes the net to 3 -> 64 -> 64 -> 6
// with ReLU, ReLU and a softplus(beta = 1) head (codec.cpp:8-12), bf16 operands,
// fp32 accumulation.
//
// One 128-pixel tile = one M = 128 tcgen05 tile row block:
//   L1  D[128 x 64]  = A1[128 x 16] . W1'^T   A1 = (r, g, b, 1, 0...) bf16, W1' = [W1 | b1 | 0]
//   L2  D[128 x 64]  = A2[128 x 64] . W2^T    A2 = bf16(relu(L1)),   epilogue adds b2
//   L3  D[128 x 16]  = A3[128 x 64] . W3'^T   A3 = bf16(relu(L2 + b2)), W3' = W3 padded to 16 rows
//   out = softplus(L3[:, :k] + b3)
// Operands live in shared memory in the canonical no-swizzle K-major UMMA layout
// (8-row x 16-byte core matrices; element (r, k) at (k/8)*LBO + r*16 + (k%8)*2),
// accumulators in TMEM (one 64-column allocation per CTA, reused by the three
// layers), the epilogue is TMEM -> registers (tcgen05.ld) -> cvt.rn.relu.bf16x2 ->
// st.shared straight into the next layer's A tile.  One elected thread issues the
// MMAs and commits them to an mbarrier.  Several CTAs per SM interleave their
// MMA and epilogue phases on the shared tensor core.  RGB tiles stream in through
// 1-D bulk copies (TMA); each thread stores its pixel's code row.
#include <cuda_bf16.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "hc_common.cuh"
#include "hc_internal.h"
#include "hc_tma.cuh"

namespace hcb {

constexpr int kMlpM = 128;    // pixels per tile (UMMA_M)
constexpr int kHid = 64;      // hidden width
constexpr int kK1 = 16;       // layer-1 K (3 inputs + bias column, padded)
constexpr int kN3 = 16;       // layer-3 N (k padded)
constexpr int kMaxK = 9;
constexpr int kThreads = 128;

// Shared-memory image offsets (bytes).
constexpr int kW1Bytes = kHid * kK1 * 2;   // 2 KB
constexpr int kW2Bytes = kHid * kHid * 2;  // 8 KB
constexpr int kW3Bytes = kN3 * kHid * 2;   // 2 KB
constexpr int kWBytes = kW1Bytes + kW2Bytes + kW3Bytes;
constexpr int kOffW1 = 0;
constexpr int kOffW2 = kOffW1 + kW1Bytes;
constexpr int kOffW3 = kOffW2 + kW2Bytes;
// A1 (128 x 16) aliases the first 4 KB of the A2/A3 buffer: A1 is dead once layer 1
// has completed, and the next tile's A1 is written after layer 3 has completed.
constexpr int kOffA2 = kOffW3 + kW3Bytes;            // 128 x 64 bf16 = 16 KB (A1, A2, A3)
constexpr int kOffA1 = kOffA2;
constexpr int kOffIn = kOffA2 + kMlpM * kHid * 2;    // 2 x 128 x 3 f32
constexpr int kInTile = kMlpM * 3 * 4;               // 1536 B
constexpr int kOffBar = kOffIn + 2 * kInTile;
constexpr int kSmemBytes = kOffBar + 64;              // ~31 KB: 7 CTAs / SM

struct MlpParams {
  float b2[kHid];
  float b3[kN3];
  const uint8_t* wimg;  // kWBytes, canonical layouts
  const float* rgb;     // P x 3
  float* out;           // P x k
  int64_t first_tile;   // tile index range [first_tile, first_tile + ntiles)
  int64_t ntiles;
  int64_t P;
  int k;
  int use_tma;          // 1: tiles are full and 16-byte aligned
};

__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFFu);
  d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFFu) << 16;
  d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFFu) << 32;
  d |= 1ull << 46;  // descriptor version (sm_100)
  return d;         // base offset 0, legacy LBO mode, SWIZZLE_NONE
}

// kind::f16 instruction descriptor: F32 accumulate, BF16 A/B, K-major A and B.
__host__ __device__ constexpr uint32_t idesc_bf16(int M, int N) {
  return (1u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(N >> 3) << 17) |
         (static_cast<uint32_t>(M >> 4) << 24);
}

__device__ __forceinline__ void mma_bf16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

#define HC_TMEM_LD16(taddr, r)                                                                          \
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];" \
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),   \
                 "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),          \
                 "=r"(r[15])                                                                            \
               : "r"(taddr))

__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ uint32_t pack_relu_bf16(float lo, float hi) {
  uint32_t d;
  asm("cvt.rn.relu.bf16x2.f32 %0, %1, %2;" : "=r"(d) : "f"(hi), "f"(lo));
  return d;
}
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  uint32_t d;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(d) : "f"(hi), "f"(lo));
  return d;
}

// softplus(x) with the reference's identity branch (codec.cpp:8-12, beta = 1):
// max(x, 0) + log1p(exp(-|x|)), log1p by series below 1e-3.
__device__ __forceinline__ float softplus1(float x) {
  if (x > 30.f) return x;
  const float e = __expf(-fabsf(x));
  const float l = e < 1e-3f ? e * (1.f - 0.5f * e) : __logf(1.f + e);
  return fmaxf(x, 0.f) + l;
}

// Epilogue for a 64-column layer: TMEM lane (row) -> bf16 relu(acc [+ bias]) row of
// the next A tile.  Thread r owns row r; chunk c of 8 bf16 goes to c*2048 + r*16.
template <bool kBias>
__device__ __forceinline__ void epilogue_hidden(uint32_t tmem_row, const float* bias, unsigned char* A, int r) {
  uint32_t va[4][16];
  HC_TMEM_LD16(tmem_row + 0, va[0]);
  HC_TMEM_LD16(tmem_row + 16, va[1]);
  HC_TMEM_LD16(tmem_row + 32, va[2]);
  HC_TMEM_LD16(tmem_row + 48, va[3]);
  tmem_wait_ld();
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const uint32_t* v = va[q];
    uint32_t pk[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      float lo = __uint_as_float(v[2 * j]), hi = __uint_as_float(v[2 * j + 1]);
      if (kBias) {
        lo += bias[q * 16 + 2 * j];
        hi += bias[q * 16 + 2 * j + 1];
      }
      pk[j] = pack_relu_bf16(lo, hi);
    }
    // columns q*16 .. q*16+15 = chunks 2q, 2q+1
    *reinterpret_cast<uint4*>(A + (2 * q) * (kMlpM * 16) + r * 16) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
    *reinterpret_cast<uint4*>(A + (2 * q + 1) * (kMlpM * 16) + r * 16) = make_uint4(pk[4], pk[5], pk[6], pk[7]);
  }
}

__global__ void __launch_bounds__(kThreads) mlp_kernel(const __grid_constant__ MlpParams p) {
  extern __shared__ __align__(1024) unsigned char sm[];
  uint64_t* bar_in = reinterpret_cast<uint64_t*>(sm + kOffBar);  // [2]
  uint64_t* bar_mma = bar_in + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar_in + 3);
  unsigned char* A1 = sm + kOffA1;
  unsigned char* A2 = sm + kOffA2;
  float* in_tiles = reinterpret_cast<float*>(sm + kOffIn);
  const int tid = threadIdx.x;
  const int warp = tid >> 5;

  // Weights: canonical images prepared on the host.
  for (int i = tid; i < kWBytes / 16; i += kThreads)
    reinterpret_cast<uint4*>(sm)[i] = reinterpret_cast<const uint4*>(p.wimg)[i];
  if (tid == 0) {
    mbar_init(&bar_in[0], 1);
    mbar_init(&bar_in[1], 1);
    mbar_init(bar_mma, 1);
    fence_mbar_init();
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 64;" ::"r"(smem_u32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t tmem_row = tmem + (static_cast<uint32_t>(warp * 32) << 16);

  const uint32_t sW1 = smem_u32(sm + kOffW1), sW2 = smem_u32(sm + kOffW2), sW3 = smem_u32(sm + kOffW3);
  const uint32_t sA1 = smem_u32(A1), sA2 = smem_u32(A2);
  constexpr uint32_t kChunkA = kMlpM * 16;  // K-chunk stride of a 128-row A tile
  const uint32_t id1 = idesc_bf16(kMlpM, kHid), id3 = idesc_bf16(kMlpM, kN3);

  auto load_tile = [&](int64_t t, int s) {
    mbar_arrive_expect_tx(&bar_in[s], kInTile);
    bulk_g2s(in_tiles + s * kMlpM * 3, p.rgb + (p.first_tile + t) * kMlpM * 3, kInTile, &bar_in[s]);
  };
  if (p.use_tma && tid == 0) {
    if (blockIdx.x < p.ntiles) load_tile(blockIdx.x, 0);
    if (blockIdx.x + gridDim.x < p.ntiles) load_tile(blockIdx.x + gridDim.x, 1);
  }

  uint32_t mma_phase = 0;
  int iter = 0;
  for (int64_t t = blockIdx.x; t < p.ntiles; t += gridDim.x, ++iter) {
    const int s = iter & 1;
    const int64_t tile = p.first_tile + t;
    const int64_t row0 = tile * kMlpM;
    const int64_t left = p.P - row0;
    const int rows = left < kMlpM ? static_cast<int>(left) : kMlpM;
    // ---- input: rgb -> (r, g, b, 1) bf16 into A1 chunk 0
    float x0 = 0.f, x1 = 0.f, x2 = 0.f;
    if (p.use_tma) {
      mbar_wait(&bar_in[s], (iter >> 1) & 1);
      const float* in = in_tiles + s * kMlpM * 3 + tid * 3;
      x0 = in[0];
      x1 = in[1];
      x2 = in[2];
    } else if (tid < rows) {
      const float* in = p.rgb + (row0 + tid) * 3;
      x0 = in[0];
      x1 = in[1];
      x2 = in[2];
    }
    *reinterpret_cast<uint4*>(A1 + tid * 16) = make_uint4(pack_bf16(x0, x1), pack_bf16(x2, 1.0f), 0u, 0u);
    *reinterpret_cast<uint4*>(A1 + kMlpM * 16 + tid * 16) = make_uint4(0u, 0u, 0u, 0u);
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();  // A1 complete; input slot s consumed
    if (tid == 0) {
      if (p.use_tma && t + 2 * gridDim.x < p.ntiles) load_tile(t + 2 * gridDim.x, s);
      tc_fence_after();
      mma_bf16(tmem, umma_desc(sA1, kChunkA, 128), umma_desc(sW1, kHid * 16, 128), id1, 0);
      mma_commit(bar_mma);
    }
    // ---- layer 1 epilogue: relu -> A2 (bias folded into W1)
    mbar_wait(bar_mma, mma_phase);
    mma_phase ^= 1;
    tc_fence_after();
    epilogue_hidden<false>(tmem_row, nullptr, A2, tid);
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    if (tid == 0) {
      tc_fence_after();
#pragma unroll
      for (int kk = 0; kk < kHid / 16; ++kk)
        mma_bf16(tmem, umma_desc(sA2 + kk * 2 * kChunkA, kChunkA, 128),
                 umma_desc(sW2 + kk * 2 * (kHid * 16), kHid * 16, 128), id1, kk > 0);
      mma_commit(bar_mma);
    }
    // ---- layer 2 epilogue: relu(acc + b2) -> A3 (reuses the A2 buffer: L2 has completed)
    mbar_wait(bar_mma, mma_phase);
    mma_phase ^= 1;
    tc_fence_after();
    epilogue_hidden<true>(tmem_row, p.b2, A2, tid);
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    if (tid == 0) {
      tc_fence_after();
#pragma unroll
      for (int kk = 0; kk < kHid / 16; ++kk)
        mma_bf16(tmem, umma_desc(sA2 + kk * 2 * kChunkA, kChunkA, 128),
                 umma_desc(sW3 + kk * 2 * (kN3 * 16), kN3 * 16, 128), id3, kk > 0);
      mma_commit(bar_mma);
    }
    // ---- layer 3 epilogue: softplus(acc + b3) -> codes
    mbar_wait(bar_mma, mma_phase);
    mma_phase ^= 1;
    tc_fence_after();
    uint32_t v[16];
    HC_TMEM_LD16(tmem_row, v);
    tmem_wait_ld();
    tc_fence_before();
    const int k = p.k;
    if (tid < rows) {
      float* o = p.out + (row0 + tid) * k;
#pragma unroll
      for (int j = 0; j < kMaxK; ++j)
        if (j < k) o[j] = softplus1(__uint_as_float(v[j]) + p.b3[j]);
    }
  }
  if (tid == 0) bulk_wait_all<0>();
  tc_fence_before();
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 64;" ::"r"(tmem));
}

}  // namespace hcb

using namespace hcb;

struct hc_mlp_s {
  hc_ctx ctx = nullptr;
  int hidden = 0, k = 0;
  uint8_t* d_wimg = nullptr;
  MlpParams base{};
  int occ = 1;
};

namespace {

uint16_t to_bf16(float f) {
  uint32_t u;
  std::memcpy(&u, &f, 4);
  u += 0x7fffu + ((u >> 16) & 1u);  // round to nearest even (finite inputs)
  return static_cast<uint16_t>(u >> 16);
}

// Canonical no-swizzle K-major image of an N x K bf16 matrix: element (n, k) at
// (k / 8) * (N * 16) + n * 16 + (k % 8) * 2 bytes.
void put_kmajor(std::vector<uint8_t>& img, int off, int N, int K, int n, int k, float v) {
  const uint16_t b = to_bf16(v);
  std::memcpy(&img[off + (k / 8) * (N * 16) + n * 16 + (k % 8) * 2], &b, 2);
}

}  // namespace

extern "C" {

int hc_mlp_create(hc_ctx ctx, int hidden, int k, const float* w1, const float* b1, const float* w2, const float* b2,
                  const float* w3, const float* b3, hc_mlp* out) {
  if (!ctx || !out || !w1 || !b1 || !w2 || !b2 || !w3 || !b3) return set_error(HC_EINVAL, "mlp: null argument");
  if (hidden != kHid) return set_error(HC_EUNSUPPORTED, "mlp: compiled for hidden = 64");
  if (k < 1 || k > kMaxK) return set_error(HC_EUNSUPPORTED, "mlp: k must be in [1, 9]");
  std::vector<uint8_t> img(kWBytes, 0);
  for (int n = 0; n < kHid; ++n) {
    for (int j = 0; j < 3; ++j) put_kmajor(img, kOffW1, kHid, kK1, n, j, w1[n * 3 + j]);
    put_kmajor(img, kOffW1, kHid, kK1, n, 3, b1[n]);  // bias via the constant-1 input column
    for (int j = 0; j < kHid; ++j) put_kmajor(img, kOffW2, kHid, kHid, n, j, w2[n * kHid + j]);
  }
  for (int n = 0; n < k; ++n)
    for (int j = 0; j < kHid; ++j) put_kmajor(img, kOffW3, kN3, kHid, n, j, w3[n * kHid + j]);
  hc_mlp m = new hc_mlp_s();
  m->ctx = ctx;
  m->hidden = hidden;
  m->k = k;
  cudaError_t e = cudaMalloc(&m->d_wimg, kWBytes);
  if (e == cudaSuccess) e = cudaMemcpy(m->d_wimg, img.data(), kWBytes, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(mlp_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(mlp_kernel, cudaFuncAttributePreferredSharedMemoryCarveout,
                             cudaSharedmemCarveoutMaxShared);
  // The occupancy API does not model TMEM (it reports 1 CTA / SM for tcgen05 kernels);
  // the real limits are shared memory and the 512 TMEM columns (64 per CTA).
  int smem_sm = 0, dev = 0;
  if (e == cudaSuccess) e = cudaGetDevice(&dev);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
  m->occ = smem_sm / (kSmemBytes + 1024);
  if (e != cudaSuccess) {
    if (m->d_wimg) cudaFree(m->d_wimg);
    delete m;
    return cuda_error(e, "hc_mlp_create");
  }
  if (const char* o = std::getenv("HC_MLP_OCC")) m->occ = std::atoi(o);
  m->occ = std::max(1, std::min(m->occ, 8));  // 8 x 64 TMEM columns = the full 512
  std::memset(&m->base, 0, sizeof(m->base));
  for (int i = 0; i < kHid; ++i) m->base.b2[i] = b2[i];
  for (int i = 0; i < k; ++i) m->base.b3[i] = b3[i];
  m->base.wimg = m->d_wimg;
  m->base.k = k;
  *out = m;
  return HC_OK;
}

int hc_mlp_destroy(hc_mlp m) {
  if (!m) return HC_OK;
  if (m->d_wimg) cudaFree(m->d_wimg);
  delete m;
  return HC_OK;
}

int hc_mlp_forward(hc_mlp m, const float* rgb, int64_t P, float* codes) {
  if (!m) return set_error(HC_EINVAL, "mlp: null handle");
  if (P < 0) return set_error(HC_EINVAL, "negative row count");
  if (P == 0) return HC_OK;
  if (!rgb || !codes) return set_error(HC_EINVAL, "mlp: null buffer");
  hc_ctx ctx = m->ctx;
  MlpParams p = m->base;
  p.rgb = rgb;
  p.out = codes;
  p.P = P;
  const bool aligned = (reinterpret_cast<uintptr_t>(rgb) & 15u) == 0;  // rgb tiles arrive by bulk copy
  // codes tile = 128 * k * 4 bytes: 16-byte multiple for any k
  const int64_t full = aligned ? P / kMlpM : 0;
  if (full > 0) {
    p.first_tile = 0;
    p.ntiles = full;
    p.use_tma = 1;
    const int grid = static_cast<int>(std::min<int64_t>(full, static_cast<int64_t>(m->occ) * ctx->sm_count));
    if (std::getenv("HC_DEBUG")) std::fprintf(stderr, "[hc] mlp_kernel grid=%d occ=%d smem=%d\n", grid, m->occ, kSmemBytes);
    mlp_kernel<<<grid, kThreads, kSmemBytes, ctx->stream>>>(p);
    HC_CHECK_LAUNCH(ctx, "mlp_kernel");
  }
  if (full * kMlpM < P) {
    p.first_tile = full;
    p.ntiles = (P - full * kMlpM + kMlpM - 1) / kMlpM;
    p.use_tma = 0;
    const int grid = static_cast<int>(std::min<int64_t>(p.ntiles, static_cast<int64_t>(m->occ) * ctx->sm_count));
    mlp_kernel<<<grid, kThreads, kSmemBytes, ctx->stream>>>(p);
    HC_CHECK_LAUNCH(ctx, "mlp_kernel(tail)");
  }
  return HC_OK;
}

}  // extern "C"
