// hadacodec-b200: RGB -> code upsampler MLP (config 5a) on 5th-gen tensor cores.
//
// Reference: forward (upsampler.cpp:42-72) and upsample's non-negative output
// (upsampler.cpp:179-190); BASELINE config 5 fixes the net to 3 -> 64 -> 64 -> 6
// with ReLU, ReLU and a softplus(beta = 1) head (codec.cpp:8-12), bf16 operands,
// fp32 accumulation.
//
// One 128-pixel tile = one M = 128 tcgen05 row block:
//   L1  D[128 x 64] = A1[128 x 16] . W1'^T   (SS: A1 = (r, g, b, 1, 0...) bf16 in smem,
//                                              W1' = [W1 | b1 | 0]: bias rides the MMA)
//   L2  D[128 x 64] = A2[128 x 80] . W2'^T   (TS: A2 = [bf16(relu(L1)) | 1 | 0] in TMEM,
//                                              W2' = [W2 | b2 | 0])
//   L3  D[128 x 16] = A3[128 x 64] . W3^T    (TS: A3 = bf16(relu(L2)) in TMEM)
//   out = softplus(L3[:, :k] + b3)
// Hidden activations never touch shared memory: the epilogue reads the fp32
// accumulator (tcgen05.ld), applies ReLU, packs bf16x2 (cvt.rn.relu.bf16x2) and
// writes the next layer's A operand back into TMEM (tcgen05.st), which the next
// MMA reads directly ("A from TMEM").  With A in shared memory (SS) the 128 x 16 A
// tile is re-read from smem by every MMA and smem bandwidth was the limit.
//
// One CTA per SM, 3 tile streams (default).  Each stream owns 144 TMEM columns of the CTA's
// 512: [0,32) the packed bf16 A2 operand, [32,64) the packed bf16 A3 operand, [64,128) the fp32
// layer-1/2 accumulator, [128,144) the layer-3 accumulator; the constant K chunk of A2 (the b2
// column) is one 8-column region at 432 shared by all streams.  With A3 and D3 in their own
// regions, layer 1 of the next tile is issued right after epilogue 2 (ahead of this tile's
// layer 3) and no epilogue waits for its own layer 3.  The chain per tile is two commit round
// trips (~470 cycles each, whatever the number of MMAs) + two epilogues (~290 each); throughput
// is tiles in flight over that latency, and TMEM caps the tiles in flight (measured variants:
// HC_MLP_STREAMS=4 with A3 over A2, 112 columns per stream; HC_MLP_PP ping-pong layout, 128
// columns; HC_MLP_A3_SMEM -- profiles/r02/mlp_ceiling_probe.txt, mma_chains.txt).
// A stream also has a 4 KB A1 tile and a 2-deep ring of rgb tiles fetched by 1-D
// bulk copies (TMA), 4 epilogue warps (one per TMEM lane quarter) and one MMA-issuer
// warp: tools/mma_probe3.cu measured that one thread can issue a tcgen05.mma only
// every ~45 cycles while several issuing warps overlap up to the tensor pipe's rate,
// so issuing from the epilogue warps put 10 x 45 cycles per tile on their critical
// path.  The warps hand off through mbarriers only:
//   issuer:   wait a2 -> L2 -> commit l2 | wait l1, next A1 | wait a3 -> L1 (next) -> commit l1
//             -> L3 -> commit l3
//   epilogue: wait l3 (previous tile) -> keep D3 | wait l1 -> relu(D) -> A2, arrive a2
//             | softplus + stores of the previous tile's codes | wait l2 -> relu(D) -> A3, arrive a3
// Weights (12 KB, canonical no-swizzle K-major UMMA images, element (n, k) at
// (k/8)*(N*16) + n*16 + (k%8)*2) are loaded once per CTA.
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
#ifndef HC_MLP_PP
#define HC_MLP_PP 0
#endif
// Ping-pong TMEM layout (measured option, off: 63.8 Gpix/s with 4 streams against 63.1-63.3 for the
// default 3 x 144 layout, 57.9 with 3 streams): each stream owns two 64-column regions X and Y.  Layer 1
// accumulates into X and its epilogue writes A2 *in place* over X's first 32 columns (+ the 8-column
// constant K chunk at X + 32); layer 2 reads A2 from X and accumulates into Y; its epilogue writes A3
// in place over Y's first 32 columns and layer 3 accumulates into Y + 32.  X is free as soon as layer
// 2 completes, so layer 1 of the next tile is issued then -- it runs under this tile's layer-2
// epilogue instead of after it -- and a stream needs 128 columns instead of 144: 4 streams fit.
// The stream's cycle is then layer-2 round trip + epilogue 2 + layer-3 round trip + accumulator read
// (~2,000 cycles under load: layer 2 of the next tile overwrites Y, so layer 3 is on the cycle), which
// 4 streams turn into ~500 cycles per tile -- the same as 3 streams of ~1,600.
constexpr bool kPP = HC_MLP_PP;
#ifndef HC_MLP_L3_SPLIT  // measured 37.2 Gpix/s: alternating two 16-column accumulators is far slower
#define HC_MLP_L3_SPLIT 0
#endif
// Layer 3 as two independent two-step K chains into two 16-column accumulators (Y + 32, Y + 48)
// summed by the codes epilogue: a dependent tcgen05.mma step costs ~100-135 cycles of latency
// whatever N (tools/mma_latency.cu), and with kPP layer 3's latency is on the stream's cycle.
constexpr bool kL3Split = HC_MLP_L3_SPLIT;
static_assert(!kL3Split || kPP, "split layer 3 needs the ping-pong layout's free Y columns");
#ifndef HC_MLP_STREAMS
#define HC_MLP_STREAMS (HC_MLP_PP ? 4 : 3)
#endif
#ifndef HC_MLP_L3_FIRST
#define HC_MLP_L3_FIRST 0
#endif
#ifndef HC_MLP_TMEM_WIDE  // epilogue TMEM access width: 0 = x16, 1 = x32 loads + one x32 store, 2 = x64 load
#define HC_MLP_TMEM_WIDE 1
#endif
#ifndef HC_MLP_B2_EPI
#define HC_MLP_B2_EPI 0
#endif
constexpr bool kB2Epi = HC_MLP_B2_EPI;     // b2 added in the layer-2 epilogue instead of a 5th MMA
constexpr int kStreams = HC_MLP_STREAMS;    // tile streams per CTA
#ifndef HC_MLP_A3_SMEM
#define HC_MLP_A3_SMEM 0
#endif
// A3 in shared memory (canonical K-major image written by the layer-2 epilogue, layer 3 is an
// SS MMA): frees 32 TMEM columns per stream, so 4 streams fit without A3 over A2.
constexpr bool kA3Smem = HC_MLP_A3_SMEM;
constexpr bool kSepA3 = kA3Smem || kStreams < 4;  // A3 not over A2 (own TMEM region or smem)
constexpr bool kL3First = HC_MLP_L3_FIRST;  // issue layer 3 of a tile before layer 1 of the next
#ifndef HC_MLP_EPI_WARPS
#define HC_MLP_EPI_WARPS 4
#endif
// Epilogue warps per stream: 4 (one per TMEM lane quarter, all 64 accumulator columns) or 8
// (two per lane quarter, 32 columns each: half the tcgen05.ld / cvt / tcgen05.st chain per warp).
constexpr int kEpiW = HC_MLP_EPI_WARPS;
static_assert(kEpiW == 4 || kEpiW == 8, "epilogue warps per stream");
static_assert(!(HC_MLP_A3_SMEM && kEpiW != 4), "A3 in smem: 4 epilogue warps");
static_assert(!(HC_MLP_PP && (kEpiW != 4 || HC_MLP_A3_SMEM || HC_MLP_B2_EPI)), "ping-pong layout: 4 epilogue warps, A3 in TMEM, b2 by MMA");
constexpr int kEpiCols = kHid * 4 / kEpiW;   // accumulator columns per epilogue warp
constexpr int kEpiThreads = 32 * kEpiW * kStreams; // warp w -> stream w / kEpiW, lane quarter w % 4
constexpr int kThreads = kEpiThreads + 32 * kStreams;  // + one MMA-issuer warp per stream
constexpr int kK2 = 80;                     // layer 2 K: 64 hidden + constant-1 column (b2 rides the MMA)
constexpr int kK3 = 64;                     // layer 3 K: b3 (6 values) is added in the epilogue instead of
                                            // paying a fifth >= 45-cycle N = 16 MMA
constexpr int kColA = 0;                    // packed bf16 A2 (and A3 of the same tile unless kSepA3): 32 columns
constexpr bool kA3Tmem = kSepA3 && !kA3Smem;
constexpr int kColA3 = kPP ? 64 : kA3Tmem ? 32 : 0;    // packed bf16 A3
constexpr int kColD = kPP ? 0 : kA3Tmem ? 64 : 32;     // fp32 accumulator of layer 1 (and 2 unless kPP): 64 columns
constexpr int kColD2 = kPP ? 64 : kColD;    // fp32 accumulator of layer 2
constexpr int kColD3 = kPP ? 96 : kColD + 64;  // fp32 accumulator of layer 3: 16 columns (separate, so layer 1
                                            // of the next tile can run while layer 3 still reads A3)
constexpr int kColsPerStream = kPP ? 128 : kColD3 + 16; // TMEM columns per stream (4 x 128, 4 x 112 or 3 x 144 of the 512)
// Constant K chunk of A2, (1, 0 x 15) bf16: one shared region after the streams, or (kPP) 8 columns
// after each stream's A2, rewritten by every layer-1 epilogue (layer 1 overwrites X).
constexpr int kColConst = kPP ? kColA + 32 : kStreams * kColsPerStream;
static_assert(kPP ? kStreams * kColsPerStream <= 512 : kColConst + 8 <= 512, "TMEM budget");

// Shared-memory image offsets (bytes).
constexpr int kW1Bytes = kHid * kK1 * 2;   // 2 KB
constexpr int kW2Bytes = kHid * kK2 * 2;   // 10 KB ([W2 | b2 | 0])
constexpr int kW3Bytes = kN3 * kK3 * 2;    // 2 KB
constexpr int kWBytes = kW1Bytes + kW2Bytes + kW3Bytes;
constexpr int kOffW1 = 0;
constexpr int kOffW2 = kOffW1 + kW1Bytes;
constexpr int kOffW3 = kOffW2 + kW2Bytes;
constexpr int kA1Bytes = kMlpM * kK1 * 2;            // 4 KB
constexpr int kInTile = kMlpM * 3 * 4;               // 1536 B
constexpr int kA3Bytes = kA3Smem ? kMlpM * kK3 * 2 : 0;  // 16 KB A3 image (kA3Smem)
constexpr int kStreamBytes = kA1Bytes + 2 * kInTile + kA3Bytes;
constexpr int kOffStreams = kWBytes;
constexpr int kOffBar = kOffStreams + kStreams * kStreamBytes;
constexpr int kBarsPerStream = 8;  // in[2], l1, l2, l3, a1, a2, a3
constexpr int kSmemBytes = kOffBar + kStreams * kBarsPerStream * 8 + 16;

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
  int use_tma;          // 1: tiles are full and the rgb base is 16-byte aligned
  long long* trace;     // debug (HC_MLP_TRACE): per-phase clock64 stamps of CTA 0
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

// D[tmem] (+)= A[smem] . B[smem]
__device__ __forceinline__ void mma_ss(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                       uint32_t accumulate) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

// D[tmem] (+)= A[tmem] . B[smem]
__device__ __forceinline__ void mma_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc, uint32_t idesc,
                                       uint32_t accumulate) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(tmem_d),
      "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}

// Warp-wide variants: every lane of the issuing warp executes them and elect.sync picks the
// one that issues.  Under `if (lane == 0)` with register operands the compiler wraps every
// UTCHMMA in a per-thread "waterfall" loop (ELECT / R2UR.BROADCAST / BRA.U.ANY): ~54 cycles per
// MMA from one thread (tools/mma_probe4.cu); warp-wide with elect.sync inside the asm: 17
// cycles (N = 16) and the full tensor rate at N = 64 (32 cycles) from a single issuer.
__device__ __forceinline__ void mma_ss_w(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n.reg .pred p, e;\nsetp.ne.b32 p, %4, 0;\nelect.sync _|e, 0xffffffff;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void mma_ts_w(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n.reg .pred p, e;\nsetp.ne.b32 p, %4, 0;\nelect.sync _|e, 0xffffffff;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(tmem_d),
      "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void mma_commit_w(uint64_t* bar) {
  asm volatile(
      "{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}\n" ::"r"(smem_u32(bar))
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

#define HC_TMEM_ST16(taddr, r)                                                                          \
  asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" \
               ::"r"(taddr), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), \
                 "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])   \
               : "memory")

#define HC_TMEM_LD8(taddr, r)                                                                           \
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"                   \
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]) \
               : "r"(taddr))
// The layer-3 accumulator has 16 columns (N = 16) but only k are codes: k <= 8 reads 8
// (TMEM reads, not writes, are the scarce direction).  k is uniform, the load warp-collective.
#define HC_TMEM_LD_D3(taddr, r, k)     \
  do {                                 \
    if ((k) <= 8) HC_TMEM_LD8(taddr, r); \
    else HC_TMEM_LD16(taddr, r);       \
  } while (0)

// kL3Split: the two partial accumulators (16 columns apart) are read and summed.
#define HC_TMEM_LD_D3S(taddr, r, k)                                                              \
  do {                                                                                           \
    if constexpr (kL3Split) {                                                                    \
      uint32_t r2_[kN3];                                                                         \
      if ((k) <= 8) {                                                                            \
        HC_TMEM_LD8(taddr, r);                                                                   \
        HC_TMEM_LD8((taddr) + kN3, r2_);                                                         \
      } else {                                                                                   \
        HC_TMEM_LD16(taddr, r);                                                                  \
        HC_TMEM_LD16((taddr) + kN3, r2_);                                                        \
      }                                                                                          \
      tmem_wait_ld();                                                                            \
      _Pragma("unroll") for (int j_ = 0; j_ < kN3; ++j_) if (j_ < 8 || (k) > 8)                  \
          r[j_] = __float_as_uint(__uint_as_float(r[j_]) + __uint_as_float(r2_[j_]));            \
    } else {                                                                                     \
      HC_TMEM_LD_D3(taddr, r, k);                                                                \
      tmem_wait_ld();                                                                            \
    }                                                                                            \
  } while (0)

#define HC_TMEM_LD64(taddr, r) \
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x64.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32,%33,%34,%35,%36,%37,%38,%39,%40,%41,%42,%43,%44,%45,%46,%47,%48,%49,%50,%51,%52,%53,%54,%55,%56,%57,%58,%59,%60,%61,%62,%63}, [%64];" \
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31]), "=r"(r[32]), "=r"(r[33]), "=r"(r[34]), "=r"(r[35]), "=r"(r[36]), "=r"(r[37]), "=r"(r[38]), "=r"(r[39]), "=r"(r[40]), "=r"(r[41]), "=r"(r[42]), "=r"(r[43]), "=r"(r[44]), "=r"(r[45]), "=r"(r[46]), "=r"(r[47]), "=r"(r[48]), "=r"(r[49]), "=r"(r[50]), "=r"(r[51]), "=r"(r[52]), "=r"(r[53]), "=r"(r[54]), "=r"(r[55]), "=r"(r[56]), "=r"(r[57]), "=r"(r[58]), "=r"(r[59]), "=r"(r[60]), "=r"(r[61]), "=r"(r[62]), "=r"(r[63]) \
               : "r"(taddr))
#define HC_TMEM_LD32(taddr, r) \
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];" \
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31]) \
               : "r"(taddr))
#define HC_TMEM_ST32(taddr, r) \
  asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" \
               ::"r"(taddr), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31]) \
               : "memory")

__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

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

// softplus(x) = max(x, 0) + ln2 * log2(1 + 2^(-|x| log2 e)) (codec.cpp:8-12, beta = 1) in
// six instructions (two MUFU): for x > 30 the log term is < 1e-13 and vanishes in fp32,
// which is the reference's identity branch; for very negative x the result is the tiny
// e = exp(x) with an absolute error ~1e-7 (ex2 / lg2.approx: 2^-22), far inside the bf16
// MLP tolerance, which is relative to the row's largest code.
__device__ __forceinline__ float softplus1(float x) {
  float e, l;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(-fabsf(x) * 1.4426950408889634f));
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(l) : "f"(1.f + e));
  return fmaf(l, 0.6931471805599453f, fmaxf(x, 0.f));
}

// Hidden-layer epilogue: fp32 accumulator row (64 TMEM columns of this thread's
// lane) -> bf16 relu(acc [+ bias]) packed in pairs (element 2j in the low half)
// -> 32 TMEM columns of the next layer's A operand.
// kCols accumulator columns starting at tmem_acc -> kCols / 2 packed A columns at tmem_a.
template <bool kBias, int kCols = 64, bool kConstChunk = false>
__device__ __forceinline__ void epilogue_hidden(uint32_t tmem_acc, uint32_t tmem_a, const float* bias) {
#ifdef HC_MLP_PROBE_NOEPI  // timing probe only: no accumulator read-out (wrong results)
  return;
#endif
  constexpr int kQ = kCols / 16;
  uint32_t va[kQ][16];
#if HC_MLP_TMEM_WIDE  // 32-column (or, = 2 with 64 columns, one 64-column) loads and one 32-column store
  static_assert(kQ % 2 == 0, "32-column chunks");
  if constexpr (HC_MLP_TMEM_WIDE == 2 && kQ == 4) {
    HC_TMEM_LD64(tmem_acc, (&va[0][0]));
  } else {
#pragma unroll
    for (int q = 0; q < kQ; q += 2) HC_TMEM_LD32(tmem_acc + q * 16, (&va[q][0]));
  }
#else
#pragma unroll
  for (int q = 0; q < kQ; ++q) HC_TMEM_LD16(tmem_acc + q * 16, va[q]);
#endif
  tmem_wait_ld();
  uint32_t pk[kQ / 2][16];
#pragma unroll
  for (int q = 0; q < kQ; ++q)
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      float lo = __uint_as_float(va[q][2 * j]), hi = __uint_as_float(va[q][2 * j + 1]);
      if (kBias) {
        lo += bias[q * 16 + 2 * j];
        hi += bias[q * 16 + 2 * j + 1];
      }
      pk[q >> 1][(q & 1) * 8 + j] = pack_relu_bf16(lo, hi);
    }
#if HC_MLP_TMEM_WIDE
  static_assert(kQ / 2 == 2, "one 32-column store");
  HC_TMEM_ST32(tmem_a, (&pk[0][0]));
#else
#pragma unroll
  for (int q = 0; q < kQ / 2; ++q) HC_TMEM_ST16(tmem_a + q * 16, pk[q]);
#endif
  if constexpr (kConstChunk) {  // K chunk (1, 0 x 15) bf16 after the 32 packed columns
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%2,%2,%2,%2,%2,%2};" ::"r"(tmem_a + kCols / 2),
                 "r"(0x3F80u), "r"(0u)
                 : "memory");
  }
  tmem_wait_st();
}

// Layer-2 epilogue with A3 in shared memory: relu(acc + bias) -> bf16 pairs -> the canonical
// no-swizzle K-major image (element (row, k) at (k / 8) * 2048 + row * 16 + (k % 8) * 2): eight
// 16-byte stores per row, a warp's 32 rows contiguous per store (conflict-free).
template <bool kBias>
__device__ __forceinline__ void epilogue_hidden_smem(uint32_t tmem_acc, unsigned char* a3, int row, const float* bias) {
  uint32_t va[4][16];
#pragma unroll
  for (int q = 0; q < 4; ++q) HC_TMEM_LD16(tmem_acc + q * 16, va[q]);
  tmem_wait_ld();
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    uint32_t w[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int e = c * 8 + 2 * j;  // element pair (e, e + 1)
      float lo = __uint_as_float(va[e >> 4][e & 15]), hi = __uint_as_float(va[e >> 4][(e & 15) + 1]);
      if (kBias) {
        lo += bias[e];
        hi += bias[e + 1];
      }
      w[j] = pack_relu_bf16(lo, hi);
    }
    *reinterpret_cast<uint4*>(a3 + c * (kMlpM * 16) + row * 16) = make_uint4(w[0], w[1], w[2], w[3]);
  }
  fence_proxy_async_smem();  // the tensor core (async proxy) reads the image
}

__global__ void __launch_bounds__(kThreads, 1) mlp_kernel(const __grid_constant__ MlpParams p) {
  extern __shared__ __align__(1024) unsigned char sm[];
  const int tid = threadIdx.x;
  const int warp = tid >> 5;
  const bool issuer = tid >= kEpiThreads;
  const int st = issuer ? (tid - kEpiThreads) >> 5 : warp / kEpiW;  // tile stream
  const int quarter = warp & 3;                                       // TMEM lane quarter (epilogue warps)
  const int half = kEpiW == 8 ? (warp >> 2) & 1 : 0;                  // column half (8 epilogue warps)
  const bool codes_warp = half == 0;  // reads D3 and stores the codes
  const int r = tid & 127;                                         // tile row = TMEM lane (epilogue)
  unsigned char* A1 = sm + kOffStreams + st * kStreamBytes;
  float* in_tiles = reinterpret_cast<float*>(A1 + kA1Bytes);
  unsigned char* A3s = A1 + kA1Bytes + 2 * kInTile;  // kA3Smem
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + kOffBar) + st * kBarsPerStream;
  uint64_t* bar_in = bars;         // [2] rgb tile landed (TMA transaction count)
  uint64_t* bar_l1 = bars + 2;     // layer-1 MMAs complete (tcgen05.commit)
  uint64_t* bar_l2 = bars + 3;     // layer-2 MMAs complete
  uint64_t* bar_l3 = bars + 4;     // layer-3 MMAs complete
  uint64_t* bar_a1 = bars + 5;     // A1 tile written to smem (4 epilogue warps)
  uint64_t* bar_a2 = bars + 6;     // A2 written to TMEM (4 epilogue warps)
  uint64_t* bar_a3 = bars + 7;     // A3 written to TMEM (4 epilogue warps)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(sm + kOffBar + kStreams * kBarsPerStream * 8);

  for (int i = tid; i < kWBytes / 16; i += kThreads)
    reinterpret_cast<uint4*>(sm)[i] = reinterpret_cast<const uint4*>(p.wimg)[i];
  if (issuer && (tid & 31) == 0) {
    for (int i = 0; i < 5; ++i) mbar_init(&bars[i], 1);
    for (int i = 5; i < 8; ++i) mbar_init(&bars[i], i == 5 ? 4 : kEpiW);
    fence_mbar_init();
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  fence_proxy_async_smem();  // weight images are read by the tensor core (async proxy)
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  if (!kPP && warp < 4) {
    // Constant K chunk of every stream's layer-2 A operand: element 64 = 1 (bias b2),
    // 65..79 = 0.  Written once per CTA (warp w: lane quarter w); the fifth layer-2 MMA
    // of all streams reads it.
    uint32_t one[8] = {0x3F80u, 0u, 0u, 0u, 0u, 0u, 0u, 0u};
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(
                     tmem + kColConst + (static_cast<uint32_t>(warp * 32) << 16)),
                 "r"(one[0]), "r"(one[1]), "r"(one[2]), "r"(one[3]), "r"(one[4]), "r"(one[5]), "r"(one[6]),
                 "r"(one[7])
                 : "memory");
    tmem_wait_st();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tcol = tmem + st * kColsPerStream;  // stream base, lane 0
  const uint32_t tA = tcol + kColA, tA3 = tcol + kColA3, tD = tcol + kColD, tD2 = tcol + kColD2, tD3 = tcol + kColD3;
  const uint32_t tC = (kPP ? tcol : tmem) + kColConst;
  const int64_t t0 = static_cast<int64_t>(blockIdx.x) * kStreams + st;
  const int64_t tstride = static_cast<int64_t>(gridDim.x) * kStreams;
  constexpr uint32_t kChunkA = kMlpM * 16;  // K-chunk stride of the 128-row A1 tile

  if (issuer) {
    // ------------------------------------------------------------ MMA-issuer warp
    // Lane 0 issues the MMAs and the rgb bulk copies; the whole warp builds each tile's
    // A1 (r, g, b, 1) rows in shared memory, so the epilogue warps never do.
    const int lane = tid & 31;
    const bool elect = lane == 0;
    const uint32_t sW1 = smem_u32(sm + kOffW1), sW2 = smem_u32(sm + kOffW2), sW3 = smem_u32(sm + kOffW3);
    const uint32_t sA1 = smem_u32(A1);
    const uint32_t id64 = idesc_bf16(kMlpM, kHid), id16 = idesc_bf16(kMlpM, kN3);
    auto load_tile = [&](int64_t t, int s) {
      mbar_arrive_expect_tx(&bar_in[s], kInTile);
      bulk_g2s(in_tiles + s * kMlpM * 3, p.rgb + (p.first_tile + t) * kMlpM * 3, kInTile, &bar_in[s]);
    };
    if (p.use_tma && elect) {
      if (t0 < p.ntiles) load_tile(t0, 0);
      if (t0 + tstride < p.ntiles) load_tile(t0 + tstride, 1);
    }
    // rgb of tile t -> (r, g, b, 1, 0 ...) bf16 rows of A1; frees rgb slot it & 1 for the
    // tile two strides on.
    auto prepare_a1 = [&](int64_t t, int it) {
      const int s = it & 1;
      const int64_t row0 = (p.first_tile + t) * kMlpM;
      const int64_t left = p.P - row0;
      if (p.use_tma) mbar_wait(&bar_in[s], (it >> 1) & 1);
#pragma unroll
      for (int q = 0; q < kMlpM / 32; ++q) {
        const int row = q * 32 + lane;
        float x0 = 0.f, x1 = 0.f, x2 = 0.f;
        if (p.use_tma) {
          const float* in = in_tiles + s * kMlpM * 3 + row * 3;
          x0 = in[0];
          x1 = in[1];
          x2 = in[2];
        } else if (row < left) {
          const float* in = p.rgb + (row0 + row) * 3;
          x0 = in[0];
          x1 = in[1];
          x2 = in[2];
        }
        *reinterpret_cast<uint4*>(A1 + row * 16) = make_uint4(pack_bf16(x0, x1), pack_bf16(x2, 1.0f), 0u, 0u);
        *reinterpret_cast<uint4*>(A1 + kChunkA + row * 16) = make_uint4(0u, 0u, 0u, 0u);
      }
      fence_proxy_async_smem();
      __syncwarp();
      if (elect && p.use_tma && t + 2 * tstride < p.ntiles) load_tile(t + 2 * tstride, s);
    };
    auto issue_l1 = [&]() {
      tc_fence_after();
      mma_ss_w(tD, umma_desc(sA1, kChunkA, 128), umma_desc(sW1, kHid * 16, 128), id64, 0);
      mma_commit_w(bar_l1);
      __syncwarp();
    };
    if (t0 < p.ntiles) {
      prepare_a1(t0, 0);
      issue_l1();
    }
    int iter = 0;
    for (int64_t t = t0; t < p.ntiles; t += tstride, ++iter) {
      const uint32_t ph = iter & 1;
      const int64_t tn = t + tstride;
      mbar_wait(bar_a2, ph);  // A2(t) in TMEM, D read out
      tc_fence_after();
#pragma unroll
      for (int kk = 0; kk < (kB2Epi ? kHid : kK2) / 16; ++kk)
        mma_ts_w(tD2, kk < kHid / 16 ? tA + kk * 8 : tC, umma_desc(sW2 + kk * 2 * (kHid * 16), kHid * 16, 128),
                 id64, kk > 0);
      mma_commit_w(bar_l2);
      __syncwarp();
      if (tn < p.ntiles) {
        mbar_wait(bar_l1, ph);  // layer 1 of tile t has read A1
        prepare_a1(tn, iter + 1);
      }
      if constexpr (kPP) {
        // Layer 2 has read A2: X is free, layer 1 of the next tile runs under this tile's
        // layer-2 epilogue.
        mbar_wait(bar_l2, ph);
        if (tn < p.ntiles) issue_l1();
      }
      mbar_wait(bar_a3, ph);  // A3(t) in TMEM, D read out, D3(t - 1) read out
      // D and D3 are separate TMEM regions, so layer 1 of the next tile (D is free, A1 is
      // ready) and layer 3 of this one run back to back.  Dependent MMAs complete in order,
      // ~100 cycles apart after a ~470-cycle first one (tools/mma_latency.cu): with A3 in the
      // A region the epilogue needs layer 3 done before it writes the next A2, so layer 3
      // goes first there.
      if (!kPP && !kL3First && tn < p.ntiles) issue_l1();
      tc_fence_after();
#pragma unroll
      for (int kk = 0; kk < kK3 / 16; ++kk) {
        if constexpr (kA3Smem)
          mma_ss_w(tD3, umma_desc(smem_u32(A3s) + kk * 2 * (kMlpM * 16), kMlpM * 16, 128),
                   umma_desc(sW3 + kk * 2 * (kN3 * 16), kN3 * 16, 128), id16, kk > 0);
        else if constexpr (kL3Split) {
          const int kc = (kk & 1) * 2 + (kk >> 1);  // K chunks 0, 2, 1, 3: chains (0, 1) and (2, 3) interleaved
          mma_ts_w(tD3 + (kc >> 1) * kN3, tA3 + kc * 8, umma_desc(sW3 + kc * 2 * (kN3 * 16), kN3 * 16, 128), id16,
                   kc & 1);
        } else
          mma_ts_w(tD3, tA3 + kk * 8, umma_desc(sW3 + kk * 2 * (kN3 * 16), kN3 * 16, 128), id16, kk > 0);
      }
      mma_commit_w(bar_l3);
      __syncwarp();
      if (!kPP && kL3First && tn < p.ntiles) issue_l1();
    }
  } else {
    // ------------------------------------------------------------ epilogue warps
    const uint32_t lane_off = static_cast<uint32_t>(quarter * 32) << 16;
    // Codes of the previous tile: the layer-3 accumulator is read right after layer 3
    // completes, softplus + the global stores run later, under the next tile's MMAs.
    uint32_t prev_v[kN3];
    int64_t prev_row0 = -1;
    int prev_rows = 0;
    const int k = p.k;
    auto store_codes = [&]() {
      if (!codes_warp || prev_row0 < 0 || r >= prev_rows) return;
      float* o = p.out + (prev_row0 + r) * k;
      if (k == 6) {
        float y[6];
#pragma unroll
        for (int j = 0; j < 6; ++j) y[j] = softplus1(__uint_as_float(prev_v[j]) + p.b3[j]);
        reinterpret_cast<float2*>(o)[0] = make_float2(y[0], y[1]);
        reinterpret_cast<float2*>(o)[1] = make_float2(y[2], y[3]);
        reinterpret_cast<float2*>(o)[2] = make_float2(y[4], y[5]);
      } else {
#pragma unroll
        for (int j = 0; j < kMaxK; ++j)
          if (j < k) o[j] = softplus1(__uint_as_float(prev_v[j]) + p.b3[j]);
      }
    };
    auto handoff = [&](uint64_t* bar) {  // TMEM stores of this warp done -> issuer
      tc_fence_before();
      __syncwarp();
      if ((tid & 31) == 0) mbar_arrive(bar);
    };

    int iter = 0;
    for (int64_t t = t0; t < p.ntiles; t += tstride, ++iter) {
      const uint32_t ph = iter & 1;
      const int64_t row0 = (p.first_tile + t) * kMlpM;
      const int64_t left = p.P - row0;
      const int rows = left < kMlpM ? static_cast<int>(left) : kMlpM;
      long long* tr = (p.trace && blockIdx.x == 0 && r == 0 && half == 0 && iter < 32) ? p.trace + (st * 32 + iter) * 8 : nullptr;
      if (tr) tr[0] = clock64();
      if (!kPP && !kSepA3 && iter > 0) {  // layer 3 of the previous tile has read A3 (the A region) and written D3
        mbar_wait(bar_l3, ph ^ 1);
        tc_fence_after();
        if (codes_warp) {
          HC_TMEM_LD_D3(tD3 + lane_off, prev_v, p.k);
          tmem_wait_ld();
        }
      }
      if (tr) tr[1] = clock64();
      mbar_wait(bar_l1, ph);
      if (tr) tr[2] = clock64();
      tc_fence_after();
      epilogue_hidden<false, kEpiCols, kPP>(tD + lane_off + half * kEpiCols, tA + lane_off + half * (kEpiCols / 2),
                                            nullptr);  // A2 over A3 of t-1 (kPP: in place over D)
      if (kPP && iter > 0) {
        // Layer 2 of this tile overwrites Y: layer 3 of the previous tile must have read A3 and
        // its accumulator (Y + 32) must be in registers before a2 is signalled.  Layer 3 was
        // issued a layer-1 wait + epilogue ago, so this wait is short.
        mbar_wait(bar_l3, ph ^ 1);
        tc_fence_after();
        HC_TMEM_LD_D3S(tD3 + lane_off, prev_v, p.k);
      }
      handoff(bar_a2);
      if (tr) tr[3] = clock64();
      if (!kPP && kSepA3 && iter > 0 && codes_warp) {  // layer 3 of the previous tile, read under this tile's layer 2
        mbar_wait(bar_l3, ph ^ 1);
        tc_fence_after();
        HC_TMEM_LD_D3(tD3 + lane_off, prev_v, p.k);
        tmem_wait_ld();
      }
      store_codes();  // the previous tile's codes, under this tile's layer 2
      if (tr) tr[4] = clock64();
      mbar_wait(bar_l2, ph);
      if (tr) tr[5] = clock64();
      tc_fence_after();
      if constexpr (kA3Smem)
        epilogue_hidden_smem<kB2Epi>(tD2 + lane_off, A3s, r, p.b2);
      else
        epilogue_hidden<kB2Epi, kEpiCols>(tD2 + lane_off + half * kEpiCols, tA3 + lane_off + half * (kEpiCols / 2),
                                          p.b2 + half * kEpiCols);  // A3 (over A2 unless kSepA3; kPP: in place over D2)
      handoff(bar_a3);
      prev_row0 = row0;
      prev_rows = rows;
      if (tr) tr[6] = clock64();
      if (tr) tr[7] = clock64();
    }
    if (iter > 0 && codes_warp) {  // the last tile's codes
      mbar_wait(bar_l3, (iter - 1) & 1);
      tc_fence_after();
      HC_TMEM_LD_D3S(tD3 + lane_off, prev_v, p.k);
      store_codes();
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

// ===================================================================== mlp2_kernel
// Layer 1 on the CUDA cores, layers 2 and 3 on the tensor cores.
//
// mlp_kernel's per-tile chain is L1 round trip + epilogue 1 + L2 round trip + epilogue 2
// (~1,900 cycles; tools/mma_latency.cu: a tcgen05.mma + commit round trip is ~474 cycles
// whatever N), and TMEM holds 3 tile streams, so the SM finishes a tile every ~630 cycles
// against a 224-cycle tensor-pipe floor.  Layer 1 is only 3 -> 64 (+ bias): per pixel
// 192 FMAs, i.e. 96 packed FFMA2 (fma.rn.f32x2) on the epilogue thread that owns the
// pixel's TMEM lane, with the same arithmetic as the tensor core (bf16 inputs and
// weights, fp32 accumulation, one cvt.rn.relu.bf16x2 per hidden pair).  The thread
// writes A2 straight into TMEM, so the layer-1 MMA, its commit round trip, the A1 smem
// tile and epilogue 1's accumulator read all disappear.  A2 of tile t+1 is computed in
// registers while layer 2 of tile t runs and stored as soon as that layer completes, so
// a stream's period is one layer-2 round trip + epilogue 2 + the A2 store.
//
// Per stream (TMEM lane = pixel row of the tile): A2 [32 cols bf16x2] | A3 [32] | D [64
// fp32] | D3 [16]; the constant-1 K chunk of A2 (b2 rides the fifth layer-2 MMA) is one
// 8-column region shared by all streams.  Warps: 4 epilogue warps per stream (one per TMEM
// lane quarter) + 1 issuer warp per stream (rgb bulk copies, MMAs).  Hand-offs:
//   epilogue: [regs] A2(t+1) | wait l2(t) -> D3(t-1) -> relu(D) -> A3(t), arrive a3
//             -> A2(t+1) -> TMEM, arrive a2 | softplus + stores of tile t-1's codes
//   issuer:   wait a2(t) -> rgb load (t + R) -> L2(t) -> commit l2 | wait a3(t) -> L3(t) -> commit l3
// One commit covers every earlier MMA of the thread, so l2(t) complete implies L3(t-1)
// complete: D3(t-1) and the A3 region are free without waiting on l3.
#ifndef HC_MLP2_STREAMS
#define HC_MLP2_STREAMS 3
#endif
#ifndef HC_MLP2_RING
#define HC_MLP2_RING 4
#endif
#ifndef HC_MLP2_L1_BF16  // 1: layer 1 in packed bf16 FMA (fma.rn.bf16x2) instead of fp32 FFMA2
#define HC_MLP2_L1_BF16 0
#endif
constexpr int kS2 = HC_MLP2_STREAMS;
constexpr int kRing2 = HC_MLP2_RING;
constexpr int kEpi2 = 128 * kS2;
constexpr int kThreads2 = kEpi2 + 32 * kS2;
constexpr int kCols2 = 144;  // A2 32 | A3 32 | D 64 | D3 16
constexpr int kColConst2 = kS2 * kCols2;
static_assert(kColConst2 + 8 <= 512, "TMEM budget");
constexpr int kOffW2b = 0;                    // W2' image (kW2Bytes)
constexpr int kOffW3b = kW2Bytes;             // W3 image (kW3Bytes)
constexpr int kOffRing2 = kW2Bytes + kW3Bytes;
constexpr int kStream2Bytes = kRing2 * kInTile;
constexpr int kOffBar2 = kOffRing2 + kS2 * kStream2Bytes;
constexpr int kBars2 = kRing2 + 4;  // in[R], l2, l3, a2, a3
constexpr int kSmem2 = kOffBar2 + kS2 * kBars2 * 8 + 16;

struct Mlp2Params {
  // layer 1, bf16-valued, as (hidden 2i, 2i + 1) pairs: w1p[c][i] = (W1[2i][c], W1[2i+1][c])
  unsigned long long w1p[3][kHid / 2];
  unsigned long long b1p[kHid / 2];
  float b3[kN3];
  const uint8_t* wimg;  // W2' | W3 canonical images (kW2Bytes + kW3Bytes)
  const float* rgb;
  float* out;
  int64_t first_tile, ntiles, P;
  int k;
  int use_tma;
  int vec2;  // codes rows 8-byte aligned (float2 stores for even k)
};

__device__ __forceinline__ uint64_t f2_pack(float lo, float hi) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}

// Layer 1 of one pixel: A2 word i = bf16x2(relu(W1 x + b1)) of hidden units (2i, 2i + 1),
// element 2i in the low half (the layout epilogue_hidden writes), x = bf16(rgb).
__device__ __forceinline__ void layer1_row(const Mlp2Params& p, float r, float g, float b, uint32_t (&w)[32]) {
  const float x0 = __bfloat162float(__float2bfloat16_rn(r));
  const float x1 = __bfloat162float(__float2bfloat16_rn(g));
  const float x2 = __bfloat162float(__float2bfloat16_rn(b));
#if HC_MLP2_L1_BF16
  const __nv_bfloat162 R = __floats2bfloat162_rn(x0, x0), G = __floats2bfloat162_rn(x1, x1),
                       B = __floats2bfloat162_rn(x2, x2);
  auto bf2 = [](unsigned long long v) {
    const float2 f = make_float2(__uint_as_float(static_cast<uint32_t>(v)), __uint_as_float(static_cast<uint32_t>(v >> 32)));
    return __floats2bfloat162_rn(f.x, f.y);
  };
#pragma unroll
  for (int i = 0; i < 32; ++i) {
    __nv_bfloat162 h = __hfma2(R, bf2(p.w1p[0][i]), bf2(p.b1p[i]));
    h = __hfma2(G, bf2(p.w1p[1][i]), h);
    h = __hfma2_relu(B, bf2(p.w1p[2][i]), h);
    w[i] = *reinterpret_cast<uint32_t*>(&h);
  }
#else
  const uint64_t R = f2_pack(x0, x0), G = f2_pack(x1, x1), B = f2_pack(x2, x2);
#pragma unroll
  for (int i = 0; i < 32; ++i) {
    uint64_t h = ffma2(R, p.w1p[0][i], p.b1p[i]);
    h = ffma2(G, p.w1p[1][i], h);
    h = ffma2(B, p.w1p[2][i], h);
    float lo, hi;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(h));
    w[i] = pack_relu_bf16(lo, hi);
  }
#endif
}

template <int ST>
__device__ __forceinline__ void mlp2_issuer(const Mlp2Params& p, unsigned char* sm, float* ring, int64_t t0,
                                            int64_t tstride) {
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + kOffBar2) + ST * kBars2;
  uint64_t* bar_in = bars;
  uint64_t* bar_l2 = bars + kRing2;
  uint64_t* bar_l3 = bars + kRing2 + 1;
  uint64_t* bar_a2 = bars + kRing2 + 2;
  uint64_t* bar_a3 = bars + kRing2 + 3;
  constexpr uint32_t tA2 = ST * kCols2, tA3 = tA2 + 32, tD = tA2 + 64, tD3 = tA2 + 128, tC = kColConst2;
  const bool elect = (threadIdx.x & 31) == 0;
  const uint32_t sW2 = smem_u32(sm + kOffW2b), sW3 = smem_u32(sm + kOffW3b);
  constexpr uint32_t id64 = idesc_bf16(kMlpM, kHid), id16 = idesc_bf16(kMlpM, kN3);
  auto load_tile = [&](int64_t t, int s) {
    mbar_arrive_expect_tx(&bar_in[s], kInTile);
    bulk_g2s(ring + s * kMlpM * 3, p.rgb + (p.first_tile + t) * kMlpM * 3, kInTile, &bar_in[s]);
  };
  if (p.use_tma && elect)
    for (int s = 0; s < kRing2; ++s)
      if (t0 + s * tstride < p.ntiles) load_tile(t0 + s * tstride, s);
  int it = 0;
  for (int64_t t = t0; t < p.ntiles; t += tstride, ++it) {
    mbar_wait(bar_a2, it & 1);  // A2(t) in TMEM; its rgb slot has been read
    if (elect && p.use_tma && t + kRing2 * tstride < p.ntiles) load_tile(t + kRing2 * tstride, it % kRing2);
    __syncwarp();
    tc_fence_after();
#pragma unroll
    for (int kk = 0; kk < kK2 / 16; ++kk)
      mma_ts_w(tD, kk < kHid / 16 ? tA2 + kk * 8 : tC, umma_desc(sW2 + kk * 2 * (kHid * 16), kHid * 16, 128), id64,
               kk > 0);
    mma_commit_w(bar_l2);
    __syncwarp();
    mbar_wait(bar_a3, it & 1);  // A3(t) in TMEM, D(t) and D3(t - 1) read out
    tc_fence_after();
#pragma unroll
    for (int kk = 0; kk < kK3 / 16; ++kk)
      mma_ts_w(tD3, tA3 + kk * 8, umma_desc(sW3 + kk * 2 * (kN3 * 16), kN3 * 16, 128), id16, kk > 0);
    mma_commit_w(bar_l3);
    __syncwarp();
  }
  (void)bar_l3;
}

__global__ void __launch_bounds__(kThreads2, 1) mlp2_kernel(const __grid_constant__ Mlp2Params p) {
  extern __shared__ __align__(1024) unsigned char sm[];
  const int tid = threadIdx.x;
  const int warp = tid >> 5;
  const bool issuer = tid >= kEpi2;
  const int st = issuer ? (tid - kEpi2) >> 5 : warp >> 2;
  const int quarter = warp & 3;
  const int r = tid & 127;
  float* ring = reinterpret_cast<float*>(sm + kOffRing2 + st * kStream2Bytes);
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + kOffBar2) + st * kBars2;
  uint64_t* bar_in = bars;               // [R] rgb tile landed
  uint64_t* bar_l2 = bars + kRing2;      // layer-2 MMAs complete (and every earlier MMA)
  uint64_t* bar_l3 = bars + kRing2 + 1;  // layer-3 MMAs complete
  uint64_t* bar_a2 = bars + kRing2 + 2;  // A2 in TMEM (4 epilogue warps)
  uint64_t* bar_a3 = bars + kRing2 + 3;  // A3 in TMEM, D and D3 read (4 epilogue warps)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(sm + kOffBar2 + kS2 * kBars2 * 8);

  for (int i = tid; i < (kW2Bytes + kW3Bytes) / 16; i += kThreads2)
    reinterpret_cast<uint4*>(sm)[i] = reinterpret_cast<const uint4*>(p.wimg)[i];
  if (issuer && (tid & 31) == 0) {
    for (int i = 0; i < kRing2 + 2; ++i) mbar_init(&bars[i], 1);
    mbar_init(bar_a2, 4);
    mbar_init(bar_a3, 4);
    fence_mbar_init();
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  if (warp < 4) {  // constant K chunk of A2: element 64 = 1 (b2), 65..79 = 0
    uint32_t one[8] = {0x3F80u, 0u, 0u, 0u, 0u, 0u, 0u, 0u};
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(
                     tmem + kColConst2 + (static_cast<uint32_t>(warp * 32) << 16)),
                 "r"(one[0]), "r"(one[1]), "r"(one[2]), "r"(one[3]), "r"(one[4]), "r"(one[5]), "r"(one[6]),
                 "r"(one[7])
                 : "memory");
    tmem_wait_st();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tcol = tmem + st * kCols2;
  const uint32_t tA2 = tcol, tA3 = tcol + 32, tD = tcol + 64, tD3 = tcol + 128, tC = tmem + kColConst2;
  const int64_t t0 = static_cast<int64_t>(blockIdx.x) * kS2 + st;
  const int64_t tstride = static_cast<int64_t>(gridDim.x) * kS2;

  if (issuer) {
    // The stream index is a template argument and the TMEM base is 0 (the CTA owns all 512
    // columns), so every MMA operand is warp-uniform at compile time: no per-MMA R2UR
    // waterfall (tools/mma_probe3.cu's ~45 cycles per issued MMA came from it).
    if (tmem != 0 && (tid & 31) == 0) __trap();
    switch (st) {
      case 0: mlp2_issuer<0>(p, sm, ring, t0, tstride); break;
#if HC_MLP2_STREAMS > 1
      case 1: mlp2_issuer<1>(p, sm, ring, t0, tstride); break;
#endif
#if HC_MLP2_STREAMS > 2
      case 2: mlp2_issuer<2>(p, sm, ring, t0, tstride); break;
#endif
#if HC_MLP2_STREAMS > 3
      case 3: mlp2_issuer<3>(p, sm, ring, t0, tstride); break;
#endif
      default: break;
    }
  } else {
    const uint32_t lane_off = static_cast<uint32_t>(quarter * 32) << 16;
    const int k = p.k;
    uint32_t prev_v[kN3];
    int64_t prev_row0 = -1;
    int prev_rows = 0;
    auto store_codes = [&]() {
      if (prev_row0 < 0 || r >= prev_rows) return;
      float* o = p.out + (prev_row0 + r) * k;
      if (k == 6 && p.vec2) {
        float y[6];
#pragma unroll
        for (int j = 0; j < 6; ++j) y[j] = softplus1(__uint_as_float(prev_v[j]) + p.b3[j]);
        reinterpret_cast<float2*>(o)[0] = make_float2(y[0], y[1]);
        reinterpret_cast<float2*>(o)[1] = make_float2(y[2], y[3]);
        reinterpret_cast<float2*>(o)[2] = make_float2(y[4], y[5]);
      } else {
#pragma unroll
        for (int j = 0; j < kMaxK; ++j)
          if (j < k) o[j] = softplus1(__uint_as_float(prev_v[j]) + p.b3[j]);
      }
    };
    auto handoff = [&](uint64_t* bar) {
      tc_fence_before();
      __syncwarp();
      if ((tid & 31) == 0) mbar_arrive(bar);
    };
    auto rgb_row = [&](int64_t t, int it, float& x0, float& x1, float& x2) {
      if (p.use_tma) {
        const int s = it % kRing2;
        mbar_wait(&bar_in[s], (it / kRing2) & 1);
        const float* in = ring + s * kMlpM * 3 + r * 3;
        x0 = in[0];
        x1 = in[1];
        x2 = in[2];
      } else {
        const int64_t row = (p.first_tile + t) * kMlpM + r;
        x0 = x1 = x2 = 0.f;
        if (row < p.P) {
          const float* in = p.rgb + row * 3;
          x0 = in[0];
          x1 = in[1];
          x2 = in[2];
        }
      }
    };
    auto store_a2 = [&](const uint32_t (&w)[32]) {
      HC_TMEM_ST16(tA2 + lane_off, w);
      HC_TMEM_ST16(tA2 + lane_off + 16, (&w[16]));
      tmem_wait_st();
      handoff(bar_a2);
    };
    uint32_t a2w[32];
    if (t0 < p.ntiles) {
      float x0, x1, x2;
      rgb_row(t0, 0, x0, x1, x2);
      layer1_row(p, x0, x1, x2, a2w);
      store_a2(a2w);
    }
    int it = 0;
    for (int64_t t = t0; t < p.ntiles; t += tstride, ++it) {
      const int64_t tn = t + tstride;
      const bool next = tn < p.ntiles;
      if (next) {  // layer 1 of the next tile, in registers, under layer 2 of this one
        float x0, x1, x2;
        rgb_row(tn, it + 1, x0, x1, x2);
        layer1_row(p, x0, x1, x2, a2w);
      }
      mbar_wait(bar_l2, it & 1);
      tc_fence_after();
      if (it > 0) {  // layer 3 of the previous tile is complete too (earlier MMA, same commit chain)
        HC_TMEM_LD_D3(tD3 + lane_off, prev_v, p.k);
      }
      // relu(D) -> bf16 A3, in two 32-column halves (register budget: 480 threads)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        uint32_t va[2][16], pk[16];
        HC_TMEM_LD16(tD + lane_off + 32 * h, va[0]);
        HC_TMEM_LD16(tD + lane_off + 32 * h + 16, va[1]);
        tmem_wait_ld();  // (covers the D3 load too)
#pragma unroll
        for (int q = 0; q < 2; ++q)
#pragma unroll
          for (int j = 0; j < 8; ++j)
            pk[q * 8 + j] = pack_relu_bf16(__uint_as_float(va[q][2 * j]), __uint_as_float(va[q][2 * j + 1]));
        HC_TMEM_ST16(tA3 + lane_off + 16 * h, pk);
      }
      tmem_wait_st();
      handoff(bar_a3);
      if (next) store_a2(a2w);
      store_codes();  // tile t - 1
      const int64_t row0 = (p.first_tile + t) * kMlpM;
      const int64_t left = p.P - row0;
      prev_row0 = row0;
      prev_rows = left < kMlpM ? static_cast<int>(left) : kMlpM;
    }
    if (it > 0) {
      mbar_wait(bar_l3, (it - 1) & 1);
      tc_fence_after();
      HC_TMEM_LD_D3(tD3 + lane_off, prev_v, p.k);
      tmem_wait_ld();
      store_codes();
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

}  // namespace hcb

using namespace hcb;

struct hc_mlp_s {
  hc_ctx ctx = nullptr;
  int hidden = 0, k = 0;
  uint8_t* d_wimg = nullptr;
  MlpParams base{};
  Mlp2Params base2{};
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
float bf16_value(float f) {
  const uint32_t u = static_cast<uint32_t>(to_bf16(f)) << 16;
  float r;
  std::memcpy(&r, &u, 4);
  return r;
}

// mlp2_kernel (layer 1 on the CUDA cores) unless HC_MLP_V1 is set or the build pins V1.
#ifndef HC_MLP_V2
#define HC_MLP_V2 0
#endif
bool use_v2() {
  const char* v1 = std::getenv("HC_MLP_V1");
  static const bool v2 = HC_MLP_V2 && !(v1 && *v1 && *v1 != '0');
  return v2;
}

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
    for (int j = 0; j < kHid; ++j) put_kmajor(img, kOffW2, kHid, kK2, n, j, w2[n * kHid + j]);
    put_kmajor(img, kOffW2, kHid, kK2, n, kHid, b2[n]);  // bias via the constant-1 A column
  }
  for (int n = 0; n < k; ++n) {
    for (int j = 0; j < kHid; ++j) put_kmajor(img, kOffW3, kN3, kK3, n, j, w3[n * kHid + j]);
  }
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
  // One CTA per SM: it allocates all 512 TMEM columns (4 streams x 128).
  m->occ = 1;
  if (e != cudaSuccess) {
    if (m->d_wimg) cudaFree(m->d_wimg);
    delete m;
    return cuda_error(e, "hc_mlp_create");
  }
  std::memset(&m->base, 0, sizeof(m->base));
  for (int i = 0; i < kHid; ++i) m->base.b2[i] = b2[i];
  for (int i = 0; i < k; ++i) m->base.b3[i] = b3[i];
  m->base.wimg = m->d_wimg;
  m->base.k = k;
  std::memset(&m->base2, 0, sizeof(m->base2));
  auto pair = [](float lo, float hi) {
    const float f[2] = {bf16_value(lo), bf16_value(hi)};
    unsigned long long v;
    std::memcpy(&v, f, 8);
    return v;
  };
  for (int i = 0; i < kHid / 2; ++i) {
    for (int c = 0; c < 3; ++c) m->base2.w1p[c][i] = pair(w1[(2 * i) * 3 + c], w1[(2 * i + 1) * 3 + c]);
    m->base2.b1p[i] = pair(b1[2 * i], b1[2 * i + 1]);
  }
  for (int i = 0; i < k; ++i) m->base2.b3[i] = b3[i];
  m->base2.wimg = m->d_wimg + kOffW2;  // W2' | W3 images are contiguous
  m->base2.k = k;
  if (use_v2()) {
    e = cudaFuncSetAttribute(mlp2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem2);
    if (e != cudaSuccess) {
      cudaFree(m->d_wimg);
      delete m;
      return cuda_error(e, "hc_mlp_create (mlp2_kernel)");
    }
  }
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
  const bool aligned = (reinterpret_cast<uintptr_t>(rgb) & 15u) == 0;  // rgb tiles arrive by bulk copy
  if (use_v2()) {
    Mlp2Params q = m->base2;
    q.rgb = rgb;
    q.out = codes;
    q.P = P;
    q.vec2 = (reinterpret_cast<uintptr_t>(codes) & 7u) == 0;  // float2 code stores need 8-byte rows
    const int64_t full = aligned ? P / kMlpM : 0;
    if (full > 0) {
      q.first_tile = 0;
      q.ntiles = full;
      q.use_tma = 1;
      const int grid = static_cast<int>(std::min<int64_t>((full + kS2 - 1) / kS2, ctx->sm_count));
      mlp2_kernel<<<grid, kThreads2, kSmem2, ctx->stream>>>(q);
      HC_CHECK_LAUNCH(ctx, "mlp2_kernel");
    }
    if (full * kMlpM < P) {
      q.first_tile = full;
      q.ntiles = (P - full * kMlpM + kMlpM - 1) / kMlpM;
      q.use_tma = 0;
      const int grid = static_cast<int>(std::min<int64_t>((q.ntiles + kS2 - 1) / kS2, ctx->sm_count));
      mlp2_kernel<<<grid, kThreads2, kSmem2, ctx->stream>>>(q);
      HC_CHECK_LAUNCH(ctx, "mlp2_kernel(tail)");
    }
    return HC_OK;
  }
  MlpParams p = m->base;
  p.rgb = rgb;
  p.out = codes;
  p.P = P;
  if (p.k == 6 && (reinterpret_cast<uintptr_t>(codes) & 7u) != 0)
    return set_error(HC_EINVAL, "mlp: codes must be 8-byte aligned (HC_MLP_V1 kernel)");
  // codes tile = 128 * k * 4 bytes: 16-byte multiple for any k
  const int64_t full = aligned ? P / kMlpM : 0;
  if (full > 0) {
    p.first_tile = 0;
    p.ntiles = full;
    p.use_tma = 1;
    const int grid = static_cast<int>(std::min<int64_t>(full, static_cast<int64_t>(m->occ) * ctx->sm_count));
    if (std::getenv("HC_DEBUG")) std::fprintf(stderr, "[hc] mlp_kernel grid=%d occ=%d smem=%d\n", grid, m->occ, kSmemBytes);
    long long* trace = nullptr;
    if (std::getenv("HC_MLP_TRACE")) {
      cudaMalloc(&trace, kStreams * 32 * 8 * sizeof(long long));
      cudaMemset(trace, 0, kStreams * 32 * 8 * sizeof(long long));
      p.trace = trace;
    }
    mlp_kernel<<<grid, kThreads, kSmemBytes, ctx->stream>>>(p);
    HC_CHECK_LAUNCH(ctx, "mlp_kernel");
    p.trace = nullptr;
    if (trace) {
      cudaStreamSynchronize(ctx->stream);
      std::vector<long long> h(kStreams * 32 * 8);
      cudaMemcpy(h.data(), trace, h.size() * sizeof(long long), cudaMemcpyDeviceToHost);
      cudaFree(trace);
      double acc[8] = {0};
      int n = 0;
      for (int st = 0; st < kStreams; ++st)
        for (int it = 4; it < 31; ++it) {
          const long long* a = &h[(st * 32 + it) * 8];
          const long long* b = &h[(st * 32 + it + 1) * 8];
          if (!a[0] || !b[0]) continue;
          for (int k = 1; k < 8; ++k) acc[k - 1] += double(a[k] - a[k - 1]);
          acc[7] += double(b[0] - a[7]);
          ++n;
        }
      if (n)
        std::fprintf(stderr, "[hc] mlp phase cycles (avg of %d tiles): prevD3 %.0f L1wait %.0f epi1 %.0f codes %.0f L2wait %.0f epi2 %.0f - %.0f loop %.0f\n",
                     n, acc[0] / n, acc[1] / n, acc[2] / n, acc[3] / n, acc[4] / n, acc[5] / n, acc[6] / n, acc[7] / n);
    }
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
