// hadacodec-b200: the codec training step on the GPU — the losses
// and their analytic gradients (trainer.cpp:49-201 forward / losses, :221-373 gradients)
// over a batch of (reflectance, illumination) pairs, and the Adam update (:399-411).
//
// Bit-identical to the reference: everything is fp64 in the reference's expression order
// (this file is compiled with -fmad=false), and every sum the reference accumulates
// sequentially over the batch is accumulated in the same order here:
//   pair_kernel      one thread per pair: forward_pair, the four per-pair loss terms and
//                    the pair's local gradient factors (dL/ds_hat, dL/dz, rec residuals);
//   grad_reduce      one thread per weight: the pairs' contributions in batch order (for a
//                    decoder weight: the s_hat backprop term, then the rec term, per pair;
//                    for an encoder weight: the code term, then the encoder-row term), the
//                    alg regularizer, and the chain through softplus;
//   loss_reduce      one thread: the batch means in batch order, loss_alg, the total.
// softplus and its derivative are evaluated on the host (glibc's exp / log1p, as the
// reference) and passed in; the device's exp differs in the last ulp.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <vector>

#include "hadacodec_b200.h"
#include "hc_internal.h"
#include "hc_tma.cuh"

namespace hcb {
namespace {

constexpr double kCosEps = 1e-12;  // trainer.cpp:18

struct LossW {
  double e2e, rec, code, col, alg;
};

// Per-pair outputs, stored transposed — [element][pair] — so that the per-weight batch
// reductions read contiguous streams (and a warp of consecutive pairs stores coalesced).
struct PairBufs {
  double* gshat;   // n x m   dL/ds_hat (e2e + col terms)
  double* grr;     // n x m   rec residual factor for R
  double* grl;     // n x m   rec residual factor for L
  double* rT;      // n x m   R, transposed
  double* lT;      // n x m   L, transposed
  double* zp;      // k x m
  double* zr;      // k x m
  double* zl;      // k x m
  double* gc;      // k x m   code-term gradient per code
  double* gzr;     // k x m   accumulated dL/dzr
  double* gzl;     // k x m   accumulated dL/dzl
  double* terms;   // 4 x m   e2e, rec, code, col per pair
};
// Rows of the transposed arrays are ld = m rounded up to an even count apart, so every
// 64-pair chunk of a row is a 16-byte-aligned 512-byte run (one bulk copy).

template <int K, int N>
__global__ void __launch_bounds__(128) pair_kernel(const double* __restrict__ E, const double* __restrict__ D,
                                                   const double* __restrict__ T, double lstep,
                                                   const double* __restrict__ refl, const double* __restrict__ illum,
                                                   int64_t m, int64_t ld, LossW lw, PairBufs pb) {
  const int64_t j = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (j >= m) return;
  const double* r = refl + j * N;
  const double* l = illum + j * N;
  double zr[K], zl[K], zp[K], zc[K];
  // forward_pair (trainer.cpp:49-62)
  for (int c = 0; c < K; ++c) {
    double ar = 0.0, al = 0.0, as = 0.0;
    for (int i = 0; i < N; ++i) {
      ar += E[c * N + i] * r[i];
      al += E[c * N + i] * l[i];
      as += E[c * N + i] * (r[i] * l[i]);
    }
    zr[c] = ar;
    zl[c] = al;
    zc[c] = as;
  }
  for (int c = 0; c < K; ++c) zp[c] = zr[c] * zl[c];
  // s_hat[i] = D zp, rec_r[i] = D zr, rec_l[i] = D zl (matvec_dec, trainer.cpp:39-47), each
  // recomputed where needed (same expression, same value) instead of kept in arrays
  auto dec3 = [&](int i, double* sh, double* rr, double* rl) {
    double a = 0.0, b = 0.0, d = 0.0;
#pragma unroll
    for (int c = 0; c < K; ++c) {
      a += D[i * K + c] * zp[c];
      b += D[i * K + c] * zr[c];
      d += D[i * K + c] * zl[c];
    }
    *sh = a;
    *rr = b;
    *rl = d;
  };
  // pass 1: the per-pair loss sums (loss_e2e / loss_rec / loss_col, trainer.cpp:108-172);
  // every accumulator runs over i in order, as in its own loop in the reference
  double mse = 0.0, dot = 0.0, na = 0.0, nb = 0.0, mr = 0.0, ml = 0.0, dcol[3] = {0.0, 0.0, 0.0};
  for (int i = 0; i < N; ++i) {
    double sh, rr, rl;
    dec3(i, &sh, &rr, &rl);
    const double s = r[i] * l[i];
    const double d = sh - s;
    mse += d * d;
    dot += sh * s;
    na += sh * sh;
    nb += s * s;
    const double dr = rr - r[i], dl = rl - l[i];
    mr += dr * dr;
    ml += dl * dl;
#pragma unroll
    for (int c = 0; c < 3; ++c) dcol[c] += T[c * N + i] * (sh - s);
  }
  mse = mse / N;
  const double a = sqrt(na), bb = sqrt(nb);
  const double cosv = dot / ((a + kCosEps) * (bb + kCosEps));
  double codes = 0.0;
  for (int c = 0; c < K; ++c) {
    const double d = zp[c] - zc[c];
    codes += d * d;
  }
  double cols = 0.0;
  for (int c = 0; c < 3; ++c) {
    dcol[c] *= lstep;
    cols += dcol[c] * dcol[c];
  }
  pb.terms[0 * ld + j] = mse * (2.0 - cosv);
  pb.terms[1 * ld + j] = mr / N + ml / N;
  pb.terms[2 * ld + j] = codes / K;
  pb.terms[3 * ld + j] = cols / 3.0;
  // pass 2: dL/ds_hat (trainer.cpp:255-285: the e2e term, then the three col terms, per i)
  // and its backprop into zp (:288-297)
  const double md = static_cast<double>(m);
  const double u = 1.0 / ((a + kCosEps) * (bb + kCosEps));
  const double cs = dot * u;
  const double w_e2e = lw.e2e / md, w_col = lw.col / md;
  double coef[3];
  for (int c = 0; c < 3; ++c) coef[c] = w_col * (2.0 / 3.0) * dcol[c] * lstep;
  double gzp[K], gzr[K], gzl[K];
  for (int c = 0; c < K; ++c) gzp[c] = gzr[c] = gzl[c] = 0.0;
  for (int i = 0; i < N; ++i) {
    double sh, rr, rl;
    dec3(i, &sh, &rr, &rl);
    double gs = 0.0;
    if (lw.e2e != 0.0) {
      const double s = r[i] * l[i];
      double gi = (2.0 - cs) * (2.0 / N) * (sh - s);
      double dcos = s * u;
      if (a > 0.0) dcos -= dot * sh / (a * (a + kCosEps) * (a + kCosEps) * (bb + kCosEps));
      gi -= mse * dcos;
      gs += w_e2e * gi;
    }
    if (lw.col != 0.0)
      for (int c = 0; c < 3; ++c) gs += coef[c] * T[c * N + i];
    pb.gshat[i * ld + j] = gs;
    if (gs == 0.0) continue;
#pragma unroll
    for (int c = 0; c < K; ++c) gzp[c] += D[i * K + c] * gs;
  }
  for (int c = 0; c < K; ++c) {  // code term (trainer.cpp:300-311)
    double gcv = 0.0;
    if (lw.code != 0.0) {
      gcv = lw.code / md * (2.0 / K) * (zp[c] - zc[c]);
      gzp[c] += gcv;
    }
    pb.gc[c * ld + j] = gcv;
  }
  for (int c = 0; c < K; ++c) {  // zp = zr o zl
    gzr[c] += gzp[c] * zl[c];
    gzl[c] += gzp[c] * zr[c];
  }
  // pass 3: rec (trainer.cpp:321-336)
  const double w_rec = lw.rec / md;
  for (int i = 0; i < N; ++i) {
    double gr = 0.0, gl = 0.0;
    if (lw.rec != 0.0) {
      double sh, rr, rl;
      dec3(i, &sh, &rr, &rl);
      gr = w_rec * (2.0 / N) * (rr - r[i]);
      gl = w_rec * (2.0 / N) * (rl - l[i]);
#pragma unroll
      for (int c = 0; c < K; ++c) {
        gzr[c] += D[i * K + c] * gr;
        gzl[c] += D[i * K + c] * gl;
      }
    }
    pb.grr[i * ld + j] = gr;
    pb.grl[i * ld + j] = gl;
    pb.rT[i * ld + j] = r[i];
    pb.lT[i * ld + j] = l[i];
  }
  for (int c = 0; c < K; ++c) {
    pb.zp[c * ld + j] = zp[c];
    pb.zr[c * ld + j] = zr[c];
    pb.zl[c * ld + j] = zl[c];
    pb.gzr[c * ld + j] = gzr[c];
    pb.gzl[c * ld + j] = gzl[c];
  }
}

// ------------------------------------------------------------------ ordered batch reductions
// Each weight's gradient (and each batch-mean loss) is a sequential sum over the pairs in
// batch order, as in the reference, so the parallelism is across weights only — and each
// chain must not wait on memory.  One warp per block: the warp's lanes own up to 32
// weights, lane -> (code lane % K, wavelength w * (32 / K) + lane / K), so their inputs are
// at most ~45 contiguous per-pair streams (rows of the transposed buffers: three per code,
// two or three per wavelength); a 4-stage ring of 128-pair chunks of all those streams is
// filled by bulk copies
// (cp.async.bulk, one mbarrier per stage) while the lanes run their chains from shared
// memory.  Stream rows in shared memory are 528 B apart, so the lanes' double2 reads of
// different streams spread over the banks.  The reference's skipped adds are adds of a
// selected 0.0 here (branch-free, so the shared-memory loads pipeline ahead of the chain):
// the same sums, since an accumulator that starts at +0.0 never holds -0.0 and x + 0.0 = x
// for every other x.
constexpr int kChunkPairs = 128;
constexpr int kStages = 4;
constexpr int kMaxStreams = 48;
constexpr int kStreamStride = kChunkPairs * 8 + 16;  // bytes
constexpr size_t kRingBytes = size_t(kStages) * kMaxStreams * kStreamStride;

struct StreamRing {
  unsigned char* buf;  // kStages x kMaxStreams x kStreamStride
  uint64_t* bar;       // kStages
  const double* const* base;
  int count;
  __device__ const double* stream(int stage, int q) const {
    return reinterpret_cast<const double*>(buf + (size_t(stage) * kMaxStreams + q) * kStreamStride);
  }
  // all lanes: copies of chunk t into its stage (lane 0 sets the byte count)
  __device__ void issue(int64_t t, int lane) const {
    const int st = static_cast<int>(t % kStages);
    if (lane == 0) mbar_arrive_expect_tx(&bar[st], static_cast<uint32_t>(count) * kChunkPairs * 8);
    for (int q = lane; q < count; q += 32)
      bulk_g2s(buf + (size_t(st) * kMaxStreams + q) * kStreamStride, base[q] + t * kChunkPairs, kChunkPairs * 8,
               &bar[st]);
  }
  __device__ void wait(int64_t t) const {
    mbar_wait(&bar[t % kStages], static_cast<uint32_t>((t / kStages) & 1));
  }
};

__device__ inline void ring_init(uint64_t* bar, int lane) {
  if (lane == 0) {
    for (int s = 0; s < kStages; ++s) mbar_init(&bar[s], 1);
    fence_mbar_init();
  }
  __syncwarp();
}

// Grid: enc warps [0, ceil(KN/32)), then dec warps.  Dynamic smem: kRingBytes.
template <int K, int N>
__device__ void loss_reduce(const double* __restrict__ D, int64_t m, int64_t ld, LossW lw,
                            const double* __restrict__ terms, double* __restrict__ out);

template <int K, int N>
__global__ void __launch_bounds__(32) grad_reduce_kernel(const double* __restrict__ D, int64_t m, int64_t ld, LossW lw,
                                                         PairBufs pb, const double* __restrict__ sd_enc,
                                                         const double* __restrict__ sd_dec,
                                                         double* __restrict__ g_enc, double* __restrict__ g_dec,
                                                         double* __restrict__ losses, int loss_block) {
  constexpr int kPerWarp = 32 / K;                          // wavelengths per warp
  constexpr int kWarpsPerHalf = (N + kPerWarp - 1) / kPerWarp;
  if (static_cast<int>(blockIdx.x) == loss_block) {  // the batch-mean losses, concurrently with the weights
    loss_reduce<K, N>(D, m, ld, lw, pb.terms, losses);
    return;
  }
  extern __shared__ __align__(128) unsigned char ring_buf[];
  __shared__ uint64_t bar[kStages];
  __shared__ const double* base[kMaxStreams];
  const int lane = threadIdx.x;
  const bool dec = blockIdx.x >= kWarpsPerHalf;
  const int w = dec ? blockIdx.x - kWarpsPerHalf : blockIdx.x;
  const int i_lo = w * kPerWarp;
  const int ni = min(kPerWarp, N - i_lo);
  const int c = lane % K;
  const int il = min(lane / K, ni - 1);  // idle lanes repeat a live weight
  const int i = i_lo + il;
  const bool live = lane < K * kPerWarp && lane / K < ni;
  const bool code = lw.code != 0.0, rec = lw.rec != 0.0;
  // streams: per code c: 3 rows [0, 3K); per wavelength: enc R, L (2) / dec gshat, grr, grl (3)
  int count, s0, s1, s2, s3, s4, s5;
  if (lane < K) {
    base[3 * lane + 0] = (dec ? pb.zp : pb.gc) + lane * ld;
    base[3 * lane + 1] = (dec ? pb.zr : pb.gzr) + lane * ld;
    base[3 * lane + 2] = (dec ? pb.zl : pb.gzl) + lane * ld;
  }
  if (!dec) {  // weight (c, i) of the encoder: gc, gzr, gzl of code c; R, L at wavelength i
    count = 3 * K + 2 * ni;
    if (lane < ni) {
      base[3 * K + lane] = pb.rT + (i_lo + lane) * ld;
      base[3 * K + ni + lane] = pb.lT + (i_lo + lane) * ld;
    }
    s0 = 3 * c;
    s1 = s0 + 1;
    s2 = s0 + 2;
    s3 = 3 * K + il;
    s4 = 3 * K + ni + il;
    s5 = 0;
  } else {  // weight (i, c) of the decoder: gshat, grr, grl at wavelength i; zp, zr, zl of code c
    count = 3 * K + 3 * ni;
    if (lane < ni) {
      base[3 * K + 3 * lane + 0] = pb.gshat + (i_lo + lane) * ld;
      base[3 * K + 3 * lane + 1] = pb.grr + (i_lo + lane) * ld;
      base[3 * K + 3 * lane + 2] = pb.grl + (i_lo + lane) * ld;
    }
    s0 = 3 * K + 3 * il;
    s1 = s0 + 1;
    s2 = s0 + 2;
    s3 = 3 * c;
    s4 = s3 + 1;
    s5 = s3 + 2;
  }
  ring_init(bar, lane);
  const StreamRing ring{ring_buf, bar, base, count};
  const int64_t nfull = m / kChunkPairs;
  for (int64_t t = 0; t < nfull && t < kStages; ++t) ring.issue(t, lane);
  double acc = 0.0;
  for (int64_t t = 0; t < nfull; ++t) {
    ring.wait(t);
    const int st = static_cast<int>(t % kStages);
    if (!dec) {
      const double2* gc = reinterpret_cast<const double2*>(ring.stream(st, s0));
      const double2* gr = reinterpret_cast<const double2*>(ring.stream(st, s1));
      const double2* gl = reinterpret_cast<const double2*>(ring.stream(st, s2));
      const double2* rv = reinterpret_cast<const double2*>(ring.stream(st, s3));
      const double2* lv = reinterpret_cast<const double2*>(ring.stream(st, s4));
#pragma unroll 8
      for (int p = 0; p < kChunkPairs / 2; ++p) {
        const double2 a = gc[p], b = gr[p], x = gl[p], y = rv[p], z = lv[p];
        acc = acc - (code ? a.x * (y.x * z.x) : 0.0);
        acc = acc + ((b.x == 0.0 && x.x == 0.0) ? 0.0 : b.x * y.x + x.x * z.x);
        acc = acc - (code ? a.y * (y.y * z.y) : 0.0);
        acc = acc + ((b.y == 0.0 && x.y == 0.0) ? 0.0 : b.y * y.y + x.y * z.y);
      }
    } else {
      const double2* gs = reinterpret_cast<const double2*>(ring.stream(st, s0));
      const double2* rr = reinterpret_cast<const double2*>(ring.stream(st, s1));
      const double2* rl = reinterpret_cast<const double2*>(ring.stream(st, s2));
      const double2* zp = reinterpret_cast<const double2*>(ring.stream(st, s3));
      const double2* zr = reinterpret_cast<const double2*>(ring.stream(st, s4));
      const double2* zl = reinterpret_cast<const double2*>(ring.stream(st, s5));
#pragma unroll 8
      for (int p = 0; p < kChunkPairs / 2; ++p) {
        const double2 a = gs[p], q = zp[p], r1 = rr[p], r2 = rl[p], w1 = zr[p], w2 = zl[p];
        acc = acc + (a.x != 0.0 ? a.x * q.x : 0.0);
        acc = acc + (rec ? r1.x * w1.x + r2.x * w2.x : 0.0);
        acc = acc + (a.y != 0.0 ? a.y * q.y : 0.0);
        acc = acc + (rec ? r1.y * w1.y + r2.y * w2.y : 0.0);
      }
    }
    __syncwarp();
    if (t + kStages < nfull) ring.issue(t + kStages, lane);
  }
  // the last m % kChunkPairs pairs straight from global memory
  for (int64_t j = nfull * kChunkPairs; j < m; ++j) {
    if (!dec) {
      const double a = base[s0][j], b = base[s1][j], x = base[s2][j], y = base[s3][j], z = base[s4][j];
      if (code) acc -= a * (y * z);
      if (!(b == 0.0 && x == 0.0)) acc += b * y + x * z;
    } else {
      const double a = base[s0][j];
      if (a != 0.0) acc += a * base[s3][j];
      if (rec) acc += base[s1][j] * base[s4][j] + base[s2][j] * base[s5][j];
    }
  }
  if (!live) return;
  if (!dec) {
    g_enc[c * N + i] = acc * sd_enc[c * N + i];
    return;
  }
  if (lw.alg != 0.0) {  // trainer.cpp:336-355
    const double off_terms = K > 1 ? static_cast<double>(K) * (K - 1) : 1.0;
    const double* wr = D + i * K;
    double gg = 0.0;
    for (int q = 0; q < K; ++q) {
      if (q == c) continue;
      gg += 4.0 * wr[c] * wr[q] * wr[q] / off_terms;
    }
    const double bi = wr[c];
    gg += 2.0 * (bi * bi - bi) * (2.0 * bi - 1.0) / K;
    acc += lw.alg * gg;
  }
  g_dec[i * K + c] = acc * sd_dec[i * K + c];
}

// Batch means in batch order (lanes 0-3: one loss term each, from the same staged ring),
// loss_alg (trainer.cpp:174-201) and the weighted total.  One warp.
template <int K, int N>
__device__ void loss_reduce(const double* __restrict__ D, int64_t m, int64_t ld, LossW lw,
                            const double* __restrict__ terms, double* __restrict__ out) {
  extern __shared__ __align__(128) unsigned char ring_buf[];
  __shared__ uint64_t bar[kStages];
  __shared__ const double* base[kMaxStreams];
  const int lane = threadIdx.x;
  if (lane < 4) base[lane] = terms + lane * ld;
  ring_init(bar, lane);
  const StreamRing ring{ring_buf, bar, base, 4};
  const int64_t nfull = m / kChunkPairs;
  for (int64_t t = 0; t < nfull && t < kStages; ++t) ring.issue(t, lane);
  const int q = lane < 4 ? lane : 0;
  double acc = 0.0;
  for (int64_t t = 0; t < nfull; ++t) {
    ring.wait(t);
    const double* v = ring.stream(static_cast<int>(t % kStages), q);
#pragma unroll 8
    for (int p = 0; p < kChunkPairs; ++p) acc += v[p];
    __syncwarp();
    if (t + kStages < nfull) ring.issue(t + kStages, lane);
  }
  for (int64_t j = nfull * kChunkPairs; j < m; ++j) acc += base[q][j];
  __shared__ double sums[4];
  if (lane < 4) sums[lane] = acc;
  __syncwarp();
  if (lane != 0) return;
  const double md = static_cast<double>(m);
  double off = 0.0, idem = 0.0;
  for (int i = 0; i < K; ++i)
    for (int j = 0; j < K; ++j) {
      if (i == j) continue;
      double s = 0.0;
      for (int a = 0; a < N; ++a) {
        const double p = D[a * K + i] * D[a * K + j];
        s += p * p;
      }
      off += s;
    }
  for (int i = 0; i < K; ++i) {
    double s = 0.0;
    for (int a = 0; a < N; ++a) {
      const double bi = D[a * K + i];
      const double d = bi * bi - bi;
      s += d * d;
    }
    idem += s;
  }
  const double off_terms = K > 1 ? static_cast<double>(K) * (K - 1) : 1.0;
  const double e2e = sums[0] / md, rec = sums[1] / md, code = sums[2] / md, col = sums[3] / md;
  const double alg = off / off_terms + idem / K;
  out[0] = e2e;
  out[1] = rec;
  out[2] = code;
  out[3] = col;
  out[4] = alg;
  out[5] = lw.e2e * e2e + lw.rec * rec + lw.code * code + lw.col * col + lw.alg * alg;
}

// adam_step (trainer.cpp:399-411); c1, c2 = 1 - beta^step from the host's pow.
__global__ void adam_kernel(double* __restrict__ p, const double* __restrict__ g, double* __restrict__ m1,
                            double* __restrict__ v1, int64_t count, double lr, double c1, double c2) {
  constexpr double b1 = 0.9, b2 = 0.999, eps = 1e-8;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < count; i += int64_t(gridDim.x) * blockDim.x) {
    m1[i] = b1 * m1[i] + (1.0 - b1) * g[i];
    v1[i] = b2 * v1[i] + (1.0 - b2) * g[i] * g[i];
    const double mh = m1[i] / c1;
    const double vh = v1[i] / c2;
    p[i] -= lr * mh / (sqrt(vh) + eps);
  }
}

double softplus_h(double raw, double beta) {  // codec.cpp:8-12
  const double t = beta * raw;
  if (t > 30.0) return raw;
  return std::log1p(std::exp(t)) / beta;
}

double softplus_derivative_h(double raw, double beta) {  // codec.cpp:14-19
  const double t = beta * raw;
  if (t > 30.0) return 1.0;
  const double e = std::exp(t);
  return e / (1.0 + e);
}

template <class F>
int dispatch_train(int k, int n, F&& f) {
  if (n == 47) {
    if (k == 3) return f(std::integral_constant<int, 3>{}, std::integral_constant<int, 47>{});
    if (k == 6) return f(std::integral_constant<int, 6>{}, std::integral_constant<int, 47>{});
    if (k == 9) return f(std::integral_constant<int, 9>{}, std::integral_constant<int, 47>{});
  } else if (n == 81) {
    if (k == 3) return f(std::integral_constant<int, 3>{}, std::integral_constant<int, 81>{});
    if (k == 6) return f(std::integral_constant<int, 6>{}, std::integral_constant<int, 81>{});
    if (k == 9) return f(std::integral_constant<int, 9>{}, std::integral_constant<int, 81>{});
  }
  return set_error(HC_EUNSUPPORTED, "codec training: compiled for n in {47, 81}, k in {3, 6, 9}");
}

}  // namespace
}  // namespace hcb

using namespace hcb;

extern "C" {

int hc_codec_train_grad(hc_ctx ctx, int k, int n, double beta, const double* raw_enc, const double* raw_dec,
                        const double* cmf, double lambda_step, const double* refl, const double* illum, int64_t m,
                        const double* loss_weights, double* g_raw_enc, double* g_raw_dec, double* losses) {
  HC_REQUIRE(ctx && raw_enc && raw_dec && cmf && loss_weights, HC_EINVAL, "codec training: null argument");
  HC_REQUIRE(k > 0 && k % 3 == 0 && n > 0, HC_EINVAL, "codec weights: bad shape");
  HC_REQUIRE(beta > 0.0, HC_EINVAL, "codec weights: beta must be positive");
  HC_REQUIRE(m > 0 && refl && illum, HC_EINVAL, "batch: empty");  // check_batch (trainer.cpp:102-107)
  HC_REQUIRE((g_raw_enc != nullptr) == (g_raw_dec != nullptr), HC_EINVAL, "codec training: both gradients or neither");
  const LossW lw{loss_weights[0], loss_weights[1], loss_weights[2], loss_weights[3], loss_weights[4]};
  // effective_weights and the softplus derivatives, on the host (glibc, as the reference)
  const size_t kn = static_cast<size_t>(k) * n;
  std::vector<double> host(4 * kn + 3 * static_cast<size_t>(n));
  double* E = host.data();
  double* D = E + kn;
  double* sde = D + kn;
  double* sdd = sde + kn;
  double* T = sdd + kn;
  for (size_t i = 0; i < kn; ++i) {
    E[i] = softplus_h(raw_enc[i], beta);
    D[i] = softplus_h(raw_dec[i], beta);
    sde[i] = softplus_derivative_h(raw_enc[i], beta);
    sdd[i] = softplus_derivative_h(raw_dec[i], beta);
  }
  for (int i = 0; i < 3 * n; ++i) T[i] = cmf[i];
  // scratch: weights | per-pair buffers (rows of ld doubles, 16-byte aligned) | gradients | losses
  const int64_t ld = (m + 1) & ~int64_t(1);
  auto up32 = [](size_t x) { return (x + 31) & ~size_t(31); };  // doubles
  const size_t wdoubles = up32(host.size());
  const size_t rows = static_cast<size_t>(5 * n + 6 * k + 4);
  const size_t pdoubles = rows * static_cast<size_t>(ld);
  const size_t wbytes = sizeof(double) * host.size();
  int rc = ensure_scratch(ctx, sizeof(double) * (wdoubles + pdoubles + 2 * kn + 8) + 256);
  if (rc != HC_OK) return rc;
  double* base = reinterpret_cast<double*>((reinterpret_cast<uintptr_t>(ctx->scratch) + 255) & ~uintptr_t(255));
  double* dW = base;
  PairBufs pb;
  double* q = base + wdoubles;
  auto take = [&](int nrows) {
    double* p = q;
    q += static_cast<size_t>(nrows) * ld;
    return p;
  };
  pb.gshat = take(n);
  pb.grr = take(n);
  pb.grl = take(n);
  pb.rT = take(n);
  pb.lT = take(n);
  pb.zp = take(k);
  pb.zr = take(k);
  pb.zl = take(k);
  pb.gc = take(k);
  pb.gzr = take(k);
  pb.gzl = take(k);
  pb.terms = take(4);
  double* dg = q;
  double* dloss = dg + 2 * kn;
  HC_CUDA_TRY(cudaMemcpyAsync(dW, host.data(), wbytes, cudaMemcpyHostToDevice, ctx->stream));
  const double* dE = dW;
  const double* dD = dW + kn;
  const double* dsde = dD + kn;
  const double* dsdd = dsde + kn;
  const double* dT = dsdd + kn;
  rc = dispatch_train(k, n, [&](auto Kc, auto Nc) {
    constexpr int K = decltype(Kc)::value, N = decltype(Nc)::value;
    pair_kernel<K, N><<<static_cast<int>((m + 127) / 128), 128, 0, ctx->stream>>>(dE, dD, dT, lambda_step, refl,
                                                                                  illum, m, ld, lw, pb);
    HC_CHECK_LAUNCH(ctx, "pair_kernel");
    if (g_raw_enc || losses) {  // weights' chains (when asked) + one warp for the losses
      auto kern = grad_reduce_kernel<K, N>;
      HC_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kRingBytes)));
      constexpr int kHalf = (N + 32 / K - 1) / (32 / K);
      const int blocks = (g_raw_enc ? 2 * kHalf : 0) + (losses ? 1 : 0);
      const int loss_block = losses ? blocks - 1 : -1;
      kern<<<blocks, 32, kRingBytes, ctx->stream>>>(dD, m, ld, lw, pb, dsde, dsdd, dg, dg + kn, dloss, loss_block);
      HC_CHECK_LAUNCH(ctx, "grad_reduce_kernel");
    }
    return HC_OK;
  });
  if (rc != HC_OK) return rc;
  if (g_raw_enc) {
    HC_CUDA_TRY(cudaMemcpyAsync(g_raw_enc, dg, sizeof(double) * kn, cudaMemcpyDeviceToHost, ctx->stream));
    HC_CUDA_TRY(cudaMemcpyAsync(g_raw_dec, dg + kn, sizeof(double) * kn, cudaMemcpyDeviceToHost, ctx->stream));
  }
  if (losses) HC_CUDA_TRY(cudaMemcpyAsync(losses, dloss, sizeof(double) * 6, cudaMemcpyDeviceToHost, ctx->stream));
  HC_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  return HC_OK;
}

int hc_adam_step(hc_ctx ctx, double* params, const double* grad, double* m1, double* v1, int64_t count, double lr,
                 int64_t step) {
  HC_REQUIRE(ctx, HC_EINVAL, "adam: null context");
  HC_REQUIRE(count >= 0 && step >= 1, HC_EINVAL, "adam: bad count / step");
  if (count == 0) return HC_OK;
  HC_REQUIRE(params && grad && m1 && v1, HC_EINVAL, "adam: null buffer");
  const double c1 = 1.0 - std::pow(0.9, static_cast<double>(step));
  const double c2 = 1.0 - std::pow(0.999, static_cast<double>(step));
  const int g = static_cast<int>(std::min<int64_t>((count + 255) / 256, int64_t(ctx->sm_count) * 8));
  adam_kernel<<<g, 256, 0, ctx->stream>>>(params, grad, m1, v1, count, lr, c1, c2);
  HC_CHECK_LAUNCH(ctx, "adam_kernel");
  return HC_OK;
}

}  // extern "C"
