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

namespace hcb {
namespace {

constexpr double kCosEps = 1e-12;  // trainer.cpp:18

struct LossW {
  double e2e, rec, code, col, alg;
};

// Per-pair outputs, structure of arrays over the batch (m pairs).
struct PairBufs {
  double* gshat;   // m x n   dL/ds_hat (e2e + col terms)
  double* grr;     // m x n   rec residual factor for R
  double* grl;     // m x n   rec residual factor for L
  double* zp;      // m x k
  double* zr;      // m x k
  double* zl;      // m x k
  double* gc;      // m x k   code-term gradient per code
  double* gzr;     // m x k   accumulated dL/dzr
  double* gzl;     // m x k   accumulated dL/dzl
  double* terms;   // m x 4   e2e, rec, code, col per pair
};

template <int K, int N>
__global__ void __launch_bounds__(128) pair_kernel(const double* __restrict__ E, const double* __restrict__ D,
                                                   const double* __restrict__ T, double lstep,
                                                   const double* __restrict__ refl, const double* __restrict__ illum,
                                                   int64_t m, LossW lw, PairBufs pb) {
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
  double shat[N], recr[N], recl[N], g[N];
  for (int i = 0; i < N; ++i) {
    double a = 0.0, b = 0.0, d = 0.0;
    for (int c = 0; c < K; ++c) {
      a += D[i * K + c] * zp[c];
      b += D[i * K + c] * zr[c];
      d += D[i * K + c] * zl[c];
    }
    shat[i] = a;
    recr[i] = b;
    recl[i] = d;
  }
  // per-pair loss terms (loss_e2e / loss_rec / loss_code / loss_col, trainer.cpp:108-172)
  double mse = 0.0, dot = 0.0, na = 0.0, nb = 0.0, mr = 0.0, ml = 0.0;
  for (int i = 0; i < N; ++i) {
    const double s = r[i] * l[i];
    const double d = shat[i] - s;
    mse += d * d;
    dot += shat[i] * s;
    na += shat[i] * shat[i];
    nb += s * s;
    const double dr = recr[i] - r[i], dl = recl[i] - l[i];
    mr += dr * dr;
    ml += dl * dl;
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
  double dcol[3];
  for (int c = 0; c < 3; ++c) {
    double d = 0.0;
    for (int i = 0; i < N; ++i) d += T[c * N + i] * (shat[i] - r[i] * l[i]);
    d *= lstep;
    dcol[c] = d;
    cols += d * d;
  }
  pb.terms[j * 4 + 0] = mse * (2.0 - cosv);
  pb.terms[j * 4 + 1] = mr / N + ml / N;
  pb.terms[j * 4 + 2] = codes / K;
  pb.terms[j * 4 + 3] = cols / 3.0;
  // gradients (trainer.cpp:236-359), per pair
  const double md = static_cast<double>(m);
  for (int i = 0; i < N; ++i) g[i] = 0.0;
  if (lw.e2e != 0.0) {
    const double u = 1.0 / ((a + kCosEps) * (bb + kCosEps));
    const double cs = dot * u;
    const double w_pair = lw.e2e / md;
    for (int i = 0; i < N; ++i) {
      const double s = r[i] * l[i];
      double gi = (2.0 - cs) * (2.0 / N) * (shat[i] - s);
      double dcos = s * u;
      if (a > 0.0) dcos -= dot * shat[i] / (a * (a + kCosEps) * (a + kCosEps) * (bb + kCosEps));
      gi -= mse * dcos;
      g[i] += w_pair * gi;
    }
  }
  if (lw.col != 0.0) {
    const double w_pair = lw.col / md;
    for (int c = 0; c < 3; ++c) {
      const double coef = w_pair * (2.0 / 3.0) * dcol[c] * lstep;
      for (int i = 0; i < N; ++i) g[i] += coef * T[c * N + i];
    }
  }
  double gzp[K], gzr[K], gzl[K];
  for (int c = 0; c < K; ++c) gzp[c] = gzr[c] = gzl[c] = 0.0;
  for (int i = 0; i < N; ++i) {  // backprop s_hat = W_dec zp
    const double gs = g[i];
    pb.gshat[j * N + i] = gs;
    if (gs == 0.0) continue;
    for (int c = 0; c < K; ++c) gzp[c] += D[i * K + c] * gs;
  }
  for (int c = 0; c < K; ++c) {  // code term
    double gcv = 0.0;
    if (lw.code != 0.0) {
      gcv = lw.code / md * (2.0 / K) * (zp[c] - zc[c]);
      gzp[c] += gcv;
    }
    pb.gc[j * K + c] = gcv;
  }
  for (int c = 0; c < K; ++c) {  // zp = zr o zl
    gzr[c] += gzp[c] * zl[c];
    gzl[c] += gzp[c] * zr[c];
  }
  const double w_rec = lw.rec / md;
  for (int i = 0; i < N; ++i) {  // rec
    double gr = 0.0, gl = 0.0;
    if (lw.rec != 0.0) {
      gr = w_rec * (2.0 / N) * (recr[i] - r[i]);
      gl = w_rec * (2.0 / N) * (recl[i] - l[i]);
      for (int c = 0; c < K; ++c) {
        gzr[c] += D[i * K + c] * gr;
        gzl[c] += D[i * K + c] * gl;
      }
    }
    pb.grr[j * N + i] = gr;
    pb.grl[j * N + i] = gl;
  }
  for (int c = 0; c < K; ++c) {
    pb.zp[j * K + c] = zp[c];
    pb.zr[j * K + c] = zr[c];
    pb.zl[j * K + c] = zl[c];
    pb.gzr[j * K + c] = gzr[c];
    pb.gzl[j * K + c] = gzl[c];
  }
}

// One thread per weight: encoder weights (c, i) first (K*N), then decoder weights (i, c).
template <int K, int N>
__global__ void __launch_bounds__(128) grad_reduce_kernel(const double* __restrict__ D,
                                                          const double* __restrict__ refl,
                                                          const double* __restrict__ illum, int64_t m, LossW lw,
                                                          PairBufs pb, const double* __restrict__ sd_enc,
                                                          const double* __restrict__ sd_dec,
                                                          double* __restrict__ g_enc, double* __restrict__ g_dec) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < K * N) {  // g_enc[c][i]
    const int c = t / N, i = t % N;
    double acc = 0.0;
    for (int64_t j = 0; j < m; ++j) {
      const double rv = refl[j * N + i], lv = illum[j * N + i];
      if (lw.code != 0.0) acc -= pb.gc[j * K + c] * (rv * lv);
      const double gr = pb.gzr[j * K + c], gl = pb.gzl[j * K + c];
      if (gr == 0.0 && gl == 0.0) continue;
      acc += gr * rv + gl * lv;
    }
    g_enc[t] = acc * sd_enc[t];
    return;
  }
  const int u = t - K * N;
  if (u >= N * K) return;
  const int i = u / K, c = u % K;  // g_dec[i][c]
  double acc = 0.0;
  for (int64_t j = 0; j < m; ++j) {
    const double gs = pb.gshat[j * N + i];
    if (gs != 0.0) acc += gs * pb.zp[j * K + c];
    if (lw.rec != 0.0) acc += pb.grr[j * N + i] * pb.zr[j * K + c] + pb.grl[j * N + i] * pb.zl[j * K + c];
  }
  if (lw.alg != 0.0) {  // trainer.cpp:336-355
    const double off_terms = K > 1 ? static_cast<double>(K) * (K - 1) : 1.0;
    const double* w = D + i * K;
    double gg = 0.0;
    for (int q = 0; q < K; ++q) {
      if (q == c) continue;
      gg += 4.0 * w[c] * w[q] * w[q] / off_terms;
    }
    const double bi = w[c];
    gg += 2.0 * (bi * bi - bi) * (2.0 * bi - 1.0) / K;
    acc += lw.alg * gg;
  }
  g_dec[u] = acc * sd_dec[u];
}

// Batch means in batch order, loss_alg (trainer.cpp:174-201), the weighted total.
template <int K, int N>
__global__ void loss_reduce_kernel(const double* __restrict__ D, int64_t m, LossW lw, const double* __restrict__ terms,
                                   double* __restrict__ out) {
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  for (int64_t j = 0; j < m; ++j)
    for (int q = 0; q < 4; ++q) acc[q] += terms[j * 4 + q];
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
  const double e2e = acc[0] / md, rec = acc[1] / md, code = acc[2] / md, col = acc[3] / md;
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
  // scratch: weights | per-pair buffers | gradients | losses
  const size_t wbytes = sizeof(double) * host.size();
  const size_t per_pair = static_cast<size_t>(3 * n + 6 * k + 4);
  const size_t pbytes = sizeof(double) * per_pair * static_cast<size_t>(m);
  const size_t gbytes = sizeof(double) * 2 * kn;
  int rc = ensure_scratch(ctx, wbytes + pbytes + gbytes + sizeof(double) * 8);
  if (rc != HC_OK) return rc;
  double* base = static_cast<double*>(ctx->scratch);
  double* dW = base;
  PairBufs pb;
  double* q = base + host.size();
  pb.gshat = q;
  q += static_cast<size_t>(m) * n;
  pb.grr = q;
  q += static_cast<size_t>(m) * n;
  pb.grl = q;
  q += static_cast<size_t>(m) * n;
  pb.zp = q;
  q += static_cast<size_t>(m) * k;
  pb.zr = q;
  q += static_cast<size_t>(m) * k;
  pb.zl = q;
  q += static_cast<size_t>(m) * k;
  pb.gc = q;
  q += static_cast<size_t>(m) * k;
  pb.gzr = q;
  q += static_cast<size_t>(m) * k;
  pb.gzl = q;
  q += static_cast<size_t>(m) * k;
  pb.terms = q;
  q += static_cast<size_t>(m) * 4;
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
                                                                                  illum, m, lw, pb);
    HC_CHECK_LAUNCH(ctx, "pair_kernel");
    if (g_raw_enc) {
      grad_reduce_kernel<K, N><<<(2 * K * N + 127) / 128, 128, 0, ctx->stream>>>(dD, refl, illum, m, lw, pb, dsde,
                                                                                 dsdd, dg, dg + kn);
      HC_CHECK_LAUNCH(ctx, "grad_reduce_kernel");
    }
    if (losses) {
      loss_reduce_kernel<K, N><<<1, 1, 0, ctx->stream>>>(dD, m, lw, pb.terms, dloss);
      HC_CHECK_LAUNCH(ctx, "loss_reduce_kernel");
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
