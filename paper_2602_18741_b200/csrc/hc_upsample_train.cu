// hadacodec-b200: the reference upsampler's training objective and its gradients
// (upsampler.cpp:207-369, upsample_loss / upsample_gradients) and the
// AdamW update (:378-391), on the GPU.
//
//   L = MSE(z, z_gt) + lambda_maxabs * E[max_i |z_i - z_gt_i|]
//       + lambda_color * E[DeltaE76(Lab(decode(z)), Lab(decode(z_gt)))]
//
// sample_kernel: one block per sample (one thread per hidden unit): the forward pass, the
// loss terms, dL/dz (MSE, the max-abs subgradient at the first argmax, the colour term
// through Lab / XYZ / decode), and the backward vectors; grad_sum_kernel: one thread per
// weight, the samples' outer products summed in sample order, as the reference does.  All
// sums run in the reference's order with -fmad=false; SiLU's exp and Lab's cbrt are CUDA's
// (within an ulp or two of glibc's), so the values agree with the reference to ~1e-12
// relative rather than bit for bit.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <vector>

#include "hadacodec_b200.h"
#include "hc_internal.h"

namespace hcb {
namespace {

constexpr int kMaxH = 512;
constexpr int kMaxK = 32;
constexpr int kMaxN = 81;
constexpr double kLabDelta = 6.0 / 29.0;  // upsampler.cpp:90-91
constexpr double kLabDelta3 = kLabDelta * kLabDelta * kLabDelta;

struct UpW {                 // device weights
  const double *w1, *b1;     // h x 3, h
  const double *w2, *w2t;    // h x h (row-major), its transpose
  const double *b2;          // h
  const double *w3, *b3;     // k x h, k
  const double *dec;         // codec decoder, n x k
  const double *wxyz;        // 3 x n: CmfTable wx / wy / wz
};

struct SampleBufs {          // per sample b (row b of each)
  double *h1, *h2, *gh2, *gi1;  // B x h
  double *z, *gz;               // B x k
  double *terms;                // B x 3: mse / k * inv_b, maxabs * inv_b, sqrt(de2) * inv_b
};

__device__ inline double silu(double x) { return x * (1.0 / (1.0 + exp(-x))); }
__device__ inline double silu_derivative(double x) {  // upsampler.cpp:21-24
  const double s = 1.0 / (1.0 + exp(-x));
  return s * (1.0 + x * (1.0 - s));
}
__device__ inline double lab_f(double t) {  // :93-96
  return t > kLabDelta3 ? cbrt(t) : t / (3.0 * kLabDelta * kLabDelta) + 4.0 / 29.0;
}
__device__ inline double lab_f_derivative(double t) {  // :98-101
  return t > kLabDelta3 ? 1.0 / (3.0 * cbrt(t * t)) : 1.0 / (3.0 * kLabDelta * kLabDelta);
}

// lab_of_spectrum (upsampler.cpp:108-126) of decode_unchecked(codec, z) (:77-86)
__device__ void lab_of_code(const UpW& W, int n, int k, const double* z, const double* white, double lab[3],
                            double fprime[3]) {
  double xyz[3] = {0.0, 0.0, 0.0};
  for (int i = 0; i < n; ++i) {
    double s = 0.0;
    for (int j = 0; j < k; ++j) s += W.dec[i * k + j] * z[j];
    xyz[0] += W.wxyz[0 * n + i] * s;
    xyz[1] += W.wxyz[1 * n + i] * s;
    xyz[2] += W.wxyz[2 * n + i] * s;
  }
  double f[3];
  for (int c = 0; c < 3; ++c) {
    const double ratio = xyz[c] / white[c];
    f[c] = lab_f(ratio);
    fprime[c] = lab_f_derivative(ratio) / white[c];
  }
  lab[0] = 116.0 * f[1] - 16.0;
  lab[1] = 500.0 * (f[0] - f[1]);
  lab[2] = 200.0 * (f[1] - f[2]);
}

__global__ void sample_kernel(UpW W, int h, int k, int n, const double* __restrict__ rgb,
                              const double* __restrict__ target, int64_t B, double lambda_maxabs, double lambda_color,
                              double wx, double wy, double wz, SampleBufs sb) {
  __shared__ double h1[kMaxH], h1pre[kMaxH], h2[kMaxH], gh2[kMaxH];
  __shared__ double z[kMaxK], gz[kMaxK];
  const int64_t b = blockIdx.x;
  const int t = threadIdx.x;
  const double inv_b = 1.0 / static_cast<double>(B);
  const double r = rgb[b * 3 + 0], g = rgb[b * 3 + 1], bl = rgb[b * 3 + 2];
  // forward (upsampler.cpp:42-72)
  double h2pre_t = 0.0;
  for (int i = t; i < h; i += blockDim.x) {
    double acc = W.b1[i];
    acc += W.w1[i * 3 + 0] * r;
    acc += W.w1[i * 3 + 1] * g;
    acc += W.w1[i * 3 + 2] * bl;
    h1pre[i] = acc;
    h1[i] = silu(acc);
  }
  __syncthreads();
  for (int i = t; i < h; i += blockDim.x) {
    double acc = W.b2[i];
    for (int j = 0; j < h; ++j) acc += W.w2t[j * h + i] * h1[j];
    h2[i] = silu(acc);
    if (i == t) h2pre_t = acc;
  }
  __syncthreads();
  if (t < k) {
    double acc = W.b3[t];
    for (int j = 0; j < h; ++j) acc += W.w3[t * h + j] * h2[j];
    z[t] = acc;
  }
  __syncthreads();
  // dL/dz and the loss terms (upsample_loss :216-238, upsample_gradients :263-317)
  if (t == 0) {
    const double* tg = target + b * k;
    double mse = 0.0, maxabs = 0.0, best = -1.0;
    int arg = 0;
    for (int i = 0; i < k; ++i) {
      const double d = z[i] - tg[i];
      mse += d * d;
      maxabs = maxabs < fabs(d) ? fabs(d) : maxabs;  // std::max
      gz[i] = 2.0 * d / k * inv_b;
      if (fabs(d) > best) {
        best = fabs(d);
        arg = i;
      }
    }
    if (best > 0.0) {
      const double d = z[arg] - tg[arg];
      gz[arg] += lambda_maxabs * (d > 0.0 ? 1.0 : -1.0) * inv_b;
    }
    const double white[3] = {wx, wy, wz};
    double lp[3], fp[3], lr[3], fr[3];
    lab_of_code(W, n, k, z, white, lp, fp);
    double tgl[kMaxK];
    for (int i = 0; i < k; ++i) tgl[i] = tg[i];
    lab_of_code(W, n, k, tgl, white, lr, fr);
    double diff[3], de2 = 0.0;
    for (int c = 0; c < 3; ++c) {
      diff[c] = lp[c] - lr[c];
      de2 += diff[c] * diff[c];
    }
    const double de = sqrt(de2);
    sb.terms[b * 3 + 0] = mse / k * inv_b;
    sb.terms[b * 3 + 1] = maxabs * inv_b;
    sb.terms[b * 3 + 2] = de * inv_b;
    if (lambda_color != 0.0 && de > 1e-12) {
      const double gl[3] = {diff[0] / de, diff[1] / de, diff[2] / de};
      const double gf[3] = {500.0 * gl[1], 116.0 * gl[0] - 500.0 * gl[1] + 200.0 * gl[2], -200.0 * gl[2]};
      const double gx[3] = {gf[0] * fp[0], gf[1] * fp[1], gf[2] * fp[2]};
      const double scale = lambda_color * inv_b;
      for (int j = 0; j < k; ++j) {
        double acc = 0.0;
        for (int i = 0; i < n; ++i) {
          const double gs = gx[0] * W.wxyz[0 * n + i] + gx[1] * W.wxyz[1 * n + i] + gx[2] * W.wxyz[2 * n + i];
          acc += gs * W.dec[i * k + j];
        }
        gz[j] += scale * acc;
      }
    }
    for (int i = 0; i < k; ++i) {
      sb.z[b * k + i] = z[i];
      sb.gz[b * k + i] = gz[i];
    }
  }
  __syncthreads();
  // backprop (:320-367): g_h2 = W3^T gz (over i in order) * silu'(h2_pre)
  for (int j = t; j < h; j += blockDim.x) {
    double acc = 0.0;
    for (int i = 0; i < k; ++i) acc += gz[i] * W.w3[i * h + j];
    double pre;
    if (j == t) {
      pre = h2pre_t;
    } else {  // blockDim < h: recompute the pre-activation
      pre = W.b2[j];
      for (int q = 0; q < h; ++q) pre += W.w2t[q * h + j] * h1[q];
    }
    gh2[j] = acc * silu_derivative(pre);
  }
  __syncthreads();
  // g_h1 = W2^T g_h2 (over i in order) * silu'(h1_pre)
  for (int j = t; j < h; j += blockDim.x) {
    double acc = 0.0;
    for (int i = 0; i < h; ++i) acc += gh2[i] * W.w2[i * h + j];
    sb.gi1[b * h + j] = acc * silu_derivative(h1pre[j]);
    sb.h1[b * h + j] = h1[j];
    sb.h2[b * h + j] = h2[j];
    sb.gh2[b * h + j] = gh2[j];
  }
}

// One thread per weight entry (w1 | b1 | w2 | b2 | w3 | b3), samples in order.
__global__ void grad_sum_kernel(int h, int k, const double* __restrict__ rgb, int64_t B, SampleBufs sb,
                                double* __restrict__ g) {
  const int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  const int64_t n1 = int64_t(h) * 3, n2 = n1 + h, n3 = n2 + int64_t(h) * h, n4 = n3 + h, n5 = n4 + int64_t(k) * h,
                n6 = n5 + k;
  if (e >= n6) return;
  double acc = 0.0;
  if (e < n1) {
    const int i = static_cast<int>(e / 3), c = static_cast<int>(e % 3);
    for (int64_t b = 0; b < B; ++b) acc += sb.gi1[b * h + i] * rgb[b * 3 + c];
  } else if (e < n2) {
    const int i = static_cast<int>(e - n1);
    for (int64_t b = 0; b < B; ++b) acc += sb.gi1[b * h + i];
  } else if (e < n3) {
    const int i = static_cast<int>((e - n2) / h), j = static_cast<int>((e - n2) % h);
    for (int64_t b = 0; b < B; ++b) acc += sb.gh2[b * h + i] * sb.h1[b * h + j];
  } else if (e < n4) {
    const int i = static_cast<int>(e - n3);
    for (int64_t b = 0; b < B; ++b) acc += sb.gh2[b * h + i];
  } else if (e < n5) {
    const int i = static_cast<int>((e - n4) / h), j = static_cast<int>((e - n4) % h);
    for (int64_t b = 0; b < B; ++b) acc += sb.gz[b * k + i] * sb.h2[b * h + j];
  } else {
    const int i = static_cast<int>(e - n5);
    for (int64_t b = 0; b < B; ++b) acc += sb.gz[b * k + i];
  }
  g[e] = acc;
}

__global__ void loss_sum_kernel(const double* __restrict__ terms, int64_t B, double lambda_maxabs,
                                double lambda_color, double* __restrict__ out) {
  double a = 0.0, m = 0.0, c = 0.0;
  for (int64_t b = 0; b < B; ++b) {
    a += terms[b * 3 + 0];
    m += terms[b * 3 + 1];
    c += terms[b * 3 + 2];
  }
  out[0] = a;
  out[1] = m;
  out[2] = c;
  out[3] = a + lambda_maxabs * m + lambda_color * c;  // :239-240
}

// adamw_step (upsampler.cpp:378-391); bc1, bc2 = 1 - beta^t from the host's pow.
__global__ void adamw_kernel(double* __restrict__ p, const double* __restrict__ g, double* __restrict__ m1,
                             double* __restrict__ v1, int64_t count, double lr, double wd, double bc1, double bc2) {
  constexpr double b1 = 0.9, b2 = 0.999, eps = 1e-8;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < count; i += int64_t(gridDim.x) * blockDim.x) {
    m1[i] = b1 * m1[i] + (1.0 - b1) * g[i];
    v1[i] = b2 * v1[i] + (1.0 - b2) * g[i] * g[i];
    const double mhat = m1[i] / bc1;
    const double vhat = v1[i] / bc2;
    p[i] -= lr * (mhat / (sqrt(vhat) + eps) + wd * p[i]);
  }
}

}  // namespace
}  // namespace hcb

using namespace hcb;

extern "C" {

int hc_upsample_train_grad(hc_ctx ctx, int k, int hidden, const double* w1, const double* b1, const double* w2,
                           const double* b2, const double* w3, const double* b3, int n, const double* codec_dec,
                           const double* wxyz, const double* white, const double* rgb, const double* target, int64_t B,
                           double lambda_maxabs, double lambda_color, double* losses, double* grads) {
  HC_REQUIRE(ctx && w1 && b1 && w2 && b2 && w3 && b3 && codec_dec && wxyz && white, HC_EINVAL,
             "upsampler training: null argument");
  HC_REQUIRE(B > 0 && rgb && target, HC_EINVAL, "upsampler: loss needs a non-empty batch");
  HC_REQUIRE(k > 0 && k <= kMaxK && hidden > 0 && hidden <= kMaxH && n > 0 && n <= kMaxN, HC_EUNSUPPORTED,
             "upsampler training: k <= 32, hidden <= 512, n <= 81");
  const size_t h = static_cast<size_t>(hidden), kk = static_cast<size_t>(k), nn = static_cast<size_t>(n);
  // device weights: w1 | b1 | w2 | w2^T | b2 | w3 | b3 | dec | wxyz
  std::vector<double> host;
  host.insert(host.end(), w1, w1 + h * 3);
  host.insert(host.end(), b1, b1 + h);
  host.insert(host.end(), w2, w2 + h * h);
  for (size_t j = 0; j < h; ++j)
    for (size_t i = 0; i < h; ++i) host.push_back(w2[i * h + j]);
  host.insert(host.end(), b2, b2 + h);
  host.insert(host.end(), w3, w3 + kk * h);
  host.insert(host.end(), b3, b3 + kk);
  host.insert(host.end(), codec_dec, codec_dec + nn * kk);
  host.insert(host.end(), wxyz, wxyz + 3 * nn);
  const size_t ng = h * 3 + h + h * h + h + kk * h + kk;
  const size_t per_sample = 4 * h + 2 * kk + 3;
  const size_t total = host.size() + per_sample * static_cast<size_t>(B) + ng + 8;
  int rc = ensure_scratch(ctx, sizeof(double) * total);
  if (rc != HC_OK) return rc;
  double* base = static_cast<double*>(ctx->scratch);
  HC_CUDA_TRY(cudaMemcpyAsync(base, host.data(), sizeof(double) * host.size(), cudaMemcpyHostToDevice, ctx->stream));
  UpW W;
  const double* q = base;
  W.w1 = q;
  q += h * 3;
  W.b1 = q;
  q += h;
  W.w2 = q;
  q += h * h;
  W.w2t = q;
  q += h * h;
  W.b2 = q;
  q += h;
  W.w3 = q;
  q += kk * h;
  W.b3 = q;
  q += kk;
  W.dec = q;
  q += nn * kk;
  W.wxyz = q;
  double* p = base + host.size();
  SampleBufs sb;
  const size_t Bs = static_cast<size_t>(B);
  sb.h1 = p;
  p += Bs * h;
  sb.h2 = p;
  p += Bs * h;
  sb.gh2 = p;
  p += Bs * h;
  sb.gi1 = p;
  p += Bs * h;
  sb.z = p;
  p += Bs * kk;
  sb.gz = p;
  p += Bs * kk;
  sb.terms = p;
  p += Bs * 3;
  double* dg = p;
  double* dl = dg + ng;
  const int threads = std::min(512, std::max(32, (hidden + 31) / 32 * 32));
  sample_kernel<<<static_cast<unsigned>(B), threads, 0, ctx->stream>>>(W, hidden, k, n, rgb, target, B, lambda_maxabs,
                                                                       lambda_color, white[0], white[1], white[2], sb);
  HC_CHECK_LAUNCH(ctx, "sample_kernel");
  if (grads) {
    grad_sum_kernel<<<static_cast<unsigned>((ng + 127) / 128), 128, 0, ctx->stream>>>(hidden, k, rgb, B, sb, dg);
    HC_CHECK_LAUNCH(ctx, "grad_sum_kernel");
    HC_CUDA_TRY(cudaMemcpyAsync(grads, dg, sizeof(double) * ng, cudaMemcpyDeviceToHost, ctx->stream));
  }
  if (losses) {
    loss_sum_kernel<<<1, 1, 0, ctx->stream>>>(sb.terms, B, lambda_maxabs, lambda_color, dl);
    HC_CHECK_LAUNCH(ctx, "loss_sum_kernel");
    HC_CUDA_TRY(cudaMemcpyAsync(losses, dl, sizeof(double) * 4, cudaMemcpyDeviceToHost, ctx->stream));
  }
  HC_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  return HC_OK;
}

int hc_adamw_step(hc_ctx ctx, double* params, const double* grad, double* m1, double* v1, int64_t count, double lr,
                  double weight_decay, int64_t step) {
  HC_REQUIRE(ctx, HC_EINVAL, "adamw: null context");
  HC_REQUIRE(count >= 0 && step >= 1, HC_EINVAL, "adamw: bad count / step");
  if (count == 0) return HC_OK;
  HC_REQUIRE(params && grad && m1 && v1, HC_EINVAL, "adamw: null buffer");
  const double bc1 = 1.0 - std::pow(0.9, static_cast<double>(step));
  const double bc2 = 1.0 - std::pow(0.999, static_cast<double>(step));
  const int g = static_cast<int>(std::min<int64_t>((count + 255) / 256, int64_t(ctx->sm_count) * 8));
  adamw_kernel<<<g, 256, 0, ctx->stream>>>(params, grad, m1, v1, count, lr, weight_decay, bc1, bc2);
  HC_CHECK_LAUNCH(ctx, "adamw_kernel");
  return HC_OK;
}

}  // extern "C"
