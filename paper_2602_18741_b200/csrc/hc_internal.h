// hadacodec-b200: host-side internals shared by the C-ABI translation units.
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <string>
#include <vector>

#include "../../include/hadacodec_b200.h"

struct hc_ctx_s {
  int device = 0;
  cudaStream_t stream = nullptr;
  int sm_count = 148;
  size_t max_smem_optin = 0;
  int* d_err = nullptr;        // latched device-side violations (hcb::kErr*)
  double* d_partials = nullptr;  // loss partial sums
  int partial_capacity = 0;
  void* scratch = nullptr;     // host-entry staging (grow-only)
  size_t scratch_bytes = 0;
#ifndef HC_AUX_STREAMS
#define HC_AUX_STREAMS 3  // measured: 3 streams 1.527 ms, 4: 1.534, 6 / 8: 1.56-1.57 per e2e frame
#endif
  static constexpr int kAux = HC_AUX_STREAMS;
  cudaStream_t aux[kAux] = {};  // host-entry copy/compute pipeline
  cudaEvent_t ev_fork = nullptr;
  std::atomic<int64_t> launches{0};
  int pdl = 1;  // programmatic dependent launch for tile kernels (HC_PDL=0 disables)
};

struct hc_codec_s {
  hc_ctx ctx = nullptr;
  int k = 0, n = 0;
  double dlambda = 0.0;
  std::vector<float> E;       // k x n
  std::vector<float> D;       // n x k
  std::vector<double> Ed;     // k x n effective weights in fp64 (renderer compile_scene)
  std::vector<double> Dd;     // n x k
  std::vector<double> cmf;    // 3 x n (unscaled)
  std::vector<float> Mxyz;    // 3 x k = dlambda * CMF * D (computed in f64)
  std::vector<float> cmf_dl;  // 3 x n = dlambda * CMF
  float Crgb[9];
};

namespace hcb {

int set_error(int code, const std::string& msg);
int cuda_error(cudaError_t e, const char* where);
void note_launch(hc_ctx ctx, int n = 1);
// Grows the context scratch to >= bytes; the first `keep` bytes survive a reallocation.
int ensure_scratch(hc_ctx ctx, size_t bytes, size_t keep = 0);
int ensure_aux_streams(hc_ctx ctx);

// Kernel attributes (cudaFuncSetAttribute: dynamic shared memory, carveout) are per device, so
// one-time configuration is tracked per device (the group API drives several GPUs from one
// process, one host thread each).  `mask` holds one bit per device ordinal (< 64).
inline uint64_t current_device_bit() {
  int dev = 0;
  cudaGetDevice(&dev);
  return 1ull << (dev & 63);
}
inline bool configured_here(const std::atomic<uint64_t>& mask) {
  return (mask.load(std::memory_order_acquire) & current_device_bit()) != 0;
}
inline void mark_configured_here(std::atomic<uint64_t>& mask) {
  mask.fetch_or(current_device_bit(), std::memory_order_release);
}

#define HC_CUDA_TRY(expr)                                        \
  do {                                                           \
    cudaError_t _e = (expr);                                     \
    if (_e != cudaSuccess) return ::hcb::cuda_error(_e, #expr);  \
  } while (0)

#define HC_REQUIRE(cond, code, msg)               \
  do {                                            \
    if (!(cond)) return ::hcb::set_error((code), (msg)); \
  } while (0)

#define HC_CHECK_LAUNCH(ctx, what)                                   \
  do {                                                               \
    cudaError_t _e = cudaGetLastError();                             \
    if (_e != cudaSuccess) return ::hcb::cuda_error(_e, what);       \
    ::hcb::note_launch(ctx);                                         \
  } while (0)

// Family entry points implemented in the kernel translation units.
int codec_launch(hc_codec c, int mode, const float* in, int64_t rows, float* o0, float* o1, float* o2,
                 float* o3, int check_negative);
int shade_latent_launch(hc_codec c, const float* pal, int n_pal, const float* light, int L,
                        const uint32_t* idx, const float* cosv, int64_t P, float* latent,
                        float* spectra, float* xyz, float* rgb);
int shade_spectral_launch(hc_codec c, const float* pal, int n_pal, const float* light, int L,
                          const uint32_t* idx, const float* cosv, int64_t P, float* spectra,
                          float* xyz, float* rgb);
int chain_latent_launch(hc_codec c, const float* pal, int n_pal, const float* ill, int n_ill,
                        const uint8_t* pidx, const uint8_t* iidx, const float* tw, int64_t P, int spp,
                        float* latent, float* xyz, float* rgb);
int chain_spectral_launch(hc_codec c, const float* pal, int n_pal, const float* ill, int n_ill,
                          const uint8_t* pidx, const uint8_t* iidx, const float* tw, int64_t P,
                          int spp, float* xyz, float* rgb);
int loss_launch(hc_codec c, const float* A, const float* B, int64_t pairs, double* sum_dev);

}  // namespace hcb
