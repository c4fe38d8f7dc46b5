// hadacodec-b200: one process driving several GPUs.
//
// The reference's only parallelism is a row-scheduled std::thread pool over one image
// (renderer.cpp:573-608, sized by HADACODEC_THREADS :615-621).  Here an image is cut into
// contiguous row bands, one per GPU (hc_row_band: sizes differ by at most one row), and
// each device is driven by its own persistent host thread with its own context, stream and
// codec.  Every pixel is independent, so nothing crosses a GPU boundary until the outputs
// are assembled; three ways of doing that:
//   HC_GATHER_HOST  each device copies its band of XYZ / sRGB straight into the caller's
//                   host image (every GPU uses its own PCIe link; no inter-GPU traffic);
//   HC_GATHER_NCCL  the bands are gathered into a full-frame buffer on the first device by
//                   one grouped ncclSend / ncclRecv per band over NVLink (NCCL has no Gather;
//                   communicators from ncclCommInitAll), then copied to the host once;
//   HC_GATHER_PEER  the same gather with cudaMemcpyPeerAsync (no NCCL; also valid when a
//                   device appears twice, which the single-GPU tests use);
//   HC_GATHER_FUSED no gather step at all: every device's shade kernel stores its band of
//                   XYZ / sRGB straight into the first device's full-frame buffer through
//                   NVLink peer memory (the kernel's bulk-copy stores take a peer address),
//                   so the transfer rides under the band's compute tile by tile; one D2H
//                   copy of the assembled frame follows.  Needs peer access from every
//                   device to the first (HC_EUNSUPPORTED otherwise).
// NCCL is loaded at run time (dlopen "libnccl.so.2": the copy PyTorch already loaded, else
// the system one); HC_GATHER_NCCL fails with HC_EUNSUPPORTED when it is absent or the
// devices are not distinct.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <condition_variable>
#include <cstring>
#include <memory>
#include <functional>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "hadacodec_b200.h"
#include "hc_internal.h"

using namespace hcb;

namespace {

// ------------------------------------------------------------------ NCCL (run-time loaded)
struct Nccl {
  bool ok = false;
  std::string why;
  ncclResult_t (*CommInitAll)(ncclComm_t*, int, const int*) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  ncclResult_t (*GetVersion)(int*) = nullptr;
};

const Nccl& nccl() {
  static Nccl n = [] {
    Nccl r;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      r.why = std::string("libnccl.so.2 not loadable: ") + dlerror();
      return r;
    }
    auto sym = [&](const char* name) { return dlsym(h, name); };
    r.CommInitAll = reinterpret_cast<decltype(r.CommInitAll)>(sym("ncclCommInitAll"));
    r.CommDestroy = reinterpret_cast<decltype(r.CommDestroy)>(sym("ncclCommDestroy"));
    r.GroupStart = reinterpret_cast<decltype(r.GroupStart)>(sym("ncclGroupStart"));
    r.GroupEnd = reinterpret_cast<decltype(r.GroupEnd)>(sym("ncclGroupEnd"));
    r.Send = reinterpret_cast<decltype(r.Send)>(sym("ncclSend"));
    r.Recv = reinterpret_cast<decltype(r.Recv)>(sym("ncclRecv"));
    r.GetErrorString = reinterpret_cast<decltype(r.GetErrorString)>(sym("ncclGetErrorString"));
    r.GetVersion = reinterpret_cast<decltype(r.GetVersion)>(sym("ncclGetVersion"));
    r.ok = r.CommInitAll && r.CommDestroy && r.GroupStart && r.GroupEnd && r.Send && r.Recv && r.GetErrorString;
    if (!r.ok) r.why = "libnccl.so.2 lacks a required symbol";
    return r;
  }();
  return n;
}

int nccl_error(ncclResult_t e, const char* where) {
  return set_error(HC_ECUDA, std::string(where) + ": " + nccl().GetErrorString(e));
}

// ------------------------------------------------------------------ persistent per-device workers
class Workers {
 public:
  explicit Workers(int n) : jobs_(n), rc_(n, HC_OK) {
    for (int i = 0; i < n; ++i) threads_.emplace_back([this, i] { loop(i); });
  }
  ~Workers() {
    {
      std::lock_guard<std::mutex> g(m_);
      stop_ = true;
      ++gen_;
    }
    cv_.notify_all();
    for (auto& t : threads_) t.join();
  }
  // Run job(i) on worker i for every i in `which` (all when empty); returns the first error.
  int run(const std::function<int(int)>& job, const std::vector<int>& which = {}) {
    std::unique_lock<std::mutex> g(m_);
    pending_ = 0;
    for (size_t i = 0; i < jobs_.size(); ++i) {
      const bool on = which.empty() || std::find(which.begin(), which.end(), static_cast<int>(i)) != which.end();
      jobs_[i] = on ? job : nullptr;
      rc_[i] = HC_OK;
      pending_ += on;
    }
    ++gen_;
    cv_.notify_all();
    done_.wait(g, [this] { return pending_ == 0; });
    for (int r : rc_)
      if (r != HC_OK) return r;
    return HC_OK;
  }

 private:
  void loop(int i) {
    uint64_t seen = 0;
    for (;;) {
      std::function<int(int)> job;
      {
        std::unique_lock<std::mutex> g(m_);
        cv_.wait(g, [&] { return gen_ != seen; });
        seen = gen_;
        if (stop_) return;
        job = jobs_[i];
      }
      if (!job) continue;
      const int r = job(i);
      std::lock_guard<std::mutex> g(m_);
      rc_[i] = r;
      if (--pending_ == 0) done_.notify_all();
    }
  }
  std::vector<std::thread> threads_;
  std::vector<std::function<int(int)>> jobs_;
  std::vector<int> rc_;
  std::mutex m_;
  std::condition_variable cv_, done_;
  uint64_t gen_ = 0;
  int pending_ = 0;
  bool stop_ = false;
};

}  // namespace

struct hc_group_s {
  int ndev = 0;
  int gather = HC_GATHER_HOST;
  std::vector<int> devices;
  std::vector<cudaStream_t> streams;
  std::vector<hc_ctx> ctx;
  std::vector<hc_codec> codec;
  std::vector<ncclComm_t> comms;
  std::unique_ptr<Workers> workers;
  // per device: band inputs / outputs (grow-only); device 0 also holds the full frame
  std::vector<void*> buf;
  std::vector<size_t> buf_bytes;
};

namespace {

int ensure_buf(hc_group g, int d, size_t bytes) {
  if (g->buf_bytes[d] >= bytes) return HC_OK;
  cudaSetDevice(g->devices[d]);
  if (g->buf[d]) cudaFree(g->buf[d]);
  g->buf[d] = nullptr;
  g->buf_bytes[d] = 0;
  HC_CUDA_TRY(cudaMalloc(&g->buf[d], bytes));
  g->buf_bytes[d] = bytes;
  return HC_OK;
}

}  // namespace

extern "C" {

int hc_row_band(int rank, int world, int64_t height, int64_t* row0, int64_t* rows) {
  HC_REQUIRE(world >= 1 && rank >= 0 && rank < world && height >= 0 && row0 && rows, HC_EINVAL,
             "row_band: bad rank / size");
  const int64_t base = height / world, extra = height % world;
  *row0 = rank * base + (rank < extra ? rank : extra);
  *rows = base + (rank < extra ? 1 : 0);
  return HC_OK;
}

int hc_group_create(const int* devices, int ndev, int gather, hc_group* out) {
  HC_REQUIRE(devices && ndev >= 1 && out, HC_EINVAL, "group: bad device list");
  HC_REQUIRE(gather == HC_GATHER_HOST || gather == HC_GATHER_NCCL || gather == HC_GATHER_PEER ||
                 gather == HC_GATHER_FUSED,
             HC_EINVAL, "group: unknown gather mode");
  if (gather == HC_GATHER_NCCL) {
    if (!nccl().ok) return set_error(HC_EUNSUPPORTED, "group: " + nccl().why);
    for (int i = 0; i < ndev; ++i)
      for (int j = 0; j < i; ++j)
        if (devices[i] == devices[j])
          return set_error(HC_EUNSUPPORTED, "group: NCCL needs distinct devices (use HC_GATHER_PEER)");
  }
  auto g = std::make_unique<hc_group_s>();
  g->ndev = ndev;
  g->gather = gather;
  g->devices.assign(devices, devices + ndev);
  g->streams.assign(ndev, nullptr);
  g->ctx.assign(ndev, nullptr);
  g->codec.assign(ndev, nullptr);
  g->buf.assign(ndev, nullptr);
  g->buf_bytes.assign(ndev, 0);
  for (int d = 0; d < ndev; ++d) {
    HC_CUDA_TRY(cudaSetDevice(devices[d]));
    HC_CUDA_TRY(cudaStreamCreateWithFlags(&g->streams[d], cudaStreamNonBlocking));
    const int rc = hc_ctx_create(devices[d], g->streams[d], &g->ctx[d]);
    if (rc != HC_OK) {
      hc_group_destroy(g.release());
      return rc;
    }
  }
  if (gather == HC_GATHER_PEER) {  // peer access where the hardware offers it (copies work either way)
    for (int d = 1; d < ndev; ++d)
      if (devices[d] != devices[0]) {
        int can = 0;
        cudaDeviceCanAccessPeer(&can, devices[0], devices[d]);
        if (can) {
          cudaSetDevice(devices[0]);
          cudaDeviceEnablePeerAccess(devices[d], 0);
          cudaGetLastError();  // already enabled is fine
        }
      }
  }
  if (gather == HC_GATHER_FUSED) {  // every device's kernels store into the first device's memory
    for (int d = 1; d < ndev; ++d)
      if (devices[d] != devices[0]) {
        int can = 0;
        cudaDeviceCanAccessPeer(&can, devices[d], devices[0]);
        if (!can) {
          hc_group_destroy(g.release());
          return set_error(HC_EUNSUPPORTED, "group: HC_GATHER_FUSED needs peer access to the first device");
        }
        cudaSetDevice(devices[d]);
        const cudaError_t e = cudaDeviceEnablePeerAccess(devices[0], 0);
        cudaGetLastError();
        if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) {
          hc_group_destroy(g.release());
          return cuda_error(e, "cudaDeviceEnablePeerAccess");
        }
      }
  }
  if (gather == HC_GATHER_NCCL) {
    g->comms.assign(ndev, nullptr);
    const ncclResult_t e = nccl().CommInitAll(g->comms.data(), ndev, devices);
    if (e != ncclSuccess) {
      g->comms.clear();
      const int rc = nccl_error(e, "ncclCommInitAll");
      hc_group_destroy(g.release());
      return rc;
    }
  }
  g->workers = std::make_unique<Workers>(ndev);
  *out = g.release();
  return HC_OK;
}

int hc_group_destroy(hc_group g) {
  if (!g) return HC_OK;
  g->workers.reset();
  for (auto c : g->comms)
    if (c) nccl().CommDestroy(c);
  for (int d = 0; d < g->ndev; ++d) {
    if (g->codec[d]) hc_codec_destroy(g->codec[d]);
    if (g->ctx[d]) hc_ctx_destroy(g->ctx[d]);
    cudaSetDevice(g->devices[d]);
    if (g->buf[d]) cudaFree(g->buf[d]);
    if (g->streams[d]) cudaStreamDestroy(g->streams[d]);
  }
  delete g;
  return HC_OK;
}

int hc_group_size(hc_group g) { return g ? g->ndev : 0; }

int hc_group_nccl_version(void) {
  int v = 0;
  if (nccl().ok && nccl().GetVersion) nccl().GetVersion(&v);
  return v;
}

int hc_group_codec_create(hc_group g, int k, int n, const float* E, const float* D, const double* cmf,
                          double dlambda) {
  HC_REQUIRE(g, HC_EINVAL, "group: null handle");
  for (int d = 0; d < g->ndev; ++d) {
    if (g->codec[d]) hc_codec_destroy(g->codec[d]);
    g->codec[d] = nullptr;
    const int rc = hc_codec_create(g->ctx[d], k, n, E, D, cmf, dlambda, &g->codec[d]);
    if (rc != HC_OK) return rc;
  }
  return HC_OK;
}

int hc_group_shade_latent_host(hc_group g, const float* pal_codes, int n_pal, const float* light_codes, int L,
                               const uint32_t* idx, const float* cosv, int64_t width, int64_t height, float* xyz,
                               float* rgb) {
  HC_REQUIRE(g && g->codec[0], HC_EINVAL, "group: no codec (hc_group_codec_create)");
  HC_REQUIRE(width >= 0 && height >= 0, HC_EINVAL, "group: negative image size");
  HC_REQUIRE(pal_codes && light_codes && idx && cosv, HC_EINVAL, "group: null input");
  const int nd = g->ndev;
  const int k = g->codec[0]->k;
  if (g->gather == HC_GATHER_HOST) {
    // every device shades its band and writes it into the host image itself
    return g->workers->run([&](int d) -> int {
      int64_t r0 = 0, nr = 0;
      hc_row_band(d, nd, height, &r0, &nr);
      cudaSetDevice(g->devices[d]);
      const int64_t p0 = r0 * width, P = nr * width;
      return hc_shade_latent_host(g->codec[d], pal_codes, n_pal, light_codes, L, idx + p0, cosv + p0 * L, P,
                                  xyz ? xyz + p0 * 3 : nullptr, rgb ? rgb + p0 * 3 : nullptr);
    });
  }
  // NCCL / PEER: bands shaded into device buffers, gathered into device 0's full frame
  const int64_t Pall = width * height;
  auto up = [](size_t b) { return (b + 255) & ~size_t(255); };
  int64_t max_band = 0;
  for (int d = 0; d < nd; ++d) {
    int64_t r0, nr;
    hc_row_band(d, nd, height, &r0, &nr);
    max_band = nr * width > max_band ? nr * width : max_band;
  }
  const size_t pal_b = up(sizeof(float) * n_pal * k);
  auto in_bytes = [&](int64_t P) { return pal_b + up(sizeof(uint32_t) * P) + up(sizeof(float) * P * L); };
  const bool fused = g->gather == HC_GATHER_FUSED;
  for (int d = 0; d < nd; ++d) {  // device 0: full-frame outputs; others: their band's (none when fused)
    const int64_t outP = d == 0 ? Pall : fused ? 0 : max_band;
    const int rc = ensure_buf(g, d, in_bytes(max_band) + 2 * up(sizeof(float) * outP * 3));
    if (rc != HC_OK) return rc;
  }
  auto layout = [&](int d, float*& d_pal, uint32_t*& d_idx, float*& d_cos, float*& d_xyz, float*& d_rgb) {
    char* b = static_cast<char*>(g->buf[d]);
    const int64_t outP = d == 0 ? Pall : fused ? 0 : max_band;
    d_pal = reinterpret_cast<float*>(b);
    d_idx = reinterpret_cast<uint32_t*>(b + pal_b);
    d_cos = reinterpret_cast<float*>(b + pal_b + up(sizeof(uint32_t) * max_band));
    d_xyz = reinterpret_cast<float*>(b + in_bytes(max_band));
    d_rgb = reinterpret_cast<float*>(b + in_bytes(max_band) + up(sizeof(float) * outP * 3));
  };
  int rc = g->workers->run([&](int d) -> int {
    int64_t r0 = 0, nr = 0;
    hc_row_band(d, nd, height, &r0, &nr);
    const int64_t p0 = r0 * width, P = nr * width;
    cudaSetDevice(g->devices[d]);
    cudaStream_t s = g->streams[d];
    float *d_pal, *d_cos, *d_xyz, *d_rgb;
    uint32_t* d_idx;
    layout(d, d_pal, d_idx, d_cos, d_xyz, d_rgb);
    if (fused && d > 0) {  // this band's slice of the first device's frame (peer memory)
      float *x0, *g0, *unused_p, *unused_c;
      uint32_t* unused_i;
      layout(0, unused_p, unused_i, unused_c, x0, g0);
      d_xyz = x0 + p0 * 3;
      d_rgb = g0 + p0 * 3;
    }
    // device 0 shades straight into its slice of the full frame (its band starts at row 0)
    HC_CUDA_TRY(cudaMemcpyAsync(d_pal, pal_codes, sizeof(float) * n_pal * k, cudaMemcpyHostToDevice, s));
    HC_CUDA_TRY(cudaMemcpyAsync(d_idx, idx + p0, sizeof(uint32_t) * P, cudaMemcpyHostToDevice, s));
    HC_CUDA_TRY(cudaMemcpyAsync(d_cos, cosv + p0 * L, sizeof(float) * P * L, cudaMemcpyHostToDevice, s));
    int r = hc_shade_latent(g->codec[d], d_pal, n_pal, light_codes, L, d_idx, d_cos, P, nullptr, nullptr,
                            xyz ? d_xyz : nullptr, rgb ? d_rgb : nullptr);
    if (r != HC_OK) return r;
    if (g->gather == HC_GATHER_NCCL) {
      // one grouped send / recv per band: rank d > 0 sends, rank 0 receives every band
      float *x0, *g0, *unused_p, *unused_c;
      uint32_t* unused_i;
      layout(0, unused_p, unused_i, unused_c, x0, g0);
      const Nccl& N = nccl();
      N.GroupStart();
      ncclResult_t e = ncclSuccess;
      if (d > 0) {
        if (xyz && e == ncclSuccess) e = N.Send(d_xyz, P * 3, ncclFloat32, 0, g->comms[d], s);
        if (rgb && e == ncclSuccess) e = N.Send(d_rgb, P * 3, ncclFloat32, 0, g->comms[d], s);
      } else {
        for (int q = 1; q < nd && e == ncclSuccess; ++q) {
          int64_t q0, qn;
          hc_row_band(q, nd, height, &q0, &qn);
          if (xyz && e == ncclSuccess) e = N.Recv(x0 + q0 * width * 3, qn * width * 3, ncclFloat32, q, g->comms[0], s);
          if (rgb && e == ncclSuccess) e = N.Recv(g0 + q0 * width * 3, qn * width * 3, ncclFloat32, q, g->comms[0], s);
        }
      }
      const ncclResult_t e2 = N.GroupEnd();
      if (e != ncclSuccess) return nccl_error(e, "ncclSend/ncclRecv");
      if (e2 != ncclSuccess) return nccl_error(e2, "ncclGroupEnd");
    } else if (d > 0 && !fused) {  // PEER
      float *x0, *g0, *unused_p, *unused_c;
      uint32_t* unused_i;
      layout(0, unused_p, unused_i, unused_c, x0, g0);
      if (xyz)
        HC_CUDA_TRY(cudaMemcpyPeerAsync(x0 + p0 * 3, g->devices[0], d_xyz, g->devices[d], sizeof(float) * P * 3, s));
      if (rgb)
        HC_CUDA_TRY(cudaMemcpyPeerAsync(g0 + p0 * 3, g->devices[0], d_rgb, g->devices[d], sizeof(float) * P * 3, s));
    }
    return hc_ctx_synchronize(g->ctx[d]);
  });
  if (rc != HC_OK) return rc;
  // the assembled frame leaves device 0 in one copy per output
  return g->workers->run(
      [&](int) -> int {
        cudaSetDevice(g->devices[0]);
        float *d_pal, *d_cos, *d_xyz, *d_rgb;
        uint32_t* d_idx;
        layout(0, d_pal, d_idx, d_cos, d_xyz, d_rgb);
        if (xyz) HC_CUDA_TRY(cudaMemcpyAsync(xyz, d_xyz, sizeof(float) * Pall * 3, cudaMemcpyDeviceToHost, g->streams[0]));
        if (rgb) HC_CUDA_TRY(cudaMemcpyAsync(rgb, d_rgb, sizeof(float) * Pall * 3, cudaMemcpyDeviceToHost, g->streams[0]));
        HC_CUDA_TRY(cudaStreamSynchronize(g->streams[0]));
        return HC_OK;
      },
      {0});
}

// ------------------------------------------------------------------ CUDA IPC frames
// One process per GPU: the destination rank's frame mapped into every rank, so each rank's
// shade kernel stores its band straight into it (the fused gather of hc_group, across
// processes).
static_assert(sizeof(cudaIpcMemHandle_t) == HC_IPC_HANDLE_BYTES, "CUDA IPC handle size");

int hc_ipc_alloc(int device, int64_t bytes, void** dptr, unsigned char* handle) {
  HC_REQUIRE(dptr && handle && bytes > 0, HC_EINVAL, "ipc_alloc: bad arguments");
  HC_CUDA_TRY(cudaSetDevice(device));
  void* p = nullptr;
  HC_CUDA_TRY(cudaMalloc(&p, static_cast<size_t>(bytes)));
  cudaIpcMemHandle_t h;
  const cudaError_t e = cudaIpcGetMemHandle(&h, p);
  if (e != cudaSuccess) {
    cudaFree(p);
    return cuda_error(e, "cudaIpcGetMemHandle");
  }
  std::memcpy(handle, &h, sizeof(h));
  *dptr = p;
  return HC_OK;
}

int hc_ipc_open(int device, const unsigned char* handle, void** dptr) {
  HC_REQUIRE(dptr && handle, HC_EINVAL, "ipc_open: bad arguments");
  HC_CUDA_TRY(cudaSetDevice(device));  // the device whose kernels will store into the frame
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, sizeof(h));
  void* p = nullptr;
  HC_CUDA_TRY(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
  *dptr = p;
  return HC_OK;
}

int hc_ipc_close(int device, void* dptr) {
  if (!dptr) return HC_OK;
  HC_CUDA_TRY(cudaSetDevice(device));
  HC_CUDA_TRY(cudaIpcCloseMemHandle(dptr));
  return HC_OK;
}

int hc_ipc_free(int device, void* dptr) {
  if (!dptr) return HC_OK;
  HC_CUDA_TRY(cudaSetDevice(device));
  HC_CUDA_TRY(cudaFree(dptr));
  return HC_OK;
}

}  // extern "C"
