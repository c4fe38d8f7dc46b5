// hadacodec-b200: RGB -> code upsampler MLP (config 5a) — placeholder until the
// tcgen05 kernel lands.
#include "hc_internal.h"

struct hc_mlp_s {
  hc_ctx ctx;
};

extern "C" {
int hc_mlp_create(hc_ctx, int, int, const float*, const float*, const float*, const float*, const float*,
                  const float*, hc_mlp* out) {
  if (out) *out = nullptr;
  return hcb::set_error(HC_EUNSUPPORTED, "mlp: not built yet");
}
int hc_mlp_destroy(hc_mlp m) {
  delete m;
  return HC_OK;
}
int hc_mlp_forward(hc_mlp, const float*, int64_t, float*) {
  return hcb::set_error(HC_EUNSUPPORTED, "mlp: not built yet");
}
}
