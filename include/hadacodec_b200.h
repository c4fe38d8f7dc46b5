/*
 * hadacodec-b200 — C ABI of the B200-native per-pixel codec / latent-shading path.
 *
 * This is the drop-in boundary for the reference's `hadacodec` static library
 * (/root/reference/proj/core, public headers core/include/hadacodec/*.hpp).
 * The reference exposes a by-value C++ API over single spectra / images; this
 * ABI exposes the same operations BATCHED, over device pointers, stream
 * ordered, with plain pointers and sizes only (no C++ or torch types).  The
 * C++ drop-in layer (include/hadacodec_b200.hpp) restores the reference
 * signatures and exception types on top of it.
 *
 * Conventions
 *   - Layouts are row-major, item-major ("HWC" as ChannelImage, renderer.hpp:73-89):
 *       spectra [rows][n] f32, codes [rows][k] f32, xyz / rgb [rows][3] f32,
 *       G-buffer idx [P] u32 + cos [P][L] f32, chain samples pidx [P][spp][4] u8,
 *       iidx [P][spp] u8, tw [P][spp][4] f32.
 *   - Pointers passed to compute entry points are DEVICE pointers of the
 *     context's device unless the name ends in `_host`.  Output pointers may be
 *     NULL to skip that output.
 *   - Every call is enqueued on the context's stream and returns without
 *     synchronising, except `_host` variants, hc_ctx_synchronize and calls
 *     that return a host value.
 *   - Return codes: HC_OK, HC_EINVAL (std::invalid_argument in the reference),
 *     HC_EDOMAIN (std::domain_error: negative code to decode, codec.cpp:56-62),
 *     HC_ECUDA, HC_ENOMEM, HC_EUNSUPPORTED.  hc_last_error() gives a message
 *     (thread-local).  Device-side range / sign violations are latched in the
 *     context and reported by the next hc_ctx_synchronize.
 *   - One context per (device, stream); a context is externally synchronised.
 */
#ifndef HADACODEC_B200_H
#define HADACODEC_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HC_OK 0
#define HC_EINVAL 1
#define HC_EDOMAIN 2
#define HC_ECUDA 3
#define HC_ENOMEM 4
#define HC_EUNSUPPORTED 5

typedef struct hc_ctx_s* hc_ctx;
typedef struct hc_codec_s* hc_codec;
typedef struct hc_mlp_s* hc_mlp;
typedef struct hc_upsampler_s* hc_upsampler;

/* ------------------------------------------------------------------ runtime */
const char* hc_last_error(void);
const char* hc_version(void);
/* Create a context on `device`, enqueuing on `stream` (a cudaStream_t; NULL =
 * legacy default stream). */
int hc_ctx_create(int device, void* stream, hc_ctx* out);
int hc_ctx_destroy(hc_ctx ctx);
int hc_ctx_set_stream(hc_ctx ctx, void* stream);
/* Synchronise the stream; returns HC_EDOMAIN / HC_EINVAL if a kernel latched a
 * negative-code or index-range violation since the last call (then clears it). */
int hc_ctx_synchronize(hc_ctx ctx);
/* Number of kernels this library has launched from `ctx` (monotonic). */
int64_t hc_ctx_launch_count(hc_ctx ctx);

/* ------------------------------------------------------------------ codec
 * Replaces CodecWeights / EffectiveWeights / CmfTable usage
 * (codec.hpp:34-60, colorimetry.hpp:25-47).
 *   E    k x n encoder (effective, non-negative), D  n x k decoder   (host, f32)
 *   cmf  3 x n colour-matching rows (xbar, ybar, zbar) on the grid   (host, f64)
 *   dlambda  grid step in nm (radiance convention, colorimetry.cpp:75-87)
 * Supported (n, k): n in {47, 81}, k in {3, 6, 9}.  k % 3 != 0 -> HC_EINVAL
 * (validate, codec.cpp:111-135). */
int hc_codec_create(hc_ctx ctx, int k, int n, const float* E, const float* D, const double* cmf,
                    double dlambda, hc_codec* out);
/* Same from raw softplus-parameterised weights (raw_enc k x n, raw_dec n x k,
 * beta): effective_weights (codec.cpp:21-34) is applied on the host. */
/* As hc_codec_create with the effective weights in fp64 (EffectiveWeights, codec.hpp:52-58),
 * kept exactly for the fp64 entry points (the fp32 kernels use them rounded to float). */
int hc_codec_create_f64(hc_ctx ctx, int k, int n, const double* E, const double* D, const double* cmf,
                        double dlambda, hc_codec* out);
int hc_codec_create_raw(hc_ctx ctx, int k, int n, double beta, const double* raw_enc,
                        const double* raw_dec, const double* cmf, double dlambda, hc_codec* out);
int hc_codec_destroy(hc_codec codec);
/* The codec's effective weights in fp64 (host copies, k x n and n x k): the doubles it was
 * created with, or softplus_beta(raw) computed as effective_weights does. */
int hc_codec_effective_f64(hc_codec codec, double* E, double* D);
int hc_codec_dims(hc_codec codec, int* k, int* n);
/* Folded 3 x k XYZ projection dlambda * CMF * D (host copy, f32). */
int hc_codec_xyz_projection(hc_codec codec, float* out_3k);

/* encode (codec.cpp:36-46), batched: Z[rows][k] = S[rows][n] . E^T. */
int hc_encode(hc_codec codec, const float* S, int64_t rows, float* Z);
/* decode (codec.cpp:52-71) / decode_image (renderer.cpp:661-690), batched,
 * with the CMF -> XYZ -> linear-sRGB projection of image_to_linear_rgb
 * (renderer.cpp:692-719) folded in.  check_negative != 0 latches HC_EDOMAIN for
 * negative codes (decode's contract); decode_image does not check (0). */
int hc_decode(hc_codec codec, const float* Z, int64_t rows, float* S, float* xyz, float* rgb,
              int check_negative);
/* Fused round trip (config 1): encode -> decode -> XYZ -> sRGB. */
int hc_roundtrip(hc_codec codec, const float* S, int64_t rows, float* Z, float* S2, float* xyz,
                 float* rgb);
/* image_to_linear_rgb (renderer.cpp:692-719) on n-channel spectra, plus XYZ. */
int hc_spectra_to_xyz_rgb(hc_codec codec, const float* S, int64_t rows, float* xyz, float* rgb);
/* blockwise_hadamard (codec.cpp:77-85), batched: out = A (.) B, [rows][k]. */
int hc_blockwise_hadamard(hc_ctx ctx, const float* A, const float* B, int64_t rows, int k,
                          float* out);

/* ------------------------------------------------------------------ shading
 * Latent G-buffer shading (configs 2/3): z_p = zR[idx_p] (.) sum_l cos_{p,l} zL_l
 * — the renderer's NEE channel loop (renderer.cpp:505-510) with the compiled
 * assets of compile_scene (renderer.cpp:161-271) — all k/3 RGB passes fused,
 * written as the reassembled HWC latent image (renderer.cpp:645-657), decoded
 * to spectra and/or projected to XYZ / linear sRGB.
 *   pal_codes  n_pal x k device codes (n_pal <= 256), light_codes L x k (host)
 *   L in {8, 32}: fused TMA kernels; any other 1 <= L <= 64: generic kernel;
 *   L > 64 -> HC_EUNSUPPORTED.  */
int hc_shade_latent(hc_codec codec, const float* pal_codes, int n_pal, const float* light_codes,
                    int L, const uint32_t* idx, const float* cosv, int64_t P, float* latent,
                    float* spectra, float* xyz, float* rgb);
/* One 3-channel render pass b < k/3 (slice_pass, renderer.cpp:274-283):
 * pass_image[P][3] = channels 3b..3b+2 of the latent shade. */
int hc_shade_latent_pass(hc_codec codec, int pass, const float* pal_codes, int n_pal,
                         const float* light_codes, int L, const uint32_t* idx, const float* cosv,
                         int64_t P, float* pass_image);
/* render_latent_multipass reassembly (renderer.cpp:645-657):
 * latent[p][3b+c] = passes[b][p][c] for b < blocks.  `passes` is a HOST array
 * of `blocks` device pointers. */
int hc_reassemble(hc_ctx ctx, const float* const* passes, int blocks, int64_t P, float* latent);
/* Naive n-sample shading (config 2/3 ground truth): S_p = R_idx (.) sum_l cos_l L_l,
 * then XYZ / sRGB (renderer.cpp:187-190 at C = n, :692-719).
 *   pal_spectra n_pal x n device, light_spectra L x n host; L as for hc_shade_latent. */
int hc_shade_spectral(hc_codec codec, const float* pal_spectra, int n_pal,
                      const float* light_spectra, int L, const uint32_t* idx, const float* cosv,
                      int64_t P, float* spectra, float* xyz, float* rgb);

/* Multi-bounce accumulation (config 4; renderer.cpp:457-551, evaluation.cpp:50-76):
 * depth 4, spp a multiple of 8, 1 <= n_pal, n_ill <= 256, pidx 4-byte and tw 16-byte aligned.
 * Latent: codes; spectral: spectra.  Out-of-range palette / illuminant indices are latched
 * and reported as HC_EINVAL by hc_ctx_synchronize.  Performance note (k = 6): spp == 64 with
 * 16-byte aligned pidx and iidx takes the bulk-copy record path (config 4's layout). */
int hc_multibounce_latent(hc_codec codec, const float* pal_codes, int n_pal, const float* ill_codes,
                          int n_ill, const uint8_t* pidx, const uint8_t* iidx, const float* tw,
                          int64_t P, int spp, float* latent, float* xyz, float* rgb);
int hc_multibounce_spectral(hc_codec codec, const float* pal_spectra, int n_pal,
                            const float* ill_spectra, int n_ill, const uint8_t* pidx,
                            const uint8_t* iidx, const float* tw, int64_t P, int spp, float* xyz,
                            float* rgb);

/* ------------------------------------------------------------------ upsampler
 * RGB -> code MLP (upsampler.cpp:42-72, :179-190): 3 -> hidden -> hidden -> k with
 * ReLU, ReLU, softplus(beta = 1) (BASELINE config 5), bf16 tcgen05 GEMMs with
 * fp32 accumulate.  Weights row-major as UpsamplerWeights (upsampler.hpp:17-24):
 * w1 hidden x 3, w2 hidden x hidden, w3 k x hidden (host f32, rounded to bf16),
 * biases host f32.  hidden = 64, k in {3, 6, 9}. */
int hc_mlp_create(hc_ctx ctx, int hidden, int k, const float* w1, const float* b1, const float* w2,
                  const float* b2, const float* w3, const float* b3, hc_mlp* out);
int hc_mlp_destroy(hc_mlp mlp);
int hc_mlp_forward(hc_mlp mlp, const float* rgb, int64_t P, float* codes);

/* ------------------------------------------------------------------ loss
 * Near-multiplicativity residual (trainer.cpp:49-71): sum over pairs and lambda
 * of (D (E a (.) E b) - a (.) b)^2 into *sum_dev (one f64 on the device). */
int hc_hadamard_loss(hc_codec codec, const float* A, const float* B, int64_t pairs, double* sum_dev);

/* ------------------------------------------------------------------ colour-metric tail
 * Consumers of the shading output.  Images are P pixels x
 * `channels` floats on the device, channels = 3 (linear sRGB) or the codec's n
 * (spectra, converted with image_to_linear_rgb in fp64).  Percentiles are exact
 * nearest-rank order statistics (evaluation.cpp:14-21).  Calls returning values
 * through host pointers synchronise the context stream. */

/* exposure_for (renderer.cpp:721-752; renderer.hpp:119, default percentile 99.5):
 * 1 / (percentile of per-pixel luminance), 1 when that is <= 1e-12.  Luminance =
 * Rec.709 luma of linear RGB, or dlambda * ybar . s of spectra. */
int hc_exposure_for(hc_codec codec, const float* img, int64_t P, int channels, double percentile,
                    double* exposure);
/* tonemap_srgb8 (renderer.cpp:754-773): out[3P] = uchar(srgb_encode(clamp(rgb * exposure, 0, 1))
 * * 255 + 0.5).  Asynchronous. */
int hc_tonemap_srgb8(hc_ctx ctx, const float* rgb, int64_t P, double exposure, uint8_t* out);
/* error_map (renderer.cpp:775-802): mse[P] (may be NULL) = mean over channels of the squared
 * linear-RGB difference, *mean_mse (host) = its mean. */
int hc_error_map(hc_codec codec, const float* a, int channels_a, const float* b, int channels_b, int64_t P,
                 float* mse, double* mean_mse);
/* scene_color_report (evaluation.cpp:122-154): out4 (host) = {mean_de76, p95_de76, mse, exposure},
 * Delta E76 in Lab under the sRGB white with the ground truth's exposure applied to both. */
int hc_scene_color_report(hc_codec codec, const float* gt, int channels_gt, const float* test,
                          int channels_test, int64_t P, double* out4);
/* Stream-ordered form (no synchronisation, capturable in a CUDA graph): out4_dev is device
 * memory; test_srgb8 (may be NULL) additionally receives tonemap_srgb8(test, exposure_for(gt))
 * from the same pass, as run_report writes next to the report (tools/main.cpp:604-623). */
int hc_scene_color_report_dev(hc_codec codec, const float* gt, int channels_gt, const float* test,
                              int channels_test, int64_t P, double* out4_dev, uint8_t* test_srgb8);
/* XYZ of rows of n fp64 values (device), fp64 out (device, rows x 3), in the reference's summation
 * order: weights == NULL is the radiance convention spectrum_to_xyz (colorimetry.cpp:75-87: CMF
 * rows, then x dlambda); otherwise `weights` (host, 3 x n) are CmfTable's D65-weighted rows and
 * the result is xyz_of_reflectance (colorimetry.cpp:89-101). */
int hc_spectra_to_xyz_f64(hc_codec codec, const double* S, int64_t rows, const double* weights, double* xyz);
/* Per-pixel Delta E94 of multibounce_eval (evaluation.cpp:59-86): Lab of both XYZ images under
 * white_xyz (host, 3 doubles; CmfTable::white_xyz) scaled to the ground truth's max(Y, 1e-6).
 * out3 (host) = {mean, median, p95}; de[P] (may be NULL) per pixel.  HC_EDOMAIN for a
 * non-positive white (xyz_to_lab, colorimetry.cpp:119-123). */
int hc_delta_e94_report(hc_ctx ctx, const float* xyz_gt, const float* xyz_test, int64_t P,
                        const double* white_xyz, float* de, double* out3);

/* ------------------------------------------------------------------ path tracer
 * The reference's unidirectional path tracer with next-event estimation
 * (renderer.hpp:93-107, renderer.cpp:437-659) on a Cornell-style scene: an axis-
 * aligned box shell with per-wall Lambertian materials, spheres / blocks and
 * parallelogram area lights (renderer.hpp:16-53).  Spectral curves are given on the
 * codec's grid (n samples).  Deterministic and identical to the reference's per-sample
 * streams (Rng::pixel_stream); see DESIGN.md for the parity statement. */
enum { HC_RENDER_SPECTRAL = 0, HC_RENDER_LATENT = 1, HC_RENDER_RGB = 2 };

typedef struct hc_scene_object {  /* SceneObject (renderer.hpp:32-39) */
  int kind;                       /* 0 sphere, 1 block */
  double center[3];
  double radius;
  double box_min[3], box_max[3];
  int material;
} hc_scene_object;

typedef struct hc_scene_light {   /* SceneLight (renderer.hpp:24-30) */
  double corner[3], edge_u[3], edge_v[3];
  const double* spd;              /* n samples, emitted radiance */
  double scale;
} hc_scene_light;

typedef struct hc_scene {         /* Scene + Camera (renderer.hpp:16-53) */
  double cam_position[3], cam_look_at[3], cam_up[3];
  double cam_vfov_degrees;
  double box_min[3], box_max[3];
  int wall_material[6];           /* left, right, floor, ceiling, back, front; -1 = absent */
  int n_materials;
  const double* materials;        /* n_materials x n reflectances in [0, 1] */
  int n_objects;
  const hc_scene_object* objects;
  int n_lights;
  const hc_scene_light* lights;
} hc_scene;

typedef struct hc_render_job {    /* RenderJob (renderer.hpp:57-72) */
  int mode;                       /* HC_RENDER_* */
  int width, height, spp;
  int max_depth;                  /* -1 = unbounded with Russian roulette from depth 5 */
  uint64_t seed;
} hc_render_job;

/* render (renderer.hpp:100-101): image (device, height x width x C floats; C = n spectral,
 * k latent, 3 rgb), path_hashes (device, width x height, may be NULL), *shading_evals (host,
 * may be NULL).  The codec supplies the grid (and the codes in latent mode); rgb mode needs
 * the grid's D65 row `d65` (n doubles, CmfTable).  Synchronous. */
int hc_render(hc_codec codec, const hc_scene* scene, const hc_render_job* job, const double* d65, float* image,
              uint64_t* path_hashes, uint64_t* shading_evals);
/* render_latent_multipass (renderer.hpp:106-107): k/3 three-channel passes, concatenated. */
int hc_render_latent_multipass(hc_codec codec, const hc_scene* scene, const hc_render_job* job, float* image,
                               uint64_t* path_hashes, uint64_t* shading_evals);

/* ------------------------------------------------------------------ formats
 * print_g17 ("%.17g", io.cpp:108-112) on the device: slots (n x 32 bytes, not NUL-
 * terminated) receive the text of v[i], lens[i] its length; bit-identical to glibc's
 * snprintf("%.17g") (exact digits, round half to even). */
int hc_format_g17(hc_ctx ctx, const double* v, int64_t n, char* slots, uint8_t* lens);
/* write_codes_csv (io.cpp:312-330) of device codes [rows][k] (float, printed as the double
 * they widen to) with ids first_id + row: header "id,c0,...\n", rows "id,v0,...\n".  With
 * out == NULL only *length (host) is returned (size query); else out (device, capacity
 * bytes) receives the file.  Synchronous. */
int hc_codes_csv_write(hc_ctx ctx, const float* codes, int64_t rows, int k, uint64_t first_id, char* out,
                       int64_t capacity, int64_t* length);
/* The general write_codes_csv (io.cpp:312-330; the reference's LatentCode values are
 * doubles): codes [rows][k] in device memory as HC_DTYPE_F32 or HC_DTYPE_F64.  Ids:
 * id_bytes (device) with id_spans (device, rows x 2 int64: start, length — the layout
 * hc_codes_csv_read / hc_spectra_csv_read return, so a file's ids pass straight through),
 * written verbatim as `f << ids[r]` does; or, with id_bytes NULL, id_prefix (host string,
 * may be NULL) followed by the decimal first_id + row (run_encode's "row" + r).  rows == 0
 * writes "id\n" (k = 0 for no codes, as the reference does).  Size query as above. */
enum { HC_DTYPE_F32 = 0, HC_DTYPE_F64 = 1 };
int hc_codes_csv_write_ids(hc_ctx ctx, const void* codes, int dtype, int64_t rows, int k, const char* id_bytes,
                           const int64_t* id_spans, const char* id_prefix, uint64_t first_id, char* out,
                           int64_t capacity, int64_t* length);
/* write_spectra_csv (io.cpp:165-186): header ["id,"] + the n wavelengths (host array, the
 * canonical grid) in %.9g, then one row per curve: [id ","] values in %.9g (print_g9,
 * io.cpp:102-106; exact, round half to even, as glibc).  values [rows][n] (device, f32 or
 * f64).  with_ids = 0: no id column (the reference's empty ids); else ids as in
 * hc_codes_csv_write_ids.  Size query with out == NULL. */
int hc_spectra_csv_write(hc_ctx ctx, const void* values, int dtype, int64_t rows, int n, const double* wavelengths,
                         int with_ids, const char* id_bytes, const int64_t* id_spans, const char* id_prefix,
                         uint64_t first_id, char* out, int64_t capacity, int64_t* length);
/* parse_double (io.cpp:78-88: std::stod of a trimmed cell, fully consumed) of n cells held
 * in fixed slots (stride bytes, lens[i] used): out[i] the correctly rounded double,
 * status[i] 0 ok, 1 not a number / trailing junk, 2 out of range (ERANGE: std::stod throws). */
int hc_parse_doubles(hc_ctx ctx, const char* slots, const uint8_t* lens, int64_t n, int stride, double* out,
                     int8_t* status);
/* read_codes_csv (io.cpp:267-310) of a file image on the device (text, len bytes): header
 * "id,c0,...,c{k-1}" on the first non-empty line, one row per non-empty line after it.
 * *k_out, *rows_out (host) always; with codes / ids NULL it is a size query, else codes
 * (device, rows x k doubles) and ids (device, rows x 2 int64: byte offset and length of the
 * trimmed id cell in text) are filled (capacity_rows >= rows).  HC_EINVAL with the 1-based
 * line in hc_last_error() for a bad header, a wrong cell count or a cell std::stod rejects. */
int hc_codes_csv_read(hc_ctx ctx, const char* text, int64_t len, int* k_out, int64_t* rows_out, double* codes,
                      int64_t* ids, int64_t capacity_rows);
/* read_spectra_csv (io.cpp:119-163) of a file image on the device: the first non-empty
 * line is the header — an optional "id" cell (*has_id), then the wavelengths (parsed as
 * the reference does, written to the host array wavelengths, up to wavelength_capacity;
 * *m_out = their count); every later non-empty line has m (+1 with ids) cells.  values
 * (device, rows x m doubles) and ids (device, rows x 2 int64 spans, only with an id
 * column) as in hc_codes_csv_read; both NULL = size query.  HC_EINVAL with the line for
 * a missing / empty / unparsable header, a wrong cell count or a cell std::stod rejects. */
int hc_spectra_csv_read(hc_ctx ctx, const char* text, int64_t len, int* has_id, double* wavelengths,
                        int wavelength_capacity, int* m_out, int64_t* rows_out, double* values, int64_t* ids,
                        int64_t capacity_rows);

/* ------------------------------------------------------------------ fp64 codec of the encode / decode tools
 * run_encode (tools/main.cpp:285-308) per curve: resample(src_wavelengths, row,
 * zero_outside) onto the canonical grid wavelength_at(i) = lambda_min + lambda_step * i
 * (spectrum.cpp:60-98; the codec's n samples), then encode (codec.cpp:36-46) in fp64
 * with the reference's summation order: codes (device, rows x k doubles) bit-identical to
 * the reference.  values: device, rows x m doubles; src_wavelengths: host, m entries,
 * strictly increasing (HC_EINVAL "resample: ..." otherwise, as the reference throws). */
int hc_encode_resampled_f64(hc_codec codec, const double* src_wavelengths, int m, const double* values, int64_t rows,
                            double lambda_min, double lambda_step, int zero_outside, double* codes);
/* run_decode (tools/main.cpp:310-328) per code: decode (codec.cpp:52-71) in fp64, spectra
 * (device, rows x n doubles) bit-identical to the reference.  A code with an entry that is
 * not >= 0 (NaN included) makes the call return HC_EDOMAIN (the reference's domain_error)
 * with *first_negative_row (host, may be NULL) = the first such row; -1 otherwise. */
int hc_decode_f64(hc_codec codec, const double* codes, int64_t rows, double* spectra, int64_t* first_negative_row);
/* encode (codec.cpp:36-46) of curves already on the canonical grid (device, rows x n
 * doubles) in fp64: codes bit-identical to the reference's.  With a codec made by
 * hc_codec_create_f64 / hc_codec_create_raw the weights are the reference's doubles. */
int hc_encode_f64(hc_codec codec, const double* spectra, int64_t rows, double* codes);

/* ------------------------------------------------------------------ codec training step
 * compute_losses + gradients (trainer.cpp:108-373) of CodecWeights {k, n, beta, raw_enc
 * (k x n), raw_dec (n x k)} (host) over a batch of m (reflectance, illumination) pairs
 * (device, m x n doubles each), with LossWeights loss_weights[5] = {e2e, rec, code, col,
 * alg}; cmf = the 3 x n colour-matching rows (CmfTable xbar / ybar / zbar), lambda_step the
 * grid step.  g_raw_enc / g_raw_dec (host, k x n / n x k; both NULL for losses only) and
 * losses[6] = {e2e, rec, code, col, alg, total} (host, may be NULL) are bit-identical to the
 * reference's gradients() / compute_losses(). */
int hc_codec_train_grad(hc_ctx ctx, int k, int n, double beta, const double* raw_enc, const double* raw_dec,
                        const double* cmf, double lambda_step, const double* refl, const double* illum, int64_t m,
                        const double* loss_weights, double* g_raw_enc, double* g_raw_dec, double* losses);
/* adam_step (trainer.cpp:399-411) on device arrays: params -= lr * mhat / (sqrt(vhat) +
 * 1e-8) with the first / second moments m1 / v1 updated in place; step >= 1.  Bit-identical. */
int hc_adam_step(hc_ctx ctx, double* params, const double* grad, double* m1, double* v1, int64_t count, double lr,
                 int64_t step);

/* ------------------------------------------------------------------ the reference's upsampler
 * UpsamplerWeights (upsampler.hpp:13-24): k, hidden (<= 512), w1 (hidden x 3), b1, w2
 * (hidden x hidden), b2, w3 (k x hidden), b3 — fp64, host; validated as validate() does.
 * hc_upsample_f64: upsample (clamp = 1: negative outputs -> 0, the count added to
 * *clamped_entries) or upsample_raw (clamp = 0) of P linear-sRGB triples (device, P x 3
 * doubles) into codes (device, P x k doubles): the reference's fp64 network and
 * summation order; SiLU's exp is CUDA's (<= 1 ulp from glibc), so results agree with the
 * reference to ~1e-15 relative. */
int hc_upsampler_create(hc_ctx ctx, int k, int hidden, const double* w1, const double* b1, const double* w2,
                        const double* b2, const double* w3, const double* b3, hc_upsampler* out);
int hc_upsampler_destroy(hc_upsampler up);
int hc_upsample_f64(hc_upsampler up, const double* rgb, int64_t P, int clamp, double* codes,
                    uint64_t* clamped_entries);

/* upsample_loss + upsample_gradients (upsampler.cpp:207-369) of UpsamplerWeights (host, as
 * hc_upsampler_create) over a batch of B samples: rgb (device, B x 3) and target codes
 * (device, B x k) of the frozen codec whose effective decoder codec_dec (host, n x k) and
 * CmfTable D65 rows wxyz (host, 3 x n: wx, wy, wz) and white (host, 3) define the colour
 * term; lambda_maxabs / lambda_color as UpsampleTrainConfig.  losses[4] = {latent_mse,
 * latent_maxabs, color, total} and grads (host, w1 | b1 | w2 | b2 | w3 | b3 concatenated in
 * UpsamplerWeights layout) may be NULL.  Within ~1e-12 of the reference (exp, cbrt). */
int hc_upsample_train_grad(hc_ctx ctx, int k, int hidden, const double* w1, const double* b1, const double* w2,
                           const double* b2, const double* w3, const double* b3, int n, const double* codec_dec,
                           const double* wxyz, const double* white, const double* rgb, const double* target, int64_t B,
                           double lambda_maxabs, double lambda_color, double* losses, double* grads);
/* adamw_step (upsampler.cpp:378-391) on device arrays, decoupled weight decay. */
int hc_adamw_step(hc_ctx ctx, double* params, const double* grad, double* m1, double* v1, int64_t count, double lr,
                  double weight_decay, int64_t step);

/* ------------------------------------------------------------------ host-buffer entry points
 * Reference-facing value calls: inputs and outputs in HOST memory (pinned for
 * full copy speed), copies and compute on the context stream, synchronised on
 * return.  These are what a caller of the reference's by-value API binds. */
int hc_shade_latent_host(hc_codec codec, const float* pal_codes, int n_pal, const float* light_codes,
                         int L, const uint32_t* idx, const float* cosv, int64_t P, float* xyz,
                         float* rgb);
/* A sequence of frames of the same scene (one palette / light table, per-frame G-buffers
 * idx[f], cosv[f] and outputs xyz[f], rgb[f], all host, each P pixels): one copy / compute
 * pipeline across all frames (frame f + 1's uploads overlap frame f's downloads), so a
 * frame stream runs at the PCIe rate instead of paying pipeline fill / drain per frame.
 * Outputs are identical to nframes hc_shade_latent_host calls.  xyz[f] / rgb[f] may be
 * NULL (not computed / copied). */
int hc_shade_latent_host_frames(hc_codec codec, const float* pal_codes, int n_pal, const float* light_codes,
                                int L, int nframes, const uint32_t* const* idx, const float* const* cosv,
                                int64_t P, float* const* xyz, float* const* rgb);
int hc_roundtrip_host(hc_codec codec, const float* S, int64_t rows, float* Z, float* S2, float* xyz,
                      float* rgb);

/* ------------------------------------------------------------------ synthetic inputs
 * Seeded generators for the BASELINE configs.  Keys are
 * hc_stream_key(seed, purpose); value i of a counter stream is
 * splitmix64(key + (i + 1) * 0x9e3779b97f4a7c15) (rng.cpp:17-22). */
uint64_t hc_stream_key(uint64_t seed, const char* purpose);
/* Gaussian-mixture spectra: item i uses Rng(ctr(key, first + i)) (rng.cpp:32-81):
 * m = 1 + index(4) bumps (centre U[380,780], sigma U[10,100], amp U[0,1]),
 * gaussian_curve sum (spectrum.cpp:97-105), clipped to [0,1]. */
int hc_synth_gm_spectra(hc_ctx ctx, uint64_t key, int64_t first, int64_t count, int n,
                        double lambda_min, double lambda_step, float* out);
/* idx[p] = ctr(key_idx, p) % n_pal ; cos[p*L+l] = u24(ctr(key_cos, p*L+l)). */
int hc_synth_gbuffer(hc_ctx ctx, uint64_t key_idx, uint64_t key_cos, int64_t first, int64_t P, int L,
                     int n_pal, uint32_t* idx, float* cosv);
int hc_synth_chain(hc_ctx ctx, uint64_t key_pidx, uint64_t key_iidx, uint64_t key_tw, int64_t first,
                   int64_t P, int spp, int n_pal, int n_ill, uint8_t* pidx, uint8_t* iidx, float* tw);
/* out[i] = u24(ctr(key, first + i)) in [0, 1). */
int hc_synth_uniform(hc_ctx ctx, uint64_t key, int64_t first, int64_t count, float* out);
/* Write `bytes` of garbage over a device buffer (L2 flush between timed steps). */
int hc_flush_l2(hc_ctx ctx, void* buf, int64_t bytes);
/* Keep the context's stream busy for `cycles` SM clocks (one spinning thread).  Measurement helper:
 * a start event queued behind it is stamped when the work after it can start, not while the
 * host is still enqueuing that work. */
int hc_spin(hc_ctx ctx, int64_t cycles);

/* ------------------------------------------------------------------ several GPUs
 * Replaces the renderer's row-scheduled thread pool (renderer.cpp:573-608,
 * HADACODEC_THREADS :615-621) across devices: an image is cut into contiguous row
 * bands, one per GPU, each driven by its own host thread, context and stream.
 * hc_row_band: rows [*row0, *row0 + *rows) of rank `rank` of `world` over `height`
 * rows; sizes differ by at most one row (the Python sharding module calls this too). */
int hc_row_band(int rank, int world, int64_t height, int64_t* row0, int64_t* rows);
typedef struct hc_group_s* hc_group;
#define HC_GATHER_HOST 0 /* each device copies its band into the host image (own PCIe link) */
#define HC_GATHER_NCCL 1 /* bands -> device 0 by grouped ncclSend / ncclRecv, one D2H copy */
#define HC_GATHER_PEER 2 /* bands -> device 0 by cudaMemcpyPeerAsync, one D2H copy */
#define HC_GATHER_FUSED 3 /* no gather step: each device's shade kernel stores its band straight into
                           * device 0's frame through NVLink peer memory, one D2H copy */
/* devices[ndev] (distinct for HC_GATHER_NCCL: ncclCommInitAll); NCCL is loaded at run time
 * (libnccl.so.2) and its absence is HC_EUNSUPPORTED for that mode. */
int hc_group_create(const int* devices, int ndev, int gather, hc_group* out);
int hc_group_destroy(hc_group g);
int hc_group_size(hc_group g);
/* Version of the NCCL library the group layer loaded (e.g. 22809), 0 if none. */
int hc_group_nccl_version(void);
/* One codec per device (the arguments of hc_codec_create). */
int hc_group_codec_create(hc_group g, int k, int n, const float* E, const float* D, const double* cmf,
                          double dlambda);
/* hc_shade_latent_host over a width x height frame split into row bands across the group:
 * host G-buffer in (idx [P], cosv [P][L]), host XYZ / sRGB out ([P][3], may be NULL);
 * bit-identical to one hc_shade_latent_host call on the whole frame. */
int hc_group_shade_latent_host(hc_group g, const float* pal_codes, int n_pal, const float* light_codes, int L,
                               const uint32_t* idx, const float* cosv, int64_t width, int64_t height, float* xyz,
                               float* rgb);

/* One process per GPU (torch.distributed / MPI ranks): the fused gather across processes.  The
 * destination rank allocates the full frame with hc_ipc_alloc and publishes the 64-byte handle
 * (CUDA IPC); every other rank maps it with hc_ipc_open (peer access from its own device is
 * enabled by the mapping) and passes its band's slice as the output pointer of hc_shade_latent,
 * so its kernels store straight into the destination GPU's frame over NVLink.  hc_ipc_close
 * unmaps (openers), hc_ipc_free releases (owner). */
#define HC_IPC_HANDLE_BYTES 64
int hc_ipc_alloc(int device, int64_t bytes, void** dptr, unsigned char* handle);
int hc_ipc_open(int device, const unsigned char* handle, void** dptr);
int hc_ipc_close(int device, void* dptr);
int hc_ipc_free(int device, void* dptr);

#ifdef __cplusplus
}
#endif
#endif /* HADACODEC_B200_H */
