/* ORACLE / TEST INFRASTRUCTURE — NOT PART OF THE PRODUCT.
 *
 * Plain-C restatement of the reference's per-pixel codec / latent-shading path
 * (hadacodec, /root/reference/proj/core).  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline leg may load it, and only as the checker.
 *
 * Conventions follow the reference exactly: fp64 accumulation for the codec
 * mat-vecs (codec.cpp:36-46, :52-71; renderer.cpp:661-690), fp32 per-sample
 * shading arithmetic with an fp64 per-pixel reduction (renderer.cpp:442-551),
 * radiance-convention XYZ with the grid step applied after the sum
 * (colorimetry.cpp:75-87) and the IEC 61966-2-1 matrix (colorimetry.cpp:22-26).
 * Parity is pinned (tests/test_oracle.py) against the compiled reference
 * (oracle/_ref, see Makefile) bit-for-bit and against the reference tests'
 * frozen known-answer values (tests/golden/reference_kats.json).
 *
 * Layouts (row-major, pixel-major): spectra [rows][n], codes [rows][k],
 * xyz / rgb [rows][3], E [k][n], D [n][k], cmf [3][n] (xbar, ybar, zbar).
 */
#ifndef HC_ORACLE_H
#define HC_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

double orc_softplus(double raw, double beta);

/* codec.cpp:36-46: z_r = sum_i E[r*n+i] * s_i in double; zd and/or zf may be NULL. */
void orc_encode(const float* E, int k, int n, const float* S, int64_t rows, double* zd, float* zf);
/* renderer.cpp:661-690: s_i = float(sum_j D[i*k+j] * double(z_j)). */
void orc_decode(const float* D, int k, int n, const float* Z, int64_t rows, float* S);
/* colorimetry.cpp:75-87 then :103-105, on fp32 spectra; xyz/rgb may be NULL. */
void orc_spectra_to_outputs(const double* cmf, double dlambda, int n, const float* S, int64_t rows,
                            float* xyz, float* rgb);
/* spectrum_to_xyz on a double curve (KAT pinning). */
void orc_spectrum_to_xyz_d(const double* cmf, double dlambda, int n, const double* s, double* xyz);
/* Config 1 round trip: encode -> fp32 code -> decode -> fp32 spectra -> XYZ / sRGB. */
void orc_codec_roundtrip(const float* E, const float* D, int k, int n, const double* cmf,
                         double dlambda, const float* S, int64_t rows, float* Z, float* S2,
                         float* xyz, float* rgb);
/* Asset codes (renderer.cpp:117-125): float(encode(E, s)). */
void orc_asset_codes(const float* E, int k, int n, const float* S, int64_t count, float* Z);

/* Configs 2/3 latent G-buffer shading (renderer.cpp:505-510, 645-657),
 * then decode + projection.  latent / S2 / xyz / rgb may be NULL. */
void orc_shade_latent(const float* D, int k, int n, const double* cmf, double dlambda,
                      const float* pal_codes, const float* light_codes, int L,
                      const uint32_t* idx, const float* cosv, int64_t P, float* latent,
                      float* S2, float* xyz, float* rgb);
/* Naive n-sample shading (renderer.cpp:187-190, :505-510 at C = n). */
void orc_shade_spectral(int n, const double* cmf, double dlambda, const float* pal_spectra,
                        const float* light_spectra, int L, const uint32_t* idx,
                        const float* cosv, int64_t P, float* S2, float* xyz, float* rgb);

/* Config 4 chain (SURVEY Appendix A #7; renderer.cpp:505-510, :530-533, :548-551). */
void orc_chain(int C, const float* pal, const float* ill, const uint8_t* pidx,
               const uint8_t* iidx, const float* tw, int64_t P, int spp, int depth, float* out);

/* Config 5a MLP (upsampler.cpp:42-72 with ReLU / softplus(beta=1)). */
float orc_bf16_round(float x);
void orc_mlp_forward(const float* rgb, int64_t P, int hidden, int k, const float* w1,
                     const float* b1, const float* w2, const float* b2, const float* w3,
                     const float* b3, float* out);

/* Config 5b loss (trainer.cpp:49-71). */
double orc_hadamard_loss(const float* E, const float* D, int k, int n, const float* A,
                         const float* B, int64_t pairs);

/* Colour-metric tail (SURVEY §8f row 1; renderer.cpp:721-802, evaluation.cpp:14-28, :59-86,
 * :122-154, colorimetry.cpp:111-162).  Images are P pixels x channels (3 = linear RGB, n =
 * spectra); cmf = [3][n] rows (xbar, ybar, zbar) of the grid. */
double orc_percentile_nearest_rank(const double* v, int64_t count, double p);
void orc_luminance(const float* img, int64_t P, int channels, const double* ybar, double dlambda, double* lum);
double orc_exposure_for(const float* img, int64_t P, int channels, const double* ybar, double dlambda,
                        double percentile);
double orc_srgb_encode(double linear);
void orc_tonemap_srgb8(const float* rgb, int64_t P, double exposure, uint8_t* out);
void orc_image_to_linear_rgb(const float* img, int64_t P, int channels, const double* cmf, double dlambda,
                             float* rgb);
double orc_error_map(const float* a, int ca, const float* b, int cb, int64_t P, const double* cmf,
                     double dlambda, float* mse);
void orc_xyz_to_lab(const double* xyz, const double* white, double* lab);
double orc_delta_e76(const double* a, const double* b);
double orc_delta_e94(const double* ref, const double* sample);
void orc_scene_color_report(const float* gt, int cgt, const float* test, int ctest, int64_t P,
                            const double* cmf, double dlambda, double* out);
void orc_delta_e94_report(const float* xyz_gt, const float* xyz_test, int64_t P, const double* white_d65,
                          float* de, double* out);

#ifdef __cplusplus
}
#endif
#endif
