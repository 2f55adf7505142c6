/* TEST INFRASTRUCTURE (oracle) — not product code.
 *
 * C signatures shared by the two CPU oracles of the flow+blend hot path:
 *   fso_*   : oracle/fs_oracle.c, a plain-C restatement of the reference
 *             algorithm (single-threaded), each function citing the
 *             reference file:line it restates;
 *   fsref_* : oracle/ref_capi.cpp, a thin extern "C" wrapper that calls the
 *             UNMODIFIED reference library compiled from /root/reference
 *             (oracle/Makefile -> oracle/_ref/libfsref.so).
 * Both export the same parameter lists so tests can run one against the
 * other and both against the CUDA path.  Only tests/, __graft_entry__.smoke()
 * and bench.py's CPU legs may load these libraries.
 *
 * Layouts follow the reference value types:
 *   image : float data[w*h*ch] interleaved (ch = 1 or 3), uint8 valid[w*h]
 *           (proj/include/flowstitch/image.hpp:32-64)
 *   flow  : float vec[w*h*2] interleaved (dx,dy), uint8 valid[w*h]
 *           (proj/include/flowstitch/flow.hpp:15-34)
 *   label : uint8 {0 Outside, 1 Area1, 2 Area2, 3 Area3}, counts int64[4]
 *           (proj/include/flowstitch/image.hpp:66-77)
 *   dist / blend : double[w*h] (proj/include/flowstitch/blend_field.hpp:12-28)
 * Status: 0 ok, 1 contract error, 2 empty region, 3 layout error.
 */
#ifndef FS_ORACLE_H
#define FS_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { FSO_OK = 0, FSO_CONTRACT = 1, FSO_EMPTY = 2, FSO_LAYOUT = 3 };

int fso_to_gray(const float* img, int w, int h, int ch, float* out);
void fso_bilinear_sample(const float* img, const uint8_t* valid, int w, int h, int ch,
                         double x, double y, float* out);
int fso_compute_partition(const uint8_t* mask_l, const uint8_t* mask_r, int w, int h,
                          uint8_t* label, int64_t* counts);
int fso_crop_box(const uint8_t* label, const int64_t* counts, int w, int h, int* box);
int fso_crop_overlap(const float* img, const uint8_t* valid, int w, int h, int ch,
                     const uint8_t* label, const int64_t* counts, float* out,
                     uint8_t* out_valid, int* box);
int fso_place_on_canvas(const float* img, const uint8_t* valid, int w, int h, int ch,
                        int ox, int oy, int cw, int chh, float* out, uint8_t* out_valid);
int fso_pyramid_depth(int w, int h, int levels);
int fso_build_pyramid(const float* img, int w, int h, int levels, float* out);
int fso_dense_pyr_lk(const float* from, const float* to, int w, int h, int levels, int radius,
                     int iters, double eps, int smoothing, float* vec, uint8_t* valid);
int fso_bidirectional_flow(const float* l, const float* r, int w, int h, int ch, int levels,
                           int radius, int iters, double eps, int smoothing, float* vec_lr,
                           uint8_t* valid_lr, float* vec_rl, uint8_t* valid_rl);
int fso_embed_flow(const float* vec, const uint8_t* valid, int w, int h, int ox, int oy,
                   int cw, int chh, float* out_vec, uint8_t* out_valid);
void fso_flow_magnitude(const float* vec, int w, int h, float* out);
int fso_distance_transform(const uint8_t* mask, int w, int h, double* out);
int fso_compute_blend(const uint8_t* label, const int64_t* counts, int w, int h, double* b);
void fso_softmax_weights(double blend_l, double blend_r, double mag_rtol, double mag_ltor,
                         double k, double coef, double* out2);
int fso_feather_blend(const float* l, const float* r, int w, int h, int ch, const double* b,
                      const uint8_t* label, float* out, uint8_t* out_valid);
int fso_warp_constituents(const float* l, const uint8_t* vl, const float* r, const uint8_t* vr,
                          int w, int h, int ch, const float* flow_lr, const float* flow_rl,
                          const double* b, const uint8_t* label, float* out_l, uint8_t* out_vl,
                          float* out_r, uint8_t* out_vr);
int fso_blend_pair(const float* l, const uint8_t* vl, const float* r, const uint8_t* vr, int w,
                   int h, int ch, const float* flow_lr, const float* flow_rl, const double* b,
                   const uint8_t* label, double k, double coef, float* out, uint8_t* out_valid);
/* misalignment_score (proj/src/pipeline.cpp:309-396, with patch_stats,
 * patch_ncc and better_candidate at :215-256): mean shift norm of the best
 * NCC match of every textured (2r+1)^2 patch fully inside Area3, searched
 * over +-2r in R.  l, r: w*h*ch images (r_valid: R's validity; L's validity
 * is not read), label/counts: the partition.  *out = the score. */
int fso_misalignment_score(const float* l, const uint8_t* l_valid, const float* r,
                           const uint8_t* r_valid, int w, int h, int ch, const uint8_t* label,
                           const int64_t* counts, int patch_radius, int stride, double* out);
/* estimate_translation (proj/src/pipeline.cpp:261-307): exhaustive integer
 * shift NCC search of B against A (grayscale, ch must be 1). */
int fso_estimate_translation(const float* a, const float* b, int w, int h, int ch, int max_shift,
                             int* dx, int* dy, double* score);
/* Fold over n placed images (proj/src/pipeline.cpp:140-212 without the
 * misalignment metrics, which never touch the panorama).  imgs[i] is
 * dims[2i] x dims[2i+1] x ch, placed at offsets[2i], offsets[2i+1].
 * stats (optional, n-1 rows of 4): overlap px, crop x0, y0 ... see .c */
int fso_stitch_placed(int n, const float* const* imgs, const uint8_t* const* valids,
                      const int* dims, const int* offsets, int ch, int cw, int chh, int levels,
                      int radius, int iters, double eps, int smoothing, double k, double coef,
                      float* out, uint8_t* out_valid);

#ifdef __cplusplus
}
#endif

#endif
