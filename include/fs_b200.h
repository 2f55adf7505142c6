/* fs_b200.h — C-ABI of the B200 flow+blend path (the drop-in boundary).
 *
 * One extern "C" entry point per function of the reference's hot-path API
 * (namespace flowstitch, /root/reference/proj/include/flowstitch/{image,flow,
 * blend_field,blender,pipeline}.hpp), each
 * citing the declaration it replaces.  Plain pointers and sizes only; the
 * data layouts are the reference's value types:
 *   image : float[w*h*ch] interleaved, ch = 1 or 3, plus uint8 valid[w*h]
 *           (image.hpp:32-64, ImageBuf)
 *   mask  : uint8[w*h] (image.hpp:17-28, Mask)
 *   label : uint8[w*h] in {0 Outside, 1 Area1, 2 Area2, 3 Area3} and
 *           int64 counts[4] (image.hpp:66-77, Region/RegionPartition)
 *   flow  : float[w*h*2] interleaved (dx, dy), uint8 valid[w*h] (flow.hpp:15-34)
 *   field : double[w*h] (blend_field.hpp:12-28, DistanceField / BlendField)
 * Buffers may live in host or device memory (CUDA unified addressing tells the
 * two apart); host buffers are staged through the device inside the call.
 * `stream` is a cudaStream_t (NULL = the legacy default stream).  Calls with
 * host outputs return after the result is in place; calls whose outputs are
 * all device pointers are asynchronous on `stream`.
 *
 * Errors: the reference throws (errors.hpp:10-37); here every call returns a
 * status and fs_last_error() gives the thread-local message, with the same
 * wording as the reference's exception where the reference tests match on it.
 * There is no CPU fallback: without a usable sm_100 GPU every compute entry
 * point returns FS_ERR_CUDA.
 */
#ifndef FS_B200_H
#define FS_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    FS_OK = 0,
    FS_ERR_CONTRACT = 1,     /* ContractError  (errors.hpp:10-14) */
    FS_ERR_EMPTY_REGION = 2, /* EmptyRegionError (errors.hpp:34-38) */
    FS_ERR_LAYOUT = 3,       /* LayoutError (errors.hpp:28-32) */
    FS_ERR_CUDA = 4,         /* device missing / CUDA failure */
    FS_ERR_OOM = 5,          /* device allocation failed */
    FS_ERR_UNSUPPORTED = 6,  /* parameter outside what the kernels implement */
    FS_ERR_IO = 7,           /* IoError (errors.hpp:16-20) */
    FS_ERR_FORMAT = 8,       /* FormatError (errors.hpp:22-26) */
    FS_ERR_SHARD_REACH = 9   /* a sharded fold read canvas pixels its GPU does not hold final:
                                the result is not certified, execute unsharded */
} fs_status;

/* FlowParams (flow.hpp:36-44); defaults 4 / 8 / 3 / 1e-4 / 2. */
typedef struct {
    int levels;
    int window_radius;
    int iterations_per_level;
    double min_eigen_eps;
    int smoothing_passes;
} fs_flow_params;

/* BlendParams (blender.hpp:12-17); defaults 10 / 0.05. */
typedef struct {
    double k_softmax_sharpness;
    double k_flow_mag_coef;
} fs_blend_params;

/* PairStats subset (pipeline.hpp:30-38) filled by the fold. */
typedef struct {
    int64_t overlap_pixels;
    double mean_flow_mag_ltor;
    double mean_flow_mag_rtol;
    double flow_seconds;  /* device time of the pair's flow stage */
    double blend_seconds; /* device time of blend field + blend + compose */
    int32_t crop_box[4];  /* x0, y0, w, h of the Area3 bounding box */
    /* misalignment_score (pipeline.cpp:184-199) of the raw pair and of the
     * flow-warped constituents, patch radius 8, stride 32; present flags
     * (bit 0 before, bit 1 after) are clear where the reference's optional
     * stays empty (no textured patch). */
    int32_t misalignment_present;
    double misalignment_before;
    double misalignment_after;
} fs_pair_stats;

const char* fs_last_error(void);
int fs_abi_version(void);
/* 1 if a usable sm_100 device is present (does not initialise the others). */
int fs_device_available(void);
/* Checks builds (make -C paper_2006_01201_b200/csrc EXTRA=-DFS_CHECKS,
 * tools/checks.sh): device-side bounds / hand-off checks counted on the
 * device; the number of violations since the last reset (0 in normal builds). */
unsigned int fs_debug_check_failures(int reset);
int fs_debug_checks_built(void);
/* checks builds only: inject a fault the checks must report (1: mis-stamped
 * producer/consumer hand-off, 2: tap copies read before they landed; 0: off) */
void fs_debug_inject(int mode);
void fs_default_flow_params(fs_flow_params* p);
void fs_default_blend_params(fs_blend_params* p);

/* ---- imagecore (image.hpp:94-108) ---- */
/* to_gray (image.hpp:94): out is w*h floats. */
fs_status fs_to_gray(const float* img, int w, int h, int ch, float* out, void* stream);
/* bilinear_sample (image.hpp:98), batched: xy = n (x, y) pairs, out = n*ch. */
fs_status fs_bilinear_sample(const float* img, const uint8_t* valid, int w, int h, int ch,
                             const double* xy, int n, float* out, void* stream);
/* compute_partition (image.hpp:100). */
fs_status fs_compute_partition(const uint8_t* mask_l, const uint8_t* mask_r, int w, int h,
                               uint8_t* label, int64_t* counts, void* stream);
/* crop_overlap (image.hpp:103): box = {offset_x, offset_y, w, h}; pass out =
 * NULL to query the box, then call again with buffers of box[2]*box[3]. */
fs_status fs_crop_overlap(const float* img, const uint8_t* valid, int w, int h, int ch,
                          const uint8_t* label, const int64_t* counts, float* out,
                          uint8_t* out_valid, int* box, void* stream);
/* place_on_canvas (image.hpp:107-108); valid may be NULL (all valid). */
fs_status fs_place_on_canvas(const float* img, const uint8_t* valid, int w, int h, int ch,
                             int offset_x, int offset_y, int canvas_w, int canvas_h, float* out,
                             uint8_t* out_valid, void* stream);

/* ---- optflow (flow.hpp:46-66) ---- */
/* pyramid depth for a w x h level 0 (flow.hpp:46-48) */
int fs_pyramid_depth(int w, int h, int levels);
/* build_pyramid (flow.hpp:48): levels concatenated, level 0 first. */
fs_status fs_build_pyramid(const float* gray, int w, int h, int levels, float* out, int* depth,
                           void* stream);
/* dense_pyr_lk (flow.hpp:52) */
fs_status fs_dense_pyr_lk(const float* from, const float* to, int w, int h,
                          const fs_flow_params* params, float* vec, uint8_t* valid,
                          void* stream);
/* bidirectional_flow (flow.hpp:56-58): returns {LtoR, RtoL}. */
fs_status fs_bidirectional_flow(const float* overlapped_l, const float* overlapped_r, int w,
                                int h, int ch, const fs_flow_params* params, float* vec_ltor,
                                uint8_t* valid_ltor, float* vec_rtol, uint8_t* valid_rtol,
                                void* stream);
/* flow_magnitude (flow.hpp:61) */
fs_status fs_flow_magnitude(const float* vec, int w, int h, float* out, void* stream);
/* embed_flow (flow.hpp:65-66) */
fs_status fs_embed_flow(const float* vec, const uint8_t* valid, int w, int h, int offset_x,
                        int offset_y, int canvas_w, int canvas_h, float* out_vec,
                        uint8_t* out_valid, void* stream);

/* ---- blendfield (blend_field.hpp:30-34) ---- */
/* distance_transform (blend_field.hpp:32) */
fs_status fs_distance_transform(const uint8_t* mask, int w, int h, double* out, void* stream);
/* compute_blend (blend_field.hpp:34) */
fs_status fs_compute_blend(const uint8_t* label, const int64_t* counts, int w, int h, double* b,
                           void* stream);

/* ---- blender (blender.hpp:19-46) ---- */
/* softmax_weights (blender.hpp:21-23): scalar, evaluated with the kernels'
 * own per-pixel routine (host copy of the same source). */
void fs_softmax_weights(double blend_l, double blend_r, double mag_rtol, double mag_ltor,
                        const fs_blend_params* params, double* sl, double* sr);
/* blend_pair (blender.hpp:30-33): all inputs canvas-sized. */
fs_status fs_blend_pair(const float* l, const uint8_t* valid_l, const float* r,
                        const uint8_t* valid_r, int w, int h, int ch, const float* flow_ltor,
                        const float* flow_rtol, const double* blend, const uint8_t* label,
                        const fs_blend_params* params, float* out, uint8_t* out_valid,
                        void* stream);
/* feather_blend (blender.hpp:36-37) */
fs_status fs_feather_blend(const float* l, const uint8_t* valid_l, const float* r,
                           const uint8_t* valid_r, int w, int h, int ch, const double* blend,
                           const uint8_t* label, float* out, uint8_t* out_valid, void* stream);
/* warp_constituents (blender.hpp:42-46) */
fs_status fs_warp_constituents(const float* l, const uint8_t* valid_l, const float* r,
                               const uint8_t* valid_r, int w, int h, int ch,
                               const float* flow_ltor, const float* flow_rtol,
                               const double* blend, const uint8_t* label, float* out_l,
                               uint8_t* out_valid_l, float* out_r, uint8_t* out_valid_r,
                               void* stream);

/* misalignment_score (pipeline.hpp:81-83; src/pipeline.cpp:309-396): the
 * seam metric of StitchReport.  l, r: w x h x ch canvases (valid_l unused,
 * as in the reference), label/counts: their partition.  Defaults in the
 * reference: patch_radius 8, stride 32.  FS_ERR_EMPTY_REGION when no patch
 * is textured. */
fs_status fs_misalignment_score(const float* l, const uint8_t* valid_l, const float* r,
                                const uint8_t* valid_r, int w, int h, int ch,
                                const uint8_t* label, const int64_t* counts, int patch_radius,
                                int stride, double* out, void* stream);

/* estimate_translation (pipeline.hpp:69-77; src/pipeline.cpp:261-307):
 * exhaustive integer-shift NCC of B against A (grayscale, ch == 1),
 * |dx|, |dy| <= max_shift <= min(w, h) / 4. */
fs_status fs_estimate_translation(const float* a, const float* b, int w, int h, int ch,
                                  int max_shift, int* dx, int* dy, double* score, void* stream);

/* ---- pre-processing (north_star stage 1) ----
 * Absent from the reference (SPEC.md:12 delegates it to Hugin/PanoTools):
 * parity UNPINNED — checked against a numpy restatement (oracle/remap.py)
 * only.  An equidistant fisheye camera (r = f * theta) at orientation
 * yaw/pitch/roll is resampled onto a rectangle of an equirectangular canvas
 * (canvas_w x canvas_h covers 360 x 180 degrees), which is then a placed view
 * of stitch_placed / fs_plan_*. */
typedef struct {
    int width, height;      /* fisheye image */
    double cx, cy;          /* optical centre (px) */
    double focal;           /* px per radian (equidistant) */
    double radius;          /* image circle radius (px); taps beyond are invalid */
    double yaw, pitch, roll;  /* radians: camera = Ry(yaw) Rx(pitch) Rz(roll) */
} fs_fisheye_camera;
/* Host-only remap table: for every pixel of the canvas rectangle
 * (x0, y0, w, h), the fisheye source position (x, y) as two floats
 * (computed in double), or (-1, -1) where the ray misses the image circle. */
fs_status fs_fisheye_map(const fs_fisheye_camera* cam, int canvas_w, int canvas_h, int x0, int y0,
                         int w, int h, float* map_xy);
/* Device remap of an RGBA8 (or RGB8 with channels = 3) fisheye image through
 * a table (device pointers), with per-channel chromaticity gains:
 * out = min(255, floor(bilinear(src) * gain + 0.5)), alpha 255 where the
 * table is valid, else the pixel is (0, 0, 0, 0).  Pointers may be host or
 * device memory (gains3: three floats, NULL = no correction). */
fs_status fs_remap_rgba8(const uint8_t* src, int sw, int sh, int channels, const float* map_xy,
                         int w, int h, const float* gains3, uint8_t* out_rgba, void* stream);

/* Chromaticity gains (exposure compensation) of n placed RGBA8 views:
 * view 0 keeps (1, 1, 1); view k's gain per channel makes its overlap with
 * the earlier views (each pixel's first covering view m, scaled by gain m)
 * agree in the mean: g_k = sum_m g_m * S[k][m] / sum_m T[k][m], where S and
 * T are the exact integer channel sums of view m and view k over the pixels
 * both cover (k valid, first covered by m < k).  gains: n x 3 floats out
 * (host memory); views host or device. */
fs_status fs_chroma_gains(int n, const uint8_t* const* views_rgba, const int* dims,
                          const int* offsets, int canvas_w, int canvas_h, float* gains,
                          void* stream);

/* ---- pipeline fold (pipeline.hpp:63-67) ---- */
/* stitch_placed: images[i] is dims[2i] x dims[2i+1] x ch at offsets[2i],
 * offsets[2i+1]; valids may be NULL or hold NULL entries (all valid).  The
 * whole fold runs device-resident; stats (optional) gets n-1 entries. */
fs_status fs_stitch_placed(int n, const float* const* images, const uint8_t* const* valids,
                           const int* dims, const int* offsets, int ch, int canvas_w,
                           int canvas_h, const fs_flow_params* flow, const fs_blend_params* blend,
                           float* out, uint8_t* out_valid, fs_pair_stats* stats, void* stream);

/* ---- production path: planned, graph-captured fold over 8-bit views ----
 * A plan fixes the layout (view sizes, offsets, fold order, canvas) and owns
 * all device memory.  Executions recompute everything per call (partition,
 * crop, pyramid, flow, distance transform, blend, compose, quantise) and
 * verify on the device that the views' masks still produce the planned Area3
 * boxes; fs_plan_check() reports a mismatch.  Views are RGBA8 (alpha >= 128
 * valid, image.hpp:86-88) and the output canvas is RGBA8 (alpha = valid). */
typedef struct fs_plan_s* fs_plan;
fs_status fs_plan_create(fs_plan* plan, int device, int n, const int* dims, const int* offsets,
                         int canvas_w, int canvas_h, const fs_flow_params* flow,
                         const fs_blend_params* blend, const uint8_t* const* views_rgba);
/* device pointer of view k's RGBA8 buffer (dims[2k]*dims[2k+1]*4 bytes) */
void* fs_plan_view_buffer(fs_plan plan, int k);
/* device pointer of the RGBA8 output canvas (canvas_w*canvas_h*4 bytes) */
void* fs_plan_output_buffer(fs_plan plan);
/* run the fold on the views already in the plan's device buffers (async) */
fs_status fs_plan_execute(fs_plan plan, void* stream);
/* end-to-end: copy host (or device) views in, fold, copy the canvas out */
fs_status fs_plan_execute_host(fs_plan plan, const uint8_t* const* views_rgba, uint8_t* out_rgba,
                               void* stream);
/* the same, asynchronous on `stream` (page-locked host buffers, DAG plans):
 * no synchronisation and no check — after synchronising, the caller calls
 * fs_plan_check (and on a status other than FS_OK repeats the execution with
 * fs_plan_execute_host).  Lets several plans (panoramas) overlap on one GPU. */
fs_status fs_plan_execute_host_async(fs_plan plan, const uint8_t* const* views_rgba,
                                     uint8_t* out_rgba, void* stream);
/* after the stream is synchronised: FS_OK or the first device-side error */
fs_status fs_plan_check(fs_plan plan);
/* number of kernel launches of one execution (for accounting) */
int fs_plan_launch_count(fs_plan plan);
/* Host buffer formats of fs_plan_execute_host / fs_plan_shard_execute:
 * views RGBA8 (4, default) or RGB8 (3: every pixel valid, expanded to RGBA8
 * on the device), canvas RGBA8 (4, default) or RGB8 (3: alpha dropped, for
 * canvases the views cover completely).  Fewer bytes cross PCIe.  With RGB8
 * views the plan also treats every view pixel as valid in the device-
 * resident fs_plan_execute (a view's validity is its placement), so views
 * written into fs_plan_view_buffer must then be fully valid as well. */
fs_status fs_plan_set_host_format(fs_plan plan, int view_channels, int out_channels);
/* bytes fs_plan_execute_host moves with page-locked buffers: views in, and
 * the canvas read back (rectangles no view covers are zeroed on the host) */
fs_status fs_plan_transfer_bytes(fs_plan plan, size_t* h2d, size_t* d2h);
/* Row/column tiles of the folds' flows (the reference has
 * no tiling — its dense_pyr_lk, src/flow.cpp:194-314, runs over a whole crop):
 * every fold whose Area3 box is longer than tile_len along its long axis is
 * cut there into interiors of about tile_len, each computed as its own crop
 * + pyramid + LK over the interior grown by the whole dependency cone (so the
 * interior's flow equals the untiled one), the crop waiting only for the
 * earlier composes its region meets; gathers are certified on the device to
 * stay `margin` px inside the tile pyramid's exact part, else the fold runs
 * untiled (fs_plan_check, then execute again).  Boxes whose long side is not
 * divisible by 2^(levels-1) stay untiled.  tile_len = 0: no tiles (default).
 * Needs the DAG schedule (<= 16 views). */
fs_status fs_plan_set_tiling(fs_plan plan, int tile_len, int margin);
/* tiles of fold k in use (0: untiled, -1: bad argument); region / interior
 * {x0, y0, w, h} box-relative (either may be NULL) */
int fs_plan_tile_count(fs_plan plan, int k);
fs_status fs_plan_tile_info(fs_plan plan, int k, int t, int* region, int* interior);
/* fold geometry: for fold k (1..n-1) the Area3 box {x0,y0,w,h} and depth */
fs_status fs_plan_fold_info(fs_plan plan, int k, int* box, int* depth);
/* fold k's crop flows of the last execution (the FlowFields bidirectional_flow
 * returns inside stitch_placed, src/pipeline.cpp:171-172): interleaved (dx,dy)
 * float + u8 valid, box w x h each; host or device destinations, any of the
 * four may be NULL.  Synchronises the plan's device. */
fs_status fs_plan_fold_flow(fs_plan plan, int k, float* ltor_vec, uint8_t* ltor_valid,
                            float* rtol_vec, uint8_t* rtol_valid);
/* one un-captured execution with CUDA events around every kernel launch on
 * `stream`; per kernel family: launches, summed device ms and algorithmic
 * bytes.  total_ms spans the whole execution. */
typedef struct {
    char name[24];
    int launches;
    double ms;
    double bytes;
} fs_kernel_stat;
/* Schedule diagnostics: one execution of the DAG (with the host copies when
 * views/out are given) launched stream by stream with timing events at its
 * schedule points; writes a
 * JSON object {"label": ms since start} into json (cap bytes). */
fs_status fs_plan_timeline(fs_plan plan, const uint8_t* const* views_rgba, uint8_t* out_rgba,
                           void* stream, char* json, int cap);
/* The same points inside the production CUDA graph itself (a one-warp
 * %globaltimer stamp kernel at each point; third replay reported). */
fs_status fs_plan_timeline_graph(fs_plan plan, const uint8_t* const* views_rgba,
                                 uint8_t* out_rgba, void* stream, char* json, int cap);
fs_status fs_plan_profile(fs_plan plan, void* stream, fs_kernel_stat* out, int max_out,
                          int* n_out, double* total_ms);
void fs_plan_destroy(fs_plan plan);

/* ---- seam sharding of one plan over GPUs ----
 * Folds are assigned to ranks (one process per GPU, each holding the same
 * plan); every rank computes the partitions and first-cover copies of all
 * views and the flow, distance transforms and blend of its own folds.  A
 * fold's Area3 "strip" (fold k's blended box, box_w*box_h float4) moves
 * between ranks only where another fold's L crop needs it (Area3 boxes that
 * meet) and to rank 0, the canvas GPU, which composes all strips in fold
 * order and holds the RGBA8 panorama.  The execution is a sequence of
 * segments; after segment s every transfer with stage s is done (by the
 * caller: NCCL send/recv of the strip buffers, or device copies).  Blend taps
 * that land outside what the rank holds final are detected on the device;
 * fs_plan_check() then returns FS_ERR_SHARD_REACH and the caller runs the
 * plan unsharded. */
typedef struct {
    int fold;   /* 1..n-1 */
    int src;    /* rank that computes the strip */
    int dst;    /* rank that needs it */
    int stage;  /* after this segment */
} fs_strip_xfer;
/* Host-only schedule (no device needed).  boxes: fold k's Area3 box at
 * boxes[4k..4k+3] (x0, y0, w, h; k >= 1).  fold_rank[k]: in, -1 (or NULL
 * array) = assign by box area, longest first, to the least loaded rank; out,
 * the rank.  stage[k]: the segment that computes fold k.  *n_segments =
 * number of segments (last stage + 2).  xfers: every transfer of every rank. */
fs_status fs_shard_schedule(int n, const int* boxes, int nranks, int* fold_rank, int* stage,
                            int* n_segments, fs_strip_xfer* xfers, int max_xfers, int* n_xfers);
/* configure `plan` as rank `rank` of `nranks` (fold_rank as above, may be
 * NULL); nranks = 1 restores the unsharded plan. */
fs_status fs_plan_shard(fs_plan plan, int nranks, int rank, const int* fold_rank);
int fs_plan_shard_segments(fs_plan plan);
/* kernel launches of this rank's captured segments (one execution) */
int fs_plan_shard_launch_count(fs_plan plan);
/* the transfers of this plan's rank after segment `segment` (sends and receives) */
fs_status fs_plan_shard_xfers(fs_plan plan, int segment, fs_strip_xfer* out, int max_out,
                              int* n_out);
/* device buffer of fold k's strip (box_w * box_h float4) */
fs_status fs_plan_strip_buffer(fs_plan plan, int fold, void** ptr, size_t* bytes);
/* run segment `segment` (async on stream).  views_rgba (segment 0): host or
 * device views copied in first (NULL: already in the plan's buffers);
 * out_rgba (last segment, rank 0): the RGBA8 canvas copied out. */
fs_status fs_plan_shard_execute(fs_plan plan, int segment, const uint8_t* const* views_rgba,
                                uint8_t* out_rgba, void* stream);

/* ---- runtime (parallel.hpp:9-18): kept for drop-in completeness; the GPU
 * path has no host worker pool, so these only record the value. ---- */
void fs_set_thread_count(int n);
int fs_thread_count(void);

#ifdef __cplusplus
}
#endif

#endif /* FS_B200_H */
