/* hp.h -- C ABI of libhp, the B200-native (sm_100a) per-tile nuclei segmentation +
 * feature pipeline of Teodoro et al., "High-throughput Execution of Hierarchical Analysis
 * Pipelines on Hybrid Cluster Platforms" (arXiv 1209.3332).
 *
 * The paper's model: a data chunk (a 4K x 4K tile,
 * PAPER.md:649-650) flows through a hierarchical pipeline -- two coarse stages,
 * segmentation then feature computation, each a chain of fine
 * operations (Table I) -- and the output is "a set of features for each
 * segmented nucleus".  The calls below are those two stage instances
 * per tile (hp_segment_tile, hp_features_tile; fused as hp_process_tile), the demand-driven
 * multi-tile driver with upload/process/download overlap (hp_run_tiles; PAPER.md:370-389,
 * 550-571) and a per-operation verification entry (hp_stage_run).
 *
 * Conventions (all entry points):
 *  - No C++ exception crosses the ABI.  Every call returns an hp_status.
 *  - Pointers documented "device" are CUDA device memory of the context's device; "host"
 *    pointers are host memory (pinned where stated).  The CALLER owns every image, label
 *    and table buffer; the context owns scratch sized at creation (max_width x max_height
 *    x n_slots), lookup tables, streams and graphs.  Hot calls never allocate.
 *  - Tile calls are asynchronous on the given stream (NULL = legacy default stream);
 *    outputs are valid once the stream has completed.  Counts (n_objects, n_rows) stay on
 *    the device, so no host synchronisation happens inside a tile.
 *  - A slot has at most one call in flight; the caller serialises per slot (the paper's
 *    "window").  Different slots may run concurrently on different streams.
 *  - Arguments are validated before any launch -> HP_ERR_INVALID.  A CUDA error ->
 *    HP_ERR_CUDA and the context is poisoned (every later call returns HP_ERR_CUDA).  More
 *    objects than a table holds -> HP_ERR_CAPACITY is NOT detectable without a host sync:
 *    the count is always written, rows beyond capacity are dropped, and hp_run_tiles
 *    reports HP_ERR_CAPACITY per tile.  On such a tile WHICH rows are kept is unspecified
 *    (the first objects to finish, not the lowest labels); the kept rows are still complete,
 *    correct and in ascending label order.  Size max_objects for the workload (a 4K tile of
 *    the synthetic recipe has ~2,000 objects) and treat HP_ERR_CAPACITY as a failed tile.
 *  - Images are row-major.  Internal planes and the per-stage I/O of hp_stage_run are dense
 *    (pitch = width elements).
 */
#ifndef HP_H
#define HP_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

struct CUstream_st;                       /* = cudaStream_t, without the CUDA headers */
typedef struct CUstream_st* hp_stream;

typedef enum {
    HP_OK = 0,
    HP_ERR_INVALID = 1,     /* bad argument or parameter; nothing was launched */
    HP_ERR_CUDA = 2,        /* CUDA runtime error; the context is poisoned */
    HP_ERR_NOMEM = 3,       /* device or pinned allocation failed at create time */
    HP_ERR_CAPACITY = 4,    /* more objects than the table capacity (count still written) */
    HP_ERR_UNSUPPORTED = 5  /* device is not sm_100 (B200) */
} hp_status;

/* Per-pixel flag bits of S1 (plane 'flags'). */
enum { HP_FLAG_RBC_HI = 1, HP_FLAG_RBC_LO = 2, HP_FLAG_R_GT_B = 4, HP_FLAG_BG = 8 };
/* Per-object flag bits of S11. */
enum { HP_OBJ_TOUCHES_BORDER = 1 };
/* Columns of a feature row (DESIGN.md "Feature table" gives the definitions). */
enum {
    HP_F_AREA = 0, HP_F_PERIMETER, HP_F_CENTROID_X, HP_F_CENTROID_Y, HP_F_BBOX_W, HP_F_BBOX_H,
    HP_F_MAJOR, HP_F_MINOR, HP_F_ECCENTRICITY, HP_F_ORIENTATION, HP_F_EQDIAM, HP_F_COMPACTNESS,
    HP_F_EXTENT,                                                           /* shape: 13 */
    HP_F_INT_MEAN, HP_F_INT_STD, HP_F_INT_MIN, HP_F_INT_MAX, HP_F_INT_MEDIAN, HP_F_INT_SKEW,
    HP_F_INT_KURT, HP_F_INT_ENTROPY, HP_F_INT_ENERGY,                      /* intensity: 9 */
    HP_F_GRAD_MEAN, HP_F_GRAD_STD, HP_F_GRAD_SKEW, HP_F_GRAD_KURT,          /* gradient: 4 */
    HP_F_GLCM_ASM, HP_F_GLCM_CONTRAST, HP_F_GLCM_CORRELATION, HP_F_GLCM_HOMOGENEITY,
    HP_F_GLCM_ENTROPY, HP_F_GLCM_SHADE, HP_F_GLCM_PROMINENCE, HP_F_GLCM_MAXPROB, /* Haralick: 8 */
    HP_F_EDGE_COUNT, HP_F_EDGE_FRAC,                                       /* edge (Canny): 2 */
    HP_NFEAT = 36
};

/* Every constant of the method (readings C3-C12 of DESIGN.md; defaults from
 * hp_default_params).  The layout is part of the ABI. */
typedef struct hp_params {
    float   q[3][3];        /* q[k][j]: optical density of channel k (R,G,B) -> stain j
                               (H, E, residual); c_j = sum_k OD_k q[k][j] */
    float   g_scale;        /* g = clamp(rint(g_scale * c_H), 0, 255); default 170 */
    int32_t bg_rgb_min;     /* flag BG iff min(R,G,B) > bg_rgb_min; default 220 */
    float   bg_skip_frac;   /* tile skipped (0 objects) iff BG count >= frac * N; > 1 = off
                               (default 2.0).  When on, hp_segment_tile syncs its stream once. */
    int32_t rbc_t1, rbc_t2; /* RBC_HI iff R > t1*G, RBC_LO iff R > t2*G (defaults 5, 4) */
    int32_t open_diam;      /* odd in [1, 63]; OpenCV MORPH_ELLIPSE diam x diam (default 19,
                               "a 19x19 disk") */
    int32_t g1;             /* candidate iff g - recon > g1 (default 50) */
    int32_t cand_min_area, cand_max_area;  /* S5 inclusive area bounds (11, 1000); max <= 131072 */
    float   h;              /* h-maxima height on the distance map, > 0 (default 1.0) */
    int32_t obj_min_area, obj_max_area;    /* S10 inclusive area bounds (21, 1000); max <= 131072
                                              (keeps S11's exact int64 moment sums in range) */
    int32_t glcm_levels;    /* must be 8 (q = g >> 5) */
    int32_t canny_low, canny_high;  /* Canny hysteresis thresholds on the L1 3x3-Sobel magnitude
                                       of g, 0 <= low <= high (defaults 100, 200; PAPER.md:604,
                                       639 "OpenCV(Canny)"; reading C22) */
} hp_params;

typedef struct hp_config {
    int32_t   device;       /* CUDA device ordinal */
    int32_t   max_width;    /* largest tile width  (>= 1, <= 16384) */
    int32_t   max_height;   /* largest tile height (>= 1, <= 16384) */
    int32_t   n_slots;      /* independent in-flight tiles (>= 1, <= 64) */
    int32_t   max_objects;  /* feature-table rows per tile (>= 1) */
    hp_params params;
} hp_config;

/* RGB u8, channels interleaved R,G,B; pitch_bytes >= 3*width.  Device or host per call. */
typedef struct hp_image {
    const uint8_t* data;
    int32_t        width, height;
    int64_t        pitch_bytes;
} hp_image;

/* Output of segmentation (S10): labels[y*pitch + x] = 1 + min linear index (y*width + x)
 * of the pixel's object, 0 = background.  Device memory. */
typedef struct hp_labels {
    int32_t* labels;
    int64_t  labels_pitch_elems;  /* >= width */
    int32_t* n_objects_dev;       /* one int32 (device) */
} hp_labels;

/* Output of feature computation (S11): rows in ascending label order.  Device memory. */
typedef struct hp_feature_table {
    int32_t* label;       /* [capacity] */
    int32_t* flags;       /* [capacity] HP_OBJ_* bits */
    float*   feat;        /* [capacity][HP_NFEAT] row-major */
    int32_t  capacity;
    int32_t* n_rows_dev;  /* one int32 (device): number of objects (may exceed capacity) */
} hp_feature_table;

typedef struct hp_ctx hp_ctx;

void        hp_default_params(hp_params* out);
hp_status   hp_ctx_create(const hp_config* cfg, hp_ctx** out);
hp_status   hp_ctx_destroy(hp_ctx* ctx);
const char* hp_status_str(hp_status st);
const char* hp_last_error(const hp_ctx* ctx);   /* ctx-local message, never NULL */
int32_t     hp_version(void);                   /* ABI version, currently 2 (2: hp_result_sink.arena) */

/* Segmentation stage (S1..S10) of one tile.  rgb: device image.  out: device labels. */
hp_status hp_segment_tile(hp_ctx* ctx, int32_t slot, const hp_image* rgb, hp_labels* out,
                          hp_stream s);
/* Feature stage (S11) of one tile: recomputes g (S1) from rgb, then the per-object rows of
 * the objects in lab.  rgb: device image; lab: device labels as produced by
 * hp_segment_tile; out: device table. */
hp_status hp_features_tile(hp_ctx* ctx, int32_t slot, const hp_image* rgb,
                           const hp_labels* lab, hp_feature_table* out, hp_stream s);
/* Both stages with the intermediate g shared (the hot path bench.py times). */
hp_status hp_process_tile(hp_ctx* ctx, int32_t slot, const hp_image* rgb, hp_labels* lab,
                          hp_feature_table* out, hp_stream s);

/* Demand-driven multi-tile driver (PAPER.md:370-389 window dispatch; 550-571 upload /
 * process / download overlap).  next() returns 0 and fills a HOST pointer to a pinned RGB
 * tile of exactly (width, height) with the given pitch and its id, or 1 when drained.
 * For each tile, done() is called (on the calling thread) with the tile's rows in HOST
 * memory owned by the context and valid only during the callback (n_rows <= max_objects
 * rows; st = HP_ERR_CAPACITY if the tile had more).  Up to n_slots tiles are in flight;
 * each slot runs H2D -> process -> D2H on its own stream.  Blocks until drained.  Errors: a
 * NULL source/sink/callback or a size outside the context -> HP_ERR_INVALID before any work;
 * a tile with a NULL pointer or pitch < 3*width -> HP_ERR_INVALID after the tiles already
 * in flight have completed (they are not delivered). */
typedef struct hp_tile_source {
    int   (*next)(void* user, const uint8_t** host_rgb, int64_t* pitch_bytes, int64_t* tile_id);
    void*   user;
    int32_t width, height;
} hp_tile_source;
/* Device row arena (S12, PAPER.md:566-571 download phase; SURVEY §8(a) S12 "feature rows
 * are appended to the device arena, or D2H per tile").  All pointers are DEVICE memory
 * owned by the caller.  Each tile's rows (at most max_objects, in label order) are appended
 * as one contiguous run at *cursor (reserved with one device atomic), with the tile id in
 * tile[].  Runs of different tiles land in completion order, so a caller that needs a
 * fixed order sorts by (tile, label).  cursor: one int64, caller-initialised (normally 0);
 * it ends at the number of rows offered, which may exceed capacity -- rows past capacity are
 * dropped and their tile is reported with HP_ERR_CAPACITY. */
typedef struct hp_row_arena {
    int64_t* tile;        /* [capacity] tile id of each row */
    int32_t* label;       /* [capacity] */
    int32_t* flags;       /* [capacity] HP_OBJ_* bits */
    float*   feat;        /* [capacity][HP_NFEAT] row-major */
    int64_t  capacity;
    int64_t* cursor;      /* one int64 (device): append position */
} hp_row_arena;
/* arena == NULL: rows are copied to the host per tile and done() receives them.  arena !=
 * NULL: rows stay on the device (appended to the arena); done() receives n_rows and NULL row
 * pointers, and only 12 bytes per tile (row count, arena offset) cross PCIe. */
typedef struct hp_result_sink {
    void (*done)(void* user, int64_t tile_id, int32_t n_rows, const int32_t* label,
                 const int32_t* flags, const float* feat, hp_status st);
    void* user;
    const hp_row_arena* arena;  /* ABI version 2 */
} hp_result_sink;
hp_status hp_run_tiles(hp_ctx* ctx, const hp_tile_source* src, const hp_result_sink* sink);

/* Compressed ingest ("the main limiting factor and bottleneck
 * is the I/O overhead of reading image tiles", 716-726).  Tiles arrive as baseline JPEG files
 * (ITU-T T.81 sequential Huffman, 8-bit, 3 components, 4:4:4 or 4:2:0 sampling (the 4:2:0
 * chroma upsampled by the IJG triangle filter, reading J4), one interleaved scan;
 * a restart interval (DRI) lets the GPU decode one interval per thread -- without one the
 * whole scan is a single serial interval).  Only the file crosses PCIe (~4 MB instead of
 * 50 MB for a quality-90 4K tile).  The host parses the marker segments (a few hundred
 * bytes); restart-marker search, Huffman decoding, dequantisation, the IDCT (the IJG "islow"
 * integer method, reading J1 of DESIGN.md) and the JFIF YCbCr->RGB conversion (reading J2)
 * run on the GPU, fused into S1: the decoded RGB tile is never written to memory.  The
 * result equals hp_process_tile on the tile cv2.imdecode would return.
 * Errors: a file outside that scope -> HP_ERR_UNSUPPORTED; a malformed header, a file larger
 * than 3 * max_width * max_height bytes or a frame larger than the context -> HP_ERR_INVALID
 * (both before any launch).  A corrupt scan (restart markers not matching the interval, an
 * invalid Huffman code) is only seen on the device: it sets the decode error word.
 *
 * hp_run_tiles_jpeg: hp_run_tiles with next() returning a HOST pointer to a JPEG file and its
 * size in bytes (pinned memory recommended; valid until the tile is delivered).  Every file
 * must decode to exactly (width, height).  A file that fails on the host, or whose scan is
 * corrupt, is delivered through done() with HP_ERR_INVALID / HP_ERR_UNSUPPORTED and no rows;
 * the run continues with the next tile.  (With a row arena, a corrupt-scan tile's run has
 * already been appended on the device when its status arrives: drop it by tile id.) */
typedef struct hp_jpeg_source {
    int   (*next)(void* user, const uint8_t** host_jpeg, int64_t* nbytes, int64_t* tile_id);
    void*   user;
    int32_t width, height;
} hp_jpeg_source;
hp_status hp_run_tiles_jpeg(hp_ctx* ctx, const hp_jpeg_source* src, const hp_result_sink* sink);
/* One JPEG tile through both stages, like hp_process_tile: host_jpeg (HOST, nbytes; keep it
 * valid until s completes) is uploaded on s.  decode_err_dev (DEVICE int32, may be NULL)
 * receives 0, or 1 (restart-marker mismatch) | 2 (invalid Huffman code). */
hp_status hp_process_tile_jpeg(hp_ctx* ctx, int32_t slot, const uint8_t* host_jpeg, int64_t nbytes,
                               hp_labels* lab, hp_feature_table* out, int32_t* decode_err_dev,
                               hp_stream s);
/* Host-only header probe (no context, no GPU): the frame size, sampling (444 or 420), the
 * restart interval in MCUs (0 = none) and the number of restart intervals of a JPEG file, or
 * HP_ERR_UNSUPPORTED / HP_ERR_INVALID as the JPEG calls would report it.  sampling,
 * restart_interval and n_intervals may be NULL. */
hp_status hp_jpeg_info(const uint8_t* host_jpeg, int64_t nbytes, int32_t* width, int32_t* height,
                       int32_t* sampling, int32_t* restart_interval, int32_t* n_intervals);
/* Verification entry of the decoder alone: the decoded RGB tile (DEVICE rgb_dev, u8 R,G,B
 * interleaved, pitch_bytes >= 3*width).  Synchronises s; a corrupt scan -> HP_ERR_INVALID. */
hp_status hp_decode_jpeg(hp_ctx* ctx, int32_t slot, const uint8_t* host_jpeg, int64_t nbytes,
                         uint8_t* rgb_dev, int64_t pitch_bytes, hp_stream s);

/* Verification ABI: run ONE operation on caller-provided DEVICE buffers (dense planes of
 * width x height).  Layouts per stage (in -> out):
 *  CD        in0 rgb u8x3 (pitch 3w)            -> out0 g u8, out1 flags u8, out2 bg count i64[1]
 *  RBC       in0 flags u8                       -> out0 rbc u8 (0/1)
 *  OPEN      in0 g u8                           -> out0 open u8
 *  RECON     in0 g u8, in1 open u8, in2 rbc u8  -> out0 cand u8 (0/1), out1 recon u8
 *  AREA      in0 cand u8                        -> out0 big0 u8 (0/1)
 *  FILL      in0 big0 u8                        -> out0 F u8 (0/1)
 *  EDT       in0 F u8                           -> out0 d2 u32, out1 dist f32
 *  MARKERS   in0 dist f32, in1 F u8             -> out0 ML i32, out1 J f32 (0 outside F)
 *  WATERSHED in0 dist f32, in1 ML i32, in2 F u8 -> out0 split u8, out1 c f32, out2 d i32,
 *                                                  out3 L i32 (c, d, L: 0 outside F)
 *  BWLABEL   in0 split u8                       -> out0 labels i32, out1 n_objects i32[1]
 *  FEATURES  in0 labels i32, in1 g u8           -> out0 label i32[cap], out1 flags i32[cap],
 *                                                  out2 feat f32[cap][36], out3 n_rows i32[1]
 *                                                  (cap = max_objects)
 *  IWPP_RAW  in0 marker u8, in1 mask u8         -> out0 recon u8, out1 stats i64[4]
 *                                                  (jobs, sweep iterations, ns regions were
 *                                                  owned, row closures attempted)
 *  CCL8/CCL4 in0 fg u8                          -> out0 labels i32 (1 + min index, 0 = bg)
 *  RECON_F32 in0 marker f32, in1 mask f32, in2 domain u8 (may be NULL) -> out0 recon f32
 *  CANNY     in0 g u8                           -> out0 edges u8 (0/1): cv2.Canny(g, low, high)
 * The whole-plane AREA .. BWLABEL kernels above are verification kernels; the pipeline runs
 * these three instead, exposed here so each hot-path kernel can be fed the oracle's input:
 *  AREA_TOPHAT in0 g u8, in1 recon u8, in2 rbc u8 -> out0 big0 u8 (0/1) = S5 of the S4
 *                                                  candidates ((g - recon) > g1) & !rbc, the
 *                                                  candidate test evaluated inside S5's CCL;
 *                                                  out1 (optional) i32[1] components kept
 *  FILL_COMP   in0 big0 u8                      -> out0 F u8 (0/1): S6 solved per 8-component
 *                                                  of big0 in its window (k_fill_fused)
 *  COMPONENTS  in0 F u8 (S6 output), in1 g u8   -> S7-S11 solved per 8-component of F
 *                                                  (k_comp_fused): out0 labels i32 (S10),
 *                                                  out1 n_objects i32[1], out2 i32[2][cap]
 *                                                  (row labels, then row flags), out3 feat
 *                                                  f32[cap][36]; cap = max_objects, rows in
 *                                                  ascending label order
 */
typedef enum {
    HP_STAGE_CD = 0, HP_STAGE_RBC, HP_STAGE_OPEN, HP_STAGE_RECON, HP_STAGE_AREA,
    HP_STAGE_FILL, HP_STAGE_EDT, HP_STAGE_MARKERS, HP_STAGE_WATERSHED, HP_STAGE_BWLABEL,
    HP_STAGE_FEATURES, HP_STAGE_IWPP_RAW, HP_STAGE_CCL8, HP_STAGE_CCL4, HP_STAGE_RECON_F32,
    HP_STAGE_CANNY, HP_STAGE_AREA_TOPHAT, HP_STAGE_FILL_COMP, HP_STAGE_COMPONENTS, HP_STAGE_COUNT
} hp_stage;
typedef struct hp_stage_io {
    const void* in[4];
    void*       out[4];
    int32_t     width, height;
} hp_stage_io;
hp_status hp_stage_run(hp_ctx* ctx, int32_t slot, hp_stage st, const hp_stage_io* io,
                       hp_stream s);

/* Per-stage timing, recorded with CUDA events on the tile's stream when enabled (off by
 * default).  Each segment/process call on a slot uses the next of 256 event sets per slot.
 * hp_get_stage_times: S1..S11 milliseconds of the slot's last tile (synchronises on it).
 * hp_stage_times_accum: sums over every tile recorded since the last accumulation or
 * enable (up to 256 per slot), writes the number of tiles to *count, and resets. */
hp_status hp_set_stage_timing(hp_ctx* ctx, int32_t enable);
hp_status hp_get_stage_times(hp_ctx* ctx, int32_t slot, float* ms11);
hp_status hp_stage_times_accum(hp_ctx* ctx, float* ms11, int32_t* count);
/* Number of libhp kernel launches issued by this process so far (diagnostics). */
int64_t   hp_launch_count(void);

/* Per-image feature aggregation (the object features of an
 * image feed the image-level classification stage).  Segmented reduction of feature rows on
 * the device: rows [off[g], off[g+1]) of feat (DEVICE, [n_rows][HP_NFEAT] f32, row-major)
 * form group g (e.g. one slide); out (DEVICE, [n_groups][HP_NFEAT][2] f64) receives per group
 * and feature the sum and the sum of squares, out_count (DEVICE, i64[n_groups]) the number of
 * rows.  off: DEVICE i64[n_groups + 1], non-decreasing.  Every thread reduces a fixed set of
 * rows and the per-group tree has a fixed shape, so the result is bit-identical run to run.
 * Async on s; HP_ERR_INVALID on null pointers or n_groups < 0 (feat may be NULL when every
 * group is empty: a rank that holds no rows).  Across GPUs the callers sum the outputs with
 * an all-reduce (paper_1209_3332_b200/dist.py aggregate_groups). */
hp_status hp_reduce_rows(hp_ctx* ctx, const float* feat, const int64_t* off, int32_t n_groups,
                         double* out, int64_t* out_count, hp_stream s);
/* Second pass of the per-group mean / standard deviation (two-pass, so the variance is never
 * formed as E[x^2] - mean^2).  sums (DEVICE, [n_groups][HP_NFEAT][2] f64, the layout of
 * hp_reduce_rows' out; only the sums [..][0] are read) and count (DEVICE, i64[n_groups]) are
 * the TOTALS over every rank (after an all-reduce of hp_reduce_rows' outputs).  mean_m2
 * (DEVICE, [n_groups][HP_NFEAT][2] f64) receives (mean = sum / count, NaN for an empty group;
 * m2 = sum over THIS caller's rows [off[g], off[g+1]) of (x - mean)^2).  Callers all-reduce
 * m2 (it is additive over ranks) and finish with hp_group_std.  feat may be NULL when every
 * group is empty.  Deterministic (fixed row ownership and tree); async on s. */
hp_status hp_group_center(hp_ctx* ctx, const float* feat, const int64_t* off, int32_t n_groups,
                          const double* sums, const int64_t* count, double* mean_m2, hp_stream s);
/* mean[g][f] = mean_m2[g][f][0]; std[g][f] = sqrt(m2 / count) (population), NaN for an
 * empty group.  All DEVICE: mean_m2 [n_groups][HP_NFEAT][2] f64, count i64[n_groups], mean and
 * std [n_groups][HP_NFEAT] f64.  Async on s. */
hp_status hp_group_std(hp_ctx* ctx, const double* mean_m2, const int64_t* count, int32_t n_groups,
                       double* mean, double* std_out, hp_stream s);

#ifdef __cplusplus
}
#endif
#endif /* HP_H */
