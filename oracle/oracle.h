/* oracle.h -- plain, slow, obviously-correct CPU oracle of the per-tile pipeline.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load liboracle.  The product path
 * (libhp, include/hp.h) shares no code, header, table or constant generator with it.
 *
 * Every function follows one step of SURVEY.md §8(c) "Oracle", which restates the
 * paper's operation list (Table I) with the readings C1-C20 that
 * DESIGN.md lists.  Images are row-major, dense (pitch = width) unless stated.
 * All functions return 0 on success, 1 on invalid arguments, 3 on allocation failure.
 * Single-threaded; compiled with g++ -O2 -ffp-contract=off (no FMA contraction;
 * where the definition says fma, std::fma is called explicitly).
 */
#ifndef ORACLE_H
#define ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Same field meaning as hp_params (include/hp.h) -- declared independently. */
typedef struct or_params {
    float   q[3][3];        /* q[k][j]: OD channel k (R,G,B) -> stain j (H,E,residual) */
    float   g_scale;        /* g = clamp(rint(g_scale * c_H), 0, 255) */
    int32_t bg_rgb_min;     /* BG flag: min(R,G,B) > bg_rgb_min */
    float   bg_skip_frac;   /* >1 disables the background-tile skip */
    int32_t rbc_t1, rbc_t2; /* RBC_HI: R > t1*G ; RBC_LO: R > t2*G */
    int32_t open_diam;      /* odd, structuring element = OpenCV MORPH_ELLIPSE diam x diam */
    int32_t g1;             /* top-hat threshold: cand = (g - recon) > g1 */
    int32_t cand_min_area, cand_max_area;
    float   h;              /* h-maxima height on the distance map */
    int32_t obj_min_area, obj_max_area;
    int32_t glcm_levels;    /* 8 */
    int32_t canny_low, canny_high;  /* Canny hysteresis thresholds on the L1 Sobel magnitude */
} or_params;

enum { OR_FLAG_RBC_HI = 1, OR_FLAG_RBC_LO = 2, OR_FLAG_R_GT_B = 4, OR_FLAG_BG = 8 };
enum { OR_OBJ_TOUCHES_BORDER = 1 };
enum { OR_NFEAT = 36 };

/* Defaults; q is computed here in double from the Ruifrok-Johnston H&E vectors. */
void or_default_params(or_params* p);

/* S1: colour deconvolution + flags.  rgb: u8 interleaved R,G,B with pitch (bytes). */
int or_cd(const uint8_t* rgb, int w, int h, int64_t pitch, const or_params* p,
          uint8_t* g, uint8_t* flags, int64_t* bg_count);
/* S2: rbc = BinRecon8(RBC_HI, RBC_LO) & R_GT_B; values 0/1. */
int or_rbc(const uint8_t* flags, int w, int h, uint8_t* rbc);
/* S3: open = dilate_D(erode_D(g)), D = OpenCV ellipse diam x diam, OOB ignored. */
int or_open(const uint8_t* g, int w, int h, int diam, uint8_t* out);
/* Brute-force erode/dilate with the same D (exposed for pins). */
int or_erode(const uint8_t* g, int w, int h, int diam, uint8_t* out);
int or_dilate(const uint8_t* g, int w, int h, int diam, uint8_t* out);
/* Grayscale reconstruction by dilation, 8-connected, Vincent's hybrid algorithm:
 * recon of min(marker, mask) under mask.  Stats (optional, may be NULL):
 * stats[0] = initial queue length, stats[1] = FIFO pops. */
int or_recon_u8(const uint8_t* marker, const uint8_t* mask, int w, int h,
                uint8_t* out, int64_t* stats);
/* Float version restricted to a domain (dom[p] != 0; dom may be NULL = all). */
int or_recon_f32(const float* marker, const float* mask, const uint8_t* dom, int w, int h,
                 float* out);
/* S4: recon = GrayRecon8(open, g); cand = ((g - recon) > g1) & !rbc. recon optional out. */
int or_recon_to_nuclei(const uint8_t* g, const uint8_t* open, const uint8_t* rbc, int w, int h,
                       int g1, uint8_t* cand, uint8_t* recon_out);
/* CCL: labels[p] = 1 + min linear index of p's component (0 = background).
 * conn = 4 or 8.  Returns the number of components in *n. */
int or_ccl(const uint8_t* fg, int w, int h, int conn, int32_t* labels, int32_t* n);
/* S5: keep 8-components of cand with amin <= area <= amax; out 0/1. */
int or_area_threshold(const uint8_t* cand, int w, int h, int amin, int amax, uint8_t* out);
/* S6: F = big0 | holes, holes = 4-components of !big0 without a tile-border pixel. */
int or_fill_holes(const uint8_t* big0, int w, int h, uint8_t* F);
/* S7: exact squared EDT (Meijster), d2 = 0 on background, UINT32_MAX everywhere if the
 * tile has no background; dist = sqrtf((float)d2) (+inf for the no-background case). */
int or_edt(const uint8_t* F, int w, int h, uint32_t* d2, float* dist);
/* S8: J = GrayRecon8_f32(dist - hh, dist) on F; M = RMAX8(J) & F; ML = CCL8(M) labels.
 * J (optional) receives J (0 outside F). n_markers optional. */
int or_markers(const float* dist, const uint8_t* F, int w, int h, float hh,
               int32_t* ML, float* J, int32_t* n_markers);
/* S9: W1 c, W2 d, W3 L, lines, split (0/1).  c/d/L optional (may be NULL). */
int or_watershed(const float* dist, const int32_t* ML, const uint8_t* F, int w, int h,
                 float* c, int32_t* d, int32_t* L, uint8_t* split);
/* S10: CCL8 of split, area filter, labels = 1 + min index, else 0. */
int or_bwlabel(const uint8_t* split, int w, int h, int amin, int amax,
               int32_t* labels, int32_t* n_objects);
/* Feature-stage Canny: cv2.Canny(g, low, high) (aperture 3, L1 norm); edges 0/1. */
int or_canny(const uint8_t* g, int w, int h, int low, int high, uint8_t* edges);
/* S11: one row per object in ascending label order: label, flags, feat[OR_NFEAT].
 * Returns 4 if more than cap objects (n_rows still written). */
int or_features(const int32_t* labels, const uint8_t* g, int w, int h, int glcm_levels,
                int canny_low, int canny_high, int32_t cap, int32_t* row_label,
                int32_t* row_flags, float* feat, int32_t* n_rows);
/* S1..S10 composed; optional per-stage seconds (11 doubles, S1..S11 order) in t_stage. */
int or_segment_tile(const uint8_t* rgb, int w, int h, int64_t pitch, const or_params* p,
                    int32_t* labels, int32_t* n_objects, double* t_stage);
/* Segmentation + features (the whole per-tile hot path). */
int or_process_tile(const uint8_t* rgb, int w, int h, int64_t pitch, const or_params* p,
                    int32_t* labels, int32_t cap, int32_t* row_label, int32_t* row_flags,
                    float* feat, int32_t* n_rows, double* t_stage);
/* NEXT-4 per-image aggregation: per group g (rows [off[g], off[g+1]) of feat [n][nfeat]),
 * count[g], mean[g][f] and population std[g][f] in fp64 (two-pass); NaN for an empty group. */
int or_aggregate(const float* feat, int nfeat, const int64_t* off, int n_groups, int64_t* count,
                 double* mean, double* stdv);
/* NEXT-3 compressed ingest (oracle/jpeg.cpp): baseline JPEG (T.81 sequential Huffman,
 * 8-bit, 3 components at 1x1 sampling, optional restart interval) -> RGB u8 interleaved,
 * pitch 3*width.  rgb == NULL: only *width / *height are written.  Returns 0, 1 (invalid
 * stream) or 5 (a JPEG feature outside that scope). */
int or_jpeg_decode(const uint8_t* data, int64_t n, int32_t* width, int32_t* height, uint8_t* rgb);

#ifdef __cplusplus
}
#endif
#endif
